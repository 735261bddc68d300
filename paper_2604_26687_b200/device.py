"""Device (B200) GNS path: Python handles over the C-ABI of include/coadapt_cuda.h.

``BucketPlan`` compiles a rank's gradient-bucket layout (segments with dedup
weights); ``GnsDevice`` is the device-resident StepAccumulator + GnsState of
one optimizer step (gns.hpp:15-73): squared-norm reductions accumulate into
its N+1 fp64 slots, ``allreduce`` sums the slots over ranks with NCCL, and
``finalize`` runs finalize_step + update_ema + gns in a device kernel.
Tensors are passed by pointer; PyTorch is used only for memory and streams.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from ._lib import GnsResult, GnsState, check, lib

TORCH_TO_DTYPE = {torch.bfloat16: L.BF16, torch.float16: L.FP16, torch.float32: L.FP32,
                  torch.float64: L.FP64}
DTYPE_TO_TORCH = {v: k for k, v in TORCH_TO_DTYPE.items()}
ESIZE = {L.BF16: 2, L.FP16: 2, L.FP32: 4, L.FP64: 8}


def _ptr(x) -> int:
    if isinstance(x, torch.Tensor):
        return x.data_ptr()
    return int(x)


def _bucket(plan: "BucketPlan", x, what: str = "bucket", host: bool = False) -> int:
    """Pointer of a bucket for `plan`, validated when it is a tensor: the
    plan's dtype, contiguous, at least bucket_numel elements, on the plan's
    GPU (host=False) or in host memory (host=True).  Raw addresses (ints,
    e.g. CUDA-IPC peer pointers) are the caller's responsibility."""
    if isinstance(x, torch.Tensor):
        want = DTYPE_TO_TORCH[plan.dtype]
        if x.dtype != want:
            raise L.ValidationError(f"{what}: dtype {x.dtype}, the plan is {want}")
        if not x.is_contiguous():
            raise L.ValidationError(f"{what}: not contiguous")
        if x.numel() < plan.bucket_numel:
            raise L.ValidationError(f"{what}: {x.numel()} elements < the plan's bucket_numel "
                                    f"{plan.bucket_numel}")
        if host:
            if x.is_cuda:
                raise L.ValidationError(f"{what}: expected host memory, got {x.device}")
        elif not x.is_cuda or x.device.index != plan.device:
            raise L.ValidationError(f"{what}: on {x.device}, the plan is on cuda:{plan.device}")
        return x.data_ptr()
    if host and hasattr(x, "ctypes"):
        if x.size < plan.bucket_numel or x.itemsize != ESIZE[plan.dtype]:
            raise L.ValidationError(f"{what}: host array smaller than the plan or wrong element size")
        return x.ctypes.data
    return int(x)


def _host_ptr(x) -> int:
    if isinstance(x, torch.Tensor):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    return int(x)


def _stream(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _seg_array(segments) -> tuple:
    segs = list(segments)
    arr = (L.Segment * max(1, len(segs)))(*[L.Segment(int(o), int(n), float(w)) for o, n, w in segs])
    return arr, len(segs)


def _gen_array(gsegs) -> tuple:
    gs = list(gsegs)
    arr = (L.GenSegment * max(1, len(gs)))(*[L.GenSegment(*map(int, g)) for g in gs])
    return arr, len(gs)


class BucketPlan:
    """A rank's flattened bucket layout: [(offset, numel, weight)] in elements."""

    def __init__(self, segments, bucket_numel: int, dtype: int, device: int = 0,
                 slice_index: Optional[int] = None, slice_count: Optional[int] = None):
        arr, n = _seg_array(segments)
        h = C.c_void_p()
        if slice_count is None:
            check(lib().coadapt_plan_create(arr, n, int(bucket_numel), int(dtype), int(device), C.byref(h)))
        else:
            check(lib().coadapt_plan_create_slice(arr, n, int(bucket_numel), int(dtype), int(device),
                                                  int(slice_index), int(slice_count), C.byref(h)))
        self.handle = h
        self.dtype = int(dtype)
        self.bucket_numel = int(bucket_numel)
        self.device = int(device)

    @property
    def active_elements(self) -> int:
        a, r = C.c_uint64(), C.c_uint64()
        check(lib().coadapt_plan_info(self.handle, C.byref(a), C.byref(r)))
        return a.value

    @property
    def num_ranges(self) -> int:
        a, r = C.c_uint64(), C.c_uint64()
        check(lib().coadapt_plan_info(self.handle, C.byref(a), C.byref(r)))
        return r.value

    @property
    def active_bytes(self) -> int:
        return self.active_elements * ESIZE[self.dtype]

    def close(self):
        if getattr(self, "handle", None):
            lib().coadapt_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GnsDevice:
    """Device StepAccumulator (gns.hpp:15-32) + GnsState (gns.hpp:53-62)."""

    def __init__(self, dp_size: int, micro_count: int, global_batch: int, device: int = 0):
        h = C.c_void_p()
        check(lib().coadapt_gns_create(int(dp_size), int(micro_count), int(global_batch), int(device),
                                       C.byref(h)))
        self.handle = h
        self.dp_size, self.micro_count, self.global_batch = int(dp_size), int(micro_count), int(global_batch)
        self.device = int(device)

    @property
    def n(self) -> int:
        return self.dp_size * self.micro_count

    def reshape(self, dp_size: int, micro_count: int, global_batch: int) -> None:
        check(lib().coadapt_gns_reshape(self.handle, int(dp_size), int(micro_count), int(global_batch)))
        self.dp_size, self.micro_count, self.global_batch = int(dp_size), int(micro_count), int(global_batch)

    def begin_step(self, stream=None) -> None:
        check(lib().coadapt_gns_begin_step(self.handle, _stream(stream)))

    def micro_sqnorm(self, plan: BucketPlan, bucket, dp_index: int, micro: int, stream=None) -> None:
        check(lib().coadapt_gns_micro_sqnorm(self.handle, plan.handle, _bucket(plan, bucket), int(dp_index),
                                             int(micro), _stream(stream)))

    def micro_sqnorm_batched(self, plan: BucketPlan, buckets: Sequence, dp_index: Sequence[int],
                             micro: Sequence[int], stream=None) -> None:
        k = len(buckets)
        ptrs = (C.c_void_p * max(1, k))(*[_bucket(plan, b) for b in buckets])
        di = (C.c_int32 * max(1, k))(*dp_index)
        mi = (C.c_int32 * max(1, k))(*micro)
        check(lib().coadapt_gns_micro_sqnorm_batched(self.handle, plan.handle, ptrs, di, mi, k,
                                                     _stream(stream)))

    def fused_sqnorm(self, plan: BucketPlan, buckets: Sequence, stream=None) -> None:
        k = len(buckets)
        ptrs = (C.c_void_p * max(1, k))(*[_bucket(plan, b) for b in buckets])
        check(lib().coadapt_gns_fused_sqnorm(self.handle, plan.handle, ptrs, k, _stream(stream)))

    def fused_sqnorm_finalize(self, plan: BucketPlan, buckets: Sequence, tokens_this_step: int,
                              stream=None) -> None:
        """The step's last fused pass with finalize (and, with mailboxes
        attached, the NVLink slot exchange) in its last CTA."""
        k = len(buckets)
        ptrs = (C.c_void_p * max(1, k))(*[_bucket(plan, b) for b in buckets])
        check(lib().coadapt_gns_fused_sqnorm_finalize(self.handle, plan.handle, ptrs, k,
                                                      int(tokens_this_step), _stream(stream)))

    def mean_sqnorm_finalize(self, plan: BucketPlan, mean_grad, tokens_this_step: int,
                             stream=None) -> None:
        """d > 1: the step's last mean-slice read with finalize in the pass."""
        check(lib().coadapt_gns_mean_sqnorm_finalize(self.handle, plan.handle,
                                                     _bucket(plan, mean_grad, "mean_grad"),
                                                     int(tokens_this_step), _stream(stream)))

    def fused_sqnorm_host(self, plan: BucketPlan, host_buckets: Sequence, stream=None) -> None:
        k = len(host_buckets)
        ptrs = (C.c_void_p * max(1, k))(*[_bucket(plan, b, "host bucket", host=True)
                                          for b in host_buckets])
        check(lib().coadapt_gns_fused_sqnorm_host(self.handle, plan.handle, ptrs, k, _stream(stream)))

    def micro_sqnorm_host(self, plan: BucketPlan, host_bucket, dp_index: int, micro: int,
                          stream=None) -> None:
        """K1 over a host (ideally pinned) bucket, streamed H2D."""
        check(lib().coadapt_gns_micro_sqnorm_host(self.handle, plan.handle,
                                                  _bucket(plan, host_bucket, "host bucket", host=True),
                                                  int(dp_index), int(micro), _stream(stream)))

    def mean_sqnorm_host(self, plan: BucketPlan, host_mean, stream=None) -> None:
        check(lib().coadapt_gns_mean_sqnorm_host(self.handle, plan.handle,
                                                 _bucket(plan, host_mean, "host mean", host=True),
                                                 _stream(stream)))

    ACC_FIRST, ACC_LAST_MEAN = 1, 2

    def accumulate(self, plan: BucketPlan, main_grad: torch.Tensor, micro_grad, dp_index: int,
                   micro: int, first: bool = False, last_mean: bool = False,
                   mean_scale_sq: Optional[float] = None, stream=None) -> None:
        """Trainer form: main_grad (+)= micro_grad (fp32) with s_m (and, on the
        last micro-batch of a d == 1 step, gbar^2) fused in."""
        if main_grad.dtype != torch.float32:
            raise L.ValidationError("main_grad must be fp32")
        if not main_grad.is_contiguous() or main_grad.numel() < plan.bucket_numel or \
                not main_grad.is_cuda or main_grad.device.index != plan.device:
            raise L.ValidationError("main_grad: contiguous fp32 on the plan's GPU with at least "
                                    "bucket_numel elements")
        flags = (self.ACC_FIRST if first else 0) | (self.ACC_LAST_MEAN if last_mean else 0)
        if mean_scale_sq is None:
            mean_scale_sq = 1.0 / float(self.micro_count) ** 2
        check(lib().coadapt_gns_accumulate(self.handle, plan.handle, main_grad.data_ptr(),
                                           _bucket(plan, micro_grad, "micro_grad"), int(dp_index),
                                           int(micro), flags,
                                           float(mean_scale_sq), _stream(stream)))

    def barrier(self, stream=None) -> None:
        """Stream-ordered cross-rank barrier (1-element NCCL all-reduce)."""
        check(lib().coadapt_gns_barrier(self.handle, _stream(stream)))

    def reduce_scatter_sqnorm(self, plan: BucketPlan, replicas: Sequence, dp_rank: int, out_slice,
                              scale: float, stream=None) -> None:
        """Fused DP reduce-scatter + gbar^2 over NVLink (peer pointers from
        ipc_open; the local replica by pointer)."""
        k = len(replicas)
        ptrs = (C.c_void_p * max(1, k))(*[_bucket(plan, r, "replica") for r in replicas])
        check(lib().coadapt_gns_reduce_scatter_sqnorm(self.handle, plan.handle, ptrs, k, int(dp_rank),
                                                      _ptr(out_slice), float(scale), _stream(stream)))

    def allreduce_sqnorm(self, plan: BucketPlan, replicas: Sequence, dp_rank: int, scale: float,
                         stream=None) -> None:
        """All-reduce form: the synchronised slice is written back into every
        replica (in place, peers' over NVLink) and its gbar^2 accumulated."""
        k = len(replicas)
        ptrs = (C.c_void_p * max(1, k))(*[_bucket(plan, r, "replica") for r in replicas])
        check(lib().coadapt_gns_allreduce_sqnorm(self.handle, plan.handle, ptrs, k, int(dp_rank),
                                                 float(scale), _stream(stream)))

    def nvls_reduce_sqnorm(self, plan: BucketPlan, bucket: "NvlsBucket", dp_rank: int, scale: float,
                           out_slice=None, stream=None) -> None:
        """Switch-reduced DP sync of an fp32 NVLS bucket + gbar^2 of this
        rank's slice in one pass: reduce-scatter into out_slice, or (out_slice
        None) all-reduce back into every GPU's copy."""
        check(lib().coadapt_gns_nvls_reduce_sqnorm(self.handle, plan.handle, C.c_void_p(bucket.multicast),
                                                   int(bucket.nranks), int(dp_rank),
                                                   None if out_slice is None else _ptr(out_slice),
                                                   float(scale), _stream(stream)))

    def mean_sqnorm(self, plan: BucketPlan, mean_grad, stream=None) -> None:
        check(lib().coadapt_gns_mean_sqnorm(self.handle, plan.handle, _bucket(plan, mean_grad, "mean_grad"),
                                            _stream(stream)))

    def attach_nccl(self, nranks: int, rank: int, unique_id: bytes) -> None:
        buf = C.create_string_buffer(bytes(unique_id), len(unique_id))
        check(lib().coadapt_gns_attach_nccl(self.handle, int(nranks), int(rank), buf, len(unique_id)))

    def allreduce(self, stream=None) -> None:
        check(lib().coadapt_gns_allreduce(self.handle, _stream(stream)))

    def mailbox(self, nranks: int) -> int:
        """This rank's NVLink slot-exchange mailbox (device address)."""
        ptr = C.c_void_p()
        check(lib().coadapt_gns_mailbox(self.handle, int(nranks), C.byref(ptr)))
        return int(ptr.value)

    def attach_mailboxes(self, nranks: int, rank: int, peers: Sequence[int]) -> None:
        arr = (C.c_void_p * len(peers))(*[int(x) for x in peers])
        check(lib().coadapt_gns_attach_mailboxes(self.handle, int(nranks), int(rank), arr))

    def allreduce_finalize_p2p(self, tokens_this_step: int, stream=None) -> None:
        """X1 + K3 in one kernel over NVLink (replaces allreduce + finalize)."""
        check(lib().coadapt_gns_allreduce_finalize_p2p(self.handle, int(tokens_this_step),
                                                       _stream(stream)))

    def finalize(self, tokens_this_step: int, stream=None) -> None:
        check(lib().coadapt_gns_finalize(self.handle, int(tokens_this_step), _stream(stream)))

    def result(self) -> GnsResult:
        r = GnsResult()
        check(lib().coadapt_gns_read_result(self.handle, C.byref(r)))
        return r

    def result_ready(self) -> bool:
        """Non-blocking: has the last finalize's result reached the host?"""
        ready = C.c_int(0)
        check(lib().coadapt_gns_result_ready(self.handle, C.byref(ready)))
        return bool(ready.value)

    def partials(self) -> np.ndarray:
        out = np.zeros(self.n + 1, np.float64)
        check(lib().coadapt_gns_read_partials(self.handle, out.ctypes.data, out.size))
        return out

    def get_state(self) -> GnsState:
        s = GnsState()
        check(lib().coadapt_gns_get_state(self.handle, C.byref(s)))
        return s

    def set_state(self, s: GnsState) -> None:
        check(lib().coadapt_gns_set_state(self.handle, C.byref(s)))

    def close(self):
        if getattr(self, "handle", None):
            lib().coadapt_gns_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def attach_nccl_all(gs: Sequence["GnsDevice"]) -> None:
    """One process driving len(gs) GPUs (one GnsDevice per device, rank order)."""
    arr = (C.c_void_p * len(gs))(*[g.handle.value for g in gs])
    check(lib().coadapt_gns_attach_nccl_all(arr, len(gs)))


def allreduce_group(gs: Sequence["GnsDevice"], streams: Sequence) -> None:
    arr = (C.c_void_p * len(gs))(*[g.handle.value for g in gs])
    sts = (C.c_void_p * len(gs))(*[_stream(s) for s in streams])
    check(lib().coadapt_gns_allreduce_group(arr, sts, len(gs)))


def ipc_handle(t: torch.Tensor) -> tuple:
    """(64-byte CUDA IPC handle of the allocation holding `t`, offset of
    t.data_ptr() inside it) — send both to the peer (ipc_open)."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64()
    check(lib().coadapt_ipc_handle(t.data_ptr(), buf, 64, C.byref(off)))
    return buf.raw, off.value


def ipc_handle_ptr(ptr: int) -> tuple:
    """ipc_handle for a raw device address (e.g. GnsDevice.mailbox)."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64()
    check(lib().coadapt_ipc_handle(C.c_void_p(int(ptr)), buf, 64, C.byref(off)))
    return buf.raw, off.value


def ipc_open(handle, device: int) -> tuple:
    """-> (device pointer to the peer tensor, base pointer to ipc_close)"""
    raw, off = handle
    ptr = C.c_void_p()
    hb = C.create_string_buffer(bytes(raw), len(raw))
    check(lib().coadapt_ipc_open(hb, len(raw), int(device), C.byref(ptr)))
    return int(ptr.value) + int(off), int(ptr.value)


def ipc_close(ptr: int) -> None:
    check(lib().coadapt_ipc_close(C.c_void_p(ptr)))


class _CudaArray:
    """__cuda_array_interface__ view of a raw device buffer (torch.as_tensor)."""

    def __init__(self, ptr: int, numel: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class NvlsBucket:
    """A gradient bucket in NVLS memory (coadapt_nvls_*): one physical buffer
    per GPU bound to a multicast object; ``tensor`` is this GPU's view.  The
    all-reduce is switch-reduced (multimem.ld_reduce / multimem.st).

    Collective setup — every rank of the DP group calls it with the same
    arguments and a torch.distributed group for the handle exchange."""

    _TYPESTR = {torch.float32: "<f4", torch.float16: "<f2"}

    def __init__(self, numel: int, dtype: torch.dtype, rank: int, nranks: int, dist_mod,
                 device: Optional[int] = None):
        dev = torch.cuda.current_device() if device is None else int(device)
        self.dtype, self.numel, self.rank, self.nranks, self.device = dtype, int(numel), rank, nranks, dev
        es = torch.empty((), dtype=dtype).element_size()
        nbytes = (self.numel * es + 15) // 16 * 16
        self.handle = C.c_void_p()
        if rank == 0:
            check(lib().coadapt_nvls_create(dev, nranks, nbytes, C.byref(self.handle)))
            buf = C.create_string_buffer(64)
            check(lib().coadapt_nvls_export(self.handle, buf, 64))
            blob = [buf.raw]
        else:
            blob = [None]
        dist_mod.broadcast_object_list(blob, src=0)
        if rank != 0:
            hb = C.create_string_buffer(bytes(blob[0]), 64)
            check(lib().coadapt_nvls_import(dev, nranks, nbytes, hb, 64, C.byref(self.handle)))
        check(lib().coadapt_nvls_add_device(self.handle))
        dist_mod.barrier()
        uc, mc = C.c_void_p(), C.c_void_p()
        check(lib().coadapt_nvls_bind(self.handle, C.byref(uc), C.byref(mc)))
        dist_mod.barrier()
        self.unicast, self.multicast = int(uc.value), int(mc.value)
        if dtype == torch.bfloat16:  # no bf16 typestr: view the bytes as int16
            raw = torch.as_tensor(_CudaArray(self.unicast, self.numel, "<i2"), device=f"cuda:{dev}")
            self.tensor = raw.view(torch.bfloat16)
        else:
            self.tensor = torch.as_tensor(_CudaArray(self.unicast, self.numel, self._TYPESTR[dtype]),
                                          device=f"cuda:{dev}")

    def allreduce(self, scale: float = 1.0, stream=None) -> None:
        """tensor <- scale * sum over the group's tensors (this rank reduces
        and broadcasts its slice; bracket with barriers)."""
        check(lib().coadapt_nvls_allreduce(self.handle, TORCH_TO_DTYPE[self.dtype], self.numel,
                                           self.rank, float(scale), _stream(stream)))

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.tensor = None
            check(lib().coadapt_nvls_destroy(self.handle))
            self.handle = None


def dp_slice(numel: int, d: int, r: int) -> tuple:
    """[lo, hi) of DP slice r of d (the cut of coadapt_plan_create_slice)."""
    cut = lambda i: numel if i >= d else (numel * i // d) & ~63
    return cut(r), cut(r + 1)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().coadapt_nccl_unique_id(buf, 128))
    return buf.raw


def sqnorm(tensor: torch.Tensor, stream=None) -> float:
    """||tensor||^2 in fp64 on the device (one-shot K1)."""
    out = C.c_double()
    check(lib().coadapt_sqnorm_device(tensor.data_ptr(), tensor.numel(), TORCH_TO_DTYPE[tensor.dtype],
                                      tensor.device.index or 0, C.byref(out), _stream(stream)))
    return out.value


def synth_fill(out: torch.Tensor, gsegs, seed: int, sample: int, g0: float, noise_unit: float,
               stream=None) -> None:
    arr, n = _gen_array(gsegs)
    check(lib().coadapt_synth_fill(out.data_ptr(), TORCH_TO_DTYPE[out.dtype], arr, n, int(seed),
                                   int(sample), float(g0), float(noise_unit), _stream(stream)))


def synth_mean_fill(out: torch.Tensor, gsegs, seed: int, sample0: int, nsamples: int, g0: float,
                    noise_unit: float, stream=None) -> None:
    arr, n = _gen_array(gsegs)
    check(lib().coadapt_synth_mean_fill(out.data_ptr(), TORCH_TO_DTYPE[out.dtype], arr, n, int(seed),
                                        int(sample0), int(nsamples), float(g0), float(noise_unit),
                                        _stream(stream)))


def l2_flush(scratch: torch.Tensor, stream=None) -> None:
    check(lib().coadapt_l2_flush(scratch.data_ptr(), scratch.numel() * scratch.element_size(),
                                 _stream(stream)))


def read_probe(buf: torch.Tensor, sink: torch.Tensor, stream=None) -> None:
    check(lib().coadapt_read_probe(buf.data_ptr(), buf.numel() * buf.element_size(), sink.data_ptr(),
                                   _stream(stream)))


def kernel_launches() -> int:
    return int(lib().coadapt_kernel_launches())
