"""ctypes binding of libcoadapt_b200.so (include/coadapt_cuda.h + coadapt_host.h).

This is the binding a Python maintainer of the reference would add (see
INTEGRATION.md).  The library is built in-tree (``make -C
paper_2604_26687_b200/csrc``); importing this module without it raises —
there is no Python or CPU fallback for the device path.
"""
from __future__ import annotations

import ctypes as C
import os
import re

# torch first: it loads its bundled libnccl.so.2, which our library then
# binds to by soname instead of pulling the (older) system copy.
import torch  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
# COADAPT_LIB_PATH: load an alternative build (kernel A/B experiments only)
LIB_PATH = os.environ.get("COADAPT_LIB_PATH") or os.path.join(_HERE, "lib", "libcoadapt_b200.so")
INCLUDE_DIR = os.path.join(os.path.dirname(_HERE), "include")

OK, E_VALIDATION, E_INTERNAL, E_CUDA, E_NCCL = 0, 1, 2, 3, 4
BF16, FP16, FP32, FP64 = 0, 1, 2, 3
NOOP, SCALE_BS, RECONFIGURE = 0, 1, 2


class ValidationError(ValueError):
    """errors.hpp:10 — a documented contract was violated (status 1)."""


class InternalError(RuntimeError):
    """errors.hpp:24 — library bug (status 2)."""


class CudaError(RuntimeError):
    """status 3: CUDA runtime / device failure."""


class NcclError(RuntimeError):
    """status 4: NCCL failure."""


class Segment(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("numel", C.c_uint64), ("weight", C.c_double)]


class GenSegment(C.Structure):
    _fields_ = [("local_off", C.c_uint64), ("numel", C.c_uint64), ("global_base", C.c_uint64),
                ("row_len", C.c_uint64), ("row_stride", C.c_uint64)]


class StepStats(C.Structure):
    """StepStats, gns.hpp:35-40."""
    _fields_ = [("signal", C.c_double), ("noise", C.c_double), ("noise_raw", C.c_double),
                ("mean_grad_sq", C.c_double)]


class GnsState(C.Structure):
    """GnsState, gns.hpp:53-62 (defaults via GnsState.default())."""
    _fields_ = [("ema_signal", C.c_double), ("ema_noise", C.c_double), ("alpha_early", C.c_double),
                ("alpha_late", C.c_double), ("phase_boundary_tokens", C.c_int64),
                ("tokens_seen", C.c_int64), ("calibration", C.c_double),
                ("initialized", C.c_int32), ("reserved_", C.c_int32)]

    @classmethod
    def default(cls) -> "GnsState":
        s = cls()
        lib().coadapt_gns_state_init(C.byref(s))
        return s

    def as_tuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_ if f != "reserved_")


class GnsResult(C.Structure):
    _fields_ = [("stats", StepStats), ("state", GnsState), ("phi", C.c_double),
                ("b_simple", C.c_double), ("sample_count", C.c_int64),
                ("phi_available", C.c_int32), ("status", C.c_int32)]


class CandidateC(C.Structure):
    _fields_ = [("d", C.c_int32), ("t", C.c_int32), ("p", C.c_int32), ("reserved_", C.c_int32),
                ("global_batch", C.c_int64), ("micro_batch", C.c_int64), ("throughput", C.c_double)]


class CostC(C.Structure):
    _fields_ = [("d", C.c_int32), ("t", C.c_int32), ("p", C.c_int32), ("reserved_", C.c_int32),
                ("t_max", C.c_double), ("b_hw", C.c_double)]


class OrchCfgC(C.Structure):
    _fields_ = [("margin", C.c_double), ("max_growth", C.c_double), ("reconfig_cost", C.c_double),
                ("reference_batch", C.c_double)]


class CommandC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("winner_index", C.c_int32), ("winner_score", C.c_double),
                ("current_score", C.c_double), ("penalized", C.c_int32), ("reserved_", C.c_int32)]


class ProfileEntryC(C.Structure):
    _fields_ = [("d", C.c_int32), ("t", C.c_int32), ("p", C.c_int32), ("reserved_", C.c_int32),
                ("global_batch", C.c_int64), ("micro_batch", C.c_int64),
                ("samples_per_sec", C.c_double), ("peak_mem_bytes", C.c_double),
                ("feasible", C.c_int32), ("reserved2_", C.c_int32)]


class DecisionRowC(C.Structure):
    _fields_ = [("step", C.c_int64), ("time_s", C.c_double), ("phi", C.c_double),
                ("current", CandidateC), ("winner", CandidateC), ("command", CommandC)]


MAXD = 4  # COADAPT_RESHARD_MAX_DIMS


class TensorDeclC(C.Structure):
    _fields_ = [("name", C.c_char_p), ("ndim", C.c_int32), ("tp_axis", C.c_int32),
                ("shape", C.c_int64 * MAXD)]


class ReshardModelC(C.Structure):
    _fields_ = [("layers", C.c_int32), ("n_tensors", C.c_int32), ("tensors", C.POINTER(TensorDeclC)),
                ("optimizer_state_multiplier", C.c_int32), ("param_bytes", C.c_int32),
                ("state_bytes", C.c_int32), ("reserved_", C.c_int32)]


class ShardC(C.Structure):
    _fields_ = [("layer", C.c_int32), ("tensor", C.c_int32), ("owner", C.c_int32),
                ("canonical", C.c_int32), ("global_shape", C.c_int64 * MAXD),
                ("global_offset", C.c_int64 * MAXD), ("local_shape", C.c_int64 * MAXD),
                ("pack_offset", C.c_uint64), ("ndim", C.c_int32), ("reserved_", C.c_int32)]


class MoveC(C.Structure):
    _fields_ = [("src_rank", C.c_int32), ("dst_rank", C.c_int32), ("layer", C.c_int32),
                ("tensor", C.c_int32), ("offset", C.c_int64 * MAXD), ("extent", C.c_int64 * MAXD),
                ("bytes", C.c_uint64), ("local", C.c_int32), ("ndim", C.c_int32)]


class ReshardInfoC(C.Structure):
    _fields_ = [("n_moves", C.c_uint64), ("total_bytes", C.c_uint64),
                ("max_bytes_per_rank", C.c_uint64), ("local_bytes", C.c_uint64),
                ("src_ranks", C.c_int32), ("dst_ranks", C.c_int32),
                ("src_max_pack_numel", C.c_uint64), ("dst_max_pack_numel", C.c_uint64)]


class GradTensorC(C.Structure):
    _fields_ = [("name", C.c_char_p), ("stage", C.c_int32), ("ndim", C.c_int32),
                ("tp_axis", C.c_int32), ("reserved_", C.c_int32), ("shape", C.c_int64 * 4)]


class GradModelC(C.Structure):
    _fields_ = [("name", C.c_char_p), ("layers", C.c_int32), ("tied", C.c_int32),
                ("tensors", C.POINTER(GradTensorC)), ("n_tensors", C.c_size_t)]


class SegmentC(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("numel", C.c_uint64), ("weight", C.c_double)]


class GenSegmentC(C.Structure):
    _fields_ = [("local_off", C.c_uint64), ("numel", C.c_uint64), ("global_base", C.c_uint64),
                ("row_len", C.c_uint64), ("row_stride", C.c_uint64)]


class ClockC(C.Structure):
    _fields_ = [("elapsed", C.c_double), ("useful", C.c_double), ("reconfig_total", C.c_double),
                ("reconfigs", C.c_int64)]


class TraceRowC(C.Structure):
    _fields_ = [("step", C.c_int64), ("tokens", C.c_int64), ("signal_raw", C.c_double),
                ("noise_raw", C.c_double), ("ema_signal", C.c_double), ("ema_noise", C.c_double),
                ("phi", C.c_double)]


P, I, I32, I64, U64, SZ, D, F = (C.c_void_p, C.c_int, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t,
                                 C.c_double, C.c_float)

# name -> (restype, argtypes); the full exported surface of both headers.
SIGNATURES = {
    # coadapt_cuda.h
    "coadapt_last_error": (C.c_char_p, []),
    "coadapt_abi_version": (I, []),
    "coadapt_kernel_launches": (U64, []),
    "coadapt_device_info": (I, [I, P, P, P, P]),
    "coadapt_plan_create": (I, [P, SZ, U64, I, I, P]),
    "coadapt_plan_create_slice": (I, [P, SZ, U64, I, I, I, I, P]),
    "coadapt_plan_destroy": (I, [P]),
    "coadapt_plan_info": (I, [P, P, P]),
    "coadapt_gns_create": (I, [I, I, I64, I, P]),
    "coadapt_gns_destroy": (I, [P]),
    "coadapt_gns_reshape": (I, [P, I, I, I64]),
    "coadapt_gns_begin_step": (I, [P, P]),
    "coadapt_gns_micro_sqnorm": (I, [P, P, P, I, I, P]),
    "coadapt_gns_micro_sqnorm_batched": (I, [P, P, P, P, P, I, P]),
    "coadapt_gns_fused_sqnorm": (I, [P, P, P, I, P]),
    "coadapt_gns_mean_sqnorm": (I, [P, P, P, P]),
    "coadapt_gns_fused_sqnorm_host": (I, [P, P, P, I, P]),
    "coadapt_gns_accumulate": (I, [P, P, P, P, I, I, I, D, P]),
    "coadapt_ipc_handle": (I, [P, P, SZ, P]),
    "coadapt_ipc_open": (I, [P, SZ, I, P]),
    "coadapt_ipc_close": (I, [P]),
    "coadapt_gns_barrier": (I, [P, P]),
    "coadapt_gns_reduce_scatter_sqnorm": (I, [P, P, P, I, I, P, D, P]),
    "coadapt_gns_allreduce_sqnorm": (I, [P, P, P, I, I, D, P]),
    "coadapt_nccl_unique_id": (I, [P, SZ]),
    "coadapt_gns_attach_nccl": (I, [P, I, I, P, SZ]),
    "coadapt_gns_allreduce": (I, [P, P]),
    "coadapt_gns_finalize": (I, [P, I64, P]),
    "coadapt_gns_fused_sqnorm_finalize": (I, [P, P, P, I, I64, P]),
    "coadapt_gns_mean_sqnorm_finalize": (I, [P, P, P, I64, P]),
    "coadapt_gns_read_result": (I, [P, P]),
    "coadapt_gns_result_ready": (I, [P, P]),
    "coadapt_gns_read_partials": (I, [P, P, SZ]),
    "coadapt_gns_get_state": (I, [P, P]),
    "coadapt_gns_set_state": (I, [P, P]),
    "coadapt_sqnorm_device": (I, [P, U64, I, I, P, P]),
    "coadapt_sqnorm_host": (I, [P, U64, I, I, P]),
    "coadapt_synth_fill": (I, [P, I, P, SZ, U64, U64, F, F, P]),
    "coadapt_synth_mean_fill": (I, [P, I, P, SZ, U64, U64, I64, F, F, P]),
    "coadapt_gns_micro_sqnorm_host": (I, [P, P, P, I, I, P]),
    "coadapt_gns_attach_nccl_all": (I, [P, I]),
    "coadapt_gns_mailbox": (I, [P, I, P]),
    "coadapt_gns_attach_mailboxes": (I, [P, I, I, P]),
    "coadapt_gns_allreduce_finalize_p2p": (I, [P, I64, P]),
    "coadapt_gns_allreduce_group": (I, [P, P, I]),
    "coadapt_gns_mean_sqnorm_host": (I, [P, P, P, P]),
    "coadapt_l2_flush": (I, [P, U64, P]),
    "coadapt_read_probe": (I, [P, U64, P, P]),
    "coadapt_nvls_create": (I, [I, I, U64, P]),
    "coadapt_nvls_export": (I, [P, P, SZ]),
    "coadapt_nvls_import": (I, [I, I, U64, P, SZ, P]),
    "coadapt_nvls_add_device": (I, [P]),
    "coadapt_nvls_bind": (I, [P, P, P]),
    "coadapt_nvls_bytes": (U64, [P]),
    "coadapt_nvls_allreduce": (I, [P, I, U64, I, D, P]),
    "coadapt_nvls_destroy": (I, [P]),
    "coadapt_gns_nvls_reduce_sqnorm": (I, [P, P, P, I, I, P, D, P]),
    # coadapt_host.h
    "coadapt_finalize_step": (I, [P, I64, I, D, I64, P]),
    "coadapt_finalize_step_vec": (I, [P, I64, I, P, U64, I64, P]),
    "coadapt_update_ema": (I, [P, P, I64]),
    "coadapt_gns_phi": (I, [P, P]),
    "coadapt_gns_state_init": (None, [P]),
    "coadapt_stat_eff": (D, [D, D]),
    "coadapt_goodput": (D, [D, D]),
    "coadapt_goodput_lr": (D, [D, D, D, D]),
    "coadapt_lr_rescale": (D, [D, D, D]),
    "coadapt_optimal_batch_continuous": (D, [D, D]),
    "coadapt_cbs_target": (I, [D, P, SZ, I, P]),
    "coadapt_synth_candidates": (I, [P, SZ, P, SZ, P, SZ, I, D, D, D, P, P]),
    "coadapt_score_candidates": (I, [P, SZ, D, P, D, D, P, P]),
    "coadapt_rank_candidates": (I, [P, SZ, D, P, D, D, P, P]),
    "coadapt_decide": (I, [P, SZ, I, D, P, D, D, P, P]),
    "coadapt_trace_csv": (I, [P, SZ, P, SZ, P]),
    "coadapt_format_double": (I, [D, P, SZ]),
    "coadapt_profile_parse": (I, [P, SZ, P, P, P]),
    "coadapt_profile_format": (I, [P, SZ, P, SZ, P]),
    "coadapt_profile_load": (I, [C.c_char_p, P, P, P]),
    "coadapt_profile_save": (I, [C.c_char_p, P, SZ]),
    "coadapt_decision_audit_csv": (I, [P, SZ, P, SZ, P]),
    "coadapt_simulate_micro_gradients": (I, [P, P, U64, I64, I, U64, P]),
    "coadapt_record_reconfig": (I, [P, P, D]),
    # coadapt_reshard.h
    "coadapt_reshard_plan_create": (I, [P, P, P, I, P]),
    "coadapt_reshard_plan_destroy": (I, [P]),
    "coadapt_reshard_plan_info": (I, [P, P]),
    "coadapt_reshard_moves": (I, [P, P, P]),
    "coadapt_reshard_shards": (I, [P, I, P, P]),
    "coadapt_reshard_pack_numel": (I, [P, I, I, P]),
    "coadapt_reshard_plan_csv": (I, [P, P, SZ, P]),
    "coadapt_reshard_latency": (I, [P, D, D, P]),
    "coadapt_reshard_execute": (I, [P, I, I, P, SZ, P, SZ, I, I, P]),
    # coadapt_segments.h
    "coadapt_model_preset": (I, [C.c_char_p, P]),
    "coadapt_gns_segments": (I, [P, I, I, I, I, P, P, SZ, P, P, P]),
    "coadapt_gns_algorithmic_bytes": (I, [P, I, I, I, I, I, I, P]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded library.  Raises ImportError when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make -C paper_2604_26687_b200/csrc` "
                              "(or __graft_entry__.build()); there is no fallback path")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().coadapt_last_error().decode(errors="replace")
    raise {E_VALIDATION: ValidationError, E_INTERNAL: InternalError, E_CUDA: CudaError,
           E_NCCL: NcclError}.get(rc, InternalError)(msg)


def header_symbols() -> list[str]:
    """Every function declared in the C-ABI headers under include/."""
    names = []
    for h in ("coadapt_cuda.h", "coadapt_host.h", "coadapt_reshard.h", "coadapt_segments.h"):
        text = open(os.path.join(INCLUDE_DIR, h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"\b(coadapt_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))
