"""Trainer hook adapter: the paper's GNS manager inside the
forward-backward loop ("backward hooks capture the
per-microbatch statistics"), for a PyTorch model, on the B200 kernels.

Megatron-style layout: every trainable parameter's ``.grad`` is a view into
one contiguous *grad bucket* (the model dtype, e.g. bf16), and an fp32
*main_grad* bucket accumulates the micro-batches.  After micro-batch m's
backward, ``coadapt_gns_accumulate`` folds the bucket into main_grad and
computes s_m = Σ w‖g_m‖² in the same pass (the norms cost no extra HBM
read); on the last micro-batch of a d = 1 step it also reduces
‖ḡ‖² = ‖main_grad / M‖².  For d > 1 the caller synchronises main_grad
across the DP group (sum) and hands it to ``finish_step``, which reads this
rank's DP slice with the 1/(d·M)² scale folded into the plan weights — or
passes ``replicas`` (every DP rank's main_grad, CUDA-IPC peer pointers),
and ``finish_step`` all-reduces main_grad itself over NVLink with ḡ² in the
same pass (``coadapt_gns_allreduce_sqnorm``): afterwards main_grad holds the
DP-averaged gradient, as after Megatron DDP's averaging all-reduce.  With
``nvls_dist`` main_grad lives in NVLS memory and the NVSwitch does the sum
(``coadapt_nvls_allreduce``; pays from 4 GPUs).

Usage::

    mgr = GnsManager(model.parameters(), micro_count=M, global_batch=B_g)
    mgr.install_hooks()                # or call mgr.after_backward() yourself
    for step in ...:
        mgr.begin_step()
        for m in range(M):
            loss_fn(model(x[m])).backward()      # hook folds grads into main_grad
        r = mgr.finish_step(tokens=B_g * seq_len)  # r.phi, r.stats, r.state
        optimizer_step_on(mgr.main_grad)

    or, without a host sync per step: ``mgr.finish_step(tokens, wait=False)``,
    the optimizer step, then ``mgr.poll()`` / ``mgr.result()`` before the
    next ``finish_step``.

Do not call ``zero_grad(set_to_none=True)`` on the model: the manager owns
the grad views and clears the bucket after each micro-batch.
"""
from __future__ import annotations

from typing import Dict, Iterable, Optional

import torch

from . import _lib as L
from . import device as D


class GnsManager:
    def __init__(self, params: Iterable[torch.nn.Parameter], micro_count: int, global_batch: int,
                 dp_size: int = 1, dp_rank: int = 0,
                 weights: Optional[Dict[torch.nn.Parameter, float]] = None, device: Optional[int] = None,
                 nvls_dist=None):
        """nvls_dist (d > 1): a torch.distributed module/group handle; main_grad
        is then allocated in NVLS memory (device.NvlsBucket, collective over
        the DP group) and finish_step all-reduces it through the NVSwitch."""
        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise L.ValidationError("no trainable parameters")
        dtypes = {p.dtype for p in self.params}
        if len(dtypes) != 1 or next(iter(dtypes)) not in D.TORCH_TO_DTYPE:
            raise L.ValidationError(f"parameters must share one of bf16/fp16/fp32, got {dtypes}")
        self.dtype = next(iter(dtypes))
        dev = self.params[0].device if device is None else torch.device("cuda", device)
        self.device = dev.index if dev.index is not None else torch.cuda.current_device()
        self.M, self.d, self.dp_rank = int(micro_count), int(dp_size), int(dp_rank)
        weights = weights or {}
        segs, off = [], 0
        self._slots = []
        for p in self.params:
            n = p.numel()
            self._slots.append((off, n))
            segs.append((off, n, float(weights.get(p, 1.0))))
            off += (n + 7) // 8 * 8  # 16-byte aligned views
        self.numel = off
        self.segments = segs
        self.grad_bucket = torch.zeros(off, dtype=self.dtype, device=f"cuda:{self.device}")
        self._nvls = None
        if nvls_dist is not None and self.d > 1:
            self._nvls = D.NvlsBucket(off, torch.float32, self.dp_rank, self.d, nvls_dist, self.device)
            self.main_grad = self._nvls.tensor  # zeroed by the bind
        else:
            self.main_grad = torch.zeros(off, dtype=torch.float32, device=f"cuda:{self.device}")
        for p, (o, n) in zip(self.params, self._slots):
            p.grad = self.grad_bucket[o:o + n].view_as(p)
        self.plan = D.BucketPlan(segs, off, D.TORCH_TO_DTYPE[self.dtype], self.device)
        self.gns = D.GnsDevice(self.d, self.M, global_batch, self.device)
        self._mean_plan = None
        self._ar_plan = None
        self._m = 0
        self._pending = 0
        self._hooks = []

    # ------------------------------------------------------------ hooks
    def install_hooks(self) -> None:
        """Run after_backward() once every parameter's gradient of the
        micro-batch has been accumulated (post-accumulate-grad hooks)."""
        def hook(_p):
            self._pending += 1
            if self._pending == len(self.params):
                self._pending = 0
                self.after_backward()
        for p in self.params:
            self._hooks.append(p.register_post_accumulate_grad_hook(hook))

    def remove_hooks(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []

    # ------------------------------------------------------------ step
    def begin_step(self, stream=None) -> None:
        self.gns.begin_step(stream)
        self._m = 0

    def after_backward(self, stream=None) -> None:
        """Fold the grad bucket (micro-batch m) into main_grad with s_m."""
        m = self._m
        if m >= self.M:
            raise L.ValidationError(f"more than M = {self.M} micro-batches in one step")
        last_mean = self.d == 1 and m == self.M - 1
        self.gns.accumulate(self.plan, self.main_grad, self.grad_bucket, self.dp_rank, m,
                            first=(m == 0), last_mean=last_mean,
                            mean_scale_sq=1.0 / float(self.M) ** 2, stream=stream)
        self.grad_bucket.zero_()
        self._m = m + 1

    def finish_step(self, tokens: int, synced_main_grad: Optional[torch.Tensor] = None,
                    replicas=None, stream=None, wait: bool = True) -> Optional[L.GnsResult]:
        """All-reduce the slots (if attached), finalize, read φ.  For d > 1
        either pass the DP-summed main_grad (this rank reads its slice of
        it) or ``replicas`` — the d ranks' main_grad buckets in DP order
        (peer pointers; this rank's own tensor or pointer at dp_rank): the
        DP all-reduce (mean) of main_grad and ḡ² then run as one NVLink pass,
        bracketed by stream-ordered barriers.

        ``wait=False`` enqueues everything and returns None without
        blocking: the host goes on to enqueue the optimizer step and the
        next forward while the GPU finishes, and reads φ with ``poll()`` or
        ``result()`` any time before the next ``finish_step``."""
        if self._m != self.M:
            raise L.ValidationError(f"step has {self._m} of {self.M} micro-batches")
        if self.d > 1 and self._nvls is not None:
            # NVLS: the switch sums the DP group's main_grad (mean) into every
            # copy, and this rank's slice's gbar^2 part is taken in the same
            # pass (coadapt_gns_nvls_reduce_sqnorm)
            if self._ar_plan is None:
                sc = 1.0 / float(self.M) ** 2  # out = mean over DP; gbar = out / M
                self._ar_plan = D.BucketPlan([(o, n, w * sc) for o, n, w in self.segments],
                                             self.numel, L.FP32, self.device)
            self.gns.barrier(stream)
            self.gns.nvls_reduce_sqnorm(self._ar_plan, self._nvls, self.dp_rank, 1.0 / self.d,
                                        stream=stream)
            self.gns.barrier(stream)
        elif self.d > 1 and replicas is not None:
            if len(replicas) != self.d:
                raise L.ValidationError(f"need {self.d} replicas, got {len(replicas)}")
            if self._ar_plan is None:
                sc = 1.0 / float(self.M) ** 2  # out = mean over DP; gbar = out / M
                self._ar_plan = D.BucketPlan([(o, n, w * sc) for o, n, w in self.segments],
                                             self.numel, L.FP32, self.device)
            self.gns.barrier(stream)
            self.gns.allreduce_sqnorm(self._ar_plan, replicas, self.dp_rank, 1.0 / self.d, stream)
            self.gns.barrier(stream)
        elif self.d > 1:
            if synced_main_grad is None:
                raise L.ValidationError("d > 1: pass the DP-summed main_grad or the replicas")
            if self._mean_plan is None:
                sc = 1.0 / float(self.d * self.M) ** 2
                self._mean_plan = D.BucketPlan([(o, n, w * sc) for o, n, w in self.segments],
                                               self.numel, L.FP32, self.device,
                                               slice_index=self.dp_rank, slice_count=self.d)
            self.gns.mean_sqnorm(self._mean_plan, synced_main_grad, stream)
        self.gns.allreduce(stream)
        self.gns.finalize(int(tokens), stream)
        return self.gns.result() if wait else None

    def poll(self) -> Optional[L.GnsResult]:
        """The last finished step's result if it has reached the host, else
        None (never blocks)."""
        return self.gns.result() if self.gns.result_ready() else None

    def result(self) -> L.GnsResult:
        """The last finished step's result (waits for it)."""
        return self.gns.result()
