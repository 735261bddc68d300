"""Multi-GPU worker for the fused DP reduce-scatter + gbar^2 over NVLink
(coadapt_gns_reduce_scatter_sqnorm), launched with torch.distributed.run.

Each rank holds one DP replica's gradient bucket; IPC handles are exchanged
with torch.distributed; every rank reduces its slice straight from the peers'
HBM.  The all-reduce form (coadapt_gns_allreduce_sqnorm) writes the slice
back into every replica in place.  Checks (rank 0 prints one JSON line):
  * the slice is bit-identical to torch: sum of the all-gathered replicas in
    replica order in fp32, times scale, rounded to the bucket dtype;
  * the all-reduced gbar^2 equals the fp64 norm of the whole synchronised
    gradient (weights applied) to 1e-12;
  * timing against NCCL reduce_scatter_tensor + the K2 slice norm;
  * all-reduce form: every replica bit-identical to the same reference over
    the WHOLE bucket, gbar^2 as above, timing against NCCL all_reduce + K2.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402
from paper_2604_26687_b200 import dist as Dist  # noqa: E402

TDT = {L.BF16: torch.bfloat16, L.FP32: torch.float32}


def check_case(rank, world, local, numel, dtype, bench_mb=0):
    torch.manual_seed(1234 + rank)
    tdt = TDT[dtype]
    n = numel
    segs = [(0, n // 3, 1.0), (n // 3, 1000, 0.0), (n // 3 + 1000, n - n // 3 - 1000, 1.0)]
    rep = (torch.randn(n, device="cuda") * (1 + rank)).to(tdt)
    plan = D.BucketPlan(segs, n, dtype, local)
    g = D.GnsDevice(world, 1, world, local)
    Dist.attach(g, dist, world, rank)
    handles = [None] * world
    dist.all_gather_object(handles, D.ipc_handle(rep))
    ptrs, bases = [], []
    for q in range(world):
        if q == rank:
            ptrs.append(rep.data_ptr())
        else:
            p, b = D.ipc_open(handles[q], local)
            ptrs.append(p)
            bases.append(b)
    lo, hi = D.dp_slice(n, world, rank)
    out = torch.empty(hi - lo, dtype=tdt, device="cuda")
    scale = 1.0 / world
    g.begin_step()
    g.barrier()
    g.reduce_scatter_sqnorm(plan, ptrs, rank, out, scale)
    g.barrier()
    g.allreduce()
    parts = g.partials()
    # reference
    allr = [torch.empty_like(rep) for _ in range(world)]
    dist.all_gather(allr, rep)
    acc = allr[0].float().clone()
    for q in range(1, world):
        acc.add_(allr[q].float())
    ref = (acc * scale).to(tdt)
    ok_slice = bool(torch.equal(out, ref[lo:hi]))
    w = torch.ones(n, dtype=torch.float64, device="cuda")
    w[n // 3:n // 3 + 1000] = 0
    g2_ref = float((w * ref.double() ** 2).sum())
    rel = abs(parts[-1] - g2_ref) / g2_ref
    res = {"dtype": "bf16" if dtype == L.BF16 else "fp32", "numel": n, "slice_bit_exact": ok_slice,
           "gbar2_rel": rel}
    if bench_mb:
        big = (bench_mb << 20) // rep.element_size()
        big -= big % (64 * world)
        x = (torch.randn(big, device="cuda") * (1 + rank)).to(tdt)
        bplan = D.BucketPlan([(0, big, 1.0)], big, dtype, local)
        hs = [None] * world
        dist.all_gather_object(hs, D.ipc_handle(x))
        bp = [x.data_ptr() if q == rank else D.ipc_open(hs[q], local)[0] for q in range(world)]
        blo, bhi = D.dp_slice(big, world, rank)
        bout = torch.empty(bhi - blo, dtype=tdt, device="cuda")
        rs_out = torch.empty(big // world, dtype=tdt, device="cuda")
        rplan = D.BucketPlan([(0, big // world, 1.0)], big // world, dtype, local)

        def fused():
            g.begin_step()
            g.barrier()
            g.reduce_scatter_sqnorm(bplan, bp, rank, bout, scale)
            g.barrier()

        def nccl_then_norm():
            # the unfused baseline: NCCL reduce-scatter, then the K2 norm of
            # the reduced slice (a second read); rs_out holds slice `rank`
            g.begin_step()
            dist.reduce_scatter_tensor(rs_out, x, op=dist.ReduceOp.SUM)
            g.mean_sqnorm(rplan, rs_out)

        def timed(fn, reps=10):
            fn()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        ms_fused = timed(fused)
        ms_rs = timed(lambda: dist.reduce_scatter_tensor(rs_out, x, op=dist.ReduceOp.SUM))
        ms_rs_norm = timed(nccl_then_norm)
        res.update({"bench_bytes_per_rank": big * rep.element_size(), "fused_ms": ms_fused,
                    "nccl_reduce_scatter_ms": ms_rs, "nccl_rs_plus_k2_ms": ms_rs_norm,
                    "fused_gbs_per_rank": big * rep.element_size() / (ms_fused / 1e3) / 1e9})
    for b in bases:
        D.ipc_close(b)
    g.close()
    return res


def _open_all(x, rank, world, local):
    hs = [None] * world
    dist.all_gather_object(hs, D.ipc_handle(x))
    ptrs, bases = [], []
    for q in range(world):
        if q == rank:
            ptrs.append(x.data_ptr())
        else:
            p, b = D.ipc_open(hs[q], local)
            ptrs.append(p)
            bases.append(b)
    return ptrs, bases


def check_allreduce(rank, world, local, numel, dtype, bench_mb=0):
    torch.manual_seed(4321 + rank)
    tdt = TDT[dtype]
    n = numel
    segs = [(0, n // 3, 1.0), (n // 3, 1000, 0.0), (n // 3 + 1000, n - n // 3 - 1000, 1.0)]
    rep = (torch.randn(n, device="cuda") * (1 + rank)).to(tdt)
    allr = [torch.empty_like(rep) for _ in range(world)]
    dist.all_gather(allr, rep)
    acc = allr[0].float().clone()
    for q in range(1, world):
        acc.add_(allr[q].float())
    scale = 1.0 / world
    ref = (acc * scale).to(tdt)
    plan = D.BucketPlan(segs, n, dtype, local)
    g = D.GnsDevice(world, 1, world, local)
    Dist.attach(g, dist, world, rank)
    ptrs, bases = _open_all(rep, rank, world, local)
    g.begin_step()
    g.barrier()
    g.allreduce_sqnorm(plan, ptrs, rank, scale)
    g.barrier()
    g.allreduce()
    parts = g.partials()
    torch.cuda.synchronize()
    ok = bool(torch.equal(rep, ref))
    w = torch.ones(n, dtype=torch.float64, device="cuda")
    w[n // 3:n // 3 + 1000] = 0
    g2_ref = float((w * ref.double() ** 2).sum())
    rel = abs(parts[-1] - g2_ref) / g2_ref
    res = {"form": "allreduce", "dtype": "bf16" if dtype == L.BF16 else "fp32", "numel": n,
           "slice_bit_exact": ok, "gbar2_rel": rel}
    if bench_mb:
        big = (bench_mb << 20) // rep.element_size()
        big -= big % (64 * world)
        x = (torch.randn(big, device="cuda") * (1 + rank)).to(tdt)
        bplan = D.BucketPlan([(0, big, 1.0)], big, dtype, local)
        bp, bb = _open_all(x, rank, world, local)
        blo, bhi = D.dp_slice(big, world, rank)
        splan = D.BucketPlan([(0, bhi - blo, 1.0)], bhi - blo, dtype, local)

        def fused():
            g.begin_step()
            g.barrier()
            g.allreduce_sqnorm(bplan, bp, rank, scale)
            g.barrier()

        def nccl_then_norm():
            # DDP's unfused form: NCCL all-reduce (sum), then the K2 norm of
            # this rank's slice (a second read; the mean scale folded in)
            g.begin_step()
            dist.all_reduce(x, op=dist.ReduceOp.SUM)
            g.mean_sqnorm(splan, x[blo:bhi])

        def timed(fn, reps=10):
            fn()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        res.update({"bench_bytes_per_rank": big * rep.element_size(),
                    "fused_allreduce_ms": timed(fused),
                    "nccl_allreduce_ms": timed(lambda: dist.all_reduce(x, op=dist.ReduceOp.SUM)),
                    "nccl_allreduce_plus_k2_ms": timed(nccl_then_norm)})
        bases += bb
    for b in bases:
        D.ipc_close(b)
    g.close()
    return res


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    cases = [check_case(rank, world, local, 1_000_003 - 3, L.BF16),
             check_case(rank, world, local, 777_216, L.FP32),
             check_case(rank, world, local, 4_000_000, L.BF16, bench_mb=int(os.environ.get("RS_BENCH_MB", "0"))),
             check_allreduce(rank, world, local, 1_000_003 - 3, L.BF16),
             check_allreduce(rank, world, local, 777_216, L.FP32),
             check_allreduce(rank, world, local, 4_000_000, L.BF16,
                             bench_mb=int(os.environ.get("RS_BENCH_MB", "0")))]
    ok = all(c["slice_bit_exact"] and c["gbar2_rel"] <= 1e-12 for c in cases)
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": world, "ok": bool(t.item()), "cases": cases}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if t.item() else 1


if __name__ == "__main__":
    sys.exit(main())
