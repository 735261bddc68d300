"""Multi-GPU worker for the NVLS (switch-reduced) DP gradient all-reduce
(coadapt_nvls_*), launched with torch.distributed.run.

Each rank owns one DP replica's bucket in NVLS memory; after the all-reduce
every rank's fp32 bucket must hold scale * fp32(sum_q replica_q) — the same
reference as the P2P form — bit-exact for d = 2 (a two-term fp32 sum has one
rounding whatever the order) and within the rounding of a d-term fp32 sum
for d > 2 (the switch's summation order is its own).  gbar^2 of the rank's
slice (K2 on the unicast view) all-reduced over the slots must equal the
fp64 norm of the reference.  bf16 buckets are refused (the switch's bf16
rounding is biased).  Optional timing (NVLS_BENCH_MB) against NCCL
all_reduce and the P2P form.  Rank 0 prints one JSON line.
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402
from paper_2604_26687_b200 import dist as Dist  # noqa: E402


def check_case(rank, world, local, numel, tdt=torch.float32):
    torch.manual_seed(99 + rank)
    buck = D.NvlsBucket(numel, tdt, rank, world, dist, local)
    x = (torch.randn(numel, device="cuda") * (1 + rank)).to(tdt)
    buck.tensor.copy_(x)
    allr = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(allr, x)
    acc = allr[0].float().clone()
    mag = allr[0].float().abs()
    for q in range(1, world):
        acc.add_(allr[q].float())
        mag.add_(allr[q].float().abs())
    scale = 1.0 / world
    ref = (acc * scale).to(tdt)
    g = D.GnsDevice(world, 1, world, local)
    Dist.attach(g, dist, world, rank)
    torch.cuda.synchronize()
    g.begin_step()
    g.barrier()
    buck.allreduce(scale)
    g.barrier()
    sl = D.BucketPlan([(0, numel, 1.0)], numel, L.FP32, local, slice_index=rank, slice_count=world)
    g.mean_sqnorm(sl, buck.tensor)
    g.allreduce()
    parts = g.partials()
    torch.cuda.synchronize()
    n_diff = int((buck.tensor != ref).sum().item())
    # d-term fp32 sum in another order: |err| <= (d - 1) u sum|x_q| (u = 2^-24)
    bound = (world - 1) * 2.0 ** -24 * mag * scale
    within = bool(((buck.tensor - ref).abs() <= bound).all().item())
    g2_ref = float((ref.double() ** 2).sum())
    g2_rel = abs(parts[-1] - g2_ref) / g2_ref
    sl.close()
    g.close()
    buck.close()
    ok = (n_diff == 0 if world == 2 else within) and g2_rel <= (1e-12 if world == 2 else 1e-9)
    return {"dtype": "fp32", "numel": numel, "mismatches": n_diff, "within_sum_bound": within,
            "gbar2_rel": g2_rel, "ok": bool(ok)}


def check_fused(rank, world, local, numel):
    """coadapt_gns_nvls_reduce_sqnorm: reduce-scatter into a local slice and
    all-reduce in place, gbar^2 of the slice (segment weights honoured) in
    the same pass — against the replica-order fp32 reference."""
    torch.manual_seed(7 + rank)
    buck = D.NvlsBucket(numel, torch.float32, rank, world, dist, local)
    x = torch.randn(numel, device="cuda") * (1 + rank)
    allr = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(allr, x)
    acc, mag = allr[0].clone(), allr[0].abs()
    for q in range(1, world):
        acc.add_(allr[q])
        mag.add_(allr[q].abs())
    scale = 1.0 / world
    ref = acc * scale
    bound = (world - 1) * 2.0 ** -24 * mag * scale
    # a weight-0 hole and a weight-0.5 range: gbar^2 honours the plan
    segs = [(0, 1000, 1.0), (1000, 3000, 0.0), (4000, 2000, 0.5), (6000, numel - 6000, 1.0)]
    w = torch.ones(numel, dtype=torch.float64, device="cuda")
    w[1000:4000] = 0.0
    w[4000:6000] = 0.5
    plan = D.BucketPlan(segs, numel, L.FP32, local)
    lo = (numel * rank // world) & ~63
    hi = numel if rank + 1 == world else (numel * (rank + 1) // world) & ~63
    res = {"numel": numel}
    ok = True
    for form in ("reduce_scatter", "allreduce"):
        buck.tensor.copy_(x)
        g = D.GnsDevice(world, 1, world, local)
        Dist.attach(g, dist, world, rank)
        out = torch.empty(hi - lo, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        g.begin_step()
        g.barrier()
        g.nvls_reduce_sqnorm(plan, buck, rank, scale, out if form == "reduce_scatter" else None)
        g.barrier()
        g.allreduce()
        parts = g.partials()
        torch.cuda.synchronize()
        got = out if form == "reduce_scatter" else buck.tensor
        want = ref[lo:hi] if form == "reduce_scatter" else ref
        bnd = bound[lo:hi] if form == "reduce_scatter" else bound
        exact = bool(torch.equal(got, want))
        within = bool(((got - want).abs() <= bnd).all().item())
        g2_ref = float((w * ref.double() ** 2).sum())
        g2_rel = abs(parts[-1] - g2_ref) / g2_ref
        res[form] = {"bit_exact": exact, "within_sum_bound": within, "gbar2_rel": g2_rel}
        ok = ok and (exact if world == 2 else within) and g2_rel <= (1e-12 if world == 2 else 1e-8)
        g.close()
    plan.close()
    buck.close()
    res["ok"] = bool(ok)
    return res


def check_bf16_refused(rank, world, local):
    buck = D.NvlsBucket(4096, torch.bfloat16, rank, world, dist, local)
    try:
        buck.allreduce(1.0 / world)
        refused = False
    except L.ValidationError:
        refused = True
    buck.close()
    return {"dtype": "bf16", "refused": refused, "ok": refused}


def bench(rank, world, local, mb, tdt=torch.float32):
    es = torch.empty((), dtype=tdt).element_size()
    n = (mb << 20) // es
    n -= n % (64 * world)
    buck = D.NvlsBucket(n, tdt, rank, world, dist, local)
    buck.tensor.copy_((torch.randn(n, device="cuda") * (1 + rank)).to(tdt))
    x = torch.randn(n, device="cuda").to(tdt)
    dt = D.TORCH_TO_DTYPE[tdt]
    g = D.GnsDevice(world, 1, world, local)
    Dist.attach(g, dist, world, rank)
    plan = D.BucketPlan([(0, n, 1.0)], n, dt, local)
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

    def nvls():
        g.barrier()
        buck.allreduce(1.0 / world)
        g.barrier()

    def p2p():
        g.barrier()
        g.allreduce_sqnorm(plan, ptrs, rank, 1.0 / world)
        g.barrier()

    lo = (n * rank // world) & ~63
    hi = n if rank + 1 == world else (n * (rank + 1) // world) & ~63
    out = torch.empty(hi - lo, dtype=tdt, device="cuda")
    outs = [torch.empty(n // world, dtype=tdt, device="cuda")]
    sl = D.BucketPlan([(0, n, 1.0)], n, dt, local, slice_index=rank, slice_count=world)
    oplan = D.BucketPlan([(0, n // world, 1.0)], n // world, dt, local)

    def nvls_rs():  # switch-reduced reduce-scatter + gbar^2, one pass
        g.barrier()
        g.nvls_reduce_sqnorm(plan, buck, rank, 1.0 / world, out)
        g.barrier()

    def nvls_ar():  # switch-reduced all-reduce + gbar^2, one pass
        g.barrier()
        g.nvls_reduce_sqnorm(plan, buck, rank, 1.0 / world)
        g.barrier()

    def p2p_rs():
        g.barrier()
        g.reduce_scatter_sqnorm(plan, ptrs, rank, out, 1.0 / world)
        g.barrier()

    def nccl_rs_norm():  # NCCL reduce-scatter, then the K2 norm of the slice
        dist.reduce_scatter_tensor(outs[0], x)
        g.mean_sqnorm(oplan, outs[0])

    def nccl_ar_norm():
        dist.all_reduce(x, op=dist.ReduceOp.SUM)
        g.mean_sqnorm(sl, x)

    res = {"dtype": str(tdt).split(".")[-1], "bytes_per_rank": n * es, "nvls_allreduce_ms": timed(nvls),
           "nvls_allreduce_sqnorm_ms": timed(nvls_ar),
           "nvls_reduce_scatter_sqnorm_ms": timed(nvls_rs),
           "p2p_allreduce_sqnorm_ms": timed(p2p),
           "p2p_reduce_scatter_sqnorm_ms": timed(p2p_rs),
           "nccl_allreduce_ms": timed(lambda: dist.all_reduce(x, op=dist.ReduceOp.SUM)),
           "nccl_allreduce_plus_norm_ms": timed(nccl_ar_norm),
           "nccl_reduce_scatter_plus_norm_ms": timed(nccl_rs_norm)}
    sl.close()
    oplan.close()
    res["nvls_busbw_gbs"] = 2 * (world - 1) / world * n * es / (res["nvls_allreduce_ms"] / 1e3) / 1e9
    for b in bases:
        D.ipc_close(b)
    plan.close()
    g.close()
    buck.close()
    return res


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    cases = [check_case(rank, world, local, 1_000_003),
             check_case(rank, world, local, 777_216),
             check_case(rank, world, local, 4_000_000),
             check_fused(rank, world, local, 1_000_003),
             check_fused(rank, world, local, 4_000_000),
             check_bf16_refused(rank, world, local)]
    ok = all(c["ok"] for c in cases)
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    out = {"world": world, "ok": bool(t.item()), "cases": cases}
    mb = int(os.environ.get("NVLS_BENCH_MB", "0"))
    if mb:
        out["bench"] = bench(rank, world, local, mb)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if t.item() else 1


if __name__ == "__main__":
    sys.exit(main())
