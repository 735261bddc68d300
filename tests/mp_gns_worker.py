"""Multi-GPU worker (launched with torch.distributed.run, one process per GPU).

Each physical rank reduces the buckets of its block of the job's d*t*p
virtual ranks into its GnsDevice slots, the library's NCCL communicator
all-reduces the N+1 scalars, and every rank finalizes.  Rank 0 then
recomputes the whole job alone on its GPU (no NCCL) and checks that the
all-reduced slots and the step result agree.  Prints one JSON line on rank 0.
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
from paper_2604_26687_b200 import layout as Lay  # noqa: E402


def run_job(g, lays, ranks, M, d, seed, unit, fused, final_tokens=None):
    """final_tokens: the rank's last reduction carries the finalize (and the
    NVLink slot exchange) in its last CTA (coadapt_gns_*_finalize)."""
    g.begin_step()
    for k, vr in enumerate(ranks):
        last = final_tokens is not None and k + 1 == len(ranks)
        lay = lays[vr]
        i_d = lay.coords[0]
        plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, torch.cuda.current_device())
        bufs = []
        for m in range(M):
            b = torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda")
            D.synth_fill(b, lay.gen, seed, i_d * M + m, Lay.G0, unit)
            bufs.append(b)
        if fused:
            if last:
                g.fused_sqnorm_finalize(plan, bufs, final_tokens)
            else:
                g.fused_sqnorm(plan, bufs)
        else:
            g.micro_sqnorm_batched(plan, bufs, [i_d] * M, list(range(M)))
            mean = torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda")
            D.synth_mean_fill(mean, lay.gen, seed, 0, d * M, Lay.G0, unit)
            sl = D.BucketPlan(lay.segments, lay.numel, L.BF16, torch.cuda.current_device(),
                              slice_index=i_d, slice_count=d)
            if last:
                g.mean_sqnorm_finalize(sl, mean, final_tokens)
            else:
                g.mean_sqnorm(sl, mean)


def graph_p2p_case(lays, mine, M, d, unit, local, world, rank):
    """X1 + K3 over NVLink captured in a CUDA graph (no eager warm-up: the
    plans built their tables at creation) and replayed on fresh data each
    step: every replay must move to the next mailbox epoch, so its phi and
    slots equal an eager NCCL step on the same data."""
    gg = D.GnsDevice(d, M, d * M, local)
    bases = Dist.attach_p2p(gg, dist, world, rank)
    ge = D.GnsDevice(d, M, d * M, local)
    Dist.attach(ge, dist, world, rank)
    s = torch.cuda.Stream()
    bufs = {vr: [torch.empty(lays[vr].numel, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
            for vr in mine}
    plans = {vr: D.BucketPlan(lays[vr].segments, lays[vr].numel, L.BF16, local) for vr in mine}

    def fill(k):
        for vr in mine:
            i_d = lays[vr].coords[0]
            for m in range(M):
                D.synth_fill(bufs[vr][m], lays[vr].gen, 0xC0905 + k, i_d * M + m, Lay.G0, unit, s)

    def body(g):
        g.begin_step(s)
        for vr in mine:
            i_d = lays[vr].coords[0]
            g.micro_sqnorm_batched(plans[vr], bufs[vr], [i_d] * M, list(range(M)), s)
            # the d > 1 mean term is not part of this check: K1 slots only
    tokens = d * M * 2048
    torch.cuda.synchronize()
    dist.barrier()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        body(gg)
        gg.allreduce_finalize_p2p(tokens, s)
    good, worst = True, 0.0
    for k in range(1, 5):
        with torch.cuda.stream(s):
            fill(k)
            graph.replay()
        rg = gg.result()
        pg = gg.partials()
        body(ge)
        ge.allreduce(s)
        ge.finalize(tokens, s)
        re = ge.result()
        pe = ge.partials()
        rel = float(np.max(np.abs(pg[:-1] - pe[:-1]) / np.abs(pe[:-1])))
        worst = max(worst, rel)
        good = good and rg.status == 0 and rel <= 1e-13 and \
            abs(rg.state.ema_signal - re.state.ema_signal) <= 1e-12 * abs(re.state.ema_signal) and \
            rg.state.tokens_seen == re.state.tokens_seen == k * tokens
    torch.cuda.synchronize()
    dist.barrier()
    for b in bases:
        D.ipc_close(b)
    return {"graph_p2p_replays": 4, "graph_p2p_max_rel_slots": worst, "graph_p2p_ok": bool(good)}


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    spec = Lay.tiny_model(layers=4, h=128, ffn=256, vocab=512, tied=True)
    unit = Lay.noise_unit_for(256.0, 1)
    report = {"world": world, "cases": []}
    ok = True
    for (d, t, p, M, fused) in [(2, 2, 2, 4, False), (1, 4, 2, 4, True), (8, 1, 1, 2, False)]:
        R = d * t * p
        lays = Lay.world_layouts(spec, d, t, p)
        mine = Dist.block_map(R, world, rank)
        g = D.GnsDevice(d, M, d * M, local)
        Dist.attach(g, dist, world, rank)
        run_job(g, lays, mine, M, d, 0xC0905, unit, fused)
        g.allreduce()
        g.finalize(d * M * 2048)
        r = g.result()
        parts = g.partials()
        dist.barrier()
        case = {"dtp": [d, t, p], "M": M, "fused": fused}
        if rank == 0:
            ref = D.GnsDevice(d, M, d * M, local)
            run_job(ref, lays, list(range(R)), M, d, 0xC0905, unit, fused)
            ref.finalize(d * M * 2048)
            rr = ref.result()
            rp = ref.partials()
            rel = float(np.max(np.abs(parts - rp) / np.maximum(np.abs(rp), 1e-300)))
            case.update({"max_rel_slots": rel, "phi": r.phi, "phi_ref": rr.phi,
                         "b_simple_rel": abs(r.b_simple - rr.b_simple) / abs(rr.b_simple)})
            ok = ok and rel <= 1e-12 and case["b_simple_rel"] <= 1e-10
        # every rank finalized the same all-reduced slots
        t_phi = torch.tensor([r.phi], dtype=torch.float64, device="cuda")
        lo, hi = t_phi.clone(), t_phi.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        case["phi_identical_on_all_ranks"] = bool(lo.item() == hi.item())
        ok = ok and case["phi_identical_on_all_ranks"]
        # the same step with X1 + K3 fused into one kernel over NVLink
        g2 = D.GnsDevice(d, M, d * M, local)
        bases = Dist.attach_p2p(g2, dist, world, rank)
        run_job(g2, lays, mine, M, d, 0xC0905, unit, fused)
        g2.allreduce_finalize_p2p(d * M * 2048)
        r2 = g2.result()
        p2 = g2.partials()
        case["p2p_max_rel_slots_vs_nccl"] = float(np.max(np.abs(p2 - parts) /
                                                         np.maximum(np.abs(parts), 1e-300)))
        case["p2p_b_simple_rel"] = abs(r2.b_simple - r.b_simple) / abs(r.b_simple)
        t2 = torch.tensor([r2.phi], dtype=torch.float64, device="cuda")
        lo2, hi2 = t2.clone(), t2.clone()
        dist.all_reduce(lo2, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi2, op=dist.ReduceOp.MAX)
        case["p2p_phi_identical_on_all_ranks"] = bool(lo2.item() == hi2.item())
        ok = ok and case["p2p_max_rel_slots_vs_nccl"] <= 1e-14 and \
            case["p2p_phi_identical_on_all_ranks"] and case["p2p_b_simple_rel"] <= 1e-12
        # the slot exchange + finalize inside the last reduction's last CTA
        g3 = D.GnsDevice(d, M, d * M, local)
        bases3 = Dist.attach_p2p(g3, dist, world, rank)
        run_job(g3, lays, mine, M, d, 0xC0905, unit, fused, final_tokens=d * M * 2048)
        r3 = g3.result()
        p3 = g3.partials()
        case["inpass_max_rel_slots_vs_nccl"] = float(np.max(np.abs(p3 - parts) /
                                                            np.maximum(np.abs(parts), 1e-300)))
        case["inpass_b_simple_rel"] = abs(r3.b_simple - r.b_simple) / abs(r.b_simple)
        case["inpass_bitwise_vs_p2p_kernel"] = bool(np.array_equal(p3, p2) and
                                                    r3.b_simple == r2.b_simple)
        ok = ok and r3.status == 0 and case["inpass_max_rel_slots_vs_nccl"] <= 1e-14 and \
            case["inpass_bitwise_vs_p2p_kernel"]
        torch.cuda.synchronize()
        dist.barrier()
        for b in bases3:
            D.ipc_close(b)
        g3.close()
        # tail latency: NCCL all-reduce + finalize vs the fused P2P kernel
        s = torch.cuda.current_stream()
        for name, fn in (("nccl", lambda: (g.allreduce(), g.finalize(1))),
                         ("p2p", lambda: g2.allreduce_finalize_p2p(1))):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(50):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            case[f"tail_us_{name}"] = e0.elapsed_time(e1) / 50 * 1e3
        dist.barrier()
        if (d, t, p) == (2, 2, 2):
            case.update(graph_p2p_case(lays, mine, M, d, unit, local, world, rank))
            ok = ok and case["graph_p2p_ok"]
        for b in bases:
            D.ipc_close(b)
        report["cases"].append(case)
        g.close()
    report["ok"] = bool(ok)
    if rank == 0:
        print(json.dumps(report), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
