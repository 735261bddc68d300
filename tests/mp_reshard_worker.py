"""Multi-GPU worker for reshard execution over NVLink,
launched with torch.distributed.run (one process per GPU, world = d*t*p of
both layouts).

Every rank fills its source pack from the deterministic global tensors,
publishes a CUDA IPC handle, maps the peers' packs and pulls its destination
pack with coadapt_reshard_execute(dst_rank = rank).  Checks (rank 0 prints
one JSON line): every destination pack equals the oracle's pack built from
the global tensors; and, for a larger TP -> PP transition, the pull
bandwidth per GPU (wire bytes received / kernel time, CUDA events).
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import reshard_oracle as O  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402
from paper_2604_26687_b200 import reshard as R  # noqa: E402


def to_oracle(m):
    return O.Model(m.layers, [O.Tensor(t.name, tuple(t.shape), t.tp_axis) for t in m.per_layer],
                   m.optimizer_state_multiplier, m.param_bytes, m.state_bytes)


def strategies(n, layers):
    return [(d, t, p) for d in range(1, n + 1) for t in range(1, n + 1) for p in range(1, n + 1)
            if d * t * p == n and layers % p == 0]


def map_peers(rank, world, mine, local):
    handles = [None] * world
    dist.all_gather_object(handles, D.ipc_handle(mine))
    ptrs, bases = [], []
    for q in range(world):
        if q == rank:
            ptrs.append(mine.data_ptr())
        else:
            p, b = D.ipc_open(handles[q], local)
            ptrs.append(p)
            bases.append(b)
    return ptrs, bases


def run_case(rank, world, local, m, a, b, dt, policy="canonical", timed=False):
    om = to_oracle(m)
    la, lb = O.layout_for(om, a), O.layout_for(om, b)
    p = R.plan_transfers(m, a, b, policy)
    es = np.dtype(dt).itemsize
    if timed:  # big: fill on device, verify by the round trip
        g = torch.Generator(device="cuda").manual_seed(rank)
        src = torch.randint(-32768, 32767, (la.pack_numel[rank],), dtype=torch.int16,
                            device="cuda", generator=g)
        want = None
    else:
        st = O.global_state(om, 3, dt)
        src = torch.from_numpy(O.pack_from_global(la, rank, st, dt)).cuda()
        want = O.pack_from_global(lb, rank, st, dt)
    dst = torch.zeros(lb.pack_numel[rank], dtype=src.dtype, device="cuda")
    ptrs, bases = map_peers(rank, world, src, local)
    torch.cuda.synchronize()
    dist.barrier()
    res = {}
    if timed:
        recv = sum(x.bytes for x in p.moves() if x.dst_rank == rank and not x.local)
        wire = recv // m.bytes_per_element * es  # this plane's wire bytes
        s = torch.cuda.current_stream()
        for _ in range(3):
            p.execute(ptrs, [dst if r == rank else None for r in range(world)], dst_rank=rank)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(s)
        for _ in range(reps):
            p.execute(ptrs, [dst if r == rank else None for r in range(world)], dst_rank=rank)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res = {"ms": ms, "wire_bytes": wire, "pack_bytes": dst.numel() * es,
               "wire_gbs": wire / ms / 1e6, "pack_gbs": dst.numel() * es / ms / 1e6}
        # round trip back into a fresh source-layout pack and compare
        back = R.plan_transfers(m, b, a, policy)
        dptrs, dbases = map_peers(rank, world, dst, local)
        again = torch.zeros_like(src)
        torch.cuda.synchronize()
        dist.barrier()
        back.execute(dptrs, [again if r == rank else None for r in range(world)], dst_rank=rank)
        torch.cuda.synchronize()
        dist.barrier()
        mask = torch.zeros(src.numel(), dtype=torch.bool, device="cuda")
        for sh in la.shards:
            if sh.owner == rank:
                mask[sh.pack_offset:sh.pack_offset + sh.numel] = True
        res["ok"] = bool(torch.equal(again[mask], src[mask]))
        for x in dbases:
            D.ipc_close(x)
    else:
        p.execute(ptrs, [dst if r == rank else None for r in range(world)], dst_rank=rank)
        torch.cuda.synchronize()
        res["ok"] = bool(np.array_equal(dst.cpu().numpy(), want))
    dist.barrier()
    for x in bases:
        D.ipc_close(x)
    return res


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    import random
    rng = random.Random(42)
    T = R.TensorDecl
    cases = []
    small = R.ModelSpec(4, (T("w", (64, 48), 0), T("o", (48, 64), 1), T("n", (48,)), T("e", (8, 6, 16), 2)))
    ss = strategies(world, small.layers)
    for a in ss:
        for b in ss:
            for dt in (np.int16, np.float32):
                pol = rng.choice(["canonical", "spread"])
                r = run_case(rank, world, local, small, a, b, dt, pol)
                cases.append({"src": a, "dst": b, "es": np.dtype(dt).itemsize, "ok": r["ok"]})
    # bandwidth: TP across all GPUs -> PP across all GPUs (each rank pulls
    # (world-1)/world of its new stage from the peers)
    big = R.ModelSpec(world * 2, (T("w", (8192, 8192), 0), T("o", (8192, 8192), 1)))
    timed = run_case(rank, world, local, big, (1, world, 1), (1, 1, world), np.int16, timed=True)
    oks = [None] * world
    dist.all_gather_object(oks, (all(c["ok"] for c in cases), timed))
    if rank == 0:
        ok = all(o[0] and o[1]["ok"] for o in oks)
        print(json.dumps({"ok": ok, "world": world, "cases": len(cases),
                          "failed": [c for c in cases if not c["ok"]][:5],
                          "bandwidth": [o[1] for o in oks]}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
