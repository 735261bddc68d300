"""Multi-GPU worker for reshard execution over NVLink,
launched with torch.distributed.run (one process per GPU, world = d*t*p of
both layouts).

Every rank fills its source pack from the deterministic global tensors and
publishes a CUDA IPC handle; in pull mode it maps the peers' source packs
and copies its destination pack (role PULL, rank = itself), in push mode it
maps the peers' destination packs and writes its source regions into them
(role PUSH).  Checks (rank 0 prints one JSON line): every destination pack
equals the oracle's pack built from the global tensors, for every strategy
pair of the world size, both modes; and, for a larger TP -> PP transition,
the copy bandwidth per GPU (CUDA events) in both modes, with a round trip
back to the source layout.
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


def run_case(rank, world, local, m, a, b, dt, policy="canonical", timed=False, mode="pull"):
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

    def go(plan, s_t, d_t, s_list, d_list):
        if mode == "pull":
            plan.execute(s_list, [d_t if r == rank else None for r in range(world)], dst_rank=rank)
        else:
            plan.execute([s_t if r == rank else None for r in range(world)], d_list, src_rank=rank)

    # pull maps the peers' sources, push the peers' destinations
    ptrs, bases = map_peers(rank, world, src if mode == "pull" else dst, local)
    sl = ptrs if mode == "pull" else None
    dl = ptrs if mode == "push" else None
    torch.cuda.synchronize()
    dist.barrier()
    res = {"mode": mode}
    if timed:
        moves = p.moves()
        mine = [x for x in moves if (x.dst_rank if mode == "pull" else x.src_rank) == rank]
        wire = sum(x.bytes for x in mine if not x.local) // m.bytes_per_element * es
        total = sum(x.bytes for x in mine) // m.bytes_per_element * es
        s = torch.cuda.current_stream()
        for _ in range(3):
            go(p, src, dst, sl, dl)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(s)
        for _ in range(reps):
            go(p, src, dst, sl, dl)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res.update({"ms": ms, "wire_bytes": wire, "bytes": total,
                    "wire_gbs": wire / ms / 1e6, "gbs": total / ms / 1e6})
        dist.barrier()
        # round trip back into a fresh source-layout pack (pulled) and compare
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
        go(p, src, dst, sl, dl)
        torch.cuda.synchronize()
        dist.barrier()  # push: peers write into this rank's dst
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
                for mode in ("pull", "push"):
                    r = run_case(rank, world, local, small, a, b, dt, pol, mode=mode)
                    cases.append({"src": a, "dst": b, "es": np.dtype(dt).itemsize, "mode": mode,
                                  "ok": r["ok"]})
    # bandwidth: TP across all GPUs -> PP across all GPUs (each rank pulls
    # (world-1)/world of its new stage from the peers)
    big = R.ModelSpec(world * 2, (T("w", (8192, 8192), 0), T("o", (8192, 8192), 1)))
    timed = [run_case(rank, world, local, big, (1, world, 1), (1, 1, world), np.int16, timed=True,
                      mode=mode) for mode in ("pull", "push")]
    oks = [None] * world
    dist.all_gather_object(oks, (all(c["ok"] for c in cases), timed))
    if rank == 0:
        ok = all(o[0] and all(t["ok"] for t in o[1]) for o in oks)
        print(json.dumps({"ok": ok, "world": world, "cases": len(cases),
                          "failed": [c for c in cases if not c["ok"]][:5],
                          "bandwidth": [o[1] for o in oks]}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
