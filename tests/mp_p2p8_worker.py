"""Eight-rank NVLink slot exchange on whatever GPUs the box has (gpurun offers
at most 4, the driver's scaling run uses 8): 8 processes over the available
GPUs (2 or 4 per GPU, CUDA IPC between processes on one device works the same
as across devices), torch.distributed over gloo for the plumbing (NCCL
refuses two ranks on one GPU).  Job: a small Qwen-like model at (1,4,2),
M = 4, one virtual rank per process.  Every rank runs 3 steps with the
exchange + finalize inside its last reduction (mailboxes of 8 peers) and one
with the standalone exchange kernel; rank 0 recomputes the whole job alone
and checks slots and phi.  Prints one JSON line on rank 0."""
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


def fill(lay, M, seed, unit):
    bufs = []
    for m in range(M):
        b = torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda")
        D.synth_fill(b, lay.gen, seed, m, Lay.G0, unit)
        bufs.append(b)
    return bufs


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    spec = Lay.tiny_model(layers=4, h=256, ffn=512, vocab=1024)
    d, t, p, M = 1, 4, 2, 4
    lays = Lay.world_layouts(spec, d, t, p)
    assert len(lays) == world == 8
    unit = Lay.noise_unit_for(256.0, 1)
    lay = lays[rank]
    plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, dev)
    g = D.GnsDevice(d, M, d * M, dev)
    bases = Dist.attach_p2p(g, dist, world, rank)
    rep = {"world": world, "gpus": torch.cuda.device_count(), "steps": []}
    ok = True
    ref_state = None
    for step in range(4):
        bufs = fill(lay, M, 0x88 + step, unit)
        g.begin_step()
        if step < 3:
            g.fused_sqnorm_finalize(plan, bufs, d * M * 2048)
        else:
            g.fused_sqnorm(plan, bufs)
            g.allreduce_finalize_p2p(d * M * 2048)
        r = g.result()
        parts = g.partials()
        phis = [None] * world
        dist.all_gather_object(phis, (r.status, r.phi, r.b_simple))
        if rank == 0:
            ref = D.GnsDevice(d, M, d * M, dev)
            if ref_state is not None:
                ref.set_state(ref_state)  # the EMA continues across steps
            ref.begin_step()
            for vr in range(world):
                ref.fused_sqnorm(D.BucketPlan(lays[vr].segments, lays[vr].numel, L.BF16, dev),
                                 fill(lays[vr], M, 0x88 + step, unit))
            ref.finalize(d * M * 2048)
            rr = ref.result()
            ref_state = ref.get_state()
            rel = float(np.max(np.abs(parts - ref.partials()) / np.abs(ref.partials())))
            same_bits = all(x == phis[0] for x in phis)
            rep["steps"].append({"form": "in-pass" if step < 3 else "standalone",
                                 "max_rel_slots": rel, "phi": r.phi,
                                 "phi_ref": rr.phi, "identical_on_all_ranks": same_bits})
            ok = ok and rel <= 1e-13 and same_bits and all(s == 0 for s, _, _ in phis) and \
                abs(r.b_simple - rr.b_simple) <= 1e-12 * abs(rr.b_simple)
            ref.close()
        dist.barrier()
    torch.cuda.synchronize()
    dist.barrier()
    for b in bases:
        D.ipc_close(b)
    rep["ok"] = bool(ok)
    if rank == 0:
        print(json.dumps(rep), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
