"""Stress of the NVLink slot exchange (the N > 1 default): every rank runs
STEPS small steps whose last reduction carries the exchange + finalize
(coadapt_gns_fused_sqnorm_finalize with mailboxes) — alternating with the
standalone exchange kernel — with random host-side delays before each launch
so ranks arrive in every order, fresh data every step.  Every step's slots are
checked against the sum of all ranks' local slots (gathered over gloo) and
phi against rank 0's (bit-identical).  Launch with torch.distributed.run.
Prints one JSON line on rank 0; exit 1 on any mismatch."""
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402
from paper_2604_26687_b200 import dist as Dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    steps = int(os.environ.get("STEPS", "2000"))
    M, n = 4, 300_000
    bufs = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, dev)
    g = D.GnsDevice(1, M, M, dev)          # the exchange under test
    loc = D.GnsDevice(1, M, M, dev)        # this rank's local slots, no exchange
    bases = Dist.attach_p2p(g, dist, world, rank)
    rng = random.Random(1000 + rank)
    bad = 0
    t0 = time.time()
    for k in range(steps):
        for m in range(M):
            D.synth_fill(bufs[m], [(0, n, 0, n, n)], 77 + k, rank * M + m, 2.0 ** -10, 1e-4)
        loc.begin_step()
        loc.fused_sqnorm(plan, bufs)
        local = loc.partials()
        time.sleep(rng.random() * 2e-3)  # arrive in every order
        g.begin_step()
        if k % 2 == 0:
            g.fused_sqnorm_finalize(plan, bufs, M * 2048)
        else:
            g.fused_sqnorm(plan, bufs)
            g.allreduce_finalize_p2p(M * 2048)
        r = g.result()
        got = g.partials()
        allp = [None] * world
        dist.all_gather_object(allp, (local.tolist(), r.status, r.phi))
        want = np.sum([np.array(x[0]) for x in allp], axis=0)  # rank-order sum
        phis = {repr(x[2]) for x in allp}  # (nan while phi is unavailable)
        if r.status != 0 or not np.allclose(got, want, rtol=1e-14, atol=0) or len(phis) != 1:
            if bad < 3 and rank == 0:
                print(json.dumps({"step": k, "form": "in-pass" if k % 2 == 0 else "standalone",
                                  "status": r.status, "got": got.tolist()[:3] + got.tolist()[-1:],
                                  "want": want.tolist()[:3] + want.tolist()[-1:],
                                  "phis": sorted(str(x) for x in phis)}), flush=True)
            bad += 1
    torch.cuda.synchronize()
    dist.barrier()
    for b in bases:
        D.ipc_close(b)
    tot = torch.tensor([bad])
    dist.all_reduce(tot)
    if rank == 0:
        print(json.dumps({"world": world, "gpus": torch.cuda.device_count(), "steps": steps,
                          "mismatched_steps": int(tot.item()), "seconds": round(time.time() - t0, 1),
                          "ok": int(tot.item()) == 0}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if tot.item() == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
