"""Two-rank run of the NVLink slot exchange for compute-sanitizer: the
standalone X1 + K3 kernel (coadapt_gns_allreduce_finalize_p2p) and the same
exchange inside the last reduction's last CTA (coadapt_gns_fused_sqnorm_
finalize with mailboxes attached).  Launch with torch.distributed.run
--nproc-per-node 2 under `compute-sanitizer --target-processes all`."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402
from paper_2604_26687_b200 import dist as Dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    n, M = 100_000, 4
    bufs = []
    for m in range(M):
        t = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        D.synth_fill(t, [(0, n, 0, n, n)], 5, rank * M + m, 2.0 ** -10, 1e-4)
        bufs.append(t)
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, torch.cuda.current_device())
    g = D.GnsDevice(1, M, M, torch.cuda.current_device())
    bases = Dist.attach_p2p(g, dist, world, rank)
    ok = True
    for step in range(3):
        g.begin_step()
        g.fused_sqnorm(plan, bufs)
        g.allreduce_finalize_p2p(M * 2048)
        r1 = g.result()
        g.begin_step()
        g.fused_sqnorm_finalize(plan, bufs, M * 2048)
        r2 = g.result()
        ok = ok and r1.status == 0 and r2.status == 0 and math.isfinite(r2.b_simple)
    torch.cuda.synchronize()
    dist.barrier()
    for b in bases:
        D.ipc_close(b)
    print(f"rank {rank}: sanitize p2p", "ok" if ok else "FAILED", flush=True)
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
