"""Multi-GPU worker: GnsManager with main_grad in NVLS memory (f1 + f2):
every DP rank runs M micro-batches of its own data through the same model;
finish_step all-reduces main_grad through the NVSwitch and takes gbar^2 of
its slice.  Checks (rank 0 prints one JSON line): main_grad on every rank
equals the DP mean of the torch references (bit-exact on 2 GPUs, within the
d-term fp32 rounding bound otherwise), the all-reduced s_m equal each rank's
torch fp64 norms, gbar^2 equals the fp64 norm of the synchronised mean / M^2,
and every rank finalizes to the same phi bits."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2604_26687_b200 import dist as Dist  # noqa: E402
from paper_2604_26687_b200.trainer import GnsManager  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    M = 3
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.GELU(),
                                torch.nn.Linear(512, 256)).cuda().to(torch.bfloat16)
    gen = torch.Generator(device="cuda").manual_seed(100 + rank)
    xs = [torch.randn(8, 256, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(M)]
    ys = [torch.randn(8, 256, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(M)]
    params = list(model.parameters())
    # torch reference: per-micro grads, fp32 accumulation in micro order
    grads = [torch.autograd.grad(torch.nn.functional.mse_loss(model(x).float(), y.float()), params)
             for x, y in zip(xs, ys)]
    s_mine = [sum(float((g.double() ** 2).sum()) for g in gm) for gm in grads]
    main_ref = [torch.zeros_like(p, dtype=torch.float32) for p in params]
    for gm in grads:
        for a, g in zip(main_ref, gm):
            a.add_(g)
    mgr = GnsManager(params, micro_count=M, global_batch=world * M * 8, dp_size=world,
                     dp_rank=rank, nvls_dist=dist)
    Dist.attach(mgr.gns, dist, world, rank)
    mgr.begin_step()
    for x, y in zip(xs, ys):
        torch.nn.functional.mse_loss(model(x).float(), y.float()).backward()
        mgr.after_backward()
    flat_mine = torch.zeros(mgr.numel, dtype=torch.float32, device="cuda")
    for (o, n), a in zip(mgr._slots, main_ref):
        flat_mine[o:o + n] = a.reshape(-1)
    r = mgr.finish_step(tokens=world * M * 8 * 2048)
    torch.cuda.synchronize()
    allm = [torch.empty_like(flat_mine) for _ in range(world)]
    dist.all_gather(allm, flat_mine)
    acc, mag = allm[0].clone(), allm[0].abs()
    for q in range(1, world):
        acc.add_(allm[q])
        mag.add_(allm[q].abs())
    mean_ref = acc * (1.0 / world)
    if world == 2:
        main_ok = bool(torch.equal(mgr.main_grad, mean_ref))
    else:
        main_ok = bool(((mgr.main_grad - mean_ref).abs() <= (world - 1) * 2.0 ** -24 * mag / world).all())
    s_all = [None] * world
    dist.all_gather_object(s_all, s_mine)
    s_ref = np.array([v for q in range(world) for v in s_all[q]])
    parts = mgr.gns.partials()
    s_ok = bool(np.allclose(parts[:-1], s_ref, rtol=1e-12, atol=0))
    g2_ref = float((mean_ref.double() ** 2).sum()) / M ** 2
    g2_rel = abs(parts[-1] - g2_ref) / g2_ref
    phis = [None] * world
    dist.all_gather_object(phis, (r.stats.signal, r.stats.noise, r.phi, r.b_simple))
    same_phi = all(p == phis[0] for p in phis)
    ok = main_ok and s_ok and g2_rel <= (1e-12 if world == 2 else 1e-9) and same_phi
    t = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"world": world, "ok": bool(t.item()), "main_grad_ok": main_ok, "s_ok": s_ok,
                          "gbar2_rel": g2_rel, "same_phi_on_all_ranks": same_phi}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if t.item() else 1


if __name__ == "__main__":
    sys.exit(main())
