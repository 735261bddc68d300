"""How does the NVSwitch round bf16 multimem.ld_reduce sums?  (torchrun,
2 or 4 GPUs; prints one JSON line from rank 0.)  Each rank fills its NVLS
bucket with bf16 values of mixed magnitude; every rank reads the whole
bucket back through ld_reduce (plain bf16 add, and .acc::f32) and compares
with RNE(exact sum) and with RNE(fp32 sum in replica order), the reference
the P2P reduce-scatter/all-reduce kernels match.  Measurement tool for
DESIGN §4 (why the NVLS form is fp32-only or not)."""
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26687_b200 import device as D  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    so = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_nvls_bf16_probe.so"))
    so.nvls_bf16_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
    n = 1 << 24
    torch.manual_seed(1234 + rank)
    buck = D.NvlsBucket(n, torch.bfloat16, rank, world, dist, local)
    x = (torch.randn(n, device="cuda") * torch.exp2(torch.randint(-6, 7, (n,), device="cuda").float()))
    x = x.to(torch.bfloat16)
    buck.tensor.copy_(x)
    allx = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(allx, x)
    exact = sum(a.double() for a in allx)
    rne_exact = exact.to(torch.bfloat16)  # double -> bf16 is RNE; the double sum is exact here
    acc = allx[0].float()
    for q in range(1, world):
        acc = acc + allx[q].float()
    rne_p2p = acc.to(torch.bfloat16)
    torch.cuda.synchronize()
    dist.barrier()
    res = {"world": world, "numel": n}
    for mode, name in ((0, "bf16_add"), (1, "acc_f32")):
        out = torch.empty_like(x)
        rc = so.nvls_bf16_probe(C.c_void_p(buck.multicast), C.c_void_p(out.data_ptr()), n // 8, mode,
                                C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        got = out.double()
        ne = (out != rne_exact)
        nm = int(ne.sum())
        up = int(((got > rne_exact.double()) & ne).sum())
        g2 = float((got ** 2).sum())
        g2r = float((rne_exact.double() ** 2).sum())
        # is the off-RNE result the truncation of the exact sum?
        trunc = int((ne & (got.abs() < exact.abs())).sum())
        res[name] = {"rc": rc, "mismatch_vs_rne_exact": nm / n, "above": up, "below": nm - up,
                     "toward_zero": trunc,
                     "mismatch_vs_rne_fp32_replica_order": int((out != rne_p2p).sum()) / n,
                     "gbar2_rel_bias": (g2 - g2r) / g2r}
    if rank == 0:
        print(json.dumps(res), flush=True)
    buck.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
