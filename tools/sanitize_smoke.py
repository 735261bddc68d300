"""Small invocations of every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck):  K0 synth + mean, K1 (aligned, unaligned,
segmented, batched), K1f TMA + LDG fallback, host streaming, mean slice,
finalize, read probe, L2 flush.  Exits 0 when all results are finite."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n = 70_001
    gen = [(0, n, 0, n, n)]
    segs = [(0, 1000, 1.0), (1000, 37, 0.0), (1037, 5, 0.5), (1042, n - 1042, 1.0)]
    bufs = []
    for m in range(4):
        raw = torch.zeros(n + 16, dtype=torch.bfloat16, device="cuda")
        D.synth_fill(raw[:n], gen, 1, m, 2.0 ** -10, 1e-4)
        bufs.append(raw)
    mean = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    D.synth_mean_fill(mean, gen, 1, 0, 4, 2.0 ** -10, 1e-4)
    plan = D.BucketPlan(segs, n, L.BF16, 0)
    sl = D.BucketPlan(segs, n, L.BF16, 0, slice_index=1, slice_count=2)
    g = D.GnsDevice(1, 4, 4, 0)
    g.begin_step()
    g.fused_sqnorm(plan, [b[:n] for b in bufs])                 # TMA
    g.fused_sqnorm(plan, [b[1:n + 1] for b in bufs])            # LDG fallback
    host = [b[:n].cpu().pin_memory() for b in bufs]
    g.fused_sqnorm_host(plan, host)                              # host streaming
    g.finalize(4096)
    r = g.result()
    g2 = D.GnsDevice(2, 2, 4, 0)
    g2.begin_step()
    g2.micro_sqnorm_batched(plan, [b[:n] for b in bufs], [0, 0, 1, 1], [0, 1, 0, 1])
    g2.micro_sqnorm(plan, bufs[0][3:n + 3], 1, 1)               # unaligned
    g2.mean_sqnorm(sl, mean)
    g2.finalize(4096)
    r2 = g2.result()
    x = torch.randn(3, dtype=torch.float64, device="cuda")
    v = D.sqnorm(x)
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    D.read_probe(bufs[0], sink)
    D.l2_flush(torch.empty(1 << 20, dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    ok = all(math.isfinite(t) for t in (r.phi if r.phi_available else 0.0, r2.b_simple, v))
    print("sanitize smoke", "ok" if ok else "FAILED", r.b_simple, r2.b_simple, v)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
