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
    # K1f at M = 16 (shape 5, both consumer groups: >= 2 chunks per CTA),
    # the batched K1 ring over 16 buckets, the in-pass finalize, KA
    n16 = 1792 * 2 * 148 + 999
    segs16 = [(0, 5000, 1.0), (5000, 4096, 0.0), (9096, n16 - 9096, 1.0)]
    b16 = []
    for m in range(16):
        t = torch.empty(n16, dtype=torch.bfloat16, device="cuda")
        D.synth_fill(t, [(0, n16, 0, n16, n16)], 2, m, 2.0 ** -10, 1e-4)
        b16.append(t)
    p16 = D.BucketPlan(segs16, n16, L.BF16, 0)
    g16 = D.GnsDevice(1, 16, 16, 0)
    g16.begin_step()
    g16.fused_sqnorm(p16, b16)
    g16.fused_sqnorm_finalize(p16, b16, 16 * 2048)
    r16 = g16.result()
    gb = D.GnsDevice(2, 16, 32, 0)
    gb.begin_step()
    gb.micro_sqnorm_batched(p16, b16, [1] * 16, list(range(16)))
    gb.finalize(32 * 2048)
    rb = gb.result()
    ga = D.GnsDevice(1, 4, 4, 0)
    ga.begin_step()
    main_grad = torch.zeros(n16, dtype=torch.float32, device="cuda")
    for m in range(4):
        ga.accumulate(p16, main_grad, b16[m], 0, m, first=m == 0, last_mean=m == 3)
    ga.finalize(4 * 2048)
    ga.result()
    x = torch.randn(3, dtype=torch.float64, device="cuda")
    v = D.sqnorm(x)
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    D.read_probe(bufs[0], sink)
    D.l2_flush(torch.empty(1 << 20, dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()
    ok = all(math.isfinite(t) for t in (r.phi if r.phi_available else 0.0, r2.b_simple, v,
                                        r16.b_simple, rb.b_simple))
    print("sanitize smoke", "ok" if ok else "FAILED", r.b_simple, r2.b_simple, v, r16.b_simple,
          rb.b_simple)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
