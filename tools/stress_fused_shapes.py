"""Flake hunt for the fused TMA ring at every shape in use: for each M, the
fused pass is repeated many times over the same buckets; every repetition must
give bit-identical s_m / gbar^2 (a ring race shows up as a changed bit) and
s_m must equal the separate K1 passes to 1e-12.
    python tools/stress_fused_shapes.py [reps] [elems_per_bucket]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n = int(sys.argv[2]) if len(sys.argv) > 2 else (24 << 20) + 12345
torch.cuda.set_device(0)
segs = [(0, 1000, 1.0), (1000, 5000, 0.0), (6000, n // 2, 1.0), (6000 + n // 2, n - 6000 - n // 2, 0.5)]
bad = 0
for M in (2, 3, 4, 7, 8, 10, 11, 12, 15, 16):
    bufs = []
    for m in range(M):
        b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        D.synth_fill(b, [(0, n, 0, n, n)], 5, m, 2.0 ** -10, 1e-4)
        bufs.append(b)
    plan = D.BucketPlan(segs, n, L.BF16, 0)
    sep = D.GnsDevice(1, M, M, 0) if M >= 2 else None
    sep.begin_step()
    for m in range(M):
        sep.micro_sqnorm(plan, bufs[m], 0, m)
    ref = sep.partials()[:M]
    g = D.GnsDevice(1, M, M, 0)
    first = None
    for r in range(reps):
        g.begin_step()
        g.fused_sqnorm(plan, bufs)
        p = g.partials()
        if first is None:
            first = p.copy()
            if not np.allclose(p[:M], ref, rtol=1e-12, atol=0):
                bad += 1
                print("M", M, "fused != separate", p[:M], ref, flush=True)
        elif not np.array_equal(p, first):
            bad += 1
            print("M", M, "rep", r, "nondeterministic", flush=True)
    print("M", M, "ok" if bad == 0 else f"bad={bad}", flush=True)
    g.close()
    sep.close()
    plan.close()
    del bufs
    torch.cuda.empty_cache()
print("total bad", bad)
sys.exit(1 if bad else 0)
