"""Repeat the fused device pass and the host-streaming pass many times on the
same data and report deviations from the first device result (race hunt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_26687_b200 import _lib as L  # noqa: E402
from paper_2604_26687_b200 import device as D  # noqa: E402

torch.cuda.set_device(0)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
numel = (16 << 20) + 12_345
segs = [(0, 1000, 1.0), (1000, 5000, 0.0), (6000, 8_000_000, 1.0),
        (8_006_000, 3, 0.5), (8_006_003, numel - 8_006_003, 1.0)]
gen = [(0, numel, 3, numel, numel)]
bufs = []
for m in range(M):
    b = torch.zeros(numel + 16, dtype=torch.bfloat16, device="cuda")
    D.synth_fill(b[:numel], gen, 5, m, 2 ** -10, 1e-4)
    bufs.append(b[:numel])
host = [b.cpu().pin_memory() for b in bufs]
plan = D.BucketPlan(segs, numel, L.BF16, 0)
ref = {}
bad = {"dev": 0, "host": 0}
cross = 0.0
for r in range(reps):
    for kind in ("dev", "host"):
        g = D.GnsDevice(1, M, M, 0)
        g.begin_step()
        if kind == "dev":
            g.fused_sqnorm(plan, bufs)
        else:
            g.fused_sqnorm_host(plan, host)
        p = g.partials()
        # each path must be bit-reproducible run to run; the two paths sum
        # in different window orders, so they agree to rounding only
        if kind not in ref:
            ref[kind] = p
        elif not np.array_equal(p, ref[kind]):
            bad[kind] += 1
            print(kind, r, "max rel", float(np.max(np.abs(p - ref[kind]) / np.abs(ref[kind]))),
                  flush=True)
        if len(ref) == 2:
            cross = max(cross, float(np.max(np.abs(ref["host"] - ref["dev"]) / np.abs(ref["dev"]))))
        g.close()
print("summary", bad, "max rel host vs dev", cross, flush=True)
