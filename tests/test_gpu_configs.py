"""Full-size BASELINE configs on the GPU against the oracle (size-independent
checks where the oracle would be too slow)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def test_c1_125m_fp32_d2_full_step():
    # C1: GPT-2-small fp32, d = 2, M = 4 (every DP rank's buckets + mean slices)
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    spec = Lay.gpt2_small()
    d, M, seed = 2, 4, 0xC0905
    lays = Lay.world_layouts(spec, d, 1, 1)
    unit = Lay.noise_unit_for(256.0, 2)
    g = D.GnsDevice(d, M, d * M * 2, 0)
    g.begin_step()
    nth = os.cpu_count() or 1
    s_ref = np.zeros(d * M)
    g2_ref = 0.0
    for lay in lays:
        i_d = lay.coords[0]
        plan = D.BucketPlan(lay.segments, lay.numel, L.FP32, 0)
        b = torch.empty(lay.numel, dtype=torch.float32, device="cuda")
        for m in range(M):
            D.synth_fill(b, lay.gen, seed, i_d * M + m, Lay.G0, unit)
            g.micro_sqnorm(plan, b, i_d, m)
            torch.cuda.synchronize()
            s_ref[i_d * M + m] = O.sqnorm_mt(b.cpu().numpy(), O.FP32, lay.segments, nth)
        mean = torch.empty(lay.numel, dtype=torch.float32, device="cuda")
        D.synth_mean_fill(mean, lay.gen, seed, 0, d * M, Lay.G0, unit)
        sl = D.BucketPlan(lay.segments, lay.numel, L.FP32, 0, slice_index=i_d, slice_count=d)
        g.mean_sqnorm(sl, mean)
        n = lay.numel
        lo = (n * i_d // d) & ~63
        hi = n if i_d + 1 == d else (n * (i_d + 1) // d) & ~63
        segs = [(max(o, lo), min(o + k, hi) - max(o, lo), w) for o, k, w in lay.segments
                if max(o, lo) < min(o + k, hi)]
        torch.cuda.synchronize()
        g2_ref += O.sqnorm_mt(mean.cpu().numpy(), O.FP32, segs, nth)
    g.finalize(d * M * 2 * 1024)
    r = g.result()
    parts = g.partials()
    assert np.allclose(parts[:-1], s_ref, rtol=1e-12, atol=0)
    assert abs(parts[-1] - g2_ref) <= 1e-12 * g2_ref
    st = O.finalize_step(s_ref, g2_ref, d * M * 2)
    assert abs(r.b_simple - st.noise / st.signal) <= 1e-9 * abs(st.noise / st.signal)
