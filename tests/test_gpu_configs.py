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


def _torch_sqnorm(b, segments, chunk=1 << 28):
    """independent fp64 reference: torch, chunked, weights applied"""
    tot = 0.0
    for o, k, w in segments:
        if w == 0.0:
            continue
        acc = torch.zeros((), dtype=torch.float64, device=b.device)
        for c in range(o, o + k, chunk):
            x = b[c:min(c + chunk, o + k)].to(torch.float64)
            acc += torch.dot(x, x)
        tot += w * acc.item()
    return tot


def test_c2_3b_bf16_d8_full_step():
    """C2: Llama-3.2-3B bf16, (d,t,p) = (8,1,1), M = 8 — all 64 micro-buckets
    (3.21 G elements each) through the batched K1 and all 8 mean slices
    through K2, against an independent chunked torch fp64 reduction."""
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    spec = Lay.llama32_3b()
    d, M, seed = 8, 8, 0xC2
    lays = Lay.world_layouts(spec, d, 1, 1)
    unit = Lay.noise_unit_for(512.0, 2)
    g = D.GnsDevice(d, M, d * M * 2, 0)
    g.begin_step()
    lay = lays[0]  # t = p = 1: every rank holds the whole model
    plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
    bufs = [torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    s_ref = np.zeros(d * M)
    for i_d in range(d):
        for m0 in range(0, M, 2):
            for j in range(2):
                D.synth_fill(bufs[j], lay.gen, seed, i_d * M + m0 + j, Lay.G0, unit)
            g.micro_sqnorm_batched(plan, bufs, [i_d, i_d], [m0, m0 + 1])
            for j in range(2):
                s_ref[i_d * M + m0 + j] = _torch_sqnorm(bufs[j], lay.segments)
    mean = bufs[0]
    D.synth_mean_fill(mean, lay.gen, seed, 0, d * M, Lay.G0, unit)
    for i_d in range(d):
        sl = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0, slice_index=i_d, slice_count=d)
        g.mean_sqnorm(sl, mean)
    g2_ref = _torch_sqnorm(mean, lay.segments)
    g.finalize(d * M * 2 * 4096)
    r = g.result()
    parts = g.partials()
    assert np.allclose(parts[:-1], s_ref, rtol=1e-12, atol=0)
    assert abs(parts[-1] - g2_ref) <= 1e-12 * g2_ref
    st = O.finalize_step(parts[:-1], parts[-1], d * M * 2)
    assert r.b_simple == st.noise / st.signal or abs(r.b_simple - st.noise / st.signal) <= 1e-12 * abs(
        st.noise / st.signal)


def test_c3_7b_bf16_d2t2p2_layout_invariance_full_size():
    """C3: Llama-2-7B bf16, (d,t,p) = (2,2,2) with TP-replicated norm dedup.
    Size-independent property at full size: the 8 ranks' shard norms
    (weight-0 duplicates skipped) sum to the norm of the unsharded 6.74 G
    element gradient, for every micro-batch and for the synchronised mean
    (DP slices) — i.e. the dedup weights and the (d,t,p) partition are
    exact."""
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    spec = Lay.llama2_7b()
    d, t, p, M, seed = 2, 2, 2, 2, 0xC3
    unit = Lay.noise_unit_for(256.0, 2)
    world = Lay.world_layouts(spec, d, t, p)
    whole = Lay.world_layouts(spec, 1, 1, 1)[0]
    gw = D.GnsDevice(d, M, d * M * 2, 0)
    gu = D.GnsDevice(d, M, d * M * 2, 0)
    gw.begin_step()
    gu.begin_step()
    plan_u = D.BucketPlan(whole.segments, whole.numel, L.BF16, 0)
    big = torch.empty(whole.numel, dtype=torch.bfloat16, device="cuda")
    shard = torch.empty(max(l.numel for l in world), dtype=torch.bfloat16, device="cuda")
    for i_d in range(d):
        for m in range(M):
            D.synth_fill(big, whole.gen, seed, i_d * M + m, Lay.G0, unit)
            gu.micro_sqnorm(plan_u, big, i_d, m)
    for lay in world:
        i_d = lay.coords[0]
        plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
        view = shard[:lay.numel]
        for m in range(M):
            D.synth_fill(view, lay.gen, seed, i_d * M + m, Lay.G0, unit)
            gw.micro_sqnorm(plan, view, i_d, m)
        D.synth_mean_fill(view, lay.gen, seed, 0, d * M, Lay.G0, unit)
        sl = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0, slice_index=i_d, slice_count=d)
        gw.mean_sqnorm(sl, view)
    D.synth_mean_fill(big, whole.gen, seed, 0, d * M, Lay.G0, unit)
    gu.mean_sqnorm(plan_u, big)
    a, b = gw.partials(), gu.partials()
    assert np.allclose(a, b, rtol=1e-12, atol=0), (a, b)
    # the replicated norms really were deduplicated: counting them on every
    # TP rank would change s by their (nonzero) contribution
    dup = sum(k for l in world for o, k, w in l.segments if w == 0.0)
    assert dup > 0


def test_c4_32b_bf16_d1t4p2_fused_full_size():
    """C4: Qwen2.5-32B bf16, (d,t,p) = (1,4,2), M = 16, the north-star job at
    full size through K1f.  Size-independent properties (the oracle would need
    131 GB per rank): (1) the 8 ranks' fused s_m and ||gbar||^2 summed over the
    world equal the same sums under the (1,8,1) layout — the partition and the
    TP-duplicate dedup are exact for this model — and (2) on rank 0 the fused
    pass equals 16 separate K1 passes for every s_m."""
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    torch.cuda.empty_cache()
    spec = Lay.qwen25_32b()
    M, seed = 16, 0xC4
    unit = Lay.noise_unit_for(1024.0, 1)
    worlds = {(1, 4, 2): Lay.world_layouts(spec, 1, 4, 2), (1, 8, 1): Lay.world_layouts(spec, 1, 8, 1)}
    cap = max(l.numel for w in worlds.values() for l in w)
    free, _ = torch.cuda.mem_get_info()
    if M * cap * 2 > free - (8 << 30):
        pytest.skip(f"needs {M * cap * 2 / 1e9:.0f} GB free, have {free / 1e9:.0f}")
    bufs = [torch.empty(cap, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    parts = {}
    for key, world in worlds.items():
        g = D.GnsDevice(1, M, M, 0)
        g.begin_step()
        for r, lay in enumerate(world):
            views = [b[:lay.numel] for b in bufs]
            for m in range(M):
                D.synth_fill(views[m], lay.gen, seed, m, Lay.G0, unit)
            plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
            g.fused_sqnorm(plan, views)
            if key == (1, 4, 2) and r == 0:
                sep = D.GnsDevice(1, M, M, 0)
                sep.begin_step()
                for m in range(M):
                    sep.micro_sqnorm(plan, views[m], 0, m)
                one = D.GnsDevice(1, M, M, 0)
                one.begin_step()
                one.fused_sqnorm(plan, views)
                a, b = one.partials()[:M], sep.partials()[:M]
                assert np.allclose(a, b, rtol=1e-12, atol=0), (a, b)
                assert b.min() > 0
                one.close()
                sep.close()
            plan.close()
        parts[key] = g.partials()
        g.close()
    a, b = parts[(1, 4, 2)], parts[(1, 8, 1)]
    assert np.allclose(a, b, rtol=1e-12, atol=0), (a, b)
    assert a[M] > 0
    del bufs
    torch.cuda.empty_cache()
