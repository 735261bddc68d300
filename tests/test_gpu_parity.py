"""GPU parity: the B200 path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): squared norms within 1e-6 relative (we hold
1e-9), B_simple within 1e-5 (we hold 1e-7), candidate ranking identical;
generator bytes and the finalize/EMA arithmetic bit-exact.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

RTOL_NORM = 1e-9
RTOL_BSIMPLE = 1e-7


@pytest.fixture(scope="module")
def D():
    from paper_2604_26687_b200 import device
    torch.cuda.set_device(0)
    return device


@pytest.fixture(scope="module")
def L():
    from paper_2604_26687_b200 import _lib
    return _lib


@pytest.fixture(scope="module")
def Lay():
    from paper_2604_26687_b200 import layout
    return layout


TDT = {0: "bfloat16", 1: "float16", 2: "float32"}


def _host_u(t):
    """device tensor -> numpy view with the oracle's element type"""
    if t.dtype == torch.float32:
        return t.cpu().numpy()
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _dev_buf(D, numel, dtype_code, gen, seed, sample, unit, offset_elems=0, g0=2.0 ** -10):
    """synthetic bucket on the device, optionally starting `offset_elems`
    into a larger allocation (unaligned base pointers)"""
    tdt = getattr(torch, TDT[dtype_code])
    raw = torch.zeros(numel + offset_elems + 16, dtype=tdt, device="cuda")
    view = raw[offset_elems:offset_elems + numel]
    D.synth_fill(view, gen, seed, sample, g0, unit)
    return raw, view


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ---------------------------------------------------------------- generator

@pytest.mark.parametrize("dtype", [0, 1, 2])
def test_generator_bit_exact(D, dtype):
    n = 100_003
    gen = [(0, 40_000, 7, 40_000, 40_000), (40_000, 60_003, 1_000_000, 101, 400)]
    unit = O.noise_unit_for(2 ** -10, 256.0, 1)
    _, v = _dev_buf(D, n, dtype, gen, 0xC0905, 3, unit)
    torch.cuda.synchronize()
    ref = O.synth_fill(n, dtype, gen, 0xC0905, 3, 2 ** -10, unit)
    assert np.array_equal(_host_u(v), ref)


@pytest.mark.parametrize("dtype", [0, 2])
def test_mean_generator_bit_exact(D, dtype):
    n = 20_011
    gen = [(0, n, 55, 97, 200)]
    unit = O.noise_unit_for(2 ** -10, 64.0, 2)
    tdt = getattr(torch, TDT[dtype])
    v = torch.empty(n, dtype=tdt, device="cuda")
    D.synth_mean_fill(v, gen, 9, 16, 8, 2 ** -10, unit)
    torch.cuda.synchronize()
    ref = O.synth_mean_fill(n, dtype, gen, 9, 16, 8, 2 ** -10, unit)
    assert np.array_equal(_host_u(v), ref)


# ---------------------------------------------------------------- K1

CASES = [
    # (numel, segments, base offset in elements)
    (1, [(0, 1, 1.0)], 0),
    (7, [(0, 7, 1.0)], 1),
    (4096, [(0, 4096, 1.0)], 0),
    (1_000_003, [(0, 1_000_003, 1.0)], 3),
    (300_001, [(0, 1, 1.0), (1, 99_999, 0.0), (100_000, 5, 1.0), (100_005, 199_996, 1.0),
               (300_005 - 4, 0, 1.0)], 5),
    (250_000, [(3, 10, 1.0), (17, 100_000, 0.5), (100_017, 149_983, 1.0)], 2),
]


@pytest.mark.parametrize("dtype", [0, 1, 2])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_micro_sqnorm_matches_oracle(D, L, dtype, case):
    numel, segs, off = CASES[case]
    segs = [s for s in segs if s[0] + s[1] <= numel]
    gen = [(0, numel, 11, numel, numel)]
    unit = O.noise_unit_for(2 ** -10, 256.0, 1)
    raw, v = _dev_buf(D, numel, dtype, gen, 1234, case, unit, offset_elems=off)
    plan = D.BucketPlan(segs, numel, dtype, 0)
    g = D.GnsDevice(2, 1, 2, 0)
    g.begin_step()
    g.micro_sqnorm(plan, v, 1, 0)
    got = g.partials()[1]
    ref = O.sqnorm(_host_u(v), dtype, segs)
    assert _rel(got, ref) <= RTOL_NORM, (got, ref)
    # deterministic: a second pass gives the identical bits
    g.begin_step()
    g.micro_sqnorm(plan, v, 1, 0)
    assert g.partials()[1] == got


def test_zero_and_extreme_values(D, L):
    n = 4096
    x = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, 0)
    g = D.GnsDevice(1, 2, 2, 0)
    g.begin_step()
    g.micro_sqnorm(plan, x, 0, 0)
    assert g.partials()[0] == 0.0
    # |x| ~ 2^70: x^2 overflows fp32 but not fp64; |x| ~ 2^-80: underflows fp32
    for mag in (2.0 ** 70, 2.0 ** -80, 3.0e38):
        x = torch.full((n,), mag, dtype=torch.bfloat16, device="cuda")
        x[::3] = -x[::3]
        g.begin_step()
        g.micro_sqnorm(plan, x, 0, 0)
        got = g.partials()[0]
        ref = O.sqnorm(_host_u(x), O.BF16, [(0, n, 1.0)])
        assert _rel(got, ref) <= 1e-12, (mag, got, ref)


def test_nonfinite_gradient_is_a_validation_error(D, L):
    n = 1000
    x = torch.ones(n, dtype=torch.bfloat16, device="cuda")
    x[17] = float("nan")
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, 0)
    g = D.GnsDevice(1, 2, 2, 0)
    st0 = g.get_state().as_tuple()
    g.begin_step()
    g.micro_sqnorm(plan, x, 0, 0)
    g.micro_sqnorm(plan, torch.ones_like(x), 0, 1)
    g.finalize(10)
    with pytest.raises(L.ValidationError):
        g.result()
    assert g.get_state().as_tuple() == st0  # state untouched


def test_argument_validation(D, L):
    n = 64
    x = torch.ones(n + 1, dtype=torch.float32, device="cuda")
    plan = D.BucketPlan([(0, n, 1.0)], n, L.FP32, 0)
    g = D.GnsDevice(2, 2, 4, 0)
    with pytest.raises(L.ValidationError):
        g.micro_sqnorm(plan, x.data_ptr() + 2, 0, 0)  # misaligned fp32
    with pytest.raises(L.ValidationError):
        g.micro_sqnorm(plan, x, 2, 0)  # dp index out of range
    with pytest.raises(L.ValidationError):
        g.fused_sqnorm(plan, [x, x])  # fused needs d == 1
    with pytest.raises(L.ValidationError):
        D.BucketPlan([(0, n + 5, 1.0)], n, L.FP32, 0)  # segment beyond bucket
    with pytest.raises(L.ValidationError):
        D.BucketPlan([(0, 10, 1.0), (5, 10, 1.0)], n, L.FP32, 0)  # overlap
    with pytest.raises(L.ValidationError):
        D.GnsDevice(1, 1, 1, 0)  # N < 2


# ---------------------------------------------------------------- K1f

@pytest.mark.parametrize("off", [0, 1])  # 0: TMA bulk-copy path, 1: unaligned LDG path
@pytest.mark.parametrize("dtype", [0, 1, 2])
@pytest.mark.parametrize("M", [1, 2, 3, 4, 8, 16])
def test_fused_matches_oracle(D, L, dtype, M, off):
    numel = 200_003
    segs = [(0, 70_001, 1.0), (70_001, 4096, 0.0), (74_097, numel - 74_097, 1.0)]
    gen = [(0, numel, 0, numel, numel)]
    unit = O.noise_unit_for(2 ** -10, 1024.0, 1)
    bufs = [_dev_buf(D, numel, dtype, gen, 77, m, unit, offset_elems=off)[1] for m in range(M)]
    plan = D.BucketPlan(segs, numel, dtype, 0)
    g = D.GnsDevice(1, max(M, 2), max(M, 2), 0) if M >= 2 else None
    if M == 1:
        # N = 1 is rejected; fused with M = 1 still reduces
        with pytest.raises(L.ValidationError):
            D.GnsDevice(1, 1, 1, 0)
        return
    g.begin_step()
    g.fused_sqnorm(plan, bufs)
    parts = g.partials()
    s, ss = O.fused_sqnorms([_host_u(b) for b in bufs], dtype, segs, 4)
    for m in range(M):
        assert _rel(parts[m], s[m]) <= RTOL_NORM
    assert _rel(parts[M], ss / (M * M)) <= RTOL_NORM


@pytest.mark.parametrize("M", [3, 4])
def test_fused_host_streaming_matches_device(D, L, M):
    numel = (16 << 20) + 12_345  # spans two staging windows
    segs = [(0, 1000, 1.0), (1000, 5000, 0.0), (6000, 8_000_000, 1.0),
            (8_006_000, 3, 0.5), (8_006_003, numel - 8_006_003, 1.0)]
    gen = [(0, numel, 3, numel, numel)]
    unit = O.noise_unit_for(2 ** -10, 256.0, 1)
    bufs = [_dev_buf(D, numel, L.BF16, gen, 5, m, unit)[1] for m in range(M)]
    host = [b.cpu().pin_memory() for b in bufs]
    plan = D.BucketPlan(segs, numel, L.BF16, 0)
    g = D.GnsDevice(1, M, M, 0)
    g.begin_step()
    g.fused_sqnorm(plan, bufs)
    a = g.partials()
    g.begin_step()
    g.fused_sqnorm_host(plan, host)
    b = g.partials()
    assert np.allclose(a, b, rtol=1e-12, atol=0)
    s, ss = O.fused_sqnorms([_host_u(x) for x in bufs], O.BF16, segs, 8)
    assert np.allclose(a[:M], s, rtol=RTOL_NORM, atol=0)
    assert _rel(a[-1], ss / (M * M)) <= RTOL_NORM


# ---------------------------------------------------------------- K2 + K3

def _emulate_world(D, L, Lay, spec, d, t, p, M, seed, unit, dtype=0, fused=False):
    """All d*t*p ranks of a layout on one GPU; returns (GnsDevice, layouts)."""
    lays = Lay.world_layouts(spec, d, t, p)
    g = D.GnsDevice(d, M, d * M * 2, 0)
    g.begin_step()
    tdt = getattr(torch, TDT[dtype])
    for lay in lays:
        i_d, i_t, i_p = lay.coords
        plan = D.BucketPlan(lay.segments, lay.numel, dtype, 0)
        bufs = []
        for m in range(M):
            b = torch.empty(lay.numel, dtype=tdt, device="cuda")
            D.synth_fill(b, lay.gen, seed, i_d * M + m, 2 ** -10, unit)
            bufs.append(b)
        if fused:
            g.fused_sqnorm(plan, bufs)
        else:
            g.micro_sqnorm_batched(plan, bufs, [i_d] * M, list(range(M)))
            mean = torch.empty(lay.numel, dtype=tdt, device="cuda")
            D.synth_mean_fill(mean, lay.gen, seed, 0, d * M, 2 ** -10, unit)
            sl = D.BucketPlan(lay.segments, lay.numel, dtype, 0, slice_index=i_d, slice_count=d)
            g.mean_sqnorm(sl, mean)
    return g, lays


def test_layout_invariance_and_dedup(D, L, Lay):
    # SPEC.md:217 analogue: the same logical gradients under (2,2,2) and
    # (2,1,1) give the same s_n and gbar^2 (pins the TP/tied dedup weights).
    spec = Lay.tiny_model(layers=4, h=128, ffn=256, vocab=512, tied=True)
    unit = Lay.noise_unit_for(256.0, 1)
    M = 2
    ga, _ = _emulate_world(D, L, Lay, spec, 2, 2, 2, M, 99, unit)
    gb, _ = _emulate_world(D, L, Lay, spec, 2, 1, 1, M, 99, unit)
    a, b = ga.partials(), gb.partials()
    assert np.allclose(a, b, rtol=1e-12, atol=0), (a, b)
    # and (1,1,1) with everything in one bucket: s_n for n < M agree too
    gc, _ = _emulate_world(D, L, Lay, spec, 1, 2, 2, M, 99, unit, fused=True)
    gd, _ = _emulate_world(D, L, Lay, spec, 1, 1, 1, M, 99, unit, fused=True)
    assert np.allclose(gc.partials(), gd.partials(), rtol=1e-12, atol=0)


@pytest.mark.parametrize("phi_true", [256.0, 4096.0])
def test_world_step_matches_oracle(D, L, Lay, phi_true):
    # nominal and stress (cancellation, SURVEY 8(d)/App. B.3) noise scales
    spec = Lay.tiny_model(layers=4, h=128, ffn=256, vocab=512, tied=False)
    d, t, p, M = 2, 2, 2, 4
    unit = Lay.noise_unit_for(phi_true, 1)
    g, lays = _emulate_world(D, L, Lay, spec, d, t, p, M, 7, unit)
    tokens = d * M * 2048
    g.finalize(tokens)
    r = g.result()
    # oracle: per-rank buffers regenerated on the CPU
    s = np.zeros(d * M)
    gb2 = 0.0
    for lay in lays:
        i_d = lay.coords[0]
        for m in range(M):
            buf = O.synth_fill(lay.numel, O.BF16, lay.gen, 7, i_d * M + m, 2 ** -10, unit)
            s[i_d * M + m] += O.sqnorm(buf, O.BF16, lay.segments)
        if i_d == 0:
            mean = O.synth_mean_fill(lay.numel, O.BF16, lay.gen, 7, 0, d * M, 2 ** -10, unit)
            gb2 += O.sqnorm(mean, O.BF16, lay.segments)
    parts = g.partials()
    assert np.allclose(parts[:-1], s, rtol=RTOL_NORM, atol=0)
    assert _rel(parts[-1], gb2) <= RTOL_NORM
    st = O.finalize_step(s, gb2, d * M * 2)
    assert _rel(r.stats.signal, st.signal) <= RTOL_BSIMPLE
    assert _rel(r.b_simple, st.noise / st.signal) <= RTOL_BSIMPLE


def test_device_finalize_bit_exact_with_host(D, L):
    # feed identical partials to the device kernel and the host C++ API
    from paper_2604_26687_b200 import gns as G
    n = 50_000
    x = torch.randn(n, device="cuda").to(torch.bfloat16)
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, 0)
    g = D.GnsDevice(2, 3, 48, 0)
    host_state = G.GnsState.default()
    for step in range(40):
        g.begin_step()
        for k in range(6):
            g.micro_sqnorm(plan, x * (1.0 + 0.01 * ((k * 7 + step) % 5)), k // 3, k % 3)
        g.mean_sqnorm(plan, x * 0.9)
        g.finalize(400_000)
        r = g.result()
        parts = g.partials()
        acc = G.StepAccumulator(2, 48)
        for v in parts[:-1]:
            acc.record_micro_batch(v)
        st = G.finalize_step(acc, parts[-1])
        G.update_ema(host_state, st, 400_000)
        assert (r.stats.signal, r.stats.noise, r.stats.noise_raw) == (st.signal, st.noise, st.noise_raw)
        assert r.state.as_tuple() == host_state.as_tuple()
        phi = G.gns(host_state)
        assert (r.phi_available == 1) == (phi is not None)
        if phi is not None:
            assert r.phi == phi
    # checkpoint round trip of the device GnsState
    s = g.get_state()
    g2 = D.GnsDevice(2, 3, 48, 0)
    g2.set_state(s)
    assert g2.get_state().as_tuple() == s.as_tuple()


def test_span_overload_runs_on_gpu(D, L):
    from paper_2604_26687_b200 import gns as G
    rng = np.random.default_rng(0)
    v = rng.normal(size=123_457)
    acc = G.StepAccumulator(1, 4)
    for x in (3.0, 5.0, 4.0, 6.0):
        acc.record_micro_batch(x)
    st = G.finalize_step(acc, v)
    ref = O.finalize_step([3.0, 5.0, 4.0, 6.0], O.sumsq_f64(v), 4)
    assert _rel(st.mean_grad_sq, ref.mean_grad_sq) <= 1e-13
    assert _rel(st.signal, ref.signal) <= 1e-12
    # SPEC.md:181 hand-worked case through the span overload
    acc = G.StepAccumulator(1, 2)
    acc.record_micro_batch(9.0)
    acc.record_micro_batch(1.0)
    st = G.finalize_step(acc, np.array([2.0, 0.0]))
    assert (st.signal, st.noise) == (3.0, 2.0)


def test_scorer_ranking_from_gpu_phi_matches_oracle(D, L, Lay):
    from paper_2604_26687_b200 import gns as G
    spec = Lay.tiny_model(layers=2, h=128, ffn=256, vocab=256)
    unit = Lay.noise_unit_for(256.0, 1)
    g, _ = _emulate_world(D, L, Lay, spec, 1, 1, 1, 8, 3, unit, fused=True)
    g.finalize(8 * 2048)
    r = g.result()
    assert r.phi_available
    costs = [(8, 1, 1, 4000.0, 256.0), (4, 2, 1, 3300.0, 96.0), (2, 2, 2, 2600.0, 40.0),
             (1, 4, 2, 2000.0, 16.0), (2, 4, 1, 2400.0, 32.0)]
    bg, bm = [16, 32, 64, 128, 256, 512, 1024, 2048], [1, 2, 4, 8]
    cands = G.synth_candidates(costs, bg, bm, True, 0.0, 0.0)
    ents = O.feasible_candidates(O.synth_profile(costs, bg, bm, True, 0.0, 0.0, 1e300))
    assert [c.key() for c in cands] == [(e.d, e.t, e.p, e.global_batch, e.micro_batch) for e in ents]
    cur = cands[3]
    ours = G.rank_candidates(cands, r.phi, cur, 900.0, 800.0, reconfig_cost=50.0)
    oscore = O.score_candidates(ents, r.phi, ents[3], 900.0, 800.0, reconfig_cost=50.0)
    # oracle ranking with the decide() tie-break
    order = sorted(range(len(ents)), key=lambda i: (-oscore[i], 0 if i == 3 else 1,
                                                    ents[i].global_batch, -ents[i].d, -ents[i].t,
                                                    ents[i].micro_batch))
    assert ours == order
    cmd = G.decide(cands, r.phi, cur, 900.0, 800.0, reconfig_cost=50.0)
    ocmd = O.decide(ents, r.phi, ents[3], 900.0, 800.0, reconfig_cost=50.0)
    assert (cmd.kind, cmd.winner_index) == (ocmd.kind, ocmd.winner_index)


def test_full_size_3b_bucket_against_oracle(D, L, Lay):
    # one full 3B-shaped (8,1,1) rank bucket: 3.21 G bf16 elements (6.4 GB)
    lay = Lay.rank_layout(Lay.llama32_3b(), 8, 1, 1, 0)
    unit = Lay.noise_unit_for(256.0, 2)
    b = torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda")
    D.synth_fill(b, lay.gen, 0xC0907, 5, 2 ** -10, unit)
    plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
    g = D.GnsDevice(8, 8, 128, 0)
    g.begin_step()
    g.micro_sqnorm(plan, b, 0, 5)
    got = g.partials()[5]
    host = b.cpu().view(torch.int16).numpy().view(np.uint16)
    # spot-check the generator bytes on three windows, then the full norm
    for lo in (0, lay.numel // 2, lay.numel - 100_000):
        win = [(0, 100_000, lo, 100_000, 100_000)]
        assert np.array_equal(O.synth_fill(100_000, O.BF16, win, 0xC0907, 5, 2 ** -10, unit),
                              host[lo:lo + 100_000])
    import os
    ref = O.sqnorm_mt(host, O.BF16, lay.segments, os.cpu_count() or 1)
    assert _rel(got, ref) <= RTOL_NORM, (got, ref)


# ---------------------------------------------------------------- KA (trainer form)

@pytest.mark.parametrize("dtype", [0, 2])
def test_accumulate_fused_into_grad_accumulation(D, L, dtype):
    M, numel = 4, 300_017
    # weighted segments with a weight-0 (TP duplicate) hole and an uncovered gap
    segs = [(0, 100_000, 1.0), (100_000, 4_096, 0.0), (104_096, 50_000, 1.0),
            (160_000, numel - 160_000, 1.0)]
    gen = [(0, numel, 0, numel, numel)]
    unit = O.noise_unit_for(2 ** -10, 256.0, 1)
    tdt = getattr(torch, TDT[dtype])
    grads = []
    for m in range(M):
        b = torch.empty(numel, dtype=tdt, device="cuda")
        D.synth_fill(b, gen, 21, m, 2 ** -10, unit)
        grads.append(b)
    plan = D.BucketPlan(segs, numel, dtype, 0)
    g = D.GnsDevice(1, M, M, 0)
    main = torch.full((numel,), 123.0, dtype=torch.float32, device="cuda")  # stale
    g.begin_step()
    for m in range(M):
        g.accumulate(plan, main, grads[m], 0, m, first=(m == 0), last_mean=(m == M - 1))
    parts = g.partials()
    # main_grad is exactly torch's sequential fp32 accumulation
    ref = grads[0].float().clone()
    for m in range(1, M):
        ref.add_(grads[m].float())
    assert torch.equal(main, ref)
    host = [_host_u(b) for b in grads]
    s, ss = O.fused_sqnorms(host, dtype, segs, 4)
    for m in range(M):
        assert _rel(parts[m], s[m]) <= RTOL_NORM
    assert _rel(parts[M], ss / (M * M)) <= RTOL_NORM
    # the same numbers as the pure GNS pass
    g2 = D.GnsDevice(1, M, M, 0)
    g2.begin_step()
    g2.fused_sqnorm(plan, grads)
    assert np.allclose(parts, g2.partials(), rtol=1e-12, atol=0)


def test_accumulate_validation(D, L):
    n = 1024
    plan = D.BucketPlan([(0, n, 1.0)], n, L.BF16, 0)
    sl = D.BucketPlan([(0, n, 1.0)], n, L.BF16, 0, slice_index=0, slice_count=2)
    g = D.GnsDevice(2, 2, 4, 0)
    main = torch.zeros(n + 4, dtype=torch.float32, device="cuda")
    grad = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(L.ValidationError):
        g.accumulate(plan, main, grad, 0, 0, last_mean=True)  # d > 1
    with pytest.raises(L.ValidationError):
        g.accumulate(sl, main, grad, 0, 0)  # slice plan
    with pytest.raises(L.ValidationError):
        g.accumulate(plan, main[1:], grad, 0, 0)  # misaligned main_grad


@pytest.mark.parametrize("dtype", [0, 2])
def test_host_streaming_k1_matches_device(D, L, dtype):
    """micro_sqnorm_host / mean_sqnorm_host (HOST buckets streamed H2D in
    whole-stage windows) equal the device-resident K1 — across window
    boundaries, weight-0 gaps, a DP-slice plan and an unaligned tail."""
    tdt = getattr(torch, TDT[dtype])
    n = (300 << 20) + 12345 if dtype == 0 else (40 << 20) + 77  # > 1 window for bf16
    segs = [(0, 70_001, 1.0), (70_001, 1 << 20, 0.0), (70_001 + (1 << 20), n - 70_001 - (1 << 20), 0.5)]
    dev_b = torch.randn(n, device="cuda").to(tdt)
    host_b = dev_b.cpu().pin_memory()
    full = D.BucketPlan(segs, n, dtype, 0)
    sl = D.BucketPlan(segs, n, dtype, 0, slice_index=1, slice_count=3)
    ga, gb = D.GnsDevice(2, 2, 8, 0), D.GnsDevice(2, 2, 8, 0)
    for g in (ga, gb):
        g.begin_step()
    ga.micro_sqnorm(full, dev_b, 1, 0)
    ga.mean_sqnorm(sl, dev_b)
    gb.micro_sqnorm_host(full, host_b, 1, 0)
    gb.mean_sqnorm_host(sl, host_b)
    a, b = ga.partials(), gb.partials()
    assert a[2] > 0 and a[-1] > 0
    assert np.allclose(a, b, rtol=1e-12, atol=0), (a, b)
    # oracle on the same bytes
    ref = O.sqnorm(_host_u(dev_b), dtype, segs)
    assert _rel(b[2], ref) <= RTOL_NORM


def test_span_overload_chunked_large_vector(D, L):
    """finalize_step(acc, span) with a host vector larger than one 32 Mi
    chunk: bounded device footprint, same value as the oracle's fp64 sum."""
    from paper_2604_26687_b200 import gns as G
    rng = np.random.default_rng(1)
    v = rng.normal(size=(32 << 20) + (5 << 20) + 3)
    acc = G.StepAccumulator(1, 4)
    for x in (3.0, 5.0):
        acc.record_micro_batch(x)
    st = G.finalize_step(acc, v)
    # 37 M fp64 terms summed in different orders: both sides carry ~sqrt(n)
    # ulp-level rounding; math.fsum of the squares is the tiebreaker
    import math
    exact = math.fsum((v * v).tolist())
    assert _rel(st.mean_grad_sq, exact) <= 1e-12
    assert _rel(O.sumsq_f64(v), exact) <= 1e-11


def _random_segments(rng, numel):
    """a random segment table: gaps, tiny and long ranges, weights 0/0.5/1/2"""
    segs, at = [], int(rng.integers(0, 9))
    while at < numel:
        kind = rng.integers(0, 4)
        n = int(rng.integers(1, 8)) if kind == 0 else int(rng.integers(8, 70_000))
        n = min(n, numel - at)
        segs.append((at, n, float(rng.choice([0.0, 0.5, 1.0, 1.0, 2.0]))))
        at += n + (int(rng.integers(0, 40)) if rng.random() < 0.3 else 0)
    return segs


@pytest.mark.parametrize("seed", range(40))
def test_randomized_layouts_k1_k1f_host(D, L, seed):
    """Randomized segment tables, base offsets, dtypes and M through every
    reduction entry point (K1, K1f TMA/LDG, K2 slice, host streaming)
    against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    dtype = int(rng.choice([0, 0, 1, 2]))
    M = int(rng.choice([2, 3, 5, 7, 8, 11, 16]))
    numel = int(rng.integers(1, 400_000))
    off = int(rng.choice([0, 0, 1, 3, 8]))
    segs = _random_segments(rng, numel)
    gen = [(0, numel, 0, numel, numel)]
    unit = O.noise_unit_for(2 ** -10, 512.0, 1)
    raws = [_dev_buf(D, numel, dtype, gen, seed, m, unit, offset_elems=off) for m in range(M)]
    bufs = [v for _, v in raws]
    hb = [_host_u(b) for b in bufs]
    plan = D.BucketPlan(segs, numel, dtype, 0)
    s_ref, ss_ref = O.fused_sqnorms(hb, dtype, segs, 4)
    # K1 (batched) and K1f
    g1, g2 = D.GnsDevice(1, M, M, 0), D.GnsDevice(1, M, M, 0)
    g1.begin_step()
    g1.micro_sqnorm_batched(plan, bufs, [0] * M, list(range(M)))
    g2.begin_step()
    g2.fused_sqnorm(plan, bufs)
    p1, p2 = g1.partials(), g2.partials()
    for m in range(M):
        assert _rel(p1[m], s_ref[m]) <= RTOL_NORM, (seed, m)
        assert _rel(p2[m], s_ref[m]) <= RTOL_NORM, (seed, m)
    assert _rel(p2[M], ss_ref / (M * M)) <= RTOL_NORM
    # host streaming: one bucket through K1, all through K1f
    g3 = D.GnsDevice(1, M, M, 0)
    g3.begin_step()
    host = [b.cpu().pin_memory() for b in bufs]
    g3.micro_sqnorm_host(plan, host[0], 0, 0)
    p3 = g3.partials()
    assert _rel(p3[0], s_ref[0]) <= RTOL_NORM
    g4 = D.GnsDevice(1, M, M, 0)
    g4.begin_step()
    g4.fused_sqnorm_host(plan, host)
    p4 = g4.partials()
    for m in range(M):
        assert _rel(p4[m], s_ref[m]) <= RTOL_NORM
    assert _rel(p4[M], ss_ref / (M * M)) <= RTOL_NORM
    # K2 over a random DP slice
    d = int(rng.integers(2, 5))
    i = int(rng.integers(0, d))
    sl = D.BucketPlan(segs, numel, dtype, 0, slice_index=i, slice_count=d)
    lo, hi = D.dp_slice(numel, d, i)
    segs_sl = [(max(o, lo), min(o + k, hi) - max(o, lo), w) for o, k, w in segs
               if max(o, lo) < min(o + k, hi)]
    g5 = D.GnsDevice(d, M, M * d, 0)
    g5.begin_step()
    g5.mean_sqnorm(sl, bufs[0])
    ref = O.sqnorm(hb[0], dtype, segs_sl)
    assert _rel(g5.partials()[-1], ref) <= RTOL_NORM


# ---------------------------------------------------------------- degenerate inputs

@pytest.mark.parametrize("dtype", [0, 2])
@pytest.mark.parametrize("kind", ["no_segments", "all_weight_zero", "zero_numel"])
def test_empty_buckets_contribute_zero(D, L, dtype, kind):
    """A rank whose bucket holds no counted element (no segments, only TP
    duplicates, or nothing at all) contributes exact zeros on every path and
    the step still finalizes (s_m is a sum over local
    parameters, empty sums are 0)."""
    tdt = getattr(torch, TDT[dtype])
    numel = 0 if kind == "zero_numel" else 10_001
    segs = {"no_segments": [], "all_weight_zero": [(0, numel, 0.0)], "zero_numel": []}[kind]
    plan = D.BucketPlan(segs, numel, dtype, 0)
    assert plan.active_elements == 0
    M = 4
    bufs = [torch.ones(max(numel, 1), dtype=tdt, device="cuda")[:numel] for _ in range(M)]
    g = D.GnsDevice(1, M, M, 0)
    g.begin_step()
    g.fused_sqnorm(plan, bufs)
    assert np.all(g.partials() == 0.0)
    g.begin_step()
    for m in range(M):
        g.micro_sqnorm(plan, bufs[m], 0, m)
    g.mean_sqnorm(plan, bufs[0])
    assert np.all(g.partials() == 0.0)
    main = torch.full((numel,), 3.0, dtype=torch.float32, device="cuda")
    g.begin_step()
    g.accumulate(plan, main, bufs[0], 0, 0, first=False)
    assert np.all(g.partials() == 0.0)
    # accumulation itself still happens on every element (gaps included)
    assert bool(torch.all(main == 4.0))
    host = [b.cpu().pin_memory() for b in bufs]
    g.begin_step()
    g.fused_sqnorm_host(plan, host)
    assert np.all(g.partials() == 0.0)
    # all-zero norms: signal 0 -> phi unavailable, never an error
    g.finalize(M * 2048)
    r = g.result()
    assert r.stats.signal == 0.0 and r.stats.noise == 0.0
    assert r.status == 0 and r.phi_available == 0


@pytest.mark.parametrize("dtype", [0, 1, 2])
@pytest.mark.parametrize("M", [2, 5, 8, 16])
def test_batched_k1_tma_ring_matches_single_passes(D, L, dtype, M):
    """micro_sqnorm_batched over one rank's aligned micro-buckets runs the TMA
    ring without its mean term; it must equal the single-bucket K1 passes
    (and the oracle), touch only the M slots, and fall back to the LDG batch
    for unaligned views with the same results."""
    numel = 300_007
    segs = [(0, 100_000, 1.0), (100_000, 3333, 0.0), (103_333, numel - 103_333 - 7, 0.5)]
    gen = [(0, numel, 0, numel, numel)]
    unit = O.noise_unit_for(2 ** -10, 64.0, 1)
    plan = D.BucketPlan(segs, numel, dtype, 0)
    d = 2
    for off in (0, 1):
        bufs = [_dev_buf(D, numel, dtype, gen, 31, m, unit, offset_elems=off)[1] for m in range(M)]
        gb = D.GnsDevice(d, M, d * M, 0)
        gb.begin_step()
        gb.micro_sqnorm_batched(plan, bufs, [1] * M, list(range(M)))
        gs = D.GnsDevice(d, M, d * M, 0)
        gs.begin_step()
        for m in range(M):
            gs.micro_sqnorm(plan, bufs[m], 1, m)
        pb, ps = gb.partials(), gs.partials()
        assert np.all(pb[:M] == 0.0) and pb[-1] == 0.0  # only dp_index 1's slots
        assert np.allclose(pb[M:2 * M], ps[M:2 * M], rtol=1e-12, atol=0), (off, pb, ps)
        for m in (0, M - 1):
            ref = O.sqnorm(_host_u(bufs[m]), dtype, segs)
            assert _rel(pb[M + m], ref) <= RTOL_NORM


@pytest.mark.parametrize("dtype", [0, 1, 2])
def test_every_m_instantiation_matches_oracle(D, L, dtype):
    """Each micro-batch count M = 2..16 is its own fused_tma_kernel
    instantiation (shape chosen per M, kBestShape), for the fused pass and
    for the batched K1 ring: every one against the oracle, on a bucket long
    enough for several chunks per CTA and with a weight-0 hole that cuts a
    tile."""
    numel = 148 * 3584 * 3 + 1234
    segs = [(0, 500_000, 1.0), (500_000, 7777, 0.0), (507_777, numel - 507_777, 1.0)]
    gen = [(0, numel, 0, numel, numel)]
    unit = O.noise_unit_for(2 ** -10, 256.0, 1)
    bufs = [_dev_buf(D, numel, dtype, gen, 404, m, unit)[1] for m in range(16)]
    host = [_host_u(b) for b in bufs]
    plan = D.BucketPlan(segs, numel, dtype, 0)
    for M in range(2, 17):
        g = D.GnsDevice(1, M, M, 0)
        g.begin_step()
        g.fused_sqnorm(plan, bufs[:M])
        parts = g.partials()
        s, ss = O.fused_sqnorms(host[:M], dtype, segs, 4)
        for m in range(M):
            assert _rel(parts[m], s[m]) <= RTOL_NORM, (M, m)
        assert _rel(parts[M], ss / (M * M)) <= RTOL_NORM, M
        g.close()
        gb = D.GnsDevice(2, M, 2 * M, 0)
        gb.begin_step()
        gb.micro_sqnorm_batched(plan, bufs[:M], [0] * M, list(range(M)))
        pb = gb.partials()
        for m in range(M):
            assert _rel(pb[m], s[m]) <= RTOL_NORM, ("batched", M, m)
        assert np.all(pb[M:] == 0.0)
        gb.close()
    plan.close()


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
@pytest.mark.parametrize("form", ["fused", "inpass", "batched", "accumulate"])
def test_nonfinite_in_every_reduction_form(D, L, bad, form):
    """A non-finite element in a counted range makes the step a validation
    error (finalize leaves the state untouched) whatever reduction carried it
    — the fused TMA pass, its in-pass finalize, the batched K1 ring, the
    trainer form — while the same value inside a weight-0 range (a TP
    duplicate, never loaded) changes nothing."""
    n = 148 * 3584 + 4096
    M = 4
    hole = (200_000, 4096)
    segs = [(0, hole[0], 1.0), (hole[0], hole[1], 0.0), (hole[0] + hole[1], n - hole[0] - hole[1], 1.0)]
    plan = D.BucketPlan(segs, n, L.BF16, 0)
    for where, expect_error in ((123_457, True), (hole[0] + 100, False)):
        bufs = [torch.full((n,), 0.5, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
        bufs[2][where] = bad
        d = 2 if form == "batched" else 1
        g = D.GnsDevice(d, M, d * M, 0)
        st0 = g.get_state().as_tuple()
        g.begin_step()
        if form == "fused":
            g.fused_sqnorm(plan, bufs)
            g.finalize(M * 2048)
        elif form == "inpass":
            g.fused_sqnorm_finalize(plan, bufs, M * 2048)
        elif form == "batched":
            g.micro_sqnorm_batched(plan, bufs, [0] * M, list(range(M)))
            g.micro_sqnorm_batched(plan, [torch.full_like(bufs[0], 0.5)] * M, [1] * M, list(range(M)))
            sl0 = D.BucketPlan(segs, n, L.BF16, 0, slice_index=0, slice_count=2)
            sl1 = D.BucketPlan(segs, n, L.BF16, 0, slice_index=1, slice_count=2)
            mean = torch.full((n,), 0.5, dtype=torch.bfloat16, device="cuda")
            g.mean_sqnorm(sl0, mean)
            g.mean_sqnorm(sl1, mean)
            g.finalize(d * M * 2048)
        else:
            main = torch.zeros(n, dtype=torch.float32, device="cuda")
            for m in range(M):
                g.accumulate(plan, main, bufs[m], 0, m, first=m == 0, last_mean=m == M - 1)
            g.finalize(M * 2048)
        if expect_error:
            with pytest.raises(L.ValidationError):
                g.result()
            assert g.get_state().as_tuple() == st0
        else:
            r = g.result()
            assert r.status == 0
            parts = g.partials()
            assert np.all(np.isfinite(parts))
            counted = n - hole[1]
            assert parts[0] == 0.25 * counted  # 0.5^2 per counted element, exact
        g.close()
    plan.close()
