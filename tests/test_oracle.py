"""Pins the CPU oracle (oracle/) to the reference's known answers.

The reference ships no tests or fixtures; its known-answer vectors are the
worked examples of SPEC.md (transcribed in tests/golden/spec_golden.json by
tests/golden/make_spec_golden.py) and its statistical properties
(acceptance #1/#2 at SPEC.md:657-658).
"""
import json
import math
import os
import sys

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_golden.json")))


def test_finalize_hand_worked_case_exact():
    # SPEC.md:181 / acceptance #2: exact match required.
    case = GOLD["finalize_step"][0]
    g = np.array(case["micro_gradients"], np.float64)
    s = [O.sumsq_f64(row) for row in g]
    mean = g.mean(axis=0)
    st = O.finalize_step(s, O.sumsq_f64(mean), case["global_batch"])
    e = case["expect"]
    assert sum(s) / len(s) == e["sbar"]
    assert st.mean_grad_sq == e["mean_grad_sq"]
    assert st.signal == e["signal"] and st.noise == e["noise"] and st.noise_raw == e["noise_raw"]


def test_finalize_identical_micro_gradients():
    case = GOLD["finalize_step"][1]
    g = np.array(case["micro_gradients"], np.float64)
    s = [O.sumsq_f64(row) for row in g]
    st = O.finalize_step(s, O.sumsq_f64(g.mean(axis=0)), case["global_batch"])
    assert st.noise == 0.0
    assert st.signal == case["expect"]["signal"]


def test_finalize_requires_two_samples():
    with pytest.raises(O.OracleError):
        O.finalize_step([9.0], 9.0, 1)


def test_finalize_rejects_negative_and_nan():
    with pytest.raises(O.OracleError):
        O.finalize_step([1.0, -1.0], 0.5, 2)
    with pytest.raises(O.OracleError):
        O.finalize_step([1.0, float("nan")], 0.5, 2)


def test_sample_variance_oracle():
    # unbiased per-component sample variance of {3,1} is 2;
    # per-sample trace with B_micro = B_g/N = 1 is 2.
    st = O.finalize_step([9.0, 1.0], 4.0, 2)
    assert st.noise == float(np.var([3.0, 1.0], ddof=1)) * 1


def test_update_ema_golden():
    case = GOLD["update_ema"][0]
    st = O.State.default()
    for step, exp in zip(case["steps"], case["expect_after"]):
        stats = O.Stats(step["signal"], step["noise"], step["noise"], 0.0)
        O.update_ema(st, stats, step["tokens"])
        assert st.ema_signal == pytest.approx(exp["ema_signal"], rel=1e-15)
        assert st.ema_noise == pytest.approx(exp["ema_noise"], rel=1e-15)
    assert st.tokens_seen == 8192


def test_update_ema_phase_switch():
    st = O.State.default()
    O.update_ema(st, O.Stats(1.0, 1.0, 1.0, 0.0), 8_000_000)
    # tokens_seen == boundary now -> alpha_late for the next update
    O.update_ema(st, O.Stats(2.0, 1.0, 1.0, 0.0), 1)
    assert st.ema_signal == 0.99 * 1.0 + (1 - 0.99) * 2.0
    # one token short of the boundary -> still alpha_early
    st2 = O.State.default()
    O.update_ema(st2, O.Stats(1.0, 1.0, 1.0, 0.0), 7_999_999)
    O.update_ema(st2, O.Stats(2.0, 1.0, 1.0, 0.0), 1)
    assert st2.ema_signal == 0.95 * 1.0 + (1 - 0.95) * 2.0


def test_update_ema_feeds_clamped_noise():
    # the clamped noise is what enters the EMA
    st = O.State.default()
    O.update_ema(st, O.Stats(1.0, 0.0, -3.0, 0.0), 10)
    assert st.ema_noise == 0.0


@pytest.mark.parametrize("case", GOLD["gns"])
def test_gns_golden(case):
    st = O.State.default()
    st.ema_signal, st.ema_noise, st.calibration = case["ema_signal"], case["ema_noise"], case["calibration"]
    st.initialized = 1
    phi = O.gns(st)
    if case["expect"] is None:
        assert phi is None
    else:
        assert phi == pytest.approx(case["expect"], rel=1e-15)


def test_scorer_golden():
    for c in GOLD["stat_eff"]:
        assert O.stat_eff(c["B_g"], c["phi"]) == pytest.approx(c["expect"], rel=1e-15)
    for c in GOLD["goodput"]:
        assert O.goodput(c["T"], c["se"]) == c["expect"]
    for c in GOLD["goodput_lr"]:
        assert O.goodput_lr(c["T"], c["B_g"], c["phi"], c["ref"]) == pytest.approx(c["expect"], rel=1e-15)
    for c in GOLD["lr_rescale"]:
        assert O.lr_rescale(c["eta"], c["b_old"], c["b_new"]) == pytest.approx(c["expect"], rel=1e-15)
    for c in GOLD["optimal_batch_continuous"]:
        assert O.optimal_batch_continuous(c["b_hw"], c["b_crit"]) == c["expect"]
    for c in GOLD["cbs_target"]:
        assert O.cbs_target(c["phi"], c["cands"]) == c["expect"]


def test_cbs_tie_goes_to_smaller():
    # phi at the geometric midpoint of 32 and 64 -> 32
    assert O.cbs_target(math.sqrt(32 * 64), [16, 32, 64]) == 32


def test_synth_profile_golden():
    c = GOLD["synth_profile"][0]
    ents = O.synth_profile([(1, 1, 1, c["t_max"], c["b_hw"])], [c["B_g"]], [1], False, 0.0, 0.0, 1e30)
    assert ents[0].throughput == c["expect_T"]
    # bubble: p=4, GA=1 -> 1/4 ; GA=16 -> 16/19
    e = O.synth_profile([(1, 1, 4, 1000.0, 0.0)], [1, 16], [1], True, 0.0, 0.0, 1e30)
    assert e[0].throughput == pytest.approx(1000.0 * 0.25, rel=1e-15)
    assert e[1].throughput == pytest.approx(1000.0 * 16 / 19, rel=1e-15)


def test_feasible_candidates_counting():
    # SPEC.md:110-112
    ents = O.synth_profile([(2, 1, 1, 1000.0, 64.0), (1, 2, 1, 800.0, 16.0)], [16, 32, 64], [1, 2],
                           False, 0.0, 0.0, 1e30)
    cands = O.feasible_candidates(ents)
    assert len(cands) == 6
    keys = [(c.global_batch, c.d, c.t, c.p) for c in cands]
    assert keys == sorted(keys)
    # infeasible (S, B_g) excluded
    ents2 = O.synth_profile([(2, 1, 1, 1000.0, 64.0)], [16, 32], [1, 2], False, 100.0, 10.0, 105.0)
    assert all(c.micro_batch == 1 for c in O.feasible_candidates(ents2))


def _decide_case(c):
    # phi = 0, ref = 16: goodput_lr = T / sqrt(B_g * 16)
    cur = O.Entry(d=2, t=1, p=1, global_batch=16, micro_batch=1, throughput=1600.0, feasible=1)
    cand_bg = 32
    T = c["cand_score"] * math.sqrt(cand_bg * 16)
    cand = O.Entry(d=2 if c["same_strategy"] else 1, t=1 if c["same_strategy"] else 2, p=1,
                   global_batch=cand_bg, micro_batch=1, throughput=T, feasible=1)
    return [cur, cand], cur


@pytest.mark.parametrize("c", GOLD["decide"])
def test_decide_golden(c):
    cands, cur = _decide_case(c)
    cmd = O.decide(cands, 0.0, cur, c["elapsed"], c["useful"], margin=0.10,
                   reconfig_cost=c["reconfig_cost"], reference_batch=16.0)
    kind = {O.NOOP: "NoOp", O.SCALE_BS: "ScaleBS", O.RECONFIGURE: "Reconfigure"}[cmd.kind]
    assert kind == c["expect"]
    assert cmd.current_score == pytest.approx(100.0, rel=1e-14)
    if "expect_winner_score" in c:
        assert cmd.winner_score == pytest.approx(c["expect_winner_score"], rel=1e-12)
    if "expect_winner_score_max" in c:
        assert cmd.winner_score <= c["expect_winner_score_max"] + 1e-9


def test_decide_phi_unavailable_is_noop():
    cands, cur = _decide_case(GOLD["decide"][1])
    assert O.decide(cands, None, cur, 1.0, 1.0).kind == O.NOOP


# ---------------------------------------------------------------- properties

def _simulate_steps(n_steps, n_dim, M, B_m, seed):
    rng = np.random.default_rng(seed)
    g_true = rng.normal(size=n_dim) * 0.5
    sigma = rng.uniform(0.5, 2.0, size=n_dim)
    sig, noi = [], []
    for k in range(n_steps):
        g = O.simulate_micro_gradients(g_true, sigma, B_m, M, seed * 100003 + k)
        s = [O.sumsq_f64(r) for r in g]
        st = O.finalize_step(s, O.sumsq_f64(g.mean(axis=0)), M * B_m)
        sig.append(st.signal)
        noi.append(st.noise_raw)
    return g_true, sigma, np.array(sig), np.array(noi)


def test_unbiasedness_three_standard_errors():
    # SPEC.md:216 / acceptance #1, 10^4 trials
    g_true, sigma, sig, noi = _simulate_steps(10_000, 4, 4, 2, 7)
    se_s = sig.std(ddof=1) / math.sqrt(sig.size)
    se_n = noi.std(ddof=1) / math.sqrt(noi.size)
    assert abs(sig.mean() - float(g_true @ g_true)) < 3 * se_s
    assert abs(noi.mean() - float(sigma.sum())) < 3 * se_n


def test_split_invariance_and_scale_equivariance():
    # SPEC.md:217-218
    rng = np.random.default_rng(3)
    g = rng.normal(size=(8, 5))
    s = [O.sumsq_f64(r) for r in g]
    gb2 = O.sumsq_f64(g.mean(axis=0))
    a = O.finalize_step(s, gb2, 16)
    b = O.finalize_step(list(reversed(s)), gb2, 16)  # relabel ranks / micro-batches
    assert a.signal == pytest.approx(b.signal, rel=1e-14)
    k = 3.0
    c = O.finalize_step([x * k * k for x in s], gb2 * k * k, 16)
    assert c.signal == pytest.approx(a.signal * k * k, rel=1e-12)
    assert c.noise == pytest.approx(a.noise * k * k, rel=1e-12)


def test_ema_convex_hull():
    # SPEC.md:219
    rng = np.random.default_rng(5)
    st = O.State.default()
    raws = []
    for i in range(300):
        x = float(rng.normal(2.0, 1.0))
        raws.append(x)
        O.update_ema(st, O.Stats(x, 1.0, 1.0, 0.0), 100_000)
        assert min(raws) - 1e-12 <= st.ema_signal <= max(raws) + 1e-12


def test_smoothed_phi_converges_within_10pct():
    # SPEC.md:212 / acceptance #1: c = 1 smoothed phi within 10% after 2000 steps
    rng = np.random.default_rng(11)
    n = 16
    g_true = rng.normal(size=n)
    sigma = np.full(n, 0.25)
    true_phi = sigma.sum() / float(g_true @ g_true)
    st = O.State.default()
    st.calibration = 1.0
    M, B_m = 8, 1
    for k in range(2000):
        g = O.simulate_micro_gradients(g_true, sigma, B_m, M, 1000 + k)
        s = [O.sumsq_f64(r) for r in g]
        stats = O.finalize_step(s, O.sumsq_f64(g.mean(axis=0)), M * B_m)
        O.update_ema(st, stats, M * B_m * 2048)
    assert abs(O.gns(st) - true_phi) / true_phi < 0.10


def test_simulate_noiseless_and_variance_halving():
    g_true = np.array([1.0, -2.0, 0.5])
    out = O.simulate_micro_gradients(g_true, np.zeros(3), 4, 10, 1)
    assert np.array_equal(out, np.tile(g_true, (10, 1)))
    sig = np.array([1.0, 1.0, 1.0])
    v1 = O.simulate_micro_gradients(g_true, sig, 1, 10_000, 2).var(axis=0).mean()
    v2 = O.simulate_micro_gradients(g_true, sig, 2, 10_000, 3).var(axis=0).mean()
    assert v1 / v2 == pytest.approx(2.0, rel=0.06)


# ---------------------------------------------------------------- norms + generator

def test_sqnorm_bf16_exact_small():
    x = np.array([0x3F80, 0x4000, 0xBF80, 0x0000], np.uint16)  # 1, 2, -1, 0
    assert O.sqnorm(x, O.BF16, [(0, 4, 1.0)]) == 6.0
    assert O.sqnorm(x, O.BF16, [(0, 2, 1.0), (2, 2, 0.0)]) == 5.0
    assert O.sqnorm_mt(x, O.BF16, [(0, 4, 1.0)], 4) == 6.0


def test_sqnorm_mt_matches_sequential():
    gs = [(0, 3_000_001, 0, 3_000_001, 3_000_001)]
    unit = O.noise_unit_for(2 ** -10, 256.0, 1)
    x = O.synth_fill(3_000_001, O.BF16, gs, 42, 0, 2 ** -10, unit)
    segs = [(0, 1_000_003, 1.0), (1_000_003, 5, 0.0), (1_000_008, 1_999_993, 1.0)]
    a = O.sqnorm(x, O.BF16, segs)
    b = O.sqnorm_mt(x, O.BF16, segs, 8)
    assert b == pytest.approx(a, rel=1e-13)


def test_generator_statistics_and_determinism():
    g0 = 2.0 ** -10
    unit = O.noise_unit_for(g0, 64.0, 1)
    gs = [(0, 200_000, 0, 200_000, 200_000)]
    a = O.synth_fill(200_000, O.FP32, gs, 9, 3, g0, unit)
    b = O.synth_fill(200_000, O.FP32, gs, 9, 3, g0, unit)
    assert O.fnv1a(a) == O.fnv1a(b)
    # mean of |G| sign pattern ~ 0, noise std ~ 8 g0
    assert abs(a.mean()) < 0.05 * g0 * 8
    assert a.std() == pytest.approx(math.sqrt(g0 ** 2 + 64 * g0 ** 2), rel=0.02)
    # a different sample index gives different noise but the same G signs
    c = O.synth_fill(200_000, O.FP32, gs, 9, 4, g0, unit)
    assert O.fnv1a(a) != O.fnv1a(c)


def test_generator_layout_independence():
    # a row-split shard of a [R, C] tensor equals the same elements of the full tensor
    R, Cc, t = 6, 8, 2
    full = O.synth_fill(R * Cc, O.BF16, [(0, R * Cc, 100, Cc, Cc)], 1, 5, 2 ** -10, 1e-6)
    for r in range(t):
        cs = Cc // t
        part = O.synth_fill(R * cs, O.BF16, [(0, R * cs, 100 + r * cs, cs, Cc)], 1, 5, 2 ** -10, 1e-6)
        assert np.array_equal(part, full.reshape(R, Cc)[:, r * cs:(r + 1) * cs].reshape(-1))


def test_fused_matches_separate_passes():
    g0 = 2.0 ** -10
    unit = O.noise_unit_for(g0, 256.0, 1)
    n = 100_003
    gs = [(0, n, 0, n, n)]
    bufs = [O.synth_fill(n, O.BF16, gs, 4, m, g0, unit) for m in range(4)]
    segs = [(0, 50_000, 1.0), (50_000, 3, 0.0), (50_003, n - 50_003, 1.0)]
    s, ss = O.fused_sqnorms(bufs, O.BF16, segs, 4)
    for m in range(4):
        assert s[m] == pytest.approx(O.sqnorm(bufs[m], O.BF16, segs), rel=1e-13)
    f = np.stack([b.astype(np.uint32) << 16 for b in bufs]).view(np.float32)
    acc = np.zeros(n, np.float32)
    for m in range(4):
        acc = acc + f[m]
    w = np.ones(n)
    w[50_000:50_003] = 0
    assert ss == pytest.approx(float((w * acc.astype(np.float64) ** 2).sum()), rel=1e-12)


def test_window_crop_helpers_reproduce_whole_bucket():
    """tests/test_gpu_fullsize_oracle.py reduces full-size buckets window by
    window; its crop helpers must reproduce the whole-bucket generator bytes
    and segment sums for every cut, including cuts inside a TP-split row."""
    import numpy as np
    from paper_2604_26687_b200 import layout as Lay
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_gpu_fullsize_oracle import crop_gen, crop_segments
    spec = Lay.tiny_model(layers=4, h=64, ffn=128, vocab=96)
    for d, t, p in [(1, 2, 2), (2, 2, 1), (1, 4, 1)]:
        for lay in Lay.world_layouts(spec, d, t, p):
            full = O.synth_fill(lay.numel, O.BF16, lay.gen, 7, 3, Lay.G0, 1e-6)
            cuts = [(0, lay.numel), (13, 777), (1000, lay.numel - 5),
                    (lay.numel // 3, lay.numel // 3 + 4097)]
            for a, b in cuts:
                w = O.synth_fill(b - a, O.BF16, crop_gen(lay.gen, a, b), 7, 3, Lay.G0, 1e-6)
                assert np.array_equal(w, full[a:b])
                s1 = O.sqnorm(full[a:b], O.BF16, crop_segments(lay.segments, a, b))
                s2 = O.sqnorm(full, O.BF16, [(o + a, k, x) for o, k, x in
                                              crop_segments(lay.segments, a, b)])
                assert s1 == s2
