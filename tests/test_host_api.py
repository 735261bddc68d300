"""CPU tests of the product's host side: the C-ABI library loads and exports
every declared symbol, and the C++ implementation of the reference API
(gns.hpp / goodput.hpp / decide) matches the spec goldens and the oracle
bit-for-bit.  No device calls."""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_golden.json")))


@pytest.fixture(scope="module")
def G():
    from paper_2604_26687_b200 import gns
    return gns


@pytest.fixture(scope="module")
def L():
    from paper_2604_26687_b200 import _lib
    return _lib


def test_library_exports_every_declared_symbol(L):
    lib = L.lib()
    declared = L.header_symbols()
    assert len(declared) >= 45
    missing = [s for s in declared if not hasattr(lib, s)]
    assert missing == []
    assert set(L.SIGNATURES) == set(declared)
    assert lib.coadapt_abi_version() == 1


def test_reference_headers_declare_the_same_api():
    # our include/coadapt/*.hpp keep every reference declaration (drop-in)
    ours = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "coadapt")
    for h in ("gns.hpp", "goodput.hpp", "strategy.hpp", "io.hpp", "errors.hpp"):
        text = open(os.path.join(ours, h)).read()
        for sym in {"gns.hpp": ["StepAccumulator(int dp_size, std::int64_t global_batch)",
                                "void record_micro_batch(double squared_norm)",
                                "StepStats finalize_step(const StepAccumulator& acc,\n                        std::span<const double> mean_gradient)",
                                "StepStats finalize_step(const StepAccumulator& acc, double mean_grad_sq)",
                                "void update_ema(GnsState& state, const StepStats& stats,\n                std::int64_t tokens_this_step)",
                                "std::optional<double> gns(const GnsState& state)",
                                "std::string gns_trace_csv(std::span<const GnsTraceRow> rows)"],
                    "goodput.hpp": ["double stat_eff(double global_batch, double phi)",
                                    "double goodput(double throughput, double stat_efficiency)",
                                    "std::int64_t cbs_target(double phi, std::span<const std::int64_t> candidates,\n                        CbsDistance metric = CbsDistance::kLog)"],
                    "strategy.hpp": ["void validate_config(const ConfigTuple& c, int n_gpus)",
                                     "ParallelStrategy parse_strategy_label(const std::string& text)"],
                    "io.hpp": ["std::string format_double(double v)",
                               "std::vector<std::string_view> split_csv_line(std::string_view line)"],
                    "errors.hpp": ["class ValidationError : public std::runtime_error",
                                   "class InternalError : public std::logic_error"]}[h]:
            assert sym in text, (h, sym)


def test_finalize_golden_and_errors(G, L):
    acc = G.StepAccumulator(1, 2)
    acc.record_micro_batch(9.0)
    acc.record_micro_batch(1.0)
    st = G.finalize_step(acc, 4.0)
    assert (st.signal, st.noise, st.noise_raw, st.mean_grad_sq) == (3.0, 2.0, 2.0, 4.0)
    with pytest.raises(L.ValidationError):
        acc.record_micro_batch(-1.0)
    one = G.StepAccumulator(1, 1)
    one.record_micro_batch(9.0)
    with pytest.raises(L.ValidationError):
        G.finalize_step(one, 9.0)
    acc3 = G.StepAccumulator(2, 8)
    for v in (4.0, 0.25, 7.0):
        acc3.record_micro_batch(v)
    assert list(acc3.squared_norms()) == [4.0, 0.25, 7.0]
    assert acc3.sample_count() == 3 and acc3.micro_count() == 1


def test_host_estimator_bit_exact_with_oracle(G):
    rng = np.random.default_rng(1)
    st_o = O.State.default()
    st_p = G.GnsState.default()
    for k in range(300):
        s = rng.uniform(0.5, 2.0, size=16)
        g2 = float(rng.uniform(0.0, 0.2))
        acc = G.StepAccumulator(2, 32)
        for v in s:
            acc.record_micro_batch(v)
        a = G.finalize_step(acc, g2)
        b = O.finalize_step(s, g2, 32)
        assert (a.signal, a.noise, a.noise_raw) == (b.signal, b.noise, b.noise_raw)
        G.update_ema(st_p, a, 200_000)
        O.update_ema(st_o, b, 200_000)
        assert (st_p.ema_signal, st_p.ema_noise, st_p.tokens_seen) == (st_o.ema_signal, st_o.ema_noise,
                                                                       st_o.tokens_seen)
        assert G.gns(st_p) == O.gns(st_o)


def test_gns_golden(G):
    for case in GOLD["gns"]:
        st = G.GnsState.default()
        st.ema_signal, st.ema_noise, st.calibration, st.initialized = (
            case["ema_signal"], case["ema_noise"], case["calibration"], 1)
        phi = G.gns(st)
        assert phi == (None if case["expect"] is None else pytest.approx(case["expect"], rel=1e-15))


def test_goodput_golden(G):
    for c in GOLD["stat_eff"]:
        assert G.stat_eff(c["B_g"], c["phi"]) == pytest.approx(c["expect"], rel=1e-15)
    assert G.goodput(500.0, 0.5) == 250.0
    assert G.goodput_lr(500.0, 64.0, 64.0, 16.0) == 507.8125
    assert G.lr_rescale(2e-4, 16, 64) == pytest.approx(4e-4, rel=1e-15)
    assert G.lr_rescale(G.lr_rescale(2e-4, 16, 32), 32, 64) == pytest.approx(4e-4, rel=1e-15)
    assert G.optimal_batch_continuous(64, 256) == 128.0
    assert G.cbs_target(48.0, [16, 32, 64]) == 64
    assert G.cbs_target(0.0, [16, 32, 64]) == 16
    assert G.cbs_target(math.sqrt(32 * 64), [16, 32, 64]) == 32
    assert G.cbs_target(48.0, [16, 32, 64], linear=True) == 32


def _cur_and_cand(same, score):
    from paper_2604_26687_b200.gns import Candidate
    cur = Candidate(2, 1, 1, 16, 1, 1600.0)
    cand = Candidate(2 if same else 1, 1 if same else 2, 1, 32, 1, score * math.sqrt(32 * 16))
    return [cur, cand], cur


@pytest.mark.parametrize("c", GOLD["decide"])
def test_decide_golden(G, c):
    cands, cur = _cur_and_cand(c["same_strategy"], c["cand_score"])
    cmd = G.decide(cands, 0.0, cur, c["elapsed"], c["useful"], reconfig_cost=c["reconfig_cost"])
    assert cmd.name == c["expect"]


def test_decide_properties(G):
    from paper_2604_26687_b200.gns import Candidate
    costs = [(8, 1, 1, 4000.0, 256.0), (4, 2, 1, 3300.0, 96.0), (2, 2, 2, 2600.0, 40.0)]
    cands = G.synth_candidates(costs, [16, 32, 64, 128, 256, 512], [1, 2, 4], True)
    rng = np.random.default_rng(4)
    for _ in range(200):
        phi = float(rng.uniform(1, 3000))
        cur = cands[int(rng.integers(len(cands)))]
        cmd = G.decide(cands, phi, cur, 1000.0, 1000.0, reconfig_cost=30.0)
        # growth clamp
        if cmd.kind != 0:
            win = cands[cmd.winner_index]
            assert win.global_batch <= 2 * cur.global_batch
        # hysteresis.  Only holds when the growth clamp does not
        # bind: SPEC.md:397 lets consecutive clamped decisions compound.
        free = G.decide(cands, phi, cur, 1000.0, 1000.0, reconfig_cost=30.0, max_growth=1e9)
        if free.kind != 0:
            again = G.decide(cands, phi, cands[free.winner_index], 1000.0, 1000.0,
                             reconfig_cost=30.0, max_growth=1e9)
            assert again.kind == 0
        # scale invariance
        scaled = [Candidate(c.d, c.t, c.p, c.global_batch, c.micro_batch, 3.0 * c.throughput) for c in cands]
        cur2 = scaled[cands.index(cur)]
        cmd2 = G.decide(scaled, phi, cur2, 1000.0, 1000.0, reconfig_cost=30.0)
        assert (cmd2.kind, cmd2.winner_index) == (cmd.kind, cmd.winner_index)


def test_candidates_and_ranking_match_oracle(G):
    costs = [(8, 1, 1, 4000.0, 256.0), (4, 2, 1, 3300.0, 96.0), (2, 2, 2, 2600.0, 40.0),
             (1, 4, 2, 2000.0, 16.0), (2, 4, 1, 2400.0, 32.0), (1, 8, 1, 1800.0, 8.0)]
    bg, bm = [16, 32, 64, 128, 256, 512, 1024, 2048], [1, 2, 4, 8]
    mine = G.synth_candidates(costs, bg, bm, True, 64e9, 1e9, 80e9)
    ents = O.feasible_candidates(O.synth_profile(costs, bg, bm, True, 64e9, 1e9, 80e9))
    assert [(c.key(), c.throughput) for c in mine] == [
        ((e.d, e.t, e.p, e.global_batch, e.micro_batch), e.throughput) for e in ents]
    for phi in (1.0, 37.0, 512.0, 4096.0):
        for ci in (0, 7, 20):
            sc = G.score_candidates(mine, phi, mine[ci], 500.0, 400.0, reconfig_cost=40.0)
            so = O.score_candidates(ents, phi, ents[ci], 500.0, 400.0, reconfig_cost=40.0)
            assert np.array_equal(sc, so)
            a = G.decide(mine, phi, mine[ci], 500.0, 400.0, reconfig_cost=40.0)
            b = O.decide(ents, phi, ents[ci], 500.0, 400.0, reconfig_cost=40.0)
            assert (a.kind, a.winner_index, a.winner_score, a.current_score) == (
                b.kind, b.winner_index, b.winner_score, b.current_score)


def test_trace_csv_is_byte_exact(G):
    rows = [G.GnsTraceRow(1, 4096, 3.0, 2.0, 3.0, 2.0, float("nan")),
            G.GnsTraceRow(2, 8192, 0.1, -0.5, 3.1, 2.0, 4.0 / 3.0)]
    text = G.gns_trace_csv(rows)
    assert text == ("step,tokens,signal_raw,noise_raw,ema_signal,ema_noise,phi\n"
                    "1,4096,3,2,3,2,nan\n2,8192,0.1,-0.5,3.1,2,1.3333333333333333\n")
    for v in (0.1, 1e-300, 123456789.125, 2.0 ** -1074):
        assert float(G.format_double(v)) == v


def test_simulate_micro_gradients_properties(G):
    g_true = np.array([1.0, -2.0, 0.5, 3.0])
    out = G.simulate_micro_gradients(g_true, np.zeros(4), 4, 5, 1)
    assert np.array_equal(out, np.tile(g_true, (5, 1)))
    a = G.simulate_micro_gradients(g_true, np.ones(4), 1, 20_000, 2)
    b = G.simulate_micro_gradients(g_true, np.ones(4), 2, 20_000, 3)
    assert np.allclose(a.mean(axis=0), g_true, atol=0.05)
    assert a.var(axis=0).mean() / b.var(axis=0).mean() == pytest.approx(2.0, rel=0.05)
    assert np.array_equal(a, G.simulate_micro_gradients(g_true, np.ones(4), 1, 20_000, 2))


def test_layout_counts_match_survey():
    from paper_2604_26687_b200 import layout as Lay
    # SURVEY App. B.1 parameter counts
    assert abs(Lay.llama32_3b().numel() - 3212.75e6) < 0.01e6
    assert abs(Lay.llama2_7b().numel() - 6738.42e6) < 0.01e6
    assert abs(Lay.qwen25_32b().numel() - 32763.88e6) < 0.01e6
    # C4: (1,4,2) -> each rank counts ~4095.7 M (+ replicated norms on tp 0)
    lays = Lay.world_layouts(Lay.qwen25_32b(), 1, 4, 2)
    assert sum(l.counted for l in lays) == Lay.qwen25_32b().numel()
    lays = Lay.world_layouts(Lay.llama32_3b(), 2, 2, 2)
    assert sum(l.counted for l in lays if l.coords[0] == 0) == Lay.llama32_3b().numel()
    lays = Lay.world_layouts(Lay.gpt2_small(), 1, 2, 2)
    assert sum(l.counted for l in lays) == Lay.gpt2_small().numel()


def test_layout_generator_covers_every_parameter_once():
    from paper_2604_26687_b200 import layout as Lay
    spec = Lay.tiny_model(layers=4, h=16, ffn=32, vocab=24, tied=True)
    for (d, t, p) in [(1, 1, 1), (1, 2, 2), (2, 4, 1), (1, 1, 4)]:
        seen = np.zeros(spec.numel(), np.int64)
        for lay in Lay.world_layouts(spec, d, t, p):
            if lay.coords[0]:
                continue
            w = {}
            for off, n, wt in lay.segments:
                w[off] = wt
            for (off, n, base, rl, rs) in lay.gen:
                if w[off] == 0.0:
                    continue
                j = np.arange(n)
                seen[base + (j // rl) * rs + (j % rl)] += 1
        assert (seen == 1).all(), (d, t, p)


def test_record_reconfig_spec_examples(G):
    """SPEC.md:377-385, through the C++ API (C-ABI) and the oracle."""
    from oracle import oracle as O
    clock = G.ClockState(elapsed=600.0, useful=600.0)
    cost = G.record_reconfig(clock, 50.0, reconfig_cost=40.0)
    assert (clock.useful, clock.elapsed) == (600.0, 650.0) and cost == 50.0
    clock = G.ClockState()
    G.record_reconfig(clock, 30.0)
    assert G.record_reconfig(clock, 56.0) == 43.0
    clock = G.ClockState(elapsed=10.0, useful=8.0)
    cost = G.record_reconfig(clock, 0.0, reconfig_cost=40.0)
    assert (clock.elapsed, clock.useful) == (10.0, 8.0) and cost == 0.0
    with pytest.raises(G.ValidationError):
        G.record_reconfig(clock, -1.0)
    # random sequences agree with the oracle bit for bit
    rng = np.random.default_rng(3)
    c, o = G.ClockState(5.0, 4.0), (5.0, 4.0, 0.0, 0, 7.0)
    cost = 7.0
    for lat in rng.uniform(0, 90, 50):
        cost = G.record_reconfig(c, lat, cost)
        o = O.record_reconfig(*o, lat)
        assert (c.elapsed, c.useful, c.reconfig_total, c.reconfigs, cost) == o


def test_python_wrappers_validate_bucket_tensors():
    """tensors handed to the device wrappers are checked against
    the plan (dtype, contiguity, element count, device) before any launch."""
    import types
    import torch
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import _lib as LL
    plan = types.SimpleNamespace(dtype=LL.BF16, bucket_numel=64, device=0)
    with pytest.raises(LL.ValidationError, match="dtype"):
        D._bucket(plan, torch.zeros(64, dtype=torch.float32))
    with pytest.raises(LL.ValidationError, match="contiguous"):
        D._bucket(plan, torch.zeros(128, dtype=torch.bfloat16)[::2])
    with pytest.raises(LL.ValidationError, match="elements"):
        D._bucket(plan, torch.zeros(63, dtype=torch.bfloat16))
    with pytest.raises(LL.ValidationError, match="cuda:0"):
        D._bucket(plan, torch.zeros(64, dtype=torch.bfloat16))  # host tensor, device plan
    host = torch.zeros(64, dtype=torch.bfloat16)
    assert D._bucket(plan, host, host=True) == host.data_ptr()
    assert D._bucket(plan, 1234) == 1234  # raw (e.g. CUDA-IPC) addresses pass through


def test_candidate_table_decides_like_the_list():
    """gns.CandidateTable (marshalled once) gives the same Command, scores
    and ranking as passing the candidate list."""
    from paper_2604_26687_b200 import gns as G
    costs = [(d, t, 8 // (d * t), 1000.0 * d ** 0.5 * (1 + 0.2 * t), 8.0 * d * d + 4.0 * (8 // (d * t)))
             for d in (1, 2, 4, 8) for t in (1, 2, 4, 8) if 8 % (d * t) == 0]
    c = G.synth_candidates(costs, [16, 32, 64, 128, 256, 512, 1024, 2048], [1, 2, 4, 8], True)
    tab = G.CandidateTable(c)
    assert len(tab) == len(c) and tab[3] == c[3] and list(tab) == c
    for phi in (None, 3.0, 500.0, 1e5):
        for cur in (c[0], c[len(c) // 2]):
            assert G.decide(tab, phi, cur, 1000.0, 900.0, reconfig_cost=40.0) == \
                G.decide(c, phi, cur, 1000.0, 900.0, reconfig_cost=40.0)
    assert list(G.score_candidates(tab, 500.0, c[1], 1000.0, 900.0)) == \
        list(G.score_candidates(c, 500.0, c[1], 1000.0, 900.0))
    assert G.rank_candidates(tab, 500.0, c[1], 1000.0, 900.0) == \
        G.rank_candidates(c, 500.0, c[1], 1000.0, 900.0)


def test_round2_entry_points_validate_without_a_device():
    """The round-2 C-ABI entry points reject bad arguments with status 1
    before touching a device (usable as a CPU-side contract check)."""
    import ctypes as C
    from paper_2604_26687_b200 import _lib as LL
    lib = LL.lib()
    ptrs = (C.c_void_p * 1)()
    assert lib.coadapt_gns_fused_sqnorm_finalize(None, None, ptrs, 1, 2048, None) == LL.E_VALIDATION
    assert lib.coadapt_gns_mean_sqnorm_finalize(None, None, None, 2048, None) == LL.E_VALIDATION
    assert lib.coadapt_gns_nvls_reduce_sqnorm(None, None, None, 2, 0, None, 0.5, None) == LL.E_VALIDATION
    assert b"NULL" in lib.coadapt_last_error()
