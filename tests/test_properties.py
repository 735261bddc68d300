"""Property tests (hypothesis) of the product's host API against the oracle:
the scalar estimator and the scorer agree bit-for-bit on arbitrary inputs."""
import math

import numpy as np
import pytest

hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

from oracle import oracle as O  # noqa: E402

pos = st.floats(min_value=0.0, max_value=1e30, allow_nan=False, allow_infinity=False)


@settings(max_examples=300, deadline=None)
@given(s=st.lists(pos, min_size=2, max_size=64), g2=pos, bg=st.integers(1, 4096),
       tokens=st.integers(0, 10 ** 9))
def test_finalize_and_ema_bit_identical(s, g2, bg, tokens):
    from paper_2604_26687_b200 import gns as G
    acc = G.StepAccumulator(1, bg)
    for v in s:
        acc.record_micro_batch(v)
    a = G.finalize_step(acc, g2)
    b = O.finalize_step(s, g2, bg)
    assert (a.signal, a.noise, a.noise_raw) == (b.signal, b.noise, b.noise_raw) or (
        math.isnan(a.signal) and math.isnan(b.signal))
    sp, so = G.GnsState.default(), O.State.default()
    for _ in range(3):
        G.update_ema(sp, a, tokens)
        O.update_ema(so, b, tokens)
    assert (sp.ema_signal, sp.ema_noise, sp.tokens_seen) == (so.ema_signal, so.ema_noise,
                                                             so.tokens_seen) or math.isnan(sp.ema_signal)
    pg, po = G.gns(sp), O.gns(so)
    assert pg == po or (pg is not None and math.isnan(pg) and math.isnan(po))


@settings(max_examples=200, deadline=None)
@given(phi=st.floats(min_value=0.0, max_value=1e5), ci=st.integers(0, 1000),
       elapsed=st.floats(min_value=1.0, max_value=1e6), frac=st.floats(min_value=0.0, max_value=1.0),
       cost=st.floats(min_value=0.0, max_value=1e4), margin=st.floats(min_value=0.0, max_value=0.5))
def test_decide_matches_oracle(phi, ci, elapsed, frac, cost, margin):
    from paper_2604_26687_b200 import gns as G
    costs = [(8, 1, 1, 4000.0, 256.0), (4, 2, 1, 3300.0, 96.0), (2, 2, 2, 2600.0, 40.0),
             (1, 8, 1, 1800.0, 8.0)]
    bg, bm = [16, 32, 64, 128, 256], [1, 2, 4]
    mine = G.synth_candidates(costs, bg, bm, True)
    ents = O.feasible_candidates(O.synth_profile(costs, bg, bm, True, 0.0, 0.0, 1e300))
    i = ci % len(mine)
    a = G.decide(mine, phi, mine[i], elapsed, elapsed * frac, margin=margin, reconfig_cost=cost)
    b = O.decide(ents, phi, ents[i], elapsed, elapsed * frac, margin=margin, reconfig_cost=cost)
    assert (a.kind, a.winner_index, a.winner_score, a.current_score) == (
        b.kind, b.winner_index, b.winner_score, b.current_score)
    order = G.rank_candidates(mine, phi, mine[i], elapsed, elapsed * frac, reconfig_cost=cost)
    sc = O.score_candidates(ents, phi, ents[i], elapsed, elapsed * frac, reconfig_cost=cost)
    assert all(sc[order[k]] >= sc[order[k + 1]] for k in range(len(order) - 1))
