"""SPEC.md's GNS properties and acceptance criterion #1 through the DEVICE
path (K0 generator -> K1f / K1 + K2 -> K3 finalize/EMA/phi), not the oracle.

* Unbiasedness (acceptance #1): over 10^4 device steps the
  mean of StepStats.signal is within 3 standard errors of |G|^2 and the mean
  of noise_raw within 3 standard errors of tr(Sigma).
* Split invariance: the same N micro-gradients and mean
  gradient, labelled as (d, M) = (1,8), (2,4), (4,2), (8,1) or permuted,
  give the same statistics (to fp64 reassociation of the slot sum).
* Scale equivariance: micro-gradients x 2 (exact in bf16)
  multiply signal and noise by 4 exactly and leave phi bit-identical.
* EMA convex hull: the device ema_signal / ema_noise stay
  inside the hull of the raw values the device produced.
* Acceptance #1: with c = 1 the device's smoothed phi is
  within 10 % of tr(Sigma)/|G|^2 after 2000 steps.

Source: the integer-exact generator (coadapt_synth_fill) — x = G_i + zeta,
G_i = +-g0 (sign hashed from the global index, fixed across samples),
zeta Irwin-Hall(4) with Var = phi_true g0^2 / B_m — so |G|^2 = n g0^2 and
tr(Sigma) = n phi_true g0^2 over the n counted elements; each
step draws fresh samples (sample index = step * N + n).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _setup(phi_true, Bm=1):
    from paper_2604_26687_b200 import _lib as L
    from paper_2604_26687_b200 import device as D
    from paper_2604_26687_b200 import layout as Lay
    torch.cuda.set_device(0)
    spec = Lay.tiny_model(layers=4, h=64, ffn=128, vocab=96)
    lay = Lay.rank_layout(spec, 1, 2, 2, 1)  # tp_rank 1: replicated norms at weight 0
    plan = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0)
    unit = Lay.noise_unit_for(phi_true, Bm)
    return L, D, Lay, lay, plan, unit


def _fill(D, Lay, bufs, lay, seed, sample0, unit):
    for j, b in enumerate(bufs):
        D.synth_fill(b, lay.gen, seed, sample0 + j, Lay.G0, unit)


def test_unbiasedness_10k_device_steps():
    phi_true, M, trials, seed = 16.0, 8, 10_000, 0xACC1
    L, D, Lay, lay, plan, unit = _setup(phi_true)
    bufs = [torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    g = D.GnsDevice(1, M, M, 0)
    sig, noi = np.empty(trials), np.empty(trials)
    for k in range(trials):
        _fill(D, Lay, bufs, lay, seed, k * M, unit)
        g.begin_step()
        g.fused_sqnorm(plan, bufs)
        g.finalize(M * 2048)
        r = g.result()
        sig[k], noi[k] = r.stats.signal, r.stats.noise_raw
    n = lay.counted
    g2_true = n * Lay.G0 ** 2
    tr_true = n * phi_true * Lay.G0 ** 2
    se_s = sig.std(ddof=1) / math.sqrt(trials)
    se_n = noi.std(ddof=1) / math.sqrt(trials)
    assert abs(sig.mean() - g2_true) < 3 * se_s, (sig.mean(), g2_true, se_s)
    assert abs(noi.mean() - tr_true) < 3 * se_n, (noi.mean(), tr_true, se_n)


def test_split_invariance_across_d_and_labels():
    N, seed = 8, 0xACC2
    L, D, Lay, lay, plan, unit = _setup(64.0)
    bufs = [torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda") for _ in range(N)]
    _fill(D, Lay, bufs, lay, seed, 0, unit)
    mean = torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda")
    D.synth_mean_fill(mean, lay.gen, seed, 0, N, Lay.G0, unit)
    B_g = 2 * N
    out = {}
    perm = [5, 2, 7, 0, 3, 6, 1, 4]
    for d in (1, 2, 4, 8):
        for order in ("id", "perm"):
            M = N // d
            g = D.GnsDevice(d, M, B_g, 0)
            g.begin_step()
            idx = list(range(N)) if order == "id" else perm
            for slot, j in enumerate(idx):
                g.micro_sqnorm(plan, bufs[j], slot // M, slot % M)
            for i_d in range(d):  # K2: every DP replica's slice of the mean
                sl = D.BucketPlan(lay.segments, lay.numel, L.BF16, 0, slice_index=i_d, slice_count=d)
                g.mean_sqnorm(sl, mean)
                torch.cuda.synchronize()
                sl.close()
            g.finalize(B_g * 2048)
            r = g.result()
            out[(d, order)] = (r.stats.signal, r.stats.noise, r.b_simple)
            g.close()
    ref = out[(1, "id")]
    for key, v in out.items():
        assert v == pytest.approx(ref, rel=1e-13), (key, v, ref)


def test_scale_equivariance_exact():
    M, seed = 8, 0xACC3
    L, D, Lay, lay, plan, unit = _setup(64.0)
    bufs = [torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    _fill(D, Lay, bufs, lay, seed, 0, unit)
    res = {}
    for k in (1.0, 2.0, 0.5):
        scaled = [b * k for b in bufs]  # powers of two: exact in bf16
        g = D.GnsDevice(1, M, M, 0)
        g.begin_step()
        g.fused_sqnorm(plan, scaled)
        g.finalize(M * 2048)
        r = g.result()
        res[k] = (r.stats.signal, r.stats.noise, r.b_simple)
        g.close()
    s1, n1, b1 = res[1.0]
    for k in (2.0, 0.5):
        s, n, b = res[k]
        assert s == s1 * k * k and n == n1 * k * k, (k, s, s1, n, n1)
        assert b == b1


def test_acceptance1_phi_within_10pct_after_2000_steps_and_ema_hull():
    phi_true, M, steps, seed = 64.0, 8, 2000, 0xACC4
    L, D, Lay, lay, plan, unit = _setup(phi_true)
    bufs = [torch.empty(lay.numel, dtype=torch.bfloat16, device="cuda") for _ in range(M)]
    g = D.GnsDevice(1, M, M, 0)
    st = L.GnsState.default()
    st.calibration = 1.0  # acceptance #1 is stated for c = 1
    g.set_state(st)
    sig, noi = [], []
    for k in range(steps):
        _fill(D, Lay, bufs, lay, seed, k * M, unit)
        g.begin_step()
        g.fused_sqnorm(plan, bufs)
        g.finalize(M * 2048)
        r = g.result()
        sig.append(r.stats.signal)
        noi.append(r.stats.noise)
        # the smoothed values stay inside the hull of the raw ones
        # (one rounding of alpha*ema + (1-alpha)*x may step an ulp outside)
        tol = 4e-16
        assert min(sig) - tol * abs(min(sig)) <= r.state.ema_signal <= max(sig) * (1 + tol)
        assert min(noi) * (1 - tol) <= r.state.ema_noise <= max(noi) * (1 + tol)
    assert r.phi_available
    assert abs(r.phi - phi_true) / phi_true < 0.10, (r.phi, phi_true)
