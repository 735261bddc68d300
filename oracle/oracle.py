"""ctypes view of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: the parity checker and the CPU baseline.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline
leg and ``--impl reference``) may import this module.  The product package
``paper_2604_26687_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

BF16, FP16, FP32 = 0, 1, 2
NOOP, SCALE_BS, RECONFIGURE = 0, 1, 2


class Segment(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("numel", C.c_uint64), ("weight", C.c_double)]


class GenSegment(C.Structure):
    _fields_ = [("local_off", C.c_uint64), ("numel", C.c_uint64),
                ("global_base", C.c_uint64), ("row_len", C.c_uint64),
                ("row_stride", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("signal", C.c_double), ("noise", C.c_double),
                ("noise_raw", C.c_double), ("mean_grad_sq", C.c_double)]


class State(C.Structure):
    _fields_ = [("ema_signal", C.c_double), ("ema_noise", C.c_double),
                ("alpha_early", C.c_double), ("alpha_late", C.c_double),
                ("phase_boundary_tokens", C.c_int64), ("tokens_seen", C.c_int64),
                ("calibration", C.c_double), ("initialized", C.c_int32),
                ("pad_", C.c_int32)]

    @classmethod
    def default(cls) -> "State":
        # gns.hpp:53-62 defaults
        return cls(0.0, 0.0, 0.95, 0.99, 8_000_000, 0, 2.0, 0, 0)


class Entry(C.Structure):
    _fields_ = [("d", C.c_int32), ("t", C.c_int32), ("p", C.c_int32), ("pad_", C.c_int32),
                ("global_batch", C.c_int64), ("micro_batch", C.c_int64),
                ("throughput", C.c_double), ("peak_memory", C.c_double),
                ("feasible", C.c_int32), ("pad2_", C.c_int32)]


class Cost(C.Structure):
    _fields_ = [("d", C.c_int32), ("t", C.c_int32), ("p", C.c_int32), ("pad_", C.c_int32),
                ("t_max", C.c_double), ("b_hw", C.c_double)]


class OrchCfg(C.Structure):
    _fields_ = [("margin", C.c_double), ("max_growth", C.c_double),
                ("reconfig_cost", C.c_double), ("reference_batch", C.c_double)]


class Command(C.Structure):
    _fields_ = [("kind", C.c_int32), ("winner_index", C.c_int32),
                ("winner_score", C.c_double), ("current_score", C.c_double),
                ("penalized", C.c_int32), ("pad_", C.c_int32)]


def build() -> None:
    """Compile liboracle.so (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        P, D, U64, I64, SZ, I = C.c_void_p, C.c_double, C.c_uint64, C.c_int64, C.c_size_t, C.c_int
        sig = {
            "orc_sqnorm": (D, [P, I, P, SZ]),
            "orc_sqnorm_mt": (D, [P, I, P, SZ, I]),
            "orc_fused_sqnorms": (None, [P, I, I, P, SZ, I, P, P]),
            "orc_finalize_step": (I, [P, I64, D, I64, P]),
            "orc_sumsq_f64": (D, [P, U64]),
            "orc_update_ema": (None, [P, P, I64]),
            "orc_gns": (I, [P, P]),
            "orc_stat_eff": (D, [D, D]),
            "orc_goodput": (D, [D, D]),
            "orc_goodput_lr": (D, [D, D, D, D]),
            "orc_lr_rescale": (D, [D, D, D]),
            "orc_optimal_batch_continuous": (D, [D, D]),
            "orc_cbs_target": (I64, [D, P, SZ, I]),
            "orc_synth_profile": (SZ, [P, SZ, P, SZ, P, SZ, I, D, D, D, P, SZ]),
            "orc_feasible_candidates": (SZ, [P, SZ, P, SZ]),
            "orc_decide": (I, [P, SZ, I, D, P, D, D, P, P]),
            "orc_record_reconfig": (I, [P, P, P, P, P, D]),
            "orc_score_candidates": (None, [P, SZ, D, P, D, D, P, P]),
            "orc_synth_fill": (None, [P, I, P, SZ, U64, U64, C.c_float, C.c_float]),
            "orc_synth_mean_fill": (None, [P, I, P, SZ, U64, U64, I64, C.c_float, C.c_float]),
            "orc_ih_std": (D, []),
            "orc_simulate_micro_gradients": (None, [P, P, U64, I64, I, U64, P]),
            "orc_fnv1a": (U64, [P, U64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _segs(segs) -> tuple:
    arr = (Segment * max(1, len(segs)))(*[Segment(int(o), int(n), float(w)) for o, n, w in segs])
    return arr, len(segs)


def _gsegs(gsegs) -> tuple:
    arr = (GenSegment * max(1, len(gsegs)))(*[GenSegment(*map(int, g)) for g in gsegs])
    return arr, len(gsegs)


def np_dtype(dtype: int):
    return np.float32 if dtype == FP32 else np.uint16


# ---------------------------------------------------------------- norms

def sqnorm(buf: np.ndarray, dtype: int, segs) -> float:
    a, n = _segs(segs)
    return lib().orc_sqnorm(_ptr(buf), dtype, a, n)


def sqnorm_mt(buf: np.ndarray, dtype: int, segs, nthreads: int) -> float:
    a, n = _segs(segs)
    return lib().orc_sqnorm_mt(_ptr(buf), dtype, a, n, nthreads)


def fused_sqnorms(bufs, dtype: int, segs, nthreads: int = 1):
    """-> (s[M], sum_i (sum_m x_mi)^2)"""
    M = len(bufs)
    ptrs = (C.c_void_p * M)(*[_ptr(b) for b in bufs])
    a, n = _segs(segs)
    s = np.zeros(M, np.float64)
    ss = C.c_double(0.0)
    lib().orc_fused_sqnorms(ptrs, M, dtype, a, n, nthreads, _ptr(s), C.byref(ss))
    return s, ss.value


def sumsq_f64(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, np.float64)
    return lib().orc_sumsq_f64(_ptr(v), v.size)


# ---------------------------------------------------------------- estimator

class OracleError(ValueError):
    pass


def finalize_step(s, mean_grad_sq: float, global_batch: int) -> Stats:
    s = np.ascontiguousarray(s, np.float64)
    out = Stats()
    rc = lib().orc_finalize_step(_ptr(s), s.size, float(mean_grad_sq), int(global_batch), C.byref(out))
    if rc:
        raise OracleError("finalize_step: validation error")
    return out


def update_ema(state: State, stats: Stats, tokens: int) -> None:
    lib().orc_update_ema(C.byref(state), C.byref(stats), int(tokens))


def gns(state: State):
    phi = C.c_double(0.0)
    return phi.value if lib().orc_gns(C.byref(state), C.byref(phi)) else None


# ---------------------------------------------------------------- goodput

def stat_eff(b, phi):
    return lib().orc_stat_eff(b, phi)


def goodput(t, se):
    return lib().orc_goodput(t, se)


def goodput_lr(t, b, phi, ref):
    return lib().orc_goodput_lr(t, b, phi, ref)


def lr_rescale(eta, b0, b1):
    return lib().orc_lr_rescale(eta, b0, b1)


def optimal_batch_continuous(bhw, bcrit):
    return lib().orc_optimal_batch_continuous(bhw, bcrit)


def cbs_target(phi, cands, linear=False):
    arr = (C.c_int64 * len(cands))(*cands)
    return lib().orc_cbs_target(phi, arr, len(cands), int(linear))


def synth_profile(costs, bg, bm, bubble, model_bytes, act_bytes, mem_cap):
    ca = (Cost * len(costs))(*[Cost(d, t, p, 0, tm, bh) for (d, t, p, tm, bh) in costs])
    bga = (C.c_int64 * len(bg))(*bg)
    bma = (C.c_int64 * len(bm))(*bm)
    n = lib().orc_synth_profile(ca, len(costs), bga, len(bg), bma, len(bm), int(bubble),
                                model_bytes, act_bytes, mem_cap, None, 0)
    out = (Entry * max(1, n))()
    lib().orc_synth_profile(ca, len(costs), bga, len(bg), bma, len(bm), int(bubble),
                            model_bytes, act_bytes, mem_cap, out, n)
    return list(out)[:n]


def feasible_candidates(entries):
    arr = (Entry * max(1, len(entries)))(*entries)
    out = (Entry * max(1, len(entries)))()
    n = lib().orc_feasible_candidates(arr, len(entries), out, len(entries))
    return list(out)[:n]


def decide(cands, phi, current: Entry, t_elapsed, t_useful, margin=0.10, max_growth=2.0,
           reconfig_cost=0.0, reference_batch=16.0) -> Command:
    arr = (Entry * max(1, len(cands)))(*cands)
    cfg = OrchCfg(margin, max_growth, reconfig_cost, reference_batch)
    out = Command()
    rc = lib().orc_decide(arr, len(cands), int(phi is not None), float(phi or 0.0), C.byref(current),
                          float(t_elapsed), float(t_useful), C.byref(cfg), C.byref(out))
    if rc:
        raise OracleError("decide: validation error")
    return out


def record_reconfig(elapsed, useful, total, count, reconfig_cost, latency):
    """SPEC.md:377-385 -> (elapsed, useful, total, count, reconfig_cost)"""
    e, u, t = C.c_double(elapsed), C.c_double(useful), C.c_double(total)
    n, c = C.c_int64(count), C.c_double(reconfig_cost)
    if lib().orc_record_reconfig(C.byref(e), C.byref(u), C.byref(t), C.byref(n), C.byref(c),
                                 float(latency)):
        raise OracleError("record_reconfig: latency must be >= 0")
    return e.value, u.value, t.value, n.value, c.value


def score_candidates(cands, phi, current, t_elapsed, t_useful, reconfig_cost=0.0, reference_batch=16.0):
    arr = (Entry * max(1, len(cands)))(*cands)
    cfg = OrchCfg(0.1, 2.0, reconfig_cost, reference_batch)
    out = np.zeros(len(cands), np.float64)
    lib().orc_score_candidates(arr, len(cands), float(phi), C.byref(current), float(t_elapsed),
                               float(t_useful), C.byref(cfg), _ptr(out))
    return out


# ---------------------------------------------------------------- synthetic data

def ih_std() -> float:
    return lib().orc_ih_std()


def noise_unit_for(g0: float, phi_true: float, micro_batch: int) -> float:
    """float32 noise unit giving Var(zeta) = phi_true * g0^2 / B_m."""
    std = g0 * (phi_true / micro_batch) ** 0.5
    return float(np.float32(std / ih_std()))


def synth_fill(numel: int, dtype: int, gsegs, seed: int, sample: int, g0: float, unit: float) -> np.ndarray:
    out = np.zeros(numel, np_dtype(dtype))
    a, n = _gsegs(gsegs)
    lib().orc_synth_fill(_ptr(out), dtype, a, n, seed, sample, g0, unit)
    return out


def synth_mean_fill(numel: int, dtype: int, gsegs, seed: int, sample0: int, nsamples: int,
                    g0: float, unit: float) -> np.ndarray:
    out = np.zeros(numel, np_dtype(dtype))
    a, n = _gsegs(gsegs)
    lib().orc_synth_mean_fill(_ptr(out), dtype, a, n, seed, sample0, nsamples, g0, unit)
    return out


def simulate_micro_gradients(g_true, sigma, micro_batch, count, seed) -> np.ndarray:
    g = np.ascontiguousarray(g_true, np.float64)
    s = np.ascontiguousarray(sigma, np.float64)
    out = np.zeros((count, g.size), np.float64)
    lib().orc_simulate_micro_gradients(_ptr(g), _ptr(s), g.size, int(micro_batch), count, seed, _ptr(out))
    return out


def fnv1a(buf: np.ndarray) -> int:
    return lib().orc_fnv1a(_ptr(buf), buf.nbytes)
