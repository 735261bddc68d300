"""Python mirror of the reference's gns / goodput / orchestrator API.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/coadapt/gns.hpp, goodput.hpp and SPEC.md's
profile/orchestrator operations, implemented by the C++ library
(libcoadapt_b200.so) through the C bindings in include/coadapt_host.h.  The
device hot path (squared norms on B200) lives in ``device.py``.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import GnsState, StepStats, ValidationError, check, lib


class StepAccumulator:
    """gns.hpp:15-32 — the N = d*M recorded squared norms of one step."""

    def __init__(self, dp_size: int, global_batch: int):
        if dp_size < 1:
            raise ValidationError("StepAccumulator: dp_size must be >= 1")
        if global_batch < 1:
            raise ValidationError("StepAccumulator: global_batch must be >= 1")
        self._dp = int(dp_size)
        self._bg = int(global_batch)
        self._s: list[float] = []

    def record_micro_batch(self, squared_norm: float) -> None:
        # gns.hpp:19 — negative (and NaN) input is rejected
        if not (squared_norm >= 0.0):
            raise ValidationError(f"record_micro_batch: squared norm must be >= 0, got {squared_norm!r}")
        self._s.append(float(squared_norm))

    def dp_size(self) -> int:
        return self._dp

    def global_batch(self) -> int:
        return self._bg

    def sample_count(self) -> int:
        return len(self._s)

    def micro_count(self) -> int:
        return len(self._s) // self._dp

    def squared_norms(self) -> np.ndarray:
        return np.asarray(self._s, np.float64)


def finalize_step(acc: StepAccumulator, mean_gradient) -> StepStats:
    """gns.hpp:47-49.  ``mean_gradient`` is either gbar^2 (float) or the mean
    gradient vector (reduced on the GPU in fp64)."""
    s = acc.squared_norms()
    out = StepStats()
    if np.isscalar(mean_gradient):
        check(lib().coadapt_finalize_step(s.ctypes.data, s.size, acc.dp_size(), float(mean_gradient),
                                          acc.global_batch(), C.byref(out)))
    else:
        v = np.ascontiguousarray(mean_gradient, np.float64)
        check(lib().coadapt_finalize_step_vec(s.ctypes.data, s.size, acc.dp_size(), v.ctypes.data,
                                              v.size, acc.global_batch(), C.byref(out)))
    return out


def update_ema(state: GnsState, stats: StepStats, tokens_this_step: int) -> None:
    """gns.hpp:64-68 (mutates ``state``)."""
    check(lib().coadapt_update_ema(C.byref(state), C.byref(stats), int(tokens_this_step)))


def gns(state: GnsState) -> Optional[float]:
    """gns.hpp:70-73: calibrated phi, or None while ema_signal <= 0."""
    phi = C.c_double()
    return phi.value if lib().coadapt_gns_phi(C.byref(state), C.byref(phi)) else None


def simulate_micro_gradients(true_gradient, sigma_diag, micro_batch_samples: int, count: int,
                             seed: int) -> np.ndarray:
    """gns.hpp:75-80 -> (count, n) array."""
    g = np.ascontiguousarray(true_gradient, np.float64)
    s = np.ascontiguousarray(sigma_diag, np.float64)
    if g.size != s.size:
        raise ValidationError("simulate_micro_gradients: size mismatch")
    out = np.zeros((max(count, 0), g.size), np.float64)
    check(lib().coadapt_simulate_micro_gradients(g.ctypes.data, s.ctypes.data, g.size,
                                                 int(micro_batch_samples), int(count), int(seed),
                                                 out.ctypes.data))
    return out


@dataclass
class GnsTraceRow:
    """gns.hpp:84-92."""
    step: int = 0
    tokens: int = 0
    signal_raw: float = 0.0
    noise_raw: float = 0.0
    ema_signal: float = 0.0
    ema_noise: float = 0.0
    phi: float = 0.0


def gns_trace_csv(rows: Sequence[GnsTraceRow]) -> str:
    """gns.hpp:94 — byte-exact via format_double (io.hpp:10-13)."""
    arr = (L.TraceRowC * max(1, len(rows)))(*[
        L.TraceRowC(r.step, r.tokens, r.signal_raw, r.noise_raw, r.ema_signal, r.ema_noise, r.phi)
        for r in rows])
    need = C.c_size_t()
    check(lib().coadapt_trace_csv(arr, len(rows), None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value + 1)
    check(lib().coadapt_trace_csv(arr, len(rows), buf, need.value + 1, C.byref(need)))
    return buf.value.decode()


def format_double(v: float) -> str:
    buf = C.create_string_buffer(64)
    check(lib().coadapt_format_double(float(v), buf, 64))
    return buf.value.decode()


# ---------------------------------------------------------------- goodput.hpp

def stat_eff(global_batch: float, phi: float) -> float:
    return lib().coadapt_stat_eff(float(global_batch), float(phi))


def goodput(throughput: float, stat_efficiency: float) -> float:
    return lib().coadapt_goodput(float(throughput), float(stat_efficiency))


def goodput_lr(throughput: float, global_batch: float, phi: float, reference_batch: float) -> float:
    return lib().coadapt_goodput_lr(float(throughput), float(global_batch), float(phi),
                                    float(reference_batch))


def lr_rescale(eta: float, batch_old: float, batch_new: float) -> float:
    return lib().coadapt_lr_rescale(float(eta), float(batch_old), float(batch_new))


def optimal_batch_continuous(batch_hw: float, batch_crit_scaled: float) -> float:
    return lib().coadapt_optimal_batch_continuous(float(batch_hw), float(batch_crit_scaled))


def cbs_target(phi: float, candidates: Sequence[int], linear: bool = False) -> int:
    arr = (C.c_int64 * max(1, len(candidates)))(*candidates)
    out = C.c_int64()
    check(lib().coadapt_cbs_target(float(phi), arr, len(candidates), int(linear), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- scorer

@dataclass(frozen=True)
class Candidate:
    d: int
    t: int
    p: int
    global_batch: int
    micro_batch: int
    throughput: float = 0.0

    def strategy(self):
        return (self.d, self.t, self.p)

    def key(self):
        return (self.d, self.t, self.p, self.global_batch, self.micro_batch)

    def _c(self) -> L.CandidateC:
        return L.CandidateC(self.d, self.t, self.p, 0, self.global_batch, self.micro_batch,
                            self.throughput)


@dataclass
class Command:
    kind: int
    winner_index: int
    winner_score: float
    current_score: float
    penalized: bool

    @property
    def name(self) -> str:
        return {L.NOOP: "NoOp", L.SCALE_BS: "ScaleBS", L.RECONFIGURE: "Reconfigure"}[self.kind]


def _carr(cands: Sequence[Candidate]):
    if isinstance(cands, CandidateTable):
        return cands._arr
    return (L.CandidateC * max(1, len(cands)))(*[c._c() for c in cands])


class CandidateTable(Sequence):
    """A candidate list marshalled for the C-ABI once.  decide() / score /
    rank accept it in place of a list; the per-step decide then costs one C
    call (microseconds) instead of rebuilding the ctypes array every step."""

    def __init__(self, cands: Sequence[Candidate]):
        self._cands = list(cands)
        self._arr = (L.CandidateC * max(1, len(self._cands)))(*[c._c() for c in self._cands])

    def __len__(self) -> int:
        return len(self._cands)

    def __getitem__(self, i):
        return self._cands[i]


def synth_candidates(costs: Iterable[tuple], batch_grid: Sequence[int], micro_grid: Sequence[int],
                     pipeline_bubble: bool = True, model_bytes: float = 0.0,
                     act_bytes_per_sample: float = 0.0, mem_capacity: float = math.inf) -> list[Candidate]:
    """synth_profile + feasible_candidates.  costs: (d, t, p, T_max, B_hw)."""
    costs = list(costs)
    ca = (L.CostC * max(1, len(costs)))(*[L.CostC(d, t, p, 0, tm, bh) for d, t, p, tm, bh in costs])
    bg = (C.c_int64 * len(batch_grid))(*batch_grid)
    bm = (C.c_int64 * len(micro_grid))(*micro_grid)
    n = C.c_size_t(0)
    args = (ca, len(costs), bg, len(batch_grid), bm, len(micro_grid), int(pipeline_bubble),
            float(model_bytes), float(act_bytes_per_sample), float(mem_capacity))
    check(lib().coadapt_synth_candidates(*args, None, C.byref(n)))
    out = (L.CandidateC * max(1, n.value))()
    check(lib().coadapt_synth_candidates(*args, out, C.byref(n)))
    return [Candidate(c.d, c.t, c.p, c.global_batch, c.micro_batch, c.throughput) for c in out[:n.value]]


def _cfg(margin, max_growth, reconfig_cost, reference_batch):
    return L.OrchCfgC(margin, max_growth, reconfig_cost, reference_batch)


def score_candidates(cands: Sequence[Candidate], phi: float, current: Candidate, t_elapsed: float,
                     t_useful: float, reconfig_cost: float = 0.0, reference_batch: float = 16.0) -> np.ndarray:
    out = np.zeros(len(cands), np.float64)
    cur = current._c()
    check(lib().coadapt_score_candidates(_carr(cands), len(cands), float(phi), C.byref(cur),
                                         float(t_elapsed), float(t_useful),
                                         C.byref(_cfg(0.1, 2.0, reconfig_cost, reference_batch)),
                                         out.ctypes.data))
    return out


def rank_candidates(cands: Sequence[Candidate], phi: float, current: Candidate, t_elapsed: float,
                    t_useful: float, reconfig_cost: float = 0.0, reference_batch: float = 16.0) -> list[int]:
    out = np.zeros(len(cands), np.int64)
    cur = current._c()
    check(lib().coadapt_rank_candidates(_carr(cands), len(cands), float(phi), C.byref(cur),
                                        float(t_elapsed), float(t_useful),
                                        C.byref(_cfg(0.1, 2.0, reconfig_cost, reference_batch)),
                                        out.ctypes.data))
    return out.tolist()


@dataclass
class ClockState:
    """T_elapsed / T_useful + the observed reconfiguration
    latencies record_reconfig averages into c_reconfig."""
    elapsed: float = 0.0
    useful: float = 0.0
    reconfig_total: float = 0.0
    reconfigs: int = 0


def record_reconfig(clock: ClockState, observed_latency: float, reconfig_cost: float = 0.0) -> float:
    """advance clock.elapsed by the latency (useful stays),
    return the new c_reconfig = mean of all observed latencies."""
    c = L.ClockC(clock.elapsed, clock.useful, clock.reconfig_total, clock.reconfigs)
    cost = C.c_double(reconfig_cost)
    check(lib().coadapt_record_reconfig(C.byref(c), C.byref(cost), float(observed_latency)))
    clock.elapsed, clock.useful = c.elapsed, c.useful
    clock.reconfig_total, clock.reconfigs = c.reconfig_total, c.reconfigs
    return cost.value


def decide(cands: Sequence[Candidate], phi: Optional[float], current: Candidate, t_elapsed: float,
           t_useful: float, margin: float = 0.10, max_growth: float = 2.0, reconfig_cost: float = 0.0,
           reference_batch: float = 16.0) -> Command:
    """Algorithm 2."""
    out = L.CommandC()
    cur = current._c()
    check(lib().coadapt_decide(_carr(cands), len(cands), int(phi is not None), float(phi or 0.0),
                               C.byref(cur), float(t_elapsed), float(t_useful),
                               C.byref(_cfg(margin, max_growth, reconfig_cost, reference_batch)),
                               C.byref(out)))
    return Command(out.kind, out.winner_index, out.winner_score, out.current_score, bool(out.penalized))


# ---------------------------------------------------------------- formats

@dataclass(frozen=True)
class ProfileEntry:
    """One row of the throughput table."""
    d: int
    t: int
    p: int
    global_batch: int
    micro_batch: int
    samples_per_sec: float
    peak_mem_bytes: float
    feasible: bool

    def _c(self) -> L.ProfileEntryC:
        return L.ProfileEntryC(self.d, self.t, self.p, 0, self.global_batch, self.micro_batch,
                               self.samples_per_sec, self.peak_mem_bytes, int(self.feasible), 0)


def _entries_out(fn, *args):
    n, g = C.c_size_t(0), C.c_int(0)
    check(fn(*args, None, C.byref(n), C.byref(g)))
    out = (L.ProfileEntryC * max(1, n.value))()
    check(fn(*args, out, C.byref(n), C.byref(g)))
    return [ProfileEntry(e.d, e.t, e.p, e.global_batch, e.micro_batch, e.samples_per_sec,
                         e.peak_mem_bytes, bool(e.feasible)) for e in out[:n.value]], g.value


def parse_profile_csv(text: str):
    """-> (entries sorted by (S, B_g, B_m), n_gpus); ValidationError on bad rows."""
    b = text.encode()
    return _entries_out(lib().coadapt_profile_parse, b, len(b))


def load_profile(path: str):
    return _entries_out(lib().coadapt_profile_load, path.encode())


def _text_out(fn, *args) -> str:
    need = C.c_size_t()
    check(fn(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value + 1)
    check(fn(*args, buf, need.value + 1, C.byref(need)))
    return buf.value.decode()


def profile_csv(entries: Sequence[ProfileEntry]) -> str:
    arr = (L.ProfileEntryC * max(1, len(entries)))(*[e._c() for e in entries])
    return _text_out(lib().coadapt_profile_format, arr, len(entries))


def save_profile(path: str, entries: Sequence[ProfileEntry]) -> None:
    arr = (L.ProfileEntryC * max(1, len(entries)))(*[e._c() for e in entries])
    check(lib().coadapt_profile_save(path.encode(), arr, len(entries)))


@dataclass
class DecisionRow:
    step: int
    time_s: float
    phi: Optional[float]
    current: Candidate
    winner: Candidate
    command: Command


def decision_audit_csv(rows: Sequence[DecisionRow]) -> str:
    """SPEC.md:404-405 decision audit log."""
    arr = (L.DecisionRowC * max(1, len(rows)))(*[
        L.DecisionRowC(r.step, r.time_s, float("nan") if r.phi is None else r.phi, r.current._c(),
                       r.winner._c(), L.CommandC(r.command.kind, r.command.winner_index,
                                                 r.command.winner_score, r.command.current_score,
                                                 int(r.command.penalized), 0))
        for r in rows])
    return _text_out(lib().coadapt_decision_audit_csv, arr, len(rows))
