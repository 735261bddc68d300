// capi.cpp — extern "C" bindings of the C++ API (include/coadapt_host.h).
// Exceptions are caught at the boundary and mapped to status codes
// (errors.hpp:8-27 -> 1 / 1 / 2).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "coadapt/errors.hpp"
#include "coadapt/gns.hpp"
#include "coadapt/goodput.hpp"
#include "coadapt/io.hpp"
#include "coadapt/orchestrator.hpp"
#include "coadapt_host.h"

// shares coadapt_last_error() storage with cabi.cu
namespace coadapt_capi {
void set_error(const char* msg);
}

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return COADAPT_OK;
  } catch (const coadapt::ValidationError& e) {
    coadapt_capi::set_error(e.what());
    return COADAPT_E_VALIDATION;
  } catch (const coadapt::ParseError& e) {
    coadapt_capi::set_error(e.what());
    return COADAPT_E_VALIDATION;
  } catch (const coadapt::InternalError& e) {
    coadapt_capi::set_error(e.what());
    return COADAPT_E_INTERNAL;
  } catch (const std::exception& e) {
    coadapt_capi::set_error(e.what());
    return COADAPT_E_INTERNAL;
  }
}

coadapt::StepAccumulator make_acc(const double* s, int64_t n, int dp,
                                  int64_t bg) {
  coadapt::StepAccumulator acc(dp, bg);
  for (int64_t i = 0; i < n; ++i) acc.record_micro_batch(s[i]);
  return acc;
}

void put(const coadapt::StepStats& st, coadapt_step_stats* out) {
  out->signal = st.signal;
  out->noise = st.noise;
  out->noise_raw = st.noise_raw;
  out->mean_grad_sq = st.mean_grad_sq;
}

coadapt::GnsState get_state(const coadapt_gns_state* s) {
  coadapt::GnsState o;
  o.ema_signal = s->ema_signal;
  o.ema_noise = s->ema_noise;
  o.alpha_early = s->alpha_early;
  o.alpha_late = s->alpha_late;
  o.phase_boundary_tokens = s->phase_boundary_tokens;
  o.tokens_seen = s->tokens_seen;
  o.calibration = s->calibration;
  o.initialized = s->initialized != 0;
  return o;
}

void put_state(const coadapt::GnsState& s, coadapt_gns_state* o) {
  o->ema_signal = s.ema_signal;
  o->ema_noise = s.ema_noise;
  o->alpha_early = s.alpha_early;
  o->alpha_late = s.alpha_late;
  o->phase_boundary_tokens = s.phase_boundary_tokens;
  o->tokens_seen = s.tokens_seen;
  o->calibration = s.calibration;
  o->initialized = s.initialized ? 1 : 0;
}

coadapt::Candidate cand(const coadapt_candidate& c) {
  return coadapt::Candidate{
      coadapt::ConfigTuple{coadapt::ParallelStrategy{c.d, c.t, c.p},
                           c.global_batch, c.micro_batch},
      c.throughput};
}

std::vector<coadapt::Candidate> cands(const coadapt_candidate* c, size_t n) {
  std::vector<coadapt::Candidate> v;
  v.reserve(n);
  for (size_t i = 0; i < n; ++i) v.push_back(cand(c[i]));
  return v;
}

coadapt::OrchestratorConfig ocfg(const coadapt_orch_cfg* c) {
  coadapt::OrchestratorConfig o;
  o.margin = c->margin;
  o.max_growth = c->max_growth;
  o.reconfig_cost = c->reconfig_cost;
  o.reference_batch = c->reference_batch;
  return o;
}

}  // namespace

extern "C" {

int coadapt_finalize_step(const double* s, int64_t n, int dp_size,
                          double mean_grad_sq, int64_t global_batch,
                          coadapt_step_stats* out) {
  return guarded([&] {
    if (!out || (n && !s)) throw coadapt::ValidationError("NULL argument");
    put(coadapt::finalize_step(make_acc(s, n, dp_size, global_batch),
                               mean_grad_sq),
        out);
  });
}

int coadapt_finalize_step_vec(const double* s, int64_t n, int dp_size,
                              const double* mean_gradient, uint64_t dim,
                              int64_t global_batch, coadapt_step_stats* out) {
  return guarded([&] {
    if (!out || (n && !s) || (dim && !mean_gradient))
      throw coadapt::ValidationError("NULL argument");
    put(coadapt::finalize_step(make_acc(s, n, dp_size, global_batch),
                               std::span<const double>(mean_gradient, dim)),
        out);
  });
}

int coadapt_update_ema(coadapt_gns_state* state, const coadapt_step_stats* st,
                       int64_t tokens) {
  return guarded([&] {
    if (!state || !st) throw coadapt::ValidationError("NULL argument");
    auto s = get_state(state);
    coadapt::update_ema(
        s, coadapt::StepStats{st->signal, st->noise, st->noise_raw,
                              st->mean_grad_sq},
        tokens);
    put_state(s, state);
  });
}

int coadapt_gns_phi(const coadapt_gns_state* state, double* phi) {
  if (!state || !phi) return 0;
  const auto r = coadapt::gns(get_state(state));
  if (!r) return 0;
  *phi = *r;
  return 1;
}

void coadapt_gns_state_init(coadapt_gns_state* state) {
  if (!state) return;
  std::memset(state, 0, sizeof(*state));
  put_state(coadapt::GnsState{}, state);
}

double coadapt_stat_eff(double b, double phi) { return coadapt::stat_eff(b, phi); }
double coadapt_goodput(double t, double se) { return coadapt::goodput(t, se); }
double coadapt_goodput_lr(double t, double b, double phi, double ref) {
  return coadapt::goodput_lr(t, b, phi, ref);
}
double coadapt_lr_rescale(double eta, double b0, double b1) {
  return coadapt::lr_rescale(eta, b0, b1);
}
double coadapt_optimal_batch_continuous(double hw, double crit) {
  return coadapt::optimal_batch_continuous(hw, crit);
}

int coadapt_cbs_target(double phi, const int64_t* c, size_t n, int linear,
                       int64_t* out) {
  return guarded([&] {
    if (!out || (n && !c)) throw coadapt::ValidationError("NULL argument");
    *out = coadapt::cbs_target(
        phi, std::span<const std::int64_t>(c, n),
        linear ? coadapt::CbsDistance::kLinear : coadapt::CbsDistance::kLog);
  });
}

int coadapt_synth_candidates(const coadapt_cost* costs, size_t ncost,
                             const int64_t* bg, size_t nbg, const int64_t* bm,
                             size_t nbm, int bubble, double model_bytes,
                             double act_bytes, double mem_cap,
                             coadapt_candidate* out, size_t* count) {
  return guarded([&] {
    if (!count || (ncost && !costs) || (nbg && !bg) || (nbm && !bm))
      throw coadapt::ValidationError("NULL argument");
    coadapt::CostModelParams p;
    int n_gpus = 0;
    for (size_t i = 0; i < ncost; ++i) {
      p.per_strategy.push_back(
          {coadapt::ParallelStrategy{costs[i].d, costs[i].t, costs[i].p},
           costs[i].t_max, costs[i].b_hw});
      n_gpus = costs[i].d * costs[i].t * costs[i].p;
    }
    p.pipeline_bubble = bubble != 0;
    p.model_bytes = model_bytes;
    p.activation_bytes_per_sample = act_bytes;
    const auto prof = coadapt::synth_profile(
        p, std::span<const std::int64_t>(bg, nbg),
        std::span<const std::int64_t>(bm, nbm), mem_cap, n_gpus);
    const auto c = coadapt::feasible_candidates(prof);
    const size_t cap = *count;
    *count = c.size();
    if (!out) return;
    for (size_t i = 0; i < std::min(cap, c.size()); ++i) {
      std::memset(&out[i], 0, sizeof(out[i]));
      out[i].d = c[i].config.strategy.d;
      out[i].t = c[i].config.strategy.t;
      out[i].p = c[i].config.strategy.p;
      out[i].global_batch = c[i].config.global_batch;
      out[i].micro_batch = c[i].config.micro_batch;
      out[i].throughput = c[i].throughput;
    }
  });
}

int coadapt_score_candidates(const coadapt_candidate* c, size_t n, double phi,
                             const coadapt_candidate* current, double elapsed,
                             double useful, const coadapt_orch_cfg* cfg,
                             double* scores) {
  return guarded([&] {
    if (!current || !cfg || !scores || (n && !c))
      throw coadapt::ValidationError("NULL argument");
    const auto v = cands(c, n);
    const auto s = coadapt::score_candidates(
        v, phi, cand(*current).config, coadapt::ClockState{elapsed, useful},
        ocfg(cfg));
    std::copy(s.begin(), s.end(), scores);
  });
}

int coadapt_rank_candidates(const coadapt_candidate* c, size_t n, double phi,
                            const coadapt_candidate* current, double elapsed,
                            double useful, const coadapt_orch_cfg* cfg,
                            int64_t* order) {
  return guarded([&] {
    if (!current || !cfg || !order || (n && !c))
      throw coadapt::ValidationError("NULL argument");
    const auto v = cands(c, n);
    const auto r = coadapt::rank_candidates(
        v, phi, cand(*current).config, coadapt::ClockState{elapsed, useful},
        ocfg(cfg));
    for (size_t i = 0; i < r.size(); ++i) order[i] = (int64_t)r[i];
  });
}

int coadapt_decide(const coadapt_candidate* c, size_t n, int phi_available,
                   double phi, const coadapt_candidate* current,
                   double elapsed, double useful, const coadapt_orch_cfg* cfg,
                   coadapt_command* out) {
  return guarded([&] {
    if (!current || !cfg || !out || (n && !c))
      throw coadapt::ValidationError("NULL argument");
    const auto v = cands(c, n);
    const auto cur = cand(*current);
    const auto cmd = coadapt::decide(
        v, phi_available ? std::optional<double>(phi) : std::nullopt,
        cur.config, coadapt::ClockState{elapsed, useful}, ocfg(cfg),
        current->throughput);
    std::memset(out, 0, sizeof(*out));
    out->kind = (int32_t)cmd.kind;
    out->winner_index = -1;
    if (cmd.winner_score != 0.0 || cmd.current_score != 0.0)
      for (size_t i = 0; i < v.size(); ++i)
        if (v[i].config == cmd.winner) out->winner_index = (int32_t)i;
    out->winner_score = cmd.winner_score;
    out->current_score = cmd.current_score;
    out->penalized = cmd.penalized ? 1 : 0;
  });
}

int coadapt_record_reconfig(coadapt_clock* clock, double* reconfig_cost,
                            double observed_latency) {
  return guarded([&] {
    if (!clock || !reconfig_cost) throw coadapt::ValidationError("NULL argument");
    coadapt::ClockState c{clock->elapsed, clock->useful, clock->reconfig_total,
                          clock->reconfigs};
    coadapt::OrchestratorConfig cfg;
    cfg.reconfig_cost = *reconfig_cost;
    coadapt::record_reconfig(c, cfg, observed_latency);
    clock->elapsed = c.elapsed;
    clock->useful = c.useful;
    clock->reconfig_total = c.reconfig_total;
    clock->reconfigs = c.reconfigs;
    *reconfig_cost = cfg.reconfig_cost;
  });
}

int coadapt_trace_csv(const coadapt_trace_row* rows, size_t n, char* buf,
                      size_t cap, size_t* needed) {
  return guarded([&] {
    if (n && !rows) throw coadapt::ValidationError("NULL argument");
    std::vector<coadapt::GnsTraceRow> v(n);
    for (size_t i = 0; i < n; ++i)
      v[i] = coadapt::GnsTraceRow{rows[i].step,       rows[i].tokens,
                                  rows[i].signal_raw, rows[i].noise_raw,
                                  rows[i].ema_signal, rows[i].ema_noise,
                                  rows[i].phi};
    const std::string s = coadapt::gns_trace_csv(v);
    if (needed) *needed = s.size();
    if (buf && cap) {
      const size_t k = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), k);
      buf[k] = '\0';
    }
  });
}

}  // extern "C"

namespace {

void profile_out(const coadapt::ThroughputProfile& prof,
                 coadapt_profile_entry* out, size_t* count, int* n_gpus) {
  const size_t cap = *count;
  *count = prof.entries.size();
  if (n_gpus) *n_gpus = prof.n_gpus;
  if (!out) return;
  size_t i = 0;
  for (const auto& [c, e] : prof.entries) {
    if (i >= cap) break;
    std::memset(&out[i], 0, sizeof(out[i]));
    out[i].d = c.strategy.d;
    out[i].t = c.strategy.t;
    out[i].p = c.strategy.p;
    out[i].global_batch = c.global_batch;
    out[i].micro_batch = c.micro_batch;
    out[i].samples_per_sec = e.samples_per_second;
    out[i].peak_mem_bytes = e.peak_memory;
    out[i].feasible = e.feasible ? 1 : 0;
    ++i;
  }
}

coadapt::ThroughputProfile profile_in(const coadapt_profile_entry* e, size_t n) {
  coadapt::ThroughputProfile prof;
  for (size_t i = 0; i < n; ++i) {
    const coadapt::ConfigTuple c{coadapt::ParallelStrategy{e[i].d, e[i].t, e[i].p},
                                 e[i].global_batch, e[i].micro_batch};
    if (prof.n_gpus == 0) prof.n_gpus = c.strategy.gpus();
    coadapt::validate_config(c, prof.n_gpus);
    if (!prof.entries
             .emplace(c, coadapt::ThroughputEntry{e[i].samples_per_sec,
                                                  e[i].peak_mem_bytes,
                                                  e[i].feasible != 0})
             .second)
      throw coadapt::ValidationError("duplicate key " + c.label());
  }
  return prof;
}

void text_out(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size();
  if (buf && cap) {
    const size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
}

}  // namespace

extern "C" {

int coadapt_profile_parse(const char* text, size_t len,
                          coadapt_profile_entry* out, size_t* count,
                          int* n_gpus) {
  return guarded([&] {
    if (!count || (len && !text)) throw coadapt::ValidationError("NULL argument");
    profile_out(coadapt::parse_profile_csv(std::string_view(text, len), "profile.csv"),
                out, count, n_gpus);
  });
}

int coadapt_profile_format(const coadapt_profile_entry* e, size_t n, char* buf,
                           size_t cap, size_t* needed) {
  return guarded([&] {
    if (n && !e) throw coadapt::ValidationError("NULL argument");
    text_out(coadapt::profile_csv(profile_in(e, n)), buf, cap, needed);
  });
}

int coadapt_profile_load(const char* path, coadapt_profile_entry* out,
                         size_t* count, int* n_gpus) {
  return guarded([&] {
    if (!path || !count) throw coadapt::ValidationError("NULL argument");
    profile_out(coadapt::load_profile(path), out, count, n_gpus);
  });
}

int coadapt_profile_save(const char* path, const coadapt_profile_entry* e,
                         size_t n) {
  return guarded([&] {
    if (!path || (n && !e)) throw coadapt::ValidationError("NULL argument");
    coadapt::save_profile(path, profile_in(e, n));
  });
}

int coadapt_decision_audit_csv(const coadapt_decision_row* rows, size_t n,
                               char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    if (n && !rows) throw coadapt::ValidationError("NULL argument");
    std::vector<coadapt::DecisionRecord> v(n);
    for (size_t i = 0; i < n; ++i) {
      v[i].step = rows[i].step;
      v[i].time_s = rows[i].time_s;
      if (!std::isnan(rows[i].phi)) v[i].phi = rows[i].phi;
      v[i].current = cand(rows[i].current).config;
      v[i].command.winner = cand(rows[i].winner).config;
      v[i].command.kind = (coadapt::CommandKind)rows[i].command.kind;
      v[i].command.current_score = rows[i].command.current_score;
      v[i].command.winner_score = rows[i].command.winner_score;
      v[i].command.penalized = rows[i].command.penalized != 0;
    }
    text_out(coadapt::decision_audit_csv(v), buf, cap, needed);
  });
}

int coadapt_format_double(double v, char* buf, size_t cap) {
  return guarded([&] {
    const std::string s = coadapt::format_double(v);
    if (!buf || cap <= s.size())
      throw coadapt::ValidationError("format_double: buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int coadapt_simulate_micro_gradients(const double* g, const double* sigma,
                                     uint64_t n, int64_t micro_batch,
                                     int count, uint64_t seed, double* out) {
  return guarded([&] {
    if ((n && (!g || !sigma)) || (count > 0 && n && !out))
      throw coadapt::ValidationError("NULL argument");
    const auto draws = coadapt::simulate_micro_gradients(
        std::span<const double>(g, n), std::span<const double>(sigma, n),
        micro_batch, count, seed);
    for (int c = 0; c < count; ++c)
      std::copy(draws[c].begin(), draws[c].end(), out + (size_t)c * n);
  });
}

}  // extern "C"
