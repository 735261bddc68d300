// orchestrator.cpp — implements coadapt/orchestrator.hpp: the candidate table
// and Algorithm 2's scoring, clamp, tie-break and margin
// (SPEC.md:361-375, 394-399).
#include "coadapt/orchestrator.hpp"

#include <algorithm>
#include <numeric>

#include "coadapt/errors.hpp"
#include "coadapt/goodput.hpp"

namespace coadapt {

ThroughputProfile synth_profile(const CostModelParams& params,
                                std::span<const std::int64_t> batch_grid,
                                std::span<const std::int64_t> micro_grid,
                                double memory_capacity, int n_gpus,
                                const std::string& hardware_id) {
  if (batch_grid.empty() || micro_grid.empty() || params.per_strategy.empty())
    throw ValidationError("synth_profile: empty grid or strategy list");
  ThroughputProfile prof;
  prof.hardware_id = hardware_id;
  prof.n_gpus = n_gpus;
  prof.memory_capacity = memory_capacity;
  for (const auto& ps : params.per_strategy) {
    validate_strategy(ps.strategy, n_gpus);
    if (!(ps.t_max > 0.0) || !(ps.b_hw > 0.0))
      throw ValidationError("synth_profile: T_max and B_hw must be > 0 for " +
                            ps.strategy.label());
    for (std::int64_t bg : batch_grid)
      for (std::int64_t bm : micro_grid) {
        ConfigTuple c{ps.strategy, bg, bm};
        if (!c.divisible()) continue;
        const std::int64_t ga = c.grad_accum();
        double t = ps.t_max * (double)bg / ((double)bg + ps.b_hw);
        if (params.pipeline_bubble)
          t *= (double)ga / (double)(ga + ps.strategy.p - 1);
        ThroughputEntry e;
        e.peak_memory =
            params.model_bytes / (double)(ps.strategy.t * ps.strategy.p) +
            params.activation_bytes_per_sample * (double)bm;
        e.feasible = e.peak_memory <= memory_capacity;
        e.samples_per_second = e.feasible ? t : 0.0;
        prof.entries[c] = e;
      }
  }
  return prof;
}

std::optional<std::pair<std::int64_t, ThroughputEntry>> best_micro_batch(
    const ThroughputProfile& profile, const ParallelStrategy& s,
    std::int64_t global_batch) {
  std::optional<std::pair<std::int64_t, ThroughputEntry>> best;
  for (const auto& [c, e] : profile.entries) {
    if (c.strategy != s || c.global_batch != global_batch || !e.feasible)
      continue;
    // fastest; ties -> smaller B_m (map order visits smaller B_m first)
    if (!best || e.samples_per_second > best->second.samples_per_second)
      best = std::make_pair(c.micro_batch, e);
  }
  return best;
}

std::optional<ParallelStrategy> optimal_strategy(
    const ThroughputProfile& profile, std::int64_t global_batch) {
  std::optional<ParallelStrategy> best;
  double best_t = 0.0;
  std::vector<ParallelStrategy> seen;
  for (const auto& [c, e] : profile.entries) {
    if (c.global_batch != global_batch) continue;
    if (std::find(seen.begin(), seen.end(), c.strategy) != seen.end()) continue;
    seen.push_back(c.strategy);
    const auto bm = best_micro_batch(profile, c.strategy, global_batch);
    if (!bm) continue;
    const double t = bm->second.samples_per_second;
    const bool better =
        !best || t > best_t ||
        (t == best_t && (c.strategy.d > best->d ||
                         (c.strategy.d == best->d && c.strategy.t > best->t)));
    if (better) {
      best = c.strategy;
      best_t = t;
    }
  }
  return best;
}

std::vector<Candidate> feasible_candidates(const ThroughputProfile& profile) {
  std::vector<Candidate> out;
  for (const auto& [c, e] : profile.entries) {
    if (!e.feasible) continue;
    const auto bm = best_micro_batch(profile, c.strategy, c.global_batch);
    if (!bm || bm->first != c.micro_batch) continue;
    out.push_back(Candidate{c, e.samples_per_second});
  }
  std::sort(out.begin(), out.end(), [](const Candidate& a, const Candidate& b) {
    const auto& x = a.config;
    const auto& y = b.config;
    if (x.global_batch != y.global_batch) return x.global_batch < y.global_batch;
    if (x.strategy.d != y.strategy.d) return x.strategy.d < y.strategy.d;
    if (x.strategy.t != y.strategy.t) return x.strategy.t < y.strategy.t;
    return x.strategy.p < y.strategy.p;
  });
  return out;
}

std::vector<double> score_candidates(std::span<const Candidate> candidates,
                                     double phi, const ConfigTuple& current,
                                     const ClockState& clock,
                                     const OrchestratorConfig& cfg) {
  std::vector<double> s(candidates.size());
  for (std::size_t i = 0; i < candidates.size(); ++i) {
    const auto& c = candidates[i];
    double g = goodput_lr(c.throughput, (double)c.config.global_batch, phi,
                          cfg.reference_batch);
    if (c.config.strategy != current.strategy)
      g = g * clock.useful / (clock.elapsed + cfg.reconfig_cost);
    s[i] = g;
  }
  return s;
}

namespace {
// strict "a ranks before b" at equal score (SPEC.md:367 + completion)
bool tie_before(const ConfigTuple& a, const ConfigTuple& b,
                const ConfigTuple& cur) {
  const bool ac = a == cur, bc = b == cur;
  if (ac != bc) return ac;
  if (a.global_batch != b.global_batch) return a.global_batch < b.global_batch;
  if (a.strategy.d != b.strategy.d) return a.strategy.d > b.strategy.d;
  if (a.strategy.t != b.strategy.t) return a.strategy.t > b.strategy.t;
  return a.micro_batch < b.micro_batch;
}
}  // namespace

std::vector<std::size_t> rank_candidates(std::span<const Candidate> candidates,
                                         double phi, const ConfigTuple& current,
                                         const ClockState& clock,
                                         const OrchestratorConfig& cfg) {
  const auto s = score_candidates(candidates, phi, current, clock, cfg);
  std::vector<std::size_t> idx(candidates.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {
    if (s[a] != s[b]) return s[a] > s[b];
    return tie_before(candidates[a].config, candidates[b].config, current);
  });
  return idx;
}

void record_reconfig(ClockState& clock, OrchestratorConfig& cfg,
                     double observed_latency) {
  if (!(observed_latency >= 0.0))
    throw ValidationError("record_reconfig: latency must be >= 0");
  clock.elapsed += observed_latency;
  clock.reconfig_total += observed_latency;
  clock.reconfigs += 1;
  cfg.reconfig_cost = clock.reconfig_total / (double)clock.reconfigs;
}

Command decide(std::span<const Candidate> candidates, std::optional<double> phi,
               const ConfigTuple& current, const ClockState& clock,
               const OrchestratorConfig& cfg,
               std::optional<double> current_throughput) {
  if (candidates.empty())
    throw ValidationError("decide: empty candidate set (SPEC.md:370)");
  Command cmd;
  cmd.target = current;
  cmd.winner = current;
  double t_cur = 0.0;
  if (current_throughput) {
    t_cur = *current_throughput;
  } else {
    auto it = std::find_if(candidates.begin(), candidates.end(),
                           [&](const Candidate& c) { return c.config == current; });
    if (it == candidates.end())
      throw ValidationError("decide: current config " + current.label() +
                            " is not a candidate and no throughput was given");
    t_cur = it->throughput;
  }
  if (!phi) {
    cmd.note = "phi unavailable";
    return cmd;
  }
  cmd.current_score = goodput_lr(t_cur, (double)current.global_batch, *phi,
                                 cfg.reference_batch);  // unpenalised
  const auto s = score_candidates(candidates, *phi, current, clock, cfg);
  long best = -1;
  for (std::size_t i = 0; i < candidates.size(); ++i) {
    if ((double)candidates[i].config.global_batch >
        cfg.max_growth * (double)current.global_batch)
      continue;  // growth clamp; shrinking is unrestricted
    if (best < 0 || s[i] > s[best] ||
        (s[i] == s[best] &&
         tie_before(candidates[i].config, candidates[best].config, current)))
      best = (long)i;
  }
  if (best < 0) {
    cmd.note = "no candidate within the growth clamp";
    return cmd;
  }
  const auto& w = candidates[best].config;
  cmd.winner = w;
  cmd.winner_score = s[best];
  cmd.penalized = w.strategy != current.strategy;
  if (w == current) return cmd;  // incumbent wins
  if ((cmd.winner_score - cmd.current_score) / cmd.current_score < cfg.margin) {
    cmd.note = "below switching margin";
    return cmd;
  }
  cmd.target = w;
  cmd.kind = w.strategy == current.strategy ? CommandKind::kScaleBS
                                            : CommandKind::kReconfigure;
  return cmd;
}

}  // namespace coadapt
