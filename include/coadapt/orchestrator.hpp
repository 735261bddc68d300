// coadapt/orchestrator.hpp — the candidate table and the scoring/ranking half
// of Algorithm 2 that consumes the GPU-produced phi.
// The reference ships no header for these modules; the declarations follow
// SPEC.md's operations: synth_profile, best_micro_batch
// (:84-92), optimal_strategy (:94-102), feasible_candidates (:104-112) and
// decide (:361-375).  Everything here is pure host arithmetic on <= a few
// hundred entries (microseconds); only phi comes from the device.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "coadapt/strategy.hpp"

namespace coadapt {

struct ThroughputEntry {
  double samples_per_second = 0.0;
  double peak_memory = 0.0;  // bytes per GPU
  bool feasible = false;
};

struct ThroughputProfile {
  std::string hardware_id;
  int n_gpus = 0;
  double memory_capacity = 0.0;
  std::map<ConfigTuple, ThroughputEntry> entries;
};

// Appendix C saturating model per strategy: T = T_max B_g / (B_g + B_hw),
// times GA / (GA + p - 1) with the pipeline-bubble switch.
struct CostModelParams {
  struct PerStrategy {
    ParallelStrategy strategy;
    double t_max = 0.0;
    double b_hw = 0.0;
  };
  std::vector<PerStrategy> per_strategy;
  bool pipeline_bubble = false;
  double model_bytes = 0.0;                  // divided by t*p
  double activation_bytes_per_sample = 0.0;  // times B_m
};

ThroughputProfile synth_profile(const CostModelParams& params,
                                std::span<const std::int64_t> batch_grid,
                                std::span<const std::int64_t> micro_grid,
                                double memory_capacity, int n_gpus,
                                const std::string& hardware_id = "synthetic");

// Fastest feasible B_m for (S, B_g); ties -> smaller B_m.
std::optional<std::pair<std::int64_t, ThroughputEntry>> best_micro_batch(
    const ThroughputProfile& profile, const ParallelStrategy& s,
    std::int64_t global_batch);

// argmax over strategies at B_g; ties -> larger d, then larger t.
std::optional<ParallelStrategy> optimal_strategy(
    const ThroughputProfile& profile, std::int64_t global_batch);

struct Candidate {
  ConfigTuple config;
  double throughput = 0.0;
};

// One candidate per feasible (S, B_g) (its fastest B_m), sorted by
// (B_g, d, t, p).
std::vector<Candidate> feasible_candidates(const ThroughputProfile& profile);

struct OrchestratorConfig {
  double margin = 0.10;        // epsilon
  double max_growth = 2.0;     // per decision
  int decision_interval = 25;  // optimizer steps
  double reconfig_cost = 0.0;  // c_reconfig, seconds
  double reference_batch = 16.0;
};

struct ClockState {
  double elapsed = 0.0;  // T_elapsed
  double useful = 0.0;   // T_useful
  // observed reconfiguration latencies so far (record_reconfig)
  double reconfig_total = 0.0;
  std::int64_t reconfigs = 0;
};

// a finished Reconfigure took `observed_latency` seconds
// (e.g. reshard::estimate or the measured device pull + process-group
// rebuild).  T_elapsed advances, T_useful does not; cfg.reconfig_cost
// becomes the mean of all observed latencies.  ValidationError if < 0.
void record_reconfig(ClockState& clock, OrchestratorConfig& cfg,
                     double observed_latency);

enum class CommandKind { kNoOp, kScaleBS, kReconfigure };

struct Command {
  CommandKind kind = CommandKind::kNoOp;
  ConfigTuple target;           // config to run next (== current for NoOp)
  ConfigTuple winner;           // argmax of the scored candidates
  double winner_score = 0.0;    // penalised if cross-strategy
  double current_score = 0.0;   // unpenalised
  bool penalized = false;
  std::string note;             // e.g. "phi unavailable"
};

// Per-candidate LR-aware goodput, penalised by T_useful/(T_elapsed+c) when
// the strategy differs from current's.
std::vector<double> score_candidates(std::span<const Candidate> candidates,
                                     double phi, const ConfigTuple& current,
                                     const ClockState& clock,
                                     const OrchestratorConfig& cfg);

// Candidate indices best-first under the decide() order: score, then prefer
// current, smaller B_g, larger d, larger t, smaller B_m.
std::vector<std::size_t> rank_candidates(std::span<const Candidate> candidates,
                                         double phi, const ConfigTuple& current,
                                         const ClockState& clock,
                                         const OrchestratorConfig& cfg);

// Algorithm 2.  `current` must be among the candidates unless its
// throughput is supplied.  nullopt phi -> NoOp.
Command decide(std::span<const Candidate> candidates, std::optional<double> phi,
               const ConfigTuple& current, const ClockState& clock,
               const OrchestratorConfig& cfg,
               std::optional<double> current_throughput = std::nullopt);

// ---- wire / disk formats ----

// Profile CSV: header exactly
//   d,t,p,global_batch,micro_batch,samples_per_sec,peak_mem_bytes,feasible
// Numbers via format_double/parse_double, so save -> load is bit-exact.
// ParseError names the line; ValidationError for invariant violations
// (d*t*p differing between rows, B_g mod d*B_m != 0, duplicate keys).
std::string profile_csv(const ThroughputProfile& profile);
ThroughputProfile parse_profile_csv(std::string_view text,
                                    const std::string& where);
ThroughputProfile load_profile(const std::string& path);
void save_profile(const std::string& path, const ThroughputProfile& profile);

// Decision audit log: header
//   step,time_s,phi,current_cfg,winner_cfg,current_score,winner_score,penalized,command
struct DecisionRecord {
  std::int64_t step = 0;
  double time_s = 0.0;
  std::optional<double> phi;  // written as nan when unavailable
  Command command;
  ConfigTuple current;
};
std::string decision_audit_csv(std::span<const DecisionRecord> rows);
const char* command_name(CommandKind kind);

}  // namespace coadapt
