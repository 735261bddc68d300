// coadapt/strategy.hpp — the (d,t,p) decision variables.
// Declarations match the reference (proj/include/coadapt/strategy.hpp:12-46).
// In the GNS hot path (d,t,p) is also the partition key of the reduction:
// d*M slots of s, model-parallel partials summed per slot.
#pragma once

#include <compare>
#include <cstdint>
#include <string>

namespace coadapt {

struct ParallelStrategy {
  int d = 1;  // data-parallel degree
  int t = 1;  // tensor-parallel degree
  int p = 1;  // pipeline-parallel degree

  int gpus() const { return d * t * p; }
  auto operator<=>(const ParallelStrategy&) const = default;

  // "d<d>t<t>p<p>", e.g. "d2t1p4"
  std::string label() const;
};

struct ConfigTuple {
  ParallelStrategy strategy;
  std::int64_t global_batch = 0;  // B_g, samples per optimizer step
  std::int64_t micro_batch = 0;   // B_m, samples per forward/backward

  // B_g % (d * B_m) == 0 with positive sizes
  bool divisible() const;
  // GA = B_g / (d * B_m): the micro-batch count M of Algorithm 1
  std::int64_t grad_accum() const;
  auto operator<=>(const ConfigTuple&) const = default;

  // "<strategy>_g<B_g>_m<B_m>", e.g. "d2t1p4_g16_m2"
  std::string label() const;
};

// ValidationError unless all degrees >= 1 and d*t*p == n_gpus.
void validate_strategy(const ParallelStrategy& s, int n_gpus);

// validate_strategy + positive batches + divisibility.
void validate_config(const ConfigTuple& c, int n_gpus);

// Accepts "2,1,4" or "d2t1p4"; ValidationError otherwise.
ParallelStrategy parse_strategy_label(const std::string& text);

}  // namespace coadapt
