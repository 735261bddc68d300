// goodput.cpp — implements coadapt/goodput.hpp (reference
// goodput.hpp:11-48).  Compiled without FMA contraction so
// values are bit-identical to the oracle's restatement.
#include "coadapt/goodput.hpp"

#include <cmath>
#include <limits>

#include "coadapt/errors.hpp"

namespace coadapt {

double EfficiencyContext::lr_at(double global_batch) const {
  return base_lr * std::sqrt(global_batch / reference_batch);
}

double stat_eff(double global_batch, double phi) {
  return (1.0 + phi) / (global_batch + phi);  // Eq. 5, goodput.hpp:20-22
}

double goodput(double throughput, double se) { return throughput * se; }

double goodput_lr(double throughput, double global_batch, double phi,
                  double reference_batch) {
  return throughput * stat_eff(global_batch, phi) *
         std::sqrt(global_batch / reference_batch);  // Eq. 7
}

double lr_rescale(double eta, double batch_old, double batch_new) {
  return eta * std::sqrt(batch_new / batch_old);  // Eq. 8
}

double optimal_batch_continuous(double batch_hw, double batch_crit_scaled) {
  return std::sqrt(batch_hw * batch_crit_scaled);  // App. C
}

std::int64_t cbs_target(double phi, std::span<const std::int64_t> candidates,
                        CbsDistance metric) {
  if (candidates.empty()) throw ValidationError("cbs_target: no candidates");
  const double target = phi > 1.0 ? phi : 1.0;
  std::int64_t best = 0;
  double best_d = std::numeric_limits<double>::infinity();
  // log2 keeps geometric (power-of-two) grids exact; distances within 1e-12
  // are ties and go to the smaller batch
  for (std::int64_t c : candidates) {
    const double d = metric == CbsDistance::kLinear
                         ? std::fabs((double)c - target)
                         : std::fabs(std::log2((double)c) - std::log2(target));
    if (d < best_d - 1e-12 || (std::fabs(d - best_d) <= 1e-12 && c < best)) {
      best_d = d;
      best = c;
    }
  }
  return best;
}

}  // namespace coadapt
