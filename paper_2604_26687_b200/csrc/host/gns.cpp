// gns.cpp — implements coadapt/gns.hpp (reference gns.hpp:15-94; Algorithm 1,
// PAPER.md:432-457).
//
// The scalar formulas here and finalize_kernel (kernels.cu) are evaluated in
// the same order with no FMA contraction (-ffp-contract=off here, explicit
// __d*_rn intrinsics there), so a device step and a host step produce
// bit-identical StepStats / GnsState from the same s and gbar^2.
#include "coadapt/gns.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <limits>

#include "coadapt/errors.hpp"
#include "coadapt/io.hpp"
#include "coadapt_cuda.h"

namespace coadapt {

StepAccumulator::StepAccumulator(int dp_size, std::int64_t global_batch)
    : dp_size_(dp_size), global_batch_(global_batch) {
  if (dp_size < 1) throw ValidationError("StepAccumulator: dp_size must be >= 1");
  if (global_batch < 1)
    throw ValidationError("StepAccumulator: global_batch must be >= 1");
}

void StepAccumulator::record_micro_batch(double squared_norm) {
  // gns.hpp:19 "Negative input is rejected"; NaN is rejected the same way
  if (!(squared_norm >= 0.0))
    throw ValidationError("record_micro_batch: squared norm must be >= 0, got " +
                          format_double(squared_norm));
  squared_norms_.push_back(squared_norm);
}

std::int64_t StepAccumulator::sample_count() const {
  return (std::int64_t)squared_norms_.size();
}

std::int64_t StepAccumulator::micro_count() const {
  return sample_count() / dp_size_;
}

StepStats finalize_step(const StepAccumulator& acc, double mean_grad_sq) {
  const std::int64_t n = acc.sample_count();
  if (n < 2)
    throw ValidationError("finalize_step: insufficient samples, N = " +
                          std::to_string(n) + " < 2 (SPEC.md:179)");
  if (!(mean_grad_sq >= 0.0) || !std::isfinite(mean_grad_sq))
    throw ValidationError("finalize_step: mean_grad_sq must be finite and >= 0");
  double sum = 0.0;
  for (double s : acc.squared_norms()) sum += s;
  const double N = (double)n;
  const double sbar = sum / N;
  StepStats st;
  st.signal = (N * mean_grad_sq - sbar) / (N - 1.0);
  st.noise_raw = (sbar - mean_grad_sq) * (double)acc.global_batch() / (N - 1.0);
  st.noise = st.noise_raw > 0.0 ? st.noise_raw : 0.0;
  st.mean_grad_sq = mean_grad_sq;
  return st;
}

StepStats finalize_step(const StepAccumulator& acc,
                        std::span<const double> mean_gradient) {
  // |mean gradient|^2 is the O(n) part: reduce it on the GPU in fp64
  // (coadapt_sqnorm_host: H2D + the K1 reduction kernel).
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess)
    throw InternalError("finalize_step: no CUDA device available");
  double g2 = 0.0;
  const int rc = coadapt_sqnorm_host(mean_gradient.data(), mean_gradient.size(),
                                     COADAPT_FP64, dev, &g2);
  if (rc == COADAPT_E_VALIDATION) throw ValidationError(coadapt_last_error());
  if (rc != COADAPT_OK) throw InternalError(coadapt_last_error());
  return finalize_step(acc, g2);
}

void update_ema(GnsState& state, const StepStats& stats,
                std::int64_t tokens_this_step) {
  const double alpha = state.tokens_seen < state.phase_boundary_tokens
                           ? state.alpha_early
                           : state.alpha_late;
  if (!state.initialized) {
    state.ema_signal = stats.signal;  // no zero bias
    state.ema_noise = stats.noise;
    state.initialized = true;
  } else {
    const double beta = 1.0 - alpha;
    state.ema_signal = alpha * state.ema_signal + beta * stats.signal;
    state.ema_noise = alpha * state.ema_noise + beta * stats.noise;
  }
  if (state.ema_noise < 0.0) state.ema_noise = 0.0;
  state.tokens_seen += tokens_this_step;
}

std::optional<double> gns(const GnsState& state) {
  if (!(state.ema_signal > 0.0)) return std::nullopt;
  return state.calibration * state.ema_noise / state.ema_signal;
}

namespace {
inline std::uint64_t splitmix(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline double unit_open(std::uint64_t h) {  // (0, 1)
  return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
}  // namespace

std::vector<std::vector<double>> simulate_micro_gradients(
    std::span<const double> true_gradient, std::span<const double> sigma_diag,
    std::int64_t micro_batch_samples, int count, std::uint64_t seed) {
  if (sigma_diag.size() != true_gradient.size())
    throw ValidationError("simulate_micro_gradients: size mismatch");
  if (micro_batch_samples < 1)
    throw ValidationError("simulate_micro_gradients: micro_batch_samples < 1");
  if (count < 0) throw ValidationError("simulate_micro_gradients: count < 0");
  for (double s : sigma_diag)
    if (!(s >= 0.0))
      throw ValidationError("simulate_micro_gradients: sigma_diag must be >= 0");
  const std::size_t n = true_gradient.size();
  std::vector<std::vector<double>> out((std::size_t)count,
                                       std::vector<double>(n));
  const double two_pi = 6.283185307179586476925286766559;
  for (int c = 0; c < count; ++c) {
    const std::uint64_t key = splitmix(seed * 0xD1B54A32D192ED03ull + (std::uint64_t)c);
    for (std::size_t i = 0; i < n; i += 2) {
      // one Box-Muller pair per two components
      const double u1 = unit_open(splitmix(key ^ (2 * i + 1)));
      const double u2 = unit_open(splitmix(key ^ (2 * i + 2)));
      const double r = std::sqrt(-2.0 * std::log(u1));
      const double z0 = r * std::cos(two_pi * u2), z1 = r * std::sin(two_pi * u2);
      out[c][i] = true_gradient[i] +
                  z0 * std::sqrt(sigma_diag[i] / (double)micro_batch_samples);
      if (i + 1 < n)
        out[c][i + 1] =
            true_gradient[i + 1] +
            z1 * std::sqrt(sigma_diag[i + 1] / (double)micro_batch_samples);
    }
  }
  return out;
}

std::string gns_trace_csv(std::span<const GnsTraceRow> rows) {
  std::string out = "step,tokens,signal_raw,noise_raw,ema_signal,ema_noise,phi\n";
  for (const auto& r : rows) {
    out += format_int(r.step) + ',' + format_int(r.tokens) + ',' +
           format_double(r.signal_raw) + ',' + format_double(r.noise_raw) + ',' +
           format_double(r.ema_signal) + ',' + format_double(r.ema_noise) + ',' +
           format_double(r.phi) + '\n';
  }
  return out;
}

}  // namespace coadapt
