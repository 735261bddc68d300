// device.cpp — implements coadapt/device.hpp on top of the C-ABI.
#include "coadapt/device.hpp"

#include <cstring>
#include <vector>

#include "coadapt/errors.hpp"
#include "coadapt_cuda.h"

namespace coadapt {
namespace {

void check(int rc) {
  if (rc == COADAPT_OK) return;
  if (rc == COADAPT_E_VALIDATION) throw ValidationError(coadapt_last_error());
  throw InternalError(coadapt_last_error());
}

std::vector<coadapt_segment> to_c(std::span<const BucketSegment> segs) {
  std::vector<coadapt_segment> v(segs.size());
  for (std::size_t i = 0; i < segs.size(); ++i)
    v[i] = coadapt_segment{segs[i].offset, segs[i].numel, segs[i].weight};
  return v;
}

GnsState from_c(const coadapt_gns_state& s) {
  GnsState o;
  o.ema_signal = s.ema_signal;
  o.ema_noise = s.ema_noise;
  o.alpha_early = s.alpha_early;
  o.alpha_late = s.alpha_late;
  o.phase_boundary_tokens = s.phase_boundary_tokens;
  o.tokens_seen = s.tokens_seen;
  o.calibration = s.calibration;
  o.initialized = s.initialized != 0;
  return o;
}

coadapt_gns_state to_c(const GnsState& s) {
  coadapt_gns_state o;
  std::memset(&o, 0, sizeof(o));
  o.ema_signal = s.ema_signal;
  o.ema_noise = s.ema_noise;
  o.alpha_early = s.alpha_early;
  o.alpha_late = s.alpha_late;
  o.phase_boundary_tokens = s.phase_boundary_tokens;
  o.tokens_seen = s.tokens_seen;
  o.calibration = s.calibration;
  o.initialized = s.initialized ? 1 : 0;
  return o;
}

}  // namespace

BucketLayout::BucketLayout(std::span<const BucketSegment> segments,
                           std::uint64_t bucket_numel, GradDType dtype,
                           int device) {
  const auto c = to_c(segments);
  check(coadapt_plan_create(c.data(), c.size(), bucket_numel, (int)dtype,
                            device, &plan_));
}

BucketLayout BucketLayout::slice(std::span<const BucketSegment> segments,
                                 std::uint64_t bucket_numel, GradDType dtype,
                                 int device, int index, int count) {
  BucketLayout out;
  const auto c = to_c(segments);
  check(coadapt_plan_create_slice(c.data(), c.size(), bucket_numel, (int)dtype,
                                  device, index, count, &out.plan_));
  return out;
}

BucketLayout::~BucketLayout() { coadapt_plan_destroy(plan_); }
BucketLayout::BucketLayout(BucketLayout&& o) noexcept : plan_(o.plan_) {
  o.plan_ = nullptr;
}
BucketLayout& BucketLayout::operator=(BucketLayout&& o) noexcept {
  if (this != &o) {
    coadapt_plan_destroy(plan_);
    plan_ = o.plan_;
    o.plan_ = nullptr;
  }
  return *this;
}

std::uint64_t BucketLayout::active_elements() const {
  std::uint64_t a = 0;
  check(coadapt_plan_info(plan_, &a, nullptr));
  return a;
}

GnsDevicePlan::GnsDevicePlan(int dp_size, int micro_count,
                             std::int64_t global_batch, int device)
    : dp_(dp_size), micro_(micro_count), global_batch_(global_batch) {
  check(coadapt_gns_create(dp_size, micro_count, global_batch, device, &g_));
}

GnsDevicePlan::~GnsDevicePlan() { coadapt_gns_destroy(g_); }

void GnsDevicePlan::reshape(int dp_size, int micro_count,
                            std::int64_t global_batch) {
  check(coadapt_gns_reshape(g_, dp_size, micro_count, global_batch));
  dp_ = dp_size;
  micro_ = micro_count;
  global_batch_ = global_batch;
}

void GnsDevicePlan::begin_step(void* stream) {
  check(coadapt_gns_begin_step(g_, stream));
}

void GnsDevicePlan::record_micro_bucket(const BucketLayout& layout,
                                        const void* bucket, int dp_index,
                                        int micro, void* stream) {
  check(coadapt_gns_micro_sqnorm(g_, layout.handle(), bucket, dp_index, micro,
                                 stream));
}

void GnsDevicePlan::record_fused(const BucketLayout& layout,
                                 std::span<const void* const> buckets,
                                 void* stream) {
  check(coadapt_gns_fused_sqnorm(g_, layout.handle(), buckets.data(),
                                 (int)buckets.size(), stream));
}

void GnsDevicePlan::record_mean_gradient(const BucketLayout& layout,
                                         const void* mean, void* stream) {
  check(coadapt_gns_mean_sqnorm(g_, layout.handle(), mean, stream));
}

void GnsDevicePlan::record_fused_finalize(const BucketLayout& layout,
                                          std::span<const void* const> buckets,
                                          std::int64_t tokens, void* stream) {
  check(coadapt_gns_fused_sqnorm_finalize(g_, layout.handle(), buckets.data(),
                                          (int)buckets.size(), tokens, stream));
}

void GnsDevicePlan::record_mean_gradient_finalize(const BucketLayout& layout,
                                                  const void* mean,
                                                  std::int64_t tokens,
                                                  void* stream) {
  check(coadapt_gns_mean_sqnorm_finalize(g_, layout.handle(), mean, tokens,
                                         stream));
}

void GnsDevicePlan::record_micro_bucket_host(const BucketLayout& layout,
                                             const void* bucket, int dp_index,
                                             int micro, void* stream) {
  check(coadapt_gns_micro_sqnorm_host(g_, layout.handle(), bucket, dp_index,
                                      micro, stream));
}

void GnsDevicePlan::record_fused_host(const BucketLayout& layout,
                                      std::span<const void* const> buckets,
                                      void* stream) {
  check(coadapt_gns_fused_sqnorm_host(g_, layout.handle(), buckets.data(),
                                      (int)buckets.size(), stream));
}

void GnsDevicePlan::record_mean_gradient_host(const BucketLayout& layout,
                                              const void* mean, void* stream) {
  check(coadapt_gns_mean_sqnorm_host(g_, layout.handle(), mean, stream));
}

void GnsDevicePlan::accumulate(const BucketLayout& layout, float* main_grad,
                               const void* micro_grad, int dp_index, int micro,
                               bool first, bool last_mean, double mean_scale_sq,
                               void* stream) {
  const int flags = (first ? COADAPT_ACC_FIRST : 0) |
                    (last_mean ? COADAPT_ACC_LAST_MEAN : 0);
  check(coadapt_gns_accumulate(g_, layout.handle(), main_grad, micro_grad,
                               dp_index, micro, flags, mean_scale_sq, stream));
}

void GnsDevicePlan::reduce_scatter_mean(const BucketLayout& layout,
                                        std::span<const void* const> replicas,
                                        int dp_rank, void* out_slice,
                                        double scale, void* stream) {
  check(coadapt_gns_reduce_scatter_sqnorm(g_, layout.handle(), replicas.data(),
                                          (int)replicas.size(), dp_rank,
                                          out_slice, scale, stream));
}

void GnsDevicePlan::allreduce_mean(const BucketLayout& layout,
                                   std::span<void* const> replicas, int dp_rank,
                                   double scale, void* stream) {
  check(coadapt_gns_allreduce_sqnorm(g_, layout.handle(), replicas.data(),
                                     (int)replicas.size(), dp_rank, scale, stream));
}

void GnsDevicePlan::barrier(void* stream) {
  check(coadapt_gns_barrier(g_, stream));
}

void GnsDevicePlan::attach_nccl(int nranks, int rank,
                                std::span<const unsigned char> id) {
  check(coadapt_gns_attach_nccl(g_, nranks, rank, id.data(), id.size()));
}

void GnsDevicePlan::allreduce(void* stream) {
  check(coadapt_gns_allreduce(g_, stream));
}

void GnsDevicePlan::finalize(std::int64_t tokens, void* stream) {
  check(coadapt_gns_finalize(g_, tokens, stream));
}

DeviceStepResult GnsDevicePlan::result() {
  coadapt_gns_result r;
  check(coadapt_gns_read_result(g_, &r));
  DeviceStepResult o;
  o.stats = StepStats{r.stats.signal, r.stats.noise, r.stats.noise_raw,
                      r.stats.mean_grad_sq};
  o.state = from_c(r.state);
  if (r.phi_available) o.phi = r.phi;
  o.b_simple = r.b_simple;
  return o;
}

bool GnsDevicePlan::result_ready() {
  int ready = 0;
  check(coadapt_gns_result_ready(g_, &ready));
  return ready != 0;
}

StepAccumulator GnsDevicePlan::accumulator() {
  std::vector<double> v((std::size_t)dp_ * micro_ + 1);
  check(coadapt_gns_read_partials(g_, v.data(), v.size()));
  StepAccumulator acc(dp_, global_batch_);
  for (std::size_t i = 0; i + 1 < v.size(); ++i) acc.record_micro_batch(v[i]);
  return acc;
}

GnsState GnsDevicePlan::state() {
  coadapt_gns_state s;
  check(coadapt_gns_get_state(g_, &s));
  return from_c(s);
}

void GnsDevicePlan::set_state(const GnsState& s) {
  const auto c = to_c(s);
  check(coadapt_gns_set_state(g_, &c));
}

}  // namespace coadapt
