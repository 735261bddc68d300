// coadapt/device.hpp — C++ face of the B200 GNS path (RAII over the C-ABI
// in coadapt_cuda.h).  This is what replaces the caller-side s_m loop +
// record_micro_batch (gns.hpp:19-20) and the host finalize_step/update_ema/
// gns (gns.hpp:47-73) inside a trainer: gradients stay in HBM, only N+1
// scalars cross NVLink (NCCL) and ~200 bytes come back to the host.
// Failures throw the reference's exception types (errors.hpp).
#pragma once

#include <cstdint>
#include <optional>
#include <span>

#include "coadapt/gns.hpp"

struct coadapt_plan;
struct coadapt_gns;

namespace coadapt {

enum class GradDType : int { kBF16 = 0, kFP16 = 1, kFP32 = 2 };

struct BucketSegment {
  std::uint64_t offset = 0;
  std::uint64_t numel = 0;
  double weight = 1.0;  // 0: counted by another rank (TP duplicate)
};

// A rank's flattened gradient bucket layout, compiled for the device.
class BucketLayout {
 public:
  BucketLayout(std::span<const BucketSegment> segments,
               std::uint64_t bucket_numel, GradDType dtype, int device);
  // DP slice `index` of `count` (the d > 1 mean-gradient read)
  static BucketLayout slice(std::span<const BucketSegment> segments,
                            std::uint64_t bucket_numel, GradDType dtype,
                            int device, int index, int count);
  ~BucketLayout();
  BucketLayout(BucketLayout&&) noexcept;
  BucketLayout& operator=(BucketLayout&&) noexcept;
  BucketLayout(const BucketLayout&) = delete;
  BucketLayout& operator=(const BucketLayout&) = delete;

  std::uint64_t active_elements() const;
  coadapt_plan* handle() const { return plan_; }

 private:
  BucketLayout() = default;
  coadapt_plan* plan_ = nullptr;
};

struct DeviceStepResult {
  StepStats stats;
  GnsState state;
  std::optional<double> phi;
  double b_simple = 0.0;  // noise / signal of this step
};

class GnsDevicePlan {
 public:
  GnsDevicePlan(int dp_size, int micro_count, std::int64_t global_batch,
                int device);
  ~GnsDevicePlan();
  GnsDevicePlan(const GnsDevicePlan&) = delete;
  GnsDevicePlan& operator=(const GnsDevicePlan&) = delete;

  void reshape(int dp_size, int micro_count, std::int64_t global_batch);
  void begin_step(void* stream);
  void record_micro_bucket(const BucketLayout& layout, const void* bucket,
                           int dp_index, int micro, void* stream);
  void record_fused(const BucketLayout& layout,
                    std::span<const void* const> buckets, void* stream);
  void record_mean_gradient(const BucketLayout& layout, const void* mean,
                            void* stream);
  // The step's last reduction with the finalize in the same pass (and the
  // NVLink slot exchange first when mailboxes are attached): replaces the
  // allreduce + finalize calls that would follow it.
  void record_fused_finalize(const BucketLayout& layout,
                             std::span<const void* const> buckets,
                             std::int64_t tokens_this_step, void* stream);
  void record_mean_gradient_finalize(const BucketLayout& layout,
                                     const void* mean,
                                     std::int64_t tokens_this_step,
                                     void* stream);
  // The same three with the buckets in HOST memory (pinned for overlap),
  // streamed H2D through the plan's staging ring; buffers must stay valid
  // until the stream work completes.
  void record_micro_bucket_host(const BucketLayout& layout, const void* bucket,
                                int dp_index, int micro, void* stream);
  void record_fused_host(const BucketLayout& layout,
                         std::span<const void* const> buckets, void* stream);
  void record_mean_gradient_host(const BucketLayout& layout, const void* mean,
                                 void* stream);
  // Trainer form (§8 f1): main_grad (+)= grad (fp32) with s_m fused in; on
  // the last micro-batch of a d == 1 step also gbar^2 (mean_scale_sq * |main|^2).
  void accumulate(const BucketLayout& layout, float* main_grad,
                  const void* micro_grad, int dp_index, int micro, bool first,
                  bool last_mean, double mean_scale_sq, void* stream);
  // Fused DP reduce-scatter + gbar^2 over NVLink (§8 f2); replicas are the
  // DP replicas' buckets mapped into this process (CUDA IPC).
  void reduce_scatter_mean(const BucketLayout& layout,
                           std::span<const void* const> replicas, int dp_rank,
                           void* out_slice, double scale, void* stream);
  // All-reduce form: the synchronised slice is written back into every
  // replica in place (DDP gradient sync + gbar^2 in one pass).
  void allreduce_mean(const BucketLayout& layout, std::span<void* const> replicas,
                      int dp_rank, double scale, void* stream);
  void barrier(void* stream);
  void attach_nccl(int nranks, int rank, std::span<const unsigned char> id);
  void allreduce(void* stream);
  void finalize(std::int64_t tokens_this_step, void* stream);
  DeviceStepResult result();
  // non-blocking: true once result() would return without waiting
  bool result_ready();
  // the N recorded values as the reference's StepAccumulator
  StepAccumulator accumulator();
  GnsState state();
  void set_state(const GnsState& s);

  int dp_size() const { return dp_; }
  std::int64_t global_batch() const { return global_batch_; }
  coadapt_gns* handle() const { return g_; }

 private:
  coadapt_gns* g_ = nullptr;
  int dp_ = 1;
  int micro_ = 1;
  std::int64_t global_batch_ = 0;
};

}  // namespace coadapt
