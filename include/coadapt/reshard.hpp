// coadapt/reshard.hpp — the Reconfigure path a Command triggers (§8 f4).
//
// The reference ships this module as specification only (SPEC.md:414-508,
// no header): shard layouts for a (d,t,p) strategy, box-intersection
// transfer plans, a latency model, and execution.  Names and semantics
// follow SPEC.md; execution here is the B200 one — every destination rank
// pulls its regions straight out of the source ranks' HBM (or every source
// rank pushes into the destinations'), NVLink peer accesses through CUDA
// IPC pointers, one kernel per state plane, instead of the paper's
// host-staged five-phase pipeline.
//
// Layout rules (plus the choices SPEC leaves open):
//   * ranks are numbered Megatron-style, tp fastest, then dp, then pp:
//     rank = i_t + t * (i_d + d * i_p)  (same as the GNS path's layout.py);
//   * stage s holds layers [s*L/p, (s+1)*L/p);
//   * a tensor with tp_axis >= 0 is cut into t equal contiguous pieces on
//     that axis; a tensor with tp_axis < 0 is held whole by every TP rank
//     (Megatron replicates norms); the i_t == 0 copy is canonical, so the
//     canonical shards of one DP replica tile every tensor exactly;
//   * DP replicates the whole layout; replica 0 is canonical.
//   * every rank stores its shards back to back in one "pack" per state
//     plane (parameters, then each optimizer state), in (layer, tensor)
//     order, each shard row-major and starting on a 64-element boundary.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "coadapt/strategy.hpp"

struct coadapt_reshard_plan;

namespace coadapt::reshard {

inline constexpr int kMaxDims = 4;

struct TensorDecl {
  std::string name;
  std::vector<std::int64_t> shape;  // 1..kMaxDims axes
  int tp_axis = -1;                 // axis split by TP, or -1 (replicated)
};

// SPEC.md:419-423.  Bytes per element of training state = param_bytes +
// optimizer_state_multiplier * state_bytes (BF16 weights, FP32 states).
struct ModelSpec {
  int layers = 0;
  std::vector<TensorDecl> per_layer;
  int optimizer_state_multiplier = 2;
  int param_bytes = 2;
  int state_bytes = 4;

  int bytes_per_element() const {
    return param_bytes + optimizer_state_multiplier * state_bytes;
  }
  std::string key(int layer, int tensor) const;  // "layer<l>.<name>"
};

// SPEC.md:425-429 (+ pack placement and the canonical flag).
struct ShardDescriptor {
  int layer = 0;
  int tensor = 0;  // index into ModelSpec::per_layer
  std::vector<std::int64_t> global_shape;
  std::vector<std::int64_t> global_offset;
  std::vector<std::int64_t> local_shape;
  int owner = 0;
  bool canonical = false;        // DP replica 0 and (replicated) TP copy 0
  std::uint64_t pack_offset = 0; // element offset in the owner's pack

  std::uint64_t numel() const;
};

// SPEC.md:431-436.
struct ShardLayout {
  ParallelStrategy strategy;
  std::vector<ShardDescriptor> shards;
  std::vector<std::vector<int>> replica_groups;  // [i_d] -> ranks
  std::vector<std::uint64_t> pack_numel;         // per rank, padded

  std::uint64_t max_pack_numel() const;
};

// Which source copy feeds a destination piece that is not already on the
// destination rank.  kCanonical is SPEC.md:492 (always DP replica 0);
// kSpread reads from source replica (dst i_d mod src d) so that several
// destination replicas do not all pull through one GPU's NVLink ports.
// Wire bytes are the same for both.
enum class SourcePolicy : int { kCanonical = 0, kSpread = 1 };

// SPEC.md:438-442.
struct Move {
  int src_rank = 0;
  int dst_rank = 0;
  int layer = 0;
  int tensor = 0;
  std::vector<std::int64_t> offset;  // global box
  std::vector<std::int64_t> extent;
  std::uint64_t bytes = 0;           // elements * bytes_per_element
  bool local = false;                // src_rank == dst_rank: no wire bytes
  std::size_t src_shard = 0;         // indices into the layouts' shards
  std::size_t dst_shard = 0;
};

struct TransferPlan {
  std::vector<Move> moves;
  std::uint64_t total_bytes = 0;         // wire bytes (non-local moves)
  std::uint64_t max_bytes_per_rank = 0;  // max wire bytes one rank receives
  std::uint64_t local_bytes = 0;
};

// ValidationError on an invalid strategy, L % p != 0, a TP axis not
// divisible by t, or a malformed tensor declaration.
ShardLayout layout_for(const ModelSpec& model, const ParallelStrategy& s,
                       int n_gpus);

// every destination shard is cut along the canonical
// source shards' boxes; a piece already held by the destination rank (any
// source copy) is a local move.  InternalError if a shard is left uncovered.
TransferPlan plan_transfers(const ModelSpec& model, const ShardLayout& src,
                            const ShardLayout& dst,
                            SourcePolicy policy = SourcePolicy::kCanonical);

// fixed_overhead + wire bytes / bandwidth.  Defaults are
// host-staged figures that put 3B-scale transitions in the paper's
// 30-56 s band; pass the NVLink figure for the device
// executor.
inline constexpr double kDefaultReshardBandwidth = 1.0e9;  // bytes/s
inline constexpr double kDefaultReshardOverhead = 20.0;    // seconds
double estimate_reconfig_latency(
    const TransferPlan& plan,
    double bandwidth_bytes_per_s = kDefaultReshardBandwidth,
    double fixed_overhead_s = kDefaultReshardOverhead);

// "key,src_rank,dst_rank,offsets,extents,bytes,local".
std::string transfer_plan_csv(const ModelSpec& model, const TransferPlan& plan);

// The device executor (RAII over coadapt_reshard.h): both layouts, the
// plan, and the copy-task tables it builds per (role, rank, element size).
// pull(r): copy every move into destination rank r (sources: this GPU's
// and NVLink peers' packs); push(r): every move out of source rank r;
// all(): every move (all packs visible to this process).  Pack pointer
// arrays are indexed by rank (nullptr where unused).  Throws
// ValidationError / InternalError like the rest of the API.
class DevicePlan {
 public:
  DevicePlan(const ModelSpec& model, const ParallelStrategy& src,
             const ParallelStrategy& dst,
             SourcePolicy policy = SourcePolicy::kCanonical);
  ~DevicePlan();
  DevicePlan(const DevicePlan&) = delete;
  DevicePlan& operator=(const DevicePlan&) = delete;

  const ShardLayout& source() const { return src_; }
  const ShardLayout& destination() const { return dst_; }
  const TransferPlan& plan() const { return plan_; }

  void pull(int dst_rank, std::span<const void* const> src_packs,
            std::span<void* const> dst_packs, int elem_bytes, int device,
            void* stream);
  void push(int src_rank, std::span<const void* const> src_packs,
            std::span<void* const> dst_packs, int elem_bytes, int device,
            void* stream);
  void all(std::span<const void* const> src_packs,
           std::span<void* const> dst_packs, int elem_bytes, int device,
           void* stream);

 private:
  void run(int role, int rank, std::span<const void* const> src_packs,
           std::span<void* const> dst_packs, int elem_bytes, int device,
           void* stream);
  ShardLayout src_, dst_;
  TransferPlan plan_;
  coadapt_reshard_plan* handle_ = nullptr;
};

}  // namespace coadapt::reshard
