// internal.h — shared between the kernels (kernels.cu) and the C-ABI layer
// (cabi.cu).  Not installed; the public boundary is include/coadapt_cuda.h.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

namespace coadapt {
namespace dev {

// NVTX range over one C-ABI call (host side: the launches it enqueues show
// under the call's name in Nsight Systems / ncu --nvtx).  Header-only NVTX3:
// a no-op unless a tool is attached.
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};
#define COADAPT_NVTX(name) ::coadapt::dev::NvtxScope coadapt_nvtx_scope_(name)

// One maximal run of same-weight, non-zero-weight bucket elements.
// cum_begin is its first index in the "active" (compacted) element space.
struct Range {
  uint64_t abs_begin;
  uint64_t cum_begin;
  uint64_t len;
  double weight;
};

constexpr int kMaxBatch = 64;  // buckets per batched launch
constexpr int kMaxFusedM = 16; // micro-buckets per fused launch

struct BatchArgs {
  const void* ptr[kMaxBatch];
  int32_t slot[kMaxBatch];
  int32_t count;
};

struct FusedArgs {
  const void* ptr[kMaxFusedM];
  int32_t slot0;     // slot of s_{dp, 0}
  int32_t gslot;     // slot of gbar^2
  double gscale;     // 1 / M^2
};

// Where a reduction writes: per-CTA partials, the ticket of the last-block
// combine, and the accumulator slots it adds into.
struct Sink {
  double* partials;
  unsigned int* ticket;
  double* slots;
};

// Compacted-space window [e_begin, e_end) that one launch covers, and the
// pointer offset that maps abs element index -> address (base - w0*es).
struct Window {
  uint64_t e_begin;
  uint64_t e_end;
};

// Kernel launchers.  Return cudaSuccess or the launch error.  `grid` is
// computed by the caller from grid_for().
cudaError_t launch_sqnorm_batched(int dtype, const Range* ranges, int nranges,
                                  Window w, const BatchArgs& jobs, Sink sink,
                                  int grid, cudaStream_t s);
cudaError_t launch_fused(int dtype, int M, const Range* ranges, int nranges,
                         Window w, const FusedArgs& args, Sink sink, int grid,
                         cudaStream_t s);
// TMA form of the fused pass (one CTA per SM).  Chunks are numbered range by
// range: range k owns chunks [prefix[k], prefix[k+1]) covering its
// intersections with the absolute windows [j*P, (j+1)*P).
int tma_chunk_elems(int dtype, int M, bool mean = true);  // P
struct Tail;
cudaError_t launch_fused_tma(int dtype, int M, const Range* ranges, int nranges,
                             const uint64_t* prefix, uint64_t c_begin,
                             uint64_t c_end, const FusedArgs& args, Sink sink,
                             int grid, cudaStream_t s, const Tail* tail = nullptr);
// max resident CTAs per SM for the kernel that launch_* would pick
int occupancy_sqnorm(int dtype);
int occupancy_fused(int dtype, int M);
int threads_sqnorm(int dtype);
int threads_fused(int M);

// Trainer form: main_grad (+)= grad over the whole bucket, s += w*grad^2
// (slot), and with flags&2 gbar^2 += gscale*w*main_grad^2 (gslot).
struct AccumArgs {
  float* main_grad;
  const void* grad;
  int flags;  // 1: first micro-batch (main_grad = grad), 2: also gbar^2
  int32_t slot, gslot;
  double gscale;
};
int occupancy_accum(int dtype, bool first);
cudaError_t launch_accum(int dtype, const Range* full, int nfull, uint64_t numel,
                         const AccumArgs& a, Sink sink, int grid, cudaStream_t s);

// Fused DP reduce-scatter + gbar^2 over peer (NVLink) memory.
constexpr int kMaxReplicas = 8;
struct RSArgs {
  const void* rep[kMaxReplicas];  // replica buckets (peer or local pointers)
  int32_t d;
  float scale;
  void* out;                      // this rank's slice, element lo at out[0]
  int32_t gslot;
  int32_t inplace;                // 1: write the slice back into every replica
  // NVLS form (fp32): rep[] unused, the switch reduces every GPU's copy of the
  // bucket through the multicast address `mc`; inplace stores go back through
  // `mc` (multimem.st into every GPU's copy)
  const void* mc;
  int32_t nvls;
};
int occupancy_rs(int dtype);
cudaError_t launch_rs(int dtype, const Range* full, int nfull, uint64_t lo,
                      uint64_t hi, const RSArgs& a, Sink sink, int grid,
                      cudaStream_t s);

struct FinalizeArgs {
  const double* slots;
  int32_t n;               // N; slots[N] = gbar^2
  int64_t global_batch;
  int64_t tokens;
  void* state;             // coadapt_gns_state*
  void* result;            // coadapt_gns_result*
};
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t s);

// X1 + K3 in one kernel over NVLink peer memory: every rank pushes its N+1
// slots into every rank's mailbox, raises a flag, waits for all flags of
// this epoch, sums the blocks in rank order (identical bits on every rank)
// and finalizes.  Mailbox of `world` ranks, `cap` doubles per block:
//   double data[2][world][cap]; uint64 flags[2][world]   (buffer = epoch & 1)
//   uint64 epoch   (this rank's step counter, read and advanced by the
//                   kernel itself, so a CUDA-graph replay moves to the next
//                   epoch and buffer parity like an eager call)
constexpr int kMaxPeers = 8;
struct P2PArgs {
  FinalizeArgs fin;
  double* slots;             // == fin.slots, receives the global sums
  int32_t world, rank, cap;
  int64_t timeout_ns;
  char* mbox[kMaxPeers];     // rank q's mailbox (peer-mapped; own = local)
};
cudaError_t launch_p2p_finalize(const P2PArgs& a, cudaStream_t s);

// Finalize carried by the step's last reduction launch (north_star item 2:
// the estimators "fused into the same pass"): after the last CTA has
// combined the partials into the slots it runs K3 (mode 1), or first
// exchanges the slots over the NVLink mailboxes like p2p_finalize_kernel
// (mode 2).  mode 0: no tail.
struct Tail {
  int32_t mode;
  int32_t reserved_;
  P2PArgs p2p;  // mode 1 uses p2p.fin only
};
inline size_t mailbox_bytes(int world, int cap) {
  return (size_t)2 * world * cap * sizeof(double) + (size_t)2 * world * 8 + 8;
}

struct GenSeg {
  uint64_t local_off, numel, global_base, row_len, row_stride;
};
cudaError_t launch_synth(void* dst, int dtype, GenSeg seg, uint64_t seed,
                         uint64_t sample, float g0, float unit,
                         cudaStream_t s);
cudaError_t launch_synth_mean(void* dst, int dtype, GenSeg seg, uint64_t seed,
                              uint64_t sample0, int64_t nsamples, float g0,
                              float unit, cudaStream_t s);
cudaError_t launch_l2_flush(void* buf, uint64_t bytes, cudaStream_t s);
cudaError_t launch_read_probe(const void* buf, uint64_t bytes, double* sink,
                              cudaStream_t s);

}  // namespace dev
}  // namespace coadapt
