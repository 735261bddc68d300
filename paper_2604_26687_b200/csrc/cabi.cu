// cabi.cu — the extern "C" boundary declared in include/coadapt_cuda.h.
// Owns plans (device range tables), step accumulators (device slots +
// GnsState), the NCCL communicator and the host-streaming staging ring.
// No C++ exception crosses this boundary; failures return a status and set
// a thread-local message (errors.hpp taxonomy, SPEC.md:635 exit codes).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/coadapt_cuda.h"
#include "internal.h"

using coadapt::dev::BatchArgs;
using coadapt::dev::FusedArgs;
using coadapt::dev::Range;
using coadapt::dev::Sink;
using coadapt::dev::Window;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace coadapt_capi {
// used by the C++-API bindings (host/capi.cpp) to share the message slot
void set_error(const char* msg) { g_err = msg ? msg : ""; }
// kernels launched from the other translation units (reshard.cu)
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace coadapt_capi

namespace {

#define CU(call)                                                          \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess)                                                \
      return fail(COADAPT_E_CUDA, std::string(#call) + ": " +             \
                                      cudaGetErrorString(e_));            \
  } while (0)

#define NC(call)                                                          \
  do {                                                                    \
    ncclResult_t r_ = (call);                                             \
    if (r_ != ncclSuccess)                                                \
      return fail(COADAPT_E_NCCL,                                         \
                  std::string(#call) + ": " + ncclGetErrorString(r_));    \
  } while (0)

// Makes `dev` current for the scope of a call and restores the caller's.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev)
      cudaSetDevice(prev);
  }
};

#define GUARD(dev)                                                        \
  DeviceGuard guard_(dev);                                                \
  if (guard_.err != cudaSuccess)                                          \
    return fail(COADAPT_E_CUDA, std::string("device ") +                  \
                                    std::to_string(dev) + ": " +          \
                                    cudaGetErrorString(guard_.err))

int esize(int dtype) {
  switch (dtype) {
    case COADAPT_BF16:
    case COADAPT_FP16: return 2;
    case COADAPT_FP32: return 4;
    case COADAPT_FP64: return 8;
  }
  return 0;
}

int sm_count(int dev) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
      cudaSuccess)
    return 0;
  return n;
}

// CTAs for a reduction over `active` elements: a full resident wave
// (SMs x occupancy) unless the pass is too small to feed it (>= 16 Ki
// elements per CTA keeps the per-CTA fixed cost below a few percent).
int grid_for(int dev, int occ, uint64_t active) {
  const int full = std::max(1, sm_count(dev) * std::max(1, occ));
  const uint64_t by_size = (active + 16383) / 16384;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(full, by_size));
}

constexpr int kMaxGridPerSM = 8;  // 2048 threads / 256
constexpr uint64_t kStageElems = 16ull << 20;  // host streaming chunk
constexpr int kStages = 3;

}  // namespace

struct coadapt_plan {
  int device = 0;
  int dtype = COADAPT_BF16;
  uint64_t bucket_numel = 0;
  uint64_t active = 0;
  std::vector<Range> host;  // ranges, sorted, merged
  Range* ranges = nullptr;  // device copy
  // TMA chunk numbering per chunk size P: prefix[k] = first chunk of range k
  struct Chunks {
    std::vector<uint64_t> prefix;
    uint64_t* dev = nullptr;
    bool pooled = false;  // dev points into chunk_pool
  };
  // deque: references stay valid while other P values are added
  std::deque<std::pair<int, Chunks>> chunks;
  // every table the TMA launches can ask for, uploaded at plan creation in
  // one allocation (so no launch path allocates or copies synchronously and
  // a step can be captured into a CUDA graph without an eager warm-up)
  uint64_t* chunk_pool = nullptr;
  std::mutex mu;  // guards the lazily built tables (chunks, full)
  // whole-bucket table for the trainer form (weight-0 ranges and gaps
  // included, abs == cum); built lazily, not for DP-slice plans
  bool is_slice = false;
  std::vector<Range> full_host;
  Range* full = nullptr;
  std::vector<coadapt_segment> segs;  // as given (sorted)
};

struct coadapt_gns {
  int device = 0;
  int dp = 1, M = 1, N = 1;
  int64_t global_batch = 0;
  int sms = 0;
  double* slots = nullptr;      // N+1 (capacity slot_cap)
  int slot_cap = 0;
  double* partials = nullptr;   // per-CTA partials
  size_t partial_cap = 0;       // doubles
  unsigned int* ticket = nullptr;
  void* state = nullptr;        // coadapt_gns_state (device)
  void* result = nullptr;       // coadapt_gns_result (device)
  coadapt_gns_result* result_host = nullptr;  // pinned
  cudaEvent_t result_ready = nullptr;
  bool finalized = false;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  double* barrier_buf = nullptr;  // coadapt_gns_barrier scratch
  // NVLink slot exchange (coadapt_gns_allreduce_finalize_p2p)
  void* mbox = nullptr;
  int mbox_world = 0, mbox_cap = 0, mbox_rank = -1;
  char* mbox_peers[coadapt::dev::kMaxPeers] = {};
  // host streaming (coadapt_gns_fused_sqnorm_host)
  void* staging = nullptr;  // kStages * 16 * kStageElems * es bytes
  size_t staging_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t stage_free[kStages] = {};
  cudaEvent_t stage_full[kStages] = {};
};

namespace {

int alloc_slots(coadapt_gns* g, int n_slots) {
  if (n_slots <= g->slot_cap) return COADAPT_OK;
  if (g->slots) cudaFree(g->slots);
  g->slots = nullptr;
  CU(cudaMalloc(&g->slots, sizeof(double) * n_slots));
  CU(cudaMemset(g->slots, 0, sizeof(double) * n_slots));
  g->slot_cap = n_slots;
  return COADAPT_OK;
}

int validate_dtype(int dtype, bool fp64_ok) {
  if (dtype == COADAPT_BF16 || dtype == COADAPT_FP16 ||
      dtype == COADAPT_FP32 || (fp64_ok && dtype == COADAPT_FP64))
    return COADAPT_OK;
  return fail(COADAPT_E_VALIDATION, "unsupported dtype " + std::to_string(dtype));
}

int build_ranges(const coadapt_segment* segs, size_t nseg,
                 uint64_t bucket_numel, uint64_t lo, uint64_t hi,
                 std::vector<Range>& out, uint64_t& active) {
  std::vector<coadapt_segment> v(segs, segs + nseg);
  for (const auto& s : v) {
    if (!std::isfinite(s.weight))
      return fail(COADAPT_E_VALIDATION, "segment weight is not finite");
    if (s.offset > bucket_numel || s.numel > bucket_numel - s.offset)
      return fail(COADAPT_E_VALIDATION,
                  "segment [" + std::to_string(s.offset) + ", +" +
                      std::to_string(s.numel) + ") exceeds bucket of " +
                      std::to_string(bucket_numel) + " elements");
  }
  std::stable_sort(v.begin(), v.end(),
                   [](const coadapt_segment& a, const coadapt_segment& b) {
                     return a.offset < b.offset;
                   });
  for (size_t i = 1; i < v.size(); ++i)
    if (v[i].offset < v[i - 1].offset + v[i - 1].numel)
      return fail(COADAPT_E_VALIDATION, "segments overlap at element " +
                                            std::to_string(v[i].offset));
  out.clear();
  active = 0;
  for (const auto& s : v) {
    if (s.weight == 0.0 || s.numel == 0) continue;
    uint64_t b = std::max(s.offset, lo), e = std::min(s.offset + s.numel, hi);
    if (b >= e) continue;
    if (!out.empty() && out.back().weight == s.weight &&
        out.back().abs_begin + out.back().len == b) {
      out.back().len += e - b;
    } else {
      out.push_back(Range{b, active, e - b, s.weight});
    }
    active += e - b;
  }
  return COADAPT_OK;
}

int plan_all_chunks(coadapt_plan* p);
int plan_full(coadapt_plan* p);

int plan_make(const coadapt_segment* segs, size_t nseg, uint64_t bucket_numel,
              int dtype, int device, uint64_t lo, uint64_t hi,
              coadapt_plan** out) {
  if (!out) return fail(COADAPT_E_VALIDATION, "out is NULL");
  *out = nullptr;
  if (nseg && !segs) return fail(COADAPT_E_VALIDATION, "segs is NULL");
  if (int rc = validate_dtype(dtype, true)) return rc;
  GUARD(device);
  auto* p = new coadapt_plan;
  p->device = device;
  p->dtype = dtype;
  p->bucket_numel = bucket_numel;
  if (int rc = build_ranges(segs, nseg, bucket_numel, lo, hi, p->host,
                            p->active)) {
    delete p;
    return rc;
  }
  p->is_slice = !(lo == 0 && hi == bucket_numel);
  p->segs.assign(segs, segs + nseg);
  std::stable_sort(p->segs.begin(), p->segs.end(),
                   [](const coadapt_segment& a, const coadapt_segment& b) {
                     return a.offset < b.offset;
                   });
  if (!p->host.empty()) {
    cudaError_t e = cudaMalloc(&p->ranges, sizeof(Range) * p->host.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(p->ranges, p->host.data(), sizeof(Range) * p->host.size(),
                     cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      if (p->ranges) cudaFree(p->ranges);
      delete p;
      return fail(COADAPT_E_CUDA, std::string("plan upload: ") +
                                      cudaGetErrorString(e));
    }
    if (int rc = plan_all_chunks(p)) {
      coadapt_plan_destroy(p);
      return rc;
    }
    if (!p->is_slice)
      if (int rc = plan_full(p)) {
        coadapt_plan_destroy(p);
        return rc;
      }
  }
  *out = p;
  return COADAPT_OK;
}

int check_bucket(const coadapt_plan* p, const void* ptr, const char* what) {
  if (!ptr && p->active) return fail(COADAPT_E_VALIDATION, std::string(what) + " is NULL");
  if (reinterpret_cast<uintptr_t>(ptr) % esize(p->dtype))
    return fail(COADAPT_E_VALIDATION,
                std::string(what) + " is not aligned to its element size");
  return COADAPT_OK;
}

int ensure_partials(coadapt_gns* g, size_t n) {
  if (n <= g->partial_cap) return COADAPT_OK;
  // growth is a synchronous cudaFree/cudaMalloc: callers size it up front
  if (g->partials) {
    CU(cudaDeviceSynchronize());
    cudaFree(g->partials);
    g->partials = nullptr;
  }
  CU(cudaMalloc(&g->partials, n * sizeof(double)));
  g->partial_cap = n;
  return COADAPT_OK;
}

int check_slot(const coadapt_gns* g, int dp_index, int micro) {
  if (dp_index < 0 || dp_index >= g->dp || micro < 0 || micro >= g->M)
    return fail(COADAPT_E_VALIDATION,
                "slot (dp=" + std::to_string(dp_index) + ", m=" +
                    std::to_string(micro) + ") outside d=" +
                    std::to_string(g->dp) + ", M=" + std::to_string(g->M));
  return COADAPT_OK;
}

int launch_batch(coadapt_gns* g, const coadapt_plan* p, const BatchArgs& jobs,
                 Window w, cudaStream_t s) {
  const uint64_t n = w.e_end - w.e_begin;
  if (n == 0 || jobs.count == 0) return COADAPT_OK;
  const int grid =
      grid_for(g->device, coadapt::dev::occupancy_sqnorm(p->dtype), n);
  if (int rc = ensure_partials(g, (size_t)grid * jobs.count)) return rc;
  Sink sink{g->partials, g->ticket, g->slots};
  CU(coadapt::dev::launch_sqnorm_batched(p->dtype, p->ranges,
                                         (int)p->host.size(), w, jobs, sink,
                                         grid, s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

int launch_fused_window(coadapt_gns* g, const coadapt_plan* p,
                        const FusedArgs& fa, int M, Window w, cudaStream_t s) {
  const uint64_t n = w.e_end - w.e_begin;
  if (n == 0) return COADAPT_OK;
  const int grid =
      grid_for(g->device, coadapt::dev::occupancy_fused(p->dtype, M), n);
  if (int rc = ensure_partials(g, (size_t)grid * (M + 1))) return rc;
  Sink sink{g->partials, g->ticket, g->slots};
  CU(coadapt::dev::launch_fused(p->dtype, M, p->ranges, (int)p->host.size(), w,
                                fa, sink, grid, s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

std::vector<uint64_t> chunk_prefix(const coadapt_plan* p, int P) {
  std::vector<uint64_t> prefix(p->host.size() + 1);
  uint64_t acc = 0;
  for (size_t k = 0; k < p->host.size(); ++k) {
    prefix[k] = acc;
    const uint64_t rb = p->host[k].abs_begin, re = rb + p->host[k].len;
    acc += (re - 1) / P - rb / P + 1;
  }
  prefix.back() = acc;
  return prefix;
}

// The chunk numbering for every chunk size P a TMA launch of this plan can
// use (K1 over 1..16 buckets, K1f for M = 2..16, the host-streaming fused
// form), built once at plan creation into one device allocation.
int plan_all_chunks(coadapt_plan* p) {
  std::vector<int> Ps;
  for (int M = 1; M <= coadapt::dev::kMaxFusedM; ++M)
    for (bool mean : {false, true}) {
      const int P = coadapt::dev::tma_chunk_elems(p->dtype, M, mean);
      if (P > 0 && std::find(Ps.begin(), Ps.end(), P) == Ps.end()) Ps.push_back(P);
    }
  if (Ps.empty()) return COADAPT_OK;
  const size_t per = p->host.size() + 1;
  std::vector<uint64_t> all;
  all.reserve(per * Ps.size());
  for (int P : Ps) {
    const auto v = chunk_prefix(p, P);
    all.insert(all.end(), v.begin(), v.end());
  }
  CU(cudaMalloc(&p->chunk_pool, sizeof(uint64_t) * all.size()));
  CU(cudaMemcpy(p->chunk_pool, all.data(), sizeof(uint64_t) * all.size(),
                cudaMemcpyHostToDevice));
  std::lock_guard<std::mutex> lock(p->mu);
  for (size_t i = 0; i < Ps.size(); ++i) {
    coadapt_plan::Chunks c;
    c.prefix.assign(all.begin() + i * per, all.begin() + (i + 1) * per);
    c.dev = p->chunk_pool + i * per;
    c.pooled = true;
    p->chunks.emplace_back(Ps[i], std::move(c));
  }
  return COADAPT_OK;
}

// chunk numbering of `p` for chunk size P: from the tables built at
// creation; any other P is built here (synchronous; not reached by the
// library's own launch shapes)
int plan_chunks(coadapt_plan* p, int P, const coadapt_plan::Chunks** out) {
  std::lock_guard<std::mutex> lock(p->mu);
  for (auto& kv : p->chunks)
    if (kv.first == P) {
      *out = &kv.second;
      return COADAPT_OK;
    }
  coadapt_plan::Chunks c;
  c.prefix = chunk_prefix(p, P);
  CU(cudaMalloc(&c.dev, sizeof(uint64_t) * c.prefix.size()));
  const cudaError_t e = cudaMemcpy(c.dev, c.prefix.data(),
                                   sizeof(uint64_t) * c.prefix.size(),
                                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(c.dev);
    return fail(COADAPT_E_CUDA, std::string("chunk table upload: ") +
                                    cudaGetErrorString(e));
  }
  p->chunks.emplace_back(P, std::move(c));
  *out = &p->chunks.back().second;
  return COADAPT_OK;
}

// number of chunks (size P) that start before absolute element x (x is a
// multiple of P, or the bucket end): per range, its chunks j with j*P < x
uint64_t chunks_before(const coadapt_plan* p, const coadapt_plan::Chunks* ch,
                       int P, uint64_t x) {
  uint64_t n = 0;
  const uint64_t jx = (x + P - 1) / P;
  for (size_t k = 0; k < p->host.size(); ++k) {
    const uint64_t rb = p->host[k].abs_begin, re = rb + p->host[k].len;
    const uint64_t j0 = rb / P, j1 = (re - 1) / P + 1;  // chunks [j0, j1)
    if (jx <= j0) break;
    n = ch->prefix[k] + (std::min(jx, j1) - j0);
  }
  return n;
}

// whole-bucket range table (every element exactly once; gaps weight 0)
int plan_full(coadapt_plan* p) {
  std::lock_guard<std::mutex> lock(p->mu);
  if (p->full || p->bucket_numel == 0) return COADAPT_OK;
  std::vector<Range>& f = p->full_host;
  f.clear();
  uint64_t at = 0;
  auto push = [&](uint64_t b, uint64_t n, double w) {
    if (n == 0) return;
    if (!f.empty() && f.back().weight == w && f.back().abs_begin + f.back().len == b)
      f.back().len += n;
    else
      f.push_back(Range{b, b, n, w});
  };
  for (const auto& s : p->segs) {
    if (s.offset > at) push(at, s.offset - at, 0.0);
    push(s.offset, s.numel, s.weight);
    at = s.offset + s.numel;
  }
  if (at < p->bucket_numel) push(at, p->bucket_numel - at, 0.0);
  Range* dev = nullptr;
  CU(cudaMalloc(&dev, sizeof(Range) * f.size()));
  const cudaError_t e = cudaMemcpy(dev, f.data(), sizeof(Range) * f.size(),
                                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(dev);
    return fail(COADAPT_E_CUDA, std::string("range table upload: ") +
                                    cudaGetErrorString(e));
  }
  p->full = dev;
  return COADAPT_OK;
}

bool use_tma_path() {
  static const char* e = getenv("COADAPT_FUSED_PATH");
  return !(e && std::string(e) == "ldg");
}

// the finalize tail as its own launch (when no TMA launch could carry it)
int launch_tail_separately(const coadapt::dev::Tail& t, cudaStream_t s) {
  if (t.mode == 2)
    CU(coadapt::dev::launch_p2p_finalize(t.p2p, s));
  else
    CU(coadapt::dev::launch_finalize(t.p2p.fin, s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

int launch_fused_tma_all(coadapt_gns* g, coadapt_plan* p, const FusedArgs& fa,
                         int M, cudaStream_t s,
                         const coadapt::dev::Tail* tail = nullptr) {
  const int P = coadapt::dev::tma_chunk_elems(p->dtype, M, fa.gslot >= 0);
  if (P <= 0) return fail(COADAPT_E_INTERNAL, "no TMA kernel for this dtype/M");
  const coadapt_plan::Chunks* ch = nullptr;
  if (int rc = plan_chunks(p, P, &ch)) return rc;
  const uint64_t nch = ch->prefix.back();
  if (nch == 0) return tail ? launch_tail_separately(*tail, s) : COADAPT_OK;
  const int grid = (int)std::min<uint64_t>(std::max(1, g->sms), nch);
  if (int rc = ensure_partials(g, (size_t)grid * (M + 1))) return rc;
  Sink sink{g->partials, g->ticket, g->slots};
  CU(coadapt::dev::launch_fused_tma(p->dtype, M, p->ranges, (int)p->host.size(),
                                    ch->dev, 0, nch, fa, sink, grid, s, tail));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

// compacted index of the first active element at or after abs index x
uint64_t cum_at(const coadapt_plan* p, uint64_t x) {
  const auto& R = p->host;
  auto it = std::upper_bound(R.begin(), R.end(), x,
                             [](uint64_t v, const Range& r) {
                               return v < r.abs_begin;
                             });
  if (it == R.begin()) return 0;
  --it;
  if (x >= it->abs_begin + it->len) return it->cum_begin + it->len;
  return it->cum_begin + (x - it->abs_begin);
}

coadapt_gns_state default_state() {
  coadapt_gns_state s;
  std::memset(&s, 0, sizeof(s));
  s.alpha_early = 0.95;
  s.alpha_late = 0.99;
  s.phase_boundary_tokens = 8000000;
  s.calibration = 2.0;
  return s;
}

std::mutex g_oneshot_mu;

// The host-streaming staging ring: kStages stages of kMaxFusedM * kStageElems
// elements (sized for 8-byte elements on first use is wasteful; it is sized
// for this element size and grown never — every later caller must fit).
int ensure_staging(coadapt_gns* g, int es) {
  const size_t need = (size_t)kStages * coadapt::dev::kMaxFusedM * kStageElems * es;
  if (!g->staging) {
    CU(cudaMalloc(&g->staging, need));
    g->staging_bytes = need;
    CU(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < kStages; ++i) {
      CU(cudaEventCreateWithFlags(&g->stage_free[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&g->stage_full[i], cudaEventDisableTiming));
    }
  } else if (g->staging_bytes < need) {
    return fail(COADAPT_E_VALIDATION,
                "host streaming: this gns's staging ring was sized for a "
                "smaller element type");
  }
  return COADAPT_OK;
}

// K1 over a HOST bucket: the plan's span of absolute elements is streamed
// through the staging ring in windows of one whole stage; each window is
// reduced (batched K1, one job) as it lands, into `slot`.
int stream_host_k1(coadapt_gns* g, const coadapt_plan* p, const void* host,
                   int slot, cudaStream_t s) {
  if (p->host.empty()) return COADAPT_OK;
  const int es = esize(p->dtype);
  if (int rc = ensure_staging(g, es)) return rc;
  const uint64_t win = (uint64_t)coadapt::dev::kMaxFusedM * kStageElems;
  const size_t stage_bytes = (size_t)win * es;
  const uint64_t lo = p->host.front().abs_begin;
  const uint64_t hi = p->host.back().abs_begin + p->host.back().len;
  for (int i = 0; i < kStages; ++i) CU(cudaEventRecord(g->stage_free[i], s));
  const uint64_t nwin = (hi - lo + win - 1) / win;
  for (uint64_t c = 0; c < nwin; ++c) {
    const uint64_t w0 = lo + c * win, w1 = std::min(hi, w0 + win);
    const uint64_t cb = cum_at(p, w0), ce = cum_at(p, w1);
    if (ce == cb) continue;  // only weight-0 data in this window
    const int st = (int)(c % kStages);
    char* stage = static_cast<char*>(g->staging) + (size_t)st * stage_bytes;
    CU(cudaStreamWaitEvent(g->copy_stream, g->stage_free[st], 0));
    CU(cudaMemcpyAsync(stage, static_cast<const char*>(host) + w0 * es,
                       (w1 - w0) * es, cudaMemcpyHostToDevice, g->copy_stream));
    CU(cudaEventRecord(g->stage_full[st], g->copy_stream));
    CU(cudaStreamWaitEvent(s, g->stage_full[st], 0));
    BatchArgs jobs;
    std::memset(&jobs, 0, sizeof(jobs));
    jobs.count = 1;
    jobs.ptr[0] = stage - w0 * es;  // abs element x lives at stage + (x-w0)*es
    jobs.slot[0] = slot;
    if (int rc = launch_batch(g, p, jobs, Window{cb, ce}, s)) return rc;
    CU(cudaEventRecord(g->stage_free[st], s));
  }
  return COADAPT_OK;
}

// K1 over 1..16 buckets sharing plan p through the fused pass's TMA ring
// without its mean term, when every bucket is 16-byte aligned: the same exact
// arithmetic as the LDG batch at a higher rate under the power cap (single
// bucket 6.77 -> 7.33 TB/s burst, 5.97 -> 6.79 sustained; C2 step +13 %,
// profiles/r01c_k1_tma.txt).  Returns false (nothing launched) when the
// buckets do not qualify; *rc is the launch status otherwise.
bool try_tma_k1(coadapt_gns* g, const coadapt_plan* p, const void* const* buckets,
                int count, int slot0, cudaStream_t s, int* rc,
                const coadapt::dev::Tail* tail = nullptr) {
  if (!use_tma_path() || count < 1 || count > coadapt::dev::kMaxFusedM) return false;
  for (int j = 0; j < count; ++j)
    if (!buckets[j] || (reinterpret_cast<uintptr_t>(buckets[j]) & 15)) return false;
  FusedArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  for (int j = 0; j < count; ++j) {
    if ((*rc = check_bucket(p, buckets[j], "bucket"))) return true;
    fa.ptr[j] = buckets[j];
  }
  fa.slot0 = slot0;
  fa.gslot = -1;
  *rc = launch_fused_tma_all(g, const_cast<coadapt_plan*>(p), fa, count, s, tail);
  return true;
}

// The step's finalize carried by its last reduction (coadapt_gns_*_finalize):
// mode 2 exchanges the slots over the attached NVLink mailboxes first.
int make_tail(coadapt_gns* g, int64_t tokens, coadapt::dev::Tail* t) {
  if (tokens < 0) return fail(COADAPT_E_VALIDATION, "tokens must be >= 0");
  std::memset(t, 0, sizeof(*t));
  t->p2p.fin = coadapt::dev::FinalizeArgs{g->slots, g->N, g->global_batch, tokens,
                                          g->state, g->result};
  t->p2p.slots = g->slots;
  if (g->mbox_rank >= 0 && g->mbox_world > 1) {
    if (g->N + 1 > g->mbox_cap)
      return fail(COADAPT_E_VALIDATION,
                  "d*M grew past the mailbox capacity: recreate the mailboxes");
    t->mode = 2;
    t->p2p.world = g->mbox_world;
    t->p2p.rank = g->mbox_rank;
    t->p2p.cap = g->mbox_cap;
    t->p2p.timeout_ns = 10'000'000'000ll;
    for (int q = 0; q < g->mbox_world; ++q) t->p2p.mbox[q] = g->mbox_peers[q];
    return COADAPT_OK;
  }
  if (g->comm && g->nranks > 1)
    return fail(COADAPT_E_VALIDATION,
                "in-pass finalize across ranks needs the NVLink mailboxes "
                "(coadapt_gns_attach_mailboxes); with NCCL use allreduce + finalize");
  t->mode = 1;
  return COADAPT_OK;
}

// result D2H + completion event, as after coadapt_gns_finalize
int finish_result(coadapt_gns* g, cudaStream_t s) {
  CU(cudaMemcpyAsync(g->result_host, g->result, sizeof(coadapt_gns_result),
                     cudaMemcpyDeviceToHost, s));
  // Under stream capture a plain record only orders nodes inside the graph;
  // an external record node makes every replay signal result_ready, so
  // read_result() after graph.replay() waits for that replay's D2H.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(s, &cap));
  if (cap == cudaStreamCaptureStatusActive)
    CU(cudaEventRecordWithFlags(g->result_ready, s, cudaEventRecordExternal));
  else
    CU(cudaEventRecord(g->result_ready, s));
  g->finalized = true;
  return COADAPT_OK;
}

}  // namespace

// ====================================================================== API

extern "C" {

const char* coadapt_last_error(void) { return g_err.c_str(); }
int coadapt_abi_version(void) { return COADAPT_ABI_VERSION; }
uint64_t coadapt_kernel_launches(void) {
  return g_launches.load(std::memory_order_relaxed);
}

int coadapt_device_info(int device, int* sm, int* l2, int* major, int* minor) {
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (sm) *sm = prop.multiProcessorCount;
  if (l2) *l2 = prop.l2CacheSize;
  if (major) *major = prop.major;
  if (minor) *minor = prop.minor;
  return COADAPT_OK;
}

int coadapt_plan_create(const coadapt_segment* segs, size_t nseg,
                        uint64_t bucket_numel, int dtype, int device,
                        coadapt_plan** out) {
  COADAPT_NVTX("coadapt_plan_create");
  return plan_make(segs, nseg, bucket_numel, dtype, device, 0, bucket_numel,
                   out);
}

int coadapt_plan_create_slice(const coadapt_segment* segs, size_t nseg,
                              uint64_t bucket_numel, int dtype, int device,
                              int index, int count, coadapt_plan** out) {
  COADAPT_NVTX("coadapt_plan_create_slice");
  if (count < 1 || index < 0 || index >= count)
    return fail(COADAPT_E_VALIDATION, "slice index/count out of range");
  auto cut = [&](int i) -> uint64_t {
    if (i >= count) return bucket_numel;
    const unsigned __int128 x = (unsigned __int128)bucket_numel * i / count;
    return (uint64_t)x & ~uint64_t(63);
  };
  return plan_make(segs, nseg, bucket_numel, dtype, device, cut(index),
                   cut(index + 1), out);
}

int coadapt_plan_destroy(coadapt_plan* p) {
  if (!p) return COADAPT_OK;
  {
    DeviceGuard guard(p->device);
    if (p->ranges) cudaFree(p->ranges);
    if (p->full) cudaFree(p->full);
    for (auto& kv : p->chunks)
      if (kv.second.dev && !kv.second.pooled) cudaFree(kv.second.dev);
    if (p->chunk_pool) cudaFree(p->chunk_pool);
  }
  delete p;
  return COADAPT_OK;
}

int coadapt_plan_info(const coadapt_plan* p, uint64_t* active,
                      uint64_t* nranges) {
  if (!p) return fail(COADAPT_E_VALIDATION, "plan is NULL");
  if (active) *active = p->active;
  if (nranges) *nranges = p->host.size();
  return COADAPT_OK;
}

int coadapt_gns_create(int dp_size, int micro_count, int64_t global_batch,
                       int device, coadapt_gns** out) {
  if (!out) return fail(COADAPT_E_VALIDATION, "out is NULL");
  *out = nullptr;
  if (dp_size < 1 || micro_count < 1)
    return fail(COADAPT_E_VALIDATION, "dp_size and micro_count must be >= 1");
  if ((int64_t)dp_size * micro_count < 2)
    return fail(COADAPT_E_VALIDATION,
                "N = d*M must be >= 2 (gns.hpp:45, SPEC.md:179)");
  if (global_batch < 1)
    return fail(COADAPT_E_VALIDATION, "global_batch must be >= 1");
  GUARD(device);
  auto* g = new coadapt_gns;
  g->device = device;
  g->dp = dp_size;
  g->M = micro_count;
  g->N = dp_size * micro_count;
  g->global_batch = global_batch;
  g->sms = sm_count(device);
  auto cleanup = [&](int rc) {
    coadapt_gns_destroy(g);
    return rc;
  };
  if (int rc = alloc_slots(g, g->N + 1)) return cleanup(rc);
  const size_t cap = (size_t)std::max(1, g->sms) * kMaxGridPerSM *
                     std::max(coadapt::dev::kMaxBatch,
                              coadapt::dev::kMaxFusedM + 1);
  if (int rc = ensure_partials(g, cap)) return cleanup(rc);
  cudaError_t e = cudaMalloc(&g->ticket, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(g->ticket, 0, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMalloc(&g->state, sizeof(coadapt_gns_state));
  if (e == cudaSuccess) {
    const coadapt_gns_state s = default_state();
    e = cudaMemcpy(g->state, &s, sizeof(s), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaMalloc(&g->result, sizeof(coadapt_gns_result));
  if (e == cudaSuccess)
    e = cudaHostAlloc((void**)&g->result_host, sizeof(coadapt_gns_result),
                      cudaHostAllocDefault);
  if (e == cudaSuccess)
    e = cudaEventCreateWithFlags(&g->result_ready, cudaEventDisableTiming);
  if (e != cudaSuccess)
    return cleanup(fail(COADAPT_E_CUDA, std::string("gns_create: ") +
                                            cudaGetErrorString(e)));
  *out = g;
  return COADAPT_OK;
}

int coadapt_gns_destroy(coadapt_gns* g) {
  if (!g) return COADAPT_OK;
  {
    DeviceGuard guard(g->device);
    cudaDeviceSynchronize();
    if (g->comm) ncclCommDestroy(g->comm);
    if (g->barrier_buf) cudaFree(g->barrier_buf);
    if (g->mbox) cudaFree(g->mbox);
    if (g->slots) cudaFree(g->slots);
    if (g->partials) cudaFree(g->partials);
    if (g->ticket) cudaFree(g->ticket);
    if (g->state) cudaFree(g->state);
    if (g->result) cudaFree(g->result);
    if (g->result_host) cudaFreeHost(g->result_host);
    if (g->result_ready) cudaEventDestroy(g->result_ready);
    if (g->staging) cudaFree(g->staging);
    if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
    for (int i = 0; i < kStages; ++i) {
      if (g->stage_free[i]) cudaEventDestroy(g->stage_free[i]);
      if (g->stage_full[i]) cudaEventDestroy(g->stage_full[i]);
    }
  }
  delete g;
  return COADAPT_OK;
}

int coadapt_gns_reshape(coadapt_gns* g, int dp_size, int micro_count,
                        int64_t global_batch) {
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  if (dp_size < 1 || micro_count < 1 || (int64_t)dp_size * micro_count < 2 ||
      global_batch < 1)
    return fail(COADAPT_E_VALIDATION, "reshape: need d, M >= 1, d*M >= 2");
  GUARD(g->device);
  CU(cudaDeviceSynchronize());
  if (int rc = alloc_slots(g, dp_size * micro_count + 1)) return rc;
  g->dp = dp_size;
  g->M = micro_count;
  g->N = dp_size * micro_count;
  g->global_batch = global_batch;
  return COADAPT_OK;
}

int coadapt_gns_begin_step(coadapt_gns* g, void* stream) {
  COADAPT_NVTX("coadapt_gns_begin_step");
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  GUARD(g->device);
  CU(cudaMemsetAsync(g->slots, 0, sizeof(double) * (g->N + 1),
                     static_cast<cudaStream_t>(stream)));
  return COADAPT_OK;
}

int coadapt_gns_micro_sqnorm(coadapt_gns* g, const coadapt_plan* p,
                             const void* bucket, int dp_index, int micro,
                             void* stream) {
  const int32_t d = dp_index, m = micro;
  return coadapt_gns_micro_sqnorm_batched(g, p, &bucket, &d, &m, 1, stream);
}

int coadapt_gns_micro_sqnorm_batched(coadapt_gns* g, const coadapt_plan* p,
                                     const void* const* buckets,
                                     const int32_t* dp_index,
                                     const int32_t* micro, int count,
                                     void* stream) {
  COADAPT_NVTX("coadapt_gns_micro_sqnorm_batched");
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64 buckets: use coadapt_sqnorm_device");
  if (count < 0 || (count && (!buckets || !dp_index || !micro)))
    return fail(COADAPT_E_VALIDATION, "bad batch arguments");
  GUARD(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // 1..16 16-byte-aligned buckets into consecutive slots (one rank's micro-
  // batches): the TMA ring of the fused pass without its mean term
  if (count >= 1 && count <= coadapt::dev::kMaxFusedM) {
    bool contiguous = true;
    for (int j = 0; j < count && contiguous; ++j) {
      if (int rc = check_slot(g, dp_index[j], micro[j])) return rc;
      contiguous = dp_index[j] * g->M + micro[j] == dp_index[0] * g->M + micro[0] + j;
    }
    if (contiguous) {
      int rc = -1;
      if (try_tma_k1(g, p, buckets, count, dp_index[0] * g->M + micro[0], s, &rc)) return rc;
    }
  }
  for (int base = 0; base < count; base += coadapt::dev::kMaxBatch) {
    BatchArgs jobs;
    std::memset(&jobs, 0, sizeof(jobs));
    jobs.count = std::min(coadapt::dev::kMaxBatch, count - base);
    for (int j = 0; j < jobs.count; ++j) {
      if (int rc = check_slot(g, dp_index[base + j], micro[base + j])) return rc;
      if (int rc = check_bucket(p, buckets[base + j], "bucket")) return rc;
      jobs.ptr[j] = buckets[base + j];
      jobs.slot[j] = dp_index[base + j] * g->M + micro[base + j];
    }
    if (int rc = launch_batch(g, p, jobs, Window{0, p->active}, s)) return rc;
  }
  return COADAPT_OK;
}

namespace {
int fused_impl(coadapt_gns* g, const coadapt_plan* p, const void* const* buckets,
               int micro_count, void* stream, const coadapt::dev::Tail* tail);
int mean_impl(coadapt_gns* g, const coadapt_plan* p, const void* mean_grad,
              void* stream, const coadapt::dev::Tail* tail);
}  // namespace

int coadapt_gns_fused_sqnorm(coadapt_gns* g, const coadapt_plan* p,
                             const void* const* buckets, int micro_count,
                             void* stream) {
  COADAPT_NVTX("coadapt_gns_fused_sqnorm");
  return fused_impl(g, p, buckets, micro_count, stream, nullptr);
}

int coadapt_gns_fused_sqnorm_finalize(coadapt_gns* g, const coadapt_plan* p,
                                      const void* const* buckets,
                                      int micro_count, int64_t tokens,
                                      void* stream) {
  COADAPT_NVTX("coadapt_gns_fused_sqnorm_finalize");
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  coadapt::dev::Tail t;
  if (int rc = make_tail(g, tokens, &t)) return rc;
  if (int rc = fused_impl(g, p, buckets, micro_count, stream, &t)) return rc;
  GUARD(g->device);
  return finish_result(g, static_cast<cudaStream_t>(stream));
}

int coadapt_gns_mean_sqnorm(coadapt_gns* g, const coadapt_plan* p,
                            const void* mean_grad, void* stream) {
  COADAPT_NVTX("coadapt_gns_mean_sqnorm");
  return mean_impl(g, p, mean_grad, stream, nullptr);
}

int coadapt_gns_mean_sqnorm_finalize(coadapt_gns* g, const coadapt_plan* p,
                                     const void* mean_grad, int64_t tokens,
                                     void* stream) {
  COADAPT_NVTX("coadapt_gns_mean_sqnorm_finalize");
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  coadapt::dev::Tail t;
  if (int rc = make_tail(g, tokens, &t)) return rc;
  if (int rc = mean_impl(g, p, mean_grad, stream, &t)) return rc;
  GUARD(g->device);
  return finish_result(g, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

int fused_impl(coadapt_gns* g, const coadapt_plan* p, const void* const* buckets,
               int micro_count, void* stream, const coadapt::dev::Tail* tail) {
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (g->dp != 1)
    return fail(COADAPT_E_VALIDATION,
                "fused pass needs d == 1 (gbar is the local micro-batch "
                "mean); use micro_sqnorm + mean_sqnorm for d > 1");
  if (micro_count != g->M || micro_count < 1 ||
      micro_count > coadapt::dev::kMaxFusedM)
    return fail(COADAPT_E_VALIDATION,
                "fused pass needs micro_count == M <= 16");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64 buckets are not supported here");
  if (!buckets) return fail(COADAPT_E_VALIDATION, "buckets is NULL");
  FusedArgs fa;
  std::memset(&fa, 0, sizeof(fa));
  const uintptr_t mod0 = reinterpret_cast<uintptr_t>(buckets[0]) & 15;
  for (int m = 0; m < micro_count; ++m) {
    if (int rc = check_bucket(p, buckets[m], "bucket")) return rc;
    if ((reinterpret_cast<uintptr_t>(buckets[m]) & 15) != mod0)
      return fail(COADAPT_E_VALIDATION,
                  "fused buckets must share their address mod 16");
    fa.ptr[m] = buckets[m];
  }
  fa.slot0 = 0;
  fa.gslot = g->N;
  fa.gscale = 1.0 / ((double)micro_count * (double)micro_count);
  GUARD(g->device);
  // TMA bulk copies need 16-byte aligned sources; unaligned bucket views use
  // the LDG form of the same pass
  if (use_tma_path() && mod0 == 0)
    return launch_fused_tma_all(g, const_cast<coadapt_plan*>(p), fa,
                                micro_count, static_cast<cudaStream_t>(stream), tail);
  if (int rc = launch_fused_window(g, p, fa, micro_count, Window{0, p->active},
                                   static_cast<cudaStream_t>(stream)))
    return rc;
  return tail ? launch_tail_separately(*tail, static_cast<cudaStream_t>(stream))
              : COADAPT_OK;
}

int mean_impl(coadapt_gns* g, const coadapt_plan* p, const void* mean_grad,
              void* stream, const coadapt::dev::Tail* tail) {
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64: use coadapt_sqnorm_device");
  if (int rc = check_bucket(p, mean_grad, "mean_grad")) return rc;
  GUARD(g->device);
  {
    int rc = -1;
    if (try_tma_k1(g, p, &mean_grad, 1, g->N, static_cast<cudaStream_t>(stream), &rc,
                   tail))
      return rc;
  }
  BatchArgs jobs;
  std::memset(&jobs, 0, sizeof(jobs));
  jobs.count = 1;
  jobs.ptr[0] = mean_grad;
  jobs.slot[0] = g->N;
  if (int rc = launch_batch(g, p, jobs, Window{0, p->active},
                            static_cast<cudaStream_t>(stream)))
    return rc;
  return tail ? launch_tail_separately(*tail, static_cast<cudaStream_t>(stream))
              : COADAPT_OK;
}

}  // namespace

extern "C" {

int coadapt_gns_fused_sqnorm_host(coadapt_gns* g, const coadapt_plan* p,
                                  const void* const* host_buckets,
                                  int micro_count, void* stream) {
  COADAPT_NVTX("coadapt_gns_fused_sqnorm_host");
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (g->dp != 1 || micro_count != g->M || micro_count < 1 ||
      micro_count > coadapt::dev::kMaxFusedM)
    return fail(COADAPT_E_VALIDATION,
                "host fused pass needs d == 1 and micro_count == M <= 16");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64 buckets are not supported here");
  if (!host_buckets) return fail(COADAPT_E_VALIDATION, "host_buckets is NULL");
  for (int m = 0; m < micro_count; ++m)
    if (!host_buckets[m] && p->active)
      return fail(COADAPT_E_VALIDATION, "host bucket is NULL");
  GUARD(g->device);
  const int es = esize(p->dtype);
  const size_t stage_stride = kStageElems * es;  // per bucket per stage
  if (int rc = ensure_staging(g, es)) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the compute stream must be done with every stage before we overwrite it
  for (int i = 0; i < kStages; ++i) CU(cudaEventRecord(g->stage_free[i], s));
  const uint64_t numel = p->bucket_numel;
  // windows are whole multiples of the TMA chunk size P, so every window is
  // a contiguous run of the plan's chunk numbering
  const int P = coadapt::dev::tma_chunk_elems(p->dtype, micro_count);
  if (P <= 0) return fail(COADAPT_E_INTERNAL, "no TMA kernel for this dtype/M");
  const coadapt_plan::Chunks* ch = nullptr;
  if (int rc = plan_chunks(const_cast<coadapt_plan*>(p), P, &ch)) return rc;
  const uint64_t win = (kStageElems / P) * P;
  const uint64_t nwin = (numel + win - 1) / win;
  for (uint64_t c = 0; c < nwin; ++c) {
    const uint64_t w0 = c * win;
    const uint64_t w1 = std::min(numel, w0 + win);
    const uint64_t cb = chunks_before(p, ch, P, w0), ce = chunks_before(p, ch, P, w1);
    if (ce == cb) continue;  // window holds only weight-0 data
    const int st = (int)(c % kStages);
    char* stage = static_cast<char*>(g->staging) +
                  (size_t)st * coadapt::dev::kMaxFusedM * stage_stride;
    CU(cudaStreamWaitEvent(g->copy_stream, g->stage_free[st], 0));
    FusedArgs fa;
    std::memset(&fa, 0, sizeof(fa));
    for (int m = 0; m < micro_count; ++m) {
      char* dst = stage + (size_t)m * stage_stride;
      CU(cudaMemcpyAsync(dst,
                         static_cast<const char*>(host_buckets[m]) + w0 * es,
                         (w1 - w0) * es, cudaMemcpyHostToDevice,
                         g->copy_stream));
      // virtual base: abs element x of the window lives at dst + (x-w0)*es
      fa.ptr[m] = dst - w0 * es;
    }
    CU(cudaEventRecord(g->stage_full[st], g->copy_stream));
    CU(cudaStreamWaitEvent(s, g->stage_full[st], 0));
    fa.slot0 = 0;
    fa.gslot = g->N;
    fa.gscale = 1.0 / ((double)micro_count * (double)micro_count);
    const int grid = (int)std::min<uint64_t>(std::max(1, g->sms), ce - cb);
    if (int rc = ensure_partials(g, (size_t)grid * (micro_count + 1))) return rc;
    Sink sink{g->partials, g->ticket, g->slots};
    CU(coadapt::dev::launch_fused_tma(p->dtype, micro_count, p->ranges,
                                      (int)p->host.size(), ch->dev, cb, ce, fa,
                                      sink, grid, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CU(cudaEventRecord(g->stage_free[st], s));
  }
  return COADAPT_OK;
}

int coadapt_gns_micro_sqnorm_host(coadapt_gns* g, const coadapt_plan* p,
                                  const void* host_bucket, int dp_index,
                                  int micro, void* stream) {
  COADAPT_NVTX("coadapt_gns_micro_sqnorm_host");
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64 buckets are not supported here");
  if (int rc = check_slot(g, dp_index, micro)) return rc;
  if (!host_bucket && p->active)
    return fail(COADAPT_E_VALIDATION, "host bucket is NULL");
  GUARD(g->device);
  return stream_host_k1(g, p, host_bucket, dp_index * g->M + micro,
                        static_cast<cudaStream_t>(stream));
}

int coadapt_gns_mean_sqnorm_host(coadapt_gns* g, const coadapt_plan* p,
                                 const void* host_mean, void* stream) {
  COADAPT_NVTX("coadapt_gns_mean_sqnorm_host");
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64 buckets are not supported here");
  if (!host_mean && p->active)
    return fail(COADAPT_E_VALIDATION, "host mean gradient is NULL");
  GUARD(g->device);
  return stream_host_k1(g, p, host_mean, g->N, static_cast<cudaStream_t>(stream));
}

int coadapt_gns_accumulate(coadapt_gns* g, const coadapt_plan* p,
                           float* main_grad, const void* micro_grad,
                           int dp_index, int micro, int flags,
                           double mean_scale_sq, void* stream) {
  COADAPT_NVTX("coadapt_gns_accumulate");
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (p->is_slice)
    return fail(COADAPT_E_VALIDATION, "accumulate needs a whole-bucket plan");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64 gradients are not supported here");
  if (flags & ~(COADAPT_ACC_FIRST | COADAPT_ACC_LAST_MEAN))
    return fail(COADAPT_E_VALIDATION, "unknown accumulate flags");
  if ((flags & COADAPT_ACC_LAST_MEAN) && g->dp != 1)
    return fail(COADAPT_E_VALIDATION,
                "LAST_MEAN needs d == 1 (the local sum is the mean gradient); "
                "for d > 1 reduce the synchronised gradient with mean_sqnorm");
  if (!(mean_scale_sq >= 0.0) || !std::isfinite(mean_scale_sq))
    return fail(COADAPT_E_VALIDATION, "mean_scale_sq must be finite and >= 0");
  if (int rc = check_slot(g, dp_index, micro)) return rc;
  if (p->bucket_numel && (!main_grad || !micro_grad))
    return fail(COADAPT_E_VALIDATION, "main_grad/micro_grad is NULL");
  if ((reinterpret_cast<uintptr_t>(main_grad) & 15) ||
      (reinterpret_cast<uintptr_t>(micro_grad) & 15))
    return fail(COADAPT_E_VALIDATION,
                "main_grad and micro_grad must be 16-byte aligned");
  GUARD(g->device);
  coadapt_plan* pm = const_cast<coadapt_plan*>(p);
  if (int rc = plan_full(pm)) return rc;
  if (p->bucket_numel == 0) return COADAPT_OK;
  const int grid = grid_for(
      g->device, coadapt::dev::occupancy_accum(p->dtype, flags & COADAPT_ACC_FIRST),
      p->bucket_numel);
  if (int rc = ensure_partials(g, (size_t)grid * 2)) return rc;
  Sink sink{g->partials, g->ticket, g->slots};
  coadapt::dev::AccumArgs a{main_grad, micro_grad, flags,
                            dp_index * g->M + micro, g->N, mean_scale_sq};
  CU(coadapt::dev::launch_accum(p->dtype, p->full, (int)p->full_host.size(),
                                p->bucket_numel, a, sink, grid,
                                static_cast<cudaStream_t>(stream)));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

int coadapt_ipc_handle(const void* dev_ptr, void* out, size_t len,
                       uint64_t* offset) {
  if (!dev_ptr || !out || len < sizeof(cudaIpcMemHandle_t))
    return fail(COADAPT_E_VALIDATION, "ipc handle buffer must be >= 64 bytes");
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  std::memcpy(out, &h, sizeof(h));
  if (offset) {
    // the handle names the whole allocation (e.g. a caching-allocator
    // block): report where dev_ptr sits in it (driver cuMemGetAddressRange)
    using range_fn = int (*)(unsigned long long*, size_t*, unsigned long long);
    static range_fn fn = nullptr;
    if (!fn) {
      void* sym = nullptr;
      cudaDriverEntryPointQueryResult q;
      CU(cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &q));
      if (!sym) return fail(COADAPT_E_CUDA, "cuMemGetAddressRange unavailable");
      fn = reinterpret_cast<range_fn>(sym);
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0)
      return fail(COADAPT_E_CUDA, "cuMemGetAddressRange failed");
    *offset = reinterpret_cast<uint64_t>(dev_ptr) - base;
  }
  return COADAPT_OK;
}

int coadapt_ipc_open(const void* handle, size_t len, int device,
                     void** dev_ptr) {
  if (!handle || !dev_ptr || len < sizeof(cudaIpcMemHandle_t))
    return fail(COADAPT_E_VALIDATION, "bad ipc handle");
  GUARD(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CU(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return COADAPT_OK;
}

int coadapt_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return COADAPT_OK;
  CU(cudaIpcCloseMemHandle(dev_ptr));
  return COADAPT_OK;
}

int coadapt_gns_barrier(coadapt_gns* g, void* stream) {
  COADAPT_NVTX("coadapt_gns_barrier");
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  if (!g->comm || g->nranks == 1) return COADAPT_OK;
  GUARD(g->device);
  // a one-element all-reduce on the stream orders every rank's prior work
  // before everything enqueued after it (no host round trip)
  if (!g->barrier_buf) CU(cudaMalloc(&g->barrier_buf, sizeof(double)));
  NC(ncclAllReduce(g->barrier_buf, g->barrier_buf, 1, ncclFloat64, ncclSum,
                   g->comm, static_cast<cudaStream_t>(stream)));
  return COADAPT_OK;
}

static int rs_common(coadapt_gns* g, const coadapt_plan* p,
                     const void* const* replicas, int d, int dp_rank,
                     void* out_slice, bool inplace, double scale, void* stream,
                     const void* multicast = nullptr) {
  if (!g || !p) return fail(COADAPT_E_VALIDATION, "gns/plan is NULL");
  if (p->device != g->device)
    return fail(COADAPT_E_VALIDATION, "plan and gns live on different devices");
  if (p->is_slice)
    return fail(COADAPT_E_VALIDATION, "reduce-scatter needs a whole-bucket plan");
  if (p->dtype == COADAPT_FP64)
    return fail(COADAPT_E_VALIDATION, "fp64 buckets are not supported here");
  if (d < 1 || d > coadapt::dev::kMaxReplicas || dp_rank < 0 || dp_rank >= d)
    return fail(COADAPT_E_VALIDATION, "need 1 <= d <= 8 and 0 <= dp_rank < d");
  if ((!replicas && !multicast) || (p->bucket_numel && !inplace && !out_slice))
    return fail(COADAPT_E_VALIDATION, "replicas/out_slice is NULL");
  if (!(scale == scale) || std::isinf(scale))
    return fail(COADAPT_E_VALIDATION, "scale must be finite");
  coadapt::dev::RSArgs a;
  std::memset(&a, 0, sizeof(a));
  if (multicast) {
    if (p->dtype != COADAPT_FP32)
      return fail(COADAPT_E_VALIDATION,
                  "NVLS reduction is fp32 only (the switch's bf16/fp16 rounding biases gbar^2)");
    if (reinterpret_cast<uintptr_t>(multicast) & 15)
      return fail(COADAPT_E_VALIDATION, "multicast address must be 16-byte aligned");
    a.mc = multicast;
    a.nvls = 1;
  } else {
    for (int q = 0; q < d; ++q) {
      if (!replicas[q] && p->bucket_numel)
        return fail(COADAPT_E_VALIDATION, "replica pointer is NULL");
      if (reinterpret_cast<uintptr_t>(replicas[q]) & 15)
        return fail(COADAPT_E_VALIDATION, "replica buffers must be 16-byte aligned");
      a.rep[q] = replicas[q];
    }
  }
  if (reinterpret_cast<uintptr_t>(out_slice) & 15)
    return fail(COADAPT_E_VALIDATION, "out_slice must be 16-byte aligned");
  // the same cut as coadapt_plan_create_slice
  const uint64_t n = p->bucket_numel;
  auto cut = [&](int i) -> uint64_t {
    if (i >= d) return n;
    return (uint64_t)((unsigned __int128)n * i / d) & ~uint64_t(63);
  };
  const uint64_t lo = cut(dp_rank), hi = cut(dp_rank + 1);
  a.d = d;
  a.scale = (float)scale;
  a.out = inplace ? nullptr : out_slice;
  a.inplace = inplace ? 1 : 0;
  a.gslot = g->N;
  GUARD(g->device);
  coadapt_plan* pm = const_cast<coadapt_plan*>(p);
  if (int rc = plan_full(pm)) return rc;
  if (hi <= lo) return COADAPT_OK;
  const int grid =
      grid_for(g->device, coadapt::dev::occupancy_rs(p->dtype), hi - lo);
  if (int rc = ensure_partials(g, (size_t)grid)) return rc;
  Sink sink{g->partials, g->ticket, g->slots};
  CU(coadapt::dev::launch_rs(p->dtype, p->full, (int)p->full_host.size(), lo,
                             hi, a, sink, grid,
                             static_cast<cudaStream_t>(stream)));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

int coadapt_gns_reduce_scatter_sqnorm(coadapt_gns* g, const coadapt_plan* p,
                                      const void* const* replicas, int d,
                                      int dp_rank, void* out_slice,
                                      double scale, void* stream) {
  COADAPT_NVTX("coadapt_gns_reduce_scatter_sqnorm");
  return rs_common(g, p, replicas, d, dp_rank, out_slice, false, scale, stream);
}

int coadapt_gns_allreduce_sqnorm(coadapt_gns* g, const coadapt_plan* p,
                                 void* const* replicas, int d, int dp_rank,
                                 double scale, void* stream) {
  COADAPT_NVTX("coadapt_gns_allreduce_sqnorm");
  return rs_common(g, p, const_cast<const void* const*>(replicas), d, dp_rank,
                   nullptr, true, scale, stream);
}

int coadapt_gns_nvls_reduce_sqnorm(coadapt_gns* g, const coadapt_plan* p,
                                   const void* multicast, int d, int dp_rank,
                                   void* out_slice, double scale, void* stream) {
  COADAPT_NVTX("coadapt_gns_nvls_reduce_sqnorm");
  if (!multicast) return fail(COADAPT_E_VALIDATION, "multicast address is NULL");
  return rs_common(g, p, nullptr, d, dp_rank, out_slice, out_slice == nullptr, scale,
                   stream, multicast);
}

int coadapt_nccl_unique_id(void* out, size_t len) {
  if (!out || len < sizeof(ncclUniqueId))
    return fail(COADAPT_E_VALIDATION, "unique id buffer must be >= 128 bytes");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return COADAPT_OK;
}

int coadapt_gns_attach_nccl(coadapt_gns* g, int nranks, int rank,
                            const void* unique_id, size_t len) {
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  if (!unique_id || len < sizeof(ncclUniqueId))
    return fail(COADAPT_E_VALIDATION, "unique id must be >= 128 bytes");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(COADAPT_E_VALIDATION, "bad nranks/rank");
  GUARD(g->device);
  if (g->comm) {
    ncclCommDestroy(g->comm);
    g->comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  NC(ncclCommInitRank(&g->comm, nranks, id, rank));
  g->nranks = nranks;
  g->rank = rank;
  return COADAPT_OK;
}

int coadapt_gns_attach_nccl_all(coadapt_gns* const* gs, int n) {
  if (!gs || n < 1) return fail(COADAPT_E_VALIDATION, "need n >= 1 gns handles");
  std::vector<int> devs(n);
  for (int i = 0; i < n; ++i) {
    if (!gs[i]) return fail(COADAPT_E_VALIDATION, "gns handle is NULL");
    devs[i] = gs[i]->device;
    for (int j = 0; j < i; ++j)
      if (devs[j] == devs[i])
        return fail(COADAPT_E_VALIDATION, "one gns per device");
  }
  std::vector<ncclComm_t> comms(n, nullptr);
  NC(ncclCommInitAll(comms.data(), n, devs.data()));
  for (int i = 0; i < n; ++i) {
    if (gs[i]->comm) ncclCommDestroy(gs[i]->comm);
    gs[i]->comm = comms[i];
    gs[i]->nranks = n;
    gs[i]->rank = i;
  }
  return COADAPT_OK;
}

int coadapt_gns_allreduce_group(coadapt_gns* const* gs, void* const* streams,
                                int n) {
  COADAPT_NVTX("coadapt_gns_allreduce_group");
  if (!gs || !streams || n < 1)
    return fail(COADAPT_E_VALIDATION, "need n >= 1 gns handles and streams");
  for (int i = 0; i < n; ++i) {
    if (!gs[i]) return fail(COADAPT_E_VALIDATION, "gns handle is NULL");
    if (gs[i]->N != gs[0]->N)
      return fail(COADAPT_E_VALIDATION, "all ranks need the same d*M");
  }
  if (n == 1 || !gs[0]->comm) return COADAPT_OK;
  NC(ncclGroupStart());
  for (int i = 0; i < n; ++i) {
    const ncclResult_t r =
        ncclAllReduce(gs[i]->slots, gs[i]->slots, (size_t)gs[i]->N + 1,
                      ncclFloat64, ncclSum, gs[i]->comm,
                      static_cast<cudaStream_t>(streams[i]));
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return fail(COADAPT_E_NCCL, std::string("ncclAllReduce: ") +
                                      ncclGetErrorString(r));
    }
  }
  NC(ncclGroupEnd());
  return COADAPT_OK;
}

int coadapt_gns_allreduce(coadapt_gns* g, void* stream) {
  COADAPT_NVTX("coadapt_gns_allreduce");
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  if (!g->comm || g->nranks == 1) return COADAPT_OK;  // local sum only
  GUARD(g->device);
  NC(ncclAllReduce(g->slots, g->slots, (size_t)g->N + 1, ncclFloat64, ncclSum,
                   g->comm, static_cast<cudaStream_t>(stream)));
  return COADAPT_OK;
}

int coadapt_gns_mailbox(coadapt_gns* g, int nranks, void** out) {
  if (!g || !out) return fail(COADAPT_E_VALIDATION, "gns/out is NULL");
  if (nranks < 1 || nranks > coadapt::dev::kMaxPeers)
    return fail(COADAPT_E_VALIDATION, "mailbox: 1 <= nranks <= 8");
  GUARD(g->device);
  const int cap = std::max(g->slot_cap, g->N + 1);
  if (!g->mbox || g->mbox_world != nranks || g->mbox_cap < cap) {
    if (g->mbox) {
      CU(cudaDeviceSynchronize());
      cudaFree(g->mbox);
      g->mbox = nullptr;
    }
    const size_t bytes = coadapt::dev::mailbox_bytes(nranks, cap);
    CU(cudaMalloc(&g->mbox, bytes));
    CU(cudaMemset(g->mbox, 0, bytes));
    g->mbox_world = nranks;
    g->mbox_cap = cap;
    g->mbox_rank = -1;  // (the zeroed mailbox restarts the epoch counter)
  }
  *out = g->mbox;
  return COADAPT_OK;
}

int coadapt_gns_attach_mailboxes(coadapt_gns* g, int nranks, int rank,
                                 const void* const* peers) {
  if (!g || !peers) return fail(COADAPT_E_VALIDATION, "gns/peers is NULL");
  if (!g->mbox || nranks != g->mbox_world)
    return fail(COADAPT_E_VALIDATION,
                "call coadapt_gns_mailbox(g, nranks) first, with the same nranks");
  if (rank < 0 || rank >= nranks)
    return fail(COADAPT_E_VALIDATION, "rank out of range");
  for (int q = 0; q < nranks; ++q) {
    if (!peers[q]) return fail(COADAPT_E_VALIDATION, "peer mailbox is NULL");
    g->mbox_peers[q] = static_cast<char*>(const_cast<void*>(peers[q]));
  }
  if (g->mbox_peers[rank] != g->mbox)
    return fail(COADAPT_E_VALIDATION, "peers[rank] must be this gns's own mailbox");
  g->mbox_rank = rank;
  return COADAPT_OK;
}

int coadapt_gns_allreduce_finalize_p2p(coadapt_gns* g, int64_t tokens,
                                       void* stream) {
  COADAPT_NVTX("coadapt_gns_allreduce_finalize_p2p");
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  if (tokens < 0) return fail(COADAPT_E_VALIDATION, "tokens must be >= 0");
  if (g->mbox_rank < 0)
    return fail(COADAPT_E_VALIDATION, "no mailboxes attached");
  if (g->N + 1 > g->mbox_cap)
    return fail(COADAPT_E_VALIDATION,
                "d*M grew past the mailbox capacity: recreate the mailboxes");
  GUARD(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  coadapt::dev::P2PArgs a;
  std::memset(&a, 0, sizeof(a));
  a.fin = coadapt::dev::FinalizeArgs{g->slots, g->N, g->global_batch, tokens,
                                     g->state, g->result};
  a.slots = g->slots;
  a.world = g->mbox_world;
  a.rank = g->mbox_rank;
  a.cap = g->mbox_cap;
  a.timeout_ns = 10'000'000'000ll;  // a peer 10 s late is a failure, not a hang
  for (int q = 0; q < a.world; ++q) a.mbox[q] = g->mbox_peers[q];
  CU(coadapt::dev::launch_p2p_finalize(a, s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return finish_result(g, s);
}

int coadapt_gns_finalize(coadapt_gns* g, int64_t tokens, void* stream) {
  COADAPT_NVTX("coadapt_gns_finalize");
  if (!g) return fail(COADAPT_E_VALIDATION, "gns is NULL");
  if (tokens < 0) return fail(COADAPT_E_VALIDATION, "tokens must be >= 0");
  GUARD(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  coadapt::dev::FinalizeArgs a{g->slots, g->N, g->global_batch, tokens,
                               g->state, g->result};
  CU(coadapt::dev::launch_finalize(a, s));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return finish_result(g, s);
}

int coadapt_gns_read_result(coadapt_gns* g, coadapt_gns_result* out) {
  if (!g || !out) return fail(COADAPT_E_VALIDATION, "gns/out is NULL");
  if (!g->finalized)
    return fail(COADAPT_E_VALIDATION, "no finalized step to read");
  GUARD(g->device);
  CU(cudaEventSynchronize(g->result_ready));
  *out = *g->result_host;
  if (out->status == COADAPT_E_INTERNAL)
    return fail(COADAPT_E_INTERNAL,
                "NVLink slot exchange timed out waiting for a peer "
                "(coadapt_gns_allreduce_finalize_p2p); GnsState left unchanged");
  if (out->status != COADAPT_OK)
    return fail(COADAPT_E_VALIDATION,
                "a squared-norm partial was negative or non-finite "
                "(gns.hpp:19); GnsState left unchanged");
  return COADAPT_OK;
}

int coadapt_gns_result_ready(coadapt_gns* g, int* ready) {
  if (!g || !ready) return fail(COADAPT_E_VALIDATION, "gns/ready is NULL");
  if (!g->finalized)
    return fail(COADAPT_E_VALIDATION, "no finalized step to query");
  GUARD(g->device);
  const cudaError_t e = cudaEventQuery(g->result_ready);
  if (e == cudaErrorNotReady) {
    *ready = 0;
    return COADAPT_OK;
  }
  CU(e);
  *ready = 1;
  return COADAPT_OK;
}

int coadapt_gns_read_partials(coadapt_gns* g, double* out, size_t n) {
  if (!g || !out) return fail(COADAPT_E_VALIDATION, "gns/out is NULL");
  if (n < (size_t)g->N + 1)
    return fail(COADAPT_E_VALIDATION, "need N+1 doubles");
  GUARD(g->device);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(out, g->slots, sizeof(double) * (g->N + 1),
                cudaMemcpyDeviceToHost));
  return COADAPT_OK;
}

int coadapt_gns_get_state(coadapt_gns* g, coadapt_gns_state* out) {
  if (!g || !out) return fail(COADAPT_E_VALIDATION, "gns/out is NULL");
  GUARD(g->device);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(out, g->state, sizeof(*out), cudaMemcpyDeviceToHost));
  return COADAPT_OK;
}

int coadapt_gns_set_state(coadapt_gns* g, const coadapt_gns_state* in) {
  if (!g || !in) return fail(COADAPT_E_VALIDATION, "gns/in is NULL");
  if (!(in->alpha_early > 0.0 && in->alpha_early <= in->alpha_late &&
        in->alpha_late < 1.0))
    return fail(COADAPT_E_VALIDATION,
                "need 0 < alpha_early <= alpha_late < 1 (SPEC.md:160)");
  GUARD(g->device);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(g->state, in, sizeof(*in), cudaMemcpyHostToDevice));
  return COADAPT_OK;
}

int coadapt_sqnorm_device(const void* v, uint64_t n, int dtype, int device,
                          double* out, void* stream) {
  COADAPT_NVTX("coadapt_sqnorm_device");
  if (!out) return fail(COADAPT_E_VALIDATION, "out is NULL");
  if (int rc = validate_dtype(dtype, true)) return rc;
  std::lock_guard<std::mutex> lock(g_oneshot_mu);
  GUARD(device);
  coadapt_segment seg{0, n, 1.0};
  coadapt_plan* p = nullptr;
  if (int rc = plan_make(&seg, 1, n, dtype, device, 0, n, &p)) return rc;
  int rc = check_bucket(p, v, "vector");
  coadapt_gns g;  // a throwaway accumulator: one slot
  g.device = device;
  g.sms = sm_count(device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!rc) rc = alloc_slots(&g, 1);
  if (!rc && cudaMalloc(&g.ticket, sizeof(unsigned int)) != cudaSuccess)
    rc = fail(COADAPT_E_CUDA, "ticket alloc");
  if (!rc && cudaMemsetAsync(g.ticket, 0, sizeof(unsigned int), s) != cudaSuccess)
    rc = fail(COADAPT_E_CUDA, "ticket init");
  if (!rc && cudaMemsetAsync(g.slots, 0, sizeof(double), s) != cudaSuccess)
    rc = fail(COADAPT_E_CUDA, "slot init");
  if (!rc) {
    BatchArgs jobs;
    std::memset(&jobs, 0, sizeof(jobs));
    jobs.count = 1;
    jobs.ptr[0] = v;
    jobs.slot[0] = 0;
    rc = launch_batch(&g, p, jobs, Window{0, p->active}, s);
  }
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(out, g.slots, sizeof(double),
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
      rc = fail(COADAPT_E_CUDA, std::string("sqnorm: ") + cudaGetErrorString(e));
  }
  if (g.slots) cudaFree(g.slots);
  if (g.partials) cudaFree(g.partials);
  if (g.ticket) cudaFree(g.ticket);
  g.slots = nullptr;
  g.partials = nullptr;
  g.ticket = nullptr;
  coadapt_plan_destroy(p);
  return rc;
}

int coadapt_sqnorm_host(const void* v, uint64_t n, int dtype, int device,
                        double* out) {
  COADAPT_NVTX("coadapt_sqnorm_host");
  if (!out) return fail(COADAPT_E_VALIDATION, "out is NULL");
  if (int rc = validate_dtype(dtype, true)) return rc;
  if (n == 0) {
    *out = 0.0;
    return COADAPT_OK;
  }
  if (!v) return fail(COADAPT_E_VALIDATION, "vector is NULL");
  GUARD(device);
  // bounded device footprint whatever n is (the span overload's host vector
  // may be larger than HBM): fixed 32 Mi-element chunks,
  // chunk sums added in chunk order on the host in fp64.  The staging
  // buffer is kept per device between calls (grown, never shrunk), so a
  // small span costs one copy and one launch, not an allocation.
  const int es = esize(dtype);
  const uint64_t chunk = std::min<uint64_t>(n, 32ull << 20);
  static std::mutex scratch_mu;
  static std::vector<std::pair<void*, size_t>> scratch;  // per device
  std::lock_guard<std::mutex> lock(scratch_mu);
  if ((int)scratch.size() <= device) scratch.resize(device + 1, {nullptr, 0});
  auto& slot = scratch[device];
  if (slot.second < (size_t)chunk * es) {
    if (slot.first) cudaFree(slot.first);
    slot = {nullptr, 0};
    CU(cudaMalloc(&slot.first, (size_t)chunk * es));
    slot.second = (size_t)chunk * es;
  }
  void* d = slot.first;
  double total = 0.0;
  int rc = COADAPT_OK;
  for (uint64_t b = 0; b < n && rc == COADAPT_OK; b += chunk) {
    const uint64_t k = std::min(chunk, n - b);
    const cudaError_t e = cudaMemcpy(d, static_cast<const char*>(v) + b * es,
                                     (size_t)k * es, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      rc = fail(COADAPT_E_CUDA,
                std::string("sqnorm_host copy: ") + cudaGetErrorString(e));
      break;
    }
    double part = 0.0;
    rc = coadapt_sqnorm_device(d, k, dtype, device, &part, nullptr);
    total += part;
  }
  if (rc == COADAPT_OK) *out = total;
  return rc;
}

int coadapt_synth_fill(void* dst, int dtype, const coadapt_gen_segment* segs,
                       size_t nseg, uint64_t seed, uint64_t sample, float g0,
                       float unit, void* stream) {
  if (int rc = validate_dtype(dtype, true)) return rc;
  if (nseg && (!segs || !dst)) return fail(COADAPT_E_VALIDATION, "NULL argument");
  for (size_t i = 0; i < nseg; ++i) {
    if (segs[i].row_len == 0 && segs[i].numel)
      return fail(COADAPT_E_VALIDATION, "gen segment row_len is 0");
    coadapt::dev::GenSeg gs{segs[i].local_off, segs[i].numel,
                            segs[i].global_base, segs[i].row_len,
                            segs[i].row_stride};
    CU(coadapt::dev::launch_synth(dst, dtype, gs, seed, sample, g0, unit,
                                  static_cast<cudaStream_t>(stream)));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return COADAPT_OK;
}

int coadapt_synth_mean_fill(void* dst, int dtype,
                            const coadapt_gen_segment* segs, size_t nseg,
                            uint64_t seed, uint64_t sample0, int64_t nsamples,
                            float g0, float unit, void* stream) {
  if (int rc = validate_dtype(dtype, true)) return rc;
  if (nsamples < 1) return fail(COADAPT_E_VALIDATION, "nsamples must be >= 1");
  if (nseg && (!segs || !dst)) return fail(COADAPT_E_VALIDATION, "NULL argument");
  for (size_t i = 0; i < nseg; ++i) {
    if (segs[i].row_len == 0 && segs[i].numel)
      return fail(COADAPT_E_VALIDATION, "gen segment row_len is 0");
    coadapt::dev::GenSeg gs{segs[i].local_off, segs[i].numel,
                            segs[i].global_base, segs[i].row_len,
                            segs[i].row_stride};
    CU(coadapt::dev::launch_synth_mean(dst, dtype, gs, seed, sample0, nsamples,
                                       g0, unit,
                                       static_cast<cudaStream_t>(stream)));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return COADAPT_OK;
}

int coadapt_l2_flush(void* scratch, uint64_t bytes, void* stream) {
  if (!scratch) return fail(COADAPT_E_VALIDATION, "scratch is NULL");
  CU(coadapt::dev::launch_l2_flush(scratch, bytes,
                                   static_cast<cudaStream_t>(stream)));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

int coadapt_read_probe(const void* buf, uint64_t bytes, double* sink,
                       void* stream) {
  if (!buf || !sink) return fail(COADAPT_E_VALIDATION, "NULL argument");
  if (reinterpret_cast<uintptr_t>(buf) & 15)
    return fail(COADAPT_E_VALIDATION, "probe buffer must be 16B aligned");
  CU(coadapt::dev::launch_read_probe(buf, bytes, sink,
                                     static_cast<cudaStream_t>(stream)));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return COADAPT_OK;
}

}  // extern "C"
