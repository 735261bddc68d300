// reshard.cu — C-ABI of the Reconfigure path (include/coadapt_reshard.h) and
// its device executor (§8 f4).
//
// Planning is coadapt::reshard (host/reshard.cpp).  Execution replaces the
// paper's host-staged pipeline with a
// pull: the destination GPU's SMs read each region straight from the source
// rank's pack — its own HBM for local moves, a peer's HBM over NVLink for the
// rest — and write it into the destination pack.  No staging buffer, no
// host round trip, one launch per state plane.
//
// Copy tasks.  A move is a box of the global tensor; in both packs the shard
// is row-major, so the box is `rows` runs of `row_bytes` contiguous bytes at
// fixed pitches.  Trailing axes that the box spans completely on both sides
// fold into the run; axes outside the last two are enumerated on the host.
// Runs are cut into tasks of <= 1 MiB so 148 SMs share the work evenly.
// Each CTA copies whole tasks with the widest access (16/8/4/2/1 B) that the
// two addresses, run length and pitches allow; 16-byte copies keep 4
// loads in flight per thread before storing (enough bytes in flight to
// cover NVLink latency with a full wave of CTAs).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/coadapt_cuda.h"
#include "internal.h"
#include "../../include/coadapt_reshard.h"
#include "coadapt/errors.hpp"
#include "coadapt/reshard.hpp"

namespace coadapt_capi {
void set_error(const char* msg);
void count_launch();
}  // namespace coadapt_capi

namespace {

namespace R = coadapt::reshard;

constexpr int kMaxRanks = 64;
// Tuned on 2 x B200 (tools/reshard_sweep.sh, TP->PP of 537 MB per rank):
// grid {4,8,16} x SMs, {4,8} 16-byte loads in flight, {256 KiB, 1 MiB}
// tasks all land at 600-670 GB/s of wire bytes — the NVLink bound; 1 MiB
// tasks, 4 loads in flight, 4 CTAs per SM is the balanced choice.
constexpr uint64_t kTaskBytes = 1u << 20;
constexpr int kGridPerSM = 4;
constexpr int kLoadsInFlight = 4;

struct CopyTask {
  uint64_t src_off, dst_off;      // bytes into the packs
  uint64_t src_pitch, dst_pitch;  // bytes between rows
  uint32_t row_bytes, rows;
  int32_t src_rank, dst_rank;
};

struct ExecArgs {
  const CopyTask* tasks;
  uint32_t n_tasks;
  const char* src[kMaxRanks];
  char* dst[kMaxRanks];
};

template <class T, int U16>
__device__ __forceinline__ void copy_rows(const char* __restrict__ s,
                                          char* __restrict__ d,
                                          const CopyTask& t) {
  const uint32_t per_row = t.row_bytes / sizeof(T);
  const uint32_t total = per_row * t.rows;
  constexpr int U = sizeof(T) == 16 ? U16 : 2;
  for (uint32_t base = threadIdx.x; base < total; base += U * blockDim.x) {
    T v[U];
    uint32_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      idx[u] = base + u * blockDim.x;
      if (idx[u] < total) {
        const uint32_t r = idx[u] / per_row, c = idx[u] - r * per_row;
        v[u] = *reinterpret_cast<const T*>(s + r * t.src_pitch + c * sizeof(T));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (idx[u] < total) {
        const uint32_t r = idx[u] / per_row, c = idx[u] - r * per_row;
        *reinterpret_cast<T*>(d + r * t.dst_pitch + c * sizeof(T)) = v[u];
      }
  }
}

template <int U16>
__global__ void __launch_bounds__(256)
reshard_copy_kernel(const __grid_constant__ ExecArgs a) {
  for (uint32_t i = blockIdx.x; i < a.n_tasks; i += gridDim.x) {
    const CopyTask t = a.tasks[i];
    const char* s = a.src[t.src_rank] + t.src_off;
    char* d = a.dst[t.dst_rank] + t.dst_off;
    const uint64_t bits = reinterpret_cast<uintptr_t>(s) |
                          reinterpret_cast<uintptr_t>(d) | t.row_bytes |
                          (t.rows > 1 ? (t.src_pitch | t.dst_pitch) : 0);
    if ((bits & 15) == 0)
      copy_rows<uint4, U16>(s, d, t);
    else if ((bits & 7) == 0)
      copy_rows<uint2, U16>(s, d, t);
    else if ((bits & 3) == 0)
      copy_rows<uint32_t, U16>(s, d, t);
    else if ((bits & 1) == 0)
      copy_rows<uint16_t, U16>(s, d, t);
    else
      copy_rows<uint8_t, U16>(s, d, t);
  }
}

int fail(int code, const std::string& msg) {
  coadapt_capi::set_error(msg.c_str());
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const coadapt::ValidationError& e) {
    return fail(COADAPT_E_VALIDATION, e.what());
  } catch (const coadapt::InternalError& e) {
    return fail(COADAPT_E_INTERNAL, e.what());
  } catch (const std::exception& e) {
    return fail(COADAPT_E_INTERNAL, e.what());
  }
}

#define CU(call)                                                        \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess)                                              \
      return fail(COADAPT_E_CUDA, std::string(#call) + ": " +           \
                                      cudaGetErrorString(e_));          \
  } while (0)

// Row-major element strides of a shard's local box.
std::vector<uint64_t> strides_of(const std::vector<int64_t>& shape) {
  std::vector<uint64_t> st(shape.size(), 1);
  for (int i = (int)shape.size() - 2; i >= 0; --i)
    st[i] = st[i + 1] * (uint64_t)shape[i + 1];
  return st;
}

void emit_tasks(const R::Move& mv, const R::ShardDescriptor& S,
                const R::ShardDescriptor& D, int eb, std::vector<CopyTask>& out) {
  const int nd = (int)mv.extent.size();
  const auto ss = strides_of(S.local_shape), ds = strides_of(D.local_shape);
  // fold trailing axes spanned completely on both sides into the run
  int j = nd - 1;
  uint64_t run = (uint64_t)mv.extent[j];
  while (j > 0 && mv.extent[j] == S.local_shape[j] &&
         mv.extent[j] == D.local_shape[j]) {
    --j;
    run *= (uint64_t)mv.extent[j];
  }
  // axis j is folded into `run`; axis j-1 (if any) is the row axis
  const int row_axis = j - 1;
  const uint64_t rows = row_axis >= 0 ? (uint64_t)mv.extent[row_axis] : 1;
  const uint64_t row_bytes = run * eb;
  const uint64_t sp = row_axis >= 0 ? ss[row_axis] * eb : 0;
  const uint64_t dp = row_axis >= 0 ? ds[row_axis] * eb : 0;
  // enumerate the outer axes [0, row_axis)
  const int outer = std::max(0, row_axis);
  std::vector<int64_t> idx(outer, 0);
  for (;;) {
    uint64_t so = S.pack_offset, dof = D.pack_offset;
    for (int i = 0; i < nd; ++i) {
      const int64_t g = mv.offset[i] + (i < outer ? idx[i] : 0);
      so += (uint64_t)(g - S.global_offset[i]) * ss[i];
      dof += (uint64_t)(g - D.global_offset[i]) * ds[i];
    }
    so *= eb;
    dof *= eb;
    if (row_bytes >= kTaskBytes) {  // long runs: split each row
      for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t b = 0; b < row_bytes; b += kTaskBytes)
          out.push_back(CopyTask{so + r * sp + b, dof + r * dp + b, 0, 0,
                                 (uint32_t)std::min(kTaskBytes, row_bytes - b),
                                 1, mv.src_rank, mv.dst_rank});
    } else {  // short runs: group rows
      const uint64_t per = std::max<uint64_t>(1, kTaskBytes / row_bytes);
      for (uint64_t r = 0; r < rows; r += per)
        out.push_back(CopyTask{so + r * sp, dof + r * dp, sp, dp,
                               (uint32_t)row_bytes,
                               (uint32_t)std::min(per, rows - r), mv.src_rank,
                               mv.dst_rank});
    }
    int k = outer - 1;
    while (k >= 0 && ++idx[k] == mv.extent[k]) idx[k--] = 0;
    if (k < 0) break;
  }
}

void to_c_shard(const R::ShardDescriptor& s, coadapt_shard& o) {
  std::memset(&o, 0, sizeof(o));
  o.layer = s.layer;
  o.tensor = s.tensor;
  o.owner = s.owner;
  o.canonical = s.canonical ? 1 : 0;
  o.ndim = (int32_t)s.global_shape.size();
  for (int i = 0; i < o.ndim; ++i) {
    o.global_shape[i] = s.global_shape[i];
    o.global_offset[i] = s.global_offset[i];
    o.local_shape[i] = s.local_shape[i];
  }
  o.pack_offset = s.pack_offset;
}

}  // namespace

struct coadapt_reshard_plan {
  R::ModelSpec model;
  R::ShardLayout src, dst;
  R::TransferPlan plan;
  struct Tasks {
    int device = -1;
    CopyTask* dev = nullptr;
    uint32_t n = 0;
  };
  std::map<std::tuple<int, int, int>, Tasks> cache;  // (role, rank, elem_bytes)
};

extern "C" {

int coadapt_reshard_plan_create(const coadapt_reshard_model* m,
                                const int32_t src_dtp[3],
                                const int32_t dst_dtp[3], int policy,
                                coadapt_reshard_plan** out) {
  if (!m || !src_dtp || !dst_dtp || !out)
    return fail(COADAPT_E_VALIDATION, "reshard: NULL argument");
  if (m->n_tensors < 0 || (m->n_tensors && !m->tensors))
    return fail(COADAPT_E_VALIDATION, "reshard: tensors is NULL");
  if (policy != COADAPT_RESHARD_CANONICAL && policy != COADAPT_RESHARD_SPREAD)
    return fail(COADAPT_E_VALIDATION, "reshard: unknown source policy");
  *out = nullptr;
  return guarded([&] {
    auto p = std::make_unique<coadapt_reshard_plan>();
    p->model.layers = m->layers;
    p->model.optimizer_state_multiplier = m->optimizer_state_multiplier;
    p->model.param_bytes = m->param_bytes;
    p->model.state_bytes = m->state_bytes;
    for (int i = 0; i < m->n_tensors; ++i) {
      const auto& t = m->tensors[i];
      if (t.ndim < 1 || t.ndim > COADAPT_RESHARD_MAX_DIMS)
        throw coadapt::ValidationError("reshard: tensor ndim must be 1..4");
      R::TensorDecl d;
      d.name = t.name ? t.name : ("t" + std::to_string(i));
      d.shape.assign(t.shape, t.shape + t.ndim);
      d.tp_axis = t.tp_axis;
      p->model.per_layer.push_back(std::move(d));
    }
    const coadapt::ParallelStrategy s{src_dtp[0], src_dtp[1], src_dtp[2]};
    const coadapt::ParallelStrategy t{dst_dtp[0], dst_dtp[1], dst_dtp[2]};
    if (s.d < 1 || s.t < 1 || s.p < 1 || t.d < 1 || t.t < 1 || t.p < 1)
      throw coadapt::ValidationError("reshard: degrees must be >= 1");
    if (s.gpus() > kMaxRanks || t.gpus() > kMaxRanks)
      throw coadapt::ValidationError("reshard: at most 64 ranks");
    p->src = R::layout_for(p->model, s, s.gpus());
    p->dst = R::layout_for(p->model, t, t.gpus());
    p->plan = R::plan_transfers(p->model, p->src, p->dst,
                                static_cast<R::SourcePolicy>(policy));
    *out = p.release();
    return COADAPT_OK;
  });
}

int coadapt_reshard_plan_destroy(coadapt_reshard_plan* p) {
  if (!p) return COADAPT_OK;
  for (auto& [k, t] : p->cache)
    if (t.dev) {
      int prev = -1;
      cudaGetDevice(&prev);
      cudaSetDevice(t.device);
      cudaFree(t.dev);
      if (prev >= 0) cudaSetDevice(prev);
    }
  delete p;
  return COADAPT_OK;
}

int coadapt_reshard_plan_info(const coadapt_reshard_plan* p,
                              coadapt_reshard_info* out) {
  if (!p || !out) return fail(COADAPT_E_VALIDATION, "reshard: NULL argument");
  std::memset(out, 0, sizeof(*out));
  out->n_moves = p->plan.moves.size();
  out->total_bytes = p->plan.total_bytes;
  out->max_bytes_per_rank = p->plan.max_bytes_per_rank;
  out->local_bytes = p->plan.local_bytes;
  out->src_ranks = p->src.strategy.gpus();
  out->dst_ranks = p->dst.strategy.gpus();
  out->src_max_pack_numel = p->src.max_pack_numel();
  out->dst_max_pack_numel = p->dst.max_pack_numel();
  return COADAPT_OK;
}

int coadapt_reshard_moves(const coadapt_reshard_plan* p, coadapt_move* out,
                          size_t* count) {
  if (!p || !count) return fail(COADAPT_E_VALIDATION, "reshard: NULL argument");
  const size_t n = p->plan.moves.size(), cap = *count;
  *count = n;
  if (cap < n) return out || cap ? fail(COADAPT_E_VALIDATION,
                                        "reshard: move buffer too small")
                                 : COADAPT_OK;
  for (size_t i = 0; i < n; ++i) {
    const auto& m = p->plan.moves[i];
    coadapt_move& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.src_rank = m.src_rank;
    o.dst_rank = m.dst_rank;
    o.layer = m.layer;
    o.tensor = m.tensor;
    o.ndim = (int32_t)m.offset.size();
    for (int k = 0; k < o.ndim; ++k) {
      o.offset[k] = m.offset[k];
      o.extent[k] = m.extent[k];
    }
    o.bytes = m.bytes;
    o.local = m.local ? 1 : 0;
  }
  return COADAPT_OK;
}

int coadapt_reshard_shards(const coadapt_reshard_plan* p, int side,
                           coadapt_shard* out, size_t* count) {
  if (!p || !count) return fail(COADAPT_E_VALIDATION, "reshard: NULL argument");
  if (side != COADAPT_RESHARD_SRC && side != COADAPT_RESHARD_DST)
    return fail(COADAPT_E_VALIDATION, "reshard: side must be SRC or DST");
  const auto& L = side == COADAPT_RESHARD_SRC ? p->src : p->dst;
  const size_t n = L.shards.size(), cap = *count;
  *count = n;
  if (cap < n) return out || cap ? fail(COADAPT_E_VALIDATION,
                                        "reshard: shard buffer too small")
                                 : COADAPT_OK;
  for (size_t i = 0; i < n; ++i) to_c_shard(L.shards[i], out[i]);
  return COADAPT_OK;
}

int coadapt_reshard_pack_numel(const coadapt_reshard_plan* p, int side,
                               int rank, uint64_t* numel) {
  if (!p || !numel) return fail(COADAPT_E_VALIDATION, "reshard: NULL argument");
  if (side != COADAPT_RESHARD_SRC && side != COADAPT_RESHARD_DST)
    return fail(COADAPT_E_VALIDATION, "reshard: side must be SRC or DST");
  const auto& L = side == COADAPT_RESHARD_SRC ? p->src : p->dst;
  if (rank < 0 || rank >= (int)L.pack_numel.size())
    return fail(COADAPT_E_VALIDATION, "reshard: rank out of range");
  *numel = L.pack_numel[rank];
  return COADAPT_OK;
}

int coadapt_reshard_plan_csv(const coadapt_reshard_plan* p, char* buf,
                             size_t cap, size_t* needed) {
  if (!p) return fail(COADAPT_E_VALIDATION, "reshard: plan is NULL");
  return guarded([&] {
    const std::string s = R::transfer_plan_csv(p->model, p->plan);
    if (needed) *needed = s.size();
    if (buf && cap) {
      const size_t k = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), k);
      buf[k] = '\0';
    }
    return COADAPT_OK;
  });
}

int coadapt_reshard_latency(const coadapt_reshard_plan* p, double bw,
                            double overhead, double* seconds) {
  if (!p || !seconds) return fail(COADAPT_E_VALIDATION, "reshard: NULL argument");
  return guarded([&] {
    *seconds = R::estimate_reconfig_latency(p->plan, bw, overhead);
    return COADAPT_OK;
  });
}

int coadapt_reshard_execute(coadapt_reshard_plan* p, int role, int rank,
                            const void* const* src_packs, size_t n_src,
                            void* const* dst_packs, size_t n_dst,
                            int elem_bytes, int device, void* stream) {
  COADAPT_NVTX("coadapt_reshard_execute");
  if (!p || !src_packs || !dst_packs)
    return fail(COADAPT_E_VALIDATION, "reshard: NULL argument");
  if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8)
    return fail(COADAPT_E_VALIDATION, "reshard: elem_bytes must be 1, 2, 4 or 8");
  const int S = p->src.strategy.gpus(), D = p->dst.strategy.gpus();
  if (n_src != (size_t)S || n_dst != (size_t)D)
    return fail(COADAPT_E_VALIDATION,
                "reshard: need " + std::to_string(S) + " source and " +
                    std::to_string(D) + " destination pack slots");
  if (role != COADAPT_RESHARD_ALL && role != COADAPT_RESHARD_PULL &&
      role != COADAPT_RESHARD_PUSH)
    return fail(COADAPT_E_VALIDATION, "reshard: unknown role");
  if (role == COADAPT_RESHARD_ALL) rank = -1;
  if (role == COADAPT_RESHARD_PULL && (rank < 0 || rank >= D))
    return fail(COADAPT_E_VALIDATION, "reshard: destination rank out of range");
  if (role == COADAPT_RESHARD_PUSH && (rank < 0 || rank >= S))
    return fail(COADAPT_E_VALIDATION, "reshard: source rank out of range");
  auto mine = [&](const R::Move& m) {
    return role == COADAPT_RESHARD_ALL ||
           (role == COADAPT_RESHARD_PULL ? m.dst_rank : m.src_rank) == rank;
  };
  // every pack this call touches must be present, and no source pack may
  // overlap a destination pack (the pull reads sources while writing)
  std::vector<char> need_src(S, 0), need_dst(D, 0);
  for (const auto& m : p->plan.moves)
    if (mine(m)) {
      need_src[m.src_rank] = 1;
      need_dst[m.dst_rank] = 1;
    }
  for (int r = 0; r < S; ++r)
    if (need_src[r] && !src_packs[r])
      return fail(COADAPT_E_VALIDATION,
                  "reshard: source pack of rank " + std::to_string(r) + " is NULL");
  for (int r = 0; r < D; ++r)
    if (need_dst[r] && !dst_packs[r])
      return fail(COADAPT_E_VALIDATION, "reshard: destination pack of rank " +
                                            std::to_string(r) + " is NULL");
  for (int a = 0; a < S; ++a) {
    if (!need_src[a]) continue;
    const auto sb = reinterpret_cast<uintptr_t>(src_packs[a]);
    const auto se = sb + p->src.pack_numel[a] * elem_bytes;
    for (int b = 0; b < D; ++b) {
      if (!need_dst[b]) continue;
      const auto db = reinterpret_cast<uintptr_t>(dst_packs[b]);
      const auto de = db + p->dst.pack_numel[b] * elem_bytes;
      if (sb < de && db < se)
        return fail(COADAPT_E_VALIDATION,
                    "reshard: source pack " + std::to_string(a) +
                        " overlaps destination pack " + std::to_string(b));
    }
  }
  int prev = -1;
  CU(cudaGetDevice(&prev));
  if (prev != device) CU(cudaSetDevice(device));
  struct Restore {
    int prev, dev;
    ~Restore() {
      if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
  } restore{prev, device};
  auto& T = p->cache[{role, rank, elem_bytes}];
  if (T.dev && T.device != device)
    return fail(COADAPT_E_VALIDATION, "reshard: plan executed on another device");
  if (!T.dev && T.n == 0) {
    std::vector<CopyTask> tasks;
    int rc = guarded([&] {
      for (const auto& m : p->plan.moves)
        if (mine(m))
          emit_tasks(m, p->src.shards[m.src_shard], p->dst.shards[m.dst_shard],
                     elem_bytes, tasks);
      return COADAPT_OK;
    });
    if (rc) return rc;
    T.device = device;
    T.n = (uint32_t)tasks.size();
    if (T.n) {
      CU(cudaMalloc(&T.dev, sizeof(CopyTask) * T.n));
      CU(cudaMemcpy(T.dev, tasks.data(), sizeof(CopyTask) * T.n,
                    cudaMemcpyHostToDevice));
    }
  }
  if (T.n == 0) return COADAPT_OK;
  ExecArgs a;
  std::memset(&a, 0, sizeof(a));
  a.tasks = T.dev;
  a.n_tasks = T.n;
  for (int r = 0; r < S; ++r) a.src[r] = static_cast<const char*>(src_packs[r]);
  for (int r = 0; r < D; ++r) a.dst[r] = static_cast<char*>(dst_packs[r]);
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int grid = (int)std::min<uint32_t>(T.n, (uint32_t)sms * kGridPerSM);
  reshard_copy_kernel<kLoadsInFlight>
      <<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
  CU(cudaGetLastError());
  coadapt_capi::count_launch();
  return COADAPT_OK;
}

}  // extern "C"
