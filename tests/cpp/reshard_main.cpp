// C++ use of coadapt/reshard.hpp (§8 f4), built by tests/test_reshard_cpp.py.
//   reshard_main        -> prints the plan CSV of a fixed case (compared with
//                          the oracle's CSV by the Python test)
//   reshard_main --gpu  -> DevicePlan::all / pull / push over virtual ranks on
//                          device 0; every destination element must equal
//                          the global tensor's value at that index
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "coadapt/errors.hpp"
#include "coadapt/reshard.hpp"

using namespace coadapt;
using namespace coadapt::reshard;

static ModelSpec model() {
  ModelSpec m;
  m.layers = 4;
  m.per_layer = {{"qkv", {96, 40}, 0}, {"out", {40, 96}, 1}, {"norm", {40}, -1},
                 {"conv", {8, 6, 24}, 2}};
  return m;
}

// value of element `flat` of (layer, tensor): a 16-bit hash
static uint16_t value(int layer, int tensor, uint64_t flat) {
  uint64_t x = flat * 0x9E3779B97F4A7C15ull + (uint64_t)layer * 1000003 + tensor;
  x ^= x >> 29;
  x *= 0xBF58476D1CE4E5B9ull;
  return (uint16_t)(x >> 48);
}

static uint64_t flat_index(const ShardDescriptor& s, const std::vector<int64_t>& local) {
  uint64_t f = 0;
  for (std::size_t i = 0; i < local.size(); ++i)
    f = f * s.global_shape[i] + (uint64_t)(s.global_offset[i] + local[i]);
  return f;
}

// fill (or check) every shard of `rank` in a host copy of its pack
static int walk(const ShardLayout& L, int rank, std::vector<uint16_t>& pack, bool fill) {
  int bad = 0;
  for (const auto& s : L.shards) {
    if (s.owner != rank) continue;
    std::vector<int64_t> idx(s.local_shape.size(), 0);
    for (uint64_t e = 0; e < s.numel(); ++e) {
      const uint16_t v = value(s.layer, s.tensor, flat_index(s, idx));
      if (fill)
        pack[s.pack_offset + e] = v;
      else if (pack[s.pack_offset + e] != v)
        ++bad;
      for (int k = (int)idx.size() - 1; k >= 0; --k) {
        if (++idx[k] < s.local_shape[k]) break;
        idx[k] = 0;
      }
    }
  }
  return bad;
}

#define CK(x)                                                    \
  do {                                                           \
    cudaError_t e_ = (x);                                        \
    if (e_ != cudaSuccess) {                                     \
      std::printf("CUDA %s: %s\n", #x, cudaGetErrorString(e_));  \
      return 1 << 20;                                            \
    }                                                            \
  } while (0)

static int gpu_case(const ParallelStrategy& a, const ParallelStrategy& b, int mode) {
  DevicePlan dp(model(), a, b, SourcePolicy::kSpread);
  const auto& S = dp.source();
  const auto& D = dp.destination();
  std::vector<void*> src(a.gpus()), dst(b.gpus());
  for (int r = 0; r < a.gpus(); ++r) {
    std::vector<uint16_t> h(S.pack_numel[r], 0);
    walk(S, r, h, true);
    CK(cudaMalloc(&src[r], h.size() * 2 + 16));
    CK(cudaMemcpy(src[r], h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  }
  for (int r = 0; r < b.gpus(); ++r) {
    CK(cudaMalloc(&dst[r], D.pack_numel[r] * 2 + 16));
    CK(cudaMemset(dst[r], 0, D.pack_numel[r] * 2));
  }
  std::vector<const void*> csrc(src.begin(), src.end());
  if (mode == 0) dp.all(csrc, dst, 2, 0, nullptr);
  if (mode == 1)
    for (int r = 0; r < b.gpus(); ++r) dp.pull(r, csrc, dst, 2, 0, nullptr);
  if (mode == 2)
    for (int r = 0; r < a.gpus(); ++r) dp.push(r, csrc, dst, 2, 0, nullptr);
  CK(cudaDeviceSynchronize());
  int bad = 0;
  for (int r = 0; r < b.gpus(); ++r) {
    std::vector<uint16_t> h(D.pack_numel[r]);
    CK(cudaMemcpy(h.data(), dst[r], h.size() * 2, cudaMemcpyDeviceToHost));
    bad += walk(D, r, h, false);
  }
  for (auto p : src) cudaFree(p);
  for (auto p : dst) cudaFree(p);
  return bad;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  if (!gpu) {
    const ModelSpec m = model();
    const auto A = layout_for(m, {1, 2, 2}, 4);
    const auto B = layout_for(m, {2, 1, 2}, 4);
    const auto plan = plan_transfers(m, A, B);
    std::printf("%s", transfer_plan_csv(m, plan).c_str());
    std::printf("#total=%llu max=%llu local=%llu latency=%.17g\n",
                (unsigned long long)plan.total_bytes,
                (unsigned long long)plan.max_bytes_per_rank,
                (unsigned long long)plan.local_bytes,
                estimate_reconfig_latency(plan, 1e9, 20.0));
    bool threw = false;
    try {
      layout_for(m, {1, 5, 1}, 5);  // 96 % 5 != 0
    } catch (const ValidationError&) {
      threw = true;
    }
    std::printf(threw ? "#validation ok\n" : "#validation MISSING\n");
    return threw ? 0 : 1;
  }
  int failures = 0;
  const ParallelStrategy ss[] = {{1, 1, 1}, {1, 2, 2}, {2, 1, 2}, {1, 4, 1},
                                 {2, 2, 1}, {1, 1, 4}, {4, 2, 1}, {2, 2, 2}};
  for (const auto& a : ss)
    for (const auto& b : ss)
      for (int mode = 0; mode < 3; ++mode) {
        const int bad = gpu_case(a, b, mode);
        if (bad) {
          std::printf("FAIL %s -> %s mode %d: %d elements\n", a.label().c_str(),
                      b.label().c_str(), mode, bad);
          ++failures;
        }
      }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
