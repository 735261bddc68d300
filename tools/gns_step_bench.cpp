// gns_step_bench — the full online-GNS goodput step (BASELINE C5) driven from
// C++ alone, the way a C++ trainer/orchestrator links the library: no Python
// in the loop.  Every optimizer step:
//   begin_step -> one fused pass per virtual rank on this GPU (K1f), the last
//   one with finalize/EMA/phi in its last CTA -> result (phi D2H) ->
//   coadapt::decide over the (d,t,p,B_g,B_m) candidate table.
// Layouts come from coadapt::gns_segments; buckets are the integer-exact
// synthetic gradients (coadapt_synth_fill); as in bench.py the job's virtual
// ranks on one GPU share one resident pool of M buckets sized for the largest
// rank, and every launch streams its rank's full bytes from HBM.
//
//   gns_step_bench [model=32b] [d t p M] [steps=10] [warmup=3]
// prints one JSON line: GB/s (algorithmic bytes per step / step time),
// ms per step, the split into device time and host decide time.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

#include "coadapt/device.hpp"
#include "coadapt/orchestrator.hpp"
#include "coadapt/segments.hpp"
#include "coadapt_cuda.h"

using namespace coadapt;

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));         \
      return 3;                                                             \
    }                                                                       \
  } while (0)

int main(int argc, char** argv) {
  const std::string key = argc > 1 ? argv[1] : "32b";
  const int d = argc > 5 ? std::atoi(argv[2]) : 1, t = argc > 5 ? std::atoi(argv[3]) : 4,
            p = argc > 5 ? std::atoi(argv[4]) : 2, M = argc > 5 ? std::atoi(argv[5]) : 16;
  const int steps = argc > 6 ? std::atoi(argv[6]) : 10, warmup = argc > 7 ? std::atoi(argv[7]) : 3;
  if (d != 1) {
    std::fprintf(stderr, "this driver runs the fused d = 1 form (K1f)\n");
    return 2;
  }
  try {
    const GradModel model = model_preset(key);
    const ParallelStrategy S{d, t, p};
    const int R = S.gpus();
    std::vector<RankSegments> ranks;
    std::uint64_t cap = 0;
    for (int r = 0; r < R; ++r) {
      ranks.push_back(gns_segments(model, S, r));
      cap = std::max(cap, ranks.back().bucket_numel);
    }
    const std::uint64_t job_bytes = gns_algorithmic_bytes(model, S, M, 2, true);
    cudaStream_t stream;
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    std::vector<void*> pool(M);
    for (auto& b : pool) {
      CK(cudaMalloc(&b, cap * 2));
      CK(cudaMemset(b, 0, cap * 2));  // past the filled rank's end: zeros
    }
    // phi_true = 256 at B_m = 1: unit = g0 * sqrt(256) / std(Irwin-Hall(4, 16-bit))
    const float g0 = 1.0f / 1024.0f;
    const float unit = (float)(g0 * 16.0 / std::sqrt((4294967296.0 - 1.0) / 3.0));
    std::vector<coadapt_gen_segment> gen;
    for (const auto& x : ranks[0].gen)
      gen.push_back({x.local_off, x.numel, x.global_base, x.row_len, x.row_stride});
    for (int m = 0; m < M; ++m)
      if (coadapt_synth_fill(pool[m], COADAPT_BF16, gen.data(), gen.size(), 0xC0905 + 3, m, g0,
                             unit, stream) != COADAPT_OK) {
        std::fprintf(stderr, "synth_fill: %s\n", coadapt_last_error());
        return 3;
      }
    std::vector<BucketLayout> layouts;
    for (const auto& rs : ranks)
      layouts.emplace_back(rs.segments, cap, GradDType::kBF16, 0);
    const std::int64_t B_g = (std::int64_t)d * M;  // B_m = 1
    GnsDevicePlan gns(d, M, B_g, 0);
    std::vector<const void*> ptrs(pool.begin(), pool.end());
    // candidate table over every (d,t,p) of the job's GPU count
    CostModelParams cp;
    for (int dd = 1; dd <= R; ++dd)
      for (int tt = 1; dd * tt <= R; ++tt)
        if (R % (dd * tt) == 0)
          cp.per_strategy.push_back({ParallelStrategy{dd, tt, R / (dd * tt)},
                                     1000.0 * std::sqrt((double)dd) * (1.0 + 0.2 * tt),
                                     8.0 * dd * dd + 4.0 * (R / (dd * tt))});
    cp.pipeline_bubble = true;
    const std::vector<std::int64_t> bg = {16, 32, 64, 128, 256, 512, 1024, 2048}, bm = {1, 2, 4, 8};
    const auto cands = feasible_candidates(synth_profile(cp, bg, bm, 1e300, R));
    ConfigTuple current = cands.front().config;  // this job's entry if the table has it
    for (const auto& c : cands)
      if (c.config.strategy == S && c.config.global_batch == B_g) {
        current = c.config;
        break;
      }
    OrchestratorConfig cfg;
    cfg.reconfig_cost = 40.0;
    ClockState clock{1000.0, 900.0, 0.0, 0};
    double decide_s = 0.0;
    auto step = [&](bool timed) {
      gns.begin_step(stream);
      for (int r = 0; r < R; ++r) {
        if (r + 1 < R)
          gns.record_fused(layouts[r], ptrs, stream);
        else
          gns.record_fused_finalize(layouts[r], ptrs, B_g * 2048, stream);
      }
      const DeviceStepResult res = gns.result();  // phi -> host, waits for the step
      const auto h0 = std::chrono::steady_clock::now();
      const Command cmd = decide(cands, res.phi, current, clock, cfg);
      (void)cmd;
      if (timed)
        decide_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
      return res;
    };
    for (int i = 0; i < warmup; ++i) step(false);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaStreamSynchronize(stream));
    CK(cudaEventRecord(a, stream));
    DeviceStepResult last;
    for (int i = 0; i < steps; ++i) last = step(true);
    CK(cudaEventRecord(b, stream));
    CK(cudaEventSynchronize(b));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, a, b));
    const double ms_step = ms / steps;
    std::printf(
        "{\"driver\": \"tools/gns_step_bench (C++ host, no Python)\", \"model\": \"%s\", "
        "\"dtp\": [%d, %d, %d], \"M\": %d, \"job_ranks_on_this_gpu\": %d, \"steps\": %d, "
        "\"bytes_per_step\": %llu, \"ms_per_step\": %.4f, \"GB_per_s\": %.1f, "
        "\"decide_ms\": %.4f, \"candidates\": %zu, \"phi\": %.6f, \"b_simple\": %.6f}\n",
        key.c_str(), d, t, p, M, R, steps, (unsigned long long)job_bytes, ms_step,
        job_bytes / (ms_step / 1e3) / 1e9, 1e3 * decide_s / steps, cands.size(),
        last.phi ? *last.phi : -1.0, last.b_simple);
    for (auto bptr : pool) cudaFree(bptr);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    return 1;
  }
}
