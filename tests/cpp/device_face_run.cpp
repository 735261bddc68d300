// Functional GPU run of the C++ device face (include/coadapt/device.hpp) in
// the sequence INTEGRATION.md §1 documents, entirely from C++:
//
//   coadapt::gns_segments -> BucketLayout -> GnsDevicePlan
//   d = 1: begin_step, record_fused, allreduce, finalize, result
//   d = 2: begin_step, record_micro_bucket x (d*M), record_mean_gradient
//          (BucketLayout::slice per DP replica), allreduce, finalize, result
//   trainer form: accumulate() over the M micro-batches (first / last_mean)
//   host form: record_fused_host from pinned host buckets
//
// The buckets are the integer-exact synthetic gradients (coadapt_synth_fill)
// of a small Llama-shaped model at (d,t,p) rank coordinates with TP dedup
// gaps.  The program checks the device result against the reference API on
// the host (finalize_step / update_ema / gns from the recorded partials:
// bit-identical) and prints every partial and result as JSON with %.17g;
// tests/test_dropin.py::test_device_face_sequence_vs_oracle recomputes them
// with the oracle from the same generator (rel 1e-9 norms, 1e-7 B_simple).
//
// usage: device_face_run <noise_unit as %a> <seed>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "coadapt/device.hpp"
#include "coadapt/errors.hpp"
#include "coadapt/gns.hpp"
#include "coadapt/segments.hpp"
#include "coadapt_cuda.h"

using namespace coadapt;

namespace {

constexpr int M = 4;
constexpr int Bm = 2;
constexpr float G0 = 1.0f / 1024.0f;

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));        \
      std::exit(3);                                                        \
    }                                                                      \
  } while (0)

void lib(int rc) {
  if (rc != COADAPT_OK) {
    std::fprintf(stderr, "C-ABI error %d: %s\n", rc, coadapt_last_error());
    std::exit(3);
  }
}

std::vector<coadapt_gen_segment> gen_of(const RankSegments& rs) {
  std::vector<coadapt_gen_segment> g;
  for (const auto& x : rs.gen)
    g.push_back({x.local_off, x.numel, x.global_base, x.row_len, x.row_stride});
  return g;
}

void print_vec(const char* key, const std::vector<double>& v) {
  std::printf("\"%s\": [", key);
  for (std::size_t i = 0; i < v.size(); ++i)
    std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]");
}

void print_result(const char* key, const DeviceStepResult& r) {
  std::printf("\"%s\": {\"signal\": %.17g, \"noise\": %.17g, \"noise_raw\": %.17g, "
              "\"mean_grad_sq\": %.17g, \"b_simple\": %.17g, \"phi\": %.17g, "
              "\"ema_signal\": %.17g, \"ema_noise\": %.17g, \"tokens_seen\": %lld}",
              key, r.stats.signal, r.stats.noise, r.stats.noise_raw, r.stats.mean_grad_sq,
              r.b_simple, r.phi ? *r.phi : NAN, r.state.ema_signal, r.state.ema_noise,
              (long long)r.state.tokens_seen);
}

bool same(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

// The device finalize (K3) must equal the reference API on the host, run on
// the device's own recorded partials, bit for bit (gns.hpp:42-73).
int check_against_host(GnsDevicePlan& plan, const DeviceStepResult& r,
                       GnsState& host_state, std::int64_t tokens, const char* what) {
  StepAccumulator acc = plan.accumulator();
  std::vector<double> parts(acc.sample_count() + 1);
  lib(coadapt_gns_read_partials(plan.handle(), parts.data(), parts.size()));
  const StepStats st = finalize_step(acc, parts.back());
  update_ema(host_state, st, tokens);
  const auto phi = gns(host_state);
  if (!same(st.signal, r.stats.signal) || !same(st.noise, r.stats.noise) ||
      !same(st.noise_raw, r.stats.noise_raw) || !same(st.mean_grad_sq, r.stats.mean_grad_sq) ||
      !same(host_state.ema_signal, r.state.ema_signal) ||
      !same(host_state.ema_noise, r.state.ema_noise) ||
      host_state.tokens_seen != r.state.tokens_seen || phi.has_value() != r.phi.has_value() ||
      (phi && !same(*phi, *r.phi))) {
    std::fprintf(stderr, "%s: device finalize differs from the host reference API\n", what);
    return 1;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s <noise_unit %%a> <seed>\n", argv[0]);
    return 2;
  }
  const float unit = std::strtof(argv[1], nullptr);
  const std::uint64_t seed = std::strtoull(argv[2], nullptr, 0);
  try {
    // h = 256, ffn = 512, vocab 1000, 4 layers, QKV bias: (1,2,2) rank 1 is
    // tp_rank 1 of stage 0 -> its norms carry weight 0 (dedup gaps)
    const GradModel model = llama_model("tiny", 1000, 256, 4, 512, 4, 2, false, true);
    const RankSegments rs = gns_segments(model, ParallelStrategy{1, 2, 2}, 1);
    const auto gen = gen_of(rs);
    const std::uint64_t n = rs.bucket_numel;
    BucketLayout layout(rs.segments, n, GradDType::kBF16, 0);
    cudaStream_t stream;
    CK(cudaStreamCreate(&stream));
    std::vector<void*> bufs(M);
    for (auto& b : bufs) CK(cudaMalloc(&b, n * 2));
    void* mean = nullptr;
    CK(cudaMalloc(&mean, n * 2));
    float* main_grad = nullptr;
    CK(cudaMalloc(&main_grad, n * 4));
    int bad = 0;
    std::printf("{\"numel\": %llu, \"counted\": %llu, ", (unsigned long long)n,
                (unsigned long long)rs.counted());

    // ---- d = 1: one fused pass (all s_m + gbar^2), INTEGRATION.md §1
    {
      for (int m = 0; m < M; ++m)
        lib(coadapt_synth_fill(bufs[m], COADAPT_BF16, gen.data(), gen.size(), seed, m, G0,
                               unit, stream));
      GnsDevicePlan gns(1, M, M * Bm, 0);
      GnsState host_state;
      std::vector<const void*> ptrs(bufs.begin(), bufs.end());
      for (int step = 0; step < 2; ++step) {  // two steps: the EMA advances
        gns.begin_step(stream);
        gns.record_fused(layout, ptrs, stream);
        gns.allreduce(stream);  // world 1: the local sum
        gns.finalize((std::int64_t)M * Bm * 2048, stream);
        while (!gns.result_ready()) {
        }  // non-blocking poll until the step's result is on the host
        const DeviceStepResult r = gns.result();
        bad |= check_against_host(gns, r, host_state, (std::int64_t)M * Bm * 2048, "d=1");
        if (step == 1) {
          std::vector<double> parts(M + 1);
          lib(coadapt_gns_read_partials(gns.handle(), parts.data(), parts.size()));
          print_vec("d1_partials", parts);
          std::printf(", ");
          print_result("d1_result", r);
          std::printf(", ");
        }
      }
      // the finalize in the same pass (record_fused_finalize) == the
      // separate record_fused + finalize, bit for bit
      {
        GnsDevicePlan sep(1, M, M * Bm, 0), inp(1, M, M * Bm, 0);
        sep.begin_step(stream);
        sep.record_fused(layout, ptrs, stream);
        sep.finalize((std::int64_t)M * Bm * 2048, stream);
        inp.begin_step(stream);
        inp.record_fused_finalize(layout, ptrs, (std::int64_t)M * Bm * 2048, stream);
        const DeviceStepResult a = sep.result(), b = inp.result();
        if (!same(a.stats.signal, b.stats.signal) || !same(a.stats.noise, b.stats.noise) ||
            !same(a.b_simple, b.b_simple) || !same(a.state.ema_signal, b.state.ema_signal)) {
          std::fprintf(stderr, "record_fused_finalize differs from record_fused + finalize\n");
          bad |= 1;
        }
      }
      // host buckets (pinned) through the same plan: record_fused_host
      std::vector<void*> host(M);
      for (int m = 0; m < M; ++m) {
        CK(cudaMallocHost(&host[m], n * 2));
        CK(cudaMemcpy(host[m], bufs[m], n * 2, cudaMemcpyDeviceToHost));
      }
      GnsDevicePlan gh(1, M, M * Bm, 0);
      gh.begin_step(stream);
      std::vector<const void*> hp(host.begin(), host.end());
      gh.record_fused_host(layout, hp, stream);
      gh.finalize((std::int64_t)M * Bm * 2048, stream);
      (void)gh.result();
      std::vector<double> hparts(M + 1);
      lib(coadapt_gns_read_partials(gh.handle(), hparts.data(), hparts.size()));
      print_vec("d1_host_partials", hparts);
      std::printf(", ");
      for (auto h : host) CK(cudaFreeHost(h));

      // trainer form: main_grad (+)= g_m with s_m fused, gbar^2 on the last
      GnsDevicePlan ga(1, M, M * Bm, 0);
      ga.begin_step(stream);
      for (int m = 0; m < M; ++m)
        ga.accumulate(layout, main_grad, bufs[m], 0, m, m == 0, m == M - 1,
                      1.0 / ((double)M * M), stream);
      ga.finalize((std::int64_t)M * Bm * 2048, stream);
      GnsState hs;
      bad |= check_against_host(ga, ga.result(), hs, (std::int64_t)M * Bm * 2048, "accumulate");
      std::vector<double> aparts(M + 1);
      lib(coadapt_gns_read_partials(ga.handle(), aparts.data(), aparts.size()));
      print_vec("accumulate_partials", aparts);
      std::printf(", ");
    }

    // ---- d = 2: per-micro-bucket passes + the DP slices of the mean
    {
      const int d = 2;
      GnsDevicePlan gns(d, M, (std::int64_t)d * M * Bm, 0);
      gns.begin_step(stream);
      for (int i_d = 0; i_d < d; ++i_d) {
        for (int m = 0; m < M; ++m) {
          lib(coadapt_synth_fill(bufs[m], COADAPT_BF16, gen.data(), gen.size(), seed,
                                 (std::uint64_t)(i_d * M + m), G0, unit, stream));
          gns.record_micro_bucket(layout, bufs[m], i_d, m, stream);
        }
        CK(cudaStreamSynchronize(stream));  // buffers are refilled next round
      }
      lib(coadapt_synth_mean_fill(mean, COADAPT_BF16, gen.data(), gen.size(), seed, 0, d * M,
                                  G0, unit, stream));
      for (int i_d = 0; i_d < d; ++i_d) {
        BucketLayout sl = BucketLayout::slice(rs.segments, n, GradDType::kBF16, 0, i_d, d);
        gns.record_mean_gradient(sl, mean, stream);
        CK(cudaStreamSynchronize(stream));
      }
      gns.allreduce(stream);
      gns.finalize((std::int64_t)d * M * Bm * 2048, stream);
      const DeviceStepResult r = gns.result();
      GnsState hs;
      bad |= check_against_host(gns, r, hs, (std::int64_t)d * M * Bm * 2048, "d=2");
      std::vector<double> parts(d * M + 1);
      lib(coadapt_gns_read_partials(gns.handle(), parts.data(), parts.size()));
      print_vec("d2_partials", parts);
      std::printf(", ");
      print_result("d2_result", r);
    }
    std::printf(", \"host_api_bit_identical\": %s}\n", bad ? "false" : "true");
    for (auto b : bufs) cudaFree(b);
    cudaFree(mean);
    cudaFree(main_grad);
    cudaStreamDestroy(stream);
    return bad;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    return 1;
  }
}
