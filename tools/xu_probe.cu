// xu_probe — achievable F2F.F64.BF16 throughput per SM on this GPU, from
// registers (no memory traffic), to tell whether the fused pass's ~79 % XU
// utilisation (profiles/r02_k1f_stalls.txt) is the pipe's practical ceiling
// or a scheduling shortfall.  Each thread converts 8 bf16 halves per
// iteration (words mutated by an integer LCG so nothing is hoisted) and
// accumulates the squares with DFMA, like vacc; variants without the DFMA
// and with the K1f micro-batch FHFMA added.  Prints conversions per clock
// per SM for several resident-warp counts.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o xu_probe xu_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double cvt(uint16_t h) {
  double d;
  asm volatile("cvt.f64.bf16 %0, %1;" : "=d"(d) : "h"(h));
  return d;
}
__device__ __forceinline__ float addbf(float s, uint16_t h) {
  asm volatile("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(s) : "h"(h), "h"((uint16_t)0x3F80));
  return s;
}

template <int MODE>  // 0: F2F + DFMA, 1: F2F + DADD only, 2: F2F + DFMA + FHFMA
__global__ void probe(int iters, double* out, float* outf, long long* cyc) {
  const long long c0 = clock64();
  uint32_t w0 = threadIdx.x * 2654435761u + blockIdx.x, w1 = w0 ^ 0x9E3779B9u;
  uint32_t w2 = w0 * 3u + 7u, w3 = w1 * 5u + 11u;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  float s = 0.f;
  for (int i = 0; i < iters; ++i) {
    const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double lo = cvt((uint16_t)(w[k] & 0x7fffu)), hi = cvt((uint16_t)((w[k] >> 16) & 0x7fffu));
      if (MODE == 1) {
        a0 += lo;
        a1 += hi;
      } else {
        a0 = fma(lo, lo, a0);
        a1 = fma(hi, hi, a1);
      }
      if (MODE == 2) {
        s = addbf(s, (uint16_t)(w[k] & 0xffffu));
        s = addbf(s, (uint16_t)(w[k] >> 16));
      }
    }
    w0 = w0 * 1664525u + 1013904223u;
    w1 = w1 * 1664525u + 1013904223u;
    w2 = w2 * 22695477u + 1u;
    w3 = w3 * 22695477u + 1u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
  outf[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = clock64() - c0;
}

int main() {
  int sms = 0;
  long long* cyc;
  cudaMallocManaged(&cyc, sizeof(long long));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  float* outf;
  cudaMalloc(&out, sizeof(double) * 148 * 1024 * 4);
  cudaMalloc(&outf, sizeof(float) * 148 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 12, 16, 24, 32}) {
      const int nt = warps * 32;
      auto launch = [&]() {
        if (mode == 0) probe<0><<<sms, nt>>>(iters, out, outf, cyc);
        if (mode == 1) probe<1><<<sms, nt>>>(iters, out, outf, cyc);
        if (mode == 2) probe<2><<<sms, nt>>>(iters, out, outf, cyc);
      };
      launch();
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      // read the SM clock the kernel ran at from a clock64 probe is awkward;
      // report conversions per ns per SM and, with the clock nvidia-smi
      // reports during the run, per clock
      const double conv = (double)sms * nt * iters * 8;
      const double ghz = (double)*cyc / (ms * 1e6);
      std::printf("{\"mode\": %d, \"warps_per_sm\": %d, \"ms\": %.3f, \"sm_ghz\": %.3f, "
                  "\"conv_per_clk_per_sm\": %.2f}\n",
                  mode, warps, ms, ghz, conv / (ms * 1e6) / sms / ghz);
    }
  return 0;
}
