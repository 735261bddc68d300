// bw_sweep.cu — read-bandwidth sweep on one B200 (development tool).
// Streams an 8 GB buffer with a trivial reduction under different load
// strategies and grid shapes, to find the read roofline the GNS kernels can
// reach:  LDG.128 variants (cache hints x loads in flight x CTAs/SM) and a
// TMA bulk-copy (cp.async.bulk + mbarrier) ring into shared memory.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/bw_sweep.cu -o tools/_bw_sweep
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

template <int H>
__device__ __forceinline__ uint4 ld(const uint4* p) {
  uint4 r;
  if (H == 0)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else if (H == 1)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else if (H == 2)
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// 256-bit loads (sm_100): H 0 = nc + L2::256B, 1 = nc + evict_first
struct u8x32 {
  uint4 a, b;
};
template <int H>
__device__ __forceinline__ u8x32 ld256(const uint4* p) {
  u8x32 r;
  if (H == 0)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.a.x), "=r"(r.a.y), "=r"(r.a.z), "=r"(r.a.w), "=r"(r.b.x), "=r"(r.b.y),
                   "=r"(r.b.z), "=r"(r.b.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.a.x), "=r"(r.a.y), "=r"(r.a.z), "=r"(r.a.w), "=r"(r.b.x), "=r"(r.b.y),
                   "=r"(r.b.z), "=r"(r.b.w)
                 : "l"(p));
  return r;
}

__device__ __forceinline__ float vsum(uint4 v) {
  return __uint_as_float(v.x << 16) + __uint_as_float(v.y << 16) +
         __uint_as_float(v.z << 16) + __uint_as_float(v.w << 16);
}

// contiguous share per CTA
template <int H, int U, int NT>
__global__ void __launch_bounds__(NT) k_contig(const uint4* __restrict__ p,
                                                uint64_t nvec, float* out) {
  const uint64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const uint64_t b = per * blockIdx.x;
  const uint64_t e = b + per < nvec ? b + per : nvec;
  float acc = 0.f;
  uint64_t i = b + threadIdx.x;
  for (; i + (uint64_t)(U - 1) * NT < e; i += (uint64_t)U * NT) {
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) r[j] = ld<H>(p + i + (uint64_t)j * NT);
#pragma unroll
    for (int j = 0; j < U; ++j) acc += vsum(r[j]);
  }
  for (; i < e; i += NT) acc += vsum(ld<H>(p + i));
  if (acc == 1234.5f) *out = acc;
}

// contiguous share per CTA, 32-byte loads (nvec counts 16-byte vectors)
template <int H, int U, int NT>
__global__ void __launch_bounds__(NT) k_contig256(const uint4* __restrict__ p,
                                                   uint64_t nvec, float* out) {
  const uint64_t n2 = nvec / 2;
  const uint64_t per = (n2 + gridDim.x - 1) / gridDim.x;
  const uint64_t b = per * blockIdx.x;
  const uint64_t e = b + per < n2 ? b + per : n2;
  float acc = 0.f;
  uint64_t i = b + threadIdx.x;
  for (; i + (uint64_t)(U - 1) * NT < e; i += (uint64_t)U * NT) {
    u8x32 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) r[j] = ld256<H>(p + 2 * (i + (uint64_t)j * NT));
#pragma unroll
    for (int j = 0; j < U; ++j) acc += vsum(r[j].a) + vsum(r[j].b);
  }
  for (; i < e; i += NT) {
    const u8x32 r = ld256<H>(p + 2 * i);
    acc += vsum(r.a) + vsum(r.b);
  }
  if (acc == 1234.5f) *out = acc;
}

// grid-stride over chunks of U*NT vectors (interleaved)
template <int H, int U, int NT>
__global__ void __launch_bounds__(NT) k_stride(const uint4* __restrict__ p,
                                                uint64_t nvec, float* out) {
  float acc = 0.f;
  const uint64_t chunk = (uint64_t)U * NT;
  for (uint64_t c = blockIdx.x; c * chunk < nvec; c += gridDim.x) {
    const uint64_t base = c * chunk + threadIdx.x;
    if (base + (uint64_t)(U - 1) * NT < nvec) {
      uint4 r[U];
#pragma unroll
      for (int j = 0; j < U; ++j) r[j] = ld<H>(p + base + (uint64_t)j * NT);
#pragma unroll
      for (int j = 0; j < U; ++j) acc += vsum(r[j]);
    } else {
      for (uint64_t i = base; i < nvec && i < c * chunk + chunk; i += NT) acc += vsum(ld<H>(p + i));
    }
  }
  if (acc == 1234.5f) *out = acc;
}

// ---- TMA bulk ring --------------------------------------------------------
__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(bar))
      : "memory");
}

template <int S, int CHUNK, int NT>
__global__ void __launch_bounds__(NT) k_tma(const char* __restrict__ p, uint64_t nbytes,
                                             float* out) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t full[S], empty[S];
  constexpr int NCW = NT / 32 - 1;  // consumer warps
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t nchunk_total = nbytes / CHUNK;
  const uint64_t per = (nchunk_total + gridDim.x - 1) / gridDim.x;
  const uint64_t c0 = per * blockIdx.x;
  const uint64_t c1 = c0 + per < nchunk_total ? c0 + per : nchunk_total;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      for (uint64_t c = c0; c < c1; ++c) {
        const uint64_t k = c - c0;
        const int st = (int)(k % S);
        if (k >= S) mbar_wait(&empty[st], (uint32_t)((k / S - 1) & 1));
        mbar_expect(&full[st], CHUNK);
        bulk_g2s(smem + st * CHUNK, p + c * CHUNK, CHUNK, &full[st]);
      }
    }
  } else {
    float acc = 0.f;
    const int ct = threadIdx.x - 32;
    for (uint64_t c = c0; c < c1; ++c) {
      const uint64_t k = c - c0;
      const int st = (int)(k % S);
      mbar_wait(&full[st], (uint32_t)((k / S) & 1));
      const uint4* v = reinterpret_cast<const uint4*>(smem + st * CHUNK);
      for (int i = ct; i < CHUNK / 16; i += NT - 32) acc += vsum(v[i]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (acc == 1234.5f) *out = acc;
  }
}

template <class P>
float time_kernel(void (*kern)(const P*, uint64_t, float*), int grid, int nt, size_t smem,
                  const P* p, uint64_t n, float* out, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<grid, nt, smem>>>(p, n, out);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) kern<<<grid, nt, smem>>>(p, n, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 8.0;
  const uint64_t nbytes = (uint64_t)(gb * 1e9) & ~uint64_t(65535);
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  char* buf;
  float* out;
  CK(cudaMalloc(&buf, nbytes));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(buf, 0x3c, nbytes));
  const uint64_t nvec = nbytes / 16;
  const int reps = 8;
  auto report = [&](const char* name, float ms) {
    printf("%-44s %8.1f GB/s\n", name, nbytes / (ms * 1e-3) / 1e9);
    fflush(stdout);
  };
  char name[128];
#define SWEEP_LDG(KERN, H, U, NT)                                                         \
  for (int occ : {1, 2, 3, 4, 6, 8}) {                                                    \
    if (occ * NT > 2048) continue;                                                        \
    snprintf(name, sizeof name, "%s H%d U%d NT%d occ%d", #KERN, H, U, NT, occ);           \
    report(name, time_kernel(KERN<H, U, NT>, sms * occ, NT, 0,                            \
                             reinterpret_cast<const uint4*>(buf), nvec, out, reps));      \
  }
  SWEEP_LDG(k_contig, 0, 8, 256)
  SWEEP_LDG(k_contig, 1, 8, 256)
  SWEEP_LDG(k_contig, 2, 8, 256)
  SWEEP_LDG(k_contig, 3, 8, 256)
  SWEEP_LDG(k_contig256, 0, 4, 256)
  SWEEP_LDG(k_contig256, 1, 4, 256)
  SWEEP_LDG(k_contig256, 0, 8, 256)
  SWEEP_LDG(k_contig, 0, 4, 256)
  SWEEP_LDG(k_contig, 0, 16, 256)
  SWEEP_LDG(k_contig, 0, 8, 512)
  SWEEP_LDG(k_contig, 0, 4, 512)
  SWEEP_LDG(k_stride, 0, 8, 256)
  SWEEP_LDG(k_stride, 1, 8, 256)
  SWEEP_LDG(k_stride, 0, 4, 512)
#define SWEEP_TMA(S, CH, NT)                                                              \
  for (int occ : {1, 2, 3, 4}) {                                                          \
    const size_t sm = (size_t)S * CH;                                                     \
    if (sm * occ > 220 * 1024) continue;                                                  \
    CK(cudaFuncSetAttribute(k_tma<S, CH, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                            (int)sm));                                                    \
    snprintf(name, sizeof name, "k_tma S%d CH%d NT%d occ%d", S, CH, NT, occ);             \
    report(name, time_kernel(k_tma<S, CH, NT>, sms * occ, NT, sm, buf, nbytes, out, reps)); \
  }
  SWEEP_TMA(4, 16384, 256)
  SWEEP_TMA(8, 16384, 256)
  SWEEP_TMA(4, 32768, 256)
  SWEEP_TMA(6, 32768, 256)
  SWEEP_TMA(3, 65536, 256)
  SWEEP_TMA(8, 8192, 128)
  SWEEP_TMA(12, 8192, 256)
  return 0;
}
