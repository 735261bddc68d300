// kernels.cu — sm_100a kernels of the GNS hot path.
//
//   K1  s += sum_ranges w * ||bucket[range]||^2 for 1..16 buckets sharing one
//       layout and the d > 1 mean-gradient read
//       (PAPER.md:444-445): fused_tma_kernel<..., MEAN=false> (TMA bulk ring)
//       for 16-byte-aligned buckets, sqnorm_kernel (LDG) for unaligned views.
//   K1f fused_tma_kernel<..., MEAN=true>: d = 1: all M micro-buckets of a
//       rank in one pass, every s_m plus ||sum_m g_m||^2; fused_kernel is
//       its LDG form for unaligned buckets.
//   KA  accum_kernel   : trainer form, fp32 grad accumulation + s_m (+ gbar^2).
//   K3  finalize_kernel: finalize_step + update_ema + gns (gns.hpp:42-73).
//   K0  synth kernels  : integer-exact synthetic gradients (test/bench data).
//
// Bandwidth design (B200, HBM3e): the reductions are pure streams.  The
// active elements are cut into chunks assigned CTA c <- chunk c mod G, so
// all CTAs sweep HBM together (7.35 TB/s read ceiling measured by
// tools/bw_sweep.cu, vs ~6.5 TB/s for contiguous per-CTA shares).  The TMA
// ring (one producer lane, cp.async.bulk into a 4-stage shared-memory ring,
// consumer warps on LDS) is the main path: under the 1 kW power cap it
// streams ~14 % faster than 128-bit LDG loads with the same arithmetic.
// Weight-0 ranges (TP duplicates) are never loaded.  Every square is
// exact in fp64 and summed in fp64; CTA partials are combined by the last
// CTA in a fixed order, so results are bit-reproducible run to run.
#include <atomic>

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <cstring>

#include "../../include/coadapt_cuda.h"
#include "internal.h"

namespace coadapt {
namespace dev {
namespace {

template <int DT>
struct Elem;
template <>
struct Elem<COADAPT_BF16> {
  static constexpr int kSize = 2, kPerVec = 8;
};
template <>
struct Elem<COADAPT_FP16> {
  static constexpr int kSize = 2, kPerVec = 8;
};
template <>
struct Elem<COADAPT_FP32> {
  static constexpr int kSize = 4, kPerVec = 4;
};
template <>
struct Elem<COADAPT_FP64> {
  static constexpr int kSize = 8, kPerVec = 2;
};
// Streaming 128-bit load: read-only path, no L1 allocation, 256B L2 prefetch.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

__device__ __forceinline__ float bf16_lo(uint32_t w) {
  return __uint_as_float(w << 16);
}
__device__ __forceinline__ float bf16_hi(uint32_t w) {
  return __uint_as_float(w & 0xffff0000u);
}

// The 8/4/2 element values of one 16-byte vector as fp32 (not for fp64).
template <int DT>
__device__ __forceinline__ void unpack(const uint4& v, float* f);
template <>
__device__ __forceinline__ void unpack<COADAPT_BF16>(const uint4& v,
                                                     float* f) {
  f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x);
  f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
  f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z);
  f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
}
template <>
__device__ __forceinline__ void unpack<COADAPT_FP16>(const uint4& v,
                                                     float* f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
    float2 t = __half22float2(h);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
template <>
__device__ __forceinline__ void unpack<COADAPT_FP32>(const uint4& v,
                                                     float* f) {
  f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
  f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
}

// bf16 -> fp64 straight from the half-word (SASS F2F.F64.BF16 with a .H1
// selector: no unpack instruction).  Exact for every bf16.
__device__ __forceinline__ double bf16_f64(uint16_t h) {
  double d;
  asm("cvt.f64.bf16 %0, %1;" : "=d"(d) : "h"(h));
  return d;
}
// fp16 -> fp64 straight from the half-word (F2F.F64.F16), exact.
__device__ __forceinline__ double f16_f64(uint16_t h) {
  double d;
  asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(h));
  return d;
}
// s + x in one fp32 rounding, x a bf16 half-word read in place (SASS
// FHADD.BF16, the mixed-precision add): identical to __fadd_rn(s, (float)x).
// (Round 1 used FHFMA.BF16, x * 1.0 + s — same result; FHADD measured
// +0.4 % on the fused pass, profiles/r02_vacc_variants.txt call 13.)
__device__ __forceinline__ float bf16_addf(float s, uint16_t h) {
  asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(s) : "h"(h));
  return s;
}

// sum[e] += x_e (fp32, one rounding each) for the values of one vector: the
// micro-batch sum of the fused pass.  bf16 via FHADD on the packed halves,
// the others unpacked and added pairwise with FADD2 (same rounding per lane).
template <int DT>
__device__ __forceinline__ void micro_add(const uint4& v, float* sum) {
  if constexpr (DT == COADAPT_BF16) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      sum[2 * i] = bf16_addf(sum[2 * i], (uint16_t)(w[i] & 0xffffu));
      sum[2 * i + 1] = bf16_addf(sum[2 * i + 1], (uint16_t)(w[i] >> 16));
    }
  } else {
    constexpr int PV = Elem<DT>::kPerVec;
    float f[PV];
    unpack<DT>(v, f);
#pragma unroll
    for (int e = 0; e < PV; e += 2) {
      const float2 t = __fadd2_rn(make_float2(sum[e], sum[e + 1]),
                                  make_float2(f[e], f[e + 1]));
      sum[e] = t.x;
      sum[e + 1] = t.y;
    }
  }
}

// acc += sum of squares of one vector, every square exact in fp64.
// Each value goes to fp64 with one F2F on the XU pipe (bf16 straight from
// the half-word) and is squared into one of two DFMA chains.  Measured
// alternatives (profiles/r01c_vacc_variants.txt, r02_vacc_variants.txt):
// fp32 squares summed in runs of 8 (+7 % K1f, +22 % K1 sustained) are not
// exact; every exact XU-free form (fp64 built from the bits on the ALU, as
// two scaled operands or one into a 2^-822-scaled accumulator, for half or
// all of the elements) moves K1 by at most +1.5 % and costs the fused pass
// 12-16 %; a chain continuing the accumulator costs 1.2 %.  This form stays.
template <int DT>
__device__ __forceinline__ void vacc(const uint4& v, double& acc) {
  if constexpr (DT == COADAPT_BF16) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    // two fp64 chains per vector halve the dependent DFMA latency
    double a0 = bf16_f64((uint16_t)(w[0] & 0xffffu));
    double a1 = bf16_f64((uint16_t)(w[0] >> 16));
    a0 *= a0;
    a1 *= a1;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      const double d0 = bf16_f64((uint16_t)(w[i] & 0xffffu));
      const double d1 = bf16_f64((uint16_t)(w[i] >> 16));
      a0 = fma(d0, d0, a0);
      a1 = fma(d1, d1, a1);
    }
    acc += a0 + a1;
    return;
  }
  if constexpr (DT == COADAPT_FP16) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    double a0 = f16_f64((uint16_t)(w[0] & 0xffffu));
    double a1 = f16_f64((uint16_t)(w[0] >> 16));
    a0 *= a0;
    a1 *= a1;
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      const double d0 = f16_f64((uint16_t)(w[i] & 0xffffu));
      const double d1 = f16_f64((uint16_t)(w[i] >> 16));
      a0 = fma(d0, d0, a0);
      a1 = fma(d1, d1, a1);
    }
    acc += a0 + a1;
  } else if constexpr (DT == COADAPT_FP32) {
    float f[4];
    unpack<DT>(v, f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double d = f[i];
      acc = fma(d, d, acc);
    }
  } else {
    const double a = __hiloint2double(v.y, v.x);
    const double b = __hiloint2double(v.w, v.z);
    acc = fma(a, a, acc);
    acc = fma(b, b, acc);
  }
}

template <int DT>
__device__ __forceinline__ double elem_f64(uintptr_t addr) {
  if constexpr (DT == COADAPT_BF16) {
    const uint16_t h = *reinterpret_cast<const uint16_t*>(addr);
    return (double)__uint_as_float((uint32_t)h << 16);
  } else if constexpr (DT == COADAPT_FP16) {
    return (double)__half2float(*reinterpret_cast<const __half*>(addr));
  } else if constexpr (DT == COADAPT_FP32) {
    return (double)*reinterpret_cast<const float*>(addr);
  } else {
    return *reinterpret_cast<const double*>(addr);
  }
}

template <int DT>
__device__ __forceinline__ float elem_f32(uintptr_t addr) {
  if constexpr (DT == COADAPT_BF16) {
    const uint16_t h = *reinterpret_cast<const uint16_t*>(addr);
    return __uint_as_float((uint32_t)h << 16);
  } else if constexpr (DT == COADAPT_FP16) {
    return __half2float(*reinterpret_cast<const __half*>(addr));
  } else {
    return *reinterpret_cast<const float*>(addr);
  }
}

// ---------------------------------------------------------------- reductions

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // red may still be read by a previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  v = 0.0;
  if (warp == 0) {
    v = lane < NT / 32 ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

// Last-CTA combine: every CTA has stored its per-output partial at
// partials[o * G + cta]; the CTA that takes the last ticket sums each
// output's G partials in a fixed order and adds scale*sum into slots[slot].
template <int NT>
__device__ __forceinline__ bool last_cta_combine(const Sink& sink, int nout,
                                                 const int32_t* out_slot,
                                                 const double* out_scale,
                                                 double* red) {
  __shared__ unsigned int is_last;
  const int G = gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(sink.ticket, 1u);
    is_last = (t == (unsigned)G - 1u);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  for (int o = 0; o < nout; ++o) {
    double v = 0.0;
    for (int c = threadIdx.x; c < G; c += NT)
      v += __ldcg(sink.partials + (size_t)o * G + c);
    v = block_sum<NT>(v, red);
    if (threadIdx.x == 0) {
      const double sc = out_scale ? out_scale[o] : 1.0;
      double* dst = sink.slots + out_slot[o];
      *dst = *dst + (sc == 1.0 ? v : v * sc);
    }
  }
  if (threadIdx.x == 0) *sink.ticket = 0u;  // ready for the next launch
  return true;
}

// defined with K3 / X1 below; the TMA kernel's last CTA may run them
__device__ void finalize_body(const FinalizeArgs& a);
__device__ void p2p_exchange_finalize(const P2PArgs& a);

// This CTA's equal share of the window [e_begin, e_end) of active elements,
// rounded to 64-element multiples so bodies stay 16B-aligned.
__device__ __forceinline__ void cta_share(const Window& w, uint64_t& e0,
                                          uint64_t& e1) {
  const uint64_t n = w.e_end - w.e_begin;
  uint64_t per = (n + gridDim.x - 1) / gridDim.x;
  per = (per + 63) & ~uint64_t(63);
  e0 = w.e_begin + min(n, per * blockIdx.x);
  e1 = w.e_begin + min(n, per * (blockIdx.x + 1));
}

__device__ __forceinline__ int find_range(const Range* __restrict__ R, int nr,
                                          uint64_t e) {
  int lo = 0, hi = nr - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (R[mid].cum_begin <= e) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// acc += ||x[a, a+n)||^2 of one stream.
template <int DT, int NT, int U>
__device__ __forceinline__ void piece_sumsq(uintptr_t base, uint64_t a,
                                            uint64_t n, double& acc) {
  constexpr int ES = Elem<DT>::kSize;
  const uintptr_t u0 = base + a * ES, u1 = u0 + n * ES;
  const uintptr_t v0 = (u0 + 15) & ~uintptr_t(15), v1 = u1 & ~uintptr_t(15);
  const unsigned tid = threadIdx.x;
  if (v0 >= v1) {
    for (uint64_t i = tid; i < n; i += NT) {
      const double x = elem_f64<DT>(u0 + i * ES);
      acc = fma(x, x, acc);
    }
    return;
  }
  const unsigned nhead = (unsigned)((v0 - u0) / ES);
  const unsigned ntail = (unsigned)((u1 - v1) / ES);
  if (tid < nhead) {
    const double x = elem_f64<DT>(u0 + tid * ES);
    acc = fma(x, x, acc);
  }
  if (tid < ntail) {
    const double x = elem_f64<DT>(v1 + tid * ES);
    acc = fma(x, x, acc);
  }
  const uint4* __restrict__ vp = reinterpret_cast<const uint4*>(v0);
  const uint64_t nv = (v1 - v0) >> 4;
  if (nv == (uint64_t)U * NT) {
    // a full aligned chunk (the common case): U unguarded loads in flight
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) r[j] = ld_stream(vp + tid + j * NT);
#pragma unroll
    for (int j = 0; j < U; ++j) vacc<DT>(r[j], acc);
    return;
  }
  // partial / misaligned piece: all U loads of an iteration still issue
  // back to back (predicated), so the piece keeps its MLP
  for (uint64_t i = tid; i < nv; i += (uint64_t)U * NT) {
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      r[j] = (i + (uint64_t)j * NT < nv) ? ld_stream(vp + i + (uint64_t)j * NT)
                                          : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int j = 0; j < U; ++j) vacc<DT>(r[j], acc);
  }
}

// ---------------------------------------------------------------- K1

// Interleaved chunks: the window of active elements is cut into chunks of
// U*NT vectors and chunk c goes to CTA c mod G, so all CTAs sweep HBM
// together (measured 7.35 TB/s read vs 6.5 TB/s for contiguous per-CTA
// shares, tools/bw_sweep.cu).  The assignment is static, so results stay
// bit-reproducible.
template <int DT, int NT, int U, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    sqnorm_kernel(const Range* __restrict__ R, int nr, Window w,
                  const BatchArgs jobs, Sink sink) {
  __shared__ double red[32];
  constexpr uint64_t CE = (uint64_t)U * NT * (16 / Elem<DT>::kSize);
  const uint64_t n = w.e_end - w.e_begin;
  const uint64_t nchunks = (n + CE - 1) / CE;
  for (int b = 0; b < jobs.count; ++b) {
    const uintptr_t base = reinterpret_cast<uintptr_t>(jobs.ptr[b]);
    double total = 0.0;
    int k = 0;  // range cursor: chunks of this CTA only move forward
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      const uint64_t e0 = w.e_begin + c * CE;
      const uint64_t e1 = min(e0 + CE, w.e_end);
      while (k + 1 < nr && R[k + 1].cum_begin <= e0) ++k;
      for (int kk = k; kk < nr && R[kk].cum_begin < e1; ++kk) {
        const uint64_t cb = R[kk].cum_begin, ce = cb + R[kk].len;
        const uint64_t s = cb > e0 ? cb : e0, e = ce < e1 ? ce : e1;
        if (s >= e) continue;
        double acc = 0.0;
        piece_sumsq<DT, NT, U>(base, R[kk].abs_begin + (s - cb), e - s, acc);
        total += R[kk].weight == 1.0 ? acc : R[kk].weight * acc;
      }
    }
    total = block_sum<NT>(total, red);
    if (threadIdx.x == 0)
      sink.partials[(size_t)b * gridDim.x + blockIdx.x] = total;
  }
  last_cta_combine<NT>(sink, jobs.count, jobs.slot, nullptr, red);
}

// ---------------------------------------------------------------- K1f

// M streams at the same element positions (all M pointers are congruent
// mod 16, checked by the host).  acc[m] += x_m^2; gacc += (sum_m x_m)^2
// with the sum in fp32, micro-batches in order (Megatron main_grad).
template <int DT, int M, int NT, int UP>
__device__ __forceinline__ void fused_piece(const FusedArgs& args, uint64_t a,
                                            uint64_t n, double* acc,
                                            double& gacc) {
  constexpr int ES = Elem<DT>::kSize;
  constexpr int PV = Elem<DT>::kPerVec;
  const uintptr_t b0 = reinterpret_cast<uintptr_t>(args.ptr[0]);
  const uintptr_t u0 = b0 + a * ES, u1 = u0 + n * ES;
  uintptr_t v0 = (u0 + 15) & ~uintptr_t(15);
  uintptr_t v1 = u1 & ~uintptr_t(15);
  const unsigned tid = threadIdx.x;
  auto scalar = [&](uint64_t i) {  // element at u0-relative byte offset i
    float sum = 0.0f;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uintptr_t p =
          reinterpret_cast<uintptr_t>(args.ptr[m]) + (u0 - b0) + i;
      const float x = elem_f32<DT>(p);
      const double xd = x;
      acc[m] = fma(xd, xd, acc[m]);
      sum = __fadd_rn(sum, x);
    }
    const double sd = sum;
    gacc = fma(sd, sd, gacc);
  };
  if (v0 >= v1) {
    for (uint64_t i = tid; i < n; i += NT) scalar(i * ES);
    return;
  }
  const unsigned nhead = (unsigned)((v0 - u0) / ES);
  const unsigned ntail = (unsigned)((u1 - v1) / ES);
  if (tid < nhead) scalar((uint64_t)tid * ES);
  if (tid < ntail) scalar((v1 - u0) + (uint64_t)tid * ES);
  const uint64_t nv = (v1 - v0) >> 4;
  const uint64_t voff = v0 - b0;  // byte offset of the first vector
  uint64_t i = tid;
  for (; i + (uint64_t)(UP - 1) * NT < nv; i += (uint64_t)UP * NT) {
    uint4 r[UP][M];
#pragma unroll
    for (int p = 0; p < UP; ++p)
#pragma unroll
      for (int m = 0; m < M; ++m)
        r[p][m] = ld_stream(reinterpret_cast<const uint4*>(
            reinterpret_cast<uintptr_t>(args.ptr[m]) + voff +
            (i + (uint64_t)p * NT) * 16));
#pragma unroll
    for (int p = 0; p < UP; ++p) {
      float sum[PV];
#pragma unroll
      for (int e = 0; e < PV; ++e) sum[e] = 0.0f;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        vacc<DT>(r[p][m], acc[m]);
        micro_add<DT>(r[p][m], sum);
      }
#pragma unroll
      for (int e = 0; e < PV; ++e) {
        const double sd = sum[e];
        gacc = fma(sd, sd, gacc);
      }
    }
  }
  for (; i < nv; i += NT) {
    float sum[PV];
#pragma unroll
    for (int e = 0; e < PV; ++e) sum[e] = 0.0f;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const uint4 v = ld_stream(reinterpret_cast<const uint4*>(
          reinterpret_cast<uintptr_t>(args.ptr[m]) + voff + i * 16));
      vacc<DT>(v, acc[m]);
      micro_add<DT>(v, sum);
    }
#pragma unroll
    for (int e = 0; e < PV; ++e) {
      const double sd = sum[e];
      gacc = fma(sd, sd, gacc);
    }
  }
}

template <int DT, int M, int NT, int UP>
__global__ void __launch_bounds__(NT)
    fused_kernel(const Range* __restrict__ R, int nr, Window w,
                 const FusedArgs args, Sink sink) {
  __shared__ double red[32];
  __shared__ int32_t out_slot[M + 1];
  __shared__ double out_scale[M + 1];
  uint64_t e0, e1;
  cta_share(w, e0, e1);
  double total[M], gtotal = 0.0;
#pragma unroll
  for (int m = 0; m < M; ++m) total[m] = 0.0;
  if (e0 < e1) {
    for (int k = find_range(R, nr, e0); k < nr && R[k].cum_begin < e1; ++k) {
      const uint64_t cb = R[k].cum_begin, ce = cb + R[k].len;
      const uint64_t s = cb > e0 ? cb : e0, e = ce < e1 ? ce : e1;
      if (s >= e) continue;
      double acc[M], gacc = 0.0;
#pragma unroll
      for (int m = 0; m < M; ++m) acc[m] = 0.0;
      fused_piece<DT, M, NT, UP>(args, R[k].abs_begin + (s - cb), e - s, acc,
                                 gacc);
      const double wt = R[k].weight;
#pragma unroll
      for (int m = 0; m < M; ++m) total[m] += wt == 1.0 ? acc[m] : wt * acc[m];
      gtotal += wt == 1.0 ? gacc : wt * gacc;
    }
  }
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const double v = block_sum<NT>(total[m], red);
    if (threadIdx.x == 0)
      sink.partials[(size_t)m * gridDim.x + blockIdx.x] = v;
  }
  {
    const double v = block_sum<NT>(gtotal, red);
    if (threadIdx.x == 0)
      sink.partials[(size_t)M * gridDim.x + blockIdx.x] = v;
  }
  if (threadIdx.x <= M) {
    out_slot[threadIdx.x] =
        threadIdx.x < M ? args.slot0 + (int)threadIdx.x : args.gslot;
    out_scale[threadIdx.x] = threadIdx.x < M ? 1.0 : args.gscale;
  }
  last_cta_combine<NT>(sink, M + 1, out_slot, out_scale, red);
}

// ---------------------------------------------------------------- K1f (TMA)
//
// The B200 form of the fused pass.  Bytes in flight are decoupled from
// registers: warp 0 (one elected lane) streams each chunk's M tiles into a
// 3-stage shared-memory ring with cp.async.bulk (TMA, SASS UBLKCP) signalled
// on an mbarrier; 8 consumer warps square/sum from shared memory and release
// the stage.  A chunk is the intersection of one range with an absolutely
// aligned P-element window, so every interior copy is 16-byte aligned and a
// chunk has one weight; the <16-byte edges of a range are read from global
// memory directly.  Chunk c goes to CTA c mod G (interleaved sweep).

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)),
               "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src,
                                         uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Shape variants of the fused TMA kernel: (consumer warps, stage bytes).
template <int V> struct TmaShape;
template <> struct TmaShape<0> { static constexpr int NW = 12, kStageBytes = 49152; };
template <> struct TmaShape<1> { static constexpr int NW = 16, kStageBytes = 49152; };
template <> struct TmaShape<2> { static constexpr int NW = 8, kStageBytes = 32768; };
template <> struct TmaShape<3> { static constexpr int NW = 8, kStageBytes = 49152; };
template <> struct TmaShape<4> { static constexpr int NW = 16, kStageBytes = 57344; };
// 14 consumer warps: a 3584 B tile (M = 16) is exactly 224 vectors, one per
// thread of a 7-warp group
template <> struct TmaShape<5> { static constexpr int NW = 14, kStageBytes = 57344; };

template <int DT, int M, int V = 0>
struct TmaCfg {
  static constexpr int ES = Elem<DT>::kSize;
  static constexpr int PV = Elem<DT>::kPerVec;
  // 4 stages; chunk i -> stage i % 4 and consumer group i % 2, so every
  // stage is always drained by the same group and each group observes every
  // mbarrier phase of its stages (parity waits cannot alias).
  static constexpr int kStages = 4;
  // tiles a multiple of 256 B
  static constexpr int kTile = (TmaShape<V>::kStageBytes / M) & ~255;
  static constexpr int P = kTile / ES;  // elements per chunk
  static constexpr int kStage = kTile * M;
  static constexpr int kSmem = kStages * kStage;
  static constexpr int NW = TmaShape<V>::NW;  // consumer warps: 2 groups
  static constexpr int CT = NW * 32;
  static constexpr int NT = CT + 32;    // + 1 producer warp
  static_assert(kStages % 2 == 0, "stages must split evenly between the groups");
};

struct ChunkMeta {
  uint64_t a;   // first element (absolute)
  uint32_t n;   // elements in the chunk
  uint32_t pad;
  double w;     // range weight
};

// Element i (absolute) of micro-bucket m, as fp32 (edges of a chunk).
template <int DT>
__device__ __forceinline__ float elem_at(const FusedArgs& args, int m,
                                         uint64_t i) {
  return elem_f32<DT>(reinterpret_cast<uintptr_t>(args.ptr[m]) +
                      i * Elem<DT>::kSize);
}

// One chunk, one consumer group (GT threads): each thread owns whole
// positions (16-byte columns across the M tiles): acc[m] += x_m^2 in fp64
// and the M values of each element are summed in micro-batch order in fp32
// (Megatron main_grad order), the sum squared in fp64.  The <16-byte edges
// of a range come from global memory.
template <int DT, int M, int V, int GT, bool WEIGHTED, bool MEAN>
__device__ __forceinline__ void tma_consume_cols(const char* stage,
                                                 const FusedArgs& args,
                                                 const ChunkMeta& cm, int gt,
                                                 double* acc, double& gacc) {
  using C = TmaCfg<DT, M, V>;
  constexpr int VE = 16 / C::ES;
  const uint64_t a = cm.a, b = cm.a + cm.n;
  uint64_t A0 = (a + VE - 1) / VE * VE, A1 = b / VE * VE;
  if (A1 <= A0) A0 = A1 = b;  // no aligned interior
  const int nhead = (int)(A0 - a), ntail = (int)(b - A1);
  const int nv = (int)((A1 - A0) / VE);
  const double w = cm.w;
  for (int v = gt; v < nv; v += GT) {
    float sum[C::PV];
#pragma unroll
    for (int e = 0; e < C::PV; ++e) sum[e] = 0.0f;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      // volatile: keeps the M shared-memory loads in program order instead of
      // hoisting all of them (register pressure, 12 warps hide the latency)
      uint4 x;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                   : "r"(smem_u32(stage + m * C::kTile + v * 16)));
      if constexpr (WEIGHTED) {
        double t = 0.0;
        vacc<DT>(x, t);
        acc[m] = fma(w, t, acc[m]);
      } else {
        vacc<DT>(x, acc[m]);
      }
      if constexpr (MEAN) micro_add<DT>(x, sum);
    }
    if constexpr (MEAN) {
      double g = 0.0;
#pragma unroll
      for (int e = 0; e < C::PV; ++e) {
        const double sd = sum[e];
        g = fma(sd, sd, g);
      }
      gacc = WEIGHTED ? fma(w, g, gacc) : gacc + g;
    }
  }
  for (int q = gt; q < nhead + ntail; q += GT) {
    const uint64_t i = q < nhead ? a + q : A1 + (q - nhead);
    float sum = 0.0f;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const float x = elem_at<DT>(args, m, i);
      const double xd = x;
      acc[m] = fma(WEIGHTED ? w * xd : xd, xd, acc[m]);
      sum = __fadd_rn(sum, x);
    }
    if constexpr (MEAN) {
      const double sd = sum;
      gacc = fma(WEIGHTED ? w * sd : sd, sd, gacc);
    }
  }
}

template <int DT, int M, int V, bool MEAN>
__global__ void __launch_bounds__(TmaCfg<DT, M, V>::NT, 1)
    fused_tma_kernel(const Range* __restrict__ R, int nr,
                     const uint64_t* __restrict__ prefix, uint64_t c_begin,
                     uint64_t c_end, const FusedArgs args, Sink sink,
                     const __grid_constant__ Tail tail) {
  // Two consumer groups of NW/2 warps take alternate chunks; every thread
  // owns whole positions of a chunk (tma_consume_cols), so per-thread state
  // is M fp64 accumulators and nothing is read twice from shared memory.
  using C = TmaCfg<DT, M, V>;
  constexpr int GW = C::NW / 2;  // warps per chunk
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint64_t full[C::kStages], empty[C::kStages];
  __shared__ ChunkMeta meta[C::kStages];
  __shared__ double red[32];
  __shared__ int32_t out_slot[M + 1];
  __shared__ double out_scale[M + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t G = gridDim.x;
  // !MEAN: batched K1 over M buckets sharing the layout (no mean term)
  double acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = 0.0;
  double gtotal = 0.0;
  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      uint64_t i = 0;
      for (uint64_t c = c_begin + blockIdx.x; c < c_end; c += G, ++i) {
        const int st = (int)(i % C::kStages);
        if (i >= (uint64_t)C::kStages)
          mbar_wait(&empty[st], (uint32_t)(((i / C::kStages) - 1) & 1));
        while (k + 1 < nr && prefix[k + 1] <= c) ++k;
        const uint64_t rb = R[k].abs_begin, re = rb + R[k].len;
        const uint64_t j = rb / C::P + (c - prefix[k]);
        const uint64_t a = max(rb, j * C::P), b = min(re, (j + 1) * C::P);
        meta[st] = ChunkMeta{a, (uint32_t)(b - a), 0u, R[k].weight};
        constexpr int VE = 16 / C::ES;
        const uint64_t A0 = (a + VE - 1) / VE * VE, A1 = b / VE * VE;
        char* dst = smem + st * C::kStage;
        if (A1 > A0) {
          const uint32_t bytes = (uint32_t)((A1 - A0) * C::ES);
          mbar_arrive_tx(&full[st], bytes * M);
#pragma unroll 1
          for (int m = 0; m < M; ++m)
            bulk_g2s(dst + m * C::kTile,
                     static_cast<const char*>(args.ptr[m]) + A0 * C::ES, bytes,
                     &full[st]);
        } else {
          mbar_arrive(&full[st]);
        }
      }
    }
  } else {
    const int grp = (warp - 1) / GW;
    const int gt = ((warp - 1) % GW) * 32 + lane;
    uint64_t i = grp;
    for (uint64_t c = c_begin + blockIdx.x + grp * G; c < c_end; c += 2 * G, i += 2) {
      const int st = (int)(i % C::kStages);
      mbar_wait(&full[st], (uint32_t)((i / C::kStages) & 1));
      const ChunkMeta cm = meta[st];
      if (cm.w == 1.0)
        tma_consume_cols<DT, M, V, GW * 32, false, MEAN>(smem + st * C::kStage, args, cm,
                                                      gt, acc, gtotal);
      else
        tma_consume_cols<DT, M, V, GW * 32, true, MEAN>(smem + st * C::kStage, args, cm,
                                                     gt, acc, gtotal);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const double v = block_sum<C::NT>(acc[m], red);
    if (threadIdx.x == 0) sink.partials[(size_t)m * G + blockIdx.x] = v;
  }
  if constexpr (MEAN) {
    const double v = block_sum<C::NT>(gtotal, red);
    if (threadIdx.x == 0) sink.partials[(size_t)M * G + blockIdx.x] = v;
  }
  if (threadIdx.x <= M) {
    out_slot[threadIdx.x] =
        threadIdx.x < M ? args.slot0 + (int)threadIdx.x : args.gslot;
    out_scale[threadIdx.x] = threadIdx.x < M ? 1.0 : args.gscale;
  }
  const bool last =
      last_cta_combine<C::NT>(sink, MEAN ? M + 1 : M, out_slot, out_scale, red);
  if (tail.mode == 0 || !last) return;
  // the step's last reduction: this CTA holds the final slots (its own
  // thread 0 wrote them; earlier launches are stream-ordered before it)
  __syncthreads();
  if (tail.mode == 2)
    p2p_exchange_finalize(tail.p2p);
  else if (threadIdx.x == 0)
    finalize_body(tail.p2p.fin);
}

// ---------------------------------------------------------------- KA
//
// Trainer form: the gradient-accumulation add a trainer
// performs anyway (Megatron: main_grad.add_(grad), fp32) with s_m fused in,
// and, on the last micro-batch of a d = 1 step, gbar^2 from the updated
// main_grad.  The norm then costs no HBM bytes beyond the accumulation's
// own (read g, read+write main_grad).  The table covers the WHOLE bucket
// (weight-0 ranges and gaps included): every element is accumulated, only
// weighted ones are counted.

__device__ __forceinline__ uint4 ld_rw(const uint4* p) {  // main_grad: read+write
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

#ifndef COADAPT_KA_NO_NORM
#define COADAPT_KA_NO_NORM 0
#endif
template <int DT>
__device__ __forceinline__ void accum_elem(float* mg, float g, double w,
                                           bool first, bool mean, double& s,
                                           double& gm) {
  const float nv = first ? g : __fadd_rn(*mg, g);
  *mg = nv;
  if (w != 0.0) {
    const double gd = g, nd = nv;
    s = fma(w * gd, gd, s);
    if (mean) gm = fma(w * nd, nd, gm);
  }
}

template <int DT, int NT, int U, bool FIRST>
__global__ void __launch_bounds__(NT, 3)
    accum_kernel(const Range* __restrict__ R, int nr, uint64_t numel,
                 float* __restrict__ mg, const void* __restrict__ gp, int flags,
                 int32_t slot, int32_t gslot, double gscale, Sink sink) {
  static_assert(DT == COADAPT_BF16 || DT == COADAPT_FP16 || DT == COADAPT_FP32, "");
  constexpr int ES = Elem<DT>::kSize, PV = Elem<DT>::kPerVec;
  constexpr uint64_t CE = (uint64_t)U * NT * PV;  // elements per chunk
  __shared__ double red[32];
  // the first micro-batch only reads the gradient (main_grad is written,
  // not read): its own instantiation keeps twice the loads in flight
  constexpr bool first = FIRST;
  const bool mean = flags & 2;
  const uint64_t nchunks = (numel + CE - 1) / CE;
  double s = 0.0, gm = 0.0;
  int k = 0;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t e0 = c * CE, e1 = min(e0 + CE, numel);
    while (k + 1 < nr && R[k + 1].abs_begin <= e0) ++k;
    for (int kk = k; kk < nr && R[kk].abs_begin < e1; ++kk) {
      const uint64_t a = max(R[kk].abs_begin, e0);
      const uint64_t b = min(R[kk].abs_begin + R[kk].len, e1);
      if (a >= b) continue;
      const double w = R[kk].weight;
      // vectors of PV elements aligned on the element index (both buffers are
      // 16-byte aligned, checked by the host), edges element by element
      const uint64_t A0 = (a + PV - 1) / PV * PV, A1 = b / PV * PV;
      const char* gb = static_cast<const char*>(gp);
      if (A1 <= A0) {
        for (uint64_t i = a + threadIdx.x; i < b; i += NT)
          accum_elem<DT>(mg + i, elem_f32<DT>(reinterpret_cast<uintptr_t>(gb + i * ES)),
                         w, first, mean, s, gm);
        continue;
      }
      if (a + threadIdx.x < A0) {
        const uint64_t i = a + threadIdx.x;
        accum_elem<DT>(mg + i, elem_f32<DT>(reinterpret_cast<uintptr_t>(gb + i * ES)), w,
                       first, mean, s, gm);
      }
      if (A1 + threadIdx.x < b) {
        const uint64_t i = A1 + threadIdx.x;
        accum_elem<DT>(mg + i, elem_f32<DT>(reinterpret_cast<uintptr_t>(gb + i * ES)), w,
                       first, mean, s, gm);
      }
      const uint64_t nv = (A1 - A0) / PV;
      const uint4* gv = reinterpret_cast<const uint4*>(gb + A0 * ES);
      uint4* mv = reinterpret_cast<uint4*>(mg + A0);  // PV floats = PV/4 uint4
      // two register sets, software-pipelined: the loads of the next set
      // are in flight while this one is converted, reduced and stored (the
      // unpipelined loop drained the memory pipe every iteration: ncu
      // long-scoreboard bound)
      auto load_set = [&](uint64_t v0, uint4(&gr)[U], uint4(&mr)[U][PV / 4]) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const uint64_t v = v0 + (uint64_t)j * NT;
          if (v < nv) {
            gr[j] = ld_stream(gv + v);
#pragma unroll
            for (int h = 0; h < PV / 4; ++h)
              mr[j][h] = first ? make_uint4(0u, 0u, 0u, 0u) : ld_rw(mv + v * (PV / 4) + h);
          }
        }
      };
      auto process_set = [&](uint64_t v0, uint4(&gr)[U], uint4(&mr)[U][PV / 4]) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const uint64_t v = v0 + (uint64_t)j * NT;
          if (v >= nv) continue;
          float* mf = reinterpret_cast<float*>(mr[j]);
          double a0 = 0.0, a1 = 0.0, m0 = 0.0, m1 = 0.0;
          float f[PV];
          if constexpr (DT != COADAPT_BF16) unpack<DT>(gr[j], f);
          const uint32_t gw[4] = {gr[j].x, gr[j].y, gr[j].z, gr[j].w};
#pragma unroll
          for (int e = 0; e < PV; ++e) {
            float nvf;
            double gd;
            if constexpr (DT == COADAPT_BF16) {
              // bf16 halves read in place: FHADD.BF16 for the fp32 add (one
              // rounding, == __fadd_rn), F2F.F64.BF16 for the square
              const uint16_t h = (e & 1) ? (uint16_t)(gw[e >> 1] >> 16)
                                         : (uint16_t)(gw[e >> 1] & 0xffffu);
              nvf = first ? __uint_as_float((uint32_t)h << 16) : bf16_addf(mf[e], h);
              gd = bf16_f64(h);
            } else {
              nvf = first ? f[e] : __fadd_rn(mf[e], f[e]);
              gd = f[e];
            }
            mf[e] = nvf;
#if !COADAPT_KA_NO_NORM  // (1: the plain accumulation, for the overhead A/B)
            if (e & 1) a1 = fma(gd, gd, a1); else a0 = fma(gd, gd, a0);
            if (mean) {
              const double nd = nvf;
              if (e & 1) m1 = fma(nd, nd, m1); else m0 = fma(nd, nd, m0);
            }
#else
            (void)gd;
#endif
          }
#pragma unroll
          for (int h = 0; h < PV / 4; ++h) st_stream(mv + v * (PV / 4) + h, mr[j][h]);
          if (w != 0.0) {
            s = fma(w, a0 + a1, s);
            if (mean) gm = fma(w, m0 + m1, gm);
          }
        }
      };
      constexpr uint64_t kStep = (uint64_t)U * NT;
      uint4 gx[U], mx[U][PV / 4], gy[U], my[U][PV / 4];
      uint64_t v0 = threadIdx.x;
      if (v0 < nv) load_set(v0, gx, mx);
      while (v0 < nv) {
        if (v0 + kStep < nv) load_set(v0 + kStep, gy, my);
        process_set(v0, gx, mx);
        v0 += kStep;
        if (v0 >= nv) break;
        if (v0 + kStep < nv) load_set(v0 + kStep, gx, mx);
        process_set(v0, gy, my);
        v0 += kStep;
      }
    }
  }
  const double vs = block_sum<NT>(s, red);
  if (threadIdx.x == 0) sink.partials[blockIdx.x] = vs;
  const double vg = block_sum<NT>(gm, red);
  if (threadIdx.x == 0) sink.partials[gridDim.x + blockIdx.x] = vg;
  __shared__ int32_t out_slot[2];
  __shared__ double out_scale[2];
  if (threadIdx.x == 0) {
    out_slot[0] = slot;
    out_slot[1] = gslot;
    out_scale[0] = 1.0;
    out_scale[1] = gscale;
  }
  last_cta_combine<NT>(sink, mean ? 2 : 1, out_slot, out_scale, red);
}

// ---------------------------------------------------------------- KR
//
// Fused DP reduce-scatter + mean-gradient norm over NVLink (SURVEY §8f row
// f2).  DP replica q's accumulated gradient bucket is mapped into this
// process (CUDA IPC peer pointer, or local for q == this rank); for every
// element of this rank's slice [lo, hi):
//   out[i - lo] = RNE_dtype( scale * fp32( sum_{q = 0..d-1} rep_q[i] ) )
// (replicas summed in fixed order) and gbar^2 += w * out^2 in fp64 — the
// synchronised mean gradient is produced and its norm taken in ONE pass, the
// loads coming straight from the peers' HBM over NVLink.  All-reduce form
// (inplace): the result is stored back into slice [lo, hi) of EVERY replica
// instead of `out` — the reduce-scatter and the all-gather of a DDP gradient
// all-reduce in the same pass (each element read once per replica and
// written once per replica, (d-1)/d of both over NVLink: the ring optimum),
// safe because only this rank ever touches [lo, hi) of any replica.

__device__ __forceinline__ uint4 ld_peer(const uint4* p) {  // no .nc on peer memory
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int DT>
__device__ __forceinline__ void pack(const float* f, uint4& v);
template <>
__device__ __forceinline__ void pack<COADAPT_BF16>(const float* f, uint4& v) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  v = make_uint4(w[0], w[1], w[2], w[3]);
}
template <>
__device__ __forceinline__ void pack<COADAPT_FP16>(const float* f, uint4& v) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  v = make_uint4(w[0], w[1], w[2], w[3]);
}
template <>
__device__ __forceinline__ void pack<COADAPT_FP32>(const float* f, uint4& v) {
  v = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]),
                 __float_as_uint(f[2]), __float_as_uint(f[3]));
}

template <int DT>
__device__ __forceinline__ float round_dt(float x) {
  if constexpr (DT == COADAPT_BF16) return __bfloat162float(__float2bfloat16_rn(x));
  else if constexpr (DT == COADAPT_FP16) return __half2float(__float2half_rn(x));
  else return x;
}

template <int DT>
__device__ __forceinline__ void store_dt(char* base, uint64_t i, float x) {
  if constexpr (DT == COADAPT_BF16)
    reinterpret_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(x);
  else if constexpr (DT == COADAPT_FP16)
    reinterpret_cast<__half*>(base)[i] = __float2half_rn(x);
  else
    reinterpret_cast<float*>(base)[i] = x;
}

// NVLS forms of the loads and stores (fp32 only: the switch adds in fp32)
__device__ __forceinline__ uint4 mm_ld_reduce_v4(const void* p) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ float mm_ld_reduce_f32(const void* p) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];"
               : "=f"(r)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ void mm_st_v4(void* p, const uint4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st_f32(void* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// NVLS = true: the d replicas are one multicast object (the DP group's fp32
// buckets bound to it, coadapt_nvls_*); every load of the slice is one
// multimem.ld_reduce (the NVSwitch sums the d copies: each GPU's link carries
// its slice once instead of (d-1)/d of the bucket), the all-reduce form stores
// through the multicast address, and gbar^2 is taken from the registers in
// the same pass.
template <int DT, int NT, int U, bool NVLS = false>
__global__ void __launch_bounds__(NT, 2)
    rs_kernel(const Range* __restrict__ R, int nr, uint64_t lo, uint64_t hi,
              const __grid_constant__ RSArgs a, Sink sink) {
  constexpr int ES = Elem<DT>::kSize, PV = Elem<DT>::kPerVec;
  constexpr uint64_t CE = (uint64_t)U * NT * PV;
  __shared__ double red[32];
  const uint64_t n = hi - lo, nchunks = (n + CE - 1) / CE;
  char* out = static_cast<char*>(a.out);
  double g = 0.0;
  int k = 0;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint64_t e0 = lo + c * CE, e1 = min(e0 + CE, hi);
    while (k + 1 < nr && R[k + 1].abs_begin <= e0) ++k;
    for (int kk = k; kk < nr && R[kk].abs_begin < e1; ++kk) {
      const uint64_t pa = max(R[kk].abs_begin, e0);
      const uint64_t pb = min(R[kk].abs_begin + R[kk].len, e1);
      if (pa >= pb) continue;
      const double w = R[kk].weight;
      const uint64_t A0 = (pa + PV - 1) / PV * PV, A1 = pb / PV * PV;
      auto scalar = [&](uint64_t i) {
        float s = 0.0f;
        if constexpr (NVLS) {
          s = mm_ld_reduce_f32(static_cast<const char*>(a.mc) + i * ES);
        } else {
          for (int q = 0; q < a.d; ++q)
            s = __fadd_rn(s, elem_f32<DT>(reinterpret_cast<uintptr_t>(a.rep[q]) + i * ES));
        }
        const float o = round_dt<DT>(__fmul_rn(s, a.scale));
        if (a.inplace) {
          if constexpr (NVLS) {
            mm_st_f32(static_cast<char*>(const_cast<void*>(a.mc)) + i * ES, o);
          } else {
            for (int q = 0; q < a.d; ++q)
              store_dt<DT>(static_cast<char*>(const_cast<void*>(a.rep[q])), i, o);
          }
        } else {
          store_dt<DT>(out, i - lo, o);
        }
        const double od = o;
        g = fma(w * od, od, g);
      };
      if (A1 <= A0) {
        for (uint64_t i = pa + threadIdx.x; i < pb; i += NT) scalar(i);
        continue;
      }
      if (pa + threadIdx.x < A0) scalar(pa + threadIdx.x);
      if (A1 + threadIdx.x < pb) scalar(A1 + threadIdx.x);
      const uint64_t nv = (A1 - A0) / PV;
      for (uint64_t v0 = threadIdx.x; v0 < nv; v0 += (uint64_t)U * NT) {
        float sum[U][PV];
#pragma unroll
        for (int j = 0; j < U; ++j)
#pragma unroll
          for (int e = 0; e < PV; ++e) sum[j][e] = 0.0f;
        for (int q = 0; q < (NVLS ? 1 : a.d); ++q) {
          uint4 r[U];
          if constexpr (NVLS) {
            const uint4* src = reinterpret_cast<const uint4*>(
                static_cast<const char*>(a.mc) + A0 * ES);
#pragma unroll
            for (int j = 0; j < U; ++j) {
              const uint64_t v = v0 + (uint64_t)j * NT;
              r[j] = v < nv ? mm_ld_reduce_v4(src + v) : make_uint4(0u, 0u, 0u, 0u);
            }
          } else {
            const uint4* src = reinterpret_cast<const uint4*>(
                static_cast<const char*>(a.rep[q]) + A0 * ES);
#pragma unroll
            for (int j = 0; j < U; ++j) {
              const uint64_t v = v0 + (uint64_t)j * NT;
              r[j] = v < nv ? ld_peer(src + v) : make_uint4(0u, 0u, 0u, 0u);
            }
          }
#pragma unroll
          for (int j = 0; j < U; ++j) {
            float f[PV];
            unpack<DT>(r[j], f);
#pragma unroll
            for (int e = 0; e < PV; ++e) sum[j][e] = __fadd_rn(sum[j][e], f[e]);
          }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const uint64_t v = v0 + (uint64_t)j * NT;
          if (v >= nv) continue;
          float o[PV];
          double gl = 0.0;
#pragma unroll
          for (int e = 0; e < PV; ++e) {
            o[e] = round_dt<DT>(__fmul_rn(sum[j][e], a.scale));
            const double od = o[e];
            gl = fma(od, od, gl);
          }
          uint4 ov;
          pack<DT>(o, ov);
          if (a.inplace) {
            // all-reduce form: this rank owns [lo, hi) of every replica, so
            // the position it just read is written back nowhere else
            if constexpr (NVLS) {
              mm_st_v4(reinterpret_cast<uint4*>(static_cast<char*>(const_cast<void*>(a.mc)) +
                                                A0 * ES) + v, ov);
            } else {
              for (int q = 0; q < a.d; ++q)
                st_stream(reinterpret_cast<uint4*>(
                              static_cast<char*>(const_cast<void*>(a.rep[q])) + A0 * ES) + v,
                          ov);
            }
          } else {
            st_stream(reinterpret_cast<uint4*>(out + (A0 - lo) * ES) + v, ov);
          }
          g = fma(w, gl, g);
        }
      }
    }
  }
  if constexpr (NVLS) {
    // the multicast stores must be visible system-wide before the peers'
    // stream-ordered barrier lets them read
    asm volatile("fence.proxy.alias;" ::: "memory");
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  }
  const double vg = block_sum<NT>(g, red);
  if (threadIdx.x == 0) sink.partials[blockIdx.x] = vg;
  __shared__ int32_t out_slot[1];
  if (threadIdx.x == 0) out_slot[0] = a.gslot;
  last_cta_combine<NT>(sink, 1, out_slot, nullptr, red);
}

// ---------------------------------------------------------------- K3

struct DevState {  // == coadapt_gns_state
  double ema_signal, ema_noise, alpha_early, alpha_late;
  int64_t phase_boundary_tokens, tokens_seen;
  double calibration;
  int32_t initialized, reserved_;
};
struct DevResult {  // == coadapt_gns_result
  double signal, noise, noise_raw, mean_grad_sq;
  DevState state;
  double phi, b_simple;
  int64_t sample_count;
  int32_t phi_available, status;
};
static_assert(sizeof(DevState) == sizeof(coadapt_gns_state), "layout");
static_assert(sizeof(DevResult) == sizeof(coadapt_gns_result), "layout");

// Single thread, explicit round-to-nearest intrinsics: no FMA contraction,
// so every value is bit-identical to the host C++ formulas
// (gns.hpp:42-44, 64-66, 70-72).
__device__ void finalize_body(const FinalizeArgs& a) {
  DevState* st = static_cast<DevState*>(a.state);
  DevResult* res = static_cast<DevResult*>(a.result);
  const int n = a.n;
  double sum = 0.0;
  bool ok = n >= 2;
  for (int i = 0; i < n; ++i) {
    const double s = a.slots[i];
    ok = ok && (s >= 0.0) && isfinite(s);  // gns.hpp:19: negative rejected
    sum = __dadd_rn(sum, s);
  }
  const double g2 = a.slots[n];
  ok = ok && (g2 >= 0.0) && isfinite(g2);
  res->sample_count = n;
  if (!ok) {
    res->status = COADAPT_E_VALIDATION;
    res->state = *st;
    res->phi_available = 0;
    res->phi = __longlong_as_double(0x7ff8000000000000ll);
    res->signal = res->noise = res->noise_raw = 0.0;
    res->mean_grad_sq = g2;
    res->b_simple = res->phi;
    return;
  }
  const double N = (double)n;
  const double nm1 = __dsub_rn(N, 1.0);
  const double sbar = __ddiv_rn(sum, N);
  const double signal = __ddiv_rn(__dsub_rn(__dmul_rn(N, g2), sbar), nm1);
  const double noise_raw = __ddiv_rn(
      __dmul_rn(__dsub_rn(sbar, g2), (double)a.global_batch), nm1);
  const double noise = noise_raw > 0.0 ? noise_raw : 0.0;
  // update_ema: alpha from tokens_seen before the increment
  DevState s = *st;
  const double alpha =
      s.tokens_seen < s.phase_boundary_tokens ? s.alpha_early : s.alpha_late;
  if (!s.initialized) {
    s.ema_signal = signal;
    s.ema_noise = noise;
    s.initialized = 1;
  } else {
    const double beta = __dsub_rn(1.0, alpha);
    s.ema_signal =
        __dadd_rn(__dmul_rn(alpha, s.ema_signal), __dmul_rn(beta, signal));
    s.ema_noise =
        __dadd_rn(__dmul_rn(alpha, s.ema_noise), __dmul_rn(beta, noise));
  }
  if (s.ema_noise < 0.0) s.ema_noise = 0.0;
  s.tokens_seen += a.tokens;
  *st = s;
  res->signal = signal;
  res->noise = noise;
  res->noise_raw = noise_raw;
  res->mean_grad_sq = g2;
  res->state = s;
  res->status = COADAPT_OK;
  res->b_simple = __ddiv_rn(noise, signal);
  if (s.ema_signal > 0.0) {
    res->phi = __ddiv_rn(__dmul_rn(s.calibration, s.ema_noise), s.ema_signal);
    res->phi_available = 1;
  } else {
    res->phi = __longlong_as_double(0x7ff8000000000000ll);
    res->phi_available = 0;
  }
}

__global__ void finalize_kernel(FinalizeArgs a) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  finalize_body(a);
}

// ---------------------------------------------------------------- X1+K3 P2P

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One CTA.  Blocks are double-buffered by epoch parity: a rank can be at
// most one epoch ahead of any reader (it needs every rank's flag of the
// current epoch before it can finish and start the next), so the block it
// overwrites next was read already.  A peer that never arrives turns into a
// status-2 result after timeout_ns instead of a hang.
__device__ void p2p_exchange_finalize(const P2PArgs& a) {
  const int nv = a.fin.n + 1, tid = threadIdx.x;
  const size_t data_doubles = (size_t)2 * a.world * a.cap;
  // the step counter lives in device memory after this rank's flags: every
  // launch (eager or a graph replay) takes the next epoch, the same on every
  // rank because every rank runs the same sequence of steps
  uint64_t* ctr = reinterpret_cast<uint64_t*>(
                      reinterpret_cast<double*>(a.mbox[a.rank]) + data_doubles) +
                  2 * a.world;
  __shared__ uint64_t s_epoch;
  if (tid == 0) s_epoch = *ctr + 1;
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int buf = (int)(epoch & 1);
  for (int q = 0; q < a.world; ++q) {
    double* dst = reinterpret_cast<double*>(a.mbox[q]) +
                  ((size_t)buf * a.world + a.rank) * a.cap;
    for (int i = tid; i < nv; i += blockDim.x) dst[i] = a.slots[i];
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    for (int q = 0; q < a.world; ++q) {
      uint64_t* f = reinterpret_cast<uint64_t*>(
                        reinterpret_cast<double*>(a.mbox[q]) + data_doubles) +
                    buf * a.world + a.rank;
      st_release_sys(f, epoch);
    }
  }
  __shared__ int timed_out;
  if (tid == 0) timed_out = 0;
  __syncthreads();
  const double* mine = reinterpret_cast<const double*>(a.mbox[a.rank]);
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(mine + data_doubles);
  if (tid < a.world) {
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(flags + buf * a.world + tid) < epoch) {
      if ((int64_t)(global_ns() - t0) > a.timeout_ns) {
        atomicExch(&timed_out, 1);
        break;
      }
      __nanosleep(64);
    }
    __threadfence_system();  // order this thread's acquire before the CTA's reads
  }
  __syncthreads();
  if (tid == 0) *ctr = epoch;  // nothing else in this launch reads it again
  if (timed_out) {
    if (tid == 0) {
      DevResult* res = static_cast<DevResult*>(a.fin.result);
      res->status = COADAPT_E_INTERNAL;
      res->sample_count = a.fin.n;
      res->phi_available = 0;
      res->phi = __longlong_as_double(0x7ff8000000000000ll);
      res->state = *static_cast<DevState*>(a.fin.state);
    }
    return;
  }
  for (int i = tid; i < nv; i += blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < a.world; ++q)
      v += mine[((size_t)buf * a.world + q) * a.cap + i];
    a.slots[i] = v;
  }
  __syncthreads();
  if (tid == 0) finalize_body(a.fin);
}

__global__ void __launch_bounds__(256) p2p_finalize_kernel(const __grid_constant__ P2PArgs a) {
  p2p_exchange_finalize(a);
}

// ---------------------------------------------------------------- K0

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t mix64_h(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t sample_key(uint64_t seed, uint64_t sample) {
  return mix64_h(seed ^ mix64_h(sample + 0x632BE59BD9B4E019ull));
}
inline uint64_t sign_key(uint64_t seed) {
  return mix64_h(seed ^ 0xA0761D6478BD642Full);
}

__device__ __forceinline__ float synth_value(uint64_t skey, uint64_t gkey,
                                             uint64_t gidx, float g0,
                                             float unit) {
  const uint64_t h = mix64(skey ^ gidx);
  const int32_t ih = (int32_t)((h & 0xffff) + ((h >> 16) & 0xffff) +
                               ((h >> 32) & 0xffff) + (h >> 48)) -
                     131070;
  const float zeta = __fmul_rn((float)ih, unit);
  const float g = (mix64(gkey ^ gidx) >> 63) ? -g0 : g0;
  return __fadd_rn(g, zeta);
}

__device__ __forceinline__ void store_elem(void* dst, int dtype, uint64_t i,
                                           float v) {
  if (dtype == COADAPT_BF16)
    reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
  else if (dtype == COADAPT_FP16)
    reinterpret_cast<__half*>(dst)[i] = __float2half_rn(v);
  else if (dtype == COADAPT_FP32)
    reinterpret_cast<float*>(dst)[i] = v;
  else
    reinterpret_cast<double*>(dst)[i] = (double)v;
}

__device__ __forceinline__ float round_trip(int dtype, float v) {
  if (dtype == COADAPT_BF16) return __bfloat162float(__float2bfloat16_rn(v));
  if (dtype == COADAPT_FP16) return __half2float(__float2half_rn(v));
  return v;
}

__global__ void synth_kernel(void* dst, int dtype, GenSeg seg, uint64_t skey,
                             uint64_t gkey, float g0, float unit) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       j < seg.numel; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t gidx = seg.global_base + (j / seg.row_len) * seg.row_stride +
                          (j % seg.row_len);
    store_elem(dst, dtype, seg.local_off + j,
               synth_value(skey, gkey, gidx, g0, unit));
  }
}

__global__ void synth_mean_kernel(void* dst, int dtype, GenSeg seg,
                                  uint64_t seed, uint64_t sample0,
                                  int64_t nsamples, uint64_t gkey, float g0,
                                  float unit, float inv_n) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       j < seg.numel; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t gidx = seg.global_base + (j / seg.row_len) * seg.row_stride +
                          (j % seg.row_len);
    float acc = 0.0f;
    for (int64_t n = 0; n < nsamples; ++n) {
      const uint64_t skey =
          mix64(seed ^ mix64(sample0 + (uint64_t)n + 0x632BE59BD9B4E019ull));
      acc = __fadd_rn(acc,
                      round_trip(dtype, synth_value(skey, gkey, gidx, g0, unit)));
    }
    store_elem(dst, dtype, seg.local_off + j, __fmul_rn(acc, inv_n));
  }
}

__global__ void l2_flush_kernel(uint4* buf, uint64_t nvec, uint32_t salt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (uint64_t)gridDim.x * blockDim.x)
    buf[i] = make_uint4(salt, (uint32_t)i, salt, (uint32_t)(i >> 32));
}

// read-only streaming probe: the same load pattern as K1 without the math
template <int NT, int U>
__global__ void __launch_bounds__(NT)
    read_probe_kernel(const uint4* __restrict__ p, uint64_t nvec,
                      double* sink) {
  uint32_t x = 0;
  const uint64_t chunk = (uint64_t)U * NT;  // interleaved, as K1
  for (uint64_t c = blockIdx.x; c * chunk < nvec; c += gridDim.x) {
    const uint64_t i = c * chunk + threadIdx.x;
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      r[j] = (i + (uint64_t)j * NT < nvec) ? ld_stream(p + i + (uint64_t)j * NT)
                                            : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int j = 0; j < U; ++j) x ^= r[j].x ^ r[j].y ^ r[j].z ^ r[j].w;
  }
  if (x == 0x9e3779b9u) *sink = (double)x;  // keeps the loads alive
}

// ---------------------------------------------------------------- configs

constexpr int kNT = 256;   // threads per CTA, K1
constexpr int kU = 8;      // 16-byte loads in flight per thread, K1
constexpr int kNTF = 256;  // threads per CTA, K1f

template <int M>
struct FusedCfg {
  // keep ~8-16 loads of 16 B in flight per thread
  static constexpr int UP = M >= 8 ? 1 : (M >= 4 ? 2 : (M >= 2 ? 4 : 8));
};

struct K1Fn {
  void* fn = nullptr;
  int nt = 0;
};

template <int DT, int NT = kNT, int U = kU, int MINB = 4>
K1Fn sqnorm_fn() {
  return K1Fn{reinterpret_cast<void*>(&sqnorm_kernel<DT, NT, U, MINB>), NT};
}

template <int DT, int M>
void* fused_fn() {
  return reinterpret_cast<void*>(&fused_kernel<DT, M, kNTF, FusedCfg<M>::UP>);
}

template <int DT>
void* fused_fn_rt(int M) {
  switch (M) {
#define F(m) \
  case m:    \
    return fused_fn<DT, m>();
    F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8) F(9) F(10) F(11) F(12) F(13) F(14)
        F(15) F(16)
#undef F
  }
  return nullptr;
}

void* fused_kernel_ptr(int dtype, int M) {
  switch (dtype) {
    case COADAPT_BF16: return fused_fn_rt<COADAPT_BF16>(M);
    case COADAPT_FP16: return fused_fn_rt<COADAPT_FP16>(M);
    case COADAPT_FP32: return fused_fn_rt<COADAPT_FP32>(M);
  }
  return nullptr;
}

K1Fn sqnorm_kernel_ptr(int dtype) {
  switch (dtype) {
    case COADAPT_BF16: return sqnorm_fn<COADAPT_BF16>();
    case COADAPT_FP16: return sqnorm_fn<COADAPT_FP16>();
    case COADAPT_FP32: return sqnorm_fn<COADAPT_FP32>();
    case COADAPT_FP64: return sqnorm_fn<COADAPT_FP64>();
  }
  return K1Fn{};
}

int occupancy_of(void* fn, int nt) {
  int occ = 0;
  if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nt, 0) !=
                 cudaSuccess)
    return 0;
  return occ;
}

struct TmaFn {
  void* fn = nullptr;
  int P = 0, smem = 0, nt = 0;
};

template <int DT, int M, int V, bool MEAN>
TmaFn tma_fn_v() {
  using C = TmaCfg<DT, M, V>;
  TmaFn f;
  f.fn = reinterpret_cast<void*>(&fused_tma_kernel<DT, M, V, MEAN>);
  f.P = C::P;
  f.smem = C::kSmem;
  f.nt = C::NT;
  // opt in to > 48 KB dynamic shared memory once per device (the attribute
  // is per device: one process may drive several GPUs)
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(f.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::kSmem);
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  return f;
}

// Best shape per M, measured on B200 (bf16, 32 GB, burst,
// profiles/r01c_tma_shapes.txt): the chunk's vectors per tile vs the group's
// threads and the register cap decide it (e.g. M=16: shape 5's 7-warp groups
// own exactly the 224 vectors of a 3584 B tile, 6.95 TB/s vs 6.59 for shape 4
// whose 8-warp groups leave 32 threads idle).
constexpr int kBestShape[17] = {4, 4, 4, 0, 4, 4, 0, 4, 0, 4, 5, 5, 0, 0, 4, 5, 5};

#ifndef COADAPT_SHAPE_SWEEP
#define COADAPT_SHAPE_SWEEP 0  // 1: every shape selectable by COADAPT_TMA_SHAPE
#endif

template <int DT, int M>
TmaFn tma_fn(bool mean) {
  // batched K1 (no mean term): the best shape only
  if (!mean) return tma_fn_v<DT, M, kBestShape[M], false>();
#if !COADAPT_SHAPE_SWEEP
  // shipped build: the measured best shape per M only (the sweep build,
  // -DCOADAPT_SHAPE_SWEEP=1, instantiates all of them: 5x the compile time)
  return tma_fn_v<DT, M, kBestShape[M], true>();
#else
  static const char* e = getenv("COADAPT_TMA_SHAPE");  // development sweep
  switch (e ? atoi(e) : kBestShape[M]) {
    case 1: return tma_fn_v<DT, M, 1, true>();
    case 2: return tma_fn_v<DT, M, 2, true>();
    case 3: return tma_fn_v<DT, M, 3, true>();
    case 4: return tma_fn_v<DT, M, 4, true>();
    case 5: return tma_fn_v<DT, M, 5, true>();
    default: return tma_fn_v<DT, M, 0, true>();
  }
#endif
}

template <int DT>
TmaFn tma_fn_rt(int M, bool mean) {
  switch (M) {
#define F(m) \
  case m:    \
    return tma_fn<DT, m>(mean);
    F(1) F(2) F(3) F(4) F(5) F(6) F(7) F(8) F(9) F(10) F(11) F(12) F(13) F(14)
        F(15) F(16)
#undef F
  }
  return TmaFn{};
}

TmaFn tma_kernel(int dtype, int M, bool mean) {
  switch (dtype) {
    case COADAPT_BF16: return tma_fn_rt<COADAPT_BF16>(M, mean);
    case COADAPT_FP16: return tma_fn_rt<COADAPT_FP16>(M, mean);
    case COADAPT_FP32: return tma_fn_rt<COADAPT_FP32>(M, mean);
  }
  return TmaFn{};
}

}  // namespace

int tma_chunk_elems(int dtype, int M, bool mean) { return tma_kernel(dtype, M, mean).P; }

cudaError_t launch_fused_tma(int dtype, int M, const Range* ranges, int nranges,
                             const uint64_t* prefix, uint64_t c_begin,
                             uint64_t c_end, const FusedArgs& fa, Sink sink,
                             int grid, cudaStream_t s, const Tail* tail) {
  const TmaFn f = tma_kernel(dtype, M, fa.gslot >= 0);
  if (!f.fn) return cudaErrorInvalidValue;
  Tail none;
  std::memset(&none, 0, sizeof(none));
  const Tail& t = tail ? *tail : none;
  void* args[] = {(void*)&ranges, (void*)&nranges, (void*)&prefix,
                  (void*)&c_begin, (void*)&c_end, (void*)&fa, (void*)&sink,
                  (void*)&t};
  return cudaLaunchKernel(f.fn, dim3(grid), dim3(f.nt), args, f.smem, s);
}

int threads_sqnorm(int dtype) { return sqnorm_kernel_ptr(dtype).nt; }
int threads_fused(int) { return kNTF; }
int occupancy_sqnorm(int dtype) {
  const K1Fn f = sqnorm_kernel_ptr(dtype);
  return occupancy_of(f.fn, f.nt);
}
int occupancy_fused(int dtype, int M) {
  return occupancy_of(fused_kernel_ptr(dtype, M), kNTF);
}

cudaError_t launch_sqnorm_batched(int dtype, const Range* ranges, int nranges,
                                  Window w, const BatchArgs& jobs, Sink sink,
                                  int grid, cudaStream_t s) {
  const K1Fn f = sqnorm_kernel_ptr(dtype);
  if (!f.fn) return cudaErrorInvalidValue;
  void* args[] = {(void*)&ranges, (void*)&nranges, (void*)&w, (void*)&jobs,
                  (void*)&sink};
  return cudaLaunchKernel(f.fn, dim3(grid), dim3(f.nt), args, 0, s);
}

cudaError_t launch_fused(int dtype, int M, const Range* ranges, int nranges,
                         Window w, const FusedArgs& fa, Sink sink, int grid,
                         cudaStream_t s) {
  void* fn = fused_kernel_ptr(dtype, M);
  if (!fn) return cudaErrorInvalidValue;
  void* args[] = {(void*)&ranges, (void*)&nranges, (void*)&w, (void*)&fa,
                  (void*)&sink};
  return cudaLaunchKernel(fn, dim3(grid), dim3(kNTF), args, 0, s);
}

namespace {
// vectors per register set (two sets in flight); measured on 1 x B200, 1 Gi
// bf16: (2, 4) 5.93 / 4.70 TB/s (add / first); (3, 6) 5.65 / 4.81;
// (4, 4) 4.71 / 4.76 (spills); unpipelined (4, 8) 5.73 / 4.76
constexpr int kNTA = 256, kUA = 2, kUA1 = 4;  // kUA1: first micro-batch
void* accum_fn(int dtype, bool first) {
  switch (dtype) {
    case COADAPT_BF16:
      return first ? reinterpret_cast<void*>(&accum_kernel<COADAPT_BF16, kNTA, kUA1, true>)
                   : reinterpret_cast<void*>(&accum_kernel<COADAPT_BF16, kNTA, kUA, false>);
    case COADAPT_FP16:
      return first ? reinterpret_cast<void*>(&accum_kernel<COADAPT_FP16, kNTA, kUA1, true>)
                   : reinterpret_cast<void*>(&accum_kernel<COADAPT_FP16, kNTA, kUA, false>);
    case COADAPT_FP32:
      return first ? reinterpret_cast<void*>(&accum_kernel<COADAPT_FP32, kNTA, kUA1, true>)
                   : reinterpret_cast<void*>(&accum_kernel<COADAPT_FP32, kNTA, kUA, false>);
  }
  return nullptr;
}
}  // namespace

int occupancy_accum(int dtype, bool first) {
  return occupancy_of(accum_fn(dtype, first), kNTA);
}

namespace {
constexpr int kNTR = 256, kUR = 2;
void* rs_fn(int dtype, bool nvls = false) {
  if (nvls)
    return dtype == COADAPT_FP32
               ? reinterpret_cast<void*>(&rs_kernel<COADAPT_FP32, kNTR, kUR, true>)
               : nullptr;
  switch (dtype) {
    case COADAPT_BF16: return reinterpret_cast<void*>(&rs_kernel<COADAPT_BF16, kNTR, kUR>);
    case COADAPT_FP16: return reinterpret_cast<void*>(&rs_kernel<COADAPT_FP16, kNTR, kUR>);
    case COADAPT_FP32: return reinterpret_cast<void*>(&rs_kernel<COADAPT_FP32, kNTR, kUR>);
  }
  return nullptr;
}
}  // namespace

int occupancy_rs(int dtype) { return occupancy_of(rs_fn(dtype), kNTR); }

cudaError_t launch_rs(int dtype, const Range* full, int nfull, uint64_t lo,
                      uint64_t hi, const RSArgs& a, Sink sink, int grid,
                      cudaStream_t s) {
  void* fn = rs_fn(dtype, a.nvls != 0);
  if (!fn) return cudaErrorInvalidValue;
  void* args[] = {(void*)&full, (void*)&nfull, (void*)&lo, (void*)&hi,
                  (void*)&a, (void*)&sink};
  return cudaLaunchKernel(fn, dim3(grid), dim3(kNTR), args, 0, s);
}

cudaError_t launch_accum(int dtype, const Range* full, int nfull, uint64_t numel,
                         const AccumArgs& a, Sink sink, int grid,
                         cudaStream_t s) {
  void* fn = accum_fn(dtype, a.flags & 1);
  if (!fn) return cudaErrorInvalidValue;
  float* mg = a.main_grad;
  const void* g = a.grad;
  int flags = a.flags;
  int32_t slot = a.slot, gslot = a.gslot;
  double gscale = a.gscale;
  void* args[] = {(void*)&full, (void*)&nfull, (void*)&numel, (void*)&mg,
                  (void*)&g,    (void*)&flags, (void*)&slot,  (void*)&gslot,
                  (void*)&gscale, (void*)&sink};
  return cudaLaunchKernel(fn, dim3(grid), dim3(kNTA), args, 0, s);
}

cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t s) {
  finalize_kernel<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_p2p_finalize(const P2PArgs& a, cudaStream_t s) {
  p2p_finalize_kernel<<<1, 256, 0, s>>>(a);
  return cudaGetLastError();
}

static int grid_for_elems(uint64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (n + 255) / 256;
  const uint64_t cap = (uint64_t)sms * 16;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

cudaError_t launch_synth(void* dst, int dtype, GenSeg seg, uint64_t seed,
                         uint64_t sample, float g0, float unit,
                         cudaStream_t s) {
  if (seg.numel == 0) return cudaSuccess;
  synth_kernel<<<grid_for_elems(seg.numel), 256, 0, s>>>(
      dst, dtype, seg, sample_key(seed, sample), sign_key(seed), g0, unit);
  return cudaGetLastError();
}

cudaError_t launch_synth_mean(void* dst, int dtype, GenSeg seg, uint64_t seed,
                              uint64_t sample0, int64_t nsamples, float g0,
                              float unit, cudaStream_t s) {
  if (seg.numel == 0) return cudaSuccess;
  const float inv_n = (float)(1.0 / (double)nsamples);
  synth_mean_kernel<<<grid_for_elems(seg.numel), 256, 0, s>>>(
      dst, dtype, seg, seed, sample0, nsamples, sign_key(seed), g0, unit,
      inv_n);
  return cudaGetLastError();
}

cudaError_t launch_l2_flush(void* buf, uint64_t bytes, cudaStream_t s) {
  static uint32_t salt = 1;
  const uint64_t nvec = bytes / 16;
  if (!nvec) return cudaSuccess;
  l2_flush_kernel<<<grid_for_elems(nvec), 256, 0, s>>>(
      static_cast<uint4*>(buf), nvec, salt++);
  return cudaGetLastError();
}

cudaError_t launch_read_probe(const void* buf, uint64_t bytes, double* sink,
                              cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // 4 CTAs x 256 threads x 8 loads per SM: the best LDG point of
  // tools/bw_sweep.cu (interleaved, 7.35 TB/s)
  read_probe_kernel<kNT, kU><<<sms * 4, kNT, 0, s>>>(
      static_cast<const uint4*>(buf), bytes / 16, sink);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace coadapt
