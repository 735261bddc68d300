// NVLink peer-read ceiling on this box: every GPU reads B bytes from each of
// its peers at once (the traffic pattern of the KR reduce-scatter), three
// ways — 16-byte LDG loads with U vectors in flight per thread (how rs_kernel
// reads), cp.async.bulk (TMA) from peer memory into a shared-memory ring, and
// the copy engines (cudaMemcpyPeerAsync) — and reports GB/s per GPU of peer
// bytes received.  Measurement tool (profiles/r02_p2p_read_probe.txt).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        tools/p2p_read_probe.cu -o tools/_p2p_read_probe
//   tools/_p2p_read_probe [MiB per peer = 1024]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x,            \
                   cudaGetErrorString(e_));                                     \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

struct Peers {
  const uint4* p[8];
  int n;
};

template <int U>
__global__ void __launch_bounds__(256) ldg_read(Peers src, uint64_t nvec, unsigned long long* sink) {
  uint32_t x = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int q = 0; q < src.n; ++q) {
    const uint4* s = src.p[q];
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nvec; v += stride * U) {
      uint4 r[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const uint64_t i = v + j * stride;
        if (i < nvec)
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(r[j].x), "=r"(r[j].y), "=r"(r[j].z), "=r"(r[j].w)
                       : "l"(s + i));
        else
          r[j] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) x ^= r[j].x ^ r[j].y ^ r[j].z ^ r[j].w;
    }
  }
  if (x == 0x9e3779b9u) atomicAdd(sink, 1ull);
}

// TMA: one elected thread streams kTile-byte pieces of the peers' buffers
// into a kStages ring; the CTA's threads fold each piece (one LDS.128 each).
constexpr int kTile = 16384, kStages = 6;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(256) tma_read(Peers src, uint64_t bytes, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  const uint64_t tiles_per_peer = bytes / kTile;
  const uint64_t total = tiles_per_peer * src.n;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(blockDim.x));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t x = 0;
  int k = 0;
  // my tiles: t = blockIdx.x + k * gridDim.x
  auto issue = [&](uint64_t t, int st) {
    const int q = (int)(t / tiles_per_peer);
    const char* g = reinterpret_cast<const char*>(src.p[q]) + (t % tiles_per_peer) * kTile;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(kTile));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm + st * kTile)),
        "l"(g), "r"(kTile), "r"(smem_u32(&full[st]))
        : "memory");
  };
  const uint64_t mine = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0)
    for (int s = 0; s < kStages && (uint64_t)s < mine; ++s) issue(blockIdx.x + (uint64_t)s * gridDim.x, s);
  for (uint64_t i = 0; i < mine; ++i) {
    const int st = (int)(i % kStages);
    const uint32_t ph = (uint32_t)((i / kStages) & 1);
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&full[st])), "r"(ph));
    const uint4* t = reinterpret_cast<const uint4*>(sm + st * kTile);
    for (int v = threadIdx.x; v < kTile / 16; v += blockDim.x) {
      const uint4 r = t[v];
      x ^= r.x ^ r.y ^ r.z ^ r.w;
    }
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(&empty[st])));
    if (threadIdx.x == 0 && i + kStages < mine) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(smem_u32(&empty[st])), "r"(ph));
      issue(blockIdx.x + (i + kStages) * gridDim.x, st);
    }
    ++k;
  }
  if (x == 0x9e3779b9u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
  const uint64_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1024;
  const uint64_t B = mib << 20;
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("{\"error\": \"needs >= 2 GPUs\"}\n");
    return 0;
  }
  std::vector<void*> buf(n);
  std::vector<unsigned long long*> sink(n);
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  int sms = 148;
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    for (int q = 0; q < n; ++q)
      if (q != d) {
        int can = 0;
        CK(cudaDeviceCanAccessPeer(&can, d, q));
        if (!can) {
          std::printf("{\"error\": \"no peer access %d->%d\"}\n", d, q);
          return 0;
        }
        CK(cudaDeviceEnablePeerAccess(q, 0));
      }
    CK(cudaMalloc(&buf[d], B));
    CK(cudaMemset(buf[d], d + 1, B));
    CK(cudaMalloc(&sink[d], 8));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    CK(cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile * kStages));
  }
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<std::vector<void*>> scratch(n);
  std::vector<std::vector<cudaStream_t>> pst(n);  // one stream per peer (mode 4)
  std::vector<std::vector<cudaEvent_t>> pev(n);
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    for (int k = 0; k < n - 1; ++k) {
      cudaStream_t s;
      cudaEvent_t e;
      CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      pst[d].push_back(s);
      pev[d].push_back(e);
    }
  }
  auto run = [&](int mode, int peers_per_gpu, int reps) -> double {
    // each GPU reads from `peers_per_gpu` peers (d+1, d+2, ...); returns
    // the slowest GPU's peer GB/s received
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(e0[d], st[d]));
      for (int r = 0; r < reps; ++r) {
        Peers P{};
        P.n = peers_per_gpu;
        for (int k = 0; k < peers_per_gpu; ++k) P.p[k] = static_cast<const uint4*>(buf[(d + 1 + k) % n]);
        if (mode == 0)
          ldg_read<4><<<sms * 4, 256, 0, st[d]>>>(P, B / 16, sink[d]);
        else if (mode == 1)
          ldg_read<8><<<sms * 4, 256, 0, st[d]>>>(P, B / 16, sink[d]);
        else if (mode == 2)
          tma_read<<<sms, 256, kTile * kStages, st[d]>>>(P, B, sink[d]);
        else {
          while ((int)scratch[d].size() < n - 1) {
            void* s = nullptr;
            CK(cudaMalloc(&s, B));
            scratch[d].push_back(s);
          }
          if (mode == 3) {
            for (int k = 0; k < peers_per_gpu; ++k)
              CK(cudaMemcpyPeerAsync(scratch[d][0], d, buf[(d + 1 + k) % n], (d + 1 + k) % n, B, st[d]));
          } else {  // mode 4: each peer's copy on its own stream, joined back into st[d]
            CK(cudaEventRecord(pev[d][0], st[d]));
            for (int k = 0; k < peers_per_gpu; ++k) {
              CK(cudaStreamWaitEvent(pst[d][k], pev[d][0], 0));
              CK(cudaMemcpyPeerAsync(scratch[d][k], d, buf[(d + 1 + k) % n], (d + 1 + k) % n, B, pst[d][k]));
            }
            for (int k = 0; k < peers_per_gpu; ++k) {
              cudaEvent_t j;
              CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
              CK(cudaEventRecord(j, pst[d][k]));
              CK(cudaStreamWaitEvent(st[d], j, 0));
              CK(cudaEventDestroy(j));
            }
          }
        }
      }
      CK(cudaEventRecord(e1[d], st[d]));
    }
    double worst = 1e30;
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventSynchronize(e1[d]));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
      const double gbs = (double)B * peers_per_gpu * reps / (ms / 1e3) / 1e9;
      if (gbs < worst) worst = gbs;
    }
    return worst;
  };
  const char* names[5] = {"ldg_u4", "ldg_u8", "tma_ring", "copy_engine", "copy_engine_stream_per_peer"};
  std::printf("{\"gpus\": %d, \"bytes_per_peer\": %llu", n, (unsigned long long)B);
  for (int peers = 1; peers < n; ++peers) {
    for (int mode = 0; mode < 5; ++mode) {
      run(mode, peers, 1);  // warm-up
      const double g = run(mode, peers, 3);
      std::printf(", \"%s_from_%d_peers_gbs\": %.1f", names[mode], peers, g);
    }
  }
  std::printf("}\n");
  return 0;
}
