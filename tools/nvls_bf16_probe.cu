// Probe: how the NVSwitch rounds a bf16 multimem.ld_reduce — plain bf16
// accumulation (LDGMC.ADD.BF16x8) vs .acc::f32 (LDGMC.HPADD.BF16x8) — read
// into a local buffer for comparison with RNE of the exact sum
// (tools/nvls_bf16_probe.py).  Measurement tool, not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        tools/nvls_bf16_probe.cu -o tools/_nvls_bf16_probe.so
#include <cuda_runtime.h>
#include <cstdint>

template <int MODE>
__global__ void probe(const char* mc, uint4* out, uint64_t nvec) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nvec;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint4 r;
    if constexpr (MODE == 0)
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc + v * 16) : "memory");
    else
      asm volatile(
          "multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
          : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(mc + v * 16) : "memory");
    out[v] = r;
  }
}

extern "C" int nvls_bf16_probe(const void* mc, void* out, uint64_t nvec, int mode,
                               void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mode == 0)
    probe<0><<<148 * 4, 256, 0, s>>>(static_cast<const char*>(mc), static_cast<uint4*>(out), nvec);
  else
    probe<1><<<148 * 4, 256, 0, s>>>(static_cast<const char*>(mc), static_cast<uint4*>(out), nvec);
  return (int)cudaGetLastError();
}
