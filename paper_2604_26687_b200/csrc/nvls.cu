// nvls.cu — NVLink SHARP (NVLS) buffers and the switch-reduced DP gradient
// all-reduce (the step after KR).
//
// KR moves 2(d-1)/d of the bucket over each GPU's NVLink in each direction
// (peer loads + peer stores) and is link-bound at ~595 GB/s per direction
// (profiles/r01c_kr_allreduce.txt).  With a multicast object the NVSwitch
// does the reduction: each GPU issues `multimem.ld_reduce` for its 1/d slice
// (the switch reads that slice from every GPU, adds, returns one copy) and
// `multimem.st` of the scaled result (the switch writes it into every GPU's
// buffer).  Per GPU and link direction that is one bucket (out: its copies
// of the other slices for their reductions + its own result; in: its
// reduced slice + the others' results) instead of 2(d-1)/d buckets for the
// P2P form — equal at d = 2, 1.5x less at d = 4, 1.75x less at d = 8.
//
// The buffers must be physical allocations bound to the multicast object,
// so the trainer allocates its main_grad / grad bucket here
// (coadapt_nvls_*).  Rank 0 creates the object and exports it as a POSIX
// file descriptor; the 64-byte handle carries (pid, fd) and every other
// rank duplicates that descriptor with pidfd_getfd (fabric handles need an
// IMEX channel this box does not grant: cuMulticastCreate returns
// CUDA_ERROR_NOT_PERMITTED for them).  Every rank then adds its device and,
// after a host barrier, binds its own physical memory and maps a unicast
// and a multicast view.  The driver API
// is reached through cudaGetDriverEntryPoint, so the library still loads
// where no driver is installed (the CPU test container).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include <poll.h>
#include <sys/socket.h>
#include <sys/syscall.h>
#include <sys/un.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <thread>

#include "../../include/coadapt_cuda.h"
#include "internal.h"

namespace coadapt_capi {
void set_error(const char* msg);
void count_launch();
}  // namespace coadapt_capi

struct coadapt_nvls {
  int device = -1, nranks = 0;
  uint64_t bytes = 0;  // rounded up to the multicast granularity
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUdeviceptr uc_va = 0, mc_va = 0;
  bool added = false, bound = false, mapped_uc = false, mapped_mc = false;
  mutable int export_fd = -1;  // exporter: kept open until destroy
};

namespace {

int fail(int code, const std::string& msg) {
  coadapt_capi::set_error(msg.c_str());
  return code;
}

template <class F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

struct Driver {
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*,
                                      CUmulticastGranularity_flags);
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle,
                               size_t, size_t, unsigned long long);
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle,
                                         CUmemAllocationHandleType, unsigned long long);
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*,
                                           CUmemAllocationHandleType);
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long);
  CUresult (*MemRelease)(CUmemGenericAllocationHandle);
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*MemAddressFree)(CUdeviceptr, size_t);
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                     unsigned long long);
  CUresult (*MemUnmap)(CUdeviceptr, size_t);
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                          CUmemAllocationGranularity_flags);
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
  bool ok = false;
};

const Driver& drv() {
  static Driver d = [] {
    Driver x;
    x.MulticastCreate = entry<decltype(x.MulticastCreate)>("cuMulticastCreate");
    x.MulticastGetGranularity =
        entry<decltype(x.MulticastGetGranularity)>("cuMulticastGetGranularity");
    x.MulticastAddDevice = entry<decltype(x.MulticastAddDevice)>("cuMulticastAddDevice");
    x.MulticastBindMem = entry<decltype(x.MulticastBindMem)>("cuMulticastBindMem");
    x.MulticastUnbind = entry<decltype(x.MulticastUnbind)>("cuMulticastUnbind");
    x.MemExportToShareableHandle =
        entry<decltype(x.MemExportToShareableHandle)>("cuMemExportToShareableHandle");
    x.MemImportFromShareableHandle =
        entry<decltype(x.MemImportFromShareableHandle)>("cuMemImportFromShareableHandle");
    x.MemCreate = entry<decltype(x.MemCreate)>("cuMemCreate");
    x.MemRelease = entry<decltype(x.MemRelease)>("cuMemRelease");
    x.MemAddressReserve = entry<decltype(x.MemAddressReserve)>("cuMemAddressReserve");
    x.MemAddressFree = entry<decltype(x.MemAddressFree)>("cuMemAddressFree");
    x.MemMap = entry<decltype(x.MemMap)>("cuMemMap");
    x.MemUnmap = entry<decltype(x.MemUnmap)>("cuMemUnmap");
    x.MemSetAccess = entry<decltype(x.MemSetAccess)>("cuMemSetAccess");
    x.MemGetAllocationGranularity =
        entry<decltype(x.MemGetAllocationGranularity)>("cuMemGetAllocationGranularity");
    x.DeviceGetAttribute = entry<decltype(x.DeviceGetAttribute)>("cuDeviceGetAttribute");
    x.ok = x.MulticastCreate && x.MulticastGetGranularity && x.MulticastAddDevice &&
           x.MulticastBindMem && x.MulticastUnbind && x.MemExportToShareableHandle &&
           x.MemImportFromShareableHandle && x.MemCreate && x.MemRelease &&
           x.MemAddressReserve && x.MemAddressFree && x.MemMap && x.MemUnmap &&
           x.MemSetAccess && x.MemGetAllocationGranularity && x.DeviceGetAttribute;
    return x;
  }();
  return d;
}

#define DRV(call)                                                             \
  do {                                                                        \
    CUresult r_ = (call);                                                     \
    if (r_ != CUDA_SUCCESS)                                                   \
      return fail(COADAPT_E_CUDA, std::string(#call) + " failed: CUresult " + \
                                      std::to_string((int)r_));               \
  } while (0)

#define RT(call)                                                          \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess)                                                \
      return fail(COADAPT_E_CUDA, std::string(#call) + ": " +             \
                                      cudaGetErrorString(e_));            \
  } while (0)

struct DevScope {  // makes `dev` current, restores the caller's
  int prev = -1;
  explicit DevScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

CUmulticastObjectProp mc_prop(int nranks, uint64_t bytes) {
  CUmulticastObjectProp p;
  std::memset(&p, 0, sizeof(p));
  p.numDevices = (unsigned)nranks;
  p.size = bytes;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

int check_args(int device, int nranks, uint64_t bytes) {
  if (nranks < 1 || nranks > 64 || bytes == 0 || device < 0)
    return fail(COADAPT_E_VALIDATION, "need 1 <= nranks <= 64, bytes > 0, device >= 0");
  if (!drv().ok)
    return fail(COADAPT_E_CUDA, "driver entry points for multicast objects are unavailable");
  int mc = 0;
  DRV(drv().DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, device));
  if (!mc) return fail(COADAPT_E_CUDA, "device does not support multicast objects (NVLS)");
  return COADAPT_OK;
}

// ------------------------------------------------------------------ kernel

template <int DT>
struct Mm;
template <>
struct Mm<COADAPT_FP32> {
  static __device__ __forceinline__ uint4 ld_reduce(const void* p) {
    uint4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p)
                 : "memory");
    return r;
  }
  static __device__ __forceinline__ void st(void* p, const uint4& v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
  static __device__ __forceinline__ uint32_t scale2(uint32_t w, float s) {
    return __float_as_uint(__uint_as_float(w) * s);
  }
};

// Vectors [v0, v1) of the bucket: switch-reduced load (fp32 adds in the
// switch), scale, multicast store.
// U vectors in flight per thread cover the NVLink round trip.
template <int DT, int U>
__global__ void __launch_bounds__(256) nvls_allreduce_kernel(char* mc, uint64_t v0, uint64_t v1,
                                                             float scale, int scaled) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = v0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < v1;
       v += stride * U) {
    uint4 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (v + j * stride < v1) r[j] = Mm<DT>::ld_reduce(mc + (v + j * stride) * 16);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (v + j * stride >= v1) continue;
      uint4 o = r[j];
      if (scaled) {
        o.x = Mm<DT>::scale2(o.x, scale);
        o.y = Mm<DT>::scale2(o.y, scale);
        o.z = Mm<DT>::scale2(o.z, scale);
        o.w = Mm<DT>::scale2(o.w, scale);
      }
      Mm<DT>::st(mc + (v + j * stride) * 16, o);
    }
  }
  // make the multicast stores visible system-wide before the kernel retires
  asm volatile("fence.proxy.alias;" ::: "memory");
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

}  // namespace

extern "C" {

int coadapt_nvls_create(int device, int nranks, uint64_t bytes, coadapt_nvls** out) {
  if (!out) return fail(COADAPT_E_VALIDATION, "out is NULL");
  *out = nullptr;
  if (int rc = check_args(device, nranks, bytes)) return rc;
  DevScope scope(device);
  CUmulticastObjectProp p = mc_prop(nranks, bytes);
  size_t gran = 0;
  DRV(drv().MulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  p.size = (bytes + gran - 1) / gran * gran;
  coadapt_nvls* o = new coadapt_nvls;
  o->device = device;
  o->nranks = nranks;
  o->bytes = p.size;
  CUresult r = drv().MulticastCreate(&o->mc, &p);
  if (r != CUDA_SUCCESS) {
    delete o;
    return fail(COADAPT_E_CUDA, "cuMulticastCreate failed: CUresult " + std::to_string((int)r));
  }
  *out = o;
  return COADAPT_OK;
}

namespace {

// The multicast handle is a POSIX fd; it reaches the other ranks the way
// NCCL passes its cuMem handles: over a Unix domain socket as SCM_RIGHTS
// ancillary data.  The exporter listens on an abstract-namespace socket
// named after (pid, fd, nonce) and serves the fd to nranks-1 importers from
// a detached thread (its own dup of the fd, 300 s deadline).  pidfd_getfd
// stays as the fallback for importers that cannot reach the socket; it
// needs ptrace rights over the exporter (Yama ptrace_scope / CAP_SYS_PTRACE).
void sock_name(sockaddr_un& a, socklen_t& len, int32_t pid, int32_t fd, int32_t nonce) {
  std::memset(&a, 0, sizeof(a));
  a.sun_family = AF_UNIX;
  const int n = std::snprintf(a.sun_path + 1, sizeof(a.sun_path) - 1,
                              "coadapt-nvls-%d-%d-%d", pid, fd, nonce);
  len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
}

int serve_fd(int fd, int32_t pid, int32_t nonce, int clients) {
  const int ls = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
  if (ls < 0) return -1;
  sockaddr_un a;
  socklen_t len;
  sock_name(a, len, pid, fd, nonce);
  if (bind(ls, reinterpret_cast<sockaddr*>(&a), len) != 0 || listen(ls, clients) != 0) {
    close(ls);
    return -1;
  }
  const int mine = dup(fd);
  std::thread([ls, mine, clients] {
    const auto end = std::chrono::steady_clock::now() + std::chrono::seconds(300);
    for (int served = 0; served < clients;) {
      const auto left = std::chrono::duration_cast<std::chrono::milliseconds>(
          end - std::chrono::steady_clock::now()).count();
      if (left <= 0) break;
      pollfd pf{ls, POLLIN, 0};
      if (poll(&pf, 1, (int)std::min<long long>(left, 1000)) <= 0) continue;
      const int c = accept4(ls, nullptr, nullptr, SOCK_CLOEXEC);
      if (c < 0) continue;
      char byte = 'F';
      iovec iov{&byte, 1};
      alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))];
      std::memset(ctl, 0, sizeof(ctl));
      msghdr m;
      std::memset(&m, 0, sizeof(m));
      m.msg_iov = &iov;
      m.msg_iovlen = 1;
      m.msg_control = ctl;
      m.msg_controllen = sizeof(ctl);
      cmsghdr* cm = CMSG_FIRSTHDR(&m);
      cm->cmsg_level = SOL_SOCKET;
      cm->cmsg_type = SCM_RIGHTS;
      cm->cmsg_len = CMSG_LEN(sizeof(int));
      std::memcpy(CMSG_DATA(cm), &mine, sizeof(int));
      if (sendmsg(c, &m, MSG_NOSIGNAL) == 1) ++served;
      close(c);
    }
    close(ls);
    close(mine);
  }).detach();
  return 0;
}

// fd from the exporter's socket, or -1 (caller falls back to pidfd_getfd)
int receive_fd(int32_t pid, int32_t fd, int32_t nonce) {
  sockaddr_un a;
  socklen_t len;
  sock_name(a, len, pid, fd, nonce);
  for (int attempt = 0; attempt < 100; ++attempt) {  // ~5 s: the server may lag
    const int c = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (c < 0) return -1;
    if (connect(c, reinterpret_cast<sockaddr*>(&a), len) == 0) {
      char byte = 0;
      iovec iov{&byte, 1};
      alignas(cmsghdr) char ctl[CMSG_SPACE(sizeof(int))];
      msghdr m;
      std::memset(&m, 0, sizeof(m));
      m.msg_iov = &iov;
      m.msg_iovlen = 1;
      m.msg_control = ctl;
      m.msg_controllen = sizeof(ctl);
      int got = -1;
      if (recvmsg(c, &m, MSG_CMSG_CLOEXEC) == 1) {
        for (cmsghdr* cm = CMSG_FIRSTHDR(&m); cm; cm = CMSG_NXTHDR(&m, cm))
          if (cm->cmsg_level == SOL_SOCKET && cm->cmsg_type == SCM_RIGHTS)
            std::memcpy(&got, CMSG_DATA(cm), sizeof(int));
      }
      close(c);
      return got;
    }
    close(c);
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
  }
  return -1;
}

std::atomic<int32_t> g_nonce{1};

}  // namespace

int coadapt_nvls_export(const coadapt_nvls* o, void* handle, size_t len) {
  if (!o || !handle || len < 64)
    return fail(COADAPT_E_VALIDATION, "need an object and a >= 64-byte handle buffer");
  DevScope scope(o->device);
  int fd = -1;
  DRV(drv().MemExportToShareableHandle(&fd, o->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  int32_t blob[16] = {0};
  blob[0] = 0x4e564c53;  // "NVLS"
  blob[1] = (int32_t)getpid();
  blob[2] = fd;  // stays open in the exporting process for the importers
  blob[3] = g_nonce.fetch_add(1) ^ (int32_t)(uintptr_t)o;
  blob[4] = serve_fd(fd, blob[1], blob[3], o->nranks - 1) == 0 ? 1 : 0;  // socket served
  if (o->export_fd >= 0) close(o->export_fd);
  o->export_fd = fd;
  std::memcpy(handle, blob, sizeof(blob));
  return COADAPT_OK;
}

int coadapt_nvls_import(int device, int nranks, uint64_t bytes, const void* handle, size_t len,
                        coadapt_nvls** out) {
  if (!out || !handle || len < 64)
    return fail(COADAPT_E_VALIDATION, "need out and a >= 64-byte handle");
  *out = nullptr;
  if (int rc = check_args(device, nranks, bytes)) return rc;
  int32_t blob[16];
  std::memcpy(blob, handle, sizeof(blob));
  if (blob[0] != 0x4e564c53) return fail(COADAPT_E_VALIDATION, "not an NVLS handle");
  // the exporter's descriptor: SCM_RIGHTS over its socket, else pidfd_getfd
  // (COADAPT_NVLS_SHARE=socket|pidfd forces one path, for tests)
  const char* force = getenv("COADAPT_NVLS_SHARE");
  const bool only_socket = force && std::string(force) == "socket";
  const bool only_pidfd = force && std::string(force) == "pidfd";
  int fd = (blob[4] && !only_pidfd) ? receive_fd(blob[1], blob[2], blob[3]) : -1;
  if (fd < 0 && only_socket)
    return fail(COADAPT_E_CUDA, "SCM_RIGHTS transfer of the multicast handle failed");
  if (fd < 0) {
    const int pidfd = (int)syscall(434 /* pidfd_open */, (pid_t)blob[1], 0);
    if (pidfd < 0) return fail(COADAPT_E_CUDA, "pidfd_open of the exporting rank failed");
    fd = (int)syscall(438 /* pidfd_getfd */, pidfd, blob[2], 0);
    close(pidfd);
    if (fd < 0)
      return fail(COADAPT_E_CUDA,
                  "neither the exporter's socket (SCM_RIGHTS) nor pidfd_getfd delivered "
                  "the multicast handle");
  }
  DevScope scope(device);
  CUmulticastObjectProp p = mc_prop(nranks, bytes);
  size_t gran = 0;
  DRV(drv().MulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  coadapt_nvls* o = new coadapt_nvls;
  o->device = device;
  o->nranks = nranks;
  o->bytes = (bytes + gran - 1) / gran * gran;
  CUresult r = drv().MemImportFromShareableHandle(
      &o->mc, reinterpret_cast<void*>((uintptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(fd);
  if (r != CUDA_SUCCESS) {
    delete o;
    return fail(COADAPT_E_CUDA,
                "cuMemImportFromShareableHandle failed: CUresult " + std::to_string((int)r));
  }
  *out = o;
  return COADAPT_OK;
}

int coadapt_nvls_add_device(coadapt_nvls* o) {
  if (!o) return fail(COADAPT_E_VALIDATION, "object is NULL");
  if (o->added) return COADAPT_OK;
  DevScope scope(o->device);
  DRV(drv().MulticastAddDevice(o->mc, (CUdevice)o->device));
  o->added = true;
  return COADAPT_OK;
}

int coadapt_nvls_bind(coadapt_nvls* o, void** unicast, void** multicast) {
  if (!o || !unicast || !multicast) return fail(COADAPT_E_VALIDATION, "NULL argument");
  if (!o->added) return fail(COADAPT_E_VALIDATION, "add the device first (then a host barrier)");
  DevScope scope(o->device);
  if (!o->bound) {
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = o->device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t g = 0;
    DRV(drv().MemGetAllocationGranularity(&g, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    if (o->bytes % g) return fail(COADAPT_E_INTERNAL, "multicast size not a multiple of the "
                                                      "allocation granularity");
    DRV(drv().MemCreate(&o->mem, o->bytes, &ap, 0));
    CUmemAccessDesc acc;
    std::memset(&acc, 0, sizeof(acc));
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = o->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DRV(drv().MemAddressReserve(&o->uc_va, o->bytes, g, 0, 0));
    DRV(drv().MemMap(o->uc_va, o->bytes, 0, o->mem, 0));
    o->mapped_uc = true;
    DRV(drv().MemSetAccess(o->uc_va, o->bytes, &acc, 1));
    DRV(drv().MulticastBindMem(o->mc, 0, o->mem, 0, o->bytes, 0));
    o->bound = true;
    DRV(drv().MemAddressReserve(&o->mc_va, o->bytes, g, 0, 0));
    DRV(drv().MemMap(o->mc_va, o->bytes, 0, o->mc, 0));
    o->mapped_mc = true;
    DRV(drv().MemSetAccess(o->mc_va, o->bytes, &acc, 1));
    RT(cudaMemset(reinterpret_cast<void*>(o->uc_va), 0, o->bytes));
    RT(cudaDeviceSynchronize());
  }
  *unicast = reinterpret_cast<void*>(o->uc_va);
  *multicast = reinterpret_cast<void*>(o->mc_va);
  return COADAPT_OK;
}

uint64_t coadapt_nvls_bytes(const coadapt_nvls* o) { return o ? o->bytes : 0; }

int coadapt_nvls_allreduce(coadapt_nvls* o, int dtype, uint64_t numel, int dp_rank,
                           double scale, void* stream) {
  COADAPT_NVTX("coadapt_nvls_allreduce");
  if (!o || !o->bound) return fail(COADAPT_E_VALIDATION, "object not bound");
  // fp32 only: the switch's bf16 reduction rounds differently from RNE and
  // the difference is one-sided (measured: ~20 % of elements 1 ulp off,
  // ||gbar||^2 biased by ~7e-4 on 2 GPUs) — far outside the GNS tolerance.
  if (dtype != COADAPT_FP32)
    return fail(COADAPT_E_VALIDATION,
                "NVLS all-reduce is fp32 only (the switch's bf16/fp16 rounding biases gbar^2)");
  const int es = 4;
  if (dp_rank < 0 || dp_rank >= o->nranks)
    return fail(COADAPT_E_VALIDATION, "dp_rank out of range");
  if (!(scale == scale) || std::isinf(scale))
    return fail(COADAPT_E_VALIDATION, "scale must be finite");
  const uint64_t per = 16 / es;
  const uint64_t nvec = (numel + per - 1) / per;  // the tail vector is padding of the buffer
  if (nvec * 16 > o->bytes) return fail(COADAPT_E_VALIDATION, "numel exceeds the buffer");
  // the same cut as coadapt_plan_create_slice (64-element multiples) in vectors
  const int d = o->nranks;
  auto cut = [&](int i) -> uint64_t {
    if (i >= d) return nvec;
    const uint64_t e = (uint64_t)((unsigned __int128)numel * i / d) & ~uint64_t(63);
    return e / per;
  };
  const uint64_t v0 = cut(dp_rank), v1 = cut(dp_rank + 1);
  if (v1 <= v0) return COADAPT_OK;
  DevScope scope(o->device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o->device);
  // flat across 1-8 vectors in flight x 1-16 CTAs per SM on 4 GPUs (4.66-4.80
  // ms for 2 GB, profiles/r01c_nvls_allreduce.txt): the switch path, not the
  // SMs, sets the rate
  constexpr int U = 4, per_sm = 4;
  const uint64_t want = (v1 - v0 + 256 * U - 1) / (256 * U);
  const int grid = (int)std::min<uint64_t>((uint64_t)sms * per_sm, std::max<uint64_t>(1, want));
  char* mc = reinterpret_cast<char*>(o->mc_va);
  const float sc = (float)scale;
  const int scaled = scale != 1.0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  nvls_allreduce_kernel<COADAPT_FP32, U><<<grid, 256, 0, s>>>(mc, v0, v1, sc, scaled);
  RT(cudaGetLastError());
  coadapt_capi::count_launch();
  return COADAPT_OK;
}

int coadapt_nvls_destroy(coadapt_nvls* o) {
  if (!o) return COADAPT_OK;
  DevScope scope(o->device);
  cudaDeviceSynchronize();
  if (o->mapped_mc) drv().MemUnmap(o->mc_va, o->bytes);
  if (o->mc_va) drv().MemAddressFree(o->mc_va, o->bytes);
  if (o->mapped_uc) drv().MemUnmap(o->uc_va, o->bytes);
  if (o->uc_va) drv().MemAddressFree(o->uc_va, o->bytes);
  if (o->bound) drv().MulticastUnbind(o->mc, (CUdevice)o->device, 0, o->bytes);
  if (o->mem) drv().MemRelease(o->mem);
  if (o->mc) drv().MemRelease(o->mc);
  if (o->export_fd >= 0) close(o->export_fd);
  delete o;
  return COADAPT_OK;
}

}  // extern "C"
