// Probe: does this box support NVLink multicast objects (NVLS, multimem.*)?
#include <cuda.h>
#include <cstdio>
int main() {
  cuInit(0);
  int n = 0;
  cuDeviceGetCount(&n);
  for (int i = 0; i < n; ++i) {
    CUdevice d;
    cuDeviceGet(&d, i);
    int mc = -1, fab = -1;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
    printf("device %d: multicast_supported=%d fabric_handles=%d\n", i, mc, fab);
  }
  if (n >= 2) {
    CUmulticastObjectProp p = {};
    p.numDevices = n;
    p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CUresult r = cuMulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    printf("granularity rc=%d gran=%zu\n", (int)r, gran);
    p.size = gran ? gran : (2u << 20);
    CUmemGenericAllocationHandle h;
    r = cuMulticastCreate(&h, &p);
    printf("cuMulticastCreate rc=%d\n", (int)r);
  }
  return 0;
}
