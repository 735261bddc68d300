// Link check of the B200-specific C++ face (include/coadapt/device.hpp) and
// of the C-ABI entry points added beside the reference API: every method's
// address is taken so the linker must resolve it in libcoadapt_b200.so.
// Without a GPU, constructing a plan must throw the reference's exception
// types (never abort); with --gpu it must succeed.
#include <cstdio>
#include <cstring>
#include <exception>

#include "coadapt/device.hpp"
#include "coadapt/errors.hpp"
#include "coadapt_cuda.h"

using coadapt::GnsDevicePlan;

int main(int argc, char** argv) {
  volatile const void* sinks[] = {
      reinterpret_cast<const void*>(&GnsDevicePlan::begin_step),
      reinterpret_cast<const void*>(&GnsDevicePlan::record_micro_bucket),
      reinterpret_cast<const void*>(&GnsDevicePlan::record_fused),
      reinterpret_cast<const void*>(&GnsDevicePlan::record_mean_gradient),
      reinterpret_cast<const void*>(&GnsDevicePlan::accumulate),
      reinterpret_cast<const void*>(&GnsDevicePlan::reduce_scatter_mean),
      reinterpret_cast<const void*>(&GnsDevicePlan::allreduce_mean),
      reinterpret_cast<const void*>(&GnsDevicePlan::barrier),
      reinterpret_cast<const void*>(&GnsDevicePlan::allreduce),
      reinterpret_cast<const void*>(&GnsDevicePlan::finalize),
      reinterpret_cast<const void*>(&coadapt_gns_allreduce_sqnorm),
      reinterpret_cast<const void*>(&coadapt_nvls_create),
      reinterpret_cast<const void*>(&coadapt_nvls_import),
      reinterpret_cast<const void*>(&coadapt_nvls_allreduce),
  };
  for (auto p : sinks)
    if (!p) return 2;
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  try {
    GnsDevicePlan plan(1, 2, 2, 0);
    if (!gpu) {
      std::printf("constructed a device plan without --gpu\n");
      return 1;
    }
  } catch (const std::exception& e) {
    if (gpu) {
      std::printf("device plan failed on a GPU box: %s\n", e.what());
      return 1;
    }
  }
  // NVLS entry points validate before touching the driver
  coadapt_nvls* o = nullptr;
  if (coadapt_nvls_create(0, 0, 1, &o) != COADAPT_E_VALIDATION) {
    std::printf("nvls_create accepted nranks = 0\n");
    return 1;
  }
  std::printf("OK\n");
  return 0;
}
