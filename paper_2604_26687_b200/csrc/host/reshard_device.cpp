// reshard_device.cpp — coadapt::reshard::DevicePlan over the C-ABI in
// coadapt_reshard.h (the executor lives in reshard.cu).
#include <cstring>
#include <vector>

#include "coadapt/errors.hpp"
#include "coadapt/reshard.hpp"
#include "coadapt_cuda.h"
#include "coadapt_reshard.h"

namespace coadapt::reshard {
namespace {

void check(int rc) {
  if (rc == COADAPT_OK) return;
  if (rc == COADAPT_E_VALIDATION) throw ValidationError(coadapt_last_error());
  throw InternalError(coadapt_last_error());
}

}  // namespace

DevicePlan::DevicePlan(const ModelSpec& model, const ParallelStrategy& src,
                       const ParallelStrategy& dst, SourcePolicy policy)
    : src_(layout_for(model, src, src.gpus())),
      dst_(layout_for(model, dst, dst.gpus())),
      plan_(plan_transfers(model, src_, dst_, policy)) {
  std::vector<coadapt_tensor_decl> decls(model.per_layer.size());
  for (std::size_t i = 0; i < decls.size(); ++i) {
    const auto& t = model.per_layer[i];
    std::memset(&decls[i], 0, sizeof(decls[i]));
    decls[i].name = t.name.c_str();
    decls[i].ndim = (int32_t)t.shape.size();
    decls[i].tp_axis = t.tp_axis;
    for (std::size_t k = 0; k < t.shape.size() && k < (std::size_t)kMaxDims; ++k)
      decls[i].shape[k] = t.shape[k];
  }
  coadapt_reshard_model m{};
  m.layers = model.layers;
  m.n_tensors = (int32_t)decls.size();
  m.tensors = decls.data();
  m.optimizer_state_multiplier = model.optimizer_state_multiplier;
  m.param_bytes = model.param_bytes;
  m.state_bytes = model.state_bytes;
  const int32_t s3[3] = {src.d, src.t, src.p}, d3[3] = {dst.d, dst.t, dst.p};
  check(coadapt_reshard_plan_create(&m, s3, d3, (int)policy, &handle_));
}

DevicePlan::~DevicePlan() { coadapt_reshard_plan_destroy(handle_); }

void DevicePlan::run(int role, int rank, std::span<const void* const> s,
                     std::span<void* const> d, int elem_bytes, int device,
                     void* stream) {
  check(coadapt_reshard_execute(handle_, role, rank, s.data(), s.size(),
                                d.data(), d.size(), elem_bytes, device, stream));
}

void DevicePlan::pull(int dst_rank, std::span<const void* const> s,
                      std::span<void* const> d, int eb, int dev, void* st) {
  run(COADAPT_RESHARD_PULL, dst_rank, s, d, eb, dev, st);
}

void DevicePlan::push(int src_rank, std::span<const void* const> s,
                      std::span<void* const> d, int eb, int dev, void* st) {
  run(COADAPT_RESHARD_PUSH, src_rank, s, d, eb, dev, st);
}

void DevicePlan::all(std::span<const void* const> s, std::span<void* const> d,
                     int eb, int dev, void* st) {
  run(COADAPT_RESHARD_ALL, -1, s, d, eb, dev, st);
}

}  // namespace coadapt::reshard
