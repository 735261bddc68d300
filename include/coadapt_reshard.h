/* coadapt_reshard.h — C-ABI of the Reconfigure path.
 *
 * Replaces the reference's reshard module, which exists as specification
 * only (layout_for :445-453, plan_transfers :455-463,
 * execute_in_memory :465-473, estimate_reconfig_latency :475-483, plan CSV
 * :501) — there is no header to bind, so these entry points are named after
 * the SPEC operations.  C++ callers use coadapt/reshard.hpp directly.
 *
 * Execution is device-side: every rank's training state is one "pack" per
 * state plane (coadapt/reshard.hpp describes the pack order);
 * coadapt_reshard_execute copies the regions between packs — local
 * pointers or NVLink peers mapped with coadapt_ipc_open — in one kernel
 * launch per plane, each GPU either pulling its destination regions or
 * pushing its source regions.  Status codes and
 * coadapt_last_error() as in coadapt_cuda.h.
 */
#ifndef COADAPT_RESHARD_H_
#define COADAPT_RESHARD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COADAPT_RESHARD_MAX_DIMS 4

typedef struct coadapt_tensor_decl {
  const char* name;
  int32_t ndim;    /* 1..4 */
  int32_t tp_axis; /* -1: replicated on every TP rank */
  int64_t shape[COADAPT_RESHARD_MAX_DIMS];
} coadapt_tensor_decl;

/* ModelSpec */
typedef struct coadapt_reshard_model {
  int32_t layers;
  int32_t n_tensors; /* per layer */
  const coadapt_tensor_decl* tensors;
  int32_t optimizer_state_multiplier;
  int32_t param_bytes; /* 2 (bf16) */
  int32_t state_bytes; /* 4 (fp32) */
  int32_t reserved_;
} coadapt_reshard_model;

/* ShardDescriptor; pack_offset in elements */
typedef struct coadapt_shard {
  int32_t layer, tensor, owner, canonical;
  int64_t global_shape[COADAPT_RESHARD_MAX_DIMS];
  int64_t global_offset[COADAPT_RESHARD_MAX_DIMS];
  int64_t local_shape[COADAPT_RESHARD_MAX_DIMS];
  uint64_t pack_offset;
  int32_t ndim, reserved_;
} coadapt_shard;

/* one TransferPlan move */
typedef struct coadapt_move {
  int32_t src_rank, dst_rank, layer, tensor;
  int64_t offset[COADAPT_RESHARD_MAX_DIMS];
  int64_t extent[COADAPT_RESHARD_MAX_DIMS];
  uint64_t bytes;
  int32_t local, ndim;
} coadapt_move;

typedef struct coadapt_reshard_info {
  uint64_t n_moves;
  uint64_t total_bytes;        /* wire bytes */
  uint64_t max_bytes_per_rank; /* max wire bytes received by one rank */
  uint64_t local_bytes;
  int32_t src_ranks, dst_ranks;
  uint64_t src_max_pack_numel, dst_max_pack_numel;
} coadapt_reshard_info;

#define COADAPT_RESHARD_CANONICAL 0 /* read DP replica 0 */
#define COADAPT_RESHARD_SPREAD 1    /* read replica (dst i_d mod src d) */

#define COADAPT_RESHARD_SRC 0
#define COADAPT_RESHARD_DST 1

typedef struct coadapt_reshard_plan coadapt_reshard_plan;

/* layout_for both strategies + plan_transfers.  strategies are {d,t,p}. */
int coadapt_reshard_plan_create(const coadapt_reshard_model* model,
                                const int32_t src_dtp[3],
                                const int32_t dst_dtp[3], int policy,
                                coadapt_reshard_plan** out);
int coadapt_reshard_plan_destroy(coadapt_reshard_plan* plan);
int coadapt_reshard_plan_info(const coadapt_reshard_plan* plan,
                              coadapt_reshard_info* out);
/* *count: in = capacity, out = number of moves (call with cap 0 to size) */
int coadapt_reshard_moves(const coadapt_reshard_plan* plan, coadapt_move* out,
                          size_t* count);
/* side: COADAPT_RESHARD_SRC / _DST */
int coadapt_reshard_shards(const coadapt_reshard_plan* plan, int side,
                           coadapt_shard* out, size_t* count);
int coadapt_reshard_pack_numel(const coadapt_reshard_plan* plan, int side,
                               int rank, uint64_t* numel);
/* "key,src_rank,dst_rank,offsets,extents,bytes,local" */
int coadapt_reshard_plan_csv(const coadapt_reshard_plan* plan, char* buf,
                             size_t cap, size_t* needed);
/* fixed_overhead_s + wire bytes / bandwidth */
int coadapt_reshard_latency(const coadapt_reshard_plan* plan,
                            double bandwidth_bytes_per_s,
                            double fixed_overhead_s, double* seconds);

/* Execute the plan for one state plane of elem_bytes (1, 2, 4 or 8) bytes
 * per element.  src_packs[r] is source rank r's pack, dst_packs[r]
 * destination rank r's pack (NULL where this call touches nothing).
 *   role COADAPT_RESHARD_ALL:  every move (all packs visible to this
 *                              process, e.g. virtual ranks on one GPU);
 *   role COADAPT_RESHARD_PULL: the moves INTO `rank` — this GPU reads the
 *                              sources (its own and NVLink peers);
 *   role COADAPT_RESHARD_PUSH: the moves OUT OF `rank` — this GPU writes
 *                              the destinations (its own and NVLink peers).
 * Every rank running PULL (or every rank running PUSH) executes the plan
 * exactly once.  Source and destination packs must not overlap; the caller
 * orders the call after the sources are final and before they are freed
 * (barriers).  Stream-ordered; one kernel launch (none if nothing to copy). */
#define COADAPT_RESHARD_ALL 0
#define COADAPT_RESHARD_PULL 1
#define COADAPT_RESHARD_PUSH 2
int coadapt_reshard_execute(coadapt_reshard_plan* plan, int role, int rank,
                            const void* const* src_packs, size_t n_src,
                            void* const* dst_packs, size_t n_dst,
                            int elem_bytes, int device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COADAPT_RESHARD_H_ */
