/*
 * coadapt_segments.h — C-ABI of the segment-table generator (
 * C++: coadapt/segments.hpp).
 *
 * A rank's flattened gradient bucket, its weighted ranges (weight 0 for the
 * TP-replicated tensors on tp_rank != 0 and the tied-embedding copy on the
 * last PP stage) and the generator map, derived from a model description
 * and (d,t,p) under SPEC.md's layout rules.
 * The reference has no such function — its estimator takes caller-computed
 * squared norms (record_micro_batch, gns.hpp:19-20) — so this is what a
 * caller binds to get the `segs` argument of coadapt_plan_create without
 * re-deriving Megatron's sharding itself.  Status codes and
 * coadapt_last_error() as in coadapt_cuda.h.
 */
#ifndef COADAPT_SEGMENTS_H_
#define COADAPT_SEGMENTS_H_

#include <stddef.h>
#include <stdint.h>

#include "coadapt_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

#define COADAPT_STAGE_EMBED 0 /* stage 0 (and the tied head copy) */
#define COADAPT_STAGE_LAYER 1 /* repeated per layer */
#define COADAPT_STAGE_FINAL 2 /* last stage, before the head */
#define COADAPT_STAGE_HEAD 3  /* last stage (untied models only) */

typedef struct coadapt_grad_tensor {
  const char* name;
  int32_t stage;   /* COADAPT_STAGE_* */
  int32_t ndim;    /* 1..4 */
  int32_t tp_axis; /* axis split by TP, -1: replicated on every TP rank */
  int32_t reserved_;
  int64_t shape[4];
} coadapt_grad_tensor;

typedef struct coadapt_grad_model {
  const char* name;
  int32_t layers;
  int32_t tied; /* head = the first embedding tensor */
  const coadapt_grad_tensor* tensors;
  size_t n_tensors;
} coadapt_grad_model;

/* The BASELINE.json shapes: "125m", "3b", "7b", "32b".  The descriptor
 * points at library-owned storage valid for the life of the process. */
int coadapt_model_preset(const char* key, coadapt_grad_model* out);

/* Rank `rank` of (d,t,p) (tp fastest, then dp, then pp): *count = number of
 * local tensors; segs[i] / gen[i] (either may be NULL; both NULL = size
 * query) the i-th tensor's weighted range and generator map; *bucket_numel
 * the bucket length; coords = (i_d, i_t, i_p) (optional).  Validation error
 * if cap < *count (count is still written), for an invalid strategy or rank,
 * layers % p != 0, or a split axis not divisible by t. */
int coadapt_gns_segments(const coadapt_grad_model* model, int d, int t, int p,
                         int rank, coadapt_segment* segs,
                         coadapt_gen_segment* gen, size_t cap, size_t* count,
                         uint64_t* bucket_numel, int32_t coords[3]);

/* Algorithmic bytes of one GNS step: every rank's counted
 * shard x micro_count x elem_bytes, plus the synchronised mean gradient
 * once per box when d > 1 or !fused. */
int coadapt_gns_algorithmic_bytes(const coadapt_grad_model* model, int d,
                                  int t, int p, int micro_count,
                                  int elem_bytes, int fused, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
