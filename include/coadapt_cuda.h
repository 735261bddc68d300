/*
 * coadapt_cuda.h — C-ABI of the B200 GNS hot path (libcoadapt_b200.so).
 *
 * The reference (arXiv 2604.26687 artifact, proj/include/coadapt/) exposes
 * the hot path as a C++ API whose inputs are host scalars and host spans:
 * callers compute s_m themselves and pass it to
 *   StepAccumulator::record_micro_batch(double)        gns.hpp:19-20
 * and the mean-gradient norm goes through
 *   finalize_step(acc, std::span<const double>)        gns.hpp:47-48
 *   finalize_step(acc, double mean_grad_sq)            gns.hpp:49
 * followed by update_ema (gns.hpp:67-68) and gns() (gns.hpp:73); the
 * all-reduce of Algorithm 1 is "modeled as summation over the
 * lists" (gns.hpp:11-14).  This header is the device-resident
 * replacement a foreign-language binding (ctypes, cgo, JNI, N-API) would bind:
 * plain pointers and sizes, no C++ or torch types, no exceptions.  Each entry
 * point names the reference interface it replaces.
 *
 * Conventions
 *  - every function returns a status: COADAPT_OK or one of the COADAPT_E_*
 *    codes, which mirror the exception taxonomy of errors.hpp:8-27 (and the
 *    CLI exit codes of SPEC.md:635); coadapt_last_error() returns the
 *    thread-local message of the last failure on the calling thread.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  All device work is asynchronous on that stream; only
 *    coadapt_gns_read_result / coadapt_gns_read_partials block
 *    (coadapt_gns_result_ready polls without blocking).
 *  - device gradient buffers are borrowed (like std::span): the library never
 *    frees or retains them past the call's stream work.  Host buffers given
 *    to coadapt_gns_fused_sqnorm_host must stay valid until that stream work
 *    completes (pinned memory for the copies to overlap).
 *  - one coadapt_gns per (device, stream); it is not thread-safe, and its
 *    launches share scratch (per-CTA partials, a completion ticket), so all
 *    calls on one coadapt_gns must be ordered on one stream (or streams
 *    joined by events).  Plans are read-only after creation and may be
 *    shared: coadapt_plan_create builds every device table any launch of
 *    the plan can use (the TMA chunk numbering for every batch size 1..16
 *    and fused M, the trainer form's whole-bucket table), so no launch
 *    allocates or copies synchronously and begin_step .. finalize (and
 *    allreduce_finalize_p2p, whose epoch counter lives in device memory)
 *    are capturable into a CUDA graph and replayable without an eager
 *    warm-up call.
 */
#ifndef COADAPT_CUDA_H
#define COADAPT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COADAPT_ABI_VERSION 1

/* status codes (errors.hpp:8-27) */
#define COADAPT_OK 0
#define COADAPT_E_VALIDATION 1 /* ValidationError: contract violated (errors.hpp:10) */
#define COADAPT_E_INTERNAL 2   /* InternalError: library bug (errors.hpp:24) */
#define COADAPT_E_CUDA 3       /* CUDA runtime / device failure */
#define COADAPT_E_NCCL 4       /* NCCL failure */

/* gradient element types */
#define COADAPT_BF16 0
#define COADAPT_FP16 1
#define COADAPT_FP32 2
#define COADAPT_FP64 3

/* A weighted range of a rank's flattened gradient bucket, in elements.
 * weight 0 marks a tensor that another rank already counts (a TP-replicated
 * norm/bias on tp_rank != 0, the tied-embedding copy on the last PP stage):
 * its bytes are never loaded.  Derived from ModelSpec.tp_split_axis = none
 * and layout_for replication. */
typedef struct coadapt_segment {
  uint64_t offset;
  uint64_t numel;
  double weight;
} coadapt_segment;

/* Synthetic-gradient layout: bucket elements [local_off, local_off+numel)
 * hold logical parameter indices
 *   global_base + (j / row_len) * row_stride + (j % row_len). */
typedef struct coadapt_gen_segment {
  uint64_t local_off;
  uint64_t numel;
  uint64_t global_base;
  uint64_t row_len;
  uint64_t row_stride;
} coadapt_gen_segment;

/* StepStats, gns.hpp:35-40 */
typedef struct coadapt_step_stats {
  double signal;
  double noise;
  double noise_raw;
  double mean_grad_sq;
} coadapt_step_stats;

/* GnsState, gns.hpp:53-62 (field order and defaults identical) */
typedef struct coadapt_gns_state {
  double ema_signal;
  double ema_noise;
  double alpha_early;           /* 0.95 */
  double alpha_late;            /* 0.99 */
  int64_t phase_boundary_tokens; /* 8'000'000 */
  int64_t tokens_seen;
  double calibration;           /* 2.0 */
  int32_t initialized;
  int32_t reserved_;
} coadapt_gns_state;

/* Everything one optimizer step produces. */
typedef struct coadapt_gns_result {
  coadapt_step_stats stats;  /* finalize_step, gns.hpp:47-49 */
  coadapt_gns_state state;   /* after update_ema, gns.hpp:67-68 */
  double phi;                /* gns(), gns.hpp:73; NaN while unavailable */
  double b_simple;           /* this step's noise / signal (uncalibrated) */
  int64_t sample_count;      /* N = d * M */
  int32_t phi_available;
  int32_t status;            /* COADAPT_OK, or COADAPT_E_VALIDATION when a
                                partial was negative/non-finite (gns.hpp:19);
                                the state is then left unchanged */
} coadapt_gns_result;

typedef struct coadapt_plan coadapt_plan; /* one bucket layout */
typedef struct coadapt_gns coadapt_gns;   /* one step accumulator + GnsState */

/* ---------------------------------------------------------------- misc */
const char* coadapt_last_error(void);
int coadapt_abi_version(void);
/* number of kernels this library has launched in this process */
uint64_t coadapt_kernel_launches(void);
/* device properties the kernels size themselves by */
int coadapt_device_info(int device, int* sm_count, int* l2_bytes,
                        int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------- plan
 * Compiles a segment table into the device range table the reductions walk.
 * Replaces nothing in the reference directly: it is the layout half of the
 * caller-side "Local squared norm" computation that feeds
 * record_micro_batch (gns.hpp:19-20). */
int coadapt_plan_create(const coadapt_segment* segs, size_t nseg,
                        uint64_t bucket_numel, int dtype, int device,
                        coadapt_plan** out);
/* the same bucket restricted to DP slice `index` of `count` equal parts of
 * its element range (the d > 1 mean-gradient read) */
int coadapt_plan_create_slice(const coadapt_segment* segs, size_t nseg,
                              uint64_t bucket_numel, int dtype, int device,
                              int index, int count, coadapt_plan** out);
int coadapt_plan_destroy(coadapt_plan* plan);
/* elements actually loaded per pass (weight != 0) and range count */
int coadapt_plan_info(const coadapt_plan* plan, uint64_t* active_elems,
                      uint64_t* nranges);

/* ---------------------------------------------------------------- step
 * coadapt_gns is the device-resident StepAccumulator (gns.hpp:15-32) of one
 * optimizer step plus a persistent GnsState (gns.hpp:53-62).  Its N+1 fp64
 * slots hold s_{i_d,m} at i_d*M + m and gbar^2 at N.
 * Replaces: StepAccumulator(int dp_size, int64_t global_batch) gns.hpp:17. */
int coadapt_gns_create(int dp_size, int micro_count, int64_t global_batch,
                       int device, coadapt_gns** out);
int coadapt_gns_destroy(coadapt_gns* g);
/* Scale-BS / Reconfigure: new (d, M, B_g) for the next step; keeps the EMA */
int coadapt_gns_reshape(coadapt_gns* g, int dp_size, int micro_count,
                        int64_t global_batch);
/* zero the slots (start of an optimizer step) */
int coadapt_gns_begin_step(coadapt_gns* g, void* stream);

/* s_{dp_index, micro} += sum_seg w * ||bucket[seg]||^2 (fp64).
 * Replaces: the caller's s_m computation + record_micro_batch, gns.hpp:19-20
 * (PAPER.md:437-440).  Partials of model-parallel ranks hosted on the same
 * device accumulate into the same slot in stream order. */
int coadapt_gns_micro_sqnorm(coadapt_gns* g, const coadapt_plan* plan,
                             const void* bucket, int dp_index, int micro,
                             void* stream);
/* `count` buckets sharing one plan in one launch */
int coadapt_gns_micro_sqnorm_batched(coadapt_gns* g, const coadapt_plan* plan,
                                     const void* const* buckets,
                                     const int32_t* dp_index,
                                     const int32_t* micro, int count,
                                     void* stream);
/* d == 1 fused pass over the M resident micro-buckets of this rank: every
 * s_{0,m} and gbar^2 += ||sum_m g_m||^2 / M^2 (fp32 micro-batch sum, as
 * Megatron's main_grad) in ONE read of the bytes.  1 <= M <= 16.
 * Replaces: M x (s_m + record_micro_batch) and finalize_step's own
 * ||mean_gradient||^2 (gns.hpp:45-48). */
int coadapt_gns_fused_sqnorm(coadapt_gns* g, const coadapt_plan* plan,
                             const void* const* buckets, int micro_count,
                             void* stream);
/* gbar^2 += ||mean_grad[plan]||^2 for the synchronised mean gradient
 * (this DP replica's slice).  Replaces finalize_step's mean-gradient
 * overload, gns.hpp:47-48. */
int coadapt_gns_mean_sqnorm(coadapt_gns* g, const coadapt_plan* plan,
                            const void* mean_grad, void* stream);
/* As coadapt_gns_fused_sqnorm, but the M buckets live in HOST memory
 * (pinned for overlap): chunks are streamed H2D through a staging ring
 * owned by g and reduced as they land.  This is the reference-facing path
 * for host-resident gradients (the reference's CPU call signature). */
int coadapt_gns_fused_sqnorm_host(coadapt_gns* g, const coadapt_plan* plan,
                                  const void* const* host_buckets,
                                  int micro_count, void* stream);
/* As coadapt_gns_micro_sqnorm / coadapt_gns_mean_sqnorm with the bucket (or
 * the synchronised mean gradient) in HOST memory: only the plan's span of
 * elements (a DP slice for slice plans) is streamed H2D, in whole-stage
 * windows through g's staging ring, each reduced as it lands.  The host
 * form of record_micro_batch's caller loop (gns.hpp:19-20) and of the d > 1
 * mean read. */
int coadapt_gns_micro_sqnorm_host(coadapt_gns* g, const coadapt_plan* plan,
                                  const void* host_bucket, int dp_index,
                                  int micro, void* stream);
int coadapt_gns_mean_sqnorm_host(coadapt_gns* g, const coadapt_plan* plan,
                                 const void* host_mean, void* stream);

/* Trainer form.  The gradient-accumulation add a trainer
 * does anyway — Megatron's fp32 main_grad.add_(grad) — with the GNS norms
 * fused in, over the WHOLE bucket (every element is accumulated; only
 * weight != 0 elements are counted):
 *   main_grad = (flags & FIRST) ? grad : main_grad + grad      (fp32, RN)
 *   s_{dp_index, micro} += sum w * grad^2                         (fp64)
 *   (flags & LAST_MEAN, d == 1): gbar^2 += mean_scale_sq * sum w * main_grad^2
 * so the estimate costs no HBM bytes beyond the accumulation's own.  Both
 * buffers 16-byte aligned; main_grad fp32, grad of the plan's dtype.
 * Replaces: the backward-hook norm of the paper's GNS manager
 * feeding record_micro_batch (gns.hpp:19-20). */
#define COADAPT_ACC_FIRST 1
#define COADAPT_ACC_LAST_MEAN 2
int coadapt_gns_accumulate(coadapt_gns* g, const coadapt_plan* plan,
                           float* main_grad, const void* micro_grad,
                           int dp_index, int micro, int flags,
                           double mean_scale_sq, void* stream);

/* Fused DP gradient sync + gbar^2 over NVLink.
 * replicas[q] (q < d <= 8) is DP replica q's gradient bucket mapped into this
 * process (coadapt_ipc_open; the local one for q == dp_rank), all laid out
 * as `plan` (a whole-bucket plan).  For this rank's slice [lo, hi) — the cut
 * of coadapt_plan_create_slice(index = dp_rank, count = d) — writes
 *   out_slice[i - lo] = RNE_dtype( scale * fp32(sum_q replicas[q][i]) )
 * (replicas summed in index order) and adds sum w * out^2 (fp64) to gbar^2:
 * the reduce-scatter of the Alg. 1 "standard gradient sync"
 * and the norm of its result in one pass whose loads come
 * from the peers' HBM over NVLink.  Bracket it with coadapt_gns_barrier so
 * peers' buffers are complete before and untouched until every rank is done.
 * Replaces: finalize_step(acc, span mean_gradient) gns.hpp:47-48 fed by a
 * separate all-reduce. */
/* handle (>= 64 B) of the allocation holding dev_ptr, and dev_ptr's offset
 * in it (pass *offset to the peer; it adds it to the opened base) */
int coadapt_ipc_handle(const void* dev_ptr, void* out, size_t len,
                       uint64_t* offset);
int coadapt_ipc_open(const void* handle, size_t len, int device, void** dev_ptr);
int coadapt_ipc_close(void* dev_ptr);
int coadapt_gns_barrier(coadapt_gns* g, void* stream);
int coadapt_gns_reduce_scatter_sqnorm(coadapt_gns* g, const coadapt_plan* plan,
                                      const void* const* replicas, int d,
                                      int dp_rank, void* out_slice,
                                      double scale, void* stream);
/* All-reduce form of the same pass (DDP without a distributed optimizer):
 * the synchronised slice is written back into [lo, hi) of EVERY replica
 * (in place, over NVLink for the peers') instead of into an out buffer, so
 * after the closing coadapt_gns_barrier every replica holds the whole
 * synchronised gradient RNE_dtype(scale * fp32(sum_q replicas[q][i])) and
 * gbar^2 has its norm: the reduce-scatter, the all-gather and the norm of
 * Alg. 1's gradient sync in one kernel.  Only this rank
 * touches [lo, hi) of any replica, so the in-place update cannot race.
 * Replaces: finalize_step(acc, span mean_gradient) gns.hpp:47-48 fed by a
 * separate all-reduce. */
int coadapt_gns_allreduce_sqnorm(coadapt_gns* g, const coadapt_plan* plan,
                                 void* const* replicas, int d, int dp_rank,
                                 double scale, void* stream);

/* NVLS (NVLink SHARP) buckets: the switch-reduced form of the DP gradient
 * all-reduce.  A multicast object binds one physical buffer per GPU; the
 * trainer keeps its gradient bucket in the unicast view.  Setup, every rank
 * (host barriers between the steps):
 *   rank 0: coadapt_nvls_create + coadapt_nvls_export (64-byte handle: the
 *           exporter's pid and POSIX fd, duplicated by importers with
 *           pidfd_getfd; keep rank 0's object alive while others import)
 *   others: coadapt_nvls_import(handle)
 *   all:    coadapt_nvls_add_device;  barrier;  coadapt_nvls_bind -> unicast /
 *           multicast pointers (buffer zeroed);  barrier
 * coadapt_nvls_allreduce(o, dtype, numel, dp_rank, scale, stream): for this
 * rank's slice (the coadapt_plan_create_slice cut) multimem.ld_reduce (the
 * switch adds every GPU's copy), scale, multimem.st into every GPU's buffer:
 * one bucket per link direction instead of the 2(d-1)/d of
 * coadapt_gns_allreduce_sqnorm (equal at d = 2, 1.5x less at d = 4).  fp32 buckets only (Megatron's main_grad):
 * the switch's bf16 rounding is biased (validation error).  Bracket it with
 * coadapt_gns_barrier; take gbar^2 of the slice with coadapt_gns_mean_sqnorm
 * on the unicast view (sliced plan).  The switch's summation order is its
 * own: bit-exact with the replica-order reference for d = 2, within the
 * fp32 rounding of a d-term sum for d > 2.
 * Replaces: the all-reduce feeding finalize_step(acc, span) gns.hpp:47-48. */
typedef struct coadapt_nvls coadapt_nvls;
int coadapt_nvls_create(int device, int nranks, uint64_t bytes, coadapt_nvls** out);
int coadapt_nvls_export(const coadapt_nvls* o, void* handle, size_t len);
int coadapt_nvls_import(int device, int nranks, uint64_t bytes, const void* handle,
                        size_t len, coadapt_nvls** out);
int coadapt_nvls_add_device(coadapt_nvls* o);
int coadapt_nvls_bind(coadapt_nvls* o, void** unicast, void** multicast);
uint64_t coadapt_nvls_bytes(const coadapt_nvls* o);
int coadapt_nvls_allreduce(coadapt_nvls* o, int dtype, uint64_t numel, int dp_rank,
                           double scale, void* stream);
int coadapt_nvls_destroy(coadapt_nvls* o);

/* The fused DP gradient sync + mean-gradient norm through the switch (§8
 * f2; Alg. 1 "standard gradient sync" + gbar^2): the DP
 * group's fp32 buckets are one NVLS object (coadapt_nvls_bind, `multicast` =
 * this rank's multicast view of the bucket start).  For this rank's slice of
 * the plan (the coadapt_plan_create_slice cut, dp_rank of d) every load is
 * one multimem.ld_reduce — the NVSwitch sums the d copies, so each GPU's
 * links carry its slice once instead of (d-1)/d of the bucket — and the
 * scaled result goes to out_slice (reduce-scatter, DistOpt) or, with
 * out_slice == NULL, back through the multicast address into every GPU's
 * copy (all-reduce, DDP); its weighted squared norm is added to slot N in
 * the same pass.  Bracket with coadapt_gns_barrier like the P2P forms.
 * fp32 only (the switch's bf16/fp16 rounding biases gbar^2). */
int coadapt_gns_nvls_reduce_sqnorm(coadapt_gns* g, const coadapt_plan* p,
                                   const void* multicast, int d, int dp_rank,
                                   void* out_slice, double scale, void* stream);

/* NCCL over NVLink: sum the N+1 slots over all ranks (Alg. 1 AllReduce,
 * PAPER.md:443; the reference models it as summation). */
int coadapt_nccl_unique_id(void* out, size_t len); /* len >= 128 */
int coadapt_gns_attach_nccl(coadapt_gns* g, int nranks, int rank,
                            const void* unique_id, size_t len);
int coadapt_gns_allreduce(coadapt_gns* g, void* stream);
/* One host thread driving n GPUs (one coadapt_gns per device, in rank
 * order): attach_nccl_all builds their communicators at once
 * (ncclCommInitAll); allreduce_group issues every rank's all-reduce inside
 * one ncclGroupStart/End so the single thread cannot deadlock. */
int coadapt_gns_attach_nccl_all(coadapt_gns* const* gs, int n);
int coadapt_gns_allreduce_group(coadapt_gns* const* gs, void* const* streams,
                                int n);

/* The all-reduce and the finalize as ONE kernel over NVLink peer memory
 * (no NCCL launch on the step's tail): every rank pushes its N+1 slots into
 * every rank's mailbox, raises a flag, waits for all ranks' flags, sums the
 * blocks in rank order (bit-identical on every rank) and runs the finalize.
 *   coadapt_gns_mailbox        allocate this rank's mailbox for nranks
 *                              (share it with coadapt_ipc_handle)
 *   coadapt_gns_attach_mailboxes  peers[q] = rank q's mailbox mapped here
 *                              (coadapt_ipc_open; peers[rank] = own)
 *   coadapt_gns_allreduce_finalize_p2p  replaces allreduce + finalize; every
 *                              rank must call it once per step.  A peer
 *                              that does not arrive within 10 s makes
 *                              coadapt_gns_read_result fail with status 2.
 * Up to 8 ranks (one NVSwitch domain). */
int coadapt_gns_mailbox(coadapt_gns* g, int nranks, void** mailbox);
int coadapt_gns_attach_mailboxes(coadapt_gns* g, int nranks, int rank,
                                 const void* const* peers);
int coadapt_gns_allreduce_finalize_p2p(coadapt_gns* g, int64_t tokens,
                                       void* stream);

/* finalize_step + update_ema + gns on the device (gns.hpp:42-73), one
 * thread, IEEE-exact twin of the host formulas.  Copies the result to
 * pinned host memory on `stream`.  Replaces: finalize_step(acc, double)
 * gns.hpp:49, update_ema gns.hpp:67-68, gns gns.hpp:73. */
int coadapt_gns_finalize(coadapt_gns* g, int64_t tokens_this_step,
                         void* stream);

/* The step's last reduction with the finalize in the same pass (north_star
 * item 2; Alg. 1): coadapt_gns_fused_sqnorm (d == 1) or
 * coadapt_gns_mean_sqnorm (d > 1, the last DP slice this rank reads), whose
 * last CTA, after combining the partials, runs finalize_step + update_ema +
 * gns — and first, when NVLink mailboxes are attached
 * (coadapt_gns_attach_mailboxes, world > 1), the slot exchange of
 * coadapt_gns_allreduce_finalize_p2p.  Replaces that call (or allreduce +
 * finalize) after the step's last reduction: one launch fewer per step,
 * identical results.  The result is copied to pinned memory as by
 * coadapt_gns_finalize.  Validation error for a gns with a multi-rank NCCL
 * communicator and no mailboxes (use allreduce + finalize there). */
int coadapt_gns_fused_sqnorm_finalize(coadapt_gns* g, const coadapt_plan* p,
                                      const void* const* buckets,
                                      int micro_count, int64_t tokens_this_step,
                                      void* stream);
int coadapt_gns_mean_sqnorm_finalize(coadapt_gns* g, const coadapt_plan* p,
                                     const void* mean_grad,
                                     int64_t tokens_this_step, void* stream);
/* waits for the last finalize and returns its result */
int coadapt_gns_read_result(coadapt_gns* g, coadapt_gns_result* out);
/* non-blocking: *ready = 1 once the last finalize's result has reached the
 * host (coadapt_gns_read_result then returns without waiting), 0 while the
 * step is still running.  Lets a trainer enqueue its optimizer step and the
 * next forward before it reads phi (the GNS never stalls the stream); the
 * result must be read before the next finalize is enqueued, which reuses
 * the host buffer.  Replaces nothing in the reference (its finalize_step is
 * synchronous, gns.hpp:42-49). */
int coadapt_gns_result_ready(coadapt_gns* g, int* ready);
/* synchronous read of the N+1 slots (s values, then gbar^2) */
int coadapt_gns_read_partials(coadapt_gns* g, double* out, size_t n);
/* checkpoint / restore of the device GnsState (synchronous) */
int coadapt_gns_get_state(coadapt_gns* g, coadapt_gns_state* out);
int coadapt_gns_set_state(coadapt_gns* g, const coadapt_gns_state* in);

/* ---------------------------------------------------------------- one-shot
 * ||v||^2 of a device vector of `dtype` (fp64 accumulation), synchronous.
 * Backs finalize_step(acc, std::span<const double>) (gns.hpp:47-48) when
 * called with host data via coadapt_sqnorm_host. */
int coadapt_sqnorm_device(const void* v, uint64_t n, int dtype, int device,
                          double* out, void* stream);
int coadapt_sqnorm_host(const void* v, uint64_t n, int dtype, int device,
                        double* out);

/* ---------------------------------------------------------------- synthetic
 * Deterministic synthetic micro-gradients (device twin of the CPU oracle's
 * integer-exact generator; test and benchmark data, K0).  Family of
 * simulate_micro_gradients, gns.hpp:75-80. */
int coadapt_synth_fill(void* dst, int dtype, const coadapt_gen_segment* segs,
                       size_t nseg, uint64_t seed, uint64_t sample, float g0,
                       float noise_unit, void* stream);
int coadapt_synth_mean_fill(void* dst, int dtype,
                            const coadapt_gen_segment* segs, size_t nseg,
                            uint64_t seed, uint64_t sample0, int64_t nsamples,
                            float g0, float noise_unit, void* stream);
/* a streaming write of `bytes` (L2 flush between timed iterations) */
int coadapt_l2_flush(void* scratch, uint64_t bytes, void* stream);
/* read-only streaming peak probe: sums `bytes` of `buf` (bench roofline) */
int coadapt_read_probe(const void* buf, uint64_t bytes, double* sink,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COADAPT_CUDA_H */
