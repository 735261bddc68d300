/*
 * oracle.h — CPU restatement of the COPUS online-GNS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 product
 * path in paper_2604_26687_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline leg and --impl reference) may load it.  The product
 * never links, imports or calls anything in oracle/.
 *
 * The reference (/root/reference, arXiv 2604.26687 artifact) ships headers
 * only (proj/include/coadapt/ headers) — there is no implementation to compile,
 * so oracle/_ref does not exist.  Every function below restates the
 * normative comments of those headers and of SPEC.md; each cites the
 * file:line it follows.  Parity pinning: the spec's golden vectors
 * are checked in tests/test_oracle.py;
 * at model-sized inputs parity is pinned only by this restatement
 * (see DESIGN.md §Oracle).
 *
 * Floating point: compiled with -O2 -ffp-contract=off (no FMA contraction)
 * so scalar formulas are IEEE-exact and reproducible.
 */
#ifndef COADAPT_ORACLE_H
#define COADAPT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types of a gradient bucket (same codes as coadapt_dtype) */
enum { ORC_BF16 = 0, ORC_FP16 = 1, ORC_FP32 = 2 };

/* weighted range of a flattened bucket, elements [offset, offset+numel) */
typedef struct {
  uint64_t offset;
  uint64_t numel;
  double weight;
} orc_segment;

/* maps a bucket range to logical (unsharded) parameter indices:
 * gidx(j) = global_base + (j / row_len) * row_stride + (j % row_len),
 * j in [0, numel), stored at bucket element local_off + j. */
typedef struct {
  uint64_t local_off;
  uint64_t numel;
  uint64_t global_base;
  uint64_t row_len;
  uint64_t row_stride;
} orc_gen_segment;

/* StepStats, gns.hpp:35-40 */
typedef struct {
  double signal;
  double noise;
  double noise_raw;
  double mean_grad_sq;
} orc_stats;

/* GnsState, gns.hpp:53-62 */
typedef struct {
  double ema_signal;
  double ema_noise;
  double alpha_early;
  double alpha_late;
  int64_t phase_boundary_tokens;
  int64_t tokens_seen;
  double calibration;
  int32_t initialized;
  int32_t pad_;
} orc_state;

/* ---- squared norms (Alg. 1 line "Local squared norm") ---- */

/* s = sum_seg weight * sum_{i in seg} x_i^2, each x_i^2 and every sum in
 * fp64, strictly sequential order.  PAPER.md:439; dedup weights per
 * SPEC.md:419-423,448 (replicated tensors carry weight 0 on tp_rank != 0). */
double orc_sqnorm(const void* buf, int dtype, const orc_segment* segs,
                  size_t nseg);

/* same value, computed with `nthreads` OpenMP threads over fixed 1 Mi-element
 * chunks combined in index order (deterministic; CPU baseline). */
double orc_sqnorm_mt(const void* buf, int dtype, const orc_segment* segs,
                     size_t nseg, int nthreads);

/* Fused d=1 pass over M resident micro-buckets:
 * s_out[m] = orc_sqnorm(bufs[m]) for every m, and
 * *sum_sq_out = sum_seg w * sum_i (S_i)^2 with S_i = fp32 sequential sum over
 * m of x_{m,i} (Megatron main_grad accumulation), squared and summed in fp64.
 * gbar^2 = *sum_sq_out / (M*M) for d = 1. */
void orc_fused_sqnorms(const void* const* bufs, int M, int dtype,
                       const orc_segment* segs, size_t nseg, int nthreads,
                       double* s_out, double* sum_sq_out);

/* ---- estimator, gns.hpp:42-73 ---- */

/* finalize_step, gns.hpp:42-49.  Returns 0 on success,
 * 1 (validation) if n < 2 or any s is negative / NaN
 * (gns.hpp:19). */
int orc_finalize_step(const double* s, int64_t n, double mean_grad_sq,
                      int64_t global_batch, orc_stats* out);

/* sum_i v_i^2 in fp64, sequential (gns.hpp:45-46: overload taking the mean
 * gradient computes gbar^2 itself). */
double orc_sumsq_f64(const double* v, uint64_t n);

/* update_ema, gns.hpp:64-68 */
void orc_update_ema(orc_state* st, const orc_stats* stats,
                    int64_t tokens_this_step);

/* gns, gns.hpp:70-73.  Returns 1 and writes *phi when available. */
int orc_gns(const orc_state* st, double* phi);

/* ---- goodput scorer, goodput.hpp:20-48; SPEC.md:253-311 ---- */
double orc_stat_eff(double global_batch, double phi);
double orc_goodput(double throughput, double se);
double orc_goodput_lr(double throughput, double global_batch, double phi,
                      double reference_batch);
double orc_lr_rescale(double eta, double b_old, double b_new);
double orc_optimal_batch_continuous(double b_hw, double b_crit_scaled);
int64_t orc_cbs_target(double phi, const int64_t* cands, size_t n,
                       int linear);

/* ---- candidate table + decide, SPEC.md:74-112, 361-375 ---- */
typedef struct {
  int32_t d, t, p, pad_;
  int64_t global_batch;
  int64_t micro_batch;
  double throughput;
  double peak_memory;
  int32_t feasible;
  int32_t pad2_;
} orc_entry;

typedef struct {
  int32_t d, t, p, pad_;
  double t_max;
  double b_hw;
} orc_cost;

/* synth_profile.  Fills up to cap entries in (strategy,
 * B_g, B_m) order; returns the count. Non-divisible (B_g mod d*B_m != 0)
 * tuples are skipped. */
size_t orc_synth_profile(const orc_cost* costs, size_t ncost,
                         const int64_t* bg, size_t nbg, const int64_t* bm,
                         size_t nbm, int bubble, double model_bytes,
                         double act_bytes_per_sample, double mem_cap,
                         orc_entry* out, size_t cap);

/* feasible_candidates, SPEC.md:104-112 (fastest B_m per (S,B_g), ties →
 * smaller B_m; sorted by B_g, d, t, p).  Returns count. */
size_t orc_feasible_candidates(const orc_entry* entries, size_t n,
                               orc_entry* out, size_t cap);

typedef struct {
  double margin;          /* epsilon */
  double max_growth;
  double reconfig_cost;   /* c_reconfig seconds */
  double reference_batch; /* B_g^ref */
} orc_orch_cfg;

enum { ORC_NOOP = 0, ORC_SCALE_BS = 1, ORC_RECONFIGURE = 2 };

typedef struct {
  int32_t kind;
  int32_t winner_index; /* index into candidates, -1 if none */
  double winner_score;
  double current_score;
  int32_t penalized;
  int32_t pad_;
} orc_command;

/* record_reconfig: T_elapsed += latency (T_useful does
 * not move); c_reconfig = mean of all observed latencies.  Returns 1 for
 * latency < 0 (validation), else 0. */
int orc_record_reconfig(double* elapsed, double* useful, double* total,
                        int64_t* count, double* reconfig_cost, double latency);

/* decide, SPEC.md:361-375 / Alg. 2 PAPER.md:490-515.  Returns 0 ok, 1 on
 * validation error (empty candidates, current absent). */
int orc_decide(const orc_entry* cands, size_t n, int phi_available,
               double phi, const orc_entry* current, double t_elapsed,
               double t_useful, const orc_orch_cfg* cfg, orc_command* out);

/* scores[i] = goodput_lr (penalised for S' != S) for every candidate. */
void orc_score_candidates(const orc_entry* cands, size_t n, double phi,
                          const orc_entry* current, double t_elapsed,
                          double t_useful, const orc_orch_cfg* cfg,
                          double* scores);

/* ---- synthetic gradient source (integer-exact) ---- */

/* x = G_i + zeta_{n,i}, G_i = +-g0 (sign from hash(seed, gidx)), zeta =
 * float(IrwinHall4 integer) * noise_unit, rounded RNE to dtype.  Bit-exact
 * twin of the device generator K0 (synth_kernel in
 * paper_2604_26687_b200/csrc/kernels.cu). */
void orc_synth_fill(void* dst, int dtype, const orc_gen_segment* segs,
                    size_t nseg, uint64_t seed, uint64_t sample, float g0,
                    float noise_unit);

/* synchronised mean gradient for d > 1: RNE_dtype( fp32_seq_sum_{n<N}
 * x_{n,i} * (1/N as float) ), samples n = sample0 .. sample0+N-1. */
void orc_synth_mean_fill(void* dst, int dtype, const orc_gen_segment* segs,
                         size_t nseg, uint64_t seed, uint64_t sample0,
                         int64_t nsamples, float g0, float noise_unit);

/* std-dev of the integer Irwin–Hall(4, 16-bit) draw; noise_unit =
 * desired_std / ORC_IH_STD. */
double orc_ih_std(void);

/* simulate_micro_gradients, gns.hpp:75-80 (statistical semantics only;
 * RNG is the oracle's own).  out is count*n doubles, row-major. */
void orc_simulate_micro_gradients(const double* g_true, const double* sigma,
                                  uint64_t n, int64_t micro_batch, int count,
                                  uint64_t seed, double* out);

/* FNV-1a over a byte range (buffer fingerprints in tests) */
uint64_t orc_fnv1a(const void* p, uint64_t nbytes);

#ifdef __cplusplus
}
#endif
#endif
