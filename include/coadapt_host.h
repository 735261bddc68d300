/*
 * coadapt_host.h — C bindings of the drop-in C++ API (gns.hpp, goodput.hpp,
 * strategy-aware scorer) for FFI callers (ctypes/cgo/JNI).  Implemented by
 * libcoadapt_b200.so in terms of the C++ functions; C++ exceptions become
 * status codes (errors.hpp:8-27 -> 1/1/2) and
 * coadapt_last_error() (coadapt_cuda.h) holds the message.
 */
#ifndef COADAPT_HOST_H
#define COADAPT_HOST_H

#include <stddef.h>
#include <stdint.h>

#include "coadapt_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* finalize_step(acc, double), gns.hpp:49: s holds the N recorded values. */
int coadapt_finalize_step(const double* s, int64_t n, int dp_size,
                          double mean_grad_sq, int64_t global_batch,
                          coadapt_step_stats* out);
/* finalize_step(acc, span<const double>), gns.hpp:47-48 (GPU fp64 norm). */
int coadapt_finalize_step_vec(const double* s, int64_t n, int dp_size,
                              const double* mean_gradient, uint64_t dim,
                              int64_t global_batch, coadapt_step_stats* out);
/* update_ema, gns.hpp:67-68 */
int coadapt_update_ema(coadapt_gns_state* state, const coadapt_step_stats* st,
                       int64_t tokens_this_step);
/* gns, gns.hpp:73: returns 1 and sets *phi when available, else 0 */
int coadapt_gns_phi(const coadapt_gns_state* state, double* phi);
/* default-initialised GnsState (gns.hpp:53-62) */
void coadapt_gns_state_init(coadapt_gns_state* state);

/* goodput.hpp:17-48 */
double coadapt_stat_eff(double global_batch, double phi);
double coadapt_goodput(double throughput, double stat_efficiency);
double coadapt_goodput_lr(double throughput, double global_batch, double phi,
                          double reference_batch);
double coadapt_lr_rescale(double eta, double batch_old, double batch_new);
double coadapt_optimal_batch_continuous(double batch_hw, double batch_crit);
int coadapt_cbs_target(double phi, const int64_t* candidates, size_t n,
                       int linear, int64_t* out);

/* candidate scoring */
typedef struct coadapt_candidate {
  int32_t d, t, p, reserved_;
  int64_t global_batch;
  int64_t micro_batch;
  double throughput;
} coadapt_candidate;

typedef struct coadapt_cost {
  int32_t d, t, p, reserved_;
  double t_max;
  double b_hw;
} coadapt_cost;

typedef struct coadapt_orch_cfg {
  double margin;
  double max_growth;
  double reconfig_cost;
  double reference_batch;
} coadapt_orch_cfg;

#define COADAPT_NOOP 0
#define COADAPT_SCALE_BS 1
#define COADAPT_RECONFIGURE 2

typedef struct coadapt_command {
  int32_t kind;
  int32_t winner_index; /* into candidates; -1 when none */
  double winner_score;
  double current_score;
  int32_t penalized;
  int32_t reserved_;
} coadapt_command;

/* synth_profile + feasible_candidates; *count in: capacity, out: needed */
int coadapt_synth_candidates(const coadapt_cost* costs, size_t ncost,
                             const int64_t* batch_grid, size_t nbg,
                             const int64_t* micro_grid, size_t nbm,
                             int pipeline_bubble, double model_bytes,
                             double act_bytes_per_sample, double mem_capacity,
                             coadapt_candidate* out, size_t* count);
int coadapt_score_candidates(const coadapt_candidate* c, size_t n, double phi,
                             const coadapt_candidate* current,
                             double t_elapsed, double t_useful,
                             const coadapt_orch_cfg* cfg, double* scores);
/* order[i] = index of the i-th best candidate */
int coadapt_rank_candidates(const coadapt_candidate* c, size_t n, double phi,
                            const coadapt_candidate* current, double t_elapsed,
                            double t_useful, const coadapt_orch_cfg* cfg,
                            int64_t* order);
/* record_reconfig: elapsed += latency (useful unchanged),
 * *reconfig_cost = mean of all observed latencies (total / count). */
typedef struct coadapt_clock {
  double elapsed;
  double useful;
  double reconfig_total;
  int64_t reconfigs;
} coadapt_clock;
int coadapt_record_reconfig(coadapt_clock* clock, double* reconfig_cost,
                            double observed_latency);
int coadapt_decide(const coadapt_candidate* c, size_t n, int phi_available,
                   double phi, const coadapt_candidate* current,
                   double t_elapsed, double t_useful,
                   const coadapt_orch_cfg* cfg, coadapt_command* out);

/* GNS trace CSV (gns.hpp:82-94).  Writes at most cap bytes (NUL-terminated
 * when room) and the full length to *needed. */
typedef struct coadapt_trace_row {
  int64_t step;
  int64_t tokens;
  double signal_raw;
  double noise_raw;
  double ema_signal;
  double ema_noise;
  double phi;
} coadapt_trace_row;
int coadapt_trace_csv(const coadapt_trace_row* rows, size_t n, char* buf,
                      size_t cap, size_t* needed);
/* Profile CSV.  *count: in = capacity of out,
 * out = number of entries.  Parse errors -> status 1 with the line number
 * in coadapt_last_error(). */
typedef struct coadapt_profile_entry {
  int32_t d, t, p, reserved_;
  int64_t global_batch;
  int64_t micro_batch;
  double samples_per_sec;
  double peak_mem_bytes;
  int32_t feasible;
  int32_t reserved2_;
} coadapt_profile_entry;
int coadapt_profile_parse(const char* text, size_t len,
                          coadapt_profile_entry* out, size_t* count,
                          int* n_gpus);
int coadapt_profile_format(const coadapt_profile_entry* entries, size_t n,
                           char* buf, size_t cap, size_t* needed);
int coadapt_profile_load(const char* path, coadapt_profile_entry* out,
                         size_t* count, int* n_gpus);
int coadapt_profile_save(const char* path, const coadapt_profile_entry* e,
                         size_t n);

/* Decision audit log, one row per decide() call */
typedef struct coadapt_decision_row {
  int64_t step;
  double time_s;
  double phi; /* NaN when unavailable */
  coadapt_candidate current;
  coadapt_candidate winner;
  coadapt_command command;
} coadapt_decision_row;
int coadapt_decision_audit_csv(const coadapt_decision_row* rows, size_t n,
                               char* buf, size_t cap, size_t* needed);

/* format_double, io.hpp:13 */
int coadapt_format_double(double v, char* buf, size_t cap);

/* simulate_micro_gradients, gns.hpp:78-80: out is count x n doubles */
int coadapt_simulate_micro_gradients(const double* g_true,
                                     const double* sigma, uint64_t n,
                                     int64_t micro_batch, int count,
                                     uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
