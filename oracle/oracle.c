/*
 * oracle.c — CPU restatement of the COPUS online-GNS hot path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked by the product.
 */
#include "oracle.h"

#include <math.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* element decode                                                     */
/* ------------------------------------------------------------------ */

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline float f16_to_f32(uint16_t h) {
  _Float16 x;
  memcpy(&x, &h, 2);
  return (float)x;
}

static inline uint16_t f32_to_f16_rne(float f) {
  _Float16 x = (_Float16)f;
  uint16_t h;
  memcpy(&h, &x, 2);
  return h;
}

static inline double load_elem(const void* buf, int dtype, uint64_t i) {
  switch (dtype) {
    case ORC_BF16:
      return (double)bf16_to_f32(((const uint16_t*)buf)[i]);
    case ORC_FP16:
      return (double)f16_to_f32(((const uint16_t*)buf)[i]);
    default:
      return (double)((const float*)buf)[i];
  }
}

static inline float load_elem_f(const void* buf, int dtype, uint64_t i) {
  switch (dtype) {
    case ORC_BF16:
      return bf16_to_f32(((const uint16_t*)buf)[i]);
    case ORC_FP16:
      return f16_to_f32(((const uint16_t*)buf)[i]);
    default:
      return ((const float*)buf)[i];
  }
}

/* ------------------------------------------------------------------ */
/* squared norms                                                      */
/* ------------------------------------------------------------------ */

double orc_sqnorm(const void* buf, int dtype, const orc_segment* segs,
                  size_t nseg) {
  double total = 0.0;
  for (size_t s = 0; s < nseg; ++s) {
    if (segs[s].weight == 0.0) continue; /* replicated copy: not counted */
    double acc = 0.0;
    const uint64_t b = segs[s].offset, e = b + segs[s].numel;
    for (uint64_t i = b; i < e; ++i) {
      const double x = load_elem(buf, dtype, i);
      acc += x * x;
    }
    total += segs[s].weight * acc;
  }
  return total;
}

/* work item: one <= 1 Mi-element piece of one weighted segment */
typedef struct {
  uint64_t begin, end;
  double weight;
} work_item;

#define ORC_CHUNK (1ull << 20)

static size_t build_items(const orc_segment* segs, size_t nseg,
                          work_item* items, size_t cap) {
  size_t k = 0;
  for (size_t s = 0; s < nseg; ++s) {
    if (segs[s].weight == 0.0) continue;
    for (uint64_t b = segs[s].offset; b < segs[s].offset + segs[s].numel;
         b += ORC_CHUNK) {
      uint64_t e = b + ORC_CHUNK;
      if (e > segs[s].offset + segs[s].numel) e = segs[s].offset + segs[s].numel;
      if (items && k < cap) {
        items[k].begin = b;
        items[k].end = e;
        items[k].weight = segs[s].weight;
      }
      ++k;
    }
  }
  return k;
}

/* 8 independent fp64 lanes (lane j takes i = j mod 8), combined in lane
 * order: a fixed association that the compiler can vectorise. */
static double range_sumsq_lanes(const void* buf, int dtype, uint64_t b,
                                uint64_t e) {
  double lane[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint64_t i = b;
  if (dtype == ORC_BF16) {
    const uint16_t* p = (const uint16_t*)buf;
    for (; i + 8 <= e; i += 8)
      for (int j = 0; j < 8; ++j) {
        const double x = (double)bf16_to_f32(p[i + j]);
        lane[j] += x * x;
      }
  } else if (dtype == ORC_FP32) {
    const float* p = (const float*)buf;
    for (; i + 8 <= e; i += 8)
      for (int j = 0; j < 8; ++j) {
        const double x = (double)p[i + j];
        lane[j] += x * x;
      }
  }
  for (; i < e; ++i) {
    const double x = load_elem(buf, dtype, i);
    lane[i & 7] += x * x;
  }
  double s = 0.0;
  for (int j = 0; j < 8; ++j) s += lane[j];
  return s;
}

#include <stdlib.h>

double orc_sqnorm_mt(const void* buf, int dtype, const orc_segment* segs,
                     size_t nseg, int nthreads) {
  const size_t n = build_items(segs, nseg, NULL, 0);
  if (n == 0) return 0.0;
  work_item* items = (work_item*)malloc(n * sizeof(work_item));
  double* part = (double*)malloc(n * sizeof(double));
  build_items(segs, nseg, items, n);
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (long k = 0; k < (long)n; ++k)
    part[k] = items[k].weight *
              range_sumsq_lanes(buf, dtype, items[k].begin, items[k].end);
  double total = 0.0;
  for (size_t k = 0; k < n; ++k) total += part[k];
  free(items);
  free(part);
  return total;
}

void orc_fused_sqnorms(const void* const* bufs, int M, int dtype,
                       const orc_segment* segs, size_t nseg, int nthreads,
                       double* s_out, double* sum_sq_out) {
  const size_t n = build_items(segs, nseg, NULL, 0);
  for (int m = 0; m < M; ++m) s_out[m] = 0.0;
  *sum_sq_out = 0.0;
  if (n == 0 || M <= 0) return;
  work_item* items = (work_item*)malloc(n * sizeof(work_item));
  double* part = (double*)malloc(n * (size_t)(M + 1) * sizeof(double));
  build_items(segs, nseg, items, n);
  if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (long k = 0; k < (long)n; ++k) {
    double* pk = part + (size_t)k * (M + 1);
    for (int m = 0; m < M; ++m)
      pk[m] = range_sumsq_lanes(bufs[m], dtype, items[k].begin, items[k].end);
    /* 8 fp64 lanes (lane j takes i = j mod 8) combined in lane order, the
     * same fixed association as range_sumsq_lanes */
    double lane[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t i = items[k].begin; i < items[k].end; ++i) {
      float sum = 0.0f; /* Megatron main_grad: fp32, micro-batches in order */
      for (int m = 0; m < M; ++m) sum = sum + load_elem_f(bufs[m], dtype, i);
      const double sd = (double)sum;
      lane[i & 7] += sd * sd;
    }
    double acc = 0.0;
    for (int j = 0; j < 8; ++j) acc += lane[j];
    for (int m = 0; m < M; ++m) pk[m] *= items[k].weight;
    pk[M] = items[k].weight * acc;
  }
  for (size_t k = 0; k < n; ++k) {
    const double* pk = part + k * (size_t)(M + 1);
    for (int m = 0; m < M; ++m) s_out[m] += pk[m];
    *sum_sq_out += pk[M];
  }
  free(items);
  free(part);
}

double orc_sumsq_f64(const double* v, uint64_t n) {
  double acc = 0.0;
  for (uint64_t i = 0; i < n; ++i) acc += v[i] * v[i];
  return acc;
}

/* ------------------------------------------------------------------ */
/* estimator                                                          */
/* ------------------------------------------------------------------ */

int orc_finalize_step(const double* s, int64_t n, double mean_grad_sq,
                      int64_t global_batch, orc_stats* out) {
  /* gns.hpp:45 "Requires N >= 2" */
  if (n < 2) return 1;
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(s[i] >= 0.0)) return 1; /* gns.hpp:19; NaN rejected too */
    sum += s[i];
  }
  const double N = (double)n;
  const double sbar = sum / N;                              /* gns.hpp:42 */
  out->signal = (N * mean_grad_sq - sbar) / (N - 1.0);       /* gns.hpp:43 */
  out->noise_raw =
      (sbar - mean_grad_sq) * (double)global_batch / (N - 1.0); /* :44 */
  out->noise = out->noise_raw > 0.0 ? out->noise_raw : 0.0;     /* :37 */
  out->mean_grad_sq = mean_grad_sq;
  return 0;
}

void orc_update_ema(orc_state* st, const orc_stats* stats,
                    int64_t tokens_this_step) {
  /* alpha chosen before tokens are added (gns.hpp:51-52, 64-65) */
  const double alpha = st->tokens_seen < st->phase_boundary_tokens
                           ? st->alpha_early
                           : st->alpha_late;
  if (!st->initialized) { /* first update adopts the raw values, :65-66 */
    st->ema_signal = stats->signal;
    st->ema_noise = stats->noise;
    st->initialized = 1;
  } else {
    st->ema_signal = alpha * st->ema_signal + (1.0 - alpha) * stats->signal;
    st->ema_noise = alpha * st->ema_noise + (1.0 - alpha) * stats->noise;
  }
  if (st->ema_noise < 0.0) st->ema_noise = 0.0; /* :66 clamp */
  st->tokens_seen += tokens_this_step;
}

int orc_gns(const orc_state* st, double* phi) {
  if (!(st->ema_signal > 0.0)) return 0; /* gns.hpp:70-72 */
  *phi = st->calibration * st->ema_noise / st->ema_signal;
  return 1;
}

/* ------------------------------------------------------------------ */
/* goodput                                                            */
/* ------------------------------------------------------------------ */

double orc_stat_eff(double b, double phi) { return (1.0 + phi) / (b + phi); }
double orc_goodput(double t, double se) { return t * se; }
double orc_goodput_lr(double t, double b, double phi, double ref) {
  return t * orc_stat_eff(b, phi) * sqrt(b / ref);
}
double orc_lr_rescale(double eta, double b_old, double b_new) {
  return eta * sqrt(b_new / b_old);
}
double orc_optimal_batch_continuous(double b_hw, double b_crit) {
  return sqrt(b_hw * b_crit);
}
int64_t orc_cbs_target(double phi, const int64_t* c, size_t n, int linear) {
  const double target = phi > 1.0 ? phi : 1.0;
  int64_t best = 0;
  double best_d = INFINITY;
  /* log2 keeps power-of-two grids exact; distances within 1e-12 are a tie
   * ("exactly at geometric midpoint -> smaller one") */
  for (size_t i = 0; i < n; ++i) {
    const double d = linear ? fabs((double)c[i] - target)
                            : fabs(log2((double)c[i]) - log2(target));
    if (d < best_d - 1e-12 || (fabs(d - best_d) <= 1e-12 && c[i] < best)) {
      best_d = d;
      best = c[i];
    }
  }
  return best;
}

/* ------------------------------------------------------------------ */
/* profile + decide                                                   */
/* ------------------------------------------------------------------ */

size_t orc_synth_profile(const orc_cost* costs, size_t ncost,
                         const int64_t* bg, size_t nbg, const int64_t* bm,
                         size_t nbm, int bubble, double model_bytes,
                         double act_bytes, double mem_cap, orc_entry* out,
                         size_t cap) {
  size_t k = 0;
  for (size_t s = 0; s < ncost; ++s)
    for (size_t i = 0; i < nbg; ++i)
      for (size_t j = 0; j < nbm; ++j) {
        const int64_t d = costs[s].d;
        if (bg[i] % (d * bm[j]) != 0) continue;
        const int64_t ga = bg[i] / (d * bm[j]);
        double t = costs[s].t_max * (double)bg[i] /
                   ((double)bg[i] + costs[s].b_hw);
        if (bubble)
          t *= (double)ga / (double)(ga + costs[s].p - 1);
        const double mem = model_bytes / (double)(costs[s].t * costs[s].p) +
                           act_bytes * (double)bm[j];
        if (k < cap) {
          orc_entry* e = out + k;
          memset(e, 0, sizeof(*e));
          e->d = costs[s].d;
          e->t = costs[s].t;
          e->p = costs[s].p;
          e->global_batch = bg[i];
          e->micro_batch = bm[j];
          e->peak_memory = mem;
          e->feasible = mem <= mem_cap;
          e->throughput = e->feasible ? t : 0.0;
        }
        ++k;
      }
  return k;
}

static int cand_order(const orc_entry* a, const orc_entry* b) {
  if (a->global_batch != b->global_batch)
    return a->global_batch < b->global_batch ? -1 : 1;
  if (a->d != b->d) return a->d < b->d ? -1 : 1;
  if (a->t != b->t) return a->t < b->t ? -1 : 1;
  if (a->p != b->p) return a->p < b->p ? -1 : 1;
  return 0;
}

size_t orc_feasible_candidates(const orc_entry* e, size_t n, orc_entry* out,
                               size_t cap) {
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    if (!e[i].feasible) continue;
    /* is there an entry with the same (S, B_g) that beats this one? */
    int dominated = 0;
    for (size_t j = 0; j < n && !dominated; ++j) {
      if (j == i || !e[j].feasible) continue;
      if (e[j].d != e[i].d || e[j].t != e[i].t || e[j].p != e[i].p ||
          e[j].global_batch != e[i].global_batch)
        continue;
      if (e[j].throughput > e[i].throughput ||
          (e[j].throughput == e[i].throughput &&
           e[j].micro_batch < e[i].micro_batch))
        dominated = 1; /* SPEC.md:87 fastest, ties -> smaller B_m */
    }
    if (!dominated && k < cap) out[k++] = e[i];
  }
  /* insertion sort by (B_g, d, t, p) */
  for (size_t i = 1; i < k; ++i) {
    orc_entry x = out[i];
    size_t j = i;
    while (j > 0 && cand_order(&out[j - 1], &x) > 0) {
      out[j] = out[j - 1];
      --j;
    }
    out[j] = x;
  }
  return k;
}

static int same_strategy(const orc_entry* a, const orc_entry* b) {
  return a->d == b->d && a->t == b->t && a->p == b->p;
}
static int same_config(const orc_entry* a, const orc_entry* b) {
  return same_strategy(a, b) && a->global_batch == b->global_batch &&
         a->micro_batch == b->micro_batch;
}

void orc_score_candidates(const orc_entry* c, size_t n, double phi,
                          const orc_entry* cur, double t_elapsed,
                          double t_useful, const orc_orch_cfg* cfg,
                          double* scores) {
  for (size_t i = 0; i < n; ++i) {
    double g = orc_goodput_lr(c[i].throughput, (double)c[i].global_batch, phi,
                              cfg->reference_batch);
    if (!same_strategy(&c[i], cur))
      g = g * t_useful / (t_elapsed + cfg->reconfig_cost);
    scores[i] = g;
  }
}

/* tie-break: prefer current, then smaller B_g, then larger d;
 * (then larger t, smaller B_m: oracle's documented completion) */
static int tie_better(const orc_entry* a, const orc_entry* b,
                      const orc_entry* cur) {
  const int ac = same_config(a, cur), bc = same_config(b, cur);
  if (ac != bc) return ac;
  if (a->global_batch != b->global_batch)
    return a->global_batch < b->global_batch;
  if (a->d != b->d) return a->d > b->d;
  if (a->t != b->t) return a->t > b->t;
  return a->micro_batch < b->micro_batch;
}

/* SPEC.md:377-385 */
int orc_record_reconfig(double* elapsed, double* useful, double* total,
                        int64_t* count, double* reconfig_cost, double latency) {
  (void)useful; /* "useful does not" advance */
  if (!(latency >= 0.0)) return 1;
  *elapsed += latency;
  *total += latency;
  *count += 1;
  *reconfig_cost = *total / (double)*count;
  return 0;
}

int orc_decide(const orc_entry* c, size_t n, int phi_available, double phi,
               const orc_entry* cur, double t_elapsed, double t_useful,
               const orc_orch_cfg* cfg, orc_command* out) {
  memset(out, 0, sizeof(*out));
  out->winner_index = -1;
  if (n == 0) return 1;
  if (!phi_available) return 0; /* NoOp */
  out->current_score = orc_goodput_lr(cur->throughput,
                                      (double)cur->global_batch, phi,
                                      cfg->reference_batch); /* unpenalised */
  long best = -1;
  double best_score = 0.0;
  for (size_t i = 0; i < n; ++i) {
    if ((double)c[i].global_batch >
        cfg->max_growth * (double)cur->global_batch)
      continue; /* growth clamp */
    double g = orc_goodput_lr(c[i].throughput, (double)c[i].global_batch, phi,
                              cfg->reference_batch);
    if (!same_strategy(&c[i], cur))
      g = g * t_useful / (t_elapsed + cfg->reconfig_cost);
    if (best < 0 || g > best_score ||
        (g == best_score && tie_better(&c[i], &c[best], cur))) {
      best = (long)i;
      best_score = g;
    }
  }
  if (best < 0) return 0;
  out->winner_index = (int32_t)best;
  out->winner_score = best_score;
  out->penalized = !same_strategy(&c[best], cur);
  if (same_config(&c[best], cur)) return 0; /* NoOp */
  if ((best_score - out->current_score) / out->current_score < cfg->margin)
    return 0; /* NoOp */
  out->kind = same_strategy(&c[best], cur) ? ORC_SCALE_BS : ORC_RECONFIGURE;
  return 0;
}

/* ------------------------------------------------------------------ */
/* synthetic gradients                                                */
/* ------------------------------------------------------------------ */

static inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline uint64_t sample_key(uint64_t seed, uint64_t sample) {
  return mix64(seed ^ mix64(sample + 0x632BE59BD9B4E019ull));
}
static inline uint64_t sign_key(uint64_t seed) {
  return mix64(seed ^ 0xA0761D6478BD642Full);
}

/* one synthetic element as fp32 before dtype rounding */
static inline float synth_value(uint64_t skey, uint64_t gkey, uint64_t gidx,
                                float g0, float noise_unit) {
  const uint64_t h = mix64(skey ^ gidx);
  const int32_t ih = (int32_t)((h & 0xffff) + ((h >> 16) & 0xffff) +
                               ((h >> 32) & 0xffff) + (h >> 48)) -
                     131070;
  const float zeta = (float)ih * noise_unit;
  const float g = (mix64(gkey ^ gidx) >> 63) ? -g0 : g0;
  return g + zeta;
}

static inline void store_elem(void* dst, int dtype, uint64_t i, float v) {
  switch (dtype) {
    case ORC_BF16:
      ((uint16_t*)dst)[i] = f32_to_bf16_rne(v);
      break;
    case ORC_FP16:
      ((uint16_t*)dst)[i] = f32_to_f16_rne(v);
      break;
    default:
      ((float*)dst)[i] = v;
  }
}

static inline float round_trip(int dtype, float v) {
  switch (dtype) {
    case ORC_BF16:
      return bf16_to_f32(f32_to_bf16_rne(v));
    case ORC_FP16:
      return f16_to_f32(f32_to_f16_rne(v));
    default:
      return v;
  }
}

static inline uint64_t gen_gidx(const orc_gen_segment* s, uint64_t j) {
  return s->global_base + (j / s->row_len) * s->row_stride + (j % s->row_len);
}

void orc_synth_fill(void* dst, int dtype, const orc_gen_segment* segs,
                    size_t nseg, uint64_t seed, uint64_t sample, float g0,
                    float noise_unit) {
  const uint64_t skey = sample_key(seed, sample), gkey = sign_key(seed);
  for (size_t s = 0; s < nseg; ++s) {
#pragma omp parallel for schedule(static)
    for (long long j = 0; j < (long long)segs[s].numel; ++j) {
      const uint64_t gidx = gen_gidx(&segs[s], (uint64_t)j);
      store_elem(dst, dtype, segs[s].local_off + (uint64_t)j,
                 synth_value(skey, gkey, gidx, g0, noise_unit));
    }
  }
}

void orc_synth_mean_fill(void* dst, int dtype, const orc_gen_segment* segs,
                         size_t nseg, uint64_t seed, uint64_t sample0,
                         int64_t nsamples, float g0, float noise_unit) {
  const uint64_t gkey = sign_key(seed);
  const float inv_n = (float)(1.0 / (double)nsamples);
  for (size_t s = 0; s < nseg; ++s) {
#pragma omp parallel for schedule(static)
    for (long long j = 0; j < (long long)segs[s].numel; ++j) {
      const uint64_t gidx = gen_gidx(&segs[s], (uint64_t)j);
      float acc = 0.0f;
      for (int64_t n = 0; n < nsamples; ++n) {
        const uint64_t skey = sample_key(seed, sample0 + (uint64_t)n);
        acc = acc + round_trip(dtype, synth_value(skey, gkey, gidx, g0,
                                                  noise_unit));
      }
      store_elem(dst, dtype, segs[s].local_off + (uint64_t)j, acc * inv_n);
    }
  }
}

double orc_ih_std(void) { return sqrt((4294967296.0 - 1.0) / 3.0); }

void orc_simulate_micro_gradients(const double* g_true, const double* sigma,
                                  uint64_t n, int64_t micro_batch, int count,
                                  uint64_t seed, double* out) {
  const double two_pi = 6.283185307179586476925286766559;
  for (int c = 0; c < count; ++c) {
    const uint64_t key = sample_key(seed, (uint64_t)c);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t h1 = mix64(key ^ (2 * i)), h2 = mix64(key ^ (2 * i + 1));
      const double u1 = ((double)(h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
      const double u2 = (double)(h2 >> 11) * (1.0 / 9007199254740992.0);
      const double z = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
      out[(size_t)c * n + i] =
          g_true[i] + z * sqrt(sigma[i] / (double)micro_batch);
    }
  }
}

uint64_t orc_fnv1a(const void* p, uint64_t nbytes) {
  const unsigned char* b = (const unsigned char*)p;
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < nbytes; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
