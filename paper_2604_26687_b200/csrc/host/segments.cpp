// segments.cpp — coadapt/segments.hpp: a rank's bucket segment table and
// generator map from a GradModel and (d,t,p),
// plus the C-ABI twin in coadapt_segments.h.
#include "coadapt/segments.hpp"

#include <cstring>
#include <string>

#include "coadapt/errors.hpp"
#include "coadapt_segments.h"

namespace coadapt {
namespace {

std::uint64_t prod(const std::vector<std::int64_t>& v, std::size_t b,
                   std::size_t e) {
  std::uint64_t p = 1;
  for (std::size_t i = b; i < e; ++i) p *= (std::uint64_t)v[i];
  return p;
}

void check_tensor(const GradTensor& ts) {
  if (ts.shape.empty() || ts.shape.size() > 4)
    throw ValidationError("tensor '" + ts.name + "': 1..4 axes required");
  for (auto n : ts.shape)
    if (n <= 0) throw ValidationError("tensor '" + ts.name + "': non-positive axis");
  if (ts.tp_axis < -1 || ts.tp_axis >= (int)ts.shape.size())
    throw ValidationError("tensor '" + ts.name + "': tp_axis out of range");
}

// logical (unsharded) order: embedding, layers, final, head (untied only)
template <class F>
void for_each_logical(const GradModel& m, F&& f) {
  for (const auto& ts : m.tensors)
    if (ts.stage == GradStage::kEmbed) f(ts, -1);
  for (int l = 0; l < m.layers; ++l)
    for (const auto& ts : m.tensors)
      if (ts.stage == GradStage::kLayer) f(ts, l);
  for (const auto& ts : m.tensors)
    if (ts.stage == GradStage::kFinal) f(ts, -1);
  if (!m.tied)
    for (const auto& ts : m.tensors)
      if (ts.stage == GradStage::kHead) f(ts, -1);
}

}  // namespace

std::uint64_t GradModel::numel() const {
  std::uint64_t n = 0;
  for_each_logical(*this, [&](const GradTensor& ts, int) {
    n += prod(ts.shape, 0, ts.shape.size());
  });
  return n;
}

std::uint64_t RankSegments::counted() const {
  std::uint64_t n = 0;
  for (const auto& s : segments)
    if (s.weight != 0.0) n += s.numel;
  return n;
}

RankSegments gns_segments(const GradModel& model, const ParallelStrategy& s,
                          int rank) {
  if (s.d < 1 || s.t < 1 || s.p < 1)
    throw ValidationError("strategy degrees must be >= 1");
  if (rank < 0 || rank >= s.gpus())
    throw ValidationError("rank " + std::to_string(rank) + " outside [0, " +
                          std::to_string(s.gpus()) + ")");
  if (model.layers < 1 || model.layers % s.p)
    throw ValidationError(model.name + ": " + std::to_string(model.layers) +
                          " layers not divisible by p=" + std::to_string(s.p));
  for (const auto& ts : model.tensors) check_tensor(ts);
  if (model.tied) {
    bool has_embed = false;
    for (const auto& ts : model.tensors) has_embed |= ts.stage == GradStage::kEmbed;
    if (!has_embed) throw ValidationError(model.name + ": tied without an embedding");
  }
  RankSegments out;
  out.rank = rank;
  out.i_t = rank % s.t;
  out.i_d = (rank / s.t) % s.d;
  out.i_p = rank / (s.t * s.d);
  const int lo = out.i_p * model.layers / s.p;
  const int hi = (out.i_p + 1) * model.layers / s.p;

  // logical base offset of every (tensor, layer)
  struct Key { const GradTensor* ts; int layer; std::uint64_t base; };
  std::vector<Key> bases;
  std::uint64_t cursor = 0;
  for_each_logical(model, [&](const GradTensor& ts, int l) {
    bases.push_back({&ts, l, cursor});
    cursor += prod(ts.shape, 0, ts.shape.size());
  });
  auto base_of = [&](const GradTensor* ts, int l) {
    for (const auto& k : bases)
      if (k.ts == ts && k.layer == l) return k.base;
    throw InternalError("tensor without a logical base");
  };

  // (tensor, layer, weight) held locally, bucket order
  struct Local { const GradTensor* ts; int layer; double w; };
  std::vector<Local> local;
  if (out.i_p == 0)
    for (const auto& ts : model.tensors)
      if (ts.stage == GradStage::kEmbed) local.push_back({&ts, -1, 1.0});
  for (int l = lo; l < hi; ++l)
    for (const auto& ts : model.tensors)
      if (ts.stage == GradStage::kLayer) local.push_back({&ts, l, 1.0});
  if (out.i_p == s.p - 1) {
    for (const auto& ts : model.tensors)
      if (ts.stage == GradStage::kFinal) local.push_back({&ts, -1, 1.0});
    if (model.tied) {
      // the head is the (first) embedding: on a separate last stage it is a
      // copy whose gradient Megatron all-reduces with stage 0's -> weight 0;
      // with p == 1 it is the embedding already in the bucket
      if (s.p > 1)
        for (const auto& ts : model.tensors)
          if (ts.stage == GradStage::kEmbed) {
            local.push_back({&ts, -1, 0.0});
            break;
          }
    } else {
      for (const auto& ts : model.tensors)
        if (ts.stage == GradStage::kHead) local.push_back({&ts, -1, 1.0});
    }
  }

  std::uint64_t off = 0;
  for (const auto& lc : local) {
    const GradTensor& ts = *lc.ts;
    const std::uint64_t b = base_of(lc.ts, lc.layer);
    const std::uint64_t full = prod(ts.shape, 0, ts.shape.size());
    std::uint64_t n = full;
    double weight = lc.w;
    if (ts.tp_axis < 0) {
      out.gen.push_back({off, n, b, n, n});
      if (out.i_t != 0) weight = 0.0;  // replicated: counted on tp_rank 0
    } else {
      const std::size_t ax = (std::size_t)ts.tp_axis;
      if (ts.shape[ax] % s.t)
        throw ValidationError(ts.name + ": axis " + std::to_string(ax) +
                              " (" + std::to_string(ts.shape[ax]) +
                              ") not divisible by t=" + std::to_string(s.t));
      n = full / (std::uint64_t)s.t;
      const std::uint64_t inner = prod(ts.shape, ax + 1, ts.shape.size());
      const std::uint64_t piece = (std::uint64_t)ts.shape[ax] / s.t;
      const std::uint64_t outer = prod(ts.shape, 0, ax);
      const std::uint64_t start = b + (std::uint64_t)out.i_t * piece * inner;
      if (outer == 1)
        out.gen.push_back({off, n, start, n, n});
      else
        out.gen.push_back({off, n, start, piece * inner,
                           (std::uint64_t)ts.shape[ax] * inner});
    }
    out.segments.push_back(BucketSegment{off, n, weight});
    out.names.push_back(lc.layer >= 0 ? ts.name + "." + std::to_string(lc.layer)
                                      : ts.name);
    off += n;
  }
  out.bucket_numel = off;
  return out;
}

std::uint64_t gns_algorithmic_bytes(const GradModel& model,
                                    const ParallelStrategy& s, int micro_count,
                                    int elem_bytes, bool fused) {
  if (micro_count < 1 || elem_bytes < 1)
    throw ValidationError("micro_count and elem_bytes must be >= 1");
  std::uint64_t micro = 0, mean = 0;
  for (int r = 0; r < s.gpus(); ++r) {
    const RankSegments rs = gns_segments(model, s, r);
    micro += rs.counted();
    if (rs.i_d == 0) mean += rs.counted();
  }
  const std::uint64_t eb = (std::uint64_t)elem_bytes;
  return micro * (std::uint64_t)micro_count * eb +
         ((fused && s.d == 1) ? 0 : mean * eb);
}

GradModel llama_model(std::string name, std::int64_t vocab, std::int64_t h,
                      int layers, std::int64_t ffn, int heads, int kv_heads,
                      bool tied, bool qkv_bias) {
  const std::int64_t hd = h / heads;
  const std::int64_t qkv_rows = h + 2 * kv_heads * hd;
  GradModel m;
  m.name = std::move(name);
  m.layers = layers;
  m.tied = tied;
  using S = GradStage;
  m.tensors.push_back({"embed", {vocab, h}, 0, S::kEmbed});
  m.tensors.push_back({"input_norm", {h}, -1, S::kLayer});
  m.tensors.push_back({"qkv", {qkv_rows, h}, 0, S::kLayer});
  if (qkv_bias) m.tensors.push_back({"qkv_bias", {qkv_rows}, 0, S::kLayer});
  m.tensors.push_back({"o_proj", {h, h}, 1, S::kLayer});
  m.tensors.push_back({"post_norm", {h}, -1, S::kLayer});
  m.tensors.push_back({"gate_up", {2 * ffn, h}, 0, S::kLayer});
  m.tensors.push_back({"down", {h, ffn}, 1, S::kLayer});
  m.tensors.push_back({"final_norm", {h}, -1, S::kFinal});
  if (!tied) m.tensors.push_back({"lm_head", {vocab, h}, 0, S::kHead});
  return m;
}

GradModel gpt2_small() {
  const std::int64_t h = 768, ffn = 3072, vocab = 50304, pos = 1024;
  using S = GradStage;
  GradModel m;
  m.name = "gpt2-125m";
  m.layers = 12;
  m.tied = true;
  m.tensors = {
      {"wte", {vocab, h}, 0, S::kEmbed},    {"wpe", {pos, h}, -1, S::kEmbed},
      {"ln1_w", {h}, -1, S::kLayer},        {"ln1_b", {h}, -1, S::kLayer},
      {"qkv_w", {3 * h, h}, 0, S::kLayer},  {"qkv_b", {3 * h}, 0, S::kLayer},
      {"proj_w", {h, h}, 1, S::kLayer},     {"proj_b", {h}, -1, S::kLayer},
      {"ln2_w", {h}, -1, S::kLayer},        {"ln2_b", {h}, -1, S::kLayer},
      {"fc_w", {ffn, h}, 0, S::kLayer},     {"fc_b", {ffn}, 0, S::kLayer},
      {"fc2_w", {h, ffn}, 1, S::kLayer},    {"fc2_b", {h}, -1, S::kLayer},
      {"lnf_w", {h}, -1, S::kFinal},        {"lnf_b", {h}, -1, S::kFinal},
  };
  return m;
}

GradModel model_preset(std::string_view key) {
  if (key == "125m") return gpt2_small();
  if (key == "3b")
    return llama_model("llama3.2-3b", 128256, 3072, 28, 8192, 24, 8, true, false);
  if (key == "7b")
    return llama_model("llama2-7b", 32000, 4096, 32, 11008, 32, 32, false, false);
  if (key == "32b")
    return llama_model("qwen2.5-32b", 152064, 5120, 64, 27648, 40, 8, false, true);
  throw ValidationError("unknown model preset '" + std::string(key) +
                        "' (125m, 3b, 7b, 32b)");
}

}  // namespace coadapt

// ------------------------------------------------------------------ C-ABI

// shares coadapt_last_error() storage with cabi.cu
namespace coadapt_capi {
void set_error(const char* msg);
}

namespace {

coadapt::GradModel from_c(const coadapt_grad_model* m) {
  if (!m) throw coadapt::ValidationError("null model");
  if (m->n_tensors && !m->tensors) throw coadapt::ValidationError("null tensor array");
  coadapt::GradModel g;
  g.name = m->name ? m->name : "";
  g.layers = m->layers;
  g.tied = m->tied != 0;
  for (std::size_t i = 0; i < m->n_tensors; ++i) {
    const coadapt_grad_tensor& t = m->tensors[i];
    if (t.ndim < 1 || t.ndim > 4) throw coadapt::ValidationError("tensor ndim must be 1..4");
    if (t.stage < 0 || t.stage > 3) throw coadapt::ValidationError("tensor stage must be 0..3");
    coadapt::GradTensor ts;
    ts.name = t.name ? t.name : "";
    ts.shape.assign(t.shape, t.shape + t.ndim);
    ts.tp_axis = t.tp_axis;
    ts.stage = (coadapt::GradStage)t.stage;
    g.tensors.push_back(std::move(ts));
  }
  return g;
}

// presets handed out as C descriptors: storage lives for the process
struct CPreset {
  coadapt::GradModel model;
  std::vector<coadapt_grad_tensor> tensors;
};

const CPreset* preset(std::string_view key) {
  static const char* keys[] = {"125m", "3b", "7b", "32b"};
  static CPreset table[4];
  static bool init = [] {
    for (int k = 0; k < 4; ++k) {
      table[k].model = coadapt::model_preset(keys[k]);
      for (const auto& ts : table[k].model.tensors) {
        coadapt_grad_tensor c;
        std::memset(&c, 0, sizeof(c));
        c.name = ts.name.c_str();
        c.stage = (int32_t)ts.stage;
        c.ndim = (int32_t)ts.shape.size();
        c.tp_axis = ts.tp_axis;
        for (std::size_t a = 0; a < ts.shape.size(); ++a) c.shape[a] = ts.shape[a];
        table[k].tensors.push_back(c);
      }
    }
    return true;
  }();
  (void)init;
  for (int k = 0; k < 4; ++k)
    if (key == keys[k]) return &table[k];
  return nullptr;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return COADAPT_OK;
  } catch (const coadapt::ValidationError& e) {
    coadapt_capi::set_error(e.what());
    return COADAPT_E_VALIDATION;
  } catch (const std::exception& e) {
    coadapt_capi::set_error(e.what());
    return COADAPT_E_INTERNAL;
  }
}

}  // namespace

extern "C" {

int coadapt_model_preset(const char* key, coadapt_grad_model* out) {
  return guard([&] {
    if (!key || !out) throw coadapt::ValidationError("null argument");
    const CPreset* p = preset(key);
    if (!p) throw coadapt::ValidationError(std::string("unknown model preset '") + key + "'");
    out->name = p->model.name.c_str();
    out->layers = p->model.layers;
    out->tied = p->model.tied ? 1 : 0;
    out->tensors = p->tensors.data();
    out->n_tensors = p->tensors.size();
  });
}

int coadapt_gns_segments(const coadapt_grad_model* model, int d, int t, int p,
                         int rank, coadapt_segment* segs, coadapt_gen_segment* gen,
                         size_t cap, size_t* count, uint64_t* bucket_numel,
                         int32_t coords[3]) {
  return guard([&] {
    if (!count) throw coadapt::ValidationError("null count");
    const auto rs = coadapt::gns_segments(from_c(model), coadapt::ParallelStrategy{d, t, p}, rank);
    *count = rs.segments.size();
    if (bucket_numel) *bucket_numel = rs.bucket_numel;
    if (coords) {
      coords[0] = rs.i_d;
      coords[1] = rs.i_t;
      coords[2] = rs.i_p;
    }
    if (!segs && !gen) return;  // size query
    if (cap < rs.segments.size())
      throw coadapt::ValidationError("segment capacity " + std::to_string(cap) + " < " +
                                     std::to_string(rs.segments.size()));
    for (std::size_t i = 0; i < rs.segments.size(); ++i) {
      if (segs)
        segs[i] = coadapt_segment{rs.segments[i].offset, rs.segments[i].numel,
                                  rs.segments[i].weight};
      if (gen) {
        const auto& g = rs.gen[i];
        gen[i] = coadapt_gen_segment{g.local_off, g.numel, g.global_base, g.row_len,
                                     g.row_stride};
      }
    }
  });
}

int coadapt_gns_algorithmic_bytes(const coadapt_grad_model* model, int d, int t,
                                  int p, int micro_count, int elem_bytes, int fused,
                                  uint64_t* out) {
  return guard([&] {
    if (!out) throw coadapt::ValidationError("null out");
    *out = coadapt::gns_algorithmic_bytes(from_c(model), coadapt::ParallelStrategy{d, t, p},
                                          micro_count, elem_bytes, fused != 0);
  });
}

}  // extern "C"
