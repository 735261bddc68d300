// coadapt/segments.hpp — a rank's gradient-bucket segment table from a model
// description and a (d,t,p) strategy.
//
// The reference has no function for this: its estimator takes a
// caller-computed s_m (record_micro_batch, gns.hpp:19-20), and the paper
// says only that the squared norm is taken "over the local parameters"
// (PAPER.md:437-440).  What a rank's parameters are follows SPEC.md's
// layout rules (contiguous PP stages holding L/p layers,
// t equal contiguous TP pieces of a split tensor, DP replication) and its
// ModelSpec (tp_split_axis = none marks a tensor every TP
// rank holds whole).  The north star adds deduplication: every logical
// parameter is counted exactly once in the world sum of s_m, so
//   * a replicated tensor (norms, row-parallel biases) has weight 1 on
//     tp_rank 0 and weight 0 elsewhere;
//   * with a tied embedding on p > 1 stages, the last stage's head copy of
//     the embedding has weight 0 (Megatron all-reduces its gradient with
//     stage 0's);
// and weight-0 ranges are never loaded by the kernels.
//
// Bucket order (Megatron): embedding tensors on stage 0, then the stage's
// layers in order (each layer's tensors in declaration order), then the
// final tensors and the head on stage p-1.  Ranks are numbered tp fastest,
// then dp, then pp (rank = i_t + t * (i_d + d * i_p)), as in
// coadapt/reshard.hpp.
//
// gns_segments() is the C++ twin of paper_2604_26687_b200/layout.py's
// rank_layout(); tests/test_segments.py holds the two bit-identical over
// every BASELINE model and layout plus random strategies.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "coadapt/device.hpp"
#include "coadapt/strategy.hpp"

namespace coadapt {

enum class GradStage : int { kEmbed = 0, kLayer = 1, kFinal = 2, kHead = 3 };

struct GradTensor {
  std::string name;
  std::vector<std::int64_t> shape;  // 1..4 axes, row-major
  int tp_axis = -1;                 // axis split by TP, or -1 (replicated)
  GradStage stage = GradStage::kLayer;
};

struct GradModel {
  std::string name;
  int layers = 0;
  std::vector<GradTensor> tensors;  // any order across stages; order within
                                    // a stage is the bucket order
  bool tied = false;  // head = the first embedding tensor (no head tensors)

  std::uint64_t numel() const;  // unique logical parameters
};

// Bucket elements [local_off, local_off + numel) hold logical parameter
// indices global_base + (j / row_len) * row_stride + (j % row_len): the
// layout-independent index the synthetic generator hashes (coadapt_synth_fill).
struct GenSegment {
  std::uint64_t local_off = 0;
  std::uint64_t numel = 0;
  std::uint64_t global_base = 0;
  std::uint64_t row_len = 0;
  std::uint64_t row_stride = 0;
};

struct RankSegments {
  int rank = 0;
  int i_d = 0, i_t = 0, i_p = 0;
  std::uint64_t bucket_numel = 0;
  std::vector<BucketSegment> segments;  // one per local tensor, bucket order
  std::vector<GenSegment> gen;          // same order
  std::vector<std::string> names;       // "<tensor>[.<layer>]"

  std::uint64_t counted() const;  // elements with weight != 0
};

// ValidationError for an invalid strategy, rank outside [0, d*t*p),
// layers % p != 0, a split axis not divisible by t, or a malformed tensor.
RankSegments gns_segments(const GradModel& model, const ParallelStrategy& s,
                          int rank);

// Bytes one GNS step reads: every rank's counted shard once
// per micro-batch, plus one read of the synchronised mean gradient (each DP
// replica its 1/d slice) when d > 1; nothing extra for the fused d == 1 pass.
std::uint64_t gns_algorithmic_bytes(const GradModel& model,
                                    const ParallelStrategy& s, int micro_count,
                                    int elem_bytes, bool fused);

// Llama-style decoder (GQA, optional QKV bias), Megatron sharding:
// vocab-parallel embedding/head, column-parallel QKV and gate/up, row-
// parallel o/down, replicated norms.
GradModel llama_model(std::string name, std::int64_t vocab, std::int64_t hidden,
                      int layers, std::int64_t ffn, int heads, int kv_heads,
                      bool tied, bool qkv_bias);
GradModel gpt2_small();  // 125M, vocab padded to 50304, tied
// "125m" (GPT-2 small), "3b" (Llama-3.2-3B), "7b" (Llama-2-7B),
// "32b" (Qwen2.5-32B): the BASELINE.json shapes.
GradModel model_preset(std::string_view key);

}  // namespace coadapt
