// reshard.cpp — shard layouts and transfer plans (§8 f4).
// Planning is a pure host function over a few hundred shards; the bytes move
// on the device (reshard.cu).
#include "coadapt/reshard.hpp"

#include <algorithm>
#include <map>
#include <tuple>

#include "coadapt/errors.hpp"
#include "coadapt/io.hpp"

namespace coadapt::reshard {
namespace {

constexpr std::uint64_t kPackAlign = 64;  // elements: 128 B for bf16

struct Coords {
  int d, t, p;
};

Coords coords_of(int rank, const ParallelStrategy& s) {
  return Coords{(rank / s.t) % s.d, rank % s.t, rank / (s.t * s.d)};
}

std::uint64_t box_numel(const std::vector<std::int64_t>& ext) {
  std::uint64_t n = 1;
  for (auto e : ext) n *= (std::uint64_t)e;
  return n;
}

// per-axis interval intersection; false when empty
bool intersect(const ShardDescriptor& a, const ShardDescriptor& b,
               std::vector<std::int64_t>& off, std::vector<std::int64_t>& ext) {
  const std::size_t nd = a.global_shape.size();
  off.assign(nd, 0);
  ext.assign(nd, 0);
  for (std::size_t i = 0; i < nd; ++i) {
    const auto lo = std::max(a.global_offset[i], b.global_offset[i]);
    const auto hi = std::min(a.global_offset[i] + a.local_shape[i],
                             b.global_offset[i] + b.local_shape[i]);
    if (hi <= lo) return false;
    off[i] = lo;
    ext[i] = hi - lo;
  }
  return true;
}

bool contains(const ShardDescriptor& s, const std::vector<std::int64_t>& off,
              const std::vector<std::int64_t>& ext) {
  for (std::size_t i = 0; i < off.size(); ++i)
    if (off[i] < s.global_offset[i] ||
        off[i] + ext[i] > s.global_offset[i] + s.local_shape[i])
      return false;
  return true;
}

void check_model(const ModelSpec& m) {
  if (m.layers < 1) throw ValidationError("reshard: layers must be >= 1");
  if (m.per_layer.empty())
    throw ValidationError("reshard: model declares no tensors");
  if (m.optimizer_state_multiplier < 0 || m.param_bytes < 1 ||
      m.state_bytes < 1)
    throw ValidationError("reshard: bad element sizes");
  for (const auto& t : m.per_layer) {
    if (t.shape.empty() || t.shape.size() > (std::size_t)kMaxDims)
      throw ValidationError("reshard: tensor " + t.name + " must have 1.." +
                            std::to_string(kMaxDims) + " axes");
    for (auto e : t.shape)
      if (e < 1)
        throw ValidationError("reshard: tensor " + t.name +
                              " has a non-positive extent");
    if (t.tp_axis < -1 || t.tp_axis >= (int)t.shape.size())
      throw ValidationError("reshard: tensor " + t.name + " tp_axis out of range");
  }
}

}  // namespace

std::string ModelSpec::key(int layer, int tensor) const {
  return "layer" + std::to_string(layer) + "." + per_layer.at(tensor).name;
}

std::uint64_t ShardDescriptor::numel() const { return box_numel(local_shape); }

std::uint64_t ShardLayout::max_pack_numel() const {
  std::uint64_t m = 0;
  for (auto n : pack_numel) m = std::max(m, n);
  return m;
}

ShardLayout layout_for(const ModelSpec& model, const ParallelStrategy& s,
                       int n_gpus) {
  validate_strategy(s, n_gpus);
  check_model(model);
  if (model.layers % s.p)
    throw ValidationError("reshard: " + std::to_string(model.layers) +
                          " layers not divisible by p=" + std::to_string(s.p));
  for (const auto& t : model.per_layer)
    if (t.tp_axis >= 0 && t.shape[t.tp_axis] % s.t)
      throw ValidationError("reshard: tensor " + t.name + " axis " +
                            std::to_string(t.tp_axis) + " (" +
                            std::to_string(t.shape[t.tp_axis]) +
                            ") not divisible by t=" + std::to_string(s.t));
  ShardLayout L;
  L.strategy = s;
  L.replica_groups.assign(s.d, {});
  L.pack_numel.assign(n_gpus, 0);
  const int per_stage = model.layers / s.p;
  for (int r = 0; r < n_gpus; ++r) {
    const Coords c = coords_of(r, s);
    L.replica_groups[c.d].push_back(r);
    std::uint64_t cursor = 0;
    for (int l = c.p * per_stage; l < (c.p + 1) * per_stage; ++l) {
      for (int ti = 0; ti < (int)model.per_layer.size(); ++ti) {
        const auto& td = model.per_layer[ti];
        ShardDescriptor sd;
        sd.layer = l;
        sd.tensor = ti;
        sd.global_shape = td.shape;
        sd.global_offset.assign(td.shape.size(), 0);
        sd.local_shape = td.shape;
        if (td.tp_axis >= 0) {
          sd.local_shape[td.tp_axis] = td.shape[td.tp_axis] / s.t;
          sd.global_offset[td.tp_axis] = c.t * sd.local_shape[td.tp_axis];
        }
        sd.owner = r;
        sd.canonical = c.d == 0 && (td.tp_axis >= 0 || c.t == 0);
        sd.pack_offset = cursor;
        cursor += (sd.numel() + kPackAlign - 1) / kPackAlign * kPackAlign;
        L.shards.push_back(std::move(sd));
      }
    }
    L.pack_numel[r] = cursor;
  }
  return L;
}

TransferPlan plan_transfers(const ModelSpec& model, const ShardLayout& src,
                            const ShardLayout& dst, SourcePolicy policy) {
  check_model(model);
  const auto& ss = src.strategy;
  // the same model must underlie both layouts
  for (const auto* lay : {&src, &dst}) {
    if ((std::uint64_t)lay->shards.size() !=
        (std::uint64_t)lay->strategy.gpus() * model.layers *
            model.per_layer.size() / lay->strategy.p)
      throw ValidationError("reshard: layout does not match the model");
    for (const auto& sd : lay->shards)
      if (sd.layer < 0 || sd.layer >= model.layers || sd.tensor < 0 ||
          sd.tensor >= (int)model.per_layer.size() ||
          sd.global_shape != model.per_layer[sd.tensor].shape)
        throw ValidationError("reshard: layout does not match the model");
  }
  // source copies per (replica, layer, tensor) that tile the tensor, and
  // every source shard per (rank, layer, tensor)
  std::map<std::tuple<int, int, int>, std::vector<std::size_t>> tiling, on_rank;
  for (std::size_t i = 0; i < src.shards.size(); ++i) {
    const auto& sd = src.shards[i];
    const Coords c = coords_of(sd.owner, ss);
    const bool split = model.per_layer[sd.tensor].tp_axis >= 0;
    if (split || c.t == 0) tiling[{c.d, sd.layer, sd.tensor}].push_back(i);
    on_rank[{sd.owner, sd.layer, sd.tensor}].push_back(i);
  }
  const std::uint64_t bpe = (std::uint64_t)model.bytes_per_element();
  TransferPlan plan;
  std::vector<std::uint64_t> received(dst.strategy.gpus(), 0);
  std::vector<std::int64_t> off, ext;
  for (std::size_t di = 0; di < dst.shards.size(); ++di) {
    const auto& D = dst.shards[di];
    const Coords dc = coords_of(D.owner, dst.strategy);
    const int replica = policy == SourcePolicy::kSpread ? dc.d % ss.d : 0;
    const auto tile = tiling.find({replica, D.layer, D.tensor});
    const auto mine = on_rank.find({D.owner, D.layer, D.tensor});
    std::uint64_t covered = 0;
    if (tile != tiling.end()) {
      for (std::size_t si : tile->second) {
        if (!intersect(D, src.shards[si], off, ext)) continue;
        Move mv;
        mv.src_shard = si;
        if (mine != on_rank.end())
          for (std::size_t li : mine->second)
            if (contains(src.shards[li], off, ext)) {
              mv.src_shard = li;
              break;
            }
        mv.src_rank = src.shards[mv.src_shard].owner;
        mv.dst_rank = D.owner;
        mv.layer = D.layer;
        mv.tensor = D.tensor;
        mv.dst_shard = di;
        mv.local = mv.src_rank == mv.dst_rank;
        const std::uint64_t n = box_numel(ext);
        mv.bytes = n * bpe;
        mv.offset = off;
        mv.extent = ext;
        covered += n;
        if (mv.local) {
          plan.local_bytes += mv.bytes;
        } else {
          plan.total_bytes += mv.bytes;
          received[mv.dst_rank] += mv.bytes;
        }
        plan.moves.push_back(std::move(mv));
      }
    }
    if (covered != D.numel())
      throw InternalError("reshard: destination shard " +
                          model.key(D.layer, D.tensor) + " on rank " +
                          std::to_string(D.owner) + " covered " +
                          std::to_string(covered) + " of " +
                          std::to_string(D.numel()) + " elements");
  }
  for (auto r : received)
    plan.max_bytes_per_rank = std::max(plan.max_bytes_per_rank, r);
  return plan;
}

double estimate_reconfig_latency(const TransferPlan& plan,
                                 double bandwidth_bytes_per_s,
                                 double fixed_overhead_s) {
  if (!(bandwidth_bytes_per_s > 0.0))
    throw ValidationError("reshard: bandwidth must be > 0");
  return fixed_overhead_s + (double)plan.total_bytes / bandwidth_bytes_per_s;
}

std::string transfer_plan_csv(const ModelSpec& model, const TransferPlan& plan) {
  std::string out = "key,src_rank,dst_rank,offsets,extents,bytes,local\n";
  auto axes = [](const std::vector<std::int64_t>& v) {
    std::string s;
    for (std::size_t i = 0; i < v.size(); ++i) {
      if (i) s += ';';
      s += format_int(v[i]);
    }
    return s;
  };
  for (const auto& m : plan.moves)
    out += model.key(m.layer, m.tensor) + ',' + format_int(m.src_rank) + ',' +
           format_int(m.dst_rank) + ',' + axes(m.offset) + ',' +
           axes(m.extent) + ',' + format_int((std::int64_t)m.bytes) + ',' +
           (m.local ? "1" : "0") + '\n';
  return out;
}

}  // namespace coadapt::reshard
