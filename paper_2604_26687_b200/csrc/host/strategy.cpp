// strategy.cpp — implements coadapt/strategy.hpp (reference
// strategy.hpp:12-46).
#include "coadapt/strategy.hpp"

#include <charconv>
#include <string_view>

#include "coadapt/errors.hpp"

namespace coadapt {

std::string ParallelStrategy::label() const {
  return "d" + std::to_string(d) + "t" + std::to_string(t) + "p" +
         std::to_string(p);
}

bool ConfigTuple::divisible() const {
  const std::int64_t unit = (std::int64_t)strategy.d * micro_batch;
  return strategy.d >= 1 && micro_batch >= 1 && global_batch >= 1 &&
         global_batch % unit == 0;
}

std::int64_t ConfigTuple::grad_accum() const {
  if (!divisible())
    throw ValidationError("config " + label() +
                          ": global_batch not divisible by d * micro_batch");
  return global_batch / ((std::int64_t)strategy.d * micro_batch);
}

std::string ConfigTuple::label() const {
  return strategy.label() + "_g" + std::to_string(global_batch) + "_m" +
         std::to_string(micro_batch);
}

void validate_strategy(const ParallelStrategy& s, int n_gpus) {
  if (s.d < 1 || s.t < 1 || s.p < 1)
    throw ValidationError("strategy " + s.label() + ": degrees must be >= 1");
  if ((long long)s.d * s.t * s.p != n_gpus)
    throw ValidationError("strategy " + s.label() + ": d*t*p != " +
                          std::to_string(n_gpus) + " GPUs");
}

void validate_config(const ConfigTuple& c, int n_gpus) {
  validate_strategy(c.strategy, n_gpus);
  if (c.global_batch < 1 || c.micro_batch < 1)
    throw ValidationError("config " + c.label() + ": batches must be >= 1");
  if (!c.divisible())
    throw ValidationError("config " + c.label() + ": global_batch " +
                          std::to_string(c.global_batch) +
                          " not divisible by d*micro_batch");
}

namespace {
int parse_degree(std::string_view s, const std::string& text) {
  int v = 0;
  auto r = std::from_chars(s.data(), s.data() + s.size(), v);
  if (s.empty() || r.ec != std::errc() || r.ptr != s.data() + s.size() || v < 1)
    throw ValidationError("bad strategy label '" + text + "'");
  return v;
}
}  // namespace

ParallelStrategy parse_strategy_label(const std::string& text) {
  std::string_view s(text);
  ParallelStrategy out;
  if (!s.empty() && s.front() == 'd') {  // "d2t1p4"
    const auto tp = s.find('t'), pp = s.find('p');
    if (tp == std::string_view::npos || pp == std::string_view::npos || pp < tp)
      throw ValidationError("bad strategy label '" + text + "'");
    out.d = parse_degree(s.substr(1, tp - 1), text);
    out.t = parse_degree(s.substr(tp + 1, pp - tp - 1), text);
    out.p = parse_degree(s.substr(pp + 1), text);
    return out;
  }
  const auto c1 = s.find(','), c2 = s.find(',', c1 == s.npos ? c1 : c1 + 1);
  if (c1 == std::string_view::npos || c2 == std::string_view::npos)
    throw ValidationError("bad strategy label '" + text + "'");
  out.d = parse_degree(s.substr(0, c1), text);
  out.t = parse_degree(s.substr(c1 + 1, c2 - c1 - 1), text);
  out.p = parse_degree(s.substr(c2 + 1), text);
  return out;
}

}  // namespace coadapt
