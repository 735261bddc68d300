// formats.cpp — profile CSV and decision audit log (SPEC.md:64-72, 129-130,
// 404-405).  Every number goes through format_double /
// parse_double (io.hpp:10-19), so save -> load round trips are bit-exact.
#include <cmath>
#include <string>

#include "coadapt/errors.hpp"
#include "coadapt/io.hpp"
#include "coadapt/orchestrator.hpp"

namespace coadapt {
namespace {
constexpr const char* kProfileHeader =
    "d,t,p,global_batch,micro_batch,samples_per_sec,peak_mem_bytes,feasible";
constexpr const char* kAuditHeader =
    "step,time_s,phi,current_cfg,winner_cfg,current_score,winner_score,"
    "penalized,command";
}  // namespace

std::string profile_csv(const ThroughputProfile& prof) {
  std::string out = std::string(kProfileHeader) + "\n";
  for (const auto& [c, e] : prof.entries) {  // map order: deterministic
    out += format_int(c.strategy.d) + ',' + format_int(c.strategy.t) + ',' +
           format_int(c.strategy.p) + ',' + format_int(c.global_batch) + ',' +
           format_int(c.micro_batch) + ',' +
           format_double(e.samples_per_second) + ',' +
           format_double(e.peak_memory) + ',' + (e.feasible ? "1" : "0") + '\n';
  }
  return out;
}

ThroughputProfile parse_profile_csv(std::string_view text,
                                    const std::string& where) {
  ThroughputProfile prof;
  prof.hardware_id = where;
  std::size_t pos = 0, line_no = 0;
  bool header = true;
  while (pos <= text.size()) {
    std::size_t nl = text.find('\n', pos);
    if (nl == std::string_view::npos) nl = text.size();
    std::string_view line = text.substr(pos, nl - pos);
    pos = nl + 1;
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
    if (line.empty()) {
      if (pos > text.size()) break;
      continue;
    }
    const std::string loc = where + " line " + std::to_string(line_no);
    if (header) {
      if (line != kProfileHeader)
        throw ParseError(loc + ": expected header '" + kProfileHeader + "'");
      header = false;
      continue;
    }
    const auto f = split_csv_line(line);
    if (f.size() != 8)
      throw ParseError(loc + ": expected 8 fields, got " + std::to_string(f.size()));
    ConfigTuple c;
    c.strategy.d = (int)parse_int(f[0], loc);
    c.strategy.t = (int)parse_int(f[1], loc);
    c.strategy.p = (int)parse_int(f[2], loc);
    c.global_batch = parse_int(f[3], loc);
    c.micro_batch = parse_int(f[4], loc);
    ThroughputEntry e;
    e.samples_per_second = parse_double(f[5], loc);
    e.peak_memory = parse_double(f[6], loc);
    const std::int64_t feas = parse_int(f[7], loc);
    if (feas != 0 && feas != 1) throw ParseError(loc + ": feasible must be 0 or 1");
    e.feasible = feas == 1;
    const int gpus = c.strategy.gpus();
    if (prof.n_gpus == 0) prof.n_gpus = gpus;
    try {
      validate_config(c, prof.n_gpus);
    } catch (const ValidationError& ex) {
      throw ValidationError(loc + ": " + ex.what());
    }
    if (e.feasible && !(e.samples_per_second > 0.0))
      throw ValidationError(loc + ": feasible entry needs samples_per_sec > 0");
    if (!prof.entries.emplace(c, e).second)
      throw ValidationError(loc + ": duplicate key " + c.label());
  }
  if (header) throw ParseError(where + ": empty profile (no header)");
  return prof;
}

ThroughputProfile load_profile(const std::string& path) {
  return parse_profile_csv(read_text_file(path), path);
}

void save_profile(const std::string& path, const ThroughputProfile& profile) {
  write_text_file(path, profile_csv(profile));
}

const char* command_name(CommandKind kind) {
  switch (kind) {
    case CommandKind::kNoOp: return "NoOp";
    case CommandKind::kScaleBS: return "ScaleBS";
    case CommandKind::kReconfigure: return "Reconfigure";
  }
  throw InternalError("unknown CommandKind");
}

std::string decision_audit_csv(std::span<const DecisionRecord> rows) {
  std::string out = std::string(kAuditHeader) + "\n";
  for (const auto& r : rows) {
    out += format_int(r.step) + ',' + format_double(r.time_s) + ',' +
           format_double(r.phi ? *r.phi : std::nan("")) + ',' + r.current.label() +
           ',' + r.command.winner.label() + ',' +
           format_double(r.command.current_score) + ',' +
           format_double(r.command.winner_score) + ',' +
           (r.command.penalized ? "1" : "0") + ',' + command_name(r.command.kind) +
           '\n';
  }
  return out;
}

}  // namespace coadapt
