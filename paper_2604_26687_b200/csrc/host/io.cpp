// io.cpp — implements coadapt/io.hpp (reference io.hpp:13-25).
#include "coadapt/io.hpp"

#include <charconv>
#include <cmath>
#include <fstream>
#include <sstream>
#include <system_error>

#include "coadapt/errors.hpp"

namespace coadapt {

std::string format_double(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);  // shortest round trip
  if (r.ec != std::errc()) throw InternalError("format_double: to_chars failed");
  return std::string(buf, r.ptr);
}

std::string format_int(std::int64_t v) {
  char buf[32];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, r.ptr);
}

double parse_double(std::string_view tok, const std::string& where) {
  if (tok.empty()) throw ParseError(where + ": empty number");
  if (tok == "nan") return std::nan("");
  if (tok == "inf") return INFINITY;
  if (tok == "-inf") return -INFINITY;
  double v = 0.0;
  auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (r.ec != std::errc() || r.ptr != tok.data() + tok.size())
    throw ParseError(where + ": not a number: '" + std::string(tok) + "'");
  return v;
}

std::int64_t parse_int(std::string_view tok, const std::string& where) {
  if (tok.empty()) throw ParseError(where + ": empty integer");
  std::int64_t v = 0;
  auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (r.ec != std::errc() || r.ptr != tok.data() + tok.size())
    throw ParseError(where + ": not an integer: '" + std::string(tok) + "'");
  return v;
}

std::vector<std::string_view> split_csv_line(std::string_view line) {
  if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
  std::vector<std::string_view> out;
  std::size_t start = 0;
  while (true) {
    const std::size_t comma = line.find(',', start);
    if (comma == std::string_view::npos) {
      out.push_back(line.substr(start));
      break;
    }
    out.push_back(line.substr(start, comma - start));
    start = comma + 1;
  }
  return out;
}

std::string read_text_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw ParseError("cannot open '" + path + "' for reading");
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void write_text_file(const std::string& path, const std::string& content) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw ParseError("cannot open '" + path + "' for writing");
  f << content;
  if (!f) throw ParseError("write to '" + path + "' failed");
}

}  // namespace coadapt
