// host_model.cpp -- parameter validation/parsing, frame writers and the
// core-count query of the drop-in library.  Behaviour (accepted syntax,
// defaults, error kinds and message text) follows the reference's
// src/model.cpp:10-28, src/io.cpp:1-230 and src/sysinfo.cpp:1-38 so that
// callers observe the same contract through include/nasch/nasch.h.
#include "host_model.hpp"

#include <cctype>
#include <charconv>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <thread>
#include <utility>

namespace nb200 {

void SimParams::validate() const {
  if (road_length < 1) throw std::invalid_argument("road_length must be at least 1");
  if (car_count < 1 || car_count > road_length) {
    throw std::invalid_argument("car_count must be in [1, road_length] (got " +
                                std::to_string(car_count) + " cars on " +
                                std::to_string(road_length) + " cells)");
  }
  // Written so that NaN fails too.
  if (!(p >= 0.0 && p <= 1.0)) throw std::invalid_argument("p must be in [0, 1]");
  if (v_max < 1) throw std::invalid_argument("v_max must be at least 1");
  if (output_stride < 1) throw std::invalid_argument("output_stride must be at least 1");
}

ParamError::ParamError(int line, std::string key, const std::string& message)
    : std::runtime_error((line > 0 ? "line " + std::to_string(line) + ": " : std::string()) +
                         key + ": " + message),
      line_(line),
      key_(std::move(key)) {}

namespace {

std::string strip(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

uint64_t to_u64(int line, const std::string& key, const std::string& text) {
  uint64_t out = 0;
  const char* end = text.data() + text.size();
  const auto res = std::from_chars(text.data(), end, out);
  if (text.empty() || res.ec != std::errc() || res.ptr != end) {
    throw ParamError(line, key, "expected a non-negative integer, got '" + text + "'");
  }
  return out;
}

double to_double(int line, const std::string& key, const std::string& text) {
  double out = 0.0;
  const char* end = text.data() + text.size();
  const auto res = std::from_chars(text.data(), end, out);
  if (text.empty() || res.ec != std::errc() || res.ptr != end) {
    throw ParamError(line, key, "expected a number, got '" + text + "'");
  }
  return out;
}

OutputMode to_mode(int line, const std::string& text) {
  if (text == "none") return OutputMode::none;
  if (text == "ascii") return OutputMode::ascii;
  if (text == "pgm") return OutputMode::pgm;
  throw ParamError(line, "output", "expected none, ascii or pgm, got '" + text + "'");
}

}  // namespace

ParamFile parse_params(const std::string& text) {
  ParamFile out;
  std::map<std::string, int> first_line;
  std::istringstream in(text);
  std::string raw;
  int line_no = 0;
  while (std::getline(in, raw)) {
    ++line_no;
    const size_t comment = raw.find('#');
    const std::string line = strip(comment == std::string::npos ? raw : raw.substr(0, comment));
    if (line.empty()) continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos) throw ParamError(line_no, line, "expected 'key = value'");
    const std::string key = strip(line.substr(0, eq));
    const std::string value = strip(line.substr(eq + 1));
    if (key.empty()) throw ParamError(line_no, value, "missing key before '='");
    const auto ins = first_line.emplace(key, line_no);
    if (!ins.second) {
      throw ParamError(line_no, key, "duplicate key, first set on line " +
                                         std::to_string(ins.first->second));
    }
    SimParams& p = out.params;
    if (key == "length") {
      p.road_length = to_u64(line_no, key, value);
    } else if (key == "ncars") {
      p.car_count = to_u64(line_no, key, value);
    } else if (key == "vmax") {
      p.v_max = to_u64(line_no, key, value);
    } else if (key == "p") {
      p.p = to_double(line_no, key, value);
    } else if (key == "steps") {
      p.steps = to_u64(line_no, key, value);
    } else if (key == "seed") {
      p.seed = to_u64(line_no, key, value);
    } else if (key == "output") {
      p.output_mode = to_mode(line_no, value);
    } else if (key == "stride") {
      p.output_stride = to_u64(line_no, key, value);
    } else if (key == "threads") {
      const uint64_t t = to_u64(line_no, key, value);
      if (t < 1) throw ParamError(line_no, key, "threads must be at least 1");
      out.threads = static_cast<unsigned>(t);
    } else {
      throw ParamError(line_no, key, "unknown key");
    }
  }
  for (const char* required : {"length", "ncars", "steps", "seed"}) {
    if (!first_line.count(required)) throw ParamError(0, required, "required key missing");
  }
  try {
    out.params.validate();
  } catch (const std::invalid_argument& e) {
    throw ParamError(0, "params", e.what());
  }
  return out;
}

ParamFile load_params(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open parameter file '" + path + "'");
  std::ostringstream buf;
  buf << f.rdbuf();
  return parse_params(buf.str());
}

const char* output_mode_name(OutputMode mode) {
  switch (mode) {
    case OutputMode::ascii: return "ascii";
    case OutputMode::pgm: return "pgm";
    case OutputMode::none: break;
  }
  return "none";
}

std::string format_params(const SimParams& p, unsigned threads) {
  std::ostringstream o;
  o << "length = " << p.road_length << "\n"
    << "ncars = " << p.car_count << "\n"
    << "vmax = " << p.v_max << "\n"
    << "p = " << p.p << "\n"
    << "steps = " << p.steps << "\n"
    << "seed = " << p.seed << "\n"
    << "output = " << output_mode_name(p.output_mode) << "\n"
    << "stride = " << p.output_stride << "\n"
    << "threads = " << threads << "\n";
  return o.str();
}

// src/io.cpp:168-184: "<step> x:v x:v ...\n" per frame.
void write_ascii_file(const std::vector<Frame>& frames, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  std::string line;
  char num[48];
  for (const Frame& f : frames) {
    line.clear();
    auto r = std::to_chars(num, num + sizeof num, f.step);
    line.append(num, r.ptr);
    for (size_t i = 0; i < f.positions.size(); ++i) {
      line.push_back(' ');
      r = std::to_chars(num, num + sizeof num, f.positions[i]);
      line.append(num, r.ptr);
      line.push_back(':');
      r = std::to_chars(num, num + sizeof num, f.velocities[i]);
      line.append(num, r.ptr);
    }
    line.push_back('\n');
    out.write(line.data(), static_cast<std::streamsize>(line.size()));
  }
  if (!out) throw IoError("write failed");
}

// src/io.cpp:186-216: P5 raster, one row per frame, occupied cells 0,
// empty cells 255.
void write_pgm_file(const std::vector<Frame>& frames, uint64_t road_length,
                    const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  out << "P5\n" << road_length << ' ' << frames.size() << "\n255\n";
  std::vector<char> row(road_length);
  for (const Frame& f : frames) {
    if (f.raster.size() == road_length) {  // rasterised on the device
      out.write(reinterpret_cast<const char*>(f.raster.data()), static_cast<std::streamsize>(road_length));
      continue;
    }
    std::fill(row.begin(), row.end(), '\xff');
    for (uint64_t x : f.positions) row[x] = '\0';
    out.write(row.data(), static_cast<std::streamsize>(row.size()));
  }
  if (!out) throw IoError("write failed");
}

// Distinct (physical id, core id) pairs from /proc/cpuinfo, else the
// hardware concurrency (src/sysinfo.cpp:11-36).
unsigned physical_cores() {
  std::ifstream info("/proc/cpuinfo");
  std::set<std::pair<long, long>> seen;
  long phys = -1;
  std::string line;
  while (info && std::getline(info, line)) {
    if (line.empty()) {
      phys = -1;
      continue;
    }
    const size_t colon = line.find(':');
    if (colon == std::string::npos) continue;
    if (line.rfind("physical id", 0) == 0) {
      phys = std::stol(line.substr(colon + 1));
    } else if (line.rfind("core id", 0) == 0) {
      seen.emplace(phys, std::stol(line.substr(colon + 1)));
    }
  }
  if (!seen.empty()) return static_cast<unsigned>(seen.size());
  return std::thread::hardware_concurrency();
}

}  // namespace nb200
