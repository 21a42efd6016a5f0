// host_model.hpp -- host-side model types of the drop-in library.
//
// Mirrors the reference's physics parameter set and its host plumbing
// (src/model.hpp:14-28, src/io.hpp:14-78, src/engine.hpp:66-70) so the
// C ABI (include/nasch/nasch.h) behaves identically; the hot path itself
// lives in engine.cu.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace nb200 {

enum class OutputMode { none, ascii, pgm };

// src/model.hpp:16-28 -- physics only; the worker count lives outside.
struct SimParams {
  uint64_t road_length = 0;
  uint64_t car_count = 0;
  uint64_t v_max = 5;
  double p = 0.13;
  uint64_t steps = 0;
  uint64_t seed = 0;
  OutputMode output_mode = OutputMode::none;
  uint64_t output_stride = 1;

  // Throws std::invalid_argument naming the violated constraint
  // (src/model.cpp:10-28).
  void validate() const;
};

// src/io.hpp:16-30
class ParamError : public std::runtime_error {
 public:
  ParamError(int line, std::string key, const std::string& message);
  int line() const { return line_; }
  const std::string& key() const { return key_; }

 private:
  int line_;
  std::string key_;
};

class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct ParamFile {
  SimParams params;
  unsigned threads = 1;
};

ParamFile parse_params(const std::string& text);      // src/io.cpp:68-142
ParamFile load_params(const std::string& path);       // src/io.cpp:144-152
std::string format_params(const SimParams& params, unsigned threads);
const char* output_mode_name(OutputMode mode);

// A recorded snapshot in rank (increasing position) order
// (src/engine.hpp:66-70).
struct Frame {
  uint64_t step = 0;
  std::vector<uint64_t> positions;
  std::vector<uint64_t> velocities;
  // output = pgm on the single-GPU engine: the frame's space-time row as
  // the P5 writer emits it (0 occupied, 255 empty), rasterised on the device
  // (positions / velocities are then not kept: only the ascii writer reads them)
  std::vector<uint8_t> raster;
};

void write_ascii_file(const std::vector<Frame>& frames, const std::string& path);
void write_pgm_file(const std::vector<Frame>& frames, uint64_t road_length,
                    const std::string& path);

unsigned physical_cores();

// FNV-1a 64 over one row (positions then velocities, each value as 8
// little-endian bytes; src/engine.hpp:15-36, src/engine.cpp:11-21).
constexpr uint64_t kFnvBasis = 14695981039346656037ull;
constexpr uint64_t kFnvPrime = 1099511628211ull;

}  // namespace nb200
