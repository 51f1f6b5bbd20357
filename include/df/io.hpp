// df/io.hpp -- the data formats either side of the GPU-actor path (SURVEY
// §8 f2): what the reference's front end reads into its source actors and
// writes from its sinks (/root/reference/proj/src/bench.cpp:25-97 read_file /
// write_file / read_pgm, :173-262 load_motion_input / load_dpd_setup), plus
// the schedule and taps text formats of the reference's DPD API
// (proj/include/dynflow/dpd.hpp:112-120, proj/src/dpd.cpp:393-462), which
// live in df/dpd.hpp.  Host code: these feed df_*_run_host / dfh_*_run, whose
// staging pipelines move the bytes to HBM.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace df::io {

// The reference's ConfigError (bench.cpp:20-23): unreadable, truncated or
// malformed input files.
class FormatError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

std::vector<char> read_file(const std::string& path);                         // bench.cpp:25-30
void write_file(const std::string& path, const void* data, std::size_t size);  // bench.cpp:32-37

// Binary PGM (P5), possibly several images concatenated in one file
// (bench.cpp:43-97): '#' comments and whitespace between header tokens,
// maxval 255, every frame the same size.
struct PgmStream {
  unsigned width = 0;
  unsigned height = 0;
  std::vector<std::uint8_t> pixels;  // concatenated frames
  std::uint64_t frames = 0;
};
PgmStream read_pgm(const std::string& path);
// Writes `frames` concatenated P5 images (the inverse of read_pgm).
void write_pgm(const std::string& path, const std::uint8_t* pixels, std::uint64_t frames, unsigned width,
               unsigned height);

// Raw frames of width x height x fmt bytes (fmt 1 gray, 3 interleaved RGB --
// the RGB form is this build's extension of bench.cpp:184-196): the file
// must hold a whole, non-zero number of frames.
std::vector<std::uint8_t> read_raw_frames(const std::string& path, unsigned width, unsigned height, unsigned fmt,
                                          std::uint64_t* frames);

// Interleaved complex-f32 samples (re, im pairs; bench.cpp:244-253).
std::vector<std::complex<float>> read_cf32(const std::string& path);

}  // namespace df::io
