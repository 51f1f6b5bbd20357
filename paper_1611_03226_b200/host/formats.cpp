// formats.cpp -- input/output formats around the GPU-actor path (df/io.hpp)
// and the DPD schedule / taps text formats (df/dpd.hpp).  Behaviour and
// error messages follow the reference: proj/src/bench.cpp:25-97 and
// :173-262, proj/src/dpd.cpp:393-462.
#include <cctype>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>

#include "df/dpd.hpp"
#include "df/io.hpp"

namespace df::io {

std::vector<char> read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw FormatError("cannot open '" + path + "'");
  return std::vector<char>((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

void write_file(const std::string& path, const void* data, std::size_t size) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw FormatError("cannot open '" + path + "' for writing");
  out.write(static_cast<const char*>(data), static_cast<std::streamsize>(size));
  if (!out) throw FormatError("short write to '" + path + "'");
}

PgmStream read_pgm(const std::string& path) {
  const std::vector<char> data = read_file(path);
  std::size_t pos = 0;
  // Header token: skips whitespace and '#'-to-end-of-line comments.
  auto token = [&]() -> std::string {
    std::string tok;
    while (pos < data.size()) {
      const char c = data[pos];
      if (c == '#') {  // comment to end of line, the newline included (bench.cpp:57-60)
        while (pos < data.size() && data[pos] != '\n') ++pos;
        if (pos < data.size()) ++pos;
        continue;
      }
      if (std::isspace(static_cast<unsigned char>(c))) {
        ++pos;
        if (!tok.empty()) return tok;
        continue;
      }
      tok.push_back(c);
      ++pos;
    }
    if (tok.empty()) throw FormatError("truncated PGM header in '" + path + "'");
    return tok;
  };
  // std::stoul as the reference (leading digits; std::invalid_argument if none).
  auto number = [](const std::string& t) -> unsigned { return static_cast<unsigned>(std::stoul(t)); };
  PgmStream s;
  while (pos < data.size()) {
    if (token() != "P5") throw FormatError("'" + path + "' is not binary PGM (P5)");
    const unsigned w = number(token());
    const unsigned h = number(token());
    const unsigned maxval = number(token());
    if (maxval != 255) throw FormatError("PGM maxval must be 255 in '" + path + "'");
    if (s.frames == 0) {
      s.width = w;
      s.height = h;
    } else if (w != s.width || h != s.height) {
      throw FormatError("PGM frames in '" + path + "' change dimensions");
    }
    // The single whitespace byte after maxval was consumed by token().
    const std::size_t size = static_cast<std::size_t>(w) * h;
    if (data.size() - pos < size) throw FormatError("truncated PGM data in '" + path + "'");
    s.pixels.insert(s.pixels.end(), data.begin() + static_cast<std::ptrdiff_t>(pos),
                    data.begin() + static_cast<std::ptrdiff_t>(pos + size));
    pos += size;
    ++s.frames;
    while (pos < data.size() && std::isspace(static_cast<unsigned char>(data[pos]))) ++pos;
  }
  if (s.frames == 0) throw FormatError("'" + path + "' holds no PGM frames");
  return s;
}

void write_pgm(const std::string& path, const std::uint8_t* pixels, std::uint64_t frames, unsigned width,
               unsigned height) {
  if (frames == 0 || width == 0 || height == 0) throw FormatError("write_pgm: nothing to write");
  std::ofstream out(path, std::ios::binary);
  if (!out) throw FormatError("cannot open '" + path + "' for writing");
  const std::string header = "P5\n" + std::to_string(width) + " " + std::to_string(height) + "\n255\n";
  const std::size_t size = static_cast<std::size_t>(width) * height;
  for (std::uint64_t f = 0; f < frames; ++f) {
    out.write(header.data(), static_cast<std::streamsize>(header.size()));
    out.write(reinterpret_cast<const char*>(pixels + f * size), static_cast<std::streamsize>(size));
  }
  if (!out) throw FormatError("short write to '" + path + "'");
}

std::vector<std::uint8_t> read_raw_frames(const std::string& path, unsigned width, unsigned height, unsigned fmt,
                                          std::uint64_t* frames) {
  if (fmt != 1 && fmt != 3) throw FormatError("raw frames: format must be 1 (gray) or 3 (RGB)");
  const std::vector<char> raw = read_file(path);
  const std::size_t size = static_cast<std::size_t>(width) * height * fmt;
  if (size == 0 || raw.empty() || raw.size() % size != 0)
    throw FormatError("'" + path + "' is not a multiple of " + std::to_string(size) + "-byte frames");
  if (frames) *frames = raw.size() / size;
  std::vector<std::uint8_t> px(raw.size());
  std::memcpy(px.data(), raw.data(), raw.size());
  return px;
}

std::vector<std::complex<float>> read_cf32(const std::string& path) {
  const std::vector<char> raw = read_file(path);
  if (raw.empty() || raw.size() % (2 * sizeof(float)) != 0)
    throw FormatError("'" + path + "' is not interleaved float re,im pairs");
  std::vector<std::complex<float>> s(raw.size() / (2 * sizeof(float)));
  std::memcpy(s.data(), raw.data(), raw.size());
  return s;
}

}  // namespace df::io

namespace df::dpd {

std::vector<ConfigToken> parse_schedule(std::istream& in) {
  std::vector<ConfigToken> schedule;
  std::string line;
  std::size_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (const auto hash = line.find('#'); hash != std::string::npos) line.erase(hash);
    std::istringstream ls(line);
    int k = 0;
    if (!(ls >> k)) continue;  // blank line
    auto fail = [&](const std::string& why) {
      throw std::runtime_error("schedule line " + std::to_string(line_no) + ": " + why);
    };
    if (k < 2 || k > static_cast<int>(kBranchCount)) fail("active count " + std::to_string(k) + " outside [2,10]");
    ConfigToken token;
    char c = 0;
    if (ls >> c) {
      if (c != ':') fail("expected ':' after count");
      for (int i = 0; i < k; ++i) {
        int branch = 0;
        if (!(ls >> branch)) fail("expected " + std::to_string(k) + " branch indices");
        if (branch < 1 || branch > static_cast<int>(kBranchCount)) fail("branch index outside 1..10");
        if (token.active(static_cast<unsigned>(branch))) fail("branch " + std::to_string(branch) + " listed twice");
        token.active_mask = static_cast<std::uint16_t>(token.active_mask | (1u << (branch - 1)));
        if (i + 1 < k && !(ls >> c && c == ',')) fail("expected ',' between branch indices");
      }
    } else {
      token = ConfigToken::first_n(static_cast<unsigned>(k));
    }
    schedule.push_back(token);
  }
  if (schedule.empty()) throw std::runtime_error("schedule file has no entries");
  return schedule;
}

std::vector<std::complex<float>> parse_taps(std::istream& in, unsigned taps_per_branch) {
  if (taps_per_branch < 1 || taps_per_branch > kMaxHistory + 1)
    throw std::invalid_argument("taps per branch outside [1,32]");
  std::vector<std::complex<float>> taps(static_cast<std::size_t>(kBranchCount) * taps_per_branch);
  const std::string expect = std::to_string(taps_per_branch);
  std::string line;
  unsigned branch = 0;
  while (branch < kBranchCount && std::getline(in, line)) {
    if (const auto hash = line.find('#'); hash != std::string::npos) line.erase(hash);
    std::istringstream ls(line);
    std::string pair;
    unsigned tap = 0;
    while (ls >> pair) {
      if (tap >= taps_per_branch)
        throw std::runtime_error("taps line for branch " + std::to_string(branch + 1) + " has more than " + expect +
                                 " entries");
      float re = 0.0f, im = 0.0f;
      char comma = 0;
      std::istringstream ps(pair);
      if (!(ps >> re >> comma >> im) || comma != ',')
        throw std::runtime_error("malformed tap '" + pair + "' (expected re,im)");
      taps[static_cast<std::size_t>(branch) * taps_per_branch + tap++] = {re, im};
    }
    if (tap == 0) continue;  // blank line
    if (tap != taps_per_branch)
      throw std::runtime_error("branch " + std::to_string(branch + 1) + " has " + std::to_string(tap) +
                               " taps, expected " + expect);
    ++branch;
  }
  if (branch != kBranchCount)
    throw std::runtime_error("taps file defines " + std::to_string(branch) + " branches, expected 10");
  return taps;
}

}  // namespace df::dpd
