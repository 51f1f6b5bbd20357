// generators.cpp -- the reference's synthetic input generators as library
// API (proj/include/dynflow/dpd.hpp:122-124, motion.hpp:77), so a caller of
// the reference's bench paths finds them here too.  Every stream is defined
// by std::mt19937_64 (a standard engine, identical across implementations)
// and the reference's mappings: a float in [-1, 1) from the top 24 bits of
// one draw (dpd.cpp:21-26), taps scaled by 0.5, schedules of 2..10 branches
// from a partial Fisher-Yates shuffle of 1..10 (dpd.cpp:467-483), frame
// bytes as the low byte of one draw (motion.cpp:254-260).
#include <array>
#include <complex>
#include <cstdint>
#include <random>
#include <vector>

#include "df/dpd.hpp"
#include "df/motion.hpp"

namespace df::dpd {
namespace {
float pm1(std::mt19937_64& g) {
  const float u = static_cast<float>(g() >> 40) * (1.0f / 16777216.0f);  // top 24 bits -> [0, 1)
  return 2.0f * u - 1.0f;
}
}  // namespace

std::vector<ConfigToken> random_schedule(std::size_t entries, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  std::array<unsigned, kBranchCount> order{};
  for (unsigned i = 0; i < kBranchCount; ++i) order[i] = i + 1;
  std::vector<ConfigToken> out(entries);
  for (ConfigToken& t : out) {
    const unsigned k = 2u + static_cast<unsigned>(g() % (kBranchCount - 1));  // 2..10 active
    for (std::size_t n = kBranchCount; n > 1; --n) std::swap(order[n - 1], order[g() % n]);
    for (unsigned j = 0; j < k; ++j) t.active_mask = static_cast<std::uint16_t>(t.active_mask | (1u << (order[j] - 1)));
  }
  return out;
}

std::vector<std::complex<float>> random_taps(std::uint64_t seed, unsigned taps_per_branch) {
  std::mt19937_64 g(seed);
  std::vector<std::complex<float>> taps(static_cast<std::size_t>(kBranchCount) * taps_per_branch);
  for (auto& t : taps) {
    const float re = 0.5f * pm1(g);
    t = {re, 0.5f * pm1(g)};
  }
  return taps;
}

std::vector<std::complex<float>> synth_samples(std::uint64_t samples, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  std::vector<std::complex<float>> out(samples);
  for (auto& s : out) {
    const float re = pm1(g);
    s = {re, pm1(g)};
  }
  return out;
}

}  // namespace df::dpd

namespace df::motion {

std::vector<std::uint8_t> synth_frames(std::uint64_t frames, unsigned width, unsigned height, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  std::vector<std::uint8_t> out(frames * static_cast<std::size_t>(width) * height);
  for (auto& px : out) px = static_cast<std::uint8_t>(g() & 0xFFu);
  return out;
}

}  // namespace df::motion
