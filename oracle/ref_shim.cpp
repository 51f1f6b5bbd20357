// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// (dynflow, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libdynflow_ref.so).  TEST INFRASTRUCTURE ONLY: used to pin
// oracle/oracle.c, to generate tests/golden fixtures, and as the timed
// "reference" CPU arm of bench.py.  Nothing here is reference source; it
// only calls the reference's public API (proj/include/dynflow/*.hpp).
#include <algorithm>
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "dynflow/bench.hpp"
#include "dynflow/channel.hpp"
#include "dynflow/dpd.hpp"
#include "dynflow/motion.hpp"
#include "dynflow/runtime.hpp"

using namespace dynflow;

namespace {
thread_local std::string g_err;

dpd::TapSet taps_from(const float* t) {
  dpd::TapSet taps{};
  for (unsigned b = 0; b < dpd::kBranchCount; ++b)
    for (unsigned k = 0; k < dpd::kTapCount; ++k)
      taps[b][k] = {t[2 * (b * dpd::kTapCount + k)], t[2 * (b * dpd::kTapCount + k) + 1]};
  return taps;
}
std::vector<dpd::ConfigToken> sched_from(const uint16_t* s, size_t n) {
  std::vector<dpd::ConfigToken> v(n);
  for (size_t i = 0; i < n; ++i) v[i].active_mask = s[i];
  return v;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

void ref_synth_samples(uint64_t n, uint64_t seed, float* out) {
  auto v = dpd::synth_samples(n, seed);
  std::memcpy(out, v.data(), n * sizeof(std::complex<float>));
}
void ref_random_taps(uint64_t seed, float* out) {
  auto t = dpd::random_taps(seed);
  for (unsigned b = 0; b < 10; ++b)
    for (unsigned k = 0; k < 10; ++k) {
      out[2 * (b * 10 + k)] = t[b][k].real();
      out[2 * (b * 10 + k) + 1] = t[b][k].imag();
    }
}
void ref_random_schedule(size_t entries, uint64_t seed, uint16_t* out) {
  auto s = dpd::random_schedule(entries, seed);
  for (size_t i = 0; i < entries; ++i) out[i] = s[i].active_mask;
}
void ref_synth_frames(uint64_t frames, unsigned w, unsigned h, uint64_t seed, uint8_t* out) {
  auto v = motion::synth_frames(frames, w, h, seed);
  std::memcpy(out, v.data(), v.size());
}

int ref_check_config(uint16_t mask) {
  try {
    dpd::check_config({mask});
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The reference's own text parsers (dpd.cpp:393-462), for parity of
// df::dpd::parse_schedule / parse_taps.  Returns the entry count, or -1.
long ref_parse_schedule(const char* text, uint16_t* out, size_t cap) {
  try {
    std::istringstream in(text);
    auto s = dpd::parse_schedule(in);
    for (size_t i = 0; i < s.size() && i < cap; ++i) out[i] = s[i].active_mask;
    return (long)s.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
int ref_parse_taps(const char* text, float* out) {
  try {
    std::istringstream in(text);
    auto t = dpd::parse_taps(in);
    for (size_t b = 0; b < t.size(); ++b)
      for (size_t k = 0; k < t[b].size(); ++k) {
        out[2 * (b * t[b].size() + k)] = t[b][k].real();
        out[2 * (b * t[b].size() + k) + 1] = t[b][k].imag();
      }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_poly_branch(unsigned b, const float* re, const float* im, size_t n, float* ore,
                     float* oim) {
  dpd::poly_branch(b, {re, n}, {im, n}, {ore, n}, {oim, n});
}
// state: 9 re then 9 im (FirState layout), updated in place.
void ref_fir10(const float* taps10, float* state, const float* re, const float* im, size_t n,
               float* ore, float* oim) {
  dpd::BranchTaps t{};
  for (unsigned k = 0; k < 10; ++k) t[k] = {taps10[2 * k], taps10[2 * k + 1]};
  dpd::FirState st;
  for (unsigned j = 0; j < 9; ++j) { st.re[j] = state[j]; st.im[j] = state[9 + j]; }
  dpd::fir10(t, st, {re, n}, {im, n}, {ore, n}, {oim, n});
  for (unsigned j = 0; j < 9; ++j) { state[j] = st.re[j]; state[9 + j] = st.im[j]; }
}

int ref_oracle_dpd(const float* in, size_t samples, const float* taps, const uint16_t* sched,
                   size_t sched_len, uint32_t period, float* out) {
  try {
    std::span<const std::complex<float>> input(reinterpret_cast<const std::complex<float>*>(in),
                                               samples);
    auto o = dpd::oracle_dpd(input, taps_from(taps), sched_from(sched, sched_len), period);
    std::memcpy(out, o.data(), samples * sizeof(std::complex<float>));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The reference's own thread-per-actor network (proj/src/dpd.cpp:151-356 run
// through proj/src/runtime.cpp:322-332), timed as cmd_dpd does it:
// samples / active_seconds("sink") (proj/src/bench.cpp:391-397).
int ref_dpd_network(const float* in, size_t samples, const float* taps, const uint16_t* sched,
                    size_t sched_len, uint32_t period, float* out, double* active_s,
                    double* wall_s) {
  try {
    dpd::Params p;
    p.period = period;
    p.samples = samples;
    p.taps = taps_from(taps);
    p.schedule = sched_from(sched, sched_len);
    p.input = {reinterpret_cast<const std::complex<float>*>(in), samples};
    p.output = {reinterpret_cast<std::complex<float>*>(out), samples};
    NetworkGraph net = dpd::build_network(p);
    ExecutionConfig cfg;
    cfg.source_firing_limit = dpd::source_firings(p);
    RunStats st = run(net, cfg);
    if (active_s) *active_s = st.active_seconds("sink");
    if (wall_s) *wall_s = std::chrono::duration<double>(st.wall).count();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_gauss5x5(const uint8_t* in, uint8_t* out, unsigned w, unsigned h) {
  motion::gauss5x5({in, size_t(w) * h}, {out, size_t(w) * h}, w, h);
}
void ref_thres_diff(const uint8_t* prev, const uint8_t* cur, uint8_t* out, unsigned w,
                    unsigned h, uint8_t thr) {
  const size_t n = size_t(w) * h;
  motion::thres_diff({prev, n}, {cur, n}, {out, n}, w, h, thr);
}
void ref_median5(const uint8_t* in, uint8_t* out, unsigned w, unsigned h) {
  motion::median5({in, size_t(w) * h}, {out, size_t(w) * h}, w, h);
}
void ref_oracle_motion(const uint8_t* frames, size_t count, unsigned w, unsigned h, uint8_t thr,
                       uint8_t* out) {
  auto o = motion::oracle_motion_detection_raw({frames, count * size_t(w) * h}, w, h, thr);
  std::memcpy(out, o.data(), o.size());
}

// proj/src/motion.cpp:107-218 network, timed like cmd_motion:
// frames / active_seconds("sink") (proj/src/bench.cpp:341-347).
int ref_motion_network(const uint8_t* frames, size_t count, unsigned w, unsigned h, uint8_t thr,
                       uint32_t rate, uint8_t* out, double* active_s, double* wall_s) {
  try {
    motion::Params p;
    p.width = w;
    p.height = h;
    p.threshold = thr;
    p.token_rate = rate;
    p.frames = count;
    p.input = {frames, count * size_t(w) * h};
    p.output = {out, count * size_t(w) * h};
    NetworkGraph net = motion::build_network(p);
    ExecutionConfig cfg;
    cfg.source_firing_limit = motion::source_firings(p);
    RunStats st = run(net, cfg);
    if (active_s) *active_s = st.active_seconds("sink");
    if (wall_s) *wall_s = std::chrono::duration<double>(st.wall).count();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

size_t ref_capacity_tokens(uint32_t rate, int has_delay) {
  ChannelSpec s{"c", 1, rate, has_delay != 0, {}};
  return capacity_tokens(s);
}
size_t ref_write_slot(uint32_t rate, int has_delay, unsigned phase) {
  ChannelSpec s{"c", 1, rate, has_delay != 0, {}};
  return write_region(s, phase).first_slot;
}
size_t ref_read_slot(uint32_t rate, int has_delay, unsigned phase) {
  ChannelSpec s{"c", 1, rate, has_delay != 0, {}};
  return read_region(s, phase).first_slot;
}
// Memory report totals (proj/src/channel.cpp:194-208 via cmd_mem's networks).
uint64_t ref_mem_total(int motion_app, unsigned w, unsigned h, uint32_t rate, uint32_t period) {
  try {
    NetworkGraph net;
    if (motion_app) {
      std::vector<uint8_t> io(size_t(w) * h * rate);
      motion::Params p;
      p.width = w; p.height = h; p.token_rate = rate; p.frames = rate;
      p.input = io; p.output = io;
      net = motion::build_network(p);
    } else {
      std::vector<std::complex<float>> io(period);
      dpd::Params p;
      p.period = period; p.samples = period;
      p.schedule = {dpd::ConfigToken::first_n(2)};
      p.input = io; p.output = io;
      net = dpd::build_network(p);
    }
    return memory_bytes(net).total_bytes;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 0;
  }
}

}  // extern "C"
