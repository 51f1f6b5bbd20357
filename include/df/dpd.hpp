// df/dpd.hpp -- the dynamic predistortion network as GPU actors.
//
// Reference: dynflow::dpd (/root/reference/proj/include/dynflow/dpd.hpp,
// proj/src/dpd.cpp:151-356): source -> split -> 10 x (poly -> fir10) ->
// adder -> sink plus a config actor driving 12 control ports, one token of
// `period` samples per firing.  B200 form: source (H2D) -> config (device
// control tokens) -> dpd (ONE dynamic GPU actor: split/branches/adder fused,
// its control token consumed on the device per logical firing) -> sink
// (D2H).  A launch covers `batch` logical firings (channels run at rate
// `batch`, one block token and one control token per logical firing).
#pragma once

#include <complex>
#include <cstdint>
#include <istream>
#include <span>
#include <vector>

#include "df/model.hpp"

struct df_dpd;

namespace df::dpd {

inline constexpr unsigned kBranchCount = 10;

// dpd.hpp:26-36
struct ConfigToken {
  std::uint16_t active_mask = 0;
  unsigned active_count() const { return __builtin_popcount(active_mask); }
  bool active(unsigned branch) const { return (active_mask >> (branch - 1)) & 1u; }
  static ConfigToken first_n(unsigned k) { return {static_cast<std::uint16_t>((1u << k) - 1)}; }
  bool operator==(const ConfigToken&) const = default;
};

// dpd.hpp:37-41: the wire form of a config token, 4 bytes little endian --
// what the config actor writes and the GPU actor reads on the device.
inline constexpr std::size_t kConfigTokenBytes = 4;
void encode_config(ConfigToken token, std::span<std::byte> out);
ConfigToken decode_config(std::span<const std::byte> in);

// check_config (dpd.cpp:49-58): k in [min_active, 10], no branch beyond
// 10.  The reference's bound is k >= 2 (the default); min_active = 1 is the
// single-branch extension BASELINE's ramp schedule needs (its oracle
// accepts any mask), enabled only through Params::allow_single_branch.
void check_config(ConfigToken token, unsigned min_active = 2);

struct Params {
  std::uint32_t period = 65536;       // samples per token (one block)
  std::uint64_t samples = 0;          // multiple of period * batch
  std::uint32_t taps_per_branch = 10;  // 10 = reference; up to 32
  std::vector<std::complex<float>> taps;  // 10 * taps_per_branch, branch-major
  std::vector<ConfigToken> schedule;      // one entry per block, cycling
  std::uint32_t batch = 1;                // logical firings per launch
  bool allow_single_branch = false;       // k = 1 masks (extension; reference: k >= 2)
  std::span<const std::complex<float>> input;  // host, interleaved re/im
  std::span<std::complex<float>> output;
};

// The reference's text formats (dpd.hpp:112-120, dpd.cpp:393-462; the
// parsers are in host/formats.cpp).  Schedule file: one entry per line, "k"
// (branches 1..k) or "k: i1,i2,...,ik"; blank lines and '#' comments
// skipped; k outside [2,10] rejected (std::runtime_error naming the line).
// Taps file: one branch per line, taps_per_branch "re,im" pairs (10 in the
// reference; up to 32 here); returned branch-major as Params::taps.
std::vector<ConfigToken> parse_schedule(std::istream& in);
std::vector<std::complex<float>> parse_taps(std::istream& in, unsigned taps_per_branch = 10);

// The reference's generators (dpd.hpp:122-124; host/generators.cpp):
// schedules of 2..10 branches, taps in [-0.5, 0.5) (10 x T, branch-major),
// samples in [-1, 1), all from std::mt19937_64(seed) as the reference draws.
std::vector<ConfigToken> random_schedule(std::size_t entries, std::uint64_t seed);
std::vector<std::complex<float>> random_taps(std::uint64_t seed, unsigned taps_per_branch = 10);
std::vector<std::complex<float>> synth_samples(std::uint64_t samples, std::uint64_t seed);

NetworkGraph build_network(const Params& params);
std::uint64_t source_firings(const Params& params);  // launches

inline constexpr unsigned kMaxHistory = 31;  // FirState samples for up to 32 taps

// The reference's own network shape (dpd.cpp:151-356: source, config,
// dynamic split, ten dynamic branches, dynamic adder, sink; 56 channels of
// one period per token) as DEVICE-RESIDENT actors: the run is one
// persistent kernel, every split/branch/adder firing reads its control
// token and dispatches its 0-or-1 port rates on the device through the
// reference's control functions (model.hpp:103-108), and the branches keep
// their FirState frozen while gated off.  Input and output spans are host
// memory (staged to HBM by the source's init, back by the sink's finish);
// params.batch is ignored (one block per firing, as the reference).  Needs
// source_firing_limit = samples / period.  branch_ctas: CTAs per branch
// actor (source, split, adder and sink get half).
NetworkGraph build_reference_network(const Params& params, int device = 0, std::uint32_t branch_ctas = 16);

}  // namespace df::dpd
