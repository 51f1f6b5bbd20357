// df/motion.hpp -- the motion-detection network as GPU actors.
//
// Reference: dynflow::motion (/root/reference/proj/src/motion.cpp:107-218):
// source -> gauss -> (cur, prev with a one-frame delay token) -> thres ->
// med -> sink.  B200 form: source (H2D) -> motion (ONE fused GPU actor:
// gray/gauss/thres/median; the prev stream is a rate-1 self-loop delay
// channel carrying gauss of the last frame, black initially) -> sink (D2H).
#pragma once

#include <cstdint>
#include <span>

#include "df/model.hpp"

namespace df::motion {

enum class Input { gray = 1, rgb = 3 };

struct Params {
  unsigned width = 320;
  unsigned height = 240;
  std::uint8_t threshold = 32;
  std::uint32_t token_rate = 1;  // frames per firing
  std::uint64_t frames = 0;      // multiple of token_rate
  Input input_format = Input::gray;
  std::span<const std::uint8_t> input;  // frames * width * height * format bytes (host)
  std::span<std::uint8_t> output;       // frames * width * height bytes (host)
};

NetworkGraph build_network(const Params& params);
std::uint64_t source_firings(const Params& params);

// The reference's own network shape (motion.cpp:107-218: source -> gauss ->
// cur + prev (delay channel, black initial frame) -> thres -> med -> sink,
// rate r on every channel) as DEVICE-RESIDENT actors, each run by `ctas`
// CTAs of one persistent kernel.  Gray input only (the reference's format);
// host spans staged to HBM by the source's init / back by the sink's finish.
NetworkGraph build_reference_network(const Params& params, int device = 0, std::uint32_t ctas = 64);

// Heterogeneous network (CPU + GPU actors on shared device channels, the
// paper's mixed mapping): source (H2D, RGB) -> gray (CPU actor: BT.601
// integer luma) -> motion (GPU actor, gray input) -> census (CPU actor:
// counts moving pixels per frame into `counts`, passes the masks on) ->
// sink (D2H).  census throws at firing `fail_at_firing` when >= 0 (fault
// injection: the run ends in ActorFault("census")).
struct MixedParams {
  Params base;                       // input_format must be rgb
  std::span<std::uint32_t> counts;   // frames entries (host)
  std::int64_t fail_at_firing = -1;
};
NetworkGraph build_mixed_network(const MixedParams& params);

// The reference's frame generator (motion.hpp:77, motion.cpp:254-260):
// one byte per draw of std::mt19937_64(seed).
std::vector<std::uint8_t> synth_frames(std::uint64_t frames, unsigned width, unsigned height, std::uint64_t seed);

}  // namespace df::motion
