// motion_net.cpp -- the motion-detection network as GPU actors
// (reference network: /root/reference/proj/src/motion.cpp:107-218).
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "df/motion.hpp"
#include "df/runtime.hpp"
#include "df_cuda.h"

namespace df::motion {

std::uint64_t source_firings(const Params& p) { return p.frames / p.token_rate; }

NetworkGraph build_network(const Params& p) {
  // motion.cpp:108-120
  if (p.width < 5 || p.height < 5) throw std::invalid_argument("motion: frame must be at least 5x5");
  if (p.token_rate < 1) throw std::invalid_argument("motion: token rate must be >= 1");
  if (p.frames % p.token_rate != 0)
    throw std::invalid_argument("motion: frame count must be a multiple of the token rate");
  const std::size_t px = std::size_t(p.width) * p.height;
  const std::size_t in_frame = px * static_cast<unsigned>(p.input_format);
  if (p.input.size() != p.frames * in_frame || p.output.size() != p.frames * px)
    throw std::invalid_argument("motion: input/output buffers must hold exactly `frames` frames");

  const std::uint32_t r = p.token_rate;
  auto input = p.input;
  auto output = p.output;
  std::vector<ChannelSpec> channels = {
      {"src_motion", in_frame, r, false, {}},
      // motion.cpp:131 "gauss_thres_prev": one-frame delay, black initial
      // token -- here a self-loop carrying gauss(last frame) across firings
      {"motion_delay", px, 1, true, {}},
      {"motion_sink", px, r, false, {}},
  };
  std::vector<ActorSpec> actors;

  ActorBehavior source;  // motion.cpp:137-142
  source.fire = [input, in_frame, r](FiringContext& ctx) {
    df_region reg;
    check(df_channel_write_start(ctx.output(0), r, &reg));
    check(df_memcpy_h2d(reg.dptr, input.data() + ctx.firing_index() * r * in_frame, in_frame * r, ctx.stream()));
    check(df_channel_write_end(ctx.output(0), &reg, ctx.stream()));
  };
  actors.push_back({"source", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "src_motion"}},
                    std::move(source)});

  struct MotionState {
    df_motion* h = nullptr;
    ~MotionState() { df_motion_destroy(h); }
  };
  auto st = std::make_shared<MotionState>();
  const unsigned w = p.width, h = p.height, thr = p.threshold;
  const int fmt = static_cast<int>(p.input_format);
  ActorBehavior fused;  // gauss + thres + med actors (motion.cpp:144-176), fused
  fused.fire = [st, w, h, fmt, thr](FiringContext& ctx) {
    if (!st->h) check(df_motion_create(ctx.device(), w, h, fmt, static_cast<std::uint8_t>(thr), &st->h));
    // inputs: src, delay; outputs: delay, sink (declaration order)
    check(df_motion_fire_channels(st->h, ctx.input(0), ctx.input(1), ctx.output(1), ctx.stream()));
  };
  actors.push_back({"motion",
                    ActorKind::static_rate,
                    {{PortDirection::input, PortKind::regular, "src_motion"},
                     {PortDirection::input, PortKind::regular, "motion_delay"},
                     {PortDirection::output, PortKind::regular, "motion_delay"},
                     {PortDirection::output, PortKind::regular, "motion_sink"}},
                    std::move(fused)});

  ActorBehavior sink;  // motion.cpp:178-183
  sink.fire = [output, px, r](FiringContext& ctx) {
    df_region reg;
    check(df_channel_read_start(ctx.input(0), r, &reg));
    check(df_memcpy_d2h(output.data() + ctx.firing_index() * r * px, reg.dptr, px * r, ctx.stream()));
    check(df_channel_read_end(ctx.input(0), &reg, ctx.stream()));
  };
  actors.push_back({"sink", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "motion_sink"}},
                    std::move(sink)});
  return df::build_network(std::move(actors), std::move(channels));
}

NetworkGraph build_mixed_network(const MixedParams& mp) {
  const Params& p = mp.base;
  if (p.input_format != Input::rgb) throw std::invalid_argument("mixed motion network: input must be RGB");
  if (p.width < 5 || p.height < 5) throw std::invalid_argument("motion: frame must be at least 5x5");
  if (p.token_rate < 1) throw std::invalid_argument("motion: token rate must be >= 1");
  if (p.frames % p.token_rate != 0)
    throw std::invalid_argument("motion: frame count must be a multiple of the token rate");
  const std::size_t px = std::size_t(p.width) * p.height;
  if (p.input.size() != p.frames * px * 3 || p.output.size() != p.frames * px || mp.counts.size() != p.frames)
    throw std::invalid_argument("mixed motion network: buffer sizes");
  const std::uint32_t r = p.token_rate;
  auto input = p.input;
  auto output = p.output;
  auto counts = mp.counts;
  const std::int64_t fail_at = mp.fail_at_firing;
  std::vector<ChannelSpec> channels = {
      {"src_gray", px * 3, r, false, {}},
      {"gray_motion", px, r, false, {}},
      {"motion_delay", px, 1, true, {}},
      {"motion_census", px, r, false, {}},
      {"census_sink", px, r, false, {}},
  };
  std::vector<ActorSpec> actors;

  ActorBehavior source;  // GPU-stream actor: H2D of the firing's frames
  source.fire = [input, px, r](FiringContext& ctx) {
    df_region reg;
    check(df_channel_write_start(ctx.output(0), r, &reg));
    check(df_memcpy_h2d(reg.dptr, input.data() + ctx.firing_index() * r * px * 3, px * 3 * r, ctx.stream()));
    check(df_channel_write_end(ctx.output(0), &reg, ctx.stream()));
  };
  actors.push_back({"source", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "src_gray"}},
                    std::move(source)});

  ActorBehavior gray;  // CPU actor
  gray.host_fire = [](HostFiringContext& ctx) {
    const auto in = ctx.input(0);
    const auto out = ctx.output(0);
    const std::size_t n = out.size();
    for (std::size_t i = 0; i < n; ++i) {
      const unsigned R = std::to_integer<unsigned>(in[3 * i]), G = std::to_integer<unsigned>(in[3 * i + 1]),
                     B = std::to_integer<unsigned>(in[3 * i + 2]);
      out[i] = static_cast<std::byte>((77u * R + 150u * G + 29u * B + 128u) >> 8);
    }
  };
  actors.push_back({"gray",
                    ActorKind::static_rate,
                    {{PortDirection::input, PortKind::regular, "src_gray"},
                     {PortDirection::output, PortKind::regular, "gray_motion"}},
                    std::move(gray)});

  struct MotionState {
    df_motion* h = nullptr;
    ~MotionState() { df_motion_destroy(h); }
  };
  auto st = std::make_shared<MotionState>();
  const unsigned w = p.width, h = p.height, thr = p.threshold;
  ActorBehavior fused;  // GPU actor
  fused.fire = [st, w, h, thr](FiringContext& ctx) {
    if (!st->h) check(df_motion_create(ctx.device(), w, h, DF_MOTION_GRAY, static_cast<std::uint8_t>(thr), &st->h));
    check(df_motion_fire_channels(st->h, ctx.input(0), ctx.input(1), ctx.output(1), ctx.stream()));
  };
  actors.push_back({"motion",
                    ActorKind::static_rate,
                    {{PortDirection::input, PortKind::regular, "gray_motion"},
                     {PortDirection::input, PortKind::regular, "motion_delay"},
                     {PortDirection::output, PortKind::regular, "motion_delay"},
                     {PortDirection::output, PortKind::regular, "motion_census"}},
                    std::move(fused)});

  ActorBehavior census;  // CPU actor
  census.host_fire = [counts, px, fail_at](HostFiringContext& ctx) {
    if (fail_at >= 0 && ctx.firing_index() == static_cast<std::uint64_t>(fail_at))
      throw std::runtime_error("census: injected fault at firing " + std::to_string(fail_at));
    const auto in = ctx.input(0);
    const auto out = ctx.output(0);
    const std::size_t frames = ctx.input_tokens(0);
    for (std::size_t f = 0; f < frames; ++f) {
      std::uint32_t c = 0;
      for (std::size_t i = 0; i < px; ++i) c += in[f * px + i] != std::byte{0};
      counts[ctx.firing_index() * frames + f] = c;
    }
    std::memcpy(out.data(), in.data(), in.size());
  };
  actors.push_back({"census",
                    ActorKind::static_rate,
                    {{PortDirection::input, PortKind::regular, "motion_census"},
                     {PortDirection::output, PortKind::regular, "census_sink"}},
                    std::move(census)});

  ActorBehavior sink;
  sink.fire = [output, px, r](FiringContext& ctx) {
    df_region reg;
    check(df_channel_read_start(ctx.input(0), r, &reg));
    check(df_memcpy_d2h(output.data() + ctx.firing_index() * r * px, reg.dptr, px * r, ctx.stream()));
    check(df_channel_read_end(ctx.input(0), &reg, ctx.stream()));
  };
  actors.push_back({"sink", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "census_sink"}},
                    std::move(sink)});
  return df::build_network(std::move(actors), std::move(channels));
}

}  // namespace df::motion
