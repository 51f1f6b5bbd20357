// dpd_net.cpp -- the dynamic predistortion network as GPU actors
// (reference network: /root/reference/proj/src/dpd.cpp:151-356).
#include <memory>
#include <stdexcept>
#include <string>

#include "df/dpd.hpp"
#include "df/runtime.hpp"
#include "df_cuda.h"

namespace df::dpd {

void encode_config(ConfigToken token, std::span<std::byte> out) {  // dpd.cpp:38-41
  if (out.size() < kConfigTokenBytes) throw std::invalid_argument("config token needs 4 bytes");
  const std::uint32_t v = token.active_mask;
  for (std::size_t i = 0; i < kConfigTokenBytes; ++i) out[i] = static_cast<std::byte>((v >> (8 * i)) & 0xFF);
}

ConfigToken decode_config(std::span<const std::byte> in) {  // dpd.cpp:43-47 (bits above 15 are dropped)
  if (in.size() < kConfigTokenBytes) throw std::invalid_argument("config token needs 4 bytes");
  std::uint32_t v = 0;
  for (std::size_t i = 0; i < kConfigTokenBytes; ++i) v |= static_cast<std::uint32_t>(in[i]) << (8 * i);
  return {static_cast<std::uint16_t>(v)};
}

void check_config(ConfigToken token, unsigned min_active) {
  // dpd.cpp:49-58 (the reference network requires k >= 2; k = 1 is the
  // north-star extension, its oracle accepts any mask; see dpd.hpp)
  if (token.active_mask >> kBranchCount) throw std::invalid_argument("config token names a branch beyond 10");
  const unsigned k = token.active_count();
  if (k < min_active || k > kBranchCount)
    throw std::invalid_argument("active branch count " + std::to_string(k) + " outside [" +
                                std::to_string(min_active) + ",10]");
}

std::uint64_t source_firings(const Params& p) { return p.samples / (std::uint64_t(p.period) * p.batch); }

NetworkGraph build_network(const Params& p) {
  if (p.period < 1) throw std::invalid_argument("dpd: period must be >= 1");
  if (p.batch < 1) throw std::invalid_argument("dpd: batch must be >= 1");
  const std::uint64_t launch = std::uint64_t(p.period) * p.batch;
  if (p.samples == 0 || p.samples % launch != 0)
    throw std::invalid_argument("dpd: sample count must be a nonzero multiple of period * batch");
  if (p.schedule.empty()) throw std::invalid_argument("dpd: schedule must not be empty");
  for (ConfigToken t : p.schedule) check_config(t, p.allow_single_branch ? 1 : 2);
  if (p.taps_per_branch < 1 || p.taps_per_branch > 32)
    throw std::invalid_argument("dpd: taps per branch outside [1,32]");
  if (p.taps.size() != std::size_t(kBranchCount) * p.taps_per_branch)
    throw std::invalid_argument("dpd: taps must hold 10 * taps_per_branch values");
  if (p.input.size() != p.samples || p.output.size() != p.samples)
    throw std::invalid_argument("dpd: input/output buffers must hold exactly `samples` samples");

  const std::uint32_t K = p.batch, period = p.period, T = p.taps_per_branch;
  const std::size_t token = std::size_t(period) * sizeof(std::complex<float>);
  auto input = p.input;
  auto output = p.output;
  auto taps = std::make_shared<std::vector<std::complex<float>>>(p.taps);
  auto sched = std::make_shared<std::vector<std::uint16_t>>();
  for (ConfigToken t : p.schedule) sched->push_back(t.active_mask);

  std::vector<ChannelSpec> channels = {
      {"src_dpd", token, K, false, {}},
      {"cfg_dpd", 4, K, false, {}},  // one control token per logical firing
      {"dpd_sink", token, K, false, {}},
  };
  std::vector<ActorSpec> actors;

  ActorBehavior source;  // dpd.cpp:189-204: host input -> channel (H2D)
  source.fire = [input, K, period, token](FiringContext& ctx) {
    df_region r;
    check(df_channel_write_start(ctx.output(0), K, &r));
    check(df_memcpy_h2d(r.dptr, input.data() + ctx.firing_index() * K * period, token * K, ctx.stream()));
    check(df_channel_write_end(ctx.output(0), &r, ctx.stream()));
  };
  actors.push_back({"source", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "src_dpd"}},
                    std::move(source)});

  ActorBehavior config;  // dpd.cpp:206-221, on device
  config.fire = [sched, K](FiringContext& ctx) {
    df_region r;
    check(df_channel_write_start(ctx.output(0), K, &r));
    check(df_dpd_config_tokens(ctx.device(), sched->data(), sched->size(), ctx.firing_index() * K, K,
                               static_cast<std::uint32_t*>(r.dptr), ctx.stream()));
    check(df_channel_write_end(ctx.output(0), &r, ctx.stream()));
  };
  actors.push_back({"config", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "cfg_dpd"}},
                    std::move(config)});

  // The dynamic actor: split + 10 x (poly_branch -> FIR) + adder, one
  // control token per logical firing consumed on the device.
  struct DpdState {
    df_dpd* h = nullptr;
    ~DpdState() { df_dpd_destroy(h); }
  };
  auto st = std::make_shared<DpdState>();
  ActorBehavior fused;
  fused.device_control = true;
  fused.fire = [st, taps, K, period, T](FiringContext& ctx) {
    if (!st->h)
      check(df_dpd_create(ctx.device(), period, T, reinterpret_cast<const float*>(taps->data()), &st->h));
    check(df_dpd_fire_channels(st->h, ctx.control(), ctx.input(0), ctx.output(0), K, ctx.stream()));
  };
  fused.finish = [st] {
    if (st->h) check(df_dpd_error(st->h));  // ControlError: a branch beyond 10
  };
  actors.push_back({"dpd",
                    ActorKind::dynamic_rate,
                    {{PortDirection::input, PortKind::control, "cfg_dpd"},
                     {PortDirection::input, PortKind::regular, "src_dpd"},
                     {PortDirection::output, PortKind::regular, "dpd_sink"}},
                    std::move(fused)});

  ActorBehavior sink;  // dpd.cpp:333-347: channel -> host output (D2H)
  sink.fire = [output, K, period, token](FiringContext& ctx) {
    df_region r;
    check(df_channel_read_start(ctx.input(0), K, &r));
    check(df_memcpy_d2h(output.data() + ctx.firing_index() * K * period, r.dptr, token * K, ctx.stream()));
    check(df_channel_read_end(ctx.input(0), &r, ctx.stream()));
  };
  actors.push_back({"sink", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "dpd_sink"}},
                    std::move(sink)});
  return df::build_network(std::move(actors), std::move(channels));
}

}  // namespace df::dpd
