// resident_net.cpp -- the reference's own network shapes as device-resident
// GPU actors (one persistent kernel per run, csrc/netrt.cu).
//
// DPD: /root/reference/proj/src/dpd.cpp:151-356 -- source, config, a dynamic
// split, ten dynamic branches (poly_branch -> fir with frozen history), a
// dynamic adder and a sink over 44 planar float channels plus 12 control
// channels (56 total, Eq. 1 memory identical to the reference's).  The
// control functions are the reference's (rates 0 or 1 per port from the
// config token), evaluated into device tables; every firing dispatches its
// token on the device.
// Motion: /root/reference/proj/src/motion.cpp:107-218 -- source, gauss,
// thres, med, sink with the one-frame delay channel gauss_thres_prev.
#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>

#include "df/dpd.hpp"
#include "df/motion.hpp"
#include "df/runtime.hpp"
#include "df_cuda.h"

namespace df {

namespace {

// Device buffers owned by a network's behaviors (freed with the last copy).
struct DeviceBuffers {
  std::vector<void*> ptrs;
  ~DeviceBuffers() {
    for (void* p : ptrs) df_free(p);
  }
  void* alloc(int device, std::size_t bytes) {
    void* p = nullptr;
    check(df_set_device(device));
    check(df_malloc(device, bytes ? bytes : 1, &p));
    ptrs.push_back(p);
    return p;
  }
};

std::string tag(unsigned b) { return b < 10 ? "0" + std::to_string(b) : std::to_string(b); }

dpd::ConfigToken decode(std::span<const std::byte> token) {
  std::uint32_t v = 0;
  for (std::size_t i = 0; i < 4 && i < token.size(); ++i) v |= std::uint32_t(token[i]) << (8 * i);
  return {static_cast<std::uint16_t>(v)};
}

}  // namespace

namespace dpd {

NetworkGraph build_reference_network(const Params& p, int device, std::uint32_t branch_ctas) {
  if (p.period < 1) throw std::invalid_argument("dpd: period must be >= 1");
  if (p.samples == 0 || p.samples % p.period != 0)
    throw std::invalid_argument("dpd: sample count must be a nonzero multiple of the period");
  if (p.schedule.empty()) throw std::invalid_argument("dpd: schedule must not be empty");
  for (ConfigToken t : p.schedule) check_config(t, p.allow_single_branch ? 1 : 2);
  if (p.taps_per_branch < 1 || p.taps_per_branch > 32) throw std::invalid_argument("dpd: taps per branch outside [1,32]");
  if (p.taps.size() != std::size_t(kBranchCount) * p.taps_per_branch)
    throw std::invalid_argument("dpd: taps must hold 10 * taps_per_branch values");
  if (p.input.size() != p.samples || p.output.size() != p.samples)
    throw std::invalid_argument("dpd: input/output buffers must hold exactly `samples` samples");
  if (branch_ctas < 1) throw std::invalid_argument("dpd: branch_ctas must be >= 1");

  const std::uint32_t period = p.period, T = p.taps_per_branch;
  const std::size_t plane = std::size_t(period) * sizeof(float), bytes = p.samples * 8;
  auto buf = std::make_shared<DeviceBuffers>();
  void* d_in = buf->alloc(device, bytes);
  void* d_out = buf->alloc(device, bytes);
  std::vector<std::uint16_t> sched;
  for (ConfigToken t : p.schedule) sched.push_back(t.active_mask);
  void* d_sched = buf->alloc(device, sched.size() * 2);
  check(df_memcpy_h2d(d_sched, sched.data(), sched.size() * 2, nullptr));
  check(df_stream_synchronize(nullptr));

  std::vector<ChannelSpec> channels;
  auto pair = [&](const std::string& base) {
    channels.push_back({base + "_re", plane, 1, false, {}});
    channels.push_back({base + "_im", plane, 1, false, {}});
  };
  pair("src_split");
  for (unsigned b = 1; b <= kBranchCount; ++b) pair("split_b" + tag(b));
  for (unsigned b = 1; b <= kBranchCount; ++b) pair("b" + tag(b) + "_adder");
  pair("adder_sink");
  channels.push_back({"cfg_split", 4, 1, false, {}});
  for (unsigned b = 1; b <= kBranchCount; ++b) channels.push_back({"cfg_b" + tag(b), 4, 1, false, {}});
  channels.push_back({"cfg_adder", 4, 1, false, {}});

  const auto in = PortDirection::input, out = PortDirection::output;
  auto reg = [](PortDirection d, const std::string& c) { return PortSpec{d, PortKind::regular, c}; };
  auto ctl = [](const std::string& c) { return PortSpec{PortDirection::input, PortKind::control, c}; };
  std::vector<ActorSpec> actors;

  const std::uint32_t io_ctas = std::max<std::uint32_t>(1, branch_ctas);
  ActorBehavior source;  // dpd.cpp:189-204 (input staged to HBM before the run)
  source.device = DeviceActor::of(DF_ACT_DPD_SOURCE, df_act_samples{d_in, period}, io_ctas);
  const auto input = p.input;
  source.init = [buf, d_in, input, bytes] {
    check(df_memcpy_h2d(d_in, input.data(), bytes, nullptr));
    check(df_stream_synchronize(nullptr));
  };
  actors.push_back({"source", ActorKind::static_rate, {reg(out, "src_split_re"), reg(out, "src_split_im")}, source});

  ActorBehavior config;  // dpd.cpp:206-221
  config.device = DeviceActor::of(DF_ACT_DPD_CONFIG, df_act_config{static_cast<const std::uint16_t*>(d_sched),
                                                                   static_cast<std::uint32_t>(sched.size())});
  std::vector<PortSpec> cfg_ports = {reg(out, "cfg_split")};
  for (unsigned b = 1; b <= kBranchCount; ++b) cfg_ports.push_back(reg(out, "cfg_b" + tag(b)));
  cfg_ports.push_back(reg(out, "cfg_adder"));
  actors.push_back({"config", ActorKind::static_rate, cfg_ports, config});

  ActorBehavior split;  // dpd.cpp:225-256: input pair every firing, active branch pairs
  split.device = DeviceActor::of(DF_ACT_DPD_SPLIT, 0, io_ctas);
  split.device.params.clear();
  split.control = [](std::span<const std::byte> token) {
    const ConfigToken cfg = decode(token);
    FiringRates r;
    r.by_regular_port.assign(2, 1);
    for (unsigned b = 1; b <= kBranchCount; ++b) {
      const std::uint32_t on = cfg.active(b) ? 1 : 0;
      r.by_regular_port.push_back(on);
      r.by_regular_port.push_back(on);
    }
    return r;
  };
  std::vector<PortSpec> split_ports = {ctl("cfg_split"), reg(in, "src_split_re"), reg(in, "src_split_im")};
  for (unsigned b = 1; b <= kBranchCount; ++b) {
    split_ports.push_back(reg(out, "split_b" + tag(b) + "_re"));
    split_ports.push_back(reg(out, "split_b" + tag(b) + "_im"));
  }
  actors.push_back({"split", ActorKind::dynamic_rate, split_ports, split});

  for (unsigned b = 1; b <= kBranchCount; ++b) {  // dpd.cpp:258-289
    void* d_taps = buf->alloc(device, std::size_t(T) * 8);
    void* d_state = buf->alloc(device, std::size_t(kMaxHistory) * 8);
    check(df_memcpy_h2d(d_taps, p.taps.data() + std::size_t(b - 1) * T, std::size_t(T) * 8, nullptr));
    check(df_memset(d_state, 0, std::size_t(kMaxHistory) * 8, nullptr));
    ActorBehavior branch;
    branch.device = DeviceActor::of(
        DF_ACT_DPD_BRANCH,
        df_act_branch{b, T, static_cast<const float*>(d_taps), static_cast<float*>(d_state), period}, branch_ctas);
    branch.control = [b](std::span<const std::byte> token) {
      return FiringRates::uniform(4, decode(token).active(b) ? 1 : 0);
    };
    branch.init = [buf, d_state] { check(df_memset(d_state, 0, std::size_t(kMaxHistory) * 8, nullptr)); };
    actors.push_back({"branch" + tag(b),
                      ActorKind::dynamic_rate,
                      {ctl("cfg_b" + tag(b)), reg(in, "split_b" + tag(b) + "_re"), reg(in, "split_b" + tag(b) + "_im"),
                       reg(out, "b" + tag(b) + "_adder_re"), reg(out, "b" + tag(b) + "_adder_im")},
                      branch});
  }
  check(df_stream_synchronize(nullptr));

  ActorBehavior adder;  // dpd.cpp:293-331
  adder.device = DeviceActor::of(DF_ACT_DPD_ADDER, 0, io_ctas);
  adder.device.params.clear();
  adder.control = [](std::span<const std::byte> token) {
    const ConfigToken cfg = decode(token);
    FiringRates r;
    for (unsigned b = 1; b <= kBranchCount; ++b) {
      const std::uint32_t on = cfg.active(b) ? 1 : 0;
      r.by_regular_port.push_back(on);
      r.by_regular_port.push_back(on);
    }
    r.by_regular_port.push_back(1);
    r.by_regular_port.push_back(1);
    return r;
  };
  std::vector<PortSpec> adder_ports = {ctl("cfg_adder")};
  for (unsigned b = 1; b <= kBranchCount; ++b) {
    adder_ports.push_back(reg(in, "b" + tag(b) + "_adder_re"));
    adder_ports.push_back(reg(in, "b" + tag(b) + "_adder_im"));
  }
  adder_ports.push_back(reg(out, "adder_sink_re"));
  adder_ports.push_back(reg(out, "adder_sink_im"));
  actors.push_back({"adder", ActorKind::dynamic_rate, adder_ports, adder});

  ActorBehavior sink;  // dpd.cpp:333-347 (output copied back after the run)
  sink.device = DeviceActor::of(DF_ACT_DPD_SINK, df_act_samples{d_out, period}, io_ctas);
  const auto output = p.output;
  sink.finish = [buf, d_out, output, bytes] {
    check(df_memcpy_d2h(output.data(), d_out, bytes, nullptr));
    check(df_stream_synchronize(nullptr));
  };
  actors.push_back({"sink", ActorKind::static_rate, {reg(in, "adder_sink_re"), reg(in, "adder_sink_im")}, sink});
  return df::build_network(std::move(actors), std::move(channels));
}

}  // namespace dpd

namespace motion {

NetworkGraph build_reference_network(const Params& p, int device, std::uint32_t ctas) {
  if (p.width < 5 || p.height < 5) throw std::invalid_argument("motion: frame must be at least 5x5");
  if (p.token_rate < 1) throw std::invalid_argument("motion: token rate must be >= 1");
  if (p.frames % p.token_rate != 0)
    throw std::invalid_argument("motion: frame count must be a multiple of the token rate");
  if (p.input_format != Input::gray)
    throw std::invalid_argument("motion: the reference network takes 8-bit gray frames");
  const std::size_t size = std::size_t(p.width) * p.height, bytes = p.frames * size;
  if (p.input.size() != bytes || p.output.size() != bytes)
    throw std::invalid_argument("motion: input/output buffers must hold exactly `frames` frames");
  if (ctas < 1) throw std::invalid_argument("motion: ctas must be >= 1");
  auto buf = std::make_shared<DeviceBuffers>();
  void* d_in = buf->alloc(device, bytes);
  void* d_out = buf->alloc(device, bytes);
  const std::uint32_t r = p.token_rate;
  std::vector<ChannelSpec> channels = {
      {"gauss_thres_cur", size, r, false, {}},
      {"gauss_thres_prev", size, r, true, {}},  // one-frame delay, black initial frame (motion.cpp:131)
      {"med_sink", size, r, false, {}},
      {"src_gauss", size, r, false, {}},
      {"thres_med", size, r, false, {}},
  };
  const df_act_frames fp{nullptr, p.width, p.height, p.threshold};
  const auto in = PortDirection::input, out = PortDirection::output;
  auto reg = [](PortDirection d, const char* c) { return PortSpec{d, PortKind::regular, c}; };
  ActorBehavior source, gauss, thres, med, sink;
  df_act_frames sp = fp, kp = fp;
  sp.frames = d_in;
  kp.frames = d_out;
  // `ctas` is the mean per actor: the group sizes follow each actor's work
  // per frame (gauss 15 loads per 4 px, median 5 + a sorting network, thres
  // 2, source / sink a copy), so the 5 * ctas CTAs of one wave are spent where
  // the firing time is (DF_NET_PROFILE: fire times 1 : 0.77 : 0.52 : 0.3).
  auto share = [ctas](std::uint32_t num, std::uint32_t den) { return std::max<std::uint32_t>(1, ctas * num / den); };
  source.device = DeviceActor::of(DF_ACT_FRAME_SOURCE, sp, share(5, 8));
  const auto input = p.input;
  source.init = [buf, d_in, input, bytes] {
    check(df_memcpy_h2d(d_in, input.data(), bytes, nullptr));
    check(df_stream_synchronize(nullptr));
  };
  gauss.device = DeviceActor::of(DF_ACT_GAUSS, fp, share(5, 3));
  thres.device = DeviceActor::of(DF_ACT_THRES, fp, share(5, 6));
  med.device = DeviceActor::of(DF_ACT_MEDIAN, fp, share(5, 4));
  sink.device = DeviceActor::of(DF_ACT_FRAME_SINK, kp, share(5, 8));
  const auto output = p.output;
  sink.finish = [buf, d_out, output, bytes] {
    check(df_memcpy_d2h(output.data(), d_out, bytes, nullptr));
    check(df_stream_synchronize(nullptr));
  };
  std::vector<ActorSpec> actors = {
      {"source", ActorKind::static_rate, {reg(out, "src_gauss")}, source},
      {"gauss", ActorKind::static_rate, {reg(in, "src_gauss"), reg(out, "gauss_thres_cur"), reg(out, "gauss_thres_prev")}, gauss},
      {"thres", ActorKind::static_rate, {reg(in, "gauss_thres_prev"), reg(in, "gauss_thres_cur"), reg(out, "thres_med")}, thres},
      {"med", ActorKind::static_rate, {reg(in, "thres_med"), reg(out, "med_sink")}, med},
      {"sink", ActorKind::static_rate, {reg(in, "med_sink")}, sink},
  };
  return df::build_network(std::move(actors), std::move(channels));
}

}  // namespace motion
}  // namespace df
