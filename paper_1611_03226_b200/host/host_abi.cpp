// host_abi.cpp -- extern "C" entry points of libdf_host.so (df_host.h).
#include <complex>
#include <cstring>
#include <memory>
#include <string>

#include <sstream>

#include "df/channel.hpp"
#include "df/dpd.hpp"
#include "df/io.hpp"
#include "df/motion.hpp"
#include "df/runtime.hpp"
#include "df_cuda.h"
#include "df_host.h"

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const df::ActorFault& e) {
    g_err = std::string("ActorFault: ") + e.what();
    return 3;
  } catch (const df::ValidationError& e) {
    g_err = std::string("ValidationError: ") + e.what();
    return 4;
  } catch (const df::BuildError& e) {
    g_err = std::string("BuildError: ") + e.what();
    return 7;
  } catch (const df::io::FormatError& e) {
    g_err = std::string("FormatError: ") + e.what();
    return 8;
  } catch (const df::ControlError& e) {
    g_err = std::string("ControlError: ") + e.what();
    return 5;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("error: ") + e.what();
    return 6;
  }
}
}  // namespace

extern "C" {

const char* dfh_last_error(void) { return g_err.c_str(); }

int dfh_dpd_run(int device, const float* in_host, float* out_host, uint64_t samples, uint32_t period,
                uint32_t T, const float* taps, const uint16_t* schedule, size_t schedule_len, uint32_t batch,
                int allow_single_branch, double* sink_active_ms, uint64_t* dpd_firings) {
  return guarded([&] {
    df::dpd::Params p;
    p.period = period;
    p.samples = samples;
    p.taps_per_branch = T;
    p.taps.resize(std::size_t(10) * T);
    for (std::size_t i = 0; i < p.taps.size(); ++i) p.taps[i] = {taps[2 * i], taps[2 * i + 1]};
    for (size_t i = 0; i < schedule_len; ++i) p.schedule.push_back({schedule[i]});
    p.batch = batch;
    p.allow_single_branch = allow_single_branch != 0;
    p.input = {reinterpret_cast<const std::complex<float>*>(in_host), samples};
    p.output = {reinterpret_cast<std::complex<float>*>(out_host), samples};
    df::NetworkGraph net = df::dpd::build_network(p);
    df::ExecutionConfig cfg;
    cfg.device = device;
    cfg.source_firing_limit = df::dpd::source_firings(p);
    df::RunStats st = df::run(net, cfg);
    if (sink_active_ms) *sink_active_ms = st.actor("sink").active_ms;
    if (dpd_firings) *dpd_firings = st.firings("dpd");
  });
}

int dfh_motion_run(int device, const uint8_t* in_host, uint8_t* out_host, uint64_t frames, unsigned width,
                   unsigned height, int fmt, uint8_t threshold, uint32_t rate, double* sink_active_ms,
                   uint64_t* delay_tokens_written) {
  return guarded([&] {
    df::motion::Params p;
    p.width = width;
    p.height = height;
    p.threshold = threshold;
    p.token_rate = rate;
    p.frames = frames;
    p.input_format = fmt == 3 ? df::motion::Input::rgb : df::motion::Input::gray;
    const std::size_t px = std::size_t(width) * height;
    p.input = {in_host, frames * px * static_cast<unsigned>(fmt == 3 ? 3 : 1)};
    p.output = {out_host, frames * px};
    df::NetworkGraph net = df::motion::build_network(p);
    df::ExecutionConfig cfg;
    cfg.device = device;
    cfg.source_firing_limit = df::motion::source_firings(p);
    df::RunStats st = df::run(net, cfg);
    if (sink_active_ms) *sink_active_ms = st.actor("sink").active_ms;
    if (delay_tokens_written)
      for (const auto& c : st.channels)
        if (c.id == "motion_delay") *delay_tokens_written = c.tokens_written;
  });
}

int dfh_dpd_run_resident(int device, const float* in_host, float* out_host, uint64_t samples, uint32_t period,
                         uint32_t T, const float* taps, const uint16_t* schedule, size_t schedule_len,
                         int allow_single_branch, uint32_t branch_ctas, double timeout_s, double* sink_active_ms,
                         uint64_t* firings, uint64_t* channel_tokens) {
  return guarded([&] {
    df::dpd::Params p;
    p.period = period;
    p.samples = samples;
    p.taps_per_branch = T;
    p.taps.resize(std::size_t(10) * T);
    for (std::size_t i = 0; i < p.taps.size(); ++i) p.taps[i] = {taps[2 * i], taps[2 * i + 1]};
    for (size_t i = 0; i < schedule_len; ++i) p.schedule.push_back({schedule[i]});
    p.allow_single_branch = allow_single_branch != 0;
    p.input = {reinterpret_cast<const std::complex<float>*>(in_host), samples};
    p.output = {reinterpret_cast<std::complex<float>*>(out_host), samples};
    df::NetworkGraph net = df::dpd::build_reference_network(p, device, branch_ctas);
    df::ExecutionConfig cfg;
    cfg.device = device;
    cfg.source_firing_limit = samples / period;
    cfg.device_timeout_s = timeout_s;
    df::RunStats st = df::run(net, cfg);
    if (sink_active_ms) *sink_active_ms = st.actor("sink").active_ms;
    if (firings)
      for (std::size_t a = 0; a < st.actors.size(); ++a) firings[a] = st.actors[a].firings;
    if (channel_tokens)
      for (std::size_t c = 0; c < st.channels.size(); ++c) channel_tokens[c] = st.channels[c].tokens_written;
  });
}

int dfh_motion_run_resident(int device, const uint8_t* in_host, uint8_t* out_host, uint64_t frames, unsigned width,
                            unsigned height, uint8_t threshold, uint32_t rate, uint32_t ctas, double timeout_s,
                            double* sink_active_ms, uint64_t* firings) {
  return guarded([&] {
    df::motion::Params p;
    p.width = width;
    p.height = height;
    p.threshold = threshold;
    p.token_rate = rate;
    p.frames = frames;
    const std::size_t px = std::size_t(width) * height;
    p.input = {in_host, frames * px};
    p.output = {out_host, frames * px};
    df::NetworkGraph net = df::motion::build_reference_network(p, device, ctas);
    df::ExecutionConfig cfg;
    cfg.device = device;
    cfg.source_firing_limit = frames / rate;
    cfg.device_timeout_s = timeout_s;
    df::RunStats st = df::run(net, cfg);
    if (sink_active_ms) *sink_active_ms = st.actor("sink").active_ms;
    if (firings)
      for (std::size_t a = 0; a < st.actors.size(); ++a) firings[a] = st.actors[a].firings;
  });
}

int dfh_motion_run_mixed(int device, const uint8_t* rgb_host, uint8_t* out_host, uint64_t frames, unsigned width,
                         unsigned height, uint8_t threshold, uint32_t rate, uint32_t* counts,
                         int64_t fail_at_firing, double* sink_active_ms) {
  return guarded([&] {
    df::motion::MixedParams mp;
    df::motion::Params& p = mp.base;
    p.width = width;
    p.height = height;
    p.threshold = threshold;
    p.token_rate = rate;
    p.frames = frames;
    p.input_format = df::motion::Input::rgb;
    const std::size_t px = std::size_t(width) * height;
    p.input = {rgb_host, frames * px * 3};
    p.output = {out_host, frames * px};
    mp.counts = {counts, frames};
    mp.fail_at_firing = fail_at_firing;
    df::NetworkGraph net = df::motion::build_mixed_network(mp);
    df::ExecutionConfig cfg;
    cfg.device = device;
    cfg.source_firing_limit = df::motion::source_firings(p);
    df::RunStats st = df::run(net, cfg);
    if (sink_active_ms) *sink_active_ms = st.actor("sink").active_ms;
  });
}

int dfh_memory(int app, unsigned width, unsigned height, uint32_t rate, uint32_t period, int shape,
               uint64_t* total_bytes) {
  int n = -1;
  int rc = guarded([&] {
    using namespace df;
    auto noop = [](FiringContext&) {};
    NetworkGraph net;
    if (shape == 0 && app == 0) {  // the B200 motion network (one firing's worth of frames shapes it)
      std::vector<std::uint8_t> io(std::size_t(width) * height * rate);
      motion::Params p;
      p.width = width;
      p.height = height;
      p.token_rate = rate;
      p.frames = rate;
      p.input = io;
      p.output = io;
      net = motion::build_network(p);
    } else if (shape == 0) {  // the B200 DPD network
      std::vector<std::complex<float>> io(period), taps(100);
      dpd::Params p;
      p.period = period;
      p.samples = period;
      p.taps = taps;
      p.schedule = {dpd::ConfigToken::first_n(2)};
      p.input = io;
      p.output = io;
      net = dpd::build_network(p);
    } else if (app == 0) {  // reference motion shape (motion.cpp:107-218)
      const std::size_t S = std::size_t(width) * height;
      std::vector<ChannelSpec> ch = {{"src_gauss", S, rate, false, {}},
                                     {"gauss_thres_cur", S, rate, false, {}},
                                     {"gauss_thres_prev", S, rate, true, {}},
                                     {"thres_med", S, rate, false, {}},
                                     {"med_sink", S, rate, false, {}}};
      ActorBehavior b;
      b.fire = noop;
      auto port = [](PortDirection d, const char* c) { return PortSpec{d, PortKind::regular, c}; };
      const auto in = PortDirection::input, out = PortDirection::output;
      std::vector<ActorSpec> a = {
          {"source", ActorKind::static_rate, {port(out, "src_gauss")}, b},
          {"gauss", ActorKind::static_rate,
           {port(in, "src_gauss"), port(out, "gauss_thres_cur"), port(out, "gauss_thres_prev")}, b},
          {"thres", ActorKind::static_rate,
           {port(in, "gauss_thres_prev"), port(in, "gauss_thres_cur"), port(out, "thres_med")}, b},
          {"med", ActorKind::static_rate, {port(in, "thres_med"), port(out, "med_sink")}, b},
          {"sink", ActorKind::static_rate, {port(in, "med_sink")}, b}};
      net = build_network(a, ch);
    } else {  // reference DPD shape (dpd.cpp:151-356): 44 float planes + 12 config channels
      const std::size_t plane = std::size_t(period) * sizeof(float);
      std::vector<ChannelSpec> ch;
      auto pair = [&](const std::string& base) {
        ch.push_back({base + "_re", plane, 1, false, {}});
        ch.push_back({base + "_im", plane, 1, false, {}});
      };
      pair("src_split");
      for (int b = 1; b <= 10; ++b) pair("split_b" + std::to_string(b));
      for (int b = 1; b <= 10; ++b) pair("b" + std::to_string(b) + "_adder");
      pair("adder_sink");
      ch.push_back({"cfg_split", 4, 1, false, {}});
      for (int b = 1; b <= 10; ++b) ch.push_back({"cfg_b" + std::to_string(b), 4, 1, false, {}});
      ch.push_back({"cfg_adder", 4, 1, false, {}});
      ActorBehavior st, dyn;
      st.fire = noop;
      dyn.fire = noop;
      dyn.device_control = true;
      const auto in = PortDirection::input, out = PortDirection::output;
      auto reg = [](PortDirection d, const std::string& c) { return PortSpec{d, PortKind::regular, c}; };
      std::vector<ActorSpec> a;
      a.push_back({"source", ActorKind::static_rate, {reg(out, "src_split_re"), reg(out, "src_split_im")}, st});
      std::vector<PortSpec> cfg_ports = {reg(out, "cfg_split")};
      for (int b = 1; b <= 10; ++b) cfg_ports.push_back(reg(out, "cfg_b" + std::to_string(b)));
      cfg_ports.push_back(reg(out, "cfg_adder"));
      a.push_back({"config", ActorKind::static_rate, cfg_ports, st});
      std::vector<PortSpec> split = {{in, PortKind::control, "cfg_split"}, reg(in, "src_split_re"),
                                     reg(in, "src_split_im")};
      for (int b = 1; b <= 10; ++b) {
        split.push_back(reg(out, "split_b" + std::to_string(b) + "_re"));
        split.push_back(reg(out, "split_b" + std::to_string(b) + "_im"));
      }
      a.push_back({"split", ActorKind::dynamic_rate, split, dyn});
      for (int b = 1; b <= 10; ++b) {
        const std::string t = std::to_string(b);
        a.push_back({"branch" + t, ActorKind::dynamic_rate,
                     {{in, PortKind::control, "cfg_b" + t}, reg(in, "split_b" + t + "_re"),
                      reg(in, "split_b" + t + "_im"), reg(out, "b" + t + "_adder_re"),
                      reg(out, "b" + t + "_adder_im")},
                     dyn});
      }
      std::vector<PortSpec> adder = {{in, PortKind::control, "cfg_adder"}};
      for (int b = 1; b <= 10; ++b) {
        adder.push_back(reg(in, "b" + std::to_string(b) + "_adder_re"));
        adder.push_back(reg(in, "b" + std::to_string(b) + "_adder_im"));
      }
      adder.push_back(reg(out, "adder_sink_re"));
      adder.push_back(reg(out, "adder_sink_im"));
      a.push_back({"adder", ActorKind::dynamic_rate, adder, dyn});
      a.push_back({"sink", ActorKind::static_rate, {reg(in, "adder_sink_re"), reg(in, "adder_sink_im")}, st});
      net = build_network(a, ch);
    }
    const auto v = validate(net);
    if (!v.empty()) throw std::invalid_argument("network shape failed validation: " + v.front().message);
    const MemoryReport r = memory_bytes(net);
    if (total_bytes) *total_bytes = r.total_bytes;
    n = (int)r.channels.size();
  });
  return rc == 0 ? n : -1;
}

int dfh_delay_chain_run(int device, uint32_t rate, int sink_first, uint64_t firings, uint64_t* out_host) {
  return guarded([&] {
    using namespace df;
    // source --(delay channel, rate r, initial token 0xFFFF...)--> sink.
    // Source firing i writes tokens with values i*r+1 .. i*r+r; the sink
    // reads r tokens per firing: the initial token, then the stream.
    auto values = std::make_shared<std::vector<std::uint64_t>>(firings * rate);
    for (std::size_t i = 0; i < values->size(); ++i) (*values)[i] = i + 1;
    std::vector<std::byte> init(8, std::byte{0xFF});
    std::vector<ChannelSpec> chans = {{"d", 8, rate, true, init}};
    ActorBehavior src, snk;
    src.fire = [values, rate](FiringContext& ctx) {
      df_region r;
      check(df_channel_write_start(ctx.output(0), rate, &r));
      check(df_memcpy_h2d(r.dptr, values->data() + ctx.firing_index() * rate, 8ull * rate, ctx.stream()));
      check(df_channel_write_end(ctx.output(0), &r, ctx.stream()));
    };
    snk.fire = [out_host, rate](FiringContext& ctx) {
      df_region r;
      check(df_channel_read_start(ctx.input(0), rate, &r));
      check(df_memcpy_d2h(out_host + ctx.firing_index() * rate, r.dptr, 8ull * rate, ctx.stream()));
      check(df_channel_read_end(ctx.input(0), &r, ctx.stream()));
    };
    ActorSpec a_src{"source", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "d"}}, src};
    ActorSpec a_snk{"sink", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "d"}}, snk};
    std::vector<ActorSpec> actors;
    if (sink_first) {
      actors = {a_snk, a_src};
    } else {
      actors = {a_src, a_snk};
    }
    ExecutionConfig cfg;
    cfg.device = device;
    cfg.source_firing_limit = firings;
    run(build_network(actors, chans), cfg);
  });
}

// The reference's dynamic DPD network shape with CPU actors on device
// channels (the static-schedule runtime): source -> split (dynamic: its
// outputs gated by the control token) -> branch1, branch2 (dynamic, gated
// in and out, each with a running state that stays frozen while gated off)
// -> adder (dynamic: gated inputs, always one output) -> sink, plus a config
// actor feeding the four control channels from `masks` (cycling).  Tokens
// are int32; source firing i emits i*r+1 .. i*r+r; branch b emits
// x * (b+1) + state_b (state_b += sum of its inputs, wrapping); the adder
// sums the active inputs.  A mask above 3 makes every control function
// return an illegal rate (ControlError -> ActorFault).
int dfh_dynamic_cpu_run(int device, const uint32_t* masks, size_t n_masks, uint32_t rate, uint64_t firings,
                        int32_t* out_host) {
  return guarded([&] {
    using namespace df;
    if (!masks || !n_masks || !out_host || !rate) throw std::invalid_argument("dfh_dynamic_cpu_run: bad argument");
    const std::vector<std::uint32_t> sched(masks, masks + n_masks);
    std::vector<ChannelSpec> chans;
    for (const char* id : {"src_split", "split_b1", "split_b2", "b1_adder", "b2_adder", "adder_sink"})
      chans.push_back({id, 4, rate, false, {}});
    for (const char* id : {"cfg_split", "cfg_b1", "cfg_b2", "cfg_adder"}) chans.push_back({id, 4, 1, false, {}});
    auto i32 = [](std::span<const std::byte> s) { return reinterpret_cast<const std::int32_t*>(s.data()); };
    auto o32 = [](std::span<std::byte> s) { return reinterpret_cast<std::int32_t*>(s.data()); };
    auto mask_of = [](std::span<const std::byte> t) {
      std::uint32_t m = 0;
      std::memcpy(&m, t.data(), 4);
      return m;
    };
    const std::uint32_t r = rate;
    auto gate = [r](std::uint32_t m, unsigned bit) -> std::uint32_t {
      if (m > 3) return 7;  // not 0 or r: control_dispatch raises ControlError
      return ((m >> bit) & 1u) ? r : 0u;
    };
    std::vector<ActorSpec> actors;
    ActorBehavior src;
    src.host_fire = [r](HostFiringContext& ctx) {
      std::int32_t* o = reinterpret_cast<std::int32_t*>(ctx.output(0).data());
      for (std::uint32_t t = 0; t < r; ++t) o[t] = static_cast<std::int32_t>(ctx.firing_index() * r + t + 1);
    };
    actors.push_back({"source", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "src_split"}}, src});
    ActorBehavior cfg;
    cfg.host_fire = [sched](HostFiringContext& ctx) {
      const std::uint32_t m = sched[ctx.firing_index() % sched.size()];
      for (std::size_t o = 0; o < ctx.output_count(); ++o) std::memcpy(ctx.output(o).data(), &m, 4);
    };
    actors.push_back({"config", ActorKind::static_rate,
                      {{PortDirection::output, PortKind::regular, "cfg_split"},
                       {PortDirection::output, PortKind::regular, "cfg_b1"},
                       {PortDirection::output, PortKind::regular, "cfg_b2"},
                       {PortDirection::output, PortKind::regular, "cfg_adder"}},
                      cfg});
    ActorBehavior split;
    split.control = [=](std::span<const std::byte> t) {
      const std::uint32_t m = mask_of(t);
      return FiringRates{{m > 3 ? 7u : r, gate(m, 0), gate(m, 1)}};
    };
    split.host_fire = [=](HostFiringContext& ctx) {
      for (std::size_t o = 0; o < ctx.output_count(); ++o)
        if (ctx.output_tokens(o)) std::memcpy(ctx.output(o).data(), ctx.input(0).data(), ctx.output(o).size());
    };
    actors.push_back({"split", ActorKind::dynamic_rate,
                      {{PortDirection::input, PortKind::control, "cfg_split"},
                       {PortDirection::input, PortKind::regular, "src_split"},
                       {PortDirection::output, PortKind::regular, "split_b1"},
                       {PortDirection::output, PortKind::regular, "split_b2"}},
                      split});
    for (unsigned b = 1; b <= 2; ++b) {
      auto state = std::make_shared<std::int32_t>(0);
      ActorBehavior br;
      br.control = [=](std::span<const std::byte> t) {
        const std::uint32_t g = gate(mask_of(t), b - 1);
        return FiringRates{{g, g}};
      };
      br.host_fire = [=](HostFiringContext& ctx) {
        if (!ctx.input_tokens(0)) return;  // gated off: no I/O, state frozen
        const std::int32_t* x = i32(ctx.input(0));
        std::int32_t* y = o32(ctx.output(0));
        std::uint32_t s = static_cast<std::uint32_t>(*state);
        for (std::uint32_t t = 0; t < r; ++t) s += static_cast<std::uint32_t>(x[t]);
        *state = static_cast<std::int32_t>(s);
        for (std::uint32_t t = 0; t < r; ++t)
          y[t] = static_cast<std::int32_t>(static_cast<std::uint32_t>(x[t]) * (b + 1) + s);
      };
      const std::string n = std::to_string(b);
      actors.push_back({"branch" + n, ActorKind::dynamic_rate,
                        {{PortDirection::input, PortKind::control, "cfg_b" + n},
                         {PortDirection::input, PortKind::regular, "split_b" + n},
                         {PortDirection::output, PortKind::regular, "b" + n + "_adder"}},
                        br});
    }
    ActorBehavior adder;
    adder.control = [=](std::span<const std::byte> t) {
      const std::uint32_t m = mask_of(t);
      return FiringRates{{gate(m, 0), gate(m, 1), m > 3 ? 7u : r}};
    };
    adder.host_fire = [=](HostFiringContext& ctx) {
      std::int32_t* y = o32(ctx.output(0));
      for (std::uint32_t t = 0; t < r; ++t) {
        std::uint32_t acc = 0;
        for (std::size_t k = 0; k < ctx.input_count(); ++k)
          if (ctx.input_tokens(k)) acc += static_cast<std::uint32_t>(i32(ctx.input(k))[t]);
        y[t] = static_cast<std::int32_t>(acc);
      }
    };
    actors.push_back({"adder", ActorKind::dynamic_rate,
                      {{PortDirection::input, PortKind::control, "cfg_adder"},
                       {PortDirection::input, PortKind::regular, "b1_adder"},
                       {PortDirection::input, PortKind::regular, "b2_adder"},
                       {PortDirection::output, PortKind::regular, "adder_sink"}},
                      adder});
    ActorBehavior sink;
    sink.host_fire = [=](HostFiringContext& ctx) {
      std::memcpy(out_host + ctx.firing_index() * r, ctx.input(0).data(), 4ull * r);
    };
    actors.push_back({"sink", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "adder_sink"}}, sink});
    ExecutionConfig ec;
    ec.device = device;
    ec.source_firing_limit = firings;
    run(build_network(actors, chans), ec);
  });
}

// source (CPU) -> doubler (bulk_kernel_adapter: int32 x -> 2x, or a wrong
// output size when bad) -> sink (CPU); out_host: firings * rate int32.
int dfh_bulk_kernel_run(int device, uint32_t rate, uint64_t firings, int bad, int32_t* out_host) {
  return guarded([&] {
    using namespace df;
    if (!out_host || !rate) throw std::invalid_argument("dfh_bulk_kernel_run: bad argument");
    std::vector<ChannelSpec> chans = {{"a", 4, rate, false, {}}, {"b", 4, rate, false, {}}};
    ActorBehavior src, snk;
    src.host_fire = [rate](HostFiringContext& ctx) {
      auto* o = reinterpret_cast<std::int32_t*>(ctx.output(0).data());
      for (std::uint32_t t = 0; t < rate; ++t) o[t] = static_cast<std::int32_t>(ctx.firing_index() * rate + t);
    };
    snk.host_fire = [out_host, rate](HostFiringContext& ctx) {
      std::memcpy(out_host + ctx.firing_index() * rate, ctx.input(0).data(), 4ull * rate);
    };
    ActorBehavior dbl = bulk_kernel_adapter([bad](const std::vector<std::span<const std::byte>>& in) {
      const auto* x = reinterpret_cast<const std::int32_t*>(in[0].data());
      std::vector<std::byte> y(in[0].size() + (bad ? 4 : 0));
      for (std::size_t t = 0; t < in[0].size() / 4; ++t) {
        const std::int32_t v = 2 * x[t];
        std::memcpy(y.data() + 4 * t, &v, 4);
      }
      return std::vector<std::vector<std::byte>>{std::move(y)};
    });
    std::vector<ActorSpec> actors = {
        {"source", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "a"}}, src},
        {"doubler", ActorKind::static_rate,
         {{PortDirection::input, PortKind::regular, "a"}, {PortDirection::output, PortKind::regular, "b"}}, dbl},
        {"sink", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "b"}}, snk}};
    ExecutionConfig ec;
    ec.device = device;
    ec.source_firing_limit = firings;
    run(build_network(actors, chans), ec);
  });
}

// df::Channel (the reference's Channel API over a device channel): a host
// producer writes `firings` regions of rate uint32 tokens (values 1, 2, ...),
// a host consumer reads them back (a delay channel first yields its initial
// token 0xFFFFFFFF); after close() the next read_start is end of stream.
// out: firings * rate tokens read; status bits: 1 = end of stream seen,
// 2 = write_start with n != rate threw logic_error, 4 = tokens_written and
// tokens_read match, 8 = a read after abort() threw RunAborted.
int dfh_channel_class_demo(int device, uint32_t rate, int delay, uint32_t firings, uint32_t* out, int* status) {
  return guarded([&] {
    using namespace df;
    if (!out || !status) throw std::invalid_argument("dfh_channel_class_demo: null argument");
    *status = 0;
    std::vector<std::byte> init(4, std::byte{0xFF});
    Channel ch({"c", 4, rate, delay != 0, delay ? init : std::vector<std::byte>{}}, device);
    try {
      ch.write_start(rate + 1);
    } catch (const std::logic_error&) {
      *status |= 2;
    }
    std::vector<std::uint32_t> v(rate);
    std::uint32_t next = 1;
    for (std::uint32_t f = 0; f < firings; ++f) {
      RegionHandle w = ch.write_start(rate);
      for (auto& x : v) x = next++;
      check(df_memcpy_h2d(w.bytes.data(), v.data(), 4ull * rate, nullptr));
      ch.write_end(w);
      std::optional<RegionHandle> r = ch.read_start(rate);
      if (!r) throw std::logic_error("unexpected end of stream");
      check(df_memcpy_d2h(out + std::size_t(f) * rate, r->bytes.data(), 4ull * rate, nullptr));
      ch.read_end(*r);
    }
    check(df_stream_synchronize(nullptr));
    if (ch.tokens_written() == std::uint64_t(firings) * rate && ch.tokens_read() == std::uint64_t(firings) * rate)
      *status |= 4;
    ch.close();
    for (int k = 0; k < 4; ++k) {  // drain what is left (a rate-1 delay channel still holds one token)
      std::optional<RegionHandle> r = ch.read_start(rate);
      if (!r) {
        *status |= 1;
        break;
      }
      ch.read_end(*r);
    }
    ch.abort();
    try {
      ch.read_start(rate);
    } catch (const RunAborted&) {
      *status |= 8;
    }
    ch.check_device();
  });
}

int dfh_validate_demo(int which) {
  int n = -1;
  int rc = guarded([&] {
    using namespace df;
    auto noop = [](FiringContext&) {};
    std::vector<ActorSpec> actors;
    std::vector<ChannelSpec> chans;
    if (which == 0) {  // the GPU DPD network shape: valid
      static std::vector<std::complex<float>> io(64), taps(100);
      dpd::Params p;
      p.period = 16;
      p.samples = 64;
      p.batch = 2;
      p.taps = taps;
      p.schedule = {dpd::ConfigToken::first_n(1), dpd::ConfigToken::first_n(10)};
      p.allow_single_branch = true;
      p.input = io;
      p.output = io;
      n = (int)validate(dpd::build_network(p)).size();
      return;
    }
    if (which == 1) {  // undelayed cycle a -> b -> a, static actor with control port
      chans = {{"ab", 4, 1, false, {}}, {"ba", 4, 1, false, {}}, {"c", 4, 1, false, {}}};
      ActorBehavior b;
      b.fire = noop;
      actors.push_back({"a", ActorKind::static_rate,
                        {{PortDirection::output, PortKind::regular, "ab"},
                         {PortDirection::input, PortKind::regular, "ba"},
                         {PortDirection::output, PortKind::regular, "c"}},
                        b});
      actors.push_back({"b", ActorKind::static_rate,
                        {{PortDirection::input, PortKind::regular, "ab"},
                         {PortDirection::output, PortKind::regular, "ba"},
                         {PortDirection::input, PortKind::control, "c"}},
                        b});
      n = (int)validate(build_network(actors, chans)).size();
      return;
    }
    if (which == 2) {  // delayed self-loop: valid
      chans = {{"loop", 8, 1, true, {}}};
      ActorBehavior b;
      b.fire = noop;
      actors.push_back({"m", ActorKind::static_rate,
                        {{PortDirection::input, PortKind::regular, "loop"},
                         {PortDirection::output, PortKind::regular, "loop"}},
                        b});
      n = (int)validate(build_network(actors, chans)).size();
      return;
    }
    if (which == 4) {  // CPU actor rules: dynamic host actor, host + device fire on one actor
      chans = {{"c", 4, 1, false, {}}, {"d", 4, 1, false, {}}, {"e", 4, 1, false, {}}};
      ActorBehavior src;
      src.fire = noop;
      actors.push_back({"src", ActorKind::static_rate,
                        {{PortDirection::output, PortKind::regular, "c"},
                         {PortDirection::output, PortKind::regular, "d"}},
                        src});
      ActorBehavior dyn;
      dyn.host_fire = [](HostFiringContext&) {};
      dyn.device_control = true;
      actors.push_back({"dyn", ActorKind::dynamic_rate,
                        {{PortDirection::input, PortKind::control, "c"},
                         {PortDirection::input, PortKind::regular, "d"},
                         {PortDirection::output, PortKind::regular, "e"}},
                        dyn});
      ActorBehavior both;
      both.fire = noop;
      both.host_fire = [](HostFiringContext&) {};
      actors.push_back({"both", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "e"}}, both});
      n = (int)validate(build_network(actors, chans)).size();
      return;
    }
    if (which == 5 || which == 6) {  // cycles whose delay channels have rate 2: unrunnable
      ActorBehavior b;
      b.fire = noop;
      if (which == 5) {  // a -> b undelayed, b -> a delayed at rate 2
        chans = {{"ab", 4, 2, false, {}}, {"ba", 4, 2, true, {}}};
        actors.push_back({"a", ActorKind::static_rate,
                          {{PortDirection::output, PortKind::regular, "ab"},
                           {PortDirection::input, PortKind::regular, "ba"}},
                          b});
        actors.push_back({"b", ActorKind::static_rate,
                          {{PortDirection::input, PortKind::regular, "ab"},
                           {PortDirection::output, PortKind::regular, "ba"}},
                          b});
      } else {  // delayed self-loop at rate 2
        chans = {{"loop", 8, 2, true, {}}};
        actors.push_back({"m", ActorKind::static_rate,
                          {{PortDirection::input, PortKind::regular, "loop"},
                           {PortDirection::output, PortKind::regular, "loop"}},
                          b});
      }
      n = (int)validate(build_network(actors, chans)).size();
      return;
    }
    if (which == 7 || which == 8) {  // batched device_control actor: control rate 4
      // 7: its regular channels carry 4 tokens per firing too (one control
      // token per port token): valid.  8: its input carries 1: "control
      // rate must be 1" (model.cpp:133-134).
      const std::uint32_t in_rate = which == 7 ? 4 : 1;
      chans = {{"c", 4, 4, false, {}}, {"x", 16, in_rate, false, {}}, {"y", 16, 4, false, {}}};
      ActorBehavior src, dyn, snk;
      src.fire = noop;
      snk.fire = noop;
      dyn.fire = noop;
      dyn.device_control = true;
      actors.push_back({"src", ActorKind::static_rate,
                        {{PortDirection::output, PortKind::regular, "c"},
                         {PortDirection::output, PortKind::regular, "x"}},
                        src});
      actors.push_back({"dyn", ActorKind::dynamic_rate,
                        {{PortDirection::input, PortKind::control, "c"},
                         {PortDirection::input, PortKind::regular, "x"},
                         {PortDirection::output, PortKind::regular, "y"}},
                        dyn});
      actors.push_back({"snk", ActorKind::static_rate, {{PortDirection::input, PortKind::regular, "y"}}, snk});
      n = (int)validate(build_network(actors, chans)).size();
      return;
    }
    // which == 3: BuildError (unknown channel)
    ActorBehavior b;
    b.fire = noop;
    actors.push_back({"x", ActorKind::static_rate, {{PortDirection::output, PortKind::regular, "nope"}}, b});
    build_network(actors, chans);
  });
  return rc == 0 ? n : -1;
}


int dfh_synth(int what, uint64_t n, uint64_t seed, void* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("dfh_synth: null output");
    if (what == 0) {  // schedule: n uint16 masks
      const auto v = df::dpd::random_schedule(n, seed);
      for (std::size_t i = 0; i < v.size(); ++i) static_cast<uint16_t*>(out)[i] = v[i].active_mask;
    } else if (what == 1) {  // taps: 10 x n complex
      const auto v = df::dpd::random_taps(seed, static_cast<unsigned>(n));
      std::memcpy(out, v.data(), v.size() * sizeof(v[0]));
    } else if (what == 2) {  // n complex samples
      const auto v = df::dpd::synth_samples(n, seed);
      std::memcpy(out, v.data(), v.size() * sizeof(v[0]));
    } else if (what == 3) {  // n frame bytes (frames * W * H)
      const auto v = df::motion::synth_frames(n, 1, 1, seed);
      std::memcpy(out, v.data(), v.size());
    } else {
      throw std::invalid_argument("dfh_synth: unknown generator");
    }
  });
}

int dfh_encode_config(uint16_t mask, uint8_t* out4) {
  return guarded([&] {
    if (!out4) throw std::invalid_argument("dfh_encode_config: null argument");
    df::dpd::encode_config({mask}, std::span<std::byte>(reinterpret_cast<std::byte*>(out4), 4));
  });
}

int dfh_decode_config(const uint8_t* in4, uint16_t* mask) {
  return guarded([&] {
    if (!in4 || !mask) throw std::invalid_argument("dfh_decode_config: null argument");
    *mask = df::dpd::decode_config(std::span<const std::byte>(reinterpret_cast<const std::byte*>(in4), 4)).active_mask;
  });
}

int dfh_parse_schedule(const char* text, uint16_t* masks, size_t cap, size_t* count) {
  return guarded([&] {
    if (!text || !count) throw std::invalid_argument("dfh_parse_schedule: null argument");
    std::istringstream in(text);
    const auto sched = df::dpd::parse_schedule(in);
    *count = sched.size();
    if (masks) {
      if (cap < sched.size()) throw std::invalid_argument("dfh_parse_schedule: buffer too small");
      for (size_t i = 0; i < sched.size(); ++i) masks[i] = sched[i].active_mask;
    }
  });
}

int dfh_parse_taps(const char* text, uint32_t taps_per_branch, float* taps_out) {
  return guarded([&] {
    if (!text || !taps_out) throw std::invalid_argument("dfh_parse_taps: null argument");
    std::istringstream in(text);
    const auto taps = df::dpd::parse_taps(in, taps_per_branch);
    std::memcpy(taps_out, taps.data(), taps.size() * sizeof(std::complex<float>));
  });
}

int dfh_read_pgm(const char* path, uint8_t* pixels, size_t cap_bytes, unsigned* width, unsigned* height,
                 uint64_t* frames) {
  return guarded([&] {
    if (!path || !width || !height || !frames) throw std::invalid_argument("dfh_read_pgm: null argument");
    const auto s = df::io::read_pgm(path);
    *width = s.width;
    *height = s.height;
    *frames = s.frames;
    if (pixels) {
      if (cap_bytes < s.pixels.size()) throw std::invalid_argument("dfh_read_pgm: buffer too small");
      std::memcpy(pixels, s.pixels.data(), s.pixels.size());
    }
  });
}

int dfh_write_pgm(const char* path, const uint8_t* pixels, uint64_t frames, unsigned width, unsigned height) {
  return guarded([&] {
    if (!path || !pixels) throw std::invalid_argument("dfh_write_pgm: null argument");
    df::io::write_pgm(path, pixels, frames, width, height);
  });
}

int dfh_read_raw_frames(const char* path, unsigned width, unsigned height, int input_format, uint8_t* pixels,
                        size_t cap_bytes, uint64_t* frames) {
  return guarded([&] {
    if (!path || !frames) throw std::invalid_argument("dfh_read_raw_frames: null argument");
    const auto px = df::io::read_raw_frames(path, width, height, static_cast<unsigned>(input_format), frames);
    if (pixels) {
      if (cap_bytes < px.size()) throw std::invalid_argument("dfh_read_raw_frames: buffer too small");
      std::memcpy(pixels, px.data(), px.size());
    }
  });
}

int dfh_read_cf32(const char* path, float* samples_out, size_t cap_samples, uint64_t* samples) {
  return guarded([&] {
    if (!path || !samples) throw std::invalid_argument("dfh_read_cf32: null argument");
    const auto s = df::io::read_cf32(path);
    *samples = s.size();
    if (samples_out) {
      if (cap_samples < s.size()) throw std::invalid_argument("dfh_read_cf32: buffer too small");
      std::memcpy(samples_out, s.data(), s.size() * sizeof(std::complex<float>));
    }
  });
}

int dfh_write_file(const char* path, const void* data, size_t size) {
  return guarded([&] {
    if (!path || (!data && size)) throw std::invalid_argument("dfh_write_file: null argument");
    df::io::write_file(path, data, size);
  });
}

}  // extern "C"
