// runtime.cpp -- static-schedule executor for GPU-actor networks.
//
// Reference: Run::execute / fire_once / actor_main
// (/root/reference/proj/src/runtime.cpp:132-299): thread per actor,
// blocking channels, control token read on the host.  Here (see
// df/runtime.hpp): one issuing thread, one CUDA stream per actor, the
// channel protocol as event dependencies, control tokens and token counts
// on the device.  Nothing synchronizes until the run ends.
#include "df/runtime.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <sstream>

#include "df_cuda.h"

namespace df {

void throw_status(int status) {
  const std::string msg = df_last_error();
  switch (status) {
    case DF_EINVAL:
      throw std::invalid_argument(msg);
    case DF_ELOGIC:
      throw std::logic_error(msg);
    case DF_EABORTED:
      throw RunAborted();
    case DF_ECONTROL:
      throw ControlError(msg);
    default:
      throw std::runtime_error("df_cuda error " + std::to_string(status) + ": " + msg);
  }
}

const RunStats::ActorStats& RunStats::actor(const std::string& id) const {
  for (const ActorStats& a : actors)
    if (a.id == id) return a;
  throw std::out_of_range("no stats for actor '" + id + "'");
}

namespace {

struct Dep {
  std::size_t actor;
  int lag;  // wait for firing (i - lag) of `actor`
};

struct ActorRun {
  const ActorSpec* spec = nullptr;
  void* stream = nullptr;
  void* done[3] = {nullptr, nullptr, nullptr};  // firing i -> done[i % 3]
  void* t_first = nullptr;
  void* t_last = nullptr;
  std::vector<Dep> deps;
  FiringContext ctx;
  std::uint64_t firings = 0;
};

// Topological order over undelayed channels (validate() rejected cycles).
std::vector<std::size_t> topo_order(const NetworkGraph& net) {
  const std::size_t n = net.actors().size();
  std::vector<int> indeg(n, 0);
  std::vector<std::vector<std::size_t>> next(n);
  for (std::size_t c = 0; c < net.channels().size(); ++c) {
    if (net.channels()[c].has_delay) continue;
    const auto& ep = net.endpoints()[c];
    if (ep.producer_actor == ep.consumer_actor) continue;
    next[ep.producer_actor].push_back(ep.consumer_actor);
    ++indeg[ep.consumer_actor];
  }
  std::vector<std::size_t> order, ready;
  for (std::size_t a = 0; a < n; ++a)
    if (indeg[a] == 0) ready.push_back(a);
  while (!ready.empty()) {
    std::size_t a = ready.front();
    ready.erase(ready.begin());
    order.push_back(a);
    for (std::size_t b : next[a])
      if (--indeg[b] == 0) ready.push_back(b);
  }
  return order;
}

}  // namespace

RunStats run(const NetworkGraph& net, const ExecutionConfig& cfg) {
  std::vector<Violation> violations = validate(net);
  if (!violations.empty()) {
    std::ostringstream msg;
    msg << "network failed validation:";
    for (const Violation& v : violations) msg << "\n  " << v.subject << ": " << v.message;
    throw ValidationError(msg.str(), std::move(violations));
  }
  const auto t0 = std::chrono::steady_clock::now();
  check(df_set_device(cfg.device));

  // Device channels (Eq. 1 storage + control block in HBM).
  std::vector<df_channel*> chans(net.channels().size(), nullptr);
  std::vector<ActorRun> runs(net.actors().size());
  auto cleanup = [&]() {
    for (ActorRun& r : runs) {
      for (void*& e : r.done)
        if (e) df_event_destroy(e);
      if (r.t_first) df_event_destroy(r.t_first);
      if (r.t_last) df_event_destroy(r.t_last);
      if (r.stream) df_stream_destroy(r.stream);
    }
    for (df_channel* c : chans) df_channel_destroy(c);
  };
  RunStats stats;
  try {
    for (std::size_t c = 0; c < chans.size(); ++c) {
      const ChannelSpec& s = net.channels()[c];
      check(df_channel_create(cfg.device, s.token_size, s.token_rate, s.has_delay,
                              s.initial_token_value.empty() ? nullptr : s.initial_token_value.data(), &chans[c]));
    }
    // Per-actor streams, events and port bindings.
    for (std::size_t a = 0; a < runs.size(); ++a) {
      ActorRun& r = runs[a];
      r.spec = &net.actors()[a];
      check(df_stream_create(cfg.device, &r.stream));
      for (void*& e : r.done) check(df_event_create(&e));
      check(df_event_create(&r.t_first));
      check(df_event_create(&r.t_last));
      std::vector<df_channel*> in, out;
      df_channel* ctrl = nullptr;
      for (std::size_t p = 0; p < r.spec->ports.size(); ++p) {
        const PortSpec& port = r.spec->ports[p];
        const std::size_t c = net.channel_index(port.channel_id);
        if (port.kind == PortKind::control)
          ctrl = chans[c];
        else if (port.direction == PortDirection::input)
          in.push_back(chans[c]);
        else
          out.push_back(chans[c]);
      }
      r.ctx.bind(std::move(in), std::move(out), ctrl);
    }
    // Dependencies encoding the channel protocol (see df/runtime.hpp).
    for (std::size_t c = 0; c < chans.size(); ++c) {
      const ChannelSpec& s = net.channels()[c];
      const auto& ep = net.endpoints()[c];
      const std::size_t p = ep.producer_actor, q = ep.consumer_actor;
      if (p == q) continue;  // self-loop: ordered by the actor's own stream
      // data: a rate-1 delay token shifts the stream by one whole firing
      runs[q].deps.push_back({p, (s.has_delay && s.token_rate == 1) ? 1 : 0});
      // capacity: the write region of firing i was read by firing i-2
      runs[p].deps.push_back({q, 2});
    }
  } catch (...) {
    cleanup();
    throw;
  }

  const std::vector<std::size_t> order = topo_order(net);
  const std::uint64_t limit = cfg.source_firing_limit.value_or(0);
  std::string fault_actor;
  try {
    for (ActorRun& r : runs) {
      fault_actor = r.spec->id;
      if (r.spec->behavior.init) r.spec->behavior.init();
    }
    fault_actor.clear();
    for (std::uint64_t i = 0; i < limit; ++i) {
      for (std::size_t a : order) {
        ActorRun& r = runs[a];
        for (const Dep& d : r.deps) {
          if (i < (std::uint64_t)d.lag) continue;
          check(df_stream_wait_event(r.stream, runs[d.actor].done[(i - d.lag) % 3]));
        }
        if (i == 0) check(df_event_record(r.t_first, r.stream));
        r.ctx.reset(i, r.stream, cfg.device);
        fault_actor = r.spec->id;
        r.spec->behavior.fire(r.ctx);
        fault_actor.clear();
        check(df_event_record(r.done[i % 3], r.stream));
        ++r.firings;
      }
    }
    for (ActorRun& r : runs) {
      check(df_event_record(r.t_last, r.stream));
      check(df_stream_synchronize(r.stream));
    }
    for (ActorRun& r : runs) {
      fault_actor = r.spec->id;
      if (r.spec->behavior.finish) r.spec->behavior.finish();
    }
    fault_actor.clear();
  } catch (const RunAborted&) {
    cleanup();
    throw;
  } catch (const std::exception& e) {
    const std::string who = fault_actor;
    cleanup();
    if (!who.empty()) throw ActorFault(who, e.what());
    throw;
  }

  // Device-side contract violations (sticky per-channel error words).
  for (std::size_t c = 0; c < chans.size(); ++c) {
    df_chan_stats st{};
    if (df_channel_stats(chans[c], &st) != DF_OK) continue;
    if (st.error) {
      const auto& ep = net.endpoints()[c];
      const std::string who = net.actors()[ep.consumer_actor].id;
      const std::string what = "channel '" + net.channels()[c].id + "': device-side token count violation (code " +
                               std::to_string(st.error) + ")";
      cleanup();
      throw ActorFault(who, what);
    }
    if (cfg.stats_enabled)
      stats.channels.push_back({net.channels()[c].id, st.tokens_written, st.tokens_read, st.tokens_available});
  }
  for (ActorRun& r : runs) {
    float ms = 0.0f;
    if (r.firings) df_event_elapsed_ms(r.t_first, r.t_last, &ms);
    stats.actors.push_back({r.spec->id, r.firings, ms});
  }
  cleanup();
  stats.wall = std::chrono::steady_clock::now() - t0;
  return stats;
}

}  // namespace df
