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
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <sstream>

#include "df_cuda.h"
#include "nvtx3/nvToolsExt.h"  // header-only NVTX v3: ranges per firing / run (no-ops without a tool)

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
  // CPU actors: pinned host copies of the firing's regions, one per
  // regular port (token_size * rate bytes).  Firings of one actor are
  // serialised on its stream, so one copy per port suffices.
  std::vector<std::byte*> stage_in, stage_out;
  std::vector<std::size_t> bytes_in, bytes_out, tokens_in, tokens_out, tsize_in, tsize_out;
  // Dynamic CPU actors: the actor's index, its control token's host copy,
  // and regular port k (declaration order) -> (is input, index).
  std::size_t index = 0;
  std::byte* stage_ctrl = nullptr;
  std::size_t ctrl_bytes = 0;
  std::vector<std::pair<bool, std::size_t>> regular_ports;
};

// Fault raised inside a CPU actor's host_fire (which runs on a CUDA
// callback thread): recorded once, rethrown as ActorFault after the run;
// later host firings are skipped (the reference aborts the run,
// runtime.cpp:232-247).
struct HostFaults {
  std::atomic<bool> failed{false};
  std::mutex mu;
  std::string actor, what;
};

struct HostJob {
  HostFaults* faults;
  const ActorRun* run;
  std::uint64_t firing;
  // This firing's tokens per port (0 on a dynamic actor's gated ports).
  std::vector<std::size_t> tokens_in, tokens_out;
};

void host_job_entry(void* p) {
  const HostJob& job = *static_cast<const HostJob*>(p);
  if (job.faults->failed.load()) return;
  const ActorRun& r = *job.run;
  try {
    std::vector<std::span<const std::byte>> in;
    std::vector<std::span<std::byte>> out;
    for (std::size_t k = 0; k < r.stage_in.size(); ++k) in.emplace_back(r.stage_in[k], job.tokens_in[k] * r.tsize_in[k]);
    for (std::size_t k = 0; k < r.stage_out.size(); ++k)
      out.emplace_back(r.stage_out[k], job.tokens_out[k] * r.tsize_out[k]);
    HostFiringContext ctx;
    ctx.bind(std::move(in), job.tokens_in, r.tsize_in, std::move(out), job.tokens_out, r.tsize_out, job.firing);
    r.spec->behavior.host_fire(ctx);
  } catch (const std::exception& e) {
    std::lock_guard<std::mutex> lock(job.faults->mu);
    if (!job.faults->failed.exchange(true)) {
      job.faults->actor = r.spec->id;
      job.faults->what = e.what();
    }
  } catch (...) {
    std::lock_guard<std::mutex> lock(job.faults->mu);
    if (!job.faults->failed.exchange(true)) {
      job.faults->actor = r.spec->id;
      job.faults->what = "unknown exception";
    }
  }
}

// One firing of a CPU actor, all in its stream: inputs' regions D2H, the
// host function, outputs' regions H2D, then the channel commits.  A dynamic
// CPU actor first reads its control token: the token's D2H copy is waited
// for on the host (one stream synchronisation per firing -- the reference's
// actor thread blocks on its control channel the same way,
// runtime.cpp:139-145), control_dispatch turns it into 0-or-r rates
// (ControlError -> ActorFault), and only the active ports' regions move and
// commit.  The host mirror of each endpoint's phase advances with its own
// commits only, so it stays exact.
void fire_host_actor(const NetworkGraph& net, ActorRun& r, std::uint64_t firing, HostFaults& faults,
                     std::deque<HostJob>& jobs) {
  const std::size_t nin = r.ctx.input_count(), nout = r.ctx.output_count();
  std::vector<std::size_t> tin = r.tokens_in, tout = r.tokens_out;
  df_region rc{};
  if (r.ctx.control()) {
    check(df_channel_read_start(r.ctx.control(), 1, &rc));
    check(df_memcpy_d2h(r.stage_ctrl, rc.dptr, r.ctrl_bytes, r.stream));
    check(df_stream_synchronize(r.stream));
    const FiringRates rates =
        control_dispatch(net, r.index, std::span<const std::byte>(r.stage_ctrl, r.ctrl_bytes));
    for (std::size_t k = 0; k < r.regular_ports.size(); ++k) {
      const auto [is_in, idx] = r.regular_ports[k];
      (is_in ? tin : tout)[idx] = rates.by_regular_port[k];
    }
  }
  std::vector<df_region> rin(nin), rout(nout);
  for (std::size_t k = 0; k < nin; ++k) {
    if (!tin[k]) continue;
    check(df_channel_read_start(r.ctx.input(k), tin[k], &rin[k]));
    check(df_memcpy_d2h(r.stage_in[k], rin[k].dptr, r.bytes_in[k], r.stream));
  }
  for (std::size_t k = 0; k < nout; ++k)
    if (tout[k]) check(df_channel_write_start(r.ctx.output(k), tout[k], &rout[k]));
  jobs.push_back({&faults, &r, firing, tin, tout});
  check(df_launch_host_func(r.stream, host_job_entry, &jobs.back()));
  for (std::size_t k = 0; k < nout; ++k) {
    if (!tout[k]) continue;
    check(df_memcpy_h2d(rout[k].dptr, r.stage_out[k], r.bytes_out[k], r.stream));
    check(df_channel_write_end(r.ctx.output(k), &rout[k], r.stream));
  }
  for (std::size_t k = 0; k < nin; ++k)
    if (tin[k]) check(df_channel_read_end(r.ctx.input(k), &rin[k], r.stream));
  if (r.ctx.control()) check(df_channel_read_end(r.ctx.control(), &rc, r.stream));
}

// Device-resident run: every actor fires inside one persistent kernel
// (df_net, csrc/netrt.cu).  The host builds the channels, registers each
// actor with its kind, ports and firing limit, turns each dynamic actor's
// `control` into a device table (control_dispatch per token value), runs
// the kernel to completion and maps a device fault back to ActorFault.
RunStats run_device(const NetworkGraph& net, const ExecutionConfig& cfg, std::chrono::steady_clock::time_point t0) {
  check(df_set_device(cfg.device));
  std::vector<df_channel*> chans(net.channels().size(), nullptr);
  df_net* dn = nullptr;
  auto cleanup = [&]() {
    df_net_destroy(dn);
    for (df_channel* c : chans) df_channel_destroy(c);
  };
  // control_dispatch failures per (actor, token value), for the fault text.
  std::vector<std::vector<std::string>> control_errors(net.actors().size());
  RunStats stats;
  try {
    for (std::size_t c = 0; c < chans.size(); ++c) {
      const ChannelSpec& s = net.channels()[c];
      check(df_channel_create(cfg.device, s.token_size, s.token_rate, s.has_delay,
                              s.initial_token_value.empty() ? nullptr : s.initial_token_value.data(), &chans[c]));
    }
    check(df_net_create(cfg.device, &dn));
    for (std::size_t a = 0; a < net.actors().size(); ++a) {
      const ActorSpec& spec = net.actors()[a];
      std::vector<df_channel*> in, out;
      std::vector<std::pair<bool, std::uint32_t>> slot;  // regular port k -> (is input, bit)
      df_channel* ctrl = nullptr;
      for (const PortSpec& port : spec.ports) {
        df_channel* ch = chans[net.channel_index(port.channel_id)];
        if (port.kind == PortKind::control) {
          ctrl = ch;
        } else if (port.direction == PortDirection::input) {
          slot.push_back({true, static_cast<std::uint32_t>(in.size())});
          in.push_back(ch);
        } else {
          slot.push_back({false, static_cast<std::uint32_t>(out.size())});
          out.push_back(ch);
        }
      }
      std::uint64_t limit = 0;
      if (in.empty() && !ctrl) {  // a source (runtime.cpp:105-107: no input, no control port)
        if (!cfg.source_firing_limit)
          throw std::invalid_argument("device-resident source '" + spec.id + "' needs a source_firing_limit");
        limit = *cfg.source_firing_limit;
        if (limit == 0) limit = ~std::uint64_t(0) >> 1;  // fires never; closes at once
      }
      const DeviceActor& d = spec.behavior.device;
      int index = -1;
      check(df_net_add_actor(dn, d.kind, d.params.empty() ? nullptr : d.params.data(), d.params.size(), d.ctas, ctrl,
                             in.data(), in.size(), out.data(), out.size(), limit, &index));
      if (ctrl) {
        const std::size_t tsize = df_channel_token_size(ctrl);
        std::uint64_t domain = spec.behavior.control_domain;
        if (tsize < 4) domain = std::min<std::uint64_t>(domain, std::uint64_t(1) << (8 * tsize));
        std::vector<std::uint32_t> rows(3 * domain, 0);
        control_errors[a].assign(domain, {});
        std::vector<std::byte> token(tsize, std::byte{0});
        for (std::uint64_t v = 0; v < domain; ++v) {
          for (std::size_t b = 0; b < tsize && b < 4; ++b) token[b] = static_cast<std::byte>((v >> (8 * b)) & 0xFF);
          try {
            const FiringRates r = control_dispatch(net, a, token);
            for (std::size_t k = 0; k < slot.size(); ++k)
              if (r.by_regular_port[k]) rows[3 * v + (slot[k].first ? 0 : 1)] |= 1u << slot[k].second;
            rows[3 * v + 2] = 1;
          } catch (const std::exception& e) {
            control_errors[a][v] = e.what();
          }
        }
        check(df_net_set_control_table(dn, index, rows.data(), static_cast<std::uint32_t>(domain)));
      }
    }
  } catch (...) {
    cleanup();
    throw;
  }
  std::string fault_actor;
  try {
    for (const ActorSpec& spec : net.actors()) {
      fault_actor = spec.id;
      if (spec.behavior.init) spec.behavior.init();
    }
    fault_actor.clear();
    nvtxRangePushA("df_net_run (device-resident network)");
    const int rc = df_net_run(dn, cfg.device_timeout_s);
    nvtxRangePop();
    if (rc != DF_OK) {
      const std::string detail = df_last_error();
      int who = -1, code = 0;
      std::uint32_t token = 0;
      df_net_fault(dn, &who, &code, &token);
      if (rc == DF_EABORTED || who < 0) throw_status(rc);
      fault_actor = net.actors()[who].id;
      if (code == DF_ECONTROL) {
        const auto& errs = control_errors[who];
        throw ControlError(token < errs.size() && !errs[token].empty()
                               ? errs[token]
                               : "actor '" + fault_actor + "': control token " + std::to_string(token) +
                                     " is outside the control domain");
      }
      throw std::runtime_error(detail);
    }
    for (const ActorSpec& spec : net.actors()) {
      fault_actor = spec.id;
      if (spec.behavior.finish) spec.behavior.finish();
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
  const bool profile = std::getenv("DF_NET_PROFILE") != nullptr;
  for (std::size_t a = 0; a < net.actors().size(); ++a) {
    std::uint64_t firings = 0;
    double ms = 0.0;
    df_net_actor_stats(dn, static_cast<int>(a), &firings, &ms);
    stats.actors.push_back({net.actors()[a].id, firings, ms});
    if (profile) {  // tracing aid: where each actor's leader spent its time
      double w = 0, f = 0, c = 0;
      df_net_actor_profile(dn, static_cast<int>(a), &w, &f, &c);
      std::fprintf(stderr, "df_net %-10s firings %8llu active %9.3f ms  wait %9.3f  fire %9.3f  commit %9.3f ms\n",
                   net.actors()[a].id.c_str(), (unsigned long long)firings, ms, w, f, c);
    }
  }
  if (cfg.stats_enabled)
    for (std::size_t c = 0; c < chans.size(); ++c) {
      df_chan_stats st{};
      if (df_channel_stats(chans[c], &st) == DF_OK)
        stats.channels.push_back({net.channels()[c].id, st.tokens_written, st.tokens_read, st.tokens_available});
    }
  cleanup();
  stats.wall = std::chrono::steady_clock::now() - t0;
  return stats;
}

}  // namespace

ActorBehavior bulk_kernel_adapter(BatchKernel kernel) {
  ActorBehavior behavior;
  behavior.host_fire = [kernel = std::move(kernel)](HostFiringContext& ctx) {
    std::vector<std::span<const std::byte>> inputs;
    for (std::size_t i = 0; i < ctx.input_count(); ++i) inputs.push_back(ctx.input(i));
    const std::vector<std::vector<std::byte>> produced = kernel(inputs);
    if (produced.size() != ctx.output_count())
      throw std::runtime_error("bulk kernel produced " + std::to_string(produced.size()) + " arrays for " +
                               std::to_string(ctx.output_count()) + " ports");
    for (std::size_t o = 0; o < produced.size(); ++o) {
      const std::span<std::byte> region = ctx.output(o);
      if (produced[o].size() != region.size())
        throw std::runtime_error("bulk kernel output " + std::to_string(o) + " is " +
                                 std::to_string(produced[o].size()) + " bytes, region is " +
                                 std::to_string(region.size()));
      std::memcpy(region.data(), produced[o].data(), region.size());
    }
  };
  return behavior;
}

RunStats run(const NetworkGraph& net, const ExecutionConfig& cfg) {
  std::vector<Violation> violations = validate(net);
  if (!violations.empty()) {
    std::ostringstream msg;
    msg << "network failed validation:";
    for (const Violation& v : violations) msg << "\n  " << v.subject << ": " << v.message;
    throw ValidationError(msg.str(), std::move(violations));
  }
  const auto t0 = std::chrono::steady_clock::now();
  if (!net.actors().empty() && net.actors().front().behavior.is_device_resident()) return run_device(net, cfg, t0);
  check(df_set_device(cfg.device));

  // Device channels (Eq. 1 storage + control block in HBM).
  std::vector<df_channel*> chans(net.channels().size(), nullptr);
  std::vector<ActorRun> runs(net.actors().size());
  auto cleanup = [&]() {
    for (ActorRun& r : runs) {
      if (r.stream) df_stream_synchronize(r.stream);  // host callbacks may still reference the stages
      for (std::byte* b : r.stage_in) df_host_free(b);
      for (std::byte* b : r.stage_out) df_host_free(b);
      if (r.stage_ctrl) df_host_free(r.stage_ctrl);
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
      if (r.spec->behavior.is_host()) {
        auto stage = [&](df_channel* ch, std::vector<std::byte*>& bufs, std::vector<std::size_t>& bytes,
                         std::vector<std::size_t>& tokens, std::vector<std::size_t>& tsize) {
          const std::size_t n = df_channel_token_rate(ch), b = n * df_channel_token_size(ch);
          void* h = nullptr;
          check(df_host_alloc(b, &h));
          bufs.push_back(static_cast<std::byte*>(h));
          bytes.push_back(b);
          tokens.push_back(n);
          tsize.push_back(df_channel_token_size(ch));
        };
        for (df_channel* ch : in) stage(ch, r.stage_in, r.bytes_in, r.tokens_in, r.tsize_in);
        for (df_channel* ch : out) stage(ch, r.stage_out, r.bytes_out, r.tokens_out, r.tsize_out);
        r.index = a;
        if (ctrl) {  // dynamic CPU actor: its control token's host copy
          r.ctrl_bytes = df_channel_token_size(ctrl);
          void* h = nullptr;
          check(df_host_alloc(r.ctrl_bytes, &h));
          r.stage_ctrl = static_cast<std::byte*>(h);
          std::size_t ni = 0, no = 0;
          for (const PortSpec& port : r.spec->ports)
            if (port.kind == PortKind::regular)
              r.regular_ports.push_back(port.direction == PortDirection::input ? std::make_pair(true, ni++)
                                                                               : std::make_pair(false, no++));
        }
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

  // validate() rejected every cycle of same-firing channels.
  const std::vector<std::size_t> order = firing_order(net).value();
  const std::uint64_t limit = cfg.source_firing_limit.value_or(0);
  std::string fault_actor;
  HostFaults host_faults;
  std::deque<HostJob> host_jobs;  // alive until every stream has drained
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
        nvtxRangePushA(r.spec->id.c_str());  // the enqueue of firing i (host timeline)
        if (r.spec->behavior.is_host())
          fire_host_actor(net, r, i, host_faults, host_jobs);
        else
          r.spec->behavior.fire(r.ctx);
        nvtxRangePop();
        fault_actor.clear();
        check(df_event_record(r.done[i % 3], r.stream));
        ++r.firings;
      }
    }
    for (ActorRun& r : runs) {
      check(df_event_record(r.t_last, r.stream));
      check(df_stream_synchronize(r.stream));
    }
    if (host_faults.failed.load()) {
      fault_actor = host_faults.actor;
      throw std::runtime_error(host_faults.what);
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
