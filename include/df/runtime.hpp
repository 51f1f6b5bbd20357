// df/runtime.hpp -- executes a network of GPU actors over device channels.
//
// Reference: dynflow::run (/root/reference/proj/src/runtime.cpp:250-332),
// which runs one OS thread per actor that blocks on mutex/condvar
// channels.  On the B200 there is nothing to block on the host: every
// actor owns a CUDA stream and a firing is an asynchronous enqueue.  The
// model's firing counts are data-independent (one control token per
// firing of a dynamic actor), so the runtime issues a static schedule --
// firing i of every actor in topological order -- and encodes the channel
// protocol as stream/event dependencies:
//   * data:      consumer firing i waits for the producer's firing i;
//   * capacity:  producer firing i waits for the consumer's firing i - 2,
//                for both layouts.  Regular channels alternate two halves, so
//                write i reuses the half read i-2 released.  A delay channel
//                (3r+1 slots) write i overlaps the region read i-2 held as
//                well: reads start one slot lower than writes, and the phase-2
//                copy into slot 0 overwrites the first slot of read phase 0.
//                Lag 3 would race; lag 2 is the correct bound for both.
// while token COUNTS (0 or r per port for dynamic actors) and region
// addresses live on the device (df_channel).  The host synchronizes once,
// at the end.  Device-side contract violations (token underflow/overflow,
// control tokens naming a branch beyond 10) surface as ActorFault.
#pragma once

#include <functional>
#include <chrono>
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "df/model.hpp"

namespace df {

// runtime.hpp:22-27 (mapping/pins are CPU-thread notions and do not apply).
struct ExecutionConfig {
  int device = 0;
  std::optional<std::uint64_t> source_firing_limit;
  bool stats_enabled = true;
  // Device-resident runs: the watchdog for any single channel wait (a
  // deadlocked network ends in ActorFault instead of hanging the GPU).
  double device_timeout_s = 30.0;
};

struct RunStats {
  struct ActorStats {
    std::string id;
    std::uint64_t firings = 0;
    double active_ms = 0.0;  // device time from first firing start to last firing end
  };
  struct ChannelStats {
    std::string id;
    std::uint64_t tokens_written = 0;
    std::uint64_t tokens_read = 0;
    std::uint64_t tokens_residual = 0;
  };
  std::vector<ActorStats> actors;
  std::vector<ChannelStats> channels;
  std::chrono::nanoseconds wall{0};
  std::vector<std::string> warnings;

  const ActorStats& actor(const std::string& id) const;
  std::uint64_t firings(const std::string& id) const { return actor(id).firings; }
  double active_seconds(const std::string& id) const { return actor(id).active_ms / 1e3; }
};

class ActorFault : public std::runtime_error {
 public:
  ActorFault(std::string actor_id, const std::string& what)
      : std::runtime_error("actor '" + actor_id + "' faulted: " + what), actor_id_(std::move(actor_id)) {}
  const std::string& actor_id() const { return actor_id_; }

 private:
  std::string actor_id_;
};

class ValidationError : public std::runtime_error {
 public:
  ValidationError(std::string what, std::vector<Violation> v)
      : std::runtime_error(std::move(what)), violations_(std::move(v)) {}
  const std::vector<Violation>& violations() const { return violations_; }

 private:
  std::vector<Violation> violations_;
};

class RunAborted : public std::runtime_error {
 public:
  RunAborted() : std::runtime_error("run aborted") {}
};

// Validates, creates the device channels and runs init, then either
//   * (device-resident actors) runs the network as one persistent kernel:
//     sources fire source_firing_limit times, every other actor until end
//     of stream, with dynamic rates dispatched on the device per firing --
//     the reference's run() semantics; or
//   * (host-issued actors) issues source_firing_limit firings of every actor
//     as a static schedule (the actors fire in lock step), synchronizes;
// then runs finish, checks device-side errors and returns the stats.
RunStats run(const NetworkGraph& net, const ExecutionConfig& cfg);

// runtime.hpp:97-108: a batch function mirroring a kernel invocation -- one
// contiguous input array per regular input port, one produced array per
// regular output port -- wrapped as a CPU actor (host_fire) that hands it
// whole r-token regions.  Wrong output count or size faults the actor.
using BatchKernel =
    std::function<std::vector<std::vector<std::byte>>(const std::vector<std::span<const std::byte>>&)>;
ActorBehavior bulk_kernel_adapter(BatchKernel kernel);

// Throws the C++ exception matching a df_* status (DF_EINVAL ->
// std::invalid_argument, DF_ELOGIC -> std::logic_error, DF_EABORTED ->
// RunAborted, DF_ECONTROL -> ControlError, DF_ECUDA -> std::runtime_error).
void throw_status(int status);
inline void check(int status) {
  if (status != 0) throw_status(status);
}

}  // namespace df
