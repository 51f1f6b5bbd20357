// df/model.hpp -- actor/port/channel model of the B200 GPU-actor runtime.
//
// Same vocabulary and rules as the reference's dynflow model
// (/root/reference/proj/include/dynflow/model.hpp:14-193): ChannelSpec,
// PortSpec, ActorSpec, ActorBehavior, FiringRates, build_network,
// validate, control_dispatch.  What changes for GPU actors: channel storage
// lives in HBM (df_channel) and control tokens are consumed on the device.
// Two kinds of GPU actor exist:
//   * device-resident actors (ActorBehavior::device): the actor fires inside
//     the network's persistent kernel (df_net); a dynamic one keeps the
//     reference's `control` function, which the runtime evaluates once per
//     possible token value into a device table, so control_dispatch happens
//     on the device per firing (0 or r per port, ControlError otherwise);
//   * host-issued actors (ActorBehavior::fire): each firing enqueues device
//     work on the actor's stream; a dynamic one (`device_control`) consumes
//     its control tokens inside its own kernels (the fused DPD actor).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <functional>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

struct df_channel;

namespace df {

enum class PortDirection { input, output };
enum class PortKind { regular, control };
enum class ActorKind { static_rate, dynamic_rate };

// model.hpp:21-25
struct PortSpec {
  PortDirection direction = PortDirection::input;
  PortKind kind = PortKind::regular;
  std::string channel_id;
};

// model.hpp:31-37 -- token_rate tokens per firing on both endpoints;
// has_delay: one initial token (initial_token_value or zeros).
struct ChannelSpec {
  std::string id;
  std::size_t token_size = 1;
  std::uint32_t token_rate = 1;
  bool has_delay = false;
  std::vector<std::byte> initial_token_value;
};

// Per-firing view handed to a GPU actor's fire function: the device
// channels bound to its ports (declaration order, regular ports only, the
// control channel separately) and the CUDA stream to enqueue on.  Region
// addresses and (for dynamic actors) token counts are resolved by the
// device; the host never dereferences channel storage.
class FiringContext {
 public:
  std::size_t input_count() const { return inputs_.size(); }
  std::size_t output_count() const { return outputs_.size(); }
  df_channel* input(std::size_t i) const { return inputs_.at(i); }
  df_channel* output(std::size_t i) const { return outputs_.at(i); }
  df_channel* control() const { return control_; }
  void* stream() const { return stream_; }
  int device() const { return device_; }
  std::uint64_t firing_index() const { return firing_index_; }

  // Assembled by the runtime.
  void reset(std::uint64_t firing, void* stream, int device) {
    firing_index_ = firing;
    stream_ = stream;
    device_ = device;
  }
  void bind(std::vector<df_channel*> in, std::vector<df_channel*> out, df_channel* ctrl) {
    inputs_ = std::move(in);
    outputs_ = std::move(out);
    control_ = ctrl;
  }

 private:
  std::vector<df_channel*> inputs_, outputs_;
  df_channel* control_ = nullptr;
  void* stream_ = nullptr;
  int device_ = 0;
  std::uint64_t firing_index_ = 0;
};

// Per-firing view handed to a CPU (host) actor: the reference's
// FiringContext (model.hpp:43-83) -- byte spans over the firing's input and
// output regions, regular ports in declaration order, tokens per port and
// the firing index.  The spans are pinned host copies: the runtime moves the
// input regions device -> host before the firing and the output regions
// host -> device after it, in the actor's stream order, so CPU and GPU
// actors share the same device channels (the paper's heterogeneous
// mapping).
class HostFiringContext {
 public:
  std::size_t input_count() const { return inputs_.size(); }
  std::size_t output_count() const { return outputs_.size(); }
  std::span<const std::byte> input(std::size_t i) const { return inputs_.at(i); }
  std::span<std::byte> output(std::size_t i) const { return outputs_.at(i); }
  std::size_t input_tokens(std::size_t i) const { return in_tokens_.at(i); }
  std::size_t output_tokens(std::size_t i) const { return out_tokens_.at(i); }
  std::size_t input_token_size(std::size_t i) const { return in_token_size_.at(i); }
  std::size_t output_token_size(std::size_t i) const { return out_token_size_.at(i); }
  std::uint64_t firing_index() const { return firing_index_; }

  // Assembled by the runtime.  A dynamic CPU actor's gated port (rate 0
  // this firing) has 0 tokens and an empty span.
  void bind(std::vector<std::span<const std::byte>> in, std::vector<std::size_t> in_tokens,
            std::vector<std::size_t> in_token_size, std::vector<std::span<std::byte>> out,
            std::vector<std::size_t> out_tokens, std::vector<std::size_t> out_token_size, std::uint64_t firing) {
    inputs_ = std::move(in);
    in_tokens_ = std::move(in_tokens);
    in_token_size_ = std::move(in_token_size);
    outputs_ = std::move(out);
    out_tokens_ = std::move(out_tokens);
    out_token_size_ = std::move(out_token_size);
    firing_index_ = firing;
  }

 private:
  std::vector<std::span<const std::byte>> inputs_;
  std::vector<std::span<std::byte>> outputs_;
  std::vector<std::size_t> in_tokens_, out_tokens_, in_token_size_, out_token_size_;
  std::uint64_t firing_index_ = 0;
};

// model.hpp:89-97: rates of one firing of a dynamic actor, one entry per
// regular port in declaration order, each 0 or the channel's rate.
struct FiringRates {
  std::vector<std::uint32_t> by_regular_port;
  static FiringRates uniform(std::size_t port_count, std::uint32_t rate) {
    FiringRates r;
    r.by_regular_port.assign(port_count, rate);
    return r;
  }
};

// An actor that fires inside the device-resident network kernel: one of
// the library's device actor kinds (DF_ACT_* in df_cuda.h) with its
// parameters, run by `ctas` CTAs.
struct DeviceActor {
  int kind = 0;  // 0: not device-resident
  std::vector<std::byte> params;
  std::uint32_t ctas = 1;
  template <typename P>
  static DeviceActor of(int kind, const P& p, std::uint32_t ctas = 1) {
    DeviceActor d;
    d.kind = kind;
    d.params.resize(sizeof(P));
    std::memcpy(d.params.data(), &p, sizeof(P));
    d.ctas = ctas;
    return d;
  }
};

// model.hpp:103-108: mandatory fire; optional init / control / finish.
//   * fire       host-issued GPU actor: enqueues device work per firing;
//   * host_fire  CPU actor: computes on host spans in stream order
//                (host-issued networks; a dynamic CPU actor's control token
//                is read on the host, one stream synchronisation per firing);
//   * device     device-resident GPU actor (see DeviceActor).
// control (the reference's signature) is required for a dynamic
// device-resident actor and a dynamic CPU actor: it maps one control token
// to FiringRates.  A CPU actor calls it per firing on the host
// (control_dispatch); a device-resident actor's control is
// evaluated for every token value v < control_domain (v little-endian in
// the token's bytes) into the device control table before the run; a
// result that is not 0-or-r per port (or a throw) makes that token a
// ControlError when a firing reads it.  device_control marks a host-issued
// dynamic actor that consumes its control tokens inside its own kernels.
struct ActorBehavior {
  std::function<void(FiringContext&)> fire;
  std::function<void(HostFiringContext&)> host_fire;
  std::function<void()> init;
  std::function<FiringRates(std::span<const std::byte>)> control;
  std::function<void()> finish;
  std::uint32_t control_domain = 1024;
  bool device_control = false;
  DeviceActor device;
  bool is_host() const { return static_cast<bool>(host_fire); }
  bool is_device_resident() const { return device.kind != 0; }
};

struct ActorSpec {
  std::string id;
  ActorKind kind = ActorKind::static_rate;
  std::vector<PortSpec> ports;
  ActorBehavior behavior;
};

struct ChannelEndpoints {
  std::size_t producer_actor = npos, producer_port = npos;
  std::size_t consumer_actor = npos, consumer_port = npos;
  static constexpr std::size_t npos = static_cast<std::size_t>(-1);
};

class BuildError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ControlError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct Violation {
  std::string subject;
  std::string message;
  bool operator==(const Violation&) const = default;
};

class NetworkGraph {
 public:
  const std::vector<ActorSpec>& actors() const { return actors_; }
  const std::vector<ChannelSpec>& channels() const { return channels_; }
  const std::vector<ChannelEndpoints>& endpoints() const { return endpoints_; }
  std::size_t actor_index(const std::string& id) const;
  std::size_t channel_index(const std::string& id) const;
  const ChannelSpec& channel(const std::string& id) const { return channels().at(channel_index(id)); }  // model.hpp:158
  std::vector<std::size_t> regular_ports(std::size_t actor) const;
  std::optional<std::size_t> control_port(std::size_t actor) const;

  friend NetworkGraph build_network(std::vector<ActorSpec> actors, std::vector<ChannelSpec> channels);

 private:
  std::vector<ActorSpec> actors_;
  std::vector<ChannelSpec> channels_;
  std::vector<ChannelEndpoints> endpoints_;
};

// Structural assembly, BuildError on defects (model.cpp:45-102 semantics).
NetworkGraph build_network(std::vector<ActorSpec> actors, std::vector<ChannelSpec> channels);

// Rule checks, ordered by channel id, actor id, then structure
// (model.cpp:104-238): rates/sizes >= 1, initial tokens only with a delay,
// control channels rate 1 without delay, one control port per dynamic
// actor, no undelayed cycles.  A delayed self-loop is legal at rate 1; a
// cycle whose delay channels all have rate > 1 is reported too (it cannot
// fire: the reference would block in read_start forever).
std::vector<Violation> validate(const NetworkGraph& net);

// Does the channel order firing i of its producer before firing i of its
// consumer?  Every channel except a rate-1 delay channel: its one initial
// token shifts the stream by a whole firing (consumer firing i reads what
// producer firing i-1 wrote); at rate r > 1 the consumer's firing i still
// needs r-1 tokens of producer firing i.
bool orders_same_firing(const ChannelSpec& spec);

// A topological order of the actors over the channels selected by
// orders_same_firing (declaration order among independent actors), or
// nullopt when they form a cycle.  The static schedule issues firing i of
// every actor in this order.
std::optional<std::vector<std::size_t>> firing_order(const NetworkGraph& net);

// model.cpp:240-265: runs the actor's control function on one token and
// checks the result (one entry per regular port, each 0 or the attached
// channel's rate); ControlError otherwise.  The device runtime evaluates
// this per token value before a run (df_net_set_control_table).
FiringRates control_dispatch(const NetworkGraph& net, std::size_t actor, std::span<const std::byte> control_token);

// One "a -> b -> a" path per cyclic component of the graph of channels
// selected by `edge` (validate()'s cycle findings).
std::vector<std::string> cycles(const NetworkGraph& net, const std::function<bool(const ChannelSpec&)>& edge);

// Eq. 1 (channel.cpp:9-16).
std::size_t capacity_tokens(const ChannelSpec& spec);
std::size_t capacity_bytes(const ChannelSpec& spec);

// Channel buffer memory of a network (channel.cpp:194-208; what cmd_mem
// prints, bench.cpp:145-164 / :491-525).  For a B200 network this is the
// HBM the device channels allocate (the per-channel control blocks and
// actor-private state such as FIR history are not channel buffers).
struct MemoryReport {
  struct Line {
    std::string channel_id;
    std::uint32_t token_rate = 0;
    std::size_t token_size = 0;
    bool has_delay = false;
    std::size_t capacity_tokens = 0;
    std::size_t capacity_bytes = 0;
  };
  std::vector<Line> channels;
  std::size_t total_bytes = 0;
};
MemoryReport memory_bytes(const NetworkGraph& net);

}  // namespace df
