// df/channel.hpp -- the reference's Channel API (proj/include/dynflow/
// channel.hpp:44-135) over the device channels of libdf_cuda.so.
//
// Same contract and the same Eq. 1 / Fig. 2 storage (2r slots, or 3r+1 with
// a delay token, the phase-2 copy of slot 3r into slot 0), but the storage
// is HBM: a RegionHandle's bytes are DEVICE memory, and the end calls are
// stream-ordered commits (the host never waits for tokens or room -- the
// device checks availability and capacity and records a violation in the
// channel's sticky error word, surfaced by check()).  read_start returns
// nullopt once the channel is closed and drained (channel.cpp:114-140);
// calls after abort() throw RunAborted; contract violations throw
// std::logic_error like the reference (channel.cpp:65-77).
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>

#include "df/model.hpp"
#include "df/runtime.hpp"
#include "df_cuda.h"

namespace df {

enum class RegionDirection { read, write };

// channel.hpp:44-57: an exclusive claim on a contiguous region of storage.
struct RegionHandle {
  std::size_t first_slot = 0;
  std::size_t tokens = 0;
  RegionDirection direction = RegionDirection::read;
  std::span<std::byte> bytes;  // device memory
  bool active() const { return raw.serial != 0; }
  df_region raw{};
};

class Channel {
 public:
  explicit Channel(const ChannelSpec& spec, int device = 0) : spec_(spec) {
    check(df_channel_create(device, spec.token_size, spec.token_rate, spec.has_delay ? 1 : 0,
                            spec.initial_token_value.empty() ? nullptr : spec.initial_token_value.data(), &ch_));
  }
  ~Channel() { df_channel_destroy(ch_); }
  Channel(const Channel&) = delete;
  Channel& operator=(const Channel&) = delete;

  const ChannelSpec& spec() const { return spec_; }
  std::size_t capacity_tokens() const { return df_channel_capacity_tokens(ch_); }
  std::size_t capacity_bytes() const { return df_channel_capacity_bytes(ch_); }
  df_channel* handle() const { return ch_; }  // for GPU actors' df_*_fire_channels

  RegionHandle write_start(std::size_t n) {
    RegionHandle h;
    check(df_channel_write_start(ch_, n, &h.raw));
    fill(h, RegionDirection::write);
    return h;
  }
  void write_end(RegionHandle& h, void* stream = nullptr) { check(df_channel_write_end(ch_, &h.raw, stream)); }

  std::optional<RegionHandle> read_start(std::size_t n) {
    RegionHandle h;
    const int rc = df_channel_read_start(ch_, n, &h.raw);
    if (rc == DF_EOS) return std::nullopt;
    check(rc);
    fill(h, RegionDirection::read);
    return h;
  }
  void read_end(RegionHandle& h, void* stream = nullptr) { check(df_channel_read_end(ch_, &h.raw, stream)); }

  void close(void* stream = nullptr) { check(df_channel_close(ch_, stream)); }
  void abort() { check(df_channel_abort(ch_)); }

  // Device state (these synchronize the channel's device).
  bool closed() const { return stats().closed != 0; }
  std::size_t tokens_available() const { return static_cast<std::size_t>(stats().tokens_available); }
  std::uint64_t tokens_written() const { return stats().tokens_written; }
  std::uint64_t tokens_read() const { return stats().tokens_read; }
  // The sticky device-side violation (overflow / underflow / write after
  // close) as the exception the reference would have thrown.
  void check_device() const { check(df_channel_check(ch_)); }

 private:
  df_chan_stats stats() const {
    df_chan_stats s{};
    check(df_channel_stats(ch_, &s));
    return s;
  }
  void fill(RegionHandle& h, RegionDirection d) const {
    h.first_slot = h.raw.first_slot;
    h.tokens = h.raw.tokens;
    h.direction = d;
    h.bytes = std::span<std::byte>(static_cast<std::byte*>(h.raw.dptr), h.raw.tokens * spec_.token_size);
  }

  ChannelSpec spec_;
  df_channel* ch_ = nullptr;
};

}  // namespace df
