// channel_host.hpp -- host handle of a device channel (opaque df_channel in
// the C ABI).  Shared by the translation units that bind GPU actors to
// channels.
#pragma once

#include <cstddef>
#include <cstdint>

#include "channel_dev.cuh"

namespace df {
enum class Endpoint { unbound, host, device };
}

struct df_channel {
  int device = 0;
  size_t token_size = 0;
  uint32_t rate = 1;
  bool has_delay = false;
  size_t capacity_tokens = 0;
  unsigned char* storage = nullptr;   // HBM, Eq. 1 layout
  df::DevChanState* state = nullptr;  // HBM control block
  unsigned int* scratch = nullptr;    // per-endpoint firing-completion counters
  // Host mirror of host-driven endpoints (their own phase only).
  unsigned host_write_phase = 0;
  unsigned host_read_phase = 0;
  uint64_t write_serial = 0, read_serial = 0, next_serial = 1;
  bool closed_host = false;
  bool aborted = false;
  df::Endpoint writer = df::Endpoint::unbound;
  df::Endpoint reader = df::Endpoint::unbound;

  df::DevChan dev() const {
    return df::DevChan{storage, state, (unsigned long long)token_size, rate, has_delay ? 1u : 0u};
  }
};
