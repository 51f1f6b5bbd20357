// channel_dev.cuh -- device-resident FIFO channel (the B200 form of the
// reference Channel, proj/include/dynflow/channel.hpp:71-135).
//
// Storage keeps the reference's Eq. 1 layout exactly: 2r slots for a
// regular channel, 3r+1 with a delay token (proj/src/channel.cpp:9-12).
// The slot walk is Fig. 2 (proj/src/channel.cpp:18-32): regular channels
// alternate halves; delay channels write [p*r+1, p*r+r] and read
// [p*r, p*r+r-1] for p = phase % 3, and the phase-2 write ends with a copy
// of slot 3r into slot 0 (proj/src/channel.cpp:97-104).
//
// The indices and counters are a control block in HBM (DevChanState).  A
// GPU actor kernel reads the phases at its start to locate its regions,
// and one thread commits the firing's token counts (0 or r per port) at
// its end -- no host round trip for data-dependent rates.
#pragma once

#include <cstdint>

namespace df {

struct DevChanState {
  unsigned long long written;    // tokens committed by the producer
  unsigned long long read;       // tokens released by the consumer
  unsigned long long available;  // committed - released (incl. the delay token)
  unsigned int write_phase;
  unsigned int read_phase;
  unsigned int closed;
  unsigned int error;            // sticky DF_* code, first error wins
};

struct DevChan {
  unsigned char* storage;
  DevChanState* st;
  unsigned long long token_size;
  unsigned int rate;
  unsigned int has_delay;
};

__host__ __device__ inline unsigned long long chan_capacity_tokens(unsigned rate, unsigned delay) {
  return delay ? 3ull * rate + 1 : 2ull * rate;
}
__host__ __device__ inline unsigned long long chan_distinct_capacity(unsigned rate, unsigned delay) {
  return delay ? 3ull * rate : 2ull * rate;  // channel.cpp:53-57
}
__host__ __device__ inline unsigned long long chan_write_slot(unsigned rate, unsigned delay,
                                                              unsigned phase) {
  return delay ? (unsigned long long)(phase % 3) * rate + 1 : (unsigned long long)(phase % 2) * rate;
}
__host__ __device__ inline unsigned long long chan_read_slot(unsigned rate, unsigned delay,
                                                             unsigned phase) {
  return delay ? (unsigned long long)(phase % 3) * rate : (unsigned long long)(phase % 2) * rate;
}
__host__ __device__ inline unsigned chan_phases(unsigned delay) { return delay ? 3u : 2u; }

#ifdef __CUDACC__
// Region of the producer's next write, resolved from the device phase.
__device__ inline unsigned char* chan_write_region(const DevChan& c) {
  const unsigned p = *(volatile unsigned*)&c.st->write_phase;
  return c.storage + chan_write_slot(c.rate, c.has_delay, p) * c.token_size;
}
__device__ inline unsigned char* chan_read_region(const DevChan& c) {
  const unsigned p = *(volatile unsigned*)&c.st->read_phase;
  return c.storage + chan_read_slot(c.rate, c.has_delay, p) * c.token_size;
}
// Delay channels: does the pending write end phase 2 (copy slot 3r -> 0)?
__device__ inline bool chan_write_wraps(const DevChan& c) {
  return c.has_delay && (*(volatile unsigned*)&c.st->write_phase % 3) == 2;
}
__device__ inline void chan_set_error(DevChanState* st, unsigned code) {
  atomicCAS(&st->error, 0u, code);
}
// Single-thread commits, called once per firing after the firing's data
// movement is complete and visible (the caller fences).  n is 0 or r.
__device__ inline void chan_commit_write(const DevChan& c, unsigned n) {
  if (n == 0) return;
  DevChanState* st = c.st;
  if (st->closed) chan_set_error(st, 2 /*DF_ELOGIC: write after close*/);
  // The producer and consumer endpoints commit concurrently (different
  // streams); `available` is the one shared counter (the reference guards it
  // with its mutex, channel.cpp:106), so it is updated atomically.  Phases
  // and written/read each have a single writer.
  const unsigned long long before = atomicAdd(&st->available, (unsigned long long)n);
  if (before + n > chan_distinct_capacity(c.rate, c.has_delay))
    chan_set_error(st, 2 /*DF_ELOGIC: overflow -- schedule violated capacity*/);
  st->write_phase = (st->write_phase + 1) % chan_phases(c.has_delay);
  st->written += n;
}
__device__ inline void chan_commit_read(const DevChan& c, unsigned n) {
  if (n == 0) return;
  DevChanState* st = c.st;
  const unsigned long long before = atomicAdd(&st->available, (unsigned long long)(-(long long)n));
  if (before < n) chan_set_error(st, 2 /*DF_ELOGIC: underflow*/);
  st->read_phase = (st->read_phase + 1) % chan_phases(c.has_delay);
  st->read += n;
}
#endif

}  // namespace df
