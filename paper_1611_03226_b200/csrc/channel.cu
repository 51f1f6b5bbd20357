// channel.cu -- device-resident channels: the B200 form of the reference
// Channel (proj/include/dynflow/channel.hpp:71-135, proj/src/channel.cpp).
//
// Storage is HBM with the Eq. 1 layout; the control block (DevChanState)
// is in HBM too.  Host-driven endpoints (source/sink actors, tests) keep a
// host mirror of their own phase -- it only ever depends on that endpoint's
// own history -- so they can name their region without reading the
// device; their commits are stream-ordered single-thread kernels.  GPU
// actor kernels resolve regions and commit directly on the device
// (channel_dev.cuh).  An endpoint is either host-driven or device-driven
// for its lifetime; mixing is a contract error (DF_ELOGIC).
#include <cstring>
#include <vector>

#include "channel_dev.cuh"
#include "channel_host.hpp"
#include "common.cuh"

#ifndef DF_CHAN_COMMIT_PDL
#define DF_CHAN_COMMIT_PDL 1
#endif

namespace df {

namespace {

// Host-endpoint commit: one thread.  Launched with programmatic dependent
// launch so it becomes resident while the previous kernel (typically the
// actor firing that produced or consumed the tokens) drains, and lets the
// next kernel do the same; it touches the control block only after that
// previous grid has completed (griddepcontrol.wait).
__global__ void chan_commit_kernel(DevChan c, unsigned n, int is_write) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (is_write)
    chan_commit_write(c, n);
  else
    chan_commit_read(c, n);
}

__global__ void chan_close_kernel(DevChanState* st) { st->closed = 1; }

int launch_commit(const DevChan& c, unsigned n, int is_write, cudaStream_t s) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(1);
  lc.blockDim = dim3(1);
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = DF_CHAN_COMMIT_PDL ? 1 : 0;
  DF_CHECK_CUDA(cudaLaunchKernelEx(&lc, chan_commit_kernel, c, n, is_write));
  return after_launch("chan_commit_kernel");
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// proj/tests/acceptance.cpp:62-66 fill_token, so device streams can be
// checked against the reference's own stream-equivalence criterion [3].
__device__ __forceinline__ unsigned char token_byte(unsigned long long seed,
                                                   unsigned long long index, size_t i) {
  return (unsigned char)(mix64(seed ^ (index * 1315423911ULL + i)) & 0xFF);
}

// Returns true in exactly one thread of the last block to finish.
__device__ bool last_block_done(unsigned int* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    *counter = 0;  // re-arm for the next firing (stream order)
    return true;
  }
  return false;
}

__global__ void chan_test_produce_kernel(DevChan c, unsigned long long first_index,
                                         unsigned long long seed, unsigned int* counter) {
  unsigned char* region = chan_write_region(c);
  const bool wraps = chan_write_wraps(c);
  const size_t bytes = (size_t)c.rate * c.token_size;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < bytes;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t t = i / c.token_size, b = i % c.token_size;
    const unsigned char v = token_byte(seed, first_index + t, b);
    region[i] = v;
    // Fig. 2 phase-2 copy of slot 3r -> slot 0, fused into the store.
    if (wraps && t == c.rate - 1) c.storage[b] = v;
  }
  if (last_block_done(counter)) chan_commit_write(c, c.rate);
}

__global__ void chan_test_consume_kernel(DevChan c, unsigned long long first_pos,
                                         unsigned long long seed, int skip_initial,
                                         unsigned long long* bad, unsigned int* counter) {
  const unsigned char* region = chan_read_region(c);
  const size_t bytes = (size_t)c.rate * c.token_size;
  unsigned long long local_bad = 0;
  if (*(volatile unsigned long long*)&c.st->available < c.rate) local_bad = 1ull << 32;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < bytes;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t t = i / c.token_size, b = i % c.token_size;
    const unsigned long long pos = first_pos + t;
    unsigned char want;
    if (skip_initial)
      want = pos == 0 ? 0 : token_byte(seed, pos - 1, b);
    else
      want = token_byte(seed, pos, b);
    local_bad += region[i] != want;
  }
  if (local_bad) atomicAdd(bad, local_bad);
  if (last_block_done(counter)) chan_commit_read(c, c.rate);
}

}  // namespace

}  // namespace df

using namespace df;

extern "C" {

size_t df_slot_capacity(uint32_t rate, int has_delay) {
  return (size_t)chan_capacity_tokens(rate, has_delay != 0);
}
size_t df_slot_write_first(uint32_t rate, int has_delay, unsigned phase) {
  return (size_t)chan_write_slot(rate, has_delay != 0, phase);
}
size_t df_slot_read_first(uint32_t rate, int has_delay, unsigned phase) {
  return (size_t)chan_read_slot(rate, has_delay != 0, phase);
}

int df_channel_create(int device, size_t token_size, uint32_t token_rate, int has_delay,
                      const void* initial_token, df_channel** out) {
  DF_REQUIRE(out, DF_EINVAL, "df_channel_create: null out pointer");
  *out = nullptr;
  // proj/src/channel.cpp:38-40
  DF_REQUIRE(token_rate >= 1 && token_size >= 1, DF_EINVAL,
             "channel: token_rate and token_size must be >= 1");
  DF_REQUIRE(!initial_token || has_delay, DF_EINVAL,
             "channel: initial token value on a channel without a delay token");
  DF_CHECK_CUDA(cudaSetDevice(device));
  auto* ch = new df_channel();
  ch->device = device;
  ch->token_size = token_size;
  ch->rate = token_rate;
  ch->has_delay = has_delay != 0;
  ch->capacity_tokens = chan_capacity_tokens(token_rate, ch->has_delay);
  const size_t bytes = ch->capacity_tokens * token_size;
  cudaError_t e = cudaMalloc(&ch->storage, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&ch->state, sizeof(DevChanState) + 64);
  if (e != cudaSuccess) {
    int rc = cuda_status(e, "df_channel_create: cudaMalloc");
    cudaFree(ch->storage);
    delete ch;
    return rc;
  }
  ch->scratch = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(ch->state) + sizeof(DevChanState));
  DevChanState init{};
  if (ch->has_delay) init.available = 1;  // channel.cpp:49
  e = cudaMemset(ch->storage, 0, bytes);
  if (e == cudaSuccess && ch->has_delay && initial_token)
    e = cudaMemcpy(ch->storage, initial_token, token_size, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(ch->state, &init, sizeof init, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(ch->scratch, 0, 64);
  if (e != cudaSuccess) {
    int rc = cuda_status(e, "df_channel_create: init");
    cudaFree(ch->storage);
    cudaFree(ch->state);
    delete ch;
    return rc;
  }
  *out = ch;
  return DF_OK;
}

int df_channel_destroy(df_channel* ch) {
  if (!ch) return DF_OK;
  cudaSetDevice(ch->device);
  cudaFree(ch->storage);
  cudaFree(ch->state);
  delete ch;
  return DF_OK;
}

size_t df_channel_capacity_tokens(const df_channel* ch) { return ch ? ch->capacity_tokens : 0; }
size_t df_channel_capacity_bytes(const df_channel* ch) {
  return ch ? ch->capacity_tokens * ch->token_size : 0;
}
size_t df_channel_token_size(const df_channel* ch) { return ch ? ch->token_size : 0; }
uint32_t df_channel_token_rate(const df_channel* ch) { return ch ? ch->rate : 0; }
int df_channel_has_delay(const df_channel* ch) { return ch ? (int)ch->has_delay : 0; }
void* df_channel_storage(const df_channel* ch) { return ch ? ch->storage : nullptr; }
void* df_channel_device_state(const df_channel* ch) { return ch ? ch->state : nullptr; }

int df_channel_write_start(df_channel* ch, size_t n, df_region* region) {
  DF_REQUIRE(ch && region, DF_EINVAL, "df_channel_write_start: null argument");
  DF_REQUIRE(!ch->aborted, DF_EABORTED, "run aborted");
  // proj/src/channel.cpp:65-74
  DF_REQUIRE(n == ch->rate, DF_ELOGIC, "channel: write of %zu tokens, rate is %u", n, ch->rate);
  DF_REQUIRE(ch->write_serial == 0, DF_ELOGIC, "channel: write already outstanding");
  DF_REQUIRE(!ch->closed_host, DF_ELOGIC, "channel: write after close");
  DF_REQUIRE(ch->writer != Endpoint::device, DF_ELOGIC,
             "channel: write endpoint is device-driven; host writes would race its phase");
  ch->writer = Endpoint::host;
  const size_t slot = chan_write_slot(ch->rate, ch->has_delay, ch->host_write_phase);
  region->first_slot = slot;
  region->tokens = n;
  region->direction = 1;
  region->dptr = ch->storage + slot * ch->token_size;
  region->serial = ch->next_serial++;
  ch->write_serial = region->serial;
  return DF_OK;
}

int df_channel_write_end(df_channel* ch, df_region* region, void* stream) {
  DF_REQUIRE(ch && region, DF_EINVAL, "df_channel_write_end: null argument");
  DF_REQUIRE(region->direction == 1 && region->serial != 0 && region->serial == ch->write_serial,
             DF_ELOGIC, "channel: write_end without matching write_start");
  DF_CHECK_CUDA(cudaSetDevice(ch->device));
  cudaStream_t s = as_stream(stream);
  if (ch->has_delay && ch->host_write_phase % 3 == 2) {
    // proj/src/channel.cpp:97-104: copy slot 3r into slot 0.
    DF_CHECK_CUDA(cudaMemcpyAsync(ch->storage, ch->storage + 3ull * ch->rate * ch->token_size,
                                  ch->token_size, cudaMemcpyDeviceToDevice, s));
  }
  DF_TRY(launch_commit(ch->dev(), (unsigned)region->tokens, 1, s));
  ch->host_write_phase = (ch->host_write_phase + 1) % chan_phases(ch->has_delay);
  ch->write_serial = 0;
  region->serial = 0;
  return DF_OK;
}

int df_channel_read_start(df_channel* ch, size_t n, df_region* region) {
  DF_REQUIRE(ch && region, DF_EINVAL, "df_channel_read_start: null argument");
  DF_REQUIRE(!ch->aborted, DF_EABORTED, "run aborted");
  DF_REQUIRE(n == ch->rate, DF_ELOGIC, "channel: read of %zu tokens, rate is %u", n, ch->rate);
  DF_REQUIRE(ch->read_serial == 0, DF_ELOGIC, "channel: read already outstanding");
  DF_REQUIRE(ch->reader != Endpoint::device || ch->closed_host, DF_ELOGIC,
             "channel: read endpoint is device-driven; host reads would race its phase");
  if (ch->closed_host) {
    // End of stream (channel.cpp:114-140: closed and fewer than n tokens ->
    // nullopt).  Once closed the producer is done, so the stream-ordered
    // state can be read after synchronizing.
    DF_CHECK_CUDA(cudaSetDevice(ch->device));
    DF_CHECK_CUDA(cudaDeviceSynchronize());
    DevChanState st;
    DF_CHECK_CUDA(cudaMemcpy(&st, ch->state, sizeof st, cudaMemcpyDeviceToHost));
    if (st.available < n) return set_error(DF_EOS, "channel: end of stream (closed, %llu < %zu tokens left)",
                                           (unsigned long long)st.available, n);
    ch->host_read_phase = st.read_phase;  // a device reader may have advanced it
  }
  ch->reader = Endpoint::host;
  const size_t slot = chan_read_slot(ch->rate, ch->has_delay, ch->host_read_phase);
  region->first_slot = slot;
  region->tokens = n;
  region->direction = 0;
  region->dptr = ch->storage + slot * ch->token_size;
  region->serial = ch->next_serial++;
  ch->read_serial = region->serial;
  return DF_OK;
}

int df_channel_read_end(df_channel* ch, df_region* region, void* stream) {
  DF_REQUIRE(ch && region, DF_EINVAL, "df_channel_read_end: null argument");
  DF_REQUIRE(region->direction == 0 && region->serial != 0 && region->serial == ch->read_serial,
             DF_ELOGIC, "channel: read_end without matching read_start");
  DF_CHECK_CUDA(cudaSetDevice(ch->device));
  DF_TRY(launch_commit(ch->dev(), (unsigned)region->tokens, 0, as_stream(stream)));
  DF_TRY(after_launch("chan_commit_kernel"));
  ch->host_read_phase = (ch->host_read_phase + 1) % chan_phases(ch->has_delay);
  ch->read_serial = 0;
  region->serial = 0;
  return DF_OK;
}

int df_channel_close(df_channel* ch, void* stream) {
  DF_REQUIRE(ch, DF_EINVAL, "df_channel_close: null channel");
  DF_CHECK_CUDA(cudaSetDevice(ch->device));
  ch->closed_host = true;
  chan_close_kernel<<<1, 1, 0, as_stream(stream)>>>(ch->state);
  return after_launch("chan_close_kernel");
}

int df_channel_abort(df_channel* ch) {
  DF_REQUIRE(ch, DF_EINVAL, "df_channel_abort: null channel");
  ch->aborted = true;
  return DF_OK;
}

int df_channel_stats(df_channel* ch, df_chan_stats* out) {
  DF_REQUIRE(ch && out, DF_EINVAL, "df_channel_stats: null argument");
  DF_CHECK_CUDA(cudaSetDevice(ch->device));
  DF_CHECK_CUDA(cudaDeviceSynchronize());
  DevChanState st;
  DF_CHECK_CUDA(cudaMemcpy(&st, ch->state, sizeof st, cudaMemcpyDeviceToHost));
  out->tokens_written = st.written;
  out->tokens_read = st.read;
  out->tokens_available = st.available;
  out->write_phase = st.write_phase;
  out->read_phase = st.read_phase;
  out->closed = st.closed;
  out->error = st.error;
  return DF_OK;
}

int df_channel_check(df_channel* ch) {
  df_chan_stats st;
  DF_TRY(df_channel_stats(ch, &st));
  if (st.error)
    return set_error((int)st.error, "channel: device-side contract violation (code %u)", st.error);
  return DF_OK;
}

int df_channel_test_produce(df_channel* ch, uint64_t first_token_index, uint32_t firings,
                            uint64_t seed, void* stream) {
  DF_REQUIRE(ch, DF_EINVAL, "df_channel_test_produce: null channel");
  DF_REQUIRE(ch->writer != Endpoint::host, DF_ELOGIC, "channel: write endpoint is host-driven");
  ch->writer = Endpoint::device;
  DF_CHECK_CUDA(cudaSetDevice(ch->device));
  const size_t bytes = (size_t)ch->rate * ch->token_size;
  const unsigned blocks = (unsigned)std::min<size_t>(148 * 4, (bytes + 255) / 256);
  for (uint32_t f = 0; f < firings; ++f) {
    chan_test_produce_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
        ch->dev(), first_token_index + (uint64_t)f * ch->rate, seed, ch->scratch);
    DF_TRY(after_launch("chan_test_produce_kernel"));
  }
  return DF_OK;
}

int df_channel_test_consume(df_channel* ch, uint64_t first_token_index, uint32_t firings,
                            uint64_t seed, int skip_initial_zero_token, uint64_t* bad_dev,
                            void* stream) {
  DF_REQUIRE(ch && bad_dev, DF_EINVAL, "df_channel_test_consume: null argument");
  DF_REQUIRE(ch->reader != Endpoint::host, DF_ELOGIC, "channel: read endpoint is host-driven");
  ch->reader = Endpoint::device;
  DF_CHECK_CUDA(cudaSetDevice(ch->device));
  const size_t bytes = (size_t)ch->rate * ch->token_size;
  const unsigned blocks = (unsigned)std::min<size_t>(148 * 4, (bytes + 255) / 256);
  for (uint32_t f = 0; f < firings; ++f) {
    chan_test_consume_kernel<<<blocks, 256, 0, as_stream(stream)>>>(
        ch->dev(), first_token_index + (uint64_t)f * ch->rate, seed, skip_initial_zero_token,
        reinterpret_cast<unsigned long long*>(bad_dev), ch->scratch + 1);
    DF_TRY(after_launch("chan_test_consume_kernel"));
  }
  return DF_OK;
}

}  // extern "C"
