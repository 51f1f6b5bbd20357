// staging.cuh -- persistent multi-buffered H2D / compute / D2H pipeline
// state of an actor's host-buffer entry point (df_*_run_host).  Allocated
// on first use, grown on demand, released with the actor.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace df {

// kSlots buffers per direction: chunk c's H2D, chunk c-1's fire and chunk
// c-2's D2H run concurrently (three stages in flight).
constexpr int kSlots = 3;

// Is `p` page-locked (cudaHostAlloc'ed or registered) host memory?
inline bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// memcpy split across host threads (pageable <-> pinned staging): one
// thread moves ~10 GB/s, the PCIe link ~55 GB/s.
inline void par_copy(void* dst, const void* src, size_t n) {
  constexpr size_t kSlice = 4u << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>(std::max(1u, std::min(8u, hw / 2)), (n + kSlice - 1) / kSlice);
  if (nt <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::vector<std::thread> ts;
  const size_t part = (n + nt - 1) / nt;
  for (size_t t = 1; t < nt; ++t) {
    const size_t a = t * part, b = std::min(n, a + part);
    if (a < b)
      ts.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
  }
  std::memcpy(dst, src, std::min(n, part));
  for (std::thread& t : ts) t.join();
}

struct Staging {
  unsigned char* in[kSlots] = {};
  unsigned char* out[kSlots] = {};
  size_t in_cap = 0, out_cap = 0;
  // Pageable caller buffers: pinned host slots between them and the DMA.
  unsigned char* hin[kSlots] = {};
  unsigned char* hout[kSlots] = {};
  size_t hin_cap = 0, hout_cap = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t in_ready[kSlots] = {}, comp_done[kSlots] = {}, out_free[kSlots] = {};
  bool init = false;

  int ensure(size_t in_bytes, size_t out_bytes) {
    if (!init) {
      DF_CHECK_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
      DF_CHECK_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
      for (int i = 0; i < kSlots; ++i) {
        DF_CHECK_CUDA(cudaEventCreateWithFlags(&in_ready[i], cudaEventDisableTiming));
        DF_CHECK_CUDA(cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming));
        DF_CHECK_CUDA(cudaEventCreateWithFlags(&out_free[i], cudaEventDisableTiming));
      }
      init = true;
    }
    if (in_bytes > in_cap || out_bytes > out_cap) {
      DF_CHECK_CUDA(cudaDeviceSynchronize());
      for (int i = 0; i < kSlots; ++i) {
        cudaFree(in[i]);
        cudaFree(out[i]);
        in[i] = out[i] = nullptr;
      }
      in_cap = std::max(in_bytes, in_cap);
      out_cap = std::max(out_bytes, out_cap);
      for (int i = 0; i < kSlots; ++i) {
        DF_CHECK_CUDA(cudaMalloc(&in[i], in_cap));
        DF_CHECK_CUDA(cudaMalloc(&out[i], out_cap));
      }
    }
    return DF_OK;
  }

  int ensure_host(size_t in_bytes, size_t out_bytes) {
    if (in_bytes <= hin_cap && out_bytes <= hout_cap) return DF_OK;
    DF_CHECK_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < kSlots; ++i) {
      cudaFreeHost(hin[i]);
      cudaFreeHost(hout[i]);
      hin[i] = hout[i] = nullptr;
    }
    hin_cap = std::max(in_bytes, hin_cap);
    hout_cap = std::max(out_bytes, hout_cap);
    for (int i = 0; i < kSlots; ++i) {
      DF_CHECK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hin[i]), hin_cap, cudaHostAllocDefault));
      DF_CHECK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hout[i]), hout_cap, cudaHostAllocDefault));
    }
    return DF_OK;
  }

  void release() {
    for (int i = 0; i < kSlots; ++i) {
      cudaFreeHost(hin[i]);
      cudaFreeHost(hout[i]);
      cudaFree(in[i]);
      cudaFree(out[i]);
      if (init) {
        cudaEventDestroy(in_ready[i]);
        cudaEventDestroy(comp_done[i]);
        cudaEventDestroy(out_free[i]);
      }
    }
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    *this = Staging();
  }

  // Chunk size in units of `unit_bytes`: at most `cap_bytes`; about 1/16 of
  // the run so H2D, fire and D2H overlap and the pipeline's fill/drain stay
  // short, but not below kMinChunkBytes -- each chunk costs ~12 us of copy
  // setup and cross-stream hand-off, which makes 2 chunks the optimum for
  // an 8 MB run (measured on B200, PCIe 5: DPD-1 e2e 1 chunk 346 us, 2
  // chunks 302 us, 8 chunks 339 us; motion 720p x300: 38-frame chunks 16.0
  // ms, 19-frame 15.6 ms, against 15.0 ms of H2D at 55.4 GB/s).
  static constexpr size_t kMinChunkBytes = 4u << 20;
  static constexpr uint64_t kTargetChunks = 16;
  static uint64_t chunk_units(uint64_t units, size_t unit_bytes, size_t cap_bytes) {
    unit_bytes = std::max<size_t>(1, unit_bytes);
    uint64_t c = std::max<uint64_t>(1, cap_bytes / unit_bytes);
    const uint64_t part = (units + kTargetChunks - 1) / kTargetChunks;
    const uint64_t floor_units = (kMinChunkBytes + unit_bytes - 1) / unit_bytes;
    c = std::min<uint64_t>(c, std::max<uint64_t>(part, floor_units));
    return std::max<uint64_t>(1, std::min<uint64_t>(c, units));
  }

  // Runs nchunks chunks: chunk c copies in_bytes(c) from host_in(c) into
  // slot c % kSlots, waits, calls fire(c, slot_in, slot_out) on `cs`, then copies
  // out_bytes(c) to host_out(c).  Slot reuse is ordered by events.  Pageable
  // caller buffers go through pinned host slots (pipeline_pageable).
  template <typename InFn, typename OutFn, typename FireFn>
  int pipeline(cudaStream_t cs, uint64_t nchunks, InFn in_of, OutFn out_of, FireFn fire) {
    if (nchunks > 0) {
      const void* hin0;
      void* hout0;
      size_t ib0, ob0;
      in_of(0, hin0, ib0);
      out_of(0, hout0, ob0);
      if (!host_pinned(hin0) || !host_pinned(hout0)) return pipeline_pageable(cs, nchunks, in_of, out_of, fire);
    }
    for (uint64_t c = 0; c < nchunks; ++c) {
      const int i = (int)(c % kSlots);
      const void* hin;
      size_t ib;
      void* hout;
      size_t ob;
      in_of(c, hin, ib);
      out_of(c, hout, ob);
      if (c >= kSlots) DF_CHECK_CUDA(cudaStreamWaitEvent(h2d, comp_done[i], 0));
      DF_CHECK_CUDA(cudaMemcpyAsync(in[i], hin, ib, cudaMemcpyHostToDevice, h2d));
      DF_CHECK_CUDA(cudaEventRecord(in_ready[i], h2d));
      DF_CHECK_CUDA(cudaStreamWaitEvent(cs, in_ready[i], 0));
      if (c >= kSlots) DF_CHECK_CUDA(cudaStreamWaitEvent(cs, out_free[i], 0));
      DF_TRY(fire(c, in[i], out[i]));
      DF_CHECK_CUDA(cudaEventRecord(comp_done[i], cs));
      DF_CHECK_CUDA(cudaStreamWaitEvent(d2h, comp_done[i], 0));
      DF_CHECK_CUDA(cudaMemcpyAsync(hout, out[i], ob, cudaMemcpyDeviceToHost, d2h));
      DF_CHECK_CUDA(cudaEventRecord(out_free[i], d2h));
    }
    DF_CHECK_CUDA(cudaStreamSynchronize(d2h));
    DF_CHECK_CUDA(cudaStreamSynchronize(cs));
    return DF_OK;
  }

  // Pageable caller buffers: the driver would bounce every copy through its
  // own staging on this thread (~6 GB/s).  Here host threads copy chunk c
  // into pinned slot c % kSlots once chunk c - kSlots's H2D has drained it,
  // and copy chunk c - 2's output back once its D2H has landed -- while the
  // DMA engines and the firing work on the chunks in between.
  template <typename InFn, typename OutFn, typename FireFn>
  int pipeline_pageable(cudaStream_t cs, uint64_t nchunks, InFn in_of, OutFn out_of, FireFn fire) {
    size_t ib_max = 0, ob_max = 0;
    for (uint64_t c = 0; c < nchunks; ++c) {
      const void* h;
      void* o;
      size_t ib, ob;
      in_of(c, h, ib);
      out_of(c, o, ob);
      ib_max = std::max(ib_max, ib);
      ob_max = std::max(ob_max, ob);
    }
    DF_TRY(ensure_host(ib_max, ob_max));
    auto drain_out = [&](uint64_t c) -> int {  // chunk c's output -> caller
      void* o;
      size_t ob;
      out_of(c, o, ob);
      DF_CHECK_CUDA(cudaEventSynchronize(out_free[c % kSlots]));
      par_copy(o, hout[c % kSlots], ob);
      return DF_OK;
    };
    for (uint64_t c = 0; c < nchunks; ++c) {
      const int i = (int)(c % kSlots);
      const void* h;
      size_t ib;
      void* o;
      size_t ob;
      in_of(c, h, ib);
      out_of(c, o, ob);
      if (c >= kSlots) DF_CHECK_CUDA(cudaEventSynchronize(in_ready[i]));  // slot drained by chunk c-3's H2D
      par_copy(hin[i], h, ib);
      if (c >= kSlots) DF_CHECK_CUDA(cudaStreamWaitEvent(h2d, comp_done[i], 0));
      DF_CHECK_CUDA(cudaMemcpyAsync(in[i], hin[i], ib, cudaMemcpyHostToDevice, h2d));
      DF_CHECK_CUDA(cudaEventRecord(in_ready[i], h2d));
      DF_CHECK_CUDA(cudaStreamWaitEvent(cs, in_ready[i], 0));
      if (c >= kSlots) DF_CHECK_CUDA(cudaStreamWaitEvent(cs, out_free[i], 0));
      DF_TRY(fire(c, in[i], out[i]));
      DF_CHECK_CUDA(cudaEventRecord(comp_done[i], cs));
      if (c >= 2) DF_TRY(drain_out(c - 2));  // frees pinned slot (c-2) % kSlots before chunk c+1 reuses it
      DF_CHECK_CUDA(cudaStreamWaitEvent(d2h, comp_done[i], 0));
      DF_CHECK_CUDA(cudaMemcpyAsync(hout[i], out[i], ob, cudaMemcpyDeviceToHost, d2h));
      DF_CHECK_CUDA(cudaEventRecord(out_free[i], d2h));
    }
    for (uint64_t c = nchunks >= 2 ? nchunks - 2 : 0; c < nchunks; ++c) DF_TRY(drain_out(c));
    DF_CHECK_CUDA(cudaStreamSynchronize(cs));
    return DF_OK;
  }
};

}  // namespace df
