// staging.cuh -- persistent double-buffered H2D / compute / D2H pipeline
// state of an actor's host-buffer entry point (df_*_run_host).  Allocated
// on first use, grown on demand, released with the actor.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace df {

struct Staging {
  unsigned char* in[2] = {nullptr, nullptr};
  unsigned char* out[2] = {nullptr, nullptr};
  size_t in_cap = 0, out_cap = 0;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t in_ready[2] = {}, comp_done[2] = {}, out_free[2] = {};
  bool init = false;

  int ensure(size_t in_bytes, size_t out_bytes) {
    if (!init) {
      DF_CHECK_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
      DF_CHECK_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        DF_CHECK_CUDA(cudaEventCreateWithFlags(&in_ready[i], cudaEventDisableTiming));
        DF_CHECK_CUDA(cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming));
        DF_CHECK_CUDA(cudaEventCreateWithFlags(&out_free[i], cudaEventDisableTiming));
      }
      init = true;
    }
    if (in_bytes > in_cap || out_bytes > out_cap) {
      DF_CHECK_CUDA(cudaDeviceSynchronize());
      for (int i = 0; i < 2; ++i) {
        cudaFree(in[i]);
        cudaFree(out[i]);
        in[i] = out[i] = nullptr;
      }
      in_cap = std::max(in_bytes, in_cap);
      out_cap = std::max(out_bytes, out_cap);
      for (int i = 0; i < 2; ++i) {
        DF_CHECK_CUDA(cudaMalloc(&in[i], in_cap));
        DF_CHECK_CUDA(cudaMalloc(&out[i], out_cap));
      }
    }
    return DF_OK;
  }

  void release() {
    for (int i = 0; i < 2; ++i) {
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

  // Runs nchunks chunks: chunk c copies in_bytes(c) from host_in(c) into
  // slot c&1, waits, calls fire(c, slot_in, slot_out) on `cs`, then copies
  // out_bytes(c) to host_out(c).  Slot reuse is ordered by events.
  template <typename InFn, typename OutFn, typename FireFn>
  int pipeline(cudaStream_t cs, uint64_t nchunks, InFn in_of, OutFn out_of, FireFn fire) {
    for (uint64_t c = 0; c < nchunks; ++c) {
      const int i = (int)(c & 1);
      const void* hin;
      size_t ib;
      void* hout;
      size_t ob;
      in_of(c, hin, ib);
      out_of(c, hout, ob);
      if (c >= 2) DF_CHECK_CUDA(cudaStreamWaitEvent(h2d, comp_done[i], 0));
      DF_CHECK_CUDA(cudaMemcpyAsync(in[i], hin, ib, cudaMemcpyHostToDevice, h2d));
      DF_CHECK_CUDA(cudaEventRecord(in_ready[i], h2d));
      DF_CHECK_CUDA(cudaStreamWaitEvent(cs, in_ready[i], 0));
      if (c >= 2) DF_CHECK_CUDA(cudaStreamWaitEvent(cs, out_free[i], 0));
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
};

}  // namespace df
