// common.cuh -- error plumbing shared by the libdf_cuda translation units.
// Every C-ABI entry point returns a DF_* status and stores a thread-local
// message (df_last_error), mirroring how the reference surfaces contract
// violations as exceptions (proj/src/channel.cpp:65-77).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "df_cuda.h"

namespace df {

int set_error(int code, const char* fmt, ...);
void clear_error();
std::atomic<uint64_t>& launch_counter();

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DF_OK;
  return set_error(DF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Counts our own kernel launches (bench "gpu_launches") and checks the
// launch configuration error immediately.
inline int after_launch(const char* what) {
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError(), what);
}

}  // namespace df

#define DF_CHECK_CUDA(expr)                                       \
  do {                                                            \
    cudaError_t df_e_ = (expr);                                   \
    if (df_e_ != cudaSuccess) return ::df::cuda_status(df_e_, #expr); \
  } while (0)

#define DF_REQUIRE(cond, code, ...)                   \
  do {                                                \
    if (!(cond)) return ::df::set_error(code, __VA_ARGS__); \
  } while (0)

#define DF_TRY(expr)              \
  do {                            \
    int df_rc_ = (expr);          \
    if (df_rc_ != DF_OK) return df_rc_; \
  } while (0)
