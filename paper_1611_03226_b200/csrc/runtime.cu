// runtime.cu -- error plumbing, devices, streams, events, memory, peer
// access and synthetic-input fills of libdf_cuda.so (the CUDA "plumbing"
// beneath the GPU actors; no reference counterpart beyond std::thread /
// host memory in proj/src/runtime.cpp).
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace df {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}
void clear_error() { g_last_error.clear(); }
std::atomic<uint64_t>& launch_counter() { return g_launches; }

namespace {
// splitmix64: counter-based, so any element is computable independently.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__global__ void fill_u8_kernel(uint4* __restrict__ dst, size_t n16, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long a = splitmix64(seed ^ (2 * i)), b = splitmix64(seed ^ (2 * i + 1));
    dst[i] = make_uint4((unsigned)a, (unsigned)(a >> 32), (unsigned)b, (unsigned)(b >> 32));
  }
}
__global__ void fill_u8_tail(unsigned char* dst, size_t start, size_t n, unsigned long long seed) {
  size_t i = start + blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (unsigned char)splitmix64(seed ^ (0x5555555555555555ULL + i));
}
// Same value distribution as the reference's uniform_pm1 (24-bit grid in
// [-1,1)), drawn from splitmix64 instead of mt19937_64.
__global__ void fill_pm1_kernel(float* __restrict__ dst, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float u = (float)(splitmix64(seed ^ i) >> 40) / (float)(1u << 24);
    dst[i] = 2.0f * u - 1.0f;
  }
}
}  // namespace

}  // namespace df

using namespace df;

extern "C" {

const char* df_last_error(void) { return g_last_error.c_str(); }
int df_abi_version(void) { return 1; }
uint64_t df_kernel_launches(void) { return g_launches.load(); }

int df_device_count(int* count) {
  DF_REQUIRE(count, DF_EINVAL, "df_device_count: null out pointer");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_status(e, "cudaGetDeviceCount");
  }
  return DF_OK;
}

int df_device_sm_count(int device, int* sms) {
  DF_REQUIRE(sms, DF_EINVAL, "df_device_sm_count: null out pointer");
  DF_CHECK_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
  return DF_OK;
}

int df_set_device(int device) {
  DF_CHECK_CUDA(cudaSetDevice(device));
  return DF_OK;
}

int df_stream_create(int device, void** stream) {
  DF_REQUIRE(stream, DF_EINVAL, "df_stream_create: null out pointer");
  DF_CHECK_CUDA(cudaSetDevice(device));
  cudaStream_t s;
  DF_CHECK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = s;
  return DF_OK;
}
int df_stream_destroy(void* stream) {
  DF_CHECK_CUDA(cudaStreamDestroy(as_stream(stream)));
  return DF_OK;
}
int df_stream_synchronize(void* stream) {
  DF_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return DF_OK;
}
int df_event_create(void** ev) {
  DF_REQUIRE(ev, DF_EINVAL, "df_event_create: null out pointer");
  cudaEvent_t e;
  DF_CHECK_CUDA(cudaEventCreate(&e));
  *ev = e;
  return DF_OK;
}
int df_event_destroy(void* ev) {
  DF_CHECK_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev)));
  return DF_OK;
}
int df_event_record(void* ev, void* stream) {
  DF_CHECK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), as_stream(stream)));
  return DF_OK;
}
int df_event_synchronize(void* ev) {
  DF_CHECK_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(ev)));
  return DF_OK;
}
int df_event_elapsed_ms(void* start, void* stop, float* ms) {
  DF_REQUIRE(ms, DF_EINVAL, "df_event_elapsed_ms: null out pointer");
  DF_CHECK_CUDA(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start),
                                     reinterpret_cast<cudaEvent_t>(stop)));
  return DF_OK;
}
int df_stream_wait_event(void* stream, void* ev) {
  DF_CHECK_CUDA(cudaStreamWaitEvent(as_stream(stream), reinterpret_cast<cudaEvent_t>(ev), 0));
  return DF_OK;
}

int df_malloc(int device, size_t bytes, void** dptr) {
  DF_REQUIRE(dptr, DF_EINVAL, "df_malloc: null out pointer");
  DF_CHECK_CUDA(cudaSetDevice(device));
  DF_CHECK_CUDA(cudaMalloc(dptr, bytes ? bytes : 1));
  return DF_OK;
}
int df_free(void* dptr) {
  DF_CHECK_CUDA(cudaFree(dptr));
  return DF_OK;
}
int df_launch_host_func(void* stream, void (*fn)(void*), void* user) {
  DF_REQUIRE(fn, DF_EINVAL, "df_launch_host_func: null function");
  DF_CHECK_CUDA(cudaLaunchHostFunc(as_stream(stream), fn, user));
  return DF_OK;
}

int df_host_alloc(size_t bytes, void** hptr) {
  DF_REQUIRE(hptr, DF_EINVAL, "df_host_alloc: null out pointer");
  DF_CHECK_CUDA(cudaHostAlloc(hptr, bytes ? bytes : 1, cudaHostAllocPortable));
  return DF_OK;
}
int df_host_free(void* hptr) {
  DF_CHECK_CUDA(cudaFreeHost(hptr));
  return DF_OK;
}
int df_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  DF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
  return DF_OK;
}
int df_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  DF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
  return DF_OK;
}
int df_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  DF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
  return DF_OK;
}
int df_memset(void* dst, int value, size_t bytes, void* stream) {
  DF_CHECK_CUDA(cudaMemsetAsync(dst, value, bytes, as_stream(stream)));
  return DF_OK;
}

int df_peer_enable(int a, int b) {
  if (a == b) return DF_OK;
  int can = 0;
  DF_CHECK_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
  DF_REQUIRE(can, DF_EINVAL, "df_peer_enable: device %d cannot access device %d", a, b);
  DF_CHECK_CUDA(cudaSetDevice(a));
  cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  DF_CHECK_CUDA(e);
  return DF_OK;
}

int df_halo_copy(int dst_device, void* dst, int src_device, const void* src, size_t bytes,
                 void* stream) {
  if (dst_device == src_device) {
    DF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
  } else {
    // Unified addressing resolves both ends -- plain peer pointers and
    // CUDA-IPC-mapped ones (df_ipc_open_handle) alike -- and the copy goes
    // peer to peer over NVLink when peer access is enabled.
    DF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  }
  return DF_OK;
}

// Cross-process peer memory (one process per GPU): a rank exports its
// shard's allocation once, its neighbour maps it and pulls the halo with
// copy-engine peer copies over NVLink -- no collective, no NCCL kernel.
int df_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }
int df_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  DF_REQUIRE(dev_ptr && handle_out, DF_EINVAL, "df_ipc_get_handle: null argument");
  cudaIpcMemHandle_t h;
  DF_CHECK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  std::memcpy(handle_out, &h, sizeof h);
  return DF_OK;
}
int df_ipc_open_handle(int device, const void* handle, void** dev_ptr) {
  DF_REQUIRE(handle && dev_ptr, DF_EINVAL, "df_ipc_open_handle: null argument");
  DF_CHECK_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  DF_CHECK_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return DF_OK;
}
int df_ipc_close_handle(void* dev_ptr) {
  DF_CHECK_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return DF_OK;
}

int df_fill_random_u8(void* dst, size_t bytes, uint64_t seed, void* stream) {
  DF_REQUIRE(dst || bytes == 0, DF_EINVAL, "df_fill_random_u8: null destination");
  if (bytes == 0) return DF_OK;
  const size_t n16 = ((uintptr_t)dst % 16 == 0) ? bytes / 16 : 0;
  cudaStream_t s = as_stream(stream);
  if (n16) {
    fill_u8_kernel<<<1184, 256, 0, s>>>(reinterpret_cast<uint4*>(dst), n16, seed);
    DF_TRY(after_launch("fill_u8_kernel"));
  }
  const size_t rest = bytes - n16 * 16;
  if (rest) {
    fill_u8_tail<<<(unsigned)((rest + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<unsigned char*>(dst), n16 * 16, bytes, seed);
    DF_TRY(after_launch("fill_u8_tail"));
  }
  return DF_OK;
}

int df_fill_random_pm1(float* dst, size_t floats, uint64_t seed, void* stream) {
  DF_REQUIRE(dst || floats == 0, DF_EINVAL, "df_fill_random_pm1: null destination");
  if (floats == 0) return DF_OK;
  fill_pm1_kernel<<<1184, 256, 0, as_stream(stream)>>>(dst, floats, seed);
  return after_launch("fill_pm1_kernel");
}

}  // extern "C"
