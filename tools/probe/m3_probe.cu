// Probes the M3 building blocks in isolation: TMEM alloc/st/ld, TMA 2D + mbarrier.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <cstring>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

#ifndef NO_TMEM
template <int MODE>
__global__ void tmem_probe(unsigned* out) {
  __shared__ unsigned slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned base = slot;
  if (MODE >= 1) {
    const unsigned ta = base + ((unsigned)(32 * warp) << 16) + 6;
    unsigned a = threadIdx.x * 3 + 1, b = threadIdx.x * 7 + 2;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(ta), "r"(a), "r"(b) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    unsigned c = 0, d = 0;
    if (MODE >= 2) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(c), "=r"(d) : "r"(ta) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(c), "+r"(d)::"memory");
    }
    out[threadIdx.x * 2] = c;
    out[threadIdx.x * 2 + 1] = d;
  }
  if (lane == 0 && warp == 0) out[1000] = base;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base) : "memory");
  }
}

#endif
template <int V>
__global__ void tma_probe(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, unsigned* out, int c0, int c1, unsigned nbytes) {
  __shared__ __align__(128) unsigned buf[192 * 4];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = smem_u32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    if (V != 3) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nbytes) : "memory");
    const uint64_t desc = V == 2 ? reinterpret_cast<uint64_t>(gmap) : reinterpret_cast<uint64_t>(&map);
    if (V == 1)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(buf)), "l"(desc), "r"(c0), "r"(c1), "r"(b) : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(buf)), "l"(desc), "r"(c0), "r"(c1), "r"(b) : "memory");
  }
  unsigned done;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b), "r"(0u) : "memory");
  } while (!done);
  for (int i = threadIdx.x; i < 192 * 4; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int V = argc > 1 ? atoi(argv[1]) : 0;
  unsigned* d;
  CK(cudaMalloc(&d, 1 << 20));
#ifndef NO_TMEM
  for (int mode = 0; mode < 3; ++mode) {
    CK(cudaMemset(d, 0, 1 << 20));
    if (mode == 0) tmem_probe<0><<<1, 128>>>(d);
    if (mode == 1) tmem_probe<1><<<1, 128>>>(d);
    if (mode == 2) tmem_probe<2><<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("tmem mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<unsigned> h(1024);
    cudaMemcpy(h.data(), d, 4096, cudaMemcpyDeviceToHost);
    int bad = 0;
    if (mode == 2) for (int t = 0; t < 128; ++t) bad += h[2 * t] != t * 3u + 1 || h[2 * t + 1] != t * 7u + 2;
    printf("  base=%u bad=%d  v[0..3]=%u %u %u %u\n", h[1000], bad, h[0], h[1], h[2], h[3]);
  }
#endif
  // TMA: a 2D uint32 tensor of 960 x 64 rows
  const int cols = 960, rows = 64;
  std::vector<unsigned> src(cols * rows);
  for (int i = 0; i < cols * rows; ++i) src[i] = i;
  unsigned* g;
  CK(cudaMalloc(&g, src.size() * 4));
  CK(cudaMemcpy(g, src.data(), src.size() * 4, cudaMemcpyHostToDevice));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  const unsigned B0 = argc > 2 ? atoi(argv[2]) : 192, B1 = argc > 3 ? atoi(argv[3]) : 4;
  cuuint32_t box[2] = {B0, B1}, es[2] = {1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, g, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d  words: %llx %llx %llx %llx\n", (int)r, (unsigned long long)map.opaque[0], (unsigned long long)map.opaque[1], (unsigned long long)map.opaque[2], (unsigned long long)map.opaque[3]);
#ifdef DIRECT
  CUtensorMap map2;
  r = cuTensorMapEncodeTiled(&map2, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, g, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("direct encode: %d same=%d\n", (int)r, memcmp(&map, &map2, sizeof(map)) == 0);
  map = map2;
#endif
  CUtensorMap* gm;
  CK(cudaMalloc(&gm, sizeof(CUtensorMap)));
  CK(cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice));
  printf("variant %d\n", V);
  int cases[3][2] = {{atoi(argc > 4 ? argv[4] : "176"), 10}, {-8, -2}, {900, 62}};
  for (auto& c : cases) {
    CK(cudaMemset(d, 0xFF, 1 << 20));
    if (V == 0) tma_probe<0><<<1, 128>>>(map, gm, d, c[0], c[1], B0 * B1 * 4);
    if (V == 1) tma_probe<1><<<1, 128>>>(map, gm, d, c[0], c[1], B0 * B1 * 4);
    if (V == 3) tma_probe<3><<<1, 128>>>(map, gm, d, c[0], c[1], B0 * B1 * 4);
    if (V == 2) tma_probe<2><<<1, 128>>>(map, gm, d, c[0], c[1], B0 * B1 * 4);
    cudaError_t e = cudaDeviceSynchronize();
    printf("tma (%d,%d): %s\n", c[0], c[1], cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<unsigned> h(768);
    cudaMemcpy(h.data(), d, 768 * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < (int)B1; ++rr)
      for (int cc = 0; cc < (int)B0; ++cc) {
        int x = c[0] + cc, y = c[1] + rr;
        unsigned want = (x >= 0 && x < cols && y >= 0 && y < rows) ? (unsigned)(y * cols + x) : 0u;
        bad += h[rr * B0 + cc] != want;
      }
    printf("  bad=%d first=%u\n", bad, h[0]);
  }
  return 0;
}
