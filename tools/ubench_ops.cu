// Pipe-throughput microbenchmark for the instruction mix of the DPD and
// motion kernels (non-fused FP32 mul/add, paired f32x2, integer SIMD ops).
// Prints warp-instructions/clk/SM and lane-ops/clk/SM per op class.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__global__ void k_fmul(float* out, float a, float b) {
  float x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __fmul_rn(x[i], b);
  }
  float s = 0; for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_fadd(float* out, float a, float b) {
  float x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __fadd_rn(x[i], b);
  }
  float s = 0; for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
// FMUL with 3 distinct register sources per op (models tap*x with tap in reg)
__global__ void k_fmul_rr(float* out, float a, float b) {
  float x[CH], y[CH];
  for (int i = 0; i < CH; ++i) { x[i] = a + threadIdx.x + i; y[i] = b + i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __fmul_rn(x[i], y[(i + it) & (CH - 1)]);
  }
  float s = 0; for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__global__ void k_fmul2(float* out, float a, float b) {
  unsigned long long x[CH];
  float2 bb = make_float2(b, b);
  unsigned long long bv = *reinterpret_cast<unsigned long long*>(&bb);
  for (int i = 0; i < CH; ++i) { float2 t = make_float2(a + threadIdx.x + i, a - i); x[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = mul2(x[i], bv);
  }
  unsigned long long s = 0; for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 12345) out[0] = 1;
}
__global__ void k_fadd2(float* out, float a, float b) {
  unsigned long long x[CH];
  float2 bb = make_float2(b, b);
  unsigned long long bv = *reinterpret_cast<unsigned long long*>(&bb);
  for (int i = 0; i < CH; ++i) { float2 t = make_float2(a + threadIdx.x + i, a - i); x[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = add2(x[i], bv);
  }
  unsigned long long s = 0; for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 12345) out[0] = 1;
}
// One complex FIR tap exactly as the reference orders it, scalar, 4 outputs/thread.
__global__ void k_tap_scalar(float* out, float a, float b) {
  float ar[4], ai[4], xr[4], xi[4];
  for (int i = 0; i < 4; ++i) { ar[i] = 0; ai[i] = 0; xr[i] = a + threadIdx.x + i; xi[i] = b - i; }
  float tr = a * 0.5f, ti = b * 0.25f;
  for (int it = 0; it < ITERS / 2; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float d = __fsub_rn(__fmul_rn(tr, xr[i]), __fmul_rn(ti, xi[i]));
      float e = __fadd_rn(__fmul_rn(tr, xi[i]), __fmul_rn(ti, xr[i]));
      ar[i] = __fadd_rn(ar[i], d);
      ai[i] = __fadd_rn(ai[i], e);
      xr[i] = __fadd_rn(xr[i], tr);  // keep the window moving (counts as 1 op)
    }
  }
  float s = 0; for (int i = 0; i < 4; ++i) s += ar[i] + ai[i] + xr[i];
  if (s == 1.2345f) out[0] = s;
}
__global__ void k_lop3(unsigned* out, unsigned a, unsigned b) {
  unsigned x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x * 7 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) { unsigned r; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(x[i]), "r"(b), "r"(x[(i + 1) & (CH - 1)])); x[i] = r; }
  }
  unsigned s = 0; for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_iadd3(unsigned* out, unsigned a, unsigned b) {
  unsigned x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x * 7 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) { unsigned r; asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(x[i]), "r"(b)); x[i] = r; }
  }
  unsigned s = 0; for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_prmt(unsigned* out, unsigned a, unsigned b) {
  unsigned x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x * 7 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __byte_perm(x[i], b, 0x5140);
  }
  unsigned s = 0; for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_dp4a(unsigned* out, unsigned a, unsigned b) {
  unsigned x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x * 7 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __dp4a(x[i], b, x[i]);
  }
  unsigned s = 0; for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_imad(unsigned* out, unsigned a, unsigned b) {
  unsigned x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x * 7 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = x[i] * b + x[(i + 3) & (CH - 1)];
  }
  unsigned s = 0; for (int i = 0; i < CH; ++i) s ^= x[i];
  if (s == 12345) out[0] = s;
}
// Mixed ALU + FMA pipe: LOP3 and IMAD interleaved (does the int work dual-issue?)
__global__ void k_mix(unsigned* out, unsigned a, unsigned b) {
  unsigned x[CH], y[CH];
  for (int i = 0; i < CH; ++i) { x[i] = a + threadIdx.x * 7 + i; y[i] = b + i; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      unsigned r; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(x[i]), "r"(b), "r"(a)); x[i] = r;
      y[i] = y[i] * b + a;
    }
  }
  unsigned s = 0; for (int i = 0; i < CH; ++i) s ^= x[i] ^ y[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_sqrt(float* out, float a, float b) {
  float x[CH];
  for (int i = 0; i < CH; ++i) x[i] = a + threadIdx.x + i;
  for (int it = 0; it < ITERS / 8; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __fadd_rn(sqrtf(x[i]), b);
  }
  float s = 0; for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 1.2345f) out[0] = s;
}

template <typename K, typename T>
double run(K kern, T* buf, T a, T b, int blocks, int threads, double ops_per_thread, const char* name, int clk_khz, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(buf, a, b);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(buf, a, b);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double t = ms / 5 * 1e-3;
  double warp_instr = ops_per_thread * blocks * threads / 32.0;
  double rate = warp_instr / t;  // warp-instr/s
  // per SM per clock at the *max* clock (upper bound on clk; reported clk also)
  double per_sm_clk = rate / sms / (clk_khz * 1e3);
  printf("%-12s %8.3f ms  %10.1f Gwarp-instr/s  %6.2f warp-instr/clk/SM (@%d MHz)  %7.1f lane-ops/clk/SM\n",
         name, t * 1e3, rate / 1e9, per_sm_clk, clk_khz / 1000, per_sm_clk * 32);
  return per_sm_clk;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s SMs=%d clk=%d kHz l2=%d MB smem/SM=%zu regs/SM=%d\n", p.name, p.multiProcessorCount, clk, p.l2CacheSize >> 20, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  float* fb; unsigned* ub; CK(cudaMalloc(&fb, 64)); CK(cudaMalloc(&ub, 64));
  int sms = p.multiProcessorCount; int blocks = sms * 8, threads = 256;
  run(k_fmul, fb, 1.0001f, 0.9999f, blocks, threads, double(ITERS) * CH, "FMUL", clk, sms);
  run(k_fadd, fb, 1.0001f, 0.9999f, blocks, threads, double(ITERS) * CH, "FADD", clk, sms);
  run(k_fmul_rr, fb, 1.0001f, 0.9999f, blocks, threads, double(ITERS) * CH, "FMUL_rr", clk, sms);
  run(k_fmul2, fb, 1.0001f, 0.9999f, blocks, threads, double(ITERS) * CH, "FMUL2(x2)", clk, sms);
  run(k_fadd2, fb, 1.0001f, 0.9999f, blocks, threads, double(ITERS) * CH, "FADD2(x2)", clk, sms);
  run(k_tap_scalar, fb, 1.0001f, 0.9999f, blocks, threads, double(ITERS / 2) * 4 * 9, "tap9ops", clk, sms);
  run(k_sqrt, fb, 1.0001f, 0.9999f, blocks, threads, double(ITERS / 8) * CH, "sqrt+add", clk, sms);
  run(k_lop3, ub, 3u, 5u, blocks, threads, double(ITERS) * CH, "LOP3", clk, sms);
  run(k_iadd3, ub, 3u, 5u, blocks, threads, double(ITERS) * CH, "IADD", clk, sms);
  run(k_prmt, ub, 3u, 5u, blocks, threads, double(ITERS) * CH, "PRMT", clk, sms);
  run(k_dp4a, ub, 3u, 5u, blocks, threads, double(ITERS) * CH, "IDP4A", clk, sms);
  run(k_imad, ub, 3u, 5u, blocks, threads, double(ITERS) * CH, "IMAD", clk, sms);
  run(k_mix, ub, 3u, 5u, blocks, threads, double(ITERS) * CH * 2, "LOP3+IMAD", clk, sms);
  return 0;
}
