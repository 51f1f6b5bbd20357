// dpd.cu -- the dynamic parallel-Hammerstein predistortion actor on sm_100a.
//
// Replaces the reference's dynamic DPD network part: split actor
// (proj/src/dpd.cpp:225-256), ten branch actors poly_branch -> fir10
// (:60-121, :258-289) and the adder (:129-145, :293-331), which the
// reference runs as 12 threads exchanging per-period tokens.  Here one GPU
// actor firing covers a batch of blocks (one block = one period = one
// token of the reference's dynamic part), each gated by one control token
// consumed on the device.  Data never round-trips through split/adder
// channels: the fan-out and the branch sum live in registers.
//
// Bit-exactness.  Every float op is the reference's, in its order, with no
// FMA contraction (__fmul_rn/__fadd_rn/__fsub_rn, IEEE __fsqrt_rn):
//   mag   = sqrt(re*re + im*im); scale_b = ((1*mag)*mag)... (b-1 muls)
//           (dpd.cpp:69-71; scale_b = scale_{b-1}*mag is the same sequence)
//   fir   acc += (tr*xr - ti*xi); acc += (tr*xi + ti*xr), k ascending
//           from 0.0f (dpd.cpp:87-104)
//   adder out = 0.0f; out += y_b for active b ascending (dpd.cpp:306-320)
// Two provable rewrites keep that bit-identical while saving work:
//   * the FIR drops its leading "0.0f +" (tap 0 initialises the
//     accumulator), which can only change the sign of an exact zero;
//   * the branch sum starts from -0.0f, the exact additive identity, and
//     the output gets one final "+ 0.0f".
// x + (+0) == x for every x != -0, and the reference's sums can never be
// -0 (they start at +0; an exact-zero sum rounds to +0), so the final
// "+ 0.0f" restores the reference's bits exactly.
//
// FIR history across blocks.  Branch b's history at block p is the last
// T-1 poly outputs of b's *active* stream before p (frozen while gated
// off, dpd.cpp:264-279, fir10's chaining for short blocks :108-120).  A
// prep kernel scans the batch's control tokens on the device (per branch:
// compacted list of active blocks), resolves each needed history sample to
// either an earlier block's input (poly recomputed -- it is memoryless) or
// the carried FirState, and writes a small per-(block, branch) history
// table.  All blocks of the batch then run fully in parallel.
// Fast path (period >= T-1, every BASELINE config): the history of block p
// is the tail of ONE block -- the branch's last earlier active block q -- so
// the main kernel resolves it itself: each block-start tile scans the
// control tokens back from p with warp ballots, and the last block-start
// tile to finish advances the FirState from the per-branch last active
// block (atomicMax).
// One launch per batch, no history table.
#include <algorithm>
#include <cstring>
#include <vector>

#include "channel_dev.cuh"
#include "channel_host.hpp"
#include "common.cuh"
#include "staging.cuh"

namespace df {
namespace {

constexpr int kBranches = 10;
constexpr int kMaxTaps = 32;

// DF_DPD_TRACE (probe builds only, tools/probe_dpd_trace.py): %globaltimer
// stamps per tile warp -- start, window loaded, FIR done, end -- stored at a
// deterministic slot (no atomics on the warp's critical path).
#ifdef DF_DPD_TRACE
__device__ unsigned long long g_dpd_trace[8 << 15];
__device__ __forceinline__ unsigned long long dpd_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void dpd_trace(unsigned slot, unsigned long long id, unsigned long long t0,
                                          unsigned long long t1, unsigned long long tf) {
  const unsigned long long t2 = dpd_gtime();
  if (slot < (1u << 15)) {
    unsigned sm, ws;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(ws));
    g_dpd_trace[8 * slot] = id | ((unsigned long long)sm << 40) | ((unsigned long long)ws << 56);
    g_dpd_trace[8 * slot + 1] = t0;
    g_dpd_trace[8 * slot + 2] = t1;
    g_dpd_trace[8 * slot + 3] = t2;
    g_dpd_trace[8 * slot + 4] = tf;
  }
}
#define DPD_TSTAMP(v) const unsigned long long v = dpd_gtime()
#define DPD_TRACE(slot, id, a, b, f) \
  if ((threadIdx.x & 31) == 0) dpd_trace(slot, id, a, b, f)
#else
#define DPD_TSTAMP(v)
#define DPD_TRACE(slot, id, a, b, f)
#endif

struct DpdIO {
  // Raw mode: direct pointers.  Channel mode: resolved from the device
  // phases at kernel start (chan_*_region) -- the host never learns them.
  const uint32_t* ctrl;
  const float2* in;
  float2* out;
  DevChan ctrl_ch, in_ch, out_ch;
  int channel_mode;
};

__device__ __forceinline__ const uint32_t* io_ctrl(const DpdIO& io) {
  return io.channel_mode ? reinterpret_cast<const uint32_t*>(chan_read_region(io.ctrl_ch)) : io.ctrl;
}
__device__ __forceinline__ const float2* io_in(const DpdIO& io) {
  return io.channel_mode ? reinterpret_cast<const float2*>(chan_read_region(io.in_ch)) : io.in;
}
__device__ __forceinline__ float2* io_out(const DpdIO& io) {
  return io.channel_mode ? reinterpret_cast<float2*>(chan_write_region(io.out_ch)) : io.out;
}

// poly_branch for one sample (dpd.cpp:67-73).
__device__ __forceinline__ float2 poly_sample(float re, float im, int b) {
  if (b == 1) return make_float2(re, im);  // scale 1.0f: re*1 == re exactly
  const float mag = __fsqrt_rn(__fadd_rn(__fmul_rn(re, re), __fmul_rn(im, im)));
  float scale = mag;  // 1.0f * mag == mag exactly
  for (int p = 2; p < b; ++p) scale = __fmul_rn(scale, mag);
  return make_float2(__fmul_rn(re, scale), __fmul_rn(im, scale));
}

// ---------------------------------------------------------------------------
// Prep: per branch (one CTA each), scan the batch's control tokens, build
// the compacted active-block list, emit the history table H[p][b][j] for
// every active (p, b), and advance the carried FirState.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) dpd_prep_kernel(DpdIO io, const float2* state_in,
                                                        float2* state_out, float2* hist,
                                                        int* act, unsigned long long K,
                                                        unsigned period, int T,
                                                        unsigned* err) {
  // Programmatic dependent launch: the main kernel may start now; only its
  // block-start tiles (which read the history table) wait for this grid.
  asm volatile("griddepcontrol.launch_dependents;");
  const int b = blockIdx.x + 1;
  const uint32_t* ctrl = io_ctrl(io);
  const float2* x = io_in(io);
  int* my_act = act + (size_t)blockIdx.x * K;
  __shared__ float2 old_state[kMaxTaps];
  __shared__ unsigned warp_counts[32];
  __shared__ unsigned long long total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (tid < T - 1) old_state[tid] = state_in[(size_t)blockIdx.x * (kMaxTaps - 1) + tid];
  if (tid == 0) total = 0;
  __syncthreads();

  // Compaction of { p : bit b-1 of ctrl[p] } with warp ballots.
  for (unsigned long long base = 0; base < K; base += blockDim.x) {
    const unsigned long long p = base + tid;
    uint32_t m = p < K ? ctrl[p] : 0;
    if (b == 1 && p < K && (m >> kBranches)) atomicCAS(err, 0u, (unsigned)DF_ECONTROL);
    const bool on = (m >> (b - 1)) & 1u;
    const unsigned ballot = __ballot_sync(0xffffffffu, on);
    if (lane == 0) warp_counts[warp] = __popc(ballot);
    __syncthreads();
    if (warp == 0) {
      unsigned v = lane < nwarps ? warp_counts[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        unsigned n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
      }
      if (lane < nwarps) warp_counts[lane] = v;  // inclusive
    }
    __syncthreads();
    const unsigned before = (warp ? warp_counts[warp - 1] : 0) + __popc(ballot & ((1u << lane) - 1));
    if (on) my_act[total + before] = (int)p;
    __syncthreads();
    if (tid == 0) total += warp_counts[nwarps - 1];
    __syncthreads();
  }
  const unsigned long long C = total;
  const int H1 = T - 1;

  // History table: entry (c, j) for the c-th active block of this branch.
  // Position of x[-(j+1)] in the branch's active stream: c*period - (j+1).
  const unsigned long long items = C * (unsigned long long)H1;
  for (unsigned long long it = tid; it < items; it += blockDim.x) {
    const unsigned long long c = it / H1;
    const int j = (int)(it % H1);
    const long long pos = (long long)(c * period) - (j + 1);
    float2 u;
    if (pos >= 0) {
      const int q = my_act[pos / period];
      const float2 v = x[(size_t)q * period + (size_t)(pos % period)];
      u = poly_sample(v.x, v.y, b);
    } else {
      u = old_state[-pos - 1];
    }
    const int p = my_act[c];
    hist[((size_t)p * kBranches + blockIdx.x) * H1 + j] = u;
  }
  // New FirState = history at the end of the batch (unchanged if C == 0).
  __syncthreads();
  if (tid < H1 && C > 0) {
    const long long pos = (long long)(C * period) - (tid + 1);
    float2 u;
    if (pos >= 0) {
      const int q = my_act[pos / period];
      const float2 v = x[(size_t)q * period + (size_t)(pos % period)];
      u = poly_sample(v.x, v.y, b);
    } else {
      u = old_state[-pos - 1];
    }
    state_out[(size_t)blockIdx.x * (kMaxTaps - 1) + tid] = u;
  }
}

// ---------------------------------------------------------------------------
// Main: one CTA = one tile of S = THREADS*V samples of one block.  Per
// active branch: poly of the tile window into smem, then a register-blocked
// FIR (V consecutive outputs per thread, sliding window over the taps), and
// the branch sum in registers.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int pad_index(int w) { return w + (w >> 3); }  // bank-conflict pad

// Resident CTAs per SM the register budget targets: 5 for the short
// T=10 FIR (more CTAs hide each tile's input-load prologue; DPD-3 -5 %);
// unconstrained (0) for T=32, whose 10 x 32-tap FIR wants the registers
// (A/B in profiles/r01_ab_dpd_variants.txt).
template <int T>
constexpr int dpd_min_blocks() { return T <= 16 ? 5 : 0; }

#ifndef DF_DPD_PREFETCH
#define DF_DPD_PREFETCH 1
#endif
#ifndef DF_DPD_BLOCK_MAJOR
#define DF_DPD_BLOCK_MAJOR 1
#endif

// 1: every CTA of a plain fast-path firing takes part in the end-of-grid
// done count (the A/B baseline); 0: only the block-start tiles do.
#ifndef DF_DPD_TAIL_ALL
#define DF_DPD_TAIL_ALL 0
#endif

// Warp-local windows for T <= DF_DPD_WARP_MAX_T: DPD-3 -1 % (1.165 vs 1.176
// ms); T=32 would need 164 registers (3 CTAs/SM) and runs DPD-5 8 % slower
// (profiles/r01_ab_dpd_variants.txt).
#ifndef DF_DPD_WARP_MAX_T
#define DF_DPD_WARP_MAX_T 16
#endif
// Window layout.  WL = 0: one CTA-wide window (thread tid owns positions
// tid + m*THREADS), a __syncthreads per branch.  WL = 1: warp-local windows
// -- warp w owns outputs [32V*w, 32V*(w+1)) of the tile and the 32V + T-1
// window positions they read (lane l owns l + 32m; the T-1 positions before
// the warp's first output are loaded and poly'd by both neighbouring warps),
// so a branch needs only __syncwarp and warps never wait for each other.
template <int T, int V, int THREADS>
struct MainCfg {
  static constexpr bool WL = T <= DF_DPD_WARP_MAX_T;
  static constexpr int S = THREADS * V;             // samples per tile
  static constexpr int NW = WL ? THREADS / 32 : 1;  // windows per CTA
  static constexpr int OW = S / NW;                 // outputs per window
  static constexpr int L = WL ? 32 : THREADS;       // threads sharing a window
  static constexpr int W = OW + T - 1;              // window incl. history
  static constexpr int WP = pad_index(W) + 1;       // padded window length
  static constexpr int M = (W + L - 1) / L;         // poly positions per thread
};

// Fast-path state (see header): state = the carried FirState (read by
// block-start tiles with no earlier active block, advanced in place by the
// grid's last CTA); last1[b] = 1 + last active block of branch b+1 in the
// batch (0: none), reset by the last CTA.
// htail[b] (optional, df_dpd_fire_halo): the last T-1 raw samples,
// oldest first, of branch b+1's last active block before the batch --
// typically a peer pointer into the previous shard's input on another GPU
// (CUDA IPC, read over NVLink by the few tiles that need it).  It replaces
// the carried state for that branch, as df_dpd_set_history would.
struct FastState {
  float2* state;
  int* last1;
  const float2* htail[kBranches];
};

// History sample u[-(j+1)] of branch bi+1 with no active block earlier in
// the batch: from the halo tail if given, else the carried FirState.
template <bool HALO>
__device__ __forceinline__ float2 carried_history(const FastState& fs, int bi, int j, int H1) {
  const float2* t = HALO ? fs.htail[bi] : nullptr;
  if (t) {
    const float2 v = t[H1 - 1 - j];
    return poly_sample(v.x, v.y, bi + 1);
  }
  return fs.state[bi * (kMaxTaps - 1) + j];
}

// Block-start tile of block p (fast path): resolve every active branch's
// FIR history into hist_s[b * H1 + j] = u_b[-(j+1)].  Warp 0 scans the
// control tokens back from p, 32 per step (lowest set lane = most recent
// block), for each branch's last earlier active block q; the history is
// poly of q's last T-1 inputs, or the carried FirState / halo when the
// branch has no earlier active block.  Also publishes p into last1 for the
// end-of-grid FirState hand-off.  CTA-collective (two __syncthreads).
template <bool HALO, int NT>
__device__ __forceinline__ void dpd_block_history(const uint32_t* ctrl, const float2* __restrict__ x,
                                                  unsigned long long p, uint32_t mask, unsigned period, int H1,
                                                  const FastState& fs, int* q_s, float2* hist_s, int tid) {
  if (tid < 32) {
    unsigned need = mask;
    for (long long base = (long long)p; need && base > 0; base -= 32) {
      const long long idx = base - 1 - tid;
      const uint32_t m = idx >= 0 ? ctrl[idx] : 0u;
      for (unsigned bits = need; bits; bits &= bits - 1) {
        const int b = __ffs(bits);
        const unsigned bal = __ballot_sync(0xffffffffu, (m >> (b - 1)) & 1u);
        if (bal) {
          if (tid == 0) q_s[b - 1] = (int)(base - __ffs(bal));
          need &= ~(1u << (b - 1));
        }
      }
    }
    if (tid == 0)
      for (unsigned bits = need; bits; bits &= bits - 1) q_s[__ffs(bits) - 1] = -1;
    if (tid < kBranches && ((mask >> tid) & 1u)) atomicMax(&fs.last1[tid], (int)p + 1);
  }
  __syncthreads();
  for (int it = tid; it < kBranches * H1; it += NT) {
    const int bi = it / H1, j = it - bi * H1;
    if (!((mask >> bi) & 1u)) continue;
    const int q = q_s[bi];
    if (q >= 0) {
      const float2 v = __ldg(&x[(size_t)q * period + (period - 1 - j)]);
      hist_s[it] = poly_sample(v.x, v.y, bi + 1);
    } else {
      hist_s[it] = carried_history<HALO>(fs, bi, j, H1);
    }
  }
  __syncthreads();
}

// End of a firing, run by the last counted CTA: advance the carried FirState
// to the tails of each branch's last active block of the batch (every
// block-start tile has read the old state by now; a branch gated off all
// batch keeps its state, or takes the halo tail), reset the batch words and
// commit a channel firing (K control tokens, K blocks in, K blocks out).
template <bool HALO, int NT>
__device__ __forceinline__ void dpd_grid_end(const DpdIO& io, const float2* x, unsigned period, int H1, bool fast,
                                             const FastState& fs, unsigned* done_counter, int tid) {
  if (fast) {
    for (int it = tid; it < kBranches * H1; it += NT) {
      const int bi = it / H1, j = it - bi * H1;
      const int q = *(volatile int*)&fs.last1[bi] - 1;
      if (q >= 0) {
        const float2 v = x[(size_t)q * period + (period - 1 - j)];
        fs.state[bi * (kMaxTaps - 1) + j] = poly_sample(v.x, v.y, bi + 1);
      } else if (HALO && fs.htail[bi]) {  // gated off all batch: the halo becomes the state
        fs.state[bi * (kMaxTaps - 1) + j] = carried_history<HALO>(fs, bi, j, H1);
      }
    }
    __syncthreads();
    if (tid < kBranches) fs.last1[tid] = 0;
  }
  if (tid == 0) {
    *done_counter = 0;
    if (io.channel_mode) {
      chan_commit_read(io.ctrl_ch, io.ctrl_ch.rate);
      chan_commit_read(io.in_ch, io.in_ch.rate);
      chan_commit_write(io.out_ch, io.out_ch.rate);
    }
  }
}

// HALO: the firing takes per-branch halo tails (df_dpd_fire_halo); a
// separate instantiation, so plain firings keep their register allocation
// (with the tails compiled in, DPD-1 ran 7 % slower).
template <int T, int V, int THREADS, bool FAST, bool HALO>
__global__ void __launch_bounds__(THREADS, dpd_min_blocks<T>()) dpd_main_kernel(DpdIO io, const float2* __restrict__ taps_g,
                                                            const float2* __restrict__ hist,
                                                            unsigned period, unsigned block_major, unsigned ahead,
                                                            unsigned* err, unsigned* done_counter,
                                                            FastState fs) {
  using C = MainCfg<T, V, THREADS>;
  constexpr int H1 = T - 1;
  constexpr int HS = H1 > 0 ? H1 : 1;
  __shared__ float2 taps_s[kBranches * T];
  __shared__ float2 us_all[C::NW][2][C::WP];
  __shared__ float2 hist_s[FAST ? kBranches * HS : 1];  // fast path: this block's history per branch
  __shared__ int q_s[kBranches];

  // Block-major grids (fast path) index blocks on x, so the block-start
  // tiles -- the only CTAs with history and FirState work -- are
  // dispatched first and the grid never ends on one of them.
  const unsigned long long p = block_major ? blockIdx.x : blockIdx.y;
  const unsigned tile = block_major ? blockIdx.y : blockIdx.x;
  const uint32_t* ctrl = io_ctrl(io);
  const float2* __restrict__ x = io_in(io);
  float2* __restrict__ y = io_out(io);

  const int tid = threadIdx.x;
  DPD_TSTAMP(tr_start);
  // L2 prefetch of the input tile of the CTA dispatched `ahead` (= the
  // resident CTA slots) after this one: it starts about when this CTA
  // retires, and finds its input in L2 instead of waiting on HBM.
  if (DF_DPD_PREFETCH && ahead && tid == 0) {
    const unsigned long long L = blockIdx.x + (unsigned long long)blockIdx.y * gridDim.x + ahead;
    if (L < (unsigned long long)gridDim.x * gridDim.y) {
      const unsigned gx = (unsigned)(L % gridDim.x), gy = (unsigned)(L / gridDim.x);
      const unsigned long long pp = block_major ? gx : gy;
      const unsigned ts = (block_major ? gy : gx) * C::S;
      const unsigned bytes = (min((unsigned)C::S, period - ts) * 8u) & ~15u;
      const float2* src = x + pp * period + ts;
      if (bytes && ((reinterpret_cast<uintptr_t>(src) & 15u) == 0))
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    }
  }
  // Window-local thread index and the window's first output in the tile.
  const int lt = C::WL ? (tid & 31) : tid;
  const int wb = C::WL ? (tid >> 5) * C::OW : 0;
  float2 (*us)[C::WP] = us_all[C::WL ? (tid >> 5) : 0];
  const unsigned t0 = tile * C::S;
  const int n = (int)min((unsigned)C::S, period - t0);  // valid outputs in this tile
  const size_t blk = (size_t)p * period;
  // Every global load of the prologue (taps, control token, the window's
  // inputs) is issued before any of them is consumed, so a CTA waits one
  // memory latency, not three in a row.
  constexpr int NTR = (kBranches * T + THREADS - 1) / THREADS;  // taps per thread
  float2 tr[NTR];
#pragma unroll
  for (int k = 0; k < NTR; ++k) {
    const int i = tid + k * THREADS;
    if (i < kBranches * T) tr[k] = __ldg(&taps_g[i]);
  }
  uint32_t mask = ctrl[p];
  // Window position w in [0, W): sample index t0 + wb - (T-1) + w of the
  // block.  Each thread owns positions w = lt + m*L; keeps x, mag, scale.
  float xr[C::M], xi[C::M], mg[C::M], sc[C::M];
#pragma unroll
  for (int m = 0; m < C::M; ++m) {
    const int w = lt + m * C::L;
    const long long s = (long long)t0 + wb - H1 + w;
    float2 v = make_float2(0.f, 0.f);
    if (w < C::W && wb + w < n + H1 && s >= 0) v = __ldg(&x[blk + s]);
    xr[m] = v.x;
    xi[m] = v.y;
  }
#pragma unroll
  for (int k = 0; k < NTR; ++k) {
    const int i = tid + k * THREADS;
    if (i < kBranches * T) taps_s[i] = tr[k];
  }
  if (mask >> kBranches) {
    if (tid == 0) atomicCAS(err, 0u, (unsigned)DF_ECONTROL);
    mask &= (1u << kBranches) - 1;
  }
#pragma unroll
  for (int m = 0; m < C::M; ++m) {
    mg[m] = __fsqrt_rn(__fadd_rn(__fmul_rn(xr[m], xr[m]), __fmul_rn(xi[m], xi[m])));
    sc[m] = 1.0f;
  }
  DPD_TSTAMP(tr_loaded);

  // Branch sum starts at -0.0f, the exact additive identity (-0 + x == x
  // for every x, including +0): the first add reproduces y_b bit for bit,
  // and the final "+ 0.0f" maps an all-zero -0 to the reference's +0.
  float outr[V], outi[V];
#pragma unroll
  for (int j = 0; j < V; ++j) outr[j] = outi[j] = -0.0f;
  constexpr bool fast = FAST;
  if (fast && tile == 0 && mask && H1 > 0)
    dpd_block_history<HALO, THREADS>(ctrl, x, p, mask, period, H1, fs, q_s, hist_s, tid);
  if (!fast && tile == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // history table from prep
  if (C::WL) __syncthreads();  // taps_s (and hist_s) before the first branch
  int prev_b = 1;
  int buf = 0;
  // Window slot of position lt + m*L: pad_index(lt) + m * (L + L/8)
  // (L % 8 == 0), so the stores use immediate offsets.
  static_assert(C::L % 8 == 0, "window padding");
  const int pt = pad_index(lt);
  // Block-start tiles: this thread's history entry for branch b is
  // hb[(b - 1) * H1] (the prep kernel's table, u[-(tid+1)]).
  const bool has_hist = tile == 0 && tid < H1;
  const float2* hb = fast ? hist_s + (has_hist ? tid : 0)
                          : hist + ((size_t)p * kBranches * H1 + (has_hist ? tid : 0));
  const int hslot = pad_index(H1 - 1 - (has_hist ? tid : 0));
#pragma unroll 1
  for (uint32_t bits = mask; bits; bits &= bits - 1) {
    const int b = __ffs(bits);  // ascending branch order
    // scale_b = mag^(b-1) as the reference's repeated product from 1.0f
    // (dpd.cpp:69-71); the first step 1.0f * mag == mag exactly.
#pragma unroll 1
    for (; prev_b < b; ++prev_b) {
#pragma unroll
      for (int m = 0; m < C::M; ++m) sc[m] = __fmul_rn(sc[m], mg[m]);
    }
    float2* u = us[buf];
#pragma unroll
    for (int m = 0; m < C::M; ++m) {
      const int w = lt + m * C::L;
      if (m < C::M - 1 || w < C::W) {
        // b == 1: sc = 1.0f and x * 1.0f == x exactly (no select needed)
        u[pt + m * (C::L + C::L / 8)] = make_float2(__fmul_rn(xr[m], sc[m]), __fmul_rn(xi[m], sc[m]));
      }
    }
    // History before the block start: the branch's frozen FIR state as
    // resolved by the prep kernel (u[-(j+1)] at window index H1-1-j).  It
    // overwrites the zero-padded poly slots 0..H1-1, stored above by other
    // lanes of warp 0: order the two stores (block-start tiles only).
    if (tile == 0) __syncwarp();
    if (has_hist) u[hslot] = hb[(b - 1) * H1];
    if (C::WL)
      __syncwarp();
    else
      __syncthreads();

    // FIR over outputs o = tid*V + j (window index o + k' with k' = T-1-k).
    const float2* tb = taps_s + (b - 1) * T;
    float ar[V], ai[V], wr[V], wi[V];
    const int o0 = lt * V;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float2 v = u[pad_index(o0 + H1 + j)];
      wr[j] = v.x;
      wi[j] = v.y;
    }
    {
      const float2 t = tb[0];
#pragma unroll
      for (int j = 0; j < V; ++j) {  // tap 0 without the leading 0.0f + (see header)
        ar[j] = __fsub_rn(__fmul_rn(t.x, wr[j]), __fmul_rn(t.y, wi[j]));
        ai[j] = __fadd_rn(__fmul_rn(t.x, wi[j]), __fmul_rn(t.y, wr[j]));
      }
    }
#pragma unroll
    for (int k = 1; k < T; ++k) {
      // Slide: window for tap k is u[o0 + H1 - k + j].
#pragma unroll
      for (int j = V - 1; j > 0; --j) {
        wr[j] = wr[j - 1];
        wi[j] = wi[j - 1];
      }
      const float2 v = u[pad_index(o0 + H1 - k)];
      wr[0] = v.x;
      wi[0] = v.y;
      const float2 t = tb[k];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        ar[j] = __fadd_rn(ar[j], __fsub_rn(__fmul_rn(t.x, wr[j]), __fmul_rn(t.y, wi[j])));
        ai[j] = __fadd_rn(ai[j], __fadd_rn(__fmul_rn(t.x, wi[j]), __fmul_rn(t.y, wr[j])));
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
      outr[j] = __fadd_rn(outr[j], ar[j]);
      outi[j] = __fadd_rn(outi[j], ai[j]);
    }
    buf ^= 1;
  }

  // Stage through smem for coalesced stores (reuse the idle buffer).
  DPD_TSTAMP(tr_fir);
  if (C::WL)
    __syncwarp();
  else
    __syncthreads();
  float2* st = us[buf];
#pragma unroll
  for (int j = 0; j < V; ++j)
    st[pad_index(lt * V + j)] = make_float2(__fadd_rn(outr[j], 0.0f), __fadd_rn(outi[j], 0.0f));
  if (C::WL) {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int o = lt + 32 * i;
      if (wb + o < n) y[blk + t0 + wb + o] = st[pad_index(o)];
    }
    DPD_TRACE((unsigned)((blockIdx.x + (unsigned long long)blockIdx.y * gridDim.x) * (THREADS / 32) + (tid >> 5)),
              p * 65536ull + tile * 4 + (tid >> 5), tr_start, tr_loaded, tr_fir);
  } else {
    __syncthreads();
    for (int o = tid; o < n; o += THREADS) y[blk + t0 + o] = st[pad_index(o)];
  }
  // The grid must not complete before the prep grid (which also advances
  // the FirState the next batch's prep reads).  Block-start tiles already
  // waited on it, and every batch has one, so no other CTA needs to: they
  // retire and free their slots while prep may still be running.

  // Only block-start tiles read the carried FirState and last1, so on a
  // plain fast-path firing only they are counted (one per block) and
  // every other CTA retires here without the fence and the atomic; a
  // channel firing counts every CTA, since its commit publishes all outputs.
  const bool counted = io.channel_mode || (fast && (DF_DPD_TAIL_ALL || tile == 0));
  if (counted) {
    // Last counted CTA: advances the FirState (fast path; every block-start
    // tile has read the old one) and commits the firing batch: K control
    // tokens, K block tokens consumed, K block tokens produced (ports always
    // at full rate).
    __shared__ bool last;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const unsigned total = io.channel_mode || DF_DPD_TAIL_ALL ? gridDim.x * gridDim.y
                             : block_major                    ? gridDim.x
                                                              : gridDim.y;
      last = atomicAdd(done_counter, 1u) == total - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    dpd_grid_end<HALO, THREADS>(io, x, period, H1, fast, fs, done_counter, tid);
  }
}

// ---------------------------------------------------------------------------
// One-wave kernel for short fast-path grids (DPD-1: 16 blocks x 64 tiles =
// 1024 CTAs).  The main kernel keeps each thread's window positions (x, |x|,
// scale: 36 registers) live across the branch loop, which caps it at 5 CTAs
// per SM -- 740 slots, so a 1024-tile grid runs a full wave and then a 38 %
// wave at ~2 warps per SM sub-partition.  Here the raw window and |x| live in
// shared memory and each branch rebuilds its poly window from them (scale_b
// = the reference's repeated product from 1.0f, recomputed per position), so
// the kernel fits DF_DPD_WAVE_MINB CTAs per SM and the whole grid is resident
// at once.  Same arithmetic, same op order as dpd_main_kernel (bit-exact).
// ---------------------------------------------------------------------------
#ifndef DF_DPD_WAVE_MINB
#define DF_DPD_WAVE_MINB 7
#endif
#ifndef DF_DPD_WAVE
#define DF_DPD_WAVE 1
#endif
#ifndef DF_DPD_WAVE_PDL
#define DF_DPD_WAVE_PDL 1
#endif
#ifndef DF_DPD_WAVE_ALL
#define DF_DPD_WAVE_ALL 0  // A/B: the shared-memory-window kernel for every T=10 fast-path grid
#endif
#ifndef DF_DPD_WAVE_L2PF
#define DF_DPD_WAVE_L2PF 1
#endif

template <int T, int V, int THREADS, bool HALO>
__global__ void __launch_bounds__(THREADS, DF_DPD_WAVE_MINB)
    dpd_wave_kernel(DpdIO io, const float2* __restrict__ taps_g, unsigned period, unsigned* err,
                    unsigned* done_counter, FastState fs) {
  using C = MainCfg<T, V, THREADS>;
  static_assert(C::WL, "warp-local windows");
  constexpr int H1 = T - 1;
  constexpr int HS = H1 > 0 ? H1 : 1;
  constexpr int NW = THREADS / 32;
  __shared__ float2 taps_s[kBranches * T];
  __shared__ float2 xs_all[NW][C::W];  // raw window
  __shared__ float mg_all[NW][C::W];   // |x| of the window
  __shared__ float2 us_all[NW][C::WP];  // poly window of the current branch (then the output staging)
  __shared__ float2 hist_s[kBranches * HS];
  __shared__ int q_s[kBranches];

  const unsigned long long p = blockIdx.x;  // block-major: block-start tiles dispatch first
  const unsigned tile = blockIdx.y;
  const int tid = threadIdx.x, lt = tid & 31, warp = tid >> 5;
#if DF_DPD_WAVE_PDL
  // Programmatic dependent launch (one-wave grids only: a multi-wave grid's
  // early dependents would sit in its later waves' slots).  The next firing
  // may launch now and becomes resident as this grid's CTAs retire; it
  // stages its taps (written by no kernel) and then waits for this whole
  // grid -- and its memory -- before touching anything a firing produces.
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  constexpr int NTR0 = (kBranches * T + THREADS - 1) / THREADS;
  float2 tr[NTR0];
#pragma unroll
  for (int k = 0; k < NTR0; ++k) {
    const int i = tid + k * THREADS;
    if (i < kBranches * T) tr[k] = __ldg(&taps_g[i]);
  }
#if DF_DPD_WAVE_PDL
  // Raw-mode firings know their input address before the previous grid is
  // done: warm L2 with this tile's window now (a prefetch only fills L2, the
  // point of coherence, so a later write by the previous grid still wins;
  // the loads proper come after the wait).  Channel firings resolve their
  // region from device state the previous grid may still commit.
  if (DF_DPD_WAVE_L2PF && !io.channel_mode && tid == 0) {
    const long long s0 = (long long)blockIdx.y * C::S - (T - 1);
    const long long a = (long long)blockIdx.x * period + (s0 > 0 ? s0 : 0);
    const long long e = (long long)blockIdx.x * period + min((long long)period, (long long)(blockIdx.y + 1) * C::S);
    const uintptr_t lo = reinterpret_cast<uintptr_t>(io.in + a) & ~(uintptr_t)15;
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(io.in + e) + 15) & ~(uintptr_t)15;
    if (hi > lo)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo)) : "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  const uint32_t* ctrl = io_ctrl(io);
  const float2* __restrict__ x = io_in(io);
  float2* __restrict__ y = io_out(io);
  const int wb = warp * C::OW;
  float2* xs = xs_all[warp];
  float* mgs = mg_all[warp];
  float2* u = us_all[warp];
  const unsigned t0 = tile * C::S;
  const int n = (int)min((unsigned)C::S, period - t0);
  const size_t blk = (size_t)p * period;
  constexpr int NTR = NTR0;
  uint32_t mask = ctrl[p];
  {
    float xr[C::M], xi[C::M];
#pragma unroll
    for (int m = 0; m < C::M; ++m) {
      const int w = lt + m * 32;
      const long long s = (long long)t0 + wb - H1 + w;
      float2 v = make_float2(0.f, 0.f);
      if (w < C::W && wb + w < n + H1 && s >= 0) v = __ldg(&x[blk + s]);
      xr[m] = v.x;
      xi[m] = v.y;
    }
#pragma unroll
    for (int k = 0; k < NTR; ++k) {
      const int i = tid + k * THREADS;
      if (i < kBranches * T) taps_s[i] = tr[k];
    }
    if (mask >> kBranches) {
      if (tid == 0) atomicCAS(err, 0u, (unsigned)DF_ECONTROL);
      mask &= (1u << kBranches) - 1;
    }
#pragma unroll
    for (int m = 0; m < C::M; ++m) {
      const int w = lt + m * 32;
      if (m < C::M - 1 || w < C::W) {
        xs[w] = make_float2(xr[m], xi[m]);
        if (mask > 1u) mgs[w] = __fsqrt_rn(__fadd_rn(__fmul_rn(xr[m], xr[m]), __fmul_rn(xi[m], xi[m])));
      }
    }
  }
  float outr[V], outi[V];
#pragma unroll
  for (int j = 0; j < V; ++j) outr[j] = outi[j] = -0.0f;
  if (tile == 0 && mask && H1 > 0) dpd_block_history<HALO, THREADS>(ctrl, x, p, mask, period, H1, fs, q_s, hist_s, tid);
  __syncthreads();  // taps_s, hist_s
  const int pt = pad_index(lt);
  const bool has_hist = tile == 0 && tid < H1;
  const int hslot = pad_index(H1 - 1 - (has_hist ? tid : 0));
#pragma unroll 1
  for (uint32_t bits = mask; bits; bits &= bits - 1) {
    const int b = __ffs(bits);
    // Poly window of branch b: scale_b = ((1*mag)*mag)... (b-1 products,
    // dpd.cpp:69-71), recomputed per position from |x| in shared memory.
#pragma unroll
    for (int m = 0; m < C::M; ++m) {
      const int w = lt + m * 32;
      if (m < C::M - 1 || w < C::W) {
        const float2 v = xs[w];
        float2 o = v;  // b == 1: scale 1.0f, x * 1.0f == x exactly
        if (b > 1) {
          const float g = mgs[w];
          float sc = g;
#pragma unroll 1
          for (int q = 2; q < b; ++q) sc = __fmul_rn(sc, g);
          o = make_float2(__fmul_rn(v.x, sc), __fmul_rn(v.y, sc));
        }
        u[pt + m * 36] = o;
      }
    }
    if (tile == 0) __syncwarp();
    if (has_hist) u[hslot] = hist_s[(b - 1) * H1 + tid];
    __syncwarp();
    const float2* tb = taps_s + (b - 1) * T;
    float ar[V], ai[V], wr[V], wi[V];
    const int o0 = lt * V;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float2 v = u[pad_index(o0 + H1 + j)];
      wr[j] = v.x;
      wi[j] = v.y;
    }
    {
      const float2 t = tb[0];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        ar[j] = __fsub_rn(__fmul_rn(t.x, wr[j]), __fmul_rn(t.y, wi[j]));
        ai[j] = __fadd_rn(__fmul_rn(t.x, wi[j]), __fmul_rn(t.y, wr[j]));
      }
    }
#pragma unroll
    for (int k = 1; k < T; ++k) {
#pragma unroll
      for (int j = V - 1; j > 0; --j) {
        wr[j] = wr[j - 1];
        wi[j] = wi[j - 1];
      }
      const float2 v = u[pad_index(o0 + H1 - k)];
      wr[0] = v.x;
      wi[0] = v.y;
      const float2 t = tb[k];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        ar[j] = __fadd_rn(ar[j], __fsub_rn(__fmul_rn(t.x, wr[j]), __fmul_rn(t.y, wi[j])));
        ai[j] = __fadd_rn(ai[j], __fadd_rn(__fmul_rn(t.x, wi[j]), __fmul_rn(t.y, wr[j])));
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
      outr[j] = __fadd_rn(outr[j], ar[j]);
      outi[j] = __fadd_rn(outi[j], ai[j]);
    }
    __syncwarp();  // the next branch (or the staging) rewrites u
  }
#pragma unroll
  for (int j = 0; j < V; ++j)
    u[pad_index(lt * V + j)] = make_float2(__fadd_rn(outr[j], 0.0f), __fadd_rn(outi[j], 0.0f));
  __syncwarp();
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int o = lt + 32 * i;
    if (wb + o < n) y[blk + t0 + wb + o] = u[pad_index(o)];
  }
  // End of grid: as dpd_main_kernel (block-start tiles counted on plain
  // firings, every CTA on channel firings).
  const bool counted = io.channel_mode || tile == 0;
  if (!counted) return;
  __shared__ bool last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned total = io.channel_mode ? gridDim.x * gridDim.y : gridDim.x;
    last = atomicAdd(done_counter, 1u) == total - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  dpd_grid_end<HALO, THREADS>(io, x, period, H1, true, fs, done_counter, tid);
}

// Generic-T fallback (T not 10/32): simple per-output loop, same op order.
__global__ void dpd_main_generic_kernel(DpdIO io, const float2* __restrict__ taps_g,
                                        const float2* __restrict__ hist, unsigned period, int T,
                                        unsigned* err, unsigned* done_counter) {
  const unsigned long long p = blockIdx.y;
  const uint32_t* ctrl = io_ctrl(io);
  const float2* x = io_in(io);
  float2* y = io_out(io);
  uint32_t mask = ctrl[p];
  if (mask >> kBranches) {
    if (threadIdx.x == 0) atomicCAS(err, 0u, (unsigned)DF_ECONTROL);
    mask &= (1u << kBranches) - 1;
  }
  const int H1 = T - 1;
  const size_t blk = (size_t)p * period;
  for (unsigned o = blockIdx.x * blockDim.x + threadIdx.x; o < period; o += gridDim.x * blockDim.x) {
    float outr = 0.0f, outi = 0.0f;
    for (uint32_t bits = mask; bits; bits &= bits - 1) {
      const int b = __ffs(bits);
      float ar = 0.0f, ai = 0.0f;
      for (int k = 0; k < T; ++k) {
        const long long s = (long long)o - k;
        float2 u;
        if (s >= 0) {
          const float2 v = x[blk + s];
          u = poly_sample(v.x, v.y, b);
        } else {
          u = hist[((size_t)p * kBranches + (b - 1)) * H1 + (size_t)(-s - 1)];
        }
        const float2 t = taps_g[(b - 1) * T + k];
        ar = __fadd_rn(ar, __fsub_rn(__fmul_rn(t.x, u.x), __fmul_rn(t.y, u.y)));
        ai = __fadd_rn(ai, __fadd_rn(__fmul_rn(t.x, u.y), __fmul_rn(t.y, u.x)));
      }
      outr = __fadd_rn(outr, ar);
      outi = __fadd_rn(outi, ai);
    }
    y[blk + o] = make_float2(outr, outi);
  }
  if (io.channel_mode) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(done_counter, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      *done_counter = 0;
      chan_commit_read(io.ctrl_ch, io.ctrl_ch.rate);
      chan_commit_read(io.in_ch, io.in_ch.rate);
      chan_commit_write(io.out_ch, io.out_ch.rate);
    }
  }
}

// History from raw halo samples: branch b's state[j] = poly_b(raw[count-1-j])
// (older state kept for j >= count), as fir10 would leave it.
__global__ void dpd_set_history_kernel(float2* state, const float2* __restrict__ raw, unsigned count,
                                       unsigned mask, int T) {
  const int b = blockIdx.x + 1;
  if (!((mask >> (b - 1)) & 1u)) return;
  const int H1 = T - 1;
  float2* st = state + (size_t)blockIdx.x * (kMaxTaps - 1);
  __shared__ float2 old[kMaxTaps];
  if ((int)threadIdx.x < H1) old[threadIdx.x] = st[threadIdx.x];
  __syncthreads();
  const int j = threadIdx.x;
  if (j < H1) {
    const long long idx = (long long)count - 1 - j;
    st[j] = idx >= 0 ? poly_sample(raw[idx].x, raw[idx].y, b) : old[-idx - 1];
  }
}

__global__ void dpd_config_kernel(const uint16_t* __restrict__ sched, unsigned len,
                                  unsigned long long first, unsigned long long count,
                                  uint32_t* __restrict__ ctrl) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < count;
       i += (unsigned long long)gridDim.x * blockDim.x)
    ctrl[i] = sched[(first + i) % len];  // LE 4-byte wire form (dpd.hpp:38-41)
}

#ifndef DF_DPD_V
#define DF_DPD_V 8
#endif
#ifndef DF_DPD_THREADS
#define DF_DPD_THREADS 128
#endif
#ifndef DF_DPD_FAST
// Fast path for T=10 (bit 0) and T=32 (bit 1).  T=32 keeps the prep kernel:
// its FAST instantiation allocates registers differently and runs DPD-5 5 %
// slower (11.21 vs 10.68 ms, profiles/r01_ab_dpd_variants.txt).
#define DF_DPD_FAST 1
#endif
constexpr int kV = DF_DPD_V;              // consecutive outputs per thread
constexpr int kThreads = DF_DPD_THREADS;  // threads per CTA (tile = kV * kThreads samples)
constexpr unsigned long long kBlockMajorMaxCtas = 4096;  // ~5.5 waves at 5 CTAs/SM

}  // namespace
}  // namespace df

using namespace df;

struct df_dpd {
  int device = 0;
  uint32_t period = 0;
  uint32_t T = 10;
  float2* taps = nullptr;      // device, 10*T
  float2* state = nullptr;     // device, 10*(kMaxTaps-1): FirState per branch
  unsigned resident_ctas = 0;  // main-kernel CTAs resident on the device (prefetch distance)
  unsigned resident_wave_ctas = 0;  // dpd_wave_kernel CTAs resident on the device (one wave)
  const char* last_kernel = "";     // main kernel of the last firing (df_dpd_kernel_name)
  unsigned* scratch = nullptr; // [0] error word, [1] done counter, [4..13] fast-path last1
  float2* hist = nullptr;      // device history table, capacity hist_blocks
  int* act = nullptr;          // device active lists, 10*hist_blocks
  unsigned long long hist_blocks = 0;
  // run_host resources
  void* ctrl_buf = nullptr;
  unsigned long long ctrl_cap = 0;
  uint16_t* sched_dev = nullptr;
  size_t sched_cap = 0;
  std::vector<uint16_t> sched_host;    // schedule the tokens in ctrl_buf were made from
  unsigned long long ctrl_blocks = 0;  // ... their count
  unsigned long long ctrl_first = 0;   // ... and the schedule position of the first
  // Blocks df_dpd_run_host has fired since create / reset: the config
  // actor's firing index (dpd.cpp:208 schedule[firing % len]) continues
  // from here, so a stream split over several calls sees one schedule.
  unsigned long long run_blocks = 0;
  df::Staging staging;  // df_dpd_run_host pipeline
};

namespace {

int ensure_hist(df_dpd* d, unsigned long long K) {
  if (K <= d->hist_blocks) return DF_OK;
  unsigned long long cap = std::max<unsigned long long>(K, 64);
  cudaFree(d->hist);
  cudaFree(d->act);
  d->hist = nullptr;
  d->act = nullptr;
  d->hist_blocks = 0;
  const size_t H1 = std::max<uint32_t>(d->T - 1, 1);
  DF_CHECK_CUDA(cudaMalloc(&d->hist, cap * kBranches * H1 * sizeof(float2)));
  DF_CHECK_CUDA(cudaMalloc(&d->act, cap * kBranches * sizeof(int)));
  d->hist_blocks = cap;
  return DF_OK;
}

bool dpd_fast_path(const df_dpd* d) {
  return ((d->T == 10 && (DF_DPD_FAST & 1)) || (d->T == 32 && (DF_DPD_FAST & 2))) && d->period >= d->T - 1;
}

// htail: optional per-branch halo tails (df_dpd_fire_halo; fast path only).
int launch_dpd(df_dpd* d, const DpdIO& io, unsigned long long K, cudaStream_t s,
               const float2* const* htail = nullptr) {
  if (K == 0) return DF_OK;
  DF_REQUIRE(K <= 0x7fffffffull / 2, DF_EINVAL, "dpd: batch of %llu blocks too large", K);
  DF_TRY(ensure_hist(d, K));
  unsigned* err = d->scratch;
  unsigned* done = d->scratch + 1;
  // Fast path (see the header): T in {10, 32} and blocks at least T-1 long.
  const bool fast = dpd_fast_path(d);
  // (FAST is a template parameter: the prep-path kernel keeps its own code.)
  FastState fs{};
  if (fast) {
    fs.state = d->state;
    fs.last1 = reinterpret_cast<int*>(d->scratch + 4);
    if (htail)
      for (int b = 0; b < kBranches; ++b) fs.htail[b] = htail[b];
  }
  if (d->T > 1 && !fast) {
    dpd_prep_kernel<<<kBranches, 1024, 0, s>>>(io, d->state, d->state, d->hist, d->act, K, d->period,
                                                (int)d->T, err);
    DF_TRY(after_launch("dpd_prep_kernel"));
  }
  const bool one_wave = d->resident_wave_ctas &&
                        K * ((d->period + kThreads * kV - 1) / (kThreads * kV)) <= d->resident_wave_ctas;
  if (fast && d->T == 10 && DF_DPD_WAVE && d->resident_wave_ctas && (one_wave || DF_DPD_WAVE_ALL) &&
      K <= 65535) {
    // Short grid that fits one wave of dpd_wave_kernel (DPD-1).
    const unsigned tiles = (d->period + kThreads * kV - 1) / (kThreads * kV);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)K, tiles);
    lc.blockDim = dim3(kThreads);
    lc.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = DF_DPD_WAVE_PDL && one_wave ? 1 : 0;
    DF_CHECK_CUDA(htail ? cudaLaunchKernelEx(&lc, dpd_wave_kernel<10, kV, kThreads, true>, io, d->taps, d->period,
                                             err, done, fs)
                        : cudaLaunchKernelEx(&lc, dpd_wave_kernel<10, kV, kThreads, false>, io, d->taps, d->period,
                                             err, done, fs));
    d->last_kernel = "dpd_wave_kernel";
    DF_TRY(after_launch("dpd_wave_kernel"));
  } else if (d->T == 10 || d->T == 32) {
    constexpr int S = kThreads * kV;
    const unsigned tiles = (d->period + S - 1) / S;
    DF_REQUIRE(K <= 65535u * 1024u, DF_EINVAL, "dpd: batch too large");
    // blockIdx.y indexes blocks: split very large batches into launches.
    for (unsigned long long base = 0; base < K; base += 65535) {
      const unsigned long long k = std::min<unsigned long long>(65535, K - base);
      DpdIO sub = io;
      if (!io.channel_mode) {
        sub.ctrl = io.ctrl + base;
        sub.in = io.in + base * d->period;
        sub.out = io.out + base * d->period;
      } else {
        DF_REQUIRE(K <= 65535, DF_EINVAL, "dpd: channel firing batch > 65535");
      }
      const float2* hist = d->hist + base * kBranches * (d->T - 1);
      cudaLaunchConfig_t lc{};
      // Block-major only for short grids (a few waves), where the grid's
      // end is the block-start tiles' FirState hand-off: DPD-1 (1024 CTAs)
      // 16.1 -> 14.1 us; DPD-3 (65536 CTAs) is 0.5 % slower block-major
      // (profiles/r01_ab_dpd_variants.txt).
      const unsigned bm =
          fast && DF_DPD_BLOCK_MAJOR && tiles <= 65535u && k * tiles <= kBlockMajorMaxCtas ? 1u : 0u;
      // Next-wave L2 prefetch, also for short grids only: DPD-1 -2.5 %;
      // DPD-3 +0.8 % and DPD-5 +1.6 % (already latency-hidden; A/B in
      // profiles/r01_ab_dpd_variants.txt).
      const unsigned ahead = DF_DPD_PREFETCH && k * tiles <= kBlockMajorMaxCtas ? d->resident_ctas : 0u;
      lc.gridDim = bm ? dim3((unsigned)k, tiles) : dim3(tiles, (unsigned)k);
      lc.blockDim = dim3(kThreads);
      lc.dynamicSmemBytes = 0;
      lc.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = attr;
      lc.numAttrs = fast ? 0 : 1;  // PDL only behind the prep kernel
      const float2* tp = d->taps;
      const bool halo = fast && htail && base == 0;
      cudaError_t le;
      if (d->T == 10)
        le = !fast ? cudaLaunchKernelEx(&lc, dpd_main_kernel<10, kV, kThreads, false, false>, sub, tp, hist, d->period, bm, ahead, err, done, fs)
             : halo ? cudaLaunchKernelEx(&lc, dpd_main_kernel<10, kV, kThreads, true, true>, sub, tp, hist, d->period, bm, ahead, err, done, fs)
                    : cudaLaunchKernelEx(&lc, dpd_main_kernel<10, kV, kThreads, true, false>, sub, tp, hist, d->period, bm, ahead, err, done, fs);
      else
        le = !fast ? cudaLaunchKernelEx(&lc, dpd_main_kernel<32, kV, kThreads, false, false>, sub, tp, hist, d->period, bm, ahead, err, done, fs)
             : halo ? cudaLaunchKernelEx(&lc, dpd_main_kernel<32, kV, kThreads, true, true>, sub, tp, hist, d->period, bm, ahead, err, done, fs)
                    : cudaLaunchKernelEx(&lc, dpd_main_kernel<32, kV, kThreads, true, false>, sub, tp, hist, d->period, bm, ahead, err, done, fs);
      DF_CHECK_CUDA(le);
      d->last_kernel = "dpd_main_kernel";
      DF_TRY(after_launch("dpd_main_kernel"));
      // Later sub-launches continue from the state this one advanced (which
      // already holds the halo of branches it never saw active).
      for (int b = 0; b < kBranches; ++b) fs.htail[b] = nullptr;
    }
  } else {
    for (unsigned long long base = 0; base < K; base += 65535) {
      const unsigned long long k = std::min<unsigned long long>(65535, K - base);
      DpdIO sub = io;
      if (!io.channel_mode) {
        sub.ctrl = io.ctrl + base;
        sub.in = io.in + base * d->period;
        sub.out = io.out + base * d->period;
      }
      const float2* hist = d->hist + base * kBranches * std::max<uint32_t>(d->T - 1, 1);
      dim3 grid(std::min<unsigned>((d->period + 255) / 256, 64), (unsigned)k);
      dpd_main_generic_kernel<<<grid, 256, 0, s>>>(sub, d->taps, hist, d->period, (int)d->T, err, done);
      d->last_kernel = "dpd_main_generic_kernel";
      DF_TRY(after_launch("dpd_main_generic_kernel"));
    }
  }
  return DF_OK;
}

}  // namespace

extern "C" {

int df_dpd_create(int device, uint32_t period, uint32_t T, const float* taps_host, df_dpd** out) {
  DF_REQUIRE(out, DF_EINVAL, "df_dpd_create: null out pointer");
  *out = nullptr;
  DF_REQUIRE(period >= 1, DF_EINVAL, "dpd: period must be >= 1");  // dpd.cpp:152-154
  DF_REQUIRE(T >= 1 && T <= kMaxTaps, DF_EINVAL, "dpd: taps per branch %u outside [1,%d]", T, kMaxTaps);
  DF_REQUIRE(taps_host, DF_EINVAL, "dpd: null taps");
  DF_CHECK_CUDA(cudaSetDevice(device));
  auto* d = new df_dpd();
  d->device = device;
  d->period = period;
  d->T = T;
  cudaError_t e = cudaMalloc(&d->taps, sizeof(float2) * kBranches * T);
  if (e == cudaSuccess) e = cudaMalloc(&d->state, sizeof(float2) * kBranches * (kMaxTaps - 1));
  if (e == cudaSuccess) e = cudaMalloc(&d->scratch, 64);
  if (e == cudaSuccess) e = cudaMemcpy(d->taps, taps_host, sizeof(float2) * kBranches * T, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(d->state, 0, sizeof(float2) * kBranches * (kMaxTaps - 1));
  if (e == cudaSuccess) e = cudaMemset(d->scratch, 0, 64);
  if (e == cudaSuccess && (T == 10 || T == 32)) {  // resident main-kernel CTAs: the L2 prefetch distance
    int per_sm = 0, sms = 0;
    e = T == 10 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dpd_main_kernel<10, kV, kThreads, true, false>,
                                                                kThreads, 0)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dpd_main_kernel<32, kV, kThreads, false, false>,
                                                                kThreads, 0);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    d->resident_ctas = (unsigned)(per_sm * sms);
    int per_sm_wave = 0;
    if (e == cudaSuccess && T == 10)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_wave, dpd_wave_kernel<10, kV, kThreads, false>,
                                                        kThreads, 0);
    d->resident_wave_ctas = (unsigned)(per_sm_wave * sms);
  }
  if (e != cudaSuccess) {
    int rc = cuda_status(e, "df_dpd_create");
    cudaFree(d->taps);
    cudaFree(d->state);
    cudaFree(d->scratch);
    delete d;
    return rc;
  }
  *out = d;
  return DF_OK;
}

int df_dpd_destroy(df_dpd* d) {
  if (!d) return DF_OK;
  cudaSetDevice(d->device);
  cudaFree(d->taps);
  cudaFree(d->state);
  cudaFree(d->scratch);
  cudaFree(d->hist);
  cudaFree(d->act);
  cudaFree(d->ctrl_buf);
  cudaFree(d->sched_dev);
  d->staging.release();
  delete d;
  return DF_OK;
}

int df_dpd_set_taps(df_dpd* d, const float* taps_host, void* stream) {
  DF_REQUIRE(d && taps_host, DF_EINVAL, "df_dpd_set_taps: null argument");
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  DF_CHECK_CUDA(cudaMemcpyAsync(d->taps, taps_host, sizeof(float2) * kBranches * d->T,
                                cudaMemcpyHostToDevice, as_stream(stream)));
  DF_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return DF_OK;
}

const char* df_dpd_kernel_name(const df_dpd* d) { return d ? d->last_kernel : ""; }

int df_dpd_reset(df_dpd* d, void* stream) {
  DF_REQUIRE(d, DF_EINVAL, "df_dpd_reset: null actor");
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  DF_CHECK_CUDA(cudaMemsetAsync(d->state, 0, sizeof(float2) * kBranches * (kMaxTaps - 1), as_stream(stream)));
  DF_CHECK_CUDA(cudaMemsetAsync(d->scratch, 0, 64, as_stream(stream)));
  d->run_blocks = 0;
  return DF_OK;
}

int df_dpd_get_state(df_dpd* d, float* state_host) {
  DF_REQUIRE(d && state_host, DF_EINVAL, "df_dpd_get_state: null argument");
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  DF_CHECK_CUDA(cudaDeviceSynchronize());
  std::vector<float2> st((size_t)kBranches * (kMaxTaps - 1));
  DF_CHECK_CUDA(cudaMemcpy(st.data(), d->state, st.size() * sizeof(float2), cudaMemcpyDeviceToHost));
  const uint32_t H1 = d->T - 1;
  for (int b = 0; b < kBranches; ++b)
    for (uint32_t j = 0; j < H1; ++j) {
      state_host[2 * (b * H1 + j)] = st[b * (kMaxTaps - 1) + j].x;
      state_host[2 * (b * H1 + j) + 1] = st[b * (kMaxTaps - 1) + j].y;
    }
  return DF_OK;
}

int df_dpd_error(df_dpd* d) {
  DF_REQUIRE(d, DF_EINVAL, "df_dpd_error: null actor");
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  DF_CHECK_CUDA(cudaDeviceSynchronize());
  unsigned err = 0;
  DF_CHECK_CUDA(cudaMemcpy(&err, d->scratch, sizeof err, cudaMemcpyDeviceToHost));
  if (err == DF_ECONTROL) return set_error(DF_ECONTROL, "config token names a branch beyond 10");
  if (err) return set_error((int)err, "dpd: device error %u", err);
  return DF_OK;
}

int df_dpd_set_history(df_dpd* d, const float* raw_dev, uint32_t count, uint32_t branch_mask, void* stream) {
  DF_REQUIRE(d, DF_EINVAL, "df_dpd_set_history: null actor");
  DF_REQUIRE(branch_mask >> kBranches == 0, DF_ECONTROL, "config token names a branch beyond 10");
  if (d->T <= 1 || count == 0 || branch_mask == 0) return DF_OK;
  DF_REQUIRE(raw_dev, DF_EINVAL, "df_dpd_set_history: null samples");
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  dpd_set_history_kernel<<<kBranches, 32, 0, as_stream(stream)>>>(d->state, reinterpret_cast<const float2*>(raw_dev),
                                                                   count, branch_mask, (int)d->T);
  return after_launch("dpd_set_history_kernel");
}

#ifdef DF_DPD_TRACE
// Probe builds only: copies out (and clears) the trace slots.
int df_debug_dpd_trace(unsigned long long* host, unsigned* count) {
  DF_CHECK_CUDA(cudaDeviceSynchronize());
  if (host) DF_CHECK_CUDA(cudaMemcpyFromSymbol(host, g_dpd_trace, (8ull << 15) * 8));
  *count = 1u << 15;
  static std::vector<unsigned long long> zeros(8 << 15);
  DF_CHECK_CUDA(cudaMemcpyToSymbol(g_dpd_trace, zeros.data(), (8ull << 15) * 8));
  return DF_OK;
}
#endif

int df_dpd_fire(df_dpd* d, const uint32_t* ctrl_dev, const float* in_dev, float* out_dev,
                uint64_t blocks, void* stream) {
  DF_REQUIRE(d, DF_EINVAL, "df_dpd_fire: null actor");
  if (blocks == 0) return DF_OK;
  DF_REQUIRE(ctrl_dev && in_dev && out_dev, DF_EINVAL, "df_dpd_fire: null buffer");
  DF_REQUIRE(in_dev != out_dev, DF_EINVAL, "df_dpd_fire: in-place firing is not supported");
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  DpdIO io{};
  io.ctrl = ctrl_dev;
  io.in = reinterpret_cast<const float2*>(in_dev);
  io.out = reinterpret_cast<float2*>(out_dev);
  io.channel_mode = 0;
  return launch_dpd(d, io, blocks, as_stream(stream));
}

int df_dpd_fire_halo(df_dpd* d, const float* const* halo_tails, const uint32_t* ctrl_dev, const float* in_dev,
                     float* out_dev, uint64_t blocks, void* stream) {
  DF_REQUIRE(d, DF_EINVAL, "df_dpd_fire_halo: null actor");
  if (blocks == 0) return DF_OK;
  DF_REQUIRE(halo_tails && ctrl_dev && in_dev && out_dev, DF_EINVAL, "df_dpd_fire_halo: null argument");
  DF_REQUIRE(in_dev != out_dev, DF_EINVAL, "df_dpd_fire_halo: in-place firing is not supported");
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  if (d->T <= 1) return df_dpd_fire(d, ctrl_dev, in_dev, out_dev, blocks, stream);
  if (!dpd_fast_path(d)) {  // prep path: set the histories, then fire
    for (int b = 0; b < kBranches; ++b)
      if (halo_tails[b]) DF_TRY(df_dpd_set_history(d, halo_tails[b], d->T - 1, 1u << b, stream));
    return df_dpd_fire(d, ctrl_dev, in_dev, out_dev, blocks, stream);
  }
  const float2* ht[kBranches];
  for (int b = 0; b < kBranches; ++b) ht[b] = reinterpret_cast<const float2*>(halo_tails[b]);
  DpdIO io{};
  io.ctrl = ctrl_dev;
  io.in = reinterpret_cast<const float2*>(in_dev);
  io.out = reinterpret_cast<float2*>(out_dev);
  io.channel_mode = 0;
  return launch_dpd(d, io, blocks, as_stream(stream), ht);
}

int df_dpd_fire_channels(df_dpd* d, df_channel* ctrl, df_channel* in, df_channel* out,
                         uint32_t firings, void* stream) {
  DF_REQUIRE(d && ctrl && in && out, DF_EINVAL, "df_dpd_fire_channels: null argument");
  if (firings == 0) return DF_OK;
  DF_REQUIRE(ctrl->token_size == 4 && ctrl->rate == firings, DF_ELOGIC,
             "dpd: control channel must carry 4-byte tokens at rate %u", firings);
  DF_REQUIRE(in->token_size == (size_t)d->period * 8 && in->rate == firings, DF_ELOGIC,
             "dpd: input channel token must be one period (%u samples) at rate %u", d->period, firings);
  DF_REQUIRE(out->token_size == (size_t)d->period * 8 && out->rate == firings, DF_ELOGIC,
             "dpd: output channel token must be one period at rate %u", firings);
  DF_REQUIRE(!ctrl->has_delay, DF_ELOGIC, "delay token on a channel into a control port");
  for (df_channel* c : {ctrl, in}) {
    DF_REQUIRE(c->reader != Endpoint::host, DF_ELOGIC, "dpd: input endpoint is host-driven");
    c->reader = Endpoint::device;
  }
  DF_REQUIRE(out->writer != Endpoint::host, DF_ELOGIC, "dpd: output endpoint is host-driven");
  out->writer = Endpoint::device;
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  DpdIO io{};
  io.channel_mode = 1;
  io.ctrl_ch = ctrl->dev();
  io.in_ch = in->dev();
  io.out_ch = out->dev();
  return launch_dpd(d, io, firings, as_stream(stream));
}

int df_dpd_config_tokens(int device, const uint16_t* schedule_host, size_t len, uint64_t first,
                         uint64_t count, uint32_t* ctrl_dev, void* stream) {
  DF_REQUIRE(schedule_host && len > 0, DF_EINVAL, "dpd: schedule must not be empty");
  if (count == 0) return DF_OK;
  DF_CHECK_CUDA(cudaSetDevice(device));
  uint16_t* sd = nullptr;
  DF_CHECK_CUDA(cudaMallocAsync(&sd, len * sizeof(uint16_t), as_stream(stream)));
  DF_CHECK_CUDA(cudaMemcpyAsync(sd, schedule_host, len * sizeof(uint16_t), cudaMemcpyHostToDevice,
                                as_stream(stream)));
  const unsigned blocks = (unsigned)std::min<uint64_t>((count + 255) / 256, 1184);
  dpd_config_kernel<<<blocks, 256, 0, as_stream(stream)>>>(sd, (unsigned)len, first, count, ctrl_dev);
  int rc = after_launch("dpd_config_kernel");
  DF_CHECK_CUDA(cudaFreeAsync(sd, as_stream(stream)));
  return rc;
}

int df_dpd_run_host(df_dpd* d, const float* in_host, float* out_host, uint64_t samples,
                    const uint16_t* schedule_host, size_t schedule_len, uint64_t chunk_blocks,
                    void* stream) {
  DF_REQUIRE(d && in_host && out_host, DF_EINVAL, "df_dpd_run_host: null argument");
  DF_REQUIRE(schedule_host && schedule_len > 0, DF_EINVAL, "dpd: schedule must not be empty");
  DF_REQUIRE(samples % d->period == 0, DF_EINVAL,
             "dpd: sample count must be a multiple of the period");
  if (samples == 0) return DF_OK;
  DF_CHECK_CUDA(cudaSetDevice(d->device));
  const uint64_t blocks = samples / d->period;
  if (chunk_blocks == 0) chunk_blocks = df::Staging::chunk_units(blocks, 8ull * d->period, 128ull << 20);
  chunk_blocks = std::min(chunk_blocks, blocks);
  const size_t chunk_bytes = chunk_blocks * d->period * 8ull;
  cudaStream_t cs = as_stream(stream);
  DF_TRY(d->staging.ensure(chunk_bytes, chunk_bytes));
  if (blocks > d->ctrl_cap) {
    DF_CHECK_CUDA(cudaDeviceSynchronize());
    cudaFree(d->ctrl_buf);
    d->ctrl_buf = nullptr;
    d->ctrl_blocks = 0;
    DF_CHECK_CUDA(cudaMalloc(&d->ctrl_buf, blocks * sizeof(uint32_t)));
    d->ctrl_cap = blocks;
  }
  if (schedule_len > d->sched_cap) {
    DF_CHECK_CUDA(cudaDeviceSynchronize());
    cudaFree(d->sched_dev);
    d->sched_dev = nullptr;
    DF_CHECK_CUDA(cudaMalloc(&d->sched_dev, schedule_len * sizeof(uint16_t)));
    d->sched_cap = schedule_len;
  }
  uint32_t* ctrl = static_cast<uint32_t*>(d->ctrl_buf);
  // Config actor: one control token per block, on device, continuing the
  // schedule from the blocks earlier calls fired.  A stream of runs with the
  // same schedule, length and schedule position reuses the tokens in HBM.
  const unsigned long long first = d->run_blocks % schedule_len;
  const bool same = d->ctrl_blocks == blocks && d->ctrl_first == first &&
                    d->sched_host.size() == schedule_len &&
                    std::memcmp(d->sched_host.data(), schedule_host, schedule_len * sizeof(uint16_t)) == 0;
  if (!same) {
    DF_CHECK_CUDA(cudaMemcpyAsync(d->sched_dev, schedule_host, schedule_len * sizeof(uint16_t),
                                  cudaMemcpyHostToDevice, cs));
    dpd_config_kernel<<<(unsigned)std::min<uint64_t>((blocks + 255) / 256, 1184), 256, 0, cs>>>(
        d->sched_dev, (unsigned)schedule_len, first, blocks, ctrl);
    DF_TRY(after_launch("dpd_config_kernel"));
    d->sched_host.assign(schedule_host, schedule_host + schedule_len);
    d->ctrl_blocks = blocks;
    d->ctrl_first = first;
  }
  d->run_blocks += blocks;
  const uint64_t nchunks = (blocks + chunk_blocks - 1) / chunk_blocks;
  auto nb = [&](uint64_t c) { return std::min(chunk_blocks, blocks - c * chunk_blocks); };
  return d->staging.pipeline(
      cs, nchunks,
      [&](uint64_t c, const void*& p, size_t& b) {
        p = in_host + 2 * c * chunk_blocks * d->period;
        b = nb(c) * d->period * 8ull;
      },
      [&](uint64_t c, void*& p, size_t& b) {
        p = out_host + 2 * c * chunk_blocks * d->period;
        b = nb(c) * d->period * 8ull;
      },
      [&](uint64_t c, unsigned char* din, unsigned char* dout) {
        DpdIO io{};
        io.ctrl = ctrl + c * chunk_blocks;
        io.in = reinterpret_cast<const float2*>(din);
        io.out = reinterpret_cast<float2*>(dout);
        return launch_dpd(d, io, nb(c), cs);
      });
}

}  // extern "C"
