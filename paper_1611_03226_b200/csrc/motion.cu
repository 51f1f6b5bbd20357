// motion.cu -- the motion-detection actor chain on sm_100a.
//
// Replaces the reference's gauss -> thres -> med actors
// (proj/src/motion.cpp:144-176) and their kernels gauss5x5 / thres_diff /
// median5 (:27-74) with ONE fused kernel per firing; the gauss -> thres
// "prev" channel with its delay token (:131, :153) becomes a gauss frame
// carried on chip between consecutive frames and, between firings, a
// device-resident delay token.  Extension: RGB input converted in the same
// kernel (gray = (77R + 150G + 29B + 128) >> 8, BT.601 integer luma).
//
// Byte-exact arithmetic, packed SIMD (HBM-bound target: 4 B/px):
//   gray   6 x IDP.4A per 4 px (weights 77/150/29, +128 in the accumulator)
//   gauss  horizontal 5-tap [1 4 6 4 1] with IDP.4A on the packed gray
//          bytes (2 per px), vertical on 16x2 packed lanes (max 65408 <
//          2^16, +128 folded into the first add), (acc+128)>>8 by byte
//          selection -- identical to motion.cpp:38-45 for every pixel
//   thres  VABSDIFF4, then a SWAR byte compare d > thr (exact for all thr)
//   median the thresholded map is binary, so the plus-shaped median of 5
//          (motion.cpp:68-71) is a bitwise majority-of-5 on byte lanes
//   out    0/255 bytes by PRMT sign replication
// Borders follow the reference exactly: gauss copies gray for the 2-px
// frame border (:34-37), median copies the threshold map for the 1-px
// border (:64-67), thres runs everywhere.
//
// Work decomposition: one warp owns a column tile (32 lanes x 8 px, lanes
// 1..30 produce output, lanes 0/31 are the horizontal halo) of a band of
// R rows, and walks a range of frames (temporal walk): gauss(prev) for its
// band lives in shared memory, so every input byte is read once per frame
// (+ vertical/horizontal halo re-reads, which hit L2).  Frame ranges that do
// not start the firing recompute gauss(f0-1) once.  No __syncthreads: warps
// are independent; neighbours are exchanged with shuffles.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "channel_dev.cuh"
#include "channel_host.hpp"
#include "common.cuh"
#include "staging.cuh"

namespace df {
namespace {

#ifndef DF_MOTION_R
#define DF_MOTION_R 48
#endif
#ifndef DF_MOTION_PF
#define DF_MOTION_PF 8
#endif
#ifndef DF_MOTION_MINB
#define DF_MOTION_MINB 14
#endif
constexpr int kBandRows = DF_MOTION_R;    // R (A/B: profiles/r01_ab_motion_variants.txt)
constexpr int kWarpsPerCta = 1;  // y0 depends on blockIdx only: warp-uniform for the compiler
constexpr int kPxPerLane = 8;
constexpr int kOutPxPerWarp = 30 * kPxPerLane;  // 240

struct MotionIO {
  const unsigned char* in;      // frames (raw mode)
  unsigned char* out;
  const unsigned char* prev;    // delay token in (gauss frame)
  unsigned char* next;          // delay token out (gauss frame)
  unsigned char* next_copy;     // Fig. 2 phase-2 duplicate (slot 0) or null
  const unsigned char* halo;    // raw mode: previous input frame replacing the delay token, or null
  DevChan in_ch, out_ch, delay_ch;
  int channel_mode;
};

struct MotionGeom {
  int W, H;
  int frames;        // frames in this firing
  int chunk;         // frames per temporal chunk
  unsigned thr_k;    // SWAR constant
  unsigned thr_sel;  // 0xFFFFFFFF if thr <= 127 else 0
  // IDP.4A weight words, passed as kernel parameters so every dp4a takes
  // its weights straight from the constant bank (no per-step UMOVs).
  unsigned wg[6];    // gray
  unsigned wh[8];    // horizontal gauss
  int l2hint;        // M3: L2 eviction hints on band-halo rows (large frames)
  int m3_chunks, m3_bands;  // M3: warp task t -> chunk t % chunks, band (t / chunks) % bands, tile
};


__device__ __forceinline__ unsigned dp4a(unsigned a, unsigned b, unsigned c) {
  return __dp4a(a, b, c);
}
__device__ __forceinline__ unsigned prmt(unsigned a, unsigned b, unsigned s) {
  unsigned d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}
__device__ __forceinline__ unsigned lop_maj(unsigned a, unsigned b, unsigned c) {
  unsigned d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ unsigned lop_or3(unsigned a, unsigned b, unsigned c) {
  unsigned d;
  asm("lop3.b32 %0, %1, %2, %3, 0xFE;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ unsigned lop_and3(unsigned a, unsigned b, unsigned c) {
  unsigned d;
  asm("lop3.b32 %0, %1, %2, %3, 0x80;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// s ? a : b  (bitwise select)
__device__ __forceinline__ unsigned lop_sel(unsigned s, unsigned a, unsigned b) {
  unsigned d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(d) : "r"(a), "r"(s), "r"(b));
  return d;
}

__device__ __forceinline__ uint2 ldg_pinned(const unsigned char* p) {
  uint2 v;
  asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

constexpr unsigned W8(unsigned a, unsigned b, unsigned c, unsigned d) {
  return a | (b << 8) | (c << 16) | (d << 24);
}

// 4 gray bytes from 12 interleaved RGB bytes (w0,w1,w2 little endian).
// wg = {W8(77,150,29,0), W8(150,29,0,0), W8(0,0,0,77), W8(29,0,0,0),
//       W8(0,0,77,150), W8(0,77,150,29)}.
__device__ __forceinline__ unsigned rgb4_to_gray(unsigned w0, unsigned w1, unsigned w2, const unsigned* wg) {
  const unsigned r0 = dp4a(w0, wg[0], 128u);
  const unsigned r1 = dp4a(w1, wg[1], dp4a(w0, wg[2], 128u));
  const unsigned r2 = dp4a(w2, wg[3], dp4a(w1, wg[4], 128u));
  const unsigned r3 = dp4a(w2, wg[5], 128u);
  const unsigned lo = prmt(r0, r1, 0x0051);  // bytes [r0.b1, r1.b1]
  const unsigned hi = prmt(r2, r3, 0x0051);
  return prmt(lo, hi, 0x5410);
}

__device__ __forceinline__ unsigned pack16x2(unsigned lo, unsigned hi) {
  unsigned d;  // hi * 65536 + lo on the FMA pipe (keeps the ALU pipe for LOP3/PRMT)
  asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(d) : "r"(hi), "r"(lo));
  return d;
}

// Horizontal [1 4 6 4 1] over 4 px of word C with neighbours L (left word)
// and R (right word): two 16x2 packed pair words.  Each sum carries a +8
// bias (dp4a accumulator): the vertical weights sum to 16, so the bias
// adds exactly the +128 of (acc + 128) >> 8 (motion.cpp:45).
// wh = {W8(0,0,1,4), W8(6,4,1,0), W8(0,0,0,1), W8(4,6,4,1), W8(1,4,6,4),
//       W8(1,0,0,0), W8(0,1,4,6), W8(4,1,0,0)}.
__device__ __forceinline__ void hgauss4(unsigned L, unsigned C, unsigned R, unsigned& p01,
                                        unsigned& p23, const unsigned* wh) {
  const unsigned h0 = dp4a(L, wh[0], dp4a(C, wh[1], 8u));
  const unsigned h1 = dp4a(L, wh[2], dp4a(C, wh[3], 8u));
  const unsigned h2 = dp4a(C, wh[4], dp4a(R, wh[5], 8u));
  const unsigned h3 = dp4a(C, wh[6], dp4a(R, wh[7], 8u));
  p01 = pack16x2(h0, h1);
  p23 = pack16x2(h2, h3);
}

// Vertical [1 4 6 4 1] on 16x2 lanes (the +128 rides in the h bias);
// max 16 * (4080 + 8) = 65408 < 2^16, so lanes never carry.
// M3's vertical gauss written as mad.lo (see vgauss_fma).
#ifndef DF_MOTION_VGAUSS_MAD
#define DF_MOTION_VGAUSS_MAD 1
#endif
__device__ __forceinline__ unsigned mad_u32(unsigned a, unsigned b, unsigned c) {
  unsigned d;  // a * b + c on the FMA pipe
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ unsigned vgauss(unsigned a, unsigned b, unsigned c, unsigned d,
                                          unsigned e) {
  const unsigned B = b + d;
  return c * 6u + (B * 4u + (a + e));
}
// The same sum written as four mad.lo (M3).  ptxas keeps some as IMAD (FMA
// pipe) and turns others into IADD3/LEA; this mix measured faster than both
// the plain form and all-IMAD (multipliers from the constant bank, which
// ptxas cannot strength-reduce): profiles/r02_ab_motion_issue.txt.
__device__ __forceinline__ unsigned vgauss_fma(unsigned a, unsigned b, unsigned c, unsigned d, unsigned e) {
#if DF_MOTION_VGAUSS_MAD
  return mad_u32(c, 6u, mad_u32(mad_u32(b, 1u, d), 4u, mad_u32(a, 1u, e)));
#else
  return vgauss(a, b, c, d, e);
#endif
}

// |cur - prev| > thr per byte -> flag in bit 7 (other bits don't-care).
__device__ __forceinline__ unsigned thres4(unsigned cur, unsigned prev, const MotionGeom& g) {
  const unsigned d = __vabsdiffu4(cur, prev);
  const unsigned t = (d & 0x7F7F7F7Fu) + g.thr_k;
  return lop_maj(t, d, g.thr_sel);
}

__device__ __forceinline__ unsigned lop_xor3(unsigned a, unsigned b, unsigned c) {
  unsigned d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Majority of 5 (bitwise): centre c, up u, down d, left l, right r, in 5
// LOP3: a full adder of (c, u, d) gives the count 2*s1 + s0, and the count
// plus l + r reaches 3 iff s1 ? (s0 | l | r) : (s0 & l & r).  (The select
// over any/majority/all of (c, u, d) by (l, r) takes 6; A/B in
// profiles/r01_ab_motion_variants.txt.)
__device__ __forceinline__ unsigned maj5(unsigned c, unsigned u, unsigned d, unsigned l,
                                         unsigned r) {
  const unsigned s0 = lop_xor3(c, u, d);
  const unsigned s1 = lop_maj(c, u, d);
  return lop_sel(s1, lop_or3(s0, l, r), lop_and3(s0, l, r));
}

// --- row I/O -----------------------------------------------------------
// One row slot of the 5-row rolling window.  It also carries the raw loads
// of the row 5 below (software prefetch riding the window rotation: slot k
// is refilled with row r+5 exactly when row r leaves the window).
template <int FMT>
struct RowSlot {
  unsigned h[4];   // horizontal sums, 16x2 packed: px (0,1), (2,3), (4,5), (6,7)
  unsigned g[2];   // gray words
  unsigned t[2];   // threshold flags (bit 7 per byte) once computed
  uint2 raw[FMT == DF_MOTION_RGB ? 3 : 1];  // prefetched input of row (this + 5)
  int raw_y;       // row index of raw (uniform)
};


// Issues the loads of row y into r.raw (FAST: aligned vector loads; the
// values are consumed five rows later).  The row index is clamped into the
// frame (warp-uniform), out-of-frame lanes read a clamped column; both are
// zeroed at conversion.
template <int FMT, bool FAST>
__device__ __forceinline__ void fetch_row(RowSlot<FMT>& r, const unsigned char* __restrict__ frame,
                                          unsigned lane_off, int y, int H, unsigned row_bytes) {
  r.raw_y = y;
  if (!FAST) return;
  const unsigned yc = (unsigned)min(max(y, 0), H - 1);
  const uint2* p = reinterpret_cast<const uint2*>(frame + (yc * row_bytes + lane_off));
  if (FMT == DF_MOTION_RGB) {
    r.raw[0] = __ldg(p);
    r.raw[1] = __ldg(p + 1);
    r.raw[2] = __ldg(p + 2);
  } else {
    r.raw[0] = __ldg(p);
  }
}

template <int FMT, bool FAST>
__device__ __forceinline__ void convert_row(const RowSlot<FMT>& r, const unsigned char* __restrict__ frame,
                                            int x, bool lane_in, int W, int H, unsigned& g0, unsigned& g1,
                                            const unsigned* wg) {
  const int y = r.raw_y;
  if (FAST) {
    const bool ok = lane_in && (unsigned)y < (unsigned)H;
    if (FMT == DF_MOTION_RGB) {
      g0 = rgb4_to_gray(r.raw[0].x, r.raw[0].y, r.raw[1].x, wg);
      g1 = rgb4_to_gray(r.raw[1].y, r.raw[2].x, r.raw[2].y, wg);
    } else {
      g0 = r.raw[0].x;
      g1 = r.raw[0].y;
    }
    g0 = ok ? g0 : 0u;
    g1 = ok ? g1 : 0u;
  } else {
    unsigned char px[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int xi = x + i;
      unsigned char v = 0;
      if (y >= 0 && y < H && xi >= 0 && xi < W) {
        if (FMT == DF_MOTION_RGB) {
          const unsigned char* q = frame + ((size_t)y * W + xi) * 3;
          v = (unsigned char)((77u * q[0] + 150u * q[1] + 29u * q[2] + 128u) >> 8);
        } else {
          v = frame[(size_t)y * W + xi];
        }
      }
      px[i] = v;
    }
    g0 = W8(px[0], px[1], px[2], px[3]);
    g1 = W8(px[4], px[5], px[6], px[7]);
  }
}

template <bool FAST>
__device__ __forceinline__ void load_bytes8(const unsigned char* __restrict__ plane, int y, int x,
                                            int W, int H, unsigned& a0, unsigned& a1) {
  a0 = a1 = 0;
  if (y < 0 || y >= H || x >= W || x + kPxPerLane <= 0) return;
  if (FAST) {
    const uint2 a = *reinterpret_cast<const uint2*>(plane + ((unsigned)y * (unsigned)W + (unsigned)x));
    a0 = a.x;
    a1 = a.y;
  } else {
    unsigned char px[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int xi = x + i;
      px[i] = (xi >= 0 && xi < W) ? plane[(size_t)y * W + xi] : 0;
    }
    a0 = W8(px[0], px[1], px[2], px[3]);
    a1 = W8(px[4], px[5], px[6], px[7]);
  }
}

template <bool FAST>
__device__ __forceinline__ void store_bytes8(unsigned char* __restrict__ plane, int y, int x, int W,
                                             unsigned a0, unsigned a1) {
  if (FAST) {
    // W % 8 == 0: an 8-px segment is entirely inside or entirely outside.
    if (x >= 0 && x < W)
      *reinterpret_cast<uint2*>(plane + ((unsigned)y * (unsigned)W + (unsigned)x)) = make_uint2(a0, a1);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int xi = x + i;
      if (xi >= 0 && xi < W) plane[(size_t)y * W + xi] = (unsigned char)((i < 4 ? a0 : a1) >> (8 * (i & 3)));
    }
  }
}

// Byte masks (0xFF per byte) of columns in the gauss border (x < 2 or
// x >= W-2) and the median border (x == 0 or x == W-1).
template <int WPL = 2>
__device__ __forceinline__ void column_masks(int x, int W, unsigned gm[WPL], unsigned mm[WPL]) {
#pragma unroll
  for (int w = 0; w < WPL; ++w) {
    unsigned a = 0, b = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int xi = x + 4 * w + i;
      if (xi < 2 || xi >= W - 2) a |= 0xFFu << (8 * i);
      if (xi == 0 || xi == W - 1) b |= 0xFFu << (8 * i);
    }
    gm[w] = a;
    mm[w] = b;
  }
}

// Processes one frame for this warp's (tile, band).  MODE 0: gauss only,
// into the prev buffer (warm-up of a frame range).  MODE 1: full chain.
// MODE 2: full chain + writes the next delay token (last frame of a firing).
// INT: interior band (FAST only) -- every row the pass touches, including
// the 5-row-ahead prefetch, lies inside the frame and no gauss/median row is
// a border row, so the pass runs with pointer-increment addressing and no
// row clamps, lane zeroing or border tests (interior_band()).
template <int FMT, bool FAST, int MODE, bool INT>
__device__ __forceinline__ void frame_pass(const unsigned char* __restrict__ frame,
                                           unsigned char* __restrict__ out,
                                           unsigned char* __restrict__ next_tok,
                                           unsigned char* __restrict__ next_copy,
                                           uint2* __restrict__ prev_s, const MotionGeom& g, int y0,
                                           int x, int xc, bool lane_in, int lane, const unsigned gm[2],
                                           const unsigned mm[2]) {
  static_assert(!INT || FAST, "interior passes need aligned 8-px segments");
  const int W = g.W, H = g.H;
  const bool out_lane = lane >= 1 && lane <= 30;
  const unsigned row_bytes = (unsigned)W * FMT;  // a frame is < 4 GiB (checked at create)
  const unsigned lane_off = (unsigned)xc * FMT;
  RowSlot<FMT> s[5];
  // INT: next row to prefetch, next output row, next prev_s row.
  const unsigned char* fptr = INT ? frame + ((size_t)(unsigned)(y0 - 3) * row_bytes + lane_off) : nullptr;
  unsigned ooff = (unsigned)y0 * (unsigned)W + (unsigned)x;  // INT: next output row (a frame is < 4 GiB)

  auto fetch = [&](RowSlot<FMT>& r, int y) {
    if (INT) {
      // volatile: keeps each row's loads in its own step (5 rows ahead of
      // use) instead of being sunk to the loop latch.
      r.raw[0] = ldg_pinned(fptr);
      if (FMT == DF_MOTION_RGB) {
        r.raw[1] = ldg_pinned(fptr + 8);
        r.raw[2] = ldg_pinned(fptr + 16);
      }
      fptr += row_bytes;
      if (DF_MOTION_PF > 0) {
        // L2 prefetch DF_MOTION_PF rows further (clamped into the frame):
        // more bytes in flight than the five register-held rows allow.
        const unsigned yp = (unsigned)min(y + DF_MOTION_PF, H - 1);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(frame + ((size_t)yp * row_bytes + lane_off)));
      }
    } else {
      fetch_row<FMT, FAST>(r, frame, lane_off, y, H, row_bytes);
    }
  };

  auto produce = [&](RowSlot<FMT>& r, int gy) {
    unsigned g0, g1;
    if (INT) {
      // Out-of-frame lanes (x < 0 or x >= W) read a clamped column; their
      // values only reach gauss/median border columns, which are copied.
      if (FMT == DF_MOTION_RGB) {
        g0 = rgb4_to_gray(r.raw[0].x, r.raw[0].y, r.raw[1].x, g.wg);
        g1 = rgb4_to_gray(r.raw[1].y, r.raw[2].x, r.raw[2].y, g.wg);
      } else {
        g0 = r.raw[0].x;
        g1 = r.raw[0].y;
      }
    } else {
      convert_row<FMT, FAST>(r, frame, x, lane_in, W, H, g0, g1, g.wg);
    }
    fetch(r, gy + 5);  // rows past the band are harmless
    const unsigned left = __shfl_up_sync(0xffffffffu, g1, 1);
    const unsigned right = __shfl_down_sync(0xffffffffu, g0, 1);
    hgauss4(left, g0, g1, r.h[0], r.h[1], g.wh);
    hgauss4(g0, g1, right, r.h[2], r.h[3], g.wh);
    r.g[0] = g0;
    r.g[1] = g1;
  };

  // gauss + thres of row gc = gy - 2 (window r4..r0 = rows gy-4..gy); ps is
  // the prev_s slot of row gc.
  auto gauss_thres = [&](RowSlot<FMT>& r4, RowSlot<FMT>& r3, RowSlot<FMT>& r2, RowSlot<FMT>& r1,
                         RowSlot<FMT>& r0, int gc, uint2* ps) {
    unsigned gw[2];
    if (!INT && (unsigned)(gc - 2) >= (unsigned)(H - 4)) {  // gc < 2 || gc >= H-2: gray copied
      gw[0] = r2.g[0];
      gw[1] = r2.g[1];
    } else {
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const unsigned v0 = vgauss(r4.h[2 * w], r3.h[2 * w], r2.h[2 * w], r1.h[2 * w], r0.h[2 * w]);
        const unsigned v1 =
            vgauss(r4.h[2 * w + 1], r3.h[2 * w + 1], r2.h[2 * w + 1], r1.h[2 * w + 1], r0.h[2 * w + 1]);
        gw[w] = lop_sel(gm[w], r2.g[w], prmt(v0, v1, 0x7531));
      }
    }
    if (MODE == 0) {
      *ps = make_uint2(gw[0], gw[1]);
      return;
    }
    const uint2 pv = *ps;
    *ps = make_uint2(gw[0], gw[1]);
    r2.t[0] = thres4(gw[0], pv.x, g);
    r2.t[1] = thres4(gw[1], pv.y, g);
    if (MODE == 2 && out_lane && gc >= y0 && gc < y0 + kBandRows && gc < H) {
      store_bytes8<FAST>(next_tok, gc, x, W, gw[0], gw[1]);
      if (next_copy) store_bytes8<FAST>(next_copy, gc, x, W, gw[0], gw[1]);
    }
  };

  // Median of row m (rows m-1, m, m+1 = r4, r3, r2); always inside the band.
  auto median = [&](RowSlot<FMT>& r4, RowSlot<FMT>& r3, RowSlot<FMT>& r2, int m) {
    const unsigned c0 = r3.t[0], c1 = r3.t[1];
    const unsigned lnb = __shfl_up_sync(0xffffffffu, c1, 1);
    const unsigned rnb = __shfl_down_sync(0xffffffffu, c0, 1);
    unsigned o0, o1;
    if (!INT && (unsigned)(m - 1) >= (unsigned)(H - 2)) {  // m == 0 || m == H-1: copied
      o0 = c0;
      o1 = c1;
    } else {
      const unsigned l0 = __funnelshift_l(lnb, c0, 8), r0w = __funnelshift_r(c0, c1, 8);
      const unsigned l1 = __funnelshift_l(c0, c1, 8), r1w = __funnelshift_r(c1, rnb, 8);
      o0 = lop_sel(mm[0], c0, maj5(c0, r4.t[0], r2.t[0], l0, r0w));
      o1 = lop_sel(mm[1], c1, maj5(c1, r4.t[1], r2.t[1], l1, r1w));
    }
    o0 = prmt(o0, 0, 0xBA98);
    o1 = prmt(o1, 0, 0xBA98);
    if (INT) {
      if (out_lane && x < W) *reinterpret_cast<uint2*>(out + ooff) = make_uint2(o0, o1);
      ooff += (unsigned)W;
    } else if (out_lane) {
      store_bytes8<FAST>(out, m, x, W, o0, o1);
    }
  };

  // One step per gauss row gc (y0-1 .. gc_end): window rows gc-2..gc+2 are
  // already produced; the step computes gauss/thres(gc) and median(gc-1)
  // from them and, independently (ILP), produces row gc+3 into the slot of
  // row gc-2 once that row has been consumed.
  const int gc_end = min(y0 + kBandRows, H);  // last gauss row needed
  // INT: the last produce (row y0+R+3) is surplus but in-frame, and the
  // break per step keeps ptxas scheduling step by step (each row's loads
  // stay five rows ahead of their use; a fixed-trip unrolled loop let it sink
  // all loads to the latch -- profiles/r01_ab_motion_variants.txt).
  auto step = [&](RowSlot<FMT>& r4, RowSlot<FMT>& r3, RowSlot<FMT>& r2, RowSlot<FMT>& r1, RowSlot<FMT>& r0,
                  int gc) {
    // r4..r0 = rows gc-2 .. gc+2
    gauss_thres(r4, r3, r2, r1, r0, gc, prev_s + (gc - (y0 - 1)) * 32 + lane);
    if (MODE != 0 && gc > y0) median(r4, r3, r2, gc - 1);  // rows gc-2, gc-1, gc
    if (INT || gc < gc_end) produce(r4, gc + 3);
  };

  int gc = y0 - 1;
#pragma unroll
  for (int k = 0; k < 5; ++k) fetch(s[k], y0 - 3 + k);
#pragma unroll
  for (int k = 0; k < 5; ++k) produce(s[k], y0 - 3 + k);
  while (true) {
    if (gc > gc_end) break;
    step(s[0], s[1], s[2], s[3], s[4], gc++);
    if (gc > gc_end) break;
    step(s[1], s[2], s[3], s[4], s[0], gc++);
    if (gc > gc_end) break;
    step(s[2], s[3], s[4], s[0], s[1], gc++);
    if (gc > gc_end) break;
    step(s[3], s[4], s[0], s[1], s[2], gc++);
    if (gc > gc_end) break;
    step(s[4], s[0], s[1], s[2], s[3], gc++);
  }
}

// A band is interior when every row a pass reads (y0-3 .. y0+R+2, plus the
// prefetch of rows up to y0+R+8) is inside the frame and no gauss row
// (y0-1 .. y0+R) or median row (y0 .. y0+R-1) is a border row.
__device__ __forceinline__ bool interior_band(int y0, int H) {
  return y0 >= 3 && y0 + kBandRows + 8 <= H - 1;
}

template <int FMT, bool FAST, bool INT>
__device__ __forceinline__ void walk_frames(const MotionIO& io, const unsigned char* in, unsigned char* out,
                                            const unsigned char* prev_tok, unsigned char* next_tok,
                                            unsigned char* next_copy, uint2* prev_s, const MotionGeom& g,
                                            int y0, int x, int xc, bool lane_in, int lane, int f_begin,
                                            int f_end) {
  const size_t in_frame = (size_t)g.W * g.H * FMT;
  const size_t frame_px = (size_t)g.W * g.H;
  unsigned gm[2], mm[2];
  column_masks(x, g.W, gm, mm);
  if (f_begin == 0) {
    // Delay token: gauss of the previous firing's last frame.
#pragma unroll 10
    for (int r = 0; r < kBandRows + 2; ++r) {
      unsigned a0, a1;
      a0 = a1 = 0u;  // null token: black (proj/src/motion.cpp:131)
      if (prev_tok) load_bytes8<FAST>(prev_tok, y0 - 1 + r, x, g.W, g.H, a0, a1);
      prev_s[r * 32 + lane] = make_uint2(a0, a1);
    }
  } else {
    frame_pass<FMT, FAST, 0, INT>(in + (size_t)(f_begin - 1) * in_frame, nullptr, nullptr, nullptr, prev_s, g,
                                  y0, x, xc, lane_in, lane, gm, mm);
  }
  const int f_last = (f_end == g.frames) ? f_end - 1 : f_end;  // frame that emits the delay token
  for (int f = f_begin; f < f_last; ++f)
    frame_pass<FMT, FAST, 1, INT>(in + (size_t)f * in_frame, out + (size_t)f * frame_px, nullptr, nullptr,
                                  prev_s, g, y0, x, xc, lane_in, lane, gm, mm);
  if (f_last < f_end)
    frame_pass<FMT, FAST, 2, INT>(in + (size_t)f_last * in_frame, out + (size_t)f_last * frame_px, next_tok,
                                  next_copy, prev_s, g, y0, x, xc, lane_in, lane, gm, mm);
}

template <int FMT, bool FAST>
__global__ void __launch_bounds__(32 * kWarpsPerCta, DF_MOTION_MINB) motion_fused_kernel(MotionIO io, MotionGeom g,
                                                                         unsigned* done_counter) {
  extern __shared__ uint2 prev_all[];  // [kWarpsPerCta][(kBandRows + 2) * 32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int band = blockIdx.y * kWarpsPerCta + warp;
  const int y0 = band * kBandRows;
  const int x = (int)blockIdx.x * kOutPxPerWarp - kPxPerLane + lane * kPxPerLane;
  const bool lane_in = x >= 0 && x < g.W;  // FAST: 8-px segments never straddle W
  const int xc = lane_in ? x : 0;
  const int f_begin = blockIdx.z * g.chunk;
  const int f_end = min(f_begin + g.chunk, g.frames);
  const unsigned char* in = io.in;
  unsigned char* out = io.out;
  const unsigned char* prev_tok = io.prev;
  unsigned char* next_tok = io.next;
  unsigned char* next_copy = io.next_copy;
  if (io.channel_mode) {
    in = chan_read_region(io.in_ch);
    out = chan_write_region(io.out_ch);
    prev_tok = chan_read_region(io.delay_ch);
    next_tok = chan_write_region(io.delay_ch);
    next_copy = chan_write_wraps(io.delay_ch) ? io.delay_ch.storage : nullptr;
  }

  if (y0 < g.H && f_begin < f_end) {
    uint2* prev_s = prev_all + warp * (kBandRows + 2) * 32;
    if (FAST && interior_band(y0, g.H))
      walk_frames<FMT, FAST, FAST>(io, in, out, prev_tok, next_tok, next_copy, prev_s, g, y0, x, xc, lane_in,
                                   lane, f_begin, f_end);
    else
      walk_frames<FMT, FAST, false>(io, in, out, prev_tok, next_tok, next_copy, prev_s, g, y0, x, xc, lane_in,
                                    lane, f_begin, f_end);
  }

  if (io.channel_mode) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(done_counter, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
    }
    __syncthreads();
    // Three independent commit chains on three threads (the delay channel's
    // read then write stay on one): each is an atomic round trip.
    if (last && threadIdx.x < 3) {
      __threadfence();
      if (threadIdx.x == 0) {
        *done_counter = 0;
        chan_commit_read(io.in_ch, io.in_ch.rate);
      } else if (threadIdx.x == 1) {
        chan_commit_read(io.delay_ch, 1);
        chan_commit_write(io.delay_ch, 1);
      } else {
        chan_commit_write(io.out_ch, io.out_ch.rate);
      }
    }
  }
}

constexpr size_t kSmemBytes = sizeof(uint2) * kWarpsPerCta * (kBandRows + 2) * 32;

// ===========================================================================
// M3: TMA-fed rows, TMEM-resident delay band.
//
// The register-prefetch kernel above is bound by bytes in flight (5 rows per
// warp in registers, shared memory full with the gauss(prev) bands).  M3
// moves gauss(prev) into tensor memory (TMEM, 256 KB/SM, otherwise idle:
// this path has no MMA) and streams the input rows through a per-warp
// shared-memory ring filled by TMA (cp.async.bulk.tensor, one box of kM3RPS
// rows per issue, mbarrier completion), kM3Stages * kM3RPS rows ahead of the
// consumer.  Out-of-frame rows and columns come back zero-filled (OOB: a 3-D
// (column, row, frame) view); they only reach border rows/columns, which the
// reference copies (motion.cpp:34-37, :64-67).
//
// CTA = kM3Warps warps on the same (tile, band), each walking its own frame
// range (temporal chunk): y0 and x stay warp-uniform, and each warp owns one
// TMEM lane quarter (warp w -> lanes 32w..32w+31, columns 2r, 2r+1 = prev
// row r).  The input must be 16-byte row aligned (W*FMT % 16 == 0).
// ===========================================================================
#ifndef DF_M3_RPS
#define DF_M3_RPS 5
#endif
// DF_M3_WARPS: warps per CTA.  4 (default): 4 CTAs per SM, each allocating
// 128 TMEM columns (one lane quarter per warp).  > 4: ONE CTA per SM that
// allocates all 512 columns; warp w uses lane quarter w % 4 and column block
// w / 4 (so R is capped by 2(R + 2) * ceil(WARPS / 4) <= 512).
#ifndef DF_M3_WARPS
#define DF_M3_WARPS 20
#endif
#ifndef DF_M3_ST
#define DF_M3_ST (DF_M3_WARPS > 4 ? 2 : 3)
#endif
// Shared-memory row loads issued at the start of a step (before the
// gauss/thres/median work) instead of right before their use: A/B
// (profiles/r01_ab_motion_variants.txt) 4K R=59 -1.8 %, 720p R=54 +1.3 %
// (ptxas allocates R=54 at the 128-register cap), so per band height.
#ifndef DF_M3_MINB
#define DF_M3_MINB (DF_M3_WARPS > 4 ? 1 : 4)  // __launch_bounds__ min blocks (register cap 65536 / (32 * WARPS * MINB))
#endif
#ifndef DF_M3_EARLY_MIN_R
#define DF_M3_EARLY_MIN_R 59
#endif
#ifndef DF_M3_ALT
#define DF_M3_ALT 1  // odd temporal chunks walk backwards (shared boundary frames hit L2)
#endif
#ifndef DF_M3_PDL
#define DF_M3_PDL 1  // programmatic dependent launch (setup overlaps the previous kernel's tail)
#endif
constexpr int kM3Warps = DF_M3_WARPS;
// Gray input: 16 px per lane (4 gray words) in 12-warp CTAs.  The kernel is
// issue-bound on gray, and the per-row per-lane fixed work (row load, the 4
// neighbour shuffles, TMEM load/store, output store, loop control, ring
// refill) is then shared by 16 px instead of 8; 12 warps x 4(R + 2) TMEM
// columns keep R = 39.  RGB keeps 8 px per lane (its 24 B/lane/row and
// RGB->gray registers) in 20-warp CTAs.
#ifndef DF_M3_GRAY_PX
#define DF_M3_GRAY_PX 16
#endif
#ifndef DF_M3_RGB_PX
#define DF_M3_RGB_PX 8
#endif
#ifndef DF_M3_WIDE_WARPS
#define DF_M3_WIDE_WARPS 12
#endif
template <int FMT>
struct M3Cfg {
  static constexpr int PX = FMT == DF_MOTION_GRAY ? DF_M3_GRAY_PX : DF_M3_RGB_PX;  // px per lane
  static constexpr int WPL = PX / 4;                                            // gray words per lane
  static constexpr int NW = PX == 16 ? DF_M3_WIDE_WARPS : kM3Warps;             // warps per CTA
  static constexpr int OUT = 30 * PX;                                           // output px per warp tile
  // A TMA box's innermost start must be 16-byte aligned.  Tile rows start at
  // FMT * (OUT t - PX) bytes: 8 bytes past a 16-byte boundary for PX = 8
  // (3 * (240 t - 8) = 720 t - 24 RGB, 240 t - 8 gray), so each box row is
  // the tile row plus 8 bytes on both sides; aligned for gray PX = 16.
  static constexpr int LEAD = (PX * FMT) % 16 == 0 ? 0 : 8;
  static constexpr int BPL = PX * FMT;  // input bytes per lane per row
  // TMA element size: a box dimension holds at most 256 elements, so rows
  // wider than 1 KB (RGB at 16 px per lane: 1536 B) use 8-byte elements.
  static constexpr int ESZ = (32 * BPL + 2 * LEAD) / 4 > 256 ? 8 : 4;
};
static_assert(DF_M3_GRAY_PX == 8 || DF_M3_GRAY_PX == 16, "gray px per lane");
static_assert(DF_M3_RGB_PX == 8 || DF_M3_RGB_PX == 16, "RGB px per lane");
// Band heights R (template parameter): a frame pass fetches rows y0-3 ..
// y0+R+2 (R + 6 rows, whole 5-row boxes), gauss(prev) holds R + 2 rows in
// WPL(R + 2) TMEM columns per warp.  launch_m3 picks R per frame geometry.
constexpr int kTmemCols = kM3Warps > 4 ? 512 : 128;
template <int FMT, int R>
constexpr int m3_warp_cols() { return M3Cfg<FMT>::WPL * (R + 2); }
template <int FMT, int R>
constexpr bool m3_valid_r() {
  return (R + 6) % 5 == 0 && m3_warp_cols<FMT, R>() * ((M3Cfg<FMT>::NW + 3) / 4) <= kTmemCols;
}
constexpr int kM3RPS = DF_M3_RPS;
constexpr int kM3Stages = DF_M3_ST;
static_assert(kM3RPS == 5, "one TMA box per 5-step iteration of the row loop (static in-box row offsets)");

template <int FMT>
constexpr int m3_row_bytes() { return 32 * M3Cfg<FMT>::BPL + 2 * M3Cfg<FMT>::LEAD; }  // 784 RGB / 512 gray B
template <int FMT>
constexpr int m3_stage_bytes() { return (kM3RPS * m3_row_bytes<FMT>() + 127) / 128 * 128; }
// Dynamic smem: NW rings (128-B aligned stages for TMA), then the
// mbarriers, then the TMEM base address slot.
template <int FMT>
constexpr size_t m3_ring_bytes() { return (size_t)kM3Stages * m3_stage_bytes<FMT>(); }
template <int FMT>
constexpr size_t m3_smem_bytes() {
  return M3Cfg<FMT>::NW * m3_ring_bytes<FMT>() + M3Cfg<FMT>::NW * kM3Stages * 8 + 16;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
#ifndef DF_M3_TMA3D
#define DF_M3_TMA3D 1
#endif
// fence.proxy.async before refilling a ring stage: not needed -- the stage's
// shared-memory loads have all been consumed (their values used) before the
// release, so no async-proxy write can overtake them (the CUTLASS consumer
// release has no fence either).  Kept as an A/B switch.
#ifndef DF_M3_PROXY_FENCE
#define DF_M3_PROXY_FENCE 0
#endif
// 3-D tensor (column word, row, frame): rows outside [0, H) of a frame are
// out of bounds and zero-filled without a DRAM read (a 2-D rows x frames
// view would fetch the neighbouring frame's rows for the top and bottom
// bands: 5.3 % extra input reads at 720p).
__device__ __forceinline__ void tma_load_3d(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// Same load with an L2 eviction-priority policy (createpolicy).
__device__ __forceinline__ void tma_load_3d_hint(unsigned dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 unsigned bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// L2 hints on the row stream (MotionGeom::l2hint; A/B in
// profiles/r02_ab_motion_l2hint.txt).  The 6 rows a band shares with the
// band above are read FIRST by this band (top of its pass) and LAST by the
// band above (bottom of its pass), one frame pass later.  At 4K that pass
// streams ~10x more bytes than at 720p and the rows are gone from L2 by the
// second read; the hint loads the first two groups of a pass with
// evict_last and the last group (the rows the band below already read) with
// evict_first.  4K RGB: 0.267 -> 0.250 ms (0.76 -> 0.81 of HBM); 720p: 1 %
// slower (its halo rows already survive), so it is enabled per geometry.
__device__ __forceinline__ void tmem_st2(unsigned taddr, unsigned a, unsigned b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tmem_ld2(unsigned taddr, unsigned& a, unsigned& b) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr) : "memory");
}
// The registers of a tcgen05.ld are undefined until wait::ld; tying them to
// the wait keeps every use after it.
__device__ __forceinline__ void tmem_wait_ld(unsigned& a, unsigned& b) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(a), "+r"(b)::"memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st4(unsigned taddr, const unsigned (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_ld4(unsigned taddr, unsigned (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld4(unsigned (&v)[4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3])::"memory");
}
// One gauss row of a lane (N = 2 or 4 words) to / from TMEM.
template <int N>
__device__ __forceinline__ void tmem_st_row(unsigned taddr, const unsigned (&v)[N]) {
  if constexpr (N == 2) tmem_st2(taddr, v[0], v[1]);
  else tmem_st4(taddr, v);
}
template <int N>
__device__ __forceinline__ void tmem_ld_row(unsigned taddr, unsigned (&v)[N]) {
  if constexpr (N == 2) tmem_ld2(taddr, v[0], v[1]);
  else tmem_ld4(taddr, v);
}
template <int N>
__device__ __forceinline__ void tmem_wait_row(unsigned (&v)[N]) {
  if constexpr (N == 2) tmem_wait_ld(v[0], v[1]);
  else tmem_wait_ld4(v);
}

// Per-warp row stream.  Group g = TMA box g = rows y0-3 + 5*(g % GPP) ..
// +4 of pass g / GPP (pass P = frame fs + dir*P, pass 0 of an inline-halo
// stream = frame 0 of hmap), in ring stage g % kM3Stages, completing its
// mbarrier phase (g / kM3Stages) & 1.  The 5-step unrolled row loop consumes
// exactly one group per iteration, so a row's offset in its box is a
// compile-time constant.  Groups are issued strictly in order, so the next
// group's coordinates advance incrementally (no divisions, warp-uniform: every
// lane advances them, lane 0 issues).
template <int FMT, int R>
struct M3Stream {
  static_assert(m3_valid_r<FMT, R>(), "band height");
  static constexpr int GPP = (R + 6) / kM3RPS;  // groups per frame pass
  const CUtensorMap* map;
  bool l2hint;        // L2 eviction hints on the band-halo rows (MotionGeom::l2hint)
  unsigned ring;      // smem address of this warp's ring
  unsigned bars;      // smem address of this warp's kM3Stages mbarriers
  unsigned stage;     // consumed group % kM3Stages
  unsigned phase;     // (consumed group / kM3Stages) & 1
  unsigned cur;       // this lane's bytes in the current group's first row
  int c0;             // tensor column (uint32 units) of the warp tile
  int H, y0;
  int dir;            // +1: pass P reads frame fs + P; -1: frame fs - P (backward chunk)
  int lane;
  // Next group to issue.
  int left;           // groups still to issue
  unsigned nin;       // its index in its pass
  int nrow;           // its first row
  int nf, fnext;      // its frame; the frame of the pass after
  const CUtensorMap* nmap;

  __device__ __forceinline__ void start(const CUtensorMap* m, const CUtensorMap* hm, bool hfirst, int fs,
                                        unsigned passes) {
    map = m;
    left = (int)passes * GPP;
    nin = 0;
    nrow = y0 - 3;
    nf = hfirst ? 0 : fs;
    fnext = fs + dir;
    nmap = hfirst ? hm : m;
  }
  // Lane 0: the TMA of the next group into stage s.
  __device__ __forceinline__ void issue(unsigned s) const {
    if (left <= 0) return;
    mbar_expect_tx(bars + 8 * s, kM3RPS * m3_row_bytes<FMT>());
#if DF_M3_TMA3D
    const int row = nrow, f = nf;
#else  // A/B baseline: frames stacked on the row axis (frame f at row f*H)
    const int row = nrow + (nmap == map ? nf * H : 0), f = 0;
#endif
    const unsigned dst = ring + s * m3_stage_bytes<FMT>();
    if (l2hint && nin < 2)
      tma_load_3d_hint(dst, nmap, c0, row, f, bars + 8 * s, policy_evict_last());
    else if (l2hint && nin == GPP - 1)
      tma_load_3d_hint(dst, nmap, c0, row, f, bars + 8 * s, policy_evict_first());
    else
      tma_load_3d(dst, nmap, c0, row, f, bars + 8 * s);
  }
  // Every lane: step the next-group state.
  __device__ __forceinline__ void advance() {
    --left;
    nrow += kM3RPS;
    if (++nin == GPP) {
      nin = 0;
      nrow = y0 - 3;
      nf = fnext;
      fnext += dir;
      nmap = map;
    }
  }
  __device__ __forceinline__ void acquire() {
    mbar_wait(bars + 8 * stage, phase);
    cur = ring + stage * m3_stage_bytes<FMT>() + M3Cfg<FMT>::LEAD + lane * M3Cfg<FMT>::BPL;
  }
  __device__ __forceinline__ unsigned row(int k) const { return cur + k * m3_row_bytes<FMT>(); }
  // After the group's bytes are in registers (and used): refill its stage
  // with group g + kM3Stages.
  __device__ __forceinline__ void release() {
    __syncwarp();
    if (lane == 0) {
#if DF_M3_PROXY_FENCE
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
      issue(stage);
    }
    advance();
    if (++stage == kM3Stages) {
      stage = 0;
      phase ^= 1;
    }
  }
};

__device__ __forceinline__ uint2 lds64(unsigned a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

__device__ __forceinline__ uint4 lds128(unsigned a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

template <int WPL>
struct M3Row {
  unsigned h[2 * WPL];  // horizontal sums, 16x2 packed
  unsigned g[WPL];      // gray words
  unsigned t[WPL];      // threshold flags
};

// WPL words (4 px each) of a lane to global memory (8 or 16 bytes).
template <int WPL>
__device__ __forceinline__ void store_words(unsigned char* p, const unsigned (&v)[WPL]) {
  if constexpr (WPL == 2) *reinterpret_cast<uint2*>(p) = make_uint2(v[0], v[1]);
  else *reinterpret_cast<uint4*>(p) = make_uint4(v[0], v[1], v[2], v[3]);
}

// One frame pass (MODE 0 warm-up / 1 chain / 2 chain + delay token / 3
// warm-up + delay token) of the warp's (tile, band).  INT: interior band (no
// border rows, full R rows).
template <int FMT, int R, int MODE, bool INT>
__device__ __forceinline__ void m3_pass(M3Stream<FMT, R>& st, unsigned char* __restrict__ out,
                                        unsigned char* __restrict__ next_tok, unsigned char* __restrict__ next_copy,
                                        unsigned tmem, const MotionGeom& g,
                                        int y0, int x, int lane, const unsigned (&gm)[M3Cfg<FMT>::WPL],
                                        const unsigned (&mm)[M3Cfg<FMT>::WPL]) {
  constexpr int WPL = M3Cfg<FMT>::WPL;
  constexpr int NIN = M3Cfg<FMT>::BPL / 4;  // input words per lane per row
  const int W = g.W, H = g.H;
  const bool out_lane = lane >= 1 && lane <= 30;
  M3Row<WPL> s[5];
  unsigned ooff = (unsigned)y0 * (unsigned)W + (unsigned)x;
  // Each prev row is read (tcgen05.ld, waited) before it is overwritten in
  // the same step; the previous pass's stores must have landed before this
  // pass's loads.
  constexpr bool CHAIN = MODE == 1 || MODE == 2;  // thres + median against TMEM's prev
  constexpr bool TOK = MODE == 2 || MODE == 3;    // this pass's gauss is the next delay token
  if (CHAIN) tmem_wait_st();

  // Row k (0..4) of the current group: the group is acquired at k == 0 and
  // released at k == 4.  fetch() reads the row's words from the ring;
  // finish() converts them (split so a step can issue its shared-memory
  // loads before the gauss/thres/median work that hides their latency).
  auto fetch = [&](int k, unsigned (&w)[NIN]) {
    if (k == 0) st.acquire();
    const unsigned a = st.row(k);
    if constexpr (NIN % 4 == 0) {
#pragma unroll
      for (int i = 0; i < NIN / 4; ++i) {
        const uint4 v = lds128(a + 16 * i);
        w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NIN / 2; ++i) {
        const uint2 v = lds64(a + 8 * i);
        w[2 * i] = v.x, w[2 * i + 1] = v.y;
      }
    }
  };
  auto finish = [&](M3Row<WPL>& r, int k, const unsigned (&w)[NIN]) {
    unsigned gw[WPL];
    if constexpr (FMT == DF_MOTION_RGB) {
#pragma unroll
      for (int i = 0; i < WPL; ++i) gw[i] = rgb4_to_gray(w[3 * i], w[3 * i + 1], w[3 * i + 2], g.wg);
    } else {
#pragma unroll
      for (int i = 0; i < WPL; ++i) gw[i] = w[i];
    }
    const unsigned left = __shfl_up_sync(0xffffffffu, gw[WPL - 1], 1);
    const unsigned right = __shfl_down_sync(0xffffffffu, gw[0], 1);
#pragma unroll
    for (int i = 0; i < WPL; ++i)
      hgauss4(i == 0 ? left : gw[i - 1], gw[i], i == WPL - 1 ? right : gw[i + 1], r.h[2 * i], r.h[2 * i + 1], g.wh);
#pragma unroll
    for (int i = 0; i < WPL; ++i) r.g[i] = gw[i];
    if (k == kM3RPS - 1) st.release();
  };
  auto produce = [&](M3Row<WPL>& r, int k) {
    unsigned w[NIN];
    fetch(k, w);
    finish(r, k, w);
  };

  auto gauss_thres = [&](M3Row<WPL>& r4, M3Row<WPL>& r3, M3Row<WPL>& r2, M3Row<WPL>& r1, M3Row<WPL>& r0, int gc) {
    const unsigned ta = tmem + (unsigned)WPL * (unsigned)(gc - (y0 - 1));
    unsigned p[WPL];
    if (CHAIN) tmem_ld_row<WPL>(ta, p);
    unsigned gw[WPL];
    if (!INT && (unsigned)(gc - 2) >= (unsigned)(H - 4)) {  // gc < 2 || gc >= H-2: gray copied
#pragma unroll
      for (int w = 0; w < WPL; ++w) gw[w] = r2.g[w];
    } else {
#pragma unroll
      for (int w = 0; w < WPL; ++w) {
        const unsigned v0 = vgauss_fma(r4.h[2 * w], r3.h[2 * w], r2.h[2 * w], r1.h[2 * w], r0.h[2 * w]);
        const unsigned v1 =
            vgauss_fma(r4.h[2 * w + 1], r3.h[2 * w + 1], r2.h[2 * w + 1], r1.h[2 * w + 1], r0.h[2 * w + 1]);
        gw[w] = lop_sel(gm[w], r2.g[w], prmt(v0, v1, 0x7531));
      }
    }
    if (CHAIN) {
      tmem_wait_row<WPL>(p);
#pragma unroll
      for (int w = 0; w < WPL; ++w) r2.t[w] = thres4(gw[w], p[w], g);
    }
    tmem_st_row<WPL>(ta, gw);
    if (TOK && out_lane && x < W && gc >= y0 && gc < y0 + R && gc < H) {
      const unsigned o = (unsigned)gc * (unsigned)W + (unsigned)x;
      store_words<WPL>(next_tok + o, gw);
      if (next_copy) store_words<WPL>(next_copy + o, gw);  // Fig. 2 phase 2
    }
  };

  auto median = [&](M3Row<WPL>& r4, M3Row<WPL>& r3, M3Row<WPL>& r2, int m) {
    const unsigned lnb = __shfl_up_sync(0xffffffffu, r3.t[WPL - 1], 1);
    const unsigned rnb = __shfl_down_sync(0xffffffffu, r3.t[0], 1);
    unsigned o[WPL];
    if (!INT && (unsigned)(m - 1) >= (unsigned)(H - 2)) {  // m == 0 || m == H-1: copied
#pragma unroll
      for (int w = 0; w < WPL; ++w) o[w] = r3.t[w];
    } else {
#pragma unroll
      for (int w = 0; w < WPL; ++w) {
        const unsigned c = r3.t[w];
        const unsigned l = __funnelshift_l(w == 0 ? lnb : r3.t[w - 1], c, 8);
        const unsigned rw = __funnelshift_r(c, w == WPL - 1 ? rnb : r3.t[w + 1], 8);
        o[w] = lop_sel(mm[w], c, maj5(c, r4.t[w], r2.t[w], l, rw));
      }
    }
#pragma unroll
    for (int w = 0; w < WPL; ++w) o[w] = prmt(o[w], 0, 0xBA98);
    if (out_lane && x < W) store_words<WPL>(out + ooff, o);
    ooff += (unsigned)W;
  };

  const int gc_end = min(y0 + R, H);  // last gauss row needed
  // Step gc produces row gc+3 = stream row gc - y0 + 6 of the pass: in-group
  // position (gc - y0 + 1) % 5, i.e. the step's position k in the unrolled
  // 5-step body (the body starts at gc = y0 - 1 + 5i).
  auto step = [&](M3Row<WPL>& r4, M3Row<WPL>& r3, M3Row<WPL>& r2, M3Row<WPL>& r1, M3Row<WPL>& r0, int gc, int k) {
    if constexpr (R >= DF_M3_EARLY_MIN_R) {
      unsigned w[NIN] = {};
      if (gc < gc_end) fetch(k, w);
      gauss_thres(r4, r3, r2, r1, r0, gc);
      if (CHAIN && gc > y0) median(r4, r3, r2, gc - 1);
      if (gc < gc_end) finish(r4, k, w);
    } else {
      gauss_thres(r4, r3, r2, r1, r0, gc);
      if (CHAIN && gc > y0) median(r4, r3, r2, gc - 1);
      if (gc < gc_end) produce(r4, k);
    }
  };

#pragma unroll
  for (int k = 0; k < 5; ++k) produce(s[k], k);
  int gc = y0 - 1;
  while (true) {
    if (gc > gc_end) break;
    step(s[0], s[1], s[2], s[3], s[4], gc++, 0);
    if (gc > gc_end) break;
    step(s[1], s[2], s[3], s[4], s[0], gc++, 1);
    if (gc > gc_end) break;
    step(s[2], s[3], s[4], s[0], s[1], gc++, 2);
    if (gc > gc_end) break;
    step(s[3], s[4], s[0], s[1], s[2], gc++, 3);
    if (gc > gc_end) break;
    step(s[4], s[0], s[1], s[2], s[3], gc++, 4);
  }
  // Bottom band (gc_end < y0 + R): rows past the frame were fetched but not
  // consumed.  Release a partly consumed group and skip the pass's rest.
  if (!INT) {
    const int produced = gc_end - y0 + 6;  // rows of this pass consumed
    int done = produced / kM3RPS;
    if (produced % kM3RPS) {
      st.release();
      ++done;
    }
    for (; done < M3Stream<FMT, R>::GPP; ++done) {
      st.acquire();
      st.release();
    }
  }
}

template <int FMT, int R, bool INT>
__device__ __forceinline__ void m3_walk(M3Stream<FMT, R>& st, bool hfirst, const unsigned char* prev_tok, unsigned char* out,
                                        unsigned char* next_tok, unsigned char* next_copy, unsigned tmem, const MotionGeom& g, int y0, int x,
                                        int lane, int f_begin, int f_end) {
  constexpr int WPL = M3Cfg<FMT>::WPL;
  const size_t frame_px = (size_t)g.W * g.H;
  unsigned gm[WPL], mm[WPL];
  column_masks<WPL>(x, g.W, gm, mm);
  // First pass: gauss of the frame before the chunk's first output (forward)
  // or of its last frame (backward, see motion_m3_kernel) into TMEM -- or
  // the delay token.  A backward chunk's first gauss is the next delay token
  // when it is the firing's last frame.
  if (st.dir < 0 && f_end == g.frames) {
    m3_pass<FMT, R, 3, INT>(st, nullptr, next_tok, next_copy, tmem, g, y0, x, lane, gm, mm);
  } else if (st.dir > 0 && f_begin == 0 && !hfirst) {
    // Delay token: gauss of the previous firing's last frame -> TMEM.
    for (int r = 0; r < R + 2; ++r) {
      unsigned v[WPL] = {};  // null token: black (proj/src/motion.cpp:131)
      if (prev_tok)
#pragma unroll
        for (int i = 0; i < WPL / 2; ++i)
          load_bytes8<true>(prev_tok, y0 - 1 + r, x + 8 * i, g.W, g.H, v[2 * i], v[2 * i + 1]);
      tmem_st_row<WPL>(tmem + (unsigned)(WPL * r), v);
    }
  } else {  // gauss of the first frame read: f_begin - 1 (or the inline halo frame), or f_end - 1
    m3_pass<FMT, R, 0, INT>(st, nullptr, nullptr, nullptr, tmem, g, y0, x, lane, gm, mm);
  }
  // Chain passes, ONE loop body for both directions (a second hot copy of the
  // pass costs instruction-cache misses).  Backward: the pass on frame k - 1
  // yields the output of frame k (|g(k) - g(k-1)| is symmetric).
  const int f_last = (st.dir > 0 && f_end == g.frames) ? f_end - 1 : f_end;
  const int n_chain = f_last - f_begin;
  for (int j = 0; j < n_chain; ++j) {
    const int f = st.dir > 0 ? f_begin + j : f_end - 1 - j;
    m3_pass<FMT, R, 1, INT>(st, out + (size_t)f * frame_px, nullptr, nullptr, tmem, g, y0, x, lane, gm, mm);
  }
  if (f_last < f_end)
    m3_pass<FMT, R, 2, INT>(st, out + (size_t)f_last * frame_px, next_tok, next_copy, tmem, g, y0, x, lane, gm, mm);
}

template <int FMT, int R>
__global__ void __launch_bounds__(32 * M3Cfg<FMT>::NW, DF_M3_MINB) motion_m3_kernel(const __grid_constant__ CUtensorMap map,
                                                                   const __grid_constant__ CUtensorMap hmap,
                                                                   MotionIO io, MotionGeom g,
                                                                   unsigned* done_counter) {
  extern __shared__ __align__(128) unsigned char m3_smem[];
  // shfl from lane 0: the compiler then treats warp-derived values (TMEM
  // addresses, ring addresses) as warp-uniform instead of emitting
  // per-unique-value loops around every tcgen05.ld/st.
  const int lane = threadIdx.x & 31, warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);
  // Warp task t (1-D grid): consecutive tasks are consecutive temporal chunks
  // of one (tile, band), so a 4-warp CTA holds 4 chunks of one band as before.
  using Cfg = M3Cfg<FMT>;
  const int task = (int)blockIdx.x * Cfg::NW + warp;
  const int chunk = task % g.m3_chunks;
  const int band = (task / g.m3_chunks) % g.m3_bands;
  const int tile = task / (g.m3_chunks * g.m3_bands);
  const int y0 = band * R;
  const int tx0 = tile * Cfg::OUT - Cfg::PX;
  const int x = tx0 + lane * Cfg::PX;
  const int f_begin = chunk * g.chunk;
  // Tasks past the last tile (the grid's last CTA) walk no frames.
  const int f_end = tx0 < g.W ? min(f_begin + g.chunk, g.frames) : f_begin;

#if DF_M3_PDL
  // Programmatic dependent launch: the next kernel in the stream (e.g. a
  // sink's commit) may launch now; this grid sets up (TMEM, barriers) and
  // waits for the previous grid before touching anything it produced.
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(m3_smem + Cfg::NW * m3_ring_bytes<FMT>() + Cfg::NW * kM3Stages * 8);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  M3Stream<FMT, R> st;
  // Inline halo (raw mode): the first chunk warms up on the halo frame
  // instead of loading a delay token -- gauss(halo) never goes through HBM.
  const bool hfirst = io.halo != nullptr && f_begin == 0;
  st.ring = smem_u32(m3_smem + warp * m3_ring_bytes<FMT>());
  st.bars = smem_u32(m3_smem + Cfg::NW * m3_ring_bytes<FMT>() + warp * kM3Stages * 8);
  st.stage = 0;
  st.phase = 0;
  st.cur = 0;
  st.c0 = (tx0 * FMT - Cfg::LEAD) / Cfg::ESZ;  // 16-byte aligned box start (see M3Cfg::LEAD)
  st.l2hint = g.l2hint;
  st.H = g.H;
  st.y0 = y0;
#if DF_M3_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  // Channel mode: the map covers the input channel's whole storage; the
  // firing's region (resolved from the device phase) starts at frame slot
  // `base` of it.  Raw mode: the map covers exactly the firing's frames.
  unsigned char* out = io.out;
  const unsigned char* prev_tok = io.prev;
  unsigned char* next_tok = io.next;
  unsigned char* next_copy = io.next_copy;
  int base = 0;
  if (io.channel_mode) {
    base = (int)((size_t)(chan_read_region(io.in_ch) - io.in_ch.storage) / io.in_ch.token_size);
    out = chan_write_region(io.out_ch);
    prev_tok = chan_read_region(io.delay_ch);
    next_tok = chan_write_region(io.delay_ch);
    next_copy = chan_write_wraps(io.delay_ch) ? io.delay_ch.storage : nullptr;
  }
  st.lane = lane;
  // Odd chunks walk their frames backwards (DF_M3_ALT).  Every chunk but the
  // first re-reads one frame its neighbour also reads -- the frame before
  // it: forward chunk c+1's warm-up frame is forward chunk c's last frame,
  // read at opposite ends of the walk, so the second read came from DRAM
  // (~9 % extra input reads at 720p).  With alternating directions the two
  // chunks sharing a boundary frame both read it FIRST (a backward chunk's
  // warm-up and the next forward chunk's warm-up) or both LAST, at about
  // the same time, and the second read hits L2.  Chunk 0 (delay token or
  // inline halo) always walks forward.
  const bool back = DF_M3_ALT && (chunk & 1) && f_begin < f_end;
  st.dir = back ? -1 : 1;
  const int f_first = back ? f_end - 1 : (f_begin > 0 || hfirst) ? f_begin - 1 : f_begin;  // first frame read
  const int passes = f_begin >= f_end ? 0 : back ? f_end - f_begin + 1 : f_end - f_first;
  st.start(&map, &hmap, hfirst, base + f_first, (unsigned)passes);
  if (lane == 0) {
    for (int s = 0; s < kM3Stages; ++s) mbar_init(st.bars + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // Lane quarter warp % 4 (a warp may only access its own quarter), column
  // block warp / 4.
  const unsigned tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0) + ((unsigned)(32 * (warp & 3)) << 16) +
                        (unsigned)((warp >> 2) * m3_warp_cols<FMT, R>());

  if (passes > 0) {
    for (int s = 0; s < kM3Stages; ++s) {
      if (lane == 0) st.issue(s);
      st.advance();
    }
    const bool interior = y0 >= 3 && y0 + R <= g.H - 3;  // no border gauss/median row
    if (interior)
      m3_walk<FMT, R, true>(st, hfirst, prev_tok, out, next_tok, next_copy, tmem, g, y0, x, lane, f_begin, f_end);
    else
      m3_walk<FMT, R, false>(st, hfirst, prev_tok, out, next_tok, next_copy, tmem, g, y0, x, lane, f_begin, f_end);
  }
  tmem_wait_st();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "n"(kTmemCols) : "memory");
  }
  if (io.channel_mode) {  // the last CTA commits the firing (as motion_fused_kernel)
    __shared__ bool last;
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(done_counter, 1u) == gridDim.x * gridDim.y * gridDim.z - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      *done_counter = 0;
      chan_commit_read(io.in_ch, io.in_ch.rate);
      chan_commit_read(io.delay_ch, 1);
      chan_commit_write(io.delay_ch, 1);
      chan_commit_write(io.out_ch, io.out_ch.rate);
    }
  }
}


// Gauss of one frame given in the input format (sets a delay token from a
// raw halo frame).
template <int FMT>
__global__ void gauss_frame_kernel(const unsigned char* __restrict__ in, unsigned char* __restrict__ out,
                                   int W, int H) {
  const int xx = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (xx >= W) return;
  auto gray = [&](int yy, int xi) -> int {
    if (FMT == DF_MOTION_RGB) {
      const unsigned char* q = in + ((size_t)yy * W + xi) * 3;
      return (int)((77u * q[0] + 150u * q[1] + 29u * q[2] + 128u) >> 8);
    }
    return in[(size_t)yy * W + xi];
  };
  const size_t idx = (size_t)y * W + xx;
  if (y < 2 || y >= H - 2 || xx < 2 || xx >= W - 2) {
    out[idx] = (unsigned char)gray(y, xx);
    return;
  }
  const int k[5] = {1, 4, 6, 4, 1};
  int acc = 0;
  for (int dy = -2; dy <= 2; ++dy)
    for (int dx = -2; dx <= 2; ++dx) acc += k[dy + 2] * k[dx + 2] * gray(y + dy, xx + dx);
  out[idx] = (unsigned char)((acc + 128) >> 8);
}

__global__ void thres_kernel(const unsigned char* prev, const unsigned char* cur, unsigned char* out,
                             size_t n, int thr) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = abs((int)cur[i] - (int)prev[i]) > thr ? 255 : 0;
}

__global__ void median_kernel(const unsigned char* in, unsigned char* out, int W, int H) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= W) return;
  const size_t i = (size_t)y * W + x;
  if (y == 0 || y == H - 1 || x == 0 || x == W - 1) {
    out[i] = in[i];
    return;
  }
  unsigned char v[5] = {in[i], in[i - W], in[i + W], in[i - 1], in[i + 1]};
  for (int a = 1; a < 5; ++a)
    for (int b = a; b > 0 && v[b - 1] > v[b]; --b) {
      unsigned char t = v[b];
      v[b] = v[b - 1];
      v[b - 1] = t;
    }
  out[i] = v[2];
}

__global__ void rgb_gray_kernel(const unsigned char* rgb, unsigned char* gray, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    gray[i] = (unsigned char)((77u * rgb[3 * i] + 150u * rgb[3 * i + 1] + 29u * rgb[3 * i + 2] + 128u) >> 8);
}

}  // namespace
}  // namespace df

using namespace df;

struct df_motion {
  int device = 0;
  int W = 0, H = 0, fmt = 1;
  uint8_t thr = 32;
  unsigned char* tok[2] = {nullptr, nullptr};  // raw-mode delay token ping-pong
  int cur = 0;
  bool black = false;  // the current token is the black initial token (not materialised)
  unsigned* scratch = nullptr;  // done counter
  int resident_ctas = 0;        // per SM, for the temporal chunking
  int m3_resident[3] = {0, 0, 0};  // motion_m3_kernel<R> CTAs per SM (0: M3 unavailable)
  int sms = 148;
  df::Staging staging;          // df_motion_run_host pipeline
};

namespace {

MotionGeom make_geom(const df_motion* m, int frames) {
  MotionGeom g;
  g.W = m->W;
  g.H = m->H;
  g.frames = frames;
  const unsigned thr = m->thr;
  if (thr <= 127) {
    g.thr_k = (127u - thr) * 0x01010101u;
    g.thr_sel = 0xFFFFFFFFu;
  } else {
    g.thr_k = (255u - thr) * 0x01010101u;
    g.thr_sel = 0u;
  }
  const unsigned wg[6] = {W8(77, 150, 29, 0), W8(150, 29, 0, 0), W8(0, 0, 0, 77),
                          W8(29, 0, 0, 0),   W8(0, 0, 77, 150), W8(0, 77, 150, 29)};
  const unsigned wh[8] = {W8(0, 0, 1, 4), W8(6, 4, 1, 0), W8(0, 0, 0, 1), W8(4, 6, 4, 1),
                          W8(1, 4, 6, 4), W8(1, 0, 0, 0), W8(0, 1, 4, 6), W8(4, 1, 0, 0)};
  for (int i = 0; i < 6; ++i) g.wg[i] = wg[i];
  for (int i = 0; i < 8; ++i) g.wh[i] = wh[i];
  // Temporal chunking: as many frame ranges as fit one wave of CTAs.
  const int tiles = (m->W + kOutPxPerWarp - 1) / kOutPxPerWarp;
  const int bands = (m->H + kBandRows - 1) / kBandRows;
  const int ctas_per_chunk = tiles * ((bands + kWarpsPerCta - 1) / kWarpsPerCta);
  const int wave = std::max(1, m->resident_ctas * m->sms);
  int chunks = std::max(1, wave / std::max(1, ctas_per_chunk));
  chunks = std::min(chunks, std::max(1, frames));
  g.chunk = (frames + chunks - 1) / chunks;
  return g;
}

template <int FMT, bool FAST>
int launch_fused(df_motion* m, const MotionIO& io, int frames, cudaStream_t s) {
  MotionGeom g = make_geom(m, frames);
  const int tiles = (m->W + kOutPxPerWarp - 1) / kOutPxPerWarp;
  const int bands = (m->H + kBandRows - 1) / kBandRows;
  dim3 grid(tiles, (bands + kWarpsPerCta - 1) / kWarpsPerCta, (frames + g.chunk - 1) / g.chunk);
  motion_fused_kernel<FMT, FAST><<<grid, 32 * kWarpsPerCta, kSmemBytes, s>>>(io, g, m->scratch);
  return after_launch("motion_fused_kernel");
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

#ifndef DF_MOTION_M3
#define DF_MOTION_M3 1
#endif

bool m3_eligible(const df_motion* m, const MotionIO& io, int frames) {
  const void* base = io.channel_mode ? (const void*)io.in_ch.storage : (const void*)io.in;
  // TMA row coordinates are int32: the mapped rows (H x frames, + halo) must fit.
  const unsigned long long map_frames =
      io.channel_mode ? chan_capacity_tokens(io.in_ch.rate, io.in_ch.has_delay) : (unsigned long long)frames;
  return DF_MOTION_M3 && m->m3_resident[0] > 0 && ((size_t)m->W * m->fmt) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(base) & 15) == 0 && (unsigned long long)m->H * map_frames < (1ull << 31) - 256 &&
         tensor_map_encoder() != nullptr;
}

// Band heights M3 is built for; launch_m3 picks the one whose grid fills
// one wave best (cost model: waves x (frames per chunk + warm-up) x rows
// fetched per pass).
#if DF_M3_WARPS > 20
constexpr int kM3Heights[3] = {29, 34, 39};  // 6 warps per lane quarter: 2(R + 2) <= 85 columns
#elif DF_M3_WARPS > 16
constexpr int kM3Heights[3] = {39, 44, 49};  // 5 warps per lane quarter: 2(R + 2) <= 102 columns
#else
constexpr int kM3Heights[3] = {49, 54, 59};
#endif
#if DF_M3_WIDE_WARPS > 12
constexpr int kM3WideHeights[3] = {19, 24, 29};  // 16 px per lane, 4 warps per lane quarter: 4(R + 2) <= 128
#else
constexpr int kM3WideHeights[3] = {29, 34, 39};  // 16 px per lane, 3 warps per lane quarter: 4(R + 2) <= 170
#endif
template <int FMT>
constexpr int m3_height(int ri) {
  return M3Cfg<FMT>::PX == 16 ? kM3WideHeights[ri] : kM3Heights[ri];
}

template <int FMT>
const void* m3_kernel_fn(int ri) {
  return ri == 0 ? (const void*)motion_m3_kernel<FMT, m3_height<FMT>(0)>
                 : ri == 1 ? (const void*)motion_m3_kernel<FMT, m3_height<FMT>(1)>
                           : (const void*)motion_m3_kernel<FMT, m3_height<FMT>(2)>;
}

struct M3Plan {
  int ri, bands, chunk, chunks, slices;
  double cost;
};

template <int FMT>
M3Plan m3_plan(const df_motion* m, int frames, int ri) {
  constexpr int NW = M3Cfg<FMT>::NW;
  const int R = m3_height<FMT>(ri);
  const int tiles = (m->W + M3Cfg<FMT>::OUT - 1) / M3Cfg<FMT>::OUT;
  M3Plan p{};
  p.ri = ri;
  p.bands = (m->H + R - 1) / R;
  const int slots = std::max(1, m->m3_resident[ri] * m->sms);  // CTAs in one wave
  const int per_slice = tiles * p.bands;  // warp tasks per temporal chunk
  // Temporal chunks (one warp task per (tile, band, chunk)): as many as fit
  // ONE wave of warps (a partial second wave would double the step time).
  p.slices = std::max(1, slots * NW / per_slice);
  p.chunks = std::min(p.slices, frames);
  if (NW == 4 && p.chunks > 4) p.chunks &= ~3;  // whole CTAs of one (tile, band)
  p.chunk = (frames + p.chunks - 1) / p.chunks;
  p.chunks = (frames + p.chunk - 1) / p.chunk;
  const int ctas = (per_slice * p.chunks + NW - 1) / NW;
  const int waves = (ctas + slots - 1) / slots;
  p.cost = (double)waves * (p.chunk + (p.chunks > 1 ? 1 : 0)) * (R + 6);
  return p;
}

template <int FMT>
int launch_m3(df_motion* m, const MotionIO& io, int frames, cudaStream_t s) {
  MotionGeom g = make_geom(m, frames);
  constexpr int NW = M3Cfg<FMT>::NW;
  M3Plan best = m3_plan<FMT>(m, frames, 0);
  for (int ri = 1; ri < 3; ++ri) {
    const M3Plan p = m3_plan<FMT>(m, frames, ri);
    if (p.cost < best.cost) best = p;
  }
  if (const char* force = getenv("DF_MOTION_M3_R")) {  // tests: pin the band height
    const int ri = atoi(force);
    if (ri >= 0 && ri < 3) best = m3_plan<FMT>(m, frames, ri);
  }
  g.chunk = best.chunk;
  g.m3_chunks = best.chunks;
  g.m3_bands = best.bands;
  // Band-halo rows need the L2 hint only when a frame pass streams more than
  // L2 can hold between their two reads (4K: 24.9 MB RGB frames; not 720p).
  g.l2hint = (size_t)m->W * m->H * FMT >= (8u << 20) ? 1 : 0;
  if (const char* force = getenv("DF_MOTION_L2HINT")) g.l2hint = atoi(force);
  // Raw mode: the map covers the firing's frames; channel mode: the input
  // channel's whole storage (the kernel offsets to its region).
  const void* base = io.channel_mode ? (const void*)io.in_ch.storage : (const void*)io.in;
  const unsigned long long map_frames =
      io.channel_mode ? chan_capacity_tokens(io.in_ch.rate, io.in_ch.has_delay) : (unsigned long long)frames;
  CUtensorMap map;
#if DF_M3_TMA3D
  const cuuint64_t dims[3] = {(cuuint64_t)m->W * FMT / M3Cfg<FMT>::ESZ, (cuuint64_t)m->H, (cuuint64_t)map_frames};
#else
  const cuuint64_t dims[3] = {(cuuint64_t)m->W * FMT / M3Cfg<FMT>::ESZ, (cuuint64_t)m->H * map_frames, 1};
#endif
  const cuuint64_t strides[2] = {(cuuint64_t)m->W * FMT, (cuuint64_t)m->W * FMT * (cuuint64_t)m->H};
  const cuuint32_t box[3] = {(cuuint32_t)(m3_row_bytes<FMT>() / M3Cfg<FMT>::ESZ), (cuuint32_t)kM3RPS, 1};
  const CUtensorMapDataType dtype = M3Cfg<FMT>::ESZ == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = tensor_map_encoder()(&map, dtype, 3, const_cast<void*>(base), dims,
                                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DF_REQUIRE(cr == CUDA_SUCCESS, DF_ECUDA, "motion: cuTensorMapEncodeTiled failed (%d)", (int)cr);
  CUtensorMap hmap = map;
  if (io.halo) {  // one frame, same box
    const cuuint64_t hdims[3] = {(cuuint64_t)m->W * FMT / M3Cfg<FMT>::ESZ, (cuuint64_t)m->H, 1};
    cr = tensor_map_encoder()(&hmap, dtype, 3, const_cast<unsigned char*>(io.halo), hdims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DF_REQUIRE(cr == CUDA_SUCCESS, DF_ECUDA, "motion: cuTensorMapEncodeTiled (halo) failed (%d)", (int)cr);
  }
  const int tiles = (m->W + M3Cfg<FMT>::OUT - 1) / M3Cfg<FMT>::OUT;
  dim3 grid((tiles * best.bands * best.chunks + NW - 1) / NW);
  if (getenv("DF_DEBUG"))
    fprintf(stderr, "motion_m3: %d px/lane, %d warps, R %d, resident %d/SM, grid %ux%ux%u, chunk %d frames, smem %zu\n",
            M3Cfg<FMT>::PX, NW, m3_height<FMT>(best.ri), m->m3_resident[best.ri], grid.x, grid.y, grid.z, g.chunk,
            m3_smem_bytes<FMT>());
  const size_t smem = m3_smem_bytes<FMT>();
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = dim3(32 * NW);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = DF_M3_PDL ? 1 : 0;
  cudaError_t le;
  if (best.ri == 0)
    le = cudaLaunchKernelEx(&lc, motion_m3_kernel<FMT, m3_height<FMT>(0)>, map, hmap, io, g, m->scratch);
  else if (best.ri == 1)
    le = cudaLaunchKernelEx(&lc, motion_m3_kernel<FMT, m3_height<FMT>(1)>, map, hmap, io, g, m->scratch);
  else
    le = cudaLaunchKernelEx(&lc, motion_m3_kernel<FMT, m3_height<FMT>(2)>, map, hmap, io, g, m->scratch);
  DF_CHECK_CUDA(le);
  return after_launch("motion_m3_kernel");
}

int launch_motion(df_motion* m, const MotionIO& io, int frames, cudaStream_t s) {
  if (frames <= 0) return DF_OK;
  if (m3_eligible(m, io, frames))
    return m->fmt == DF_MOTION_RGB ? launch_m3<DF_MOTION_RGB>(m, io, frames, s)
                                   : launch_m3<DF_MOTION_GRAY>(m, io, frames, s);
  const bool fast = (m->W % 8 == 0);
  if (m->fmt == DF_MOTION_RGB)
    return fast ? launch_fused<DF_MOTION_RGB, true>(m, io, frames, s)
                : launch_fused<DF_MOTION_RGB, false>(m, io, frames, s);
  return fast ? launch_fused<DF_MOTION_GRAY, true>(m, io, frames, s)
              : launch_fused<DF_MOTION_GRAY, false>(m, io, frames, s);
}

}  // namespace

extern "C" {

int df_motion_create(int device, unsigned width, unsigned height, int fmt, uint8_t thr,
                     df_motion** out) {
  DF_REQUIRE(out, DF_EINVAL, "df_motion_create: null out pointer");
  *out = nullptr;
  // proj/src/motion.cpp:108-110
  DF_REQUIRE(width >= 5 && height >= 5, DF_EINVAL, "motion: frame must be at least 5x5");
  DF_REQUIRE(fmt == DF_MOTION_GRAY || fmt == DF_MOTION_RGB, DF_EINVAL, "motion: input format must be GRAY or RGB");
  DF_REQUIRE(width <= (1u << 20) && height <= (1u << 20) && (uint64_t)width * height * 3 < (1ull << 32),
             DF_EINVAL, "motion: frame too large");
  DF_CHECK_CUDA(cudaSetDevice(device));
  auto* m = new df_motion();
  m->device = device;
  m->W = (int)width;
  m->H = (int)height;
  m->fmt = fmt;
  m->thr = thr;
  const size_t px = (size_t)width * height;
  cudaError_t e = cudaMalloc(&m->tok[0], px);
  if (e == cudaSuccess) e = cudaMalloc(&m->tok[1], px);
  if (e == cudaSuccess) e = cudaMalloc(&m->scratch, 64);
  if (e == cudaSuccess) e = cudaMemset(m->tok[0], 0, px);  // black initial token
  if (e == cudaSuccess) e = cudaMemset(m->scratch, 0, 64);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&m->sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) {
    const bool fast = width % 8 == 0;
    const void* fn = fmt == DF_MOTION_RGB
                         ? (fast ? (const void*)motion_fused_kernel<DF_MOTION_RGB, true>
                                 : (const void*)motion_fused_kernel<DF_MOTION_RGB, false>)
                         : (fast ? (const void*)motion_fused_kernel<DF_MOTION_GRAY, true>
                                 : (const void*)motion_fused_kernel<DF_MOTION_GRAY, false>);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m->resident_ctas, fn, 32 * kWarpsPerCta, kSmemBytes);
    if (e == cudaSuccess && DF_MOTION_M3 && ((size_t)width * fmt) % 16 == 0) {
      const int sm3 = (int)(fmt == DF_MOTION_RGB ? m3_smem_bytes<DF_MOTION_RGB>() : m3_smem_bytes<DF_MOTION_GRAY>());
      int smem_sm = 0;
      e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
      for (int ri = 0; ri < 3 && e == cudaSuccess; ++ri) {
        const void* f3 = fmt == DF_MOTION_RGB ? m3_kernel_fn<DF_MOTION_RGB>(ri) : m3_kernel_fn<DF_MOTION_GRAY>(ri);
        e = cudaFuncSetAttribute(f3, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
        // Residency from the kernel's resources (the occupancy API reports 1
        // CTA/SM for kernels that allocate TMEM): TMEM (kTmemCols of 512
        // columns per CTA), registers, shared memory (+1 KB reserved per CTA).
        cudaFuncAttributes fa{};
        if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, f3);
        if (e == cudaSuccess) {
          const int nw = fmt == DF_MOTION_RGB ? M3Cfg<DF_MOTION_RGB>::NW : M3Cfg<DF_MOTION_GRAY>::NW;
          const int by_regs = 65536 / std::max(1, fa.numRegs * 32 * nw);
          const int by_smem = smem_sm / (sm3 + (int)fa.sharedSizeBytes + 1024);
          m->m3_resident[ri] = std::max(0, std::min({512 / kTmemCols, by_regs, by_smem}));
        }
      }
      if (e != cudaSuccess || m->m3_resident[0] == 0 || m->m3_resident[1] == 0 || m->m3_resident[2] == 0) {
        m->m3_resident[0] = 0;  // M3 unavailable: the register-prefetch kernel runs
        e = cudaSuccess;
        cudaGetLastError();
      }
    }
  }
  if (e != cudaSuccess) {
    int rc = cuda_status(e, "df_motion_create");
    cudaFree(m->tok[0]);
    cudaFree(m->tok[1]);
    cudaFree(m->scratch);
    delete m;
    return rc;
  }
  *out = m;
  return DF_OK;
}

int df_motion_destroy(df_motion* m) {
  if (!m) return DF_OK;
  cudaSetDevice(m->device);
  m->staging.release();
  cudaFree(m->tok[0]);
  cudaFree(m->tok[1]);
  cudaFree(m->scratch);
  delete m;
  return DF_OK;
}

int df_motion_set_prev_frame(df_motion* m, const void* frame_dev, void* stream) {
  DF_REQUIRE(m, DF_EINVAL, "df_motion_set_prev_frame: null actor");
  DF_CHECK_CUDA(cudaSetDevice(m->device));
  cudaStream_t s = as_stream(stream);
  if (!frame_dev) {  // black: the next firing loads zeros instead of a token
    m->black = true;
    return DF_OK;
  }
  m->black = false;
  dim3 grid((m->W + 127) / 128, m->H);
  if (m->fmt == DF_MOTION_RGB)
    gauss_frame_kernel<DF_MOTION_RGB><<<grid, 128, 0, s>>>((const unsigned char*)frame_dev, m->tok[m->cur], m->W, m->H);
  else
    gauss_frame_kernel<DF_MOTION_GRAY><<<grid, 128, 0, s>>>((const unsigned char*)frame_dev, m->tok[m->cur], m->W, m->H);
  return after_launch("gauss_frame_kernel");
}

int df_motion_fire(df_motion* m, const void* in_dev, uint8_t* out_dev, uint32_t frames, void* stream) {
  DF_REQUIRE(m, DF_EINVAL, "df_motion_fire: null actor");
  if (frames == 0) return DF_OK;
  DF_REQUIRE(in_dev && out_dev, DF_EINVAL, "df_motion_fire: null buffer");
  DF_REQUIRE(frames <= (1u << 30), DF_EINVAL, "df_motion_fire: too many frames");
  DF_CHECK_CUDA(cudaSetDevice(m->device));
  MotionIO io{};
  io.in = (const unsigned char*)in_dev;
  io.out = out_dev;
  io.prev = m->black ? nullptr : m->tok[m->cur];
  io.next = m->tok[m->cur ^ 1];
  io.next_copy = nullptr;
  io.channel_mode = 0;
  DF_TRY(launch_motion(m, io, (int)frames, as_stream(stream)));
  m->cur ^= 1;
  m->black = false;
  return DF_OK;
}

int df_motion_fire_halo(df_motion* m, const void* halo_dev, const void* in_dev, uint8_t* out_dev,
                        uint32_t frames, void* stream) {
  DF_REQUIRE(m, DF_EINVAL, "df_motion_fire_halo: null actor");
  if (frames == 0) return DF_OK;
  DF_REQUIRE(halo_dev && in_dev && out_dev, DF_EINVAL, "df_motion_fire_halo: null buffer");
  DF_REQUIRE(frames <= (1u << 30), DF_EINVAL, "df_motion_fire_halo: too many frames");
  DF_CHECK_CUDA(cudaSetDevice(m->device));
  MotionIO io{};
  io.in = (const unsigned char*)in_dev;
  io.out = out_dev;
  io.prev = m->tok[m->cur];
  io.next = m->tok[m->cur ^ 1];
  io.halo = (const unsigned char*)halo_dev;
  const bool halo_ok = (reinterpret_cast<uintptr_t>(halo_dev) & 15) == 0;
  if (!m3_eligible(m, io, (int)frames) || !halo_ok) {
    // Register-prefetch kernel: the halo becomes the delay token first.
    DF_TRY(df_motion_set_prev_frame(m, halo_dev, stream));
    return df_motion_fire(m, in_dev, out_dev, frames, stream);
  }
  DF_TRY(launch_motion(m, io, (int)frames, as_stream(stream)));
  m->cur ^= 1;
  m->black = false;
  return DF_OK;
}

int df_motion_fire_channels(df_motion* m, df_channel* in, df_channel* delay, df_channel* out,
                            void* stream) {
  DF_REQUIRE(m && in && delay && out, DF_EINVAL, "df_motion_fire_channels: null argument");
  const size_t px = (size_t)m->W * m->H;
  DF_REQUIRE(in->token_size == px * (size_t)m->fmt, DF_ELOGIC, "motion: input token must be one frame");
  DF_REQUIRE(out->token_size == px && out->rate == in->rate, DF_ELOGIC,
             "motion: output token must be one W*H mask at the input's rate");
  DF_REQUIRE(delay->token_size == px && delay->rate == 1 && delay->has_delay, DF_ELOGIC,
             "motion: delay channel must be a rate-1 self-loop with a delay token of W*H bytes");
  DF_REQUIRE(in->reader != Endpoint::host && out->writer != Endpoint::host &&
                 delay->reader != Endpoint::host && delay->writer != Endpoint::host,
             DF_ELOGIC, "motion: channel endpoint is host-driven");
  in->reader = out->writer = delay->reader = delay->writer = Endpoint::device;
  DF_CHECK_CUDA(cudaSetDevice(m->device));
  MotionIO io{};
  io.channel_mode = 1;
  io.in_ch = in->dev();
  io.out_ch = out->dev();
  io.delay_ch = delay->dev();
  return launch_motion(m, io, (int)in->rate, as_stream(stream));
}

int df_motion_run_host(df_motion* m, const void* in_host, uint8_t* out_host, uint64_t frames,
                       uint32_t chunk_frames, void* stream) {
  DF_REQUIRE(m && in_host && out_host, DF_EINVAL, "df_motion_run_host: null argument");
  if (frames == 0) return DF_OK;
  DF_CHECK_CUDA(cudaSetDevice(m->device));
  const size_t in_frame = (size_t)m->W * m->H * m->fmt, out_frame = (size_t)m->W * m->H;
  if (chunk_frames == 0) chunk_frames = (uint32_t)df::Staging::chunk_units(frames, in_frame, 256ull << 20);
  chunk_frames = (uint32_t)std::min<uint64_t>(chunk_frames, frames);
  cudaStream_t cs = as_stream(stream);
  DF_TRY(m->staging.ensure(chunk_frames * in_frame, chunk_frames * out_frame));
  const uint64_t nchunks = (frames + chunk_frames - 1) / chunk_frames;
  auto nf = [&](uint64_t c) { return (uint32_t)std::min<uint64_t>(chunk_frames, frames - c * chunk_frames); };
  return m->staging.pipeline(
      cs, nchunks,
      [&](uint64_t c, const void*& p, size_t& b) {
        p = (const unsigned char*)in_host + c * chunk_frames * in_frame;
        b = nf(c) * in_frame;
      },
      [&](uint64_t c, void*& p, size_t& b) {
        p = out_host + c * chunk_frames * out_frame;
        b = nf(c) * out_frame;
      },
      [&](uint64_t c, unsigned char* din, unsigned char* dout) { return df_motion_fire(m, din, dout, nf(c), cs); });
}

const char* df_motion_kernel_name(const df_motion* m) {
  if (!m) return "";
  return DF_MOTION_M3 && m->m3_resident[0] > 0 && ((size_t)m->W * m->fmt) % 16 == 0 && tensor_map_encoder()
             ? "motion_m3_kernel"
             : "motion_fused_kernel";
}

int df_motion_gauss5x5(const uint8_t* in_dev, uint8_t* out_dev, unsigned w, unsigned h, void* stream) {
  DF_REQUIRE(in_dev && out_dev, DF_EINVAL, "gauss5x5: null buffer");
  DF_REQUIRE(w >= 5 && h >= 5, DF_EINVAL, "gauss5x5: frame smaller than the 5x5 kernel");
  dim3 grid((w + 127) / 128, h);
  gauss_frame_kernel<DF_MOTION_GRAY><<<grid, 128, 0, as_stream(stream)>>>(in_dev, out_dev, (int)w, (int)h);
  return after_launch("gauss_frame_kernel");
}

int df_motion_thres_diff(const uint8_t* prev_dev, const uint8_t* cur_dev, uint8_t* out_dev, unsigned w,
                         unsigned h, uint8_t thr, void* stream) {
  DF_REQUIRE(prev_dev && cur_dev && out_dev, DF_EINVAL, "thres_diff: null buffer");
  const size_t n = (size_t)w * h;
  if (n == 0) return DF_OK;
  thres_kernel<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, as_stream(stream)>>>(
      prev_dev, cur_dev, out_dev, n, thr);
  return after_launch("thres_kernel");
}

int df_motion_median5(const uint8_t* in_dev, uint8_t* out_dev, unsigned w, unsigned h, void* stream) {
  DF_REQUIRE(in_dev && out_dev, DF_EINVAL, "median5: null buffer");
  DF_REQUIRE(w >= 3 && h >= 3, DF_EINVAL, "median5: frame smaller than 3x3");
  dim3 grid((w + 127) / 128, h);
  median_kernel<<<grid, 128, 0, as_stream(stream)>>>(in_dev, out_dev, (int)w, (int)h);
  return after_launch("median_kernel");
}

int df_motion_rgb_to_gray(const uint8_t* rgb_dev, uint8_t* gray_dev, size_t pixels, void* stream) {
  DF_REQUIRE(rgb_dev && gray_dev, DF_EINVAL, "rgb_to_gray: null buffer");
  if (pixels == 0) return DF_OK;
  rgb_gray_kernel<<<(unsigned)std::min<size_t>((pixels + 255) / 256, 4096), 256, 0, as_stream(stream)>>>(
      rgb_dev, gray_dev, pixels);
  return after_launch("rgb_gray_kernel");
}

}  // extern "C"
