// netrt.cu -- device-resident actor networks: persistent actors on sm_100a.
//
// The reference runs a network as one OS thread per actor, each looping
// Run::fire_once over blocking mutex/condvar channels, with end of stream,
// drain and abort (proj/src/runtime.cpp:132-299, proj/src/channel.cpp:
// 63-177).  Here the whole network is ONE cooperative persistent kernel:
// every actor is a group of co-resident CTAs.  The group leader (CTA 0,
// thread 0) plays the actor thread:
//
//   control token -> rates   read 1 token from the control ring, look it up
//                            in the actor's control table (the device form of
//                            ActorBehavior::control + control_dispatch,
//                            proj/src/model.cpp:240-265): per regular port 0
//                            or r, or illegal -> ControlError fault;
//   read_start / write_start spin on the ring's `available` counter in HBM
//                            until r tokens are there (or the channel is
//                            closed and fewer remain: end of stream) / until
//                            r slots are free;
//   fire                     publish the regions (a frame) to the group's
//                            CTAs, which all fire on them;
//   write_end / read_end     after the group is done: the Fig. 2 phase-2
//                            copy (slot 3r -> 0) of a delay channel, then
//                            commit outputs, then inputs (release order).
//
// At its firing limit (sources) or end of stream the leader closes its
// outputs and drains its inputs (proj/src/runtime.cpp:216-231).  A fault
// records (actor, code, token) and sets the abort word; every spin loop
// watches it (and a host-mapped abort word, and a watchdog), so a fault or
// df_net_abort ends every actor (RunAborted, channel.cpp:170-177).
//
// Memory ordering: data is written with plain stores and read with
// ld.global.cg (L2; a ring slot is rewritten every 2-3 firings, so an L1
// copy could be stale); counters are published with a fence + atomic and
// read with ld.acquire.gpu.
#include <algorithm>
#include <cstring>
#include <vector>

#include "channel_dev.cuh"
#include "channel_host.hpp"
#include "common.cuh"

namespace df {
namespace {

constexpr int kMaxPorts = 24;
constexpr unsigned kMaxPairs = 10;  // DPD adder: up to 10 (re, im) input pairs
constexpr int kNetThreads = 256;
constexpr int kParamBytes = 96;

struct ActorDesc {
  int kind;
  unsigned cta0, ctas;
  unsigned n_in, n_out;
  int has_ctrl;
  unsigned long long limit;  // firing limit (0: none)
  DevChan ctrl;
  DevChan in[kMaxPorts];
  DevChan out[kMaxPorts];
  const uint32_t* table;  // [domain][3] = in bits, out bits, legal
  unsigned domain;
  alignas(16) unsigned char params[kParamBytes];
};

struct Frame {
  unsigned long long firing;
  unsigned stop;
  unsigned in_on, out_on, out_wrap;
  unsigned char* in_ptr[kMaxPorts];
  unsigned char* out_ptr[kMaxPorts];
};

struct ActorRt {
  unsigned gen;   // frame generation published by the leader
  unsigned done;  // CTAs finished with the current frame
  Frame frame;
  unsigned long long firings, t_first, t_stop;
  // Leader time split (ns, summed over firings): waiting in read_start /
  // write_start (incl. the control token), firing (publish -> every CTA
  // done), commit (phase-2 copies + counter updates).
  unsigned long long t_wait, t_fire, t_commit;
  unsigned long long state[4];  // kind state (test stream positions)
};

struct NetCtl {
  unsigned abort;  // set by a fault (device) -- every spin loop watches it
  unsigned fault_actor, fault_code, fault_token;
  unsigned long long timeout_ns;
  const volatile unsigned* host_abort;  // mapped pinned host word (df_net_abort)
};

// ---- memory-model helpers ---------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acq32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- waits (leader thread only) ------------------------------------------
enum Wait : int { kOk = 0, kEos = 1, kAbort = 2 };

__device__ void raise_fault(NetCtl* ctl, int actor, unsigned code, unsigned token) {
  if (atomicCAS(&ctl->fault_code, 0u, code) == 0u) {
    ctl->fault_actor = (unsigned)actor;
    ctl->fault_token = token;
  }
  __threadfence();
  atomicExch(&ctl->abort, 1u);
}

// Polls the mapped host abort word (df_net_abort) -- a PCIe read, so only
// group leaders poll it, at most every kHostPollNs -- and promotes it to the
// device word every actor watches.
constexpr unsigned long long kHostPollNs = 20000;
__device__ bool host_abort_poll(NetCtl* ctl, unsigned long long* last) {
  const unsigned long long t = now_ns();
  if (t - *last < kHostPollNs) return false;
  *last = t;
  if (!*ctl->host_abort) return false;
  atomicCAS(&ctl->fault_code, 0u, (unsigned)DF_EABORTED);
  atomicExch(&ctl->abort, 1u);
  return true;
}

// Is the run aborted (a device fault, or df_net_abort from the host)?
__device__ bool aborted_now(NetCtl* ctl, unsigned long long* last_host_poll) {
  if (*(volatile unsigned*)&ctl->abort) return true;
  return last_host_poll && host_abort_poll(ctl, last_host_poll);
}

// A wait loop: backs off from 32 ns to 256 ns between polls, watches the
// abort words, and (leaders) a watchdog over the whole wait.
struct Spin {
  unsigned long long t0 = 0;
  unsigned long long* host_poll = nullptr;  // leaders: their last host-abort poll time
  unsigned n = 0;
  bool watchdog = true;
  // Returns kAbort when the run is aborted or this wait timed out.
  __device__ int tick(NetCtl* ctl, int actor) {
    if (aborted_now(ctl, (++n & 15) == 0 ? host_poll : nullptr)) return kAbort;
    if (watchdog && (n & 15) == 0) {
      const unsigned long long t = now_ns();
      if (t0 == 0) t0 = t;
      if (t - t0 > ctl->timeout_ns) {
        raise_fault(ctl, actor, DF_ETIMEOUT, 0);
        return kAbort;
      }
    }
    __nanosleep(32u << min(n / 8, 3u));  // 32 ns .. 256 ns
    return kOk;
  }
};

// read_start (channel.cpp:114-140): r tokens, or end of stream once closed.
__device__ int wait_readable(const DevChan& c, unsigned r, NetCtl* ctl, int actor, unsigned long long* poll) {
  Spin s;
  s.host_poll = poll;
  for (;;) {
    if (ld_acq64(&c.st->available) >= r) return kOk;
    if (ld_acq32(&c.st->closed)) return ld_acq64(&c.st->available) >= r ? kOk : kEos;
    if (s.tick(ctl, actor) != kOk) return kAbort;
  }
}
// write_end / read_end.  The CALLER fences once before a firing's commits
// (every CTA's data accesses of the firing are complete by then); the
// counter updates themselves are relaxed reductions.
// `phase` is the endpoint's phase, cached by the leader (it is the only
// writer); the control block's copy is written for the host's stats.
__device__ void commit_write(const DevChan& c, unsigned r, unsigned& phase) {
  DevChanState* st = c.st;
  phase = (phase + 1) % chan_phases(c.has_delay);
  st->write_phase = phase;
  atomicAdd(&st->written, (unsigned long long)r);
  atomicAdd(&st->available, (unsigned long long)r);
}
__device__ void commit_read(const DevChan& c, unsigned r, unsigned& phase) {
  DevChanState* st = c.st;
  phase = (phase + 1) % chan_phases(c.has_delay);
  st->read_phase = phase;
  atomicAdd(&st->read, (unsigned long long)r);
  atomicAdd(&st->available, (unsigned long long)(-(long long)r));
}

// The leader's cached endpoint phases (shared memory of the leader CTA).
struct Phases {
  unsigned in[kMaxPorts], out[kMaxPorts], ctrl;
};
__device__ __forceinline__ unsigned long long ld_rlx64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void close_channel(const DevChan& c) {
  __threadfence();
  st_rel32(&c.st->closed, 1u);
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// acceptance.cpp:62-66 fill_token (as channel.cu's test actors)
__device__ __forceinline__ unsigned char token_byte(unsigned long long seed, unsigned long long index, size_t i) {
  return (unsigned char)(mix64(seed ^ (index * 1315423911ULL + i)) & 0xFF);
}

template <typename P>
__device__ __forceinline__ const P& params(const ActorDesc& A) {
  return *reinterpret_cast<const P*>(A.params);
}

// ---- leader: one firing's control, regions and waits ----------------------
// Fills rt->frame and publishes it (returns false once the actor stops).
__device__ bool leader_prepare(const ActorDesc& A, int a, ActorRt* rt, NetCtl* ctl, bool* aborted,
                               unsigned long long* poll, Phases& ph) {
  Frame& F = rt->frame;
  const unsigned long long i = rt->firings;
  bool stop = false;
  if (A.limit && i >= A.limit) stop = true;  // source firing limit (runtime.cpp:217-219)
  if (!stop && aborted_now(ctl, poll)) {  // checked once per firing, not only inside waits
    stop = true;
    *aborted = true;
  }
  unsigned in_on = A.n_in >= 32 ? 0xffffffffu : (1u << A.n_in) - 1;
  unsigned out_on = A.n_out >= 32 ? 0xffffffffu : (1u << A.n_out) - 1;
  if (!stop && A.kind == DF_ACT_TEST_PRODUCE) {  // scripted stalls (concurrency tests)
    const df_act_test& P = params<df_act_test>(A);
    unsigned long long pause = P.hold_ns;
    if (P.stall_mask && (mix64(P.seed ^ (i * 0x51ed27ull)) & P.stall_mask) == 0) pause += 2000;
    const unsigned long long t0 = now_ns();
    while (pause && now_ns() - t0 < pause) {
      if (aborted_now(ctl, poll)) {
        stop = true;
        *aborted = true;
        break;
      }
      __nanosleep(1000);
    }
  }
  if (!stop && A.has_ctrl) {  // fire_once: one control token, then rates
    const int w = wait_readable(A.ctrl, 1, ctl, a, poll);
    if (w != kOk) {
      stop = true;
      *aborted = w == kAbort;
    } else {
      const unsigned char* tok = A.ctrl.storage + chan_read_slot(A.ctrl.rate, A.ctrl.has_delay, ph.ctrl) * A.ctrl.token_size;
      unsigned v = 0;
      for (unsigned b = 0; b < 4 && b < A.ctrl.token_size; ++b) v |= (unsigned)__ldcg(tok + b) << (8 * b);
      unsigned extra = 0;  // bytes beyond the 4th must be zero for v to name the token
      for (unsigned b = 4; b < A.ctrl.token_size && b < 64; ++b) extra |= __ldcg(tok + b);
      __threadfence();  // the token bytes are read before the slot is released
      commit_read(A.ctrl, 1, ph.ctrl);  // the control region is released before the firing (runtime.cpp:144)
      const uint32_t* row = A.table + 3ull * (v < A.domain ? v : 0);
      if (v >= A.domain || extra || !row[2]) {
        raise_fault(ctl, a, DF_ECONTROL, v);
        stop = true;
        *aborted = true;
      } else {
        in_on = row[0];
        out_on = row[1];
      }
    }
  }
  // read_start on every active input and write_start on every active
  // output, polled together: each round issues all the counter loads
  // (relaxed, independent) and spins only while some port is not ready; one
  // acquire fence then orders the firing's data accesses after them.
  if (!stop) {
    unsigned in_wait = in_on & (A.n_in >= 32 ? 0xffffffffu : (1u << A.n_in) - 1);
    unsigned out_wait = out_on & (A.n_out >= 32 ? 0xffffffffu : (1u << A.n_out) - 1);
    Spin sp;
    sp.host_poll = poll;
    while (in_wait | out_wait) {
      // Up to 4 counters per batch are loaded before any is compared, so
      // their L2 round trips overlap (a 20-input adder polled one port at a
      // time waited ~20 sequential round trips per firing).
      constexpr int kB = 4;
      for (unsigned pend = in_wait; pend;) {
        unsigned long long v[kB];
        int idx[kB], n = 0;
        for (; pend && n < kB; pend &= pend - 1, ++n) {
          idx[n] = __ffs(pend) - 1;
          v[n] = ld_rlx64(&A.in[idx[n]].st->available);
        }
        for (int k = 0; k < n; ++k) {
          const DevChan& c = A.in[idx[k]];
          if (v[k] >= c.rate)
            in_wait &= ~(1u << idx[k]);
          else if (ld_rlx32(&c.st->closed) && ld_rlx64(&c.st->available) < c.rate)
            stop = true;  // end of stream (read_start -> nullopt)
        }
      }
      for (unsigned pend = out_wait; pend;) {
        unsigned long long v[kB];
        int idx[kB], n = 0;
        for (; pend && n < kB; pend &= pend - 1, ++n) {
          idx[n] = __ffs(pend) - 1;
          v[n] = ld_rlx64(&A.out[idx[n]].st->available);
        }
        for (int k = 0; k < n; ++k) {
          const DevChan& c = A.out[idx[k]];
          if (v[k] + c.rate <= chan_distinct_capacity(c.rate, c.has_delay)) out_wait &= ~(1u << idx[k]);
        }
      }
      if (stop || !(in_wait | out_wait)) break;
      if (sp.tick(ctl, a) != kOk) {
        stop = true;
        *aborted = true;
      }
      if (stop) break;
    }
    __threadfence();
  }
  unsigned wrap = 0;
  for (unsigned p = 0; !stop && p < A.n_in; ++p)
    if ((in_on >> p) & 1u)
      F.in_ptr[p] = A.in[p].storage + chan_read_slot(A.in[p].rate, A.in[p].has_delay, ph.in[p]) * A.in[p].token_size;
  for (unsigned p = 0; !stop && p < A.n_out; ++p) {
    if (!((out_on >> p) & 1u)) continue;
    const unsigned wp = ph.out[p];
    F.out_ptr[p] = A.out[p].storage + chan_write_slot(A.out[p].rate, A.out[p].has_delay, wp) * A.out[p].token_size;
    if (A.out[p].has_delay && wp % 3 == 2) wrap |= 1u << p;
  }
  F.firing = i;
  F.stop = stop ? 1u : 0u;
  F.in_on = in_on;
  F.out_on = out_on;
  F.out_wrap = wrap;
  if (!stop && i == 0) rt->t_first = now_ns();
  __threadfence();
  st_rel32(&rt->gen, rt->gen + 1);
  return !stop;
}

// ---- kinds: the firing, run by every thread of the actor's CTAs -----------
// Grid-stride index over the group: [g*blockDim + tid, ...) step ctas*blockDim.
struct Group {
  unsigned g, ctas;
  __device__ unsigned long long first() const { return (unsigned long long)g * blockDim.x + threadIdx.x; }
  __device__ unsigned long long step() const { return (unsigned long long)ctas * blockDim.x; }
};

__device__ float2 poly_sample(float re, float im, int b) {  // poly_branch, dpd.cpp:67-73
  if (b == 1) return make_float2(re, im);
  const float mag = __fsqrt_rn(__fadd_rn(__fmul_rn(re, re), __fmul_rn(im, im)));
  float scale = mag;
  for (int p = 2; p < b; ++p) scale = __fmul_rn(scale, mag);
  return make_float2(__fmul_rn(re, scale), __fmul_rn(im, scale));
}

// Grid-stride loop over [0, n) that issues U independent loads per thread
// before any store: an actor's few CTAs move a whole token per firing, so
// memory-level parallelism, not bandwidth, bounds them (one load in flight
// per thread made the DPD split / source / sink latency-bound).
template <int U, typename T, typename L, typename S>
__device__ __forceinline__ void batched(const Group& G, unsigned long long n, L load, S store) {
  const unsigned long long step = G.step();
  for (unsigned long long k = G.first(); k < n; k += U * step) {
    T v[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (k + j * step < n) v[j] = load(k + j * step);
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (k + j * step < n) store(k + j * step, v[j]);
  }
}

struct U4x2 {
  uint4 re, im;
};

__device__ __noinline__ void copy_bytes(unsigned char* dst, const unsigned char* src, unsigned long long n, const Group& G) {
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | n) & 15) == 0) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    batched<4, uint4>(G, n / 16, [&](unsigned long long k) { return __ldcg(s + k); },
                      [&](unsigned long long k, const uint4& v) { d[k] = v; });
  } else {
    batched<4, unsigned char>(G, n, [&](unsigned long long k) { return __ldcg(src + k); },
                              [&](unsigned long long k, unsigned char v) { dst[k] = v; });
  }
}

// DPD split fire on 16-byte words: each word of re and im is loaded once
// and stored to every active output of its plane.
__device__ __noinline__ void split_planes(const ActorDesc& A, const Frame& F, const Group& G, unsigned long long n16) {
  const uint4* re = reinterpret_cast<const uint4*>(F.in_ptr[0]);
  const uint4* im = reinterpret_cast<const uint4*>(F.in_ptr[1]);
  batched<2, U4x2>(G, n16, [&](unsigned long long k) { return U4x2{__ldcg(re + k), __ldcg(im + k)}; },
                   [&](unsigned long long k, const U4x2& v) {
                     for (unsigned o = 0; o < A.n_out; ++o)
                       if ((F.out_on >> o) & 1u) reinterpret_cast<uint4*>(F.out_ptr[o])[k] = o & 1u ? v.im : v.re;
                   });
}


// The branch actor's window: kBranchV consecutive outputs per thread.
constexpr int kBranchV = 4;

__device__ void fire_dpd_branch(const ActorDesc& A, const Frame& F, const Group& G, float2* win) {
  const df_act_branch& P = params<df_act_branch>(A);
  if (!(F.in_on & 1u)) return;  // inactive this period: no I/O, state frozen (dpd.cpp:272)
  const float* re = reinterpret_cast<const float*>(F.in_ptr[0]);
  const float* im = reinterpret_cast<const float*>(F.in_ptr[1]);
  float* ore = reinterpret_cast<float*>(F.out_ptr[0]);
  float* oim = reinterpret_cast<float*>(F.out_ptr[1]);
  const float2* taps = reinterpret_cast<const float2*>(P.taps);
  const float2* state = reinterpret_cast<const float2*>(P.state);
  const int T = (int)P.taps_per_branch, H1 = T - 1, b = (int)P.branch;
  const unsigned n = P.period;
  // Chunks of C = kBranchV * blockDim outputs, round-robin over the group's
  // CTAs; the poly window (chunk + T-1 history) is staged in shared memory
  // and each thread runs a register-blocked FIR over kBranchV consecutive
  // outputs (a sliding window over the taps: kBranchV independent
  // accumulation chains per component).  The raw inputs of the next chunk
  // are loaded before this chunk's FIR.
  constexpr int V = kBranchV;
  const unsigned C = V * blockDim.x;
  const unsigned stride = G.ctas * C;
  constexpr int MW = V + 1;  // window positions per thread: C + T-1 <= (V+1) * blockDim for T <= 33
  auto raw = [&](unsigned c0, int w) -> float2 {
    const long long j = (long long)c0 - H1 + w;
    if (w >= (int)C + H1 || j >= (long long)n) return make_float2(0.f, 0.f);
    if (j >= 0) return make_float2(__ldcg(re + j), __ldcg(im + j));
    return __ldcg(state - j - 1);  // FirState x[-(j+1)] (fir10, dpd.cpp:92-97), written by the leader CTA
  };
  float2 nx[MW];
#pragma unroll
  for (int m = 0; m < MW; ++m) nx[m] = raw(G.g * C, threadIdx.x + m * blockDim.x);
  for (unsigned c0 = G.g * C; c0 < n; c0 += stride) {
    float2 x[MW];
#pragma unroll
    for (int m = 0; m < MW; ++m) x[m] = nx[m];
    if (c0 + stride < n) {
#pragma unroll
      for (int m = 0; m < MW; ++m) nx[m] = raw(c0 + stride, threadIdx.x + m * blockDim.x);
    }
    __syncthreads();  // the previous chunk's FIR has read the window
    // poly of the raw samples; history positions before the block start are
    // already poly outputs (the FirState).
#pragma unroll
    for (int m = 0; m < MW; ++m) {
      const int w = threadIdx.x + m * blockDim.x;
      if (w < (int)C + H1) {
        const long long j = (long long)c0 - H1 + w;
        win[w] = j >= 0 ? poly_sample(x[m].x, x[m].y, b) : x[m];
      }
    }
    __syncthreads();
    const unsigned o0 = c0 + V * threadIdx.x;
    if (o0 < n) {
      // fir10's accumulation order per output (dpd.cpp:87-104): 0.0f, then
      // taps k ascending.  Output o0 + j reads window index V*tid + j + H1 - k.
      float ar[V], ai[V], wr[V], wi[V];
      const int base = V * threadIdx.x + H1;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float2 v = win[base + j];
        wr[j] = v.x;
        wi[j] = v.y;
        ar[j] = ai[j] = 0.0f;
      }
      for (int k = 0; k < T; ++k) {
        if (k > 0) {
#pragma unroll
          for (int j = V - 1; j > 0; --j) {
            wr[j] = wr[j - 1];
            wi[j] = wi[j - 1];
          }
          const float2 v = win[base - k];
          wr[0] = v.x;
          wi[0] = v.y;
        }
        const float2 t = taps[k];
#pragma unroll
        for (int j = 0; j < V; ++j) {
          ar[j] = __fadd_rn(ar[j], __fsub_rn(__fmul_rn(t.x, wr[j]), __fmul_rn(t.y, wi[j])));
          ai[j] = __fadd_rn(ai[j], __fadd_rn(__fmul_rn(t.x, wi[j]), __fmul_rn(t.y, wr[j])));
        }
      }
#pragma unroll
      for (int j = 0; j < V; ++j)
        if (o0 + j < n) {
          ore[o0 + j] = ar[j];
          oim[o0 + j] = ai[j];
        }
    }
  }
}

// After every CTA fired (leader CTA): the branch's FirState becomes the
// block's last T-1 poly outputs, older state filling short blocks
// (dpd.cpp:108-120).
__device__ void post_dpd_branch(const ActorDesc& A, const Frame& F) {
  const df_act_branch& P = params<df_act_branch>(A);
  if (!(F.in_on & 1u)) return;
  const float* re = reinterpret_cast<const float*>(F.in_ptr[0]);
  const float* im = reinterpret_cast<const float*>(F.in_ptr[1]);
  float2* state = reinterpret_cast<float2*>(P.state);
  const int H1 = (int)P.taps_per_branch - 1;
  const long long n = P.period;
  __shared__ float2 next[32];
  if ((int)threadIdx.x < H1) {
    const long long idx = n - 1 - threadIdx.x;
    next[threadIdx.x] = idx >= 0 ? poly_sample(__ldcg(re + idx), __ldcg(im + idx), (int)P.branch) : __ldcg(state - idx - 1);
  }
  __syncthreads();
  if ((int)threadIdx.x < H1) state[threadIdx.x] = next[threadIdx.x];
}

// ---- motion actors, 4 px per thread (frames with W % 4 == 0) -------------
// The same integer arithmetic as the fused motion kernel (motion.cu): the
// horizontal [1 4 6 4 1] as IDP.4A dot products on packed bytes with a +8
// bias per row sum (the vertical weights sum to 16, so the bias adds the
// reference's +128 rounding, motion.cpp:45), the vertical pass on 16x2
// packed lanes.  Ring slots are read with ld.global.cg (L2) as elsewhere;
// each word's 15 (gauss) / 5 (median) loads are independent and issued
// together (a variant sharing neighbour words through shuffles measured
// 2-3x slower: tools/probe_resident_profile.py).
__device__ __forceinline__ unsigned m_prmt(unsigned a, unsigned b, unsigned sel) {
  unsigned d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
constexpr unsigned mW8(unsigned a, unsigned b, unsigned c, unsigned d) { return a | (b << 8) | (c << 16) | (d << 24); }

// Gauss of the 4 px of word C (neighbour words L, R) in one row: 16x2 pairs.
__device__ __forceinline__ void m_hgauss4(unsigned L, unsigned C, unsigned R, unsigned& p01, unsigned& p23) {
  const unsigned h0 = __dp4a(L, mW8(0, 0, 1, 4), __dp4a(C, mW8(6, 4, 1, 0), 8u));
  const unsigned h1 = __dp4a(L, mW8(0, 0, 0, 1), __dp4a(C, mW8(4, 6, 4, 1), 8u));
  const unsigned h2 = __dp4a(C, mW8(1, 4, 6, 4), __dp4a(R, mW8(1, 0, 0, 0), 8u));
  const unsigned h3 = __dp4a(C, mW8(0, 1, 4, 6), __dp4a(R, mW8(4, 1, 0, 0), 8u));
  p01 = h1 * 65536u + h0;
  p23 = h3 * 65536u + h2;
}

__device__ void fire_gauss4(const ActorDesc& A, const Frame& F, const Group& G, unsigned W, unsigned H) {
  const unsigned Wq = W / 4;
  const unsigned long long Sq = (unsigned long long)Wq * H, totalq = Sq * A.in[0].rate;
  for (unsigned long long k = G.first(); k < totalq; k += G.step()) {
    const unsigned long long f = k / Sq, idx = k % Sq;
    const unsigned y = (unsigned)(idx / Wq), xq = (unsigned)(idx % Wq);
    const unsigned* fr = reinterpret_cast<const unsigned*>(F.in_ptr[0]) + f * Sq;
    const unsigned c = __ldcg(fr + idx);
    unsigned v = c;  // rows y < 2 or >= H-2: gray copied (motion.cpp:34-37)
    if (y >= 2 && y < H - 2) {
      unsigned a0 = 0, a1 = 0;
#pragma unroll
      for (int dy = -2; dy <= 2; ++dy) {
        const unsigned* row = fr + (unsigned long long)(y + dy) * Wq + xq;
        const unsigned C = dy == 0 ? c : __ldcg(row);
        const unsigned L = xq > 0 ? __ldcg(row - 1) : 0u, R = xq + 1 < Wq ? __ldcg(row + 1) : 0u;
        unsigned p01, p23;
        m_hgauss4(L, C, R, p01, p23);
        const unsigned w = dy == 0 ? 6u : (dy == -1 || dy == 1) ? 4u : 1u;
        a0 += w * p01;
        a1 += w * p23;
      }
      v = m_prmt(a0, a1, 0x7531);  // (sum + 128) >> 8 per px: byte 1 of each 16-bit lane
      // Columns x < 2 or x >= W-2: gray copied.
      const unsigned x = 4 * xq;
      if (x < 2) v = (v & 0xFFFF0000u) | (c & 0x0000FFFFu);
      if (x + 4 > W - 2) v = (v & 0x0000FFFFu) | (c & 0xFFFF0000u);
    }
    for (unsigned o = 0; o < A.n_out; ++o) {
      reinterpret_cast<unsigned*>(F.out_ptr[o])[k] = v;
      // Fig. 2 phase-2 copy (slot 3r -> slot 0, channel.cpp:97-104) done by
      // the writer of each word instead of the leader CTA afterwards.
      const unsigned long long last = (unsigned long long)(A.out[o].rate - 1) * Sq;
      if (((F.out_wrap >> o) & 1u) && k >= last) reinterpret_cast<unsigned*>(A.out[o].storage)[k - last] = v;
    }
  }
}

__device__ __forceinline__ void m_sort2(unsigned& p, unsigned& q) {
  const unsigned t = __vminu4(p, q);
  q = __vmaxu4(p, q);
  p = t;
}

__device__ void fire_median4(const ActorDesc& A, const Frame& F, const Group& G, unsigned W, unsigned H) {
  const unsigned Wq = W / 4;
  const unsigned long long Sq = (unsigned long long)Wq * H, totalq = Sq * A.in[0].rate;
  for (unsigned long long k = G.first(); k < totalq; k += G.step()) {
    const unsigned long long f = k / Sq, idx = k % Sq;
    const unsigned y = (unsigned)(idx / Wq), xq = (unsigned)(idx % Wq);
    const unsigned* fr = reinterpret_cast<const unsigned*>(F.in_ptr[0]) + f * Sq;
    const unsigned c = __ldcg(fr + idx);
    unsigned v = c;  // rows 0 and H-1: copied (motion.cpp:64-67)
    if (y >= 1 && y < H - 1) {
      unsigned a = c, b = __ldcg(fr + idx - Wq), cc = __ldcg(fr + idx + Wq);
      const unsigned lw = xq > 0 ? __ldcg(fr + idx - 1) : 0u, rw = xq + 1 < Wq ? __ldcg(fr + idx + 1) : 0u;
      unsigned d = __funnelshift_l(lw, c, 8), e = __funnelshift_r(c, rw, 8);  // left / right neighbours
      // median of 5 per byte: the scalar actor's sorting network on 4 lanes
      m_sort2(a, b); m_sort2(d, e); m_sort2(a, cc); m_sort2(b, cc); m_sort2(a, d);
      m_sort2(cc, d); m_sort2(b, e); m_sort2(b, cc); m_sort2(d, e);
      v = cc;
      const unsigned x = 4 * xq;
      if (x == 0) v = (v & 0xFFFFFF00u) | (c & 0xFFu);              // column 0 copied
      if (x + 4 == W) v = (v & 0x00FFFFFFu) | (c & 0xFF000000u);    // column W-1 copied
    }
    reinterpret_cast<unsigned*>(F.out_ptr[0])[k] = v;
  }
}

// 16 px per thread (frames with W % 16 == 0, 16-byte aligned regions): one
// 16-byte load per row plus the two neighbour words, so a gauss output word
// costs 15/4 load requests instead of 15, a median word 5/4 instead of 5.
#ifndef DF_NET_V16
#define DF_NET_V16 1
#endif
#ifndef DF_NET_NCH
#define DF_NET_NCH 2
#endif
// NCH adjacent 16-px chunks per thread (the row's chunk count a multiple of
// NCH): per row NCH 16-byte loads plus the two outer neighbour words.
template <int NCH>
__device__ void gauss16_n(const ActorDesc& A, const Frame& F, const Group& G, unsigned W, unsigned H) {
  const unsigned Wc = W / 16 / NCH, Wq = W / 4;  // Wc: thread items per row
  const unsigned long long Sc = (unsigned long long)Wc * H, Sq = (unsigned long long)Wq * H, total = Sc * A.in[0].rate;
  for (unsigned long long k = G.first(); k < total; k += G.step()) {
    const unsigned long long f = k / Sc, idx = k % Sc;
    const unsigned y = (unsigned)(idx / Wc), xc = (unsigned)(idx % Wc);
    const unsigned* fr = reinterpret_cast<const unsigned*>(F.in_ptr[0]) + f * Sq;
    const unsigned long long cw = (unsigned long long)y * Wq + 4ull * NCH * xc;  // first word of the item
    uint4 c[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) c[j] = __ldcg(reinterpret_cast<const uint4*>(fr + cw) + j);
    uint4 v[NCH];
#pragma unroll
    for (int j = 0; j < NCH; ++j) v[j] = c[j];  // rows y < 2 or >= H-2: gray copied (motion.cpp:34-37)
    if (y >= 2 && y < H - 2) {
      unsigned a0[4 * NCH] = {}, a1[4 * NCH] = {};
#pragma unroll
      for (int dy = -2; dy <= 2; ++dy) {
        const unsigned* row = fr + cw + (long long)dy * Wq;
        unsigned wd[4 * NCH + 2];
        wd[0] = xc > 0 ? __ldcg(row - 1) : 0u;
        wd[4 * NCH + 1] = xc + 1 < Wc ? __ldcg(row + 4 * NCH) : 0u;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const uint4 C = dy == 0 ? c[j] : __ldcg(reinterpret_cast<const uint4*>(row) + j);
          wd[1 + 4 * j] = C.x, wd[2 + 4 * j] = C.y, wd[3 + 4 * j] = C.z, wd[4 + 4 * j] = C.w;
        }
        const unsigned w = dy == 0 ? 6u : (dy == -1 || dy == 1) ? 4u : 1u;
#pragma unroll
        for (int i = 0; i < 4 * NCH; ++i) {
          unsigned p01, p23;
          m_hgauss4(wd[i], wd[i + 1], wd[i + 2], p01, p23);
          a0[i] += w * p01, a1[i] += w * p23;
        }
      }
#pragma unroll
      for (int j = 0; j < NCH; ++j)
        v[j] = make_uint4(m_prmt(a0[4 * j], a1[4 * j], 0x7531), m_prmt(a0[4 * j + 1], a1[4 * j + 1], 0x7531),
                          m_prmt(a0[4 * j + 2], a1[4 * j + 2], 0x7531), m_prmt(a0[4 * j + 3], a1[4 * j + 3], 0x7531));
      // Columns x < 2 or x >= W-2: gray copied.
      if (xc == 0) v[0].x = (v[0].x & 0xFFFF0000u) | (c[0].x & 0x0000FFFFu);
      if (xc + 1 == Wc) v[NCH - 1].w = (v[NCH - 1].w & 0x0000FFFFu) | (c[NCH - 1].w & 0xFFFF0000u);
    }
    for (unsigned o = 0; o < A.n_out; ++o) {
      const unsigned long long last = (unsigned long long)(A.out[o].rate - 1) * Sc;
      const bool wrap = ((F.out_wrap >> o) & 1u) && k >= last;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        reinterpret_cast<uint4*>(F.out_ptr[o])[NCH * k + j] = v[j];
        // Fig. 2 phase-2 copy (slot 3r -> slot 0, channel.cpp:97-104) by the writer
        if (wrap) reinterpret_cast<uint4*>(A.out[o].storage)[NCH * (k - last) + j] = v[j];
      }
    }
  }
}

__device__ void fire_gauss16(const ActorDesc& A, const Frame& F, const Group& G, unsigned W, unsigned H) {
  const unsigned Wc = W / 16, Wq = W / 4;
  const unsigned long long Sc = (unsigned long long)Wc * H, Sq = (unsigned long long)Wq * H, total = Sc * A.in[0].rate;
  for (unsigned long long k = G.first(); k < total; k += G.step()) {
    const unsigned long long f = k / Sc, idx = k % Sc;
    const unsigned y = (unsigned)(idx / Wc), xc = (unsigned)(idx % Wc);
    const unsigned* fr = reinterpret_cast<const unsigned*>(F.in_ptr[0]) + f * Sq;  // frame f, in words
    const unsigned long long cw = (unsigned long long)y * Wq + 4ull * xc;          // this chunk's first word
    const uint4 c = __ldcg(reinterpret_cast<const uint4*>(fr + cw));
    uint4 v = c;  // rows y < 2 or >= H-2: gray copied (motion.cpp:34-37)
    if (y >= 2 && y < H - 2) {
      unsigned a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
#pragma unroll
      for (int dy = -2; dy <= 2; ++dy) {
        const unsigned* row = fr + cw + (long long)dy * Wq;
        const uint4 C = dy == 0 ? c : __ldcg(reinterpret_cast<const uint4*>(row));
        const unsigned L = xc > 0 ? __ldcg(row - 1) : 0u, R = xc + 1 < Wc ? __ldcg(row + 4) : 0u;
        const unsigned w = dy == 0 ? 6u : (dy == -1 || dy == 1) ? 4u : 1u;
        unsigned p01, p23;
        m_hgauss4(L, C.x, C.y, p01, p23);
        a0[0] += w * p01, a1[0] += w * p23;
        m_hgauss4(C.x, C.y, C.z, p01, p23);
        a0[1] += w * p01, a1[1] += w * p23;
        m_hgauss4(C.y, C.z, C.w, p01, p23);
        a0[2] += w * p01, a1[2] += w * p23;
        m_hgauss4(C.z, C.w, R, p01, p23);
        a0[3] += w * p01, a1[3] += w * p23;
      }
      // (sum + 128) >> 8 per px: byte 1 of each 16-bit lane
      v = make_uint4(m_prmt(a0[0], a1[0], 0x7531), m_prmt(a0[1], a1[1], 0x7531), m_prmt(a0[2], a1[2], 0x7531),
                     m_prmt(a0[3], a1[3], 0x7531));
      // Columns x < 2 or x >= W-2: gray copied.
      if (xc == 0) v.x = (v.x & 0xFFFF0000u) | (c.x & 0x0000FFFFu);
      if (xc + 1 == Wc) v.w = (v.w & 0x0000FFFFu) | (c.w & 0xFFFF0000u);
    }
    for (unsigned o = 0; o < A.n_out; ++o) {
      reinterpret_cast<uint4*>(F.out_ptr[o])[k] = v;
      // Fig. 2 phase-2 copy (slot 3r -> slot 0, channel.cpp:97-104) done by
      // the writer of each chunk instead of the leader CTA afterwards.
      const unsigned long long last = (unsigned long long)(A.out[o].rate - 1) * Sc;
      if (((F.out_wrap >> o) & 1u) && k >= last) reinterpret_cast<uint4*>(A.out[o].storage)[k - last] = v;
    }
  }
}

__device__ __forceinline__ unsigned m_med5w(unsigned c, unsigned up, unsigned dn, unsigned lw, unsigned rw) {
  unsigned a = c, b = up, cc = dn;
  unsigned d = __funnelshift_l(lw, c, 8), e = __funnelshift_r(c, rw, 8);  // left / right neighbours
  // median of 5 per byte: the scalar actor's sorting network on 4 lanes
  m_sort2(a, b); m_sort2(d, e); m_sort2(a, cc); m_sort2(b, cc); m_sort2(a, d);
  m_sort2(cc, d); m_sort2(b, e); m_sort2(b, cc); m_sort2(d, e);
  return cc;
}

__device__ void fire_median16(const ActorDesc& A, const Frame& F, const Group& G, unsigned W, unsigned H) {
  const unsigned Wc = W / 16, Wq = W / 4;
  const unsigned long long Sc = (unsigned long long)Wc * H, Sq = (unsigned long long)Wq * H, total = Sc * A.in[0].rate;
  for (unsigned long long k = G.first(); k < total; k += G.step()) {
    const unsigned long long f = k / Sc, idx = k % Sc;
    const unsigned y = (unsigned)(idx / Wc), xc = (unsigned)(idx % Wc);
    const unsigned* fr = reinterpret_cast<const unsigned*>(F.in_ptr[0]) + f * Sq;
    const unsigned long long cw = (unsigned long long)y * Wq + 4ull * xc;
    const uint4 c = __ldcg(reinterpret_cast<const uint4*>(fr + cw));
    uint4 v = c;  // rows 0 and H-1: copied (motion.cpp:64-67)
    if (y >= 1 && y < H - 1) {
      const uint4 u = __ldcg(reinterpret_cast<const uint4*>(fr + cw - Wq));
      const uint4 dn = __ldcg(reinterpret_cast<const uint4*>(fr + cw + Wq));
      const unsigned lw = xc > 0 ? __ldcg(fr + cw - 1) : 0u, rw = xc + 1 < Wc ? __ldcg(fr + cw + 4) : 0u;
      v.x = m_med5w(c.x, u.x, dn.x, lw, c.y);
      v.y = m_med5w(c.y, u.y, dn.y, c.x, c.z);
      v.z = m_med5w(c.z, u.z, dn.z, c.y, c.w);
      v.w = m_med5w(c.w, u.w, dn.w, c.z, rw);
      if (xc == 0) v.x = (v.x & 0xFFFFFF00u) | (c.x & 0xFFu);              // column 0 copied
      if (xc + 1 == Wc) v.w = (v.w & 0x00FFFFFFu) | (c.w & 0xFF000000u);   // column W-1 copied
    }
    reinterpret_cast<uint4*>(F.out_ptr[0])[k] = v;
  }
}

__device__ __forceinline__ bool chunks16_ok(const Frame& F, const ActorDesc& A, unsigned W) {
  uintptr_t m = W & 15u;
  for (unsigned p = 0; p < A.n_in; ++p) m |= reinterpret_cast<uintptr_t>(F.in_ptr[p]);
  for (unsigned p = 0; p < A.n_out; ++p) m |= reinterpret_cast<uintptr_t>(F.out_ptr[p]) | reinterpret_cast<uintptr_t>(A.out[p].storage);
  return DF_NET_V16 && (m & 15u) == 0;
}

__device__ __forceinline__ bool words_ok(const Frame& F, const ActorDesc& A, unsigned W) {
  uintptr_t m = W & 3u;
  for (unsigned p = 0; p < A.n_in; ++p) m |= reinterpret_cast<uintptr_t>(F.in_ptr[p]);
  for (unsigned p = 0; p < A.n_out; ++p) m |= reinterpret_cast<uintptr_t>(F.out_ptr[p]);
  return (m & 3u) == 0;
}

__device__ void fire_kind(const ActorDesc& A, const Frame& F, const Group& G, ActorRt* rt, float2* win) {
  switch (A.kind) {
    case DF_ACT_DPD_SOURCE: {  // dpd.cpp:189-204
      const df_act_samples& P = params<df_act_samples>(A);
      const float2* x = reinterpret_cast<const float2*>(P.samples) + F.firing * P.period;
      float* re = reinterpret_cast<float*>(F.out_ptr[0]);
      float* im = reinterpret_cast<float*>(F.out_ptr[1]);
      batched<4, float2>(G, P.period, [&](unsigned long long k) { return x[k]; },
                         [&](unsigned long long k, const float2& v) {
                           re[k] = v.x;
                           im[k] = v.y;
                         });
      break;
    }
    case DF_ACT_DPD_SINK: {  // dpd.cpp:333-347
      const df_act_samples& P = params<df_act_samples>(A);
      float2* y = reinterpret_cast<float2*>(P.samples) + F.firing * P.period;
      const float* re = reinterpret_cast<const float*>(F.in_ptr[0]);
      const float* im = reinterpret_cast<const float*>(F.in_ptr[1]);
      batched<4, float2>(G, P.period, [&](unsigned long long k) { return make_float2(__ldcg(re + k), __ldcg(im + k)); },
                         [&](unsigned long long k, const float2& v) { y[k] = v; });
      break;
    }
    case DF_ACT_DPD_CONFIG: {  // dpd.cpp:206-221: the same LE token on every output
      const df_act_config& P = params<df_act_config>(A);
      const unsigned v = P.schedule[F.firing % P.len];
      for (unsigned long long k = G.first(); k < 4ull * A.n_out; k += G.step()) {
        const unsigned o = (unsigned)(k / 4), byte = (unsigned)(k % 4);
        if ((F.out_on >> o) & 1u) F.out_ptr[o][byte] = (unsigned char)(v >> (8 * byte));
      }
      break;
    }
    case DF_ACT_DPD_SPLIT: {  // dpd.cpp:246-256: inputs 0,1 (re, im) -> active pairs
      // Every output of a pair carries the same plane: load each 16-byte
      // word of re and im once and store it to every active output, so a
      // firing costs one load latency instead of one per active output.
      const unsigned long long bytes = (unsigned long long)A.in[0].rate * A.in[0].token_size;
      uintptr_t al = reinterpret_cast<uintptr_t>(F.in_ptr[0]) | reinterpret_cast<uintptr_t>(F.in_ptr[1]) | bytes;
      for (unsigned o = 0; o < A.n_out; ++o)
        if ((F.out_on >> o) & 1u) al |= reinterpret_cast<uintptr_t>(F.out_ptr[o]);
      if ((al & 15) == 0 && A.in[1].rate * A.in[1].token_size == bytes) {
        split_planes(A, F, G, bytes / 16);
        break;
      }
      for (unsigned o = 0; o < A.n_out; ++o)
        if ((F.out_on >> o) & 1u)
          copy_bytes(F.out_ptr[o], F.in_ptr[o & 1], (unsigned long long)A.out[o].rate * A.out[o].token_size, G);
      break;
    }
    case DF_ACT_DPD_BRANCH:
      fire_dpd_branch(A, F, G, win);
      break;
    case DF_ACT_DPD_ADDER: {  // dpd.cpp:306-320: +0.0f, then active inputs in port order
      const unsigned n = (unsigned)(A.out[0].token_size / 4) * A.out[0].rate;
      float* ore = reinterpret_cast<float*>(F.out_ptr[0]);
      float* oim = reinterpret_cast<float*>(F.out_ptr[1]);
      for (unsigned long long s0 = G.first(); s0 < n; s0 += 2 * G.step()) {
        // two outputs per iteration: their loads are independent
        const unsigned long long s1 = s0 + G.step();
        const bool two = s1 < n;
        float r0 = 0.0f, i0 = 0.0f, r1 = 0.0f, i1 = 0.0f;
        // Unrolled over the (at most 10) input pairs so every active input's
        // loads are issued before the adds consume them.
#pragma unroll
        for (unsigned p = 0; p + 1 < 2 * kMaxPairs && p + 1 < A.n_in; p += 2) {
          if (!((F.in_on >> p) & 1u)) continue;
          const float* pr = reinterpret_cast<const float*>(F.in_ptr[p]);
          const float* pi = reinterpret_cast<const float*>(F.in_ptr[p + 1]);
          const float a0 = __ldcg(pr + s0), b0 = __ldcg(pi + s0);
          const float a1 = two ? __ldcg(pr + s1) : 0.f, b1 = two ? __ldcg(pi + s1) : 0.f;
          r0 = __fadd_rn(r0, a0);
          i0 = __fadd_rn(i0, b0);
          r1 = __fadd_rn(r1, a1);
          i1 = __fadd_rn(i1, b1);
        }
        ore[s0] = r0;
        oim[s0] = i0;
        if (two) {
          ore[s1] = r1;
          oim[s1] = i1;
        }
      }
      break;
    }
    case DF_ACT_TEST_PRODUCE: {
      if (!(F.out_on & 1u)) break;
      const df_act_test& P = params<df_act_test>(A);
      const DevChan& c = A.out[0];
      const unsigned long long first = rt->state[0];
      for (unsigned long long k = G.first(); k < (unsigned long long)c.rate * c.token_size; k += G.step())
        F.out_ptr[0][k] = token_byte(P.seed, first + k / c.token_size, k % c.token_size);
      break;
    }
    case DF_ACT_TEST_CONSUME: {
      if (!(F.in_on & 1u)) break;
      const df_act_test& P = params<df_act_test>(A);
      const DevChan& c = A.in[0];
      const unsigned long long first = rt->state[0];
      unsigned long long bad = 0;
      for (unsigned long long k = G.first(); k < (unsigned long long)c.rate * c.token_size; k += G.step()) {
        const unsigned long long pos = first + k / c.token_size;
        const unsigned char want = P.skip_initial ? (pos == 0 ? 0 : token_byte(P.seed, pos - 1, k % c.token_size))
                                                  : token_byte(P.seed, pos, k % c.token_size);
        bad += __ldcg(F.in_ptr[0] + k) != want;
      }
      if (bad) atomicAdd(reinterpret_cast<unsigned long long*>(P.counters) + 1, bad);
      break;
    }
    case DF_ACT_FRAME_SOURCE: {  // motion.cpp:123-129: r frames per firing
      const df_act_frames& P = params<df_act_frames>(A);
      const unsigned long long bytes = (unsigned long long)A.out[0].rate * A.out[0].token_size;
      copy_bytes(F.out_ptr[0], reinterpret_cast<const unsigned char*>(P.frames) + F.firing * bytes, bytes, G);
      break;
    }
    case DF_ACT_FRAME_SINK: {  // motion.cpp:178-183
      const df_act_frames& P = params<df_act_frames>(A);
      const unsigned long long bytes = (unsigned long long)A.in[0].rate * A.in[0].token_size;
      copy_bytes(reinterpret_cast<unsigned char*>(P.frames) + F.firing * bytes, F.in_ptr[0], bytes, G);
      break;
    }
    case DF_ACT_GAUSS: {  // gauss5x5 (motion.cpp:27-48) of every frame, to every output
      const df_act_frames& P = params<df_act_frames>(A);
      const unsigned W = P.width, H = P.height;
      if (DF_NET_NCH == 2 && W % 32 == 0 && W >= 64 && H >= 5 && chunks16_ok(F, A, W)) {
        gauss16_n<2>(A, F, G, W, H);
        break;
      }
      if (W >= 32 && H >= 5 && chunks16_ok(F, A, W)) {
        fire_gauss16(A, F, G, W, H);
        break;
      }
      if (W >= 8 && H >= 5 && words_ok(F, A, W)) {
        fire_gauss4(A, F, G, W, H);
        break;
      }
      const unsigned long long S = (unsigned long long)W * H, total = S * A.in[0].rate;
      const unsigned char* in = F.in_ptr[0];
      for (unsigned long long k = G.first(); k < total; k += G.step()) {
        const unsigned long long f = k / S, idx = k % S;
        const unsigned y = (unsigned)(idx / W), x = (unsigned)(idx % W);
        const unsigned char* fr = in + f * S;
        unsigned v;
        if (y < 2 || y >= H - 2 || x < 2 || x >= W - 2) {
          v = __ldcg(fr + idx);
        } else {
          const int bn[5] = {1, 4, 6, 4, 1};
          int acc = 0;
          for (int dy = -2; dy <= 2; ++dy)
            for (int dx = -2; dx <= 2; ++dx)
              acc += bn[dy + 2] * bn[dx + 2] * (int)__ldcg(fr + (unsigned long long)(y + dy) * W + (x + dx));
          v = (unsigned)((acc + 128) >> 8);
        }
        for (unsigned o = 0; o < A.n_out; ++o) {
          F.out_ptr[o][k] = (unsigned char)v;
          const unsigned long long last = (unsigned long long)(A.out[o].rate - 1) * S;  // phase-2 copy inline
          if (((F.out_wrap >> o) & 1u) && k >= last) A.out[o].storage[k - last] = (unsigned char)v;
        }
      }
      break;
    }
    case DF_ACT_THRES: {  // thres_diff (motion.cpp:50-57): in0 prev, in1 cur
      const df_act_frames& P = params<df_act_frames>(A);
      const unsigned long long total = (unsigned long long)A.in[0].rate * A.in[0].token_size;
      if (((reinterpret_cast<uintptr_t>(F.in_ptr[0]) | reinterpret_cast<uintptr_t>(F.in_ptr[1]) |
            reinterpret_cast<uintptr_t>(F.out_ptr[0]) | total) & 3) == 0) {
        // 4 px per word: |cur - prev| per byte (VABSDIFF4), > thr per byte -> 0xFF
        const unsigned* prev = reinterpret_cast<const unsigned*>(F.in_ptr[0]);
        const unsigned* cur = reinterpret_cast<const unsigned*>(F.in_ptr[1]);
        unsigned* out = reinterpret_cast<unsigned*>(F.out_ptr[0]);
        const unsigned thr4 = 0x01010101u * P.threshold;
        batched<4, uint2>(G, total / 4, [&](unsigned long long k) { return make_uint2(__ldcg(prev + k), __ldcg(cur + k)); },
                          [&](unsigned long long k, const uint2& v) { out[k] = __vcmpgtu4(__vabsdiffu4(v.y, v.x), thr4); });
      } else {
        for (unsigned long long k = G.first(); k < total; k += G.step()) {
          const int d = (int)__ldcg(F.in_ptr[1] + k) - (int)__ldcg(F.in_ptr[0] + k);
          F.out_ptr[0][k] = (d < 0 ? -d : d) > (int)P.threshold ? 255 : 0;
        }
      }
      break;
    }
    case DF_ACT_MEDIAN: {  // median5 (motion.cpp:59-74): plus-shaped median, 1-px border copy
      const df_act_frames& P = params<df_act_frames>(A);
      const unsigned W = P.width, H = P.height;
      if (W >= 32 && H >= 3 && chunks16_ok(F, A, W)) {
        fire_median16(A, F, G, W, H);
        break;
      }
      if (W >= 8 && H >= 3 && words_ok(F, A, W)) {
        fire_median4(A, F, G, W, H);
        break;
      }
      const unsigned long long S = (unsigned long long)W * H, total = S * A.in[0].rate;
      for (unsigned long long k = G.first(); k < total; k += G.step()) {
        const unsigned long long f = k / S, idx = k % S;
        const unsigned y = (unsigned)(idx / W), x = (unsigned)(idx % W);
        const unsigned char* fr = F.in_ptr[0] + f * S;
        unsigned v;
        if (y == 0 || y == H - 1 || x == 0 || x == W - 1) {
          v = __ldcg(fr + idx);
        } else {
          unsigned a = __ldcg(fr + idx), b = __ldcg(fr + idx - W), c = __ldcg(fr + idx + W), d = __ldcg(fr + idx - 1),
                   e = __ldcg(fr + idx + 1);
          // median of 5: max(min(max(a,b), max(c,d)), min(...)) via a sorting network
          unsigned t;
#define DF_SORT2(p, q) t = min(p, q), q = max(p, q), p = t
          DF_SORT2(a, b); DF_SORT2(d, e); DF_SORT2(a, c); DF_SORT2(b, c); DF_SORT2(a, d);
          DF_SORT2(c, d); DF_SORT2(b, e); DF_SORT2(b, c); DF_SORT2(d, e);
#undef DF_SORT2
          v = c;
        }
        F.out_ptr[0][k] = (unsigned char)v;
      }
      break;
    }
    default:
      break;
  }
}

// Leader CTA, after every CTA fired: kind state that needs the whole firing.
__device__ void post_kind(const ActorDesc& A, const Frame& F, ActorRt* rt) {
  switch (A.kind) {
    case DF_ACT_DPD_BRANCH:
      post_dpd_branch(A, F);
      break;
    case DF_ACT_TEST_PRODUCE:
    case DF_ACT_TEST_CONSUME: {
      const bool on = A.kind == DF_ACT_TEST_PRODUCE ? (F.out_on & 1u) : (F.in_on & 1u);
      const DevChan& c = A.kind == DF_ACT_TEST_PRODUCE ? A.out[0] : A.in[0];
      if (on && threadIdx.x == 0) {
        rt->state[0] += c.rate;
        *params<df_act_test>(A).counters = rt->state[0];
      }
      break;
    }
    default:
      break;
  }
}

// Leader, after the loop: close outputs, then drain inputs until their
// producers close (runtime.cpp:223-229, drain_channel :199-204).
__device__ void leader_finish(const ActorDesc& A, int a, ActorRt* rt, NetCtl* ctl, bool aborted,
                              unsigned long long* poll, Phases& ph) {
  rt->t_stop = now_ns();
  for (unsigned p = 0; p < A.n_out; ++p) close_channel(A.out[p]);
  if (aborted) return;
  auto drain = [&](const DevChan& c, unsigned& phase) {  // discards: nothing is read before the release
    while (wait_readable(c, c.rate, ctl, a, poll) == kOk) commit_read(c, c.rate, phase);
  };
  for (unsigned p = 0; p < A.n_in; ++p) drain(A.in[p], ph.in[p]);
  if (A.has_ctrl) drain(A.ctrl, ph.ctrl);
}

__global__ void __launch_bounds__(kNetThreads, 4) net_kernel(const ActorDesc* __restrict__ actors, unsigned n_actors,
                                                          ActorRt* rts, NetCtl* ctl) {
  __shared__ int s_actor;
  __shared__ Frame s_frame;
  __shared__ float2 win[kBranchV * kNetThreads + 32];  // DPD branch window (chunk + T-1 history)
  __shared__ bool s_aborted;
  __shared__ Phases s_ph;  // leader CTA: the actor's endpoint phases
  __shared__ unsigned long long s_t;  // leader: timestamp of the current phase
  if (threadIdx.x == 0) {
    s_actor = -1;
    for (unsigned a = 0; a < n_actors; ++a)
      if (blockIdx.x >= actors[a].cta0 && blockIdx.x < actors[a].cta0 + actors[a].ctas) s_actor = (int)a;
    s_aborted = false;
  }
  __syncthreads();
  const int a = s_actor;
  if (a < 0) return;
  const ActorDesc& A = actors[a];
  ActorRt* rt = rts + a;
  const Group G{blockIdx.x - A.cta0, A.ctas};
  const bool leader_cta = G.g == 0;
  if (leader_cta && threadIdx.x < kMaxPorts) {
    s_ph.in[threadIdx.x] = threadIdx.x < A.n_in ? A.in[threadIdx.x].st->read_phase : 0;
    s_ph.out[threadIdx.x] = threadIdx.x < A.n_out ? A.out[threadIdx.x].st->write_phase : 0;
    if (threadIdx.x == 0) s_ph.ctrl = A.has_ctrl ? A.ctrl.st->read_phase : 0;
  }
  __syncthreads();
  unsigned gen = 0;
  unsigned long long host_poll = 0;  // leader thread: last poll of the host abort word
  for (;;) {
    if (threadIdx.x == 0) {
      if (leader_cta) {
        bool ab = false;
        const unsigned long long t0 = now_ns();
        leader_prepare(A, a, rt, ctl, &ab, &host_poll, s_ph);
        s_aborted = ab;
        const unsigned long long t1 = now_ns();
        rt->t_wait += t1 - t0;
        s_t = t1;
      } else {
        Spin s;
        s.watchdog = false;  // the leader's own waits carry the watchdog
        while (ld_acq32(&rt->gen) == gen)
          if (s.tick(ctl, a) != kOk) break;  // an abort cannot strand this CTA
      }
      if (ld_acq32(&rt->gen) == gen) {
        s_frame.stop = 1;  // aborted while waiting
      } else {
        const volatile Frame* vf = &rt->frame;
        s_frame.firing = vf->firing;
        s_frame.stop = vf->stop;
        s_frame.in_on = vf->in_on;
        s_frame.out_on = vf->out_on;
        s_frame.out_wrap = vf->out_wrap;
        for (unsigned p = 0; p < A.n_in; ++p) s_frame.in_ptr[p] = vf->in_ptr[p];
        for (unsigned p = 0; p < A.n_out; ++p) s_frame.out_ptr[p] = vf->out_ptr[p];
      }
    }
    __syncthreads();
    ++gen;
    if (s_frame.stop) break;
    fire_kind(A, s_frame, G, rt, win);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&rt->done, 1u);
    }
    if (!leader_cta) continue;
    if (threadIdx.x == 0) {
      Spin s;
      s.watchdog = false;
      bool ab = false;
      while (ld_acq32(&rt->done) < A.ctas)
        if (s.tick(ctl, a) != kOk) {
          ab = true;
          break;
        }
      rt->done = 0;
      s_aborted = ab;
      const unsigned long long t = now_ns();
      rt->t_fire += t - s_t;
      s_t = t;
    }
    __syncthreads();
    if (s_aborted) break;
    post_kind(A, s_frame, rt);
    // Fig. 2 phase-2 write: copy slot 3r into slot 0 (channel.cpp:97-104).
    for (unsigned p = 0; p < A.n_out; ++p)
      if (((s_frame.out_wrap >> p) & 1u) && A.kind != DF_ACT_GAUSS) {  // GAUSS writes it inline
        const DevChan& c = A.out[p];
        copy_bytes(c.storage, c.storage + 3ull * c.rate * c.token_size, c.token_size, Group{0, 1});
      }
    __syncthreads();
    // write_end / read_end of every port at once: lane p of warp 0 commits
    // output p and input p (each lane fences its own view first), instead
    // of one thread walking up to 48 ports.
    if (threadIdx.x < 32) {
      const unsigned p = threadIdx.x;
      __threadfence();
      if (p < A.n_out && ((s_frame.out_on >> p) & 1u)) commit_write(A.out[p], A.out[p].rate, s_ph.out[p]);
      if (p < A.n_in && ((s_frame.in_on >> p) & 1u)) commit_read(A.in[p], A.in[p].rate, s_ph.in[p]);
      if (p == 0) {
        ++rt->firings;
        rt->t_commit += now_ns() - s_t;
      }
    }
  }
  if (leader_cta && threadIdx.x == 0)
    leader_finish(A, a, rt, ctl, s_aborted || *(volatile unsigned*)&ctl->abort, &host_poll, s_ph);
}

}  // namespace
}  // namespace df

using namespace df;

struct df_net {
  int device = 0;
  std::vector<ActorDesc> actors;
  std::vector<std::vector<uint32_t>> tables;
  std::vector<df_channel*> channels;  // every channel bound (for endpoint bookkeeping)
  unsigned total_ctas = 0;
  ActorDesc* d_actors = nullptr;
  ActorRt* d_rt = nullptr;
  NetCtl* d_ctl = nullptr;
  uint32_t* d_tables = nullptr;
  unsigned* h_abort = nullptr;  // mapped pinned
  std::vector<ActorRt> rt;      // after a run
  NetCtl ctl{};
  bool ran = false;
};

namespace {
void net_free_device(df_net* n) {
  cudaFree(n->d_actors);
  cudaFree(n->d_rt);
  cudaFree(n->d_ctl);
  cudaFree(n->d_tables);
  n->d_actors = nullptr;
  n->d_rt = nullptr;
  n->d_ctl = nullptr;
  n->d_tables = nullptr;
}
size_t kind_params(int kind) {
  switch (kind) {
    case DF_ACT_DPD_SOURCE:
    case DF_ACT_DPD_SINK:
      return sizeof(df_act_samples);
    case DF_ACT_DPD_CONFIG:
      return sizeof(df_act_config);
    case DF_ACT_DPD_BRANCH:
      return sizeof(df_act_branch);
    case DF_ACT_TEST_PRODUCE:
    case DF_ACT_TEST_CONSUME:
      return sizeof(df_act_test);
    case DF_ACT_FRAME_SOURCE:
    case DF_ACT_FRAME_SINK:
    case DF_ACT_GAUSS:
    case DF_ACT_THRES:
    case DF_ACT_MEDIAN:
      return sizeof(df_act_frames);
    case DF_ACT_DPD_SPLIT:
    case DF_ACT_DPD_ADDER:
      return 0;
    default:
      return (size_t)-1;
  }
}
}  // namespace

extern "C" {

int df_net_create(int device, df_net** out) {
  DF_REQUIRE(out, DF_EINVAL, "df_net_create: null out pointer");
  DF_CHECK_CUDA(cudaSetDevice(device));
  auto* n = new df_net();
  n->device = device;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&n->h_abort), sizeof(unsigned), cudaHostAllocMapped);
  if (e != cudaSuccess) {
    delete n;
    return cuda_status(e, "df_net_create: cudaHostAlloc");
  }
  *n->h_abort = 0;
  *out = n;
  return DF_OK;
}

int df_net_destroy(df_net* n) {
  if (!n) return DF_OK;
  cudaSetDevice(n->device);
  net_free_device(n);
  cudaFreeHost(n->h_abort);
  delete n;
  return DF_OK;
}

int df_net_add_actor(df_net* n, int kind, const void* params, size_t params_bytes, uint32_t ctas, df_channel* control,
                     df_channel* const* inputs, size_t n_in, df_channel* const* outputs, size_t n_out,
                     uint64_t firing_limit, int* index) {
  DF_REQUIRE(n, DF_EINVAL, "df_net_add_actor: null network");
  const size_t need = kind_params(kind);
  DF_REQUIRE(need != (size_t)-1, DF_EINVAL, "df_net_add_actor: unknown actor kind %d", kind);
  DF_REQUIRE(params_bytes == need && (need == 0 || params), DF_EINVAL,
             "df_net_add_actor: kind %d takes %zu parameter bytes, got %zu", kind, need, params_bytes);
  DF_REQUIRE(n_in <= (size_t)kMaxPorts && n_out <= (size_t)kMaxPorts, DF_EINVAL,
             "df_net_add_actor: at most %d inputs and %d outputs", kMaxPorts, kMaxPorts);
  DF_REQUIRE(ctas >= 1, DF_EINVAL, "df_net_add_actor: an actor needs at least one CTA");
  DF_REQUIRE(!n->ran, DF_ELOGIC, "df_net_add_actor: the network already ran");
  ActorDesc A{};
  A.kind = kind;
  A.cta0 = n->total_ctas;
  A.ctas = ctas;
  A.n_in = (unsigned)n_in;
  A.n_out = (unsigned)n_out;
  A.limit = firing_limit;
  if (need) std::memcpy(A.params, params, need);
  auto bind = [&](df_channel* c, bool reader, DevChan& slot) -> int {
    DF_REQUIRE(c, DF_EINVAL, "df_net_add_actor: null channel");
    DF_REQUIRE(c->device == n->device, DF_EINVAL, "df_net_add_actor: channel on another device");
    Endpoint& ep = reader ? c->reader : c->writer;
    DF_REQUIRE(ep != Endpoint::host, DF_ELOGIC, "channel endpoint is host-driven; a network actor would race it");
    ep = Endpoint::device;
    slot = c->dev();
    n->channels.push_back(c);
    return DF_OK;
  };
  if (control) {
    DF_REQUIRE(!control->has_delay, DF_ELOGIC, "delay token on a channel into a control port");
    DF_REQUIRE(control->rate == 1, DF_ELOGIC, "control rate must be 1");
    DF_TRY(bind(control, true, A.ctrl));
    A.has_ctrl = 1;
  }
  for (size_t i = 0; i < n_in; ++i) DF_TRY(bind(inputs[i], true, A.in[i]));
  for (size_t i = 0; i < n_out; ++i) DF_TRY(bind(outputs[i], false, A.out[i]));
  // Kind port contracts (what fire_kind assumes).
  switch (kind) {
    case DF_ACT_DPD_SOURCE:
    case DF_ACT_DPD_SINK: {
      const auto& P = *static_cast<const df_act_samples*>(params);
      const size_t plane = (size_t)P.period * 4;
      const bool src = kind == DF_ACT_DPD_SOURCE;
      DF_REQUIRE((src ? n_out : n_in) == 2 && (src ? n_in : n_out) == 0 && P.samples && P.period, DF_EINVAL,
                 "dpd source/sink: two planes (re, im) and a sample buffer");
      for (int k = 0; k < 2; ++k) {
        const df_channel* c = src ? outputs[k] : inputs[k];
        DF_REQUIRE(c->token_size == plane && c->rate == 1, DF_EINVAL, "dpd source/sink: planes of `period` floats, rate 1");
      }
      break;
    }
    case DF_ACT_DPD_CONFIG:
      DF_REQUIRE(n_in == 0 && static_cast<const df_act_config*>(params)->len > 0, DF_EINVAL, "dpd config: no inputs, non-empty schedule");
      for (size_t i = 0; i < n_out; ++i)
        DF_REQUIRE(outputs[i]->token_size == 4 && outputs[i]->rate == 1, DF_EINVAL, "dpd config: 4-byte tokens, rate 1");
      break;
    case DF_ACT_DPD_SPLIT:
      DF_REQUIRE(n_in == 2 && n_out % 2 == 0, DF_EINVAL, "dpd split: inputs re, im; outputs in pairs");
      for (size_t i = 0; i < n_out; ++i)
        DF_REQUIRE(outputs[i]->token_size * outputs[i]->rate == inputs[i & 1]->token_size * inputs[i & 1]->rate,
                   DF_EINVAL, "dpd split: outputs carry the input planes");
      break;
    case DF_ACT_DPD_BRANCH: {
      const auto& P = *static_cast<const df_act_branch*>(params);
      DF_REQUIRE(n_in == 2 && n_out == 2, DF_EINVAL, "dpd branch: inputs re, im; outputs re, im");
      DF_REQUIRE(P.branch >= 1 && P.branch <= 10 && P.taps_per_branch >= 1 && P.taps_per_branch <= 32 && P.taps &&
                     (P.state || P.taps_per_branch == 1),
                 DF_EINVAL, "dpd branch: branch 1..10, 1..32 taps, taps and state buffers");
      for (int k = 0; k < 2; ++k)
        DF_REQUIRE(inputs[k]->token_size == (size_t)P.period * 4 && outputs[k]->token_size == (size_t)P.period * 4 &&
                       inputs[k]->rate == 1 && outputs[k]->rate == 1,
                   DF_EINVAL, "dpd branch: planes of `period` floats, rate 1");
      break;
    }
    case DF_ACT_DPD_ADDER:
      DF_REQUIRE(n_in % 2 == 0 && n_out == 2, DF_EINVAL, "dpd adder: input pairs, outputs re, im");
      for (size_t i = 0; i < n_in; ++i)
        DF_REQUIRE(inputs[i]->token_size * inputs[i]->rate == outputs[0]->token_size * outputs[0]->rate &&
                       outputs[0]->token_size % 4 == 0,
                   DF_EINVAL, "dpd adder: input planes match the output plane");
      break;
    case DF_ACT_TEST_PRODUCE:
      DF_REQUIRE(n_in == 0 && n_out == 1 && static_cast<const df_act_test*>(params)->counters, DF_EINVAL,
                 "test producer: one output and a counter buffer");
      break;
    case DF_ACT_TEST_CONSUME:
      DF_REQUIRE(n_in == 1 && n_out == 0 && static_cast<const df_act_test*>(params)->counters, DF_EINVAL,
                 "test consumer: one input and a counter buffer");
      break;
    default: {  // frame kinds
      const auto& P = *static_cast<const df_act_frames*>(params);
      const size_t S = (size_t)P.width * P.height;
      DF_REQUIRE(P.width >= 5 && P.height >= 5, DF_EINVAL, "motion: frame must be at least 5x5");
      const size_t ins = kind == DF_ACT_FRAME_SOURCE ? 0 : kind == DF_ACT_THRES ? 2 : 1;
      DF_REQUIRE(n_in == ins && (kind == DF_ACT_FRAME_SINK ? n_out == 0 : n_out >= 1), DF_EINVAL,
                 "frame actor kind %d: wrong port count", kind);
      DF_REQUIRE((kind != DF_ACT_FRAME_SOURCE && kind != DF_ACT_FRAME_SINK) || P.frames, DF_EINVAL,
                 "frame source/sink: null frame buffer");
      uint32_t r = 0;
      for (size_t i = 0; i < n_in + n_out; ++i) {
        const df_channel* c = i < n_in ? inputs[i] : outputs[i - n_in];
        DF_REQUIRE(c->token_size == S, DF_EINVAL, "frame actors: tokens are W*H bytes");
        if (!r) r = c->rate;
        DF_REQUIRE(c->rate == r, DF_EINVAL, "frame actors: every port at the same token rate");
      }
      break;
    }
  }
  n->actors.push_back(A);
  n->tables.emplace_back();
  n->total_ctas += ctas;
  if (index) *index = (int)n->actors.size() - 1;
  return DF_OK;
}

int df_net_set_control_table(df_net* n, int actor, const uint32_t* rows, uint32_t domain) {
  DF_REQUIRE(n && rows && domain > 0, DF_EINVAL, "df_net_set_control_table: null argument or empty domain");
  DF_REQUIRE(actor >= 0 && (size_t)actor < n->actors.size(), DF_EINVAL, "df_net_set_control_table: no actor %d", actor);
  DF_REQUIRE(n->actors[actor].has_ctrl, DF_EINVAL, "static actor with a control function");
  n->tables[actor].assign(rows, rows + 3ull * domain);
  n->actors[actor].domain = domain;
  return DF_OK;
}

int df_net_abort(df_net* n) {
  DF_REQUIRE(n, DF_EINVAL, "df_net_abort: null network");
  *(volatile unsigned*)n->h_abort = 1;
  return DF_OK;
}

int df_net_run(df_net* n, double timeout_s) {
  DF_REQUIRE(n, DF_EINVAL, "df_net_run: null network");
  DF_REQUIRE(!n->ran, DF_ELOGIC, "df_net_run: a network runs once (its channels hold the end state)");
  DF_REQUIRE(!n->actors.empty(), DF_EINVAL, "df_net_run: empty network");
  for (size_t a = 0; a < n->actors.size(); ++a)
    DF_REQUIRE(!n->actors[a].has_ctrl || n->actors[a].domain > 0, DF_EINVAL,
               "dynamic actor %zu without a control table", a);
  DF_CHECK_CUDA(cudaSetDevice(n->device));
  int per_sm = 0, sms = 0, coop = 0;
  DF_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, net_kernel, kNetThreads, 0));
  DF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, n->device));
  DF_CHECK_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, n->device));
  DF_REQUIRE(n->total_ctas <= (unsigned)(per_sm * sms), DF_EINVAL,
             "df_net_run: %u CTAs exceed the %d that can be co-resident", n->total_ctas, per_sm * sms);
  // Control tables, concatenated.
  std::vector<uint32_t> all;
  std::vector<size_t> off(n->actors.size(), 0);
  for (size_t a = 0; a < n->actors.size(); ++a) {
    off[a] = all.size();
    all.insert(all.end(), n->tables[a].begin(), n->tables[a].end());
  }
  if (all.empty()) all.assign(3, 0);
  DF_CHECK_CUDA(cudaMalloc(&n->d_tables, all.size() * sizeof(uint32_t)));
  DF_CHECK_CUDA(cudaMemcpy(n->d_tables, all.data(), all.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  std::vector<ActorDesc> desc = n->actors;
  for (size_t a = 0; a < desc.size(); ++a) desc[a].table = n->d_tables + off[a];
  DF_CHECK_CUDA(cudaMalloc(&n->d_actors, desc.size() * sizeof(ActorDesc)));
  DF_CHECK_CUDA(cudaMemcpy(n->d_actors, desc.data(), desc.size() * sizeof(ActorDesc), cudaMemcpyHostToDevice));
  DF_CHECK_CUDA(cudaMalloc(&n->d_rt, desc.size() * sizeof(ActorRt)));
  DF_CHECK_CUDA(cudaMemset(n->d_rt, 0, desc.size() * sizeof(ActorRt)));
  NetCtl ctl{};
  ctl.timeout_ns = (unsigned long long)((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
  unsigned* dev_abort = nullptr;
  DF_CHECK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev_abort), n->h_abort, 0));
  ctl.host_abort = dev_abort;
  DF_CHECK_CUDA(cudaMalloc(&n->d_ctl, sizeof(NetCtl)));
  DF_CHECK_CUDA(cudaMemcpy(n->d_ctl, &ctl, sizeof ctl, cudaMemcpyHostToDevice));
  DF_CHECK_CUDA(cudaDeviceSynchronize());  // channel initialisation and earlier host-endpoint work
  n->ran = true;
  unsigned na = (unsigned)desc.size();
  void* args[] = {&n->d_actors, &na, &n->d_rt, &n->d_ctl};
  cudaError_t e = coop ? cudaLaunchCooperativeKernel((const void*)net_kernel, dim3(n->total_ctas), dim3(kNetThreads), args, 0, nullptr)
                       : cudaLaunchKernel((const void*)net_kernel, dim3(n->total_ctas), dim3(kNetThreads), args, 0, nullptr);
  DF_CHECK_CUDA(e);
  DF_TRY(after_launch("net_kernel"));
  DF_CHECK_CUDA(cudaDeviceSynchronize());
  n->rt.resize(desc.size());
  DF_CHECK_CUDA(cudaMemcpy(n->rt.data(), n->d_rt, desc.size() * sizeof(ActorRt), cudaMemcpyDeviceToHost));
  DF_CHECK_CUDA(cudaMemcpy(&n->ctl, n->d_ctl, sizeof(NetCtl), cudaMemcpyDeviceToHost));
  for (df_channel* c : n->channels) c->closed_host = true;  // every output was closed on the device
  if (n->ctl.fault_code == DF_EABORTED) return set_error(DF_EABORTED, "run aborted");
  if (n->ctl.fault_code == DF_ECONTROL)
    return set_error(DF_ECONTROL, "actor %u: control token %u maps to no legal rates", n->ctl.fault_actor,
                     n->ctl.fault_token);
  if (n->ctl.fault_code == DF_ETIMEOUT)
    return set_error(DF_ETIMEOUT, "actor %u: waited longer than %.3g s on a channel (deadlock watchdog)",
                     n->ctl.fault_actor, timeout_s > 0 ? timeout_s : 30.0);
  if (n->ctl.fault_code) return set_error((int)n->ctl.fault_code, "actor %u faulted", n->ctl.fault_actor);
  return DF_OK;
}

int df_net_fault(const df_net* n, int* actor, int* code, uint32_t* token) {
  DF_REQUIRE(n, DF_EINVAL, "df_net_fault: null network");
  if (actor) *actor = n->ctl.fault_code ? (int)n->ctl.fault_actor : -1;
  if (code) *code = (int)n->ctl.fault_code;
  if (token) *token = n->ctl.fault_token;
  return DF_OK;
}

int df_net_actor_profile(const df_net* n, int actor, double* wait_ms, double* fire_ms, double* commit_ms) {
  DF_REQUIRE(n && actor >= 0 && (size_t)actor < n->actors.size(), DF_EINVAL, "df_net_actor_profile: no such actor");
  DF_REQUIRE(n->ran && n->rt.size() == n->actors.size(), DF_ELOGIC, "df_net_actor_profile: the network has not run");
  const ActorRt& r = n->rt[actor];
  if (wait_ms) *wait_ms = (double)r.t_wait / 1e6;
  if (fire_ms) *fire_ms = (double)r.t_fire / 1e6;
  if (commit_ms) *commit_ms = (double)r.t_commit / 1e6;
  return DF_OK;
}

int df_net_actor_stats(const df_net* n, int actor, uint64_t* firings, double* active_ms) {
  DF_REQUIRE(n && actor >= 0 && (size_t)actor < n->actors.size(), DF_EINVAL, "df_net_actor_stats: no such actor");
  DF_REQUIRE(n->ran && n->rt.size() == n->actors.size(), DF_ELOGIC, "df_net_actor_stats: the network has not run");
  const ActorRt& r = n->rt[actor];
  if (firings) *firings = r.firings;
  if (active_ms) *active_ms = r.firings && r.t_stop > r.t_first ? (double)(r.t_stop - r.t_first) / 1e6 : 0.0;
  return DF_OK;
}

}  // extern "C"
