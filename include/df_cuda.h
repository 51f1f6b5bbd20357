/*
 * df_cuda.h -- the C ABI of libdf_cuda.so, the B200 (sm_100a) GPU-actor
 * path of the dynflow dataflow framework (arXiv 1611.03226 artifact).
 *
 * This is the drop-in boundary.  Every entry point uses plain pointers,
 * sizes and opaque handles (no CUDA or C++ types), returns an int status
 * (DF_OK = 0) and leaves a thread-local message in df_last_error().
 * Stream arguments are cudaStream_t passed as void* (NULL = legacy default
 * stream).  Device pointers are never dereferenced by the host.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   channels      Channel, capacity_tokens, write_region/read_region
 *                 (include/dynflow/channel.hpp:15-135, src/channel.cpp:9-192)
 *   DPD actor     poly_branch + fir10 + dpd_adder behind the split / branch /
 *                 adder actors (src/dpd.cpp:60-145, :225-331), control tokens
 *                 ConfigToken (include/dynflow/dpd.hpp:26-45)
 *   DPD e2e       oracle_dpd / the dpd network run (src/dpd.cpp:151-391,
 *                 src/bench.cpp:383-441)
 *   motion actor  gauss5x5 + thres_diff + median5 behind the gauss / thres /
 *                 med actors (src/motion.cpp:27-74, :144-176)
 *   motion e2e    oracle_motion_detection_raw / the motion network run
 *                 (src/motion.cpp:107-252, src/bench.cpp:328-381)
 *   errors        std::invalid_argument / std::logic_error / RunAborted /
 *                 ControlError (src/channel.cpp:65-77, src/model.cpp:240-265)
 */
#ifndef DF_CUDA_H
#define DF_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define DF_OK 0
#define DF_EINVAL 1    /* bad argument or spec        -> std::invalid_argument */
#define DF_ELOGIC 2    /* contract misuse (n != r, outstanding handle, write
                          after close, token count mismatch on device)
                                                        -> std::logic_error */
#define DF_EABORTED 3  /* channel aborted               -> RunAborted */
#define DF_ECUDA 4     /* CUDA runtime / launch failure */
#define DF_ECONTROL 5  /* control token maps to an illegal rate -> ControlError */
#define DF_EOS 6       /* read_start on a closed channel holding fewer than r
                          tokens (nullopt, channel.cpp:114-140) */

const char* df_last_error(void);
int df_abi_version(void); /* bumps on any signature change */

/* ---- devices, streams, events, memory (plumbing) ------------------------ */
int df_device_count(int* count);
int df_device_sm_count(int device, int* sms);
int df_set_device(int device);
int df_stream_create(int device, void** stream);
int df_stream_destroy(void* stream);
int df_stream_synchronize(void* stream);
int df_event_create(void** ev);
int df_event_destroy(void* ev);
int df_event_record(void* ev, void* stream);
int df_event_synchronize(void* ev);
int df_event_elapsed_ms(void* start, void* stop, float* ms);
int df_stream_wait_event(void* stream, void* ev);
int df_malloc(int device, size_t bytes, void** dptr);
int df_free(void* dptr);
int df_host_alloc(size_t bytes, void** hptr); /* pinned */
int df_host_free(void* hptr);
int df_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int df_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int df_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);
int df_memset(void* dst, int value, size_t bytes, void* stream);
/* Runs fn(user) on a host thread in `stream` order (cudaLaunchHostFunc):
 * the firing of a CPU actor between its inputs' D2H and outputs' H2D.
 * fn must not call CUDA. */
int df_launch_host_func(void* stream, void (*fn)(void*), void* user);

/* ---- device channels (Eq. 1 capacity, Fig. 2 slot walk, state in HBM) ---
 * Replaces Channel (include/dynflow/channel.hpp:71-135).  Storage is
 * capacity_tokens * token_size bytes of HBM laid out exactly as the
 * reference buffer (delay token in slot 0, phase-2 copy of slot 3r -> 0).
 * The read/write phases and the available/written/read counters live in a
 * device control block, so a GPU actor kernel resolves its regions and
 * commits its per-firing token counts (0 or r) on the device.  The host
 * calls below are stream-ordered device operations (tiny kernels), never
 * host reads of device state, except df_channel_stats which synchronizes.
 */
typedef struct df_channel df_channel;

typedef struct df_chan_stats {
  uint64_t tokens_written;
  uint64_t tokens_read;
  uint64_t tokens_available; /* committed, not yet released (incl. delay) */
  uint32_t write_phase;
  uint32_t read_phase;
  uint32_t closed;
  uint32_t error; /* sticky device-side error word (DF_E* code), 0 = none */
} df_chan_stats;

/* initial_token: host pointer to token_size bytes, or NULL for all-zero
 * (proj/src/channel.cpp:34-51).  Only meaningful with has_delay. */
int df_channel_create(int device, size_t token_size, uint32_t token_rate, int has_delay,
                      const void* initial_token, df_channel** ch);
int df_channel_destroy(df_channel* ch);
size_t df_channel_capacity_tokens(const df_channel* ch);   /* channel.cpp:9-12 */
size_t df_channel_capacity_bytes(const df_channel* ch);    /* channel.cpp:14-16 */
size_t df_channel_token_size(const df_channel* ch);
uint32_t df_channel_token_rate(const df_channel* ch);
int df_channel_has_delay(const df_channel* ch);
void* df_channel_storage(const df_channel* ch);            /* device base */
void* df_channel_device_state(const df_channel* ch);       /* device control block */

/* Pure slot arithmetic (channel.cpp:18-32), host-side, for tests/tools. */
size_t df_slot_capacity(uint32_t rate, int has_delay);
size_t df_slot_write_first(uint32_t rate, int has_delay, unsigned phase);
size_t df_slot_read_first(uint32_t rate, int has_delay, unsigned phase);

/* Stream-ordered host-side transfers for host-driven endpoints (source /
 * sink actors, tests).  *_start with n != token_rate -> DF_ELOGIC, as the
 * reference (channel.cpp:65-68).  A host-driven endpoint owns its phase, so
 * its region address is known without a device round trip.  Blocking is
 * replaced by stream order: the host does not wait for tokens or room --
 * availability and capacity are checked on the device, where a violation
 * sets the sticky error word (df_channel_stats / df_channel_check).
 * End of stream: read_start on a channel that has been closed (by
 * df_channel_close or by the end of a device-resident run) synchronizes
 * and returns DF_EOS when fewer than n tokens remain. */
typedef struct df_region {
  void* dptr;          /* device address of the first token of the region */
  size_t first_slot;
  size_t tokens;
  uint64_t serial;     /* nonzero while outstanding */
  int direction;       /* 0 read, 1 write */
} df_region;
int df_channel_write_start(df_channel* ch, size_t n, df_region* region);
int df_channel_write_end(df_channel* ch, df_region* region, void* stream);
int df_channel_read_start(df_channel* ch, size_t n, df_region* region);
int df_channel_read_end(df_channel* ch, df_region* region, void* stream);
int df_channel_close(df_channel* ch, void* stream);
int df_channel_abort(df_channel* ch);
/* Synchronizes the channel's device and reads the control block. */
int df_channel_stats(df_channel* ch, df_chan_stats* out);
/* Returns the sticky device error (DF_OK if none) after synchronizing. */
int df_channel_check(df_channel* ch);

/* Device-resident channel test actors (exercise the device-side index
 * arithmetic exactly like a GPU actor does): a producer kernel writing
 * `firings` firings of rate-r tokens filled from splitmix64(seed, index),
 * and a consumer kernel checking them (mismatches counted into *bad_dev,
 * a device uint64).  Both resolve their regions from the device phase. */
int df_channel_test_produce(df_channel* ch, uint64_t first_token_index, uint32_t firings,
                            uint64_t seed, void* stream);
int df_channel_test_consume(df_channel* ch, uint64_t first_token_index, uint32_t firings,
                            uint64_t seed, int skip_initial_zero_token, uint64_t* bad_dev,
                            void* stream);

/* ---- DPD: dynamic parallel-Hammerstein predistortion actor -------------
 * One actor instance owns the taps and the per-branch FIR history
 * (FirState, include/dynflow/dpd.hpp:70-73), resident in HBM.  A firing
 * processes one block of `period` complex-f32 samples (interleaved re,im)
 * governed by one 4-byte little-endian control token (bit b-1 = branch b,
 * include/dynflow/dpd.hpp:26-41).  Branch b active: poly_branch -> FIR; all
 * active branches summed in ascending b; inactive: no output, state frozen
 * (src/dpd.cpp:258-320).  Arithmetic is op-for-op the reference's (no FMA
 * contraction), so outputs are bit-identical to oracle_dpd.
 * Extensions: taps_per_branch in {1..32} (reference: 10), masks with any
 * number of active branches including 1 (the reference network requires
 * [2,10]; its oracle accepts any).  A mask naming a branch beyond 10 sets
 * DF_ECONTROL in the actor's error word (check_config, src/dpd.cpp:49-58). */
typedef struct df_dpd df_dpd;

int df_dpd_create(int device, uint32_t period, uint32_t taps_per_branch,
                  const float* taps_host /* 10*T*2 floats, branch-major (re,im) */,
                  df_dpd** dpd);
int df_dpd_destroy(df_dpd* dpd);
int df_dpd_set_taps(df_dpd* dpd, const float* taps_host, void* stream);
int df_dpd_reset(df_dpd* dpd, void* stream); /* zero FIR history */
/* Name of the main kernel the actor's last firing launched ("dpd_wave_kernel"
 * for grids that fit one wave, else "dpd_main_kernel" / "dpd_main_generic_kernel";
 * "" before the first firing).  Static storage. */
const char* df_dpd_kernel_name(const df_dpd* dpd);
/* Reads the FIR history (10 branches x (T-1) complex) to host; synchronizes. */
int df_dpd_get_state(df_dpd* dpd, float* state_host);
int df_dpd_error(df_dpd* dpd); /* sticky device error word; synchronizes */
/* Sets the FIR history of every branch in branch_mask from `count` raw
 * input samples preceding the next firing (interleaved, device): exactly
 * the state fir10 leaves after processing them (dpd.cpp:108-120) --
 * poly recomputed, older history kept when count < T-1.  This is the
 * FIR-history halo of a block-range shard. */
int df_dpd_set_history(df_dpd* dpd, const float* raw_dev, uint32_t count, uint32_t branch_mask, void* stream);
/* Batched firing on raw device buffers: `blocks` consecutive firings, block
 * i governed by ctrl_dev[i] (uint32 LE) and reading/writing samples
 * [i*period, (i+1)*period) of in_dev / out_dev.  Equivalent to `blocks`
 * sequential firings of the reference's dynamic part. */
int df_dpd_fire(df_dpd* dpd, const uint32_t* ctrl_dev, const float* in_dev, float* out_dev,
                uint64_t blocks, void* stream);
/* Raw-buffer firing of a block-range shard with its FIR-history halo:
 * halo_tails[b-1] is a device pointer -- local, or a peer pointer into the
 * previous shard's input on another GPU (df_ipc_open_handle) -- to the
 * last T-1 raw interleaved samples, oldest first, of branch b's last
 * active block before this shard, or NULL (branch b keeps its carried
 * history).  Equivalent to df_dpd_set_history(dpd, halo_tails[b-1], T-1,
 * 1 << (b-1)) for each non-NULL b followed by df_dpd_fire; on the fast path
 * the tiles that need a halo read it directly (over NVLink for a peer
 * pointer) inside the firing. */
int df_dpd_fire_halo(df_dpd* dpd, const float* const* halo_tails, const uint32_t* ctrl_dev,
                     const float* in_dev, float* out_dev, uint64_t blocks, void* stream);/* Channel-bound firing: consumes `firings` control tokens from `ctrl`
 * (token 4 B, rate 1) and one block token per firing from `in`
 * (token = period*8 B); produces one block token per firing into `out`.
 * All three channels must have token_rate == firings (a batched GPU actor
 * sees its channels at the batch rate); regions and commits are resolved
 * on the device. */
int df_dpd_fire_channels(df_dpd* dpd, df_channel* ctrl, df_channel* in, df_channel* out,
                         uint32_t firings, void* stream);
/* Config actor (src/dpd.cpp:206-221) on device: writes
 * schedule[(first_firing + i) % len] for i < count into ctrl_dev. */
int df_dpd_config_tokens(int device, const uint16_t* schedule_host, size_t schedule_len,
                         uint64_t first_firing, uint64_t count, uint32_t* ctrl_dev, void* stream);
/* End to end from HOST buffers (drop-in for oracle_dpd / cmd_dpd's run):
 * samples % period == 0; H2D, config tokens, firings and D2H are pipelined
 * in chunks of `chunk_blocks` blocks on `stream` plus internal copy streams.
 * Continues from the actor's current FIR history and from its schedule
 * position: block i of this call is governed by schedule[(n + i) % len],
 * n = blocks fired by earlier run_host calls since create / df_dpd_reset, so
 * one stream split over several calls equals one call (df_dpd_reset starts a
 * fresh run).  Synchronizes before returning. */
int df_dpd_run_host(df_dpd* dpd, const float* in_host, float* out_host, uint64_t samples,
                    const uint16_t* schedule_host, size_t schedule_len, uint64_t chunk_blocks,
                    void* stream);

/* ---- motion detection actor ---------------------------------------------
 * Fused gray -> gauss5x5 -> |cur - prev| > thr -> median5 over a firing of
 * `frames` frames (rate r = frames), byte-exact to the reference chain
 * (src/motion.cpp:27-74, :236-252).  prev of the firing's first frame is
 * the delay token (gauss of the previous firing's last frame; black at
 * start, src/motion.cpp:131), and the firing produces the next delay
 * token.  Input format: DF_MOTION_GRAY (reference, 1 B/px) or
 * DF_MOTION_RGB (extension: interleaved RGB, gray = (77R+150G+29B+128)>>8). */
#define DF_MOTION_GRAY 1
#define DF_MOTION_RGB 3
typedef struct df_motion df_motion;

int df_motion_create(int device, unsigned width, unsigned height, int input_format,
                     uint8_t threshold, df_motion** m);
int df_motion_destroy(df_motion* m);
/* Sets the delay token: gauss(gray) of one frame given in the input format
 * (the one-frame halo of a frame-range shard), or black when NULL. */
int df_motion_set_prev_frame(df_motion* m, const void* frame_dev, void* stream);
/* Raw-buffer firing: frames in_dev[0..frames) -> masks out_dev; consumes
 * and replaces the actor's internal delay token. */
int df_motion_fire(df_motion* m, const void* in_dev, uint8_t* out_dev, uint32_t frames,
                   void* stream);
/* Raw-buffer firing of a frame-range shard: like df_motion_set_prev_frame
 * (m, halo_dev) followed by df_motion_fire, byte for byte, but gauss(halo)
 * is computed inside the firing by the warps that start the shard (no
 * separate gauss pass, no token round trip through HBM).  halo_dev is the
 * previous shard's last input frame in the input format. */
int df_motion_fire_halo(df_motion* m, const void* halo_dev, const void* in_dev, uint8_t* out_dev,
                        uint32_t frames, void* stream);
/* Channel-bound firing: `in` (token = one input frame, rate r), `delay`
 * (self-loop delay channel, token = W*H gauss bytes, rate 1, has_delay)
 * and `out` (token = W*H mask bytes, rate r).  Regions and the Fig. 2
 * delay walk are resolved on the device. */
int df_motion_fire_channels(df_motion* m, df_channel* in, df_channel* delay, df_channel* out,
                            void* stream);
/* End to end from HOST buffers (drop-in for the motion network run):
 * pipelined H2D / fire / D2H in chunks of chunk_frames.  Continues from the
 * current delay token.  Synchronizes before returning. */
int df_motion_run_host(df_motion* m, const void* in_host, uint8_t* out_host, uint64_t frames,
                       uint32_t chunk_frames, void* stream);
/* Name of the kernel a firing of this actor launches when its input is
 * 16-byte aligned: "motion_m3_kernel" (TMA-fed rows, TMEM-resident delay
 * band; needs width * input_format % 16 == 0) or "motion_fused_kernel"
 * (register-prefetch kernel, any width).  Static storage. */
const char* df_motion_kernel_name(const df_motion* m);
/* Individual stages (unit-level parity with gauss5x5 / thres_diff /
 * median5 / rgb->gray); one frame each, device buffers. */
int df_motion_gauss5x5(const uint8_t* in_dev, uint8_t* out_dev, unsigned w, unsigned h,
                       void* stream);
int df_motion_thres_diff(const uint8_t* prev_dev, const uint8_t* cur_dev, uint8_t* out_dev,
                         unsigned w, unsigned h, uint8_t thr, void* stream);
int df_motion_median5(const uint8_t* in_dev, uint8_t* out_dev, unsigned w, unsigned h,
                      void* stream);
int df_motion_rgb_to_gray(const uint8_t* rgb_dev, uint8_t* gray_dev, size_t pixels,
                          void* stream);

/* ---- device-resident networks (persistent actors) ----------------------
 * Replaces the reference's thread-per-actor run (Run::execute / actor_main
 * / fire_once, src/runtime.cpp:132-299) for networks whose actors all fire
 * on the GPU.  ONE cooperative persistent kernel runs the whole network:
 * each actor is a group of CTAs whose leader loops over the actor's
 * firings exactly as fire_once does -- read one control token (dynamic
 * actors) and dispatch it to per-port rates of 0 or r through the actor's
 * control table (control_dispatch, src/model.cpp:240-265), wait by spinning
 * on the HBM ring counters for r tokens on each active input and room for
 * r on each active output (read_start / write_start), publish the regions
 * to its CTAs, which fire, then commit outputs before inputs (write_end
 * with the Fig. 2 phase-2 copy, read_end).  A source stops at its firing
 * limit; an actor stops at end of stream on any input (read_start ->
 * nullopt: closed and fewer than r tokens left), then closes its outputs
 * and drains its inputs (src/runtime.cpp:206-231).  A fault (illegal
 * control token -> DF_ECONTROL, watchdog -> DF_ETIMEOUT) or df_net_abort
 * aborts every actor (RunAborted, src/channel.cpp:170-177).  No host round
 * trip happens between firings; token counts never leave the device. */
#define DF_ETIMEOUT 7 /* watchdog: an actor waited longer than the run's timeout */

#define DF_ACT_DPD_SOURCE 1   /* interleaved complex f32 -> re, im planes (dpd.cpp:189-204) */
#define DF_ACT_DPD_CONFIG 2   /* schedule[firing % len] -> every output (dpd.cpp:206-221) */
#define DF_ACT_DPD_SPLIT 3    /* in re,im -> active branch pairs (dpd.cpp:225-256) */
#define DF_ACT_DPD_BRANCH 4   /* poly_branch -> fir with frozen history (dpd.cpp:258-289) */
#define DF_ACT_DPD_ADDER 5    /* +0.0f then active pairs ascending (dpd.cpp:293-331) */
#define DF_ACT_DPD_SINK 6     /* re, im planes -> interleaved complex f32 (dpd.cpp:333-347) */
#define DF_ACT_TEST_PRODUCE 7 /* splitmix64 token stream on output 0 (acceptance.cpp:62-66) */
#define DF_ACT_TEST_CONSUME 8 /* checks that stream on input 0 */
#define DF_ACT_FRAME_SOURCE 9 /* u8 frames -> output 0 (motion.cpp:123-129) */
#define DF_ACT_GAUSS 10       /* gauss5x5, result to every output (motion.cpp:144-154) */
#define DF_ACT_THRES 11       /* in0 prev, in1 cur -> thres_diff (motion.cpp:157-166) */
#define DF_ACT_MEDIAN 12      /* median5 (motion.cpp:168-176) */
#define DF_ACT_FRAME_SINK 13  /* input 0 -> u8 frames (motion.cpp:178-183) */

/* Kind parameters (passed by value to df_net_add_actor).  Buffers are
 * device pointers or mapped pinned host pointers (df_host_alloc memory is
 * mapped; the actor then streams over PCIe). */
typedef struct df_act_samples { /* DPD_SOURCE (read) / DPD_SINK (write) */
  void* samples;                 /* interleaved complex f32, firing i = block i */
  uint32_t period;
} df_act_samples;
typedef struct df_act_config { /* DPD_CONFIG */
  const uint16_t* schedule;     /* device */
  uint32_t len;
} df_act_config;
typedef struct df_act_branch { /* DPD_BRANCH */
  uint32_t branch;              /* 1..10: poly order */
  uint32_t taps_per_branch;     /* 1..32 */
  const float* taps;            /* device, taps_per_branch complex */
  float* state;                 /* device, taps_per_branch-1 complex FirState, x[-(j+1)] */
  uint32_t period;
} df_act_branch;
typedef struct df_act_test { /* TEST_PRODUCE / TEST_CONSUME */
  uint64_t seed;
  uint64_t* counters;           /* device: [0] tokens produced / consumed, [1] mismatches */
  uint32_t stall_mask;          /* leader pauses ~2 us before a firing when (hash & mask) == 0; 0 = never */
  uint32_t skip_initial;        /* consumer: the first token is the channel's zero delay token */
  uint64_t hold_ns;             /* pause before every firing (abort tests) */
} df_act_test;
typedef struct df_act_frames { /* FRAME_SOURCE (read) / FRAME_SINK (write) / GAUSS / THRES / MEDIAN */
  void* frames;                 /* W*H bytes per token, firing i = tokens [i*r, (i+1)*r) */
  uint32_t width, height;
  uint8_t threshold;            /* THRES */
} df_act_frames;

typedef struct df_net df_net;
int df_net_create(int device, df_net** net);
int df_net_destroy(df_net* net);
/* Adds an actor of `kind` run by `ctas` CTAs.  control: the control channel
 * of a dynamic actor (NULL for static), inputs / outputs: regular ports in
 * declaration order (at most 24 each).  firing_limit: a source's
 * source_firing_limit (0 = stop only at end of stream).  Channels bound to
 * a network are device-driven at both ends. */
int df_net_add_actor(df_net* net, int kind, const void* params, size_t params_bytes, uint32_t ctas,
                     df_channel* control, df_channel* const* inputs, size_t n_in, df_channel* const* outputs,
                     size_t n_out, uint64_t firing_limit, int* index);
/* The device form of ActorBehavior::control (model.hpp:103-108) for a
 * dynamic actor: row v (v < domain, the control token read as a
 * little-endian integer) = { bits of the active inputs, bits of the active
 * outputs, 1 if legal }.  A token >= domain or an illegal row faults the
 * actor with DF_ECONTROL (ControlError), recording the token value. */
int df_net_set_control_table(df_net* net, int actor, const uint32_t* rows, uint32_t domain);
/* Runs the network to completion: one cooperative kernel; synchronizes.
 * timeout_s: watchdog for any single wait (<= 0: 30 s).  Returns DF_OK, or
 * the first fault's code (see df_net_fault) / DF_EABORTED. */
int df_net_run(df_net* net, double timeout_s);
/* From any host thread while df_net_run blocks: aborts the run. */
int df_net_abort(df_net* net);
int df_net_fault(const df_net* net, int* actor, int* code, uint32_t* token);
/* After a run: firings, and device time from the first firing's start to
 * the actor's stop (RunStats::active_seconds, bench.cpp:346-347). */
int df_net_actor_stats(const df_net* net, int actor, uint64_t* firings, double* active_ms);
/* After a run, the actor leader's time split over all its firings (device
 * timestamps): waiting for tokens / room (read_start + write_start and the
 * control token), firing (frame published -> every CTA done), committing
 * (phase-2 copies + counter updates).  Tracing aid (RunStats has no
 * counterpart). */
int df_net_actor_profile(const df_net* net, int actor, double* wait_ms, double* fire_ms, double* commit_ms);

/* ---- multi-GPU halos (NVLink peer copies; no collectives) ---------------
 * No reference counterpart: dynflow is one CPU process.  These serve the
 * frame-range / block-range sharding of the two actors (one process per
 * GPU; df_motion_fire_halo / df_dpd_fire_halo take the halos). */
int df_peer_enable(int device_a, int device_b);
int df_halo_copy(int dst_device, void* dst, int src_device, const void* src, size_t bytes,
                 void* stream);
/* One process per GPU: export a cudaMalloc'ed shard buffer (handle of
 * df_ipc_handle_size() bytes), map a neighbour's exported buffer (peer
 * access enabled lazily), and unmap it.  The mapped pointer is a peer
 * pointer for df_halo_copy (src_device = the exporting rank's device). */
int df_ipc_handle_size(void);
int df_ipc_get_handle(const void* dev_ptr, void* handle_out);
int df_ipc_open_handle(int device, const void* handle, void** dev_ptr);
int df_ipc_close_handle(void* dev_ptr);

/* ---- synthetic inputs on device (bench data; not the reference streams) */
int df_fill_random_u8(void* dst, size_t bytes, uint64_t seed, void* stream);
int df_fill_random_pm1(float* dst, size_t floats, uint64_t seed, void* stream);

/* ---- launch accounting (for bench "gpu_launches") ----------------------- */
uint64_t df_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* DF_CUDA_H */
