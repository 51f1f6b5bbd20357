/*
 * df_host.h -- C ABI of libdf_host.so: the C++ GPU-actor runtime (include/df/)
 * running the two reference networks end to end from HOST buffers.
 *
 * These are the drop-in calls for the reference's network runs
 * (/root/reference/proj/src/bench.cpp:383-441 cmd_dpd and :328-381
 * cmd_motion: build_network(params) + run(net, cfg) with host spans), as a
 * cgo/ctypes/JNI binding would call them.  Status 0 = OK; on failure
 * dfh_last_error() describes the exception (ValidationError,
 * std::invalid_argument, ActorFault naming the actor, ...).
 */
#ifndef DF_HOST_H
#define DF_HOST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* dfh_last_error(void);

/* taps: 10 * taps_per_branch complex (re, im) floats, branch-major;
 * schedule: one 10-bit mask per block (bit b-1 = branch b), cycling, each
 * with 2..10 active branches as the reference's check_config demands
 * (src/dpd.cpp:49-58), or 1..10 with allow_single_branch (extension).
 * samples % (period * batch) == 0.  sink_active_ms: device time of the
 * sink actor from its first to its last firing (like active_seconds). */
int dfh_dpd_run(int device, const float* in_host, float* out_host, uint64_t samples, uint32_t period,
                uint32_t taps_per_branch, const float* taps, const uint16_t* schedule, size_t schedule_len,
                uint32_t batch, int allow_single_branch, double* sink_active_ms, uint64_t* dpd_firings);

/* input_format: 1 gray, 3 RGB; frames % token_rate == 0. */
int dfh_motion_run(int device, const uint8_t* in_host, uint8_t* out_host, uint64_t frames, unsigned width,
                   unsigned height, int input_format, uint8_t threshold, uint32_t token_rate,
                   double* sink_active_ms, uint64_t* delay_tokens_written);

/* The reference's own network shapes as DEVICE-RESIDENT actors, run as one
 * persistent kernel (df::dpd / df::motion ::build_reference_network):
 * DPD: 15 actors / 56 channels, split / branches / adder dynamic with their
 * control tokens dispatched on the device per firing (0 or 1 per port);
 * firings[15] receives each actor's firing count in declaration order
 * (source, config, split, branch01..10, adder, sink), channel_tokens[56]
 * each channel's tokens written (channel declaration order, dpd.cpp:
 * 167-184).  Motion: 5 actors (source, gauss, thres, med, sink) with the
 * delay channel gauss_thres_prev; gray frames; firings[5].  timeout_s is
 * the device watchdog (a deadlock ends in ActorFault). */
int dfh_dpd_run_resident(int device, const float* in_host, float* out_host, uint64_t samples, uint32_t period,
                         uint32_t taps_per_branch, const float* taps, const uint16_t* schedule, size_t schedule_len,
                         int allow_single_branch, uint32_t branch_ctas, double timeout_s, double* sink_active_ms,
                         uint64_t* firings, uint64_t* channel_tokens);
int dfh_motion_run_resident(int device, const uint8_t* in_host, uint8_t* out_host, uint64_t frames, unsigned width,
                            unsigned height, uint8_t threshold, uint32_t token_rate, uint32_t ctas, double timeout_s,
                            double* sink_active_ms, uint64_t* firings);

/* Heterogeneous CPU + GPU network (df::motion::build_mixed_network):
 * RGB in; the gray conversion and a per-frame moving-pixel census run as
 * CPU actors, the motion chain as a GPU actor, all on device channels.
 * counts: `frames` entries.  fail_at_firing >= 0 injects a fault into the
 * census actor (the call then fails with ActorFault). */
int dfh_motion_run_mixed(int device, const uint8_t* rgb_host, uint8_t* out_host, uint64_t frames, unsigned width,
                         unsigned height, uint8_t threshold, uint32_t token_rate, uint32_t* counts,
                         int64_t fail_at_firing, double* sink_active_ms);

/* Channel buffer memory (cmd_mem, proj/src/bench.cpp:491-525), no device:
 * app 0 = motion (width, height, token_rate), 1 = dpd (period).
 * shape 0 = the B200 network this library runs; shape 1 = the reference's
 * network shape (5 motion channels / 56 DPD channels) restated with this
 * library's model types, whose Eq. 1 total must equal the reference's.
 * Returns the channel count (or -1, dfh_last_error). */
int dfh_memory(int app, unsigned width, unsigned height, uint32_t token_rate, uint32_t period, int shape,
               uint64_t* total_bytes);

/* Host-side rule checks (no device): builds the named reference network
 * shape and returns the number of validate() violations (0 = runnable);
 * -1 with dfh_last_error() on a BuildError / invalid_argument. */
int dfh_validate_demo(int which);  /* which: 0..6, see host_abi.cpp */

/* Ordering check of the static schedule (device needed): source -> sink
 * over ONE delay channel of 8-byte tokens at token_rate, initial token all
 * 0xFF bytes, the sink optionally declared first.  Source firing i writes
 * the values i*r+1 .. i*r+r; out_host receives the sink's firings*r tokens:
 * the initial token, then 1, 2, ... (a delay channel of rate r > 1 orders
 * the producer's firing i before the consumer's firing i). */
int dfh_delay_chain_run(int device, uint32_t token_rate, int sink_first, uint64_t firings, uint64_t* out_host);

/* Dynamic-rate CPU actors (the static-schedule runtime): the reference's
 * dynamic DPD network shape -- split, two gated branches with frozen state,
 * adder -- as CPU actors on device channels, int32 tokens, masks cycling
 * (bit b-1 = branch b active; a mask above 3 is an illegal rate ->
 * ActorFault).  out_host: firings * rate int32. */
int dfh_dynamic_cpu_run(int device, const uint32_t* masks, size_t n_masks, uint32_t rate, uint64_t firings,
                        int32_t* out_host);

/* df::bulk_kernel_adapter (runtime.hpp:97-108): source -> a CPU actor made
 * from a batch kernel (int32 x -> 2x; bad != 0: a wrong output size, which
 * faults the actor) -> sink.  out_host: firings * rate int32. */
int dfh_bulk_kernel_run(int device, uint32_t rate, uint64_t firings, int bad, int32_t* out_host);

/* df::Channel (include/df/channel.hpp, the reference's Channel API over a
 * device channel): see host_abi.cpp for the scripted walk and status bits. */
int dfh_channel_class_demo(int device, uint32_t rate, int delay, uint32_t firings, uint32_t* out, int* status);

/* ---- data formats either side of the path (df/io.hpp, df/dpd.hpp) -------
 * The reference's text and file formats (proj/src/dpd.cpp:393-462
 * parse_schedule / parse_taps; proj/src/bench.cpp:25-97, :173-262 read_file
 * / write_file / read_pgm and the raw-frame / cf32 inputs).  Status 8 =
 * FormatError (the reference's ConfigError: unreadable, truncated or
 * malformed file); parse errors are status 6 with the reference's message.
 * Size queries: pass a NULL buffer to get the sizes, then call again. */
/* The reference's generators (df::dpd::random_schedule / random_taps /
 * synth_samples, df::motion::synth_frames): what 0 = n uint16 schedule
 * masks, 1 = 10 x n complex taps, 2 = n complex samples, 3 = n frame bytes. */
int dfh_synth(int what, uint64_t n, uint64_t seed, void* out);

/* The config token's wire form (dpd.cpp:38-47): 4 bytes little endian. */
int dfh_encode_config(uint16_t mask, uint8_t* out4);
int dfh_decode_config(const uint8_t* in4, uint16_t* mask);
int dfh_parse_schedule(const char* text, uint16_t* masks, size_t cap, size_t* count);
int dfh_parse_taps(const char* text, uint32_t taps_per_branch, float* taps_out /* 10*T*2 floats */);
int dfh_read_pgm(const char* path, uint8_t* pixels, size_t cap_bytes, unsigned* width, unsigned* height,
                 uint64_t* frames);
int dfh_write_pgm(const char* path, const uint8_t* pixels, uint64_t frames, unsigned width, unsigned height);
int dfh_read_raw_frames(const char* path, unsigned width, unsigned height, int input_format, uint8_t* pixels,
                        size_t cap_bytes, uint64_t* frames);
int dfh_read_cf32(const char* path, float* samples_out, size_t cap_samples, uint64_t* samples);
int dfh_write_file(const char* path, const void* data, size_t size);

#ifdef __cplusplus
}
#endif
#endif
