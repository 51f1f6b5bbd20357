/*
 * oracle.h -- CPU restatement of the reference (dynflow, arXiv 1611.03226
 * artifact) hot-path arithmetic.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker
 * or the timed CPU baseline.  The product path (libdf_cuda.so) never
 * links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference compiled from /root/reference/proj/src (oracle/_ref, built by
 * oracle/Makefile) and against the committed fixtures in tests/golden/.
 * Extensions with no reference counterpart (RGB->gray, T != 10 taps,
 * k = 1 masks in the network, 3x3 morphology) are labelled "restatement
 * only" below; for T = 10 / gray input they reduce to the pinned code.
 *
 * Build flags are part of the pin: -O2 -ffp-contract=off (FMA contraction
 * changes the reference's own DPD output).
 */
#ifndef DF_ORACLE_H
#define DF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- generators (std::mt19937_64 restated) ---------------------------- */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);

/* proj/src/dpd.cpp:496-505 synth_samples: interleaved (re, im) floats. */
void orc_synth_samples(uint64_t samples, uint64_t seed, float* out_interleaved);
/* proj/src/dpd.cpp:485-494 random_taps, generalised to T taps per branch
 * (branch-major, taps[b*T + k] = (re, im) interleaved).  T = 10 is the
 * reference; other T continue the same stream (restatement only). */
void orc_random_taps(uint64_t seed, unsigned taps_per_branch, float* out_interleaved);
/* proj/src/dpd.cpp:467-483 random_schedule: masks with k in [2,10]. */
void orc_random_schedule(size_t entries, uint64_t seed, uint16_t* out_masks);
/* proj/src/motion.cpp:254-260 synth_frames: rng() & 0xFF per byte. */
void orc_synth_bytes(uint64_t bytes, uint64_t seed, uint8_t* out);

/* ---- DPD (proj/src/dpd.cpp) --------------------------------------------- */
/* proj/src/dpd.cpp:60-75 poly_branch on planar spans. */
void orc_poly_branch(unsigned branch, const float* re_in, const float* im_in, size_t n,
                     float* re_out, float* im_out);
/* proj/src/dpd.cpp:83-121 fir10 generalised to T taps (T = 10 is fir10).
 * state_re/state_im hold T-1 history samples, [j] = x[-(j+1)]. */
void orc_fir(unsigned T, const float* taps_interleaved, float* state_re, float* state_im,
             const float* re_in, const float* im_in, size_t n, float* re_out, float* im_out);
/* proj/src/dpd.cpp:358-391 oracle_dpd, T-generic, accepts any mask
 * (including k = 1 and 0, which the oracle never rejects).  Returns 0, or
 * -1 on a bad schedule/period exactly where the reference throws. */
int orc_dpd(const float* in_interleaved, size_t samples, const float* taps_interleaved,
            unsigned T, const uint16_t* schedule, size_t schedule_len, uint32_t period,
            float* out_interleaved);

/* ---- motion (proj/src/motion.cpp) -------------------------------------- */
void orc_gauss5x5(const uint8_t* in, uint8_t* out, unsigned w, unsigned h);   /* :27-48 */
void orc_thres_diff(const uint8_t* prev, const uint8_t* cur, uint8_t* out, unsigned w,
                    unsigned h, uint8_t threshold);                            /* :50-57 */
void orc_median5(const uint8_t* in, uint8_t* out, unsigned w, unsigned h);    /* :59-74 */
/* :236-252 oracle_motion_detection_raw over concatenated gray frames. */
void orc_motion_gray(const uint8_t* frames, size_t count, unsigned w, unsigned h,
                     uint8_t threshold, uint8_t* out);
/* Extension (restatement only): integer BT.601 luma,
 * gray = (77 R + 150 G + 29 B + 128) >> 8, over interleaved RGB. */
void orc_rgb_to_gray(const uint8_t* rgb, size_t pixels, uint8_t* gray);
/* gray(RGB) followed by the pinned gray chain; prev = black initially, or
 * the gauss of `prev_rgb` (one-frame halo) when non-NULL. */
void orc_motion_rgb(const uint8_t* rgb, size_t count, unsigned w, unsigned h, uint8_t threshold,
                    const uint8_t* prev_rgb, uint8_t* out);

/* ---- multi-threaded drivers (bit-identical to the serial functions) ----
 * orc_dpd_mt: block ranges per thread, each starting from branch b's FIR
 * history = poly of the last T-1 samples of b's active stream before the
 * range (dpd.cpp:108-120).  orc_motion_mt: frame ranges, each starting
 * from gauss(gray(frame f0-1)); fmt 1 gray / 3 RGB; prev0 = RGB halo frame
 * before frame 0 or NULL (black). */
int orc_dpd_mt(const float* in_interleaved, size_t samples, const float* taps_interleaved, unsigned T,
               const uint16_t* schedule, size_t schedule_len, uint32_t period, float* out_interleaved,
               unsigned threads);
void orc_motion_mt(const uint8_t* frames, size_t count, unsigned w, unsigned h, int fmt, uint8_t threshold,
                   const uint8_t* prev0, uint8_t* out, unsigned threads);

/* ---- channel slot walk (proj/src/channel.cpp:9-32) ---------------------- */
size_t orc_capacity_tokens(uint32_t rate, int has_delay);
size_t orc_write_slot(uint32_t rate, int has_delay, unsigned phase);
size_t orc_read_slot(uint32_t rate, int has_delay, unsigned phase);

/* proj/src/bench.cpp:307-326 compare_samples: index of the first sample
 * with |g-w|/max(|w|,1e-3) > tol, or -1. */
int64_t orc_compare_samples(const float* got, const float* want, size_t samples, double tol,
                            double* worst_err);

#ifdef __cplusplus
}
#endif
#endif
