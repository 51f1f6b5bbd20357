/*
 * oracle.c -- CPU restatement of the dynflow hot path.  TEST
 * INFRASTRUCTURE ONLY (see oracle.h): the checker for the CUDA path and
 * the "port" CPU baseline, never part of the shipped product.
 *
 * Every function follows the reference op-for-op so float results are
 * bit-identical when compiled with -ffp-contract=off.  Citations are
 * /root/reference/proj/... file:line.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------
 * std::mt19937_64 (the generator every reference fixture is drawn from:
 * proj/src/dpd.cpp:21-26, :467-505, proj/src/motion.cpp:254-260).
 * Parameters are the standard ones (w=64, n=312, m=156, r=31).
 * ---------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  g->idx = MT_N;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->idx >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* proj/src/dpd.cpp:21-26 uniform_pm1: top 24 bits -> [0,1) -> [-1,1). */
static float uniform_pm1(orc_mt64* g) {
  const float u = (float)(orc_mt64_next(g) >> 40) / (float)(1u << 24);
  return 2.0f * u - 1.0f;
}

void orc_synth_samples(uint64_t samples, uint64_t seed, float* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < samples; ++i) {  /* dpd.cpp:499-503: re then im */
    out[2 * i] = uniform_pm1(&g);
    out[2 * i + 1] = uniform_pm1(&g);
  }
}

void orc_random_taps(uint64_t seed, unsigned T, float* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  for (unsigned b = 0; b < 10; ++b) {      /* dpd.cpp:488-492, branch-major */
    for (unsigned k = 0; k < T; ++k) {
      const float re = 0.5f * uniform_pm1(&g);
      const float im = 0.5f * uniform_pm1(&g);
      out[2 * (b * T + k)] = re;
      out[2 * (b * T + k) + 1] = im;
    }
  }
}

void orc_random_schedule(size_t entries, uint64_t seed, uint16_t* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  unsigned branches[10];
  for (unsigned i = 0; i < 10; ++i) branches[i] = i + 1;  /* dpd.cpp:471-472 iota */
  for (size_t i = 0; i < entries; ++i) {
    const unsigned k = 2 + (unsigned)(orc_mt64_next(&g) % 9);  /* dpd.cpp:474 */
    for (size_t j = 10; j > 1; --j) {                           /* dpd.cpp:475-477 */
      const size_t r = (size_t)(orc_mt64_next(&g) % j);
      const unsigned t = branches[j - 1];
      branches[j - 1] = branches[r];
      branches[r] = t;
    }
    uint16_t mask = 0;
    for (unsigned j = 0; j < k; ++j) mask |= (uint16_t)(1u << (branches[j] - 1));
    out[i] = mask;
  }
}

void orc_synth_bytes(uint64_t bytes, uint64_t seed, uint8_t* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < bytes; ++i) out[i] = (uint8_t)(orc_mt64_next(&g) & 0xFF);
}

/* ------------------------------------------------------------------------
 * DPD
 * ---------------------------------------------------------------------- */
void orc_poly_branch(unsigned branch, const float* re_in, const float* im_in, size_t n,
                     float* re_out, float* im_out) {
  for (size_t i = 0; i < n; ++i) {        /* dpd.cpp:66-74 */
    const float re = re_in[i];
    const float im = im_in[i];
    const float mag = sqrtf(re * re + im * im);
    float scale = 1.0f;
    for (unsigned p = 1; p < branch; ++p) scale *= mag;
    re_out[i] = re * scale;
    im_out[i] = im * scale;
  }
}

void orc_fir(unsigned T, const float* taps, float* state_re, float* state_im, const float* re_in,
             const float* im_in, size_t n_, float* re_out, float* im_out) {
  const ptrdiff_t n = (ptrdiff_t)n_;
  for (ptrdiff_t i = 0; i < n; ++i) {     /* dpd.cpp:86-107 */
    float acc_re = 0.0f;
    float acc_im = 0.0f;
    for (unsigned k = 0; k < T; ++k) {
      const ptrdiff_t j = i - (ptrdiff_t)k;
      float x_re, x_im;
      if (j >= 0) {
        x_re = re_in[j];
        x_im = im_in[j];
      } else {
        x_re = state_re[-j - 1];
        x_im = state_im[-j - 1];
      }
      const float t_re = taps[2 * k];
      const float t_im = taps[2 * k + 1];
      acc_re += t_re * x_re - t_im * x_im;
      acc_im += t_re * x_im + t_im * x_re;
    }
    re_out[i] = acc_re;
    im_out[i] = acc_im;
  }
  /* dpd.cpp:108-120: history = last T-1 inputs, older state fills short blocks. */
  float next_re[64], next_im[64];
  for (unsigned j = 0; j + 1 < T; ++j) {
    const ptrdiff_t idx = n - 1 - (ptrdiff_t)j;
    if (idx >= 0) {
      next_re[j] = re_in[idx];
      next_im[j] = im_in[idx];
    } else {
      next_re[j] = state_re[-idx - 1];
      next_im[j] = state_im[-idx - 1];
    }
  }
  memcpy(state_re, next_re, sizeof(float) * (T - 1));
  memcpy(state_im, next_im, sizeof(float) * (T - 1));
}

int orc_dpd(const float* in, size_t samples, const float* taps, unsigned T,
            const uint16_t* schedule, size_t schedule_len, uint32_t period, float* out) {
  /* dpd.cpp:362-364 */
  if (schedule_len == 0 || period == 0 || samples % period != 0) return -1;
  if (T < 1 || T > 64) return -1;
  const size_t periods = samples / period;
  float* state = (float*)calloc((size_t)10 * 2 * 64, sizeof(float));
  float* bre = (float*)malloc(sizeof(float) * period);
  float* bim = (float*)malloc(sizeof(float) * period);
  float* pre = (float*)malloc(sizeof(float) * period);
  float* pim = (float*)malloc(sizeof(float) * period);
  float* fre = (float*)malloc(sizeof(float) * period);
  float* fim = (float*)malloc(sizeof(float) * period);
  float* are = (float*)malloc(sizeof(float) * period);
  float* aim = (float*)malloc(sizeof(float) * period);
  for (size_t p = 0; p < periods; ++p) {  /* dpd.cpp:370-389 */
    const uint16_t cfg = schedule[p % schedule_len];
    for (size_t i = 0; i < period; ++i) {
      bre[i] = in[2 * (p * period + i)];
      bim[i] = in[2 * (p * period + i) + 1];
      are[i] = 0.0f;
      aim[i] = 0.0f;
    }
    for (unsigned b = 1; b <= 10; ++b) {
      if (!((cfg >> (b - 1)) & 1u)) continue;
      orc_poly_branch(b, bre, bim, period, pre, pim);
      float* st = state + (size_t)(b - 1) * 128;
      orc_fir(T, taps + 2 * (size_t)(b - 1) * T, st, st + 64, pre, pim, period, fre, fim);
      for (size_t i = 0; i < period; ++i) {
        are[i] += fre[i];
        aim[i] += fim[i];
      }
    }
    for (size_t i = 0; i < period; ++i) {
      out[2 * (p * period + i)] = are[i];
      out[2 * (p * period + i) + 1] = aim[i];
    }
  }
  free(state); free(bre); free(bim); free(pre); free(pim);
  free(fre); free(fim); free(are); free(aim);
  return 0;
}

/* ------------------------------------------------------------------------
 * Motion detection
 * ---------------------------------------------------------------------- */
static const int kBinomial[5] = {1, 4, 6, 4, 1};  /* motion.cpp:14 */

void orc_gauss5x5(const uint8_t* in, uint8_t* out, unsigned w, unsigned h) {
  for (unsigned y = 0; y < h; ++y) {      /* motion.cpp:29-47 */
    for (unsigned x = 0; x < w; ++x) {
      const size_t idx = (size_t)y * w + x;
      if (y < 2 || y >= h - 2 || x < 2 || x >= w - 2) {
        out[idx] = in[idx];
        continue;
      }
      int acc = 0;
      for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx)
          acc += kBinomial[dy + 2] * kBinomial[dx + 2] * in[(size_t)(y + dy) * w + (x + dx)];
      out[idx] = (uint8_t)((acc + 128) >> 8);
    }
  }
}

void orc_thres_diff(const uint8_t* prev, const uint8_t* cur, uint8_t* out, unsigned w, unsigned h,
                    uint8_t threshold) {
  const size_t n = (size_t)w * h;         /* motion.cpp:53-56 */
  for (size_t i = 0; i < n; ++i) out[i] = abs((int)cur[i] - (int)prev[i]) > threshold ? 255 : 0;
}

void orc_median5(const uint8_t* in, uint8_t* out, unsigned w, unsigned h) {
  for (unsigned y = 0; y < h; ++y) {      /* motion.cpp:61-73 */
    for (unsigned x = 0; x < w; ++x) {
      const size_t idx = (size_t)y * w + x;
      if (y == 0 || y == h - 1 || x == 0 || x == w - 1) {
        out[idx] = in[idx];
        continue;
      }
      uint8_t v[5] = {in[idx], in[idx - w], in[idx + w], in[idx - 1], in[idx + 1]};
      /* nth_element(v, v+2) == the 3rd smallest; a 5-element sort gives it. */
      for (int i = 1; i < 5; ++i) {
        uint8_t t = v[i];
        int j = i - 1;
        while (j >= 0 && v[j] > t) { v[j + 1] = v[j]; --j; }
        v[j + 1] = t;
      }
      out[idx] = v[2];
    }
  }
}

void orc_motion_gray(const uint8_t* frames, size_t count, unsigned w, unsigned h,
                     uint8_t threshold, uint8_t* out) {
  const size_t size = (size_t)w * h;      /* motion.cpp:239-251 */
  uint8_t* prev = (uint8_t*)calloc(size, 1);
  uint8_t* filt = (uint8_t*)malloc(size);
  uint8_t* diff = (uint8_t*)malloc(size);
  for (size_t f = 0; f < count; ++f) {
    orc_gauss5x5(frames + f * size, filt, w, h);
    orc_thres_diff(prev, filt, diff, w, h, threshold);
    orc_median5(diff, out + f * size, w, h);
    uint8_t* t = prev; prev = filt; filt = t;
  }
  free(prev); free(filt); free(diff);
}

void orc_rgb_to_gray(const uint8_t* rgb, size_t pixels, uint8_t* gray) {
  for (size_t i = 0; i < pixels; ++i) {
    const unsigned r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
    gray[i] = (uint8_t)((77u * r + 150u * g + 29u * b + 128u) >> 8);
  }
}

void orc_motion_rgb(const uint8_t* rgb, size_t count, unsigned w, unsigned h, uint8_t threshold,
                    const uint8_t* prev_rgb, uint8_t* out) {
  const size_t size = (size_t)w * h;
  uint8_t* gray = (uint8_t*)malloc(size);
  uint8_t* prev = (uint8_t*)calloc(size, 1);
  uint8_t* filt = (uint8_t*)malloc(size);
  uint8_t* diff = (uint8_t*)malloc(size);
  if (prev_rgb) {  /* one-frame halo: the delay token is gauss(gray(f0-1)) */
    orc_rgb_to_gray(prev_rgb, size, gray);
    orc_gauss5x5(gray, prev, w, h);
  }
  for (size_t f = 0; f < count; ++f) {
    orc_rgb_to_gray(rgb + f * size * 3, size, gray);
    orc_gauss5x5(gray, filt, w, h);
    orc_thres_diff(prev, filt, diff, w, h, threshold);
    orc_median5(diff, out + f * size, w, h);
    uint8_t* t = prev; prev = filt; filt = t;
  }
  free(gray); free(prev); free(filt); free(diff);
}

/* ------------------------------------------------------------------------
 * Multi-threaded drivers of the restatements above (whole-output parity at
 * BASELINE sizes).  They split the stream into block / frame ranges and
 * give each range exactly the state the serial run has at its start, so
 * the result is bit-identical to orc_dpd / orc_motion_rgb / orc_motion_gray
 * (checked against them in tests/test_oracle.py):
 *   DPD     branch b's FIR history at block p0 is the poly of the last T-1
 *           samples of b's ACTIVE input stream before p0 (fir10's state
 *           update, dpd.cpp:108-120; poly_branch is memoryless), zeros if
 *           fewer were seen;
 *   motion  the delay token of frame f0 is gauss(gray(f0 - 1)) (black for
 *           frame 0, motion.cpp:239-251).
 * ---------------------------------------------------------------------- */
#include <pthread.h>

typedef struct {
  const float* in; const float* taps; unsigned T; const uint16_t* sched; size_t len;
  uint32_t period; size_t p0, p1; float* out;
} dpd_job;

static void* dpd_range(void* arg) {
  const dpd_job* j = (const dpd_job*)arg;
  const uint32_t period = j->period;
  const unsigned H1 = j->T - 1;
  float* state = (float*)calloc((size_t)10 * 128, sizeof(float));
  float* bre = (float*)malloc(sizeof(float) * period);
  float* bim = (float*)malloc(sizeof(float) * period);
  float* pre = (float*)malloc(sizeof(float) * period);
  float* pim = (float*)malloc(sizeof(float) * period);
  float* fre = (float*)malloc(sizeof(float) * period);
  float* fim = (float*)malloc(sizeof(float) * period);
  float* are = (float*)malloc(sizeof(float) * period);
  float* aim = (float*)malloc(sizeof(float) * period);
  /* History at p0: walk back over each branch's active blocks. */
  for (unsigned b = 1; b <= 10; ++b) {
    float* st = state + (size_t)(b - 1) * 128;
    unsigned got = 0;
    for (size_t q = j->p0; q-- > 0 && got < H1;) {
      if (!((j->sched[q % j->len] >> (b - 1)) & 1u)) continue;
      for (size_t i = period; i-- > 0 && got < H1; ++got) {
        float re, im;
        orc_poly_branch(b, &j->in[2 * (q * period + i)], &j->in[2 * (q * period + i) + 1], 1, &re, &im);
        st[got] = re;
        st[64 + got] = im;
      }
    }
  }
  for (size_t p = j->p0; p < j->p1; ++p) {  /* the serial loop of orc_dpd, dpd.cpp:370-389 */
    const uint16_t cfg = j->sched[p % j->len];
    for (size_t i = 0; i < period; ++i) {
      bre[i] = j->in[2 * (p * period + i)];
      bim[i] = j->in[2 * (p * period + i) + 1];
      are[i] = 0.0f;
      aim[i] = 0.0f;
    }
    for (unsigned b = 1; b <= 10; ++b) {
      if (!((cfg >> (b - 1)) & 1u)) continue;
      orc_poly_branch(b, bre, bim, period, pre, pim);
      float* st = state + (size_t)(b - 1) * 128;
      orc_fir(j->T, j->taps + 2 * (size_t)(b - 1) * j->T, st, st + 64, pre, pim, period, fre, fim);
      for (size_t i = 0; i < period; ++i) {
        are[i] += fre[i];
        aim[i] += fim[i];
      }
    }
    for (size_t i = 0; i < period; ++i) {
      j->out[2 * (p * period + i)] = are[i];
      j->out[2 * (p * period + i) + 1] = aim[i];
    }
  }
  free(state); free(bre); free(bim); free(pre); free(pim);
  free(fre); free(fim); free(are); free(aim);
  return NULL;
}

int orc_dpd_mt(const float* in, size_t samples, const float* taps, unsigned T, const uint16_t* schedule,
               size_t schedule_len, uint32_t period, float* out, unsigned threads) {
  if (schedule_len == 0 || period == 0 || samples % period != 0) return -1;
  if (T < 1 || T > 64) return -1;
  const size_t periods = samples / period;
  if (threads < 1) threads = 1;
  if (threads > periods) threads = periods ? (unsigned)periods : 1;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  dpd_job* jobs = (dpd_job*)malloc(sizeof(dpd_job) * threads);
  for (unsigned t = 0; t < threads; ++t) {
    dpd_job jb = {in, taps, T, schedule, schedule_len, period, periods * t / threads, periods * (t + 1) / threads, out};
    jobs[t] = jb;
    pthread_create(&tid[t], NULL, dpd_range, &jobs[t]);
  }
  for (unsigned t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid); free(jobs);
  return 0;
}

typedef struct {
  const uint8_t* frames; size_t f0, f1; unsigned w, h; uint8_t thr; int rgb; const uint8_t* prev0; uint8_t* out;
} motion_job;

static void* motion_range(void* arg) {
  const motion_job* j = (const motion_job*)arg;
  const size_t px = (size_t)j->w * j->h, fb = px * (j->rgb ? 3 : 1);
  const uint8_t* prev = j->f0 ? j->frames + (j->f0 - 1) * fb : j->prev0;
  if (j->rgb) {
    orc_motion_rgb(j->frames + j->f0 * fb, j->f1 - j->f0, j->w, j->h, j->thr, prev, j->out + j->f0 * px);
  } else if (!prev) {
    orc_motion_gray(j->frames + j->f0 * fb, j->f1 - j->f0, j->w, j->h, j->thr, j->out + j->f0 * px);
  } else {  /* gray with a halo frame: run from f0 - 1 and drop its mask */
    uint8_t* tmp = (uint8_t*)malloc((j->f1 - j->f0 + 1) * px);
    orc_motion_gray(prev, j->f1 - j->f0 + 1, j->w, j->h, j->thr, tmp);
    memcpy(j->out + j->f0 * px, tmp + px, (j->f1 - j->f0) * px);
    free(tmp);
  }
  return NULL;
}

/* fmt 1 = gray, 3 = RGB; prev0: the halo frame before frame 0 (RGB only),
 * or NULL for the black initial token. */
void orc_motion_mt(const uint8_t* frames, size_t count, unsigned w, unsigned h, int fmt, uint8_t threshold,
                   const uint8_t* prev0, uint8_t* out, unsigned threads) {
  if (threads < 1) threads = 1;
  if (threads > count) threads = count ? (unsigned)count : 1;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  motion_job* jobs = (motion_job*)malloc(sizeof(motion_job) * threads);
  for (unsigned t = 0; t < threads; ++t) {
    motion_job jb = {frames, count * t / threads, count * (t + 1) / threads, w, h, threshold, fmt == 3,
                     fmt == 3 ? prev0 : NULL, out};
    jobs[t] = jb;
    pthread_create(&tid[t], NULL, motion_range, &jobs[t]);
  }
  for (unsigned t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid); free(jobs);
}

/* ------------------------------------------------------------------------
 * Channel slot walk (channel.cpp:9-32) and comparator (bench.cpp:307-326)
 * ---------------------------------------------------------------------- */
size_t orc_capacity_tokens(uint32_t r, int has_delay) {
  return has_delay ? (size_t)r * 3 + 1 : (size_t)r * 2;
}
size_t orc_write_slot(uint32_t r, int has_delay, unsigned phase) {
  return has_delay ? (size_t)(phase % 3) * r + 1 : (size_t)(phase % 2) * r;
}
size_t orc_read_slot(uint32_t r, int has_delay, unsigned phase) {
  return has_delay ? (size_t)(phase % 3) * r : (size_t)(phase % 2) * r;
}

int64_t orc_compare_samples(const float* got, const float* want, size_t samples, double tol,
                            double* worst_err) {
  int64_t first = -1;
  double worst = 0.0;
  for (size_t i = 0; i < samples; ++i) {
    const double gr = got[2 * i], gi = got[2 * i + 1];
    const double wr = want[2 * i], wi = want[2 * i + 1];
    const double mag = hypot(wr, wi);
    const double err = hypot(gr - wr, gi - wi) / (mag > 1e-3 ? mag : 1e-3);
    if (err > worst || err != err) worst = err;
    if ((err > tol || err != err) && first < 0) first = (int64_t)i;
  }
  if (worst_err) *worst_err = worst;
  return first;
}
