/*
 * dedisp_oracle.c -- CPU restatement of the reference dedispersion hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: it may be
 * loaded by tests/, by __graft_entry__.smoke() and by bench.py's
 * cpu_baseline / --impl reference legs, never by the product path
 * (paper_1601_05052_b200/).  It restates, in plain C, the algorithms of
 * /root/reference/proj/core (C++20), citing the file:line each function
 * follows.  Parity is pinned by tests/test_oracle.py against the golden
 * fingerprints in tests/golden/golden.json, which were produced by the
 * reference itself (oracle/_ref, built from the unmodified reference sources
 * by oracle/Makefile; generating script tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared -pthread -lm
 * (-ffp-contract=off: the reference is built for baseline x86-64, which has
 * no FMA, so no contraction ever happens there either.)
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_CAPACITY 2

/* ------------------------------------------------------------------ */
/* FNV-1a 64 over raw little-endian bytes.       */
/* ------------------------------------------------------------------ */
uint64_t or_fnv1a(const void* data, uint64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ------------------------------------------------------------------ */
/* Geometry: setup.hpp:23-29 (channel_frequency, highest_frequency,     */
/* trial_dm) and setup.cpp:31-46 (ObservationSetup::validate).          */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t samples_per_second;
  uint32_t channels;
  double f_min;
  double channel_width;
  double dm_first;
  double dm_step;
} or_setup;

static double ch_freq(const or_setup* s, uint32_t ch) {
  return s->f_min + (double)ch * s->channel_width;
}
static double top_freq(const or_setup* s) { return ch_freq(s, s->channels - 1); }
static double dm_value(const or_setup* s, uint32_t i) {
  return s->dm_first + (double)i * s->dm_step;
}

int or_setup_validate(const or_setup* s) {
  if (s->samples_per_second < 1 || s->channels < 1) return OR_INVALID;
  if (!(s->f_min > 0.0) || !isfinite(s->f_min)) return OR_INVALID;
  if (!(s->channel_width > 0.0) || !isfinite(s->channel_width)) return OR_INVALID;
  if (!(s->dm_step > 0.0) || !isfinite(s->dm_step)) return OR_INVALID;
  if (!(s->dm_first >= 0.0) || !isfinite(s->dm_first)) return OR_INVALID;
  return OR_OK;
}

/* setup.cpp:48-62 -- Eq. 1 in FP64 with k = 4150 (setup.cpp:19). */
int or_delay_seconds(double dm, double f_ch, double f_hi, double* out) {
  if (!isfinite(dm) || !isfinite(f_ch) || !isfinite(f_hi)) return OR_INVALID;
  if (dm < 0.0 || f_ch <= 0.0 || f_hi <= 0.0 || f_ch > f_hi) return OR_INVALID;
  const double inv_low = 1.0 / (f_ch * f_ch);
  const double inv_high = 1.0 / (f_hi * f_hi);
  *out = 4150.0 * dm * (inv_low - inv_high);
  return OR_OK;
}

/* setup.cpp:66-105 (make_table_shell + build_delay_table) and :107-110
 * (build_zero_delay_table).  DM-major uint32 [num_dms][channels]. */
int or_build_delay_table(const or_setup* s, uint32_t num_dms, uint64_t cap_bytes, int zero,
                         uint32_t* shifts, uint32_t* max_delay_out) {
  if (or_setup_validate(s) != OR_OK || num_dms < 1) return OR_INVALID;
  const unsigned __int128 bytes = (unsigned __int128)num_dms * s->channels * 4u;
  if (bytes > cap_bytes) return OR_CAPACITY;
  const uint64_t entries = (uint64_t)num_dms * s->channels;
  if (zero) {
    memset(shifts, 0, entries * 4u);
    *max_delay_out = 0;
    return OR_OK;
  }
  const double f_hi = top_freq(s);
  const double rate = (double)s->samples_per_second;
  uint32_t mx = 0;
  for (uint32_t dm = 0; dm < num_dms; ++dm) {
    const double trial = dm_value(s, dm);
    uint32_t* row = shifts + (uint64_t)dm * s->channels;
    for (uint32_t ch = 0; ch < s->channels; ++ch) {
      double sec = 0.0;
      if (or_delay_seconds(trial, ch_freq(s, ch), f_hi, &sec) != OR_OK) return OR_INVALID;
      row[ch] = (uint32_t)llround(sec * rate);
      if (row[ch] > mx) mx = row[ch];
    }
  }
  *max_delay_out = mx;
  return OR_OK;
}

/* setup.cpp:112-137 -- t = s * ceil((s + max_delay) / s), flop = d*s*c. */
int or_instance_sizing(const or_setup* s, uint32_t num_dms, uint64_t* num_samples,
                       uint64_t* flop, uint32_t* max_delay) {
  if (or_setup_validate(s) != OR_OK || num_dms < 1) return OR_INVALID;
  double worst = 0.0;
  if (or_delay_seconds(dm_value(s, num_dms - 1), ch_freq(s, 0), top_freq(s), &worst) != OR_OK)
    return OR_INVALID;
  const double worst_samples = worst * (double)s->samples_per_second;
  if (worst_samples >= 4294967295.0) return OR_CAPACITY;
  const uint32_t md = (uint32_t)llround(worst_samples);
  const uint64_t rate = s->samples_per_second;
  const uint64_t blocks = (rate + md + rate - 1) / rate;
  *num_samples = blocks * rate;
  *flop = (uint64_t)num_dms * rate * s->channels;
  *max_delay = md;
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Noise: filterbank.cpp:22-49 (GaussianStream: mt19937_64, top-53-bit  */
/* uniforms, Box-Muller returning r*cos first and caching r*sin) and    */
/* filterbank.cpp:60-80 (channel-major fill, float(sigma * g)).         */
/* mt19937_64 is restated from its published definition (the C++11     */
/* standard's parameters), since the reference takes it from libstdc++. */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_mt64;

static void mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(or_mt64* g) {
  static const uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (g->mt[i] & kUpper) | (g->mt[(i + 1) % 312] & kLower);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1u) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static double unit53(or_mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

int or_noise_filterbank(uint32_t channels, uint64_t num_samples, float sigma, uint64_t seed,
                        float* out) {
  if (channels < 1 || num_samples < 1 || !isfinite(sigma) || sigma < 0.0f) return OR_INVALID;
  const uint64_t n = (uint64_t)channels * num_samples;
  if (!(sigma > 0.0f)) {
    memset(out, 0, n * sizeof(float));
    return OR_OK;
  }
  or_mt64* g = (or_mt64*)malloc(sizeof(or_mt64));
  if (!g) return OR_CAPACITY;
  mt64_seed(g, seed);
  const double kPi = 3.14159265358979323846;
  int have_spare = 0;
  double spare = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    double z;
    if (have_spare) {
      have_spare = 0;
      z = spare;
    } else {
      const double u1 = 1.0 - unit53(g);
      const double u2 = unit53(g);
      const double radius = sqrt(-2.0 * log(u1));
      const double angle = 2.0 * kPi * u2;
      spare = radius * sin(angle);
      have_spare = 1;
      z = radius * cos(angle);
    }
    out[i] = (float)((double)sigma * z);
  }
  free(g);
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* kernels.cpp:44-56 (config_valid); the four parameters of             */
/* kernels.hpp:40-52.                                                   */
/* ------------------------------------------------------------------ */
typedef struct {
  uint32_t items_time, items_dm, work_time, work_dm;
} or_config;

int or_config_valid(const or_config* k, uint32_t num_dms, uint32_t s, uint32_t max_block_items,
                    uint32_t max_accumulators) {
  if (!k->items_time || !k->items_dm || !k->work_time || !k->work_dm) return 0;
  const uint64_t tt = (uint64_t)k->items_time * k->work_time;
  const uint64_t td = (uint64_t)k->items_dm * k->work_dm;
  if (tt > s || s % tt) return 0;
  if (td > num_dms || num_dms % td) return 0;
  if ((uint64_t)k->items_time * k->items_dm > max_block_items) return 0;
  if ((uint64_t)k->work_time * k->work_dm > max_accumulators) return 0;
  return 1;
}

/* kernels.cpp:16-28 (check_pair): t >= s + max_delay. */
static int pair_ok(uint64_t t, uint32_t s, const uint32_t* shifts, uint64_t entries) {
  uint32_t mx = 0;
  for (uint64_t i = 0; i < entries; ++i)
    if (shifts[i] > mx) mx = shifts[i];
  return t >= (uint64_t)s + mx;
}

/* kernels.cpp:83-108 -- Algorithm 1: one fp32 accumulator per output,
 * initialised to 0.0f, channels added in ascending order. */
int or_dedisperse_reference(const float* in, uint32_t channels, uint64_t t,
                            const uint32_t* shifts, uint32_t num_dms, uint32_t s, float* out) {
  if (!pair_ok(t, s, shifts, (uint64_t)num_dms * channels)) return OR_INVALID;
  for (uint32_t dm = 0; dm < num_dms; ++dm) {
    const uint32_t* row = shifts + (uint64_t)dm * channels;
    float* o = out + (uint64_t)dm * s;
    for (uint32_t j = 0; j < s; ++j) {
      float acc = 0.0f;
      for (uint32_t ch = 0; ch < channels; ++ch) acc += in[(uint64_t)ch * t + j + row[ch]];
      o[j] = acc;
    }
  }
  return OR_OK;
}

/* kernels.cpp:117-206 -- tiled restatement (run_tile :134-188): per tile
 * and channel, stage [t0+lo, t0+hi+tile_time) then lane-blocked adds into
 * private accumulators, ascending channels.  Tiles are claimed dynamically
 * by `threads` pthreads, as ThreadPool::for_each_index does
 * (thread_pool.cpp:70-99).  Used as the "port" CPU baseline. */
typedef struct {
  const float* in;
  uint32_t c;
  uint64_t t;
  const uint32_t* shifts;
  uint32_t d, s;
  or_config k;
  float* out;
  uint64_t tiles;
  uint32_t tiles_time;
  volatile uint64_t next;
  pthread_mutex_t lock;
  uint64_t staged;
} tiled_job;

static void run_tile(tiled_job* j, uint64_t tile, float* acc, float** stage, uint64_t* cap,
                     uint64_t* fetched) {
  const uint32_t tt = j->k.items_time * j->k.work_time;
  const uint32_t td = j->k.items_dm * j->k.work_dm;
  const uint32_t dm0 = (uint32_t)(tile / j->tiles_time) * td;
  const uint32_t t0 = (uint32_t)(tile % j->tiles_time) * tt;
  memset(acc, 0, (uint64_t)td * tt * sizeof(float));
  for (uint32_t ch = 0; ch < j->c; ++ch) {
    uint32_t lo = j->shifts[(uint64_t)dm0 * j->c + ch], hi = lo;
    for (uint32_t ld = 1; ld < td; ++ld) {
      const uint32_t v = j->shifts[(uint64_t)(dm0 + ld) * j->c + ch];
      if (v < lo) lo = v;
      if (v > hi) hi = v;
    }
    const uint64_t span = (uint64_t)(hi - lo) + tt;
    if (span > *cap) {
      free(*stage);
      *stage = (float*)malloc(span * sizeof(float));
      *cap = span;
    }
    memcpy(*stage, j->in + (uint64_t)ch * j->t + t0 + lo, span * sizeof(float));
    *fetched += span;
    for (uint32_t wd = 0; wd < j->k.work_dm; ++wd)
      for (uint32_t id = 0; id < j->k.items_dm; ++id) {
        const uint32_t ld = wd * j->k.items_dm + id;
        const float* src = *stage + (j->shifts[(uint64_t)(dm0 + ld) * j->c + ch] - lo);
        float* a = acc + (uint64_t)ld * tt;
        for (uint32_t wt = 0; wt < j->k.work_time; ++wt) {
          const uint32_t base = wt * j->k.items_time;
          for (uint32_t it = 0; it < j->k.items_time; ++it) a[base + it] += src[base + it];
        }
      }
  }
  for (uint32_t ld = 0; ld < td; ++ld)
    memcpy(j->out + (uint64_t)(dm0 + ld) * j->s + t0, acc + (uint64_t)ld * tt, tt * sizeof(float));
}

static void* tiled_worker(void* arg) {
  tiled_job* j = (tiled_job*)arg;
  const uint32_t tt = j->k.items_time * j->k.work_time;
  const uint32_t td = j->k.items_dm * j->k.work_dm;
  float* acc = (float*)malloc((uint64_t)tt * td * sizeof(float));
  float* stage = NULL;
  uint64_t cap = 0, fetched = 0;
  for (;;) {
    const uint64_t tile = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (tile >= j->tiles) break;
    run_tile(j, tile, acc, &stage, &cap, &fetched);
  }
  free(acc);
  free(stage);
  __atomic_fetch_add(&j->staged, fetched, __ATOMIC_RELAXED);
  return NULL;
}

int or_dedisperse_tiled(const float* in, uint32_t channels, uint64_t t, const uint32_t* shifts,
                        uint32_t num_dms, uint32_t s, const or_config* k, int threads,
                        float* out, uint64_t* staged_out) {
  if (!or_config_valid(k, num_dms, s, 0xFFFFFFFFu, 0xFFFFFFFFu)) return OR_INVALID;
  if (!pair_ok(t, s, shifts, (uint64_t)num_dms * channels)) return OR_INVALID;
  tiled_job j;
  memset(&j, 0, sizeof(j));
  j.in = in;
  j.c = channels;
  j.t = t;
  j.shifts = shifts;
  j.d = num_dms;
  j.s = s;
  j.k = *k;
  j.out = out;
  j.tiles_time = s / (k->items_time * k->work_time);
  j.tiles = (uint64_t)j.tiles_time * (num_dms / (k->items_dm * k->work_dm));
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 1; i < threads; ++i) pthread_create(&th[i], NULL, tiled_worker, &j);
  tiled_worker(&j);
  for (int i = 1; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
  if (staged_out) *staged_out = j.staged;
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* count_loads.cpp:9-68 -- staged (:33-45) and ideal (:50-65) loads.    */
/* ------------------------------------------------------------------ */
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

int or_count_loads(const uint32_t* shifts, uint32_t channels, uint32_t num_dms, uint32_t s,
                   const or_config* k, uint64_t* staged, uint64_t* ideal) {
  if (!or_config_valid(k, num_dms, s, 0xFFFFFFFFu, 0xFFFFFFFFu)) return OR_INVALID;
  const uint64_t tt = (uint64_t)k->items_time * k->work_time;
  const uint32_t td = k->items_dm * k->work_dm;
  const uint64_t tiles_time = s / tt;
  uint64_t st = 0, id = 0;
  for (uint32_t dm0 = 0; dm0 < num_dms; dm0 += td)
    for (uint32_t ch = 0; ch < channels; ++ch) {
      uint32_t lo = shifts[(uint64_t)dm0 * channels + ch], hi = lo;
      for (uint32_t ld = 1; ld < td; ++ld) {
        const uint32_t v = shifts[(uint64_t)(dm0 + ld) * channels + ch];
        if (v < lo) lo = v;
        if (v > hi) hi = v;
      }
      st += ((uint64_t)(hi - lo) + tt) * tiles_time;
    }
  uint32_t* col = (uint32_t*)malloc((size_t)num_dms * 4u);
  for (uint32_t ch = 0; ch < channels; ++ch) {
    for (uint32_t dm = 0; dm < num_dms; ++dm) col[dm] = shifts[(uint64_t)dm * channels + ch];
    qsort(col, num_dms, 4u, cmp_u32);
    uint64_t begin = col[0], end = (uint64_t)col[0] + s;
    for (uint32_t dm = 1; dm < num_dms; ++dm) {
      if (col[dm] > end) {
        id += end - begin;
        begin = col[dm];
      }
      end = (uint64_t)col[dm] + s;
    }
    id += end - begin;
  }
  free(col);
  *staged = st;
  *ideal = id;
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* tuner.cpp:19-30 + :103-134 -- lexicographic divisor enumeration.     */
/* Writes up to `cap` configs, returns the total count (0 = empty).     */
/* ------------------------------------------------------------------ */
static uint32_t divisors(uint32_t n, uint32_t* out) {
  uint32_t ns = 0, nl = 0;
  uint32_t large[2048];
  for (uint64_t k = 1; k * k <= n; ++k)
    if (n % k == 0) {
      out[ns++] = (uint32_t)k;
      if (k != n / k) large[nl++] = (uint32_t)(n / k);
    }
  for (uint32_t i = 0; i < nl; ++i) out[ns + i] = large[nl - 1 - i];
  return ns + nl;
}

uint64_t or_enumerate_configs(uint32_t num_dms, uint32_t s, uint32_t max_block_items,
                              uint32_t max_accumulators, or_config* out, uint64_t cap) {
  if (!num_dms || !s) return 0;
  uint32_t tdiv[4096], ddiv[4096];
  const uint32_t nt = divisors(s, tdiv), nd = divisors(num_dms, ddiv);
  uint64_t n = 0;
  for (uint32_t a = 0; a < nt; ++a) {
    const uint32_t it = tdiv[a];
    if (it > max_block_items) break;
    for (uint32_t b = 0; b < nd; ++b) {
      const uint32_t idm = ddiv[b];
      if ((uint64_t)it * idm > max_block_items) break;
      for (uint32_t c = 0; c < nt; ++c) {
        const uint32_t wt = tdiv[c];
        if (wt > max_accumulators) break;
        const uint64_t tt = (uint64_t)it * wt;
        if (tt > s || s % tt) continue;
        for (uint32_t e = 0; e < nd; ++e) {
          const uint32_t wd = ddiv[e];
          if ((uint64_t)wt * wd > max_accumulators) break;
          const uint64_t td = (uint64_t)idm * wd;
          if (td > num_dms || num_dms % td) continue;
          if (n < cap) {
            out[n].items_time = it;
            out[n].items_dm = idm;
            out[n].work_time = wt;
            out[n].work_dm = wd;
          }
          ++n;
        }
      }
    }
  }
  return n;
}
