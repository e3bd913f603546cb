/*
 * synth.c -- seeded synthetic input generators shared by the oracle tests and
 * the product tests / bench.  Holds NONE of the method's arithmetic (no rANS,
 * no model quantisation, no metadata): it only turns counter-based SplitMix64
 * draws into bytes through integer inverse-CDF threshold tables that the
 * Python side (synth/__init__.py) computes from the workload recipes in
 * DESIGN.md "Input recipe".
 *
 * Draw i of a stream with seed s is  u_i = mix64(s + (i + 1) * GAMMA)
 * (the SplitMix64 output at position i), so any sub-range can be generated
 * independently and the result does not depend on the thread count.
 * Byte_i = #{k : thr[k] <= u_i} clamped to 255, where thr[] is the table's
 * cumulative distribution scaled to 2^64.
 */
#include <stdint.h>
#include <stddef.h>
#include <pthread.h>

#define GAMMA 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint8_t draw_byte(uint64_t u, const uint64_t *thr) {
  /* branch-free lower bound over 256 sorted thresholds: count of thr[k] <= u */
  uint32_t k = 0;
  for (uint32_t step = 128; step > 0; step >>= 1)
    if (thr[k + step - 1] <= u) k += step;
  return (uint8_t)(k > 255 ? 255 : k);
}

typedef struct {
  uint8_t *out;
  uint64_t begin, end; /* absolute draw indices */
  uint64_t seed;
  const uint64_t *tables; /* n_tables x 256 */
  uint32_t n_tables;
  uint64_t tile; /* symbols per tile (table chosen per tile); 0 = single table */
} job_t;

static void *run_job(void *arg) {
  job_t *j = (job_t *)arg;
  const uint64_t *thr = j->tables;
  uint64_t cur_tile = UINT64_MAX;
  for (uint64_t i = j->begin; i < j->end; ++i) {
    if (j->tile) {
      uint64_t t = i / j->tile;
      if (t != cur_tile) {
        cur_tile = t;
        uint64_t h = mix64((j->seed ^ 0xD1B54A32D192ED03ULL) + (t + 1) * GAMMA);
        thr = j->tables + 256 * (h % j->n_tables);
      }
    }
    uint64_t u = mix64(j->seed + (i + 1) * GAMMA);
    j->out[i - j->begin] = draw_byte(u, thr);
  }
  return NULL;
}

/* Fill out[0..count) with draws [start, start+count) of stream `seed`.
 * tables: n_tables x 256 thresholds (uint64, non-decreasing per table).
 * tile == 0: table 0 for every draw; else draw i uses the table picked by a
 * hash of (seed, i / tile).  threads <= 0 means 1. Returns 0. */
int synth_fill(uint8_t *out, uint64_t start, uint64_t count, uint64_t seed,
               const uint64_t *tables, uint32_t n_tables, uint64_t tile,
               int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  if (count < (1u << 20)) threads = 1;
  pthread_t th[64];
  job_t jobs[64];
  for (int t = 0; t < threads; ++t) {
    uint64_t b = count * (uint64_t)t / (uint64_t)threads;
    uint64_t e = count * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].out = out + b;
    jobs[t].begin = start + b;
    jobs[t].end = start + e;
    jobs[t].seed = seed;
    jobs[t].tables = tables;
    jobs[t].n_tables = n_tables ? n_tables : 1;
    jobs[t].tile = tile;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, run_job, &jobs[t]);
  run_job(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* Raw SplitMix64 draws (for tests that need random words / fuzz parameters). */
void synth_u64(uint64_t *out, uint64_t start, uint64_t count, uint64_t seed) {
  for (uint64_t i = 0; i < count; ++i) out[i] = mix64(seed + (start + i + 1) * GAMMA);
}

/* Index-keyed draws for the adaptive workload: value_i = base[k] + j where
 * k = mid[i] and j = #{t < len[k] : thr[off[k] + t] <= u_i} (clamped), u_i the
 * SplitMix64 draw i.  thr: per model, len[k] non-decreasing cumulative
 * thresholds scaled to 2^64.  threads <= 0 means 1. */
typedef struct {
  uint16_t *out;
  const uint8_t *mid;
  uint64_t begin, end, seed;
  const uint64_t *thr, *off;
  const uint32_t *base, *len;
} ljob_t;

static void *run_ljob(void *arg) {
  ljob_t *j = (ljob_t *)arg;
  for (uint64_t i = j->begin; i < j->end; ++i) {
    uint32_t k = j->mid[i - j->begin];
    const uint64_t *t = j->thr + j->off[k];
    uint64_t u = mix64(j->seed + (i + 1) * GAMMA);
    uint32_t lo = 0, hi = j->len[k] - 1; /* first t with u < thr[t] */
    while (lo < hi) {
      uint32_t m = (lo + hi) >> 1;
      if (t[m] <= u) lo = m + 1; else hi = m;
    }
    j->out[i - j->begin] = (uint16_t)(j->base[k] + lo);
  }
  return NULL;
}

int synth_fill_models(uint16_t *out, const uint8_t *mid, uint64_t start, uint64_t count, uint64_t seed,
                      const uint64_t *thr, const uint64_t *off, const uint32_t *base, const uint32_t *len,
                      int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  if (count < (1u << 20)) threads = 1;
  pthread_t th[64];
  ljob_t jobs[64];
  for (int t = 0; t < threads; ++t) {
    uint64_t b = count * (uint64_t)t / (uint64_t)threads;
    uint64_t e = count * (uint64_t)(t + 1) / (uint64_t)threads;
    ljob_t jb = {out + b, mid + b, start + b, start + e, seed, thr, off, base, len};
    jobs[t] = jb;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, run_ljob, &jobs[t]);
  run_ljob(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* Byte histogram of x[0..n) (input statistics for the model the tests and the
 * bench build; no method arithmetic), on up to `threads` threads. */
typedef struct {
  const uint8_t *x;
  uint64_t n;
  uint64_t h[256];
} hjob_t;

static void *run_hjob(void *arg) {
  hjob_t *j = (hjob_t *)arg;
  uint64_t h4[4][256] = {{0}};
  uint64_t i = 0;
  for (; i + 4 <= j->n; i += 4) {
    ++h4[0][j->x[i]];
    ++h4[1][j->x[i + 1]];
    ++h4[2][j->x[i + 2]];
    ++h4[3][j->x[i + 3]];
  }
  for (; i < j->n; ++i) ++h4[0][j->x[i]];
  for (int k = 0; k < 256; ++k) j->h[k] = h4[0][k] + h4[1][k] + h4[2][k] + h4[3][k];
  return NULL;
}

void synth_histogram(const uint8_t *x, uint64_t n, uint64_t *hist, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  if (n < (1u << 22)) threads = 1;
  pthread_t th[64];
  hjob_t jobs[64];
  for (int t = 0; t < threads; ++t) {
    uint64_t b = n * (uint64_t)t / (uint64_t)threads, e = n * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].x = x + b;
    jobs[t].n = e - b;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, run_hjob, &jobs[t]);
  run_hjob(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  for (int k = 0; k < 256; ++k) {
    uint64_t s = 0;
    for (int t = 0; t < threads; ++t) s += jobs[t].h[k];
    hist[k] = s;
  }
}
