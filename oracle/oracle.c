/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain, slow, single-threaded C11 reference of Recoil, arXiv 2306.12141
 * (/root/reference/PAPER.md, cited P:<line>).  Every function follows the
 * paper's definition or algorithm in the paper's order; where the paper is
 * silent or ambiguous the reading is named (Z<k> = SURVEY.md §8(c) table,
 * also listed in DESIGN.md "Readings").  No blocking, fusion or reordering.
 *
 * Constants: tab:rans_params -- 32-bit state, L = 2^16, b = 16.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

#define L_BOUND 65536u  /* L = 2^16 */
#define B_BITS 16u      /* b = 16 */

static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

/* ------------------------------------------------------------------ */
/* Model (quantiser = reading Z19, the paper gives none)      */
/* ------------------------------------------------------------------ */

/* Floor of hist*2^n/total, every present symbol at least 1, then the
 * shortfall handed out by largest remainder (ties: smaller symbol); an
 * excess (caused by the min-1 rule) is taken from the largest f (ties:
 * smaller count, then smaller symbol).  `count` entries (256 for bytes; a
 * model of the adaptive codec may have up to 2^16). */
int or_quantize(const uint64_t *hist, uint32_t count, uint32_t n, uint32_t *f) {
  if (n < 1 || n > 16 || count < 1) return OR_E_ARG;
  uint64_t total = 0, distinct = 0, R = 1ull << n;
  for (uint32_t s = 0; s < count; ++s) {
    total += hist[s];
    if (hist[s]) distinct++;
  }
  if (total == 0 || distinct > R) return OR_E_MODEL;
  uint64_t *rem = (uint64_t *)calloc(count, sizeof(uint64_t));
  int *given = (int *)calloc(count, sizeof(int));
  if (!rem || !given) { free(rem); free(given); return OR_E_NOMEM; }
  uint64_t sum = 0;
  for (uint32_t s = 0; s < count; ++s) {
    if (!hist[s]) {
      f[s] = 0;
      rem[s] = 0;
      continue;
    }
    /* hist * R may exceed 64 bits for large counts: 128-bit product */
    unsigned __int128 prod = (unsigned __int128)hist[s] * R;
    uint64_t q = (uint64_t)(prod / total);
    rem[s] = (uint64_t)(prod % total);
    f[s] = (uint32_t)(q < 1 ? 1 : q);
    if (q < 1) given[s] = 1; /* raised to 1: already rounded up */
    sum += f[s];
  }
  /* largest remainder: the shortfall is < the number of symbols not raised
   * to 1, so each gets at most one extra count */
  while (sum < R) {
    int64_t best = -1;
    for (uint32_t s = 0; s < count; ++s)
      if (hist[s] && !given[s] && (best < 0 || rem[s] > rem[best])) best = s;
    if (best < 0) { free(rem); free(given); return OR_E_MODEL; } /* unreachable */
    given[best] = 1;
    f[best]++;
    sum++;
  }
  while (sum > R) { /* largest f first; ties: smaller count, then smaller symbol */
    int64_t best = -1;
    for (uint32_t s = 0; s < count; ++s)
      if (f[s] > 1 && (best < 0 || f[s] > f[best] || (f[s] == f[best] && hist[s] < hist[best]))) best = s;
    f[best]--;
    sum--;
  }
  free(rem);
  free(given);
  return OR_OK;
}

int or_build_model(const uint64_t hist[256], uint32_t n, uint32_t f[256]) {
  return or_quantize(hist, 256, n, f);
}

static void cdf_of(const uint32_t f[256], uint32_t F[256]) {
  uint32_t acc = 0;
  for (int t = 0; t < 256; ++t) {
    F[t] = acc; /* F(t) = sum_{u<t} f(u) */
    acc += f[t];
  }
}

/* Eq. 1: x_i = 2^n floor(x_{i-1}/f(s_i)) + F(s_i) + (x_{i-1} mod f(s_i)) */
uint64_t or_encode_step(uint64_t x, uint32_t f, uint32_t F, uint32_t n) {
  return ((x / f) << n) + F + (x % f);
}

/* Eq. 2: s = t with F(t) <= x mod 2^n < F(t+1), found by a
 * plain scan of the CDF; x_{i-1} = f(s) floor(x/2^n) - F(s) + (x mod 2^n). */
int or_decode_step(uint32_t x, const uint32_t f[256], uint32_t n, uint32_t *s, uint32_t *x_prev) {
  uint32_t F[256];
  cdf_of(f, F);
  uint32_t slot = x & ((1u << n) - 1);
  for (uint32_t t = 0; t < 256; ++t) {
    if (f[t] && F[t] <= slot && slot < F[t] + f[t]) {
      *s = t;
      *x_prev = f[t] * (x >> n) - F[t] + slot;
      return OR_OK;
    }
  }
  return OR_E_MODEL;
}

/* Eq. 3: while x >= (2^b / 2^n) L f(s_{i+1}): B_p = x mod 2^b,
 * x = floor(x / 2^b), p++.  (2^b/2^n) L f = f * 2^(32-n); compared in 64
 * bits so f = 2^n does not overflow (reading Z2). */
int or_renorm_encode(uint64_t *x, uint32_t f_next, uint32_t n, uint16_t *words, uint64_t *p) {
  uint64_t threshold = ((uint64_t)1 << B_BITS) * L_BOUND / ((uint64_t)1 << n) * f_next;
  int steps = 0;
  while (*x >= threshold) {
    words[*p] = (uint16_t)(*x % (1u << B_BITS));
    *x = *x / (1u << B_BITS);
    (*p)++;
    steps++;
  }
  return steps;
}

/* Eq. 4: while x < L: x = x 2^b + B_p, p--. */
int or_renorm_decode(uint64_t *x, const uint16_t *words, int64_t *p) {
  int steps = 0;
  while (*x < L_BOUND) {
    if (*p < 0) return OR_E_UNDERFLOW;
    *x = *x * (1u << B_BITS) + words[*p];
    (*p)--;
    steps++;
  }
  return steps;
}

/* ------------------------------------------------------------------ */
/* W-way interleaved rANS (fig:interleaved_rans)            */
/* ------------------------------------------------------------------ */

/* Symbols are processed in groups of W; lane j encodes symbols i with
 * i mod W = j.  Before a lane encodes symbol i it is renormalised against
 * that symbol (Eq. 3 with s_{i+1} = the lane's next symbol), and the
 * renormalisation outputs of a group boundary are interleaved into the one
 * stream in increasing lane ID (reading Z4).  A lane without a
 * symbol in the last group neither renormalises nor encodes (Z5).  Initial
 * state L (Z3).  Each emitted word is logged as an event carrying the
 * lane's most recently encoded symbol index (i - W) and the post-emission
 * state (Z7), which the Lemma bounds by L. */
int64_t or_interleaved_encode(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                              uint32_t W, uint16_t *words, uint32_t *final_states,
                              or_event *events, uint64_t *max_renorm_steps) {
  if (W < 1 || W > 32 || n < 1 || n > 16) return OR_E_ARG;
  uint32_t F[256];
  cdf_of(f, F);
  for (uint64_t i = 0; i < N; ++i)
    if (f[sym[i]] == 0) return OR_E_MODEL;
  uint64_t x[32];
  for (uint32_t j = 0; j < W; ++j) x[j] = L_BOUND;
  uint64_t G = (N + W - 1) / W, p = 0, maxsteps = 0;
  for (uint64_t g = 0; g < G; ++g) {
    /* renormalisation outputs of this group boundary, increasing lane ID */
    for (uint32_t j = 0; j < W; ++j) {
      uint64_t i = g * W + j;
      if (i >= N) continue;
      uint64_t p_before = p;
      int steps = or_renorm_encode(&x[j], f[sym[i]], n, words, &p);
      if ((uint64_t)steps > maxsteps) maxsteps = (uint64_t)steps;
      for (uint64_t q = p_before; q < p; ++q) {
        if (events) {
          events[q].idx = (int64_t)i - (int64_t)W;
          events[q].lane = j;
          events[q].state = (uint32_t)x[j]; /* state after the (last) emission */
        }
      }
    }
    /* encode the group (Eq. 1) */
    for (uint32_t j = 0; j < W; ++j) {
      uint64_t i = g * W + j;
      if (i >= N) continue;
      x[j] = or_encode_step(x[j], f[sym[i]], F[sym[i]], n);
      if (x[j] >> 32) return OR_E_OVERFLOW; /* 32-bit state */
    }
  }
  for (uint32_t j = 0; j < W; ++j) final_states[j] = (uint32_t)x[j];
  if (max_renorm_steps) *max_renorm_steps = maxsteps;
  return (int64_t)p;
}

/* Plain slot -> symbol table built from Eq. 2's definition. */
static void lut_of(const uint32_t f[256], uint32_t n, uint8_t *lut) {
  uint32_t F[256];
  cdf_of(f, F);
  (void)n;
  for (uint32_t t = 0; t < 256; ++t) /* lut[slot] = t  <=>  F(t) <= slot < F(t) + f(t) */
    for (uint32_t slot = F[t]; slot < F[t] + f[t]; ++slot) lut[slot] = (uint8_t)t;
}

/* Serial decoder: the stream is read backwards from the end;
 * per group, decoders that need to renormalise read in decreasing lane ID,
 * then the group's symbols are decoded.  The stack property means
 * the decode of the whole stream ends with every lane back at the initial
 * state L and the stream exhausted. */
int or_interleaved_decode(const uint16_t *words, uint64_t B, const uint32_t *final_states,
                          uint64_t N, const uint32_t f[256], uint32_t n, uint32_t W, uint8_t *out) {
  if (W < 1 || W > 32) return OR_E_ARG;
  uint32_t F[256];
  cdf_of(f, F);
  uint8_t *lut = (uint8_t *)malloc(1u << n);
  if (!lut) return OR_E_NOMEM;
  lut_of(f, n, lut);
  uint64_t x[32];
  for (uint32_t j = 0; j < W; ++j) x[j] = final_states[j];
  int64_t p = (int64_t)B - 1;
  int64_t G = (int64_t)((N + W - 1) / W);
  int rc = OR_OK;
  for (int64_t g = G - 1; g >= -1 && rc == OR_OK; --g) {
    for (int32_t j = (int32_t)W - 1; j >= 0; --j) /* refill, decreasing lane ID */
      if (or_renorm_decode(&x[j], words, &p) < 0) { rc = OR_E_UNDERFLOW; break; }
    if (g < 0) break; /* g = -1: the outputs emitted before group 0 (n = 16, f = 1 only) */
    for (uint32_t j = 0; j < W; ++j) {
      uint64_t i = (uint64_t)g * W + j;
      if (i >= N) continue;
      uint32_t slot = (uint32_t)(x[j] & ((1u << n) - 1));
      uint32_t s = lut[slot];
      x[j] = (uint64_t)f[s] * (x[j] >> n) - F[s] + slot; /* Eq. 2 */
      out[i] = (uint8_t)s;
    }
  }
  free(lut);
  if (rc) return rc;
  if (p != -1) return OR_E_END;
  for (uint32_t j = 0; j < W; ++j)
    if (x[j] != L_BOUND) return OR_E_END;
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Backward scan, heuristic, split selection               */
/* ------------------------------------------------------------------ */

/* from the split position, scan backwards and keep, per lane, the
 * first event seen (its last renormalisation); ignore earlier ones; stop
 * when all W lanes are recorded.  The Synchronization Section starts at the
 * smallest recorded symbol index. */
int or_backward_scan(const or_event *ev, uint64_t e, uint32_t W, uint32_t *anchor_state,
                     int64_t *anchor_idx, int64_t *sync_start) {
  int found[32] = {0};
  uint32_t count = 0;
  for (int64_t o = (int64_t)e; o >= 0 && count < W; --o) {
    uint32_t j = ev[o].lane;
    if (found[j]) continue; /* "we ignore the previous renormalizations" */
    found[j] = 1;
    anchor_state[j] = ev[o].state;
    anchor_idx[j] = ev[o].idx;
    count++;
  }
  if (count < W) return 0; /* reading Z8: infeasible */
  int64_t mn = anchor_idx[0];
  for (uint32_t j = 0; j < W; ++j) {
    if (anchor_idx[j] < 0) return 0;
    if (anchor_idx[j] < mn) mn = anchor_idx[j];
  }
  *sync_start = mn;
  return 1;
}

static int64_t iabs64(int64_t v) { return v < 0 ? -v : v; }

/* H(t, t_s) = |t - T| + |t - t_s - T| */
int64_t or_heuristic(int64_t t, int64_t ts, int64_t T) { return iabs64(t - T) + iabs64(t - ts - T); }

/* Reading Z10' of P:325-333: the boundary index of the
 * previous split point is prev (-1 before the first); t = idx(e) - prev is
 * the number of symbols between the previous and the candidate split point
 * (this split's Synchronization Section included) and t_s = idx(e) -
 * sync_start(e) + 1.  T is the rounded-up average of the symbols still to be
 * split, T_m = ceil((N - prev - 1) / (M - m + 1)); for m = 1 this is the
 * printed T = ceil(N/M).  (With T fixed for every m the boundaries drift by
 * ~t_s/2 per split, since H is flat on t in [T, T + t_s], and the stream runs
 * out before M splits: 2159 of 2176 on a 10 MB rand_10.)  For boundary
 * m = 1..M-1 every event e with 0 < t <= 2 T_m whose backward scan is
 * feasible, whose Synchronization Section starts after prev and whose group
 * differences fit 16 bits is a candidate; the one with minimum
 * H(t, t_s) wins, ties to the smaller word offset.  No candidate: stop with
 * fewer splits. */
int64_t or_choose_splits(const or_event *ev, uint64_t n_ev, uint64_t N, uint32_t W, uint32_t M,
                         uint64_t *chosen) {
  return or_choose_splits_ex(ev, n_ev, N, W, M, 0, chosen);
}

/* flags & OR_SPLIT_PRINTED_T: the printed T = ceil(N/M) of P:329 for every
 * boundary instead of Z10''s T_m (kept to compare the two readings). */
int64_t or_choose_splits_ex(const or_event *ev, uint64_t n_ev, uint64_t N, uint32_t W, uint32_t M,
                            uint32_t flags, uint64_t *chosen) {
  if (M <= 1 || N == 0) return 0;
  int64_t prev = -1;
  int64_t count = 0;
  uint64_t first = 0; /* event idx is strictly increasing with the word offset (pinned by a test) */
  uint32_t st[32];
  int64_t ai[32];
  for (uint32_t m = 1; m < M; ++m) {
    int64_t T = (flags & OR_SPLIT_PRINTED_T) ? (int64_t)ceil_div(N, M)
                                             : (int64_t)ceil_div(N - (uint64_t)(prev + 1), M - m + 1);
    while (first < n_ev && ev[first].idx <= prev) first++;
    int64_t best = -1, best_h = 0;
    /* candidates with 0 < t <= 2T; a window without a feasible candidate is
     * doubled until one is found or the stream ends (reading Z10'') */
    for (int64_t limit = 2 * T; best < 0; limit *= 2) {
      for (uint64_t e = first; e < n_ev && ev[e].idx - prev <= limit; ++e) {
        int64_t ss;
        if (!or_backward_scan(ev, e, W, st, ai, &ss)) continue;
        if (ss <= prev) continue;
        if (ev[e].idx / W - ss / W > 65535) continue;
        int64_t t = ev[e].idx - prev;
        int64_t ts = ev[e].idx - ss + 1;
        int64_t h = or_heuristic(t, ts, T);
        if (best < 0 || h < best_h) {
          best = (int64_t)e;
          best_h = h;
        }
      }
      if (n_ev == 0 || ev[n_ev - 1].idx - prev <= limit) break; /* the window covers the rest */
    }
    if (best < 0) break;
    chosen[count++] = (uint64_t)best;
    prev = ev[best].idx;
  }
  return count;
}

/* ------------------------------------------------------------------ */
/* Data series                                              */
/* ------------------------------------------------------------------ */

static void put_bits(uint8_t *buf, uint64_t *pos, uint64_t value, uint32_t nbits) {
  for (int32_t k = (int32_t)nbits - 1; k >= 0; --k) { /* MSB first */
    if ((value >> k) & 1) buf[*pos >> 3] |= (uint8_t)(0x80u >> (*pos & 7));
    (*pos)++;
  }
}

static uint64_t get_bits(const uint8_t *buf, uint64_t *pos, uint32_t nbits) {
  uint64_t v = 0;
  for (uint32_t k = 0; k < nbits; ++k) {
    v = (v << 1) | ((buf[*pos >> 3] >> (7 - (*pos & 7))) & 1);
    (*pos)++;
  }
  return v;
}

static uint32_t bitlen(uint64_t v) { /* bits to hold v; one bit for zero (P:388 footnote) */
  uint32_t w = 1;
  while (w < 64 && (v >> w)) w++;
  return w;
}

/* Width field (field_bits wide) = w - 1, w = max bitlen(|v_i|) (reading Z14),
 * then each element's magnitude in w bits and, for a signed series, a sign
 * bit after it (1 = negative, reading Z16).  buf must be zeroed.  Returns
 * the bit position after the series. */
uint64_t or_pack_series(const int64_t *v, uint64_t count, int is_signed, uint32_t field_bits,
                        uint8_t *buf, uint64_t bitpos) {
  uint32_t w = 1;
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t b = bitlen((uint64_t)iabs64(v[i]));
    if (b > w) w = b;
  }
  put_bits(buf, &bitpos, w - 1, field_bits);
  for (uint64_t i = 0; i < count; ++i) {
    put_bits(buf, &bitpos, (uint64_t)iabs64(v[i]), w);
    if (is_signed) put_bits(buf, &bitpos, v[i] < 0 ? 1 : 0, 1);
  }
  return bitpos;
}

int64_t or_unpack_series(const uint8_t *buf, uint64_t buf_bits, uint64_t bitpos, uint64_t count,
                         int is_signed, uint32_t field_bits, int64_t *v) {
  if (bitpos + field_bits > buf_bits) return OR_E_CONTAINER;
  uint32_t w = (uint32_t)get_bits(buf, &bitpos, field_bits) + 1;
  if (bitpos + count * (w + (is_signed ? 1 : 0)) > buf_bits) return OR_E_CONTAINER;
  for (uint64_t i = 0; i < count; ++i) {
    int64_t mag = (int64_t)get_bits(buf, &bitpos, w);
    int neg = is_signed ? (int)get_bits(buf, &bitpos, 1) : 0;
    v[i] = neg ? -mag : mag;
  }
  return (int64_t)bitpos;
}

/* ------------------------------------------------------------------ */
/* The 3-phase decoder of one split                         */
/* ------------------------------------------------------------------ */

/* Entry: cursor0 = first word this task reads (the split's bitstream
 * offset, Z18), start_group = the split's max Symbol Group ID.  Lane j is
 * initialised with init_state[j] in the group init_group[j], immediately
 * before its first read.  Per group: refill pass in decreasing lane
 * ID, then every initialised lane decodes its symbol.  Phases:
 *  - Synchronization Phase: groups where some lane is not yet initialised;
 *    uninitialised lanes neither read nor decode (s_15, s_13 skipped).
 *  - Decoding Phase: all lanes initialised, down to the split boundary.
 *  - Cross-Boundary Phase: the same loop continues into the previous split's
 *    Synchronization Section and stops at its completion point commit_lo.
 * A symbol is written to out iff commit_lo <= i <= commit_hi (readings Z13,
 * Z20).  Every decoded i < N is flagged in produced (if non-NULL).  If the
 * task reaches the stream start it must end with every lane at L and the
 * cursor at -1 (P:124 stack property). */
int or_decode_from(const uint16_t *words, uint64_t B, const uint32_t f[256], uint32_t n,
                   uint32_t W, uint64_t N, int64_t cursor0, int64_t start_group,
                   const uint32_t *init_state, const int64_t *init_group,
                   uint64_t commit_lo, uint64_t commit_hi, uint8_t *out, uint8_t *produced,
                   int64_t *cursor_end) {
  (void)B;
  uint32_t F[256];
  cdf_of(f, F);
  uint8_t *lut = (uint8_t *)malloc(1u << n);
  if (!lut) return OR_E_NOMEM;
  lut_of(f, n, lut);
  uint64_t x[32] = {0};
  int inited[32] = {0};
  int64_t p = cursor0;
  int64_t lo_group = (int64_t)(commit_lo / W);
  int rc = OR_OK;
  for (int64_t g = start_group; g >= lo_group && rc == OR_OK; --g) {
    for (int32_t j = (int32_t)W - 1; j >= 0; --j) {
      if (!inited[j] && init_group[j] == g) {
        x[j] = init_state[j];
        inited[j] = 1;
      }
      if (inited[j] && or_renorm_decode(&x[j], words, &p) < 0) { rc = OR_E_UNDERFLOW; break; }
    }
    if (rc) break;
    for (uint32_t j = 0; j < W; ++j) {
      uint64_t i = (uint64_t)g * W + j;
      if (!inited[j] || i >= N) continue;
      uint32_t slot = (uint32_t)(x[j] & ((1u << n) - 1));
      uint32_t s = lut[slot];
      x[j] = (uint64_t)f[s] * (x[j] >> n) - F[s] + slot; /* Eq. 2 */
      if (produced) produced[i] = 1;
      if (i >= commit_lo && i <= commit_hi) out[i] = (uint8_t)s;
    }
  }
  if (rc == OR_OK && commit_lo == 0) {
    /* reached the stream start: outputs emitted before group 0, then the end state */
    for (int32_t j = (int32_t)W - 1; j >= 0 && rc == OR_OK; --j)
      if (inited[j] && or_renorm_decode(&x[j], words, &p) < 0) rc = OR_E_UNDERFLOW;
    if (rc == OR_OK) {
      if (p != -1) rc = OR_E_END;
      for (uint32_t j = 0; j < W; ++j)
        if (!inited[j] || x[j] != L_BOUND) rc = OR_E_END;
    }
  }
  if (cursor_end) *cursor_end = p;
  free(lut);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Recoil container                 */
/* ------------------------------------------------------------------ */

static void put_le(uint8_t *b, uint64_t v, int nbytes) {
  for (int k = 0; k < nbytes; ++k) b[k] = (uint8_t)(v >> (8 * k));
}
static uint64_t get_le(const uint8_t *b, int nbytes) {
  uint64_t v = 0;
  for (int k = 0; k < nbytes; ++k) v |= (uint64_t)b[k] << (8 * k);
  return v;
}

typedef struct {
  uint32_t n, W, M;
  uint64_t N, B, G;
  uint32_t kind;        /* 0: "RCL1" static 8-bit model; 1: "RCA1" adaptive model set, 16-bit symbols */
  uint32_t f[256];      /* kind 0 */
  uint32_t K;           /* kind 1: model set (see "Adaptive coding" below) */
  uint32_t *mbase, *mlen, *mf;
  uint32_t final_state[32];
  uint64_t *offset;     /* M-1 */
  uint64_t *maxg;       /* M-1 */
  uint32_t *state;      /* (M-1) x W */
  int64_t *gdiff;       /* (M-1) x W */
  const uint8_t *words; /* B little-endian u16 */
  uint64_t meta_bytes, model_bytes, header_bytes;
} or_box;

static void box_free(or_box *b) {
  free(b->mbase);
  free(b->mlen);
  free(b->mf);
  free(b->offset);
  free(b->maxg);
  free(b->state);
  free(b->gdiff);
}

/* Serialise. out == NULL: only *len is computed. */
static int box_write(const or_box *bx, const uint16_t *words, uint8_t *out, uint64_t *len) {
  uint32_t M = bx->M, W = bx->W;
  uint64_t P = M - 1;
  uint32_t count = 0;
  uint64_t msum = 0;
  for (int s = 0; s < 256; ++s) count += bx->f[s] ? 1 : 0;
  for (uint32_t k = 0; bx->kind == 1 && k < bx->K; ++k) msum += bx->mlen[k];
  /* sizes; adaptive model block: u32 K, K x (u32 base, u32 len), sum(len) x u32 f */
  uint64_t header = 28, finals = 4ull * W;
  uint64_t model = bx->kind == 1 ? 4 + 8ull * bx->K + 4 * msum : 2 + 5ull * count;
  int64_t *d_off = (int64_t *)calloc(P + 1, sizeof(int64_t));
  int64_t *d_g = (int64_t *)calloc(P + 1, sizeof(int64_t));
  if (!d_off || !d_g) { free(d_off); free(d_g); return OR_E_NOMEM; }
  uint64_t Eb = ceil_div(bx->B, M), Eg = ceil_div(bx->G, M); /* P:382, reading Z15 */
  for (uint64_t k = 1; k <= P; ++k) {
    d_off[k - 1] = (int64_t)bx->offset[k - 1] - (int64_t)(k * Eb); /* actual - expected (tab:metadata_split_point) */
    d_g[k - 1] = (int64_t)bx->maxg[k - 1] - (int64_t)(k * Eg);
    if (iabs64(d_off[k - 1]) >> 32 || iabs64(d_g[k - 1]) >> 32) { free(d_off); free(d_g); return OR_E_OVERFLOW; }
  }
  /* global block: two signed series with 5-bit width fields */
  uint32_t w1 = 1, w2 = 1;
  for (uint64_t k = 0; k < P; ++k) {
    if (bitlen((uint64_t)iabs64(d_off[k])) > w1) w1 = bitlen((uint64_t)iabs64(d_off[k]));
    if (bitlen((uint64_t)iabs64(d_g[k])) > w2) w2 = bitlen((uint64_t)iabs64(d_g[k]));
  }
  uint64_t gbits = 5 + P * (w1 + 1) + 5 + P * (w2 + 1);
  uint64_t gbytes = (gbits + 7) / 8;
  uint64_t pbytes = 0;
  for (uint64_t k = 0; k < P; ++k) {
    uint32_t w = 1;
    for (uint32_t j = 0; j < W; ++j)
      if (bitlen((uint64_t)bx->gdiff[k * W + j]) > w) w = bitlen((uint64_t)bx->gdiff[k * W + j]);
    if (w > 16) { free(d_off); free(d_g); return OR_E_OVERFLOW; } /* 4-bit width field */
    pbytes += 2ull * W + (4 + (uint64_t)W * w + 7) / 8;
  }
  uint64_t total = header + model + finals + gbytes + pbytes + 2 * bx->B;
  if (!out) {
    *len = total;
    free(d_off);
    free(d_g);
    return OR_OK;
  }
  if (*len < total) { *len = total; free(d_off); free(d_g); return OR_E_BUFFER; }
  memset(out, 0, total);
  uint8_t *q = out;
  memcpy(q, bx->kind == 1 ? "RCA1" : "RCL1", 4);
  q[4] = 1;  /* version */
  q[5] = bx->kind == 1 ? 16 : 8;  /* symbol bits (8 or 16) */
  q[6] = (uint8_t)bx->n;
  q[7] = (uint8_t)W;
  put_le(q + 8, M, 4);
  put_le(q + 12, bx->N, 8);
  put_le(q + 20, bx->B, 8); /* M, B, N stored as-is */
  q += header;
  if (bx->kind == 1) {
    put_le(q, bx->K, 4);
    q += 4;
    for (uint32_t k = 0; k < bx->K; ++k, q += 8) {
      put_le(q, bx->mbase[k], 4);
      put_le(q + 4, bx->mlen[k], 4);
    }
    for (uint64_t e = 0; e < msum; ++e, q += 4) put_le(q, bx->mf[e], 4);
  } else {
    put_le(q, count, 2);
    q += 2;
    for (int s = 0; s < 256; ++s)
      if (bx->f[s]) {
        q[0] = (uint8_t)s;
        put_le(q + 1, bx->f[s], 4);
        q += 5;
      }
  }
  for (uint32_t j = 0; j < W; ++j, q += 4) put_le(q, bx->final_state[j], 4);
  uint64_t bp = or_pack_series(d_off, P, 1, 5, q, 0);
  bp = or_pack_series(d_g, P, 1, 5, q, bp);
  q += gbytes;
  for (uint64_t k = 0; k < P; ++k) {
    for (uint32_t j = 0; j < W; ++j, q += 2) put_le(q, bx->state[k * W + j], 2); /* states as-is */
    uint64_t bits = or_pack_series(bx->gdiff + k * W, W, 0, 4, q, 0);
    q += (bits + 7) / 8;
  }
  for (uint64_t w = 0; w < bx->B; ++w, q += 2) put_le(q, words[w], 2);
  *len = total;
  free(d_off);
  free(d_g);
  return OR_OK;
}

static int box_read(const uint8_t *c, uint64_t len, or_box *bx) {
  memset(bx, 0, sizeof(*bx));
  if (len < 28) return OR_E_CONTAINER;
  if (memcmp(c, "RCL1", 4) == 0 && c[4] == 1 && c[5] == 8) bx->kind = 0;
  else if (memcmp(c, "RCA1", 4) == 0 && c[4] == 1 && c[5] == 16) bx->kind = 1;
  else return OR_E_CONTAINER;
  bx->n = c[6];
  bx->W = c[7];
  bx->M = (uint32_t)get_le(c + 8, 4);
  bx->N = get_le(c + 12, 8);
  bx->B = get_le(c + 20, 8);
  if (bx->n < 1 || bx->n > 16 || bx->W < 1 || bx->W > 32 || bx->M < 1) return OR_E_CONTAINER;
  bx->G = ceil_div(bx->N, bx->W);
  uint64_t pos = 28;
  if (bx->kind == 1) {
    if (pos + 4 > len) return OR_E_CONTAINER;
    bx->K = (uint32_t)get_le(c + pos, 4);
    pos += 4;
    if (bx->K < 1 || bx->K > 256 || pos + 8ull * bx->K > len) return OR_E_CONTAINER;
    bx->mbase = (uint32_t *)calloc(bx->K, 4);
    bx->mlen = (uint32_t *)calloc(bx->K, 4);
    if (!bx->mbase || !bx->mlen) { box_free(bx); return OR_E_NOMEM; }
    uint64_t msum = 0;
    for (uint32_t k = 0; k < bx->K; ++k, pos += 8) {
      bx->mbase[k] = (uint32_t)get_le(c + pos, 4);
      bx->mlen[k] = (uint32_t)get_le(c + pos + 4, 4);
      if (bx->mlen[k] < 1 || (uint64_t)bx->mbase[k] + bx->mlen[k] > 65536) { box_free(bx); return OR_E_CONTAINER; }
      msum += bx->mlen[k];
    }
    if (pos + 4 * msum > len) { box_free(bx); return OR_E_CONTAINER; }
    bx->mf = (uint32_t *)calloc(msum + 1, 4);
    if (!bx->mf) { box_free(bx); return OR_E_NOMEM; }
    for (uint64_t e = 0; e < msum; ++e, pos += 4) bx->mf[e] = (uint32_t)get_le(c + pos, 4);
    uint64_t e0 = 0;
    for (uint32_t k = 0; k < bx->K; ++k) { /* every model sums to 2^n */
      uint64_t fsum = 0;
      for (uint32_t j = 0; j < bx->mlen[k]; ++j) fsum += bx->mf[e0 + j];
      e0 += bx->mlen[k];
      if (fsum != (1ull << bx->n)) { box_free(bx); return OR_E_CONTAINER; }
    }
    bx->model_bytes = 4 + 8ull * bx->K + 4 * msum;
  } else {
    if (pos + 2 > len) return OR_E_CONTAINER;
    uint32_t count = (uint32_t)get_le(c + pos, 2);
    pos += 2;
    if (pos + 5ull * count > len) return OR_E_CONTAINER;
    uint64_t fsum = 0;
    for (uint32_t k = 0; k < count; ++k, pos += 5) {
      bx->f[c[pos]] = (uint32_t)get_le(c + pos + 1, 4);
      fsum += bx->f[c[pos]];
    }
    if (fsum != (1ull << bx->n)) return OR_E_CONTAINER;
    bx->model_bytes = 2 + 5ull * count;
  }
  bx->header_bytes = 28;
  if (pos + 4ull * bx->W > len) { box_free(bx); return OR_E_CONTAINER; }
  for (uint32_t j = 0; j < bx->W; ++j, pos += 4) bx->final_state[j] = (uint32_t)get_le(c + pos, 4);
  uint64_t meta_start = pos;
  uint64_t P = bx->M - 1, W = bx->W;
  bx->offset = (uint64_t *)calloc(P + 1, 8);
  bx->maxg = (uint64_t *)calloc(P + 1, 8);
  bx->state = (uint32_t *)calloc(P * W + 1, 4);
  bx->gdiff = (int64_t *)calloc(P * W + 1, 8);
  int64_t *d = (int64_t *)calloc(P + 1, 8);
  if (!bx->offset || !bx->maxg || !bx->state || !bx->gdiff || !d) { free(d); box_free(bx); return OR_E_NOMEM; }
  uint64_t Eb = ceil_div(bx->B, bx->M), Eg = ceil_div(bx->G, bx->M);
  int64_t bp = or_unpack_series(c + pos, 8 * (len - pos), 0, P, 1, 5, d);
  if (bp < 0) { free(d); box_free(bx); return OR_E_CONTAINER; }
  for (uint64_t k = 1; k <= P; ++k) bx->offset[k - 1] = (uint64_t)((int64_t)(k * Eb) + d[k - 1]);
  bp = or_unpack_series(c + pos, 8 * (len - pos), (uint64_t)bp, P, 1, 5, d);
  if (bp < 0) { free(d); box_free(bx); return OR_E_CONTAINER; }
  for (uint64_t k = 1; k <= P; ++k) bx->maxg[k - 1] = (uint64_t)((int64_t)(k * Eg) + d[k - 1]);
  free(d);
  pos += ((uint64_t)bp + 7) / 8;
  for (uint64_t k = 0; k < P; ++k) {
    if (pos + 2 * W > len) { box_free(bx); return OR_E_CONTAINER; }
    for (uint32_t j = 0; j < W; ++j, pos += 2) bx->state[k * W + j] = (uint32_t)get_le(c + pos, 2);
    int64_t b2 = or_unpack_series(c + pos, 8 * (len - pos), 0, W, 0, 4, bx->gdiff + k * W);
    if (b2 < 0) { box_free(bx); return OR_E_CONTAINER; }
    pos += ((uint64_t)b2 + 7) / 8;
  }
  bx->meta_bytes = pos - meta_start;
  if (pos + 2 * bx->B != len) { box_free(bx); return OR_E_CONTAINER; }
  bx->words = c + pos;
  /* consistency (S:366 InconsistentMetadata): offsets inside the stream,
   * group IDs inside the symbol range, sync starts strictly increasing */
  int64_t prev_ss = -1;
  for (uint64_t k = 0; k < P; ++k) {
    if (bx->offset[k] >= bx->B || bx->maxg[k] >= bx->G) { box_free(bx); return OR_E_CONTAINER; }
    int64_t ss = -1;
    for (uint32_t j = 0; j < W; ++j) {
      if ((uint64_t)bx->gdiff[k * W + j] > bx->maxg[k]) { box_free(bx); return OR_E_CONTAINER; }
      int64_t idx = (int64_t)(bx->maxg[k] - (uint64_t)bx->gdiff[k * W + j]) * (int64_t)W + j;
      if ((uint64_t)idx >= bx->N) { box_free(bx); return OR_E_CONTAINER; }
      if (ss < 0 || idx < ss) ss = idx;
    }
    if (ss <= prev_ss) { box_free(bx); return OR_E_CONTAINER; }
    prev_ss = ss;
  }
  return OR_OK;
}

static uint16_t *box_words(const or_box *bx) {
  uint16_t *w = (uint16_t *)malloc(2 * bx->B + 2);
  if (!w) return NULL;
  for (uint64_t i = 0; i < bx->B; ++i) w[i] = (uint16_t)get_le(bx->words + 2 * i, 2);
  return w;
}

/* sync_start and boundary index of point k (0-based array index) */
static void point_span(const or_box *bx, uint64_t k, int64_t *ss, int64_t *bidx) {
  int64_t mn = -1, mx = -1;
  for (uint32_t j = 0; j < bx->W; ++j) {
    int64_t idx = (int64_t)(bx->maxg[k] - (uint64_t)bx->gdiff[k * bx->W + j]) * (int64_t)bx->W + j;
    if (mn < 0 || idx < mn) mn = idx;
    if (idx > mx) mx = idx;
  }
  *ss = mn;
  *bidx = mx;
}

int or_recoil_encode(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                     uint32_t W, uint32_t M, uint8_t *out, uint64_t *len) {
  return or_recoil_encode_ex(sym, N, f, n, W, M, 0, out, len);
}

int or_recoil_encode_ex(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                        uint32_t W, uint32_t M, uint32_t split_flags, uint8_t *out, uint64_t *len) {
  if (M < 1 || W < 1 || W > 32 || n < 1 || n > 16) return OR_E_ARG;
  uint64_t fs = 0;
  for (int s = 0; s < 256; ++s) fs += f[s];
  if (fs != (1ull << n)) return OR_E_MODEL;
  uint16_t *words = (uint16_t *)malloc(2 * N + 2);
  or_event *ev = (or_event *)malloc(sizeof(or_event) * (N + 1));
  if (!words || !ev) { free(words); free(ev); return OR_E_NOMEM; }
  or_box bx;
  memset(&bx, 0, sizeof(bx));
  bx.n = n;
  bx.W = W;
  bx.N = N;
  bx.G = ceil_div(N, W);
  memcpy(bx.f, f, sizeof(bx.f));
  int64_t B = or_interleaved_encode(sym, N, f, n, W, words, bx.final_state, ev, NULL);
  if (B < 0) { free(words); free(ev); return (int)B; }
  bx.B = (uint64_t)B;
  uint64_t *chosen = (uint64_t *)malloc(8ull * M);
  int64_t P = or_choose_splits_ex(ev, bx.B, N, W, M, split_flags, chosen);
  bx.M = (uint32_t)P + 1;
  bx.offset = (uint64_t *)calloc((uint64_t)P + 1, 8);
  bx.maxg = (uint64_t *)calloc((uint64_t)P + 1, 8);
  bx.state = (uint32_t *)calloc((uint64_t)P * W + 1, 4);
  bx.gdiff = (int64_t *)calloc((uint64_t)P * W + 1, 8);
  for (int64_t k = 0; k < P; ++k) {
    int64_t ai[32], ss;
    uint32_t st[32];
    or_backward_scan(ev, chosen[k], W, st, ai, &ss);
    bx.offset[k] = chosen[k];                            /* bitstream offset of the split (Z18) */
    bx.maxg[k] = (uint64_t)ev[chosen[k]].idx / W;        /* max Symbol Group ID = anchor */
    for (uint32_t j = 0; j < W; ++j) {
      bx.state[k * W + j] = st[j];                       /* < L by the Lemma: 16 bits */
      bx.gdiff[k * W + j] = (int64_t)bx.maxg[k] - ai[j] / (int64_t)W; /* |group - anchor| */
    }
  }
  int rc = box_write(&bx, words, out, len);
  box_free(&bx);
  free(chosen);
  free(words);
  free(ev);
  return rc;
}

/* Combine (readings Z11, Z12): keep the points at 1-based
 * positions k, 2k, ... with k = ceil(M / target); target >= M: unchanged. */
int or_combine(const uint8_t *in, uint64_t in_len, uint32_t target, uint8_t *out, uint64_t *len) {
  if (target < 1) return OR_E_ARG;
  or_box bx;
  int rc = box_read(in, in_len, &bx);
  if (rc) return rc;
  if (target >= bx.M) {
    box_free(&bx);
    if (!out) { *len = in_len; return OR_OK; }
    if (*len < in_len) { *len = in_len; return OR_E_BUFFER; }
    memcpy(out, in, in_len);
    *len = in_len;
    return OR_OK;
  }
  uint64_t k = ceil_div(bx.M, target), P = bx.M - 1, kept = 0;
  for (uint64_t pos = k; pos <= P; pos += k) { /* 1-based position pos -> array index pos-1 */
    bx.offset[kept] = bx.offset[pos - 1];
    bx.maxg[kept] = bx.maxg[pos - 1];
    for (uint32_t j = 0; j < bx.W; ++j) {
      bx.state[kept * bx.W + j] = bx.state[(pos - 1) * bx.W + j];
      bx.gdiff[kept * bx.W + j] = bx.gdiff[(pos - 1) * bx.W + j];
    }
    kept++;
  }
  bx.M = (uint32_t)kept + 1;
  uint16_t *w = box_words(&bx);
  rc = box_write(&bx, w, out, len);
  free(w);
  box_free(&bx);
  return rc;
}

int or_container_info(const uint8_t *c, uint64_t len, uint64_t info[8]) {
  or_box bx;
  int rc = box_read(c, len, &bx);
  if (rc) return rc;
  info[0] = bx.N;
  info[1] = bx.B;
  info[2] = bx.M;
  info[3] = bx.n;
  info[4] = bx.W;
  info[5] = bx.header_bytes + bx.model_bytes;
  info[6] = bx.meta_bytes; /* final states + global series + split records */
  info[7] = 2 * bx.B;
  box_free(&bx);
  return OR_OK;
}

int or_container_points(const uint8_t *c, uint64_t len, uint64_t *offset, uint64_t *maxg,
                        uint64_t *sync_start, uint64_t *bidx) {
  or_box bx;
  int rc = box_read(c, len, &bx);
  if (rc) return rc;
  for (uint64_t k = 0; k + 1 < bx.M; ++k) {
    int64_t ss, bi;
    point_span(&bx, k, &ss, &bi);
    offset[k] = bx.offset[k];
    maxg[k] = bx.maxg[k];
    sync_start[k] = (uint64_t)ss;
    bidx[k] = (uint64_t)bi;
  }
  box_free(&bx);
  return OR_OK;
}

/* Task t of M: t < M-1 enters at split point t+1 (1-based); task M-1 enters
 * from the explicitly transmitted final states.  Task t commits
 * [sync_start(point t), sync_start(point t+1) - 1] (Z13). */
static int box_task(const or_box *bx, const uint16_t *w, uint32_t t, uint8_t *out, uint64_t *lo_out,
                    uint64_t *hi_out) {
  if (bx->kind != 0) return OR_E_ARG; /* adaptive containers: or_ad_recoil_decode* (needs the model ids) */
  uint32_t W = bx->W;
  uint32_t st[32];
  int64_t ig[32];
  int64_t cursor0, start_group, ss, bi;
  uint64_t lo = 0, hi;
  if (t > 0) {
    point_span(bx, t - 1, &ss, &bi);
    lo = (uint64_t)ss;
  }
  if (t + 1 < bx->M) {
    point_span(bx, t, &ss, &bi);
    hi = (uint64_t)ss - 1;
    cursor0 = (int64_t)bx->offset[t];
    start_group = (int64_t)bx->maxg[t];
    for (uint32_t j = 0; j < W; ++j) {
      st[j] = bx->state[t * W + j];
      ig[j] = (int64_t)bx->maxg[t] - bx->gdiff[t * W + j];
    }
  } else {
    hi = bx->N - 1;
    cursor0 = (int64_t)bx->B - 1;
    start_group = (int64_t)bx->G - 1;
    for (uint32_t j = 0; j < W; ++j) {
      st[j] = bx->final_state[j];
      ig[j] = start_group;
    }
  }
  if (lo_out) *lo_out = lo;
  if (hi_out) *hi_out = hi;
  return or_decode_from(w, bx->B, bx->f, bx->n, W, bx->N, cursor0, start_group, st, ig, lo, hi,
                        out, NULL, NULL);
}

int or_recoil_decode(const uint8_t *c, uint64_t len, uint8_t *out) {
  or_box bx;
  int rc = box_read(c, len, &bx);
  if (rc) return rc;
  if (bx.N == 0) { box_free(&bx); return OR_OK; }
  uint16_t *w = box_words(&bx);
  for (uint32_t t = 0; t < bx.M && rc == OR_OK; ++t) rc = box_task(&bx, w, t, out, NULL, NULL);
  free(w);
  box_free(&bx);
  return rc;
}

/* Decode a list of tasks with one parse of the container (bounded samples for
 * the CPU baseline).  *n_symbols = committed symbols decoded. */
int or_recoil_decode_tasks(const uint8_t *c, uint64_t len, const uint32_t *tasks, uint32_t n_tasks,
                           uint8_t *out, uint64_t *n_symbols) {
  or_box bx;
  int rc = box_read(c, len, &bx);
  if (rc) return rc;
  uint16_t *w = box_words(&bx);
  uint64_t total = 0;
  for (uint32_t k = 0; k < n_tasks && rc == OR_OK; ++k) {
    uint64_t lo = 0, hi = 0;
    if (tasks[k] >= bx.M || bx.N == 0) { rc = OR_E_ARG; break; }
    rc = box_task(&bx, w, tasks[k], out, &lo, &hi);
    total += hi - lo + 1;
  }
  if (n_symbols) *n_symbols = total;
  free(w);
  box_free(&bx);
  return rc;
}

/* A container parsed once (box_read + box_words) for repeated task decodes:
 * the reference arm times or_opened_decode_tasks only, with the parse outside
 * its timed region. */
struct or_opened {
  or_box bx;
  uint16_t *w;
};

int or_open(const uint8_t *c, uint64_t len, or_opened **out) {
  or_opened *h = (or_opened *)calloc(1, sizeof(or_opened));
  if (!h) return OR_E_ARG;
  int rc = box_read(c, len, &h->bx);
  if (rc) { free(h); return rc; }
  h->w = box_words(&h->bx);
  *out = h;
  return OR_OK;
}

int or_opened_decode_tasks(or_opened *h, const uint32_t *tasks, uint32_t n_tasks, uint8_t *out,
                           uint64_t *n_symbols) {
  int rc = OR_OK;
  uint64_t total = 0;
  for (uint32_t k = 0; k < n_tasks && rc == OR_OK; ++k) {
    uint64_t lo = 0, hi = 0;
    if (tasks[k] >= h->bx.M || h->bx.N == 0) { rc = OR_E_ARG; break; }
    rc = box_task(&h->bx, h->w, tasks[k], out, &lo, &hi);
    total += hi - lo + 1;
  }
  if (n_symbols) *n_symbols = total;
  return rc;
}

void or_close(or_opened *h) {
  if (!h) return;
  free(h->w);
  box_free(&h->bx);
  free(h);
}

int or_recoil_decode_task(const uint8_t *c, uint64_t len, uint32_t task, uint8_t *out,
                          uint64_t *lo, uint64_t *hi) {
  or_box bx;
  int rc = box_read(c, len, &bx);
  if (rc) return rc;
  if (task >= bx.M || bx.N == 0) { box_free(&bx); return OR_E_ARG; }
  uint16_t *w = box_words(&bx);
  rc = box_task(&bx, w, task, out, lo, hi);
  free(w);
  box_free(&bx);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Conventional partitioned codec (partition bounds Z25')    */
/* ------------------------------------------------------------------ */

/* Partition p covers groups [floor(pG/P), floor((p+1)G/P)), i.e. symbols
 * [W floor(pG/P), min(N, W floor((p+1)G/P))); each is encoded by its own
 * W-way interleaved codec; sub-streams concatenated plus an offset table
 * (P:192).  Layout: "RCV1", version, symbol bits, n, W, u32 P, u64 N, u64 B,
 * model block, P x u32 word counts, P x W x u32 final states, words. */
int or_partitioned_encode(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                          uint32_t W, uint32_t P, uint8_t *out, uint64_t *len) {
  if (P < 1 || W < 1 || W > 32) return OR_E_ARG;
  uint64_t G = ceil_div(N, W);
  uint16_t *words = (uint16_t *)malloc(2 * N + 2);
  uint32_t *cnt = (uint32_t *)calloc(P, 4);
  uint32_t *fin = (uint32_t *)calloc((uint64_t)P * W, 4);
  if (!words || !cnt || !fin) { free(words); free(cnt); free(fin); return OR_E_NOMEM; }
  uint64_t B = 0;
  for (uint64_t p = 0; p < P; ++p) {
    uint64_t lo = W * (p * G / P), hi = W * ((p + 1) * G / P);
    if (hi > N) hi = N;
    if (lo > hi) lo = hi;
    int64_t b = or_interleaved_encode(sym + lo, hi - lo, f, n, W, words + B, fin + p * W, NULL, NULL);
    if (b < 0 || (uint64_t)b >> 32) { free(words); free(cnt); free(fin); return b < 0 ? (int)b : OR_E_OVERFLOW; }
    cnt[p] = (uint32_t)b;
    B += (uint64_t)b;
  }
  uint32_t count = 0;
  for (int s = 0; s < 256; ++s) count += f[s] ? 1 : 0;
  uint64_t total = 28 + 2 + 5ull * count + 4ull * P + 4ull * P * W + 2 * B;
  if (!out) { *len = total; free(words); free(cnt); free(fin); return OR_OK; }
  if (*len < total) { *len = total; free(words); free(cnt); free(fin); return OR_E_BUFFER; }
  uint8_t *q = out;
  memcpy(q, "RCV1", 4);
  q[4] = 1;
  q[5] = 8;
  q[6] = (uint8_t)n;
  q[7] = (uint8_t)W;
  put_le(q + 8, P, 4);
  put_le(q + 12, N, 8);
  put_le(q + 20, B, 8);
  q += 28;
  put_le(q, count, 2);
  q += 2;
  for (int s = 0; s < 256; ++s)
    if (f[s]) { q[0] = (uint8_t)s; put_le(q + 1, f[s], 4); q += 5; }
  for (uint64_t p = 0; p < P; ++p, q += 4) put_le(q, cnt[p], 4);
  for (uint64_t k = 0; k < (uint64_t)P * W; ++k, q += 4) put_le(q, fin[k], 4);
  for (uint64_t w = 0; w < B; ++w, q += 2) put_le(q, words[w], 2);
  *len = total;
  free(words);
  free(cnt);
  free(fin);
  return OR_OK;
}

int or_partitioned_decode(const uint8_t *c, uint64_t len, uint8_t *out) {
  if (len < 30 || memcmp(c, "RCV1", 4) != 0 || c[4] != 1 || c[5] != 8) return OR_E_CONTAINER;
  uint32_t n = c[6], W = c[7], P = (uint32_t)get_le(c + 8, 4);
  uint64_t N = get_le(c + 12, 8), B = get_le(c + 20, 8), G = ceil_div(N, W);
  uint64_t pos = 28;
  uint32_t count = (uint32_t)get_le(c + pos, 2), f[256] = {0};
  pos += 2;
  for (uint32_t k = 0; k < count; ++k, pos += 5) f[c[pos]] = (uint32_t)get_le(c + pos + 1, 4);
  uint64_t cnt_pos = pos, fin_pos = pos + 4ull * P, w_pos = fin_pos + 4ull * P * W;
  if (w_pos + 2 * B != len) return OR_E_CONTAINER;
  uint16_t *words = (uint16_t *)malloc(2 * B + 2);
  for (uint64_t i = 0; i < B; ++i) words[i] = (uint16_t)get_le(c + w_pos + 2 * i, 2);
  uint64_t base = 0;
  int rc = OR_OK;
  for (uint64_t p = 0; p < P && rc == OR_OK; ++p) {
    uint64_t lo = W * (p * G / P), hi = W * ((p + 1) * G / P);
    if (hi > N) hi = N;
    if (lo > hi) lo = hi;
    uint32_t fin[32];
    for (uint32_t j = 0; j < W; ++j) fin[j] = (uint32_t)get_le(c + fin_pos + 4 * (p * W + j), 4);
    uint64_t b = get_le(c + cnt_pos + 4 * p, 4);
    rc = or_interleaved_decode(words + base, b, fin, hi - lo, f, n, W, out + lo);
    base += b;
  }
  free(words);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Adaptive coding: index-keyed models, 16-bit symbols                 */
/* (P:227 item (3); P:411 sizeof(s_i) = 8 or 16 bits)           */
/* ------------------------------------------------------------------ */

/* A model set has K models.  Model k covers the symbol values base[k] ..
 * base[k] + len[k] - 1 with frequencies mf[off_k + j] (sum 2^n; 0 = not in
 * the model), off_k = len[0] + ... + len[k-1].  Symbol i is coded with
 * model mid[i] -- the "symbol index as a key" of P:227 -- and Eq. 1-4 are
 * used unchanged with f, F of that model.  The renormalisation before
 * symbol i (Eq. 3) uses f of model mid[i], so the split metadata (events,
 * backward scan, H, series) is exactly that of the static codec. */
typedef struct {
  uint32_t K;
  const uint32_t *base, *len, *mf;
  uint64_t *off;  /* K + 1 */
  uint32_t *F;    /* per entry: F_k(j) = sum of mf[off_k .. off_k + j - 1] */
} or_ad_models;

static int ad_models_init(or_ad_models *m, uint32_t K, const uint32_t *base, const uint32_t *len,
                          const uint32_t *mf, uint32_t n) {
  memset(m, 0, sizeof(*m));
  if (K < 1 || K > 256) return OR_E_ARG;
  m->K = K;
  m->base = base;
  m->len = len;
  m->mf = mf;
  m->off = (uint64_t *)calloc(K + 1, 8);
  if (!m->off) return OR_E_NOMEM;
  for (uint32_t k = 0; k < K; ++k) {
    if (len[k] < 1 || (uint64_t)base[k] + len[k] > 65536) { free(m->off); return OR_E_MODEL; }
    m->off[k + 1] = m->off[k] + len[k];
  }
  m->F = (uint32_t *)calloc(m->off[K] + 1, 4);
  if (!m->F) { free(m->off); return OR_E_NOMEM; }
  for (uint32_t k = 0; k < K; ++k) {
    uint64_t acc = 0;
    for (uint32_t j = 0; j < len[k]; ++j) {
      m->F[m->off[k] + j] = (uint32_t)acc;
      acc += mf[m->off[k] + j];
    }
    if (acc != (1ull << n)) { free(m->off); free(m->F); return OR_E_MODEL; }
  }
  return OR_OK;
}

static void ad_models_free(or_ad_models *m) {
  free(m->off);
  free(m->F);
}

/* f and F of symbol value v under model k; 0 if v is not in the model */
static int ad_fF(const or_ad_models *m, uint32_t k, uint32_t v, uint32_t *f, uint32_t *F) {
  if (k >= m->K || v < m->base[k] || v - m->base[k] >= m->len[k]) return 0;
  uint64_t e = m->off[k] + (v - m->base[k]);
  *f = m->mf[e];
  *F = m->F[e];
  return *f > 0;
}

/* Eq. 2 under model k: the value v with F_k(v) <= x mod 2^n < F_k(v) + f_k(v),
 * by a plain scan of the model's entries. */
static int ad_decode_step(const or_ad_models *m, uint32_t k, uint32_t n, uint64_t *x, uint32_t *v) {
  uint32_t slot = (uint32_t)(*x & ((1u << n) - 1));
  for (uint32_t j = 0; j < m->len[k]; ++j) {
    uint64_t e = m->off[k] + j;
    if (m->mf[e] && m->F[e] <= slot && slot < m->F[e] + m->mf[e]) {
      *x = (uint64_t)m->mf[e] * (*x >> n) - m->F[e] + slot;
      *v = m->base[k] + j;
      return OR_OK;
    }
  }
  return OR_E_MODEL;
}

/* The interleaved encoder of P:166-170 (see or_interleaved_encode) with the
 * model of every symbol taken from mid[i]. */
int64_t or_ad_interleaved_encode(const uint16_t *sym, uint64_t N, const uint8_t *mid, uint32_t K,
                                 const uint32_t *base, const uint32_t *len, const uint32_t *mf, uint32_t n,
                                 uint32_t W, uint16_t *words, uint32_t *final_states, or_event *events) {
  if (W < 1 || W > 32 || n < 1 || n > 16) return OR_E_ARG;
  or_ad_models m;
  int rc = ad_models_init(&m, K, base, len, mf, n);
  if (rc) return rc;
  uint32_t f, F;
  for (uint64_t i = 0; i < N; ++i)
    if (!ad_fF(&m, mid[i], sym[i], &f, &F)) { ad_models_free(&m); return OR_E_MODEL; }
  uint64_t x[32];
  for (uint32_t j = 0; j < W; ++j) x[j] = L_BOUND;
  uint64_t G = (N + W - 1) / W, p = 0;
  for (uint64_t g = 0; g < G; ++g) {
    for (uint32_t j = 0; j < W; ++j) { /* renormalisation outputs, increasing lane ID (Z4) */
      uint64_t i = g * W + j;
      if (i >= N) continue;
      ad_fF(&m, mid[i], sym[i], &f, &F);
      uint64_t p_before = p;
      or_renorm_encode(&x[j], f, n, words, &p);
      for (uint64_t q = p_before; q < p; ++q)
        if (events) {
          events[q].idx = (int64_t)i - (int64_t)W;
          events[q].lane = j;
          events[q].state = (uint32_t)x[j];
        }
    }
    for (uint32_t j = 0; j < W; ++j) { /* Eq. 1 */
      uint64_t i = g * W + j;
      if (i >= N) continue;
      ad_fF(&m, mid[i], sym[i], &f, &F);
      x[j] = or_encode_step(x[j], f, F, n);
      if (x[j] >> 32) { ad_models_free(&m); return OR_E_OVERFLOW; }
    }
  }
  for (uint32_t j = 0; j < W; ++j) final_states[j] = (uint32_t)x[j];
  ad_models_free(&m);
  return (int64_t)p;
}

/* Serial decoder of the adaptive stream (see or_interleaved_decode). */
int or_ad_interleaved_decode(const uint16_t *words, uint64_t B, const uint32_t *final_states, uint64_t N,
                             const uint8_t *mid, uint32_t K, const uint32_t *base, const uint32_t *len,
                             const uint32_t *mf, uint32_t n, uint32_t W, uint16_t *out) {
  if (W < 1 || W > 32) return OR_E_ARG;
  or_ad_models m;
  int rc = ad_models_init(&m, K, base, len, mf, n);
  if (rc) return rc;
  uint64_t x[32];
  for (uint32_t j = 0; j < W; ++j) x[j] = final_states[j];
  int64_t p = (int64_t)B - 1;
  int64_t G = (int64_t)((N + W - 1) / W);
  for (int64_t g = G - 1; g >= -1 && rc == OR_OK; --g) {
    for (int32_t j = (int32_t)W - 1; j >= 0; --j)
      if (or_renorm_decode(&x[j], words, &p) < 0) { rc = OR_E_UNDERFLOW; break; }
    if (g < 0 || rc) break;
    for (uint32_t j = 0; j < W && rc == OR_OK; ++j) {
      uint64_t i = (uint64_t)g * W + j;
      if (i >= N) continue;
      uint32_t v;
      if (mid[i] >= K) { rc = OR_E_MODEL; break; }
      rc = ad_decode_step(&m, mid[i], n, &x[j], &v);
      out[i] = (uint16_t)v;
    }
  }
  ad_models_free(&m);
  if (rc) return rc;
  if (p != -1) return OR_E_END;
  for (uint32_t j = 0; j < W; ++j)
    if (x[j] != L_BOUND) return OR_E_END;
  return OR_OK;
}

/* The 3-phase task decoder of P:303-315 (see or_decode_from) for the
 * adaptive codec. */
int or_ad_decode_from(const uint16_t *words, const uint8_t *mid, uint32_t K, const uint32_t *base,
                      const uint32_t *len, const uint32_t *mf, uint32_t n, uint32_t W, uint64_t N,
                      int64_t cursor0, int64_t start_group, const uint32_t *init_state,
                      const int64_t *init_group, uint64_t commit_lo, uint64_t commit_hi, uint16_t *out) {
  or_ad_models m;
  int rc = ad_models_init(&m, K, base, len, mf, n);
  if (rc) return rc;
  uint64_t x[32] = {0};
  int inited[32] = {0};
  int64_t p = cursor0;
  int64_t lo_group = (int64_t)(commit_lo / W);
  for (int64_t g = start_group; g >= lo_group && rc == OR_OK; --g) {
    for (int32_t j = (int32_t)W - 1; j >= 0; --j) {
      if (!inited[j] && init_group[j] == g) {
        x[j] = init_state[j];
        inited[j] = 1;
      }
      if (inited[j] && or_renorm_decode(&x[j], words, &p) < 0) { rc = OR_E_UNDERFLOW; break; }
    }
    for (uint32_t j = 0; j < W && rc == OR_OK; ++j) {
      uint64_t i = (uint64_t)g * W + j;
      if (!inited[j] || i >= N) continue;
      uint32_t v;
      if (mid[i] >= K) { rc = OR_E_MODEL; break; }
      rc = ad_decode_step(&m, mid[i], n, &x[j], &v);
      if (rc == OR_OK && i >= commit_lo && i <= commit_hi) out[i] = (uint16_t)v;
    }
  }
  if (rc == OR_OK && commit_lo == 0) {
    for (int32_t j = (int32_t)W - 1; j >= 0 && rc == OR_OK; --j)
      if (inited[j] && or_renorm_decode(&x[j], words, &p) < 0) rc = OR_E_UNDERFLOW;
    if (rc == OR_OK) {
      if (p != -1) rc = OR_E_END;
      for (uint32_t j = 0; j < W; ++j)
        if (!inited[j] || x[j] != L_BOUND) rc = OR_E_END;
    }
  }
  ad_models_free(&m);
  return rc;
}

/* Recoil container of an adaptive stream ("RCA1": 16-bit symbols, the model
 * set in the model block; everything else as "RCL1"). */
int or_ad_recoil_encode(const uint16_t *sym, uint64_t N, const uint8_t *mid, uint32_t K, const uint32_t *base,
                        const uint32_t *len, const uint32_t *mf, uint32_t n, uint32_t W, uint32_t M,
                        uint8_t *out, uint64_t *outlen) {
  if (M < 1 || W < 1 || W > 32 || n < 1 || n > 16 || K < 1 || K > 256) return OR_E_ARG;
  uint16_t *words = (uint16_t *)malloc(2 * N + 2);
  or_event *ev = (or_event *)malloc(sizeof(or_event) * (N + 1));
  uint64_t *chosen = (uint64_t *)malloc(8ull * M);
  if (!words || !ev || !chosen) { free(words); free(ev); free(chosen); return OR_E_NOMEM; }
  or_box bx;
  memset(&bx, 0, sizeof(bx));
  bx.kind = 1;
  bx.n = n;
  bx.W = W;
  bx.N = N;
  bx.G = ceil_div(N, W);
  bx.K = K;
  uint64_t msum = 0;
  for (uint32_t k = 0; k < K; ++k) msum += len[k];
  bx.mbase = (uint32_t *)malloc(4ull * K);
  bx.mlen = (uint32_t *)malloc(4ull * K);
  bx.mf = (uint32_t *)malloc(4 * msum + 4);
  int64_t B = (!bx.mbase || !bx.mlen || !bx.mf) ? OR_E_NOMEM
              : or_ad_interleaved_encode(sym, N, mid, K, base, len, mf, n, W, words, bx.final_state, ev);
  if (B < 0) { box_free(&bx); free(words); free(ev); free(chosen); return (int)B; }
  memcpy(bx.mbase, base, 4ull * K);
  memcpy(bx.mlen, len, 4ull * K);
  memcpy(bx.mf, mf, 4 * msum);
  bx.B = (uint64_t)B;
  int64_t P = or_choose_splits_ex(ev, bx.B, N, W, M, 0, chosen);
  bx.M = (uint32_t)P + 1;
  bx.offset = (uint64_t *)calloc((uint64_t)P + 1, 8);
  bx.maxg = (uint64_t *)calloc((uint64_t)P + 1, 8);
  bx.state = (uint32_t *)calloc((uint64_t)P * W + 1, 4);
  bx.gdiff = (int64_t *)calloc((uint64_t)P * W + 1, 8);
  for (int64_t k = 0; k < P; ++k) { /* same split records as or_recoil_encode */
    int64_t ai[32], ss;
    uint32_t st[32];
    or_backward_scan(ev, chosen[k], W, st, ai, &ss);
    bx.offset[k] = chosen[k];
    bx.maxg[k] = (uint64_t)ev[chosen[k]].idx / W;
    for (uint32_t j = 0; j < W; ++j) {
      bx.state[k * W + j] = st[j];
      bx.gdiff[k * W + j] = (int64_t)bx.maxg[k] - ai[j] / (int64_t)W;
    }
  }
  int rc = box_write(&bx, words, out, outlen);
  box_free(&bx);
  free(chosen);
  free(words);
  free(ev);
  return rc;
}

static int box_task_ad(const or_box *bx, const uint16_t *w, const uint8_t *mid, uint32_t t, uint16_t *out,
                       uint64_t *lo_out, uint64_t *hi_out) {
  if (bx->kind != 1) return OR_E_ARG;
  uint32_t W = bx->W;
  uint32_t st[32];
  int64_t ig[32];
  int64_t cursor0, start_group, ss, bi;
  uint64_t lo = 0, hi;
  if (t > 0) {
    point_span(bx, t - 1, &ss, &bi);
    lo = (uint64_t)ss;
  }
  if (t + 1 < bx->M) {
    point_span(bx, t, &ss, &bi);
    hi = (uint64_t)ss - 1;
    cursor0 = (int64_t)bx->offset[t];
    start_group = (int64_t)bx->maxg[t];
    for (uint32_t j = 0; j < W; ++j) {
      st[j] = bx->state[t * W + j];
      ig[j] = (int64_t)bx->maxg[t] - bx->gdiff[t * W + j];
    }
  } else {
    hi = bx->N - 1;
    cursor0 = (int64_t)bx->B - 1;
    start_group = (int64_t)bx->G - 1;
    for (uint32_t j = 0; j < W; ++j) {
      st[j] = bx->final_state[j];
      ig[j] = start_group;
    }
  }
  if (lo_out) *lo_out = lo;
  if (hi_out) *hi_out = hi;
  return or_ad_decode_from(w, mid, bx->K, bx->mbase, bx->mlen, bx->mf, bx->n, W, bx->N, cursor0, start_group,
                           st, ig, lo, hi, out);
}

int or_ad_recoil_decode(const uint8_t *c, uint64_t len, const uint8_t *mid, uint16_t *out) {
  or_box bx;
  int rc = box_read(c, len, &bx);
  if (rc) return rc;
  if (bx.kind != 1) { box_free(&bx); return OR_E_ARG; }
  if (bx.N == 0) { box_free(&bx); return OR_OK; }
  uint16_t *w = box_words(&bx);
  for (uint32_t t = 0; t < bx.M && rc == OR_OK; ++t) rc = box_task_ad(&bx, w, mid, t, out, NULL, NULL);
  free(w);
  box_free(&bx);
  return rc;
}

int or_ad_recoil_decode_task(const uint8_t *c, uint64_t len, const uint8_t *mid, uint32_t task, uint16_t *out,
                             uint64_t *lo, uint64_t *hi) {
  or_box bx;
  int rc = box_read(c, len, &bx);
  if (rc) return rc;
  if (bx.kind != 1 || task >= bx.M || bx.N == 0) { box_free(&bx); return OR_E_ARG; }
  uint16_t *w = box_words(&bx);
  rc = box_task_ad(&bx, w, mid, task, out, lo, hi);
  free(w);
  box_free(&bx);
  return rc;
}
