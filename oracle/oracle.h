/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded C11 reference of Recoil (Lin et al.,
 * arXiv 2306.12141, /root/reference/PAPER.md, cited as P:<line>).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  It shares no code, header, table or constant
 * generator with the product (paper_2306_12141_b200/, include/recoil.h).
 *
 * Parameters (tab:rans_params P:400-423): 32-bit state, L = 2^16, b = 16,
 * 8-bit symbols, 1 <= n <= 16, 1 <= W <= 32 interleaved lanes.
 * Indices are 0-based: symbol i belongs to lane i mod W and group i / W.
 *
 * Parity pins: every function is pinned by tests/test_oracle_pins.py
 * (worked examples of the paper / SPEC, closed forms, invariants, brute
 * force).  Functions marked "parity unpinned" have no such pin.
 */
#ifndef RECOIL_ORACLE_H
#define RECOIL_ORACLE_H
#include <stdint.h>

#define OR_OK 0
#define OR_E_ARG -1
#define OR_E_MODEL -2
#define OR_E_UNDERFLOW -3
#define OR_E_END -4
#define OR_E_CONTAINER -5
#define OR_E_NOMEM -6
#define OR_E_BUFFER -7
#define OR_E_OVERFLOW -8

/* One renormalisation event = one emitted word (the word's offset is the
 * event's position in the log).  idx = the lane's most recently encoded
 * symbol (reading Z7), state = lane state right after the emission. */
typedef struct {
  int64_t idx;
  uint32_t lane;
  uint32_t state;
} or_event;

/* model */
int or_quantize(const uint64_t *hist, uint32_t count, uint32_t n, uint32_t *f);
int or_build_model(const uint64_t hist[256], uint32_t n, uint32_t f[256]);
uint64_t or_encode_step(uint64_t x, uint32_t f, uint32_t F, uint32_t n);
int or_decode_step(uint32_t x, const uint32_t f[256], uint32_t n, uint32_t *s, uint32_t *x_prev);
/* Eq. 3 / Eq. 4 on one lane; return number of words moved */
int or_renorm_encode(uint64_t *x, uint32_t f_next, uint32_t n, uint16_t *words, uint64_t *p);
int or_renorm_decode(uint64_t *x, const uint16_t *words, int64_t *p);

/* W-way interleaved encoder: returns B (words written) or <0. */
int64_t or_interleaved_encode(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                              uint32_t W, uint16_t *words, uint32_t *final_states,
                              or_event *events, uint64_t *max_renorm_steps);
/* Serial interleaved decoder: full stream, from the final states. */
int or_interleaved_decode(const uint16_t *words, uint64_t B, const uint32_t *final_states,
                          uint64_t N, const uint32_t f[256], uint32_t n, uint32_t W, uint8_t *out);

/* Backward scan: anchors of the split at event e. Returns 1 if
 * feasible, 0 if not (a lane has no event at or before e, or an anchor idx < 0). */
int or_backward_scan(const or_event *ev, uint64_t e, uint32_t W, uint32_t *anchor_state,
                     int64_t *anchor_idx, int64_t *sync_start);
/* Heuristic H */
int64_t or_heuristic(int64_t t, int64_t ts, int64_t T);
/* Split selection (reading Z10): writes chosen event offsets, returns count. */
int64_t or_choose_splits(const or_event *ev, uint64_t n_ev, uint64_t N, uint32_t W, uint32_t M,
                         uint64_t *chosen);
/* The same with flags: OR_SPLIT_PRINTED_T = T fixed at the printed ceil(N/M)
 * instead of reading Z10''s per-boundary T_m. */
#define OR_SPLIT_PRINTED_T 1u
int64_t or_choose_splits_ex(const or_event *ev, uint64_t n_ev, uint64_t N, uint32_t W, uint32_t M,
                            uint32_t flags, uint64_t *chosen);

/* Data series: bit-packed, MSB first. */
uint64_t or_pack_series(const int64_t *v, uint64_t count, int is_signed, uint32_t field_bits,
                        uint8_t *buf, uint64_t bitpos);
int64_t or_unpack_series(const uint8_t *buf, uint64_t buf_bits, uint64_t bitpos, uint64_t count,
                         int is_signed, uint32_t field_bits, int64_t *v);

/* Task entry decoded by the 3-phase decoder. */
int or_decode_from(const uint16_t *words, uint64_t B, const uint32_t f[256], uint32_t n,
                   uint32_t W, uint64_t N, int64_t cursor0, int64_t start_group,
                   const uint32_t *init_state, const int64_t *init_group,
                   uint64_t commit_lo, uint64_t commit_hi, uint8_t *out, uint8_t *produced,
                   int64_t *cursor_end);

/* Whole-pipeline helpers: Recoil container. */
int or_recoil_encode(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                     uint32_t W, uint32_t M, uint8_t *out, uint64_t *len);
int or_recoil_encode_ex(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                        uint32_t W, uint32_t M, uint32_t split_flags, uint8_t *out, uint64_t *len);
int or_combine(const uint8_t *in, uint64_t in_len, uint32_t target, uint8_t *out, uint64_t *len);
int or_container_info(const uint8_t *c, uint64_t len, uint64_t info[8]);
/* split table of a container: per point (M-1): offset, max_group, sync_start, boundary idx */
int or_container_points(const uint8_t *c, uint64_t len, uint64_t *offset, uint64_t *maxg,
                        uint64_t *sync_start, uint64_t *bidx);
int or_recoil_decode(const uint8_t *c, uint64_t len, uint8_t *out);
/* A container parsed once for repeated task decodes (bounded CPU samples). */
typedef struct or_opened or_opened;
int or_open(const uint8_t *c, uint64_t len, or_opened **out);
int or_opened_decode_tasks(or_opened *h, const uint32_t *tasks, uint32_t n_tasks, uint8_t *out,
                           uint64_t *n_symbols);
void or_close(or_opened *h);
int or_recoil_decode_task(const uint8_t *c, uint64_t len, uint32_t task, uint8_t *out,
                          uint64_t *lo, uint64_t *hi);
int or_recoil_decode_tasks(const uint8_t *c, uint64_t len, const uint32_t *tasks, uint32_t n_tasks,
                           uint8_t *out, uint64_t *n_symbols);

/* Conventional partitioned codec. */
int or_partitioned_encode(const uint8_t *sym, uint64_t N, const uint32_t f[256], uint32_t n,
                          uint32_t W, uint32_t P, uint8_t *out, uint64_t *len);
int or_partitioned_decode(const uint8_t *c, uint64_t len, uint8_t *out);

/* Adaptive coding with index-keyed models and 16-bit symbols (P:227 item
 * (3)): K models, model k = values base[k] .. base[k]+len[k]-1
 * with frequencies mf[off_k + j] (sum 2^n); symbol i uses model mid[i].
 * Container "RCA1" (16-bit symbols, model set in the model block). */
int64_t or_ad_interleaved_encode(const uint16_t *sym, uint64_t N, const uint8_t *mid, uint32_t K,
                                 const uint32_t *base, const uint32_t *len, const uint32_t *mf, uint32_t n,
                                 uint32_t W, uint16_t *words, uint32_t *final_states, or_event *events);
int or_ad_interleaved_decode(const uint16_t *words, uint64_t B, const uint32_t *final_states, uint64_t N,
                             const uint8_t *mid, uint32_t K, const uint32_t *base, const uint32_t *len,
                             const uint32_t *mf, uint32_t n, uint32_t W, uint16_t *out);
int or_ad_decode_from(const uint16_t *words, const uint8_t *mid, uint32_t K, const uint32_t *base,
                      const uint32_t *len, const uint32_t *mf, uint32_t n, uint32_t W, uint64_t N,
                      int64_t cursor0, int64_t start_group, const uint32_t *init_state,
                      const int64_t *init_group, uint64_t commit_lo, uint64_t commit_hi, uint16_t *out);
int or_ad_recoil_encode(const uint16_t *sym, uint64_t N, const uint8_t *mid, uint32_t K, const uint32_t *base,
                        const uint32_t *len, const uint32_t *mf, uint32_t n, uint32_t W, uint32_t M,
                        uint8_t *out, uint64_t *outlen);
int or_ad_recoil_decode(const uint8_t *c, uint64_t len, const uint8_t *mid, uint16_t *out);
int or_ad_recoil_decode_task(const uint8_t *c, uint64_t len, const uint8_t *mid, uint32_t task, uint16_t *out,
                             uint64_t *lo, uint64_t *hi);

#endif
