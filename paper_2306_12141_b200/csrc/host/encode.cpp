// encode.cpp -- model quantiser, serial interleaved rANS encoder with a
// streaming split selector, and the partitioned (conventional) encoder.
//
// Paper: Eq. 1, Eq. 3, interleaving,
// backward scan, heuristic H (reading Z10' in DESIGN.md),
// metadata.  The split choices must equal the oracle's exactly
// (tests/test_host_parity.py compares containers byte for byte); the
// selector here is a streaming re-formulation: the backward scan's sync start
// is the oldest entry of an LRU list of the lanes' last events, and candidate
// windows are evaluated from a bounded event buffer.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <deque>
#include <new>
#include <thread>
#include <vector>

#include "../recoil_internal.h"

namespace recoil {
namespace {

// Exact floor(x / f) for x < 2^32, 1 <= f <= 2^16: q = (x * m) >> (32 + l),
// l = ceil(log2 f), m = ceil(2^(32+l) / f)  (error < 2^-l <= 1/f).
struct Recip {
  uint64_t m;
  uint32_t shift;
};

inline Recip make_recip(uint32_t f) {
  uint32_t l = 0;
  while ((1ull << l) < f) ++l;
  unsigned __int128 num = (unsigned __int128)1 << (32 + l);
  uint64_t m = (uint64_t)((num + f - 1) / f);
  return {m, 32 + l};
}

inline uint32_t div_recip(uint32_t x, const Recip &r) {
  return (uint32_t)(((unsigned __int128)x * r.m) >> r.shift);
}

struct SymInfo {
  uint64_t thr;  // Eq. 3 threshold f * 2^(32-n)
  uint32_t f, F;
  Recip rcp;
};

int check_model(const uint32_t freqs[256], uint32_t n, SymInfo *si) {
  if (n < 1 || n > 16) return RECOIL_E_ARG;
  uint64_t sum = 0;
  for (int s = 0; s < 256; ++s) {
    si[s].f = freqs[s];
    si[s].F = (uint32_t)sum;
    sum += freqs[s];
    si[s].thr = (uint64_t)freqs[s] << (32 - n);
    if (freqs[s]) si[s].rcp = make_recip(freqs[s]);
  }
  return sum == (1ull << n) ? RECOIL_OK : RECOIL_E_ARG;
}

// Streaming split selector (see file comment).  Events arrive in word order.
class Selector {
 public:
  Selector(uint64_t N, uint32_t M) : N_(N), M_(M) {
    done_ = (M <= 1 || N == 0);
    T_ = done_ ? 0 : (int64_t)ceil_div(N, M);
    win_ = 2 * T_;
    for (uint32_t j = 0; j < kLanes; ++j) {
      last_idx_[j] = -1;
      prev_lane_[j] = next_lane_[j] = -1;
    }
  }

  void on_event(uint64_t offset, uint32_t lane, int64_t idx, uint32_t state) {
    // LRU of lanes by the time of their last event: tail = oldest = sync start.
    if (!seen_[lane]) {
      seen_[lane] = true;
      nseen_++;
    } else {
      unlink(lane);
    }
    push_front(lane);
    last_idx_[lane] = idx;
    if (done_) return;
    int64_t ss = (nseen_ == (int)kLanes) ? last_idx_[tail_] : -1;  // min over the lanes' last events
    while (!done_ && idx > prev_ + win_) finalize(false);
    if (done_) return;
    if (buf_.empty()) buf_base_ = offset;
    buf_.push_back(Ev{idx, ss, (uint16_t)state, (uint8_t)lane});
  }

  void finish() {
    while (!done_) finalize(true);
  }

  struct Point {
    uint64_t offset, maxg;
    uint16_t state[32];
    uint16_t gdiff[32];
  };
  std::vector<Point> points;

 private:
  struct Ev {
    int64_t idx, ss;  // ss < 0: infeasible
    uint16_t state;
    uint8_t lane;
  };

  void unlink(int j) {
    int p = prev_lane_[j], n = next_lane_[j];
    if (p >= 0) next_lane_[p] = n; else head_ = n;
    if (n >= 0) prev_lane_[n] = p; else tail_ = p;
  }
  void push_front(int j) {
    prev_lane_[j] = -1;
    next_lane_[j] = head_;
    if (head_ >= 0) prev_lane_[head_] = j;
    head_ = j;
    if (tail_ < 0) tail_ = j;
  }

  // Close the window of boundary m: pick the minimum-H candidate with
  // 0 < t <= win_ (2T, doubled while empty: reading Z10'').  at_end: no more
  // events will arrive, so an empty window is doubled until it covers the buffer.
  void finalize(bool at_end) {
    int64_t best = -1, best_h = 0;
    for (size_t q = 0; q < buf_.size(); ++q) {
      const Ev &e = buf_[q];
      if (e.idx <= prev_) continue;
      if (e.idx - prev_ > win_) break;
      if (e.ss < 0 || e.ss <= prev_) continue;
      if (e.idx / kLanes - e.ss / kLanes > 65535) continue;
      int64_t t = e.idx - prev_, ts = e.idx - e.ss + 1;
      int64_t h = (t > T_ ? t - T_ : T_ - t) + (t - ts > T_ ? t - ts - T_ : T_ - (t - ts));
      if (best < 0 || h < best_h) {
        best = (int64_t)q;
        best_h = h;
      }
    }
    if (best < 0) {
      const bool covers = buf_.empty() || buf_.back().idx - prev_ <= win_;
      if (at_end && covers) {
        done_ = true;
        buf_.clear();
      } else {
        win_ *= 2;
      }
      return;
    }
    // anchors: backward scan from the chosen event over the buffer
    Point pt;
    const Ev &be = buf_[(size_t)best];
    pt.offset = buf_base_ + (uint64_t)best;
    pt.maxg = (uint64_t)be.idx / kLanes;
    uint32_t found = 0, cnt = 0;
    for (int64_t q = best; q >= 0 && cnt < kLanes; --q) {
      const Ev &e = buf_[(size_t)q];
      if (found & (1u << e.lane)) continue;
      found |= 1u << e.lane;
      cnt++;
      pt.state[e.lane] = e.state;
      pt.gdiff[e.lane] = (uint16_t)(pt.maxg - (uint64_t)e.idx / kLanes);
    }
    points.push_back(pt);
    prev_ = be.idx;
    size_t drop = (size_t)best + 1;
    buf_.erase(buf_.begin(), buf_.begin() + (ptrdiff_t)drop);
    buf_base_ += drop;
    m_++;
    if (m_ >= M_) {
      done_ = true;
      buf_.clear();
      return;
    }
    T_ = (int64_t)ceil_div(N_ - (uint64_t)(prev_ + 1), M_ - m_ + 1);
    win_ = 2 * T_;
  }

  uint64_t N_;
  uint32_t M_;
  uint32_t m_ = 1;
  bool done_;
  int64_t T_, win_;
  int64_t prev_ = -1;
  std::deque<Ev> buf_;
  uint64_t buf_base_ = 0;
  bool seen_[32] = {false};
  int nseen_ = 0;
  int64_t last_idx_[32];
  int prev_lane_[32], next_lane_[32];
  int head_ = -1, tail_ = -1;
};

// Serial 32-way interleaved encoder (Eq. 1 + Eq. 3, renormalisation outputs of
// a group boundary in increasing lane order, initial state L).  info(i) gives
// f, F and the Eq. 3 threshold of symbol i: the symbol's entry of the static
// model, or of model mid[i] for the adaptive codec (P:227 item (3)).
template <bool kLog, class Info>
int interleaved_encode_gen(uint64_t N, const Info &info, uint32_t n, std::vector<uint16_t> *words,
                           uint32_t final_states[32], Selector *sel) {
  uint32_t x[32];
  for (uint32_t j = 0; j < kLanes; ++j) x[j] = kL;
  for (uint64_t i = 0; i < N; ++i)
    if (info(i).f == 0) return RECOIL_E_ZERO_FREQ;
  uint64_t G = ceil_div(N, kLanes);
  for (uint64_t g = 0; g < G; ++g) {
    uint64_t base = g * kLanes;
    uint32_t lanes = (uint32_t)std::min<uint64_t>(kLanes, N - base);
    for (uint32_t j = 0; j < lanes; ++j) {
      const SymInfo &s = info(base + j);
      if (x[j] >= s.thr) {  // single step suffices since b >= n
        if (kLog) sel->on_event(words->size(), j, (int64_t)(base + j) - (int64_t)kLanes, x[j] >> kWordBits);
        words->push_back((uint16_t)x[j]);
        x[j] >>= kWordBits;
      }
    }
    for (uint32_t j = 0; j < lanes; ++j) {
      const SymInfo &s = info(base + j);
      uint32_t q = div_recip(x[j], s.rcp);
      x[j] = (q << n) + s.F + (x[j] - q * s.f);
    }
  }
  for (uint32_t j = 0; j < kLanes; ++j) final_states[j] = x[j];
  return RECOIL_OK;
}

template <bool kLog>
int interleaved_encode(const uint8_t *sym, uint64_t N, const SymInfo *si, uint32_t n,
                       std::vector<uint16_t> *words, uint32_t final_states[32], Selector *sel) {
  auto info = [&](uint64_t i) -> const SymInfo & { return si[sym[i]]; };
  return interleaved_encode_gen<kLog>(N, info, n, words, final_states, sel);
}

// Fill c's split metadata from the selector's points.
void take_points(const Selector &sel, Container *c) {
  size_t P = sel.points.size();
  c->M = (uint32_t)P + 1;
  c->offset.resize(P);
  c->maxg.resize(P);
  c->state.resize(P * kLanes);
  c->gdiff.resize(P * kLanes);
  for (size_t k = 0; k < P; ++k) {
    c->offset[k] = sel.points[k].offset;
    c->maxg[k] = sel.points[k].maxg;
    std::memcpy(&c->state[k * kLanes], sel.points[k].state, 64);
    std::memcpy(&c->gdiff[k * kLanes], sel.points[k].gdiff, 64);
  }
}

}  // namespace

int encode_recoil(const uint8_t *sym, uint64_t N, const uint32_t freqs[256], uint32_t n, uint32_t M,
                  Container *c, std::vector<uint16_t> *words) {
  SymInfo si[256];
  int rc = check_model(freqs, n, si);
  if (rc) return rc;
  if (M < 1) return RECOIL_E_ARG;
  words->clear();
  words->reserve(N / 2 + 64);
  c->partitioned = false;
  c->n = n;
  c->W = kLanes;
  c->N = N;
  c->G = ceil_div(N, kLanes);
  std::memcpy(c->f, freqs, sizeof(c->f));
  c->finals.assign(kLanes, 0);
  Selector sel(N, M);
  if (M > 1)
    rc = interleaved_encode<true>(sym, N, si, n, words, c->finals.data(), &sel);
  else
    rc = interleaved_encode<false>(sym, N, si, n, words, c->finals.data(), &sel);
  if (rc) return rc;
  sel.finish();
  c->B = words->size();
  take_points(sel, c);
  return RECOIL_OK;
}

// Adaptive codec (index-keyed models, 16-bit symbols; P:227 item (3), P:411,
// P:514): model k covers values base[k] .. base[k]+len[k]-1 with frequencies
// freqs[off_k + j]; symbol i is coded with model mid[i].  Same split selector.
int encode_recoil_adaptive(const uint16_t *sym, uint64_t N, const uint8_t *mid, uint32_t K, const uint32_t *base,
                           const uint32_t *len, const uint32_t *freqs, uint32_t n, uint32_t M, Container *c,
                           std::vector<uint16_t> *words) {
  if (n < 1 || n > 16 || K < 1 || K > 256 || M < 1) return RECOIL_E_ARG;
  std::vector<uint64_t> off(K + 1, 0);
  for (uint32_t k = 0; k < K; ++k) {
    if (len[k] < 1 || (uint64_t)base[k] + len[k] > 65536) return RECOIL_E_ARG;
    off[k + 1] = off[k] + len[k];
  }
  std::vector<SymInfo> si(off[K]);
  for (uint32_t k = 0; k < K; ++k) {
    uint64_t sum = 0;
    for (uint32_t j = 0; j < len[k]; ++j) {
      SymInfo &e = si[off[k] + j];
      const uint32_t f = freqs[off[k] + j];
      e.f = f;
      e.F = (uint32_t)sum;
      e.thr = (uint64_t)f << (32 - n);
      if (f) e.rcp = make_recip(f);
      sum += f;
    }
    if (sum != (1ull << n)) return RECOIL_E_ARG;
  }
  static const SymInfo kAbsent{};  // f = 0: rejected as E_ZERO_FREQ
  for (uint64_t i = 0; i < N; ++i)
    if (mid[i] >= K || sym[i] < base[mid[i]] || sym[i] - base[mid[i]] >= len[mid[i]]) return RECOIL_E_ZERO_FREQ;
  auto info = [&](uint64_t i) -> const SymInfo & {
    const uint32_t k = mid[i];
    return (k < K) ? si[off[k] + (sym[i] - base[k])] : kAbsent;
  };
  words->clear();
  words->reserve(N / 2 + 64);
  c->partitioned = false;
  c->adaptive = true;
  c->n = n;
  c->W = kLanes;
  c->N = N;
  c->G = ceil_div(N, kLanes);
  c->K = K;
  c->mbase.assign(base, base + K);
  c->mlen.assign(len, len + K);
  c->mf.assign(freqs, freqs + off[K]);
  c->finals.assign(kLanes, 0);
  Selector sel(N, M);
  int rc = M > 1 ? interleaved_encode_gen<true>(N, info, n, words, c->finals.data(), &sel)
                 : interleaved_encode_gen<false>(N, info, n, words, c->finals.data(), &sel);
  if (rc) return rc;
  sel.finish();
  c->B = words->size();
  take_points(sel, c);
  return RECOIL_OK;
}

static void put_le(uint8_t *b, uint64_t v, int nbytes) {
  for (int k = 0; k < nbytes; ++k) b[k] = (uint8_t)(v >> (8 * k));
}

int encode_partitioned(const uint8_t *sym, uint64_t N, const uint32_t freqs[256], uint32_t n,
                       uint32_t P, uint8_t *out, uint64_t *len) {
  SymInfo si[256];
  int rc = check_model(freqs, n, si);
  if (rc) return rc;
  if (P < 1) return RECOIL_E_ARG;
  uint32_t count = 0;
  for (int s = 0; s < 256; ++s) count += freqs[s] ? 1 : 0;
  uint64_t fixed = 28 + 2 + 5ull * count + 4ull * P + 4ull * P * kLanes;
  if (!out) {
    *len = fixed + 2 * N + 64;  // upper bound: at most one word per symbol (b >= n)
    return RECOIL_OK;
  }
  uint64_t G = ceil_div(N, kLanes);
  // partitions are independent codecs: encode them on several threads,
  // each into its own word vector, then concatenate in partition order
  std::vector<std::vector<uint16_t>> parts(P);
  std::vector<uint32_t> cnt(P), fin((size_t)P * kLanes);
  std::vector<int> prc(P, RECOIL_OK);
  std::atomic<uint64_t> next{0};
  auto worker = [&]() {
    for (uint64_t p; (p = next.fetch_add(1)) < P;) {
      uint64_t lo = kLanes * (p * G / P), hi = std::min<uint64_t>(N, kLanes * ((p + 1) * G / P));
      if (lo > hi) lo = hi;
      parts[p].reserve((hi - lo) / 2 + 64);
      prc[p] = interleaved_encode<false>(sym + lo, hi - lo, si, n, &parts[p], &fin[p * kLanes], nullptr);
      if (!prc[p] && (parts[p].size() >> 32)) prc[p] = RECOIL_E_OVERFLOW;
    }
  };
  const uint32_t nt = (uint32_t)std::min<uint64_t>({P, (uint64_t)std::max(1u, std::thread::hardware_concurrency()),
                                                    std::max<uint64_t>(1, N >> 22)});
  std::vector<std::thread> pool;
  for (uint32_t i = 1; i < nt; ++i) pool.emplace_back(worker);
  worker();
  for (auto &th : pool) th.join();
  uint64_t n_words = 0;
  for (uint64_t p = 0; p < P; ++p) {
    if (prc[p]) return prc[p];
    cnt[p] = (uint32_t)parts[p].size();
    n_words += parts[p].size();
  }
  uint64_t total = fixed + 2 * n_words;
  if (*len < total) {
    *len = total;
    return RECOIL_E_BUFFER;
  }
  uint8_t *q = out;
  std::memcpy(q, "RCV1", 4);
  q[4] = 1;
  q[5] = 8;
  q[6] = (uint8_t)n;
  q[7] = (uint8_t)kLanes;
  put_le(q + 8, P, 4);
  put_le(q + 12, N, 8);
  put_le(q + 20, n_words, 8);
  q += 28;
  put_le(q, count, 2);
  q += 2;
  for (int s = 0; s < 256; ++s)
    if (freqs[s]) {
      q[0] = (uint8_t)s;
      put_le(q + 1, freqs[s], 4);
      q += 5;
    }
  for (uint64_t p = 0; p < P; ++p, q += 4) put_le(q, cnt[p], 4);
  for (size_t k = 0; k < fin.size(); ++k, q += 4) put_le(q, fin[k], 4);
  for (uint64_t p = 0; p < P; ++p)  // u16 little endian (host is little endian, as the container)
    for (size_t w = 0; w < parts[p].size(); ++w, q += 2) put_le(q, parts[p][w], 2);
  *len = total;
  return RECOIL_OK;
}

}  // namespace recoil

using namespace recoil;

extern "C" int recoil_quantize(const uint64_t *hist, uint32_t count, uint32_t n, uint32_t *f) {
  if (!hist || !f || count < 1 || n < 1 || n > 16) return RECOIL_E_ARG;
  uint64_t total = 0, distinct = 0, R = 1ull << n;
  for (uint32_t s = 0; s < count; ++s) {
    total += hist[s];
    distinct += hist[s] ? 1 : 0;
  }
  if (total == 0) return RECOIL_E_EMPTY;
  if (distinct > R) return RECOIL_E_ALPHABET;
  try {
    // order of symbols by (remainder desc, symbol asc) for the largest-remainder pass
    std::vector<uint64_t> rem(count, 0);
    std::vector<uint8_t> raised(count, 0);
    uint64_t sum = 0;
    for (uint32_t s = 0; s < count; ++s) {
      f[s] = 0;
      if (!hist[s]) continue;
      unsigned __int128 prod = (unsigned __int128)hist[s] * R;
      uint64_t q = (uint64_t)(prod / total);
      rem[s] = (uint64_t)(prod % total);
      if (q < 1) {
        q = 1;
        raised[s] = 1;
      }
      f[s] = (uint32_t)q;
      sum += q;
    }
    if (sum < R) {
      std::vector<uint32_t> order;
      for (uint32_t s = 0; s < count; ++s)
        if (hist[s] && !raised[s]) order.push_back(s);
      std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return rem[a] > rem[b]; });
      for (size_t i = 0; sum < R && i < order.size(); ++i, ++sum) f[order[i]]++;
      if (sum < R) return RECOIL_E_ARG;  // unreachable (shortfall < #non-raised symbols)
    }
    while (sum > R) {
      int64_t best = -1;
      for (uint32_t s = 0; s < count; ++s)
        if (f[s] > 1 && (best < 0 || f[s] > f[best] || (f[s] == f[best] && hist[s] < hist[best]))) best = s;
      f[best]--;
      sum--;
    }
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_build_model(const uint64_t hist[256], uint32_t n, uint32_t f[256]) {
  return recoil_quantize(hist, 256, n, f);
}

extern "C" int recoil_encode(const uint8_t *symbols, uint64_t N, const uint32_t freqs[256],
                             uint32_t n, uint32_t M, uint8_t *out, uint64_t *len) {
  if (!len || !freqs || (N && !symbols) || M < 1 || n < 1 || n > 16) return RECOIL_E_ARG;
  if (!out) {
    uint32_t count = 0;
    for (int s = 0; s < 256; ++s) count += freqs[s] ? 1 : 0;
    // header + model + finals + global series (<= 2*(5 + 33 (M-1)) bits) + records + words
    *len = 28 + 2 + 5ull * count + 4ull * kLanes + (10 + 66ull * M) / 8 + 2 + 131ull * M + 2 * N + 64;
    return RECOIL_OK;
  }
  try {
    Container c;
    std::vector<uint16_t> words;
    int rc = encode_recoil(symbols, N, freqs, n, M, &c, &words);
    if (rc) return rc;
    std::vector<uint8_t> wbytes(2 * words.size());
    for (size_t i = 0; i < words.size(); ++i) {
      wbytes[2 * i] = (uint8_t)words[i];
      wbytes[2 * i + 1] = (uint8_t)(words[i] >> 8);
    }
    return write_recoil_container(c, wbytes.data(), out, len);
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_encode_adaptive(const uint16_t *symbols, uint64_t N, const uint8_t *model_ids,
                                      uint32_t n_models, const uint32_t *model_base, const uint32_t *model_len,
                                      const uint32_t *freqs, uint32_t n, uint32_t M, uint8_t *out, uint64_t *len) {
  if (!len || !freqs || !model_base || !model_len || (N && (!symbols || !model_ids)) || M < 1 || n < 1 || n > 16 ||
      n_models < 1 || n_models > 256)
    return RECOIL_E_ARG;
  if (!out) {
    uint64_t msum = 0;
    for (uint32_t k = 0; k < n_models; ++k) msum += model_len[k];
    *len = 28 + 4 + 8ull * n_models + 4 * msum + 4ull * kLanes + (10 + 66ull * M) / 8 + 2 + 131ull * M + 2 * N + 64;
    return RECOIL_OK;
  }
  try {
    Container c;
    std::vector<uint16_t> words;
    int rc = encode_recoil_adaptive(symbols, N, model_ids, n_models, model_base, model_len, freqs, n, M, &c, &words);
    if (rc) return rc;
    std::vector<uint8_t> wbytes(2 * words.size());
    for (size_t i = 0; i < words.size(); ++i) {
      wbytes[2 * i] = (uint8_t)words[i];
      wbytes[2 * i + 1] = (uint8_t)(words[i] >> 8);
    }
    return write_recoil_container(c, wbytes.data(), out, len);
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_partitioned_encode(const uint8_t *symbols, uint64_t N, const uint32_t freqs[256],
                                         uint32_t n, uint32_t P, uint8_t *out, uint64_t *len) {
  if (!len || !freqs || (N && !symbols) || P < 1 || n < 1 || n > 16) return RECOIL_E_ARG;
  try {
    return encode_partitioned(symbols, N, freqs, n, P, out, len);
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}
