// container.cpp -- Recoil ("RCL1") and partitioned ("RCV1") containers:
// parse, write, combine, inspect.
//
// Layout (adapted from SPEC S:323-361):
//   header  : "RCL1" u8 version=1, u8 symbol_bits=8, u8 n, u8 W, u32 M, u64 N, u64 B
//   model   : u16 count, count x (u8 symbol, u32 f)
//   finals  : W x u32 final states ("explicitly transmitted")
//   global  : signed series (5-bit width field) of offset diffs actual - k ceil(B/M),
//             then signed series of max-group diffs actual - k ceil(G/M)  (P:382-384,
//             tab:metadata_split_point), byte padded
//   points  : per split point: W x u16 states (as-is) + unsigned series (4-bit
//             width field) of max_group - group_j, byte padded
//   words   : B x u16
// Series: width field = w - 1, w = max bit length (zero takes one bit),
// then w-bit magnitudes MSB first, signed series append a sign bit (1 = negative).
#include <algorithm>
#include <cstring>
#include <new>

#include "../recoil_internal.h"

namespace recoil {
namespace {

inline uint64_t get_le(const uint8_t *b, int nbytes) {
  uint64_t v = 0;
  for (int k = 0; k < nbytes; ++k) v |= (uint64_t)b[k] << (8 * k);
  return v;
}
inline void put_le(uint8_t *b, uint64_t v, int nbytes) {
  for (int k = 0; k < nbytes; ++k) b[k] = (uint8_t)(v >> (8 * k));
}
inline uint32_t bit_length(uint64_t v) { return v ? 64 - (uint32_t)__builtin_clzll(v) : 1; }

struct BitWriter {
  uint8_t *buf;
  uint64_t pos = 0;
  void put(uint64_t v, uint32_t nbits) {
    for (int32_t k = (int32_t)nbits - 1; k >= 0; --k, ++pos)
      if ((v >> k) & 1) buf[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
  }
};

struct BitReader {
  const uint8_t *buf;
  uint64_t nbits;
  uint64_t pos = 0;
  // MSB-first read of n <= 33 bits: one unaligned big-endian 64-bit load when
  // 8 bytes are available, else byte by byte at the end of the buffer.
  bool get(uint32_t n, uint64_t *v) {
    if (pos + n > nbits) return false;
    const uint64_t byte = pos >> 3;
    uint64_t word;
    if (byte + 8 <= (nbits + 7) >> 3) {
      std::memcpy(&word, buf + byte, 8);
      word = __builtin_bswap64(word);
    } else {
      word = 0;
      for (uint64_t k = 0; k < 8; ++k) word = (word << 8) | (byte + k < ((nbits + 7) >> 3) ? buf[byte + k] : 0);
    }
    *v = n ? (word << (pos & 7)) >> (64 - n) : 0;
    pos += n;
    return true;
  }
};

inline uint64_t uabs(int64_t v) { return v < 0 ? (uint64_t)(-v) : (uint64_t)v; }

uint32_t series_width(const int64_t *v, uint64_t count) {
  uint32_t w = 1;
  for (uint64_t i = 0; i < count; ++i) w = std::max(w, bit_length(uabs(v[i])));
  return w;
}

void put_series(BitWriter *bw, const int64_t *v, uint64_t count, bool is_signed, uint32_t field) {
  uint32_t w = series_width(v, count);
  bw->put(w - 1, field);
  for (uint64_t i = 0; i < count; ++i) {
    bw->put(uabs(v[i]), w);
    if (is_signed) bw->put(v[i] < 0 ? 1 : 0, 1);
  }
}

bool get_series(BitReader *br, int64_t *v, uint64_t count, bool is_signed, uint32_t field) {
  uint64_t wf;
  if (!br->get(field, &wf)) return false;
  uint32_t w = (uint32_t)wf + 1;
  if (br->pos + count * (w + (is_signed ? 1 : 0)) > br->nbits) return false;
  for (uint64_t i = 0; i < count; ++i) {
    uint64_t mag = 0, sign = 0;
    br->get(w, &mag);
    if (is_signed) br->get(1, &sign);
    v[i] = sign ? -(int64_t)mag : (int64_t)mag;
  }
  return true;
}

int parse_model(const uint8_t *c, uint64_t len, uint64_t *pos, uint32_t n, uint32_t f[256]) {
  if (*pos + 2 > len) return RECOIL_E_TRUNCATED;
  uint32_t count = (uint32_t)get_le(c + *pos, 2);
  *pos += 2;
  if (*pos + 5ull * count > len) return RECOIL_E_TRUNCATED;
  uint64_t sum = 0;
  for (uint32_t k = 0; k < count; ++k, *pos += 5) {
    uint32_t s = c[*pos];
    if (f[s]) return RECOIL_E_INCONSISTENT;
    f[s] = (uint32_t)get_le(c + *pos + 1, 4);
    if (!f[s]) return RECOIL_E_INCONSISTENT;
    sum += f[s];
  }
  return sum == (1ull << n) ? RECOIL_OK : RECOIL_E_INCONSISTENT;
}

// Adaptive model block ("RCA1"): u32 K, K x (u32 base, u32 len), sum(len) x u32 f;
// every model sums to 2^n and stays inside the 16-bit symbol range.
int parse_models(const uint8_t *c, uint64_t len, uint64_t *pos, Container *o) {
  if (*pos + 4 > len) return RECOIL_E_TRUNCATED;
  o->K = (uint32_t)get_le(c + *pos, 4);
  *pos += 4;
  if (o->K < 1 || o->K > 256) return RECOIL_E_INCONSISTENT;
  if (*pos + 8ull * o->K > len) return RECOIL_E_TRUNCATED;
  o->mbase.resize(o->K);
  o->mlen.resize(o->K);
  uint64_t msum = 0;
  for (uint32_t k = 0; k < o->K; ++k, *pos += 8) {
    o->mbase[k] = (uint32_t)get_le(c + *pos, 4);
    o->mlen[k] = (uint32_t)get_le(c + *pos + 4, 4);
    if (o->mlen[k] < 1 || (uint64_t)o->mbase[k] + o->mlen[k] > 65536) return RECOIL_E_INCONSISTENT;
    msum += o->mlen[k];
  }
  if (*pos + 4 * msum > len) return RECOIL_E_TRUNCATED;
  o->mf.resize(msum);
  for (uint64_t e = 0; e < msum; ++e, *pos += 4) o->mf[e] = (uint32_t)get_le(c + *pos, 4);
  uint64_t e0 = 0;
  for (uint32_t k = 0; k < o->K; ++k) {
    uint64_t sum = 0;
    for (uint32_t j = 0; j < o->mlen[k]; ++j) sum += o->mf[e0 + j];
    e0 += o->mlen[k];
    if (sum != (1ull << o->n)) return RECOIL_E_INCONSISTENT;
  }
  return RECOIL_OK;
}

int parse_partitioned(const uint8_t *c, uint64_t len, Container *o) {
  uint64_t pos = 28;
  int rc = parse_model(c, len, &pos, o->n, o->f);
  if (rc) return rc;
  uint64_t P = o->M;
  if (pos + 4 * P + 4 * P * o->W > len) return RECOIL_E_TRUNCATED;
  o->part_words.resize(P);
  uint64_t sum = 0;
  for (uint64_t p = 0; p < P; ++p) sum += (o->part_words[p] = get_le(c + pos + 4 * p, 4));
  pos += 4 * P;
  o->finals.resize(P * o->W);
  for (uint64_t k = 0; k < P * o->W; ++k) o->finals[k] = (uint32_t)get_le(c + pos + 4 * k, 4);
  pos += 4 * P * o->W;
  o->meta_bytes = 4 * P + 4 * P * o->W;
  if (sum != o->B) return RECOIL_E_INCONSISTENT;
  if (len < pos + 2 * o->B) return RECOIL_E_TRUNCATED;
  if (len != pos + 2 * o->B) return RECOIL_E_INCONSISTENT;
  o->words = c + pos;
  return RECOIL_OK;
}

}  // namespace

void point_span(const Container &c, uint64_t k, int64_t *sync_start, int64_t *bidx) {
  int64_t mn = INT64_MAX, mx = -1;
  for (uint32_t j = 0; j < c.W; ++j) {
    int64_t idx = (int64_t)(c.maxg[k] - c.gdiff[k * c.W + j]) * (int64_t)c.W + j;
    mn = std::min(mn, idx);
    mx = std::max(mx, idx);
  }
  *sync_start = mn;
  *bidx = mx;
}

int parse_container(const uint8_t *c, uint64_t len, Container *o, bool light) {
  if (!c || len < 28) return c ? RECOIL_E_TRUNCATED : RECOIL_E_ARG;
  bool part = std::memcmp(c, "RCV1", 4) == 0;
  bool adapt = std::memcmp(c, "RCA1", 4) == 0;
  if (!part && !adapt && std::memcmp(c, "RCL1", 4) != 0) return RECOIL_E_BAD_MAGIC;
  if (c[4] != 1 || c[5] != (adapt ? 16 : 8)) return RECOIL_E_VERSION;
  *o = Container();
  o->partitioned = part;
  o->adaptive = adapt;
  o->bytes = c;
  o->n = c[6];
  o->W = c[7];
  o->M = (uint32_t)get_le(c + 8, 4);
  o->N = get_le(c + 12, 8);
  o->B = get_le(c + 20, 8);
  o->total_bytes = len;
  if (o->n < 1 || o->n > 16 || o->W != kLanes || o->M < 1) return RECOIL_E_INCONSISTENT;
  if (o->B > o->N + 1) return RECOIL_E_INCONSISTENT;  // at most one word per symbol (b >= n)
  o->G = ceil_div(o->N, o->W);
  // every split record takes >= 2W + 1 bytes, every partition 4 + 4W bytes
  if ((uint64_t)(o->M - 1) * (2 * kLanes + 1) > len || (part && (uint64_t)o->M * (4 + 4 * kLanes) > len))
    return RECOIL_E_TRUNCATED;
  if (part) {
    int rc = parse_partitioned(c, len, o);
    o->header_bytes = len - o->meta_bytes - 2 * o->B;
    return rc;
  }
  uint64_t pos = 28;
  int rc = adapt ? parse_models(c, len, &pos, o) : parse_model(c, len, &pos, o->n, o->f);
  if (rc) return rc;
  o->header_bytes = pos;
  const uint32_t W = o->W;
  if (pos + 4ull * W > len) return RECOIL_E_TRUNCATED;
  o->finals.resize(W);
  for (uint32_t j = 0; j < W; ++j) o->finals[j] = (uint32_t)get_le(c + pos + 4 * j, 4);
  uint64_t meta_start = pos;
  pos += 4ull * W;
  const uint64_t P = o->M - 1;
  std::vector<int64_t> d(P + 1);
  BitReader br{c + pos, 8 * (len - pos)};
  if (!get_series(&br, d.data(), P, true, 5)) return RECOIL_E_TRUNCATED;
  o->offset.resize(P);
  uint64_t Eb = ceil_div(o->B, o->M), Eg = ceil_div(o->G, o->M);
  for (uint64_t k = 1; k <= P; ++k) o->offset[k - 1] = (uint64_t)((int64_t)(k * Eb) + d[k - 1]);
  if (!get_series(&br, d.data(), P, true, 5)) return RECOIL_E_TRUNCATED;
  o->maxg.resize(P);
  for (uint64_t k = 1; k <= P; ++k) o->maxg[k - 1] = (uint64_t)((int64_t)(k * Eg) + d[k - 1]);
  pos += (br.pos + 7) / 8;
  if (light) {  // record offsets only: record k = W u16 states + 1 width byte + 4 w bytes of series
    o->light = true;
    o->rec_off.resize(P + 1);
    for (uint64_t k = 0; k < P; ++k) {
      o->rec_off[k] = pos;
      if (pos + 2ull * W + 1 > len) return RECOIL_E_TRUNCATED;
      const uint32_t w = (c[pos + 2ull * W] >> 4) + 1;
      pos += 2ull * W + (4 + (uint64_t)W * w + 7) / 8;
    }
    o->rec_off[P] = pos;
    o->meta_bytes = pos - meta_start;
    if (len < pos + 2 * o->B) return RECOIL_E_TRUNCATED;
    if (len != pos + 2 * o->B) return RECOIL_E_INCONSISTENT;
    o->words = c + pos;
    for (uint64_t k = 0; k < P; ++k)
      if (o->offset[k] >= o->B || o->maxg[k] >= o->G || (k && o->offset[k] <= o->offset[k - 1]))
        return RECOIL_E_INCONSISTENT;
    return RECOIL_OK;
  }
  o->state.resize(P * W);
  o->gdiff.resize(P * W);
  int64_t dv[32];
  static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "container words/states are little endian");
  for (uint64_t k = 0; k < P; ++k) {
    if (pos + 2ull * W + 1 > len) return RECOIL_E_TRUNCATED;
    std::memcpy(&o->state[k * W], c + pos, 2ull * W);  // W x u16 LE anchor states
    pos += 2ull * W;
    // unsigned series, 4-bit width field: all W elements share one width w <= 16
    const uint32_t w = (c[pos] >> 4) + 1;
    const uint64_t bits = 4 + (uint64_t)W * w, bytes = (bits + 7) / 8;
    if (pos + bytes > len) return RECOIL_E_TRUNCATED;
    uint16_t *gd = &o->gdiff[k * W];
    if (pos + bytes + 8 <= len) {  // fast path: one unaligned big-endian load per element
      for (uint32_t j = 0; j < W; ++j) {
        const uint64_t bp = 4 + (uint64_t)j * w;
        uint64_t word;
        std::memcpy(&word, c + pos + (bp >> 3), 8);
        gd[j] = (uint16_t)((__builtin_bswap64(word) << (bp & 7)) >> (64 - w));
      }
    } else {
      BitReader pr{c + pos, 8 * (len - pos)};
      if (!get_series(&pr, dv, W, false, 4)) return RECOIL_E_TRUNCATED;
      for (uint32_t j = 0; j < W; ++j) gd[j] = (uint16_t)dv[j];
    }
    pos += bytes;
  }
  o->meta_bytes = pos - meta_start;
  if (len < pos + 2 * o->B) return RECOIL_E_TRUNCATED;
  if (len != pos + 2 * o->B) return RECOIL_E_INCONSISTENT;
  o->words = c + pos;
  // consistency: points inside the stream, sync starts strictly increasing
  int64_t prev_ss = -1;
  o->sync_start.resize(P);
  o->bidx.resize(P);
  for (uint64_t k = 0; k < P; ++k) {
    if (o->offset[k] >= o->B || o->maxg[k] >= o->G || (k && o->offset[k] <= o->offset[k - 1]))
      return RECOIL_E_INCONSISTENT;
    // anchor index of lane j = (maxg - d_j) W + j: its min / max over lanes via d_j W - j
    const uint16_t *gd = &o->gdiff[k * W];
    int32_t dmax = 0, vmax = INT32_MIN, vmin = INT32_MAX;
    for (uint32_t j = 0; j < W; ++j) {
      const int32_t v = (int32_t)gd[j] * (int32_t)W - (int32_t)j;
      dmax = std::max(dmax, (int32_t)gd[j]);
      vmax = std::max(vmax, v);
      vmin = std::min(vmin, v);
    }
    if ((uint64_t)dmax > o->maxg[k]) return RECOIL_E_INCONSISTENT;
    const int64_t ss = (int64_t)o->maxg[k] * W - vmax, bi = (int64_t)o->maxg[k] * W - vmin;
    if ((uint64_t)bi >= o->N || ss <= prev_ss) return RECOIL_E_INCONSISTENT;
    o->sync_start[k] = ss;
    o->bidx[k] = bi;
    prev_ss = ss;
  }
  return RECOIL_OK;
}

int point_span_light(const Container &c, uint64_t k, int64_t *sync_start, int64_t *bidx) {
  if (!c.light) {
    *sync_start = c.sync_start[k];
    *bidx = c.bidx[k];
    return RECOIL_OK;
  }
  const uint8_t *r = c.bytes + c.rec_off[k] + 2 * c.W;
  BitReader br{r, 8 * (c.rec_off[k + 1] - c.rec_off[k] - 2 * c.W)};
  int64_t d[32];
  if (!get_series(&br, d, c.W, false, 4)) return RECOIL_E_TRUNCATED;
  int64_t mn = INT64_MAX, mx = -1;
  for (uint32_t j = 0; j < c.W; ++j) {
    if ((uint64_t)d[j] > c.maxg[k]) return RECOIL_E_INCONSISTENT;
    const int64_t idx = (int64_t)(c.maxg[k] - (uint64_t)d[j]) * c.W + j;
    mn = std::min(mn, idx);
    mx = std::max(mx, idx);
  }
  *sync_start = mn;
  *bidx = mx;
  return RECOIL_OK;
}

int write_recoil_container(const Container &c, const uint8_t *words, uint8_t *out, uint64_t *len) {
  const uint32_t W = c.W, M = c.M;
  const uint64_t P = M - 1;
  uint32_t count = 0;
  for (int s = 0; s < 256; ++s) count += c.f[s] ? 1 : 0;
  const uint64_t model_bytes = c.adaptive ? 4 + 8ull * c.K + 4ull * c.mf.size() : 2 + 5ull * count;
  std::vector<int64_t> doff(P + 1), dg(P + 1);
  uint64_t Eb = ceil_div(c.B, M), Eg = ceil_div(c.G, M);
  for (uint64_t k = 1; k <= P; ++k) {
    doff[k - 1] = (int64_t)c.offset[k - 1] - (int64_t)(k * Eb);
    dg[k - 1] = (int64_t)c.maxg[k - 1] - (int64_t)(k * Eg);
    if ((uabs(doff[k - 1]) >> 32) || (uabs(dg[k - 1]) >> 32)) return RECOIL_E_OVERFLOW;
  }
  uint64_t gbits = 5 + P * (series_width(doff.data(), P) + 1) + 5 + P * (series_width(dg.data(), P) + 1);
  uint64_t pbytes = 0;
  std::vector<uint8_t> pw(P);
  for (uint64_t k = 0; k < P; ++k) {
    uint32_t w = 1;
    for (uint32_t j = 0; j < W; ++j) w = std::max(w, bit_length(c.gdiff[k * W + j]));
    if (w > 16) return RECOIL_E_OVERFLOW;
    pw[k] = (uint8_t)w;
    pbytes += 2ull * W + (4 + (uint64_t)W * w + 7) / 8;
  }
  uint64_t total = 28 + model_bytes + 4ull * W + (gbits + 7) / 8 + pbytes + 2 * c.B;
  if (!out) {
    *len = total;
    return RECOIL_OK;
  }
  if (*len < total) {
    *len = total;
    return RECOIL_E_BUFFER;
  }
  uint64_t meta_end = total - 2 * c.B;
  std::memset(out, 0, meta_end);
  uint8_t *q = out;
  std::memcpy(q, c.adaptive ? "RCA1" : "RCL1", 4);
  q[4] = 1;
  q[5] = c.adaptive ? 16 : 8;
  q[6] = (uint8_t)c.n;
  q[7] = (uint8_t)W;
  put_le(q + 8, M, 4);
  put_le(q + 12, c.N, 8);
  put_le(q + 20, c.B, 8);
  q += 28;
  if (c.adaptive) {
    put_le(q, c.K, 4);
    q += 4;
    for (uint32_t k = 0; k < c.K; ++k, q += 8) {
      put_le(q, c.mbase[k], 4);
      put_le(q + 4, c.mlen[k], 4);
    }
    for (size_t e = 0; e < c.mf.size(); ++e, q += 4) put_le(q, c.mf[e], 4);
  } else {
    put_le(q, count, 2);
    q += 2;
    for (int s = 0; s < 256; ++s)
      if (c.f[s]) {
        q[0] = (uint8_t)s;
        put_le(q + 1, c.f[s], 4);
        q += 5;
      }
  }
  for (uint32_t j = 0; j < W; ++j, q += 4) put_le(q, c.finals[j], 4);
  BitWriter bw{q};
  put_series(&bw, doff.data(), P, true, 5);
  put_series(&bw, dg.data(), P, true, 5);
  q += (bw.pos + 7) / 8;
  int64_t dv[32];
  for (uint64_t k = 0; k < P; ++k) {
    for (uint32_t j = 0; j < W; ++j, q += 2) put_le(q, c.state[k * W + j], 2);
    for (uint32_t j = 0; j < W; ++j) dv[j] = c.gdiff[k * W + j];
    BitWriter pb{q};
    put_series(&pb, dv, W, false, 4);
    q += (pb.pos + 7) / 8;
  }
  if (c.B) std::memcpy(q, words, 2 * c.B);
  *len = total;
  return RECOIL_OK;
}

}  // namespace recoil

using namespace recoil;

extern "C" int recoil_combine_splits(const uint8_t *in, uint64_t in_len, uint32_t target, uint8_t *out,
                                     uint64_t *out_len) {
  if (!in || !out_len || target < 1) return RECOIL_E_ARG;
  try {
    Container c;
    int rc = parse_container(in, in_len, &c);
    if (rc) return rc;
    if (c.partitioned) return RECOIL_E_ARG;  // partitions cannot be combined
    if (target >= c.M) {
      if (!out) {
        *out_len = in_len;
        return RECOIL_OK;
      }
      if (*out_len < in_len) {
        *out_len = in_len;
        return RECOIL_E_BUFFER;
      }
      std::memcpy(out, in, in_len);
      *out_len = in_len;
      return RECOIL_OK;
    }
    uint64_t k = ceil_div(c.M, target), P = c.M - 1, kept = 0;
    for (uint64_t pos = k; pos <= P; pos += k, ++kept) {  // 1-based positions k, 2k, ...
      c.offset[kept] = c.offset[pos - 1];
      c.maxg[kept] = c.maxg[pos - 1];
      std::memmove(&c.state[kept * c.W], &c.state[(pos - 1) * c.W], 2 * c.W);
      std::memmove(&c.gdiff[kept * c.W], &c.gdiff[(pos - 1) * c.W], 2 * c.W);
    }
    c.M = (uint32_t)kept + 1;
    return write_recoil_container(c, c.words, out, out_len);
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_inspect(const uint8_t *container, uint64_t len, recoil_info *info) {
  if (!container || !info) return RECOIL_E_ARG;
  try {
    Container c;
    int rc = parse_container(container, len, &c);
    if (rc) return rc;
    info->n_symbols = c.N;
    info->n_words = c.B;
    info->n_splits = c.M;
    info->prob_bits = c.n;
    info->lanes = c.W;
    info->partitioned = c.partitioned ? 1 : 0;
    info->symbol_bits = c.adaptive ? 16 : 8;
    info->n_models = c.adaptive ? c.K : 1;
    info->header_bytes = c.header_bytes;
    info->meta_bytes = c.meta_bytes;
    info->word_bytes = 2 * c.B;
    info->total_bytes = len;
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" const char *recoil_strerror(int s) {
  switch (s) {
    case RECOIL_OK: return "ok";
    case RECOIL_E_ARG: return "invalid argument";
    case RECOIL_E_EMPTY: return "empty histogram";
    case RECOIL_E_ALPHABET: return "alphabet larger than 2^n";
    case RECOIL_E_ZERO_FREQ: return "symbol with zero frequency";
    case RECOIL_E_OVERFLOW: return "metadata value overflows its field";
    case RECOIL_E_BAD_MAGIC: return "bad magic";
    case RECOIL_E_VERSION: return "unsupported version";
    case RECOIL_E_TRUNCATED: return "truncated container";
    case RECOIL_E_INCONSISTENT: return "inconsistent metadata";
    case RECOIL_E_UNDERFLOW: return "bitstream underflow";
    case RECOIL_E_SYNC: return "synchronisation / end-state failure";
    case RECOIL_E_CUDA: return "CUDA error";
    case RECOIL_E_NOMEM: return "out of memory";
    case RECOIL_E_BUFFER: return "buffer too small";
    case RECOIL_E_UNSUPPORTED: return "unsupported on the GPU path";
    default: return "unknown error";
  }
}
