// plan.cpp -- row a1 of the hot path: expand the container's
// split metadata into the per-warp task table, pack the LUT, plan
// the word slice / output span, and shard task ranges across GPUs (§8(e)).
//
// Task t < M-1 enters at split point t+1 (1-based): cursor0 = the point's
// bitstream offset (the boundary event's word, the first word the task reads),
// start group = the anchor (max Symbol Group ID), lane j initialised with its
// 16-bit state in group anchor - diff_j (tab:metadata_codec).  The
// last task enters from the explicitly transmitted final states; a
// lane without a symbol in the last group starts one group lower, so the
// kernel needs no i < N test.  Task t commits [sync_start(point t),
// sync_start(point t+1) - 1] (reading Z13).
#include <algorithm>
#include <cstring>
#include <new>

#include "../recoil_internal.h"

namespace recoil {

void pack_lut(const uint32_t f[256], uint32_t n, std::vector<uint8_t> *lut) {
  if (n <= 12) {  // packed: s | bias << 8 | f << 20 (symbol, f and F in one 32-bit entry)
    std::vector<uint32_t> w((size_t)1 << n, 0);
    uint32_t F = 0;
    for (uint32_t s = 0; s < 256; ++s) {
      for (uint32_t k = 0; k < f[s]; ++k) w[F + k] = s | (k << 8) | (f[s] << 20);
      F += f[s];
    }
    lut->resize(4 * w.size());
    std::memcpy(lut->data(), w.data(), lut->size());
    return;
  }
  // n = 13..16: slot -> symbol bytes, then per symbol f | F << 16
  lut->assign(((size_t)1 << n) + 1024, 0);
  uint32_t F = 0, fF[256];
  for (uint32_t s = 0; s < 256; ++s) {
    std::memset(lut->data() + F, (int)s, f[s]);
    fF[s] = (f[s] & 0xFFFFu) | (F << 16);
    F += f[s];
  }
  std::memcpy(lut->data() + ((size_t)1 << n), fF, 1024);
}

int pack_adaptive(const Container &c, uint32_t cbits, std::vector<uint8_t> *blob, uint32_t *Kout, uint32_t *Eout) {
  const uint32_t K = c.K, n = c.n;
  // per model: entries up to the last value with f > 0 (trailing zero-f values
  // cannot be decoded and would carry F = 2^n, which does not fit 16 bits)
  std::vector<uint32_t> off(K + 1, 0), keep(K);
  std::vector<uint64_t> moff(K + 1, 0);
  for (uint32_t k = 0; k < K; ++k) {
    moff[k + 1] = moff[k] + c.mlen[k];
    uint32_t last = 0;
    for (uint32_t j = 0; j < c.mlen[k]; ++j)
      if (c.mf[moff[k] + j]) last = j;
    keep[k] = last + 1;
    off[k + 1] = off[k] + keep[k];
  }
  const uint32_t E = off[K];
  if (E > 65535) return RECOIL_E_UNSUPPORTED;
  const uint32_t Epad = (E + 3) & ~3u;
  // 2^cbits coarse buckets per model: the u16 entry index containing each
  // bucket's first slot, 2^cbits + 1 boundaries (+1 pad) per model; bucket b's entries lie in
  // [lo[b], lo[b+1]] (a superset by at most one entry, excluded by the search)
  const uint32_t nbk = 1u << cbits, crow = coarse_row(cbits);
  const size_t cwords = ((size_t)K * crow * 2 + 15) / 16 * 4;  // u16 rows, 16-B aligned
  std::vector<uint32_t> w(cwords + Epad + K, 0);
  uint16_t *coarse = reinterpret_cast<uint16_t *>(w.data());
  uint32_t *ent = w.data() + cwords, *delta = ent + Epad;
  const uint32_t shift = n > cbits ? n - cbits : 0, nb = 1u << (n - shift);
  std::vector<uint32_t> F;
  for (uint32_t k = 0; k < K; ++k) {
    F.assign(keep[k], 0);
    uint32_t acc = 0;
    for (uint32_t j = 0; j < keep[k]; ++j) {
      const uint32_t f = c.mf[moff[k] + j];
      F[j] = acc;
      acc += f;
      ent[off[k] + j] = F[j] | (((f - 1) & 0xFFFFu) << 16);
    }
    delta[k] = c.mbase[k] - off[k];  // value = entry index + delta (mod 2^32)
    // largest j with F_j <= slot (F non-decreasing)
    auto entry_of = [&](uint32_t slot) {
      uint32_t j = (uint32_t)(std::upper_bound(F.begin(), F.end(), slot) - F.begin());
      return off[k] + (j ? j - 1 : 0);
    };
    for (uint32_t b = 0; b <= nbk; ++b)
      coarse[k * crow + b] = (uint16_t)(b < nb ? entry_of(b << shift) : off[k] + keep[k] - 1);
  }
  blob->resize(4 * w.size());
  std::memcpy(blob->data(), w.data(), blob->size());
  *Kout = K;
  *Eout = E;
  return RECOIL_OK;
}

static uint64_t align16(uint64_t v) { return (v + 15) & ~15ull; }

int build_decoder(const uint8_t *cbytes, uint64_t len, uint64_t task_begin, uint64_t task_end, Decoder *d,
                  bool for_gpu) {
  auto parsed = std::make_shared<Container>();
  // Recoil on the GPU: the host expands every task's record (row a1, O(M W), the full
  // parse) and the kernel streams the prebuilt records, as for partitioned containers:
  // measured 1-4 % faster than expanding the records inside the decode kernel (same box,
  // 10656 / 21312 splits).  Adaptive containers keep the fused plan (the
  // light parse: task heads + raw records expanded in the kernel).
  const bool adaptive = cbytes && len >= 4 && std::memcmp(cbytes, "RCA1", 4) == 0;
  int rc = parse_container(cbytes, len, parsed.get(), /*light=*/for_gpu && adaptive);
  if (rc) return rc;
  return build_decoder_from(std::move(parsed), task_begin, task_end, d, for_gpu);
}

// Recoil on the GPU: task heads only (row a1 split: the O(M) global series and
// record offsets are decoded here, the per-lane anchors in the kernel).
static int build_fused(Decoder *d, uint64_t tb, uint64_t te) {
  const Container &c = *d->c;
  d->fused = true;
  if (c.adaptive) {
    // the most coarse bucket bits in 9..7 whose tables fit beside the 32-warp kernel's
    // layout in one block's shared memory, else 6-bit buckets on the 8-warp kernel
    int rc0 = RECOIL_OK;
    d->ad_narrow = true;
    for (uint32_t cb = kCoarseBitsWide; cb >= kCoarseBitsWideMin && d->ad_narrow && !rc0; --cb) {
      rc0 = pack_adaptive(c, cb, &d->lut, &d->ad_K, &d->ad_E);
      d->ad_cbits = cb;
      d->ad_narrow = kAdaptiveWideLayoutBytes + d->lut.size() > kSmemOptinBytes;
    }
    if (!rc0 && d->ad_narrow) {
      rc0 = pack_adaptive(c, kCoarseBitsNarrow, &d->lut, &d->ad_K, &d->ad_E);
      d->ad_cbits = kCoarseBitsNarrow;
    }
    if (rc0) return rc0;
  } else {
    pack_lut(c.f, c.n, &d->lut);
  }
  d->finals = c.finals;
  d->heads.clear();
  d->tasks.clear();
  const uint64_t P = c.M - 1;
  recoil_plan &p = d->plan;
  std::memset(&p, 0, sizeof(p));
  p.task_begin = tb;
  p.task_end = te;
  p.prob_bits = c.n;
  uint64_t word_lo = 0, word_hi = 0;
  int64_t ss, bi;
  int rc;
  for (uint64_t t = tb; t < te; ++t) {
    if (c.N == 0) break;
    TaskHead h;
    std::memset(&h, 0, sizeof(h));
    h.task_id = (uint32_t)t;
    if (t < P) {
      h.cursor0 = (int32_t)0;  // set below (slice relative)
      h.start_group = (int32_t)c.maxg[t];
    } else {
      h.start_group = (int32_t)(c.G - 1);
      h.flags |= kHeadLast;
    }
    if (t > 0)
      h.maxg_prev = (uint32_t)c.maxg[t - 1];
    else
      h.flags |= kHeadFirst;
    d->heads.push_back(h);
  }
  if (!d->heads.empty()) {
    const uint64_t t_last = tb + d->heads.size() - 1;
    word_hi = (t_last < P ? c.offset[t_last] : c.B - 1) + 1;
    if (tb >= 2) {
      int64_t ss1, bi1, ss2, bi2;
      if ((rc = point_span_light(c, tb - 1, &ss1, &bi1)) || (rc = point_span_light(c, tb - 2, &ss2, &bi2))) return rc;
      if (ss1 > bi2 && c.offset[tb - 2] >= kLanes - 1) word_lo = c.offset[tb - 2] - (kLanes - 1);
    }
    if (tb > 0) {
      if ((rc = point_span_light(c, tb - 1, &ss, &bi))) return rc;
      p.out_lo = (uint64_t)ss;
    }
    uint64_t write_end;
    if (t_last < P) {
      if ((rc = point_span_light(c, t_last, &ss, &bi))) return rc;
      p.out_hi = (uint64_t)ss;
      write_end = kLanes * ((uint64_t)ss / kLanes + 1);
    } else {
      p.out_hi = c.N;
      write_end = (c.N + 15) & ~15ull;
    }
    p.out_base = p.out_lo & ~(uint64_t)(kBlockBytes - 1);
    p.out_count = ((std::max(write_end, p.out_hi) + 15) & ~15ull) - p.out_base;
  }
  word_lo &= ~(uint64_t)(kChunkWords - 1);
  word_hi = ceil_div(std::max(word_hi, word_lo + 1), kChunkWords) * kChunkWords;
  if (word_hi - word_lo >= (1ull << 31)) return RECOIL_E_UNSUPPORTED;  // 32-bit slice cursor
  p.word_lo = word_lo;
  p.word_count = word_hi - word_lo;
  // records needed: points [tb - 1, min(te, P)) (task t reads points t and t - 1)
  const uint64_t r0 = tb > 0 ? tb - 1 : 0, r1 = std::min<uint64_t>(te, P);
  d->rec_src = r1 > r0 ? c.rec_off[r0] : 0;
  d->rec_len = r1 > r0 ? c.rec_off[r1] - c.rec_off[r0] : 0;
  for (size_t i = 0; i < d->heads.size(); ++i) {
    TaskHead &h = d->heads[i];
    const uint64_t t = tb + i;
    h.cursor0 = (int32_t)((t < P ? (int64_t)c.offset[t] : (int64_t)c.B - 1) - (int64_t)word_lo);
    if (t < P) h.rec = (uint32_t)(c.rec_off[t] - d->rec_src);
    if (t > 0) h.rec_prev = (uint32_t)(c.rec_off[t - 1] - d->rec_src);
    if (h.flags & kHeadFirst) h.end_cursor = (int32_t)(-1 - (int64_t)word_lo);
  }
  d->n_tasks = (uint32_t)d->heads.size();
  p.n_tasks = d->n_tasks;
  p.symbol_bytes = c.adaptive ? 2 : 1;
  p.n_models = c.adaptive ? c.K : 1;
  p.coarse_bits = c.adaptive ? d->ad_cbits : 0;
  p.warps_per_block = c.adaptive ? (d->ad_narrow ? kWarpsAdaptiveNarrow : kWarpsAdaptive) : kWarpsStatic;
  d->lut_off = 16;
  d->finals_off = align16(d->lut_off + d->lut.size());
  d->tasks_off = align16(d->finals_off + 4 * d->finals.size());
  d->rec_off = align16(d->tasks_off + sizeof(TaskHead) * d->heads.size());
  p.workspace_bytes = align16(d->rec_off + d->rec_len + 256);  // + over-read pad of the record windows
  p.upload_bytes = (p.workspace_bytes - 16) + 2 * std::min<uint64_t>(p.word_count, c.B > word_lo ? c.B - word_lo : 0);
  return RECOIL_OK;
}

int build_decoder_from(std::shared_ptr<const Container> cptr, uint64_t task_begin, uint64_t task_end, Decoder *d,
                       bool for_gpu) {
  d->c = std::move(cptr);
  const Container &c = *d->c;
  if (task_end > c.M) task_end = c.M;
  if (task_begin > task_end) return RECOIL_E_ARG;
  // adaptive containers: GPU decode only (fused plan; recoil_decode_adaptive)
  if (c.adaptive && !(for_gpu && c.light)) return RECOIL_E_UNSUPPORTED;
  {
    int present = 0;
    for (int s = 0; s < 256; ++s)
      if (c.f[s]) {
        present++;
        d->single_symbol = s;
      }
    if (present != 1) d->single_symbol = -1;
  }
  if (for_gpu && !c.partitioned && c.light) return build_fused(d, task_begin, task_end);
  if (task_end > c.M) task_end = c.M;
  if (task_begin > task_end) return RECOIL_E_ARG;
  if (for_gpu && c.n > kMaxGpuProbBits) return RECOIL_E_UNSUPPORTED;
  int present = 0;
  for (int s = 0; s < 256; ++s)
    if (c.f[s]) {
      present++;
      d->single_symbol = s;
    }
  if (present != 1) d->single_symbol = -1;
  if (for_gpu) pack_lut(c.f, c.n, &d->lut);
  d->tasks.clear();
  d->finals.clear();
  std::vector<uint64_t> part_start;
  if (c.partitioned) {
    part_start.resize(c.M + 1, 0);
    for (uint32_t p = 0; p < c.M; ++p) part_start[p + 1] = part_start[p] + c.part_words[p];
  }
  for (uint64_t t = task_begin; t < task_end; ++t) {
    TaskRec r;
    std::memset(&r, 0, sizeof(r));
    r.task_id = (uint32_t)t;
    if (!c.partitioned) {
      const uint64_t lo = t > 0 ? (uint64_t)c.sync_start[t - 1] : 0;
      r.commit_lo = lo;
      r.end_cursor = lo == 0 ? -1 : kNoEndCheck;
      if (t + 1 < c.M) {
        const int64_t ss = c.sync_start[t];
        r.commit_hi = (uint64_t)ss - 1;
        r.write_hi = kLanes * ((uint64_t)ss / kLanes + 1);  // through the sync completion group
        r.cursor0 = (int64_t)c.offset[t];
        r.start_group = (int32_t)c.maxg[t];
        r.finals_idx = kNoFinals;
        for (uint32_t j = 0; j < kLanes; ++j)
          r.lanes[j] = c.state[t * kLanes + j] | ((uint32_t)c.gdiff[t * kLanes + j] << 16);
      } else {
        if (c.N == 0) continue;
        r.commit_hi = c.N - 1;
        r.write_hi = (c.N + 15) & ~15ull;
        r.cursor0 = (int64_t)c.B - 1;
        r.start_group = (int32_t)(c.G - 1);
        r.finals_idx = (uint32_t)(d->finals.size() / kLanes);
        d->finals.insert(d->finals.end(), c.finals.begin(), c.finals.end());
        for (uint32_t j = 0; j < kLanes; ++j) r.lanes[j] = (32 * (c.G - 1) + j < c.N ? 0u : 1u) << 16;
      }
    } else {
      uint64_t gl = t * c.G / c.M, gh = (t + 1) * c.G / c.M;
      uint64_t lo = kLanes * gl, hi = std::min<uint64_t>(c.N, kLanes * gh);
      if (lo >= hi) continue;  // empty partition
      r.commit_lo = lo;
      r.commit_hi = hi - 1;
      r.write_hi = (hi + 15) & ~15ull;
      r.cursor0 = (int64_t)(part_start[t] + c.part_words[t]) - 1;
      r.end_cursor = (int64_t)part_start[t] - 1;
      r.start_group = (int32_t)(gh - 1);
      r.finals_idx = (uint32_t)(d->finals.size() / kLanes);
      d->finals.insert(d->finals.end(), c.finals.begin() + t * kLanes, c.finals.begin() + (t + 1) * kLanes);
      for (uint32_t j = 0; j < kLanes; ++j) r.lanes[j] = (kLanes * (gh - 1) + j < hi ? 0u : 1u) << 16;
    }
    d->tasks.push_back(r);
  }
  // word slice [word_lo, word_hi): chunk aligned, padded
  recoil_plan &p = d->plan;
  std::memset(&p, 0, sizeof(p));
  p.task_begin = task_begin;
  p.task_end = task_end;
  p.n_tasks = (uint32_t)d->tasks.size();
  p.prob_bits = c.n;
  uint64_t word_lo = 0, word_hi = 0;
  if (!d->tasks.empty()) {
    int64_t mx = -1;
    for (const TaskRec &r : d->tasks) mx = std::max(mx, r.cursor0);
    word_hi = (uint64_t)(mx + 1);
    if (c.partitioned) {
      word_lo = part_start[task_begin];
    } else if (task_begin >= 2) {
      // task a reads no word below offset(point a-2) - 31 when sync_start(point a-1) >
      // boundary(point a-2) (reading Z9, enforced by the encoder); else start at 0.
      if (c.sync_start[task_begin - 1] > c.bidx[task_begin - 2] && c.offset[task_begin - 2] >= kLanes - 1)
        word_lo = c.offset[task_begin - 2] - (kLanes - 1);
    }
  }
  word_lo &= ~(uint64_t)(kChunkWords - 1);
  word_hi = ceil_div(std::max(word_hi, word_lo + 1), kChunkWords) * kChunkWords;
  if (for_gpu && word_hi - word_lo >= (1ull << 31)) return RECOIL_E_UNSUPPORTED;  // 32-bit slice cursor
  p.word_lo = word_lo;
  p.word_count = word_hi - word_lo;
  for (TaskRec &r : d->tasks) {
    r.cursor0 -= (int64_t)word_lo;
    if (r.end_cursor != kNoEndCheck) r.end_cursor -= (int64_t)word_lo;
  }
  if (!d->tasks.empty()) {
    p.out_lo = d->tasks.front().commit_lo;
    p.out_hi = d->tasks.back().commit_hi + 1;
  }
  p.out_base = p.out_lo & ~(uint64_t)(kBlockBytes - 1);
  uint64_t write_end = p.out_hi;
  for (const TaskRec &r : d->tasks) write_end = std::max(write_end, r.write_hi);
  p.out_count = ((write_end + 15) & ~15ull) - p.out_base;
  p.warps_per_block = kWarpsStatic;
  d->lut_off = 16;
  d->finals_off = align16(d->lut_off + d->lut.size());
  d->tasks_off = align16(d->finals_off + 4 * d->finals.size());
  d->n_tasks = (uint32_t)d->tasks.size();
  p.workspace_bytes = align16(d->tasks_off + sizeof(TaskRec) * d->tasks.size());
  p.symbol_bytes = 1;
  p.n_models = 1;
  p.upload_bytes = (p.workspace_bytes - 16) + 2 * std::min<uint64_t>(p.word_count, c.B > word_lo ? c.B - word_lo : 0);
  return RECOIL_OK;
}

}  // namespace recoil

using namespace recoil;

extern "C" int recoil_decoder_create(const uint8_t *container, uint64_t len, uint64_t task_begin,
                                     uint64_t task_end, recoil_decoder **out) {
  if (!container || !out) return RECOIL_E_ARG;
  *out = nullptr;
  try {
    Decoder *d = new Decoder();
    int rc = build_decoder(container, len, task_begin, task_end, d, true);
    if (rc) {
      delete d;
      return rc;
    }
    *out = reinterpret_cast<recoil_decoder *>(d);
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

namespace recoil {
namespace {

// Parse for a decoder-side combine: the full parse (host-expanded task records, the default
// GPU plan) for static containers, the light parse (fused plan) for adaptive ones.
int parse_for_subset(const uint8_t *container, uint64_t len, std::shared_ptr<Container> *out) {
  auto full = std::make_shared<Container>();
  const bool adaptive = container && len >= 4 && std::memcmp(container, "RCA1", 4) == 0;
  int rc = parse_container(container, len, full.get(), /*light=*/adaptive);
  if (rc) return rc;
  if (full->partitioned) return RECOIL_E_ARG;  // partitions cannot be combined
  *out = std::move(full);
  return RECOIL_OK;
}

// The container viewed with only the split points `keep` (ascending point indices): the
// decode runs through the dropped points.  Full parse: the kept points' anchors,
// differences and spans; light parse: their record offsets (rec_off[j + 1] bounds kept record
// j's bytes: the next kept record, a looser but valid bound; the last bound is the last kept
// record's end).
std::shared_ptr<Container> select_points(const Container &full, const std::vector<uint64_t> &keep) {
  auto view = std::make_shared<Container>(full);
  const uint32_t W = full.W;
  view->offset.clear();
  view->maxg.clear();
  view->rec_off.clear();
  view->state.clear();
  view->gdiff.clear();
  view->sync_start.clear();
  view->bidx.clear();
  for (uint64_t k : keep) {
    view->offset.push_back(full.offset[k]);
    view->maxg.push_back(full.maxg[k]);
    if (full.light) {
      view->rec_off.push_back(full.rec_off[k]);
    } else {
      view->state.insert(view->state.end(), full.state.begin() + k * W, full.state.begin() + (k + 1) * W);
      view->gdiff.insert(view->gdiff.end(), full.gdiff.begin() + k * W, full.gdiff.begin() + (k + 1) * W);
      view->sync_start.push_back(full.sync_start[k]);
      view->bidx.push_back(full.bidx[k]);
    }
  }
  if (full.light) view->rec_off.push_back(keep.empty() ? full.rec_off[0] : full.rec_off[keep.back() + 1]);
  view->M = (uint32_t)keep.size() + 1;
  return view;
}

int finish_decoder(std::shared_ptr<const Container> view, uint64_t tb, uint64_t te, recoil_decoder **out) {
  Decoder *d = new Decoder();
  int rc = build_decoder_from(std::move(view), tb, te, d, true);
  if (rc) {
    delete d;
    return rc;
  }
  *out = reinterpret_cast<recoil_decoder *>(d);
  return RECOIL_OK;
}

// the split points recoil_combine_splits(c, target) keeps: 1-based positions k, 2k, ...
std::vector<uint64_t> combine_keep(const Container &c, uint32_t target) {
  std::vector<uint64_t> keep;
  const uint64_t P = c.M - 1;
  if (target >= c.M) {
    for (uint64_t k = 0; k < P; ++k) keep.push_back(k);
  } else {
    const uint64_t step = ceil_div(c.M, target);
    for (uint64_t pos = step; pos <= P; pos += step) keep.push_back(pos - 1);
  }
  return keep;
}

}  // namespace
}  // namespace recoil

extern "C" int recoil_decoder_create_subset(const uint8_t *container, uint64_t len, uint32_t target_splits,
                                            uint64_t task_begin, uint64_t task_end, recoil_decoder **out) {
  if (!container || !out || target_splits < 1) return RECOIL_E_ARG;
  *out = nullptr;
  try {
    std::shared_ptr<Container> full;
    int rc = parse_for_subset(container, len, &full);
    if (rc) return rc;
    return finish_decoder(select_points(*full, combine_keep(*full, target_splits)), task_begin, task_end, out);
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_decoder_create_for_device(const uint8_t *container, uint64_t len, int device, uint32_t waves_x100,
                                                recoil_decoder **out) {
  if (!container || !out || len < 8) return RECOIL_E_ARG;
  *out = nullptr;
  try {
    std::shared_ptr<Container> full;
    int rc = parse_for_subset(container, len, &full);
    if (rc) return rc;
    int warps = 0, sms = 0;
    if (full->adaptive) {
      uint64_t e = 0;
      for (uint32_t k = 0; k < full->K; ++k) e += full->mlen[k];
      rc = recoil_decode_occupancy_adaptive(device, full->K, e, &warps, &sms);
    } else {
      rc = recoil_decode_occupancy(device, full->n, &warps, &sms);
    }
    if (rc) return rc;
    const uint64_t target = std::max<uint64_t>(1, (uint64_t)warps * sms * (waves_x100 ? waves_x100 : 150) / 100);
    return finish_decoder(select_points(*full, combine_keep(*full, (uint32_t)std::min<uint64_t>(target, full->M))),
                          0, UINT64_MAX, out);
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_decoder_create_grouped(const uint8_t *container, uint64_t len, uint32_t n_runs,
                                             const uint32_t *run_tasks, const uint32_t *run_splits,
                                             recoil_decoder **out) {
  if (!container || !out || n_runs < 1 || !run_tasks || !run_splits) return RECOIL_E_ARG;
  *out = nullptr;
  try {
    std::shared_ptr<Container> full;
    int rc = parse_for_subset(container, len, &full);
    if (rc) return rc;
    for (uint32_t r = 0; r < n_runs; ++r)
      if (run_splits[r] == 0) return RECOIL_E_ARG;
    // task i spans run_splits[r] consecutive encoder splits (segments) for the run r it
    // falls in; the point after its last segment is kept, every other point is dropped
    // (the decode runs through it); the last task takes the segments that remain
    const uint64_t P = full->M - 1;
    std::vector<uint64_t> keep;
    uint64_t seg = 0;
    for (uint32_t r = 0; r < n_runs; ++r)
      for (uint32_t i = 0; i < run_tasks[r]; ++i) {
        seg += run_splits[r];
        if (seg > P) break;
        keep.push_back(seg - 1);  // point k closes segment k
      }
    return finish_decoder(select_points(*full, keep), 0, UINT64_MAX, out);
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_decoder_plan(const recoil_decoder *dec, recoil_plan *plan) {
  if (!dec || !plan) return RECOIL_E_ARG;
  *plan = reinterpret_cast<const Decoder *>(dec)->plan;
  return RECOIL_OK;
}

extern "C" void recoil_decoder_destroy(recoil_decoder *dec) { delete reinterpret_cast<Decoder *>(dec); }

namespace recoil {

void shard_bounds_range(const Container &c, uint64_t tb, uint64_t te, uint32_t n_shards, uint64_t *bounds) {
  // shard s starts at the first task whose start reaches lo(tb) + s (lo(te) - lo(tb)) / n
  // balance on the anchor group of the entry point below each task (within one
  // Synchronization Section of the committed start; available from a light parse)
  auto lo_of = [&](uint64_t t) -> uint64_t {
    if (t >= c.M) return c.N;
    if (c.partitioned) return kLanes * (t * c.G / c.M);
    return t == 0 ? 0 : kLanes * c.maxg[t - 1];
  };
  te = std::min<uint64_t>(te, c.M);
  tb = std::min(tb, te);
  std::vector<uint64_t> lo(te - tb);
  for (uint64_t t = tb; t < te; ++t) lo[t - tb] = lo_of(t);
  const uint64_t a = lo_of(tb), span = lo_of(te) - a;
  bounds[0] = tb;
  for (uint32_t s = 1; s < n_shards; ++s) {
    uint64_t target = a + ceil_div((uint64_t)s * span, n_shards);
    uint64_t b = tb + (uint64_t)(std::lower_bound(lo.begin(), lo.end(), target) - lo.begin());
    bounds[s] = std::max(bounds[s - 1], std::min<uint64_t>(b, te));
  }
  bounds[n_shards] = te;
}

void shard_bounds(const Container &c, uint32_t n_shards, uint64_t *bounds) {
  shard_bounds_range(c, 0, c.M, n_shards, bounds);
}

}  // namespace recoil

extern "C" int recoil_shard_plan(const uint8_t *container, uint64_t len, uint32_t n_shards,
                                 uint64_t *bounds) {
  if (!container || !bounds || n_shards < 1) return RECOIL_E_ARG;
  try {
    recoil::Container c;
    int rc = recoil::parse_container(container, len, &c);
    if (rc) return rc;
    recoil::shard_bounds(c, n_shards, bounds);
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}
