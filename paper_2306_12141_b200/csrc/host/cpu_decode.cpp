// cpu_decode.cpp -- multithreaded host decoder (baseline, NOT a fallback of the
// GPU path): the same task table as the GPU kernel, one task per split, one
// thread per core (P:429 recommends no SMT).  Decodes Recoil and partitioned
// containers for any 1 <= n <= 16.  Three task decoders (NEXT row 3; the
// paper's CPU decoders are AVX2 8-way x 4 and AVX-512 16-way x 2):
//  - scalar;
//  - AVX-512: the 32 lanes are two 16 x u32 vectors, the refill of a group is
//    one masked expand-load of the needing lanes' words (ascending lanes take
//    ascending words, i.e. the interleaved decreasing-lane read order of P:168);
//  - AVX2: four 8 x u32 vectors; per vector one 16-byte load of the words its
//    needing lanes take (a contiguous run below the cursor) and a permutation
//    from a 256-entry table indexed by the needing-lane mask;
// in both SIMD decoders the symbol lookup is a gather from the LUT.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <new>
#include <thread>

#include "../recoil_internal.h"

namespace recoil {
namespace {

struct Tables {
  std::vector<uint8_t> sym;
  std::vector<uint32_t> f, bias;
  std::vector<uint32_t> fb, symw;  // AVX-512: f | bias << 16 and the symbol, per slot (u32 for gathers)
};

int decode_task(const Decoder &d, const Tables &tb, const TaskRec &t, const uint16_t *w, uint8_t *out) {
  const uint32_t n = d.c->n, mask = (1u << n) - 1;
  uint32_t x[32], st[32];
  int32_t ig[32];
  bool inited[32];
  for (uint32_t j = 0; j < kLanes; ++j) {
    st[j] = t.finals_idx == kNoFinals ? (t.lanes[j] & 0xFFFF) : d.finals[t.finals_idx * kLanes + j];
    ig[j] = t.start_group - (int32_t)(t.lanes[j] >> 16);
    inited[j] = false;
    x[j] = 0;
  }
  int64_t cur = t.cursor0;
  const int64_t lo_group = (int64_t)(t.commit_lo / kLanes);
  const uint64_t out_base = d.plan.out_base;
  for (int64_t g = t.start_group; g >= lo_group; --g) {
    for (int32_t j = kLanes - 1; j >= 0; --j) {  // refill, decreasing lane
      if (!inited[j] && g == ig[j]) {
        x[j] = st[j];
        inited[j] = true;
      }
      if (inited[j] && x[j] < kL) {
        if (cur < 0) return RECOIL_E_UNDERFLOW;
        x[j] = (x[j] << kWordBits) | w[cur--];
      }
    }
    const uint64_t base = (uint64_t)g * kLanes;
    for (uint32_t j = 0; j < kLanes; ++j) {
      if (!inited[j]) continue;
      uint32_t slot = x[j] & mask;
      x[j] = tb.f[slot] * (x[j] >> n) + tb.bias[slot];
      uint64_t i = base + j;
      if (i >= t.commit_lo && i <= t.commit_hi) out[i - out_base] = tb.sym[slot];
    }
  }
  if (t.end_cursor != kNoEndCheck) {
    // reached the codec's first symbol: outputs emitted before group 0 (n = 16, f = 1)
    for (int32_t j = kLanes - 1; j >= 0; --j)
      if (inited[j] && x[j] < kL) {
        if (cur < 0) return RECOIL_E_UNDERFLOW;
        x[j] = (x[j] << kWordBits) | w[cur--];
      }
    if (cur != t.end_cursor) return RECOIL_E_SYNC;
    for (uint32_t j = 0; j < kLanes; ++j)
      if (inited[j] && x[j] != kL) return RECOIL_E_SYNC;
  }
  return RECOIL_OK;
}

// One group's refill (Eq. 4 renormalisation, P:168 read order): lanes with
// x < L, in decreasing lane order, each take the next word below the cursor;
// the expand-load hands the lowest of the `total` words to the lowest lane.
__attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi2,popcnt"))) inline bool simd_refill(
    __m512i &x0, __m512i &x1, int64_t &cur, const uint16_t *w) {
  const __m512i vL = _mm512_set1_epi32((int)kL);
  const __mmask16 k0 = _mm512_cmplt_epu32_mask(x0, vL), k1 = _mm512_cmplt_epu32_mask(x1, vL);
  const uint32_t m = (uint32_t)k0 | ((uint32_t)k1 << 16);
  const int total = __builtin_popcount(m);
  if (!total) return true;
  if (cur - total + 1 < 0) return false;
  const __m512i wv = _mm512_maskz_expandloadu_epi16(m, w + (cur - total + 1));
  const __m512i w0 = _mm512_cvtepu16_epi32(_mm512_castsi512_si256(wv));
  const __m512i w1 = _mm512_cvtepu16_epi32(_mm512_extracti64x4_epi64(wv, 1));
  x0 = _mm512_mask_or_epi32(x0, k0, _mm512_slli_epi32(x0, 16), w0);
  x1 = _mm512_mask_or_epi32(x1, k1, _mm512_slli_epi32(x1, 16), w1);
  cur -= total;
  return true;
}

__attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi2,popcnt")))
int decode_task_avx512(const Decoder &d, const Tables &tb, const TaskRec &t, const uint16_t *w, uint8_t *out) {
  const uint32_t n = d.c->n;
  const __m512i vmask = _mm512_set1_epi32((int)((1u << n) - 1)), vL = _mm512_set1_epi32((int)kL);
  const __m512i v16 = _mm512_set1_epi32(0xFFFF), vall = _mm512_set1_epi32(-1);
  const __m128i vn = _mm_cvtsi32_si128((int)n);
  alignas(64) uint32_t st[32];
  alignas(64) int32_t ig[32];
  for (uint32_t j = 0; j < kLanes; ++j) {
    st[j] = t.finals_idx == kNoFinals ? (t.lanes[j] & 0xFFFF) : d.finals[t.finals_idx * kLanes + j];
    ig[j] = t.start_group - (int32_t)(t.lanes[j] >> 16);
  }
  const __m512i st0 = _mm512_load_si512(st), st1 = _mm512_load_si512(st + 16);
  const __m512i ig0 = _mm512_load_si512(ig), ig1 = _mm512_load_si512(ig + 16);
  __m512i x0 = vall, x1 = vall;  // uninitialised lanes: never < L
  __mmask16 in0 = 0, in1 = 0;
  int64_t cur = t.cursor0;
  const int64_t lo_group = (int64_t)(t.commit_lo / kLanes);
  const uint64_t out_base = d.plan.out_base;
  for (int64_t g = t.start_group; g >= lo_group; --g) {
    const __m512i gv = _mm512_set1_epi32((int)g);
    const __mmask16 i0 = _mm512_cmpeq_epi32_mask(ig0, gv), i1 = _mm512_cmpeq_epi32_mask(ig1, gv);
    x0 = _mm512_mask_mov_epi32(x0, i0, st0);
    x1 = _mm512_mask_mov_epi32(x1, i1, st1);
    in0 |= i0;
    in1 |= i1;
    if (!simd_refill(x0, x1, cur, w)) return RECOIL_E_UNDERFLOW;
    const __m512i s0 = _mm512_and_si512(x0, vmask), s1 = _mm512_and_si512(x1, vmask);
    __m512i y0, y1, sym0, sym1;
    if (n <= 12) {  // packed s | bias << 8 | f << 20
      const __m512i e0 = _mm512_i32gather_epi32(s0, tb.fb.data(), 4), e1 = _mm512_i32gather_epi32(s1, tb.fb.data(), 4);
      sym0 = e0;
      sym1 = e1;
      const __m512i b0 = _mm512_and_si512(_mm512_srli_epi32(e0, 8), _mm512_set1_epi32(0xFFF));
      const __m512i b1 = _mm512_and_si512(_mm512_srli_epi32(e1, 8), _mm512_set1_epi32(0xFFF));
      y0 = _mm512_add_epi32(_mm512_mullo_epi32(_mm512_srli_epi32(e0, 20), _mm512_srl_epi32(x0, vn)), b0);
      y1 = _mm512_add_epi32(_mm512_mullo_epi32(_mm512_srli_epi32(e1, 20), _mm512_srl_epi32(x1, vn)), b1);
    } else {  // f | bias << 16, symbol separately
      const __m512i e0 = _mm512_i32gather_epi32(s0, tb.fb.data(), 4), e1 = _mm512_i32gather_epi32(s1, tb.fb.data(), 4);
      sym0 = _mm512_i32gather_epi32(s0, tb.symw.data(), 4);
      sym1 = _mm512_i32gather_epi32(s1, tb.symw.data(), 4);
      y0 = _mm512_add_epi32(_mm512_mullo_epi32(_mm512_and_si512(e0, v16), _mm512_srl_epi32(x0, vn)),
                            _mm512_srli_epi32(e0, 16));
      y1 = _mm512_add_epi32(_mm512_mullo_epi32(_mm512_and_si512(e1, v16), _mm512_srl_epi32(x1, vn)),
                            _mm512_srli_epi32(e1, 16));
    }
    x0 = _mm512_mask_mov_epi32(x0, in0, y0);
    x1 = _mm512_mask_mov_epi32(x1, in1, y1);
    const uint64_t i0s = (uint64_t)g * kLanes;
    if (i0s + 31 < t.commit_lo || i0s > t.commit_hi) continue;
    const __m128i b0 = _mm512_cvtepi32_epi8(sym0), b1 = _mm512_cvtepi32_epi8(sym1);
    uint8_t *dst = out + (i0s - out_base);
    if (i0s >= t.commit_lo && i0s + 31 <= t.commit_hi) {
      _mm_storeu_si128(reinterpret_cast<__m128i *>(dst), b0);
      _mm_storeu_si128(reinterpret_cast<__m128i *>(dst + 16), b1);
    } else {
      uint32_t keep = 0;
      for (uint32_t j = 0; j < kLanes; ++j)
        if (i0s + j >= t.commit_lo && i0s + j <= t.commit_hi) keep |= 1u << j;
      _mm_mask_storeu_epi8(dst, (__mmask16)(keep & 0xFFFF), b0);
      _mm_mask_storeu_epi8(dst + 16, (__mmask16)(keep >> 16), b1);
    }
  }
  if (t.end_cursor != kNoEndCheck) {
    if (!simd_refill(x0, x1, cur, w)) return RECOIL_E_UNDERFLOW;  // outputs emitted before group 0 (n = 16, f = 1)
    if (cur != t.end_cursor) return RECOIL_E_SYNC;
    const __mmask16 ok0 = _mm512_cmpeq_epi32_mask(x0, vL), ok1 = _mm512_cmpeq_epi32_mask(x1, vL);
    if ((ok0 & in0) != in0 || (ok1 & in1) != in1) return RECOIL_E_SYNC;
  }
  return RECOIL_OK;
}

// AVX2 refill (P:168 read order): vector v holds lanes 8v..8v+7; the vectors are
// visited from the highest lanes down, and the c needing lanes of a vector take the
// c words just below the cursor, ascending lane <- ascending word.
struct Avx2Perm {
  alignas(32) uint32_t idx[256][8];  // needing-lane mask -> for each lane, its rank among the needing lanes
  Avx2Perm() {
    for (uint32_t m = 0; m < 256; ++m)
      for (uint32_t j = 0; j < 8; ++j) idx[m][j] = (uint32_t)__builtin_popcount(m & ((1u << j) - 1)) & 7u;
  }
};
const Avx2Perm &avx2_perm() {
  static const Avx2Perm p;
  return p;
}

__attribute__((target("avx2,popcnt"))) inline bool avx2_refill(__m256i x[4], int64_t &cur, const uint16_t *w,
                                                               const Avx2Perm &pm) {
  for (int v = 3; v >= 0; --v) {
    const __m256i need = _mm256_cmpeq_epi32(_mm256_srli_epi32(x[v], 16), _mm256_setzero_si256());  // x < L = 2^16
    const uint32_t m = (uint32_t)_mm256_movemask_ps(_mm256_castsi256_ps(need));
    if (!m) continue;
    const int c = __builtin_popcount(m);
    if (cur - c + 1 < 0) return false;
    // words [cur - c + 1, cur - c + 8]: the container copy has 8 words of padding past B
    const __m256i wv = _mm256_cvtepu16_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i *>(w + (cur - c + 1))));
    const __m256i pw = _mm256_permutevar8x32_epi32(wv, _mm256_load_si256(reinterpret_cast<const __m256i *>(pm.idx[m])));
    x[v] = _mm256_blendv_epi8(x[v], _mm256_or_si256(_mm256_slli_epi32(x[v], 16), pw), need);
    cur -= c;
  }
  return true;
}

__attribute__((target("avx2,popcnt")))
int decode_task_avx2(const Decoder &d, const Tables &tb, const TaskRec &t, const uint16_t *w, uint8_t *out) {
  const uint32_t n = d.c->n;
  const Avx2Perm &pm = avx2_perm();
  const __m256i vmask = _mm256_set1_epi32((int)((1u << n) - 1)), vL = _mm256_set1_epi32((int)kL);
  const __m256i v16 = _mm256_set1_epi32(0xFFFF), v12 = _mm256_set1_epi32(0xFFF), vff = _mm256_set1_epi32(0xFF);
  const __m128i vn = _mm_cvtsi32_si128((int)n);
  const __m256i order = _mm256_setr_epi32(0, 4, 1, 5, 2, 6, 3, 7);
  alignas(32) uint32_t st[32];
  alignas(32) int32_t ig[32];
  for (uint32_t j = 0; j < kLanes; ++j) {
    st[j] = t.finals_idx == kNoFinals ? (t.lanes[j] & 0xFFFF) : d.finals[t.finals_idx * kLanes + j];
    ig[j] = t.start_group - (int32_t)(t.lanes[j] >> 16);
  }
  __m256i x[4], stv[4], igv[4], in[4];
  for (int v = 0; v < 4; ++v) {
    stv[v] = _mm256_load_si256(reinterpret_cast<const __m256i *>(st + 8 * v));
    igv[v] = _mm256_load_si256(reinterpret_cast<const __m256i *>(ig + 8 * v));
    x[v] = _mm256_set1_epi32(-1);  // uninitialised lanes: never < L
    in[v] = _mm256_setzero_si256();
  }
  int64_t cur = t.cursor0;
  const int64_t lo_group = (int64_t)(t.commit_lo / kLanes);
  const uint64_t out_base = d.plan.out_base;
  for (int64_t g = t.start_group; g >= lo_group; --g) {
    const __m256i gv = _mm256_set1_epi32((int)g);
    for (int v = 0; v < 4; ++v) {
      const __m256i now = _mm256_cmpeq_epi32(igv[v], gv);
      x[v] = _mm256_blendv_epi8(x[v], stv[v], now);
      in[v] = _mm256_or_si256(in[v], now);
    }
    if (!avx2_refill(x, cur, w, pm)) return RECOIL_E_UNDERFLOW;
    __m256i sym[4];
    for (int v = 0; v < 4; ++v) {
      const __m256i slot = _mm256_and_si256(x[v], vmask);
      const __m256i e = _mm256_i32gather_epi32(reinterpret_cast<const int *>(tb.fb.data()), slot, 4);
      __m256i y;
      if (n <= 12) {  // packed s | bias << 8 | f << 20
        sym[v] = _mm256_and_si256(e, vff);
        y = _mm256_add_epi32(_mm256_mullo_epi32(_mm256_srli_epi32(e, 20), _mm256_srl_epi32(x[v], vn)),
                             _mm256_and_si256(_mm256_srli_epi32(e, 8), v12));
      } else {  // f | bias << 16, symbol separately
        sym[v] = _mm256_i32gather_epi32(reinterpret_cast<const int *>(tb.symw.data()), slot, 4);
        y = _mm256_add_epi32(_mm256_mullo_epi32(_mm256_and_si256(e, v16), _mm256_srl_epi32(x[v], vn)),
                             _mm256_srli_epi32(e, 16));
      }
      x[v] = _mm256_blendv_epi8(x[v], y, in[v]);
    }
    const uint64_t i0s = (uint64_t)g * kLanes;
    if (i0s + 31 < t.commit_lo || i0s > t.commit_hi) continue;
    // 32 symbols (u32) -> 32 bytes in lane order
    const __m256i p = _mm256_packus_epi16(_mm256_packus_epi32(sym[0], sym[1]), _mm256_packus_epi32(sym[2], sym[3]));
    const __m256i bytes = _mm256_permutevar8x32_epi32(p, order);
    uint8_t *dst = out + (i0s - out_base);
    if (i0s >= t.commit_lo && i0s + 31 <= t.commit_hi) {
      _mm256_storeu_si256(reinterpret_cast<__m256i *>(dst), bytes);
    } else {
      alignas(32) uint8_t b[32];
      _mm256_store_si256(reinterpret_cast<__m256i *>(b), bytes);
      for (uint32_t j = 0; j < kLanes; ++j)
        if (i0s + j >= t.commit_lo && i0s + j <= t.commit_hi) dst[j] = b[j];
    }
  }
  if (t.end_cursor != kNoEndCheck) {
    if (!avx2_refill(x, cur, w, pm)) return RECOIL_E_UNDERFLOW;  // outputs emitted before group 0 (n = 16, f = 1)
    if (cur != t.end_cursor) return RECOIL_E_SYNC;
    for (int v = 0; v < 4; ++v) {
      const __m256i bad = _mm256_andnot_si256(_mm256_cmpeq_epi32(x[v], vL), in[v]);
      if (!_mm256_testz_si256(bad, bad)) return RECOIL_E_SYNC;
    }
  }
  return RECOIL_OK;
}

bool have_avx2() {
  static const bool ok = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("popcnt");
  return ok;
}

bool have_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                         __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512vbmi2");
  return ok;
}

}  // namespace
}  // namespace recoil

using namespace recoil;

extern "C" int recoil_decode_cpu_ex(const uint8_t *container, uint64_t len, uint8_t *out, uint32_t threads,
                                    uint32_t flags) {
  if (!container) return RECOIL_E_ARG;
  try {
    Decoder d;
    int rc = build_decoder(container, len, 0, UINT64_MAX, &d, false);
    if (rc) return rc;
    if (d.c->N == 0) return RECOIL_OK;
    if (!out) return RECOIL_E_ARG;
    if (d.single_symbol >= 0) {
      std::memset(out, d.single_symbol, d.c->N);
      return RECOIL_OK;
    }
    Tables tb;
    const uint32_t n = d.c->n;
    // ISA: AVX-512 when the CPU has it, else AVX2; RECOIL_CPU_AVX2 forces AVX2, RECOIL_CPU_SCALAR scalar
    const int isa = (flags & RECOIL_CPU_SCALAR) ? 0 : (!(flags & RECOIL_CPU_AVX2) && have_avx512()) ? 2
                                                                                                   : have_avx2() ? 1 : 0;
    if ((flags & RECOIL_CPU_AVX2) && !(flags & RECOIL_CPU_SCALAR) && !have_avx2()) return RECOIL_E_UNSUPPORTED;
    const bool simd = isa != 0;
    tb.sym.resize(1u << n);
    tb.f.resize(1u << n);
    tb.bias.resize(1u << n);
    if (simd) {
      tb.fb.resize(1u << n);
      if (n > 12) tb.symw.resize(1u << n);
    }
    uint32_t F = 0;
    for (uint32_t s = 0; s < 256; ++s) {
      for (uint32_t k = 0; k < d.c->f[s]; ++k) {
        tb.sym[F + k] = (uint8_t)s;
        tb.f[F + k] = d.c->f[s];
        tb.bias[F + k] = k;
        if (simd) {
          if (n <= 12)
            tb.fb[F + k] = s | (k << 8) | (d.c->f[s] << 20);
          else {
            tb.fb[F + k] = (d.c->f[s] & 0xFFFFu) | (k << 16);
            tb.symw[F + k] = s;
          }
        }
      }
      F += d.c->f[s];
    }
    // the container's words as a host u16 array (little-endian host)
    std::vector<uint16_t> w(d.c->B + 16);  // + padding: the AVX2 refill loads 8 words at a time
    if (d.c->B) std::memcpy(w.data(), d.c->words, 2 * d.c->B);
    const uint16_t *slice = w.data() + d.plan.word_lo;
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    threads = std::min<uint32_t>(threads, (uint32_t)std::max<size_t>(1, d.tasks.size()));
    std::atomic<size_t> next{0};
    std::atomic<int> err{RECOIL_OK};
    auto worker = [&]() {
      for (size_t k; (k = next.fetch_add(1)) < d.tasks.size() && err.load() == RECOIL_OK;) {
        int r = isa == 2   ? decode_task_avx512(d, tb, d.tasks[k], slice, out)
                : isa == 1 ? decode_task_avx2(d, tb, d.tasks[k], slice, out)
                           : decode_task(d, tb, d.tasks[k], slice, out);
        if (r) err.store(r);
      }
    };
    std::vector<std::thread> pool;
    for (uint32_t i = 1; i < threads; ++i) pool.emplace_back(worker);
    worker();
    for (auto &th : pool) th.join();
    return err.load();
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_decode_cpu(const uint8_t *container, uint64_t len, uint8_t *out, uint32_t threads) {
  return recoil_decode_cpu_ex(container, len, out, threads, 0);
}

extern "C" int recoil_cpu_simd(void) { return have_avx512() ? 2 : have_avx2() ? 1 : 0; }
