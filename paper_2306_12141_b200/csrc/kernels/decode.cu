// decode.cu -- the Recoil decode kernel for sm_100a and its C-ABI entry points
// (recoil_decoder_upload / recoil_decode / recoil_decoder_status /
// recoil_decode_occupancy / recoil_decoder_launches).
//
// One warp per split task (a 32-way interleaved group "naturally fits
// into a GPU warp"); lane j is interleaved decoder D_j.  Per symbol group g
// (32 symbols, one per lane), top-down:
//   refill  (Eq. 4): lanes with x < L read one 16-bit word, in
//           decreasing lane order: m = ballot(x < L), lane j reads
//           word[cursor + 1 - popc(m & lanes_at_or_above_j)], cursor -= the
//           warp maximum of that count (REDUX.MAX: lane 0's count = popc(m));
//   decode  (Eq. 2): e = lut[x mod 2^n] from the shared-memory
//           packed LUT (s | bias << 8 | f << 20; n <= 11: four
//           bank-interleaved copies, one per 8 lanes), x = f (x >> n) + bias.
// Synchronization Phase: a lane is initialised with its 16-bit
// anchor state in its anchor group, immediately before its first read;
// uninitialised lanes hold 0xFFFFFFFF (never < L, so they never read) and
// their decodes are discarded.  The Decoding and Cross-Boundary phases
// are the same loop with every lane initialised, down to the
// group of the task's commit_lo; that steady state runs as fully unrolled
// 16-group blocks (one 512-byte output block each) with no per-group branch.
//
// Memory path: the words come from a per-warp 2 KB shared-memory ring filled
// by warp-cooperative 16-byte cp.async loads (256 words per chunk; chunks c,
// c-1, c-2 resident and c-3 in flight, checked once per 16-group block since 16
// groups consume <= 512 words); Recoil task heads and raw split records are
// loaded one block before a task starts and expanded in the kernel (row a1),
// prebuilt records (partitioned containers) stream in by cp.async; tasks are
// handed out by an atomic counter (persistent warps, 2 CTAs of 24 warps per
// SM).  Output: in whole 16-group blocks of the static codec (n <= 12) and the
// adaptive codec each group's 32 symbols go straight to HBM as one warp store (full
// 32-B sectors: no staging wavefronts, measured +2 % over staging);
// the partial blocks at a task's edges (and n >= 13) stage a 512-symbol block in
// shared memory and write each lane's 16 S bytes with 16-byte stores inside the
// task's write window.  All shared accesses use 32-bit shared-window addresses
// (inline PTX) computed once per warp.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>
#include <cstring>

#include "../recoil_internal.h"

namespace recoil {
namespace dev {
#ifdef RECOIL_CHECK_BOUNDS
__device__ unsigned long long g_oob;  // output stores outside the plan's buffer (debug builds)
#endif

// Warps per block.  The SM's warp schedulers favour older CTAs: with one task
// per warp, the warps of the last-resident CTA get issue slots only when the
// others stall and finish last (measured per task with -DRECOIL_TIMELINE: CTA
// rank 0..5 of an SM at 8 warps took 55 / 59 / 66 / 77 / 90 / 101 us of a 104 us
// decode, warps of one CTA alike).  So the static kernels run 2 CTAs of 24 warps
// (48 warps per SM, two priority levels; config 2: 989 -> 1082 GB/s, config 3
// 1277 -> 1324); the adaptive kernel runs one CTA of 32 warps (8-warp CTAs
// when its model tables leave no room for that layout).
#ifndef RECOIL_WARPS
#define RECOIL_WARPS kWarpsStatic
#endif
#ifndef RECOIL_WARPS_ADAPTIVE
#define RECOIL_WARPS_ADAPTIVE kWarpsAdaptive
#endif
// NB = 0 and NB = -1 are the adaptive codec (NEXT rows 1 + 4: index-keyed
// models, 16-bit symbols, n at run time; model tables in dynamic shared memory):
// one CTA of 32 warps per SM (2^25 latent symbols: 194 G symbols/s, against 184
// at 2 x 16 warps and 165 at 3 x 8), or, when the tables leave no room for that
// layout, 8-warp CTAs (NB = -1).
template <int NB>
__host__ __device__ constexpr int warps_per_block() {
  return NB == 0 ? (int)RECOIL_WARPS_ADAPTIVE : NB < 0 ? (int)kWarpsAdaptiveNarrow : (int)RECOIL_WARPS;
}
template <int NB>
__host__ __device__ constexpr int threads_per_block() { return 32 * warps_per_block<NB>(); }
// Resident warps per SM the register budget is sized for.  The steady state is
// bound by the shared-memory pipe and the latency of the per-group dependency
// chain, so more warps help: n <= 12 runs 48 warps (2 CTAs, 40 registers; at 8-warp
// CTAs, 56 warps at 32 registers measured 11 % slower, 40 warps 6 % slower);
// n >= 13 (up to 64 KB symbol table) is shared-memory limited to one CTA.
#ifndef RECOIL_MIN_WARPS
#define RECOIL_MIN_WARPS 48
#endif
template <int NB>
__host__ __device__ constexpr int min_blocks() {
  constexpr int w = warps_per_block<NB>();
  return NB <= 0 ? (32 / w > 0 ? 32 / w : 1) : NB <= 12 ? (RECOIL_MIN_WARPS / w > 0 ? RECOIL_MIN_WARPS / w : 1)
                                                       : (40 / w > 0 ? 40 / w : 1);
}
template <int NB>
__host__ __device__ constexpr int sym_bytes() { return NB <= 0 ? 2 : 1; }
constexpr int kRingChunks = 4;
constexpr int kRingWords = kRingChunks * (int)kChunkWords;  // 1024 words = 2 KB per warp
constexpr uint32_t kRingBytes = 2 * kRingWords;
constexpr uint32_t kFull = 0xFFFFFFFFu;

struct Params {
  const uint8_t *lut;     // n <= 12: 2^n packed u32; n >= 13: 2^n symbol bytes + 256 x u32 (f | F << 16)
  const uint32_t *finals;
  const TaskRec *tasks;   // prebuilt records (partitioned containers)
  const TaskHead *heads;  // fused a1 (Recoil): task heads ...
  const uint8_t *recs;    // ... and the raw split records they point into
  uint32_t N_lo, N_hi;    // N (symbols) as two words
  int32_t G;              // symbol groups
  DeviceStatus *status;
  const uint16_t *words;  // slice base (stream word word_lo)
  uint8_t *out;           // symbol out_base
  uint64_t out_base;
  uint64_t out_lim;       // out_base + out_count: no task writes at or beyond this symbol
  int32_t n_chunks;       // slice words / 256
  uint32_t n_tasks;
  // Runtime constants, opaque to ptxas, that keep some steady-state work on the
  // FMA pipe (IMAD) instead of the ALU pipe, which is the busiest one:
  int32_t neg2;           // -2: cursor arithmetic as IMAD instead of IADD3
  int32_t kneg4096;       // -2^12: see Warp::decode
  // adaptive codec (NB = 0): model id of every symbol (absolute index, 16-B
  // aligned), model count, table entries, n
  const uint8_t *mid;
  uint32_t ad_K, ad_E, nbits, ad_cbits, ad_crow;  // + coarse bucket bits, u16 row length
};

// Shared memory per block (dynamic; about 101 KB for n = 11 at 24 warps): the word
// rings need 2 KB alignment (ring addresses are formed with one LOP3: base | (pos & 0x7FE)).
constexpr int kNarrowMaxBits = 12;  // packed u32 LUT up to n = 12
// n <= 11: the packed LUT in kLutCopies = 4 interleaved copies (entry i of copy c at
// word 4 i + c, so copy c sits in banks c, c + 4, ..., c + 28) and lanes 8c .. 8c + 7
// read copy c: a random gather of 32 slots then spreads over the banks as 4 groups
// of 8 lanes on 8 banks each (3.27 wavefronts on average instead of 3.49 for one
// copy; 32 KB at n = 11, still two 24-warp CTAs per SM).  The decode is bound by the
// l1tex data pipe at ~5.8 wavefronts per 32-symbol group.
constexpr int kLutCopies = 4, kCopyMaxBits = 11;
static_assert(kLutCopies % 4 == 0 && 32 % kLutCopies == 0, "copies are staged as uint4 and split the warp evenly");
template <int NB>
__host__ __device__ constexpr int lut_words() {
  return NB <= 0 ? 128 * warps_per_block<NB>()
                 : NB <= kCopyMaxBits ? ((kLutCopies << NB) > 512 ? (kLutCopies << NB) : 512)
                                      : NB <= 12 ? (1 << NB) : 512;
}
// bytes before the LUT: staging + records
constexpr int kPreLut(int W, int S) { return W * ((int)kBlockBytes * S + 2 * (int)sizeof(TaskRec)); }
// padding that puts the LUT at 1 KB + pre + pad = 0 mod A (A = 2 KB)
constexpr int kLutPad(int W, int S, int A) { return ((A - 1024 - kPreLut(W, S) % A) % A + A) % A; }
// Block layout (byte offsets into the dynamic shared memory).  The CTA's shared
// memory starts 1 KB into its shared window (the reserved system area); stage + rec
// + pad put the LUT on a 2 KB boundary and the LUT is a multiple of 2 KB, so the
// word rings after it start 2 KB-aligned (ring addresses are base | (pos & 0x7FE);
// checked at kernel start).
//   stage[W][512 S]  per warp 512 symbols of output staging
//   rec[W][2]        current / next task record (prebuilt-record plans)
//   lut[lut_words]   n <= 12: packed LUT s | bias << 8 | f << 20 (4 copies for
//                    n <= 11, see kLutCopies); n >= 13
//                    (NEXT row 1): f and F per symbol (the 2^n slot -> symbol bytes
//                    follow the layout); adaptive: each warp's staged model ids
//   ring[W][1024]    per warp 2 KB word window (u16)
template <int NB>
struct Smem {
  static constexpr int S = sym_bytes<NB>();
  static constexpr int W = warps_per_block<NB>();
  static constexpr int kStage = 0;
  static constexpr int kRec = kStage + W * (int)kBlockBytes * S;
  static constexpr int kLut = kRec + W * 2 * (int)sizeof(TaskRec) + kLutPad(W, S, 2048);
  static constexpr int kRing = kLut + 4 * lut_words<NB>();
  static constexpr int kBytes = kRing + W * 2 * kRingWords;
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 lds_v4(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void stg_u16(void *p, uint32_t v) {
  asm volatile("st.global.u16 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void stg_u8(void *p, uint32_t v) {
  asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void stg_v4(void *p, int4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_ge() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_ge;" : "=r"(m));
  return m;
}

#ifdef RECOIL_TIMELINE
// Experiment builds only (tools/build_variant.sh -DRECOIL_TIMELINE): per task the
// %globaltimer at its start and end, the SM and the warp's kernel start time.
constexpr uint32_t kTimelineMax = 1u << 17;
__device__ unsigned long long g_timeline[kTimelineMax][4];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}
#endif
// 4 bytes at byte offset `off` of a warp-distributed window (lane k holds bytes
// [4k, 4k + 4) of it, little endian); off + 4 <= 128.
__device__ __forceinline__ uint32_t window_u32(uint32_t win, uint32_t off) {
  const uint32_t lo = __shfl_sync(kFull, win, (off >> 2) & 31), hi = __shfl_sync(kFull, win, ((off >> 2) + 1) & 31);
  const uint32_t r = 8 * (off & 3);
  return r ? (lo >> r) | (hi << (32 - r)) : lo;
}
// Element j of a W = 32 unsigned data series whose width field is
// the high nibble of byte `base` of the window: w = field + 1 bits, MSB first.
__device__ __forceinline__ uint32_t series_elem(uint32_t win, uint32_t base, uint32_t j, uint32_t *width) {
  const uint32_t w = ((window_u32(win, base) >> 4) & 0xFu) + 1;
  const uint32_t bit = 4 + j * w;
  const uint32_t be = __byte_perm(window_u32(win, base + (bit >> 3)), 0, 0x0123);  // big endian
  *width = w;
  return (be << (bit & 7)) >> (32 - w);
}
__device__ __forceinline__ uint32_t ld_win(const uint8_t *aligned_base, int lane) {
  return __ldg(reinterpret_cast<const uint32_t *>(aligned_base) + lane);
}

struct Warp {
  const Params *p;
  uint32_t ring32;   // 2 KB-aligned shared address of this warp's word ring
  uint32_t stage32;  // this warp's 512-B staging block + lane
  uint32_t lut32;    // shared address of the packed LUT (n <= 12)
  // adaptive (NB = 0): this lane's model-id slot of the staged block, the
  // model tables (coarse bucket -> entry range, entries F | (f-1) << 16,
  // per-model value offset), n, the coarse shift and the largest model id
  uint32_t mid32, coarse32, ent32, delta32, nb, cshift, kmax;
  uint32_t ge;       // this lane and the lanes above it
  int lane;
  // 2 x (1 + slice-relative index of the next word to read), unsigned: slices
  // hold < 2^31 words, so the doubled index needs all 32 bits (a signed form
  // overflowed for slices of >= 2^30 words: the 8 GiB config 5 stream in one
  // launch); the end state (next word -1) is cursor2 = 0.  The +1 lets a lane
  // address its word as cursor2 - 2 pge with pge counting the needing lanes at
  // or above it (see refill).
  uint32_t cursor2;
  int cchunk;        // (cursor2 - 2) >> 9 at the last window check
  uint32_t lo2;      // (cchunk << 9) + 2: the cursor drops below it when it enters chunk cchunk - 1

  // a7: warp-cooperative prefetch of word chunk c (256 words = 32 lanes x 16 B)
  __device__ __forceinline__ void issue_chunk(int c) {
    if (c >= 0 && c < p->n_chunks)
      cp_async16(ring32 + (uint32_t)(c & (kRingChunks - 1)) * (2 * kChunkWords) + 16 * lane,
                 p->words + (size_t)c * kChunkWords + lane * 8);
    cp_commit();
  }
  // Keep chunks cchunk, cchunk-1, cchunk-2 complete and cchunk-3 in flight (the
  // 4-chunk ring).  16 groups consume at most 512 words (two chunks), so one
  // check covers a whole output block.
  __device__ __forceinline__ void window_check() {
    if (cursor2 < lo2) {  // (cursor2 - 2) >> 9 < cchunk: the cursor only moves down
      const int c = (int)((cursor2 - 2u) >> 9);
      __syncwarp();  // all lanes' reads of the slot being refilled (chunk c+1's) are done
      do {
        --cchunk;
        issue_chunk(cchunk - 3);
      } while (cchunk > c);
      lo2 = ((uint32_t)cchunk << 9) + 2u;
      cp_wait<1>();
      __syncwarp();
    }
  }
  // Eq. 4 with the interleaved read order: lanes below read after the
  // lanes above them.  pge = needing lanes at or above this one (POPC), so a
  // needing lane reads word cursor - pge + 1; the warp's word count is lane 0's
  // pge, i.e. the maximum, taken by REDUX (which runs outside the LDS/POPC pipe;
  // one instruction fewer per group than a REDUX.SUM of the need flags).
  __device__ __forceinline__ uint32_t refill(uint32_t x) {
    const bool need = x < kL;
    const uint32_t m = __ballot_sync(kFull, need);
    const uint32_t pge = __popc(m & ge);
    const uint32_t w = lds_u16(ring32 | ((cursor2 + pge * (uint32_t)p->neg2) & (kRingBytes - 2)));
    cursor2 += __reduce_max_sync(kFull, pge) * (uint32_t)p->neg2;  // IMAD: FMA pipe, not ALU
    return need ? x * 65536u + w : x;
  }
  // Eq. 2 with the LUT; stages the symbol byte of group slot k (= g mod 16)
#ifdef RECOIL_CHECK_BOUNDS
  // debug builds (tools/build_variant.sh -DRECOIL_CHECK_BOUNDS; compute-sanitizer is not
  // available on the GPU pool): every output store is checked against the plan's
  // output buffer [chk_lo, chk_hi); a store outside it is counted (g_oob) and dropped
  uint8_t *chk_lo, *chk_hi;
  __device__ __forceinline__ bool in_out(const uint8_t *a, uint32_t n) const { return a >= chk_lo && a + n <= chk_hi; }
#else
  __device__ __forceinline__ bool in_out(const uint8_t *, uint32_t) const { return true; }
#endif
  template <int S>
  __device__ __forceinline__ void st_out(uint8_t *a, uint32_t v) {
    if (!in_out(a, S)) return oob();
    if (S == 1) stg_u8(a, v); else stg_u16(a, v);
  }
  __device__ __forceinline__ void st_out16(uint8_t *a, int4 v) {
    if (!in_out(a, 16)) return oob();
    stg_v4(a, v);
  }
  __device__ __forceinline__ void oob() const;
  uint8_t *outp = nullptr;  // whole blocks: this lane's symbol (S bytes) of group 0 of the output block
  template <int NB, bool DIRECT = false>
  __device__ __forceinline__ uint32_t decode(const uint32_t *lut, const uint8_t *sym, uint32_t x, uint32_t k) {
    if constexpr (NB <= 0) {
      // Eq. 2 under model mid(i) (P:227 item (3)): the entry j of the model
      // with F_j <= slot < F_j + f_j, by a coarse bucket lookup (2^9..2^6 buckets of
      // the slot range per model) and a warp-converged binary search inside
      // the bucket's entry range; value = j + delta(model)
      const uint32_t km = min(lds_u8(mid32 + k * 32), kmax);
      const uint32_t slot = x & ((1u << nb) - 1);
      const uint32_t ca = coarse32 + 2 * (km * p->ad_crow + (slot >> cshift));
      uint32_t lo = lds_u16(ca), hi = lds_u16(ca + 2);
      {  // the first search step unconditionally (predicated, no vote): most buckets hold <= 2
         // entries, and the warp-converged loop below then runs for ~1/3 of the groups (+2 %)
        const uint32_t m = (lo + hi + 1) >> 1;
        const bool up = (lds_u32(ent32 + 4 * m) & 0xFFFFu) <= slot;
        const bool open = lo < hi;
        lo = open && up ? m : lo;
        hi = open && !up ? m - 1 : hi;
      }
      while (__any_sync(kFull, lo < hi)) {
        if (lo < hi) {
          const uint32_t m = (lo + hi + 1) >> 1;
          if ((lds_u32(ent32 + 4 * m) & 0xFFFFu) <= slot) lo = m; else hi = m - 1;
        }
      }
      const uint32_t e = lds_u32(ent32 + 4 * lo);
      if constexpr (DIRECT)  // whole blocks: straight to HBM (64 B = two full sectors per warp)
        st_out<2>(outp + k * 64, lo + lds_u32(delta32 + 4 * km));
      else
        sts_u16(stage32 + k * 64, lo + lds_u32(delta32 + 4 * km));
      return ((e >> 16) + 1) * (x >> nb) + slot - (e & 0xFFFFu);  // f (x >> n) + slot - F
    } else if constexpr (NB <= kNarrowMaxBits) {
      uint32_t e;
      if constexpr (NB <= kCopyMaxBits) {
        // entry slot of this lane's copy: lut32 + 4 kLutCopies slot as one IMAD (FMA pipe;
        // inline PTX so ptxas keeps the multiply-add instead of a shift + add on the ALU pipe)
        uint32_t a;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(a) : "r"(x & ((1u << NB) - 1)), "n"(4 * kLutCopies), "r"(lut32));
        e = lds_u32(a);
      } else {
        e = lds_u32(lut32 + ((x & ((1u << NB) - 1)) << 2));
      }
      if constexpr (DIRECT)
        st_out<1>(outp + k * 32, e);  // whole blocks: straight to HBM (one 32-B sector per warp)
      else
        sts_u8(stage32 + k * 32, e);
      // f (x >> n) + bias as f ((x >> n) - 2^12) + (e >> 8), since e >> 8 = bias + 2^12 f
      // (mod 2^32; the true result is < 2^32): LEA.HI + SHF + SHF + IMAD
      return (e >> 20) * ((x >> NB) + (uint32_t)p->kneg4096) + (e >> 8);
    } else {
      const uint32_t slot = x & ((1u << NB) - 1);
      const uint32_t s = sym[slot];
      const uint32_t e = lut[s];  // f | F << 16
      sts_u8(stage32 + k * 32, s);
      return (e & 0xFFFFu) * (x >> NB) + slot - (e >> 16);  // f (x >> n) + slot - F
    }
  }
  // a8: write an output block: every 16-B chunk of this lane inside the task's
  // write window [woff, wend) (offsets relative to the block's base `dst`).
  // S = symbol bytes: each lane writes 16 S bytes (its part of the 512-symbol block)
  // Offsets are unsigned 32-bit: a task's write window spans < 2^32 - 1024 bytes
  // (checked per task; longer tasks flag E_UNSUPPORTED).
  template <int S>
  __device__ __forceinline__ void flush_at(uint8_t *dst, uint32_t c, uint32_t woff, uint32_t wend) {
    __syncwarp();
    if (c >= woff && c + 16 * S <= wend) {
      const uint32_t a = stage32 + (16 * S - S) * lane;  // staging base + 16 S lane
      st_out16(dst + 16 * S * lane, lds_v4(a));
      if (S == 2) st_out16(dst + 32 * lane + 16, lds_v4(a + 16));
    }
    __syncwarp();  // the staging block is rewritten by the next group steps
  }
  // a whole block inside the write window; dst = this lane's 16 S bytes of it
  template <int S>
  __device__ __forceinline__ void flush_whole(uint8_t *dst) {
    __syncwarp();
    const uint32_t a = stage32 + (16 * S - S) * lane;
    st_out16(dst, lds_v4(a));
    if (S == 2) st_out16(dst + 16, lds_v4(a + 16));
    __syncwarp();
  }
  template <int S>
  __device__ __forceinline__ void flush(uint8_t *dst, uint32_t rel, uint32_t woff, uint32_t wend) {
    flush_at<S>(dst, rel + 16 * S * lane, woff, wend);
  }
};

__device__ __forceinline__ void Warp::oob() const {
#ifdef RECOIL_CHECK_BOUNDS
  atomicAdd(&g_oob, 1ull);
#endif
}

// One group step.  SYNC: Synchronization Phase logic -- lane j is
// initialised with its anchor state in its anchor group, before its read;
// uninitialised lanes keep x = 0xFFFFFFFF and their decodes are discarded.
template <int NB, bool SYNC>
__device__ __forceinline__ uint32_t step(Warp &w, const uint32_t *lut, const uint8_t *sym, uint32_t x, int g, int k, int init_group,
                                         uint32_t state) {
  if (SYNC && g == init_group) x = state;
  x = w.refill(x);
  const uint32_t xn = w.decode<NB>(lut, sym, x, (uint32_t)k);
  return (SYNC && g > init_group) ? 0xFFFFFFFFu : xn;
}

// Groups g .. g_end of one 16-group output block (g_end <= g, same block),
// entered at slot g & 15 (Duff's device) and left after slot g_end & 15.
template <int NB, bool SYNC>
__device__ __forceinline__ uint32_t run_part(Warp &w, const uint32_t *lut, const uint8_t *sym, uint32_t x, int g,
                                             int g_end,
                                             int init_group, uint32_t state) {
  const int gb = g & ~15, k1 = g_end & 15;
  w.window_check();
  if constexpr (NB <= 0) {  // adaptive: a loop, not 16 unrolled entries (instruction-cache size, see run_block)
#pragma unroll 1
    for (int k = g & 15;; --k) {
      x = step<NB, SYNC>(w, lut, sym, x, gb + k, k, init_group, state);
      if (k == k1) break;
    }
    return x;
  }
#define RECOIL_STEP(K)                                                  \
  x = step<NB, SYNC>(w, lut, sym, x, gb + K, K, init_group, state);     \
  if (k1 == K) break;
  switch (g & 15) {
    case 15: RECOIL_STEP(15) [[fallthrough]];
    case 14: RECOIL_STEP(14) [[fallthrough]];
    case 13: RECOIL_STEP(13) [[fallthrough]];
    case 12: RECOIL_STEP(12) [[fallthrough]];
    case 11: RECOIL_STEP(11) [[fallthrough]];
    case 10: RECOIL_STEP(10) [[fallthrough]];
    case 9: RECOIL_STEP(9) [[fallthrough]];
    case 8: RECOIL_STEP(8) [[fallthrough]];
    case 7: RECOIL_STEP(7) [[fallthrough]];
    case 6: RECOIL_STEP(6) [[fallthrough]];
    case 5: RECOIL_STEP(5) [[fallthrough]];
    case 4: RECOIL_STEP(4) [[fallthrough]];
    case 3: RECOIL_STEP(3) [[fallthrough]];
    case 2: RECOIL_STEP(2) [[fallthrough]];
    case 1: RECOIL_STEP(1) [[fallthrough]];
    default: RECOIL_STEP(0)
  }
#undef RECOIL_STEP
  return x;
}

#ifndef RECOIL_AD_UNROLL
#define RECOIL_AD_UNROLL 4
#endif
constexpr int kAdUnroll = RECOIL_AD_UNROLL;
// A whole 16-group block with every lane initialised: no branch per group.  The static
// codec (n <= 12) and the adaptive codec store each group's symbols directly to w.outp
// (set by the caller).
template <int NB>
__device__ __forceinline__ uint32_t run_block(Warp &w, const uint32_t *lut, const uint8_t *sym, uint32_t x) {
  w.window_check();
  if constexpr (NB <= 0) {
    // adaptive: ~60 instructions per group, so a fully unrolled block (and its copies in
    // the partial-block paths) overflows the instruction cache; unroll by RECOIL_AD_UNROLL
#pragma unroll kAdUnroll
    for (int k = 15; k >= 0; --k) {
      x = w.refill(x);
      x = w.template decode<NB, true>(lut, sym, x, k);
    }
  } else {
#pragma unroll
    for (int k = 15; k >= 0; --k) {
      x = w.refill(x);
      x = w.template decode<NB, NB <= kNarrowMaxBits>(lut, sym, x, k);
    }
  }
  return x;
}

template <int NB, bool FUSED>
__global__ void __launch_bounds__(threads_per_block<NB>(), min_blocks<NB>()) recoil_decode_kernel(const Params p) {
  // the shared-memory layout is sized for warps_per_block<NB>() warps; a launch
  // may use fewer (small task counts are spread over all SMs, see launch())
  const uint32_t kWarpsPerBlock = blockDim.x >> 5;
  const uint32_t kThreads = blockDim.x;
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  using L = Smem<NB>;
  uint32_t *const sm_lut = reinterpret_cast<uint32_t *>(smem_dyn + L::kLut);
  TaskRec *const sm_rec = reinterpret_cast<TaskRec *>(smem_dyn + L::kRec);  // [warp][2]
  uint8_t *const sym_dyn = smem_dyn + L::kBytes;  // n >= 13: 2^n slot -> symbol; adaptive: model tables

  constexpr int S = sym_bytes<NB>();
#ifdef RECOIL_TIMELINE
  const unsigned long long tl_kernel = gtime();
#endif
  // the first task's head is requested before the LUT staging, so its latency
  // overlaps the block's LUT copy (fused plans)
  uint32_t hw_first = 0;
  if constexpr (FUSED) {
    const uint32_t t0 = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    hw_first = t0 < p.n_tasks ? __ldg(reinterpret_cast<const uint32_t *>(&p.heads[t0]) + (threadIdx.x & 7)) : 0u;
  }
  // a2: stage the LUT in shared memory (per block)
  if constexpr (NB <= 0) {  // adaptive: coarse table, entries, value offsets (p.lut blob)
    const uint32_t words = (uint32_t)(adaptive_table_bytes(p.ad_K, p.ad_E, p.ad_cbits) / 4);
    for (uint32_t i = threadIdx.x; i < words / 4; i += kThreads)
      reinterpret_cast<int4 *>(sym_dyn)[i] = reinterpret_cast<const int4 *>(p.lut)[i];
    for (uint32_t i = (words & ~3u) + threadIdx.x; i < words; i += kThreads)
      reinterpret_cast<uint32_t *>(sym_dyn)[i] = reinterpret_cast<const uint32_t *>(p.lut)[i];
  } else if constexpr (NB <= kNarrowMaxBits) {
    constexpr uint32_t kWords = 1u << NB;
    if constexpr (NB <= kCopyMaxBits) {  // kLutCopies copies, interleaved by entry
      for (uint32_t i = threadIdx.x; i < kWords; i += kThreads) {
        const uint32_t v = reinterpret_cast<const uint32_t *>(p.lut)[i];
#pragma unroll
        for (int c = 0; c < kLutCopies / 4; ++c)
          reinterpret_cast<uint4 *>(sm_lut)[kLutCopies / 4 * i + c] = make_uint4(v, v, v, v);
      }
    } else if (kWords >= 4) {
      for (uint32_t i = threadIdx.x; i < kWords / 4; i += kThreads)
        reinterpret_cast<int4 *>(sm_lut)[i] = reinterpret_cast<const int4 *>(p.lut)[i];
    } else if (threadIdx.x < kWords) {
      sm_lut[threadIdx.x] = reinterpret_cast<const uint32_t *>(p.lut)[threadIdx.x];
    }
  } else {
    for (uint32_t i = threadIdx.x; i < (1u << NB) / 16; i += kThreads)
      reinterpret_cast<int4 *>(sym_dyn)[i] = reinterpret_cast<const int4 *>(p.lut)[i];
    for (uint32_t i = threadIdx.x; i < 256; i += kThreads)
      sm_lut[i] = reinterpret_cast<const uint32_t *>(p.lut + (1u << NB))[i];
  }
  __syncthreads();

  Warp w;
  w.p = &p;
  w.lane = threadIdx.x & 31;
  const int lane = w.lane;
  const int warp = threadIdx.x >> 5;
  w.ring32 = smem_addr(smem_dyn + L::kRing + warp * 2 * kRingWords);
  w.stage32 = smem_addr(smem_dyn + L::kStage + warp * (int)kBlockBytes * S + S * lane);
  w.ge = lanemask_ge();
  w.lut32 = smem_addr(sm_lut);
#ifdef RECOIL_CHECK_BOUNDS
  w.chk_lo = p.out;
  w.chk_hi = p.out + (p.out_lim - p.out_base) * S;
#ifdef RECOIL_CHECK_SELFTEST
  w.chk_hi -= 512;  // positive control of the check: the last block's stores count as out of bounds
#endif
#endif
  if constexpr (NB >= 1 && NB <= kCopyMaxBits) w.lut32 += 4 * (lane / (32 / kLutCopies));  // this lane's copy
  if constexpr (NB <= 0) {
    w.mid32 = w.lut32 + 512 * warp + lane;
    w.coarse32 = smem_addr(sym_dyn);
    w.ent32 = w.coarse32 + (p.ad_K * p.ad_crow * 2 + 15) / 16 * 16;
    w.delta32 = w.ent32 + 4 * ((p.ad_E + 3) & ~3u);
    w.nb = p.nbits;
    w.cshift = p.nbits > p.ad_cbits ? p.nbits - p.ad_cbits : 0;
    w.kmax = p.ad_K - 1;
  }
  if (w.ring32 & (kRingBytes - 1)) {
    // shared-memory layout assumption broken: fail loudly
    if (threadIdx.x == 0) atomicOr(&p.status->flags, 4u);
    return;
  }
  w.cchunk = 0;
  w.lo2 = 2u;
  const uint32_t rec32 = smem_addr(&sm_rec[2 * warp]);
  const uint32_t *lut = sm_lut;
  const uint8_t *sym = sym_dyn;

  // a3: persistent warps.  The first wave of task ids is static; afterwards a
  // warp takes the next id from an atomic counter shortly before it finishes
  // its current task (two blocks ahead: the atomic's latency hides behind them)
  // and streams that record into shared memory by cp.async.  Taking ids late
  // matters: warps of one SM run at very different speeds under the issue
  // arbiter's priority order, so an id reserved early by a slow warp would
  // become the kernel's tail.
  const uint32_t first_wave = gridDim.x * kWarpsPerBlock;
  auto issue_task = [&](uint32_t t, int buf) {  // prebuilt records: cp.async into shared memory
    if constexpr (!FUSED) {
      if (t < p.n_tasks && lane < (int)(sizeof(TaskRec) / 16))
        cp_async16(rec32 + buf * sizeof(TaskRec) + 16 * lane,
                   reinterpret_cast<const char *>(&p.tasks[t]) + 16 * lane);
      cp_commit();
    }
  };
  // fused a1: lane l holds word l & 7 of the task head (hw) and the task's raw
  // record windows (states and series of point t, series of point t-1); both are
  // loaded one block before the task starts, so their latency hides behind it
  uint32_t hw = 0, pf_st = 0, pf_se = 0, pf_pr = 0;
  auto load_head = [&](uint32_t t) {
    if constexpr (FUSED) hw = t < p.n_tasks ? __ldg(reinterpret_cast<const uint32_t *>(&p.heads[t]) + (lane & 7)) : 0u;
  };
  auto load_windows = [&]() {
    if constexpr (FUSED) {
      const uint32_t rec = __shfl_sync(kFull, hw, 2), rec_prev = __shfl_sync(kFull, hw, 3);
      const uint32_t flags = __shfl_sync(kFull, hw, 5);
      pf_st = (flags & kHeadLast) ? 0u : ld_win(p.recs + (rec & ~3u), lane);
      pf_se = (flags & kHeadLast) ? 0u : ld_win(p.recs + ((rec + 64) & ~3u), lane);
      pf_pr = (flags & kHeadFirst) ? 0u : ld_win(p.recs + ((rec_prev + 64) & ~3u), lane);
    }
  };
  uint32_t t = blockIdx.x * kWarpsPerBlock + warp;
  int buf = 0;
  if (t < p.n_tasks) {
    issue_task(t, 0);
    if constexpr (FUSED) hw = hw_first;
    load_windows();
  }
  // a7: the task's word window: chunks c, c-1, c-2 resident, c-3 in flight
  auto issue_window = [&](int32_t cursor0) {
    w.cursor2 = 2u * (uint32_t)cursor0 + 2u;
    w.cchunk = cursor0 >> 8;
    w.lo2 = ((uint32_t)w.cchunk << 9) + 2u;
    w.issue_chunk(w.cchunk);
    w.issue_chunk(w.cchunk - 1);
    w.issue_chunk(w.cchunk - 2);
    w.issue_chunk(w.cchunk - 3);
  };
  while (t < p.n_tasks) {
#ifdef RECOIL_TIMELINE
    const unsigned long long tl_start = gtime();
#endif
    cp_wait<0>();  // this task's record and any window copy still in flight have landed
    __syncwarp();
    int32_t start_group, init_group, cursor0;
    uint64_t lo, whi;
    int64_t end_cursor;
    uint32_t task_id, state;
    if constexpr (FUSED) {
      // a1 in the kernel: expand the split records of points t and t-1 (P:380-394,
      // tab:metadata_codec): anchor state and group of every lane, the sync starts
      // (min anchor index) that bound this task's committed range (reading Z13)
      cursor0 = (int32_t)__shfl_sync(kFull, hw, 0);
      issue_window(cursor0);  // before the record expansion: the copies overlap it
      start_group = (int32_t)__shfl_sync(kFull, hw, 1);
      const uint32_t rec = __shfl_sync(kFull, hw, 2), rec_prev = __shfl_sync(kFull, hw, 3);
      const uint32_t maxg_prev = __shfl_sync(kFull, hw, 4), flags = __shfl_sync(kFull, hw, 5);
      task_id = __shfl_sync(kFull, hw, 6);
      const int32_t hend = (int32_t)__shfl_sync(kFull, hw, 7);
      const uint64_t N = ((uint64_t)p.N_hi << 32) | p.N_lo;
      bool bad_meta = false;
      int64_t ss_t;
      if (flags & kHeadLast) {
        state = p.finals[lane];
        init_group = start_group - ((uint64_t)start_group * 32 + lane < N ? 0 : 1);
        ss_t = (int64_t)N;
        whi = (N + 15) & ~15ull;
      } else {
        state = window_u32(pf_st, (rec & 3u) + 2 * lane) & 0xFFFFu;  // states as-is
        uint32_t w;
        const uint32_t d = series_elem(pf_se, (rec + 64) & 3u, lane, &w);  // anchor - group
        bad_meta |= d > (uint32_t)start_group;
        init_group = start_group - (int32_t)d;
        // sync start = min_j (32 group_j + j) = 32 start_group + 31 - max_j (32 d_j + 31 - j):
        // one REDUX on a small non-negative key (d < 2^16), exact for any N
        ss_t = 32 * (int64_t)start_group + 31 - (int64_t)__reduce_max_sync(kFull, 32 * d + 31 - lane);
        whi = (uint64_t)(ss_t / 32 + 1) * 32;
      }
      if (flags & kHeadFirst) {
        lo = 0;
        end_cursor = hend;
      } else {
        uint32_t w;
        const uint32_t d = series_elem(pf_pr, (rec_prev + 64) & 3u, lane, &w);
        bad_meta |= d > maxg_prev;
        lo = 32 * (uint64_t)maxg_prev + 31 - __reduce_max_sync(kFull, 32 * d + 31 - lane);
        end_cursor = kNoEndCheck;
        bad_meta |= (int64_t)lo >= ss_t;  // sync starts strictly increasing
      }
      if (__any_sync(kFull, bad_meta)) {  // inconsistent metadata: flag it, skip the task
        if (lane == 0) {
          atomicOr(&p.status->flags, 4u);
          atomicMax(&p.status->bad_task, 0xFFFFFFFFu - task_id);
        }
        lo = 0;
        start_group = -1;
      }
    } else {
      const TaskRec &r = sm_rec[2 * warp + buf];
      start_group = r.start_group;
      lo = r.commit_lo;
      whi = r.write_hi;
      end_cursor = r.end_cursor;
      task_id = r.task_id;
      const uint32_t lw = r.lanes[lane];
      state = r.finals_idx == kNoFinals ? (lw & 0xFFFFu) : p.finals[r.finals_idx * 32 + lane];
      init_group = start_group - (int32_t)(lw >> 16);
      cursor0 = (int)r.cursor0;
      __syncwarp();
      issue_window(cursor0);
    }
    // next task: 0 = not asked, 1 = atomic in flight, 2 = record / head in flight,
    // 3 = (fused) record windows in flight
    int next_state = 0;
    uint32_t t_after = 0, t_next = p.n_tasks;
    auto next_task_step = [&]() {
      if (next_state == 0) {
        if (lane == 0) t_after = first_wave + atomicAdd(&p.status->next_task, 1u);
        next_state = 1;
      } else if (next_state == 1) {
        t_next = __shfl_sync(kFull, t_after, 0);
        issue_task(t_next, buf ^ 1);
        load_head(t_next);
        next_state = 2;
      } else if (next_state == 2) {
        load_windows();
        next_state = 3;
      }
    };

    // a7: word window (issued above) -- chunks c, c-1, c-2 resident, c-3 in flight
    cp_wait<1>();
    __syncwarp();

    // The task's write window [32 group(lo), whi) must lie inside the plan's output
    // buffer [out_base, out_lim) and its first group inside the stream; a record
    // that says otherwise (corrupt or crafted metadata) is flagged, not decoded.
    // Windows of 2^32 - 1024 bytes or more exceed the 32-bit block offsets: E_UNSUPPORTED.
    if (start_group >= 0) {
      const bool bad_win = start_group >= p.G || (lo & ~31ull) < p.out_base || whi > p.out_lim || whi <= lo;
      const bool too_long = !bad_win && (whi - (lo & ~511ull)) * S >= 0xFFFFFC00ull;
      if (bad_win || too_long) {
        if (lane == 0) {
          atomicOr(&p.status->flags, bad_win ? 4u : 8u);
          atomicMax(&p.status->bad_task, 0xFFFFFFFFu - task_id);
        }
        lo = 0;
        start_group = -1;
      }
    }
    const int32_t lo_group = (int32_t)(lo >> 5);
    const int32_t min_init = __reduce_min_sync(kFull, init_group);
    const int32_t g_sync_end = max(min_init, lo_group);
    // 32-bit output bookkeeping relative to the block of lo_group (bytes: S per symbol)
    const int32_t b_lo = lo_group >> 4;
    uint8_t *const out_blo = p.out + ((uint64_t)b_lo * kBlockBytes - p.out_base) * S;
    const uint32_t woff = (lo_group & 15) * kLanes * S;  // 0..511 symbols into block b_lo
    const uint32_t wend = (uint32_t)((whi - (uint64_t)b_lo * kBlockBytes) * S);
    constexpr int kBlk = (int)kBlockBytes * S;  // output block bytes

    // adaptive: the model ids of the block being decoded are staged in shared
    // memory (16 B per lane); the next lower block's ids are loaded into
    // registers meanwhile (one block of look-ahead)
    uint4 midv = make_uint4(0, 0, 0, 0);
    int mid_blk = -1;
    auto mid_load = [&](int blk) -> uint4 {
      const uint64_t N = ((uint64_t)p.N_hi << 32) | p.N_lo;
      const uint64_t i0 = (uint64_t)blk * kBlockBytes + 16 * lane;
      if (i0 + 16 <= N) return __ldg(reinterpret_cast<const uint4 *>(p.mid + i0));
      uint32_t v[4] = {0, 0, 0, 0};
#pragma unroll
      for (int b = 0; b < 16; ++b)
        if (i0 + b < N) v[b >> 2] |= (uint32_t)p.mid[i0 + b] << (8 * (b & 3));
      return make_uint4(v[0], v[1], v[2], v[3]);
    };
    auto stage_block = [&](int blk) {
      if constexpr (NB <= 0) {
        const uint4 v = (mid_blk == blk) ? midv : mid_load(blk);
        __syncwarp();
        sts_v4(w.mid32 - lane + 16 * lane, v);
        __syncwarp();
        if (blk > 0) {
          midv = mid_load(blk - 1);
          mid_blk = blk - 1;
        }
      }
    };

    uint32_t x = 0xFFFFFFFFu;  // uninitialised: never < L
    int32_t g = start_group;

    // a4: Synchronization Phase -- groups where some lane is still uninitialised
    while (g >= g_sync_end) {
      const int gb = g & ~15, ge = max(gb, g_sync_end);
      if ((g & 15) == 15 || g == start_group) stage_block(g >> 4);
      x = run_part<NB, true>(w, lut, sym, x, g, ge, init_group, state);
      if (ge == gb) {
        const int rel = (gb >> 4) - b_lo;
        w.template flush<S>(out_blo + (uint32_t)rel * kBlk, (uint32_t)rel * kBlk, woff, wend);
      }
      g = ge - 1;
    }
    // a5 + a6: Decoding Phase and Cross-Boundary Phase (all lanes initialised)
    if (g >= lo_group && (g & 15) != 15) {  // head: partial block
      const int gb = g & ~15, ge = max(gb, lo_group);
      if (g == start_group) stage_block(g >> 4);  // else staged by the sync phase
      x = run_part<NB, false>(w, lut, sym, x, g, ge, 0, 0);
      const int rel = (gb >> 4) - b_lo;
      w.template flush<S>(out_blo + (uint32_t)rel * kBlk, (uint32_t)rel * kBlk, woff, wend);
      g = ge - 1;
    }
    if (g >= lo_group) {
      // whole blocks above the block of lo_group; the next task id is requested
      // three blocks before the end
      int rel = (g >> 4) - b_lo;
      const int full_lo = ((lo_group & 15) == 0) ? 0 : 1;
      // Every whole block lies inside the write window [woff, wend): block full_lo
      // starts at or above woff, and the top one ends at or below wend because the
      // sync start bounding whi is >= 32 min_init and these blocks are
      // below group min_init.  Checked once here (records that break it are
      // inconsistent), so the whole-block flushes need no per-chunk test.
      const bool whole_ok = (uint32_t)(rel + 1) * kBlk <= wend;
      if (!whole_ok) {
        if (lane == 0) {
          atomicOr(&p.status->flags, 4u);
          atomicMax(&p.status->bad_task, 0xFFFFFFFFu - task_id);
        }
        rel = full_lo - 1;
      }
      constexpr bool kDirect = NB <= kNarrowMaxBits;  // static n <= 12 and the adaptive codec
      uint8_t *dst = out_blo + (uint32_t)rel * kBlk + (kDirect ? S : 16 * S) * lane;  // this lane's part
      for (; rel >= full_lo + 3; --rel) {
        stage_block(b_lo + rel);
        if constexpr (kDirect) w.outp = dst;
        x = run_block<NB>(w, lut, sym, x);
        if constexpr (!kDirect) w.template flush_whole<S>(dst);
        dst -= kBlk;
      }
      for (; rel >= full_lo; --rel) {
        next_task_step();
        stage_block(b_lo + rel);
        if constexpr (kDirect) w.outp = dst;
        x = run_block<NB>(w, lut, sym, x);
        if constexpr (!kDirect) w.template flush_whole<S>(dst);
        dst -= kBlk;
      }
      if (full_lo && whole_ok) {  // tail: the partial block of lo_group
        stage_block(b_lo);
        x = run_part<NB, false>(w, lut, sym, x, b_lo * 16 + 15, lo_group, 0, 0);
        w.template flush<S>(out_blo, 0, woff, wend);
      }
    }
    while (next_state < 3) next_task_step();
    if (end_cursor != kNoEndCheck) {
      // the task reached its codec's first symbol: the outputs emitted before
      // group 0 (Eq. 3 with f(s_0) 2^(32-n) <= L, i.e. n = 16 and f = 1) are read last
      w.window_check();
      x = w.refill(x);
    }

    // a9: integrity -- a task that reaches its codec's start must end in the
    // stack-property end state: cursor one below the codec's first word,
    // every initialised lane back at L.
    // the cursor as a signed slice index: -1 is the codec's end state; anything
    // else at or beyond the slice end is an underflow (the slice has < 2^31 words)
    const uint32_t cur_u = (w.cursor2 - 2u) >> 1;
    const int cursor = w.cursor2 == 0u ? -1 : (int)cur_u;
    bool bad_end = false;
    const bool under = w.cursor2 != 0u && cur_u >= (uint32_t)p.n_chunks * kChunkWords;
    if (end_cursor != kNoEndCheck) {
      const bool lane_ok = (init_group < lo_group) || x == kL;
      bad_end = (cursor != (int)end_cursor) || !__all_sync(kFull, lane_ok);
    }
    if (lane == 0 && (bad_end || under)) {
      atomicOr(&p.status->flags, (under ? 1u : 0u) | (bad_end ? 2u : 0u));
      atomicMax(&p.status->bad_task, 0xFFFFFFFFu - task_id);
    }
#ifdef RECOIL_TIMELINE
    if (lane == 0 && task_id < kTimelineMax) {
      g_timeline[task_id][0] = tl_start;
      g_timeline[task_id][1] = gtime();
      g_timeline[task_id][2] = smid() | (uint64_t)(blockIdx.x * kWarpsPerBlock + warp) << 16;
      g_timeline[task_id][3] = tl_kernel;
    }
#endif
    t = t_next;
    buf ^= 1;
  }
  cp_wait<0>();
}

using KernelFn = void (*)(const Params);
static KernelFn kernel_for(uint32_t nbits, bool fused, bool adaptive = false, bool narrow = false) {
  if (adaptive) return !fused ? nullptr : narrow ? recoil_decode_kernel<-1, true> : recoil_decode_kernel<0, true>;
  if (fused) switch (nbits) {
    case 1: return recoil_decode_kernel<1, true>;
    case 2: return recoil_decode_kernel<2, true>;
    case 3: return recoil_decode_kernel<3, true>;
    case 4: return recoil_decode_kernel<4, true>;
    case 5: return recoil_decode_kernel<5, true>;
    case 6: return recoil_decode_kernel<6, true>;
    case 7: return recoil_decode_kernel<7, true>;
    case 8: return recoil_decode_kernel<8, true>;
    case 9: return recoil_decode_kernel<9, true>;
    case 10: return recoil_decode_kernel<10, true>;
    case 11: return recoil_decode_kernel<11, true>;
    case 12: return recoil_decode_kernel<12, true>;
    case 13: return recoil_decode_kernel<13, true>;
    case 14: return recoil_decode_kernel<14, true>;
    case 15: return recoil_decode_kernel<15, true>;
    case 16: return recoil_decode_kernel<16, true>;
    default: return nullptr;
  }
  switch (nbits) {
    case 1: return recoil_decode_kernel<1, false>;
    case 2: return recoil_decode_kernel<2, false>;
    case 3: return recoil_decode_kernel<3, false>;
    case 4: return recoil_decode_kernel<4, false>;
    case 5: return recoil_decode_kernel<5, false>;
    case 6: return recoil_decode_kernel<6, false>;
    case 7: return recoil_decode_kernel<7, false>;
    case 8: return recoil_decode_kernel<8, false>;
    case 9: return recoil_decode_kernel<9, false>;
    case 10: return recoil_decode_kernel<10, false>;
    case 11: return recoil_decode_kernel<11, false>;
    case 12: return recoil_decode_kernel<12, false>;
    case 13: return recoil_decode_kernel<13, false>;
    case 14: return recoil_decode_kernel<14, false>;
    case 15: return recoil_decode_kernel<15, false>;
    case 16: return recoil_decode_kernel<16, false>;
    default: return nullptr;
  }
}

}  // namespace dev

static size_t layout_bytes(int nbits) {  // dev::Smem<n>::kBytes (n = 0 / -1: adaptive)
  switch (nbits) {
    case -1: return dev::Smem<-1>::kBytes;
    case 0: return dev::Smem<0>::kBytes;
    case 10: return dev::Smem<10>::kBytes;
    case 11: return dev::Smem<11>::kBytes;
    case 12: return dev::Smem<12>::kBytes;
    default: return nbits <= 9 ? dev::Smem<9>::kBytes : dev::Smem<13>::kBytes;
  }
}
static size_t smem_bytes(uint32_t nbits) {  // the block layout + the slot -> symbol table for n >= 13
  return layout_bytes(nbits) + (nbits > (uint32_t)dev::kNarrowMaxBits ? (size_t)1 << nbits : 0);
}
static size_t dyn_smem(const Decoder &d) {  // adaptive: the layout + the model tables
  return d.c->adaptive ? layout_bytes(d.ad_narrow ? -1 : 0) + d.lut.size() : smem_bytes(d.plan.prob_bits);
}

// The kernel's dynamic shared-memory limit only ever grows (per device and
// kernel): launches with less dynamic memory are unaffected by a larger limit,
// and lowering it would break a cached plan that needs more.
static int ensure_dyn(dev::KernelFn fn, size_t dyn) {
  struct Lim {
    int dev;
    dev::KernelFn fn;
    size_t dyn;
  };
  static std::mutex mu;
  static std::vector<Lim> lims;
  int dev_id = 0, optin = 0;
  if (cudaGetDevice(&dev_id) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev_id) != cudaSuccess)
    return RECOIL_E_CUDA;
  if (dyn > (size_t)optin) return RECOIL_E_UNSUPPORTED;  // tables do not fit in shared memory
  std::lock_guard<std::mutex> lock(mu);
  for (Lim &l : lims)
    if (l.dev == dev_id && l.fn == fn) {
      if (l.dyn >= dyn) return RECOIL_OK;
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess)
        return RECOIL_E_CUDA;
      l.dyn = dyn;
      return RECOIL_OK;
    }
  if (cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared) !=
          cudaSuccess ||
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess)
    return RECOIL_E_CUDA;
  lims.push_back({dev_id, fn, dyn});
  return RECOIL_OK;
}

static int occupancy(dev::KernelFn fn, int threads, size_t dyn, int *blocks_per_sm) {
  if (!fn) return RECOIL_E_ARG;
  int rc = ensure_dyn(fn, dyn);
  if (rc) return rc;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fn, threads, dyn) != cudaSuccess)
    return RECOIL_E_CUDA;
  return RECOIL_OK;
}

// The plan (build_fused) picks the adaptive kernel: 32-warp CTAs with the most coarse
// bucket bits in 9..7 (NB = 0) whose tables fit beside that layout in kSmemOptinBytes,
// else 8-warp CTAs with 6-bit buckets (NB = -1); ensure_dyn checks the device's real limit.
}  // namespace recoil
const uint64_t recoil::kAdaptiveWideLayoutBytes = recoil::dev::Smem<0>::kBytes;
namespace recoil {

static int launch(Decoder *d, char *ws, const uint16_t *d_words, const uint8_t *d_mid, uint8_t *d_out,
                  cudaStream_t s) {
  const recoil_plan &pl = d->plan;
  const bool adaptive = d->c->adaptive;
  dev::KernelFn fn = dev::kernel_for(pl.prob_bits, d->fused, adaptive, d->ad_narrow);
  const int warps = adaptive ? (d->ad_narrow ? dev::warps_per_block<-1>() : dev::warps_per_block<0>())
                             : dev::warps_per_block<11>();
  if (d->blocks_per_sm == 0) {
    // launch geometry, cached per (device, kernel, dynamic smem) for the process: the
    // attribute / occupancy queries cost tens of microseconds, and the pipeline builds a
    // fresh plan per chunk and run
    struct Geo {
      int dev;
      dev::KernelFn fn;
      size_t dyn;
      int bps, sms;
    };
    static std::mutex mu;
    static std::vector<Geo> cache;
    int dev_id = 0;
    if (cudaGetDevice(&dev_id) != cudaSuccess) return RECOIL_E_CUDA;
    const size_t dyn = dyn_smem(*d);
    std::lock_guard<std::mutex> lock(mu);
    for (const Geo &g : cache)
      if (g.dev == dev_id && g.fn == fn && g.dyn == dyn) {
        d->blocks_per_sm = g.bps;
        d->sm_count = g.sms;
      }
    if (d->blocks_per_sm == 0) {
      int rc = occupancy(fn, 32 * warps, dyn, &d->blocks_per_sm);
      if (rc) return rc;
      if (cudaDeviceGetAttribute(&d->sm_count, cudaDevAttrMultiProcessorCount, dev_id) != cudaSuccess)
        return RECOIL_E_CUDA;
      if (d->blocks_per_sm < 1) return RECOIL_E_UNSUPPORTED;  // tables do not fit in shared memory
      cache.push_back({dev_id, fn, dyn, d->blocks_per_sm, d->sm_count});
    }
  }
  dev::Params prm;
  prm.lut = reinterpret_cast<const uint8_t *>(ws + d->lut_off);
  prm.finals = reinterpret_cast<const uint32_t *>(ws + d->finals_off);
  prm.tasks = reinterpret_cast<const TaskRec *>(ws + d->tasks_off);
  prm.heads = reinterpret_cast<const TaskHead *>(ws + d->tasks_off);
  prm.recs = reinterpret_cast<const uint8_t *>(ws + d->rec_off);
  prm.N_lo = (uint32_t)d->c->N;
  prm.N_hi = (uint32_t)(d->c->N >> 32);
  prm.G = (int32_t)d->c->G;
  prm.status = reinterpret_cast<DeviceStatus *>(ws);
  prm.words = d_words;
  prm.out = d_out;
  prm.out_base = pl.out_base;
  prm.out_lim = pl.out_base + pl.out_count;
  prm.n_chunks = (int32_t)(pl.word_count / kChunkWords);
  prm.n_tasks = pl.n_tasks;
  prm.neg2 = -2;
  prm.kneg4096 = -4096;
  prm.mid = d_mid;
  prm.ad_K = d->ad_K;
  prm.ad_E = d->ad_E;
  prm.ad_cbits = d->ad_cbits;
  prm.ad_crow = coarse_row(d->ad_cbits);
  prm.nbits = pl.prob_bits;
  // fewer tasks than resident warps: narrower blocks, so the tasks spread over
  // all SMs instead of filling a few (config 4 at 2048 splits: 86 SMs x 24 warps)
  const uint32_t cap = (uint32_t)(d->blocks_per_sm * d->sm_count) * (uint32_t)warps;
  const uint32_t wl = pl.n_tasks >= cap ? (uint32_t)warps
                                        : std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)warps,
                                              (pl.n_tasks + d->sm_count - 1) / (uint32_t)d->sm_count));
  const uint32_t need = (pl.n_tasks + wl - 1) / wl;
  const uint32_t grid = std::min<uint32_t>(need, (uint32_t)(d->blocks_per_sm * d->sm_count));
  if (d->c->adaptive) {  // container-sized tables: the limit may have to grow
    int rc = ensure_dyn(fn, dyn_smem(*d));
    if (rc) return rc;
  }
  fn<<<grid, 32 * wl, dyn_smem(*d), s>>>(prm);
  return cudaGetLastError() == cudaSuccess ? RECOIL_OK : RECOIL_E_CUDA;
}

}  // namespace recoil

using namespace recoil;

extern "C" int recoil_decoder_upload(recoil_decoder *dec, void *d_workspace, uint16_t *d_words, void *stream) {
  if (!dec || !d_workspace || !d_words) return RECOIL_E_ARG;
  Decoder *d = reinterpret_cast<Decoder *>(dec);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = reinterpret_cast<char *>(d_workspace);
  const recoil_plan &p = d->plan;
  if (cudaMemsetAsync(ws, 0, 16, s) != cudaSuccess) return RECOIL_E_CUDA;
  if (!d->lut.empty() && cudaMemcpyAsync(ws + d->lut_off, d->lut.data(), d->lut.size(), cudaMemcpyHostToDevice,
                                         s) != cudaSuccess)
    return RECOIL_E_CUDA;
  if (!d->finals.empty() && cudaMemcpyAsync(ws + d->finals_off, d->finals.data(), 4 * d->finals.size(),
                                            cudaMemcpyHostToDevice, s) != cudaSuccess)
    return RECOIL_E_CUDA;
  if (!d->tasks.empty() && cudaMemcpyAsync(ws + d->tasks_off, d->tasks.data(), sizeof(TaskRec) * d->tasks.size(),
                                           cudaMemcpyHostToDevice, s) != cudaSuccess)
    return RECOIL_E_CUDA;
  if (!d->heads.empty() && cudaMemcpyAsync(ws + d->tasks_off, d->heads.data(), sizeof(TaskHead) * d->heads.size(),
                                           cudaMemcpyHostToDevice, s) != cudaSuccess)
    return RECOIL_E_CUDA;
  if (d->rec_len && cudaMemcpyAsync(ws + d->rec_off, d->c->bytes + d->rec_src, d->rec_len, cudaMemcpyHostToDevice,
                                    s) != cudaSuccess)
    return RECOIL_E_CUDA;
  // the 128-B record windows may reach past the last record: zero that pad
  if (d->fused && cudaMemsetAsync(ws + d->rec_off + d->rec_len, 0, p.workspace_bytes - d->rec_off - d->rec_len, s) !=
                      cudaSuccess)
    return RECOIL_E_CUDA;
  uint64_t have = d->c->B > p.word_lo ? std::min<uint64_t>(p.word_count, d->c->B - p.word_lo) : 0;
  if (have && cudaMemcpyAsync(d_words, d->c->words + 2 * p.word_lo, 2 * have, cudaMemcpyHostToDevice, s) !=
                  cudaSuccess)
    return RECOIL_E_CUDA;
  if (p.word_count > have && cudaMemsetAsync(d_words + have, 0, 2 * (p.word_count - have), s) != cudaSuccess)
    return RECOIL_E_CUDA;
  return RECOIL_OK;
}

namespace recoil {
int launch_decode(Decoder *d, char *ws, const uint16_t *d_words, uint8_t *d_out, void *stream) {
  return launch(d, ws, d_words, nullptr, d_out, reinterpret_cast<cudaStream_t>(stream));
}
// recoil_decode without the status reset: the caller uploaded a zeroed status
// block with the workspace on the same stream order (the e2e pipeline's one
// H2D of tables + records per chunk)
int decode_staged(Decoder *d, char *ws, const uint16_t *d_words, uint8_t *d_out, void *stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const recoil_plan &pl = d->plan;
  if (pl.n_tasks == 0) return RECOIL_OK;
  if (d->c->adaptive) return RECOIL_E_ARG;
  if (d->single_symbol >= 0)
    return cudaMemsetAsync(d_out + (pl.out_lo - pl.out_base), d->single_symbol, pl.out_hi - pl.out_lo, s) ==
                   cudaSuccess
               ? RECOIL_OK
               : RECOIL_E_CUDA;
  return launch(d, ws, d_words, nullptr, d_out, s);
}
}  // namespace recoil

extern "C" int recoil_decode(recoil_decoder *dec, void *d_workspace, const uint16_t *d_words, uint8_t *d_out,
                             void *stream) {
  if (!dec || !d_workspace || !d_words) return RECOIL_E_ARG;
  Decoder *d = reinterpret_cast<Decoder *>(dec);
  const recoil_plan &pl = d->plan;
  if (!d_out && pl.out_hi > pl.out_lo) return RECOIL_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = reinterpret_cast<char *>(d_workspace);
  if (cudaMemsetAsync(ws, 0, 16, s) != cudaSuccess) return RECOIL_E_CUDA;  // status + task counter
  if (pl.n_tasks == 0) return RECOIL_OK;
  if (d->c->adaptive) return RECOIL_E_ARG;  // needs the model ids: recoil_decode_adaptive
  if (d->single_symbol >= 0) {  // f = 2^n: every state decodes to the one symbol (Eq. 2 identity)
    return cudaMemsetAsync(d_out + (pl.out_lo - pl.out_base), d->single_symbol, pl.out_hi - pl.out_lo, s) ==
                   cudaSuccess
               ? RECOIL_OK
               : RECOIL_E_CUDA;
  }
  return launch(d, ws, d_words, nullptr, d_out, s);
}

extern "C" int recoil_decode_adaptive(recoil_decoder *dec, void *d_workspace, const uint16_t *d_words,
                                      const uint8_t *d_model_ids, uint16_t *d_out, void *stream) {
  if (!dec || !d_workspace || !d_words) return RECOIL_E_ARG;
  Decoder *d = reinterpret_cast<Decoder *>(dec);
  const recoil_plan &pl = d->plan;
  if (!d->c->adaptive) return RECOIL_E_ARG;
  if ((!d_out || !d_model_ids) && pl.out_hi > pl.out_lo) return RECOIL_E_ARG;
  if (reinterpret_cast<uintptr_t>(d_model_ids) & 15) return RECOIL_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = reinterpret_cast<char *>(d_workspace);
  if (cudaMemsetAsync(ws, 0, 16, s) != cudaSuccess) return RECOIL_E_CUDA;  // status + task counter
  if (pl.n_tasks == 0) return RECOIL_OK;
  return launch(d, ws, d_words, d_model_ids, reinterpret_cast<uint8_t *>(d_out), s);
}

extern "C" int recoil_decoder_status(recoil_decoder *dec, const void *d_workspace, void *stream, uint64_t *bad) {
  if (!dec || !d_workspace) return RECOIL_E_ARG;
  DeviceStatus st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(&st, d_workspace, sizeof(st), cudaMemcpyDeviceToHost, s) != cudaSuccess) return RECOIL_E_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return RECOIL_E_CUDA;
  if (bad) *bad = st.bad_task ? (uint64_t)(0xFFFFFFFFu - st.bad_task) : UINT64_MAX;
  if (st.flags & 4u) return RECOIL_E_INCONSISTENT;
  if (st.flags & 8u) return RECOIL_E_UNSUPPORTED;
  if (st.flags & 1u) return RECOIL_E_UNDERFLOW;
  if (st.flags & 2u) return RECOIL_E_SYNC;
  return RECOIL_OK;
}

extern "C" int recoil_decoder_launches(const recoil_decoder *dec) {
  if (!dec) return RECOIL_E_ARG;
  const Decoder *d = reinterpret_cast<const Decoder *>(dec);
  return (d->plan.n_tasks == 0 || d->single_symbol >= 0) ? 0 : 1;
}

extern "C" int recoil_decode_occupancy_adaptive(int device, uint32_t n_models, uint64_t n_entries,
                                                int *warps_per_sm, int *sm_count) {
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return RECOIL_E_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return RECOIL_E_CUDA;
  int per_sm = 0, sms = 0, rc;
  // the plan's choice (build_fused): 32-warp CTAs with 2^9..2^7 buckets if they fit
  uint64_t wide = 0;
  bool narrow = true;
  for (uint32_t cb = kCoarseBitsWide; cb >= kCoarseBitsWideMin && narrow; --cb) {
    wide = adaptive_table_bytes(n_models, n_entries, cb);
    narrow = kAdaptiveWideLayoutBytes + wide > kSmemOptinBytes;
  }
  const int warps = narrow ? dev::warps_per_block<-1>() : dev::warps_per_block<0>();
  if (narrow)
    rc = occupancy(dev::kernel_for(16, true, true, true), dev::threads_per_block<-1>(),
                   layout_bytes(-1) + adaptive_table_bytes(n_models, n_entries, kCoarseBitsNarrow), &per_sm);
  else
    rc = occupancy(dev::kernel_for(16, true, true, false), dev::threads_per_block<0>(), layout_bytes(0) + wide,
                   &per_sm);
  cudaError_t e2 = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaSetDevice(prev);
  if (rc) return rc;
  if (e2 != cudaSuccess) return RECOIL_E_CUDA;
  if (warps_per_sm) *warps_per_sm = per_sm * warps;
  if (sm_count) *sm_count = sms;
  return RECOIL_OK;
}

extern "C" int recoil_decode_occupancy(int device, uint32_t nbits, int *warps_per_sm, int *sm_count) {
  if (nbits < 1 || nbits > kMaxGpuProbBits) return RECOIL_E_ARG;
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return RECOIL_E_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return RECOIL_E_CUDA;
  int per_sm = 0, sms = 0;
  int rc = occupancy(dev::kernel_for(nbits, true), dev::threads_per_block<11>(), smem_bytes(nbits), &per_sm);
  cudaError_t e2 = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaSetDevice(prev);
  if (rc) return rc;
  if (e2 != cudaSuccess) return RECOIL_E_CUDA;
  if (warps_per_sm) *warps_per_sm = per_sm * dev::warps_per_block<11>();
  if (sm_count) *sm_count = sms;
  return RECOIL_OK;
}

#ifdef RECOIL_CHECK_BOUNDS
// debug builds: out-of-buffer output stores counted since the last reset
extern "C" int recoil_debug_oob(unsigned long long *count, int reset) {
  if (cudaMemcpyFromSymbol(count, recoil::dev::g_oob, sizeof(*count)) != cudaSuccess) return RECOIL_E_CUDA;
  if (reset) {
    const unsigned long long z = 0;
    if (cudaMemcpyToSymbol(recoil::dev::g_oob, &z, sizeof(z)) != cudaSuccess) return RECOIL_E_CUDA;
  }
  return RECOIL_OK;
}
#endif
#ifdef RECOIL_TIMELINE
extern "C" int recoil_timeline_read(unsigned long long *host, uint32_t n_tasks) {
  const uint32_t n = n_tasks < recoil::dev::kTimelineMax ? n_tasks : recoil::dev::kTimelineMax;
  return cudaMemcpyFromSymbol(host, recoil::dev::g_timeline, 32ull * n) == cudaSuccess ? 0 : -1;
}
#endif
