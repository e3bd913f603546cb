// device_meta.cu -- the on-device metadata path (P:272,
// P:380-396): a client copies the received container to the GPU as it is and
// everything after the fixed header is decoded there.  The host reads only the
// 28-byte header and the model block (to size buffers); the GPU
//   1. decodes the two global series (offset and max-group differences against
//      k ceil(B/M) and k ceil(G/M), tab:metadata_split_point) -- fixed-width
//      elements, one thread each;
//   2. finds the byte offset of every split record.  A record is W u16 states
//      plus an unsigned series whose 4-bit width field w - 1 sits in byte 64, so
//      its size is 65 + 4w in [69, 129] and record k+1's position depends on
//      record k's: a list, not a prefix sum.  The points section is cut into
//      chunks; for every chunk and every possible position 0..129 of its first
//      record the chunk is parsed speculatively (exit position, record count),
//      one thread per (chunk, entry) from a shared-memory copy; one thread then
//      follows the real entry through the chunk summaries, and every chunk
//      writes its records' offsets;
//   3. builds the packed LUT from the model block and expands every
//      task's record (row a1: anchor states, group differences, sync starts; one
//      warp per task reading the split records inside the container's copy);
// then the decode kernel runs.  recoil_device_combine (the server
// shrinks parallelism per client) does the same parse and writes the combined
// container on the GPU: new global series, the kept records copied verbatim
// (a record depends only on its own point), the word stream (device-to-device copy).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>

#include "../recoil_internal.h"

namespace recoil {
namespace dm {

constexpr uint32_t kEntries = 130;   // first-record positions 0..129 in a chunk (record sizes 69..129)
constexpr uint32_t kMaxChunks = 384; // chunk summaries staged in one block's shared memory by the resolver
constexpr uint32_t kBadSpec = 0xFFFFFFFFu;

// Host-side view of the fixed header + model block.
struct Head {
  uint32_t n = 0, M = 0, count = 0;
  uint64_t N = 0, B = 0, G = 0, len = 0, P = 0;
  uint64_t model_pos = 28, finals_pos = 0, gpos = 0, wstart = 0;
  uint32_t f[256] = {0};
};

// Device results of the metadata kernels (workspace layout, see DevPlanLayout).
struct Misc {
  unsigned long long rpos;  // byte offset of the first split record
  uint32_t flags;           // bit 2: inconsistent metadata (as DeviceStatus)
  uint32_t pad;
};

struct Layout {
  uint64_t lut, finals, heads, offset, maxg, rec_off, spec, chunk, misc, total;
  uint32_t chunk_bytes, n_chunks;
};

inline uint64_t a256(uint64_t v) { return (v + 255) & ~255ull; }

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

// MSB-first read of n <= 33 bits at bit position bp of b[0..lim) (bytes past lim read as 0).
__device__ __forceinline__ uint64_t get_bits(const uint8_t *b, uint64_t lim, uint64_t bp, uint32_t n) {
  const uint64_t byte = bp >> 3;
  uint64_t v = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) v = (v << 8) | (byte + k < lim ? b[byte + k] : 0u);
  return (v << (16 + (bp & 7))) >> (64 - n);  // 48 bits loaded: bits [bp, bp + n) with n + 7 <= 48
}

__device__ __forceinline__ uint32_t le32(const uint8_t *b) {
  return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

__device__ __forceinline__ void flag_bad(DeviceStatus *st, Misc *misc) {
  atomicOr(&st->flags, 4u);
  if (misc) atomicOr(&misc->flags, 4u);
}

struct GArgs {
  const uint8_t *c;  // container (device copy)
  uint64_t len, P, B, G, M, N, gpos, finals_pos, wstart;
};

// 1. global series: offset_k = (k+1) ceil(B/M) + d1_k, maxg_k = (k+1) ceil(G/M) + d2_k;
// also the record section start and the final states
__global__ void k_global(GArgs a, uint64_t *offset, uint32_t *maxg, uint32_t *finals, Misc *misc, DeviceStatus *st) {
  const uint8_t *g = a.c + a.gpos;
  const uint64_t lim = a.wstart > a.gpos ? a.wstart - a.gpos : 0;  // the series lie before the words
  const uint32_t w1 = (uint32_t)get_bits(g, lim, 0, 5) + 1;
  const uint64_t s2 = 5 + a.P * (w1 + 1);
  const uint32_t w2 = (uint32_t)get_bits(g, lim, s2, 5) + 1;
  const uint64_t gbits = s2 + 5 + a.P * (w2 + 1);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) {
    misc->rpos = a.gpos + (gbits + 7) / 8;
    if (a.gpos + (gbits + 7) / 8 > a.wstart) flag_bad(st, misc);
  }
  if (tid < 32) finals[tid] = le32(a.c + a.finals_pos + 4 * tid);
  if (tid >= a.P) return;
  if (w1 > 33 || w2 > 33) {  // widths of 32-bit differences with a sign (writer: |d| < 2^32)
    flag_bad(st, misc);
    offset[tid] = 0;
    maxg[tid] = 0;
    return;
  }
  const uint64_t Eb = (a.B + a.M - 1) / a.M, Eg = (a.G + a.M - 1) / a.M;
  auto elem = [&](uint64_t base, uint32_t w, uint64_t k) -> int64_t {
    const uint64_t bp = base + k * (w + 1);
    const int64_t mag = (int64_t)get_bits(g, lim, bp, w);
    return get_bits(g, lim, bp + w, 1) ? -mag : mag;
  };
  const int64_t off = (int64_t)((tid + 1) * Eb) + elem(5, w1, tid);
  const int64_t mg = (int64_t)((tid + 1) * Eg) + elem(s2 + 5, w2, tid);
  bool bad = off < 0 || (uint64_t)off >= a.B || mg < 0 || (uint64_t)mg >= a.G;
  if (tid > 0 && !bad) {  // offsets strictly increasing (the points are in stream order)
    const int64_t prev = (int64_t)(tid * Eb) + elem(5, w1, tid - 1);
    bad = off <= prev;
  }
  if (bad) flag_bad(st, misc);
  offset[tid] = bad ? 0 : (uint64_t)off;
  maxg[tid] = bad ? 0 : (uint32_t)mg;
}

// Stage bytes [src, src + n) into shared memory with aligned 16-B loads of the covering range;
// returns the shared pointer of src's first byte (smbuf must hold n + 32 bytes).  The covering
// range stays inside the device buffer: the metadata precedes the (padded) word stream.
__device__ __forceinline__ const uint8_t *stage_bytes(uint8_t *smbuf, const uint8_t *src, uint32_t n) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
  const uint32_t lead = (uint32_t)(reinterpret_cast<uintptr_t>(src) - a);
  const uint32_t n16 = (lead + n + 15) / 16;
  for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x)
    reinterpret_cast<uint4 *>(smbuf)[i] = reinterpret_cast<const uint4 *>(a)[i];
  __syncthreads();
  return smbuf + lead;
}

// 2a. speculative parse: block t stages chunk t (+ 130 bytes) of the points section and thread e
// parses from chunk position e; spec[t][e] = end position (chunk relative) | record count << 16
__global__ void k_spec(const uint8_t *c, uint64_t wstart, uint32_t C, uint32_t T, const Misc *misc, uint32_t *spec) {
  extern __shared__ __align__(16) uint8_t smbuf[];
  const uint64_t rpos = misc->rpos;
  const uint64_t Ls = wstart > rpos ? wstart - rpos : 0;
  const uint64_t cs = (uint64_t)blockIdx.x * C;
  if (cs >= Ls) {
    for (uint32_t e = threadIdx.x; e < kEntries; e += blockDim.x) spec[(uint64_t)blockIdx.x * kEntries + e] = kBadSpec;
    return;
  }
  const uint32_t have = (uint32_t)(Ls - cs < (uint64_t)C + kEntries + 64 ? Ls - cs : (uint64_t)C + kEntries + 64);
  const uint8_t *sm = stage_bytes(smbuf, c + rpos + cs, have);
  for (uint32_t e = threadIdx.x; e < kEntries; e += blockDim.x) {
    uint32_t p = e, cnt = 0;
    bool bad = false;
    while (p < C && cs + p < Ls) {
      if (p + 64 >= have) {  // the width byte lies past the section: no record starts here
        bad = true;
        break;
      }
      p += 65 + 4 * ((sm[p + 64] >> 4) + 1);
      ++cnt;
    }
    spec[(uint64_t)blockIdx.x * kEntries + e] = bad ? kBadSpec : (p | (cnt << 16));
  }
}

// 2b. follow the real entry (position 0 of chunk 0) through the chunk summaries
__global__ void k_resolve(uint32_t C, uint32_t T, uint64_t P, uint64_t wstart, const uint32_t *spec, uint32_t *chunk,
                          Misc *misc, DeviceStatus *st) {
  extern __shared__ uint32_t ssum[];
  const uint64_t rpos = misc->rpos;
  const uint64_t Ls = wstart > rpos ? wstart - rpos : 0;
  for (uint32_t i = threadIdx.x; i < T * kEntries; i += blockDim.x) ssum[i] = spec[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t e = 0;
  uint64_t idx = 0, end = 0;
  bool bad = false;
  for (uint32_t t = 0; t < T && (uint64_t)t * C < Ls; ++t) {
    chunk[2 * t] = e;
    chunk[2 * t + 1] = (uint32_t)idx;
    if (e >= kEntries) {
      bad = true;
      break;
    }
    const uint32_t v = ssum[t * kEntries + e];
    if (v == kBadSpec) {
      bad = true;
      break;
    }
    const uint32_t p = v & 0xFFFFu;
    idx += v >> 16;
    end = (uint64_t)t * C + p;
    e = p >= C ? p - C : kEntries;  // a chunk's parse leaves it past its end (or at the section end)
  }
  if (bad || idx != P || end != Ls) flag_bad(st, misc);
}

// 2c. every chunk writes the offsets of the records that start in it
__global__ void k_write(const uint8_t *c, uint64_t wstart, uint32_t C, uint64_t P, const uint32_t *chunk,
                        const Misc *misc, uint64_t *rec_off) {
  extern __shared__ __align__(16) uint8_t smbuf[];
  if (misc->flags) return;
  const uint64_t rpos = misc->rpos;
  const uint64_t Ls = wstart - rpos;
  const uint64_t cs = (uint64_t)blockIdx.x * C;
  if (cs >= Ls) return;
  const uint32_t have = (uint32_t)(Ls - cs < (uint64_t)C + kEntries + 64 ? Ls - cs : (uint64_t)C + kEntries + 64);
  const uint8_t *sm = stage_bytes(smbuf, c + rpos + cs, have);
  if (threadIdx.x != 0) return;
  uint32_t p = chunk[2 * blockIdx.x];
  uint64_t idx = chunk[2 * blockIdx.x + 1];
  while (p < C && cs + p < Ls && idx < P) {
    rec_off[idx++] = rpos + cs + p;
    p += 65 + 4 * ((sm[p + 64] >> 4) + 1);
  }
  if (cs + C >= Ls) rec_off[P] = wstart;  // the last chunk closes the list
}

// 3a. the packed LUT from the model block: n <= 12 s | bias << 8 | f << 20; n >= 13 slot ->
// symbol bytes + per-symbol f | F << 16 (the layouts of pack_lut)
__global__ void k_lut(const uint8_t *c, uint64_t model_pos, uint32_t count, uint32_t n, uint8_t *lut) {
  __shared__ uint32_t f[256], F[257];
  for (uint32_t s = threadIdx.x; s < 256; s += blockDim.x) f[s] = 0;
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < count; k += blockDim.x) {
    const uint8_t *e = c + model_pos + 2 + 5 * (uint64_t)k;
    f[e[0]] = le32(e + 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    F[0] = 0;
    for (int s = 0; s < 256; ++s) F[s + 1] = F[s] + f[s];
  }
  __syncthreads();
  const uint32_t slots = 1u << n;
  for (uint32_t slot = threadIdx.x; slot < slots; slot += blockDim.x) {
    uint32_t lo = 0, hi = 255;  // the symbol s with F[s] <= slot < F[s + 1]
    while (lo < hi) {
      const uint32_t m = (lo + hi + 1) >> 1;
      if (F[m] <= slot) lo = m; else hi = m - 1;
    }
    if (n <= 12)
      reinterpret_cast<uint32_t *>(lut)[slot] = lo | ((slot - F[lo]) << 8) | (f[lo] << 20);
    else
      lut[slot] = (uint8_t)lo;
  }
  if (n > 12)
    for (uint32_t s = threadIdx.x; s < 256; s += blockDim.x)
      reinterpret_cast<uint32_t *>(lut + slots)[s] = (f[s] & 0xFFFFu) | (F[s] << 16);
}

// 3b. task records (the host-expanded TaskRec of build_decoder_from, row a1) on the device: one
// warp per task, lane j decodes element j of its point's group-difference series and
// the warp takes the point's sync start (min anchor index) and boundary (max) by REDUX; the checks
// of the host's full parse: differences <= the anchor group, boundary < N, sync starts
// strictly increasing.  Inconsistent metadata: the task gets start group G, which the kernel flags
// and skips.
__device__ __forceinline__ bool point_of(const uint8_t *c, uint64_t rec, uint32_t mg, uint64_t N, uint32_t lane,
                                         uint32_t *state, uint32_t *d, int64_t *ss) {
  const uint8_t *r = c + rec;
  *state = (uint32_t)r[2 * lane] | ((uint32_t)r[2 * lane + 1] << 8);  // W x u16 anchor states
  const uint32_t w = (r[2 * kLanes] >> 4) + 1;
  *d = (uint32_t)get_bits(r + 2 * kLanes, 5 + 4 * w, 4 + lane * w, w);
  const bool bad = *d > mg;
  // min_j (32 (mg - d_j) + j) = 32 mg + 31 - max_j (32 d_j + 31 - j); max_j (...) = 32 mg + 31 - min_j (...)
  const uint32_t key = 32 * *d + 31 - lane;
  *ss = 32 * (int64_t)mg + 31 - (int64_t)__reduce_max_sync(0xFFFFFFFFu, key);
  const int64_t bidx = 32 * (int64_t)mg + 31 - (int64_t)__reduce_min_sync(0xFFFFFFFFu, key);
  return __any_sync(0xFFFFFFFFu, bad) || bidx >= (int64_t)N;
}

// tasks [tb, te) of the container; record t - tb holds task t (task_id t)
__global__ void k_taskrecs(uint64_t M, uint64_t tb, uint64_t te, uint64_t N, uint64_t B, uint64_t G, const uint8_t *c,
                           const uint64_t *offset, const uint32_t *maxg, const uint64_t *rec_off, Misc *misc,
                           DeviceStatus *st, TaskRec *tasks) {
  const uint64_t t = tb + (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (t >= te) return;
  const uint64_t P = M - 1;
  TaskRec r;
  bool bad = misc->flags != 0;
  uint32_t state = 0, d = 0;
  int64_t ss = (int64_t)N, ss_prev = 0;
  if (!bad && t < P) bad |= point_of(c, rec_off[t], maxg[t], N, lane, &state, &d, &ss);
  if (!bad && t > 0) {
    uint32_t s2, d2;
    bad |= point_of(c, rec_off[t - 1], maxg[t - 1], N, lane, &s2, &d2, &ss_prev);
    bad |= ss <= ss_prev && t < P;
  }
  if (bad && lane == 0) flag_bad(st, nullptr);
  r.task_id = (uint32_t)t;
  r.pad[0] = r.pad[1] = r.pad[2] = 0;
  r.commit_lo = t > 0 ? (uint64_t)ss_prev : 0;
  r.end_cursor = r.commit_lo == 0 ? -1 : kNoEndCheck;
  if (t < P) {
    r.commit_hi = (uint64_t)ss - 1;
    r.write_hi = kLanes * ((uint64_t)ss / kLanes + 1);  // through the sync completion group
    r.cursor0 = (int64_t)offset[t];
    r.start_group = (int32_t)maxg[t];
    r.finals_idx = kNoFinals;
    r.lanes[lane] = state | (d << 16);
  } else {
    r.commit_hi = N - 1;
    r.write_hi = (N + 15) & ~15ull;
    r.cursor0 = (int64_t)B - 1;
    r.start_group = (int32_t)(G - 1);
    r.finals_idx = 0;
    r.lanes[lane] = (kLanes * (G - 1) + lane < N ? 0u : 1u) << 16;
  }
  if (bad) {  // the kernel rejects start_group >= G before decoding
    r.start_group = (int32_t)G;
    r.cursor0 = 0;
    r.commit_lo = 0;
    r.end_cursor = kNoEndCheck;
  }
  // lane j stores lanes[j]; lane 0 the scalar fields (16-B aligned record)
  tasks[t - tb].lanes[lane] = r.lanes[lane];
  if (lane == 0) {
    TaskRec &o = tasks[t - tb];
    o.cursor0 = r.cursor0;
    o.end_cursor = r.end_cursor;
    o.commit_lo = r.commit_lo;
    o.commit_hi = r.commit_hi;
    o.write_hi = r.write_hi;
    o.start_group = r.start_group;
    o.finals_idx = r.finals_idx;
    o.task_id = r.task_id;
    o.pad[0] = o.pad[1] = o.pad[2] = 0;
  }
}

// ---------------------------------------------------------------------------
// combine on the GPU: keep points k, 2k, ... (k = ceil(M / target))
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t bitlen64(uint64_t v) { return v ? 64 - __clzll((long long)v) : 1; }

// widths of the new global series (max bit length of |diff|), into wmax[0..1]
__global__ void k_cmb_width(uint64_t P2, uint64_t kstep, uint64_t Eb2, uint64_t Eg2, const uint64_t *offset,
                            const uint32_t *maxg, uint32_t *wmax) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t w1 = 1, w2 = 1;
  if (i < P2) {
    const uint64_t src = (i + 1) * kstep - 1;
    const int64_t d1 = (int64_t)offset[src] - (int64_t)((i + 1) * Eb2);
    const int64_t d2 = (int64_t)maxg[src] - (int64_t)((i + 1) * Eg2);
    w1 = bitlen64(d1 < 0 ? (uint64_t)(-d1) : (uint64_t)d1);
    w2 = bitlen64(d2 < 0 ? (uint64_t)(-d2) : (uint64_t)d2);
  }
  // warp max, then one atomic per warp
  for (int o = 16; o; o >>= 1) {
    w1 = max(w1, __shfl_xor_sync(0xFFFFFFFFu, w1, o));
    w2 = max(w2, __shfl_xor_sync(0xFFFFFFFFu, w2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&wmax[0], w1);
    atomicMax(&wmax[1], w2);
  }
}

// OR `nbits` (<= 34) bits of v, MSB first, into the big-endian bit stream at bit position bp
__device__ __forceinline__ void or_bits(uint8_t *out, uint64_t bp, uint64_t v, uint32_t nbits) {
  // bits land in bytes bp >> 3 .. (bp + nbits - 1) >> 3 (at most 6); OR byte by byte via 32-bit atomics
  const uint32_t sh = (uint32_t)(bp & 7);
  const uint64_t aligned = v << (64 - nbits - sh);  // the field's bits, left aligned after sh leading bits
  const uint64_t b0 = bp >> 3;
  const uint32_t nbytes = (sh + nbits + 7) >> 3;
  for (uint32_t k = 0; k < nbytes; ++k) {
    const uint32_t byte = (uint32_t)((aligned >> (56 - 8 * k)) & 0xFFu);
    if (!byte) continue;
    const uint64_t a = b0 + k;
    uint32_t *word = reinterpret_cast<uint32_t *>(reinterpret_cast<uintptr_t>(out + a) & ~(uintptr_t)3);
    atomicOr(word, byte << (8 * (reinterpret_cast<uintptr_t>(out + a) & 3)));
  }
}

struct CmbArgs {
  uint64_t P2, kstep, Eb2, Eg2;
  uint64_t gpos;        // byte offset of the global series in the output
  uint64_t rec_out;     // byte offset of the first kept record in the output
};

// the new global series bits (the region is zeroed first); thread i writes element i of both series
__global__ void k_cmb_series(CmbArgs a, const uint64_t *offset, const uint32_t *maxg, const uint32_t *wmax,
                             uint8_t *out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t w1 = wmax[0], w2 = wmax[1];
  uint8_t *g = out + a.gpos;
  const uint64_t s2 = 5 + a.P2 * (w1 + 1);
  if (i == 0) {
    or_bits(g, 0, w1 - 1, 5);
    or_bits(g, s2, w2 - 1, 5);
  }
  if (i >= a.P2) return;
  const uint64_t src = (i + 1) * a.kstep - 1;
  const int64_t d1 = (int64_t)offset[src] - (int64_t)((i + 1) * a.Eb2);
  const int64_t d2 = (int64_t)maxg[src] - (int64_t)((i + 1) * a.Eg2);
  const uint64_t m1 = d1 < 0 ? (uint64_t)(-d1) : (uint64_t)d1, m2 = d2 < 0 ? (uint64_t)(-d2) : (uint64_t)d2;
  or_bits(g, 5 + i * (w1 + 1), (m1 << 1) | (d1 < 0 ? 1u : 0u), w1 + 1);
  or_bits(g, s2 + 5 + i * (w2 + 1), (m2 << 1) | (d2 < 0 ? 1u : 0u), w2 + 1);
}

// kept record sizes -> exclusive prefix (one block; the record list is short: M <= ~300k)
__global__ void k_cmb_scan(uint64_t P2, uint64_t kstep, const uint64_t *rec_off, uint64_t *rec_out) {
  __shared__ uint64_t part[1024];
  const uint32_t T = blockDim.x;
  const uint64_t per = (P2 + T - 1) / T;
  const uint64_t lo = threadIdx.x * per, hi = min(P2, lo + per);
  uint64_t s = 0;
  for (uint64_t i = lo; i < hi; ++i) {
    const uint64_t src = (i + 1) * kstep - 1;
    s += rec_off[src + 1] - rec_off[src];
  }
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (uint32_t k = 0; k < T; ++k) {
      const uint64_t v = part[k];
      part[k] = acc;
      acc += v;
    }
    rec_out[P2] = acc;  // total bytes of the kept records
  }
  __syncthreads();
  uint64_t acc = part[threadIdx.x];
  for (uint64_t i = lo; i < hi; ++i) {
    const uint64_t src = (i + 1) * kstep - 1;
    rec_out[i] = acc;
    acc += rec_off[src + 1] - rec_off[src];
  }
}

// kept records, verbatim: one warp per record
__global__ void k_cmb_records(uint64_t P2, uint64_t kstep, const uint8_t *in, const uint64_t *rec_off,
                              const uint64_t *rec_out, uint64_t out_rec_base, uint8_t *out) {
  const uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (i >= P2) return;
  const uint64_t src = (i + 1) * kstep - 1;
  const uint64_t a = rec_off[src], n = rec_off[src + 1] - a, d = out_rec_base + rec_out[i];
  for (uint64_t k = lane; k < n; k += 32) out[d + k] = in[a + k];
}

__global__ void k_cmb_total(uint64_t fixed, const uint64_t *rec_out, uint64_t P2, uint64_t words_bytes,
                            unsigned long long *total) {
  *total = fixed + rec_out[P2] + words_bytes;
}

}  // namespace dm

namespace {

int read_head(const uint8_t *h, uint64_t head_len, uint64_t len, dm::Head *o) {
  if (!h) return RECOIL_E_ARG;
  if (head_len < 28 || len < 28) return RECOIL_E_TRUNCATED;
  if (std::memcmp(h, "RCL1", 4) != 0) return std::memcmp(h, "RCA1", 4) == 0 || std::memcmp(h, "RCV1", 4) == 0
                                                  ? RECOIL_E_UNSUPPORTED
                                                  : RECOIL_E_BAD_MAGIC;
  if (h[4] != 1 || h[5] != 8) return RECOIL_E_VERSION;
  auto le = [&](uint64_t pos, int nb) {
    uint64_t v = 0;
    for (int k = 0; k < nb; ++k) v |= (uint64_t)h[pos + k] << (8 * k);
    return v;
  };
  o->n = h[6];
  if (o->n < 1 || o->n > 16 || h[7] != kLanes) return RECOIL_E_INCONSISTENT;
  o->M = (uint32_t)le(8, 4);
  o->N = le(12, 8);
  o->B = le(20, 8);
  o->len = len;
  if (o->M < 1 || o->B > o->N + 1) return RECOIL_E_INCONSISTENT;
  o->G = ceil_div(o->N, kLanes);
  o->P = o->M - 1;
  if (head_len < 30) return RECOIL_E_TRUNCATED;
  o->count = (uint32_t)le(28, 2);
  if (head_len < 30 + 5ull * o->count) return RECOIL_E_TRUNCATED;
  uint64_t sum = 0;
  for (uint32_t k = 0; k < o->count; ++k) {
    const uint32_t s = h[30 + 5 * k];
    const uint32_t f = (uint32_t)le(30 + 5 * k + 1, 4);
    if (!f || o->f[s]) return RECOIL_E_INCONSISTENT;
    o->f[s] = f;
    sum += f;
  }
  if (sum != (1ull << o->n)) return RECOIL_E_INCONSISTENT;
  o->finals_pos = 30 + 5ull * o->count;
  o->gpos = o->finals_pos + 4ull * kLanes;
  if (2 * o->B > len || len - 2 * o->B < o->gpos + 2 + o->P * (2 * kLanes + 1)) return RECOIL_E_TRUNCATED;
  o->wstart = len - 2 * o->B;
  return RECOIL_OK;
}

dm::Layout layout_for(const dm::Head &h) {
  dm::Layout L{};
  const uint64_t Ls = h.wstart - h.gpos;  // upper bound of the points section
  uint32_t C = 8192;
  while (ceil_div(Ls, C) + 1 > dm::kMaxChunks && C < 60000) C += 4096;
  L.chunk_bytes = C;
  L.n_chunks = (uint32_t)std::max<uint64_t>(1, ceil_div(Ls, C) + 1);
  const uint64_t lut_bytes = h.n <= 12 ? 4ull << h.n : (1ull << h.n) + 1024;
  L.lut = 256;  // status + misc first
  L.misc = 16;
  L.finals = dm::a256(L.lut + lut_bytes);
  L.heads = dm::a256(L.finals + 128);
  L.offset = dm::a256(L.heads + sizeof(TaskRec) * h.M);
  L.maxg = dm::a256(L.offset + 8 * h.P);
  L.rec_off = dm::a256(L.maxg + 4 * h.P);
  L.spec = dm::a256(L.rec_off + 8 * (h.P + 1));
  L.chunk = dm::a256(L.spec + 4ull * dm::kEntries * L.n_chunks);
  L.total = dm::a256(L.chunk + 8ull * L.n_chunks) + 256;
  return L;
}

struct DeviceDecoder {
  dm::Head h;
  dm::Layout L;
  Decoder dec;
  uint64_t coff = 0;       // container offset in the caller's buffer (words 512-B aligned)
  uint64_t buf_bytes = 0;  // caller's buffer size
  uint64_t words_pad = 0;  // zero bytes after the words (chunk padding + over-read)
};

// the parse kernels into workspace ws for the container at buf + coff
int run_parse(const dm::Head &h, const dm::Layout &L, const uint8_t *buf, uint64_t coff, char *ws, cudaStream_t s) {
  const uint8_t *c = buf + coff;
  DeviceStatus *st = reinterpret_cast<DeviceStatus *>(ws);
  dm::Misc *misc = reinterpret_cast<dm::Misc *>(ws + L.misc);
  uint64_t *offset = reinterpret_cast<uint64_t *>(ws + L.offset);
  uint32_t *maxg = reinterpret_cast<uint32_t *>(ws + L.maxg);
  uint64_t *rec_off = reinterpret_cast<uint64_t *>(ws + L.rec_off);
  uint32_t *spec = reinterpret_cast<uint32_t *>(ws + L.spec);
  uint32_t *chunk = reinterpret_cast<uint32_t *>(ws + L.chunk);
  if (cudaMemsetAsync(ws, 0, 256, s) != cudaSuccess) return RECOIL_E_CUDA;  // status + misc
  dm::GArgs ga{c, h.len, h.P, h.B, h.G, h.M, h.N, h.gpos, h.finals_pos, h.wstart};
  const uint32_t gb = (uint32_t)std::max<uint64_t>(1, ceil_div(std::max<uint64_t>(h.P, 32), 256));
  dm::k_global<<<gb, 256, 0, s>>>(ga, offset, maxg, reinterpret_cast<uint32_t *>(ws + L.finals), misc, st);
  if (h.P) {
    const size_t stage = L.chunk_bytes + dm::kEntries + 64 + 32;
    // dynamic shared memory beyond 48 KB (per device: set on every call, it is cheap)
    if (cudaFuncSetAttribute(dm::k_spec, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(dm::k_write, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024) != cudaSuccess ||
        cudaFuncSetAttribute(dm::k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             4 * dm::kEntries * dm::kMaxChunks) != cudaSuccess)
      return RECOIL_E_CUDA;
    dm::k_spec<<<L.n_chunks, 160, stage, s>>>(c, h.wstart, L.chunk_bytes, L.n_chunks, misc, spec);
    dm::k_resolve<<<1, 1024, 4 * dm::kEntries * L.n_chunks, s>>>(L.chunk_bytes, L.n_chunks, h.P, h.wstart, spec,
                                                                 chunk, misc, st);
    dm::k_write<<<L.n_chunks, 128, stage, s>>>(c, h.wstart, L.chunk_bytes, h.P, chunk, misc, rec_off);
  }
  return cudaGetLastError() == cudaSuccess ? RECOIL_OK : RECOIL_E_CUDA;
}

}  // namespace
}  // namespace recoil

using namespace recoil;

extern "C" int recoil_device_decoder_create_range(const uint8_t *head, uint64_t head_len, uint64_t container_len,
                                                  uint64_t task_begin, uint64_t task_end,
                                                  recoil_device_decoder **out) {
  if (!out) return RECOIL_E_ARG;
  *out = nullptr;
  try {
    DeviceDecoder *dd = new DeviceDecoder();
    int rc = read_head(head, head_len, container_len, &dd->h);
    if (rc) {
      delete dd;
      return rc;
    }
    if (dd->h.M > 1 && dd->h.wstart - dd->h.gpos > (uint64_t)dm::kMaxChunks * 60000) {
      delete dd;
      return RECOIL_E_UNSUPPORTED;  // more split metadata than the resolver stages (~23 MB)
    }
    const dm::Head &h = dd->h;
    dd->L = layout_for(h);
    dd->coff = (512 - (h.wstart & 511)) & 511;
    const uint64_t word_count = std::max<uint64_t>(kChunkWords, ceil_div(h.B, kChunkWords) * kChunkWords);
    if (word_count >= (1ull << 31)) {
      delete dd;
      return RECOIL_E_UNSUPPORTED;
    }
    dd->words_pad = 2 * (word_count - h.B) + 256;
    dd->buf_bytes = dd->coff + container_len + dd->words_pad;
    // the decode plan: tasks [tb, te) (the whole stream by default), task records built
    // on the device; the output is addressed by absolute symbol index (out_base 0)
    const uint64_t M = h.N ? h.M : 0;
    const uint64_t tb = task_begin, te = task_end == ~0ull ? M : task_end;
    if (tb > te || te > M || (M && tb == te)) {
      delete dd;
      return RECOIL_E_ARG;
    }
    auto c = std::make_shared<Container>();
    c->n = h.n;
    c->W = kLanes;
    c->M = h.M;
    c->N = h.N;
    c->B = h.B;
    c->G = h.G;
    c->light = true;
    std::memcpy(c->f, h.f, sizeof(c->f));
    Decoder &d = dd->dec;
    d.c = c;
    d.fused = false;  // device-built task records (k_taskrecs), streamed by the kernel
    d.single_symbol = -1;
    int present = 0;
    for (int s = 0; s < 256; ++s)
      if (h.f[s]) {
        ++present;
        d.single_symbol = s;
      }
    if (present != 1) d.single_symbol = -1;
    recoil_plan &p = d.plan;
    std::memset(&p, 0, sizeof(p));
    p.task_begin = tb;
    p.task_end = te;
    p.n_tasks = (uint32_t)(te - tb);
    p.prob_bits = h.n;
    p.word_lo = 0;
    p.word_count = word_count;
    p.out_lo = 0;
    p.out_hi = h.N;
    p.out_base = 0;
    p.out_count = (h.N + 15) & ~15ull;
    p.workspace_bytes = dd->L.total;
    p.upload_bytes = container_len;
    p.symbol_bytes = 1;
    p.n_models = 1;
    p.warps_per_block = kWarpsStatic;
    d.n_tasks = p.n_tasks;
    d.lut_off = dd->L.lut;
    d.finals_off = dd->L.finals;
    d.tasks_off = dd->L.heads;
    *out = reinterpret_cast<recoil_device_decoder *>(dd);
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_device_decoder_create(const uint8_t *head, uint64_t head_len, uint64_t container_len,
                                            recoil_device_decoder **out) {
  return recoil_device_decoder_create_range(head, head_len, container_len, 0, ~0ull, out);
}

extern "C" int recoil_device_decoder_span(const recoil_device_decoder *dec, const void *d_workspace, void *stream,
                                          uint64_t *out_lo, uint64_t *out_hi) {
  if (!dec || !d_workspace || !out_lo || !out_hi) return RECOIL_E_ARG;
  const DeviceDecoder *dd = reinterpret_cast<const DeviceDecoder *>(dec);
  const recoil_plan &p = dd->dec.plan;
  *out_lo = *out_hi = 0;
  if (!p.n_tasks) return RECOIL_OK;
  // the committed range of the first and the last task of the range (device task records)
  const TaskRec *recs = reinterpret_cast<const TaskRec *>(static_cast<const char *>(d_workspace) + dd->L.heads);
  uint64_t lo = 0, hi = 0;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(&lo, &recs[0].commit_lo, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(&hi, &recs[p.n_tasks - 1].commit_hi, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return RECOIL_E_CUDA;
  *out_lo = lo;
  *out_hi = hi + 1;
  return RECOIL_OK;
}

extern "C" int recoil_device_decoder_plan(const recoil_device_decoder *dec, recoil_device_plan *plan) {
  if (!dec || !plan) return RECOIL_E_ARG;
  const DeviceDecoder *dd = reinterpret_cast<const DeviceDecoder *>(dec);
  plan->container_offset = dd->coff;
  plan->buffer_bytes = dd->buf_bytes;
  plan->workspace_bytes = dd->L.total;
  plan->out_count = dd->dec.plan.out_count;
  plan->n_symbols = dd->h.N;
  plan->n_tasks = dd->dec.plan.n_tasks;
  plan->prob_bits = dd->h.n;
  return RECOIL_OK;
}

extern "C" int recoil_device_upload(const recoil_device_decoder *dec, const uint8_t *container, void *d_buffer,
                                    void *stream) {
  if (!dec || !container || !d_buffer) return RECOIL_E_ARG;
  const DeviceDecoder *dd = reinterpret_cast<const DeviceDecoder *>(dec);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *b = static_cast<char *>(d_buffer);
  if (cudaMemcpyAsync(b + dd->coff, container, dd->h.len, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemsetAsync(b + dd->coff + dd->h.len, 0, dd->words_pad, s) != cudaSuccess)
    return RECOIL_E_CUDA;
  return RECOIL_OK;
}

extern "C" int recoil_device_decode(recoil_device_decoder *dec, void *d_buffer, void *d_workspace, uint8_t *d_out,
                                    void *stream) {
  if (!dec || !d_buffer || !d_workspace) return RECOIL_E_ARG;
  DeviceDecoder *dd = reinterpret_cast<DeviceDecoder *>(dec);
  const dm::Head &h = dd->h;
  if (h.N && !d_out) return RECOIL_E_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = static_cast<char *>(d_workspace);
  const uint8_t *buf = static_cast<const uint8_t *>(d_buffer);
  int rc = run_parse(h, dd->L, buf, dd->coff, ws, s);
  if (rc) return rc;
  if (!h.N) return RECOIL_OK;
  dm::k_lut<<<1, 256, 0, s>>>(buf + dd->coff, h.model_pos, h.count, h.n, reinterpret_cast<uint8_t *>(ws + dd->L.lut));
  const recoil_plan &pl = dd->dec.plan;
  const uint32_t hb = (uint32_t)ceil_div(32 * (uint64_t)pl.n_tasks, 256);
  dm::k_taskrecs<<<hb, 256, 0, s>>>(h.M, pl.task_begin, pl.task_end, h.N, h.B, h.G, buf + dd->coff,
                                    reinterpret_cast<const uint64_t *>(ws + dd->L.offset),
                                    reinterpret_cast<const uint32_t *>(ws + dd->L.maxg),
                                    reinterpret_cast<const uint64_t *>(ws + dd->L.rec_off),
                                    reinterpret_cast<dm::Misc *>(ws + dd->L.misc),
                                    reinterpret_cast<DeviceStatus *>(ws), reinterpret_cast<TaskRec *>(ws + dd->L.heads));
  if (cudaGetLastError() != cudaSuccess) return RECOIL_E_CUDA;
  if (dd->dec.single_symbol >= 0)
    return cudaMemsetAsync(d_out, dd->dec.single_symbol, h.N, s) == cudaSuccess ? RECOIL_OK : RECOIL_E_CUDA;
  const uint16_t *words = reinterpret_cast<const uint16_t *>(buf + dd->coff + h.wstart);
  return launch_decode(&dd->dec, ws, words, d_out, s);
}

extern "C" int recoil_device_decoder_status(recoil_device_decoder *dec, const void *d_workspace, void *stream,
                                            uint64_t *bad_task) {
  if (!dec) return RECOIL_E_ARG;
  return recoil_decoder_status(reinterpret_cast<recoil_decoder *>(&reinterpret_cast<DeviceDecoder *>(dec)->dec),
                               d_workspace, stream, bad_task);
}

extern "C" int recoil_device_decoder_launches(const recoil_device_decoder *dec) {
  if (!dec) return RECOIL_E_ARG;
  const DeviceDecoder *dd = reinterpret_cast<const DeviceDecoder *>(dec);
  const int parse = dd->h.P ? 4 : 1;  // k_global (+ k_spec, k_resolve, k_write)
  if (!dd->h.N) return parse;
  return parse + 2 + (dd->dec.single_symbol >= 0 ? 0 : 1);  // + k_lut, k_heads, the decode kernel
}

extern "C" void recoil_device_decoder_destroy(recoil_device_decoder *dec) {
  delete reinterpret_cast<DeviceDecoder *>(dec);
}

// ---------------------------------------------------------------------------
// combine on the GPU
// ---------------------------------------------------------------------------

extern "C" int recoil_device_combine_plan(const uint8_t *head, uint64_t head_len, uint64_t container_len,
                                          uint32_t target_splits, uint64_t *out_capacity, uint64_t *workspace_bytes) {
  if (!out_capacity || !workspace_bytes || target_splits < 1) return RECOIL_E_ARG;
  dm::Head h;
  int rc = read_head(head, head_len, container_len, &h);
  if (rc) return rc;
  if (h.M > 1 && h.wstart - h.gpos > (uint64_t)dm::kMaxChunks * 60000) return RECOIL_E_UNSUPPORTED;
  const dm::Layout L = layout_for(h);
  const uint64_t P2 = target_splits >= h.M ? h.P : h.P / ceil_div(h.M, target_splits);
  // header + model + finals, new global series (<= 2 x (5 + 34 bits per point)), kept records, words
  *out_capacity = h.gpos + (10 + 68 * P2 + 7) / 8 + (h.wstart - h.gpos) + 2 * h.B + 16;
  *workspace_bytes = L.total + dm::a256(8 * (P2 + 1)) + 256;
  return RECOIL_OK;
}

extern "C" int recoil_device_combine(const uint8_t *head, uint64_t head_len, const uint8_t *d_in, uint64_t in_len,
                                     uint32_t target_splits, uint8_t *d_out, uint64_t out_capacity, void *d_workspace,
                                     uint64_t *d_out_len, void *stream) {
  if (!d_in || !d_out || !d_workspace || !d_out_len || target_splits < 1) return RECOIL_E_ARG;
  dm::Head h;
  int rc = read_head(head, head_len, in_len, &h);
  if (rc) return rc;
  uint64_t cap = 0, wsb = 0;
  if ((rc = recoil_device_combine_plan(head, head_len, in_len, target_splits, &cap, &wsb))) return rc;
  if (out_capacity < cap) return RECOIL_E_BUFFER;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long *tot = reinterpret_cast<unsigned long long *>(d_out_len);
  if (target_splits >= h.M) {  // identity (nothing to drop)
    if (cudaMemcpyAsync(d_out, d_in, in_len, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(d_out_len, &h.len, 8, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return RECOIL_E_CUDA;
    return RECOIL_OK;
  }
  const dm::Layout L = layout_for(h);
  char *ws = static_cast<char *>(d_workspace);
  if ((rc = run_parse(h, L, d_in, 0, ws, s))) return rc;
  const uint64_t kstep = ceil_div(h.M, target_splits), P2 = h.P / kstep, M2 = P2 + 1;
  const uint64_t Eb2 = ceil_div(h.B, M2), Eg2 = ceil_div(h.G, M2);
  uint64_t *rec_out = reinterpret_cast<uint64_t *>(ws + L.total);
  uint32_t *wmax = reinterpret_cast<uint32_t *>(ws + L.total + dm::a256(8 * (P2 + 1)));
  const uint64_t *offset = reinterpret_cast<const uint64_t *>(ws + L.offset);
  const uint32_t *maxg = reinterpret_cast<const uint32_t *>(ws + L.maxg);
  const uint64_t *rec_off = reinterpret_cast<const uint64_t *>(ws + L.rec_off);
  // widths of the new series, then the header / model / finals (copied, M patched) and the series bits
  const uint32_t init[2] = {1, 1};
  if (cudaMemcpyAsync(wmax, init, 8, cudaMemcpyHostToDevice, s) != cudaSuccess) return RECOIL_E_CUDA;
  const uint32_t gb = (uint32_t)std::max<uint64_t>(1, ceil_div(P2, 256));
  dm::k_cmb_width<<<gb, 256, 0, s>>>(P2, kstep, Eb2, Eg2, offset, maxg, wmax);
  // the series region's size depends on the widths: read them back (one 8-byte sync), as the
  // host must size the output anyway
  uint32_t w[2];
  if (cudaMemcpyAsync(w, wmax, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return RECOIL_E_CUDA;
  DeviceStatus st;
  if (cudaMemcpy(&st, ws, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) return RECOIL_E_CUDA;
  if (st.flags) return RECOIL_E_INCONSISTENT;
  if (w[0] > 33 || w[1] > 33) return RECOIL_E_OVERFLOW;
  const uint64_t gbits = 10 + P2 * (w[0] + 1) + P2 * (w[1] + 1), gbytes = (gbits + 7) / 8;
  const uint64_t rec_base = h.gpos + gbytes;
  uint8_t hdr[28];
  if (cudaMemcpyAsync(d_out, d_in, h.gpos, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(hdr, d_in, 28, cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess)
    return RECOIL_E_CUDA;
  for (int k = 0; k < 4; ++k) hdr[8 + k] = (uint8_t)(M2 >> (8 * k));
  if (cudaMemcpyAsync(d_out + 8, hdr + 8, 4, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemsetAsync(d_out + h.gpos, 0, gbytes, s) != cudaSuccess)
    return RECOIL_E_CUDA;
  dm::CmbArgs ca{P2, kstep, Eb2, Eg2, h.gpos, rec_base};
  dm::k_cmb_series<<<gb, 256, 0, s>>>(ca, offset, maxg, wmax, d_out);
  dm::k_cmb_scan<<<1, 1024, 0, s>>>(P2, kstep, rec_off, rec_out);
  const uint32_t rb = (uint32_t)std::max<uint64_t>(1, ceil_div(32 * P2, 256));
  dm::k_cmb_records<<<rb, 256, 0, s>>>(P2, kstep, d_in, rec_off, rec_out, rec_base, d_out);
  dm::k_cmb_total<<<1, 1, 0, s>>>(rec_base, rec_out, P2, 2 * h.B, tot);
  if (cudaGetLastError() != cudaSuccess) return RECOIL_E_CUDA;
  // the word stream follows the kept records: one more 8-byte read-back places it, then a
  // device-to-device copy (the driver's copy engine handles the byte misalignment)
  uint64_t rec_bytes = 0;
  if (cudaMemcpyAsync(&rec_bytes, rec_out + P2, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return RECOIL_E_CUDA;
  if (rec_base + rec_bytes + 2 * h.B > out_capacity) return RECOIL_E_BUFFER;
  if (h.B && cudaMemcpyAsync(d_out + rec_base + rec_bytes, d_in + h.wstart, 2 * h.B, cudaMemcpyDeviceToDevice, s) !=
                 cudaSuccess)
    return RECOIL_E_CUDA;
  return RECOIL_OK;
}
