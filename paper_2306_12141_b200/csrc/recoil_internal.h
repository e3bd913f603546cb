// recoil_internal.h -- internal types of librecoil (host C++ and CUDA).
// Not part of the ABI; the ABI is include/recoil.h.
#pragma once
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "recoil.h"

namespace recoil {

constexpr uint32_t kLanes = 32;          // W (tab:rans_params P:419)
constexpr uint32_t kL = 1u << 16;        // L
constexpr uint32_t kWordBits = 16;       // b
constexpr uint32_t kChunkWords = 256;    // device word-window chunk: 32 lanes x 16 B
constexpr uint32_t kBlockBytes = 512;    // device output block: 16 groups x 32 symbols
constexpr uint32_t kMaxGpuProbBits = 16; // GPU decode: packed u32 LUT up to n = 12, split tables above
constexpr uint32_t kNoFinals = 0xFFFFFFFFu;
constexpr int64_t kNoEndCheck = INT64_MIN;
// Adaptive model tables: per model 2^cbits coarse slot buckets, a row of 2^cbits + 2
// u16 entry indices (2^cbits + 1 boundaries + 1 pad).  The 32-warp adaptive kernel
// takes the most bits in 9..7 whose tables fit beside its layout (fewer binary-
// search steps: 2^25 latent symbols 193 / 248 / 275 G symbols/s at 6 / 8 / 9 bits);
// the 8-warp fallback for large model sets uses 6.
constexpr uint32_t kCoarseBitsWide = 9, kCoarseBitsWideMin = 7, kCoarseBitsNarrow = 6;
// Decode kernel CTA sizes in warps (decode.cu): static codec 2 CTAs x 24 per SM;
// adaptive one CTA of 32, or 8-warp CTAs when the model tables need the room.
constexpr uint32_t kWarpsStatic = 24, kWarpsAdaptive = 32, kWarpsAdaptiveNarrow = 8;
#ifdef __CUDACC__
#define RECOIL_HD __host__ __device__
#else
#define RECOIL_HD
#endif
RECOIL_HD constexpr uint32_t coarse_row(uint32_t cbits) { return (1u << cbits) + 2; }
// Bytes of the packed adaptive tables (pack_adaptive) for K models, E entries.
RECOIL_HD constexpr uint64_t adaptive_table_bytes(uint32_t K, uint64_t E, uint32_t cbits) {
  return ((uint64_t)K * coarse_row(cbits) * 2 + 15) / 16 * 16 + 4 * (((E + 3) & ~3ull) + K);
}
// Shared-memory layout bytes of the 32-warp adaptive kernel and the opt-in limit it
// is planned against (sm_100: 227 KB per block); decode.cu checks both at run time.
extern const uint64_t kAdaptiveWideLayoutBytes;
constexpr uint64_t kSmemOptinBytes = 232448;

// Parsed container of either kind. Recoil: M tasks, M-1 split points.
// Partitioned: M partitions (tasks), no points.
struct Container {
  bool partitioned = false;
  bool adaptive = false;          // "RCA1": 16-bit symbols, index-keyed model set (P:227 (3))
  uint32_t n = 0, W = 0, M = 0;
  uint64_t N = 0, B = 0, G = 0;
  uint32_t f[256] = {0};          // static model ("RCL1" / "RCV1")
  uint32_t K = 0;                 // adaptive: model k = values mbase[k] .. + mlen[k] - 1,
  std::vector<uint32_t> mbase, mlen, mf;  // frequencies mf[off_k + j] (sum 2^n each)
  std::vector<uint32_t> finals;   // Recoil: W final states; partitioned: M x W
  std::vector<uint64_t> offset;   // Recoil: M-1 split offsets (word index of the boundary event)
  std::vector<uint64_t> maxg;     // Recoil: M-1 anchor (max) group IDs
  std::vector<uint16_t> state;    // Recoil: (M-1) x W anchor states (< L)
  std::vector<uint16_t> gdiff;    // Recoil: (M-1) x W group differences to the anchor
  std::vector<int64_t> sync_start, bidx;  // Recoil: per point min / max anchor index (full parse)
  bool light = false;             // Recoil light parse: state/gdiff/sync_start/bidx left empty
  std::vector<uint64_t> rec_off;  // Recoil: container byte offset of each split record (P + 1 entries)
  const uint8_t *bytes = nullptr; // the container
  std::vector<uint64_t> part_words; // partitioned: M word counts
  const uint8_t *words = nullptr; // B little-endian u16
  uint64_t header_bytes = 0, meta_bytes = 0, total_bytes = 0;
};

int parse_container(const uint8_t *c, uint64_t len, Container *out, bool light = false);
// Light parse helper: sync start and boundary index of split point k (decodes one record).
int point_span_light(const Container &c, uint64_t k, int64_t *sync_start, int64_t *bidx);
// Serialise a Recoil container (offset/maxg/state/gdiff/finals/f from `c`,
// words from `words` (B little-endian u16 bytes)).  out == nullptr: size only.
int write_recoil_container(const Container &c, const uint8_t *words, uint8_t *out, uint64_t *len);

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Anchor span of split point k: sync start (min anchor index) and boundary index (max).
void point_span(const Container &c, uint64_t k, int64_t *sync_start, int64_t *bidx);

// ---------------------------------------------------------------------------
// Device task record: 176 B, 16-B aligned.
// ---------------------------------------------------------------------------
struct alignas(16) TaskRec {
  int64_t cursor0;      // slice-relative word index of the task's first read
  int64_t end_cursor;   // slice-relative cursor the task must end at, or kNoEndCheck
  uint64_t commit_lo;   // first committed symbol (absolute)
  uint64_t commit_hi;   // last committed symbol (absolute, inclusive)
  uint64_t write_hi;    // GPU writes the 16-B chunks inside [32 group(commit_lo), write_hi):
                        // every symbol there is decoded by this task after it is synchronised
  int32_t start_group;  // group of the first decode step
  uint32_t finals_idx;  // kNoFinals: lanes[] low 16 bits are the init states; else 32 u32 states
  uint32_t task_id;     // container task index (error reporting)
  uint32_t pad[3];
  uint32_t lanes[32];   // (state16 | diff16 << 16), diff = start_group - init_group
};
static_assert(sizeof(TaskRec) == 192, "TaskRec layout");

// Fused-a1 task header (Recoil containers on the GPU, DESIGN.md row a1): the
// O(M) sequential part of the metadata (global series, record offsets) is
// decoded on the host; the kernel expands the O(M W) per-lane part (anchor
// states and group differences) from the raw records itself.
struct alignas(16) TaskHead {
  int32_t cursor0;      // slice-relative first word (offset of point t; B - 1 for the last task)
  int32_t start_group;  // anchor group of point t (G - 1 for the last task)
  uint32_t rec;         // byte offset of point t's record in the device record area
  uint32_t rec_prev;    // byte offset of point t-1's record
  uint32_t maxg_prev;   // anchor group of point t-1
  uint32_t flags;       // kHeadLast: entered from the final states; kHeadFirst: t == 0
  uint32_t task_id;
  int32_t end_cursor;   // t == 0: slice-relative end cursor (-1 - word_lo)
};
static_assert(sizeof(TaskHead) == 32, "TaskHead layout");
constexpr uint32_t kHeadLast = 1, kHeadFirst = 2;

struct DeviceStatus {   // first 16 B of the workspace, zeroed before every decode
  uint32_t flags;       // bit 0 underflow, bit 1 end-state mismatch, bit 2 inconsistent metadata,
                        // bit 3 a task window too long for the 32-bit block offsets (E_UNSUPPORTED)
  uint32_t bad_task;    // atomicMax of (0xFFFFFFFF - failing task id); 0 = none
  uint32_t next_task;   // persistent-warp task counter
  uint32_t pad;
};

// Host-side decode plan (the recoil_decoder handle).
struct Decoder {
  std::shared_ptr<const Container> c;  // parsed container (shared by the chunks of a pipeline)
  recoil_plan plan{};
  std::vector<uint8_t> lut;        // n <= 12: 2^n packed u32 s | bias << 8 | f << 20;
                                   // n >= 13: 2^n symbol bytes + 256 x u32 (f | F << 16)
  std::vector<uint32_t> finals;    // K x 32 u32 states referenced by finals_idx
  std::vector<TaskRec> tasks;      // prebuilt records (partitioned containers, CPU decoder)
  bool fused = false;              // Recoil on the GPU: heads + raw records, expanded in-kernel
  std::vector<TaskHead> heads;
  uint64_t rec_src = 0, rec_len = 0;  // container byte span of the records the plan needs
  uint64_t lut_off = 0, finals_off = 0, tasks_off = 0, rec_off = 0;  // workspace byte offsets
  uint32_t n_tasks = 0;
  int single_symbol = -1;          // >= 0: the model has one symbol (f = 2^n): decode = fill
  uint32_t ad_K = 0, ad_E = 0;     // adaptive: models, table entries (lut = coarse | entries | offsets)
  int blocks_per_sm = 0, sm_count = 0;  // launch geometry (occupancy API), cached
  bool ad_narrow = false;          // adaptive: 8-warp CTAs (the model tables leave no room for 32 warps)
  uint32_t ad_cbits = 0;           // adaptive: coarse bucket bits of the packed tables
};

int build_decoder(const uint8_t *c, uint64_t len, uint64_t task_begin, uint64_t task_end, Decoder *d,
                  bool for_gpu);
// Plan tasks [task_begin, task_end) of an already parsed container.
int build_decoder_from(std::shared_ptr<const Container> c, uint64_t task_begin, uint64_t task_end, Decoder *d,
                       bool for_gpu);
// recoil_decode for a workspace whose zeroed status block was uploaded with it
// (no reset; decode.cu).
int decode_staged(Decoder *d, char *ws, const uint16_t *d_words, uint8_t *d_out, void *stream);
// Launch the decode kernel of a prepared plan (no status reset, no single-symbol shortcut).
int launch_decode(Decoder *d, char *ws, const uint16_t *d_words, uint8_t *d_out, void *stream);
// Contiguous task ranges with ~equal committed symbols (recoil_shard_plan).
void shard_bounds(const Container &c, uint32_t n_shards, uint64_t *bounds);
void shard_bounds_range(const Container &c, uint64_t task_begin, uint64_t task_end, uint32_t n_shards,
                        uint64_t *bounds);
void pack_lut(const uint32_t f[256], uint32_t n, std::vector<uint8_t> *lut);
// Adaptive model tables for the GPU: K rows of 2^cbits + 2 u16
// coarse bucket boundaries (entry holding each of the 2^cbits buckets' first slot,
// + end, + pad; 16-B aligned), E entries F | (f-1) << 16 (padded to 4), K value
// offsets.  cbits is chosen per plan: 9..7 on the 32-warp kernel, 6 on the 8-warp one.
// E_UNSUPPORTED if E > 65535.
int pack_adaptive(const Container &c, uint32_t cbits, std::vector<uint8_t> *blob, uint32_t *K, uint32_t *E);


}  // namespace recoil
