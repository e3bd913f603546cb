/*
 * recoil.h -- C ABI of the B200-native Recoil library (librecoil.so).
 *
 * Recoil (Lin et al., arXiv 2306.12141; /root/reference/PAPER.md cited as
 * P:<line>) makes ONE W = 32-way interleaved rANS bitstream decodable from
 * the middle by storing, at chosen renormalisation points ("splits"), each
 * lane's 16-bit state and symbol group and the bitstream offset; decoding of
 * the splits then runs in parallel, one warp per split, on sm_100a.
 *
 * Fixed parameters (tab:rans_params P:400-423): 32-bit states, L = 2^16,
 * b = 16-bit words, 8-bit symbols, W = 32 lanes, 1 <= n <= 16 probability
 * bits.  The GPU decoder packs s, f, F into one u32 LUT entry for n <= 12
 * and uses a slot -> symbol byte table plus a per-symbol (f, F)
 * table for 13 <= n <= 16.
 * Symbol i (0-based) belongs to lane i mod 32 and group i / 32.
 *
 * Conventions for every call:
 *  - Return value: RECOIL_OK (0) or a negative RECOIL_E_* code; no call
 *    aborts the process.  recoil_strerror() names a code.
 *  - The caller owns every buffer passed in, host or device; the library
 *    never frees or retains them past the call, except as stated for
 *    recoil_decoder_upload (host source must stay valid until the stream
 *    passes the copy).  Handles own only host memory.
 *  - Device memory and streams come from the caller (PyTorch in this repo);
 *    `cuda_stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Sizes: passing out == NULL stores the required (for encode: an upper
 *    bound) length in *len and returns RECOIL_OK; a too-small buffer returns
 *    RECOIL_E_BUFFER with the required length in *len.
 *  - Reentrant; no global state.  A handle is used by one thread at a time.
 *  - Containers are little-endian byte strings; see DESIGN.md "Container".
 */
#ifndef RECOIL_H
#define RECOIL_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RECOIL_OK 0
#define RECOIL_E_ARG (-1)          /* bad argument (NULL pointer, range)          */
#define RECOIL_E_EMPTY (-2)        /* model from an empty histogram        */
#define RECOIL_E_ALPHABET (-3)     /* more distinct symbols than 2^n       */
#define RECOIL_E_ZERO_FREQ (-4)    /* symbol to encode has f = 0          */
#define RECOIL_E_OVERFLOW (-5)     /* a metadata value does not fit its field     */
#define RECOIL_E_BAD_MAGIC (-6)    /* not a Recoil / partitioned container        */
#define RECOIL_E_VERSION (-7)      /* unsupported version / symbol width          */
#define RECOIL_E_TRUNCATED (-8)    /* container shorter than its header says      */
#define RECOIL_E_INCONSISTENT (-9) /* metadata inconsistent               */
#define RECOIL_E_UNDERFLOW (-10)   /* device: a task read below its word slice    */
#define RECOIL_E_SYNC (-11)        /* device: end state != (x = L, cursor = -1)   */
#define RECOIL_E_CUDA (-12)        /* a CUDA runtime call failed                  */
#define RECOIL_E_NOMEM (-13)       /* host allocation failed                      */
#define RECOIL_E_BUFFER (-14)      /* output buffer too small (*len = required)   */
#define RECOIL_E_UNSUPPORTED (-15) /* valid but outside the GPU path (slice >= 2^31 words) */

const char *recoil_strerror(int status);

/* ---------------------------------------------------------------------- */
/* Model                                                                   */
/* ---------------------------------------------------------------------- */

/* Quantised PDF f(t) with sum f = 2^prob_bits.  The paper does not
 * give its quantiser: floor(h 2^n / total), present symbols raised to
 * 1, shortfall by largest remainder (ties: smaller symbol), excess (from the
 * raise) taken from the largest f (ties: smaller count, then smaller symbol).
 * hist: 256 counts.  freqs_out: 256 entries.  Errors: E_ARG (n outside 1..16),
 * E_EMPTY, E_ALPHABET. */
/* Reading Z19's quantiser over `count` entries (recoil_build_model = 256):
 * f = floor(hist 2^n / total), present entries raised to 1, shortfall by
 * largest remainder (ties: lower index), excess from the largest f.  Used for
 * the per-model frequencies of the adaptive codec.  Errors as recoil_build_model. */
int recoil_quantize(const uint64_t *hist, uint32_t count, uint32_t prob_bits, uint32_t *freqs_out);

int recoil_build_model(const uint64_t hist[256], uint32_t prob_bits, uint32_t freqs_out[256]);

/* ---------------------------------------------------------------------- */
/* Encode / combine / inspect (host)                                       */
/* ---------------------------------------------------------------------- */

/* Serial 32-way interleaved rANS encode (Eq. 1, Eq. 3) of
 * symbols[0..n_symbols) under freqs (sum = 2^prob_bits), plus the split
 * heuristic (reading Z10') choosing up to n_splits - 1
 * split points (the backward scan of P:301 gives each point's anchors), and
 * the difference-coded metadata.  Result: a Recoil container
 * ("RCL1") in container[0..*container_len).  Fewer splits than requested are
 * produced when the stream has too few renormalisation points.
 * container == NULL: *container_len = an upper bound on the size.
 * Errors: E_ARG, E_ZERO_FREQ, E_OVERFLOW, E_BUFFER, E_NOMEM. */
int recoil_encode(const uint8_t *symbols, uint64_t n_symbols, const uint32_t freqs[256],
                  uint32_t prob_bits, uint32_t n_splits, uint8_t *container,
                  uint64_t *container_len);

/* Adaptive Recoil encode (P:227 item (3)): 16-bit symbols,
 * symbol i coded with model model_ids[i] < n_models (<= 256).  Model k covers
 * the values model_base[k] .. model_base[k] + model_len[k] - 1 (<= 65535) with
 * frequencies freqs[off_k + j], off_k = model_len[0] + ... + model_len[k-1],
 * each model summing to 2^prob_bits.  Same split heuristic and metadata as
 * recoil_encode; container "RCA1" (the model set replaces the model block).
 * Errors: E_ARG, E_ZERO_FREQ (a symbol outside its model or with f = 0),
 * E_OVERFLOW, E_BUFFER, E_NOMEM. */
int recoil_encode_adaptive(const uint16_t *symbols, uint64_t n_symbols, const uint8_t *model_ids,
                           uint32_t n_models, const uint32_t *model_base, const uint32_t *model_len,
                           const uint32_t *freqs, uint32_t prob_bits, uint32_t n_splits, uint8_t *container,
                           uint64_t *container_len);

/* Decoder-adaptive combine: keep the split points at
 * 1-based positions k, 2k, ... with k = ceil(M / target_splits) and rewrite
 * the metadata for the new M; the word stream is copied verbatim.
 * target_splits >= M: byte-identical copy.  Errors: E_ARG, container errors,
 * E_BUFFER. */
int recoil_combine_splits(const uint8_t *in, uint64_t in_len, uint32_t target_splits, uint8_t *out,
                          uint64_t *out_len);

typedef struct {
  uint64_t n_symbols;    /* N */
  uint64_t n_words;      /* B (16-bit words) */
  uint32_t n_splits;     /* M (tasks); partitions for a partitioned container */
  uint32_t prob_bits;    /* n */
  uint32_t lanes;        /* W (32) */
  uint32_t partitioned;  /* 0 = Recoil "RCL1", 1 = partitioned "RCV1" */
  uint64_t header_bytes; /* fixed header + model block */
  uint64_t meta_bytes;   /* final states + split metadata (or offset table + states) */
  uint64_t word_bytes;   /* 2 B */
  uint64_t total_bytes;
  uint32_t symbol_bits;  /* 8 ("RCL1", "RCV1") or 16 ("RCA1", adaptive) */
  uint32_t n_models;     /* 1, or K for an adaptive container */
} recoil_info;

/* Parse and validate a container (either kind).  Errors: container errors. */
int recoil_inspect(const uint8_t *container, uint64_t len, recoil_info *info);

/* Conventional "partitioning symbols" codec for the paper's
 * comparison: partition p = groups [floor(p G/P), floor((p+1) G/P)), each an
 * independent 32-way interleaved codec; offset table + final states.
 * container == NULL: upper bound.  Errors as recoil_encode. */
int recoil_partitioned_encode(const uint8_t *symbols, uint64_t n_symbols, const uint32_t freqs[256],
                              uint32_t prob_bits, uint32_t n_partitions, uint8_t *container,
                              uint64_t *container_len);

/* ---------------------------------------------------------------------- */
/* GPU decode (sm_100a)                                                    */
/* ---------------------------------------------------------------------- */

typedef struct recoil_decoder recoil_decoder;

/* Layout of one decode plan.  All device buffers are provided by the caller. */
typedef struct {
  uint64_t task_begin, task_end; /* tasks [begin, end) of the container            */
  uint32_t n_tasks;              /* tasks with work in this plan                    */
  uint32_t prob_bits;
  uint64_t word_lo;              /* d_words[0] holds stream word word_lo (mult. of 256) */
  uint64_t word_count;           /* d_words must hold word_count words (mult. of 256)   */
  uint64_t out_lo, out_hi;       /* this plan writes symbols [out_lo, out_hi)            */
  uint64_t out_base;             /* d_out[0] is symbol out_base (out_lo & ~511)          */
  uint64_t out_count;            /* d_out must hold out_count (>= out_hi - out_base) symbols */
  uint64_t workspace_bytes;      /* d_workspace size (LUT + task table + status)       */
  uint64_t upload_bytes;         /* bytes recoil_decoder_upload copies host->device     */
  uint32_t symbol_bytes;         /* 1 (8-bit symbols) or 2 (adaptive "RCA1", uint16_t)   */
  uint32_t n_models;             /* adaptive: K models; else 1                          */
  uint32_t coarse_bits;          /* adaptive: coarse slot buckets per model = 2^coarse_bits; else 0 */
  uint32_t warps_per_block;      /* the decode kernel's CTA size for this plan (warps)  */
} recoil_plan;

/* Host half of the path (DESIGN.md row a1): parse the container
 * and expand the split metadata of tasks [task_begin, task_end) into the
 * per-warp task table (task_end = UINT64_MAX: all tasks).  Task t < M-1
 * enters at split point t+1; task M-1 enters from the final
 * states.  Works on either container kind (partitions = tasks).
 * The container bytes must stay valid while the handle is used.
 * Errors: container errors, E_ARG, E_NOMEM, E_UNSUPPORTED (word slice of
 * 2^31 words or more). */
int recoil_decoder_create(const uint8_t *container, uint64_t len, uint64_t task_begin,
                          uint64_t task_end, recoil_decoder **out);

/* Decoder-side combine (P:266-272 on the client): plan the decode with only
 * the split points recoil_combine_splits(container, target_splits) would keep
 * (1-based positions k, 2k, ..., k = ceil(M / target_splits)), reading the
 * kept records in place -- no rewritten container, no copy of the word
 * stream.  Output identical to decoding the combined container; task indices
 * refer to the kept splits.  Errors as recoil_decoder_create; E_ARG for a
 * partitioned container. */
int recoil_decoder_create_subset(const uint8_t *container, uint64_t len, uint32_t target_splits,
                                 uint64_t task_begin, uint64_t task_end, recoil_decoder **out);
/* Decoder-side combine into tasks of unequal length (P:266-272 on the client:
 * which split points a decoder uses is its choice).  Tasks in stream order:
 * the first run_tasks[0] tasks each span run_splits[0] consecutive encoder
 * splits, the next run_tasks[1] span run_splits[1], ...; the last task takes
 * the splits that remain (fewer tasks if the splits run out).  The kernel's
 * first wave takes tasks 0, 1, ... and later ones come from its atomic
 * counter, so long tasks first and short ones last (longest-processing-time
 * order) let the warps the SM schedulers favour take more of the tail.  Output
 * identical to any other plan.  Errors as recoil_decoder_create_subset; E_ARG
 * for n_runs = 0 or a run of 0 splits. */
int recoil_decoder_create_grouped(const uint8_t *container, uint64_t len, uint32_t n_runs,
                                  const uint32_t *run_tasks, const uint32_t *run_splits, recoil_decoder **out);
/* Decoder-adaptive scalability in one call: the whole stream planned for the
 * parallelism of `device` -- when the container holds more split points than
 * waves_x100 / 100 waves of the decode kernel's resident warps (0: 150, the measured
 * best), the decode uses the points recoil_combine_splits would keep for
 * that count (in place, nothing rewritten); else all of them.  Errors as
 * recoil_decoder_create, E_CUDA (occupancy query). */
int recoil_decoder_create_for_device(const uint8_t *container, uint64_t len, int device, uint32_t waves_x100,
                                     recoil_decoder **out);
int recoil_decoder_plan(const recoil_decoder *dec, recoil_plan *plan);

/* Asynchronous host->device copy on cuda_stream of the packed LUT and task
 * table into d_workspace and of the plan's word slice (zero padded) into
 * d_words.  Source = the handle's host table and the container bytes.
 * Errors: E_ARG, E_CUDA. */
int recoil_decoder_upload(recoil_decoder *dec, void *d_workspace, uint16_t *d_words, void *cuda_stream);

/* Launch the decode kernel on cuda_stream (asynchronous; stream-ordered):
 * one warp per split, smem LUT, cp.async word window, ballot/popc
 * refills, 16-byte output stores.  Writes symbols [out_lo, out_hi) to
 * d_out[i - out_base]; it may also write, inside d_out[0, out_count), the
 * neighbouring symbols of partially committed 32-symbol groups (always their
 * correct decoded values) and padding past N.  Clears and then sets the
 * device status word.  Errors: E_ARG, E_CUDA. */
int recoil_decode(recoil_decoder *dec, void *d_workspace, const uint16_t *d_words, uint8_t *d_out,
                  void *cuda_stream);

/* Synchronise cuda_stream and read the device status word of the last
 * decode: RECOIL_OK, RECOIL_E_UNDERFLOW or RECOIL_E_SYNC.
 * *bad_task (may be NULL) = first failing task or UINT64_MAX. */
int recoil_decoder_status(recoil_decoder *dec, const void *d_workspace, void *cuda_stream,
                          uint64_t *bad_task);

/* Number of kernel launches one recoil_decode issues (for launch accounting). */
int recoil_decoder_launches(const recoil_decoder *dec);

void recoil_decoder_destroy(recoil_decoder *dec);

/* Adaptive decode ("RCA1" containers; NEXT rows 1 + 4 of SURVEY.md §8(f)):
 * symbol i was coded with model d_model_ids[i] (P:227 item (3): "the
 * probability distribution used in every iteration is dynamic, determined
 * using symbol index as a key"), 16-bit symbols.  d_model_ids: device,
 * one byte per symbol of the WHOLE stream (indexed from symbol 0, 16-byte
 * aligned; ids >= K are clamped).  d_out: uint16_t symbols, d_out[i - out_base]
 * (plan.symbol_bytes = 2).  Otherwise as recoil_decode.  The model tables go
 * to shared memory: E_UNSUPPORTED if they exceed it (more than 65535 table
 * entries in total, or too large for one block).  Errors: E_ARG (static
 * container, misaligned ids), E_CUDA, E_UNSUPPORTED. */
int recoil_decode_adaptive(recoil_decoder *dec, void *d_workspace, const uint16_t *d_words,
                           const uint8_t *d_model_ids, uint16_t *d_out, void *cuda_stream);

/* Resident warps per SM of the decode kernel on `device` and the SM count
 * (cudaOccupancyMaxActiveBlocksPerMultiprocessor): the split count
 * that fills the GPU is warps_per_sm * sm_count * waves. */
int recoil_decode_occupancy(int device, uint32_t prob_bits, int *warps_per_sm, int *sm_count);  /* 1 <= n <= 16 */
/* The same for the adaptive kernel of a container with n_models models and
 * n_entries model-table entries in total (the decoded values of all models up to
 * each model's last nonzero frequency): the plan runs 32-warp CTAs with 2^9,
 * 2^8 or 2^7 coarse buckets per model (the most that fit beside that layout in
 * one block's shared memory), else 8-warp CTAs with 2^6 buckets. */
int recoil_decode_occupancy_adaptive(int device, uint32_t n_models, uint64_t n_entries, int *warps_per_sm,
                                     int *sm_count);

/* ---------------------------------------------------------------------- */
/* End-to-end pipelined decode on one GPU (host container -> host symbols)  */
/* ---------------------------------------------------------------------- */

typedef struct recoil_pipeline recoil_pipeline;

/* Cut the container's tasks [task_begin, task_end) (UINT64_MAX: all) into
 * n_chunks contiguous ranges of ~equal committed symbols (as recoil_shard_plan).  The container bytes must stay
 * valid while the handle is used (its words are copied from them; pinned
 * memory lets those copies run asynchronously).  Owns pinned host staging
 * and CUDA events.  Errors: container errors, E_ARG, E_NOMEM, E_CUDA. */
int recoil_pipeline_create(const uint8_t *container, uint64_t len, uint64_t task_begin, uint64_t task_end,
                           uint32_t n_chunks, recoil_pipeline **out);

/* Device scratch the caller must provide to recoil_pipeline_run with
 * n_streams streams (1 <= n_streams <= 8): one buffer set per stream. */
int recoil_pipeline_device_bytes(const recoil_pipeline *p, uint32_t n_streams, uint64_t *bytes);

/* One end-to-end decode: per chunk k, in device buffer set k % n_streams, the
 * host expands the chunk's tasks (a1), then H2D of LUT + task table (from
 * pinned staging) and of the chunk's word slice on streams[0], the decode
 * kernel on streams[1], and D2H of the chunk's symbols into host_out[out_lo,
 * out_hi) (absolute symbol indices: host_out is indexed from symbol 0) and of
 * its status word on streams[2] (with fewer streams the roles share), chained
 * by events.  Copies in of later chunks overlap copies out of earlier ones.  Returns
 * once everything is enqueued; call recoil_pipeline_status to wait.
 * host_out: N bytes (pinned for asynchronous copies).  Errors: E_ARG, E_CUDA,
 * container errors. */
int recoil_pipeline_run(recoil_pipeline *p, void *d_scratch, uint8_t *host_out, void *const *streams,
                        uint32_t n_streams);

/* recoil_pipeline_run with host_out indexed from symbol host_first instead of 0:
 * the chunk symbols [out_lo, out_hi) go to host_out[out_lo - host_first, ...),
 * so a shard's caller needs only a buffer of its own span (host_first = the
 * span's out_lo from recoil_pipeline_span).  E_ARG if host_first > out_lo. */
int recoil_pipeline_run_at(recoil_pipeline *p, void *d_scratch, uint8_t *host_out, uint64_t host_first,
                           void *const *streams, uint32_t n_streams);

/* Committed symbols [*out_lo, *out_hi) of the pipeline's task range. */
int recoil_pipeline_span(const recoil_pipeline *p, uint64_t *out_lo, uint64_t *out_hi);

/* Synchronise the streams and fold the chunks' status words (as
 * recoil_decoder_status).  *bad_task (may be NULL): first failing task. */
int recoil_pipeline_status(recoil_pipeline *p, void *const *streams, uint32_t n_streams, uint64_t *bad_task);

/* Kernel launches of the last run. */
int recoil_pipeline_launches(const recoil_pipeline *p);

void recoil_pipeline_destroy(recoil_pipeline *p);

/* ---------------------------------------------------------------------- */
/* On-device metadata path          */
/* ---------------------------------------------------------------------- */

/* The client copies the received container to the GPU unchanged; the split
 * metadata is decoded there (global series, split-record offsets by a
 * speculative chunked parse, LUT, the 192-B task records of every split task)
 * and the decode kernel streams those records.  The host reads only the fixed
 * header and the model block.  Whole stream, "RCL1" only. */
typedef struct recoil_device_decoder recoil_device_decoder;
typedef struct {
  uint64_t container_offset; /* copy the container to d_buffer + container_offset (puts its words 512-B aligned) */
  uint64_t buffer_bytes;     /* d_buffer size: offset + container + zeroed word padding (>= 256 words + 256 B) */
  uint64_t workspace_bytes;  /* d_workspace size (status, parse results, LUT, task records) */
  uint64_t out_count;        /* d_out bytes (N rounded up to 16) */
  uint64_t n_symbols;        /* N */
  uint32_t n_tasks;          /* split tasks (M; 0 for N = 0) */
  uint32_t prob_bits;        /* n */
} recoil_device_plan;

/* head: the first head_len bytes of the container (the 28-byte header and the
 * model block at least: 30 + 5 x symbols); container_len: its full length.
 * Errors: E_ARG, E_BAD_MAGIC, E_VERSION, E_TRUNCATED, E_INCONSISTENT (header or
 * model), E_UNSUPPORTED ("RCA1" / "RCV1", more than ~23 MB of split metadata,
 * a word stream of >= 2^31 words), E_NOMEM. */
int recoil_device_decoder_create(const uint8_t *head, uint64_t head_len, uint64_t container_len,
                                 recoil_device_decoder **out);
/* The split tasks [task_begin, task_end) only (a multi-GPU shard: the tasks
 * are independent; task_end = UINT64_MAX: to the last task).  Every split record is
 * still parsed on the device (the series and record offsets are a list), the task
 * records and the decode cover the range; the output keeps absolute symbol indices
 * (d_out holds out_count = N rounded up to 16 bytes; the range writes its committed
 * span, recoil_device_decoder_span, plus at most the 16-B chunks around it, whose
 * bytes are the stream's own).  Errors: as recoil_device_decoder_create, E_ARG for an
 * empty or out-of-range task range. */
int recoil_device_decoder_create_range(const uint8_t *head, uint64_t head_len, uint64_t container_len,
                                       uint64_t task_begin, uint64_t task_end, recoil_device_decoder **out);
/* After recoil_device_decode (synchronises the stream: two 8-byte read-backs of the
 * device task records): the committed symbol span [*out_lo, *out_hi) of the
 * decoder's task range (sync start of the point before the range .. sync start of
 * its last point, Z13; the whole [0, N) for the full range).  Errors: E_ARG, E_CUDA. */
int recoil_device_decoder_span(const recoil_device_decoder *dec, const void *d_workspace, void *cuda_stream,
                               uint64_t *out_lo, uint64_t *out_hi);
int recoil_device_decoder_plan(const recoil_device_decoder *dec, recoil_device_plan *plan);
/* Convenience H2D (stream-ordered): container -> d_buffer + container_offset, and the
 * zero padding after it.  A caller that copies the container itself must zero
 * buffer_bytes - container_offset - container_len bytes after it. */
int recoil_device_upload(const recoil_device_decoder *dec, const uint8_t *container, void *d_buffer, void *cuda_stream);
/* Stream-ordered: the metadata kernels, then the decode kernel, writing the N
 * symbols to d_out[0, N) (it may write d_out up to out_count).  Metadata that
 * fails its checks (offsets out of range or not increasing, record list not
 * ending at the words, widths out of range, a group difference above its anchor
 * group, a boundary past N, sync starts not increasing) sets E_INCONSISTENT in
 * the status word and the affected tasks do not decode.  Errors: E_ARG, E_CUDA. */
int recoil_device_decode(recoil_device_decoder *dec, void *d_buffer, void *d_workspace, uint8_t *d_out,
                         void *cuda_stream);
/* As recoil_decoder_status for the last recoil_device_decode. */
int recoil_device_decoder_status(recoil_device_decoder *dec, const void *d_workspace, void *cuda_stream,
                                 uint64_t *bad_task);
/* Kernel launches one recoil_device_decode issues. */
int recoil_device_decoder_launches(const recoil_device_decoder *dec);
void recoil_device_decoder_destroy(recoil_device_decoder *dec);

/* Combine on the GPU (the server shrinks parallelism per
 * client): the result of recoil_combine_splits(container, target_splits),
 * written from the device copy d_in (in_len bytes, any alignment) to d_out.
 * recoil_device_combine_plan: the d_out capacity and d_workspace size to
 * provide.  recoil_device_combine writes the output length to the device word
 * *d_out_len (stream-ordered); it synchronises the stream twice (8-byte
 * read-backs: the new series widths, then the kept records' total size,
 * place the series and the word stream).  target_splits >= M: a copy.  Errors: as
 * recoil_device_decoder_create, E_BUFFER (capacity), E_INCONSISTENT
 * (metadata checks), E_OVERFLOW, E_CUDA. */
int recoil_device_combine_plan(const uint8_t *head, uint64_t head_len, uint64_t container_len, uint32_t target_splits,
                               uint64_t *out_capacity, uint64_t *workspace_bytes);
int recoil_device_combine(const uint8_t *head, uint64_t head_len, const uint8_t *d_in, uint64_t in_len,
                          uint32_t target_splits, uint8_t *d_out, uint64_t out_capacity, void *d_workspace,
                          uint64_t *d_out_len, void *cuda_stream);

/* ---------------------------------------------------------------------- */
/* Multi-GPU sharding (host planning; each GPU decodes its own task range) */
/* ---------------------------------------------------------------------- */

/* Split the container's tasks into n_shards contiguous ranges whose
 * committed symbol counts are as equal as task granularity allows.
 * task_bounds: n_shards + 1 entries, task_bounds[0] = 0,
 * task_bounds[n_shards] = M.  Errors: E_ARG, container errors. */
int recoil_shard_plan(const uint8_t *container, uint64_t len, uint32_t n_shards, uint64_t *task_bounds);

/* Single-process multi-GPU decode (the split tasks
 * are "completely independent" and "can be scaled over multiple cores").
 * recoil_multi_plan: the decode plan of each of n_dev shards (recoil_shard_plan
 * ranges); plans[d].out_count symbols is the size of d_outs[d], laid out as for
 * recoil_decode (d_outs[d][i - plans[d].out_base]).  plans: n_dev entries.
 * Errors: container errors, E_ARG, E_NOMEM, E_UNSUPPORTED (adaptive container:
 * it needs per-symbol model ids, use recoil_decode_adaptive per device). */
int recoil_multi_plan(const uint8_t *container, uint64_t len, uint32_t n_dev, recoil_plan *plans);

/* Decode shard d on CUDA device devices[d] into the caller's device buffer
 * d_outs[d] (on that device, plans[d].out_count bytes).  Each device gets its
 * own stream, workspace and word slice (allocated stream-ordered from that
 * device's pool, freed before return); all devices are enqueued before any is
 * waited on, so distinct GPUs decode concurrently.  Synchronous: returns after
 * every device finished.  gather_root >= 0: afterwards every shard's committed
 * span [out_lo, out_hi) is copied into d_gather[out_lo, out_hi) on
 * devices[gather_root] (d_gather: N bytes on that device) -- one NCCL group of
 * ncclSend/ncclRecv (libnccl.so.2, loaded at run time) when the devices are
 * distinct, else (shards sharing a GPU, or no NCCL) cudaMemcpyPeerAsync; the
 * gather is skipped when a decode failed.  gather_root = -1: no gather.
 * kernel_ms (may be NULL): n_dev decode-kernel times (CUDA events per device).
 * Returns the most severe device status (E_INCONSISTENT, E_UNSUPPORTED,
 * E_UNDERFLOW, E_SYNC) or RECOIL_OK.  The current device is restored.
 * Errors: as recoil_multi_plan, E_ARG (NULL d_outs[d] of a shard with tasks,
 * gather_root >= n_dev, gather without d_gather), E_CUDA. */
int recoil_multi_decode(const uint8_t *container, uint64_t len, uint32_t n_dev, const int *devices,
                        uint8_t *const *d_outs, int gather_root, uint8_t *d_gather, float *kernel_ms);

/* 1 if recoil_multi_decode can gather over NCCL (libnccl.so.2 loadable), else 0. */
int recoil_multi_nccl_available(void);

/* ---------------------------------------------------------------------- */
/* Host baselines (NOT a fallback of the GPU path: separate entry points)  */
/* ---------------------------------------------------------------------- */

/* Multithreaded CPU Recoil / partitioned decoder: one task per split, up to
 * `threads` threads (0 = hardware concurrency; P:429 recommends one per
 * physical core, no SMT).  Task decoder (P:429's CPU decoders): AVX-512 (16
 * lanes per instruction, two vectors per 32-lane group) when the CPU has
 * AVX-512 F/BW/VL/VBMI2, else AVX2 (8 lanes per instruction, four vectors per
 * group), else scalar.  out: N bytes.
 * Errors: container errors, E_UNDERFLOW, E_SYNC. */
int recoil_decode_cpu(const uint8_t *container, uint64_t len, uint8_t *out, uint32_t threads);

#define RECOIL_CPU_SCALAR 1u /* recoil_decode_cpu_ex flag: force the scalar task decoder */
#define RECOIL_CPU_AVX2 2u   /* recoil_decode_cpu_ex flag: force the AVX2 task decoder (E_UNSUPPORTED without AVX2) */
int recoil_decode_cpu_ex(const uint8_t *container, uint64_t len, uint8_t *out, uint32_t threads, uint32_t flags);

/* The SIMD task decoder recoil_decode_cpu uses on this CPU: 2 = AVX-512,
 * 1 = AVX2, 0 = none (scalar). */
int recoil_cpu_simd(void);

#ifdef __cplusplus
}
#endif
#endif
