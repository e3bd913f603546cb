// pipeline.cpp -- end-to-end host -> host decode on one GPU, pipelined.
//
// The task list is cut into contiguous chunks of ~equal committed symbols
// (the multi-GPU shard plan, §8(e), used here on one device).  For chunk k the
// host expands its tasks (row a1), stages LUT + task table in pinned memory,
// and enqueues, into buffer set k % S: the H2D of tables and the chunk's word
// slice on the copy-in stream, the decode kernel on the compute stream, the
// D2H of the chunk's symbols and status word on the copy-out stream, chained
// by events.  The H2D of later chunks overlaps the D2H of earlier ones (PCIe
// is full duplex), and the host's a1 work for chunk k+1 overlaps the device
// work of chunk k.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>

#include "../recoil_internal.h"

namespace recoil {
namespace {

constexpr uint32_t kMaxStreams = 8;

uint64_t align256(uint64_t v) { return (v + 255) & ~255ull; }

struct Pipeline {
  const uint8_t *bytes = nullptr;
  uint64_t len = 0;
  uint32_t chunks = 0;
  uint64_t task_begin = 0, task_end = 0;
  uint64_t N = 0;
  uint64_t ws_bytes = 0, word_bytes = 0, out_bytes = 0, set_bytes = 0;
  // pinned host staging per buffer set (LUT + finals + task table) and status words
  uint8_t *staging[kMaxStreams] = {nullptr};
  uint64_t staging_bytes = 0;
  cudaEvent_t staged[kMaxStreams] = {nullptr};
  // per buffer set: its H2D done, its kernel done, its D2H done (role streams below)
  cudaEvent_t ev_in[kMaxStreams] = {nullptr}, ev_k[kMaxStreams] = {nullptr}, ev_out[kMaxStreams] = {nullptr};
  DeviceStatus *status = nullptr;  // pinned, one per chunk
  std::vector<uint64_t> bounds;
  std::vector<Decoder> dec;        // the last run's chunk plans (alive until status)
  int single_symbol = -1;
  uint32_t prev_streams = 0;       // buffer sets the previous run used (its work may still be queued)
  uint64_t out_lo = 0, out_hi = 0; // committed symbols of the task range

  ~Pipeline() {
    for (auto &p : staging)
      if (p) cudaFreeHost(p);
    for (auto *arr : {staged, ev_in, ev_k, ev_out})
      for (uint32_t i = 0; i < kMaxStreams; ++i)
        if (arr[i]) cudaEventDestroy(arr[i]);
    if (status) cudaFreeHost(status);
  }
};

int plan_chunks(Pipeline *pl, std::shared_ptr<const Container> c) {
  pl->bounds.assign(pl->chunks + 1, 0);
  shard_bounds_range(*c, pl->task_begin, pl->task_end, pl->chunks, pl->bounds.data());
  pl->dec.clear();
  pl->dec.resize(pl->chunks);
  for (uint32_t k = 0; k < pl->chunks; ++k) {
    int rc = build_decoder_from(c, pl->bounds[k], pl->bounds[k + 1], &pl->dec[k], true);
    if (rc) return rc;
  }
  return RECOIL_OK;
}

}  // namespace
}  // namespace recoil

using namespace recoil;

extern "C" int recoil_pipeline_create(const uint8_t *container, uint64_t len, uint64_t task_begin,
                                      uint64_t task_end, uint32_t n_chunks, recoil_pipeline **out) {
  if (!container || !out || n_chunks < 1) return RECOIL_E_ARG;
  *out = nullptr;
  try {
    auto c = std::make_shared<Container>();
    int rc = parse_container(container, len, c.get(), /*light=*/true);
    if (rc) return rc;
    if (c->adaptive) return RECOIL_E_UNSUPPORTED;  // needs the model ids (recoil_decode_adaptive)
    Pipeline *pl = new Pipeline();
    pl->bytes = container;
    pl->len = len;
    pl->task_end = std::min<uint64_t>(task_end, c->M);
    pl->task_begin = std::min(task_begin, pl->task_end);
    pl->chunks = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(n_chunks, pl->task_end - pl->task_begin));
    pl->N = c->N;
    rc = plan_chunks(pl, c);
    if (rc) {
      delete pl;
      return rc;
    }
    pl->out_lo = pl->dec.front().plan.out_lo;
    pl->out_hi = pl->dec.back().plan.out_hi;
    for (const Decoder &d : pl->dec) {
      pl->out_lo = std::min(pl->out_lo, d.plan.out_lo);
      pl->out_hi = std::max(pl->out_hi, d.plan.out_hi);
      pl->ws_bytes = std::max(pl->ws_bytes, align256(d.plan.workspace_bytes));
      pl->word_bytes = std::max(pl->word_bytes, align256(2 * d.plan.word_count));
      pl->out_bytes = std::max(pl->out_bytes, align256(d.plan.out_count));
      pl->staging_bytes = std::max(pl->staging_bytes, d.plan.workspace_bytes);
      pl->single_symbol = d.single_symbol;
    }
    pl->set_bytes = pl->ws_bytes + pl->word_bytes + pl->out_bytes;
    if (cudaHostAlloc(reinterpret_cast<void **>(&pl->status), sizeof(DeviceStatus) * pl->chunks,
                      cudaHostAllocDefault) != cudaSuccess) {
      delete pl;
      return RECOIL_E_CUDA;
    }
    *out = reinterpret_cast<recoil_pipeline *>(pl);
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_pipeline_device_bytes(const recoil_pipeline *p, uint32_t n_streams, uint64_t *bytes) {
  if (!p || !bytes || n_streams < 1 || n_streams > kMaxStreams) return RECOIL_E_ARG;
  *bytes = (uint64_t)n_streams * reinterpret_cast<const Pipeline *>(p)->set_bytes;
  return RECOIL_OK;
}

extern "C" int recoil_pipeline_span(const recoil_pipeline *p, uint64_t *out_lo, uint64_t *out_hi) {
  if (!p || !out_lo || !out_hi) return RECOIL_E_ARG;
  const Pipeline *pl = reinterpret_cast<const Pipeline *>(p);
  *out_lo = pl->out_lo;
  *out_hi = pl->out_hi;
  return RECOIL_OK;
}

extern "C" int recoil_pipeline_run(recoil_pipeline *p, void *d_scratch, uint8_t *host_out, void *const *streams,
                                   uint32_t n_streams) {
  return recoil_pipeline_run_at(p, d_scratch, host_out, 0, streams, n_streams);
}

extern "C" int recoil_pipeline_run_at(recoil_pipeline *p, void *d_scratch, uint8_t *host_out, uint64_t host_first,
                                      void *const *streams, uint32_t n_streams) {
  if (!p || !d_scratch || !streams || n_streams < 1 || n_streams > kMaxStreams) return RECOIL_E_ARG;
  Pipeline *pl = reinterpret_cast<Pipeline *>(p);
  if (pl->N && !host_out) return RECOIL_E_ARG;
  if (pl->out_hi > pl->out_lo && host_first > pl->out_lo) return RECOIL_E_ARG;
  try {
    // a previous run enqueued without an intervening status call may still be
    // reading its buffer sets, staging and status words: wait for its last D2H per
    // set (each set's work is chained, so that event follows all of it)
    for (uint32_t s = 0; s < pl->prev_streams; ++s)
      if (pl->ev_out[s] && cudaEventSynchronize(pl->ev_out[s]) != cudaSuccess) return RECOIL_E_CUDA;
    pl->prev_streams = 0;
    // per run: parse and plan again (this is the host half of the path)
    auto c = std::make_shared<Container>();
    int rc = parse_container(pl->bytes, pl->len, c.get(), /*light=*/true);
    if (rc) return rc;
    pl->bounds.assign(pl->chunks + 1, 0);
    shard_bounds_range(*c, pl->task_begin, pl->task_end, pl->chunks, pl->bounds.data());
    pl->dec.clear();
    pl->dec.resize(pl->chunks);
    for (uint32_t s = 0; s < n_streams; ++s) {
      if (!pl->staging[s] && cudaHostAlloc(reinterpret_cast<void **>(&pl->staging[s]), pl->staging_bytes,
                                           cudaHostAllocDefault) != cudaSuccess)
        return RECOIL_E_CUDA;
      for (cudaEvent_t *e : {&pl->staged[s], &pl->ev_in[s], &pl->ev_k[s], &pl->ev_out[s]})
        if (!*e && cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return RECOIL_E_CUDA;
    }
    // stream roles: copies in on streams[0], kernels on streams[1], copies out on
    // streams[2] (fewer streams: shared roles).  Chunk k uses buffer set k % n_streams;
    // the H2D of chunk k waits for the D2H of chunk k - n_streams (same set).  So the
    // H2D of later chunks overlaps the D2H of earlier ones (PCIe is full duplex).
    cudaStream_t sh = reinterpret_cast<cudaStream_t>(streams[0]);
    cudaStream_t sc = reinterpret_cast<cudaStream_t>(streams[std::min<uint32_t>(1, n_streams - 1)]);
    cudaStream_t so = reinterpret_cast<cudaStream_t>(streams[std::min<uint32_t>(2, n_streams - 1)]);
    std::memset(pl->status, 0, sizeof(DeviceStatus) * pl->chunks);
    pl->prev_streams = std::min<uint32_t>(n_streams, pl->chunks);
    for (uint32_t k = 0; k < pl->chunks; ++k) {
      const uint32_t s = k % n_streams;
      cudaStream_t st = sh;
      Decoder &d = pl->dec[k];
      rc = build_decoder_from(c, pl->bounds[k], pl->bounds[k + 1], &d, true);  // a1 for this chunk
      if (rc) return rc;
      const recoil_plan &pn = d.plan;
      if (pn.workspace_bytes > pl->staging_bytes || 2 * pn.word_count > pl->word_bytes ||
          pn.out_count > pl->out_bytes)
        return RECOIL_E_INCONSISTENT;  // the container changed since create
      char *set = static_cast<char *>(d_scratch) + (uint64_t)s * pl->set_bytes;
      char *ws = set;
      uint16_t *words = reinterpret_cast<uint16_t *>(set + pl->ws_bytes);
      uint8_t *dout = reinterpret_cast<uint8_t *>(set + pl->ws_bytes + pl->word_bytes);
      // stage LUT + finals + tasks (+ records) in pinned memory once the set's previous H2D has consumed it
      if (k >= n_streams && cudaEventSynchronize(pl->staged[s]) != cudaSuccess) return RECOIL_E_CUDA;
      uint8_t *stg = pl->staging[s];
      std::memset(stg, 0, 16);
      if (!d.lut.empty()) std::memcpy(stg + d.lut_off, d.lut.data(), d.lut.size());
      if (!d.finals.empty()) std::memcpy(stg + d.finals_off, d.finals.data(), 4 * d.finals.size());
      if (!d.tasks.empty()) std::memcpy(stg + d.tasks_off, d.tasks.data(), sizeof(TaskRec) * d.tasks.size());
      if (!d.heads.empty()) std::memcpy(stg + d.tasks_off, d.heads.data(), sizeof(TaskHead) * d.heads.size());
      if (d.fused) {  // the raw split records and the zero pad under their windows: one H2D with the tables
        if (d.rec_len) std::memcpy(stg + d.rec_off, c->bytes + d.rec_src, d.rec_len);
        std::memset(stg + d.rec_off + d.rec_len, 0, pn.workspace_bytes - d.rec_off - d.rec_len);
      }
      if (k >= n_streams && cudaStreamWaitEvent(sh, pl->ev_out[s], 0) != cudaSuccess) return RECOIL_E_CUDA;
      if (cudaMemcpyAsync(ws, stg, pn.workspace_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaEventRecord(pl->staged[s], st) != cudaSuccess)
        return RECOIL_E_CUDA;
      const uint64_t have = c->B > pn.word_lo ? std::min<uint64_t>(pn.word_count, c->B - pn.word_lo) : 0;
      if (have && cudaMemcpyAsync(words, c->words + 2 * pn.word_lo, 2 * have, cudaMemcpyHostToDevice, st) !=
                      cudaSuccess)
        return RECOIL_E_CUDA;
      if (pn.word_count > have &&
          cudaMemsetAsync(words + have, 0, 2 * (pn.word_count - have), st) != cudaSuccess)
        return RECOIL_E_CUDA;
      if (cudaEventRecord(pl->ev_in[s], sh) != cudaSuccess || cudaStreamWaitEvent(sc, pl->ev_in[s], 0) != cudaSuccess)
        return RECOIL_E_CUDA;
      rc = decode_staged(&d, ws, words, dout, sc);  // the status block came zeroed with the tables
      if (rc) return rc;
      if (cudaEventRecord(pl->ev_k[s], sc) != cudaSuccess || cudaStreamWaitEvent(so, pl->ev_k[s], 0) != cudaSuccess)
        return RECOIL_E_CUDA;
      if (pn.out_hi > pn.out_lo &&
          cudaMemcpyAsync(host_out + (pn.out_lo - host_first), dout + (pn.out_lo - pn.out_base), pn.out_hi - pn.out_lo,
                          cudaMemcpyDeviceToHost, so) != cudaSuccess)
        return RECOIL_E_CUDA;
      if (cudaMemcpyAsync(&pl->status[k], ws, sizeof(DeviceStatus), cudaMemcpyDeviceToHost, so) != cudaSuccess ||
          cudaEventRecord(pl->ev_out[s], so) != cudaSuccess)
        return RECOIL_E_CUDA;
    }
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_pipeline_status(recoil_pipeline *p, void *const *streams, uint32_t n_streams,
                                      uint64_t *bad_task) {
  if (!p || !streams || n_streams < 1) return RECOIL_E_ARG;
  Pipeline *pl = reinterpret_cast<Pipeline *>(p);
  for (uint32_t s = 0; s < n_streams; ++s)
    if (cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(streams[s])) != cudaSuccess) return RECOIL_E_CUDA;
  int rc = RECOIL_OK;
  uint64_t bad = UINT64_MAX;
  for (uint32_t k = 0; k < pl->chunks && k < pl->dec.size(); ++k) {
    const DeviceStatus &st = pl->status[k];
    if (st.bad_task) bad = std::min<uint64_t>(bad, 0xFFFFFFFFu - st.bad_task);
    if (st.flags & 4u) rc = RECOIL_E_INCONSISTENT;
    else if ((st.flags & 8u) && rc != RECOIL_E_INCONSISTENT) rc = RECOIL_E_UNSUPPORTED;
    else if ((st.flags & 1u) && rc != RECOIL_E_INCONSISTENT && rc != RECOIL_E_UNSUPPORTED) rc = RECOIL_E_UNDERFLOW;
    else if ((st.flags & 2u) && rc == RECOIL_OK) rc = RECOIL_E_SYNC;
  }
  if (bad_task) *bad_task = bad;
  return rc;
}

extern "C" int recoil_pipeline_launches(const recoil_pipeline *p) {
  if (!p) return RECOIL_E_ARG;
  const Pipeline *pl = reinterpret_cast<const Pipeline *>(p);
  int n = 0;
  for (const Decoder &d : pl->dec) n += recoil_decoder_launches(reinterpret_cast<const recoil_decoder *>(&d));
  return n;
}

extern "C" void recoil_pipeline_destroy(recoil_pipeline *p) { delete reinterpret_cast<Pipeline *>(p); }
