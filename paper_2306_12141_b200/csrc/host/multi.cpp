// multi.cpp -- single-process multi-GPU decode (P:223:
// the split tasks are "completely independent" and "can be scaled over multiple
// cores").  The container's tasks are cut into contiguous ranges of ~equal
// committed symbols (recoil_shard_plan); device d uploads only the word slice
// and records its range needs and decodes its own span, with no exchange.  The
// optional final gather of the spans into one buffer on a root device is one
// NCCL group of point-to-point sends/receives when the devices are distinct
// (NCCL is dlopen'ed, so the library loads without it), and a device-to-device
// copy for a span that already lives on the root's GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: the entry points are resolved with dlsym

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <vector>

#include "../recoil_internal.h"

namespace recoil {
namespace {

struct NcclApi {
  decltype(&ncclCommInitAll) comm_init_all = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  bool ok = false;
};

// libnccl.so.2 of the process if one is already loaded (PyTorch's), else the system's
const NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.comm_init_all = reinterpret_cast<decltype(&ncclCommInitAll)>(dlsym(h, "ncclCommInitAll"));
    api.comm_destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.group_start = reinterpret_cast<decltype(&ncclGroupStart)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.send = reinterpret_cast<decltype(&ncclSend)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(&ncclRecv)>(dlsym(h, "ncclRecv"));
    api.ok = api.comm_init_all && api.comm_destroy && api.group_start && api.group_end && api.send && api.recv;
  });
  return api;
}

int plan_shards(const uint8_t *container, uint64_t len, uint32_t n_dev, std::vector<Decoder> *dec) {
  auto c = std::make_shared<Container>();
  // full parse: the shards use the host-expanded task records, as recoil_decoder_create
  if (container && len >= 4 && std::memcmp(container, "RCA1", 4) == 0)
    return RECOIL_E_UNSUPPORTED;  // needs per-device model ids (recoil_decode_adaptive)
  int rc = parse_container(container, len, c.get(), /*light=*/false);
  if (rc) return rc;
  std::vector<uint64_t> bounds(n_dev + 1, 0);
  shard_bounds_range(*c, 0, c->M, n_dev, bounds.data());
  dec->clear();
  dec->resize(n_dev);
  for (uint32_t d = 0; d < n_dev; ++d) {
    rc = build_decoder_from(c, bounds[d], bounds[d + 1], &(*dec)[d], true);
    if (rc) return rc;
  }
  return RECOIL_OK;
}

// Per-device resources of one call; released (stream-ordered frees, then the
// stream) on every exit path.
struct DevRun {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  char *ws = nullptr;
  uint16_t *words = nullptr;
  ~DevRun() {
    if (!stream) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (ws) cudaFreeAsync(ws, stream);
    if (words) cudaFreeAsync(words, stream);
    cudaStreamSynchronize(stream);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    cudaStreamDestroy(stream);
    cudaSetDevice(prev);
  }
};

int worst(int a, int b) {  // the more severe of two status codes (metadata > unsupported > underflow > sync)
  auto rank = [](int r) {
    return r == RECOIL_OK ? 0 : r == RECOIL_E_SYNC ? 1 : r == RECOIL_E_UNDERFLOW ? 2 : r == RECOIL_E_UNSUPPORTED ? 3
                                                                                                                : 4;
  };
  return rank(b) > rank(a) ? b : a;
}

}  // namespace
}  // namespace recoil

using namespace recoil;

extern "C" int recoil_multi_plan(const uint8_t *container, uint64_t len, uint32_t n_dev, recoil_plan *plans) {
  if (!container || !plans || n_dev < 1 || n_dev > 1024) return RECOIL_E_ARG;
  try {
    std::vector<Decoder> dec;
    int rc = plan_shards(container, len, n_dev, &dec);
    if (rc) return rc;
    for (uint32_t d = 0; d < n_dev; ++d) plans[d] = dec[d].plan;
    return RECOIL_OK;
  } catch (const std::bad_alloc &) {
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_multi_decode(const uint8_t *container, uint64_t len, uint32_t n_dev, const int *devices,
                                   uint8_t *const *d_outs, int gather_root, uint8_t *d_gather, float *kernel_ms) {
  if (!container || !devices || !d_outs || n_dev < 1 || n_dev > 1024) return RECOIL_E_ARG;
  if (gather_root >= (int)n_dev || (gather_root >= 0 && !d_gather)) return RECOIL_E_ARG;
  int prev_dev = 0;
  if (cudaGetDevice(&prev_dev) != cudaSuccess) return RECOIL_E_CUDA;
  try {
    std::vector<Decoder> dec;
    int rc = plan_shards(container, len, n_dev, &dec);
    if (rc) return rc;
    std::vector<std::unique_ptr<DevRun>> run(n_dev);
    auto fail = [&](int code) {
      run.clear();
      cudaSetDevice(prev_dev);
      return code;
    };
    // enqueue every device's upload + decode before waiting on any (the GPUs run concurrently)
    for (uint32_t d = 0; d < n_dev; ++d) {
      run[d].reset(new DevRun());
      DevRun &r = *run[d];
      const recoil_plan &p = dec[d].plan;
      r.device = devices[d];
      if (cudaSetDevice(r.device) != cudaSuccess) return fail(RECOIL_E_CUDA);
      if (cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking) != cudaSuccess) return fail(RECOIL_E_CUDA);
      if (cudaEventCreate(&r.t0) != cudaSuccess || cudaEventCreate(&r.t1) != cudaSuccess)
        return fail(RECOIL_E_CUDA);
      if (p.n_tasks == 0) continue;
      if (!d_outs[d]) return fail(RECOIL_E_ARG);
      if (cudaMallocAsync(reinterpret_cast<void **>(&r.ws), std::max<uint64_t>(p.workspace_bytes, 16), r.stream) !=
              cudaSuccess ||
          cudaMallocAsync(reinterpret_cast<void **>(&r.words), std::max<uint64_t>(2 * p.word_count, 2), r.stream) !=
              cudaSuccess)
        return fail(RECOIL_E_CUDA);
      recoil_decoder *h = reinterpret_cast<recoil_decoder *>(&dec[d]);
      if ((rc = recoil_decoder_upload(h, r.ws, r.words, r.stream)) != RECOIL_OK) return fail(rc);
      if (cudaEventRecord(r.t0, r.stream) != cudaSuccess) return fail(RECOIL_E_CUDA);
      if ((rc = recoil_decode(h, r.ws, r.words, d_outs[d], r.stream)) != RECOIL_OK) return fail(rc);
      if (cudaEventRecord(r.t1, r.stream) != cudaSuccess) return fail(RECOIL_E_CUDA);
    }
    int status = RECOIL_OK;
    for (uint32_t d = 0; d < n_dev; ++d) {
      DevRun &r = *run[d];
      if (cudaSetDevice(r.device) != cudaSuccess) return fail(RECOIL_E_CUDA);
      if (kernel_ms) kernel_ms[d] = 0.f;
      if (dec[d].plan.n_tasks == 0) continue;
      uint64_t bad = 0;
      const int st = recoil_decoder_status(reinterpret_cast<recoil_decoder *>(&dec[d]), r.ws, r.stream, &bad);
      if (st == RECOIL_E_CUDA) return fail(st);
      status = worst(status, st);
      if (kernel_ms && cudaEventElapsedTime(&kernel_ms[d], r.t0, r.t1) != cudaSuccess) return fail(RECOIL_E_CUDA);
    }
    if (gather_root >= 0 && status == RECOIL_OK) {
      // optional final gather: span of device d -> d_gather[out_lo_d, out_hi_d) on the root
      const int root_dev = devices[gather_root];
      bool distinct = n_dev > 1;
      for (uint32_t a = 0; a < n_dev && distinct; ++a)
        for (uint32_t b = a + 1; b < n_dev; ++b)
          if (devices[a] == devices[b]) distinct = false;
      auto span_src = [&](uint32_t d) { return d_outs[d] + (dec[d].plan.out_lo - dec[d].plan.out_base); };
      auto span_len = [&](uint32_t d) { return dec[d].plan.out_hi - dec[d].plan.out_lo; };
      const NcclApi &api = nccl();
      if (distinct && api.ok) {
        std::vector<ncclComm_t> comms(n_dev, nullptr);
        std::vector<int> devs(devices, devices + n_dev);
        if (api.comm_init_all(comms.data(), (int)n_dev, devs.data()) != ncclSuccess) return fail(RECOIL_E_CUDA);
        bool ok = api.group_start() == ncclSuccess;
        for (uint32_t d = 0; d < n_dev && ok; ++d) {
          if ((int)d == gather_root || span_len(d) == 0) continue;
          ok = api.send(span_src(d), span_len(d), ncclUint8, gather_root, comms[d], run[d]->stream) == ncclSuccess &&
               api.recv(d_gather + dec[d].plan.out_lo, span_len(d), ncclUint8, (int)d, comms[gather_root],
                        run[gather_root]->stream) == ncclSuccess;
        }
        ok = (api.group_end() == ncclSuccess) && ok;
        cudaSetDevice(root_dev);
        if (ok && span_len(gather_root))
          ok = cudaMemcpyAsync(d_gather + dec[gather_root].plan.out_lo, span_src(gather_root), span_len(gather_root),
                               cudaMemcpyDeviceToDevice, run[gather_root]->stream) == cudaSuccess;
        for (uint32_t d = 0; d < n_dev; ++d) {
          cudaSetDevice(devices[d]);
          ok = cudaStreamSynchronize(run[d]->stream) == cudaSuccess && ok;
        }
        for (ncclComm_t cm : comms)
          if (cm) api.comm_destroy(cm);
        if (!ok) return fail(RECOIL_E_CUDA);
      } else {
        // one GPU (or NCCL absent): peer / device copies on the root's stream
        if (cudaSetDevice(root_dev) != cudaSuccess) return fail(RECOIL_E_CUDA);
        for (uint32_t d = 0; d < n_dev; ++d)
          if (span_len(d) && cudaMemcpyPeerAsync(d_gather + dec[d].plan.out_lo, root_dev, span_src(d), devices[d],
                                                 span_len(d), run[gather_root]->stream) != cudaSuccess)
            return fail(RECOIL_E_CUDA);
        if (cudaStreamSynchronize(run[gather_root]->stream) != cudaSuccess) return fail(RECOIL_E_CUDA);
      }
    }
    run.clear();
    cudaSetDevice(prev_dev);
    return status;
  } catch (const std::bad_alloc &) {
    cudaSetDevice(prev_dev);
    return RECOIL_E_NOMEM;
  }
}

extern "C" int recoil_multi_nccl_available(void) { return nccl().ok ? 1 : 0; }
