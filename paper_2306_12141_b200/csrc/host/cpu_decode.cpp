// cpu_decode.cpp -- multithreaded host decoder (baseline, NOT a fallback of the
// GPU path): the same task table as the GPU kernel, one task per split, one
// thread per core (P:429 recommends no SMT), scalar code.  Decodes Recoil and
// partitioned containers for any 1 <= n <= 16.
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

}  // namespace
}  // namespace recoil

using namespace recoil;

extern "C" int recoil_decode_cpu(const uint8_t *container, uint64_t len, uint8_t *out, uint32_t threads) {
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
    tb.sym.resize(1u << n);
    tb.f.resize(1u << n);
    tb.bias.resize(1u << n);
    uint32_t F = 0;
    for (uint32_t s = 0; s < 256; ++s) {
      for (uint32_t k = 0; k < d.c->f[s]; ++k) {
        tb.sym[F + k] = (uint8_t)s;
        tb.f[F + k] = d.c->f[s];
        tb.bias[F + k] = k;
      }
      F += d.c->f[s];
    }
    // the container's words as a host u16 array (little-endian host)
    std::vector<uint16_t> w(d.c->B + 1);
    if (d.c->B) std::memcpy(w.data(), d.c->words, 2 * d.c->B);
    const uint16_t *slice = w.data() + d.plan.word_lo;
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    threads = std::min<uint32_t>(threads, (uint32_t)std::max<size_t>(1, d.tasks.size()));
    std::atomic<size_t> next{0};
    std::atomic<int> err{RECOIL_OK};
    auto worker = [&]() {
      for (size_t k; (k = next.fetch_add(1)) < d.tasks.size() && err.load() == RECOIL_OK;) {
        int r = decode_task(d, tb, d.tasks[k], slice, out);
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
