/*
 * c_client.c -- the C ABI (include/recoil.h) used from plain C, no Python and no torch:
 * encode a synthetic byte stream with split points, shrink the metadata for a smaller
 * client (recoil_combine_splits), decode on the GPU through
 * recoil_decoder_create / upload / decode / status with cudaMalloc'd buffers, then
 * decode again as shards on several "devices" with recoil_multi_decode and gather the
 * spans; every byte is compared with the input.
 *
 *   usage: c_client [n_symbols] [splits] [devices...]     (default 4000000 1000 0 0)
 *   exit 0 = bit-exact everywhere
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "recoil.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    int rc_ = (call);                                                            \
    if (rc_ != RECOIL_OK) {                                                      \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, recoil_strerror(rc_)); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)
#define CUDA(call)                                                               \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

static uint64_t splitmix(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int main(int argc, char **argv) {
  const uint64_t N = argc > 1 ? strtoull(argv[1], NULL, 10) : 4000000;
  const uint32_t M = argc > 2 ? (uint32_t)strtoul(argv[2], NULL, 10) : 1000;
  int n_dev = argc > 3 ? argc - 3 : 2;
  int devices[16] = {0, 0};
  for (int d = 0; d < n_dev && d < 16; ++d) devices[d] = argc > 3 ? atoi(argv[3 + d]) : 0;

  /* skewed bytes: geometric-like distribution over 0..63 */
  uint8_t *sym = (uint8_t *)malloc(N);
  uint64_t seed = 12345, hist[256] = {0};
  for (uint64_t i = 0; i < N; ++i) {
    uint64_t u = splitmix(&seed);
    uint32_t s = 0;
    while (s < 63 && (u & 3) == 0) {
      u >>= 2;
      ++s;
    }
    sym[i] = (uint8_t)s;
    ++hist[sym[i]];
  }
  uint32_t freqs[256];
  CHECK(recoil_build_model(hist, 11, freqs));

  uint64_t cap = 0;
  CHECK(recoil_encode(sym, N, freqs, 11, M, NULL, &cap));
  uint8_t *c = (uint8_t *)malloc(cap);
  uint64_t clen = cap;
  CHECK(recoil_encode(sym, N, freqs, 11, M, c, &clen));
  recoil_info info;
  CHECK(recoil_inspect(c, clen, &info));
  printf("encoded %llu symbols into %llu bytes, %u splits\n", (unsigned long long)N, (unsigned long long)clen,
         info.n_splits);

  /* the server shrinks the metadata for a smaller client */
  uint64_t slen = 0;
  CHECK(recoil_combine_splits(c, clen, info.n_splits / 4 + 1, NULL, &slen));
  uint8_t *small = (uint8_t *)malloc(slen);
  CHECK(recoil_combine_splits(c, clen, info.n_splits / 4 + 1, small, &slen));

  /* one-GPU decode of the shrunk container */
  recoil_decoder *dec = NULL;
  CHECK(recoil_decoder_create(small, slen, 0, UINT64_MAX, &dec));
  recoil_plan plan;
  CHECK(recoil_decoder_plan(dec, &plan));
  void *ws = NULL, *words = NULL, *out = NULL;
  cudaStream_t st;
  CUDA(cudaSetDevice(devices[0]));
  CUDA(cudaStreamCreate(&st));
  CUDA(cudaMalloc(&ws, plan.workspace_bytes));
  CUDA(cudaMalloc(&words, 2 * plan.word_count));
  CUDA(cudaMalloc(&out, plan.out_count));
  CHECK(recoil_decoder_upload(dec, ws, (uint16_t *)words, st));
  CHECK(recoil_decode(dec, ws, (const uint16_t *)words, (uint8_t *)out, st));
  uint64_t bad = 0;
  CHECK(recoil_decoder_status(dec, ws, st, &bad));
  uint8_t *host = (uint8_t *)malloc(N + 16);
  CUDA(cudaMemcpy(host, (uint8_t *)out + (plan.out_lo - plan.out_base), plan.out_hi - plan.out_lo,
                  cudaMemcpyDeviceToHost));
  if (plan.out_lo != 0 || plan.out_hi != N || memcmp(host, sym, N) != 0) {
    fprintf(stderr, "single-GPU decode mismatch\n");
    return 1;
  }
  printf("single GPU: %u tasks, bit-exact\n", plan.n_tasks);
  recoil_decoder_destroy(dec);
  cudaFree(ws);
  cudaFree(words);
  cudaFree(out);

  /* shards on n_dev devices of the full container, gathered on device 0 */
  recoil_plan plans[16];
  CHECK(recoil_multi_plan(c, clen, (uint32_t)n_dev, plans));
  uint8_t *outs[16];
  for (int d = 0; d < n_dev; ++d) {
    CUDA(cudaSetDevice(devices[d]));
    CUDA(cudaMalloc((void **)&outs[d], plans[d].out_count ? plans[d].out_count : 16));
  }
  uint8_t *gathered = NULL;
  CUDA(cudaSetDevice(devices[0]));
  CUDA(cudaMalloc((void **)&gathered, N));
  float ms[16];
  CHECK(recoil_multi_decode(c, clen, (uint32_t)n_dev, devices, outs, 0, gathered, ms));
  memset(host, 0, N);
  CUDA(cudaMemcpy(host, gathered, N, cudaMemcpyDeviceToHost));
  if (memcmp(host, sym, N) != 0) {
    fprintf(stderr, "multi-device decode mismatch\n");
    return 1;
  }
  printf("%d shards, gather %s: bit-exact (kernel ms:", n_dev, recoil_multi_nccl_available() ? "NCCL-capable" : "peer");
  for (int d = 0; d < n_dev; ++d) printf(" %.3f", ms[d]);
  printf(")\n");
  for (int d = 0; d < n_dev; ++d) cudaFree(outs[d]);
  cudaFree(gathered);
  free(sym);
  free(c);
  free(small);
  free(host);
  return 0;
}
