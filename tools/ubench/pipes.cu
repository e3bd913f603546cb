// Microbenchmark: per-SM throughput of the instruction classes the decode loop uses.
// Each kernel runs ITER iterations of 8 independent chains per thread; clock64 per
// block gives cycles; report warp-instructions per SM-cycle for the op under test.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#define ITER 4096
__device__ uint32_t sink;
template <int OP>
__global__ void __launch_bounds__(256, 6) bench(uint32_t seed, long long* cyc) {
  __shared__ uint32_t sm[2048];
  for (int i = threadIdx.x; i < 2048; i += 256) sm[i] = i * 2654435761u;
  __syncthreads();
  uint32_t a[8];
  for (int k = 0; k < 8; ++k) a[k] = seed ^ (threadIdx.x * 977 + k * 131);
  uint32_t gt; asm("mov.u32 %0, %%lanemask_gt;" : "=r"(gt));
  uint32_t sh = seed & 7 | 8;
  long long t0 = clock64();
  #pragma unroll 1
  for (int it = 0; it < ITER; ++it) {
    #pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) a[k] = __popc(a[k] ^ gt) + a[k];                  // POPC (+IADD)
      if (OP == 1) a[k] = __umulhi(a[k], seed | 1) + a[k];           // IMAD.HI (+IADD)
      if (OP == 2) a[k] = (a[k] >> sh) ^ (a[k] + 0x9e3779b9u);       // SHF + LOP3/IADD
      if (OP == 3) a[k] = a[k] * (seed | 1) + 12345u;               // IMAD
      if (OP == 4) a[k] = __ballot_sync(0xffffffffu, a[k] & 1) + a[k];  // VOTE (+IADD)
      if (OP == 5) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm) + ((a[k] & 2047) << 2))); a[k] += v; }  // random LDS
      if (OP == 6) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm) + ((threadIdx.x & 31) << 2) + ((a[k] & 7) << 7))); a[k] += v; }  // conflict-free LDS
      if (OP == 7) a[k] = __reduce_add_sync(0xffffffffu, a[k] & 1) + a[k];  // REDUX
      if (OP == 8) a[k] = __shfl_sync(0xffffffffu, a[k], a[k] & 31) + 1u;  // SHFL
      if (OP == 9) a[k] = (a[k] ^ gt) + (a[k] & 0xFFF) ;                // 2 ALU-ish
      if (OP == 10) a[k] = __popc(a[k] ^ gt) + __ballot_sync(0xffffffffu, a[k] & 1);      // POPC + VOTE
      if (OP == 11) a[k] = __popc(a[k] ^ gt) + __shfl_sync(0xffffffffu, a[k], 3);          // POPC + SHFL
      if (OP == 12) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm) + ((a[k] & 2047) << 2))); a[k] = v + __shfl_sync(0xffffffffu, a[k], 5); }  // LDS + SHFL
      if (OP == 13) a[k] = __popc(a[k] ^ gt) + __umulhi(a[k], seed | 1);                   // POPC + IMAD.HI
      if (OP == 14) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm) + ((a[k] & 2047) << 2))); a[k] = v + __popc(a[k] ^ gt); }  // LDS + POPC
      if (OP == 15) { asm volatile("st.shared.u8 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x & 31) + ((k & 3) << 5)), "r"(a[k])); a[k] = a[k] * 3u + 1u; }  // STS.U8 + IMAD
      if (OP == 16) { uint32_t v; asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm) + ((a[k] & 31) << 1) + 64 * (k & 3))); a[k] = v + a[k] * 3u; }  // LDS.U16 consecutive
      if (OP == 17) a[k] = __ballot_sync(0xffffffffu, a[k] & 1) + (a[k] >> 3);             // VOTE + SHF
      if (OP == 18) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm) + ((a[k] & 2047) << 2))); a[k] = v + __reduce_add_sync(0xffffffffu, a[k] & 1); }  // LDS + REDUX
      if (OP == 19) a[k] = __popc(a[k] ^ gt) + __reduce_add_sync(0xffffffffu, a[k] & 1);   // POPC + REDUX
      if (OP == 20) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(sm) + ((a[k] & 2047) << 2))); a[k] = v + __ballot_sync(0xffffffffu, a[k] & 1); }  // LDS + VOTE
      if (OP == 21) { asm volatile("st.shared.u8 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x & 31) + ((k & 3) << 5)), "r"(a[k])); a[k] = __popc(a[k] ^ gt) + a[k]; }  // STS.U8 + POPC
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 0x12345678u) sink = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, int per_sm_blocks) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * per_sm_blocks;
  long long* d; cudaMalloc(&d, grid * sizeof(long long));
  bench<OP><<<grid, 256>>>(1u, d); cudaDeviceSynchronize();
  bench<OP><<<grid, 256>>>(3u, d); cudaDeviceSynchronize();
  long long* h = new long long[grid]; cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  double warp_ops = (double)per_sm_blocks * 8 /*warps*/ * ITER * 8 /*chains*/;
  printf("%-28s blocks/SM=%d  cycles=%lld  op-iterations per SM-cycle = %.3f (warp-level)\n", name, per_sm_blocks, mx, warp_ops / mx);
  delete[] h; cudaFree(d);
}
int main(int argc, char** argv) {
  int b = 6; int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0) {
    run<0>("POPC+IADD", b); run<1>("IMAD.HI+IADD", b); run<2>("SHF+LOP/IADD", b); run<3>("IMAD", b);
    run<4>("VOTE+IADD", b); run<5>("LDS random (2048 words)", b); run<6>("LDS conflict-free", b);
    run<7>("REDUX+IADD", b); run<8>("SHFL+IADD", b); run<9>("LOP3+IADD(2 ALU)", b);
    run<10>("POPC+VOTE", b); run<11>("POPC+SHFL", b); run<12>("LDS+SHFL", b); run<13>("POPC+IMAD.HI", b);
    run<14>("LDS+POPC", b); run<15>("STS.U8+IMAD", b); run<16>("LDS.U16 near+IMAD", b); run<17>("VOTE+SHF", b);
  }
  run<18>("LDS+REDUX", b); run<19>("POPC+REDUX", b); run<20>("LDS+VOTE", b); run<21>("STS.U8+POPC", b);
  return 0;
}
