// Microbenchmark: stable warp rank of 7-bit digits (the distribute kernel's
// inner step) on skewed digit streams, at the kernel's occupancy (one
// 512-thread CTA per SM, 8 items per thread).  Variants:
//   0 atomicOr peer masks + shared counters (dist.cuh radix_rank)
//   1 7-ballot peers + shared counters
//   2 match_any peers + shared counters
// HOT = percentage of lanes drawing one of 4 hot digits.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/rank_bench.cu -o tools/rank_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rnd(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; return x ^ (x >> 16);
}
__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

template <int MODE, int HOT>
__global__ void __launch_bounds__(512, 1) k(uint32_t* out, int iters) {
  __shared__ uint32_t cnt[16][128];
  __shared__ uint32_t msk[16][128];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  for (int i = lane; i < 128; i += 32) { cnt[w][i] = 0; msk[w][i] = 0; }
  __syncwarp();
  uint32_t x = blockIdx.x * 512 + threadIdx.x, acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      x = rnd(x + q);
      d[q] = ((x >> 8) % 100 + 1 <= HOT) ? (x & 3) * 37 : (x >> 20) & 127;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t peers;
      if constexpr (MODE == 0) {
        atomicOr(&msk[w][d[q]], 1u << lane);
        __syncwarp();
        peers = msk[w][d[q]];
      } else if constexpr (MODE == 1) {
        peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 7; ++b) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (d[q] >> b) & 1u);
          peers &= ((d[q] >> b) & 1u) ? bal : ~bal;
        }
      } else if constexpr (MODE == 2) {
        peers = __match_any_sync(0xffffffffu, d[q]);
      } else if constexpr (MODE == 4) {   // hardware-aggregated increment: old value = rank
        acc += atomicAdd(&cnt[w][d[q]], 1u);
        __syncwarp();
        continue;
      } else {   // baseline: digit generation only
        acc += d[q];
        continue;
      }
      const uint32_t base = cnt[w][d[q]];
      __syncwarp();
      if (lane == 31 - __clz(peers)) {
        cnt[w][d[q]] = base + __popc(peers);
        if constexpr (MODE == 0) msk[w][d[q]] = 0;
      }
      acc += base + __popc(peers & lt);
      __syncwarp();
    }
  }
  out[blockIdx.x * 512 + threadIdx.x] = acc;
}

// Checks atomicAdd(+1) old values against base + popc(peers & lanemask_lt)
// (lane-order ranks) on random and skewed digits; counts mismatches.
__global__ void verify(unsigned long long* bad, int iters, int hot) {
  __shared__ uint32_t cnt[16][128];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  for (int i = lane; i < 128; i += 32) cnt[w][i] = 0;
  __syncwarp();
  uint32_t x = blockIdx.x * 512 + threadIdx.x * 7919u, nbad = 0;
  for (int it = 0; it < iters; ++it) {
    x = rnd(x + it);
    const uint32_t d = ((x >> 8) % 100 + 1 <= (uint32_t)hot) ? (x & 3) * 37 : (x >> 20) & 127;
    const bool active = ((x >> 4) & 15) != 0 || hot == 100;   // some inactive lanes
    const uint32_t peers = __match_any_sync(0xffffffffu, active ? d : 1000u + lane);
    const uint32_t before = cnt[w][d];
    __syncwarp();
    uint32_t old = 0;
    if (active) old = atomicAdd(&cnt[w][d], 1u);
    __syncwarp();
    if (active && old != before + __popc(peers & lt)) ++nbad;
    __syncwarp();
  }
  atomicAdd(bad, (unsigned long long)nbad);
}

template <int MODE, int HOT>
void run(const char* name, uint32_t* out) {
  const int iters = 2048;
  k<MODE, HOT><<<148, 512>>>(out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, HOT><<<148, 512>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double warp_items = 16.0 * 8 * iters;   // per SM
  printf("%-10s hot=%3d%%  %.3f ms  %6.2f SM-cycles per warp-item (1.965 GHz)\n", name, HOT, ms,
         ms * 1e-3 * 1.965e9 / warp_items);
}

int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 512 * 4);
  unsigned long long* bad; cudaMalloc(&bad, 8);
  for (int hot : {0, 50, 90, 100}) {
    cudaMemset(bad, 0, 8);
    verify<<<148 * 4, 512>>>(bad, 20000, hot);
    unsigned long long h = 0;
    cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    printf("verify lane-order ranks hot=%3d%%: %llu mismatches of %.2e lane-ops\n", hot, h, 148.0 * 4 * 512 * 20000);
  }
  run<0, 0>("atomicOr", out);  run<0, 50>("atomicOr", out);  run<0, 90>("atomicOr", out);
  run<1, 0>("ballot7", out);   run<1, 50>("ballot7", out);   run<1, 90>("ballot7", out);
  run<3, 50>("baseline", out);
  run<4, 0>("popc_inc", out);  run<4, 50>("popc_inc", out);  run<4, 90>("popc_inc", out);
  run<2, 0>("match_any", out); run<2, 50>("match_any", out); run<2, 90>("match_any", out);
  return 0;
}
