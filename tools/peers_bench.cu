// Microbenchmark: cost of warp peer masks / shared counters on sm_100
// (MATCH.ANY vs ballots vs shared-memory atomicOr masks vs atomicAdd), to
// choose the ranking primitive of the distribute and leaf kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t rnd(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; return x ^ (x >> 16); }

// MODE 0 match_any, 1 ballot peers, 2 atomicOr masks, 3 atomicAdd counters,
// 6 baseline (no peers).  HOT: ~60% of lanes draw one of 4 values.
template <int MODE, int BITS, bool HOT>
__global__ void k(uint32_t* out, int iters) {
  __shared__ uint32_t masks[8][MODE >= 2 ? (1 << BITS) : 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = lane; i < (MODE >= 2 ? (1 << BITS) : 1); i += 32) masks[w][i] = 0;
  __syncwarp();
  uint32_t acc = 0, x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    x = rnd(x);
    uint32_t v = x & ((1u << BITS) - 1);
    if (HOT && (x >> 28) < 10) v = (x >> 24) & 3;
    uint32_t peers = 0;
    if constexpr (MODE == 0) {
      peers = __match_any_sync(0xffffffffu, v);
    } else if constexpr (MODE == 1) {
      uint32_t m = 0xffffffffu;
#pragma unroll
      for (int j = 0; j < BITS; ++j) {
        const uint32_t bit = (v >> j) & 1u;
        const uint32_t b = __ballot_sync(0xffffffffu, bit);
        m &= bit ? b : ~b;
      }
      peers = m;
    } else if constexpr (MODE == 2) {
      atomicOr(&masks[w][v], 1u << lane);
      __syncwarp();
      peers = masks[w][v];
      __syncwarp();
      masks[w][v] = 0;
      __syncwarp();
    } else if constexpr (MODE == 3) {
      atomicAdd(&masks[w][v], 1u);
      peers = v;
    } else {
      peers = v;
    }
    acc += __popc(peers & ((1u << lane) - 1)) + peers;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + masks[w][lane & 1];
}

template <int MODE, int BITS, bool HOT>
void run(const char* name, uint32_t* out) {
  const int iters = 4096, grid = 148 * 8, block = 256;
  k<MODE, BITS, HOT><<<grid, block>>>(out, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, BITS, HOT><<<grid, block>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double warp_ops = double(grid) * (block / 32) * iters;
  printf("%-16s bits=%2d hot=%d  %.3f ms  %6.2f SM-cycles/warp-op (1.965 GHz)\n", name, BITS, int(HOT), ms,
         ms * 1e-3 * 1.965e9 * 148 / warp_ops);
}

int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<6, 7, false>("baseline", out);
  run<0, 7, false>("match_any", out);
  run<0, 7, true>("match_any", out);
  run<1, 7, false>("ballot_peers", out);
  run<1, 11, false>("ballot_peers", out);
  run<2, 7, false>("atomicOr-masks", out);
  run<2, 7, true>("atomicOr-masks", out);
  run<2, 10, false>("atomicOr-masks", out);
  run<3, 10, false>("atomicAdd", out);
  run<3, 10, true>("atomicAdd", out);
  return 0;
}
