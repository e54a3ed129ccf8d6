// Microbenchmark: cycles per call of the distribute kernel's block scans at
// 512 threads (one CTA per SM): u32 / u64 block_excl_scan and radix_scan.
// Build: nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -I paper_2304_10078_b200/csrc tools/scan_bench.cu -o tools/scan_bench
#include <cstdio>
#include "common.cuh"
#include "dist.cuh"

using namespace ss;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters) {
  __shared__ uint32_t dh[16 * kDhStride];
  __shared__ unsigned long long red64[33];
  __shared__ uint32_t red32[33];
  for (int i = threadIdx.x; i < 16 * kDhStride; i += 512) dh[i] = i & 3;
  __syncthreads();
  unsigned long long acc = 0, t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
      uint32_t tot;
      acc += block_excl_scan<uint32_t>(threadIdx.x + it, red32, tot);
    } else if constexpr (MODE == 1) {
      unsigned long long tot;
      acc += block_excl_scan<unsigned long long>(threadIdx.x + it, red64, tot);
    } else if constexpr (MODE == 2) {
      acc += radix_scan<16>(dh, red64, threadIdx.x);
      __syncthreads();
    } else {
      __syncthreads();
      acc += it;
    }
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  if (acc == 12345) out[1000] = acc;
}

template <int MODE>
void run(const char* name, unsigned long long* d) {
  k<MODE><<<148, 512>>>(d, 2000);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-22s %8.1f cycles per call\n", name, s / 148);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1001 * 8);
  run<3>("syncthreads only", d);
  run<0>("block_excl_scan u32", d);
  run<1>("block_excl_scan u64", d);
  run<2>("radix_scan<16>+sync", d);
  return 0;
}
