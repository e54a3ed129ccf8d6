// Measurement helper: the memory-system ceiling of the blocked-distributing
// store pattern, with NO ranking work.  148 persistent CTAs each stream their
// own contiguous chunk of 16-byte records (coalesced loads) and write every
// tile out as per-bucket runs of RUN records at the CTA's private cursor of
// each of NB buckets (the X-row layout: bucket-major, CTA-minor).  RUN = T/NB
// is what a T-record tile gives a uniform bucket.  Reports GB/s (read+write)
// against a plain copy.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/runs_bench.cu -o tools/runs_bench
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <typename R>
__global__ void __launch_bounds__(512, 2) k_runs(const R* __restrict__ in, R* __restrict__ out, uint64_t per_cta,
                                                 uint32_t nb, uint32_t run, uint32_t shift) {
  // per_cta records per CTA; per bucket the CTA owns per_cta / nb output slots
  const uint64_t cta = blockIdx.x, G = gridDim.x;
  const uint64_t slots = per_cta / nb;              // per (bucket, cta)
  const R* src = in + cta * per_cta;
  const uint32_t T = nb * run;
  for (uint64_t t = 0; t * T < per_cta; ++t) {
    for (uint32_t i = threadIdx.x; i < T; i += blockDim.x) {
      const uint32_t b = i / run, r = i % run;
      const R v = src[t * T + i];
      out[(static_cast<uint64_t>(b) * G + cta) * slots + shift + t * run + r] = v;
    }
  }
}

template <typename R>
__global__ void k_copy(const R* __restrict__ in, R* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) out[i] = in[i];
}

template <typename R>
void run_all(const char* name, uint64_t n) {
  R *in, *out;
  CK(cudaMalloc(&in, n * sizeof(R)));
  CK(cudaMalloc(&out, (n + 64) * sizeof(R)));
  CK(cudaMemset(in, 1, n * sizeof(R)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_copy<R><<<148 * 8, 512>>>(in, out, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("%s copy: %.3f ms  %.0f GB/s\n", name, ms, 2.0 * n * sizeof(R) / ms / 1e6);
  const uint32_t nb = 1024;
  const int G = 148 * 2;
  for (uint32_t shift = 0; shift <= 1; ++shift)
    for (uint32_t run = 1; run <= 64; run *= 2) {
      const uint64_t per_cta = (n / G) / (nb * 64) * (nb * 64);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_runs<R><<<G, 512>>>(in, out, per_cta, nb, run, shift);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
      }
      printf("%s runs of %2u records (%4zu B)%s: %.3f ms  %.0f GB/s\n", name, run, run * sizeof(R),
             shift ? " misaligned by one record" : "", ms, 2.0 * per_cta * G * sizeof(R) / ms / 1e6);
    }
  cudaFree(in);
  cudaFree(out);
}

int main() {
  run_all<ulonglong2>("16B", 1ull << 28);
  run_all<uint64_t>("8B", 1ull << 29);
  run_all<uint32_t>("4B", 1ull << 30);
  return 0;
}
