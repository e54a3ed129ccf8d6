// Measurement helper: can TMA bulk stores (cp.async.bulk.global.shared::cta)
// write the blocked-distributing output -- ~1024 runs of 64..256 bytes per
// 4096-record tile, each at its own cursor -- faster than lane stores?
// 148 CTAs x 512 threads; a 64 KB shared tile is written out every
// iteration as NB runs of RUN bytes, run r of CTA c at
// out[(r * 148 + c) * slot + it * RUN + shift].  Write-only traffic.
//   bulk : thread t issues the bulk stores of runs t, t + 512, ...; one
//          commit + wait_group.read per iteration
//   lanes: RUN/16 adjacent lanes store one run with 16-byte stores
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/bulk_store_bench.cu -o tools/bulk_store_bench
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

constexpr int kTileBytes = 65536;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <bool BULK>
__global__ void __launch_bounds__(512, 1) k_store(unsigned char* __restrict__ out, uint64_t slot, uint32_t run,
                                                  uint32_t shift, uint32_t iters) {
  extern __shared__ __align__(128) unsigned char tile[];
  for (uint32_t i = threadIdx.x; i < kTileBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(tile)[i] = make_uint4(i, blockIdx.x, 3, 4);
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint32_t nb = kTileBytes / run;
  for (uint32_t it = 0; it < iters; ++it) {
    if constexpr (BULK) {
      for (uint32_t r = threadIdx.x; r < nb; r += blockDim.x) {
        unsigned char* dst = out + (static_cast<uint64_t>(r) * gridDim.x + blockIdx.x) * slot + static_cast<uint64_t>(it) * run + shift;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(tile + r * run)), "r"(run) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    } else {
      const uint32_t per = run / 16;   // lanes per run
      for (uint32_t q = threadIdx.x; q < kTileBytes / 16; q += blockDim.x) {
        const uint32_t r = q / per, o = q % per;
        unsigned char* dst = out + (static_cast<uint64_t>(r) * gridDim.x + blockIdx.x) * slot + static_cast<uint64_t>(it) * run + shift;
        reinterpret_cast<uint4*>(dst)[o] = reinterpret_cast<const uint4*>(tile)[q];
      }
    }
    __syncthreads();
  }
}

int main() {
  const uint32_t iters = 400;
  const int G = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  CK(cudaFuncSetAttribute(k_store<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes));
  CK(cudaFuncSetAttribute(k_store<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes));
  for (uint32_t run : {64u, 128u, 256u, 1024u}) {
    const uint32_t nb = kTileBytes / run;
    const uint64_t slot = static_cast<uint64_t>(iters) * run + 64;   // bytes per (run, CTA) stream, 64-byte aligned streams
    const uint64_t bytes = static_cast<uint64_t>(nb) * G * slot + 64;
    unsigned char* out;
    CK(cudaMalloc(&out, bytes));
    for (uint32_t shift : {0u, 16u}) {
      for (int bulk = 1; bulk >= 0; --bulk) {
        float ms = 0;
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (bulk) k_store<true><<<G, 512, kTileBytes>>>(out, slot, run, shift, iters);
          else k_store<false><<<G, 512, kTileBytes>>>(out, slot, run, shift, iters);
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          cudaEventElapsedTime(&ms, e0, e1);
        }
        const double gb = double(kTileBytes) * G * iters / 1e9;
        printf("run %4u B shift %2u %-5s: %.3f ms  %.0f GB/s written  (%.0f cycles per 64 KB tile at 1.965 GHz)\n", run, shift,
               bulk ? "bulk" : "lanes", ms, gb / (ms / 1e3), ms * 1e-3 * 1.965e9 / iters);
      }
    }
    CK(cudaFree(out));
  }
  return 0;
}
