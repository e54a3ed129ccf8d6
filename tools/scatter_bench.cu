// Measurement helper: how fast can a stable multisplit scatter write
// 16-byte records without shared-memory staging?  Compares
//   copy   : coalesced SoA -> pair copy (the HBM ceiling for this traffic)
//   free   : per-record shared atomicAdd on CTA cursors (unordered across
//            warps), scattered 16-byte stores
//   token  : the same, but warps take the cursor atomics in input order
//            (a shared token passed warp to warp) -> stable
// Buckets: 1024 light (mix64 of the key) + 39 hot keys holding HOT% of the
// records (the c2 level-0 shape).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/scatter_bench.cu -o tools/scatter_bench
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

constexpr int NL = 1024, NH = 39, NB = NL + NH;

__device__ __forceinline__ uint32_t bucket(uint64_t k) {
  if (k < NH) return NL + static_cast<uint32_t>(k);
  return static_cast<uint32_t>(mix64(k)) & (NL - 1);
}

__global__ void k_gen(uint64_t* keys, uint64_t* vals, uint64_t n, uint32_t hot_pct) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = mix64(i * 0x9e3779b97f4a7c15ull + 12345);
    keys[i] = (r % 100) < hot_pct ? (r >> 32) % NH : NH + (r >> 20);
    vals[i] = i;
  }
}

__global__ void k_count(const uint64_t* keys, uint64_t n, uint64_t chunk, uint32_t* C) {
  __shared__ uint32_t c[NB];
  const uint64_t row = blockIdx.x;
  for (int b = threadIdx.x; b < NB; b += blockDim.x) c[b] = 0;
  __syncthreads();
  const uint64_t lo = row * chunk, hi = (n < lo + chunk ? n : lo + chunk);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&c[bucket(keys[i])], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += blockDim.x) C[row * NB + b] = c[b];
}

__global__ void k_copy(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, ulonglong2* __restrict__ out,
                       uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = make_ulonglong2(__ldg(keys + i), __ldg(vals + i));
}

// One CTA per row at a time (rows claimed in order from a counter); 16 warps,
// each warp owns 256 consecutive records of a 4096-record tile.
template <bool TOKEN, int ITEMS, int MINB = 1>
__global__ void __launch_bounds__(512, MINB)
k_scatter(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, ulonglong2* __restrict__ out, uint64_t n,
          uint64_t chunk, uint32_t nrows, const uint64_t* __restrict__ X, uint32_t* ctr) {
  __shared__ uint32_t cur[NB];
  __shared__ uint64_t rbase;
  __shared__ uint32_t srow;
  __shared__ volatile uint32_t token;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = 16, WT = 32 * ITEMS, T = NW * WT;
  for (;;) {
    if (threadIdx.x == 0) srow = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t row = srow;
    if (row >= nrows) return;
    const uint64_t* xr = X + (uint64_t)row * NB;
    if (threadIdx.x == 0) { rbase = xr[0]; token = 0; }
    __syncthreads();
    for (int b = threadIdx.x; b < NB; b += 512) cur[b] = (uint32_t)(xr[b] - rbase);
    __syncthreads();
    const uint64_t lo = (uint64_t)row * chunk, hi = (n < lo + chunk ? n : lo + chunk);
    const uint64_t rb = rbase;
    uint32_t seq = w;
    for (uint64_t t0 = lo; t0 < hi; t0 += T, seq += NW) {
      const uint64_t base = t0 + (uint64_t)w * WT;
      uint64_t k[ITEMS], v[ITEMS];
      uint32_t b[ITEMS], d[ITEMS];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const uint64_t idx = base + i * 32 + lane;
        const bool ok = idx < hi;
        k[i] = ok ? __ldg(keys + idx) : 0;
        v[i] = ok ? __ldg(vals + idx) : 0;
        b[i] = ok ? bucket(k[i]) : 0xFFFFFFFFu;
      }
      if (TOKEN) {
        if (lane == 0) while (token != seq) {}
        __syncwarp();
      }
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        d[i] = b[i] != 0xFFFFFFFFu ? atomicAdd(&cur[b[i]], 1u) : 0;
        __syncwarp();
      }
      if (TOKEN) {
        __threadfence_block();
        __syncwarp();
        if (lane == 0) token = seq + 1;
      }
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (b[i] != 0xFFFFFFFFu) out[rb + d[i]] = make_ulonglong2(k[i], v[i]);
    }
    __syncthreads();
  }
}

__global__ void k_check(const ulonglong2* out, uint64_t n, const uint64_t* off, uint32_t* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const ulonglong2 r = out[i];
    const uint32_t b = bucket(r.x);
    if (i < off[b] || i >= off[b + 1]) { atomicAdd(bad, 1u); continue; }
    if (i > off[b] && out[i - 1].y >= r.y) atomicAdd(bad + 1, 1u);   // stability
  }
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 29);
  const uint32_t hot = argc > 2 ? atoi(argv[2]) : 58;
  const uint64_t chunk = ((n + 4735) / 4736 + 4095) & ~4095ull;
  const uint32_t nrows = (uint32_t)((n + chunk - 1) / chunk);
  uint64_t *keys, *vals, *X, *off;
  ulonglong2* out;
  uint32_t *C, *ctr, *bad;
  CK(cudaMalloc(&keys, n * 8)); CK(cudaMalloc(&vals, n * 8)); CK(cudaMalloc(&out, n * 16));
  CK(cudaMalloc(&C, (size_t)nrows * NB * 4)); CK(cudaMalloc(&X, (size_t)nrows * NB * 8));
  CK(cudaMalloc(&off, (NB + 1) * 8)); CK(cudaMalloc(&ctr, 4)); CK(cudaMalloc(&bad, 8));
  k_gen<<<1184, 256>>>(keys, vals, n, hot);
  k_count<<<nrows, 512>>>(keys, n, chunk, C);
  std::vector<uint32_t> hC((size_t)nrows * NB);
  std::vector<uint64_t> hX((size_t)nrows * NB), hoff(NB + 1);
  CK(cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost));
  uint64_t run = 0;
  for (int b = 0; b < NB; ++b) {
    hoff[b] = run;
    for (uint32_t r = 0; r < nrows; ++r) { hX[(size_t)r * NB + b] = run; run += hC[(size_t)r * NB + b]; }
  }
  hoff[NB] = run;
  CK(cudaMemcpy(X, hX.data(), hX.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(off, hoff.data(), hoff.size() * 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn, bool check) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemset(ctr, 0, 4));
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    uint32_t hb[2] = {0, 0};
    if (check) {
      CK(cudaMemset(bad, 0, 8));
      k_check<<<1184, 256>>>(out, n, off, bad);
      CK(cudaMemcpy(hb, bad, 8, cudaMemcpyDeviceToHost));
    }
    printf("%-12s n=%llu hot=%u%%: %.3f ms  %.0f GB/s (32 B/rec)  misplaced=%u unstable=%u\n", name,
           (unsigned long long)n, hot, best, 32.0 * n / best / 1e6, hb[0], hb[1]);
  };
  timeit("copy", [&] { k_copy<<<148 * 8, 512>>>(keys, vals, out, n); }, false);
  timeit("free8", [&] { k_scatter<false, 8><<<148, 512>>>(keys, vals, out, n, chunk, nrows, X, ctr); }, true);
  timeit("token8", [&] { k_scatter<true, 8><<<148, 512>>>(keys, vals, out, n, chunk, nrows, X, ctr); }, true);
  timeit("token4", [&] { k_scatter<true, 4><<<148, 512>>>(keys, vals, out, n, chunk, nrows, X, ctr); }, true);
  timeit("token8x2", [&] { k_scatter<true, 8, 2><<<296, 512>>>(keys, vals, out, n, chunk, nrows, X, ctr); }, true);
  timeit("token4x2", [&] { k_scatter<true, 4, 2><<<296, 512>>>(keys, vals, out, n, chunk, nrows, X, ctr); }, true);
  timeit("token16", [&] { k_scatter<true, 16><<<148, 512>>>(keys, vals, out, n, chunk, nrows, X, ctr); }, true);
  CK(cudaGetLastError());
  return 0;
}
