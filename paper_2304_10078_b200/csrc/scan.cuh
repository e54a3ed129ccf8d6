// Device-wide exclusive scan (reduce-then-scan, three launches) used to
// place variable-length outputs deterministically (aggregate result pairs,
// partition counts).
#pragma once

#include "common.cuh"

namespace ss {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr uint64_t kScanTile = static_cast<uint64_t>(kScanThreads) * kScanItems;

template <typename T>
static __global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(const T* __restrict__ in, uint64_t n, uint64_t* __restrict__ part) {
  __shared__ uint64_t red[33];
  const uint64_t base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  uint64_t s = 0;
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += in[base + k];
  uint64_t tot;
  block_excl_scan<uint64_t>(s, red, tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

static __global__ void __launch_bounds__(kScanThreads)
k_scan_parts(uint64_t* __restrict__ part, uint64_t nparts, uint64_t* __restrict__ total) {
  __shared__ uint64_t red[33];
  uint64_t carry = 0;
  for (uint64_t b = 0; b < nparts; b += kScanThreads) {
    const uint64_t i = b + threadIdx.x;
    const uint64_t v = i < nparts ? part[i] : 0;
    uint64_t t;
    const uint64_t ex = block_excl_scan<uint64_t>(v, red, t);
    if (i < nparts) part[i] = carry + ex;
    carry += t;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

template <typename T>
static __global__ void __launch_bounds__(kScanThreads)
k_scan_apply(const T* __restrict__ in, uint64_t n, const uint64_t* __restrict__ part, uint64_t* __restrict__ out) {
  __shared__ uint64_t red[33];
  const uint64_t base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  T v[kScanItems];
  uint64_t s = 0;
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : T(0);
    s += v[k];
  }
  uint64_t tot;
  uint64_t run = part[blockIdx.x] + block_excl_scan<uint64_t>(s, red, tot);
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

inline uint64_t scan_parts_needed(uint64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

// out[i] = sum(in[0..i)); *total (device) = sum(in).  `part` needs
// scan_parts_needed(n) entries.
template <typename T>
inline void device_exclusive_scan(const T* in, uint64_t n, uint64_t* out, uint64_t* part, uint64_t* total,
                                  cudaStream_t st) {
  if (n == 0) {
    cudaMemsetAsync(total, 0, sizeof(uint64_t), st);
    return;
  }
  const uint64_t nb = (n + kScanTile - 1) / kScanTile;
  k_scan_reduce<T><<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(in, n, part);
  k_scan_parts<<<1, kScanThreads, 0, st>>>(part, nb, total);
  k_scan_apply<T><<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(in, n, part, out);
}

}  // namespace ss
