// Record-dump rows <-> SoA device columns (records.py:149-202).
//
// A dump stores n packed little-endian rows, key bytes then value bytes
// (row = (key_width + value_width) / 8 bytes).  The reference splits them
// with numpy views and copies on the host; here the raw payload is copied
// to HBM as-is and split (or packed) by one bandwidth-bound kernel: each CTA
// stages a tile of whole rows in shared memory with coalesced 4-byte loads,
// then writes the key and value columns of those rows as contiguous runs.
// Widths are multiples of 4 bytes (keys 4/8/16, values 4*k), so the kernel
// works in 32-bit words; rows wider than kRowsDirectWords go word by word
// straight through global memory.
#include <cuda_runtime.h>

#include "abi.cuh"

namespace ss {
namespace {

constexpr uint32_t kRowsThreads = 512;
constexpr uint32_t kRowsTileWords = 12288;   // 48 KB of staged rows per CTA
constexpr uint32_t kRowsDirectWords = 384;    // wider rows skip the staging

// unpack: rows -> (keys, values); pack: the reverse.  kw / vw = key / value
// words per row, rw = kw + vw; T = rows per tile.
template <bool UNPACK>
__global__ void __launch_bounds__(kRowsThreads)
k_rows(uint32_t* __restrict__ rows, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, uint64_t n,
       uint32_t kw, uint32_t vw, uint32_t T) {
  extern __shared__ uint32_t tile[];
  const uint32_t rw = kw + vw;
  for (uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * T; r0 < n; r0 += static_cast<uint64_t>(gridDim.x) * T) {
    const uint32_t nr = static_cast<uint32_t>(n - r0 < T ? n - r0 : T);
    const uint64_t kbase = r0 * kw, vbase = r0 * vw, rbase = r0 * rw;
    if constexpr (UNPACK) {
      for (uint32_t i = threadIdx.x; i < nr * rw; i += blockDim.x) tile[i] = __ldcs(rows + rbase + i);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nr * kw; i += blockDim.x) keys[kbase + i] = tile[(i / kw) * rw + i % kw];
      for (uint32_t i = threadIdx.x; i < nr * vw; i += blockDim.x)
        vals[vbase + i] = tile[(i / vw) * rw + kw + i % vw];
    } else {
      for (uint32_t i = threadIdx.x; i < nr * kw; i += blockDim.x) tile[(i / kw) * rw + i % kw] = __ldcs(keys + kbase + i);
      for (uint32_t i = threadIdx.x; i < nr * vw; i += blockDim.x)
        tile[(i / vw) * rw + kw + i % vw] = __ldcs(vals + vbase + i);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nr * rw; i += blockDim.x) rows[rbase + i] = tile[i];
    }
    __syncthreads();
  }
}

template <bool UNPACK>
__global__ void k_rows_direct(uint32_t* __restrict__ rows, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                              uint64_t n, uint32_t kw, uint32_t vw) {
  const uint32_t rw = kw + vw;
  const uint64_t total = n * rw;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / rw;
    const uint32_t c = static_cast<uint32_t>(i % rw);
    uint32_t* col = c < kw ? keys + r * kw + c : vals + r * vw + (c - kw);
    if constexpr (UNPACK) *col = rows[i];
    else rows[i] = *col;
  }
}

template <bool UNPACK>
void run_rows(void* rows, void* keys, void* vals, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
              cudaStream_t st) {
  if (key_bytes != 4 && key_bytes != 8 && key_bytes != 16)
    throw Fail(SS_ERR_CONTRACT, "key_bytes must be 4, 8 or 16");
  if (value_bytes % 4) throw Fail(SS_ERR_CONTRACT, "value_bytes must be a multiple of 4");
  if (n && (!rows || !keys || (value_bytes && !vals))) throw Fail(SS_ERR_CONTRACT, "NULL buffer");
  if ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(vals)) & 3)
    throw Fail(SS_ERR_CONTRACT, "buffers must be 4-byte aligned");
  if (!n) return;
  const uint32_t kw = key_bytes / 4, vw = value_bytes / 4, rw = kw + vw;
  auto* r = static_cast<uint32_t*>(rows);
  auto* k = static_cast<uint32_t*>(keys);
  auto* v = static_cast<uint32_t*>(vals);
  if (rw > kRowsDirectWords) {
    k_rows_direct<UNPACK><<<148 * 8, 256, 0, st>>>(r, k, v, n, kw, vw);
  } else {
    const uint32_t T = kRowsTileWords / rw;
    const uint64_t tiles = (n + T - 1) / T;
    const uint32_t grid = static_cast<uint32_t>(tiles < 148ull * 4 ? tiles : 148ull * 4);
    const size_t smem = static_cast<size_t>(T) * rw * 4;
    k_rows<UNPACK><<<grid, kRowsThreads, smem, st>>>(r, k, v, n, kw, vw, T);
  }
  SS_CUDA(cudaGetLastError());
}

}  // namespace
}  // namespace ss

extern "C" {

int ss_records_unpack(const void* rows, uint64_t n, uint32_t key_bytes, uint32_t value_bytes, void* keys,
                      void* values, void* stream) {
  return ss::guarded([&] {
    ss::run_rows<true>(const_cast<void*>(rows), keys, values, n, key_bytes, value_bytes, ss::as_stream(stream));
  });
}

int ss_records_pack(const void* keys, const void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                    void* rows, void* stream) {
  return ss::guarded([&] {
    ss::run_rows<false>(rows, const_cast<void*>(keys), const_cast<void*>(values), n, key_bytes, value_bytes,
                        ss::as_stream(stream));
  });
}

}  // extern "C"
