// Byte-view keys (adapters.py:200-275, hashing.py:56-106, ngrams.py): keys
// are (offset, length) views into a caller-owned byte arena; hash, equality
// and order are those of the referenced bytes.
//
// The device path reduces them to 128-bit identity keys (paper_2304_10078_b200/
// bytes_keys.py): lo = the content hash, hi = the length (eq) or the exact
// lexicographic rank of the content (lt).  The semisort then takes the same
// buckets (the hash is the reference's), the same heavy keys and the same
// leaf order (chained by hash, or by (rank, ...) = content order) as the
// reference does with content comparisons.  These kernels compute the
// hashes, the 7-byte chunks the lt rank is refined on, and the content
// equality checks that make a (hash, length) collision between different
// contents fail loudly instead of merging groups.
#include <cstdint>

#include "abi.cuh"
#include "common.cuh"

namespace ss {

constexpr uint64_t kPolyMult = 0x00000100000001B3ull;   // hashing.py:19 (the FNV-1a prime)

// polynomial over the bytes, then mix64(poly ^ mix64(len)) (hashing.py:56-66,
// BytePrefixHasher.hash_views :98-106)
__global__ void k_bytes_hash(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ views, uint64_t n,
                             uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t off = views[2 * i], len = views[2 * i + 1];
    const uint8_t* p = arena + off;
    uint64_t acc = 0;
    uint64_t j = 0;
    // 8 bytes per step where the view is 8-byte aligned inside the arena
    if (((reinterpret_cast<uintptr_t>(p)) & 7) == 0)
      for (; j + 8 <= len; j += 8) {
        const uint64_t w = __ldg(reinterpret_cast<const unsigned long long*>(p + j));
#pragma unroll
        for (int b = 0; b < 8; ++b) acc = acc * kPolyMult + ((w >> (8 * b)) & 0xFF);
      }
    for (; j < len; ++j) acc = acc * kPolyMult + __ldg(p + j);
    out[i] = mix64(acc ^ mix64(len));
  }
}

// Bytes [7c, 7c + 7) of each view as 9-bit digits (byte + 1; 0 past the end),
// most significant first: comparing these words for c = 0, 1, ... is the
// lexicographic byte order with a proper prefix sorting first.  Signed
// int64 (63 bits used) so torch can sort them.
__global__ void k_bytes_chunk(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ views, uint64_t n,
                              uint64_t c, int64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t off = views[2 * i], len = views[2 * i + 1];
    uint64_t w = 0;
#pragma unroll
    for (int b = 0; b < 7; ++b) {
      const uint64_t j = 7 * c + b;
      const uint64_t d = j < len ? static_cast<uint64_t>(__ldg(arena + off + j)) + 1 : 0;
      w = (w << 9) | d;
    }
    out[i] = static_cast<int64_t>(w);
  }
}

// mismatches += [content(a[i]) != content(b[i])]
__global__ void k_bytes_equal(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ va,
                              const uint64_t* __restrict__ vb, uint64_t n, unsigned long long* __restrict__ bad) {
  unsigned long long mine = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t oa = va[2 * i], la = va[2 * i + 1], ob = vb[2 * i], lb = vb[2 * i + 1];
    bool eq = la == lb;
    for (uint64_t j = 0; eq && j < la; ++j) eq = __ldg(arena + oa + j) == __ldg(arena + ob + j);
    mine += eq ? 0 : 1;
  }
  if (mine) atomicAdd(bad, mine);
}

// every view inside the arena (records.py: views are caller-owned data)
__global__ void k_bytes_bounds(const uint64_t* __restrict__ views, uint64_t n, uint64_t arena_len,
                               unsigned long long* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t off = views[2 * i], len = views[2 * i + 1];
    if (off > arena_len || len > arena_len - off) atomicAdd(bad, 1ull);
  }
}

static uint32_t grid_for(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return static_cast<uint32_t>(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

// scratch word for the counters: the caller passes one u64 of device memory
static uint64_t read_counter(unsigned long long* d, cudaStream_t st) {
  unsigned long long h = 0;
  SS_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  return h;
}

}  // namespace ss

using namespace ss;

extern "C" {

int ss_bytes_hash(const void* arena, uint64_t arena_len, const void* views, uint64_t n, void* out_hash,
                  void* counter, void* stream) {
  return guarded([&] {
    cudaStream_t st = as_stream(stream);
    if (!n) return;
    if (!arena || !views || !out_hash || !counter) throw Fail(SS_ERR_CONFIG, "null pointer");
    auto* bad = static_cast<unsigned long long*>(counter);
    SS_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st));
    k_bytes_bounds<<<grid_for(n), 256, 0, st>>>(static_cast<const uint64_t*>(views), n, arena_len, bad);
    check_launch();
    if (read_counter(bad, st)) throw Fail(SS_ERR_CONFIG, "a byte view lies outside the arena");
    k_bytes_hash<<<grid_for(n), 256, 0, st>>>(static_cast<const uint8_t*>(arena), static_cast<const uint64_t*>(views),
                                              n, static_cast<uint64_t*>(out_hash));
    check_launch();
  });
}

int ss_bytes_chunk(const void* arena, const void* views, uint64_t n, uint64_t chunk, void* out, void* stream) {
  return guarded([&] {
    if (!n) return;
    k_bytes_chunk<<<grid_for(n), 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(arena),
                                                              static_cast<const uint64_t*>(views), n, chunk,
                                                              static_cast<int64_t*>(out));
    check_launch();
  });
}

int ss_bytes_equal(const void* arena, const void* views_a, const void* views_b, uint64_t n, void* counter,
                   uint64_t* out_mismatches, void* stream) {
  return guarded([&] {
    cudaStream_t st = as_stream(stream);
    if (!out_mismatches || !counter) throw Fail(SS_ERR_CONFIG, "null pointer");
    *out_mismatches = 0;
    if (!n) return;
    auto* bad = static_cast<unsigned long long*>(counter);
    SS_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st));
    k_bytes_equal<<<grid_for(n), 256, 0, st>>>(static_cast<const uint8_t*>(arena), static_cast<const uint64_t*>(views_a),
                                               static_cast<const uint64_t*>(views_b), n, bad);
    check_launch();
    *out_mismatches = read_counter(bad, st);
  });
}

}  // extern "C"
