// semisort< base cases in shared memory (core.py:425-429: a stable sort by
// key; adapters.py:132-135).  Sorting (key, index) makes equal keys keep
// input order, so a bitonic network gives exactly numpy's stable argsort.
//
//   k_leaf_lt_warp  one warp per leaf of <= kLeafWarpMax records: keys,
//                   values and indices in the warp's shared memory, the
//                   network synchronised by __syncwarp only;
//   k_leaf_lt_smem  one CTA per leaf of <= kLeafSmemMax records.
// Larger leaves keep the global-scratch k_leaf_lt (leaf.cuh).  Records are
// staged before any store, so in-place leaves (src == dst) are safe; ss is
// the source element stride (2 when the leaf lives in the pair scratch).
#pragma once

#include "common.cuh"
#include "leaf.cuh"
#include "types.cuh"

namespace ss {

// (key, index) order with padding (index >= m) last.
template <typename K>
__device__ __forceinline__ bool lt_after(K a, uint32_t ia, K b, uint32_t ib, uint32_t m) {
  if (ia >= m) return ib < m || ia > ib;
  if (ib >= m) return false;
  return a > b || (a == b && ia > ib);
}

// Bitonic network over N (power of two) entries; `lanes` threads starting at
// thread `t0` of the group cooperate; sync() separates stages.
template <typename K, typename Sync>
__device__ __forceinline__ void bitonic_kv(K* key, uint16_t* idx, uint32_t N, uint32_t m, uint32_t t, uint32_t lanes,
                                           Sync sync) {
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = t; i < N; i += lanes) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const K a = key[i], b = key[ixj];
          const uint32_t ia = idx[i], ib = idx[ixj];
          const bool up = (i & k) == 0;
          if (lt_after(a, ia, b, ib, m) == up) {
            key[i] = b;
            key[ixj] = a;
            idx[i] = static_cast<uint16_t>(ib);
            idx[ixj] = static_cast<uint16_t>(ia);
          }
        }
      }
      sync();
    }
  }
}

template <typename K, typename V>
struct LtWarpSmem {
  K key[kLeafWarpMax];
  V val[ValTraits<V>::bytes ? kLeafWarpMax : 1];
  uint16_t idx[kLeafWarpMax];
};

template <typename K, typename V>
__global__ void __launch_bounds__(kLeafWarpWarps * 32)
k_leaf_lt_warp(const K* __restrict__ src_k, const V* __restrict__ src_v, K* __restrict__ dst_k,
               V* __restrict__ dst_v, const Leaf* __restrict__ leaves, uint32_t n_leaves, uint32_t ss) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  LtWarpSmem<K, V>& w = reinterpret_cast<LtWarpSmem<K, V>*>(smem)[warp_id()];
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kLeafWarpWarps + warp_id(), nw = gridDim.x * kLeafWarpWarps;
  for (uint32_t l = gw; l < n_leaves; l += nw) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (m <= 1) {
      if (m == 1 && lane == 0 && (src_k != dst_k || ss != 1)) {
        dst_k[lf.lo] = src_k[lf.lo * ss];
        if constexpr (kHasV) dst_v[lf.lo] = src_v[lf.lo * ss];
      }
      continue;
    }
    const uint32_t N = 1u << (32 - __clz(m - 1));   // pow2 >= m
    for (uint32_t i = lane; i < N; i += 32) {
      w.key[i] = i < m ? src_k[(lf.lo + i) * ss] : K(0);
      w.idx[i] = static_cast<uint16_t>(i);
      if constexpr (kHasV) {
        if (i < m) w.val[i] = src_v[(lf.lo + i) * ss];
      }
    }
    __syncwarp();
    bitonic_kv(w.key, w.idx, N, m, lane, 32u, [] { __syncwarp(); });
    for (uint32_t i = lane; i < m; i += 32) {
      dst_k[lf.lo + i] = w.key[i];
      if constexpr (kHasV) dst_v[lf.lo + i] = w.val[w.idx[i]];
    }
    __syncwarp();
  }
}

template <typename K, typename V>
__host__ inline size_t leaf_lt_smem_bytes() {
  return static_cast<size_t>(kLeafSmemMax) * (sizeof(K) + ValTraits<V>::bytes + sizeof(uint16_t)) + 64;
}

template <typename K, typename V>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_lt_smem(const K* __restrict__ src_k, const V* __restrict__ src_v, K* __restrict__ dst_k,
               V* __restrict__ dst_v, const Leaf* __restrict__ leaves, uint32_t n_leaves, uint32_t ss) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  K* key = reinterpret_cast<K*>(smem);
  V* val = reinterpret_cast<V*>(key + kLeafSmemMax);
  uint16_t* idx = reinterpret_cast<uint16_t*>(kHasV ? reinterpret_cast<unsigned char*>(val + kLeafSmemMax)
                                                    : reinterpret_cast<unsigned char*>(val));
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (m <= 1) {
      if (m == 1 && threadIdx.x == 0 && (src_k != dst_k || ss != 1)) {
        dst_k[lf.lo] = src_k[lf.lo * ss];
        if constexpr (kHasV) dst_v[lf.lo] = src_v[lf.lo * ss];
      }
      continue;
    }
    const uint32_t N = 1u << (32 - __clz(m - 1));
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
      key[i] = i < m ? src_k[(lf.lo + i) * ss] : K(0);
      idx[i] = static_cast<uint16_t>(i);
      if constexpr (kHasV) {
        if (i < m) val[i] = src_v[(lf.lo + i) * ss];
      }
    }
    __syncthreads();
    bitonic_kv(key, idx, N, m, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      dst_k[lf.lo + i] = key[i];
      if constexpr (kHasV) dst_v[lf.lo + i] = val[idx[i]];
    }
    __syncthreads();
  }
}

}  // namespace ss
