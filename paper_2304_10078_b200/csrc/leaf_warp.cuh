// Warp-per-leaf semisort= base case for leaves of up to kLeafWarpMax records
// (the common leaf: core.py:404-422 on light buckets < alpha).
//
// Output order (eq_leaf_order in oracle/semisort_oracle.py): groups of equal
// keys ordered by (cell = hash & (cap-1), first index), records of a group in
// input order.  Computed as two stable counting passes, O(m + cap):
//   pass 1  records by (first index, index): dedup table -> first index per
//           record, per-first counts, scan, in-order ranks;
//   pass 2  the pass-1 sequence stably by cell; skipped when every record
//           shares one cell.  That is the usual case: a leaf below the root
//           holds one light bucket of every level above it, so its records
//           share the low b*depth hash bits and cap <= 2^(b*depth).
// The dedup table probes from a multiplicative hash of the folded key hash
// (not the cell), so the shared low bits do not pile every key into one
// probe cluster; probe placement never affects the output order.
#pragma once

#include "common.cuh"
#include "leaf.cuh"
#include "types.cuh"

namespace ss {

__device__ __forceinline__ uint32_t leaf_cap_fast(uint32_t m) {   // smallest pow2 >= 2m (>= 2)
  return m <= 1 ? 2u : 1u << (32 - __clz(2 * m - 1));
}

// Exclusive scan in place of a[0, L), L a multiple of 128, 16-byte aligned.
__device__ __forceinline__ void warp_excl_scan_vec(uint32_t* a, uint32_t L) {
  const uint32_t per4 = L >> 7;   // uint4 chunks per lane: 1, 2 or 4
  uint4* v = reinterpret_cast<uint4*>(a) + lane_id() * per4;
  uint32_t local = 0;
  for (uint32_t q = 0; q < per4; ++q) {
    const uint4 x = v[q];
    local += x.x + x.y + x.z + x.w;
  }
  uint32_t run = warp_incl_scan(local) - local;
  for (uint32_t q = 0; q < per4; ++q) {
    const uint4 x = v[q];
    uint4 y;
    y.x = run; run += x.x;
    y.y = run; run += x.y;
    y.z = run; run += x.z;
    y.w = run; run += x.w;
    v[q] = y;
  }
}

template <typename K, typename V, int ITEMS>
__device__ __forceinline__ void warp_leaf(const K* __restrict__ src_k, const V* __restrict__ src_v,
                                          K* __restrict__ dst_k, V* __restrict__ dst_v, uint64_t lo, uint32_t m,
                                          bool identity, WarpLeafSmem<K>& ws, bool hw, uint32_t ss) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const uint32_t lane = lane_id(), lt = lanemask_lt();
  const uint32_t cap = leaf_cap_fast(m), cmask = cap - 1;
  const uint32_t pshift = 32 - (31 - __clz(cap));   // probe start: top log2(cap) bits
  const uint32_t n_it = (m + 31) >> 5;             // warp-uniform
  K key[ITEMS];
  V val[ITEMS];
  uint32_t cell[ITEMS], aux[ITEMS];                // aux: probe slot -> first index -> position
  uint32_t cmin = 0xFFFFFFFFu, cmax = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t i = lane + 32 * k;
    cell[k] = 0;
    aux[k] = 0;
    if (k < n_it && i < m) {
      key[k] = src_k[(lo + i) * ss];   // ss 2: the leaf lives in the pair scratch layout
      if constexpr (kHasV) val[k] = src_v[(lo + i) * ss];
      ws.keys[i] = key[k];
      const uint64_t h = key_hash(key[k], identity);
      cell[k] = static_cast<uint32_t>(h) & cmask;
      aux[k] = (static_cast<uint32_t>(h ^ (h >> 32)) * 0x9E3779B1u) >> pshift;
      cmin = min(cmin, cell[k]);
      cmax = max(cmax, cell[k]);
    }
  }
  const uint32_t mpad = (m + 127) & ~127u, cpad = cap < 128 ? 128u : cap;
  for (uint32_t s = lane; s < cap; s += 32) ws.T[s] = kEmpty32;
  for (uint32_t f = lane; f < mpad; f += 32) ws.cnt[f] = 0;
  __syncwarp();
  // dedup: lock-free linear probing, the minimum index wins each group
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t i = lane + 32 * k;
    if (k < n_it && i < m) {
      uint32_t s = aux[k];
      while (true) {
        uint32_t t = ws.T[s];
        if (t == kEmpty32) {
          t = atomicCAS(&ws.T[s], kEmpty32, i);
          if (t == kEmpty32) break;
        }
        if (ws.keys[t] == key[k]) {
          if (i < t) atomicMin(&ws.T[s], i);   // T[s] only decreases: skip when already smaller
          break;
        }
        s = (s + 1) & cmask;
      }
      aux[k] = s;
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (k < n_it && lane + 32 * k < m) {
      aux[k] = ws.T[aux[k]];
      atomicAdd(&ws.cnt[aux[k]], 1u);
    }
  }
  const bool one_cell = __reduce_min_sync(0xFFFFFFFFu, cmin) == __reduce_max_sync(0xFFFFFFFFu, cmax);
  __syncwarp();
  warp_excl_scan_vec(ws.cnt, mpad);
  __syncwarp();
  // pass 1: position in (first index, index) order
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (k < n_it) aux[k] = warp_rank_item(lane + 32 * k < m, aux[k], ws.mask, ws.cnt, lane, lt, hw);
  }
  if (!one_cell) {
    // pass 2: stable by cell over the pass-1 sequence
    for (uint32_t s = lane; s < cpad; s += 32) ws.T[s] = 0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      if (k < n_it && lane + 32 * k < m) {
        atomicAdd(&ws.T[cell[k]], 1u);
        ws.arr[aux[k]] = static_cast<uint16_t>(cell[k]);
      }
    }
    __syncwarp();
    warp_excl_scan_vec(ws.T, cpad);
    __syncwarp();
    for (uint32_t j = 0; j < n_it; ++j) {
      const uint32_t p = j * 32 + lane;
      const bool valid = p < m;
      const uint32_t c = valid ? ws.arr[p] : 0u;
      const uint32_t d = warp_rank_item(valid, c, ws.mask, ws.T, lane, lt, hw);
      if (valid) ws.dest[p] = static_cast<uint16_t>(d);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
      if (k < n_it && lane + 32 * k < m) aux[k] = ws.dest[aux[k]];
  }
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    if (k < n_it && lane + 32 * k < m) {
      dst_k[lo + aux[k]] = key[k];
      if constexpr (kHasV) dst_v[lo + aux[k]] = val[k];
    }
  }
  __syncwarp();   // shared arrays reusable by the next leaf
}

template <typename K, typename V>
__global__ void __launch_bounds__(kLeafWarpWarps * 32, 3)
k_leaf_eq_warp(const K* __restrict__ src_k, const V* __restrict__ src_v, K* __restrict__ dst_k,
               V* __restrict__ dst_v, const Leaf* __restrict__ leaves, uint32_t n_leaves, int identity, int hw,
               uint32_t ss = 1) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  WarpLeafSmem<K>& ws = reinterpret_cast<WarpLeafSmem<K>*>(smem)[warp_id()];
  const uint32_t gw = blockIdx.x * kLeafWarpWarps + warp_id(), nw = gridDim.x * kLeafWarpWarps;
  const bool ident = identity != 0;
  for (uint32_t s = lane_id(); s < kLeafWarpCap; s += 32) ws.mask[s] = 0;   // leaders re-zero after use
  __syncwarp();
  for (uint32_t l = gw; l < n_leaves; l += nw) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (m <= 1) {
      if (m == 1 && lane_id() == 0 && src_k != dst_k) {
        dst_k[lf.lo] = src_k[lf.lo * ss];
        if constexpr (kHasV) dst_v[lf.lo] = src_v[lf.lo * ss];
      }
      continue;
    }
    // one instantiation: several inlined variants cost registers (occupancy)
    warp_leaf<K, V, kLeafWarpItems>(src_k, src_v, dst_k, dst_v, lf.lo, m, ident, ws, hw != 0, ss);
  }
}

}  // namespace ss
