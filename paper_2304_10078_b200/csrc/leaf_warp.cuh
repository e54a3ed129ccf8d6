// Warp-per-leaf semisort= base case for leaves of up to kLeafWarpMax records
// (the common leaf: core.py:404-422 on light buckets < alpha).
//
// Same chained-hash order as leaf_eq (groups by (hash & (cap-1), first
// index), records of a group in input order), with every step
// warp-synchronous.  The records of a leaf live in registers (ITEMS per
// lane, record index lane + 32k), so in-place leaves need no staging; the
// per-leaf code is instantiated for ITEMS = 1, 2, 4, 8 so small leaves do not
// iterate empty items.
#pragma once

#include "common.cuh"
#include "leaf.cuh"
#include "types.cuh"

namespace ss {

__device__ __forceinline__ uint32_t leaf_cap_fast(uint32_t m) {   // smallest pow2 >= 2m (>= 2)
  return m <= 1 ? 2u : 1u << (32 - __clz(2 * m - 1));
}

template <typename K, typename V, int ITEMS>
__device__ __forceinline__ void warp_leaf(const K* __restrict__ src_k, const V* __restrict__ src_v,
                                          K* __restrict__ dst_k, V* __restrict__ dst_v, uint64_t lo, uint32_t m,
                                          bool identity, WarpLeafSmem<K>& ws) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const uint32_t lane = lane_id(), lt = lanemask_lt();
  const uint32_t cap = leaf_cap_fast(m), mask = cap - 1;
  K* keys = ws.keys();
  K key[ITEMS];
  V val[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t i = lane + 32 * k;
    if (i < m) {
      key[k] = src_k[lo + i];
      if constexpr (kHasV) val[k] = src_v[lo + i];
      keys[i] = key[k];
    }
  }
  for (uint32_t s = lane; s < cap; s += 32) {
    ws.T[s] = kEmpty32;
    ws.cell[s] = 0;
    ws.gcnt[s] = 0;
  }
  __syncwarp();
  // groups: open addressing from the chained-hash cell, min index per group
  uint32_t slot[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t i = lane + 32 * k;
    slot[k] = 0;
    if (i < m) {
      const uint32_t c = static_cast<uint32_t>(key_hash(key[k], identity)) & mask;
      atomicAdd(&ws.cell[c], 1u);
      uint32_t s = c;
      while (true) {
        uint32_t t = ws.T[s];
        if (t == kEmpty32) {
          const uint32_t prev = atomicCAS(&ws.T[s], kEmpty32, i);
          if (prev == kEmpty32) {
            ws.home[s] = static_cast<uint16_t>(c);
            break;
          }
          t = prev;
        }
        if (keys[t] == key[k]) {
          atomicMin(&ws.T[s], i);
          break;
        }
        s = (s + 1) & mask;
      }
      slot[k] = s;
    }
  }
  __syncwarp();
  // in-order ranks within groups; the dead key copies hold the peer masks
  uint32_t* pmask = ws.masks();
  for (uint32_t s = lane; s < cap; s += 32) pmask[s] = 0;
  __syncwarp();
  uint32_t rank[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const bool valid = lane + 32 * k < m;
    if (valid) atomicOr(&pmask[slot[k]], 1u << lane);
    __syncwarp();
    const uint32_t peers = valid ? pmask[slot[k]] : 0u;
    const uint32_t cnt = valid ? ws.gcnt[slot[k]] : 0u;
    __syncwarp();
    if (valid && lane == 31u - __clz(peers)) {
      ws.gcnt[slot[k]] = static_cast<uint16_t>(cnt + __popc(peers));
      pmask[slot[k]] = 0;
    }
    rank[k] = cnt + __popc(peers & lt);
    __syncwarp();   // mask cleared and count published before the next item
  }
  // exclusive scan of records per cell (cap/32 contiguous cells per lane)
  {
    const uint32_t per = cap >= 32 ? cap / 32 : 1;
    const uint32_t c0 = min(cap, lane * per), c1 = min(cap, c0 + per);
    uint32_t local = 0;
    for (uint32_t c = c0; c < c1; ++c) local += ws.cell[c];
    uint32_t run = warp_incl_scan(local) - local;
    for (uint32_t c = c0; c < c1; ++c) {
      const uint32_t v = ws.cell[c];
      ws.cell[c] = run;
      run += v;
    }
  }
  __syncwarp();
  // group starts in (cell, first index) order
  for (uint32_t s = lane; s < cap; s += 32) {
    const uint32_t f = ws.T[s];
    if (f == kEmpty32) continue;
    const uint32_t c = ws.home[s];
    uint32_t st = ws.cell[c];
    for (uint32_t t = c; t != s; t = (t + 1) & mask)   // groups of cell c before slot s
      if (ws.home[t] == c && ws.T[t] < f) st += ws.gcnt[t];
    for (uint32_t t = (s + 1) & mask; ws.T[t] != kEmpty32; t = (t + 1) & mask)   // and after it
      if (ws.home[t] == c && ws.T[t] < f) st += ws.gcnt[t];
    ws.gstart[s] = static_cast<uint16_t>(st);
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t i = lane + 32 * k;
    if (i < m) {
      const uint32_t pos = ws.gstart[slot[k]] + rank[k];
      dst_k[lo + pos] = key[k];
      if constexpr (kHasV) dst_v[lo + pos] = val[k];
    }
  }
  __syncwarp();
}

template <typename K, typename V>
__global__ void __launch_bounds__(kLeafWarpWarps * 32)
k_leaf_eq_warp(const K* __restrict__ src_k, const V* __restrict__ src_v, K* __restrict__ dst_k,
               V* __restrict__ dst_v, const Leaf* __restrict__ leaves, uint32_t n_leaves, int identity) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  WarpLeafSmem<K>& ws = reinterpret_cast<WarpLeafSmem<K>*>(smem)[warp_id()];
  const uint32_t gw = blockIdx.x * kLeafWarpWarps + warp_id(), nw = gridDim.x * kLeafWarpWarps;
  const bool ident = identity != 0;
  for (uint32_t l = gw; l < n_leaves; l += nw) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (m <= 1) {
      if (m == 1 && lane_id() == 0 && src_k != dst_k) {
        dst_k[lf.lo] = src_k[lf.lo];
        if constexpr (kHasV) dst_v[lf.lo] = src_v[lf.lo];
      }
      continue;
    }
    // one instantiation: several inlined variants cost registers (occupancy)
    warp_leaf<K, V, kLeafWarpItems>(src_k, src_v, dst_k, dst_v, lf.lo, m, ident, ws);
  }
}

}  // namespace ss
