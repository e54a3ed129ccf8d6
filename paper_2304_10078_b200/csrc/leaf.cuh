// Base cases (core.py:388-429; aggregate.py:239-264), one CTA per leaf.
//
// semisort= reproduces the reference's chained-hash order exactly: groups
// (distinct keys) are emitted by (hash & (cap-1), first index), cap the
// smallest power of two >= 2m, records of a group in input order
// (core.py:388-422, pinned by test_core_ops.py:309-335).  We never sort:
//   1. open-addressing table with home slot = the chained-hash cell; a
//      group's entry holds its minimum record index (atomicMin);
//   2. one warp walks the records in index order: match_any on the group
//      slot gives each record its rank inside its group (stable);
//   3. records per cell -> block scan -> cell starts;
//   4. a group's start = its cell start + the sizes of the groups with the
//      same home cell and a smaller first index (found in the probe run
//      from the home cell, which linear probing keeps contiguous);
//   5. record i goes to gstart[slot(i)] + rank(i).
// Work arrays live in SMEM for leaves up to kLeafSmemMax records and in a
// per-CTA global scratch (L2-resident) above that.
#pragma once

#include "common.cuh"
#include "types.cuh"

namespace ss {

constexpr int kLeafThreads = 256;
constexpr uint32_t kLeafSmemMax = 1024;             // records per SMEM leaf
constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;

struct LeafArrays {
  uint32_t* T;       // [cap] min record index of the slot's group
  uint32_t* home;    // [cap] home cell of the slot's group
  uint32_t* gcnt;    // [cap] group size (after the rank pass)
  uint32_t* cell;    // [cap] records per cell -> cell start
  uint32_t* gstart;  // [cap] group start
  uint32_t* rslot;   // [m]
  uint32_t* rank;    // [m]
  unsigned long long* gsum;  // [cap] (aggregation only)
};

__host__ __device__ inline uint32_t leaf_cap(uint64_t m) {
  uint64_t c = 2;
  while (c < 2 * m) c <<= 1;
  return static_cast<uint32_t>(c);
}

__host__ __device__ inline uint64_t leaf_words(uint64_t m, bool agg) {
  uint64_t cap = leaf_cap(m);
  return 5 * cap + 2 * m + (agg ? 2 * cap : 0) + 8;
}

__device__ __forceinline__ LeafArrays leaf_arrays(uint32_t* base, uint32_t cap, uint32_t m, bool agg) {
  LeafArrays a;
  uint32_t* p = base;
  if (agg) {
    a.gsum = reinterpret_cast<unsigned long long*>(p);
    p += 2 * cap;
  } else {
    a.gsum = nullptr;
  }
  a.T = p; p += cap;
  a.home = p; p += cap;
  a.gcnt = p; p += cap;
  a.cell = p; p += cap;
  a.gstart = p; p += cap;
  a.rslot = p; p += m;
  a.rank = p;
  return a;
}

// Steps 1-2: groups, per-record slot and in-group rank, group sizes.
template <typename K>
__device__ void leaf_group(const K* rk, uint32_t m, uint32_t cap, bool identity, LeafArrays a) {
  const uint32_t mask = cap - 1;
  for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
    a.T[s] = kEmpty32;
    a.gcnt[s] = 0;
    a.cell[s] = 0;
    a.gstart[s] = 0;   // peer-mask scratch of the rank pass
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const K k = rk[i];
    const uint32_t c = static_cast<uint32_t>(key_hash(k, identity)) & mask;
    atomicAdd(&a.cell[c], 1u);
    uint32_t s = c;
    while (true) {
      uint32_t t = a.T[s];
      if (t == kEmpty32) {
        uint32_t prev = atomicCAS(&a.T[s], kEmpty32, i);
        if (prev == kEmpty32) { a.home[s] = c; break; }
        t = prev;
      }
      if (rk[t] == k) { atomicMin(&a.T[s], i); break; }
      s = (s + 1) & mask;
    }
    a.rslot[i] = s;
  }
  __syncthreads();
  if (warp_id() == 0) {
    // in-order pass: peers of the same group among 32 consecutive records
    // via atomicOr masks in a.gstart (not yet in use)
    const uint32_t lt = lanemask_lt();
    for (uint32_t base = 0; base < m; base += 32) {
      const uint32_t i = base + lane_id();
      const bool valid = i < m;
      const uint32_t s = valid ? a.rslot[i] : 0;
      if (valid) atomicOr(&a.gstart[s], 1u << lane_id());
      __syncwarp();
      uint32_t peers = 0, cnt = 0;
      if (valid) {
        peers = a.gstart[s];
        cnt = a.gcnt[s];
      }
      __syncwarp();
      if (valid) {
        if (lane_id() == 31 - __clz(peers)) {
          a.gcnt[s] = cnt + __popc(peers);
          a.gstart[s] = 0;
        }
        a.rank[i] = cnt + __popc(peers & lt);
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

// Step 3: exclusive scan of cell[0..cap) in place (contiguous per thread).
__device__ inline void leaf_scan_cells(uint32_t* cell, uint32_t cap, uint32_t* red) {
  const uint32_t per = (cap + blockDim.x - 1) / blockDim.x;
  const uint32_t c0 = min(cap, threadIdx.x * per), c1 = min(cap, c0 + per);
  uint32_t local = 0;
  for (uint32_t c = c0; c < c1; ++c) local += cell[c];
  uint32_t tot;
  uint32_t run = block_excl_scan<uint32_t>(local, red, tot);
  for (uint32_t c = c0; c < c1; ++c) {
    uint32_t v = cell[c];
    cell[c] = run;
    run += v;
  }
  __syncthreads();
}

// Step 4: group starts in chained-hash order.  With count_groups, positions
// are in units of groups (the aggregation output order) instead of records.
__device__ inline void leaf_group_starts(uint32_t cap, LeafArrays a, bool count_groups) {
  const uint32_t mask = cap - 1;
  for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
    const uint32_t f = a.T[s];
    if (f == kEmpty32) continue;
    const uint32_t c = a.home[s];
    uint32_t st = a.cell[c];
    for (uint32_t t = c; a.T[t] != kEmpty32; t = (t + 1) & mask) {
      if (t != s && a.home[t] == c && a.T[t] < f) st += count_groups ? 1u : a.gcnt[t];
    }
    a.gstart[s] = st;
  }
  __syncthreads();
}

// Full semisort= leaf: records rk/rv (leaf-relative) -> ok/ov.
template <typename K, typename V>
__device__ void leaf_eq(const K* rk, const V* rv, K* ok, V* ov, uint32_t m, bool identity,
                        LeafArrays a, uint32_t* red) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const uint32_t cap = leaf_cap(m);
  leaf_group(rk, m, cap, identity, a);
  leaf_scan_cells(a.cell, cap, red);
  leaf_group_starts(cap, a, false);
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t pos = a.gstart[a.rslot[i]] + a.rank[i];
    ok[pos] = rk[i];
    if constexpr (kHasV) ov[pos] = rv[i];
  }
}

// Leaves up to kLeafSmemMax records, fully in SMEM.  src_* is the side the
// leaves live on, dst_* the caller's array A (same index range).
template <typename K, typename V>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_eq_smem(const K* __restrict__ src_k, const V* __restrict__ src_v, K* __restrict__ dst_k,
               V* __restrict__ dst_v, const Leaf* __restrict__ leaves, uint32_t n_leaves, int identity) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t red[33];
  constexpr uint32_t kCap = 2 * kLeafSmemMax;
  K* rk = reinterpret_cast<K*>(smem);
  V* rv = reinterpret_cast<V*>(rk + kLeafSmemMax);
  uint32_t* work = reinterpret_cast<uint32_t*>(kHasV ? reinterpret_cast<unsigned char*>(rv + kLeafSmemMax)
                                                     : reinterpret_cast<unsigned char*>(rv));
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (m == 1) {
      if (threadIdx.x == 0 && src_k != dst_k) {
        dst_k[lf.lo] = src_k[lf.lo];
        if constexpr (kHasV) dst_v[lf.lo] = src_v[lf.lo];
      }
      continue;
    }
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      rk[i] = src_k[lf.lo + i];
      if constexpr (kHasV) rv[i] = src_v[lf.lo + i];
    }
    __syncthreads();
    const uint32_t cap = leaf_cap(m);
    LeafArrays a = leaf_arrays(work, cap <= kCap ? cap : kCap, m, false);
    leaf_eq(rk, rv, dst_k + lf.lo, dst_v + lf.lo, m, identity != 0, a, red);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// warp-per-leaf base case (leaves up to kLeafWarpMax records)
// ---------------------------------------------------------------------------
//
// Same chained-hash order as leaf_eq, computed as two stable counting
// passes (leaf_warp.cuh).  Records live in registers (up to 8 per lane,
// index lane + 32k), so in-place leaves need no staging.

constexpr uint32_t kLeafWarpMax = 256;
constexpr uint32_t kLeafWarpCap = 2 * kLeafWarpMax;
constexpr int kLeafWarpItems = kLeafWarpMax / 32;
constexpr int kLeafWarpWarps = 8;

template <typename K>
struct WarpLeafSmem {
  alignas(16) uint32_t T[kLeafWarpCap];      // dedup table (first index); pass 2: per-cell cursors
  alignas(16) uint32_t cnt[kLeafWarpMax];    // records per first index; pass 1: cursors
  alignas(16) uint32_t mask[kLeafWarpCap];   // peer masks (zero between uses)
  alignas(16) K keys[kLeafWarpMax];          // key copies for the dedup compares
  uint16_t arr[kLeafWarpMax];                // pass 2: cell at each pass-1 position
  uint16_t dest[kLeafWarpMax];               // pass 2: final position of each pass-1 position
};

__host__ inline size_t leaf_smem_bytes(int key_bytes, int val_bytes) {
  return static_cast<size_t>(kLeafSmemMax) * (key_bytes + val_bytes) +
         (5 * 2 * kLeafSmemMax + 2 * kLeafSmemMax) * 4 + 64;
}

// Leaves with work arrays in global scratch (any size).  If the leaf lives
// in A (in_a), it is first copied to the free S range, then S -> A.
template <typename K, typename V>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_eq_global(K* __restrict__ S_k, V* __restrict__ S_v, K* __restrict__ A_k, V* __restrict__ A_v,
                 const Leaf* __restrict__ leaves, uint32_t n_leaves, int in_a, int identity,
                 uint32_t* __restrict__ scratch, uint64_t words_per_cta) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  __shared__ uint32_t red[33];
  uint32_t* mine = scratch + static_cast<uint64_t>(blockIdx.x) * words_per_cta;
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (in_a) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        S_k[lf.lo + i] = A_k[lf.lo + i];
        if constexpr (kHasV) S_v[lf.lo + i] = A_v[lf.lo + i];
      }
      __syncthreads();
    }
    if (m <= 1) {
      if (m == 1 && threadIdx.x == 0) {
        A_k[lf.lo] = S_k[lf.lo];
        if constexpr (kHasV) A_v[lf.lo] = S_v[lf.lo];
      }
      __syncthreads();
      continue;
    }
    const uint32_t cap = leaf_cap(m);
    LeafArrays a = leaf_arrays(mine, cap, m, false);
    leaf_eq(S_k + lf.lo, S_v + lf.lo, A_k + lf.lo, A_v + lf.lo, m, identity != 0, a, red);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// semisort< base case: stable sort by key (core.py:425-429)
// ---------------------------------------------------------------------------

// Bitonic sort of (key, index) pairs at generic pointers, N a power of two;
// padding entries carry index 0xFFFFFFFF and sort last.
template <typename K>
__device__ void bitonic_key_idx(K* key, uint32_t* idx, uint32_t N) {
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        uint32_t ixj = i ^ j;
        if (ixj > i) {
          K a = key[i], b = key[ixj];
          uint32_t ia = idx[i], ib = idx[ixj];
          bool a_gt_b = (ia == kEmpty32) ? true : (ib == kEmpty32 ? false : (a > b || (a == b && ia > ib)));
          bool up = (i & k) == 0;
          if (a_gt_b == up) { key[i] = b; key[ixj] = a; idx[i] = ib; idx[ixj] = ia; }
        }
      }
      __syncthreads();
    }
  }
}

// One CTA per leaf; keys/indices in `scratch` (per CTA, 2*pow2(max m) words
// for u64 keys) or SMEM.  Always reads S (leaf copied there first if in A).
template <typename K, typename V>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_lt(K* __restrict__ S_k, V* __restrict__ S_v, K* __restrict__ A_k, V* __restrict__ A_v,
          const Leaf* __restrict__ leaves, uint32_t n_leaves, int in_a,
          uint32_t* __restrict__ scratch, uint64_t words_per_cta) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  uint32_t* mine = scratch + static_cast<uint64_t>(blockIdx.x) * words_per_cta;
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (in_a) {
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        S_k[lf.lo + i] = A_k[lf.lo + i];
        if constexpr (kHasV) S_v[lf.lo + i] = A_v[lf.lo + i];
      }
      __syncthreads();
    }
    uint32_t N = 1;
    while (N < m) N <<= 1;
    K* key = reinterpret_cast<K*>(mine);
    uint32_t* idx = reinterpret_cast<uint32_t*>(key + N);
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
      key[i] = i < m ? S_k[lf.lo + i] : K(0);
      idx[i] = i < m ? i : kEmpty32;
    }
    __syncthreads();
    bitonic_key_idx(key, idx, N);
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint32_t src = idx[i];
      A_k[lf.lo + i] = key[i];
      if constexpr (kHasV) A_v[lf.lo + i] = S_v[lf.lo + src];
    }
    __syncthreads();
  }
}

}  // namespace ss
