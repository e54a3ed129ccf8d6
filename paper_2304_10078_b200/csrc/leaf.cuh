// Base cases (core.py:388-429; aggregate.py:239-264), one CTA per leaf.
//
// semisort= reproduces the reference's chained-hash order exactly: groups
// (distinct keys) are emitted by (cell = hash & (cap-1), first index), cap
// the smallest power of two >= 2m, records of a group in input order
// (core.py:388-422, pinned by test_core_ops.py:309-335).  Computed as two
// stable counting passes, O(m + cap), no comparison sort:
//   1. dedup: lock-free linear probing from a multiplicative hash of the
//      folded key hash; a group's slot keeps its minimum record index
//      (atomicMin), which every record of the group then reads (fidx);
//   2. pass 1: records per first index -> block scan -> one warp walks the
//      records in index order, ranking peers of equal fidx (stable);
//   3. pass 2 (skipped when all records share one cell -- the usual case
//      below the root, where a leaf is one light bucket of every level above
//      it and so shares the low b*depth hash bits): records per cell ->
//      scan -> one warp walks the pass-1 sequence, ranking peers of equal
//      cell (stable);
//   4. record i goes to its final position.
// The dedup probes do not start at the cell: with every record in one cell
// that would be one cluster of all groups, quadratic in the group count.
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
  uint32_t* T;       // [cap] dedup table (min record index); pass 2: per-cell cursors
  uint32_t* cnt;     // [m]   records per first index -> cursors
  uint32_t* mask;    // [cap] peer masks (cap >= 2m)
  uint32_t* pos;     // [m]   first index -> pass-1 position -> final position
  uint32_t* arr;     // [m]   pass 2: cell at each pass-1 position -> final position
  unsigned long long* gsum;  // [m] (aggregation only) sum per first index
};

__host__ __device__ inline uint32_t leaf_cap(uint64_t m) {   // smallest pow2 >= 2m (>= 2)
#ifdef __CUDA_ARCH__
  return m <= 1 ? 2u : static_cast<uint32_t>(1ull << (64 - __clzll(2 * m - 1)));
#else
  uint64_t c = 2;
  while (c < 2 * m) c <<= 1;
  return static_cast<uint32_t>(c);
#endif
}

__host__ __device__ inline uint64_t leaf_words(uint64_t m, bool agg) {
  const uint64_t cap = leaf_cap(m);
  return (2 * cap + 3 * m + (agg ? 2 * m + 2 : 0) + 16 + 3) & ~uint64_t(3);   // 16-byte multiple: per-CTA slices stay aligned
}

__device__ __forceinline__ LeafArrays leaf_arrays(uint32_t* base, uint32_t cap, uint32_t m, bool agg) {
  LeafArrays a;
  uint32_t* p = base;
  a.mask = p; p += cap;   // cap is even: the u64 sums below stay 8-byte aligned
  if (agg) {
    a.gsum = reinterpret_cast<unsigned long long*>(p);
    p += 2 * m + 2;
  } else {
    a.gsum = nullptr;
  }
  a.T = p; p += cap;
  a.cnt = p; p += m;
  a.pos = p; p += m;
  a.arr = p;
  return a;
}

// Probe start of the dedup table: top log2(cap) bits of a multiplicative
// hash of the folded key hash (independent of the cell bits).
__device__ __forceinline__ uint32_t leaf_probe(uint64_t h, uint32_t cap) {
  return (static_cast<uint32_t>(h ^ (h >> 32)) * 0x9E3779B1u) >> (32 - (31 - __clz(cap)));
}

// Stable in-order ranks of one 32-wide item: `key` < mask capacity; `cur`
// holds each key's cursor and advances by the item's count.
__device__ __forceinline__ uint32_t warp_rank_item(bool valid, uint32_t key, uint32_t* mask, uint32_t* cur,
                                                   uint32_t lane, uint32_t lt, bool hw = false) {
  if (hw) {   // lane-ordered atomicAdd returns (probe.cuh): the cursor is the rank
    const uint32_t r = valid ? atomicAdd(&cur[key], 1u) : 0u;
    __syncwarp();
    return r;
  }
  if (valid) atomicOr(&mask[key], 1u << lane);
  __syncwarp();
  const uint32_t peers = valid ? mask[key] : 0u;
  const uint32_t base = valid ? cur[key] : 0u;
  __syncwarp();
  if (valid && lane == 31u - __clz(peers)) {
    cur[key] = base + __popc(peers);
    mask[key] = 0;
  }
  __syncwarp();
  return base + __popc(peers & lt);
}

// One warp: out[p] = stable rank of key_of[p] (p in [0, L), in order) at the
// cursors cur; invalid positions (valid_of[p] == 0 when given) are skipped.
// out may alias key_of.
__device__ __forceinline__ void warp_walk(const uint32_t* key_of, const uint32_t* valid_of, uint32_t L,
                                          uint32_t* mask, uint32_t* cur, uint32_t* out, bool hw = false) {
  const uint32_t lane = lane_id(), lt = lanemask_lt();
  for (uint32_t base = 0; base < L; base += 32) {
    const uint32_t p = base + lane;
    const bool valid = p < L && (valid_of == nullptr || valid_of[p] != 0);
    const uint32_t k = valid ? key_of[p] : 0u;
    const uint32_t r = warp_rank_item(valid, k, mask, cur, lane, lt, hw);
    if (valid) out[p] = r;
  }
}

// Exclusive scan of a[0, L) in place (contiguous chunk per thread).
__device__ inline void leaf_scan(uint32_t* a, uint32_t L, uint32_t* red) {
  const uint32_t per = (L + blockDim.x - 1) >> (31 - __clz(blockDim.x));   // blockDim is a power of two
  const uint32_t c0 = min(L, threadIdx.x * per), c1 = min(L, c0 + per);
  uint32_t local = 0;
  for (uint32_t c = c0; c < c1; ++c) local += a[c];
  uint32_t tot;
  uint32_t run = block_excl_scan<uint32_t>(local, red, tot);
  for (uint32_t c = c0; c < c1; ++c) {
    const uint32_t v = a[c];
    a[c] = run;
    run += v;
  }
  __syncthreads();
}

// Step 1 + record counts per first index: a.pos[i] = first index of record
// i's group, a.cnt[f] = size of the group whose first index is f (0 when f
// is not a first index).  Returns whether every record shares one cell.
// ks: element stride of rk (2 when the records are (key, value) pairs).
template <typename K>
__device__ bool leaf_dedup(const K* rk, uint32_t m, uint32_t cap, bool identity, LeafArrays a, bool count = true,
                           uint32_t ks = 1, uint32_t* groups = nullptr) {   // groups: distinct keys (shared)
  __shared__ uint32_t s_cmin, s_cmax, s_groups;
  const uint32_t cmask = cap - 1;
  for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
    a.T[s] = kEmpty32;
    a.mask[s] = 0;
  }
  for (uint32_t f = threadIdx.x; f < m; f += blockDim.x) a.cnt[f] = 0;
  if (threadIdx.x == 0) {
    s_cmin = 0xFFFFFFFFu;
    s_cmax = 0;
    s_groups = 0;
  }
  __syncthreads();
  uint32_t cmin = 0xFFFFFFFFu, cmax = 0, mine = 0;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const K k = rk[i * ks];
    const uint64_t h = key_hash(k, identity);
    const uint32_t c = static_cast<uint32_t>(h) & cmask;
    cmin = min(cmin, c);
    cmax = max(cmax, c);
    uint32_t s = leaf_probe(h, cap);
    while (true) {
      uint32_t t = a.T[s];
      if (t == kEmpty32) {
        t = atomicCAS(&a.T[s], kEmpty32, i);
        if (t == kEmpty32) {
          ++mine;
          break;
        }
      }
      if (rk[t * ks] == k) {
        if (i < t) atomicMin(&a.T[s], i);   // T[s] only decreases: skip when already smaller
        break;
      }
      s = (s + 1) & cmask;
    }
    a.pos[i] = s;
  }
  cmin = __reduce_min_sync(0xFFFFFFFFu, cmin);
  cmax = __reduce_max_sync(0xFFFFFFFFu, cmax);
  mine = __reduce_add_sync(0xFFFFFFFFu, mine);
  if (lane_id() == 0) {
    atomicMin(&s_cmin, cmin);
    atomicMax(&s_cmax, cmax);
    atomicAdd(&s_groups, mine);
  }
  __syncthreads();
  if (groups) *groups = s_groups;
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t f = a.T[a.pos[i]];
    a.pos[i] = f;
    if (count) atomicAdd(&a.cnt[f], 1u);
  }
  __syncthreads();
  return s_cmin == s_cmax;
}

// Full semisort= leaf: records rk/rv (leaf-relative) -> ok/ov.
template <typename K, typename V>
__device__ void leaf_eq(const K* rk, const V* rv, K* ok, V* ov, uint32_t m, bool identity,
                        LeafArrays a, uint32_t* red, bool hw = false) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const uint32_t cap = leaf_cap(m);
  uint32_t groups = 0;
  const bool one_cell = leaf_dedup(rk, m, cap, identity, a, true, 1, &groups);
  if (groups == m) {
    // every key distinct (uniform keys): each record is its own group, so
    // pass 1's (first index, index) order is the input order
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) a.pos[i] = i;
  } else if (hw) {
    // Pass 1 with lane-ordered atomics (probe.cuh), walking only records of
    // groups with more than one record: a singleton group's record goes to
    // its group start directly (all-distinct leaves -- uniform keys --
    // skip the serial walk entirely).  Flags in mask[0, m) and arr (the
    // non-hw walk's peer masks are not used), the list of walked records in
    // T (free after the dedup).
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint32_t multi = a.cnt[a.pos[i]] > 1 ? 1u : 0u;
      a.mask[i] = multi;
      a.arr[i] = multi;
    }
    __syncthreads();
    leaf_scan(a.cnt, m, red);   // group starts by first index
    leaf_scan(a.arr, m, red);   // list positions
    const uint32_t L = a.arr[m - 1] + a.mask[m - 1];
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      if (a.mask[i]) a.T[a.arr[i]] = i;
      else a.pos[i] = a.cnt[a.pos[i]];
    }
    __syncthreads();
    if (warp_id() == 0) {
      const uint32_t lane = lane_id();
      for (uint32_t b = 0; b < L; b += 32) {   // in index order: ranks inside each group
        const uint32_t q = b + lane;
        const uint32_t i = q < L ? a.T[q] : 0u;
        const uint32_t f = q < L ? a.pos[i] : 0u;
        const uint32_t r = q < L ? atomicAdd(&a.cnt[f], 1u) : 0u;
        __syncwarp();
        if (q < L) a.pos[i] = r;
      }
    }
  } else {
    leaf_scan(a.cnt, m, red);
    if (warp_id() == 0) warp_walk(a.pos, nullptr, m, a.mask, a.cnt, a.pos);   // pass 1
  }
  __syncthreads();
  if (!one_cell) {   // pass 2
    for (uint32_t c = threadIdx.x; c < cap; c += blockDim.x) a.T[c] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint32_t c = static_cast<uint32_t>(key_hash(rk[i], identity)) & (cap - 1);
      atomicAdd(&a.T[c], 1u);
      a.arr[a.pos[i]] = c;
    }
    __syncthreads();
    leaf_scan(a.T, cap, red);
    if (warp_id() == 0) warp_walk(a.arr, nullptr, m, a.mask, a.T, a.arr, hw);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) a.pos[i] = a.arr[a.pos[i]];
  }
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t p = a.pos[i];
    ok[p] = rk[i];
    if constexpr (kHasV) ov[p] = rv[i];
  }
}

__host__ inline size_t leaf_smem_bytes(int key_bytes, int val_bytes) {
  return static_cast<size_t>(kLeafSmemMax) * (key_bytes + val_bytes) + leaf_words(kLeafSmemMax, false) * 4 + 64;
}

// Leaves up to kLeafSmemMax records, fully in SMEM.  src_* is the side the
// leaves live on, dst_* the caller's array A (same index range).
template <typename K, typename V>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_eq_smem(const K* __restrict__ src_k, const V* __restrict__ src_v, K* __restrict__ dst_k,
               V* __restrict__ dst_v, const Leaf* __restrict__ leaves, uint32_t n_leaves, int identity, int hw,
               uint32_t ss = 1) {   // ss 2: the leaves live in the pair scratch layout
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t red[33];
  K* rk = reinterpret_cast<K*>(smem);
  V* rv = reinterpret_cast<V*>(rk + kLeafSmemMax);
  uint32_t* work = reinterpret_cast<uint32_t*>(kHasV ? reinterpret_cast<unsigned char*>(rv + kLeafSmemMax)
                                                     : reinterpret_cast<unsigned char*>(rv));
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (m == 1) {
      if (threadIdx.x == 0 && src_k != dst_k) {
        dst_k[lf.lo] = src_k[lf.lo * ss];
        if constexpr (kHasV) dst_v[lf.lo] = src_v[lf.lo * ss];
      }
      continue;
    }
    {   // all of the leaf's loads in flight at once (<= 4 records per thread)
      constexpr int kPer = kLeafSmemMax / kLeafThreads;
      K kr[kPer];
      V vr[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const uint32_t i = threadIdx.x + u * kLeafThreads;
        if (i < m) {
          kr[u] = src_k[(lf.lo + i) * ss];
          if constexpr (kHasV) vr[u] = src_v[(lf.lo + i) * ss];
        }
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const uint32_t i = threadIdx.x + u * kLeafThreads;
        if (i < m) {
          rk[i] = kr[u];
          if constexpr (kHasV) rv[i] = vr[u];
        }
      }
    }
    __syncthreads();
    LeafArrays a = leaf_arrays(work, leaf_cap(m), m, false);
    leaf_eq(rk, rv, dst_k + lf.lo, dst_v + lf.lo, m, identity != 0, a, red, hw != 0);
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

// SoA staging of one scratch-side leaf for the CTA kernels below: sk / sv
// receive the leaf's records (leaf-relative).  Without the pair layout the
// staging is S's own range; with it (s_pairs), the leaf's 2m K-words of
// the pair array are viewed as m keys then m values -- a leaf living there
// (!in_a) is first unpacked to its final range in A, which is free, and
// restaged from A like an A-resident leaf.
template <typename K, typename V>
__device__ __forceinline__ void leaf_stage(K* S_k, V* S_v, K* A_k, V* A_v, const Leaf& lf, int in_a, int s_pairs,
                                           K*& sk, V*& sv) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const uint32_t m = static_cast<uint32_t>(lf.size);
  if (s_pairs) {
    K* base = S_k + 2 * lf.lo;
    sk = base;
    sv = reinterpret_cast<V*>(base + m);
    if (!in_a) {   // pairs -> A
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const K k = base[2 * i];
        const K v = base[2 * i + 1];
        A_k[lf.lo + i] = k;
        if constexpr (std::is_same_v<K, V>) A_v[lf.lo + i] = v;   // pairs imply K == V
      }
      __syncthreads();
    }
  } else {
    sk = S_k + lf.lo;
    sv = S_v + lf.lo;
    if (!in_a) return;
  }
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {   // A -> staging
    sk[i] = A_k[lf.lo + i];
    if constexpr (kHasV) sv[i] = A_v[lf.lo + i];
  }
  __syncthreads();
}

// Leaves with work arrays in global scratch (any size).  If the leaf lives
// in A (in_a), it is first copied to the free S range, then S -> A.
template <typename K, typename V>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_eq_global(K* __restrict__ S_k, V* __restrict__ S_v, K* __restrict__ A_k, V* __restrict__ A_v,
                 const Leaf* __restrict__ leaves, uint32_t n_leaves, int in_a, int identity,
                 uint32_t* __restrict__ scratch, uint64_t words_per_cta, int hw, int s_pairs = 0) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  __shared__ uint32_t red[33];
  uint32_t* mine = scratch + static_cast<uint64_t>(blockIdx.x) * words_per_cta;
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    K* sk;
    V* sv;
    leaf_stage(S_k, S_v, A_k, A_v, lf, in_a, s_pairs, sk, sv);
    if (m <= 1) {
      if (m == 1 && threadIdx.x == 0) {
        A_k[lf.lo] = sk[0];
        if constexpr (kHasV) A_v[lf.lo] = sv[0];
      }
      __syncthreads();
      continue;
    }
    const uint32_t cap = leaf_cap(m);
    LeafArrays a = leaf_arrays(mine, cap, m, false);
    leaf_eq(sk, sv, A_k + lf.lo, A_v + lf.lo, m, identity != 0, a, red, hw != 0);
    __syncthreads();
  }
}

// Mid-size leaves (kLeafSmemMax, alpha): up to kLeafMidMax<K, V> records
// stage records and work arrays in shared memory (one CTA per SM); larger
// ones keep k_leaf_eq_global's global-scratch path.  The global path costs
// ~10x per record (its probes and counters are L2 round trips): c2's 2053
// mid leaves took 0.42 ms there.
template <typename K, typename V>
constexpr uint32_t kLeafMidMax = sizeof(K) + ValTraits<V>::bytes <= 16 ? 4096u : 2048u;
// When every mid leaf of a launch has <= 2048 records (c5: all of them, c2's
// too), the 2048-record shape holds two CTAs per SM (89 KB each for 16-byte
// records instead of 179 KB).
constexpr uint32_t kLeafMidSmall = 2048;

template <typename K, typename V, uint32_t M = kLeafMidMax<K, V>>
__host__ inline size_t leaf_mid_smem_bytes() {
  return static_cast<size_t>(M) * (sizeof(K) + ValTraits<V>::bytes) + leaf_words(M, false) * 4 + 64;
}

template <typename K, typename V, uint32_t M = kLeafMidMax<K, V>>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_eq_mid(K* __restrict__ S_k, V* __restrict__ S_v, K* __restrict__ A_k, V* __restrict__ A_v,
              const Leaf* __restrict__ leaves, uint32_t n_leaves, int in_a, int identity,
              uint32_t* __restrict__ scratch, uint64_t words_per_cta, int hw, int s_pairs = 0,
              uint64_t size_lo = 0, uint64_t size_hi = ~0ull) {   // leaves outside [size_lo, size_hi]: another launch
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t red[33];
  K* rk = reinterpret_cast<K*>(smem);
  V* rv = reinterpret_cast<V*>(rk + M);
  uint32_t* work = reinterpret_cast<uint32_t*>(kHasV ? reinterpret_cast<unsigned char*>(rv + M)
                                                     : reinterpret_cast<unsigned char*>(rv));
  uint32_t* mine = scratch + static_cast<uint64_t>(blockIdx.x) * words_per_cta;
  // where the leaf lives: A, or S (pair records when s_pairs)
  const K* src_k = in_a ? A_k : S_k;
  const V* src_v = in_a ? A_v : S_v;
  const uint32_t ss = in_a ? 1u : (s_pairs ? 2u : 1u);
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    if (lf.size < size_lo || lf.size > size_hi) continue;
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if (m <= M) {
      if (m <= 1) {
        if (m == 1 && threadIdx.x == 0 && !in_a) {
          A_k[lf.lo] = src_k[lf.lo * ss];
          if constexpr (kHasV) A_v[lf.lo] = src_v[lf.lo * ss];
        }
        __syncthreads();
        continue;
      }
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        rk[i] = src_k[(lf.lo + i) * ss];
        if constexpr (kHasV) rv[i] = src_v[(lf.lo + i) * ss];
      }
      __syncthreads();
      LeafArrays a = leaf_arrays(work, leaf_cap(m), m, false);
      leaf_eq(rk, rv, A_k + lf.lo, A_v + lf.lo, m, identity != 0, a, red, hw != 0);
      __syncthreads();
      continue;
    }
    K* sk;
    V* sv;
    leaf_stage(S_k, S_v, A_k, A_v, lf, in_a, s_pairs, sk, sv);
    LeafArrays a = leaf_arrays(mine, leaf_cap(m), m, false);
    leaf_eq(sk, sv, A_k + lf.lo, A_v + lf.lo, m, identity != 0, a, red, hw != 0);
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
          uint32_t* __restrict__ scratch, uint64_t words_per_cta, int s_pairs = 0) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  uint32_t* mine = scratch + static_cast<uint64_t>(blockIdx.x) * words_per_cta;
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    K* sk;
    V* sv;
    leaf_stage(S_k, S_v, A_k, A_v, lf, in_a, s_pairs, sk, sv);
    uint32_t N = 1;
    while (N < m) N <<= 1;
    K* key = reinterpret_cast<K*>(mine);
    uint32_t* idx = reinterpret_cast<uint32_t*>(key + N);
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
      key[i] = i < m ? sk[i] : K(0);
      idx[i] = i < m ? i : kEmpty32;
    }
    __syncthreads();
    bitonic_key_idx(key, idx, N);
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint32_t src = idx[i];
      A_k[lf.lo + i] = key[i];
      if constexpr (kHasV) A_v[lf.lo + i] = sv[src];
    }
    __syncthreads();
  }
}

}  // namespace ss
