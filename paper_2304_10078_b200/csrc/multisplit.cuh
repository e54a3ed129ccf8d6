// Blocked Distributing on the GPU: counting matrix, column-major scan and the
// stable scatter (core.py:268-380, aggregate.py:172-193), batched over every
// node of a recursion level.
//
// * k_count     one CTA per subarray (work item): bucket ids are recomputed
//               from the key (hash + SMEM heavy table), aggregated per warp
//               with __match_any_sync and added to SMEM counters; one row of
//               C is written.  Reads K bytes / record.
// * scan        three small kernels: partial column sums per row group,
//               per-node bucket-major scan, and the cursor matrix
//               X[row][b] = out_base + (column-major exclusive prefix).
// * k_distribute
//               one CTA per subarray owns its X row as SMEM cursors and walks
//               the subarray in 2048-record tiles.  Each warp ranks its 256
//               records in index order (match_any + per-warp u16 histograms),
//               a per-bucket prefix over warps orders warps, the tile is
//               staged bucket-sorted in SMEM and written out as contiguous
//               runs per bucket.  Stability and race freedom come from the
//               disjoint cursor ranges, never from atomics.
#pragma once

#include "common.cuh"
#include "types.cuh"

namespace ss {

// ---------------------------------------------------------------------------
// bucket functors
// ---------------------------------------------------------------------------

// Semisort / aggregate buckets: heavy table lookup, else the light slice.
struct KeyBuckets {
  const uint64_t* heavy;   // [node][max_heavy]
  uint32_t max_heavy;
  uint32_t n_light;
  uint32_t light_bits;
  uint32_t identity;
  // per node, set by prepare()
  HeavySmem* tab;
  LightCfg lc;
  uint32_t n_heavy;

  static constexpr bool kUsesTable = true;

  __device__ __forceinline__ void prepare(const Node& nd, uint32_t node_idx, HeavySmem* t) {
    tab = t;
    n_heavy = nd.n_heavy;
    lc = LightCfg::make(nd.depth, light_bits, n_light);
    heavy_build(*tab, heavy + static_cast<uint64_t>(node_idx) * max_heavy, n_heavy);
  }
  __device__ __forceinline__ uint32_t n_buckets() const { return n_light + n_heavy; }
  template <typename K>
  __device__ __forceinline__ uint32_t operator()(K key, uint64_t) const {
    return bucket_of(key, *tab, n_heavy, lc, identity != 0, n_light);
  }
};

// Precomputed ids (the reference's _counts_from_ids / _distribute_ids).
struct IdBuckets {
  const int32_t* ids;      // indexed by absolute source position
  uint32_t nb;
  static constexpr bool kUsesTable = false;
  __device__ __forceinline__ void prepare(const Node&, uint32_t, HeavySmem*) {}
  __device__ __forceinline__ uint32_t n_buckets() const { return nb; }
  template <typename K>
  __device__ __forceinline__ uint32_t operator()(K, uint64_t pos) const {
    return static_cast<uint32_t>(ids[pos]);
  }
};

// ---------------------------------------------------------------------------
// counting matrix
// ---------------------------------------------------------------------------

constexpr int kCountThreads = 256;
constexpr int kCountItems = 8;

template <typename K, typename BF>
__global__ void __launch_bounds__(kCountThreads)
k_count(const K* __restrict__ src, const Work* __restrict__ work, uint32_t n_work,
        const Node* __restrict__ nodes, uint32_t* __restrict__ C, uint32_t stride, BF bf) {
  extern __shared__ __align__(16) uint32_t cnt[];
  __shared__ HeavySmem tab;
  for (uint32_t wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
    const Work wk = work[wi];
    const Node nd = nodes[wk.node];
    bf.prepare(nd, wk.node, &tab);
    const uint32_t nb = bf.n_buckets();
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    const uint64_t begin = wk.begin;
    const uint32_t len = wk.len;
    for (uint32_t base = 0; base < len; base += kCountThreads * kCountItems) {
      K keys[kCountItems];
#pragma unroll
      for (int k = 0; k < kCountItems; ++k) {
        uint32_t i = base + k * kCountThreads + threadIdx.x;
        keys[k] = i < len ? ldg_key(src, begin + i) : K(0);
      }
#pragma unroll
      for (int k = 0; k < kCountItems; ++k) {
        uint32_t i = base + k * kCountThreads + threadIdx.x;
        bool valid = i < len;
        uint32_t act = __ballot_sync(0xffffffffu, valid);
        if (valid) {
          uint32_t b = bf(keys[k], begin + i);
          uint32_t peers = __match_any_sync(act, b);
          if (lane_id() == __ffs(peers) - 1) atomicAdd(&cnt[b], __popc(peers));
        }
      }
    }
    __syncthreads();
    uint32_t* row = C + wk.row * stride;
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) row[b] = cnt[b];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// column-major exclusive scan (core.py:302-318), batched over nodes
// ---------------------------------------------------------------------------

// Columns of node j: n_light + n_heavy (all buckets) or n_light only.
__device__ __forceinline__ uint32_t node_cols(const Node& nd, uint32_t n_light, int light_only, uint32_t fixed) {
  if (fixed) return fixed;
  return light_only ? n_light : n_light + nd.n_heavy;
}

// P[g][b] = sum of C over the rows of group g.
template <typename CT>
static __global__ void k_colsum_groups(const CT* __restrict__ C, const Node* __restrict__ nodes,
                                const uint32_t* __restrict__ grp_node, uint32_t n_grps,
                                uint64_t* __restrict__ P, uint32_t stride, uint32_t n_light,
                                int light_only, uint32_t fixed_cols) {
  for (uint32_t g = blockIdx.x; g < n_grps; g += gridDim.x) {
    const Node nd = nodes[grp_node[g]];
    const uint32_t cols = node_cols(nd, n_light, light_only, fixed_cols);
    const uint32_t gi = g - nd.grp_base;
    const uint64_t r0 = nd.row_base + static_cast<uint64_t>(gi) * kRowGroup;
    const uint64_t r1 = min(r0 + kRowGroup, nd.row_base + nd.n_rows);
    for (uint32_t b = threadIdx.x; b < cols; b += blockDim.x) {
      uint64_t s = 0;
      for (uint64_t r = r0; r < r1; ++r) s += C[r * stride + b];
      P[static_cast<uint64_t>(g) * stride + b] = s;
    }
  }
}

// Per node: bucket totals, bucket-major exclusive scan, group starts (in P),
// bucket offsets (relative to the node) and the node total.
static __global__ void __launch_bounds__(1024)
k_scan_nodes(const Node* __restrict__ nodes, uint32_t n_nodes, uint64_t* __restrict__ P,
             uint64_t* __restrict__ off, uint32_t stride, uint32_t n_light, int light_only,
             uint32_t fixed_cols, uint64_t* __restrict__ node_total) {
  __shared__ uint64_t red[33];
  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const Node nd = nodes[j];
    const uint32_t cols = node_cols(nd, n_light, light_only, fixed_cols);
    // each thread owns a contiguous run of buckets
    const uint32_t per = (cols + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = min(cols, threadIdx.x * per), b1 = min(cols, b0 + per);
    uint64_t local = 0;
    for (uint32_t b = b0; b < b1; ++b) {
      uint64_t t = 0;
      for (uint32_t g = 0; g < nd.n_grps; ++g) t += P[static_cast<uint64_t>(nd.grp_base + g) * stride + b];
      local += t;
    }
    uint64_t total;
    uint64_t run = block_excl_scan<uint64_t>(local, red, total);
    uint64_t* o = off + static_cast<uint64_t>(j) * (stride + 1);
    for (uint32_t b = b0; b < b1; ++b) {
      o[b] = run;
      for (uint32_t g = 0; g < nd.n_grps; ++g) {
        uint64_t* p = P + static_cast<uint64_t>(nd.grp_base + g) * stride + b;
        uint64_t v = *p;
        *p = run;
        run += v;
      }
    }
    if (threadIdx.x == 0) {
      o[cols] = total;
      if (node_total) node_total[j] = total;
    }
    __syncthreads();
  }
}

// X[r][b] = base(node) + group start + prefix of C inside the group.
// base = node_base[j] if given, else nodes[j].out_base.
template <typename CT, typename XT>
__global__ void k_write_X(const CT* __restrict__ C, const Node* __restrict__ nodes,
                          const uint32_t* __restrict__ grp_node, uint32_t n_grps,
                          const uint64_t* __restrict__ P, XT* __restrict__ X, uint32_t stride,
                          uint32_t n_light, int light_only, uint32_t fixed_cols,
                          const uint64_t* __restrict__ node_base) {
  for (uint32_t g = blockIdx.x; g < n_grps; g += gridDim.x) {
    const uint32_t j = grp_node[g];
    const Node nd = nodes[j];
    const uint64_t base = node_base ? node_base[j] : nd.out_base;
    const uint32_t cols = node_cols(nd, n_light, light_only, fixed_cols);
    const uint32_t gi = g - nd.grp_base;
    const uint64_t r0 = nd.row_base + static_cast<uint64_t>(gi) * kRowGroup;
    const uint64_t r1 = min(r0 + kRowGroup, nd.row_base + nd.n_rows);
    for (uint32_t b = threadIdx.x; b < cols; b += blockDim.x) {
      uint64_t run = base + P[static_cast<uint64_t>(g) * stride + b];
      for (uint64_t r = r0; r < r1; ++r) {
        X[r * stride + b] = static_cast<XT>(run);
        run += C[r * stride + b];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// the stable scatter
// ---------------------------------------------------------------------------

constexpr int kDistThreads = 256;
constexpr int kDistWarps = kDistThreads / 32;
constexpr int kDistItems = 8;
constexpr int kDistTile = kDistThreads * kDistItems;     // 2048 records

// Dynamic SMEM layout (bytes) for a stride.
__host__ __device__ inline size_t dist_smem_bytes(uint32_t stride, int key_bytes, int val_bytes) {
  size_t s2 = (stride + 1) & ~1u;
  return s2 * kDistWarps * 2          // per-warp u16 histograms
         + static_cast<size_t>(stride) * 8   // cursors
         + static_cast<size_t>(stride) * 4   // tile offsets
         + static_cast<size_t>(kDistTile) * (key_bytes + val_bytes + 2) + 64;
}

template <typename K, typename V, typename BF>
__global__ void __launch_bounds__(kDistThreads)
k_distribute(const K* __restrict__ sk, const V* __restrict__ sv, K* __restrict__ dk, V* __restrict__ dv,
             const Work* __restrict__ work, uint32_t n_work, const Node* __restrict__ nodes,
             const uint64_t* __restrict__ X, uint32_t stride, uint32_t keep_below, BF bf) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ HeavySmem tab;
  __shared__ uint32_t red[33];
  const uint32_t s2 = (stride + 1) & ~1u;
  uint64_t* cursor = reinterpret_cast<uint64_t*>(smem);
  K* stage_k = reinterpret_cast<K*>(cursor + stride);
  V* stage_v = reinterpret_cast<V*>(stage_k + kDistTile);
  uint32_t* toff = reinterpret_cast<uint32_t*>(kHasV ? reinterpret_cast<unsigned char*>(stage_v + kDistTile)
                                                     : reinterpret_cast<unsigned char*>(stage_v));
  uint16_t* whist = reinterpret_cast<uint16_t*>(toff + stride);
  uint16_t* sb = whist + s2 * kDistWarps;

  const int w = warp_id(), lane = lane_id();
  const uint32_t lt = lanemask_lt();

  for (uint32_t wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
    const Work wk = work[wi];
    const Node nd = nodes[wk.node];
    bf.prepare(nd, wk.node, &tab);
    uint32_t nb = bf.n_buckets();
    if (nb > keep_below) nb = keep_below;
    // thread-owned contiguous bucket range (for the per-tile scans)
    const uint32_t per = (nb + kDistThreads - 1) / kDistThreads;
    const uint32_t b0 = min(nb, threadIdx.x * per), b1 = min(nb, b0 + per);
    const uint64_t* xrow = X + wk.row * stride;
    for (uint32_t b = threadIdx.x; b < nb; b += kDistThreads) cursor[b] = xrow[b];
    for (uint32_t i = threadIdx.x; i < s2 * kDistWarps / 2; i += kDistThreads)
      reinterpret_cast<uint32_t*>(whist)[i] = 0;
    __syncthreads();

    const uint64_t begin = wk.begin;
    const uint32_t len = wk.len;
    for (uint32_t tb = 0; tb < len; tb += kDistTile) {
      // -- load (warp-striped: warp w owns tile positions [w*256, w*256+256))
      K key[kDistItems];
      V val[kDistItems];
      uint32_t bkt[kDistItems], rk[kDistItems];
#pragma unroll
      for (int k = 0; k < kDistItems; ++k) {
        uint32_t i = tb + w * (32 * kDistItems) + k * 32 + lane;
        bool valid = i < len;
        key[k] = valid ? ldg_key(sk, begin + i) : K(0);
        if constexpr (kHasV) { if (valid) val[k] = sv[begin + i]; }
        bkt[k] = kNoBucket;
        if (valid) {
          uint32_t b = bf(key[k], begin + i);
          if (b < nb) bkt[k] = b;
        }
      }
      // -- per-warp stable ranks
      uint16_t* wh = whist + w * s2;
#pragma unroll
      for (int k = 0; k < kDistItems; ++k) {
        const bool valid = bkt[k] != kNoBucket;
        const uint32_t act = __ballot_sync(0xffffffffu, valid);
        uint32_t peers = 0, base = 0;
        if (valid) {
          peers = __match_any_sync(act, bkt[k]);
          base = wh[bkt[k]];
        }
        __syncwarp();
        if (valid && lane == 31 - __clz(peers)) wh[bkt[k]] = static_cast<uint16_t>(base + __popc(peers));
        rk[k] = base + __popc(peers & lt);
        __syncwarp();
      }
      __syncthreads();
      // -- per-bucket prefix over warps, then bucket-major tile offsets
      uint32_t local = 0;
      for (uint32_t b = b0; b < b1; ++b) {
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < kDistWarps; ++ww) {
          uint32_t t = whist[ww * s2 + b];
          whist[ww * s2 + b] = static_cast<uint16_t>(run);
          run += t;
        }
        toff[b] = run;           // temporarily the bucket's tile count
        local += run;
      }
      uint32_t tile_total;
      uint32_t at = block_excl_scan<uint32_t>(local, red, tile_total);
      for (uint32_t b = b0; b < b1; ++b) {
        uint32_t c = toff[b];
        toff[b] = at;
        at += c;
      }
      __syncthreads();
      // -- stage bucket-sorted
#pragma unroll
      for (int k = 0; k < kDistItems; ++k) {
        if (bkt[k] == kNoBucket) continue;
        uint32_t s = toff[bkt[k]] + whist[w * s2 + bkt[k]] + rk[k];
        stage_k[s] = key[k];
        if constexpr (kHasV) stage_v[s] = val[k];
        sb[s] = static_cast<uint16_t>(bkt[k]);
      }
      __syncthreads();
      // -- write contiguous runs
      for (uint32_t s = threadIdx.x; s < tile_total; s += kDistThreads) {
        const uint32_t b = sb[s];
        const uint64_t d = cursor[b] + (s - toff[b]);
        dk[d] = stage_k[s];
        if constexpr (kHasV) dv[d] = stage_v[s];
      }
      __syncthreads();
      // -- advance cursors, clear histograms
      for (uint32_t b = b0; b < b1; ++b) {
        uint32_t next = (b + 1 < nb) ? toff[b + 1] : tile_total;
        cursor[b] += next - toff[b];
      }
      for (uint32_t i = threadIdx.x; i < s2 * kDistWarps / 2; i += kDistThreads)
        reinterpret_cast<uint32_t*>(whist)[i] = 0;
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// heavy copy-back S -> A (core.py:478-482)
// ---------------------------------------------------------------------------

template <typename K, typename V>
__global__ void k_copy_heavy(const K* __restrict__ sk, const V* __restrict__ sv, K* __restrict__ dk,
                             V* __restrict__ dv, const Node* __restrict__ nodes, uint32_t n_nodes,
                             const uint64_t* __restrict__ off, uint32_t stride, uint32_t n_light) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  for (uint32_t j = blockIdx.y; j < n_nodes; j += gridDim.y) {
    const Node nd = nodes[j];
    const uint64_t h0 = nd.lo + off[static_cast<uint64_t>(j) * (stride + 1) + n_light];
    const uint64_t h1 = nd.lo + nd.size;
    for (uint64_t i = h0 + blockIdx.x * blockDim.x + threadIdx.x; i < h1;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
      dk[i] = sk[i];
      if constexpr (kHasV) dv[i] = sv[i];
    }
  }
}

template <typename K, typename V>
__global__ void k_copy_range(const K* __restrict__ sk, const V* __restrict__ sv, K* __restrict__ dk,
                             V* __restrict__ dv, uint64_t lo, uint64_t hi) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  for (uint64_t i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    dk[i] = sk[i];
    if constexpr (kHasV) dv[i] = sv[i];
  }
}

// ---------------------------------------------------------------------------
// children: leaves and next-level nodes (core.py:484-498, aggregate.py:166-170)
// ---------------------------------------------------------------------------

// Per node: count light buckets by class.  cls: 0 empty, 1 small leaf in
// SMEM range, 2 small leaf (global path), 3 child node.  With
// all_nodes != 0 (aggregation), every non-empty bucket is a node() call;
// small ones are still leaves but classified the same way.
__device__ __forceinline__ int child_class(uint64_t sz, uint64_t alpha, uint64_t smem_max) {
  if (sz == 0) return 0;
  if (sz < alpha) return sz <= smem_max ? 1 : 2;
  return 3;
}

static __global__ void k_children_count(const Node* __restrict__ nodes, uint32_t n_nodes,
                                 const uint64_t* __restrict__ off, uint32_t stride, uint32_t n_light,
                                 uint64_t alpha, uint64_t smem_max, uint32_t* __restrict__ counts) {
  __shared__ uint32_t red[33];
  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const uint64_t* o = off + static_cast<uint64_t>(j) * (stride + 1);
    uint32_t c1 = 0, c2 = 0, c3 = 0;
    for (uint32_t b = threadIdx.x; b < n_light; b += blockDim.x) {
      int c = child_class(o[b + 1] - o[b], alpha, smem_max);
      c1 += c == 1; c2 += c == 2; c3 += c == 3;
    }
    uint32_t t1, t2, t3;
    block_excl_scan<uint32_t>(c1, red, t1);
    block_excl_scan<uint32_t>(c2, red, t2);
    block_excl_scan<uint32_t>(c3, red, t3);
    if (threadIdx.x == 0) {
      counts[3 * j + 0] = t1;
      counts[3 * j + 1] = t2;
      counts[3 * j + 2] = t3;
    }
  }
}

// Exclusive scan of the 3 count columns over nodes (single CTA); totals and
// the max leaf size land in tot[0..3].
static __global__ void __launch_bounds__(1024)
k_children_scan(uint32_t* __restrict__ counts, uint32_t n_nodes, uint64_t* __restrict__ tot) {
  __shared__ uint32_t red[33];
  for (int c = 0; c < 3; ++c) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n_nodes; base += blockDim.x) {
      uint32_t j = base + threadIdx.x;
      uint32_t v = j < n_nodes ? counts[3 * j + c] : 0;
      uint32_t t;
      uint32_t ex = block_excl_scan<uint32_t>(v, red, t);
      if (j < n_nodes) counts[3 * j + c] = carry + ex;
      carry += t;
    }
    if (threadIdx.x == 0) tot[c] = carry;
  }
}

// Emit, in (node, bucket) order: SMEM leaves, global leaves, child nodes.
// Child depth / stall bookkeeping follows core.py:452-460 (applied to the
// child here instead of on entry, which is equivalent).
static __global__ void k_children_emit(const Node* __restrict__ nodes, uint32_t n_nodes,
                                const uint64_t* __restrict__ off, uint32_t stride, uint32_t n_light,
                                uint64_t alpha, uint64_t smem_max, const uint32_t* __restrict__ counts,
                                const uint64_t* __restrict__ child_base, uint32_t rounds,
                                Leaf* __restrict__ leaf_s, Leaf* __restrict__ leaf_g,
                                Node* __restrict__ next, uint64_t* __restrict__ max_leaf) {
  __shared__ uint32_t red[33];
  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const Node nd = nodes[j];
    const uint64_t* o = off + static_cast<uint64_t>(j) * (stride + 1);
    const uint64_t base = child_base ? child_base[j] : nd.lo;
    uint32_t a1 = counts[3 * j + 0], a2 = counts[3 * j + 1], a3 = counts[3 * j + 2];
    uint64_t mx = 0;
    for (uint32_t bb = 0; bb < n_light; bb += blockDim.x) {
      const uint32_t b = bb + threadIdx.x;
      int c = 0;
      uint64_t lo = 0, sz = 0;
      if (b < n_light) {
        lo = o[b];
        sz = o[b + 1] - lo;
        c = child_class(sz, alpha, smem_max);
      }
      uint32_t t1, t2, t3;
      uint32_t e1 = block_excl_scan<uint32_t>(c == 1, red, t1);
      uint32_t e2 = block_excl_scan<uint32_t>(c == 2, red, t2);
      uint32_t e3 = block_excl_scan<uint32_t>(c == 3, red, t3);
      if (c == 1) leaf_s[a1 + e1] = Leaf{base + lo, sz};
      if (c == 2) { leaf_g[a2 + e2] = Leaf{base + lo, sz}; mx = sz > mx ? sz : mx; }
      if (c == 3) {
        Node ch{};
        ch.lo = base + lo;
        ch.size = sz;
        ch.path = mix64_pair(nd.path, static_cast<uint64_t>(b) + 1);
        ch.parent_size = nd.size;
        uint32_t depth = nd.depth + 1, stalled = nd.stalled;
        if (2 * sz > nd.size) {
          stalled += 1;
          if (stalled == 1) depth = (depth / rounds + 1) * rounds;
        }
        ch.depth = depth;
        ch.stalled = stalled;
        next[a3 + e3] = ch;
      }
      a1 += t1; a2 += t2; a3 += t3;
    }
    if (mx) atomicMax(reinterpret_cast<unsigned long long*>(max_leaf), static_cast<unsigned long long>(mx));
  }
}

}  // namespace ss
