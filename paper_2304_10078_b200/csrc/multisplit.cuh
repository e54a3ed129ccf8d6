// Blocked Distributing on the GPU: counting matrix, column-major scan and the
// stable scatter (core.py:268-380, aggregate.py:172-193), batched over every
// node of a recursion level.
//
// * k_count     one CTA per subarray (work item): bucket ids are recomputed
//               from the key (hash + SMEM heavy table with a home-bit
//               prefilter) and added to SMEM counters with plain shared
//               atomics (cheaper on sm_100 than any warp aggregation, see
//               tools/peers_bench.cu).  One row of C is written.  Reads K
//               bytes / record.
// * scan        three small kernels: partial column sums per row group,
//               per-node bucket-major scan, and the cursor matrix
//               X[row][b] = out_base + (column-major exclusive prefix).
// * k_distribute (dist.cuh) consumes the u16 bucket ids the count pass
//               stores, and scatters each subarray stably through its X row.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "dist.cuh"
#include "tma.cuh"
#include "types.cuh"

namespace ss {

// ---------------------------------------------------------------------------
// bucket functors
// ---------------------------------------------------------------------------

// Semisort / aggregate buckets: heavy table lookup, else the light slice.
// S: heavy-key storage (KeyStore<K>: u64 for u32/u64 keys, U128).
template <typename S = uint64_t>
struct KeyBucketsT {
  const S* heavy;   // [node][max_heavy]
  uint32_t max_heavy;
  uint32_t n_light;
  uint32_t light_bits;
  uint32_t identity;
  // per node, set by prepare()
  HeavySmemT<S>* tab;
  LightCfg lc;
  uint32_t n_heavy;

  __device__ __forceinline__ void prepare(const Node& nd, uint32_t node_idx, HeavySmemT<S>* t) {
    tab = t;
    n_heavy = nd.n_heavy;
    lc = LightCfg::make(nd.depth, light_bits, n_light);
    heavy_build(*tab, heavy + static_cast<uint64_t>(node_idx) * max_heavy, n_heavy, identity != 0);
  }
  __device__ __forceinline__ uint32_t n_buckets() const { return n_light + n_heavy; }
  __device__ __forceinline__ uint32_t first_hot() const { return n_light; }
  template <typename K>
  __device__ __forceinline__ uint32_t operator()(K key, uint64_t) const {
    return bucket_of(key, *tab, n_heavy, lc, identity != 0, n_light);
  }
  // the kernel's own __shared__ table: no generic-to-shared conversions
  template <typename K>
  __device__ __forceinline__ uint32_t operator()(K key, uint64_t, const HeavySmemT<S>& t) const {
    return bucket_of(key, t, n_heavy, lc, identity != 0, n_light);
  }
};
using KeyBuckets = KeyBucketsT<uint64_t>;

// Precomputed ids (the reference's _counts_from_ids / _distribute_ids).
struct IdBuckets {
  const int32_t* ids;      // indexed by absolute source position
  uint32_t nb;
  template <typename T>
  __device__ __forceinline__ void prepare(const Node&, uint32_t, T*) { __syncthreads(); }
  __device__ __forceinline__ uint32_t n_buckets() const { return nb; }
  __device__ __forceinline__ uint32_t first_hot() const { return nb; }
  template <typename K>
  __device__ __forceinline__ uint32_t operator()(K, uint64_t pos) const {
    return static_cast<uint32_t>(ids[pos]);
  }
  template <typename K, typename T>
  __device__ __forceinline__ uint32_t operator()(K k, uint64_t pos, const T&) const {
    return (*this)(k, pos);
  }
};

// ---------------------------------------------------------------------------
// counting matrix
// ---------------------------------------------------------------------------

constexpr int kCountThreads = 256;
constexpr int kCountItems = 8;

// Adds one record per valid lane to cnt[b].  Shared-memory atomicAdd on
// sm_100 costs ~1.3 SM cycles per warp op even when most lanes hit one hot
// (heavy) counter (tools/peers_bench.cu), far below any warp aggregation
// (MATCH.ANY ~53, 7-bit ballot peers ~21), so no aggregation is done.
__device__ __forceinline__ void count_add(uint32_t* cnt, uint32_t b, bool valid, uint32_t, int) {
  if (valid) atomicAdd(&cnt[b], 1u);
}

template <typename K, typename BF>
__global__ void __launch_bounds__(kCountThreads, 6)
k_count(const K* __restrict__ src, const Work* __restrict__ work, uint32_t n_work,
        const Node* __restrict__ nodes, uint32_t* __restrict__ C, uint32_t stride, BF bf,
        uint16_t* __restrict__ ids_out, uint32_t kstride = 1) {   // kstride 2: pair scratch layout
  extern __shared__ __align__(16) uint32_t cnt[];
  __shared__ HeavySmemT<KeyStore<K>> tab;
  for (uint32_t wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
    const Work wk = work[wi];
    const Node nd = nodes[wk.node];
    bf.prepare(nd, wk.node, &tab);
    const uint32_t nb = bf.n_buckets();
    const uint32_t hot = bf.first_hot();
    const int hot_bits = bits_for(nb > hot ? nb - hot : 1);
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
    __syncthreads();
    const uint64_t begin = wk.begin;
    const uint32_t len = wk.len;
    const K* ws = src + begin * kstride;                         // 32-bit offsets below
    uint16_t* wids = ids_out ? ids_out + begin : nullptr;
    constexpr uint32_t kBatch = kCountThreads * kCountItems;
    const uint32_t full = len - len % kBatch;
    auto full_batches = [&](auto write_ids) {   // no bounds checks; id store decided at compile time
      for (uint32_t base = 0; base < full; base += kBatch) {
        K keys[kCountItems];
#pragma unroll
        for (int k = 0; k < kCountItems; ++k) keys[k] = ldg_key(ws, (base + k * kCountThreads + threadIdx.x) * kstride);
#pragma unroll
        for (int k = 0; k < kCountItems; ++k) {
          const uint32_t i = base + k * kCountThreads + threadIdx.x;
          const uint32_t b = bf(keys[k], begin + i, tab);
          atomicAdd(&cnt[b], 1u);
          if constexpr (decltype(write_ids)::value) wids[i] = static_cast<uint16_t>(b);   // consumed by k_distribute
        }
      }
    };
    // 16-byte key loads and packed id stores when the item is aligned (work
    // items start at multiples of 8 records: the root's are, deeper nodes'
    // mostly not); thread t owns records 2048b + V (256 k + t) + [0, V)
    constexpr uint32_t V = (sizeof(K) == 4 || sizeof(K) == 8) ? 16 / sizeof(K) : 1;
    const bool vec = V > 1 && kstride == 1 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(wids) & (2 * V - 1)) == 0;
    auto vec_batches = [&](auto write_ids) {
      if constexpr (V > 1) {
        using VT = std::conditional_t<sizeof(K) == 8, ulonglong2, uint4>;
        using IT = std::conditional_t<V == 2, uint32_t, uint2>;   // V packed u16 ids
        constexpr uint32_t NV = kCountItems / V;
        for (uint32_t base = 0; base < full; base += kBatch) {
          VT kv[NV];
#pragma unroll
          for (uint32_t k = 0; k < NV; ++k)
            kv[k] = __ldg(reinterpret_cast<const VT*>(ws + base) + k * kCountThreads + threadIdx.x);
#pragma unroll
          for (uint32_t k = 0; k < NV; ++k) {
            const K* kk = reinterpret_cast<const K*>(&kv[k]);
            const uint32_t i0 = base + V * (k * kCountThreads + threadIdx.x);
            uint32_t bb[V];
#pragma unroll
            for (uint32_t v = 0; v < V; ++v) {
              bb[v] = bf(kk[v], begin + i0 + v, tab);
              atomicAdd(&cnt[bb[v]], 1u);
            }
            if constexpr (decltype(write_ids)::value) {
              IT packed;
              uint32_t* pw = reinterpret_cast<uint32_t*>(&packed);
#pragma unroll
              for (uint32_t v = 0; v < V; v += 2) pw[v / 2] = bb[v] | (bb[v + 1] << 16);
              *reinterpret_cast<IT*>(wids + i0) = packed;
            }
          }
        }
      }
    };
    if (vec) {
      if (wids) vec_batches(std::true_type{});
      else vec_batches(std::false_type{});
    } else if (wids) {
      full_batches(std::true_type{});
    } else {
      full_batches(std::false_type{});
    }
    for (uint32_t base = full; base < len; base += kBatch) {    // tail
      K keys[kCountItems];
#pragma unroll
      for (int k = 0; k < kCountItems; ++k) {
        uint32_t i = base + k * kCountThreads + threadIdx.x;
        keys[k] = i < len ? ldg_key(ws, i * kstride) : K(0);
      }
#pragma unroll
      for (int k = 0; k < kCountItems; ++k) {
        const uint32_t i = base + k * kCountThreads + threadIdx.x;
        const bool valid = i < len;
        const uint32_t b = valid ? bf(keys[k], begin + i) : 0u;
        count_add(cnt, b, valid, hot, hot_bits);
        if (wids && valid) wids[i] = static_cast<uint16_t>(b);
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
                                int light_only, uint32_t fixed_cols, uint32_t rg = kRowGroup) {
  for (uint32_t g = blockIdx.x; g < n_grps; g += gridDim.x) {
    const Node nd = nodes[grp_node[g]];
    const uint32_t cols = node_cols(nd, n_light, light_only, fixed_cols);
    const uint32_t gi = g - nd.grp_base;
    const uint64_t r0 = nd.row_base + static_cast<uint64_t>(gi) * rg;
    const uint64_t r1 = min(r0 + rg, nd.row_base + nd.n_rows);
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
    constexpr uint32_t kG = 8;   // group loads in flight per thread (the loop is latency-bound)
    for (uint32_t b = b0; b < b1; ++b) {
      uint64_t t = 0;
      const uint64_t* p = P + static_cast<uint64_t>(nd.grp_base) * stride + b;
      uint32_t g = 0;
      for (; g + kG <= nd.n_grps; g += kG) {
        uint64_t v[kG];
#pragma unroll
        for (uint32_t u = 0; u < kG; ++u) v[u] = p[static_cast<uint64_t>(g + u) * stride];
#pragma unroll
        for (uint32_t u = 0; u < kG; ++u) t += v[u];
      }
      for (; g < nd.n_grps; ++g) t += p[static_cast<uint64_t>(g) * stride];
      local += t;
    }
    uint64_t total;
    uint64_t run = block_excl_scan<uint64_t>(local, red, total);
    uint64_t* o = off + static_cast<uint64_t>(j) * (stride + 1);
    for (uint32_t b = b0; b < b1; ++b) {
      o[b] = run;
      uint64_t* p = P + static_cast<uint64_t>(nd.grp_base) * stride + b;
      uint32_t g = 0;
      for (; g + kG <= nd.n_grps; g += kG) {
        uint64_t v[kG];
#pragma unroll
        for (uint32_t u = 0; u < kG; ++u) v[u] = p[static_cast<uint64_t>(g + u) * stride];
#pragma unroll
        for (uint32_t u = 0; u < kG; ++u) {
          p[static_cast<uint64_t>(g + u) * stride] = run;
          run += v[u];
        }
      }
      for (; g < nd.n_grps; ++g) {
        const uint64_t v = p[static_cast<uint64_t>(g) * stride];
        p[static_cast<uint64_t>(g) * stride] = run;
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
                          const uint64_t* __restrict__ node_base, uint32_t rg = kRowGroup) {
  for (uint32_t g = blockIdx.x; g < n_grps; g += gridDim.x) {
    const uint32_t j = grp_node[g];
    const Node nd = nodes[j];
    const uint64_t base = node_base ? node_base[j] : nd.out_base;
    const uint32_t cols = node_cols(nd, n_light, light_only, fixed_cols);
    const uint32_t gi = g - nd.grp_base;
    const uint64_t r0 = nd.row_base + static_cast<uint64_t>(gi) * rg;
    const uint64_t r1 = min(r0 + rg, nd.row_base + nd.n_rows);
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
// heavy copy-back S -> A (core.py:478-482), vectorised when aligned
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ void copy_span(T* __restrict__ dst, const T* __restrict__ src, uint64_t lo, uint64_t hi,
                                          uint64_t tid, uint64_t nthreads) {
  if (hi <= lo) return;
  // 16-byte vectors when src and dst share alignment
  const uintptr_t a = reinterpret_cast<uintptr_t>(src + lo), b = reinterpret_cast<uintptr_t>(dst + lo);
  if (sizeof(T) < 16 && ((a ^ b) & 15) == 0) {
    constexpr uint64_t per = 16 / sizeof(T);
    uint64_t head = ((16 - (a & 15)) & 15) / sizeof(T);
    if (head > hi - lo) head = hi - lo;
    for (uint64_t i = lo + tid; i < lo + head; i += nthreads) dst[i] = src[i];
    const uint64_t v0 = lo + head, nv = (hi - v0) / per;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + v0);
    uint4* d4 = reinterpret_cast<uint4*>(dst + v0);
    uint64_t i = tid;
    for (; i + 3 * nthreads < nv; i += 4 * nthreads) {   // 4 loads in flight per thread
      const uint4 x0 = __ldcs(s4 + i), x1 = __ldcs(s4 + i + nthreads), x2 = __ldcs(s4 + i + 2 * nthreads),
                  x3 = __ldcs(s4 + i + 3 * nthreads);
      __stcs(d4 + i, x0);
      __stcs(d4 + i + nthreads, x1);
      __stcs(d4 + i + 2 * nthreads, x2);
      __stcs(d4 + i + 3 * nthreads, x3);
    }
    for (; i < nv; i += nthreads) d4[i] = s4[i];
    for (uint64_t i = v0 + nv * per + tid; i < hi; i += nthreads) dst[i] = src[i];
  } else if (sizeof(T) == 4 || sizeof(T) == 8) {
    // misaligned by a multiple of 4 bytes: aligned 16-byte stores, each fed
    // by two aligned 16-byte loads funnel-shifted by r words
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(src + lo);
    uint32_t* dw = reinterpret_cast<uint32_t*>(dst + lo);
    const uint64_t words = (hi - lo) * (sizeof(T) / 4);
    uint64_t head = ((16 - (b & 15)) & 15) / 4;
    if (head > words) head = words;
    for (uint64_t i = tid; i < head; i += nthreads) dw[i] = sw[i];
    const uint64_t nv = (words - head) / 4;
    uint4* d4 = reinterpret_cast<uint4*>(dw + head);
    const uint32_t* s0 = sw + head;                      // source word of d4[0].x
    const uint32_t r = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(s0) & 15) / 4);   // 1..3
    const uint4* s4 = reinterpret_cast<const uint4*>(s0 - r);
    auto pick = [r](const uint4& x, const uint4& y) {
      const uint32_t w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
      return r == 1 ? make_uint4(w[1], w[2], w[3], w[4]) : r == 2 ? make_uint4(w[2], w[3], w[4], w[5])
                                                                  : make_uint4(w[3], w[4], w[5], w[6]);
    };
    uint64_t i = tid;
    for (; i + 3 * nthreads < nv; i += 4 * nthreads) {
      uint4 o[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = pick(__ldcs(s4 + i + u * nthreads), __ldcs(s4 + i + u * nthreads + 1));
#pragma unroll
      for (int u = 0; u < 4; ++u) __stcs(d4 + i + u * nthreads, o[u]);
    }
    for (; i < nv; i += nthreads) d4[i] = pick(__ldcs(s4 + i), __ldcs(s4 + i + 1));
    for (uint64_t k = head + nv * 4 + tid; k < words; k += nthreads) dw[k] = sw[k];
  } else {
    for (uint64_t i = lo + tid; i < hi; i += nthreads) dst[i] = src[i];
  }
}

template <typename K, typename V>
__global__ void k_copy_heavy(const K* __restrict__ sk, const V* __restrict__ sv, K* __restrict__ dk,
                             V* __restrict__ dv, const Node* __restrict__ nodes, uint32_t n_nodes,
                             const uint64_t* __restrict__ off, uint32_t stride, uint32_t n_light) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint32_t j = blockIdx.y; j < n_nodes; j += gridDim.y) {
    const Node nd = nodes[j];
    const uint64_t h0 = nd.lo + off[static_cast<uint64_t>(j) * (stride + 1) + n_light];
    const uint64_t h1 = nd.lo + nd.size;
    copy_span(dk, sk, h0, h1, tid, nth);
    if constexpr (kHasV) copy_span(dv, sv, h0, h1, tid, nth);
  }
}

// Heavy copy-back with key fill (semisort=): a heavy bucket holds a single
// key, so the distribute skipped its keys (key_below) and only the values
// move S -> A; the keys are filled from the node's heavy table.  off[j] are
// node-relative bucket offsets ([n_light + t] = start of heavy bucket t,
// [n_light + n_heavy] = node size); heavy[j * mh + t] its key.
constexpr uint64_t kFillChunk = 1 << 16;

template <typename K>
__device__ __forceinline__ void fill_span(K* __restrict__ dst, uint64_t lo, uint64_t hi, K key) {
  if (hi <= lo) return;
  constexpr uint64_t per = 16 / sizeof(K);
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst + lo);
  uint64_t head = ((16 - (a & 15)) & 15) / sizeof(K);
  if (head > hi - lo) head = hi - lo;
  for (uint64_t i = lo + threadIdx.x; i < lo + head; i += blockDim.x) dst[i] = key;
  const uint64_t v0 = lo + head, nv = (hi - v0) / per;
  uint4 pat;
  K* pk = reinterpret_cast<K*>(&pat);
#pragma unroll
  for (uint64_t q = 0; q < per; ++q) pk[q] = key;
  uint4* d4 = reinterpret_cast<uint4*>(dst + v0);
  for (uint64_t i = threadIdx.x; i < nv; i += blockDim.x) __stcs(d4 + i, pat);
  for (uint64_t i = v0 + nv * per + threadIdx.x; i < hi; i += blockDim.x) dst[i] = key;
}

template <typename K, typename V>
__global__ void k_copy_heavy_fill(K* __restrict__ dk, const V* __restrict__ sv, V* __restrict__ dv,
                                  const Node* __restrict__ nodes, uint32_t n_nodes, const uint64_t* __restrict__ off,
                                  uint32_t stride, uint32_t n_light, const KeyStore<K>* __restrict__ heavy, uint32_t mh,
                                  int pairs = 0) {   // pairs: S is the pair layout (heavy values at words h0 + p)
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  __shared__ uint32_t s_t0;
  for (uint32_t j = blockIdx.y; j < n_nodes; j += gridDim.y) {
    const Node nd = nodes[j];
    const uint64_t* o = off + static_cast<uint64_t>(j) * (stride + 1) + n_light;   // o[t]: heavy bucket t
    const uint64_t h0 = o[0], h1 = nd.size;
    if (kHasV) {
      const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
      const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
      // pair layout: heavy value of position p at K-word h0abs + p (dist1.cuh)
      const V* src = pairs ? reinterpret_cast<const V*>(reinterpret_cast<const K*>(sv) + nd.lo + h0) : sv;
      copy_span(dv, src, nd.lo + h0, nd.lo + h1, tid, nth);
    }
    for (uint64_t c0 = h0 + blockIdx.x * kFillChunk; c0 < h1; c0 += gridDim.x * kFillChunk) {
      const uint64_t c1 = min(h1, c0 + kFillChunk);
      if (threadIdx.x == 0) {   // last bucket starting at or before c0
        uint32_t lo = 0, hi = nd.n_heavy;   // o[lo] <= c0 < o[hi]
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (o[mid] <= c0) lo = mid;
          else hi = mid;
        }
        s_t0 = lo;
      }
      __syncthreads();
      for (uint32_t t = s_t0; t < nd.n_heavy && o[t] < c1; ++t) {
        const uint64_t b0 = max(c0, o[t]), b1 = min(c1, o[t + 1]);
        fill_span(dk, nd.lo + b0, nd.lo + b1, static_cast<K>(heavy[static_cast<uint64_t>(j) * mh + t]));
      }
      __syncthreads();
    }
  }
}

template <typename K, typename V>
__global__ void k_copy_range(const K* __restrict__ sk, const V* __restrict__ sv, K* __restrict__ dk,
                             V* __restrict__ dv, uint64_t lo, uint64_t hi) {
  constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nth = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  copy_span(dk, sk, lo, hi, tid, nth);
  if constexpr (kHasV) copy_span(dv, sv, lo, hi, tid, nth);
}

// ---------------------------------------------------------------------------
// children: leaves and next-level nodes (core.py:484-498, aggregate.py:166-170)
// ---------------------------------------------------------------------------

// Leaf size classes: 1 warp leaves (<= t1), 2 SMEM CTA leaves (<= t2),
// 3 global-scratch CTA leaves (< alpha); 4 = child node (>= alpha).
struct LeafClasses {
  uint64_t t1, t2, alpha;
  __device__ __forceinline__ int of(uint64_t sz) const {
    if (sz == 0) return 0;
    if (sz >= alpha) return 4;
    if (sz <= t1) return 1;
    return sz <= t2 ? 2 : 3;
  }
};

static __global__ void k_children_count(const Node* __restrict__ nodes, uint32_t n_nodes,
                                        const uint64_t* __restrict__ off, uint32_t stride, uint32_t n_light,
                                        LeafClasses lc, uint32_t* __restrict__ counts) {
  __shared__ uint32_t red[33];
  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const uint64_t* o = off + static_cast<uint64_t>(j) * (stride + 1);
    uint32_t c[4] = {0, 0, 0, 0};
    for (uint32_t b = threadIdx.x; b < n_light; b += blockDim.x) {
      int k = lc.of(o[b + 1] - o[b]);
      if (k) c[k - 1] += 1;
    }
    for (int k = 0; k < 4; ++k) {
      uint32_t t;
      block_excl_scan<uint32_t>(c[k], red, t);
      if (threadIdx.x == 0) counts[4 * j + k] = t;
    }
  }
}

// Exclusive scan of the 4 count columns over nodes (single CTA); totals in tot[0..3].
static __global__ void __launch_bounds__(1024)
k_children_scan(uint32_t* __restrict__ counts, uint32_t n_nodes, uint64_t* __restrict__ tot) {
  __shared__ uint32_t red[33];
  for (int c = 0; c < 4; ++c) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n_nodes; base += blockDim.x) {
      uint32_t j = base + threadIdx.x;
      uint32_t v = j < n_nodes ? counts[4 * j + c] : 0;
      uint32_t t;
      uint32_t ex = block_excl_scan<uint32_t>(v, red, t);
      if (j < n_nodes) counts[4 * j + c] = carry + ex;
      carry += t;
    }
    if (threadIdx.x == 0) tot[c] = carry;
  }
}

// Emit, in (node, bucket) order, the three leaf lists and the child nodes.
// Child depth / stall bookkeeping follows core.py:452-460 (applied to the
// child here instead of on entry, which is equivalent).
static __global__ void k_children_emit(const Node* __restrict__ nodes, uint32_t n_nodes,
                                       const uint64_t* __restrict__ off, uint32_t stride, uint32_t n_light,
                                       LeafClasses lc, const uint32_t* __restrict__ counts,
                                       const uint64_t* __restrict__ child_base, uint32_t rounds,
                                       Leaf* __restrict__ leaf1, Leaf* __restrict__ leaf2, Leaf* __restrict__ leaf3,
                                       Node* __restrict__ next, uint64_t* __restrict__ max_leaf) {
  __shared__ uint32_t red[33];
  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const Node nd = nodes[j];
    const uint64_t* o = off + static_cast<uint64_t>(j) * (stride + 1);
    const uint64_t base = child_base ? child_base[j] : nd.lo;
    uint32_t a[4];
    for (int k = 0; k < 4; ++k) a[k] = counts[4 * j + k];
    uint64_t mx = 0;
    for (uint32_t bb = 0; bb < n_light; bb += blockDim.x) {
      const uint32_t b = bb + threadIdx.x;
      int c = 0;
      uint64_t lo = 0, sz = 0;
      if (b < n_light) {
        lo = o[b];
        sz = o[b + 1] - lo;
        c = lc.of(sz);
      }
      uint32_t ex[4], t[4];
      for (int k = 0; k < 4; ++k) ex[k] = block_excl_scan<uint32_t>(c == k + 1, red, t[k]);
      if (c == 1) leaf1[a[0] + ex[0]] = Leaf{base + lo, sz};
      if (c == 2) leaf2[a[1] + ex[1]] = Leaf{base + lo, sz};
      if (c == 3) { leaf3[a[2] + ex[2]] = Leaf{base + lo, sz}; mx = sz > mx ? sz : mx; }
      if (c == 4) {
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
        next[a[3] + ex[3]] = ch;
      }
      for (int k = 0; k < 4; ++k) a[k] += t[k];
    }
    if (mx) atomicMax(reinterpret_cast<unsigned long long*>(max_leaf), static_cast<unsigned long long>(mx));
  }
}

}  // namespace ss
