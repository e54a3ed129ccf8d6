// collect-reduce / histogram on the GPU (aggregate.py:122-299), level by
// level like the semisort scheduler.
//
// Per level: sample heavy keys; count the matrix while folding heavy values
// into SMEM accumulators (heavy records never move, aggregate.py:156-157);
// scan the light columns; scatter light records only into a compacted child
// buffer (aggregate.py:159-165); light buckets >= alpha become next-level
// nodes, smaller ones are folded in a shared-memory hash table (the
// chained-hash group order of _base_fold, aggregate.py:239-264).  Integer
// sums are order independent (wrapping uint64, aggregate.py:67-79), so the
// result pairs are bit-exact.  Pairs are emitted in a deterministic order:
// by level, heavy pairs by node then leaves by (node, bucket).
#pragma once

#include <type_traits>

#include "engine.cuh"
#include "leaf.cuh"
#include "multisplit.cuh"
#include "sample.cuh"
#include "scan.cuh"
#include "sort_engine.cuh"

namespace ss {

// Fold leaves up to this size keep records and work arrays in shared memory:
// 2048 when the staged record (key, + value for sums) is <= 8 bytes, 1024
// above (two staging buffers per CTA must leave room for >= 2 CTAs per SM).
__host__ __device__ constexpr uint32_t agg_smem_max(int staged_bytes) { return staged_bytes <= 8 ? 2048u : 1024u; }
template <typename K, typename V, bool SUM>
constexpr uint32_t kFoldMax = agg_smem_max(static_cast<int>(sizeof(K)) + (SUM ? ValTraits<V>::bytes : 0));

template <typename V> __device__ __forceinline__ uint64_t val_u64(const V& v) { return static_cast<uint64_t>(v); }
template <> __device__ __forceinline__ uint64_t val_u64<NoVal>(const NoVal&) { return 0; }
template <> __device__ __forceinline__ uint64_t val_u64<V16>(const V16& v) { return v.lo; }

}  // namespace ss

#include "node_fold.cuh"

namespace ss {

// Counting matrix + per-row heavy partial sums.
template <typename K, typename V, bool SUM>
__global__ void __launch_bounds__(kCountThreads)
k_count_agg(const K* __restrict__ src, const V* __restrict__ sv, Work* __restrict__ work, uint32_t n_work,
            const Node* __restrict__ nodes, uint32_t* __restrict__ C, uint32_t stride, KeyBucketsT<KeyStore<K>> bf,
            unsigned long long* __restrict__ HS, uint32_t hs_stride, uint16_t* __restrict__ ids_out,
            uint32_t ss = 1) {   // ss 2: (key, value) pair records
  extern __shared__ __align__(16) uint32_t cnt[];
  __shared__ HeavySmemT<KeyStore<K>> tab;
  // heavy partial sums as native 32-bit atomics: low half, carries out of
  // it, high half (a 64-bit shared atomicAdd is a CAS spin loop on sm_100)
  __shared__ uint32_t hlo[kMaxHeavyDevice], hhi[kMaxHeavyDevice], hcy[kMaxHeavyDevice];
  for (uint32_t wi = blockIdx.x; wi < n_work; wi += gridDim.x) {
    const Work wk = work[wi];
    const Node nd = nodes[wk.node];
    bf.prepare(nd, wk.node, &tab);
    const uint32_t nb = bf.n_buckets();
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
    if (SUM)
      for (uint32_t t = threadIdx.x; t < nd.n_heavy; t += blockDim.x) hlo[t] = hhi[t] = hcy[t] = 0;
    __syncthreads();
    const uint64_t begin = wk.begin;
    const uint32_t len = wk.len;
    const uint32_t nl = bf.n_light;
    uint32_t done = 0;
    // values matter only for heavy records (their partial sums): a node
    // without heavy keys (c3's root) never reads its value column here
    const bool need_v = SUM && nd.n_heavy > 0;
    if constexpr (sizeof(K) == 4 || sizeof(K) == 8) {
      // keys only: 16-byte key loads and packed id stores over the aligned
      // full batches (work items start at multiples of 8 records)
      constexpr uint32_t V = 16 / sizeof(K), NV = kCountItems / V, kBatch = kCountThreads * kCountItems;
      using VT = std::conditional_t<sizeof(K) == 8, ulonglong2, uint4>;
      using IT = std::conditional_t<V == 2, uint32_t, uint2>;
      const K* ws = src + begin;
      uint16_t* wids = ids_out + begin;
      if (!need_v && ss == 1 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0 &&
          (reinterpret_cast<uintptr_t>(wids) & (2 * V - 1)) == 0) {
        done = len - len % kBatch;
        for (uint32_t base = 0; base < done; base += kBatch) {
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
              bb[v] = bf(kk[v], begin + i0 + v);
              atomicAdd(&cnt[bb[v]], 1u);
            }
            IT packed;
            uint32_t* pw = reinterpret_cast<uint32_t*>(&packed);
#pragma unroll
            for (uint32_t v = 0; v < V; v += 2) pw[v / 2] = bb[v] | (bb[v + 1] << 16);
            *reinterpret_cast<IT*>(wids + i0) = packed;
          }
        }
      }
    }
    for (uint32_t base = done; base < len; base += kCountThreads * kCountItems) {
      K keys[kCountItems];
      uint64_t vals[SUM ? kCountItems : 1];
#pragma unroll
      for (int k = 0; k < kCountItems; ++k) {
        uint32_t i = base + k * kCountThreads + threadIdx.x;
        keys[k] = i < len ? ldg_key(src, (begin + i) * ss) : K(0);
        if constexpr (SUM) vals[k] = need_v && i < len ? val_u64(sv[(begin + i) * ss]) : 0ull;
      }
#pragma unroll
      for (int k = 0; k < kCountItems; ++k) {
        uint32_t i = base + k * kCountThreads + threadIdx.x;
        if (i < len) {
          const uint32_t b = bf(keys[k], begin + i);
          atomicAdd(&cnt[b], 1u);   // shared atomics are ~free on sm_100 (see count_add)
          ids_out[begin + i] = static_cast<uint16_t>(b);
          if constexpr (SUM) {
            if (b >= nl) {
              const uint32_t t = b - nl, lo = static_cast<uint32_t>(vals[k]), hi = static_cast<uint32_t>(vals[k] >> 32);
              const uint32_t old = atomicAdd(&hlo[t], lo);
              if (old + lo < old) atomicAdd(&hcy[t], 1u);
              if (hi) atomicAdd(&hhi[t], hi);
            }
          }
        }
      }
    }
    __syncthreads();
    uint32_t* row = C + wk.row * stride;
    __shared__ uint32_t kept;
    if (threadIdx.x == 0) kept = 0;
    __syncthreads();
    uint32_t mine = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
      row[b] = cnt[b];
      if (b < nl) mine += cnt[b];
    }
    if (mine) atomicAdd(&kept, mine);
    __syncthreads();
    // no light record in this row: the light-only distribute skips it (len 0)
    if (threadIdx.x == 0 && kept == 0) work[wi].len = 0;
    if (SUM)
      for (uint32_t t = threadIdx.x; t < nd.n_heavy; t += blockDim.x)   // wrapping u64
        HS[wk.row * hs_stride + t] = (static_cast<unsigned long long>(hhi[t] + hcy[t]) << 32) | hlo[t];
    __syncthreads();
  }
}

// Heavy totals per node: column sums of C (count) or of HS (sum64).
template <typename K, bool SUM>
__global__ void k_heavy_fold(const Node* __restrict__ nodes, uint32_t n_nodes, const uint32_t* __restrict__ C,
                             uint32_t stride, uint32_t n_light, const unsigned long long* __restrict__ HS,
                             uint32_t hs_stride, const KeyStore<K>* __restrict__ heavy, uint32_t mh,
                             K* __restrict__ hk, uint64_t* __restrict__ ha) {
  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const Node nd = nodes[j];
    for (uint32_t t = threadIdx.x; t < nd.n_heavy; t += blockDim.x) {
      uint64_t s = 0;
      for (uint32_t r = 0; r < nd.n_rows; ++r) {
        const uint64_t row = nd.row_base + r;
        s += SUM ? static_cast<uint64_t>(HS[row * hs_stride + t]) : C[row * stride + n_light + t];
      }
      hk[static_cast<uint64_t>(j) * mh + t] = static_cast<K>(heavy[static_cast<uint64_t>(j) * mh + t]);
      ha[static_cast<uint64_t>(j) * mh + t] = s;
    }
  }
}

// Base fold of one leaf: groups in chained-hash order, (cell, first index)
// (aggregate.py:239-264), with count or sum; leaf.cuh's dedup and passes.
// ss: element stride of rk / rv (2 for (key, value) pair records).
template <typename K, typename V, bool SUM>
__device__ void leaf_fold(const K* rk, const V* rv, uint32_t m, bool identity, LeafArrays a, uint32_t* red,
                          K* out_k, uint64_t* out_a, uint32_t* g_out, uint32_t ss = 1) {
  const uint32_t cap = leaf_cap(m);
  if (SUM)
    for (uint32_t f = threadIdx.x; f < m; f += blockDim.x) a.gsum[f] = 0;
  const bool one_cell = leaf_dedup(rk, m, cap, identity, a, true, ss);
  if (SUM)
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
      atomicAdd(&a.gsum[a.pos[i]], static_cast<unsigned long long>(val_u64(rv[i * ss])));
  // rank of each group (first index f) in (cell, f) order -> a.arr[f]
  if (one_cell) {
    for (uint32_t f = threadIdx.x; f < m; f += blockDim.x) a.arr[f] = a.cnt[f] ? 1u : 0u;
    __syncthreads();
    leaf_scan(a.arr, m, red);
  } else {
    for (uint32_t c = threadIdx.x; c < cap; c += blockDim.x) a.T[c] = 0;
    __syncthreads();
    for (uint32_t f = threadIdx.x; f < m; f += blockDim.x) {
      if (!a.cnt[f]) continue;
      const uint32_t c = static_cast<uint32_t>(key_hash(rk[f * ss], identity)) & (cap - 1);
      atomicAdd(&a.T[c], 1u);
      a.arr[f] = c;
    }
    __syncthreads();
    leaf_scan(a.T, cap, red);
    if (warp_id() == 0) warp_walk(a.arr, a.cnt, m, a.mask, a.T, a.arr);
    __syncthreads();
  }
  uint32_t groups = 0;
  for (uint32_t f = threadIdx.x; f < m; f += blockDim.x) {
    const uint32_t c = a.cnt[f];
    if (!c) continue;
    const uint32_t g = a.arr[f];
    out_k[g] = rk[f * ss];
    out_a[g] = SUM ? static_cast<uint64_t>(a.gsum[f]) : c;
    ++groups;
  }
  uint32_t tot;
  block_excl_scan<uint32_t>(groups, red, tot);
  if (threadIdx.x == 0) *g_out = tot;
}

// Staging buffer of one leaf: the 16-byte aligned superset of its keys
// (values), as Bulk16 plans it.
__host__ __device__ constexpr size_t fold_buf_bytes(uint32_t maxm, int elem_bytes) {
  return elem_bytes ? ((static_cast<size_t>(maxm) + 2 * (16 / elem_bytes)) * elem_bytes + 15) & ~size_t(15) : 0;
}

__host__ inline size_t leaf_fold_smem_bytes(int key_bytes, int val_bytes) {
  const uint32_t maxm = agg_smem_max(key_bytes + val_bytes);
  return 2 * (fold_buf_bytes(maxm, key_bytes) + fold_buf_bytes(maxm, val_bytes)) + leaf_words(maxm, true) * 4 + 64;
}

// SMEM folds: the next leaf's keys (and values) stream in by TMA bulk copies
// into the second buffer while this leaf folds (the plain per-leaf load
// left the CTA waiting on memory at 2 CTAs per SM).
template <typename K, typename V, bool SUM>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_fold_smem(const K* __restrict__ src_k, const V* __restrict__ src_v, uint64_t n_src,
                 const Leaf* __restrict__ leaves, uint32_t n_leaves, int identity, K* __restrict__ st_k,
                 uint64_t* __restrict__ st_a, uint32_t* __restrict__ G, uint32_t ss = 1) {
  // ss 2: src_k is an array of (key, value) pair records (K == V, sums)
  constexpr bool kPairsOk = SUM && std::is_same_v<K, V>;
  const bool pairs = kPairsOk && ss == 2;
  constexpr uint32_t kMax = kFoldMax<K, V, SUM>;
  constexpr size_t kBK = fold_buf_bytes(kMax, sizeof(K));
  constexpr size_t kBV = SUM ? fold_buf_bytes(kMax, ValTraits<V>::bytes) : 0;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t red[33];
  __shared__ __align__(8) uint64_t bar[2];
  auto bufK = [&](int b) { return reinterpret_cast<K*>(smem + b * (kBK + kBV)); };
  auto bufV = [&](int b) { return reinterpret_cast<V*>(smem + b * (kBK + kBV) + kBK); };
  uint32_t* work = reinterpret_cast<uint32_t*>(smem + 2 * (kBK + kBV));   // 16-byte aligned
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t l, int b) {   // thread 0: stage leaf l into buffer b
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    if constexpr (kPairsOk) {
      if (pairs) {   // one stream of pairs into the key + value areas
        const Bulk16<Pair2<K>> bp(reinterpret_cast<const Pair2<K>*>(src_k), n_src, lf.lo, m);
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[b], bp.ok ? bp.bytes : 0u);
        if (bp.ok) bulk_g2s(bufK(b), bp.src, bp.bytes, &bar[b]);
        return;
      }
    }
    const Bulk16<K> bk(src_k, n_src, lf.lo, m);
    Bulk16<V> bv(src_v, n_src, lf.lo, m);
    uint32_t bytes = bk.ok ? bk.bytes : 0;
    if (SUM && bv.ok) bytes += bv.bytes;
    fence_proxy_async();
    mbar_arrive_expect_tx(&bar[b], bytes);
    if (bk.ok) bulk_g2s(bufK(b), bk.src, bk.bytes, &bar[b]);
    if (SUM && bv.ok) bulk_g2s(bufV(b), bv.src, bv.bytes, &bar[b]);
  };
  if (threadIdx.x == 0 && blockIdx.x < n_leaves) issue(blockIdx.x, 0);
  uint32_t it = 0;
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x, ++it) {
    const int b = it & 1;
    if (threadIdx.x == 0 && l + gridDim.x < n_leaves) issue(l + gridDim.x, b ^ 1);   // buffer b^1 is free
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    const Bulk16<K> bk(src_k, n_src, lf.lo, m);
    const Bulk16<V> bv(src_v, n_src, lf.lo, m);
    mbar_wait(&bar[b], (it >> 1) & 1);
    const K* rk = bk.ok ? bufK(b) + bk.sh : src_k + lf.lo;   // misfit supersets read global
    const V* rv = (!SUM || bv.ok) ? bufV(b) + bv.sh : src_v + lf.lo;
    if constexpr (kPairsOk) {
      if (pairs) {
        const Bulk16<Pair2<K>> bp(reinterpret_cast<const Pair2<K>*>(src_k), n_src, lf.lo, m);
        rk = bp.ok ? bufK(b) + 2 * bp.sh : src_k + 2 * lf.lo;
        rv = reinterpret_cast<const V*>(rk + 1);
      }
    }
    const uint32_t cap = leaf_cap(m);
    LeafArrays a = leaf_arrays(work, cap, m, true);
    leaf_fold<K, V, SUM>(rk, rv, m, identity != 0, a, red, st_k + lf.lo, st_a + lf.lo, G + l, pairs ? 2u : 1u);
    __syncthreads();
  }
}

template <typename K, typename V, bool SUM>
__global__ void __launch_bounds__(kLeafThreads)
k_leaf_fold_global(const K* __restrict__ src_k, const V* __restrict__ src_v, const Leaf* __restrict__ leaves,
                   uint32_t n_leaves, int identity, K* __restrict__ st_k, uint64_t* __restrict__ st_a,
                   uint32_t* __restrict__ G, uint32_t* __restrict__ scratch, uint64_t words_per_cta,
                   uint32_t ss = 1) {   // ss 2: (key, value) pair records at src_k
  __shared__ uint32_t red[33];
  uint32_t* mine = scratch + static_cast<uint64_t>(blockIdx.x) * words_per_cta;
  for (uint32_t l = blockIdx.x; l < n_leaves; l += gridDim.x) {
    const Leaf lf = leaves[l];
    const uint32_t m = static_cast<uint32_t>(lf.size);
    LeafArrays a = leaf_arrays(mine, leaf_cap(m), m, true);
    const K* rk = src_k + lf.lo * ss;
    const V* rv = ss == 2 ? reinterpret_cast<const V*>(rk + 1) : src_v + lf.lo;
    leaf_fold<K, V, SUM>(rk, rv, m, identity != 0, a, red, st_k + lf.lo, st_a + lf.lo, G + l, ss);
    __syncthreads();
  }
}

template <typename K>
__global__ void k_emit_heavy(const Node* __restrict__ nodes, uint32_t n_nodes, const uint64_t* __restrict__ hoff,
                             const K* __restrict__ hk, const uint64_t* __restrict__ ha, uint32_t mh,
                             K* __restrict__ out_k, uint64_t* __restrict__ out_a, const uint64_t* __restrict__ cursor) {
  const uint64_t c0 = *cursor;
  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const uint64_t base = c0 + hoff[j];
    for (uint32_t t = threadIdx.x; t < nodes[j].n_heavy; t += blockDim.x) {
      out_k[base + t] = hk[static_cast<uint64_t>(j) * mh + t];
      out_a[base + t] = ha[static_cast<uint64_t>(j) * mh + t];
    }
  }
}

template <typename K>
__global__ void k_emit_leaves(const Leaf* __restrict__ leaves, uint32_t n_leaves, const uint32_t* __restrict__ G,
                              const uint64_t* __restrict__ loff, const K* __restrict__ st_k,
                              const uint64_t* __restrict__ st_a, K* __restrict__ out_k, uint64_t* __restrict__ out_a,
                              const uint64_t* __restrict__ cursor) {
  const uint64_t c0 = *cursor;
  // one warp per leaf
  const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t l = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; l < n_leaves; l += warps) {
    const uint64_t base = c0 + loff[l], lo = leaves[l].lo;
    const uint32_t g = G[l];
    for (uint32_t t = lane_id(); t < g; t += 32) {
      out_k[base + t] = st_k[lo + t];
      out_a[base + t] = st_a[lo + t];
    }
  }
}

static __global__ void k_bump(uint64_t* cursor, const uint64_t* add_dev, uint64_t add_host) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *cursor += (add_dev ? *add_dev : 0) + add_host;
}

template <typename K, typename V>
struct AggEngine {
  static constexpr bool kHasV = ValTraits<V>::bytes > 0;
  const K* in_k = nullptr;
  const V* in_v = nullptr;
  uint64_t n = 0;
  int kind = SS_AGG_COUNT;
  int identity = 0;
  Params P{};
  cudaStream_t st = nullptr;
  ss_telemetry* tel = nullptr;

  uint32_t stride = 0, mh = 1, sample_grid = 0, leafg_grid = 0;
  uint64_t max_nodes = 0, max_rows = 0, max_grps = 0, max_leaves = 0, s_cap = 0, leafg_words = 0, max_pairs = 0;
  // workspace; d_out_* first so ss_result_copy can find them with a minimal carve
  K* d_out_k = nullptr;
  uint64_t* d_out_a = nullptr;
  K* B_k[2] = {nullptr, nullptr};
  V* B_v[2] = {nullptr, nullptr};
  K* st_k = nullptr;
  uint64_t* st_a = nullptr;
  Node* d_nodes = nullptr;
  Node* d_next = nullptr;
  KeyStore<K>* d_heavy = nullptr;
  Work* d_work = nullptr;
  uint32_t* d_grp_node = nullptr;
  uint32_t* d_C = nullptr;
  uint64_t* d_X = nullptr;
  uint64_t* d_P = nullptr;
  uint64_t* d_off = nullptr;
  uint32_t* d_ccnt = nullptr;
  uint64_t* d_misc = nullptr;
  Leaf* d_leaf_s = nullptr;
  Leaf* d_leaf_g = nullptr;
  uint64_t* d_samp = nullptr;
  uint32_t* d_leafscr = nullptr;
  unsigned long long* d_HS = nullptr;
  uint64_t* d_ntot = nullptr;
  uint64_t* d_nbase = nullptr;
  uint32_t* d_G = nullptr;
  uint64_t* d_loff = nullptr;
  uint64_t* d_part = nullptr;
  uint16_t* d_ids = nullptr;
  K* d_hk = nullptr;
  uint64_t* d_ha = nullptr;
  uint64_t* d_hoff = nullptr;
  uint64_t* d_cursor = nullptr;
  uint32_t* d_ord = nullptr;
  uint32_t* d_claim = nullptr;
  uint64_t* d_fstat = nullptr;

  void plan(Arena& a) {
    stride = even_stride(P);
    mh = std::max<uint32_t>(P.max_heavy, 1);
    const uint64_t alpha = P.base_case_cutoff;
    max_nodes = std::max<uint64_t>(1, n / alpha);
    max_rows = std::min<uint64_t>(kTargetRows, cdiv(n, kMinChunk)) + max_nodes;   // rows <= R / chunk + nodes
    max_grps = max_rows / kRowGroup + max_nodes + 1;
    max_leaves = std::max<uint64_t>(1, std::min<uint64_t>(n, max_nodes * P.light_buckets));
    s_cap = std::max<uint64_t>(1, std::min<uint64_t>(n, P.sample_count));
    sample_grid = static_cast<uint32_t>(std::min<uint64_t>(kSampleGridMax, max_nodes));
    const uint64_t mmax = std::max<uint64_t>(1, std::min<uint64_t>(n, alpha > 1 ? alpha - 1 : 1));
    leafg_words = leaf_words(mmax, true);
    leafg_grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kLeafGlobalGridMax, cdiv(n, agg_smem_max(16) + 1))));   // kind-independent (the workspace query has no kind)
    max_pairs = std::max<uint64_t>(n, 1);
    d_out_k = a.take<K>(max_pairs);
    d_out_a = a.take<uint64_t>(max_pairs);
    d_cursor = a.take<uint64_t>(1);
    for (int i = 0; i < 2; ++i) {
      if constexpr (std::is_same_v<K, V>) {   // one 2n-word block: SoA halves or pair records (run())
        B_k[i] = a.take<K>(2 * n);
        B_v[i] = reinterpret_cast<V*>(B_k[i] + n);
      } else {
        B_k[i] = a.take<K>(n);
        if (kHasV) B_v[i] = a.take<V>(n);
      }
    }
    st_k = a.take<K>(n);
    st_a = a.take<uint64_t>(n);
    d_nodes = a.take<Node>(max_nodes);
    d_next = a.take<Node>(max_nodes);
    d_heavy = a.take<KeyStore<K>>(max_nodes * mh);
    d_work = a.take<Work>(max_rows);
    d_grp_node = a.take<uint32_t>(max_grps);
    d_C = a.take<uint32_t>(max_rows * stride);
    d_X = a.take<uint64_t>(max_rows * stride);
    d_P = a.take<uint64_t>(max_grps * stride);
    d_off = a.take<uint64_t>(max_nodes * (stride + 1));
    d_ccnt = a.take<uint32_t>(max_nodes * 4);
    d_misc = a.take<uint64_t>(8);
    d_leaf_s = a.take<Leaf>(max_leaves);
    d_leaf_g = a.take<Leaf>(max_leaves);
    d_samp = a.take<uint64_t>(static_cast<uint64_t>(sample_grid) * sample_scratch_words(s_cap, sizeof(KeyStore<K>)));
    d_leafscr = a.take<uint32_t>(static_cast<uint64_t>(leafg_grid) * leafg_words);
    d_HS = a.take<unsigned long long>(max_rows * mh);
    d_ntot = a.take<uint64_t>(max_nodes);
    d_nbase = a.take<uint64_t>(max_nodes);
    d_G = a.take<uint32_t>(max_leaves);
    d_loff = a.take<uint64_t>(max_leaves);
    d_part = a.take<uint64_t>(scan_parts_needed(std::max(max_leaves, max_nodes)) + 8);
    d_hk = a.take<K>(max_nodes * mh);
    d_ha = a.take<uint64_t>(max_nodes * mh);
    d_ids = a.take<uint16_t>(n);
    d_hoff = a.take<uint64_t>(max_nodes);
    d_ord = a.take<uint32_t>(max_nodes);
    d_claim = a.take<uint32_t>(1);
    d_fstat = a.take<uint64_t>(2 * max_nodes);
  }

  bool sum() const { return kind == SS_AGG_SUM64; }
  // SS_NODE_FOLD=0 sends every node through the level path (A/B runs, tests)
  static bool fold_enabled() {
    const char* e = std::getenv("SS_NODE_FOLD");
    return !(e && e[0] == '0');
  }
  // Pair buffers (K == V, sum64, chosen in run()): B holds (key, value)
  // records, element stride 2 -- the light scatter then writes one 16-byte
  // record instead of two partial-sector stores (c3's level 0 is all light).
  bool pairs = false;
  uint32_t bss() const { return pairs ? 2u : 1u; }
  uint32_t fold_max() const {   // the SMEM fold's leaf bound for this engine's staged record
    return agg_smem_max(static_cast<int>(sizeof(K)) + (sum() ? ValTraits<V>::bytes : 0));
  }

  // fold + emit one device leaf list living in `src`
  void fold_list(Tracker& tr, const K* sk, const V* sv, const Leaf* d_list, uint64_t count, bool smem_ok,
                 uint32_t* scr, uint64_t words, uint32_t grid_cap, uint32_t ss = 1) {
    if (!count) return;
    const uint32_t cnt = static_cast<uint32_t>(count);
    if (smem_ok) {
      const size_t sm = leaf_fold_smem_bytes(sizeof(K), sum() ? ValTraits<V>::bytes : 0);
      auto launch = [&](auto kern) {
        SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        int per_sm = 0;
        SS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLeafThreads, sm));
        const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(count, 148u * std::max(per_sm, 1)));
        kern<<<grid, kLeafThreads, sm, st>>>(sk, sv, n, d_list, cnt, identity, st_k, st_a, d_G, ss);
      };
      if (sum()) launch(k_leaf_fold_smem<K, V, true>);
      else launch(k_leaf_fold_smem<K, V, false>);
      if (tel) tel->leaves_smem += count;
    } else {
      const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(count, grid_cap));
      if (sum())
        k_leaf_fold_global<K, V, true><<<grid, kLeafThreads, 0, st>>>(sk, sv, d_list, cnt, identity, st_k, st_a, d_G,
                                                                     scr, words, ss);
      else
        k_leaf_fold_global<K, V, false><<<grid, kLeafThreads, 0, st>>>(sk, sv, d_list, cnt, identity, st_k, st_a, d_G,
                                                                      scr, words, ss);
      if (tel) tel->leaves_global += count;
    }
    check_launch();
    device_exclusive_scan<uint32_t>(d_G, count, d_loff, d_part, d_misc + 6, st);
    k_emit_leaves<K><<<static_cast<uint32_t>(std::min<uint64_t>(cdiv(count, 8), 148 * 16)), 256, 0, st>>>(
        d_list, cnt, d_G, d_loff, st_k, st_a, d_out_k, d_out_a, d_cursor);
    k_bump<<<1, 32, 0, st>>>(d_cursor, d_misc + 6, 0);
    check_launch();
    tr.launched(6);
  }

  // host-built leaves of any size (root leaf, forced leaves)
  void fold_host(Tracker& tr, const K* sk, const V* sv, const std::vector<Leaf>& leaves, uint32_t ss = 1) {
    const uint64_t mmax = std::max<uint64_t>(1, std::min<uint64_t>(n, P.base_case_cutoff > 1 ? P.base_case_cutoff - 1 : 1));
    for (const Leaf& l : leaves) {
      SS_CUDA(cudaMemcpyAsync(d_leaf_g, &l, sizeof(Leaf), cudaMemcpyHostToDevice, st));
      if (l.size <= fold_max()) {
        fold_list(tr, sk, sv, d_leaf_g, 1, true, nullptr, 0, 1, ss);
      } else if (l.size <= mmax) {
        fold_list(tr, sk, sv, d_leaf_g, 1, false, d_leafscr, leafg_words, 1, ss);
      } else {
        const uint64_t words = leaf_words(l.size, true);
        uint32_t* scr = nullptr;
        SS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scr), words * 4, st));
        fold_list(tr, sk, sv, d_leaf_g, 1, false, scr, words, 1, ss);
        SS_CUDA(cudaFreeAsync(scr, st));
      }
      SS_CUDA(cudaStreamSynchronize(st));   // &l must outlive the copy
    }
  }

  // Node folds (node_fold.cuh): every node of a level below the root whose
  // light children would all be leaves is reduced in one pass; returns the
  // nodes that need the regular level path (children >= alpha, or more
  // distinct keys than the shared-memory table holds).
  std::vector<Node> fold_nodes(Tracker& tr, std::vector<Node>& cur, int lvl) {
    if constexpr (sizeof(K) > 8) return cur;   // 128-bit keys: the level path (no 16-byte fold table)
    else return fold_nodes_impl(tr, cur, lvl);
  }
  std::vector<Node> fold_nodes_impl(Tracker& tr, std::vector<Node>& cur, int lvl) {
    const K* sk = B_k[lvl & 1];
    const V* sv = B_v[lvl & 1];
    std::vector<Node> rest, fold;
    // the table's shared memory (+ ~12 KB static) must fit a CTA: large
    // light_buckets settings keep the level path
    const size_t sm = node_fold_smem(sizeof(K), sum(), P.light_buckets);
    if (sm + 12 * 1024 > 227 * 1024) return cur;
    for (const Node& nd : cur) (nd.size >> 32 ? rest : fold).push_back(nd);
    if (fold.empty()) return rest;
    const uint32_t nn = static_cast<uint32_t>(fold.size());
    std::vector<uint32_t> ord(nn);
    std::vector<Leaf> lv(nn);
    for (uint32_t j = 0; j < nn; ++j) {
      ord[j] = j;
      lv[j] = Leaf{fold[j].lo, fold[j].size};
    }
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return fold[a].size > fold[b].size; });
    SS_CUDA(cudaMemcpyAsync(d_nodes, fold.data(), nn * sizeof(Node), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemcpyAsync(d_ord, ord.data(), nn * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemcpyAsync(d_leaf_g, lv.data(), nn * sizeof(Leaf), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemsetAsync(d_claim, 0, sizeof(uint32_t), st));

    tr.begin(kPhSample);
    SS_CUDA(cudaFuncSetAttribute(k_sample<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSampleSmem)));
    k_sample<K><<<std::min<uint32_t>(sample_grid, nn), kSampleThreads, kSampleSmem, st>>>(
        sk, d_nodes, nn, d_heavy, d_samp, s_cap, P, 0, 0, bss());
    check_launch();
    tr.launched();

    KeyBuckets bf{};
    bf.heavy = d_heavy;
    bf.max_heavy = mh;
    bf.n_light = P.light_buckets;
    bf.light_bits = P.light_bits;
    bf.identity = identity;
    tr.begin(kPhLeaves);
    auto launch = [&](auto kern) {
      SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
      int dev = 0, sms = 148;
      SS_CUDA(cudaGetDevice(&dev));
      SS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      kern<<<std::min<uint32_t>(nn, static_cast<uint32_t>(sms)), kFoldThreads, sm, st>>>(
          sk, sv, bss(), d_nodes, d_ord, nn, d_claim, bf, P.base_case_cutoff, st_k, st_a, d_G, d_fstat);
    };
    if (sum()) launch(k_fold_nodes<K, V, true>);
    else launch(k_fold_nodes<K, V, false>);
    check_launch();
    device_exclusive_scan<uint32_t>(d_G, nn, d_loff, d_part, d_misc + 6, st);
    k_emit_leaves<K><<<static_cast<uint32_t>(std::min<uint64_t>(cdiv(nn, 8), 148 * 16)), 256, 0, st>>>(
        d_leaf_g, nn, d_G, d_loff, st_k, st_a, d_out_k, d_out_a, d_cursor);
    k_bump<<<1, 32, 0, st>>>(d_cursor, d_misc + 6, 0);
    check_launch();
    tr.launched(5);
    tr.end();

    std::vector<uint64_t> fst(2 * static_cast<size_t>(nn));
    SS_CUDA(cudaMemcpyAsync(fst.data(), d_fstat, fst.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaMemcpyAsync(fold.data(), d_nodes, nn * sizeof(Node), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    uint64_t done = 0;
    for (uint32_t j = 0; j < nn; ++j) {
      if (fst[2 * j + 1] >> 32) {
        Node nd = fold[j];
        nd.n_heavy = 0;
        rest.push_back(nd);
        continue;
      }
      ++done;
      if (!tel) continue;
      tel->fold_records += fold[j].size;
      const uint64_t kids = fst[2 * j + 1] & 0xFFFFFFFFull;
      tel->bucket_assignments += fold[j].size;
      if (lvl <= 64)
        tel->matrix_cells_by_level[lvl] += cdiv(fold[j].size, P.subarray_len) * (P.light_buckets + fold[j].n_heavy);
      tel->scratch_moves += fst[2 * j];
      tel->nodes += kids;
      if (kids && static_cast<uint64_t>(lvl + 1) > tel->max_depth) tel->max_depth = lvl + 1;
    }
    if (tel) tel->nodes_folded += done;
    return rest;
  }

  std::vector<Node> level(Tracker& tr, std::vector<Node>& cur, int lvl) {
    if (lvl >= 2 && fold_enabled()) {
      cur = fold_nodes(tr, cur, lvl);
      if (cur.empty()) {
        if (tel) tel->levels += 1;
        return {};
      }
    }
    const K* sk = lvl == 1 ? in_k : B_k[lvl & 1];
    const V* sv = lvl == 1 ? in_v : B_v[lvl & 1];
    K* dk = B_k[(lvl + 1) & 1];
    V* dv = B_v[(lvl + 1) & 1];
    const uint32_t nn = static_cast<uint32_t>(cur.size());
    uint64_t R = 0;
    for (auto& nd : cur) R += nd.size;
    const uint64_t chunk = (std::max<uint64_t>(kMinChunk, cdiv(R, kTargetRows)) + 7) & ~uint64_t(7);   // aligned items
    uint64_t max_nrows = 0;   // rows per scan group: <= 128 groups per node (see SortEngine::level)
    for (auto& nd : cur) max_nrows = std::max<uint64_t>(max_nrows, cdiv(nd.size, chunk));
    const uint32_t rg = static_cast<uint32_t>(std::max<uint64_t>(kRowGroup, cdiv(max_nrows, 128)));
    std::vector<Work> work;
    std::vector<uint32_t> grp_node;
    for (uint32_t j = 0; j < nn; ++j) {
      Node& nd = cur[j];
      nd.row_base = work.size();
      nd.n_rows = static_cast<uint32_t>(cdiv(nd.size, chunk));
      nd.grp_base = static_cast<uint32_t>(grp_node.size());
      nd.n_grps = static_cast<uint32_t>(cdiv(nd.n_rows, rg));
      for (uint32_t r = 0; r < nd.n_rows; ++r) {
        Work w;
        w.begin = nd.lo + r * chunk;
        w.len = static_cast<uint32_t>(std::min<uint64_t>(chunk, nd.size - r * chunk));
        w.node = j;
        w.row = nd.row_base + r;
        work.push_back(w);
      }
      for (uint32_t g = 0; g < nd.n_grps; ++g) grp_node.push_back(j);
    }
    if (work.size() > max_rows || grp_node.size() > max_grps || nn > max_nodes)
      throw Fail(SS_ERR_RESOURCE, "level plan exceeds workspace bounds");
    const uint32_t nwork = static_cast<uint32_t>(work.size());
    const uint32_t ngrp = static_cast<uint32_t>(grp_node.size());
    SS_CUDA(cudaMemcpyAsync(d_nodes, cur.data(), nn * sizeof(Node), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemcpyAsync(d_work, work.data(), nwork * sizeof(Work), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemcpyAsync(d_grp_node, grp_node.data(), ngrp * sizeof(uint32_t), cudaMemcpyHostToDevice, st));

    tr.begin(kPhSample);
    SS_CUDA(cudaFuncSetAttribute(k_sample<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSampleSmem)));
    const uint32_t sss = lvl == 1 ? 1u : bss();   // element stride of the source side
    k_sample<K><<<std::min<uint32_t>(sample_grid, nn), kSampleThreads, kSampleSmem, st>>>(
        sk, d_nodes, nn, d_heavy, d_samp, s_cap, P, 0, 0, sss);
    check_launch();
    tr.launched();

    KeyBucketsT<KeyStore<K>> bf{};
    bf.heavy = d_heavy;
    bf.max_heavy = mh;
    bf.n_light = P.light_buckets;
    bf.light_bits = P.light_bits;
    bf.identity = identity;

    tr.begin(kPhCount);
    if (sum())
      k_count_agg<K, V, true><<<nwork, kCountThreads, stride * 4, st>>>(sk, sv, d_work, nwork, d_nodes, d_C, stride, bf,
                                                                        d_HS, mh, d_ids, sss);
    else
      k_count_agg<K, V, false><<<nwork, kCountThreads, stride * 4, st>>>(sk, sv, d_work, nwork, d_nodes, d_C, stride,
                                                                         bf, d_HS, mh, d_ids, sss);
    check_launch();
    tr.launched();

    tr.begin(kPhScan);
    k_colsum_groups<uint32_t><<<ngrp, 256, 0, st>>>(d_C, d_nodes, d_grp_node, ngrp, d_P, stride, P.light_buckets, 1, 0, rg);
    k_scan_nodes<<<nn, 1024, 0, st>>>(d_nodes, nn, d_P, d_off, stride, P.light_buckets, 1, 0, d_ntot);
    device_exclusive_scan<uint64_t>(d_ntot, nn, d_nbase, d_part, d_misc + 5, st);
    k_write_X<uint32_t, uint64_t><<<ngrp, 256, 0, st>>>(d_C, d_nodes, d_grp_node, ngrp, d_P, d_X, stride,
                                                         P.light_buckets, 1, 0, d_nbase, rg);
    check_launch();
    tr.launched(6);

    tr.begin(kPhDistribute);
    launch_distribute<K, V>(sk, sv, d_ids, dk, dv, d_work, nwork, d_nodes, d_X, stride, P.light_buckets,
                            P.light_buckets, 0, st, n, reinterpret_cast<uint32_t*>(d_misc + 7), 0xFFFFFFFFu,
                            pairs && lvl > 1, pairs);
    tr.launched();

    tr.begin(kPhCopy);
    if (sum())
      k_heavy_fold<K, true><<<nn, 128, 0, st>>>(d_nodes, nn, d_C, stride, P.light_buckets, d_HS, mh, d_heavy, mh, d_hk, d_ha);
    else
      k_heavy_fold<K, false><<<nn, 128, 0, st>>>(d_nodes, nn, d_C, stride, P.light_buckets, d_HS, mh, d_heavy, mh, d_hk,
                                                 d_ha);
    check_launch();
    tr.launched();

    tr.begin(kPhChildren);
    SS_CUDA(cudaMemsetAsync(d_misc, 0, 5 * sizeof(uint64_t), st));
    const LeafClasses lcls{0, fold_max(), P.base_case_cutoff};
    k_children_count<<<nn, 256, 0, st>>>(d_nodes, nn, d_off, stride, P.light_buckets, lcls, d_ccnt);
    k_children_scan<<<1, 1024, 0, st>>>(d_ccnt, nn, d_misc);
    k_children_emit<<<nn, 256, 0, st>>>(d_nodes, nn, d_off, stride, P.light_buckets, lcls, d_ccnt, d_nbase,
                                        rounds_per_hash(P.light_bits), d_leaf_s, d_leaf_s, d_leaf_g, d_next,
                                        d_misc + 4);
    check_launch();
    tr.launched(3);
    tr.end();

    uint64_t misc[8];
    std::vector<uint64_t> ntot(nn);
    SS_CUDA(cudaMemcpyAsync(misc, d_misc, sizeof(misc), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaMemcpyAsync(cur.data(), d_nodes, nn * sizeof(Node), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaMemcpyAsync(ntot.data(), d_ntot, nn * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    const uint64_t n_s = misc[1], n_g = misc[2], n_next = misc[3];
    std::vector<Node> next(n_next);
    if (n_next) {
      SS_CUDA(cudaMemcpyAsync(next.data(), d_next, n_next * sizeof(Node), cudaMemcpyDeviceToHost, st));
      SS_CUDA(cudaStreamSynchronize(st));
    }
    if (tel) {
      for (uint32_t j = 0; j < nn; ++j) {
        tel->bucket_assignments += cur[j].size;
        if (lvl <= 64)
          tel->matrix_cells_by_level[lvl] += cdiv(cur[j].size, P.subarray_len) * (P.light_buckets + cur[j].n_heavy);
        tel->scratch_moves += ntot[j];
      }
      const uint64_t kids = n_s + n_g + n_next;
      tel->nodes += kids;
      if (kids && static_cast<uint64_t>(lvl + 1) > tel->max_depth) tel->max_depth = lvl + 1;
      tel->levels += 1;
    }

    // emit: heavy pairs (by node), then leaves (by node, bucket)
    tr.begin(kPhLeaves);
    std::vector<uint64_t> hoff(nn);
    uint64_t htot = 0;
    for (uint32_t j = 0; j < nn; ++j) {
      hoff[j] = htot;
      htot += cur[j].n_heavy;
    }
    if (htot) {
      SS_CUDA(cudaMemcpyAsync(d_hoff, hoff.data(), nn * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
      k_emit_heavy<K><<<std::min<uint32_t>(nn, 1184), 128, 0, st>>>(d_nodes, nn, d_hoff, d_hk, d_ha, mh, d_out_k, d_out_a,
                                                                   d_cursor);
      k_bump<<<1, 32, 0, st>>>(d_cursor, nullptr, htot);
      check_launch();
      tr.launched(2);
    }
    fold_list(tr, dk, dv, d_leaf_s, n_s, true, nullptr, 0, 1, bss());
    fold_list(tr, dk, dv, d_leaf_g, n_g, false, d_leafscr, leafg_words, leafg_grid, bss());
    std::vector<Node> keep;
    std::vector<Leaf> forced;
    for (const Node& c : next) {
      if (c.stalled >= 2 || lvl + 1 >= kDepthLimit) forced.push_back(Leaf{c.lo, c.size});
      else keep.push_back(c);
    }
    fold_host(tr, dk, dv, forced, bss());
    SS_CUDA(cudaStreamSynchronize(st));   // hoff must outlive its copy
    tr.end();
    return keep;
  }

  uint64_t run(Tracker& tr) {
    if constexpr (std::is_same_v<K, V>) {   // pair buffers when summing through the single-pass kernel
      if (sum() && hw_rank_ok() && dist1_tile<K, V>(stride, n) != 0) {
        pairs = true;
        for (int i = 0; i < 2; ++i) B_v[i] = reinterpret_cast<V*>(B_k[i] + 1);
      }
    }
    SS_CUDA(cudaMemsetAsync(d_cursor, 0, sizeof(uint64_t), st));
    if (tel) {
      tel->nodes += 1;
      tel->max_depth = std::max<uint64_t>(tel->max_depth, 1);
    }
    if (n == 0) return 0;
    if (n < P.base_case_cutoff) {
      fold_host(tr, in_k, in_v, {Leaf{0, n}});
    } else {
      Node root{};
      root.lo = 0;
      root.size = n;
      std::vector<Node> cur{root};
      int lvl = 1;
      while (!cur.empty()) {
        cur = level(tr, cur, lvl);
        ++lvl;
      }
    }
    uint64_t count = 0;
    SS_CUDA(cudaMemcpyAsync(&count, d_cursor, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    return count;
  }
};

}  // namespace ss
