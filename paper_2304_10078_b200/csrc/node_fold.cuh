// Node folds for collect-reduce / histogram: a recursion node whose light
// children would all be base-case leaves is reduced in ONE pass over its
// records, in a shared-memory hash table, instead of count -> scan -> light
// distribute -> one base fold per child (aggregate.py:133-170 followed by
// _base_fold :239-264 on every child).
//
// Why this is the same computation: the result of collect_reduce/histogram
// is one (key, aggregate) pair per distinct key, the aggregate being a
// wrapping-u64 sum or a count over ALL of the key's records (aggregate.py:
// 62-79) -- order and grouping independent.  Heavy keys (folded by
// _heavy_fold :205-228) and light keys (folded in their child leaf) end up
// as one pair each either way.  What the recursion shape changes is only the
// Telemetry, and that is reproduced exactly: the node is still sampled with
// its reference Philox stream (n_heavy feeds matrix_cells, and heavy keys do
// not count as light records), and the fold table yields, per distinct key,
// its light bucket (core.py:139-151) and record count, hence every light
// child's size: nodes += non-empty light buckets, scratch_moves += light
// records, max_depth = level + 1.  A node is only folded when every light
// child is < alpha (a child >= alpha would recurse, aggregate.py:139-141)
// and its distinct keys fit the table; otherwise it reports failure and
// takes the regular level path (the table is discarded, nothing was
// written; u32 counting also falls back when a 16-bit count wrapped).
//
// Table (u32 counting, c4: ~9.8K keys per node at load 0.3): buckets of 16
// bytes (4 slots), one shared load each;
// a key's home bucket is a multiplicative fold of the raw key (independent
// of the hash bits the node's ancestors bucketed on); slots fill a bucket
// left to right, the next bucket takes the overflow, the ones after it
// when both are full (fold_probe2).  Per record: one vector load (two when
// the home bucket is full), compares, one shared atomicAdd.  Other key /
// aggregate types (few keys per node, e.g. c3's ~120): single-slot linear
// probing, one 8-byte load per record, + 1-2 atomics for sums.
// The kernel is bound by shared-memory wavefronts (bank conflicts of the
// random bucket loads and counter atomics), not by HBM.
//
// Output order per node (deterministic whatever the insertion races): by
// (home bucket, key) -- a counting sort over home buckets, then a key sort
// inside each (small) home group in the L2-resident staging area.
//
// Algorithmic bytes: one read of the node's records (K [+ V] bytes each)
// plus the pairs; measured bound: shared-memory wavefronts (above).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "multisplit.cuh"
#include "types.cuh"

namespace ss {

constexpr int kFoldThreads = 1024;

template <typename K> struct FoldKey;
template <> struct FoldKey<uint32_t> {
  using T = uint32_t;
  static constexpr uint32_t kEmpty = 0xFFFFFFFFu;
};
template <> struct FoldKey<uint64_t> {
  using T = unsigned long long;
  static constexpr unsigned long long kEmpty = ~0ull;
};

// Table geometry: key + record count (+ sum as low and high words -- 32-bit
// shared atomics, carries out of the low word go to the high word; a 64-bit
// shared atomicAdd is a CAS spin loop on sm_100) + one counter per bucket
// for the emission sort.  u32 counting (c4: ~9.8K keys per node) packs the
// record counts and the bucket counters as 16-bit halves: 32K slots fit
// (load 0.3, overflow past both candidate buckets is rare); a count that
// wraps is caught by the node total (the node then takes the level path).
template <typename K, bool SUM>
struct FoldShape {
  static constexpr bool kC16 = sizeof(K) == 4 && !SUM;
  static constexpr uint32_t kLog2T = kC16 ? 15u : 13u;
  static constexpr uint32_t kT = 1u << kLog2T;
  static constexpr uint32_t kW = 16 / sizeof(K);   // slots per bucket: one 16-byte shared load
  static constexpr uint32_t kLog2B = kLog2T - (sizeof(K) == 4 ? 2u : 1u);
  static constexpr uint32_t kB = kT / kW;
  static constexpr uint32_t kLimit = kT / 4 * 3;   // distinct keys (load 0.75)
  static constexpr uint32_t kPer = kT / kFoldThreads;
  static constexpr size_t kBytes = static_cast<size_t>(kT) * (sizeof(K) + (kC16 ? 2 : SUM ? 12 : 4)) + kB * (kC16 ? 2 : 4);
};

__host__ inline size_t node_fold_smem(int key_bytes, bool sum, uint32_t n_light) {
  const size_t b = key_bytes == 4 ? (sum ? FoldShape<uint32_t, true>::kBytes : FoldShape<uint32_t, false>::kBytes)
                                  : (sum ? FoldShape<uint64_t, true>::kBytes : FoldShape<uint64_t, false>::kBytes);
  return b + static_cast<size_t>(n_light) * 4;
}

// the keys of bucket b (volatile: other threads insert concurrently)
__device__ __forceinline__ void bucket_keys(const volatile uint32_t* tk, uint32_t b, uint32_t (&q)[4]) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(const_cast<uint32_t*>(tk + 4 * b)));
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]) : "r"(a));
}
__device__ __forceinline__ void bucket_keys(const volatile unsigned long long* tk, uint32_t b,
                                            unsigned long long (&q)[2]) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(const_cast<unsigned long long*>(tk + 2 * b)));
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(q[0]), "=l"(q[1]) : "r"(a));
}
// (No "memory" clobber: a stale read can only show a slot as empty that has
// since been filled -- filled slots never change -- and the CAS that claims
// an empty slot returns its current key.)

// Claims (or finds) the slot of key k when the caller's reads of its two
// candidate buckets b1, b2 missed.  Placement rule, whatever the races: b1's
// first empty slot; b2 only when b1 is full; past b2 (next buckets in
// order) only when both are full -- buckets never lose keys, so a lookup
// that finds an empty slot in b1 (or, with b1 full, in b2) knows k is
// absent.  Every CAS result is checked, so a slot another thread filled
// with k is found.  Returns T when the table is full.  Out of line: only
// inserts that lost a race and keys past both buckets come here.
template <typename TK, uint32_t T, uint32_t W>
__device__ __noinline__ uint32_t fold_probe2(volatile TK* tk, TK k, uint32_t b1, uint32_t b2, uint32_t* used,
                                             uint32_t* fail, uint32_t limit) {
  constexpr uint32_t NB = T / W;
  constexpr TK kEmpty = ~TK(0);
  auto in_bucket = [&](uint32_t b, uint32_t& slot) -> bool {   // true: k found or placed in b
    TK q[W];
    bucket_keys(tk, b, q);
    uint32_t e = W;
#pragma unroll
    for (int i = W - 1; i >= 0; --i) {
      if (q[i] == k) {
        slot = W * b + i;
        return true;
      }
      if (q[i] == kEmpty) e = i;
    }
    for (; e < W; ++e) {
      const TK old = atomicCAS(const_cast<TK*>(tk + W * b + e), kEmpty, k);
      if (old == kEmpty) {
        if (atomicAdd(used, 1u) >= limit) *fail = 1;
        slot = W * b + e;
        return true;
      }
      if (old == k) {
        slot = W * b + e;
        return true;
      }
    }
    return false;   // b is full and does not hold k
  };
  uint32_t slot = T;
  if (in_bucket(b1, slot) || in_bucket(b2, slot)) return slot;
  for (uint32_t step = 1, b = b2; step < NB; ++step) {
    b = (b + 1) & (NB - 1);
    if (b != b1 && in_bucket(b, slot)) return slot;
  }
  return T;
}

template <typename K, typename V, bool SUM>
__global__ void __launch_bounds__(kFoldThreads, 1)
k_fold_nodes(const K* __restrict__ src_k, const V* __restrict__ src_v, uint32_t ss, const Node* __restrict__ nodes,
             const uint32_t* __restrict__ order, uint32_t n_nodes, uint32_t* __restrict__ claim, KeyBuckets bf,
             uint64_t alpha, K* __restrict__ st_k, uint64_t* __restrict__ st_a, uint32_t* __restrict__ G,
             uint64_t* __restrict__ stat) {   // stat[2j] = light records, stat[2j+1] = kids | failed << 32
  using FK = FoldKey<K>;
  using TK = typename FK::T;
  using Sh = FoldShape<K, SUM>;
  constexpr uint32_t T = Sh::kT, NB = Sh::kB;
  constexpr TK kEmpty = FK::kEmpty;
  extern __shared__ __align__(16) unsigned char smem[];
  volatile TK* tk = reinterpret_cast<volatile TK*>(smem);
  constexpr bool C16 = Sh::kC16;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + T * sizeof(TK));   // C16: two 16-bit counts per word
  uint32_t* slo = cnt + T;   // SUM only
  uint32_t* shi = slo + T;
  uint32_t* hcnt = SUM ? shi + T : cnt + (C16 ? T / 2 : T);   // per home bucket: keys, bases, cursors
  uint32_t* lcnt = hcnt + (C16 ? NB / 2 : NB);
  // 16-bit-or-32-bit counter access
  auto c_add = [&](uint32_t* a, uint32_t i) {   // returns the old value
    if constexpr (C16) {
      const uint32_t sh = (i & 1u) << 4;
      return (atomicAdd(&a[i >> 1], 1u << sh) >> sh) & 0xFFFFu;
    } else {
      return atomicAdd(&a[i], 1u);
    }
  };
  auto c_red = [&](uint32_t* a, uint32_t i) {   // no return value
    if constexpr (C16) atomicAdd(&a[i >> 1], 1u << ((i & 1u) << 4));
    else atomicAdd(&a[i], 1u);
  };
  auto c_get = [&](const uint32_t* a, uint32_t i) -> uint32_t {
    if constexpr (C16) return (a[i >> 1] >> ((i & 1u) << 4)) & 0xFFFFu;
    else return a[i];
  };
  __shared__ HeavySmem tab;
  __shared__ uint32_t red[33];
  __shared__ uint32_t s_node, s_used, s_fail, s_kids, s_max, s_light;
  __shared__ uint32_t e_cnt, e_lo, e_hi;   // the key equal to the empty marker
  const bool identity = bf.identity != 0;
  const volatile uint32_t* vfail = &s_fail;

  auto home = [](TK k) { return static_cast<uint32_t>((static_cast<uint64_t>(k) * kGamma) >> (64 - Sh::kLog2B)); };
  auto probe_start = [](TK k) {   // first slot of the single-slot probe (!C16)
    const uint32_t x = static_cast<uint32_t>(k) ^ static_cast<uint32_t>(static_cast<uint64_t>(k) >> 32);
    return (x * 0x9E3779B1u) >> (32 - Sh::kLog2T);
  };
  auto add_sum = [&](uint32_t* lo, uint32_t* hi, uint64_t v) {
    const uint32_t l = static_cast<uint32_t>(v), h = static_cast<uint32_t>(v >> 32);
    const uint32_t old = atomicAdd(lo, l);
    const uint32_t up = h + (old + l < old ? 1u : 0u);
    if (up) atomicAdd(hi, up);
  };
  // one record into the table (sets s_fail once the node overflows)
  auto add = [&](K key, uint64_t v) {
    const TK k = static_cast<TK>(key);
    if (k == kEmpty) {
      atomicAdd(&e_cnt, 1u);
      if constexpr (SUM) add_sum(&e_lo, &e_hi, v);
      return;
    }
    if constexpr (!C16) {
      // few distinct keys per node (c3: ~120): single-slot linear probing
      // from a multiplicative hash of the raw key -- one 8-byte shared load
      // per record instead of a 16-byte bucket scan (c3 fold 3.79 -> 3.28
      // ms).  At c4's load 0.3 the probe chains diverged (max over a warp
      // ~3 probes): u32 counting keeps the bucket scan below.
      uint32_t slot = probe_start(k);
      for (uint32_t n = 0;; ++n) {
        TK t = tk[slot];
        if (t == k) break;
        if (t == kEmpty) {
          t = atomicCAS(const_cast<TK*>(tk + slot), kEmpty, k);
          if (t == kEmpty) {
            if (atomicAdd(&s_used, 1u) >= Sh::kLimit) s_fail = 1;
            break;
          }
          if (t == k) break;
        }
        if (n + 1 >= T) {   // table full
          s_fail = 1;
          return;
        }
        slot = (slot + 1) & (T - 1);
      }
      c_red(cnt, slot);
      if constexpr (SUM) add_sum(&slo[slot], &shi[slot], v);
      return;
    }
    // the home bucket, then the next one only when it is full (a second
    // candidate bucket read for every record was measured slower: the
    // fold is bound by shared-memory wavefronts, and at load <= 0.3 / small
    // key counts the overflow it avoids is rare)
    constexpr uint32_t W = Sh::kW;
    const uint32_t b1 = home(k);
    TK q1[W], q2[W];
    bucket_keys(tk, b1, q1);
    {   // fast path: the key is already in its home bucket (~99% of c4's
        // records; an out-of-line slow path with a 16-key unrolled stream
        // loop was measured slower: 2.75 -> 4.33 ms)
      uint32_t hit = 0;
#pragma unroll
      for (int i = 0; i < static_cast<int>(W); ++i) hit |= (q1[i] == k ? 1u : 0u) << i;
      if (hit) {
        c_red(cnt, W * b1 + (__ffs(hit) - 1));
        return;
      }
    }
    const uint32_t b2 = (b1 + 1) & (NB - 1);
    uint32_t slot = T, e1 = W, e2 = W;
#pragma unroll
    for (int i = W - 1; i >= 0; --i) {
      if (q1[i] == k) slot = W * b1 + i;
      if (q1[i] == kEmpty) e1 = i;
    }
    if (slot == T && e1 == W) {   // home bucket full: read the next one
      bucket_keys(tk, b2, q2);
#pragma unroll
      for (int i = W - 1; i >= 0; --i) {
        if (q2[i] == k) slot = W * b2 + i;
        if (q2[i] == kEmpty) e2 = i;
      }
    }
    if (slot == T) {   // absent (or beyond both buckets): one inline claim attempt
      const bool at1 = e1 < W;
      if (at1 || e2 < W) {
        const uint32_t cs = at1 ? W * b1 + e1 : W * b2 + e2;
        const TK old = atomicCAS(const_cast<TK*>(tk + cs), kEmpty, k);
        if (old == kEmpty) {
          slot = cs;
          if (atomicAdd(&s_used, 1u) >= Sh::kLimit) s_fail = 1;
        } else if (old == k) {
          slot = cs;
        }
      }
      if (slot == T) slot = fold_probe2<TK, T, W>(tk, k, b1, b2, &s_used, &s_fail, Sh::kLimit);
    }
    if (slot == T) {   // full: only after the limit was passed
      s_fail = 1;
      return;
    }
    c_red(cnt, slot);
    if constexpr (SUM) add_sum(&slo[slot], &shi[slot], v);
  };

  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t c = atomicAdd(claim, 1u);
      s_node = c < n_nodes ? order[c] : 0xFFFFFFFFu;
      s_used = s_fail = 0;
      s_kids = s_max = 0;
      s_light = 0;
      e_cnt = e_lo = e_hi = 0;
    }
    __syncthreads();
    const uint32_t j = s_node;
    if (j == 0xFFFFFFFFu) break;
    const Node nd = nodes[j];
    bf.prepare(nd, j, &tab);
    for (uint32_t s = threadIdx.x; s < T; s += kFoldThreads) {
      tk[s] = kEmpty;
      if constexpr (SUM) slo[s] = shi[s] = 0;
    }
    for (uint32_t s = threadIdx.x; s < (C16 ? T / 2 : T); s += kFoldThreads) cnt[s] = 0;
    for (uint32_t b = threadIdx.x; b < (C16 ? NB / 2 : NB); b += kFoldThreads) hcnt[b] = 0;
    for (uint32_t b = threadIdx.x; b < bf.n_light; b += kFoldThreads) lcnt[b] = 0;
    __syncthreads();

    // ---- stream the node's records once --------------------------------
    const uint64_t lo = nd.lo, m = nd.size;
    if constexpr (!SUM && std::is_same_v<K, uint32_t>) {
      // keys only, 4 per 16-byte load between a scalar head and tail
      const uint64_t end = lo + m, a4 = (lo + 3) >> 2, b4 = end >> 2;
      const uint64_t h_end = end < (a4 << 2) ? end : (a4 << 2);
      for (uint64_t i = lo + threadIdx.x; i < h_end; i += kFoldThreads) add(__ldg(src_k + i), 0);
      if ((a4 << 2) < end) {
        const uint4* p = reinterpret_cast<const uint4*>(src_k);
        constexpr int U = 4;
        for (uint64_t q = a4; q < b4 && !*vfail; q += static_cast<uint64_t>(kFoldThreads) * U) {
          uint4 w[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint64_t x = q + u * kFoldThreads + threadIdx.x;
            w[u] = x < b4 ? __ldcs(p + x) : make_uint4(0, 0, 0, 0);
          }
          // rolled over the loaded vectors (registers rotate): four inlined
          // probes instead of sixteen keep the kernel in the I-cache
#pragma unroll 1
          for (int u = 0; u < U; ++u) {
            if (q + u * kFoldThreads + threadIdx.x < b4) {
              add(w[0].x, 0);
              add(w[0].y, 0);
              add(w[0].z, 0);
              add(w[0].w, 0);
            }
#pragma unroll
            for (int r = 0; r + 1 < U; ++r) w[r] = w[r + 1];
          }
        }
        for (uint64_t i = (b4 << 2) + threadIdx.x; i < end; i += kFoldThreads) add(__ldg(src_k + i), 0);
      }
    } else if (std::is_same_v<K, V> && sizeof(K) == 8 && ss == 2) {
      // (key, value) pair records, one 16-byte load each
      const ulonglong2* p = reinterpret_cast<const ulonglong2*>(src_k) + lo;
      constexpr int U = 4;
      for (uint64_t q = 0; q < m && !*vfail; q += static_cast<uint64_t>(kFoldThreads) * U) {
        ulonglong2 w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t x = q + u * kFoldThreads + threadIdx.x;
          w[u] = x < m ? __ldcs(p + x) : make_ulonglong2(0, 0);
        }
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
          if (q + u * kFoldThreads + threadIdx.x < m) add(static_cast<K>(w[0].x), w[0].y);
#pragma unroll
          for (int r = 0; r + 1 < U; ++r) w[r] = w[r + 1];
        }
      }
    } else {
      constexpr int U = 8;
      for (uint64_t q = 0; q < m && !*vfail; q += static_cast<uint64_t>(kFoldThreads) * U) {
        K kk[U];
        uint64_t vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t x = q + u * kFoldThreads + threadIdx.x;
          kk[u] = x < m ? ldg_key(src_k, (lo + x) * ss) : K(0);
          if constexpr (SUM) vv[u] = x < m ? val_u64(src_v[(lo + x) * ss]) : 0ull;
          else vv[u] = 0;
        }
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
          if (q + u * kFoldThreads + threadIdx.x < m) add(kk[0], vv[0]);
#pragma unroll
          for (int r = 0; r + 1 < U; ++r) {
            kk[r] = kk[r + 1];
            vv[r] = vv[r + 1];
          }
        }
      }
    }
    __syncthreads();
    if (*vfail) {
      if (threadIdx.x == 0) {
        G[j] = 0;
        stat[2 * j] = 0;
        stat[2 * j + 1] = 1ull << 32;
      }
      __syncthreads();
      continue;
    }

    // ---- per distinct key: light child (bucket, records), home-group size
    uint32_t counted = 0;   // C16: all records seen through the 16-bit counts
#pragma unroll 4
    for (uint32_t r = 0; r < Sh::kPer; ++r) {
      const uint32_t s = r * kFoldThreads + threadIdx.x;
      const TK k = tk[s];
      if (k == kEmpty) continue;
      c_red(hcnt, home(k));
      const uint32_t c = c_get(cnt, s);
      counted += c;
      const K key = static_cast<K>(k);
      const uint64_t h = key_hash(key, identity);
      if (bf.n_heavy && heavy_find(tab, KeyTraits<K>::widen(key), h, identity) >= 0) continue;
      atomicAdd(&lcnt[bf.lc.id(h)], c);
    }
    if constexpr (C16) {   // a wrapped 16-bit count loses records: the node takes the level path
      if (counted) atomicAdd(&s_used, counted);   // (s_used is free after the stream)
    }
    if (threadIdx.x == 0 && e_cnt) {
      const K key = static_cast<K>(kEmpty);
      const uint64_t h = key_hash(key, identity);
      if (!(bf.n_heavy && heavy_find(tab, KeyTraits<K>::widen(key), h, identity) >= 0))
        atomicAdd(&lcnt[bf.lc.id(h)], e_cnt);
    }
    __syncthreads();
    {
      uint32_t kids = 0, mx = 0, tot = 0;   // node sizes are < 2^32
      for (uint32_t b = threadIdx.x; b < bf.n_light; b += kFoldThreads) {
        const uint32_t c = lcnt[b];
        kids += c != 0;
        mx = c > mx ? c : mx;
        tot += c;
      }
      if (kids) {
        atomicAdd(&s_kids, kids);
        atomicMax(&s_max, mx);
        atomicAdd(&s_light, tot);
      }
    }
    // home-group bases: exclusive scan of hcnt (NB / kFoldThreads per thread)
    constexpr uint32_t kBP = NB / kFoldThreads;
    uint32_t hc[kBP], run = 0;
#pragma unroll
    for (uint32_t r = 0; r < kBP; ++r) {
      hc[r] = c_get(hcnt, threadIdx.x * kBP + r);
      run += hc[r];
    }
    uint32_t total;
    uint32_t before = block_excl_scan<uint32_t>(run, red, total);   // (its barriers order the atomics above)
    bool wrapped = false;   // s_used = inserts (= total) + all records counted
    if constexpr (C16) wrapped = s_used - total != static_cast<uint32_t>(m) - e_cnt;
    if (s_max >= alpha || wrapped) {   // a child would recurse (aggregate.py:139-141): the level path takes the node
      if (threadIdx.x == 0) {
        G[j] = 0;
        stat[2 * j] = 0;
        stat[2 * j + 1] = 1ull << 32;
      }
      __syncthreads();
      continue;
    }
    if constexpr (C16) {   // this thread's kBP (even) buckets are whole words
#pragma unroll
      for (uint32_t r = 0; r < kBP; r += 2) {
        hcnt[(threadIdx.x * kBP + r) >> 1] = before | ((before + hc[r]) << 16);
        before += hc[r] + hc[r + 1];
      }
    } else {
#pragma unroll
      for (uint32_t r = 0; r < kBP; ++r) {
        hcnt[threadIdx.x * kBP + r] = before;
        before += hc[r];
      }
    }
    __syncthreads();

    // ---- emit by (home bucket, key) --------------------------------------
    const uint32_t g0 = e_cnt ? 1u : 0u;
    K* ok = st_k + lo + g0;
    uint64_t* oa = st_a + lo + g0;
    // cursor per home bucket (its base, advanced here): arbitrary order inside
    // a group, fixed by the key sort below
#pragma unroll 4
    for (uint32_t r = 0; r < Sh::kPer; ++r) {
      const uint32_t s = r * kFoldThreads + threadIdx.x;
      const TK k = tk[s];
      if (k == kEmpty) continue;
      const uint32_t at = c_add(hcnt, home(k));
      ok[at] = static_cast<K>(k);
      if constexpr (SUM) oa[at] = (static_cast<uint64_t>(shi[s]) << 32) | slo[s];
      else oa[at] = c_get(cnt, s);
    }
    if (threadIdx.x == 0) {
      if (g0) {
        st_k[lo] = static_cast<K>(kEmpty);
        st_a[lo] = SUM ? (static_cast<uint64_t>(e_hi) << 32) | e_lo : e_cnt;
      }
      G[j] = total + g0;
      stat[2 * j] = s_light;
      stat[2 * j + 1] = s_kids;
    }
    __syncthreads();   // the staged pairs are visible to the whole CTA
    // key order inside each home group (groups are small: ~load x 4 keys);
    // the cursors now hold each group's end
    for (uint32_t b = threadIdx.x; b < NB; b += kFoldThreads) {
      const uint32_t a = b ? c_get(hcnt, b - 1) : 0u, e = c_get(hcnt, b);
      for (uint32_t x = a + 1; x < e; ++x) {
        const K kx = ok[x];
        const uint64_t vx = oa[x];
        uint32_t y = x;
        for (; y > a && ok[y - 1] > kx; --y) {
          ok[y] = ok[y - 1];
          oa[y] = oa[y - 1];
        }
        ok[y] = kx;
        oa[y] = vx;
      }
    }
    __syncthreads();
  }
}

}  // namespace ss
