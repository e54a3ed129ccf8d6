// Sampling and heavy-key detection, one CTA per node (core.py:221-260).
//
// The draw positions are exactly numpy's
//   Generator(Philox(key=mix64_pair(seed, path))).integers(0, m, size=draws)
// i.e. Lemire bounded draws over the Philox4x64-10 stream (32-bit words for
// m < 2^32, 64-bit words above), where a rejected word is simply skipped;
// the accepted words are therefore a stream compaction, which we compute
// with a block scan instead of a sequential loop.  Sampled keys are counted
// in a shared-memory open-addressing table keyed by the key itself (exact
// equality, core.py:193-213), keeping the first stream position of every
// key.  Keys with count >= ceil(log2 n) become heavy, capped at max_heavy by
// (-count, first position) and returned in discovery order.
#pragma once

#include "common.cuh"
#include "types.cuh"

namespace ss {

constexpr int kSampleThreads = 1024;
constexpr uint32_t kSampleSmemCap = 1u << 15;     // table slots kept in SMEM

// Block-wide bitonic sort of N (power of two) uint64 values at generic `d`.
__device__ inline void block_bitonic_u64(uint64_t* d, uint32_t N) {
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        uint32_t ixj = i ^ j;
        if (ixj > i) {
          uint64_t a = d[i], b = d[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) { d[i] = b; d[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ uint32_t pow2_at_least(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Table entry: first stream position in the high half, count in the low
// half.  E = uint32_t (16+16 bits, SMEM) or unsigned long long (32+32, global).
template <typename E> struct Entry;
template <> struct Entry<uint32_t> {
  static constexpr uint32_t kEmpty = 0xFFFFFFFFu;
  static __device__ __forceinline__ uint32_t make(uint32_t first, uint32_t cnt) { return (first << 16) | cnt; }
  static __device__ __forceinline__ uint32_t first(uint32_t e) { return e >> 16; }
  static __device__ __forceinline__ uint32_t count(uint32_t e) { return e & 0xFFFFu; }
};
template <> struct Entry<unsigned long long> {
  static constexpr unsigned long long kEmpty = ~0ull;
  static __device__ __forceinline__ unsigned long long make(uint32_t first, uint32_t cnt) {
    return (static_cast<unsigned long long>(first) << 32) | cnt;
  }
  static __device__ __forceinline__ uint32_t first(unsigned long long e) { return static_cast<uint32_t>(e >> 32); }
  static __device__ __forceinline__ uint32_t count(unsigned long long e) { return static_cast<uint32_t>(e); }
};

// Lanes of `act` holding the same key (both words for 128-bit keys).
__device__ __forceinline__ uint32_t match_key(uint32_t act, uint64_t key) { return __match_any_sync(act, key); }
__device__ __forceinline__ uint32_t match_key(uint32_t act, const U128& key) {
  return __match_any_sync(act, key.lo) & __match_any_sync(act, key.hi);
}

template <typename E, typename S>
__device__ void sample_table_insert(E* tab, uint32_t cap, const S* samp, uint32_t draws) {
  using X = Entry<E>;
  const uint32_t mask = cap - 1;
  for (uint32_t base = 0; base < draws; base += blockDim.x) {
    uint32_t s = base + threadIdx.x;
    bool valid = s < draws;
    const S key = valid ? samp[s] : S(0);
    // lanes holding the same key aggregate; the lowest lane has the
    // smallest stream position
    uint32_t act = __ballot_sync(0xffffffffu, valid);
    if (!valid) continue;
    uint32_t peers = match_key(act, key);
    if (lane_id() != __ffs(peers) - 1) continue;
    uint32_t c = __popc(peers);
    // probe start from the top bits of a multiplicative hash of the folded
    // mix: a node's keys share the low hash bits its ancestors bucketed on,
    // so `mix64(key) & mask` would start every probe in a few slots
    const uint64_t h = key_hash(key, false);
    uint32_t slot = (static_cast<uint32_t>(h ^ (h >> 32)) * 0x9E3779B1u) >> (32 - (31 - __clz(cap)));
    while (true) {
      E old = tab[slot];
      if (old == X::kEmpty) {
        E prev = atomicCAS(&tab[slot], X::kEmpty, X::make(s, c));
        if (prev == X::kEmpty) break;
        old = prev;
      }
      if (samp[X::first(old)] == key) {
        // count: one atomicAdd on the low field (counts < 2^16 resp. 2^32,
        // no carry into the first position); a CAS retry loop here stormed
        // on hot keys (8M retries for 0.5M warp inserts per level-1 launch)
        old = atomicAdd(&tab[slot], static_cast<E>(c));
        // first position: lowered only when this lane's is smaller (rare)
        while (s < X::first(old)) {
          const E prev = atomicCAS(&tab[slot], old, X::make(s, X::count(old)));
          if (prev == old) break;
          old = prev;
        }
        break;
      }
      slot = (slot + 1) & mask;
    }
  }
}

// Per-CTA scratch words (u64): samples (KeyStore x s_cap), candidates
// (s_cap) and the global-memory fallback table (2 * pow2(s_cap)).
__host__ __device__ inline uint64_t sample_scratch_words(uint64_t s_cap, uint32_t key_store_bytes) {
  uint64_t p = 1;
  while (p < s_cap) p <<= 1;
  return s_cap * (key_store_bytes / 8) + s_cap + 2 * p;
}

// One CTA per node (grid-strided over nodes); `scratch` as above.
template <typename K>
__global__ void __launch_bounds__(kSampleThreads)
k_sample(const K* __restrict__ src, Node* __restrict__ nodes, uint32_t n_nodes,
         KeyStore<K>* __restrict__ heavy_out, uint64_t* __restrict__ scratch,
         uint64_t s_cap, Params P, int use_fixed_key, uint64_t fixed_key, uint32_t kstride = 1) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint64_t red[33];
  __shared__ uint32_t n_cand;
  uint32_t* stab = reinterpret_cast<uint32_t*>(smem_raw);
  using S = KeyStore<K>;
  constexpr uint32_t kSW = sizeof(S) / 8;
  uint64_t* mine = scratch + static_cast<uint64_t>(blockIdx.x) * sample_scratch_words(s_cap, sizeof(S));
  S* samp = reinterpret_cast<S*>(mine);
  uint64_t* cand = mine + kSW * s_cap;
  unsigned long long* gtab = reinterpret_cast<unsigned long long*>(cand + s_cap);

  for (uint32_t j = blockIdx.x; j < n_nodes; j += gridDim.x) {
    const uint64_t lo = nodes[j].lo, m = nodes[j].size;
    const uint64_t draws64 = m < P.sample_count ? m : P.sample_count;
    const uint32_t draws = static_cast<uint32_t>(draws64);
    if (draws == 0 || P.max_heavy == 0) {
      if (threadIdx.x == 0) nodes[j].n_heavy = 0;
      continue;
    }
    const uint64_t rkey = use_fixed_key ? fixed_key : mix64_pair(P.seed, nodes[j].path);

    // ---- 1. draw positions, gather the sampled keys ------------------------
    // mode 0: m == 1 (no words consumed); 1: 32-bit Lemire; 2: raw 32-bit
    // words (m == 2^32); 3: 64-bit Lemire.
    const uint64_t rng = m - 1;
    const int mode = rng == 0 ? 0 : (rng < 0xFFFFFFFFull ? 1 : (rng == 0xFFFFFFFFull ? 2 : 3));
    const uint32_t thr32 = mode == 1 ? static_cast<uint32_t>((1ull << 32) % m) : 0;
    const uint64_t thr64 = mode == 3 ? (0ull - m) % m : 0;
    uint64_t accepted = 0, blk = 0;
    while (accepted < draws) {
      uint64_t pos[8];
      uint32_t flags = 0;
      if (mode == 0) {
        for (int w = 0; w < 8; ++w) pos[w] = 0;
        flags = 0xFF;
      } else {
        U64x4 r = philox4x64_10(blk + threadIdx.x + 1, rkey);
        if (mode == 3) {
          for (int w = 0; w < 4; ++w) {
            uint64_t hi, lo2;
            mulhilo64(r.v[w], m, hi, lo2);
            pos[w] = hi;
            if (lo2 >= thr64) flags |= 1u << w;
          }
        } else {
          for (int w = 0; w < 8; ++w) {
            uint32_t word = static_cast<uint32_t>(r.v[w >> 1] >> (32 * (w & 1)));
            if (mode == 2) { pos[w] = word; flags |= 1u << w; continue; }
            uint64_t prod = static_cast<uint64_t>(word) * m;
            pos[w] = prod >> 32;
            if (static_cast<uint32_t>(prod) >= thr32) flags |= 1u << w;
          }
        }
      }
      uint64_t mine_cnt = __popc(flags), total;
      uint64_t at = accepted + block_excl_scan<uint64_t>(mine_cnt, red, total);
      for (int w = 0; w < 8; ++w) {
        if (!(flags >> w & 1)) continue;
        if (at < draws) samp[at] = static_cast<S>(src[(lo + pos[w]) * kstride]);   // 2: pair layout
        ++at;
      }
      accepted += total;
      blk += blockDim.x;
    }
    __syncthreads();

    // ---- 2. count sampled keys in a hash table -----------------------------
    uint32_t cap = pow2_at_least(2 * draws);
    if (cap < 64) cap = 64;
    const bool in_smem = cap <= kSampleSmemCap && draws < 0xFFFFu;
    if (in_smem) {
      for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) stab[s] = Entry<uint32_t>::kEmpty;
    } else {
      for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) gtab[s] = Entry<unsigned long long>::kEmpty;
    }
    if (threadIdx.x == 0) n_cand = 0;
    __syncthreads();
    if (in_smem) sample_table_insert<uint32_t>(stab, cap, samp, draws);
    else sample_table_insert<unsigned long long>(gtab, cap, samp, draws);
    __syncthreads();

    // ---- 3. candidates: count >= ceil(threshold) ---------------------------
    const uint32_t thr = static_cast<uint32_t>(P.heavy_threshold_int);
    for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
      uint32_t f, c;
      bool occ;
      if (in_smem) {
        uint32_t e = stab[s];
        occ = e != Entry<uint32_t>::kEmpty; f = Entry<uint32_t>::first(e); c = Entry<uint32_t>::count(e);
      } else {
        unsigned long long e = gtab[s];
        occ = e != Entry<unsigned long long>::kEmpty;
        f = Entry<unsigned long long>::first(e); c = Entry<unsigned long long>::count(e);
      }
      if (occ && c >= thr) {
        uint32_t at = atomicAdd(&n_cand, 1u);
        cand[at] = (static_cast<uint64_t>(c) << 32) | f;
      }
    }
    __syncthreads();
    const uint32_t n_k = n_cand;
    const uint32_t keep = n_k < P.max_heavy ? n_k : P.max_heavy;
    if (n_k > 0) {
      // sort buffer: reuse the SMEM table when it fits, else sort in place
      uint32_t N = pow2_at_least(n_k);
      uint64_t* buf = (N * 8 <= kSampleSmemCap * 4) ? reinterpret_cast<uint64_t*>(smem_raw) : cand;
      if (n_k > P.max_heavy) {
        // order by (-count, first): key = (~count << 32) | first
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
          uint64_t v = ~0ull;
          if (i < n_k) {
            uint64_t e = cand[i];
            v = (static_cast<uint64_t>(~static_cast<uint32_t>(e >> 32)) << 32) | (e & 0xFFFFFFFFu);
          }
          if (buf != cand) buf[i] = v;
          else if (i < n_k) cand[i] = v;
          else cand[i] = ~0ull;
        }
        __syncthreads();
        block_bitonic_u64(buf, N);
        // keep the first `keep`, re-sort by first position
        N = pow2_at_least(keep);
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x)
          buf[i] = i < keep ? (buf[i] & 0xFFFFFFFFu) : ~0ull;   // own element only
        __syncthreads();
      } else {
        for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
          uint64_t v = i < n_k ? (cand[i] & 0xFFFFFFFFu) : ~0ull;
          if (buf != cand) buf[i] = v;
          else cand[i] = v;
        }
        __syncthreads();
      }
      block_bitonic_u64(buf, N);
      for (uint32_t t = threadIdx.x; t < keep; t += blockDim.x)
        heavy_out[static_cast<uint64_t>(j) * P.max_heavy + t] = samp[buf[t]];
    }
    if (threadIdx.x == 0) nodes[j].n_heavy = keep;
    __syncthreads();
  }
}

}  // namespace ss
