// Shared device primitives for the B200 semisort hot path (sm_100a).
//
// Everything here is integer work: the splitmix64 finalizer the reference
// uses as its key hash (hashing.py:25-47), the numpy-compatible
// Philox4x64-10 stream that drives sampling (core.py:238-239, numpy's
// Generator.integers -> Lemire bounded draws), the per-depth light-id bit
// slice (core.py:139-151), and a shared-memory heavy-key table
// (core.py:64-104, 193-213).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ss {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;   // hashing.py:14
constexpr uint64_t kMul1 = 0xBF58476D1CE4E5B9ull;    // hashing.py:15
constexpr uint64_t kMul2 = 0x94D049BB133111EBull;    // hashing.py:16
constexpr int kDepthLimit = 64;                      // core.py:39
constexpr uint32_t kNoBucket = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + kGamma;
  z = (z ^ (z >> 30)) * kMul1;
  z = (z ^ (z >> 27)) * kMul2;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix64_pair(uint64_t a, uint64_t b) {
  return mix64(a ^ mix64(b));
}

// Value payload of a record: the reference's values column may be absent or
// any fixed-width layout; the hot path only moves it.
struct NoVal {};
struct alignas(16) V16 { uint64_t lo, hi; };

template <typename T> struct ValTraits { static constexpr int bytes = sizeof(T); };
template <> struct ValTraits<NoVal> { static constexpr int bytes = 0; };

template <typename V>
__device__ __forceinline__ V load_val(const V* p, uint64_t i) { return p[i]; }
template <>
__device__ __forceinline__ NoVal load_val<NoVal>(const NoVal*, uint64_t) { return NoVal{}; }
template <typename V>
__device__ __forceinline__ void store_val(V* p, uint64_t i, const V& v) { p[i] = v; }
template <>
__device__ __forceinline__ void store_val<NoVal>(NoVal*, uint64_t, const NoVal&) {}

// 128-bit key (UInt128KeyAdapter, adapters.py:147-197): (lo, hi) words;
// equality on both words, order lexicographic by (hi, lo) (np.lexsort((lo,
// hi)), adapters.py:186-190).
struct alignas(16) U128 {
  uint64_t lo, hi;
  U128() = default;
  __host__ __device__ explicit constexpr U128(uint64_t v) : lo(v), hi(0) {}   // K(0) padding
  __host__ __device__ constexpr U128(uint64_t l, uint64_t h) : lo(l), hi(h) {}
};
__host__ __device__ __forceinline__ bool operator==(const U128& a, const U128& b) { return a.lo == b.lo && a.hi == b.hi; }
__host__ __device__ __forceinline__ bool operator!=(const U128& a, const U128& b) { return !(a == b); }
__host__ __device__ __forceinline__ bool operator<(const U128& a, const U128& b) {
  return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
__host__ __device__ __forceinline__ bool operator>(const U128& a, const U128& b) { return b < a; }

// How a key is stored in heavy tables and sample buffers: u32 keys widen to
// u64 (adapters.py:113), u64 and U128 keys are kept as they are.
template <typename K> struct KeyTraits {
  using Store = uint64_t;
  __host__ __device__ static uint64_t widen(K k) { return static_cast<uint64_t>(k); }
};
template <> struct KeyTraits<U128> {
  using Store = U128;
  __host__ __device__ static U128 widen(U128 k) { return k; }
};
template <typename K> using KeyStore = typename KeyTraits<K>::Store;

__host__ __device__ __forceinline__ uint64_t low_word(uint64_t k) { return k; }
__host__ __device__ __forceinline__ uint64_t low_word(const U128& k) { return k.lo; }

// Read-only streaming load of one key.
template <typename K>
__device__ __forceinline__ K ldg_key(const K* p, uint64_t i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ U128 ldg_key<U128>(const U128* p, uint64_t i) {
  const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(p) + i);
  return U128(w.x, w.y);
}

// ---------------------------------------------------------------------------
// key hash and light ids
// ---------------------------------------------------------------------------

template <typename K>
__host__ __device__ __forceinline__ uint64_t key_hash(K key, bool identity) {
  uint64_t k = static_cast<uint64_t>(key);   // u32 keys widen (adapters.py:113)
  return identity ? k : mix64(k);
}
// 128-bit keys: mix64(mix64(hi) ^ lo), identity: lo (adapters.py:158-168)
__host__ __device__ __forceinline__ uint64_t key_hash(const U128& key, bool identity) {
  return identity ? key.lo : mix64(mix64(key.hi) ^ key.lo);
}

// Per-node light-id slice: rnd, slot = divmod(depth, rounds) (core.py:146-151).
struct LightCfg {
  uint64_t salt;     // mix64(rnd), used when remix != 0
  uint32_t shift;    // slot * light_bits
  uint32_t mask;     // n_light - 1
  uint32_t remix;    // rnd > 0

  __host__ __device__ static LightCfg make(uint32_t depth, uint32_t light_bits, uint32_t n_light) {
    uint32_t rounds = 64u / (light_bits > 1 ? light_bits : 1u);
    if (rounds < 1) rounds = 1;
    uint32_t rnd = depth / rounds, slot = depth % rounds;
    LightCfg c;
    c.salt = mix64(static_cast<uint64_t>(rnd));
    c.shift = slot * light_bits;
    c.mask = n_light - 1;
    c.remix = rnd != 0;
    return c;
  }
  __device__ __forceinline__ uint32_t id(uint64_t h) const {
    if (remix) h = mix64(h ^ salt);
    return static_cast<uint32_t>(h >> shift) & mask;
  }
};

// ---------------------------------------------------------------------------
// shared-memory heavy table: key -> heavy slot (discovery order)
// ---------------------------------------------------------------------------

constexpr int kHeavySlots = 1024;   // >= 2 * max_heavy (500); power of two
constexpr int kMaxHeavyDevice = 512;

// Open-addressing table keyed by the heavy key (stored as KeyStore<K>); the
// home slot is the top 10 bits of the key's (mixed) hash, and a 1024-bit
// home bitmap lets the common light record leave after one shared-memory
// word test.
template <typename S>
struct HeavySmemT {
  S keys[kHeavySlots];
  unsigned short ids[kHeavySlots];
  uint32_t home_bits[kHeavySlots / 32];
};
using HeavySmem = HeavySmemT<uint64_t>;

// 64-bit hash used for the table home slot (mixed for identity keys too).
template <typename S>
__device__ __forceinline__ uint64_t heavy_hash(const S& key, uint64_t h, bool identity) {
  return identity ? low_word(key) * kGamma : h;
}
__device__ __forceinline__ uint32_t heavy_home_of(uint64_t hh) { return static_cast<uint32_t>(hh >> 54); }

// Cooperative parallel build; caller must __syncthreads() afterwards.
template <typename S>
__device__ __forceinline__ void heavy_build(HeavySmemT<S>& t, const S* heavy, uint32_t n_heavy, bool identity) {
  for (int s = threadIdx.x; s < kHeavySlots; s += blockDim.x) t.ids[s] = 0xFFFF;
  for (int s = threadIdx.x; s < kHeavySlots / 32; s += blockDim.x) t.home_bits[s] = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n_heavy; i += blockDim.x) {
    const S k = heavy[i];
    const uint32_t home = heavy_home_of(heavy_hash(k, key_hash(k, identity), identity));
    atomicOr(&t.home_bits[home >> 5], 1u << (home & 31));
    uint32_t s = home;
    while (atomicCAS(&t.ids[s], static_cast<unsigned short>(0xFFFF), static_cast<unsigned short>(i)) != 0xFFFF)
      s = (s + 1) & (kHeavySlots - 1);
    t.keys[s] = k;
  }
}

// Returns the heavy slot of key (with 64-bit hash h) or -1.
template <typename S>
__device__ __forceinline__ int heavy_find(const HeavySmemT<S>& t, const S& key, uint64_t h, bool identity) {
  uint32_t s = heavy_home_of(heavy_hash(key, h, identity));
  if (!(t.home_bits[s >> 5] & (1u << (s & 31)))) return -1;
  while (true) {
    uint16_t id = t.ids[s];
    if (id == 0xFFFF) return -1;
    if (t.keys[s] == key) return id;
    s = (s + 1) & (kHeavySlots - 1);
  }
}

// Bucket id of a key at a node: heavy -> n_light + slot, else the light slice.
template <typename K>
__device__ __forceinline__ uint32_t bucket_of(K key, const HeavySmemT<KeyStore<K>>& t, uint32_t n_heavy,
                                              const LightCfg& lc, bool identity, uint32_t n_light) {
  const KeyStore<K> k = KeyTraits<K>::widen(key);
  const uint64_t h = key_hash(k, identity);
  if (n_heavy) {
    int hv = heavy_find(t, k, h, identity);
    if (hv >= 0) return n_light + static_cast<uint32_t>(hv);
  }
  return lc.id(h);
}

// Lanes of `active` whose value equals this lane's, from `bits` ballots
// (a multisplit peer mask without MATCH.ANY, whose ADU issue cost is ~57
// SM cycles per warp instruction on sm_100).  All 32 lanes must call it.
__device__ __forceinline__ uint32_t ballot_peers(uint32_t v, uint32_t active, int bits) {
  uint32_t m = active;
  for (int j = 0; j < bits; ++j) {
    const uint32_t bit = (v >> j) & 1u;
    const uint32_t b = __ballot_sync(0xffffffffu, bit);
    m &= bit ? b : ~b;
  }
  return m;
}

template <int BITS>
__device__ __forceinline__ uint32_t ballot_peers_t(uint32_t v, uint32_t active) {
  uint32_t m = active;
#pragma unroll
  for (int j = 0; j < BITS; ++j) {
    const uint32_t bit = (v >> j) & 1u;
    const uint32_t b = __ballot_sync(0xffffffffu, bit);
    m &= bit ? b : ~b;
  }
  return m;
}

__device__ __forceinline__ int bits_for(uint32_t n) {   // ceil(log2(n)), n >= 1
  return n <= 1 ? 0 : 32 - __clz(n - 1);
}

// ---------------------------------------------------------------------------
// numpy Philox4x64-10 + Generator.integers(0, m) (Lemire, no masking)
// ---------------------------------------------------------------------------

struct U64x4 { uint64_t v[4]; };

__host__ __device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = static_cast<unsigned __int128>(a) * b;
  lo = static_cast<uint64_t>(p);
  hi = static_cast<uint64_t>(p >> 64);
#endif
}

// Counter block `ctr` (numpy increments the 256-bit counter before each
// block, so block j of a fresh generator uses counter j+1), key (k0, 0).
__host__ __device__ __forceinline__ U64x4 philox4x64_10(uint64_t ctr, uint64_t k0) {
  uint64_t c0 = ctr, c1 = 0, c2 = 0, c3 = 0, k1 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ull, c0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ull, c2, hi1, lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  U64x4 out;
  out.v[0] = c0; out.v[1] = c1; out.v[2] = c2; out.v[3] = c3;
  return out;
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane_id() >= d) v += o;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; `tmp` needs
// blockDim/32 + 1 entries.  Returns the exclusive prefix, writes the total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* tmp, T& total) {
  T inc = warp_incl_scan(v);
  const int w = warp_id(), nw = blockDim.x >> 5;
  if (lane_id() == 31) tmp[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane_id() < nw ? tmp[lane_id()] : T(0);
    T xi = warp_incl_scan(x);
    if (lane_id() < nw) tmp[lane_id()] = xi - x;
    if (lane_id() == nw - 1) tmp[32] = xi;
  }
  __syncthreads();
  T out = tmp[w] + inc - v;
  total = tmp[32];
  __syncthreads();
  return out;
}

}  // namespace ss
