// Blocked Distributing scatter (core.py:321-380, aggregate.py:172-193).
//
// Persistent, one 512-thread CTA per SM; each CTA walks its subarrays (work
// items) in 4096-record tiles.  The bucket id of every record was written
// by the count pass (u16, 2 bytes / record), so this kernel never rehashes.
// Per tile:
//   * TMA bulk copies (cp.async.bulk + mbarrier) stream ids, keys and
//     values of tile t+1 into the second half of a double buffer while
//     tile t is processed;
//   * a shared-atomic histogram of the tile's ids and one block scan give
//     every bucket's start inside the tile (no run-boundary pass);
//   * a stable two-pass 7-bit LSD radix sort of (id << 12 | index) in
//     shared memory orders the tile by (bucket, input position); peers of
//     a digit inside a warp come from shared atomicOr masks, which cost
//     ~5-8 SM cycles per warp op on sm_100 against ~53 for MATCH.ANY
//     (tools/peers_bench.cu);
//   * records leave as contiguous per-bucket runs at the subarray's SMEM
//     cursors (its X row), then the cursors advance by the tile histogram.
// Stability and race freedom come from disjoint cursor ranges, never from
// atomics deciding order.
#pragma once

#include "common.cuh"
#include "tma.cuh"
#include "types.cuh"

namespace ss {

constexpr int kDistThreads = 512;
constexpr int kDistWarps = kDistThreads / 32;
constexpr int kDistCtasPerSm = 1;
constexpr int kRadixBits = 7;
constexpr int kRadixBins = 1 << kRadixBits;
constexpr uint32_t kIdxBits = 12;                              // tile index bits (tile <= 4096)
constexpr uint32_t kSentinel = (1u << (2 * kRadixBits)) - 1;   // bucket sorting last
constexpr uint32_t kMaxDistBuckets = kSentinel;                // ids must stay below

// Debug / measurement knob (SS_DIST_DEBUG): 0 normal, 1 skip the scattered
// stores, 2 store linearly (tile-contiguous).  Outputs are wrong unless 0.
__device__ int g_dist_debug = 0;

template <typename K, typename V, int TILE>
struct DistCfg {
  static constexpr int kValBytes = ValTraits<V>::bytes;
  static constexpr int kTile = TILE;
  static constexpr int kItems = kTile / kDistThreads;
  static constexpr size_t up16(size_t x) { return (x + 15) & ~size_t(15); }
  static constexpr size_t kBufI = up16((static_cast<size_t>(kTile) + 8) * 2);
  static constexpr size_t kBufK = up16((static_cast<size_t>(kTile) + 16 / sizeof(K)) * sizeof(K));
  static constexpr size_t kBufV = kValBytes ? up16((static_cast<size_t>(kTile) + 16) * kValBytes) : 0;
  static size_t smem_bytes(uint32_t stride) {
    return 2 * (kBufI + kBufK + kBufV) + 2 * static_cast<size_t>(kTile) * 4 + up16(static_cast<size_t>(stride) * 8) +
           2 * up16(static_cast<size_t>(stride) * 4) + 2 * kDistWarps * kRadixBins * 4 + 64;
  }
};

constexpr size_t kMaxDynSmem = 227 * 1024;

// Largest tile (4096, 2048 or 1024 records) whose buffers fit shared memory.
template <typename K, typename V>
__host__ inline int dist_tile_for(uint32_t stride) {
  if (DistCfg<K, V, 4096>::smem_bytes(stride) <= kMaxDynSmem) return 4096;
  if (DistCfg<K, V, 2048>::smem_bytes(stride) <= kMaxDynSmem) return 2048;
  return 1024;
}

// One stable LSD pass over the tile: entries e[k] sit at logical positions
// w*(32*ITEMS) + k*32 + lane; digit = (e >> shift) & 127.  Writes the
// entries to `out` ordered by (digit, logical position).
template <int ITEMS>
__device__ __forceinline__ void radix_pass(const uint32_t (&e)[ITEMS], int shift, uint32_t* dh, uint32_t* out,
                                           uint32_t* red, uint32_t* pm) {
  const int w = warp_id(), lane = lane_id();
  const uint32_t lt = lanemask_lt();
  uint32_t* mine = dh + w * kRadixBins;
  uint32_t* mask = pm + w * kRadixBins;
  for (int i = lane; i < kRadixBins; i += 32) mine[i] = 0;
  __syncwarp();
  uint32_t rk[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t d = (e[k] >> shift) & (kRadixBins - 1);
    atomicOr(&mask[d], 1u << lane);
    __syncwarp();
    const uint32_t peers = mask[d];
    const uint32_t base = mine[d];
    __syncwarp();
    if (lane == 31 - __clz(peers)) {
      mine[d] = base + __popc(peers);
      mask[d] = 0;
    }
    rk[k] = base + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan in (digit, warp) order: kPer consecutive entries per thread
  constexpr int kEntries = kDistWarps * kRadixBins;
  constexpr int kPer = kEntries / kDistThreads;
  uint32_t v[kPer], s = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x * kPer + q;          // j = d * kDistWarps + w
    v[q] = dh[(j % kDistWarps) * kRadixBins + j / kDistWarps];
    s += v[q];
  }
  uint32_t tot;
  uint32_t run = block_excl_scan<uint32_t>(s, red, tot);
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x * kPer + q;
    dh[(j % kDistWarps) * kRadixBins + j / kDistWarps] = run;
    run += v[q];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t d = (e[k] >> shift) & (kRadixBins - 1);
    out[mine[d] + rk[k]] = e[k];
  }
}

// ids: u16 bucket id per source record (absolute index), written by the
// count pass.  Buckets kept: [0, nb) with nb = min(fixed_nb or
// n_light + node.n_heavy, keep_below); others are dropped.
template <typename K, typename V, int TILE>
__global__ void __launch_bounds__(kDistThreads, kDistCtasPerSm)
k_distribute(const K* __restrict__ sk, const V* __restrict__ sv, const uint16_t* __restrict__ ids,
             K* __restrict__ dk, V* __restrict__ dv, const Work* __restrict__ work, uint32_t n_work,
             const Node* __restrict__ nodes, const uint64_t* __restrict__ X, uint32_t stride, uint32_t keep_below,
             uint32_t n_light, uint32_t fixed_nb) {
  using Cfg = DistCfg<K, V, TILE>;
  constexpr bool kHasV = Cfg::kValBytes > 0;
  constexpr int T = Cfg::kTile;
  constexpr int ITEMS = Cfg::kItems;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t red[33];
  __shared__ __align__(8) uint64_t bars[2];

  unsigned char* p = smem;
  uint16_t* bufI[2];
  K* bufK[2];
  V* bufV[2];
  for (int b = 0; b < 2; ++b) {
    bufI[b] = reinterpret_cast<uint16_t*>(p); p += Cfg::kBufI;
    bufK[b] = reinterpret_cast<K*>(p); p += Cfg::kBufK;
    bufV[b] = reinterpret_cast<V*>(p); p += Cfg::kBufV;
  }
  uint32_t* srtA = reinterpret_cast<uint32_t*>(p); p += T * 4;
  uint32_t* srtB = reinterpret_cast<uint32_t*>(p); p += T * 4;
  uint64_t* cursor = reinterpret_cast<uint64_t*>(p); p += Cfg::up16(static_cast<size_t>(stride) * 8);
  uint32_t* hist = reinterpret_cast<uint32_t*>(p); p += Cfg::up16(static_cast<size_t>(stride) * 4);
  uint32_t* toff = reinterpret_cast<uint32_t*>(p); p += Cfg::up16(static_cast<size_t>(stride) * 4);
  uint32_t* dh = reinterpret_cast<uint32_t*>(p);
  uint32_t* pm = dh + kDistWarps * kRadixBins;
  for (int i = threadIdx.x; i < kDistWarps * kRadixBins; i += blockDim.x) pm[i] = 0;
  const int dbg = g_dist_debug;
  const int w = warp_id(), lane = lane_id();

  struct It {
    uint32_t wi;
    uint32_t tb;
  };
  auto first_it = [&](uint32_t wi0) {
    It it{wi0, 0};
    while (it.wi < n_work && work[it.wi].len == 0) it.wi += gridDim.x;
    return it;
  };
  auto next_it = [&](It it) {
    it.tb += T;
    if (it.tb >= work[it.wi].len) it = first_it(it.wi + gridDim.x);
    return it;
  };
  auto issue = [&](It it, int b) {   // one thread
    const Work wk = work[it.wi];
    const uint64_t begin = wk.begin + it.tb;
    const uint32_t cnt = min(static_cast<uint32_t>(T), wk.len - it.tb);
    uint32_t bytes = span_body_bytes(ids, begin, cnt) + span_body_bytes(sk, begin, cnt);
    if constexpr (kHasV) bytes += span_body_bytes(sv, begin, cnt);
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[b], bytes);
    stage_span(bufI[b], ids, begin, cnt, &bars[b]);
    stage_span(bufK[b], sk, begin, cnt, &bars[b]);
    if constexpr (kHasV) stage_span(bufV[b], sv, begin, cnt, &bars[b]);
  };

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();

  It cur = first_it(blockIdx.x);
  if (cur.wi >= n_work) return;
  if (threadIdx.x == 0) issue(cur, 0);
  uint32_t q = 0, nb = 0;
  while (cur.wi < n_work) {
    const int buf = q & 1;
    const It nxt = next_it(cur);
    if (threadIdx.x == 0 && nxt.wi < n_work) issue(nxt, buf ^ 1);
    const Work wk = work[cur.wi];
    if (cur.tb == 0) {   // new subarray: its X row and bucket count
      nb = fixed_nb ? fixed_nb : n_light + nodes[wk.node].n_heavy;
      if (nb > keep_below) nb = keep_below;
      const uint64_t* xrow = X + wk.row * stride;
      for (uint32_t b = threadIdx.x; b < nb; b += kDistThreads) cursor[b] = xrow[b];
    }
    for (uint32_t b = threadIdx.x; b < nb; b += kDistThreads) hist[b] = 0;
    const uint64_t begin = wk.begin + cur.tb;
    const uint32_t cnt = min(static_cast<uint32_t>(T), wk.len - cur.tb);
    const uint32_t shI = Span16<uint16_t>(ids, begin, cnt).sh;
    const uint32_t shK = Span16<K>(sk, begin, cnt).sh;
    uint32_t shV = 0;
    if constexpr (kHasV) shV = Span16<V>(sv, begin, cnt).sh;
    mbar_wait(&bars[buf], (q >> 1) & 1);
    __syncthreads();   // head/tail elements, cursors, zeroed histogram visible

    // ids of the tile -> histogram + (bucket << 12 | index) entries
    uint32_t e[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t i = w * (32 * ITEMS) + k * 32 + lane;
      uint32_t b = kSentinel;
      if (i < cnt) {
        b = bufI[buf][i + shI];
        if (b >= nb) b = kSentinel;
        else atomicAdd(&hist[b], 1u);
      }
      e[k] = (b << kIdxBits) | i;
    }
    radix_pass<ITEMS>(e, kIdxBits, dh, srtA, red, pm);
    // bucket starts inside the sorted tile (scan of the histogram)
    {
      const uint32_t per = (nb + kDistThreads - 1) / kDistThreads;
      const uint32_t b0 = min(nb, threadIdx.x * per), b1 = min(nb, b0 + per);
      uint32_t local = 0;
      for (uint32_t b = b0; b < b1; ++b) local += hist[b];
      uint32_t tot;
      uint32_t run = block_excl_scan<uint32_t>(local, red, tot);   // also fences the pass-1 scatter
      for (uint32_t b = b0; b < b1; ++b) {
        toff[b] = run;
        run += hist[b];
      }
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) e[k] = srtA[w * (32 * ITEMS) + k * 32 + lane];
    radix_pass<ITEMS>(e, kIdxBits + kRadixBits, dh, srtB, red, pm);
    __syncthreads();
    // contiguous per-bucket runs out of the staged tile
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t s = threadIdx.x + k * kDistThreads;
      const uint32_t ent = srtB[s];
      const uint32_t b = ent >> kIdxBits;
      if (b == kSentinel) continue;
      const uint32_t i = ent & ((1u << kIdxBits) - 1);
      uint64_t d = cursor[b] + (s - toff[b]);
      if (dbg) d = begin + s;
      if (dbg != 1) {
        dk[d] = bufK[buf][i + shK];
        if constexpr (kHasV) dv[d] = bufV[buf][i + shV];
      }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += kDistThreads) cursor[b] += hist[b];
    __syncthreads();   // buffer `buf` may be refilled; cursors final for the next tile
    cur = nxt;
    ++q;
  }
}

}  // namespace ss
