// Blocked Distributing scatter (core.py:321-380, aggregate.py:172-193).
//
// Persistent, one 512-thread CTA per SM; each CTA walks its subarrays (work
// items) in 4096-record tiles.  The bucket id of every record was written
// by the count pass (u16, 2 bytes / record), so this kernel never rehashes.
// Per tile:
//   * TMA bulk copies (cp.async.bulk + mbarrier) stream ids, keys and
//     values of tile t+1 into the second half of a double buffer while
//     tile t is processed (the 16-byte aligned superset of the tile, so the
//     issuing thread never waits on a global load);
//   * a shared-atomic histogram of the tile's ids and one block scan give
//     every bucket's start inside the tile (no run-boundary pass);
//   * a stable two-pass 7-bit LSD radix sort of (id << 12 | index) in
//     shared memory orders the tile by (bucket, input position); peers of
//     a digit inside a warp come from shared atomicOr masks, which cost
//     ~5-8 SM cycles per warp op on sm_100 against ~53 for MATCH.ANY
//     (tools/peers_bench.cu);
//   * records leave as contiguous per-bucket runs at the subarray's
//     cursors (its X row); the cursors advance by the tile histogram.
// Stability and race freedom come from disjoint cursor ranges, never from
// atomics deciding order.
#pragma once

#include "common.cuh"
#include "tma.cuh"
#include "types.cuh"

namespace ss {

constexpr int kRadixBits = 7;
constexpr int kRadixBins = 1 << kRadixBits;
constexpr uint32_t kIdxBits = 12;                              // tile index bits (tile <= 4096)
constexpr uint32_t kSentinel = (1u << (2 * kRadixBits)) - 1;   // bucket sorting last
constexpr uint32_t kMaxDistBuckets = kSentinel;                // ids must stay below
// Row stride of the per-warp digit counters: 130 = 2 (mod 32) makes the
// (digit, warp)-major scan reads conflict-free.
constexpr int kDhStride = kRadixBins + 2;

// Debug / measurement knob (SS_DIST_DEBUG): 0 normal, 1 skip the scattered
// stores, 2 store linearly (tile-contiguous).  Outputs are wrong unless 0.
__device__ int g_dist_debug = 0;
// Phase profile (SS_DIST_DEBUG bit 4): cycles per phase summed over CTAs.
__device__ unsigned long long g_dist_prof[12];   // [10] CTAs, [11] max cycles of one CTA

// Launch shape: NT threads per CTA, STAGES input buffers, TILE records.
template <typename K, typename V, int TILE, int NT = 512, int STAGES = 2>
struct DistCfg {
  static constexpr int kValBytes = ValTraits<V>::bytes;
  static constexpr int kTile = TILE;
  static constexpr int kThreads = NT;
  static constexpr int kWarps = NT / 32;
  static constexpr int kStages = STAGES;
  static constexpr int kItems = kTile / kThreads;
  static constexpr size_t up16(size_t x) { return (x + 15) & ~size_t(15); }
  // +2 x (16 / element size) elements: the aligned superset of a tile
  static constexpr size_t kBufI = up16((static_cast<size_t>(kTile) + 16) * 2);
  static constexpr size_t kBufK = up16((static_cast<size_t>(kTile) + 2 * (16 / sizeof(K))) * sizeof(K));
  static constexpr size_t kBufV =
      kValBytes ? up16((static_cast<size_t>(kTile) + 2 * (16 / kValBytes > 0 ? 16 / kValBytes : 1)) * kValBytes) : 0;
  static constexpr size_t kSet = kBufI + kBufK + kBufV;   // one pipeline stage
  static size_t smem_bytes(uint32_t stride) {
    return kStages * kSet + 2 * static_cast<size_t>(kTile) * 4 + 2 * up16(static_cast<size_t>(stride) * 8) +
           up16(static_cast<size_t>(stride) * 4) + 2 * kWarps * kDhStride * 4 + 64;
  }
};

constexpr size_t kMaxDynSmem = 227 * 1024 - 1024;   // leave room for static shared memory

// Largest tile (4096, 2048 or 1024 records) whose buffers fit shared memory.
template <typename K, typename V>
__host__ inline int dist_tile_for(uint32_t stride) {
  if (DistCfg<K, V, 4096>::smem_bytes(stride) <= kMaxDynSmem) return 4096;
  if (DistCfg<K, V, 2048>::smem_bytes(stride) <= kMaxDynSmem) return 2048;
  return 1024;
}

// Per-warp stable ranks of one LSD digit: e[k] at logical position
// w*(32*ITEMS) + k*32 + lane, digit = (e >> shift) & 127.  Leaves the warp's
// digit counts in dh[w][*] and each item's rank among equal digits of its
// warp (index order) in rk[k].
//
// HW: a shared atomicAdd of 1 returns each lane its rank among the lanes
// of the warp instruction that hit the same counter, in lane order, on
// sm_100 (probed at load time by ss::hw_rank_ok(); HW is false if the probe
// fails).  Otherwise peers come from shared atomicOr masks.
template <int ITEMS, int NW, bool HW>
__device__ __forceinline__ void radix_rank(const uint32_t (&e)[ITEMS], int shift, uint32_t* dh, uint32_t* pm,
                                           uint32_t (&rk)[ITEMS]) {
  const int w = warp_id(), lane = lane_id();
  const uint32_t lt = lanemask_lt();
  uint32_t* mine = dh + w * kDhStride;
  uint32_t* mask = pm + w * kDhStride;
  for (int i = lane; i < kRadixBins; i += 32) mine[i] = 0;
  __syncwarp();
  if constexpr (HW) {
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      rk[k] = atomicAdd(&mine[(e[k] >> shift) & (kRadixBins - 1)], 1u);
      __syncwarp();   // item k's increments precede item k+1's
    }
    return;
  }
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
}

// Barrier of the NW consumer warps only (named barrier 1): the producer
// warp never joins it.
template <int NW>
__device__ __forceinline__ void csync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
}

// Exclusive scan over the NW consumer warps, one value per thread, with a
// single barrier: every warp rescans the NW warp totals itself.  `red`
// (NW entries) must not be rewritten before all warps have read it (the
// callers separate two scans by at least one barrier).
template <int NW>
__device__ __forceinline__ unsigned long long cscan_u64(unsigned long long v, unsigned long long* red,
                                                        unsigned long long& total) {
  const int w = warp_id(), lane = lane_id();
  const unsigned long long inc = warp_incl_scan(v);
  if (lane == 31) red[w] = inc;
  csync<NW>();
  const unsigned long long x = lane < NW ? red[lane] : 0ull;
  const unsigned long long xi = warp_incl_scan(x);
  total = __shfl_sync(0xffffffffu, xi, NW - 1);
  const unsigned long long before = __shfl_sync(0xffffffffu, xi - x, w);
  return before + inc - v;
}

// (digit, warp)-major exclusive scan of dh in place: kPer entries per
// thread.  `extra` (< 2^32 in total) is scanned alongside in the high half.
template <int NW>
__device__ __forceinline__ uint32_t radix_scan(uint32_t* dh, unsigned long long* red64, uint32_t extra) {
  constexpr int kDistWarps = NW;
  constexpr int kEntries = NW * kRadixBins;
  constexpr int kPer = kEntries / (NW * 32);
  uint32_t v[kPer], s = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x * kPer + q;          // j = d * kDistWarps + w
    v[q] = dh[(j % kDistWarps) * kDhStride + j / kDistWarps];
    s += v[q];
  }
  unsigned long long tot;
  const unsigned long long packed = (static_cast<unsigned long long>(extra) << 32) | s;
  const unsigned long long ex = cscan_u64<NW>(packed, red64, tot);
  uint32_t run = static_cast<uint32_t>(ex);
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = threadIdx.x * kPer + q;
    dh[(j % kDistWarps) * kDhStride + j / kDistWarps] = run;
    run += v[q];
  }
  return static_cast<uint32_t>(ex >> 32);
}

template <int ITEMS>
__device__ __forceinline__ void radix_scatter(const uint32_t (&e)[ITEMS], const uint32_t (&rk)[ITEMS], int shift,
                                              const uint32_t* dh, uint32_t* out) {
  const uint32_t* mine = dh + warp_id() * kDhStride;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const uint32_t d = (e[k] >> shift) & (kRadixBins - 1);
    out[mine[d] + rk[k]] = e[k];
  }
}

// Tile descriptor the producer publishes with each staged tile.
struct TileDesc {
  uint64_t begin;     // first record (absolute)
  uint32_t cnt;       // records in the tile (0: no more work, exit)
  uint32_t node;
  uint64_t row;       // X row of the work item
  uint32_t fresh;     // first tile of its work item
  uint32_t pad;       // staging plan (tile_plan): which streams landed, their element shifts
};

// Staging plan of a tile, packed by the producer so the consumers do not
// recompute the Bulk16 supersets: bit 0 ids staged, bit 1 records staged
// (keys [+ values], or the pair stream), bits 8-11 / 12-15 / 16-19 the
// element shifts of ids / keys (pairs) / values.
__device__ __forceinline__ uint32_t tile_plan(bool i_ok, uint32_t i_sh, bool r_ok, uint32_t k_sh, uint32_t v_sh) {
  return (i_ok ? 1u : 0u) | (r_ok ? 2u : 0u) | (i_sh << 8) | (k_sh << 12) | (v_sh << 16);
}

// Producer (one thread of the producer warp): claims work items from the
// global counter *ctr (zeroed by the launcher; items listed longest first),
// keeps Cfg::kStages tiles in flight, publishes each tile's descriptor next
// to its data (the mbarrier phase that delivers the bytes also orders the
// descriptor: arrive = release, try_wait = acquire), and ends with an exit
// marker (cnt = 0).  A work item's tiles stay on one CTA, in order.
// A (key, value) record of the pair scratch layout (K == V): keys at even,
// values at odd K-words (sort_engine.cuh, SortEngine::aos).
template <typename K>
struct alignas(2 * sizeof(K)) Pair2 {
  K k, v;
};

// SA: the source is an array of Pair2<K> records (one bulk copy per tile
// into the key + value areas of the stage) instead of two SoA columns.
template <typename K, typename V, typename Cfg, bool SA = false>
__device__ __forceinline__ void dist_producer(unsigned char* smem, const K* __restrict__ sk, const V* __restrict__ sv,
                                              const uint16_t* __restrict__ ids, uint64_t n_src,
                                              const Work* __restrict__ work, uint32_t n_work, uint32_t* ctr,
                                              uint64_t* full, uint64_t* empty, TileDesc* sdesc, int dbg) {
  constexpr bool kHasV = Cfg::kValBytes > 0;
  constexpr int T = Cfg::kTile;
  constexpr int STAGES = Cfg::kStages;
  auto stI = [&](int b) { return reinterpret_cast<uint16_t*>(smem + b * Cfg::kSet); };
  auto stK = [&](int b) { return reinterpret_cast<K*>(smem + b * Cfg::kSet + Cfg::kBufI); };
  auto stV = [&](int b) { return reinterpret_cast<V*>(smem + b * Cfg::kSet + Cfg::kBufI + Cfg::kBufK); };
  auto claim = [&]() {   // next non-empty work item, or n_work
    uint32_t i;
    do {
      i = atomicAdd(ctr, 1u);
    } while (i < n_work && work[i].len == 0);
    return i;
  };
  const uint64_t pol = l2_evict_first_policy();
  const bool l2_hint = !(dbg & 8);   // SS_DIST_DEBUG bit 8: plain loads (measurement)
  uint32_t pwi = claim(), ptb = 0;
  Work pw, pwn;
  pw.len = 0;
  pwn.len = 0;
  if (pwi < n_work) pw = work[pwi];
  uint32_t pnext = pwi < n_work ? claim() : n_work;   // one item ahead
  if (pnext < n_work) pwn = work[pnext];
  for (uint32_t j = 0;; ++j) {
    const int b = j % STAGES;
    if (j >= STAGES) mbar_wait(&empty[b], ((j / STAGES) - 1) & 1);   // tile j - STAGES consumed
    if (pwi >= n_work) {   // exit marker
      sdesc[b].cnt = 0;
      mbar_arrive(&full[b]);
      return;
    }
    const uint64_t begin = pw.begin + ptb;
    const uint32_t cnt = min(static_cast<uint32_t>(T), pw.len - ptb);
    TileDesc d;
    d.begin = begin;
    d.cnt = cnt;
    d.node = pw.node;
    d.row = pw.row;
    d.fresh = ptb == 0;
    const Bulk16<uint16_t> bi(ids, n_src, begin, cnt);
    if constexpr (SA) {
      const Bulk16<Pair2<K>> bp(reinterpret_cast<const Pair2<K>*>(sk), n_src, begin, cnt);
      d.pad = tile_plan(bi.ok, bi.sh, bp.ok, bp.sh, 0);
    } else {
      const Bulk16<K> bk(sk, n_src, begin, cnt);
      const Bulk16<V> bv(sv, n_src, begin, cnt);
      d.pad = tile_plan(bi.ok, bi.sh, bk.ok && (!kHasV || bv.ok), bk.sh, kHasV ? bv.sh : 0);
    }
    sdesc[b] = d;
    if constexpr (SA) {   // pair records: one stream into the key + value areas
      const Bulk16<Pair2<K>> bp(reinterpret_cast<const Pair2<K>*>(sk), n_src, begin, cnt);
      fence_proxy_async();
      mbar_arrive_expect_tx(&full[b], bi.bytes + bp.bytes);
      if (bi.ok) bulk_g2s_hint(stI(b), bi.src, bi.bytes, &full[b], pol);
      if (bp.ok) bulk_g2s_hint(stK(b), bp.src, bp.bytes, &full[b], pol);
    } else {
      const Bulk16<K> bk(sk, n_src, begin, cnt);
      const Bulk16<V> bv(sv, n_src, begin, cnt);
      uint32_t bytes = bi.bytes + bk.bytes;
      if constexpr (kHasV) bytes += bv.bytes;
      fence_proxy_async();
      mbar_arrive_expect_tx(&full[b], bytes);
      if (l2_hint) {
        if (bi.ok) bulk_g2s_hint(stI(b), bi.src, bi.bytes, &full[b], pol);
        if (bk.ok) bulk_g2s_hint(stK(b), bk.src, bk.bytes, &full[b], pol);
        if constexpr (kHasV) {
          if (bv.ok) bulk_g2s_hint(stV(b), bv.src, bv.bytes, &full[b], pol);
        }
      } else {
        if (bi.ok) bulk_g2s(stI(b), bi.src, bi.bytes, &full[b]);
        if (bk.ok) bulk_g2s(stK(b), bk.src, bk.bytes, &full[b]);
        if constexpr (kHasV) {
          if (bv.ok) bulk_g2s(stV(b), bv.src, bv.bytes, &full[b]);
        }
      }
    }
    // L2 prefetch of the tile `pf` tiles ahead in this CTA's sequence (the
    // current work item, then the one already claimed): the bulk copy into
    // the stage then finds its lines in L2 instead of waiting behind the
    // scattered stores (c2 distribute 12.64 -> 12.35 ms at pf = 2; 3 and 4
    // tiles ahead were slower, 4-byte records did not gain; with evict_last
    // stores and an evict_last hint on the prefetch, one tile ahead is best:
    // 12.11 -> 11.96 ms).  SS_DIST_DEBUG bits 8-11 override pf (15 = off).
    constexpr uint32_t kPfDefault = sizeof(K) + Cfg::kValBytes >= 16 ? 1u : 0u;
    const uint32_t pf_dbg = (static_cast<uint32_t>(dbg) >> 8) & 15u;
    if (const uint32_t pf = pf_dbg == 15u ? 0u : pf_dbg ? pf_dbg : kPfDefault) {
      uint64_t fb = 0;
      uint32_t fc = 0;
      const uint64_t ahead = static_cast<uint64_t>(ptb) + static_cast<uint64_t>(pf) * T;
      if (ahead < pw.len) {
        fb = pw.begin + ahead;
        fc = static_cast<uint32_t>(min(static_cast<uint64_t>(T), pw.len - ahead));
      } else if (pnext < n_work) {
        const uint64_t rem = (static_cast<uint64_t>(pw.len - ptb) + T - 1) / T;   // tiles left in the item, this one included
        const uint64_t off = (pf - rem) * static_cast<uint64_t>(T);
        if (pf >= rem && off < pwn.len) {
          fb = pwn.begin + off;
          fc = static_cast<uint32_t>(min(static_cast<uint64_t>(T), pwn.len - off));
        }
      }
      if (fc) {
        // prefetched lines are evict_last until the stage copy (evict_first) takes them
        const uint64_t ppol = l2_evict_last_policy();
        auto bulk_prefetch_l2 = [&](const void* src, uint32_t bytes) { ss::bulk_prefetch_l2_hint(src, bytes, ppol); };
        const Bulk16<uint16_t> fi(ids, n_src, fb, fc);
        if (fi.ok) bulk_prefetch_l2(fi.src, fi.bytes);
        if constexpr (SA) {
          const Bulk16<Pair2<K>> fp(reinterpret_cast<const Pair2<K>*>(sk), n_src, fb, fc);
          if (fp.ok) bulk_prefetch_l2(fp.src, fp.bytes);
        } else {
          const Bulk16<K> fk(sk, n_src, fb, fc);
          if (fk.ok) bulk_prefetch_l2(fk.src, fk.bytes);
          if constexpr (kHasV) {
            const Bulk16<V> fv(sv, n_src, fb, fc);
            if (fv.ok) bulk_prefetch_l2(fv.src, fv.bytes);
          }
        }
      }
    }
    ptb += T;
    if (ptb >= pw.len) {   // advance to the prefetched item, prefetch the next
      pwi = pnext;
      pw = pwn;
      ptb = 0;
      if (pwi < n_work) {
        pnext = claim();
        if (pnext < n_work) pwn = work[pnext];
      }
    }
  }
}

// ids: u16 bucket id per source record (absolute index), written by the
// count pass.  Buckets kept: [0, nb) with nb = min(fixed_nb or
// n_light + node.n_heavy, keep_below); others are dropped.  n_src: element
// count of the source arrays (bounds of the aligned TMA supersets).
//
// NT consumer threads + one producer warp (dist_producer).  A work item's
// tiles stay on one CTA, in order: its X-row cursors advance tile by tile,
// which keeps the scatter stable.  This two-pass LSD kernel is the general
// path; dist1.cuh's single-pass kernel serves when its tables fit.
template <typename K, typename V, int TILE, int NT, int STAGES, bool HW>
__global__ void __launch_bounds__(NT + 32, 1)   // 17 warps: one sub-partition holds 5 -> <= 96 registers

k_distribute(const K* __restrict__ sk, const V* __restrict__ sv, const uint16_t* __restrict__ ids, uint64_t n_src,
             K* __restrict__ dk, V* __restrict__ dv, const Work* __restrict__ work, uint32_t n_work,
             const Node* __restrict__ nodes, const uint64_t* __restrict__ X, uint32_t stride, uint32_t keep_below,
             uint32_t n_light, uint32_t fixed_nb, uint32_t* __restrict__ ctr) {
  using Cfg = DistCfg<K, V, TILE, NT, STAGES>;
  constexpr int kDistThreads = NT;
  constexpr int kDistWarps = NT / 32;
  constexpr bool kHasV = Cfg::kValBytes > 0;
  constexpr int T = Cfg::kTile;
  constexpr int ITEMS = Cfg::kItems;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long red64[33];
  __shared__ __align__(8) uint64_t full[STAGES];    // tile bytes landed (producer arrive + TMA tx)
  __shared__ __align__(8) uint64_t empty[STAGES];   // stage consumed (consumer thread 0 arrive)
  __shared__ TileDesc sdesc[STAGES];

  // stage b: [ids | keys | values] at smem + b * kSet (arithmetic keeps the
  // shared address space visible to the compiler: LDS, no local arrays)
  auto stI = [&](int b) { return reinterpret_cast<uint16_t*>(smem + b * Cfg::kSet); };
  auto stK = [&](int b) { return reinterpret_cast<K*>(smem + b * Cfg::kSet + Cfg::kBufI); };
  auto stV = [&](int b) { return reinterpret_cast<V*>(smem + b * Cfg::kSet + Cfg::kBufI + Cfg::kBufK); };
  unsigned char* p = smem + STAGES * Cfg::kSet;
  uint32_t* srtA = reinterpret_cast<uint32_t*>(p); p += T * 4;
  uint32_t* srtB = reinterpret_cast<uint32_t*>(p); p += T * 4;
  uint64_t* cursor = reinterpret_cast<uint64_t*>(p); p += Cfg::up16(static_cast<size_t>(stride) * 8);
  uint64_t* wbase = reinterpret_cast<uint64_t*>(p); p += Cfg::up16(static_cast<size_t>(stride) * 8);
  uint32_t* hist = reinterpret_cast<uint32_t*>(p); p += Cfg::up16(static_cast<size_t>(stride) * 4);
  uint32_t* dh = reinterpret_cast<uint32_t*>(p);
  uint32_t* pm = dh + kDistWarps * kDhStride;
  for (int i = threadIdx.x; i < kDistWarps * kDhStride; i += blockDim.x) pm[i] = 0;
  const int dbg = g_dist_debug;
  const int w = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int b = 0; b < STAGES; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // ---- producer warp (lane 0): claims work items, stages tiles ----
  if (w == kDistWarps) {
    if (lane == 0) dist_producer<K, V, Cfg>(smem, sk, sv, ids, n_src, work, n_work, ctr, full, empty, sdesc, dbg);
    return;
  }

  uint32_t nb = 0;
  const bool prof = (dbg & 4) && threadIdx.x == 0;
  unsigned long long pacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tlast = prof ? clock64() : 0;
  auto mark = [&](int ph) {
    if (prof) {
      const unsigned long long t = clock64();
      pacc[ph] += t - tlast;
      tlast = t;
    }
  };
  for (uint32_t q = 0;; ++q) {
    const int buf = q % STAGES;
    mark(9);
    mbar_wait(&full[buf], (q / STAGES) & 1);
    const TileDesc td = sdesc[buf];
    if (td.cnt == 0) break;   // uniform: every thread read the same marker
    const uint64_t begin = td.begin;
    const uint32_t cnt = td.cnt;
    if (td.fresh) {   // new work item: its X row and bucket count
      nb = fixed_nb ? fixed_nb : n_light + nodes[td.node].n_heavy;
      if (nb > keep_below) nb = keep_below;
      const uint64_t* xrow = X + td.row * stride;
      for (uint32_t b = threadIdx.x; b < nb; b += kDistThreads) {
        cursor[b] = xrow[b];
        hist[b] = 0;
      }
    }
    const Bulk16<uint16_t> pi(ids, n_src, begin, cnt);
    const Bulk16<K> pk(sk, n_src, begin, cnt);
    const Bulk16<V> pv(sv, n_src, begin, cnt);
    const uint16_t* tI = stI(buf) + pi.sh;
    const K* tK = stK(buf) + pk.sh;
    const V* tV = stV(buf) + pv.sh;
    mark(0);
    csync<kDistWarps>();   // cursors and zeroed histogram visible
    mark(1);

    // ids -> histogram + (bucket << 12 | index) entries; pass-1 ranks
    uint32_t e[ITEMS], rk[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t i = w * (32 * ITEMS) + k * 32 + lane;
      uint32_t b = kSentinel;
      if (i < cnt) {
        b = pi.ok ? tI[i] : ids[begin + i];
        if (b >= nb) b = kSentinel;
        else atomicAdd(&hist[b], 1u);
      }
      e[k] = (b << kIdxBits) | i;
    }
    radix_rank<ITEMS, kDistWarps, HW>(e, kIdxBits, dh, pm, rk);
    csync<kDistWarps>();
    mark(2);
    // one fused scan: pass-1 digit bases and the histogram (bucket starts)
    const uint32_t per = (nb + kDistThreads - 1) / kDistThreads;
    const uint32_t b0 = min(nb, threadIdx.x * per), b1 = min(nb, b0 + per);
    uint32_t hl = 0;
    for (uint32_t b = b0; b < b1; ++b) hl += hist[b];
    uint32_t trun = radix_scan<kDistWarps>(dh, red64, hl);
    for (uint32_t b = b0; b < b1; ++b) {   // thread-owned buckets: no races
      const uint32_t h = hist[b];
      wbase[b] = cursor[b] - trun;
      cursor[b] += h;
      hist[b] = 0;
      trun += h;
    }
    csync<kDistWarps>();
    mark(3);
    radix_scatter<ITEMS>(e, rk, kIdxBits, dh, srtA);
    csync<kDistWarps>();
    mark(4);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) e[k] = srtA[w * (32 * ITEMS) + k * 32 + lane];
    radix_rank<ITEMS, kDistWarps, HW>(e, kIdxBits + kRadixBits, dh, pm, rk);
    csync<kDistWarps>();
    mark(5);
    radix_scan<kDistWarps>(dh, red64, 0);
    csync<kDistWarps>();
    mark(6);
    radix_scatter<ITEMS>(e, rk, kIdxBits + kRadixBits, dh, srtB);
    csync<kDistWarps>();
    mark(7);
    // contiguous per-bucket runs out of the staged tile
    if (pk.ok && (!kHasV || pv.ok) && !(dbg & 3)) {
      // batches of loads first (no branches between them), then the stores
      constexpr int kB = ITEMS >= 4 ? 4 : ITEMS;
#pragma unroll
      for (int k0 = 0; k0 < ITEMS; k0 += kB) {
        uint64_t dd[kB];
        K kk[kB];
        V vv[kB];
        bool ok[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
          const uint32_t s = threadIdx.x + (k0 + k) * kDistThreads;
          const uint32_t ent = srtB[s];
          const uint32_t b = ent >> kIdxBits, i = ent & ((1u << kIdxBits) - 1);
          ok[k] = b != kSentinel;
          dd[k] = wbase[ok[k] ? b : 0u] + s;
          kk[k] = tK[i];
          if constexpr (kHasV) vv[k] = tV[i];
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
          if (ok[k]) {
            dk[dd[k]] = kk[k];
            if constexpr (kHasV) dv[dd[k]] = vv[k];
          }
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const uint32_t s = threadIdx.x + k * kDistThreads;
        const uint32_t ent = srtB[s];
        const uint32_t b = ent >> kIdxBits;
        if (b == kSentinel) continue;
        const uint32_t i = ent & ((1u << kIdxBits) - 1);
        uint64_t d = wbase[b] + s;
        if (dbg & 2) d = begin + s;
        if (!(dbg & 1)) {
          dk[d] = pk.ok ? tK[i] : sk[begin + i];
          if constexpr (kHasV) dv[d] = pv.ok ? tV[i] : sv[begin + i];
        }
      }
    }
    csync<kDistWarps>();   // stage `buf` may be refilled; wbase / srtB / sdesc reusable
    if (threadIdx.x == 0) mbar_arrive(&empty[buf]);
    mark(8);
  }
  if (prof) {
    unsigned long long tot = 0;
    for (int p = 0; p < 10; ++p) {
      atomicAdd(&g_dist_prof[p], pacc[p]);
      tot += pacc[p];
    }
    atomicAdd(&g_dist_prof[10], 1ull);
    atomicMax(&g_dist_prof[11], tot);
  }
}

}  // namespace ss
