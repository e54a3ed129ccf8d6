// Single-pass blocked distributing (core.py:321-380, aggregate.py:172-193):
// the fast path of the stable scatter when its tables fit shared memory and
// every node's output range is below 2^32 records.
//
// Same pipeline as dist.cuh (persistent CTAs, a producer warp staging
// 4096-record tiles of [ids | keys | values] by TMA, dynamic claiming of
// work items), but each tile is ordered by bucket in ONE counting pass
// instead of two 7-bit LSD passes:
//   A. every warp walks its 256 records in index order; a shared atomicAdd
//      on the warp's private u16 counter of the record's bucket (two
//      buckets packed per word, +1 / +65536) returns the record's rank
//      among the warp's earlier records of that bucket -- in lane order
//      within one instruction on sm_100 (probe.cuh checks it at load time;
//      without it dist.cuh's kernel runs instead);
//   B. per bucket, an exclusive scan over the warps' counters plus one
//      CTA scan of the bucket totals turn counters into tile positions
//      (bucket start + earlier warps), and advance the row cursors;
//   C. records scatter their (bucket, index) into the sorted order;
//   D. threads write sorted positions, so lanes emit contiguous per-bucket
//      runs, and re-zero their counters.
// Positions are row-relative u32 (X[row][0] + offset): 5 barriers per
// tile instead of 9, and the counters replace the radix buffers.
// key_below: keys of buckets >= key_below are not written (semisort's heavy
// buckets hold one key; the copy-back fills it, k_copy_heavy_fill).
#pragma once

#include <type_traits>

#include "dist.cuh"

namespace ss {

template <typename K, typename V, int TILE, int NT, int STAGES>
struct Dist1Cfg : DistCfg<K, V, TILE, NT, STAGES> {
  using Base = DistCfg<K, V, TILE, NT, STAGES>;
  static constexpr int kWarps = NT / 32;
  // counter pairs a thread owns in the per-bucket scan: 2 (uint2 rows) at
  // 512 consumer threads, 4 (uint4 rows) at 256
  static constexpr int kQP = NT >= 512 ? 2 : 4;
  // u16 counter pairs per warp row: ceil(nb / 2) rounded up to kQP (vector loads)
  __host__ __device__ static uint32_t pair_stride(uint32_t stride) {
    return ((stride + 1) / 2 + kQP - 1) & ~static_cast<uint32_t>(kQP - 1);
  }
  static size_t smem_bytes(uint32_t stride) {
    return STAGES * Base::kSet + static_cast<size_t>(TILE) * 4 + 2 * Base::up16(static_cast<size_t>(stride) * 4) +
           static_cast<size_t>(kWarps) * pair_stride(stride) * 4 + 64;
  }
};

// Store with an L2 eviction policy (8- and 16-byte values; others plain).
template <typename T>
__device__ __forceinline__ void st_pol(T* p, const T& v, uint64_t pol) {
  if constexpr (sizeof(T) == 16) {
    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(&v);
    asm volatile("st.global.L2::cache_hint.v2.b64 [%0], {%1, %2}, %3;" ::"l"(p), "l"(u.x), "l"(u.y), "l"(pol) : "memory");
  } else if constexpr (sizeof(T) == 8) {
    const unsigned long long u = *reinterpret_cast<const unsigned long long*>(&v);
    asm volatile("st.global.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(u), "l"(pol) : "memory");
  } else if constexpr (sizeof(T) == 4) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(&v);
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(u), "l"(pol) : "memory");
  } else {
    *p = v;
  }
}

// SA: source in the pair scratch layout (keys at even, values at odd
// K-words; sk points at the first key, sv is unused); DA: destination in
// the pair layout -- a light record leaves as ONE 16-byte (8-byte for u32)
// store instead of two partial-sector stores, a heavy record writes only
// its value at K-word hbase + d of the pair array, hbase = start of the
// node's heavy region, so a node's heavy values lie contiguous inside its
// heavy region's own words [2 hbase, hbase + h1) (the copy-back streams them;
// keys are filled there).  Both need V == K.
// MINB: CTAs per SM (2 with NT = 256: two independent consumer groups per SM)
template <typename K, typename V, int TILE, int NT, int STAGES, bool SA = false, bool DA = false, int MINB = 1>
__global__ void __launch_bounds__(NT + 32, MINB)   // 17 warps: one sub-partition holds 5 -> <= 96 registers

k_distribute1(const K* __restrict__ sk, const V* __restrict__ sv, const uint16_t* __restrict__ ids, uint64_t n_src,
              K* __restrict__ dk, V* __restrict__ dv, const Work* __restrict__ work, uint32_t n_work,
              const Node* __restrict__ nodes, const uint64_t* __restrict__ X, uint32_t stride, uint32_t keep_below,
              uint32_t n_light, uint32_t fixed_nb, uint32_t* __restrict__ ctr, uint32_t key_below,
              uint32_t cstride) {   // cstride: shared counter / cursor rows (>= every work item's nb)
  using Cfg = Dist1Cfg<K, V, TILE, NT, STAGES>;
  constexpr int NW = NT / 32;
  constexpr bool kHasV = Cfg::kValBytes > 0;
  constexpr int T = TILE;
  constexpr int ITEMS = T / NT;
  static_assert(T <= 8192 && ITEMS * NT == T, "tile index is 12 or 13 bits");
  constexpr uint32_t IB = T <= 4096 ? kIdxBits : kIdxBits + 1;   // (bucket << IB) | index
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long red64[33];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ TileDesc sdesc[STAGES];

  auto stI = [&](int b) { return reinterpret_cast<uint16_t*>(smem + b * Cfg::kSet); };
  auto stK = [&](int b) { return reinterpret_cast<K*>(smem + b * Cfg::kSet + Cfg::kBufI); };
  auto stV = [&](int b) { return reinterpret_cast<V*>(smem + b * Cfg::kSet + Cfg::kBufI + Cfg::kBufK); };
  const uint32_t pstride = Cfg::pair_stride(cstride);
  unsigned char* p = smem + STAGES * Cfg::kSet;
  uint32_t* srt = reinterpret_cast<uint32_t*>(p); p += T * 4;
  uint32_t* cursor = reinterpret_cast<uint32_t*>(p); p += Cfg::up16(static_cast<size_t>(cstride) * 4);
  uint32_t* wbase = reinterpret_cast<uint32_t*>(p); p += Cfg::up16(static_cast<size_t>(cstride) * 4);
  uint32_t* cntw = reinterpret_cast<uint32_t*>(p);   // [NW][pstride] u16 pairs
  for (uint32_t i = threadIdx.x; i < NW * pstride; i += blockDim.x) cntw[i] = 0;
  const int dbg = g_dist_debug;
  // The scattered stores keep their lines in L2 (evict_last) until the
  // work item's following tiles have completed them; the streamed input is
  // evict_first (dist_producer).  Measured against plain stores: c3
  // distribute 9.98 -> 9.50 ms, c2 12.62 -> 12.28; evict_first and
  // evict_unchanged on the stores: no change.
  uint64_t spol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(spol));
  const int w = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int b = 0; b < STAGES; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (w == NW) {
    if (lane == 0) dist_producer<K, V, Cfg, SA>(smem, sk, sv, ids, n_src, work, n_work, ctr, full, empty, sdesc, dbg);
    return;
  }

  uint32_t nb = 0, npairs = 0;
  uint64_t rbase = 0;   // X[row][0]: positions below are relative to it
  uint64_t hbase = 0;   // DA: start of the node's heavy region (X[node's first row][n_light])
  uint32_t* mine = cntw + w * pstride;
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
    mbar_wait(&full[buf], (q / STAGES) & 1);
    const TileDesc td = sdesc[buf];
    if (td.cnt == 0) break;
    const uint64_t begin = td.begin;
    const uint32_t cnt = td.cnt;
    if (td.fresh) {   // new work item: its X row (row-relative) and bucket count
      nb = fixed_nb ? fixed_nb : n_light + nodes[td.node].n_heavy;
      if (nb > keep_below) nb = keep_below;
      npairs = (nb + 1) >> 1;
      const uint64_t* xrow = X + td.row * stride;
      rbase = xrow[0];   // bucket-major layout: bucket 0's cursor is the row minimum
      if constexpr (DA) hbase = n_light < nb ? X[static_cast<uint64_t>(nodes[td.node].row_base) * stride + n_light] : 0;
      for (uint32_t b = threadIdx.x; b < nb; b += NT) cursor[b] = static_cast<uint32_t>(xrow[b] - rbase);
    }
    static_assert(!(SA || DA) || (sizeof(K) == sizeof(V) && ValTraits<V>::bytes == sizeof(K)), "pair layout needs V == K");
    // staging plan from the producer (tile_plan): staged streams and shifts
    const uint32_t plan = td.pad;
    const bool i_ok = plan & 1u;
    const bool staged = (plan >> 1) & 1u;
    const uint32_t i_sh = (plan >> 8) & 15u, k_sh = (plan >> 12) & 15u, v_sh = (plan >> 16) & 15u;
    const Pair2<K>* gP = reinterpret_cast<const Pair2<K>*>(sk);
    const Pair2<K>* tP = reinterpret_cast<const Pair2<K>*>(stK(buf)) + k_sh;
    auto rec_key = [&](uint32_t i) -> K {   // record i of the tile, staged or from global
      if constexpr (SA) return staged ? tP[i].k : gP[begin + i].k;
      else return staged ? stK(buf)[k_sh + i] : sk[begin + i];
    };
    auto rec_val = [&](uint32_t i) -> V {
      if constexpr (SA) return static_cast<V>(staged ? tP[i].v : gP[begin + i].v);
      else return staged ? stV(buf)[v_sh + i] : sv[begin + i];
    };
    const uint16_t* tI = stI(buf) + i_sh;
    mark(0);

    // A. in-warp ranks: old value of the warp's packed counter
    uint32_t bk[ITEMS], rk[ITEMS];
    if (cnt == T && i_ok) {   // full staged tile: no bounds or source checks
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        uint32_t b = tI[w * (32 * ITEMS) + k * 32 + lane];
        b = b < nb ? b : kSentinel;
        bk[k] = b;
        rk[k] = 0;
        if (b != kSentinel) {
          const uint32_t sh = (b & 1u) << 4;
          rk[k] = (atomicAdd(&mine[b >> 1], 1u << sh) >> sh) & 0xFFFFu;
        }
        __syncwarp();   // item k's increments precede item k+1's
      }
    } else {
#pragma unroll
      for (int k = 0; k < ITEMS; ++k) {
        const uint32_t i = w * (32 * ITEMS) + k * 32 + lane;
        uint32_t b = kSentinel;
        if (i < cnt) {
          b = i_ok ? tI[i] : ids[begin + i];
          if (b >= nb) b = kSentinel;
        }
        bk[k] = b;
        rk[k] = 0;
        if (b != kSentinel) {
          const uint32_t sh = (b & 1u) << 4;
          rk[k] = (atomicAdd(&mine[b >> 1], 1u << sh) >> sh) & 0xFFFFu;
        }
        __syncwarp();   // item k's increments precede item k+1's
      }
    }
    csync<NW>();
    mark(2);

    // B. per bucket pair: exclusive scan over warps, then over buckets.
    //    Thread t owns pairs 2t, 2t+1 (one uint2 per warp row);
    //    thread-contiguous pairs keep the CTA scan in bucket order.
    uint32_t n_valid;
    constexpr int QP = Cfg::kQP;
    using QV = std::conditional_t<QP == 2, uint2, uint4>;
    if (npairs <= QP * NT) {
      // thread t owns pairs QP t .. QP t + QP - 1 (one vector per warp row);
      // thread-contiguous pairs keep the CTA scan in bucket order
      const uint32_t j0 = QP * threadIdx.x;
      const bool own = j0 < npairs;
      uint32_t lo[QP], hi[QP];
#pragma unroll
      for (int q = 0; q < QP; ++q) lo[q] = hi[q] = 0;
#pragma unroll
      for (int v = 0; v < NW; ++v) {
        QV c{};
        if (own) c = *reinterpret_cast<const QV*>(cntw + v * pstride + j0);
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(&c);
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          lo[q] += cw[q] & 0xFFFFu;
          hi[q] += cw[q] >> 16;
        }
      }
      uint32_t mine_tot = 0;
#pragma unroll
      for (int q = 0; q < QP; ++q) mine_tot += lo[q] + hi[q];
      unsigned long long total64;
      uint32_t a = static_cast<uint32_t>(cscan_u64<NW>(mine_tot, red64, total64));
      n_valid = static_cast<uint32_t>(total64);
      if (own) {
        uint32_t st[QP];   // packed tile starts of each owned pair (low | high << 16)
        // the owned buckets' cursors as one vector per thread (scalar accesses
        // at a stride of 2 QP words were 2 QP-way bank conflicts); entries at
        // or past nb are padding of the 16-byte rounded rows
        static_assert(QP == 2, "cursor rows are padded to 4 words: one uint4 (two pairs) per thread");
        using CV = uint4;
        constexpr int kCV = 1;
        CV cur[kCV], wb[kCV];
#pragma unroll
        for (int c = 0; c < kCV; ++c) cur[c] = reinterpret_cast<const CV*>(cursor + 2 * j0)[c];
        uint32_t* cw = reinterpret_cast<uint32_t*>(cur);
        uint32_t* ww = reinterpret_cast<uint32_t*>(wb);
#pragma unroll
        for (int q = 0; q < QP; ++q) {
          const uint32_t alo = a, ahi = a + lo[q];
          a = ahi + hi[q];
          st[q] = alo | (ahi << 16);
          ww[2 * q] = cw[2 * q] - alo;   // modular: cursor + (s - start) below
          cw[2 * q] += lo[q];
          ww[2 * q + 1] = cw[2 * q + 1] - ahi;
          cw[2 * q + 1] += hi[q];
        }
#pragma unroll
        for (int c = 0; c < kCV; ++c) {
          reinterpret_cast<CV*>(wbase + 2 * j0)[c] = wb[c];
          reinterpret_cast<CV*>(cursor + 2 * j0)[c] = cur[c];
        }
#pragma unroll
        for (int v = 0; v < NW; ++v) {   // tile position of warp v's first record per bucket
          QV* cp = reinterpret_cast<QV*>(cntw + v * pstride + j0);
          QV c = *cp, o;
          const uint32_t* cw = reinterpret_cast<const uint32_t*>(&c);
          uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
          for (int q = 0; q < QP; ++q) {
            ow[q] = st[q];
            st[q] += cw[q];   // both halves advance; no carry (positions < 2^16)
          }
          *cp = o;
        }
      }
    } else {   // many buckets: contiguous chunks of pairs, counters re-read
      const uint32_t per = (npairs + NT - 1) / NT;
      const uint32_t j0 = min(npairs, threadIdx.x * per), j1 = min(npairs, j0 + per);
      uint32_t tot_local = 0;
      for (uint32_t j = j0; j < j1; ++j)
#pragma unroll
        for (int v = 0; v < NW; ++v) {
          const uint32_t cv = cntw[v * pstride + j];
          tot_local += (cv & 0xFFFFu) + (cv >> 16);
        }
      unsigned long long total64;
      uint32_t run = static_cast<uint32_t>(cscan_u64<NW>(tot_local, red64, total64));
      n_valid = static_cast<uint32_t>(total64);
      for (uint32_t j = j0; j < j1; ++j) {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int v = 0; v < NW; ++v) {
          const uint32_t cv = cntw[v * pstride + j];
          lo += cv & 0xFFFFu;
          hi += cv >> 16;
        }
        uint32_t alo = run, ahi = run + lo;
        const uint32_t b0 = 2 * j;
        wbase[b0] = cursor[b0] - alo;
        cursor[b0] += lo;
        if (b0 + 1 < nb) {
          wbase[b0 + 1] = cursor[b0 + 1] - ahi;
          cursor[b0 + 1] += hi;
        }
#pragma unroll
        for (int v = 0; v < NW; ++v) {
          const uint32_t cv = cntw[v * pstride + j];
          cntw[v * pstride + j] = alo | (ahi << 16);
          alo += cv & 0xFFFFu;
          ahi += cv >> 16;
        }
        run += lo + hi;
      }
    }
    csync<NW>();
    mark(3);

    // C. scatter (bucket << 12 | index) into the sorted order
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint32_t b = bk[k];
      if (b == kSentinel) continue;
      const uint32_t sh = (b & 1u) << 4;
      const uint32_t s = ((mine[b >> 1] >> sh) & 0xFFFFu) + rk[k];
      srt[s] = (b << IB) | (w * (32 * ITEMS) + k * 32 + lane);
    }
    csync<NW>();
    mark(4);

    // D. sorted write-out (contiguous per-bucket runs); re-zero counters
    if (npairs <= QP * NT) {
      const uint32_t j0 = QP * threadIdx.x;
      if (j0 < npairs)
#pragma unroll
        for (int v = 0; v < NW; ++v) *reinterpret_cast<QV*>(cntw + v * pstride + j0) = QV{};
    } else {
      for (uint32_t j = threadIdx.x; j < npairs; j += NT)
#pragma unroll
        for (int v = 0; v < NW; ++v) cntw[v * pstride + j] = 0;
    }
    if (staged && !(dbg & 3)) {
      constexpr int kB = ITEMS >= 4 ? 4 : ITEMS;
#pragma unroll
      for (int k0 = 0; k0 < ITEMS; k0 += kB) {
        uint64_t dd[kB];
        K kk[kB];
        V vv[kB];
        bool ok[kB], wk[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
          const uint32_t s = threadIdx.x + (k0 + k) * NT;
          ok[k] = s < n_valid;
          const uint32_t ent = ok[k] ? srt[s] : 0u;   // srt beyond n_valid is stale
          const uint32_t b = ent >> IB, i = ent & ((1u << IB) - 1);
          wk[k] = ok[k] && b < key_below;
          dd[k] = rbase + static_cast<uint32_t>(wbase[b] + s);
          kk[k] = rec_key(i);
          if constexpr (kHasV) vv[k] = rec_val(i);
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
          if constexpr (DA) {
            Pair2<K>* dP = reinterpret_cast<Pair2<K>*>(dk);
            if (wk[k]) st_pol(dP + dd[k], Pair2<K>{kk[k], static_cast<K>(vv[k])}, spol);
            else if (ok[k]) st_pol(reinterpret_cast<K*>(dk) + hbase + dd[k], static_cast<K>(vv[k]), spol);
          } else {
            if (wk[k]) st_pol(dk + dd[k], kk[k], spol);
            if constexpr (kHasV) {
              if (ok[k]) st_pol(dv + dd[k], vv[k], spol);
            }
          }
        }
      }
    } else {
      for (uint32_t s = threadIdx.x; s < n_valid; s += NT) {
        const uint32_t ent = srt[s];
        const uint32_t b = ent >> IB, i = ent & ((1u << IB) - 1);
        uint64_t d = rbase + static_cast<uint32_t>(wbase[b] + s);
        if (dbg & 2) d = begin + s;
        if (!(dbg & 1)) {
          if constexpr (DA) {
            if (b < key_below) reinterpret_cast<Pair2<K>*>(dk)[d] = Pair2<K>{rec_key(i), static_cast<K>(rec_val(i))};
            else reinterpret_cast<K*>(dk)[hbase + d] = static_cast<K>(rec_val(i));
          } else {
            if (b < key_below) dk[d] = rec_key(i);
            if constexpr (kHasV) dv[d] = rec_val(i);
          }
        }
      }
    }
    csync<NW>();   // stage, srt, wbase and sdesc reusable; counters zero
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
