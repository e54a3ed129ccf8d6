// Level-synchronous semisort scheduler (core.py:437-598 re-designed for the
// GPU).
//
// The reference recurses node by node (big buckets sequentially,
// core.py:496-498).  Every node's result depends only on its own descriptor
// (range, depth, path, stall state), so we process all nodes of a recursion
// level together: one launch per phase for the whole level, with one
// device->host sync per level to learn the next level's node list.  Leaves
// (light buckets < alpha) are resolved right after the level that produced
// them.  Buffer roles follow core.py:117-131 / PAPER §3.4: level L reads A
// when L is odd and S when L is even; heavy buckets written to S are copied
// back, leaves living in S are written to A by their base case.
#pragma once

#include <cstdio>
#include <type_traits>
#include <vector>

#include "engine.cuh"
#include "leaf.cuh"
#include "leaf_lt.cuh"
#include "leaf_warp.cuh"
#include "dist1.cuh"
#include "multisplit.cuh"
#include "probe.cuh"
#include "sample.cuh"

namespace ss {

constexpr uint64_t kTargetRows = 148 * 32;   // subarrays per level (~32 per SM: dynamic scheduling granularity)
constexpr uint64_t kMinChunk = 4096;
constexpr uint32_t kSampleGridMax = 148;
constexpr uint32_t kLeafGlobalGridMax = 296;
constexpr size_t kSampleSmem = kSampleSmemCap * 4;

inline uint64_t lt_leaf_words(uint64_t m, int key_bytes) {
  return pow2_ge(std::max<uint64_t>(m, 1)) * (key_bytes + 4) / 4 + 16;
}

template <typename K, typename V, int TILE, int NT, int STAGES, bool HW>
inline void launch_distribute_t(const K* sk, const V* sv, const uint16_t* ids, uint64_t n_src, K* dk, V* dv,
                                const Work* d_work, uint32_t nwork, const Node* d_nodes, const uint64_t* d_X,
                                uint32_t stride, uint32_t keep_below, uint32_t n_light, uint32_t fixed_nb,
                                cudaStream_t st, uint32_t* ctr) {
  const size_t dsm = DistCfg<K, V, TILE, NT, STAGES>::smem_bytes(stride);
  auto kern = k_distribute<K, V, TILE, NT, STAGES, HW>;
  SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm)));
  int per_sm = 0;
  SS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT + 32, dsm));
  const uint32_t grid = std::min<uint32_t>(nwork, 148u * static_cast<uint32_t>(std::max(per_sm, 1)));
  SS_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
  kern<<<grid, NT + 32, dsm, st>>>(sk, sv, ids, n_src, dk, dv, d_work, nwork, d_nodes, d_X, stride, keep_below, n_light,
                              fixed_nb, ctr);
  check_launch();
}

template <typename K, typename V, int TILE, bool SA, bool DA, int STAGES = 2>
inline void launch_distribute1_t(const K* sk, const V* sv, const uint16_t* ids, uint64_t n_src, K* dk, V* dv,
                                 const Work* d_work, uint32_t nwork, const Node* d_nodes, const uint64_t* d_X,
                                 uint32_t stride, uint32_t keep_below, uint32_t n_light, uint32_t fixed_nb,
                                 cudaStream_t st, uint32_t* ctr, uint32_t key_below, uint32_t cstride) {
  const size_t dsm = Dist1Cfg<K, V, TILE, 512, STAGES>::smem_bytes(cstride);
  auto kern = k_distribute1<K, V, TILE, 512, STAGES, SA, DA>;
  SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm)));
  const uint32_t grid = std::min<uint32_t>(nwork, 148u);
  SS_CUDA(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
  kern<<<grid, 512 + 32, dsm, st>>>(sk, sv, ids, n_src, dk, dv, d_work, nwork, d_nodes, d_X, stride, keep_below,
                                    n_light, fixed_nb, ctr, key_below, cstride);
  check_launch();
}

// Which distribute kernel (SS_DIST_KERNEL=radix forces dist.cuh's; tests use it).
inline bool dist_radix_forced() {
  const char* e = std::getenv("SS_DIST_KERNEL");
  return e && std::strcmp(e, "radix") == 0;
}

// 8192-record tiles when a staged record is <= 8 bytes (measured: c4's u32
// distribute 7.1 -> 5.3 ms).  For 16-byte records the stage would not fit;
// an ids-only stage with the records prefetched into L2 and gathered by the
// write-out was measured slower than 4096 staged (c2 13.3 -> 15.6 ms), and
// so were three stages of 3072 (12.8 -> 14.1 ms; c3 10.1 -> 11.0 ms).
template <typename K, typename V>
constexpr bool kDist8k = sizeof(K) + ValTraits<V>::bytes <= 8;

// Tile of the single-pass kernel for this launch, 0 when the radix kernel
// serves it (no hardware rank order, positions beyond u32, tables too big).
template <typename K, typename V>
inline int dist1_tile(uint32_t stride, uint64_t n_src) {
  if (!hw_rank_ok() || dist_radix_forced() || n_src > 0xFFFFFFFFull) return 0;
  if constexpr (kDist8k<K, V>)   // small records: twice the records per tile, longer per-bucket runs
    if (Dist1Cfg<K, V, 8192, 512, 2>::smem_bytes(stride) <= kMaxDynSmem) return 8192;
  if (Dist1Cfg<K, V, 4096, 512, 2>::smem_bytes(stride) <= kMaxDynSmem) return 4096;
  if (Dist1Cfg<K, V, 2048, 512, 2>::smem_bytes(stride) <= kMaxDynSmem) return 2048;
  return 0;
}

// Stable scatter of every work item through its X row, by the u16 bucket
// ids `ids` the count pass stored; n_src = element count of the sources;
// ctr = one workspace word (the dynamic work counter, zeroed here).
// key_below: heavy buckets (>= key_below) do not write keys.  src_pairs /
// dst_pairs: that side is the pair scratch layout (K == V, single-pass
// kernel only; the caller checks dist1_tile).
template <typename K, typename V>
inline void launch_distribute(const K* sk, const V* sv, const uint16_t* ids, K* dk, V* dv, const Work* d_work,
                              uint32_t nwork, const Node* d_nodes, const uint64_t* d_X, uint32_t stride,
                              uint32_t keep_below, uint32_t n_light, uint32_t fixed_nb, cudaStream_t st,
                              uint64_t n_src, uint32_t* ctr, uint32_t key_below = 0xFFFFFFFFu,
                              bool src_pairs = false, bool dst_pairs = false, uint32_t max_nb = 0) {
  if (!nwork) return;
  // shared counter rows: the largest bucket count a work item can have
  // (max_nb: n_light + the level's largest n_heavy, when the caller knows it)
  uint32_t cstride = stride;
  if (fixed_nb && fixed_nb < cstride) cstride = fixed_nb;
  if (keep_below < cstride) cstride = keep_below;
  if (max_nb && max_nb < cstride) cstride = max_nb;
  cstride = std::max<uint32_t>(2, std::min<uint32_t>(stride, (cstride + 1) & ~1u));
  static const int dbg = [] {
    const char* e = std::getenv("SS_DIST_DEBUG");
    const int v = e ? std::atoi(e) : 0;
    cudaMemcpyToSymbol(g_dist_debug, &v, sizeof(int));
    return v;
  }();
  (void)dbg;
  if (stride >= kMaxDistBuckets) throw Fail(SS_ERR_CONFIG, "too many buckets for the GPU distribute");
#define SS_DIST_ARGS \
  sk, sv, ids, n_src, dk, dv, d_work, nwork, d_nodes, d_X, stride, keep_below, n_light, fixed_nb, st, ctr
  const int t1 = dist1_tile<K, V>(cstride, n_src);
  if (t1) {
    auto go = [&]<int TILE>() {
      if constexpr (std::is_same_v<K, V>) {
        if (src_pairs && dst_pairs)
          return launch_distribute1_t<K, V, TILE, true, true>(SS_DIST_ARGS, key_below, cstride);
        if (src_pairs) return launch_distribute1_t<K, V, TILE, true, false>(SS_DIST_ARGS, key_below, cstride);
        if (dst_pairs) return launch_distribute1_t<K, V, TILE, false, true>(SS_DIST_ARGS, key_below, cstride);
      }
      launch_distribute1_t<K, V, TILE, false, false>(SS_DIST_ARGS, key_below, cstride);
    };
    bool done = false;
    if constexpr (kDist8k<K, V>) {
      if (t1 == 8192) {
        go.template operator()<8192>();
        done = true;
      }
    }
    if (done) {
    } else if (t1 == 4096) go.template operator()<4096>();
    else go.template operator()<2048>();
  } else {
    if (src_pairs || dst_pairs) throw Fail(SS_ERR_RESOURCE, "pair scratch layout needs the single-pass distribute");
    const bool hw = hw_rank_ok();
    switch (dist_tile_for<K, V>(stride)) {
      case 4096:
        hw ? launch_distribute_t<K, V, 4096, 512, 2, true>(SS_DIST_ARGS)
           : launch_distribute_t<K, V, 4096, 512, 2, false>(SS_DIST_ARGS);
        break;
      case 2048:
        hw ? launch_distribute_t<K, V, 2048, 512, 2, true>(SS_DIST_ARGS)
           : launch_distribute_t<K, V, 2048, 512, 2, false>(SS_DIST_ARGS);
        break;
      default:
        hw ? launch_distribute_t<K, V, 1024, 512, 2, true>(SS_DIST_ARGS)
           : launch_distribute_t<K, V, 1024, 512, 2, false>(SS_DIST_ARGS);
    }
  }
#undef SS_DIST_ARGS
  if (dbg & 4) {   // phase profile of this launch on stderr
    unsigned long long pr[12];
    SS_CUDA(cudaStreamSynchronize(st));
    SS_CUDA(cudaMemcpyFromSymbol(pr, g_dist_prof, sizeof(pr)));
    static const char* names[10] = {"top", "wait", "rank1", "scan1", "scat1", "rank2", "scan2", "scat2", "write",
                                    "issue"};
    unsigned long long tot = 0;
    for (int p = 0; p < 10; ++p) tot += pr[p];
    std::fprintf(stderr, "[dist_prof] nwork=%u ctas=%llu cyc/cta avg=%.0f max=%llu |", nwork, pr[10],
                 double(tot) / double(pr[10] ? pr[10] : 1), pr[11]);
    for (int p = 0; p < 10; ++p)
      std::fprintf(stderr, " %s %.1f%%", names[p], 100.0 * double(pr[p]) / double(tot ? tot : 1));
    std::fprintf(stderr, "\n");
    const unsigned long long zero[12] = {};
    SS_CUDA(cudaMemcpyToSymbol(g_dist_prof, zero, sizeof(zero)));
  }
}

// Measurement knob (SS_LEAF_STATS=1): leaf size histogram per launch on stderr.
inline void leaf_stats(const char* what, const Leaf* d_list, uint64_t count, cudaStream_t st) {
  static const bool on = std::getenv("SS_LEAF_STATS") != nullptr;
  if (!on || !count) return;
  std::vector<Leaf> h(count);
  SS_CUDA(cudaMemcpyAsync(h.data(), d_list, count * sizeof(Leaf), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  uint64_t bins[16] = {}, recs = 0;
  for (const Leaf& l : h) {
    int b = 0;
    while (b < 15 && (1ull << b) < l.size) ++b;
    ++bins[b];
    recs += l.size;
  }
  std::fprintf(stderr, "[leaf_stats] %s leaves=%llu records=%llu |", what, (unsigned long long)count,
               (unsigned long long)recs);
  for (int b = 0; b < 16; ++b)
    if (bins[b]) std::fprintf(stderr, " <=%llu:%llu", 1ull << b, (unsigned long long)bins[b]);
  std::fprintf(stderr, "\n");
}

template <typename K, typename V>
struct SortEngine {
  static constexpr bool kHasV = ValTraits<V>::bytes > 0;
  // inputs
  K* A_k;
  V* A_v;
  uint64_t n;
  int mode;
  int identity;
  Params P;
  cudaStream_t st;
  ss_telemetry* tel;
  // plan
  uint32_t stride = 0;
  uint64_t max_nodes = 0, max_rows = 0, max_grps = 0, max_leaves = 0, s_cap = 0, leafg_words = 0;
  uint32_t sample_grid = 0, leafg_grid = 0;
  // workspace
  K* S_k = nullptr;
  V* S_v = nullptr;
  // Pair scratch layout (K == V, chosen in run()): S holds (key, value)
  // records, S_k = record base, S_v = S_k + 1, element stride 2.  Light
  // records then leave the distribute as one 16-byte store instead of two
  // partial-sector stores (the level-0 store path of c2 was bound by them).
  bool aos = false;
  uint32_t s_ss() const { return aos ? 2u : 1u; }
  // where the copy-back reads heavy values: S_v, or the pair array's words
  V* heavy_src() const { return aos ? reinterpret_cast<V*>(S_k) : S_v; }
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
  uint32_t* d_ctr = nullptr;   // distribute work counter
  Leaf* d_leaf_w = nullptr;   // warp leaves (<= kLeafWarpMax)
  Leaf* d_leaf_s = nullptr;   // SMEM CTA leaves (<= kLeafSmemMax)
  Leaf* d_leaf_g = nullptr;   // global-scratch CTA leaves
  uint64_t* d_samp = nullptr;
  uint32_t* d_leafscr = nullptr;
  uint16_t* d_ids = nullptr;   // per-record bucket ids of the current level
  bool external_scratch = false;
  // Root source in the pair layout (ss_semisort_pairs): level 1 reads the
  // (key, value) records at R_pairs instead of A; A aliases that memory as
  // SoA columns and is first written by the root's heavy copy-back, after the
  // level-1 distribute has consumed every record of R (stream order).
  const K* R_pairs = nullptr;

  void plan(Arena& a, bool carve_scratch = true) {
    stride = even_stride(P);
    const uint64_t alpha = P.base_case_cutoff;
    max_nodes = std::max<uint64_t>(1, n / alpha);
    max_rows = std::min<uint64_t>(kTargetRows, cdiv(n, kMinChunk)) + max_nodes;   // rows <= R / chunk + nodes
    max_grps = max_rows / kRowGroup + max_nodes + 1;
    max_leaves = std::max<uint64_t>(1, std::min<uint64_t>(n, max_nodes * P.light_buckets));
    s_cap = std::max<uint64_t>(1, std::min<uint64_t>(n, P.sample_count));
    sample_grid = static_cast<uint32_t>(std::min<uint64_t>(kSampleGridMax, max_nodes));
    const uint64_t mmax = std::max<uint64_t>(1, std::min<uint64_t>(n, alpha > 1 ? alpha - 1 : 1));
    leafg_words = std::max(leaf_words(mmax, false), lt_leaf_words(mmax, sizeof(K)));
    leafg_grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kLeafGlobalGridMax, cdiv(n, kLeafSmemMax + 1))));
    if (carve_scratch) {
      if constexpr (std::is_same_v<K, V>) {   // one 2n-word block: SoA halves or pair records
        S_k = a.take<K>(2 * n);
        S_v = reinterpret_cast<V*>(S_k + n);
      } else {
        S_k = a.take<K>(n);
        if (kHasV) S_v = a.take<V>(n);
      }
    }
    d_nodes = a.take<Node>(max_nodes);
    d_next = a.take<Node>(max_nodes);
    d_heavy = a.take<KeyStore<K>>(max_nodes * std::max<uint32_t>(P.max_heavy, 1));
    d_work = a.take<Work>(max_rows);
    d_grp_node = a.take<uint32_t>(max_grps);
    d_C = a.take<uint32_t>(max_rows * stride);
    d_X = a.take<uint64_t>(max_rows * stride);
    d_P = a.take<uint64_t>(max_grps * stride);
    d_off = a.take<uint64_t>(max_nodes * (stride + 1));
    d_ccnt = a.take<uint32_t>(max_nodes * 4);
    d_misc = a.take<uint64_t>(8);
    d_ctr = a.take<uint32_t>(4);
    d_leaf_w = a.take<Leaf>(max_leaves);
    d_leaf_s = a.take<Leaf>(max_leaves);
    d_leaf_g = a.take<Leaf>(max_leaves);
    d_samp = a.take<uint64_t>(static_cast<uint64_t>(sample_grid) * sample_scratch_words(s_cap, sizeof(KeyStore<K>)));
    d_leafscr = a.take<uint32_t>(static_cast<uint64_t>(leafg_grid) * leafg_words);
    d_ids = a.take<uint16_t>(n);
  }

  bool src_is_A(int level, bool flip) const { return ((level & 1) == 1) != flip; }

  // ---- leaves ---------------------------------------------------------------
  void run_leaves_warp(Tracker& tr, const Leaf* d_list, uint64_t count, bool in_a) {
    if (!count) return;
    if (mode == SS_MODE_LT) {   // semisort<: (key, index) bitonic per warp
      const size_t sm = sizeof(LtWarpSmem<K, V>) * kLeafWarpWarps;
      SS_CUDA(cudaFuncSetAttribute(k_leaf_lt_warp<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(sm)));
      int per_sm = 0;
      SS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_leaf_lt_warp<K, V>, kLeafWarpWarps * 32, sm));
      const uint32_t grid = static_cast<uint32_t>(
          std::min<uint64_t>(cdiv(count, kLeafWarpWarps), 148u * std::max(per_sm, 1)));
      k_leaf_lt_warp<K, V><<<grid, kLeafWarpWarps * 32, sm, st>>>(in_a ? A_k : S_k, in_a ? A_v : S_v, A_k, A_v,
                                                                 d_list, static_cast<uint32_t>(count),
                                                                 in_a ? 1u : s_ss());
      check_launch();
      tr.launched();
      if (tel) tel->leaves_smem += count;
      return;
    }
    leaf_stats("warp", d_list, count, st);
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(cdiv(count, kLeafWarpWarps), 148 * 3));
    const size_t sm = sizeof(WarpLeafSmem<K>) * kLeafWarpWarps;
    SS_CUDA(cudaFuncSetAttribute(k_leaf_eq_warp<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    k_leaf_eq_warp<K, V><<<grid, kLeafWarpWarps * 32, sm, st>>>(in_a ? A_k : S_k, in_a ? A_v : S_v, A_k, A_v,
                                                               d_list, static_cast<uint32_t>(count), identity,
                                                               hw_rank_ok() ? 1 : 0, in_a ? 1u : s_ss());
    check_launch();
    tr.launched();
    if (tel) tel->leaves_smem += count;
  }

  void run_leaves_smem(Tracker& tr, const Leaf* d_list, uint64_t count, bool in_a) {
    if (!count) return;
    if (mode == SS_MODE_LT) {   // semisort<: (key, index) bitonic per CTA in shared memory
      const size_t sm = leaf_lt_smem_bytes<K, V>();
      auto kern = k_leaf_lt_smem<K, V>;
      SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
      int per_sm = 0;
      SS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLeafThreads, sm));
      const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(count, 148u * std::max(per_sm, 1)));
      kern<<<grid, kLeafThreads, sm, st>>>(in_a ? A_k : S_k, in_a ? A_v : S_v, A_k, A_v, d_list,
                                           static_cast<uint32_t>(count), in_a ? 1u : s_ss());
      check_launch();
      tr.launched();
      if (tel) tel->leaves_smem += count;
      return;
    }
    leaf_stats("smem", d_list, count, st);
    const size_t smem = leaf_smem_bytes(sizeof(K), kHasV ? sizeof(V) : 0);
    auto kern = k_leaf_eq_smem<K, V>;
    SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    SS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLeafThreads, smem));
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(count, 148u * std::max(per_sm, 1)));
    kern<<<grid, kLeafThreads, smem, st>>>(in_a ? A_k : S_k, in_a ? A_v : S_v, A_k, A_v, d_list,
                                           static_cast<uint32_t>(count), identity, hw_rank_ok() ? 1 : 0,
                                           in_a ? 1u : s_ss());
    check_launch();
    tr.launched();
    if (tel) tel->leaves_smem += count;
  }

  // Global-scratch leaves; scr == nullptr uses the planned scratch.
  void run_leaves_global(Tracker& tr, const Leaf* d_list, uint64_t count, bool in_a, uint32_t* scr,
                         uint64_t words, uint64_t max_size = ~0ull) {
    if (!count) return;
    leaf_stats("global", d_list, count, st);
    uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(count, leafg_grid));
    if (!scr) { scr = d_leafscr; words = leafg_words; }
    else grid = 1;
    if (mode == SS_MODE_LT) {
      k_leaf_lt<K, V><<<grid, kLeafThreads, 0, st>>>(S_k, S_v, A_k, A_v, d_list, static_cast<uint32_t>(count),
                                                    in_a, scr, words, aos ? 1 : 0);
    } else if (grid > 1) {   // planned mid leaves: shared-memory path up to kLeafMidMax
      auto launch = [&](auto kern, size_t sm, uint64_t lo, uint64_t hi) {
        SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        int per_sm = 0;
        SS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLeafThreads, sm));
        const uint32_t g = static_cast<uint32_t>(std::min<uint64_t>(count, 148u * std::max(per_sm, 1)));
        kern<<<std::min(g, grid), kLeafThreads, sm, st>>>(S_k, S_v, A_k, A_v, d_list, static_cast<uint32_t>(count),
                                                         in_a, identity, scr, words, hw_rank_ok() ? 1 : 0,
                                                         aos ? 1 : 0, lo, hi);
      };
      if constexpr (kLeafMidSmall < kLeafMidMax<K, V>) {
        // leaves <= 2048 records at two CTAs per SM, the larger rest (c5: 5%)
        // in a second launch of the one-CTA shape; each skips the other's
        launch(k_leaf_eq_mid<K, V, kLeafMidSmall>, leaf_mid_smem_bytes<K, V, kLeafMidSmall>(), 0, kLeafMidSmall);
        if (max_size > kLeafMidSmall)
          launch(k_leaf_eq_mid<K, V>, leaf_mid_smem_bytes<K, V>(), kLeafMidSmall + 1, ~0ull);
      } else {
        launch(k_leaf_eq_mid<K, V>, leaf_mid_smem_bytes<K, V>(), 0, ~0ull);
      }
    } else {
      k_leaf_eq_global<K, V><<<grid, kLeafThreads, 0, st>>>(S_k, S_v, A_k, A_v, d_list,
                                                            static_cast<uint32_t>(count), in_a, identity, scr, words,
                                                            hw_rank_ok() ? 1 : 0, aos ? 1 : 0);
    }
    check_launch();
    tr.launched();
    if (tel) tel->leaves_global += count;
  }

  // Leaves built on the host (root leaf, local_refine small buckets, forced
  // leaves after a stall / at DEPTH_LIMIT): any size.
  void run_host_leaves(Tracker& tr, const std::vector<Leaf>& leaves, bool in_a) {
    if (leaves.empty()) return;
    std::vector<Leaf> tiny, small, mid, huge;
    const uint64_t mmax_planned = std::max<uint64_t>(1, std::min<uint64_t>(n, P.base_case_cutoff > 1 ? P.base_case_cutoff - 1 : 1));
    for (const Leaf& l : leaves) {
      if (l.size <= kLeafWarpMax) tiny.push_back(l);
      else if (l.size <= kLeafSmemMax) small.push_back(l);
      else if (l.size <= mmax_planned) mid.push_back(l);
      else huge.push_back(l);
    }
    if (!tiny.empty()) {
      SS_CUDA(cudaMemcpyAsync(d_leaf_w, tiny.data(), tiny.size() * sizeof(Leaf), cudaMemcpyHostToDevice, st));
      run_leaves_warp(tr, d_leaf_w, tiny.size(), in_a);
    }
    if (!small.empty()) {
      SS_CUDA(cudaMemcpyAsync(d_leaf_s, small.data(), small.size() * sizeof(Leaf), cudaMemcpyHostToDevice, st));
      run_leaves_smem(tr, d_leaf_s, small.size(), in_a);
    }
    if (!mid.empty()) {
      SS_CUDA(cudaMemcpyAsync(d_leaf_g, mid.data(), mid.size() * sizeof(Leaf), cudaMemcpyHostToDevice, st));
      run_leaves_global(tr, d_leaf_g, mid.size(), in_a, nullptr, 0);
    }
    for (const Leaf& l : huge) {
      // rare: a stalled bucket larger than alpha; dedicated scratch
      const uint64_t words = std::max(leaf_words(l.size, false), lt_leaf_words(l.size, sizeof(K)));
      uint32_t* scr = nullptr;
      SS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scr), words * 4, st));
      SS_CUDA(cudaMemcpyAsync(d_leaf_g, &l, sizeof(Leaf), cudaMemcpyHostToDevice, st));
      run_leaves_global(tr, d_leaf_g, 1, in_a, scr, words);
      SS_CUDA(cudaFreeAsync(scr, st));
    }
    // the host vectors must outlive the async copies
    SS_CUDA(cudaStreamSynchronize(st));
  }

  // ---- one recursion level -------------------------------------------------
  std::vector<Node> level(Tracker& tr, std::vector<Node>& cur, int lvl, bool flip) {
    const bool from_a = src_is_A(lvl, flip);
    const bool from_r = R_pairs && lvl == 1 && !flip;   // root of ss_semisort_pairs
    const K* sk = from_r ? R_pairs : from_a ? A_k : S_k;
    const V* sv = from_r ? reinterpret_cast<const V*>(R_pairs + 1) : from_a ? A_v : S_v;
    K* dk = from_a ? S_k : A_k;
    V* dv = from_a ? S_v : A_v;
    const uint32_t nn = static_cast<uint32_t>(cur.size());

    uint64_t R = 0;
    for (auto& nd : cur) R += nd.size;
    const uint64_t chunk = (std::max<uint64_t>(kMinChunk, cdiv(R, kTargetRows)) + 7) & ~uint64_t(7);   // aligned items
    // rows per scan group: <= 128 groups per node (k_scan_nodes walks a node's
    // groups sequentially; 592 groups at the root cost 0.3 ms)
    uint64_t max_nrows = 0;
    for (auto& nd : cur) max_nrows = std::max<uint64_t>(max_nrows, cdiv(nd.size, chunk));
    const uint32_t rg = static_cast<uint32_t>(std::max<uint64_t>(kRowGroup, cdiv(max_nrows, 128)));
    std::vector<Work> work;
    std::vector<uint32_t> grp_node;
    for (uint32_t j = 0; j < nn; ++j) {
      Node& nd = cur[j];
      nd.out_base = nd.lo;
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
    // longest first: the distribute kernel claims work items dynamically
    std::stable_sort(work.begin(), work.end(), [](const Work& x, const Work& y) { return x.len > y.len; });
    const uint32_t nwork = static_cast<uint32_t>(work.size());
    const uint32_t ngrp = static_cast<uint32_t>(grp_node.size());
    tr.begin(kPhOther);
    SS_CUDA(cudaMemcpyAsync(d_nodes, cur.data(), nn * sizeof(Node), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemcpyAsync(d_work, work.data(), nwork * sizeof(Work), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemcpyAsync(d_grp_node, grp_node.data(), ngrp * sizeof(uint32_t), cudaMemcpyHostToDevice, st));

    // sampling + heavy tables
    tr.begin(kPhSample);
    SS_CUDA(cudaFuncSetAttribute(k_sample<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSampleSmem)));
    const uint32_t kss = from_r ? 2u : from_a ? 1u : s_ss();   // key stride of the source side
    k_sample<K><<<std::min<uint32_t>(sample_grid, nn), kSampleThreads, kSampleSmem, st>>>(
        sk, d_nodes, nn, d_heavy, d_samp, s_cap, P, 0, 0, kss);
    check_launch();
    tr.launched();

    using BF = KeyBucketsT<KeyStore<K>>;
    BF bf{};
    bf.heavy = d_heavy;
    bf.max_heavy = std::max<uint32_t>(P.max_heavy, 1);
    bf.n_light = P.light_buckets;
    bf.light_bits = P.light_bits;
    bf.identity = identity;

    // counting matrix
    tr.begin(kPhCount);
    k_count<K, BF><<<nwork, kCountThreads, stride * 4, st>>>(sk, d_work, nwork, d_nodes, d_C, stride, bf,
                                                                     d_ids, kss);
    check_launch();
    tr.launched();

    // column-major scan -> X, offsets
    tr.begin(kPhScan);
    k_colsum_groups<uint32_t><<<ngrp, 256, 0, st>>>(d_C, d_nodes, d_grp_node, ngrp, d_P, stride, P.light_buckets, 0, 0, rg);
    check_launch();
    k_scan_nodes<<<nn, 1024, 0, st>>>(d_nodes, nn, d_P, d_off, stride, P.light_buckets, 0, 0, nullptr);
    check_launch();
    k_write_X<uint32_t, uint64_t><<<ngrp, 256, 0, st>>>(d_C, d_nodes, d_grp_node, ngrp, d_P, d_X, stride,
                                               P.light_buckets, 0, 0, nullptr, rg);
    check_launch();
    tr.launched(3);

    // blocked distributing
    tr.begin(kPhDistribute);
    // even levels (A -> S, copied back): heavy keys are filled by the copy
    launch_distribute<K, V>(sk, sv, d_ids, dk, dv, d_work, nwork, d_nodes, d_X, stride, 0xFFFFFFFFu,
                            P.light_buckets, 0, st, n, d_ctr, from_a ? P.light_buckets : 0xFFFFFFFFu,
                            from_r || (aos && !from_a), aos && from_a);
    check_launch();
    tr.launched();

    // heavy buckets are final: copy them back when they landed in S (their
    // keys were not scattered: one key per bucket, filled here).  In order on
    // the caller's stream: overlapping it with the next level took SMs from
    // the distribute (the two kernels cannot share an SM's registers).
    if (from_a) {
      tr.begin(kPhCopy);
      const uint32_t gy = std::min<uint32_t>(nn, 65535);
      const uint32_t gx = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(1184, cdiv(1184, gy))));
      k_copy_heavy_fill<K, V><<<dim3(gx, gy), 256, 0, st>>>(A_k, heavy_src(), A_v, d_nodes, nn, d_off, stride,
                                                           P.light_buckets, d_heavy, bf.max_heavy, aos ? 1 : 0);
      check_launch();
      tr.launched();
    }

    // children
    tr.begin(kPhChildren);
    SS_CUDA(cudaMemsetAsync(d_misc, 0, 8 * sizeof(uint64_t), st));
    const LeafClasses lcls{kLeafWarpMax, kLeafSmemMax, P.base_case_cutoff};
    k_children_count<<<nn, 256, 0, st>>>(d_nodes, nn, d_off, stride, P.light_buckets, lcls, d_ccnt);
    check_launch();
    k_children_scan<<<1, 1024, 0, st>>>(d_ccnt, nn, d_misc);
    check_launch();
    k_children_emit<<<nn, 256, 0, st>>>(d_nodes, nn, d_off, stride, P.light_buckets, lcls, d_ccnt, nullptr,
                                        rounds_per_hash(P.light_bits), d_leaf_w, d_leaf_s, d_leaf_g, d_next,
                                        d_misc + 4);
    check_launch();
    tr.launched(3);
    tr.end();

    uint64_t misc[8];
    SS_CUDA(cudaMemcpyAsync(misc, d_misc, sizeof(misc), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaMemcpyAsync(cur.data(), d_nodes, nn * sizeof(Node), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    const uint64_t n_w = misc[0], n_s = misc[1], n_g = misc[2], n_next = misc[3], max_mid = misc[4];
    std::vector<Node> next(n_next);
    if (n_next) {
      SS_CUDA(cudaMemcpyAsync(next.data(), d_next, n_next * sizeof(Node), cudaMemcpyDeviceToHost, st));
      SS_CUDA(cudaStreamSynchronize(st));
    }

    // telemetry with the reference's counter semantics (core.py:451-482)
    if (tel) {
      for (const Node& nd : cur) {
        tel->bucket_assignments += nd.size;
        if (lvl <= 64)
          tel->matrix_cells_by_level[lvl] += cdiv(nd.size, P.subarray_len) * (P.light_buckets + nd.n_heavy);
        if (from_a) tel->scratch_moves += nd.size;
      }
      const uint64_t kids = n_w + n_s + n_g + n_next;
      tel->nodes += kids;
      if (kids && static_cast<uint64_t>(lvl + 1) > tel->max_depth) tel->max_depth = lvl + 1;
      tel->levels += 1;
    }

    // leaves of this level live on the destination side
    const bool leaves_in_a = !from_a;
    tr.begin(kPhLeaves);
    run_leaves_warp(tr, d_leaf_w, n_w, leaves_in_a);
    run_leaves_smem(tr, d_leaf_s, n_s, leaves_in_a);
    run_leaves_global(tr, d_leaf_g, n_g, leaves_in_a, nullptr, 0, max_mid);

    // forced leaves (stall valve / depth limit, core.py:459)
    std::vector<Node> keep;
    std::vector<Leaf> forced;
    for (const Node& c : next) {
      if (c.stalled >= 2 || lvl + 1 >= kDepthLimit) forced.push_back(Leaf{c.lo, c.size});
      else keep.push_back(c);
    }
    run_host_leaves(tr, forced, leaves_in_a);
    tr.end();
    return keep;
  }

  // Drive levels from an initial frontier of internal nodes at `lvl`.
  void drive(Tracker& tr, std::vector<Node> cur, int lvl, bool flip) {
    while (!cur.empty()) {
      cur = level(tr, cur, lvl, flip);
      ++lvl;
    }
  }

  void run(Tracker& tr) {
    if constexpr (std::is_same_v<K, V>) {   // pair scratch layout when the single-pass kernel serves
      if (!external_scratch && S_k && hw_rank_ok() && dist1_tile<K, V>(stride, n) != 0) {
        aos = true;
        S_v = reinterpret_cast<V*>(S_k + 1);
      }
    }
    run_levels(tr);
  }

  void run_levels(Tracker& tr) {
    if (tel) tel->scratch_allocations += 1;   // one scratch per call (core.py:591-592)
    if (tel) {
      tel->nodes += 1;
      tel->max_depth = std::max<uint64_t>(tel->max_depth, 1);
    }
    if (n == 0) return;
    if (n < P.base_case_cutoff) {   // root is a leaf (core.py:459)
      run_host_leaves(tr, {Leaf{0, n}}, true);
      return;
    }
    Node root{};
    root.lo = 0;
    root.size = n;
    root.path = 0;
    root.depth = 0;
    root.stalled = 0;
    drive(tr, {root}, 1, false);
  }
};

}  // namespace ss
