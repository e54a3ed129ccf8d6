// C-ABI exports (include/semisort_b200.h): argument checking, key/value
// type dispatch, workspace carving and the phase-level entry points.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "abi.cuh"
#include "agg_engine.cuh"
#include "engine.cuh"
#include "sort_engine.cuh"

namespace ss {

thread_local std::string g_last_error;

// Calls f.template operator()<K, V>() for the runtime widths.
template <typename F>
void dispatch_kv(uint32_t kb, uint32_t vb, F&& f) {
  check_widths(kb, vb);
  if (kb == 8) {
    switch (vb) {
      case 0: f.template operator()<uint64_t, NoVal>(); return;
      case 4: f.template operator()<uint64_t, uint32_t>(); return;
      case 8: f.template operator()<uint64_t, uint64_t>(); return;
      default: f.template operator()<uint64_t, V16>(); return;
    }
  } else {
    switch (vb) {
      case 0: f.template operator()<uint32_t, NoVal>(); return;
      case 4: f.template operator()<uint32_t, uint32_t>(); return;
      case 8: f.template operator()<uint32_t, uint64_t>(); return;
      default: f.template operator()<uint32_t, V16>(); return;
    }
  }
}

// dispatch_kv plus 128-bit keys (records.py:8-10): the semisort and
// aggregation entry points; the phase-level API stays 32/64-bit.
template <typename F>
void dispatch_sort(uint32_t kb, uint32_t vb, F&& f) {
  check_widths(kb, vb, true);
  if (kb != 16) return dispatch_kv(kb, vb, f);
  switch (vb) {
    case 0: f.template operator()<U128, NoVal>(); return;
    case 4: f.template operator()<U128, uint32_t>(); return;
    case 8: f.template operator()<U128, uint64_t>(); return;
    default: f.template operator()<U128, V16>(); return;
  }
}

template <typename F>
void dispatch_k(uint32_t kb, F&& f) {
  if (kb == 8) f.template operator()<uint64_t>();
  else if (kb == 4) f.template operator()<uint32_t>();
  else throw Fail(SS_ERR_CONTRACT, "key_bytes must be 4 or 8");
}

// ---------------------------------------------------------------------------
// single-node helpers for the phase-level API (explicit subarray_len)
// ---------------------------------------------------------------------------

struct PhasePlan {
  uint32_t stride;
  uint64_t rows, grps;
  Node* d_node;
  Work* d_work;
  uint32_t* d_grp_node;
  uint32_t* d_C;
  uint64_t* d_X;
  uint64_t* d_P;
  uint64_t* d_off;
  uint64_t* d_heavy;
  uint32_t* d_ctr;
  uint32_t* d_leafscr;
  uint64_t* d_samp;
  uint64_t leaf_words_n;
  uint64_t s_cap;
  uint16_t* d_ids;

  void carve(Arena& a, uint64_t n, uint32_t stride_, const Params& P, int key_bytes) {
    stride = (stride_ + 1) & ~1u;
    const uint64_t l = std::max<uint64_t>(P.subarray_len, 1);
    rows = std::max<uint64_t>(1, cdiv(n, l));
    grps = cdiv(rows, kRowGroup) + 1;
    d_node = a.take<Node>(1);
    d_work = a.take<Work>(rows);
    d_grp_node = a.take<uint32_t>(grps);
    d_C = a.take<uint32_t>(rows * stride);
    d_X = a.take<uint64_t>(rows * stride);
    d_P = a.take<uint64_t>(grps * stride);
    d_off = a.take<uint64_t>(stride + 1);
    d_heavy = a.take<uint64_t>(kMaxHeavyDevice);
    d_ctr = a.take<uint32_t>(4);
    leaf_words_n = std::max(leaf_words(std::max<uint64_t>(n, 1), false), lt_leaf_words(n, key_bytes));
    d_leafscr = a.take<uint32_t>(leaf_words_n);
    s_cap = std::max<uint64_t>(1, std::min<uint64_t>(n, P.sample_count));
    d_samp = a.take<uint64_t>(sample_scratch_words(s_cap, 8));
    d_ids = a.take<uint16_t>(n);
  }

  // One node spanning [0, n), rows of exactly subarray_len records.
  void upload_single(uint64_t n, uint32_t depth, uint32_t n_heavy, uint64_t l, cudaStream_t st,
                     std::vector<Work>& work, std::vector<uint32_t>& gn, Node& nd) {
    nd = Node{};
    nd.lo = 0;
    nd.size = n;
    nd.depth = depth;
    nd.n_heavy = n_heavy;
    nd.out_base = 0;
    nd.row_base = 0;
    nd.n_rows = static_cast<uint32_t>(cdiv(n, l));
    nd.grp_base = 0;
    nd.n_grps = static_cast<uint32_t>(cdiv(nd.n_rows, kRowGroup));
    work.clear();
    for (uint64_t r = 0; r < nd.n_rows; ++r) {
      Work w;
      w.begin = r * l;
      w.len = static_cast<uint32_t>(std::min<uint64_t>(l, n - r * l));
      w.node = 0;
      w.row = r;
      work.push_back(w);
    }
    gn.assign(nd.n_grps, 0);
    SS_CUDA(cudaMemcpyAsync(d_node, &nd, sizeof(Node), cudaMemcpyHostToDevice, st));
    if (!work.empty())
      SS_CUDA(cudaMemcpyAsync(d_work, work.data(), work.size() * sizeof(Work), cudaMemcpyHostToDevice, st));
    if (!gn.empty())
      SS_CUDA(cudaMemcpyAsync(d_grp_node, gn.data(), gn.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  }
};

// Caller-supplied bucket ids index shared-memory counters: reject any id
// outside [0, nb) before a kernel uses it (the reference raises for them).
__global__ void k_check_ids(const int32_t* ids, uint64_t n, uint32_t nb, uint32_t* bad) {
  uint32_t local = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    local |= static_cast<uint32_t>(ids[i]) >= nb ? 1u : 0u;
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1u);
}

inline void check_ids(const void* ids, uint64_t n, uint32_t nb, uint32_t* d_flag, cudaStream_t st) {
  SS_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(uint32_t), st));
  k_check_ids<<<static_cast<uint32_t>(std::min<uint64_t>(cdiv(n, 256), 1184)), 256, 0, st>>>(
      static_cast<const int32_t*>(ids), n, nb, d_flag);
  check_launch();
  uint32_t bad = 0;
  SS_CUDA(cudaMemcpyAsync(&bad, d_flag, sizeof(bad), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  if (bad) throw Fail(SS_ERR_CONFIG, "bucket ids must lie in [0, n_buckets)");
}

__global__ void k_u32_to_i64(const uint32_t* src, uint64_t rows, uint32_t cols, uint32_t stride, int64_t* dst) {
  uint64_t total = rows * cols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t r = i / cols, c = i % cols;
    dst[i] = static_cast<int64_t>(src[r * stride + c]);
  }
}

__global__ void k_i64_to_u32_strided(const int64_t* src, uint64_t rows, uint32_t cols, uint32_t stride, uint32_t* dst) {
  uint64_t total = rows * cols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t r = i / cols, c = i % cols;
    dst[r * stride + c] = static_cast<uint32_t>(src[i]);
  }
}

__global__ void k_i64_to_u64_strided(const int64_t* src, uint64_t rows, uint32_t cols, uint32_t stride, uint64_t* dst) {
  uint64_t total = rows * cols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t r = i / cols, c = i % cols;
    dst[r * stride + c] = static_cast<uint64_t>(src[i]);
  }
}

__global__ void k_u64_to_i64_strided(const uint64_t* src, uint64_t rows, uint32_t cols, uint32_t stride, int64_t* dst) {
  uint64_t total = rows * cols;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t r = i / cols, c = i % cols;
    dst[i] = static_cast<int64_t>(src[r * stride + c]);
  }
}

template <typename K>
__global__ void k_assign_ids(const K* __restrict__ keys, uint64_t n, const uint64_t* __restrict__ heavy,
                             uint32_t n_heavy, LightCfg lc, int identity, uint32_t n_light,
                             int32_t* __restrict__ out) {
  __shared__ HeavySmem tab;
  heavy_build(tab, heavy, n_heavy, identity != 0);
  __syncthreads();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(bucket_of(keys[i], tab, n_heavy, lc, identity != 0, n_light));
}

inline uint32_t grid_for(uint64_t n, uint32_t threads = 256, uint32_t cap = 148 * 16) {
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(cap, cdiv(n, threads))));
}

}  // namespace ss

using namespace ss;

extern "C" {

const char* ss_last_error(void) { return g_last_error.c_str(); }

int ss_version(void) { return 1; }

uint64_t ss_semisort_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                                     const ss_params* params) {
  uint64_t out = 0;
  int rc = guarded([&] {
    Params P = to_params(params, n, false);
    dispatch_sort(key_bytes, value_bytes, [&]<typename K, typename V>() {
      SortEngine<K, V> e{};
      e.n = n;
      e.P = P;
      Arena a(nullptr, 0);
      e.plan(a);
      out = a.used + 4096;
    });
  });
  return rc == SS_OK ? out : 0;
}

int ss_semisort(void* keys, void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes, int mode,
                int identity, const ss_params* params, void* workspace, uint64_t workspace_bytes,
                ss_telemetry* telemetry, void* stream) {
  return guarded([&] {
    if (mode != SS_MODE_EQ && mode != SS_MODE_LT) throw Fail(SS_ERR_CONFIG, "mode must be 'eq' or 'lt'");
    Params P = to_params(params, n, true);
    if (value_bytes && !values && n) throw Fail(SS_ERR_CONTRACT, "values pointer is NULL");
    reset_tel(telemetry);
    dispatch_sort(key_bytes, value_bytes, [&]<typename K, typename V>() {
      SortEngine<K, V> e{};
      e.A_k = static_cast<K*>(keys);
      e.A_v = static_cast<V*>(values);
      e.n = n;
      e.mode = mode;
      e.identity = identity;
      e.P = P;
      e.st = as_stream(stream);
      e.tel = telemetry;
      Arena a(workspace, workspace_bytes);
      e.plan(a);
      Tracker tr(e.st, telemetry);
      e.run(tr);
      tr.finish();
      SS_CUDA(cudaGetLastError());
    });
  });
}

int ss_local_refine(void* keys, void* values, void* scratch_keys, void* scratch_values, uint64_t n,
                    uint32_t key_bytes, uint32_t value_bytes, int mode, int identity, const ss_params* params,
                    const int64_t* offsets, uint32_t n_buckets, int live_in_primary, uint32_t depth,
                    void* workspace, uint64_t workspace_bytes, ss_telemetry* telemetry, void* stream) {
  return guarded([&] {
    if (mode != SS_MODE_EQ && mode != SS_MODE_LT) throw Fail(SS_ERR_CONFIG, "mode must be 'eq' or 'lt'");
    Params P = to_params(params, n, false);
    if (!offsets || n_buckets < P.light_buckets) throw Fail(SS_ERR_CONFIG, "offsets do not match light_buckets");
    reset_tel(telemetry);
    dispatch_kv(key_bytes, value_bytes, [&]<typename K, typename V>() {
      SortEngine<K, V> e{};
      e.A_k = static_cast<K*>(keys);
      e.A_v = static_cast<V*>(values);
      e.n = n;
      e.mode = mode;
      e.identity = identity;
      e.P = P;
      e.st = as_stream(stream);
      e.tel = telemetry;
      Arena a(workspace, workspace_bytes);
      e.plan(a, false);
      e.S_k = static_cast<K*>(scratch_keys);
      e.S_v = static_cast<V*>(scratch_values);
      Tracker tr(e.st, telemetry);
      const uint64_t total = static_cast<uint64_t>(offsets[n_buckets]);
      const bool live_a = live_in_primary != 0;
      if (!live_a) {   // heavy buckets are final: copy back (core.py:549-552)
        const uint64_t h0 = static_cast<uint64_t>(offsets[P.light_buckets]);
        if (h0 < total) {
          k_copy_range<K, V><<<grid_for(total - h0), 256, 0, e.st>>>(e.S_k, e.S_v, e.A_k, e.A_v, h0, total);
          check_launch();
          tr.launched();
        }
      }
      std::vector<Leaf> small;
      std::vector<Node> big;
      const uint32_t rounds = rounds_per_hash(P.light_bits);
      for (uint32_t b = 0; b < P.light_buckets; ++b) {
        const uint64_t lo = offsets[b], hi = offsets[b + 1];
        if (hi == lo) continue;
        if (hi - lo < P.base_case_cutoff) {
          small.push_back(Leaf{lo, hi - lo});
          continue;
        }
        Node c{};
        c.lo = lo;
        c.size = hi - lo;
        c.path = mix64_pair(P.seed, static_cast<uint64_t>(b) + 1);
        c.parent_size = total;
        uint32_t d = depth + 1, stalled = 0;
        if (2 * c.size > total) {
          stalled = 1;
          d = (d / rounds + 1) * rounds;
        }
        c.depth = d;
        c.stalled = stalled;
        big.push_back(c);
      }
      if (telemetry) {
        telemetry->nodes += small.size() + big.size();
        if (!small.empty() || !big.empty()) telemetry->max_depth = std::max<uint64_t>(telemetry->max_depth, 1);
      }
      // level-1 nodes live on the live side: flip the parity when that is S
      e.run_host_leaves(tr, small, live_a);
      e.drive(tr, big, 1, !live_a);
      tr.finish();
      SS_CUDA(cudaGetLastError());
    });
  });
}

// ---- aggregation --------------------------------------------------------------

uint64_t ss_aggregate_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                                      const ss_params* params) {
  uint64_t out = 0;
  int rc = guarded([&] {
    Params P = to_params(params, n, false);
    dispatch_sort(key_bytes, value_bytes, [&]<typename K, typename V>() {
      AggEngine<K, V> e{};
      e.n = n;
      e.P = P;
      Arena a(nullptr, 0);
      e.plan(a);
      out = a.used + 4096;
    });
  });
  return rc == SS_OK ? out : 0;
}

int ss_collect_reduce(const void* keys, const void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                      int kind, int identity, const ss_params* params, void* workspace, uint64_t workspace_bytes,
                      uint64_t* out_count, ss_telemetry* telemetry, void* stream) {
  return guarded([&] {
    if (kind != SS_AGG_COUNT && kind != SS_AGG_SUM64) throw Fail(SS_ERR_CONFIG, "unknown aggregate kind");
    Params P = to_params(params, n, true);
    if (kind == SS_AGG_SUM64 && n && (!values || value_bytes == 0))
      throw Fail(SS_ERR_CONFIG, "summing64 needs a value column");
    if (!out_count) throw Fail(SS_ERR_CONFIG, "out_count must not be NULL");
    reset_tel(telemetry);
    dispatch_sort(key_bytes, value_bytes, [&]<typename K, typename V>() {
      AggEngine<K, V> e{};
      e.in_k = static_cast<const K*>(keys);
      e.in_v = static_cast<const V*>(values);
      e.n = n;
      e.kind = kind;
      e.identity = identity;
      e.P = P;
      e.st = as_stream(stream);
      e.tel = telemetry;
      Arena a(workspace, workspace_bytes);
      e.plan(a);
      Tracker tr(e.st, telemetry);
      *out_count = e.run(tr);
      tr.finish();
      SS_CUDA(cudaGetLastError());
    });
  });
}

int ss_histogram(const void* keys, uint64_t n, uint32_t key_bytes, int identity, const ss_params* params,
                 void* workspace, uint64_t workspace_bytes, uint64_t* out_count, ss_telemetry* telemetry,
                 void* stream) {
  return ss_collect_reduce(keys, nullptr, n, key_bytes, 0, SS_AGG_COUNT, identity, params, workspace,
                           workspace_bytes, out_count, telemetry, stream);
}

int ss_result_copy(const void* workspace, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                   const ss_params* params, void* out_keys, void* out_aggs, uint64_t count, void* stream) {
  return guarded([&] {
    Params P = to_params(params, n, false);
    dispatch_sort(key_bytes, value_bytes, [&]<typename K, typename V>() {
      AggEngine<K, V> e{};
      e.n = n;
      e.P = P;
      Arena a(const_cast<void*>(workspace), ~0ull);
      e.plan(a);
      if (count > e.max_pairs) throw Fail(SS_ERR_CONFIG, "count exceeds the result capacity");
      cudaStream_t st = as_stream(stream);
      if (count) {
        SS_CUDA(cudaMemcpyAsync(out_keys, e.d_out_k, count * sizeof(K), cudaMemcpyDeviceToDevice, st));
        SS_CUDA(cudaMemcpyAsync(out_aggs, e.d_out_a, count * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
      }
    });
  });
}

// ---- phase level ----------------------------------------------------------------

uint64_t ss_phase_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes, const ss_params* params) {
  uint64_t out = 0;
  int rc = guarded([&] {
    check_widths(key_bytes, value_bytes);
    Params P = to_params(params, n, false);
    PhasePlan pp{};
    Arena a(nullptr, 0);
    pp.carve(a, n, P.light_buckets + P.max_heavy, P, key_bytes);
    out = a.used + 4096;
  });
  return rc == SS_OK ? out : 0;
}

int ss_sample_heavy(const void* keys, uint64_t n, uint32_t key_bytes, const ss_params* params, uint64_t rng_key,
                    void* out_heavy, uint32_t* out_n_heavy, void* workspace, uint64_t workspace_bytes,
                    void* stream) {
  return guarded([&] {
    Params P = to_params(params, n, false);
    cudaStream_t st = as_stream(stream);
    PhasePlan pp{};
    Arena a(workspace, workspace_bytes);
    pp.carve(a, n, P.light_buckets + P.max_heavy, P, key_bytes);
    // the phase API receives the Philox key itself (core.py:222, rng arg)
    Node nd{};
    nd.lo = 0;
    nd.size = n;
    SS_CUDA(cudaMemcpyAsync(pp.d_node, &nd, sizeof(Node), cudaMemcpyHostToDevice, st));
    dispatch_k(key_bytes, [&]<typename K>() {
      SS_CUDA(cudaFuncSetAttribute(k_sample<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(kSampleSmem)));
      k_sample<K><<<1, kSampleThreads, kSampleSmem, st>>>(static_cast<const K*>(keys), pp.d_node, 1,
                                                          static_cast<uint64_t*>(out_heavy), pp.d_samp,
                                                          pp.s_cap, P, 1, rng_key);
      check_launch();
    });
    SS_CUDA(cudaMemcpyAsync(&nd, pp.d_node, sizeof(Node), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    *out_n_heavy = nd.n_heavy;
  });
}

int ss_assign_bucket_ids(const void* keys, uint64_t n, uint32_t key_bytes, int identity, const ss_params* params,
                         uint32_t depth, const void* heavy_keys, uint32_t n_heavy, void* out_ids, void* workspace,
                         uint64_t workspace_bytes, void* stream) {
  return guarded([&] {
    (void)workspace;
    (void)workspace_bytes;
    Params P = to_params(params, n, false);
    if (n_heavy > static_cast<uint32_t>(kMaxHeavyDevice)) throw Fail(SS_ERR_CONFIG, "too many heavy keys");
    cudaStream_t st = as_stream(stream);
    LightCfg lc = LightCfg::make(depth, P.light_bits, P.light_buckets);
    dispatch_k(key_bytes, [&]<typename K>() {
      k_assign_ids<K><<<grid_for(n), 256, 0, st>>>(static_cast<const K*>(keys), n,
                                                   static_cast<const uint64_t*>(heavy_keys), n_heavy, lc,
                                                   identity, P.light_buckets, static_cast<int32_t*>(out_ids));
      check_launch();
    });
  });
}

int ss_count_matrix(const void* keys, const void* ids, uint64_t n, uint32_t key_bytes, int identity,
                    const ss_params* params, uint32_t depth, const void* heavy_keys, uint32_t n_heavy,
                    uint32_t n_buckets, void* out_counts, void* workspace, uint64_t workspace_bytes, void* stream) {
  return guarded([&] {
    Params P = to_params(params, n, false);
    cudaStream_t st = as_stream(stream);
    if (n == 0) return;
    if (!ids && n_buckets != P.light_buckets + n_heavy) throw Fail(SS_ERR_CONFIG, "n_buckets mismatch");
    if (n_buckets > 8192) throw Fail(SS_ERR_CONFIG, "too many buckets for the GPU counting matrix");
    PhasePlan pp{};
    Arena a(workspace, workspace_bytes);
    pp.carve(a, n, std::max<uint32_t>(n_buckets, P.light_buckets + P.max_heavy), P, key_bytes);
    std::vector<Work> work;
    std::vector<uint32_t> gn;
    Node nd;
    pp.upload_single(n, depth, n_heavy, P.subarray_len, st, work, gn, nd);
    if (n_heavy)
      SS_CUDA(cudaMemcpyAsync(pp.d_heavy, heavy_keys, n_heavy * 8, cudaMemcpyDeviceToDevice, st));
    if (ids) check_ids(ids, n, n_buckets, pp.d_ctr, st);
    dispatch_k(key_bytes, [&]<typename K>() {
      const uint32_t nw = static_cast<uint32_t>(work.size());
      if (ids) {
        IdBuckets bf{static_cast<const int32_t*>(ids), n_buckets};
        k_count<K, IdBuckets><<<nw, kCountThreads, pp.stride * 4, st>>>(static_cast<const K*>(keys), pp.d_work, nw,
                                                                       pp.d_node, pp.d_C, pp.stride, bf, nullptr);
      } else {
        KeyBuckets bf{};
        bf.heavy = pp.d_heavy;
        bf.max_heavy = kMaxHeavyDevice;
        bf.n_light = P.light_buckets;
        bf.light_bits = P.light_bits;
        bf.identity = identity;
        k_count<K, KeyBuckets><<<nw, kCountThreads, pp.stride * 4, st>>>(static_cast<const K*>(keys), pp.d_work, nw,
                                                                        pp.d_node, pp.d_C, pp.stride, bf, nullptr);
      }
      check_launch();
    });
    k_u32_to_i64<<<grid_for(pp.rows * n_buckets), 256, 0, st>>>(pp.d_C, nd.n_rows, n_buckets, pp.stride,
                                                                  static_cast<int64_t*>(out_counts));
    check_launch();
    SS_CUDA(cudaStreamSynchronize(st));
  });
}

int ss_column_scan(const void* counts, uint64_t rows, uint32_t n_buckets, void* out_prefix, void* out_offsets,
                   void* workspace, uint64_t workspace_bytes, void* stream) {
  return guarded([&] {
    cudaStream_t st = as_stream(stream);
    const uint32_t stride = (n_buckets + 1) & ~1u;
    Arena a(workspace, workspace_bytes);
    const uint64_t grps = std::max<uint64_t>(1, cdiv(rows, kRowGroup));
    Node* d_node = a.take<Node>(1);
    uint32_t* d_gn = a.take<uint32_t>(grps);
    uint64_t* d_C = a.take<uint64_t>(std::max<uint64_t>(rows, 1) * stride);
    uint64_t* d_P = a.take<uint64_t>(grps * stride);
    uint64_t* d_X = a.take<uint64_t>(std::max<uint64_t>(rows, 1) * stride);
    uint64_t* d_off = a.take<uint64_t>(stride + 1);
    if (n_buckets == 0) return;
    if (rows == 0) {
      SS_CUDA(cudaMemsetAsync(out_offsets, 0, (n_buckets + 1) * sizeof(int64_t), st));
      SS_CUDA(cudaStreamSynchronize(st));
      return;
    }
    Node nd{};
    nd.n_rows = static_cast<uint32_t>(rows);
    nd.n_grps = static_cast<uint32_t>(cdiv(rows, kRowGroup));
    std::vector<uint32_t> gn(nd.n_grps, 0);
    SS_CUDA(cudaMemcpyAsync(d_node, &nd, sizeof(Node), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaMemcpyAsync(d_gn, gn.data(), gn.size() * 4, cudaMemcpyHostToDevice, st));
    k_i64_to_u64_strided<<<grid_for(rows * n_buckets), 256, 0, st>>>(static_cast<const int64_t*>(counts), rows,
                                                                       n_buckets, stride, d_C);
    k_colsum_groups<uint64_t><<<nd.n_grps, 256, 0, st>>>(d_C, d_node, d_gn, nd.n_grps, d_P, stride, 0, 0, n_buckets);
    k_scan_nodes<<<1, 1024, 0, st>>>(d_node, 1, d_P, d_off, stride, 0, 0, n_buckets, nullptr);
    k_write_X<uint64_t, uint64_t><<<nd.n_grps, 256, 0, st>>>(d_C, d_node, d_gn, nd.n_grps, d_P, d_X, stride, 0, 0,
                                                               n_buckets, nullptr);
    k_u64_to_i64_strided<<<grid_for(rows * n_buckets), 256, 0, st>>>(d_X, rows, n_buckets, stride,
                                                                       static_cast<int64_t*>(out_prefix));
    k_u64_to_i64_strided<<<1, 256, 0, st>>>(d_off, 1, n_buckets + 1, n_buckets + 1, static_cast<int64_t*>(out_offsets));
    check_launch();
    SS_CUDA(cudaStreamSynchronize(st));
  });
}

int ss_distribute(const void* src_keys, const void* src_values, void* dst_keys, void* dst_values, const void* ids,
                  uint64_t n, uint32_t key_bytes, uint32_t value_bytes, int identity, const ss_params* params,
                  uint32_t depth, const void* heavy_keys, uint32_t n_heavy, uint32_t n_buckets, const void* prefix,
                  void* workspace, uint64_t workspace_bytes, void* stream) {
  return guarded([&] {
    Params P = to_params(params, n, false);
    cudaStream_t st = as_stream(stream);
    if (n == 0) return;
    if (n_buckets >= kSentinel) throw Fail(SS_ERR_CONFIG, "too many buckets for the GPU distribute");
    PhasePlan pp{};
    Arena a(workspace, workspace_bytes);
    pp.carve(a, n, std::max<uint32_t>(n_buckets, P.light_buckets + P.max_heavy), P, key_bytes);
    std::vector<Work> work;
    std::vector<uint32_t> gn;
    Node nd;
    pp.upload_single(n, depth, n_heavy, P.subarray_len, st, work, gn, nd);
    if (n_heavy)
      SS_CUDA(cudaMemcpyAsync(pp.d_heavy, heavy_keys, n_heavy * 8, cudaMemcpyDeviceToDevice, st));
    k_i64_to_u64_strided<<<grid_for(nd.n_rows * static_cast<uint64_t>(n_buckets)), 256, 0, st>>>(
        static_cast<const int64_t*>(prefix), nd.n_rows, n_buckets, pp.stride, pp.d_X);
    check_launch();
    if (ids) check_ids(ids, n, n_buckets, pp.d_ctr, st);
    const uint32_t nw = static_cast<uint32_t>(work.size());
    dispatch_kv(key_bytes, value_bytes, [&]<typename K, typename V>() {
      // bucket ids (u16) by the count kernel, then the stable scatter
      const K* sk = static_cast<const K*>(src_keys);
      if (ids) {
        IdBuckets bf{static_cast<const int32_t*>(ids), n_buckets};
        k_count<K, IdBuckets><<<nw, kCountThreads, pp.stride * 4, st>>>(sk, pp.d_work, nw, pp.d_node, pp.d_C,
                                                                       pp.stride, bf, pp.d_ids);
      } else {
        KeyBuckets bf{};
        bf.heavy = pp.d_heavy;
        bf.max_heavy = kMaxHeavyDevice;
        bf.n_light = P.light_buckets;
        bf.light_bits = P.light_bits;
        bf.identity = identity;
        k_count<K, KeyBuckets><<<nw, kCountThreads, pp.stride * 4, st>>>(sk, pp.d_work, nw, pp.d_node, pp.d_C,
                                                                        pp.stride, bf, pp.d_ids);
      }
      check_launch();
      launch_distribute<K, V>(sk, static_cast<const V*>(src_values), pp.d_ids, static_cast<K*>(dst_keys),
                              static_cast<V*>(dst_values), pp.d_work, nw, pp.d_node, pp.d_X, pp.stride, 0xFFFFFFFFu,
                              P.light_buckets, n_buckets, st, n, pp.d_ctr);
    });
    SS_CUDA(cudaStreamSynchronize(st));
  });
}

int ss_base_case(void* keys, void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes, int mode,
                 int identity, void* workspace, uint64_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (mode != SS_MODE_EQ && mode != SS_MODE_LT) throw Fail(SS_ERR_CONFIG, "mode must be 'eq' or 'lt'");
    cudaStream_t st = as_stream(stream);
    if (n < 2) return;
    dispatch_kv(key_bytes, value_bytes, [&]<typename K, typename V>() {
      Arena a(workspace, workspace_bytes);
      K* S_k = a.take<K>(n);
      V* S_v = ValTraits<V>::bytes ? a.take<V>(n) : nullptr;
      Leaf* d_leaf = a.take<Leaf>(1);
      const uint64_t words = std::max(leaf_words(n, false), lt_leaf_words(n, sizeof(K)));
      uint32_t* scr = a.take<uint32_t>(words);
      Leaf lf{0, n};
      SS_CUDA(cudaMemcpyAsync(d_leaf, &lf, sizeof(Leaf), cudaMemcpyHostToDevice, st));
      if (mode == SS_MODE_LT)
        k_leaf_lt<K, V><<<1, kLeafThreads, 0, st>>>(S_k, S_v, static_cast<K*>(keys), static_cast<V*>(values), d_leaf, 1,
                                                   1, scr, words);
      else
        k_leaf_eq_global<K, V><<<1, kLeafThreads, 0, st>>>(S_k, S_v, static_cast<K*>(keys), static_cast<V*>(values),
                                                          d_leaf, 1, 1, identity, scr, words, hw_rank_ok() ? 1 : 0);
      check_launch();
      SS_CUDA(cudaStreamSynchronize(st));
    });
  });
}

uint64_t ss_base_case_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes) {
  return n * (key_bytes + value_bytes) + std::max(leaf_words(std::max<uint64_t>(n, 1), false),
                                                  lt_leaf_words(n, key_bytes)) * 4 + 8192;
}

}  // extern "C"
