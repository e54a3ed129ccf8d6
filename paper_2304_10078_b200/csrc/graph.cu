// Graph transpose and CSR construction on the semisort path (SURVEY.md
// §8(f) row 1; reference graphs.py:59-105).
//
// transpose: expand the CSR offsets to one source id per edge, semisort the
// (target u32, source u32) records with the identity hash (graphs.py:88-89),
// then rebuild offsets and targets from the runs of equal keys
// (graphs.py:91-104).  Each target's run is contiguous and in input order
// (stable), so placing run v at offset[v] yields ascending sources -- the
// same CSR the reference returns, independent of the semisort's group order.
// from_edges is the same rebuild keyed by source (stable argsort by source,
// graphs.py:59-71).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "abi.cuh"
#include "engine.cuh"
#include "scan.cuh"
#include "sort_engine.cuh"

namespace ss {
namespace {

constexpr int kGThreads = 256;

inline uint32_t grid_for(uint64_t n, uint32_t cap = 148 * 16) {
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(cap, cdiv(n, kGThreads))));
}

// mark[off[u]] = u for every vertex with edges (two vertices with edges
// never share an offset); mark is zeroed first.
__global__ void k_csr_mark(const uint64_t* __restrict__ off, uint64_t nv, uint32_t* __restrict__ mark) {
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < nv;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    if (off[u + 1] > off[u]) mark[off[u]] = static_cast<uint32_t>(u);
}

// Inclusive max-scan in place, three phases (tile maxima, their scan, apply):
// turns the marks into the source id of every edge (sources are
// nondecreasing along a CSR edge array, vertex 0's edges carry 0).
constexpr uint64_t kMaxTile = static_cast<uint64_t>(kScanThreads) * kScanItems;

__global__ void __launch_bounds__(kScanThreads) k_max_tiles(const uint32_t* __restrict__ a, uint64_t n,
                                                           uint32_t* __restrict__ part) {
  __shared__ uint32_t red[32];
  const uint64_t base = blockIdx.x * kMaxTile + threadIdx.x * kScanItems;
  uint32_t m = 0;
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) m = max(m, a[base + k]);
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane_id() == 0) red[warp_id()] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t x = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0;
    x = __reduce_max_sync(0xffffffffu, x);
    if (threadIdx.x == 0) part[blockIdx.x] = x;
  }
}

__global__ void __launch_bounds__(1024) k_max_parts(uint32_t* __restrict__ part, uint64_t np) {
  // exclusive running max of the tile maxima (one CTA; np is small)
  __shared__ uint32_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint64_t b = 0; b < np; b += blockDim.x) {
    const uint64_t i = b + threadIdx.x;
    uint32_t v = i < np ? part[i] : 0;
    // inclusive max-scan within the block
    uint32_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, x, d);
      if (lane_id() >= d) x = max(x, o);
    }
    __shared__ uint32_t wmax[32];
    if (lane_id() == 31) wmax[warp_id()] = x;
    __syncthreads();
    uint32_t before = carry_s;
    for (int w = 0; w < warp_id(); ++w) before = max(before, wmax[w]);
    const uint32_t excl_in_warp = __shfl_up_sync(0xffffffffu, x, 1);
    const uint32_t excl = lane_id() ? max(before, excl_in_warp) : before;
    __syncthreads();
    if (i < np) part[i] = excl;
    if (threadIdx.x == blockDim.x - 1) {
      uint32_t all = carry_s;
      for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) all = max(all, wmax[w]);
      carry_s = all;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kScanThreads) k_max_apply(uint32_t* __restrict__ a, uint64_t n,
                                                           const uint32_t* __restrict__ part) {
  __shared__ uint32_t wmax[32];
  const uint64_t base = blockIdx.x * kMaxTile + threadIdx.x * kScanItems;
  uint32_t v[kScanItems], m = 0;
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? a[base + k] : 0u;
    m = max(m, v[k]);
  }
  // exclusive max over earlier threads of the tile
  uint32_t x = m;
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, x, d);
    if (lane_id() >= d) x = max(x, o);
  }
  if (lane_id() == 31) wmax[warp_id()] = x;
  __syncthreads();
  uint32_t run = part[blockIdx.x];
  for (int w = 0; w < warp_id(); ++w) run = max(run, wmax[w]);
  const uint32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane_id()) run = max(run, prev);
  for (int k = 0; k < kScanItems; ++k) {
    run = max(run, v[k]);
    if (base + k < n) a[base + k] = run;
  }
}

// Run bounds of equal keys in the semisorted key column: rs[v] = first
// position, re[v] = one past the last (each key forms one run).
__global__ void k_run_bounds(const uint32_t* __restrict__ k, uint64_t m, uint64_t* __restrict__ rs,
                             uint64_t* __restrict__ re) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = k[i];
    if (i == 0 || k[i - 1] != v) rs[v] = i;
    if (i + 1 == m || k[i + 1] != v) re[v] = i + 1;
  }
}

__global__ void k_run_counts(const uint64_t* __restrict__ rs, uint64_t* __restrict__ re, uint64_t nv) {
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    re[v] -= rs[v];   // count (0 for vertices without a run: both stay 0)
}

// out_targets[offsets[v] + (i - rs[v])] = values[i] for key v = keys[i]
__global__ void k_run_scatter(const uint32_t* __restrict__ k, const uint32_t* __restrict__ val, uint64_t m,
                              const uint64_t* __restrict__ rs, const uint64_t* __restrict__ off,
                              uint32_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = k[i];
    out[off[v] + (i - rs[v])] = val[i];
  }
}

// Workspace of the shared CSR rebuild: pairs, per-vertex run bounds, scan
// parts, then the semisort's own workspace.
struct CsrPlan {
  uint32_t* pk = nullptr;   // keys (m)
  uint32_t* pv = nullptr;   // values (m)
  uint64_t* rs = nullptr;   // nv
  uint64_t* re = nullptr;   // nv (counts after k_run_counts)
  uint64_t* part = nullptr;
  uint64_t* total = nullptr;
  uint32_t* mpart = nullptr;
  SortEngine<uint32_t, uint32_t> eng{};
  void plan(Arena& a, uint64_t nv, uint64_t m, const Params& P) {
    pk = a.take<uint32_t>(std::max<uint64_t>(m, 1));
    pv = a.take<uint32_t>(std::max<uint64_t>(m, 1));
    rs = a.take<uint64_t>(std::max<uint64_t>(nv, 1));
    re = a.take<uint64_t>(std::max<uint64_t>(nv, 1));
    part = a.take<uint64_t>(scan_parts_needed(std::max<uint64_t>(nv, 1)) + 2);
    total = a.take<uint64_t>(2);
    mpart = a.take<uint32_t>(cdiv(std::max<uint64_t>(m, 1), kMaxTile) + 2);
    eng.n = m;
    eng.P = P;
    eng.A_k = pk;
    eng.A_v = pv;
    eng.plan(a);
  }
};

uint64_t csr_workspace(uint64_t nv, uint64_t m, const ss_params* params) {
  Params P = to_params(params, m, false);
  CsrPlan cp;
  Arena a(nullptr, 0);
  cp.plan(a, nv, m, P);
  return a.used + 4096;
}

// pk/pv hold the (key, value) edge records; semisort them and rebuild CSR.
void csr_rebuild(CsrPlan& cp, uint64_t nv, uint64_t m, uint64_t* out_off, uint32_t* out_t, cudaStream_t st,
                 ss_telemetry* tel) {
  cp.eng.mode = SS_MODE_EQ;
  cp.eng.identity = 1;   // UIntKeyAdapter(identity=True), graphs.py:88
  cp.eng.st = st;
  cp.eng.tel = tel;
  Tracker tr(st, tel);
  cp.eng.run(tr);
  tr.finish();
  SS_CUDA(cudaMemsetAsync(cp.rs, 0, std::max<uint64_t>(nv, 1) * 8, st));
  SS_CUDA(cudaMemsetAsync(cp.re, 0, std::max<uint64_t>(nv, 1) * 8, st));
  if (m) k_run_bounds<<<grid_for(m), kGThreads, 0, st>>>(cp.pk, m, cp.rs, cp.re);
  if (nv) k_run_counts<<<grid_for(nv), kGThreads, 0, st>>>(cp.rs, cp.re, nv);
  device_exclusive_scan<uint64_t>(cp.re, nv, out_off, cp.part, out_off + nv, st);   // offsets[n] = m
  if (m) k_run_scatter<<<grid_for(m), kGThreads, 0, st>>>(cp.pk, cp.pv, m, cp.rs, out_off, out_t);
  SS_CUDA(cudaGetLastError());
}

}  // namespace
}  // namespace ss

using namespace ss;

extern "C" {

uint64_t ss_csr_workspace_bytes(uint64_t n_vertices, uint64_t m, const ss_params* params) {
  uint64_t out = 0;
  const int rc = guarded([&] { out = csr_workspace(n_vertices, m, params); });
  return rc == SS_OK ? out : 0;
}

int ss_csr_from_edges(uint64_t n_vertices, uint64_t m, const uint32_t* sources, const uint32_t* targets,
                      uint64_t* out_offsets, uint32_t* out_targets, const ss_params* params, void* workspace,
                      uint64_t workspace_bytes, ss_telemetry* telemetry, void* stream) {
  return guarded([&] {
    if (n_vertices >= (1ull << 32)) throw Fail(SS_ERR_CONFIG, "vertex ids are 32-bit");
    if (m && (!sources || !targets)) throw Fail(SS_ERR_CONTRACT, "edge arrays are NULL");
    Params P = to_params(params, m, true);
    reset_tel(telemetry);
    cudaStream_t st = as_stream(stream);
    CsrPlan cp;
    Arena a(workspace, workspace_bytes);
    cp.plan(a, n_vertices, m, P);
    if (m) {
      SS_CUDA(cudaMemcpyAsync(cp.pk, sources, m * 4, cudaMemcpyDeviceToDevice, st));
      SS_CUDA(cudaMemcpyAsync(cp.pv, targets, m * 4, cudaMemcpyDeviceToDevice, st));
    }
    csr_rebuild(cp, n_vertices, m, out_offsets, out_targets, st, telemetry);
  });
}

int ss_graph_transpose(uint64_t n_vertices, uint64_t m, const uint64_t* offsets, const uint32_t* targets,
                       uint64_t* out_offsets, uint32_t* out_targets, const ss_params* params, void* workspace,
                       uint64_t workspace_bytes, ss_telemetry* telemetry, void* stream) {
  return guarded([&] {
    if (n_vertices >= (1ull << 32)) throw Fail(SS_ERR_CONFIG, "vertex ids are 32-bit");
    if (!offsets || (m && !targets)) throw Fail(SS_ERR_CONTRACT, "graph arrays are NULL");
    Params P = to_params(params, m, true);
    reset_tel(telemetry);
    cudaStream_t st = as_stream(stream);
    CsrPlan cp;
    Arena a(workspace, workspace_bytes);
    cp.plan(a, n_vertices, m, P);
    if (m) {
      // (target, source) records: keys = targets, values = expanded sources
      SS_CUDA(cudaMemcpyAsync(cp.pk, targets, m * 4, cudaMemcpyDeviceToDevice, st));
      SS_CUDA(cudaMemsetAsync(cp.pv, 0, m * 4, st));
      k_csr_mark<<<grid_for(n_vertices), kGThreads, 0, st>>>(offsets, n_vertices, cp.pv);
      const uint64_t nt = cdiv(m, kMaxTile);
      k_max_tiles<<<static_cast<uint32_t>(nt), kScanThreads, 0, st>>>(cp.pv, m, cp.mpart);
      k_max_parts<<<1, 1024, 0, st>>>(cp.mpart, nt);
      k_max_apply<<<static_cast<uint32_t>(nt), kScanThreads, 0, st>>>(cp.pv, m, cp.mpart);
    }
    csr_rebuild(cp, n_vertices, m, out_offsets, out_targets, st, telemetry);
  });
}

}  // extern "C"
