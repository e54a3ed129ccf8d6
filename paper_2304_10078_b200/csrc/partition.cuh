// Multi-GPU hash partition: dest = top log2(G) bits of
// mix64(key), always hashed so identity-mode keys spread too.  The plan and
// the count + scan phases are shared by ss_partition (SoA output) and
// ss_partition_pairs (packed (key, value) records for one exchange).
#pragma once

#include <vector>

#include "engine.cuh"
#include "multisplit.cuh"

namespace ss {

struct PartBuckets {
  uint32_t shift;   // 64 - log2(parts); 64 means a single part
  uint32_t nb;
  template <typename T>
  __device__ __forceinline__ void prepare(const Node&, uint32_t, T*) { __syncthreads(); }
  __device__ __forceinline__ uint32_t n_buckets() const { return nb; }
  __device__ __forceinline__ uint32_t first_hot() const { return nb; }
  template <typename K>
  __device__ __forceinline__ uint32_t operator()(K key, uint64_t) const {
    return shift >= 64 ? 0u : static_cast<uint32_t>(mix64(static_cast<uint64_t>(key)) >> shift);
  }
  template <typename K, typename T>
  __device__ __forceinline__ uint32_t operator()(K key, uint64_t pos, const T&) const {
    return (*this)(key, pos);
  }
};

struct PartPlan {
  uint64_t rows, grps;
  uint32_t stride;
  Node* d_node;
  Work* d_work;
  uint32_t* d_gn;
  uint32_t* d_C;
  uint64_t* d_X;
  uint64_t* d_P;
  uint64_t* d_off;
  uint16_t* d_ids;
  uint32_t* d_ctr;
  void carve(Arena& a, uint64_t n, uint32_t parts) {
    stride = (parts + 1) & ~1u;
    rows = std::max<uint64_t>(1, std::min<uint64_t>(1184, cdiv(n, 4096)));
    grps = cdiv(rows, kRowGroup) + 1;
    d_node = a.take<Node>(1);
    d_work = a.take<Work>(rows);
    d_gn = a.take<uint32_t>(grps);
    d_C = a.take<uint32_t>(rows * stride);
    d_X = a.take<uint64_t>(rows * stride);
    d_P = a.take<uint64_t>(grps * stride);
    d_off = a.take<uint64_t>(stride + 1);
    d_ids = a.take<uint16_t>(n);
    d_ctr = a.take<uint32_t>(4);
  }
};

// Plan work items, count per (item, part) and scan: X and the part offsets
// are ready in pp afterwards.  Returns the work item count.
inline uint32_t partition_count_scan(PartPlan& pp, const void* keys, uint64_t n, uint32_t key_bytes, uint32_t parts,
                                     Node& nd, cudaStream_t st) {
  uint32_t bits = 0;
  while ((1u << bits) < parts) ++bits;
  PartBuckets bf{64u - bits, parts};
  const uint64_t chunk = (cdiv(n, pp.rows) + 7) & ~uint64_t(7);
  nd = Node{};
  nd.lo = 0;
  nd.size = n;
  nd.out_base = 0;
  nd.n_rows = static_cast<uint32_t>(cdiv(n, chunk));
  nd.n_grps = static_cast<uint32_t>(cdiv(nd.n_rows, kRowGroup));
  std::vector<Work> work(nd.n_rows);
  for (uint32_t r = 0; r < nd.n_rows; ++r) {
    work[r].begin = r * chunk;
    work[r].len = static_cast<uint32_t>(std::min<uint64_t>(chunk, n - r * chunk));
    work[r].node = 0;
    work[r].row = r;
  }
  std::vector<uint32_t> gn(nd.n_grps, 0);
  SS_CUDA(cudaMemcpyAsync(pp.d_node, &nd, sizeof(Node), cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemcpyAsync(pp.d_work, work.data(), work.size() * sizeof(Work), cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemcpyAsync(pp.d_gn, gn.data(), gn.size() * 4, cudaMemcpyHostToDevice, st));
  const uint32_t nw = nd.n_rows;
  auto count = [&](auto kt) {
    using K = decltype(kt);
    k_count<K, PartBuckets><<<nw, kCountThreads, pp.stride * 4, st>>>(static_cast<const K*>(keys), pp.d_work, nw,
                                                                    pp.d_node, pp.d_C, pp.stride, bf, pp.d_ids);
  };
  if (key_bytes == 8) count(uint64_t{});
  else count(uint32_t{});
  k_colsum_groups<uint32_t><<<nd.n_grps, 256, 0, st>>>(pp.d_C, pp.d_node, pp.d_gn, nd.n_grps, pp.d_P, pp.stride, 0, 0,
                                                       parts);
  k_scan_nodes<<<1, 1024, 0, st>>>(pp.d_node, 1, pp.d_P, pp.d_off, pp.stride, 0, 0, parts, nullptr);
  k_write_X<uint32_t, uint64_t><<<nd.n_grps, 256, 0, st>>>(pp.d_C, pp.d_node, pp.d_gn, nd.n_grps, pp.d_P, pp.d_X,
                                                            pp.stride, 0, 0, parts, nullptr);
  check_launch();
  return nw;
}

// Per-part counts (host) from the part offsets.
inline void partition_counts(const PartPlan& pp, uint32_t parts, uint64_t* out_counts, cudaStream_t st) {
  std::vector<uint64_t> off(parts + 1);
  SS_CUDA(cudaMemcpyAsync(off.data(), pp.d_off, (parts + 1) * 8, cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  for (uint32_t p = 0; p < parts; ++p) out_counts[p] = off[p + 1] - off[p];
}

}  // namespace ss
