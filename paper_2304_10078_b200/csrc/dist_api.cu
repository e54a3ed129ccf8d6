// Multi-GPU entry points: the packed partition that
// feeds ONE exchange, the semisort that starts from the received packed
// records and finishes in the same memory (buffer reuse for strong scaling),
// and the whole per-rank pipeline over an NCCL communicator
// (ss_dist_semisort: partition -> count exchange -> all-to-allv of 16-byte
// records as grouped ncclSend/ncclRecv -> local semisort).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2; inside a torch
// process that is the already-loaded torch copy), so the library loads on
// hosts without NCCL and only the ss_nccl_* / ss_dist_* calls need it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "abi.cuh"
#include "engine.cuh"
#include "partition.cuh"
#include "sort_engine.cuh"

namespace ss {

// (key, value) pair records -> SoA columns keys[0, n), values[0, n)
template <typename K>
__global__ void k_unpack_pairs(const K* __restrict__ pairs, uint64_t n, K* __restrict__ keys, K* __restrict__ vals) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    keys[i] = pairs[2 * i];
    vals[i] = pairs[2 * i + 1];
  }
}

inline uint32_t dgrid(uint64_t n) {
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(148 * 16, cdiv(n, 256))));
}

template <typename F>
void dispatch_pair(uint32_t kb, F&& f) {
  if (kb == 8) f.template operator()<uint64_t>();
  else if (kb == 4) f.template operator()<uint32_t>();
  else throw Fail(SS_ERR_CONTRACT, "packed records need 4- or 8-byte keys with values of the key width");
}

// TuningParams.for_input (params.py:64-86) for the size a rank received.
inline Params params_for(uint64_t m, const ss_params* tmpl) {
  if (!tmpl) throw Fail(SS_ERR_CONFIG, "params must not be NULL");
  ss_params p = *tmpl;
  p.input_size = m;
  const uint64_t nl = p.light_buckets;
  p.subarray_len = std::max<uint64_t>(std::max<uint64_t>(1, cdiv(m, 5000)), nl);
  const double log_n = std::log2(static_cast<double>(std::max<uint64_t>(m, 2)));
  p.sample_count = std::max<uint64_t>(1, static_cast<uint64_t>(std::nearbyint(p.sample_factor * log_n)));
  p.heavy_threshold = log_n;
  p.heavy_threshold_int = std::max<uint64_t>(1, static_cast<uint64_t>(std::ceil(log_n)));
  return to_params(&p, m, true);
}

// Semisort of n packed records in `pairs` (2n key-width words), finishing as
// SoA columns in the same memory: keys = words [0, n), values = [n, 2n).
// scratch: 2n words, or nullptr to carve it from the workspace.
template <typename K>
void semisort_pairs(K* pairs, uint64_t n, int mode, int identity, const Params& P, K* scratch, void* workspace,
                    uint64_t workspace_bytes, ss_telemetry* tel, cudaStream_t st) {
  SortEngine<K, K> e{};
  e.A_k = pairs;
  e.A_v = pairs + n;
  e.n = n;
  e.mode = mode;
  e.identity = identity;
  e.P = P;
  e.st = st;
  e.tel = tel;
  Arena a(workspace, workspace_bytes);
  e.plan(a, scratch == nullptr);
  if (scratch) {
    e.S_k = scratch;
    e.S_v = scratch + n;
  }
  Tracker tr(st, tel);
  const bool pair_path = n >= P.base_case_cutoff && hw_rank_ok() && dist1_tile<K, K>(e.stride, n) != 0;
  if (pair_path) {
    e.R_pairs = pairs;
    e.run(tr);   // picks the pair scratch layout (same conditions)
  } else {
    // small input (the root is a leaf) or no single-pass distribute:
    // unpack through the scratch first, then the ordinary path
    if (n) {
      SS_CUDA(cudaMemcpyAsync(e.S_k, pairs, n * 2 * sizeof(K), cudaMemcpyDeviceToDevice, st));
      k_unpack_pairs<K><<<dgrid(n), 256, 0, st>>>(e.S_k, n, e.A_k, e.A_v);
      check_launch();
      tr.launched();
    }
    e.run_levels(tr);
  }
  tr.finish();
  SS_CUDA(cudaGetLastError());
}

template <typename K>
uint64_t semisort_pairs_ws(uint64_t n, const Params& P, bool with_scratch) {
  SortEngine<K, K> e{};
  e.n = n;
  e.P = P;
  Arena a(nullptr, 0);
  e.plan(a, with_scratch);
  return a.used + 4096;
}

// Stable packed partition: (keys, values) -> pairs grouped by part.
template <typename K>
void partition_pairs(const K* keys, const K* values, uint64_t n, uint32_t parts, K* dst_pairs, uint64_t* out_counts,
                     void* workspace, uint64_t workspace_bytes, cudaStream_t st) {
  PartPlan pp{};
  Arena a(workspace, workspace_bytes);
  pp.carve(a, n, parts);
  if (n == 0) {
    for (uint32_t p = 0; p < parts; ++p) out_counts[p] = 0;
    return;
  }
  if (!hw_rank_ok() || dist1_tile<K, K>(pp.stride, n) == 0)
    throw Fail(SS_ERR_RESOURCE, "packed partition needs the single-pass distribute");
  Node nd{};
  const uint32_t nw = partition_count_scan(pp, keys, n, sizeof(K), parts, nd, st);
  launch_distribute<K, K>(keys, values, pp.d_ids, dst_pairs, dst_pairs + 1, pp.d_work, nw, pp.d_node, pp.d_X,
                          pp.stride, 0xFFFFFFFFu, parts, parts, st, n, pp.d_ctr, 0xFFFFFFFFu, false, true, parts);
  partition_counts(pp, parts, out_counts, st);
}

// ---- NCCL, resolved at run time -------------------------------------------

struct Nccl {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

inline const Nccl& nccl() {
  static Nccl api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) err = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw Fail(SS_ERR_COMM, err);
  return api;
}

inline void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Fail(SS_ERR_COMM, std::string(what) + ": " + nccl().error_string(r));
}

// all-to-allv as grouped point-to-point calls: send[p] = counts[p] elements
// at send + soff[p] to rank p; receive rcounts[p] from rank p at recv +
// roff[p] (source-rank order).
inline void alltoallv(ncclComm_t comm, uint32_t world, const void* send, const std::vector<uint64_t>& scnt,
                      void* recv, const std::vector<uint64_t>& rcnt, size_t elem_bytes, cudaStream_t st) {
  const Nccl& N = nccl();
  uint64_t so = 0, ro = 0;
  nccl_ok(N.group_start(), "ncclGroupStart");
  for (uint32_t p = 0; p < world; ++p) {
    if (scnt[p])
      nccl_ok(N.send(static_cast<const unsigned char*>(send) + so * elem_bytes, scnt[p] * elem_bytes, ncclUint8,
                     static_cast<int>(p), comm, st),
              "ncclSend");
    if (rcnt[p])
      nccl_ok(N.recv(static_cast<unsigned char*>(recv) + ro * elem_bytes, rcnt[p] * elem_bytes, ncclUint8,
                     static_cast<int>(p), comm, st),
              "ncclRecv");
    so += scnt[p];
    ro += rcnt[p];
  }
  nccl_ok(N.group_end(), "ncclGroupEnd");
}

}  // namespace ss

using namespace ss;

extern "C" {

int ss_params_for_input(uint64_t n, const ss_params* tmpl, ss_params* out) {
  return guarded([&] {
    const Params P = params_for(n, tmpl);
    *out = *tmpl;
    out->input_size = n;
    out->subarray_len = P.subarray_len;
    out->sample_count = P.sample_count;
    out->heavy_threshold = P.heavy_threshold;
    out->heavy_threshold_int = P.heavy_threshold_int;
  });
}

uint64_t ss_partition_pairs_workspace_bytes(uint64_t n, uint32_t parts) {
  PartPlan pp{};
  Arena a(nullptr, 0);
  pp.carve(a, n, std::max<uint32_t>(parts, 1));
  return a.used + 4096;
}

int ss_partition_pairs(const void* keys, const void* values, uint64_t n, uint32_t key_bytes, uint32_t parts,
                       void* dst_pairs, uint64_t* out_counts, void* workspace, uint64_t workspace_bytes,
                       void* stream) {
  return guarded([&] {
    if (parts < 1 || (parts & (parts - 1)) || parts > 4096) throw Fail(SS_ERR_CONFIG, "parts must be a power of two <= 4096");
    if (n && (!keys || !values || !dst_pairs)) throw Fail(SS_ERR_CONTRACT, "NULL buffer");
    dispatch_pair(key_bytes, [&]<typename K>() {
      partition_pairs<K>(static_cast<const K*>(keys), static_cast<const K*>(values), n, parts, static_cast<K*>(dst_pairs),
                         out_counts, workspace, workspace_bytes, as_stream(stream));
    });
  });
}

uint64_t ss_semisort_pairs_workspace_bytes(uint64_t n, uint32_t key_bytes, const ss_params* params, int with_scratch) {
  uint64_t out = 0;
  const int rc = guarded([&] {
    const Params P = to_params(params, n, false);
    dispatch_pair(key_bytes, [&]<typename K>() { out = semisort_pairs_ws<K>(n, P, with_scratch != 0); });
  });
  return rc == SS_OK ? out : 0;
}

int ss_semisort_pairs(void* pairs, uint64_t n, uint32_t key_bytes, int mode, int identity, const ss_params* params,
                      void* scratch, void* workspace, uint64_t workspace_bytes, ss_telemetry* telemetry,
                      void* stream) {
  return guarded([&] {
    if (mode != SS_MODE_EQ && mode != SS_MODE_LT) throw Fail(SS_ERR_CONFIG, "mode must be 'eq' or 'lt'");
    const Params P = to_params(params, n, true);
    if (n && !pairs) throw Fail(SS_ERR_CONTRACT, "pairs pointer is NULL");
    reset_tel(telemetry);
    dispatch_pair(key_bytes, [&]<typename K>() {
      semisort_pairs<K>(static_cast<K*>(pairs), n, mode, identity, P, static_cast<K*>(scratch), workspace,
                        workspace_bytes, telemetry, as_stream(stream));
    });
  });
}

int ss_nccl_unique_id(unsigned char* out128) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_ok(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int ss_nccl_comm_init(const unsigned char* id128, int world, int rank, void** out_comm) {
  return guarded([&] {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    nccl_ok(nccl().comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
    *out_comm = c;
  });
}

int ss_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (comm) nccl_ok(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

uint64_t ss_dist_semisort_workspace_bytes(uint64_t capacity, uint32_t key_bytes, uint32_t world,
                                          const ss_params* params) {
  uint64_t out = 0;
  const int rc = guarded([&] {
    const Params P = params_for(capacity, params);
    PartPlan pp{};
    Arena a(nullptr, 0);
    pp.carve(a, capacity, std::max<uint32_t>(world, 1));
    dispatch_pair(key_bytes, [&]<typename K>() {
      out = std::max<uint64_t>(a.used, semisort_pairs_ws<K>(capacity, P, false)) + 2 * 8 * 4096 + 8192;
    });
  });
  return rc == SS_OK ? out : 0;
}

int ss_dist_semisort(void* comm, uint32_t world, uint32_t rank, const void* keys, const void* values, uint64_t n_local,
                     uint32_t key_bytes, int mode, int identity, const ss_params* params, void* recv_block,
                     void* scratch, uint64_t capacity, void* workspace, uint64_t workspace_bytes, uint64_t* out_n,
                     ss_telemetry* telemetry, void* stream) {
  return guarded([&] {
    if (mode != SS_MODE_EQ && mode != SS_MODE_LT) throw Fail(SS_ERR_CONFIG, "mode must be 'eq' or 'lt'");
    if (world < 1 || (world & (world - 1)) || world > 4096 || rank >= world)
      throw Fail(SS_ERR_CONFIG, "world must be a power of two <= 4096 and rank < world");
    if (n_local > capacity) throw Fail(SS_ERR_CONFIG, "n_local exceeds capacity");
    cudaStream_t st = as_stream(stream);
    reset_tel(telemetry);
    dispatch_pair(key_bytes, [&]<typename K>() {
      // counts exchange buffers at the top of the workspace
      unsigned char* ws = static_cast<unsigned char*>(workspace);
      uint64_t* d_cnt = reinterpret_cast<uint64_t*>(ws);
      const uint64_t cnt_bytes = 2 * 8 * 4096;
      if (workspace_bytes < cnt_bytes + 8192) throw Fail(SS_ERR_RESOURCE, "workspace too small");
      void* rest = ws + cnt_bytes;
      const uint64_t rest_bytes = workspace_bytes - cnt_bytes;
      // 1. stable packed partition into the scratch
      std::vector<uint64_t> scnt(world), rcnt(world);
      partition_pairs<K>(static_cast<const K*>(keys), static_cast<const K*>(values), n_local, world,
                         static_cast<K*>(scratch), scnt.data(), rest, rest_bytes, st);
      // 2. per-peer counts
      SS_CUDA(cudaMemcpyAsync(d_cnt, scnt.data(), world * 8, cudaMemcpyHostToDevice, st));
      std::vector<uint64_t> ones(world, 1);
      alltoallv(static_cast<ncclComm_t>(comm), world, d_cnt, ones, d_cnt + 4096, ones, 8, st);
      SS_CUDA(cudaMemcpyAsync(rcnt.data(), d_cnt + 4096, world * 8, cudaMemcpyDeviceToHost, st));
      SS_CUDA(cudaStreamSynchronize(st));
      uint64_t m = 0;
      for (uint64_t c : rcnt) m += c;
      *out_n = m;
      if (m > capacity) throw Fail(SS_ERR_RESOURCE, "received records exceed capacity: " + std::to_string(m));
      // 3. one exchange of packed records, received in source-rank order
      alltoallv(static_cast<ncclComm_t>(comm), world, scratch, scnt, recv_block, rcnt, 2 * sizeof(K), st);
      // 4. local semisort from the packed records (scratch is free again)
      const Params P = params_for(m, params);
      semisort_pairs<K>(static_cast<K*>(recv_block), m, mode, identity, P, static_cast<K*>(scratch), rest, rest_bytes,
                        telemetry, st);
    });
  });
}

}  // extern "C"
