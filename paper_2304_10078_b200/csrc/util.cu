// Device utilities behind the C ABI: synthetic workload generation for the
// benchmark (the reference generator families, datagen.py:72-158), O(n)
// semisort validation, distinct-key counting, and the
// multi-GPU hash partition (stable, so global stability survives the
// exchange).
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "engine.cuh"
#include "multisplit.cuh"
#include "partition.cuh"

namespace ss {

extern thread_local std::string g_last_error;

template <typename F>
int guarded_u(F&& f) {
  try {
    f();
    return SS_OK;
  } catch (const Fail& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SS_ERR_RESOURCE;
  }
}

// ---------------------------------------------------------------------------
// generation
// ---------------------------------------------------------------------------

struct ZipfCfg {
  double s, one_minus, lo, hi, cut, n;
  bool s_is_one;
};

__host__ __device__ inline double zH(const ZipfCfg& z, double x) {
  return z.s_is_one ? log(x) : expm1(z.one_minus * log(x)) / z.one_minus;
}
__host__ __device__ inline double zHinv(const ZipfCfg& z, double x) {
  return z.s_is_one ? exp(x) : exp(log1p(x * z.one_minus) / z.one_minus);
}
__host__ __device__ inline double zh(const ZipfCfg& z, double x) { return exp(-z.s * log(x)); }

inline ZipfCfg make_zipf(double s, uint64_t n) {
  ZipfCfg z{};
  z.s = s;
  z.s_is_one = s == 1.0;
  z.one_minus = 1.0 - s;
  z.n = static_cast<double>(n);
  z.lo = zH(z, 1.5) - 1.0;
  z.hi = zH(z, z.n + 0.5);
  z.cut = 2.0 - zHinv(z, zH(z, 2.5) - zh(z, 2.0));
  return z;
}

__device__ inline double u01(uint64_t w) { return static_cast<double>(w >> 11) * (1.0 / 9007199254740992.0); }

// Rejection-inversion draw of a rank in [1, n] (Hörmann & Derflinger), the
// same sampler the reference uses, driven by a counter-based stream.
__device__ inline uint64_t zipf_draw(const ZipfCfg& z, uint64_t key, uint64_t ctr) {
  for (uint64_t round = 0;; ++round) {
    U64x4 r = philox4x64_10(ctr + (round << 40), key);
    for (int t = 0; t < 4; ++t) {
      double u = z.lo + u01(r.v[t]) * (z.hi - z.lo);
      double x = zHinv(z, u);
      double k = floor(x + 0.5);
      k = k < 1.0 ? 1.0 : (k > z.n ? z.n : k);
      if (k - x <= z.cut || u >= zH(z, k + 0.5) - zh(z, k)) return static_cast<uint64_t>(k);
    }
  }
}

// Key of global record g (a pure function of g: any shard, or any single
// record, regenerates independently).
__device__ inline uint64_t gen_key(int family, double param, const ZipfCfg& z, uint64_t kkey, int hash_ranks,
                                   uint64_t g) {
  U64x4 r = philox4x64_10(g + 1, kkey);
  switch (family) {
    case 0: {   // uniform [0, param)
      uint64_t hi, lo;
      mulhilo64(r.v[0], static_cast<uint64_t>(param), hi, lo);
      return hi;
    }
    case 1:     // floor(exponential(scale = 1/param))
      return static_cast<uint64_t>(floor(-log1p(-u01(r.v[0])) / param));
    case 2: {   // zipf rank in [1, universe]
      const uint64_t k = zipf_draw(z, kkey ^ 0x5A5Aull, g + 1);
      return hash_ranks ? mix64(k - 1) : k;
    }
    case 3:
      return r.v[0];
    default:    // config-5 mix: uniform 64-bit or zipf(param) rank - 1
      return (r.v[1] & 1) ? r.v[0] : zipf_draw(z, kkey ^ 0x5A5Aull, g + 1) - 1;
  }
}

__host__ __device__ inline uint64_t gen_kkey(uint64_t seed, int family) { return mix64_pair(seed, 0xA11CEull + family); }

template <typename K, typename V>
__global__ void k_generate(int family, double param, uint64_t universe, uint64_t n, uint64_t first, uint64_t seed,
                           int hash_ranks, ZipfCfg z, K* __restrict__ keys, V* __restrict__ vals, int values_mode,
                           uint32_t value_shift) {
  const uint64_t kkey = gen_kkey(seed, family);
  const uint64_t vkey = mix64_pair(seed, 0xB0Bull);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t g = first + i;
    keys[i] = static_cast<K>(gen_key(family, param, z, kkey, hash_ranks, g));
    if (values_mode == 1) {
      vals[i] = static_cast<V>(g);
    } else if (values_mode == 2) {
      U64x4 q = philox4x64_10(g + 1, vkey);
      vals[i] = static_cast<V>(q.v[0] >> value_shift);
    }
  }
}

// Shard validation for generated inputs whose value is the global record
// index: record integrity against the generator itself
// (key_out[i] == key(value_out[i])), stability inside runs, dest(key) ==
// rank (top `bits` of mix64), run count, and the permutation fingerprints
// count / sum v / sum v^2 / sum mix64(v) (mod 2^64) that the ranks add up
// and compare with those of [0, N).
// acc: [0] bad record, [1] runs, [2] bad stability, [3] bad dest,
//      [4] sum v, [5] sum v^2, [6] sum mix64(v)
template <typename K>
__global__ void k_validate_shard(int family, double param, ZipfCfg z, uint64_t kkey, int hash_ranks,
                                 const K* __restrict__ ko, const uint64_t* __restrict__ vo, uint64_t m,
                                 uint32_t bits, uint32_t rank, unsigned long long* __restrict__ acc) {
  unsigned long long c[7] = {0, 0, 0, 0, 0, 0, 0};
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = vo[i];
    const K k = ko[i];
    c[0] += static_cast<K>(gen_key(family, param, z, kkey, hash_ranks, v)) != k;
    if (i == 0 || ko[i - 1] != k) ++c[1];
    else c[2] += vo[i - 1] >= v;
    if (bits) c[3] += static_cast<uint32_t>(mix64(static_cast<uint64_t>(k)) >> (64 - bits)) != rank;
    c[4] += v;
    c[5] += v * v;
    c[6] += mix64(v);
  }
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    unsigned long long x = c[j];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(&acc[j], x);
  }
}

// The same fingerprints over the index range [lo, hi).
__global__ void k_index_fingerprint(uint64_t lo, uint64_t hi, unsigned long long* __restrict__ acc) {
  unsigned long long a = 0, b = 0, c = 0;
  for (uint64_t v = lo + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < hi;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    a += v;
    b += v * v;
    c += mix64(v);
  }
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[0], a);
    atomicAdd(&acc[1], b);
    atomicAdd(&acc[2], c);
  }
}

// ---------------------------------------------------------------------------
// validation
// ---------------------------------------------------------------------------

template <typename K, typename V>
__global__ void k_validate(const K* __restrict__ ki, const K* __restrict__ ko, const V* __restrict__ vo, uint64_t n,
                           uint32_t* __restrict__ bitmap, unsigned long long* __restrict__ acc) {
  // acc: [0] bad perm, [1] bad record, [2] runs, [3] bad stability
  __shared__ unsigned long long sacc[4];
  if (threadIdx.x < 4) sacc[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long bp = 0, br = 0, runs = 0, bs = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = static_cast<uint64_t>(vo[i]);
    const K k = ko[i];
    if (v >= n) {
      ++bp;
    } else {
      uint32_t bit = 1u << (v & 31);
      if (atomicOr(&bitmap[v >> 5], bit) & bit) ++bp;
      if (ki[v] != k) ++br;
    }
    if (i == 0 || ko[i - 1] != k) ++runs;
    else if (static_cast<uint64_t>(vo[i - 1]) >= v) ++bs;
  }
  atomicAdd(&sacc[0], bp);
  atomicAdd(&sacc[1], br);
  atomicAdd(&sacc[2], runs);
  atomicAdd(&sacc[3], bs);
  __syncthreads();
  if (threadIdx.x < 4) atomicAdd(&acc[threadIdx.x], sacc[threadIdx.x]);
}

template <typename K>
__global__ void k_count_distinct(const K* __restrict__ keys, uint64_t n, uint64_t* __restrict__ tk,
                                 uint32_t* __restrict__ occ, uint64_t mask, unsigned long long* __restrict__ count) {
  unsigned long long mine = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = static_cast<uint64_t>(keys[i]);
    uint64_t s = mix64(k) & mask;
    while (true) {
      uint32_t o = atomicAdd(&occ[s], 0u);
      if (o == 0) {
        if (atomicCAS(&occ[s], 0u, 1u) == 0u) {
          tk[s] = k;
          __threadfence();
          atomicExch(&occ[s], 2u);
          ++mine;
          break;
        }
        continue;
      }
      while (o == 1) o = atomicAdd(&occ[s], 0u);
      // the key was published by another SM: read it from L2, not a stale L1 line
      if (__ldcg(&tk[s]) == k) break;
      s = (s + 1) & mask;
    }
  }
  atomicAdd(count, mine);
}

// ---------------------------------------------------------------------------
// partition by the top bits of mix64(key)
// ---------------------------------------------------------------------------

inline uint32_t ugrid(uint64_t n) {
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(148 * 16, cdiv(n, 256))));
}

}  // namespace ss

using namespace ss;

extern "C" {

int ss_generate(int family, double param, uint64_t universe, uint64_t n, uint64_t first_index, uint32_t key_bytes,
                uint64_t seed, int hash_ranks, void* out_keys, void* out_values, uint32_t value_bytes,
                int values_mode, uint32_t value_shift, void* stream) {
  return guarded_u([&] {
    if (family < 0 || family > 4) throw Fail(SS_ERR_CONFIG, "unknown family");
    if ((family == 2 || family == 4) && (param <= 0 || universe < 1)) throw Fail(SS_ERR_CONFIG, "bad zipf parameters");
    if (family == 0 && param < 1) throw Fail(SS_ERR_CONFIG, "uniform mu must be >= 1");
    if (family == 1 && param <= 0) throw Fail(SS_ERR_CONFIG, "exponential lambda must be > 0");
    if (values_mode && value_bytes != 4 && value_bytes != 8) throw Fail(SS_ERR_CONTRACT, "value_bytes must be 4 or 8");
    ZipfCfg z = make_zipf((family == 2 || family == 4) ? param : 1.2, std::max<uint64_t>(universe, 2));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t grid = ugrid(n);
    auto go = [&](auto kt, auto vt) {
      using K = decltype(kt);
      using V = decltype(vt);
      k_generate<K, V><<<grid, 256, 0, st>>>(family, param, universe, n, first_index, seed, hash_ranks, z,
                                             static_cast<K*>(out_keys), static_cast<V*>(out_values), values_mode,
                                             value_shift);
    };
    if (key_bytes == 8) {
      if (value_bytes == 4) go(uint64_t{}, uint32_t{});
      else go(uint64_t{}, uint64_t{});
    } else if (key_bytes == 4) {
      if (value_bytes == 8) go(uint32_t{}, uint64_t{});
      else go(uint32_t{}, uint32_t{});
    } else {
      throw Fail(SS_ERR_CONTRACT, "key_bytes must be 4 or 8");
    }
    check_launch();
  });
}

int ss_validate_shard(int family, double param, uint64_t universe, uint64_t seed, int hash_ranks,
                      const void* keys_out, const void* values_out, uint64_t m, uint32_t key_bytes, uint32_t parts,
                      uint32_t rank, void* workspace, uint64_t workspace_bytes, uint64_t* out, void* stream) {
  return guarded_u([&] {
    if (family < 0 || family > 4) throw Fail(SS_ERR_CONFIG, "unknown family");
    if (parts < 1 || (parts & (parts - 1)) || rank >= parts) throw Fail(SS_ERR_CONFIG, "bad parts / rank");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(workspace, workspace_bytes);
    unsigned long long* acc = a.take<unsigned long long>(8);
    SS_CUDA(cudaMemsetAsync(acc, 0, 8 * 8, st));
    uint32_t bits = 0;
    while ((1u << bits) < parts) ++bits;
    ZipfCfg z = make_zipf((family == 2 || family == 4) ? param : 1.2, std::max<uint64_t>(universe, 2));
    const uint64_t kkey = gen_kkey(seed, family);
    if (m) {
      if (key_bytes == 8)
        k_validate_shard<uint64_t><<<ugrid(m), 256, 0, st>>>(family, param, z, kkey, hash_ranks,
                                                             static_cast<const uint64_t*>(keys_out),
                                                             static_cast<const uint64_t*>(values_out), m, bits, rank, acc);
      else if (key_bytes == 4)
        k_validate_shard<uint32_t><<<ugrid(m), 256, 0, st>>>(family, param, z, kkey, hash_ranks,
                                                             static_cast<const uint32_t*>(keys_out),
                                                             static_cast<const uint64_t*>(values_out), m, bits, rank, acc);
      else
        throw Fail(SS_ERR_CONTRACT, "key_bytes must be 4 or 8");
      check_launch();
    }
    unsigned long long h[8];
    SS_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < 7; ++j) out[j] = h[j];
  });
}

int ss_index_fingerprint(uint64_t lo, uint64_t hi, void* workspace, uint64_t workspace_bytes, uint64_t* out,
                         void* stream) {
  return guarded_u([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(workspace, workspace_bytes);
    unsigned long long* acc = a.take<unsigned long long>(4);
    SS_CUDA(cudaMemsetAsync(acc, 0, 4 * 8, st));
    if (hi > lo) {
      k_index_fingerprint<<<ugrid(hi - lo), 256, 0, st>>>(lo, hi, acc);
      check_launch();
    }
    unsigned long long h[4];
    SS_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    for (int j = 0; j < 3; ++j) out[j] = h[j];
  });
}

uint64_t ss_validate_workspace_bytes(uint64_t n) { return (n / 32 + 1) * 4 + 4096; }

int ss_validate_indexed(const void* keys_in, const void* keys_out, const void* values_out, uint64_t n,
                        uint32_t key_bytes, uint32_t value_bytes, uint64_t distinct_keys, void* workspace,
                        uint64_t workspace_bytes, int32_t* out_flags, void* stream) {
  return guarded_u([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Arena a(workspace, workspace_bytes);
    uint32_t* bitmap = a.take<uint32_t>(n / 32 + 1);
    unsigned long long* acc = a.take<unsigned long long>(4);
    SS_CUDA(cudaMemsetAsync(bitmap, 0, (n / 32 + 1) * 4, st));
    SS_CUDA(cudaMemsetAsync(acc, 0, 32, st));
    auto go = [&](auto kt, auto vt) {
      using K = decltype(kt);
      using V = decltype(vt);
      k_validate<K, V><<<ugrid(n), 256, 0, st>>>(static_cast<const K*>(keys_in), static_cast<const K*>(keys_out),
                                                 static_cast<const V*>(values_out), n, bitmap, acc);
    };
    if (key_bytes == 8 && value_bytes == 8) go(uint64_t{}, uint64_t{});
    else if (key_bytes == 8 && value_bytes == 4) go(uint64_t{}, uint32_t{});
    else if (key_bytes == 4 && value_bytes == 4) go(uint32_t{}, uint32_t{});
    else if (key_bytes == 4 && value_bytes == 8) go(uint32_t{}, uint64_t{});
    else throw Fail(SS_ERR_CONTRACT, "validation needs 4/8-byte keys and index values");
    check_launch();
    unsigned long long h[4];
    SS_CUDA(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    out_flags[0] = h[0] == 0;
    out_flags[1] = h[1] == 0;
    out_flags[2] = n == 0 ? 1 : (h[2] == distinct_keys);
    out_flags[3] = h[3] == 0;
  });
}

uint64_t ss_count_distinct_workspace_bytes(uint64_t n) {
  uint64_t cap = pow2_ge(std::max<uint64_t>(2 * n, 64));
  return cap * 12 + 8192;
}

int ss_count_distinct(const void* keys, uint64_t n, uint32_t key_bytes, void* workspace, uint64_t workspace_bytes,
                      uint64_t* out_count, void* stream) {
  return guarded_u([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint64_t cap = pow2_ge(std::max<uint64_t>(2 * n, 64));
    Arena a(workspace, workspace_bytes);
    uint64_t* tk = a.take<uint64_t>(cap);
    uint32_t* occ = a.take<uint32_t>(cap);
    unsigned long long* cnt = a.take<unsigned long long>(1);
    SS_CUDA(cudaMemsetAsync(occ, 0, cap * 4, st));
    SS_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
    if (key_bytes == 8)
      k_count_distinct<uint64_t><<<ugrid(n), 256, 0, st>>>(static_cast<const uint64_t*>(keys), n, tk, occ, cap - 1, cnt);
    else if (key_bytes == 4)
      k_count_distinct<uint32_t><<<ugrid(n), 256, 0, st>>>(static_cast<const uint32_t*>(keys), n, tk, occ, cap - 1, cnt);
    else
      throw Fail(SS_ERR_CONTRACT, "key_bytes must be 4 or 8");
    check_launch();
    unsigned long long h = 0;
    SS_CUDA(cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    *out_count = h;
  });
}

uint64_t ss_partition_workspace_bytes(uint64_t n, uint32_t parts) {
  PartPlan pp{};
  Arena a(nullptr, 0);
  pp.carve(a, n, std::max<uint32_t>(parts, 1));
  return a.used + 4096;
}

int ss_partition(const void* keys, const void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                 uint32_t parts, void* dst_keys, void* dst_values, uint64_t* out_counts, void* workspace,
                 uint64_t workspace_bytes, void* stream) {
  return guarded_u([&] {
    if (parts < 1 || (parts & (parts - 1)) || parts > 4096) throw Fail(SS_ERR_CONFIG, "parts must be a power of two <= 4096");
    check_widths(key_bytes, value_bytes);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PartPlan pp{};
    Arena a(workspace, workspace_bytes);
    pp.carve(a, n, parts);
    if (n == 0) {
      for (uint32_t p = 0; p < parts; ++p) out_counts[p] = 0;
      return;
    }
    Node nd{};
    const uint32_t nw = partition_count_scan(pp, keys, n, key_bytes, parts, nd, st);
    auto go = [&](auto kt, auto vt) {
      using K = decltype(kt);
      using V = decltype(vt);
      constexpr int kTile = 2048;   // parts <= 4096 always fit this tile
      const size_t dsm = DistCfg<K, V, kTile, 512, 2>::smem_bytes(pp.stride);
      auto kern = k_distribute<K, V, kTile, 512, 2, false>;
      SS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm)));
      SS_CUDA(cudaMemsetAsync(pp.d_ctr, 0, sizeof(uint32_t), st));
      kern<<<std::min<uint32_t>(nw, 148), 512 + 32, dsm, st>>>(   // + producer warp
          static_cast<const K*>(keys), static_cast<const V*>(values), pp.d_ids, n, static_cast<K*>(dst_keys),
          static_cast<V*>(dst_values), pp.d_work, nw, pp.d_node, pp.d_X, pp.stride, 0xFFFFFFFFu, 0, parts,
          pp.d_ctr);
    };
    auto withv = [&](auto kt) {
      using K = decltype(kt);
      switch (value_bytes) {
        case 0: go(K{}, NoVal{}); break;
        case 4: go(K{}, uint32_t{}); break;
        case 8: go(K{}, uint64_t{}); break;
        default: go(K{}, V16{}); break;
      }
    };
    if (key_bytes == 8) withv(uint64_t{});
    else withv(uint32_t{});
    check_launch();
    partition_counts(pp, parts, out_counts, st);
  });
}

}  // extern "C"
