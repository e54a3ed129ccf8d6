// Host-side runtime shared by the C-ABI entry points: error plumbing,
// workspace arena, parameter validation, launch accounting and per-phase
// device timing.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "semisort_b200.h"
#include "common.cuh"
#include "types.cuh"

namespace ss {

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SS_CUDA(x)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw ::ss::Fail(SS_ERR_RESOURCE, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
inline uint64_t pow2_ge(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Bump allocator over the caller's workspace.  With base == nullptr it only
// measures (size queries use the same code path as the real carve).
struct Arena {
  char* base;
  uint64_t cap;
  uint64_t used = 0;
  Arena(void* b, uint64_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(uint64_t count) {
    used = (used + 255) & ~uint64_t(255);
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += std::max<uint64_t>(count, 1) * sizeof(T);
    if (base && used > cap)
      throw Fail(SS_ERR_RESOURCE, "workspace too small: need more than " + std::to_string(cap) + " bytes");
    return p;
  }
};

inline Params to_params(const ss_params* p, uint64_t n, bool check_n) {
  if (!p) throw Fail(SS_ERR_CONFIG, "params must not be NULL");
  Params P{};
  P.input_size = p->input_size;
  P.light_buckets = p->light_buckets;
  P.light_bits = p->light_bits;
  P.subarray_len = p->subarray_len;
  P.base_case_cutoff = p->base_case_cutoff;
  P.max_heavy = p->max_heavy;
  P.sample_factor = p->sample_factor;
  P.seed = p->seed;
  P.sample_count = p->sample_count;
  P.heavy_threshold_int = p->heavy_threshold_int;
  P.heavy_threshold = p->heavy_threshold;
  const uint32_t nl = P.light_buckets;
  if (nl < 1 || (nl & (nl - 1)))
    throw Fail(SS_ERR_CONFIG, "light_buckets must be a power of two, got " + std::to_string(nl));
  if (nl != (1u << P.light_bits)) throw Fail(SS_ERR_CONFIG, "light_bits inconsistent with light_buckets");
  if (P.subarray_len < nl) throw Fail(SS_ERR_CONFIG, "subarray_len smaller than light_buckets");
  if (P.base_case_cutoff < 1) throw Fail(SS_ERR_CONFIG, "base_case_cutoff must be >= 1");
  if (nl > 4096)
    throw Fail(SS_ERR_CONFIG, "light_buckets > 4096 exceeds the per-CTA shared-memory histograms of the GPU path");
  if (P.max_heavy > static_cast<uint32_t>(kMaxHeavyDevice))
    throw Fail(SS_ERR_CONFIG, "max_heavy > 512 exceeds the shared-memory heavy table of the GPU path");
  if (check_n && P.input_size != n)
    throw Fail(SS_ERR_CONFIG, "params derived for n=" + std::to_string(P.input_size) + " used on n=" +
                                  std::to_string(n));
  if (P.heavy_threshold_int == 0) P.heavy_threshold_int = 1;
  return P;
}

inline void check_widths(uint32_t kb, uint32_t vb, bool allow_u128 = false) {
  if (kb != 4 && kb != 8 && !(allow_u128 && kb == 16))
    throw Fail(SS_ERR_CONTRACT, allow_u128 ? "key_bytes must be 4, 8 or 16" : "key_bytes must be 4 or 8");
  if (vb != 0 && vb != 4 && vb != 8 && vb != 16)
    throw Fail(SS_ERR_CONTRACT, "value_bytes must be 0, 4, 8 or 16");
}

inline uint32_t rounds_per_hash(uint32_t light_bits) { return std::max(1u, 64u / std::max(light_bits, 1u)); }

inline uint32_t even_stride(const Params& P) { return (P.light_buckets + P.max_heavy + 1) & ~1u; }

// Launch accounting + optional per-phase CUDA-event timing.
enum Phase { kPhSample = 0, kPhCount, kPhScan, kPhDistribute, kPhCopy, kPhChildren, kPhLeaves, kPhOther };

struct Tracker {
  cudaStream_t st;
  ss_telemetry* tel;
  bool timing;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> spans;
  int open_phase = -1;
  cudaEvent_t open_ev = nullptr;

  Tracker(cudaStream_t s, ss_telemetry* t) : st(s), tel(t), timing(t && t->timing) {}
  void launched(uint64_t k = 1) {
    if (tel) tel->kernel_launches += k;
  }
  void begin(int ph) {
    if (!timing) return;
    end();
    SS_CUDA(cudaEventCreate(&open_ev));
    SS_CUDA(cudaEventRecord(open_ev, st));
    open_phase = ph;
  }
  void end() {
    if (!timing || open_phase < 0) return;
    cudaEvent_t e;
    SS_CUDA(cudaEventCreate(&e));
    SS_CUDA(cudaEventRecord(e, st));
    spans.push_back({open_phase, {open_ev, e}});
    open_phase = -1;
  }
  void finish() {
    if (!timing) return;
    end();
    SS_CUDA(cudaStreamSynchronize(st));
    for (auto& s : spans) {
      float ms = 0;
      SS_CUDA(cudaEventElapsedTime(&ms, s.second.first, s.second.second));
      tel->phase_ms[s.first] += ms;
      cudaEventDestroy(s.second.first);
      cudaEventDestroy(s.second.second);
    }
    spans.clear();
  }
  ~Tracker() {
    for (auto& s : spans) {
      cudaEventDestroy(s.second.first);
      cudaEventDestroy(s.second.second);
    }
    if (open_phase >= 0 && open_ev) cudaEventDestroy(open_ev);
  }
};

inline void check_launch() { SS_CUDA(cudaGetLastError()); }

template <typename F>
int guarded(F&& f);

}  // namespace ss
