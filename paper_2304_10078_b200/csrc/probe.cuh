// Load-time probe of the hardware rank property the distribute kernels' fast
// paths rely on (dist.cuh radix_rank<HW = true>, dist1.cuh): a shared
// atomicAdd returns, to the lanes of one warp instruction that hit the same
// counter, old values accumulated in lane order -- for +1 counters and for
// u16 pairs packed in one word (+1 / +65536).  The probe compares those values
// with ranks from __match_any_sync on random and skewed digits; any
// mismatch (or SS_HW_RANK=0) selects the atomicOr-mask path instead.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace ss {

constexpr int kProbeBins = 128;

static __global__ void __launch_bounds__(512) k_probe_hw_rank(unsigned long long* bad, int iters) {
  __shared__ uint32_t cnt[16][kProbeBins];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  for (int i = lane; i < kProbeBins; i += 32) cnt[w][i] = 0;
  __syncwarp();
  uint64_t x = (static_cast<uint64_t>(blockIdx.x) << 32) | threadIdx.x;
  uint32_t nbad = 0;
  for (int it = 0; it < iters; ++it) {
    x = mix64(x + it);
    const uint32_t hot = (it >> 6) % 4;   // 0%, ~50%, ~90%, 100% of lanes on 4 digits
    const uint32_t r = static_cast<uint32_t>(x >> 8) % 100u;
    const bool on_hot = hot == 3 || (hot == 1 && r < 50) || (hot == 2 && r < 90);
    const uint32_t d = on_hot ? static_cast<uint32_t>(x & 3) * 37u : static_cast<uint32_t>(x >> 40) % kProbeBins;
    const bool active = ((x >> 20) & 7) != 0;
    const uint32_t peers = __match_any_sync(0xffffffffu, active ? d : 0x10000u + lane);
    // +1 counters (radix_rank) and u16 pairs packed in one word (+1 low /
    // +65536 high, dist1.cuh) must both hand out lane-ordered old values
    const bool packed = (it & 1) != 0;
    uint32_t* word = packed ? &cnt[w][d >> 1] : &cnt[w][d];
    const uint32_t sh = packed ? 16u * (d & 1u) : 0u;
    const uint32_t before = *word;
    __syncwarp();
    uint32_t old = 0;
    if (active) old = atomicAdd(word, 1u << sh);
    __syncwarp();
    const uint32_t got = packed ? (old >> sh) & 0xFFFFu : old;
    const uint32_t want = (packed ? (before >> sh) & 0xFFFFu : before) + __popc(peers & lt);
    if (active && got != want) ++nbad;
    __syncwarp();
    if (packed && lane == 0) {   // keep packed halves far from overflow
      for (int i = 0; i < kProbeBins; ++i) cnt[w][i] &= 0x00FF00FFu;
    }
    __syncwarp();
  }
  if (nbad) atomicAdd(bad, static_cast<unsigned long long>(nbad));
}

inline bool hw_rank_probe() {
  unsigned long long* d_bad = nullptr;
  if (cudaMalloc(&d_bad, sizeof(unsigned long long)) != cudaSuccess) return false;
  unsigned long long h_bad = 1;
  bool ok = cudaMemset(d_bad, 0, sizeof(unsigned long long)) == cudaSuccess;
  if (ok) {
    k_probe_hw_rank<<<4, 512>>>(d_bad, 4096);
    ok = cudaGetLastError() == cudaSuccess &&
         cudaMemcpy(&h_bad, d_bad, sizeof(h_bad), cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaFree(d_bad);
  return ok && h_bad == 0;
}

// Probed once per process; SS_HW_RANK=0 forces the fallback (tests use it).
inline bool hw_rank_ok() {
  static const bool probed = hw_rank_probe();
  const char* e = std::getenv("SS_HW_RANK");
  if (e && e[0] == '0') return false;
  return probed;
}

}  // namespace ss
