// Bulk-async (TMA 1-D) global->shared copies tracked by an mbarrier
// (cp.async.bulk + mbarrier complete_tx), for the streaming kernels.
#pragma once

#include <cstdint>

namespace ss {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Orders this thread's prior generic-proxy shared accesses before later
// async-proxy (bulk copy) accesses.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// L2 policy for streamed-once inputs: evict first, so scattered partial
// writes elsewhere in the kernel keep their lines until they complete.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// L2 prefetch of a 16-byte aligned global range (no shared memory, no barrier).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2_hint(const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(pol) : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Plain arrival (no transaction bytes): completes a count-1 phase.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Bulk-copy plan for elements [begin, begin+cnt) of a T array of n_total
// elements: one TMA copy of the 16-byte aligned superset of the range.
// Element i of the range lands at index i + sh of the (16-byte aligned)
// shared buffer.  When the superset would leave the array (misaligned array
// start or end only), `ok` is false and consumers read global memory
// directly for that tile -- the producer never does synchronous loads.
template <typename T>
struct Bulk16 {
  const unsigned char* src;
  uint32_t bytes, sh;
  bool ok;
  __device__ __forceinline__ Bulk16(const T* base, uint64_t n_total, uint64_t begin, uint32_t cnt) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(base), a1 = reinterpret_cast<uintptr_t>(base + n_total);
    const uintptr_t a = reinterpret_cast<uintptr_t>(base + begin), e = reinterpret_cast<uintptr_t>(base + begin + cnt);
    const uintptr_t lo = a & ~uintptr_t(15), hi = (e + 15) & ~uintptr_t(15);
    ok = cnt > 0 && lo >= a0 && hi <= a1;
    src = reinterpret_cast<const unsigned char*>(lo);
    bytes = ok ? static_cast<uint32_t>(hi - lo) : 0u;
    sh = static_cast<uint32_t>((a - lo) / sizeof(T));
  }
};

// Split [begin, begin+cnt) of a T array into an unaligned head, a 16-byte
// aligned bulk body and a tail.  `sh` is the element shift that makes the
// body land 16-byte aligned in shared memory (element i of the range is
// stored at index i + sh of a 16-byte aligned buffer).
template <typename T>
struct Span16 {
  uint32_t sh, head, body;
  __device__ __forceinline__ Span16(const T* base, uint64_t begin, uint32_t cnt) {
    constexpr uint32_t per = 16 / sizeof(T) > 0 ? 16 / sizeof(T) : 1;
    const uint32_t mis = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(base + begin) & 15u) / sizeof(T));
    sh = mis;
    head = mis ? min(per - mis, cnt) : 0;
    body = ((cnt - head) / per) * per;
  }
};

// Issued by one thread: bulk copy of the body (returns its bytes, already
// armed on `bar` by the caller) plus synchronous head/tail element copies.
template <typename T>
__device__ __forceinline__ void stage_span(T* buf, const T* src, uint64_t begin, uint32_t cnt, uint64_t* bar) {
  Span16<T> sp(src, begin, cnt);
  if (sp.body) bulk_g2s(buf + sp.sh + sp.head, src + begin + sp.head, sp.body * sizeof(T), bar);
  for (uint32_t i = 0; i < sp.head; ++i) buf[sp.sh + i] = src[begin + i];
  for (uint32_t i = sp.head + sp.body; i < cnt; ++i) buf[sp.sh + i] = src[begin + i];
}

template <typename T>
__device__ __forceinline__ uint32_t span_body_bytes(const T* src, uint64_t begin, uint32_t cnt) {
  Span16<T> sp(src, begin, cnt);
  return sp.body * sizeof(T);
}

}  // namespace ss
