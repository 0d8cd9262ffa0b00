// Shared device helpers for the im2win sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define IM2WIN_DEVICE __device__ __forceinline__

// Records which kernel the last library call on this host thread launched
// (im2win_last_kernel(); capi.cu).  Static strings only.
void im2win_note_kernel(const char* name);
// relabel the call's kernel without counting a launch (a call made of several launches)
void im2win_label_kernel(const char* name);

namespace im2win {

// Unsigned division by a runtime-invariant divisor via multiply-high
// (round-up method).  Exact for 0 <= n < 2^31 and 1 <= d < 2^31.
struct FastDiv {
  uint32_t d;
  uint32_t mul;
  uint32_t shr;

  FastDiv() = default;
  __host__ __device__ explicit FastDiv(uint32_t divisor) : d(divisor), mul(0), shr(0) {
    while ((1ull << shr) < divisor) ++shr;
    mul = static_cast<uint32_t>(((1ull << 32) * ((1ull << shr) - divisor)) / divisor + 1);
  }
  IM2WIN_DEVICE uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shr; }
  IM2WIN_DEVICE void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

IM2WIN_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 4-byte async copy global->shared (L1-allocating); src_bytes==0 zero-fills.
IM2WIN_DEVICE void cp_async_4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}

// 4-byte async copy with an ignore-src predicate: zero-fills when `zero` is true.
IM2WIN_DEVICE void cp_async_4_zfill(uint32_t dst, const void* src, bool zero) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "cp.async.ca.shared.global [%0], [%1], 4, p;\n\t}\n" ::"r"(dst),
      "l"(src), "r"(static_cast<int>(zero)));
}

// 16-byte async copy (L2 only); src_bytes==0 zero-fills.
IM2WIN_DEVICE void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes));
}

IM2WIN_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// mbarrier primitives for cp.async pipelines (SIMT kernels).
IM2WIN_DEVICE void mbarrier_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
IM2WIN_DEVICE void mbarrier_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
IM2WIN_DEVICE void mbarrier_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Arrive on `bar` once all of this thread's prior cp.async copies have landed.
IM2WIN_DEVICE void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int N>
IM2WIN_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace im2win
