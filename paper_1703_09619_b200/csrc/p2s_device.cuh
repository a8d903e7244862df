// p2s_device.cuh -- sm_100a device helpers: compile-time loops, mbarrier and
// bulk-copy (TMA engine, cp.async.bulk) wrappers.
#pragma once

#include <cstdint>
#include <type_traits>
#include <utility>

namespace p2s {

// ---------------------------------------------------------------- static_for
template <int Begin, int End, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (Begin < End) {
    f(std::integral_constant<int, Begin>{});
    static_for<Begin + 1, End>(static_cast<F&&>(f));
  }
}

// Work items 0..N-1 over THREADS threads as ceil(N/THREADS) unrolled rounds
// (no runtime loop: keeps ptxas from hoisting per-item constant-bank loads
// into registers across items).
template <int N, int THREADS, class F>
__device__ __forceinline__ void for_items(F&& body) {
  static_for<0, (N + THREADS - 1) / THREADS>([&](auto rc) {
    const int f = decltype(rc)::value * THREADS + static_cast<int>(threadIdx.x);
    if (f < N) body(f);
  });
}

// ---------------------------------------------------------------- smem / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// 1-D bulk copy global -> shared through the TMA engine (UBLKCP); bytes and
// both addresses must be multiples of 16.  Completion is signalled on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy shared -> global through the TMA engine (UBLKCP), evict-first in
// L2 (the element matrices are written once); bytes and both addresses multiples
// of 16.  Completion is tracked per thread in bulk groups (commit / wait below).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N of this thread's bulk groups are still READING shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Prefetch the line holding p into L1 (no register, no scoreboard).
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Bulk prefetch of global memory into L2 (bytes multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Streaming (evict-first) 8-byte store: element matrices are written once and
// never re-read by the fill.
#ifdef P2S_STORE_WB
__device__ __forceinline__ void st_cs(double* p, double v) { *p = v; }
__device__ __forceinline__ void st_cs2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
#else
__device__ __forceinline__ void st_cs(double* p, double v) { __stcs(p, v); }
// 16-B streaming store of two adjacent doubles (p 16-B aligned)
__device__ __forceinline__ void st_cs2(double* p, double a, double b) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(a, b));
}
#endif

// 32-B read-only load of four adjacent doubles (p 32-B aligned; sm_100 LDG.256)
__device__ __forceinline__ void ld_nc4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}

// 8-B read-only load that does not allocate in L1: alpha is read once, and a
// kernel that spills keeps its local-memory lines in the (small, mostly carved
// out for shared memory) L1 instead of losing them to the alpha stream
__device__ __forceinline__ double ld_nc_na(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// 32-B streaming store of four adjacent doubles (p 32-B aligned; sm_100 STG.256)
__device__ __forceinline__ void st_cs4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
// four adjacent doubles with the widest store the alignment allows (w = 4, 2 or 1)
__device__ __forceinline__ void st_cs_n(double* p, const double* v, int w) {
  if (w >= 4) {
    st_cs4(p, v[0], v[1], v[2], v[3]);
  } else if (w == 2) {
    st_cs2(p, v[0], v[1]);
    st_cs2(p + 2, v[2], v[3]);
  } else {
    st_cs(p, v[0]);
    st_cs(p + 1, v[1]);
    st_cs(p + 2, v[2]);
    st_cs(p + 3, v[3]);
  }
}

}  // namespace p2s
