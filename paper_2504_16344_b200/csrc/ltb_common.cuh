// ltb_common.cuh -- shared device helpers for the B200 (sm_100a) hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define LTB_DEV __device__ __forceinline__

namespace ltb {

// complex FP64 as double2 (x = re, y = im); F-hat and all spectra use the
// same interleaved layout as std::complex<double> / fftw_complex.
LTB_DEV double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
LTB_DEV double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
LTB_DEV double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
LTB_DEV double2 conjg(double2 a) { return make_double2(a.x, -a.y); }

// acc += a * x
LTB_DEV void cmac(double2& acc, double2 a, double2 x) {
  acc.x = fma(a.x, x.x, acc.x);
  acc.x = fma(-a.y, x.y, acc.x);
  acc.y = fma(a.x, x.y, acc.y);
  acc.y = fma(a.y, x.x, acc.y);
}
// acc += conj(a) * x
LTB_DEV void cmac_conj(double2& acc, double2 a, double2 x) {
  acc.x = fma(a.x, x.x, acc.x);
  acc.x = fma(a.y, x.y, acc.x);
  acc.y = fma(a.x, x.y, acc.y);
  acc.y = fma(-a.y, x.x, acc.y);
}

// Streaming read of F-hat: read-only path, do not allocate in L1 (every
// byte is touched exactly once per matvec).
LTB_DEV double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}
// 256-bit streaming read (sm_100a LDG.E.NA.256): two consecutive complex
// values, 32-byte aligned, L2 evict-first so the stream does not push the
// small re-read vectors out of L2.
LTB_DEV void ld_stream2(const double2* p, double2& a, double2& b) {
  long long r0, r1, r2, r3;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.b64 {%0,%1,%2,%3}, [%4];"
               : "=l"(r0), "=l"(r1), "=l"(r2), "=l"(r3)
               : "l"(p));
  a = make_double2(__longlong_as_double(r0), __longlong_as_double(r1));
  b = make_double2(__longlong_as_double(r2), __longlong_as_double(r3));
}

LTB_DEV double shfl_xor_d(double v, int m, int width = 32) {
  return __shfl_xor_sync(0xffffffffu, v, m, width);
}

// ---- bulk async copy (TMA 1-D, cp.async.bulk) + mbarrier helpers ----
LTB_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

LTB_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
LTB_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// arrive (count 1) and register `bytes` of expected transaction volume
LTB_DEV void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// global -> shared bulk copy completing on `bar`; 16-byte aligned, size % 16 == 0
LTB_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

LTB_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

LTB_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LTB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LTB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace ltb
