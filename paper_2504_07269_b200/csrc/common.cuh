// Shared helpers for the stfem_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <string>

#include "../../include/stfem_b200.h"

namespace stfem {

// ---- error reporting (thread-local message behind stfem_last_error) -------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define STFEM_CUDA_TRY(expr)                                          \
  do {                                                                \
    cudaError_t _e = (expr);                                          \
    if (_e != cudaSuccess) return ::stfem::cuda_fail(_e, #expr);      \
  } while (0)

#define STFEM_LAUNCH_CHECK(where)                                     \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::stfem::cuda_fail(_e, where);      \
  } while (0)

// Per-device "first use" latch for cudaFuncSetAttribute opt-ins: function attributes are per
// device, so a process that moves to another GPU must set them again there.
//   static DeviceOnce once;  if (once.first()) { cudaFuncSetAttribute(...); }
struct DeviceOnce {
  std::atomic<uint64_t> mask{0};
  bool first() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
    const uint64_t bit = 1ull << dev;
    return (mask.fetch_or(bit) & bit) == 0;
  }
};

// ---- complex128 as double2 ------------------------------------------------
struct __align__(16) cplx {
  double re, im;
};

__host__ __device__ __forceinline__ cplx cmk(double r, double i) { return cplx{r, i}; }
__host__ __device__ __forceinline__ cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
__host__ __device__ __forceinline__ cplx csub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
__host__ __device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return cplx{fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
// a - b*c
__host__ __device__ __forceinline__ cplx cfms(cplx a, cplx b, cplx c) {
  return cplx{fma(-b.im, -c.im, fma(-b.re, c.re, a.re)), fma(-b.re, c.im, fma(-b.im, c.re, a.im))};
}
// a + b*c
__host__ __device__ __forceinline__ cplx cfma(cplx b, cplx c, cplx a) {
  return cplx{fma(-b.im, c.im, fma(b.re, c.re, a.re)), fma(b.re, c.im, fma(b.im, c.re, a.im))};
}
__host__ __device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  // Smith's algorithm
  if (fabs(b.re) >= fabs(b.im)) {
    double r = b.im / b.re, den = b.re + b.im * r;
    return cplx{(a.re + a.im * r) / den, (a.im - a.re * r) / den};
  } else {
    double r = b.re / b.im, den = b.re * r + b.im;
    return cplx{(a.re * r + a.im) / den, (a.im * r - a.re) / den};
  }
}
__host__ __device__ __forceinline__ cplx crecip(cplx b) { return cdiv(cplx{1.0, 0.0}, b); }
// 1/b with one division: conj(b)/|b|^2 (pivots here are far from over/underflow)
// principal square root (branch cut on the negative real axis)
__host__ __device__ __forceinline__ cplx csqrt_(cplx z) {
  const double r = hypot(z.re, z.im);
  if (r == 0.0) return cplx{0.0, 0.0};
  if (z.re >= 0.0) {
    const double t = sqrt(0.5 * (r + z.re));
    return cplx{t, z.im / (2.0 * t)};
  }
  const double t = sqrt(0.5 * (r - z.re));
  return cplx{fabs(z.im) / (2.0 * t), z.im >= 0.0 ? t : -t};
}
__host__ __device__ __forceinline__ cplx crecip_fast(cplx b) {
  double s = 1.0 / fma(b.re, b.re, b.im * b.im);
  return cplx{b.re * s, -b.im * s};
}
__host__ __device__ __forceinline__ double cabs2(cplx a) { return a.re * a.re + a.im * a.im; }

#ifdef __CUDACC__
__device__ __forceinline__ cplx ldc(const cplx* p) {
  double2 v = *reinterpret_cast<const double2*>(p);
  return cplx{v.x, v.y};
}
__device__ __forceinline__ void stc(cplx* p, cplx v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.re, v.im);
}

// ---- FP64 tensor core: mma.sync m16n8k4 f64 (lowers to DMMA on sm_100a) ---
// Fragment layout (CuTe SM90_16x8x4_F64F64F64F64_TN):
//   g = lane>>2, t = lane&3
//   A (16x4, row): a0 = A[g][t], a1 = A[g+8][t]
//   B (4x8, col):  b0 = B[t][g]
//   C (16x8):      c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1]
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// ---- cp.async 16-byte with zero fill ---------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
// 8-byte variant (one double; .ca: the 16-byte-only .cg form does not exist for 8 bytes)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- mbarrier + 1-D bulk copies (the TMA engine) --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.b32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// a wait that cannot hang the GPU: a protocol bug traps (kernel error) instead of spinning forever
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  for (uint32_t spin = 0; !mbar_try_wait(b, parity); ++spin)
    if (spin > (1u << 28)) __trap();
}
// 1-D bulk copy global -> shared (TMA engine), bytes a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
// arrive on b once every cp.async this thread issued so far has landed (counts as one expected arrival)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}

#endif  // __CUDACC__

}  // namespace stfem
