// f32x2.cuh — device primitives shared by the E-step kernels (sm_100a):
// packed FP32 pairs (fma/add/mul.rn.f32x2 -> FFMA2/FADD2/FMUL2), MUFU
// ex2/lg2/rcp, warp reduce-scatter, mbarriers and TMA bulk copies.
#pragma once
#include <cuda_runtime.h>

#ifndef GMMB_F2F_ALU
#define GMMB_F2F_ALU 0          // 1: FP32 -> FP64 widening on the integer ALU
#endif

namespace gmmb {
namespace dev {

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int P>
struct Log2 {
  static constexpr int v = P == 1 ? 0 : 1 + Log2<P / 2>::v;
};
template <>
struct Log2<1> {
  static constexpr int v = 0;
};

// Warp reduce-scatter over 32 lanes of P per-lane values (one per point).
// On return v[0] of lane l holds the reduction for point l >> (5 - log2 P)
// over all 32 lanes. Fixed butterfly order => deterministic.
template <int P, bool MAX>
__device__ __forceinline__ float warp_reduce_scatter(float (&v)[P], int lane) {
#pragma unroll
  for (int h = P / 2, off = 16; h >= 1; h >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const float send = up ? v[i] : v[i + h];
      const float keep = up ? v[i + h] : v[i];
      const float got = __shfl_xor_sync(0xffffffffu, send, off);
      v[i] = MAX ? fmaxf(keep, got) : keep + got;
    }
  }
#pragma unroll
  for (int off = 16 / P; off >= 1; off >>= 1) {
    const float got = __shfl_xor_sync(0xffffffffu, v[0], off);
    v[0] = MAX ? fmaxf(v[0], got) : v[0] + got;
  }
  return v[0];
}

__device__ __forceinline__ float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// f32x2 register pairs (lo = component tid, hi = component T + tid)
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo2(f2_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}
__device__ __forceinline__ float hi2(f2_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2n(float x) {  // 2^-x
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-x));
  return y;
}

// FP32 -> FP64 widening. The XU pipe (F2F) also carries the ex2 of every
// unit; GMMB_F2F_ALU = 1 widens on the integer ALU instead (exact for
// normal numbers; FP32 subnormals, ~1e-38, flush to zero).
__device__ __forceinline__ double f32_to_f64(float f) {
#if GMMB_F2F_ALU
  const unsigned b = __float_as_uint(f);
  const unsigned e = b & 0x7f800000u;
  const unsigned hi = e ? (((b >> 3) & 0x0fffffffu) + 0x38000000u) | (b & 0x80000000u) : 0u;
  const unsigned lo = e ? (b << 29) : 0u;
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
#else
  return static_cast<double>(f);
#endif
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

}  // namespace dev
}  // namespace gmmb
