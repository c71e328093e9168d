// factor.cuh — small dense FP64 linear algebra for D = 3, 4 components
// (kernels.cpp:10-50): Cholesky, L^-1, and the E-step constants.
#pragma once
#include "common.cuh"

namespace gmmb {

// ---------------------------------------------------------------------------
// Small dense FP64 linear algebra (kernels.cpp:10-50), D = 3 or 4.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ bool cholesky_d(const double (&a)[D][D], double (&l)[D][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) l[i][j] = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double d = a[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(l[j][k], l[j][k]));
    if (!(d > 0.0) || !isfinite(d)) return false;
    const double ljj = sqrt(d);
    l[j][j] = ljj;
#pragma unroll
    for (int i = j + 1; i < D; ++i) {
      double s = a[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(l[i][k], l[j][k]));
      l[i][j] = s / ljj;
    }
  }
  return true;
}

template <int D>
__device__ __forceinline__ void lower_inverse_d(const double (&l)[D][D], double (&inv)[D][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) inv[i][j] = 0.0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double x[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) s = __dsub_rn(s, __dmul_rn(l[i][k], x[k]));
      x[i] = s / l[i][i];
    }
#pragma unroll
    for (int r = c; r < D; ++r) inv[r][c] = x[r];
  }
}

// Cholesky + precision factor + E constants for one covariance.
// Returns false if not SPD. This feeds only the FP32 E-step constants and the
// log-determinant, so it trades the exact divisions / square roots of
// cholesky_d / lower_inverse_d (kept for the factor and scoring APIs) for one
// reciprocal square root per pivot: l_jj = d r_j, columns scaled by r_j =
// 1 / l_jj, P = L^-1 by multiplications, and one log of the product of the
// r_j (each within 1-2 ulp of the exact forms; ~3x shorter dependent chain on
// the per-iteration critical path).
template <int D>
__device__ __forceinline__ bool factor_component(const double* cov_packed, float* pc,
                                                 double* logdet) {
  double a[D][D];
#pragma unroll
  for (int k = 0; k < npacked(D); ++k) {
    a[packed_row(k)][packed_col(k)] = cov_packed[k];
    a[packed_col(k)][packed_row(k)] = cov_packed[k];
  }
  double l[D][D], r[D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) l[i][j] = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double d = a[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= l[j][k] * l[j][k];
    if (!(d > 0.0) || !isfinite(d)) return false;
    r[j] = rsqrt(d);
    l[j][j] = d * r[j];
#pragma unroll
    for (int i = j + 1; i < D; ++i) {
      double s = a[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= l[i][k] * l[j][k];
      l[i][j] = s * r[j];
    }
  }
  double p[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) p[i][j] = 0.0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    p[c][c] = r[c];
#pragma unroll
    for (int i = c + 1; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int k = c; k < i; ++k) s -= l[i][k] * p[k][c];
      p[i][c] = s * r[i];
    }
  }
  double prod = 1.0, ld = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) prod *= r[j];
  if (prod > 1e-300 && prod < 1e300) {
    ld = log(prod);
  } else {
#pragma unroll
    for (int j = 0; j < D; ++j) ld += log(r[j]);
  }
  *logdet = ld;
  const double sc = sqrt(0.5 * kLog2E);
#pragma unroll
  for (int k = 0; k < npacked(D); ++k) {
    pc[k] = static_cast<float>(p[packed_row(k)][packed_col(k)] * sc);
  }
  return true;
}

}  // namespace gmmb
