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
// Returns false if not SPD.
template <int D>
__device__ __forceinline__ bool factor_component(const double* cov_packed, float* pc,
                                 double* logdet) {
  double a[D][D];
#pragma unroll
  for (int k = 0; k < npacked(D); ++k) {
    a[packed_row(k)][packed_col(k)] = cov_packed[k];
    a[packed_col(k)][packed_row(k)] = cov_packed[k];
  }
  double l[D][D], p[D][D];
  if (!cholesky_d<D>(a, l)) return false;
  lower_inverse_d<D>(l, p);
  double ld = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) ld += log(p[j][j]);
  *logdet = ld;
  const double sc = sqrt(0.5 * kLog2E);
#pragma unroll
  for (int k = 0; k < npacked(D); ++k) {
    pc[k] = static_cast<float>(p[packed_row(k)][packed_col(k)] * sc);
  }
  return true;
}

}  // namespace gmmb
