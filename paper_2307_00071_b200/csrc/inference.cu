// inference.cu — model evaluation kernels beyond the fit:
//   score               inference.cpp:141-172 (average log-likelihood)
//   e_step (API)        sogmm.cpp:341-395 (dense log-responsibilities)
//   joint_dist_sample   inference.cpp:17-54
//   color_conditional   inference.cpp:56-139
// All FP64 (the API results are reported numbers, not an inner loop): per
// component factors are computed once per call (FP64 Cholesky / L^-1, the
// reference's cholesky_cache) and streamed through shared memory in chunks;
// one thread per point / sample / query.
#include <cmath>

#include "factor.cuh"
#include "inference.cuh"

namespace gmmb {

namespace {

constexpr int kChunk = 128;  // components per shared-memory chunk
constexpr int kFac = 16;     // doubles per component: P packed [0..9], mu [10..13], base [14]

// factors: P = L^-1 (packed lower, FP64), mu, base = ln w + sum ln P_jj - D/2 ln 2 pi;
// lower (packed) for sampling; err = first non-SPD component (atomicMin)
template <int D>
__global__ void factors_kernel(const double* __restrict__ w, const double* __restrict__ mu,
                               const double* __restrict__ cov, int m, double* __restrict__ fac,
                               double* __restrict__ lower, int* __restrict__ err) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double a[D][D];
#pragma unroll
  for (int q = 0; q < npacked(D); ++q) {
    a[packed_row(q)][packed_col(q)] = cov[k * npacked(D) + q];
    a[packed_col(q)][packed_row(q)] = cov[k * npacked(D) + q];
  }
  double l[D][D], p[D][D];
  double* f = fac + static_cast<int64_t>(k) * kFac;
  if (!cholesky_d<D>(a, l)) {
    atomicMin(err, k);
    for (int q = 0; q < kFac; ++q) f[q] = 0.0;
    return;
  }
  lower_inverse_d<D>(l, p);
  double ld = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) ld += log(p[j][j]);
#pragma unroll
  for (int q = 0; q < 10; ++q) f[q] = q < npacked(D) ? p[packed_row(q)][packed_col(q)] : 0.0;
#pragma unroll
  for (int j = 0; j < 4; ++j) f[10 + j] = j < D ? mu[k * D + j] : 0.0;
  f[14] = log(w[k]) + ld - 0.5 * D * kLog2Pi;
  f[15] = 0.0;
  if (lower) {
#pragma unroll
    for (int q = 0; q < 10; ++q)
      lower[static_cast<int64_t>(k) * 10 + q] = q < npacked(D) ? l[packed_row(q)][packed_col(q)] : 0.0;
  }
}

// log density of point x under the component at f (sogmm.cpp:351-364 tree)
template <int D>
__device__ __forceinline__ double log_dens(const double* f, const double (&x)[D]) {
  double d[D];
#pragma unroll
  for (int j = 0; j < D; ++j) d[j] = x[j] - f[10 + j];
  double q = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double y = f[i * (i + 1) / 2] * d[0];
#pragma unroll
    for (int j = 1; j <= i; ++j) y = y + f[i * (i + 1) / 2 + j] * d[j];
    q = q + y * y;
  }
  return f[14] - 0.5 * q;
}

// Per point: lse over all components (online max / rescaled sum), per-CTA
// partial of sum lse (fixed tree), optional dense log-responsibilities
// log_gamma[k * n + i] = l - lse (N x M column-major, the reference layout).
template <int D>
__global__ void __launch_bounds__(256) dense_kernel(const double* __restrict__ x64, int64_t n,
                                                    const double* __restrict__ fac, int m,
                                                    double* __restrict__ lse_out,
                                                    double* __restrict__ part,
                                                    double* __restrict__ log_gamma) {
  __shared__ double sf[kChunk * kFac];
  __shared__ double red[256];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool v = i < n;
  double x[D];
#pragma unroll
  for (int j = 0; j < D; ++j) x[j] = v ? x64[j * n + i] : 0.0;
  double mx = -INFINITY, acc = 0.0;
  for (int c0 = 0; c0 < m; c0 += kChunk) {
    const int len = min(kChunk, m - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < len * kFac; t += blockDim.x) sf[t] = fac[c0 * kFac + t];
    __syncthreads();
    if (v) {
      for (int c = 0; c < len; ++c) {
        const double l = log_dens<D>(sf + c * kFac, x);
        if (l > mx) {
          acc = acc * exp(mx - l) + 1.0;  // (exp(-inf) = 0 on the first)
          mx = l;
        } else {
          acc += exp(fmax(l - mx, -700.0));  // kernels.cpp:123-127
        }
      }
    }
  }
  const double lse = (mx == -INFINITY) ? -INFINITY : mx + log(acc);
  if (v && lse_out) lse_out[i] = lse;
  red[threadIdx.x] = v ? lse : 0.0;
  __syncthreads();
  for (int off = 128; off >= 1; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
  if (!log_gamma) return;
  for (int c0 = 0; c0 < m; c0 += kChunk) {
    const int len = min(kChunk, m - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < len * kFac; t += blockDim.x) sf[t] = fac[c0 * kFac + t];
    __syncthreads();
    if (v) {
      for (int c = 0; c < len; ++c)
        log_gamma[static_cast<int64_t>(c0 + c) * n + i] = log_dens<D>(sf + c * kFac, x) - lse;
    }
  }
}

// running sum of the weights in order, last entry pinned to 1
// (inference.cpp:22-28)
__global__ void cdf_kernel(const double* __restrict__ w, int m, double* __restrict__ cdf) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (int b = 0; b < m; ++b) {
    acc += w[b];
    cdf[b] = acc;
  }
  cdf[m - 1] = 1.0;
}

__device__ __forceinline__ void normal_pair(uint64_t seed, uint64_t stream, uint64_t counter,
                                            double& z0, double& z1) {  // rng.hpp:45-53
  const double u1 = static_cast<double>((rng_bits(seed, stream, counter) >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(rng_bits(seed, stream, counter + 1) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.14159265358979323846 * u2;
  z0 = r * cos(a);
  z1 = r * sin(a);
}

template <int D>
__global__ void sample_kernel(const double* __restrict__ cdf, const double* __restrict__ fac,
                              const double* __restrict__ lower, int m, int64_t n,
                              uint64_t seed, double* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // component: first b < m - 1 with u < cdf[b], else m - 1 (the linear scan
  // of inference.cpp:39-40 on a non-decreasing prefix)
  const double u = static_cast<double>(rng_bits(seed, 0, static_cast<uint64_t>(i)) >> 11) * 0x1.0p-53;
  int lo = 0, hi = m - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (u >= cdf[mid]) lo = mid + 1;
    else hi = mid;
  }
  const int b = lo;
  double z[4];
  normal_pair(seed, 1, static_cast<uint64_t>(i) * 4, z[0], z[1]);
  normal_pair(seed, 1, static_cast<uint64_t>(i) * 4 + 2, z[2], z[3]);
  const double* L = lower + static_cast<int64_t>(b) * 10;
  const double* f = fac + static_cast<int64_t>(b) * kFac;
#pragma unroll
  for (int r = 0; r < D; ++r) {
    double v = __dmul_rn(L[r * (r + 1) / 2], z[0]);
#pragma unroll
    for (int j = 1; j <= r; ++j) v = __dadd_rn(v, __dmul_rn(L[r * (r + 1) / 2 + j], z[j]));
    out[r * n + i] = __dadd_rn(f[10 + r], v);
  }
}

// color_conditional per-component terms (inference.cpp:64-88), 20 doubles:
// xx_inv (9, column-major), mu_x (3), mu_i, regression (3), cond_var, gate_base
constexpr int kCnd = 20;

__device__ bool cholesky3(const double (&a)[3][3], double (&l)[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) l[i][j] = 0.0;
  for (int j = 0; j < 3; ++j) {
    double d = a[j][j];
    for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(l[j][k], l[j][k]));
    if (!(d > 0.0) || !isfinite(d)) return false;
    const double ljj = sqrt(d);
    l[j][j] = ljj;
    for (int i = j + 1; i < 3; ++i) {
      double s = a[i][j];
      for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(l[i][k], l[j][k]));
      l[i][j] = s / ljj;
    }
  }
  return true;
}
__device__ void llt_solve3(const double (&l)[3][3], const double (&b)[3], double (&x)[3]) {
  double y[3];
  for (int i = 0; i < 3; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s = __dsub_rn(s, __dmul_rn(l[i][k], y[k]));
    y[i] = s / l[i][i];
  }
  for (int i = 2; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < 3; ++k) s = __dsub_rn(s, __dmul_rn(l[k][i], x[k]));
    x[i] = s / l[i][i];
  }
}

__global__ void conditional_prep_kernel(const double* __restrict__ w,
                                        const double* __restrict__ mu,
                                        const double* __restrict__ cov, int m,
                                        double* __restrict__ cnd, int* __restrict__ err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= m) return;
  double c4[4][4];
  for (int q = 0; q < 10; ++q) {
    c4[packed_row(q)][packed_col(q)] = cov[b * 10 + q];
    c4[packed_col(q)][packed_row(q)] = cov[b * 10 + q];
  }
  double sxx[3][3], sxi[3], l[3][3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) sxx[i][j] = c4[i][j];
    sxi[i] = c4[i][3];
  }
  double* o = cnd + static_cast<int64_t>(b) * kCnd;
  if (!cholesky3(sxx, l)) {
    atomicMin(err, b);
    for (int q = 0; q < kCnd; ++q) o[q] = 0.0;
    return;
  }
  for (int col = 0; col < 3; ++col) {
    double e[3] = {0.0, 0.0, 0.0}, x[3];
    e[col] = 1.0;
    llt_solve3(l, e, x);
    for (int i = 0; i < 3; ++i) o[col * 3 + i] = x[i];
  }
  double reg[3];
  llt_solve3(l, sxi, reg);
  for (int i = 0; i < 3; ++i) {
    o[9 + i] = mu[b * 4 + i];
    o[13 + i] = reg[i];
  }
  o[12] = mu[b * 4 + 3];
  o[16] = c4[3][3] - (sxi[0] * reg[0] + sxi[1] * reg[1] + sxi[2] * reg[2]);
  const double log_det = 2.0 * ((log(l[0][0]) + log(l[1][1])) + log(l[2][2]));
  o[17] = log(w[b]) - 0.5 * (3.0 * kLog2Pi + log_det);
  o[18] = o[19] = 0.0;
}

__global__ void __launch_bounds__(256) conditional_kernel(const double* __restrict__ locs,
                                                          int64_t n,
                                                          const double* __restrict__ cnd, int m,
                                                          int clamp, double* __restrict__ expct,
                                                          double* __restrict__ var,
                                                          int* __restrict__ err) {
  __shared__ double sc[kChunk * kCnd];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool v = i < n;
  double x[3];
  for (int j = 0; j < 3; ++j) x[j] = v ? locs[j * n + i] : 0.0;
  // online gated sums; fallback: nearest component by Mahalanobis distance
  double mx = -INFINITY, norm = 0.0, e = 0.0, second = 0.0;
  double best_q = INFINITY, best_cm = 0.0, best_cv = 0.0;
  for (int c0 = 0; c0 < m; c0 += kChunk) {
    const int len = min(kChunk, m - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < len * kCnd; t += blockDim.x) sc[t] = cnd[c0 * kCnd + t];
    __syncthreads();
    if (!v) continue;
    for (int c = 0; c < len; ++c) {
      const double* o = sc + c * kCnd;
      const double d[3] = {x[0] - o[9], x[1] - o[10], x[2] - o[11]};
      double q = 0.0;
      for (int r = 0; r < 3; ++r) {
        const double ad = o[0 * 3 + r] * d[0] + o[1 * 3 + r] * d[1] + o[2 * 3 + r] * d[2];
        q += d[r] * ad;
      }
      const double lg = o[17] - 0.5 * q;
      const double cm = o[12] + (o[13] * d[0] + o[14] * d[1] + o[15] * d[2]);
      const double cv = o[16];
      if (q < best_q) {
        best_q = q;
        best_cm = cm;
        best_cv = cv;
      }
      if (lg > mx) {
        const double s = exp(mx - lg);
        norm = norm * s + 1.0;
        e = e * s + cm;
        second = second * s + (cv + cm * cm);
        mx = lg;
      } else {
        const double w = exp(lg - mx);
        norm += w;
        e += w * cm;
        second += w * (cv + cm * cm);
      }
    }
  }
  if (!v) return;
  if (mx == -INFINITY || !isfinite(mx)) {  // every gate underflowed
    e = best_cm;
    second = best_cv + e * e;
  } else {
    e /= norm;
    second /= norm;
  }
  double vv = second - e * e;
  if (vv < -1e-12) atomicMin(err, static_cast<int>(min64(i, 0x7ffffffe)));
  if (vv < 0.0) vv = 0.0;
  var[i] = vv;
  expct[i] = clamp ? fmin(fmax(e, 0.0), 1.0) : e;
}

}  // namespace

cudaError_t launch_factors(int d, const double* w, const double* mu, const double* cov, int m,
                           double* fac, double* lower, int* err, cudaStream_t s) {
  const int grid = (m + 127) / 128;
  if (d == 4)
    factors_kernel<4><<<grid, 128, 0, s>>>(w, mu, cov, m, fac, lower, err);
  else
    factors_kernel<3><<<grid, 128, 0, s>>>(w, mu, cov, m, fac, lower, err);
  return cudaGetLastError();
}

int dense_blocks(int64_t n) { return static_cast<int>((n + 255) / 256); }

cudaError_t launch_dense(int d, const double* x64, int64_t n, const double* fac, int m,
                         double* lse, double* part, double* log_gamma, cudaStream_t s) {
  const int grid = dense_blocks(n);
  if (d == 4)
    dense_kernel<4><<<grid, 256, 0, s>>>(x64, n, fac, m, lse, part, log_gamma);
  else
    dense_kernel<3><<<grid, 256, 0, s>>>(x64, n, fac, m, lse, part, log_gamma);
  return cudaGetLastError();
}

cudaError_t launch_sample(int d, const double* w, const double* fac, const double* lower, int m,
                          int64_t n, uint64_t seed, double* cdf, double* out, cudaStream_t s) {
  cdf_kernel<<<1, 32, 0, s>>>(w, m, cdf);
  const int grid = static_cast<int>((n + 255) / 256);
  if (d == 4)
    sample_kernel<4><<<grid, 256, 0, s>>>(cdf, fac, lower, m, n, seed, out);
  else
    sample_kernel<3><<<grid, 256, 0, s>>>(cdf, fac, lower, m, n, seed, out);
  return cudaGetLastError();
}

cudaError_t launch_conditional(const double* w, const double* mu, const double* cov, int m,
                               const double* locs, int64_t n, int clamp, double* cnd,
                               double* expct, double* var, int* err, cudaStream_t s) {
  conditional_prep_kernel<<<(m + 127) / 128, 128, 0, s>>>(w, mu, cov, m, cnd, err);
  conditional_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(locs, n, cnd, m, clamp,
                                                                      expct, var, err + 1);
  return cudaGetLastError();
}

}  // namespace gmmb
