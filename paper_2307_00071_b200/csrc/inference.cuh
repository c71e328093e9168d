// inference.cuh — score / dense E step / sampling / conditional intensity.
#pragma once
#include "common.cuh"

namespace gmmb {

// Per-component FP64 factors (16 doubles: P packed, mu, base) for a model
// with weights w[m], means mu[m][d], covariances cov[m][d(d+1)/2] (packed
// lower, row-major); lower (optional) = packed Cholesky factors [m][10].
// err[0] = first non-SPD component (atomicMin; initialise to INT_MAX).
cudaError_t launch_factors(int d, const double* w, const double* mu, const double* cov, int m,
                           double* fac, double* lower, int* err, cudaStream_t s);

int dense_blocks(int64_t n);
// lse[n] (optional), part[dense_blocks(n)] = per-CTA sums of lse,
// log_gamma (optional) = N x M column-major log-responsibilities.
cudaError_t launch_dense(int d, const double* x64, int64_t n, const double* fac, int m,
                         double* lse, double* part, double* log_gamma, cudaStream_t s);

// n draws, out = n x d column-major; cdf = scratch [m].
cudaError_t launch_sample(int d, const double* w, const double* fac, const double* lower, int m,
                          int64_t n, uint64_t seed, double* cdf, double* out, cudaStream_t s);

// 4D model; locs n x 3 column-major; cnd = scratch [m][20];
// err[0] = first non-SPD spatial block, err[1] = first query whose
// conditional variance is below -1e-12 (both INT_MAX when fine).
cudaError_t launch_conditional(const double* w, const double* mu, const double* cov, int m,
                               const double* locs, int64_t n, int clamp, double* cnd,
                               double* expct, double* var, int* err, cudaStream_t s);

}  // namespace gmmb
