// mstep_hard.cuh — initial M step from hard labels (sort + segmented moments).
#pragma once
#include "em_kernels.cuh"

namespace gmmb {

struct HardScratch {
  int32_t* idx_in;    // [n]
  int32_t* idx_out;   // [n]  point indices sorted by label (stable)
  int32_t* keys_out;  // [n]  sorted labels
  void* temp;         // CUB radix-sort temp
  size_t temp_bytes;
};

size_t hard_moments_temp_bytes(int64_t n, int m);

// Records (count, mean, regularised covariance, factor, flags) of the
// per-label moments, for launch_commit(mode = 1). Single device.
cudaError_t launch_hard_moments(int d, const double* x64, int64_t n, const int32_t* labels,
                                int m, double cov_reg, HardScratch scr, RecBuf rec,
                                cudaStream_t s);

}  // namespace gmmb
