// layout.cuh — validation + Morton-sorted, tile-recentred FP32 point copy.
#pragma once
#include "common.cuh"

namespace gmmb {

constexpr int kBboxParts = 1024;

struct LayoutScratch {
  double* bbox_part;   // [kBboxParts][6]
  uint64_t* keys_in;   // [n]
  uint64_t* keys_out;  // [n]
  int32_t* idx_in;     // [n]
  void* temp;          // CUB radix-sort temp
  size_t temp_bytes;
};

// flags |= 1 non-finite, |= 2 intensity outside [0, 1] (point_cloud.hpp:15-24)
cudaError_t launch_validate(const double* x64, int64_t n, int d, int* flags,
                            cudaStream_t s);
size_t layout_sort_temp_bytes(int64_t n);
cudaError_t launch_layout(const double* x64, int64_t n, LayoutScratch scr,
                          float4* xt, double* tc, int32_t* perm, int sm_count,
                          cudaStream_t s);

}  // namespace gmmb
