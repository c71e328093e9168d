// mstep_hard.cu — the initial M step from hard k-means++ labels.
//
// Reference: m_step on the one-hot responsibilities kinit returns
// (sogmm.cpp:481 -> m_step_impl :399-455 -> weighted_moments_fn
// kernels.hpp:82-181 with weights exp(0) = 1 / exp(-inf) = 0). With 0/1
// weights the weighted moments are plain per-label moments, so instead of
// testing every (point, component) pair the points are stably sorted by
// label (CUB radix sort on the label bits) and one warp per component
// reduces its contiguous segment in a fixed order: pass 1 sum x -> mean,
// pass 2 sum (x - mean)(x - mean)^T in packed order, then the usual record
// (count, mean, scatter / count + cov_reg I, FP64 Cholesky). Deterministic;
// O(N log K) instead of O(N K).
#include <cub/device/device_radix_sort.cuh>

#include "em_kernels.cuh"
#include "factor.cuh"
#include "mstep_hard.cuh"

namespace gmmb {

namespace {

__global__ void iota_kernel(int32_t* __restrict__ idx, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) idx[i] = static_cast<int32_t>(i);
}

// first position with key >= v in sorted keys[0, n)
__device__ __forceinline__ int64_t lower_bound(const int32_t* keys, int64_t n, int v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Block-wide FP64 sum of NV values per thread (fixed tree: deterministic).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*red)[NV]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) red[warp][q] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[w][q];
    v[q] = s;
  }
  __syncthreads();
}

// One CTA per component (the segment of its points in label-sorted order):
// large clusters (the back wall of cfg2 holds tens of thousands of points)
// spread over 256 threads with independent loads in flight.
constexpr int kHardThreads = 256;
template <int D>
__global__ void __launch_bounds__(kHardThreads) hard_moments_kernel(
    const double* __restrict__ x64, int64_t n, const int32_t* __restrict__ skeys,
    const int32_t* __restrict__ sidx, int m, double cov_reg, RecBuf rec) {
  constexpr int NP = npacked(D);
  __shared__ double red1[kHardThreads / 32][D];
  __shared__ double red2[kHardThreads / 32][NP];
  const int k = blockIdx.x;
  if (k >= m) return;
  const int64_t b = lower_bound(skeys, n, k), e = lower_bound(skeys, n, k + 1);
  const double cnt = static_cast<double>(e - b);
  // pass 1: sum x (kernels.hpp:91-119)
  double sx[D];
#pragma unroll
  for (int j = 0; j < D; ++j) sx[j] = 0.0;
#pragma unroll 4
  for (int64_t i = b + threadIdx.x; i < e; i += kHardThreads) {
    const int64_t p = sidx[i];
#pragma unroll
    for (int j = 0; j < D; ++j) sx[j] += x64[j * n + p];
  }
  block_sum<D>(sx, red1);
  const bool keep = !(cnt < kDegenerateCount);  // kernels.hpp:121-128
  double mean[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < D; ++j) mean[j] = keep ? sx[j] / cnt : 0.0;
  // pass 2: centred second moments in packed order (kernels.hpp:131-179)
  double sc[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) sc[q] = 0.0;
#pragma unroll 4
  for (int64_t i = b + threadIdx.x; i < e; i += kHardThreads) {
    const int64_t p = sidx[i];
    double d[D];
#pragma unroll
    for (int j = 0; j < D; ++j) d[j] = x64[j * n + p] - mean[j];
#pragma unroll
    for (int q = 0; q < NP; ++q) sc[q] += d[packed_row(q)] * d[packed_col(q)];
  }
  block_sum<NP>(sc, red2);
  if (threadIdx.x != 0) return;
  const double inv = keep ? 1.0 / cnt : 0.0;
  double cov[10];
#pragma unroll
  for (int q = 0; q < 10; ++q) cov[q] = 0.0;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    cov[q] = sc[q] * inv;
    if (packed_row(q) == packed_col(q)) cov[q] += cov_reg;
  }
  float pc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) pc[j] = 0.f;
  double logdet = 0.0;
  int flags = keep ? 1 : 0;
  if (keep && factor_component<D>(cov, pc, &logdet)) flags |= 2;
  rec.count[k] = cnt;
#pragma unroll
  for (int j = 0; j < 4; ++j) rec.mean[k * 4 + j] = mean[j];
#pragma unroll
  for (int j = 0; j < 10; ++j) rec.cov[k * 10 + j] = cov[j];
  rec.logdet[k] = logdet;
#pragma unroll
  for (int j = 0; j < 16; ++j) rec.pc[k * 16 + j] = pc[j];
  rec.flags[k] = flags;
}

int label_bits(int m) {
  int b = 1;
  while ((1 << b) < m) ++b;
  return b;
}

}  // namespace

size_t hard_moments_temp_bytes(int64_t n, int m) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr,
                                  static_cast<int>(n), 0, label_bits(m));
  return bytes;
}

cudaError_t launch_hard_moments(int d, const double* x64, int64_t n, const int32_t* labels,
                                int m, double cov_reg, HardScratch scr, RecBuf rec,
                                cudaStream_t s) {
  iota_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(scr.idx_in, n);
  size_t bytes = scr.temp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(scr.temp, bytes, labels, scr.keys_out,
                                                  scr.idx_in, scr.idx_out, static_cast<int>(n),
                                                  0, label_bits(m), s);
  if (e != cudaSuccess) return e;
  if (d == 4)
    hard_moments_kernel<4><<<m, kHardThreads, 0, s>>>(x64, n, scr.keys_out, scr.idx_out, m,
                                                      cov_reg, rec);
  else
    hard_moments_kernel<3><<<m, kHardThreads, 0, s>>>(x64, n, scr.keys_out, scr.idx_out, m,
                                                      cov_reg, rec);
  return cudaGetLastError();
}

}  // namespace gmmb
