// layout.cu — input validation and the E/M data layout.
//
// Points arrive as the reference's N x D column-major FP64 matrix
// (common.hpp:11) and stay resident in that form for kinit, which must be
// bit-exact in FP64. The EM pass streams a second copy: points Morton-sorted
// on xyz (E/M sums are order-independent up to rounding) and stored as FP32
// float4 offsets from the FP64 centroid of their 128-point tile. Within a
// compact tile, fp32(x - c_t) - fp32(mu - c_t) reproduces the exact FP64
// difference x - mu to ~1e-7 relative of the tile extent, which is what the
// 1e-4 parameter tolerance needs.
#include <cub/device/device_radix_sort.cuh>

#include "layout.cuh"

namespace gmmb {

namespace {

__global__ void validate_kernel(const double* __restrict__ x64, int64_t n,
                                int d, int* __restrict__ flags) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int f = 0;
  for (int j = 0; j < 4; ++j) {
    const double v = x64[j * n + i];
    if (!isfinite(v)) f |= 1;
  }
  if (d == 4) {
    const double w = x64[3 * n + i];
    if (w < 0.0 || w > 1.0) f |= 2;  // point_cloud.hpp:20-23
  }
  if (f) atomicOr(flags, f);
}

__global__ void bbox_kernel(const double* __restrict__ x64, int64_t n,
                            double* __restrict__ part) {
  __shared__ double lo[3][256], hi[3][256];
  const int tid = threadIdx.x;
  double l[3] = {INFINITY, INFINITY, INFINITY};
  double h[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + tid; i < n;
       i += static_cast<int64_t>(gridDim.x) * 256) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double v = x64[j * n + i];
      l[j] = fmin(l[j], v);
      h[j] = fmax(h[j], v);
    }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    lo[j][tid] = l[j];
    hi[j][tid] = h[j];
  }
  __syncthreads();
  for (int off = 128; off >= 1; off >>= 1) {
    if (tid < off) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        lo[j][tid] = fmin(lo[j][tid], lo[j][tid + off]);
        hi[j][tid] = fmax(hi[j][tid], hi[j][tid + off]);
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      part[blockIdx.x * 6 + j] = lo[j][0];
      part[blockIdx.x * 6 + 3 + j] = hi[j][0];
    }
  }
}

// The tiles only need spatial compactness: sorting on the top 30 Morton bits
// (10 per axis, cells of 1/1024 of the bounding box; the radix sort runs 4
// passes instead of 8) keeps 128-point tiles within a few cells.
constexpr int kMortonLoBit = 33;

__device__ __forceinline__ uint64_t spread3(uint64_t v) {  // 21 bits -> 63
  v &= 0x1fffffULL;
  v = (v | (v << 32)) & 0x1f00000000ffffULL;
  v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
  v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
  v = (v | (v << 2)) & 0x1249249249249249ULL;
  return v;
}

__global__ void morton_kernel(const double* __restrict__ x64, int64_t n,
                              const double* __restrict__ part, int nparts,
                              uint32_t* __restrict__ keys,
                              int32_t* __restrict__ idx) {
  // the bounding box from the per-CTA partials: all threads, then a fixed
  // tree (min / max are order-independent anyway)
  __shared__ double red[6][256];
  __shared__ double bb[6];
  {
    double v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
#pragma unroll
      for (int j = 0; j < 6; ++j)
        v[j] = j < 3 ? fmin(v[j], part[p * 6 + j]) : fmax(v[j], part[p * 6 + j]);
    }
#pragma unroll
    for (int j = 0; j < 6; ++j) red[j][threadIdx.x] = v[j];
    __syncthreads();
    for (int off = blockDim.x / 2; off >= 1; off >>= 1) {
      if (threadIdx.x < off) {
#pragma unroll
        for (int j = 0; j < 6; ++j)
          red[j][threadIdx.x] = j < 3 ? fmin(red[j][threadIdx.x], red[j][threadIdx.x + off])
                                      : fmax(red[j][threadIdx.x], red[j][threadIdx.x + off]);
      }
      __syncthreads();
    }
    if (threadIdx.x < 6) bb[threadIdx.x] = red[threadIdx.x][0];
    __syncthreads();
  }
  double lo[3], ex[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    lo[j] = bb[j];
    ex[j] = bb[3 + j] - bb[j];
  }
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t key = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double t = ex[j] > 0.0 ? (x64[j * n + i] - lo[j]) / ex[j] : 0.0;
      t = fmin(fmax(t, 0.0), 1.0);
      const uint64_t q = static_cast<uint64_t>(t * 2097151.0);
      key |= spread3(q) << j;
    }
    keys[i] = static_cast<uint32_t>(key >> kMortonLoBit);  // the top 30 bits (4 radix passes)
    idx[i] = static_cast<int32_t>(i);
  }
}

// One CTA per 128-point tile: FP64 centroid, then FP32 offsets.
__global__ void __launch_bounds__(kTile)
    tile_kernel(const double* __restrict__ x64, int64_t n,
                const int32_t* __restrict__ perm, float4* __restrict__ xt,
                double* __restrict__ tc) {
  __shared__ double red[4][kTile];
  const int t = blockIdx.x, tid = threadIdx.x;
  const int64_t i = static_cast<int64_t>(t) * kTile + tid;
  const bool v = i < n;
  double x[4] = {0, 0, 0, 0};
  if (v) {
    const int64_t src = perm[i];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = x64[j * n + src];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) red[j][tid] = x[j];
  __syncthreads();
  for (int off = kTile / 2; off >= 1; off >>= 1) {
    if (tid < off) {
#pragma unroll
      for (int j = 0; j < 4; ++j) red[j][tid] += red[j][tid + off];
    }
    __syncthreads();
  }
  const int cnt = static_cast<int>(min64(kTile, n - static_cast<int64_t>(t) * kTile));
  double c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = red[j][0] / cnt;
  if (tid < 4) tc[static_cast<int64_t>(t) * 4 + tid] = c[tid];
  // padding points of the last tile are zero (the E kernel copies whole tiles)
  xt[i] = v ? make_float4(static_cast<float>(x[0] - c[0]), static_cast<float>(x[1] - c[1]),
                          static_cast<float>(x[2] - c[2]), static_cast<float>(x[3] - c[3]))
            : make_float4(0.f, 0.f, 0.f, 0.f);
}

}  // namespace

cudaError_t launch_validate(const double* x64, int64_t n, int d, int* flags,
                            cudaStream_t s) {
  const int grid = static_cast<int>((n + 255) / 256);
  validate_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(x64, n, d, flags);
  return cudaGetLastError();
}

size_t layout_sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, static_cast<int>(n), 0, 63 - kMortonLoBit);
  return bytes;
}

cudaError_t launch_layout(const double* x64, int64_t n, LayoutScratch scr,
                          float4* xt, double* tc, int32_t* perm, int sm_count,
                          cudaStream_t s) {
  int nparts = sm_count * 2;
  if (nparts > kBboxParts) nparts = kBboxParts;
  bbox_kernel<<<nparts, 256, 0, s>>>(x64, n, scr.bbox_part);
  const int64_t need = (n + 255) / 256;
  const int grid = static_cast<int>(need < sm_count * 4 ? need : sm_count * 4);
  uint32_t* kin = reinterpret_cast<uint32_t*>(scr.keys_in);
  uint32_t* kout = reinterpret_cast<uint32_t*>(scr.keys_out);
  morton_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(x64, n, scr.bbox_part, nparts, kin,
                                                   scr.idx_in);
  size_t bytes = scr.temp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(
      scr.temp, bytes, kin, kout, scr.idx_in, perm, static_cast<int>(n), 0, 63 - kMortonLoBit, s);
  if (e != cudaSuccess) return e;
  const int ntiles = static_cast<int>((n + kTile - 1) / kTile);
  tile_kernel<<<ntiles, kTile, 0, s>>>(x64, n, perm, xt, tc);
  return cudaGetLastError();
}

}  // namespace gmmb
