// ingest.cu — depth/intensity image pair -> resident 4D cloud on the device
// (SURVEY.md §8(f) row 2): decimate (ingest.cpp:59-75) fused with
// image_pair_to_cloud (ingest.cpp:27-57). Only the two 16-bit images cross
// PCIe/NVLink-C2C (1.2 MB for 640x480 instead of the 9.8 MB FP64 cloud).
// Order and arithmetic follow the reference: row-major over the decimated
// image, zero depths dropped (a stable compaction: flag -> CUB exclusive
// scan -> scatter), z = d * (1 / scale), x = (u - cx) * z / fx,
// y = (v - cy) * z / fy, intensity = I * (1 / max) — so the device cloud
// is bit-identical to the host restatement.
#include <cub/device/device_scan.cuh>

#include "ingest.cuh"

namespace gmmb {

namespace {

__global__ void ingest_flags_kernel(const uint16_t* __restrict__ depth, int width, int wd, int hd,
                                    int f, int* __restrict__ flags) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= static_cast<int64_t>(wd) * hd) return;
  const int v = static_cast<int>(p / wd), u = static_cast<int>(p % wd);
  flags[p] = depth[static_cast<int64_t>(v) * f * width + static_cast<int64_t>(u) * f] > 0;
}

__global__ void ingest_scatter_kernel(const uint16_t* __restrict__ depth,
                                      const uint16_t* __restrict__ inten, int width, int wd,
                                      int hd, int f, const int* __restrict__ flags,
                                      const int* __restrict__ offs, IngestParams ip,
                                      double* __restrict__ x64, int64_t* __restrict__ n_out) {
  const int64_t np = static_cast<int64_t>(wd) * hd;
  const int64_t n = static_cast<int64_t>(offs[np - 1]) + flags[np - 1];
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p == 0) *n_out = n;
  if (p >= np || !flags[p]) return;
  const int v = static_cast<int>(p / wd), u = static_cast<int>(p % wd);
  const int64_t src = static_cast<int64_t>(v) * f * width + static_cast<int64_t>(u) * f;
  const int64_t k = offs[p];
  const double z = __dmul_rn(static_cast<double>(depth[src]), ip.inv_scale);
  x64[k] = __ddiv_rn(__dmul_rn(__dsub_rn(static_cast<double>(u), ip.cx), z), ip.fx);
  x64[n + k] = __ddiv_rn(__dmul_rn(__dsub_rn(static_cast<double>(v), ip.cy), z), ip.fy);
  x64[2 * n + k] = z;
  x64[3 * n + k] = __dmul_rn(static_cast<double>(inten[src]), ip.inv_max);
}

}  // namespace

size_t ingest_temp_bytes(int64_t np) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const int*)nullptr, (int*)nullptr,
                                static_cast<int>(np));
  return bytes;
}

cudaError_t launch_ingest(const uint16_t* depth, const uint16_t* inten, int width, int wd, int hd,
                          int f, IngestParams ip, IngestScratch scr, double* x64,
                          int64_t* n_dev, cudaStream_t s) {
  const int64_t np = static_cast<int64_t>(wd) * hd;
  const int grid = static_cast<int>((np + 255) / 256);
  ingest_flags_kernel<<<grid, 256, 0, s>>>(depth, width, wd, hd, f, scr.flags);
  size_t bytes = scr.temp_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(scr.temp, bytes, scr.flags, scr.offs,
                                                static_cast<int>(np), s);
  if (e != cudaSuccess) return e;
  ingest_scatter_kernel<<<grid, 256, 0, s>>>(depth, inten, width, wd, hd, f, scr.flags, scr.offs,
                                             ip, x64, n_dev);
  return cudaGetLastError();
}

}  // namespace gmmb
