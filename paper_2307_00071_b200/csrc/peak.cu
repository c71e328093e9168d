// peak.cu — FP32 FFMA throughput microbenchmark: the roofline denominator
// of the CUDA-core-bound fused E step (MEASURED_PEAKS.json only carries HBM
// and bf16 tensor peaks). Register-operand FFMA (the form the E step uses),
// 8 independent chains per thread, 32 warps per SM.
#include <cuda_runtime.h>

#include "../../include/gmmb.h"

namespace {
__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float s) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  float x[8], y[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = s * (t + j);
    y[j] = 0.9999f - s * j;
  }
  const float z = s * 0.5f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], y[j], z);
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += x[j];
  out[t] = acc;
}
}  // namespace

extern "C" int gmmb_ffma_peak_impl(int sm_count, void* stream, double ms_target,
                                   double* tflops, double* ms_out) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = sm_count * 8, threads = 256;
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * blocks * threads) != cudaSuccess) return 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 256;
  float ms = 0.f;
  for (int pass = 0; pass < 4; ++pass) {
    cudaEventRecord(a, s);
    ffma_kernel<<<blocks, threads, 0, s>>>(out, iters, 1e-7f);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass < 3 && ms > 0.f) {
      const double scale = ms_target / ms;
      iters = static_cast<int>(iters * (scale > 64 ? 64 : scale)) + 1;
    }
  }
  const double flops = 2.0 * 16 * 8 * static_cast<double>(iters) * blocks * threads;
  *tflops = flops / (ms * 1e-3) / 1e12;
  *ms_out = ms;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const cudaError_t e = cudaGetLastError();
  cudaFree(out);
  return e == cudaSuccess ? 0 : 1;
}
