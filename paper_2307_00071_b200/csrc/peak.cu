// peak.cu — FP32 FMA throughput microbenchmark: the roofline denominator
// of the CUDA-core-bound fused E step (MEASURED_PEAKS.json only carries HBM
// and bf16 tensor peaks). Packed fma.rn.f32x2 (FFMA2, the form the E step
// uses): 8 independent chains per thread, 16 warps per SM. Scalar FFMA with
// three distinct register sources tops out at ~47 TFLOP/s (register-bank
// reads), the two-register form at ~66; FFMA2 reaches the ~74 TFLOP/s
// nominal (148 SMs x 128 lanes x 2 x 1.965 GHz), scripts/micro/ffma2_bench.cu.
#include <cuda_runtime.h>

#include "../../include/gmmb.h"

namespace {
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t pk(float a, float b) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__global__ void __launch_bounds__(256) ffma_kernel(float* out, int iters, float s) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  f2_t x[8], a[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = pk(s * (t + j), s * (t - j));
    a[j] = pk(0.9999f - s * j, 0.9998f - s * j);
    b[j] = pk(1e-3f * s * (j + 1), 2e-3f * s * (j + 1));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        f2_t d;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a[j]), "l"(b[(j + u) & 7]), "l"(x[j]));
        x[j] = d;
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[j]));
    acc += lo + hi;
  }
  out[t] = acc;
}
}  // namespace

extern "C" int gmmb_ffma_peak_impl(int sm_count, void* stream, double ms_target,
                                   double* tflops, double* ms_out) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = sm_count * 2, threads = 256;
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
  const double flops = 2.0 * 2 * 8 * 8 * static_cast<double>(iters) * blocks * threads;
  *tflops = flops / (ms * 1e-3) / 1e12;
  *ms_out = ms;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const cudaError_t e = cudaGetLastError();
  cudaFree(out);
  return e == cudaSuccess ? 0 : 1;
}
