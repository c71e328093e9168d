// FP64 add latency / throughput on this GPU (dependent chain vs independent
// chains), to size the FP64 work on kinit's critical path.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dadd_kernel(double* out, double a, double b, int iters, long long* cyc) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = a + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __dadd_rn(x[c], b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CHAINS>
void run(int warps, int blocks) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * blocks * warps * 32);
  cudaMalloc(&cyc, sizeof(long long));
  const int iters = 4096;
  dadd_kernel<CHAINS><<<blocks, warps * 32>>>(out, 1.0, 1e-9, iters, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dadd_kernel<CHAINS><<<blocks, warps * 32>>>(out, 1.0, 1e-9, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double ops = double(iters) * CHAINS * warps * 32 * blocks;
  printf("chains %d warps/CTA %2d CTAs %3d: %.2f cycles per dependent add (warp 0), %.2f TFLOP/s DADD\n",
         CHAINS, warps, blocks, double(c) / (iters), ops / (ms * 1e-3) / 1e12);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<1>(1, 1);
  run<1>(4, 1);
  run<8>(4, 1);
  run<8>(12, 148);
  run<8>(32, 148);
  return 0;
}
