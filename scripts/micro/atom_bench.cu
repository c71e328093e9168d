// Global 64-bit atomic throughput on B200 (sm_100a): N threads each add to
// addresses among A (K x stats x limbs), with return (atom) or without (red).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 atom_bench.cu -o atom_bench
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atom(unsigned long long* a, int nadr, int iters, int ret, unsigned long long* sink) {
  unsigned long long s = 0;
  unsigned x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const int idx = (x >> 8) % nadr;
    if (ret) s += atomicAdd(a + idx, 1ull);
    else atomicAdd(a + idx, 1ull);
  }
  if (ret && s == 12345) sink[0] = s;
}
int main() {
  unsigned long long *a, *sink;
  cudaMalloc(&a, sizeof(unsigned long long) * (1 << 24));
  cudaMalloc(&sink, 8);
  cudaMemset(a, 0, sizeof(unsigned long long) * (1 << 24));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nadrs[] = {64, 1024, 15360, 61440, 1 << 20};
  for (int ret = 0; ret < 2; ++ret)
    for (int na : nadrs) {
      const int blocks = 148 * 8, threads = 256, iters = 64;
      k_atom<<<blocks, threads>>>(a, na, iters, ret, sink);
      cudaEventRecord(e0);
      k_atom<<<blocks, threads>>>(a, na, iters, ret, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = double(blocks) * threads * iters;
      printf("%s addresses %8d: %.1f G atomics/s (%.3f ms)\n", ret ? "atom" : "red ", na, ops / (ms * 1e-3) / 1e9, ms);
    }
  return 0;
}
