// Latency of warp reductions on this GPU: redux.sync.min.u32 vs a 5-round
// shfl.xor min (one warp, dependent chain).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(unsigned* out, long long* cyc, int iters) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_min_sync(0xffffffffu, v) + threadIdx.x;
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, off));
    v += threadIdx.x;
  }
  long long t2 = clock64();
  unsigned long long k = v;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, off);
      k = o < k ? o : k;
    }
    k += threadIdx.x;
  }
  long long t3 = clock64();
  out[threadIdx.x] = v + (unsigned)k;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / iters;
    cyc[1] = (t2 - t1) / iters;
    cyc[2] = (t3 - t2) / iters;
  }
}

int main() {
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, 4 * 32);
  cudaMalloc(&cyc, 8 * 3);
  lat_kernel<<<1, 32>>>(out, cyc, 1000);
  lat_kernel<<<1, 32>>>(out, cyc, 1000);
  long long h[3];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("redux.min.u32: %lld cycles; 5-round shfl min u32: %lld; 5-round shfl min u64: %lld\n", h[0],
         h[1], h[2]);
  return 0;
}
