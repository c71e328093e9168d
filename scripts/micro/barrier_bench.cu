// Microbenchmark: per-round cost of grid-wide exchange variants (1 CTA/SM).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_release(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory"); }
__device__ __forceinline__ void red_relaxed(unsigned* p) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory"); }
__device__ __forceinline__ void fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

struct Slot { double c; long long i; long long pad[6]; };

template <int MODE>
__global__ void bench(unsigned* counter, Slot* slots, int rounds, double* out) {
  __shared__ double best;
  const int nblk = gridDim.x;
  double acc = 0;
  for (int r = 0; r < rounds; ++r) {
    Slot* sl = slots + (r & 1) * nblk;
    if (MODE == 3) {
      if (threadIdx.x == 0) { sl[blockIdx.x].c = r + blockIdx.x; }
      cg::this_grid().sync();
    } else if (threadIdx.x == 0) {
      sl[blockIdx.x].c = r + blockIdx.x * 1e-3;
      unsigned target = nblk * (r + 1);
      if (MODE == 0) { red_release(counter); while (ld_relaxed(counter) < target) {} fence(); }
      if (MODE == 1) { red_release(counter); while (ld_acquire(counter) < target) {} }
      if (MODE == 2) { __threadfence(); red_relaxed(counter); while (ld_relaxed(counter) < target) {} __threadfence(); }
      if (MODE == 4) { red_release(counter); while (ld_relaxed(counter) < target) { __nanosleep(32); } fence(); }
    }
    __syncthreads();
    if (MODE != 5) {
      // read all slots (threads < nblk), min-reduce
      double v = 1e300;
      if (threadIdx.x < nblk) v = ((volatile Slot*)sl)[threadIdx.x].c;
      for (int off = 16; off; off >>= 1) v = fmin(v, __shfl_xor_sync(~0u, v, off));
      if ((threadIdx.x & 31) == 0) atomicMin((unsigned long long*)&best, 0);  // placeholder
      acc += v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

template <int MODE>
void run(const char* name, int nblk, int threads) {
  unsigned* counter; Slot* slots; double* out;
  cudaMalloc(&counter, 4); cudaMalloc(&slots, sizeof(Slot) * 2 * nblk); cudaMalloc(&out, 8);
  int rounds = 2000;
  void* args[] = {&counter, &slots, &rounds, &out};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(counter, 0, 4);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)bench<MODE>, dim3(nblk), dim3(threads), args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep == 2) printf("%-28s blocks %4d threads %4d : %.3f us/round  (%s)\n", name, nblk, threads, ms * 1000 / rounds, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int sm; cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {384, 1024}) {
    run<0>("red.release+relaxed+fence", sm, t);
    run<1>("red.release+ld.acquire", sm, t);
    run<2>("threadfence+red+relaxed", sm, t);
    run<3>("cg grid.sync", sm, t);
    run<4>("release+nanosleep poll", sm, t);
  }
  run<0>("red.release+relaxed+fence", sm * 2, 384);
  run<0>("red.release+relaxed+fence", 32, 384);
  return 0;
}
