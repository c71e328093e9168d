// Microbenchmark: grid exchange latency per round (148 CTAs x 384 threads,
// 1 CTA/SM) for LL-protocol (payload, tag) words vs an arrival counter.
//   mode 0: counter (red.release + spin + fence) then read all slots
//   mode 1: LL all-to-all, warp 0 of every CTA polls every slot (contiguous)
//   mode 2: LL all-to-all, slots spread 256 B apart
//   mode 3: LL master: CTA 0 gathers, publishes 16 record copies 1 KB apart
//   mode 4: LL all-to-all, only lane 0..4 poll (one 16 B load per slot)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_ll(uint2* p, unsigned v, unsigned tag) {
  asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v), "r"(tag) : "memory");
}
__device__ __forceinline__ bool ld_ll2(const uint2* p, unsigned tag, unsigned& a, unsigned& b) {
  unsigned t0, t1;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(t0), "=r"(b), "=r"(t1) : "l"(p) : "memory");
  return t0 == tag && t1 == tag;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_release(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory"); }

template <int MODE>
__global__ void __launch_bounds__(384, 1) bench(unsigned* counter, uint2* ll, double* slots, int rounds, float* out) {
  __shared__ float best;
  const int nblk = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float acc = 0.f;
  for (int r = 0; r < rounds; ++r) {
    const unsigned tag = r + 1;
    const float mine = (float)((blockIdx.x * 7919 + r * 104729) % 1000);
    __syncthreads();
    if (warp == 0) {
      float m = 1e30f;
      if (MODE == 0) {
        double* sl = slots + (r & 1) * nblk * 8;
        if (lane == 0) {
          sl[blockIdx.x * 8] = mine;
          red_release(counter);
          while (ld_relaxed(counter) < (unsigned)nblk * (r + 1)) {}
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncwarp();
        for (int b = lane; b < nblk; b += 32) m = fminf(m, (float)((volatile double*)sl)[b * 8]);
      } else if (MODE == 1 || MODE == 2 || MODE == 4) {
        const int stride = MODE == 2 ? 32 : 2;  // words
        uint2* sl = ll + (r & 1) * nblk * 32;
        if (lane == 0) { st_ll(sl + blockIdx.x * stride, __float_as_uint(mine), tag); st_ll(sl + blockIdx.x * stride + 1, 0u, tag); }
        if (MODE == 4) {
          if (lane < 5) {
            for (int b = lane * 30; b < nblk && b < lane * 30 + 30; ++b) {
              unsigned a, c;
              while (!ld_ll2(sl + b * stride, tag, a, c)) {}
              m = fminf(m, __uint_as_float(a));
            }
          }
        } else {
          unsigned pend = 0;
          for (int b = lane, q = 0; b < nblk; b += 32, ++q) pend |= 1u << q;
          while (pend) {
#pragma unroll
            for (int q = 0; q < 5; ++q) {
              if ((pend >> q) & 1) {
                unsigned a, c;
                if (ld_ll2(sl + (lane + 32 * q) * stride, tag, a, c)) { m = fminf(m, __uint_as_float(a)); pend &= ~(1u << q); }
              }
            }
          }
        }
      } else if (MODE == 3) {
        uint2* sl = ll + (r & 1) * nblk * 2;
        uint2* rec = ll + 4096 + (r & 1) * 16 * 128;
        if (lane == 0) { st_ll(sl + blockIdx.x * 2, __float_as_uint(mine), tag); st_ll(sl + blockIdx.x * 2 + 1, 0u, tag); }
        if (blockIdx.x == 0) {
          unsigned pend = 0;
          for (int b = lane, q = 0; b < nblk; b += 32, ++q) pend |= 1u << q;
          while (pend) {
#pragma unroll
            for (int q = 0; q < 5; ++q) {
              if ((pend >> q) & 1) {
                unsigned a, c;
                if (ld_ll2(sl + (lane + 32 * q) * 2, tag, a, c)) { m = fminf(m, __uint_as_float(a)); pend &= ~(1u << q); }
              }
            }
          }
          for (int off = 16; off; off >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, off));
          if (lane < 16) { st_ll(rec + lane * 128, __float_as_uint(m), tag); st_ll(rec + lane * 128 + 1, 0u, tag); }
        }
        if (lane == 0) {
          unsigned a, c;
          while (!ld_ll2(rec + (blockIdx.x % 16) * 128, tag, a, c)) {}
          m = __uint_as_float(a);
        }
      }
      for (int off = 16; off; off >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, off));
      if (lane == 0) best = m;
    }
    __syncthreads();
    acc += best;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

template <int MODE>
void run(const char* name, int sms) {
  unsigned* counter; uint2* ll; double* slots; float* out;
  cudaMalloc(&counter, 4); cudaMalloc(&ll, 1 << 20); cudaMalloc(&slots, 1 << 20); cudaMalloc(&out, 4096);
  const int rounds = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(counter, 0, 4); cudaMemset(ll, 0, 1 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    bench<MODE><<<sms, 384>>>(counter, ll, slots, rounds, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep == 1) printf("%-40s %.3f us/round (%s)\n", name, ms * 1000 / rounds, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("counter + fence + read slots", sms);
  run<1>("LL all-to-all, contiguous, 32 lanes", sms);
  run<2>("LL all-to-all, 256 B spread, 32 lanes", sms);
  run<3>("LL master + 16 record copies", sms);
  run<4>("LL all-to-all, 5 lanes sequential", sms);
  return 0;
}
