// FP32 issue-rate microbenchmark: scalar FFMA with 2 vs 3 distinct register
// sources, and packed fma.rn.f32x2 (FFMA2). Run: ./ffma2_bench
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// mode 0: x = fma(x, y, z) (z shared)   mode 1: x = fma(a, b, x) distinct a,b per chain
template <int MODE>
__global__ void __launch_bounds__(512) k_scalar(float* out, int iters, float s) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  float x[8], a[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = s * (t + j);
    a[j] = 0.9999f - s * j;
    b[j] = 1e-3f * s * (j + 1);
  }
  const float z = s * 0.5f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (MODE == 0) x[j] = fmaf(x[j], a[j], z);
        else x[j] = fmaf(a[j], b[(j + u) & 7], x[j]);
      }
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += x[j];
  out[t] = acc;
}

__global__ void __launch_bounds__(512) k_pair(float* out, int iters, float s) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long x[8], a[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = f2(s * (t + j), s * (t - j));
    a[j] = f2(0.9999f - s * j, 0.9998f - s * j);
    b[j] = f2(1e-3f * s * (j + 1), 2e-3f * s * (j + 1));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma2(a[j], b[(j + u) & 7], x[j]);
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

// mode 0: all pairs; 1: scalar broadcast operand; 2: FADD2 chains; 3: FMUL2 chains
template <int MODE>
__global__ void __launch_bounds__(256) k_pair2(float* out, int iters, float s) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long x[8], a[8];
  float b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = f2(s * (t + j), s * (t - j));
    a[j] = f2(0.9999f - s * j, 0.9998f - s * j);
    b[j] = 1e-3f * s * (j + 1);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float bb = b[(j + u) & 7];
        if (MODE == 1) x[j] = fma2(a[j], f2(bb, bb), x[j]);
        if (MODE == 2) {
          unsigned long long d;
          asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a[(j + u) & 7]), "l"(x[j]));
          x[j] = d;
        }
        if (MODE == 3) {
          unsigned long long d;
          asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a[(j + u) & 7]), "l"(x[j]));
          x[j] = d;
        }
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

template <typename K>
double run_t(K kern, int blocks, int threads, float* out, int iters, double fma_per_thread_iter) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, threads>>>(out, iters, 1e-7f);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(out, iters, 1e-7f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 2.0 * fma_per_thread_iter * iters * blocks * threads / (ms * 1e-3) / 1e12;
}

template <typename K>
double run(K kern, int blocks, float* out, int iters, double fma_per_thread_iter) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, 256>>>(out, iters, 1e-7f);
  cudaEventRecord(a);
  kern<<<blocks, 256>>>(out, iters, 1e-7f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return 2.0 * fma_per_thread_iter * iters * blocks * 256 / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  const int iters = 20000;
  for (int occ : {2, 4, 8}) {
    const int blocks = sms * occ;
    printf("CTAs/SM %d: scalar 2-reg %.1f TF | scalar 3-reg %.1f TF | f32x2 %.1f TF | "
           "f32x2 bcast %.1f | fadd2 %.1f | fmul2 %.1f (lane-ops x2 /s)\n", occ,
           run(k_scalar<0>, blocks, out, iters, 128), run(k_scalar<1>, blocks, out, iters, 128),
           run(k_pair, blocks, out, iters, 256), run(k_pair2<1>, blocks, out, iters, 256),
           run(k_pair2<2>, blocks, out, iters, 256), run(k_pair2<3>, blocks, out, iters, 256));
  }
  for (int w : {1, 2, 3, 4}) {
    printf("warps/SMSP %d (1 CTA/SM of %d threads): f32x2 %.1f TF | scalar 2-reg %.1f TF\n", w, 128 * w,
           run_t(k_pair, sms, 128 * w, out, iters, 256), run_t(k_scalar<0>, sms, 128 * w, out, iters, 128));
  }
  return 0;
}
