// Cost of kinit's fold phase in isolation: W warps per CTA, PPT points per
// thread in shared memory (SoA like kpp_seed_kernel), two FP64 centres per
// step, strict-< update. Prints cycles per step for warp 0.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kT = 352;

__device__ __forceinline__ double dist2(double x0, double x1, double x2, double x3, const double* c) {
  const double e0 = __dsub_rn(x0, c[0]), e1 = __dsub_rn(x1, c[1]);
  const double e2 = __dsub_rn(x2, c[2]), e3 = __dsub_rn(x3, c[3]);
  double s = __dadd_rn(__dmul_rn(e0, e0), __dmul_rn(e1, e1));
  s = __dadd_rn(s, __dmul_rn(e2, e2));
  return __dadd_rn(s, __dmul_rn(e3, e3));
}

template <int MODE>
__global__ void fold_kernel(int ppt, int steps, int active_warps, long long* out, int* sink) {
  extern __shared__ double sm[];
  double* x = sm;                    // [4][ppt][kT]
  double* d2 = sm + 4 * ppt * kT;    // [ppt][kT]
  int* lab = reinterpret_cast<int*>(d2 + ppt * kT);
  const int t = threadIdx.x, warp = t >> 5;
  for (int j = 0; j < ppt; ++j) {
    for (int q = 0; q < 4; ++q) x[(q * ppt + j) * kT + t] = (t * 7 + j * 13 + q) * 0.001;
    d2[j * kT + t] = 1e30;
    lab[j * kT + t] = 0;
  }
  __syncthreads();
  if (warp >= active_warps) return;
  double cf[2][4];
  unsigned cm = 0;
  const long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    for (int f = 0; f < 2; ++f)
      for (int q = 0; q < 4; ++q) cf[f][q] = 0.5 + 0.01 * ((s * 2 + f) * 4 + q) * (1 + (s & 3));
    if (MODE == 0) {
#pragma unroll 1
      for (int j = 0; j < ppt; ++j) {
        const int o = j * kT + t;
        const double x0 = x[o], x1 = x[o + ppt * kT], x2 = x[o + 2 * ppt * kT], x3 = x[o + 3 * ppt * kT];
        double dj = d2[o];
        int lb = -1;
        for (int f = 0; f < 2; ++f) {
          const double dd = dist2(x0, x1, x2, x3, cf[f]);
          if (dd < dj) {
            dj = dd;
            lb = s * 2 + f;
          }
        }
        if (lb >= 0) {
          d2[o] = dj;
          lab[o] = lb;
          cm |= 1u << j;
        }
      }
    } else if (MODE == 2) {
      // all PPT (= 6) points at once, branch-free: 12 independent chains
      constexpr int P = 6;
      double dj[P];
      int lb[P];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const int o = j * kT + t;
        const double x0 = x[o], x1 = x[o + P * kT], x2 = x[o + 2 * P * kT], x3 = x[o + 3 * P * kT];
        const double d = d2[o];
        const double e0 = dist2(x0, x1, x2, x3, cf[0]);
        const double e1 = dist2(x0, x1, x2, x3, cf[1]);
        const bool c0 = e0 < d;
        const double m0 = c0 ? e0 : d;
        const bool c1 = e1 < m0;
        dj[j] = c1 ? e1 : m0;
        lb[j] = c1 ? s * 2 + 1 : c0 ? s * 2 : -1;
      }
#pragma unroll
      for (int j = 0; j < P; ++j) {
        if (lb[j] >= 0) {
          const int o = j * kT + t;
          d2[o] = dj[j];
          lab[o] = lb[j];
          cm |= 1u << j;
        }
      }
    } else {
      // registers only (no shared memory): the arithmetic floor
#pragma unroll 1
      for (int j = 0; j < ppt; ++j) {
        const double x0 = t * 0.001 + j, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
        double dj = 1e30 + s;
        int lb = -1;
        for (int f = 0; f < 2; ++f) {
          const double dd = dist2(x0, x1, x2, x3, cf[f]);
          if (dd < dj) {
            dj = dd;
            lb = s * 2 + f;
          }
        }
        cm += lb;
      }
    }
  }
  const long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = (t1 - t0) / steps;
  if (cm == 12345) sink[0] = 1;
}

int main() {
  long long* out;
  int* sink;
  cudaMalloc(&out, sizeof(long long) * 148);
  cudaMalloc(&sink, 4);
  const int ppt = 6;
  const size_t bytes = static_cast<size_t>(ppt) * kT * (5 * 8 + 4);
  cudaFuncSetAttribute(fold_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cudaFuncSetAttribute(fold_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cudaFuncSetAttribute(fold_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  for (int mode = 0; mode < 3; ++mode)
    for (int aw : {1, 4, 11}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) fold_kernel<0><<<148, kT, bytes>>>(ppt, 200, aw, out, sink);
        else if (mode == 1) fold_kernel<1><<<148, kT, bytes>>>(ppt, 200, aw, out, sink);
        else fold_kernel<2><<<148, kT, bytes>>>(ppt, 200, aw, out, sink);
      }
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      printf("mode %s, %2d active warps: %lld cycles per fold step (6 points x 2 centres), CTA 0\n",
             mode == 0 ? "smem" : mode == 1 ? "regs" : "smem, 6-way", aw, h[0]);
    }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
