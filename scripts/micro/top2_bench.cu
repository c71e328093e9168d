// Latency of kinit's warp top-2 (both levels, redux- and shuffle-based) for
// one warp, inputs from shared memory like the communication warp's CTA
// reduce.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void merge_top2(float& a1, int& i1, float& a2, float b1, int j1, float b2) {
  const bool take = (j1 >= 0) & ((i1 < 0) | (b1 < a1) | ((b1 == a1) & (j1 < i1)));
  const float n2 = take ? fminf(a1, b2) : fminf(a2, b1);
  a1 = take ? b1 : a1;
  i1 = take ? j1 : i1;
  a2 = n2;
}
__device__ __forceinline__ void merge_top2d(float& a1, int& i1, float& a2, double& d, float b1, int j1,
                                            float b2, double e) {
  const bool take = (j1 >= 0) & ((i1 < 0) | (b1 < a1) | ((b1 == a1) & (j1 < i1)));
  merge_top2(a1, i1, a2, b1, j1, b2);
  d = take ? e : d;
}
__device__ __forceinline__ void top2_redux(float& a1, int& i1, float& a2) {
  const unsigned u1 = __float_as_uint(a1);
  const unsigned m1 = __reduce_min_sync(0xffffffffu, u1);
  const unsigned mi = __reduce_min_sync(0xffffffffu, u1 == m1 ? static_cast<unsigned>(i1) : ~0u);
  const unsigned u2 = static_cast<unsigned>(i1) == mi ? __float_as_uint(a2) : u1;
  a2 = __uint_as_float(__reduce_min_sync(0xffffffffu, u2));
  a1 = __uint_as_float(m1);
  i1 = static_cast<int>(mi);
}
template <int MODE>
__device__ __forceinline__ void top2s(float& a1, int& i1, float& a2, float& b1, int& j1, float& b2,
                                      double& bd) {
  if (MODE == 0) {
    top2_redux(a1, i1, a2);
    const unsigned u1 = __float_as_uint(b1);
    const unsigned m1 = __reduce_min_sync(0xffffffffu, u1);
    const unsigned mj = __reduce_min_sync(0xffffffffu, u1 == m1 ? static_cast<unsigned>(j1) : ~0u);
    const bool holder = static_cast<unsigned>(j1) == mj;
    const unsigned u2 = holder ? __float_as_uint(b2) : u1;
    b2 = __uint_as_float(__reduce_min_sync(0xffffffffu, u2));
    const int src = __ffs(__ballot_sync(0xffffffffu, holder)) - 1;
    bd = __shfl_sync(0xffffffffu, bd, src);
    b1 = __uint_as_float(m1);
    j1 = static_cast<int>(mj);
  } else {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const float o1 = __shfl_xor_sync(0xffffffffu, a1, off);
      const int oi = __shfl_xor_sync(0xffffffffu, i1, off);
      const float o2 = __shfl_xor_sync(0xffffffffu, a2, off);
      const float p1 = __shfl_xor_sync(0xffffffffu, b1, off);
      const int pj = __shfl_xor_sync(0xffffffffu, j1, off);
      const float p2 = __shfl_xor_sync(0xffffffffu, b2, off);
      const double pd = __shfl_xor_sync(0xffffffffu, bd, off);
      merge_top2(a1, i1, a2, o1, oi, o2);
      merge_top2d(b1, j1, b2, bd, p1, pj, p2, pd);
    }
  }
}

template <int MODE>
__global__ void k(const float* in, float* out, long long* cyc, int iters) {
  __shared__ float sa1[32], sa2[32], sb1[32], sb2[32];
  __shared__ int si1[32], sj1[32];
  __shared__ double sd[32];
  const int l = threadIdx.x;
  float acc = 0;
  long long tot = 0;
  for (int it = 0; it < iters; ++it) {
    sa1[l] = in[l] + it; sa2[l] = in[l] + 2 + it; sb1[l] = in[l + 32]; sb2[l] = in[l + 32] + 1;
    si1[l] = l < 11 ? l * 7 + it : -1; sj1[l] = l < 11 ? l * 5 : -1; sd[l] = l;
    __syncwarp();
    const long long t0 = clock64();
    float a1 = sa1[l], a2 = sa2[l], b1 = sb1[l], b2 = sb2[l];
    int i1 = si1[l], j1 = sj1[l];
    double bd = sd[l];
    top2s<MODE>(a1, i1, a2, b1, j1, b2, bd);
    acc += a1 + a2 + b1 + b2 + i1 + j1 + (float)bd;
    __syncwarp();
    const long long t1 = clock64();
    tot += t1 - t0;
  }
  out[l] = acc;
  if (l == 0) *cyc = tot / iters;
}

int main() {
  float *in, *out;
  long long* cyc;
  cudaMalloc(&in, 64 * 4);
  cudaMalloc(&out, 32 * 4);
  cudaMalloc(&cyc, 8);
  float h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1.0f + (i * 37 % 64);
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  long long c;
  k<0><<<1, 32>>>(in, out, cyc, 100);
  k<0><<<1, 32>>>(in, out, cyc, 100);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("redux top2s (smem loads + reduce): %lld cycles\n", c);
  k<1><<<1, 32>>>(in, out, cyc, 100);
  k<1><<<1, 32>>>(in, out, cyc, 100);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("shfl top2s (smem loads + reduce): %lld cycles\n", c);
  return 0;
}
