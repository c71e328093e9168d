// common.cuh — shared device helpers for the B200 GMM learner (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gmmb {

constexpr double kLog2Pi = 1.8378770664093454836;   // sogmm.cpp:19
constexpr double kLog2E = 1.4426950408889634074;
constexpr double kLn2 = 0.69314718055994530942;
constexpr double kDegenerateCount = 1e-10;          // kernels.hpp:61
constexpr int kTile = 128;       // points per recentring super-tile
constexpr int kMaxK = 4096;      // largest K the fused E/M kernel supports
constexpr int kCtaComps = 512;   // components per CTA of the fused kernel

// packed lower triangle, row-major (packed10.hpp:11-14); D=3 uses the first 6
__host__ __device__ constexpr int packed_row(int k) {
  return k < 1 ? 0 : k < 3 ? 1 : k < 6 ? 2 : 3;
}
__host__ __device__ constexpr int packed_col(int k) {
  return k < 1 ? k : k < 3 ? k - 1 : k < 6 ? k - 3 : k - 6;
}
__host__ __device__ constexpr int npacked(int d) { return d * (d + 1) / 2; }
// sufficient statistics per component: count, D first moments, packed second
__host__ __device__ constexpr int nstats(int d) { return 1 + d + npacked(d); }

__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---- counter-based RNG, bit-exact port of rng.hpp:16-70 -----------------
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t rng_bits(uint64_t seed, uint64_t stream,
                                             uint64_t counter) {
  constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
  uint64_t h = mix64(seed ^ 0x2545f4914f6cdd1dULL);
  h = mix64(h + stream * kGolden);
  h = mix64(h + counter * kGolden);
  return h;
}

// Per-component E-step constants, FP32 (16 floats = 4 x float4):
//   p[0..npacked(D)-1] : sqrt(0.5*log2 e) * P (P = L^{-1}), packed lower
//   p[10]              : base2 = log2(e) * (ln w + sum ln diag P - D/2 ln 2pi)
// so that log2 of w*N(x) = base2 - |p (x - mu)|^2.
struct __align__(16) CompConst {
  float p[16];
};

// Device state of one EM run (one per context, lives in device memory).
struct EmState {
  int iter;          // E steps completed
  int done;          // 1 once converged / max_iters / error
  int k_cur;         // components of the current model
  int cur;           // which model buffer is current (0/1)
  int removed;       // removed_components accumulated
  int error;         // 0 ok, 3 numerical
  int error_index;   // component index for the message
  int error_kind;    // 1 non-SPD, 2 all degenerate, 3 cholesky(prep)
  double ll_prev;
  double ll;
  int converged;     // 1 if the exit was the tolerance break
  int max_iters;
  double tol;
  double cov_reg;
  double npts;       // global point count (for the unit counter)
  double units;      // sum over E steps of N * K_t
};

}  // namespace gmmb
