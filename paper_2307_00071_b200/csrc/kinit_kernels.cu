// kinit_kernels.cu — k-means++ seeding with exponential clocks (sm_100a).
//
// Reference: /root/reference/proj/src/sogmm.cpp:197-337 (kinit).
// Bit-exactness: keys and draws are 64-bit integer ports of rng.hpp; the
// distance d2 = ((e0^2 + e1^2) + e2^2) + e3^2 is evaluated with explicit
// round-to-nearest FP64 intrinsics (no FMA contraction, like the SSE2
// reference build); the clock is an IEEE FP64 division. The only inexact
// ingredient is -log(u): CUDA's FP64 log and glibc's may differ by 1 ulp,
// which can only flip a round whose two best clocks are within ~2 ulp.
// Ties are resolved on (clock, index) lexicographically = the reference's
// strict-< scan in index order, and identical keys produce identical clocks.
//
// The nearest-centre pass (sogmm.cpp:290-312) is folded into the seeding
// rounds: round r already evaluates d(x, c_{r-1}) for every point, so the
// running argmin with strict < over ascending centre index is tracked for
// free; one extra fold of c_{k-1} completes the labels. This removes the
// reference's N x K distance pass entirely.
#include <climits>

#include "kinit_kernels.cuh"

namespace gmmb {

namespace {

__device__ __forceinline__ double dist2(double x0, double x1, double x2,
                                        double x3, const double (&c)[4]) {
  const double e0 = __dsub_rn(x0, c[0]);
  const double e1 = __dsub_rn(x1, c[1]);
  const double e2 = __dsub_rn(x2, c[2]);
  const double e3 = __dsub_rn(x3, c[3]);
  double s = __dadd_rn(__dmul_rn(e0, e0), __dmul_rn(e1, e1));
  s = __dadd_rn(s, __dmul_rn(e2, e2));
  return __dadd_rn(s, __dmul_rn(e3, e3));
}

__device__ __forceinline__ double neg_log_u(uint64_t seed, int r, uint64_t key) {
  const uint64_t b = rng_bits(seed, static_cast<uint64_t>(r), key);
  const double u = static_cast<double>((b >> 11) + 1) * 0x1.0p-53;  // rng.hpp:37-41
  return -log(u);
}

// lexicographic (clock, idx) minimum; idx -1 = none
__device__ __forceinline__ void cand_min(double& c, long long& i, double c2,
                                         long long i2) {
  if (i2 < 0) return;
  if (i < 0 || c2 < c || (c2 == c && i2 < i)) {
    c = c2;
    i = i2;
  }
}

__device__ __forceinline__ void warp_cand_min(double& c, long long& i,
                                              long long& u) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double c2 = __shfl_xor_sync(0xffffffffu, c, off);
    const long long i2 = __shfl_xor_sync(0xffffffffu, i, off);
    const long long u2 = __shfl_xor_sync(0xffffffffu, u, off);
    cand_min(c, i, c2, i2);
    u = u2 < u ? u2 : u;
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void keys_kernel(const double* __restrict__ x64, int64_t n,
                            const double* __restrict__ tail,
                            uint64_t* __restrict__ keys) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t h = 0x6a09e667f3bcc909ULL;  // rng.hpp:64-70
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double v = i + j < n ? x64[i + j] : tail[i + j - n];
    h = mix64(h ^ static_cast<uint64_t>(__double_as_longlong(v)));
  }
  keys[i] = h;
}

constexpr int kSeedThreads = 512;

// PPT > 0: each thread keeps PPT points (stride = grid threads) in registers.
// PPT == 0: points, d2, labels and chosen flags live in global memory.
template <int PPT>
__global__ void __launch_bounds__(kSeedThreads)
    kpp_seed_kernel(const double* __restrict__ x64, int64_t n, int k,
                    uint64_t seed, KinitScratch scr) {
  __shared__ double s_c[kSeedThreads / 32];
  __shared__ long long s_i[kSeedThreads / 32];
  __shared__ long long s_u[kSeedThreads / 32];
  __shared__ long long s_win;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = gridDim.x;
  const int64_t G = static_cast<int64_t>(nblk) * kSeedThreads;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * kSeedThreads + tid;
  constexpr int R = PPT > 0 ? PPT : 1;
  double px[R][4], d2[R];
  uint64_t key[R];
  int lab[R];
  bool chosen[R];
  if constexpr (PPT > 0) {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int64_t i = g0 + j * G;
      const bool v = i < n;
#pragma unroll
      for (int q = 0; q < 4; ++q) px[j][q] = v ? x64[q * n + i] : 0.0;
      key[j] = v ? scr.keys[i] : 0;
      d2[j] = INFINITY;
      lab[j] = 0;
      chosen[j] = false;
    }
  }
  double c[4] = {0, 0, 0, 0};
  long long prev = -1;
  for (int r = 0; r <= k; ++r) {
    // fold centre c_{r-1} into d2 and the running nearest-centre label
    double bc = INFINITY;
    long long bi = -1, bu = LLONG_MAX;
    if constexpr (PPT > 0) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int64_t i = g0 + j * G;
        if (i >= n) continue;
        if (r > 0) {
          const double dd = dist2(px[j][0], px[j][1], px[j][2], px[j][3], c);
          if (dd < d2[j]) {
            d2[j] = dd;
            lab[j] = r - 1;
          }
          if (i == prev) chosen[j] = true;
        }
        if (r == k) continue;
        const double nl = neg_log_u(seed, r, key[j]);
        if (r == 0) {
          cand_min(bc, bi, nl, i);
        } else if (d2[j] > 0.0) {
          const double clk = nl / d2[j];
          if (clk < INFINITY) cand_min(bc, bi, clk, i);
        }
        if (!chosen[j] && i < bu) bu = i;
      }
    } else {
      for (int64_t i = g0; i < n; i += G) {
        double dcur = r > 0 ? scr.d2[i] : INFINITY;
        if (r > 0) {
          const double dd = dist2(x64[i], x64[n + i], x64[2 * n + i], x64[3 * n + i], c);
          if (dd < dcur) {
            dcur = dd;
            scr.d2[i] = dd;
            scr.labels[i] = r - 1;
          }
          if (i == prev) scr.chosen[i] = 1;
        } else {
          scr.d2[i] = INFINITY;
          scr.labels[i] = 0;
          scr.chosen[i] = 0;
        }
        if (r == k) continue;
        const double nl = neg_log_u(seed, r, scr.keys[i]);
        if (r == 0) {
          cand_min(bc, bi, nl, i);
        } else if (dcur > 0.0) {
          const double clk = nl / dcur;
          if (clk < INFINITY) cand_min(bc, bi, clk, i);
        }
        if (!scr.chosen[i] && i < bu) bu = i;
      }
    }
    if (r == k) break;
    // CTA reduce
    warp_cand_min(bc, bi, bu);
    if (lane == 0) {
      s_c[warp] = bc;
      s_i[warp] = bi;
      s_u[warp] = bu;
    }
    __syncthreads();
    KppSlot* slots = scr.slots + (r & 1) * nblk;
    if (warp == 0) {
      bc = lane < kSeedThreads / 32 ? s_c[lane] : INFINITY;
      bi = lane < kSeedThreads / 32 ? s_i[lane] : -1;
      bu = lane < kSeedThreads / 32 ? s_u[lane] : LLONG_MAX;
      warp_cand_min(bc, bi, bu);
      if (lane == 0) {
        KppSlot& sl = slots[blockIdx.x];
        sl.clock = bc;
        sl.idx = bi;
        sl.unchosen = bu;
        __threadfence();
        st_release(&sl.tag, r + 1);
      }
    }
    // all-gather: every CTA reduces every CTA's candidate (same order => same
    // winner everywhere), which doubles as the grid barrier of this round
    bc = INFINITY;
    bi = -1;
    bu = LLONG_MAX;
    for (int b = tid; b < nblk; b += kSeedThreads) {
      const KppSlot& sl = slots[b];
      while (ld_acquire(&sl.tag) != r + 1) {
      }
      const double c2 = *reinterpret_cast<const volatile double*>(&sl.clock);
      const long long i2 = *reinterpret_cast<const volatile long long*>(&sl.idx);
      const long long u2 = *reinterpret_cast<const volatile long long*>(&sl.unchosen);
      cand_min(bc, bi, c2, i2);
      bu = u2 < bu ? u2 : bu;
    }
    warp_cand_min(bc, bi, bu);
    __syncthreads();  // s_* reuse
    if (lane == 0) {
      s_c[warp] = bc;
      s_i[warp] = bi;
      s_u[warp] = bu;
    }
    __syncthreads();
    if (warp == 0) {
      bc = lane < kSeedThreads / 32 ? s_c[lane] : INFINITY;
      bi = lane < kSeedThreads / 32 ? s_i[lane] : -1;
      bu = lane < kSeedThreads / 32 ? s_u[lane] : LLONG_MAX;
      warp_cand_min(bc, bi, bu);
      if (lane == 0) {
        // sogmm.cpp:276-284 fallback: lowest unchosen index
        const long long win = bi >= 0 && bc < INFINITY ? bi : bu;
        s_win = win;
        if (blockIdx.x == 0) scr.centers[r] = win;
      }
    }
    __syncthreads();
    prev = s_win;
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = x64[q * n + prev];
  }
  // labels + owned counts (every point's final nearest centre)
  if constexpr (PPT > 0) {
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      const int64_t i = g0 + j * G;
      if (i >= n) continue;
      scr.labels[i] = lab[j];
      atomicAdd(&scr.owned[lab[j]], 1);
    }
  } else {
    for (int64_t i = g0; i < n; i += G) atomicAdd(&scr.owned[scr.labels[i]], 1);
  }
}

// Owned fix-up, single CTA (sogmm.cpp:315-331).
__global__ void __launch_bounds__(1024)
    fixup_kernel(int64_t n, int k, int32_t* __restrict__ labels,
                 int* __restrict__ owned) {
  __shared__ int s_any;
  __shared__ int s_v[1024];
  __shared__ long long s_l[1024];
  const int tid = threadIdx.x;
  if (tid == 0) s_any = 0;
  __syncthreads();
  for (int b = tid; b < k; b += 1024)
    if (owned[b] == 0) s_any = 1;
  __syncthreads();
  if (!s_any) return;
  for (int b = 0; b < k; ++b) {
    if (owned[b] > 0) continue;  // uniform: owned[] only changes below
    // donor = argmax owned, lowest index on ties (strict >)
    int bv = -1, bidx = 0;
    for (int c = tid; c < k; c += 1024) {
      if (owned[c] > bv) {
        bv = owned[c];
        bidx = c;
      }
    }
    s_v[tid] = bv;
    s_l[tid] = bidx;
    __syncthreads();
    for (int off = 512; off >= 1; off >>= 1) {
      if (tid < off) {
        const int v2 = s_v[tid + off];
        const long long i2 = s_l[tid + off];
        if (v2 > s_v[tid] || (v2 == s_v[tid] && i2 < s_l[tid])) {
          s_v[tid] = v2;
          s_l[tid] = i2;
        }
      }
      __syncthreads();
    }
    const int donor = static_cast<int>(s_l[0]);
    __syncthreads();
    long long lo = LLONG_MAX;
    for (int64_t i = tid; i < n; i += 1024) {
      if (labels[i] == donor) {
        lo = i;
        break;
      }
    }
    s_l[tid] = lo;
    __syncthreads();
    for (int off = 512; off >= 1; off >>= 1) {
      if (tid < off && s_l[tid + off] < s_l[tid]) s_l[tid] = s_l[tid + off];
      __syncthreads();
    }
    if (tid == 0 && s_l[0] != LLONG_MAX) {
      labels[s_l[0]] = b;
      owned[donor]--;
      owned[b]++;
    }
    __syncthreads();
  }
}

// ---- sharded rounds ----
__device__ __forceinline__ void winner_from(const KppRankSlot* prev, int world,
                                            long long& win, double (&c)[4]) {
  double bc = INFINITY;
  long long bi = -1, bu = LLONG_MAX;
  int ri = -1, ru = -1;
  for (int w = 0; w < world; ++w) {
    const double c2 = prev[w].clock;
    const long long i2 = prev[w].idx;
    if (i2 >= 0 && (bi < 0 || c2 < bc || (c2 == bc && i2 < bi))) {
      bc = c2;
      bi = i2;
      ri = w;
    }
    if (prev[w].unchosen < bu) {
      bu = prev[w].unchosen;
      ru = w;
    }
  }
  if (bi >= 0 && bc < INFINITY) {
    win = bi;
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = prev[ri].x[q];
  } else {
    win = bu;
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = ru >= 0 ? prev[ru].ux[q] : 0.0;
  }
}

__global__ void __launch_bounds__(512)
    kpp_round_kernel(const double* __restrict__ x64, int64_t n, int64_t offset,
                     int r, uint64_t seed, const KppRankSlot* __restrict__ prev,
                     int world, KinitScratch scr, KppRankSlot* out,
                     int* ticket) {
  __shared__ double s_c[16];
  __shared__ long long s_i[16];
  __shared__ long long s_u[16];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = static_cast<int64_t>(gridDim.x) * 512;
  double c[4] = {0, 0, 0, 0};
  long long win = -1;
  if (r > 0) winner_from(prev, world, win, c);
  double bc = INFINITY;
  long long bi = -1, bu = LLONG_MAX;
  for (int64_t li = static_cast<int64_t>(blockIdx.x) * 512 + tid; li < n; li += G) {
    const long long gi = offset + li;
    double dcur;
    if (r > 0) {
      dcur = scr.d2[li];
      const double dd = dist2(x64[li], x64[n + li], x64[2 * n + li], x64[3 * n + li], c);
      if (dd < dcur) {
        dcur = dd;
        scr.d2[li] = dd;
        scr.labels[li] = r - 1;
      }
      if (gi == win) scr.chosen[li] = 1;
    } else {
      dcur = INFINITY;
      scr.d2[li] = INFINITY;
      scr.labels[li] = 0;
      scr.chosen[li] = 0;
    }
    const double nl = neg_log_u(seed, r, scr.keys[li]);
    if (r == 0) {
      cand_min(bc, bi, nl, gi);
    } else if (dcur > 0.0) {
      const double clk = nl / dcur;
      if (clk < INFINITY) cand_min(bc, bi, clk, gi);
    }
    if (!scr.chosen[li] && gi < bu) bu = gi;
  }
  warp_cand_min(bc, bi, bu);
  if (lane == 0) {
    s_c[warp] = bc;
    s_i[warp] = bi;
    s_u[warp] = bu;
  }
  __syncthreads();
  if (warp == 0) {
    bc = lane < 16 ? s_c[lane] : INFINITY;
    bi = lane < 16 ? s_i[lane] : -1;
    bu = lane < 16 ? s_u[lane] : LLONG_MAX;
    warp_cand_min(bc, bi, bu);
    if (lane == 0) {
      KppSlot& sl = scr.slots[blockIdx.x];
      sl.clock = bc;
      sl.idx = bi;
      sl.unchosen = bu;
      __threadfence();
      s_last = (atomicAdd(ticket, 1) == static_cast<int>(gridDim.x) - 1);
    }
  }
  __syncthreads();
  if (!s_last) return;
  // last CTA: reduce all CTA slots in order -> this rank's candidate
  __threadfence();
  bc = INFINITY;
  bi = -1;
  bu = LLONG_MAX;
  for (int b = tid; b < static_cast<int>(gridDim.x); b += 512) {
    const volatile KppSlot& sl = scr.slots[b];
    cand_min(bc, bi, sl.clock, sl.idx);
    bu = sl.unchosen < bu ? sl.unchosen : bu;
  }
  warp_cand_min(bc, bi, bu);
  __syncthreads();
  if (lane == 0) {
    s_c[warp] = bc;
    s_i[warp] = bi;
    s_u[warp] = bu;
  }
  __syncthreads();
  if (warp == 0) {
    bc = lane < 16 ? s_c[lane] : INFINITY;
    bi = lane < 16 ? s_i[lane] : -1;
    bu = lane < 16 ? s_u[lane] : LLONG_MAX;
    warp_cand_min(bc, bi, bu);
    if (lane == 0) {
      out->clock = bc;
      out->idx = bi;
      out->unchosen = bu;
      for (int q = 0; q < 4; ++q) {
        out->x[q] = bi >= 0 ? x64[q * n + (bi - offset)] : 0.0;
        out->ux[q] = bu != LLONG_MAX ? x64[q * n + (bu - offset)] : 0.0;
      }
      *ticket = 0;
      if (r > 0) scr.centers[r - 1] = win;
    }
  }
}

__global__ void kpp_final_kernel(const double* __restrict__ x64, int64_t n,
                                 int64_t offset, int k,
                                 const KppRankSlot* __restrict__ prev,
                                 int world, KinitScratch scr) {
  double c[4];
  long long win;
  winner_from(prev, world, win, c);
  const int64_t li = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (li == 0) scr.centers[k - 1] = win;
  if (li >= n) return;
  int lab = scr.labels[li];
  const double dd = dist2(x64[li], x64[n + li], x64[2 * n + li], x64[3 * n + li], c);
  if (dd < scr.d2[li]) lab = k - 1;
  scr.labels[li] = lab;
  atomicAdd(&scr.owned[lab], 1);
}

}  // namespace

cudaError_t launch_keys(const double* x64, int64_t n, const double* tail,
                        uint64_t* keys, cudaStream_t s) {
  const int grid = static_cast<int>((n + 255) / 256);
  keys_kernel<<<grid, 256, 0, s>>>(x64, n, tail, keys);
  return cudaGetLastError();
}

template <int PPT>
static cudaError_t launch_seed_t(const double* x64, int64_t n, int k,
                                 uint64_t seed, KinitScratch scr, int nblk,
                                 cudaStream_t s) {
  void* args[] = {(void*)&x64, (void*)&n, (void*)&k, (void*)&seed, (void*)&scr};
  return cudaLaunchCooperativeKernel((void*)kpp_seed_kernel<PPT>, dim3(nblk),
                                     dim3(kSeedThreads), args, 0, s);
}

cudaError_t launch_kpp_seed(const double* x64, int64_t n, int k, uint64_t seed,
                            KinitScratch scr, int sm_count, cudaStream_t s) {
  // pick the smallest register-resident variant that covers n
  auto blocks_for = [&](const void* f) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, kSeedThreads, 0);
    return per < 1 ? 1 : per;
  };
  struct V {
    int ppt;
    const void* f;
  } vs[] = {{1, (const void*)kpp_seed_kernel<1>},
            {2, (const void*)kpp_seed_kernel<2>},
            {4, (const void*)kpp_seed_kernel<4>},
            {8, (const void*)kpp_seed_kernel<8>}};
  for (const V& v : vs) {
    const int nblk = sm_count * blocks_for(v.f);
    if (static_cast<int64_t>(nblk) * kSeedThreads * v.ppt >= n) {
      switch (v.ppt) {
        case 1: return launch_seed_t<1>(x64, n, k, seed, scr, nblk, s);
        case 2: return launch_seed_t<2>(x64, n, k, seed, scr, nblk, s);
        case 4: return launch_seed_t<4>(x64, n, k, seed, scr, nblk, s);
        default: return launch_seed_t<8>(x64, n, k, seed, scr, nblk, s);
      }
    }
  }
  const int nblk = sm_count * blocks_for((const void*)kpp_seed_kernel<0>);
  return launch_seed_t<0>(x64, n, k, seed, scr, nblk, s);
}

cudaError_t launch_fixup(int64_t n, int k, KinitScratch scr, cudaStream_t s) {
  fixup_kernel<<<1, 1024, 0, s>>>(n, k, scr.labels, scr.owned);
  return cudaGetLastError();
}

cudaError_t launch_kpp_round(const double* x64, int64_t n, int64_t offset,
                             int r, uint64_t seed, const KppRankSlot* prev,
                             int world, KinitScratch scr, KppRankSlot* out,
                             int* ticket, int sm_count, cudaStream_t s) {
  int grid = static_cast<int>((n + 511) / 512);
  if (grid > sm_count * 4) grid = sm_count * 4;
  if (grid < 1) grid = 1;
  kpp_round_kernel<<<grid, 512, 0, s>>>(x64, n, offset, r, seed, prev, world,
                                        scr, out, ticket);
  return cudaGetLastError();
}

cudaError_t launch_kpp_final(const double* x64, int64_t n, int64_t offset,
                             int k, const KppRankSlot* prev, int world,
                             KinitScratch scr, cudaStream_t s) {
  const int grid = static_cast<int>((n + 255) / 256);
  kpp_final_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(x64, n, offset, k, prev, world, scr);
  return cudaGetLastError();
}

}  // namespace gmmb
