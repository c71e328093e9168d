// kinit_tile.cu — k-means++ seeding for clouds beyond the shared-memory-
// resident kernel (cfg4: 4M points), with per-tile pruning (sm_100a).
//
// Reference: /root/reference/proj/src/sogmm.cpp:197-337 (kinit): round r
// picks argmin_i (-ln u_{r,i}) / d2_i over the points with d2_i > 0 (round 0:
// argmin -ln u), u from the coordinate-keyed counter RNG (rng.hpp:22-28),
// d2 the squared distance to the nearest chosen centre (FP64, folded one
// centre per round), ties to the lowest index; the labels are the running
// nearest centre (strict <, ascending centre index).
//
// Every round of the memory-resident kernel reads every point's state. Here
// the points are in the layout's Morton order, grouped in the layout's
// 128-point tiles, and two bounds skip almost all of that work without
// changing any decision:
//  * fold: the new centre c can only lower d2 inside a tile if the distance
//    from c to the tile's FP64 bounding box is below the tile's largest d2
//    (kept per tile, exact FP64); other tiles are not touched;
//  * clocks: a point can only win round r if its clock E / d2 < tau, i.e.
//    E < tau * Dmax_t (Dmax_t the tile's largest d2), i.e. its uniform
//    u > exp(-tau * Dmax_t): one compare on the top 32 bits of the draw
//    (u <= (hi32 + 1) 2^-32). Only those candidates get the exact FP64
//    clock (log + division, as the reference). If the best candidate's clock
//    is below tau, no other point can beat it: that is the round's exact
//    winner. Otherwise (rare) the round is repeated with a 64x larger tau,
//    up to tau = inf (every point with d2 > 0). tau = 12 / sum(d2) (the sum
//    from the previous exchange) leaves ~12 x (sum_t n_t Dmax_t / sum d2)
//    candidates per round and fails with probability ~e^-12.
// The draws (one mix64 per point per round, on keys stored in Morton order)
// remain; they are the reference's RNG and decide the candidates.
//
// One cooperative persistent launch: a CTA per SM owns a contiguous range of
// tiles; rounds end with a grid exchange of per-CTA (clock, index, sum d2)
// slots (arrival counter + fence), reduced by every CTA in the same order.
#include <climits>

#include "kinit_kernels.cuh"

namespace gmmb {

namespace {

constexpr int kTileKppThreads = 1024;
constexpr int kTileKppWarps = kTileKppThreads / 32;
constexpr uint64_t kGoldenT = 0x9e3779b97f4a7c15ULL;
constexpr double kTauAlpha = 12.0;

__device__ __forceinline__ uint64_t round_prefix_t(uint64_t seed, int r) {
  return mix64(mix64(seed ^ 0x2545f4914f6cdd1dULL) + static_cast<uint64_t>(r) * kGoldenT);
}

__device__ __forceinline__ double nlu_exact_t(uint64_t bits) {
  return -log(static_cast<double>((bits >> 11) + 1) * 0x1.0p-53);
}

__device__ __forceinline__ bool better(double c2, long long i2, double c, long long i) {
  return i2 >= 0 && (i < 0 || c2 < c || (c2 == c && i2 < i));
}

__device__ __forceinline__ void st_ll_t(uint2* p, unsigned v, unsigned tag) {
  asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v), "r"(tag)
               : "memory");
}
// six LL words of one slot (three 16-byte loads per attempt)
__device__ __forceinline__ void ld_ll6(const uint2* p, unsigned tag, unsigned (&v)[6]) {
  bool ok;
  do {
    ok = true;
#pragma unroll
    for (int i = 0; i < 6; i += 2) {
      unsigned t0, t1;
      asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[i]), "=r"(t0), "=r"(v[i + 1]), "=r"(t1)
                   : "l"(p + i)
                   : "memory");
      ok = ok && t0 == tag && t1 == tag;
    }
  } while (!ok);
}

__device__ __forceinline__ double dist2_t(const double (&x)[4], const double (&c)[4]) {
  const double e0 = __dsub_rn(x[0], c[0]);
  const double e1 = __dsub_rn(x[1], c[1]);
  const double e2 = __dsub_rn(x[2], c[2]);
  const double e3 = __dsub_rn(x[3], c[3]);
  double s = __dadd_rn(__dmul_rn(e0, e0), __dmul_rn(e1, e1));
  s = __dadd_rn(s, __dmul_rn(e2, e2));
  return __dadd_rn(s, __dmul_rn(e3, e3));
}

// Morton-order working copies + per-tile state (one thread per point)
__global__ void kpp_tile_init_kernel(const double* __restrict__ x64, int64_t n,
                                     const int32_t* __restrict__ perm,
                                     const uint64_t* __restrict__ keys, KppTileScratch ts) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t src = perm[i];
#pragma unroll
  for (int j = 0; j < 4; ++j) ts.xm[j * n + i] = x64[j * n + src];
  ts.mkey[i] = keys[src];
  ts.md2[i] = INFINITY;
  ts.mlab[i] = 0;
}

// per-tile FP64 bounding boxes; Dmax = inf, sum = 0 (one warp per tile)
__global__ void kpp_tile_box_kernel(int64_t n, int ntiles, KppTileScratch ts) {
  const int t = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= ntiles) return;
  double lo[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  double hi[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int q = 0; q < 4; ++q) {
    const int64_t i = static_cast<int64_t>(t) * kTile + lane + 32 * q;
    if (i < n) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double v = ts.xm[j * n + i];
        lo[j] = fmin(lo[j], v);
        hi[j] = fmax(hi[j], v);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      lo[j] = fmin(lo[j], __shfl_xor_sync(0xffffffffu, lo[j], off));
      hi[j] = fmax(hi[j], __shfl_xor_sync(0xffffffffu, hi[j], off));
    }
  }
  if (lane < 4) {
    ts.tbox[static_cast<int64_t>(t) * 8 + lane] = lo[lane];
    ts.tbox[static_cast<int64_t>(t) * 8 + 4 + lane] = hi[lane];
  }
  if (lane == 0) {
    ts.tdmax[t] = INFINITY;
    ts.tsum[t] = 0.0;
  }
}

// labels back to the original order + owned counts (sogmm.cpp:315-318)
__global__ void kpp_tile_scatter_kernel(int64_t n, const int32_t* __restrict__ perm,
                                        const int32_t* __restrict__ mlab,
                                        int32_t* __restrict__ labels, int* __restrict__ owned) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t l = mlab[i];
  labels[perm[i]] = l;
  atomicAdd(&owned[l], 1);
}

// the 32 warps' (clock, index) and sums -> warp 0 (the CTA best / total
// in thread 0)
__device__ __forceinline__ void cta_best(double& bc, long long& bi, double& sm, double* s_c,
                                         long long* s_i, double* s_s, int lane, int warp) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
    const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
    sm += __shfl_xor_sync(0xffffffffu, sm, off);
    if (better(c2, i2, bc, bi)) {
      bc = c2;
      bi = i2;
    }
  }
  if (lane == 0) {
    s_c[warp] = bc;
    s_i[warp] = bi;
    s_s[warp] = sm;
  }
  __syncthreads();
  if (warp == 0) {
    bc = s_c[lane];
    bi = s_i[lane];
    sm = s_s[lane];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
      const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
      sm += __shfl_xor_sync(0xffffffffu, sm, off);
      if (better(c2, i2, bc, bi)) {
        bc = c2;
        bi = i2;
      }
    }
  }
}

// Dynamic shared memory: the CTA's tiles' state (box, largest d2, d2 sum,
// round threshold) for at most kMaxCtaTiles tiles.
constexpr int kMaxCtaTiles = 1024;
struct TileSmem {
  double box[8];
  double dmax;
  double sum;
};

__global__ void __launch_bounds__(kTileKppThreads, 1)
    kpp_tile_kernel(const double* __restrict__ x64, int64_t n, int ntiles, int k, uint64_t seed,
                    KppTileScratch ts, KinitScratch scr, unsigned long long* arrive) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double s_c[kTileKppWarps];
  __shared__ long long s_i[kTileKppWarps];
  __shared__ double s_sum[kTileKppWarps];
  __shared__ double s_gc, s_gsum;
  __shared__ long long s_gi, s_u[kTileKppWarps];
  __shared__ double s_delta[kTileKppWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = gridDim.x;
  const int t0 = static_cast<int>(static_cast<int64_t>(blockIdx.x) * ntiles / nblk);
  const int t1 = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * ntiles / nblk);
  const int nt = t1 - t0;
  TileSmem* tsm = reinterpret_cast<TileSmem*>(smem_raw);
  unsigned* thr = reinterpret_cast<unsigned*>(tsm + kMaxCtaTiles);
  for (int q = tid; q < nt; q += kTileKppThreads) {
#pragma unroll
    for (int j = 0; j < 8; ++j) tsm[q].box[j] = ts.tbox[static_cast<int64_t>(t0 + q) * 8 + j];
    tsm[q].dmax = INFINITY;
    tsm[q].sum = 0.0;
  }
  __syncthreads();
  const double* __restrict__ xm = ts.xm;
  const int64_t p0 = static_cast<int64_t>(t0) * kTile;
  const int64_t p1 = min64(n, static_cast<int64_t>(t1) * kTile);
  double c[4] = {0, 0, 0, 0};
  double cta_sum = 0.0;       // sum of d2 over this CTA's points (finite after round 1)
  double gsum = INFINITY;     // global sum of d2 from the last exchange
  unsigned long long xchg = 0;  // exchanges so far (arrival target, slot parity)
  for (int r = 0; r <= k; ++r) {
    // ---- fold centre r - 1 into the tiles it can reach (box test in shared memory)
    if (r > 0) {
      double delta = 0.0;
      for (int q = warp; q < nt; q += kTileKppWarps) {
        TileSmem& tt = tsm[q];
        double lb = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double g = fmax(fmax(tt.box[j] - c[j], c[j] - tt.box[4 + j]), 0.0);
          lb = fma(g, g, lb);
        }
        if (lb * (1.0 - 1e-12) >= tt.dmax) continue;  // no point of the tile gets closer
        const int t = t0 + q;
        double mx = 0.0, sm = 0.0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int64_t i = static_cast<int64_t>(t) * kTile + lane + 32 * h;
          if (i < n) {
            double x[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = xm[j * n + i];
            const double dd = dist2_t(x, c);
            double d2 = ts.md2[i];
            if (dd < d2) {
              d2 = dd;
              ts.md2[i] = dd;
              ts.mlab[i] = r - 1;
            }
            mx = fmax(mx, d2);
            sm += d2;
          }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          sm += __shfl_xor_sync(0xffffffffu, sm, off);
        }
        if (lane == 0) {
          tt.dmax = mx;
          delta += sm - tt.sum;
          tt.sum = sm;
        }
      }
      if (lane == 0) s_delta[warp] = delta;
      __syncthreads();
      if (tid == 0) {
        for (int w = 0; w < kTileKppWarps; ++w) cta_sum += s_delta[w];
      }
    }
    if (r == k) break;
    // ---- candidates, exact clocks, grid exchange (repeated with a larger tau
    // if the best candidate does not beat tau)
    const uint64_t pre = round_prefix_t(seed, r);
    double tau = r == 0 ? kTauAlpha / static_cast<double>(n)
                        : (isfinite(gsum) && gsum > 0.0 ? kTauAlpha / gsum : INFINITY);
    long long win = -1;
    for (;;) {
      // per-tile thresholds on the top 32 bits of the draw
      for (int q = tid; q < nt; q += kTileKppThreads) {
        const double dmax = r == 0 ? 1.0 : tsm[q].dmax;
        unsigned th = 0xffffffffu;  // dmax == 0: no eligible point (d2 > 0 fails)
        if (dmax > 0.0) {
          const double e = exp(-tau * dmax) * (1.0 - 1e-12);
          th = e > 0.0 ? static_cast<unsigned>(fmin(e * 4294967296.0, 4294967295.0)) : 0u;
        }
        thr[q] = th;
      }
      __syncthreads();
      double bc = INFINITY;
      long long bi = -1;
      // every point of the CTA: one mix64 + one compare on the top 32 bits.
      // Point j = tid + 1024 m of the CTA range lies in tile (tid >> 7) + 8 m
      // (ranges start at a tile boundary); 32-bit offsets, four keys in flight,
      // bounds checks only in the last chunk.
      auto exact = [&](int j, uint64_t bits) {
        const int64_t i = p0 + j;
#ifdef GMMB_KPP_TILE_STATS
        atomicAdd(reinterpret_cast<unsigned long long*>(scr.status + 4), 1ull);
#endif
        const double nl = nlu_exact_t(bits);
        double clk = nl;
        if (r > 0) {
          const double d2 = ts.md2[i];
          if (!(d2 > 0.0)) return;
          clk = nl / d2;
        }
        const long long oi = ts.perm[i];
        if (better(clk, oi, bc, bi)) {
          bc = clk;
          bi = oi;
        }
      };
      {
        const int np = static_cast<int>(p1 - p0);
        const uint64_t* __restrict__ kp = ts.mkey + p0;
        const int q0 = tid >> 7;
        int j = tid, q = q0;
        for (; j + 3 * kTileKppThreads < np; j += 4 * kTileKppThreads, q += 32) {
          uint64_t kv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) kv[u] = __ldg(kp + j + u * kTileKppThreads);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint64_t bits = mix64(pre + kv[u]);
            if (static_cast<unsigned>(bits >> 32) >= thr[q + 8 * u]) exact(j + u * kTileKppThreads, bits);
          }
        }
        for (; j < np; j += kTileKppThreads, q += 8) {
          const uint64_t bits = mix64(pre + __ldg(kp + j));
          if (static_cast<unsigned>(bits >> 32) >= thr[q]) exact(j, bits);
        }
      }
      double unused = 0.0;
      cta_best(bc, bi, unused, s_c, s_i, s_sum, lane, warp);
      // LL exchange (warp 0): the CTA's (clock, index, sum d2) as six 8-byte
      // (payload, tag) words, each single-copy atomic, so no fence or arrival
      // counter; every CTA polls every slot (lanes over slots, three 16-byte
      // loads per slot per attempt) and reduces. Slot sets alternate by
      // exchange parity: a CTA cannot publish exchange x + 2 before every CTA
      // has published x + 1, i.e. finished reading x.
      if (warp == 0) {
        const unsigned tag = static_cast<unsigned>(xchg) + 1u;
        uint2* base = reinterpret_cast<uint2*>(scr.slots) + static_cast<size_t>(xchg & 1) * nblk * 8;
        const double csum = __shfl_sync(0xffffffffu, cta_sum, 0);
        bc = __shfl_sync(0xffffffffu, bc, 0);
        bi = __shfl_sync(0xffffffffu, bi, 0);
        if (lane < 6) {
          const unsigned long long w[3] = {static_cast<unsigned long long>(__double_as_longlong(bc)),
                                           static_cast<unsigned long long>(bi),
                                           static_cast<unsigned long long>(__double_as_longlong(csum))};
          const unsigned long long v = w[lane >> 1];
          st_ll_t(base + blockIdx.x * 8 + lane, (lane & 1) ? static_cast<unsigned>(v >> 32)
                                                         : static_cast<unsigned>(v), tag);
        }
        double gc = INFINITY, gs = 0.0;
        long long gi = -1;
        for (int b = lane; b < nblk; b += 32) {
          unsigned v[6];
          ld_ll6(base + b * 8, tag, v);
          const double c2 = __longlong_as_double(static_cast<long long>(
              (static_cast<unsigned long long>(v[1]) << 32) | v[0]));
          const long long i2 = static_cast<long long>((static_cast<unsigned long long>(v[3]) << 32) | v[2]);
          gs += __longlong_as_double(static_cast<long long>(
              (static_cast<unsigned long long>(v[5]) << 32) | v[4]));
          if (better(c2, i2, gc, gi)) {
            gc = c2;
            gi = i2;
          }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          const double c2 = __shfl_xor_sync(0xffffffffu, gc, off);
          const long long i2 = __shfl_xor_sync(0xffffffffu, gi, off);
          gs += __shfl_xor_sync(0xffffffffu, gs, off);
          if (better(c2, i2, gc, gi)) {
            gc = c2;
            gi = i2;
          }
        }
        if (lane == 0) {
          s_gc = gc;
          s_gi = gi;
          s_gsum = gs;
        }
      }
      __syncthreads();
      ++xchg;
      const double gc = s_gc;
      const long long gi = s_gi;
      if (r > 0) gsum = s_gsum;
      if (gi >= 0 && gc < tau * (1.0 - 1e-12)) {
        win = gi;
        break;
      }
      if (tau == INFINITY) break;  // no point with d2 > 0 anywhere
      tau = tau * 64.0 > 1e300 ? INFINITY : tau * 64.0;
      if (xchg > 64ull * (k + 1)) tau = INFINITY;  // (cannot happen; bounded anyway)
    }
    if (win < 0) {
      // sogmm.cpp:276-284: the lowest unchosen index, among 0 .. r (CTA 0
      // fenced its centre stores before publishing later exchanges)
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      long long lo = LLONG_MAX;
      for (long long cnd = tid; cnd <= r && cnd < n; cnd += kTileKppThreads) {
        bool taken = false;
        for (int q = 0; q < r && !taken; ++q) taken = __ldcg(scr.centers + q) == cnd;
        if (!taken && cnd < lo) lo = cnd;
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const long long u2 = __shfl_xor_sync(0xffffffffu, lo, off);
        lo = u2 < lo ? u2 : lo;
      }
      if (lane == 0) s_u[warp] = lo;
      __syncthreads();
      if (tid == 0) {
        for (int q = 0; q < kTileKppWarps; ++q) lo = s_u[q] < lo ? s_u[q] : lo;
        s_gi = lo;
      }
      __syncthreads();
      win = s_gi;
    }
    if (blockIdx.x == 0 && tid == 0) {
      scr.centers[r] = win;
      __threadfence();
      if (r == k - 1) *reinterpret_cast<unsigned long long*>(scr.status + 2) = xchg;  // diagnostics
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = x64[j * n + win];
    __syncthreads();  // shared words reused next round
  }
}

}  // namespace

bool kpp_tile_wanted(int64_t n, int sm_count) {
  // the shared-memory-resident kernel holds up to ~365k points (148 SMs);
  // a CTA keeps at most kMaxCtaTiles tiles' state (19M points on 148 SMs;
  // beyond: the memory-resident rounds)
  return n > static_cast<int64_t>(sm_count) * 2400 &&
         n <= static_cast<int64_t>(sm_count) * kMaxCtaTiles * kTile;
}

cudaError_t launch_kpp_tile(const double* x64, int64_t n, int ntiles, const int32_t* perm,
                            int k, uint64_t seed, KinitScratch scr, KppTileScratch ts,
                            int sm_count, cudaStream_t s) {
  const int grid = static_cast<int>((n + 255) / 256);
  ts.perm = perm;
  kpp_tile_init_kernel<<<grid, 256, 0, s>>>(x64, n, perm, scr.keys, ts);
  kpp_tile_box_kernel<<<(ntiles + 7) / 8, 256, 0, s>>>(n, ntiles, ts);
  unsigned long long* arrive = reinterpret_cast<unsigned long long*>(scr.status + 6);
  // LL tags start from zero (two slot sets of 64 bytes per CTA)
  cudaError_t e = cudaMemsetAsync(scr.slots, 0, sizeof(KppSlot) * 2 * sm_count, s);
  if (e != cudaSuccess) return e;
  int nblk = sm_count;  // one CTA per SM
  if (nblk > ntiles) nblk = ntiles;
  if ((ntiles + nblk - 1) / nblk > kMaxCtaTiles) return cudaErrorInvalidValue;
  const size_t smem = sizeof(TileSmem) * kMaxCtaTiles + sizeof(unsigned) * kMaxCtaTiles;
  e = cudaFuncSetAttribute(kpp_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kpp_tile_kernel, kTileKppThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  void* args[] = {(void*)&x64, (void*)&n, (void*)&ntiles, (void*)&k, (void*)&seed,
                  (void*)&ts, (void*)&scr, (void*)&arrive};
  e = cudaLaunchCooperativeKernel((const void*)kpp_tile_kernel, dim3(nblk), dim3(kTileKppThreads),
                                  args, smem, s);
  if (e != cudaSuccess) return e;
  kpp_tile_scatter_kernel<<<grid, 256, 0, s>>>(n, perm, ts.mlab, scr.labels, scr.owned);
  return cudaGetLastError();
}

}  // namespace gmmb
