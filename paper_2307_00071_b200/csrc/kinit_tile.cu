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
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

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

// the top 32 bits of mix64(z) (the candidate test) without the low half of
// the last product: hi32(z2 * C2) = umulhi(lo, C2lo) + lo C2hi + hi C2lo
// (mod 2^32), then hi ^ (hi >> 31) (z ^ (z >> 31) restricted to the top
// word). Equal to static_cast<unsigned>(mix64(z) >> 32) for every z.
__device__ __forceinline__ unsigned mix64_hi32(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = z ^ (z >> 27);
  const unsigned lo = static_cast<unsigned>(z), hi = static_cast<unsigned>(z >> 32);
  const unsigned h = __umulhi(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
  return h ^ (h >> 31);
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


// Every slot of the exchange (4 LL words: clock, index, FP32 sum of d2):
// lane l owns slots l, l + 32, ... (up to 5); each attempt issues the
// 16-byte loads of all its not-yet-seen slots back to back and checks every
// tag (one L2 round trip per attempt, not one per slot).
constexpr int kPollSlots = 5;  // nblk <= 160 (one CTA per SM)
__device__ __forceinline__ void poll_slots(const uint2* base, unsigned tag, int nblk, int lane,
                                           double& gc, long long& gi, double& gs) {
  unsigned v[kPollSlots][4];
  unsigned pending = 0;
#pragma unroll
  for (int q = 0; q < kPollSlots; ++q)
    if (lane + 32 * q < nblk) pending |= 1u << q;
  while (pending) {
#pragma unroll
    for (int q = 0; q < kPollSlots; ++q) {
      if (!((pending >> q) & 1u)) continue;
      const uint2* p = base + (lane + 32 * q) * 8;
      bool ok = true;
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        unsigned t0, t1;
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[q][i]), "=r"(t0), "=r"(v[q][i + 1]), "=r"(t1)
                     : "l"(p + i)
                     : "memory");
        ok = ok && t0 == tag && t1 == tag;
      }
      if (ok) pending &= ~(1u << q);
    }
    // (no __nanosleep between attempts: it sleeps far longer than asked on B200)
  }
#pragma unroll
  for (int q = 0; q < kPollSlots; ++q) {
    if (lane + 32 * q >= nblk) continue;
    const double c2 = __longlong_as_double(
        static_cast<long long>((static_cast<unsigned long long>(v[q][1]) << 32) | v[q][0]));
    const long long i2 = static_cast<long long>(static_cast<int>(v[q][2]));
    gs += static_cast<double>(__uint_as_float(v[q][3]));
    if (better(c2, i2, gc, gi)) {
      gc = c2;
      gi = i2;
    }
  }
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
        if (lane < 4) {  // slot: clock (2 words), index, sum of d2 (FP32)
          const unsigned long long cb = static_cast<unsigned long long>(__double_as_longlong(bc));
          const unsigned w = lane == 0 ? static_cast<unsigned>(cb)
                           : lane == 1 ? static_cast<unsigned>(cb >> 32)
                           : lane == 2 ? static_cast<unsigned>(static_cast<int>(bi))
                                       : __float_as_uint(static_cast<float>(csum));
          st_ll_t(base + blockIdx.x * 8 + lane, w, tag);
        }
        double gc = INFINITY, gs = 0.0;
        long long gi = -1;
        poll_slots(base, tag, nblk, lane, gc, gi, gs);
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


// ---------------------------------------------------------------------------
// Warp-specialised variant: warp 0 runs the grid exchange of round r while
// warps 1..31 already draw round r + 1 for every point and keep its
// candidates (speculative: thresholds from the tiles' largest d2 BEFORE
// centre r is folded, which can only be larger than after, and tau from the
// last known sum of d2), so the draws hide behind the exchange. After the
// exchange the compute warps fold centre r and evaluate only the kept
// candidates; the exact-winner test (best clock < tau) is unchanged.
// Rounds 0 and 1, and a round whose test fails, are drawn synchronously.
// ---------------------------------------------------------------------------
#ifdef GMMB_KPP_TPROF
// per exchange (first 4096) and CTA: publish time, all-slots-seen time, and
// the compute warps' draw-done time (ns, globaltimer)
__device__ unsigned long long g_tprof[6][4096][160];  // + round start, fold end, nfold
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
constexpr int kWsCompute = kTileKppThreads - 32;  // compute threads (warps 1..31)
constexpr int kWsCWarps = kWsCompute / 32;
constexpr int kCandCap = 1024;                    // kept candidates per CTA and round
constexpr double kSpecAlpha = 16.0;

// Dynamic shared memory of the warp-specialised kernel, for mt tiles per CTA:
// tile state | thresholds | fold list | kept candidates | as many of the
// CTA's keys as fit (the rest stay in global memory). Keeping the keys
// on-chip takes the per-round stream of draws off L2, where it would slow
// the grid exchange it runs beside.
struct WsLayout {
  TileSmem* tsm;
  unsigned* thr;
  int* fold;
  int* cand_j;
  double* cand_nl;   // -ln u (FP64, as the reference)
  uint64_t* keys;
};
__host__ __device__ inline size_t ws_fixed_bytes(int mt) {
  return (sizeof(TileSmem) * mt + sizeof(unsigned) * mt + sizeof(int) * mt + 15) / 16 * 16 +
         (sizeof(int) + sizeof(double)) * kCandCap;
}
__device__ inline WsLayout ws_layout(unsigned char* base, int mt) {
  WsLayout l;
  l.tsm = reinterpret_cast<TileSmem*>(base);
  l.thr = reinterpret_cast<unsigned*>(l.tsm + mt);
  l.fold = reinterpret_cast<int*>(l.thr + mt);
  unsigned char* q = base + (sizeof(TileSmem) * mt + sizeof(unsigned) * mt + sizeof(int) * mt + 15) / 16 * 16;
  l.cand_nl = reinterpret_cast<double*>(q);
  l.cand_j = reinterpret_cast<int*>(l.cand_nl + kCandCap);
  l.keys = reinterpret_cast<uint64_t*>(base + ws_fixed_bytes(mt));
  return l;
}

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(kTileKppThreads, 1)
    kpp_tile_ws_kernel(const double* __restrict__ x64, int64_t n, int ntiles, int k, uint64_t seed,
                       KppTileScratch ts, KinitScratch scr, int mt, int kcache) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const WsLayout sm = ws_layout(smem_raw, mt);
  __shared__ double s_bc[kWsCWarps];
  __shared__ long long s_bi[kWsCWarps];
  __shared__ double s_delta[kWsCWarps];
  __shared__ double s_cta_sum, s_tau, s_gsum;
  __shared__ long long s_win;
  __shared__ int s_nfold, s_ncand, s_cover;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = gridDim.x;
  // CTA b owns tiles b, b + nblk, b + 2 nblk, ...: a new centre's
  // neighbourhood (consecutive Morton tiles) is folded by many CTAs, not one
  const int b0 = blockIdx.x;
  const int nt = ntiles > b0 ? (ntiles - 1 - b0) / nblk + 1 : 0;
  auto gtile = [&](int q) { return b0 + q * nblk; };
  for (int q = tid; q < nt; q += kTileKppThreads) {
#pragma unroll
    for (int j = 0; j < 8; ++j) sm.tsm[q].box[j] = ts.tbox[static_cast<int64_t>(gtile(q)) * 8 + j];
    sm.tsm[q].dmax = INFINITY;
    sm.tsm[q].sum = 0.0;
  }
  if (tid == 0) {
    s_nfold = 0;
    s_ncand = 0;
    s_cover = 0;
    s_cta_sum = 0.0;
  }
  // CTA point j: offset j % 128 of tile j / 128 (the last tile may be short)
  auto gidx = [&](int j) -> int64_t {
    return static_cast<int64_t>(gtile(j >> 7)) * kTile + (j & (kTile - 1));
  };
  const int np = nt * kTile;
  const int ncache = np < kcache ? np : kcache;
  for (int j = tid; j < ncache; j += kTileKppThreads) {
    const int64_t i = gidx(j);
    sm.keys[j] = i < n ? ts.mkey[i] : 0ull;
  }
  __syncthreads();

  if (warp == 0) {
    // ======================= communication warp =======================
    unsigned xchg = 0;
    for (int r = 0; r < k;) {
      bar_sync(2, kTileKppThreads);  // the compute warps' bests of this attempt
      double bc = INFINITY;
      long long bi = -1;
      if (lane < kWsCWarps) {
        bc = s_bc[lane];
        bi = s_bi[lane];
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
        const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
        if (better(c2, i2, bc, bi)) {
          bc = c2;
          bi = i2;
        }
      }
      const double tau = s_tau;
      const double csum = s_cta_sum;
      const unsigned tag = xchg + 1u;
#ifdef GMMB_KPP_TPROF
      if (lane == 0 && xchg < 4096 && blockIdx.x < 160) g_tprof[0][xchg][blockIdx.x] = gtime();
#endif
      uint2* base = reinterpret_cast<uint2*>(scr.slots) + static_cast<size_t>(xchg & 1) * nblk * 8;
      if (lane < 4) {  // slot: clock (2 words), index, sum of d2 (FP32)
        const unsigned long long cb = static_cast<unsigned long long>(__double_as_longlong(bc));
        const unsigned w = lane == 0 ? static_cast<unsigned>(cb)
                         : lane == 1 ? static_cast<unsigned>(cb >> 32)
                         : lane == 2 ? static_cast<unsigned>(static_cast<int>(bi))
                                     : __float_as_uint(static_cast<float>(csum));
        st_ll_t(base + blockIdx.x * 8 + lane, w, tag);
      }
      double gc = INFINITY, gs = 0.0;
      long long gi = -1;
      poll_slots(base, tag, nblk, lane, gc, gi, gs);
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
#ifdef GMMB_KPP_TPROF
      if (lane == 0 && xchg < 4096 && blockIdx.x < 160) g_tprof[1][xchg][blockIdx.x] = gtime();
#endif
      ++xchg;
      long long win = -1;
      if (gi >= 0 && gc < tau * (1.0 - 1e-12)) {
        win = gi;
      } else if (tau == INFINITY) {
        // sogmm.cpp:276-284: no point with d2 > 0: the lowest unchosen
        // index among 0 .. r (CTA 0 fenced its centre stores)
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        long long lo = LLONG_MAX;
        for (long long cnd = lane; cnd <= r && cnd < n; cnd += 32) {
          bool taken = false;
          for (int q = 0; q < r && !taken; ++q) taken = __ldcg(scr.centers + q) == cnd;
          if (!taken && cnd < lo) lo = cnd;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          const long long u2 = __shfl_xor_sync(0xffffffffu, lo, off);
          lo = u2 < lo ? u2 : lo;
        }
        win = lo;
      }
      if (lane == 0) {
        s_win = win;  // -1: repeat the round with a larger tau
        s_gsum = gs;
        if (win >= 0 && blockIdx.x == 0) {
          scr.centers[r] = win;
          __threadfence();
          if (r == k - 1) *reinterpret_cast<unsigned long long*>(scr.status + 2) = xchg;
        }
      }
      __syncwarp();
      bar_arrive(3, kTileKppThreads);
      if (win >= 0) ++r;
    }
    return;
  }

  // ========================= compute warps =========================
  const int ct = tid - 32, cw = warp - 1;
  const uint64_t* __restrict__ kp = ts.mkey;
  double c[4] = {0, 0, 0, 0};
  double gsum = INFINITY;   // last known global sum of d2
  double cta_sum = 0.0;     // (ct == 0)
  bool spec = false;        // candidates of this round were kept during the last exchange
  double tau_kept = 0.0;    // the tau they were drawn with
  // best (clock, index) of this thread over the candidates it evaluates
  double bc;
  long long bi;
  auto eval = [&](int j, uint64_t bits, int r) {
    const int64_t i = gidx(j);
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
  // a kept candidate of round r >= 2: its -ln u was computed while drawing
  auto eval_nl = [&](int j, double nl) {
    const int64_t i = gidx(j);
    const double d2 = ts.md2[i];
    if (!(d2 > 0.0)) return;
    const double clk = nl / d2;
    const long long oi = ts.perm[i];
    if (better(clk, oi, bc, bi)) {
      bc = clk;
      bi = oi;
    }
  };
  // per-tile thresholds on the draw's top 32 bits for (tau, r)
  auto thresholds = [&](double tau, int r) {
    for (int q = ct; q < nt; q += kWsCompute) {
      const double dmax = r == 0 ? 1.0 : sm.tsm[q].dmax;
      unsigned th = 0xffffffffu;
      if (dmax > 0.0) {
        const double e = exp(-tau * dmax) * (1.0 - 1e-12);
        th = e > 0.0 ? static_cast<unsigned>(fmin(e * 4294967296.0, 4294967295.0)) : 0u;
      }
      sm.thr[q] = th;
    }
    bar_sync(1, kWsCompute);
  };
  // draw round r for every point: KEEP = 0 evaluates the candidates, 1 keeps them
  // draw round r for every point. keep = false (rounds drawn after their
  // exchange: 0, 1, 2, repeats): candidates are evaluated on the spot.
  // keep = true (the next round, behind the exchange): a warp per tile, the
  // tile's threshold uniform, four points per lane; the rare candidates are
  // only appended to the kept list (draw bits), their -ln u comes after.
  auto draw = [&](int r, bool keep) {
    const uint64_t pre = round_prefix_t(seed, r);
    if (keep) {
      for (int q = cw; q < nt; q += kWsCWarps) {
        const unsigned th = sm.thr[q];
        const int jb = q * kTile;
        uint64_t kv[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int jj = jb + lane + 32 * h;
          kv[h] = jj < ncache ? sm.keys[jj] : 0ull;
        }
        if (jb + kTile > ncache) {  // keys beyond the on-chip cache
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int jj = jb + lane + 32 * h;
            const int64_t ii = gidx(jj);
            if (jj >= ncache && ii < n) kv[h] = __ldg(kp + ii);
          }
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const uint64_t bits = mix64(pre + kv[h]);
          if (static_cast<unsigned>(bits >> 32) >= th) {
            const int jj = jb + lane + 32 * h;
            if (gidx(jj) < n) {
              const int slot = atomicAdd(&s_ncand, 1);
              if (slot < kCandCap) {
                sm.cand_j[slot] = jj;
                sm.cand_nl[slot] = __longlong_as_double(static_cast<long long>(bits));
              } else {
                s_cover = 1;
              }
            }
          }
        }
      }
      bar_sync(1, kWsCompute);
      const int nc = s_ncand < kCandCap ? s_ncand : kCandCap;
      for (int q = ct; q < nc; q += kWsCompute)
        sm.cand_nl[q] = nlu_exact_t(static_cast<uint64_t>(__double_as_longlong(sm.cand_nl[q])));
      return;
    }
    for (int j = ct; j < np; j += kWsCompute) {
      const int64_t ii = gidx(j);
      if (ii >= n) continue;
      const uint64_t bits = mix64(pre + (j < ncache ? sm.keys[j] : __ldg(kp + ii)));
      if (static_cast<unsigned>(bits >> 32) >= sm.thr[j >> 7]) eval(j, bits, r);
    }
  };
  auto publish_best = [&](double tau) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
      const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
      if (better(c2, i2, bc, bi)) {
        bc = c2;
        bi = i2;
      }
    }
    if (lane == 0) {
      s_bc[cw] = bc;
      s_bi[cw] = bi;
    }
    if (ct == 0) {
      s_tau = tau;
      s_cta_sum = cta_sum;
    }
    bar_arrive(2, kTileKppThreads);
  };

  for (int r = 0; r <= k; ++r) {
#ifdef GMMB_KPP_TPROF
    if (ct == 0 && r < 4096 && blockIdx.x < 160) g_tprof[3][r][blockIdx.x] = gtime();
#endif
    // ---- fold centre r - 1: box tests by threads, listed tiles by warps
    if (r > 0) {
      for (int q = ct; q < nt; q += kWsCompute) {
        const TileSmem& tt = sm.tsm[q];
        double lb = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double g = fmax(fmax(tt.box[j] - c[j], c[j] - tt.box[4 + j]), 0.0);
          lb = fma(g, g, lb);
        }
        if (!(lb * (1.0 - 1e-12) >= tt.dmax)) sm.fold[atomicAdd(&s_nfold, 1)] = q;
      }
      bar_sync(1, kWsCompute);
      const int nf = s_nfold;
      double delta = 0.0;
      for (int f = cw; f < nf; f += kWsCWarps) {
        const int q = sm.fold[f];
        TileSmem& tt = sm.tsm[q];
        const int64_t ib = static_cast<int64_t>(gtile(q)) * kTile;
        double mx = 0.0, smv = 0.0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int64_t i = ib + lane + 32 * h;
          if (i < n) {
            double x[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = ts.xm[j * n + i];
            const double dd = dist2_t(x, c);
            double d2 = ts.md2[i];
            if (dd < d2) {
              d2 = dd;
              ts.md2[i] = dd;
              ts.mlab[i] = r - 1;
            }
            mx = fmax(mx, d2);
            smv += d2;
          }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          smv += __shfl_xor_sync(0xffffffffu, smv, off);
        }
        if (lane == 0) {
          tt.dmax = mx;
          delta += smv - tt.sum;
          tt.sum = smv;
        }
      }
      if (lane == 0) s_delta[cw] = delta;
      bar_sync(1, kWsCompute);
      if (ct == 0) {
        for (int w = 0; w < kWsCWarps; ++w) cta_sum += s_delta[w];
#ifdef GMMB_KPP_TPROF
        if (r < 4096 && blockIdx.x < 160) {
          g_tprof[4][r][blockIdx.x] = gtime();
          g_tprof[5][r][blockIdx.x] = s_nfold;
        }
#endif
        s_nfold = 0;
      }
    }
    if (r == k) break;
    // ---- round r: evaluate the kept candidates, or draw now
    double tau = r == 0 ? kTauAlpha / static_cast<double>(n)
                        : (isfinite(gsum) && gsum > 0.0 ? kTauAlpha / gsum : INFINITY);
    bool first = true;
    bool spec_next = false;
    double tau_next = 0.0;
    for (;;) {
      bc = INFINITY;
      bi = -1;
      if (first && spec) {
        tau = tau_kept;  // the kept candidates were drawn with it
        const int nc = s_ncand;
        for (int q = ct; q < nc; q += kWsCompute) eval_nl(sm.cand_j[q], sm.cand_nl[q]);
      } else {
        thresholds(tau, r);
        draw(r, false);
      }
      publish_best(tau);
      // ---- meanwhile: keep round r + 1's candidates (first attempt only)
      bool kept = false;
      if (first && r + 1 < k && r >= 1 && isfinite(gsum) && gsum > 0.0) {
        bar_sync(1, kWsCompute);  // kept list consumed; s_tau published
        if (ct == 0) {
          s_ncand = 0;
          s_cover = 0;
        }
        tau_next = kSpecAlpha / gsum;
        thresholds(tau_next, r + 1);  // (its barrier orders the reset before the draws)
        draw(r + 1, true);
        kept = true;
#ifdef GMMB_KPP_TPROF
        bar_sync(1, kWsCompute);
        if (ct == 0 && r < 4096 && blockIdx.x < 160) g_tprof[2][r][blockIdx.x] = gtime();
#endif
      }
      bar_sync(3, kTileKppThreads);  // the exchange result (and every kept candidate)
      const long long win = s_win;
      gsum = s_gsum;
      if (kept) spec_next = s_cover == 0;
      if (win >= 0) {
        spec = spec_next;
        tau_kept = tau_next;
#pragma unroll
        for (int j = 0; j < 4; ++j) c[j] = x64[j * n + win];
        break;
      }
      first = false;
      tau = tau * 64.0 > 1e300 ? INFINITY : tau * 64.0;
    }
  }
}
// ---------------------------------------------------------------------------
// Two rounds per exchange (kpp_tile_ws2_kernel). The kept candidates of
// round r + 1 are evaluated in the same epoch as round r, with the d2 from
// before centre c_r is folded (speculative clocks); the exchange decides c_r
// as above and, from the speculative argmin s of round r + 1, c_{r+1} = s iff
// (a) its clock is below the tau its candidates were kept with (no other
// point's speculative clock can be smaller), and (b) c_r leaves its d2
// unchanged (exact FP64 test, the fold's strict <): every other point's true
// clock of round r + 1 can only be larger than its speculative one, since
// folding a centre only lowers d2. Otherwise round r + 1 runs again in the
// next epoch from the same kept list (still a superset: its thresholds came
// from a larger d2). The kept lists live in a ring by round (r % 4); during
// each exchange the compute warps draw the missing lists of the next rounds
// (two per exchange in the steady state), so the draws, not the exchange,
// now bound the epoch, and one exchange decides two centres.
// ---------------------------------------------------------------------------
constexpr int kW2Cap = 128;        // kept candidates per list and CTA (more: the list is not used)
constexpr int kW2Lists = 4;        // ring of kept lists (round % 4)
constexpr int kW2SlotWords = 16;   // LL words per CTA slot (10 used)

struct Ws2Layout {
  TileSmem* tsm;
  unsigned* thr;
  unsigned* thr2;  // a second round's thresholds (two lists drawn in one pass)
  int* fold;
  int* cand_j;       // [kW2Lists][kW2Cap]
  double* cand_nl;   // [kW2Lists][kW2Cap] -ln u (FP64, as the reference)
  uint64_t* keys;
};
__host__ __device__ inline size_t ws2_fixed_bytes(int mt) {
  return (sizeof(TileSmem) * mt + 2 * sizeof(unsigned) * mt + sizeof(int) * mt + 15) / 16 * 16 +
         (sizeof(int) + sizeof(double)) * kW2Lists * kW2Cap;
}
__device__ inline Ws2Layout ws2_layout(unsigned char* base, int mt) {
  Ws2Layout l;
  l.tsm = reinterpret_cast<TileSmem*>(base);
  l.thr = reinterpret_cast<unsigned*>(l.tsm + mt);
  l.thr2 = l.thr + mt;
  l.fold = reinterpret_cast<int*>(l.thr2 + mt);
  unsigned char* q = base + (sizeof(TileSmem) * mt + 2 * sizeof(unsigned) * mt + sizeof(int) * mt + 15) / 16 * 16;
  l.cand_nl = reinterpret_cast<double*>(q);
  l.cand_j = reinterpret_cast<int*>(l.cand_nl + kW2Lists * kW2Cap);
  l.keys = reinterpret_cast<uint64_t*>(base + ws2_fixed_bytes(mt));
  return l;
}

// the CTA slots of one exchange: level 0 (clock, index, sum of d2) and
// level 1 (clock, index, the best's FP64 d2). A slot is folded into the
// lane's bests as soon as its tags check ((clock, index) is a total order, so
// the minima do not depend on arrival order); its sum goes to psum[slot],
// summed in slot order afterwards.
__device__ __forceinline__ void poll_slots2(const uint2* base, unsigned tag, int nblk, int lane,
                                            double& gc0, long long& gi0, float* psum, double& gc1,
                                            long long& gi1, double& gd1) {
  unsigned pending = 0;
#pragma unroll
  for (int q = 0; q < kPollSlots; ++q)
    if (lane + 32 * q < nblk) pending |= 1u << q;
  while (pending) {
    // the loads of every unseen slot go out back to back: which slots to read
    // is fixed before the attempt (a predicate on the previous slot's tags
    // would serialise one L2 round trip per slot)
    const unsigned pend0 = pending;
#pragma unroll
    for (int q = 0; q < kPollSlots; ++q) {
      if (!((pend0 >> q) & 1u)) continue;
      const uint2* p = base + (lane + 32 * q) * kW2SlotWords;
      unsigned v[10];
      bool ok = true;
#pragma unroll
      for (int i = 0; i < 10; i += 2) {
        unsigned t0, t1;
        asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[i]), "=r"(t0), "=r"(v[i + 1]), "=r"(t1)
                     : "l"(p + i)
                     : "memory");
        ok = ok && t0 == tag && t1 == tag;
      }
      if (!ok) continue;
      pending &= ~(1u << q);
      const double c0 = __longlong_as_double(
          static_cast<long long>((static_cast<unsigned long long>(v[1]) << 32) | v[0]));
      const long long i0 = static_cast<long long>(static_cast<int>(v[2]));
      psum[lane + 32 * q] = __uint_as_float(v[3]);
      if (better(c0, i0, gc0, gi0)) {
        gc0 = c0;
        gi0 = i0;
      }
      const double c1 = __longlong_as_double(
          static_cast<long long>((static_cast<unsigned long long>(v[5]) << 32) | v[4]));
      const long long i1 = static_cast<long long>(static_cast<int>(v[6]));
      const double d1 = __longlong_as_double(
          static_cast<long long>((static_cast<unsigned long long>(v[8]) << 32) | v[7]));
      if (better(c1, i1, gc1, gi1)) {
        gc1 = c1;
        gi1 = i1;
        gd1 = d1;
      }
    }
    // (no __nanosleep between attempts: even 32 ns sleeps far longer on
    // B200; with it the cfg4 seeding took 21.7 ms instead of 20.2)
  }
}

__global__ void __launch_bounds__(kTileKppThreads, 1)
    kpp_tile_ws2_kernel(const double* __restrict__ x64, int64_t n, int ntiles, int k, uint64_t seed,
                        KppTileScratch ts, KinitScratch scr, int mt, int kcache) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Ws2Layout sm = ws2_layout(smem_raw, mt);
  __shared__ double s_bc[2][kWsCWarps];
  __shared__ long long s_bi[2][kWsCWarps];
  __shared__ double s_bd[kWsCWarps];
  __shared__ double s_delta[kWsCWarps];
  __shared__ double s_cta_sum, s_tau[2], s_gsum;
  __shared__ long long s_win[2];
  __shared__ int s_r, s_mode, s_nfold;
  __shared__ int s_lround[kW2Lists], s_lcount[kW2Lists], s_lcover[kW2Lists];
  __shared__ float s_psum[32 * kPollSlots];
  __shared__ double s_ltau[kW2Lists];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = gridDim.x;
  const int b0 = blockIdx.x;
  const int nt = ntiles > b0 ? (ntiles - 1 - b0) / nblk + 1 : 0;
  auto gtile = [&](int q) { return b0 + q * nblk; };
  for (int q = tid; q < nt; q += kTileKppThreads) {
#pragma unroll
    for (int j = 0; j < 8; ++j) sm.tsm[q].box[j] = ts.tbox[static_cast<int64_t>(gtile(q)) * 8 + j];
    sm.tsm[q].dmax = INFINITY;
    sm.tsm[q].sum = 0.0;
  }
  if (tid < kW2Lists) {
    s_lround[tid] = -1;
    s_lcount[tid] = 0;
    s_lcover[tid] = 0;
    s_ltau[tid] = 0.0;
  }
  if (tid == 0) {
    s_nfold = 0;
    s_cta_sum = 0.0;
  }
  auto gidx = [&](int j) -> int64_t {
    return static_cast<int64_t>(gtile(j >> 7)) * kTile + (j & (kTile - 1));
  };
  const int np = nt * kTile;
  const int ncache = np < kcache ? np : kcache;
  for (int j = tid; j < ncache; j += kTileKppThreads) {
    const int64_t i = gidx(j);
    sm.keys[j] = i < n ? ts.mkey[i] : 0ull;
  }
  __syncthreads();

  if (warp == 0) {
    // ======================= communication warp =======================
    unsigned xchg = 0;
    for (;;) {
      bar_sync(2, kTileKppThreads);  // the compute warps' bests of this epoch
      const int r = s_r;
      if (r >= k) break;
      const int mode = s_mode;
      double c0 = INFINITY, c1 = INFINITY, d1 = 0.0;
      long long i0 = -1, i1 = -1;
      if (lane < kWsCWarps) {
        c0 = s_bc[0][lane];
        i0 = s_bi[0][lane];
        c1 = s_bc[1][lane];
        i1 = s_bi[1][lane];
        d1 = s_bd[lane];
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const double a0 = __shfl_xor_sync(0xffffffffu, c0, off);
        const long long j0 = __shfl_xor_sync(0xffffffffu, i0, off);
        const double a1 = __shfl_xor_sync(0xffffffffu, c1, off);
        const long long j1 = __shfl_xor_sync(0xffffffffu, i1, off);
        const double e1 = __shfl_xor_sync(0xffffffffu, d1, off);
        if (better(a0, j0, c0, i0)) {
          c0 = a0;
          i0 = j0;
        }
        if (better(a1, j1, c1, i1)) {
          c1 = a1;
          i1 = j1;
          d1 = e1;
        }
      }
      const double tau0 = s_tau[0], tau1 = s_tau[1];
      const double csum = s_cta_sum;
      const unsigned tag = xchg + 1u;
      uint2* base = reinterpret_cast<uint2*>(scr.slots) + static_cast<size_t>(xchg & 1) * nblk * kW2SlotWords;
#ifdef GMMB_KPP_TPROF
      if (lane == 0 && xchg < 4096 && blockIdx.x < 160) g_tprof[0][xchg][blockIdx.x] = gtime();
#endif
      if (lane < 10) {
        const unsigned long long b0w = static_cast<unsigned long long>(__double_as_longlong(c0));
        const unsigned long long b1w = static_cast<unsigned long long>(__double_as_longlong(c1));
        const unsigned long long dw = static_cast<unsigned long long>(__double_as_longlong(d1));
        unsigned w = 0u;
        w = lane == 0 ? static_cast<unsigned>(b0w) : w;
        w = lane == 1 ? static_cast<unsigned>(b0w >> 32) : w;
        w = lane == 2 ? static_cast<unsigned>(static_cast<int>(i0)) : w;
        w = lane == 3 ? __float_as_uint(static_cast<float>(csum)) : w;
        w = lane == 4 ? static_cast<unsigned>(b1w) : w;
        w = lane == 5 ? static_cast<unsigned>(b1w >> 32) : w;
        w = lane == 6 ? static_cast<unsigned>(static_cast<int>(i1)) : w;
        w = lane == 7 ? static_cast<unsigned>(dw) : w;
        w = lane == 8 ? static_cast<unsigned>(dw >> 32) : w;
        st_ll_t(base + blockIdx.x * kW2SlotWords + lane, w, tag);
      }
      double gc0 = INFINITY, gc1 = INFINITY, gd1 = 0.0;
      long long gi0 = -1, gi1 = -1;
      poll_slots2(base, tag, nblk, lane, gc0, gi0, s_psum, gc1, gi1, gd1);
      __syncwarp();
#ifdef GMMB_KPP_TPROF
      if (lane == 0 && xchg < 4096 && blockIdx.x < 160) g_tprof[1][xchg][blockIdx.x] = gtime();
#endif
      double gs = 0.0;  // the CTAs' d2 sums in a fixed order
      for (int q = lane; q < nblk; q += 32) gs += static_cast<double>(s_psum[q]);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const double a0 = __shfl_xor_sync(0xffffffffu, gc0, off);
        const long long j0 = __shfl_xor_sync(0xffffffffu, gi0, off);
        const double a1 = __shfl_xor_sync(0xffffffffu, gc1, off);
        const long long j1 = __shfl_xor_sync(0xffffffffu, gi1, off);
        const double e1 = __shfl_xor_sync(0xffffffffu, gd1, off);
        gs += __shfl_xor_sync(0xffffffffu, gs, off);
        if (better(a0, j0, gc0, gi0)) {
          gc0 = a0;
          gi0 = j0;
        }
        if (better(a1, j1, gc1, gi1)) {
          gc1 = a1;
          gi1 = j1;
          gd1 = e1;
        }
      }
      ++xchg;
      long long win = -1, win2 = -1;
      if (gi0 >= 0 && gc0 < tau0 * (1.0 - 1e-12)) {
        win = gi0;
      } else if (tau0 == INFINITY) {
        // sogmm.cpp:276-284: no point with d2 > 0: the lowest unchosen
        // index among 0 .. r (CTA 0 fenced its centre stores)
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        long long lo = LLONG_MAX;
        for (long long cnd = lane; cnd <= r && cnd < n; cnd += 32) {
          bool taken = false;
          for (int q = 0; q < r && !taken; ++q) taken = __ldcg(scr.centers + q) == cnd;
          if (!taken && cnd < lo) lo = cnd;
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          const long long u2 = __shfl_xor_sync(0xffffffffu, lo, off);
          lo = u2 < lo ? u2 : lo;
        }
        win = lo;
      }
      if (mode == 2 && win >= 0 && gi1 >= 0 && gc1 < tau1 * (1.0 - 1e-12)) {
        // c_r must leave the speculative winner's d2 unchanged (fold: strict <)
        double xa[4], xb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          xa[j] = x64[j * n + win];
          xb[j] = x64[j * n + gi1];
        }
        const double dd = dist2_t(xb, xa);
        if (!(dd < gd1)) win2 = gi1;
      }
      if (lane == 0) {
        s_win[0] = win;  // -1: repeat round r with a larger tau
        s_win[1] = win2;
        s_gsum = gs;
        if (win >= 0 && blockIdx.x == 0) {
          scr.centers[r] = win;
          if (win2 >= 0) scr.centers[r + 1] = win2;
          __threadfence();
          if (r + (win2 >= 0 ? 2 : 1) >= k)
            *reinterpret_cast<unsigned long long*>(scr.status + 2) = xchg;
        }
      }
      __syncwarp();
      bar_arrive(3, kTileKppThreads);
    }
    return;
  }

  // ========================= compute warps =========================
  const int ct = tid - 32, cw = warp - 1;
  const uint64_t* __restrict__ kp = ts.mkey;
  double cf[2][4];          // centres to fold (in round order)
  int nfc = 0, rfc = 0;     // how many, the round of the first
  double gsum = INFINITY;   // last known global sum of d2
  double cta_sum = 0.0;     // (ct == 0)
  double bc0, bc1, bd1;
  long long bi0, bi1;
  auto eval0 = [&](int j, uint64_t bits, int r) {
    const int64_t i = gidx(j);
    const double nl = nlu_exact_t(bits);
    double clk = nl;
    if (r > 0) {
      const double d2 = ts.md2[i];
      if (!(d2 > 0.0)) return;
      clk = nl / d2;
    }
    const long long oi = ts.perm[i];
    if (better(clk, oi, bc0, bi0)) {
      bc0 = clk;
      bi0 = oi;
    }
  };
  auto thresholds = [&](double tau, int r, unsigned* thr, bool sync) {
    for (int q = ct; q < nt; q += kWsCompute) {
      const double dmax = r == 0 ? 1.0 : sm.tsm[q].dmax;
      unsigned th = 0xffffffffu;
      if (dmax > 0.0) {
        const double e = exp(-tau * dmax) * (1.0 - 1e-12);
        th = e > 0.0 ? static_cast<unsigned>(fmin(e * 4294967296.0, 4294967295.0)) : 0u;
      }
      thr[q] = th;
    }
    if (sync) bar_sync(1, kWsCompute);
  };
  // round r drawn now, its candidates evaluated on the spot
  auto draw_now = [&](int r) {
    const uint64_t pre = round_prefix_t(seed, r);
    for (int j = ct; j < np; j += kWsCompute) {
      const int64_t ii = gidx(j);
      if (ii >= n) continue;
      const uint64_t bits = mix64(pre + (j < ncache ? sm.keys[j] : __ldg(kp + ii)));
      if (static_cast<unsigned>(bits >> 32) >= sm.thr[j >> 7]) eval0(j, bits, r);
    }
  };
  // rounds ra (and rb >= 0) kept in lists ra % 4 (rb % 4) in one pass over
  // the keys (a warp per tile, the tile's thresholds uniform, four points per
  // lane; -ln u after the pass)
  auto draw_keep = [&](int ra, int rb, double tau) {
    const int La = ra & (kW2Lists - 1), Lb = rb >= 0 ? (rb & (kW2Lists - 1)) : La;
    if (ct == 0) {
      s_lcount[La] = 0;
      s_lcover[La] = 0;
      s_ltau[La] = tau;
      s_lround[La] = ra;
      if (rb >= 0) {
        s_lcount[Lb] = 0;
        s_lcover[Lb] = 0;
        s_ltau[Lb] = tau;
        s_lround[Lb] = rb;
      }
    }
    thresholds(tau, ra, sm.thr, false);
    if (rb >= 0) thresholds(tau, rb, sm.thr2, false);
    bar_sync(1, kWsCompute);  // (orders the resets before the draws)
    const uint64_t prea = round_prefix_t(seed, ra);
    const uint64_t preb = round_prefix_t(seed, rb >= 0 ? rb : ra);
    auto keep = [&](int L, int jj, uint64_t bits) {
      const int slot = atomicAdd(&s_lcount[L], 1);
      if (slot < kW2Cap) {
        sm.cand_j[L * kW2Cap + slot] = jj;
        sm.cand_nl[L * kW2Cap + slot] = __longlong_as_double(static_cast<long long>(bits));
      } else {
        s_lcover[L] = 1;
      }
    };
    for (int q = cw; q < nt; q += kWsCWarps) {
      const unsigned tha = sm.thr[q];
      const unsigned thb = rb >= 0 ? sm.thr2[q] : 0xffffffffu;
      const int jb = q * kTile;
      uint64_t kv[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int jj = jb + lane + 32 * h;
        kv[h] = jj < ncache ? sm.keys[jj] : 0ull;
      }
      if (jb + kTile > ncache) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int jj = jb + lane + 32 * h;
          const int64_t ii = gidx(jj);
          if (jj >= ncache && ii < n) kv[h] = __ldg(kp + ii);
        }
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const bool ca = mix64_hi32(prea + kv[h]) >= tha;
        const bool cb = rb >= 0 && mix64_hi32(preb + kv[h]) >= thb;
        if (ca || cb) {  // (rare) the full draws
          const int jj = jb + lane + 32 * h;
          if (gidx(jj) < n) {
            if (ca) keep(La, jj, mix64(prea + kv[h]));
            if (cb) keep(Lb, jj, mix64(preb + kv[h]));
          }
        }
      }
    }
    bar_sync(1, kWsCompute);
    const int na = s_lcount[La] < kW2Cap ? s_lcount[La] : kW2Cap;
    for (int q = ct; q < na; q += kWsCompute)
      sm.cand_nl[La * kW2Cap + q] = nlu_exact_t(static_cast<uint64_t>(__double_as_longlong(sm.cand_nl[La * kW2Cap + q])));
    if (rb >= 0) {
      const int nb = s_lcount[Lb] < kW2Cap ? s_lcount[Lb] : kW2Cap;
      for (int q = ct; q < nb; q += kWsCompute)
        sm.cand_nl[Lb * kW2Cap + q] = nlu_exact_t(static_cast<uint64_t>(__double_as_longlong(sm.cand_nl[Lb * kW2Cap + q])));
    }
    bar_sync(1, kWsCompute);
  };
  auto list_ok = [&](int rr) {
    const int L = rr & (kW2Lists - 1);
    return s_lround[L] == rr && s_lcover[L] == 0;
  };

  int r = 0;
  unsigned xe = 0;  // exchanges so far (profiling)
  for (;;) {
#ifdef GMMB_KPP_TPROF
    if (ct == 0 && xe < 4096 && blockIdx.x < 160) g_tprof[3][xe][blockIdx.x] = gtime();
#endif
    // ---- fold the centres decided in the last epoch (in round order)
    if (nfc > 0) {
      for (int q = ct; q < nt; q += kWsCompute) {
        const TileSmem& tt = sm.tsm[q];
        bool hit = false;
#pragma unroll
        for (int f = 0; f < 2; ++f) {
          if (f >= nfc) break;
          double lb = 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double g = fmax(fmax(tt.box[j] - cf[f][j], cf[f][j] - tt.box[4 + j]), 0.0);
            lb = fma(g, g, lb);
          }
          hit = hit || !(lb * (1.0 - 1e-12) >= tt.dmax);
        }
        if (hit) sm.fold[atomicAdd(&s_nfold, 1)] = q;
      }
      bar_sync(1, kWsCompute);
      const int nf = s_nfold;
      double delta = 0.0;
      for (int fi = cw; fi < nf; fi += kWsCWarps) {
        const int q = sm.fold[fi];
        TileSmem& tt = sm.tsm[q];
        const int64_t ib = static_cast<int64_t>(gtile(q)) * kTile;
        double mx = 0.0, smv = 0.0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int64_t i = ib + lane + 32 * h;
          if (i < n) {
            double x[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = ts.xm[j * n + i];
            double d2 = ts.md2[i];
            int lab = -1;
#pragma unroll
            for (int f = 0; f < 2; ++f) {
              if (f >= nfc) break;
              const double dd = dist2_t(x, cf[f]);
              if (dd < d2) {
                d2 = dd;
                lab = rfc + f;
              }
            }
            if (lab >= 0) {
              ts.md2[i] = d2;
              ts.mlab[i] = lab;
            }
            mx = fmax(mx, d2);
            smv += d2;
          }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          smv += __shfl_xor_sync(0xffffffffu, smv, off);
        }
        if (lane == 0) {
          tt.dmax = mx;
          delta += smv - tt.sum;
          tt.sum = smv;
        }
      }
      if (lane == 0) s_delta[cw] = delta;
      bar_sync(1, kWsCompute);
      if (ct == 0) {
        for (int w = 0; w < kWsCWarps; ++w) cta_sum += s_delta[w];
#ifdef GMMB_KPP_TPROF
        if (xe < 4096 && blockIdx.x < 160) {
          g_tprof[4][xe][blockIdx.x] = gtime();
          g_tprof[5][xe][blockIdx.x] = s_nfold;
        }
#endif
        s_nfold = 0;
      }
    }
    if (r >= k) {
      if (ct == 0) s_r = k;  // releases the communication warp
      bar_arrive(2, kTileKppThreads);
      break;
    }
    // ---- epoch: round r (exact), and round r + 1 from its kept list
    // (speculative) when both lists are there
    double tau = r == 0 ? kTauAlpha / static_cast<double>(n)
                        : (isfinite(gsum) && gsum > 0.0 ? kTauAlpha / gsum : INFINITY);
    bool first = true;
    for (;;) {
      const bool use0 = first && list_ok(r);
      const bool mode2 = first && use0 && r + 1 < k && list_ok(r + 1);
      bc0 = INFINITY;
      bi0 = -1;
      bc1 = INFINITY;
      bi1 = -1;
      bd1 = 0.0;
      double tau1 = 0.0;
      if (use0) {
        const int L = r & (kW2Lists - 1);
        tau = s_ltau[L];
        const int nc = s_lcount[L];
        for (int q = ct; q < nc; q += kWsCompute) {
          const int64_t i = gidx(sm.cand_j[L * kW2Cap + q]);
          const double d2 = ts.md2[i];
          if (!(d2 > 0.0)) continue;
          const double clk = sm.cand_nl[L * kW2Cap + q] / d2;
          const long long oi = ts.perm[i];
          if (better(clk, oi, bc0, bi0)) {
            bc0 = clk;
            bi0 = oi;
          }
        }
      } else {
        thresholds(tau, r, sm.thr, true);
        draw_now(r);
      }
      if (mode2) {
        const int L = (r + 1) & (kW2Lists - 1);
        tau1 = s_ltau[L];
        const int nc = s_lcount[L];
        for (int q = ct; q < nc; q += kWsCompute) {
          const int64_t i = gidx(sm.cand_j[L * kW2Cap + q]);
          const double d2 = ts.md2[i];
          if (!(d2 > 0.0)) continue;
          const double clk = sm.cand_nl[L * kW2Cap + q] / d2;
          const long long oi = ts.perm[i];
          if (better(clk, oi, bc1, bi1)) {
            bc1 = clk;
            bi1 = oi;
            bd1 = d2;
          }
        }
      }
      // ---- publish both levels
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const double a0 = __shfl_xor_sync(0xffffffffu, bc0, off);
        const long long j0 = __shfl_xor_sync(0xffffffffu, bi0, off);
        const double a1 = __shfl_xor_sync(0xffffffffu, bc1, off);
        const long long j1 = __shfl_xor_sync(0xffffffffu, bi1, off);
        const double e1 = __shfl_xor_sync(0xffffffffu, bd1, off);
        if (better(a0, j0, bc0, bi0)) {
          bc0 = a0;
          bi0 = j0;
        }
        if (better(a1, j1, bc1, bi1)) {
          bc1 = a1;
          bi1 = j1;
          bd1 = e1;
        }
      }
      if (lane == 0) {
        s_bc[0][cw] = bc0;
        s_bi[0][cw] = bi0;
        s_bc[1][cw] = bc1;
        s_bi[1][cw] = bi1;
        s_bd[cw] = bd1;
      }
      if (ct == 0) {
        s_r = r;
        s_mode = mode2 ? 2 : 1;
        s_tau[0] = tau;
        s_tau[1] = tau1;
        s_cta_sum = cta_sum;
      }
      bar_arrive(2, kTileKppThreads);
      // ---- meanwhile: the kept lists of the next rounds that are missing
      // (at most two; first attempt only, once d2 is known everywhere)
      if (first && r >= 1 && isfinite(gsum) && gsum > 0.0) {
        // which lists (every compute thread decides from the same state,
        // then a barrier before the first list is rewritten)
        int todo[2] = {-1, -1}, nd = 0;
        for (int rr = r + 1; rr <= r + 3 && rr < k && nd < 2; ++rr) {
          // (lists r and, in a pair epoch, r + 1 are in use this epoch)
          if (list_ok(rr) || (rr == r + 1 && mode2)) continue;
          todo[nd++] = rr;
        }
        bar_sync(1, kWsCompute);
        if (nd > 0) draw_keep(todo[0], nd > 1 ? todo[1] : -1, kSpecAlpha / gsum);
#ifdef GMMB_KPP_TPROF
        if (ct == 0 && xe < 4096 && blockIdx.x < 160) g_tprof[2][xe][blockIdx.x] = gtime();
#endif
      }
      ++xe;
      bar_sync(3, kTileKppThreads);  // the exchange result
      const long long win = s_win[0], win2 = s_win[1];
      gsum = s_gsum;
      if (win >= 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) cf[0][j] = x64[j * n + win];
        nfc = 1;
        rfc = r;
        if (win2 >= 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) cf[1][j] = x64[j * n + win2];
          nfc = 2;
        }
        r += nfc;
        break;
      }
      first = false;
      // (no point with d2 > 0 left: straight to the fallback)
      tau = !(isfinite(gsum) && gsum > 0.0) || tau * 64.0 > 1e300 ? INFINITY : tau * 64.0;
    }
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
  // (the two-round kernel's slots are twice as wide: 2 x 128 B per CTA)
  cudaError_t e = cudaMemsetAsync(scr.slots, 0, sizeof(KppSlot) * 4 * sm_count, s);
  if (e != cudaSuccess) return e;
  int nblk = sm_count;  // one CTA per SM
  if (nblk > ntiles) nblk = ntiles;
  if ((ntiles + nblk - 1) / nblk > kMaxCtaTiles || nblk > 32 * kPollSlots) return cudaErrorInvalidValue;
  // GMMB_KPP_TILE=sync: the single-role kernel (every round drawn after its
  // exchange); =ws1: warp-specialised, one round per exchange; default: two
  static const int variant = [] {
    const char* v = getenv("GMMB_KPP_TILE");
    if (v && v[0] == 's') return 0;
    if (v && std::strcmp(v, "ws1") == 0) return 1;
    return 2;
  }();
  const bool ws = variant != 0;
  const void* fn = variant == 0 ? (const void*)kpp_tile_kernel
                 : variant == 1 ? (const void*)kpp_tile_ws_kernel
                                : (const void*)kpp_tile_ws2_kernel;
  int mt = (ntiles + nblk - 1) / nblk;
  int max_smem = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t statics = 4096;  // the kernels' static shared words (ws2: 2.3 KB)
  int kcache = 0;
  size_t smem = sizeof(TileSmem) * kMaxCtaTiles + sizeof(unsigned) * kMaxCtaTiles;
  if (ws) {
    const size_t fixed = variant == 2 ? ws2_fixed_bytes(mt) : ws_fixed_bytes(mt);
    const size_t avail = static_cast<size_t>(max_smem) > fixed + statics ? max_smem - fixed - statics : 0;
    kcache = static_cast<int>(std::min<size_t>(avail / sizeof(uint64_t), static_cast<size_t>(mt) * kTile));
    smem = fixed + sizeof(uint64_t) * kcache;
  }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kTileKppThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  void* args_ws[] = {(void*)&x64, (void*)&n, (void*)&ntiles, (void*)&k, (void*)&seed,
                     (void*)&ts, (void*)&scr, (void*)&mt, (void*)&kcache};
  void* args[] = {(void*)&x64, (void*)&n, (void*)&ntiles, (void*)&k, (void*)&seed,
                  (void*)&ts, (void*)&scr, (void*)&arrive};
  e = cudaLaunchCooperativeKernel(fn, dim3(nblk), dim3(kTileKppThreads), ws ? args_ws : args, smem, s);
  if (e != cudaSuccess) return e;
  kpp_tile_scatter_kernel<<<grid, 256, 0, s>>>(n, perm, ts.mlab, scr.labels, scr.owned);
  return cudaGetLastError();
}

}  // namespace gmmb

#ifdef GMMB_KPP_TPROF
extern "C" int gmmb_debug_kpp_tprof(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, gmmb::g_tprof, sizeof(gmmb::g_tprof)));
}
#endif
