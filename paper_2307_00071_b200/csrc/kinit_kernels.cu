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
// Work per point per round is cut three ways:
//  * the (seed, round) half of the counter hash is hoisted out of the point
//    loop and keys are stored pre-multiplied, leaving one mix64 per point;
//  * clocks are first evaluated in FP32 with a proven relative error bound
//    (< 1e-4); only points within 4e-4 of their warp's approximate minimum
//    (typically one per warp) get the exact FP64 log and division, which
//    therefore decide the argmin exactly;
//  * the nearest-centre pass (sogmm.cpp:290-312) is folded into the rounds:
//    round r already evaluates d(x, c_{r-1}), so the running argmin with
//    strict < over ascending centre index gives the labels for free.
// The per-round grid exchange: each CTA publishes one 64-byte slot, arrives
// on a monotonic counter with a release reduction, one thread per CTA polls
// the counter (relaxed loads, one acquire fence), then every CTA reduces all
// slots in the same order.
#include <climits>

#include "kinit_kernels.cuh"

namespace gmmb {

namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr float kBand = 1.0f + 4e-4f;  // >> 2x the approx-clock error bound

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

// rng.hpp:22-28 with the per-point tail split off:
//   bits = mix64(prefix(seed, r) + key * golden)
__device__ __forceinline__ uint64_t round_prefix(uint64_t seed, int r) {
  return mix64(mix64(seed ^ 0x2545f4914f6cdd1dULL) +
               static_cast<uint64_t>(r) * kGolden);
}

// -ln(uniform_pos) exactly as sogmm.cpp:240-241 (FP64)
__device__ __forceinline__ double nlu_exact(uint64_t bits) {
  return -log(static_cast<double>((bits >> 11) + 1) * 0x1.0p-53);
}

// FP32 approximation of -ln(u) with relative error < 3e-5 (the candidate
// band kBand is 4e-4, > 2x the bound plus the 1/d2 rounding), where
// u = (m + 1) 2^-53 and m = bits >> 11:
//  * v = 1 - u < 2^-4: -ln u = v + v^2/2 + v^3/3 + v^4/4 + O(v^5), the
//    truncation is < v^4/5 < 3e-6 relative; v is read from its top 32 bits
//    (w = v >> 17, midpoint => < 2^-17 relative once w >= 2^16, else the
//    exact 64-bit conversion);
//  * u <= 1 - 2^-4 (so -ln u >= 0.0645): u from the top 32 bits of the hash
//    (t = bits >> 32, midpoint => < 2^-21 relative once t >= 2^20, i.e.
//    < 7.4e-6 on -ln u; smaller t use the exact 64-bit conversion) and
//    lg2.approx (relative ~2^-22).
__device__ __forceinline__ float nlu_approx(uint64_t bits) {
  const uint64_t m = bits >> 11;
  const uint64_t v = ((1ULL << 53) - 1) - m;
  float out;
  if (v < (1ULL << 49)) {
    const unsigned w = static_cast<unsigned>(v >> 17);
    const float vf = w >= (1u << 16) ? (__uint2float_rn(w) + 0.5f) * 0x1p-36f
                                     : __ull2float_rn(v) * 0x1p-53f;
    out = vf * fmaf(vf, fmaf(vf, fmaf(vf, 0.25f, 0.333333343f), 0.5f), 1.0f);
  } else {
    const unsigned t = static_cast<unsigned>(bits >> 32);
    const float uf = t >= (1u << 20) ? (__uint2float_rn(t) + 0.5f) * 0x1p-32f
                                     : __ull2float_rn(m + 1) * 0x1p-53f;
    float lg;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(uf));
    out = -lg * 0.693147182f;
  }
  return out;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// lexicographic (clock, idx) order; idx -1 = none
__device__ __forceinline__ bool cand_better(double c2, long long i2, double c,
                                            long long i) {
  return i2 >= 0 && (i < 0 || c2 < c || (c2 == c && i2 < i));
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
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
  keys[i] = h * kGolden;
}

constexpr int kSeedPPT = 8;
constexpr int kSeedThreads = 384;
constexpr int kSeedWarps = kSeedThreads / 32;
constexpr int kMaxSeedBlocks = 1024;

struct SeedSmem {
  double wc[kSeedWarps];
  long long wi[kSeedWarps];
  int wo[kSeedWarps];
  double wx[kSeedWarps][4];
  double gc[kMaxSeedBlocks / 32];
  long long gi[kMaxSeedBlocks / 32];
  int gs[kMaxSeedBlocks / 32];
  long long gu[kMaxSeedBlocks / 32];
  long long win;
  int win_owner;
  int fallbacks;
  double cx[4];
  double scx[kMaxSeedBlocks][4];   // gathered slot coordinates
  int sown[kMaxSeedBlocks];
};

__device__ __forceinline__ void shfl_cand(double& c, long long& i, int& s,
                                          int off) {
  const double c2 = __shfl_xor_sync(0xffffffffu, c, off);
  const long long i2 = __shfl_xor_sync(0xffffffffu, i, off);
  const int s2 = __shfl_xor_sync(0xffffffffu, s, off);
  if (cand_better(c2, i2, c, i)) {
    c = c2;
    i = i2;
    s = s2;
  }
}

// arrive on a monotonic grid counter and wait for all CTAs (one thread)
__device__ __forceinline__ void grid_exchange(unsigned* counter, unsigned target) {
  red_release_add(counter, 1u);
  while (ld_relaxed_u32(counter) < target) {
  }
  fence_acq_rel();
}

// Each thread keeps PPT points (stride = grid threads) in registers.
__global__ void __launch_bounds__(kSeedThreads, 1)
    kpp_seed_kernel(const double* __restrict__ x64, int64_t n, int k,
                    uint64_t seed, KinitScratch scr) {
  constexpr int PPT = kSeedPPT;
  __shared__ SeedSmem sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nblk = gridDim.x;
  const long long G = static_cast<long long>(nblk) * kSeedThreads;
  const long long g0 = static_cast<long long>(blockIdx.x) * kSeedThreads + tid;
  double px[PPT][4], d2[PPT];
  float inv[PPT];  // ~1/d2 in FP32 (approximate clocks only)
  uint64_t kp[PPT];
  int lab[PPT];
  unsigned chosen = 0, valid = 0;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const long long i = g0 + j * G;
    const bool v = i < n;
    if (v) valid |= 1u << j;
#pragma unroll
    for (int q = 0; q < 4; ++q) px[j][q] = v ? x64[q * n + i] : 0.0;
    kp[j] = v ? scr.keys[i] : 0;
    d2[j] = INFINITY;
    inv[j] = 0.f;
    lab[j] = 0;
  }
  // slots beyond the warp's last valid point are skipped (warp-uniform)
  const unsigned wvalid = __reduce_or_sync(0xffffffffu, valid);
  if (tid == 0) sm.fallbacks = 0;
  double c[4] = {0, 0, 0, 0};
  unsigned epoch = 0;  // completed grid exchanges
  for (int r = 0; r <= k; ++r) {
    const uint64_t pre = round_prefix(seed, r);
    float a[PPT];
    float amin = INFINITY;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      a[j] = INFINITY;
      if (!((wvalid >> j) & 1)) continue;
      if (r > 0) {  // fold c_{r-1} (sogmm.cpp:229-238) + running label
        const double dd = dist2(px[j][0], px[j][1], px[j][2], px[j][3], c);
        if (dd < d2[j]) {
          d2[j] = dd;
          lab[j] = r - 1;
          // 1/d2 for the approximate clock; d2 == 0 (a chosen point or a
          // duplicate) is ineligible (sogmm.cpp:254)
          const float f = __double2float_rn(dd);
          inv[j] = dd > 0.0 ? (isinf(f) ? 1e-38f : rcp_approx(f)) : 0.f;
        }
      }
      if (r == k) continue;
      const float na = nlu_approx(mix64(pre + kp[j]));
      const float aj = r == 0 ? na : (inv[j] > 0.f ? na * inv[j] : INFINITY);
      a[j] = ((valid >> j) & 1) ? aj : INFINITY;
      amin = fminf(amin, a[j]);
    }
    if (r == k) break;
    // warp filter, then exact FP64 clocks for the few candidates
    float wmin = amin;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
      wmin = fminf(wmin, __shfl_xor_sync(0xffffffffu, wmin, off));
    const float thr = wmin * kBand;
    double bc = INFINITY;
    long long bi = -1;
    int bj = 0;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      if (!((wvalid >> j) & 1)) continue;
      const bool cj = ((valid >> j) & 1) && (r == 0 || d2[j] > 0.0) && !(a[j] > thr);
      if (__any_sync(0xffffffffu, cj)) {
        if (cj) {
          const double nl = nlu_exact(mix64(pre + kp[j]));
          const double clk = r == 0 ? nl : nl / d2[j];
          const long long i = g0 + j * G;
          if (clk < INFINITY && cand_better(clk, i, bc, bi)) {
            bc = clk;
            bi = i;
            bj = j;
          }
        }
      }
    }
    // warp argmin: usually a single lane holds a candidate
    const unsigned has = __ballot_sync(0xffffffffu, bi >= 0);
    int src = has ? __ffs(has) - 1 : 0;
    if (__popc(has) > 1) {
      double wc = bc;
      long long wi = bi;
      int ws = lane;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) shfl_cand(wc, wi, ws, off);
      src = ws;
    }
    if (has && lane == src) {
      double x0 = px[0][0], x1 = px[0][1], x2 = px[0][2], x3 = px[0][3];
#pragma unroll
      for (int j = 1; j < PPT; ++j) {
        if (bj == j) {
          x0 = px[j][0]; x1 = px[j][1]; x2 = px[j][2]; x3 = px[j][3];
        }
      }
      sm.wc[warp] = bc;
      sm.wi[warp] = bi;
      sm.wo[warp] = static_cast<int>(g0);
      sm.wx[warp][0] = x0; sm.wx[warp][1] = x1; sm.wx[warp][2] = x2; sm.wx[warp][3] = x3;
    } else if (!has && lane == 0) {
      sm.wc[warp] = INFINITY;
      sm.wi[warp] = -1;
      sm.wo[warp] = -1;
    }
    __syncthreads();
    KppSlot* slots = scr.slots + (r & 1) * nblk;
    if (warp == 0) {
      double c1 = lane < kSeedWarps ? sm.wc[lane] : INFINITY;
      long long i1 = lane < kSeedWarps ? sm.wi[lane] : -1;
      int s1 = lane;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) shfl_cand(c1, i1, s1, off);
      if (lane == 0) {
        KppSlot& sl = slots[blockIdx.x];
        sl.clock = c1;
        sl.idx = i1;
        sl.owner = i1 >= 0 ? sm.wo[s1] : -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) sl.cx[q] = i1 >= 0 ? sm.wx[s1][q] : 0.0;
        ++epoch;
        grid_exchange(scr.counter, static_cast<unsigned>(nblk) * epoch);
      }
    }
    __syncthreads();
    // every CTA reduces every CTA's slot in the same order => same winner
    if (tid < ((nblk + 31) & ~31)) {
      double gc = INFINITY;
      long long gi = -1;
      int gs = -1;
      for (int b = tid; b < nblk; b += kSeedThreads) {
        const volatile KppSlot& vs = slots[b];
        const double c2 = vs.clock;
        const long long i2 = vs.idx;
        sm.sown[b] = vs.owner;
#pragma unroll
        for (int q = 0; q < 4; ++q) sm.scx[b][q] = vs.cx[q];
        if (cand_better(c2, i2, gc, gi)) {
          gc = c2;
          gi = i2;
          gs = b;
        }
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) shfl_cand(gc, gi, gs, off);
      if (lane == 0) {
        sm.gc[warp] = gc;
        sm.gi[warp] = gi;
        sm.gs[warp] = gs;
      }
    }
    __syncthreads();
    if (warp == 0) {
      const int nw = (nblk + 31) >> 5;
      double c1 = lane < nw ? sm.gc[lane] : INFINITY;
      long long i1 = lane < nw ? sm.gi[lane] : -1;
      int s1 = lane < nw ? sm.gs[lane] : -1;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) shfl_cand(c1, i1, s1, off);
      if (lane == 0) {
        if (i1 >= 0 && c1 < INFINITY) {
          sm.win = i1;
          sm.win_owner = sm.sown[s1];
#pragma unroll
          for (int q = 0; q < 4; ++q) sm.cx[q] = sm.scx[s1][q];
        } else {
          sm.win = -1;  // no eligible point anywhere: fallback below
        }
      }
    }
    __syncthreads();
    if (sm.win < 0) {
      // sogmm.cpp:276-284: lowest unchosen index (rare; a second exchange)
      const unsigned freem = valid & ~chosen;
      long long bu = freem ? g0 + static_cast<long long>(__ffs(freem) - 1) * G : LLONG_MAX;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const long long u2 = __shfl_xor_sync(0xffffffffu, bu, off);
        bu = u2 < bu ? u2 : bu;
      }
      if (lane == 0) sm.gu[warp] = bu;
      __syncthreads();
      if (tid == 0) {
        long long m = LLONG_MAX;
        for (int w = 0; w < kSeedWarps; ++w) m = sm.gu[w] < m ? sm.gu[w] : m;
        KppSlot* fs = scr.slots + 2 * nblk;
        fs[blockIdx.x].unchosen = m;
        ++epoch;
        grid_exchange(scr.counter, static_cast<unsigned>(nblk) * epoch);
        m = LLONG_MAX;
        for (int b = 0; b < nblk; ++b) {
          const long long u2 = reinterpret_cast<volatile KppSlot*>(fs)[b].unchosen;
          m = u2 < m ? u2 : m;
        }
        sm.win = m;
        sm.win_owner = static_cast<int>(m % G);
#pragma unroll
        for (int q = 0; q < 4; ++q) sm.cx[q] = x64[q * n + m];
      }
      __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) scr.centers[r] = sm.win;
#pragma unroll
    for (int q = 0; q < 4; ++q) c[q] = sm.cx[q];
    if (sm.win_owner == static_cast<int>(g0)) {
      chosen |= 1u << static_cast<int>((sm.win - g0) / G);
    }
    // sm.win / sm.cx are rewritten only after the next round's exchange,
    // which every thread reaches after these reads (two barriers later)
  }
  // labels + owned counts (every point's final nearest centre)
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const long long i = g0 + j * G;
    if (i >= n) continue;
    scr.labels[i] = lab[j];
    atomicAdd(&scr.owned[lab[j]], 1);
  }
}

// Memory-resident variant (N beyond the register budget): plain exact FP64
// clocks, state in global memory, one launch per round (grid barrier =
// kernel boundary), CTA slots reduced by the last CTA to finish.
__global__ void __launch_bounds__(512)
    kpp_mem_round_kernel(const double* __restrict__ x64, int64_t n, int r,
                         int k, uint64_t seed, KinitScratch scr, int* ticket,
                         long long* win_io) {
  __shared__ double s_c[16];
  __shared__ long long s_i[16];
  __shared__ long long s_u[16];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = static_cast<int64_t>(gridDim.x) * 512;
  const long long win = r > 0 ? win_io[0] : -1;
  double c[4] = {0, 0, 0, 0};
  if (r > 0)
    for (int q = 0; q < 4; ++q) c[q] = x64[q * n + win];
  const uint64_t pre = round_prefix(seed, r);
  double bc = INFINITY;
  long long bi = -1, bu = LLONG_MAX;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 512 + tid; i < n; i += G) {
    double dcur;
    if (r > 0) {
      dcur = scr.d2[i];
      const double dd = dist2(x64[i], x64[n + i], x64[2 * n + i], x64[3 * n + i], c);
      if (dd < dcur) {
        dcur = dd;
        scr.d2[i] = dd;
        scr.labels[i] = r - 1;
      }
      if (i == win) scr.chosen[i] = 1;
    } else {
      dcur = INFINITY;
      scr.d2[i] = INFINITY;
      scr.labels[i] = 0;
      scr.chosen[i] = 0;
    }
    if (r == k) continue;
    const double nl = nlu_exact(mix64(pre + scr.keys[i]));
    if (r == 0) {
      if (cand_better(nl, i, bc, bi)) { bc = nl; bi = i; }
    } else if (dcur > 0.0) {
      const double clk = nl / dcur;
      if (clk < INFINITY && cand_better(clk, i, bc, bi)) { bc = clk; bi = i; }
    }
    if (!scr.chosen[i] && i < bu) bu = i;
  }
  if (r == k) return;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
    const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
    const long long u2 = __shfl_xor_sync(0xffffffffu, bu, off);
    if (cand_better(c2, i2, bc, bi)) { bc = c2; bi = i2; }
    bu = u2 < bu ? u2 : bu;
  }
  if (lane == 0) { s_c[warp] = bc; s_i[warp] = bi; s_u[warp] = bu; }
  __syncthreads();
  if (warp == 0) {
    bc = lane < 16 ? s_c[lane] : INFINITY;
    bi = lane < 16 ? s_i[lane] : -1;
    bu = lane < 16 ? s_u[lane] : LLONG_MAX;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
      const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
      const long long u2 = __shfl_xor_sync(0xffffffffu, bu, off);
      if (cand_better(c2, i2, bc, bi)) { bc = c2; bi = i2; }
      bu = u2 < bu ? u2 : bu;
    }
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
  if (!s_last || tid != 0) return;
  __threadfence();
  double gc = INFINITY;
  long long gi = -1, gu = LLONG_MAX;
  for (int b = 0; b < static_cast<int>(gridDim.x); ++b) {
    const volatile KppSlot& sl = scr.slots[b];
    if (cand_better(sl.clock, sl.idx, gc, gi)) { gc = sl.clock; gi = sl.idx; }
    gu = sl.unchosen < gu ? sl.unchosen : gu;
  }
  const long long w = (gi >= 0 && gc < INFINITY) ? gi : gu;
  win_io[0] = w;
  scr.centers[r] = w;
  *ticket = 0;
}

__global__ void owned_kernel(int64_t n, const int32_t* __restrict__ labels,
                             int* __restrict__ owned) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&owned[labels[i]], 1);
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
    if (cand_better(prev[w].clock, prev[w].idx, bc, bi)) {
      bc = prev[w].clock;
      bi = prev[w].idx;
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
  const uint64_t pre = round_prefix(seed, r);
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
    const double nl = nlu_exact(mix64(pre + scr.keys[li]));
    if (r == 0) {
      if (cand_better(nl, gi, bc, bi)) { bc = nl; bi = gi; }
    } else if (dcur > 0.0) {
      const double clk = nl / dcur;
      if (clk < INFINITY && cand_better(clk, gi, bc, bi)) { bc = clk; bi = gi; }
    }
    if (!scr.chosen[li] && gi < bu) bu = gi;
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
    const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
    const long long u2 = __shfl_xor_sync(0xffffffffu, bu, off);
    if (cand_better(c2, i2, bc, bi)) { bc = c2; bi = i2; }
    bu = u2 < bu ? u2 : bu;
  }
  if (lane == 0) { s_c[warp] = bc; s_i[warp] = bi; s_u[warp] = bu; }
  __syncthreads();
  if (warp == 0) {
    bc = lane < 16 ? s_c[lane] : INFINITY;
    bi = lane < 16 ? s_i[lane] : -1;
    bu = lane < 16 ? s_u[lane] : LLONG_MAX;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const double c2 = __shfl_xor_sync(0xffffffffu, bc, off);
      const long long i2 = __shfl_xor_sync(0xffffffffu, bi, off);
      const long long u2 = __shfl_xor_sync(0xffffffffu, bu, off);
      if (cand_better(c2, i2, bc, bi)) { bc = c2; bi = i2; }
      bu = u2 < bu ? u2 : bu;
    }
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
  if (!s_last || tid != 0) return;
  __threadfence();
  double gc = INFINITY;
  long long gi2 = -1, gu = LLONG_MAX;
  for (int b = 0; b < static_cast<int>(gridDim.x); ++b) {
    const volatile KppSlot& sl = scr.slots[b];
    if (cand_better(sl.clock, sl.idx, gc, gi2)) { gc = sl.clock; gi2 = sl.idx; }
    gu = sl.unchosen < gu ? sl.unchosen : gu;
  }
  out->clock = gc;
  out->idx = gi2;
  out->unchosen = gu;
  for (int q = 0; q < 4; ++q) {
    out->x[q] = gi2 >= 0 ? x64[q * n + (gi2 - offset)] : 0.0;
    out->ux[q] = gu != LLONG_MAX ? x64[q * n + (gu - offset)] : 0.0;
  }
  *ticket = 0;
  if (r > 0) scr.centers[r - 1] = win;
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

cudaError_t launch_kpp_seed(const double* x64, int64_t n, int k, uint64_t seed,
                            KinitScratch scr, int sm_count, cudaStream_t s) {
  // one CTA per SM, points register-resident while they fit
  const int nblk = sm_count < kMaxSeedBlocks ? sm_count : kMaxSeedBlocks;
  if (n <= static_cast<int64_t>(nblk) * kSeedThreads * kSeedPPT) {
    void* args[] = {(void*)&x64, (void*)&n, (void*)&k, (void*)&seed, (void*)&scr};
    return cudaLaunchCooperativeKernel((void*)kpp_seed_kernel, dim3(nblk),
                                       dim3(kSeedThreads), args, 0, s);
  }
  // memory-resident fallback: one launch per round
  const int grid = sm_count * 4;
  int* ticket = scr.status;
  long long* win = reinterpret_cast<long long*>(scr.status + 2);
  cudaError_t e = cudaMemsetAsync(scr.status, 0, sizeof(int) * 4, s);
  if (e != cudaSuccess) return e;
  for (int r = 0; r <= k; ++r) {
    kpp_mem_round_kernel<<<grid, 512, 0, s>>>(x64, n, r, k, seed, scr, ticket, win);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  owned_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, s>>>(n, scr.labels, scr.owned);
  return cudaGetLastError();
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
