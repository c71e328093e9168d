// estep_chunked.cu — the fused E step + sufficient statistics for K > 512:
// two passes over the points, components in chunks of 512 (one CTA holds a
// chunk: thread j the pair (c*512 + j, c*512 + 256 + j)), any K.
//
// Reference semantics: e_step_into (sogmm.cpp:341-383, logsumexp_rows
// kernels.cpp:104-135) and m_step_impl's moments (sogmm.cpp:399-455,
// weighted_moments_fn kernels.hpp:82-181), like em_kernels.cu.
//
// The responsibility of (point n, component k) needs the normaliser over ALL
// K components. One CTA cannot hold more than 512 components' constants and
// statistics in registers, and the cluster kernels that exchanged per-point
// partial sums between CTAs after every 16-point sub-tile spent a third of
// their time synchronising. Here the exchange is a pass:
//
//  A  lse_part_kernel    chunk c x point range: e = 2^-Q in FP32 (the same
//                        FFMA chains as the single-CTA kernel), per-point
//                        sums over the chunk (warp reduce-scatter + a fixed-
//                        order combine of the 8 warps) -> part[c][n]
//     lse_combine_kernel L_n = log2(sum_c part[c][n]) (fixed chunk order);
//                        a point whose sum leaves [2^-64, 2^64] (far from
//                        every component) is listed for ...
//     lse_exact_kernel   ... the exact max-shifted log-sum-exp (warp per
//                        point, fixed order)
//  B  stats_chunk_kernel chunk c x point range: r = 2^-(Q + L_n) directly
//                        (no normaliser in the pass), statistics centred at
//                        mu_old (sum r, sum r d, sum r d d^T) in FP32 pairs
//                        widened to FP64 shared memory every 16 points; per
//                        (range, component) FP64 partials + the ll partials
//                        (chunk 0 CTAs) for the ordered reduce.
//
// No CTA ever waits for another: pass B has no synchronisation at all (each
// warp streams its own points; tiles are broadcast loads through L1), pass A
// one CTA barrier per 128-point tile. Cost: the 14 FFMA2 of the density are
// evaluated twice per (point, component pair), against the single-CTA
// kernel's cross-warp hand-off.
#include "em_kernels.cuh"
#include "f32x2.cuh"

namespace gmmb {

namespace {

using namespace dev;

#ifndef GMMB_CHUNK_WS
#define GMMB_CHUNK_WS 1  // 1: pass B on the warp-specialised kernel; 0: stats_chunk_kernel
#endif

constexpr int kT = 256;      // threads per CTA (component pairs of a chunk)
constexpr int kP = 16;       // points per sub-tile (pass A reduce-scatter)
constexpr int kSPT = kTile / kP;

// ---- a thread's component pair ------------------------------------------
template <int D>
struct PairConsts {
  static constexpr int NP = npacked(D);
  f2_t PP[NP];  // sqrt(0.5 log2 e) P, packed lower
  f2_t NBASE;   // -base2
  int ka, kb;   // the two components
};

template <int D>
__device__ __forceinline__ void load_pair(const ModelBuf& mb, int k_cur, int ka, int kb,
                                          PairConsts<D>& pc) {
  constexpr int NP = npacked(D);
  float pp[2][NP], nb[2];
  const int ks[2] = {ka, kb};
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    nb[c] = INFINITY;  // padding component: e = 2^-inf = 0
#pragma unroll
    for (int q = 0; q < NP; ++q) pp[c][q] = 0.f;
    if (ks[c] < k_cur) {
      const float4* c4 = reinterpret_cast<const float4*>(mb.cst + ks[c]);
      const float4 a = c4[0], b = c4[1], e = c4[2];
      const float cc[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, e.x, e.y, e.z, e.w};
#pragma unroll
      for (int q = 0; q < NP; ++q) pp[c][q] = cc[q];
      nb[c] = -cc[10];
    }
  }
#pragma unroll
  for (int q = 0; q < NP; ++q) pc.PP[q] = pk(pp[0][q], pp[1][q]);
  pc.NBASE = pk(nb[0], nb[1]);
  pc.ka = ka;
  pc.kb = kb;
}

// -P'(mu - c_t) per tile: FP64 dot of the FP32 factor with the FP32-rounded
// tile-relative mean, rounded once (the single-CTA kernel's formula), and
// -(mu - c_t) in FP32 for the statistics' d = x - mu.
template <int D, typename MuF>
__device__ __forceinline__ void tile_terms(MuF&& mean, const PairConsts<D>& pc,
                                           const double* __restrict__ ct, f2_t (&NB)[D],
                                           f2_t (&NMU)[D]) {
  float nbf[2][D], nm[2][D];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float muf[D];
#pragma unroll
    for (int q = 0; q < D; ++q) {
      const double mu = mean(c, q);  // 0 for a padding component
      muf[q] = static_cast<float>(mu - ct[q]);
      nm[c][q] = static_cast<float>(-(mu - ct[q]));
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q <= i; ++q) {
        const f2_t pij = pc.PP[i * (i + 1) / 2 + q];
        s = fma(static_cast<double>(c ? hi2(pij) : lo2(pij)), static_cast<double>(muf[q]), s);
      }
      nbf[c][i] = static_cast<float>(-s);
    }
  }
#pragma unroll
  for (int q = 0; q < D; ++q) {
    NB[q] = pk(nbf[0][q], nbf[1][q]);
    NMU[q] = pk(nm[0][q], nm[1][q]);
  }
}

// the chunk's means (FP64, [q][local component]) staged once per CTA: the
// per-tile terms then read shared memory instead of a global round trip
template <int D>
__device__ __forceinline__ void stage_means(const ModelBuf& mb, int k_cur, int kbase,
                                            double (*smu)[2 * kT]) {
  for (int i = threadIdx.x; i < 2 * kT; i += blockDim.x) {
    const int k = kbase + i;
#pragma unroll
    for (int q = 0; q < 4; ++q) smu[q][i] = k < k_cur ? mb.mu[k * 4 + q] : 0.0;
  }
  __syncthreads();
}

// Q + shift for both components of the pair (Q = -log2 of w N(x)):
// the single-CTA kernel's FFMA tree, started from nbase.
template <int D>
__device__ __forceinline__ f2_t dens_pair(const float4 x, const f2_t (&PP)[npacked(D)],
                                          const f2_t (&NB)[D], f2_t nbase) {
  const f2_t X0 = pk(x.x, x.x), X1 = pk(x.y, x.y), X2 = pk(x.z, x.z);
  const f2_t Y0 = fma2(PP[0], X0, NB[0]);
  const f2_t Y1 = fma2(PP[2], X1, fma2(PP[1], X0, NB[1]));
  const f2_t Y2 = fma2(PP[5], X2, fma2(PP[4], X1, fma2(PP[3], X0, NB[2])));
  f2_t qv = fma2(Y2, Y2, fma2(Y1, Y1, fma2(Y0, Y0, nbase)));
  if constexpr (D == 4) {
    const f2_t X3 = pk(x.w, x.w);
    const f2_t Y3 = fma2(PP[9], X3, fma2(PP[8], X2, fma2(PP[7], X1, fma2(PP[6], X0, NB[3]))));
    qv = fma2(Y3, Y3, qv);
  }
  return qv;
}

// L1 prefetch of a 128-point tile (2 KB of float4 points + the normalisers),
// issued a tile ahead by one warp: the first touch of a line from L2 costs
// hundreds of cycles that one point's work cannot cover
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void prefetch_tile(const float4* xt, const float2* lse, int t,
                                              int ntiles, int lane) {
  if (t >= ntiles) return;
  const char* xb = reinterpret_cast<const char*>(xt + static_cast<int64_t>(t) * kTile);
  if (lane < 16) prefetch_l1(xb + lane * 128);
  if (lse && lane >= 16 && lane < 24) {
    const char* lb = reinterpret_cast<const char*>(lse + static_cast<int64_t>(t) * kTile);
    prefetch_l1(lb + (lane - 16) * 128);
  }
}

// balanced contiguous sub-tile range of one (chunk, range) CTA
struct Range {
  int64_t g_begin, g_end;
};
__device__ __forceinline__ Range sub_range(int64_t n, int ntiles, int grp, int ngrp) {
  const int64_t last_pts = n - static_cast<int64_t>(ntiles - 1) * kTile;
  const int64_t total = static_cast<int64_t>(ntiles - 1) * kSPT + (last_pts + kP - 1) / kP;
  return Range{grp * total / ngrp, (grp + 1) * total / ngrp};
}

// ---- pass A: per-chunk per-point sums of e ---------------------------------
// NPR component pairs per thread (chunk = 512 NPR components): with 2 pairs
// the per-point warp reduce-scatter and the point loads serve 4 components.
// Tiles are staged in shared memory by cp.async one tile ahead.
#ifndef GMMB_LSE_NPR
#define GMMB_LSE_NPR 2
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}

template <int D, int NPR>
__global__ void __launch_bounds__(kT, NPR == 1 ? 3 : 2)
    lse_part_kernel(const float4* __restrict__ xt, const double* __restrict__ tc, int64_t n,
                    int ntiles, ModelBuf b0, ModelBuf b1, const EmState* __restrict__ st,
                    int nch, int64_t npad, float* __restrict__ part) {
  constexpr int CW = 2 * kT * NPR;  // components per chunk
  __shared__ float red[kT / 32][kTile];
  __shared__ __align__(16) float4 xs[2][kTile];
  __shared__ __align__(16) double cts[2][4];
  __shared__ double smu[4][CW];
  if (st->done) return;
  const int c = blockIdx.x % nch, grp = blockIdx.x / nch, ngrp = gridDim.x / nch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ModelBuf& mb = st->cur ? b1 : b0;
  const int k_cur = st->k_cur;
  PairConsts<D> pc[NPR];
#pragma unroll
  for (int h = 0; h < NPR; ++h)
    load_pair<D>(mb, k_cur, c * CW + h * 2 * kT + tid, c * CW + h * 2 * kT + kT + tid, pc[h]);
  for (int i = tid; i < CW; i += kT) {
    const int k = c * CW + i;
#pragma unroll
    for (int q = 0; q < 4; ++q) smu[q][i] = k < k_cur ? mb.mu[k * 4 + q] : 0.0;
  }
  const Range rg = sub_range(n, ntiles, grp, ngrp);
  const int t_first = static_cast<int>(rg.g_begin / kSPT);
  const int t_last = rg.g_end > rg.g_begin ? static_cast<int>((rg.g_end - 1) / kSPT) : t_first - 1;
  auto issue = [&](int t, int buf) {  // this thread's 16-byte pieces of tile t
    if (t <= t_last) {
      if (tid < kTile) cp_async16(&xs[buf][tid], xt + static_cast<int64_t>(t) * kTile + tid);
      else if (tid < kTile + 2) cp_async16(&cts[buf][2 * (tid - kTile)], tc + static_cast<int64_t>(t) * 4 + 2 * (tid - kTile));
    }
    cp_async_commit();
  };
  issue(t_first, 0);
  for (int t = t_first, ti = 0; t <= t_last; ++t, ++ti) {
    const int buf = ti & 1;
    issue(t + 1, buf ^ 1);
    cp_async_wait1();
    __syncthreads();  // tile t staged (every thread's pieces); smu written
    const int64_t tb0 = static_cast<int64_t>(t) * kSPT;
    const int s0 = static_cast<int>((rg.g_begin > tb0 ? rg.g_begin : tb0) - tb0);
    const int s1 = static_cast<int>((rg.g_end < tb0 + kSPT ? rg.g_end : tb0 + kSPT) - tb0);
    const double ct[4] = {cts[buf][0], cts[buf][1], cts[buf][2], cts[buf][3]};
    f2_t NB[NPR][D];
#pragma unroll
    for (int h = 0; h < NPR; ++h) {
      f2_t NMU[D];
      tile_terms<D>([&](int hh, int q) { return smu[q][h * 2 * kT + hh * kT + tid]; }, pc[h], ct,
                    NB[h], NMU);
    }
    for (int s = s0; s < s1; ++s) {
      float v[kP];
#pragma unroll
      for (int p = 0; p < kP; ++p) {
        const float4 x = xs[buf][s * kP + p];
        float e = 0.f;
#pragma unroll
        for (int h = 0; h < NPR; ++h) {
          const f2_t q = dens_pair<D>(x, pc[h].PP, NB[h], pc[h].NBASE);
          e += ex2n(lo2(q)) + ex2n(hi2(q));
        }
        v[p] = e;
      }
      const float r = warp_reduce_scatter<kP, false>(v, lane);
      if ((lane & 1) == 0) red[warp][s * kP + (lane >> 1)] = r;
    }
    __syncthreads();
    if (tid < kTile) {
      const int64_t i = static_cast<int64_t>(t) * kTile + tid;
      if (tid >= s0 * kP && tid < s1 * kP && i < n) {
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < kT / 32; ++w) sum += red[w][tid];
        part[c * npad + i] = sum;
      }
    }
    __syncthreads();  // red and the tile buffer are reused
  }
}

__global__ void lse_combine_kernel(const float* __restrict__ part, int nch, int64_t npad,
                                   int64_t n, const EmState* __restrict__ st,
                                   float2* __restrict__ lse, int* __restrict__ xlist,
                                   int* __restrict__ xcount, int exact_mode) {
  if (st->done) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = part[i];
  for (int c = 1; c < nch; ++c) s += part[c * npad + i];
  if (exact_mode || !(s >= 0x1p-64f && s <= 0x1p64f)) {
    xlist[atomicAdd(xcount, 1)] = static_cast<int>(i);
    lse[i] = make_float2(0.f, 0.f);
  } else {
    lse[i] = make_float2(0.f, lg2f(s));
  }
}

// exact log2-sum-exp of the listed points: one warp per point, lanes over
// components (lane l: l, l + 32, ...), max then shifted sum, fixed butterflies
template <int D>
__global__ void __launch_bounds__(256)
    lse_exact_kernel(const float4* __restrict__ xt, const double* __restrict__ tc, ModelBuf b0,
                     ModelBuf b1, const EmState* __restrict__ st, float2* __restrict__ lse,
                     const int* __restrict__ xlist, const int* __restrict__ xcount) {
  if (st->done) return;
  const int cnt = *xcount;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const ModelBuf& mb = st->cur ? b1 : b0;
  const int k_cur = st->k_cur;
  for (int q = gw; q < cnt; q += nw) {
    const int i = xlist[q];
    const float4 x = xt[i];
    const double* ct = tc + static_cast<int64_t>(i / kTile) * 4;
    auto neg_q = [&](int k) {  // -Q of component k (the pair formula, lane lo)
      PairConsts<D> pc;
      load_pair<D>(mb, k_cur, k, k_cur, pc);
      f2_t NB[D], NMU[D];
      tile_terms<D>([&](int h, int q) { return h == 0 ? mb.mu[k * 4 + q] : 0.0; }, pc, ct, NB,
                    NMU);
      return -lo2(dens_pair<D>(x, pc.PP, NB, pc.NBASE));
    };
    float m = -INFINITY;
    for (int k = lane; k < k_cur; k += 32) m = fmaxf(m, neg_q(k));
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float sum = 0.f;
    if (m > -INFINITY)
      for (int k = lane; k < k_cur; k += 32) sum += ex2f(neg_q(k) - m);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    // kept apart: m = -Q_min is bitwise the dominant component's -Q, so pass
    // B forms Q - Q_min exactly before adding the small log2 of the sum
    if (lane == 0) lse[i] = make_float2(m, lg2f(sum));
  }
}

// ---- pass B: statistics with the known normaliser ---------------------------
template <int D>
__global__ void __launch_bounds__(kT, 2)
    stats_chunk_kernel(const float4* __restrict__ xt, const double* __restrict__ tc, int64_t n,
                       int ntiles, ModelBuf b0, ModelBuf b1, const EmState* __restrict__ st,
                       int nch, int kpad, const float2* __restrict__ lse,
                       double* __restrict__ partials, double* __restrict__ ll_part) {
  constexpr int NS = nstats(D);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* acc64 = reinterpret_cast<double2*>(smem_raw);  // [NS][kT]
  double (*smu)[2 * kT] = reinterpret_cast<double (*)[2 * kT]>(acc64 + NS * kT);
  if (st->done) return;
  const int c = blockIdx.x % nch, grp = blockIdx.x / nch, ngrp = gridDim.x / nch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ModelBuf& mb = st->cur ? b1 : b0;
  const int k_cur = st->k_cur;
  PairConsts<D> pc;
  load_pair<D>(mb, k_cur, c * 2 * kT + tid, c * 2 * kT + kT + tid, pc);
  stage_means<D>(mb, k_cur, c * 2 * kT, smu);
  auto mean = [&](int h, int q) { return smu[q][h * kT + tid]; };
  f2_t ACC[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    ACC[s] = 0ull;
    acc64[s * kT + tid] = make_double2(0.0, 0.0);
  }
  auto promote = [&]() {  // FP32 register sums -> FP64 shared accumulators
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      double2 v = acc64[s * kT + tid];
      v.x += f32_to_f64(lo2(ACC[s]));
      v.y += f32_to_f64(hi2(ACC[s]));
      ACC[s] = 0ull;
      acc64[s * kT + tid] = v;
    }
  };
  const bool ll_warp = c == 0 && warp == 0;
  double ll = 0.0;
  const Range rg = sub_range(n, ntiles, grp, ngrp);
  for (int64_t g = rg.g_begin; g < rg.g_end;) {
    const int t = static_cast<int>(g / kSPT);
    const int s0 = static_cast<int>(g - static_cast<int64_t>(t) * kSPT);
    const int64_t tend = static_cast<int64_t>(t + 1) * kSPT;
    const int s1 = static_cast<int>((rg.g_end < tend ? rg.g_end : tend) - static_cast<int64_t>(t) * kSPT);
    const int64_t base = static_cast<int64_t>(t) * kTile;
    const int p0 = s0 * kP;
    const int p1 = static_cast<int>(min64(static_cast<int64_t>(s1) * kP, n - base));
    double ct[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ct[q] = __ldg(tc + static_cast<int64_t>(t) * 4 + q);
    f2_t NB[D], NMU[D];
    tile_terms<D>(mean, pc, ct, NB, NMU);
    const float4* xs = xt + base;
    const float2* ls = lse + base;
    if (warp == 0) prefetch_tile(xt, lse, t + 1, ntiles, lane);
    // responsibilities of a point for the pair: common case (L.x = 0) the
    // shift starts the FFMA chain; a far point (L.x = -Q_min, warp-uniform
    // branch) takes Q first, then Q - Q_min, then the small remainder, as
    // the exact path of the single-CTA kernel
    auto resp = [&](const float4 x, const float2 L) {
      const bool far = L.x != 0.f;
      f2_t q = dens_pair<D>(x, pc.PP, NB, far ? pc.NBASE : add2(pc.NBASE, pk(L.y, L.y)));
      if (far) q = add2(add2(q, pk(L.x, L.x)), pk(L.y, L.y));
      return pk(ex2n(lo2(q)), ex2n(hi2(q)));
    };
    auto accum = [&](const float4 x, const f2_t R) {
      const float xv[4] = {x.x, x.y, x.z, x.w};
      f2_t DD[D], W[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        DD[i] = add2(pk(xv[i], xv[i]), NMU[i]);
        W[i] = mul2(R, DD[i]);
      }
      ACC[0] = add2(ACC[0], R);
#pragma unroll
      for (int i = 0; i < D; ++i) ACC[1 + i] = add2(ACC[1 + i], W[i]);
      int qq = 1 + D;
#pragma unroll
      for (int i = 0; i < D; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
          ACC[qq] = fma2(W[i], DD[j], ACC[qq]);
          ++qq;
        }
      }
    };
    // two points per step: their density chains are independent, so the
    // FFMA2 / MUFU latencies of one hide behind the other's work
    int p = p0;
    for (; p + 1 < p1; p += 2) {
      const float4 xa = __ldg(xs + p), xb = __ldg(xs + p + 1);
      const float2 La = __ldg(ls + p), Lb = __ldg(ls + p + 1);
      const f2_t Ra = resp(xa, La), Rb = resp(xb, Lb);
      accum(xa, Ra);
      accum(xb, Rb);
      if ((p & (kP - 1)) == kP - 2) promote();  // every 16 points (sub-tile aligned)
    }
    if (p < p1) {
      const float4 x = __ldg(xs + p);
      accum(x, resp(x, __ldg(ls + p)));
    }
    if ((p1 & (kP - 1)) != 0) promote();        // a partial last sub-tile
    if (ll_warp) {
      for (int p = p0 + lane; p < p1; p += 32) {
        const float2 L = __ldg(ls + p);
        ll += static_cast<double>(L.x) + static_cast<double>(L.y);
      }
    }
    g = static_cast<int64_t>(t) * kSPT + s1;
  }
  const int ks[2] = {pc.ka, pc.kb};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (ks[h] < kpad) {
      double* out = partials + (static_cast<int64_t>(grp) * kpad + ks[h]) * NS;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double2 v = acc64[s * kT + tid];
        out[s] = h ? v.y : v.x;
      }
    }
  }
  if (ll_warp) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, off);
    if (lane == 0) ll_part[grp] = ll * kLn2;
  }
}

template <int D>
cudaError_t launch_d(const PointsDev& pts, const ModelBuf* bufs, const EmState* st, int k0,
                     double* partials, double* ll_part, int exact_mode, int sm_count,
                     cudaStream_t s, int* ncl_out, const ChunkScratch* scr) {
  const int nch = (k0 + 2 * kT - 1) / (2 * kT);
  constexpr int NS = nstats(D);
  const size_t smem_b = sizeof(double2) * NS * kT + sizeof(double) * 4 * 2 * kT;
  static int occ_dev[64][2] = {};  // co-resident CTAs per SM (pass A, pass B) per device
  int dev = 0;
  cudaGetDevice(&dev);
  int* occ = occ_dev[dev & 63];
  if (occ[0] == 0) {
    cudaError_t e = cudaFuncSetAttribute(stats_chunk_kernel<D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_b));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[0], lse_part_kernel<D, GMMB_LSE_NPR>,
                                                      kT, 0);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[1], stats_chunk_kernel<D>, kT, smem_b);
    if (e != cudaSuccess) return e;
    if (occ[0] < 1) occ[0] = 1;
    if (occ[1] < 1) occ[1] = 1;
  }
  // point ranges: one co-resident wave of (chunk, range) CTAs
  auto groups = [&](int per_sm) {
    int g = sm_count * per_sm / nch;
    if (g < 1) g = 1;
    const int64_t total_sub = (pts.n + kP - 1) / kP;
    if (g > total_sub) g = static_cast<int>(total_sub);
    return g;
  };
  constexpr int CWA = 2 * kT * GMMB_LSE_NPR;  // pass A chunk
  const int ncha = (k0 + CWA - 1) / CWA;
  auto groups_a = [&](int per_sm) {
    int g = sm_count * per_sm / ncha;
    if (g < 1) g = 1;
    const int64_t total_sub = (pts.n + kP - 1) / kP;
    if (g > total_sub) g = static_cast<int>(total_sub);
    return g;
  };
  const int ga = groups_a(occ[0]), gb = groups(occ[1]);
#if GMMB_CHUNK_WS
  // pass B on the warp-specialised kernel (one CTA per SM)
  {
    const cudaError_t e = launch_estep_ws_pre(pts, bufs, st, k0, nch, nullptr, nullptr, nullptr,
                                              sm_count, s, ncl_out);
    if (e != cudaSuccess) return e;
  }
#else
  *ncl_out = gb;
#endif
  if (!partials) return cudaSuccess;  // size query
  const int64_t npad = static_cast<int64_t>(pts.ntiles) * kTile;
  cudaError_t e = cudaMemsetAsync(scr->xcount, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  lse_part_kernel<D, GMMB_LSE_NPR><<<ncha * ga, kT, 0, s>>>(
      pts.xt, pts.tc, pts.n, pts.ntiles, bufs[0], bufs[1], st, ncha, npad, scr->part);
  lse_combine_kernel<<<static_cast<int>((pts.n + 255) / 256), 256, 0, s>>>(
      scr->part, ncha, npad, pts.n, st, scr->lse, scr->xlist, scr->xcount, exact_mode);
  lse_exact_kernel<D><<<sm_count, 256, 0, s>>>(pts.xt, pts.tc, bufs[0], bufs[1], st, scr->lse,
                                               scr->xlist, scr->xcount);
#if GMMB_CHUNK_WS
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int ncl = 0;
  return launch_estep_ws_pre(pts, bufs, st, k0, nch, scr->lse, partials, ll_part, sm_count, s,
                             &ncl);
#else
  stats_chunk_kernel<D><<<nch * gb, kT, smem_b, s>>>(pts.xt, pts.tc, pts.n, pts.ntiles, bufs[0],
                                                      bufs[1], st, nch, k0, scr->lse, partials,
                                                      ll_part);
  return cudaGetLastError();
#endif
}

}  // namespace

size_t chunk_scratch_floats(int k0, int64_t n) {
  const int64_t npad = (n + kTile - 1) / kTile * kTile;
  const int nch = (k0 + 2 * kT - 1) / (2 * kT);
  return static_cast<size_t>(npad) * (nch + 2);  // part[nch][npad] + lse float2[npad]
}

cudaError_t launch_estep_chunked(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                                 int k0, double* partials, double* ll_part, int exact_mode,
                                 int sm_count, cudaStream_t s, int* ncl_out,
                                 const ChunkScratch* scr) {
  if (pts.d == 4)
    return launch_d<4>(pts, bufs, st, k0, partials, ll_part, exact_mode, sm_count, s, ncl_out, scr);
  return launch_d<3>(pts, bufs, st, k0, partials, ll_part, exact_mode, sm_count, s, ncl_out, scr);
}

}  // namespace gmmb
