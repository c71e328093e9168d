// em_kernels.cu — the EM hot path on sm_100a.
//
// Reference semantics (paths under /root/reference/proj):
//   cholesky_cache          src/gmm.cpp:33-48, src/kernels.cpp:10-77
//   e_step_into             src/sogmm.cpp:341-383, logsumexp_rows kernels.cpp:104-135
//   m_step_impl             src/sogmm.cpp:399-455, weighted_moments_fn kernels.hpp:82-181
//   EM loop bookkeeping     src/sogmm.cpp:484-509
//
// The fused kernel never materialises the N x K responsibility matrix: a CTA
// owns up to 512 components (one per thread; K > 512 uses a thread-block
// cluster whose CTAs split the components and exchange per-point
// log-sum-exp partials through distributed shared memory), streams
// 128-point tiles of spatially sorted, tile-recentred FP32 points through
// shared memory, evaluates log2-domain log densities in FP32 registers,
// normalises them with warp reduce-scatter butterflies + a CTA combine,
// and accumulates the centred sufficient statistics (sum r, sum r d,
// sum r d d^T, d = x - mu_old) in FP32 registers, promoted to FP64 every
// tile. Per-cluster FP64 partials are reduced in a fixed order by a second
// kernel, so results are bit-reproducible run to run.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "em_kernels.cuh"
#include "factor.cuh"
#include "f32x2.cuh"

namespace cg = cooperative_groups;

// Precision / schedule switches (defaults = production).
#ifndef GMMB_REDUCE_CTA_NCL
#define GMMB_REDUCE_CTA_NCL 256  // above this many partials per component: a CTA per component
#endif
#ifndef GMMB_FLUSH_SUBTILES
#define GMMB_FLUSH_SUBTILES 2   // 8-point groups per FP32 -> FP64 promotion
#endif
#ifndef GMMB_PIPE
#define GMMB_PIPE 1             // 1: warp-specialised packed kernel when one CTA holds all K
#endif
#ifndef GMMB_WS_P
#define GMMB_WS_P 16            // points per sub-tile of the warp-specialised kernel
#endif
#ifndef GMMB_F2F_ALU
#define GMMB_F2F_ALU 0          // 1: FP32 -> FP64 widening on the integer ALU
#endif
#ifndef GMMB_CHUNKED
#define GMMB_CHUNKED 1          // 1: K > 512 through the chunked two-pass kernels
#endif
#ifndef GMMB_PXB
#define GMMB_PXB 1              // 1: y = P'x - P'mu (FFMA chains); 0: y = P'(x - mu)
#endif

namespace gmmb {

namespace {

using namespace dev;



// ---------------------------------------------------------------------------
// Fused E-step + sufficient statistics.
// ---------------------------------------------------------------------------
template <int D, int NW, int C, int P>
struct EstepSmem {
  float4 xs[kTile];
  float red[2][P][NW];    // per-warp partials per point, double-buffered
  float xm[2][P];         // cluster exchange: CTA max per point
  float xsum[2][P];       // cluster exchange: CTA sum per point
};

// Combines the NW per-warp partials of P points inside one warp: lane
// (p = lane / G, q = lane % G), G = 32 / P, folds warps q, q+G, ... in
// order, then log2(G) xor steps. Every warp computes the identical
// (order-fixed) value.
template <int NW, int P, bool MAX>
__device__ __forceinline__ float cta_combine(const float (&red)[P][NW], int lane) {
  constexpr int G = 32 / P;  // lanes per point
  const int p = lane / G, q = lane % G;
  float v = MAX ? -INFINITY : 0.f;
#pragma unroll
  for (int w = q; w < NW; w += G) v = MAX ? fmaxf(v, red[p][w]) : v + red[p][w];
#pragma unroll
  for (int off = 1; off < G; off <<= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, v, off);
    v = MAX ? fmaxf(v, o) : v + o;
  }
  return v;
}

// Cluster-wide combine of per-CTA values xs[p][rank]: lane (p, q) folds
// ranks q, q+4, then two xor steps (fixed order on every CTA).
template <int C, bool MAX>
__device__ __forceinline__ float cluster_combine(float* local_slot, int lane) {
  cg::cluster_group cl = cg::this_cluster();
  const int q = lane & 3;
  float v = MAX ? -INFINITY : 0.f;
#pragma unroll
  for (int r = q; r < C; r += 4) {
    const float o = *cl.map_shared_rank(local_slot, r);
    v = MAX ? fmaxf(v, o) : v + o;
  }
#pragma unroll
  for (int off = 1; off <= 2; off <<= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, v, off);
    v = MAX ? fmaxf(v, o) : v + o;
  }
  return v;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}


// CPT components per thread: thread tid of CTA rank r owns components
// r * kCtaComps + c * (32 NW) + tid, c < CPT. Per 8-point sub-tile: phase A
// (log2 densities), phase B (normalise: one CTA barrier, every warp combines
// the per-warp partials itself; clusters add one cluster barrier), phase C
// (responsibilities + statistics centred at the previous means).
//
// Phase A evaluates y = P'x - P'mu' as FFMA chains (P'mu' is formed once
// per tile in FP64), so a unit costs 10 + D FFMA (D = 4) instead of
// D FADD + D FMUL + 6 FFMA + D FFMA. Phase B sums ex2(l) with no shift: the
// log2 densities of any point that matters lie far inside FP32's exponent
// range; a sub-tile whose sum leaves [2^-64, 2^64] (outliers far from every
// component) is redone with the exact max shift.
template <int D, int NW, int C, int P, int CPT>
__global__ void __launch_bounds__(NW * 32, 16 / NW)
    estep_stats_kernel(const float4* __restrict__ xt,
                       const double* __restrict__ tc, int64_t n, int ntiles,
                       ModelBuf b0, ModelBuf b1, const EmState* __restrict__ st,
                       int kpad, double* __restrict__ partials,
                       double* __restrict__ ll_part, int exact_mode) {
  constexpr int NP = npacked(D);
  constexpr int NS = nstats(D);
  constexpr int T = NW * 32;
  using Smem = EstepSmem<D, NW, C, P>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);


  if (st->done) return;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  // FP64 accumulators, stat pairs as double2 [(c * NSP + s / 2) * T + tid]:
  // conflict-free 16-byte shared loads/stores when promoting
  constexpr int NSP = (NS + 1) / 2;
  double2* acc64 = reinterpret_cast<double2*>(smem_raw + ((sizeof(Smem) + 15) & ~size_t(15)));
  auto promote = [&](float (&a)[CPT][NS]) {
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
      for (int s2 = 0; s2 < NSP; ++s2) {
        double2 v = acc64[(c * NSP + s2) * T + tid];
        v.x += static_cast<double>(a[c][2 * s2]);
        a[c][2 * s2] = 0.f;
        if (2 * s2 + 1 < NS) {
          v.y += static_cast<double>(a[c][2 * s2 + 1]);
          a[c][2 * s2 + 1] = 0.f;
        }
        acc64[(c * NSP + s2) * T + tid] = v;
      }
  };  int rank = 0, cid = blockIdx.x, ncl = gridDim.x;
  if constexpr (C > 1) {
    rank = static_cast<int>(cg::this_cluster().block_rank());
    cid = blockIdx.x / C;
    ncl = gridDim.x / C;
  }
  const int k_cur = st->k_cur;
  const ModelBuf& mb = st->cur ? b1 : b0;

  // component constants in registers
  float pp[CPT][NP];
  float base2[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int k = rank * kCtaComps + c * T + tid;
    base2[c] = -INFINITY;
#pragma unroll
    for (int j = 0; j < NP; ++j) pp[c][j] = 0.f;
    if (k < k_cur) {
      const float4* c4 = reinterpret_cast<const float4*>(mb.cst + k);
      float cc[12];
      const float4 a = c4[0], b = c4[1], e = c4[2];
      cc[0] = a.x; cc[1] = a.y; cc[2] = a.z; cc[3] = a.w;
      cc[4] = b.x; cc[5] = b.y; cc[6] = b.z; cc[7] = b.w;
      cc[8] = e.x; cc[9] = e.y; cc[10] = e.z; cc[11] = e.w;
#pragma unroll
      for (int j = 0; j < NP; ++j) pp[c][j] = cc[j];
      base2[c] = cc[10];
    }
  }

  float acc[CPT][NS];
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[c][s] = 0.f;
#pragma unroll
  for (int i = 0; i < CPT * NSP; ++i) acc64[i * T + tid] = make_double2(0.0, 0.0);
  double ll_acc = 0.0;   // warp 0, lanes with lane % 4 == 0 (one point each)
  int rb = 0;            // red[] buffer rotation (one flip per CTA barrier)
  int xb = 0;            // cluster exchange buffer rotation
  const bool finisher = warp == 0 && (lane & 3) == 0;
  const int fp = lane >> 2;  // point of this lane's group

  for (int t = cid; t < ntiles; t += ncl) {
    const int64_t t0 = static_cast<int64_t>(t) * kTile;
    const int npts = static_cast<int>(min64(kTile, n - t0));
    __syncthreads();  // previous tile fully consumed
    for (int i = tid; i < kTile; i += T) {
      sm.xs[i] = i < npts ? xt[t0 + i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // tile-relative means mu' = fp32(mu - c_t) and nb = -P' mu' (FP64 dot)
    float muf[CPT][D];
    float nb[CPT][D];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int k = rank * kCtaComps + c * T + tid;
      double rel[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double m = k < k_cur ? mb.mu[k * 4 + j] : 0.0;
        rel[j] = m - tc[static_cast<int64_t>(t) * 4 + j];
        muf[c][j] = static_cast<float>(rel[j]);
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j <= i; ++j) {
          s = fma(static_cast<double>(pp[c][i * (i + 1) / 2 + j]),
                  static_cast<double>(muf[c][j]), s);
        }
        nb[c][i] = static_cast<float>(-s);
      }
    }
    __syncthreads();

    for (int q = 0; q < npts; q += P) {
      // ---- phase A: log2 densities l = base2 - |y|^2 ----
      float l[CPT][P], e[CPT][P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float4 x = sm.xs[q + p];
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
#if GMMB_PXB
          const float y0 = fmaf(pp[c][0], x.x, nb[c][0]);
          const float y1 = fmaf(pp[c][2], x.y, fmaf(pp[c][1], x.x, nb[c][1]));
          const float y2 = fmaf(pp[c][5], x.z, fmaf(pp[c][4], x.y, fmaf(pp[c][3], x.x, nb[c][2])));
#else
          const float d0 = x.x - muf[c][0], d1 = x.y - muf[c][1], d2 = x.z - muf[c][2];
          const float y0 = pp[c][0] * d0;
          const float y1 = fmaf(pp[c][2], d1, pp[c][1] * d0);
          const float y2 = fmaf(pp[c][5], d2, fmaf(pp[c][4], d1, pp[c][3] * d0));
#endif
          float lv = fmaf(-y2, y2, fmaf(-y1, y1, fmaf(-y0, y0, base2[c])));
          if constexpr (D == 4) {
#if GMMB_PXB
            const float y3 = fmaf(pp[c][9], x.w, fmaf(pp[c][8], x.z,
                                  fmaf(pp[c][7], x.y, fmaf(pp[c][6], x.x, nb[c][3]))));
#else
            const float d3 = x.w - muf[c][3];
            const float y3 = fmaf(pp[c][9], d3, fmaf(pp[c][8], d2, fmaf(pp[c][7], d1, pp[c][6] * d0)));
#endif
            lv = fmaf(-y3, y3, lv);
          }
          l[c][p] = lv;
        }
      }
      const bool valid_g = q + fp < npts;  // this lane group's point
      float S = 1.f, M = 0.f;              // lane group's sum and shift
      bool exact = exact_mode != 0;
      if (!exact) {
        // ---- phase B: unshifted sum of 2^l over all components ----
        float v[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          v[p] = 0.f;
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            e[c][p] = ex2f(l[c][p]);
            v[p] += e[c][p];
          }
        }
        const float r = warp_reduce_scatter<P, false>(v, lane);
        if ((lane & 3) == 0) sm.red[rb][lane >> 2][warp] = r;
        __syncthreads();
        S = cta_combine<NW, P, false>(sm.red[rb], lane);
        rb ^= 1;
        if constexpr (C > 1) {
          if (finisher) sm.xsum[xb][fp] = S;
          cluster_sync_all();
          S = cluster_combine<C, false>(&sm.xsum[xb][fp], lane);
          xb ^= 1;
        }
        // identical inputs in every warp => warp-, CTA- and cluster-uniform
        exact = __any_sync(0xffffffffu, valid_g && !(S >= 0x1p-64f && S <= 0x1p64f));
      }
      if (exact) {
        // ---- exact max-shift path (forced, or the plain sum left range) ----
        float v[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          v[p] = l[0][p];
#pragma unroll
          for (int c = 1; c < CPT; ++c) v[p] = fmaxf(v[p], l[c][p]);
        }
        float r = warp_reduce_scatter<P, true>(v, lane);
        if ((lane & 3) == 0) sm.red[rb][lane >> 2][warp] = r;
        __syncthreads();
        M = cta_combine<NW, P, true>(sm.red[rb], lane);
        rb ^= 1;
        if constexpr (C > 1) {
          if (finisher) sm.xm[xb][fp] = M;
          cluster_sync_all();
          M = cluster_combine<C, true>(&sm.xm[xb][fp], lane);
          xb ^= 1;
        }
        M = M == -INFINITY ? 0.f : M;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float mp = __shfl_sync(0xffffffffu, M, p * 4);
          v[p] = 0.f;
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            e[c][p] = ex2f(l[c][p] - mp);
            v[p] += e[c][p];
          }
        }
        r = warp_reduce_scatter<P, false>(v, lane);
        if ((lane & 3) == 0) sm.red[rb][lane >> 2][warp] = r;
        __syncthreads();
        S = cta_combine<NW, P, false>(sm.red[rb], lane);
        rb ^= 1;
        if constexpr (C > 1) {
          if (finisher) sm.xsum[xb][fp] = S;
          cluster_sync_all();
          S = cluster_combine<C, false>(&sm.xsum[xb][fp], lane);
          xb ^= 1;
        }
      }
      if (finisher && valid_g && rank == 0) ll_acc += static_cast<double>(M + lg2f(S));
      const float scale_g = valid_g ? rcpf(S) : 0.f;
      // ---- phase C: responsibilities and statistics centred at mu_old ----
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float sc = __shfl_sync(0xffffffffu, scale_g, p * 4);
        const float4 x = sm.xs[q + p];
        const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const float r = e[c][p] * sc;
          float dd[D], w[D];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            dd[j] = xv[j] - muf[c][j];
            w[j] = r * dd[j];
          }
          acc[c][0] += r;
#pragma unroll
          for (int j = 0; j < D; ++j) acc[c][1 + j] += w[j];
          int s = 1 + D;
#pragma unroll
          for (int i = 0; i < D; ++i) {
#pragma unroll
            for (int j = 0; j <= i; ++j) {
              acc[c][s] = fmaf(w[i], dd[j], acc[c][s]);
              ++s;
            }
          }
        }
      }
      if (GMMB_FLUSH_SUBTILES < 16 && ((q / P + 1) % GMMB_FLUSH_SUBTILES) == 0) promote(acc);
    }
    promote(acc);  // the tile's remaining FP32 partial sums
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int k = rank * kCtaComps + c * T + tid;
    if (k < kpad) {
      double* out = partials + (static_cast<int64_t>(cid) * kpad + k) * NS;
#pragma unroll
      for (int s2 = 0; s2 < NSP; ++s2) {
        const double2 v = acc64[(c * NSP + s2) * T + tid];
        out[2 * s2] = v.x;
        if (2 * s2 + 1 < NS) out[2 * s2 + 1] = v.y;
      }
    }
  }
  if (warp == 0) {  // ll partial of this cluster: the 8 finisher lanes, in order
    double s = 0.0;
#pragma unroll
    for (int p = 0; p < P; ++p) s += __shfl_sync(0xffffffffu, ll_acc, p * 4);
    if (lane == 0 && rank == 0) ll_part[cid] = s * kLn2;
  }
  if constexpr (C > 1) {
    // keep smem alive until every CTA of the cluster finished its DSMEM reads
    cg::this_cluster().sync();
  }
}
// ---------------------------------------------------------------------------
// Packed, software-pipelined fused E step (one CTA holds all K <= 512
// components; thread tid owns the component pair (tid, T + tid)).
//
// * Packed FP32: every per-(point, component) operation is identical for the
//   thread's two components, so phases A and C run on f32x2 register pairs
//   (FFMA2 / FADD2 / FMUL2: 64 lane-operations per warp instruction; B200
//   reaches its 74 TFLOP/s FP32 peak only through this form, and it issues
//   half the instructions). Points enter as scalar broadcast operands.
// * Phase A evaluates q - base = |P'x - P'mu'|^2 - base with FFMA chains
//   (P'mu' formed once per tile in FP64); e = 2^-(q - base) on the MUFU.
// * Phase B sums e with no shift: log2 densities of any point that matters
//   lie far inside FP32's exponent range; a sub-tile whose sum leaves
//   [2^-64, 2^64] is redone with the exact max shift (CTA-uniform decision).
// * Software pipelining: the CTA-wide sum of sub-tile s is posted to a ring
//   slot + mbarrier, and the thread computes the densities of s+1 before
//   waiting for s, so shuffle/barrier latency hides behind FFMA work. Three
//   slots suffice: a thread that writes slot s % 3 has passed the wait for
//   s - 1, so every thread has finished reading sub-tile s - 3.
// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// Warp-specialised fused E step (one CTA holds all K <= 512 components).
//
// Producer warps own the log densities, consumer warps own the statistics:
//   producer thread j (component pair j, T + j), per P-point sub-tile:
//     Q = |P'x - P'mu'|^2 - base2 (FFMA chains; P'mu' = P'mu - P'c_t per
//     tile in FP64), e = 2^-Q (MUFU), e pairs -> e ring slot, a warp
//     reduce-scatter of the per-point sums -> red ring slot, arrive full;
//   consumer thread j: wait full, combine the per-warp partials (fixed
//     order) into S, copy its e pairs, arrive empty, then r = e / S and the
//     centred statistics sum r, sum r d, sum r d d^T (d = x - mu_old) in FP32
//     pairs, promoted to FP64 shared memory every GMMB_FLUSH_SUBTILES
//     sub-tiles.
// Point tiles (2 KB) and tile centres arrive by TMA bulk copies into a
// double buffer, issued a tile ahead by one producer thread.
// Every per-(point, component) operation is identical for a thread's two
// components, so both roles run on f32x2 register pairs (FFMA2 / FADD2 /
// FMUL2): B200 reaches its FP32 peak only through that form, and it issues
// half the instructions. Splitting the roles halves each thread's live
// registers, which keeps enough independent FFMA2 chains in flight.
//
// The normaliser is an unshifted sum: the log2 densities of any point that
// matters lie far inside FP32's exponent range. A sub-tile whose sum leaves
// [2^-64, 2^64] (outliers far from every component) is redone by the
// consumers with the exact max shift (uniform decision: S is identical in
// every consumer warp), reloading the constants from global memory.
// ---------------------------------------------------------------------------
#ifndef GMMB_RING
#define GMMB_RING 4
#endif
// sub-tile slots in flight between the roles: 4 for one CTA (measured ~1 %
// faster than 3); the cluster kernels keep 3 (their shared memory is larger,
// and K = 2048 measured 3 % slower with 4)
template <int C>
constexpr int ring_slots() {
  return C > 1 ? (GMMB_RING < 3 ? GMMB_RING : 3) : GMMB_RING;
}

template <int NWH, int P, int C>
struct WsSmem {
  float4 xs[2][kTile];                   // point tiles (TMA destination)
  double tcs[2][4];                      // tile centres (TMA destination)
  float2 ls[2][kTile];                   // PRE: the tile's log2 normalisers (TMA destination)
  static constexpr int kRing = ring_slots<C>();
  float4 ering[kRing][P / 2][NWH * 32];  // e pairs: [slot][point pair][thread]
  float red[kRing][P][C * NWH];          // per-warp partial sums of every CTA of the cluster
  float xred[2][P][C * NWH];             // consumer exact-path scratch
  double mu[4][2 * NWH * 32];            // mu (FP64), [q][component of this CTA]
  unsigned long long full[kRing], empty[kRing], xs_full[2], xs_free[2], xbar[2];
};

// distributed shared memory (thread-block clusters)
__device__ __forceinline__ unsigned mapa_u32(unsigned addr, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(unsigned addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(unsigned addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* b, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}


// PRE (pass B of the chunked K > 512 E step, estep_chunked.cu): the
// per-point log2 normalisers L_n over ALL K are known (pass A), so the CTA
// holds one 512-component chunk c = blockIdx.x % nch of them; producers
// emit r = 2^-(Q + L_n) directly (no reduce-scatter, no per-warp partials),
// consumers accumulate with no combine / rescale / exact path.
template <int D, int NWH, int P, int C, bool PRE = false>
__global__ void __launch_bounds__(2 * NWH * 32, 8 / NWH)
    estep_ws_kernel(const float4* __restrict__ xt, const double* __restrict__ tc,
                    int64_t n, int ntiles, ModelBuf b0, ModelBuf b1,
                    const EmState* __restrict__ st, int kpad,
                    double* __restrict__ partials, double* __restrict__ ll_part,
                    int exact_mode, int split_sub, const float2* __restrict__ lse = nullptr,
                    int nch = 1) {
  static_assert(!PRE || C == 1, "pre-normalised pass: one CTA per chunk");
  constexpr int NP = npacked(D);
  constexpr int NS = nstats(D);
  constexpr int T = NWH * 32;  // threads per role
  constexpr int G = 32 / P;    // lanes per point after the warp reduce-scatter
  constexpr int NWC = C * NWH; // producer warps of the cluster
  using Smem = WsSmem<NWH, P, C>;
  constexpr int kRing = Smem::kRing;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  // consumer FP64 accumulators: acc64[s * T + j] = (component j, component T + j)
  double2* acc64 = reinterpret_cast<double2*>(smem_raw + ((sizeof(Smem) + 15) & ~size_t(15)));

  if (st->done) return;
  const bool producer = threadIdx.x < T;
  const int lane = (threadIdx.x % T) & 31;
  const int warp = (threadIdx.x % T) >> 5;
  // K > 512: a cluster of C CTAs splits the components; every CTA streams
  // the same tiles and the per-point sums go to every CTA through DSMEM
  int rank = 0, cid = blockIdx.x, ncl = gridDim.x;
  if constexpr (C > 1) {
    rank = static_cast<int>(cg::this_cluster().block_rank());
    cid = blockIdx.x / C;
    ncl = gridDim.x / C;
  }
  int chunk = 0;
  if constexpr (PRE) {
    chunk = blockIdx.x % nch;
    cid = blockIdx.x / nch;
    ncl = gridDim.x / nch;
  }
  // component pair (rank * 2T + j, rank * 2T + T + j); j is the local index
  const int j = static_cast<int>(threadIdx.x) % T;
  const int kb = (PRE ? chunk : rank) * 2 * T;
  const int k_cur = st->k_cur;
  const ModelBuf& mb = st->cur ? b1 : b0;
  constexpr unsigned kTileBytes =
      kTile * sizeof(float4) + 4 * sizeof(double) + (PRE ? kTile * sizeof(float2) : 0);
  auto issue_tile = [&](int t, int buf) {  // one thread: TMA bulk copy of tile t
    mbar_expect_tx(&sm.xs_full[buf], kTileBytes);
    bulk_g2s(sm.xs[buf], xt + static_cast<int64_t>(t) * kTile, kTile * sizeof(float4),
             &sm.xs_full[buf]);
    bulk_g2s(sm.tcs[buf], tc + static_cast<int64_t>(t) * 4, 4 * sizeof(double), &sm.xs_full[buf]);
    if constexpr (PRE)
      bulk_g2s(sm.ls[buf], lse + static_cast<int64_t>(t) * kTile, kTile * sizeof(float2),
               &sm.xs_full[buf]);
  };
  // Each CTA (cluster) takes a contiguous, balanced range of P-point
  // sub-tiles (a round-robin over 128-point tiles leaves 16 or 17 tiles per
  // CTA on cfg2: a 5 % tail); the first and last tiles of a range may be
  // partial. Sub-tile g is sub-tile g % SPT of tile g / SPT. With several
  // CTAs per SM (small K) the SM averages its CTAs' imbalance, and the
  // round-robin over whole tiles measured faster (split_sub = 0).
  constexpr int SPT = kTile / P;
  const int64_t last_pts = n - static_cast<int64_t>(ntiles - 1) * kTile;
  const int64_t total_sub = static_cast<int64_t>(ntiles - 1) * SPT + (last_pts + P - 1) / P;
  // range boundaries floor(c * units / ncl): sizes differ by at most one
  const int64_t g_begin = static_cast<int64_t>(cid) * total_sub / ncl;
  const int64_t g_end = static_cast<int64_t>(cid + 1) * total_sub / ncl;
  const int t_first = static_cast<int>(g_begin / SPT);
  const int t_last = g_end > g_begin ? static_cast<int>((g_end - 1) / SPT) : t_first - 1;
  // this CTA's tiles: ti-th tile, and the sub-tiles [s0, s1) it processes
  const int ntiles_cta = split_sub ? t_last - t_first + 1
                                   : (cid < ntiles ? (ntiles - 1 - cid) / ncl + 1 : 0);
  auto tile_of = [&](int ti) { return split_sub ? t_first + ti : cid + ti * ncl; };
  auto sub_range = [&](int t, int nsub, int& s0, int& s1) {
    s0 = 0;
    s1 = nsub;
    if (split_sub) {
      if (t == t_first) s0 = static_cast<int>(g_begin % SPT);
      if (t == t_last) s1 = static_cast<int>((g_end - 1) % SPT) + 1;
    }
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kRing; ++i) {
      // C > 1: one arrival per warp of every CTA of the cluster; C = 1: per thread
      mbar_init(&sm.full[i], C > 1 ? C * NWH : T);
      mbar_init(&sm.empty[i], C > 1 ? C * NWH : T);
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.xs_full[b], 1);
      mbar_init(&sm.xs_free[b], T);
      mbar_init(&sm.xbar[b], C * NWH);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ntiles_cta > 0) issue_tile(tile_of(0), 0);
  }

  // component constants as pairs (lo = component j, hi = component T + j)
  auto load_consts = [&](f2_t (&PP)[NP], f2_t& NBASE) {
    float pp[2][NP], base2[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int k = kb + c * T + j;
      base2[c] = -INFINITY;
#pragma unroll
      for (int q = 0; q < NP; ++q) pp[c][q] = 0.f;
      if (k < k_cur) {
        const float4* c4 = reinterpret_cast<const float4*>(mb.cst + k);
        float cc[12];
        const float4 a = c4[0], b = c4[1], e = c4[2];
        cc[0] = a.x; cc[1] = a.y; cc[2] = a.z; cc[3] = a.w;
        cc[4] = b.x; cc[5] = b.y; cc[6] = b.z; cc[7] = b.w;
        cc[8] = e.x; cc[9] = e.y; cc[10] = e.z; cc[11] = e.w;
#pragma unroll
        for (int q = 0; q < NP; ++q) pp[c][q] = cc[q];
        base2[c] = cc[10];
      }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) PP[q] = pk(pp[0][q], pp[1][q]);
    NBASE = pk(-base2[0], -base2[1]);
  };
  // NB = -P'(mu - c_t): FP64 dot of the FP32 factor with the FP32-rounded
  // tile-relative mean (the same mu' the consumers centre on), rounded once
  auto tile_nb = [&](const double* ct, const f2_t (&PP)[NP], f2_t (&NB)[D]) {
    float nbf[2][D];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float muf[D];
#pragma unroll
      for (int q = 0; q < D; ++q) muf[q] = static_cast<float>(sm.mu[q][c * T + j] - ct[q]);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q <= i; ++q) {
          const f2_t pij = PP[i * (i + 1) / 2 + q];
          s = fma(static_cast<double>(c ? hi2(pij) : lo2(pij)), static_cast<double>(muf[q]), s);
        }
        nbf[c][i] = static_cast<float>(-s);
      }
    }
#pragma unroll
    for (int q = 0; q < D; ++q) NB[q] = pk(nbf[0][q], nbf[1][q]);
  };
  // one point (the same FFMA tree as dens), chain started from nbase
  auto dens1 = [&](const float4 x, const f2_t (&PP)[NP], const f2_t (&NB)[D], f2_t nbase,
                   f2_t& Q) {
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
    Q = qv;
  };
  // Q = q - base2 = -(log2 density) of the P points at xs, both components
  auto dens = [&](const float4* xs, const f2_t (&PP)[NP], const f2_t (&NB)[D], f2_t NBASE,
                  f2_t (&Q)[P]) {
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const float4 x = xs[p];
      const f2_t X0 = pk(x.x, x.x), X1 = pk(x.y, x.y), X2 = pk(x.z, x.z);
      const f2_t Y0 = fma2(PP[0], X0, NB[0]);
      const f2_t Y1 = fma2(PP[2], X1, fma2(PP[1], X0, NB[1]));
      const f2_t Y2 = fma2(PP[5], X2, fma2(PP[4], X1, fma2(PP[3], X0, NB[2])));
      f2_t qv = fma2(Y2, Y2, fma2(Y1, Y1, fma2(Y0, Y0, NBASE)));
      if constexpr (D == 4) {
        const f2_t X3 = pk(x.w, x.w);
        const f2_t Y3 = fma2(PP[9], X3, fma2(PP[8], X2, fma2(PP[7], X1, fma2(PP[6], X0, NB[3]))));
        qv = fma2(Y3, Y3, qv);
      }
      Q[p] = qv;
    }
  };

  if (!producer) {  // mu (FP64) of both components, read by both roles
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int k = kb + c * T + j;
#pragma unroll
      for (int q = 0; q < 4; ++q) sm.mu[q][c * T + j] = k < k_cur ? mb.mu[k * 4 + q] : 0.0;
    }
  }
  if constexpr (C > 1) {
    cluster_sync_all();  // barriers initialised everywhere before any remote access
  } else {
    __syncthreads();
  }
  if (producer) {
    // ======================= producer warps =======================
    f2_t PP[NP], NBASE, NB[D];
    load_consts(PP, NBASE);
    unsigned g = 0;  // global sub-tile counter
    int ti = 0;      // tile iteration
    for (; ti < ntiles_cta; ++ti) {
      const int t = tile_of(ti);
      const int npts = static_cast<int>(min64(kTile, n - static_cast<int64_t>(t) * kTile));
      int s0, s1;
      sub_range(t, (npts + P - 1) / P, s0, s1);
      const int tb = ti & 1;
      mbar_wait(&sm.xs_full[tb], (ti >> 1) & 1u);
      {
        double ct[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) ct[q] = sm.tcs[tb][q];
        tile_nb(ct, PP, NB);
      }
      for (int s = s0; s < s1; ++s, ++g) {
        if (j == 0 && s == min(s0 + kRing, s1 - 1)) {
          // prefetch the next tile: consumers have started this tile (they
          // read sub-tile g - kRing), so they released the other buffer
          if (ti + 1 < ntiles_cta) {
            const int tn = tile_of(ti + 1);
            if (ti >= 1) mbar_wait(&sm.xs_free[tb ^ 1], ((ti - 1) >> 1) & 1u);
            issue_tile(tn, tb ^ 1);
          }
        }
        const int slot = g % kRing;
        if (g >= kRing) {
          if constexpr (C > 1) {
            mbar_wait_cluster(&sm.empty[slot], ((g / kRing) - 1) & 1u);
          } else {
            mbar_wait(&sm.empty[slot], ((g / kRing) - 1) & 1u);
          }
        }
        f2_t E[P];
        if constexpr (PRE) {
          // r = 2^-(Q + L): the shift starts the FFMA chain (L.x = 0), or a
          // far point (L.x = -Q_min, uniform) adds Q - Q_min first, then the
          // small remainder (estep_chunked.cu)
#pragma unroll
          for (int p = 0; p < P; ++p) {
            const float2 L = sm.ls[tb][s * P + p];
            const bool far = L.x != 0.f;
            f2_t q1[1];
            const f2_t nb1 = far ? NBASE : add2(NBASE, pk(L.y, L.y));
            dens1(sm.xs[tb][s * P + p], PP, NB, nb1, q1[0]);
            E[p] = far ? add2(add2(q1[0], pk(L.x, L.x)), pk(L.y, L.y)) : q1[0];
          }
#pragma unroll
          for (int p = 0; p < P; p += 2) {
            sm.ering[slot][p / 2][j] = make_float4(ex2n(lo2(E[p])), ex2n(hi2(E[p])),
                                                   ex2n(lo2(E[p + 1])), ex2n(hi2(E[p + 1])));
          }
          mbar_arrive(&sm.full[slot]);
          continue;
        }
        dens(&sm.xs[tb][s * P], PP, NB, NBASE, E);
        float v[P];
#pragma unroll
        for (int p = 0; p < P; p += 2) {
          const float e0 = ex2n(lo2(E[p])), e1 = ex2n(hi2(E[p]));
          const float e2 = ex2n(lo2(E[p + 1])), e3 = ex2n(hi2(E[p + 1]));
          sm.ering[slot][p / 2][j] = make_float4(e0, e1, e2, e3);
          v[p] = e0 + e1;
          v[p + 1] = e2 + e3;
        }
        const float r = warp_reduce_scatter<P, false>(v, lane);
        if constexpr (C > 1) {
          // the warp's per-point partial to every CTA of the cluster, then an
          // arrival on each CTA's full barrier (release.cluster orders them)
          const unsigned ra = smem_u32(&sm.red[slot][lane / G][rank * NWH + warp]);
          const unsigned fa = smem_u32(&sm.full[slot]);
#pragma unroll
          for (int q = 0; q < C; ++q) {
            if ((lane % G) == 0) st_cluster_f32(mapa_u32(ra, q), r);
          }
          __syncwarp();  // the warp's stores before its lane-0 release arrivals
          if (lane < C) mbar_arrive_cluster(mapa_u32(fa, lane));
        } else {
          if ((lane % G) == 0) sm.red[slot][lane / G][warp] = r;
          mbar_arrive(&sm.full[slot]);
        }
      }
    }
  } else {  // producers hold no statistics

  // ======================= consumer warps =======================
  f2_t ACC[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    ACC[s] = 0ull;
    acc64[s * T + j] = make_double2(0.0, 0.0);
  }
  // FP32 register sums are widened into the FP64 shared accumulators every
  // GMMB_FLUSH_SUBTILES x 8 points (a second FP32 level, or a
  // longer cadence, costs accuracy that EM amplifies ~25x).
  auto promote = [&]() {  // registers -> acc64
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      double2 v = acc64[s * T + j];
      v.x += f32_to_f64(lo2(ACC[s]));
      v.y += f32_to_f64(hi2(ACC[s]));
      ACC[s] = 0ull;
      acc64[s * T + j] = v;
    }
  };
  unsigned xcount = 0;  // exact-path events (xbar parity)
  // exact path: this warp's per-point partial to every CTA's xred[b], then
  // wait until all consumer warps of the cluster posted theirs
  auto xpost = [&](float r, int b) {
    if constexpr (C > 1) {
      const unsigned ra = smem_u32(&sm.xred[b][lane / G][rank * NWH + warp]);
      const unsigned xa = smem_u32(&sm.xbar[b]);
#pragma unroll
      for (int q = 0; q < C; ++q) {
        if ((lane % G) == 0) st_cluster_f32(mapa_u32(ra, q), r);
      }
      __syncwarp();
      if (lane < C) mbar_arrive_cluster(mapa_u32(xa, lane));
      mbar_wait_cluster(&sm.xbar[b], xcount & 1u);
    } else {
      if ((lane % G) == 0) sm.xred[b][lane / G][warp] = r;
      asm volatile("bar.sync 2, %0;" ::"r"(T) : "memory");
    }
  };
  double ll_acc = 0.0;  // consumer warp 0, lanes with lane % G == 0 (one point each)
  const bool finisher = warp == 0 && (lane % G) == 0;
  const int fp = lane / G;
  int xb = 0;
  unsigned g = 0;
  int ti = 0;
  for (; ti < ntiles_cta; ++ti) {
    const int t = tile_of(ti);
    const int npts = static_cast<int>(min64(kTile, n - static_cast<int64_t>(t) * kTile));
    int s0, s1;
    sub_range(t, (npts + P - 1) / P, s0, s1);
    const int tb = ti & 1;
    mbar_wait(&sm.xs_full[tb], (ti >> 1) & 1u);
    f2_t NMU[D];  // -(mu - c_t) as FP32 pairs
    {
      float nm[2][D];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < D; ++q)
          nm[c][q] = static_cast<float>(-(sm.mu[q][c * T + j] - sm.tcs[tb][q]));
#pragma unroll
      for (int q = 0; q < D; ++q) NMU[q] = pk(nm[0][q], nm[1][q]);
    }
    for (int s = s0; s < s1; ++s, ++g) {
      const int q0 = s * P;
      const int slot = g % kRing;
      if constexpr (C > 1) {
        mbar_wait_cluster(&sm.full[slot], (g / kRing) & 1u);
      } else {
        mbar_wait(&sm.full[slot], (g / kRing) & 1u);
      }
      float S = PRE ? 1.f : cta_combine<NWC, P, false>(sm.red[slot], lane);
      f2_t E[P];
#pragma unroll
      for (int p = 0; p < P; p += 2) {
        const float4 v = sm.ering[slot][p / 2][j];
        E[p] = pk(v.x, v.y);
        E[p + 1] = pk(v.z, v.w);
      }
      if constexpr (C > 1) {
        __syncwarp();  // the warp's reads of the slot before its release arrivals
        if (lane < C) mbar_arrive_cluster(mapa_u32(smem_u32(&sm.empty[slot]), lane));
      } else {
        mbar_arrive(&sm.empty[slot]);
      }
      float M = 0.f;
      const bool valid_g = q0 + fp < npts;
      const bool exact = !PRE && __any_sync(0xffffffffu, valid_g && (exact_mode != 0 ||
                                                             !(S >= 0x1p-64f && S <= 0x1p64f)));
      if (exact) {  // uniform over consumer warps: identical S everywhere
        f2_t PP[NP], NBASE, NB[D];
        load_consts(PP, NBASE);
        float nbf[2][D];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int i = 0; i < D; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q <= i; ++q) {
              const f2_t pij = PP[i * (i + 1) / 2 + q];
              acc = fma(static_cast<double>(c ? hi2(pij) : lo2(pij)),
                        sm.mu[q][c * T + j] - sm.tcs[tb][q], acc);
            }
            nbf[c][i] = static_cast<float>(-acc);
          }
        }
#pragma unroll
        for (int q = 0; q < D; ++q) NB[q] = pk(nbf[0][q], nbf[1][q]);
        dens(&sm.xs[tb][q0], PP, NB, NBASE, E);
        float v[P];
#pragma unroll
        for (int p = 0; p < P; ++p) v[p] = fmaxf(-lo2(E[p]), -hi2(E[p]));
        float r = warp_reduce_scatter<P, true>(v, lane);
        xpost(r, xb);
        M = cta_combine<NWC, P, true>(sm.xred[xb], lane);
        xb ^= 1;
        M = M == -INFINITY ? 0.f : M;
#pragma unroll
        for (int p = 0; p < P; ++p) {
          const float mp = __shfl_sync(0xffffffffu, M, p * G);
          const float e0 = ex2n(lo2(E[p]) + mp), e1 = ex2n(hi2(E[p]) + mp);
          E[p] = pk(e0, e1);
          v[p] = e0 + e1;
        }
        r = warp_reduce_scatter<P, false>(v, lane);
        xpost(r, xb);
        S = cta_combine<NWC, P, false>(sm.xred[xb], lane);
        xb ^= 1;
        ++xcount;
      }
      if constexpr (PRE) {
        if (finisher && valid_g && chunk == 0) {
          const float2 L = sm.ls[tb][q0 + fp];
          ll_acc += static_cast<double>(L.x) + static_cast<double>(L.y);
        }
      } else {
        if (finisher && valid_g && rank == 0) ll_acc += static_cast<double>(M + lg2f(S));
      }
      const float scale_g = valid_g ? rcpf(S) : 0.f;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const float4 x = sm.xs[tb][q0 + p];
        const float xv[4] = {x.x, x.y, x.z, x.w};
        f2_t R;
        if constexpr (PRE) {
          R = q0 + p < npts ? E[p] : 0ull;  // padding points of a partial tile
        } else {
          const float sc = __shfl_sync(0xffffffffu, scale_g, p * G);
          R = mul2(E[p], pk(sc, sc));
        }
        f2_t DD[D], W[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          DD[i] = add2(pk(xv[i], xv[i]), NMU[i]);
          W[i] = mul2(R, DD[i]);
        }
        ACC[0] = add2(ACC[0], R);
#pragma unroll
        for (int i = 0; i < D; ++i) ACC[1 + i] = add2(ACC[1 + i], W[i]);
        int q = 1 + D;
#pragma unroll
        for (int i = 0; i < D; ++i) {
#pragma unroll
          for (int c = 0; c <= i; ++c) {
            ACC[q] = fma2(W[i], DD[c], ACC[q]);
            ++q;
          }
        }
        if (GMMB_FLUSH_SUBTILES < 16 && ((q0 + p + 1) % (GMMB_FLUSH_SUBTILES * 8)) == 0) promote();
      }
    }
    promote();  // the tile's remaining FP32 partial sums
    mbar_arrive(&sm.xs_free[tb]);  // this consumer is done with tile buffer tb
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int k = kb + c * T + j;
    if (k < kpad) {
      double* out = partials + (static_cast<int64_t>(cid) * kpad + k) * NS;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double2 v = acc64[s * T + j];
        out[s] = c ? v.y : v.x;
      }
    }
  }
  if (warp == 0) {  // ll partial of this cluster: the P finisher lanes, in order
    double s = 0.0;
#pragma unroll
    for (int p = 0; p < P; ++p) s += __shfl_sync(0xffffffffu, ll_acc, p * G);
    if (lane == 0 && rank == 0 && chunk == 0) ll_part[cid] = s * kLn2;
  }
  }  // consumers
  if constexpr (C > 1) {
    // no CTA leaves while cluster peers may still write its shared memory
    cluster_sync_all();
  }
}

template <int D, int NWH, int C>
cudaError_t launch_estep_ws(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                            int kpad, double* partials, double* ll_part, int exact_mode,
                            int sm_count, cudaStream_t s, int* ncl_out) {
  constexpr int P = GMMB_WS_P;
  using Smem = WsSmem<NWH, P, C>;
  auto kern = estep_ws_kernel<D, NWH, P, C>;
  const size_t smem = ((sizeof(Smem) + 15) & ~size_t(15)) + sizeof(double2) * nstats(D) * NWH * 32;
  static int slots_dev[64] = {0};  // co-resident CTAs (C = 1) or clusters (C > 1), per device
  int dev = 0;
  cudaGetDevice(&dev);
  int& slots = slots_dev[dev & 63];
  if (slots == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (C > 1) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(C * (sm_count / C));
      q.blockDim = dim3(2 * NWH * 32);
      q.dynamicSmemBytes = smem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = C;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      e = cudaOccupancyMaxActiveClusters(&slots, kern, &q);  // one wave of clusters
    } else {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&slots, kern, 2 * NWH * 32, smem);
      slots *= sm_count;
    }
    if (e != cudaSuccess) return e;
    if (slots < 1) slots = 1;
    if (getenv("GMMB_DEBUG"))
      fprintf(stderr, "gmmb: estep_ws D=%d NWH=%d C=%d smem=%zu -> %d co-resident %s\n", D, NWH, C,
              smem, slots, C > 1 ? "clusters" : "CTAs");
  }
  int ncl = slots;
  if (ncl > pts.ntiles) ncl = pts.ntiles;
  if (ncl < 1) ncl = 1;
  *ncl_out = ncl;
  if (!partials) return cudaSuccess;  // size query only
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * C);
  cfg.blockDim = dim3(2 * NWH * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  const int split_sub = ncl * C <= sm_count ? 1 : 0;  // one CTA per SM: balance sub-tiles
  return cudaLaunchKernelEx(&cfg, kern, pts.xt, pts.tc, pts.n, pts.ntiles, bufs[0], bufs[1], st,
                            kpad, partials, ll_part, exact_mode, split_sub,
                            static_cast<const float2*>(nullptr), 1);
}

// pass B of the chunked E step (K > 512): the warp-specialised kernel with
// known normalisers, one CTA per (512-component chunk, point range), one CTA
// per SM (groups = sm_count / nch point ranges)
template <int D>
cudaError_t launch_estep_ws_pre_d(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                                  int kpad, int nch, const float2* lse, double* partials,
                                  double* ll_part, int sm_count, cudaStream_t s, int* ncl_out) {
  constexpr int P = GMMB_WS_P, NWH = 8;
  using Smem = WsSmem<NWH, P, 1>;
  auto kern = estep_ws_kernel<D, NWH, P, 1, true>;
  const size_t smem = ((sizeof(Smem) + 15) & ~size_t(15)) + sizeof(double2) * nstats(D) * NWH * 32;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set[dev & 63] = true;
  }
  int groups = sm_count / nch;
  if (groups < 1) groups = 1;
  if (groups > pts.ntiles) groups = pts.ntiles;
  *ncl_out = groups;
  if (!partials) return cudaSuccess;
  kern<<<nch * groups, 2 * NWH * 32, smem, s>>>(pts.xt, pts.tc, pts.n, pts.ntiles, bufs[0],
                                                bufs[1], st, kpad, partials, ll_part, 0, 1, lse,
                                                nch);
  return cudaGetLastError();
}

template <int D, int NW, int C, int P, int CPT>
cudaError_t launch_estep_t(const PointsDev& pts, const ModelBuf* bufs,
                           const EmState* st, int kpad, double* partials,
                           double* ll_part, int exact_mode, int sm_count,
                           cudaStream_t s, int* ncl_out) {
  using Smem = EstepSmem<D, NW, C, P>;
  auto kern = estep_stats_kernel<D, NW, C, P, CPT>;
  const size_t smem = ((sizeof(Smem) + 15) & ~size_t(15)) +
                      sizeof(double2) * ((nstats(D) + 1) / 2) * CPT * NW * 32;
  static int per_sm_dev[64] = {0};  // per template instance and device
  int dev = 0;
  cudaGetDevice(&dev);
  int& per_sm = per_sm_dev[dev & 63];
  if (per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  int ncl = sm_count * per_sm / C;
  if (ncl > pts.ntiles) ncl = pts.ntiles;
  if (ncl < 1) ncl = 1;
  *ncl_out = ncl;
  if (!partials) return cudaSuccess;  // size query only
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * C);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (C > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, pts.xt, pts.tc, pts.n, pts.ntiles,
                            bufs[0], bufs[1], st, kpad, partials, ll_part,
                            exact_mode);
}

template <int D>
cudaError_t launch_estep_d(const PointsDev& pts, const ModelBuf* bufs,
                           const EmState* st, int k0, double* partials,
                           double* ll_part, int exact_mode, int sm_count,
                           cudaStream_t s, int* ncl) {
  constexpr int P = 8;
  const int kpad = k0;
#define GMMB_L(NW, C, CPT) \
  return launch_estep_t<D, NW, C, P, CPT>(pts, bufs, st, kpad, partials, ll_part, \
                                          exact_mode, sm_count, s, ncl)
#define GMMB_W(NWH, C) \
  return launch_estep_ws<D, NWH, C>(pts, bufs, st, kpad, partials, ll_part, exact_mode, \
                                    sm_count, s, ncl)
#if GMMB_PIPE
  // warp-specialised packed kernel: K <= 64 NWH per CTA, clusters of C CTAs above 512
  if (k0 <= 64) GMMB_W(1, 1);
  if (k0 <= 128) GMMB_W(2, 1);
  if (k0 <= 256) GMMB_W(4, 1);
  if (k0 <= 512) GMMB_W(8, 1);
  if (k0 <= 1024) GMMB_W(8, 2);
  if (k0 <= 2048) GMMB_W(8, 4);
  // K = 4096 (clusters of 8): only 15 clusters co-reside (120 SMs) and the
  // cross-CTA hand-off per sub-tile dominates; the barrier-per-sub-tile
  // cluster kernel below is faster there (5.2 vs 5.8 ms per iteration)
#undef GMMB_W
#else
  if (k0 <= 32) GMMB_L(1, 1, 1);
  if (k0 <= 64) GMMB_L(2, 1, 1);
  if (k0 <= 128) GMMB_L(4, 1, 1);
  if (k0 <= 256) GMMB_L(8, 1, 1);
  if (k0 <= 512) GMMB_L(8, 1, 2);
#endif
  if (k0 <= 1024) GMMB_L(8, 2, 2);
  if (k0 <= 2048) GMMB_L(8, 4, 2);
  if (k0 <= 4096) GMMB_L(8, 8, 2);
#undef GMMB_L
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Second-stage reduce: one warp per component, fixed lane/shuffle order.
// ---------------------------------------------------------------------------
template <int D>
__global__ void em_reduce_kernel(const double* __restrict__ partials,
                                 const double* __restrict__ ll_part, int ncl,
                                 int kpad, const EmState* __restrict__ st,
                                 double* __restrict__ red,
                                 double* __restrict__ red_ll) {
  constexpr int NS = nstats(D);
  if (st->done) return;
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (k == kpad) {  // one extra warp reduces the log-likelihood partials
    double s = 0.0;
    for (int c = lane; c < ncl; c += 32) s += ll_part[c];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) red_ll[0] = s;
    return;
  }
  if (k > kpad || k >= st->k_cur) return;
  double acc[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) acc[j] = 0.0;
  for (int c = lane; c < ncl; c += 32) {
    const double* src = partials + (static_cast<int64_t>(c) * kpad + k) * NS;
#pragma unroll
    for (int j = 0; j < NS; ++j) acc[j] += src[j];
  }
#pragma unroll
  for (int j = 0; j < NS; ++j) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NS; ++j) red[static_cast<int64_t>(k) * NS + j] = acc[j];
  }
}

// ---------------------------------------------------------------------------
// Finalize: centred stats about mu_old -> mean, covariance, factor.
//   mean = mu_old + S_d / n_k;  scatter = S_dd / n_k - delta delta^T
// (the reference's two passes, sogmm.cpp:410-416 / kernels.hpp:91-179,
// fused into one pass centred at the previous mean).
// ---------------------------------------------------------------------------
// Finalize one component from its reduced statistics s[NS] (centred at the
// old mean): mean, covariance + cov_reg, FP64 Cholesky / precision factor.
template <int D>
// The mean, covariance and precision factor go straight into the fresh model
// buffer (the one the commit makes current) at index k; the commit then only
// adds weights and log-normalisers, or compacts when components are dropped.
__device__ __forceinline__ void finalize_component(const double* s, int k, const ModelBuf& mb,
                                                   double cov_reg, RecBuf& rec,
                                                   const ModelBuf& fresh) {
  constexpr int NP = npacked(D);
  const double cnt = s[0];
  int flags = 0;
  double mean[4] = {0, 0, 0, 0};
  double cov[10];
#pragma unroll
  for (int j = 0; j < 10; ++j) cov[j] = 0.0;
  float pc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) pc[j] = 0.f;
  double logdet = 0.0;
  if (!(cnt < kDegenerateCount)) {
    flags |= 1;
    double delta[D];
    const double inv = 1.0 / cnt;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      delta[j] = s[1 + j] * inv;
      mean[j] = mb.mu[k * 4 + j] + delta[j];
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int i = packed_row(q), j = packed_col(q);
      cov[q] = s[1 + D + q] * inv - delta[i] * delta[j];
      if (i == j) cov[q] += cov_reg;
    }
    if (factor_component<D>(cov, pc, &logdet)) flags |= 2;
  }
  rec.count[k] = cnt;
  double2* dm = reinterpret_cast<double2*>(fresh.mu + k * 4);
  dm[0] = make_double2(mean[0], mean[1]);
  dm[1] = make_double2(mean[2], mean[3]);
  double2* dc = reinterpret_cast<double2*>(fresh.cov + k * 10);
#pragma unroll
  for (int j = 0; j < 5; ++j) dc[j] = make_double2(cov[2 * j], cov[2 * j + 1]);
  rec.logdet[k] = logdet;
  float4* dp = reinterpret_cast<float4*>(&fresh.cst[k]);
#pragma unroll
  for (int j = 0; j < 4; ++j) dp[j] = make_float4(pc[4 * j], pc[4 * j + 1], pc[4 * j + 2], pc[4 * j + 3]);
  rec.flags[k] = flags;
}

template <int D>
__global__ void em_finalize_kernel(const double* __restrict__ red,
                                   ModelBuf b0, ModelBuf b1,
                                   const EmState* __restrict__ st, RecBuf rec) {
  if (st->done) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= st->k_cur) return;
  const ModelBuf& mb = st->cur ? b1 : b0;
  const ModelBuf& fresh = st->cur ? b0 : b1;
  finalize_component<D>(red + static_cast<int64_t>(k) * nstats(D), k, mb, st->cov_reg, rec, fresh);
}

// Single-device fused second stage: one warp per component reduces the
// per-CTA partials in a fixed order (lane-strided sums, fixed butterfly) and
// its lane 0 finalizes the component.
// WPC warps per component: one (K large) or the whole 128-thread CTA (small
// K, where the E kernel runs many CTAs and leaves ncl ~ 1000 partials per
// component). Lane-strided sums, a fixed butterfly, and (WPC > 1) the warps'
// sums in warp order: deterministic.
template <int D, int WPC>
__global__ void __launch_bounds__(128) em_reduce_finalize_kernel(
    const double* __restrict__ partials, int ncl, int kpad, ModelBuf b0, ModelBuf b1,
    const EmState* __restrict__ st, RecBuf rec) {
  constexpr int NS = nstats(D);
  __shared__ double red[4][NS];
  if (st->done) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = WPC == 1 ? blockIdx.x * 4 + w : blockIdx.x;
  const int sub = WPC == 1 ? 0 : w;
  if (k >= kpad || k >= st->k_cur) return;  // uniform over the CTA when WPC > 1
  double acc[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) acc[j] = 0.0;
#pragma unroll 4
  for (int c = sub * 32 + lane; c < ncl; c += 32 * WPC) {
    const double* src = partials + (static_cast<int64_t>(c) * kpad + k) * NS;
#pragma unroll
    for (int j = 0; j < NS; ++j) acc[j] += src[j];
  }
#pragma unroll
  for (int j = 0; j < NS; ++j) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
  }
  if constexpr (WPC > 1) {
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < NS; ++j) red[w][j] = acc[j];
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      double t = red[0][j];
#pragma unroll
      for (int q = 1; q < WPC; ++q) t += red[q][j];
      acc[j] = t;
    }
  } else {
    if (lane != 0) return;
  }
  const ModelBuf& mb = st->cur ? b1 : b0;
  const ModelBuf& fresh = st->cur ? b0 : b1;
  finalize_component<D>(acc, k, mb, st->cov_reg, rec, fresh);
}

// ---------------------------------------------------------------------------
// Commit (single CTA of 1024 threads): sogmm.cpp:418-453 + :488-504.
// The kernel is a chain of dependent memory round trips, so it issues every
// independent load first (state, ll partials, the components' keep flags,
// counts and log-dets), scans the keep flags chunk by chunk in component
// order (component k = chunk * T + tid, order-preserving compaction), and
// copies the kept records with 16-byte vector accesses (coalesced: thread j
// writes compacted component j).
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void commit_body(
    int mode, const RecBuf& rec, int k_in_arg, const double* __restrict__ red_ll,
    const double* __restrict__ ll_part, int ncl,
    const ModelBuf& b0, const ModelBuf& b1, EmState* st, double* __restrict__ ll_trace) {
  constexpr int T = 1024;
  constexpr int CH = kMaxK / T;  // chunks of T components (<= 4)
  __shared__ int s_wcnt[32];
  __shared__ double s_wtot[32];
  __shared__ int s_woff[32];
  __shared__ int s_base[CH + 1];
  __shared__ double s_ctot[CH];
  __shared__ int s_flag;
  __shared__ short s_map[kMaxK];  // compacted index -> component
  static_assert(T == 1024, "one CTA of 1024 threads");
  static_assert(kMaxK <= 32767, "short map");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- every independent load up front (one round trip) ----
  const int done0 = st->done;
  const int kcur0 = st->k_cur;
  const int cur0 = st->cur;
  int iter0 = 0, maxit0 = 0, removed0 = 0;
  double units0 = 0.0, npts0 = 0.0, llprev0 = 0.0, tol0 = 0.0;
  if (tid == 0) {  // the rest of the state thread 0 needs
    iter0 = st->iter;
    maxit0 = st->max_iters;
    removed0 = st->removed;
    units0 = st->units;
    npts0 = st->npts;
    llprev0 = st->ll_prev;
    tol0 = st->tol;
  }
  const int kcap = k_in_arg;  // rec holds at least this many records
  int flg[CH];
  double cntv[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int k = c * T + tid;
    flg[c] = k < kcap ? rec.flags[k] : 0;
    cntv[c] = k < kcap ? rec.count[k] : 0.0;
  }
  double llv = 0.0;
  if (mode == 0 && warp == 0) {
    if (ll_part) {
      for (int c = lane; c < ncl; c += 32) llv += ll_part[c];
    } else if (lane == 0) {
      llv = red_ll[0];
    }
  }
  if (done0) return;
  const int k_in = mode == 0 ? kcur0 : k_in_arg;

  if (mode == 0) {
    // log-likelihood: the per-CTA partials of the fused E kernel in a fixed
    // order (lane-strided sums, then a fixed butterfly), or a reduced value
    double ll = llv;
    if (warp == 0 && ll_part) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, off);
    }
    // EM bookkeeping: sogmm.cpp:490-498
    if (tid == 0) {
      const int iter = iter0;
      st->units = units0 + npts0 * static_cast<double>(k_in);
      if (ll_trace) ll_trace[iter] = ll;
      st->ll = ll;
      st->iter = iter + 1;
      int conv = 0;
      if (iter > 0) {
        const double rel = fabs(ll - llprev0) / fmax(fabs(llprev0), 1e-12);
        if (rel < tol0) conv = 1;
      }
      if (conv) {
        st->converged = 1;
        st->done = 1;
      }
      st->ll_prev = ll;
      s_flag = conv;
    }
    __syncthreads();
    if (s_flag) return;
  }

  // keep flags -> per-chunk exclusive scans (compaction preserves component
  // order, sogmm.cpp:418-429); chunk totals and kept counts with fixed-shape
  // reductions (deterministic)
  int keep[CH], excl[CH];
  const int nch = (k_in + T - 1) / T;
#pragma unroll
  for (int c = 0; c < CH; ++c) keep[c] = excl[c] = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if (c >= nch) break;  // uniform: only the chunks that hold components
    const int k = c * T + tid;
    keep[c] = (c < nch && k < k_in) ? (flg[c] & 1) : 0;
    int incl = keep[c];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    double wt = keep[c] ? cntv[c] : 0.0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) wt += __shfl_xor_sync(0xffffffffu, wt, off);
    if (c < nch) {
      if (lane == 31) s_wcnt[warp] = incl;
      if (lane == 0) s_wtot[warp] = wt;
    }
    __syncthreads();
    if (c < nch && warp == 0) {
      const int wc = s_wcnt[lane];
      int wi = wc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, wi, off);
        if (lane >= off) wi += v;
      }
      s_woff[lane] = wi - wc;
      double t = s_wtot[lane];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
      if (lane == 31) s_base[c + 1] = wi;  // kept in this chunk
      if (lane == 0) s_ctot[c] = t;
    }
    __syncthreads();
    excl[c] = c < nch ? s_woff[warp] + incl - keep[c] : 0;
    __syncthreads();  // s_wcnt / s_woff reused by the next chunk
  }
  if (tid == 0) {
    int b = 0;
    double tot = 0.0;
    s_base[0] = 0;
    for (int c = 0; c < nch; ++c) {
      const int kc = s_base[c + 1];
      s_base[c + 1] = b + kc;
      b += kc;
      tot += s_ctot[c];
    }
    s_ctot[0] = tot;
    s_flag = 0x7fffffff;
  }
  __syncthreads();
  const int k_new = s_base[nch];
  const double total = s_ctot[0];
  if (k_new == 0) {
    if (tid == 0) {
      st->error = 3;
      st->error_kind = 2;
      st->error_index = 0;
      st->done = 1;
    }
    return;
  }
  // first non-SPD kept component (compacted index), sogmm.cpp:447-452; the
  // compaction map
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    if (keep[c]) {
      const int j = s_base[c] + excl[c];
      s_map[j] = static_cast<short>(c * T + tid);
      if (!(flg[c] & 2)) atomicMin(&s_flag, j);
    }
  }
  __syncthreads();
  if (s_flag != 0x7fffffff) {
    if (tid == 0) {
      st->error = 3;
      st->error_kind = 1;
      st->error_index = s_flag;
      st->done = 1;
    }
    return;
  }
  const double half_d_ln2pi = 0.5 * D * kLog2Pi;
  int dst_sel;
  if (mode == 0 && k_new == k_in) {
    // nothing dropped (the common case): the finalize already wrote means,
    // covariances and factors into the fresh buffer in place; add the
    // weights and log-normalisers
    dst_sel = cur0 ^ 1;
    const ModelBuf& dst = dst_sel ? b1 : b0;
    for (int k = tid; k < k_new; k += T) {
      const double w = rec.count[k] / total;
      dst.w[k] = w;
      const double b2 = kLog2E * (log(w) + rec.logdet[k] - half_d_ln2pi);
      const float hi = static_cast<float>(b2);
      *reinterpret_cast<float2*>(&dst.cst[k].p[10]) =
          make_float2(hi, static_cast<float>(b2 - static_cast<double>(hi)));
    }
  } else {
    // compaction: mode 0 from the fresh buffer (written by the finalize) into
    // the other one (the previous model, consumed by now); mode 1 from the
    // record buffers into the current one
    dst_sel = cur0;
    const ModelBuf& dst = dst_sel ? b1 : b0;
    const ModelBuf& src_m = cur0 ? b0 : b1;
    for (int j = tid; j < k_new; j += T) {
      const int k = s_map[j];
      const double w = rec.count[k] / total;
      dst.w[j] = w;
      const double2* sm2 = reinterpret_cast<const double2*>(mode == 0 ? src_m.mu + k * 4 : rec.mean + k * 4);
      double2* dm2 = reinterpret_cast<double2*>(dst.mu + j * 4);
      dm2[0] = sm2[0];
      dm2[1] = sm2[1];
      const double2* sc2 = reinterpret_cast<const double2*>(mode == 0 ? src_m.cov + k * 10 : rec.cov + k * 10);
      double2* dc2 = reinterpret_cast<double2*>(dst.cov + j * 10);
#pragma unroll
      for (int q = 0; q < 5; ++q) dc2[q] = sc2[q];
      const float4* sp4 = mode == 0 ? reinterpret_cast<const float4*>(&src_m.cst[k])
                                    : reinterpret_cast<const float4*>(rec.pc + k * 16);
      float4* dp4 = reinterpret_cast<float4*>(&dst.cst[j]);
      float4 v2 = sp4[2];
      const double b2 = kLog2E * (log(w) + rec.logdet[k] - half_d_ln2pi);
      v2.z = static_cast<float>(b2);                              // c.p[10]
      v2.w = static_cast<float>(b2 - static_cast<double>(v2.z));  // c.p[11]
      dp4[0] = sp4[0];
      dp4[1] = sp4[1];
      dp4[2] = v2;
      dp4[3] = sp4[3];
    }
  }
  __syncthreads();
  if (tid == 0) {
    st->removed = removed0 + (k_in - k_new);
    st->k_cur = k_new;
    if (mode == 0) {
      st->cur = dst_sel;
      if (iter0 + 1 >= maxit0) st->done = 1;
    }
  }
}

// Commit kernel. Inside the EM while-graph (use_cond = 1) it also sets the
// loop condition from the device state: the whole EM loop runs without a
// host round trip (CUDA conditional graph node).
// Any K (k_in > kMaxK): the same commit with the chunk loop at run time and
// the compaction map in global memory (rec.map[k] = compacted index of a
// kept component). Chunk totals are combined serially in chunk order, so
// the result does not depend on the schedule.
template <int D>
__device__ __forceinline__ void commit_body_big(
    int mode, const RecBuf& rec, int k_in_arg, const double* __restrict__ red_ll,
    const double* __restrict__ ll_part, int ncl,
    const ModelBuf& b0, const ModelBuf& b1, EmState* st, double* __restrict__ ll_trace) {
  constexpr int T = 1024;
  __shared__ int s_wcnt[32];
  __shared__ double s_wtot[32];
  __shared__ int s_woff[32];
  __shared__ int s_base;
  __shared__ double s_tot;
  __shared__ int s_flag;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (st->done) return;
  const int cur0 = st->cur;
  const int k_in = mode == 0 ? st->k_cur : k_in_arg;
  if (mode == 0) {  // EM bookkeeping: sogmm.cpp:490-498
    double ll = 0.0;
    if (warp == 0) {
      if (ll_part) {
        for (int c = lane; c < ncl; c += 32) ll += ll_part[c];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, off);
      } else {
        ll = red_ll[0];
      }
    }
    if (tid == 0) {
      const int iter = st->iter;
      st->units = st->units + st->npts * static_cast<double>(k_in);
      if (ll_trace) ll_trace[iter] = ll;
      st->ll = ll;
      st->iter = iter + 1;
      int conv = 0;
      if (iter > 0) {
        const double rel = fabs(ll - st->ll_prev) / fmax(fabs(st->ll_prev), 1e-12);
        if (rel < st->tol) conv = 1;
      }
      if (conv) {
        st->converged = 1;
        st->done = 1;
      }
      st->ll_prev = ll;
      s_flag = conv;
    }
    __syncthreads();
    if (s_flag) return;
  }
  if (tid == 0) {
    s_base = 0;
    s_tot = 0.0;
    s_flag = 0x7fffffff;
  }
  __syncthreads();
  // order-preserving compaction map + kept weight total (sogmm.cpp:418-433)
  for (int k0 = 0; k0 < k_in; k0 += T) {
    const int k = k0 + tid;
    const int fl = k < k_in ? rec.flags[k] : 0;
    const int keep = fl & 1;
    int incl = keep;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    double wt = keep ? rec.count[k] : 0.0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) wt += __shfl_xor_sync(0xffffffffu, wt, off);
    if (lane == 31) s_wcnt[warp] = incl;
    if (lane == 0) s_wtot[warp] = wt;
    __syncthreads();
    if (warp == 0) {
      const int wc = s_wcnt[lane];
      int wi = wc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, wi, off);
        if (lane >= off) wi += v;
      }
      s_woff[lane] = wi - wc;
      double t = s_wtot[lane];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
      if (lane == 31) s_wcnt[0] = wi;  // kept in this chunk (read after the barrier)
      if (lane == 0) s_wtot[0] = t;
    }
    __syncthreads();
    const int base = s_base;
    if (keep) {
      const int j = base + s_woff[warp] + incl - keep;
      rec.map[k] = j;
      if (!(fl & 2)) atomicMin(&s_flag, j);
    }
    __syncthreads();
    if (tid == 0) {
      s_base = base + s_wcnt[0];
      s_tot += s_wtot[0];
    }
    __syncthreads();
  }
  const int k_new = s_base;
  const double total = s_tot;
  if (k_new == 0) {
    if (tid == 0) {
      st->error = 3;
      st->error_kind = 2;
      st->error_index = 0;
      st->done = 1;
    }
    return;
  }
  if (s_flag != 0x7fffffff) {
    if (tid == 0) {
      st->error = 3;
      st->error_kind = 1;
      st->error_index = s_flag;
      st->done = 1;
    }
    return;
  }
  const double half_d_ln2pi = 0.5 * D * kLog2Pi;
  int dst_sel;
  if (mode == 0 && k_new == k_in) {
    dst_sel = cur0 ^ 1;
    const ModelBuf& dst = dst_sel ? b1 : b0;
    for (int k = tid; k < k_new; k += T) {
      const double w = rec.count[k] / total;
      dst.w[k] = w;
      const double b2 = kLog2E * (log(w) + rec.logdet[k] - half_d_ln2pi);
      const float hi = static_cast<float>(b2);
      *reinterpret_cast<float2*>(&dst.cst[k].p[10]) =
          make_float2(hi, static_cast<float>(b2 - static_cast<double>(hi)));
    }
  } else {
    dst_sel = cur0;
    const ModelBuf& dst = dst_sel ? b1 : b0;
    const ModelBuf& src_m = cur0 ? b0 : b1;
    for (int k = tid; k < k_in; k += T) {
      if (!(rec.flags[k] & 1)) continue;
      const int j = rec.map[k];
      const double w = rec.count[k] / total;
      dst.w[j] = w;
      const double* sm = mode == 0 ? src_m.mu + k * 4 : rec.mean + k * 4;
      for (int q = 0; q < 4; ++q) dst.mu[j * 4 + q] = sm[q];
      const double* sc = mode == 0 ? src_m.cov + k * 10 : rec.cov + k * 10;
      for (int q = 0; q < 10; ++q) dst.cov[j * 10 + q] = sc[q];
      const float* sp = mode == 0 ? src_m.cst[k].p : rec.pc + k * 16;
      float v[16];
      for (int q = 0; q < 16; ++q) v[q] = sp[q];
      const double b2 = kLog2E * (log(w) + rec.logdet[k] - half_d_ln2pi);
      v[10] = static_cast<float>(b2);
      v[11] = static_cast<float>(b2 - static_cast<double>(v[10]));
      for (int q = 0; q < 16; ++q) dst.cst[j].p[q] = v[q];
    }
  }
  __syncthreads();
  if (tid == 0) {
    st->removed = st->removed + (k_in - k_new);
    st->k_cur = k_new;
    if (mode == 0) {
      st->cur = dst_sel;
      if (st->iter >= st->max_iters) st->done = 1;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(1024) commit_kernel(
    int mode, RecBuf rec, int k_in_arg, const double* __restrict__ red_ll,
    const double* __restrict__ ll_part, int ncl,
    ModelBuf b0, ModelBuf b1, EmState* st, double* __restrict__ ll_trace,
    cudaGraphConditionalHandle cond, int use_cond) {
  if (k_in_arg > kMaxK)
    commit_body_big<D>(mode, rec, k_in_arg, red_ll, ll_part, ncl, b0, b1, st, ll_trace);
  else
    commit_body<D>(mode, rec, k_in_arg, red_ll, ll_part, ncl, b0, b1, st, ll_trace);
  if (use_cond) {
    __syncthreads();
    if (threadIdx.x == 0) cudaGraphSetConditional(cond, st->done ? 0u : 1u);
  }
}

// ---------------------------------------------------------------------------
// Prep: FP64 model in buffer st->cur -> constants (gmm.cpp:33-48).
// ---------------------------------------------------------------------------
template <int D>
__global__ void prep_kernel(ModelBuf b0, ModelBuf b1, EmState* st, int m) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const ModelBuf& mb = st->cur ? b1 : b0;
  CompConst c;
#pragma unroll
  for (int q = 0; q < 16; ++q) c.p[q] = 0.f;
  double logdet = 0.0;
  if (!factor_component<D>(mb.cov + k * 10, c.p, &logdet)) {
    atomicMin(&st->error_index, k);
    st->error = 3;
    st->error_kind = 3;
    st->done = 1;
    return;
  }
  const double b2 = kLog2E * (log(mb.w[k]) + logdet - 0.5 * D * kLog2Pi);
  c.p[10] = static_cast<float>(b2);
  c.p[11] = static_cast<float>(b2 - static_cast<double>(c.p[10]));
  mb.cst[k] = c;
}

// ---------------------------------------------------------------------------
// FP64 two-pass weighted moments (kernels.hpp:82-181).
// grid: (point chunks, component groups of 128); one thread per component.
// ---------------------------------------------------------------------------
constexpr int kMomChunk = 4096;  // points per CTA chunk (= kPointBlock)
constexpr int kMomTile = 256;

template <int D, bool LABELS, int PASS>
__global__ void __launch_bounds__(128) moments_kernel(
    const double* __restrict__ x64, int64_t n, const int32_t* __restrict__ labels,
    const double* __restrict__ log_gamma, int m,
    const double* __restrict__ means, double* __restrict__ part) {
  __shared__ double xs[4][kMomTile];
  __shared__ int ls[kMomTile];
  const int k = blockIdx.y * 128 + threadIdx.x;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kMomChunk;
  const int64_t c1 = min64(n, c0 + kMomChunk);
  double mu[D];
#pragma unroll
  for (int j = 0; j < D; ++j) mu[j] = (PASS == 2 && k < m) ? means[k * 4 + j] : 0.0;
  double acc[10];
#pragma unroll
  for (int j = 0; j < 10; ++j) acc[j] = 0.0;
  for (int64_t t0 = c0; t0 < c1; t0 += kMomTile) {
    const int len = static_cast<int>(min64(kMomTile, c1 - t0));
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += 128) {
#pragma unroll
      for (int j = 0; j < D; ++j) xs[j][i] = x64[j * n + t0 + i];
      if (LABELS) ls[i] = labels[t0 + i];
    }
    __syncthreads();
    if (k < m) {
      for (int i = 0; i < len; ++i) {
        double w;
        if (LABELS) {
          if (ls[i] != k) continue;
          w = 1.0;
        } else {
          const double g = log_gamma[static_cast<int64_t>(k) * n + t0 + i];
          if (g < -700.0) continue;  // sogmm.cpp:415 select(0.0, ...)
          w = exp(g);
        }
        if (PASS == 1) {
          acc[0] += w;
#pragma unroll
          for (int j = 0; j < D; ++j) acc[1 + j] += __dmul_rn(w, xs[j][i]);
        } else {
          double d[D];
#pragma unroll
          for (int j = 0; j < D; ++j) d[j] = xs[j][i] - mu[j];
#pragma unroll
          for (int q = 0; q < npacked(D); ++q) {
            acc[q] += __dmul_rn(__dmul_rn(w, d[packed_row(q)]), d[packed_col(q)]);
          }
        }
      }
    }
  }
  if (k < m) {
    double* o = part + (static_cast<int64_t>(blockIdx.x) * m + k) * 10;
#pragma unroll
    for (int j = 0; j < 10; ++j) o[j] = acc[j];
  }
}

// reduce chunks in order; PASS 1 -> sums[m][5]; PASS 2 -> sums[m][10]
__global__ void moments_reduce_kernel(const double* __restrict__ part,
                                      int nchunks, int m, int width,
                                      double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m * width) return;
  const int k = i / width, j = i % width;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += part[(static_cast<int64_t>(c) * m + k) * 10 + j];
  out[k * width + j] = s;
}

template <int D>
__global__ void moments_means_kernel(const double* __restrict__ sums, int m,
                                     double* __restrict__ means,
                                     double* __restrict__ counts) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const double c = sums[k * 5];
  counts[k] = c;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    // degenerate: mean 0 (kernels.hpp:121-128)
    means[k * 4 + j] = (j < D && !(c < kDegenerateCount)) ? sums[k * 5 + 1 + j] / c : 0.0;
  }
}

template <int D>
__global__ void moments_finish_kernel(const double* __restrict__ sums2,
                                      const double* __restrict__ means,
                                      const double* __restrict__ counts, int m,
                                      double cov_reg, RecBuf rec) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const double cnt = counts[k];
  const bool keep = !(cnt < kDegenerateCount);
  const double inv = keep ? 1.0 / cnt : 0.0;
  double cov[10];
#pragma unroll
  for (int q = 0; q < 10; ++q) cov[q] = 0.0;
#pragma unroll
  for (int q = 0; q < npacked(D); ++q) {
    cov[q] = sums2[k * 10 + q] * inv;
    if (packed_row(q) == packed_col(q)) cov[q] += cov_reg;
  }
  float pc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) pc[j] = 0.f;
  double logdet = 0.0;
  int flags = keep ? 1 : 0;
  if (keep && factor_component<D>(cov, pc, &logdet)) flags |= 2;
  rec.count[k] = cnt;
#pragma unroll
  for (int j = 0; j < 4; ++j) rec.mean[k * 4 + j] = means[k * 4 + j];
#pragma unroll
  for (int j = 0; j < 10; ++j) rec.cov[k * 10 + j] = cov[j];
  rec.logdet[k] = logdet;
#pragma unroll
  for (int j = 0; j < 16; ++j) rec.pc[k * 16 + j] = pc[j];
  rec.flags[k] = flags;
}

// FP64 factors of buffer st->cur for the cholesky_cache API:
// out[k*33 + 0..15] = L (4x4 row-major), [16..31] = P = L^-1, [32] = logdet.
template <int D>
__global__ void factor_dump_kernel(ModelBuf b0, ModelBuf b1,
                                   const EmState* __restrict__ st, int m,
                                   double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const ModelBuf& mb = st->cur ? b1 : b0;
  double a[D][D];
#pragma unroll
  for (int q = 0; q < npacked(D); ++q) {
    a[packed_row(q)][packed_col(q)] = mb.cov[k * 10 + q];
    a[packed_col(q)][packed_row(q)] = mb.cov[k * 10 + q];
  }
  double l[D][D], p[D][D];
  double* o = out + static_cast<int64_t>(k) * 33;
  for (int i = 0; i < 33; ++i) o[i] = 0.0;
  if (!cholesky_d<D>(a, l)) return;
  lower_inverse_d<D>(l, p);
  double ld = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) ld += log(p[j][j]);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      o[i * 4 + j] = l[i][j];
      o[16 + i * 4 + j] = p[i][j];
    }
  o[32] = ld;
}

}  // namespace

cudaError_t launch_factor_dump(int d, const ModelBuf* bufs, const EmState* st,
                               int m, double* out, cudaStream_t s) {
  const int grid = (m + 127) / 128;
  if (d == 4)
    factor_dump_kernel<4><<<grid, 128, 0, s>>>(bufs[0], bufs[1], st, m, out);
  else
    factor_dump_kernel<3><<<grid, 128, 0, s>>>(bufs[0], bufs[1], st, m, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
cudaError_t launch_estep_ws_pre(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                                int kpad, int nch, const float2* lse, double* partials,
                                double* ll_part, int sm_count, cudaStream_t s, int* ncl_out) {
  if (pts.d == 4)
    return launch_estep_ws_pre_d<4>(pts, bufs, st, kpad, nch, lse, partials, ll_part, sm_count,
                                    s, ncl_out);
  return launch_estep_ws_pre_d<3>(pts, bufs, st, kpad, nch, lse, partials, ll_part, sm_count, s,
                                  ncl_out);
}

cudaError_t launch_estep_stats(const PointsDev& pts, const ModelBuf* bufs,
                               const EmState* st, int k0, double* partials,
                               double* ll_part, int exact_mode,
                               int sm_count, cudaStream_t s, int* ncl_out,
                               const ChunkScratch* chunk, const SparseScratch* sparse) {
  if (sparse)
    return launch_estep_sparse(pts, bufs, st, k0, partials, ll_part, exact_mode, sm_count, s,
                               ncl_out, *sparse);
  if (GMMB_CHUNKED && k0 > kCtaComps) {
    if (partials && !chunk) return cudaErrorInvalidValue;
    return launch_estep_chunked(pts, bufs, st, k0, partials, ll_part, exact_mode, sm_count, s,
                                ncl_out, chunk);
  }
  if (pts.d == 4)
    return launch_estep_d<4>(pts, bufs, st, k0, partials, ll_part, exact_mode,
                             sm_count, s, ncl_out);
  return launch_estep_d<3>(pts, bufs, st, k0, partials, ll_part, exact_mode,
                           sm_count, s, ncl_out);
}

cudaError_t launch_em_reduce(int d, const double* partials,
                             const double* ll_part, int ncl, int k0,
                             const EmState* st, double* red, double* red_ll,
                             cudaStream_t s) {
  const int warps = k0 + 1;
  const int wpb = 8;
  const int grid = (warps + wpb - 1) / wpb;
  if (d == 4)
    em_reduce_kernel<4><<<grid, wpb * 32, 0, s>>>(partials, ll_part, ncl, k0, st, red, red_ll);
  else
    em_reduce_kernel<3><<<grid, wpb * 32, 0, s>>>(partials, ll_part, ncl, k0, st, red, red_ll);
  return cudaGetLastError();
}

cudaError_t launch_em_reduce_finalize(int d, const double* partials, int ncl, int k0,
                                     const ModelBuf* bufs, const EmState* st, RecBuf rec,
                                     cudaStream_t s) {
  // many partials per component (small K: many E CTAs): a CTA per component
  if (ncl > GMMB_REDUCE_CTA_NCL) {
    if (d == 4)
      em_reduce_finalize_kernel<4, 4><<<k0, 128, 0, s>>>(partials, ncl, k0, bufs[0], bufs[1], st, rec);
    else
      em_reduce_finalize_kernel<3, 4><<<k0, 128, 0, s>>>(partials, ncl, k0, bufs[0], bufs[1], st, rec);
    return cudaGetLastError();
  }
  const int grid = (k0 + 3) / 4;
  if (d == 4)
    em_reduce_finalize_kernel<4, 1><<<grid, 128, 0, s>>>(partials, ncl, k0, bufs[0], bufs[1], st, rec);
  else
    em_reduce_finalize_kernel<3, 1><<<grid, 128, 0, s>>>(partials, ncl, k0, bufs[0], bufs[1], st, rec);
  return cudaGetLastError();
}

cudaError_t launch_em_finalize(int d, const double* red, const ModelBuf* bufs,
                               const EmState* st, int k0, RecBuf rec,
                               cudaStream_t s) {
  const int grid = (k0 + 127) / 128;
  if (d == 4)
    em_finalize_kernel<4><<<grid, 128, 0, s>>>(red, bufs[0], bufs[1], st, rec);
  else
    em_finalize_kernel<3><<<grid, 128, 0, s>>>(red, bufs[0], bufs[1], st, rec);
  return cudaGetLastError();
}

cudaError_t launch_commit(int d, int mode, const RecBuf rec, int k_in,
                          const double* red_ll, ModelBuf* bufs, EmState* st,
                          double* ll_trace, cudaStream_t s,
                          const cudaGraphConditionalHandle* cond,
                          const double* ll_part, int ncl) {
  const cudaGraphConditionalHandle h = cond ? *cond : cudaGraphConditionalHandle{};
  const int use = cond ? 1 : 0;
  if (d == 4)
    commit_kernel<4><<<1, 1024, 0, s>>>(mode, rec, k_in, red_ll, ll_part, ncl, bufs[0], bufs[1],
                                        st, ll_trace, h, use);
  else
    commit_kernel<3><<<1, 1024, 0, s>>>(mode, rec, k_in, red_ll, ll_part, ncl, bufs[0], bufs[1],
                                        st, ll_trace, h, use);
  return cudaGetLastError();
}

cudaError_t launch_prep(int d, ModelBuf* bufs, EmState* st, int k,
                        cudaStream_t s) {
  const int grid = (k + 127) / 128;
  if (d == 4)
    prep_kernel<4><<<grid, 128, 0, s>>>(bufs[0], bufs[1], st, k);
  else
    prep_kernel<3><<<grid, 128, 0, s>>>(bufs[0], bufs[1], st, k);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_moments_d(const double* x64, int64_t n,
                                    const int32_t* labels,
                                    const double* log_gamma, int m,
                                    double cov_reg, MomentsScratch scr,
                                    RecBuf rec, cudaStream_t s,
                                    void (*allreduce)(double*, int64_t, void*),
                                    void* ar_ctx) {
  const int nchunks = static_cast<int>((n + kMomChunk - 1) / kMomChunk);
  const dim3 grid(nchunks, (m + 127) / 128);
  const int rg1 = (m * 5 + 255) / 256, rg2 = (m * 10 + 255) / 256;
  if (labels)
    moments_kernel<D, true, 1><<<grid, 128, 0, s>>>(x64, n, labels, log_gamma, m, nullptr, scr.part);
  else
    moments_kernel<D, false, 1><<<grid, 128, 0, s>>>(x64, n, labels, log_gamma, m, nullptr, scr.part);
  moments_reduce_kernel<<<rg1, 256, 0, s>>>(scr.part, nchunks, m, 5, scr.sums);
  if (allreduce) allreduce(scr.sums, static_cast<int64_t>(m) * 5, ar_ctx);
  moments_means_kernel<D><<<(m + 127) / 128, 128, 0, s>>>(scr.sums, m, scr.means, scr.counts);
  if (labels)
    moments_kernel<D, true, 2><<<grid, 128, 0, s>>>(x64, n, labels, log_gamma, m, scr.means, scr.part);
  else
    moments_kernel<D, false, 2><<<grid, 128, 0, s>>>(x64, n, labels, log_gamma, m, scr.means, scr.part);
  moments_reduce_kernel<<<rg2, 256, 0, s>>>(scr.part, nchunks, m, 10, scr.sums);
  if (allreduce) allreduce(scr.sums, static_cast<int64_t>(m) * 10, ar_ctx);
  moments_finish_kernel<D><<<(m + 127) / 128, 128, 0, s>>>(scr.sums, scr.means, scr.counts, m, cov_reg, rec);
  return cudaGetLastError();
}

cudaError_t launch_moments(int d, const double* x64, int64_t n,
                           const int32_t* labels, const double* log_gamma,
                           int m, double cov_reg, MomentsScratch scr,
                           RecBuf rec, int /*sm_count*/, cudaStream_t s,
                           void (*allreduce)(double*, int64_t, void*),
                           void* ar_ctx) {
  if (d == 4)
    return launch_moments_d<4>(x64, n, labels, log_gamma, m, cov_reg, scr, rec, s, allreduce, ar_ctx);
  return launch_moments_d<3>(x64, n, labels, log_gamma, m, cov_reg, scr, rec, s, allreduce, ar_ctx);
}



}  // namespace gmmb
