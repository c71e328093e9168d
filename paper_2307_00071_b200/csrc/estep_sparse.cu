// estep_sparse.cu — the fused E step + sufficient statistics with exact-zero
// tile pruning (sm_100a).
//
// Reference semantics: e_step_into + m_step's weighted moments
// (/root/reference/proj/src/sogmm.cpp:341-383, 399-416; kernels.hpp:82-181),
// evaluated exactly like the dense kernels of em_kernels.cu: log2 densities
// Q = |P'x - P'mu'|^2 - base2 in FP32 on tile-recentred points, densities
// e = ex2.approx.ftz(-Q), an unshifted per-point normaliser (the exact max
// shift when it leaves [2^-64, 2^64]), centred statistics in FP32 pairs
// widened to FP64 every 16 points.
//
// Exact-zero pruning. ex2.approx.ftz returns exactly +0 for Q > 126 (the
// result would be subnormal), and a zero density adds exactly nothing to the
// normaliser or to any statistic (0 * finite = 0, s + 0 = s). So a
// (tile, component) pair whose Q exceeds 126 at every point of the tile can
// be skipped without changing a single bit the dense evaluation would add.
// An interval bound over the tile's bounding box decides it: with
// y = P'(x - mu) affine in x, each y_i ranges over [yc_i - r_i, yc_i + r_i]
// (yc at the box centre, r_i = sum_j |P'_ij| h_j), so
// Q >= sum_i max(0, |yc_i| - r_i)^2 - base2 =: LB. A pair is a candidate iff
// LB < 134 (8 of margin over 126 for FP32 rounding in the kernel and in the
// bound). On the cfg2 frame a 128-point tile keeps ~30 of 512 components.
//
// Points whose normaliser leaves [2^-64, 2^64] need the max-shifted sum,
// in which components with Q > 134 may no longer vanish; a tile with such a
// point (or exact_mode) is evaluated over all K components (same arithmetic
// as the dense kernel's exact path).
//
// Kernels per EM iteration:
//   block_cand_kernel  per block of 16 tiles (2048 points, static FP64 box):
//                      coarse candidate list (a superset of every tile's)
//   estep_sparse_kernel one warp per tile (dynamic tile queue): tile box,
//                      fine candidates (ascending), pass 1 (normalisers,
//                      lanes = candidates, point pairs in f32x2), pass 2
//                      (densities recomputed, responsibilities, statistics);
//                      per-(tile, candidate) FP64 statistics to a CSR pool,
//                      the tile's candidate bitmask + per-word prefix counts
//   sparse_reduce_kernel per (32-component word, tile range): fixed-order sums
//                      -> per-range partials [R][K][NS] + ll partials [R], the
//                      layout of the dense kernels (em_reduce_finalize / the
//                      sharded em_reduce + all-reduce + em_finalize follow)
// Every sum has a fixed order independent of scheduling: bit-reproducible.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "em_kernels.cuh"
#include "f32x2.cuh"

namespace gmmb {

namespace {

using namespace dev;

#ifdef GMMB_SP_PROF
__device__ unsigned long long g_sp_prof[4 * 262144];  // per unit: t0, t1, (sm, C), flags
__device__ unsigned g_sp_ph[6 * 262144];             // per unit: phase durations (cycles)
#define SP_PH(i) unsigned long long ph##i = clock64()
#else
#define SP_PH(i)
#endif
constexpr int kSpEvCalls = 256;
cudaEvent_t g_sp_ev[kSpEvCalls][4] = {};
int g_sp_nev = 0;
constexpr int kBlkTiles = 16;     // tiles per culling block
#ifndef GMMB_RED_STEP
#define GMMB_RED_STEP 2
#endif
#ifndef GMMB_RED_UNITS
#define GMMB_RED_UNITS 128
#endif
constexpr int kRedStep = GMMB_RED_STEP;  // units whose statistics the reduce loads together
constexpr int kItem = 32;         // points per item (one per lane); a work unit is U = 1, 2
constexpr int kItemsPerTile = kTile / kItem;  // or 4 consecutive items of one layout tile
constexpr int kSpWarps = 8;       // warps per CTA of the main kernel
#ifndef GMMB_SP_MINB
#define GMMB_SP_MINB 2
#endif
constexpr int kSpMinBlocks = GMMB_SP_MINB;  // two CTAs per SM (128 registers)
constexpr int kListCap = 1024;    // candidate list entries per warp (more: every component)
constexpr int kSlice = 16;        // points per FP32 partial (widened to FP64 after)
constexpr float kQCut = 134.f;    // candidates: LB < 134 (ex2.approx.ftz(-Q) = 0 for Q > 126)
// (GMMB_SPARSE_QCUT overrides it: a validation knob, e.g. 1e30 keeps every pair)

// pool entries: the nstats(D) FP64 statistics of one (unit, candidate),
// padded to an even count (16-byte loads in the reduce). (FP32 entries halve
// the bytes but measured slower: the reduce is latency-bound, and the
// conversions lengthen its dependent chain: cfg4 E reduce 373 -> 480 us.)
__host__ __device__ constexpr int pool_stride(int d) { return (nstats(d) + 1) & ~1; }
// Heavy units (many candidates) are split over up to kMaxSplit warps by
// 16-point slices: a unit whose previous iteration had C > kHeavyC candidates
// is queued first, split into S = 2^j sub-units while C / S > split_c, where
// split_c = (96, or 160 for K > 1024) x (units per 4 warps, at least 1): a split only pays when
// one unit is a large share of a warp's work (each sub-unit repeats the
// unit's loads and candidate filter).
constexpr int kMaxSplit = kSparseMaxSplit;
#ifndef GMMB_HEAVY_C
#define GMMB_HEAVY_C 48
#endif
constexpr int kHeavyC = GMMB_HEAVY_C;
#ifndef GMMB_SPLIT_C
#define GMMB_SPLIT_C 0  // 0: by K (below)
#endif
constexpr int kSplitC = GMMB_SPLIT_C;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// interval lower bound of |P'(x - mu)|^2 over the box centre v = bc - mu'
// (FP32) and half-widths h; P' packed lower triangle (CompConst.p)
template <int D>
__device__ __forceinline__ float box_lb(const float* P, const float (&v)[4], const float (&h)[4]) {
  float lb = 0.f;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float yc = 0.f, r = 0.f;
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      const float p = P[i * (i + 1) / 2 + j];
      yc = fmaf(p, v[j], yc);
      r = fmaf(fabsf(p), h[j], r);
    }
    const float dlt = fmaxf(fabsf(yc) - r, 0.f);
    lb = fmaf(dlt, dlt, lb);
  }
  return lb;
}

// interval upper bound of |P'(x - mu)|^2 over the same box
template <int D>
__device__ __forceinline__ float box_ub(const float* P, const float (&v)[4], const float (&h)[4]) {
  float ub = 0.f;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    float yc = 0.f, r = 0.f;
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      const float p = P[i * (i + 1) / 2 + j];
      yc = fmaf(p, v[j], yc);
      r = fmaf(fabsf(p), h[j], r);
    }
    const float dlt = fabsf(yc) + r;
    ub = fmaf(dlt, dlt, ub);
  }
  return ub;
}

// ---- static per-layout block boxes (FP64 centre, FP32 half-widths rounded up)
__global__ void __launch_bounds__(kTile)
    block_box_kernel(const float4* __restrict__ xt, const double* __restrict__ tc, int64_t n,
                     int ntiles, double* __restrict__ bc, float4* __restrict__ bh) {
  __shared__ double red[8][kTile];
  const int b = blockIdx.x, tid = threadIdx.x;
  double lo[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  double hi[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  const int t1 = min(ntiles, (b + 1) * kBlkTiles);
  for (int t = b * kBlkTiles; t < t1; ++t) {
    const int64_t i = static_cast<int64_t>(t) * kTile + tid;
    if (i >= n) break;
    const float4 x = xt[i];
    const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double a = tc[static_cast<int64_t>(t) * 4 + j] + static_cast<double>(xv[j]);
      lo[j] = fmin(lo[j], a);
      hi[j] = fmax(hi[j], a);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    red[j][tid] = lo[j];
    red[4 + j][tid] = hi[j];
  }
  __syncthreads();
  for (int off = kTile / 2; off >= 1; off >>= 1) {
    if (tid < off) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        red[j][tid] = fmin(red[j][tid], red[j][tid + off]);
        red[4 + j][tid] = fmax(red[4 + j][tid], red[4 + j][tid + off]);
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    float h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double c = 0.5 * (red[j][0] + red[4 + j][0]);
      bc[static_cast<int64_t>(b) * 4 + j] = c;
      const double hw = fmax(red[4 + j][0] - c, c - red[j][0]);
      h[j] = __double2float_ru(hw * (1.0 + 0x1p-20) + 1e-30);
    }
    bh[b] = make_float4(h[0], h[1], h[2], h[3]);
  }
}

// ---- coarse candidates per block (ascending component order) --------------
#ifndef GMMB_BC_THREADS
#define GMMB_BC_THREADS 256
#endif
constexpr int kBcThreads = GMMB_BC_THREADS;  // components per pass of block_cand
template <int D>
__global__ void __launch_bounds__(kBcThreads)
    block_cand_kernel(const double* __restrict__ bc, const float4* __restrict__ bh, ModelBuf b0,
                      ModelBuf b1, const EmState* __restrict__ st, int kcap,
                      int* __restrict__ blist, float4* __restrict__ brec, int* __restrict__ bcnt,
                      int* __restrict__ ctl, float qcut) {
  __shared__ int wcnt[kBcThreads / 32];
  __shared__ int s_base;
  if (st->done) return;
  // item queues and pool cursor restart every iteration (ctl[2] overflow and
  // ctl[4..5] evaluated units accumulate over the fit; zeroed by the driver);
  // the heavy list this iteration appends to (parity of iter + 1) restarts;
  // ctl[8] is the item epoch (never reset)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl[0] = 0;
    ctl[1] = 0;
    ctl[3] = 0;
    ctl[6 + ((st->iter + 1) & 1)] = 0;
    ctl[9 + ((st->iter + 1) & 1)] = 0;
    // +2 at a run's first iteration: marks left by an abandoned run (pool
    // overflow re-run) can never match
    ctl[8] += st->iter == 0 ? 2 : 1;
  }
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int k_cur = st->k_cur;
  const ModelBuf& mb = st->cur ? b1 : b0;
  double c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = bc[static_cast<int64_t>(b) * 4 + j];
  const float4 hb = bh[b];
  const float h[4] = {hb.x, hb.y, hb.z, hb.w};
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int k0 = 0; k0 < k_cur; k0 += kBcThreads) {
    const int k = k0 + tid;
    bool cand = false;
    float4 a0, a1, a2;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (k < k_cur) {
      const float4* c4 = reinterpret_cast<const float4*>(mb.cst + k);
      a0 = c4[0];
      a1 = c4[1];
      a2 = c4[2];
      const float P[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = j < D ? -static_cast<float>(mb.mu[k * 4 + j] - c[j]) : 0.f;
      const float lb = box_lb<D>(P, v, h);
      // superset of the fine test (looser slack, +1)
      cand = fmaf(lb, -0x1p-9f, lb) - P[10] < qcut + 1.f;
    }
    const unsigned m = __ballot_sync(0xffffffffu, cand);
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    int pre = s_base;
    for (int q = 0; q < w; ++q) pre += wcnt[q];
    if (cand) {
      // the candidate's id + bound record (factor, base2, mean relative to the
      // block centre in FP32): the units' filters read these contiguously
      const int64_t pos = static_cast<int64_t>(b) * kcap + pre + __popc(m & lanemask_lt());
      blist[pos] = k;
      float4* rec = brec + pos * 4;
      rec[0] = a0;
      rec[1] = a1;
      rec[2] = a2;
      rec[3] = make_float4(-v[0], -v[1], -v[2], -v[3]);
    }
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int q = 0; q < kBcThreads / 32; ++q) tot += wcnt[q];
      s_base += tot;
    }
    __syncthreads();
  }
  if (tid == 0) bcnt[b] = s_base;
}

// One candidate's tile-relative constants (lane-private scalars).
template <int D>
struct Cand {
  float P[npacked(D)];
  float nb[D];   // -P' mu' (FP64 dot of the FP32 factor with the FP32-rounded mu')
  float nbase;   // -base2
  float nmu[D];  // -mu' (statistics centre: x - mu')
};

template <int D>
__device__ __forceinline__ void load_cand(Cand<D>& cd, int k, const ModelBuf& mb, const double (&ct)[4]) {
  constexpr int NP = npacked(D);
  if (k < 0) {
#pragma unroll
    for (int q = 0; q < NP; ++q) cd.P[q] = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      cd.nb[i] = 0.f;
      cd.nmu[i] = 0.f;
    }
    cd.nbase = INFINITY;  // e = 2^-inf = 0
    return;
  }
  const float4* c4 = reinterpret_cast<const float4*>(mb.cst + k);
  const float4 a0 = c4[0], a1 = c4[1], a2 = c4[2];
  const float cc[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
#pragma unroll
  for (int q = 0; q < NP; ++q) cd.P[q] = cc[q];
  cd.nbase = -cc[10];
  float muf[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    muf[j] = static_cast<float>(mb.mu[k * 4 + j] - ct[j]);
    cd.nmu[j] = -muf[j];
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q <= i; ++q)
      s = fma(static_cast<double>(cd.P[i * (i + 1) / 2 + q]), static_cast<double>(muf[q]), s);
    cd.nb[i] = static_cast<float>(-s);
  }
}

// Q of the point pair (p, p + 1) for the lane's candidate (FFMA2 chains with
// the broadcast constant operand), points from the warp's SoA tile
template <int D>
__device__ __forceinline__ f2_t dens_pair(const Cand<D>& cd, const f2_t (&X)[D]) {
  const f2_t Y0 = fma2(X[0], pk(cd.P[0], cd.P[0]), pk(cd.nb[0], cd.nb[0]));
  const f2_t Y1 = fma2(X[1], pk(cd.P[2], cd.P[2]), fma2(X[0], pk(cd.P[1], cd.P[1]), pk(cd.nb[1], cd.nb[1])));
  const f2_t Y2 =
      fma2(X[2], pk(cd.P[5], cd.P[5]),
           fma2(X[1], pk(cd.P[4], cd.P[4]), fma2(X[0], pk(cd.P[3], cd.P[3]), pk(cd.nb[2], cd.nb[2]))));
  f2_t q = fma2(Y2, Y2, fma2(Y1, Y1, fma2(Y0, Y0, pk(cd.nbase, cd.nbase))));
  if constexpr (D == 4) {
    const f2_t Y3 = fma2(
        X[3], pk(cd.P[9], cd.P[9]),
        fma2(X[2], pk(cd.P[8], cd.P[8]),
             fma2(X[1], pk(cd.P[7], cd.P[7]), fma2(X[0], pk(cd.P[6], cd.P[6]), pk(cd.nb[3], cd.nb[3])))));
    q = fma2(Y3, Y3, q);
  }
  return q;
}

template <int D>
__device__ __forceinline__ void load_pair(const float (*xs)[kTile], int p, f2_t (&X)[D]) {
#pragma unroll
  for (int j = 0; j < D; ++j) X[j] = *reinterpret_cast<const f2_t*>(&xs[j][p]);
}

struct SpWarpSmem {
  double acc[15][32];   // FP64 statistics of the lanes' candidates (one group)
  float xs[4][kTile];   // the unit's points (SoA, tile-relative)
  float ssum[kTile];    // per-point normaliser partials (pass 1), then 1/S
  float sh[kTile];      // per-point shift (exact path), else 0
  unsigned short list[kListCap];  // fine candidates, ascending
};
// per warp: SpWarpSmem | candidate bitmask (K/32 words)
__host__ __device__ inline size_t warp_smem_bytes(int kcap) {
  return (sizeof(SpWarpSmem) + sizeof(unsigned) * ((kcap + 31) / 32) + 15) & ~size_t(15);
}

// ---- main kernel ------------------------------------------------------------
// Dynamic smem: kSpWarps x [SpWarpSmem | list (kcap ints) | mask (kw words)].
template <int D>
__global__ void __launch_bounds__(kSpWarps * 32, kSpMinBlocks)
    estep_sparse_kernel(const float4* __restrict__ xt, const double* __restrict__ tc, int64_t n,
                        int nitems, ModelBuf b0, ModelBuf b1, const EmState* __restrict__ st,
                        int kcap, const int* __restrict__ blist, const float4* __restrict__ brec,
                        const int* __restrict__ bcnt, const double* __restrict__ bcen, int ucap,
                        int* __restrict__ ctl, double* __restrict__ pool, int64_t pool_cap,
                        int* __restrict__ toff, unsigned* __restrict__ maskT,
                        unsigned short* __restrict__ preT, double* __restrict__ ll_tile,
                        int* __restrict__ heavy, unsigned* __restrict__ done,
                        int exact_mode, float qcut, int U, int split_c) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kNSP = pool_stride(D);
  if (st->done) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kw = (kcap + 31) / 32;
  const size_t wbytes = warp_smem_bytes(kcap);
  SpWarpSmem& ws = *reinterpret_cast<SpWarpSmem*>(smem_raw + wbytes * warp);
  unsigned* mw = reinterpret_cast<unsigned*>(smem_raw + wbytes * warp + sizeof(SpWarpSmem));
  unsigned short* list = ws.list;
  double (*facc)[32] = ws.acc;
  const int k_cur = st->k_cur;
  const ModelBuf& mb = st->cur ? b1 : b0;
  unsigned long long evaluated = 0;  // units evaluated (lane 0)

  // Work order: first the units that were heavy in the previous iteration
  // (more than kHeavyC candidates; longest first is the classic fix for a
  // tail): the split ones' sub-units (list front), then the rest (list back);
  // then every unit in index order, skipping the heavy ones (marked with this
  // epoch by the previous iteration, before this kernel started, so no unit
  // is ever taken twice). The order changes no result: a (sub-)unit's output
  // depends only on the unit, its slices and the split S, and S is a function
  // of the previous iteration's candidate count.
  const int par = st->iter & 1;
  const int hcap = kMaxSplit * nitems;
  const int nA = ctl[6 + par], nheavy = nA + ctl[9 + par];
  const int* hl_cur = heavy + static_cast<int64_t>(par) * hcap;
  int* hl_next = heavy + static_cast<int64_t>(par ^ 1) * hcap;
  const unsigned epoch = static_cast<unsigned>(ctl[8]);
  // marks by parity: this iteration reads its own, the pushes below write the
  // next iteration's (a shared array would let a heavy unit re-marked early
  // be taken again by the normal queue)
  const unsigned* done_cur = done + static_cast<int64_t>(par) * nitems;
  unsigned* done_next = done + static_cast<int64_t>(par ^ 1) * nitems;
  int* toffS = toff + nitems;          // [nitems][kMaxSplit] sub-unit pool bases
  double* llS = ll_tile + nitems;      // [nitems][kMaxSplit] sub-unit ll
  for (;;) {
    // task = (unit << 6) | (sub << 3) | (S - 1)
    int task = 0;
    if (lane == 0) {
      const int h = nheavy > 0 ? atomicAdd(&ctl[3], 1) : nheavy;
      if (h < nA) {
        task = hl_cur[h];
      } else if (h < nheavy) {
        task = hl_cur[hcap - 1 - (h - nA)];
      } else {
        int u;
        do {
          u = atomicAdd(&ctl[0], 1);
        } while (u < nitems && done_cur[u] == epoch);
        task = u < nitems ? (u << 6) : -1;
      }
    }
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task < 0) break;
#ifdef GMMB_SP_COUNT
    if (lane == 0) atomicAdd(&ctl[12], 1);
#endif
    const int it = task >> 6;
    const int sub = (task >> 3) & 7, nsub = (task & 7) + 1;
    // unit it: points [it U 32, (it + 1) U 32) of the sorted cloud, one tile;
    // this task: its 16-point slices [sl0, sl1)
    const int64_t p0 = static_cast<int64_t>(it) * U * kItem;
    const int t = static_cast<int>(p0 / kTile);
    const int nsl = 2 * U;  // 16-point slices
    const int sl0 = sub * nsl / nsub, sl1 = (sub + 1) * nsl / nsub;
#ifdef GMMB_SP_PROF
    unsigned long long prof_t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_t0));
#endif
    SP_PH(0);
    const int npts = static_cast<int>(min64(U * kItem, n - p0));  // may be <= 0 (padding)
    // issued first, independent of the points: the block's candidate count,
    // centre and first group of records (the filter below needs the box)
    const int blk = t / kBlkTiles;
    const int* bl = blist + static_cast<int64_t>(blk) * kcap;
    const float4* br = brec + static_cast<int64_t>(blk) * kcap * 4;
    const int cb_ld = bcnt[blk];
    double bce[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) bce[j] = bcen[blk * 4 + j];
    int kn = -1;
    float4 n0 = make_float4(0.f, 0.f, 0.f, 0.f), n1 = n0, n2 = n0, n3 = n0;
    if (lane < kcap) {
      kn = __ldcg(bl + lane);
      const float4* rec = br + static_cast<int64_t>(lane) * 4;
      n0 = __ldcg(rec);
      n1 = __ldcg(rec + 1);
      n2 = __ldcg(rec + 2);
      n3 = __ldcg(rec + 3);
    }
    double ct[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ct[j] = tc[static_cast<int64_t>(t) * 4 + j];
    // ---- tile points -> SoA smem + bounding box of the valid points
    float lo[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    float hi[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int q = 0; q < U; ++q) {
      const int p = lane + 32 * q;
      const float4 x = xt[p0 + p];  // (the padding of the last tile is zero)
      const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        ws.xs[j][p] = xv[j];
        if (p < npts) {
          lo[j] = fminf(lo[j], xv[j]);
          hi[j] = fmaxf(hi[j], xv[j]);
        }
      }
      ws.ssum[p] = 0.f;
      ws.sh[p] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        lo[j] = fminf(lo[j], __shfl_xor_sync(0xffffffffu, lo[j], off));
        hi[j] = fmaxf(hi[j], __shfl_xor_sync(0xffffffffu, hi[j], off));
      }
    }
    float bcv[4], hw[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      bcv[j] = 0.5f * (lo[j] + hi[j]);
      // half-width rounded up (covers the rounding of the centre)
      hw[j] = fmaxf(hi[j] - bcv[j], bcv[j] - lo[j]) * (1.f + 0x1p-20f) + 1e-30f;
    }
    SP_PH(1);
    // ---- fine candidates (ascending): the block's list filtered by the tile box
    const int cb = npts > 0 ? cb_ld : 0;
    // box centre relative to the block centre (the records' frame); the
    // FP32 rounding of the two frames (~1e-7 of the block extent) is far
    // inside the 8-unit margin of the cut
    float bcb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) bcb[j] = bcv[j] + static_cast<float>(ct[j] - bce[j]);
    int C = 0;
    for (int c0 = 0; c0 < cb; c0 += 32) {
      const int ci = c0 + lane;
      bool cand = false;
      int k = -1;
      // this group's records (prefetched), then the next group's in flight
      const float4 a0 = n0, a1 = n1, a2 = n2, mr = n3;
      const int kc = kn;
      if (c0 + 32 < cb && ci + 32 < cb) {
        kn = __ldcg(bl + ci + 32);
        const float4* rec = br + static_cast<int64_t>(ci + 32) * 4;
        n0 = __ldcg(rec);
        n1 = __ldcg(rec + 1);
        n2 = __ldcg(rec + 2);
        n3 = __ldcg(rec + 3);
      }
      if (ci < cb) {
        k = kc;
        const float P[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
        const float mu_b[4] = {mr.x, mr.y, mr.z, mr.w};
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = j < D ? bcb[j] - mu_b[j] : 0.f;
        // slack: 2^-10 relative + the frames' rounding (hw already rounds up)
        const float lb = box_lb<D>(P, v, hw);
        cand = fmaf(lb, -0x1p-10f, lb) - P[10] < qcut;
      }
      const unsigned m = __ballot_sync(0xffffffffu, cand);
      if (cand && C + __popc(m) <= kListCap)
        list[C + __popc(m & lanemask_lt())] = static_cast<unsigned short>(k);
      C += __popc(m);
    }
    // more candidates than the list holds: every component (a superset)
    bool allk = C > kListCap;
    if (allk) C = k_cur;
    __syncwarp();
    auto cand_at = [&](int i) -> int { return allk ? i : list[i]; };
    // the atomics whose results are needed only after the passes go out now
    // (their latency hides behind the passes): the overflow-region slots and
    // the next iteration's heavy-list slots (lane 0 holds the results)
    const int C_pre = C;
    int o_pre = 0, h_pre = 0, ns_pre = 0;
    if (lane == 0) {
      if (C > ucap || nsub > 1) o_pre = atomicAdd(&ctl[1], C);
      if (sub == 0 && C > kHeavyC) {
        ns_pre = 1;
        while (ns_pre < nsl && ns_pre < kMaxSplit && C > split_c * ns_pre) ns_pre *= 2;
        h_pre = atomicAdd(&ctl[(ns_pre > 1 ? 6 : 9) + (par ^ 1)], ns_pre > 1 ? ns_pre : 1);
      }
    }
    SP_PH(2);

    // ---- one group (C <= 32, most tiles): both passes per 16-point slice, the
    // densities kept in registers between them (no recomputation). A slice
    // that needs the exact path abandons it for the general path below.
    constexpr int NS = nstats(D);
    bool fused = false;
    if (C <= 32 && exact_mode == 0) {
      fused = true;
      Cand<D> cd;
      load_cand<D>(cd, lane < C ? cand_at(lane) : -1, mb, ct);
#pragma unroll
      for (int q = 0; q < NS; ++q) facc[q][lane] = 0.0;
      double fll = 0.0;
      #pragma unroll 1
        for (int s = sl0; s < sl1; ++s) {
        float e[kSlice], v[kSlice];
#pragma unroll
        for (int pp = 0; pp < kSlice; pp += 2) {
          f2_t X[D];
          load_pair<D>(ws.xs, s * kSlice + pp, X);
          const f2_t Q = dens_pair<D>(cd, X);
          e[pp] = ex2n(lo2(Q));
          e[pp + 1] = ex2n(hi2(Q));
          v[pp] = e[pp];
          v[pp + 1] = e[pp + 1];
        }
        const float S = warp_reduce_scatter<kSlice, false>(v, lane);
        const int pq = s * kSlice + (lane >> 1);
        const bool valid = pq < npts;
        if (__any_sync(0xffffffffu, valid && !(S >= 0x1p-64f && S <= 0x1p64f))) {
          fused = false;
          break;
        }
        if (valid && (lane & 1) == 0) fll += static_cast<double>(lg2f(S));
        if ((lane & 1) == 0) ws.ssum[pq] = valid ? rcpf(S) : 0.f;
        __syncwarp();
        f2_t ACC[NS];
#pragma unroll
        for (int q = 0; q < NS; ++q) ACC[q] = 0ull;
#pragma unroll
        for (int pp = 0; pp < kSlice; pp += 2) {
          const int p = s * kSlice + pp;
          f2_t X[D];
          load_pair<D>(ws.xs, p, X);
          const f2_t R = mul2(pk(e[pp], e[pp + 1]), *reinterpret_cast<const f2_t*>(&ws.ssum[p]));
          f2_t DD[D], W[D];
#pragma unroll
          for (int i = 0; i < D; ++i) {
            DD[i] = add2(X[i], pk(cd.nmu[i], cd.nmu[i]));
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
        }
#pragma unroll
        for (int q = 0; q < NS; ++q) facc[q][lane] += f32_to_f64(lo2(ACC[q]) + hi2(ACC[q]));
      }
      if (fused) {
        // the slices' ll in point order: lanes 0, 2, .. hold points 0..15 of each slice
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) fll += __shfl_xor_sync(0xffffffffu, fll, off);
        if (lane == 0) {
          if (nsub == 1) ll_tile[it] = fll;
          else llS[it * kMaxSplit + sub] = fll;
        }
      } else {
        for (int q = 0; q < U; ++q) ws.ssum[lane + 32 * q] = 0.f;
        __syncwarp();
      }
    }

    // ---- pass 1: normalisers over the candidates
    auto pass1 = [&](int nc) {
      for (int g = 0; g < nc; g += 32) {
        Cand<D> cd;
        load_cand<D>(cd, g + lane < nc ? cand_at(g + lane) : -1, mb, ct);
        #pragma unroll 1
        for (int s = sl0; s < sl1; ++s) {
          float v[kSlice];
#pragma unroll
          for (int pp = 0; pp < kSlice; pp += 2) {
            f2_t X[D];
            load_pair<D>(ws.xs, s * kSlice + pp, X);
            const f2_t Q = dens_pair<D>(cd, X);
            v[pp] = ex2n(lo2(Q));
            v[pp + 1] = ex2n(hi2(Q));
          }
          const float r = warp_reduce_scatter<kSlice, false>(v, lane);
          if ((lane & 1) == 0) ws.ssum[s * kSlice + (lane >> 1)] += r;
        }
      }
      __syncwarp();
    };
    unsigned xslices = 0;
    if (!fused) {
    pass1(C);
    // exact path needed anywhere in the item? (per 16-point slice, like the
    // dense kernel's sub-tiles)
    for (int q = 0; q < U; ++q) {
      const int p = lane + 32 * q;
      const float S = ws.ssum[p];
      const bool own = p >= sl0 * kSlice && p < sl1 * kSlice;
      const bool bad = own && p < npts && (exact_mode != 0 || !(S >= 0x1p-64f && S <= 0x1p64f));
      const unsigned m = __ballot_sync(0xffffffffu, bad);
      // lanes 0..15 -> slice 2q, 16..31 -> slice 2q + 1
      if (m & 0xffffu) xslices |= 1u << (2 * q);
      if (m & 0xffff0000u) xslices |= 2u << (2 * q);
    }
    if (xslices) {
      // a split unit's sub-units could re-select different candidate lists
      // here: flag it, the EM run is repeated without splits
      if (nsub > 1 && lane == 0) atomicOr(&ctl[2], 2);
      // Max shift on the flagged slices (the dense kernel's exact path). The
      // components that can matter: with UB_min the smallest upper bound of
      // Q over the tile box among ALL components, every point's minimum Q is
      // <= UB_min, so a component whose lower bound is >= max(UB_min, 0) + 134
      // has density 0 both shifted (Q - min Q >= 134) and unshifted.
      float ubmin = INFINITY;
      for (int k = lane; k < k_cur; k += 32) {
        const float4* c4 = reinterpret_cast<const float4*>(mb.cst + k);
        const float4 a0 = c4[0], a1 = c4[1], a2 = c4[2];
        const float P[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[j] = j < D ? bcv[j] - static_cast<float>(mb.mu[k * 4 + j] - ct[j]) : 0.f;
        ubmin = fminf(ubmin, box_ub<D>(P, v, hw) * (1.f + 0x1p-10f) - P[10]);
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1)
        ubmin = fminf(ubmin, __shfl_xor_sync(0xffffffffu, ubmin, off));
      const float xcut = fmaxf(ubmin, 0.f) + qcut;
      C = 0;
      allk = false;
      for (int k0 = 0; k0 < k_cur; k0 += 32) {
        const int k = k0 + lane;
        bool cand = false;
        if (k < k_cur) {
          const float4* c4 = reinterpret_cast<const float4*>(mb.cst + k);
          const float4 a0 = c4[0], a1 = c4[1], a2 = c4[2];
          const float P[12] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            v[j] = j < D ? bcv[j] - static_cast<float>(mb.mu[k * 4 + j] - ct[j]) : 0.f;
          const float lb = box_lb<D>(P, v, hw);
          cand = !(fmaf(lb, -0x1p-10f, lb) - P[10] >= xcut);  // NaN / inf bounds: keep
        }
        const unsigned m = __ballot_sync(0xffffffffu, cand);
        if (cand && C + __popc(m) <= kListCap)
          list[C + __popc(m & lanemask_lt())] = static_cast<unsigned short>(k);
        C += __popc(m);
      }
      if (C > kListCap) {
        C = k_cur;
        allk = true;
      }
      __syncwarp();
      for (int q = 0; q < U; ++q) ws.ssum[lane + 32 * q] = -INFINITY;
      __syncwarp();
      for (int g = 0; g < C; g += 32) {  // per-point max of -Q
        Cand<D> cd;
        load_cand<D>(cd, g + lane < C ? cand_at(g + lane) : -1, mb, ct);
        #pragma unroll 1
        for (int s = 0; s < nsl; ++s) {
          if (!((xslices >> s) & 1u)) continue;
          float v[kSlice];
#pragma unroll
          for (int pp = 0; pp < kSlice; pp += 2) {
            f2_t X[D];
            load_pair<D>(ws.xs, s * kSlice + pp, X);
            const f2_t Q = dens_pair<D>(cd, X);
            v[pp] = -lo2(Q);
            v[pp + 1] = -hi2(Q);
          }
          const float r = warp_reduce_scatter<kSlice, true>(v, lane);
          if ((lane & 1) == 0) {
            float& o = ws.ssum[s * kSlice + (lane >> 1)];
            o = fmaxf(o, r);
          }
        }
      }
      __syncwarp();
      for (int q = 0; q < U; ++q) {
        const int p = lane + 32 * q;
        const float M = ws.ssum[p];
        ws.sh[p] = ((xslices >> (p / kSlice)) & 1u) ? (M == -INFINITY ? 0.f : M) : 0.f;
        ws.ssum[p] = 0.f;
      }
      __syncwarp();
      // normalisers (shifted on flagged slices)
      for (int g = 0; g < C; g += 32) {
        Cand<D> cd;
        load_cand<D>(cd, g + lane < C ? cand_at(g + lane) : -1, mb, ct);
        #pragma unroll 1
        for (int s = sl0; s < sl1; ++s) {
          float v[kSlice];
#pragma unroll
          for (int pp = 0; pp < kSlice; pp += 2) {
            f2_t X[D];
            load_pair<D>(ws.xs, s * kSlice + pp, X);
            f2_t Q = dens_pair<D>(cd, X);
            Q = add2(Q, *reinterpret_cast<const f2_t*>(&ws.sh[s * kSlice + pp]));
            v[pp] = ex2n(lo2(Q));
            v[pp + 1] = ex2n(hi2(Q));
          }
          const float r = warp_reduce_scatter<kSlice, false>(v, lane);
          if ((lane & 1) == 0) ws.ssum[s * kSlice + (lane >> 1)] += r;
        }
      }
      __syncwarp();
    }
    // 1/S, log-likelihood (log2 units; one lane per point, fixed order)
    double ll = 0.0;
    for (int q = 0; q < U; ++q) {
      const int p = lane + 32 * q;
      const bool own = p >= sl0 * kSlice && p < sl1 * kSlice && p < npts;
      const float S = ws.ssum[p];
      if (own) ll += static_cast<double>(ws.sh[p] + lg2f(S));
      ws.ssum[p] = own ? rcpf(S) : 0.f;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, off);
    if (lane == 0) {
      if (nsub == 1) ll_tile[it] = ll;
      else llS[it * kMaxSplit + sub] = ll;
    }
    }  // !fused

    SP_PH(3);
    // ---- output slots (CSR pool) + the unit's candidate bitmask
    // fixed slots of ucap entries per whole unit; more candidates, and every
    // sub-unit of a split unit: the overflow region after them (cursor ctl[1])
    int64_t base = static_cast<int64_t>(it) * ucap;
    if (C > ucap || nsub > 1) {
      int o = o_pre;
      // (the exact path may have re-selected the candidates: new slots)
      if (lane == 0 && (C != C_pre || !(C_pre > ucap || nsub > 1))) o = atomicAdd(&ctl[1], C);
      base = static_cast<int64_t>(nitems) * ucap + __shfl_sync(0xffffffffu, o, 0);
    }
    const bool fits = base + C <= pool_cap;
    if (lane == 0) {
      if (nsub == 1) {
        toff[it] = fits ? static_cast<int>(base) : -1;
      } else {
        toff[it] = -nsub;  // split: the reduce adds the sub-units' entries
        toffS[it * kMaxSplit + sub] = fits ? static_cast<int>(base) : -1;
      }
      if (!fits) atomicOr(&ctl[2], 1);  // pool overflow: the host re-runs larger
    }
    // the next iteration's heavy list (from the whole unit's count: every
    // sub-unit has the same list; sub-unit 0 reports it)
    // (the candidate count before any exact-path re-selection decides)
    if (lane == 0 && ns_pre > 0) {
      if (ns_pre > 1) {
        for (int q = 0; q < ns_pre; ++q) hl_next[h_pre + q] = (it << 6) | (q << 3) | (ns_pre - 1);
      } else {
        hl_next[hcap - 1 - h_pre] = it << 6;
      }
      done_next[it] = epoch + 1;  // the next iteration's normal queue skips it
    }
    // the bitmask: identical for every sub-unit; sub-unit 0 writes it
    const bool wmask = sub == 0;
    for (int w = lane; w < kw; w += 32) mw[w] = 0u;
    __syncwarp();
    // the candidates' bits, grouped per word in registers (no shared atomics:
    // ascending candidates share words, which would serialise them)
    for (int i0 = 0; i0 < C; i0 += 32) {
      const int i = i0 + lane;
      const int k = i < C ? cand_at(i) : -1;
      const int wk = k >= 0 ? (k >> 5) : -1;
      // ascending: each word's candidates are a run of lanes; segmented
      // inclusive OR-scan, the run's last lane writes
      unsigned bits = k >= 0 ? 1u << (k & 31) : 0u;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned ob = __shfl_up_sync(0xffffffffu, bits, off);
        const int ow = __shfl_up_sync(0xffffffffu, wk, off);
        if (lane >= off && ow == wk) bits |= ob;
      }
      const int nw = __shfl_down_sync(0xffffffffu, wk, 1);
      if (k >= 0 && (lane == 31 || nw != wk)) mw[wk] |= bits;
      __syncwarp();
    }
    {
      int run = 0;
      for (int w0 = 0; w0 < kw; w0 += 32) {
        const int w = w0 + lane;
        const unsigned word = w < kw ? mw[w] : 0u;
        int c = __popc(word);
        int incl = c;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += o;
        }
        if (w < kw && wmask) {
          // a sub-unit that did not fit leaves its base -1: the reduce skips it
          maskT[static_cast<int64_t>(w) * nitems + it] = (fits || nsub > 1) ? word : 0u;
          preT[static_cast<int64_t>(w) * nitems + it] = static_cast<unsigned short>(run + incl - c);
        }
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0) {
      const int own = min(npts, sl1 * kSlice) - sl0 * kSlice;
      if (own > 0) evaluated += static_cast<unsigned long long>(own) * C;
    }
#ifdef GMMB_SP_PROF
    const int prof_c = C, prof_f = fused ? 1 : 0, prof_x = xslices ? 1 : 0;
#endif
    SP_PH(4);

    if (fused) {
      if (fits && lane < C) {
        double2* dst = reinterpret_cast<double2*>(pool + (base + lane) * kNSP);
#pragma unroll
        for (int q = 0; q < kNSP / 2; ++q)
          dst[q] = make_double2(facc[2 * q][lane], 2 * q + 1 < NS ? facc[2 * q + 1][lane] : 0.0);
      }
    } else
    // ---- pass 2: responsibilities + centred statistics
    for (int g = 0; g < C; g += 32) {
      const int ci = g + lane;
      Cand<D> cd;
      load_cand<D>(cd, ci < C ? cand_at(ci) : -1, mb, ct);
      double acc[NS];
#pragma unroll
      for (int q = 0; q < NS; ++q) acc[q] = 0.0;
      #pragma unroll 1
        for (int s = sl0; s < sl1; ++s) {
        const bool xs_s = (xslices >> s) & 1u;
        f2_t ACC[NS];
#pragma unroll
        for (int q = 0; q < NS; ++q) ACC[q] = 0ull;
#pragma unroll
        for (int pp = 0; pp < kSlice; pp += 2) {
          const int p = s * kSlice + pp;
          f2_t X[D];
          load_pair<D>(ws.xs, p, X);
          f2_t Q = dens_pair<D>(cd, X);
          if (xs_s) Q = add2(Q, *reinterpret_cast<const f2_t*>(&ws.sh[p]));
          const f2_t E = pk(ex2n(lo2(Q)), ex2n(hi2(Q)));
          const f2_t R = mul2(E, *reinterpret_cast<const f2_t*>(&ws.ssum[p]));
          f2_t DD[D], W[D];
#pragma unroll
          for (int i = 0; i < D; ++i) {
            DD[i] = add2(X[i], pk(cd.nmu[i], cd.nmu[i]));
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
        }
#pragma unroll
        for (int q = 0; q < NS; ++q) acc[q] += f32_to_f64(lo2(ACC[q]) + hi2(ACC[q]));
      }
      if (fits && ci < C) {
        double2* dst = reinterpret_cast<double2*>(pool + (base + ci) * kNSP);
#pragma unroll
        for (int q = 0; q < kNSP / 2; ++q)
          dst[q] = make_double2(acc[2 * q], 2 * q + 1 < NS ? acc[2 * q + 1] : 0.0);
      }
    }
    __syncwarp();
#ifdef GMMB_SP_PROF
    SP_PH(5);
    if (lane == 0) {
      g_sp_ph[it * 6 + 0] = static_cast<unsigned>(ph1 - ph0);
      g_sp_ph[it * 6 + 1] = static_cast<unsigned>(ph2 - ph1);
      g_sp_ph[it * 6 + 2] = static_cast<unsigned>(ph3 - ph2);
      g_sp_ph[it * 6 + 3] = static_cast<unsigned>(ph4 - ph3);
      g_sp_ph[it * 6 + 4] = static_cast<unsigned>(ph5 - ph4);
    }
    if (lane == 0) {
      unsigned long long prof_t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_t1));
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      g_sp_prof[it * 4 + 0] = prof_t0;
      g_sp_prof[it * 4 + 1] = prof_t1;
      g_sp_prof[it * 4 + 2] = (static_cast<unsigned long long>(smid) << 32) | static_cast<unsigned>(prof_c);
      g_sp_prof[it * 4 + 3] = prof_f | (prof_x << 1);
    }
#endif
  }
  if (lane == 0 && evaluated)
    atomicAdd(reinterpret_cast<unsigned long long*>(&ctl[4]), evaluated);
}

// ---- fixed-order reduce of the per-(tile, candidate) statistics -----------
// CTA (w, r): components 32 w + lane over tile range r (8 warps split it
// into contiguous sub-ranges, combined in warp order).
template <int D>
__global__ void __launch_bounds__(256)
    sparse_reduce_kernel(const unsigned* __restrict__ maskT, const unsigned short* __restrict__ preT,
                         const int* __restrict__ toff, const double* __restrict__ pool,
                         int64_t pool_cap, const double* __restrict__ ll_tile, int ntiles, int kw,
                         int R, int kpad, const EmState* __restrict__ st,
                         double* __restrict__ partials, double* __restrict__ ll_part) {
  constexpr int NS = nstats(D);
  constexpr int kNSP = pool_stride(D);
  __shared__ double red[8][NS][32];
  __shared__ double lred[8];
  if (st->done) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = blockIdx.x % kw, r = blockIdx.x / kw;
  const int t0 = static_cast<int>(static_cast<int64_t>(r) * ntiles / R);
  const int t1 = static_cast<int>(static_cast<int64_t>(r + 1) * ntiles / R);
  const int a0 = t0 + static_cast<int>(static_cast<int64_t>(warp) * (t1 - t0) / 8);
  const int a1 = t0 + static_cast<int>(static_cast<int64_t>(warp + 1) * (t1 - t0) / 8);
  double acc[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) acc[q] = 0.0;
  const unsigned below = lanemask_lt();
  const int* toffS = toff + ntiles;  // split units' sub-unit bases (ntiles = units)
  for (int tb = a0; tb < a1; tb += 32) {
    const int tt = tb + lane;
    const unsigned wv = tt < a1 ? maskT[static_cast<int64_t>(w) * ntiles + tt] : 0u;
    const int pv = tt < a1 ? preT[static_cast<int64_t>(w) * ntiles + tt] : 0;
    const int ov = tt < a1 ? toff[tt] : 0;
    unsigned any = __ballot_sync(0xffffffffu, wv != 0u);
    // split units of this chunk first (rare), each sub-unit's entries in
    // sub-unit order; then the plain units below
    unsigned spl = __ballot_sync(0xffffffffu, wv != 0u && ov < -1);
    any &= ~spl;
    while (spl) {
      const int j = __ffs(spl) - 1;
      spl &= spl - 1;
      const unsigned word = __shfl_sync(0xffffffffu, wv, j);
      const int pre = __shfl_sync(0xffffffffu, pv, j);
      const int ns = -__shfl_sync(0xffffffffu, ov, j);
      const bool mine = (word >> lane) & 1u;
      const int idx = pre + __popc(word & below);
      for (int sb = 0; sb < ns; ++sb) {
        const int b = toffS[static_cast<int64_t>(tb + j) * kMaxSplit + sb];
        const double2* src = reinterpret_cast<const double2*>(pool + (static_cast<int64_t>(b) + idx) * kNSP);
        const bool ld = mine && b >= 0;
#pragma unroll
        for (int q = 0; q < kNSP / 2; ++q) {
          const double2 x = ld ? __ldcg(src + q) : make_double2(0.0, 0.0);
          acc[2 * q] += x.x;
          if (2 * q + 1 < NS) acc[2 * q + 1] += x.y;
        }
      }
    }
    while (any) {
      // kRedStep units per step: their loads in flight before the (ordered) adds
      double v[kRedStep][NS];
#pragma unroll
      for (int u = 0; u < kRedStep; ++u) {
        const int j = any ? __ffs(any) - 1 : 0;
        const bool on = any != 0u;
        any &= any - 1;
        const unsigned word = on ? __shfl_sync(0xffffffffu, wv, j) : 0u;
        const int pre = __shfl_sync(0xffffffffu, pv, j);
        const int off = __shfl_sync(0xffffffffu, ov, j);
        const bool mine = (word >> lane) & 1u;
        const int64_t e = static_cast<int64_t>(off) + pre + __popc(word & below);
        const double2* src = reinterpret_cast<const double2*>(pool + e * kNSP);
#pragma unroll
        for (int q = 0; q < kNSP / 2; ++q) {
          const double2 x = mine ? __ldcg(src + q) : make_double2(0.0, 0.0);
          v[u][2 * q] = x.x;
          if (2 * q + 1 < NS) v[u][2 * q + 1] = x.y;
        }
      }
#pragma unroll
      for (int u = 0; u < kRedStep; ++u)
#pragma unroll
        for (int q = 0; q < NS; ++q) acc[q] += v[u][q];
    }
  }
#pragma unroll
  for (int q = 0; q < NS; ++q) red[warp][q][lane] = acc[q];
  double l = 0.0;
  if (w == 0) {
    const double* llS = ll_tile + ntiles;
    for (int tt = a0 + lane; tt < a1; tt += 32) {
      const int o = toff[tt];
      if (o < -1) {
        for (int sb = 0; sb < -o; ++sb) l += llS[static_cast<int64_t>(tt) * kMaxSplit + sb];
      } else {
        l += ll_tile[tt];
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
    if (lane == 0) lred[warp] = l;
  }
  __syncthreads();
  if (warp == 0) {
    const int k = 32 * w + lane;
    if (k < kpad) {
      double* out = partials + (static_cast<int64_t>(r) * kpad + k) * NS;
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        double s = 0.0;
#pragma unroll
        for (int v = 0; v < 8; ++v) s += red[v][q][lane];
        out[q] = s;
      }
    }
    if (w == 0 && lane == 0) {
      double s = 0.0;
#pragma unroll
      for (int v = 0; v < 8; ++v) s += lred[v];
      ll_part[r] = s * kLn2;
    }
  }
}


size_t main_smem_bytes(int kcap) { return warp_smem_bytes(kcap) * kSpWarps; }

int reduce_ranges(int kcap, int nunits, int sm_count) {
  // enough CTAs to fill the device, and at most GMMB_RED_UNITS units per CTA
  // (the scan over units is a chain of dependent loads; 128 units, two per
  // step, measured best: cfg2 E 132 -> 123 us, K = 2048 439 -> 404 us)
  const int kw = (kcap + 31) / 32;
  int R = (2 * sm_count + kw - 1) / kw;
  const int r2 = (nunits + GMMB_RED_UNITS - 1) / GMMB_RED_UNITS;  // units per CTA
  if (R < r2) R = r2;
  const int maxr = (nunits + 63) / 64;  // at least 8 units per warp
  if (R > maxr) R = maxr;
  return R < 1 ? 1 : R;
}

}  // namespace

bool sparse_supported(int k0, int ntiles) {
  const int nblk = (ntiles + kBlkTiles - 1) / kBlkTiles;
  return k0 <= 65535 && static_cast<int64_t>(nblk) * k0 <= (int64_t{1} << 26) &&
         static_cast<int64_t>(ntiles) * kItemsPerTile < (int64_t{1} << 24) &&
         main_smem_bytes(k0) <= 200 * 1024;
}

int sparse_blocks(int ntiles) { return (ntiles + kBlkTiles - 1) / kBlkTiles; }

int sparse_items(int ntiles) { return ntiles * kItemsPerTile; }

// points per work unit: one item (32 points) while the cloud has few tiles per
// warp (balance, tight boxes), whole tiles when there are plenty (4x fewer
// per-unit statistics records to write and reduce)
int sparse_unit_items(int ntiles, int sm_count, int k0) {
  static const int forced = [] {  // GMMB_SPARSE_U=1|2|4 (experiments)
    const char* e = getenv("GMMB_SPARSE_U");
    const int u = e ? atoi(e) : 0;
    return (u == 1 || u == 2 || u == 4) ? u : 0;
  }();
  if (forced) return forced;
  const int warps = sm_count * kSpWarps * kSpMinBlocks;
  const int nitems = sparse_items(ntiles);
  // Measured EM ms per fit, U = 1 / 2 / 4 (scripts/ab_fits.py, fits to tol
  // 1e-3; the heavy-unit split keeps larger units balanced):
  //   frame (9,600 items) K = 64: 1.27 / 1.14 / 1.16, K = 256: 1.72 / 1.48 / 1.81,
  //   K = 512: 1.90 / 1.61 / 1.79, K = 1024: 2.40 / 2.00 / 1.93,
  //   K = 2048: 4.73 / 4.08 / 3.94, K = 4096: 9.20 / 7.73 / 7.60;
  //   cfg4 (125k items, K = 2048): 10.65 / 6.74 / 4.94
  if (nitems >= 32 * warps) return 4;
  if (nitems >= 2 * warps) return k0 > 512 ? 4 : 2;
  return 1;
}

int sparse_ranges(int k0, int ntiles, int sm_count) {
  return reduce_ranges(k0, sparse_items(ntiles) / sparse_unit_items(ntiles, sm_count, k0), sm_count);
}

cudaError_t launch_sparse_layout(const PointsDev& pts, const SparseScratch& sp, cudaStream_t s) {
  const int nblk = sparse_blocks(pts.ntiles);
  block_box_kernel<<<nblk, kTile, 0, s>>>(pts.xt, pts.tc, pts.n, pts.ntiles, sp.bc, sp.bh);
  return cudaGetLastError();
}

cudaError_t launch_estep_sparse(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                                int k0, double* partials, double* ll_part, int exact_mode,
                                int sm_count, cudaStream_t s, int* ncl_out,
                                const SparseScratch& sp) {
  const int ntiles = pts.ntiles;
  const int U = sparse_unit_items(ntiles, sm_count, k0);
  const int nitems = sparse_items(ntiles) / U;  // work units
  const int R = reduce_ranges(k0, nitems, sm_count);
  *ncl_out = R;
  if (!partials) return cudaSuccess;
  const int nblk = sparse_blocks(ntiles);
  const int kw = (k0 + 31) / 32;
  const size_t smem = main_smem_bytes(k0);
  static int occ_dev[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& occ = occ_dev[dev & 63][pts.d == 4 ? 1 : 0];
  auto kern = pts.d == 4 ? estep_sparse_kernel<4> : estep_sparse_kernel<3>;
  if (occ == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(200 * 1024));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kSpWarps * 32, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
    if (getenv("GMMB_DEBUG"))
      fprintf(stderr, "gmmb: estep_sparse D=%d K=%d smem=%zu -> %d CTAs/SM\n", pts.d, k0, smem, occ);
  }
  int grid = sm_count * occ;
  const int need = (nitems + kSpWarps - 1) / kSpWarps;
  if (grid > need) grid = need;
  static const float qcut = [] {
    const char* e = getenv("GMMB_SPARSE_QCUT");
    return e ? static_cast<float>(atof(e)) : kQCut;
  }();
  // GMMB_SP_EVENTS=1 (diagnostic; plain launches only, i.e. timing mode):
  // events around each of the three kernels, read by gmmb_debug_sp_events
  static const bool evs = getenv("GMMB_SP_EVENTS") != nullptr;
  cudaEvent_t* ev = nullptr;
  if (evs && g_sp_nev < kSpEvCalls) {
    ev = g_sp_ev[g_sp_nev++];
    for (int i = 0; i < 4; ++i)
      if (!ev[i]) cudaEventCreate(&ev[i]);
  }
  if (ev) cudaEventRecord(ev[0], s);
  if (pts.d == 4)
    block_cand_kernel<4><<<nblk, kBcThreads, 0, s>>>(sp.bc, sp.bh, bufs[0], bufs[1], st, k0, sp.blist,
                                              sp.brec, sp.bcnt, sp.ctl, qcut);
  else
    block_cand_kernel<3><<<nblk, kBcThreads, 0, s>>>(sp.bc, sp.bh, bufs[0], bufs[1], st, k0, sp.blist,
                                              sp.brec, sp.bcnt, sp.ctl, qcut);
  const int ucap = sp.item_cap * U;
  const int warps_all = sm_count * occ * kSpWarps;
  // GMMB_SPARSE_NOSPLIT=1 / GMMB_SPARSE_EXACT=1: validation knobs (no
  // heavy-unit splits / the max-shift path on every slice)
  static const bool env_nosplit = getenv("GMMB_SPARSE_NOSPLIT") != nullptr;
  static const bool env_exact = getenv("GMMB_SPARSE_EXACT") != nullptr;
  if (env_exact) exact_mode = 1;
  // (measured: 96 best up to K = 1024, 160 above: K = 2048 3.96 -> 3.80 ms,
  // K = 4096 7.47 -> 6.43 ms of EM per fit; K = 1024 1.96 vs 2.17)
  const int split_base = kSplitC > 0 ? kSplitC : (k0 > 1024 ? 160 : 96);
  const int split_c = (sp.no_split || env_nosplit) ? (1 << 30)
                                                    : split_base * std::max(1, nitems / (4 * warps_all));
  if (ev) cudaEventRecord(ev[1], s);
  kern<<<grid, kSpWarps * 32, smem, s>>>(pts.xt, pts.tc, pts.n, nitems, bufs[0], bufs[1], st, k0,
                                         sp.blist, sp.brec, sp.bcnt, sp.bc, ucap, sp.ctl, sp.pool,
                                         sp.pool_cap, sp.toff,
                                         sp.maskT, sp.preT, sp.ll_tile, sp.heavy, sp.done,
                                         exact_mode, qcut, U, split_c);
  if (ev) cudaEventRecord(ev[2], s);
  if (pts.d == 4)
    sparse_reduce_kernel<4><<<kw * R, 256, 0, s>>>(sp.maskT, sp.preT, sp.toff, sp.pool, sp.pool_cap,
                                                   sp.ll_tile, nitems, kw, R, k0, st, partials,
                                                   ll_part);
  else
    sparse_reduce_kernel<3><<<kw * R, 256, 0, s>>>(sp.maskT, sp.preT, sp.toff, sp.pool, sp.pool_cap,
                                                   sp.ll_tile, nitems, kw, R, k0, st, partials,
                                                   ll_part);
  if (ev) cudaEventRecord(ev[3], s);
  return cudaGetLastError();
}

}  // namespace gmmb

// per recorded E step: ms of block_cand, the main kernel, the reduce;
// returns the number of steps and resets the recorder
extern "C" int gmmb_debug_sp_events(float* out, int max_steps) {
  using namespace gmmb;
  const int n = g_sp_nev < max_steps ? g_sp_nev : max_steps;
  cudaDeviceSynchronize();
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 3; ++j) cudaEventElapsedTime(&out[3 * i + j], g_sp_ev[i][j], g_sp_ev[i][j + 1]);
  g_sp_nev = 0;
  return n;
}

#ifdef GMMB_SP_PROF
extern "C" int gmmb_debug_sp_prof(unsigned long long* out, int count) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, gmmb::g_sp_prof, sizeof(unsigned long long) * count));
}
extern "C" int gmmb_debug_sp_ph(unsigned* out, int count) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, gmmb::g_sp_ph, sizeof(unsigned) * count));
}
#endif
