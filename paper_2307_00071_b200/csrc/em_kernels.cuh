// em_kernels.cuh — EM iteration kernels (declarations + launch helpers).
#pragma once
#include "common.cuh"

namespace gmmb {

// Device model buffer (one of two, ping-ponged across M steps).
struct ModelBuf {
  double* w;        // [kcap]
  double* mu;       // [kcap][4]
  double* cov;      // [kcap][10] packed (D=3 uses the first 6)
  CompConst* cst;   // [kcap] FP32 E-step constants
};

// Per-component M-step record (output of finalize, input of commit).
struct RecBuf {
  double* count;    // [kcap]
  double* mean;     // [kcap][4]
  double* cov;      // [kcap][10]  regularised covariance
  double* logdet;   // [kcap]      sum ln diag P
  float* pc;        // [kcap][16]  scaled precision factor
  int* flags;       // [kcap]      bit0 keep, bit1 SPD ok
  int* map;         // [kcap]      compacted index (commit, K > kMaxK)
};

struct PointsDev {
  int64_t n;
  int d;
  const double* x64;   // [4][n] column-major FP64 (original order)
  const float4* xt;    // [n] sorted, tile-recentred FP32
  const double* tc;    // [ntiles][4] tile centres
  int ntiles;
};

// Scratch of the chunked two-pass E step (K > 512, estep_chunked.cu):
// part[nch][npad] per-chunk per-point sums, lse[npad] per-point log2
// normalisers as (shift, remainder) pairs (shift = 0 except for points that
// needed the exact max-shifted log-sum-exp), xlist[npad] + *xcount those
// points (npad = ntiles * kTile, nch = ceil(K / 512)).
struct ChunkScratch {
  float* part;
  float2* lse;
  int* xlist;
  int* xcount;
};
size_t chunk_scratch_floats(int k0, int64_t n);  // part + lse
cudaError_t launch_estep_chunked(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                                 int k0, double* partials, double* ll_part, int exact_mode,
                                 int sm_count, cudaStream_t s, int* ncl_out,
                                 const ChunkScratch* scr);

// Exact-zero-pruned E step (estep_sparse.cu). Per-layout: bc/bh block boxes;
// per iteration: block candidate lists, a pool of per-(tile, candidate) FP64
// statistics (SoA [nstats][pool_cap]), per-tile pool offsets, candidate
// bitmasks + per-word prefix counts (word-major [K/32][ntiles]), per-tile ll.
// ctl[0] tile queue, ctl[1] pool cursor, ctl[2] pool overflow (the fit is
// re-run with a larger pool), ctl[4..5] units evaluated (u64).
struct SparseScratch {
  double* bc;            // [nblk][4]
  float4* bh;            // [nblk]
  int* blist;            // [nblk][K]
  float4* brec;          // [nblk][K][4] candidate bound records (factor, base2, mean - block centre)
  int item_cap;          // pool entries reserved per 32-point item (overflow region after)
  int* bcnt;             // [nblk]
  int* ctl;              // [16]
  int* heavy;            // [2][kSparseMaxSplit * nunits] heavy-unit task lists (iteration parity)
  unsigned* done;        // [2][nunits] epoch stamps of units queued as heavy (iteration parity)
  double* pool;          // [pool_cap][stride] per-(unit, candidate) statistics
  int64_t pool_cap;
  int* toff;             // [nunits] pool base (-S: split) + [nunits][kSparseMaxSplit] sub-unit bases
  unsigned* maskT;       // [K/32][nunits]
  unsigned short* preT;  // [K/32][nunits]
  double* ll_tile;       // [nunits] + [nunits][kSparseMaxSplit] (split units)
  int no_split;          // 1: no heavy-unit splits (the retry after a split unit hit the exact path)
};
constexpr int kSparseMaxSplit = 8;  // sub-units per heavy unit (estep_sparse.cu)
bool sparse_supported(int k0, int ntiles);
int sparse_blocks(int ntiles);
int sparse_items(int ntiles);  // work items (32-point quarter tiles)
int sparse_ranges(int k0, int ntiles, int sm_count);
cudaError_t launch_sparse_layout(const PointsDev& pts, const SparseScratch& sp, cudaStream_t s);
cudaError_t launch_estep_sparse(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                                int k0, double* partials, double* ll_part, int exact_mode,
                                int sm_count, cudaStream_t s, int* ncl_out,
                                const SparseScratch& sp);

// Pass B of the chunked E step on the warp-specialised kernel (normalisers
// known): grid nch x (sm_count / nch); *ncl_out = point ranges.
cudaError_t launch_estep_ws_pre(const PointsDev& pts, const ModelBuf* bufs, const EmState* st,
                                int kpad, int nch, const float2* lse, double* partials,
                                double* ll_part, int sm_count, cudaStream_t s, int* ncl_out);

// Fused E-step + sufficient statistics (one EM iteration's data pass).
// Writes per-cluster FP64 partial statistics [ncl][kpad][nstats(D)] and
// per-cluster log-likelihood partials (natural log) [ncl]. exact_mode = 1
// forces the max-shifted normalisation on every sub-tile (validation).
cudaError_t launch_estep_stats(const PointsDev& pts, const ModelBuf* bufs,
                               const EmState* st, int k0, double* partials,
                               double* ll_part, int exact_mode,
                               int sm_count, cudaStream_t s, int* ncl_out,
                               const ChunkScratch* chunk = nullptr,
                               const SparseScratch* sparse = nullptr);

// (partials == nullptr: only report the cluster count *ncl_out.) K > 512
// runs the chunked two-pass kernels (chunk scratch required) unless
// GMMB_CHUNKED=0 at build time (the cluster kernels, K <= 4096).

// FP64 L, P, logdet of buffer st->cur (cholesky_cache API), 33 doubles/comp.
cudaError_t launch_factor_dump(int d, const ModelBuf* bufs, const EmState* st,
                               int m, double* out, cudaStream_t s);

// Deterministic second-stage reduce: red[k][nstats] (+ red_ll[0]).
cudaError_t launch_em_reduce(int d, const double* partials,
                             const double* ll_part, int ncl, int k0,
                             const EmState* st, double* red, double* red_ll,
                             cudaStream_t s);

// Per-component finalize: centred stats about mu_old -> record.
cudaError_t launch_em_finalize(int d, const double* red, const ModelBuf* bufs,
                               const EmState* st, int k0, RecBuf rec,
                               cudaStream_t s);

// Single-CTA commit: convergence bookkeeping, compaction, new model.
// mode 0: EM iteration (uses red_ll, ll_trace); mode 1: plain M step
// (initial hard M step / m_step API: always commits, no EM bookkeeping).
// cond != nullptr: the launch is the tail of the EM while-graph body and
// sets the loop condition (1 = run another iteration) from st->done.
cudaError_t launch_commit(int d, int mode, const RecBuf rec, int k_in,
                          const double* red_ll, ModelBuf* bufs, EmState* st,
                          double* ll_trace, cudaStream_t s,
                          const cudaGraphConditionalHandle* cond = nullptr,
                          const double* ll_part = nullptr, int ncl = 0);
// (mode 0: the log-likelihood comes from ll_part[ncl] if given, else red_ll[0])

// Single-device fused reduce of the per-CTA partials + finalize (replaces
// launch_em_reduce + launch_em_finalize when there is no cross-rank sum).
cudaError_t launch_em_reduce_finalize(int d, const double* partials, int ncl, int k0,
                                     const ModelBuf* bufs, const EmState* st, RecBuf rec,
                                     cudaStream_t s);

// Model (FP64) -> E-step constants for buffer st->cur; sets error on
// a non-SPD covariance (first failing index, gmm.cpp:33-48 semantics).
cudaError_t launch_prep(int d, ModelBuf* bufs, EmState* st, int k,
                        cudaStream_t s);

// FP64 two-pass weighted moments (kernels.hpp:82-181) with weights either
// from hard labels (kinit one-hot) or from a dense N x M log_gamma.
// Produces records (count/mean/cov/...) for launch_commit(mode=1).
struct MomentsScratch {
  double* part;      // [nchunks][m][10]
  double* sums;      // [m][5]   reduced pass-1 sums
  double* means;     // [m][4]
  double* counts;    // [m]
};
cudaError_t launch_moments(int d, const double* x64, int64_t n,
                           const int32_t* labels, const double* log_gamma,
                           int m, double cov_reg, MomentsScratch scr,
                           RecBuf rec, int sm_count, cudaStream_t s,
                           void (*allreduce)(double*, int64_t, void*),
                           void* ar_ctx);



}  // namespace gmmb
