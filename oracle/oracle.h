/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * C ABI of the FP64 CPU restatement of the gmmscape hot path
 * (k-means++ kinit -> hard M-step -> full-covariance EM). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library, and only as the checker / CPU baseline.
 * The product (paper_2307_00071_b200/, libgmmb.so) never links it.
 *
 * Parity status: the reference (/root/reference/proj) cannot be compiled
 * here (Eigen3 and libpng are absent, no network), so there is no
 * oracle/_ref. This restatement is pinned against every known-answer test
 * SPEC.md states for the path (tests/test_oracle_kats.py); the reference
 * ships no golden vectors, so bit-level agreement with an Eigen build is
 * "parity unpinned" beyond those KATs.
 *
 * Layouts follow the reference:
 *   points  : N x 4 column-major doubles (Eigen MatX4, common.hpp:11),
 *             i.e. pts[j*N + i] is coordinate j of point i.
 *   means   : M x 4 row-major (one row per component).
 *   covs    : M x 10 packed lower triangle, row-major order
 *             (0,0),(1,0),(1,1),(2,0),... (packed10.hpp:11-14).
 *   4x4     : column-major 16 doubles (Eigen Matrix4d default).
 *   log_gamma: N x M column-major (Eigen MatX).
 * Return codes: 0 ok, 2 invalid argument, 3 numerical error
 * (gmmscape_cli.cpp:508-528 exit-code classes).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
void orc_set_num_threads(int n);      /* common.cpp:13 */
int orc_num_threads(void);            /* common.cpp:15-21 */

/* rng.hpp:16-70 */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_bits(uint64_t seed, uint64_t stream, uint64_t counter);
double orc_uniform(uint64_t seed, uint64_t stream, uint64_t counter);
double orc_uniform_pos(uint64_t seed, uint64_t stream, uint64_t counter);
void orc_normal_pair(uint64_t seed, uint64_t stream, uint64_t counter,
                     double* z0, double* z1);
uint64_t orc_hash_coords(const double* x, int n);

/* kernels.cpp:10-50 */
int orc_cholesky4(const double* a16, double* lower16);
void orc_lower_inverse4(const double* lower16, double* inv16);
/* kernels.cpp:52-77 ; returns 3 and sets *bad to the first failing block */
int orc_batched_cholesky(const double* blocks, int count, double* lower,
                         int* bad);
/* kernels.cpp:104-135 */
void orc_logsumexp_rows(const double* mat, int64_t n, int64_t m, double* out);
/* kernels.hpp:82-181 + kernels.cpp:321-331 (linear-domain resp) */
int orc_weighted_moments(const double* pts, int64_t n, const double* resp,
                         int64_t m, double* counts, double* means,
                         double* scatters16, int* degenerate_flags);
/* gmm.cpp:33-48 */
int orc_cholesky_cache(const double* covs, int m, double* lower16,
                       double* precision16, double* log_det_terms);

/* point_cloud.hpp:15-24 */
int orc_validate_cloud(const double* pts, int64_t n);

/* sogmm.cpp:197-337. centers[k], labels[n] (the argmax-one-hot of the
 * returned Responsibilities). */
int orc_kinit(const double* pts, int64_t n, int k, uint64_t seed,
              int64_t* centers, int32_t* labels);
/* sogmm.cpp:341-383; log_gamma is N x M col-major caller buffer. */
int orc_e_step(const double* pts, int64_t n, int m, const double* weights,
               const double* means, const double* covs, double* log_gamma,
               double* ll);
/* sogmm.cpp:399-455. Outputs sized for m components; *m_out <= m. */
int orc_m_step(const double* pts, int64_t n, const double* log_gamma, int m,
               double cov_reg, double* w_out, double* mu_out, double* cov_out,
               int* m_out, int* removed);
/* Hard-label M-step: identical to orc_m_step on the one-hot (0/-inf)
 * log_gamma kinit returns (sogmm.cpp:333-336, :481), without building it. */
int orc_m_step_labels(const double* pts, int64_t n, const int32_t* labels,
                      int m, double cov_reg, double* w_out, double* mu_out,
                      double* cov_out, int* m_out, int* removed);

typedef struct {
  int max_iters;      /* sogmm.hpp:37 */
  double ll_rel_tol;  /* 0 = run max_iters (extension; reference needs > 0) */
  double cov_reg;
  uint64_t seed;
  /* subtracted from every ll before the convergence test and the outputs:
   * the 3D embedding constant N(-1/2 ln 2pi - 1/2 ln cov_reg), so a 3D cloud
   * fitted through [x,y,z,0] reports (and converges on) the 3D ll. */
  double ll_offset;
} orc_em_params;

typedef struct {
  int em_iterations;          /* E steps executed (sogmm.cpp:492) */
  double final_log_likelihood;
  int removed_components;
  int k_out;
  int k_init;                 /* k = min(K, N) (sogmm.cpp:477) */
} orc_fit_stats;

/* EM loop sogmm.cpp:484-509 from a given model (m0 components).
 * ll_trace[max_iters] receives the ll of every E step. */
int orc_fit_from(const double* pts, int64_t n, int m0, const double* w0,
                 const double* mu0, const double* cov0,
                 const orc_em_params* em, double* w_out, double* mu_out,
                 double* cov_out, double* ll_trace, orc_fit_stats* stats);
/* sogmm.cpp:477-509 with K given: kinit -> m_step -> EM loop.
 * centers/labels may be NULL. */
int orc_fit_k(const double* pts, int64_t n, int K, const orc_em_params* em,
              double* w_out, double* mu_out, double* cov_out,
              double* ll_trace, orc_fit_stats* stats, int64_t* centers,
              int32_t* labels);

/* Streaming EM: same arithmetic as orc_fit_from but recomputes log_gamma
 * per 4096-point block instead of materialising N x M (for configs whose
 * N x M FP64 matrix exceeds host RAM). Sums differ from orc_fit_from only
 * by association order. */
int orc_fit_from_streaming(const double* pts, int64_t n, int m0,
                           const double* w0, const double* mu0,
                           const double* cov0, const orc_em_params* em,
                           double* w_out, double* mu_out, double* cov_out,
                           double* ll_trace, orc_fit_stats* stats);

/* inference.cpp:141-172 score (average ll), :17-54 joint_dist_sample
 * (n x 4 column-major out), :56-139 color_conditional (locs n x 3
 * column-major). */
int orc_score(const double* pts, int64_t n, int m, const double* w, const double* mu,
              const double* cov, double* out);
int orc_sample(int m, const double* w, const double* mu, const double* cov, int64_t n,
               uint64_t seed, double* out);
int orc_color_conditional(int m, const double* w, const double* mu, const double* cov,
                          const double* locs, int64_t n, int clamp, double* expected,
                          double* variance);

/* gbms_estimate_components (sogmm.cpp:22-195) with the reference's kd-tree
 * (kdtree.hpp); points N x 4 column-major; modes (optional) components x 4
 * row-major, up to modes_capacity rows. */
int orc_gbms(const double* pts, int64_t n, double bandwidth, int max_iters, double tol,
             double merge_radius, int* components, int* iterations, int* seeds0,
             double* modes, int modes_capacity);

/* benchmark inputs (reference synthetic.cpp / ingest.cpp restated) */
int orc_synthetic_frame_cloud(int width, int height, double depth_scale, double* pts,
                              int64_t* n_out);
int orc_structured_scene(int64_t n, uint64_t seed, double noise_sigma, double* pts);
int orc_jitter_cloud(double* pts, int64_t n, double sigma, uint64_t seed);

#ifdef __cplusplus
}
#endif
