/*
 * gmmb.h — C ABI of the B200-native Gaussian-mixture learner
 * (libgmmb.so, package paper_2307_00071_b200).
 *
 * Drop-in boundary for the reference's fit path (gmmscape, C++ library,
 * /root/reference/proj). The reference exposes no FFI; its public C++ API is
 * include/gmmscape/sogmm.hpp + gmm.hpp. Each entry point below names the
 * reference symbol it replaces. include/gmmb.hpp wraps this ABI back into the
 * reference's C++ shape (exceptions, value types) and INTEGRATION.md shows
 * the bindings.
 *
 * Conventions (all follow the reference):
 *  - points: N x D column-major doubles, D in {3, 4}: pts[j*N + i] is
 *    coordinate j of point i (Eigen MatX4, common.hpp:11). D = 4 is
 *    xyz + intensity in [0, 1] (point_cloud.hpp:7-24); D = 3 is xyz.
 *  - model: weights[M]; means[M*D] row-major; covs[M*D(D+1)/2] packed lower
 *    triangle in row-major order (0,0),(1,0),(1,1),(2,0),... (packed10.hpp).
 *  - log_gamma: N x M column-major (sogmm.hpp Responsibilities).
 *  - return codes: 0 ok, 1 I/O / device failure, 2 invalid argument
 *    (std::invalid_argument), 3 numerical error (NumericalError) — the
 *    CLI's exit-code classes, gmmscape_cli.cpp:508-528. The message is in
 *    gmmb_last_error() (thread-local).
 *  - all calls are blocking; the library copies host buffers in and out and
 *    keeps no pointer after return. A context owns one CUDA device/stream
 *    and reusable device buffers; calls on one context must not overlap.
 */
#ifndef GMMB_H_
#define GMMB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gmmb_ctx gmmb_ctx;

/* EmParams (sogmm.hpp:36-41). ll_rel_tol = 0 runs exactly max_iters E steps
 * (extension: the reference requires > 0, sogmm.cpp:468). */
typedef struct {
  int max_iters;      /* default 100 */
  double ll_rel_tol;  /* default 1e-5 */
  double cov_reg;     /* default 1e-6 */
  uint64_t seed;      /* default 0 (kinit) */
} gmmb_em_params;

/* FitResult (sogmm.hpp:65-71) minus gbms_components, plus K bookkeeping and
 * device-side stage timings (CUDA events, milliseconds). */
typedef struct {
  int em_iterations;           /* E steps executed */
  double final_log_likelihood; /* natural log, D-dimensional density */
  int removed_components;      /* degenerate components removed */
  int k_out;                   /* components in the returned model */
  int k_init;                  /* min(K, N) (sogmm.cpp:477) */
  int converged;               /* 1 if the tolerance test ended the loop */
  double ms_layout;            /* validate + Morton sort + recentring */
  double ms_kinit;             /* keys + k-means++ + fix-up */
  double ms_mstep0;            /* initial hard-assignment M step */
  double ms_em;                /* EM loop */
  double units;                /* sum over E steps of N * K_t */
  double ms_total;             /* layout start -> EM end (device) */
  double ms_estep;             /* fused E-step kernel, executed iterations */
  long long launches;          /* kernels this library enqueued (CUB excluded) */
  double units_evaluated;      /* (point, component) pairs the E step evaluated:
                                  the pruned E step skips pairs whose FP32
                                  density is provably exactly 0 (= units for
                                  the dense kernels) */
} gmmb_fit_stats;

const char* gmmb_last_error(void);
void gmmb_em_params_default(gmmb_em_params* p);

/* Context on a CUDA device (one process may hold several). */
int gmmb_ctx_create(int device, gmmb_ctx** out);
/* Sharded context: this rank holds points [offset, offset+n) of a cloud
 * split over `world` ranks; sufficient statistics and k-means++ candidates
 * are combined with NCCL (libnccl.so.2, loaded at run time). nccl_id is the
 * 128-byte ncclUniqueId from gmmb_nccl_unique_id on rank 0, broadcast by the
 * caller (e.g. torch.distributed). */
int gmmb_nccl_unique_id(void* out128);
int gmmb_ctx_create_sharded(int device, int rank, int world,
                            const void* nccl_id128, gmmb_ctx** out);
/* Virtual shards (no reference counterpart; the validation mode of the
 * sharded path): `world` in-process ranks on ONE device. The
 * caller creates one context per rank with gmmb_ctx_create_virtual and
 * drives each from its own host thread with the same calls as NCCL ranks
 * (e.g. gmmb_fit_k on contiguous shards); the collectives are fixed-order
 * device reductions over the ranks' buffers instead of NCCL. A failure on
 * one rank, or destroying one rank's context, aborts the group (its peers'
 * pending collectives return 1). The group lives until it is released and
 * every context of it is destroyed. */
typedef struct gmmb_vgroup gmmb_vgroup;
int gmmb_vgroup_create(int device, int world, gmmb_vgroup** out);
void gmmb_vgroup_release(gmmb_vgroup* g);
int gmmb_ctx_create_virtual(gmmb_vgroup* g, int rank, gmmb_ctx** out);
void gmmb_ctx_destroy(gmmb_ctx* ctx);
/* EM loop execution mode (no reference counterpart; measurement aid).
 * 0 (default): the EM loop of a fit is one CUDA graph with a conditional
 * WHILE node, the loop condition set on the device — no host round trip.
 * 1: iterations are enqueued in chunks with CUDA events around every fused
 * E kernel (gmmb_fit_stats.ms_estep), for kernel timing. Same results. */
int gmmb_ctx_set_timing(gmmb_ctx* ctx, int per_kernel_events);
/* E-step kernels: 0 (default) the exact-zero-pruned E step whenever it
 * applies (K <= 8192), 1 the dense kernels (every (point, component) pair).
 * Both give the same results up to FP32 summation order. The environment
 * variable GMMB_ESTEP=dense sets 1 at context creation. */
int gmmb_ctx_set_estep_mode(gmmb_ctx* ctx, int mode);

int gmmb_device_info(gmmb_ctx* ctx, int* sm_count, int* cc_major,
                     int* cc_minor);

/* ---- full fits ---------------------------------------------------------
 * fit(cloud, bandwidth, em) (sogmm.hpp:74-75, sogmm.cpp:465-510) with the
 * component count given instead of estimated by GBMS:
 * k = min(K, N) -> kinit -> m_step -> EM loop (sogmm.cpp:477-509).
 * Outputs are sized for min(K, N) components; stats->k_out says how many
 * are valid. ll_trace[max_iters] (nullable) receives every E step's ll.
 * labels[N] / centers[k] (nullable) receive the kinit assignment.
 * offset: global index of this rank's first point (0 unless sharded). */
int gmmb_fit_k(gmmb_ctx* ctx, const double* pts, int64_t n, int d, int K,
               const gmmb_em_params* em, double* w_out, double* mu_out,
               double* cov_out, double* ll_trace, gmmb_fit_stats* stats,
               int32_t* labels, int64_t* centers);

/* A batch of independent frames (BASELINE cfg3), the reference's serial
 * loop of fit calls (gmmscape_cli.cpp:208-227) on one device: frame f is
 * fitted exactly as gmmb_fit_k(pts[f], n[f], d, K, em with seed seeds[f])
 * (seeds nullable: em->seed for all), while frame f+1's points are copied to
 * the device on a second stream (pinned host frames overlap fully; frames
 * already in device memory are accepted too). Outputs
 * per frame at f*K (w), f*K*d (mu), f*K*d(d+1)/2 (cov); stats[f]. Sharded
 * contexts: shard the frames over the ranks instead (returns 2). */
int gmmb_fit_k_batch(gmmb_ctx* ctx, int frames, const double* const* pts, const int64_t* n,
                     int d, int K, const gmmb_em_params* em, const uint64_t* seeds,
                     double* w_out, double* mu_out, double* cov_out, gmmb_fit_stats* stats);

/* EM loop of fit (sogmm.cpp:484-509) from a caller-supplied initial model
 * (the "fixed init" configuration). */
int gmmb_fit_from(gmmb_ctx* ctx, const double* pts, int64_t n, int d, int m,
                  const double* w0, const double* mu0, const double* cov0,
                  const gmmb_em_params* em, double* w_out, double* mu_out,
                  double* cov_out, double* ll_trace, gmmb_fit_stats* stats);

/* Device-resident variants (points uploaded once, fits re-run on them):
 * gmmb_upload validates and lays out the cloud (PointCloud4D::validate,
 * point_cloud.hpp:15-24). */
int gmmb_upload(gmmb_ctx* ctx, const double* pts, int64_t n, int d,
                int64_t offset, int64_t n_global);
int gmmb_fit_k_resident(gmmb_ctx* ctx, int K, const gmmb_em_params* em,
                        double* w_out, double* mu_out, double* cov_out,
                        double* ll_trace, gmmb_fit_stats* stats,
                        int32_t* labels, int64_t* centers);
int gmmb_fit_from_resident(gmmb_ctx* ctx, int m, const double* w0,
                           const double* mu0, const double* cov0,
                           const gmmb_em_params* em, double* w_out,
                           double* mu_out, double* cov_out, double* ll_trace,
                           gmmb_fit_stats* stats);

/* ---- single steps (teacher forcing / API parity) -----------------------
 * These calls stage their own input in the context's buffers: afterwards
 * the context holds no resident cloud (gmmb_fit_*_resident return 2 until
 * the next gmmb_upload / gmmb_fit_k / gmmb_ingest_images). */
/* kinit (sogmm.hpp:52, sogmm.cpp:197-337): labels[N] = column of the 0 in
 * each row of the one-hot log_gamma; centers[k] = k-means++ seed indices. */
int gmmb_kinit(gmmb_ctx* ctx, const double* pts, int64_t n, int d, int k,
               uint64_t seed, int32_t* labels, int64_t* centers);

/* e_step (sogmm.hpp:55-57, sogmm.cpp:341-395) in FP64: ll and optionally
 * the N x M log responsibilities (nullable). */
int gmmb_e_step(gmmb_ctx* ctx, const double* pts, int64_t n, int d, int m,
                const double* w, const double* mu, const double* cov,
                double* ll_out, double* log_gamma_out);

/* Device ingest (ingest.hpp:27-35, ingest.cpp:27-75): decimate(depth, f),
 * decimate(intensity, f) and image_pair_to_cloud with intrinsics.decimated(f),
 * on the GPU. Images are width x height row-major uint16; the resulting
 * N x 4 cloud (row-major pixel order, zero depths dropped) becomes the
 * context's resident cloud for gmmb_fit_k_resident; pts_out (optional, N x 4
 * column-major, capacity (width/f)*(height/f)*4) receives a copy, n_out its
 * size. Errors: invalid_argument (2) for bad factor / intrinsics,
 * NumericalError (3) when every depth is zero. */
int gmmb_ingest_images(gmmb_ctx* ctx, const uint16_t* depth, const uint16_t* intensity, int width,
                       int height, double intensity_max, double fx, double fy, double cx,
                       double cy, double depth_scale, int factor, double* pts_out,
                       int64_t* n_out);

/* GbmsParams (sogmm.hpp:12-22). */
typedef struct gmmb_gbms_params {
  double bandwidth;        /* in (0, 1], normalised units; default 0.015 */
  int max_iters;           /* default 100 */
  double convergence_tol;  /* mean seed displacement; default 1e-5 */
  double merge_radius;     /* <= 0: bandwidth / 2 */
} gmmb_gbms_params;
void gmmb_gbms_params_default(gmmb_gbms_params* p);

/* gbms_estimate_components (sogmm.hpp:33-34, sogmm.cpp:22-195) on the
 * device: binned seeding, blurring mean shift with seed folding, single-
 * linkage merge. modes (optional): components x 4 row-major, original
 * coordinates, up to modes_capacity rows. D = 3 runs on the 4D embedding. */
int gmmb_gbms(gmmb_ctx* ctx, const double* pts, int64_t n, int d, const gmmb_gbms_params* gp,
              int* components, int* iterations, double* modes, int modes_capacity);

/* fit (sogmm.hpp:74-75, sogmm.cpp:465-510): GBMS decides K, then the fit of
 * gmmb_fit_k. Outputs sized for capacity components (returns 2 with
 * *gbms_components set when K exceeds it). */
int gmmb_fit(gmmb_ctx* ctx, const double* pts, int64_t n, int d, const gmmb_gbms_params* gp,
             const gmmb_em_params* em, int capacity, double* w_out, double* mu_out,
             double* cov_out, double* ll_trace, gmmb_fit_stats* stats, int* gbms_components);

/* score (inference.hpp:33, inference.cpp:141-172): average log-likelihood
 * of the cloud under the model (natural log, FP64); point_ll_out (n,
 * optional) receives each point's log-sum-exp. D = 3 or 4; 4 is the
 * reference's Gmm4. */
int gmmb_score(gmmb_ctx* ctx, const double* pts, int64_t n, int d, int m, const double* w,
               const double* mu, const double* cov, double* avg_ll_out, double* point_ll_out);

/* joint_dist_sample (inference.hpp:13-14, inference.cpp:17-54): n draws,
 * out = n x d column-major; draw i depends only on (seed, i) through the
 * reference's counter RNG (component: rng::uniform(seed, 0, i); normals:
 * rng::normal_pair(seed, 1, 4i) and (seed, 1, 4i + 2)). */
int gmmb_sample(gmmb_ctx* ctx, int d, int m, const double* w, const double* mu,
                const double* cov, int64_t n, uint64_t seed, double* out);

/* color_conditional (inference.hpp:25-27, inference.cpp:56-139): expected
 * intensity and variance at n 3D locations (locs n x 3 column-major) under
 * a 4D model; clamp != 0 clamps the expectation to [0, 1]. */
int gmmb_color_conditional(gmmb_ctx* ctx, int m, const double* w, const double* mu,
                           const double* cov, const double* locs, int64_t n, int clamp,
                           double* expected, double* variance);

/* m_step (sogmm.hpp:62-63, sogmm.cpp:399-463) from an N x M log_gamma.
 * Outputs sized for m; *m_out = kept components; *removed = m - *m_out. */
int gmmb_m_step(gmmb_ctx* ctx, const double* pts, int64_t n, int d,
                const double* log_gamma, int m, double cov_reg, double* w_out,
                double* mu_out, double* cov_out, int* m_out, int* removed);

/* One fused EM iteration of the production path (E step + sufficient
 * statistics + M step) on a given model: ll of the E step and the model
 * the next iteration would use. */
int gmmb_em_step(gmmb_ctx* ctx, const double* pts, int64_t n, int d, int m,
                 const double* w, const double* mu, const double* cov,
                 double cov_reg, double* ll_out, double* w_out,
                 double* mu_out, double* cov_out, int* m_out, int* removed);

/* cholesky_cache (gmm.hpp:44-52, gmm.cpp:33-48) on the device, FP64:
 * lower/precision as M x D x D row-major, log_det_terms[M]. */
int gmmb_cholesky_cache(gmmb_ctx* ctx, int d, int m, const double* covs,
                        double* lower, double* precision,
                        double* log_det_terms);

/* Sharded k-means++ keys (sogmm.cpp:210-213 hash 4 contiguous doubles of
 * the GLOBAL column-major buffer): the 3 doubles that follow shard `rank`'s
 * last x value. heads[r*8 + 0..2] = first 3 x of shard r, [3..5] = its first
 * 3 y, [6] = its point count. Host-only helper (no device needed). */
int gmmb_shard_key_tail(const double* heads, int world, int rank,
                        double* tail3);

/* FP32 FFMA throughput microbenchmark (the E step's roofline denominator):
 * runs ~`ms_target` ms of dependent-free FFMA chains on every SM and
 * returns TFLOP/s (2 flops per FFMA) and the elapsed device ms. */
int gmmb_ffma_peak(gmmb_ctx* ctx, double ms_target, double* tflops,
                   double* ms);

/* ---- model I/O (gmm_io.hpp:21-33, gmm_io.cpp:71-177), host ------------
 * Binary "SGMM4D01" (f32 payload) and the JSON mirror (full precision), 4D
 * models (means m x 4, covariances m x 10 packed). Load applies the
 * reference's checks (finalize_loaded): returns 1 for format / truncation /
 * open errors (GmmFormatError / GmmTruncatedError / IoError), 3 for
 * non-finite, non-positive or non-normalised weights and non-SPD
 * covariances, 2 if capacity < M (*m_out still set). Messages via
 * gmmb_io_last_error. */
const char* gmmb_io_last_error(void);
int gmmb_save_model(const char* path, int m, const double* w, const double* mu,
                    const double* cov);
int gmmb_load_model(const char* path, int capacity, double* w, double* mu, double* cov,
                    int* m_out);
int gmmb_save_model_json(const char* path, int m, const double* w, const double* mu,
                         const double* cov);
int gmmb_load_model_json(const char* path, int capacity, double* w, double* mu, double* cov,
                         int* m_out);

/* ---- synthetic inputs (synthetic.cpp / ingest.cpp restated, host) ------
 * make_synthetic_frame + image_pair_to_cloud (synthetic.cpp:9-72,
 * ingest.cpp:27-57): writes up to width*height points (col-major, D=4,
 * capacity width*height rows, leading dimension = *n_out). */
int gmmb_synthetic_frame_cloud(int width, int height, double depth_scale,
                               double* pts_out, int64_t* n_out);
/* make_synthetic_frame (synthetic.cpp:9-72): the depth (depth_scale units)
 * and 8-bit intensity images, width x height row-major; intr_out (optional)
 * = fx, fy, cx, cy. */
int gmmb_synthetic_frame_images(int width, int height, double depth_scale, uint16_t* depth_out,
                                uint16_t* intensity_out, double* intr_out);
/* make_structured_scene (synthetic.cpp:94-129): N x 4 col-major. */
int gmmb_structured_scene(int64_t n, uint64_t seed, double noise_sigma,
                          double* pts_out);
/* make_blob_cloud (synthetic.cpp:74-92): centers[k*4] row-major. */
int gmmb_blob_cloud(const double* centers, int k, double sigma,
                    int64_t per_blob, uint64_t seed, double* pts_out);
/* cfg3 frame jitter: xyz += sigma * normal_pair(seed, 13, 4i..) (D=4). */
int gmmb_jitter_cloud(double* pts, int64_t n, double sigma, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif /* GMMB_H_ */
