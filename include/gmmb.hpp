// gmmb.hpp — header-only C++ API over the C ABI (gmmb.h), shaped like the
// reference's gmmscape API (/root/reference/proj/include/gmmscape/sogmm.hpp,
// gmm.hpp, point_cloud.hpp) with Eigen-free value types:
//
//   gmmscape::EmParams          sogmm.hpp:36-41   -> gmmb::EmParams
//   gmmscape::PointCloud4D      point_cloud.hpp   -> gmmb::PointCloud (D = 3|4)
//   gmmscape::Gmm4              gmm.hpp:15-34     -> gmmb::Gmm
//   gmmscape::Responsibilities  sogmm.hpp:44-46   -> gmmb::Responsibilities
//   gmmscape::FitResult         sogmm.hpp:65-71   -> gmmb::FitResult
//   gmmscape::CholeskyCache     gmm.hpp:44-48     -> gmmb::CholeskyCache
//   kinit / e_step / m_step     sogmm.hpp:52-63   -> same names
//   fit(cloud, bandwidth, em)   sogmm.hpp:74-75   -> fit_k(cloud, K, em) / fit_from
//   NumericalError              common.hpp:27-30  -> gmmb::NumericalError
//   IoError                     common.hpp:23-25  -> gmmb::IoError (device errors)
//   std::invalid_argument       (unchanged)
//
// Points are stored exactly like Eigen's column-major MatX4 (x column, then
// y, z, intensity), so a reference caller can pass cloud.points.data()
// without copying.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gmmb.h"

namespace gmmb {

struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int code) {
  if (code == 0) return;
  const std::string msg = gmmb_last_error();
  if (code == 2) throw std::invalid_argument(msg);
  if (code == 3) throw NumericalError(msg);
  throw IoError(msg);
}

struct EmParams {
  int max_iters = 100;
  double ll_rel_tol = 1e-5;  // 0: exactly max_iters E steps (extension)
  double cov_reg = 1e-6;
  std::uint64_t seed = 0;
  gmmb_em_params c() const { return {max_iters, ll_rel_tol, cov_reg, seed}; }
};

// N x D column-major (D = 4: xyz + intensity in [0, 1]; D = 3: xyz).
struct PointCloud {
  int dim = 4;
  std::vector<double> points;
  std::int64_t size() const { return dim ? static_cast<std::int64_t>(points.size()) / dim : 0; }
};

// Packed symmetric storage (packed10.hpp): lower triangle, row-major order.
struct Gmm {
  int dim = 4;
  std::vector<double> weights;      // M
  std::vector<double> means;        // M x D, row-major
  std::vector<double> covariances;  // M x D(D+1)/2
  int components() const { return static_cast<int>(weights.size()); }
  int packed() const { return dim * (dim + 1) / 2; }
  std::int64_t memory_footprint() const {  // gmm.hpp:38-40 (4-byte floats)
    return std::int64_t{4} * components() * (1 + dim + packed());
  }
};

struct Responsibilities {
  std::int64_t n = 0;
  int m = 0;
  std::vector<double> log_gamma;  // N x M column-major
};

struct CholeskyCache {
  std::vector<double> lower;          // M x D x D row-major
  std::vector<double> precision;      // L^-1
  std::vector<double> log_det_terms;  // sum ln diag P = -1/2 ln|Sigma|
};

struct FitResult {
  Gmm model;
  int em_iterations = 0;  // E steps executed
  double final_log_likelihood = 0.0;
  int removed_components = 0;
  int k_init = 0;  // min(K, N)
  bool converged = false;
  std::vector<double> ll_trace;
  gmmb_fit_stats stats{};
};

class Context {
 public:
  explicit Context(int device = 0) { check(gmmb_ctx_create(device, &h_)); }
  Context(int device, int rank, int world, const void* nccl_id) {
    check(gmmb_ctx_create_sharded(device, rank, world, nccl_id, &h_));
  }
  ~Context() { gmmb_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  gmmb_ctx* get() const { return h_; }

 private:
  gmmb_ctx* h_ = nullptr;
};

namespace detail {
inline FitResult finish(Gmm&& m, std::vector<double>&& ll, const gmmb_fit_stats& st) {
  FitResult r;
  m.weights.resize(st.k_out);
  m.means.resize(static_cast<size_t>(st.k_out) * m.dim);
  m.covariances.resize(static_cast<size_t>(st.k_out) * m.packed());
  ll.resize(st.em_iterations);
  r.model = std::move(m);
  r.ll_trace = std::move(ll);
  r.em_iterations = st.em_iterations;
  r.final_log_likelihood = st.final_log_likelihood;
  r.removed_components = st.removed_components;
  r.k_init = st.k_init;
  r.converged = st.converged != 0;
  r.stats = st;
  return r;
}
inline Gmm alloc(int dim, int m) {
  Gmm g;
  g.dim = dim;
  g.weights.resize(m);
  g.means.resize(static_cast<size_t>(m) * dim);
  g.covariances.resize(static_cast<size_t>(m) * g.packed());
  return g;
}
}  // namespace detail

// fit with K given (sogmm.cpp:477-509): kinit -> m_step -> EM loop.
inline FitResult fit_k(Context& ctx, const PointCloud& cloud, int K, const EmParams& em = {}) {
  const std::int64_t n = cloud.size();
  const int k = static_cast<int>(K < n ? K : n);
  Gmm m = detail::alloc(cloud.dim, k > 0 ? k : 1);
  std::vector<double> ll(em.max_iters > 0 ? em.max_iters : 1);
  gmmb_fit_stats st{};
  const gmmb_em_params p = em.c();
  check(gmmb_fit_k(ctx.get(), cloud.points.data(), n, cloud.dim, K, &p, m.weights.data(),
                   m.means.data(), m.covariances.data(), ll.data(), &st, nullptr, nullptr));
  return detail::finish(std::move(m), std::move(ll), st);
}

// EM loop (sogmm.cpp:484-509) from a given model.
inline FitResult fit_from(Context& ctx, const PointCloud& cloud, const Gmm& init,
                          const EmParams& em = {}) {
  Gmm m = detail::alloc(cloud.dim, init.components());
  std::vector<double> ll(em.max_iters > 0 ? em.max_iters : 1);
  gmmb_fit_stats st{};
  const gmmb_em_params p = em.c();
  check(gmmb_fit_from(ctx.get(), cloud.points.data(), cloud.size(), cloud.dim,
                      init.components(), init.weights.data(), init.means.data(),
                      init.covariances.data(), &p, m.weights.data(), m.means.data(),
                      m.covariances.data(), ll.data(), &st));
  return detail::finish(std::move(m), std::move(ll), st);
}

// kinit (sogmm.cpp:197-337): the one-hot log responsibilities.
inline Responsibilities kinit(Context& ctx, const PointCloud& cloud, int k, std::uint64_t seed) {
  const std::int64_t n = cloud.size();
  std::vector<std::int32_t> labels(static_cast<size_t>(n));
  std::vector<std::int64_t> centers(k > 0 ? k : 1);
  check(gmmb_kinit(ctx.get(), cloud.points.data(), n, cloud.dim, k, seed, labels.data(),
                   centers.data()));
  Responsibilities r;
  r.n = n;
  r.m = k;
  r.log_gamma.assign(static_cast<size_t>(n) * k, -std::numeric_limits<double>::infinity());
  for (std::int64_t i = 0; i < n; ++i) r.log_gamma[static_cast<size_t>(labels[i]) * n + i] = 0.0;
  return r;
}

// e_step (sogmm.cpp:387-395): (responsibilities, log-likelihood).
inline std::pair<Responsibilities, double> e_step(Context& ctx, const PointCloud& cloud,
                                                  const Gmm& model) {
  Responsibilities r;
  r.n = cloud.size();
  r.m = model.components();
  r.log_gamma.resize(static_cast<size_t>(r.n) * r.m);
  double ll = 0.0;
  check(gmmb_e_step(ctx.get(), cloud.points.data(), r.n, cloud.dim, r.m, model.weights.data(),
                    model.means.data(), model.covariances.data(), &ll, r.log_gamma.data()));
  return {std::move(r), ll};
}

// m_step (sogmm.cpp:459-463).
inline Gmm m_step(Context& ctx, const PointCloud& cloud, const Responsibilities& resp,
                  double cov_reg, int* removed_out = nullptr) {
  Gmm m = detail::alloc(cloud.dim, resp.m);
  int kept = 0, removed = 0;
  check(gmmb_m_step(ctx.get(), cloud.points.data(), cloud.size(), cloud.dim,
                    resp.log_gamma.data(), resp.m, cov_reg, m.weights.data(), m.means.data(),
                    m.covariances.data(), &kept, &removed));
  m.weights.resize(kept);
  m.means.resize(static_cast<size_t>(kept) * m.dim);
  m.covariances.resize(static_cast<size_t>(kept) * m.packed());
  if (removed_out) *removed_out = removed;
  return m;
}

// cholesky_cache (gmm.cpp:33-48).
inline CholeskyCache cholesky_cache(Context& ctx, const Gmm& model) {
  CholeskyCache c;
  const int m = model.components(), d = model.dim;
  c.lower.resize(static_cast<size_t>(m) * d * d);
  c.precision.resize(static_cast<size_t>(m) * d * d);
  c.log_det_terms.resize(m);
  check(gmmb_cholesky_cache(ctx.get(), d, m, model.covariances.data(), c.lower.data(),
                            c.precision.data(), c.log_det_terms.data()));
  return c;
}

// score (inference.cpp:141-172): average log-likelihood.
inline double score(Context& ctx, const Gmm& model, const PointCloud& cloud) {
  double avg = 0.0;
  check(gmmb_score(ctx.get(), cloud.points.data(), cloud.size(), cloud.dim, model.components(),
                   model.weights.data(), model.means.data(), model.covariances.data(), &avg,
                   nullptr));
  return avg;
}

// joint_dist_sample (inference.cpp:17-54).
inline PointCloud joint_dist_sample(Context& ctx, const Gmm& model, std::int64_t n,
                                    std::uint64_t seed) {
  PointCloud out;
  out.dim = model.dim;
  out.points.resize(static_cast<size_t>(n > 0 ? n : 0) * model.dim);
  check(gmmb_sample(ctx.get(), model.dim, model.components(), model.weights.data(),
                    model.means.data(), model.covariances.data(), n, seed, out.points.data()));
  return out;
}

// color_conditional (inference.cpp:56-139); locs is N x 3 column-major.
struct ConditionalResult {
  std::vector<double> expected_intensity;
  std::vector<double> variance;
};
inline ConditionalResult color_conditional(Context& ctx, const Gmm& model,
                                           const std::vector<double>& locs, bool clamp = true) {
  const std::int64_t n = static_cast<std::int64_t>(locs.size() / 3);
  ConditionalResult r;
  r.expected_intensity.resize(n);
  r.variance.resize(n);
  check(gmmb_color_conditional(ctx.get(), model.components(), model.weights.data(),
                               model.means.data(), model.covariances.data(), locs.data(), n,
                               clamp ? 1 : 0, r.expected_intensity.data(), r.variance.data()));
  return r;
}

}  // namespace gmmb
