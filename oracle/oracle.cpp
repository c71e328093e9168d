// oracle.cpp — TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Eigen-free FP64 restatement of the gmmscape hot path. Every function cites
// the reference file:line it follows (paths relative to
// /root/reference/proj). The reference's data-parallel structure is kept:
// fixed 4096-point blocks (common.hpp:46-53) handed to a spawn-per-call
// std::thread pool with an atomic block counter (common.cpp:25-47), so the
// reduction order is independent of the thread count and the library
// doubles as the multithreaded CPU baseline (kind "port").
//
// Arithmetic notes (Appendix A of SURVEY.md):
//  * built with -O3 -ffp-contract=off and no -march (SSE2, no FMA), like the
//    reference Release build (CMakeLists.txt:8-10);
//  * Eigen's element-wise expressions are evaluated left-to-right per
//    element, which this file reproduces exactly (k-means++ distances are
//    therefore bit-identical);
//  * Eigen's vectorised .sum() and packet exp/log are replaced by
//    left-to-right sums and glibc exp/log: rounding-level differences only
//    (this is the unpinned part of the oracle).

#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <string>
#include <thread>
#include <vector>
#include <array>
#include <numeric>
#include <map>

namespace {

constexpr int64_t kPointBlock = 4096;              // common.hpp:49
constexpr double kDegenerateCount = 1e-10;         // kernels.hpp:61
constexpr double kLog2Pi = 1.8378770664093454836;  // sogmm.cpp:19
constexpr double kNegInf = -std::numeric_limits<double>::infinity();
constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr int kRow[10] = {0, 1, 1, 2, 2, 2, 3, 3, 3, 3};  // packed10.hpp:13
constexpr int kCol[10] = {0, 0, 1, 0, 1, 2, 0, 1, 2, 3};  // packed10.hpp:14

thread_local std::string g_err;
std::atomic<int> g_num_threads{0};

struct ArgError {
  std::string msg;
};
struct NumError {
  std::string msg;
};

int64_t num_blocks(int64_t n) { return (n + kPointBlock - 1) / kPointBlock; }

// common.cpp:25-47 — spawn/join per call, dynamic block hand-out.
void parallel_for_blocks(int64_t nb, const std::function<void(int64_t)>& fn) {
  if (nb <= 0) return;
  const int workers =
      static_cast<int>(std::min<int64_t>(orc_num_threads(), nb));
  if (workers <= 1) {
    for (int64_t b = 0; b < nb; ++b) fn(b);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  pool.reserve(workers);
  for (int w = 0; w < workers; ++w) {
    pool.emplace_back([&] {
      for (;;) {
        const int64_t b = next.fetch_add(1);
        if (b >= nb) break;
        fn(b);
      }
    });
  }
  for (auto& t : pool) t.join();
}

// 4x4 column-major helpers (Eigen Matrix4d default storage).
inline double& at(double* m, int r, int c) { return m[c * 4 + r]; }
inline double at(const double* m, int r, int c) { return m[c * 4 + r]; }

void unpack_symmetric4(const double* p, double* m) {  // packed10.hpp:22-29
  for (int k = 0; k < 10; ++k) {
    at(m, kRow[k], kCol[k]) = p[k];
    at(m, kCol[k], kRow[k]) = p[k];
  }
}

bool cholesky4(const double* a, double* lower) {  // kernels.cpp:10-25
  for (int i = 0; i < 16; ++i) lower[i] = 0.0;
  for (int j = 0; j < 4; ++j) {
    double d = at(a, j, j);
    for (int k = 0; k < j; ++k) d -= at(lower, j, k) * at(lower, j, k);
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    const double ljj = std::sqrt(d);
    at(lower, j, j) = ljj;
    for (int i = j + 1; i < 4; ++i) {
      double s = at(a, i, j);
      for (int k = 0; k < j; ++k) s -= at(lower, i, k) * at(lower, j, k);
      at(lower, i, j) = s / ljj;
    }
  }
  return true;
}

void tri_lower_solve4(const double* lower, const double* b, double* x) {
  for (int i = 0; i < 4; ++i) {  // kernels.cpp:27-39
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= at(lower, i, k) * x[k];
    if (at(lower, i, i) == 0.0) {
      throw NumError{"triangular solve: zero diagonal at row " +
                     std::to_string(i)};
    }
    x[i] = s / at(lower, i, i);
  }
}

void lower_inverse4(const double* lower, double* inv) {  // kernels.cpp:41-50
  for (int i = 0; i < 16; ++i) inv[i] = 0.0;
  for (int c = 0; c < 4; ++c) {
    double e[4] = {0, 0, 0, 0};
    e[c] = 1.0;
    double x[4];
    tri_lower_solve4(lower, e, x);
    for (int r = c; r < 4; ++r) at(inv, r, c) = x[r];
  }
}

struct Model {
  std::vector<double> w, mu, cov;  // M, M x 4 row-major, M x 10 packed
  int m() const { return static_cast<int>(w.size()); }
};

struct Cache {
  std::vector<double> lower, prec, logdet;  // M x 16, M x 16, M
};

Cache cholesky_cache(const Model& model) {  // gmm.cpp:33-48
  const int m = model.m();
  Cache c;
  c.lower.assign(static_cast<size_t>(m) * 16, 0.0);
  c.prec.assign(static_cast<size_t>(m) * 16, 0.0);
  c.logdet.assign(m, 0.0);
  // batched_cholesky (kernels.cpp:52-77): one 4096-block covers M <= 4096;
  // report the first failing index.
  int first_bad = m;
  for (int b = 0; b < m; ++b) {
    double a[16];
    unpack_symmetric4(&model.cov[b * 10], a);
    if (!cholesky4(a, &c.lower[b * 16])) {
      first_bad = std::min(first_bad, b);
      break;
    }
  }
  if (first_bad < m) {
    throw NumError{"cholesky failed: block " + std::to_string(first_bad) +
                   " is not positive definite"};
  }
  for (int b = 0; b < m; ++b) {
    double* p = &c.prec[b * 16];
    lower_inverse4(&c.lower[b * 16], p);
    // Eigen's fixed-size 4-element sum unrolls pairwise (gmm.cpp:45).
    c.logdet[b] = (std::log(at(p, 0, 0)) + std::log(at(p, 1, 1))) +
                  (std::log(at(p, 2, 2)) + std::log(at(p, 3, 3)));
  }
  return c;
}

// kernels.cpp:104-135
void logsumexp_rows(const double* mat, int64_t n, int64_t m, double* out) {
  if (n == 0) return;
  parallel_for_blocks(num_blocks(n), [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
    std::vector<double> mx(mat + r0, mat + r0 + len);
    for (int64_t j = 1; j < m; ++j) {
      const double* col = mat + j * n + r0;
      for (int64_t i = 0; i < len; ++i) mx[i] = std::max(mx[i], col[i]);
    }
    std::vector<double> acc(len, 0.0);
    for (int64_t j = 0; j < m; ++j) {
      const double* col = mat + j * n + r0;
      for (int64_t i = 0; i < len; ++i) {
        acc[i] += std::exp(std::max(col[i] - mx[i], -700.0));
      }
    }
    for (int64_t i = 0; i < len; ++i) {
      out[r0 + i] = mx[i] == kNegInf ? kNegInf : mx[i] + std::log(acc[i]);
    }
  });
}

struct Moments {
  std::vector<double> counts, means, scatters;  // M, M x 4, M x 16
  std::vector<int> degenerate;
};

// kernels.hpp:82-181. fill(b, r0, len, out) writes linear-domain weights.
template <typename Fill>
Moments weighted_moments_fn(const double* pts, int64_t n, int64_t m,
                            Fill&& fill) {
  const int64_t nb = num_blocks(n);
  std::vector<double> part1(static_cast<size_t>(nb) * m * 5, 0.0);
  parallel_for_blocks(nb, [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
    std::vector<double> w(len);
    double* out = part1.data() + static_cast<size_t>(blk) * m * 5;
    const double* x0 = pts + 0 * n + r0;
    const double* x1 = pts + 1 * n + r0;
    const double* x2 = pts + 2 * n + r0;
    const double* x3 = pts + 3 * n + r0;
    for (int64_t b = 0; b < m; ++b) {
      fill(b, r0, len, w.data());
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
      for (int64_t i = 0; i < len; ++i) {
        s0 += w[i];
        s1 += w[i] * x0[i];
        s2 += w[i] * x1[i];
        s3 += w[i] * x2[i];
        s4 += w[i] * x3[i];
      }
      double* o = out + b * 5;
      o[0] = s0; o[1] = s1; o[2] = s2; o[3] = s3; o[4] = s4;
    }
  });

  Moments wm;
  wm.counts.assign(m, 0.0);
  wm.means.assign(static_cast<size_t>(m) * 4, 0.0);
  for (int64_t blk = 0; blk < nb; ++blk) {  // serial block-order reduce
    const double* in = part1.data() + static_cast<size_t>(blk) * m * 5;
    for (int64_t b = 0; b < m; ++b) {
      wm.counts[b] += in[b * 5 + 0];
      for (int d = 0; d < 4; ++d) wm.means[b * 4 + d] += in[b * 5 + 1 + d];
    }
  }
  for (int64_t b = 0; b < m; ++b) {
    if (wm.counts[b] < kDegenerateCount) {
      wm.degenerate.push_back(static_cast<int>(b));
      for (int d = 0; d < 4; ++d) wm.means[b * 4 + d] = 0.0;
    } else {
      for (int d = 0; d < 4; ++d) wm.means[b * 4 + d] /= wm.counts[b];
    }
  }

  std::vector<double> part2(static_cast<size_t>(nb) * m * 10, 0.0);
  parallel_for_blocks(nb, [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
    std::vector<double> w(len);
    double* out = part2.data() + static_cast<size_t>(blk) * m * 10;
    const double* x0 = pts + 0 * n + r0;
    const double* x1 = pts + 1 * n + r0;
    const double* x2 = pts + 2 * n + r0;
    const double* x3 = pts + 3 * n + r0;
    for (int64_t b = 0; b < m; ++b) {
      fill(b, r0, len, w.data());
      const double m0 = wm.means[b * 4 + 0], m1 = wm.means[b * 4 + 1];
      const double m2 = wm.means[b * 4 + 2], m3 = wm.means[b * 4 + 3];
      double s[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int64_t i = 0; i < len; ++i) {
        const double d0 = x0[i] - m0, d1 = x1[i] - m1;
        const double d2 = x2[i] - m2, d3 = x3[i] - m3;
        // (w * d_r * d_c): Eigen evaluates (w*d_r)*d_c (kernels.hpp:147-156)
        s[0] += w[i] * d0 * d0;
        s[1] += w[i] * d1 * d0;
        s[2] += w[i] * d1 * d1;
        s[3] += w[i] * d2 * d0;
        s[4] += w[i] * d2 * d1;
        s[5] += w[i] * d2 * d2;
        s[6] += w[i] * d3 * d0;
        s[7] += w[i] * d3 * d1;
        s[8] += w[i] * d3 * d2;
        s[9] += w[i] * d3 * d3;
      }
      std::memcpy(out + b * 10, s, sizeof(s));
    }
  });

  wm.scatters.assign(static_cast<size_t>(m) * 16, 0.0);
  std::vector<double> packed(static_cast<size_t>(m) * 10, 0.0);
  for (int64_t blk = 0; blk < nb; ++blk) {
    const double* in = part2.data() + static_cast<size_t>(blk) * m * 10;
    for (int64_t b = 0; b < m; ++b) {
      for (int k = 0; k < 10; ++k) packed[b * 10 + k] += in[b * 10 + k];
    }
  }
  for (int64_t b = 0; b < m; ++b) {
    double* blockb = &wm.scatters[b * 16];
    const double inv =
        wm.counts[b] >= kDegenerateCount ? 1.0 / wm.counts[b] : 0.0;
    for (int k = 0; k < 10; ++k) {
      const double v = packed[b * 10 + k] * inv;
      at(blockb, kRow[k], kCol[k]) = v;
      at(blockb, kCol[k], kRow[k]) = v;
    }
  }
  return wm;
}

// sogmm.cpp:418-455 (everything after weighted_moments_fn).
Model finish_m_step(const Moments& wm, int64_t m, double cov_reg,
                    int* removed_out) {
  std::vector<int> keep;
  size_t di = 0;
  for (int64_t b = 0; b < m; ++b) {
    if (di < wm.degenerate.size() && wm.degenerate[di] == b) {
      ++di;
    } else {
      keep.push_back(static_cast<int>(b));
    }
  }
  if (removed_out) *removed_out = static_cast<int>(m - keep.size());
  if (keep.empty()) throw NumError{"m_step: all components degenerate"};
  Model model;
  const size_t mk = keep.size();
  model.w.resize(mk);
  model.mu.resize(mk * 4);
  model.cov.resize(mk * 10);
  double total = 0.0;
  for (size_t j = 0; j < mk; ++j) total += wm.counts[keep[j]];
  for (size_t j = 0; j < mk; ++j) {
    const int b = keep[j];
    model.w[j] = wm.counts[b] / total;
    for (int d = 0; d < 4; ++d) model.mu[j * 4 + d] = wm.means[b * 4 + d];
    double cov[16];
    std::memcpy(cov, &wm.scatters[b * 16], sizeof(cov));
    for (int d = 0; d < 4; ++d) at(cov, d, d) += cov_reg;
    for (int k = 0; k < 10; ++k) model.cov[j * 10 + k] = at(cov, kRow[k], kCol[k]);
    double lower[16];
    if (!cholesky4(cov, lower)) {
      throw NumError{"m_step: component " + std::to_string(j) +
                     " covariance not positive definite after regularization"};
    }
  }
  return model;
}

// sogmm.cpp:399-416: fill = exp(log_gamma) with < -700 -> 0.
Model m_step_impl(const double* pts, int64_t n, const double* log_gamma,
                  int64_t m, double cov_reg, int* removed_out) {
  if (cov_reg < 0.0) throw ArgError{"cov_reg must be >= 0"};
  Moments wm = weighted_moments_fn(
      pts, n, m, [&](int64_t b, int64_t r0, int64_t len, double* out) {
        const double* seg = log_gamma + b * n + r0;
        for (int64_t i = 0; i < len; ++i) {
          out[i] = seg[i] < -700.0 ? 0.0 : std::exp(std::max(seg[i], -700.0));
        }
      });
  return finish_m_step(wm, m, cov_reg, removed_out);
}

// E-step column value (sogmm.cpp:351-364); identical expression tree.
inline double log_density(const double* p, double base, double d0, double d1,
                          double d2, double d3) {
  const double y0 = at(p, 0, 0) * d0;
  const double y1 = at(p, 1, 0) * d0 + at(p, 1, 1) * d1;
  const double y2 = at(p, 2, 0) * d0 + at(p, 2, 1) * d1 + at(p, 2, 2) * d2;
  const double y3 = at(p, 3, 0) * d0 + at(p, 3, 1) * d1 + at(p, 3, 2) * d2 +
                    at(p, 3, 3) * d3;
  return base - 0.5 * (y0 * y0 + y1 * y1 + y2 * y2 + y3 * y3);
}

// sogmm.cpp:341-383
double e_step_into(const double* pts, int64_t n, const Model& model,
                   const Cache& cache, double* log_gamma) {
  const int m = model.m();
  parallel_for_blocks(m, [&](int64_t b) {
    const double* mu = &model.mu[b * 4];
    const double* p = &cache.prec[b * 16];
    const double base =
        std::log(model.w[b]) + cache.logdet[b] - 2.0 * kLog2Pi;
    double* col = log_gamma + b * n;
    for (int64_t i = 0; i < n; ++i) {
      col[i] = log_density(p, base, pts[i] - mu[0], pts[n + i] - mu[1],
                           pts[2 * n + i] - mu[2], pts[3 * n + i] - mu[3]);
    }
  });
  std::vector<double> row_lse(n);
  logsumexp_rows(log_gamma, n, m, row_lse.data());
  parallel_for_blocks(m, [&](int64_t b) {
    double* col = log_gamma + b * n;
    for (int64_t i = 0; i < n; ++i) col[i] -= row_lse[i];
  });
  const int64_t nb = num_blocks(n);
  std::vector<double> partials(nb, 0.0);
  parallel_for_blocks(nb, [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
    double s = 0.0;
    for (int64_t i = 0; i < len; ++i) s += row_lse[r0 + i];
    partials[blk] = s;
  });
  double ll = 0.0;
  for (double p : partials) ll += p;
  return ll;
}

void validate_cloud(const double* pts, int64_t n) {  // point_cloud.hpp:15-24
  if (n < 1) throw NumError{"point cloud is empty"};
  for (int64_t i = 0; i < 4 * n; ++i) {
    if (!std::isfinite(pts[i])) {
      throw NumError{"point cloud contains non-finite values"};
    }
  }
  double lo = kInf, hi = -kInf;
  for (int64_t i = 0; i < n; ++i) {
    lo = std::min(lo, pts[3 * n + i]);
    hi = std::max(hi, pts[3 * n + i]);
  }
  if (lo < 0.0 || hi > 1.0) throw NumError{"intensity outside [0, 1]"};
}

// kinit: sogmm.cpp:197-337 (returns labels; log_gamma is the one-hot of it)
void kinit(const double* pts, int64_t n, int k, uint64_t seed,
           int64_t* centers_out, int32_t* labels_out) {
  validate_cloud(pts, n);
  if (k < 1 || k > n) {
    throw ArgError{"kinit: k must satisfy 1 <= k <= N"};
  }
  const int64_t nb = num_blocks(n);
  // keys[i] = hash_coords(pts.row(i).data(), 4) on a column-major MatX4:
  // reads the 4 contiguous doubles starting at x_i (sogmm.cpp:210-213).
  std::vector<uint64_t> keys(n);
  for (int64_t i = 0; i < n; ++i) keys[i] = orc_hash_coords(pts + i, 4);

  std::vector<int64_t> centers;
  centers.reserve(k);
  std::vector<char> chosen(n, 0);
  std::vector<double> d2(n, kInf), neg_log_u(n);
  std::vector<int64_t> block_arg(nb);
  std::vector<double> block_min(nb);

  for (int r = 0; r < k; ++r) {
    parallel_for_blocks(nb, [&](int64_t blk) {
      const int64_t r0 = blk * kPointBlock;
      const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
      if (r > 0) {  // :229-238
        const int64_t c = centers.back();
        const double c0 = pts[c], c1 = pts[n + c], c2 = pts[2 * n + c],
                     c3 = pts[3 * n + c];
        for (int64_t i = r0; i < r0 + len; ++i) {
          const double e0 = pts[i] - c0, e1 = pts[n + i] - c1;
          const double e2 = pts[2 * n + i] - c2, e3 = pts[3 * n + i] - c3;
          const double dd = e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3;
          d2[i] = std::min(d2[i], dd);
        }
      }
      for (int64_t i = r0; i < r0 + len; ++i) {  // :239-242
        neg_log_u[i] =
            -std::log(orc_uniform_pos(seed, static_cast<uint64_t>(r), keys[i]));
      }
      int64_t arg = -1;
      double best = kInf;
      if (r == 0) {  // :245-251
        for (int64_t i = r0; i < r0 + len; ++i) {
          if (neg_log_u[i] < best) {
            best = neg_log_u[i];
            arg = i;
          }
        }
      } else {  // :253-261
        for (int64_t i = r0; i < r0 + len; ++i) {
          if (d2[i] > 0.0) {
            const double clock = neg_log_u[i] / d2[i];
            if (clock < best) {
              best = clock;
              arg = i;
            }
          }
        }
      }
      block_arg[blk] = arg;
      block_min[blk] = best;
    });
    int64_t best = -1;  // :267-275
    double best_clock = kInf;
    for (int64_t blk = 0; blk < nb; ++blk) {
      if (block_arg[blk] >= 0 && block_min[blk] < best_clock) {
        best_clock = block_min[blk];
        best = block_arg[blk];
      }
    }
    if (best < 0) {  // :276-284
      for (int64_t i = 0; i < n; ++i) {
        if (!chosen[i]) {
          best = i;
          break;
        }
      }
    }
    chosen[best] = 1;
    centers.push_back(best);
  }

  // :290-312 nearest centre, lower centre index wins ties.
  std::vector<double> cp(static_cast<size_t>(k) * 4);
  for (int b = 0; b < k; ++b) {
    for (int d = 0; d < 4; ++d) cp[b * 4 + d] = pts[d * n + centers[b]];
  }
  std::vector<int32_t> assign(n);
  parallel_for_blocks(nb, [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
    std::vector<double> best(len, kInf);
    for (int b = 0; b < k; ++b) {
      const double c0 = cp[b * 4], c1 = cp[b * 4 + 1], c2 = cp[b * 4 + 2],
                   c3 = cp[b * 4 + 3];
      for (int64_t i = 0; i < len; ++i) {
        const int64_t g = r0 + i;
        const double e0 = pts[g] - c0, e1 = pts[n + g] - c1;
        const double e2 = pts[2 * n + g] - c2, e3 = pts[3 * n + g] - c3;
        const double dd = e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3;
        if (dd < best[i]) {
          best[i] = dd;
          assign[g] = b;
        }
      }
    }
  });

  // :315-331 every component owns a point.
  std::vector<int64_t> owned(k, 0);
  for (int64_t i = 0; i < n; ++i) owned[assign[i]]++;
  for (int b = 0; b < k; ++b) {
    if (owned[b] > 0) continue;
    int donor = 0;
    for (int c = 1; c < k; ++c) {
      if (owned[c] > owned[donor]) donor = c;
    }
    for (int64_t i = 0; i < n; ++i) {
      if (assign[i] == donor) {
        assign[i] = b;
        owned[donor]--;
        owned[b]++;
        break;
      }
    }
  }
  if (centers_out) std::copy(centers.begin(), centers.end(), centers_out);
  if (labels_out) std::copy(assign.begin(), assign.end(), labels_out);
}

Model m_step_labels(const double* pts, int64_t n, const int32_t* labels,
                    int64_t m, double cov_reg, int* removed_out) {
  // exp of the one-hot log_gamma: exactly 1 at the label, 0 elsewhere.
  Moments wm = weighted_moments_fn(
      pts, n, m, [&](int64_t b, int64_t r0, int64_t len, double* out) {
        for (int64_t i = 0; i < len; ++i) {
          out[i] = labels[r0 + i] == b ? 1.0 : 0.0;
        }
      });
  return finish_m_step(wm, m, cov_reg, removed_out);
}

Model model_from(int m, const double* w, const double* mu, const double* cov) {
  Model md;
  md.w.assign(w, w + m);
  md.mu.assign(mu, mu + static_cast<size_t>(m) * 4);
  md.cov.assign(cov, cov + static_cast<size_t>(m) * 10);
  return md;
}

void model_to(const Model& md, double* w, double* mu, double* cov) {
  if (w) std::copy(md.w.begin(), md.w.end(), w);
  if (mu) std::copy(md.mu.begin(), md.mu.end(), mu);
  if (cov) std::copy(md.cov.begin(), md.cov.end(), cov);
}

void check_em(const orc_em_params* em) {
  // sogmm.cpp:468-470, relaxed to ll_rel_tol >= 0 (0 = fixed iterations).
  if (!em || em->max_iters < 1 || !(em->ll_rel_tol >= 0.0)) {
    throw ArgError{"bad EM parameters"};
  }
}

// sogmm.cpp:484-509
void em_loop(const double* pts, int64_t n, Model model,
             const orc_em_params* em, int removed0, double* w_out,
             double* mu_out, double* cov_out, double* ll_trace,
             orc_fit_stats* stats) {
  std::vector<double> log_gamma(static_cast<size_t>(n) * model.m());
  double ll_prev = kNegInf, ll = kNegInf;
  int iters = 0, removed_total = removed0;
  for (int iter = 0; iter < em->max_iters; ++iter) {
    Cache cache = cholesky_cache(model);
    ll = e_step_into(pts, n, model, cache, log_gamma.data()) - em->ll_offset;
    if (ll_trace) ll_trace[iter] = ll;
    ++iters;
    if (iter > 0) {
      const double rel =
          std::abs(ll - ll_prev) / std::max(std::abs(ll_prev), 1e-12);
      if (rel < em->ll_rel_tol) break;
    }
    ll_prev = ll;
    int removed = 0;
    model = m_step_impl(pts, n, log_gamma.data(), model.m(), em->cov_reg,
                        &removed);
    removed_total += removed;
  }
  model_to(model, w_out, mu_out, cov_out);
  if (stats) {
    stats->em_iterations = iters;
    stats->final_log_likelihood = ll;
    stats->removed_components = removed_total;
    stats->k_out = model.m();
  }
}

// Streaming EM: lse per point is kept; log_gamma(b, i) = l_b(x_i) - lse_i is
// recomputed on demand with the identical expression, so every value the
// M-step sees equals the materialised one bit for bit.
void em_loop_streaming(const double* pts, int64_t n, Model model,
                       const orc_em_params* em, double* w_out, double* mu_out,
                       double* cov_out, double* ll_trace,
                       orc_fit_stats* stats) {
  double ll_prev = kNegInf, ll = kNegInf;
  int iters = 0, removed_total = 0;
  std::vector<double> lse(n);
  const int64_t nb = num_blocks(n);
  for (int iter = 0; iter < em->max_iters; ++iter) {
    Cache cache = cholesky_cache(model);
    const int m = model.m();
    std::vector<double> base(m);
    for (int b = 0; b < m; ++b) {
      base[b] = std::log(model.w[b]) + cache.logdet[b] - 2.0 * kLog2Pi;
    }
    auto logd = [&](int64_t b, int64_t i) {
      const double* mu = &model.mu[b * 4];
      return log_density(&cache.prec[b * 16], base[b], pts[i] - mu[0],
                         pts[n + i] - mu[1], pts[2 * n + i] - mu[2],
                         pts[3 * n + i] - mu[3]);
    };
    std::vector<double> partials(nb, 0.0);
    parallel_for_blocks(nb, [&](int64_t blk) {
      const int64_t r0 = blk * kPointBlock;
      const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
      std::vector<double> tile(static_cast<size_t>(len) * m);
      for (int b = 0; b < m; ++b) {
        for (int64_t i = 0; i < len; ++i) tile[b * len + i] = logd(b, r0 + i);
      }
      std::vector<double> mx(tile.begin(), tile.begin() + len);
      for (int b = 1; b < m; ++b) {
        for (int64_t i = 0; i < len; ++i) mx[i] = std::max(mx[i], tile[b * len + i]);
      }
      std::vector<double> acc(len, 0.0);
      for (int b = 0; b < m; ++b) {
        for (int64_t i = 0; i < len; ++i) {
          acc[i] += std::exp(std::max(tile[b * len + i] - mx[i], -700.0));
        }
      }
      double s = 0.0;
      for (int64_t i = 0; i < len; ++i) {
        lse[r0 + i] = mx[i] == kNegInf ? kNegInf : mx[i] + std::log(acc[i]);
        s += lse[r0 + i];
      }
      partials[blk] = s;
    });
    ll = 0.0;
    for (double p : partials) ll += p;
    ll -= em->ll_offset;
    if (ll_trace) ll_trace[iter] = ll;
    ++iters;
    if (iter > 0) {
      const double rel =
          std::abs(ll - ll_prev) / std::max(std::abs(ll_prev), 1e-12);
      if (rel < em->ll_rel_tol) break;
    }
    ll_prev = ll;
    if (em->cov_reg < 0.0) throw ArgError{"cov_reg must be >= 0"};
    Moments wm = weighted_moments_fn(
        pts, n, m, [&](int64_t b, int64_t r0, int64_t len, double* out) {
          for (int64_t i = 0; i < len; ++i) {
            const double g = logd(b, r0 + i) - lse[r0 + i];
            out[i] = g < -700.0 ? 0.0 : std::exp(std::max(g, -700.0));
          }
        });
    int removed = 0;
    model = finish_m_step(wm, m, em->cov_reg, &removed);
    removed_total += removed;
  }
  model_to(model, w_out, mu_out, cov_out);
  if (stats) {
    stats->em_iterations = iters;
    stats->final_log_likelihood = ll;
    stats->removed_components = removed_total;
    stats->k_out = model.m();
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ArgError& e) {
    g_err = e.msg;
    return 2;
  } catch (const NumError& e) {
    g_err = e.msg;
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

}  // namespace

// ---- inference.cpp restatements (score, joint_dist_sample, color_conditional)

// 3x3 Cholesky (Eigen LLT semantics: column algorithm) and L L^T x = b solve
bool cholesky3(const double* a, double* l) {  // a, l column-major 3x3
  for (int i = 0; i < 9; ++i) l[i] = 0.0;
  for (int j = 0; j < 3; ++j) {
    double d = a[j * 3 + j];
    for (int k = 0; k < j; ++k) d -= l[k * 3 + j] * l[k * 3 + j];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    const double ljj = std::sqrt(d);
    l[j * 3 + j] = ljj;
    for (int i = j + 1; i < 3; ++i) {
      double s2 = a[j * 3 + i];
      for (int k = 0; k < j; ++k) s2 -= l[k * 3 + i] * l[k * 3 + j];
      l[j * 3 + i] = s2 / ljj;
    }
  }
  return true;
}
void llt_solve3(const double* l, const double* b, double* x) {
  double y[3];
  for (int i = 0; i < 3; ++i) {
    double s2 = b[i];
    for (int k = 0; k < i; ++k) s2 -= l[k * 3 + i] * y[k];
    y[i] = s2 / l[i * 3 + i];
  }
  for (int i = 2; i >= 0; --i) {
    double s2 = y[i];
    for (int k = i + 1; k < 3; ++k) s2 -= l[i * 3 + k] * x[k];
    x[i] = s2 / l[i * 3 + i];
  }
}

// inference.cpp:141-172: average log-likelihood
double score(const double* pts, int64_t n, const Model& md) {
  const Cache c = cholesky_cache(md);
  const int m = md.m();
  std::vector<double> base(m);
  for (int b = 0; b < m; ++b) base[b] = std::log(md.w[b]) + c.logdet[b] - 2.0 * kLog2Pi;
  const int64_t nb = num_blocks(n);
  std::vector<double> partials(nb, 0.0);
  parallel_for_blocks(nb, [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t len = std::min<int64_t>(n, r0 + kPointBlock) - r0;
    std::vector<double> block(static_cast<size_t>(len) * m), lse(len);
    for (int b = 0; b < m; ++b) {
      const double* mu = &md.mu[b * 4];
      const double* p = &c.prec[b * 16];
      for (int64_t i = 0; i < len; ++i) {
        const int64_t g = r0 + i;
        block[b * len + i] = log_density(p, base[b], pts[g] - mu[0], pts[n + g] - mu[1],
                                         pts[2 * n + g] - mu[2], pts[3 * n + g] - mu[3]);
      }
    }
    logsumexp_rows(block.data(), len, m, lse.data());
    double s2 = 0.0;
    for (int64_t i = 0; i < len; ++i) s2 += lse[i];
    partials[blk] = s2;
  });
  double total = 0.0;
  for (double p : partials) total += p;
  return total / static_cast<double>(n);
}

// inference.cpp:17-54: draws (n x 4 column-major)
void joint_dist_sample(const Model& md, int64_t n, uint64_t seed, double* out) {
  const Cache c = cholesky_cache(md);
  const int m = md.m();
  std::vector<double> cdf(m);
  double acc = 0.0;
  for (int b = 0; b < m; ++b) {
    acc += md.w[b];
    cdf[b] = acc;
  }
  cdf[m - 1] = 1.0;
  parallel_for_blocks(num_blocks(n), [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t r1 = std::min<int64_t>(n, r0 + kPointBlock);
    for (int64_t i = r0; i < r1; ++i) {
      const double u = orc_uniform(seed, 0, static_cast<uint64_t>(i));
      int b = 0;
      while (b < m - 1 && u >= cdf[b]) ++b;
      double z[4];
      orc_normal_pair(seed, 1, static_cast<uint64_t>(i) * 4, &z[0], &z[1]);
      orc_normal_pair(seed, 1, static_cast<uint64_t>(i) * 4 + 2, &z[2], &z[3]);
      const double* L = &c.lower[b * 16];
      for (int r = 0; r < 4; ++r) {
        double v = at(L, r, 0) * z[0];
        for (int j = 1; j < 4; ++j) v = v + at(L, r, j) * z[j];
        out[r * n + i] = md.mu[b * 4 + r] + v;
      }
    }
  });
}

// inference.cpp:56-139: E[intensity | xyz] and Var
void color_conditional(const Model& md, const double* locs, int64_t n, int clamp,
                       double* expected, double* variance) {
  const int m = md.m();
  std::vector<double> xx_inv(m * 9), mux(m * 3), reg(m * 3), mui(m), cvar(m), gbase(m);
  for (int b = 0; b < m; ++b) {
    double cov[16];
    unpack_symmetric4(&md.cov[b * 10], cov);
    double sxx[9], sxi[3], l[9];
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) sxx[j * 3 + i] = at(cov, i, j);
      sxi[i] = at(cov, i, 3);
    }
    if (!cholesky3(sxx, l)) {
      throw NumError{"spatial covariance of component " + std::to_string(b) +
                     " is not positive definite"};
    }
    for (int col = 0; col < 3; ++col) {
      double e[3] = {0, 0, 0}, x[3];
      e[col] = 1.0;
      llt_solve3(l, e, x);
      for (int i = 0; i < 3; ++i) xx_inv[b * 9 + col * 3 + i] = x[i];
    }
    llt_solve3(l, sxi, &reg[b * 3]);
    for (int i = 0; i < 3; ++i) mux[b * 3 + i] = md.mu[b * 4 + i];
    mui[b] = md.mu[b * 4 + 3];
    cvar[b] = at(cov, 3, 3) - (sxi[0] * reg[b * 3] + sxi[1] * reg[b * 3 + 1] + sxi[2] * reg[b * 3 + 2]);
    const double log_det = 2.0 * ((std::log(l[0]) + std::log(l[4])) + std::log(l[8]));
    gbase[b] = std::log(md.w[b]) - 0.5 * (3.0 * kLog2Pi + log_det);
  }
  std::atomic<int> bad{0};
  std::atomic<int64_t> bad_idx{-1};
  std::vector<double> vbad(1, 0.0);
  parallel_for_blocks(num_blocks(n), [&](int64_t blk) {
    const int64_t r0 = blk * kPointBlock;
    const int64_t r1 = std::min<int64_t>(n, r0 + kPointBlock);
    std::vector<double> lg(m), cm(m), mh(m);
    for (int64_t i = r0; i < r1; ++i) {
      const double x[3] = {locs[i], locs[n + i], locs[2 * n + i]};
      double mx = kNegInf;
      for (int b = 0; b < m; ++b) {
        const double d[3] = {x[0] - mux[b * 3], x[1] - mux[b * 3 + 1], x[2] - mux[b * 3 + 2]};
        const double* A = &xx_inv[b * 9];
        double q = 0.0;
        for (int r = 0; r < 3; ++r) {
          const double ad = A[0 * 3 + r] * d[0] + A[1 * 3 + r] * d[1] + A[2 * 3 + r] * d[2];
          q += d[r] * ad;
        }
        mh[b] = q;
        lg[b] = gbase[b] - 0.5 * q;
        cm[b] = mui[b] + (reg[b * 3] * d[0] + reg[b * 3 + 1] * d[1] + reg[b * 3 + 2] * d[2]);
        if (lg[b] > mx) mx = lg[b];
      }
      double e = 0.0, second = 0.0;
      if (mx == kNegInf || !std::isfinite(mx)) {
        int b = 0;
        for (int q = 1; q < m; ++q)
          if (mh[q] < mh[b]) b = q;
        e = cm[b];
        second = cvar[b] + e * e;
      } else {
        double norm = 0.0;
        for (int b = 0; b < m; ++b) {
          const double w = std::exp(lg[b] - mx);
          norm += w;
          e += w * cm[b];
          second += w * (cvar[b] + cm[b] * cm[b]);
        }
        e /= norm;
        second /= norm;
      }
      double v = second - e * e;
      if (v < -1e-12) {
        bad = 1;
        bad_idx = i;
      }
      if (v < 0.0) v = 0.0;
      variance[i] = v;
      expected[i] = clamp ? std::min(std::max(e, 0.0), 1.0) : e;
    }
  });
  if (bad) throw NumError{"conditional variance below tolerance"};
}

// ---- GBMS component estimation (sogmm.cpp:22-195, kdtree.hpp:13-99) -------

// KdTree4 (kdtree.hpp): median split on the widest axis, leaf size 16,
// std::nth_element partitions — restated verbatim so radius queries visit
// points in the reference's order (it fixes the FP summation order).
class KdTree4 {
 public:
  KdTree4(const std::vector<double>& pts, int n, int leaf = 16)
      : pts_(pts), n_(n), leaf_(leaf) {
    idx_.resize(n);
    std::iota(idx_.begin(), idx_.end(), 0);
    if (n > 0) {
      nodes_.reserve(2 * n / leaf_ + 2);
      build(0, n);
    }
  }
  template <typename V>
  void for_each_in_radius(const double* q, double r, V&& visit) const {
    if (!nodes_.empty()) search(0, q, r * r, r, visit);
  }

 private:
  struct Node {
    int begin, end, axis = -1;
    double split = 0.0;
    int left = -1, right = -1;
  };
  double at(int row, int d) const { return pts_[static_cast<size_t>(row) * 4 + d]; }
  int build(int begin, int end) {
    const int id = static_cast<int>(nodes_.size());
    nodes_.push_back({begin, end});
    if (end - begin <= leaf_) return id;
    double lo[4], hi[4];
    for (int d = 0; d < 4; ++d) lo[d] = hi[d] = at(idx_[begin], d);
    for (int i = begin + 1; i < end; ++i)
      for (int d = 0; d < 4; ++d) {
        lo[d] = std::min(lo[d], at(idx_[i], d));
        hi[d] = std::max(hi[d], at(idx_[i], d));
      }
    int axis = 0;  // Eigen maxCoeff: first maximum
    for (int d = 1; d < 4; ++d)
      if (hi[d] - lo[d] > hi[axis] - lo[axis]) axis = d;
    if (hi[axis] - lo[axis] <= 0.0) return id;
    const int mid = begin + (end - begin) / 2;
    std::nth_element(idx_.begin() + begin, idx_.begin() + mid, idx_.begin() + end,
                     [&](int a, int b) { return at(a, axis) < at(b, axis); });
    nodes_[id].axis = axis;
    nodes_[id].split = at(idx_[mid], axis);
    const int l = build(begin, mid);
    const int r = build(mid, end);
    nodes_[id].left = l;
    nodes_[id].right = r;
    return id;
  }
  template <typename V>
  void search(int id, const double* q, double r2, double r, V&& visit) const {
    const Node& nd = nodes_[id];
    if (nd.axis < 0) {
      for (int i = nd.begin; i < nd.end; ++i) {
        const int p = idx_[i];
        const double e0 = at(p, 0) - q[0], e1 = at(p, 1) - q[1], e2 = at(p, 2) - q[2],
                     e3 = at(p, 3) - q[3];
        if (((e0 * e0 + e1 * e1) + e2 * e2) + e3 * e3 <= r2) visit(p);
      }
      return;
    }
    const double d = q[nd.axis] - nd.split;
    if (d <= r) search(nd.left, q, r2, r, visit);
    if (d >= -r) search(nd.right, q, r2, r, visit);
  }
  const std::vector<double>& pts_;
  int n_, leaf_;
  std::vector<int> idx_;
  std::vector<Node> nodes_;
};

struct GbmsOut {
  int components = 0, iterations = 0, seeds0 = 0;
  std::vector<double> modes;  // components x 4 row-major
};

GbmsOut gbms(const double* pts, int64_t n, double bw, int max_iters, double tol, double merge_r) {
  if (!(bw > 0.0) || bw > 1.0) throw ArgError{"bandwidth must be in (0, 1]"};
  if (max_iters < 1) throw ArgError{"max_iters must be >= 1"};
  if (!(tol > 0.0)) throw ArgError{"convergence_tol must be > 0"};
  validate_cloud(pts, n);
  double mins[4], ranges[4];
  for (int d = 0; d < 4; ++d) {
    double lo = pts[d * n], hi = pts[d * n];
    for (int64_t i = 1; i < n; ++i) {
      lo = std::min(lo, pts[d * n + i]);
      hi = std::max(hi, pts[d * n + i]);
    }
    mins[d] = lo;
    ranges[d] = hi - lo;
  }
  auto norm = [&](int64_t i, int d) {
    return ranges[d] > 0.0 ? (pts[d * n + i] - mins[d]) / ranges[d] : 0.0;
  };
  std::map<uint64_t, std::pair<std::array<double, 4>, int>> bins;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t key = 0;
    double v[4];
    for (int d = 0; d < 4; ++d) {
      v[d] = norm(i, d);
      const auto cell = static_cast<uint64_t>(v[d] / bw);
      key = (key << 16) | (cell & 0xffff);
    }
    auto it = bins.try_emplace(key, std::array<double, 4>{0, 0, 0, 0}, 0).first;
    for (int d = 0; d < 4; ++d) it->second.first[d] += v[d];
    it->second.second += 1;
  }
  int S = static_cast<int>(bins.size());
  std::vector<double> seeds(static_cast<size_t>(S) * 4), weights(S, 1.0);
  {
    int s = 0;
    for (const auto& kv : bins) {
      for (int d = 0; d < 4; ++d) seeds[s * 4 + d] = kv.second.first[d] / kv.second.second;
      ++s;
    }
  }
  GbmsOut out;
  out.seeds0 = S;
  double total_weight = 0.0;
  for (double w : weights) total_weight += w;
  const double fold_eps = std::max(1e-12, tol * 1e-3);
  for (int iter = 0; iter < max_iters; ++iter) {
    ++out.iterations;
    std::vector<double> next(static_cast<size_t>(S) * 4);
    KdTree4 tree(seeds, S);
    parallel_for_blocks(num_blocks(S), [&](int64_t blk) {
      const int64_t r0 = blk * kPointBlock, r1 = std::min<int64_t>(S, r0 + kPointBlock);
      for (int64_t s = r0; s < r1; ++s) {
        double sum[4] = {0, 0, 0, 0}, mass = 0.0;
        tree.for_each_in_radius(&seeds[s * 4], bw, [&](int j) {
          for (int d = 0; d < 4; ++d) sum[d] += weights[j] * seeds[j * 4 + d];
          mass += weights[j];
        });
        for (int d = 0; d < 4; ++d) next[s * 4 + d] = sum[d] / mass;
      }
    });
    double shift = 0.0;
    for (int s = 0; s < S; ++s) {
      double q = 0.0;
      for (int d = 0; d < 4; ++d) {
        const double e = next[s * 4 + d] - seeds[s * 4 + d];
        q += e * e;
      }
      shift += weights[s] * std::sqrt(q);
    }
    shift /= total_weight;
    seeds.swap(next);
    std::vector<uint64_t> keys(S);
    std::map<uint64_t, std::pair<int, double>> fold;
    std::vector<int> keep;
    for (int s = 0; s < S; ++s) {
      uint64_t key = 0;
      for (int d = 0; d < 4; ++d) {
        const auto cell = static_cast<uint64_t>((seeds[s * 4 + d] + 1.0) / fold_eps);
        key = orc_mix64(key ^ cell);
      }
      keys[s] = key;
      auto [it, ins] = fold.try_emplace(key, s, 0.0);
      if (ins) keep.push_back(s);
      it->second.second += weights[s];
    }
    if (static_cast<int>(keep.size()) < S) {
      std::vector<double> fs(keep.size() * 4), fw(keep.size());
      for (size_t o = 0; o < keep.size(); ++o) {
        for (int d = 0; d < 4; ++d) fs[o * 4 + d] = seeds[keep[o] * 4 + d];
        fw[o] = fold.at(keys[keep[o]]).second;
      }
      seeds.swap(fs);
      weights.swap(fw);
      S = static_cast<int>(keep.size());
    }
    if (shift < tol) break;
  }
  const double mr = merge_r > 0.0 ? merge_r : bw * 0.5;
  std::vector<int> parent(S);
  std::iota(parent.begin(), parent.end(), 0);
  auto find = [&](int a) {
    while (parent[a] != a) {
      parent[a] = parent[parent[a]];
      a = parent[a];
    }
    return a;
  };
  KdTree4 tree(seeds, S);
  for (int s = 0; s < S; ++s) {
    tree.for_each_in_radius(&seeds[s * 4], mr, [&](int j) {
      const int ra = find(s), rb = find(j);
      if (ra != rb) parent[std::max(ra, rb)] = std::min(ra, rb);
    });
  }
  std::vector<int> root_to_mode(S, -1);
  std::vector<std::array<double, 4>> sums;
  std::vector<double> masses;
  for (int s = 0; s < S; ++s) {
    const int r = find(s);
    if (root_to_mode[r] < 0) {
      root_to_mode[r] = static_cast<int>(sums.size());
      sums.push_back({0, 0, 0, 0});
      masses.push_back(0.0);
    }
    for (int d = 0; d < 4; ++d) sums[root_to_mode[r]][d] += weights[s] * seeds[s * 4 + d];
    masses[root_to_mode[r]] += weights[s];
  }
  out.components = static_cast<int>(sums.size());
  out.modes.resize(sums.size() * 4);
  for (size_t m = 0; m < sums.size(); ++m)
    for (int d = 0; d < 4; ++d) {
      const double y = sums[m][d] / masses[m];
      out.modes[m * 4 + d] = ranges[d] > 0.0 ? y * ranges[d] + mins[d] : mins[d];
    }
  return out;
}

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void orc_set_num_threads(int n) { g_num_threads.store(std::max(0, n)); }

int orc_num_threads(void) {
  const int n = g_num_threads.load();
  if (n > 0) return n;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

// rng.hpp:16-20
uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// rng.hpp:22-28
uint64_t orc_bits(uint64_t seed, uint64_t stream, uint64_t counter) {
  constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
  uint64_t h = orc_mix64(seed ^ 0x2545f4914f6cdd1dULL);
  h = orc_mix64(h + stream * kGolden);
  h = orc_mix64(h + counter * kGolden);
  return h;
}

double orc_uniform(uint64_t seed, uint64_t stream, uint64_t counter) {
  return static_cast<double>(orc_bits(seed, stream, counter) >> 11) * 0x1.0p-53;
}

double orc_uniform_pos(uint64_t seed, uint64_t stream, uint64_t counter) {
  return static_cast<double>((orc_bits(seed, stream, counter) >> 11) + 1) *
         0x1.0p-53;
}

void orc_normal_pair(uint64_t seed, uint64_t stream, uint64_t counter,
                     double* z0, double* z1) {  // rng.hpp:45-53
  const double u1 = orc_uniform_pos(seed, stream, counter);
  const double u2 = orc_uniform(seed, stream, counter + 1);
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * M_PI * u2;
  *z0 = r * std::cos(a);
  *z1 = r * std::sin(a);
}

uint64_t orc_hash_coords(const double* x, int n) {  // rng.hpp:64-70
  uint64_t h = 0x6a09e667f3bcc909ULL;
  for (int i = 0; i < n; ++i) h = orc_mix64(h ^ std::bit_cast<uint64_t>(x[i]));
  return h;
}

int orc_cholesky4(const double* a16, double* lower16) {
  return cholesky4(a16, lower16) ? 0 : 3;
}

void orc_lower_inverse4(const double* lower16, double* inv16) {
  try {
    lower_inverse4(lower16, inv16);
  } catch (const NumError& e) {
    g_err = e.msg;
    for (int i = 0; i < 16; ++i) inv16[i] = std::nan("");
  }
}

int orc_batched_cholesky(const double* blocks, int count, double* lower,
                         int* bad) {
  std::atomic<int> first_bad{count};  // kernels.cpp:52-77
  parallel_for_blocks(num_blocks(count), [&](int64_t blk) {
    const int r0 = static_cast<int>(blk * kPointBlock);
    const int r1 = std::min<int>(count, r0 + static_cast<int>(kPointBlock));
    for (int i = r0; i < r1; ++i) {
      double l[16];
      if (!cholesky4(blocks + 16 * i, l)) {
        int expected = first_bad.load();
        while (i < expected && !first_bad.compare_exchange_weak(expected, i)) {
        }
        return;
      }
      std::memcpy(lower + 16 * i, l, sizeof(l));
    }
  });
  if (bad) *bad = first_bad.load() < count ? first_bad.load() : -1;
  if (first_bad.load() < count) {
    g_err = "cholesky failed: block " + std::to_string(first_bad.load()) +
            " is not positive definite";
    return 3;
  }
  return 0;
}

void orc_logsumexp_rows(const double* mat, int64_t n, int64_t m, double* out) {
  logsumexp_rows(mat, n, m, out);
}

int orc_weighted_moments(const double* pts, int64_t n, const double* resp,
                         int64_t m, double* counts, double* means,
                         double* scatters16, int* degenerate_flags) {
  return guarded([&] {
    Moments wm = weighted_moments_fn(
        pts, n, m, [&](int64_t b, int64_t r0, int64_t len, double* out) {
          std::memcpy(out, resp + b * n + r0, sizeof(double) * len);
        });
    std::copy(wm.counts.begin(), wm.counts.end(), counts);
    std::copy(wm.means.begin(), wm.means.end(), means);
    std::copy(wm.scatters.begin(), wm.scatters.end(), scatters16);
    if (degenerate_flags) {
      for (int64_t b = 0; b < m; ++b) degenerate_flags[b] = 0;
      for (int b : wm.degenerate) degenerate_flags[b] = 1;
    }
  });
}

int orc_cholesky_cache(const double* covs, int m, double* lower16,
                       double* precision16, double* log_det_terms) {
  return guarded([&] {
    Model md;
    md.w.assign(m, 1.0 / m);
    md.mu.assign(static_cast<size_t>(m) * 4, 0.0);
    md.cov.assign(covs, covs + static_cast<size_t>(m) * 10);
    Cache c = cholesky_cache(md);
    if (lower16) std::copy(c.lower.begin(), c.lower.end(), lower16);
    if (precision16) std::copy(c.prec.begin(), c.prec.end(), precision16);
    if (log_det_terms) std::copy(c.logdet.begin(), c.logdet.end(), log_det_terms);
  });
}

int orc_validate_cloud(const double* pts, int64_t n) {
  return guarded([&] { validate_cloud(pts, n); });
}

int orc_kinit(const double* pts, int64_t n, int k, uint64_t seed,
              int64_t* centers, int32_t* labels) {
  return guarded([&] { kinit(pts, n, k, seed, centers, labels); });
}

int orc_e_step(const double* pts, int64_t n, int m, const double* weights,
               const double* means, const double* covs, double* log_gamma,
               double* ll) {
  return guarded([&] {
    Model md = model_from(m, weights, means, covs);
    Cache c = cholesky_cache(md);
    std::vector<double> tmp;
    double* lg = log_gamma;
    if (!lg) {
      tmp.resize(static_cast<size_t>(n) * m);
      lg = tmp.data();
    }
    const double v = e_step_into(pts, n, md, c, lg);
    if (ll) *ll = v;
  });
}

int orc_m_step(const double* pts, int64_t n, const double* log_gamma, int m,
               double cov_reg, double* w_out, double* mu_out, double* cov_out,
               int* m_out, int* removed) {
  return guarded([&] {
    Model md = m_step_impl(pts, n, log_gamma, m, cov_reg, removed);
    model_to(md, w_out, mu_out, cov_out);
    if (m_out) *m_out = md.m();
  });
}

int orc_m_step_labels(const double* pts, int64_t n, const int32_t* labels,
                      int m, double cov_reg, double* w_out, double* mu_out,
                      double* cov_out, int* m_out, int* removed) {
  return guarded([&] {
    if (cov_reg < 0.0) throw ArgError{"cov_reg must be >= 0"};
    Model md = m_step_labels(pts, n, labels, m, cov_reg, removed);
    model_to(md, w_out, mu_out, cov_out);
    if (m_out) *m_out = md.m();
  });
}

int orc_fit_from(const double* pts, int64_t n, int m0, const double* w0,
                 const double* mu0, const double* cov0,
                 const orc_em_params* em, double* w_out, double* mu_out,
                 double* cov_out, double* ll_trace, orc_fit_stats* stats) {
  return guarded([&] {
    validate_cloud(pts, n);
    check_em(em);
    if (m0 < 1) throw ArgError{"model has no components"};
    if (stats) stats->k_init = m0;
    em_loop(pts, n, model_from(m0, w0, mu0, cov0), em, 0, w_out, mu_out,
            cov_out, ll_trace, stats);
  });
}

int orc_fit_from_streaming(const double* pts, int64_t n, int m0,
                           const double* w0, const double* mu0,
                           const double* cov0, const orc_em_params* em,
                           double* w_out, double* mu_out, double* cov_out,
                           double* ll_trace, orc_fit_stats* stats) {
  return guarded([&] {
    validate_cloud(pts, n);
    check_em(em);
    if (m0 < 1) throw ArgError{"model has no components"};
    if (stats) stats->k_init = m0;
    em_loop_streaming(pts, n, model_from(m0, w0, mu0, cov0), em, w_out,
                      mu_out, cov_out, ll_trace, stats);
  });
}

int orc_fit_k(const double* pts, int64_t n, int K, const orc_em_params* em,
              double* w_out, double* mu_out, double* cov_out,
              double* ll_trace, orc_fit_stats* stats, int64_t* centers,
              int32_t* labels) {
  return guarded([&] {
    validate_cloud(pts, n);
    check_em(em);
    if (K < 1) throw ArgError{"kinit: k must satisfy 1 <= k <= N"};
    const int k = static_cast<int>(std::min<int64_t>(K, n));  // sogmm.cpp:477
    std::vector<int32_t> lab(n);
    std::vector<int64_t> cen(k);
    kinit(pts, n, k, em->seed, cen.data(), lab.data());
    int removed = 0;
    Model md = m_step_labels(pts, n, lab.data(), k, em->cov_reg, &removed);
    if (centers) std::copy(cen.begin(), cen.end(), centers);
    if (labels) std::copy(lab.begin(), lab.end(), labels);
    if (stats) stats->k_init = k;
    em_loop(pts, n, std::move(md), em, removed, w_out, mu_out, cov_out,
            ll_trace, stats);
  });
}


int orc_score(const double* pts, int64_t n, int m, const double* w, const double* mu,
              const double* cov, double* out) {
  return guarded([&] {
    if (n < 1) throw ArgError{"empty cloud"};
    Model md = model_from(m, w, mu, cov);
    *out = score(pts, n, md);
  });
}

int orc_sample(int m, const double* w, const double* mu, const double* cov, int64_t n,
               uint64_t seed, double* out) {
  return guarded([&] {
    if (n < 1) throw ArgError{"sample count must be >= 1"};
    Model md = model_from(m, w, mu, cov);
    joint_dist_sample(md, n, seed, out);
  });
}

int orc_color_conditional(int m, const double* w, const double* mu, const double* cov,
                          const double* locs, int64_t n, int clamp, double* expected,
                          double* variance) {
  return guarded([&] {
    Model md = model_from(m, w, mu, cov);
    color_conditional(md, locs, n, clamp, expected, variance);
  });
}

int orc_gbms(const double* pts, int64_t n, double bandwidth, int max_iters, double tol,
             double merge_radius, int* components, int* iterations, int* seeds0,
             double* modes, int modes_capacity) {
  return guarded([&] {
    GbmsOut g = gbms(pts, n, bandwidth, max_iters, tol, merge_radius);
    *components = g.components;
    *iterations = g.iterations;
    if (seeds0) *seeds0 = g.seeds0;
    if (modes)
      std::memcpy(modes, g.modes.data(),
                  sizeof(double) * 4 * std::min(g.components, modes_capacity));
  });
}
// ---- benchmark inputs, restated from the reference -----
// make_synthetic_frame (synthetic.cpp:9-72) + image_pair_to_cloud
// (ingest.cpp:27-57, row-major pixels, zero depths dropped): N x 4 col-major
// into pts (capacity width*height rows), *n_out = N. Vec3 dot / squaredNorm
// are ((a0 b0 + a1 b1) + a2 b2), the order Eigen's fixed-size redux yields.
int orc_synthetic_frame_cloud(int width, int height, double depth_scale, double* pts,
                              int64_t* n_out) {
  return guarded([&] {
    if (width < 1 || height < 1 || !(depth_scale > 0.0)) throw ArgError{"bad frame size"};
    const double fx = 525.0 * width / 640.0, fy = 525.0 * width / 640.0;  // :12-13
    const double cx = width * 0.5 - 0.5, cy = height * 0.5 - 0.5;         // :14-15
    const size_t npx = static_cast<size_t>(width) * height;
    std::vector<uint16_t> depth(npx), inten(npx);
    const double scx = 0.35, scy = -0.1, scz = 2.1, sr = 0.35;             // :27-28
    for (int v = 0; v < height; ++v) {
      for (int u = 0; u < width; ++u) {
        const double rx = (u - cx) / fx, ry = (v - cy) / fy;               // :33-34
        double z = 3.0;                                                    // :38
        const double denom = ry + 0.18;                                    // :42-46
        if (denom > 1e-9) {
          const double zd = 0.45 / denom;
          if (zd > 0.4 && zd < z) z = zd;
        }
        const double a = (rx * rx + ry * ry) + 1.0 * 1.0;                  // :49-56
        const double bq = -2.0 * ((rx * scx + ry * scy) + 1.0 * scz);
        const double c = ((scx * scx + scy * scy) + scz * scz) - sr * sr;
        const double disc = bq * bq - 4.0 * a * c;
        if (disc > 0.0) {
          const double t = (-bq - std::sqrt(disc)) / (2.0 * a);
          if (t > 0.0 && t < z) z = t;
        }
        const double px = rx * z, py = ry * z, pz = 1.0 * z;               // :58
        depth[static_cast<size_t>(v) * width + u] =
            static_cast<uint16_t>(std::min(depth_scale * z, 65535.0));     // :59-61
        double in = 0.55 + 0.25 * std::sin(7.0 * px) * std::cos(5.0 * py) +
                    0.15 * std::sin(3.0 * pz);                             // :64-66
        in = std::clamp(in, 0.0, 1.0);
        inten[static_cast<size_t>(v) * width + u] =
            static_cast<uint16_t>(std::lround(in * 255.0));                // :67-68
      }
    }
    int64_t n = 0;
    for (const uint16_t d : depth) n += d > 0;                             // ingest.cpp:33-36
    const double inv_scale = 1.0 / depth_scale, inv_max = 1.0 / 255.0;     // :41-42
    int64_t k = 0;
    for (int v = 0; v < height; ++v) {
      for (int u = 0; u < width; ++u) {
        const uint16_t d = depth[static_cast<size_t>(v) * width + u];
        if (d == 0) continue;
        const double z = d * inv_scale;                                    // :48-53
        pts[0 * n + k] = (u - cx) * z / fx;
        pts[1 * n + k] = (v - cy) * z / fy;
        pts[2 * n + k] = z;
        pts[3 * n + k] = inten[static_cast<size_t>(v) * width + u] * inv_max;
        ++k;
      }
    }
    *n_out = n;
  });
}

// make_structured_scene (synthetic.cpp:94-129): n x 4 col-major.
int orc_structured_scene(int64_t n, uint64_t seed, double noise_sigma, double* pts) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      const auto ctr = static_cast<uint64_t>(i);
      const double u = orc_uniform(seed, 11, ctr * 8), v = orc_uniform(seed, 11, ctr * 8 + 1);
      double nz0, nz1, nz2, unused;
      orc_normal_pair(seed, 12, ctr * 8 + 2, &nz0, &nz1);
      orc_normal_pair(seed, 12, ctr * 8 + 4, &nz2, &unused);
      double x, y, z;
      if (i % 3 == 0) {          // ground plane z = 0
        x = 2.0 * u - 1.0; y = 2.0 * v - 1.0; z = 0.0;
      } else if (i % 3 == 1) {   // wall plane x = 0
        x = 0.0; y = 2.0 * u - 1.0; z = 1.2 * v;
      } else {                   // cylinder along z
        const double ang = 2.0 * M_PI * u;
        x = 0.55 + 0.3 * std::cos(ang); y = -0.35 + 0.3 * std::sin(ang); z = 1.1 * v;
      }
      x += noise_sigma * nz0;
      y += noise_sigma * nz1;
      z += noise_sigma * nz2;
      pts[0 * n + i] = x;
      pts[1 * n + i] = y;
      pts[2 * n + i] = z;
      pts[3 * n + i] =
          std::clamp(0.5 + 0.3 * std::sin(4.0 * x) + 0.2 * std::cos(3.0 * y + z), 0.0, 1.0);
    }
  });
}

// cfg3 frame f (a generator new to this build): xyz of the
// cfg2 frame jittered by sigma * normal_pair(seed = f, stream 13, 4i ...).
int orc_jitter_cloud(double* pts, int64_t n, double sigma, uint64_t seed) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i) {
      double z0, z1, z2, z3;
      orc_normal_pair(seed, 13, static_cast<uint64_t>(i) * 4, &z0, &z1);
      orc_normal_pair(seed, 13, static_cast<uint64_t>(i) * 4 + 2, &z2, &z3);
      pts[0 * n + i] += sigma * z0;
      pts[1 * n + i] += sigma * z1;
      pts[2 * n + i] += sigma * z2;
    }
  });
}
}  // extern "C"
