// Minimal C++ caller of the drop-in API (include/gmmb.hpp): three 4D blobs,
// K = 3, k-means++ + EM; prints the fit. Exit codes follow the reference CLI
// (gmmscape_cli.cpp:508-528): 1 I/O/device, 2 invalid argument, 3 numerical.
#include <cstdio>
#include <vector>

#include "gmmb.hpp"

int main() {
  const double centers[12] = {0.1, 0.1, 0.1, 0.2, 0.5, 0.5, 0.5, 0.5, 0.9, 0.9, 0.9, 0.8};
  gmmb::PointCloud cloud;
  cloud.dim = 4;
  cloud.points.resize(4 * 3 * 1000);
  gmmb::check(gmmb_blob_cloud(centers, 3, 0.02, 1000, 7, cloud.points.data()));
  try {
    gmmb::Context ctx(0);
    gmmb::EmParams em;
    em.max_iters = 50;
    em.ll_rel_tol = 1e-6;
    const gmmb::FitResult r = gmmb::fit_k(ctx, cloud, 3, em);
    std::printf("K=%d iters=%d ll=%.6f removed=%d\n", r.model.components(), r.em_iterations,
                r.final_log_likelihood, r.removed_components);
    for (int k = 0; k < r.model.components(); ++k) {
      std::printf("  w=%.4f mu=(%.4f %.4f %.4f %.4f)\n", r.model.weights[k],
                  r.model.means[4 * k], r.model.means[4 * k + 1], r.model.means[4 * k + 2],
                  r.model.means[4 * k + 3]);
    }
    return 0;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "invalid argument: %s\n", e.what());
    return 2;
  } catch (const gmmb::NumericalError& e) {
    std::fprintf(stderr, "numerical error: %s\n", e.what());
    return 3;
  } catch (const gmmb::IoError& e) {
    std::fprintf(stderr, "device error: %s\n", e.what());
    return 1;
  }
}
