// synthetic.cpp — host-side input generators for the benchmark configs.
//
// Restates the reference's data sources so both arms see identical clouds:
//   make_synthetic_frame   /root/reference/proj/src/synthetic.cpp:9-72
//   image_pair_to_cloud    /root/reference/proj/src/ingest.cpp:27-57
//   make_blob_cloud        /root/reference/proj/src/synthetic.cpp:74-92
//   make_structured_scene  /root/reference/proj/src/synthetic.cpp:94-129
// (glibc libm + the rng.hpp counter RNG, evaluated in the same order).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/gmmb.h"
#include "common.cuh"

namespace {

double uniform(uint64_t seed, uint64_t stream, uint64_t counter) {  // rng.hpp:31-34
  return static_cast<double>(gmmb::rng_bits(seed, stream, counter) >> 11) * 0x1.0p-53;
}
double uniform_pos(uint64_t seed, uint64_t stream, uint64_t counter) {
  return static_cast<double>((gmmb::rng_bits(seed, stream, counter) >> 11) + 1) * 0x1.0p-53;
}
void normal_pair(uint64_t seed, uint64_t stream, uint64_t counter, double& z0,
                 double& z1) {  // rng.hpp:45-53
  const double u1 = uniform_pos(seed, stream, counter);
  const double u2 = uniform(seed, stream, counter + 1);
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * M_PI * u2;
  z0 = r * std::cos(a);
  z1 = r * std::sin(a);
}

}  // namespace

extern "C" {

int gmmb_synthetic_frame_images(int width, int height, double depth_scale, uint16_t* depth_out,
                                uint16_t* intensity_out, double* intr_out) {
  if (width < 1 || height < 1 || !(depth_scale > 0.0) || !depth_out || !intensity_out) return 2;
  const double fx = 525.0 * width / 640.0, fy = 525.0 * width / 640.0;
  const double cx = width * 0.5 - 0.5, cy = height * 0.5 - 0.5;
  uint16_t* depth = depth_out;
  uint16_t* inten = intensity_out;
  if (intr_out) {
    intr_out[0] = fx;
    intr_out[1] = fy;
    intr_out[2] = cx;
    intr_out[3] = cy;
  }
  const double sc[3] = {0.35, -0.1, 2.1};
  const double sr = 0.35;
  for (int v = 0; v < height; ++v) {
    for (int u = 0; u < width; ++u) {
      const double rx = (u - cx) / fx;
      const double ry = (v - cy) / fy;
      const double dir[3] = {rx, ry, 1.0};
      double z = 3.0;
      const double denom = ry + 0.18;
      if (denom > 1e-9) {
        const double zd = 0.45 / denom;
        if (zd > 0.4 && zd < z) z = zd;
      }
      // Eigen squaredNorm / dot on Vector3d: ((a0*b0 + a1*b1) + a2*b2)
      const double a = dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2];
      const double bq = -2.0 * (dir[0] * sc[0] + dir[1] * sc[1] + dir[2] * sc[2]);
      const double c = (sc[0] * sc[0] + sc[1] * sc[1] + sc[2] * sc[2]) - sr * sr;
      const double disc = bq * bq - 4.0 * a * c;
      if (disc > 0.0) {
        const double t = (-bq - std::sqrt(disc)) / (2.0 * a);
        if (t > 0.0 && t < z) z = t;
      }
      const double p[3] = {dir[0] * z, dir[1] * z, dir[2] * z};
      const double raw = depth_scale * z;
      depth[static_cast<size_t>(v) * width + u] =
          static_cast<uint16_t>(std::min(raw, 65535.0));
      double in = 0.55 + 0.25 * std::sin(7.0 * p[0]) * std::cos(5.0 * p[1]) +
                  0.15 * std::sin(3.0 * p[2]);
      in = std::clamp(in, 0.0, 1.0);
      inten[static_cast<size_t>(v) * width + u] =
          static_cast<uint16_t>(std::lround(in * 255.0));
    }
  }
  return 0;
}

int gmmb_synthetic_frame_cloud(int width, int height, double depth_scale,
                               double* pts_out, int64_t* n_out) {
  if (width < 1 || height < 1 || !(depth_scale > 0.0) || !pts_out || !n_out) return 2;
  const size_t np = static_cast<size_t>(width) * height;
  std::vector<uint16_t> depth(np), inten(np);
  double intr[4];
  gmmb_synthetic_frame_images(width, height, depth_scale, depth.data(), inten.data(), intr);
  const double fx = intr[0], fy = intr[1], cx = intr[2], cy = intr[3];
  // image_pair_to_cloud (ingest.cpp:27-57): row-major pixels, drop zero depth
  int64_t n = 0;
  for (uint16_t d : depth) n += d > 0;
  const double inv_scale = 1.0 / depth_scale, inv_max = 1.0 / 255.0;
  int64_t k = 0;
  for (int v = 0; v < height; ++v) {
    for (int u = 0; u < width; ++u) {
      const uint16_t d = depth[static_cast<size_t>(v) * width + u];
      if (d == 0) continue;
      const double z = d * inv_scale;
      pts_out[0 * n + k] = (u - cx) * z / fx;
      pts_out[1 * n + k] = (v - cy) * z / fy;
      pts_out[2 * n + k] = z;
      pts_out[3 * n + k] = inten[static_cast<size_t>(v) * width + u] * inv_max;
      ++k;
    }
  }
  *n_out = n;
  return 0;
}

int gmmb_structured_scene(int64_t n, uint64_t seed, double noise_sigma,
                          double* pts_out) {
  if (n < 0 || !pts_out) return 2;
  for (int64_t i = 0; i < n; ++i) {
    const auto ctr = static_cast<uint64_t>(i);
    const double u = uniform(seed, 11, ctr * 8);
    const double v = uniform(seed, 11, ctr * 8 + 1);
    double nz0, nz1, nz2, unused;
    normal_pair(seed, 12, ctr * 8 + 2, nz0, nz1);
    normal_pair(seed, 12, ctr * 8 + 4, nz2, unused);
    double p[3];
    switch (i % 3) {
      case 0:
        p[0] = 2.0 * u - 1.0; p[1] = 2.0 * v - 1.0; p[2] = 0.0;
        break;
      case 1:
        p[0] = 0.0; p[1] = 2.0 * u - 1.0; p[2] = 1.2 * v;
        break;
      default: {
        const double ang = 2.0 * M_PI * u;
        p[0] = 0.55 + 0.3 * std::cos(ang);
        p[1] = -0.35 + 0.3 * std::sin(ang);
        p[2] = 1.1 * v;
        break;
      }
    }
    p[0] += noise_sigma * nz0;
    p[1] += noise_sigma * nz1;
    p[2] += noise_sigma * nz2;
    const double in = std::clamp(
        0.5 + 0.3 * std::sin(4.0 * p[0]) + 0.2 * std::cos(3.0 * p[1] + p[2]), 0.0, 1.0);
    pts_out[0 * n + i] = p[0];
    pts_out[1 * n + i] = p[1];
    pts_out[2 * n + i] = p[2];
    pts_out[3 * n + i] = in;
  }
  return 0;
}

int gmmb_blob_cloud(const double* centers, int k, double sigma,
                    int64_t per_blob, uint64_t seed, double* pts_out) {
  if (k < 0 || per_blob < 0 || !pts_out || (k > 0 && !centers)) return 2;
  const int64_t n = static_cast<int64_t>(k) * per_blob;
  for (int64_t b = 0; b < k; ++b) {
    for (int64_t i = 0; i < per_blob; ++i) {
      const auto counter = static_cast<uint64_t>(b * per_blob + i) * 4;
      double z[4];
      normal_pair(seed, 7, counter, z[0], z[1]);
      normal_pair(seed, 7, counter + 2, z[2], z[3]);
      for (int j = 0; j < 4; ++j) {
        double v = centers[b * 4 + j] + sigma * z[j];
        if (j == 3) v = std::min(std::max(v, 0.0), 1.0);
        pts_out[j * n + b * per_blob + i] = v;
      }
    }
  }
  return 0;
}

int gmmb_jitter_cloud(double* pts, int64_t n, double sigma, uint64_t seed) {
  if (n < 0 || !pts) return 2;
  for (int64_t i = 0; i < n; ++i) {
    double z0, z1, z2, z3;
    normal_pair(seed, 13, static_cast<uint64_t>(i) * 4, z0, z1);
    normal_pair(seed, 13, static_cast<uint64_t>(i) * 4 + 2, z2, z3);
    pts[0 * n + i] += sigma * z0;
    pts[1 * n + i] += sigma * z1;
    pts[2 * n + i] += sigma * z2;
  }
  return 0;
}

}  // extern "C"
