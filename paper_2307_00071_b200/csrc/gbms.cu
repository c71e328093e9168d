// gbms.cu — GBMS component estimation on the device:
// gbms_estimate_components (sogmm.cpp:22-195), the step fit(cloud,
// bandwidth) runs before kinit. The reference's kd-tree radius queries
// (kdtree.hpp) become a uniform grid of bandwidth-sized cells: a seed's
// neighbours within the bandwidth lie in the 3^4 cells around its own, found
// by binary search in the cell-sorted seed keys.
//   binning   : per-point 4 x 16-bit cell key, CUB sort (stable), run-length
//               segments -> seed = centroid summed in point order (exactly
//               the reference's std::map accumulation);
//   blurring  : flat-kernel weighted mean of the seeds within the bandwidth,
//               shift = sum w |next - seed| / total (fixed-order reduction);
//   folding   : mix64 cell keys at fold_eps, CUB sort, representative = first
//               seed of each key, weights summed in seed order, order kept;
//   merging   : single linkage at the merge radius by min-label propagation
//               (the reference's union-by-min roots), modes = weighted means
//               in seed order, mapped back to the original coordinates.
// The blur sums visit neighbours in grid order rather than kd-tree order, so
// seeds differ from the reference at the rounding level (1e-16 relative);
// fold keys (1e-8 cells) and the radius tests absorb that.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include "gbms.cuh"

namespace gmmb {

namespace {

__global__ void minmax_kernel(const double* __restrict__ x64, int64_t n, double* __restrict__ out) {
  // one block per coordinate: out[d] = min, out[4 + d] = max
  __shared__ double lo[256], hi[256];
  const int d = blockIdx.x;
  double a = INFINITY, b = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = x64[d * n + i];
    a = fmin(a, v);
    b = fmax(b, v);
  }
  lo[threadIdx.x] = a;
  hi[threadIdx.x] = b;
  __syncthreads();
  for (int off = 128; off >= 1; off >>= 1) {
    if (threadIdx.x < off) {
      lo[threadIdx.x] = fmin(lo[threadIdx.x], lo[threadIdx.x + off]);
      hi[threadIdx.x] = fmax(hi[threadIdx.x], hi[threadIdx.x + off]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[d] = lo[0];
    out[4 + d] = hi[0];
  }
}

// detail::normalize_cloud (sogmm.cpp:35-49) + the bin key (:62-68)
__global__ void bin_keys_kernel(const double* __restrict__ x64, int64_t n,
                                const double* __restrict__ mm, double bw,
                                double* __restrict__ norm, uint64_t* __restrict__ keys,
                                int32_t* __restrict__ idx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t key = 0;
  for (int d = 0; d < 4; ++d) {
    const double range = mm[4 + d] - mm[d];
    const double v = range > 0.0 ? (x64[d * n + i] - mm[d]) / range : 0.0;
    norm[i * 4 + d] = v;
    const uint64_t cell = static_cast<uint64_t>(v / bw);
    key = (key << 16) | (cell & 0xffff);
  }
  keys[i] = key;
  idx[i] = static_cast<int32_t>(i);
}

// seed = centroid of the run, summed in point order (std::map accumulation)
__global__ void seed_centroid_kernel(const double* __restrict__ norm,
                                     const int32_t* __restrict__ sidx,
                                     const int* __restrict__ counts, const int* __restrict__ offs,
                                     const int* __restrict__ nruns, double* __restrict__ seeds,
                                     double* __restrict__ weights) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= *nruns) return;
  double sum[4] = {0, 0, 0, 0};
  const int b = offs[s], c = counts[s];
  for (int q = 0; q < c; ++q) {
    const int64_t p = sidx[b + q];
    for (int d = 0; d < 4; ++d) sum[d] += norm[p * 4 + d];
  }
  for (int d = 0; d < 4; ++d) seeds[s * 4 + d] = sum[d] / c;
  weights[s] = 1.0;
}

// Grid cell key: a 64-bit hash of the four integer cell coordinates (no
// range limit, so any bandwidth works). Different cells that collide only
// share a sorted run; every visit re-checks the exact distance.
__device__ __forceinline__ uint64_t cell_hash(const int64_t (&c)[4]) {
  uint64_t key = 0x243f6a8885a308d3ULL;
  for (int d = 0; d < 4; ++d) key = mix64(key ^ static_cast<uint64_t>(c[d]));
  return key;
}
__device__ __forceinline__ uint64_t cell_key(const double* x, double cell) {
  int64_t c[4];
  for (int d = 0; d < 4; ++d) c[d] = static_cast<int64_t>(floor(x[d] / cell));
  return cell_hash(c);
}

__global__ void grid_keys_kernel(const double* __restrict__ seeds, int S, double bw,
                                 uint64_t* __restrict__ keys, int32_t* __restrict__ idx) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  keys[s] = cell_key(seeds + s * 4, bw);
  idx[s] = s;
}

__device__ __forceinline__ int lower_bound_u64(const uint64_t* k, int n, uint64_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (k[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// visit every seed j within radius r <= cell of q through the cell grid
// (the 3^4 cells around q's own); a hash collision that puts another cell's
// seeds in a visited run is filtered by the distance check (two of the 81
// neighbour cells sharing one 64-bit hash, which would visit a run twice,
// has probability ~2^-52)
template <typename V>
__device__ __forceinline__ void for_each_near(const double* q, double r, double cell,
                                              const double* __restrict__ seeds,
                                              const uint64_t* __restrict__ gk,
                                              const int32_t* __restrict__ gi, int S, V&& visit) {
  int64_t c[4];
  for (int d = 0; d < 4; ++d) c[d] = static_cast<int64_t>(floor(q[d] / cell));
  const double r2 = r * r;
  for (int nb = 0; nb < 81; ++nb) {
    int t = nb;
    int64_t cc[4];
    for (int d = 0; d < 4; ++d) {
      cc[d] = c[d] + (t % 3) - 1;
      t /= 3;
    }
    const uint64_t key = cell_hash(cc);
    for (int p = lower_bound_u64(gk, S, key); p < S && gk[p] == key; ++p) {
      const int j = gi[p];
      const double* x = seeds + j * 4;
      const double e0 = x[0] - q[0], e1 = x[1] - q[1], e2 = x[2] - q[2], e3 = x[3] - q[3];
      if (((e0 * e0 + e1 * e1) + e2 * e2) + e3 * e3 <= r2) visit(j);
    }
  }
}

// one blurring step (sogmm.cpp:92-110) + the seed's shift term
__global__ void blur_kernel(const double* __restrict__ seeds, const double* __restrict__ w, int S,
                            double bw, const uint64_t* __restrict__ gk,
                            const int32_t* __restrict__ gi, double* __restrict__ next,
                            double* __restrict__ shift_terms) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const double* q = seeds + s * 4;
  double sum[4] = {0, 0, 0, 0}, mass = 0.0;
  for_each_near(q, bw, bw, seeds, gk, gi, S, [&](int j) {
    for (int d = 0; d < 4; ++d) sum[d] += w[j] * seeds[j * 4 + d];
    mass += w[j];
  });
  double e2 = 0.0;
  for (int d = 0; d < 4; ++d) {
    next[s * 4 + d] = sum[d] / mass;
    const double e = next[s * 4 + d] - q[d];
    e2 += e * e;
  }
  shift_terms[s] = w[s] * sqrt(e2);
}

__global__ void sum_kernel(const double* __restrict__ v, int n, double* __restrict__ out) {
  __shared__ double red[1024];
  double a = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a += v[i];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int off = 512; off >= 1; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void fold_keys_kernel(const double* __restrict__ seeds, int S, double eps,
                                 uint64_t* __restrict__ keys, int32_t* __restrict__ idx) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  uint64_t key = 0;
  for (int d = 0; d < 4; ++d) {
    const uint64_t cell = static_cast<uint64_t>((seeds[s * 4 + d] + 1.0) / eps);
    key = mix64(key ^ cell);
  }
  keys[s] = key;
  idx[s] = s;
}

// per fold run: representative = first (lowest) seed index, weights summed in seed order
__global__ void fold_runs_kernel(const int32_t* __restrict__ sidx, const int* __restrict__ counts,
                                 const int* __restrict__ offs, const int* __restrict__ nruns,
                                 const double* __restrict__ w, int32_t* __restrict__ rep,
                                 double* __restrict__ rw) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= *nruns) return;
  const int b = offs[r], c = counts[r];
  double a = 0.0;
  for (int q = 0; q < c; ++q) a += w[sidx[b + q]];
  rep[r] = sidx[b];
  rw[r] = a;
}

__global__ void gather_seeds_kernel(const double* __restrict__ seeds, const int32_t* __restrict__ rep,
                                    int R, double* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  for (int d = 0; d < 4; ++d) out[r * 4 + d] = seeds[rep[r] * 4 + d];
}

__global__ void iota_kernel32(int32_t* __restrict__ v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

// single linkage: min-label propagation + pointer jumping
__global__ void link_kernel(const double* __restrict__ seeds, int S, double r, double bw,
                            const uint64_t* __restrict__ gk, const int32_t* __restrict__ gi,
                            int32_t* __restrict__ label, int* __restrict__ changed) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  int m = label[s];
  for_each_near(seeds + s * 4, r, bw, seeds, gk, gi, S, [&](int j) { m = min(m, label[j]); });
  m = min(m, label[m]);
  if (m < label[s]) {
    atomicMin(&label[s], m);
    *changed = 1;
  }
}

// modes: one thread per component (root = lowest seed index), members in seed order
__global__ void modes_kernel(const int32_t* __restrict__ sidx, const int* __restrict__ counts,
                             const int* __restrict__ offs, const int* __restrict__ nruns,
                             const double* __restrict__ seeds, const double* __restrict__ w,
                             const double* __restrict__ mm, double* __restrict__ modes) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= *nruns) return;
  const int b = offs[r], c = counts[r];
  double sum[4] = {0, 0, 0, 0}, mass = 0.0;
  for (int q = 0; q < c; ++q) {
    const int s = sidx[b + q];
    for (int d = 0; d < 4; ++d) sum[d] += w[s] * seeds[s * 4 + d];
    mass += w[s];
  }
  for (int d = 0; d < 4; ++d) {
    const double y = sum[d] / mass;
    const double range = mm[4 + d] - mm[d];
    modes[r * 4 + d] = range > 0.0 ? y * range + mm[d] : mm[d];
  }
}

}  // namespace

size_t gbms_temp_bytes(int64_t n) {
  size_t a = 0, b = 0, c = 0, d = 0, e = 0;
  const int ni = static_cast<int>(n);
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, ni);
  cub::DeviceRunLengthEncode::Encode(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                     (int*)nullptr, (int*)nullptr, ni);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (const int*)nullptr, (int*)nullptr, ni);
  cub::DeviceRadixSort::SortPairs(nullptr, d, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const double*)nullptr, (double*)nullptr, ni);
  cub::DeviceRunLengthEncode::Encode(nullptr, e, (const int32_t*)nullptr, (int32_t*)nullptr,
                                     (int*)nullptr, (int*)nullptr, ni);
  return std::max(std::max(std::max(a, b), std::max(c, d)), e);
}

#define GB_CK(x)                          \
  do {                                    \
    cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) return e_;     \
  } while (0)

static int blocks(int64_t n, int t = 256) { return static_cast<int>((n + t - 1) / t); }

// sorted runs of keys[0, n): counts, offsets, run count (device)
static cudaError_t runs_u64(GbmsScratch& g, const uint64_t* keys_sorted, int n, int* counts,
                            int* offs, int* nruns, cudaStream_t s) {
  size_t bytes = g.temp_bytes;
  GB_CK(cub::DeviceRunLengthEncode::Encode(g.temp, bytes, keys_sorted, g.ukeys, counts, nruns, n,
                                           s));
  bytes = g.temp_bytes;
  return cub::DeviceScan::ExclusiveSum(g.temp, bytes, counts, offs, n, s);
}

cudaError_t gbms_run(const double* x64, int64_t n, GbmsParamsDev prm, GbmsScratch g,
                     GbmsResultHost* res, cudaStream_t s) {
  const int ni = static_cast<int>(n);
  minmax_kernel<<<4, 256, 0, s>>>(x64, n, g.mm);
  bin_keys_kernel<<<blocks(n), 256, 0, s>>>(x64, n, g.mm, prm.bandwidth, g.norm, g.k0, g.i0);
  size_t bytes = g.temp_bytes;
  GB_CK(cub::DeviceRadixSort::SortPairs(g.temp, bytes, g.k0, g.k1, g.i0, g.i1, ni, 0, 64, s));
  GB_CK(runs_u64(g, g.k1, ni, g.counts, g.offs, g.nruns, s));
  int S = 0;
  GB_CK(cudaMemcpyAsync(&S, g.nruns, sizeof(int), cudaMemcpyDeviceToHost, s));
  GB_CK(cudaStreamSynchronize(s));
  seed_centroid_kernel<<<blocks(S), 256, 0, s>>>(g.norm, g.i1, g.counts, g.offs, g.nruns, g.seeds,
                                                 g.w);
  res->seeds0 = S;
  const double total_weight = static_cast<double>(S);  // weights start at one
  const double fold_eps = fmax(1e-12, prm.tol * 1e-3);
  int iterations = 0;
  for (int iter = 0; iter < prm.max_iters; ++iter) {
    ++iterations;
    grid_keys_kernel<<<blocks(S), 256, 0, s>>>(g.seeds, S, prm.bandwidth, g.k0, g.i0);
    bytes = g.temp_bytes;
    GB_CK(cub::DeviceRadixSort::SortPairs(g.temp, bytes, g.k0, g.k1, g.i0, g.i1, S, 0, 64, s));
    blur_kernel<<<blocks(S), 256, 0, s>>>(g.seeds, g.w, S, prm.bandwidth, g.k1, g.i1, g.next,
                                          g.terms);
    sum_kernel<<<1, 1024, 0, s>>>(g.terms, S, g.scal);
    std::swap(g.seeds, g.next);
    // fold coincident seeds (sogmm.cpp:121-143)
    fold_keys_kernel<<<blocks(S), 256, 0, s>>>(g.seeds, S, fold_eps, g.k0, g.i0);
    bytes = g.temp_bytes;
    GB_CK(cub::DeviceRadixSort::SortPairs(g.temp, bytes, g.k0, g.k1, g.i0, g.i1, S, 0, 64, s));
    GB_CK(runs_u64(g, g.k1, S, g.counts, g.offs, g.nruns, s));
    fold_runs_kernel<<<blocks(S), 256, 0, s>>>(g.i1, g.counts, g.offs, g.nruns, g.w, g.i0, g.terms);
    int R = 0;
    double shift = 0.0;
    GB_CK(cudaMemcpyAsync(&R, g.nruns, sizeof(int), cudaMemcpyDeviceToHost, s));
    GB_CK(cudaMemcpyAsync(&shift, g.scal, sizeof(double), cudaMemcpyDeviceToHost, s));
    GB_CK(cudaStreamSynchronize(s));
    shift /= total_weight;
    if (R < S) {
      // keep first-occurrence order: sort the representatives by index
      bytes = g.temp_bytes;
      GB_CK(cub::DeviceRadixSort::SortPairs(g.temp, bytes, g.i0, g.i1, g.terms, g.w2, R, 0, 32, s));
      gather_seeds_kernel<<<blocks(R), 256, 0, s>>>(g.seeds, g.i1, R, g.next);
      std::swap(g.seeds, g.next);
      std::swap(g.w, g.w2);
      S = R;
    }
    if (shift < prm.tol) break;
  }
  // single-linkage merge (sogmm.cpp:148-168): cells at least as wide as the
  // merge radius, so the 3^4 neighbourhood covers every link
  const double mcell = fmax(prm.bandwidth, prm.merge_radius);
  grid_keys_kernel<<<blocks(S), 256, 0, s>>>(g.seeds, S, mcell, g.k0, g.i0);
  bytes = g.temp_bytes;
  GB_CK(cub::DeviceRadixSort::SortPairs(g.temp, bytes, g.k0, g.k1, g.i0, g.i1, S, 0, 64, s));
  int32_t* label = g.i2;
  iota_kernel32<<<blocks(S), 256, 0, s>>>(label, S);
  for (int pass = 0; pass < S + 1; ++pass) {
    GB_CK(cudaMemsetAsync(g.flag, 0, sizeof(int), s));
    link_kernel<<<blocks(S), 256, 0, s>>>(g.seeds, S, prm.merge_radius, mcell, g.k1, g.i1,
                                          label, g.flag);
    int changed = 0;
    GB_CK(cudaMemcpyAsync(&changed, g.flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    GB_CK(cudaStreamSynchronize(s));
    if (!changed) break;
  }
  // modes: components ordered by root (lowest seed index), members in seed order
  iota_kernel32<<<blocks(S), 256, 0, s>>>(g.i0, S);
  bytes = g.temp_bytes;
  GB_CK(cub::DeviceRadixSort::SortPairs(g.temp, bytes, label, g.i3, g.i0, g.i1, S, 0, 32, s));
  bytes = g.temp_bytes;
  GB_CK(cub::DeviceRunLengthEncode::Encode(g.temp, bytes, g.i3, g.i0, g.counts, g.nruns, S, s));
  bytes = g.temp_bytes;
  GB_CK(cub::DeviceScan::ExclusiveSum(g.temp, bytes, g.counts, g.offs, S, s));
  modes_kernel<<<blocks(S), 256, 0, s>>>(g.i1, g.counts, g.offs, g.nruns, g.seeds, g.w, g.mm,
                                         g.modes);
  int C = 0;
  GB_CK(cudaMemcpyAsync(&C, g.nruns, sizeof(int), cudaMemcpyDeviceToHost, s));
  GB_CK(cudaStreamSynchronize(s));
  res->components = C;
  res->iterations = iterations;
  return cudaGetLastError();
}

}  // namespace gmmb
