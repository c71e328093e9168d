// gbms.cuh — GBMS component estimation on the device.
#pragma once
#include "common.cuh"

namespace gmmb {

struct GbmsParamsDev {
  double bandwidth, tol, merge_radius;
  int max_iters;
};
struct GbmsResultHost {
  int components, iterations, seeds0;
};
// device scratch, all sized for n points (seeds never exceed n)
struct GbmsScratch {
  double* mm;      // [8] mins, maxs
  double* norm;    // [n][4]
  double* seeds;   // [n][4]
  double* next;    // [n][4]
  double* w;       // [n]
  double* w2;      // [n]
  double* terms;   // [n]
  double* scal;    // [1]
  double* modes;   // [n][4]
  uint64_t *k0, *k1, *ukeys;  // [n]
  int32_t *i0, *i1, *i2, *i3; // [n]
  int *counts, *offs;         // [n]
  int* nruns;                 // [1]
  int* flag;                  // [1]
  void* temp;
  size_t temp_bytes;
};

size_t gbms_temp_bytes(int64_t n);
// Runs GBMS on the N x 4 column-major cloud; modes land in scratch.modes
// (components x 4 row-major, original coordinates).
cudaError_t gbms_run(const double* x64, int64_t n, GbmsParamsDev prm, GbmsScratch g,
                     GbmsResultHost* res, cudaStream_t s);

}  // namespace gmmb
