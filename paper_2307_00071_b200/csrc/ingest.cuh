// ingest.cuh — device back-projection of a (decimated) depth/intensity pair.
#pragma once
#include "common.cuh"

namespace gmmb {

struct IngestParams {  // decimated intrinsics (ingest.cpp:16-25)
  double fx, fy, cx, cy, inv_scale, inv_max;
};
struct IngestScratch {
  int* flags;  // [wd * hd]
  int* offs;   // [wd * hd]
  void* temp;
  size_t temp_bytes;
};

size_t ingest_temp_bytes(int64_t np);
// x64 must hold 4 * wd * hd doubles; the cloud is N x 4 column-major with
// N = *n_dev (device) = non-zero depths of the decimated image.
cudaError_t launch_ingest(const uint16_t* depth, const uint16_t* inten, int width, int wd, int hd,
                          int f, IngestParams ip, IngestScratch scr, double* x64,
                          int64_t* n_dev, cudaStream_t s);

}  // namespace gmmb
