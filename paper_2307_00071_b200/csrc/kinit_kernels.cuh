// kinit_kernels.cuh — k-means++ seeding + nearest-centre labels on sm_100a.
#pragma once
#include "common.cuh"

namespace gmmb {

// One candidate per CTA per round, published with a round tag (64 B).
struct __align__(64) KppSlot {
  double clock;         // exact FP64 clock of the CTA's best candidate
  long long idx;        // its global index, -1 if none eligible
  long long unchosen;   // lowest unchosen global index in the CTA
  int tag;              // round + 1 once valid
  int owner;            // grid thread id owning idx (or -1)
  double cx[4];         // coordinates of idx
};

struct KinitScratch {
  uint64_t* keys;     // [n]  key * golden (pre-multiplied hash counter)
  double* d2;         // [n]  (memory-resident variant / sharded)
  int32_t* labels;    // [n]
  unsigned char* chosen;  // [n] (memory-resident variant / sharded)
  KppSlot* slots;     // [2][max_blocks]
  int* owned;         // [k]
  long long* centers; // [k]
  int* status;        // [4]
  unsigned* counter;  // [2] grid-barrier arrival counter, max |coordinate| (zeroed per launch)
  // memory-resident rounds: FP32 coordinates, fold-prefilter thresholds, 1/d2
  float4* xf;         // [n]
  float* tp;          // [n]
  float* inv;         // [n]
};

// Keys (sogmm.cpp:210-213): key_i = hash of the 4 doubles starting at x_i in
// the column-major N x 4 buffer (the reference's pts.row(i).data() quirk).
// Stored pre-multiplied by the golden ratio constant (rng.hpp:26).
// tail[0..2] = the 3 doubles that follow x_{n-1} in the (global) buffer:
// x64 + n (the y column) on one device; the next shard's x or the global y
// column when the cloud is sharded.
cudaError_t launch_keys(const double* x64, int64_t n, const double* tail,
                        uint64_t* keys, cudaStream_t s);

// Persistent k-means++ seeding for one device holding all points
// (sogmm.cpp:224-287), followed by the final centre fold that yields the
// nearest-centre labels (:290-312) and owned counts. Cooperative launch.
cudaError_t launch_kpp_seed(const double* x64, int64_t n, int d, int k, uint64_t seed,
                            KinitScratch scr, int sm_count, cudaStream_t s);

// Tile-pruned seeding for clouds beyond the shared-memory-resident kernel
// (kinit_tile.cu): Morton-order copies of the points / keys / state and
// per-tile FP64 boxes, largest d2 and d2 sums (ntiles = layout tiles).
struct KppTileScratch {
  double* xm;           // [4][n] FP64 coordinates, Morton order
  uint64_t* mkey;       // [n]
  double* md2;          // [n]
  int32_t* mlab;        // [n]
  const int32_t* perm;  // [n] Morton position -> original index
  double* tbox;         // [ntiles][8] lo[4], hi[4]
  double* tdmax;        // [ntiles]
  double* tsum;         // [ntiles]
};
bool kpp_tile_wanted(int64_t n, int sm_count);

// keys must be computed; owned[] zeroed; labels (original order), owned and
// centres are written (the fix-up follows).
cudaError_t launch_kpp_tile(const double* x64, int64_t n, int ntiles, const int32_t* perm,
                            int k, uint64_t seed, KinitScratch scr, KppTileScratch ts,
                            int sm_count, cudaStream_t s);

// Owned fix-up (sogmm.cpp:315-331), single CTA, no-op when nothing is empty.
cudaError_t launch_fixup(int64_t n, int k, KinitScratch scr, cudaStream_t s);

// ---- sharded (multi-rank) seeding: one kernel per round + allgather ----
// Each rank holds points [offset, offset + n) of the global cloud.
struct __align__(64) KppRankSlot {
  double clock;
  long long idx;        // global index, -1 if none eligible
  long long unchosen;   // lowest unchosen global index
  double x[4];          // coordinates of idx (if >= 0)
  double ux[4];         // coordinates of unchosen (if valid)
};
cudaError_t launch_kpp_round(const double* x64, int64_t n, int64_t offset,
                             int r, uint64_t seed, const KppRankSlot* prev,
                             int world, KinitScratch scr, KppRankSlot* out,
                             int* ticket, int sm_count, cudaStream_t s);
// final fold of centre k-1 (from prev slots) + labels + owned counts
cudaError_t launch_kpp_final(const double* x64, int64_t n, int64_t offset,
                             int k, const KppRankSlot* prev, int world,
                             KinitScratch scr, cudaStream_t s);

// sharded fix-up: *out = lowest global index i with labels[i - offset] ==
// donor on this shard, LLONG_MAX if none
cudaError_t launch_first_label(int64_t n, int64_t offset, KinitScratch scr, int donor,
                               long long* out, cudaStream_t s);

}  // namespace gmmb
