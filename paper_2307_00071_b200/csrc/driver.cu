// driver.cu — host driver + extern "C" ABI (include/gmmb.h).
//
// One context = one CUDA device + stream + grow-only device buffers. The
// fit path mirrors gmmscape::fit with K given (sogmm.cpp:477-509):
//   upload (validate + layout) -> kinit (keys, k-means++, fix-up)
//   -> initial M step from labels -> EM loop on the device.
// The EM loop runs in chunks of iterations enqueued back to back; each
// iteration is [fused E+stats] -> [ordered reduce] -> (NCCL allreduce when
// sharded) -> [per-component finalize] -> [commit]. Convergence is decided on
// the device (commit kernel); the host reads the 64-byte state once per
// chunk to stop enqueuing.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gmmb.h"
#include "em_kernels.cuh"
#include "kinit_kernels.cuh"
#include "layout.cuh"
#include "mstep_hard.cuh"
#include "inference.cuh"
#include "ingest.cuh"
#include "gbms.cuh"
#include "comm.cuh"

using namespace gmmb;

// NVTX ranges around the fit's stages (header-only nvtx3: free without a
// profiler; visible in Nsight Systems / ncu --nvtx)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace {

thread_local std::string g_err;

struct Err {
  int code;
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Err{1, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  void ensure(size_t count) {
    if (count <= cap && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t c = std::max<size_t>(count, 1);
    ck(cudaMalloc(&p, c * sizeof(T)), "cudaMalloc");
    cap = c;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Shape + buffer identity of a built EM graph (rebuild when any differs).
struct EmGraphKey {
  int k0, d, world, sparse;
  int64_t n;
  const void* p[32];
  bool operator==(const EmGraphKey& o) const {
    if (k0 != o.k0 || d != o.d || n != o.n || world != o.world || sparse != o.sparse) return false;
    for (int i = 0; i < 32; ++i)
      if (p[i] != o.p[i]) return false;
    return true;
  }
};

}  // namespace

struct gmmb_ctx {
  int device = 0;
  int sm_count = 148;
  int cc_major = 0, cc_minor = 0;
  cudaStream_t s = nullptr;
  cudaStream_t s_copy = nullptr;  // batch fits: next frame's H2D alongside this frame's fit
  cudaEvent_t ev_copy = nullptr;
  cudaEvent_t ev[8] = {};
  std::vector<cudaEvent_t> ev_e;  // [2*i], [2*i+1] bracket the E kernel of iteration i
  long long launches = 0;         // kernels of this library enqueued by the current call
  // sharding
  int rank = 0, world = 1;
  Comm* comm = nullptr;            // world > 1: NCCL or virtual ranks (comm.cuh)
  // resident cloud
  int64_t n = 0, offset = 0, n_global = 0;
  int d = 0;
  bool have_cloud = false;
  DevBuf<double> x64;
  DevBuf<double> x64_next;        // batch fits: the prefetched next frame
  DevBuf<float4> xt;
  DevBuf<double> tc;
  DevBuf<int32_t> perm;
  DevBuf<double> bbox_part;
  DevBuf<uint64_t> mkeys_in, mkeys_out;
  DevBuf<int32_t> midx;
  DevBuf<unsigned char> sort_tmp;
  DevBuf<int32_t> hidx;           // hard M step: [3][n] sort indices / keys
  // inference (score / sample / conditional / e_step API)
  DevBuf<double> iw, imu, icov, ifac, ilow, iout, iout2;
  DevBuf<int> ierr;
  DevBuf<uint16_t> img;        // ingest: depth + intensity images
  DevBuf<int> iflags;          // ingest: flags + offsets
  DevBuf<int64_t> in_n;
  DevBuf<unsigned char> gb;    // GBMS scratch (one allocation)
  DevBuf<int> flags;
  // kinit
  DevBuf<uint64_t> keys;
  DevBuf<double> kd2;
  DevBuf<int32_t> labels;
  DevBuf<unsigned char> chosen;
  DevBuf<float4> kxf;
  DevBuf<float> ktp, kinv;
  DevBuf<KppSlot> slots;
  DevBuf<int> owned;
  DevBuf<long long> centers;
  DevBuf<KppRankSlot> rslots;  // [world] gathered + [1] own
  DevBuf<int> ticket;
  DevBuf<int> kstatus;
  DevBuf<long long> ll64;      // sharded fix-up scratch
  int kinit_tile = 1;          // 1: tile-pruned seeding past the resident kernel (GMMB_KINIT=mem: off)
  int kinit_gather = 1;        // sharded: gather the cloud and seed it whole (GMMB_KINIT_SHARDED=rounds: 0)
  DevBuf<double> kgather;
  DevBuf<double> kt_xm, kt_d2, kt_tile;
  DevBuf<uint64_t> kt_key;
  DevBuf<int32_t> kt_lab;
  // model
  DevBuf<double> mw[2], mmu[2], mcov[2];
  DevBuf<CompConst> mcst[2];
  DevBuf<double> rcount, rmean, rcov, rlogdet;
  DevBuf<float> rpc;
  DevBuf<int> rflags, rmap;
  DevBuf<double> mpart, msums, mmeans, mcounts;
  DevBuf<double> partials, ll_part, red, ll_trace;
  DevBuf<float> chunkf;          // chunked E step (K > 512): per-chunk sums + normalisers
  DevBuf<int> chunki;            // ... exact-path point list + count
  ChunkScratch chunk{};
  // exact-zero-pruned E step (estep_sparse.cu)
  int estep_mode = 0;             // 0: pruned when supported, 1: dense kernels
  bool sparse_on = false;         // the current EM run uses the pruned E step
  int pool_mult = 1;              // pool growth after an overflow
  int sp_nosplit = 0;             // this EM run's retry without heavy-unit splits
  DevBuf<double> sp_bc, sp_pool, sp_ll;
  DevBuf<float4> sp_bh, sp_brec;
  DevBuf<int> sp_blist, sp_bcnt, sp_ctl, sp_toff, sp_heavy;
  DevBuf<unsigned> sp_done;
  DevBuf<unsigned> sp_mask;
  DevBuf<unsigned short> sp_pre;
  SparseScratch sparse{};
  double units_eval = 0.0;        // units evaluated by the last EM run (pruned E step)
  DevBuf<EmState> st_bak;         // EM-start snapshot (pool overflow re-run)
  DevBuf<double> bak_w[2], bak_mu[2], bak_cov[2];
  DevBuf<CompConst> bak_cst[2];
  DevBuf<double> dense;  // log_gamma staging for m_step / e_step
  DevBuf<EmState> st;
  EmState* st_host = nullptr;  // pinned
  int timing = 0;                // 1: chunked EM loop with per-iteration E-kernel events
  bool last_timed = false;       // the last EM run recorded those events
  cudaGraphExec_t em_graph = nullptr;
  EmGraphKey em_key{};
  ModelBuf bufs[2];
  RecBuf rec;
};

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Err& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// guarded() for calls that may run collectives: a failure on this rank
// aborts a virtual group so that its peers do not wait forever
template <typename F>
int guarded_coll(gmmb_ctx* c, F&& f) {
  const int rc = guarded(f);
  if (rc != 0 && c && c->comm) c->comm->abort();
  return rc;
}

void set_device(gmmb_ctx* c) { ck(cudaSetDevice(c->device), "cudaSetDevice"); }

// Copies ordered on the context's (non-blocking) stream: a plain cudaMemcpy
// runs on the legacy stream, which does not wait for work on c->s.
void copy_sync(gmmb_ctx* c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  ck(cudaMemcpyAsync(dst, src, bytes, kind, c->s), "cudaMemcpyAsync");
  ck(cudaStreamSynchronize(c->s), "cudaStreamSynchronize");
}

void check_d(int d) {
  if (d != 3 && d != 4) throw Err{2, "dimension must be 3 (xyz) or 4 (xyz+intensity)"};
}

void check_em(const gmmb_em_params* em) {
  // sogmm.cpp:468-470 (ll_rel_tol = 0 allowed: fixed iteration count)
  if (!em || em->max_iters < 1 || !(em->ll_rel_tol >= 0.0)) {
    throw Err{2, "bad EM parameters"};
  }
  if (em->cov_reg < 0.0) throw Err{2, "cov_reg must be >= 0"};
}

// ---- device allocation ----------------------------------------------------
void ensure_model(gmmb_ctx* c, int k) {
  const size_t kc = std::max(k, 32);
  for (int b = 0; b < 2; ++b) {
    c->mw[b].ensure(kc);
    c->mmu[b].ensure(kc * 4);
    c->mcov[b].ensure(kc * 10);
    c->mcst[b].ensure(kc);
    c->bufs[b] = ModelBuf{c->mw[b].p, c->mmu[b].p, c->mcov[b].p, c->mcst[b].p};
  }
  c->rcount.ensure(kc);
  c->rmean.ensure(kc * 4);
  c->rcov.ensure(kc * 10);
  c->rlogdet.ensure(kc);
  c->rpc.ensure(kc * 16);
  c->rflags.ensure(kc);
  c->rmap.ensure(kc);
  c->rec = RecBuf{c->rcount.p, c->rmean.p, c->rcov.p, c->rlogdet.p, c->rpc.p, c->rflags.p,
                  c->rmap.p};
  c->red.ensure(kc * 16 + 1);
  c->st.ensure(1);
}

void reset_state(gmmb_ctx* c, int k, const gmmb_em_params* em, int removed0) {
  EmState h{};
  h.iter = 0;
  h.done = 0;
  h.k_cur = k;
  h.cur = 0;
  h.removed = removed0;
  h.error = 0;
  h.error_index = std::numeric_limits<int>::max();
  h.error_kind = 0;
  h.ll_prev = -INFINITY;
  h.ll = -INFINITY;
  h.converged = 0;
  h.max_iters = em ? em->max_iters : 1;
  h.tol = em ? em->ll_rel_tol : 0.0;
  h.cov_reg = em ? em->cov_reg : 0.0;
  h.npts = static_cast<double>(c->n_global);
  h.units = 0.0;
  ck(cudaMemcpyAsync(c->st.p, &h, sizeof(h), cudaMemcpyHostToDevice, c->s), "state H2D");
}

EmState read_state(gmmb_ctx* c) {
  ck(cudaMemcpyAsync(c->st_host, c->st.p, sizeof(EmState), cudaMemcpyDeviceToHost, c->s),
     "state D2H");
  ck(cudaStreamSynchronize(c->s), "stream sync");
  return *c->st_host;
}

void raise_state_error(const EmState& h) {
  if (!h.error) return;
  switch (h.error_kind) {
    case 1:
      throw Err{3, "m_step: component " + std::to_string(h.error_index) +
                       " covariance not positive definite after regularization"};
    case 2:
      throw Err{3, "m_step: all components degenerate"};
    case 3:
      throw Err{3, "cholesky failed: block " + std::to_string(h.error_index) +
                       " is not positive definite"};
    default:
      throw Err{3, "numerical error"};
  }
}

// Collectives of a sharded context (comm.cuh): NCCL or in-process virtual
// ranks.
void coll(gmmb_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  throw Err{1, std::string(what) + ": " + c->comm->last_error()};
}

void allreduce_sum(gmmb_ctx* c, double* p, int64_t count) {
  if (c->world <= 1) return;
  coll(c, c->comm->allreduce(p, static_cast<size_t>(count), DType::kF64, RedOp::kSum, c->s),
       "allreduce (statistics)");
}

void moments_allreduce_cb(double* p, int64_t count, void* ctx) {
  allreduce_sum(static_cast<gmmb_ctx*>(ctx), p, count);
}

// ---- upload + layout ------------------------------------------------------
void upload(gmmb_ctx* c, const double* pts, int64_t n, int d, int64_t offset,
            int64_t n_global) {
  check_d(d);
  if (n < 1) throw Err{3, "point cloud is empty"};
  if (!pts) throw Err{2, "null point buffer"};
  if (n > (int64_t{1} << 31) - 1) throw Err{2, "too many points for one device"};
  set_device(c);
  c->x64.ensure(static_cast<size_t>(n) * 4 + 4);
  // column-major D columns; D = 3 gets an all-zero intensity column so the
  // 4D key quirk (sogmm.cpp:212) sees exactly the embedded cloud
  ck(cudaMemcpyAsync(c->x64.p, pts, sizeof(double) * n * d, cudaMemcpyHostToDevice, c->s),
     "points H2D");
  if (d == 3) ck(cudaMemsetAsync(c->x64.p + 3 * n, 0, sizeof(double) * n, c->s), "memset");
  c->n = n;
  c->d = d;
  c->offset = offset;
  c->n_global = n_global;
  c->have_cloud = true;
}

void validate(gmmb_ctx* c) {
  c->flags.ensure(4);
  ck(cudaMemsetAsync(c->flags.p, 0, sizeof(int) * 4, c->s), "memset");
  ck(launch_validate(c->x64.p, c->n, c->d, c->flags.p, c->s), "validate");
}

void layout(gmmb_ctx* c) {
  NvtxRange nv("gmmb.layout");
  const int64_t n = c->n;
  validate(c);
  const int ntiles = static_cast<int>((n + kTile - 1) / kTile);
  c->xt.ensure(static_cast<size_t>(ntiles) * kTile);
  c->tc.ensure(static_cast<size_t>(ntiles) * 4);
  c->perm.ensure(n);
  c->bbox_part.ensure(kBboxParts * 6);
  c->mkeys_in.ensure(n);
  c->mkeys_out.ensure(n);
  c->midx.ensure(n);
  const size_t tb = layout_sort_temp_bytes(n);
  c->sort_tmp.ensure(tb);
  LayoutScratch ls{c->bbox_part.p, c->mkeys_in.p, c->mkeys_out.p, c->midx.p,
                   c->sort_tmp.p, c->sort_tmp.cap};
  ck(launch_layout(c->x64.p, n, ls, c->xt.p, c->tc.p, c->perm.p, c->sm_count, c->s),
     "layout");
  c->launches += 4;  // bbox, morton, tile + validate (CUB's sort kernels not counted)
  // static culling-block boxes of the pruned E step
  const int nblk = sparse_blocks(ntiles);
  c->sp_bc.ensure(static_cast<size_t>(nblk) * 4);
  c->sp_bh.ensure(nblk);
  c->sparse.bc = c->sp_bc.p;
  c->sparse.bh = c->sp_bh.p;
  PointsDev pts{n, c->d, c->x64.p, c->xt.p, c->tc.p, ntiles};
  ck(launch_sparse_layout(pts, c->sparse, c->s), "block boxes");
  c->launches += 1;
}

void check_cloud_flags(gmmb_ctx* c) {
  int f[4];
  ck(cudaMemcpyAsync(f, c->flags.p, sizeof(f), cudaMemcpyDeviceToHost, c->s), "flags D2H");
  ck(cudaStreamSynchronize(c->s), "sync");
  if (c->world > 1) {
    // PointCloud4D::validate over the whole (sharded) cloud: every rank
    // reports the same error
    int v[2] = {(f[0] & 1) ? 1 : 0, (f[0] & 2) ? 1 : 0};
    c->kstatus.ensure(8);
    copy_sync(c, c->kstatus.p + 6, v, sizeof(v), cudaMemcpyHostToDevice);
    coll(c, c->comm->allreduce(c->kstatus.p + 6, 2, DType::kI32, RedOp::kSum, c->s),
         "allreduce (cloud flags)");
    copy_sync(c, v, c->kstatus.p + 6, sizeof(v), cudaMemcpyDeviceToHost);
    f[0] = (v[0] ? 1 : 0) | (v[1] ? 2 : 0);
  }
  if (f[0] & 1) throw Err{3, "point cloud contains non-finite values"};
  if (f[0] & 2) throw Err{3, "intensity outside [0, 1]"};
}

// ---- kinit ----------------------------------------------------------------
KinitScratch kinit_scratch(gmmb_ctx* c, int k) {
  const int64_t n = c->n;
  c->keys.ensure(n + 4);
  c->kd2.ensure(n);
  c->labels.ensure(n);
  c->chosen.ensure(n);
  // persistent kernel: LL words + fallback slots; memory-resident rounds:
  // one slot per CTA (n / 8192 CTAs beyond 4 per SM)
  c->slots.ensure(std::max<size_t>(static_cast<size_t>(c->sm_count) * 8 * 2,
                                   static_cast<size_t>(n / 8192 + 1)));
  c->owned.ensure(std::max(k, 1));
  c->centers.ensure(std::max(k, 1));
  c->kstatus.ensure(8);
  c->kxf.ensure(n);
  c->ktp.ensure(n);
  c->kinv.ensure(n);
  return KinitScratch{c->keys.p, c->kd2.p, c->labels.p, c->chosen.p,
                      c->slots.p, c->owned.p, c->centers.p, c->kstatus.p,
                      reinterpret_cast<unsigned*>(c->kstatus.p + 4), c->kxf.p, c->ktp.p,
                      c->kinv.p};
}

void run_kinit(gmmb_ctx* c, int k, uint64_t seed) {
  NvtxRange nv("gmmb.kinit");
  const int64_t n = c->n;
  KinitScratch ks = kinit_scratch(c, k);
  ck(cudaMemsetAsync(c->owned.p, 0, sizeof(int) * k, c->s), "memset");
  if (c->world == 1 && c->kinit_tile && (c->kinit_tile == 2 || kpp_tile_wanted(n, c->sm_count))) {
    // beyond the shared-memory-resident kernel: tile-pruned rounds over the
    // layout's Morton tiles (kinit_tile.cu)
    const int ntiles = static_cast<int>((n + kTile - 1) / kTile);
    c->kt_xm.ensure(static_cast<size_t>(n) * 4);
    c->kt_key.ensure(n);
    c->kt_d2.ensure(n);
    c->kt_lab.ensure(n);
    c->kt_tile.ensure(static_cast<size_t>(ntiles) * 10);
    KppTileScratch ts{c->kt_xm.p, c->kt_key.p, c->kt_d2.p, c->kt_lab.p, c->perm.p, c->kt_tile.p,
                      c->kt_tile.p + static_cast<size_t>(ntiles) * 8,
                      c->kt_tile.p + static_cast<size_t>(ntiles) * 9};
    ck(launch_keys(c->x64.p, n, c->x64.p + n, c->keys.p, c->s), "keys");
    ck(cudaMemsetAsync(c->kstatus.p, 0, sizeof(int) * 8, c->s), "memset");
    ck(launch_kpp_tile(c->x64.p, n, ntiles, c->perm.p, k, seed, ks, ts, c->sm_count, c->s),
       "kpp_tile");
    ck(launch_fixup(n, k, ks, c->s), "fixup");
    c->launches += 6;  // keys, init, boxes, rounds (persistent), scatter, fixup
    if (getenv("GMMB_DEBUG")) {
      unsigned long long xc[2] = {0, 0};
      copy_sync(c, xc, c->kstatus.p + 2, sizeof(xc), cudaMemcpyDeviceToHost);
      fprintf(stderr, "gmmb: kpp_tile n=%lld k=%d: %llu grid exchanges, %llu exact clocks\n",
              static_cast<long long>(n), k, xc[0], xc[1]);
    }
    return;
  }
  if (c->world == 1) {
    ck(launch_keys(c->x64.p, n, c->x64.p + n, c->keys.p, c->s), "keys");
    ck(cudaMemsetAsync(c->kstatus.p, 0, sizeof(int) * 8, c->s), "memset");
    // LL exchange words carry round tags: start from all-zero tags
    ck(cudaMemsetAsync(c->slots.p, 0, sizeof(KppSlot) * c->slots.cap, c->s), "memset");
    ck(launch_kpp_seed(c->x64.p, n, c->d, k, seed, ks, c->sm_count, c->s), "kpp_seed");
    ck(launch_fixup(n, k, ks, c->s), "fixup");
    c->launches += 3;  // keys, seed (persistent), fixup
    return;
  }
  if (c->world > 1 && c->kinit_gather) {
    // Sharded clouds: k-means++ is K strictly sequential rounds, so a
    // per-round collective (the path below) costs K network round trips
    // (cfg4: 2048). Instead every rank gathers the whole cloud once (one
    // all-gather, 128 MB for cfg4 over NVLink), seeds it exactly like one
    // device would (identical centres and labels on every rank, no
    // collective per round) and keeps the labels of its own shard.
    const int W = c->world;
    const int64_t N = c->n_global;
    c->ll64.ensure(static_cast<size_t>(2 * W) + 2);
    long long ext[2] = {static_cast<long long>(c->offset), static_cast<long long>(n)};
    long long* dext = c->ll64.p + 2 * W;
    copy_sync(c, dext, ext, sizeof(ext), cudaMemcpyHostToDevice);
    coll(c, c->comm->allgather(dext, c->ll64.p, sizeof(ext), c->s), "allgather (shard extents)");
    std::vector<long long> all(static_cast<size_t>(2 * W));
    copy_sync(c, all.data(), c->ll64.p, sizeof(long long) * 2 * W, cudaMemcpyDeviceToHost);
    long long max_n = 0, tot = 0;
    for (int r = 0; r < W; ++r) {
      max_n = std::max(max_n, all[2 * r + 1]);
      tot += all[2 * r + 1];
    }
    if (tot != N) throw Err{2, "bad shard layout"};
    c->dense.ensure(static_cast<size_t>(4) * max_n);
    c->kgather.ensure(static_cast<size_t>(4) * max_n * W);
    for (int j = 0; j < 4; ++j)
      ck(cudaMemcpyAsync(c->dense.p + j * max_n, c->x64.p + j * n, sizeof(double) * n,
                         cudaMemcpyDeviceToDevice, c->s), "D2D");
    coll(c, c->comm->allgather(c->dense.p, c->kgather.p, sizeof(double) * 4 * max_n, c->s),
         "allgather (cloud)");
    c->x64_next.ensure(static_cast<size_t>(N) * 4 + 4);
    for (int r = 0; r < W; ++r)
      for (int j = 0; j < 4; ++j)
        ck(cudaMemcpyAsync(c->x64_next.p + j * N + all[2 * r],
                           c->kgather.p + (static_cast<size_t>(r) * 4 + j) * max_n,
                           sizeof(double) * all[2 * r + 1], cudaMemcpyDeviceToDevice, c->s),
           "D2D");
    // the whole cloud as a one-device context (layout + seeding), then back
    const int64_t off = c->offset, ng = c->n_global;
    std::swap(c->x64.p, c->x64_next.p);
    std::swap(c->x64.cap, c->x64_next.cap);
    c->n = N;
    c->offset = 0;
    c->world = 1;
    try {
      layout(c);
      run_kinit(c, k, seed);
    } catch (...) {
      std::swap(c->x64.p, c->x64_next.p);
      std::swap(c->x64.cap, c->x64_next.cap);
      c->n = n;
      c->offset = off;
      c->world = W;
      throw;
    }
    std::swap(c->x64.p, c->x64_next.p);
    std::swap(c->x64.cap, c->x64_next.cap);
    c->n = n;
    c->offset = off;
    c->n_global = ng;
    c->world = W;
    // this shard's labels to the front (through scratch: the ranges overlap)
    c->hidx.ensure(static_cast<size_t>(n));
    ck(cudaMemcpyAsync(c->hidx.p, c->labels.p + off, sizeof(int32_t) * n,
                       cudaMemcpyDeviceToDevice, c->s), "D2D");
    ck(cudaMemcpyAsync(c->labels.p, c->hidx.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice,
                       c->s), "D2D");
    layout(c);  // the shard's own layout for its E steps
    return;
  }
  // Sharded k-means++ (GMMB_KINIT_SHARDED=rounds): local candidate per round
  // -> allgather -> every rank picks the same global (clock, index) winner. Keys hash x[i..i+3] of the
  // GLOBAL column-major buffer, so the last 3 local keys need the 3 doubles
  // that follow this shard's x column: the next shards' first x values, or
  // the global y column (rank 0's first y values) for the last shard.
  const int W = c->world;
  {
    c->ll64.ensure(static_cast<size_t>(W) * 8 + 8);
    double* g = reinterpret_cast<double*>(c->ll64.p);  // [W][8]: 3 x, 3 y, n, pad
    std::vector<double> mine(8, 0.0);
    std::vector<double> hx(std::min<int64_t>(3, n)), hy(std::min<int64_t>(3, n));
    copy_sync(c, hx.data(), c->x64.p, sizeof(double) * hx.size(), cudaMemcpyDeviceToHost);
    copy_sync(c, hy.data(), c->x64.p + n, sizeof(double) * hy.size(), cudaMemcpyDeviceToHost);
    for (size_t q = 0; q < hx.size(); ++q) {
      mine[q] = hx[q];
      mine[3 + q] = hy[q];
    }
    mine[6] = static_cast<double>(n);
    c->dense.ensure(8);
    copy_sync(c, c->dense.p, mine.data(), sizeof(double) * 8, cudaMemcpyHostToDevice);
    coll(c, c->comm->allgather(c->dense.p, g, 8 * sizeof(double), c->s), "allgather (shard heads)");
    std::vector<double> all(static_cast<size_t>(W) * 8);
    ck(cudaMemcpyAsync(all.data(), g, sizeof(double) * W * 8, cudaMemcpyDeviceToHost, c->s), "D2H");
    ck(cudaStreamSynchronize(c->s), "sync");
    double tail[3] = {0, 0, 0};
    if (gmmb_shard_key_tail(all.data(), W, c->rank, tail) != 0) throw Err{2, "bad shard layout"};
    copy_sync(c, c->dense.p, tail, sizeof(tail), cudaMemcpyHostToDevice);
    ck(launch_keys(c->x64.p, n, c->dense.p, c->keys.p, c->s), "keys");
  }
  c->rslots.ensure(static_cast<size_t>(W) + 1);
  c->ticket.ensure(1);
  ck(cudaMemsetAsync(c->ticket.p, 0, sizeof(int), c->s), "memset");
  KppRankSlot* all = c->rslots.p;
  KppRankSlot* mine = c->rslots.p + W;
  for (int r = 0; r < k; ++r) {
    ck(launch_kpp_round(c->x64.p, n, c->offset, r, seed, all, W, ks, mine, c->ticket.p,
                        c->sm_count, c->s),
       "kpp_round");
    coll(c, c->comm->allgather(mine, all, sizeof(KppRankSlot), c->s), "allgather (k-means++)");
  }
  ck(launch_kpp_final(c->x64.p, n, c->offset, k, all, W, ks, c->s), "kpp_final");
  // global owned counts; the (rare) fix-up (sogmm.cpp:315-331) runs as a
  // host loop over the empty components, each step one device search for
  // the donor's lowest local index and a min over ranks
  coll(c, c->comm->allreduce(c->owned.p, k, DType::kI32, RedOp::kSum, c->s), "allreduce (owned)");
  std::vector<int> owned(k);
  copy_sync(c, owned.data(), c->owned.p, sizeof(int) * k, cudaMemcpyDeviceToHost);
  c->ll64.ensure(2);
  for (int b = 0; b < k; ++b) {
    if (owned[b] > 0) continue;
    int donor = 0;
    for (int q = 1; q < k; ++q)
      if (owned[q] > owned[donor]) donor = q;
    ck(launch_first_label(n, c->offset, ks, donor, c->ll64.p, c->s), "first_label");
    coll(c, c->comm->allreduce(c->ll64.p, 1, DType::kI64, RedOp::kMin, c->s), "allreduce (fix-up)");
    long long lo = 0;
    copy_sync(c, &lo, c->ll64.p, sizeof(lo), cudaMemcpyDeviceToHost);
    if (lo == std::numeric_limits<long long>::max()) continue;  // donor owns nothing anywhere
    if (lo >= c->offset && lo < c->offset + n) {
      const int32_t v = b;
      copy_sync(c, c->labels.p + (lo - c->offset), &v, sizeof(v), cudaMemcpyHostToDevice);
    }
    owned[donor]--;
    owned[b]++;
  }
}

// ---- M step from labels / dense log_gamma -> model buffer st->cur -------
void run_moments_commit(gmmb_ctx* c, const int32_t* labels,
                        const double* log_gamma, int m, double cov_reg) {
  const int64_t n = c->n;
  if (labels && c->world == 1) {
    // hard labels on one device: stable sort by label + segmented moments
    c->hidx.ensure(static_cast<size_t>(n) * 3);
    const size_t tb = hard_moments_temp_bytes(n, m);
    c->sort_tmp.ensure(tb);
    HardScratch hs{c->hidx.p, c->hidx.p + n, c->hidx.p + 2 * n, c->sort_tmp.p, c->sort_tmp.cap};
    ck(launch_hard_moments(c->d, c->x64.p, n, labels, m, cov_reg, hs, c->rec, c->s),
       "hard_moments");
    ck(launch_commit(c->d, 1, c->rec, m, nullptr, c->bufs, c->st.p, nullptr, c->s), "commit");
    c->launches += 3;  // iota, moments, commit (CUB's sort kernels not counted)
    return;
  }
  const int nchunks = static_cast<int>((n + 4095) / 4096);
  c->mpart.ensure(static_cast<size_t>(nchunks) * m * 10);
  c->msums.ensure(static_cast<size_t>(m) * 10);
  c->mmeans.ensure(static_cast<size_t>(m) * 4);
  c->mcounts.ensure(m);
  MomentsScratch ms{c->mpart.p, c->msums.p, c->mmeans.p, c->mcounts.p};
  ck(launch_moments(c->d, c->x64.p, n, labels, log_gamma, m, cov_reg, ms, c->rec,
                    c->sm_count, c->s, c->world > 1 ? moments_allreduce_cb : nullptr, c),
     "moments");
  ck(launch_commit(c->d, 1, c->rec, m, nullptr, c->bufs, c->st.p, nullptr, c->s), "commit");
  c->launches += 8;
}

// ---- model upload / download -------------------------------------------
void upload_model(gmmb_ctx* c, int m, const double* w, const double* mu,
                  const double* cov) {
  const int d = c->d, np = d * (d + 1) / 2;
  if (m < 1) throw Err{2, "model has no components"};
  if (!w || !mu || !cov) throw Err{2, "null model buffer"};
  std::vector<double> hmu(static_cast<size_t>(m) * 4, 0.0), hcov(static_cast<size_t>(m) * 10, 0.0);
  for (int k = 0; k < m; ++k) {
    for (int j = 0; j < d; ++j) hmu[k * 4 + j] = mu[k * d + j];
    for (int j = 0; j < np; ++j) hcov[k * 10 + j] = cov[k * np + j];
  }
  ck(cudaMemcpyAsync(c->bufs[0].w, w, sizeof(double) * m, cudaMemcpyHostToDevice, c->s), "H2D");
  ck(cudaMemcpyAsync(c->bufs[0].mu, hmu.data(), sizeof(double) * m * 4, cudaMemcpyHostToDevice, c->s), "H2D");
  ck(cudaMemcpyAsync(c->bufs[0].cov, hcov.data(), sizeof(double) * m * 10, cudaMemcpyHostToDevice, c->s), "H2D");
  ck(cudaStreamSynchronize(c->s), "sync");  // host vectors die here
}

void download_model(gmmb_ctx* c, int buf, int m, double* w, double* mu,
                    double* cov) {
  const int d = c->d, np = d * (d + 1) / 2;
  std::vector<double> hmu(static_cast<size_t>(m) * 4), hcov(static_cast<size_t>(m) * 10);
  if (w) ck(cudaMemcpyAsync(w, c->bufs[buf].w, sizeof(double) * m, cudaMemcpyDeviceToHost, c->s), "D2H");
  ck(cudaMemcpyAsync(hmu.data(), c->bufs[buf].mu, sizeof(double) * m * 4, cudaMemcpyDeviceToHost, c->s), "D2H");
  ck(cudaMemcpyAsync(hcov.data(), c->bufs[buf].cov, sizeof(double) * m * 10, cudaMemcpyDeviceToHost, c->s), "D2H");
  ck(cudaStreamSynchronize(c->s), "sync");
  for (int k = 0; k < m; ++k) {
    if (mu)
      for (int j = 0; j < d; ++j) mu[k * d + j] = hmu[k * 4 + j];
    if (cov)
      for (int j = 0; j < np; ++j) cov[k * np + j] = hcov[k * 10 + j];
  }
}

// ---- EM loop ----------------------------------------------------------
// kernels of the fused E step + statistics per iteration (the chunked
// K > 512 path: per-chunk sums, combine, exact list, statistics)
int estep_launches(const gmmb_ctx* c, int k0) {
  return c->sparse_on ? 3 : k0 > kCtaComps ? 4 : 1;
}

void em_iteration(gmmb_ctx* c, int k0, int it,
                  const cudaGraphConditionalHandle* cond = nullptr) {
  const int NS = nstats(c->d);
  PointsDev pts{c->n, c->d, c->x64.p, c->xt.p, c->tc.p,
                static_cast<int>((c->n + kTile - 1) / kTile)};
  int ncl = 0;
  const bool timed = it >= 0 && static_cast<size_t>(2 * it + 1) < c->ev_e.size();
  if (timed) ck(cudaEventRecord(c->ev_e[2 * it], c->s), "event");
  ck(launch_estep_stats(pts, c->bufs, c->st.p, k0, c->partials.p, c->ll_part.p, 0,
                        c->sm_count, c->s, &ncl, &c->chunk,
                        c->sparse_on ? &c->sparse : nullptr),
     "estep_stats");
  if (timed) ck(cudaEventRecord(c->ev_e[2 * it + 1], c->s), "event");
  c->launches += estep_launches(c, k0) + 3;
  if (c->world == 1) {
    c->launches += -1;  // fused reduce + finalize
    ck(launch_em_reduce_finalize(c->d, c->partials.p, ncl, k0, c->bufs, c->st.p, c->rec, c->s),
       "em_reduce_finalize");
    ck(launch_commit(c->d, 0, c->rec, k0, nullptr, c->bufs, c->st.p, c->ll_trace.p, c->s, cond,
                     c->ll_part.p, ncl),
       "commit");
    return;
  }
  double* red_ll = c->red.p + static_cast<size_t>(k0) * NS;
  ck(launch_em_reduce(c->d, c->partials.p, c->ll_part.p, ncl, k0, c->st.p, c->red.p, red_ll,
                      c->s),
     "em_reduce");
  allreduce_sum(c, c->red.p, static_cast<int64_t>(k0) * NS + 1);
  ck(launch_em_finalize(c->d, c->red.p, c->bufs, c->st.p, k0, c->rec, c->s), "em_finalize");
  ck(launch_commit(c->d, 0, c->rec, k0, red_ll, c->bufs, c->st.p, c->ll_trace.p, c->s, cond),
     "commit");
}

// The whole EM loop as one CUDA graph: a conditional WHILE node whose body
// is one iteration (E+stats -> reduce -> finalize -> commit); the commit
// kernel sets the loop condition from the device state, so a fit's EM loop
// is one graph launch with no host round trip. Rebuilt only when the
// problem shape or a device buffer changes.
EmGraphKey em_graph_key(gmmb_ctx* c, int k0) {
  EmGraphKey k{};
  k.k0 = k0;
  k.d = c->d;
  k.n = c->n;
  k.world = c->world;
  k.sparse = c->sparse_on ? 1 + c->sp_nosplit : 0;
  // every device buffer the captured kernels address (a grown buffer moves)
  const void* ps[32] = {c->xt.p, c->tc.p, c->partials.p, c->ll_part.p, c->red.p, c->ll_trace.p,
                        c->st.p, c->bufs[0].w, c->bufs[1].w, c->rec.count, c->bufs[0].cst,
                        c->bufs[1].cst, c->chunkf.p, c->chunki.p, c->sp_pool.p, c->sp_blist.p,
                        c->sp_mask.p, c->sp_ctl.p, c->sp_bc.p, c->sp_toff.p, c->sp_bh.p,
                        c->sp_brec.p, c->sp_bcnt.p, c->sp_heavy.p, c->sp_done.p, c->sp_pre.p,
                        c->sp_ll.p, c->bufs[0].mu, c->bufs[1].mu, c->bufs[0].cov, c->bufs[1].cov,
                        c->x64.p};
  for (int i = 0; i < 32; ++i) k.p[i] = ps[i];
  return k;
}

void launch_em_graph(gmmb_ctx* c, int k0) {
  const EmGraphKey key = em_graph_key(c, k0);
  if (!c->em_graph || !(key == c->em_key)) {
    if (c->em_graph) cudaGraphExecDestroy(c->em_graph);
    c->em_graph = nullptr;
    cudaGraph_t g = nullptr;
    ck(cudaGraphCreate(&g, 0), "cudaGraphCreate");
    cudaGraphConditionalHandle h;
    ck(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault),
       "cudaGraphConditionalHandleCreate");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    ck(cudaGraphAddNode(&node, g, nullptr, 0, &cp), "cudaGraphAddNode");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    ck(cudaStreamBeginCaptureToGraph(c->s, body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeRelaxed),
       "cudaStreamBeginCaptureToGraph");
    const long long launches = c->launches;
    try {
      em_iteration(c, k0, -1, &h);
      c->launches = launches;
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamEndCapture(c->s, &dummy);
      cudaGraphDestroy(g);
      throw;
    }
    ck(cudaStreamEndCapture(c->s, &body), "cudaStreamEndCapture");
    ck(cudaGraphInstantiate(&c->em_graph, g, 0), "cudaGraphInstantiate");
    cudaGraphDestroy(g);
    c->em_key = key;
  }
  ck(cudaGraphLaunch(c->em_graph, c->s), "cudaGraphLaunch");
}

void ensure_em_buffers(gmmb_ctx* c, int k0, int max_iters) {
  const int NS = nstats(c->d);
  PointsDev pts{c->n, c->d, c->x64.p, c->xt.p, c->tc.p,
                static_cast<int>((c->n + kTile - 1) / kTile)};
  c->sparse_on = c->estep_mode == 0 && sparse_supported(k0, pts.ntiles);
  if (c->sparse_on) {
    const int ntiles = pts.ntiles;
    const int nitems = sparse_items(ntiles);
    const int nblk = sparse_blocks(ntiles);
    const int kw = (k0 + 31) / 32;
    // pool of per-(item, candidate) statistics: ~20-45 candidates per 32-point
    // item on the BASELINE clouds; 32 + K/64 per item (or all K) up front,
    // doubled after an overflow (the EM run is repeated, see run_em)
    // (GMMB_SPARSE_ITEM_CAP: the initial per-item reservation, a test knob
    // that exercises the overflow region and the re-run)
    static const int64_t cap0 = [] {
      const char* e = getenv("GMMB_SPARSE_ITEM_CAP");
      return e ? std::max<int64_t>(1, atoll(e)) : int64_t{0};
    }();
    const int64_t per_item =
        std::min<int64_t>(k0, (cap0 ? cap0 : 32 + k0 / 64) * int64_t{c->pool_mult});
    // fixed slots per unit + as many again for units with more candidates
    // (K >= 1024 has many units above the reservation; an overflow costs a
    // repeated EM run)
    const int64_t cap = std::max<int64_t>(static_cast<int64_t>(nitems) * per_item * 2, 1024);
    c->sp_blist.ensure(static_cast<size_t>(nblk) * k0);
    c->sp_brec.ensure(static_cast<size_t>(nblk) * k0 * 4);
    c->sp_bcnt.ensure(nblk);
    c->sp_ctl.ensure(16);
    c->sp_heavy.ensure(static_cast<size_t>(2) * kSparseMaxSplit * nitems);
    if (c->sp_done.cap < static_cast<size_t>(2) * nitems) {
      c->sp_done.ensure(static_cast<size_t>(2) * nitems);  // epoch stamps: zero once per allocation
      ck(cudaMemsetAsync(c->sp_done.p, 0, sizeof(unsigned) * c->sp_done.cap, c->s), "memset");
      ck(cudaMemsetAsync(c->sp_ctl.p, 0, sizeof(int) * 16, c->s), "memset");
    }

    const int NSP = (NS + 1) & ~1;  // pool entry stride (estep_sparse.cu)
    c->sp_pool.ensure(static_cast<size_t>(cap) * NSP);
    c->sp_toff.ensure(static_cast<size_t>(1 + kSparseMaxSplit) * nitems);
    c->sp_mask.ensure(static_cast<size_t>(kw) * nitems);
    c->sp_pre.ensure(static_cast<size_t>(kw) * nitems);
    c->sp_ll.ensure(static_cast<size_t>(1 + kSparseMaxSplit) * nitems);
    c->sparse = SparseScratch{c->sp_bc.p, c->sp_bh.p, c->sp_blist.p, c->sp_brec.p,
                              static_cast<int>(per_item), c->sp_bcnt.p, c->sp_ctl.p,
                              c->sp_heavy.p, c->sp_done.p,
                              c->sp_pool.p, static_cast<int64_t>(c->sp_pool.cap / NSP),
                              c->sp_toff.p, c->sp_mask.p, c->sp_pre.p, c->sp_ll.p, c->sp_nosplit};
  }
  int ncl = 0;
  ck(launch_estep_stats(pts, c->bufs, c->st.p, k0, nullptr, nullptr, 0,
                        c->sm_count, c->s, &ncl, nullptr, c->sparse_on ? &c->sparse : nullptr),
     "estep query");
  c->partials.ensure(static_cast<size_t>(ncl) * k0 * NS);
  c->ll_part.ensure(ncl);
  if (!c->sparse_on && k0 > kCtaComps) {  // chunked two-pass E step
    const int64_t npad = static_cast<int64_t>(pts.ntiles) * kTile;
    const int nch = (k0 + kCtaComps - 1) / kCtaComps;
    c->chunkf.ensure(chunk_scratch_floats(k0, c->n));
    c->chunki.ensure(static_cast<size_t>(npad) + 1);
    c->chunk = ChunkScratch{c->chunkf.p,
                            reinterpret_cast<float2*>(c->chunkf.p + static_cast<size_t>(nch) * npad),
                            c->chunki.p, c->chunki.p + npad};
  }
  c->red.ensure(static_cast<size_t>(k0) * NS + 1);
  c->ll_trace.ensure(std::max(max_iters, 1));
}

// Runs EM from the model in buffer st->cur (st already reset). Returns the
// final state.
EmState run_em_once(gmmb_ctx* c, int k0, const gmmb_em_params* em);

// The pruned E step writes per-(tile, candidate) statistics to a pool sized
// up front; if an iteration overflows it (a cloud where most components
// reach most tiles), the EM run is repeated from its starting model with a
// larger pool, so results never depend on the pool size.
EmState run_em(gmmb_ctx* c, int k0, const gmmb_em_params* em) {
  NvtxRange nv("gmmb.em");
  c->sp_nosplit = 0;
  for (int attempt = 0;; ++attempt) {
    ensure_em_buffers(c, k0, em->max_iters);
    if (!c->sparse_on) {
      c->units_eval = 0.0;
      return run_em_once(c, k0, em);
    }
    // snapshot of the EM start (state + both model buffers; device copies,
    // no host round trip)
    c->st_bak.ensure(1);
    const size_t kc = c->mw[0].cap;
    auto d2d = [&](void* dst, const void* src, size_t bytes) {
      ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->s), "snapshot");
    };
    d2d(c->st_bak.p, c->st.p, sizeof(EmState));
    for (int b = 0; b < 2; ++b) {
      c->bak_w[b].ensure(kc);
      c->bak_mu[b].ensure(kc * 4);
      c->bak_cov[b].ensure(kc * 10);
      c->bak_cst[b].ensure(kc);
      d2d(c->bak_w[b].p, c->mw[b].p, sizeof(double) * kc);
      d2d(c->bak_mu[b].p, c->mmu[b].p, sizeof(double) * kc * 4);
      d2d(c->bak_cov[b].p, c->mcov[b].p, sizeof(double) * kc * 10);
      d2d(c->bak_cst[b].p, c->mcst[b].p, sizeof(CompConst) * kc);
    }
    // per-fit counters (queues, pool cursor, overflow, evaluated units, heavy
    // counts); ctl[8] (the unit epoch) keeps counting
    ck(cudaMemsetAsync(c->sp_ctl.p, 0, sizeof(int) * 8, c->s), "memset");
    ck(cudaMemsetAsync(c->sp_ctl.p + 9, 0, sizeof(int) * 7, c->s), "memset");
    EmState h = run_em_once(c, k0, em);
    int ctl[16];
    copy_sync(c, ctl, c->sp_ctl.p, sizeof(ctl), cudaMemcpyDeviceToHost);
    // ctl[2] bit 0: pool overflow (retry with a larger pool); bit 1: a split
    // heavy unit needed the exact path, whose re-selected candidates could
    // differ between its sub-units (retry without splits)
    int redo[2] = {ctl[2] & 1, (ctl[2] >> 1) & 1};
    if (getenv("GMMB_DEBUG"))
      fprintf(stderr,
              "gmmb: sparse run: iters %d pool cursor %d redo flags %d heavy split tasks %d/%d "
              "whole %d/%d epoch %d tasks %d (GMMB_SP_COUNT builds)\n",
              h.iter, ctl[1], ctl[2], ctl[6], ctl[7], ctl[9], ctl[10], ctl[8], ctl[12]);
    if (c->world > 1) {  // every rank repeats together
      c->kstatus.ensure(8);
      copy_sync(c, c->kstatus.p + 6, redo, sizeof(redo), cudaMemcpyHostToDevice);
      coll(c, c->comm->allreduce(c->kstatus.p + 6, 2, DType::kI32, RedOp::kSum, c->s),
           "allreduce (pool overflow)");
      copy_sync(c, redo, c->kstatus.p + 6, sizeof(redo), cudaMemcpyDeviceToHost);
    }
    const bool overflow = redo[0] != 0 || redo[1] != 0;
    unsigned long long ev = 0;
    std::memcpy(&ev, &ctl[4], sizeof(ev));
    c->units_eval = static_cast<double>(ev);
    if (!overflow || attempt >= 8) return h;
    d2d(c->st.p, c->st_bak.p, sizeof(EmState));
    for (int b = 0; b < 2; ++b) {
      d2d(c->mw[b].p, c->bak_w[b].p, sizeof(double) * kc);
      d2d(c->mmu[b].p, c->bak_mu[b].p, sizeof(double) * kc * 4);
      d2d(c->mcov[b].p, c->bak_cov[b].p, sizeof(double) * kc * 10);
      d2d(c->mcst[b].p, c->bak_cst[b].p, sizeof(CompConst) * kc);
    }
    // (an attempt that overflowed ran on partial statistics: only its
    // overflow counts, a split conflict there says nothing)
    if (redo[0]) c->pool_mult *= 2;
    else if (redo[1]) c->sp_nosplit = 1;
  }
}

EmState run_em_once(gmmb_ctx* c, int k0, const gmmb_em_params* em) {
  while (c->ev_e.size() < static_cast<size_t>(2 * em->max_iters)) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    c->ev_e.push_back(e);
  }
  c->last_timed = !(c->world == 1 && !c->timing);
  if (!c->last_timed) {
    launch_em_graph(c, k0);
    EmState h = read_state(c);
    c->launches += static_cast<long long>(estep_launches(c, k0) + 2) * h.iter;
    return h;
  }
  int launched = 0;
  int chunk = 2;
  EmState h{};
  while (true) {
    const int todo = std::min(chunk, em->max_iters - launched);
    for (int i = 0; i < todo; ++i) em_iteration(c, k0, launched + i);
    launched += todo;
    h = read_state(c);
    if (h.done || h.error || launched >= em->max_iters) break;
    chunk = std::min(chunk * 2, 8);
  }
  return h;
}

void finish_fit(gmmb_ctx* c, const EmState& h, const gmmb_em_params* em,
                double* w_out, double* mu_out, double* cov_out,
                double* ll_trace, gmmb_fit_stats* stats) {
  raise_state_error(h);
  download_model(c, h.cur, h.k_cur, w_out, mu_out, cov_out);
  if (ll_trace && h.iter > 0) {
    copy_sync(c, ll_trace, c->ll_trace.p, sizeof(double) * h.iter, cudaMemcpyDeviceToHost);
  }
  if (stats) {
    stats->em_iterations = h.iter;
    stats->final_log_likelihood = h.ll;
    stats->removed_components = h.removed;
    stats->k_out = h.k_cur;
    stats->converged = h.converged;
    stats->units = h.units;
    stats->units_evaluated = c->sparse_on ? c->units_eval : h.units;
    double me = 0.0;
    for (int i = 0; c->last_timed && i < h.iter && static_cast<size_t>(2 * i + 1) < c->ev_e.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev_e[2 * i], c->ev_e[2 * i + 1]);
      me += ms;
    }
    stats->ms_estep = c->last_timed ? me : 0.0;  // per-kernel events only in timing mode
  }
  (void)em;
}

float elapsed(gmmb_ctx* c, int a, int b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]);
  return ms;
}

void fit_k_resident(gmmb_ctx* c, int K, const gmmb_em_params* em, double* w_out,
                    double* mu_out, double* cov_out, double* ll_trace,
                    gmmb_fit_stats* stats, int32_t* labels_out,
                    int64_t* centers_out) {
  NvtxRange nv("gmmb.fit");
  if (!c->have_cloud) throw Err{2, "no point cloud uploaded"};
  check_em(em);
  if (K < 1) throw Err{2, "kinit: k must satisfy 1 <= k <= N"};
  set_device(c);
  const int64_t ng = c->n_global;
  const int k = static_cast<int>(std::min<int64_t>(K, ng));  // sogmm.cpp:477
  c->launches = 0;
  ck(cudaEventRecord(c->ev[0], c->s), "event");
  layout(c);
  ck(cudaEventRecord(c->ev[1], c->s), "event");
  ensure_model(c, k);
  run_kinit(c, k, em->seed);
  ck(cudaEventRecord(c->ev[2], c->s), "event");
  reset_state(c, k, em, 0);
  run_moments_commit(c, c->labels.p, nullptr, k, em->cov_reg);
  ck(cudaEventRecord(c->ev[3], c->s), "event");
  // the mode-1 commit leaves k_cur / removed of the initial M step in the
  // state and does not touch iter / ll, so EM continues from it
  // (sogmm.cpp:481-487). Errors (invalid cloud, non-SPD) stop the device
  // loop and are reported after it, cloud errors first.
  ck(cudaEventRecord(c->ev[4], c->s), "event");
  EmState h = run_em(c, k, em);
  ck(cudaEventRecord(c->ev[5], c->s), "event");
  ck(cudaEventSynchronize(c->ev[5]), "sync");
  check_cloud_flags(c);
  finish_fit(c, h, em, w_out, mu_out, cov_out, ll_trace, stats);
  if (labels_out)
    copy_sync(c, labels_out, c->labels.p, sizeof(int32_t) * c->n, cudaMemcpyDeviceToHost);
  if (centers_out) {
    std::vector<long long> cc(k);
    copy_sync(c, cc.data(), c->centers.p, sizeof(long long) * k, cudaMemcpyDeviceToHost);
    for (int i = 0; i < k; ++i) centers_out[i] = cc[i];
  }
  if (stats) {
    stats->k_init = k;
    stats->ms_layout = elapsed(c, 0, 1);
    stats->ms_kinit = elapsed(c, 1, 2);
    stats->ms_mstep0 = elapsed(c, 2, 3);
    stats->ms_em = elapsed(c, 4, 5);
    stats->ms_total = elapsed(c, 0, 5);
    stats->launches = c->launches;
  }
}

void fit_from_resident(gmmb_ctx* c, int m, const double* w0, const double* mu0,
                       const double* cov0, const gmmb_em_params* em,
                       double* w_out, double* mu_out, double* cov_out,
                       double* ll_trace, gmmb_fit_stats* stats) {
  if (!c->have_cloud) throw Err{2, "no point cloud uploaded"};
  check_em(em);
  if (m < 1) throw Err{2, "model has no components"};
  set_device(c);
  c->launches = 0;
  ck(cudaEventRecord(c->ev[0], c->s), "event");
  layout(c);
  ck(cudaEventRecord(c->ev[1], c->s), "event");
  ensure_model(c, m);
  upload_model(c, m, w0, mu0, cov0);
  reset_state(c, m, em, 0);
  ck(launch_prep(c->d, c->bufs, c->st.p, m, c->s), "prep");
  c->launches += 1;
  ck(cudaEventRecord(c->ev[4], c->s), "event");
  EmState h = run_em(c, m, em);
  ck(cudaEventRecord(c->ev[5], c->s), "event");
  ck(cudaEventSynchronize(c->ev[5]), "sync");
  check_cloud_flags(c);
  finish_fit(c, h, em, w_out, mu_out, cov_out, ll_trace, stats);
  if (stats) {
    stats->k_init = m;
    stats->ms_layout = elapsed(c, 0, 1);
    stats->ms_kinit = 0.0;
    stats->ms_mstep0 = 0.0;
    stats->ms_em = elapsed(c, 4, 5);
    stats->ms_total = elapsed(c, 0, 5);
    stats->launches = c->launches;
  }
}


// ---- frame batches (cfg3): the reference's serial loop of fit calls ----
// (gmmscape_cli.cpp:208-227) with frame f+1's host-to-device copy on a copy
// stream while frame f fits (pinned host frames overlap fully).
void fit_batch(gmmb_ctx* c, int F, const double* const* pts, const int64_t* ns, int d, int K,
               const gmmb_em_params* em, const uint64_t* seeds, double* w_out, double* mu_out,
               double* cov_out, gmmb_fit_stats* stats) {
  if (F < 1) throw Err{2, "empty frame batch"};
  if (!pts || !ns) throw Err{2, "null frame list"};
  if (c->world > 1) throw Err{2, "frame batches run per device (shard the frames, not the points)"};
  check_d(d);
  check_em(em);
  if (K < 1) throw Err{2, "kinit: k must satisfy 1 <= k <= N"};
  for (int f = 0; f < F; ++f) {
    if (!pts[f]) throw Err{2, "null point buffer"};
    if (ns[f] < 1) throw Err{3, "point cloud is empty"};
    if (ns[f] > (int64_t{1} << 31) - 1) throw Err{2, "too many points for one device"};
  }
  set_device(c);
  if (!c->s_copy) {
    ck(cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreateWithFlags(&c->ev_copy, cudaEventDisableTiming), "cudaEventCreate");
  }
  const int np = d * (d + 1) / 2;
  auto prefetch = [&](int f) {  // frame f -> x64_next on the copy stream
    const int64_t n = ns[f];
    c->x64_next.ensure(static_cast<size_t>(n) * 4 + 4);
    // host (ideally pinned) or device-resident frames (unified addressing)
    ck(cudaMemcpyAsync(c->x64_next.p, pts[f], sizeof(double) * n * d, cudaMemcpyDefault,
                       c->s_copy),
       "points H2D");
    if (d == 3)
      ck(cudaMemsetAsync(c->x64_next.p + 3 * n, 0, sizeof(double) * n, c->s_copy), "memset");
    ck(cudaEventRecord(c->ev_copy, c->s_copy), "event");
  };
  prefetch(0);
  for (int f = 0; f < F; ++f) {
    // frame f becomes the resident cloud (buffer swap, ordered after its copy)
    ck(cudaStreamWaitEvent(c->s, c->ev_copy, 0), "cudaStreamWaitEvent");
    std::swap(c->x64.p, c->x64_next.p);
    std::swap(c->x64.cap, c->x64_next.cap);
    c->n = ns[f];
    c->d = d;
    c->offset = 0;
    c->n_global = ns[f];
    c->have_cloud = true;
    // the previous frame (now in x64_next) is finished: its fit synchronised
    if (f + 1 < F) prefetch(f + 1);
    gmmb_em_params ef = *em;
    ef.seed = seeds ? seeds[f] : em->seed;
    const size_t kk = static_cast<size_t>(K);
    fit_k_resident(c, K, &ef, w_out ? w_out + f * kk : nullptr,
                   mu_out ? mu_out + f * kk * d : nullptr,
                   cov_out ? cov_out + f * kk * np : nullptr, nullptr,
                   stats ? stats + f : nullptr, nullptr, nullptr);
  }
}

// ---- inference helpers ----------------------------------------------------
// gmm.cpp:8-31 Gmm4::validate (host part: sizes, finiteness, weights); the
// SPD check runs on the device (factors kernel).
void validate_model(int m, int d, const double* w, const double* mu, const double* cov) {
  if (m < 1) throw Err{3, "model has no components"};
  if (!w || !mu || !cov) throw Err{2, "null model buffer"};
  const int np = d * (d + 1) / 2;
  double sum = 0.0, wmin = INFINITY;
  bool finite = true;
  for (int k = 0; k < m; ++k) {
    finite = finite && std::isfinite(w[k]);
    for (int j = 0; j < d; ++j) finite = finite && std::isfinite(mu[k * d + j]);
    for (int j = 0; j < np; ++j) finite = finite && std::isfinite(cov[k * np + j]);
    sum += w[k];
    wmin = std::min(wmin, w[k]);
  }
  if (!finite) throw Err{3, "model contains non-finite values"};
  if (wmin <= 0.0) throw Err{3, "model weights must be positive"};
  if (std::abs(sum - 1.0) > 1e-9) throw Err{3, "model weights sum to " + std::to_string(sum)};
}

// model -> device, FP64 factors; returns the first non-SPD component or -1
int upload_factors(gmmb_ctx* c, int m, int d, const double* w, const double* mu,
                   const double* cov, bool want_lower) {
  set_device(c);
  const int np = d * (d + 1) / 2;
  c->iw.ensure(m);
  c->imu.ensure(static_cast<size_t>(m) * d);
  c->icov.ensure(static_cast<size_t>(m) * np);
  c->ifac.ensure(static_cast<size_t>(m) * 16);
  if (want_lower) c->ilow.ensure(static_cast<size_t>(m) * 10);
  c->ierr.ensure(4);
  ck(cudaMemcpyAsync(c->iw.p, w, sizeof(double) * m, cudaMemcpyHostToDevice, c->s), "H2D");
  ck(cudaMemcpyAsync(c->imu.p, mu, sizeof(double) * m * d, cudaMemcpyHostToDevice, c->s), "H2D");
  ck(cudaMemcpyAsync(c->icov.p, cov, sizeof(double) * m * np, cudaMemcpyHostToDevice, c->s), "H2D");
  const int init[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
  ck(cudaMemcpyAsync(c->ierr.p, init, sizeof(init), cudaMemcpyHostToDevice, c->s), "H2D");
  ck(launch_factors(d, c->iw.p, c->imu.p, c->icov.p, m, c->ifac.p,
                    want_lower ? c->ilow.p : nullptr, c->ierr.p, c->s),
     "factors");
  int err[4];
  copy_sync(c, err, c->ierr.p, sizeof(err), cudaMemcpyDeviceToHost);
  return err[0] == INT_MAX ? -1 : err[0];
}

// GBMS on the resident cloud (sogmm.cpp:22-195); modes copied to the host
GbmsResultHost run_gbms(gmmb_ctx* c, const gmmb_gbms_params* gp, double* modes, int capacity) {
  if (!gp) throw Err{2, "null GBMS parameters"};
  // GbmsParams::validate (sogmm.cpp:22-30)
  if (!(gp->bandwidth > 0.0) || gp->bandwidth > 1.0) throw Err{2, "bandwidth must be in (0, 1]"};
  if (gp->max_iters < 1) throw Err{2, "max_iters must be >= 1"};
  if (!(gp->convergence_tol > 0.0)) throw Err{2, "convergence_tol must be > 0"};
  const int64_t n = c->n;
  if (n > (int64_t{1} << 31) - 2) throw Err{2, "too many points for GBMS on one device"};
  // carve the scratch: 8 + 5n*4... doubles, uint64 and int32 arrays
  const size_t nn = static_cast<size_t>(n) + 1;
  const size_t tb = gbms_temp_bytes(n);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_mm = take(8 * 8), o_norm = take(nn * 32), o_seeds = take(nn * 32),
               o_next = take(nn * 32), o_w = take(nn * 8), o_w2 = take(nn * 8),
               o_terms = take(nn * 8), o_scal = take(8), o_modes = take(nn * 32),
               o_k0 = take(nn * 8), o_k1 = take(nn * 8), o_uk = take(nn * 8), o_i0 = take(nn * 4),
               o_i1 = take(nn * 4), o_i2 = take(nn * 4), o_i3 = take(nn * 4),
               o_cnt = take(nn * 4), o_off = take(nn * 4), o_nr = take(4), o_fl = take(4),
               o_tmp = take(tb);
  c->gb.ensure(off);
  unsigned char* b = c->gb.p;
  GbmsScratch g{reinterpret_cast<double*>(b + o_mm), reinterpret_cast<double*>(b + o_norm),
                reinterpret_cast<double*>(b + o_seeds), reinterpret_cast<double*>(b + o_next),
                reinterpret_cast<double*>(b + o_w), reinterpret_cast<double*>(b + o_w2),
                reinterpret_cast<double*>(b + o_terms), reinterpret_cast<double*>(b + o_scal),
                reinterpret_cast<double*>(b + o_modes), reinterpret_cast<uint64_t*>(b + o_k0),
                reinterpret_cast<uint64_t*>(b + o_k1), reinterpret_cast<uint64_t*>(b + o_uk),
                reinterpret_cast<int32_t*>(b + o_i0), reinterpret_cast<int32_t*>(b + o_i1),
                reinterpret_cast<int32_t*>(b + o_i2), reinterpret_cast<int32_t*>(b + o_i3),
                reinterpret_cast<int*>(b + o_cnt), reinterpret_cast<int*>(b + o_off),
                reinterpret_cast<int*>(b + o_nr), reinterpret_cast<int*>(b + o_fl),
                b + o_tmp, tb};
  const double mr = gp->merge_radius > 0.0 ? gp->merge_radius : gp->bandwidth * 0.5;
  GbmsParamsDev prm{gp->bandwidth, gp->convergence_tol, mr, gp->max_iters};
  GbmsResultHost res{};
  ck(gbms_run(c->x64.p, n, prm, g, &res, c->s), "gbms");
  if (modes && capacity > 0) {
    const int m = std::min(res.components, capacity);
    copy_sync(c, modes, g.modes, sizeof(double) * 4 * m, cudaMemcpyDeviceToHost);
  }
  return res;
}

// Sharded entry: runs `checks` (which may throw Err), then one all-reduce of
// [shard sizes..., error codes...] so that every rank learns the global size,
// its offset and whether ANY rank failed; all ranks then fail together (the
// failing rank with its own message, the others naming the first bad rank).
template <typename F>
void shard_exchange(gmmb_ctx* c, int64_t n, F&& checks, int64_t* off, int64_t* tot) {
  set_device(c);
  const int W = c->world;
  int code = 0;
  std::string msg;
  try {
    checks();
  } catch (const Err& e) {
    code = e.code;
    msg = e.msg;
  }
  c->ll64.ensure(static_cast<size_t>(2 * W) + 1);
  std::vector<long long> v(2 * W, 0);
  v[c->rank] = code ? 0 : n;
  v[W + c->rank] = code;
  copy_sync(c, c->ll64.p, v.data(), sizeof(long long) * 2 * W, cudaMemcpyHostToDevice);
  coll(c, c->comm->allreduce(c->ll64.p, 2 * W, DType::kI64, RedOp::kSum, c->s),
       "allreduce (shard sizes)");
  copy_sync(c, v.data(), c->ll64.p, sizeof(long long) * 2 * W, cudaMemcpyDeviceToHost);
  if (code) throw Err{code, msg};
  for (int r = 0; r < W; ++r) {
    if (v[W + r]) {
      throw Err{static_cast<int>(v[W + r]),
                "sharded fit: rank " + std::to_string(r) + " rejected its input"};
    }
  }
  *off = 0;
  *tot = 0;
  for (int r = 0; r < W; ++r) {
    if (r < c->rank) *off += v[r];
    *tot += v[r];
  }
}

}  // namespace

// ===========================================================================
extern "C" {

const char* gmmb_last_error(void) { return g_err.c_str(); }

int gmmb_ffma_peak_impl(int sm_count, void* stream, double ms_target, double* tflops,
                        double* ms);

int gmmb_ffma_peak(gmmb_ctx* c, double ms_target, double* tflops, double* ms) {
  return guarded([&] {
    if (!c || !tflops || !ms) throw Err{2, "null argument"};
    set_device(c);
    if (gmmb_ffma_peak_impl(c->sm_count, c->s, ms_target, tflops, ms) != 0)
      throw Err{1, "ffma microbenchmark failed"};
  });
}

int gmmb_shard_key_tail(const double* heads, int world, int rank, double* tail3) {
  if (!heads || !tail3 || world < 1 || rank < 0 || rank >= world) return 2;
  // flat global column-major sequence after this shard's last x: the next
  // shards' x values, then (wrapping) the global y column = rank 0's y...
  int got = 0;
  for (int r = rank + 1; r < world && got < 3; ++r) {
    const int nr = static_cast<int>(std::min(3.0, heads[r * 8 + 6]));
    for (int q = 0; q < nr && got < 3; ++q) tail3[got++] = heads[r * 8 + q];
  }
  for (int r = 0; r < world && got < 3; ++r) {
    const int nr = static_cast<int>(std::min(3.0, heads[r * 8 + 6]));
    for (int q = 0; q < nr && got < 3; ++q) tail3[got++] = heads[r * 8 + 3 + q];
  }
  for (; got < 3; ++got) tail3[got] = 0.0;  // N < 3 overall: z column
  return 0;
}

void gmmb_gbms_params_default(gmmb_gbms_params* p) {
  if (!p) return;
  p->bandwidth = 0.015;
  p->max_iters = 100;
  p->convergence_tol = 1e-5;
  p->merge_radius = -1.0;
}

void gmmb_em_params_default(gmmb_em_params* p) {
  if (!p) return;
  p->max_iters = 100;
  p->ll_rel_tol = 1e-5;
  p->cov_reg = 1e-6;
  p->seed = 0;
}

static int create(int device, int rank, int world, const void* id, VGroup* vg,
                  gmmb_ctx** out) {
  return guarded([&] {
    if (!out) throw Err{2, "null output"};
    *out = nullptr;
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw Err{2, "invalid device index"};
    gmmb_ctx* c = new gmmb_ctx();
    c->device = device;
    c->rank = rank;
    c->world = world;
    {  // GMMB_ESTEP=dense selects the dense E kernels (A/B, validation)
      const char* m = getenv("GMMB_ESTEP");
      c->estep_mode = (m && std::strcmp(m, "dense") == 0) ? 1 : 0;
      const char* ks = getenv("GMMB_KINIT_SHARDED");
      c->kinit_gather = (ks && std::strcmp(ks, "rounds") == 0) ? 0 : 1;
      const char* ki = getenv("GMMB_KINIT");
      // GMMB_KINIT=mem: memory-resident rounds past the shared-memory kernel;
      // =tile: the tile-pruned kernel at any size (A/B)
      c->kinit_tile = (ki && std::strcmp(ki, "mem") == 0) ? 0 : (ki && std::strcmp(ki, "tile") == 0) ? 2 : 1;
    }
    try {
      ck(cudaSetDevice(device), "cudaSetDevice");
      cudaDeviceProp prop{};
      ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
      c->sm_count = prop.multiProcessorCount;
      c->cc_major = prop.major;
      c->cc_minor = prop.minor;
      ck(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking), "cudaStreamCreate");
      for (auto& e : c->ev) ck(cudaEventCreate(&e), "cudaEventCreate");
      ck(cudaMallocHost(&c->st_host, sizeof(EmState)), "cudaMallocHost");
      if (vg) {
        c->comm = make_virtual_comm(vg, rank);
      } else if (world > 1) {
        try {
          c->comm = make_nccl_comm(id, rank, world);
        } catch (const std::exception& e) {
          throw Err{1, e.what()};
        }
      }
    } catch (...) {
      gmmb_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

int gmmb_ctx_create(int device, gmmb_ctx** out) {
  return create(device, 0, 1, nullptr, nullptr, out);
}

int gmmb_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) throw Err{2, "null output"};
    const char* err = nullptr;
    if (nccl_unique_id(out128, &err) != 0) throw Err{1, std::string("ncclGetUniqueId: ") + err};
  });
}

struct gmmb_vgroup {
  VGroup* g;
};

int gmmb_vgroup_create(int device, int world, gmmb_vgroup** out) {
  return guarded([&] {
    if (!out) throw Err{2, "null output"};
    *out = nullptr;
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) throw Err{2, "invalid device index"};
    if (world < 1 || world > 64) throw Err{2, "virtual world must be 1..64"};
    try {
      *out = new gmmb_vgroup{vgroup_create(device, world)};
    } catch (const std::exception& e) {
      throw Err{1, e.what()};
    }
  });
}

void gmmb_vgroup_release(gmmb_vgroup* g) {
  if (!g) return;
  vgroup_release(g->g);
  delete g;
}

int gmmb_ctx_create_virtual(gmmb_vgroup* g, int rank, gmmb_ctx** out) {
  if (!g || rank < 0 || rank >= vgroup_world(g->g)) {
    g_err = "invalid virtual group / rank";
    return 2;
  }
  return create(vgroup_device(g->g), rank, vgroup_world(g->g), nullptr, g->g, out);
}

int gmmb_ctx_create_sharded(int device, int rank, int world, const void* nccl_id128,
                            gmmb_ctx** out) {
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_id128)) {
    g_err = "invalid rank/world";
    return 2;
  }
  return create(device, rank, world, nccl_id128, nullptr, out);
}

void gmmb_ctx_destroy(gmmb_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->s) cudaStreamSynchronize(c->s);
  delete c->comm;
  c->x64.release(); c->x64_next.release(); c->xt.release(); c->tc.release(); c->perm.release();
  c->bbox_part.release(); c->mkeys_in.release(); c->mkeys_out.release();
  c->midx.release(); c->sort_tmp.release(); c->flags.release(); c->hidx.release();
  c->iw.release(); c->imu.release(); c->icov.release(); c->ifac.release(); c->ilow.release();
  c->iout.release(); c->iout2.release(); c->ierr.release(); c->img.release();
  c->iflags.release(); c->in_n.release(); c->gb.release();
  c->keys.release(); c->kd2.release(); c->labels.release(); c->chosen.release();
  c->kxf.release(); c->ktp.release(); c->kinv.release();
  c->slots.release(); c->owned.release(); c->centers.release(); c->rslots.release();
  c->ticket.release(); c->kstatus.release(); c->ll64.release();
  c->kt_xm.release(); c->kt_d2.release(); c->kt_tile.release(); c->kt_key.release();
  c->kt_lab.release(); c->kgather.release();
  for (int b = 0; b < 2; ++b) {
    c->mw[b].release(); c->mmu[b].release(); c->mcov[b].release(); c->mcst[b].release();
  }
  c->rcount.release(); c->rmean.release(); c->rcov.release(); c->rlogdet.release();
  c->rpc.release(); c->rflags.release(); c->rmap.release(); c->mpart.release(); c->msums.release();
  c->mmeans.release(); c->mcounts.release(); c->partials.release(); c->ll_part.release();
  c->red.release(); c->ll_trace.release(); c->dense.release(); c->st.release();
  c->chunkf.release(); c->chunki.release();
  c->sp_bc.release(); c->sp_pool.release(); c->sp_ll.release(); c->sp_bh.release();
  c->sp_blist.release(); c->sp_bcnt.release(); c->sp_ctl.release(); c->sp_toff.release();
  c->sp_mask.release(); c->sp_pre.release(); c->st_bak.release();
  c->sp_heavy.release(); c->sp_done.release(); c->sp_brec.release();
  for (int b = 0; b < 2; ++b) {
    c->bak_w[b].release(); c->bak_mu[b].release(); c->bak_cov[b].release(); c->bak_cst[b].release();
  }
  if (c->em_graph) cudaGraphExecDestroy(c->em_graph);
  if (c->st_host) cudaFreeHost(c->st_host);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_e) cudaEventDestroy(e);
  if (c->s) cudaStreamDestroy(c->s);
  if (c->s_copy) cudaStreamDestroy(c->s_copy);
  if (c->ev_copy) cudaEventDestroy(c->ev_copy);
  delete c;
}

int gmmb_ctx_set_timing(gmmb_ctx* c, int per_kernel_events) {
  if (!c) return 2;
  c->timing = per_kernel_events ? 1 : 0;
  return 0;
}

int gmmb_ctx_set_estep_mode(gmmb_ctx* c, int mode) {
  if (!c || mode < 0 || mode > 1) return 2;
  c->estep_mode = mode;
  return 0;
}

int gmmb_device_info(gmmb_ctx* c, int* sm_count, int* cc_major, int* cc_minor) {
  if (!c) return 2;
  if (sm_count) *sm_count = c->sm_count;
  if (cc_major) *cc_major = c->cc_major;
  if (cc_minor) *cc_minor = c->cc_minor;
  return 0;
}

int gmmb_upload(gmmb_ctx* c, const double* pts, int64_t n, int d, int64_t offset,
                int64_t n_global) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    upload(c, pts, n, d, offset, n_global > 0 ? n_global : n);
  });
}

int gmmb_fit_k_resident(gmmb_ctx* c, int K, const gmmb_em_params* em, double* w_out,
                        double* mu_out, double* cov_out, double* ll_trace,
                        gmmb_fit_stats* stats, int32_t* labels, int64_t* centers) {
  return guarded_coll(c, [&] {
    if (!c) throw Err{2, "null context"};
    fit_k_resident(c, K, em, w_out, mu_out, cov_out, ll_trace, stats, labels, centers);
  });
}

int gmmb_fit_from_resident(gmmb_ctx* c, int m, const double* w0, const double* mu0,
                           const double* cov0, const gmmb_em_params* em,
                           double* w_out, double* mu_out, double* cov_out,
                           double* ll_trace, gmmb_fit_stats* stats) {
  return guarded_coll(c, [&] {
    if (!c) throw Err{2, "null context"};
    fit_from_resident(c, m, w0, mu0, cov0, em, w_out, mu_out, cov_out, ll_trace, stats);
  });
}

int gmmb_fit_k(gmmb_ctx* c, const double* pts, int64_t n, int d, int K,
               const gmmb_em_params* em, double* w_out, double* mu_out,
               double* cov_out, double* ll_trace, gmmb_fit_stats* stats,
               int32_t* labels, int64_t* centers) {
  return guarded_coll(c, [&] {
    if (!c) throw Err{2, "null context"};
    if (c->world > 1) {
      // every rank validates, then one exchange of (size, error) decides
      // for all: a rank that failed alone must not leave its peers blocked
      // in a later collective
      int64_t off = 0, tot = 0;
      shard_exchange(c, n, [&] {
        check_d(d);
        if (n < 1) throw Err{3, "point cloud is empty"};
        if (!pts) throw Err{2, "null point buffer"};
        if (n > (int64_t{1} << 31) - 1) throw Err{2, "too many points for one device"};
        check_em(em);
        if (K < 1) throw Err{2, "kinit: k must satisfy 1 <= k <= N"};
      }, &off, &tot);
      upload(c, pts, n, d, off, tot);
    } else {
      check_d(d);
      if (n < 1) throw Err{3, "point cloud is empty"};
      check_em(em);
      upload(c, pts, n, d, 0, n);
    }
    fit_k_resident(c, K, em, w_out, mu_out, cov_out, ll_trace, stats, labels, centers);
  });
}

int gmmb_fit_k_batch(gmmb_ctx* c, int frames, const double* const* pts, const int64_t* n, int d,
                     int K, const gmmb_em_params* em, const uint64_t* seeds, double* w_out,
                     double* mu_out, double* cov_out, gmmb_fit_stats* stats) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    fit_batch(c, frames, pts, n, d, K, em, seeds, w_out, mu_out, cov_out, stats);
  });
}

int gmmb_fit_from(gmmb_ctx* c, const double* pts, int64_t n, int d, int m,
                  const double* w0, const double* mu0, const double* cov0,
                  const gmmb_em_params* em, double* w_out, double* mu_out,
                  double* cov_out, double* ll_trace, gmmb_fit_stats* stats) {
  return guarded_coll(c, [&] {
    if (!c) throw Err{2, "null context"};
    if (c->world > 1) {
      int64_t off = 0, tot = 0;
      shard_exchange(c, n, [&] {
        check_d(d);
        if (n < 1) throw Err{3, "point cloud is empty"};
        if (!pts) throw Err{2, "null point buffer"};
        if (n > (int64_t{1} << 31) - 1) throw Err{2, "too many points for one device"};
        check_em(em);
        if (m < 1) throw Err{2, "model has no components"};
      }, &off, &tot);
      upload(c, pts, n, d, off, tot);
    } else {
      upload(c, pts, n, d, 0, n);
    }
    fit_from_resident(c, m, w0, mu0, cov0, em, w_out, mu_out, cov_out, ll_trace, stats);
  });
}

int gmmb_kinit(gmmb_ctx* c, const double* pts, int64_t n, int d, int k, uint64_t seed,
               int32_t* labels, int64_t* centers) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    if (c->world > 1) throw Err{2, "gmmb_kinit is single-device; use gmmb_fit_k"};
    upload(c, pts, n, d, 0, n);
    c->have_cloud = false;  // single-step input: not a resident cloud for *_resident fits
    // the tile-pruned seeding (large clouds) runs on the Morton layout
    if (c->kinit_tile && (c->kinit_tile == 2 || kpp_tile_wanted(n, c->sm_count)))
      layout(c);
    else
      validate(c);
    check_cloud_flags(c);
    if (k < 1 || k > n) throw Err{2, "kinit: k must satisfy 1 <= k <= N"};  // sogmm.cpp:200
    ensure_model(c, k);
    run_kinit(c, k, seed);
    ck(cudaStreamSynchronize(c->s), "sync");
    if (labels)
      copy_sync(c, labels, c->labels.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost);
    if (centers) {
      std::vector<long long> cc(k);
      copy_sync(c, cc.data(), c->centers.p, sizeof(long long) * k, cudaMemcpyDeviceToHost);
      for (int i = 0; i < k; ++i) centers[i] = cc[i];
    }
  });
}

int gmmb_e_step(gmmb_ctx* c, const double* pts, int64_t n, int d, int m, const double* w,
                const double* mu, const double* cov, double* ll_out, double* log_gamma_out) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    upload(c, pts, n, d, 0, n);
    c->have_cloud = false;  // single-step input: not a resident cloud for *_resident fits
    validate(c);
    check_cloud_flags(c);
    if (m < 1 || !w || !mu || !cov) throw Err{2, "model has no components"};
    // cholesky_cache semantics (gmm.cpp:33-48, kernels.cpp:71-75)
    const int bad = upload_factors(c, m, d, w, mu, cov, false);
    if (bad >= 0)
      throw Err{3, "cholesky failed: block " + std::to_string(bad) + " is not positive definite"};
    const int nblk = dense_blocks(n);
    c->ll_part.ensure(nblk);
    if (log_gamma_out) c->dense.ensure(static_cast<size_t>(n) * m);
    ck(launch_dense(d, c->x64.p, n, c->ifac.p, m, nullptr, c->ll_part.p,
                    log_gamma_out ? c->dense.p : nullptr, c->s),
       "dense");
    std::vector<double> parts(nblk);
    copy_sync(c, parts.data(), c->ll_part.p, sizeof(double) * nblk, cudaMemcpyDeviceToHost);
    double ll = 0.0;
    for (double p : parts) ll += p;
    if (ll_out) *ll_out = ll;
    if (log_gamma_out)
      copy_sync(c, log_gamma_out, c->dense.p, sizeof(double) * n * m, cudaMemcpyDeviceToHost);
  });
}

int gmmb_ingest_images(gmmb_ctx* c, const uint16_t* depth, const uint16_t* intensity, int width,
                       int height, double intensity_max, double fx, double fy, double cx,
                       double cy, double depth_scale, int factor, double* pts_out,
                       int64_t* n_out) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    if (!depth || !intensity) throw Err{2, "null image"};
    // decimate (ingest.cpp:59-63)
    if (factor < 1) throw Err{2, "decimation factor must be >= 1"};
    if (factor > width || factor > height)
      throw Err{2, "decimation factor exceeds image dimensions"};
    if (!(intensity_max > 0.0)) throw Err{2, "intensity max_value must be > 0"};
    // CameraIntrinsics::decimated + validate (ingest.cpp:7-25)
    const int wd = width / factor, hd = height / factor;
    IngestParams ip{fx / factor, fy / factor, cx / factor, cy / factor, 1.0 / depth_scale,
                    1.0 / intensity_max};
    if (ip.fx <= 0.0 || ip.fy <= 0.0 || depth_scale <= 0.0)
      throw Err{2, "intrinsics: fx, fy, depth_scale must be > 0"};
    if (!(ip.cx > 0.0 && ip.cx < wd) || !(ip.cy > 0.0 && ip.cy < hd))
      throw Err{2, "intrinsics: principal point outside image"};
    set_device(c);
    const int64_t npx = static_cast<int64_t>(width) * height;
    const int64_t np = static_cast<int64_t>(wd) * hd;
    c->img.ensure(static_cast<size_t>(npx) * 2);
    c->iflags.ensure(static_cast<size_t>(np) * 2);
    c->in_n.ensure(1);
    const size_t tb = ingest_temp_bytes(np);
    c->sort_tmp.ensure(tb);
    c->x64.ensure(static_cast<size_t>(np) * 4 + 4);
    ck(cudaMemcpyAsync(c->img.p, depth, sizeof(uint16_t) * npx, cudaMemcpyHostToDevice, c->s),
       "depth H2D");
    ck(cudaMemcpyAsync(c->img.p + npx, intensity, sizeof(uint16_t) * npx, cudaMemcpyHostToDevice,
                       c->s),
       "intensity H2D");
    IngestScratch is{c->iflags.p, c->iflags.p + np, c->sort_tmp.p, c->sort_tmp.cap};
    ck(launch_ingest(c->img.p, c->img.p + npx, width, wd, hd, factor, ip, is, c->x64.p,
                     c->in_n.p, c->s),
       "ingest");
    int64_t n = 0;
    copy_sync(c, &n, c->in_n.p, sizeof(n), cudaMemcpyDeviceToHost);
    if (n == 0) throw Err{3, "all depth pixels are zero: empty cloud"};
    c->n = n;
    c->d = 4;
    c->offset = 0;
    c->n_global = n;
    c->have_cloud = true;
    if (n_out) *n_out = n;
    if (pts_out)
      copy_sync(c, pts_out, c->x64.p, sizeof(double) * n * 4, cudaMemcpyDeviceToHost);
  });
}

int gmmb_gbms(gmmb_ctx* c, const double* pts, int64_t n, int d, const gmmb_gbms_params* gp,
              int* components, int* iterations, double* modes, int modes_capacity) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    upload(c, pts, n, d, 0, n);
    c->have_cloud = false;  // single-step input: not a resident cloud for *_resident fits
    validate(c);
    check_cloud_flags(c);  // cloud.validate() (sogmm.cpp:36)
    const GbmsResultHost r = run_gbms(c, gp, modes, modes_capacity);
    if (components) *components = r.components;
    if (iterations) *iterations = r.iterations;
  });
}

int gmmb_fit(gmmb_ctx* c, const double* pts, int64_t n, int d, const gmmb_gbms_params* gp,
             const gmmb_em_params* em, int capacity, double* w_out, double* mu_out,
             double* cov_out, double* ll_trace, gmmb_fit_stats* stats, int* gbms_components) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    if (c->world > 1) throw Err{2, "gmmb_fit is single-device; use gmmb_fit_k when sharded"};
    upload(c, pts, n, d, 0, n);
    validate(c);
    check_cloud_flags(c);  // sogmm.cpp:466
    check_em(em);          // :468-470
    const GbmsResultHost r = run_gbms(c, gp, nullptr, 0);  // :472-475
    if (gbms_components) *gbms_components = r.components;
    const int k = static_cast<int>(std::min<int64_t>(r.components, n));  // :477
    if (k > capacity) throw Err{2, "output capacity smaller than the GBMS component count"};
    fit_k_resident(c, k, em, w_out, mu_out, cov_out, ll_trace, stats, nullptr, nullptr);
  });
}

int gmmb_score(gmmb_ctx* c, const double* pts, int64_t n, int d, int m, const double* w,
               const double* mu, const double* cov, double* avg_ll_out, double* point_ll_out) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    check_d(d);
    if (n < 1) throw Err{2, "empty cloud"};  // inference.cpp:143
    validate_model(m, d, w, mu, cov);
    upload(c, pts, n, d, 0, n);
    c->have_cloud = false;  // single-step input: not a resident cloud for *_resident fits
    validate(c);
    check_cloud_flags(c);
    const int bad = upload_factors(c, m, d, w, mu, cov, false);
    if (bad >= 0)
      throw Err{3, "covariance of component " + std::to_string(bad) + " is not positive definite"};
    const int nblk = dense_blocks(n);
    c->ll_part.ensure(nblk);
    if (point_ll_out) c->iout.ensure(n);
    ck(launch_dense(d, c->x64.p, n, c->ifac.p, m, point_ll_out ? c->iout.p : nullptr,
                    c->ll_part.p, nullptr, c->s),
       "dense");
    std::vector<double> parts(nblk);
    copy_sync(c, parts.data(), c->ll_part.p, sizeof(double) * nblk, cudaMemcpyDeviceToHost);
    double ll = 0.0;
    for (double p : parts) ll += p;
    if (avg_ll_out) *avg_ll_out = ll / static_cast<double>(n);
    if (point_ll_out)
      copy_sync(c, point_ll_out, c->iout.p, sizeof(double) * n, cudaMemcpyDeviceToHost);
  });
}

int gmmb_sample(gmmb_ctx* c, int d, int m, const double* w, const double* mu, const double* cov,
                int64_t n, uint64_t seed, double* out) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    check_d(d);
    if (n < 1) throw Err{2, "sample count must be >= 1"};  // inference.cpp:19
    if (!out) throw Err{2, "null output"};
    validate_model(m, d, w, mu, cov);
    const int bad = upload_factors(c, m, d, w, mu, cov, true);
    if (bad >= 0)
      throw Err{3, "covariance of component " + std::to_string(bad) + " is not positive definite"};
    c->iout.ensure(static_cast<size_t>(n) * d);
    c->iout2.ensure(m);
    ck(launch_sample(d, c->iw.p, c->ifac.p, c->ilow.p, m, n, seed, c->iout2.p, c->iout.p, c->s),
       "sample");
    copy_sync(c, out, c->iout.p, sizeof(double) * n * d, cudaMemcpyDeviceToHost);
  });
}

int gmmb_color_conditional(gmmb_ctx* c, int m, const double* w, const double* mu,
                           const double* cov, const double* locs, int64_t n, int clamp,
                           double* expected, double* variance) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    validate_model(m, 4, w, mu, cov);
    if (n < 1) return;
    if (!locs || !expected || !variance) throw Err{2, "null buffer"};
    const int bad = upload_factors(c, m, 4, w, mu, cov, false);
    if (bad >= 0)
      throw Err{3, "covariance of component " + std::to_string(bad) + " is not positive definite"};
    c->iout.ensure(static_cast<size_t>(n) * 5 + static_cast<size_t>(m) * 20);
    double* dl = c->iout.p;                 // locs n x 3
    double* de = dl + 3 * n;                // expected
    double* dv = de + n;                    // variance
    double* cnd = dv + n;                   // [m][20]
    ck(cudaMemcpyAsync(dl, locs, sizeof(double) * n * 3, cudaMemcpyHostToDevice, c->s), "H2D");
    const int init[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
    ck(cudaMemcpyAsync(c->ierr.p, init, sizeof(init), cudaMemcpyHostToDevice, c->s), "H2D");
    ck(launch_conditional(c->iw.p, c->imu.p, c->icov.p, m, dl, n, clamp, cnd, de, dv, c->ierr.p,
                          c->s),
       "conditional");
    int err[4];
    copy_sync(c, err, c->ierr.p, sizeof(err), cudaMemcpyDeviceToHost);
    if (err[0] != INT_MAX)
      throw Err{3, "spatial covariance of component " + std::to_string(err[0]) +
                       " is not positive definite"};
    if (err[1] != INT_MAX) throw Err{3, "conditional variance below tolerance"};
    copy_sync(c, expected, de, sizeof(double) * n, cudaMemcpyDeviceToHost);
    copy_sync(c, variance, dv, sizeof(double) * n, cudaMemcpyDeviceToHost);
  });
}

int gmmb_m_step(gmmb_ctx* c, const double* pts, int64_t n, int d, const double* log_gamma,
                int m, double cov_reg, double* w_out, double* mu_out, double* cov_out,
                int* m_out, int* removed) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    if (cov_reg < 0.0) throw Err{2, "cov_reg must be >= 0"};
    if (!log_gamma || m < 1) throw Err{2, "responsibility rows != point count"};
    upload(c, pts, n, d, 0, n);
    c->have_cloud = false;  // single-step input: not a resident cloud for *_resident fits
    ensure_model(c, m);
    c->dense.ensure(static_cast<size_t>(n) * m);
    ck(cudaMemcpyAsync(c->dense.p, log_gamma, sizeof(double) * n * m, cudaMemcpyHostToDevice, c->s), "H2D");
    gmmb_em_params em{1, 0.0, cov_reg, 0};
    reset_state(c, m, &em, 0);
    run_moments_commit(c, nullptr, c->dense.p, m, cov_reg);
    EmState h = read_state(c);
    raise_state_error(h);
    download_model(c, h.cur, h.k_cur, w_out, mu_out, cov_out);
    if (m_out) *m_out = h.k_cur;
    if (removed) *removed = h.removed;
  });
}

int gmmb_em_step(gmmb_ctx* c, const double* pts, int64_t n, int d, int m, const double* w,
                 const double* mu, const double* cov, double cov_reg, double* ll_out,
                 double* w_out, double* mu_out, double* cov_out, int* m_out, int* removed) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    gmmb_em_params em{1, 0.0, cov_reg, 0};
    upload(c, pts, n, d, 0, n);
    c->have_cloud = false;  // single-step input: not a resident cloud for *_resident fits
    layout(c);
    check_cloud_flags(c);
    ensure_model(c, m);
    upload_model(c, m, w, mu, cov);
    reset_state(c, m, &em, 0);
    ck(launch_prep(c->d, c->bufs, c->st.p, m, c->s), "prep");
    raise_state_error(read_state(c));
    // one iteration through run_em: per-run counters and the pruned E step's
    // pool-overflow re-run live there
    EmState h = run_em(c, m, &em);
    raise_state_error(h);
    if (ll_out) *ll_out = h.ll;
    download_model(c, h.cur, h.k_cur, w_out, mu_out, cov_out);
    if (m_out) *m_out = h.k_cur;
    if (removed) *removed = h.removed;
  });
}

int gmmb_cholesky_cache(gmmb_ctx* c, int d, int m, const double* covs, double* lower,
                        double* precision, double* log_det_terms) {
  return guarded([&] {
    if (!c) throw Err{2, "null context"};
    check_d(d);
    if (m < 1 || !covs) throw Err{2, "model has no components"};
    // host FP64 restatement is not allowed on the product path: use prep on
    // the device and read back the FP64 factors through a dedicated pass
    set_device(c);
    c->d = d;
    c->have_cloud = false;  // the resident cloud's D no longer holds
    ensure_model(c, m);
    std::vector<double> w(m, 1.0 / m), mu(static_cast<size_t>(m) * d, 0.0);
    upload_model(c, m, w.data(), mu.data(), covs);
    reset_state(c, m, nullptr, 0);
    ck(launch_prep(d, c->bufs, c->st.p, m, c->s), "prep");
    raise_state_error(read_state(c));
    // factors: recompute in FP64 on the device via the dense helper
    c->dense.ensure(static_cast<size_t>(m) * 33);
    ck(launch_factor_dump(d, c->bufs, c->st.p, m, c->dense.p, c->s), "factor_dump");
    std::vector<double> f(static_cast<size_t>(m) * 33);
    copy_sync(c, f.data(), c->dense.p, sizeof(double) * m * 33, cudaMemcpyDeviceToHost);
    for (int k = 0; k < m; ++k) {
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
          if (lower) lower[(k * d + i) * d + j] = f[k * 33 + i * 4 + j];
          if (precision) precision[(k * d + i) * d + j] = f[k * 33 + 16 + i * 4 + j];
        }
      if (log_det_terms) log_det_terms[k] = f[k * 33 + 32];
    }
  });
}

}  // extern "C"
