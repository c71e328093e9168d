// comm.cu — NCCL and in-process virtual-rank collectives (comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "comm.cuh"

namespace gmmb {

namespace {

// ---- NCCL, loaded lazily (only sharded contexts need it) -----------------
struct NcclLib {
  void* h = nullptr;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok() const { return GetUniqueId && CommInitRank && AllReduce && AllGather; }
};

NcclLib& nccl_lib() {
  static NcclLib n;
  static std::once_flag once;
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) {
      n.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
    n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
    n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
    n.AllReduce = (decltype(n.AllReduce))dlsym(n.h, "ncclAllReduce");
    n.AllGather = (decltype(n.AllGather))dlsym(n.h, "ncclAllGather");
    n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
    if (!n.ok()) n.err = "libnccl.so.2 lacks required symbols";
  });
  return n;
}

ncclDataType_t nccl_type(DType t) {
  return t == DType::kF64 ? ncclFloat64 : t == DType::kI32 ? ncclInt32 : ncclInt64;
}
ncclRedOp_t nccl_op(RedOp o) {
  return o == RedOp::kSum ? ncclSum : o == RedOp::kMin ? ncclMin : ncclMax;
}
size_t dtype_bytes(DType t) { return t == DType::kI32 ? 4 : 8; }

class NcclComm final : public Comm {
 public:
  NcclComm(const void* id128, int rank, int world) : rank_(rank), world_(world) {
    NcclLib& n = nccl_lib();
    if (!n.ok()) throw std::runtime_error(n.err);
    ncclUniqueId uid;
    std::memcpy(&uid, id128, sizeof(uid));
    const ncclResult_t r = n.CommInitRank(&comm_, world, uid, rank);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclCommInitRank: ") + str(r));
  }
  ~NcclComm() override {
    if (comm_ && nccl_lib().CommDestroy) nccl_lib().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  cudaError_t allreduce(void* buf, size_t count, DType t, RedOp op, cudaStream_t s) override {
    return check(nccl_lib().AllReduce(buf, buf, count, nccl_type(t), nccl_op(op), comm_, s),
                 "ncclAllReduce");
  }
  cudaError_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    return check(nccl_lib().AllGather(send, recv, bytes, ncclUint8, comm_, s), "ncclAllGather");
  }
  const char* last_error() const override { return err_.c_str(); }

 private:
  static const char* str(ncclResult_t r) {
    return nccl_lib().GetErrorString ? nccl_lib().GetErrorString(r) : "nccl error";
  }
  cudaError_t check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return cudaSuccess;
    err_ = std::string(what) + ": " + str(r);
    return cudaErrorUnknown;
  }
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
  std::string err_;
};

// ---- virtual ranks: G host threads driving G contexts on one device ------
constexpr int kMaxVRanks = 64;
struct PtrPack {
  const void* p[kMaxVRanks];
};

template <typename T, int OP>
__global__ void vreduce_kernel(PtrPack src, int nsrc, T* __restrict__ dst, size_t count) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    T v = static_cast<const T*>(src.p[0])[i];
    for (int r = 1; r < nsrc; ++r) {  // fixed rank order: deterministic sums
      const T o = static_cast<const T*>(src.p[r])[i];
      v = OP == 0 ? v + o : OP == 1 ? (o < v ? o : v) : (o > v ? o : v);
    }
    dst[i] = v;
  }
}

template <typename T>
cudaError_t launch_vreduce(const PtrPack& pk, int g, void* dst, size_t count, RedOp op,
                           cudaStream_t s) {
  const int grid = static_cast<int>(count / 256 + 1 < 1024 ? count / 256 + 1 : 1024);
  T* d = static_cast<T*>(dst);
  if (op == RedOp::kSum) vreduce_kernel<T, 0><<<grid, 256, 0, s>>>(pk, g, d, count);
  else if (op == RedOp::kMin) vreduce_kernel<T, 1><<<grid, 256, 0, s>>>(pk, g, d, count);
  else vreduce_kernel<T, 2><<<grid, 256, 0, s>>>(pk, g, d, count);
  return cudaGetLastError();
}

}  // namespace

struct VGroup {
  int device = 0;
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool aborted = false;
  struct Slot {
    const void* send = nullptr;
    cudaEvent_t ready = nullptr;
  };
  std::vector<Slot> slots;
  cudaEvent_t done = nullptr;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int refs = 0;  // live virtual comms + the creator's handle

  // returns false if the group was aborted (a rank failed)
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (aborted) return false;
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    return !aborted || gen != g;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    aborted = true;
    cv.notify_all();
  }
};

namespace {

class VirtualComm final : public Comm {
 public:
  VirtualComm(VGroup* g, int rank) : g_(g), rank_(rank) {
    std::lock_guard<std::mutex> lk(g->m);
    ++g->refs;
  }
  ~VirtualComm() override {
    // a rank that goes away mid-sequence must not leave its peers waiting
    g_->abort();
    vgroup_release(g_);
  }
  void abort() override { g_->abort(); }
  int rank() const override { return rank_; }
  int size() const override { return g_->world; }
  const char* last_error() const override { return err_.c_str(); }

  cudaError_t allreduce(void* buf, size_t count, DType t, RedOp op, cudaStream_t s) override {
    const size_t bytes = count * dtype_bytes(t);
    return run(buf, buf, bytes, s, [&](const PtrPack& pk, cudaStream_t s0) -> cudaError_t {
      switch (t) {
        case DType::kF64: return launch_vreduce<double>(pk, g_->world, g_->scratch, count, op, s0);
        case DType::kI32: return launch_vreduce<int>(pk, g_->world, g_->scratch, count, op, s0);
        default: return launch_vreduce<long long>(pk, g_->world, g_->scratch, count, op, s0);
      }
    }, bytes);
  }

  cudaError_t allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    return run(send, recv, bytes, s, [&](const PtrPack& pk, cudaStream_t s0) -> cudaError_t {
      for (int r = 0; r < g_->world; ++r) {
        const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(g_->scratch) + r * bytes,
                                              pk.p[r], bytes, cudaMemcpyDeviceToDevice, s0);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }, bytes * g_->world);
  }

 private:
  // Rendezvous: every rank publishes its send buffer and an event after its
  // prior work; rank 0 waits for all of them, combines into the group
  // scratch, records `done`; every rank waits for `done` and copies the
  // scratch into its receive buffer. The next collective's rank-0 combine
  // waits for every rank's events again, i.e. after their copies, so the
  // scratch is never overwritten while a rank still reads it.
  template <typename F>
  cudaError_t run(const void* send, void* recv, size_t send_bytes, cudaStream_t s, F&& combine,
                  size_t out_bytes) {
    (void)send_bytes;
    VGroup& g = *g_;
    cudaError_t e = cudaEventRecord(g.slots[rank_].ready, s);
    if (e != cudaSuccess) return fail(e, "cudaEventRecord");
    g.slots[rank_].send = send;
    if (!g.barrier()) return fail(cudaErrorUnknown, "virtual rank group aborted");
    if (rank_ == 0) {
      if (out_bytes > g.scratch_bytes) {
        // every rank is parked at the barrier with its work enqueued; the
        // device sync makes the old scratch safe to free
        cudaDeviceSynchronize();
        if (g.scratch) cudaFree(g.scratch);
        g.scratch = nullptr;
        g.scratch_bytes = 0;
        const size_t want = out_bytes < (1u << 20) ? (1u << 20) : out_bytes;
        e = cudaMalloc(&g.scratch, want);
        if (e != cudaSuccess) {
          g.abort();
          return fail(e, "cudaMalloc (virtual comm scratch)");
        }
        g.scratch_bytes = want;
      }
      PtrPack pk{};
      for (int r = 0; r < g.world; ++r) {
        pk.p[r] = g.slots[r].send;
        e = cudaStreamWaitEvent(s, g.slots[r].ready, 0);
        if (e != cudaSuccess) break;
      }
      if (e == cudaSuccess) e = combine(pk, s);
      if (e == cudaSuccess) e = cudaEventRecord(g.done, s);
      if (e != cudaSuccess) {
        g.abort();
        return fail(e, "virtual collective");
      }
    }
    if (!g.barrier()) return fail(cudaErrorUnknown, "virtual rank group aborted");
    e = cudaStreamWaitEvent(s, g.done, 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(recv, g.scratch, out_bytes, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return fail(e, "virtual collective copy-out");
    return cudaSuccess;
  }
  cudaError_t fail(cudaError_t e, const char* what) {
    err_ = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaSuccess ? cudaErrorUnknown : e;
  }
  VGroup* g_;
  int rank_;
  std::string err_;
};

}  // namespace

namespace {
void vgroup_destroy(VGroup* g);
}

Comm* make_nccl_comm(const void* nccl_id128, int rank, int world) {
  return new NcclComm(nccl_id128, rank, world);
}

int nccl_unique_id(void* out128, const char** err) {
  NcclLib& n = nccl_lib();
  if (!n.ok()) {
    *err = n.err.c_str();
    return 1;
  }
  ncclUniqueId uid;
  const ncclResult_t r = n.GetUniqueId(&uid);
  if (r != ncclSuccess) {
    *err = n.GetErrorString ? n.GetErrorString(r) : "ncclGetUniqueId failed";
    return 1;
  }
  std::memcpy(out128, &uid, sizeof(uid));
  return 0;
}

VGroup* vgroup_create(int device, int world) {
  if (world < 1 || world > kMaxVRanks) throw std::runtime_error("virtual world must be 1..64");
  VGroup* g = new VGroup();
  g->device = device;
  g->world = world;
  g->slots.resize(world);
  g->refs = 1;
  cudaSetDevice(device);
  for (auto& sl : g->slots) {
    if (cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming) != cudaSuccess) {
      vgroup_destroy(g);
      throw std::runtime_error("cudaEventCreate failed");
    }
  }
  if (cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming) != cudaSuccess) {
    vgroup_destroy(g);
    throw std::runtime_error("cudaEventCreate failed");
  }
  return g;
}

namespace {
void vgroup_destroy(VGroup* g) {
  cudaSetDevice(g->device);
  for (auto& sl : g->slots)
    if (sl.ready) cudaEventDestroy(sl.ready);
  if (g->done) cudaEventDestroy(g->done);
  if (g->scratch) cudaFree(g->scratch);
  delete g;
}
}  // namespace

void vgroup_release(VGroup* g) {
  if (!g) return;
  bool last = false;
  {
    std::lock_guard<std::mutex> lk(g->m);
    last = --g->refs == 0;
  }
  if (last) vgroup_destroy(g);
}
int vgroup_world(const VGroup* g) { return g->world; }
int vgroup_device(const VGroup* g) { return g->device; }

Comm* make_virtual_comm(VGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->world) throw std::runtime_error("invalid virtual rank");
  return new VirtualComm(g, rank);
}

}  // namespace gmmb
