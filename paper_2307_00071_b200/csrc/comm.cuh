// comm.cuh — collectives of the point-sharded fit (one rank per shard).
//
// The reference has no collectives (threads in one process, common.cpp:25-47);
// the sharded fit adds exactly the exchanges SURVEY.md §8(e) names: the
// per-iteration sum of the K x (1 + D + D(D+1)/2) sufficient statistics + ll,
// the per-round k-means++ candidate all-gather, the shard-size exchange and
// the owned-count sum / lowest-index min of the kinit fix-up.
//
// Two implementations of one interface, chosen at context creation:
//  * NcclComm — one process per GPU, NCCL over NVLink (libnccl.so.2 loaded
//    at run time);
//  * VirtualComm — G in-process ranks on ONE device (host thread per rank,
//    each with its own context and stream), the collective computed by a
//    fixed-order device kernel over the ranks' buffers. It runs the exact
//    sharded driver logic without G GPUs (SURVEY.md §4 "virtual-shard mode").
// Every call is collective: all ranks must make the same sequence of calls.
// Operations are enqueued on the caller's stream (no host synchronisation
// beyond what the implementation needs to rendezvous).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace gmmb {

enum class RedOp { kSum, kMin, kMax };
enum class DType { kF64, kI32, kI64 };

class Comm {
 public:
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // in place: buf[0..count) = op over ranks
  virtual cudaError_t allreduce(void* buf, size_t count, DType t, RedOp op,
                                cudaStream_t s) = 0;
  // recv[r * bytes .. (r + 1) * bytes) = rank r's send
  virtual cudaError_t allgather(const void* send, void* recv, size_t bytes,
                                cudaStream_t s) = 0;
  virtual const char* last_error() const = 0;
  // after a failure on this rank: release peers blocked in a collective
  // (virtual ranks; a no-op for NCCL, where validation is agreed up front)
  virtual void abort() {}
};

// NCCL communicator (throws std::runtime_error on failure to create).
Comm* make_nccl_comm(const void* nccl_id128, int rank, int world);
int nccl_unique_id(void* out128, const char** err);

// In-process group of `world` virtual ranks on `device`, reference-counted:
// the creator holds one reference, every virtual comm one more.
struct VGroup;
VGroup* vgroup_create(int device, int world);
void vgroup_release(VGroup* g);
int vgroup_world(const VGroup* g);
int vgroup_device(const VGroup* g);
Comm* make_virtual_comm(VGroup* g, int rank);

}  // namespace gmmb
