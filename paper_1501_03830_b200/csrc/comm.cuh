// Multi-GPU plumbing for the column-sharded solve.
//
// One process per GPU.  The only exchanges on the path are broadcasts of a
// rank's column block to every other rank (the congruence W = L^T M L and the
// recovered X1/X2), issued as one NCCL group of per-root broadcasts on the
// solve stream so every block moves concurrently over NVLink/NVSwitch.
//
// Two transports implement the same Comm:
//  * NcclComm: libnccl (dlopen'ed, so the library loads without it), one
//    communicator per process, collectives ordered on the solve stream;
//  * HostComm: host-staged broadcast through a caller callback (a gloo
//    process group in the tests) -- lets two ranks share one GPU without any
//    kernel waiting on another rank's kernel.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <string>

namespace bse {

struct Comm {
  int rank = 0;
  int world = 1;
  virtual ~Comm() = default;
  // Broadcast `count` doubles at dptr from `root` (in place) on stream s.
  // Calls between group_begin/group_end may be fused by the transport.
  virtual cudaError_t group_begin() { return cudaSuccess; }
  virtual cudaError_t bcast(double* dptr, size_t count, int root, cudaStream_t s) = 0;
  virtual cudaError_t group_end(cudaStream_t s) { (void)s; return cudaSuccess; }
  // Sum of `count` doubles at dptr over all ranks, in place, the same bits on
  // every rank (panel products of the distributed band reduction, gathers of
  // disjoint pieces padded with zeros).
  virtual cudaError_t allreduce_sum(double* dptr, size_t count, cudaStream_t s) = 0;
  virtual std::string error() const { return err; }
  std::string err;
};

// Contiguous column block of `rank` among `world` ranks: [c0, c1).
inline void shard_range(long long n, int world, int rank, long long* c0, long long* c1) {
  *c0 = n * rank / world;
  *c1 = n * (rank + 1) / world;
}

// Every rank's column block [c0_r, c1_r) of the n-column matrix A (ld) is
// broadcast from r: afterwards all ranks hold all n columns.
cudaError_t allgather_cols(Comm& c, double* A, long long ld, long long n, cudaStream_t s);

// NCCL transport.  id128: ncclUniqueId bytes from nccl_unique_id() on rank 0.
Comm* make_nccl_comm(int rank, int world, const void* id128, std::string* err);
int nccl_unique_id(void* id128, std::string* err);

// Host-staged transport: fn(ctx, host_buf, bytes, root) must broadcast the
// host buffer from root to every rank and return 0 on success.
typedef int (*HostBcastFn)(void* ctx, void* host_buf, size_t bytes, int root);
Comm* make_host_comm(int rank, int world, HostBcastFn fn, void* ctx);

// Measurement-only: rank `rank` of `world` with no data movement.
Comm* make_solo_comm(int rank, int world);

}  // namespace bse
