// Transports for the column-sharded multi-GPU solve (comm.cuh).
#include <dlfcn.h>
#include <nccl.h>
#include <cstring>
#include <mutex>
#include <vector>
#include "comm.cuh"

namespace bse {

cudaError_t allgather_cols(Comm& c, double* A, long long ld, long long n, cudaStream_t s) {
  if (c.world <= 1 || n <= 0) return cudaSuccess;
  cudaError_t e = c.group_begin();
  for (int r = 0; r < c.world && e == cudaSuccess; ++r) {
    long long c0, c1;
    shard_range(n, c.world, r, &c0, &c1);
    if (c1 > c0) e = c.bcast(A + c0 * ld, (size_t)((c1 - c0) * ld), r, s);
  }
  cudaError_t e2 = c.group_end(s);
  return e != cudaSuccess ? e : e2;
}

// ---------------------------------------------------------------------------
// NCCL, resolved at run time (the system libnccl.so.2, or the copy torch has
// already loaded under the same soname).

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast &&
             api.AllReduce && api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  cudaError_t check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return cudaSuccess;
    err = std::string(what) + ": " + nccl().GetErrorString(r);
    return cudaErrorUnknown;
  }
  cudaError_t group_begin() override { return check(nccl().GroupStart(), "ncclGroupStart"); }
  cudaError_t bcast(double* p, size_t count, int root, cudaStream_t s) override {
    return check(nccl().Broadcast(p, p, count, ncclFloat64, root, comm, s), "ncclBroadcast");
  }
  cudaError_t group_end(cudaStream_t) override { return check(nccl().GroupEnd(), "ncclGroupEnd"); }
  cudaError_t allreduce_sum(double* p, size_t count, cudaStream_t s) override {
    return check(nccl().AllReduce(p, p, count, ncclFloat64, ncclSum, comm, s), "ncclAllReduce");
  }
};

// Host-staged broadcast: D2H of the root's block, the caller's host
// broadcast, H2D everywhere.  Synchronous with respect to the stream.
struct HostComm final : Comm {
  HostBcastFn fn = nullptr;
  void* ctx = nullptr;
  std::vector<double> buf;
  cudaError_t bcast(double* p, size_t count, int root, cudaStream_t s) override {
    buf.resize(count);
    cudaError_t e;
    if (rank == root) {
      if ((e = cudaMemcpyAsync(buf.data(), p, count * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return e;
    }
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if (fn(ctx, buf.data(), count * 8, root) != 0) {
      err = "host broadcast callback failed";
      return cudaErrorUnknown;
    }
    if (rank != root) {
      if ((e = cudaMemcpyAsync(p, buf.data(), count * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return e;
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  // every rank's block goes round by the host broadcast and is added in rank
  // order, so all ranks form the same bits
  std::vector<double> acc, mine;
  cudaError_t allreduce_sum(double* p, size_t count, cudaStream_t s) override {
    cudaError_t e;
    mine.resize(count);
    acc.assign(count, 0.0);
    if ((e = cudaMemcpyAsync(mine.data(), p, count * 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    for (int r = 0; r < world; ++r) {
      buf.resize(count);
      if (r == rank) std::memcpy(buf.data(), mine.data(), count * 8);
      if (fn(ctx, buf.data(), count * 8, r) != 0) {
        err = "host broadcast callback failed";
        return cudaErrorUnknown;
      }
      for (size_t i = 0; i < count; ++i) acc[i] += buf[i];
    }
    if ((e = cudaMemcpyAsync(p, acc.data(), count * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return e;
    return cudaStreamSynchronize(s);
  }
};

// Measurement-only transport: behaves as rank `rank` of `world` but moves
// nothing (other ranks' column blocks are left as they are).  Lets one GPU
// time exactly the kernels one rank of a P-GPU solve executes.
struct SoloComm final : Comm {
  cudaError_t bcast(double*, size_t, int, cudaStream_t) override { return cudaSuccess; }
  cudaError_t allreduce_sum(double*, size_t, cudaStream_t) override { return cudaSuccess; }
};

}  // namespace

Comm* make_solo_comm(int rank, int world) {
  auto* c = new SoloComm;
  c->rank = rank;
  c->world = world;
  return c;
}

int nccl_unique_id(void* id128, std::string* err) {
  const NcclApi& api = nccl();
  if (!api.ok) { *err = api.why; return 1; }
  ncclUniqueId id;
  ncclResult_t r = api.GetUniqueId(&id);
  if (r != ncclSuccess) { *err = api.GetErrorString(r); return 1; }
  std::memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

Comm* make_nccl_comm(int rank, int world, const void* id128, std::string* err) {
  const NcclApi& api = nccl();
  if (!api.ok) { *err = api.why; return nullptr; }
  ncclUniqueId id;
  std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  auto* c = new NcclComm;
  c->rank = rank;
  c->world = world;
  ncclResult_t r = api.CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    *err = std::string("ncclCommInitRank: ") + api.GetErrorString(r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

Comm* make_host_comm(int rank, int world, HostBcastFn fn, void* ctx) {
  auto* c = new HostComm;
  c->rank = rank;
  c->world = world;
  c->fn = fn;
  c->ctx = ctx;
  return c;
}

}  // namespace bse
