// Communicators for the sharded factorisation.
//
// The exchanges are sums and one gather: the l x l Grams of a row-sharded
// sketch (CholQR), the n x l partials A_g^T Q_g (row shards) or m x l
// partials A_g X_g (column shards), and the all-gather of the local TSQR R
// factors when a sharded sketch needs the Householder fallback.
//
// * NcclComm — production: ncclAllReduce / ncclAllGather on the library's
//   compute stream (stream-ordered with the kernels around them, no host
//   round trip; NVLink/NVSwitch, NVLS when NCCL selects it). NCCL's
//   reductions give bitwise-identical results on every rank, which keeps the
//   replicated QRs and small SVD identical. libnccl is dlopen'ed on first
//   use ("libnccl.so.2": torch's bundled copy when torch already loaded it,
//   else the system one), so single-GPU users need no NCCL at all.
// * HostComm — the caller's own collectives on host copies
//   (xb_comm_init_host): the stream is drained, the operand copied to pinned
//   memory, the callback run, the result copied back. Ranks meet only on the
//   host, so several processes may share one GPU — how the real sharded
//   engine is tested at world size 2 on a single-GPU box.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace xb {
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return;
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(a.h, "ncclCommInitRank"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(a.h, "ncclAllReduce"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(a.h, "ncclAllGather"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.getErrorString =
        reinterpret_cast<decltype(a.getErrorString)>(dlsym(a.h, "ncclGetErrorString"));
  });
  XB_REQUIRE(a.h && a.getUniqueId && a.commInitRank && a.allReduce && a.allGather &&
                 a.commDestroy,
             XB_ENCCL, "NCCL (libnccl.so.2) could not be loaded");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = api().getErrorString ? api().getErrorString(r) : "unknown";
    throw Error(XB_ENCCL, std::string(what) + ": " + msg);
  }
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) api().commDestroy(comm);
  }
  void allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
    if (count) check(api().allReduce(buf, buf, count, ncclDouble, ncclSum, comm, st), "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    if (count) check(api().allGather(send, recv, count, ncclDouble, comm, st), "ncclAllGather");
  }
};

struct HostComm final : Comm {
  xb_host_collective_fn fn = nullptr;
  void* user = nullptr;
  double* stage = nullptr;
  size_t stage_count = 0;
  ~HostComm() override {
    if (stage) cudaFreeHost(stage);
  }
  double* staging(size_t count) {
    if (count > stage_count) {
      if (stage) XB_CUDA(cudaFreeHost(stage));
      XB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stage), count * sizeof(double),
                            cudaHostAllocDefault));
      stage_count = count;
    }
    return stage;
  }
  void call(int op, double* buf, size_t count) {
    const int rc = fn(user, op, buf, (int64_t)count);
    XB_REQUIRE(rc == 0, XB_ENCCL, "host collective callback failed (op " + std::to_string(op) +
                                      ", rc " + std::to_string(rc) + ")");
  }
  void allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
    if (!count) return;
    double* h = staging(count);
    XB_CUDA(cudaMemcpyAsync(h, buf, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    XB_CUDA(cudaStreamSynchronize(st));
    call(XB_COLL_ALLREDUCE_SUM, h, count);
    XB_CUDA(cudaMemcpyAsync(buf, h, count * sizeof(double), cudaMemcpyHostToDevice, st));
    XB_CUDA(cudaStreamSynchronize(st));  // h is reused by the next collective
  }
  void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
    if (!count) return;
    double* h = staging(count * world);
    XB_CUDA(cudaMemcpyAsync(h + (size_t)rank * count, send, count * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    XB_CUDA(cudaStreamSynchronize(st));
    call(XB_COLL_ALLGATHER, h, count);
    XB_CUDA(cudaMemcpyAsync(recv, h, count * world * sizeof(double), cudaMemcpyHostToDevice, st));
    XB_CUDA(cudaStreamSynchronize(st));
  }
};

}  // namespace

void nccl_unique_id(unsigned char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  check(api().getUniqueId(&id), "ncclGetUniqueId");
  memcpy(out, &id, 128);
}

Comm* nccl_comm_create(const unsigned char id_bytes[128], int world, int rank) {
  ncclUniqueId id;
  memcpy(&id, id_bytes, 128);
  auto* c = new NcclComm();
  c->world = world;
  c->rank = rank;
  ncclResult_t r = api().commInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    c->comm = nullptr;
    delete c;
    check(r, "ncclCommInitRank");
  }
  return c;
}

Comm* host_comm_create(int world, int rank, xb_host_collective_fn fn, void* user) {
  XB_REQUIRE(fn != nullptr, XB_EVALUE, "null collective callback");
  auto* c = new HostComm();
  c->world = world;
  c->rank = rank;
  c->fn = fn;
  c->user = user;
  return c;
}

}  // namespace xb
