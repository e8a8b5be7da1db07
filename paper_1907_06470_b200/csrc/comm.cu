// NCCL communicator for the row-sharded factorisation.
//
// A's rows are split over the ranks (one process per GPU). The only
// exchanges are sums: the l x l Gram of a row-sharded sketch (CholQR) and the
// n x l partial products A_g^T Q_g. Both are ncclAllReduce(sum) on the
// library's compute stream, so they are stream-ordered with the kernels
// around them; NCCL's reductions give bitwise-identical results on every
// rank, which keeps the replicated n-side QR and small SVD identical.
//
// NCCL is dlopen'ed on first use ("libnccl.so.2": torch's bundled copy when
// torch already loaded it, else the system one), so single-GPU users need no
// NCCL at all.
#include <dlfcn.h>
#include <nccl.h>

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
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.getErrorString =
        reinterpret_cast<decltype(a.getErrorString)>(dlsym(a.h, "ncclGetErrorString"));
  });
  XB_REQUIRE(a.h && a.getUniqueId && a.commInitRank && a.allReduce && a.commDestroy, XB_ENCCL,
             "NCCL (libnccl.so.2) could not be loaded");
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = api().getErrorString ? api().getErrorString(r) : "unknown";
    throw Error(XB_ENCCL, std::string(what) + ": " + msg);
  }
}

}  // namespace

void nccl_unique_id(unsigned char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  check(api().getUniqueId(&id), "ncclGetUniqueId");
  memcpy(out, &id, 128);
}

void* nccl_comm_init(const unsigned char id_bytes[128], int world, int rank) {
  ncclUniqueId id;
  memcpy(&id, id_bytes, 128);
  ncclComm_t comm = nullptr;
  check(api().commInitRank(&comm, world, id, rank), "ncclCommInitRank");
  return comm;
}

void nccl_comm_destroy(void* comm) {
  if (comm) api().commDestroy(static_cast<ncclComm_t>(comm));
}

void nccl_allreduce_sum(void* comm, double* buf, size_t count, cudaStream_t st) {
  check(api().allReduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), st),
        "ncclAllReduce");
}

}  // namespace xb
