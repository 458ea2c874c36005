// Seam-statistics exchange for camera-sharded arrays: a thin
// binding of the NCCL communicator API, resolved at run time from the
// libnccl.so.2 the process already has loaded (PyTorch's), so the library
// has no link-time NCCL dependency and shares NCCL's version with
// torch.distributed.  The unique id travels between ranks over
// torch.distributed (dist.py); after that every batch's exchange is one
// ncclAllGather issued from C on the caller's stream, between K1 and K2 of
// camx_correct_batch_sharded - no Python on the per-batch path.
#include <dlfcn.h>

#include <mutex>

#include "camx_common.cuh"

namespace camx {

namespace nccl {
// ABI subset of nccl.h (stable across NCCL 2.x).
constexpr int kUniqueIdBytes = 128;
struct UniqueId {
  char internal[kUniqueIdBytes];
};
using Comm = void *;
using Result = int;       // ncclResult_t: 0 = ncclSuccess
constexpr int kUint8 = 1;  // ncclDataType_t ncclUint8

using GetUniqueIdFn = Result (*)(UniqueId *);
using CommInitRankFn = Result (*)(Comm *, int, UniqueId, int);
using AllGatherFn = Result (*)(const void *, void *, size_t, int, Comm, cudaStream_t);
using CommDestroyFn = Result (*)(Comm);
using GetErrorStringFn = const char *(*)(Result);

struct Api {
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  AllGatherFn all_gather = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  GetErrorStringFn error_string = nullptr;
  bool ok = false;
};

const Api &api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    a.get_unique_id = reinterpret_cast<GetUniqueIdFn>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<CommInitRankFn>(dlsym(h, "ncclCommInitRank"));
    a.all_gather = reinterpret_cast<AllGatherFn>(dlsym(h, "ncclAllGather"));
    a.comm_destroy = reinterpret_cast<CommDestroyFn>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<GetErrorStringFn>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_gather && a.comm_destroy;
  });
  return a;
}

int status(Result r) { return r == 0 ? CAMX_OK : CAMX_ENCCL_BASE + r; }
}  // namespace nccl

// Used by camx_correct_batch_sharded (camx_apply.cu).
int comm_all_gather(const void *send, void *recv, size_t bytes, void *comm, cudaStream_t s) {
  const nccl::Api &a = nccl::api();
  if (!a.ok) return CAMX_ENONCCL;
  return nccl::status(a.all_gather(send, recv, bytes, nccl::kUint8, comm, s));
}

const char *nccl_error_string(int r) {
  const nccl::Api &a = nccl::api();
  return (a.ok && a.error_string) ? a.error_string(r) : "NCCL error";
}

}  // namespace camx

using namespace camx;

extern "C" int camx_comm_available(void) { return nccl::api().ok ? 1 : 0; }

extern "C" int camx_comm_unique_id(uint8_t *id_out) {
  if (id_out == nullptr) return CAMX_EINVAL;
  const nccl::Api &a = nccl::api();
  if (!a.ok) return CAMX_ENONCCL;
  nccl::UniqueId id;
  const int st = nccl::status(a.get_unique_id(&id));
  if (st != CAMX_OK) return st;
  memcpy(id_out, id.internal, nccl::kUniqueIdBytes);
  return CAMX_OK;
}

extern "C" int camx_comm_init(void **comm_out, const uint8_t *id, int32_t n_ranks,
                              int32_t rank) {
  if (comm_out == nullptr || id == nullptr || n_ranks < 1 || rank < 0 || rank >= n_ranks)
    return CAMX_EINVAL;
  const nccl::Api &a = nccl::api();
  if (!a.ok) return CAMX_ENONCCL;
  nccl::UniqueId uid;
  memcpy(uid.internal, id, nccl::kUniqueIdBytes);
  nccl::Comm c = nullptr;
  const int st = nccl::status(a.comm_init_rank(&c, n_ranks, uid, rank));
  if (st != CAMX_OK) return st;
  *comm_out = c;
  return CAMX_OK;
}

extern "C" int camx_comm_destroy(void *comm) {
  if (comm == nullptr) return CAMX_OK;
  const nccl::Api &a = nccl::api();
  if (!a.ok) return CAMX_ENONCCL;
  return nccl::status(a.comm_destroy(comm));
}
