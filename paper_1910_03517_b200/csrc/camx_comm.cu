// Seam-statistics exchange for camera-sharded arrays: a thin
// binding of the NCCL communicator API, resolved at run time from the
// libnccl.so.2 the process already has loaded (PyTorch's), so the library
// has no link-time NCCL dependency and shares NCCL's version with
// torch.distributed.  The unique id travels between ranks over
// torch.distributed (dist.py); after that every batch's exchange is one
// ncclAllGather issued from C on the caller's stream, between K1 and K2 of
// camx_correct_batch_sharded - no Python on the per-batch path.
#include <dlfcn.h>

#include <condition_variable>
#include <mutex>
#include <set>
#include <vector>

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

// ---- loopback communicator (tests: W ranks inside ONE process on one GPU) --
// NCCL refuses two ranks on one device, so with a single GPU the sharded
// path's world > 1 code (record padding, in-place all-gather, rank-major K2,
// the pipelined step) would never run.  A loopback group is W handles
// driven from W host threads, each rank on its own stream; its all-gather
// moves the bytes through one shared device staging buffer:
//   (a) wait until every rank finished reading the previous call's staging
//   (b) copy send -> staging[rank], record posted[rank]
//   (c) host barrier: every rank has posted
//   (d) wait on every posted[q], copy staging -> recv, record consumed[rank]
//   (e) host barrier: every rank has enqueued its reads (so no rank's next
//       call can re-post before they are ordered)
// Only stream-order waits on events: no kernel ever spins on another rank.
namespace loopback {
struct Group {
  int world = 0, live = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0, status = CAMX_OK;
  uint64_t gen = 0;
  uint8_t *staging = nullptr;
  size_t staging_bytes = 0;
  std::vector<cudaEvent_t> posted, consumed;
};
struct Handle {
  Group *g;
  int rank;
};
std::mutex reg_mu;
std::set<const void *> &registry() {
  static std::set<const void *> r;
  return r;
}
bool is_loopback(const void *h) {
  std::lock_guard<std::mutex> lock(reg_mu);
  return registry().count(h) != 0;
}
// host barrier; `last` runs once, by the last thread to arrive, before the
// others are released
template <class F>
int barrier(Group &g, F last) {
  std::unique_lock<std::mutex> lock(g.mu);
  const uint64_t gen = g.gen;
  if (++g.arrived == g.world) {
    g.status = last();
    g.arrived = 0;
    ++g.gen;
    g.cv.notify_all();
  } else {
    g.cv.wait(lock, [&] { return g.gen != gen; });
  }
  return g.status;  // the last arriver's result, seen by every rank
}
int all_gather(const void *send, void *recv, size_t bytes, Handle &h, cudaStream_t s) {
  Group &g = *h.g;
  const size_t need = bytes * g.world;
  // staging (re)allocation by the last arriver while every rank waits (the
  // first call, or a larger message: cudaFree orders after in-flight reads)
  int st = barrier(g, [&]() -> int {
    if (g.staging_bytes >= need) return CAMX_OK;
    if (g.staging) cudaFree(g.staging);
    g.staging = nullptr;
    g.staging_bytes = 0;
    cudaError_t e = cudaMalloc(&g.staging, need);
    if (e != cudaSuccess) return static_cast<int>(e);
    g.staging_bytes = need;
    return CAMX_OK;
  });
  if (st != CAMX_OK) return st;
  cudaError_t e = cudaSuccess;
  for (int q = 0; e == cudaSuccess && q < g.world; ++q) e = cudaStreamWaitEvent(s, g.consumed[q], 0);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(g.staging + bytes * h.rank, send, bytes, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaEventRecord(g.posted[h.rank], s);
  if (e != cudaSuccess) return static_cast<int>(e);
  barrier(g, [] { return CAMX_OK; });
  for (int q = 0; e == cudaSuccess && q < g.world; ++q) e = cudaStreamWaitEvent(s, g.posted[q], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(recv, g.staging, need, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaEventRecord(g.consumed[h.rank], s);
  if (e != cudaSuccess) return static_cast<int>(e);
  barrier(g, [] { return CAMX_OK; });
  return CAMX_OK;
}
}  // namespace loopback

// Used by camx_correct_batch_sharded (camx_shard.cu).
int comm_all_gather(const void *send, void *recv, size_t bytes, void *comm, cudaStream_t s) {
  if (comm != nullptr && loopback::is_loopback(comm))
    return loopback::all_gather(send, recv, bytes, *static_cast<loopback::Handle *>(comm), s);
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

extern "C" int camx_comm_loopback_create(int32_t world, void **comms_out) {
  if (world < 1 || world > 64 || comms_out == nullptr) return CAMX_EINVAL;
  auto *g = new loopback::Group();
  g->world = g->live = world;
  g->posted.resize(world);
  g->consumed.resize(world);
  for (int r = 0; r < world; ++r) {
    cudaError_t e = cudaEventCreateWithFlags(&g->posted[r], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->consumed[r], cudaEventDisableTiming);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  std::lock_guard<std::mutex> lock(loopback::reg_mu);
  for (int r = 0; r < world; ++r) {
    auto *h = new loopback::Handle{g, r};
    loopback::registry().insert(h);
    comms_out[r] = h;
  }
  return CAMX_OK;
}

extern "C" int camx_comm_destroy(void *comm) {
  if (comm == nullptr) return CAMX_OK;
  if (loopback::is_loopback(comm)) {
    auto *h = static_cast<loopback::Handle *>(comm);
    loopback::Group *g = h->g;
    bool last = false;
    {
      std::lock_guard<std::mutex> lock(loopback::reg_mu);
      loopback::registry().erase(h);
      last = --g->live == 0;
    }
    delete h;
    if (last) {
      cudaDeviceSynchronize();
      if (g->staging) cudaFree(g->staging);
      for (int r = 0; r < g->world; ++r) {
        cudaEventDestroy(g->posted[r]);
        cudaEventDestroy(g->consumed[r]);
      }
      delete g;
    }
    return CAMX_OK;
  }
  const nccl::Api &a = nccl::api();
  if (!a.ok) return CAMX_ENONCCL;
  return nccl::status(a.comm_destroy(comm));
}
