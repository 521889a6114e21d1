// NCCL for multi-GPU chains, loaded with dlopen on first use so that single-GPU use never needs it.
// libnccl.so.2 is the one PyTorch ships (already loaded in a torch process; the same soname resolves to it).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "mabd_plan.h"

namespace mabd {

namespace {
// minimal ABI subset of nccl.h (2.x): opaque comm, 128-byte unique id, enums as int
typedef struct {
  char internal[128];
} UniqueId;
typedef void* Comm;
enum { kNcclDouble = 8 };  // ncclFloat64
typedef int (*GetUniqueIdFn)(UniqueId*);
typedef int (*CommInitRankFn)(Comm*, int, UniqueId, int);
typedef int (*AllGatherFn)(const void*, void*, size_t, int, Comm, cudaStream_t);
typedef int (*BroadcastFn)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*GroupFn)();
typedef int (*CommDestroyFn)(Comm);
typedef const char* (*ErrStrFn)(int);

struct Api {
  void* h = nullptr;
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  AllGatherFn all_gather = nullptr;
  BroadcastFn broadcast = nullptr;
  GroupFn group_start = nullptr, group_end = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  ErrStrFn err_str = nullptr;
} g_api;
std::mutex g_mu;
thread_local int g_step_rc = 0;  // first NCCL failure inside a step's launch sequence (nccl_take_step_error)
}  // namespace

int nccl_step_failed(int rc) {
  if (rc != 0 && g_step_rc == 0) g_step_rc = rc;
  return rc;
}
int nccl_take_step_error() {
  const int rc = g_step_rc;
  g_step_rc = 0;
  return rc;
}

bool nccl_load(std::string* err) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_api.h) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    if (err) *err = std::string("dlopen(libnccl.so.2): ") + dlerror();
    return false;
  }
  Api a;
  a.h = h;
  a.get_unique_id = (GetUniqueIdFn)dlsym(h, "ncclGetUniqueId");
  a.comm_init_rank = (CommInitRankFn)dlsym(h, "ncclCommInitRank");
  a.all_gather = (AllGatherFn)dlsym(h, "ncclAllGather");
  a.broadcast = (BroadcastFn)dlsym(h, "ncclBroadcast");
  a.group_start = (GroupFn)dlsym(h, "ncclGroupStart");
  a.group_end = (GroupFn)dlsym(h, "ncclGroupEnd");
  a.comm_destroy = (CommDestroyFn)dlsym(h, "ncclCommDestroy");
  a.err_str = (ErrStrFn)dlsym(h, "ncclGetErrorString");
  if (!a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.broadcast || !a.group_start || !a.group_end ||
      !a.comm_destroy) {
    if (err) *err = "libnccl.so.2 lacks a required symbol";
    return false;
  }
  g_api = a;
  return true;
}

int nccl_unique_id(void* out128) {
  if (!nccl_load(nullptr)) return -1;
  UniqueId id;
  const int rc = g_api.get_unique_id(&id);
  if (rc == 0) memcpy(out128, &id, sizeof(id));
  return rc;
}

int nccl_comm_init(void** comm, int world, const void* id128, int rank) {
  if (!nccl_load(nullptr)) return -1;
  UniqueId id;
  memcpy(&id, id128, sizeof(id));
  Comm c = nullptr;
  const int rc = g_api.comm_init_rank(&c, world, id, rank);
  *comm = c;
  return rc;
}

// in-place all-gather: rank r's block of count_per_rank doubles sits at buf + r·count
int nccl_allgather_doubles(void* comm, double* buf, size_t count, int rank, cudaStream_t st) {
  return g_api.all_gather(buf + (size_t)rank * count, buf, count, kNcclDouble, (Comm)comm, st);
}

// every rank broadcasts its own position range of each of ncomp SoA rows (rows of stride ld)
int nccl_bcast_ranges(void* comm, double* base, const std::vector<std::pair<int64_t, int64_t>>& ranges, int64_t ld,
                      int ncomp, cudaStream_t st) {
  int rc = g_api.group_start();
  for (int c = 0; c < ncomp && rc == 0; ++c)
    for (int r = 0; r < (int)ranges.size() && rc == 0; ++r) {
      const int64_t lo = ranges[r].first, hi = ranges[r].second;
      if (hi <= lo) continue;
      double* p = base + c * ld + lo;
      rc = g_api.broadcast(p, p, (size_t)(hi - lo), kNcclDouble, r, (Comm)comm, st);
    }
  const int rc2 = g_api.group_end();
  return rc ? rc : rc2;
}

void nccl_comm_destroy(void* comm) {
  if (comm && g_api.comm_destroy) g_api.comm_destroy((Comm)comm);
}

const char* nccl_err(int code) { return g_api.err_str ? g_api.err_str(code) : "NCCL error"; }

}  // namespace mabd
