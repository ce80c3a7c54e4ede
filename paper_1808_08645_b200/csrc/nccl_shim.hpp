// Minimal run-time binding to NCCL (dlopen), so that libbbwadg.so loads and runs
// single-GPU without NCCL and reuses the libnccl.so.2 that torch already mapped
// (NCCL 2.28 from the nvidia-nccl wheel) for multi-GPU runs.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

namespace bbw {
namespace nccl {

typedef void* Comm;
enum { kFloat = 7, kDouble = 8 };  // ncclFloat32, ncclFloat64
struct UniqueId { char internal[128]; };

typedef int (*GetUniqueIdFn)(UniqueId*);
typedef int (*CommInitRankFn)(Comm*, int, UniqueId, int);
typedef int (*CommDestroyFn)(Comm);
typedef int (*SendFn)(const void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*RecvFn)(void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*GroupFn)();
typedef const char* (*LastErrorFn)(Comm);
typedef int (*AsyncErrorFn)(Comm, int*);

struct Api {
  void* handle = nullptr;
  GetUniqueIdFn getUniqueId = nullptr;
  CommInitRankFn commInitRank = nullptr;
  CommDestroyFn commDestroy = nullptr;
  SendFn send = nullptr;
  RecvFn recv = nullptr;
  GroupFn groupStart = nullptr, groupEnd = nullptr;
  LastErrorFn lastError = nullptr;
  AsyncErrorFn asyncError = nullptr;
};

inline Api& api() {
  static Api a;
  return a;
}

inline bool load(std::string& why) {
  Api& a = api();
  if (a.handle) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    a.handle = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // already loaded by torch?
    if (a.handle) break;
  }
  if (!a.handle) {
    const char* env = getenv("BBWADG_NCCL_LIB");
    if (env) a.handle = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!a.handle) a.handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!a.handle) {
    why = std::string("cannot load libnccl.so.2: ") + dlerror();
    return false;
  }
  a.getUniqueId = (GetUniqueIdFn)dlsym(a.handle, "ncclGetUniqueId");
  a.commInitRank = (CommInitRankFn)dlsym(a.handle, "ncclCommInitRank");
  a.commDestroy = (CommDestroyFn)dlsym(a.handle, "ncclCommDestroy");
  a.send = (SendFn)dlsym(a.handle, "ncclSend");
  a.recv = (RecvFn)dlsym(a.handle, "ncclRecv");
  a.groupStart = (GroupFn)dlsym(a.handle, "ncclGroupStart");
  a.groupEnd = (GroupFn)dlsym(a.handle, "ncclGroupEnd");
  a.lastError = (LastErrorFn)dlsym(a.handle, "ncclGetLastError");
  a.asyncError = (AsyncErrorFn)dlsym(a.handle, "ncclCommGetAsyncError");
  if (!a.getUniqueId || !a.commInitRank || !a.send || !a.recv || !a.groupStart || !a.groupEnd) {
    why = "libnccl.so.2 lacks required symbols";
    return false;
  }
  return true;
}

inline int get_unique_id(void* out) {
  UniqueId id;
  int r = api().getUniqueId(&id);
  memcpy(out, &id, sizeof(id));
  return r;
}
inline int comm_init_rank(Comm* c, int n, const void* id, int rank) {
  UniqueId u;
  memcpy(&u, id, sizeof(u));
  return api().commInitRank(c, n, u, rank);
}
inline int comm_destroy(Comm c) { return api().commDestroy ? api().commDestroy(c) : 0; }
inline int send(const void* b, size_t n, int dt, int peer, Comm c, cudaStream_t s) { return api().send(b, n, dt, peer, c, s); }
inline int recv(void* b, size_t n, int dt, int peer, Comm c, cudaStream_t s) { return api().recv(b, n, dt, peer, c, s); }
inline int group_start() { return api().groupStart(); }
inline int group_end() { return api().groupEnd(); }
inline const char* last_error(Comm c) { return api().lastError ? api().lastError(c) : ""; }
// ncclCommGetAsyncError: 0 = ncclSuccess, 7 = ncclInProgress (non-blocking init), else a failure
inline int async_error(Comm c) {
  int e = 0;
  if (!api().asyncError || api().asyncError(c, &e) != 0) return 0;
  return e;
}

}  // namespace nccl
}  // namespace bbw
