// Minimal run-time binding of NCCL (dlopen), so the single-GPU library has no
// link-time NCCL dependency and reuses whichever libnccl.so.2 the process
// already loaded (torch's bundled NCCL when torch.distributed is in use).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

typedef struct ncclComm* ncclComm_t;

namespace nccl {

enum { kUint64 = 5, kDouble = 8 };           // ncclUint64, ncclFloat64
enum { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };  // ncclRedOp_t

struct UniqueId {
  char internal[128];
};

struct Api {
  int (*getUniqueId_)(UniqueId*);
  int (*commInitRank_)(ncclComm_t*, int, UniqueId, int);
  int (*commDestroy_)(ncclComm_t);
  int (*send_)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*recv_)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*groupStart_)();
  int (*groupEnd_)();
  int (*allReduce_)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*allGather_)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);

  int getUniqueId(void* out) { return getUniqueId_(reinterpret_cast<UniqueId*>(out)); }
  int commInitRank(ncclComm_t* c, int n, const void* uid, int r) {
    UniqueId u;
    __builtin_memcpy(&u, uid, sizeof u);
    return commInitRank_(c, n, u, r);
  }
  int commDestroy(ncclComm_t c) { return commDestroy_(c); }
  int send(const void* b, size_t n, int t, int peer, ncclComm_t c, cudaStream_t s) { return send_(b, n, t, peer, c, s); }
  int recv(void* b, size_t n, int t, int peer, ncclComm_t c, cudaStream_t s) { return recv_(b, n, t, peer, c, s); }
  int groupStart() { return groupStart_(); }
  int groupEnd() { return groupEnd_(); }
  int allReduce(const void* a, void* b, size_t n, int t, int op, ncclComm_t c, cudaStream_t s) {
    return allReduce_(a, b, n, t, op, c, s);
  }
  int allGather(const void* a, void* b, size_t n, int t, ncclComm_t c, cudaStream_t s) {
    return allGather_(a, b, n, t, c, s);
  }
};

inline Api* api() {
  static Api a;
  static int state = 0;  // 0 untried, 1 ok, -1 missing
  if (state) return state > 0 ? &a : nullptr;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    state = -1;
    return nullptr;
  }
#define PC_SYM(f, n) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, n))
  PC_SYM(getUniqueId_, "ncclGetUniqueId");
  PC_SYM(commInitRank_, "ncclCommInitRank");
  PC_SYM(commDestroy_, "ncclCommDestroy");
  PC_SYM(send_, "ncclSend");
  PC_SYM(recv_, "ncclRecv");
  PC_SYM(groupStart_, "ncclGroupStart");
  PC_SYM(groupEnd_, "ncclGroupEnd");
  PC_SYM(allReduce_, "ncclAllReduce");
  PC_SYM(allGather_, "ncclAllGather");
#undef PC_SYM
  state = (a.getUniqueId_ && a.commInitRank_ && a.send_ && a.recv_ && a.allReduce_) ? 1 : -1;
  return state > 0 ? &a : nullptr;
}

}  // namespace nccl
