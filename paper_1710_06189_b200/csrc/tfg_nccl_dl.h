// tfg_nccl_dl.h — NCCL resolved at run time (dlopen, RTLD_LOCAL) on the first
// multi-GPU call, instead of a link-time DT_NEEDED on libnccl.so.2.
//
// Why: a process that maps one libnccl.so.2 keeps it for every later user of
// that soname. Linking the system NCCL (2.27) into libtexforge_cuda.so made a
// later `import torch` bind libtorch_cuda.so to it and fail on a symbol that
// only torch's bundled NCCL (2.28) exports. Resolution order:
//   1. TEXFORGE_NCCL_LIB (the Python binding points it at torch's bundled copy),
//   2. a libnccl.so.2 the process has already mapped (RTLD_NOLOAD),
//   3. libnccl.so.2 from the default search path.
// Only the entry points tfg_multi_gpu.inc uses are wrapped; a missing library
// surfaces as ncclSystemError -> TFG_COLLECTIVE_ERROR, never at load time.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>

namespace tfg_nccl {

struct Api {
  void* h = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

inline const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    if (const char* p = std::getenv("TEXFORGE_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    auto sym = [h](auto& fp, const char* name) { fp = reinterpret_cast<std::decay_t<decltype(fp)>>(dlsym(h, name)); };
    sym(a.get_error_string, "ncclGetErrorString");
    sym(a.comm_init_all, "ncclCommInitAll");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.reduce, "ncclReduce");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    a.h = h;
  });
  return a;
}

#define TFG_NCCL_CALL(field, ...) \
  (api().field ? api().field(__VA_ARGS__) : ncclSystemError)

inline const char* GetErrorString(ncclResult_t r) {
  if (!api().get_error_string) return "NCCL library not found (set TEXFORGE_NCCL_LIB to libnccl.so.2)";
  return api().get_error_string(r);
}
inline ncclResult_t CommInitAll(ncclComm_t* c, int n, const int* devs) { return TFG_NCCL_CALL(comm_init_all, c, n, devs); }
inline ncclResult_t CommInitRank(ncclComm_t* c, int n, ncclUniqueId id, int r) {
  return TFG_NCCL_CALL(comm_init_rank, c, n, id, r);
}
inline ncclResult_t GetUniqueId(ncclUniqueId* id) { return TFG_NCCL_CALL(get_unique_id, id); }
inline ncclResult_t CommDestroy(ncclComm_t c) { return TFG_NCCL_CALL(comm_destroy, c); }
inline ncclResult_t GroupStart() { return TFG_NCCL_CALL(group_start); }
inline ncclResult_t GroupEnd() { return TFG_NCCL_CALL(group_end); }
inline ncclResult_t Reduce(const void* s, void* r, size_t n, ncclDataType_t t, ncclRedOp_t o, int root, ncclComm_t c,
                           cudaStream_t st) {
  return TFG_NCCL_CALL(reduce, s, r, n, t, o, root, c, st);
}
inline ncclResult_t AllReduce(const void* s, void* r, size_t n, ncclDataType_t t, ncclRedOp_t o, ncclComm_t c,
                              cudaStream_t st) {
  return TFG_NCCL_CALL(all_reduce, s, r, n, t, o, c, st);
}
inline ncclResult_t Send(const void* s, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
  return TFG_NCCL_CALL(send, s, n, t, peer, c, st);
}
inline ncclResult_t Recv(void* r, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
  return TFG_NCCL_CALL(recv, r, n, t, peer, c, st);
}
#undef TFG_NCCL_CALL

}  // namespace tfg_nccl
