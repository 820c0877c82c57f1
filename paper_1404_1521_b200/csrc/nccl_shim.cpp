// nccl_shim.cpp -- see nccl_shim.h.
#include "nccl_shim.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

namespace {
struct Api {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  // symmetric memory (NCCL >= 2.27): optional -- the PEER exchange needs them
  ncclResult_t (*memAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*memFree)(void*) = nullptr;
  ncclResult_t (*winRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*winDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
  struct Team { int nRanks, rank, stride; };   // ncclTeam_t (nccl_device/core.h)
  Team (*teamLsa)(ncclComm_t) = nullptr;
};
Api g_api;
std::once_flag g_once;
std::string g_load_err;

void load() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    // prefer an already-mapped copy (torch's), then the normal search path
    g_api.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!g_api.h) g_api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_api.h) break;
  }
  if (!g_api.h) { g_load_err = std::string("cannot load libnccl.so.2: ") + dlerror(); return; }
  g_api.getUniqueId = (decltype(g_api.getUniqueId))dlsym(g_api.h, "ncclGetUniqueId");
  g_api.commInitRank = (decltype(g_api.commInitRank))dlsym(g_api.h, "ncclCommInitRank");
  g_api.allGather = (decltype(g_api.allGather))dlsym(g_api.h, "ncclAllGather");
  g_api.commDestroy = (decltype(g_api.commDestroy))dlsym(g_api.h, "ncclCommDestroy");
  g_api.groupStart = (decltype(g_api.groupStart))dlsym(g_api.h, "ncclGroupStart");
  g_api.groupEnd = (decltype(g_api.groupEnd))dlsym(g_api.h, "ncclGroupEnd");
  g_api.getErrorString = (decltype(g_api.getErrorString))dlsym(g_api.h, "ncclGetErrorString");
  g_api.allReduce = (decltype(g_api.allReduce))dlsym(g_api.h, "ncclAllReduce");
  g_api.memAlloc = (decltype(g_api.memAlloc))dlsym(g_api.h, "ncclMemAlloc");
  g_api.memFree = (decltype(g_api.memFree))dlsym(g_api.h, "ncclMemFree");
  g_api.winRegister = (decltype(g_api.winRegister))dlsym(g_api.h, "ncclCommWindowRegister");
  g_api.winDeregister = (decltype(g_api.winDeregister))dlsym(g_api.h, "ncclCommWindowDeregister");
  g_api.teamLsa = (decltype(g_api.teamLsa))dlsym(g_api.h, "ncclTeamLsa");
  if (!g_api.getUniqueId || !g_api.commInitRank || !g_api.allGather || !g_api.commDestroy || !g_api.groupStart ||
      !g_api.groupEnd || !g_api.allReduce)
    g_load_err = "libnccl.so.2 lacks required symbols";
}

bool ready(std::string* err) {
  std::call_once(g_once, load);
  if (!g_load_err.empty()) { if (err) *err = g_load_err; return false; }
  return true;
}

int check(ncclResult_t r, const char* what, std::string* err) {
  if (r == ncclSuccess) return 0;
  if (err) *err = std::string(what) + ": " + (g_api.getErrorString ? g_api.getErrorString(r) : "nccl error");
  return 1;
}
}  // namespace

int nccl_shim_unique_id(void* out128, std::string* err) {
  if (!ready(err)) return 1;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  return check(g_api.getUniqueId(reinterpret_cast<ncclUniqueId*>(out128)), "ncclGetUniqueId", err);
}

int nccl_shim_init(void** comm, int rank, int world, const void* uid128, std::string* err) {
  if (!ready(err)) return 1;
  ncclUniqueId id;
  memcpy(&id, uid128, sizeof id);
  ncclComm_t c = nullptr;
  if (check(g_api.commInitRank(&c, world, id, rank), "ncclCommInitRank", err)) return 1;
  *comm = c;
  return 0;
}

int nccl_shim_allgather_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s,
                            std::string* err) {
  if (!ready(err)) return 1;
  return check(g_api.allGather(send, recv, count, ncclFloat32, static_cast<ncclComm_t>(comm), s),
               "ncclAllGather", err);
}

int nccl_shim_destroy(void* comm) {
  if (!comm || !ready(nullptr)) return 1;
  return g_api.commDestroy(static_cast<ncclComm_t>(comm)) != ncclSuccess;
}

int nccl_shim_group(bool start, std::string* err) {
  if (!ready(err)) return 1;
  return check(start ? g_api.groupStart() : g_api.groupEnd(), start ? "ncclGroupStart" : "ncclGroupEnd", err);
}

int nccl_shim_allgather_bytes(const void* send, void* recv, size_t bytes, void* comm, cudaStream_t s,
                              std::string* err) {
  if (!ready(err)) return 1;
  return check(g_api.allGather(send, recv, bytes, ncclChar, static_cast<ncclComm_t>(comm), s), "ncclAllGather", err);
}

int nccl_shim_allreduce_sum_f32(const float* send, float* recv, size_t count, void* comm, cudaStream_t s,
                                std::string* err) {
  if (!ready(err)) return 1;
  return check(g_api.allReduce(send, recv, count, ncclFloat32, ncclSum, static_cast<ncclComm_t>(comm), s),
               "ncclAllReduce", err);
}

bool nccl_shim_has_symmetric() {
  return ready(nullptr) && g_api.memAlloc && g_api.memFree && g_api.winRegister && g_api.winDeregister &&
         g_api.teamLsa;
}

int nccl_shim_lsa_size(void* comm) {
  if (!nccl_shim_has_symmetric()) return 0;
  return g_api.teamLsa(static_cast<ncclComm_t>(comm)).nRanks;
}

int nccl_shim_mem_alloc(void** ptr, size_t bytes, std::string* err) {
  if (!nccl_shim_has_symmetric()) { if (err) *err = "NCCL symmetric memory unavailable"; return 1; }
  return check(g_api.memAlloc(ptr, bytes), "ncclMemAlloc", err);
}

int nccl_shim_mem_free(void* ptr) {
  if (!ptr || !nccl_shim_has_symmetric()) return 1;
  return g_api.memFree(ptr) != ncclSuccess;
}

int nccl_shim_window_register(void* comm, void* buf, size_t bytes, void** win, std::string* err) {
  if (!nccl_shim_has_symmetric()) { if (err) *err = "NCCL symmetric memory unavailable"; return 1; }
  ncclWindow_t w = nullptr;
  if (check(g_api.winRegister(static_cast<ncclComm_t>(comm), buf, bytes, &w, NCCL_WIN_COLL_SYMMETRIC),
            "ncclCommWindowRegister", err))
    return 1;
  *win = w;
  return 0;
}

int nccl_shim_window_deregister(void* comm, void* win) {
  if (!win || !nccl_shim_has_symmetric()) return 1;
  return g_api.winDeregister(static_cast<ncclComm_t>(comm), static_cast<ncclWindow_t>(win)) != ncclSuccess;
}
