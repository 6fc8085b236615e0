// nccl_dl.cpp -- run-time NCCL binding (see nccl_dl.h).
#include "nccl_dl.h"

#include <dlfcn.h>

#include <mutex>

namespace mrf {

namespace {
NcclApi g_api;
bool g_ok = false;
const char* g_why = "NCCL not loaded";
std::once_flag g_once;

void load() {
  // Prefer a libnccl already mapped into the process (e.g. by torch.distributed).
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { g_why = "dlopen(libnccl.so.2) failed"; return; }
  g_api.GetUniqueId = (int (*)(NcclUniqueId*))dlsym(h, "ncclGetUniqueId");
  g_api.CommInitRank = (int (*)(NcclComm*, int, NcclUniqueId, int))dlsym(h, "ncclCommInitRank");
  g_api.AllReduce = (int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t))dlsym(h, "ncclAllReduce");
  g_api.CommDestroy = (int (*)(NcclComm))dlsym(h, "ncclCommDestroy");
  g_api.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  if (!g_api.GetUniqueId || !g_api.CommInitRank || !g_api.AllReduce || !g_api.CommDestroy || !g_api.GetErrorString) {
    g_why = "libnccl is missing required symbols";
    return;
  }
  g_ok = true;
}
}  // namespace

const NcclApi* nccl_api(const char** why) {
  std::call_once(g_once, load);
  if (!g_ok) {
    if (why) *why = g_why;
    return nullptr;
  }
  return &g_api;
}

}  // namespace mrf
