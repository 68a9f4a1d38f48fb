// nccl_dyn.cpp — see nccl_dyn.h.
#include "nccl_dyn.h"

#include <dlfcn.h>

#include <mutex>

namespace irgl {
namespace {
NcclApi g_api;
std::once_flag g_once;
std::string g_why;

template <class F>
bool bind(void* h, const char* name, F& fn) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  return fn != nullptr;
}

void load() {
  const char* cands[] = {"libnccl.so.2", "libnccl.so",
                         "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
  void* h = nullptr;
  for (const char* c : cands) {  // prefer a copy already mapped into the process (torch's)
    h = dlopen(c, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (h) { g_api.path = c; break; }
  }
  if (!h)
    for (const char* c : cands) {
      h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
      if (h) { g_api.path = c; break; }
    }
  if (!h) {
    g_why = std::string("E_NCCL: cannot dlopen libnccl.so.2: ") + (dlerror() ? dlerror() : "?");
    return;
  }
  bool ok = bind(h, "ncclGetUniqueId", g_api.GetUniqueId) &&
            bind(h, "ncclCommInitRank", g_api.CommInitRank) &&
            bind(h, "ncclCommDestroy", g_api.CommDestroy) &&
            bind(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError) &&
            bind(h, "ncclGetErrorString", g_api.GetErrorString) &&
            bind(h, "ncclGroupStart", g_api.GroupStart) && bind(h, "ncclGroupEnd", g_api.GroupEnd) &&
            bind(h, "ncclSend", g_api.Send) && bind(h, "ncclRecv", g_api.Recv) &&
            bind(h, "ncclAllReduce", g_api.AllReduce) && bind(h, "ncclAllGather", g_api.AllGather);
  if (!ok) {
    g_why = "E_NCCL: libnccl is missing a required symbol";
    return;
  }
  g_api.ok = true;
}
}  // namespace

const NcclApi* nccl_api(std::string* why) {
  std::call_once(g_once, load);
  if (!g_api.ok) {
    if (why) *why = g_why;
    return nullptr;
  }
  return &g_api;
}
}  // namespace irgl
