// ltb_nccl.cu -- run-time binding of NCCL (see ltb_nccl.h).
#include <dlfcn.h>

#include <mutex>

#include "ltb_nccl.h"

namespace ltb {

namespace {
Nccl g_api;
const Nccl* g_ok = nullptr;
const char* g_why = "NCCL not loaded";
std::once_flag g_once;

template <class F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

void load() {
  // RTLD_NOLOAD first: reuse the copy PyTorch already mapped (one NCCL per process)
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    g_why = "libnccl.so.2 not found";
    return;
  }
  bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) && sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
            sym(h, "ncclCommDestroy", g_api.CommDestroy) && sym(h, "ncclBroadcast", g_api.Broadcast) &&
            sym(h, "ncclAllGather", g_api.AllGather) && sym(h, "ncclSend", g_api.Send) &&
            sym(h, "ncclRecv", g_api.Recv) && sym(h, "ncclGroupStart", g_api.GroupStart) &&
            sym(h, "ncclGroupEnd", g_api.GroupEnd) && sym(h, "ncclGetErrorString", g_api.GetErrorString);
  if (!ok) {
    g_why = "libnccl.so.2 lacks a required symbol";
    return;
  }
  g_ok = &g_api;
}
}  // namespace

const Nccl* nccl_api(const char** why) {
  std::call_once(g_once, load);
  if (!g_ok && why) *why = g_why;
  return g_ok;
}

}  // namespace ltb
