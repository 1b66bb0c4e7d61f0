// NCCL entry points resolved at run time (dlopen "libnccl.so.2").
//
// The z-slab exchanges run inside the library on the context's stream (and
// inside its CUDA graphs).  NCCL is resolved at run time rather than linked:
// in a process that already imported torch, dlopen returns torch's bundled
// libnccl.so.2 (one NCCL per process); otherwise the system library.  Only
// the types come from nccl.h.
#include <dlfcn.h>

#include <mutex>
#include <string>

#include "nccl_dyn.h"

namespace pppm {

static NcclApi g_api;
static std::string g_api_err;
static std::once_flag g_once;

template <typename F> static bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

static void load_nccl() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) {
    const char* e = dlerror();
    g_api_err = std::string("libnccl.so.2 not found: ") + (e ? e : "");
    return;
  }
  bool ok = sym(h, "ncclGetUniqueId", g_api.GetUniqueId) && sym(h, "ncclCommInitRank", g_api.CommInitRank) &&
            sym(h, "ncclCommDestroy", g_api.CommDestroy) && sym(h, "ncclCommAbort", g_api.CommAbort) &&
            sym(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError) &&
            sym(h, "ncclGetErrorString", g_api.GetErrorString) && sym(h, "ncclGroupStart", g_api.GroupStart) &&
            sym(h, "ncclGroupEnd", g_api.GroupEnd) && sym(h, "ncclSend", g_api.Send) &&
            sym(h, "ncclRecv", g_api.Recv) && sym(h, "ncclAllReduce", g_api.AllReduce) &&
            sym(h, "ncclGetVersion", g_api.GetVersion);
  if (!ok) {
    g_api_err = "libnccl.so.2 lacks a required entry point";
    return;
  }
  g_api.ok = true;
}

const NcclApi* nccl_api(std::string* err) {
  std::call_once(g_once, load_nccl);
  if (!g_api.ok) {
    if (err) *err = g_api_err;
    return nullptr;
  }
  return &g_api;
}

}  // namespace pppm
