// NCCL for the E1 sharded path (include/hyde.h
// hyde_hyres_sharded), resolved at run time: the libnccl.so.2 already in the
// process (PyTorch's) is reused when present, so one NCCL serves both the
// caller's process group and the library; a process without NCCL keeps every
// single-GPU entry point (the sharded call then returns HYDE_ENCCL).
#include "nccl_shim.h"

#include <dlfcn.h>

#include <mutex>

namespace {
NcclApi g_api;
bool g_tried = false;
std::mutex g_mu;

template <typename F>
bool sym(void* lib, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(lib, name));
  return out != nullptr;
}
}  // namespace

const NcclApi* nccl_api() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_tried) return g_api.ok ? &g_api : nullptr;
  g_tried = true;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return nullptr;
  bool ok = sym(lib, "ncclGetVersion", g_api.GetVersion) && sym(lib, "ncclGetUniqueId", g_api.GetUniqueId) &&
            sym(lib, "ncclCommInitRank", g_api.CommInitRank) && sym(lib, "ncclCommDestroy", g_api.CommDestroy) &&
            sym(lib, "ncclCommCount", g_api.CommCount) && sym(lib, "ncclCommUserRank", g_api.CommUserRank) &&
            sym(lib, "ncclAllReduce", g_api.AllReduce) && sym(lib, "ncclSend", g_api.Send) &&
            sym(lib, "ncclRecv", g_api.Recv) && sym(lib, "ncclGroupStart", g_api.GroupStart) &&
            sym(lib, "ncclGroupEnd", g_api.GroupEnd) && sym(lib, "ncclGetErrorString", g_api.GetErrorString);
  g_api.ok = ok;
  return ok ? &g_api : nullptr;
}
