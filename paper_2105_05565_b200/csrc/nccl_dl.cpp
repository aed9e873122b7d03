// NCCL loaded on demand (dlopen) so that single-GPU use never needs libnccl.  Looks for
// RS_NCCL_LIB, then the libnccl.so.2 shipped next to torch (nvidia/nccl/lib), then the system one.
#include "nccl_dl.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace rs {

static NcclApi g_api;
static std::once_flag g_once;
static std::string g_load_err;

static void* try_open(const char* path) { return path ? dlopen(path, RTLD_NOW | RTLD_GLOBAL) : nullptr; }

static void load() {
  void* h = try_open(std::getenv("RS_NCCL_LIB"));
  if (!h) h = try_open(RS_NCCL_WHEEL_PATH);
  if (!h) h = try_open("libnccl.so.2");
  if (!h) {
    g_load_err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
    return;
  }
#define RS_SYM(name)                                                            \
  g_api.name = reinterpret_cast<decltype(g_api.name)>(dlsym(h, #name));        \
  if (!g_api.name) {                                                            \
    g_load_err = "libnccl missing symbol " #name;                               \
    return;                                                                     \
  }
  RS_SYM(ncclGetUniqueId)
  RS_SYM(ncclCommInitRank)
  RS_SYM(ncclCommDestroy)
  RS_SYM(ncclCommAbort)
  RS_SYM(ncclCommGetAsyncError)
  RS_SYM(ncclGetErrorString)
  RS_SYM(ncclAllReduce)
#undef RS_SYM
  g_api.ok = true;
}

const NcclApi* nccl_api(std::string* err) {
  std::call_once(g_once, load);
  if (!g_api.ok && err) *err = g_load_err;
  return g_api.ok ? &g_api : nullptr;
}

}  // namespace rs
