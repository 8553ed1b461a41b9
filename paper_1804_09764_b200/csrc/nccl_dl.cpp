// nccl_dl.cpp -- dlopen/dlsym of the NCCL entry points used by the halo
// exchange (grouped ncclSend/ncclRecv, ncclAlltoAll, the device API's
// symmetric windows) and the final 1-double all-reduce.
#include "nccl_dl.h"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

namespace cc {

namespace {
template <typename F>
bool sym(void *h, const char *name, F &out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}
}  // namespace

NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = nullptr;
    if (const char *p = std::getenv("CC_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = "libnccl.so.2 not found (set CC_NCCL_LIB)";
      return;
    }
    bool ok = sym(h, "ncclGetUniqueId", api.GetUniqueId) && sym(h, "ncclCommInitRank", api.CommInitRank) &&
              sym(h, "ncclCommDestroy", api.CommDestroy) &&
              sym(h, "ncclCommGetAsyncError", api.CommGetAsyncError) && sym(h, "ncclSend", api.Send) &&
              sym(h, "ncclRecv", api.Recv) && sym(h, "ncclGroupStart", api.GroupStart) &&
              sym(h, "ncclGroupEnd", api.GroupEnd) && sym(h, "ncclAllReduce", api.AllReduce) &&
              sym(h, "ncclGetErrorString", api.GetErrorString);
    sym(h, "ncclAlltoAll", api.AlltoAll);
    api.dev_ok = sym(h, "ncclMemAlloc", api.MemAlloc) && sym(h, "ncclMemFree", api.MemFree) &&
                 sym(h, "ncclCommWindowRegister", api.CommWindowRegister) &&
                 sym(h, "ncclCommWindowDeregister", api.CommWindowDeregister) &&
                 sym(h, "ncclDevCommCreate", api.DevCommCreate) && sym(h, "ncclDevCommDestroy", api.DevCommDestroy);
    api.ok = ok;
    api.why = ok ? "" : "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

}  // namespace cc
