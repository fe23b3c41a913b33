#include "nccl_dyn.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "engine.h"

namespace h3db {

namespace {

void* open_nccl() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names)
    if (void* h = dlopen(n, RTLD_NOW | RTLD_NOLOAD)) return h;  // already in the process
  for (const char* n : names)
    if (void* h = dlopen(n, RTLD_NOW | RTLD_GLOBAL)) return h;
  return nullptr;
}

template <class F>
void bind(void* h, F& fn, const char* sym) {
  fn = reinterpret_cast<F>(dlsym(h, sym));
  if (!fn) throw NcclFailure(std::string("libnccl lacks ") + sym);
}

}  // namespace

const NcclApi& nccl() {
  static NcclApi api{};
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = open_nccl();
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    try {
      bind(h, api.GetUniqueId, "ncclGetUniqueId");
      bind(h, api.CommInitRank, "ncclCommInitRank");
      bind(h, api.CommDestroy, "ncclCommDestroy");
      bind(h, api.GroupStart, "ncclGroupStart");
      bind(h, api.GroupEnd, "ncclGroupEnd");
      bind(h, api.Broadcast, "ncclBroadcast");
      bind(h, api.GetErrorString, "ncclGetErrorString");
    } catch (const NcclFailure& e) {
      err = e.what();
    }
  });
  if (!err.empty()) throw NcclFailure(err);
  return api;
}

}  // namespace h3db
