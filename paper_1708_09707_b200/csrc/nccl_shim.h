// nccl_shim.h -- NCCL resolved at run time (dlopen), not at link time.
//
// The engine only needs NCCL for the y allgather of row-sliced products.  Linking
// libnccl.so.2 directly would pin whichever copy the dynamic loader finds first; a
// process that later imports torch (which ships its own, newer libnccl.so.2) would then
// bind torch to the older copy.  Resolving the handful of entry points lazily, and
// preferring an already-loaded libnccl (RTLD_NOLOAD), keeps exactly one NCCL per process.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include "common.cuh"

namespace hmb {

struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;

  static const NcclApi& get() {
    static NcclApi api = load();
    if (!api.GetUniqueId) raise(kEnccl, "libnccl.so.2 could not be loaded");
    return api;
  }

 private:
  static NcclApi load() {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(dlsym(h, "ncclBroadcast"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    if (!a.CommInitRank || !a.CommDestroy || !a.GroupStart || !a.GroupEnd || !a.Broadcast || !a.AllGather)
      a.GetUniqueId = nullptr;
    return a;
  }
};

}  // namespace hmb
