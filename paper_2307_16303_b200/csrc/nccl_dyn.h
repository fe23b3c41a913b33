// NCCL resolved at first use (dlopen), not at link time: a process that also
// runs PyTorch must see ONE libnccl (torch bundles its own, newer than the
// system copy), so an already-loaded libnccl.so.2 is reused (RTLD_NOLOAD)
// before any other is opened. Only the entry points the x all-gather needs.
#pragma once

#include <nccl.h>

namespace h3db {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

// Throws NcclFailure (engine.h) when no libnccl can be loaded.
const NcclApi& nccl();

}  // namespace h3db
