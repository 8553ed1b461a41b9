// nccl_dl.h -- NCCL loaded at run time (dlopen), so libcc.so has no link-time
// dependency on a particular libnccl; the process's already-loaded copy
// (torch's bundled NCCL 2.28) is reused when present.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

struct ncclDevComm;              // nccl_device/core.h (device API, NCCL >= 2.28)
struct ncclDevCommRequirements;

namespace cc {

struct NcclApi {
  bool ok = false;
  const char *why = "not loaded";
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*AlltoAll)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  // device API (NCCL >= 2.28): symmetric windows + device communicator; dev_ok
  // when every entry point below resolved
  bool dev_ok = false;
  ncclResult_t (*MemAlloc)(void **, size_t) = nullptr;
  ncclResult_t (*MemFree)(void *) = nullptr;
  ncclResult_t (*CommWindowRegister)(ncclComm_t, void *, size_t, ncclWindow_t *, int) = nullptr;
  ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
  ncclResult_t (*DevCommCreate)(ncclComm_t, const struct ncclDevCommRequirements *, struct ncclDevComm *) = nullptr;
  ncclResult_t (*DevCommDestroy)(ncclComm_t, const struct ncclDevComm *) = nullptr;
};

NcclApi &nccl();

}  // namespace cc
