// nccl_dyn.h — NCCL bound at run time with dlopen.  The process may already hold torch's bundled
// libnccl.so.2 (2.28.9); binding to the already-loaded copy (RTLD_NOLOAD first) avoids two NCCL
// instances in one process.  Falls back to the system libnccl.so.2 (2.27.3).  Types come from the
// system nccl.h (ABI-stable for the calls used here).
#pragma once
#include <nccl.h>

#include <string>

namespace irgl {
struct NcclApi {
  bool ok = false;
  std::string path;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
};
// Loads once; returns nullptr (with *why set) if no NCCL could be bound.
const NcclApi* nccl_api(std::string* why);
}  // namespace irgl
