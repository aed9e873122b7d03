#pragma once
#include <nccl.h>

#include <string>

#ifndef RS_NCCL_WHEEL_PATH
#define RS_NCCL_WHEEL_PATH nullptr
#endif

namespace rs {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*ncclGetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*ncclCommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*ncclCommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*ncclCommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*ncclCommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*ncclGetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*ncclAllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
};

// nullptr (and *err set) if NCCL cannot be loaded.
const NcclApi* nccl_api(std::string* err);

}  // namespace rs
