// ltb_nccl.h -- the few NCCL entry points the distributed offline phase
// uses, resolved at run time from the libnccl.so.2 already in the process
// (PyTorch's) or the system one.  libltb.so does not link NCCL: a process
// that never runs a distributed factorisation never loads it.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace ltb {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

// nullptr (with *why set) when no NCCL library can be loaded
const Nccl* nccl_api(const char** why);

}  // namespace ltb
