// NCCL entry points loaded at run time (dlopen), so libsnexec.so has no link
// dependency on a particular libnccl: in a PyTorch process the libnccl.so.2
// torch already loaded is the one used (same soname); SN_NCCL_LIB overrides.
#pragma once
#include <nccl.h>

#include <string>

namespace sndp {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// nullptr (with *err set) when no usable libnccl can be loaded.
const Nccl* nccl(std::string* err);

}  // namespace sndp
