// nccl_dl.h -- NCCL resolved at run time (dlopen/dlsym), so libmrfnufft.so has no link-time NCCL
// dependency and uses the NCCL already loaded into the process (PyTorch's) when there is one.
#pragma once
#include <cuda_runtime.h>

namespace mrf {

typedef struct { char internal[128]; } NcclUniqueId;
typedef void* NcclComm;
enum { kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0 };

struct NcclApi {
  int (*GetUniqueId)(NcclUniqueId*);
  int (*CommInitRank)(NcclComm*, int, NcclUniqueId, int);
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
  int (*CommDestroy)(NcclComm);
  const char* (*GetErrorString)(int);
};

// Returns nullptr (and a message in *why) when NCCL cannot be loaded.
const NcclApi* nccl_api(const char** why);

}  // namespace mrf
