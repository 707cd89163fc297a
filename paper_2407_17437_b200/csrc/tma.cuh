// Tensor Memory Accelerator helpers shared by the TMA kernels (sm_100a):
// the driver's tensor-map encoder and the PTX wrappers for mbarriers and
// bulk tensor copies.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace smb {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// cuTensorMapEncodeTiled (null when the driver does not provide it)
EncodeTiledFn encode_fn();

}  // namespace smb
