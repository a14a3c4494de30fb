// Host-side TMA descriptor encoding without a link-time libcuda dependency:
// cuTensorMapEncodeTiled is resolved once through the runtime's
// cudaGetDriverEntryPoint, so libbpx.so still loads (and exports its
// symbols) on a machine without the driver -- only a call that needs a
// device fails, with BPX_ERR_INVALID_ARGUMENT from the caller.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

namespace bpx {

inline CUresult encode_tiled(CUtensorMap* map, CUtensorMapDataType dtype, cuuint32_t rank,
                             void* addr, const cuuint64_t* dims, const cuuint64_t* strides,
                             const cuuint32_t* box, const cuuint32_t* estrides,
                             CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                             CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return CUDA_ERROR_NOT_FOUND;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn(map, dtype, rank, addr, dims, strides, box, estrides, il, sw, l2, oob);
}

}  // namespace bpx
