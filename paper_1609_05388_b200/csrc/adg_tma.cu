// adg_tma.cu -- cuTensorMapEncodeTiled through the runtime's driver entry
// point (no link-time dependency on libcuda).
#include "adg_tma.cuh"

#include <cudaTypedefs.h>

#include <mutex>

namespace adg {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) fail(ADG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_tensor_map_2d(const void* base, CUtensorMapDataType elem, uint64_t inner,
                               uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                               uint32_t box_outer, CUtensorMapSwizzle swizzle) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult rc = encode_fn()(&m, elem, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS)
    fail(ADG_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)rc));
  return m;
}

}  // namespace adg
