// Host-side TMA descriptor construction (driver entry point, no -lcuda).
#include "tma.cuh"

namespace sdmp {

int make_tmap_3d(CUtensorMap* map, const float* base, const int64_t full[3], int bz, int by,
                 bool evict_first) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    SDMP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode,
                                      cudaEnableDefault, &q));
    SDMP_CHECK(encode && q == cudaDriverEntryPointSuccess, "cuTensorMapEncodeTiled unavailable");
  }
  SDMP_CHECK(((uintptr_t)base & 15) == 0, "TMA base must be 16-byte aligned");
  SDMP_CHECK(full[2] % 4 == 0, "TMA needs the FULL z extent to be a multiple of 4");
  cuuint64_t dims[3] = {(cuuint64_t)full[2], (cuuint64_t)full[1], (cuuint64_t)full[0]};
  cuuint64_t strides[2] = {(cuuint64_t)full[2] * 4, (cuuint64_t)(full[1] * full[2] * 4)};
  cuuint32_t box[3] = {(cuuint32_t)bz, (cuuint32_t)by, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      evict_first ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                  : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SDMP_ECUDA;
  }
  return SDMP_OK;
}

}  // namespace sdmp
