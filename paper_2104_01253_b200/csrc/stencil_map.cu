// Host side of the TMA-staged stencil (stencil_tma.cuh): the 3-D tensor map
// of a rank's grid block, encoded through the driver entry point
// cuTensorMapEncodeTiled (no libcuda link needed) and cached per operand.
#include "stencil_tma.cuh"

namespace kls {
bool stencil7_tensor_map(const double* x, int64_t nx, int64_t ny, int64_t nz, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (encode == nullptr || nx > INT32_MAX) return false;
  struct Entry {
    const double* x;
    int64_t nx, ny, nz;
    CUtensorMap map;
  };
  static thread_local Entry cache[8];
  static thread_local int next = 0;
  for (auto& e : cache)
    if (e.x == x && e.nx == nx && e.ny == ny && e.nz == nz) {
      *map = e.map;
      return true;
    }
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(nz), static_cast<cuuint64_t>(ny),
                              static_cast<cuuint64_t>(nx)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(nz) * sizeof(double),
                                 static_cast<cuuint64_t>(ny * nz) * sizeof(double)};
  const cuuint32_t box[3] = {kRowD, kRowsS, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(x), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[next] = Entry{x, nx, ny, nz, *map};
  next = (next + 1) % 8;
  return true;
}
}  // namespace kls
