// Probe: which rank-1 tensor-map encodings does the driver accept (run on the GPU box).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  printf("fn %p q %d\n", fn, (int)q);
  void* buf;
  cudaMalloc(&buf, 1 << 24);
  alignas(64) CUtensorMap m;
  cuuint64_t strides[1] = {16};
  for (int t = 0; t < 2; ++t)
    for (int nullstr = 0; nullstr < 2; ++nullstr)
      for (int l2 = 0; l2 < 2; ++l2) {
        CUtensorMapDataType ty = t ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
        cuuint64_t dims[1] = {t ? 100000ull : 100000ull};
        cuuint32_t box[1] = {t ? 198u : 80u}, es[1] = {1};
        CUresult r = enc(&m, ty, 1, buf, dims, nullstr ? nullptr : strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("type %s nullstrides %d l2 %d -> %d\n", t ? "f64" : "u8", nullstr, l2, (int)r);
      }
  // odd sizes / small dims
  cuuint32_t es[1] = {1};
  for (cuuint64_t d : {64ull, 79ull, 80ull, 81ull, 2146689ull}) {
    cuuint64_t dims[1] = {d};
    cuuint32_t box[1] = {80};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("u8 dim %llu box 80 -> %d\n", (unsigned long long)d, (int)r);
  }
  for (cuuint32_t b : {16u, 64u, 128u, 192u, 198u, 256u}) {
    cuuint64_t dims[1] = {6440067ull};
    cuuint32_t box[1] = {b};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("f64 box %u -> %d\n", b, (int)r);
  }
  // 2D view as a fallback: rows of 3 doubles? dims {3*NX, rows}, stride 3*NX*8 (must be 16-multiple)
  {
    cuuint64_t dims[2] = {2ull * 200, 1000}, st[1] = {2ull * 200 * 8};
    cuuint32_t box[2] = {198, 6}, es2[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, st, box, es2, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("f64 2d -> %d\n", (int)r);
  }
  return 0;
}
