// Probe: rank-1 TMA loads (double and uint8 boxes) through a __grid_constant__ map, on the GPU box.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2604_22087_b200/csrc/tma.cuh"
namespace afem {
void encode_map_1d(CUtensorMap* map, const void* base, uint64_t n, CUtensorMapDataType type, uint32_t box) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const cuuint64_t dims[1] = {n}, st[1] = {16};
  const cuuint32_t boxd[1] = {box}, es[1] = {1};
  CUresult r = enc(map, type, 1, const_cast<void*>(base), dims, st, boxd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode -> %d\n", (int)r);
}
}  // namespace afem
using namespace afem;
template <int BOX, int MODE>
__global__ void k(const __grid_constant__ CUtensorMap m, int c, double* out) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(smem_u32(&bar), BOX * 8);
    if (MODE == 0) tma_load_1d(smem_u32(buf), &m, c, smem_u32(&bar));
    else {
      asm volatile(
          "cp.async.bulk.tensor.1d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(
              smem_u32(buf)),
          "l"(reinterpret_cast<uint64_t>(&m)), "r"(c), "r"(smem_u32(&bar))
          : "memory");
    }
  }
  mbar_wait(smem_u32(&bar), 0);
  for (int i = threadIdx.x; i < BOX; i += blockDim.x) out[i] = buf[i];
}
int main() {
  double *x, *out;
  int n = 100000;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&out, 256 * 8);
  double* h = new double[n];
  for (int i = 0; i < n; ++i) h[i] = i;
  cudaMemcpy(x, h, n * 8, cudaMemcpyHostToDevice);
  CUtensorMap m;
  for (int box : {16, 198}) {
    encode_map_1d(&m, x, n, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, box);
    for (int mode = 0; mode < 2; ++mode)
      for (int c : {0, 2, 4, -2, -4, 6, 99998, 99996}) {
        cudaMemset(out, 0, 256 * 8);
        if (box == 16) mode ? k<16, 1><<<1, 32>>>(m, c, out) : k<16, 0><<<1, 32>>>(m, c, out);
        else mode ? k<198, 1><<<1, 32>>>(m, c, out) : k<198, 0><<<1, 32>>>(m, c, out);
        cudaError_t e = cudaDeviceSynchronize();
        double r[4];
        cudaMemcpy(r, out, 32, cudaMemcpyDeviceToHost);
        printf("box %d mode %d c %d -> %s  %g %g %g %g\n", box, mode, c, cudaGetErrorString(e), r[0], r[1], r[2], r[3]);
        if (e != cudaSuccess) return 1;
      }
  }
  return 0;
}
