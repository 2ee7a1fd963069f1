// Staging-throughput probe for the structured stencil's main kernel: how fast can
// the per-plane halo windows of x (TY + 2 rows of the 66-node window, interleaved dofs) be brought
// into shared memory on one B200, with no stencil arithmetic and no y stores? Same decomposition as
// k_stencil_tma (64 x TY node tiles, 4 CTAs / SM, each CTA an equal contiguous range of (tile,
// plane) units, one CTA barrier per plane), x = 3 * 129^3 doubles.
//   mode 0: rank-1 TMA boxes (cp.async.bulk.tensor.1d, one per row), 4-slot mbarrier ring
//   mode 1: rank-2 TMA box (rows x 200 doubles) over a padded copy of x (row pitch 16-byte aligned)
//   mode 2: synchronous LDG.64 by all threads into the slot (coalesced), then the barrier
//   mode 3: the same loads as mode 2 issued one plane ahead into registers (software pipeline)
//   mode 4: plain grid-stride streaming read of x (the HBM floor)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stage_probe stage_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                             \
  do {                                                                                    \
    cudaError_t e = (x);                                                                  \
    if (e != cudaSuccess) {                                                               \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                           \
    }                                                                                     \
  } while (0)

constexpr int TY = 4, NT = 128, RING = 4, XBOX = 200, RSP = 208;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
          bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma1(uint32_t dst, const CUtensorMap* m, int c, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

struct Geo {
  int NX, NY, NZ, ntx, nty, pitch;  // pitch: doubles per padded row (mode 1)
};

template <int MODE>
__global__ void __launch_bounds__(NT, 4) k_stage(const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m2,
                                                 Geo g, const double* __restrict__ x, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double (*xs)[TY + 2][RSP] = reinterpret_cast<double (*)[TY + 2][RSP]>(sm);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + sizeof(double) * RING * (TY + 2) * RSP);
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int q = 0; q < RING; ++q) mbar_init(su32(&bars[q]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  uint32_t phase = 0;
  double acc = 0;
  const int64_t U = (int64_t)g.ntx * g.nty * g.NZ;
  int64_t u = U * blockIdx.x / gridDim.x;
  const int64_t ue = U * (blockIdx.x + 1) / gridDim.x;
  while (u < ue) {
    const int tile = static_cast<int>(u / g.NZ), kk = static_cast<int>(u % g.NZ);
    const int kl = static_cast<int>(min(static_cast<int64_t>(g.NZ), kk + (ue - u)));
    u += kl - kk;
    const int i0 = (tile % g.ntx) * 64, j0 = (tile / g.ntx) * TY;
    const int k0 = kk, k1 = kl;  // planes k0 - 1 .. k1 staged (as the stencil: one halo plane below)
    auto issue = [&](int p) {
      const int sl = (p + 1) % RING;
      if (p < 0 || p >= g.NZ) p = 0;  // keep the phase structure simple: stage plane 0 again
      const uint32_t bar = su32(&bars[sl]);
      if constexpr (MODE == 0) {
        if ((tid & 31) != 0) return;
        const int w = tid >> 5;
        if (w == 0) mbar_expect(bar, (TY + 2) * XBOX * 8);
        for (int r = w; r < TY + 2; r += TY) {
          int jj = j0 - 1 + r;
          jj = jj < 0 ? 0 : (jj >= g.NY ? g.NY - 1 : jj);
          const int c = 3 * (i0 - 1 + g.NX * (jj + g.NY * p));
          tma1(su32(&xs[sl][r][0]), &m1, c & ~1, bar);
        }
      } else if constexpr (MODE == 1) {
        if (tid != 0) return;
        mbar_expect(bar, (TY + 2) * XBOX * 8);
        tma2(su32(&xs[sl][0][0]), &m2, 3 * (i0 - 1) & ~1, j0 - 1 + g.NY * p, bar);
      }
    };
    auto wait = [&](int p) {
      const int sl = (p + 1) % RING;
      mbar_wait(su32(&bars[sl]), (phase >> sl) & 1u);
      phase ^= 1u << sl;
    };
    if constexpr (MODE <= 1) {
      for (int q = 0; q < RING - 1; ++q)
        if (k0 - 1 + q <= k1) issue(k0 - 1 + q);
      wait(k0 - 1);
      __syncthreads();
      for (int p = k0 - 1; p <= k1; ++p) {
        const int sl = (p + 1) % RING;
        acc += xs[sl][tid >> 5][6 * (tid & 31)] + xs[sl][(tid >> 5) + 2][6 * (tid & 31) + 7];
        if (p + 1 <= k1) wait(p + 1);
        __syncthreads();
        if (p + RING - 1 <= k1) issue(p + RING - 1);
      }
    } else if constexpr (MODE == 2 || MODE == 3) {
      // 6 rows x 200 doubles = 1200 doubles per plane: 128 threads x 10 loads (last partial)
      double v[10];
      auto load = [&](int p) {
        const int pp = p < 0 || p >= g.NZ ? 0 : p;
#pragma unroll
        for (int q = 0; q < 10; ++q) {
          const int e = tid + NT * q;
          v[q] = 0.0;
          if (e < (TY + 2) * XBOX) {
            const int r = e / XBOX, c = e % XBOX;
            int jj = j0 - 1 + r;
            jj = jj < 0 ? 0 : (jj >= g.NY ? g.NY - 1 : jj);
            const int64_t gi = 3ll * (i0 - 1 + (int64_t)g.NX * (jj + g.NY * pp)) + c;
            if (gi >= 0 && gi < 3ll * g.NX * g.NY * g.NZ) v[q] = __ldg(&x[gi]);
          }
        }
      };
      auto store = [&](int p) {
        const int sl = (p + 1) % RING;
#pragma unroll
        for (int q = 0; q < 10; ++q) {
          const int e = tid + NT * q;
          if (e < (TY + 2) * XBOX) xs[sl][e / XBOX][e % XBOX] = v[q];
        }
      };
      load(k0 - 1);
      for (int p = k0 - 1; p <= k1; ++p) {
        if constexpr (MODE == 2) {
          store(p);
          if (p + 1 <= k1) load(p + 1);
        } else {
          store(p);
          if (p + 1 <= k1) load(p + 1);  // in flight across the barrier and the "compute"
        }
        __syncthreads();
        const int sl = (p + 1) % RING;
        acc += xs[sl][tid >> 5][6 * (tid & 31)] + xs[sl][(tid >> 5) + 2][6 * (tid & 31) + 7];
      }
    }
  }
  if (acc == 1.2345e300) out[0] = acc;
}

__global__ void k_stream(const double2* __restrict__ x, int64_t n2, double* out) {
  double a = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = __ldg(&x[i]);
    a += v.x + v.y;
  }
  if (a == 1.2345e300) out[0] = a;
}

__global__ void k_pad(const double* __restrict__ x, double* xp, Geo g) {
  const int64_t rows = (int64_t)g.NY * g.NZ, rl = 3ll * g.NX;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < rows * g.pitch; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = q / g.pitch, c = q % g.pitch;
    xp[q] = c < rl ? x[r * rl + c] : 0.0;
  }
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 129;
  Geo g{N, N, N, (N - 1 + 63) / 64, (N + TY - 1) / TY, 0};
  g.pitch = ((3 * N + 1) + 1) & ~1;  // even -> 16-byte aligned rows
  const int64_t n = 3ll * N * N * N;
  double *x, *xp, *out;
  CK(cudaMalloc(&x, n * 8 + 64));
  CK(cudaMalloc(&xp, (int64_t)g.pitch * N * N * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, n * 8));
  k_pad<<<1184, 256>>>(x, xp, g);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap m1{}, m2{};
  {
    cuuint64_t dim[1] = {static_cast<cuuint64_t>(n)}, str[1] = {8};
    cuuint32_t box[1] = {XBOX}, es[1] = {1};
    if (enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, x, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      std::printf("encode m1 failed\n");
  }
  {
    cuuint64_t dim[2] = {static_cast<cuuint64_t>(g.pitch), static_cast<cuuint64_t>(N) * N},
               str[1] = {static_cast<cuuint64_t>(g.pitch) * 8};
    cuuint32_t box[2] = {XBOX, TY + 2}, es[2] = {1, 1};
    if (enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, xp, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      std::printf("encode m2 failed\n");
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = sizeof(double) * RING * (TY + 2) * RSP + 8 * RING + 128;
  CK(cudaFuncSetAttribute(k_stage<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_stage<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_stage<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_stage<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // L2 flush buffer (> 126 MB)
  double* fl;
  const size_t fln = 256ull << 20;
  CK(cudaMalloc(&fl, fln));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const char* names[5] = {"tma rank-1 rows", "tma rank-2 box (padded x)", "LDG -> STS, synchronous",
                          "LDG one plane ahead", "stream read of x"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int blocks_per_sm : {4}) {
      const int grid = sms * blocks_per_sm;
      float best = 1e30f, sum = 0;
      const int reps = 20;
      for (int r = 0; r < reps + 2; ++r) {
        CK(cudaMemsetAsync(fl, r & 1, fln));
        CK(cudaEventRecord(a));
        switch (mode) {
          case 0: k_stage<0><<<grid, NT, smem>>>(m1, m2, g, x, out); break;
          case 1: k_stage<1><<<grid, NT, smem>>>(m1, m2, g, x, out); break;
          case 2: k_stage<2><<<grid, NT, smem>>>(m1, m2, g, x, out); break;
          case 3: k_stage<3><<<grid, NT, smem>>>(m1, m2, g, x, out); break;
          default: k_stream<<<sms * 8, 512>>>(reinterpret_cast<const double2*>(x), n / 2, out);
        }
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (r >= 2) {
          best = ms < best ? ms : best;
          sum += ms;
        }
      }
      std::printf("mode %d %-28s N=%d: mean %.2f us, best %.2f us, x %.1f MB -> %.0f GB/s (mean)\n", mode, names[mode], N,
                  sum / reps * 1e3, best * 1e3, n * 8 / 1e6, n * 8 / (sum / reps * 1e-3) / 1e9);
    }
  }
  return 0;
}
