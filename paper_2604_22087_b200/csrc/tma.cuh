// Blackwell bulk-async data movement used by the structured kernels: TMA tensor copies
// (cp.async.bulk.tensor, SASS UTMALDG) completing on shared-memory mbarriers (SASS SYNCS), and the
// host-side tensor-map encoding (cuTensorMapEncodeTiled through the runtime's driver entry point, so
// the library does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "common.cuh"

namespace afem {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}

// makes initialised barriers visible to the async proxy (TMA completes on them)
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// orders this thread's earlier generic-proxy shared-memory accesses before later async-proxy ones
// (a TMA write into a slot the threads have just read or patched)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// 1D tiled tensor copy global -> shared: box of the map's boxDim elements starting at element c
// (any integer; out-of-range elements are zero-filled), completion counted on mbarrier bar.
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const CUtensorMap* map, int c, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(bar)
      : "memory");
}

// Host: encode a rank-1 tiled map over `n` elements of `elem_bytes` at `base` (16-byte aligned)
// with box `box` (box * elem_bytes a multiple of 16).
void encode_map_1d(CUtensorMap* map, const void* base, uint64_t n, CUtensorMapDataType type, uint32_t box);

}  // namespace afem
