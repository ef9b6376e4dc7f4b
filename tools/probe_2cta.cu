// Hardware probe (dev tool): semantics of tcgen05.mma.cta_group::2.
// A 256x64 (rows 0-127 in CTA0, 128-255 in CTA1), B 64x64, D = A B^T.
//   variant 0 ("split"): CTA r holds B rows [32r, 32r+32)
//   variant 1 ("full") : both CTAs hold all 64 B rows
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../paper_2204_01701_b200/csrc/qd_ptx.cuh"

using namespace qd;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe2_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, float* out,
                  int variant) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;            // 16 KB
  uint8_t* sB = sm + 16384;    // 8 KB
  uint64_t* full = (uint64_t*)(sm + 32768);
  uint64_t* done = full + 1;
  uint32_t* slot = (uint32_t*)(full + 2);
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(full, 1);
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(slot)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  ptx::tc_fence_before();
  cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tbase = *slot;
  const int brows = variant == 0 ? 32 : 64;
  if (threadIdx.x == 0) {
    uint32_t bar0 = ptx::smem_u32(full) & 0xFEFFFFFFu;  // CTA0's barrier in the cluster window
    if (rank == 0) ptx::mbar_arrive_expect_tx(full, 2 * (16384 + brows * 128));
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(sA)),
        "l"(&mA), "r"(bar0), "r"(0), "r"((int)(128 * rank))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(ptx::smem_u32(sB)),
        "l"(&mB), "r"(bar0), "r"(0), "r"(variant == 0 ? (int)(32 * rank) : 0)
        : "memory");
    if (rank == 0) {
      ptx::mbar_wait(full, 0);
      ptx::tc_fence_after();
      uint32_t a0 = ptx::smem_u32(sA), b0 = ptx::smem_u32(sB);
      uint32_t idesc = ptx::idesc_bf16(256, 64, false, false);
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = ptx::sw128_desc(a0 + k * 32, 16, 1024);
        uint64_t bd = ptx::sw128_desc(b0 + k * 32, 16, 1024);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
            "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(k > 0))
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              ptx::smem_u32(done)),
          "h"((uint16_t)3)
          : "memory");
    }
  }
  __syncwarp();
  ptx::mbar_wait(done, 0);
  ptx::tc_fence_after();
  int row = warp * 32 + lane;
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    ptx::tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    ptx::tmem_wait_ld();
    for (int e = 0; e < 16; ++e) out[(128 * rank + row) * 64 + c + e] = v[e];
  }
  ptx::tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(64));
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
static void map2d(CUtensorMap* m, const void* p, int inner, int rows, int box_inner, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)inner * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, str, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

extern "C" int probe2_run(const void* A, const void* B, float* out, int variant) {
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  CUtensorMap mA, mB;
  map2d(&mA, A, 64, 256, 64, 128);
  map2d(&mB, B, 64, 64, 64, variant == 0 ? 32 : 64);
  int smem = 1024 + 32768 + 1024;
  cudaFuncSetAttribute(probe2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe2_kernel<<<2, 128, smem>>>(mA, mB, out, variant);
  return (int)cudaDeviceSynchronize();
}
