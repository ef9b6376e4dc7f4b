// Dev probe: cycles per back-to-back tcgen05.mma (bf16, K=16) for 1-CTA M=128
// and 2-CTA M=256 at several N, issued by one elected lane of a converged warp.
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../paper_2204_01701_b200/csrc/qd_ptx.cuh"

using namespace qd;

template <int CG, int N, int UNROLL>
__global__ void __launch_bounds__(128, 1) mma_rate(unsigned long long* out, int iters) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(sm + 65536);
  uint32_t* slot = (uint32_t*)(bar + 1);
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::fence_barrier_init(); }
  if (warp == 0) {
    if (CG == 1) {
      ptx::tmem_alloc(slot, 256);
      ptx::tmem_relinquish();
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(slot)), "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  ptx::tc_fence_before();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  ptx::tc_fence_after();
  uint32_t tmem = *slot;
  if (warp == 1 && rank == 0) {
    constexpr uint32_t IDESC = ptx::idesc_bf16(CG == 2 ? 256 : 128, N, false, false);
    constexpr uint32_t DHI = ptx::sw128_desc_hi(1024);
    const bool leader = ptx::elect_one();
    uint32_t a_lo = ptx::sw128_desc_lo(ptx::smem_u32(sm), 16);
    uint32_t b_lo = ptx::sw128_desc_lo(ptx::smem_u32(sm + 32768), 16);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += UNROLL) {
      if (leader) {
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          if (CG == 1)
            ptx::mma_bf16(tmem, ptx::mk_desc(DHI, a_lo + 2 * (k & 3)), ptx::mk_desc(DHI, b_lo + 2 * (k & 3)), IDESC, 1);
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(ptx::mk_desc(DHI, a_lo + 2 * (k & 3))), "l"(ptx::mk_desc(DHI, b_lo + 2 * (k & 3))), "r"(IDESC), "r"(1u) : "memory");
        }
      }
      __syncwarp();
    }
    unsigned long long t1 = clock64();
    if (leader) {
      if (CG == 1) ptx::mma_commit(bar);
      else asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(ptx::smem_u32(bar)), "h"((uint16_t)3) : "memory");
    }
    __syncwarp();
    ptx::mbar_wait(bar, 0);
    unsigned long long t2 = clock64();
    if (leader && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  } else if (CG == 2 && warp == 1 && rank == 1) {
    ptx::mbar_wait(bar, 0);
  }
  ptx::tc_fence_before();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    if (CG == 1) ptx::tmem_dealloc(tmem, 256);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

template <int CG, int N, int U>
static void launch(unsigned long long* out, int iters, int grid) {
  int smem = 1024 + 65536 + 1024;
  cudaFuncSetAttribute(mma_rate<CG, N, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, mma_rate<CG, N, U>, out, iters);
}

extern "C" int mma_rate_run(unsigned long long* out, int cg, int n, int unroll, int iters, int grid) {
#define L(C, NN, U) if (cg == C && n == NN && unroll == U) launch<C, NN, U>(out, iters, grid);
  L(1, 64, 4) L(1, 128, 4) L(1, 192, 4) L(1, 256, 4) L(2, 64, 4) L(2, 128, 4) L(2, 192, 4) L(2, 256, 4)
  L(1, 64, 16) L(2, 64, 16) L(2, 192, 16)
  return (int)cudaDeviceSynchronize();
}
