// Dev probe: halo-box TMA pipeline in the conv2 pattern (cluster of 2).
// mode 0: each CTA loads its box with .cta_group::2, completion on CTA0's barrier;
//         CTA0's consumer waits and releases both CTAs' slot (remote arrive).
// mode 1: each CTA loads with the plain form into its own barrier; own consumer.
// A consumer "tile" costs nothing (no MMA): the rate is the TMA pipeline rate.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include "../paper_2204_01701_b200/csrc/qd_ptx.cuh"
using namespace qd;

struct A2 {
  int iters, slots, mode, W, H, N, bw, bh, w0;
  uint32_t box_bytes, slot_bytes;
};
__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1) probe2(const __grid_constant__ CUtensorMap m, A2 a,
                                                                         unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + a.slots * a.slot_bytes);  // [8] full, [8] empty, [8] pfull
  uint64_t* empty = full + 8;
  uint64_t* pfull = empty + 8;  // mode 2: CTA1's data ready (relayed by CTA1's consumer warp)
  const uint32_t rank = crank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.slots; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
      ptx::mbar_init(&pfull[i], 1);
    }
    ptx::fence_barrier_init();
  }
  csync();
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < a.iters; ++i) {
      ptx::mbar_wait(&empty[s], ph ^ 1);
      int t = (blockIdx.x >> 1) * 7919 + i * 104729;
      int n = (2 * (t % (a.N / 2)) + (int)rank), h = (t / a.N) % (a.H - a.bh + 1);
      if (a.mode == 0) {
        uint32_t bar = ptx::smem_u32(&full[s]) & 0xFEFFFFFFu;
        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], 2 * a.box_bytes);
        asm volatile(
            "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(ptx::smem_u32(sm + s * a.slot_bytes)),
            "l"(&m), "r"(bar), "r"(0), "r"(a.w0), "r"(h), "r"(n)
            : "memory");
      } else {
        ptx::mbar_arrive_expect_tx(&full[s], a.box_bytes);
        ptx::tma_load_4d(&m, &full[s], sm + s * a.slot_bytes, 0, a.w0, h, n);
      }
      if (++s == a.slots) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    if (a.mode == 0 && rank == 1) {
      // CTA1 has no consumer; its empty barrier is released remotely by CTA0
    } else if (a.mode == 2 && rank == 1) {
      // relay: own data landed -> tell CTA0
      for (int i = 0; i < a.iters; ++i) {
        ptx::mbar_wait(&full[s], ph);
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(ptx::smem_u32(&pfull[s])));
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        if (++s == a.slots) { s = 0; ph ^= 1; }
      }
    } else if (a.mode == 2) {
      for (int i = 0; i < a.iters; ++i) {
        ptx::mbar_wait(&full[s], ph);
        ptx::mbar_wait(&pfull[s], ph);
        uint32_t e = ptx::smem_u32(&empty[s]);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(e) : "memory");
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(remote) : "r"(e));
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        if (++s == a.slots) { s = 0; ph ^= 1; }
      }
    } else {
      for (int i = 0; i < a.iters; ++i) {
        ptx::mbar_wait(&full[s], ph);
        if (a.mode == 0) {
          uint32_t e = ptx::smem_u32(&empty[s]);
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(e) : "memory");
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(remote) : "r"(e));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        } else {
          ptx::mbar_arrive(&empty[s]);
        }
        if (++s == a.slots) { s = 0; ph ^= 1; }
      }
    }
  }
  __syncthreads();
  csync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
extern "C" float probe2_run(const void* x, int N, int H, int W, int mode, int bw, int bh, int w0, int slots,
                            int iters, int clusters, unsigned long long* cyc_dev) {
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  CUtensorMap m;
  cuuint32_t es[4] = {1, 1, 1, 1};
  cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t str[3] = {128, (cuuint64_t)W * 128, (cuuint64_t)W * H * 128};
  cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  A2 a{};
  a.iters = iters; a.slots = slots; a.mode = mode; a.W = W; a.H = H; a.N = N; a.bw = bw; a.bh = bh; a.w0 = w0;
  a.box_bytes = bw * bh * 128;
  a.slot_bytes = (a.box_bytes + 1023) / 1024 * 1024;
  int smem = 1024 + slots * a.slot_bytes + 1024;
  cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe2<<<2 * clusters, 64, smem>>>(m, a, cyc_dev);
  cudaEventRecord(e0);
  probe2<<<2 * clusters, 64, smem>>>(m, a, cyc_dev);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return -1.f; }
  return ms;
}
