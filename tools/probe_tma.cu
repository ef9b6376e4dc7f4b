// Dev probe: TMA load throughput for the box shapes the conv kernels use.
// Each CTA streams `iters` boxes through a `stages`-deep smem ring (no compute).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include "../paper_2204_01701_b200/csrc/qd_ptx.cuh"

using namespace qd;

struct PArgs {
  int iters, stages, mode;  // mode 0: 4-D box; 1: 2-D box
  int W, H, N, bw, bh, w0, rows2d, npix;
  uint32_t box_bytes, slot_bytes;
};

__global__ void __launch_bounds__(32, 1) tma_probe(const __grid_constant__ CUtensorMap m, PArgs a) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + a.stages * a.slot_bytes);
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) ptx::mbar_init(&full[i], 1);
    ptx::fence_barrier_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < a.iters + a.stages; ++i) {
    if (i < a.iters) {
      int st = i % a.stages;
      if (i >= a.stages) ptx::mbar_wait(&full[st], ((i / a.stages) - 1) & 1);  // slot free
      int t = blockIdx.x * 7919 + i * 104729;
      ptx::mbar_arrive_expect_tx(&full[st], a.box_bytes);
      if (a.mode == 0) {
        int n = t % a.N, h = (t / a.N) % (a.H - a.bh + 1);
        ptx::tma_load_4d(&m, &full[st], sm + st * a.slot_bytes, 0, a.w0, h, n);
      } else {
        int r0 = (int)(((long long)t * 131) % (a.npix - a.rows2d));
        ptx::tma_load_2d(&m, &full[st], sm + st * a.slot_bytes, 0, r0);
      }
    }
  }
  // drain
  for (int i = a.iters; i < a.iters + a.stages; ++i) {
    int j = i - a.stages;
    if (j >= 0) ptx::mbar_wait(&full[j % a.stages], (j / a.stages) & 1);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;

extern "C" float tma_probe_run(const void* x, int N, int H, int W, int mode, int bw, int bh, int w0, int rows2d,
                               int stages, int iters, int ctas) {
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  CUtensorMap m;
  cuuint32_t es[4] = {1, 1, 1, 1};
  PArgs a{};
  a.iters = iters; a.stages = stages; a.mode = mode; a.W = W; a.H = H; a.N = N; a.bw = bw; a.bh = bh; a.w0 = w0;
  a.rows2d = rows2d; a.npix = N * H * W;
  if (mode == 0) {
    cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t str[3] = {128, (cuuint64_t)W * 128, (cuuint64_t)W * H * 128};
    cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.box_bytes = bw * bh * 128;
  } else {
    cuuint64_t dims[2] = {64, (cuuint64_t)a.npix};
    cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)rows2d};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, str, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    a.box_bytes = rows2d * 128;
  }
  a.slot_bytes = (a.box_bytes + 1023) / 1024 * 1024;
  int smem = 1024 + stages * a.slot_bytes + 1024;
  cudaError_t e2 = cudaFuncSetAttribute(tma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e2 != cudaSuccess) printf("attr err %s\n", cudaGetErrorString(e2));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tma_probe<<<ctas, 32, smem>>>(m, a);  // warm
  cudaEventRecord(e0);
  tma_probe<<<ctas, 32, smem>>>(m, a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return -1.f; }
  return ms;
}
