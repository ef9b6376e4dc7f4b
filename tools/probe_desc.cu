// Hardware probe (dev tool, not part of the product): does a SWIZZLE_128B
// UMMA descriptor whose start address is shifted by s 128-B rows (not a
// multiple of the 1024-B swizzle atom) read rows s.. of a TMA-written tile,
// and what must the descriptor's base_offset field hold? Answers decide
// whether one halo tile can feed all filter taps.
//   mode 0: K-major A (row shift), K-major B      D[m][n] = sum_k A[s+m][k] B[n][k]
//   mode 1: MN-major A (K-row shift), MN-major B  D[m][n] = sum_k A[s+k][m] B[k][n]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include "../paper_2204_01701_b200/csrc/qd_ptx.cuh"

using namespace qd;

__global__ void __launch_bounds__(128, 1) probe_kernel(const __grid_constant__ CUtensorMap mA0,
                                                       const __grid_constant__ CUtensorMap mA1,
                                                       const __grid_constant__ CUtensorMap mB, float* out,
                                                       int mode, int shift, int base_off) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;              // 64 KB
  uint8_t* sB = sm + 65536;      // 32 KB
  uint64_t* bar = (uint64_t*)(sm + 98304);
  uint64_t* mbar = bar + 1;
  uint32_t* slot = (uint32_t*)(bar + 2);
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::mbar_init(mbar, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 0) { ptx::tmem_alloc(slot, 64); ptx::tmem_relinquish(); }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  uint32_t tbase = *slot;
  if (threadIdx.x == 0) {
    if (mode == 0) {
      ptx::mbar_arrive_expect_tx(bar, 256 * 128 + 64 * 128);
      ptx::tma_load_2d(&mA0, bar, sA, 0, 0);      // [256 rows][64 k]
      ptx::tma_load_2d(&mB, bar, sB, 0, 0);       // [64 rows][64 k]
    } else if (mode == 2) {
      ptx::mbar_arrive_expect_tx(bar, 256 * 128 + 256 * 128);
      ptx::tma_load_2d(&mA0, bar, sA, 0, 0);      // [256 q][64 m] single atom
      ptx::tma_load_2d(&mB, bar, sB, 0, 0);       // [256 q][64 n]
    } else if (mode == 3) {
      ptx::mbar_arrive_expect_tx(bar, 192 * 128 + 64 * 128);
      ptx::tma_load_2d(&mA0, bar, sA + base_off * 128, 0, 0);  // [192 rows][64 k] at misaligned dst
      ptx::tma_load_2d(&mB, bar, sB, 0, 0);
    } else {
      ptx::mbar_arrive_expect_tx(bar, 2 * 256 * 128 + 256 * 128);
      ptx::tma_load_2d(&mA0, bar, sA, 0, 0);      // [256 q][64 m] atom 0
      ptx::tma_load_2d(&mA1, bar, sA + 32768, 64, 0);  // atom 1 (m 64..127)
      ptx::tma_load_2d(&mB, bar, sB, 0, 0);       // [256 q][64 n]
    }
    ptx::mbar_wait(bar, 0);
    ptx::tc_fence_after();
    uint32_t a0 = ptx::smem_u32(sA), b0 = ptx::smem_u32(sB);
    for (int k = 0; k < 4; ++k) {
      uint64_t ad, bd;
      uint32_t idesc;
      if (mode == 2) {
        // M atoms: atom 1 = atom 0 shifted by base_off K-rows (LBO = base_off*128 B)
        ad = ptx::sw128_desc(a0 + (shift + 16 * k) * 128, base_off * 128, 1024);
        bd = ptx::sw128_desc(b0 + (16 * k) * 128, 32768, 1024);
        idesc = ptx::idesc_bf16(128, 64, true, true);
      } else if (mode == 3) {
        ad = ptx::sw128_desc(a0 + (base_off + shift) * 128 + k * 32, 16, 1024);
        bd = ptx::sw128_desc(b0 + k * 32, 16, 1024);
        idesc = ptx::idesc_bf16(128, 64, false, false);
      } else if (mode == 0) {
        ad = ptx::sw128_desc(a0 + shift * 128 + k * 32, 16, 1024);
        bd = ptx::sw128_desc(b0 + k * 32, 16, 1024);
        idesc = ptx::idesc_bf16(128, 64, false, false);
      } else {
        ad = ptx::sw128_desc(a0 + (shift + 16 * k) * 128, 32768, 1024);
        bd = ptx::sw128_desc(b0 + (16 * k) * 128, 32768, 1024);
        idesc = ptx::idesc_bf16(128, 64, true, true);
      }
      if (mode <= 1) ad |= (uint64_t)(base_off & 7) << 49;
      ptx::mma_bf16(tbase, ad, bd, idesc, k > 0);
    }
    ptx::mma_commit(mbar);
  }
  __syncwarp();
  ptx::mbar_wait(mbar, 0);
  ptx::tc_fence_after();
  int row = warp * 32 + lane;
  for (int c = 0; c < 64; c += 16) {
    float v[16];
    ptx::tmem_ld16(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    ptx::tmem_wait_ld();
    for (int e = 0; e < 16; ++e) out[row * 64 + c + e] = v[e];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 64); }
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

extern "C" int probe_run(const void* A, const void* B, float* out, int mode, int shift, int base_off) {
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  CUtensorMap mA0, mA1, mB;
  if (mode == 0) {
    map2d(&mA0, A, 64, 256, 64, 256);
    mA1 = mA0;
    map2d(&mB, B, 64, 64, 64, 64);
  } else if (mode == 2) {
    map2d(&mA0, A, 64, 256, 64, 256);
    mA1 = mA0;
    map2d(&mB, B, 64, 256, 64, 256);
  } else if (mode == 3) {
    map2d(&mA0, A, 64, 192, 64, 192);
    mA1 = mA0;
    map2d(&mB, B, 64, 64, 64, 64);
  } else {
    map2d(&mA0, A, 128, 256, 64, 256);  // A_mn [256 q][128 m]
    mA1 = mA0;
    map2d(&mB, B, 64, 256, 64, 256);    // B_mn [256 q][64 n]
  }
  int smem = 1024 + 98304 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(mA0, mA1, mB, out, mode, shift, base_off);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
