// Generic tiled CUDA-core GEMM shared by the translation units:
//   out[s][m][n] = sum_{k in split s} A(m,k) * B(n,k)   (fp32 FFMA, functor operands)
#pragma once
#include "qd_kernels.h"

namespace qd {
constexpr int SG_BM = 128, SG_BN = 128, SG_BK = 8;

// Operand functors declare their contiguous direction: kfast (A(m, k) / B(n, k)
// contiguous along k) loads 8 consecutive k of a row per lane group, otherwise
// the 32 lanes of a warp read 32 consecutive m (or n).
// 128 x 128 tile, 256 threads, 8 x 8 FFMA micro-tile per thread (2 x 2 blocks of
// 4 x 4: float4 shared reads without bank conflicts), shared memory double
// buffered with the next k-tile staged in registers during the FFMAs.
template <class F, int ROWS>
__device__ __forceinline__ void sg_load(const F& f, int r0, int R, long long k0, long long ke, float v[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = threadIdx.x + 256 * u;
    const int rr = F::kfast ? i / SG_BK : i % ROWS, kk = F::kfast ? i % SG_BK : i / ROWS;
    const int row = r0 + rr;
    const long long k = k0 + kk;
    v[u] = (row < R && k < ke) ? f(row, k) : 0.f;
  }
}
template <class F, int ROWS>
__device__ __forceinline__ void sg_store(float (*S)[ROWS + 4], const float v[4]) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = threadIdx.x + 256 * u;
    const int rr = F::kfast ? i / SG_BK : i % ROWS, kk = F::kfast ? i % SG_BK : i / ROWS;
    S[kk][rr] = v[u];
  }
}

template <class LA, class LB>
__global__ void __launch_bounds__(256) simt_gemm_kernel(LA la, LB lb, int M, int N, long long K,
                                                        long long kper, float* out) {
  __shared__ __align__(16) float As[2][SG_BK][SG_BM + 4];
  __shared__ __align__(16) float Bs[2][SG_BK][SG_BN + 4];
  const int m0 = blockIdx.x * SG_BM, n0 = blockIdx.y * SG_BN, s = blockIdx.z;
  const long long kb = (long long)s * kper;
  long long ke = kb + kper;
  if (ke > K) ke = K;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  float ra[4], rb[4];
  int buf = 0;
  if (kb < ke) {
    sg_load<LA, SG_BM>(la, m0, M, kb, ke, ra);
    sg_load<LB, SG_BN>(lb, n0, N, kb, ke, rb);
    sg_store<LA, SG_BM>(As[0], ra);
    sg_store<LB, SG_BN>(Bs[0], rb);
  }
  __syncthreads();
  for (long long k0 = kb; k0 < ke; k0 += SG_BK) {
    const bool more = k0 + SG_BK < ke;
    if (more) {  // next k-tile into registers while this one is multiplied
      sg_load<LA, SG_BM>(la, m0, M, k0 + SG_BK, ke, ra);
      sg_load<LB, SG_BN>(lb, n0, N, k0 + SG_BK, ke, rb);
    }
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      sg_store<LA, SG_BM>(As[buf ^ 1], ra);
      sg_store<LB, SG_BN>(Bs[buf ^ 1], rb);
    }
    __syncthreads();
    buf ^= 1;
  }
  float* o = out + (size_t)s * M * N;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n < N) o[(size_t)m * N + n] = acc[i][j];
    }
  }
}

template <class LA, class LB>
inline void simt_gemm_ext(LA la, LB lb, int M, int N, long long K, int split, float* out, cudaStream_t st) {
  long long kper = (K + split - 1) / split;
  kper = (kper + SG_BK - 1) / SG_BK * SG_BK;
  dim3 grid((M + SG_BM - 1) / SG_BM, (N + SG_BN - 1) / SG_BN, split);
  simt_gemm_kernel<<<grid, 256, 0, st>>>(la, lb, M, N, K, kper, out);
  count_launch(st, "simt_gemm");
}


}  // namespace qd
