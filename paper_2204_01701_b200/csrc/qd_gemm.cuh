// Generic tiled CUDA-core GEMM shared by the translation units:
//   out[s][m][n] = sum_{k in split s} A(m,k) * B(n,k)   (fp32 FFMA, functor operands)
#pragma once
#include "qd_kernels.h"

namespace qd {
constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

template <class LA, class LB>
__global__ void __launch_bounds__(256) simt_gemm_kernel(LA la, LB lb, int M, int N, long long K,
                                                        long long kper, float* out) {
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Bs[SG_BK][SG_BN + 4];
  int m0 = blockIdx.x * SG_BM, n0 = blockIdx.y * SG_BN, s = blockIdx.z;
  long long kb = (long long)s * kper, ke = kb + kper;
  if (ke > K) ke = K;
  int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (long long k0 = kb; k0 < ke; k0 += SG_BK) {
    for (int i = threadIdx.x; i < SG_BM * SG_BK; i += 256) {
      int mm = i % SG_BM, kk = i / SG_BM;
      int m = m0 + mm;
      long long k = k0 + kk;
      As[kk][mm] = (m < M && k < ke) ? la(m, k) : 0.f;
    }
    for (int i = threadIdx.x; i < SG_BN * SG_BK; i += 256) {
      int nn = i % SG_BN, kk = i / SG_BN;
      int n = n0 + nn;
      long long k = k0 + kk;
      Bs[kk][nn] = (n < N && k < ke) ? lb(n, k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* o = out + (size_t)s * M * N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx * 4 + j;
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
