// T1 families (t1_pure, t1_full, t1and2): one output unit carrying a full-rank
// quadratic form, fc only (neurons.py:58-65, forward :245-254, backward :320-348):
//   y = sum_i (x Wq)_i x_i  [+ x Wb (t1_full) | + (x*x) Wb (t1and2)]
// The n x n GEMMs run on the generic CUDA-core GEMM (qd_simt.cu) in fp32; the
// quadratic form's row dot and the elementwise backward terms are small kernels.
// Weights are packed as fp32 [Wq (n*n) | Wb (n)] for both dtypes.
#include <stdio.h>
#include "qd_kernels.h"
#include "qd_gemm.cuh"

namespace qd {

bool is_t1(int family) {
  return family == QD_FAM_T1_PURE || family == QD_FAM_T1_FULL || family == QD_FAM_T1AND2;
}
size_t t1_pack_bytes(const Plan& P) { return ((size_t)P.C * P.C + P.C) * 4; }

__global__ void t1_pack_kernel(int n, const float* wq, const float* wb, float* out) {
  const long long tot = (long long)n * n + n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = i < (long long)n * n ? wq[i] : (wb ? wb[i - (long long)n * n] : 0.f);
}
void t1_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st) {
  t1_pack_kernel<<<128, 256, 0, st>>>(P.C, w[0], P.family == QD_FAM_T1_PURE ? nullptr : w[1], (float*)wpack);
  count_launch(st, "t1_pack");
}

// workspace: V (N x n), dv (N x n), Q (N x n) fp32, wgrad partials [S][n][n]
Workspace t1_workspace(const Plan& P) {
  Workspace L;
  memset(&L, 0, sizeof(L));
  const size_t nn = (size_t)P.N * P.C * 4;
  L.sz_P = 3 * nn;
  long long S = (2 * 148 + 0) / (((P.C + 63) / 64) * ((P.C + 63) / 64));
  if (S > P.N / 32) S = P.N / 32;
  if (S < 1) S = 1;
  L.wg_split = (int)S;
  L.sz_WG = (size_t)S * P.C * P.C * 4;
  size_t off = 0;
  L.off_P = off; off = (off + L.sz_P + 255) / 256 * 256;
  L.off_WG = off; off = (off + L.sz_WG + 255) / 256 * 256;
  L.total = off;
  return L;
}

template <typename T>
struct T1RowA {  // A(m, k) = x[m][k] (optionally squared)
  static constexpr bool kfast = true;
  const T* x; int n;
  __device__ float operator()(int m, long long k) const { return ld(x + (size_t)m * n + k); }
};
struct T1ColB {  // B(j, k) = W[k][j] (x @ W)
  static constexpr bool kfast = false;
  const float* w; int n;
  __device__ float operator()(int j, long long k) const { return w[(size_t)k * n + j]; }
};
struct T1RowB {  // B(i, k) = W[i][k] (dv @ W^T)
  static constexpr bool kfast = true;
  const float* w; int n;
  __device__ float operator()(int i, long long k) const { return w[(size_t)i * n + k]; }
};
template <typename T>
struct T1XtA {  // A(i, m) = x[m][i]   (x^T dv)
  static constexpr bool kfast = false;
  const T* x; int n;
  __device__ float operator()(int i, long long m) const { return ld(x + (size_t)m * n + i); }
};
struct T1DvB {  // B(j, m) = dv[m][j]
  static constexpr bool kfast = false;
  const float* dv; int n;
  __device__ float operator()(int j, long long m) const { return dv[(size_t)m * n + j]; }
};

// y[m] = sum_i V[m][i] x[m][i] + linear term; one warp per row, fixed order
template <typename T>
__global__ void t1_fwd_kernel(int family, int N, int n, const T* x, const float* V, const float* wb, T* y) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= N) return;
  const T* xr = x + (size_t)warp * n;
  const float* vr = V + (size_t)warp * n;
  float q = 0.f, l = 0.f;
  for (int i = lane; i < n; i += 32) {
    const float xv = ld(xr + i);
    q = fmaf(vr[i], xv, q);
    if (family == QD_FAM_T1_FULL) l = fmaf(xv, wb[i], l);
    if (family == QD_FAM_T1AND2) l = fmaf(xv * xv, wb[i], l);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    q += __shfl_xor_sync(0xffffffffu, q, o);
    l += __shfl_xor_sync(0xffffffffu, l, o);
  }
  if (lane == 0) y[warp] = cvt<T>(q + l);
}

// dv = g x (dh = broadcast g)
template <typename T>
__global__ void t1_dv_kernel(int N, int n, const T* x, const T* g, float* dv) {
  const long long tot = (long long)N * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x)
    dv[i] = ld(g + i / n) * ld(x + i);
}

// dx = g V + dv Wq^T (+ g Wb^T | + 2 (g Wb^T) x), in the reference's term order
template <typename T>
__global__ void t1_dx_kernel(int family, int N, int n, const T* x, const T* g, const float* V, const float* Q,
                             const float* wb, T* dx) {
  const long long tot = (long long)N * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % n);
    const float gv = ld(g + i / n);
    float v;
    if (family == QD_FAM_T1_FULL) {
      v = gv * wb[k];
      v = v + gv * V[i];
      v = v + Q[i];
    } else {
      v = gv * V[i];
      v = v + Q[i];
      if (family == QD_FAM_T1AND2) {
        const float t = (gv * wb[k]) * ld(x + i);
        v = v + t;
        v = v + t;
      }
    }
    dx[i] = cvt<T>(v);
  }
}

// dWb[i] = sum_m g[m] x[m][i] (t1_full) or g[m] x[m][i]^2 (t1and2); fixed order
template <typename T>
__global__ void t1_dwb_kernel(int family, int N, int n, const T* x, const T* g, float* dwb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
  for (int m = 0; m < N; ++m) {
    const float xv = ld(x + (size_t)m * n + i);
    acc = fmaf(ld(g + m), family == QD_FAM_T1AND2 ? xv * xv : xv, acc);
  }
  dwb[i] = acc;
}

__global__ void t1_sum_kernel(long long tot, int S, const float* part, float* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += part[(size_t)s * tot + i];
    out[i] = acc;
  }
}

template <typename T>
static int t1_forward_t(const Plan& P, const T* x, const float* wp, T* y, char* ws, const Workspace& L,
                        cudaStream_t st) {
  const int N = P.N, n = P.C;
  float* V = (float*)(ws + L.off_P);
  simt_gemm_ext(T1RowA<T>{x, n}, T1ColB{wp, n}, N, n, n, 1, V, st);
  t1_fwd_kernel<T><<<(N * 32 + 255) / 256, 256, 0, st>>>(P.family, N, n, x, V, wp + (size_t)n * n, y);
  count_launch(st, "t1_fwd");
  return check_launch("t1 forward");
}

int t1_forward(const Plan& P, const void* x, const void* wpack, void* y, char* ws, const Workspace& L,
               cudaStream_t st) {
  if (P.dtype == QD_BF16) return t1_forward_t<bf16>(P, (const bf16*)x, (const float*)wpack, (bf16*)y, ws, L, st);
  return t1_forward_t<float>(P, (const float*)x, (const float*)wpack, (float*)y, ws, L, st);
}

template <typename T>
static int t1_backward_t(const Plan& P, const T* x, const float* wp, const T* g, T* dx, float* const dW[3],
                         char* ws, const Workspace& L, cudaStream_t st) {
  const int N = P.N, n = P.C;
  float* V = (float*)(ws + L.off_P);
  float* dv = V + (size_t)N * n;
  float* Q = dv + (size_t)N * n;
  const float* wb = wp + (size_t)n * n;
  simt_gemm_ext(T1RowA<T>{x, n}, T1ColB{wp, n}, N, n, n, 1, V, st);  // v = x Wq (recomputed)
  const long long tot = (long long)N * n;
  const int grid = (int)((tot + 255) / 256 > 148 * 16 ? 148 * 16 : (tot + 255) / 256);
  t1_dv_kernel<T><<<grid, 256, 0, st>>>(N, n, x, g, dv);
  count_launch(st, "t1_dv");
  if (dW[0]) {
    float* part = (float*)(ws + L.off_WG);
    simt_gemm_ext(T1XtA<T>{x, n}, T1DvB{dv, n}, n, n, N, L.wg_split, part, st);  // dWq = x^T dv
    t1_sum_kernel<<<(int)(((long long)n * n + 255) / 256), 256, 0, st>>>((long long)n * n, L.wg_split, part, dW[0]);
    count_launch(st, "t1_sum");
    if (P.family != QD_FAM_T1_PURE && dW[1]) {
      t1_dwb_kernel<T><<<(n + 127) / 128, 128, 0, st>>>(P.family, N, n, x, g, dW[1]);
      count_launch(st, "t1_dwb");
    }
  }
  if (dx) {
    simt_gemm_ext(T1RowA<float>{dv, n}, T1RowB{wp, n}, N, n, n, 1, Q, st);  // dv Wq^T
    t1_dx_kernel<T><<<grid, 256, 0, st>>>(P.family, N, n, x, g, V, Q, wb, dx);
    count_launch(st, "t1_dx");
  }
  return check_launch("t1 backward");
}

int t1_backward(const Plan& P, const void* x, const void* wpack, const void* dy, void* dx, float* const dW[3],
                char* ws, const Workspace& L, cudaStream_t st) {
  if (P.dtype == QD_BF16)
    return t1_backward_t<bf16>(P, (const bf16*)x, (const float*)wpack, (const bf16*)dy, (bf16*)dx, dW, ws, L, st);
  return t1_backward_t<float>(P, (const float*)x, (const float*)wpack, (const float*)dy, (float*)dx, dW, ws, L, st);
}

}  // namespace qd
