#include <stdlib.h>
// Batch norm (+ ReLU) fused around the quadratic conv.
// Reference semantics: tensor.py:423-470 (forward: biased batch variance for the
// normalisation AND for the running-variance update, eps 1e-5, momentum 0.1)
// and tensor.py:552-570 (backward: dx = inv/m (m dxhat - sum dxhat - xhat
// sum dxhat xhat), dgamma = sum g xhat, dbeta = sum g).
//
// Forward: per-channel shifted sums (sum y-K, sum (y-K)^2, K = row 0, for a
// stable variance) as fixed-order partials -> mean / inv_std / running stats ->
// one normalise(+ReLU) pass.
// Backward: one reduction pass over (dz, y) for sum g and sum g xhat (g = dz
// masked by the recomputed ReLU), then ONE elementwise pass that applies the BN
// backward and directly emits the quadratic layer's backward operand
// D = [dy b | dy a | dy] (or [dy b | dy a], or dy) plus the layer's bias
// partial sums -- the BN-backward output dy is never written to memory.
// NHWC [M][C] tensors; fp32 arithmetic for both dtypes.
#include <stdio.h>
#include "qd_kernels.h"
#include "qd_ptx.cuh"

namespace qd {

// row blocks: ~16K elements each (enough blocks for small-M / large-C layers too)
static int bn_splits(long long M, int C) {
  static const long long cap = getenv("QD_BN_SPLITS_MAX") ? atoll(getenv("QD_BN_SPLITS_MAX")) : 592;  // dev knob
  long long S = (M * C + 16383) / 16384;
  if (S > cap) S = cap;
  if (S > M) S = M;
  return (int)(S < 1 ? 1 : S);
}
// 8-channel vector kernels when C % 8 == 0 and C / 8 <= 256
static bool bn_vec(int C) { return C % 8 == 0 && C / 8 <= 256 && 256 % (C / 8) == 0; }

// 4-channel chunks (the backward kernels: their per-channel constants and
// partial sums would otherwise hold 8 x 12 registers per thread and halve the
// resident warps of these HBM-bound passes)
static bool bn_c4(int C) { return C % 4 == 0 && C / 4 <= 256 && 256 % (C / 4) == 0; }

template <typename T> struct BV;
template <> struct BV<bf16> {
  __device__ static void ld8(const bf16* p, float v[8]) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h[e]);
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
  }
  __device__ static void ld4(const bf16* p, float v[4]) {
    uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
    v[0] = f0.x; v[1] = f0.y; v[2] = f1.x; v[3] = f1.y;
  }
  __device__ static void st4(bf16* p, const float v[4]) {
    uint2 u;
    __nv_bfloat162 h0 = __floats2bfloat162_rn(v[0], v[1]), h1 = __floats2bfloat162_rn(v[2], v[3]);
    u.x = *reinterpret_cast<uint32_t*>(&h0);
    u.y = *reinterpret_cast<uint32_t*>(&h1);
    *reinterpret_cast<uint2*>(p) = u;
  }
  __device__ static void st8(bf16* p, const float v[8]) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      w[e] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct BV<float> {
  __device__ static void ld8(const float* p, float v[8]) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ static void ld4(const float* p, float v[4]) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
  __device__ static void st4(float* p, const float v[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
  __device__ static void st8(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

// vector reduction: thread = (8-channel chunk q, row lane); rows [r0, r1) of block s;
// lane partials folded in a fixed order through shared memory
template <typename T, int MODE>
__global__ void __launch_bounds__(256) bn_reduce_vec_kernel(long long M, int C, const T* __restrict__ y,
                                                            const T* __restrict__ dz, const float* mean,
                                                            const float* invstd, const float* gamma,
                                                            const float* beta, int relu, float* part) {
  ptx::pdl_wait();  // predecessor outputs complete (PDL launch)
  ptx::pdl_launch();
  __shared__ float red[2][256 * 8];
  const int CQ = C / 8, lanes = 256 / CQ;
  const int q = threadIdx.x % CQ, lane = threadIdx.x / CQ, c0 = q * 8;
  const int S = gridDim.x, s = blockIdx.x;
  const long long rows = (M + S - 1) / S;
  const long long r0 = (long long)s * rows;
  long long r1 = r0 + rows;
  if (r1 > M) r1 = M;
  float a0[8], a1[8], K[8], mu[8], is[8], ga[8], be[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) a0[e] = a1[e] = 0.f;
  if (lane < lanes) {
    if (MODE == 0) {
      BV<T>::ld8(y + c0, K);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        mu[e] = mean[c0 + e]; is[e] = invstd[c0 + e]; ga[e] = gamma[c0 + e]; be[e] = beta[c0 + e];
      }
    }
    long long r = r0 + lane;
    constexpr int U = MODE == 0 ? 8 : 2;  // rows whose loads are issued before any use
    for (; r + (U - 1) * lanes < r1; r += U * lanes) {
      float v[U][8], gv[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        BV<T>::ld8(y + (size_t)(r + u * lanes) * C + c0, v[u]);
        if (MODE != 0) BV<T>::ld8(dz + (size_t)(r + u * lanes) * C + c0, gv[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (MODE == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float d = v[u][e] - K[e];
            a0[e] += d;
            a1[e] = fmaf(d, d, a1[e]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float xh = (v[u][e] - mu[e]) * is[e];
            const float gg = (relu && !(fmaf(ga[e], xh, be[e]) > 0.f)) ? 0.f : gv[u][e];
            a0[e] += gg;
            a1[e] = fmaf(gg, xh, a1[e]);
          }
        }
      }
    }
    for (; r < r1; r += lanes) {
      float v[8];
      BV<T>::ld8(y + (size_t)r * C + c0, v);
      if (MODE == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = v[e] - K[e];
          a0[e] += d;
          a1[e] = fmaf(d, d, a1[e]);
        }
      } else {
        float g[8];
        BV<T>::ld8(dz + (size_t)r * C + c0, g);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xh = (v[e] - mu[e]) * is[e];
          const float gg = (relu && !(fmaf(ga[e], xh, be[e]) > 0.f)) ? 0.f : g[e];
          a0[e] += gg;
          a1[e] = fmaf(gg, xh, a1[e]);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red[0][threadIdx.x * 8 + e] = a0[e];
    red[1][threadIdx.x * 8 + e] = a1[e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int qq = c / 8, e = c % 8;
    float t0 = 0.f, t1 = 0.f;
    for (int l = 0; l < lanes; ++l) {
      t0 += red[0][(l * CQ + qq) * 8 + e];
      t1 += red[1][(l * CQ + qq) * 8 + e];
    }
    part[((size_t)s * 2 + 0) * C + c] = t0;
    part[((size_t)s * 2 + 1) * C + c] = t1;
  }
}

// thread = (8-channel chunk q, row lane) with 256 % (C / 8) == 0: the chunk's
// BN constants stay in registers (packed fp32 pairs) and rows stride by the
// grid's lane count; residual and ReLU are template parameters, so the
// no-residual instantiation keeps only 4 rows x 16 B of loads in registers
// (4 blocks per SM, one wave of a 4-per-SM grid)
template <typename T, bool RES, bool RELU>
__global__ void __launch_bounds__(256, 4) bn_apply_vec_kernel(long long rows, int C, const T* __restrict__ y,
                                                              const float* mean, const float* invstd,
                                                              const float* gamma, const float* beta,
                                                              T* __restrict__ z, const T* __restrict__ res) {
  ptx::pdl_wait();  // predecessor outputs complete (PDL launch)
  ptx::pdl_launch();
  const int CQ = C / 8, lanes = 256 / CQ;
  const int q = threadIdx.x % CQ, c0 = q * 8;
  float2 sc[4], sh[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {  // z = sc * y + sh (the backward's mask uses the same fmaf)
    float a[2], b[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int c = c0 + 2 * h + u;
      a[u] = gamma[c] * invstd[c];
      b[u] = beta[c] - a[u] * mean[c];
    }
    sc[h] = make_float2(a[0], a[1]);
    sh[h] = make_float2(b[0], b[1]);
  }
  const long long step = (long long)gridDim.x * lanes;
  long long r = (long long)blockIdx.x * lanes + threadIdx.x / CQ;
  auto emit = [&](long long rr, float (&v)[8], const float (&rv)[8]) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      float2 t = __ffma2_rn(sc[h], make_float2(v[2 * h], v[2 * h + 1]), sh[h]);
      if (RES) t = __fadd2_rn(t, make_float2(rv[2 * h], rv[2 * h + 1]));
      if (RELU) {
        t.x = t.x < 0.f ? 0.f : t.x;
        t.y = t.y < 0.f ? 0.f : t.y;
      }
      v[2 * h] = t.x;
      v[2 * h + 1] = t.y;
    }
    BV<T>::st8(z + (size_t)rr * C + c0, v);
  };
  // main loop: 4 rows whose loads are all issued before any use
  for (; r + 3 * step < rows; r += 4 * step) {
    float v[4][8], rv[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      BV<T>::ld8(y + (size_t)(r + u * step) * C + c0, v[u]);
      if (RES) BV<T>::ld8(res + (size_t)(r + u * step) * C + c0, rv[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) emit(r + u * step, v[u], rv[u]);
  }
  for (; r < rows; r += step) {
    float v[8], rv[8];
    BV<T>::ld8(y + (size_t)r * C + c0, v);
    if (RES) BV<T>::ld8(res + (size_t)r * C + c0, rv);
    emit(r, v, rv);
  }
}

template <typename T>
static void launch_apply_vec(long long M, int C, const T* y, const float* sm, const float* si, const float* gamma,
                             const float* beta, int relu, T* z, const T* res, cudaStream_t st) {
  long long g = ((M * C / 8) + 255) / 256;
  g = (g + 3) / 4;  // each thread takes >= 4 rows (the unguarded batch)
  const long long cap = 4LL * tc_num_sms();
  if (g > cap) g = cap;
#define QD_APPLY(R_, L_)                                                                                         \
  launch_pdl(bn_apply_vec_kernel<T, R_, L_>, dim3((unsigned)g), dim3(256), 0, st, M, C, y, sm, si, gamma, beta, z, \
             res)
  if (res)
    relu ? QD_APPLY(true, true) : QD_APPLY(true, false);
  else
    relu ? QD_APPLY(false, true) : QD_APPLY(false, false);
#undef QD_APPLY
}

template <typename T>
__global__ void __launch_bounds__(256, 3) bn_emit_D_vec_kernel(Plan P, const T* __restrict__ dz,
                                                               const T* __restrict__ y, const T* __restrict__ a,
                                                               const T* __restrict__ b, const float* mean,
                                                               const float* invstd, const float* gamma,
                                                               const float* beta, const float* dgamma,
                                                               const float* dbeta, int relu, T* __restrict__ D,
                                                               float* bpart) {
  ptx::pdl_wait();  // predecessor outputs complete (PDL launch)
  ptx::pdl_launch();
  // per-channel constants in shared memory (registers go to the loads in flight:
  // 3 blocks per SM); the same buffer takes the partial-sum fold afterwards.
  //   dy = kA g' + kC y + kB, g' = g masked where kA y + kQ <= 0 (the forward
  //   apply's z = kA y + kQ, same fmaf); kA = gamma inv, kC = -gamma inv^2 dgamma / M,
  //   kB = -gamma inv dbeta / M - kC mean
  __shared__ __align__(16) float sm[4 * 2048];
  const long long M = P.Mout;
  const int C = P.F, CQ = C / 8, lanes = 256 / CQ;
  const int q = threadIdx.x % CQ, lane = threadIdx.x / CQ, c0 = q * 8;
  const int S = gridDim.x, s = blockIdx.x;
  const long long rows = (M + S - 1) / S;
  const long long r0 = (long long)s * rows;
  long long r1 = r0 + rows;
  if (r1 > M) r1 = M;
  const bool mat = caches_ab(P.family), hasg = d_has_g(P.family);
  float* kA = sm;
  float* kB = sm + C;
  float* kC = sm + 2 * C;
  float* kQ = sm + 3 * C;
  {
    const float inv_m = 1.f / (float)M;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      const float mu = mean[c], is = invstd[c];
      const float ka = gamma[c] * is, kc = -ka * is * dgamma[c] * inv_m;
      kA[c] = ka;
      kQ[c] = beta[c] - ka * mu;
      kC[c] = kc;
      kB[c] = -ka * dbeta[c] * inv_m - kc * mu;
    }
  }
  __syncthreads();
  float s0[8], s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s0[e] = s1[e] = s2[e] = 0.f;
  if (lane < lanes) {
    for (long long r = r0 + lane; r < r1; r += lanes) {
      const size_t i = (size_t)r * C + c0;
      float v[8], g[8], av[8], bv[8];
      BV<T>::ld8(y + i, v);
      BV<T>::ld8(dz + i, g);
      if (mat) {
        BV<T>::ld8(a + i, av);
        BV<T>::ld8(b + i, bv);
      }
      float dyv[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float4 A4 = *reinterpret_cast<const float4*>(kA + c0 + 4 * h);
        const float4 B4 = *reinterpret_cast<const float4*>(kB + c0 + 4 * h);
        const float4 C4 = *reinterpret_cast<const float4*>(kC + c0 + 4 * h);
        const float4 Q4 = *reinterpret_cast<const float4*>(kQ + c0 + 4 * h);
        const float ka[4] = {A4.x, A4.y, A4.z, A4.w}, kb[4] = {B4.x, B4.y, B4.z, B4.w};
        const float kc[4] = {C4.x, C4.y, C4.z, C4.w}, kq[4] = {Q4.x, Q4.y, Q4.z, Q4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int f = 4 * h + e;
          const float gg = (relu && !(fmaf(ka[e], v[f], kq[e]) > 0.f)) ? 0.f : g[f];
          dyv[f] = fmaf(ka[e], gg, fmaf(kc[e], v[f], kb[e]));
        }
      }
      T* drow = D + (size_t)r * P.Jd + c0;
      if (mat) {
        float d0[8], d1[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          d0[e] = dyv[e] * bv[e];
          d1[e] = dyv[e] * av[e];
          s0[e] += d0[e];
          s1[e] += d1[e];
          s2[e] += dyv[e];
        }
        BV<T>::st8(drow, d0);
        BV<T>::st8(drow + C, d1);
        if (hasg) BV<T>::st8(drow + 2 * C, dyv);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) s0[e] += dyv[e];
        BV<T>::st8(drow, dyv);
      }
    }
  }
  __syncthreads();  // constants no longer read: the buffer takes the fold
  float (*red)[256 * 8] = reinterpret_cast<float (*)[256 * 8]>(sm);
  // 3 x 256 x 8 floats > 4 x 2048: fold in two rounds (s0, s1), then s2
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red[0][threadIdx.x * 8 + e] = s0[e];
    red[1][threadIdx.x * 8 + e] = s1[e];
  }
  __syncthreads();
  float* o = bpart + (size_t)s * P.Jd;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int qq = c / 8, e = c % 8;
    float t0 = 0.f, t1 = 0.f;
    for (int l = 0; l < lanes; ++l) {
      t0 += red[0][(l * CQ + qq) * 8 + e];
      t1 += red[1][(l * CQ + qq) * 8 + e];
    }
    o[c] = t0;
    if (mat) o[C + c] = t1;
  }
  if (mat && hasg) {
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 8; ++e) red[0][threadIdx.x * 8 + e] = s2[e];
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
      const int qq = c / 8, e = c % 8;
      float t2 = 0.f;
      for (int l = 0; l < lanes; ++l) t2 += red[0][(l * CQ + qq) * 8 + e];
      o[2 * C + c] = t2;
    }
  }
}

// Backward kernels on 4-channel chunks: thread = (chunk q, row lane), rows
// [r0, r1) of block s, two rows' loads issued before any use. The BN backward is
// folded into per-channel constants:
//   dy = kA g' + kC y + kB,  g' = g masked where kP y + kQ <= 0 (the ReLU of the
//   forward apply, z = kP y + kQ, evaluated with the same fmaf)
// with kA = gamma inv, kC = -gamma inv^2 dgamma / M, kB = -gamma inv dbeta / M - kC mean.
struct BnBwdK {
  float kA[4], kB[4], kC[4], kP[4], kQ[4];
  __device__ void load(int c0, long long M, const float* mean, const float* invstd, const float* gamma,
                       const float* beta, const float* dgamma, const float* dbeta) {
    const float inv_m = 1.f / (float)M;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float mu = mean[c0 + e], is = invstd[c0 + e], ga = gamma[c0 + e];
      kP[e] = ga * is;
      kQ[e] = beta[c0 + e] - kP[e] * mu;
      kA[e] = kP[e];
      kC[e] = dgamma ? -kP[e] * is * dgamma[c0 + e] * inv_m : 0.f;
      kB[e] = dbeta ? -kP[e] * dbeta[c0 + e] * inv_m - kC[e] * mu : 0.f;
    }
  }
};

template <typename T>
__global__ void __launch_bounds__(256, 4) bn_emit_D_c4_kernel(Plan P, const T* __restrict__ dz, const T* __restrict__ y,
                                                           const T* __restrict__ a, const T* __restrict__ b,
                                                           const float* mean, const float* invstd,
                                                           const float* gamma, const float* beta,
                                                           const float* dgamma, const float* dbeta, int relu,
                                                           T* __restrict__ D, float* bpart) {
  ptx::pdl_wait();  // dgamma / dbeta come from the finalize kernel (PDL launch)
  ptx::pdl_launch();
  __shared__ float red[3][256 * 4];
  const long long M = P.Mout;
  const int C = P.F, CQ = C / 4, lanes = 256 / CQ;
  const int q = threadIdx.x % CQ, lane = threadIdx.x / CQ, c0 = q * 4;
  const int S = gridDim.x, s = blockIdx.x;
  const long long rows = (M + S - 1) / S;
  const long long r0 = (long long)s * rows;
  long long r1 = r0 + rows;
  if (r1 > M) r1 = M;
  const bool mat = caches_ab(P.family), hasg = d_has_g(P.family);
  float s0[4], s1[4], s2[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) s0[e] = s1[e] = s2[e] = 0.f;
  if (lane < lanes) {
    BnBwdK k;
    k.load(c0, M, mean, invstd, gamma, beta, dgamma, dbeta);
    long long r = r0 + lane;
    constexpr int U = 2;
    for (; r < r1; r += U * lanes) {
      float v[U][4], g[U][4], av[U][4], bv[U][4];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // all loads of the batch in flight (clamped rows)
        const long long ru = r + u * lanes;
        ok[u] = ru < r1;
        const size_t i = (size_t)(ok[u] ? ru : r) * C + c0;
        BV<T>::ld4(y + i, v[u]);
        BV<T>::ld4(dz + i, g[u]);
        if (mat) {
          BV<T>::ld4(a + i, av[u]);
          BV<T>::ld4(b + i, bv[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        float dy[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float gg = (relu && !(fmaf(k.kP[e], v[u][e], k.kQ[e]) > 0.f)) ? 0.f : g[u][e];
          dy[e] = fmaf(k.kA[e], gg, fmaf(k.kC[e], v[u][e], k.kB[e]));
        }
        T* drow = D + (size_t)(r + u * lanes) * P.Jd + c0;
        if (mat) {
          float d0[4], d1[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            d0[e] = dy[e] * bv[u][e];
            d1[e] = dy[e] * av[u][e];
            s0[e] += d0[e];
            s1[e] += d1[e];
            s2[e] += dy[e];
          }
          BV<T>::st4(drow, d0);
          BV<T>::st4(drow + C, d1);
          if (hasg) BV<T>::st4(drow + 2 * C, dy);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) s0[e] += dy[e];
          BV<T>::st4(drow, dy);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    red[0][threadIdx.x * 4 + e] = s0[e];
    red[1][threadIdx.x * 4 + e] = s1[e];
    red[2][threadIdx.x * 4 + e] = s2[e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int qq = c / 4, e = c % 4;
    float t0 = 0.f, t1 = 0.f, t2 = 0.f;
    for (int l = 0; l < lanes; ++l) {
      t0 += red[0][(l * CQ + qq) * 4 + e];
      t1 += red[1][(l * CQ + qq) * 4 + e];
      t2 += red[2][(l * CQ + qq) * 4 + e];
    }
    float* o = bpart + (size_t)s * P.Jd;
    if (mat) {
      o[c] = t0;
      o[C + c] = t1;
      if (hasg) o[2 * C + c] = t2;
    } else {
      o[c] = t0;
    }
  }
}

// backward reduction (sum g', sum g' xhat) on 4-channel chunks, four rows' loads
// in flight; xhat = (y - mean) inv
template <typename T>
__global__ void __launch_bounds__(256, 4) bn_bwd_reduce_c4_kernel(long long M, int C, const T* __restrict__ y,
                                                               const T* __restrict__ dz, const float* mean,
                                                               const float* invstd, const float* gamma,
                                                               const float* beta, int relu, float* part) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  __shared__ float red[2][256 * 4];
  const int CQ = C / 4, lanes = 256 / CQ;
  const int q = threadIdx.x % CQ, lane = threadIdx.x / CQ, c0 = q * 4;
  const int S = gridDim.x, s = blockIdx.x;
  const long long rows = (M + S - 1) / S;
  const long long r0 = (long long)s * rows;
  long long r1 = r0 + rows;
  if (r1 > M) r1 = M;
  float a0[4], a1[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) a0[e] = a1[e] = 0.f;
  if (lane < lanes) {
    float mu[4], is[4], kP[4], kQ[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      mu[e] = mean[c0 + e]; is[e] = invstd[c0 + e];
      kP[e] = gamma[c0 + e] * is[e];
      kQ[e] = beta[c0 + e] - kP[e] * mu[e];
    }
    constexpr int U = 4;
    for (long long r = r0 + lane; r < r1; r += U * lanes) {
      float v[U][4], g[U][4];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long ru = r + u * lanes;
        ok[u] = ru < r1;
        const size_t i = (size_t)(ok[u] ? ru : r) * C + c0;
        BV<T>::ld4(y + i, v[u]);
        BV<T>::ld4(dz + i, g[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float xh = (v[u][e] - mu[e]) * is[e];
          const float gg = (relu && !(fmaf(kP[e], v[u][e], kQ[e]) > 0.f)) ? 0.f : g[u][e];
          a0[e] += gg;
          a1[e] = fmaf(gg, xh, a1[e]);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    red[0][threadIdx.x * 4 + e] = a0[e];
    red[1][threadIdx.x * 4 + e] = a1[e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int qq = c / 4, e = c % 4;
    float t0 = 0.f, t1 = 0.f;
    for (int l = 0; l < lanes; ++l) {
      t0 += red[0][(l * CQ + qq) * 4 + e];
      t1 += red[1][(l * CQ + qq) * 4 + e];
    }
    part[((size_t)s * 2 + 0) * C + c] = t0;
    part[((size_t)s * 2 + 1) * C + c] = t1;
  }
}

// workspace: [reduction partial rows][2C] then [D-emission partial rows][Jd]
// (the register-streaming emit: S rows; the streaming emit: <= bn_stream_rows(),
// its fold group rows included)
static size_t bn_emit_rows(long long M, int C) {
  const size_t a = (size_t)bn_splits(M, C), b = bn_stream_rows();
  return a > b ? a : b;
}
size_t bn_workspace_bytes(long long M, int C, int Jd) {
  return (size_t)bn_splits(M, C) * 2 * C * 4 + bn_emit_rows(M, C) * Jd * 4 + 256;
}

// per-block partials over rows [r0, r1): thread = (channel c = tid % C? no: strided)
// Scalar channel loop per thread keeps it general (any C); rows are split over
// the block's thread groups and folded in a fixed order through shared memory.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) bn_reduce_kernel(long long M, int C, const T* __restrict__ y,
                                                        const T* __restrict__ dz, const float* mean,
                                                        const float* invstd, const float* gamma,
                                                        const float* beta, int relu, float* part) {
  // MODE 0: sum(y - K), sum((y - K)^2) with K = y[0][c]
  // MODE 1: sum(g), sum(g xhat), g = dz * [relu ? z > 0 : 1]
  __shared__ float red[2][256];
  const int S = gridDim.x, s = blockIdx.x;
  const long long rows = (M + S - 1) / S;
  const long long r0 = (long long)s * rows;
  long long r1 = r0 + rows;
  if (r1 > M) r1 = M;
  const int G = blockDim.x < C ? 1 : blockDim.x / C;  // row groups
  const int cpt = blockDim.x < C ? 1 : 0;
  for (int c0 = 0; c0 < C; c0 += (cpt ? blockDim.x : C)) {
    int c = c0 + (cpt ? (int)threadIdx.x : (int)threadIdx.x % C);
    const int grp = cpt ? 0 : (int)threadIdx.x / C;
    float a0 = 0.f, a1 = 0.f;
    const bool act = c < C && grp < G;
    if (act) {
      if (MODE == 0) {
        const float K = ld(y + c);
        for (long long r = r0 + grp; r < r1; r += G) {
          const float v = ld(y + (size_t)r * C + c) - K;
          a0 += v;
          a1 = fmaf(v, v, a1);
        }
      } else {
        const float mu = mean[c], is = invstd[c], ga = gamma[c], be = beta[c];
        for (long long r = r0 + grp; r < r1; r += G) {
          const size_t i = (size_t)r * C + c;
          const float xh = (ld(y + i) - mu) * is;
          float g = ld(dz + i);
          if (relu && !(fmaf(ga, xh, be) > 0.f)) g = 0.f;
          a0 += g;
          a1 = fmaf(g, xh, a1);
        }
      }
    }
    red[0][threadIdx.x] = a0;
    red[1][threadIdx.x] = a1;
    __syncthreads();
    if (act && grp == 0) {
      float t0 = 0.f, t1 = 0.f;
      for (int gq = 0; gq < G; ++gq) {
        t0 += red[0][gq * C + (c - c0)];
        t1 += red[1][gq * C + (c - c0)];
      }
      part[((size_t)s * 2 + 0) * C + c] = t0;
      part[((size_t)s * 2 + 1) * C + c] = t1;
    }
    __syncthreads();
  }
}

// fold the S x (2, C) partials: block = 8 channels x both sums (16 columns) x 64
// row groups; group g sums rows g, g + 64, ... in order (~S/64 <= 10 loads, all
// issued before use: the fold is L2-latency bound, and 32 channels x 16 groups
// took five dependent rounds, ~10 us per finalize), then 8 threads per column
// add 8 group totals each and one adds those 8, in order (deterministic).
constexpr int kFoldCh = 8;
__device__ __forceinline__ bool bn_fold2(int C, int S, const float* part, float& s1, float& s2) {
  __shared__ float red[64][2 * kFoldCh + 1];
  __shared__ float red8[8][2 * kFoldCh + 1];
  const int col = threadIdx.x % (2 * kFoldCh), grp = threadIdx.x / (2 * kFoldCh);
  const int k = col / kFoldCh, c = blockIdx.x * kFoldCh + col % kFoldCh;
  float acc = 0.f;
  if (c < C) {
    const float* p = part + (size_t)k * C + c;
    const size_t step = (size_t)2 * C;
    int sp = grp;
    for (; sp + 7 * 64 < S; sp += 8 * 64) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = p[(size_t)(sp + 64 * u) * step];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = sp + 64 * u < S ? p[(size_t)(sp + 64 * u) * step] : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  red[grp][col] = acc;
  __syncthreads();
  if (grp < 8) {
    float t = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) t += red[grp * 8 + g][col];
    red8[grp][col] = t;
  }
  __syncthreads();
  if (threadIdx.x >= kFoldCh || blockIdx.x * kFoldCh + (int)threadIdx.x >= C) return false;
  s1 = 0.f;
  s2 = 0.f;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    s1 += red8[g][threadIdx.x];
    s2 += red8[g][threadIdx.x + kFoldCh];
  }
  return true;
}

template <typename T>
__global__ void __launch_bounds__(1024) bn_stats_finalize(long long M, int C, int S, const T* y, const float* part,
                                                          float eps, float momentum, int training, float* run_mean,
                                                          float* run_var, float* save_mean, float* save_invstd) {
  ptx::pdl_wait();  // predecessor outputs complete (PDL launch)
  ptx::pdl_launch();
  float s1, s2;
  if (!bn_fold2(C, S, part, s1, s2)) return;
  const int c = blockIdx.x * kFoldCh + threadIdx.x;
  const float inv_m = 1.f / (float)M;
  const float dm = s1 * inv_m;
  float var = s2 * inv_m - dm * dm;  // biased (tensor.py:444)
  if (var < 0.f) var = 0.f;
  const float mean = ld(y + c) + dm;
  save_mean[c] = mean;
  save_invstd[c] = rsqrtf(var + eps);
  if (training && run_mean) {  // tensor.py:445-450 (biased var in the running update too)
    run_mean[c] = run_mean[c] * (1.f - momentum) + momentum * mean;
    run_var[c] = run_var[c] * (1.f - momentum) + momentum * var;
  }
}

template <typename T>
__global__ void bn_apply_kernel(long long n, int C, const T* y, const float* mean, const float* invstd,
                                const float* gamma, const float* beta, int relu, T* z, const T* res) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    float v = fmaf(gamma[c], (ld(y + i) - mean[c]) * invstd[c], beta[c]) + (res ? ld(res + i) : 0.f);
    if (relu && v < 0.f) v = 0.f;
    z[i] = cvt<T>(v);
  }
}

__global__ void __launch_bounds__(1024) bn_grad_finalize(int C, int S, const float* part, float* dgamma,
                                                          float* dbeta) {
  ptx::pdl_wait();  // predecessor outputs complete (PDL launch)
  ptx::pdl_launch();
  float s1, s2;
  if (!bn_fold2(C, S, part, s1, s2)) return;
  const int c = blockIdx.x * kFoldCh + threadIdx.x;
  dbeta[c] = s1;
  dgamma[c] = s2;
}

// dy = gamma inv / m (m g - dbeta - xhat dgamma) (tensor.py:558-566 with s1 = gamma dbeta,
// s2 = gamma dgamma), then D and the layer's bias partials; block s covers rows [r0, r1)
template <typename T>
__global__ void __launch_bounds__(256) bn_emit_D_kernel(Plan P, const T* __restrict__ dz, const T* __restrict__ y,
                                                        const T* __restrict__ a, const T* __restrict__ b,
                                                        const float* mean, const float* invstd, const float* gamma,
                                                        const float* beta, const float* dgamma, const float* dbeta,
                                                        int relu, T* D, float* bpart) {
  __shared__ float red[3][256];
  const long long M = P.Mout;
  const int C = P.F, S = gridDim.x, s = blockIdx.x;
  const long long rows = (M + S - 1) / S;
  const long long r0 = (long long)s * rows;
  long long r1 = r0 + rows;
  if (r1 > M) r1 = M;
  const bool mat = caches_ab(P.family), hasg = d_has_g(P.family);
  const int G = blockDim.x < C ? 1 : blockDim.x / C;
  const int cpt = blockDim.x < C ? 1 : 0;
  const float inv_m = 1.f / (float)M;
  for (int c0 = 0; c0 < C; c0 += (cpt ? blockDim.x : C)) {
    int c = c0 + (cpt ? (int)threadIdx.x : (int)threadIdx.x % C);
    const int grp = cpt ? 0 : (int)threadIdx.x / C;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
    const bool act = c < C && grp < G;
    if (act) {
      const float mu = mean[c], is = invstd[c], ga = gamma[c], be = beta[c], dg = dgamma[c], db = dbeta[c];
      const float k = ga * is * inv_m;
      for (long long r = r0 + grp; r < r1; r += G) {
        const size_t i = (size_t)r * C + c;
        const float xh = (ld(y + i) - mu) * is;
        float g = ld(dz + i);
        if (relu && !(fmaf(ga, xh, be) > 0.f)) g = 0.f;
        const float dyv = k * ((float)M * g - db - xh * dg);
        T* drow = D + (size_t)r * P.Jd;
        if (mat) {
          const float d0 = dyv * ld(b + i), d1 = dyv * ld(a + i);
          drow[c] = cvt<T>(d0);
          drow[C + c] = cvt<T>(d1);
          if (hasg) drow[2 * C + c] = cvt<T>(dyv);
          s0 += d0;
          s1 += d1;
          s2 += dyv;
        } else {
          drow[c] = cvt<T>(dyv);
          s0 += dyv;
        }
      }
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    red[2][threadIdx.x] = s2;
    __syncthreads();
    if (act && grp == 0) {
      float t0 = 0.f, t1 = 0.f, t2 = 0.f;
      for (int gq = 0; gq < G; ++gq) {
        t0 += red[0][gq * C + (c - c0)];
        t1 += red[1][gq * C + (c - c0)];
        t2 += red[2][gq * C + (c - c0)];
      }
      float* o = bpart + (size_t)s * P.Jd;
      if (mat) {
        o[c] = t0;
        o[C + c] = t1;
        if (hasg) o[2 * C + c] = t2;
      } else {
        o[c] = t0;
      }
    }
    __syncthreads();
  }
}

template <typename T>
static int bn_forward_t(long long M, int C, const T* y, const float* gamma, const float* beta, float* rm, float* rv,
                        float momentum, float eps, int relu, int training, T* z, float* sm, float* si, char* ws,
                        cudaStream_t st, const T* res) {
  if (dev_skip("bn")) return QD_OK;
  const int S = bn_splits(M, C);
  float* part = (float*)ws;
  if (training) {
    if (bn_vec(C))
      launch_pdl(bn_reduce_vec_kernel<T, 0>, dim3(S), dim3(256), 0, st, M, C, y, (const T*)nullptr, (const float*)nullptr,
                 (const float*)nullptr, (const float*)nullptr, (const float*)nullptr, 0, part);
    else
      bn_reduce_kernel<T, 0><<<S, 256, 0, st>>>(M, C, y, nullptr, nullptr, nullptr, nullptr, nullptr, 0, part);
    count_launch(st, "bn_stats");
    launch_pdl(bn_stats_finalize<T>, dim3((C + kFoldCh - 1) / kFoldCh), dim3(1024), 0, st, M, C, S, y, (const float*)part, eps,
               momentum, 1, rm, rv, sm, si);
    count_launch(st, "bn_stats_finalize");
  }
  const long long n = M * C;
  if (bn_vec(C)) {
    launch_apply_vec<T>(M, C, y, sm, si, gamma, beta, relu, z, res, st);
  } else {
    long long g = (n + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    bn_apply_kernel<T><<<(int)g, 256, 0, st>>>(n, C, y, sm, si, gamma, beta, relu, z, res);
  }
  count_launch(st, "bn_apply");
  return check_launch("bn forward");
}

template <typename T>
static int bn_backward_D_t(const Plan& P, const T* dz, const T* y, const T* a, const T* b, const float* gamma,
                           const float* beta, const float* sm, const float* si, int relu, T* D, float* dgamma,
                           float* dbeta, float* const db[3], char* ws, cudaStream_t st) {
  if (dev_skip("bn")) return QD_OK;
  const long long M = P.Mout;
  const int C = P.F, S = bn_splits(M, C);
  float* part = (float*)ws;
  float* bpart = part + (size_t)S * 2 * C;
  if (bn_c4(C) && !getenv("QD_BN_C8"))
    launch_pdl(bn_bwd_reduce_c4_kernel<T>, dim3(S), dim3(256), 0, st, M, C, y, dz, sm, si, gamma, beta, relu, part);
  else if (bn_vec(C))
    launch_pdl(bn_reduce_vec_kernel<T, 1>, dim3(S), dim3(256), 0, st, M, C, y, dz, sm, si, gamma, beta, relu, part);
  else
    bn_reduce_kernel<T, 1><<<S, 256, 0, st>>>(M, C, y, dz, sm, si, gamma, beta, relu, part);
  count_launch(st, "bn_bwd_reduce");
  launch_pdl(bn_grad_finalize, dim3((C + kFoldCh - 1) / kFoldCh), dim3(1024), 0, st, C, S, (const float*)part, dgamma,
             dbeta);
  count_launch(st, "bn_bwd_finalize");
  if (bn_stream_ok(M, C, P.dtype))  // qd_bnstream.cu: bulk-copy streaming emit, bias folded in-kernel
    return bn_emit_stream(P, dz, y, a, b, gamma, beta, sm, si, relu, D, dgamma, dbeta, db, bpart, st);
  if (bn_c4(C) && getenv("QD_BN_C4"))  // dev: the 4-channel emit (slower, measured)
    launch_pdl(bn_emit_D_c4_kernel<T>, dim3(S), dim3(256), 0, st, P, dz, y, a, b, sm, si, gamma, beta,
               (const float*)dgamma, (const float*)dbeta, relu, D, bpart);
  else if (bn_vec(C))
    launch_pdl(bn_emit_D_vec_kernel<T>, dim3(S), dim3(256), 0, st, P, dz, y, a, b, sm, si, gamma, beta,
               (const float*)dgamma, (const float*)dbeta, relu, D, bpart);
  else
    bn_emit_D_kernel<T><<<S, 256, 0, st>>>(P, dz, y, a, b, sm, si, gamma, beta, dgamma, dbeta, relu, D, bpart);
  count_launch(st, "bn_emit_D");
  if (db && db[0] && P.nbias) launch_bias_finish(P, bpart, S, db, st);
  return check_launch("bn backward");
}

int bn_forward(long long M, int C, int dtype, const void* y, const float* gamma, const float* beta, float* rm,
               float* rv, float momentum, float eps, int relu, int training, void* z, float* sm, float* si, char* ws,
               cudaStream_t st, const void* res) {
  if (dtype == QD_BF16)
    return bn_forward_t<bf16>(M, C, (const bf16*)y, gamma, beta, rm, rv, momentum, eps, relu, training, (bf16*)z, sm,
                              si, ws, st, (const bf16*)res);
  return bn_forward_t<float>(M, C, (const float*)y, gamma, beta, rm, rv, momentum, eps, relu, training, (float*)z,
                             sm, si, ws, st, (const float*)res);
}

// Chan's parallel-variance merge of two (count, mean, M2) groups
__device__ __forceinline__ void chan_merge(float& n, float& mean, float& m2, float nb, float mb, float m2b) {
  const float nt = n + nb;
  if (nb == 0.f) return;
  if (n == 0.f) {
    n = nb; mean = mb; m2 = m2b;
    return;
  }
  const float d = mb - mean, f = nb / nt;
  mean += d * f;
  m2 += m2b + d * d * n * f;
  n = nt;
}

// statistics rows of the fprop epilogue -> batch mean / invstd (+ running update):
// block = 32 channels x 32 row groups; group g merges rows g, g + 32, ... in order,
// then the 32 group results merge in order (fixed order: deterministic)
__global__ void __launch_bounds__(1024) bn_merge_finalize(int C, int R, const float* __restrict__ stats, float eps,
                                                          float momentum, int training, float* run_mean,
                                                          float* run_var, float* save_mean, float* save_invstd) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  __shared__ float sn[32][33], sm_[32][33], sq[32][33];
  const int col = threadIdx.x % 32, grp = threadIdx.x / 32;
  const int c = blockIdx.x * 32 + col;
  const float* mean_r = stats;
  const float* m2_r = stats + (size_t)R * C;
  const float* cnt_r = stats + (size_t)2 * R * C;
  float n = 0.f, mean = 0.f, m2 = 0.f;
  if (c < C)
    for (int r = grp; r < R; r += 32) chan_merge(n, mean, m2, __ldg(cnt_r + r), __ldg(mean_r + (size_t)r * C + c),
                                                 __ldg(m2_r + (size_t)r * C + c));
  sn[grp][col] = n; sm_[grp][col] = mean; sq[grp][col] = m2;
  __syncthreads();
  if (grp != 0 || c >= C) return;
  n = 0.f; mean = 0.f; m2 = 0.f;
  for (int g = 0; g < 32; ++g) chan_merge(n, mean, m2, sn[g][col], sm_[g][col], sq[g][col]);
  const float var = n > 0.f ? m2 / n : 0.f;  // biased (tensor.py:444)
  save_mean[c] = mean;
  save_invstd[c] = rsqrtf(var + eps);
  if (training && run_mean) {  // tensor.py:445-450 (biased var in the running update too)
    run_mean[c] = run_mean[c] * (1.f - momentum) + momentum * mean;
    run_var[c] = run_var[c] * (1.f - momentum) + momentum * var;
  }
}

template <typename T>
static int bn_forward_stats_t(long long M, int C, const T* y, const T* res, const float* stats, int R,
                              const float* gamma, const float* beta, float* rm, float* rv, float momentum, float eps,
                              int relu, int training, T* z, float* sm, float* si, cudaStream_t st) {
  if (dev_skip("bn")) return QD_OK;
  launch_pdl(bn_merge_finalize, dim3((C + 31) / 32), dim3(1024), 0, st, C, R, stats, eps, momentum, training, rm, rv,
             sm, si);
  count_launch(st, "bn_stats_merge");
  const long long n = M * C;
  if (bn_vec(C)) {
    launch_apply_vec<T>(M, C, y, sm, si, gamma, beta, relu, z, res, st);
  } else {
    long long g = (n + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    bn_apply_kernel<T><<<(int)g, 256, 0, st>>>(n, C, y, sm, si, gamma, beta, relu, z, res);
  }
  count_launch(st, "bn_apply");
  return check_launch("bn forward (epilogue statistics)");
}

int bn_forward_stats(long long M, int C, int dtype, const void* y, const void* res, const float* stats, int rows,
                     const float* gamma, const float* beta, float* rm, float* rv, float momentum, float eps, int relu,
                     int training, void* z, float* sm, float* si, cudaStream_t st) {
  if (dtype == QD_BF16)
    return bn_forward_stats_t<bf16>(M, C, (const bf16*)y, (const bf16*)res, stats, rows, gamma, beta, rm, rv, momentum,
                                    eps, relu, training, (bf16*)z, sm, si, st);
  return bn_forward_stats_t<float>(M, C, (const float*)y, (const float*)res, stats, rows, gamma, beta, rm, rv,
                                   momentum, eps, relu, training, (float*)z, sm, si, st);
}

int bn_backward_D(const Plan& P, const void* dz, const void* y, const void* a, const void* b, const float* gamma,
                  const float* beta, const float* sm, const float* si, int relu, void* D, float* dgamma,
                  float* dbeta, float* const db[3], char* ws, cudaStream_t st) {
  if (P.dtype == QD_BF16)
    return bn_backward_D_t<bf16>(P, (const bf16*)dz, (const bf16*)y, (const bf16*)a, (const bf16*)b, gamma, beta, sm,
                                 si, relu, (bf16*)D, dgamma, dbeta, db, ws, st);
  return bn_backward_D_t<float>(P, (const float*)dz, (const float*)y, (const float*)a, (const float*)b, gamma, beta,
                                sm, si, relu, (float*)D, dgamma, dbeta, db, ws, st);
}

}  // namespace qd
