// Depth-wise quadratic convolution (kind = dwconv, one r x r filter per channel,
// C == F): the MobileNet rows of the paper. Reference:
// tensor.py:367-418 (dw_im2col, dwconv_forward_raw, dwconv_backward_raw) under the
// family algebra of neurons.py:235-276 / :393-444.
//
// This work is memory-bound (r*r MACs per loaded element), so it runs as direct
// CUDA-core kernels over NHWC tensors with one thread per (pixel, channel):
// consecutive threads touch consecutive channels, i.e. contiguous bytes, for x,
// y, D and dx alike. fp32 accumulation for both dtypes.
//
//   forward  acc_r = dwconv(xin_r, W_r) per weight role, family epilogue fused
//   backward D from the shared prologue kernels (g b | g a | g, or 2 g a for t3),
//            dgrad as the transposed gather over the taps (x*x branches get the
//            2 x factor), wgrad as per-(role, tap, channel) partial sums over
//            pixel ranges folded in a fixed order (deterministic).
#include <stdio.h>
#include "qd_kernels.h"
#include "qd_dw.cuh"

namespace qd {

static DwArgs dw_args(const Plan& P) {
  DwArgs a;
  a.family = P.family; a.N = P.N; a.C = P.C; a.H = P.H; a.W = P.W; a.OH = P.OH; a.OW = P.OW;
  a.r = P.r; a.s = P.s; a.p = P.p; a.Min = P.Min; a.Mout = P.Mout; a.Jd = P.Jd;
  return a;
}

static inline int dw_grid(long long n) {
  long long g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return (int)(g < 1 ? 1 : g);
}

// plain = 1: write acc of role 0 only (t3 backward recompute of a = Wa x)
template <typename T>
__global__ void __launch_bounds__(256) dw_fwd_kernel(DwArgs A, const T* __restrict__ x,
                                                     const float* __restrict__ Wp, const float* b0,
                                                     const float* b1, const float* b2, T* y, T* oa, T* ob,
                                                     int plain) {
  const DwFam fm = dw_fam(A.family);
  const int rr = A.r * A.r;
  const long long total = A.Mout * A.C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % A.C);
    const long long m = i / A.C;
    const int ow = (int)(m % A.OW);
    const long long t = m / A.OW;
    const int oh = (int)(t % A.OH), n = (int)(t / A.OH);
    float acc[3] = {0.f, 0.f, 0.f};
    for (int dy = 0; dy < A.r; ++dy) {
      const int ih = oh * A.s + dy - A.p;
      if (ih < 0 || ih >= A.H) continue;
      for (int dx = 0; dx < A.r; ++dx) {
        const int iw = ow * A.s + dx - A.p;
        if (iw < 0 || iw >= A.W) continue;
        const float v = ld(x + (((size_t)n * A.H + ih) * A.W + iw) * A.C + c);
        const int tap = dy * A.r + dx;
#pragma unroll
        for (int ro = 0; ro < 3; ++ro)
          if (ro < fm.nroles) {
            const float w = __ldg(Wp + ((size_t)ro * rr + tap) * A.C + c);
            acc[ro] = fmaf(w, fm.sq[ro] ? v * v : v, acc[ro]);
          }
      }
    }
    if (plain) {
      y[i] = cvt<T>(acc[0]);
      continue;
    }
    float out;
    switch (A.family) {
      case QD_FAM_FIRST_ORDER: out = acc[0] + b0[c]; break;
      case QD_FAM_T3: out = acc[0] * acc[0]; break;
      case QD_FAM_T4:
        oa[i] = cvt<T>(acc[0]); ob[i] = cvt<T>(acc[1]);
        out = acc[0] * acc[1];
        break;
      case QD_FAM_PROPOSED: {
        const float av = acc[0] + b0[c], bv = acc[1] + b1[c];
        oa[i] = cvt<T>(av); ob[i] = cvt<T>(bv);
        out = av * bv + (acc[2] + b2[c]);
        break;
      }
      case QD_FAM_T2_LINEAR: out = acc[0] + acc[1]; break;
      case QD_FAM_T2AND4:
        oa[i] = cvt<T>(acc[0]); ob[i] = cvt<T>(acc[1]);
        out = acc[0] * acc[1] + acc[2];
        break;
      default: out = acc[0]; break;  // t2
    }
    y[i] = cvt<T>(out);
  }
}

// dx[n, ih, iw, c] = sum over roles and taps of D_din(r)[o(tap)] W_r[c, tap];
// x*x roles accumulate separately and get the 2 x factor (neurons.py:400-405)
template <typename T>
__global__ void __launch_bounds__(256) dw_dgrad_kernel(DwArgs A, const T* __restrict__ x, const T* __restrict__ D,
                                                       const float* __restrict__ Wp, T* dx) {
  const DwFam fm = dw_fam(A.family);
  const int rr = A.r * A.r;
  const long long total = A.Min * A.C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % A.C);
    const long long m = i / A.C;
    const int iw = (int)(m % A.W);
    const long long t = m / A.W;
    const int ih = (int)(t % A.H), n = (int)(t / A.H);
    float lin = 0.f, sq = 0.f;
    for (int dy = 0; dy < A.r; ++dy) {
      int th = ih + A.p - dy;
      if (th < 0 || th % A.s) continue;
      const int oh = th / A.s;
      if (oh >= A.OH) continue;
      for (int dxx = 0; dxx < A.r; ++dxx) {
        int tw = iw + A.p - dxx;
        if (tw < 0 || tw % A.s) continue;
        const int ow = tw / A.s;
        if (ow >= A.OW) continue;
        const size_t orow = (((size_t)n * A.OH + oh) * A.OW + ow) * A.Jd;
        const int tap = dy * A.r + dxx;
#pragma unroll
        for (int ro = 0; ro < 3; ++ro)
          if (ro < fm.nroles) {
            const float d = ld(D + orow + (size_t)fm.din[ro] * A.C + c);
            const float w = __ldg(Wp + ((size_t)ro * rr + tap) * A.C + c);
            if (fm.sq[ro]) sq = fmaf(d, w, sq);
            else lin = fmaf(d, w, lin);
          }
      }
    }
    float v = lin;
    if (fm.sq[0] || fm.sq[1] || fm.sq[2]) {
      const float tt = sq * ld(x + i);
      v += tt + tt;
    }
    dx[i] = cvt<T>(v);
  }
}

// part[s][role][tap][c] = sum over output pixels of range s of D_din(role) * xin_role(tap)
template <typename T>
__global__ void __launch_bounds__(256) dw_wgrad_kernel(DwArgs A, const T* __restrict__ x, const T* __restrict__ D,
                                                       float* part, long long rows_per) {
  const DwFam fm = dw_fam(A.family);
  const int rr = A.r * A.r;
  const int nrc = fm.nroles * rr * A.C;
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nrc) return;
  const int c = id % A.C, rt = id / A.C, tap = rt % rr, ro = rt / rr;
  const int dy = tap / A.r, dxx = tap % A.r;
  const int s = blockIdx.y;
  const long long m0 = (long long)s * rows_per;
  long long m1 = m0 + rows_per;
  if (m1 > A.Mout) m1 = A.Mout;
  const int dofs = fm.din[ro] * A.C + c;
  const bool sq = fm.sq[ro] != 0;
  float acc0 = 0.f, acc1 = 0.f;
  int ow = (int)(m0 % A.OW);
  long long t = m0 / A.OW;
  int oh = (int)(t % A.OH), n = (int)(t / A.OH);
  for (long long m = m0; m < m1; ++m) {
    const int ih = oh * A.s + dy - A.p, iw = ow * A.s + dxx - A.p;
    if (ih >= 0 && ih < A.H && iw >= 0 && iw < A.W) {
      const float v = ld(x + (((size_t)n * A.H + ih) * A.W + iw) * A.C + c);
      const float d = ld(D + (size_t)m * A.Jd + dofs);
      if (m & 1) acc1 = fmaf(d, sq ? v * v : v, acc1);
      else acc0 = fmaf(d, sq ? v * v : v, acc0);
    }
    if (++ow == A.OW) {
      ow = 0;
      if (++oh == A.OH) { oh = 0; ++n; }
    }
  }
  part[(size_t)s * nrc + id] = acc0 + acc1;
}

// ---- 8-channel vector versions (C % 8 == 0): 16-B loads/stores for bf16 ---------
template <typename T> struct Vec8;
template <> struct Vec8<bf16> {
  __device__ static void load(const bf16* p, float v[8]) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(h[e]);
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
  }
  __device__ static void store(bf16* p, const float v[8]) {
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
template <> struct Vec8<float> {
  __device__ static void load(const float* p, float v[8]) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ static void store(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};
__device__ __forceinline__ void ldw8(const float* p, float w[8]) {
  float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

template <typename T>
__global__ void __launch_bounds__(256) dw_fwd_vec_kernel(DwArgs A, const T* __restrict__ x,
                                                         const float* __restrict__ Wp, const float* b0,
                                                         const float* b1, const float* b2, T* y, T* oa, T* ob,
                                                         int plain) {
  extern __shared__ float sW[];  // [role][tap][C], the layer's filters
  const DwFam fm = dw_fam(A.family);
  const int rr = A.r * A.r, CQ = A.C / 8;
  for (int i = threadIdx.x; i < fm.nroles * rr * A.C / 4; i += blockDim.x)
    reinterpret_cast<float4*>(sW)[i] = __ldg(reinterpret_cast<const float4*>(Wp) + i);
  __syncthreads();
  const int total = (int)(A.Mout * CQ);  // < 2^31 (host check): 32-bit index math
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i % CQ, c0 = q * 8;
    const int m = i / CQ;
    const int ow = m % A.OW;
    const int t = m / A.OW;
    const int oh = t % A.OH, n = t / A.OH;
    float acc[3][8];
#pragma unroll
    for (int ro = 0; ro < 3; ++ro)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[ro][e] = 0.f;
    for (int dy = 0; dy < A.r; ++dy) {
      const int ih = oh * A.s + dy - A.p;
      if (ih < 0 || ih >= A.H) continue;
      for (int dx = 0; dx < A.r; ++dx) {
        const int iw = ow * A.s + dx - A.p;
        if (iw < 0 || iw >= A.W) continue;
        float v[8], v2[8];
        Vec8<T>::load(x + (((size_t)n * A.H + ih) * A.W + iw) * A.C + c0, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) v2[e] = v[e] * v[e];
        const int tap = dy * A.r + dx;
#pragma unroll
        for (int ro = 0; ro < 3; ++ro)
          if (ro < fm.nroles) {
            const float4* wp = reinterpret_cast<const float4*>(sW + (ro * rr + tap) * A.C + c0);
            const float4 w0 = wp[0], w1 = wp[1];
            const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[ro][e] = fmaf(w[e], fm.sq[ro] ? v2[e] : v[e], acc[ro][e]);
          }
      }
    }
    const size_t o = (size_t)m * A.C + c0;
    if (plain) {
      Vec8<T>::store(y + o, acc[0]);
      continue;
    }
    float out[8], av[8], bv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = c0 + e;
      switch (A.family) {
        case QD_FAM_FIRST_ORDER: out[e] = acc[0][e] + b0[c]; break;
        case QD_FAM_T3: out[e] = acc[0][e] * acc[0][e]; break;
        case QD_FAM_T4: av[e] = acc[0][e]; bv[e] = acc[1][e]; out[e] = av[e] * bv[e]; break;
        case QD_FAM_PROPOSED:
          av[e] = acc[0][e] + b0[c]; bv[e] = acc[1][e] + b1[c];
          out[e] = av[e] * bv[e] + (acc[2][e] + b2[c]);
          break;
        case QD_FAM_T2_LINEAR: out[e] = acc[0][e] + acc[1][e]; break;
        case QD_FAM_T2AND4: av[e] = acc[0][e]; bv[e] = acc[1][e]; out[e] = av[e] * bv[e] + acc[2][e]; break;
        default: out[e] = acc[0][e]; break;
      }
    }
    Vec8<T>::store(y + o, out);
    if (caches_ab(A.family)) {
      Vec8<T>::store(oa + o, av);
      Vec8<T>::store(ob + o, bv);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) dw_dgrad_vec_kernel(DwArgs A, const T* __restrict__ x,
                                                           const T* __restrict__ D, const float* __restrict__ Wp,
                                                           T* dx) {
  extern __shared__ float sW[];
  const DwFam fm = dw_fam(A.family);
  const int rr = A.r * A.r, CQ = A.C / 8;
  for (int i = threadIdx.x; i < fm.nroles * rr * A.C / 4; i += blockDim.x)
    reinterpret_cast<float4*>(sW)[i] = __ldg(reinterpret_cast<const float4*>(Wp) + i);
  __syncthreads();
  const bool anysq = fm.sq[0] || fm.sq[1] || fm.sq[2];
  const int total = (int)(A.Min * CQ);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i % CQ, c0 = q * 8;
    const int m = i / CQ;
    const int iw = m % A.W;
    const int t = m / A.W;
    const int ih = t % A.H, n = t / A.H;
    float lin[8], sq[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) lin[e] = sq[e] = 0.f;
    for (int dy = 0; dy < A.r; ++dy) {
      const int th = ih + A.p - dy;
      if (th < 0 || th % A.s) continue;
      const int oh = th / A.s;
      if (oh >= A.OH) continue;
      for (int dxx = 0; dxx < A.r; ++dxx) {
        const int tw = iw + A.p - dxx;
        if (tw < 0 || tw % A.s) continue;
        const int ow = tw / A.s;
        if (ow >= A.OW) continue;
        const size_t orow = (((size_t)n * A.OH + oh) * A.OW + ow) * A.Jd;
        const int tap = dy * A.r + dxx;
#pragma unroll
        for (int ro = 0; ro < 3; ++ro)
          if (ro < fm.nroles) {
            float d[8];
            Vec8<T>::load(D + orow + (size_t)fm.din[ro] * A.C + c0, d);
            const float4* wp = reinterpret_cast<const float4*>(sW + (ro * rr + tap) * A.C + c0);
            const float4 w0 = wp[0], w1 = wp[1];
            const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            if (fm.sq[ro]) {
#pragma unroll
              for (int e = 0; e < 8; ++e) sq[e] = fmaf(d[e], w[e], sq[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) lin[e] = fmaf(d[e], w[e], lin[e]);
            }
          }
      }
    }
    if (anysq) {
      float xv[8];
      Vec8<T>::load(x + (size_t)m * A.C + c0, xv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float tt = sq[e] * xv[e];
        lin[e] += tt + tt;
      }
    }
    Vec8<T>::store(dx + (size_t)m * A.C + c0, lin);
  }
}

// block (tap = blockIdx.x, pixel range = blockIdx.y); thread = (8-channel chunk, pixel lane);
// per-lane partials reduced across lanes in smem in a fixed order
template <typename T>
__global__ void __launch_bounds__(256) dw_wgrad_vec_kernel(DwArgs A, const T* __restrict__ x,
                                                           const T* __restrict__ D, float* part,
                                                           long long rows_per) {
  extern __shared__ float sred[];  // [lanes][nroles][C]
  const DwFam fm = dw_fam(A.family);
  const int rr = A.r * A.r, CQ = A.C / 8;
  const int tap = blockIdx.x, dy = tap / A.r, dxx = tap % A.r;
  const int q = threadIdx.x % CQ, lane = threadIdx.x / CQ, lanes = blockDim.x / CQ;
  const int c0 = q * 8;
  const long long m0 = (long long)blockIdx.y * rows_per;
  long long m1 = m0 + rows_per;
  if (m1 > A.Mout) m1 = A.Mout;
  float acc[3][8];
#pragma unroll
  for (int ro = 0; ro < 3; ++ro)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[ro][e] = 0.f;
  if (lane < lanes) {
    long long m = m0 + lane;
    int ow = (int)(m % A.OW);
    long long t = m / A.OW;
    int oh = (int)(t % A.OH), n = (int)(t / A.OH);
    for (; m < m1; m += lanes) {
      const int ih = oh * A.s + dy - A.p, iw = ow * A.s + dxx - A.p;
      if (ih >= 0 && ih < A.H && iw >= 0 && iw < A.W) {
        float v[8], v2[8];
        Vec8<T>::load(x + (((size_t)n * A.H + ih) * A.W + iw) * A.C + c0, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) v2[e] = v[e] * v[e];
#pragma unroll
        for (int ro = 0; ro < 3; ++ro)
          if (ro < fm.nroles) {
            float d[8];
            Vec8<T>::load(D + (size_t)m * A.Jd + (size_t)fm.din[ro] * A.C + c0, d);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[ro][e] = fmaf(d[e], fm.sq[ro] ? v2[e] : v[e], acc[ro][e]);
          }
      }
      ow += lanes;
      while (ow >= A.OW) {
        ow -= A.OW;
        if (++oh == A.OH) { oh = 0; ++n; }
      }
    }
  }
  // fixed-order reduction over the pixel lanes
  const int nr = fm.nroles;
  if (lane < lanes)
    for (int ro = 0; ro < nr; ++ro)
#pragma unroll
      for (int e = 0; e < 8; ++e) sred[((size_t)lane * nr + ro) * A.C + c0 + e] = acc[ro][e];
  __syncthreads();
  const int nrc_t = nr * A.C;  // outputs of this (tap, range)
  for (int o = threadIdx.x; o < nrc_t; o += blockDim.x) {
    float s = 0.f;
    for (int l = 0; l < lanes; ++l) s += sred[(size_t)l * nrc_t + o];
    const int ro = o / A.C, c = o - ro * A.C;
    // part[s][ro][tap][c] (same indexing as the scalar kernel: id = (ro*rr + tap)*C + c)
    part[(size_t)blockIdx.y * nr * rr * A.C + ((size_t)ro * rr + tap) * A.C + c] = s;
  }
}

__global__ void dw_wgrad_finish_kernel(int nrc, int S, const float* part, int rrC, float* w0, float* w1,
                                       float* w2, int rr, int C) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nrc) return;
  float acc = 0.f;
  int s = 0;
  for (; s + 8 <= S; s += 8) {  // eight rows in flight, added in row order
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = part[(size_t)(s + u) * nrc + id];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  for (; s < S; ++s) acc += part[(size_t)s * nrc + id];
  const int c = id % C, rt = id / C, tap = rt % rr, ro = rt / rr;
  float* dst = ro == 0 ? w0 : (ro == 1 ? w1 : w2);
  if (dst) dst[(size_t)c * rr + tap] = acc;  // reference layout (C, r, r)
  (void)rrC;
}

// packed depth-wise weights: fp32 [role][tap][C] (channel fastest: 8-channel vectors)
__global__ void dw_pack_kernel(int C, int rr, const float* w0, const float* w1, const float* w2, float* out,
                               int nroles) {
  const int n = nroles * C * rr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int ro = i / (C * rr), j = i - ro * C * rr, tap = j / C, c = j - tap * C;
    const float* w = ro == 0 ? w0 : (ro == 1 ? w1 : w2);
    out[i] = w[(size_t)c * rr + tap];  // reference (C, r, r)
  }
}

size_t dw_pack_bytes(const Plan& P) { return (size_t)dw_fam(P.family).nroles * P.C * P.r * P.r * 4; }

void dw_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st) {
  const int nr = dw_fam(P.family).nroles, rr = P.r * P.r;
  dw_pack_kernel<<<dw_grid((long long)nr * P.C * rr), 256, 0, st>>>(P.C, rr, w[0], nr > 1 ? w[1] : nullptr,
                                                                  nr > 2 ? w[2] : nullptr, (float*)wpack, nr);
  count_launch(st, "dw_pack");
}

static size_t dw_wsmem(const Plan& P) { return (size_t)dw_fam(P.family).nroles * P.r * P.r * P.C * 4; }
static bool dw_vec(const Plan& P) {
  return P.C % 8 == 0 && P.C <= 2048 && dw_wsmem(P) <= 200 * 1024 && P.Min * P.C < (1LL << 31) &&
         P.Mout * P.C < (1LL << 31);
}
template <typename K>
static void dw_smem_attr(K kernel, size_t smem) {
  raise_smem_attr((const void*)kernel, smem);
}

int dw_wgrad_split(const Plan& P) {
  if (dw_tile_ok(P)) return dw_tile_wgrad_split(P);
  if (dw_vec(P)) {  // grid (taps, ranges) ~ 4 blocks per SM
    const int rr = P.r * P.r;
    long long S = (4LL * 148 + rr - 1) / rr;
    long long cap = P.Mout / 16;
    if (cap < 1) cap = 1;
    if (S > cap) S = cap;
    return (int)(S < 1 ? 1 : S);
  }
  const long long nrc = (long long)dw_fam(P.family).nroles * P.r * P.r * P.C;
  long long S = (148LL * 2048 + nrc - 1) / nrc;
  long long cap = P.Mout / 32;
  if (cap < 1) cap = 1;
  if (S > cap) S = cap;
  if (S > 1024) S = 1024;
  return (int)(S < 1 ? 1 : S);
}

template <typename T>
static int dw_forward_t(const Plan& P, const T* x, const float* Wp, const float* const bias[3], T* y, T* a, T* b,
                        cudaStream_t st) {
  DwArgs A = dw_args(P);
  if (dw_tile_ok(P)) return dw_tile_forward<T>(P, A, x, Wp, bias, y, a, b, 0, st);
  if (dw_vec(P)) {
    dw_smem_attr(dw_fwd_vec_kernel<T>, dw_wsmem(P));
    dw_fwd_vec_kernel<T><<<dw_grid(P.Mout * (P.C / 8)), 256, dw_wsmem(P), st>>>(A, x, Wp, bias[0], bias[1], bias[2], y,
                                                                               a, b, 0);
  }
  else
    dw_fwd_kernel<T><<<dw_grid(P.Mout * P.C), 256, 0, st>>>(A, x, Wp, bias[0], bias[1], bias[2], y, a, b, 0);
  count_launch(st, "dw_fwd");
  return check_launch("dwconv forward");
}

int dw_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3], void* y, void* a,
               void* b, char* ws, const Workspace& L, cudaStream_t st) {
  (void)ws; (void)L;
  if (P.dtype == QD_BF16)
    return dw_forward_t<bf16>(P, (const bf16*)x, (const float*)wpack, bias, (bf16*)y, (bf16*)a, (bf16*)b, st);
  return dw_forward_t<float>(P, (const float*)x, (const float*)wpack, bias, (float*)y, (float*)a, (float*)b, st);
}

template <typename T>
static int dw_backward_t(const Plan& P, const T* x, const float* Wp, const T* a, const T* b, const T* dy, T* dx,
                         float* const dW[3], float* const db[3], char* ws, const Workspace& L, cudaStream_t st) {
  DwArgs A = dw_args(P);
  float* bpart = (float*)(ws + L.off_BS);
  const T* D = dy;
  if (P.family == QD_FAM_T3) {
    T* Dw = (T*)(ws + L.off_D);
    const float* nob[3] = {nullptr, nullptr, nullptr};
    if (dw_tile_ok(P)) {
      int rc = dw_tile_forward<T>(P, A, x, Wp, nob, Dw, nullptr, nullptr, 1, st);
      if (rc) return rc;
    } else if (dw_vec(P)) {
      dw_smem_attr(dw_fwd_vec_kernel<T>, dw_wsmem(P));
      dw_fwd_vec_kernel<T><<<dw_grid(P.Mout * (P.C / 8)), 256, dw_wsmem(P), st>>>(A, x, Wp, nob[0], nob[1], nob[2], Dw,
                                                                                 nullptr, nullptr, 1);
    }
    else
      dw_fwd_kernel<T><<<dw_grid(P.Mout * P.C), 256, 0, st>>>(A, x, Wp, nob[0], nob[1], nob[2], Dw, nullptr,
                                                              nullptr, 1);
    if (!dw_tile_ok(P)) count_launch(st, "dw_fwd_plain");
    launch_t3_prologue(P, dy, Dw, false, Dw, st);
    D = Dw;
  } else {
    if (caches_ab(P.family)) D = (const T*)(ws + L.off_D);
    if (P.dtype == QD_BF16 && P.F % 8 == 0 && 256 % (P.F / 8) == 0)
      launch_bwd_prologue_vec(P, dy, a, b, (void*)D, bpart, L.bs_split, st);
    else
      launch_bwd_prologue(P, dy, a, b, (void*)D, bpart, L.bs_split, st);
    if (db[0]) launch_bias_finish(P, bpart, L.bs_split, db, st);
  }
  if (dw_tile_ok(P)) {  // tiled wgrad + dgrad, then the fixed-order fold of the wgrad rows
    const DwFam fm = dw_fam(P.family);
    const int nrc = fm.nroles * P.r * P.r * P.C;
    float* part = dW[0] ? (float*)(ws + L.off_WG) : nullptr;
    int rc = dw_tile_backward<T>(P, A, x, D, Wp, dx, part, L.wg_split, st);
    if (rc) return rc;
    if (part) {
      dw_wgrad_finish_kernel<<<(nrc + 255) / 256, 256, 0, st>>>(nrc, L.wg_split, part, P.r * P.r * P.C, dW[0], dW[1],
                                                                dW[2], P.r * P.r, P.C);
      count_launch(st, "dw_wgrad_finish");
    }
    return check_launch("dwconv backward");
  }
  if (dW[0]) {
    const DwFam fm = dw_fam(P.family);
    const int nrc = fm.nroles * P.r * P.r * P.C;
    const int S = L.wg_split;
    float* part = (float*)(ws + L.off_WG);
    const long long rows_per = (P.Mout + S - 1) / S;
    if (dw_vec(P)) {
      const int CQ = P.C / 8, lanes = 256 / CQ;
      const size_t smem = (size_t)lanes * fm.nroles * P.C * 4;
      dw_wgrad_vec_kernel<T><<<dim3(P.r * P.r, S), lanes * CQ, smem, st>>>(A, x, D, part, rows_per);
    } else {
      dim3 grid((nrc + 255) / 256, S);
      dw_wgrad_kernel<T><<<grid, 256, 0, st>>>(A, x, D, part, rows_per);
    }
    count_launch(st, "dw_wgrad");
    dw_wgrad_finish_kernel<<<(nrc + 255) / 256, 256, 0, st>>>(nrc, S, part, P.r * P.r * P.C, dW[0], dW[1], dW[2],
                                                              P.r * P.r, P.C);
    count_launch(st, "dw_wgrad_finish");
  }
  if (dx) {
    if (dw_vec(P)) {
      dw_smem_attr(dw_dgrad_vec_kernel<T>, dw_wsmem(P));
      dw_dgrad_vec_kernel<T><<<dw_grid(P.Min * (P.C / 8)), 256, dw_wsmem(P), st>>>(A, x, D, Wp, dx);
    }
    else
      dw_dgrad_kernel<T><<<dw_grid(P.Min * P.C), 256, 0, st>>>(A, x, D, Wp, dx);
    count_launch(st, "dw_dgrad");
  }
  return check_launch("dwconv backward");
}

int dw_backward(const Plan& P, const void* x, const void* wpack, const void* a, const void* b, const void* dy,
                void* dx, float* const dW[3], float* const db[3], char* ws, const Workspace& L, cudaStream_t st) {
  if (P.dtype == QD_BF16)
    return dw_backward_t<bf16>(P, (const bf16*)x, (const float*)wpack, (const bf16*)a, (const bf16*)b,
                               (const bf16*)dy, (bf16*)dx, dW, db, ws, L, st);
  return dw_backward_t<float>(P, (const float*)x, (const float*)wpack, (const float*)a, (const float*)b,
                              (const float*)dy, (float*)dx, dW, db, ws, L, st);
}

}  // namespace qd
