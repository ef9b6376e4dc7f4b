// Max pooling (NHWC) for the QuadraNet training step around the quadratic
// layers: the ResNet stem pool (3x3/2, pad 1) and the VGG 2x2/2 pools.
//
// Forward: one thread per (output pixel, 8 channels) takes the window max in
// scan order (ky, kx) with torch.nn.MaxPool2d's rule (first maximum wins, NaN
// propagates) and records the winning window offset in one byte per channel.
// Backward is a gather, not a scatter: one thread per (input pixel, 8 channels)
// sums, in a fixed window order, the output gradients whose recorded offset
// points at it -- no atomics, deterministic, every store coalesced.
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "qd_kernels.h"

namespace qd {

template <typename T> struct PV;
template <> struct PV<bf16> {
  __device__ static void ld8(const bf16* p, float v[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
  }
  __device__ static void st8(bf16* p, const float v[8]) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      w[e] = *reinterpret_cast<const uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct PV<float> {
  __device__ static void ld8(const float* p, float v[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ static void st8(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

struct PoolGeo {
  int N, C, H, W, OH, OW, k, s, p;
};

// KW = window size at compile time (2, 3) so every window load of a thread is
// issued before any use (a runtime-bound loop waits on each load in turn); 0 = runtime
template <typename T, int KW>
__global__ void __launch_bounds__(256) maxpool_fwd_kernel(PoolGeo g, const T* __restrict__ x, T* __restrict__ y,
                                                          uint8_t* __restrict__ arg) {
  // 32-bit index math (the host checks the element count)
  const unsigned c8 = g.C / 8;
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (unsigned)g.N * g.OH * g.OW * c8) return;
  const unsigned cq = i % c8;
  unsigned t = i / c8;
  const int ow = (int)(t % (unsigned)g.OW);
  t /= (unsigned)g.OW;
  const int oh = (int)(t % (unsigned)g.OH);
  const int n = (int)(t / (unsigned)g.OH);
  const int k = KW ? KW : g.k;
  const int h0 = oh * g.s - g.p, w0 = ow * g.s - g.p;
  // torch's initial index: the window's first in-bounds position
  const uint8_t first = (uint8_t)((h0 < 0 ? -h0 : 0) * k + (w0 < 0 ? -w0 : 0));
  float best[8];
  uint8_t bi[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    best[e] = -__int_as_float(0x7f800000);  // -inf: padding never wins
    bi[e] = first;
  }
  const T* xn = x + ((size_t)n * g.H * g.W) * g.C + cq * 8;
  if (KW) {
    constexpr int KK = KW ? KW * KW : 1;
    float v[KK][8];
    bool ok[KK];
#pragma unroll
    for (int o = 0; o < KW * KW; ++o) {
      const int h = h0 + o / KW, w = w0 + o % KW;
      ok[o] = h >= 0 && h < g.H && w >= 0 && w < g.W;
      if (ok[o]) PV<T>::ld8(xn + ((size_t)h * g.W + w) * g.C, v[o]);
    }
#pragma unroll
    for (int o = 0; o < KW * KW; ++o) {
      if (!ok[o]) continue;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (v[o][e] > best[e] || v[o][e] != v[o][e]) {  // torch's rule: first maximum, a NaN always takes over
          best[e] = v[o][e];
          bi[e] = (uint8_t)o;
        }
    }
  } else {
    for (int ky = 0; ky < k; ++ky) {
      const int h = h0 + ky;
      if (h < 0 || h >= g.H) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int w = w0 + kx;
        if (w < 0 || w >= g.W) continue;
        float v[8];
        PV<T>::ld8(xn + ((size_t)h * g.W + w) * g.C, v);
        const uint8_t o = (uint8_t)(ky * k + kx);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (v[e] > best[e] || v[e] != v[e]) {
            best[e] = v[e];
            bi[e] = o;
          }
      }
    }
  }
  const size_t oidx = (size_t)i * 8;
  PV<T>::st8(y + oidx, best);
  uint2 packed;
  packed.x = bi[0] | (bi[1] << 8) | (bi[2] << 16) | ((uint32_t)bi[3] << 24);
  packed.y = bi[4] | (bi[5] << 8) | (bi[6] << 16) | ((uint32_t)bi[7] << 24);
  *reinterpret_cast<uint2*>(arg + oidx) = packed;
}

// backward gather; NW = max windows per axis covering one input position
// (ceil(k / s): 2 for 3x3/2 and 2x2/2) at compile time so all index and
// gradient loads of a thread are in flight together; 0 = runtime loop
template <typename T, int NW>
__global__ void __launch_bounds__(256) maxpool_bwd_kernel(PoolGeo g, const T* __restrict__ dy,
                                                          const uint8_t* __restrict__ arg, T* __restrict__ dx) {
  const unsigned c8 = g.C / 8;
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (unsigned)g.N * g.H * g.W * c8) return;
  const unsigned cq = i % c8;
  unsigned t = i / c8;
  const int w = (int)(t % (unsigned)g.W);
  t /= (unsigned)g.W;
  const int h = (int)(t % (unsigned)g.H);
  const int n = (int)(t / (unsigned)g.H);
  // windows (oh, ow) with oh*s - p <= h <= oh*s - p + k - 1
  int oh_lo = (h + g.p - g.k + g.s) / g.s, oh_hi = (h + g.p) / g.s;  // h + p - k + 1 >= 0 ? ceil : 0
  if (h + g.p - g.k + 1 < 0) oh_lo = 0;
  int ow_lo = (w + g.p - g.k + g.s) / g.s, ow_hi = (w + g.p) / g.s;
  if (w + g.p - g.k + 1 < 0) ow_lo = 0;
  if (oh_hi >= g.OH) oh_hi = g.OH - 1;
  if (ow_hi >= g.OW) ow_hi = g.OW - 1;
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  const size_t nbase = (size_t)n * g.OH * g.OW;
  if (NW) {
    constexpr int NN = NW ? NW * NW : 1;
    uint2 av[NN];
    float v[NN][8];
    bool ok[NN];
    uint8_t o[NN];
#pragma unroll
    for (int u = 0; u < NW * NW; ++u) {
      const int oh = oh_lo + u / NW, ow = ow_lo + u % NW;
      ok[u] = oh <= oh_hi && ow <= ow_hi;
      o[u] = (uint8_t)((h - (oh * g.s - g.p)) * g.k + (w - (ow * g.s - g.p)));
      const size_t oidx = ((nbase + (size_t)oh * g.OW + ow) * g.C) + cq * 8;
      if (ok[u]) {
        av[u] = __ldg(reinterpret_cast<const uint2*>(arg + oidx));
        PV<T>::ld8(dy + oidx, v[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < NW * NW; ++u) {
      if (!ok[u]) continue;
      const uint8_t* ab = reinterpret_cast<const uint8_t*>(&av[u]);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (ab[e] == o[u]) acc[e] += v[u][e];
    }
  } else {
    for (int oh = oh_lo; oh <= oh_hi; ++oh) {
      const int ky = h - (oh * g.s - g.p);
      for (int ow = ow_lo; ow <= ow_hi; ++ow) {
        const int kx = w - (ow * g.s - g.p);
        const uint8_t o = (uint8_t)(ky * g.k + kx);
        const size_t oidx = ((nbase + (size_t)oh * g.OW + ow) * g.C) + cq * 8;
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(arg + oidx));
        const uint8_t* ab = reinterpret_cast<const uint8_t*>(&a);
        float v[8];
        PV<T>::ld8(dy + oidx, v);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (ab[e] == o) acc[e] += v[e];
      }
    }
  }
  PV<T>::st8(dx + (size_t)i * 8, acc);
}

// k3 s2 p1 (the ResNet stem), even H and W: one thread per 2x2 input block x 8
// channels. The block's pixels are covered by windows (i, j), (i, j+1),
// (i+1, j), (i+1, j+1) only (i = h/2, j = w/2), so each window's argmax bytes
// and dy are loaded once for four pixels (the per-pixel gather loaded 9 window
// reads per 4 pixels and redid the index math for each); the per-pixel sums
// keep the window order of the general kernel (bit-identical results).
template <typename T>
__global__ void __launch_bounds__(256) maxpool_bwd_k3s2_kernel(PoolGeo g, const T* __restrict__ dy,
                                                               const uint8_t* __restrict__ arg, T* __restrict__ dx) {
  const unsigned c8 = g.C / 8, BW = g.W / 2, BH = g.H / 2;
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (unsigned)g.N * BH * BW * c8) return;
  const unsigned cq = i % c8;
  unsigned t = i / c8;
  const int bj = (int)(t % BW);
  t /= BW;
  const int bi = (int)(t % BH);
  const int n = (int)(t / BH);
  float acc[4][8];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[q][e] = 0.f;
  uint2 av[4];
  float v[4][8];
  bool ok[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {  // windows (bi + u/2, bj + u%2), all loads in flight
    const int oh = bi + u / 2, ow = bj + u % 2;
    ok[u] = oh < g.OH && ow < g.OW;
    const size_t oidx = (((size_t)n * g.OH + oh) * g.OW + ow) * g.C + cq * 8;
    if (ok[u]) {
      av[u] = __ldg(reinterpret_cast<const uint2*>(arg + oidx));
      PV<T>::ld8(dy + oidx, v[u]);
    }
  }
  // pixel (dh, dw) of the block sits at window offset ky * 3 + kx with
  // ky = dh + 1 (window row bi) or dh - 1 (row bi + 1, only dh = 1); kx alike
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (!ok[u]) continue;
    const uint8_t* ab = reinterpret_cast<const uint8_t*>(&av[u]);
    const int wy = u / 2, wx = u % 2;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int dh = q / 2, dw = q % 2;
      const int ky = wy == 0 ? dh + 1 : dh - 1, kx = wx == 0 ? dw + 1 : dw - 1;
      if (ky < 0 || kx < 0) continue;
      const uint8_t o = (uint8_t)(ky * 3 + kx);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (ab[e] == o) acc[q][e] += v[u][e];
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int h = 2 * bi + q / 2, w = 2 * bj + q % 2;
    PV<T>::st8(dx + ((((size_t)n * g.H + h) * g.W + w) * g.C) + cq * 8, acc[q]);
  }
}

static int pool_geo(int N, int C, int H, int W, int k, int s, int p, PoolGeo& g) {
  if (N < 1 || C < 8 || C % 8 || H < 1 || W < 1) return set_error(QD_ERR_DIM, "maxpool: N %d C %d H %d W %d", N, C, H, W);
  if (k < 1 || k > 15 || s < 1 || p < 0 || 2 * p > k) return set_error(QD_ERR_CONFIG, "maxpool: k %d s %d p %d", k, s, p);
  g.N = N; g.C = C; g.H = H; g.W = W; g.k = k; g.s = s; g.p = p;
  g.OH = (H + 2 * p - k) / s + 1;
  g.OW = (W + 2 * p - k) / s + 1;
  if (g.OH < 1 || g.OW < 1) return set_error(QD_ERR_DIM, "maxpool: empty output");
  return QD_OK;
}

int maxpool_forward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* x, void* y, void* arg,
                    cudaStream_t st) {
  PoolGeo g;
  int rc = pool_geo(N, C, H, W, k, s, p, g);
  if (rc) return rc;
  if (dev_skip("pool")) return QD_OK;
  const long long n = (long long)N * g.OH * g.OW * (C / 8);
  if (n >= (1LL << 31)) return set_error(QD_ERR_DIM, "maxpool: %lld channel groups (max 2^31)", n);
  const unsigned blocks = (unsigned)((n + 255) / 256);
#define QD_MPF(T, KW) maxpool_fwd_kernel<T, KW><<<blocks, 256, 0, st>>>(g, (const T*)x, (T*)y, (uint8_t*)arg)
  // the runtime-loop forward measured at least as fast as the unrolled one (64 regs)
  // on the ResNet stem pool; QD_MPF_UNROLL=1 selects the unrolled variant
  static const bool unr = getenv("QD_MPF_UNROLL") != nullptr;
  if (unr && k == 3) {
    if (dtype == QD_BF16) QD_MPF(bf16, 3); else QD_MPF(float, 3);
  } else if (unr && k == 2) {
    if (dtype == QD_BF16) QD_MPF(bf16, 2); else QD_MPF(float, 2);
  } else {
    if (dtype == QD_BF16) QD_MPF(bf16, 0); else QD_MPF(float, 0);
  }
#undef QD_MPF
  count_launch(st, "maxpool_fwd");
  return check_launch("maxpool forward");
}

int maxpool_backward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* dy, const void* arg,
                     void* dx, cudaStream_t st) {
  PoolGeo g;
  int rc = pool_geo(N, C, H, W, k, s, p, g);
  if (rc) return rc;
  if (dev_skip("pool")) return QD_OK;
  const long long n = (long long)N * H * W * (C / 8);
  if (n >= (1LL << 31)) return set_error(QD_ERR_DIM, "maxpool: %lld channel groups (max 2^31)", n);
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (k == 3 && s == 2 && p == 1 && H % 2 == 0 && W % 2 == 0 && g.OH == H / 2 && g.OW == W / 2) {
    const unsigned b4 = (unsigned)((n / 4 + 255) / 256);
    if (dtype == QD_BF16)
      maxpool_bwd_k3s2_kernel<bf16><<<b4, 256, 0, st>>>(g, (const bf16*)dy, (const uint8_t*)arg, (bf16*)dx);
    else
      maxpool_bwd_k3s2_kernel<float><<<b4, 256, 0, st>>>(g, (const float*)dy, (const uint8_t*)arg, (float*)dx);
    count_launch(st, "maxpool_bwd");
    return check_launch("maxpool backward");
  }
  // windows per axis covering an input position: ceil(k / s); 2 is the common case
  const int nw = (k + s - 1) / s;
#define QD_MPB(T, NW) maxpool_bwd_kernel<T, NW><<<blocks, 256, 0, st>>>(g, (const T*)dy, (const uint8_t*)arg, (T*)dx)
  if (dtype == QD_BF16) {
    if (nw == 2) QD_MPB(bf16, 2); else if (nw == 1) QD_MPB(bf16, 1); else QD_MPB(bf16, 0);
  } else {
    if (nw == 2) QD_MPB(float, 2); else if (nw == 1) QD_MPB(float, 1); else QD_MPB(float, 0);
  }
#undef QD_MPB
  count_launch(st, "maxpool_bwd");
  return check_launch("maxpool backward");
}

}  // namespace qd

namespace qd {

// im2col for small-channel convs run as one fc GEMM (the ResNet stem 7x7/2 over
// 3 channels, the VGG stem 3x3 over 3 channels): NHWC x -> col[M][Kp] in the
// run-padded layout k = ky runp + kx C + c (runp = r C rounded up to 8; zeros
// in the run tails and up to Kp, a multiple of 8).
// block = (n, oh, up to 112 output pixels of that row): the r input rows the
// block needs are staged in shared memory (row stride rounded to 8 elements,
// the zero padding materialised, coalesced NHWC loads). For a pixel, the kx, c
// columns of filter row ky are ONE contiguous run of the staged row ky, so a
// thread copies a whole run (pixel, ky) as 32-bit words (funnel-shifted when
// the run starts at an odd element) into runp / 8 16-byte stores (measured:
// 0.30 ms on the ResNet stem vs 0.34 with one 16-byte chunk per thread).
constexpr int IM2COL_TW = 112;  // a whole ResNet stem output row per block (32: 4x the blocks, latency-bound)
template <typename T, int CT, int RT>  // CT / RT: C and r at compile time (0: runtime)
__global__ void __launch_bounds__(256) im2col_kernel(int N, int C_, int H, int W, int OH, int OW, int r_, int s,
                                                     int p, int Kp, const T* __restrict__ x, T* __restrict__ col) {
  // the kernel is instruction-bound (ncu: issue slots 80% busy): index math by
  // compile-time C and r (the stems: C = 3, r = 7 / 3) and per-row staging loops
  const int C = CT ? CT : C_, r = RT ? RT : r_;
  extern __shared__ __align__(16) unsigned char im2col_smem[];
  T* rows = reinterpret_cast<T*>(im2col_smem);  // [r][RCp]
  const int owt = (OW + IM2COL_TW - 1) / IM2COL_TW;
  int b = blockIdx.x;
  const int ot = b % owt;
  b /= owt;
  const int oh = b % OH, n = b / OH;
  const int ow0 = ot * IM2COL_TW, tw = min(IM2COL_TW, OW - ow0);
  const int RW = (IM2COL_TW - 1) * s + r, RC = RW * C, RCp = (RC + 7) & ~7;
  const int h0 = oh * s - p, w0 = ow0 * s - p;
  // staging, one input row at a time: 4 elements per thread per pass, all 4
  // loads issued before the shared stores; valid w is a contiguous q range
  const int qlo = (w0 < 0 ? -w0 : 0) * C, qhi = min(RC, (W - w0) * C);
  for (int j = 0; j < r; ++j) {
    const int h = h0 + j;
    const bool hok = h >= 0 && h < H;
    const T* src = x + (((size_t)n * H + (hok ? h : 0)) * W) * C + (long long)w0 * C;
    T* dst = rows + j * RCp;
    for (int q0 = threadIdx.x; q0 < RCp; q0 += 4 * blockDim.x) {
      T v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * blockDim.x;
        v[u] = (hok && q >= qlo && q < qhi) ? src[q] : cvt<T>(0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * blockDim.x;
        if (q < RCp) dst[q] = v[u];
      }
    }
  }
  __syncthreads();
  const int rc = r * C, runp = (rc + 7) & ~7;
  T* dst0 = col + ((size_t)(n * OH + oh) * OW + ow0) * Kp;
  for (int id = threadIdx.x; id < tw * r; id += blockDim.x) {
    const int l = id / r, ky = id - l * r;
    const int off = ky * RCp + l * s * C;  // first element of the run
    T* dst = dst0 + (size_t)l * Kp + ky * runp;
    if (sizeof(T) == 2) {
      const uint32_t* ws = reinterpret_cast<const uint32_t*>(rows) + (off >> 1);
      const uint32_t sh = (off & 1) * 16;
      uint32_t prev = ws[0];
      for (int c8 = 0; c8 < runp / 8; ++c8) {
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t nxt = ws[c8 * 4 + e + 1];
          uint32_t v = __funnelshift_r(prev, nxt, sh);
          prev = nxt;
          const int kk = c8 * 8 + 2 * e;  // run elements kk, kk + 1
          if (kk >= rc) v = 0u;
          else if (kk + 1 >= rc) v &= 0xFFFFu;
          o[e] = v;
        }
        *reinterpret_cast<uint4*>(dst + c8 * 8) = make_uint4(o[0], o[1], o[2], o[3]);
      }
    } else {
      for (int k = 0; k < runp; ++k) dst[k] = k < rc ? rows[off + k] : cvt<T>(0.f);
    }
    if (ky == r - 1)  // K padding after the last run
      for (int k = r * runp; k < Kp; k += 8) {
        if (sizeof(T) == 2) {
          *reinterpret_cast<uint4*>(dst0 + (size_t)l * Kp + k) = make_uint4(0u, 0u, 0u, 0u);
        } else {
          for (int e = 0; e < 8; ++e) dst0[(size_t)l * Kp + k + e] = cvt<T>(0.f);
        }
      }
  }
}

int im2col(int N, int C, int H, int W, int r, int s, int p, int Kp, int dtype, const void* x, void* col,
           cudaStream_t st) {
  if (N < 1 || C < 1 || H < 1 || W < 1 || r < 1 || s < 1 || p < 0)
    return set_error(QD_ERR_DIM, "im2col: N %d C %d H %d W %d r %d s %d p %d", N, C, H, W, r, s, p);
  const int runp = (r * C + 7) & ~7;
  if (Kp % 8 || Kp < r * runp)
    return set_error(QD_ERR_CONFIG, "im2col: Kp %d (need a multiple of 8 >= %d)", Kp, r * runp);
  const int OH = (H + 2 * p - r) / s + 1, OW = (W + 2 * p - r) / s + 1;
  if (OH < 1 || OW < 1) return set_error(QD_ERR_DIM, "im2col: empty output");
  if (dev_skip("im2col")) return QD_OK;
  const long long blocks = (long long)N * OH * ((OW + IM2COL_TW - 1) / IM2COL_TW);
  if (blocks >= (1LL << 31)) return set_error(QD_ERR_DIM, "im2col: %lld blocks", blocks);
  const size_t es = dtype == QD_BF16 ? 2 : 4;
  // staged rows + slack for the word past the last run
  const size_t smem = (size_t)r * ((((IM2COL_TW - 1) * s + r) * C + 7) & ~7) * es + (size_t)(runp + 8) * es;
  if (smem > 48 * 1024) return set_error(QD_ERR_UNSUPPORTED, "im2col: %zu B of staged rows (r %d, s %d, C %d)", smem, r, s, C);
  if (dtype == QD_BF16) {
    if (C == 3 && r == 7)
      im2col_kernel<bf16, 3, 7><<<(unsigned)blocks, 256, smem, st>>>(N, C, H, W, OH, OW, r, s, p, Kp, (const bf16*)x,
                                                                     (bf16*)col);
    else if (C == 3 && r == 3)
      im2col_kernel<bf16, 3, 3><<<(unsigned)blocks, 256, smem, st>>>(N, C, H, W, OH, OW, r, s, p, Kp, (const bf16*)x,
                                                                     (bf16*)col);
    else
      im2col_kernel<bf16, 0, 0><<<(unsigned)blocks, 256, smem, st>>>(N, C, H, W, OH, OW, r, s, p, Kp, (const bf16*)x,
                                                                     (bf16*)col);
  } else {
    im2col_kernel<float, 0, 0><<<(unsigned)blocks, 256, smem, st>>>(N, C, H, W, OH, OW, r, s, p, Kp,
                                                                    (const float*)x, (float*)col);
  }
  count_launch(st, "im2col");
  return check_launch("im2col");
}

}  // namespace qd
