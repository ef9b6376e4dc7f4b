// fp32 layers on the bf16 tensor cores (device path 3, "x3").
//
// Every fp32 GEMM operand v is split into two bf16 terms, hi = bf16(v) and
// lo = bf16(v - hi) (|v - hi - lo| <= 2^-17 |v|: 16 significant bits), and each
// product is formed as hi*hi + hi*lo + lo*hi with fp32 accumulation in TMEM
// (the dropped lo*lo term is below 2^-16 of the product). On the existing
// tcgen05 kernels that is ONE GEMM with K tripled: A = [hi | hi | lo] through
// two TMA maps (segment 2 from the second map), B = [W_hi | W_lo | W_hi]
// packed once. The layer's error is ~1e-5 relative -- inside the north star's
// 1e-4 fp32 bound (plain TF32, one 11-bit product, is not: SURVEY.md §0.4) --
// at the bf16 MMA rate (twice the TF32 rate, so 3 bf16 products cost what 1.5
// TF32 products would).
//
// This file: the operand split, the x3 weight pack, the fp32 backward prologue
// (D = [g b | g a | g] split into hi / lo, bias partial sums from fp32 values)
// and the fp32 epilogue passes over the raw accumulators.
#include <stdio.h>
#include "qd_kernels.h"
#include "qd_ptx.cuh"

namespace qd {

__device__ __forceinline__ void x3_split1(float v, bf16& hi, bf16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

__device__ __forceinline__ void x3_split8(const float* v, uint4& hi, uint4& lo) {
  bf16 h[8], l[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) x3_split1(v[e], h[e], l[e]);
  hi = *reinterpret_cast<const uint4*>(h);
  lo = *reinterpret_cast<const uint4*>(l);
}

// n elements (n % 8 == 0): hi / lo halves, 8 per thread-iteration (2 x float4 in, 2 x uint4 out)
__global__ void __launch_bounds__(256) x3_split_kernel(const float* __restrict__ x, bf16* __restrict__ hi,
                                                       bf16* __restrict__ lo, long long n8) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n8; i += (long long)gridDim.x * blockDim.x) {
    const float4* src = reinterpret_cast<const float4*>(x) + 2 * i;
    float4 p = __ldg(src), q = __ldg(src + 1);
    const float v[8] = {p.x, p.y, p.z, p.w, q.x, q.y, q.z, q.w};
    uint4 h, l;
    x3_split8(v, h, l);
    reinterpret_cast<uint4*>(hi)[i] = h;
    reinterpret_cast<uint4*>(lo)[i] = l;
  }
}

void launch_x3_split(const float* x, bf16* hi, bf16* lo, long long n, cudaStream_t st) {
  const long long n8 = n / 8;
  long long g = (n8 + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  if (g < 1) g = 1;
  launch_pdl(x3_split_kernel, dim3((unsigned)g), dim3(256), 0, st, x, hi, lo, n8);
  count_launch(st, "x3_split");
}

// packed weights, x3 layout: fprop rows [nb F][3 Kf] = [hi | lo | hi] of the bf16
// fprop layout (fprop_src / fprop_row), then dgrad rows [Cd][3 Kd] likewise.
// Elements [i0, nf + nd) of that (fprop, dgrad) sequence.
__global__ void x3_pack_kernel(Plan P, const float* w0, const float* w1, const float* w2, bf16* out, long long i0) {
  const long long nf = (long long)P.nb * P.F * P.Kf, nd = (long long)P.Cd * P.Kd;
  for (long long i = i0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf + nd;
       i += (long long)gridDim.x * blockDim.x) {
    float v;
    bf16* base;
    int k, K;
    if (i < nf) {
      const int R = (int)(i / P.Kf);
      k = (int)(i % P.Kf);
      K = P.Kf;
      const int grp = P.nb * P.FT;
      const int tile = R / grp, rem = R % grp;
      const int br = rem / P.FT, f = tile * P.FT + rem % P.FT;
      int role, kk;
      const bool nz = fprop_src(P, br, k, role, kk);
      const int tap = kk / P.C, c = kk % P.C, dy = tap / P.r, dx = tap % P.r;
      const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
      v = !nz ? 0.f
              : (P.kind == QD_KIND_FC) ? w[(size_t)c * P.F + f] : w[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx];
      base = out + (size_t)R * 3 * P.Kf;
    } else {
      const long long i2 = i - nf;
      const int cp = (int)(i2 / P.Kd);
      k = (int)(i2 % P.Kd);
      K = P.Kd;
      const int e = k / P.Jd, j = k % P.Jd;
      const int ey = e / P.r, ex = e % P.r, dy = P.r - 1 - ey, dx = P.r - 1 - ex;
      int role, f, c;
      const bool nz = dgrad_src(P, cp, j, role, c, f);
      const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
      v = !nz ? 0.f
              : (P.kind == QD_KIND_FC) ? w[(size_t)c * P.F + f] : w[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx];
      base = out + 3 * nf + (size_t)cp * 3 * P.Kd;
    }
    bf16 hi, lo;
    x3_split1(v, hi, lo);
    base[k] = hi;
    base[K + k] = lo;
    base[2 * K + k] = hi;
  }
}

// fc fprop part of the x3 pack as 32 x 32 transposes: the fc weights are (in, out)
// = w[c F + f] while a packed fprop row runs over c (fprop_row for the f index);
// reads coalesced along f, writes along c. grid (F / 32, C / 32, roles).
__global__ void __launch_bounds__(256) x3_pack_fc_kernel(Plan P, const float* w0, const float* w1, const float* w2,
                                                         bf16* out) {
  __shared__ float t[32][33];
  const int role = blockIdx.z, f0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + ty + 8 * i, f = f0 + tx;
    t[ty + 8 * i][tx] = (c < P.C && f < P.F) ? __ldg(w + (size_t)c * P.F + f) : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int f = f0 + ty + 8 * i, c = c0 + tx;
    if (f >= P.F || c >= P.C) continue;
    const int R = fprop_row(role, f, P.nb, P.FT);
    bf16 hi, lo;
    x3_split1(t[tx][ty + 8 * i], hi, lo);
    bf16* row = out + (size_t)R * 3 * P.Kf;
    row[c] = hi;
    row[P.Kf + c] = lo;
    row[2 * P.Kf + c] = hi;
  }
}

// fc dgrad rows [hi | lo | hi] of the split pack: row cp = input channel, column j =
// D channel (one tap); block (x, cp) covers 256 consecutive j -- the fc weights
// are read along f (coalesced) and no per-element 64-bit index division remains
__global__ void __launch_bounds__(256) x3_pack_fc_dgrad_kernel(Plan P, const float* w0, const float* w1,
                                                               const float* w2, bf16* out) {
  const int cp = blockIdx.y, j = blockIdx.x * 256 + threadIdx.x;
  if (j >= P.Kd) return;
  int role, c, f;
  const bool nz = dgrad_src(P, cp, j, role, c, f);
  const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
  const float v = nz ? __ldg(w + (size_t)c * P.F + f) : 0.f;
  bf16 hi, lo;
  x3_split1(v, hi, lo);
  bf16* row = out + 3 * (size_t)P.nb * P.F * P.Kf + (size_t)cp * 3 * P.Kd;
  row[j] = hi;
  row[P.Kd + j] = lo;
  row[2 * P.Kd + j] = hi;
}

void launch_x3_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st) {
  const long long nf = (long long)P.nb * P.F * P.Kf;
  long long i0 = 0;
  if (P.kind == QD_KIND_FC && P.sq == 0) {
    x3_pack_fc_kernel<<<dim3((P.F + 31) / 32, (P.C + 31) / 32, P.nroles), 256, 0, st>>>(P, w[0], w[1], w[2],
                                                                                         (bf16*)wpack);
    x3_pack_fc_dgrad_kernel<<<dim3((P.Kd + 255) / 256, P.Cd), 256, 0, st>>>(P, w[0], w[1], w[2], (bf16*)wpack);
    count_launch(st, "x3_pack");
    return;
  }
  const long long n = nf + (long long)P.Cd * P.Kd - i0;
  long long g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  x3_pack_kernel<<<(unsigned)g, 256, 0, st>>>(P, w[0], w[1], w[2], (bf16*)wpack, i0);
  count_launch(st, "x3_pack");
}

// backward prologue in fp32: D = [g b | g a | g] (proposed), [g b | g a] (t4) or
// g (first order), each block written as hi / lo bf16 rows [M][Jd]; bias partial
// sums (fixed order: per thread, then per block over its row lanes) of the fp32
// products: block 0 = sum g b, 1 = sum g a, 2 = sum g (proposed), or sum g
// (first order). One thread = 8 channels of one row.
__global__ void __launch_bounds__(256) x3_prologue_kernel(Plan P, const float* __restrict__ dy,
                                                          const float* __restrict__ a, const float* __restrict__ b,
                                                          bf16* __restrict__ Dh, bf16* __restrict__ Dl,
                                                          float* __restrict__ part, long long rows_per) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  const int F = P.F, chunks = F / 8;
  const int lanes = 256 / chunks;
  const int ch = threadIdx.x % chunks, rl = threadIdx.x / chunks;
  const bool mat = caches_ab(P.family);
  const int nblk = P.Jd / F;
  long long r0 = (long long)blockIdx.x * rows_per, r1 = r0 + rows_per;
  if (r1 > P.Mout) r1 = P.Mout;
  float s[3][8];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int e = 0; e < 8; ++e) s[q][e] = 0.f;
  auto ld8 = [](const float* p, float v[8]) {
    const float4 u = __ldg(reinterpret_cast<const float4*>(p)), w = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
  };
  auto emit = [&](long long m, const float* g, const float* av, const float* bv) {
    bf16* hrow = Dh + (size_t)m * P.Jd + ch * 8;
    bf16* lrow = Dl + (size_t)m * P.Jd + ch * 8;
    uint4 h, l;
    if (mat) {
      float gb[8], ga[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        gb[e] = g[e] * bv[e];
        ga[e] = g[e] * av[e];
        s[0][e] += gb[e];
        s[1][e] += ga[e];
        s[2][e] += g[e];
      }
      x3_split8(gb, h, l);
      *reinterpret_cast<uint4*>(hrow) = h;
      *reinterpret_cast<uint4*>(lrow) = l;
      x3_split8(ga, h, l);
      *reinterpret_cast<uint4*>(hrow + F) = h;
      *reinterpret_cast<uint4*>(lrow + F) = l;
      if (nblk == 3) {
        x3_split8(g, h, l);
        *reinterpret_cast<uint4*>(hrow + 2 * F) = h;
        *reinterpret_cast<uint4*>(lrow + 2 * F) = l;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) s[0][e] += g[e];
      x3_split8(g, h, l);
      *reinterpret_cast<uint4*>(hrow) = h;
      *reinterpret_cast<uint4*>(lrow) = l;
    }
  };
  if (rl < lanes) {
    // two rows per iteration: all twelve 16-B loads in flight before any use
    long long m = r0 + rl;
    for (; m + lanes < r1; m += 2 * lanes) {
      float g0[8], a0[8], b0[8], g1[8], a1[8], b1[8];
      const size_t o0 = (size_t)m * F + ch * 8, o1 = (size_t)(m + lanes) * F + ch * 8;
      ld8(dy + o0, g0);
      ld8(dy + o1, g1);
      if (mat) {
        ld8(a + o0, a0); ld8(b + o0, b0);
        ld8(a + o1, a1); ld8(b + o1, b1);
      }
      emit(m, g0, a0, b0);
      emit(m + lanes, g1, a1, b1);
    }
    if (m < r1) {
      float g0[8], a0[8], b0[8];
      const size_t o0 = (size_t)m * F + ch * 8;
      ld8(dy + o0, g0);
      if (mat) {
        ld8(a + o0, a0);
        ld8(b + o0, b0);
      }
      emit(m, g0, a0, b0);
    }
  }
  if (!part) return;
  __shared__ float red[256][9];
  const int nsum = mat ? nblk : 1;
  for (int q = 0; q < nsum; ++q) {
#pragma unroll
    for (int e = 0; e < 8; ++e) red[threadIdx.x][e] = q == 0 ? s[0][e] : (q == 1 ? s[1][e] : s[2][e]);
    __syncthreads();
    for (int tcol = threadIdx.x; tcol < chunks * 8; tcol += 256) {
      const int c = tcol / 8, e = tcol % 8;
      float acc = 0.f;
      for (int l2 = 0; l2 < lanes; ++l2) acc += red[l2 * chunks + c][e];
      part[(size_t)blockIdx.x * P.Jd + q * F + c * 8 + e] = acc;
    }
    __syncthreads();
  }
}

void launch_x3_prologue(const Plan& P, const float* dy, const float* a, const float* b, bf16* Dh, bf16* Dl,
                        float* part, int split, cudaStream_t st) {
  const long long rows_per = (P.Mout + split - 1) / split;
  launch_pdl(x3_prologue_kernel, dim3(split), dim3(256), 0, st, P, dy, a, b, Dh, Dl, part, rows_per);
  count_launch(st, "x3_prologue");
}

// fprop epilogue over the raw accumulators [S][M][ld] (column of branch br, channel
// f: (f / 64) nb 64 + br 64 + f % 64; plain: f): slices summed in order, then
// a = ra + ba, b = rb + bb, y = a b + rc + bc (proposed) / y = a b (t4) /
// y = r + bias (plain); fp32 outputs. One thread = 4 channels of one pixel.
__global__ void __launch_bounds__(256) x3_fprop_finish_kernel(const float* __restrict__ raw, int S, long long M,
                                                              int ld, int F, int nb, int epi, float* __restrict__ y,
                                                              float* __restrict__ ao, float* __restrict__ bo,
                                                              const float* __restrict__ b0,
                                                              const float* __restrict__ b1,
                                                              const float* __restrict__ b2) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  const int f4 = F / 4;
  const long long n = M * f4;
  const long long slice = M * (long long)ld;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / f4;
    const int f = (int)(i - m * f4) * 4;
    const float* rp = raw + m * ld;
    float4 acc[3];
    const int nbr = epi == 2 ? 1 : nb;
    for (int br = 0; br < nbr; ++br) {
      const int col = epi == 2 ? f : (f / 64) * nb * 64 + br * 64 + (f % 64);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < S; ++s) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(rp + s * slice + col));
        v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
      }
      acc[br] = v;
    }
    float4 out;
    if (epi == 0) {  // proposed
      const float4 ba = *reinterpret_cast<const float4*>(b0 + f), bb = *reinterpret_cast<const float4*>(b1 + f),
                   bc = *reinterpret_cast<const float4*>(b2 + f);
      float4 a = make_float4(acc[0].x + ba.x, acc[0].y + ba.y, acc[0].z + ba.z, acc[0].w + ba.w);
      float4 b = make_float4(acc[1].x + bb.x, acc[1].y + bb.y, acc[1].z + bb.z, acc[1].w + bb.w);
      out = make_float4(fmaf(a.x, b.x, acc[2].x + bc.x), fmaf(a.y, b.y, acc[2].y + bc.y),
                        fmaf(a.z, b.z, acc[2].z + bc.z), fmaf(a.w, b.w, acc[2].w + bc.w));
      *reinterpret_cast<float4*>(ao + m * F + f) = a;
      *reinterpret_cast<float4*>(bo + m * F + f) = b;
    } else if (epi == 1) {  // t4
      const float4 a = acc[0], b = acc[1];
      out = make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
      *reinterpret_cast<float4*>(ao + m * F + f) = a;
      *reinterpret_cast<float4*>(bo + m * F + f) = b;
    } else {
      out = acc[0];
      if (b0) {
        const float4 bz = *reinterpret_cast<const float4*>(b0 + f);
        out.x += bz.x; out.y += bz.y; out.z += bz.z; out.w += bz.w;
      }
    }
    *reinterpret_cast<float4*>(y + m * F + f) = out;
  }
}

void launch_x3_fprop_finish(const float* raw, int S, long long M, int ld, int F, int nb, int epi, float* y,
                            float* a, float* b, const float* const bias[3], cudaStream_t st) {
  const long long n = M * (F / 4);
  long long g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  launch_pdl(x3_fprop_finish_kernel, dim3((unsigned)g), dim3(256), 0, st, (const float*)raw, S, M, ld, F, nb, epi, y,
             a, b, bias[0], bias[1], bias[2]);
  count_launch(st, "x3_finish");
}

// sum of S raw slices [S][n] into out[n] (dgrad with a split K)
__global__ void __launch_bounds__(256) x3_sum_kernel(const float* __restrict__ raw, int S, long long n4,
                                                     float* __restrict__ out) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < S; ++s) {
      const float4 u = __ldg(reinterpret_cast<const float4*>(raw) + s * n4 + i);
      v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
    }
    reinterpret_cast<float4*>(out)[i] = v;
  }
}

void launch_x3_sum(const float* raw, int S, long long n, float* out, cudaStream_t st) {
  const long long n4 = n / 4;
  long long g = (n4 + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  launch_pdl(x3_sum_kernel, dim3((unsigned)g), dim3(256), 0, st, raw, S, n4, out);
  count_launch(st, "x3_sum");
}

}  // namespace qd
