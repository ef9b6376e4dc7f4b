// Generic CUDA-core kernels: weight packing, the elementwise/reduction pieces
// of the backward pass (shared with the tcgen05 path), and a fully general
// implicit-GEMM fallback that covers every geometry (any stride/pad/kernel,
// any channel count, fp32 and bf16). The fallback is the fp32 path (exact
// FFMA accumulation) and the path for shapes the tcgen05 kernels do not
// tile; it is never a CPU path.
//
// Math follows the reference closed forms (neurons.py:235-276 forward,
// neurons.py:295-445 backward) with the conv lowered as an implicit GEMM
// instead of materialising the patch matrix (tensor.py:283-331).
#include <stdio.h>
#include <stdlib.h>
#include "qd_kernels.h"
#include "qd_gemm.cuh"
#include "qd_ptx.cuh"

namespace qd {

// ---------------------------------------------------------------------------
// packing
// ---------------------------------------------------------------------------
size_t pack_fprop_elems(const Plan& P) { return (size_t)P.nb * P.F * P.Kf; }
size_t pack_dgrad_elems(const Plan& P) { return (size_t)P.Cd * P.Kd; }

static inline int grid_for(long long n, int bs = 256, int cap = 148 * 16) {
  long long g = (n + bs - 1) / bs;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

template <typename T>
__global__ void pack_one_kernel(Plan P, const float* w0, const float* w1, const float* w2, T* out) {
  long long nf = (long long)P.nb * P.F * P.Kf;
  int nfb = (int)((nf + 255) / 256);
  if ((int)blockIdx.x < nfb) {
    long long i = (long long)blockIdx.x * 256 + threadIdx.x;
    if (i >= nf) return;
    int R = (int)(i / P.Kf), k = (int)(i % P.Kf);
    int grp = P.nb * P.FT;
    int tile = R / grp, rem = R % grp;
    int br = rem / P.FT, f = tile * P.FT + rem % P.FT;
    int role, kk;
    const bool nz = fprop_src(P, br, k, role, kk);
    int tap = kk / P.C, c = kk % P.C, dy = tap / P.r, dx = tap % P.r;
    const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
    float v = !nz ? 0.f
                  : (P.kind == QD_KIND_FC) ? w[(size_t)c * P.F + f]
                                           : w[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx];
    out[i] = cvt<T>(v);
  } else {
    long long i = (long long)(blockIdx.x - nfb) * 256 + threadIdx.x;
    if (i >= (long long)P.Cd * P.Kd) return;
    int cp = (int)(i / P.Kd), k = (int)(i % P.Kd);
    int e = k / P.Jd, j = k % P.Jd;
    int ey = e / P.r, ex = e % P.r, dy = P.r - 1 - ey, dx = P.r - 1 - ex;
    int role, f, c;
    const bool nz = dgrad_src(P, cp, j, role, c, f);
    const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
    float v = !nz ? 0.f
                  : (P.kind == QD_KIND_FC) ? w[(size_t)c * P.F + f]
                                           : w[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx];
    out[nf + i] = cvt<T>(v);
  }
}

template <typename T>
__global__ void pack_all_kernel(Plan P, const float* w0, const float* w1, const float* w2, T* out) {
  // blocks [0, nfb) pack the fprop layout, the rest the dgrad layout; 4 consecutive
  // k (same row, so the row decode is shared) per thread
  const long long nf = (long long)P.nb * P.F * P.Kf;
  const int nfb = (int)((nf / 4 + 255) / 256);
  if ((int)blockIdx.x < nfb) {
    long long i0 = ((long long)blockIdx.x * 256 + threadIdx.x) * 4;
    if (i0 >= nf) return;
    int R = (int)(i0 / P.Kf), k0 = (int)(i0 % P.Kf);
    int grp = P.nb * P.FT;
    int tile = R / grp, rem = R % grp;
    int br = rem / P.FT, f = tile * P.FT + rem % P.FT;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int k = k0 + e, role, kk;
      const bool nz = fprop_src(P, br, k, role, kk);
      int tap = kk / P.C, c = kk % P.C, dy = tap / P.r, dx = tap % P.r;
      const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
      float v = !nz ? 0.f
                    : (P.kind == QD_KIND_FC) ? w[(size_t)c * P.F + f]
                                             : w[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx];
      out[i0 + e] = cvt<T>(v);
    }
  } else {
    long long i0 = ((long long)(blockIdx.x - nfb) * 256 + threadIdx.x) * 4;
    if (i0 >= (long long)P.Cd * P.Kd) return;
    int cp = (int)(i0 / P.Kd), k0 = (int)(i0 % P.Kd);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int k = k0 + e;
      int ee = k / P.Jd, j = k % P.Jd;
      int ey = ee / P.r, ex = ee % P.r, dy = P.r - 1 - ey, dx = P.r - 1 - ex;
      int role, f, c;
      const bool nz = dgrad_src(P, cp, j, role, c, f);
      const float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
      float v = !nz ? 0.f
                    : (P.kind == QD_KIND_FC) ? w[(size_t)c * P.F + f]
                                             : w[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx];
      out[nf + i0 + e] = cvt<T>(v);
    }
  }
}

// conv, no squared operand: one block per packed row, the row's source block staged in
// smem so both the reads of w and the writes of the packed row are contiguous.
//   fprop row (role br, filter f):  k = tap*C + c   <- w_br[f][c][tap]
//   dgrad row c:                    k = e*Jd + j    <- w_{j/F}[j%F][c][r*r-1-e]
template <typename T>
__global__ void __launch_bounds__(256) pack_conv_kernel(Plan P, const float* w0, const float* w1, const float* w2,
                                                        T* out) {
  extern __shared__ float sbuf[];
  ptx::pdl_launch();  // the forward kernel may start its setup while we pack
  const int rr = P.r * P.r;
  const int nrow = P.nb * P.F;
  if ((int)blockIdx.x < nrow) {
    const int br = blockIdx.x / P.F, f = blockIdx.x - br * P.F;
    const float* w = (br == 0 ? w0 : (br == 1 ? w1 : w2)) + (size_t)f * P.C * rr;
    const int nsrc = P.C * rr;
    for (int i0 = threadIdx.x; i0 < nsrc; i0 += 8 * blockDim.x) {  // 8 loads in flight per thread
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        v[u] = i < nsrc ? __ldg(w + i) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < nsrc) sbuf[i] = v[u];
      }
    }
    __syncthreads();
    const int R = (f / P.FT) * (P.nb * P.FT) + br * P.FT + f % P.FT;
    T* o = out + (size_t)R * P.Kf;
    for (int k = threadIdx.x; k < P.Kf; k += blockDim.x) {
      const int tap = k / P.C, c = k - tap * P.C;
      o[k] = cvt<T>(sbuf[c * rr + tap]);
    }
  } else {
    const int c = blockIdx.x - nrow;
    const int nsrc = P.Jd * rr;
    for (int i0 = threadIdx.x; i0 < nsrc; i0 += 8 * blockDim.x) {  // 8 loads in flight per thread
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        v[u] = 0.f;
        if (i < nsrc) {
          const int j = i / rr, t = i - j * rr;
          const int br = j / P.F, f = j - br * P.F;
          const float* w = br == 0 ? w0 : (br == 1 ? w1 : w2);
          v[u] = __ldg(w + ((size_t)f * P.C + c) * rr + t);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * blockDim.x;
        if (i < nsrc) sbuf[i] = v[u];
      }
    }
    __syncthreads();
    T* o = out + (size_t)nrow * P.Kf + (size_t)c * P.Kd;
    for (int k = threadIdx.x; k < P.Kd; k += blockDim.x) {
      const int e = k / P.Jd, j = k - e * P.Jd;
      o[k] = cvt<T>(sbuf[j * rr + (rr - 1 - e)]);
    }
  }
}

template <typename T>
static void launch_pack_conv(const Plan& P, const float* const w[3], T* out, size_t smem, cudaStream_t st) {
  raise_smem_attr((const void*)pack_conv_kernel<T>, smem);
  pack_conv_kernel<T><<<P.nb * P.F + P.C, 256, smem, st>>>(P, w[0], w[1], w[2], out);
}

// threads per tile block: 16 warps share a 32 x 32 tile's filter rows (more loads in flight)
#define QD_SGD_THREADS 512
template <typename T, int TF, int TC, int RR, bool UPD>
__global__ void sgd_pack_tiled_kernel(Plan P, float* w0, float* w1, float* w2, float* m0, float* m1, float* m2,
                                      const float* g0, const float* g1, const float* g2, float lr, float mom,
                                      float wd, int first, T* out);

template <typename T>
static void launch_pack_tiled(const Plan& P, const float* const w[3], T* out, cudaStream_t st) {
  float* wm[3] = {(float*)w[0], (float*)w[1], (float*)w[2]};
  const size_t smem = (size_t)32 * (32 * 9 + 1) * 4;
  const int blocks = P.nroles * ((P.F + 31) / 32) * ((P.C + 31) / 32);
  sgd_pack_tiled_kernel<T, 32, 32, 9, false><<<blocks, QD_SGD_THREADS, smem, st>>>(P, wm[0], wm[1], wm[2], nullptr, nullptr,
                                                                          nullptr, nullptr, nullptr, nullptr, 0.f,
                                                                          0.f, 0.f, 0, out);
}

void launch_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st) {
  if (dev_skip("pack")) return;
  long long nf = (long long)pack_fprop_elems(P), nd = (long long)pack_dgrad_elems(P);
  // every packed position is a weight (no structural zeros): the tiled kernel
  // reads the roles once, coalesced, and writes both layouts in contiguous runs
  // (large layers only: the row-per-block kernel below has more blocks for small ones)
  if (P.kind == QD_KIND_CONV && P.r == 3 && P.sq == 0 && P.Jd == P.nb * P.F && P.Cd == P.C &&
      (long long)P.nroles * ((P.F + 31) / 32) * ((P.C + 31) / 32) >= 2 * 148 && !getenv("QD_OLD_PACK")) {
    if (P.dtype == QD_BF16)
      launch_pack_tiled<bf16>(P, w, (bf16*)wpack, st);
    else
      launch_pack_tiled<float>(P, w, (float*)wpack, st);
    count_launch(st, "pack");
    return;
  }
  if (P.kind == QD_KIND_CONV && P.sq == 0 && P.Jd == P.nb * P.F && P.Cd == P.C) {
    const int rr = P.r * P.r;
    size_t smem = (size_t)(P.C > P.Jd ? P.C : P.Jd) * rr * 4;
    if (smem <= 200 * 1024) {
      if (P.dtype == QD_BF16)
        launch_pack_conv<bf16>(P, w, (bf16*)wpack, smem, st);
      else
        launch_pack_conv<float>(P, w, (float*)wpack, smem, st);
      count_launch(st, "pack");
      return;
    }
  }
  if (P.Kf % 4 || P.Kd % 4) {  // rows not a multiple of 4: one element per thread
    int blocks1 = (int)((nf + 255) / 256 + (nd + 255) / 256);
    if (P.dtype == QD_BF16)
      pack_one_kernel<bf16><<<blocks1, 256, 0, st>>>(P, w[0], w[1], w[2], (bf16*)wpack);
    else
      pack_one_kernel<float><<<blocks1, 256, 0, st>>>(P, w[0], w[1], w[2], (float*)wpack);
    count_launch(st, "pack");
    return;
  }
  int blocks = (int)((nf / 4 + 255) / 256 + (nd / 4 + 255) / 256);
  if (P.dtype == QD_BF16)
    pack_all_kernel<bf16><<<blocks, 256, 0, st>>>(P, w[0], w[1], w[2], (bf16*)wpack);
  else
    pack_all_kernel<float><<<blocks, 256, 0, st>>>(P, w[0], w[1], w[2], (float*)wpack);
  count_launch(st, "pack");
}

// fused SGD (trainer.py:50-61) + pack: one thread per weight element of every role
template <typename T>
__global__ void sgd_pack_kernel(Plan P, float* w0, float* w1, float* w2, float* m0, float* m1, float* m2,
                                const float* g0, const float* g1, const float* g2, float lr, float mom, float wd,
                                int first, T* out) {
  const int rr = P.r * P.r;
  const long long per = (long long)P.F * P.C * rr;  // elements of one role
  const long long nf = (long long)P.nb * P.F * P.Kf;
  const long long tot = per * P.nroles;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int role = (int)(i / per);
    const long long o = i - role * per;
    float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
    float* m = role == 0 ? m0 : (role == 1 ? m1 : m2);
    const float* g = role == 0 ? g0 : (role == 1 ? g1 : g2);
    const float d = g[o] + wd * w[o];
    const float v = first ? d : mom * m[o] + d;
    m[o] = v;
    const float nw = w[o] - lr * v;
    w[o] = nw;
    int f, c, tap;
    if (P.kind == QD_KIND_FC) {  // reference fc layout (in, out)
      c = (int)(o / P.F);
      f = (int)(o - (long long)c * P.F);
      tap = 0;
    } else {  // (F, C, r, r)
      f = (int)(o / ((long long)P.C * rr));
      const int rem = (int)(o - (long long)f * P.C * rr);
      c = rem / rr;
      tap = rem - c * rr;
    }
    int R, kf, cp, kd;
    pack_positions(P, role, f, c, tap, R, kf, cp, kd);
    const T pv = cvt<T>(nw);
    out[(size_t)R * P.Kf + kf] = pv;
    out[nf + (size_t)cp * P.Kd + kd] = pv;
  }
}

// tiled variant: block = (role, TF filters, TC channels) with all r*r taps. The
// update streams the role's contiguous (F, C, r, r) / (C, F) rows; the new weights
// go through shared memory so the packed fprop rows (c fastest) and dgrad rows
// (filter fastest) are written as contiguous runs instead of scattered 2-B stores.
// UPD = false: pack only (the weights are read, nothing is updated).
// Conv layouts only. Warp-row loops: phase 1 streams each filter's contiguous
// (c0..c0+TC) x r*r run into the tile in source order (tile row = [cl][tap] + 1
// pad float, an odd stride), phase 2 writes fprop rows (lane = channel), phase 3
// dgrad rows (lane = filter) -- no per-element index division anywhere.
template <typename T, int TF, int TC, int RR, bool UPD>  // RR = r*r at compile time (0: runtime)
__global__ void __launch_bounds__(512) sgd_pack_tiled_kernel(Plan P, float* w0, float* w1, float* w2, float* m0,
                                                             float* m1, float* m2, const float* g0,
                                                             const float* g1, const float* g2, float lr, float mom,
                                                             float wd, int first, T* out) {
  extern __shared__ float tile[];  // [TF][TC * rr + 1]
  __shared__ int Rrow[TF];
  const int rr = RR ? RR : P.r * P.r;
  const int RT = TC * rr, RS = RT + 1;
  const int ftiles = (P.F + TF - 1) / TF, ctiles = (P.C + TC - 1) / TC;
  int b = blockIdx.x;
  const int ct = b % ctiles;
  b /= ctiles;
  const int ft = b % ftiles, role = b / ftiles;
  const int f0 = ft * TF, c0 = ct * TC;
  float* w = role == 0 ? w0 : (role == 1 ? w1 : w2);
  float* m = role == 0 ? m0 : (role == 1 ? m1 : m2);
  const float* g = role == 0 ? g0 : (role == 1 ? g1 : g2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  // packed positions are affine in (c, tap) for a fixed (role, f) and in f for a
  // fixed (role, c, tap): take the offsets from pack_positions once
  int R0, kf0, cp0, kdl;
  pack_positions(P, role, f0, c0, rr - 1, R0, kf0, cp0, kdl);  // tap rr-1: kd = j(f0)
  kf0 -= (rr - 1) * P.C;                                          // kf of (f0, c0, tap 0)
  if ((int)threadIdx.x < TF) {
    int R, kf, cp, kd;
    const int f = f0 + threadIdx.x < P.F ? f0 + threadIdx.x : f0;
    pack_positions(P, role, f, c0, 0, R, kf, cp, kd);
    Rrow[threadIdx.x] = R;
  }
  const int fmax = min(TF, P.F - f0), cmax = min(TC, P.C - c0);
  const int qmax = cmax * rr;  // valid run length of one filter row
  for (int fi = warp; fi < fmax; fi += nw) {
    const size_t base = ((size_t)(f0 + fi) * P.C + c0) * rr;
    float* trow = tile + fi * RS;
#pragma unroll 3
    for (int q0 = 0; q0 < RT; q0 += 96) {
      float wv[3], gv[3], mv[3];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int q = q0 + lane + 32 * u;
        const bool ok = q < qmax;
        wv[u] = ok ? w[base + q] : 0.f;
        gv[u] = (UPD && ok) ? g[base + q] : 0.f;
        mv[u] = (UPD && ok && !first) ? m[base + q] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int q = q0 + lane + 32 * u;
        if (q >= qmax) continue;
        float nw_ = wv[u];
        if (UPD) {
          const float d = gv[u] + wd * wv[u];
          const float v = first ? d : mom * mv[u] + d;
          m[base + q] = v;
          nw_ = wv[u] - lr * v;
          w[base + q] = nw_;
        }
        trow[q] = nw_;
      }
    }
  }
  __syncthreads();
  // fprop rows (role, f): columns kf0 + tap C + c, channel fastest
  for (int row = warp; row < fmax * rr; row += nw) {
    const int fi = row / rr, tap = row - fi * rr;
    T* o = out + (size_t)Rrow[fi] * P.Kf + kf0 + tap * P.C;
    const float* t = tile + fi * RS + tap;
    for (int cl = lane; cl < cmax; cl += 32) o[cl] = cvt<T>(t[cl * rr]);
  }
  // dgrad rows (c): columns (rr-1-tap) Jd + j(f0) + fi, filter fastest
  T* od = out + (long long)P.nb * P.F * P.Kf + (size_t)cp0 * P.Kd + kdl;
  for (int row = warp; row < cmax * rr; row += nw) {
    const int cl = row / rr, tap = row - cl * rr;
    T* o = od + (size_t)cl * P.Kd + (rr - 1 - tap) * P.Jd;
    const float* t = tile + cl * rr + tap;
    for (int fi = lane; fi < fmax; fi += 32) o[fi] = cvt<T>(t[fi * RS]);
  }
}

template <typename T, int TF, int TC>
static void launch_sgd_tiled(const Plan& P, float* const w[3], float* const mom[3], const float* const grad[3],
                             float lr, float momentum, float wd, int first, T* out, cudaStream_t st) {
  const size_t smem = (size_t)TF * (TC * P.r * P.r + 1) * 4;
  const int blocks = P.nroles * ((P.F + TF - 1) / TF) * ((P.C + TC - 1) / TC);
  if (P.r == 3) {
    sgd_pack_tiled_kernel<T, TF, TC, 9, true><<<blocks, QD_SGD_THREADS, smem, st>>>(P, w[0], w[1], w[2], mom[0], mom[1], mom[2],
                                                                    grad[0], grad[1], grad[2], lr, momentum, wd,
                                                                    first, out);
    return;
  }
  raise_smem_attr((const void*)sgd_pack_tiled_kernel<T, TF, TC, 0, true>, smem);
  sgd_pack_tiled_kernel<T, TF, TC, 0, true><<<blocks, QD_SGD_THREADS, smem, st>>>(P, w[0], w[1], w[2], mom[0], mom[1], mom[2],
                                                                  grad[0], grad[1], grad[2], lr, momentum, wd,
                                                                  first, out);
}

void launch_sgd_pack(const Plan& P, float* const w[3], float* const mom[3], const float* const grad[3], float lr,
                     float momentum, float wd, int first, void* wpack, cudaStream_t st) {
  if (dev_skip("sgd")) return;
  const int rr = P.r * P.r;
  // 32 x 32 tiles unless that leaves most SMs idle (small layers: 16 x 16)
  const bool big = (long long)P.nroles * ((P.F + 31) / 32) * ((P.C + 31) / 32) >= 2 * 148;
  if (!getenv("QD_SGD_ELEM") && rr <= 49 && P.kind == QD_KIND_CONV) {
    if (P.dtype == QD_BF16) {
      if (rr <= 9 && big) launch_sgd_tiled<bf16, 32, 32>(P, w, mom, grad, lr, momentum, wd, first, (bf16*)wpack, st);
      else launch_sgd_tiled<bf16, 16, 16>(P, w, mom, grad, lr, momentum, wd, first, (bf16*)wpack, st);
    } else {
      if (rr <= 9 && big) launch_sgd_tiled<float, 32, 32>(P, w, mom, grad, lr, momentum, wd, first, (float*)wpack, st);
      else launch_sgd_tiled<float, 16, 16>(P, w, mom, grad, lr, momentum, wd, first, (float*)wpack, st);
    }
    count_launch(st, "sgd_pack");
    return;
  }
  const long long tot = (long long)P.F * P.C * rr * P.nroles;
  const int grid = grid_for(tot);
  if (P.dtype == QD_BF16)
    sgd_pack_kernel<bf16><<<grid, 256, 0, st>>>(P, w[0], w[1], w[2], mom[0], mom[1], mom[2], grad[0], grad[1],
                                                grad[2], lr, momentum, wd, first, (bf16*)wpack);
  else
    sgd_pack_kernel<float><<<grid, 256, 0, st>>>(P, w[0], w[1], w[2], mom[0], mom[1], mom[2], grad[0], grad[1],
                                                 grad[2], lr, momentum, wd, first, (float*)wpack);
  count_launch(st, "sgd_pack");
}

// ---------------------------------------------------------------------------
// generic tiled SIMT GEMM:  out[s][m][n] = sum_{k in split s} A(m,k) * B(n,k)
// ---------------------------------------------------------------------------
template <class LA, class LB>
static void simt_gemm(LA la, LB lb, int M, int N, long long K, int split, float* out, cudaStream_t st) {
  simt_gemm_ext(la, lb, M, N, K, split, out, st);
}

// fprop A: implicit im2col of x (optionally squared), m = output pixel
template <typename T>
struct FpropA {
  static constexpr bool kfast = true;  // k = (tap, c): channels contiguous
  const T* x; int H, W, C, OH, OW, r, s, p, K0, sq;
  __device__ float operator()(int m, long long kl) const {
    int k = (int)kl;
    int ow = m % OW, t = m / OW, oh = t % OH, n = t / OH;
    bool square = (sq == 1) || (sq == 2 && k < K0);
    int kk = k % K0;
    int tap = kk / C, c = kk % C, dy = tap / r, dx = tap % r;
    int h = oh * s + dy - p, w = ow * s + dx - p;
    if (h < 0 || h >= H || w < 0 || w >= W) return 0.f;
    float v = ld(x + (((size_t)n * H + h) * W + w) * C + c);
    return square ? v * v : v;
  }
};
// fprop B: GEMM column n = br*F + f -> packed row
template <typename T>
struct FpropB {
  static constexpr bool kfast = true;
  const T* wf; int F, nb, FT, Kf;
  __device__ float operator()(int n, long long k) const {
    int br = n / F, f = n % F;
    return ld(wf + (size_t)fprop_row(br, f, nb, FT) * Kf + k);
  }
};
// dgrad A: transposed-conv gather of D, m = input pixel, k = (e, j)
template <typename T>
struct DgradA {
  static constexpr bool kfast = true;  // k = (e, j): D channels contiguous
  const T* D; int H, W, OH, OW, r, s, p, Jd;
  __device__ float operator()(int m, long long kl) const {
    int k = (int)kl;
    int w = m % W, t = m / W, h = t % H, n = t / H;
    int e = k / Jd, j = k % Jd;
    int dy = r - 1 - e / r, dx = r - 1 - e % r;
    int th = h + p - dy, tw = w + p - dx;
    if (th < 0 || tw < 0 || th % s || tw % s) return 0.f;
    int oh = th / s, ow = tw / s;
    if (oh >= OH || ow >= OW) return 0.f;
    return ld(D + (((size_t)n * OH + oh) * OW + ow) * Jd + j);
  }
};
template <typename T>
struct RowMajorB {  // B(n, k) = w[n*K + k]
  static constexpr bool kfast = true;
  const T* w; long long K;
  __device__ float operator()(int n, long long k) const { return ld(w + (size_t)n * K + k); }
};
// wgrad A: A(j, pixel) = D[pixel][j]
template <typename T>
struct WgradA {
  static constexpr bool kfast = false;  // consecutive j contiguous
  const T* D; int Jd;
  __device__ float operator()(int j, long long q) const { return ld(D + (size_t)q * Jd + j); }
};
// wgrad B: B(kw, pixel) = im2col(x or x*x)[pixel][kw]
template <typename T>
struct WgradB {
  static constexpr bool kfast = false;  // consecutive kw (channels) contiguous
  FpropA<T> a;
  __device__ float operator()(int kw, long long q) const { return a((int)q, kw); }
};

// ---------------------------------------------------------------------------
// elementwise / reduction pieces
// ---------------------------------------------------------------------------
template <typename T>
__global__ void fwd_epilogue_kernel(Plan P, const float* G, int S, const float* b0, const float* b1,
                                    const float* b2, T* y, T* a, T* b) {
  long long total = P.Mout * P.F;
  int NG = P.nb * P.F;
  const size_t slice = (size_t)P.Mout * NG;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long m = i / P.F;
    int f = (int)(i % P.F);
    // the K slices of the GEMM output, summed in slice order (deterministic)
    float gv[3] = {0.f, 0.f, 0.f};
    for (int s = 0; s < S; ++s) {
      const float* gs = G + s * slice + m * NG;
      for (int br = 0; br < P.nb; ++br) gv[br] += gs[br * P.F + f];
    }
#define g_(br) gv[br]
    float out;
    if (P.family == QD_FAM_PROPOSED) {
      float av = g_(0) + b0[f], bv = g_(1) + b1[f];
      out = av * bv + (g_(2) + b2[f]);
      a[i] = cvt<T>(av); b[i] = cvt<T>(bv);
    } else if (P.family == QD_FAM_T4) {
      float av = g_(0), bv = g_(1);
      out = av * bv;
      a[i] = cvt<T>(av); b[i] = cvt<T>(bv);
    } else if (P.family == QD_FAM_T2AND4) {
      float av = g_(0), bv = g_(1);
      out = av * bv + g_(2);
      a[i] = cvt<T>(av); b[i] = cvt<T>(bv);
    } else if (P.family == QD_FAM_T3) {
      out = g_(0) * g_(0);
    } else if (P.family == QD_FAM_FIRST_ORDER) {
      out = g_(0) + b0[f];
    } else {
      out = g_(0);
    }
#undef g_
    y[i] = cvt<T>(out);
  }
}

// D = [dy*b | dy*a | dy] / [dy*b | dy*a]; column partial sums of D (fp32 products)
// or of dy (t2 / t2_linear / first_order) for the bias gradients.
template <typename T>
__global__ void bwd_prologue_kernel(Plan P, const T* dy, const T* a, const T* b, T* D,
                                    float* part, long long rows_per) {
  int s = blockIdx.x;
  long long r0 = (long long)s * rows_per, r1 = r0 + rows_per;
  if (r1 > P.Mout) r1 = P.Mout;
  bool mat = caches_ab(P.family);
  int F = P.F;
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
    for (long long m = r0; m < r1; ++m) {
      size_t i = (size_t)m * F + f;
      float g = ld(dy + i);
      if (mat) {
        float av = ld(a + i), bv = ld(b + i);
        float d0 = g * bv, d1 = g * av;
        T* drow = D + (size_t)m * P.Jd;
        drow[f] = cvt<T>(d0);
        drow[F + f] = cvt<T>(d1);
        if (d_has_g(P.family)) drow[2 * F + f] = cvt<T>(g);
        s0 += d0; s1 += d1; s2 += g;
      } else {
        s0 += g;
      }
    }
    float* o = part + (size_t)s * P.Jd;
    if (d_has_g(P.family)) { o[f] = s0; o[F + f] = s1; o[2 * F + f] = s2; }
    else if (P.family == QD_FAM_T4) { o[f] = s0; o[F + f] = s1; }
    else o[f] = s0;
  }
}

// t3 (neurons.py:406-411): a = Wa x is recomputed (never cached); D = 2 g a.
// `a` is the fp32 recompute (SIMT) or the stored bf16 recompute (tcgen05, in place).
template <typename T, typename A>
__global__ void t3_prologue_kernel(long long n, const T* dy, const A* a, T* D) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float t = ld(dy + i) * ld(a + i);
    D[i] = cvt<T>(t + t);
  }
}
void launch_t3_prologue(const Plan& P, const void* dy, const void* a, bool a_fp32, void* D, cudaStream_t st) {
  const long long n = P.Mout * P.F;
  if (P.dtype == QD_BF16) {
    if (a_fp32)
      t3_prologue_kernel<bf16, float><<<grid_for(n), 256, 0, st>>>(n, (const bf16*)dy, (const float*)a, (bf16*)D);
    else
      t3_prologue_kernel<bf16, bf16><<<grid_for(n), 256, 0, st>>>(n, (const bf16*)dy, (const bf16*)a, (bf16*)D);
  } else {
    t3_prologue_kernel<float, float><<<grid_for(n), 256, 0, st>>>(n, (const float*)dy, (const float*)a,
                                                                  (float*)D);
  }
  count_launch(st, "prologue_t3");
}

void launch_bwd_prologue(const Plan& P, const void* dy, const void* a, const void* b, void* D,
                         float* part, int split, cudaStream_t st) {
  long long rows_per = (P.Mout + split - 1) / split;
  int threads = P.F >= 256 ? 256 : ((P.F + 31) / 32) * 32;
  if (P.dtype == QD_BF16)
    bwd_prologue_kernel<bf16><<<split, threads, 0, st>>>(P, (const bf16*)dy, (const bf16*)a,
                                                         (const bf16*)b, (bf16*)D, part, rows_per);
  else
    bwd_prologue_kernel<float><<<split, threads, 0, st>>>(P, (const float*)dy, (const float*)a,
                                                          (const float*)b, (float*)D, part, rows_per);
  count_launch(st, "prologue_simt");
}

// bias gradient per role: proposed ba <- sum(dy*b) (block 0), bb <- sum(dy*a)
// (block 1), bc <- sum(dy) (block 2); first_order b <- sum(dy).
// One block per 32 columns; 8 row-groups sum strided partials, then a
// fixed-order combine (deterministic).
__global__ void __launch_bounds__(256) bias_finish_kernel(Plan P, const float* part, int S, float* d0,
                                                          float* d1, float* d2) {
  __shared__ float red[8][33];
  int col = threadIdx.x % 32, grp = threadIdx.x / 32;
  int j = blockIdx.x * 32 + col;
  float acc = 0.f;
  if (j < P.Jd)
    for (int s = grp; s < S; s += 8) acc += part[(size_t)s * P.Jd + j];
  red[grp][col] = acc;
  __syncthreads();
  if (grp == 0 && j < P.Jd) {
    float t = 0.f;
    for (int g = 0; g < 8; ++g) t += red[g][col];
    int role = j / P.F, f = j % P.F;
    float* dst = role == 0 ? d0 : (role == 1 ? d1 : d2);
    if (dst) dst[f] = t;
  }
}

void launch_bias_finish(const Plan& P, const float* part, int S, float* const db[3], cudaStream_t st) {
  if (P.nbias == 0) return;
  bias_finish_kernel<<<(P.Jd + 31) / 32, 256, 0, st>>>(P, part, S, db[0], db[1], db[2]);
  count_launch(st, "bias_finish");
}

// wgrad partials [S][Jd][Kf] -> reference layouts
__global__ void wgrad_finish_kernel(Plan P, const float* part, int S, float* w0, float* w1, float* w2) {
  long long total = (long long)P.Jd * P.Kf;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    int j = (int)(i / P.Kf), k = (int)(i % P.Kf);
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += part[(size_t)s * total + i];
    int role, f, kk;
    if (!wgrad_dst(P, j, k, role, f, kk)) continue;  // t2and4 structural zero
    int tap = kk / P.C, c = kk % P.C, dy = tap / P.r, dx = tap % P.r;
    float* dst = role == 0 ? w0 : (role == 1 ? w1 : w2);
    if (!dst) continue;
    if (P.kind == QD_KIND_FC) dst[(size_t)c * P.F + f] = acc;
    else dst[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx] = acc;
  }
}

void launch_wgrad_finish(const Plan& P, const float* part, int S, float* const dW[3], cudaStream_t st) {
  long long total = (long long)P.Jd * P.Kf;
  wgrad_finish_kernel<<<grid_for(total), 256, 0, st>>>(P, part, S, dW[0], dW[1], dW[2]);
  count_launch(st, "wgrad_finish");
}

template <typename T>
__global__ void square_kernel(const T* x, T* xs, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float v = ld(x + i);
    xs[i] = cvt<T>(v * v);
  }
}

void launch_square_out(const Plan& P, void* y, cudaStream_t st) {
  long long n = P.Mout * P.F;
  if (P.dtype == QD_BF16) square_kernel<bf16><<<grid_for(n), 256, 0, st>>>((const bf16*)y, (bf16*)y, n);
  else square_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)y, (float*)y, n);
  count_launch(st, "square_out");
}

// x*x for bf16, 8 elements per 16-B vector, 4 vectors in flight per thread (the
// element-wise kernel above ran at ~2.5 TB/s with its 2-byte accesses)
__global__ void __launch_bounds__(256) square_vec_kernel(const uint4* __restrict__ x, uint4* __restrict__ xs,
                                                         long long n8) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  constexpr int U = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n8; i0 += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      v[u] = i < n8 ? __ldg(x + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long i = i0 + u * stride;
      if (i >= n8) break;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v[u]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(h[e]);
        h[e] = __floats2bfloat162_rn(f.x * f.x, f.y * f.y);
      }
      xs[i] = v[u];
    }
  }
}

void launch_square(const Plan& P, const void* x, void* xs, cudaStream_t st) {
  long long n = P.Min * P.C;
  if (P.dtype == QD_BF16 && n % 8 == 0 && (uintptr_t)x % 16 == 0 && (uintptr_t)xs % 16 == 0) {
    const long long n8 = n / 8;
    long long g = (n8 + 4 * 256 - 1) / (4 * 256);
    if (g > 148 * 8) g = 148 * 8;
    launch_pdl(square_vec_kernel, dim3((unsigned)(g < 1 ? 1 : g)), dim3(256), 0, st, (const uint4*)x, (uint4*)xs, n8);
  } else if (P.dtype == QD_BF16) {
    square_kernel<bf16><<<grid_for(n), 256, 0, st>>>((const bf16*)x, (bf16*)xs, n);
  } else {
    square_kernel<float><<<grid_for(n), 256, 0, st>>>((const float*)x, (float*)xs, n);
  }
  count_launch(st, "square");
}

// dgrad epilogue: dx = Q (first_order/t4/proposed), 2 x Q (t2),
// 2 x Q[:, :C] + Q[:, C:] (t2_linear)  -- neurons.py:400-405 "t = ds*x; dx = t + t"
template <typename T>
__global__ void dgrad_epilogue_kernel(Plan P, const float* Q, int S, const T* x, T* dx) {
  long long total = P.Min * P.C;
  const size_t slice = (size_t)P.Min * P.Cd;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long m = i / P.C;
    int c = (int)(i % P.C);
    float q0 = 0.f, q1 = 0.f;  // K slices summed in slice order (deterministic)
    for (int s = 0; s < S; ++s) {
      q0 += Q[s * slice + m * P.Cd + c];
      if (P.sq == 2) q1 += Q[s * slice + m * P.Cd + P.C + c];
    }
    float v;
    if (P.sq == 0) v = q0;
    else {
      float t = q0 * ld(x + i);
      v = t + t;
      if (P.sq == 2) v += q1;
    }
    dx[i] = cvt<T>(v);
  }
}

// ---------------------------------------------------------------------------
// full SIMT forward / backward
// ---------------------------------------------------------------------------
template <typename T>
static int simt_forward_t(const Plan& P, const T* x, const T* wf, const float* const bias[3], T* y,
                          T* a, T* b, char* ws, const Workspace& L, cudaStream_t st) {
  float* G = (float*)(ws + L.off_P);
  FpropA<T> la{x, P.H, P.W, P.C, P.OH, P.OW, P.r, P.s, P.p, P.K0, P.sq};
  FpropB<T> lb{wf, P.F, P.nb, P.FT, P.Kf};
  const int S = L.sk_f > 0 ? L.sk_f : 1;
  simt_gemm(la, lb, (int)P.Mout, P.nb * P.F, P.Kf, S, G, st);
  long long total = P.Mout * P.F;
  fwd_epilogue_kernel<T><<<grid_for(total), 256, 0, st>>>(P, G, S, bias[0], bias[1], bias[2], y, a, b);
  count_launch(st, "fwd_epilogue_simt");
  return check_launch("simt forward");
}

int simt_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3],
                 void* y, void* a, void* b, char* ws, const Workspace& L, cudaStream_t st) {
  if (P.dtype == QD_BF16)
    return simt_forward_t<bf16>(P, (const bf16*)x, (const bf16*)wpack, bias, (bf16*)y, (bf16*)a,
                                (bf16*)b, ws, L, st);
  return simt_forward_t<float>(P, (const float*)x, (const float*)wpack, bias, (float*)y, (float*)a,
                               (float*)b, ws, L, st);
}

template <typename T>
static int simt_backward_t(const Plan& P, const T* x, const T* wpack, const T* a, const T* b,
                           const T* dy, T* dx, float* const dW[3], float* const db[3], char* ws,
                           const Workspace& L, cudaStream_t st, bool want_dx) {
  const T* wd = wpack + pack_fprop_elems(P);
  float* bpart = (float*)(ws + L.off_BS);
  const T* D = dy;
  if (caches_ab(P.family) && !(P.flags & QD_FLAG_D_GIVEN)) D = (const T*)(ws + L.off_D);
  if (P.flags & QD_FLAG_D_GIVEN) {
    // `dy` is the operand D already (qd_bn_backward_D formed it and the bias grads)
  } else if (P.family == QD_FAM_T3) {
    // recompute a = Wa x (fp32, the forward GEMM) and form D = 2 g a
    float* G = (float*)(ws + L.off_P);
    FpropA<T> la{x, P.H, P.W, P.C, P.OH, P.OW, P.r, P.s, P.p, P.K0, P.sq};
    FpropB<T> lb{wpack, P.F, P.nb, P.FT, P.Kf};
    simt_gemm(la, lb, (int)P.Mout, P.F, P.Kf, 1, G, st);
    D = (const T*)(ws + L.off_D);
    launch_t3_prologue(P, dy, G, true, (void*)D, st);
  } else {
    launch_bwd_prologue(P, dy, a, b, (void*)D, bpart, L.bs_split, st);
  }
  if (db[0]) launch_bias_finish(P, bpart, L.bs_split, db, st);
  if (dW[0]) {
    // wgrad: [Jd][Kf] = D^T * im2col(x | x*x), split over pixels
    float* part = (float*)(ws + L.off_WG);
    WgradA<T> wa{D, P.Jd};
    WgradB<T> wb{FpropA<T>{x, P.H, P.W, P.C, P.OH, P.OW, P.r, P.s, P.p, P.K0, P.sq}};
    simt_gemm(wa, wb, P.Jd, P.Kf, P.Mout, L.wg_split, part, st);
    launch_wgrad_finish(P, part, L.wg_split, dW, st);
  }
  if (want_dx) {
    float* Q = (float*)(ws + L.off_P);
    DgradA<T> da{D, P.H, P.W, P.OH, P.OW, P.r, P.s, P.p, P.Jd};
    RowMajorB<T> dbm{wd, P.Kd};
    const int S = L.sk_d > 0 ? L.sk_d : 1;
    simt_gemm(da, dbm, (int)P.Min, P.Cd, P.Kd, S, Q, st);
    long long total = P.Min * P.C;
    dgrad_epilogue_kernel<T><<<grid_for(total), 256, 0, st>>>(P, Q, S, x, dx);
    count_launch(st, "dgrad_epilogue_simt");
  }
  return check_launch("simt backward");
}

int simt_backward(const Plan& P, const void* x, const void* wpack, const void* a, const void* b,
                  const void* dy, void* dx, float* const dW[3], float* const db[3], char* ws,
                  const Workspace& L, cudaStream_t st) {
  bool want_dx = dx != nullptr;
  if (P.dtype == QD_BF16)
    return simt_backward_t<bf16>(P, (const bf16*)x, (const bf16*)wpack, (const bf16*)a,
                                 (const bf16*)b, (const bf16*)dy, (bf16*)dx, dW, db, ws, L, st,
                                 want_dx);
  return simt_backward_t<float>(P, (const float*)x, (const float*)wpack, (const float*)a,
                                (const float*)b, (const float*)dy, (float*)dx, dW, db, ws, L, st,
                                want_dx);
}

}  // namespace qd

namespace qd {
// One launch folds both fixed-order reductions of the backward pass:
// blocks [0, nwb) sum the wgrad split-K partials -- 32 float4 columns x 8
// partial groups per block, combined in a fixed order (deterministic) -- and
// scatter them into the reference layouts; the rest sum the bias partials.
// bias columns: 8 columns x 32 partial groups per block, 4 independent chains per thread
__device__ __forceinline__ void finish_bias_block(const Plan& P, int bblk, const float* __restrict__ bpart, int SB,
                                                  float* d0, float* d1, float* d2) {
  if (P.nbias == 0 || !d0) return;
  __shared__ float redb[32][9];
  const int bc = threadIdx.x % 8, bg = threadIdx.x / 8;
  int j = bblk * 8 + bc;
  float a[8];  // eight chains: 8 partial loads in flight per thread (latency-bound fold)
#pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = 0.f;
  if (j < P.Jd) {
    int s = bg;
    for (; s + 7 * 32 < SB; s += 8 * 32) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = bpart[(size_t)(s + 32 * u) * P.Jd + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += v[u];
    }
    for (; s < SB; s += 32) a[0] += bpart[(size_t)s * P.Jd + j];
  }
  redb[bg][bc] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  __syncthreads();
  if (bg == 0 && j < P.Jd) {
    float t = 0.f;
    for (int gq = 0; gq < 32; ++gq) t += redb[gq][bc];
    int role = j / P.F, f = j % P.F;
    float* dst = role == 0 ? d0 : (role == 1 ? d1 : d2);
    if (dst) dst[f] = t;
  }
}

__global__ void __launch_bounds__(256) bwd_finish_kernel(Plan P, const float* __restrict__ wpart, int S, WSplits wsp,
                                                         float* w0, float* w1, float* w2,
                                                         const float* __restrict__ bpart, int SB, float* d0,
                                                         float* d1, float* d2, int nwb) {
  __shared__ float4 red4[8][33];
  __shared__ float red[8][33];
  const int col = threadIdx.x % 32, grp = threadIdx.x / 32;
  if ((int)blockIdx.x < nwb) {
    if (!w0) return;
    const long long total = (long long)P.Jd * P.Kf;
    const long long i4 = ((long long)blockIdx.x * 32 + col) * 4;
    int Sk = S;
    if (i4 < total && wsp.ng > 0) {
      int k = (int)(i4 % P.Kf), kk = k % P.K0;
      int tg = (kk / P.C / 2) / wsp.pp;
#pragma unroll
      for (int t = 0; t < 16; ++t)  // static indexing: no local-memory copy of wsp
        if (t == tg) Sk = wsp.s[t];
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i4 < total) {
      const float4* src = reinterpret_cast<const float4*>(wpart + i4);
      const long long stride4 = total / 4;
      // four independent chains (loads in flight), combined in a fixed order
      float4 c1 = make_float4(0.f, 0.f, 0.f, 0.f), c2 = c1, c3 = c1;
      int s = grp;
      for (; s + 24 < Sk; s += 32) {
        float4 v0 = __ldg(src + s * stride4), v1 = __ldg(src + (s + 8) * stride4);
        float4 v2 = __ldg(src + (s + 16) * stride4), v3 = __ldg(src + (s + 24) * stride4);
        acc.x += v0.x; acc.y += v0.y; acc.z += v0.z; acc.w += v0.w;
        c1.x += v1.x; c1.y += v1.y; c1.z += v1.z; c1.w += v1.w;
        c2.x += v2.x; c2.y += v2.y; c2.z += v2.z; c2.w += v2.w;
        c3.x += v3.x; c3.y += v3.y; c3.z += v3.z; c3.w += v3.w;
      }
      for (; s < Sk; s += 8) {
        float4 v = __ldg(src + s * stride4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      acc.x += c1.x + (c2.x + c3.x); acc.y += c1.y + (c2.y + c3.y);
      acc.z += c1.z + (c2.z + c3.z); acc.w += c1.w + (c2.w + c3.w);
    }
    red4[grp][col] = acc;
    __syncthreads();
    if (grp != 0 || i4 >= total) return;
    float4 t = red4[0][col];
    for (int gq = 1; gq < 8; ++gq) {
      float4 v = red4[gq][col];
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    float av[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      long long i = i4 + e;
      int j = (int)(i / P.Kf), k = (int)(i % P.Kf);
      int role, f, kk;
      if (!wgrad_dst(P, j, k, role, f, kk)) continue;  // t2and4 structural zero
      int tap = kk / P.C, c = kk % P.C, dy = tap / P.r, dx = tap % P.r;
      float* dst = role == 0 ? w0 : (role == 1 ? w1 : w2);
      if (!dst) continue;
      if (P.kind == QD_KIND_FC) dst[(size_t)c * P.F + f] = av[e];
      else dst[(((size_t)f * P.C + c) * P.r + dy) * P.r + dx] = av[e];
    }
  } else {
    finish_bias_block(P, (int)blockIdx.x - nwb, bpart, SB, d0, d1, d2);
  }
}

// fc weight fold: 32 x 32 tiles of the [Jd][Kf] partials, slices summed in order,
// transposed through shared memory into the fc layout (in, out) = dst[c F + f]:
// reads coalesced along c, writes along f (the element-wise fold above writes
// with stride F). Blocks [0, ntile) fold weights, the rest the bias partials.
__global__ void __launch_bounds__(256) wfinish_fc_kernel(Plan P, const float* __restrict__ wpart, int S,
                                                         float* w0, float* w1, float* w2,
                                                         const float* __restrict__ bpart, int SB, float* d0,
                                                         float* d1, float* d2, int ntile) {
  __shared__ float t[32][33];
  if ((int)blockIdx.x >= ntile) {
    finish_bias_block(P, (int)blockIdx.x - ntile, bpart, SB, d0, d1, d2);
    return;
  }
  if (!w0) return;
  const int tk = (P.Kf + 31) / 32;
  const int j0 = (blockIdx.x / tk) * 32, k0 = (blockIdx.x % tk) * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const size_t slice = (size_t)P.Jd * P.Kf;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = j0 + ty + 8 * i, k = k0 + tx;
    float acc = 0.f;
    if (j < P.Jd && k < P.Kf)
      for (int sl = 0; sl < S; ++sl) acc += __ldg(wpart + sl * slice + (size_t)j * P.Kf + k);
    t[ty + 8 * i][tx] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty + 8 * i, j = j0 + tx;  // k = input channel c, j = role F + f
    if (j >= P.Jd || k >= P.Kf) continue;
    const int role = j / P.F, f = j - role * P.F;
    float* dst = role == 0 ? w0 : (role == 1 ? w1 : w2);
    if (dst) dst[(size_t)k * P.F + f] = t[tx][ty + 8 * i];
  }
}

// conv weight fold: block = (NJ D channels j, K half, 64-channel chunk). G warp
// groups sum interleaved split subsets (fixed order) of the block's NJ x rr x 64
// partial values (G x NJ = 8: with few splits the lanes cover more rows, so every
// block keeps ~1k independent loads in flight), and the totals are written
// transposed into the reference (F, C, r, r) layout: partial reads and gradient
// writes are both coalesced (the element-wise fold above writes with stride r*r).
template <int RR>  // r*r at compile time (0: runtime)
__global__ void __launch_bounds__(256) wfinish_conv_kernel(Plan P, const float* __restrict__ wpart, int S,
                                                           WSplits wsp, float* w0, float* w1, float* w2,
                                                           const float* __restrict__ bpart, int SB, float* d0,
                                                           float* d1, float* d2, int nwb) {
  extern __shared__ float4 red[];  // [G][NJ][rr][17]: 64 channels + 4 pad floats per tap row
  if ((int)blockIdx.x >= nwb) {
    finish_bias_block(P, (int)blockIdx.x - nwb, bpart, SB, d0, d1, d2);
    return;
  }
  if (!w0) return;
  const int G = S >= 8 ? 8 : (S >= 4 ? 4 : (S >= 2 ? 2 : 1)), NJ = 8 / G, L = 256 / G;
  const int rr = RR ? RR : P.r * P.r, nv = rr * 16, nvb = NJ * nv;
  const int cch = P.C / 64, nh = P.Kf / P.K0;
  int b = blockIdx.x;
  const int cb = b % cch;
  b /= cch;
  const int half = b % nh, j0 = (b / nh) * NJ;
  const int lane = threadIdx.x % L, grp = threadIdx.x / L;
  const long long stride4 = (long long)P.Jd * P.Kf / 4;
  const float4* src = reinterpret_cast<const float4*>(wpart + half * P.K0 + cb * 64) + (long long)j0 * (P.Kf / 4);
  const int c4s = P.C / 4, kf4 = P.Kf / 4;
  for (int v0 = 0; v0 < nvb; v0 += 4 * L) {
    float4 acc[4];
    int off[4], soff[4], sk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      const int vb = v0 + lane + L * u, jj = vb / nv, v = vb - jj * nv, tap = v >> 4, c4 = v & 15;
      off[u] = jj * kf4 + tap * c4s + c4;
      soff[u] = (jj * rr + tap) * 17 + c4;
      int sv = S;
      if (wsp.ng > 0) {
        const int tg = (tap / 2) / wsp.pp;
#pragma unroll
        for (int t = 0; t < 16; ++t)  // static indexing: no local-memory copy of wsp
          if (t == tg) sv = wsp.s[t];
      }
      sk[u] = (vb < nvb && j0 + jj < P.Jd) ? sv : 0;
    }
#pragma unroll 2
    for (int s = grp; s < S; s += G) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (s < sk[u]) {
          const float4 x = __ldg(src + s * stride4 + off[u]);
          acc[u].x += x.x; acc[u].y += x.y; acc[u].z += x.z; acc[u].w += x.w;
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + lane + L * u < nvb) red[grp * NJ * rr * 17 + soff[u]] = acc[u];
  }
  __shared__ float* rowdst[8];
  if ((int)threadIdx.x < NJ) {
    const int j = j0 + threadIdx.x;
    float* o = nullptr;
    int role, f, kk;
    if (j < P.Jd && wgrad_dst(P, j, half * P.K0, role, f, kk)) {  // else t2and4 structural zero
      float* dst = role == 0 ? w0 : (role == 1 ? w1 : w2);
      if (dst) o = dst + ((size_t)f * P.C + cb * 64) * rr;
    }
    rowdst[threadIdx.x] = o;
  }
  __syncthreads();
  const float* redf = reinterpret_cast<const float*>(red);
  const int gstride = NJ * rr * 68;  // floats per split group
  const int per = 64 * rr;           // outputs per row, a multiple of 4
  for (int q = threadIdx.x; q < NJ * per / 4; q += blockDim.x) {
    const int e4 = 4 * q, jj = e4 / per, e = e4 - jj * per;
    float* o = rowdst[jj];
    if (!o) continue;
    const float* rj = redf + jj * rr * 68;
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = (e + k) / rr, tap = e + k - c * rr;
      const float* qp = rj + tap * 68 + c;
      float t = qp[0];
      for (int g = 1; g < G; ++g) t += qp[g * gstride];
      v[k] = t;
    }
    *reinterpret_cast<float4*>(o + e) = make_float4(v[0], v[1], v[2], v[3]);  // (f C + 64 cb) rr % 4 == 0
  }
}

// phase 1 of the conv fold when S > 1: the S partial slices summed in place into
// slice 0. Block = L float4 columns x G split groups (G = min(S, 8) rounded down
// to a power of two, L = 256 / G: every thread loads); group g sums splits
// g, g+G, ... with 4 loads in flight and the groups are added in order --
// contiguous reads and writes; the transposing fold then reads one slice
__global__ void __launch_bounds__(256) wsum_kernel(Plan P, float* __restrict__ part, int S, WSplits wsp, int G) {
  __shared__ float4 red[256];
  const int L = 256 / G;
  const int col = threadIdx.x % L, grp = threadIdx.x / L;
  const long long n4 = (long long)P.Jd * P.Kf / 4;
  float4* p4 = reinterpret_cast<float4*>(part);
  // grid-stride over column tiles: a few resident blocks per SM do all the work
  // (one short block per tile spent its time in block launch, not in loads)
  for (long long i0 = (long long)blockIdx.x * L; i0 < n4; i0 += (long long)gridDim.x * L) {
    const long long i = i0 + col;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n4) {
      int Sk = S;
      if (wsp.ng > 0) {
        const int k = (int)((i * 4) % P.Kf), kk = k % P.K0, tg = (kk / P.C / 2) / wsp.pp;
#pragma unroll
        for (int t = 0; t < 16; ++t)  // static indexing: no local-memory copy of wsp
          if (t == tg) Sk = wsp.s[t];
      }
      // eight chains: 8 slice loads in flight per thread (L2-latency bound)
      float4 c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) c[u] = acc;
      int s = grp;
      for (; s + 7 * G < Sk; s += 8 * G) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p4[(s + u * G) * n4 + i];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          c[u].x += v[u].x; c[u].y += v[u].y; c[u].z += v[u].z; c[u].w += v[u].w;
        }
      }
      for (; s < Sk; s += G) {
        const float4 v = p4[s * n4 + i];
        c[0].x += v.x; c[0].y += v.y; c[0].z += v.z; c[0].w += v.w;
      }
#pragma unroll
      for (int e = 4; e > 0; e >>= 1)
#pragma unroll
        for (int u = 0; u < e; ++u) {
          c[u].x += c[u + e].x; c[u].y += c[u + e].y; c[u].z += c[u + e].z; c[u].w += c[u + e].w;
        }
      acc = c[0];
    }
    red[threadIdx.x] = acc;
    __syncthreads();  // every group has read slice 0 before it is overwritten
    if (grp == 0 && i < n4) {
      float4 t = red[col];
      for (int g = 1; g < G; ++g) {
        const float4 v = red[g * L + col];
        t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
      }
      p4[i] = t;
    }
    __syncthreads();  // red is reused by the next tile
  }
}

void launch_bwd_finish(const Plan& P, const float* wpart, int S, const WSplits& ws, float* const dW[3],
                       const float* bpart, int SB, float* const db[3], cudaStream_t st) {
  if (dev_skip("finish")) return;
  long long total = (long long)P.Jd * P.Kf;  // Kf is a multiple of 64 on the tcgen05 path
  int nwb = dW[0] ? (int)((total / 4 + 31) / 32) : 0;
  int nbb = (P.nbias && db[0]) ? (P.Jd + 7) / 8 : 0;
  if (nwb + nbb == 0) return;
  bool al16 = true;  // the transposing fold writes float4
  for (int i = 0; i < 3; ++i) al16 = al16 && ((uintptr_t)dW[i] % 16 == 0);
  if (P.kind == QD_KIND_CONV && P.C % 64 == 0 && P.r <= 7 && al16 && !getenv("QD_OLD_FINISH")) {
    WSplits ws1 = ws;
    if (S > 1 && dW[0] && !getenv("QD_FOLD_1PASS")) {
      // sum the slices first (contiguous, all SMs busy), then transpose one slice
      const long long n4 = (long long)P.Jd * P.Kf / 4;
      // split groups per column only while the columns alone leave threads
      // idle (~300K threads fill the GPU): a group of one slice-load per
      // thread per tile is L2-latency bound (measured 21 us on 7 MB slices)
      int G = 1;
      while (G < 8 && 2 * G <= S && n4 * G < 150000) G *= 2;
      const int L = 256 / G;
      const long long tiles = (n4 + L - 1) / L;
      wsum_kernel<<<(unsigned)(tiles < 148 * 8 ? tiles : 148 * 8), 256, 0, st>>>(P, const_cast<float*>(wpart), S, ws,
                                                                                 G);
      count_launch(st, "wsum");
      S = 1;
      ws1.ng = 0;
    }
    const int G = S >= 8 ? 8 : (S >= 4 ? 4 : (S >= 2 ? 2 : 1)), NJ = 8 / G;  // as in the kernel
    const int nwc = dW[0] ? (P.Jd + NJ - 1) / NJ * (P.Kf / P.K0) * (P.C / 64) : 0;
    const size_t smem = (size_t)8 * P.r * P.r * 17 * sizeof(float4);
    raise_smem_attr((const void*)wfinish_conv_kernel<0>, smem);  // r = 3 / 1 stay under 48 KB
    if (P.r == 3)
      wfinish_conv_kernel<9><<<nwc + nbb, 256, smem, st>>>(P, wpart, S, ws1, dW[0], dW[1], dW[2], bpart, SB, db[0],
                                                           db[1], db[2], nwc);
    else if (P.r == 1)
      wfinish_conv_kernel<1><<<nwc + nbb, 256, smem, st>>>(P, wpart, S, ws1, dW[0], dW[1], dW[2], bpart, SB, db[0],
                                                           db[1], db[2], nwc);
    else
      wfinish_conv_kernel<0><<<nwc + nbb, 256, smem, st>>>(P, wpart, S, ws1, dW[0], dW[1], dW[2], bpart, SB, db[0],
                                                           db[1], db[2], nwc);
  } else if (P.kind == QD_KIND_FC && P.sq == 0 && ws.ng == 0 && !getenv("QD_OLD_FINISH")) {
    const int ntile = dW[0] ? ((P.Jd + 31) / 32) * ((P.Kf + 31) / 32) : 0;
    wfinish_fc_kernel<<<ntile + nbb, 256, 0, st>>>(P, wpart, S, dW[0], dW[1], dW[2], bpart, SB, db[0], db[1], db[2],
                                                   ntile);
  } else {
    if (getenv("QD_VERBOSE"))
      fprintf(stderr, "[qd] generic bwd_finish: kind %d fam %d C %d F %d r %d Jd %d Kf %d S %d ng %d SB %d nbb %d\n", P.kind,
              P.family, P.C, P.F, P.r, P.Jd, P.Kf, S, ws.ng, SB, nbb);
    bwd_finish_kernel<<<nwb + nbb, 256, 0, st>>>(P, wpart, S, ws, dW[0], dW[1], dW[2], bpart, SB, db[0], db[1],
                                                  db[2], nwb);
  }
  count_launch(st, "bwd_finish");
}
}  // namespace qd
