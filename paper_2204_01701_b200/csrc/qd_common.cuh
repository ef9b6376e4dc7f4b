// Shared host/device definitions for the quadratic-layer kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/quadra_b200.h"

namespace qd {

typedef __nv_bfloat16 bf16;

// Derived sizes of one layer (host and device).
struct Plan {
  int family, kind, dtype;
  int N, C, H, W, F, r, s, p;
  int OH, OW;
  long long Min;   // N*H*W input pixels
  long long Mout;  // N*OH*OW output pixels
  int nb;          // fprop GEMM branches sharing x: proposed 3, t4 2, else 1
  int sq;          // 0 none, 1 all of K squared (t2), 2 first half squared (t2_linear)
  int K0;          // r*r*C
  int Kf;          // fprop K: K0, or 2*K0 for t2_linear
  int FT;          // branch interleave tile for the packed fprop weights
  int Jd;          // channels of the backward operand D: proposed 3F, t4 2F, else F
  int Cd;          // dgrad GEMM N: C, or 2C for t2_linear
  int Kd;          // dgrad K: r*r*Jd
  int nroles;      // weight roles
  int nbias;       // bias roles
  unsigned flags;  // qd_desc flags
};

__host__ __device__ inline int conv_out(int size, int r, int s, int p) {
  // floor division like Python's // for the (always >= -r) numerator
  int num = size + 2 * p - r;
  return (num >= 0 ? num / s : -((-num + s - 1) / s)) + 1;
}

inline Plan make_plan(const qd_desc& d) {
  Plan P;
  P.family = d.family; P.kind = d.kind; P.dtype = d.dtype;
  P.N = d.N; P.C = d.C; P.H = d.H; P.W = d.W; P.F = d.F;
  P.r = d.r; P.s = d.stride; P.p = d.pad;
  P.flags = d.flags;
  P.OH = conv_out(P.H, P.r, P.s, P.p);
  P.OW = conv_out(P.W, P.r, P.s, P.p);
  P.Min = (long long)P.N * P.H * P.W;
  P.Mout = (long long)P.N * P.OH * P.OW;
  switch (P.family) {
    case QD_FAM_PROPOSED: P.nb = 3; P.sq = 0; P.Jd = 3 * P.F; P.nroles = 3; P.nbias = 3; break;
    case QD_FAM_T4:       P.nb = 2; P.sq = 0; P.Jd = 2 * P.F; P.nroles = 2; P.nbias = 0; break;
    case QD_FAM_T2:       P.nb = 1; P.sq = 1; P.Jd = P.F;     P.nroles = 1; P.nbias = 0; break;
    case QD_FAM_T2_LINEAR:P.nb = 1; P.sq = 2; P.Jd = P.F;     P.nroles = 2; P.nbias = 0; break;
    default:              P.nb = 1; P.sq = 0; P.Jd = P.F;     P.nroles = 1; P.nbias = 1; break;
  }
  P.K0 = P.r * P.r * P.C;
  P.Kf = (P.sq == 2) ? 2 * P.K0 : P.K0;
  P.FT = (P.F % 64 == 0) ? 64 : P.F;
  P.Cd = (P.sq == 2) ? 2 * P.C : P.C;
  P.Kd = P.r * P.r * P.Jd;
  return P;
}

// Row of branch `br`, channel `f` inside the packed fprop weights: branches are
// interleaved per FT-wide channel tile so one TMA box of nb*FT rows carries
// [Wa_tile; Wb_tile; Wc_tile] for the same output channels.
__host__ __device__ inline int fprop_row(int br, int f, int nb, int FT) {
  return (f / FT) * nb * FT + br * FT + (f % FT);
}

template <typename T> __device__ inline float ld(const T* p);
template <> __device__ inline float ld<float>(const float* p) { return *p; }
template <> __device__ inline float ld<bf16>(const bf16* p) { return __bfloat162float(*p); }
template <typename T> __device__ inline T cvt(float v);
template <> __device__ inline float cvt<float>(float v) { return v; }
template <> __device__ inline bf16 cvt<bf16>(float v) { return __float2bfloat16_rn(v); }

}  // namespace qd
