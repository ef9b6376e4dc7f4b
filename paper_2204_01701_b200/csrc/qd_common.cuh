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
    case QD_FAM_T3:       P.nb = 1; P.sq = 0; P.Jd = P.F;     P.nroles = 1; P.nbias = 0; break;
    // t2and4: K = [x*x | x] like t2_linear, three branches like proposed (a, b read
    // the x half, c the x*x half; the other halves are structural zeros)
    case QD_FAM_T2AND4:   P.nb = 3; P.sq = 2; P.Jd = 3 * P.F; P.nroles = 3; P.nbias = 0; break;
    case QD_FAM_T1_PURE:  P.nb = 1; P.sq = 0; P.Jd = P.F;     P.nroles = 1; P.nbias = 0; break;
    case QD_FAM_T1_FULL:
    case QD_FAM_T1AND2:   P.nb = 1; P.sq = 0; P.Jd = P.F;     P.nroles = 2; P.nbias = 0; break;
    default:              P.nb = 1; P.sq = 0; P.Jd = P.F;     P.nroles = 1; P.nbias = 1; break;
  }
  P.K0 = P.r * P.r * P.C;
  P.Kf = (P.sq == 2) ? 2 * P.K0 : P.K0;
  P.FT = (P.F % 64 == 0) ? 64 : P.F;
  P.Cd = (P.sq == 2) ? 2 * P.C : P.C;
  P.Kd = P.r * P.r * P.Jd;
  return P;
}

// families whose forward caches a and b (neurons.py:110-111)
__host__ __device__ inline bool caches_ab(int family) {
  return family == QD_FAM_PROPOSED || family == QD_FAM_T4 || family == QD_FAM_T2AND4;
}
// D = [g b | g a | g] (three blocks) for proposed and t2and4
__host__ __device__ inline bool d_has_g(int family) {
  return family == QD_FAM_PROPOSED || family == QD_FAM_T2AND4;
}

// packed fprop weight (branch br, GEMM column k): source role and tap-major index kk;
// false for t2and4's structural zeros. K = [x*x | x] when sq == 2.
__host__ __device__ inline bool fprop_src(const Plan& P, int br, int k, int& role, int& kk) {
  if (P.sq == 2) {
    const int half = k / P.K0;
    kk = k - half * P.K0;
    if (P.family == QD_FAM_T2AND4) {
      role = br;
      return (br == 2) == (half == 0);
    }
    role = half;  // t2_linear: Wa on x*x, Wc on x
    return true;
  }
  role = br;
  kk = k;
  return true;
}
// packed dgrad weight (row cp, D channel j): source role, input channel c, filter f.
// sq == 2: rows [0, C) produce the x*x-branch gradient, rows [C, 2C) the linear one.
__host__ __device__ inline bool dgrad_src(const Plan& P, int cp, int j, int& role, int& c, int& f) {
  if (P.family == QD_FAM_T2AND4) {
    const int part = cp / P.C, jb = j / P.F;
    c = cp - part * P.C;
    f = j - jb * P.F;
    role = jb;  // D blocks: g b -> Wa, g a -> Wb, g -> Wc
    return (part == 0) == (jb == 2);
  }
  if (P.sq == 2) {
    role = cp / P.C;
    c = cp % P.C;
    f = j;
    return true;
  }
  role = j / P.F;
  f = j % P.F;
  c = cp;
  return true;
}
// wgrad partial (D channel j, GEMM K index k) -> gradient role, filter f, tap-major kk
__host__ __device__ inline bool wgrad_dst(const Plan& P, int j, int k, int& role, int& f, int& kk) {
  f = j % P.F;
  if (P.sq == 2) {
    const int half = k / P.K0;
    kk = k - half * P.K0;
    if (P.family == QD_FAM_T2AND4) {
      role = j / P.F;
      return (role == 2) == (half == 0);
    }
    role = half;
    return true;
  }
  role = j / P.F;
  kk = k;
  return true;
}

// inverse of fprop_src / dgrad_src: where weight element (role, f, c, tap) lives in
// the packed fprop matrix (row R, column kf) and the packed dgrad matrix (row cp, column kd)
__host__ __device__ inline void pack_positions(const Plan& P, int role, int f, int c, int tap, int& R, int& kf,
                                               int& cp, int& kd) {
  const int rr = P.r * P.r, e = rr - 1 - tap;
  int br = role, half = 0, j = role * P.F + f;
  cp = c;
  if (P.family == QD_FAM_T2AND4) {
    half = role == 2 ? 0 : 1;
    cp = (role == 2 ? 0 : 1) * P.C + c;
  } else if (P.sq == 2) {  // t2_linear: one branch, role = K half
    br = 0;
    half = role;
    j = f;
    cp = role * P.C + c;
  }
  const int tile = f / P.FT;
  R = tile * P.nb * P.FT + br * P.FT + (f - tile * P.FT);
  kf = half * P.K0 + tap * P.C + c;
  kd = e * P.Jd + j;
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
