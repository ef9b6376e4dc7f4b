// Depth-wise quadratic convolution, shared-memory tiled (kind = dwconv, r = 3,
// stride 1 or 2, C % 32 == 0): the MobileNet rows of SURVEY.md §8(f) row 3.
// Reference: tensor.py:367-418 (dw_im2col, dwconv_forward_raw,
// dwconv_backward_raw) under the family algebra of neurons.py:235-276 / :393-444;
// the same arithmetic as the direct kernels of qd_dw.cu, restructured for HBM:
//   - a CTA owns an 8 x 16 pixel tile of one image and 32 channels; its input
//     halo (and, backward, its D tile) is staged in shared memory once with
//     16-byte loads (zero fill = the padding), so each element leaves HBM once
//     instead of once per tap;
//   - a thread owns a channel pair: its 3 x 9 filter taps live in registers
//     (fp32 pairs, FFMA2), the family (roles, squared-input roles, epilogue) is a
//     template parameter, so the inner loops are straight-line FFMA2;
//   - the wgrad CTA walks a range of tiles, accumulates its 27 x 32 partials in
//     registers, folds its warps in a fixed order through shared memory, and
//     writes one partial row; dw_wgrad_finish folds the rows in order
//     (deterministic).
#include <stdio.h>
#include "qd_kernels.h"
#include "qd_dw.cuh"

namespace qd {

namespace {
constexpr int TH = 8, TW = 16, CB = 32, NT = 256;

template <typename T> struct P2;  // a channel pair in shared or global memory
template <> struct P2<bf16> {
  __device__ static float2 ld(const bf16* p) { return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p)); }
  __device__ static void st(bf16* p, float2 v) { *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v.x, v.y); }
};
template <> struct P2<float> {
  __device__ static float2 ld(const float* p) { return *reinterpret_cast<const float2*>(p); }
  __device__ static void st(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
};

// shared-memory bytes of each kernel (dynamic: the stride-2 / fp32 tiles pass 48 KB)
// two stages each (the next tile's loads in flight)
template <typename T, int S> constexpr int halo_bytes() { return ((TH - 1) * S + 3) * ((TW - 1) * S + 3) * CB * (int)sizeof(T); }
template <typename T, int S> constexpr int fwd_smem() { return 2 * halo_bytes<T, S>(); }
template <typename T, int S> constexpr int dgrad_smem(int nd) {
  return 2 * nd * ((TH + 1) / S + 2) * ((TW + 1) / S + 2) * CB * (int)sizeof(T);
}
template <typename T, int S> constexpr int wgrad_smem(int nd, int nr) {
  return 2 * (halo_bytes<T, S>() + nd * TH * TW * CB * (int)sizeof(T)) > 8 * nr * 9 * CB * 4
             ? 2 * (halo_bytes<T, S>() + nd * TH * TW * CB * (int)sizeof(T))
             : 8 * nr * 9 * CB * 4;
}

// family traits: roles, squared-input role mask, D block of each role
template <int FAM> struct DwF;
template <> struct DwF<QD_FAM_FIRST_ORDER> { static constexpr int NR = 1, SQ = 0, D1 = 0, D2 = 0; };
template <> struct DwF<QD_FAM_T2> { static constexpr int NR = 1, SQ = 1, D1 = 0, D2 = 0; };
template <> struct DwF<QD_FAM_T3> { static constexpr int NR = 1, SQ = 0, D1 = 0, D2 = 0; };
template <> struct DwF<QD_FAM_T4> { static constexpr int NR = 2, SQ = 0, D1 = 1, D2 = 0; };
template <> struct DwF<QD_FAM_PROPOSED> { static constexpr int NR = 3, SQ = 0, D1 = 1, D2 = 2; };
template <> struct DwF<QD_FAM_T2_LINEAR> { static constexpr int NR = 2, SQ = 1, D1 = 0, D2 = 0; };
template <> struct DwF<QD_FAM_T2AND4> { static constexpr int NR = 3, SQ = 4, D1 = 1, D2 = 2; };
template <int FAM> constexpr int dw_nd() {  // distinct D blocks the roles read
  return DwF<FAM>::NR == 1 ? 1 : (DwF<FAM>::D2 ? 3 : (DwF<FAM>::D1 ? 2 : 1));
}

__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }

struct TileGeo {
  int tilesW, tilesH, n, y0, x0;  // tile origin in the tile's own grid (outputs or inputs)
};
__device__ __forceinline__ TileGeo tile_of(int t, int H, int W) {
  TileGeo g;
  g.tilesW = (W + TW - 1) / TW;
  g.tilesH = (H + TH - 1) / TH;
  const int tw = t % g.tilesW;
  t /= g.tilesW;
  const int th = t % g.tilesH;
  g.n = t / g.tilesH;
  g.y0 = th * TH;
  g.x0 = tw * TW;
  return g;
}

// [rows][cols][CB] box of an NHWC tensor (row stride `cs` elements, channels
// c0..c0+31) at (n, y0, x0) into shared memory through cp.async (16-byte, zero
// fill via src-size 0 = the padding): the next tile's loads fly while the current
// one is computed
template <int ROWS, int COLS, typename T>
__device__ __forceinline__ void load_box_async(const T* __restrict__ src, int cs, int c0, int n, int H, int W,
                                               int y0, int x0, T* dst) {
  constexpr int VPP = CB * (int)sizeof(T) / 16;
  constexpr int EPV = 16 / (int)sizeof(T);
  constexpr int total = ROWS * COLS * VPP, cols = COLS;  // compile-time: the index splits are shifts / mul-hi
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int v = i % VPP, pix = i / VPP;
    const int yy = y0 + pix / cols, xx = x0 + pix % cols;
    const bool ok = yy >= 0 && yy < H && xx >= 0 && xx < W;
    const T* g = ok ? src + (((size_t)n * H + yy) * W + xx) * cs + c0 + v * EPV : src;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(
                     reinterpret_cast<uint4*>(dst) + i)),
                 "l"(g), "r"(ok ? 16 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// contiguous range of tiles of this CTA (persistent CTAs, blockIdx.x of gridDim.x)
__device__ __forceinline__ void tile_range(int ntiles, int& t0, int& t1) {
  t0 = (int)((long long)blockIdx.x * ntiles / gridDim.x);
  t1 = (int)((long long)(blockIdx.x + 1) * ntiles / gridDim.x);
}
}  // namespace

// ---- forward: y (and a, b) of 8 x 16 x 32 output tiles, two tiles in flight per CTA -------
template <typename T, int S, int FAM>
__global__ void __launch_bounds__(NT) dw_fwd_tile_kernel(DwArgs A, const T* __restrict__ x,
                                                         const float* __restrict__ Wp, const float* b0,
                                                         const float* b1, const float* b2, T* y, T* oa, T* ob,
                                                         int plain, int ntiles) {
  using F = DwF<FAM>;
  constexpr int R = 3, HR = (TH - 1) * S + R, HC = (TW - 1) * S + R, STG = HR * HC * CB;
  extern __shared__ __align__(16) uint8_t dsm[];
  T* sbuf = reinterpret_cast<T*>(dsm);  // two stages of STG
  const int c0 = blockIdx.y * CB;
  int t0, t1;
  tile_range(ntiles, t0, t1);
  auto issue = [&](int t, T* dst) {
    const TileGeo tg = tile_of(t, A.OH, A.OW);
    load_box_async<HR, HC>(x, A.C, c0, tg.n, A.H, A.W, tg.y0 * S - A.p, tg.x0 * S - A.p, dst);
  };
  if (t0 < t1) issue(t0, sbuf);
  cp_commit();
  const int cp = threadIdx.x % (CB / 2), col = threadIdx.x / (CB / 2), c = c0 + 2 * cp;
  float2 w[F::NR][R * R];
#pragma unroll
  for (int ro = 0; ro < F::NR; ++ro)
#pragma unroll
    for (int t = 0; t < R * R; ++t) w[ro][t] = __ldg(reinterpret_cast<const float2*>(Wp + (ro * R * R + t) * A.C + c));
  float2 bb[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  if (FAM == QD_FAM_FIRST_ORDER || FAM == QD_FAM_PROPOSED) {
    bb[0] = make_float2(b0[c], b0[c + 1]);
    if (FAM == QD_FAM_PROPOSED) {
      bb[1] = make_float2(b1[c], b1[c + 1]);
      bb[2] = make_float2(b2[c], b2[c + 1]);
    }
  }
  for (int t = t0, it = 0; t < t1; ++t, ++it) {
    if (t + 1 < t1) issue(t + 1, sbuf + ((it + 1) & 1) * STG);
    cp_commit();
    cp_wait1();
    __syncthreads();  // tile t staged by every thread
    const T* sx = sbuf + (it & 1) * STG;
    const TileGeo tg = tile_of(t, A.OH, A.OW);
    const int ow = tg.x0 + col;
    if (ow < A.OW) {
      // 3 x 3 input window in registers, slid down the column: each output row loads
      // only its S new input rows (rows past the image read the zero-filled halo)
      float2 win[R][R];
      const T* base = sx + (col * S) * CB + 2 * cp;
      T* yb = y + (((size_t)tg.n * A.OH + tg.y0) * A.OW + ow) * A.C + c;
      const size_t rs = (size_t)A.OW * A.C;
#pragma unroll
      for (int dy = 0; dy < R - S; ++dy)
#pragma unroll
        for (int dx = 0; dx < R; ++dx) win[dy + S][dx] = P2<T>::ld(base + (dy * HC + dx) * CB);
#pragma unroll
      for (int rl = 0; rl < TH; ++rl) {
#pragma unroll
        for (int dy = 0; dy < R; ++dy)
#pragma unroll
          for (int dx = 0; dx < R; ++dx) {
            if (dy < R - S)
              win[dy][dx] = win[dy + S][dx];
            else
              win[dy][dx] = P2<T>::ld(base + ((rl * S + dy) * HC + dx) * CB);
          }
        float2 acc[F::NR];
#pragma unroll
        for (int ro = 0; ro < F::NR; ++ro) acc[ro] = make_float2(0.f, 0.f);
#pragma unroll
        for (int dy = 0; dy < R; ++dy)
#pragma unroll
          for (int dx = 0; dx < R; ++dx) {
            const float2 v = win[dy][dx];
            const float2 v2 = F::SQ ? f2mul(v, v) : v;
#pragma unroll
            for (int ro = 0; ro < F::NR; ++ro)
              acc[ro] = f2fma(w[ro][dy * R + dx], (F::SQ >> ro) & 1 ? v2 : v, acc[ro]);
          }
        if (tg.y0 + rl >= A.OH) continue;
        const size_t o = rl * rs;
        if (plain) {
          P2<T>::st(yb + o, acc[0]);
          continue;
        }
        float2 out;
        if (FAM == QD_FAM_FIRST_ORDER) {
          out = f2add(acc[0], bb[0]);
        } else if (FAM == QD_FAM_T3) {
          out = f2mul(acc[0], acc[0]);
        } else if (FAM == QD_FAM_T4) {
          P2<T>::st(oa + (yb - y) + o, acc[0]);
          P2<T>::st(ob + (yb - y) + o, acc[F::NR - 1]);
          out = f2mul(acc[0], acc[F::NR - 1]);
        } else if (FAM == QD_FAM_PROPOSED) {
          const float2 av = f2add(acc[0], bb[0]), bv = f2add(acc[1 % F::NR], bb[1]);
          P2<T>::st(oa + (yb - y) + o, av);
          P2<T>::st(ob + (yb - y) + o, bv);
          out = f2add(f2mul(av, bv), f2add(acc[2 % F::NR], bb[2]));
        } else if (FAM == QD_FAM_T2_LINEAR) {
          out = f2add(acc[0], acc[1 % F::NR]);
        } else if (FAM == QD_FAM_T2AND4) {
          P2<T>::st(oa + (yb - y) + o, acc[0]);
          P2<T>::st(ob + (yb - y) + o, acc[1 % F::NR]);
          out = f2add(f2mul(acc[0], acc[1 % F::NR]), acc[2 % F::NR]);
        } else {
          out = acc[0];  // t2
        }
        P2<T>::st(yb + o, out);
      }
    }
    __syncthreads();  // stage it & 1 free for tile t + 2
  }
}

// ---- dgrad: dx of one 8 x 16 x 32 input tile per CTA --------------------------------
// dx[i] = sum_roles sum_taps D_din(ro)[o(i, tap)] W_ro[tap] (+ 2 x * the x*x roles'
// sum, neurons.py:400-405); o(i, tap) = (i + p - tap) / s where divisible
template <typename T, int S, int FAM>
__global__ void __launch_bounds__(NT) dw_dgrad_tile_kernel(DwArgs A, const T* __restrict__ x,
                                                           const T* __restrict__ D, const float* __restrict__ Wp,
                                                           T* dx, int ntiles) {
  using F = DwF<FAM>;
  constexpr int R = 3;
  // output rows / cols a tile of TH x TW inputs reaches: ((TH - 1) + R - 1) / S + 1 (+1 for flooring)
  constexpr int DR = (TH + R - 2) / S + 2, DC = (TW + R - 2) / S + 2;
  constexpr int ND = dw_nd<FAM>(), STG = ND * DR * DC * CB;
  extern __shared__ __align__(16) uint8_t dsm[];
  T* sbuf = reinterpret_cast<T*>(dsm);  // two stages of STG
  const int c0 = blockIdx.y * CB;
  int t0, t1;
  tile_range(ntiles, t0, t1);
  // first output row / col any input of the tile reaches (floor division)
  auto org = [&](int t, TileGeo& tg, int& oy0, int& ox0) {
    tg = tile_of(t, A.H, A.W);
    oy0 = (tg.y0 + A.p - (R - 1) + S * 64) / S - 64;
    ox0 = (tg.x0 + A.p - (R - 1) + S * 64) / S - 64;
  };
  auto issue = [&](int t, T* dst) {
    TileGeo tg;
    int oy0, ox0;
    org(t, tg, oy0, ox0);
    for (int k = 0; k < ND; ++k)
      load_box_async<DR, DC>(D, A.Jd, k * A.C + c0, tg.n, A.OH, A.OW, oy0, ox0, dst + k * DR * DC * CB);
  };
  if (t0 < t1) issue(t0, sbuf);
  cp_commit();
  const int cp = threadIdx.x % (CB / 2), col = threadIdx.x / (CB / 2), c = c0 + 2 * cp;
  float2 w[F::NR][R * R];
#pragma unroll
  for (int ro = 0; ro < F::NR; ++ro)
#pragma unroll
    for (int t = 0; t < R * R; ++t) w[ro][t] = __ldg(reinterpret_cast<const float2*>(Wp + (ro * R * R + t) * A.C + c));
  for (int t = t0, it = 0; t < t1; ++t, ++it) {
    if (t + 1 < t1) issue(t + 1, sbuf + ((it + 1) & 1) * STG);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const T* sd = sbuf + (it & 1) * STG;
    TileGeo tg;
    int oy0, ox0;
    org(t, tg, oy0, ox0);
    const int iw = tg.x0 + col;
    if (iw < A.W) {
      if constexpr (S == 1) {
        // input (rl, col) reads halo rows rl..rl+2, cols col..col+2 (tap (2 - j, 2 - k)):
        // a 3 x 3 window per D block slid down the column, one new halo row per input row
        float2 win[ND][R][R];
        const T* base = sd + col * CB + 2 * cp;
#pragma unroll
        for (int k = 0; k < ND; ++k)
#pragma unroll
          for (int j = 0; j < R - 1; ++j)
#pragma unroll
            for (int kk = 0; kk < R; ++kk) win[k][j + 1][kk] = P2<T>::ld(base + (k * DR * DC + j * DC + kk) * CB);
        T* db = dx + (((size_t)tg.n * A.H + tg.y0) * A.W + iw) * A.C + c;
        const T* xb = x + (db - dx);
        const size_t rs = (size_t)A.W * A.C;
#pragma unroll
        for (int rl = 0; rl < TH; ++rl) {
#pragma unroll
          for (int k = 0; k < ND; ++k)
#pragma unroll
            for (int j = 0; j < R; ++j)
#pragma unroll
              for (int kk = 0; kk < R; ++kk) {
                if (j < R - 1)
                  win[k][j][kk] = win[k][j + 1][kk];
                else
                  win[k][j][kk] = P2<T>::ld(base + (k * DR * DC + (rl + j) * DC + kk) * CB);
              }
          float2 lin = make_float2(0.f, 0.f), sq = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < R; ++j)
#pragma unroll
            for (int kk = 0; kk < R; ++kk)
#pragma unroll
              for (int ro = 0; ro < F::NR; ++ro) {
                const int k = ro == 0 ? 0 : (ro == 1 ? F::D1 : F::D2);
                const float2 wt = w[ro][(R - 1 - j) * R + (R - 1 - kk)];
                if ((F::SQ >> ro) & 1)
                  sq = f2fma(win[k][j][kk], wt, sq);
                else
                  lin = f2fma(win[k][j][kk], wt, lin);
              }
          if (tg.y0 + rl >= A.H) continue;
          if (F::SQ) {
            const float2 xv = P2<T>::ld(xb + rl * rs), t2 = f2mul(sq, xv);
            lin = f2add(lin, f2add(t2, t2));
          }
          P2<T>::st(db + rl * rs, lin);
        }
      } else {
        for (int rl = 0; rl < TH; ++rl) {
          const int ih = tg.y0 + rl;
          if (ih >= A.H) break;
          float2 lin = make_float2(0.f, 0.f), sq = make_float2(0.f, 0.f);
#pragma unroll
          for (int dy = 0; dy < R; ++dy) {
            const int th = ih + A.p - dy;
            if (th & 1) continue;
            const int oyl = (th + S * 64) / S - 64 - oy0;
#pragma unroll
            for (int dxx = 0; dxx < R; ++dxx) {
              const int tw = iw + A.p - dxx;
              if (tw & 1) continue;
              const int oxl = (tw + S * 64) / S - 64 - ox0;
              const int pix = oyl * DC + oxl;
#pragma unroll
              for (int ro = 0; ro < F::NR; ++ro) {
                const int k = ro == 0 ? 0 : (ro == 1 ? F::D1 : F::D2);
                const float2 d = P2<T>::ld(sd + (k * DR * DC + pix) * CB + 2 * cp);
                if ((F::SQ >> ro) & 1)
                  sq = f2fma(d, w[ro][dy * R + dxx], sq);
                else
                  lin = f2fma(d, w[ro][dy * R + dxx], lin);
              }
            }
          }
          const size_t i = (((size_t)tg.n * A.H + ih) * A.W + iw) * A.C + c;
          if (F::SQ) {
            const float2 xv = P2<T>::ld(x + i), t2 = f2mul(sq, xv);
            lin = f2add(lin, f2add(t2, t2));
          }
          P2<T>::st(dx + i, lin);
        }
      }
    }
    __syncthreads();
  }
}

// ---- wgrad: per (role, tap, channel) sums over the CTA's range of output tiles ------
// thread = (channel pair cp, tile column pg of 16): pg walks the column's TH rows;
// the 16 columns fold in a fixed order (xor-16 shuffle within the warp, then the
// 8 warps through shared memory)
template <typename T, int S, int FAM>
__global__ void __launch_bounds__(NT) dw_wgrad_tile_kernel(DwArgs A, const T* __restrict__ x,
                                                           const T* __restrict__ D, float* part, int ntiles) {
  using F = DwF<FAM>;
  constexpr int R = 3, HR = (TH - 1) * S + R, HC = (TW - 1) * S + R;
  constexpr int ND = dw_nd<FAM>();
  constexpr int XS = HR * HC * CB, STG = XS + ND * TH * TW * CB;
  extern __shared__ __align__(16) uint8_t dsm[];  // two stages of (x halo, D tile), then the fold
  T* sbuf = reinterpret_cast<T*>(dsm);
  const int c0 = blockIdx.y * CB;
  const int cp = threadIdx.x % (CB / 2), pg = threadIdx.x / (CB / 2);
  float2 acc[F::NR][R * R];
#pragma unroll
  for (int ro = 0; ro < F::NR; ++ro)
#pragma unroll
    for (int t = 0; t < R * R; ++t) acc[ro][t] = make_float2(0.f, 0.f);
  int t0, t1;
  tile_range(ntiles, t0, t1);
  auto issue = [&](int t, T* dst) {
    const TileGeo tg = tile_of(t, A.OH, A.OW);
    load_box_async<HR, HC>(x, A.C, c0, tg.n, A.H, A.W, tg.y0 * S - A.p, tg.x0 * S - A.p, dst);
    for (int k = 0; k < ND; ++k)
      load_box_async<TH, TW>(D, A.Jd, k * A.C + c0, tg.n, A.OH, A.OW, tg.y0, tg.x0, dst + XS + k * TH * TW * CB);
  };
  if (t0 < t1) issue(t0, sbuf);
  cp_commit();
  for (int t = t0, it = 0; t < t1; ++t, ++it) {
    if (t + 1 < t1) issue(t + 1, sbuf + ((it + 1) & 1) * STG);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const T* sx = sbuf + (it & 1) * STG;
    const T* sd = sx + XS;
    // thread column pg walks the tile's TH rows with a 3 x 3 x window slid down
    // (S new rows per output row); pixels outside the image have D = 0 (zero
    // filled), so no bounds checks are needed
    float2 win[R][R];
    const T* xb = sx + (pg * S) * CB + 2 * cp;
#pragma unroll
    for (int dy = 0; dy < R - S; ++dy)
#pragma unroll
      for (int dxx = 0; dxx < R; ++dxx) win[dy + S][dxx] = P2<T>::ld(xb + (dy * HC + dxx) * CB);
#pragma unroll
    for (int rl = 0; rl < TH; ++rl) {
#pragma unroll
      for (int dy = 0; dy < R; ++dy)
#pragma unroll
        for (int dxx = 0; dxx < R; ++dxx) {
          if (dy < R - S)
            win[dy][dxx] = win[dy + S][dxx];
          else
            win[dy][dxx] = P2<T>::ld(xb + ((rl * S + dy) * HC + dxx) * CB);
        }
      float2 d[F::NR];
#pragma unroll
      for (int ro = 0; ro < F::NR; ++ro) {
        const int k = ro == 0 ? 0 : (ro == 1 ? F::D1 : F::D2);
        d[ro] = P2<T>::ld(sd + (k * TH * TW + rl * TW + pg) * CB + 2 * cp);
      }
#pragma unroll
      for (int dy = 0; dy < R; ++dy)
#pragma unroll
        for (int dxx = 0; dxx < R; ++dxx) {
          const float2 v = win[dy][dxx];
          const float2 v2 = F::SQ ? f2mul(v, v) : v;
#pragma unroll
          for (int ro = 0; ro < F::NR; ++ro)
            acc[ro][dy * R + dxx] = f2fma(d[ro], (F::SQ >> ro) & 1 ? v2 : v, acc[ro][dy * R + dxx]);
        }
    }
    __syncthreads();  // stage it & 1 free for tile t + 2
  }
  // fold the 16 pixel groups: xor-16 lanes (groups 2w, 2w + 1 of warp w), then warps in order
#pragma unroll
  for (int ro = 0; ro < F::NR; ++ro)
#pragma unroll
    for (int t = 0; t < R * R; ++t) {
      float2& a = acc[ro][t];
      const float ox = __shfl_xor_sync(0xffffffffu, a.x, 16), oy = __shfl_xor_sync(0xffffffffu, a.y, 16);
      a = (threadIdx.x & 16) ? f2add(make_float2(ox, oy), a) : f2add(a, make_float2(ox, oy));
    }
  __syncthreads();  // tiles no longer read: the buffer takes the fold
  float2* red = reinterpret_cast<float2*>(dsm);  // [warp][ro * 9 + t][cp]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane < 16)
#pragma unroll
    for (int ro = 0; ro < F::NR; ++ro)
#pragma unroll
      for (int t = 0; t < R * R; ++t) red[(warp * F::NR * R * R + ro * R * R + t) * (CB / 2) + cp] = acc[ro][t];
  __syncthreads();
  const int nout = F::NR * R * R * (CB / 2);
  float* o = part + (size_t)blockIdx.x * F::NR * R * R * A.C;
  for (int j = threadIdx.x; j < nout; j += NT) {
    float2 s = red[j];
    for (int w8 = 1; w8 < NT / 32; ++w8) s = f2add(s, red[w8 * nout + j]);
    const int rt = j / (CB / 2), q = j % (CB / 2);  // rt = ro * 9 + tap
    // part[s][ro][tap][c], the layout dw_wgrad_finish folds
    o[(size_t)rt * A.C + c0 + 2 * q] = s.x;
    o[(size_t)rt * A.C + c0 + 2 * q + 1] = s.y;
  }
}

// ---- host ---------------------------------------------------------------------------
bool dw_tile_ok(const Plan& P) {
  if (getenv("QD_DW_DIRECT")) return false;  // dev A/B: the direct kernels of qd_dw.cu
  // fp32 at stride 2: two wgrad stages (x halo + D tile) exceed shared memory
  return P.r == 3 && (P.s == 1 || (P.s == 2 && P.dtype == QD_BF16)) && P.C % CB == 0 && P.p >= 0 && P.p <= 2 &&
         P.Min * P.C < (1LL << 31) && P.Mout * P.C < (1LL << 31);
}

static long long dw_tiles(const Plan& P, bool input_space) {
  const int h = input_space ? P.H : P.OH, w = input_space ? P.W : P.OW;
  return (long long)P.N * ((h + TH - 1) / TH) * ((w + TW - 1) / TW);
}

int dw_tile_wgrad_split(const Plan& P) {
  const long long nt = dw_tiles(P, false), cbs = P.C / CB;
  long long s = (2LL * tc_num_sms() + cbs - 1) / cbs;
  if (s > nt) s = nt;
  return (int)(s < 1 ? 1 : s);
}

#define QD_DW_FAMS(X) X(QD_FAM_FIRST_ORDER) X(QD_FAM_T2) X(QD_FAM_T3) X(QD_FAM_T4) X(QD_FAM_PROPOSED) \
  X(QD_FAM_T2_LINEAR) X(QD_FAM_T2AND4)

// persistent CTAs per channel block: ~2 resident per SM over all channel blocks
static int dw_ctas(const Plan& P, long long tiles) {
  const long long cbs = P.C / CB;
  long long n = (2LL * tc_num_sms() + cbs - 1) / cbs;
  if (n > tiles) n = tiles;
  return (int)(n < 1 ? 1 : n);
}

template <typename T, int S>
static void fwd_s(const Plan& P, const DwArgs& A, const T* x, const float* Wp, const float* const bias[3], T* y,
                  T* a, T* b, int plain, cudaStream_t st) {
  const int nt = (int)dw_tiles(P, false);
  const dim3 grid((unsigned)dw_ctas(P, nt), (unsigned)(P.C / CB));
  switch (P.family) {
#define X(f)                                                                                         \
  case f:                                                                                            \
    raise_smem_attr((const void*)dw_fwd_tile_kernel<T, S, f>, fwd_smem<T, S>());                      \
    dw_fwd_tile_kernel<T, S, f><<<grid, NT, fwd_smem<T, S>(), st>>>(A, x, Wp, bias[0], bias[1], bias[2], y, a, b, \
                                                                   plain, nt);                         \
    break;
    QD_DW_FAMS(X)
#undef X
    default: break;
  }
}

template <typename T>
int dw_tile_forward(const Plan& P, const DwArgs& A, const T* x, const float* Wp, const float* const bias[3], T* y,
                    T* a, T* b, int plain, cudaStream_t st) {
  if (P.s == 1)
    fwd_s<T, 1>(P, A, x, Wp, bias, y, a, b, plain, st);
  else
    fwd_s<T, 2>(P, A, x, Wp, bias, y, a, b, plain, st);
  count_launch(st, plain ? "dw_fwd_plain" : "dw_fwd");
  return check_launch("dwconv forward (tiled)");
}

template <typename T, int S>
static void bwd_s(const Plan& P, const DwArgs& A, const T* x, const T* D, const float* Wp, T* dx, float* part,
                  int split, cudaStream_t st) {
  const int nt = (int)dw_tiles(P, false), ntin = (int)dw_tiles(P, true);
  const dim3 gw((unsigned)split, (unsigned)(P.C / CB)), gd((unsigned)dw_ctas(P, ntin), (unsigned)(P.C / CB));
  switch (P.family) {
#define X(f)                                                                                \
  case f:                                                                                   \
    if (part) {                                                                             \
      constexpr int sm = wgrad_smem<T, S>(dw_nd<f>(), DwF<f>::NR);                          \
      raise_smem_attr((const void*)dw_wgrad_tile_kernel<T, S, f>, sm);                      \
      dw_wgrad_tile_kernel<T, S, f><<<gw, NT, sm, st>>>(A, x, D, part, nt);                 \
      count_launch(st, "dw_wgrad");                                                         \
    }                                                                                       \
    if (dx) {                                                                               \
      constexpr int sm = dgrad_smem<T, S>(dw_nd<f>());                                      \
      raise_smem_attr((const void*)dw_dgrad_tile_kernel<T, S, f>, sm);                      \
      dw_dgrad_tile_kernel<T, S, f><<<gd, NT, sm, st>>>(A, x, D, Wp, dx, ntin);             \
      count_launch(st, "dw_dgrad");                                                         \
    }                                                                                       \
    break;
    QD_DW_FAMS(X)
#undef X
    default: break;
  }
}

template <typename T>
int dw_tile_backward(const Plan& P, const DwArgs& A, const T* x, const T* D, const float* Wp, T* dx, float* part,
                     int split, cudaStream_t st) {
  if (P.s == 1)
    bwd_s<T, 1>(P, A, x, D, Wp, dx, part, split, st);
  else
    bwd_s<T, 2>(P, A, x, D, Wp, dx, part, split, st);
  return check_launch("dwconv backward (tiled)");
}

template int dw_tile_forward<bf16>(const Plan&, const DwArgs&, const bf16*, const float*, const float* const[3],
                                   bf16*, bf16*, bf16*, int, cudaStream_t);
template int dw_tile_forward<float>(const Plan&, const DwArgs&, const float*, const float*, const float* const[3],
                                    float*, float*, float*, int, cudaStream_t);
template int dw_tile_backward<bf16>(const Plan&, const DwArgs&, const bf16*, const bf16*, const float*, bf16*,
                                    float*, int, cudaStream_t);
template int dw_tile_backward<float>(const Plan&, const DwArgs&, const float*, const float*, const float*, float*,
                                     float*, int, cudaStream_t);

}  // namespace qd
