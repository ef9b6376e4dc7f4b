// tcgen05 / TMEM / TMA kernels for the quadratic conv (and fc as a 1x1 conv
// over an N x 1 x 1 grid), bf16 operands, fp32 accumulation in TMEM.
//
//  K1  conv_gemm<EPI_PROPOSED|EPI_T4|EPI_PLAIN>  fprop: one implicit GEMM over
//      the branch-interleaved [Wa;Wb;Wc] weights; A tiles are 4-D TMA boxes of
//      the NHWC activations shifted per filter tap (OOB zero fill = padding);
//      the a*b + c + bias epilogue runs on the TMEM accumulator in registers
//      and the y / a / b tiles leave through TMA stores. The raw Wa.x, Wb.x,
//      Wc.x and a*b never reach HBM (neurons.py:268-274).
//  K3  conv_gemm<EPI_PLAIN|EPI_SQ>  stride-1 dgrad: the same kernel run as a
//      conv of D = [dy*b | dy*a | dy] with the flipped packed weights, so
//      dX = Wa^T(dy*b) + Wb^T(dy*a) + Wc^T dy is ONE GEMM with K = r*r*3F
//      (neurons.py:433-444); t2's "t = ds*x; dx = t + t" (:400-405) is the
//      EPI_SQ epilogue.
//  K4  wgrad: dW^T tiles = im2col(x)^T . D with both operands MN-major
//      straight from TMA boxes, split over pixels into fp32 partials that a
//      fixed-order reduce folds into the reference layouts (deterministic).
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (one lane),
// w2 TMEM allocator, w4-7 epilogue (TMEM lane quarter = warp % 4).
// Persistent over output tiles, TMEM accumulators double-buffered so the
// epilogue of tile i overlaps the main loop of tile i+1.
#include <cudaTypedefs.h>
#include <stdio.h>
#include <string.h>
#include "qd_kernels.h"
#include "qd_ptx.cuh"

namespace qd {

enum { EPI_PROPOSED = 0, EPI_T4 = 1, EPI_PLAIN = 2, EPI_SQ = 3 };

struct ConvArgs {
  int tiles_w, tiles_h, tiles_nn, total_tiles;
  int Wb, Hb, Nb, box_rows;
  int OHg, OWg, Ng;         // output grid (epilogue validity)
  int r, pad_eff, cblks;    // taps, shift, 64-channel blocks of the A tensor
  int kb_half, dual;        // k-blocks per A map; dual = second half from map A1 (t2_linear)
  int b_rs_tile, b_rs_blk;  // B row offset per N tile / per 64-row block
  int out_c_tile;           // output channel offset per N tile
  int Cout;                 // channels of the output tensor (and of x for EPI_SQ)
  const float* bias0;
  const float* bias1;
  const float* bias2;
  const bf16* xres;         // x (NHWC) for EPI_SQ
  // split-K (small output grids): work item = (tile, K slice); the epilogue then
  // writes fp32 partials [ksplit][Mpix][part_ld] and splitk_finish applies EPI
  int ksplit, kb_per, part_ld;
  long long Mpix;
  float* part;
  // stride 2 without the stride-1 grid: the fprop's A map walks x with traversal
  // stride `sstride` (box origin sstride * output + tap - pad); the dgrad runs as
  // four output-parity classes (cls = 1): class (ph, pw) is a stride-1 conv of D
  // over the taps with ey = ph + pad_eff (mod 2) (resp. ex), D row offset
  // (ph + ey - pad_eff) / 2, written to dx pixels (2h + ph, 2w + pw)
  int sstride;
  int cls, cls_tiles;       // class mode; tiles per class (all classes share the grid)
  int cls_code[4];          // per class in work order: ph | pw << 1 | k-blocks << 2
  int Hx, Wx;               // dx extent (class mode)
  bf16* out;                // dx, direct row stores (class mode)
};

// work item -> (tile, K slice, parity class, k-block range)
struct ConvWork { int t, ks, ph, pw, kb0, kb1; };
__device__ __forceinline__ ConvWork conv_work(const ConvArgs& a, int wi, int KB) {
  ConvWork w;
  if (a.cls) {
    const int ci = wi / a.cls_tiles;
    int code = a.cls_code[0];
#pragma unroll
    for (int i = 1; i < 4; ++i)  // static indexing: no local copy of the array
      if (i == ci) code = a.cls_code[i];
    w.t = wi - ci * a.cls_tiles; w.ks = 0;
    w.ph = code & 1; w.pw = (code >> 1) & 1;
    w.kb0 = 0; w.kb1 = code >> 2;
    return w;
  }
  w.t = wi / a.ksplit; w.ks = wi - w.t * a.ksplit;
  w.ph = w.pw = 0;
  w.kb0 = w.ks * a.kb_per; w.kb1 = min(KB, w.kb0 + a.kb_per);
  return w;
}

// PAIR: the CTA-pair form (cta_group::2, M = 256 over two SMs), each CTA holding
// its own A tile but only half of B (NB x 32 rows)
template <int EPI, int NB, int PAIR = 0>
struct ConvCfg {
  static constexpr int A_BYTES = 128 * 128;
  static constexpr int B_BYTES = NB * 64 * 128 / (PAIR ? 2 : 1);
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int NOUT = (EPI == EPI_PROPOSED || EPI == EPI_T4) ? 3 : (EPI == EPI_PLAIN ? NB : 1);
  static constexpr int STG = NOUT * 128 * 128;
  static constexpr int BUDGET = 220 * 1024;
  static constexpr int S0 = (BUDGET - STG - 1024) / STAGE;
  static constexpr int STAGES = S0 > 6 ? 6 : S0;
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE + STG + 1024 /*barriers*/;
  static constexpr int ACC_COLS = NB * 64;
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// write 16 fp32 values (channels 16j..16j+15 of a 64-channel row) as bf16 into a
// SWIZZLE_128B staging tile: 16-B chunk q of row `row` lives at chunk q ^ (row & 7)
__device__ __forceinline__ void stage_store16(uint8_t* tile, int row, int j, const float* v) {
  uint4 lo, hi;
  lo.x = pack_bf16x2(v[0], v[1]);   lo.y = pack_bf16x2(v[2], v[3]);
  lo.z = pack_bf16x2(v[4], v[5]);   lo.w = pack_bf16x2(v[6], v[7]);
  hi.x = pack_bf16x2(v[8], v[9]);   hi.y = pack_bf16x2(v[10], v[11]);
  hi.z = pack_bf16x2(v[12], v[13]); hi.w = pack_bf16x2(v[14], v[15]);
  uint8_t* rowp = tile + row * 128;
  int q0 = 2 * j, q1 = 2 * j + 1;
  *reinterpret_cast<uint4*>(rowp + ((q0 ^ (row & 7)) << 4)) = lo;
  *reinterpret_cast<uint4*>(rowp + ((q1 ^ (row & 7)) << 4)) = hi;
}

template <int EPI, int NB, int PAIR = 0>
__global__ void __launch_bounds__(256, 1)
    conv_gemm_kernel(const __grid_constant__ CUtensorMap mapA0, const __grid_constant__ CUtensorMap mapA1,
                     const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapO0,
                     const __grid_constant__ CUtensorMap mapO1, const __grid_constant__ CUtensorMap mapO2,
                     const ConvArgs args) {
  using Cfg = ConvCfg<EPI, NB, PAIR>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint8_t* sOut = sB + STAGES * Cfg::B_BYTES;
  uint64_t* full = (uint64_t*)(sOut + Cfg::STG);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // PAIR: CTA r of a cluster takes M tile 2 m + r of the pair's work item; every
  // stage completes on CTA0's full barrier, the MMA (CTA0) commits to both CTAs
  const uint32_t rank = PAIR ? ptx::cluster_rank() : 0;
  const int wstart = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int wstep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  auto tile_of = [&](int t, int& ntile, int& w0, int& h0, int& n0) {
    ntile = t % args.tiles_nn;
    const int mt = PAIR ? 2 * (t / args.tiles_nn) + (int)rank : t / args.tiles_nn;
    const int tw = mt % args.tiles_w, th = (mt / args.tiles_w) % args.tiles_h;
    const int tn = mt / (args.tiles_w * args.tiles_h);  // >= tiles_n: an empty tile (all OOB)
    w0 = tw * args.Wb; h0 = th * args.Hb; n0 = tn * args.Nb;
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&mapA0);
    ptx::prefetch_tmap(&mapA1);
    ptx::prefetch_tmap(&mapB);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], PAIR ? 8 : 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    if (PAIR) {
      ptx::tmem_alloc2(tmem_slot, 512);
    } else {
      ptx::tmem_alloc(tmem_slot, 512);
      ptx::tmem_relinquish();
    }
  }
  ptx::tc_fence_before();
  if (PAIR) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // dual = extra K segments: 1 = [x*x | x] (t2_linear; segment 1 from A1), 2 = the
  // fp32 split [hi | hi | lo] (qd_x3.cu; segment 2 from A1)
  const int KB = args.kb_half * (1 + args.dual);
  const int NWORK = args.cls ? 4 * args.cls_tiles : args.total_tiles * args.ksplit;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t bytes = (uint32_t)(args.box_rows * 128 + Cfg::B_BYTES) * (PAIR ? 2 : 1);
      const int ss = args.sstride;
      for (int wi = wstart; wi < NWORK; wi += wstep) {
        const ConvWork cw = conv_work(args, wi, KB);
        const int t = cw.t;
        int ntile, w0, h0, n0;
        tile_of(t, ntile, w0, h0, n0);
        // class mode: first tap of the class's parity and its tap count along x
        const int ey0 = (args.pad_eff - cw.ph) & 1, ex0 = (args.pad_eff - cw.pw) & 1;
        const int ntx = (args.r - ex0 + 1) >> 1;
        // k-block -> (K half, tap, channel block) walked incrementally: the divisions
        // run once per work item, not per k-block (the single producer thread issues
        // 1 + NB boxes per ~400 MMA cycles and was the limiter with them, ncu)
        int half = cw.kb0 / args.kb_half, kk0 = cw.kb0 - half * args.kb_half;
        int tap = kk0 / args.cblks, cb = kk0 - tap * args.cblks;
        int ty = args.cls ? tap / ntx : tap / args.r;  // class: tap row in the class; else ey
        int tx = args.cls ? tap - ty * ntx : tap - ty * args.r;
        int kk = kk0;
        int brow[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const int j0 = (int)rank * NB * 32 + i * 32;
          brow[i] = PAIR ? ntile * args.b_rs_tile + (j0 / 64) * args.b_rs_blk + j0 % 64
                         : ntile * args.b_rs_tile + i * args.b_rs_blk;
        }
        for (int kb = cw.kb0; kb < cw.kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], bytes);
          int ax, ay, bk = kb;
          if (args.cls) {
            const int ey = ey0 + 2 * ty, ex = ex0 + 2 * tx;
            ay = h0 + ((cw.ph + ey - args.pad_eff) >> 1);  // even numerator: exact
            ax = w0 + ((cw.pw + ex - args.pad_eff) >> 1);
            bk = (ey * args.r + ex) * args.cblks + cb;
          } else {
            ax = ss * w0 + tx - args.pad_eff;
            ay = ss * h0 + ty - args.pad_eff;
          }
          const CUtensorMap* ma = (half > 0 && half == args.dual) ? &mapA1 : &mapA0;
          if (PAIR) {
            // this CTA's half of the B tile: rows j in [rank NB 32, (rank + 1) NB 32) as 32-row boxes
            const uint32_t fb = ptx::peer0(&full[stage]);
            ptx::tma4_cg2(ma, fb, sA + stage * Cfg::A_BYTES, cb * 64, ax, ay, n0);
#pragma unroll
            for (int i = 0; i < NB; ++i)
              ptx::tma2_cg2(&mapB, fb, sB + stage * Cfg::B_BYTES + i * 4096, bk * 64, brow[i]);
          } else {
            ptx::tma_load_4d(ma, &full[stage], sA + stage * Cfg::A_BYTES, cb * 64, ax, ay, n0);
#pragma unroll
            for (int i = 0; i < NB; ++i)
              ptx::tma_load_2d(&mapB, &full[stage], sB + stage * Cfg::B_BYTES + i * 8192, bk * 64, brow[i]);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          // next k-block: channel block, then tap (x, then y), then K half
          if (++cb == args.cblks) {
            cb = 0;
            if (++tx == (args.cls ? ntx : args.r)) { tx = 0; ++ty; }
          }
          if (++kk == args.kb_half) { kk = 0; ++half; ty = 0; tx = 0; cb = 0; }
        }
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ===== MMA issuer: warp-wide loop (uniform datapath), one elected lane issues =====
    constexpr uint32_t IDESC = ptx::idesc_bf16(PAIR ? 256 : 128, NB * 64, false, false);
    constexpr uint32_t DHI = ptx::sw128_desc_hi(1024);
    const bool leader = ptx::elect_one();
    const uint32_t a_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sA), 16);
    const uint32_t b_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sB), 16);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int wi = wstart; wi < NWORK; wi += wstep, ++it) {
      const ConvWork cw = conv_work(args, wi, KB);
      const int kb0 = cw.kb0, kb1 = cw.kb1;
      int as = it & 1;
      uint32_t aph = (it >> 1) & 1;
      ptx::mbar_wait(&tempty[as], aph ^ 1);
      ptx::tc_fence_after();
      uint32_t d_tmem = tmem_base + as * Cfg::ACC_COLS;
      for (int kb = kb0; kb < kb1; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a_lo = a_lo0 + stage * (Cfg::A_BYTES >> 4);
        const uint32_t b_lo = b_lo0 + stage * (Cfg::B_BYTES >> 4);
        if (leader) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (PAIR)
              ptx::mma_cg2(d_tmem, ptx::mk_desc(DHI, a_lo + 2 * k), ptx::mk_desc(DHI, b_lo + 2 * k), IDESC,
                           ((kb != kb0) || (k != 0)) ? 1u : 0u);
            else
              ptx::mma_bf16(d_tmem, ptx::mk_desc(DHI, a_lo + 2 * k), ptx::mk_desc(DHI, b_lo + 2 * k), IDESC,
                            (kb != kb0) || (k != 0));
          }
          if (PAIR) ptx::commit_mc(&empty[stage]);
          else ptx::mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (leader) {
        if (PAIR) ptx::commit_mc(&tfull[as]);
        else ptx::mma_commit(&tfull[as]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===== epilogue =====
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int etid = threadIdx.x - 128;
    // TMEM hand-back: PAIR -> CTA0's barrier (count 8: both CTAs' epilogue warps)
    const uint32_t tempty0 = PAIR ? ptx::peer0(&tempty[0]) : 0u;
    auto hand_back = [&](int as_) {
      if (PAIR) ptx::arrive_remote(tempty0 + as_ * 8);
      else ptx::mbar_arrive(&tempty[as_]);
    };
    int it = 0;
    for (int wi = wstart; wi < NWORK; wi += wstep, ++it) {
      const ConvWork cw = conv_work(args, wi, KB);
      const int t = cw.t, ks = cw.ks;
      int ntile, w0, h0, n0;
      tile_of(t, ntile, w0, h0, n0);
      int as = it & 1;
      uint32_t aph = (it >> 1) & 1;
      if (EPI == EPI_PLAIN && args.cls) {
        // parity class (ph, pw): each row is one dx pixel (2h + ph, 2w + pw), its
        // NB x 64 channels stored straight from registers (full 128-B lines)
        ptx::mbar_wait(&tfull[as], aph);
        ptx::tc_fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + as * Cfg::ACC_COLS;
        const int ww = row % args.Wb, hh = (row / args.Wb) % args.Hb, nn = row / (args.Wb * args.Hb);
        const int n = n0 + nn, h = h0 + hh, w = w0 + ww;
        const int ih = 2 * h + cw.ph, iw = 2 * w + cw.pw;
        const bool ok = row < args.box_rows && n < args.Ng && h < args.OHg && w < args.OWg && ih < args.Hx &&
                        iw < args.Wx;
        const bool zero = cw.kb1 == cw.kb0;  // a class no tap reaches (r = 1): dx = 0 there
        bf16* orow = args.out + (((size_t)n * args.Hx + ih) * args.Wx + iw) * args.Cout + ntile * args.out_c_tile;
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          float v[NB][16];
#pragma unroll
          for (int i = 0; i < NB; ++i) ptx::tmem_ld16(tb + i * 64 + j * 16, v[i]);
          ptx::tmem_wait_ld();
          if (zero) {
#pragma unroll
            for (int i = 0; i < NB; ++i)
#pragma unroll
              for (int e = 0; e < 16; ++e) v[i][e] = 0.f;
          }
          if (ok) {
#pragma unroll
            for (int i = 0; i < NB; ++i) {
              uint4 lo, hi;
              lo.x = pack_bf16x2(v[i][0], v[i][1]);   lo.y = pack_bf16x2(v[i][2], v[i][3]);
              lo.z = pack_bf16x2(v[i][4], v[i][5]);   lo.w = pack_bf16x2(v[i][6], v[i][7]);
              hi.x = pack_bf16x2(v[i][8], v[i][9]);   hi.y = pack_bf16x2(v[i][10], v[i][11]);
              hi.z = pack_bf16x2(v[i][12], v[i][13]); hi.w = pack_bf16x2(v[i][14], v[i][15]);
              uint4* op = reinterpret_cast<uint4*>(orow + i * 64 + j * 16);
              op[0] = lo;
              op[1] = hi;
            }
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) hand_back(as);
        continue;
      }
      if (args.part) {
        // split-K slice: raw fp32 accumulator rows into the partial buffer
        ptx::mbar_wait(&tfull[as], aph);
        ptx::tc_fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + as * Cfg::ACC_COLS;
        const int ww = row % args.Wb, hh = (row / args.Wb) % args.Hb, nn = row / (args.Wb * args.Hb);
        const int n = n0 + nn, h = h0 + hh, w = w0 + ww;
        const bool ok = row < args.box_rows && n < args.Ng && h < args.OHg && w < args.OWg;
        float* prow = args.part + ((size_t)ks * args.Mpix + ((size_t)n * args.OHg + h) * args.OWg + w) * args.part_ld +
                      (size_t)ntile * NB * 64;
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          float v[NB][16];
#pragma unroll
          for (int i = 0; i < NB; ++i) ptx::tmem_ld16(tb + i * 64 + j * 16, v[i]);
          ptx::tmem_wait_ld();
          if (ok) {
#pragma unroll
            for (int i = 0; i < NB; ++i)
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                *reinterpret_cast<float4*>(prow + i * 64 + j * 16 + e) =
                    make_float4(v[i][e], v[i][e + 1], v[i][e + 2], v[i][e + 3]);
          }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) hand_back(as);
        continue;
      }
      // previous tile's TMA stores must have finished reading the staging tiles
      if (etid == 0) ptx::bulk_wait_read0();
      ptx::named_bar_sync(1, 128);
      ptx::mbar_wait(&tfull[as], aph);
      ptx::tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + as * Cfg::ACC_COLS;
      const int c_base = ntile * args.out_c_tile;
      // pixel of this row (for EPI_SQ's x operand)
      bool valid = false;
      size_t pix = 0;
      if (EPI == EPI_SQ) {
        int ww = row % args.Wb, hh = (row / args.Wb) % args.Hb, nn = row / (args.Wb * args.Hb);
        int n = n0 + nn, h = h0 + hh, w = w0 + ww;
        valid = row < args.box_rows && n < args.Ng && h < args.OHg && w < args.OWg;
        pix = ((size_t)n * args.OHg + h) * args.OWg + w;
      }
#pragma unroll 1
      for (int j = 0; j < 4; ++j) {
        float v[NB][16];
#pragma unroll
        for (int i = 0; i < NB; ++i) ptx::tmem_ld16(tbase + i * 64 + j * 16, v[i]);
        ptx::tmem_wait_ld();
        if (EPI == EPI_PROPOSED || EPI == EPI_T4) {
          float y[16], a[16], b[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            int c = c_base + j * 16 + e;
            if (EPI == EPI_PROPOSED) {
              a[e] = v[0][e] + __ldg(args.bias0 + c);
              b[e] = v[1][e] + __ldg(args.bias1 + c);
              y[e] = fmaf(a[e], b[e], v[2 % NB][e] + __ldg(args.bias2 + c));
            } else {
              a[e] = v[0][e];
              b[e] = v[1 % NB][e];
              y[e] = a[e] * b[e];
            }
          }
          stage_store16(sOut, row, j, y);
          stage_store16(sOut + 16384, row, j, a);
          stage_store16(sOut + 32768, row, j, b);
        } else if (EPI == EPI_PLAIN) {
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            if (args.bias0) {
#pragma unroll
              for (int e = 0; e < 16; ++e) v[i][e] += __ldg(args.bias0 + c_base + i * 64 + j * 16 + e);
            }
            stage_store16(sOut + i * 16384, row, j, v[i]);
          }
        } else {  // EPI_SQ: dx = 2 x acc0 (+ acc1)
          float o[16];
          float xv[16];
          if (valid) {
            const uint4* xp = reinterpret_cast<const uint4*>(args.xres + pix * args.Cout + c_base + j * 16);
            uint4 u0 = __ldg(xp), u1 = __ldg(xp + 1);
            const __nv_bfloat162* h0p = reinterpret_cast<const __nv_bfloat162*>(&u0);
            const __nv_bfloat162* h1p = reinterpret_cast<const __nv_bfloat162*>(&u1);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float2 f0 = __bfloat1622float2(h0p[e]);
              float2 f1 = __bfloat1622float2(h1p[e]);
              xv[2 * e] = f0.x; xv[2 * e + 1] = f0.y;
              xv[8 + 2 * e] = f1.x; xv[8 + 2 * e + 1] = f1.y;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) xv[e] = 0.f;
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float tt = v[0][e] * xv[e];
            o[e] = tt + tt;
            if (NB == 2) o[e] += v[NB - 1][e];
          }
          stage_store16(sOut, row, j, o);
        }
      }
      // accumulator drained: hand it back to the MMA warp
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) hand_back(as);
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, 128);
      if (etid == 0) {
        if (EPI == EPI_PROPOSED || EPI == EPI_T4) {
          ptx::tma_store_4d(&mapO0, sOut, c_base, w0, h0, n0);
          ptx::tma_store_4d(&mapO1, sOut + 16384, c_base, w0, h0, n0);
          ptx::tma_store_4d(&mapO2, sOut + 32768, c_base, w0, h0, n0);
        } else if (EPI == EPI_PLAIN) {
#pragma unroll
          for (int i = 0; i < NB; ++i) ptx::tma_store_4d(&mapO0, sOut + i * 16384, c_base + i * 64, w0, h0, n0);
        } else {
          ptx::tma_store_4d(&mapO0, sOut, c_base, w0, h0, n0);
        }
        ptx::bulk_commit();
      }
    }
    if (etid == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  if (PAIR) {
    ptx::cluster_sync();
    if (warp == 2) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc2(tmem_base, 512);
    }
  } else {
    __syncthreads();
    if (warp == 2) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc(tmem_base, 512);
    }
  }
}

// split-K fold: one thread per (pixel, 8 output channels) sums the K slices in
// order and applies the conv_gemm epilogue (same math as above)
template <int EPI, int NB>
__global__ void __launch_bounds__(256) splitk_finish_kernel(const float* __restrict__ part, int S, long long Mpix,
                                                            int ld, int Cout, bf16* o0, bf16* o1, bf16* o2,
                                                            const float* __restrict__ bias0,
                                                            const float* __restrict__ bias1,
                                                            const float* __restrict__ bias2,
                                                            const bf16* __restrict__ xres) {
  const int c8n = Cout / 8;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Mpix * c8n) return;
  const long long pix = idx / c8n;
  const int c = (int)(idx - pix * c8n) * 8;
  constexpr int NACC = (EPI == EPI_PLAIN) ? 1 : NB;
  // partial column of accumulator i for output channel c
  int col[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i)
    col[i] = (EPI == EPI_PLAIN) ? c : (c / 64) * NB * 64 + i * 64 + c % 64;
  float acc[NACC][8];
#pragma unroll
  for (int i = 0; i < NACC; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[i][e] = 0.f;
  for (int s = 0; s < S; ++s) {
    const float* prow = part + ((size_t)s * Mpix + pix) * ld;
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const float4 u0 = __ldg(reinterpret_cast<const float4*>(prow + col[i]));
      const float4 u1 = __ldg(reinterpret_cast<const float4*>(prow + col[i] + 4));
      acc[i][0] += u0.x; acc[i][1] += u0.y; acc[i][2] += u0.z; acc[i][3] += u0.w;
      acc[i][4] += u1.x; acc[i][5] += u1.y; acc[i][6] += u1.z; acc[i][7] += u1.w;
    }
  }
  const size_t off = (size_t)pix * Cout + c;
  uint4 outv[3];
  uint32_t* p0 = reinterpret_cast<uint32_t*>(&outv[0]);
  uint32_t* p1 = reinterpret_cast<uint32_t*>(&outv[1]);
  uint32_t* p2 = reinterpret_cast<uint32_t*>(&outv[2]);
  if (EPI == EPI_PROPOSED || EPI == EPI_T4) {
    float y[8], a[8], b[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (EPI == EPI_PROPOSED) {
        a[e] = acc[0][e] + __ldg(bias0 + c + e);
        b[e] = acc[1 % NACC][e] + __ldg(bias1 + c + e);
        y[e] = fmaf(a[e], b[e], acc[2 % NACC][e] + __ldg(bias2 + c + e));
      } else {
        a[e] = acc[0][e];
        b[e] = acc[1 % NACC][e];
        y[e] = a[e] * b[e];
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      p0[e] = pack_bf16x2(y[2 * e], y[2 * e + 1]);
      p1[e] = pack_bf16x2(a[2 * e], a[2 * e + 1]);
      p2[e] = pack_bf16x2(b[2 * e], b[2 * e + 1]);
    }
    *reinterpret_cast<uint4*>(o0 + off) = outv[0];
    *reinterpret_cast<uint4*>(o1 + off) = outv[1];
    *reinterpret_cast<uint4*>(o2 + off) = outv[2];
  } else if (EPI == EPI_PLAIN) {
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = acc[0][e] + (bias0 ? __ldg(bias0 + c + e) : 0.f);
#pragma unroll
    for (int e = 0; e < 4; ++e) p0[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
    *reinterpret_cast<uint4*>(o0 + off) = outv[0];
  } else {  // EPI_SQ
    const uint4 xu = __ldg(reinterpret_cast<const uint4*>(xres + off));
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xu);
    float v[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 xf = __bfloat1622float2(x2[e]);
      float t0 = acc[0][2 * e] * xf.x, t1 = acc[0][2 * e + 1] * xf.y;
      v[2 * e] = t0 + t0 + (NB == 2 ? acc[NACC - 1][2 * e] : 0.f);
      v[2 * e + 1] = t1 + t1 + (NB == 2 ? acc[NACC - 1][2 * e + 1] : 0.f);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) p0[e] = pack_bf16x2(v[2 * e], v[2 * e + 1]);
    *reinterpret_cast<uint4*>(o0 + off) = outv[0];
  }
}

// ---------------------------------------------------------------------------
// K4 wgrad
// ---------------------------------------------------------------------------
struct WgArgs {
  int mtiles, ntiles, splits;
  int pb_w, pb_h, pb_n;                 // pixel box (product 64)
  int pt_w, pt_h, ptiles;               // pixel tiles along w, h; total
  int r, pad, cblks, kb_half, nkb;      // 64-row k-block decode
  int Jd, Kf;
  int sstride;                          // x traversal stride (stride-2 layers, strided x maps)
  float* part;                          // [splits][Jd][Kf]
};

template <int NBLK>
struct WgCfg {
  static constexpr int A_BYTES = 2 * 8192;
  static constexpr int B_BYTES = NBLK * 8192;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int S0 = (220 * 1024 - 2048) / STAGE;
  static constexpr int STAGES = S0 > 8 ? 8 : S0;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 1024;
  static constexpr int TCOLS = NBLK * 64 <= 32 ? 32 : (NBLK * 64 <= 64 ? 64 : (NBLK * 64 <= 128 ? 128 : 256));
};

template <int NBLK>
__global__ void __launch_bounds__(256, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap mapX0, const __grid_constant__ CUtensorMap mapX1,
                 const __grid_constant__ CUtensorMap mapD, const WgArgs args) {
  using Cfg = WgCfg<NBLK>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = (uint64_t*)(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int b = blockIdx.x;
  const int ntile = b % args.ntiles;
  b /= args.ntiles;
  const int mtile = b % args.mtiles;
  const int split = b / args.mtiles;
  const int p_beg = (int)((long long)split * args.ptiles / args.splits);
  const int p_end = (int)((long long)(split + 1) * args.ptiles / args.splits);
  const int nA = (2 * mtile + 1 < args.nkb) ? 2 : 1;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&mapX0);
    ptx::prefetch_tmap(&mapX1);
    ptx::prefetch_tmap(&mapD);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(tmem_slot, Cfg::TCOLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t bytes = (uint32_t)(nA * 8192 + Cfg::B_BYTES);
      // the CTA's two x k-blocks are fixed: decoded once; the pixel tile walks
      // (w, h, n) incrementally (no divisions per stage in the producer thread)
      int a_c[2] = {0, 0}, a_dx[2] = {0, 0}, a_dy[2] = {0, 0}, a_h[2] = {0, 0};
      for (int a = 0; a < nA; ++a) {
        const int kb = 2 * mtile + a;
        const int half = kb / args.kb_half, kk = kb % args.kb_half;
        const int tap = kk / args.cblks, cb = kk % args.cblks;
        a_h[a] = half;
        a_c[a] = cb * 64;
        a_dx[a] = tap % args.r - args.pad;
        a_dy[a] = tap / args.r - args.pad;
      }
      int tw = p_beg % args.pt_w, th = (p_beg / args.pt_w) % args.pt_h, tn = p_beg / (args.pt_w * args.pt_h);
      for (int pt = p_beg; pt < p_end; ++pt) {
        const int w0 = tw * args.pb_w, h0 = th * args.pb_h, n0 = tn * args.pb_n;
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], bytes);
        for (int a = 0; a < nA; ++a)
          ptx::tma_load_4d(a_h[a] ? &mapX1 : &mapX0, &full[stage], sA + stage * Cfg::A_BYTES + a * 8192, a_c[a],
                           args.sstride * w0 + a_dx[a], args.sstride * h0 + a_dy[a], n0);
        if (++tw == args.pt_w) {
          tw = 0;
          if (++th == args.pt_h) { th = 0; ++tn; }
        }
#pragma unroll
        for (int i = 0; i < NBLK; ++i)
          ptx::tma_load_4d(&mapD, &full[stage], sB + stage * Cfg::B_BYTES + i * 8192,
                           (ntile * NBLK + i) * 64, w0, h0, n0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // warp-wide loop, elected lane issues (descriptors stay on the uniform datapath)
    constexpr uint32_t IDESC = ptx::idesc_bf16(128, NBLK * 64, true, true);
    constexpr uint32_t DHI = ptx::sw128_desc_hi(1024);
    const bool leader = ptx::elect_one();
    const uint32_t a_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sA), 8192);
    const uint32_t b_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sB), 8192);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t accum = 0;
    for (int pt = p_beg; pt < p_end; ++pt) {
      ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      const uint32_t a_lo = a_lo0 + stage * (Cfg::A_BYTES >> 4);
      const uint32_t b_lo = b_lo0 + stage * (Cfg::B_BYTES >> 4);
      if (leader) {
#pragma unroll
        for (int k = 0; k < 4; ++k)  // 16 pixels (K) per MMA = two 8-row groups of 128 B
          ptx::mma_bf16(tmem_base, ptx::mk_desc(DHI, a_lo + 128 * k), ptx::mk_desc(DHI, b_lo + 128 * k), IDESC,
                        accum | (uint32_t)k);
        ptx::mma_commit(&empty[stage]);
      }
      accum = 1;
      __syncwarp();
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if (leader) ptx::mma_commit(done);
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int kglob = mtile * 128 + row;
    const bool has_work = p_end > p_beg;
    if (has_work) {
      ptx::mbar_wait(done, 0);
      ptx::tc_fence_after();
    }
    const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16);
    float* dst = args.part + (size_t)split * args.Jd * args.Kf;
#pragma unroll 1
    for (int c = 0; c < NBLK * 64; c += 16) {
      float v[16];
      if (has_work) {
        ptx::tmem_ld16(tbase + c, v);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = 0.f;
      }
      if (kglob < args.Kf && row < nA * 64) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          int j = ntile * NBLK * 64 + c + e;
          dst[(size_t)j * args.Kf + kglob] = v[e];
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, Cfg::TCOLS);
  }
}

// K4 v1 on CTA pairs. The v1 wgrad is bound by TMA delivery (every stage brings
// 16 KB of x boxes and NBLK x 8 KB of D boxes for 128 x 64 NBLK x 64 MACs; the
// chip-wide TMA throughput, ~6300 B/cycle, caps it at ~30% tensor-pipe use on the
// 512-channel layers). The two CTAs of a cluster take M tiles 2m and 2m + 1 of the
// same N tile and pixel range and issue M = 256 MMAs (cta_group::2): each holds its
// own x boxes but only HALF of the D boxes (its NBLK / 2 64-column blocks), so every
// D byte reaches one SM instead of two: 16 + 4 NBLK KB per SM and stage instead of
// 16 + 8 NBLK. Same partial-slot output as wgrad_kernel.
template <int NBLK>
struct WpCfg {
  static constexpr int HB = NBLK / 2;  // D boxes per CTA
  static constexpr int A_BYTES = 2 * 8192;
  static constexpr int B_BYTES = HB * 8192;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int S0 = (220 * 1024 - 2048) / STAGE;
  static constexpr int STAGES = S0 > 8 ? 8 : S0;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 1024;
  static constexpr int TCOLS = NBLK * 64 <= 128 ? 128 : 256;
};

template <int NBLK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    wgrad_pair_kernel(const __grid_constant__ CUtensorMap mapX0, const __grid_constant__ CUtensorMap mapX1,
                      const __grid_constant__ CUtensorMap mapD, const WgArgs args) {
  using Cfg = WpCfg<NBLK>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * Cfg::A_BYTES;
  uint64_t* full = (uint64_t*)(sB + STAGES * Cfg::B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_rank();
  int b = blockIdx.x >> 1;
  const int ntile = b % args.ntiles;
  b /= args.ntiles;
  const int mpairs = (args.mtiles + 1) / 2;
  const int mpair = b % mpairs;
  const int split = b / mpairs;
  const int mtile = 2 * mpair + (int)rank;
  const int p_beg = (int)((long long)split * args.ptiles / args.splits);
  const int p_end = (int)((long long)(split + 1) * args.ptiles / args.splits);
  // 64-row k-blocks of x this CTA loads (a missing second M tile loads none: its
  // TMEM rows are computed from stale smem and never stored)
  auto n_a = [&](int mt) { return mt >= args.mtiles ? 0 : ((2 * mt + 1 < args.nkb) ? 2 : 1); };
  const int nA = n_a(mtile);

  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&mapX0);
    ptx::prefetch_tmap(&mapX1);
    ptx::prefetch_tmap(&mapD);
    for (int i = 0; i < STAGES; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc2(tmem_slot, Cfg::TCOLS);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // both CTAs' boxes complete on CTA0's full barrier; CTA0 expects the pair's bytes
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t bytes = (uint32_t)((n_a(2 * mpair) + n_a(2 * mpair + 1)) * 8192 + 2 * Cfg::B_BYTES);
      int a_c[2] = {0, 0}, a_dx[2] = {0, 0}, a_dy[2] = {0, 0}, a_h[2] = {0, 0};
      for (int a = 0; a < nA; ++a) {
        const int kb = 2 * mtile + a;
        const int half = kb / args.kb_half, kk = kb % args.kb_half;
        const int tap = kk / args.cblks, cb = kk % args.cblks;
        a_h[a] = half;
        a_c[a] = cb * 64;
        a_dx[a] = tap % args.r - args.pad;
        a_dy[a] = tap / args.r - args.pad;
      }
      int tw = p_beg % args.pt_w, th = (p_beg / args.pt_w) % args.pt_h, tn = p_beg / (args.pt_w * args.pt_h);
      for (int pt = p_beg; pt < p_end; ++pt) {
        const int w0 = tw * args.pb_w, h0 = th * args.pb_h, n0 = tn * args.pb_n;
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], bytes);
        const uint32_t fb = ptx::peer0(&full[stage]);
        for (int a = 0; a < nA; ++a)
          ptx::tma4_cg2(a_h[a] ? &mapX1 : &mapX0, fb, sA + stage * Cfg::A_BYTES + a * 8192, a_c[a],
                        args.sstride * w0 + a_dx[a], args.sstride * h0 + a_dy[a], n0);
        if (++tw == args.pt_w) {
          tw = 0;
          if (++th == args.pt_h) { th = 0; ++tn; }
        }
#pragma unroll
        for (int i = 0; i < Cfg::HB; ++i)
          ptx::tma4_cg2(&mapD, fb, sB + stage * Cfg::B_BYTES + i * 8192, (ntile * NBLK + (int)rank * Cfg::HB + i) * 64,
                        w0, h0, n0);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // M = 256 over the pair (CTA r: rows of M tile 2m + r), N = NBLK x 64 (CTA r
      // holds columns [r N/2, (r+1) N/2) of B); commits reach both CTAs' barriers
      constexpr uint32_t IDESC = ptx::idesc_bf16(256, NBLK * 64, true, true);
      constexpr uint32_t DHI = ptx::sw128_desc_hi(1024);
      const bool leader = ptx::elect_one();
      const uint32_t a_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sA), 8192);
      const uint32_t b_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sB), 8192);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t accum = 0;
      for (int pt = p_beg; pt < p_end; ++pt) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a_lo = a_lo0 + stage * (Cfg::A_BYTES >> 4);
        const uint32_t b_lo = b_lo0 + stage * (Cfg::B_BYTES >> 4);
        if (leader) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            ptx::mma_cg2(tmem_base, ptx::mk_desc(DHI, a_lo + 128 * k), ptx::mk_desc(DHI, b_lo + 128 * k), IDESC,
                         accum | (uint32_t)k);
          ptx::commit_mc(&empty[stage]);
        }
        accum = 1;
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (leader) ptx::commit_mc(done);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int kglob = mtile * 128 + row;
    const bool has_work = p_end > p_beg;
    if (has_work) {
      ptx::mbar_wait(done, 0);
      ptx::tc_fence_after();
    }
    const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16);
    float* dst = args.part + (size_t)split * args.Jd * args.Kf;
#pragma unroll 1
    for (int c = 0; c < NBLK * 64; c += 16) {
      float v[16];
      if (has_work) {
        ptx::tmem_ld16(tbase + c, v);
        ptx::tmem_wait_ld();
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = 0.f;
      }
      if (kglob < args.Kf && row < nA * 64) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          int j = ntile * NBLK * 64 + c + e;
          dst[(size_t)j * args.Kf + kglob] = v[e];
        }
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem_base, Cfg::TCOLS);
  }
}

// ---------------------------------------------------------------------------
// vectorised backward prologue for the tcgen05 path:
// D = [dy*b | dy*a | dy] (proposed) / [dy*b | dy*a] (t4) in bf16 plus
// fixed-order column partial sums (bias gradients) of the fp32 products.
// ---------------------------------------------------------------------------
// up = 1 (stride-2 layers): D rows live on the stride-1 grid (OH1 x OW1); rows
// at odd positions are written as zeros (the zero-upsampled gradient operand).
__global__ void __launch_bounds__(256) bwd_prologue_vec_kernel(Plan P, const bf16* __restrict__ dy,
                                                               const bf16* __restrict__ a,
                                                               const bf16* __restrict__ b, bf16* __restrict__ D,
                                                               float* __restrict__ part, long long rows_per,
                                                               int up, int OH1, int OW1, int dstride) {
  ptx::pdl_wait();  // a, b come from the forward kernel
  ptx::pdl_launch();
  const int F = P.F, chunks = F / 8;
  const int lanes = 256 / chunks;  // rows processed concurrently
  const int ch = threadIdx.x % chunks, rl = threadIdx.x / chunks;
  const bool mat = caches_ab(P.family);
  const bool prop = d_has_g(P.family);
  const long long rows = up ? (long long)P.N * OH1 * OW1 : P.Mout;
  long long r0 = (long long)blockIdx.x * rows_per, r1 = r0 + rows_per;
  if (r1 > rows) r1 = rows;
  float s0[8], s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s0[e] = s1[e] = s2[e] = 0.f;
  if (rl < lanes && !up && mat) {
    // fast path (stride 1, D materialised): 4 rows per iteration, all 12 loads in flight
    constexpr int U = 4;
    for (long long m0 = r0 + rl; m0 < r1; m0 += (long long)U * lanes) {
      uint4 gu[U], au[U], bu[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        long long m = m0 + (long long)u * lanes;
        ok[u] = m < r1;
        size_t off = (size_t)(ok[u] ? m : r0) * F + ch * 8;
        gu[u] = __ldg(reinterpret_cast<const uint4*>(dy + off));
        au[u] = __ldg(reinterpret_cast<const uint4*>(a + off));
        bu[u] = __ldg(reinterpret_cast<const uint4*>(b + off));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        long long m = m0 + (long long)u * lanes;
        const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gu[u]);
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&au[u]);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bu[u]);
        uint4 d0, d1;
        uint32_t* d0p = reinterpret_cast<uint32_t*>(&d0);
        uint32_t* d1p = reinterpret_cast<uint32_t*>(&d1);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 g = __bfloat1622float2(g2[e]), av = __bfloat1622float2(a2[e]), bv = __bfloat1622float2(b2[e]);
          float x0 = g.x * bv.x, x1 = g.y * bv.y, y0 = g.x * av.x, y1 = g.y * av.y;
          d0p[e] = pack_bf16x2(x0, x1);
          d1p[e] = pack_bf16x2(y0, y1);
          s0[2 * e] += x0; s0[2 * e + 1] += x1;
          s1[2 * e] += y0; s1[2 * e + 1] += y1;
          s2[2 * e] += g.x; s2[2 * e + 1] += g.y;
        }
        bf16* drow = D + (size_t)m * dstride + ch * 8;
        *reinterpret_cast<uint4*>(drow) = d0;
        *reinterpret_cast<uint4*>(drow + F) = d1;
        if (prop && dstride == P.Jd) *reinterpret_cast<uint4*>(drow + 2 * F) = gu[u];
      }
    }
  } else if (rl < lanes) {
    for (long long md = r0 + rl; md < r1; md += lanes) {
      long long m = md;
      if (up) {
        long long n = md / ((long long)OH1 * OW1), rem = md % ((long long)OH1 * OW1);
        int h1 = (int)(rem / OW1), w1 = (int)(rem % OW1);
        bool real = !(h1 & 1) && !(w1 & 1) && (h1 >> 1) < P.OH && (w1 >> 1) < P.OW;
        if (!real) {
          bf16* drow = D + (size_t)md * P.Jd + ch * 8;
          uint4 z = make_uint4(0u, 0u, 0u, 0u);
          for (int blk = 0; blk < P.Jd / F; ++blk) *reinterpret_cast<uint4*>(drow + blk * F) = z;
          continue;
        }
        m = (n * P.OH + (h1 >> 1)) * P.OW + (w1 >> 1);
      }
      size_t off = (size_t)m * F + ch * 8;
      uint4 gu = __ldg(reinterpret_cast<const uint4*>(dy + off));
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gu);
      if (mat) {
        uint4 au = __ldg(reinterpret_cast<const uint4*>(a + off));
        uint4 bu = __ldg(reinterpret_cast<const uint4*>(b + off));
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&au);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&bu);
        uint4 d0, d1;
        uint32_t* d0p = reinterpret_cast<uint32_t*>(&d0);
        uint32_t* d1p = reinterpret_cast<uint32_t*>(&d1);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 g = __bfloat1622float2(g2[e]), av = __bfloat1622float2(a2[e]), bv = __bfloat1622float2(b2[e]);
          float x0 = g.x * bv.x, x1 = g.y * bv.y, y0 = g.x * av.x, y1 = g.y * av.y;
          d0p[e] = pack_bf16x2(x0, x1);
          d1p[e] = pack_bf16x2(y0, y1);
          s0[2 * e] += x0; s0[2 * e + 1] += x1;
          s1[2 * e] += y0; s1[2 * e + 1] += y1;
          s2[2 * e] += g.x; s2[2 * e + 1] += g.y;
        }
        bf16* drow = D + (size_t)md * P.Jd + ch * 8;
        *reinterpret_cast<uint4*>(drow) = d0;
        *reinterpret_cast<uint4*>(drow + F) = d1;
        if (prop) *reinterpret_cast<uint4*>(drow + 2 * F) = gu;
      } else {
        if (up) *reinterpret_cast<uint4*>(D + (size_t)md * P.Jd + ch * 8) = gu;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 g = __bfloat1622float2(g2[e]);
          s0[2 * e] += g.x; s0[2 * e + 1] += g.y;
        }
      }
    }
  }
  if (!part) return;  // no bias sums wanted (D only)
  // reduce over the row lanes of this block in a fixed order
  __shared__ float red[256][9];
  const int nsum = mat ? (prop ? 3 : 2) : 1;
  for (int sidx = 0; sidx < nsum; ++sidx) {
    float* src = sidx == 0 ? s0 : (sidx == 1 ? s1 : s2);
#pragma unroll
    for (int e = 0; e < 8; ++e) red[threadIdx.x][e] = src[e];
    __syncthreads();
    for (int tcol = threadIdx.x; tcol < chunks * 8; tcol += 256) {
      int c = tcol / 8, e = tcol % 8;
      float acc = 0.f;
      for (int l = 0; l < lanes; ++l) acc += red[l * chunks + c][e];
      int jcol = sidx * F + c * 8 + e;
      // proposed/t4: block 0 = sum(dy*b), 1 = sum(dy*a), 2 = sum(dy); else block 0 = sum(dy)
      part[(size_t)blockIdx.x * P.Jd + jcol] = acc;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static int g_num_sms = 0;
static int g_arch_ok = -1;

static bool init_driver_once() {
  int dev = 0;
  cudaDeviceProp prop;
  g_arch_ok = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return false; }
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) { cudaGetLastError(); return false; }
  g_num_sms = prop.multiProcessorCount;
  if (prop.major != 10) return false;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  g_arch_ok = 1;
  return true;
}
// first call from any thread initialises (a function-local static: thread-safe)
static bool init_driver() {
  static const bool ok = init_driver_once();
  return ok;
}

PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() { return g_encode; }

// the driver call needs a current context: a host thread whose first CUDA call is
// ours (e.g. torch's autograd worker running a backward) has none yet
// (CUDA_ERROR_INVALID_CONTEXT); binding the device's primary context through the
// runtime and retrying fixes that
CUresult tc_encode_tiled(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* ptr, const cuuint64_t* dims,
                         const cuuint64_t* strides, const cuuint32_t* box, const cuuint32_t* es,
                         CUtensorMapInterleave il, CUtensorMapSwizzle sw, CUtensorMapL2promotion l2,
                         CUtensorMapFloatOOBfill oob) {
  CUresult r = g_encode(m, dt, rank, ptr, dims, strides, box, es, il, sw, l2, oob);
  if (r == CUDA_ERROR_INVALID_CONTEXT) {
    cudaFree(nullptr);  // binds the current device's primary context to this thread
    cudaGetLastError();
    r = g_encode(m, dt, rank, ptr, dims, strides, box, es, il, sw, l2, oob);
  }
  return r;
}
int tc_num_sms() { return g_num_sms > 0 ? g_num_sms : 148; }

static int plain_blocks(int ch);

// fprop / dgrad kernel configurations (shared by dispatch and eligibility)
struct GemmCfg {
  int epi, nbk, tiles_nn, b_rs_tile, b_rs_blk, out_c_tile, nout, nbias;
};
static GemmCfg fprop_cfg(const Plan& P) {
  GemmCfg c;
  if (P.family == QD_FAM_PROPOSED || P.family == QD_FAM_T2AND4) { c.epi = EPI_PROPOSED; c.nbk = 3; }
  else if (P.family == QD_FAM_T4) { c.epi = EPI_T4; c.nbk = 2; }
  else { c.epi = EPI_PLAIN; c.nbk = plain_blocks(P.F); }
  if (c.epi == EPI_PLAIN) {
    c.tiles_nn = P.F / (64 * c.nbk); c.b_rs_tile = 64 * c.nbk; c.out_c_tile = 64 * c.nbk; c.nout = c.nbk;
    c.nbias = P.family == QD_FAM_FIRST_ORDER ? 1 : 0;
  } else {
    c.tiles_nn = P.F / 64; c.b_rs_tile = c.nbk * 64; c.out_c_tile = 64; c.nout = 3;
    c.nbias = (P.family == QD_FAM_PROPOSED || P.family == QD_FAM_T2AND4) ? 3 : 0;  // t2and4: zero biases
  }
  c.b_rs_blk = 64;
  return c;
}
static GemmCfg dgrad_cfg(const Plan& P) {
  GemmCfg c;
  c.epi = P.sq == 0 ? EPI_PLAIN : EPI_SQ;
  c.nbk = P.sq == 0 ? plain_blocks(P.C) : (P.sq == 1 ? 1 : 2);
  c.tiles_nn = P.sq == 0 ? P.C / (64 * c.nbk) : P.C / 64;
  c.b_rs_tile = P.sq == 0 ? 64 * c.nbk : 64;
  c.b_rs_blk = P.sq == 2 ? P.C : 64;
  c.out_c_tile = P.sq == 0 ? 64 * c.nbk : 64;
  c.nout = P.sq == 0 ? c.nbk : 1;
  c.nbias = 0;
  return c;
}

// stride-2 layers: only via the CTA-pair / halo kernels on the stride-1 grid
static bool s2_fits(const Plan& P) {
  if (P.s != 2 || P.r < 2) return false;
  Plan P1 = stride1_plan(P);
  GemmCfg f = fprop_cfg(P), d = dgrad_cfg(P);
  if (!conv2_fits(P.N, P.C, P.W, P.H, P1.OW, P1.OH, P.p, P.r, P.sq == 2, f.nbk, f.nout, f.tiles_nn, P.F, f.nbias))
    return false;
  if (!conv2_fits(P.N, P.Jd, P1.OW, P1.OH, P.W, P.H, P.r - 1 - P.p, P.r, 0, d.nbk, d.nout, d.tiles_nn, P.C, 0))
    return false;
  return wgrad2_split(P1) > 0;
}

// stride 2 on its own output grid (v1 kernels): fprop and wgrad read x through
// traversal-stride-2 TMA maps, the dgrad runs as four output-parity classes of
// D (no zero-upsampled operand, no 4x work); a class no tap reaches (r = 1)
// stores zeros. The squared-input families keep the stride-1-grid path (x*x operand, EPI_SQ
// dgrad). QD_S2_UPSAMPLE=1 forces the stride-1-grid path (A/B checks).
bool tc_s2_direct(const Plan& P) {
  static const bool off = getenv("QD_S2_UPSAMPLE") && atoi(getenv("QD_S2_UPSAMPLE"));
  return P.s == 2 && P.kind == QD_KIND_CONV && P.r >= 1 && P.sq == 0 && P.family != QD_FAM_T3 && !off &&
         P.OW <= 128 && P.OH <= 128 && P.dtype == QD_BF16 && P.C % 64 == 0 && P.F % 64 == 0;
}

bool tc_supported(const Plan& P, unsigned flags) {
  if (flags & QD_FLAG_FORCE_SIMT) return false;
  if (P.dtype != QD_BF16) return false;
  if (P.C % 64 || P.F % 64) return false;
  if (P.OH < 1 || P.OW < 1) return false;
  if (!init_driver()) return false;
  if (P.s == 1) return true;
  if (P.family == QD_FAM_T3) return false;  // t3 stride 2: CUDA-core path
  if (tc_s2_direct(P)) return true;
  return !(flags & QD_FLAG_TC_V1) && s2_fits(P);
}

static int make_map(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims, const cuuint32_t* box,
                    int trav = 1) {
  cuuint64_t strides[4];
  cuuint64_t acc = dims[0] * 2;
  for (int i = 1; i < rank; ++i) {
    strides[i - 1] = acc;
    acc *= dims[i];
  }
  // trav > 1: traversal stride along W and H (the box spans trav x the pixels it loads)
  cuuint32_t es[5] = {1, (cuuint32_t)trav, (cuuint32_t)trav, 1, 1};
  CUresult r = tc_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box,
                               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(QD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return QD_OK;
}

// NHWC activation map with a (64, Wb, Hb, Nb) box; trav = 2 loads every second
// pixel along W and H (Wb x Hb pixels from a 2Wb x 2Hb window)
static int map_act(CUtensorMap* m, const void* p, int Cch, int W, int H, int N, int Wb, int Hb, int Nb,
                   int trav = 1) {
  cuuint64_t dims[4] = {(cuuint64_t)Cch, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint32_t box[4] = {64, (cuuint32_t)(Wb * trav), (cuuint32_t)(Hb * trav), (cuuint32_t)Nb};
  return make_map(m, p, 4, dims, box, trav);
}
static int map_rows(CUtensorMap* m, const void* p, int K, int rows, int box_rows = 64) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  return make_map(m, p, 2, dims, box);
}

struct Box { int Wb, Hb, Nb, tw, th, tn; };

// choose the (Wb, Hb, Nb) pixel box with Wb*Hb*Nb <= cap that covers the grid
// with the fewest tiles (ties: wider boxes, longer TMA rows)
static Box choose_box(int W, int H, int N, int cap, bool exact) {
  Box best{1, 1, 1, W, H, N};
  long long best_tiles = -1;
  if (exact) {
    // box product must be exactly `cap` (a power of two); dims may overhang the
    // tensor (TMA zero-fills), so any grid works
    for (int wb = cap; wb >= 1; wb /= 2)
      for (int hb = cap / wb; hb >= 1; hb /= 2) {
        int nb = cap / (wb * hb);
        long long tiles = (long long)((W + wb - 1) / wb) * ((H + hb - 1) / hb) * ((N + nb - 1) / nb);
        if (best_tiles < 0 || tiles < best_tiles) {
          best_tiles = tiles;
          best = Box{wb, hb, nb, (W + wb - 1) / wb, (H + hb - 1) / hb, (N + nb - 1) / nb};
        }
      }
    return best;
  }
  for (int wb = (W < cap ? W : cap); wb >= 1; --wb) {
    for (int hb = (H < cap / wb ? H : cap / wb); hb >= 1; --hb) {
      int nb = cap / (wb * hb);
      if (nb > N) nb = N;
      if (nb < 1) continue;
      if (nb > 256 || wb > 256 || hb > 256) continue;
      if (exact && wb * hb * nb != cap) continue;
      long long tiles = (long long)((W + wb - 1) / wb) * ((H + hb - 1) / hb) * ((N + nb - 1) / nb);
      if (best_tiles < 0 || tiles < best_tiles) {
        best_tiles = tiles;
        best = Box{wb, hb, nb, (W + wb - 1) / wb, (H + hb - 1) / hb, (N + nb - 1) / nb};
      }
    }
  }
  return best;
}

// co-resident 2-CTA clusters of a kernel at this smem (cached per kernel / device)
template <typename K>
static int conv_pair_clusters(K kernel, size_t smem) {
  thread_local int maxc_[kMaxDev] = {};
  int& maxc = maxc_[cur_device()];
  if (maxc == 0) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(2 * 148, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)kernel, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    maxc = n > 0 ? n : g_num_sms / 2;
  }
  return maxc;
}

template <int EPI, int NB, int PAIR = 0>
static int launch_conv(const CUtensorMap& A0, const CUtensorMap& A1, const CUtensorMap& B, const CUtensorMap& O0,
                       const CUtensorMap& O1, const CUtensorMap& O2, const ConvArgs& args, cudaStream_t st) {
  using Cfg = ConvCfg<EPI, NB, PAIR>;
  auto kernel = conv_gemm_kernel<EPI, NB, PAIR>;
  raise_smem_attr((const void*)kernel, Cfg::SMEM);
  const int nwork = args.cls ? 4 * args.cls_tiles : args.total_tiles * args.ksplit;
  if (!PAIR) {
    int grid = nwork < g_num_sms ? nwork : g_num_sms;
    kernel<<<grid, 256, Cfg::SMEM, st>>>(A0, A1, B, O0, O1, O2, args);
  } else {
    int clusters = conv_pair_clusters(kernel, Cfg::SMEM);
    if (nwork < clusters) clusters = nwork;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(2 * clusters, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, A0, A1, B, O0, O1, O2, args);
  }
  count_launch(st, "conv_gemm");
  return check_launch("conv_gemm");
}

template <int EPI, int NB>
static int launch_conv_split(const CUtensorMap& A0, const CUtensorMap& A1, const CUtensorMap& B,
                             const CUtensorMap& O0, const CUtensorMap& O1, const CUtensorMap& O2,
                             const ConvArgs& args, void* o0, void* o1, void* o2, cudaStream_t st, bool pair) {
  int rc = pair ? launch_conv<EPI, NB, 1>(A0, A1, B, O0, O1, O2, args, st)
                : launch_conv<EPI, NB>(A0, A1, B, O0, O1, O2, args, st);
  if (rc || args.ksplit <= 1) return rc;
  const long long n = args.Mpix * (args.Cout / 8);
  splitk_finish_kernel<EPI, NB><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      args.part, args.ksplit, args.Mpix, args.part_ld, args.Cout, (bf16*)o0, (bf16*)(o1 ? o1 : o0),
      (bf16*)(o2 ? o2 : o0), args.bias0, args.bias1, args.bias2, args.xres);
  count_launch(st, "splitk_finish");
  return check_launch("splitk_finish");
}

// K slices for a conv_gemm launch: only when the output grid leaves most SMs idle,
// each slice >= 8 k-blocks (K 512); QD_NO_SPLITK=1 disables
static int conv_ksplit(long long tiles, int KB, int sms = 0) {
  if (sms <= 0) sms = tc_num_sms();
  if (getenv("QD_NO_SPLITK") || tiles * 2 > sms) return 1;
  long long S = sms / tiles;
  if (S > KB / 8) S = KB / 8;
  return S < 1 ? 1 : (int)S;
}

template <int NBLK>
static int launch_wgrad(const CUtensorMap& X0, const CUtensorMap& X1, const CUtensorMap& Dm, const WgArgs& args,
                        cudaStream_t st) {
  using Cfg = WgCfg<NBLK>;
  raise_smem_attr((const void*)wgrad_kernel<NBLK>, Cfg::SMEM);
  int grid = args.mtiles * args.ntiles * args.splits;
  wgrad_kernel<NBLK><<<grid, 256, Cfg::SMEM, st>>>(X0, X1, Dm, args);
  count_launch(st, "wgrad_v1");
  return check_launch("wgrad");
}
template <int NBLK>
static int launch_wgrad_pair(const CUtensorMap& X0, const CUtensorMap& X1, const CUtensorMap& Dm,
                             const WgArgs& args, cudaStream_t st) {
  using Cfg = WpCfg<NBLK>;
  raise_smem_attr((const void*)wgrad_pair_kernel<NBLK>, Cfg::SMEM);
  int grid = 2 * ((args.mtiles + 1) / 2) * args.ntiles * args.splits;
  wgrad_pair_kernel<NBLK><<<grid, 256, Cfg::SMEM, st>>>(X0, X1, Dm, args);
  count_launch(st, "wgrad_v1");
  return check_launch("wgrad pair");
}

// v1 wgrad shape: N tile (64-column blocks: 4 / 3 / 2 / 1 dividing Jd) and the
// pixel split S. One CTA per SM, so the grid (tiles x S) should fill whole waves:
// S = SMs / tiles when there are few tiles, and among the N tiles the one with the
// best wave fill wins (narrower N pays a little in operand bytes per MMA), e.g.
// Jd 1536, Kf 4608: 216 tiles (1.46 waves) at N 256 vs 288 (1.95) at N 192.
static long long wgrad_split_for(long long tiles, long long ptiles, int sms) {
  long long S = sms / tiles;
  long long cap = ptiles / 4;
  if (cap < 1) cap = 1;
  if (S > cap) S = cap;
  return S < 1 ? 1 : S;
}

static int wgrad_ntile_blocks(const Plan& P, long long ptiles) {
  const int nb = P.Jd / 64, mtiles = (P.Kf / 64 + 1) / 2, sms = tc_num_sms();
  if (const char* e = getenv("QD_WG_NBLK")) {  // dev: pin the N tile (64-column blocks)
    const int c = atoi(e);
    if (c >= 1 && c <= 4 && nb % c == 0) return c;
  }
  int best = 1;
  double best_eff = -1.0;
  for (int c = 4; c >= 1; --c) {
    if (nb % c) continue;
    const long long tiles = (long long)mtiles * (nb / c);
    const long long ctas = tiles * wgrad_split_for(tiles, ptiles, sms);
    const long long waves = (ctas + sms - 1) / sms;
    const double fill = (double)ctas / (double)(waves * sms);
    const double eff = fill * (c == 4 ? 1.0 : (c == 3 ? 0.97 : (c == 2 ? 0.9 : 0.75)));
    if (eff > best_eff + 1e-9) { best_eff = eff; best = c; }
  }
  return best;
}

static long long wgrad_ptiles(const Plan& P) {
  Box pb = choose_box(P.OW, P.OH, P.N, 64, true);
  return (long long)pb.tw * pb.th * pb.tn;
}

// v1 wgrad launch shape: CTA pairs or single CTAs, the N tile (64-column blocks)
// and the pixel split S. Pairs (wgrad_pair_kernel) need an even block count and
// two M tiles; they are taken when a small cost model says so: per tile, MACs /
// (per-SM MMA rate x TMA factor) with the factor min(1, 7 / operand KB per
// 64-pixel k-step and 8K MACs) -- the single kernel at N = 256 delivers 48 KB per
// 16 x 8K MACs, the pair 32 -- times whole waves of the grid, plus the fold's
// S x Jd x Kf x 8 bytes of partial traffic; pairs take S = 1 (QD_WPAIR=0: never).
struct WgShape { int pair, nblk, S; };
static WgShape wgrad_v1_shape(const Plan& P) {
  const long long ptiles = wgrad_ptiles(P);
  const int sms = tc_num_sms(), nb = P.Jd / 64, mtiles = (P.Kf / 64 + 1) / 2;
  WgShape s{0, wgrad_ntile_blocks(P, ptiles), 1};
  s.S = (int)wgrad_split_for((long long)mtiles * (nb / s.nblk), ptiles, sms);
  const char* on = getenv("QD_WPAIR");  // QD_WPAIR=0: single CTAs only
  if ((on && !atoi(on)) || mtiles < 2 || nb % 2) return s;
  const double px = (double)ptiles * 64;
  auto cost = [&](int pair, int c, int S) {
    const long long units = (long long)(pair ? (mtiles + 1) / 2 : mtiles) * (nb / c) * S;
    const int slots = pair ? sms / 2 : sms;
    const long long waves = (units + slots - 1) / slots;
    const double kb = pair ? (16.0 + 4.0 * c) / c : (16.0 + 8.0 * c) / c;  // KB per k-step and 8K MACs
    const double rate = kb > 7.0 ? 7.0 / kb : 1.0;
    const double tile_us = 128.0 * 64 * c * (px / S) / 5.5e6 / rate;
    const double fold_us = (double)S * P.Jd * P.Kf * 8 / 6.0e6;
    return waves * tile_us + fold_us;
  };
  double best = cost(0, s.nblk, s.S);
  // pairs without extra pixel splits: an S = 2 pair's partial fold (~22 µs at
  // 512@7) costs more than the split saves (measured); QD_WPAIR_SMAX=K (dev) allows K
  const int smax = getenv("QD_WPAIR_SMAX") ? atoi(getenv("QD_WPAIR_SMAX")) : 1;
  for (int c = 4; c >= 2; c -= 2) {
    if (nb % c) continue;
    for (int S = 1; S <= smax && ptiles / S >= 4; ++S) {
      const double t = cost(1, c, S);
      if (t < best * 0.97) { best = t; s = WgShape{1, c, S}; }
    }
  }
  return s;
}

int tc_wgrad_split(const Plan& P) {
  if (!(P.flags & QD_FLAG_TC_V1)) {
    int s3 = wgrad3_split(P);
    if (s3 > 0) return s3;
    int s2 = wgrad2_split(P);
    if (s2 > 0) return s2;
  }
  return wgrad_v1_shape(P).S;
}

// generic conv-GEMM launch (fprop or dgrad)
static int run_conv(int epi, int nbk, const void* a0, const void* a1, int Cin, int Win, int Hin, int N,
                    int OWg, int OHg, int pad_eff, int r, int dual, const void* wmat, int wrows, int wK,
                    int b_rs_tile, int b_rs_blk, int tiles_nn, int out_c_tile, void* o0, void* o1, void* o2,
                    int Cout, const float* const bias[3], const void* xres, cudaStream_t st,
                    float* skpart = nullptr, size_t skbytes = 0, int trav = 1, int cls = 0, int Hx = 0,
                    int Wx = 0, int force_part = 0, int* ksplit_out = nullptr) {
  Box bx = choose_box(OWg, OHg, N, 128, false);
  const long long mtiles = (long long)bx.tw * bx.th * bx.tn;
  // CTA pairs (M = 256 over two SMs, each holding half of the weight tile): only
  // with QD_CPAIR=1 while being measured, never for the raw-accumulator modes
  const char* cp = getenv("QD_CPAIR");
  const bool pair = cp && atoi(cp) && mtiles >= 2 && !force_part;
  CUtensorMap A0, A1, B, O0, O1, O2;
  int rc;
  if ((rc = map_act(&A0, a0, Cin, Win, Hin, N, bx.Wb, bx.Hb, bx.Nb, trav))) return rc;
  if ((rc = map_act(&A1, a1 ? a1 : a0, Cin, Win, Hin, N, bx.Wb, bx.Hb, bx.Nb, trav))) return rc;
  if ((rc = map_rows(&B, wmat, wK, wrows, pair ? 32 : 64))) return rc;
  if ((rc = map_act(&O0, o0, Cout, OWg, OHg, N, bx.Wb, bx.Hb, bx.Nb))) return rc;
  if ((rc = map_act(&O1, o1 ? o1 : o0, Cout, OWg, OHg, N, bx.Wb, bx.Hb, bx.Nb))) return rc;
  if ((rc = map_act(&O2, o2 ? o2 : o0, Cout, OWg, OHg, N, bx.Wb, bx.Hb, bx.Nb))) return rc;
  ConvArgs g;
  memset(&g, 0, sizeof(g));
  g.tiles_w = bx.tw; g.tiles_h = bx.th; g.tiles_nn = tiles_nn;
  g.total_tiles = (int)((pair ? (mtiles + 1) / 2 : mtiles) * tiles_nn);  // PAIR: pair tiles
  g.Wb = bx.Wb; g.Hb = bx.Hb; g.Nb = bx.Nb; g.box_rows = bx.Wb * bx.Hb * bx.Nb;
  g.OHg = OHg; g.OWg = OWg; g.Ng = N;
  g.r = r; g.pad_eff = pad_eff; g.cblks = Cin / 64;
  g.kb_half = r * r * (Cin / 64); g.dual = dual;
  g.b_rs_tile = b_rs_tile; g.b_rs_blk = b_rs_blk; g.out_c_tile = out_c_tile; g.Cout = Cout;
  g.bias0 = bias[0]; g.bias1 = bias[1]; g.bias2 = bias[2];
  g.xres = (const bf16*)xres;
  const int KB = g.kb_half * (1 + dual);
  g.ksplit = 1;
  g.kb_per = KB;
  g.Mpix = (long long)N * OHg * OWg;
  g.part_ld = tiles_nn * nbk * 64;
  const int S = conv_ksplit(g.total_tiles, KB, pair ? tc_num_sms() / 2 : 0);
  if (S > 1 && skpart && (size_t)S * g.Mpix * g.part_ld * 4 <= skbytes) {
    g.kb_per = (KB + S - 1) / S;
    g.ksplit = (KB + g.kb_per - 1) / g.kb_per;
    g.part = skpart;
  }
  // raw fp32 accumulators whatever the split (fp32 x3 path): force_part 1 -> skpart,
  // 2 -> o0 itself when unsplit (a plain epilogue's raw rows ARE the fp32 output)
  if (force_part && !g.part) {
    g.part = force_part == 2 ? (float*)o0 : skpart;
    if (!g.part || (force_part == 1 && (size_t)g.Mpix * g.part_ld * 4 > skbytes))
      return set_error(QD_ERR_UNSUPPORTED, "x3: raw accumulator buffer too small");
  }
  if (ksplit_out) *ksplit_out = g.ksplit;
  g.sstride = trav;
  if (g.part && force_part) {
    // the split-K finish of the bf16 epilogues must not run: the caller folds
#define QD_LCP(E, NBV) launch_conv<E, NBV>(A0, A1, B, O0, O1, O2, g, st)
    if (epi == EPI_PROPOSED) return QD_LCP(EPI_PROPOSED, 3);
    if (epi == EPI_T4) return QD_LCP(EPI_T4, 2);
    if (nbk == 4) return QD_LCP(EPI_PLAIN, 4);
    if (nbk == 2) return QD_LCP(EPI_PLAIN, 2);
    return QD_LCP(EPI_PLAIN, 1);
#undef QD_LCP
  }
  g.sstride = trav;
  if (cls) {
    if (epi != EPI_PLAIN || dual) return set_error(QD_ERR_UNSUPPORTED, "parity-class dgrad: plain epilogue only");
    // the four output-parity classes of a stride-2 dgrad, most k-blocks first
    // (static round-robin over the persistent grid then balances like LPT)
    int code[4], n = 0;
    for (int ph = 0; ph < 2; ++ph)
      for (int pw = 0; pw < 2; ++pw) {
        // a class no tap reaches (r = 1) keeps 0 k-blocks: its tiles store zeros
        const int nty = (r - ((pad_eff - ph) & 1) + 1) / 2, ntx = (r - ((pad_eff - pw) & 1) + 1) / 2;
        code[n++] = ph | pw << 1 | (nty * ntx * g.cblks) << 2;
      }
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j)
        if ((code[j] >> 2) > (code[i] >> 2)) { int t = code[i]; code[i] = code[j]; code[j] = t; }
    for (int i = 0; i < 4; ++i) g.cls_code[i] = code[i];
    g.cls = 1;
    g.cls_tiles = g.total_tiles;
    g.Hx = Hx; g.Wx = Wx;
    g.out = (bf16*)o0;
  }
#define QD_LC(E, NBV) launch_conv_split<E, NBV>(A0, A1, B, O0, O1, O2, g, o0, o1, o2, st, pair)
  if (epi == EPI_PROPOSED) return QD_LC(EPI_PROPOSED, 3);
  if (epi == EPI_T4) return QD_LC(EPI_T4, 2);
  if (epi == EPI_PLAIN) {
    if (nbk == 4) return QD_LC(EPI_PLAIN, 4);
    if (nbk == 2) return QD_LC(EPI_PLAIN, 2);
    return QD_LC(EPI_PLAIN, 1);
  }
  if (nbk == 2) return QD_LC(EPI_SQ, 2);
  return QD_LC(EPI_SQ, 1);
#undef QD_LC
}

// split-K partial bytes the stride-1 v1 fprop / dgrad of P may use (workspace)
size_t tc_splitk_bytes(const Plan& P) {
  if (P.s != 1 || P.dtype != QD_BF16) return 0;
  size_t need = 0;
  {
    GemmCfg c = fprop_cfg(P);
    Box bx = choose_box(P.OW, P.OH, P.N, 128, false);
    const long long tiles = (long long)bx.tw * bx.th * bx.tn * c.tiles_nn;
    const int KB = P.r * P.r * (P.C / 64) * (P.sq == 2 ? 2 : 1);
    const int S = conv_ksplit(tiles, KB);
    if (S > 1) need = (size_t)S * P.N * P.OH * P.OW * c.tiles_nn * c.nbk * 64 * 4;
  }
  {
    GemmCfg c = dgrad_cfg(P);
    Box bx = choose_box(P.W, P.H, P.N, 128, false);
    const long long tiles = (long long)bx.tw * bx.th * bx.tn * c.tiles_nn;
    const int KB = P.r * P.r * (P.Jd / 64);
    const int S = conv_ksplit(tiles, KB);
    const size_t b = S > 1 ? (size_t)S * P.N * P.H * P.W * c.tiles_nn * c.nbk * 64 * 4 : 0;
    if (b > need) need = b;
  }
  return need;
}

static int plain_blocks(int ch) { return ch % 256 == 0 ? 4 : (ch % 128 == 0 ? 2 : 1); }

// plain fprop GEMM (no bias, one output) -- the t3 forward and its backward recompute
static int tc_fprop_plain(const Plan& P, const void* a0, const void* a1, const void* wpack, void* out,
                          cudaStream_t st) {
  GemmCfg c = fprop_cfg(P);
  const float* nob[3] = {nullptr, nullptr, nullptr};
  if (P.s == 2) {
    Plan P1 = stride1_plan(P);
    return run_conv2(c.epi, c.nbk, a0, a1, P.C, P.W, P.H, P.N, P1.OW, P1.OH, P.p, P.r, 0, wpack, P.nb * P.F, P.Kf,
                     c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, out, nullptr, nullptr, P.F, nob, nullptr, st, 2);
  }
  if (!(P.flags & QD_FLAG_TC_V1)) {
    int rc2 = run_conv2(c.epi, c.nbk, a0, a1, P.C, P.W, P.H, P.N, P.OW, P.OH, P.p, P.r, 0, wpack, P.nb * P.F,
                        P.Kf, c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, out, nullptr, nullptr, P.F, nob, nullptr, st);
    if (rc2 != QD_ERR_UNSUPPORTED) return rc2;
  }
  return run_conv(c.epi, c.nbk, a0, a1, P.C, P.W, P.H, P.N, P.OW, P.OH, P.p, P.r, 0, wpack, P.nb * P.F, P.Kf,
                  c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, out, nullptr, nullptr, P.F, nob, nullptr, st);
}

// the vectorised prologue for other callers (depth-wise path), bf16 only
void launch_bwd_prologue_vec(const Plan& P, const void* dy, const void* a, const void* b, void* D, float* part,
                             int split, cudaStream_t st) {
  long long rows_per = (P.Mout + split - 1) / split;
  bwd_prologue_vec_kernel<<<split, 256, 0, st>>>(P, (const bf16*)dy, (const bf16*)a, (const bf16*)b, (bf16*)D,
                                                 part, rows_per, 0, P.OH, P.OW, P.Jd);
  count_launch(st, "prologue");
}

__device__ float g_zero_bias[3 * 2048];  // zero-initialised at module load, never written

// rows of BN statistics the forward epilogue can write for P (0: the forward takes
// a path without them -- the caller then reduces y separately)
int tc_stat_rows(const Plan& P, int path) {
  if (P.kind != QD_KIND_CONV || P.s != 1 || (P.flags & QD_FLAG_TC_V1)) return 0;
  if (P.family != QD_FAM_PROPOSED && P.family != QD_FAM_T4) return 0;
  GemmCfg c = fprop_cfg(P);
  if (path == 1)
    return conv2_stat_rows(P.N, P.C, P.W, P.H, P.OW, P.OH, P.p, P.r, 0, c.nbk, c.nout, c.tiles_nn, P.F, c.nbias);
  if (path == 3)
    return conv2_stat_rows(P.N, P.C, P.W, P.H, P.OW, P.OH, P.p, P.r, 2, c.nbk, c.nout, c.tiles_nn, P.F, c.nbias);
  return 0;
}

int tc_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3], void* y, void* a,
               void* b, char* ws, const Workspace& L, cudaStream_t st, float* stats) {
  const void* a0 = x;
  const void* a1 = nullptr;
  // squared-input families: x * x into the workspace by one vectorised pass, the
  // GEMM reads it as its first K half. QD_XFS=1 (measured slower):
  // the conv2 kernels square x in their transform warps instead (C2Args::xf = 1)
  const bool xfs = P.sq && getenv("QD_XFS") && atoi(getenv("QD_XFS"));
  const C2Xform xsq{xfs ? 1 : 0, P.C, 0, x, nullptr, nullptr};
  auto square_x = [&]() {
    if (!P.sq) return;
    void* xs = ws + L.off_XS;
    launch_square(P, x, xs, st);
    a0 = xs;
  };
  if (P.sq == 2) a1 = x;
  if (P.sq && !xfs) square_x();
  const float* nb3[3] = {bias[0], bias[1], bias[2]};
  GemmCfg c = fprop_cfg(P);
  if (c.nbias == 0) nb3[0] = nb3[1] = nb3[2] = nullptr;
  if (P.family == QD_FAM_T2AND4) {
    // y = a b + c through the proposed epilogue with zero biases: a static zero
    // vector (no per-forward memset) when the layer is narrow enough
    thread_local float* zdev_[kMaxDev] = {};
    float*& zdev = zdev_[cur_device()];
    if (!zdev && cudaGetSymbolAddress((void**)&zdev, g_zero_bias) != cudaSuccess) {
      cudaGetLastError();
      zdev = nullptr;
    }
    float* z = (float*)(ws + L.off_ZB);
    if (zdev && 3 * P.F <= (int)(sizeof(g_zero_bias) / sizeof(float))) z = zdev;
    else cudaMemsetAsync(z, 0, (size_t)3 * P.F * 4, st);
    nb3[0] = z; nb3[1] = z + P.F; nb3[2] = z + 2 * P.F;
  }
  if (P.family == QD_FAM_T3) {
    // y = (Wa x)^2: the plain GEMM, then the square in place
    if (xfs) square_x();
    int rc = tc_fprop_plain(P, a0, a1, wpack, y, st);
    if (rc) return rc;
    launch_square_out(P, y, st);
    return check_launch("t3 forward");
  }
  if (tc_s2_direct(P)) {
    if (dev_skip("fprop")) return QD_OK;
    return run_conv(c.epi, c.nbk, a0, a1, P.C, P.W, P.H, P.N, P.OW, P.OH, P.p, P.r, 0, wpack, P.nb * P.F, P.Kf,
                    c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, y, a, b, P.F, nb3, nullptr, st, nullptr, 0, 2);
  }
  if (P.s == 2) {
    // stride-1 grid, epilogue keeps the even positions
    Plan P1 = stride1_plan(P);
    return run_conv2(c.epi, c.nbk, a0, a1, P.C, P.W, P.H, P.N, P1.OW, P1.OH, P.p, P.r, P.sq == 2 ? 1 : 0, wpack,
                     P.nb * P.F, P.Kf, c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, y, a, b, P.F, nb3, nullptr, st, 2,
                     nullptr, 0, 1, 0, nullptr, &xsq);
  }
  if (dev_skip("fprop")) return QD_OK;
  if (!(P.flags & QD_FLAG_TC_V1)) {
    int rc2 = run_conv2(c.epi, c.nbk, a0, a1, P.C, P.W, P.H, P.N, P.OW, P.OH, P.p, P.r, P.sq == 2 ? 1 : 0, wpack,
                        P.nb * P.F, P.Kf, c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, y, a, b, P.F, nb3, nullptr, st,
                        1, nullptr, 0, 1, 0, stats, &xsq);
    if (rc2 != QD_ERR_UNSUPPORTED) return rc2;
  }
  if (stats) return set_error(QD_ERR_UNSUPPORTED, "BN statistics: the conv2 forward does not fit this layer");
  if (xfs) square_x();
  return run_conv(c.epi, c.nbk, a0, a1, P.C, P.W, P.H, P.N, P.OW, P.OH, P.p, P.r, P.sq == 2 ? 1 : 0, wpack,
                  P.nb * P.F, P.Kf, c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, y, a, b, P.F, nb3, nullptr, st,
                  (float*)(ws + L.off_SK), L.sz_SK);
}

// side stream for work that can overlap the main chain (one per device/thread pair
// would be more general; the library drives one device per process)
// per (host thread, device): one side stream and its fork / join events, so
// concurrent callers never record into each other's events
struct SideState {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideState& side_state() {
  thread_local SideState s[kMaxDev];
  return s[cur_device()];
}
static cudaStream_t fork_side(cudaStream_t st) {
  SideState& s = side_state();
  if (!s.side) {
    if (cudaStreamCreateWithFlags(&s.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      s.side = nullptr;
      return nullptr;
    }
  }
  cudaEventRecord(s.fork, st);
  cudaStreamWaitEvent(s.side, s.fork, 0);
  return s.side;
}
static void join_side(cudaStream_t st, cudaStream_t side) {
  SideState& s = side_state();
  cudaEventRecord(s.join, side);
  cudaStreamWaitEvent(st, s.join, 0);
}

// one v1 wgrad product (x taps from x0 / x1 by K half, D) into `splits` fp32
// partial slots at `part`; single CTAs or CTA pairs per wgrad_v1_shape
static int run_wgrad_v1(const Plan& P, const void* x0, const void* x1, const void* D, float* part, int splits,
                        cudaStream_t st) {
  Box pb = choose_box(P.OW, P.OH, P.N, 64, true);
  CUtensorMap X0, X1, Dm;
  int rc;
  if ((rc = map_act(&X0, x0, P.C, P.W, P.H, P.N, pb.Wb, pb.Hb, pb.Nb, P.s))) return rc;
  if ((rc = map_act(&X1, x1 ? x1 : x0, P.C, P.W, P.H, P.N, pb.Wb, pb.Hb, pb.Nb, P.s))) return rc;
  if ((rc = map_act(&Dm, D, P.Jd, P.OW, P.OH, P.N, pb.Wb, pb.Hb, pb.Nb))) return rc;
  const WgShape sh = wgrad_v1_shape(P);
  WgArgs g;
  memset(&g, 0, sizeof(g));
  g.nkb = P.Kf / 64;
  g.mtiles = (g.nkb + 1) / 2;
  g.ntiles = (P.Jd / 64) / sh.nblk;
  g.splits = splits;
  g.pb_w = pb.Wb; g.pb_h = pb.Hb; g.pb_n = pb.Nb;
  g.pt_w = pb.tw; g.pt_h = pb.th; g.ptiles = pb.tw * pb.th * pb.tn;
  g.r = P.r; g.pad = P.p; g.cblks = P.C / 64; g.kb_half = P.K0 / 64;
  g.Jd = P.Jd; g.Kf = P.Kf;
  g.sstride = P.s;
  g.part = part;
  if (sh.pair) {
    if (sh.nblk == 4) return launch_wgrad_pair<4>(X0, X1, Dm, g, st);
    return launch_wgrad_pair<2>(X0, X1, Dm, g, st);
  }
  if (sh.nblk == 4) return launch_wgrad<4>(X0, X1, Dm, g, st);
  if (sh.nblk == 3) return launch_wgrad<3>(X0, X1, Dm, g, st);
  if (sh.nblk == 2) return launch_wgrad<2>(X0, X1, Dm, g, st);
  return launch_wgrad<1>(X0, X1, Dm, g, st);
}

int tc_backward(const Plan& P0, const void* x, const void* wpack, const void* a, const void* b, const void* dy,
                void* dx, float* const dW[3], float* const db[3], char* ws, const Workspace& L,
                cudaStream_t st) {
  // stride-2 layers: on their own grid when tc_s2_direct, else the GEMMs run on
  // the stride-1 grid over the zero-upsampled D
  const bool s2d = tc_s2_direct(P0);
  const bool up = P0.s == 2 && !s2d;
  const Plan P = up ? stride1_plan(P0) : P0;
  const bf16* wd = (const bf16*)wpack + pack_fprop_elems(P);
  const bool mat = caches_ab(P.family);
  const bf16* D = (const bf16*)dy;
  float* bpart = (float*)(ws + L.off_BS);
  cudaStream_t side = nullptr;
  // proposed, stride 1, both GEMMs on the v2 kernels: D holds only [g b, g a]
  // and the consumers read its third block (g itself) straight from dy
  const bool w3 = !(P.flags & QD_FLAG_TC_V1) && wgrad3_split(P) == L.wg_split;
  const bool w2 = !w3 && !(P.flags & QD_FLAG_TC_V1) && wgrad2_split(P) == L.wg_split;
  const bool dgiven = (P.flags & QD_FLAG_D_GIVEN) != 0;  // `dy` is D already (qd_bn_backward_D)
  bool d2 = P.family == QD_FAM_PROPOSED && !up && dW[0] && (w2 || w3) && !dgiven && !getenv("QD_NO_D2");
  if (d2 && dx) {
    GemmCfg c = dgrad_cfg(P);
    d2 = conv2_fits(P.N, P.Jd, P.OW, P.OH, P.W, P.H, P.r - 1 - P.p, P.r, 0, c.nbk, c.nout, c.tiles_nn, P.C, 0);
  }
  const int dsplit = d2 ? 2 * P.F / 64 : 0;
  int rc;
  // SM partition: the v3 wgrad runs on ~54% of the SM pairs (side stream) while
  // the dgrad runs on the rest, both persistent and concurrent -- their tails
  // (partial-store drain, last-tile imbalance) overlap instead of adding up.
  // 54% balances the two on the measured C2 step; QD_PART=K pins
  // K pairs, QD_NO_PART=1 runs them back to back on all SMs.
  int part = 0, dg_pairs = 0;
  if (w3 && dx && dW[0] && !P.sq && !getenv("QD_NO_PART") && !getenv("QD_BR2")) {
    const int per = wgrad3_pairs_per_split(P);
    const int total = L.wg_split * per;  // pairs the wgrad alone would fill
    // measured best: 54% of the pairs on the C2 step (32x32 images), 50% on the
    // ResNet 64@56 layers (287.5 vs 299.2 us at 37 vs 40 pairs); QD_PART pins
    const int pct = P.OH >= 48 ? 50 : 54;
    part = getenv("QD_PART") ? atoi(getenv("QD_PART")) : (total * pct / per + 50) / 100;
    dg_pairs = total - part * per;
    // one pair per split only: with several (wide C) the split granularity is too
    // coarse to balance the two (measured: 256x14 loses 15%)
    if (per != 1 || part < 1 || part >= L.wg_split || dg_pairs < total / 4) part = 0;
  }
  // QD_XFD=1 (measured slower): the dgrad forms its own D blocks
  // (dy * b, dy * a) in its transform warps (C2Args::xf = 2) and no longer waits
  // for the backward prologue, which then runs on the side stream ahead of the
  // wgrad, beside the dgrad
  const bool xfd = d2 && dx && part > 0 && P.kind == QD_KIND_CONV && getenv("QD_XFD") && atoi(getenv("QD_XFD"));
  if (xfd) {
    side = fork_side(st);
    if (!side) return set_error(QD_ERR_CUDA, "side stream");
  }
  cudaStream_t pst = xfd ? side : st;  // the prologue's stream
  bool wg_pdl = false;  // a PDL-launched v2/v3 wgrad immediately precedes the dgrad on `st`
  if (dgiven) {
    D = (const bf16*)dy;
  } else if (P.family == QD_FAM_T3) {
    // a = Wa x is recomputed into the D buffer, then D = 2 dy a in place
    // (on the stride-1 grid for stride 2 the prologue below upsamples it)
    bf16* Dw = (bf16*)(ws + L.off_D);
    if (up) return set_error(QD_ERR_UNSUPPORTED, "t3 stride 2 on the tcgen05 path");
    int rc0 = tc_fprop_plain(P0, x, nullptr, wpack, Dw, st);
    if (rc0) return rc0;
    launch_t3_prologue(P, dy, Dw, false, Dw, st);
    D = Dw;
  } else if (mat || up || (P.nbias && db[0])) {  // (bias sums only when asked for)
    long long rows = up ? P.Mout : P0.Mout;
    long long rows_per = (rows + L.bs_split - 1) / L.bs_split;
    bf16* Dw = (mat || up) ? (bf16*)(ws + L.off_D) : nullptr;
    if (!dev_skip("prologue")) launch_pdl(bwd_prologue_vec_kernel, dim3(L.bs_split), dim3(256), 0, pst, P0, (const bf16*)dy, (const bf16*)a,
               (const bf16*)b, Dw, bpart, rows_per, up ? 1 : 0, P.OH, P.OW, d2 ? 2 * P.F : P.Jd);
    count_launch(pst, "prologue");
    if (mat || up) D = Dw;
  }
  // v1 wgrad + fold on stream `ws_`, x operands chosen below
  bool v1_side = false;
  const void* v1_x0 = x;
  auto run_v1_wgrad_and_fold = [&](cudaStream_t ws_) -> int {
    int rc1 = run_wgrad_v1(P, v1_x0, x, D, (float*)(ws + L.off_WG), L.wg_split, ws_);
    if (rc1) return rc1;
    WSplits uni;
    memset(&uni, 0, sizeof(uni));
    launch_bwd_finish(P, (float*)(ws + L.off_WG), L.wg_split, uni, dW, bpart, L.bs_split, db, ws_);
    return QD_OK;
  };
  // ---- wgrad ----
  if (dW[0]) {
    const void* x0 = x;
    const void* x1 = x;
    if (P.sq) {
      void* xs = ws + L.off_XS;
      launch_square(P, x, xs, st);
      x0 = xs;
    }
    v1_x0 = x0;
    rc = QD_ERR_UNSUPPORTED;
    WSplits wsp;
    memset(&wsp, 0, sizeof(wsp));
    wg_pdl = false;
    // dev: QD_BR2=1 runs wgrad + fold on the side stream concurrently with the dgrad
    const bool br2 = (w2 || w3) && dx && !P.sq && getenv("QD_BR2") && atoi(getenv("QD_BR2"));
    cudaStream_t wst = st;
    if (br2 || part) {
      if (!side) side = fork_side(st);
      if (side) wst = side;
      else part = 0;
    }
    // partitioned (wgrad3 beside the dgrad): wgrad3 folds its own partials (grid
    // barrier + fixed-order sums, written transposed; C2 step 116 -> 111 us) --
    // no wsum / transpose launches behind it. Unpartitioned, the separate fold on
    // the side stream overlaps the dgrad instead. QD_W3_NOFOLD=1 forces the latter.
    bool fold3 = false;
    if (w3) {
      const int ns = part ? part : L.wg_split;
      bool al16 = true;
      for (int i = 0; i < 3; ++i) al16 = al16 && ((uintptr_t)dW[i] % 16 == 0);
      fold3 = part > 0 && al16 && P.kind == QD_KIND_CONV &&
              !(getenv("QD_W3_NOFOLD") && atoi(getenv("QD_W3_NOFOLD")));
      bool folded = false;
      rc = run_wgrad3(P, x0, P.sq == 2 ? x1 : nullptr, D, (float*)(ws + L.off_WG), ns, wst, dy, dsplit,
                      fold3 ? dW : nullptr, bpart, L.bs_split, db, &folded);
      fold3 = folded;  // the driver may refuse the cooperative launch: then fold separately
      wsp.pp = (P.r * P.r + 1) / 2;  // every tap in every split slot
      wsp.ng = 1;
      wsp.s[0] = ns;
    } else if (w2) {
      rc = run_wgrad2(P, x0, P.sq == 2 ? x1 : nullptr, D, (float*)(ws + L.off_WG), L.wg_split, wst, dy, dsplit);
      wsp = wgrad2_splits(P);
    }
    if (rc == QD_OK) wg_pdl = (w2 || w3) && pdl_enabled() && wst == st;
    if (rc == QD_OK) {
      // the memory-bound fold overlaps the (smem-bound) dgrad: it runs on the side
      // stream, forked after wgrad and joined before this call returns
      // (QD_FOLD_MAIN=1: on `st`, for per-kernel timing with one stream of marks)
      const bool fold_main = getenv("QD_FOLD_MAIN") && atoi(getenv("QD_FOLD_MAIN"));
      if (!fold3) {
        if (wst == st && !fold_main) side = fork_side(st);
        launch_bwd_finish(P, (float*)(ws + L.off_WG), L.wg_split, wsp, dW, bpart, L.bs_split, db,
                          side ? side : st);
      }
    } else if (rc != QD_ERR_UNSUPPORTED) {
      return rc;
    } else {
      // v1 wgrad + its fold: with a dgrad, on the side stream AFTER the dgrad is
      // enqueued (below), so the persistent dgrad takes its SMs first and the
      // wgrad's CTAs fill the ones it leaves (512@7: 98 of 148) and then the rest;
      // QD_V1_SERIAL=1: wgrad, fold, dgrad in order on `st`
      v1_side = dx && !(getenv("QD_V1_SERIAL") && atoi(getenv("QD_V1_SERIAL")));
      if (v1_side && !side) side = fork_side(st);
      if (!side) v1_side = false;
      if (!v1_side) {
        rc = run_v1_wgrad_and_fold(st);
        if (rc) return rc;
      }
    }
  } else if (db[0] && (mat || P.nbias)) {
    launch_bias_finish(P, bpart, L.bs_split, db, st);
  }
  if (up && dx && (P.flags & QD_FLAG_TC_V1)) return set_error(QD_ERR_UNSUPPORTED, "stride 2 needs conv2");
  // ---- dgrad (stride 1: a conv of D with the flipped packed weights) ----
  if (dx) {
    const float* nob[3] = {nullptr, nullptr, nullptr};
    int pad_eff = P.r - 1 - P.p;
    GemmCfg c = dgrad_cfg(P);
    const void* xr = P.sq ? x : nullptr;
    rc = QD_ERR_UNSUPPORTED;
    if (part) set_conv2_cap(dg_pairs);
    if (dev_skip("dgrad")) rc = QD_OK;
    else if (s2d)
      rc = run_conv(c.epi, c.nbk, D, nullptr, P.Jd, P.OW, P.OH, P.N, (P.W + 1) / 2, (P.H + 1) / 2, pad_eff, P.r, 0,
                    wd, P.Cd, P.Kd, c.b_rs_tile, c.b_rs_blk, c.tiles_nn, c.out_c_tile, dx, nullptr, nullptr, P.C,
                    nob, xr, st, nullptr, 0, 1, 1, P.H, P.W);
    else if (!(P.flags & QD_FLAG_TC_V1))
      // D is complete once the (PDL-launched) v2/v3 wgrad is running, and nothing
      // the dgrad reads is written by it: the dgrad need not wait for the wgrad
    {
      C2Xform xfm{xfd ? 2 : 0, P.F, P.F / 64, dy, a, b};
      rc = run_conv2(c.epi, c.nbk, D, nullptr, P.Jd, P.OW, P.OH, P.N, P.W, P.H, pad_eff, P.r, 0, wd, P.Cd, P.Kd,
                     c.b_rs_tile, c.b_rs_blk, c.tiles_nn, c.out_c_tile, dx, nullptr, nullptr, P.C, nob, xr, st, 1,
                     dy, dsplit, (wg_pdl && !xfd) ? 0 : 1, 0, nullptr, &xfm);
    }
    if (part) set_conv2_cap(0);
    if (d2 && rc == QD_ERR_UNSUPPORTED) return set_error(QD_ERR_UNSUPPORTED, "dgrad conv2 plan changed");
    if (rc == QD_ERR_UNSUPPORTED && !up)
      rc = run_conv(c.epi, c.nbk, D, nullptr, P.Jd, P.OW, P.OH, P.N, P.W, P.H, pad_eff, P.r, 0, wd, P.Cd, P.Kd,
                    c.b_rs_tile, c.b_rs_blk, c.tiles_nn, c.out_c_tile, dx, nullptr, nullptr, P.C, nob, xr, st,
                    (float*)(ws + L.off_SK), L.sz_SK);
    if (rc) return rc;
  }
  if (v1_side) {
    rc = run_v1_wgrad_and_fold(side);
    if (rc) return rc;
  }
  if (side) join_side(st, side);
  return check_launch("tc backward");
}

// ===========================================================================
// fp32 layers on the tensor cores (device path 3; kernels in qd_x3.cu): the
// v1 conv GEMM over the K-tripled split operands, raw fp32 accumulators, fp32
// epilogue passes; three v1 wgrad products into one fixed-order fold
// ===========================================================================
bool x3_supported(const Plan& P, unsigned flags) {
  if ((flags & QD_FLAG_FORCE_SIMT) || P.dtype != QD_F32) return false;
  const char* e = getenv("QD_NO_X3");  // read per call: tests switch the exact FFMA path on and off
  if (e && atoi(e)) return false;
  if (P.family != QD_FAM_PROPOSED && P.family != QD_FAM_T4 && P.family != QD_FAM_FIRST_ORDER) return false;
  if (P.kind != QD_KIND_FC && P.kind != QD_KIND_CONV) return false;
  if (P.s != 1 || P.C % 64 || P.F % 64 || P.OH < 1 || P.OW < 1) return false;
  return init_driver();
}

static int x3_fprop_split(const Plan& P) {
  GemmCfg c = fprop_cfg(P);
  Box bx = choose_box(P.OW, P.OH, P.N, 128, false);
  const long long tiles = (long long)bx.tw * bx.th * bx.tn * c.tiles_nn;
  const int KB = 3 * P.r * P.r * (P.C / 64);
  int S = conv_ksplit(tiles, KB);
  if (S > 1) {
    const int per = (KB + S - 1) / S;
    S = (KB + per - 1) / per;
  }
  return S;
}
static int x3_dgrad_split(const Plan& P) {
  GemmCfg c = dgrad_cfg(P);
  Box bx = choose_box(P.W, P.H, P.N, 128, false);
  const long long tiles = (long long)bx.tw * bx.th * bx.tn * c.tiles_nn;
  const int KB = 3 * P.r * P.r * (P.Jd / 64);
  int S = conv_ksplit(tiles, KB);
  if (S > 1) {
    const int per = (KB + S - 1) / S;
    S = (KB + per - 1) / per;
  }
  return S;
}
size_t x3_raw_bytes(const Plan& P) {
  GemmCfg c = fprop_cfg(P);
  const size_t f = (size_t)x3_fprop_split(P) * P.Mout * c.tiles_nn * c.nbk * 64 * 4;
  const int sd = x3_dgrad_split(P);
  const size_t d = sd > 1 ? (size_t)sd * P.Min * P.C * 4 : 0;
  return f > d ? f : d;
}
int x3_wgrad_split(const Plan& P) {
  if (!(P.flags & QD_FLAG_TC_V1)) {
    const int s3 = wgrad3_split(P);  // r = 3 on CTA pairs (one product per launch, no in-kernel fold)
    if (s3 > 0) return s3;
  }
  return wgrad_v1_shape(P).S;
}

int x3_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3], void* y, void* a,
               void* b, char* ws, const Workspace& L, cudaStream_t st, float* stats) {
  bf16* xh = (bf16*)(ws + L.off_XS);
  bf16* xl = xh + (size_t)P.Min * P.C;
  launch_x3_split((const float*)x, xh, xl, P.Min * P.C, st);
  GemmCfg c = fprop_cfg(P);
  const float* nob[3] = {nullptr, nullptr, nullptr};
  const float* bz[3] = {bias[0], bias[1], bias[2]};
  if (c.nbias == 0) bz[0] = bz[1] = bz[2] = nullptr;
  if (!(P.flags & QD_FLAG_TC_V1) && P.kind == QD_KIND_CONV) {
    // CTA-pair halo kernel with the fp32 epilogue in registers: y, a, b written
    // once, no raw accumulator pass
    int rc2 = run_conv2(c.epi, c.nbk, xh, xl, P.C, P.W, P.H, P.N, P.OW, P.OH, P.p, P.r, 2, wpack, P.nb * P.F,
                        3 * P.Kf, c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, y, a, b, P.F, bz, nullptr, st, 1,
                        nullptr, 0, 1, 1, stats);
    if (rc2 != QD_ERR_UNSUPPORTED) return rc2 ? rc2 : check_launch("x3 forward");
  }
  if (stats) return set_error(QD_ERR_UNSUPPORTED, "BN statistics: the conv2 forward does not fit this layer");
  int S = 1;
  int rc = run_conv(c.epi, c.nbk, xh, xl, P.C, P.W, P.H, P.N, P.OW, P.OH, P.p, P.r, 2, wpack, P.nb * P.F, 3 * P.Kf,
                    c.b_rs_tile, 64, c.tiles_nn, c.out_c_tile, y, a, b, P.F, nob, nullptr, st,
                    (float*)(ws + L.off_P), L.sz_P, 1, 0, 0, 0, 1, &S);
  if (rc) return rc;
  launch_x3_fprop_finish((const float*)(ws + L.off_P), S, P.Mout, c.tiles_nn * c.nbk * 64, P.F, P.nb,
                         c.epi == EPI_PROPOSED ? 0 : (c.epi == EPI_T4 ? 1 : 2), (float*)y, (float*)a, (float*)b, bz,
                         st);
  return check_launch("x3 forward");
}

int x3_backward(const Plan& P, const void* x, const void* wpack, const void* a, const void* b, const void* dy,
                void* dx, float* const dW[3], float* const db[3], char* ws, const Workspace& L, cudaStream_t st) {
  const bf16* wd = (const bf16*)wpack + 3 * pack_fprop_elems(P);
  bf16* Dh = (bf16*)(ws + L.off_D);
  bf16* Dl = Dh + (size_t)P.Mout * P.Jd;
  bf16* xh = (bf16*)(ws + L.off_XS);
  bf16* xl = xh + (size_t)P.Min * P.C;
  float* bpart = (float*)(ws + L.off_BS);
  const bool dgiven = (P.flags & QD_FLAG_D_GIVEN) != 0;
  // the HBM-bound passes first, back to back: x for the weight products, then D
  if (dW[0]) launch_x3_split((const float*)x, xh, xl, P.Min * P.C, st);
  if (dgiven) {
    // `dy` is the fp32 operand D (qd_bn_backward_D formed it and the bias grads)
    launch_x3_split((const float*)dy, Dh, Dl, P.Mout * P.Jd, st);
  } else {
    const bool need_part = P.nbias && db[0];
    launch_x3_prologue(P, (const float*)dy, (const float*)a, (const float*)b, Dh, Dl, need_part ? bpart : nullptr,
                       L.bs_split, st);
  }
  int rc;
  const GemmCfg dc = dgrad_cfg(P);
  const bool c2d = dx && !(P.flags & QD_FLAG_TC_V1) && P.kind == QD_KIND_CONV &&
                   conv2_fits(P.N, P.Jd, P.OW, P.OH, P.W, P.H, P.r - 1 - P.p, P.r, 2, dc.nbk, dc.nout, dc.tiles_nn,
                              P.C, 0);
  const bool w3 = dW[0] && !(P.flags & QD_FLAG_TC_V1) && wgrad3_split(P) == L.wg_split &&
                  wgrad3_pairs_per_split(P) == 1;
  // SM partition as in the bf16 backward: the three wgrad3 products (and their fold)
  // on ~half of the pairs on the side stream, the persistent dgrad capped to the rest
  int S = L.wg_split, dg_pairs = 0;
  if (w3 && c2d && !getenv("QD_NO_PART")) {
    // measured on C2-fp32 (tools/x3_part_sweep.sh): 39 of 74 pairs with the grouped B stream
    // of the 64-channel dgrad (254 vs 222 TFLOP/s at the old 26, the best for the per-tap ring)
    const int pct = P.C == 64 ? 53 : 35;
    const int part = getenv("QD_X3_PART") ? atoi(getenv("QD_X3_PART")) : (L.wg_split * pct + 50) / 100;
    if (part >= 1 && part < L.wg_split) {
      S = part;
      dg_pairs = L.wg_split - part;
    }
  }
  // the weight-gradient chain (three products, fold) runs on the side stream beside
  // the dgrad: both only read D, x and the packed weights
  cudaStream_t side = (dW[0] && dx) ? fork_side(st) : nullptr;
  cudaStream_t wst = side ? side : st;
  if (dW[0]) {
    float* part = (float*)(ws + L.off_WG);
    const size_t slot = (size_t)P.Jd * P.Kf;
    const bf16* xa[3] = {xh, xh, xl};
    const bf16* da[3] = {Dh, Dl, Dh};
    for (int i = 0; i < 3; ++i) {
      float* pi = part + (size_t)i * S * slot;  // 3 S contiguous slots
      rc = w3 ? run_wgrad3(P, xa[i], nullptr, da[i], pi, S, wst) : run_wgrad_v1(P, xa[i], nullptr, da[i], pi, S, wst);
      if (rc) return rc;
    }
    WSplits uni;
    memset(&uni, 0, sizeof(uni));
    float* const nodb[3] = {nullptr, nullptr, nullptr};
    launch_bwd_finish(P, part, 3 * S, uni, dW, bpart, L.bs_split, (dgiven || !P.nbias) ? nodb : db, wst);
  } else if (!dgiven && db[0] && P.nbias) {
    launch_bias_finish(P, bpart, L.bs_split, db, st);
  }
  if (dx) {
    const float* nob[3] = {nullptr, nullptr, nullptr};
    rc = QD_ERR_UNSUPPORTED;
    if (c2d) {
      if (dg_pairs) set_conv2_cap(dg_pairs);
      rc = run_conv2(dc.epi, dc.nbk, Dh, Dl, P.Jd, P.OW, P.OH, P.N, P.W, P.H, P.r - 1 - P.p, P.r, 2, wd, P.Cd,
                     3 * P.Kd, dc.b_rs_tile, dc.b_rs_blk, dc.tiles_nn, dc.out_c_tile, dx, nullptr, nullptr, P.C, nob,
                     nullptr, st, 1, nullptr, 0, 1, 1);
      set_conv2_cap(0);
    }
    if (rc == QD_ERR_UNSUPPORTED) {
      int Sd = 1;
      rc = run_conv(dc.epi, dc.nbk, Dh, Dl, P.Jd, P.OW, P.OH, P.N, P.W, P.H, P.r - 1 - P.p, P.r, 2, wd, P.Cd,
                    3 * P.Kd, dc.b_rs_tile, dc.b_rs_blk, dc.tiles_nn, dc.out_c_tile, dx, nullptr, nullptr, P.C, nob,
                    nullptr, st, (float*)(ws + L.off_P), L.sz_P, 1, 0, 0, 0, 2, &Sd);
      if (rc) return rc;
      if (Sd > 1) launch_x3_sum((const float*)(ws + L.off_P), Sd, P.Min * P.C, (float*)dx, st);
    } else if (rc) {
      return rc;
    }
  }
  if (side) join_side(st, side);
  return check_launch("x3 backward");
}

}  // namespace qd
