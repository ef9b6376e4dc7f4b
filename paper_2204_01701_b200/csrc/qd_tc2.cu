// K1/K3 v2: stride-1 implicit-GEMM conv on CTA pairs (cta_group::2) with
// halo reuse. Used for fprop (A = x) and dgrad (A = D, flipped weights) when
// r >= 2, channels are multiples of 64 and the image is wide enough.
//
// Tiling. Each image's output grid is walked in the "padded flat" index
// q = oh * Wp + ow (Wp = W + 2 pe): output (oh, ow) reads padded input rows
// q + ey * Wp + ex, so a tile of 128 consecutive q needs ONE halo box of whole
// padded rows (4-D TMA box {64 ch, Wp, HR, 1}, OOB zero fill = the padding),
// and every filter tap is the same smem tile read through a descriptor
// shifted by ey*Wp + ex rows -- SWIZZLE_128B is address based on sm_100a
// (profiles/r1_probe_sw128_row_shift.log), so row shifts need no re-layout.
// The last r-1 columns of each padded row are junk outputs and are not stored.
//
// Pairs. The two CTAs of a cluster take the same tile index of images 2p and
// 2p+1 (identical halo geometry, so one descriptor address serves both) and
// issue M = 256 MMAs: CTA r holds A rows 128r.. and N rows [r N/2, (r+1) N/2)
// of B (profiles/r1_probe_2cta.log). When half of B fits in smem (C = F = 64:
// 108 KB) it is loaded once per CTA and stays resident; otherwise B streams
// per (tap, channel block) through a ring.
//
// Epilogue. Per warp, TMEM rows -> registers (a*b + c + bias, or 2 x acc) ->
// swizzled 4 KB warp staging -> 16-B coalesced global stores that skip the
// junk columns; TMEM accumulators are double-buffered so this overlaps the
// next tile's main loop.
#include <cudaTypedefs.h>
#include <atomic>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "qd_kernels.h"
#include "qd_ptx.cuh"

namespace qd {

enum { E2_PROPOSED = 0, E2_T4 = 1, E2_PLAIN = 2, E2_SQ = 3 };

struct C2Args {
  int N, Cin, Win, Hin;
  int OHg, OWg;
  int ss, OHo, OWo;  // output subsampling (stride-2 conv = stride-1 grid, even positions)
  int pe, r, Wp, HR;
  int T_img, tiles_nn, total;
  int cblks, ablocks, KBtot;
  int resident;
  int b_rs_tile, b_rs_blk, b_contig;
  int Cout, out_c_tile;
  uint32_t halo_bytes, halo_tx, b_stage_bytes;
  int b_slots, a_slots, stg_tiles;
  int b_group;  // streamed B: taps per ring slot (1, or r*r = one barrier per channel block)
  int nbias;  // bias vectors staged in smem (3 proposed, 1 first_order, else 0), Cout floats each
  int direct;  // epilogue stores straight from registers (no smem staging)
  int pf;      // L2 prefetch distance of the A halo boxes, in this cluster's tiles (0 = off)
  int pdl_wait;  // 1: wait for the previous kernel's outputs (PDL) before the first global read
  ptx::FastDiv fd_nn, fd_T, fd_Wp;  // tiles_nn, T_img, Wp
  int csplit;  // A channel blocks >= csplit come from the second map (dgrad: D = [g b, g a] then dy)
  int dual;    // extra K segments of A: 1 = [x*x | x] (segment 1 from the second map), 2 = the fp32
               // split [hi | hi | lo] (segment 2 from the second map)
  int f32out;  // fp32 outputs stored straight from registers (the fp32 split path)
  // BN statistics of y (the batch norm that follows the layer, bn.QuadConvBN):
  // per (tile, CTA, 32-row warp) and channel, the mean and M2 of the stored y
  // values of the tile's valid pixels; stats = [mean: rows x Cout][M2: rows x
  // Cout][count: rows], merged in a fixed order by bn_merge_finalize
  float* stats;
  int stat_rows;
  int dbg;  // QD_DEBUG bits (dev only): 1 = epilogue only releases TMEM, 2 = no MMA
  unsigned long long* trace;  // QD_TRACE (dev only): per-role clock64 timeline of cluster 0
  const float* bias0;
  const float* bias1;
  const float* bias2;
  bf16* out0;
  bf16* out1;
  bf16* out2;
  const bf16* xres;
  // operand transform (XF kernels): A halo slots computed by the transform warps
  // from global tensors instead of TMA-loaded. xf = 1: x * x for the blocks of the
  // first K half (squared-input families, neurons.py:255-256); xf = 2: the dgrad's
  // D blocks cb < csplit, dy * b (block cb < xf_fb) and dy * a (neurons.py:437-444),
  // bit-identical to the backward prologue's bf16(dy * b) / bf16(dy * a)
  int xf, xf_cs, xf_fb;  // mode; channels of the source tensors; F / 64
  const bf16* xf_x;      // x (xf 1) or dy (xf 2)
  const bf16* xf_a;
  const bf16* xf_b;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
namespace c2 {
// dev-only timeline: slot = (role * 64 + tile) * 16 + event, CTA 0 only
#define C2_TRACE(role, tile, ev)                                                                  \
  do {                                                                                            \
    if (g.trace && blockIdx.x == 0 && (tile) < 64)                                                \
      g.trace[((role) * 64 + (tile)) * 16 + (ev)] = (unsigned long long)clock64();                \
  } while (0)
// same slots, written by CTA `blk` (dev only)
#define C2_TRACE_B(blk, role, tile, ev)                                                           \
  do {                                                                                            \
    if (g.trace && blockIdx.x == (blk) && (tile) < 64)                                            \
      g.trace[((role) * 64 + (tile)) * 16 + (ev)] = (unsigned long long)clock64();                \
  } while (0)
using ptx::cluster_rank;
using ptx::cluster_sync;
using ptx::peer0;
using ptx::tma4_cg2;
using ptx::tma2_cg2;
using ptx::mma_cg2;
using ptx::commit_mc;
using ptx::arrive_remote;
// L2 prefetch of a future box (fire and forget; the later load then hits L2)
__device__ __forceinline__ void tma4_prefetch(const CUtensorMap* m, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(m), "r"(c0), "r"(c1),
               "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// 16 values (channels 16j..16j+15) of warp-local row `row` into a 32x128 B
// staging tile, 16-B chunk q stored at q ^ (row & 7) (bank-conflict free)
__device__ __forceinline__ void stage16(uint8_t* tile, int row, int j, const float* v) {
  uint4 lo, hi;
  lo.x = pack2(v[0], v[1]);   lo.y = pack2(v[2], v[3]);   lo.z = pack2(v[4], v[5]);   lo.w = pack2(v[6], v[7]);
  hi.x = pack2(v[8], v[9]);   hi.y = pack2(v[10], v[11]); hi.z = pack2(v[12], v[13]); hi.w = pack2(v[14], v[15]);
  uint8_t* rp = tile + row * 128;
  *reinterpret_cast<uint4*>(rp + (((2 * j) ^ (row & 7)) << 4)) = lo;
  *reinterpret_cast<uint4*>(rp + (((2 * j + 1) ^ (row & 7)) << 4)) = hi;
}
}  // namespace c2

// 16 packed bf16 (channels 16j..16j+15) into a 32-row staging tile of RB-byte rows
// (RB = 2 x channels per warp); chunk c of row r at c ^ ((r / (128/RB)) & (RB/16-1)),
// conflict free for the row-per-lane writes and the lanes-per-row reads below
template <int RB>
__device__ __forceinline__ void c2_stage_rb(uint8_t* tile, int row, int j, const uint4& lo, const uint4& hi) {
  constexpr int CH = RB / 16, RPL = 128 / RB;
  uint8_t* rp = tile + row * RB;
  const int f = (row / RPL) & (CH - 1);
  *reinterpret_cast<uint4*>(rp + (((2 * j) ^ f) << 4)) = lo;
  *reinterpret_cast<uint4*>(rp + (((2 * j + 1) ^ f) << 4)) = hi;
}
template <int RB>
__device__ __forceinline__ void c2_store_rb(const C2Args& g, const uint8_t* st, bf16* dst, int ch, int pix,
                                            int lane) {
  constexpr int CH = RB / 16, RPL = 128 / RB, RPI = 32 / CH;  // chunks per row, rows per instr
#pragma unroll
  for (int i = 0; i < 32 / RPI; ++i) {
    const int Rw = RPI * i + lane / CH, c = lane % CH;
    const int rp = __shfl_sync(0xffffffffu, pix, Rw);
    uint4 val = *reinterpret_cast<const uint4*>(st + Rw * RB + ((c ^ ((Rw / RPL) & (CH - 1))) << 4));
    if (rp >= 0) *reinterpret_cast<uint4*>(dst + (size_t)rp * g.Cout + ch + c * 8) = val;
  }
}
// store pass with the per-row element offsets (pixel * Cout + channel chunk, -1 =
// skip) computed once per tile for the 32/RPI rows this lane stores
template <int RB>
__device__ __forceinline__ void c2_store_rb_pre(const uint8_t* st, bf16* dst, const long long* roff, int lane) {
  constexpr int CH = RB / 16, RPL = 128 / RB, RPI = 32 / CH;
#pragma unroll
  for (int i = 0; i < 32 / RPI; ++i) {
    const int Rw = RPI * i + lane / CH, c = lane % CH;
    uint4 val = *reinterpret_cast<const uint4*>(st + Rw * RB + ((c ^ ((Rw / RPL) & (CH - 1))) << 4));
    if (roff[i] >= 0) *reinterpret_cast<uint4*>(dst + roff[i]) = val;
  }
}
// sum over the warp's 32 lanes of v[c] for 32 channels at once: recursive halving
// (each lane gives away the half of its vector it does not keep: 16+8+4+2+1
// shuffles), after which lane c holds channel c's sum
__device__ __forceinline__ float c2_lane_sums32(float (&v)[32], int lane) {
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool up = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? v[i] : v[i + half];
      const float keep = up ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  return v[0];
}

__device__ __forceinline__ void c2_pack16(const float* v, uint4& lo, uint4& hi) {
  lo = make_uint4(c2::pack2(v[0], v[1]), c2::pack2(v[2], v[3]), c2::pack2(v[4], v[5]), c2::pack2(v[6], v[7]));
  hi = make_uint4(c2::pack2(v[8], v[9]), c2::pack2(v[10], v[11]), c2::pack2(v[12], v[13]), c2::pack2(v[14], v[15]));
}

// coalesced store of one 32 x 128 B warp staging tile: 4 rows (512 B) per instruction
template <int EPI>
__device__ __forceinline__ void c2_store_pass(const C2Args& g, const uint8_t* st, int o, int c_base, int pix,
                                              int lane) {
  bf16* dst = (EPI == E2_PROPOSED || EPI == E2_T4) ? (o == 0 ? g.out0 : (o == 1 ? g.out1 : g.out2)) : g.out0;
  const int ch = (EPI == E2_PLAIN) ? c_base + o * 64 : c_base;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int Rw = 4 * i + (lane >> 3), c = lane & 7;
    int rp = __shfl_sync(0xffffffffu, pix, Rw);
    uint4 val = *reinterpret_cast<const uint4*>(st + Rw * 128 + ((c ^ (Rw & 7)) << 4));
    if (rp >= 0) *reinterpret_cast<uint4*>(dst + (size_t)rp * g.Cout + ch + c * 8) = val;
  }
}

#ifndef C2_EPW
#define C2_EPW 2
#endif

// transform warps' slot wait: polls with a back-off so the spinning warps leave
// the issue slots to the MMA warp on their sub-partition
__device__ __forceinline__ void c2_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = ptx::smem_u32(bar);
  while (!ptx::mbar_try_wait(addr, parity)) __nanosleep(200);
}
template <int EPI, int NB, int XF = 0>
struct C2Threads {
  static constexpr int NPASS = (EPI == E2_PROPOSED || EPI == E2_T4) ? 3 : (EPI == E2_PLAIN ? NB : 1);
  // proposed / t4: C2_EPW epilogue warpgroups, each owning 64 / C2_EPW channels of y, a, b
  static constexpr int NEPI = NPASS == 3 ? 4 * C2_EPW : 4;
  // operand-transform warps (XF kernels): 8 beside one epilogue warpgroup, else 4
  static constexpr int XW = XF ? (NEPI == 4 ? 8 : 4) : 0;
  static constexpr int THREADS = 128 + NEPI * 32 + XW * 32;
};

// release arrive on a (possibly remote) cluster barrier: publishes this warp's
// shared-memory writes (after fence.proxy.async) to the MMA that waits on it
// (CTA-scope release, as the usual 2-SM producer pattern: a cluster-scope release
// compiles to MEMBAR.ALL.GPU + ERRBAR per arrival, profiled)
__device__ __forceinline__ void c2_arrive_release(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ uint4 c2_bf16_mul(uint4 u, uint4 v) {
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
  const __nv_bfloat162* k = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 a = __bfloat1622float2(h[e]), b = __bfloat1622float2(k[e]);
    h[e] = __floats2bfloat162_rn(a.x * b.x, a.y * b.y);
  }
  return u;
}

template <int EPI, int NB, int R, int XF = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(C2Threads<EPI, NB, XF>::THREADS, 1)
    conv2_kernel(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
                 const __grid_constant__ CUtensorMap mB, const C2Args g) {
  // output "passes": proposed/t4 write y, a, b; plain writes NB 64-channel blocks
  constexpr int NPASS = C2Threads<EPI, NB, XF>::NPASS;
  constexpr int NEPI = C2Threads<EPI, NB, XF>::NEPI;
  constexpr int XW = C2Threads<EPI, NB, XF>::XW;
  constexpr int ACC = NB * 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sHalo = sm;
  uint8_t* sB = sHalo + g.a_slots * g.halo_bytes;
  uint8_t* sStg = sB + g.b_slots * g.b_group * g.b_stage_bytes;
  float* sBias = (float*)(sStg + 4 * g.stg_tiles * 4096);
  uint64_t* afull = (uint64_t*)(sBias + g.nbias * g.Cout);
  uint64_t* aempty = afull + 4;
  uint64_t* tfull = aempty + 4;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres = tempty + 2;
  uint64_t* bfull = bres + 1;
  uint64_t* bempty = bfull + g.b_slots;
  uint32_t* tslot = (uint32_t*)(bempty + g.b_slots);

  if (g.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    g.trace[4096 + 2 * blockIdx.x] = gtimer();
    g.trace[6144 + 2 * blockIdx.x] = clock64();
  }
  const uint32_t rank = c2::cluster_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int r = R > 0 ? R : g.r;
  const int rr = r * r;

  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&mA0);
    ptx::prefetch_tmap(&mA1);
    ptx::prefetch_tmap(&mB);
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&afull[i], 1 + 2 * XW);  // XF: every transform warp of both CTAs arrives per slot use
      ptx::mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 2 * NEPI);
    }
    ptx::mbar_init(bres, 1);
    for (int i = 0; i < g.b_slots; ++i) {
      ptx::mbar_init(&bfull[i], 1);
      ptx::mbar_init(&bempty[i], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  ptx::tc_fence_before();
  c2::cluster_sync();
  ptx::tc_fence_after();
  if (g.pdl_wait) ptx::pdl_wait();  // before any read of the previous kernel's outputs
  ptx::pdl_launch();                 // the next kernel's CTAs may take SMs as ours retire
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ===== TMA producer (whole warp loops, one elected lane issues; both CTAs,
    // completions land on CTA0's barriers) =====
    const int half_rows = NB * 32;
    const bool leader = ptx::elect_one();
    auto brow = [&](int j) {
      return g.b_contig ? j * g.b_rs_tile + (int)rank * half_rows : j * g.b_rs_tile + (int)rank * g.b_rs_blk;
    };
    if (g.resident && leader) {
      if (rank == 0) ptx::mbar_arrive_expect_tx(bres, 2u * g.KBtot * g.b_stage_bytes);
      for (int kb = 0; kb < g.KBtot; ++kb)
        c2::tma2_cg2(&mB, c2::peer0(bres), sB + kb * g.b_stage_bytes, kb * 64, brow(0));
    }
    int as = 0, bs = 0;
    uint32_t aph = 0, bph = 0;
    int it = 0;
    for (int w = cluster; w < g.total; w += nclusters, ++it) {
      const int rest = ptx::fdiv(w, g.fd_nn), j = w - rest * g.tiles_nn;
      const int p = ptx::fdiv(rest, g.fd_T), t = rest - p * g.T_img;
      int n = 2 * p + (int)rank;
      int hq_lo = ptx::fdiv(128 * t, g.fd_Wp);
      for (int ab = 0; ab < g.ablocks; ++ab) {
        int half = ab / g.cblks, cb = ab % g.cblks;
        if (leader) C2_TRACE(0, it, 2 * ab);
        if (leader) C2_TRACE_B(1, 0, it, 8 + 2 * ab);
        ptx::mbar_wait(&aempty[as], aph ^ 1);
        const bool xblk = XF && (g.xf == 1 ? half == 0 : (g.xf == 2 && cb < g.csplit));  // filled by the transform warps
        if (xblk) {
          if (leader && rank == 0) ptx::mbar_arrive(&afull[as]);
        } else if (leader) {
          C2_TRACE(0, it, 2 * ab + 1);
          C2_TRACE_B(1, 0, it, 9 + 2 * ab);
          if (rank == 0) ptx::mbar_arrive_expect_tx(&afull[as], 2u * g.halo_tx);
          const bool tail = g.csplit && cb >= g.csplit;
          const bool second = (half > 0 && half == g.dual) || tail;
          c2::tma4_cg2(second ? &mA1 : &mA0, c2::peer0(&afull[as]), sHalo + as * g.halo_bytes,
                       (tail ? cb - g.csplit : cb) * 64, -g.pe, hq_lo - g.pe, n);
          if (ab == 0) C2_TRACE(0, it, 7);
          const int wf = w + g.pf * nclusters;
          if (g.pf && wf < g.total) {
            const int rf = wf / g.tiles_nn;
            const int tf = rf % g.T_img, nf = 2 * (rf / g.T_img) + (int)rank;
            if (nf < g.N)
              c2::tma4_prefetch(second ? &mA1 : &mA0, (tail ? cb - g.csplit : cb) * 64, -g.pe,
                                (128 * tf) / g.Wp - g.pe, nf);
          }
        }
        if (++as == g.a_slots) { as = 0; aph ^= 1; }
        if (!g.resident && g.b_group > 1) {
          // all taps of this channel block on one barrier (one wait / commit per block on the MMA side)
          ptx::mbar_wait(&bempty[bs], bph ^ 1);
          if (leader) {
            if (rank == 0) ptx::mbar_arrive_expect_tx(&bfull[bs], 2u * rr * g.b_stage_bytes);
            for (int tap = 0; tap < rr; ++tap)
              c2::tma2_cg2(&mB, c2::peer0(&bfull[bs]), sB + (bs * rr + tap) * g.b_stage_bytes,
                           ((half * rr + tap) * g.cblks + cb) * 64, brow(j));
          }
          if (++bs == g.b_slots) { bs = 0; bph ^= 1; }
        } else if (!g.resident) {
          for (int tap = 0; tap < rr; ++tap) {
            int kbi = (half * rr + tap) * g.cblks + cb;
            ptx::mbar_wait(&bempty[bs], bph ^ 1);
            if (leader) {
              if (rank == 0) ptx::mbar_arrive_expect_tx(&bfull[bs], 2u * g.b_stage_bytes);
              c2::tma2_cg2(&mB, c2::peer0(&bfull[bs]), sB + bs * g.b_stage_bytes, kbi * 64, brow(j));
            }
            if (++bs == g.b_slots) { bs = 0; bph ^= 1; }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ===== MMA issuer (CTA0 only, M = 256 over the pair); warp-wide loop,
      // descriptors on the uniform datapath, one elected lane issues =====
      constexpr uint32_t IDESC = ptx::idesc_bf16(256, ACC, false, false);
      constexpr uint32_t DHI = ptx::sw128_desc_hi(1024);
      const bool leader = ptx::elect_one();
      if (g.resident) {
        ptx::mbar_wait(bres, 0);
        ptx::tc_fence_after();
      }
      const uint32_t halo_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sHalo), 16);
      const uint32_t b_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sB), 16);
      const uint32_t halo_step = g.halo_bytes >> 4, b_step = g.b_stage_bytes >> 4;
      const uint32_t wp8 = (uint32_t)g.Wp * 8;
      int as = 0, bs = 0;
      uint32_t aph = 0, bph = 0;
      int it = 0;
      for (int w = cluster; w < g.total; w += nclusters, ++it) {
        const int rest = ptx::fdiv(w, g.fd_nn);
        const int t = rest - ptx::fdiv(rest, g.fd_T) * g.T_img;
        const int q0 = 128 * t;
        const int row_off = q0 - ptx::fdiv(q0, g.fd_Wp) * g.Wp;
        int acs = it & 1;
        uint32_t tph = (it >> 1) & 1;
        if (leader) C2_TRACE(1, it, 0);
        ptx::mbar_wait(&tempty[acs], tph ^ 1);
        if (leader) C2_TRACE(1, it, 1);
        ptx::tc_fence_after();
        if (leader) C2_TRACE(1, it, 11);
        const uint32_t d = tmem + acs * ACC;
        uint32_t accum = 0;
        for (int ab = 0; ab < g.ablocks; ++ab) {
          int half = ab / g.cblks, cb = ab % g.cblks;
          ptx::mbar_wait(&afull[as], aph);
          if (leader) C2_TRACE(1, it, 2 + ab);
          ptx::tc_fence_after();
          const uint32_t a_lo = halo_lo0 + as * halo_step + row_off * 8;
          const bool grouped = !g.resident && g.b_group > 1;
          if ((g.resident && !(g.dbg & 2)) || grouped) {
            // all taps of this channel block back to back (B resident: no waits;
            // grouped stream: one wait and one commit per block)
            if (grouped) {
              ptx::mbar_wait(&bfull[bs], bph);
              ptx::tc_fence_after();
            }
            const uint32_t bb = grouped ? b_lo0 + bs * rr * b_step : b_lo0 + (half * rr * g.cblks + cb) * b_step;
            const uint32_t tap_b = grouped ? b_step : g.cblks * b_step;
            if (leader) {
              if (R > 0) {
#pragma unroll
                for (int ey = 0; ey < R; ++ey)
#pragma unroll
                  for (int ex = 0; ex < R; ++ex) {
                    const uint32_t at = a_lo + ey * wp8 + ex * 8, bt = bb + (ey * R + ex) * tap_b;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                      c2::mma_cg2(d, ptx::mk_desc(DHI, at + 2 * k), ptx::mk_desc(DHI, bt + 2 * k), IDESC, accum);
                      accum = 1;
                    }
                  }
              } else {
                for (int ey = 0; ey < r; ++ey)
                  for (int ex = 0; ex < r; ++ex) {
                    const uint32_t at = a_lo + ey * wp8 + ex * 8, bt = bb + (ey * r + ex) * tap_b;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                      c2::mma_cg2(d, ptx::mk_desc(DHI, at + 2 * k), ptx::mk_desc(DHI, bt + 2 * k), IDESC, accum);
                      accum = 1;
                    }
                  }
              }
            }
            accum = 1;
            __syncwarp();
            if (grouped) {
              if (leader) c2::commit_mc(&bempty[bs]);
              if (++bs == g.b_slots) { bs = 0; bph ^= 1; }
            }
          } else {
            for (int ey = 0; ey < r; ++ey) {
              for (int ex = 0; ex < r; ++ex) {
                uint32_t b_lo;
                if (g.resident) {
                  b_lo = b_lo0 + ((half * rr + ey * r + ex) * g.cblks + cb) * b_step;
                } else {
                  ptx::mbar_wait(&bfull[bs], bph);
                  ptx::tc_fence_after();
                  b_lo = b_lo0 + bs * b_step;
                }
                const uint32_t at = a_lo + ey * wp8 + ex * 8;
                if (leader && !(g.dbg & 2)) {
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    c2::mma_cg2(d, ptx::mk_desc(DHI, at + 2 * k), ptx::mk_desc(DHI, b_lo + 2 * k), IDESC,
                                accum | (uint32_t)k);
                }
                accum = 1;
                __syncwarp();
                if (!g.resident) {
                  if (leader) c2::commit_mc(&bempty[bs]);
                  if (++bs == g.b_slots) { bs = 0; bph ^= 1; }
                }
              }
            }
          }
          if (leader) c2::commit_mc(&aempty[as]);
          if (++as == g.a_slots) { as = 0; aph ^= 1; }
        }
        if (leader) c2::commit_mc(&tfull[acs]);
        if (leader) C2_TRACE(1, it, 15);
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 4 + NEPI) {
    // ===== epilogue (both CTAs, own TMEM rows); one 4 KB staging tile per warp,
    // one output pass at a time =====
    const int q = warp & 3;
    const int eg = (warp - 4) >> 2;  // epilogue warpgroup
    {
      // every bias of the layer into smem once; read back as float4 broadcasts
      const int et = threadIdx.x - 128;
      for (int i = et; i < g.nbias * g.Cout; i += NEPI * 32) {
        int role = i / g.Cout, c = i - role * g.Cout;
        const float* src = role == 0 ? g.bias0 : (role == 1 ? g.bias1 : g.bias2);
        sBias[i] = __ldg(src + c);
      }
      ptx::named_bar_sync(1, NEPI * 32);
    }
    // passes of this warp: with two warpgroups, group 0 writes y and group 1 a, b
    constexpr bool SPLIT = NEPI > 4;  // proposed / t4: channel-split warpgroups
    constexpr int CW = SPLIT ? 64 / (NEPI / 4) : 64;  // channels per warp
    const int o_beg = 0;
    const int o_end = NPASS;
    // split: warp (eg, q) owns a CW x 32-row staging tile (16 KB in all); else stg_tiles 4 KB tiles
    uint8_t* stg = SPLIT ? sStg + (warp - 4) * (CW * 64) : sStg + q * g.stg_tiles * 4096;
    const bool multi = g.stg_tiles > 1;
    const bool tracer = q == 0 && eg == 0 && lane == 0;
    const bool tracer1 = q == 0 && eg == 1 && lane == 0;
    const uint32_t tempty0 = c2::peer0(&tempty[0]);
    int it = 0;
    for (int w = cluster; w < g.total; w += nclusters, ++it) {
      const int rest = ptx::fdiv(w, g.fd_nn), j = w - rest * g.tiles_nn;
      const int p = ptx::fdiv(rest, g.fd_T), t = rest - p * g.T_img;
      int n = 2 * p + (int)rank;
      int acs = it & 1;
      uint32_t tph = (it >> 1) & 1;
      int qq = 128 * t + q * 32 + lane;
      int hq = ptx::fdiv(qq, g.fd_Wp), wq = qq - hq * g.Wp;
      bool valid = n < g.N && hq < g.OHg && wq < g.OWg;
      int pix;
      if (g.ss > 1) {
        valid = valid && (hq % g.ss) == 0 && (wq % g.ss) == 0;
        pix = valid ? (n * g.OHo + hq / g.ss) * g.OWo + wq / g.ss : -1;
      } else {
        pix = valid ? (n * g.OHo + hq) * g.OWo + wq : -1;
      }
      const int c_base = j * g.out_c_tile;
      if (tracer) C2_TRACE(2, it, 0);
      ptx::mbar_wait(&tfull[acs], tph);
      if (tracer) C2_TRACE(2, it, 1);
      if (tracer1) C2_TRACE(2, it, 10);
      ptx::tc_fence_after();
      if (g.dbg & 1) {
        __syncwarp();
        if (lane == 0) c2::arrive_remote(tempty0 + acs * 8);
        continue;
      }
      const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + acs * ACC;
      if (SPLIT) {
        // warpgroup eg takes channels [CW eg, CW eg + CW) of all three outputs:
        // (a, b, c) TMEM loads per 16 channels, y / a / b packed to bf16 in
        // registers, the accumulator handed back, then three staged store passes
        constexpr int JJ = CW / 16;
        uint4 pk[3][JJ][2];  // [y|a|b][jj][lo|hi]
        float ysv[CW == 32 ? 32 : 1];  // BN statistics: the stored y of this lane's pixel, 32 channels
#pragma unroll
        for (int jj = 0; jj < JJ; ++jj) {
          const int col = eg * CW + jj * 16;
          const int c0 = c_base + col;
          float va[16], vb[16], vc[16];
          ptx::tmem_ld16(tb + col, va);
          ptx::tmem_ld16(tb + 64 + col, vb);
          if (EPI == E2_PROPOSED) {
            ptx::tmem_ld16(tb + 128 + col, vc);
            const float4* pa = reinterpret_cast<const float4*>(sBias + c0);
            const float4* pb = reinterpret_cast<const float4*>(sBias + g.Cout + c0);
            const float4* pc = reinterpret_cast<const float4*>(sBias + 2 * g.Cout + c0);
            float ba[16], bbv[16], bc[16];
#pragma unroll
            for (int v4 = 0; v4 < 4; ++v4) {
              float4 x0 = pa[v4], x1 = pb[v4], x2 = pc[v4];
              ba[4 * v4] = x0.x; ba[4 * v4 + 1] = x0.y; ba[4 * v4 + 2] = x0.z; ba[4 * v4 + 3] = x0.w;
              bbv[4 * v4] = x1.x; bbv[4 * v4 + 1] = x1.y; bbv[4 * v4 + 2] = x1.z; bbv[4 * v4 + 3] = x1.w;
              bc[4 * v4] = x2.x; bc[4 * v4 + 1] = x2.y; bc[4 * v4 + 2] = x2.z; bc[4 * v4 + 3] = x2.w;
            }
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              va[e] += ba[e];
              vb[e] += bbv[e];
              vc[e] = fmaf(va[e], vb[e], vc[e] + bc[e]);
            }
          } else {
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) vc[e] = va[e] * vb[e];
          }
          if constexpr (CW == 32) if (g.stats) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              ysv[jj * 16 + e] = pix < 0 ? 0.f : (g.f32out ? vc[e] : __bfloat162float(__float2bfloat16_rn(vc[e])));
          }
          if (g.f32out) {
            // fp32 y, a, b rows of this lane's pixel, straight from registers
            if (pix >= 0) {
              float* dy_ = reinterpret_cast<float*>(g.out0) + (size_t)pix * g.Cout + c0;
              float* da_ = reinterpret_cast<float*>(g.out1) + (size_t)pix * g.Cout + c0;
              float* db_ = reinterpret_cast<float*>(g.out2) + (size_t)pix * g.Cout + c0;
#pragma unroll
              for (int v4 = 0; v4 < 4; ++v4) {
                reinterpret_cast<float4*>(dy_)[v4] = make_float4(vc[4 * v4], vc[4 * v4 + 1], vc[4 * v4 + 2], vc[4 * v4 + 3]);
                reinterpret_cast<float4*>(da_)[v4] = make_float4(va[4 * v4], va[4 * v4 + 1], va[4 * v4 + 2], va[4 * v4 + 3]);
                reinterpret_cast<float4*>(db_)[v4] = make_float4(vb[4 * v4], vb[4 * v4 + 1], vb[4 * v4 + 2], vb[4 * v4 + 3]);
              }
            }
            continue;
          }
          c2_pack16(vc, pk[0][jj][0], pk[0][jj][1]);
          c2_pack16(va, pk[1][jj][0], pk[1][jj][1]);
          c2_pack16(vb, pk[2][jj][0], pk[2][jj][1]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) c2::arrive_remote(tempty0 + acs * 8);
        if (tracer) C2_TRACE(2, it, 2);
        if (tracer1) C2_TRACE(2, it, 11);
        if constexpr (CW == 32) if (g.stats) {
          // this warp's 32 rows: per-channel mean and M2 (the finalize merges rows
          // with Chan's formula); the squares first, while ysv still holds y
          float sq[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) sq[e] = ysv[e] * ysv[e];
          const float s2 = c2_lane_sums32(sq, lane);
          const float s1 = c2_lane_sums32(ysv, lane);
          const int cnt = __popc(__ballot_sync(0xffffffffu, pix >= 0));
          const int row = (rest * 2 + (int)rank) * 4 + q;
          const float mean = cnt ? s1 / (float)cnt : 0.f;
          const float m2 = cnt ? fmaxf(s2 - s1 * mean, 0.f) : 0.f;
          const int cg = c_base + eg * 32 + lane;
          g.stats[(size_t)row * g.Cout + cg] = mean;
          g.stats[(size_t)g.stat_rows * g.Cout + (size_t)row * g.Cout + cg] = m2;
          if (lane == 0 && eg == 0 && j == 0) g.stats[(size_t)2 * g.stat_rows * g.Cout + row] = (float)cnt;
        }
        if (g.f32out) continue;  // stored above
        if (g.direct) {
          // straight from registers: this lane's pixel row, CW channels per output
          if (pix >= 0 && !(g.dbg & 4)) {
#pragma unroll
            for (int o = 0; o < 3; ++o) {
              bf16* dst = (o == 0 ? g.out0 : (o == 1 ? g.out1 : g.out2)) + (size_t)pix * g.Cout + c_base + eg * CW;
#pragma unroll
              for (int jj = 0; jj < JJ; ++jj) {
                reinterpret_cast<uint4*>(dst + jj * 16)[0] = pk[o][jj][0];
                reinterpret_cast<uint4*>(dst + jj * 16)[1] = pk[o][jj][1];
              }
            }
          }
          if (tracer) C2_TRACE(2, it, 3);
          if (tracer1) C2_TRACE(2, it, 12);
          continue;
        }
        // rows this lane stores in every pass: shuffles and address math once per tile
        constexpr int SCH = (2 * CW) / 16, SRPI = 32 / SCH, NRI = 32 / SRPI;
        long long roff[NRI];
#pragma unroll
        for (int i = 0; i < NRI; ++i) {
          const int rp = __shfl_sync(0xffffffffu, pix, SRPI * i + lane / SCH);
          roff[i] = rp >= 0 ? (long long)rp * g.Cout + c_base + eg * CW + (lane % SCH) * 8 : -1;
        }
#pragma unroll
        for (int o = 0; o < 3; ++o) {
#pragma unroll
          for (int jj = 0; jj < JJ; ++jj) c2_stage_rb<2 * CW>(stg, lane, jj, pk[o][jj][0], pk[o][jj][1]);
          __syncwarp();
          if (!(g.dbg & 4))  // dev knob: skip the global stores
            c2_store_rb_pre<2 * CW>(stg, o == 0 ? g.out0 : (o == 1 ? g.out1 : g.out2), roff, lane);
          __syncwarp();
        }
        if (tracer) C2_TRACE(2, it, 3);
        if (tracer1) C2_TRACE(2, it, 12);
        continue;
      }
#pragma unroll 1
      for (int o = o_beg; o < o_end; ++o) {
#pragma unroll 1
        for (int jj = 0; jj < 4; ++jj) {
          float out[16];
          const int c0 = c_base + jj * 16;
          if (EPI == E2_PROPOSED || EPI == E2_T4) {
            float va[16], vb[16];
            if (o != 2) ptx::tmem_ld16(tb + jj * 16, va);            // a
            if (o != 1) ptx::tmem_ld16(tb + 64 + jj * 16, vb);       // b
            float vc[16];
            if (EPI == E2_PROPOSED && o == 0) ptx::tmem_ld16(tb + 128 + jj * 16, vc);
            // biases: 16 channels as 4 x float4 per role, loaded together (a per-element
            // __ldg chain serialised at ~86 cycles each -- traced)
            float ba[16], bbv[16], bc[16];
            if (EPI == E2_PROPOSED) {
              const float4* pa = reinterpret_cast<const float4*>(sBias + c0);
              const float4* pb = reinterpret_cast<const float4*>(sBias + g.Cout + c0);
              const float4* pc = reinterpret_cast<const float4*>(sBias + 2 * g.Cout + c0);
#pragma unroll
              for (int v4 = 0; v4 < 4; ++v4) {
                float4 x0 = pa[v4], x1 = pb[v4], x2 = pc[v4];
                ba[4 * v4] = x0.x; ba[4 * v4 + 1] = x0.y; ba[4 * v4 + 2] = x0.z; ba[4 * v4 + 3] = x0.w;
                bbv[4 * v4] = x1.x; bbv[4 * v4 + 1] = x1.y; bbv[4 * v4 + 2] = x1.z; bbv[4 * v4 + 3] = x1.w;
                bc[4 * v4] = x2.x; bc[4 * v4 + 1] = x2.y; bc[4 * v4 + 2] = x2.z; bc[4 * v4 + 3] = x2.w;
              }
            }
            ptx::tmem_wait_ld();
            if (EPI == E2_PROPOSED) {
              if (o == 0) {
#pragma unroll
                for (int e = 0; e < 16; ++e) out[e] = fmaf(va[e] + ba[e], vb[e] + bbv[e], vc[e] + bc[e]);
              } else if (o == 1) {
#pragma unroll
                for (int e = 0; e < 16; ++e) out[e] = va[e] + ba[e];
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) out[e] = vb[e] + bbv[e];
              }
            } else {
              if (o == 0) {
#pragma unroll
                for (int e = 0; e < 16; ++e) out[e] = va[e] * vb[e];
              } else if (o == 1) {
#pragma unroll
                for (int e = 0; e < 16; ++e) out[e] = va[e];
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) out[e] = vb[e];
              }
            }
          } else if (EPI == E2_PLAIN) {
            ptx::tmem_ld16(tb + o * 64 + jj * 16, out);
            float bz[16];
            if (g.nbias) {
              const float4* pz = reinterpret_cast<const float4*>(sBias + c0 + o * 64);
#pragma unroll
              for (int v4 = 0; v4 < 4; ++v4) {
                float4 x0 = pz[v4];
                bz[4 * v4] = x0.x; bz[4 * v4 + 1] = x0.y; bz[4 * v4 + 2] = x0.z; bz[4 * v4 + 3] = x0.w;
              }
            }
            ptx::tmem_wait_ld();
            if (g.nbias) {
#pragma unroll
              for (int e = 0; e < 16; ++e) out[e] += bz[e];
            }
          } else {  // E2_SQ: dx = 2 x acc0 (+ acc1)
            float v0[16], v1[16], xv[16];
            ptx::tmem_ld16(tb + jj * 16, v0);
            if (NB == 2) ptx::tmem_ld16(tb + 64 + jj * 16, v1);
            if (valid) {
              const uint4* xp = reinterpret_cast<const uint4*>(g.xres + (size_t)pix * g.Cout + c0);
              uint4 u0 = __ldg(xp), u1 = __ldg(xp + 1);
              const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&u0);
              const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&u1);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float2 f0 = __bfloat1622float2(h0[e]), f1 = __bfloat1622float2(h1[e]);
                xv[2 * e] = f0.x; xv[2 * e + 1] = f0.y; xv[8 + 2 * e] = f1.x; xv[9 + 2 * e] = f1.y;
              }
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) xv[e] = 0.f;
            }
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float tt = v0[e] * xv[e];
              out[e] = tt + tt;
              if (NB == 2) out[e] += v1[e];
            }
          }
          if (g.f32out) {
            // fp32 rows straight from registers (64 B: four 16-B stores)
            if (pix >= 0) {
              const int ch = ((EPI == E2_PLAIN) ? c_base + o * 64 : c_base) + jj * 16;
              float* dst = reinterpret_cast<float*>((EPI == E2_PROPOSED || EPI == E2_T4)
                                                        ? (o == 0 ? g.out0 : (o == 1 ? g.out1 : g.out2))
                                                        : g.out0) + (size_t)pix * g.Cout + ch;
#pragma unroll
              for (int v4 = 0; v4 < 4; ++v4)
                reinterpret_cast<float4*>(dst)[v4] =
                    make_float4(out[4 * v4], out[4 * v4 + 1], out[4 * v4 + 2], out[4 * v4 + 3]);
            }
          } else if (g.direct) {
            // 32 B of this row's output straight from registers (two 16-B stores)
            if (pix >= 0) {
              bf16* dst = (EPI == E2_PROPOSED || EPI == E2_T4) ? (o == 0 ? g.out0 : (o == 1 ? g.out1 : g.out2))
                                                               : g.out0;
              const int ch = ((EPI == E2_PLAIN) ? c_base + o * 64 : c_base) + jj * 16;
              uint4 lo, hi;
              lo.x = c2::pack2(out[0], out[1]);   lo.y = c2::pack2(out[2], out[3]);
              lo.z = c2::pack2(out[4], out[5]);   lo.w = c2::pack2(out[6], out[7]);
              hi.x = c2::pack2(out[8], out[9]);   hi.y = c2::pack2(out[10], out[11]);
              hi.z = c2::pack2(out[12], out[13]); hi.w = c2::pack2(out[14], out[15]);
              uint4* p = reinterpret_cast<uint4*>(dst + (size_t)pix * g.Cout + ch);
              p[0] = lo;
              p[1] = hi;
            }
          } else {
            c2::stage16(stg + (multi ? (o - o_beg) * 4096 : 0), lane, jj, out);
          }
        }
        if (tracer) C2_TRACE(2, it, 4 + 2 * o);
        if (o == o_end - 1) {
          // every TMEM read of this tile is done -> hand the accumulator back
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) c2::arrive_remote(tempty0 + acs * 8);
          if (tracer) C2_TRACE(2, it, 2);
          if (tracer1) C2_TRACE(2, it, 11);
        }
        if (!multi && !g.direct) {
          __syncwarp();
          c2_store_pass<EPI>(g, stg, o, c_base, pix, lane);
          __syncwarp();
          if (tracer) C2_TRACE(2, it, 5 + 2 * o);
        }
      }
      if (multi && !g.direct) {
        __syncwarp();
#pragma unroll 1
        for (int o = o_beg; o < o_end; ++o) c2_store_pass<EPI>(g, stg + (o - o_beg) * 4096, o, c_base, pix, lane);
        __syncwarp();
      }
      if (tracer) C2_TRACE(2, it, 3);
      if (tracer1) C2_TRACE(2, it, 12);
    }
  } else if (XF && warp >= 4 + NEPI) {
    // ===== operand transform (XF): the A halo slots of the transformed blocks are
    // written here -- 16-B chunks of the source rows loaded (ld.global.nc), the
    // elementwise op in fp32, bf16 stored at the SWIZZLE_128B position the TMA
    // would use (chunk c of halo row ri at c ^ (ri & 7)); out-of-image rows and
    // columns are zeros (the TMA's OOB fill = the padding). Each warp then
    // fences the generic-proxy writes for the tensor core and arrives (release)
    // on CTA0's full barrier; it also arrives for TMA-loaded blocks so the
    // barrier count stays fixed.
    constexpr int U = 8;
    const int xt = threadIdx.x - (128 + NEPI * 32);
    const int nchunk = g.Wp * g.HR * 8;
    const size_t img = (size_t)g.Hin * g.Win;
    int as = 0;
    uint32_t aph = 0;
    const bool xtr = xt == 0;  // dev trace: role 3 = transform warp 0 of CTA 0
    int it = 0;
    for (int w = cluster; w < g.total; w += nclusters, ++it) {
      const int rest = ptx::fdiv(w, g.fd_nn);
      const int p = ptx::fdiv(rest, g.fd_T), t = rest - p * g.T_img;
      const int n = 2 * p + (int)rank;
      const int h0 = ptx::fdiv(128 * t, g.fd_Wp) - g.pe;
      for (int ab = 0; ab < g.ablocks; ++ab) {
        const int half = ab / g.cblks, cb = ab % g.cblks;
        const bool xblk = g.xf == 1 ? half == 0 : (g.xf == 2 && cb < g.csplit);  // 3: none (dev)
        if (xblk) {
          const bf16* s0 = g.xf_x;
          const bf16* s1 = nullptr;
          int ch = cb * 64;
          if (g.xf == 2) {
            const int seg = cb >= g.xf_fb ? 1 : 0;
            ch = (cb - seg * g.xf_fb) * 64;
            s1 = seg == 0 ? g.xf_b : g.xf_a;
          }
          uint8_t* slot = sHalo + as * g.halo_bytes;
          // the first pass's loads go out before the wait for the slot (registers
          // only), so their latency overlaps the MMAs still reading it. Thread xt
          // owns 16-B chunk (xt & 7) of halo rows (xt >> 3) + 32 k (XW = 8: 256
          // threads = 32 rows per step): the row -> (image row, column) walk and
          // the source offsets advance incrementally (the transform is issue-bound)
          bool waited = false;
          constexpr int RSTEP = XW * 32 / 8;  // halo rows per step of all transform threads
          const int cc = xt & 7;
          int r_ = xt >> 3;
          int hi = ptx::fdiv(r_, g.fd_Wp), wc = r_ - hi * g.Wp;
          const size_t rowpix = (size_t)g.Win * g.xf_cs;
          const bf16* b0 = s0 + (size_t)n * img * g.xf_cs + ch + cc * 8;
          const bf16* b1 = s1 ? s1 + (size_t)n * img * g.xf_cs + ch + cc * 8 : nullptr;
          const int nrows = g.Wp * g.HR;
          const bool nok = n < g.N && !(g.dbg & 8);
          while (r_ < nrows) {
            uint4 v0[U], v1[U];
            int ri[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int hh = h0 + hi, ww = wc - g.pe;
              ri[u] = r_ < nrows ? r_ : -1;
              const bool ok = r_ < nrows && nok && hh >= 0 && hh < g.Hin && ww >= 0 && ww < g.Win;
              const size_t off = (size_t)hh * rowpix + (size_t)ww * g.xf_cs;
              v0[u] = ok ? __ldg(reinterpret_cast<const uint4*>(b0 + off)) : make_uint4(0, 0, 0, 0);
              if (g.xf == 2) v1[u] = ok ? __ldg(reinterpret_cast<const uint4*>(b1 + off)) : make_uint4(0, 0, 0, 0);
              r_ += RSTEP;
              wc += RSTEP;
              while (wc >= g.Wp) { wc -= g.Wp; ++hi; }
            }
            if (!waited) {
              if (xtr) C2_TRACE(3, it, 2 * ab);
              if (lane == 0) c2_wait_sleep(&aempty[as], aph ^ 1);
              if (xtr) C2_TRACE(3, it, 2 * ab + 1);
              __syncwarp();
              waited = true;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (ri[u] < 0) continue;
              const uint4 val = c2_bf16_mul(v0[u], g.xf == 2 ? v1[u] : v0[u]);
              if (!(g.dbg & 128)) *reinterpret_cast<uint4*>(slot + ri[u] * 128 + ((cc ^ (ri[u] & 7)) << 4)) = val;
            }
          }
          if (!waited) {
            if (lane == 0) c2_wait_sleep(&aempty[as], aph ^ 1);
            __syncwarp();
          }
          if (!(g.dbg & 64)) ptx::fence_proxy_async_smem();
        } else {
          if (lane == 0) c2_wait_sleep(&aempty[as], aph ^ 1);
        }
        __syncwarp();
        if (xtr) C2_TRACE(3, it, 8 + ab);
        if (lane == 0) c2_arrive_release(c2::peer0(&afull[as]));
        if (++as == g.a_slots) { as = 0; aph ^= 1; }
      }
    }
  }
  ptx::tc_fence_before();
  c2::cluster_sync();
  if (g.trace && threadIdx.x == 0 && blockIdx.x < 1024) {
    g.trace[4096 + 2 * blockIdx.x + 1] = gtimer();
    g.trace[6144 + 2 * blockIdx.x + 1] = clock64();
  }
  if (warp == 2) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static unsigned long long* g_trace = nullptr;
static unsigned long long* trace_buffer() {
  if (!g_trace) {
    cudaMalloc(&g_trace, 8192 * sizeof(unsigned long long));
  }
  cudaMemset(g_trace, 0, 8192 * sizeof(unsigned long long));
  return g_trace;
}
}  // namespace qd
// dev-only: spin `cycles` SM clocks on every SM and record clock64 / globaltimer
// at both ends of block 0 into out[4] (clock-rate probe under the caller's load)
__global__ void qd_spin_kernel(long long cycles, unsigned long long* out) {
  unsigned long long c0 = clock64(), t0 = qd::gtimer();
  while ((long long)(clock64() - c0) < cycles) {
  }
  unsigned long long c1 = clock64(), t1 = qd::gtimer();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = c0; out[1] = c1; out[2] = t0; out[3] = t1;
  }
}
extern "C" int qd_debug_spin(long long cycles, unsigned long long* dev_out, void* stream) {
  qd_spin_kernel<<<148, 32, 0, (cudaStream_t)stream>>>(cycles, dev_out);
  return (int)cudaGetLastError();
}
// dev-only: copy the last QD_TRACE buffer (8192 u64: 3 roles x 64 tiles x 16 events of
// clock64; wgrad: per-CTA globaltimer pairs from slot 3072, clock64 pairs from 2048;
// conv2: per-CTA globaltimer pairs from 4096, clock64 pairs from 6144)
extern "C" int qd_debug_trace_copy(unsigned long long* host) {
  if (!qd::g_trace) return -1;
  cudaDeviceSynchronize();
  return (int)cudaMemcpy(host, qd::g_trace, 8192 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
}
namespace qd {
// co-resident clusters of size 2 for a kernel at this smem / block size (cached per kernel)
template <typename K>
static int max_pair_clusters(K kernel, int threads, size_t smem) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(2 * 148, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
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
  if (getenv("QD_VERBOSE")) fprintf(stderr, "[qd] max active 2-CTA clusters: %d (smem %zu)\n", n, smem);
  return n;
}
extern PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn();
extern CUresult tc_encode_tiled(CUtensorMap* m, CUtensorMapDataType dt, cuuint32_t rank, void* ptr,
                                const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                                const cuuint32_t* es, CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                                CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob);
extern int tc_num_sms();

struct C2Plan {
  bool ok;
  C2Args g;
  size_t smem;
};

static int c2_map(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims, const cuuint32_t* box) {
  cuuint64_t strides[4];
  cuuint64_t acc = dims[0] * 2;
  for (int i = 1; i < rank; ++i) {
    strides[i - 1] = acc;
    acc *= dims[i];
  }
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = tc_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), dims, strides, box,
                              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(QD_ERR_CUDA, "cuTensorMapEncodeTiled (conv2) failed (%d)", (int)r);
  return QD_OK;
}

// geometry + smem plan; ok=false if this conv does not fit the v2 kernel
static C2Plan c2_plan(int N, int Cin, int Win, int Hin, int OWg, int OHg, int pe, int r, int dual, int NB, int NOUT,
                      int tiles_nn, int Cout, int nbias) {
  C2Plan pl;
  memset(&pl, 0, sizeof(pl));
  C2Args& g = pl.g;
  if (r < 2 || Cin % 64 || Cout % 64) return pl;
  int Wp = Win + 2 * pe;
  if (OWg != Wp - r + 1 || Wp > 256 || OWg < 12) return pl;
  int T_img = (OHg * Wp + 127) / 128;
  int HR = 0;
  for (int t = 0; t < T_img; ++t) {
    int q0 = 128 * t, lo = q0 / Wp, hi = (q0 + 127 + (r - 1) * Wp + (r - 1)) / Wp;
    if (hi - lo + 1 > HR) HR = hi - lo + 1;
  }
  if (HR > 256) return pl;
  uint32_t halo_tx = (uint32_t)Wp * HR * 128;
  uint32_t halo = (halo_tx + 1023) / 1024 * 1024;
  if (halo > 64 * 1024) return pl;
  int cblks = Cin / 64;
  int ablocks = cblks * (1 + dual);
  int KBtot = ablocks * r * r;
  uint32_t bstage = NB * 32 * 128;
  // staging: one 4 KB tile per warp per output pass (single epilogue pass over TMEM,
  // stores after the hand-back) when smem allows, else one tile reused per pass
  // (proposed / t4: 8 warps x 2 KB half-row tiles = 4 x 4 KB)
  int stg_tiles = NOUT == 3 ? 1 : NOUT;
  {
    const char* e = getenv("QD_C2_STG");
    if (e && NOUT != 3) stg_tiles = atoi(e) > 1 ? NOUT : 1;
  }
  const size_t bias_bytes = (size_t)nbias * Cout * 4;
  const size_t fixed0 = 1024 + 4 * (size_t)stg_tiles * 4096 + bias_bytes + 1024;  // slack, staging, biases, barriers
  const size_t limit = 227 * 1024;
  int resident = 0, slots, aslots = 0, bgroup = 1;
  // prefer resident B with >= 3 halo buffers; else stream B with a 4-deep halo ring
  if (tiles_nn == 1 && KBtot <= 48) {
    size_t rest = limit - fixed0 - (size_t)KBtot * bstage;
    if ((long long)rest >= 2 * (long long)halo) {
      resident = 1;
      slots = KBtot;
      aslots = (int)(rest / halo);
      if (aslots > 4) aslots = 4;
      // fprop: two halo buffers -- the smaller footprint lets the next PDL-launched
      // kernel's CTAs land beside this one's tail (C2 step 115.7 -> 113.0 us, t4
      // 64@56 +5%; neutral on the other C5 shapes and both nets; tools/aslot_ab.sh);
      // dgrad: four (112.1 us)
      int want = NOUT == 3 ? 2 : 4;
      const char* e = getenv(NOUT == 3 ? "QD_ASLOTS" : "QD_ASLOTS_DG");  // dev knobs: 1..4 (fprop / other)
      if (e && atoi(e) >= 1) want = atoi(e);
      if (want < aslots) aslots = want;
    }
  }
  if (!resident) {
    aslots = 4;
    while (aslots > 2 && fixed0 + (size_t)aslots * halo + 4 * (size_t)bstage > limit) --aslots;
    if (fixed0 + (size_t)aslots * halo + 2 * (size_t)bstage > limit) return pl;
    slots = (int)((limit - fixed0 - (size_t)aslots * halo) / bstage);
    // ring depth cap 8: deeper rings for the small (4 / 8 KB) stages were measured neutral
    // to slower (the larger footprint delays the next PDL-launched kernel's CTAs)
    int cap = 8;
    {
      const char* e = getenv("QD_C2_BSLOTS");  // dev knob: B ring depth cap (2..48)
      if (e && atoi(e) >= 2 && atoi(e) <= 48) cap = atoi(e);
    }
    if (slots > cap) slots = cap;
    // grouped stream (all r*r taps of a channel block per ring slot) where two groups fit
    // beside the halo ring: the MMA warp then waits / commits once per block, not per tap
    const char* eg = getenv("QD_C2_BGROUP");  // dev knob: 0 = per-tap ring, 1 = grouped wherever it fits
    const int gmode = eg ? atoi(eg) : -1;
    const size_t gbytes = (size_t)r * r * bstage;
    const bool gwant = gmode == 1 || (gmode < 0 && bstage <= 4096);
    if (gwant) {
      int ga = aslots;
      while (ga > 2 && fixed0 + (size_t)ga * halo + 2 * gbytes > limit) --ga;
      if (fixed0 + (size_t)ga * halo + 2 * gbytes <= limit) {
        aslots = ga;
        bgroup = r * r;
        slots = (int)((limit - fixed0 - (size_t)aslots * halo) / gbytes);
        if (slots > 3) slots = 3;
      }
    }
  }
  const size_t fixed = fixed0 + (size_t)aslots * halo;
  g.N = N; g.Cin = Cin; g.Win = Win; g.Hin = Hin; g.OHg = OHg; g.OWg = OWg;
  g.pe = pe; g.r = r; g.Wp = Wp; g.HR = HR;
  g.T_img = T_img; g.tiles_nn = tiles_nn; g.total = ((N + 1) / 2) * T_img * tiles_nn;
  g.fd_nn = ptx::make_fastdiv(tiles_nn); g.fd_T = ptx::make_fastdiv(T_img); g.fd_Wp = ptx::make_fastdiv(Wp);
  g.cblks = cblks; g.ablocks = ablocks; g.KBtot = KBtot; g.resident = resident;
  g.halo_bytes = halo; g.halo_tx = halo_tx; g.b_stage_bytes = bstage; g.b_slots = slots; g.b_group = bgroup; g.a_slots = aslots; g.stg_tiles = stg_tiles; g.nbias = nbias;
  g.Cout = Cout;
  pl.smem = fixed + (size_t)slots * bgroup * bstage;
  pl.ok = true;
  return pl;
}

// cap on the persistent conv2 grid (pairs) for the next launches; 0 = all SMs
static thread_local int g_conv2_cap = 0;  // per host thread (set around one launch)
void set_conv2_cap(int pairs) { g_conv2_cap = pairs; }

template <int EPI, int NB, int R, int XF = 0>
static int c2_launch_r(const CUtensorMap& A0, const CUtensorMap& A1, const CUtensorMap& B, const C2Plan& pl,
                       cudaStream_t st) {
  using Th = C2Threads<EPI, NB, XF>;
  raise_smem_attr((const void*)conv2_kernel<EPI, NB, R, XF>, pl.smem);
  // persistent grid: only as many pairs as can be co-resident (GPCs with an odd
  // number of free SMs cannot host a pair; a second wave would double the time)
  thread_local int maxc_[kMaxDev] = {};
  thread_local size_t maxc_smem_[kMaxDev] = {};
  int& maxc = maxc_[cur_device()];
  size_t& maxc_smem = maxc_smem_[cur_device()];
  if (maxc == 0 || maxc_smem != pl.smem) {
    maxc = max_pair_clusters(conv2_kernel<EPI, NB, R, XF>, Th::THREADS, pl.smem);
    maxc_smem = pl.smem;
  }
  int clusters = tc_num_sms() / 2;
  if (maxc > 0 && maxc < clusters) clusters = maxc;
  if (pl.g.total < clusters) clusters = pl.g.total;
  if (g_conv2_cap > 0 && g_conv2_cap < clusters) clusters = g_conv2_cap;
  const cudaError_t le = launch_pdl(conv2_kernel<EPI, NB, R, XF>, dim3(2 * clusters), dim3(Th::THREADS),
                                    pl.smem, st, A0, A1, B, pl.g);
  if (le != cudaSuccess) {
    cudaGetLastError();
    cudaFuncAttributes fa;
    memset(&fa, 0, sizeof(fa));
    const cudaError_t fe = cudaFuncGetAttributes(&fa, conv2_kernel<EPI, NB, R, XF>);
    const int again = max_pair_clusters(conv2_kernel<EPI, NB, R, XF>, Th::THREADS, pl.smem);
    int dev = -1;
    cudaGetDevice(&dev);
    return set_error(QD_ERR_CUDA,
                     "conv2 launch (%d CTAs, %d threads, %zu B smem, maxc %d, tiles %d; function: "
                     "max dyn smem %d static %zu (%s), clusters now %d, device %d): %s",
                     2 * clusters, Th::THREADS, pl.smem, maxc, (int)pl.g.total,
                     fa.maxDynamicSharedSizeBytes, fa.sharedSizeBytes, cudaGetErrorString(fe), again, dev,
                     cudaGetErrorString(le));
  }
  count_launch(st, "conv2");
  return check_launch("conv2");
}
template <int EPI, int NB>
static int c2_launch(const CUtensorMap& A0, const CUtensorMap& A1, const CUtensorMap& B, const C2Plan& pl,
                     cudaStream_t st) {
  if (pl.g.xf) {
    if (pl.g.r == 3) return c2_launch_r<EPI, NB, 3, 1>(A0, A1, B, pl, st);
    return c2_launch_r<EPI, NB, 0, 1>(A0, A1, B, pl, st);
  }
  if (pl.g.r == 3) return c2_launch_r<EPI, NB, 3>(A0, A1, B, pl, st);
  return c2_launch_r<EPI, NB, 0>(A0, A1, B, pl, st);
}

// fprop / dgrad entry: returns QD_ERR_UNSUPPORTED when the geometry does not
// fit (the caller then uses the v1 kernel)
int run_conv2(int epi, int nbk, const void* a0, const void* a1, int Cin, int Win, int Hin, int N, int OWg, int OHg,
              int pe, int r, int dual, const void* wmat, int wrows, int wK, int b_rs_tile, int b_rs_blk,
              int tiles_nn, int out_c_tile, void* o0, void* o1, void* o2, int Cout, const float* const bias[3],
              const void* xres, cudaStream_t st, int ss, const void* a_tail, int csplit, int pdl_wait,
              int f32out, float* stats, const C2Xform* xf) {
  int NOUT = (epi == E2_PROPOSED || epi == E2_T4) ? 3 : (epi == E2_PLAIN ? nbk : 1);
  int nbias = epi == E2_PROPOSED ? 3 : ((epi == E2_PLAIN && bias[0]) ? 1 : 0);
  C2Plan pl = c2_plan(N, Cin, Win, Hin, OWg, OHg, pe, r, dual, nbk, NOUT, tiles_nn, Cout, nbias);
  if (!pl.ok) return QD_ERR_UNSUPPORTED;
  C2Args& g = pl.g;
  g.b_rs_tile = b_rs_tile;
  g.b_rs_blk = b_rs_blk;
  g.b_contig = (b_rs_blk == 64) ? 1 : 0;
  if (!g.b_contig && nbk != 2) return QD_ERR_UNSUPPORTED;
  g.out_c_tile = out_c_tile;
  g.ss = ss;
  g.dual = dual;
  g.f32out = f32out;
  g.stats = stats;
  g.stat_rows = ((N + 1) / 2) * g.T_img * 8;
  if (stats && !(epi == E2_PROPOSED || epi == E2_T4)) return QD_ERR_UNSUPPORTED;
  if (f32out && (ss != 1 || epi == E2_SQ)) return QD_ERR_UNSUPPORTED;
  {
    const char* e = getenv("QD_C2_DIRECT");
    g.direct = f32out ? 1 : (e ? atoi(e) : 0);
    const char* f = getenv("QD_PF");
    g.pf = f ? atoi(f) : 0;  // measured: no gain on C2 (the pipe is MMA-bound)

  }
  g.OHo = (OHg - 1) / ss + 1;
  g.OWo = (OWg - 1) / ss + 1;
  {
    const char* e = getenv("QD_DEBUG");
    g.dbg = e ? atoi(e) : 0;
    g.trace = getenv("QD_TRACE") ? trace_buffer() : nullptr;
  }
  g.bias0 = bias[0]; g.bias1 = bias[1]; g.bias2 = bias[2];
  g.out0 = (bf16*)o0; g.out1 = (bf16*)o1; g.out2 = (bf16*)o2;
  g.xres = (const bf16*)xres;
  g.pdl_wait = pdl_wait;
  if (xf && xf->mode) {
    if (f32out || (xf->mode == 1 && dual > 1) || (xf->mode == 2 && !(a_tail && csplit > 0)))
      return QD_ERR_UNSUPPORTED;
    g.xf = xf->mode;
    if (getenv("QD_XF_NULL")) g.xf = 3;  // dev: transform warps present, every block TMA-loaded (timing)
    g.xf_cs = xf->cs;
    g.xf_fb = xf->fb;
    g.xf_x = (const bf16*)xf->x;
    g.xf_a = (const bf16*)xf->a;
    g.xf_b = (const bf16*)xf->b;
  }
  CUtensorMap A0, A1, B;
  int rc;
  cuuint32_t bA[4] = {64, (cuuint32_t)g.Wp, (cuuint32_t)g.HR, 1};
  g.csplit = (a_tail && csplit > 0 && csplit < Cin / 64) ? csplit : 0;
  if (g.csplit) {
    cuuint64_t d0[4] = {(cuuint64_t)(64 * g.csplit), (cuuint64_t)Win, (cuuint64_t)Hin, (cuuint64_t)N};
    cuuint64_t d1[4] = {(cuuint64_t)(Cin - 64 * g.csplit), (cuuint64_t)Win, (cuuint64_t)Hin, (cuuint64_t)N};
    if ((rc = c2_map(&A0, a0, 4, d0, bA))) return rc;
    if ((rc = c2_map(&A1, a_tail, 4, d1, bA))) return rc;
  } else {
    cuuint64_t dA[4] = {(cuuint64_t)Cin, (cuuint64_t)Win, (cuuint64_t)Hin, (cuuint64_t)N};
    if ((rc = c2_map(&A0, a0, 4, dA, bA))) return rc;
    if ((rc = c2_map(&A1, a1 ? a1 : a0, 4, dA, bA))) return rc;
  }
  cuuint64_t dB[2] = {(cuuint64_t)wK, (cuuint64_t)wrows};
  cuuint32_t bB[2] = {64, (cuuint32_t)(nbk * 32)};
  if ((rc = c2_map(&B, wmat, 2, dB, bB))) return rc;
  if (epi == E2_PROPOSED) return c2_launch<E2_PROPOSED, 3>(A0, A1, B, pl, st);
  if (epi == E2_T4) return c2_launch<E2_T4, 2>(A0, A1, B, pl, st);
  if (epi == E2_PLAIN) {
    if (nbk == 4) return c2_launch<E2_PLAIN, 4>(A0, A1, B, pl, st);
    if (nbk == 2) return c2_launch<E2_PLAIN, 2>(A0, A1, B, pl, st);
    return c2_launch<E2_PLAIN, 1>(A0, A1, B, pl, st);
  }
  if (nbk == 2) return c2_launch<E2_SQ, 2>(A0, A1, B, pl, st);
  return c2_launch<E2_SQ, 1>(A0, A1, B, pl, st);
}


// ===========================================================================
// K4 v2: wgrad with halo reuse.
//   dW^T[(tap, c)][j] = sum_q x_pad[q + off(tap)][c] * D[q][j]
// over the same padded-flat q of conv2. Per stage: one D box {64 j, Wp, RD}
// (columns >= OW are out of bounds -> 0, so junk q contribute nothing) and one
// x halo box {64 c, Wp, RX}. A = x^T (MN-major): M = 128 rows = TWO taps, the
// second tap's 64-channel atom being the same halo shifted by
// off(t1) - off(t0) rows (LBO = that shift; overlapping atoms are legal,
// profiles/r1_probe_lbo_overlap_and_tma_dst.log). B = D (MN-major, N = 64 j).
// All r*r taps accumulate in one CTA: ceil(r*r/2) accumulators x 64 columns.
// Output: fp32 split-K partials [S][Jd][Kf], folded by wgrad_finish.
// ===========================================================================
struct W2Args {
  int N, OHg, OWg, Jd, Kf, K0, C;
  int pe, r, Wp, RD, RX;
  int T_img, cblks, ablocks, jtiles, splits;
  int NT, ntb;          // N tile (j) width and its 64-wide boxes
  int npairs, pp, tgroups;  // tap pairs, pairs per CTA (TMEM: pp * NT <= 512), tap groups
  int gsplit[16];           // split-K count per tap group (weighted by its pairs)
  int gstart[17];           // prefix sums of gsplit
  uint32_t d_tx, x_tx, d_bytes, x_bytes;  // d_* per 64-j box
  int stages;
  int jsplit;  // D channel blocks >= jsplit are loaded from the second D map (dy)
  float* part;
  unsigned long long* trace;  // QD_TRACE (dev only)
};


__global__ void __launch_bounds__(256, 1)
    wgrad2_kernel(const __grid_constant__ CUtensorMap mX0, const __grid_constant__ CUtensorMap mX1,
                  const __grid_constant__ CUtensorMap mD, const __grid_constant__ CUtensorMap mD1,
                  const W2Args g) {
  if (g.trace && threadIdx.x == 0 && blockIdx.x < 512) g.trace[3072 + 2 * blockIdx.x] = gtimer();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t stage_bytes = g.ntb * g.d_bytes + g.x_bytes;
  uint64_t* full = (uint64_t*)(sm + g.stages * stage_bytes);
  uint64_t* empty = full + g.stages;
  uint64_t* done = empty + g.stages;
  uint32_t* tslot = (uint32_t*)(done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int b = blockIdx.x;
  const int jt = b % g.jtiles;
  b /= g.jtiles;
  const int ab = b % g.ablocks;
  b /= g.ablocks;
  int tg = 0;
  while (tg + 1 < g.tgroups && b >= g.gstart[tg + 1]) ++tg;
  const int split = b - g.gstart[tg];
  const int gs = g.gsplit[tg];
  const int half = ab / g.cblks, cb = ab % g.cblks;
  const int nblk = g.N * g.T_img;
  const int q_beg = (int)((long long)split * nblk / gs);
  const int q_end = (int)((long long)(split + 1) * nblk / gs);
  const int rr = g.r * g.r;
  const int p_beg = tg * g.pp;
  const int p_end = min(g.npairs, p_beg + g.pp);

  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&mX0);
    ptx::prefetch_tmap(&mX1);
    ptx::prefetch_tmap(&mD);
    if (g.jsplit) ptx::prefetch_tmap(&mD1);
    for (int i = 0; i < g.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(tslot, 512);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::pdl_wait();
  ptx::pdl_launch();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    const bool leader = ptx::elect_one();
    int st = 0;
    uint32_t ph = 0;
    int n = q_beg / g.T_img, t = q_beg % g.T_img;  // walked incrementally below
    for (int qb = q_beg; qb < q_end; ++qb, (++t == g.T_img ? (t = 0, ++n) : 0)) {
      int hq_lo = (128 * t) / g.Wp;
      if (leader) C2_TRACE(0, qb - q_beg, 0);
      ptx::mbar_wait(&empty[st], ph ^ 1);
      if (leader) {
        C2_TRACE(0, qb - q_beg, 1);
        uint8_t* s = sm + st * stage_bytes;
        ptx::mbar_arrive_expect_tx(&full[st], g.ntb * g.d_tx + g.x_tx);
        for (int i = 0; i < g.ntb; ++i) {
          const int jb = jt * g.ntb + i;
          if (g.jsplit && jb >= g.jsplit)
            ptx::tma_load_4d(&mD1, &full[st], s + i * g.d_bytes, (jb - g.jsplit) * 64, 0, hq_lo, n);
          else
            ptx::tma_load_4d(&mD, &full[st], s + i * g.d_bytes, jb * 64, 0, hq_lo, n);
        }
        ptx::tma_load_4d(half ? &mX1 : &mX0, &full[st], s + g.ntb * g.d_bytes, cb * 64, -g.pe, hq_lo - g.pe, n);
      }
      __syncwarp();
      if (++st == g.stages) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    // B = D (MN-major, N = NT j over ntb atoms g.d_bytes apart); A = x^T, M = two
    // taps as two 64-channel atoms of the same halo, LBO = their row shift
    const uint32_t IDESC = ptx::idesc_bf16(128, g.NT, true, true);
    constexpr uint32_t DHI = ptx::sw128_desc_hi(1024);
    const bool leader = ptx::elect_one();
    const uint32_t s_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sm), 0);
    const uint32_t d_lbo = (g.d_bytes >> 4) << 16;
    int st = 0;
    uint32_t ph = 0;
    uint32_t accum = 0;
    int t = q_beg % g.T_img;
    for (int qb = q_beg; qb < q_end; ++qb, (++t == g.T_img ? (t = 0) : 0)) {
      int q0 = 128 * t;
      int row_off = q0 - (q0 / g.Wp) * g.Wp;
      if (leader) C2_TRACE(1, qb - q_beg, 0);
      ptx::mbar_wait(&full[st], ph);
      if (leader) C2_TRACE(1, qb - q_beg, 1);
      ptx::tc_fence_after();
      const uint32_t d_lo = s_lo0 + st * (stage_bytes >> 4) + row_off * 8 + d_lbo;
      const uint32_t x_lo = s_lo0 + st * (stage_bytes >> 4) + ((g.ntb * g.d_bytes) >> 4) + row_off * 8;
      if (leader) {
        for (int p = p_beg; p < p_end; ++p) {
          int t0 = 2 * p, t1 = (2 * p + 1 < rr) ? 2 * p + 1 : 2 * p;
          int o0 = (t0 / g.r) * g.Wp + t0 % g.r, o1 = (t1 / g.r) * g.Wp + t1 % g.r;
          const uint32_t a_lo = x_lo + o0 * 8 + ((uint32_t)((o1 - o0) * 8) << 16);
          const uint32_t dt = tmem + (p - p_beg) * g.NT;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            ptx::mma_bf16(dt, ptx::mk_desc(DHI, a_lo + 128 * k), ptx::mk_desc(DHI, d_lo + 128 * k), IDESC,
                          accum | (uint32_t)k);
        }
        ptx::mma_commit(&empty[st]);
        C2_TRACE(1, qb - q_beg, 2);
      }
      accum = 1;
      __syncwarp();
      if (++st == g.stages) { st = 0; ph ^= 1; }
    }
    if (leader) ptx::mma_commit(done);
    __syncwarp();
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const bool has_work = q_end > q_beg;
    if (has_work) {
      ptx::mbar_wait(done, 0);
      ptx::tc_fence_after();
    }
    float* dst = g.part + (size_t)split * g.Jd * g.Kf;
    for (int p = p_beg; p < p_end; ++p) {
      int tap = row < 64 ? 2 * p : 2 * p + 1;
      bool ok = tap < rr;
      int k = half * g.K0 + tap * g.C + cb * 64 + (row & 63);
#pragma unroll 1
      for (int c = 0; c < g.NT; c += 16) {
        float v[16];
        if (has_work) {
          ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (p - p_beg) * g.NT + c, v);
          ptx::tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = 0.f;
        }
        if (ok) {
#pragma unroll
          for (int e = 0; e < 16; ++e) dst[(size_t)(jt * g.NT + c + e) * g.Kf + k] = v[e];
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (g.trace && threadIdx.x == 0 && blockIdx.x < 512) g.trace[3072 + 2 * blockIdx.x + 1] = gtimer();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

struct W2Plan {
  bool ok;
  W2Args g;
  size_t smem;
};

static W2Plan w2_plan(const Plan& P) {
  W2Plan pl;
  memset(&pl, 0, sizeof(pl));
  W2Args& g = pl.g;
  if (P.s != 1 || P.r < 2 || P.C % 64 || P.Jd % 64) return pl;
  int Wp = P.W + 2 * P.p;
  if (P.OW != Wp - P.r + 1 || Wp > 256 || P.OW < 12) return pl;
  int T_img = (P.OH * Wp + 127) / 128;
  int RD = 0;
  for (int t = 0; t < T_img; ++t) {
    int q0 = 128 * t, lo = q0 / Wp, hi = (q0 + 127) / Wp;
    if (hi - lo + 1 > RD) RD = hi - lo + 1;
  }
  int RX = 0;  // x halo rows: q0 .. q0 + 127 + (r-1)(Wp+1)
  for (int t = 0; t < T_img; ++t) {
    int q0 = 128 * t, lo = q0 / Wp, hi = (q0 + 127 + (P.r - 1) * (Wp + 1)) / Wp;
    if (hi - lo + 1 > RX) RX = hi - lo + 1;
  }
  if (RX > 256) return pl;
  uint32_t d_tx = (uint32_t)Wp * RD * 128, x_tx = (uint32_t)Wp * RX * 128;
  uint32_t d_bytes = (d_tx + 1023) / 1024 * 1024, x_bytes = (x_tx + 1023) / 1024 * 1024;
  // N tile: the widest multiple of 64 (<= 256, dividing Jd) whose stage still
  // double-buffers in smem (192 for proposed F = 64 at 32x32; narrower for wide images)
  int ntb = 0, stages = 0;
  for (int c = 4; c >= 1; --c) {
    if ((P.Jd / 64) % c) continue;
    uint32_t stg = c * d_bytes + x_bytes;
    int sn = (int)((212 * 1024) / stg);
    if (sn >= 2) { ntb = c; stages = sn > 4 ? 4 : sn; break; }
  }
  if (ntb == 0) return pl;
  const int NT = ntb * 64;
  const int npairs = (P.r * P.r + 1) / 2;
  int pp = 512 / NT;
  if (pp > npairs) pp = npairs;
  const int tgroups = (npairs + pp - 1) / pp;
  g.N = P.N; g.OHg = P.OH; g.OWg = P.OW; g.Jd = P.Jd; g.Kf = P.Kf; g.K0 = P.K0; g.C = P.C;
  g.pe = P.p; g.r = P.r; g.Wp = Wp; g.RD = RD; g.RX = RX;
  g.T_img = T_img; g.cblks = P.C / 64; g.ablocks = g.cblks * (P.sq == 2 ? 2 : 1); g.jtiles = P.Jd / NT;
  g.NT = NT; g.ntb = ntb; g.npairs = npairs; g.pp = pp; g.tgroups = tgroups;
  if (tgroups > 16) return pl;
  // CTA budget per (j tile, channel block), shared among tap groups by their pair count
  int budget = tc_num_sms() / (g.jtiles * g.ablocks);
  if (budget < tgroups) budget = tgroups;
  int nblk = P.N * T_img;
  // per-q-block cost of a group ~ max(MMA issue, TMA fill): traced at ~NT/2 cycles per
  // M128 MMA (+~400 loop) and ~64 B/cycle of TMA per SM
  const double tma_cyc = (double)(ntb * d_bytes + x_bytes) / 64.0;
  double wsum = 0, wg[16];
  for (int t = 0; t < tgroups; ++t) {
    int pg = min(pp, npairs - t * pp);
    double mma_cyc = pg * 8 * (NT / 2.0) + 400.0;
    wg[t] = mma_cyc > tma_cyc ? mma_cyc : tma_cyc;
    wsum += wg[t];
  }
  int smax = 1, tot = 0;
  for (int t = 0; t < tgroups; ++t) {
    int sg = (int)(budget * wg[t] / wsum);
    if (sg < 1) sg = 1;
    if (sg > nblk) sg = nblk;
    g.gsplit[t] = sg;
    g.gstart[t] = tot;
    tot += sg;
    if (sg > smax) smax = sg;
  }
  g.gstart[tgroups] = tot;
  g.splits = smax;  // partial slots; rows of group t use slots [0, gsplit[t])
  g.d_tx = d_tx; g.x_tx = x_tx; g.d_bytes = d_bytes; g.x_bytes = x_bytes; g.stages = stages;
  pl.smem = 1024 + (size_t)stages * (ntb * d_bytes + x_bytes) + 1024;
  pl.ok = true;
  return pl;
}

// ===========================================================================
// K4 v3 (r = 3): wgrad on CTA pairs sharing every stage load.
//   Both CTAs of a cluster walk the same q blocks; each issues half of the
//   stage's TMA boxes (D boxes, x halo) multicast to both, so D and x are read
//   from L2 once per pair instead of once per tap group. CTA r accumulates tap
//   pairs {2r, 2r+1} over the whole N tile plus the ninth tap over its share
//   of the N boxes (CTA0: the first ntb/2 boxes, CTA1: the rest), so the
//   pair's TMEM holds every tap: 2 NT + ceil(ntb/2) 64 <= 512 columns.
//   Stage release needs both CTAs' MMAs: each commit is multicast to both
//   CTAs' empty barriers (count 2). Partials: one slot per cluster.
// ===========================================================================
struct W3Args {
  int N, OHg, OWg, Jd, Kf, K0, C;
  int pe, Wp, RD, RX;
  int T_img, cblks, ablocks, jtiles, nsplit;
  int NT, ntb;
  int R, ksteps;  // a q block = R whole rows of the padded grid (R Wp positions), ksteps x 16 MMA K
  uint32_t d_tx, x_tx, d_bytes, x_bytes;
  int stages;
  int jsplit;
  float* part;
  unsigned long long* trace;  // QD_TRACE (dev only)
  // in-kernel fold (fold_bar != null): after a grid barrier each CTA sums whole
  // (j, half, channel block) units of the partial slots in a fixed order and
  // writes them transposed into the reference (F, C, 3, 3) layouts
  int fold_slot;  // >= 0: fold in-kernel, grid barrier on counter slot fold_slot
  float* dw0;
  float* dw1;
  float* dw2;
  const float* bpart;  // bias partial sums [SB][Jd] (prologue / BN emit), folded here too
  int SB;
  float* db0;
  float* db1;
  float* db2;
  Plan P;
};

// grid barrier of the in-kernel fold: a sense-reversing barrier per slot. Each
// CTA reads the slot's generation, arrives on the count; the last arrival
// re-arms the count and publishes generation + 1, the others wait for the
// generation to move. Nothing is reset "after" the barrier, so a replay (or
// a launch of another shape on the same slot) never sees a stale count.
// Launches take slots from a host-side atomic round-robin allocator; only 64
// fold launches in flight at once could share a slot.
__device__ unsigned g_w3_count[64];
__device__ unsigned g_w3_gen[64];

// grid barrier over a co-resident grid (thread 0 of each CTA calls it between
// two __syncthreads). A wait past `timeout_ns` traps: a co-residency violation
// becomes a loud launch failure instead of a hang.
__device__ __forceinline__ void w3_grid_barrier(int slot, unsigned long long timeout_ns) {
  unsigned* cnt = &g_w3_count[slot];
  unsigned* gen = &g_w3_gen[slot];
  unsigned my;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(my) : "l"(gen) : "memory");
  __threadfence();  // this CTA's partial stores before its arrival
  if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
    atomicExch(cnt, 0u);
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(my + 1u) : "memory");
  } else {
    const unsigned long long t0 = gtimer();
    unsigned g;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
      if (g != my) break;
      __nanosleep(64);
      if (gtimer() - t0 > timeout_ns) __trap();
    }
  }
}

__device__ __forceinline__ void w3_tma4_mc(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                           int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(ptx::smem_u32(dst)),
      "l"(m), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void w3_commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          ptx::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    wgrad3_kernel(const __grid_constant__ CUtensorMap mX0, const __grid_constant__ CUtensorMap mX1,
                  const __grid_constant__ CUtensorMap mD, const __grid_constant__ CUtensorMap mD1,
                  const W3Args g) {
  if (g.trace && threadIdx.x == 0 && blockIdx.x < 512) {
    g.trace[3072 + 2 * blockIdx.x] = gtimer();
    g.trace[2048 + 2 * blockIdx.x] = clock64();
  }
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t stage_bytes = g.ntb * g.d_bytes + g.x_bytes;
  uint64_t* full = (uint64_t*)(sm + g.stages * stage_bytes);
  uint64_t* empty = full + g.stages;
  uint64_t* done = empty + g.stages;
  uint32_t* tslot = (uint32_t*)(done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = c2::cluster_rank();
  int b = blockIdx.x >> 1;
  const int jt = b % g.jtiles;
  b /= g.jtiles;
  const int ab = b % g.ablocks;
  const int split = b / g.ablocks;
  const int half = ab / g.cblks, cb = ab % g.cblks;
  const int nblk = g.N * g.T_img;
  const int q_beg = (int)((long long)split * nblk / g.nsplit);
  const int q_end = (int)((long long)(split + 1) * nblk / g.nsplit);
  // ninth tap: CTA r takes N boxes [nlo, nhi)
  const int nlo = rank == 0 ? 0 : g.ntb / 2;
  const int nhi = rank == 0 ? g.ntb / 2 : g.ntb;

  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&mX0);
    ptx::prefetch_tmap(&mX1);
    ptx::prefetch_tmap(&mD);
    if (g.jsplit) ptx::prefetch_tmap(&mD1);
    for (int i = 0; i < g.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 2);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(tslot, 512);
    ptx::tmem_relinquish();
  }
  {
    // the slot tails past each box (K padding to 16 positions; the x rows the
    // last K step may touch) are never written by TMA: zero them once. They
    // only ever meet zero D / finite x, so they add nothing.
    const uint32_t d_box = (uint32_t)g.RD * g.Wp * 128, x_box = (uint32_t)g.RX * g.Wp * 128;
    for (int s = 0; s < g.stages; ++s) {
      uint8_t* base = sm + s * stage_bytes;
      for (int i = 0; i <= g.ntb; ++i) {
        uint8_t* slot = base + i * g.d_bytes;
        const uint32_t lo = i < g.ntb ? d_box : x_box, hi = i < g.ntb ? g.d_bytes : g.x_bytes;
        for (uint32_t o = lo + 16 * threadIdx.x; o < hi; o += 16 * blockDim.x)
          *(uint4*)(slot + o) = make_uint4(0, 0, 0, 0);
      }
    }
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  c2::cluster_sync();  // barriers of both CTAs initialised before any multicast lands
  ptx::tc_fence_after();
  ptx::pdl_wait();
  ptx::pdl_launch();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    const bool leader = ptx::elect_one();
    int st = 0;
    uint32_t ph = 0;
    // box i < ntb: D box i; i == ntb: the x halo. CTA0 issues [0, nsh), CTA1 the rest.
    const int nsh = (g.ntb + 1) / 2;
    int n = q_beg / g.T_img, t = q_beg % g.T_img;  // walked incrementally below
    for (int qb = q_beg; qb < q_end; ++qb, (++t == g.T_img ? (t = 0, ++n) : 0)) {
      int hq_lo = g.R * t;
      if (leader) C2_TRACE(0, qb - q_beg, 0);
      ptx::mbar_wait(&empty[st], ph ^ 1);
      if (leader) {
        C2_TRACE(0, qb - q_beg, 1);
        uint8_t* s = sm + st * stage_bytes;
        ptx::mbar_arrive_expect_tx(&full[st], g.ntb * g.d_tx + g.x_tx);
        const int i0 = rank == 0 ? 0 : nsh, i1 = rank == 0 ? nsh : g.ntb + 1;
        for (int i = i0; i < i1; ++i) {
          if (i == g.ntb) {
            w3_tma4_mc(half ? &mX1 : &mX0, &full[st], s + g.ntb * g.d_bytes, cb * 64, -g.pe, hq_lo - g.pe, n);
          } else {
            const int jb = jt * g.ntb + i;
            if (g.jsplit && jb >= g.jsplit)
              w3_tma4_mc(&mD1, &full[st], s + i * g.d_bytes, (jb - g.jsplit) * 64, 0, hq_lo, n);
            else
              w3_tma4_mc(&mD, &full[st], s + i * g.d_bytes, jb * 64, 0, hq_lo, n);
          }
        }
      }
      __syncwarp();
      if (++st == g.stages) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    const uint32_t IDESC = ptx::idesc_bf16(128, g.NT, true, true);
    const uint32_t IDESC9 = ptx::idesc_bf16(128, (nhi - nlo) * 64, true, true);
    constexpr uint32_t DHI = ptx::sw128_desc_hi(1024);
    const bool leader = ptx::elect_one();
    const uint32_t s_lo0 = ptx::sw128_desc_lo(ptx::smem_u32(sm), 0);
    const uint32_t d_lbo = (g.d_bytes >> 4) << 16;
    // tap offsets in the halo (rows): pairs {2r, 2r+1}, {2r+2... } of this CTA; tap 8 = (2, 2)
    const int ta = 4 * (int)rank;  // taps ta .. ta+3
    int off[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) off[i] = ((ta + i) / 3) * g.Wp + (ta + i) % 3;
    const int off8 = 2 * g.Wp + 2;
    int st = 0;
    uint32_t ph = 0;
    uint32_t accum = 0;
    const int ks = g.ksteps;
    for (int qb = q_beg; qb < q_end; ++qb) {
      if (leader) C2_TRACE(1, qb - q_beg, 0);
      ptx::mbar_wait(&full[st], ph);
      if (leader) C2_TRACE(1, qb - q_beg, 1);
      ptx::tc_fence_after();
      const uint32_t base = s_lo0 + st * (stage_bytes >> 4);
      const uint32_t d_lo = base + d_lbo;
      const uint32_t x_lo = base + ((g.ntb * g.d_bytes) >> 4);
      if (leader) {
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
          const int o0 = off[2 * pr], o1 = off[2 * pr + 1];
          const uint32_t a_lo = x_lo + o0 * 8 + ((uint32_t)((o1 - o0) * 8) << 16);
          const uint32_t dt = tmem + pr * g.NT;
#pragma unroll 4
          for (int k = 0; k < ks; ++k)
            ptx::mma_bf16(dt, ptx::mk_desc(DHI, a_lo + 128 * k), ptx::mk_desc(DHI, d_lo + 128 * k), IDESC,
                          accum | (uint32_t)(k > 0));
        }
        if (nhi > nlo) {
          const uint32_t a_lo = x_lo + off8 * 8;  // both 64-row atoms: tap 8 (second discarded)
          const uint32_t b_lo = d_lo + nlo * (g.d_bytes >> 4);
          const uint32_t dt = tmem + 2 * g.NT;
#pragma unroll 4
          for (int k = 0; k < ks; ++k)
            ptx::mma_bf16(dt, ptx::mk_desc(DHI, a_lo + 128 * k), ptx::mk_desc(DHI, b_lo + 128 * k), IDESC9,
                          accum | (uint32_t)(k > 0));
        }
        w3_commit_mc(&empty[st]);
        C2_TRACE(1, qb - q_beg, 2);
      }
      accum = 1;
      __syncwarp();
      if (++st == g.stages) { st = 0; ph ^= 1; }
    }
    if (leader) ptx::mma_commit(done);
    __syncwarp();
  }
  {
    // ===== epilogue on all 8 warps: warp w reads TMEM lanes 32 (w % 4) and
    // stores half h = w / 4 of every accumulator's columns =====
    const int q = warp & 3, hh = warp >> 2;
    const int row = q * 32 + lane;
    const bool has_work = q_end > q_beg;
    if (has_work) {
      ptx::mbar_wait(done, 0);
      ptx::tc_fence_after();
    }
    if (g.trace && threadIdx.x == 0 && blockIdx.x < 1024) g.trace[4096 + blockIdx.x] = gtimer();  // main loop done
    float* dst = g.part + (size_t)split * g.Jd * g.Kf;
    // accumulators: 0, 1 = tap pairs of this CTA over NT; 2 = tap 8 over boxes [nlo, nhi)
    for (int acc = 0; acc < 3; ++acc) {
      int tap, c_lo, c_hi;
      if (acc < 2) {
        tap = 4 * (int)rank + 2 * acc + (row < 64 ? 0 : 1);
        c_lo = 0;
        c_hi = g.NT;
      } else {
        tap = 8;
        c_lo = nlo * 64;
        c_hi = nhi * 64;
        if (q >= 2) continue;  // rows 64..127 hold the duplicate atom (warp-uniform skip)
      }
      const bool ok = c_hi > c_lo;
      const int k = half * g.K0 + tap * g.C + cb * 64 + (row & 63);
      const int ncols = (acc < 2) ? g.NT : (nhi - nlo) * 64;
      const int cw = ncols / 2;
#pragma unroll 1
      for (int c = hh * cw; c < (hh + 1) * cw; c += 16) {
        float v[16];
        if (has_work) {
          ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * g.NT + c, v);
          ptx::tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = 0.f;
        }
        if (ok) {
          const int j0 = jt * g.NT + c_lo + c;
#pragma unroll
          for (int e = 0; e < 16; ++e) dst[(size_t)(j0 + e) * g.Kf + k] = v[e];
        }
      }
    }
  }
  ptx::tc_fence_before();
  c2::cluster_sync();  // no CTA exits while its partner may still multicast into it
  if (g.fold_slot >= 0) {
    // ===== in-kernel fold. Every CTA of the (persistent, co-resident) grid has
    // stored its slot region: grid barrier (release / acquire at GPU scope) =====
    __syncthreads();
    if (threadIdx.x == 0) w3_grid_barrier(g.fold_slot, 20000000000ull);
    __syncthreads();
    const Plan& P = g.P;
    // bias partial sums: 8 columns x 32 split groups per pass, fixed order
    if (g.db0 && P.nbias) {
      float* redb = reinterpret_cast<float*>(sm);
      const int bc = threadIdx.x % 8, bg = threadIdx.x / 8;
      for (int bb = blockIdx.x; bb * 8 < P.Jd; bb += gridDim.x) {
        const int j = bb * 8 + bc;
        float a0 = 0.f, a1 = 0.f;
        if (j < P.Jd) {
          int s2 = bg;
          for (; s2 + 32 < g.SB; s2 += 64) {
            a0 += __ldcg(g.bpart + (size_t)s2 * P.Jd + j);
            a1 += __ldcg(g.bpart + (size_t)(s2 + 32) * P.Jd + j);
          }
          for (; s2 < g.SB; s2 += 32) a0 += __ldcg(g.bpart + (size_t)s2 * P.Jd + j);
        }
        redb[bg * 9 + bc] = a0 + a1;
        __syncthreads();
        if (bg == 0 && j < P.Jd) {
          float t = 0.f;
          for (int gq = 0; gq < 32; ++gq) t += redb[gq * 9 + bc];
          const int role = j / P.F, f = j % P.F;
          float* dst = role == 0 ? g.db0 : (role == 1 ? g.db1 : g.db2);
          if (dst) dst[f] = t;
        }
        __syncthreads();
      }
    }
    // unit = (j, half, 64-channel block): 9 taps x 64 channels = 144 float4
    // columns of partial row j, summed over the slots in a fixed order (four
    // interleaved chains, combined in order), transposed through shared memory
    // (the stage buffers are idle: every load landed and every MMA retired) and
    // written as one contiguous 576-float run of dW[role][f][cb*64 ..][9]
    const int nh = P.Kf / P.K0, units = P.Jd * nh * g.cblks, S = g.nsplit;
    const long long slot4 = (long long)P.Jd * P.Kf / 4;
    const float4* part4 = reinterpret_cast<const float4*>(g.part);
    float* red = reinterpret_cast<float*>(sm);
    // units per batch: as many 576-float tiles as the stage buffers hold (<= 64)
    const int UB = min(64, (int)((g.stages * stage_bytes) / 2304));
    for (int u0 = blockIdx.x; u0 < units; u0 += UB * gridDim.x) {
      int nu = 0;
      for (int u = u0; u < units && nu < UB; u += gridDim.x) ++nu;
      for (int i = threadIdx.x; i < nu * 144; i += blockDim.x) {
        const int ul = i / 144, col = i - ul * 144, u = u0 + ul * gridDim.x;
        const int cbk = u % g.cblks, rest = u / g.cblks, hf = rest % nh, j = rest / nh;
        const int tap = col >> 4, c4 = col & 15;
        const long long o4 = ((long long)j * P.Kf + hf * P.K0 + tap * P.C + cbk * 64) / 4 + c4;
        // eight independent chains (8 loads in flight per thread: the fold is
        // L2-latency bound), combined in a fixed order
        float4 ac[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) ac[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        int sl = 0;
        for (; sl + 7 < S; sl += 8) {
          float4 v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __ldcg(part4 + (sl + e) * slot4 + o4);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            ac[e].x += v[e].x; ac[e].y += v[e].y; ac[e].z += v[e].z; ac[e].w += v[e].w;
          }
        }
        for (; sl < S; ++sl) {
          const float4 v = __ldcg(part4 + sl * slot4 + o4);
          ac[0].x += v.x; ac[0].y += v.y; ac[0].z += v.z; ac[0].w += v.w;
        }
#pragma unroll
        for (int e = 4; e > 0; e >>= 1)
#pragma unroll
          for (int i2 = 0; i2 < e; ++i2) {
            ac[i2].x += ac[i2 + e].x; ac[i2].y += ac[i2 + e].y; ac[i2].z += ac[i2 + e].z; ac[i2].w += ac[i2 + e].w;
          }
        const float t[4] = {ac[0].x, ac[0].y, ac[0].z, ac[0].w};
        float* ru = red + ul * 576;
#pragma unroll
        for (int e = 0; e < 4; ++e) ru[(c4 * 4 + e) * 9 + tap] = t[e];  // (c, tap) order
      }
      __syncthreads();
      for (int i = threadIdx.x; i < nu * 144; i += blockDim.x) {
        const int ul = i / 144, q4 = i - ul * 144, u = u0 + ul * gridDim.x;
        const int cbk = u % g.cblks, rest = u / g.cblks, hf = rest % nh, j = rest / nh;
        int role, f, kk;
        if (!wgrad_dst(P, j, hf * P.K0, role, f, kk)) continue;  // t2and4 structural zero
        float* dst = role == 0 ? g.dw0 : (role == 1 ? g.dw1 : g.dw2);
        if (!dst) continue;
        const float4 v = *reinterpret_cast<const float4*>(red + ul * 576 + 4 * q4);
        reinterpret_cast<float4*>(dst + ((size_t)f * P.C + cbk * 64) * 9)[q4] = v;
      }
      __syncthreads();
    }
  }
  if (g.trace && threadIdx.x == 0 && blockIdx.x < 512) {
    g.trace[3072 + 2 * blockIdx.x + 1] = gtimer();
    g.trace[2048 + 2 * blockIdx.x + 1] = clock64();
  }
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

struct W3Plan {
  bool ok;
  W3Args g;
  size_t smem;
};

static W3Plan w3_plan(const Plan& P) {
  W3Plan pl;
  memset(&pl, 0, sizeof(pl));
  W3Args& g = pl.g;
  if (getenv("QD_NO_W3")) return pl;
  if (P.s != 1 || P.r != 3 || P.C % 64 || P.Jd % 64) return pl;
  int Wp = P.W + 2 * P.p;
  if (P.OW != Wp - P.r + 1 || Wp > 256 || P.OW < 12) return pl;
  // q blocks of R whole rows: the D box is exactly the block (no row overfetch)
  // and K = R Wp padded to 16. Pick R by MMA efficiency (positions computed /
  // positions issued, incl. the rows past OH of the last block), then by bytes
  // staged per position, with at least 2 stages.
  int ntb = 0, stages = 0, R = 0, ksteps = 0;
  uint32_t d_tx = 0, x_tx = 0, d_bytes = 0, x_bytes = 0;
  for (int c = 3; c >= 1 && !ntb; --c) {  // 2 NT + ceil(c/2) 64 <= 512
    if ((P.Jd / 64) % c) continue;
    double best = 0.0;
    const int rpin = getenv("QD_W3_R") ? atoi(getenv("QD_W3_R")) : 0;  // dev: pin R
    for (int rr = 1; rr <= P.OH && rr + P.r - 1 <= 256; ++rr) {
      const int kst = (rr * Wp + 15) / 16;
      const uint32_t db = (uint32_t)kst * 16 * 128;  // multiple of 2048
      const uint32_t xb = ((uint32_t)(kst * 16 + (P.r - 1) * (Wp + 1)) * 128 + 1023) / 1024 * 1024;
      const uint32_t stg = c * db + xb;
      const int sn = (int)((212 * 1024) / stg);
      if (sn < 2) break;
      const int tb = (P.OH + rr - 1) / rr;
      const double eff = (double)P.OH * Wp / ((double)tb * kst * 16);
      const double score = rpin ? (rr == rpin ? 1.0 : 0.0) : eff - 1e-7 * stg / (rr * Wp);
      if (score > best) {
        best = score;
        ntb = c; stages = sn > 4 ? 4 : sn; R = rr; ksteps = kst;
        d_tx = (uint32_t)Wp * rr * 128; x_tx = (uint32_t)Wp * (rr + P.r - 1) * 128;
        d_bytes = db; x_bytes = xb;
      }
    }
  }
  const int RD = R, RX = R + P.r - 1, T_img = R ? (P.OH + R - 1) / R : 0;
  // narrow N tiles (wide images) re-read x per j tile and run N = 64 MMAs: wgrad2 is better there
  if (ntb < 2) return pl;
  g.N = P.N; g.OHg = P.OH; g.OWg = P.OW; g.Jd = P.Jd; g.Kf = P.Kf; g.K0 = P.K0; g.C = P.C;
  g.pe = P.p; g.Wp = Wp; g.RD = RD; g.RX = RX; g.R = R; g.ksteps = ksteps;
  g.T_img = T_img; g.cblks = P.C / 64; g.ablocks = g.cblks * (P.sq == 2 ? 2 : 1);
  g.NT = ntb * 64; g.ntb = ntb; g.jtiles = P.Jd / g.NT;
  const int nblk = P.N * T_img;
  pl.smem = 1024 + (size_t)stages * (ntb * d_bytes + x_bytes) + 1024;
  thread_local int maxc_[kMaxDev] = {};
  thread_local size_t maxc_smem_[kMaxDev] = {};
  int& maxc = maxc_[cur_device()];
  size_t& maxc_smem = maxc_smem_[cur_device()];
  if (maxc == 0 || maxc_smem != pl.smem) {
    raise_smem_attr((const void*)wgrad3_kernel, pl.smem);
    maxc = max_pair_clusters(wgrad3_kernel, 256, pl.smem);
    maxc_smem = pl.smem;
  }
  int pairs = tc_num_sms() / 2;
  if (maxc > 0 && maxc < pairs) pairs = maxc;
  int ns = pairs / (g.jtiles * g.ablocks);
  if (ns < 1) ns = 1;
  if (ns > nblk) ns = nblk;
  g.nsplit = ns;
  g.d_tx = d_tx; g.x_tx = x_tx; g.d_bytes = d_bytes; g.x_bytes = x_bytes; g.stages = stages;
  pl.smem = 1024 + (size_t)stages * (ntb * d_bytes + x_bytes) + 1024;
  pl.ok = true;
  return pl;
}

int wgrad3_split(const Plan& P) {
  W3Plan pl = w3_plan(P);
  return pl.ok ? pl.g.nsplit : 0;
}

// SM pairs one split of the v3 wgrad occupies (its grid is this x nsplit pairs)
int wgrad3_pairs_per_split(const Plan& P) {
  W3Plan pl = w3_plan(P);
  return pl.ok ? pl.g.jtiles * pl.g.ablocks : 0;
}

int run_wgrad3(const Plan& P, const void* x0, const void* x1, const void* D, float* part, int splits,
               cudaStream_t st, const void* Dtail, int jsplit, float* const* dW, const float* bpart, int SB,
               float* const* db, bool* folded) {
  if (dev_skip("wgrad")) return QD_OK;
  W3Plan pl = w3_plan(P);
  // splits < the plan's: a partitioned launch sharing the SMs with a concurrent kernel
  if (!pl.ok || splits < 1 || splits > pl.g.nsplit) return QD_ERR_UNSUPPORTED;
  W3Args& g = pl.g;
  g.nsplit = splits;
  g.part = part;
  g.fold_slot = -1;
  g.P = P;
  if (folded) *folded = false;
  if (dW && dW[0]) {
    // the grid barrier needs every CTA resident at once: the grid never exceeds
    // the co-resident clusters (w3_plan), and the launch is cooperative (the
    // driver then guarantees co-residency even beside other kernels)
    static std::atomic<unsigned> slot{0};
    g.fold_slot = (int)(slot.fetch_add(1u) % 64u);
    g.dw0 = dW[0]; g.dw1 = dW[1]; g.dw2 = dW[2];
    g.bpart = bpart; g.SB = SB;
    g.db0 = db ? db[0] : nullptr; g.db1 = db ? db[1] : nullptr; g.db2 = db ? db[2] : nullptr;
  }
  g.trace = getenv("QD_TRACE") ? trace_buffer() : nullptr;
  CUtensorMap X0, X1, Dm, Dm1;
  int rc;
  cuuint64_t dX[4] = {(cuuint64_t)P.C, (cuuint64_t)P.W, (cuuint64_t)P.H, (cuuint64_t)P.N};
  cuuint32_t bX[4] = {64, (cuuint32_t)g.Wp, (cuuint32_t)g.RX, 1};
  if ((rc = c2_map(&X0, x0, 4, dX, bX))) return rc;
  if ((rc = c2_map(&X1, x1 ? x1 : x0, 4, dX, bX))) return rc;
  g.jsplit = (Dtail && jsplit > 0 && jsplit < P.Jd / 64) ? jsplit : 0;
  cuuint64_t dD[4] = {(cuuint64_t)(g.jsplit ? 64 * g.jsplit : P.Jd), (cuuint64_t)P.OW, (cuuint64_t)P.OH,
                      (cuuint64_t)P.N};
  cuuint32_t bD[4] = {64, (cuuint32_t)g.Wp, (cuuint32_t)g.RD, 1};
  if ((rc = c2_map(&Dm, D, 4, dD, bD))) return rc;
  Dm1 = Dm;
  if (g.jsplit) {
    cuuint64_t d1[4] = {(cuuint64_t)(P.Jd - 64 * g.jsplit), (cuuint64_t)P.OW, (cuuint64_t)P.OH, (cuuint64_t)P.N};
    if ((rc = c2_map(&Dm1, Dtail, 4, d1, bD))) return rc;
  }
  raise_smem_attr((const void*)wgrad3_kernel, pl.smem);
  const dim3 grid(2 * g.jtiles * g.ablocks * g.nsplit);
  if (g.fold_slot >= 0) {
    // in-kernel fold: cooperative launch (co-residency guaranteed by the driver);
    // if the driver refuses it, the caller folds with separate kernels instead
    const char* ce = getenv("QD_W3_COOP");
    const bool coop = !(ce && atoi(ce) == 0);
    if (cudaLaunchCoop(wgrad3_kernel, grid, dim3(256), pl.smem, st, coop, X0, X1, Dm, Dm1, g) == cudaSuccess) {
      if (folded) *folded = true;
      count_launch(st, "wgrad3");
      return check_launch("wgrad3");
    }
    cudaGetLastError();
    g.fold_slot = -1;
  }
  launch_pdl(wgrad3_kernel, grid, dim3(256), pl.smem, st, X0, X1, Dm, Dm1, g);
  count_launch(st, "wgrad3");
  return check_launch("wgrad3");
}

// rows of BN statistics the conv2 fprop epilogue writes for this geometry (0: not eligible)
int conv2_stat_rows(int N, int Cin, int Win, int Hin, int OWg, int OHg, int pe, int r, int dual, int nbk, int nout,
                    int tiles_nn, int Cout, int nbias) {
  C2Plan pl = c2_plan(N, Cin, Win, Hin, OWg, OHg, pe, r, dual, nbk, nout, tiles_nn, Cout, nbias);
  return pl.ok ? ((N + 1) / 2) * pl.g.T_img * 8 : 0;
}

bool conv2_fits(int N, int Cin, int Win, int Hin, int OWg, int OHg, int pe, int r, int dual, int nbk, int nout,
                int tiles_nn, int Cout, int nbias) {
  return c2_plan(N, Cin, Win, Hin, OWg, OHg, pe, r, dual, nbk, nout, tiles_nn, Cout, nbias).ok;
}

int wgrad2_split(const Plan& P) {
  W2Plan pl = w2_plan(P);
  return pl.ok ? pl.g.splits : 0;
}

WSplits wgrad2_splits(const Plan& P) {
  W2Plan pl = w2_plan(P);
  WSplits w;
  memset(&w, 0, sizeof(w));
  if (!pl.ok) return w;
  w.pp = pl.g.pp;
  w.ng = pl.g.tgroups;
  for (int t = 0; t < w.ng; ++t) w.s[t] = pl.g.gsplit[t];
  return w;
}

int run_wgrad2(const Plan& P, const void* x0, const void* x1, const void* D, float* part, int splits,
               cudaStream_t st, const void* Dtail, int jsplit) {
  W2Plan pl = w2_plan(P);
  if (!pl.ok || pl.g.splits != splits) return QD_ERR_UNSUPPORTED;
  W2Args& g = pl.g;
  g.part = part;
  g.trace = getenv("QD_TRACE") ? trace_buffer() : nullptr;
  CUtensorMap X0, X1, Dm, Dm1;
  int rc;
  cuuint64_t dX[4] = {(cuuint64_t)P.C, (cuuint64_t)P.W, (cuuint64_t)P.H, (cuuint64_t)P.N};
  cuuint32_t bX[4] = {64, (cuuint32_t)g.Wp, (cuuint32_t)g.RX, 1};
  if ((rc = c2_map(&X0, x0, 4, dX, bX))) return rc;
  if ((rc = c2_map(&X1, x1 ? x1 : x0, 4, dX, bX))) return rc;
  g.jsplit = (Dtail && jsplit > 0 && jsplit < P.Jd / 64) ? jsplit : 0;
  cuuint64_t dD[4] = {(cuuint64_t)(g.jsplit ? 64 * g.jsplit : P.Jd), (cuuint64_t)P.OW, (cuuint64_t)P.OH,
                      (cuuint64_t)P.N};
  cuuint32_t bD[4] = {64, (cuuint32_t)g.Wp, (cuuint32_t)g.RD, 1};
  if ((rc = c2_map(&Dm, D, 4, dD, bD))) return rc;
  Dm1 = Dm;
  if (g.jsplit) {
    cuuint64_t d1[4] = {(cuuint64_t)(P.Jd - 64 * g.jsplit), (cuuint64_t)P.OW, (cuuint64_t)P.OH, (cuuint64_t)P.N};
    if ((rc = c2_map(&Dm1, Dtail, 4, d1, bD))) return rc;
  }
  raise_smem_attr((const void*)wgrad2_kernel, pl.smem);
  launch_pdl(wgrad2_kernel, dim3(g.jtiles * g.ablocks * g.gstart[g.tgroups]), dim3(256), pl.smem, st, X0, X1, Dm,
             Dm1, g);
  count_launch(st, "wgrad2");
  return check_launch("wgrad2");
}

}  // namespace qd
