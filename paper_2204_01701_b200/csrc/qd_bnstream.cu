// The BN backward's D emission in streaming form (
// tensor.py:552-570 as qd_bn.cu states it): dy = kA g' + kC y + kB ->
// D = [dy b | dy a | dy] with the layer's bias gradients folded in-kernel.
// An HBM-bound byte stream (4 tensors in, 3 out), built for bytes in flight:
//   - one persistent CTA per SM: 16 consumer warps + one producer warp; the CTA's
//     contiguous range of row tiles ([TR rows][C channels], 16 KB per tensor) is
//     staged into shared memory by 1-D bulk copies (cp.async.bulk ...
//     mbarrier::complete_tx) NST tiles ahead, full / empty mbarriers per stage,
//     so the loads in flight are set by shared memory (192 KB per SM), not by
//     registers, and no consumer waits for another at a CTA barrier;
//   - each thread owns one 16-byte channel chunk (512 % (C / VEC) == 0), so its
//     per-channel constants and bias partial sums stay in registers; packed
//     fp32 pairs (FFMA2 / FADD2 / FMUL2) halve the arithmetic issue;
//   - the bias sums end in the deterministic grid fold of qd_bnfold.cuh: no
//     bias_finish launch.
// The same design for the statistics, apply and backward-reduction passes was
// measured slower than the register-streaming kernels of qd_bn.cu (DESIGN.md
// §9); those keep LDG streaming and take the same in-kernel grid fold.
#include <stdio.h>
#include "qd_kernels.h"
#include "qd_ptx.cuh"
#include "qd_bnfold.cuh"
#include <atomic>

namespace qd {

namespace {
constexpr int kNT = 512;           // consumer threads per CTA (16 warps)
constexpr int kThreads = kNT + 32; // + the producer warp
constexpr int kHdr = 256;          // full / empty mbarriers (<= 16 stages)
// stage geometry per kernel: tile bytes per tensor x stages (128-192 KB per CTA)
constexpr int kEmitTile = 16384, kEmitNst = 4, kEmitNstMat = 3;

struct BnGrid {
  long long M;  // rows
  int C;        // channels
  int TR;       // rows per tile
  long long T;  // tiles
  int S;        // CTAs
};

template <typename T> struct SV;  // 16-byte vectors: shared-memory loads, global stores
template <> struct SV<bf16> {
  static constexpr int V = 8;
  __device__ static void lds(const bf16* p, float v[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      v[2 * e] = f.x;
      v[2 * e + 1] = f.y;
    }
  }
  __device__ static void stg(bf16* p, const float v[8]) {
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
template <> struct SV<float> {
  static constexpr int V = 4;
  __device__ static void lds(const float* p, float v[4]) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
  __device__ static void stg(float* p, const float v[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   ptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
               : "memory");
}

// packed fp32 pairs: FFMA2 / FADD2 / FMUL2 on sm_100 (IEEE round-to-nearest,
// bit-identical to the scalar fmaf / + / *) halve the arithmetic issue of these
// issue-limited passes
__device__ __forceinline__ float2 pr(const float* v, int h) { return make_float2(v[2 * h], v[2 * h + 1]); }

// Stream the CTA's tiles of NIN [M][C] tensors through NST shared-memory stages
// of TB bytes per tensor. Producer warp: waits for a stage to drain, issues its
// bulk copies. Consumer thread i owns chunk q = i % CQ of rows i / CQ + j * lanes
// of each tile: body(in[NIN] (shared pointers to the chunk), global row).
// The producer warp returns at once; consumers return with every copy consumed.
template <typename T, int NIN, int NST, int TB, typename F>
__device__ __forceinline__ void bn_stream(const BnGrid& g, const T* const* src, uint8_t* sm, F&& body) {
  constexpr int V = SV<T>::V;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + NST;
  uint8_t* buf = sm + kHdr;
  const int t0 = (int)((long long)blockIdx.x * g.T / g.S), t1 = (int)((long long)(blockIdx.x + 1) * g.T / g.S);
  const int TR = g.TR;
  if (threadIdx.x >= kNT) {
    // the whole warp walks the loop (lane 0 issues): it leaves converged, so the
    // CTA barriers after the stream (aligned bar.sync) see the full warp
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      if (threadIdx.x == kNT) {
        const int st = i % NST;
        if (i >= NST) ptx::mbar_wait(&empty[st], ((i / NST) - 1) & 1);
        const long long r0 = (long long)t * TR;
        long long nr = g.M - r0;
        if (nr > TR) nr = TR;
        const uint32_t bytes = (uint32_t)(nr * g.C * (long long)sizeof(T));
        ptx::mbar_arrive_expect_tx(&full[st], bytes * NIN);
#pragma unroll
        for (int k = 0; k < NIN; ++k) bulk_g2s(buf + (st * NIN + k) * TB, src[k] + r0 * g.C, bytes, &full[st]);
      }
      __syncwarp();
    }
    return;
  }
  const int CQ = g.C / V, lanes = kNT / CQ, lrow = threadIdx.x / CQ;
  for (int t = t0, i = 0; t < t1; ++t, ++i) {
    const int st = i % NST;
    ptx::mbar_wait_warp(&full[st], (i / NST) & 1);
    const long long r0 = (long long)t * TR;
    const int nr = t == g.T - 1 ? (int)(g.M - r0) : TR;
    const T* base = reinterpret_cast<const T*>(buf + st * NIN * TB) + threadIdx.x * V;
#pragma unroll 2
    for (int rr = lrow; rr < nr; rr += lanes) {
      const T* in[NIN];
#pragma unroll
      for (int k = 0; k < NIN; ++k) in[k] = base + (size_t)k * (TB / sizeof(T)) + (rr - lrow) * g.C;
      body(in, r0 + rr);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&empty[st]);
  }
}

// barriers of the stream: full (one arrival + the tile bytes), empty (one
// arrival per consumer warp)
template <int NST>
__device__ __forceinline__ void bn_stream_init(uint8_t* sm) {
  if (threadIdx.x == 0) {
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    for (int i = 0; i < NST; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&full[NST + i], kNT / 32);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
}

// Per-thread accumulators acc[NACC][V] (chunk q = tid % CQ) -> the CTA's partial
// row part[s][NACC * C] (lane order fixed) -> grid_fold (qd_bnfold.cuh). Returns
// true in the one CTA that then holds the finished sums in fin[NACC * C].
template <int NACC, int V>
__device__ bool bn_grid_fold(const BnGrid& g, float (&acc)[NACC][V], float* part, unsigned* cnt, uint8_t* sm,
                             float* fin) {
  const int C = g.C, CQ = C / V, lanes = kNT / CQ, W = NACC * C, s = blockIdx.x;
  float* red = reinterpret_cast<float*>(sm);  // [NACC][kNT * V]
  __syncthreads();  // red overlays the stage buffers: every warp is done streaming
  if (threadIdx.x < kNT) {
#pragma unroll
    for (int k = 0; k < NACC; ++k)
#pragma unroll
      for (int e = 0; e < V; ++e) red[(k * kNT + threadIdx.x) * V + e] = acc[k][e];
  }
  __syncthreads();
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    const int k = w / C, c = w % C, q = c / V, e = c % V;
    const float* r = red + (size_t)k * kNT * V + q * V + e;
    float t = 0.f;
    for (int l = 0; l < lanes; ++l) t += r[(size_t)l * CQ * V];
    part[(size_t)s * W + w] = t;
  }
  return grid_fold(part, W, fold_geom(g.S), cnt, fin, reinterpret_cast<float4*>(fin + 3 * 2048));
}

// ---- backward D emission ------------------------------------------------------------
// dy = kA g' + kC y + kB (tensor.py:558-566), g' = g masked where kA y + kQ <= 0;
// D row r = [dy b | dy a | dy] (MAT, HASG), [dy b | dy a] (MAT) or dy; NACC sums
// of the written columns are the layer's bias gradients.
template <typename T, bool MAT, bool HASG, bool RELU>
__global__ void __launch_bounds__(kThreads, 1) bns_emit_kernel(BnGrid g, int Jd, const T* __restrict__ dz,
                                                          const T* __restrict__ y, const T* __restrict__ a,
                                                          const T* __restrict__ b, const float* mean,
                                                          const float* invstd, const float* gamma,
                                                          const float* beta, const float* dgamma,
                                                          const float* dbeta, T* __restrict__ D,
                                                          float* part, unsigned* cnt, float* db0,
                                                          float* db1, float* db2) {
  constexpr int V = SV<T>::V, NIN = MAT ? 4 : 2, NST = MAT ? kEmitNstMat : kEmitNst, TB = kEmitTile;
  constexpr int NACC = MAT ? (HASG ? 3 : 2) : 1;
  extern __shared__ __align__(128) uint8_t sm[];
  bn_stream_init<NST>(sm);
  ptx::pdl_wait();  // dgamma / dbeta complete (PDL launch)
  ptx::pdl_launch();
  const int C = g.C, c0 = (threadIdx.x % (C / V)) * V;
  float2 kA[V / 2], kB[V / 2], kC[V / 2], kQ[V / 2], ac[NACC][V / 2];
  {
    const float inv_m = 1.f / (float)g.M;
#pragma unroll
    for (int h = 0; h < V / 2; ++h) {
      float a2[2], b2[2], c2[2], q2[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = c0 + 2 * h + u;
        const float mu = mean[c], is = invstd[c];
        a2[u] = gamma[c] * is;
        q2[u] = beta[c] - a2[u] * mu;
        c2[u] = -a2[u] * is * dgamma[c] * inv_m;
        b2[u] = -a2[u] * dbeta[c] * inv_m - c2[u] * mu;
      }
      kA[h] = make_float2(a2[0], a2[1]);
      kB[h] = make_float2(b2[0], b2[1]);
      kC[h] = make_float2(c2[0], c2[1]);
      kQ[h] = make_float2(q2[0], q2[1]);
#pragma unroll
      for (int k = 0; k < NACC; ++k) ac[k][h] = make_float2(0.f, 0.f);
    }
  }
  const T* src[NIN];
  src[0] = y;
  src[1] = dz;
  if (MAT) {
    src[2 % NIN] = a;
    src[3 % NIN] = b;
  }
  bn_stream<T, NIN, NST, TB>(g, src, sm, [&](const T* const* in, long long r) {
    float v[V], gv[V], dyv[V];
    SV<T>::lds(in[0], v);
    SV<T>::lds(in[1], gv);
    float2 dy2[V / 2];
#pragma unroll
    for (int h = 0; h < V / 2; ++h) {
      const float2 vv = pr(v, h);
      float2 gg = pr(gv, h);
      if (RELU) {  // g' = g where the forward's kA y + kQ > 0
        const float2 t = __ffma2_rn(kA[h], vv, kQ[h]);
        gg.x = t.x > 0.f ? gg.x : 0.f;
        gg.y = t.y > 0.f ? gg.y : 0.f;
      }
      dy2[h] = __ffma2_rn(kA[h], gg, __ffma2_rn(kC[h], vv, kB[h]));
      dyv[2 * h] = dy2[h].x;
      dyv[2 * h + 1] = dy2[h].y;
    }
    T* drow = D + (size_t)r * Jd + c0;
    if (MAT) {
      float av[V], bv[V];
      SV<T>::lds(in[2 % NIN], av);
      SV<T>::lds(in[3 % NIN], bv);
#pragma unroll
      for (int h = 0; h < V / 2; ++h) {
        const float2 d0 = __fmul2_rn(dy2[h], pr(bv, h)), d1 = __fmul2_rn(dy2[h], pr(av, h));
        ac[0][h] = __fadd2_rn(ac[0][h], d0);
        ac[1 % NACC][h] = __fadd2_rn(ac[1 % NACC][h], d1);
        if (HASG) ac[2 % NACC][h] = __fadd2_rn(ac[2 % NACC][h], dy2[h]);
        bv[2 * h] = d0.x;
        bv[2 * h + 1] = d0.y;
        av[2 * h] = d1.x;
        av[2 * h + 1] = d1.y;
      }
      SV<T>::stg(drow, bv);
      SV<T>::stg(drow + C, av);
      if (HASG) SV<T>::stg(drow + 2 * C, dyv);
    } else {
#pragma unroll
      for (int h = 0; h < V / 2; ++h) ac[0][h] = __fadd2_rn(ac[0][h], dy2[h]);
      SV<T>::stg(drow, dyv);
    }
  });
  float acc[NACC][V];
#pragma unroll
  for (int k = 0; k < NACC; ++k)
#pragma unroll
    for (int h = 0; h < V / 2; ++h) {
      acc[k][2 * h] = ac[k][h].x;
      acc[k][2 * h + 1] = ac[k][h].y;
    }
  if (!db0 && !db1 && !db2) return;
  float* fin = reinterpret_cast<float*>(sm + kHdr + (size_t)NACC * kNT * V * 4);
  if (!bn_grid_fold<NACC, V>(g, acc, part, cnt, sm + kHdr, fin)) return;
  for (int j = threadIdx.x; j < NACC * C; j += blockDim.x) {
    float* dst = j < C ? db0 : (j < 2 * C ? db1 : db2);
    if (dst) dst[j % C] = fin[j];
  }
}

// ---- host side ------------------------------------------------------------------------
template <typename T>
BnGrid bn_grid(long long M, int C, int tile_bytes) {
  BnGrid g;
  g.M = M;
  g.C = C;
  int TR = tile_bytes / (C * (int)sizeof(T));
  if (TR < 1) TR = 1;
  const int sms = tc_num_sms();
  const long long want = (long long)sms * 4;  // >= 4 tiles per CTA when the tensor allows
  long long T0 = (M + TR - 1) / TR;
  if (T0 < want && TR > 1) {
    long long tr = (M + want - 1) / want;
    TR = (int)(tr < 1 ? 1 : tr);
    T0 = (M + TR - 1) / TR;
  }
  g.TR = TR;
  g.T = T0;
  g.S = (int)(T0 < sms ? T0 : sms);
  return g;
}

static size_t stage_bytes(int nin, int nst, int tb) { return kHdr + (size_t)nin * nst * tb; }

// the fold's shared buffer (NACC x 512 x V fp32 partials + the W results) fits
// inside the stage buffer
static_assert(3 * kNT * 8 * 4 + 3 * 2048 * 4 + kThreads * 16 <= 2 * kEmitNst * kEmitTile, "emit fold buffer");
static_assert(3 * kNT * 8 * 4 + 3 * 2048 * 4 + kThreads * 16 <= 4 * kEmitNstMat * kEmitTile, "emit fold buffer");

constexpr int kFoldSlots = 1024;
__device__ unsigned g_fold_cnt[kFoldSlots * kFoldWords];

template <typename T, bool MAT, bool HASG, bool RELU>
static void launch_emit(const BnGrid& g, int Jd, const T* dz, const T* y, const T* a, const T* b, const float* sm,
                        const float* si, const float* gamma, const float* beta, const float* dgamma,
                        const float* dbeta, T* D, float* bpart, unsigned* cnt, float* const db[3], cudaStream_t st) {
  const int smb = (int)stage_bytes(MAT ? 4 : 2, MAT ? kEmitNstMat : kEmitNst, kEmitTile);
  raise_smem_attr((const void*)bns_emit_kernel<T, MAT, HASG, RELU>, smb);
  launch_pdl(bns_emit_kernel<T, MAT, HASG, RELU>, dim3(g.S), dim3(kThreads), smb, st, g, Jd, dz, y, a, b, sm, si, gamma,
             beta, dgamma, dbeta, D, bpart, cnt, db ? db[0] : (float*)nullptr, db ? db[1] : (float*)nullptr,
             db ? db[2] : (float*)nullptr);
}

template <typename T>
static int bns_emit_t(const Plan& P, const T* dz, const T* y, const T* a, const T* b, const float* gamma,
                      const float* beta, const float* sm, const float* si, int relu, T* D, const float* dgamma,
                      const float* dbeta, float* const db[3], float* bpart, cudaStream_t st) {
  const BnGrid g = bn_grid<T>(P.Mout, P.F, kEmitTile);
  const bool want_db = db && db[0] && P.nbias;
  float* const* dbp = want_db ? db : nullptr;
  unsigned* cnt = want_db ? fold_counters() : nullptr;
  const bool mat = caches_ab(P.family), hasg = d_has_g(P.family);
#define QD_EMIT(M_, H_)                                                                                              \
  (relu ? launch_emit<T, M_, H_, true>(g, P.Jd, dz, y, a, b, sm, si, gamma, beta, dgamma, dbeta, D, bpart, cnt, dbp, st) \
        : launch_emit<T, M_, H_, false>(g, P.Jd, dz, y, a, b, sm, si, gamma, beta, dgamma, dbeta, D, bpart, cnt, dbp, st))
  if (mat && hasg)
    QD_EMIT(true, true);
  else if (mat)
    QD_EMIT(true, false);
  else
    QD_EMIT(false, false);
#undef QD_EMIT
  count_launch(st, "bn_emit_D");
  return check_launch("bn emit (stream)");
}

}  // namespace

unsigned* fold_counters() {
  static std::atomic<unsigned> next{0};
  static unsigned* base[kMaxDev] = {};
  const int d = cur_device();
  if (!base[d]) {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_fold_cnt);
    base[d] = static_cast<unsigned*>(p);
  }
  return base[d] + (size_t)(next.fetch_add(1u, std::memory_order_relaxed) % kFoldSlots) * kFoldWords;
}

// Large tensors only: one persistent wave plus the in-kernel fold (~8 us of
// serial GPU-scope steps) lose to the register-streaming emit + bias_finish
// below ~16M elements (measured: 128x128x28x28 even, 256x14 / 512x7 slower;
// 64x56 / 64x112 faster by ~10%).
bool bn_stream_ok(long long M, int C, int dtype) {
  if (getenv("QD_BN_OLD")) return false;  // dev A/B: the register-streaming emit + bias_finish
  const int V = dtype == QD_BF16 ? 8 : 4;
  if (M < 1 || C % V || C > 2048 || kNT % (C / V)) return false;
  return M * (long long)C >= (16ll << 20);
}

// emit partial rows (S <= SMs) + fold group rows
size_t bn_stream_rows() { return 160 + 16; }

int bn_emit_stream(const Plan& P, const void* dz, const void* y, const void* a, const void* b, const float* gamma,
                   const float* beta, const float* sm, const float* si, int relu, void* D, const float* dgamma,
                   const float* dbeta, float* const db[3], float* bpart, cudaStream_t st) {
  if (P.dtype == QD_BF16)
    return bns_emit_t<bf16>(P, (const bf16*)dz, (const bf16*)y, (const bf16*)a, (const bf16*)b, gamma, beta, sm, si,
                            relu, (bf16*)D, dgamma, dbeta, db, bpart, st);
  return bns_emit_t<float>(P, (const float*)dz, (const float*)y, (const float*)a, (const float*)b, gamma, beta, sm, si,
                           relu, (float*)D, dgamma, dbeta, db, bpart, st);
}

}  // namespace qd
