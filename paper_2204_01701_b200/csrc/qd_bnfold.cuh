// Deterministic in-kernel grid fold of per-CTA partial rows (the BN reductions):
// every CTA writes its partial row part[s][0..W); the last CTA to arrive in each
// group of ~sqrt(S) CTAs folds that group's rows in order into part[S + g]; the
// last group folder folds the G group rows in order. The result does not depend
// on which CTA arrives when (fixed grouping, fixed order), and no finalize
// launch follows the reduction.
#pragma once
#include "qd_kernels.h"

namespace qd {

struct FoldGeom {
  int S;   // CTAs (partial rows)
  int GS;  // CTAs per group
  int G;   // groups (<= kFoldWords - 1)
};
constexpr int kFoldWords = 32;  // arrival counters per fold: [0] groups, [1 + g] group g

__host__ __device__ inline FoldGeom fold_geom(int S) {
  int gs = 1;
  while (gs * gs < S) ++gs;
  FoldGeom f;
  f.S = S;
  f.GS = gs;
  f.G = (S + gs - 1) / gs;
  return f;
}

// arrival index among n arrivals; the last arrival re-arms the count to 0 (the
// counters are zero at rest: device globals, zero at load, see fold_counters)
__device__ __forceinline__ unsigned fold_arrive(unsigned* cnt, unsigned n) {
  const unsigned c = atomicAdd(cnt, 1u);
  if (c == n - 1) atomicExch(cnt, 0u);
  return c;
}

// out[0..W) = column sums of rows [b0, b1) of p[rows][W] (W % 4 == 0), float4
// columns. Narrow rows (W / 4 < blockDim): tpc threads per column group each sum
// a contiguous run of rows (in order), combined in thread order through scratch
// (blockDim float4, shared) -- fixed order, so deterministic; few L2 round trips.
__device__ __forceinline__ void fold_rows(const float* p, int W, int b0, int b1, float* out, float4* scratch) {
  const int W4 = W / 4, nb = (int)blockDim.x;
  const float4* p4 = reinterpret_cast<const float4*>(p);
  float4* o4 = reinterpret_cast<float4*>(out);
  if (W4 >= nb) {
    for (int q = threadIdx.x; q < W4; q += nb) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      int b = b0;
      for (; b + 8 <= b1; b += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p4 + (size_t)(b + u) * W4 + q);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
      }
      for (; b < b1; ++b) {
        const float4 v = __ldcg(p4 + (size_t)b * W4 + q);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      o4[q] = acc;
    }
    return;
  }
  const int tpc = nb / W4, q = threadIdx.x % W4, k = threadIdx.x / W4;
  const int chunk = (b1 - b0 + tpc - 1) / tpc;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k < tpc) {
    const int r0 = b0 + k * chunk, r1 = min(b1, r0 + chunk);
    int b = r0;
    for (; b + 4 <= r1; b += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(p4 + (size_t)(b + u) * W4 + q);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
      }
    }
    for (; b < r1; ++b) {
      const float4 v = __ldcg(p4 + (size_t)b * W4 + q);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  scratch[threadIdx.x] = acc;
  __syncthreads();
  if (k == 0) {
    float4 t = scratch[q];
    for (int j = 1; j < tpc; ++j) {
      const float4 v = scratch[j * W4 + q];
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    o4[q] = t;
  }
  __syncthreads();
}

// Call with every thread of the CTA once its partial row is stored. Returns true
// in the single CTA that then holds the totals in fin[0..W) (shared memory,
// 16-byte aligned; written only after the CTA's own reads of any buffer fin
// overlays are done). scratch: blockDim float4 of shared memory apart from fin.
__device__ __forceinline__ bool grid_fold(float* part, int W, const FoldGeom f, unsigned* cnt, float* fin,
                                          float4* scratch) {
  __shared__ int last;
  const int s = blockIdx.x, grp = s / f.GS, b0 = grp * f.GS, b1 = min(f.S, b0 + f.GS);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = fold_arrive(&cnt[1 + grp], (unsigned)(b1 - b0)) == (unsigned)(b1 - b0 - 1);
  __syncthreads();
  if (!last) return false;
  __threadfence();
  float* gpart = part + (size_t)f.S * W;
  fold_rows(part, W, b0, b1, gpart + (size_t)grp * W, scratch);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = fold_arrive(&cnt[0], (unsigned)f.G) == (unsigned)(f.G - 1);
  __syncthreads();
  if (!last) return false;
  __threadfence();
  fold_rows(gpart, W, 0, f.G, fin, scratch);
  __syncthreads();
  return true;
}

// kFoldWords zeroed counters for one fold launch (qd_bnstream.cu): a ring of
// slots in a device global; a slot is re-armed by the fold that used it
unsigned* fold_counters();

}  // namespace qd
