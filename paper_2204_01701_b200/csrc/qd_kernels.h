#include <stdlib.h>
// Host launchers shared between the translation units of libquadra_b200.so.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <string.h>
#include <mutex>
#include <utility>
#include "qd_common.cuh"

namespace qd {

// ---- per-(thread, device) host state ------------------------------------------
// The side stream / fork-join events of the concurrent backward are per host
// thread: those caches are thread_local arrays indexed by the current device.
// Kernel attributes are per (function, device) for the whole process: see
// raise_smem_attr.
constexpr int kMaxDev = 16;
inline int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  return d < 0 ? 0 : (d >= kMaxDev ? kMaxDev - 1 : d);
}

// Raise a kernel's opt-in dynamic shared memory on the current device to at
// least `bytes`; never lowers it. The attribute is process-wide, so the record
// of what was set is too (one mutex): a per-thread "largest so far" let the
// autograd thread set a smaller value under a launch of the main thread's larger
// plan (conv2 launch: invalid argument).
inline cudaError_t raise_smem_attr(const void* fn, size_t bytes) {
  struct Rec {
    const void* fn;
    int dev;
    size_t bytes;
  };
  static std::mutex mu;
  static Rec recs[512];
  static int n = 0;
  if (bytes <= 48 * 1024) return cudaSuccess;
  const int d = cur_device();
  std::lock_guard<std::mutex> lock(mu);
  int i = 0;
  for (; i < n; ++i)
    if (recs[i].fn == fn && recs[i].dev == d) break;
  if (i < n && recs[i].bytes >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return e;
  if (i < n)
    recs[i].bytes = bytes;
  else if (n < 512)
    recs[n++] = Rec{fn, d, bytes};
  return cudaSuccess;
}

// ---- bookkeeping -----------------------------------------------------------
// counts a launch of ours on `st`; with profiling on, also records a timing event
void count_launch(cudaStream_t st, const char* name);
int set_error(int status, const char* fmt, ...);
int check_launch(const char* what);

// ---- workspace layout ------------------------------------------------------
struct Workspace {
  size_t total;
  size_t off_P, sz_P;      // SIMT fprop / dgrad fp32 GEMM output
  size_t off_D, sz_D;      // backward operand D (dtype), proposed/t4
  size_t off_WG, sz_WG;    // wgrad split-K partials (fp32)
  size_t off_BS, sz_BS;    // bias-sum partials (fp32)
  size_t off_XS, sz_XS;    // squared input (dtype), t2/t2_linear tcgen05 path
  size_t off_ZB, sz_ZB;    // zero bias vectors (t2and4 reuses the proposed epilogue)
  size_t off_SK, sz_SK;    // split-K fp32 partials of the v1 fprop / dgrad (small output grids)
  int wg_split;            // number of wgrad partials
  int bs_split;            // number of bias-sum partials
  int sk_f, sk_d;          // SIMT fprop / dgrad K slices (slices of P, summed by the epilogues)
};
// SIMT GEMM K slices: enough CTAs for two per SM, each slice >= 64 of K
inline int simt_ksplit(long long M, long long N, long long K) {
  const long long tiles = ((M + 127) / 128) * ((N + 127) / 128);  // SG_BM x SG_BN tiles
  long long S = (2 * 148 + tiles - 1) / tiles;
  if (S > K / 64) S = K / 64;
  return S < 1 ? 1 : (int)S;
}
Workspace plan_workspace(const Plan& P, int path);
size_t tc_splitk_bytes(const Plan& P);

// ---- packing (both paths) --------------------------------------------------
size_t pack_fprop_elems(const Plan& P);
size_t pack_dgrad_elems(const Plan& P);
void launch_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st);

// ---- generic CUDA-core path ------------------------------------------------
int simt_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3],
                 void* y, void* a, void* b, char* ws, const Workspace& L, cudaStream_t st);
int simt_backward(const Plan& P, const void* x, const void* wpack, const void* a, const void* b,
                  const void* dy, void* dx, float* const dW[3], float* const db[3], char* ws,
                  const Workspace& L, cudaStream_t st);

// ---- shared backward pieces (elementwise / reductions) ---------------------
// D = [dy*b | dy*a | dy] (proposed) or [dy*b | dy*a] (t4), plus column-sum
// partials of D (or of dy) for the bias gradients.
void launch_bwd_prologue(const Plan& P, const void* dy, const void* a, const void* b,
                         void* D, float* bsum_part, int bs_split, cudaStream_t st);
// t3: D = 2 dy a from the recomputed a (fp32 SIMT GEMM output or dtype, may alias D)
void launch_t3_prologue(const Plan& P, const void* dy, const void* a, bool a_fp32, void* D, cudaStream_t st);
void launch_bwd_prologue_vec(const Plan& P, const void* dy, const void* a, const void* b, void* D, float* part,
                             int split, cudaStream_t st);  // bf16, F % 8 == 0
void launch_bias_finish(const Plan& P, const float* bsum_part, int bs_split,
                        float* const db[3], cudaStream_t st);
// sum the wgrad partials [S][Jd][Kf] and scatter into reference layouts
void launch_wgrad_finish(const Plan& P, const float* part, int S, float* const dW[3],
                         cudaStream_t st);
// split-K partial counts of the wgrad rows: rows of tap pair p (tap / 2) have
// s[p / pp] partials (ng == 0: every row has the uniform count)
struct WSplits {
  int pp, ng;
  int s[16];
};
WSplits wgrad2_splits(const Plan& P);
// tcgen05 path: wgrad partial fold + bias partial fold in one launch (Kf % 4 == 0)
void launch_bwd_finish(const Plan& P, const float* wpart, int S, const WSplits& ws, float* const dW[3],
                       const float* bpart, int SB, float* const db[3], cudaStream_t st);
void launch_square(const Plan& P, const void* x, void* xs, cudaStream_t st);
void launch_square_out(const Plan& P, void* y, cudaStream_t st);  // y <- y*y in place (t3)

// Launch with programmatic stream serialization (PDL): the kernel may start while
// the previous kernel of the stream drains; it must call ptx::pdl_wait() before
// touching that kernel's outputs. QD_NO_PDL=1 falls back to ordinary launches.
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("QD_NO_PDL");
    on = (e && atoi(e)) ? 0 : 1;
  }
  return on == 1;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  if (!pdl_enabled()) {
    kernel<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// PDL launch with the cooperative attribute (coop = 1): the driver launches the
// grid only when every CTA can be resident at once (software grid barriers)
template <typename... KArgs, typename... Args>
inline cudaError_t cudaLaunchCoop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                  bool coop, Args&&... args) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (coop) {
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

void launch_sgd_pack(const Plan& P, float* const w[3], float* const mom[3], const float* const grad[3], float lr,
                     float momentum, float wd, int first, void* wpack, cudaStream_t st);

// ---- BN (+ReLU) around the quadratic conv (qd_bn.cu) ------------------------
size_t bn_workspace_bytes(long long M, int C, int Jd);
// the streaming D emission of the BN backward (qd_bnstream.cu): persistent CTAs,
// bulk-copy staged tiles, bias gradients folded in-kernel
bool bn_stream_ok(long long M, int C, int dtype);
size_t bn_stream_rows();
int bn_emit_stream(const Plan& P, const void* dz, const void* y, const void* a, const void* b, const float* gamma,
                   const float* beta, const float* sm, const float* si, int relu, void* D, const float* dgamma,
                   const float* dbeta, float* const db[3], float* bpart, cudaStream_t st);
int tc_num_sms();
int bn_forward(long long M, int C, int dtype, const void* y, const float* gamma, const float* beta, float* rm,
               float* rv, float momentum, float eps, int relu, int training, void* z, float* sm, float* si, char* ws,
               cudaStream_t st, const void* res = nullptr);
// BN forward from the statistics rows of the fprop epilogue (mean / M2 / count per
// row, merged with Chan's formula in a fixed order), then the apply pass
int bn_forward_stats(long long M, int C, int dtype, const void* y, const void* res, const float* stats, int rows,
                     const float* gamma, const float* beta, float* rm, float* rv, float momentum, float eps, int relu,
                     int training, void* z, float* sm, float* si, cudaStream_t st);
int bn_backward_D(const Plan& P, const void* dz, const void* y, const void* a, const void* b, const float* gamma,
                  const float* beta, const float* sm, const float* si, int relu, void* D, float* dgamma,
                  float* dbeta, float* const db[3], char* ws, cudaStream_t st);

// ---- T1 families (qd_t1.cu): fc, one output, CUDA-core path ----------------
bool is_t1(int family);
size_t t1_pack_bytes(const Plan& P);
void t1_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st);
Workspace t1_workspace(const Plan& P);
int t1_forward(const Plan& P, const void* x, const void* wpack, void* y, char* ws, const Workspace& L,
               cudaStream_t st);
int t1_backward(const Plan& P, const void* x, const void* wpack, const void* dy, void* dx, float* const dW[3],
                char* ws, const Workspace& L, cudaStream_t st);

// ---- depth-wise path (qd_dw.cu): qd_path() == 2 ------------------------------
size_t dw_pack_bytes(const Plan& P);
void dw_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st);
int dw_wgrad_split(const Plan& P);
int dw_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3], void* y, void* a,
               void* b, char* ws, const Workspace& L, cudaStream_t st);
int dw_backward(const Plan& P, const void* x, const void* wpack, const void* a, const void* b, const void* dy,
                void* dx, float* const dW[3], float* const db[3], char* ws, const Workspace& L, cudaStream_t st);

// ---- fp32 on the tensor cores (path 3, qd_x3.cu + qd_tc.cu) -----------------
bool x3_supported(const Plan& P, unsigned flags);
size_t x3_raw_bytes(const Plan& P);
int x3_wgrad_split(const Plan& P);
void launch_x3_split(const float* x, bf16* hi, bf16* lo, long long n, cudaStream_t st);
void launch_x3_pack(const Plan& P, const float* const w[3], void* wpack, cudaStream_t st);
void launch_x3_prologue(const Plan& P, const float* dy, const float* a, const float* b, bf16* Dh, bf16* Dl,
                        float* part, int split, cudaStream_t st);
void launch_x3_fprop_finish(const float* raw, int S, long long M, int ld, int F, int nb, int epi, float* y, float* a,
                            float* b, const float* const bias[3], cudaStream_t st);
void launch_x3_sum(const float* raw, int S, long long n, float* out, cudaStream_t st);
int x3_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3], void* y, void* a,
               void* b, char* ws, const Workspace& L, cudaStream_t st, float* stats = nullptr);
int tc_stat_rows(const Plan& P, int path);
int x3_backward(const Plan& P, const void* x, const void* wpack, const void* a, const void* b, const void* dy,
                void* dx, float* const dW[3], float* const db[3], char* ws, const Workspace& L, cudaStream_t st);

// ---- tcgen05 path ----------------------------------------------------------
bool tc_supported(const Plan& P, unsigned flags);
int tc_wgrad_split(const Plan& P);
// v2 wgrad with halo reuse (qd_tc2.cu); wgrad2_split() == 0 when not eligible
int wgrad2_split(const Plan& P);
// Dtail / jsplit: D channel blocks >= jsplit are read from Dtail (the dy tensor) instead of D
int run_wgrad2(const Plan& P, const void* x0, const void* x1, const void* D, float* part, int splits,
               cudaStream_t st, const void* Dtail = nullptr, int jsplit = 0);
// v3 wgrad (r = 3) on CTA pairs with multicast stage loads; 0 when not eligible
void set_conv2_cap(int pairs);
bool dev_skip(const char* name);
int maxpool_forward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* x, void* y, void* arg,
                    cudaStream_t st);
int maxpool_backward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* dy, const void* arg,
                     void* dx, cudaStream_t st);
int im2col(int N, int C, int H, int W, int r, int s, int p, int Kp, int dtype, const void* x, void* col,
           cudaStream_t st);
int wgrad3_pairs_per_split(const Plan& P);
int wgrad3_split(const Plan& P);
int run_wgrad3(const Plan& P, const void* x0, const void* x1, const void* D, float* part, int splits,
               cudaStream_t st, const void* Dtail = nullptr, int jsplit = 0, float* const* dW = nullptr,
               const float* bpart = nullptr, int SB = 0, float* const* db = nullptr, bool* folded = nullptr);
// operand transform of the conv2 A operand (C2Args::xf): mode 1 = x * x for the
// first K half (x = the layer input), 2 = the dgrad's D blocks dy * b, dy * a
// (x = dy; cs = channels of dy / a / b, fb = F / 64)
struct C2Xform {
  int mode, cs, fb;
  const void* x;
  const void* a;
  const void* b;
};
// v2 stride-1 conv on CTA pairs (qd_tc2.cu); QD_ERR_UNSUPPORTED if the shape does not fit
int run_conv2(int epi, int nbk, const void* a0, const void* a1, int Cin, int Win, int Hin, int N, int OWg, int OHg,
              int pe, int r, int dual, const void* wmat, int wrows, int wK, int b_rs_tile, int b_rs_blk,
              int tiles_nn, int out_c_tile, void* o0, void* o1, void* o2, int Cout, const float* const bias[3],
              const void* xres, cudaStream_t st, int ss = 1, const void* a_tail = nullptr, int csplit = 0,
              int pdl_wait = 1, int f32out = 0, float* stats = nullptr, const C2Xform* xf = nullptr);
int conv2_stat_rows(int N, int Cin, int Win, int Hin, int OWg, int OHg, int pe, int r, int dual, int nbk, int nout,
                    int tiles_nn, int Cout, int nbias);
bool conv2_fits(int N, int Cin, int Win, int Hin, int OWg, int OHg, int pe, int r, int dual, int nbk, int nout,
                int tiles_nn, int Cout, int nbias);
// stride 2 on its own output grid (strided x maps, parity-class dgrad)
bool tc_s2_direct(const Plan& P);
// otherwise stride-2 layers run as their stride-1 equivalent: forward subsamples the
// output, backward uses the zero-upsampled gradient operand
inline Plan stride1_plan(const Plan& P) {
  Plan Q = P;
  Q.s = 1;
  Q.OH = P.H + 2 * P.p - P.r + 1;
  Q.OW = P.W + 2 * P.p - P.r + 1;
  Q.Mout = (long long)P.N * Q.OH * Q.OW;
  return Q;
}
int tc_forward(const Plan& P, const void* x, const void* wpack, const float* const bias[3],
               void* y, void* a, void* b, char* ws, const Workspace& L, cudaStream_t st, float* stats = nullptr);
// dW[0] == nullptr skips the weight/bias gradient GEMM (QD_FLAG_NO_DW)
int tc_backward(const Plan& P, const void* x, const void* wpack, const void* a, const void* b,
                const void* dy, void* dx, float* const dW[3], float* const db[3], char* ws,
                const Workspace& L, cudaStream_t st);

}  // namespace qd
