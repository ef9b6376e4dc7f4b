#include <stdlib.h>
// C-ABI entry points of libquadra_b200.so (declared in include/quadra_b200.h).
// Validation mirrors the reference's error conventions; dispatch picks the
// tcgen05 kernels when the shape tiles onto them and the generic CUDA-core
// kernels otherwise. There is no host fallback.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <atomic>
#include <vector>
#include "qd_kernels.h"

namespace qd {

static std::atomic<unsigned long long> g_launches{0};
static thread_local char g_err[512] = "";

// ---- lightweight per-kernel profiling (bench.py roofline): an event after each
// launch of ours, recorded on the launching stream (capturable into graphs) ----
static bool g_prof = false;
static std::vector<cudaEvent_t> g_prof_ev;
static std::vector<const char*> g_prof_name;
static std::vector<cudaStream_t> g_prof_st;
static size_t g_prof_used = 0;

static void prof_mark(cudaStream_t st, const char* name) {
  if (g_prof_used == g_prof_ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    g_prof_ev.push_back(e);
    g_prof_name.push_back(name);
    g_prof_st.push_back(st);
  }
  g_prof_name[g_prof_used] = name;
  g_prof_st[g_prof_used] = st;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)  // becomes an event-record node that fires on replay
    cudaEventRecordWithFlags(g_prof_ev[g_prof_used], st, cudaEventRecordExternal);
  else
    cudaEventRecord(g_prof_ev[g_prof_used], st);
  ++g_prof_used;
}

// dev (timing ablation only; results are wrong): QD_SKIP=pack,fprop,prologue,wgrad,finish,dgrad
bool dev_skip(const char* name) {
  static const char* s = getenv("QD_SKIP");
  if (!s) return false;
  const size_t n = strlen(name);
  for (const char* p = strstr(s, name); p; p = strstr(p + 1, name))
    if ((p == s || p[-1] == ',') && (p[n] == 0 || p[n] == ',')) return true;
  return false;
}

void count_launch(cudaStream_t st, const char* name) {
  g_launches.fetch_add(1ull, std::memory_order_relaxed);
  if (g_prof) prof_mark(st, name);
}

int set_error(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(QD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return QD_OK;
}

static size_t align_up(size_t v, size_t a = 256) { return (v + a - 1) / a * a; }

static int device_path(const Plan& P, unsigned flags) {
  if (P.kind == QD_KIND_DWCONV) return 2;
  if (is_t1(P.family)) return 0;
  if (x3_supported(P, flags)) return 3;
  return tc_supported(P, flags) ? 1 : 0;
}

Workspace plan_workspace(const Plan& P, int path) {
  Workspace L;
  memset(&L, 0, sizeof(L));
  size_t es = P.dtype == QD_BF16 ? 2 : 4;
  if (is_t1(P.family)) return t1_workspace(P);
  if (path == 3) {  // fp32 split operands (hi / lo bf16), raw accumulators, 3 wgrad products
    L.sz_XS = (size_t)2 * P.Min * P.C * 2;
    L.sz_D = (size_t)2 * P.Mout * P.Jd * 2;
    L.sz_P = x3_raw_bytes(P);
    L.wg_split = x3_wgrad_split(P);
    L.sz_WG = (size_t)3 * L.wg_split * P.Jd * P.Kf * 4;
    // one row-lane iteration per thread where the rows allow (256 / (F / 8) rows per block)
    const long long lanes = 256 / (P.F / 8 > 0 ? P.F / 8 : 1);
    long long bs = (P.Mout + lanes - 1) / (lanes > 0 ? lanes : 1);
    if (bs > 2 * 148) bs = 2 * 148;
    L.bs_split = (int)(bs < 1 ? 1 : bs);
    L.sz_BS = (size_t)L.bs_split * P.Jd * 4;
    size_t off = 0;
    L.off_P = off; off = align_up(off + L.sz_P);
    L.off_D = off; off = align_up(off + L.sz_D);
    L.off_WG = off; off = align_up(off + L.sz_WG);
    L.off_BS = off; off = align_up(off + L.sz_BS);
    L.off_XS = off; off = align_up(off + L.sz_XS);
    L.total = off;
    return L;
  }
  if (path == 2) {  // depth-wise: D, bias partials, wgrad partials
    if (caches_ab(P.family) || P.family == QD_FAM_T3) L.sz_D = (size_t)P.Mout * P.Jd * es;
    L.wg_split = dw_wgrad_split(P);
    int nroles = P.nroles;
    L.sz_WG = (size_t)L.wg_split * nroles * P.r * P.r * P.C * 4;
    long long bs = (P.Mout + 255) / 256;
    if (bs > 2 * 148) bs = 2 * 148;
    L.bs_split = (int)(bs < 1 ? 1 : bs);
    L.sz_BS = (size_t)L.bs_split * P.Jd * 4;
    size_t off = 0;
    L.off_D = off; off = align_up(off + L.sz_D);
    L.off_WG = off; off = align_up(off + L.sz_WG);
    L.off_BS = off; off = align_up(off + L.sz_BS);
    L.total = off;
    return L;
  }
  if (path == 0) {
    // SIMT fprop / dgrad outputs, one fp32 slice per K split (small grids: C1's
    // 256 x 1536 fprop would fill 96 CTAs, its 256 x 512 dgrad 32)
    L.sk_f = simt_ksplit(P.Mout, (long long)P.nb * P.F, P.Kf);
    L.sk_d = simt_ksplit(P.Min, P.Cd, P.Kd);
    size_t a = (size_t)L.sk_f * P.Mout * P.nb * P.F, b = (size_t)L.sk_d * P.Min * P.Cd;
    L.sz_P = (a > b ? a : b) * 4;
  }
  // stride-2 layers on the tcgen05 path run their backward on the stride-1 grid
  const Plan Pg = (path == 1 && P.s == 2 && !tc_s2_direct(P)) ? stride1_plan(P) : P;
  if (caches_ab(P.family) || P.family == QD_FAM_T3 || Pg.s != P.s) L.sz_D = (size_t)Pg.Mout * P.Jd * es;
  if (path == 1 && P.family == QD_FAM_T2AND4) L.sz_ZB = (size_t)3 * P.F * 4;
  if (path == 0) {
    long long tiles = (long long)((P.Jd + 127) / 128) * ((P.Kf + 127) / 128);  // SIMT GEMM tiles
    long long S = (2 * 148 + tiles - 1) / tiles;
    long long cap = P.Mout / 64;
    if (cap < 1) cap = 1;
    if (S > cap) S = cap;
    if (S < 1) S = 1;
    L.wg_split = (int)S;
  } else {
    L.wg_split = tc_wgrad_split(Pg);
  }
  L.sz_WG = (size_t)L.wg_split * P.Jd * P.Kf * 4;
  long long bs = (Pg.Mout + 255) / 256;
  if (path == 0) bs = Pg.Mout < 2 * 148 ? Pg.Mout : (bs > 2 * 148 ? bs : 2 * 148);  // row blocks for every SM
  if (path == 1 && P.F % 8 == 0 && P.F <= 2048) {
    // the vectorised prologue covers 4 x (2048 / F) rows per block iteration:
    // wide layers need more blocks for the same rows
    const long long rows_it = 4LL * (2048 / P.F);
    bs = (Pg.Mout + rows_it - 1) / rows_it;
  }
  {
    const char* e = getenv("QD_BS_MULT");
    int mult = e ? atoi(e) : 2;
    if (bs > mult * 148) bs = mult * 148;
  }
  if (bs < 1) bs = 1;
  L.bs_split = (int)bs;
  L.sz_BS = (size_t)L.bs_split * P.Jd * 4;
  if (path == 1 && P.sq) L.sz_XS = (size_t)P.Min * P.C * es;
  if (path == 1 && !(P.flags & QD_FLAG_FORCE_SIMT)) L.sz_SK = tc_splitk_bytes(P);
  size_t off = 0;
  L.off_P = off; off = align_up(off + L.sz_P);
  L.off_D = off; off = align_up(off + L.sz_D);
  L.off_WG = off; off = align_up(off + L.sz_WG);
  L.off_BS = off; off = align_up(off + L.sz_BS);
  L.off_XS = off; off = align_up(off + L.sz_XS);
  L.off_ZB = off; off = align_up(off + L.sz_ZB);
  L.off_SK = off; off = align_up(off + L.sz_SK);
  L.total = off;
  return L;
}

static int validate(const qd_desc* d) {
  if (!d) return set_error(QD_ERR_ARG, "null descriptor");
  if (d->family < 0 || d->family > QD_FAM_T1AND2)
    return set_error(QD_ERR_CONFIG, "unknown family %d", d->family);
  if (d->kind != QD_KIND_FC && d->kind != QD_KIND_CONV && d->kind != QD_KIND_DWCONV)
    return set_error(QD_ERR_CONFIG, "unknown layer kind %d", d->kind);
  if (d->dtype != QD_F32 && d->dtype != QD_BF16)
    return set_error(QD_ERR_CONFIG, "unknown dtype %d", d->dtype);
  if (d->C < 1 || d->F < 1)
    return set_error(QD_ERR_CONFIG, "layer dims must be positive: %d->%d", d->C, d->F);
  if (is_t1(d->family)) {  // neurons.py:58-65
    static const char* names[3] = {"t1_pure", "t1_full", "t1and2"};
    const char* nm = names[d->family - QD_FAM_T1_PURE];
    if (d->kind != QD_KIND_FC)
      return set_error(QD_ERR_CONFIG,
                       "%s carries a full-rank quadratic weight and is restricted to fc layers (got kind=%s)", nm,
                       d->kind == QD_KIND_CONV ? "conv" : "dwconv");
    if (d->F != 1) return set_error(QD_ERR_CONFIG, "%s defines a single output unit; got out=%d", nm, d->F);
  }
  if (d->kind == QD_KIND_DWCONV && d->C != d->F)  // neurons.py:73-75
    return set_error(QD_ERR_CONFIG, "dwconv requires in == out channels, got %d->%d", d->C, d->F);
  if (d->N < 1 || d->H < 1 || d->W < 1)
    return set_error(QD_ERR_DIM, "tensor dimensions must be positive, got (%d, %d, %d, %d)", d->N,
                     d->C, d->H, d->W);
  if (d->kind == QD_KIND_FC) {
    if (d->r != 1 || d->stride != 1 || d->pad != 0)
      return set_error(QD_ERR_CONFIG, "fc layers must use k=1 s=1 p=0");
    if (d->H != 1 || d->W != 1) return set_error(QD_ERR_DIM, "fc input must be (N, C)");
  } else {
    if (d->r < 1 || d->stride < 1 || d->pad < 0)
      return set_error(QD_ERR_CONFIG, "bad conv geometry k=%d s=%d p=%d", d->r, d->stride, d->pad);
    if (d->r > d->H + 2 * d->pad || d->r > d->W + 2 * d->pad)
      return set_error(QD_ERR_DIM, "kernel %d larger than padded input (%d, %d, %d, %d) with pad %d",
                       d->r, d->N, d->C, d->H, d->W, d->pad);
  }
  long long elems = (long long)d->N * d->C * d->H * d->W;
  if (elems >= (1LL << 40)) return set_error(QD_ERR_DIM, "input too large");
  return QD_OK;
}

}  // namespace qd

using namespace qd;

extern "C" {

int qd_validate(const qd_desc* d) { return validate(d); }

int qd_out_shape(const qd_desc* d, int* OH, int* OW) {
  int st = validate(d);
  if (st) return st;
  Plan P = make_plan(*d);
  if (OH) *OH = P.OH;
  if (OW) *OW = P.OW;
  return QD_OK;
}

size_t qd_pack_bytes(const qd_desc* d) {
  if (validate(d)) return 0;
  Plan P = make_plan(*d);
  if (P.kind == QD_KIND_DWCONV) return dw_pack_bytes(P);
  if (is_t1(P.family)) return t1_pack_bytes(P);
  if (device_path(P, d->flags) == 3) return (pack_fprop_elems(P) + pack_dgrad_elems(P)) * 3 * 2;  // [hi|lo|hi] bf16
  size_t es = P.dtype == QD_BF16 ? 2 : 4;
  return (pack_fprop_elems(P) + pack_dgrad_elems(P)) * es;
}

int qd_path(const qd_desc* d) {
  if (validate(d)) return -1;
  Plan P = make_plan(*d);
  return device_path(P, d->flags);
}

size_t qd_workspace_bytes(const qd_desc* d) {
  if (validate(d)) return 0;
  Plan P = make_plan(*d);
  return plan_workspace(P, device_path(P, d->flags)).total;
}

int qd_pack_weights(const qd_desc* d, const float* const w[3], void* wpack, void* stream) {
  int st = validate(d);
  if (st) return st;
  Plan P = make_plan(*d);
  for (int i = 0; i < P.nroles; ++i)
    if (!w || !w[i]) return set_error(QD_ERR_ARG, "weight role %d is NULL", i);
  if (!wpack) return set_error(QD_ERR_ARG, "wpack is NULL");
  if (P.kind == QD_KIND_DWCONV)
    dw_pack(P, w, wpack, (cudaStream_t)stream);
  else if (is_t1(P.family))
    t1_pack(P, w, wpack, (cudaStream_t)stream);
  else if (device_path(P, d->flags) == 3)
    launch_x3_pack(P, w, wpack, (cudaStream_t)stream);
  else
    launch_pack(P, w, wpack, (cudaStream_t)stream);
  return check_launch("pack weights");
}

size_t qd_bn_workspace_bytes(long long M, int C, int Jd) { return bn_workspace_bytes(M, C, Jd); }

int qd_bn_forward(long long M, int C, int dtype, const void* y, const float* gamma, const float* beta,
                  float* run_mean, float* run_var, float momentum, float eps, int relu, int training, void* z,
                  float* save_mean, float* save_invstd, void* ws, void* stream) {
  if (M < 1 || C < 1) return set_error(QD_ERR_DIM, "batchnorm over %lld rows x %d channels", M, C);
  if (dtype != QD_F32 && dtype != QD_BF16) return set_error(QD_ERR_CONFIG, "unknown dtype %d", dtype);
  if (!(eps > 0.f)) return set_error(QD_ERR_CONFIG, "batchnorm eps must be positive");
  if (!y || !gamma || !beta || !z || !save_mean || !save_invstd || (training && !ws))
    return set_error(QD_ERR_ARG, "qd_bn_forward: NULL argument");
  return bn_forward(M, C, dtype, y, gamma, beta, run_mean, run_var, momentum, eps, relu, training, z, save_mean,
                    save_invstd, (char*)ws, (cudaStream_t)stream);
}

int qd_bn_forward_res(long long M, int C, int dtype, const void* y, const void* res, const float* gamma,
                      const float* beta, float* run_mean, float* run_var, float momentum, float eps, int relu,
                      int training, void* z, float* save_mean, float* save_invstd, void* ws, void* stream) {
  if (!res) return set_error(QD_ERR_ARG, "qd_bn_forward_res: NULL residual");
  if (M < 1 || C < 1) return set_error(QD_ERR_DIM, "batchnorm over %lld rows x %d channels", M, C);
  if (dtype != QD_F32 && dtype != QD_BF16) return set_error(QD_ERR_CONFIG, "unknown dtype %d", dtype);
  if (!(eps > 0.f)) return set_error(QD_ERR_CONFIG, "batchnorm eps must be positive");
  if (!y || !gamma || !beta || !z || !save_mean || !save_invstd || (training && !ws))
    return set_error(QD_ERR_ARG, "qd_bn_forward_res: NULL argument");
  return bn_forward(M, C, dtype, y, gamma, beta, run_mean, run_var, momentum, eps, relu, training, z, save_mean,
                    save_invstd, (char*)ws, (cudaStream_t)stream, res);
}

int qd_bn_backward_D(const qd_desc* d, const void* dz, const void* y, const void* a, const void* b,
                     const float* gamma, const float* beta, const float* save_mean, const float* save_invstd,
                     int relu, void* D, float* dgamma, float* dbeta, float* const db[3], void* ws, void* stream) {
  int st = validate(d);
  if (st) return st;
  Plan P = make_plan(*d);
  if (P.family == QD_FAM_T3 || is_t1(P.family))
    return set_error(QD_ERR_UNSUPPORTED, "qd_bn_backward_D: t3 / T1 families recompute their operand");
  if (caches_ab(P.family) && (!a || !b)) return set_error(QD_ERR_INTEGRITY, "cache for this family must hold a and b");
  if (!dz || !y || !gamma || !beta || !save_mean || !save_invstd || !D || !dgamma || !dbeta || !ws)
    return set_error(QD_ERR_ARG, "qd_bn_backward_D: NULL argument");
  return bn_backward_D(P, dz, y, a, b, gamma, beta, save_mean, save_invstd, relu, D, dgamma, dbeta, db, (char*)ws,
                       (cudaStream_t)stream);
}

int qd_maxpool_forward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* x, void* y,
                       void* argmax, void* stream) {
  if (dtype != QD_F32 && dtype != QD_BF16) return set_error(QD_ERR_CONFIG, "unknown dtype %d", dtype);
  if (!x || !y || !argmax) return set_error(QD_ERR_ARG, "qd_maxpool_forward: NULL argument");
  return maxpool_forward(N, C, H, W, k, s, p, dtype, x, y, argmax, (cudaStream_t)stream);
}

int qd_maxpool_backward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* dy,
                        const void* argmax, void* dx, void* stream) {
  if (dtype != QD_F32 && dtype != QD_BF16) return set_error(QD_ERR_CONFIG, "unknown dtype %d", dtype);
  if (!dy || !dx || !argmax) return set_error(QD_ERR_ARG, "qd_maxpool_backward: NULL argument");
  return maxpool_backward(N, C, H, W, k, s, p, dtype, dy, argmax, dx, (cudaStream_t)stream);
}

int qd_im2col(int N, int C, int H, int W, int r, int s, int p, int Kp, int dtype, const void* x, void* col,
              void* stream) {
  if (dtype != QD_F32 && dtype != QD_BF16) return set_error(QD_ERR_CONFIG, "unknown dtype %d", dtype);
  if (!x || !col) return set_error(QD_ERR_ARG, "qd_im2col: NULL argument");
  return im2col(N, C, H, W, r, s, p, Kp, dtype, x, col, (cudaStream_t)stream);
}

int qd_sgd_pack(const qd_desc* d, float* const w[3], float* const mom[3], const float* const grad[3],
                float lr, float momentum, float weight_decay, int first, void* wpack, void* stream) {
  int st = validate(d);
  if (st) return st;
  Plan P = make_plan(*d);
  if (P.kind == QD_KIND_DWCONV || is_t1(P.family))
    return set_error(QD_ERR_UNSUPPORTED, "qd_sgd_pack: fc / conv kinds of the non-T1 families only");
  if (device_path(P, d->flags) == 3)
    return set_error(QD_ERR_UNSUPPORTED, "qd_sgd_pack: fp32 layers on the split tensor-core path pack themselves");
  if (!w || !mom || !grad || !wpack) return set_error(QD_ERR_ARG, "qd_sgd_pack: NULL argument");
  for (int i = 0; i < P.nroles; ++i)
    if (!w[i] || !mom[i] || !grad[i]) return set_error(QD_ERR_ARG, "qd_sgd_pack: role %d has a NULL pointer", i);
  launch_sgd_pack(P, w, mom, grad, lr, momentum, weight_decay, first, wpack, (cudaStream_t)stream);
  return check_launch("sgd pack");
}

int qd_forward(const qd_desc* d, const void* x, const void* wpack, const float* const bias[3],
               void* y, void* a_cache, void* b_cache, void* workspace, void* stream) {
  int st = validate(d);
  if (st) return st;
  Plan P = make_plan(*d);
  if (!x || !wpack || !y) return set_error(QD_ERR_ARG, "null tensor pointer");
  for (int i = 0; i < P.nbias; ++i)
    if (!bias || !bias[i]) return set_error(QD_ERR_ARG, "bias role %d is NULL", i);
  bool cache = caches_ab(P.family);
  if (cache && (!a_cache || !b_cache))
    return set_error(QD_ERR_ARG, "family caches a and b: a_cache/b_cache must be given");
  const float* nob[3] = {nullptr, nullptr, nullptr};
  const float* const* bs = bias ? bias : nob;
  int path = device_path(P, d->flags);
  Workspace L = plan_workspace(P, path);
  if (L.total && !workspace) return set_error(QD_ERR_ARG, "workspace is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  if (is_t1(P.family)) return t1_forward(P, x, wpack, y, (char*)workspace, L, s);
  if (path == 2) return dw_forward(P, x, wpack, bs, y, a_cache, b_cache, (char*)workspace, L, s);
  if (path == 1) return tc_forward(P, x, wpack, bs, y, a_cache, b_cache, (char*)workspace, L, s);
  if (path == 3) return x3_forward(P, x, wpack, bs, y, a_cache, b_cache, (char*)workspace, L, s);
  return simt_forward(P, x, wpack, bs, y, a_cache, b_cache, (char*)workspace, L, s);
}

int qd_bn_stats_rows(const qd_desc* d) {
  if (validate(d)) return 0;
  Plan P = make_plan(*d);
  const int path = device_path(P, d->flags);
  return (path == 1 || path == 3) ? tc_stat_rows(P, path) : 0;
}

int qd_forward_bnstats(const qd_desc* d, const void* x, const void* wpack, const float* const bias[3], void* y,
                       void* a_cache, void* b_cache, void* workspace, float* stats, void* stream) {
  int st = validate(d);
  if (st) return st;
  Plan P = make_plan(*d);
  if (!x || !wpack || !y || !stats) return set_error(QD_ERR_ARG, "null tensor pointer");
  for (int i = 0; i < P.nbias; ++i)
    if (!bias || !bias[i]) return set_error(QD_ERR_ARG, "bias role %d is NULL", i);
  if (caches_ab(P.family) && (!a_cache || !b_cache))
    return set_error(QD_ERR_ARG, "family caches a and b: a_cache/b_cache must be given");
  const int path = device_path(P, d->flags);
  if (!((path == 1 || path == 3) && tc_stat_rows(P, path) > 0))
    return set_error(QD_ERR_UNSUPPORTED, "qd_forward_bnstats: no epilogue statistics on this layer's path");
  Workspace L = plan_workspace(P, path);
  if (L.total && !workspace) return set_error(QD_ERR_ARG, "workspace is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  if (path == 3) return x3_forward(P, x, wpack, bias, y, a_cache, b_cache, (char*)workspace, L, s, stats);
  return tc_forward(P, x, wpack, bias, y, a_cache, b_cache, (char*)workspace, L, s, stats);
}

int qd_bn_forward_stats(long long M, int C, int dtype, const void* y, const void* res, const float* stats, int rows,
                        const float* gamma, const float* beta, float* run_mean, float* run_var, float momentum,
                        float eps, int relu, int training, void* z, float* save_mean, float* save_invstd,
                        void* stream) {
  if (M < 1 || C < 1 || rows < 1) return set_error(QD_ERR_DIM, "batchnorm over %lld rows x %d channels", M, C);
  if (dtype != QD_F32 && dtype != QD_BF16) return set_error(QD_ERR_CONFIG, "unknown dtype %d", dtype);
  if (!(eps > 0.f)) return set_error(QD_ERR_CONFIG, "batchnorm eps must be positive");
  if (!y || !stats || !gamma || !beta || !z || !save_mean || !save_invstd)
    return set_error(QD_ERR_ARG, "qd_bn_forward_stats: NULL argument");
  return bn_forward_stats(M, C, dtype, y, res, stats, rows, gamma, beta, run_mean, run_var, momentum, eps, relu,
                          training, z, save_mean, save_invstd, (cudaStream_t)stream);
}

int qd_backward(const qd_desc* d, const void* x, const void* wpack, const void* a_cache,
                const void* b_cache, const void* dy, void* dx, float* const dW[3],
                float* const db[3], void* workspace, void* stream) {
  int st = validate(d);
  if (st) return st;
  Plan P = make_plan(*d);
  if (!x || !wpack || !dy) return set_error(QD_ERR_ARG, "null tensor pointer");
  const bool dgiven = (d->flags & QD_FLAG_D_GIVEN) != 0;
  bool cache = caches_ab(P.family) && !dgiven;
  if (cache && (!a_cache || !b_cache))
    return set_error(QD_ERR_INTEGRITY, "cache for this family must hold a and b");
  // stride 2 only on its own output grid (the D the caller emits is on that grid)
  const bool s2ok = P.s == 2 && tc_supported(P, d->flags) && tc_s2_direct(P);
  if (dgiven && ((P.s != 1 && !s2ok) || P.family == QD_FAM_T3 || is_t1(P.family) || P.kind == QD_KIND_DWCONV))
    return set_error(QD_ERR_UNSUPPORTED,
                     "QD_FLAG_D_GIVEN: stride-1 fc / conv layers or direct stride-2 convs, not t3 / T1");
  if (!(d->flags & QD_FLAG_NO_DX) && !dx) return set_error(QD_ERR_ARG, "dx is NULL");
  float* nof[3] = {nullptr, nullptr, nullptr};
  float* const* w = (dW && !(d->flags & QD_FLAG_NO_DW)) ? dW : nof;
  float* const* b = (db && !(d->flags & QD_FLAG_NO_DW) && !dgiven) ? db : nof;
  int path = device_path(P, d->flags);
  Workspace L = plan_workspace(P, path);
  if (L.total && !workspace) return set_error(QD_ERR_ARG, "workspace is NULL");
  void* dxp = (d->flags & QD_FLAG_NO_DX) ? nullptr : dx;
  cudaStream_t s = (cudaStream_t)stream;
  if (is_t1(P.family)) return t1_backward(P, x, wpack, dy, dxp, w, (char*)workspace, L, s);
  if (path == 2) return dw_backward(P, x, wpack, a_cache, b_cache, dy, dxp, w, b, (char*)workspace, L, s);
  if (path == 1) return tc_backward(P, x, wpack, a_cache, b_cache, dy, dxp, w, b, (char*)workspace, L, s);
  if (path == 3) return x3_backward(P, x, wpack, a_cache, b_cache, dy, dxp, w, b, (char*)workspace, L, s);
  return simt_backward(P, x, wpack, a_cache, b_cache, dy, dxp, w, b, (char*)workspace, L, s);
}

const char* qd_error_string(int status) {
  switch (status) {
    case QD_OK: return "ok";
    case QD_ERR_CONFIG: return "ConfigError";
    case QD_ERR_DIM: return "DimensionError";
    case QD_ERR_INTEGRITY: return "IntegrityError";
    case QD_ERR_CUDA: return "CUDA error";
    case QD_ERR_UNSUPPORTED: return "unsupported on this device path";
    case QD_ERR_ARG: return "invalid argument";
  }
  return "unknown status";
}

const char* qd_last_error(void) { return g_err; }

unsigned long long qd_launch_count(void) { return g_launches.load(); }

int qd_profile(int enable) {
  g_prof = enable != 0;
  if (g_prof) g_prof_used = 0;
  return QD_OK;
}

int qd_profile_mark(void* stream) {
  if (g_prof) prof_mark((cudaStream_t)stream, "begin");
  return QD_OK;
}

int qd_profile_count(void) { return (int)g_prof_used; }

int qd_profile_read(int i, const char** name, float* ms) {
  if (i <= 0 || (size_t)i >= g_prof_used) return QD_ERR_ARG;
  if (name) *name = g_prof_name[i];
  // interval from the latest earlier mark on the same stream (a kernel on a
  // forked side stream: from the latest earlier mark, the fork point)
  size_t j = (size_t)i - 1;
  for (size_t k = (size_t)i - 1; k >= 1; --k)
    if (g_prof_st[k] == g_prof_st[i]) { j = k; break; }
  float t = 0.f;
  cudaError_t e = cudaEventElapsedTime(&t, g_prof_ev[j], g_prof_ev[i]);
  if (e != cudaSuccess) return set_error(QD_ERR_CUDA, "qd_profile_read: %s", cudaGetErrorString(e));
  if (ms) *ms = t;
  return QD_OK;
}

const char* qd_version(void) { return "quadra_b200 0.1.0 (sm_100a)"; }

}  // extern "C"
