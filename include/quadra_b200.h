/*
 * quadra_b200.h -- C ABI of the B200-native quadratic-layer hot path.
 *
 * The reference (QuadraLib, /root/reference/pkg/src/quadra) is a pure-Python
 * numpy library with no FFI; its hot-path interface is the Python pair
 *
 *   neurons.forward(spec, params, x) -> (y, LayerCache(x, a, b))
 *       /root/reference/pkg/src/quadra/neurons.py:235-276
 *   neurons.symbolic_backward(spec, params, cache, dy) -> ({role: dW}, dx)
 *       /root/reference/pkg/src/quadra/neurons.py:295-445
 *
 * plus the integer helpers validate_spec / param_shapes / conv_out_size
 * (neurons.py:50-107, tensor.py:279-280). Each entry point below replaces one
 * of those (cited per function); the Python package
 * paper_2204_01701_b200.neurons binds them with ctypes and keeps the
 * reference's Python signatures.
 *
 * Conventions: every tensor pointer is DEVICE memory, caller-allocated;
 * every call is stream-ordered on `stream` with no host synchronisation and
 * no allocation inside. Activations are NHWC (channels_last; fc = (N, C)) in
 * the descriptor's dtype; weights and weight/bias gradients are fp32 in the
 * reference layouts (conv (F, C, r, r); fc (in, out) = (C, F)).
 */
#ifndef QUADRA_B200_H
#define QUADRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* family tags: reference neurons.py:40-41 (+ t2_linear) */
enum {
  QD_FAM_FIRST_ORDER = 0, /* W x + b                                  */
  QD_FAM_T2 = 1,          /* Wa (x*x)                                 */
  QD_FAM_T4 = 2,          /* (Wa x) * (Wb x)                          */
  QD_FAM_PROPOSED = 3,    /* (Wa x + ba) * (Wb x + bb) + (Wc x + bc)  */
  QD_FAM_T2_LINEAR = 4,   /* Wa (x*x) + Wc x                          */
  QD_FAM_T3 = 5,          /* (Wa x)^2                                 */
  QD_FAM_T2AND4 = 6,      /* (Wa x) * (Wb x) + Wc (x*x)               */
  QD_FAM_T1_PURE = 7,     /* x^T Wq x              (fc, one output)   */
  QD_FAM_T1_FULL = 8,     /* x^T Wq x + x Wb       (fc, one output)   */
  QD_FAM_T1AND2 = 9       /* x^T Wq x + (x*x) Wb   (fc, one output)   */
};
enum { QD_KIND_FC = 0, QD_KIND_CONV = 1, QD_KIND_DWCONV = 2 /* depth-wise, C == F */ };
enum { QD_F32 = 0, QD_BF16 = 1 };

/* status codes; the Python layer re-raises the reference exception classes
 * (errors.py:8-38): CONFIG->ConfigError, DIM->DimensionError,
 * INTEGRITY->IntegrityError, CUDA/UNSUPPORTED/ARG->DeviceError */
enum {
  QD_OK = 0,
  QD_ERR_CONFIG = 1,
  QD_ERR_DIM = 2,
  QD_ERR_INTEGRITY = 3,
  QD_ERR_CUDA = 4,
  QD_ERR_UNSUPPORTED = 5,
  QD_ERR_ARG = 6
};

/* flags */
#define QD_FLAG_NO_DX 1u      /* backward: skip the input gradient        */
#define QD_FLAG_FORCE_SIMT 2u /* use the generic CUDA-core kernels even    \
                                 where a tcgen05 kernel exists (tests)     */
#define QD_FLAG_NO_DW 4u      /* backward: skip weight and bias gradients  \
                                 (frozen layers; per-kernel timing)        */
#define QD_FLAG_TC_V1 8u      /* tcgen05 path without the CTA-pair / halo \
                                 conv kernel (tests compare the two)       */
#define QD_FLAG_D_GIVEN 16u   /* backward: `dy` already is the operand D   \
                                 (qd_bn_backward_D); bias grads not formed */

typedef struct {
  int family, kind, dtype;
  int N, C, H, W; /* input  (fc: H = W = 1)                            */
  int F;          /* output channels / features                        */
  int r, stride, pad;
  unsigned flags;
} qd_desc;

/* Replaces validate_spec + _check_x + _check_conv_pre
 * (neurons.py:50-77, :212-220; tensor.py:334-352) for the device path. */
int qd_validate(const qd_desc* d);

/* conv_out_size semantics, tensor.py:279-280. */
int qd_out_shape(const qd_desc* d, int* OH, int* OW);

/* Bytes of the packed-weight buffer and of the scratch workspace one layer
 * needs (forward and backward share it). */
size_t qd_pack_bytes(const qd_desc* d);
size_t qd_workspace_bytes(const qd_desc* d);

/* Cast + re-layout the fp32 reference-layout weights of the branches into
 * the kernels' packed layouts (fprop [Wa;Wb;Wc] K-major, dgrad flipped).
 * w[i] are the family's weight roles in order: proposed (Wa, Wb, Wc),
 * t4 (Wa, Wb), t2 (Wa), first_order (W), t2_linear (Wa, Wc). Unused = NULL.
 * Replaces the implicit W.reshape(f,-1) of tensor.py:317, :329. */
int qd_pack_weights(const qd_desc* d, const float* const w[3], void* wpack,
                    void* stream);

/* Batch norm (+ ReLU) around the quadratic conv,
 * reference semantics tensor.py:423-470 / :552-570 (biased batch variance, also
 * in the running update). NHWC tensors of M = N*OH*OW rows and C channels.
 * Forward: z = relu?(gamma (y - mean) inv_std + beta); training computes the
 * batch statistics (save_mean / save_invstd out) and folds them into
 * run_mean / run_var; eval uses save_mean / save_invstd as given.
 * Workspace: qd_bn_workspace_bytes of caller memory, any content, one call at a
 * time. Reductions are deterministic (fixed-order partial rows); the streaming
 * D emission of large tensors folds its bias sums in-kernel with arrival
 * counters from a library-owned device ring (1024 slots, re-armed by each use). */
size_t qd_bn_workspace_bytes(long long M, int C, int Jd);
int qd_bn_forward(long long M, int C, int dtype, const void* y, const float* gamma, const float* beta,
                  float* run_mean, float* run_var, float momentum, float eps, int relu, int training,
                  void* z, float* save_mean, float* save_invstd, void* ws, void* stream);
/* Same with a residual added before the ReLU (a ResNet block tail):
 * z = relu?(BN(y) + res), res of y's shape and dtype. Not in the reference
 * (its nets have no residual); the ReLU mask for the backward is z > 0. */
int qd_bn_forward_res(long long M, int C, int dtype, const void* y, const void* res, const float* gamma,
                      const float* beta, float* run_mean, float* run_var, float momentum, float eps, int relu,
                      int training, void* z, float* save_mean, float* save_invstd, void* ws, void* stream);
/* BN forward statistics in the layer's fprop epilogue:
 * qd_bn_stats_rows(d) = rows of per-(tile, 32-pixel warp) statistics the fprop
 * epilogue can write for d (0: this layer's forward path has none -- use
 * qd_bn_forward). qd_forward_bnstats = qd_forward that also writes them into
 * `stats` (float [rows*F mean | rows*F M2 | rows count], of the stored y
 * values); qd_bn_forward_stats merges the rows (Chan's formula, fixed order)
 * into the batch mean / biased variance (+ running update) and applies
 * z = relu?(BN(y) (+ res)) -- no reduction pass over y. */
int qd_bn_stats_rows(const qd_desc* d);
int qd_forward_bnstats(const qd_desc* d, const void* x, const void* wpack, const float* const bias[3], void* y,
                       void* a_cache, void* b_cache, void* workspace, float* stats, void* stream);
int qd_bn_forward_stats(long long M, int C, int dtype, const void* y, const void* res, const float* stats, int rows,
                        const float* gamma, const float* beta, float* run_mean, float* run_var, float momentum,
                        float eps, int relu, int training, void* z, float* save_mean, float* save_invstd,
                        void* stream);
/* BN(+ReLU) backward fused with the quadratic layer's backward prologue: from
 * dz (gradient of z) and the layer's y, a, b it forms dgamma, dbeta, the layer's
 * bias gradients db[] and the operand D the layer backward consumes; then call
 * qd_backward with QD_FLAG_D_GIVEN and D as `dy`. Stride-1 layers; not t3. */
int qd_bn_backward_D(const qd_desc* d, const void* dz, const void* y, const void* a, const void* b,
                     const float* gamma, const float* beta, const float* save_mean, const float* save_invstd,
                     int relu, void* D, float* dgamma, float* dbeta, float* const db[3], void* ws, void* stream);

/* Fused SGD + weight pack: the reference sgd_step
 * (trainer.py:50-61) on the fp32 weight roles, in place,
 *   v <- momentum v + (g + weight_decay w)   (v = g + weight_decay w when first != 0)
 *   w <- w - lr v
 * and, in the same pass, the updated weights written into wpack in the layout
 * qd_pack_weights produces (structural zeros of the layout are left as they
 * are: pass a wpack that was packed once before). fc / conv kinds, families
 * other than the T1 ones. Biases are not touched. */
int qd_sgd_pack(const qd_desc* d, float* const w[3], float* const mom[3], const float* const grad[3],
                float lr, float momentum, float weight_decay, int first, void* wpack, void* stream);

/* Max pooling around the quadratic layers in the QuadraNet training step
 * (QuadraVGG 2x2/2, QuadraResNet stem 3x3/2 pad 1), torch.nn.MaxPool2d
 * semantics (floor mode, -inf padding, first maximum wins, NaN propagates).
 * NHWC, C % 8 == 0. argmax: one byte per output element (window offset
 * ky*k + kx), written by the forward and read by the backward, which gathers
 * (no atomics: deterministic) and writes every element of dx. */
int qd_maxpool_forward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* x, void* y,
                       void* argmax, void* stream);
int qd_maxpool_backward(int N, int C, int H, int W, int k, int s, int p, int dtype, const void* dy,
                        const void* argmax, void* dx, void* stream);

/* im2col of an NHWC tensor for small-channel convs run as one fc GEMM (the
 * QuadraResNet 7x7/2 stem, the QuadraVGG first layer -- 3 input channels):
 * col[m][k], m = (n, oh, ow), run-padded columns k = ky runp + kx C + c with
 * runp = r*C rounded up to 8 (zeros in the run tails and from r*runp up to Kp,
 * a multiple of 8). Same geometry rules as conv_out_size (tensor.py:279). */
int qd_im2col(int N, int C, int H, int W, int r, int s, int p, int Kp, int dtype, const void* x, void* col,
              void* stream);

/* Forward: neurons.forward (neurons.py:235-276).
 * bias[i]: fp32 (F) per role (proposed ba, bb, bc; first_order b; else NULL).
 * y: output NHWC; a_cache/b_cache: the LayerCache a, b (proposed/t4, NHWC,
 * dtype) -- may be NULL when not needed by the family. */
int qd_forward(const qd_desc* d, const void* x, const void* wpack,
               const float* const bias[3], void* y, void* a_cache,
               void* b_cache, void* workspace, void* stream);

/* Backward: neurons.symbolic_backward (neurons.py:295-445).
 * dW[i]: fp32 reference-layout gradient per weight role (same order as
 * qd_pack_weights); db[i]: fp32 (F) per bias role; dx NHWC (may be NULL with
 * QD_FLAG_NO_DX). */
int qd_backward(const qd_desc* d, const void* x, const void* wpack,
                const void* a_cache, const void* b_cache, const void* dy,
                void* dx, float* const dW[3], float* const db[3],
                void* workspace, void* stream);

/* Which implementation qd_forward / qd_backward will use for d:
 * 0 = generic CUDA-core (SIMT) kernels (exact fp32 FFMA / bf16),
 * 1 = tcgen05/TMA kernels (bf16), 2 = depth-wise direct kernels,
 * 3 = fp32 on the tcgen05 kernels: each fp32 operand split into two bf16 terms
 *     (hi = bf16(v), lo = bf16(v - hi)), products hi*hi + hi*lo + lo*hi
 *     accumulated in fp32 -- one K-tripled GEMM; error ~1e-5 relative.
 *     proposed / t4 / first_order, stride 1, C and F multiples of 64.
 *     qd_pack_bytes / qd_pack_weights then use the [hi | lo | hi] layout and
 *     qd_sgd_pack returns QD_ERR_UNSUPPORTED (the layer packs itself). */
int qd_path(const qd_desc* d);

const char* qd_error_string(int status);
const char* qd_last_error(void); /* detail of the last failure (thread-local) */

/* Number of kernels this library has launched since load (benchmarks report
 * it as gpu_launches). */
unsigned long long qd_launch_count(void);

/* Per-kernel timing for benchmarks: with profiling on, the library records a
 * CUDA event on the launching stream after each of its kernels (also inside
 * CUDA-graph capture). qd_profile_mark records a start mark; qd_profile_read(i)
 * returns the name of the i-th mark and the ms since mark i-1 (i >= 1; the
 * caller synchronises first). */
int qd_profile(int enable);
int qd_profile_mark(void* stream);
int qd_profile_count(void);
int qd_profile_read(int i, const char** name, float* ms);

/* Library version string. */
const char* qd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QUADRA_B200_H */
