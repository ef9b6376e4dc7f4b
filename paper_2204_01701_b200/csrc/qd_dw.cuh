// Depth-wise quadratic convolution: the role table and kernel arguments shared by
// the direct (qd_dw.cu) and shared-memory tiled (qd_dwtile.cu) kernels.
#pragma once
#include "qd_kernels.h"

namespace qd {

// role table: which D block and which input (x or x*x) each weight role uses
struct DwFam {
  int nroles;
  int din[3];  // D block of role r (backward)
  int sq[3];   // role r reads x*x
};
__host__ __device__ inline DwFam dw_fam(int family) {
  DwFam f = {1, {0, 0, 0}, {0, 0, 0}};
  switch (family) {
    case QD_FAM_T2: f.sq[0] = 1; break;
    case QD_FAM_T4: f.nroles = 2; f.din[1] = 1; break;
    case QD_FAM_PROPOSED: f.nroles = 3; f.din[1] = 1; f.din[2] = 2; break;
    case QD_FAM_T2_LINEAR: f.nroles = 2; f.sq[0] = 1; break;  // Wa on x*x, Wc on x, both with D = g
    case QD_FAM_T2AND4: f.nroles = 3; f.din[1] = 1; f.din[2] = 2; f.sq[2] = 1; break;
    default: break;  // first_order, t3 (D = 2 g a)
  }
  return f;
}

struct DwArgs {
  int family, N, C, H, W, OH, OW, r, s, p;
  long long Min, Mout;
  int Jd;
};

// the tiled kernels (qd_dwtile.cu): r = 3, stride 1 / 2, C % 32 == 0
bool dw_tile_ok(const Plan& P);
int dw_tile_wgrad_split(const Plan& P);
template <typename T>
int dw_tile_forward(const Plan& P, const DwArgs& A, const T* x, const float* Wp, const float* const bias[3], T* y,
                    T* a, T* b, int plain, cudaStream_t st);
template <typename T>
int dw_tile_backward(const Plan& P, const DwArgs& A, const T* x, const T* D, const float* Wp, T* dx, float* part,
                     int split, cudaStream_t st);

}  // namespace qd
