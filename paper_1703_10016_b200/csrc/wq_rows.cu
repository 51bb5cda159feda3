// Row blocks of the general (non-circulant) path for multi-GPU assembly
// (SURVEY 8(e)): X[rows] = IK1[rows] + X2[rows], X2 = (2 Theta - C^T D) C with
// C = H^{-1} S, so for rows i in [i0, i1)
//   Phi[:, i] = 2 H^{-1} Theta^T[:, i] - F S[:, i],   F = H^{-1} D H^{-1}
//   X2[i][j]  = sum_t S[s_j + t][j] Phi[s_j + t][i]
// (assembly.py:233-245 in the X-form).  Theta^T columns of the block come from
// the row-restricted Theta kernels; D and F are replicated per rank.
#include "wq_common.cuh"

namespace wq {

// P[m][i - i0] = alpha P[m][i - i0] - sum_t F[m][(s_i + t) mod nf] S_i[t]
__global__ void gather_fs_rows_kernel(wq_logpart_t lp, double alpha, const double* F, double* P,
                                      int64_t i0, int64_t i1, int64_t ldp) {
  const int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = blockIdx.y;
  if (i >= i1) return;
  const int64_t nf = lp.n_fine;
  double acc = alpha * P[m * ldp + (i - i0)];
  const int64_t si = pmod(lp.s_start[i], nf);
  for (int t = 0; t < lp.ws; ++t) {
    const double s = lp.s_w[i * lp.ws + t];
    if (s != 0.0) acc = fma(-F[m * nf + wrap1(si + t, nf)], s, acc);
  }
  P[m * ldp + (i - i0)] = acc;
}

// X[i - i0][j] (+)= sum_t S_j[t] PhiT[i - i0][(s_j + t) mod nf]   (threads over j)
__global__ void phi_s_rows_kernel(wq_logpart_t lp, const double* PhiT, int64_t i0, double* X,
                                  int64_t ldx, int accumulate) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t il = blockIdx.y;
  if (j >= lp.n_rows) return;
  const int64_t nf = lp.n_fine;
  const double* ph = PhiT + il * nf;
  double acc = 0.0;
  const int64_t sj = pmod(lp.s_start[j], nf);
  for (int t = 0; t < lp.ws; ++t) {
    const double s = lp.s_w[j * lp.ws + t];
    if (s != 0.0) acc = fma(s, ph[wrap1(sj + t, nf)], acc);
  }
  double* dst = X + il * ldx + j;
  *dst = accumulate ? *dst + acc : acc;
}

}  // namespace wq

using namespace wq;

extern "C" {

int wq_gather_fs_rows(const wq_logpart_t* lp, double alpha, const double* F, double* P,
                      int64_t i0, int64_t i1, int64_t ldp, void* stream) {
  if (!lp || !F || !P || i0 < 0 || i1 > lp->n_rows || i1 <= i0 || ldp < i1 - i0) {
    set_error("wq_gather_fs_rows: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(i1 - i0, 128), (unsigned)lp->n_fine);
  gather_fs_rows_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(*lp, alpha, F, P, i0, i1, ldp);
  return check_launch("wq_gather_fs_rows");
}

int wq_phi_s_rows(const wq_logpart_t* lp, const double* PhiT, int64_t i0, int64_t i1, double* X,
                  int64_t ldx, int accumulate, void* stream) {
  if (!lp || !PhiT || !X || i0 < 0 || i1 > lp->n_rows || i1 <= i0 || ldx < lp->n_rows) {
    set_error("wq_phi_s_rows: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(lp->n_rows, 128), (unsigned)(i1 - i0));
  phi_s_rows_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(*lp, PhiT, i0, X, ldx, accumulate);
  return check_launch("wq_phi_s_rows");
}

}  // extern "C"
