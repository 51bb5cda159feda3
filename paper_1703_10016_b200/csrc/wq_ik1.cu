// Fused smooth-kernel grid + banded sum-factorised contraction (north_star
// (a)+(b)); replaces assemble_ik1 (assembly.py:175-183) and the K1 grid of
// KernelSplit.K1_grid (geometry.py:225-248):
//
//   IK1[i, j] = sum_q sum_r G[i,q] K1(eta_q, eta_r) G[j,r],
//   K1 = 1/2 ln(|f(s) - f(t)|^2 / p(s,t)^2),  K1(s,s) = ln J(s).
//
// One CTA owns a TI x TJ output tile.  The node rows/columns its rules touch
// (a contiguous, seam-wrapping range of span <= 2*T + wg) are staged in
// shared memory, the K1 tile is evaluated there once (never written to HBM),
// then contracted as T = K1 G^T (per outer node) and X = G T.
#include "wq_common.cuh"
#include "wq_log.cuh"

namespace wq {

constexpr int IK1_TI = WQ_TILE;
constexpr int IK1_TJ = WQ_TILE;
constexpr int IK1_THREADS = 256;

struct NodeRec {
  double s, fx, fy, J;
};

__device__ __forceinline__ double k1_value(const wq_smooth_t& sm, int64_t qa, const NodeRec& a,
                                           int64_t ra, const NodeRec& b, int* bad,
                                           const double2* ltab) {
  double R;
  if (qa == ra) {
    R = a.J * a.J;  // continuity limit J^2 (geometry.py:240-245)
  } else if (sm.near_k > 0 && near_pair_j2(sm, qa, ra, &R)) {
    // distinct nodes within eps_diag: J^2 at the pair midpoint (geometry.py:237-245)
  } else {
    double dx = a.fx - b.fx, dy = a.fy - b.fy;
    double dist2 = dx * dx + dy * dy;
    if (sm.k1_mode == WQ_K1_TABLE) {
      int64_t g = ra > qa ? ra - qa : qa - ra;
      R = dist2 * sm.invp2[g];
    } else if (sm.k1_mode == WQ_K1_OPEN) {
      double p = fabs(b.s - a.s);
      R = dist2 / (p * p);
    } else {
      // periodic distance from the UNWRAPPED |t - s| (geometry.py:136-138)
      double x = fabs(b.s - a.s);
      double p = (sm.period / kPi) * fabs(sin(kPi * x / sm.period));
      R = dist2 / (p * p);
    }
  }
  if (!(R > 0.0)) {
    *bad = 1;
    return 0.5 * log(R);
  }
  return half_ln64t(R, ltab);   // table-based 0.5 ln, ~1 ulp (tests/test_gpu_kernels.py)
}

__global__ void __launch_bounds__(IK1_THREADS)
ik1_tile_kernel(wq_smooth_t sm, int64_t row0, int64_t row1, int64_t col0, int64_t col1, double* X,
                int64_t ldx, int accumulate, int span, int qc, int* flag, int sym) {
  extern __shared__ double smem[];
  __shared__ double2 ltab[64];
  // sym: rows == cols; only tiles on or above the diagonal, mirrored (K1 is
  // symmetric in (q, r), so IK1 = G K1 G^T is)
  if (sym && blockIdx.x < blockIdx.y) return;
  const int wg = (int)sm.wg;
  const int64_t I0 = row0 + (int64_t)blockIdx.y * IK1_TI;
  const int64_t J0 = col0 + (int64_t)blockIdx.x * IK1_TJ;
  const int ni = (int)(row1 - I0 < IK1_TI ? row1 - I0 : IK1_TI);
  const int nj = (int)(col1 - J0 < IK1_TJ ? col1 - J0 : IK1_TJ);
  const int64_t qlo = sm.g_start[I0];
  const int nQ = (int)(sm.g_start[I0 + ni - 1] + wg - qlo);
  const int64_t rlo = sm.g_start[J0];
  const int nR = (int)(sm.g_start[J0 + nj - 1] + wg - rlo);

  NodeRec* qn = reinterpret_cast<NodeRec*>(smem);         // span
  NodeRec* rn = qn + span;                                // span
  double* K = reinterpret_cast<double*>(rn + span);       // qc * span (a chunk of q rows)
  double* T = K + (size_t)qc * span;                      // span * TJ
  double* Gi = T + (size_t)span * IK1_TJ;                 // TI * wg
  double* Gj = Gi + IK1_TI * wg;                          // TJ * wg
  int* qidx = reinterpret_cast<int*>(Gj + IK1_TJ * wg);   // span
  int* ridx = qidx + span;                                // span

  for (int k = threadIdx.x; k < 128; k += blockDim.x) reinterpret_cast<double*>(ltab)[k] = kTang64[k];
  for (int k = threadIdx.x; k < nQ; k += blockDim.x) {
    int64_t a = pmod(qlo + k, sm.nq);
    qidx[k] = (int)a;
    qn[k] = NodeRec{sm.s[a], sm.fx[a], sm.fy[a], sm.J[a]};
  }
  for (int k = threadIdx.x; k < nR; k += blockDim.x) {
    int64_t a = pmod(rlo + k, sm.nq);
    ridx[k] = (int)a;
    rn[k] = NodeRec{sm.s[a], sm.fx[a], sm.fy[a], sm.J[a]};
  }
  for (int k = threadIdx.x; k < IK1_TI * wg; k += blockDim.x) {
    int ii = k / wg;
    Gi[k] = ii < ni ? sm.g_w[(I0 + ii) * wg + (k - ii * wg)] : 0.0;
  }
  for (int k = threadIdx.x; k < IK1_TJ * wg; k += blockDim.x) {
    int jj = k / wg;
    Gj[k] = jj < nj ? sm.g_w[(J0 + jj) * wg + (k - jj * wg)] : 0.0;
  }
  __syncthreads();

  // K1 rows in chunks of qc outer nodes (the whole span x span tile does not fit
  // shared memory for wide rules, e.g. p = 5 with nref = 2), each chunk
  // contracted into T[q][jj] = sum_w K[q][r_j + w] G[j][w] before the next
  int bad = 0;
  for (int q0c = 0; q0c < nQ; q0c += qc) {
    const int nq_c = min(qc, nQ - q0c);
    for (int k = threadIdx.x; k < nq_c * nR; k += blockDim.x) {
      int a = k / nR, b = k - a * nR;
      K[a * span + b] = k1_value(sm, qidx[q0c + a], qn[q0c + a], ridx[b], rn[b], &bad, ltab);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nq_c * IK1_TJ; k += blockDim.x) {
      int a = k / IK1_TJ, jj = k - a * IK1_TJ;
      double acc = 0.0;
      if (jj < nj) {
        int r0 = (int)(sm.g_start[J0 + jj] - rlo);
        const double* kr = K + a * span + r0;
        const double* gj = Gj + jj * wg;
        for (int w = 0; w < wg; ++w) acc = fma(kr[w], gj[w], acc);
      }
      T[(q0c + a) * IK1_TJ + jj] = acc;
    }
    __syncthreads();
  }
  if (bad) atomicOr(flag, WQ_FLAG_R_NONPOSITIVE);

  // X[i][j] = sum_w G[i][w] T[q_i + w][jj]
  for (int k = threadIdx.x; k < ni * IK1_TJ; k += blockDim.x) {
    int ii = k / IK1_TJ, jj = k - ii * IK1_TJ;
    if (jj >= nj) continue;
    int q0 = (int)(sm.g_start[I0 + ii] - qlo);
    const double* gi = Gi + ii * wg;
    double acc = 0.0;
    for (int w = 0; w < wg; ++w) acc = fma(gi[w], T[(q0 + w) * IK1_TJ + jj], acc);
    double* dst = X + (I0 - row0 + ii) * ldx + (J0 - col0 + jj);
    *dst = accumulate ? *dst + acc : acc;
    if (sym && J0 > I0) {
      double* mir = X + (J0 - col0 + jj) * ldx + (I0 - row0 + ii);
      *mir = accumulate ? *mir + acc : acc;
    }
  }
}

}  // namespace wq

using namespace wq;

extern "C" int wq_ik1(const wq_smooth_t* sm, int64_t row0, int64_t row1, int64_t col0, int64_t col1,
                      double* X, int64_t ldx, int accumulate, int64_t max_span, int* flag,
                      void* stream) {
  if (!sm || !X || !flag || row0 < 0 || row1 > sm->n_rows || col0 < 0 || col1 > sm->n_rows ||
      row1 <= row0 || col1 <= col0 || sm->wg <= 0 || max_span < sm->wg) {
    set_error("wq_ik1: bad arguments");
    return WQ_EINVAL;
  }
  if (sm->k1_mode == WQ_K1_TABLE && !sm->invp2) {
    set_error("wq_ik1: table mode without invp2");
    return WQ_EINVAL;
  }
  int span = (int)max_span;
  const size_t fixed = (size_t)2 * span * sizeof(NodeRec) + (size_t)span * IK1_TJ * 8 +
                       (size_t)(IK1_TI + IK1_TJ) * sm->wg * 8 + (size_t)2 * span * sizeof(int);
  const size_t budget = 225 * 1024;   // + the static ln table, under the 227 KB opt-in limit
  // K1 rows per chunk: the whole span when it fits, else as many as fit
  const int64_t qfit = fixed < budget ? (int64_t)((budget - fixed) / ((size_t)span * 8)) : 0;
  const int qc = (int)(qfit < span ? qfit : span);
  if (qc < 1) {
    set_error("wq_ik1: node span %d too large for one tile", span);
    return WQ_EUNSUPPORTED;
  }
  const size_t smem = fixed + (size_t)qc * span * 8;
  cudaFuncSetAttribute(ik1_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(ceil_div(col1 - col0, IK1_TJ), ceil_div(row1 - row0, IK1_TI));
  // the full square (the assemble_ik1 / general-path call) uses the symmetry
  const int sym = row0 == col0 && row1 == col1 && IK1_TI == IK1_TJ;
  ik1_tile_kernel<<<grid, IK1_THREADS, smem, (cudaStream_t)stream>>>(*sm, row0, row1, col0, col1, X,
                                                                     ldx, accumulate, span, qc, flag, sym);
  return check_launch("wq_ik1");
}
