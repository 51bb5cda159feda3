// v2 closed-uniform (circulant) assembly: two sm_100a kernels over the
// UPPER-TRIANGLE tile pairs (I <= J) of the N x N matrix.
//
//  ik1_sym_kernel   IK1(I,J) = G_I K1 G_J^T (assemble_ik1, assembly.py:175-183;
//                   K1_grid, geometry.py:225-248).  K1 is evaluated once per
//                   node pair of the tile in shared memory (table-based ln on
//                   the FP64 pipe, never stored to HBM), then contracted with
//                   the rule band with register reuse.  Only the upper tile
//                   (I,J) is written: IK1 is symmetric.
//  x2_pairs_kernel  X2(I,J) and X2(J,I) of the log part (assemble_ik2,
//                   assembly.py:186-245, X-form) on the FP64 tensor cores
//                   (DMMA m8n8k4): Phi = Zext * Uext^T in skewed (diagonal)
//                   coordinates, the banded S contraction as a second DMMA,
//                   then the fused epilogue
//                     A(I,J) = alpha (w IK1(I,J) + X2(I,J) + X2(J,I)^T),
//                     A(J,I) = A(I,J)^T      (scale_and_symmetrize, :262-271).
//
// Both kernels are deterministic (no atomics on values).
#include <math.h>

#include "wq_common.cuh"

namespace wq {

constexpr int FT = 64;          // tile rows/cols
constexpr int FTHREADS = 256;   // 8 warps

// ---------------------------------------------------------------------------
// 0.5*ln(x), x > 0 normal: x = 2^e m, m in [1,2); c_j ~ 1/m on 128 mantissa
// bins; r = m c_j - 1 with one FMA rounding (|r| <= 2^-8); ln(1+r) by its
// degree-7 series; -ln c_j as a double-double table.  About 1 ulp.
// ---------------------------------------------------------------------------

__device__ double g_logtab[3 * 128];  // c_j | 0.5*(-ln c_j)_hi | 0.5*(-ln c_j)_lo
static bool g_logtab_ready[64];

int ensure_logtab() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && g_logtab_ready[dev]) return WQ_OK;
  double tab[3 * 128];
  for (int j = 0; j < 128; ++j) {
    long double mid = 1.0L + (j + 0.5L) / 128.0L;
    double c = (double)(1.0L / mid);
    long double nl = -logl((long double)c);
    double hi = (double)nl;
    double lo = (double)(nl - (long double)hi);
    tab[j] = c;
    tab[128 + j] = 0.5 * hi;
    tab[256 + j] = 0.5 * lo;
  }
  cudaError_t e = cudaMemcpyToSymbol(g_logtab, tab, sizeof(tab));
  if (e != cudaSuccess) {
    set_error("log table upload: %s", cudaGetErrorString(e));
    return WQ_ECUDA;
  }
  if (dev >= 0 && dev < 64) g_logtab_ready[dev] = true;
  return WQ_OK;
}

// 0.5 ln 2 = HLN2_A + HLN2_B, HLN2_A with 41 significant bits (e*A exact)
constexpr double HLN2_A = 0.3465735902798315;
constexpr double HLN2_B = 1.4117645281515789e-13;

__device__ __forceinline__ double half_ln(double x, const double* __restrict__ tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 13) & 127;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double r = fma(m, tab[j], -1.0);
  // 0.5 ln(1+r) = 0.5 r + r^2 q(r)
  double q = fma(r, 0.5 / 7.0, -0.5 / 6.0);
  q = fma(r, q, 0.5 / 5.0);
  q = fma(r, q, -0.5 / 4.0);
  q = fma(r, q, 0.5 / 3.0);
  q = fma(r, q, -0.25);
  const double r2 = r * r;
  const double de = (double)e;
  const double t_hi = fma(de, HLN2_A, tab[128 + j]);
  const double t_lo = fma(de, HLN2_B, tab[256 + j]);
  return t_hi + fma(r, 0.5, fma(r2, q, t_lo));
}

// upper-triangle tile pair index -> (bi, bj), bi <= bj, row bi holds nb - bi pairs
__device__ __forceinline__ void tri_index(int64_t t, int nb, int& bi, int& bj) {
  // start(b) = b*nb - b*(b-1)/2
  double B = 2.0 * nb + 1.0;
  int b = (int)floor((B - sqrt(B * B - 8.0 * (double)t)) * 0.5);
  if (b < 0) b = 0;
  if (b > nb - 1) b = nb - 1;
  auto start = [nb](int64_t x) { return x * nb - x * (x - 1) / 2; };
  while (b > 0 && start(b) > t) --b;
  while (b + 1 < nb && start(b + 1) <= t) ++b;
  bi = b;
  bj = b + (int)(t - start(b));
}

// ---------------------------------------------------------------------------
// ik1_sym_kernel
// ---------------------------------------------------------------------------

constexpr int QS = 16;  // K1 strip rows

__global__ void __launch_bounds__(FTHREADS, 2)
ik1_sym_kernel(wq_smooth_t sm, int nb, double* X, int64_t ldx, int span, int* flag) {
  extern __shared__ double smem[];
  const int wg = (int)sm.wg;
  const int64_t N = sm.n_rows;
  int bi, bj;
  tri_index(blockIdx.x, nb, bi, bj);
  const int64_t I0 = (int64_t)bi * FT, J0 = (int64_t)bj * FT;
  const int ni = (int)min((int64_t)FT, N - I0);
  const int nj = (int)min((int64_t)FT, N - J0);
  const int64_t qlo = sm.g_start[I0];
  const int nQ = (int)(sm.g_start[I0 + ni - 1] + wg - qlo);
  const int64_t rlo = sm.g_start[J0];
  const int nR = (int)(sm.g_start[J0 + nj - 1] + wg - rlo);
  const int nRp = span + 1;  // strip row stride

  double* tab = smem;                         // 384
  double* qx = tab + 384;                     // span each: q fx, fy, s, J
  double* qy = qx + span;
  double* qs = qy + span;
  double* qJ = qs + span;
  double* rx = qJ + span;                     // r fx, fy, s, J
  double* ry = rx + span;
  double* rs = ry + span;
  double* rJ = rs + span;
  double* Gi = rJ + span;                     // FT * wg
  double* Gj = Gi + FT * wg;                  // FT * wg
  double* K = Gj + FT * wg;                   // QS * nRp
  double* T1 = K + QS * nRp;                  // span * FT
  int* qa = reinterpret_cast<int*>(T1 + (size_t)span * FT);  // span
  int* ra = qa + span;                        // span
  int* jr0 = ra + span;                       // FT: first r (tile-local) of column j
  int* iq0 = jr0 + FT;                        // FT: first q (tile-local) of row i

  const int tid = threadIdx.x;
  for (int k = tid; k < 384; k += FTHREADS) tab[k] = g_logtab[k];
  for (int k = tid; k < nQ; k += FTHREADS) {
    int64_t a = pmod(qlo + k, sm.nq);
    qa[k] = (int)a;
    qx[k] = sm.fx[a]; qy[k] = sm.fy[a]; qs[k] = sm.s[a]; qJ[k] = sm.J[a];
  }
  for (int k = tid; k < nR; k += FTHREADS) {
    int64_t a = pmod(rlo + k, sm.nq);
    ra[k] = (int)a;
    rx[k] = sm.fx[a]; ry[k] = sm.fy[a]; rs[k] = sm.s[a]; rJ[k] = sm.J[a];
  }
  for (int k = tid; k < FT * wg; k += FTHREADS) {
    int ii = k / wg;
    Gi[k] = ii < ni ? sm.g_w[(I0 + ii) * wg + (k - ii * wg)] : 0.0;
    Gj[k] = ii < nj ? sm.g_w[(J0 + ii) * wg + (k - ii * wg)] : 0.0;
  }
  for (int k = tid; k < FT; k += FTHREADS) {
    jr0[k] = k < nj ? (int)(sm.g_start[J0 + k] - rlo) : 0;
    iq0[k] = k < ni ? (int)(sm.g_start[I0 + k] - qlo) : 0;
  }
  for (int k = tid; k < span * FT; k += FTHREADS) T1[k] = 0.0;
  __syncthreads();

  int bad = 0;
  const int mode = (int)sm.k1_mode;
  const double* __restrict__ invp2 = sm.invp2;
  for (int q0 = 0; q0 < nQ; q0 += QS) {
    const int nq_s = min(QS, nQ - q0);
    for (int e = tid; e < nq_s * nR; e += FTHREADS) {
      const int qq = e / nR, r = e - qq * nR;
      const int q = q0 + qq;
      const int a = qa[q], b = ra[r];
      double R;
      if (a == b) {
        R = qJ[q] * qJ[q];
      } else {
        const double dx = qx[q] - rx[r], dy = qy[q] - ry[r];
        const double d2 = fma(dx, dx, dy * dy);
        if (mode == WQ_K1_TABLE) {
          R = d2 * __ldg(invp2 + (a > b ? a - b : b - a));
        } else if (mode == WQ_K1_OPEN) {
          const double p = fabs(rs[r] - qs[q]);
          R = d2 / (p * p);
        } else {
          const double xx = fabs(rs[r] - qs[q]);
          const double p = (sm.period / kPi) * fabs(sin(kPi * xx / sm.period));
          R = d2 / (p * p);
        }
      }
      if (!(R > 0.0) || !(R < 1e300)) {
        bad = 1;
        R = 1.0;
      }
      K[qq * nRp + r] = half_ln(R, tab);
    }
    __syncthreads();
    // T1[q][j] = sum_w K[q][jr0_j + w] G_j[w]; thread: one q row, 4 consecutive j
    for (int e = tid; e < nq_s * (FT / 4); e += FTHREADS) {
      const int qq = e / (FT / 4), jc = (e - qq * (FT / 4)) * 4;
      const double* kr = K + qq * nRp;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = jc + u;
        const double* gj = Gj + j * wg;
        const double* kk = kr + jr0[j];
        for (int w = 0; w < wg; ++w) acc[u] = fma(kk[w], gj[w], acc[u]);
      }
      double* t = T1 + (size_t)(q0 + qq) * FT + jc;
      t[0] = acc[0]; t[1] = acc[1]; t[2] = acc[2]; t[3] = acc[3];
    }
    __syncthreads();
  }
  if (bad) atomicOr(flag, WQ_FLAG_R_NONPOSITIVE);

  // IK1[i][j] = sum_w G_i[w] T1[iq0_i + w][j]; thread: column j, 16 rows
  const int j = tid & (FT - 1);
  const int ig = tid / FT;  // 0..3
  for (int ib = 0; ib < FT / 4; ++ib) {
    const int i = ib * 4 + ig;
    if (i >= ni || j >= nj) continue;
    const double* gi = Gi + i * wg;
    const double* t = T1 + (size_t)iq0[i] * FT + j;
    double acc = 0.0;
    for (int w = 0; w < wg; ++w) acc = fma(gi[w], t[(size_t)w * FT], acc);
    X[(I0 + i) * ldx + J0 + j] = acc;
  }
}

// ---------------------------------------------------------------------------
// x2_pairs_kernel (DMMA)
// ---------------------------------------------------------------------------

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct X2Params {
  int64_t N, n;         // rows, circulant period (= N)
  int p, d;             // degrees (p = d, nref = 1)
  int nA, nApad;        // Z' columns (P+1) and padded to a multiple of 4
  int tu;               // elements per support (p+1)
  int ws, wspad;        // S band width (2d+1) and padded
  int ktot;             // tu*nApad + wspad
  int ustride;          // Usm row stride (== 12 mod 16 doubles)
  int zstride;          // Zext row stride (== 4 mod 16 doubles, >= nApad+1)
  int zrows;            // Zsm rows
  int amax;             // max row offset (max(tu, wspad) - 1)
  int ks;               // S-DMMA K (8 + 2d padded to mult of 4)
  double alpha, w_ik1;
};

constexpr int PSTRIDE = 76;  // Phi smem row stride (== 12 mod 16)
constexpr int TSTRIDE = 65;  // transpose staging stride

// Phi[m][i] for m in [M0, M0 + FT + 2d), i in tile rows (Usm), into Phs[i][m - M0]
template <int NKB>
__device__ __forceinline__ void phi_block(const X2Params& P, const double* Usm, const double* Zsm,
                                          double* Phs, int64_t M0, int64_t R0, int64_t gmin) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, c = lane & 3;
  // rows of this warp: R0 + 8*warp + (0..7); k-block base
  const int64_t kb0 = M0 - (R0 + 8 * warp + 7);
  double acc[NKB][2];
#pragma unroll
  for (int kb = 0; kb < NKB; ++kb) acc[kb][0] = acc[kb][1] = 0.0;
  const int sZ = P.tu * P.nApad / 4;
  const int nsteps = P.ktot / 4;
  const double* urow = Usm + (8 * warp + r) * P.ustride + c;
  const int zbase = (int)(kb0 + r + P.p - gmin);  // Zsm row of (kb=0, a=0)
  for (int s = 0; s < nsteps; ++s) {
    int off, col;
    if (s < sZ) {
      const int K = 4 * s;
      off = K / P.nApad;              // a
      col = (K - off * P.nApad) + c;  // alpha
    } else {
      off = 4 * (s - sZ) + c;         // t
      col = P.nApad;
    }
    const double b = urow[4 * s];
    const double* z = Zsm + (zbase - off) * P.zstride + col;
#pragma unroll
    for (int kb = 0; kb < NKB; ++kb) dmma(acc[kb][0], acc[kb][1], z[kb * 8 * P.zstride], b);
  }
  // scatter to Phs[i][m - M0], m = k + i
  const int span = FT + 2 * P.d;
#pragma unroll
  for (int kb = 0; kb < NKB; ++kb) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int il = 8 * warp + 2 * c + e;                 // tile-local row
      const int64_t k = kb0 + 8 * kb + r;
      const int mm = (int)(k + R0 + il - M0);
      if (mm >= 0 && mm < span) Phs[il * PSTRIDE + mm] = acc[kb][e];
    }
  }
}

// X2 block: out[a][b] = sum_m Phs[a][m] S_b[m - b + d] (a: tile rows of Phi, b: band columns)
// warp owns output row block `warp`, all 8 column blocks; acc in fragment layout
__device__ __forceinline__ void s_contract(const X2Params& P, const double* Phs, const double* Ssm,
                                           double (&acc)[8][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, c = lane & 3;
#pragma unroll
  for (int jb = 0; jb < 8; ++jb) acc[jb][0] = acc[jb][1] = 0.0;
  const int nks = P.ks / 4;
  const int bw = 2 * P.d;
#pragma unroll
  for (int jb = 0; jb < 8; ++jb) {
    for (int s = 0; s < nks; ++s) {
      const int mm = 4 * s + c;
      const double a = Phs[(8 * warp + r) * PSTRIDE + 8 * jb + mm];
      // B[mm][jcol]: jcol = r (lane>>2), t = mm - r
      const int t = mm - r;
      const double b = (t >= 0 && t <= bw) ? Ssm[(8 * jb + r) * 16 + t] : 0.0;
      dmma(acc[jb][0], acc[jb][1], a, b);
    }
  }
}

template <int NKB>
__global__ void __launch_bounds__(FTHREADS, 1)
x2_pairs_kernel(X2Params P, const double* __restrict__ Uext, const double* __restrict__ Zext,
                const double* __restrict__ sw, double* X, int64_t ldx, int nb) {
  extern __shared__ double smem[];
  double* Usm = smem;                              // FT * ustride
  double* Zsm = Usm + FT * P.ustride;              // zrows * zstride
  double* Phs = Zsm + P.zrows * P.zstride;         // FT * PSTRIDE (also transpose staging)
  double* Ssm = Phs + FT * PSTRIDE;                // FT * 16 (S band of the contraction side)
  int bi, bj;
  tri_index(blockIdx.x, nb, bi, bj);
  const int64_t I0 = (int64_t)bi * FT, J0 = (int64_t)bj * FT;
  const int64_t N = P.N, n = P.n;
  const int ni = (int)min((int64_t)FT, N - I0);
  const int nj = (int)min((int64_t)FT, N - J0);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, c = lane & 3;

  // Phs padding columns must be finite (they multiply zero B entries)
  for (int k = tid; k < FT * PSTRIDE; k += FTHREADS) Phs[k] = 0.0;

  double accA[8][2], accB[8][2];
  for (int orient = 0; orient < 2; ++orient) {
    // orient 0: Phi rows = I (Uext of I), m over J-range; contraction with S_J
    // orient 1: Phi rows = J, m over I-range; contraction with S_I
    const int64_t R0 = orient == 0 ? I0 : J0;
    const int nr = orient == 0 ? ni : nj;
    const int64_t C0 = orient == 0 ? J0 : I0;
    const int nc = orient == 0 ? nj : ni;
    const int64_t M0 = C0 - P.d;
    const int64_t kb0_min = M0 - (R0 + 8 * 7 + 7);
    const int64_t gmin = kb0_min + P.p - P.amax;
    __syncthreads();
    for (int k = tid; k < FT * P.ktot; k += FTHREADS) {
      const int row = k / P.ktot, col = k - row * P.ktot;
      Usm[row * P.ustride + col] = row < nr ? Uext[(R0 + row) * P.ktot + col] : 0.0;
    }
    for (int k = tid; k < P.zrows * P.zstride; k += FTHREADS) {
      const int row = k / P.zstride;
      const int64_t g = pmod(gmin + row, n);
      Zsm[k] = Zext[g * P.zstride + (k - row * P.zstride)];
    }
    for (int k = tid; k < FT * 16; k += FTHREADS) {
      const int row = k >> 4, t = k & 15;
      Ssm[k] = (row < nc && t < P.ws) ? sw[(C0 + row) * P.ws + t] : 0.0;
    }
    __syncthreads();
    phi_block<NKB>(P, Usm, Zsm, Phs, M0, R0, gmin);
    __syncthreads();
    if (orient == 0)
      s_contract(P, Phs, Ssm, accA);
    else
      s_contract(P, Phs, Ssm, accB);
  }
  __syncthreads();
  // stage X2(J,I) transposed: accB lane holds (j = 8warp + r, i = 8ib + 2c + e)
  double* Tst = Phs;  // FT * TSTRIDE <= FT * PSTRIDE
#pragma unroll
  for (int ib = 0; ib < 8; ++ib)
#pragma unroll
    for (int e = 0; e < 2; ++e) Tst[(8 * ib + 2 * c + e) * TSTRIDE + 8 * warp + r] = accB[ib][e];
  __syncthreads();
  // A(I,J)[i][j], accA lane holds (i = 8warp + r, j = 8jb + 2c + e)
  double vals[8][2];
  const int i_l = 8 * warp + r;
#pragma unroll
  for (int jb = 0; jb < 8; ++jb)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j_l = 8 * jb + 2 * c + e;
      double ik1 = 0.0;
      if (P.w_ik1 != 0.0 && i_l < ni && j_l < nj) ik1 = X[(I0 + i_l) * ldx + J0 + j_l];
      vals[jb][e] = P.alpha * (P.w_ik1 * ik1 + accA[jb][e] + Tst[i_l * TSTRIDE + j_l]);
    }
  __syncthreads();
#pragma unroll
  for (int jb = 0; jb < 8; ++jb)
#pragma unroll
    for (int e = 0; e < 2; ++e) Tst[i_l * TSTRIDE + 8 * jb + 2 * c + e] = vals[jb][e];
  __syncthreads();
  // coalesced writes of A(I,J) and A(J,I) = A(I,J)^T; diagonal tiles are
  // mirrored from their upper triangle so A is exactly symmetric
  for (int k = tid; k < FT * FT; k += FTHREADS) {
    const int a = k >> 6, b = k & 63;
    if (a < ni && b < nj) {
      const double v = (bi == bj && a > b) ? Tst[b * TSTRIDE + a] : Tst[a * TSTRIDE + b];
      X[(I0 + a) * ldx + J0 + b] = v;
    }
  }
  if (bi != bj) {
    for (int k = tid; k < FT * FT; k += FTHREADS) {
      const int a = k >> 6, b = k & 63;  // row J0+a, col I0+b
      if (a < nj && b < ni) X[(J0 + a) * ldx + I0 + b] = Tst[b * TSTRIDE + a];
    }
  }
}

// Zext[g] = [Z'[g][0..nA-1], 0.., ff[g] at column nApad, 0..]
__global__ void zext_kernel(int64_t n, int nA, int nApad, int zstride, const double* Zp,
                            const double* ff, double* Zext) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * zstride) return;
  int64_t g = e / zstride;
  int col = (int)(e - g * zstride);
  double v = 0.0;
  if (col < nA) v = Zp[g * nA + col];
  else if (col == nApad) v = ff[g];
  Zext[e] = v;
}

// self-test hooks: custom ln vs libdevice, and a DMMA fragment-layout GEMM
__global__ void selftest_log_kernel(int64_t n, const double* x, double* out_fast, double* out_ref) {
  __shared__ double tab[384];
  for (int k = threadIdx.x; k < 384; k += blockDim.x) tab[k] = g_logtab[k];
  __syncthreads();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out_fast[i] = half_ln(x[i], tab);
  out_ref[i] = 0.5 * log(x[i]);
}

__global__ void selftest_dmma_kernel(const double* A, const double* B, double* C) {
  // C(8x8) = A(8x4 row-major) B(4x8 row-major), one warp
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  double c0 = 0.0, c1 = 0.0;
  dmma(c0, c1, A[r * 4 + c], B[c * 8 + r]);
  C[r * 8 + 2 * c] = c0;
  C[r * 8 + 2 * c + 1] = c1;
}

}  // namespace wq

using namespace wq;

extern "C" {

int wq_ik1_sym(const wq_smooth_t* sm, double* X, int64_t ldx, int64_t max_span, int* flag,
               void* stream) {
  if (!sm || !X || !flag || sm->wg <= 0 || max_span < sm->wg || sm->n_rows <= 0) {
    set_error("wq_ik1_sym: bad arguments");
    return WQ_EINVAL;
  }
  if (sm->k1_mode == WQ_K1_TABLE && !sm->invp2) {
    set_error("wq_ik1_sym: table mode without invp2");
    return WQ_EINVAL;
  }
  int rc = ensure_logtab();
  if (rc) return rc;
  const int span = (int)max_span;
  const int wg = (int)sm->wg;
  size_t smem = (size_t)(384 + 8 * span + 2 * FT * wg + QS * (span + 1) + (size_t)span * FT) * 8 +
                (size_t)(2 * span + 2 * FT) * 4;
  if (smem > 227 * 1024) {
    set_error("wq_ik1_sym: node span %d too large (%zu B smem)", span, smem);
    return WQ_EUNSUPPORTED;
  }
  cudaFuncSetAttribute(ik1_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nb = ceil_div(sm->n_rows, FT);
  const int64_t pairs = (int64_t)nb * (nb + 1) / 2;
  ik1_sym_kernel<<<(unsigned)pairs, FTHREADS, smem, (cudaStream_t)stream>>>(*sm, nb, X, ldx, span,
                                                                            flag);
  return check_launch("wq_ik1_sym");
}

int wq_zext(int64_t n, int nA, int nApad, int zstride, const double* Zp, const double* ff,
            double* Zext, void* stream) {
  if (n <= 0 || !Zp || !ff || !Zext || nApad < nA || zstride < nApad + 1) {
    set_error("wq_zext: bad arguments");
    return WQ_EINVAL;
  }
  zext_kernel<<<ceil_div(n * zstride, 256), 256, 0, (cudaStream_t)stream>>>(n, nA, nApad, zstride,
                                                                            Zp, ff, Zext);
  return check_launch("wq_zext");
}

int wq_x2_pairs(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                const double* Uext, const double* Zext, const double* s_w, double alpha,
                double w_ik1, double* X, int64_t ldx, void* stream) {
  if (N <= 0 || p < 1 || !Uext || !Zext || !s_w || !X || nApad % 4 || ktot % 4 ||
      zstride < nApad + 1 || ws > 16 || 2 * p > 14) {
    set_error("wq_x2_pairs: bad arguments");
    return WQ_EINVAL;
  }
  X2Params P;
  P.N = N;
  P.n = N;
  P.p = p;
  P.d = p;
  P.nA = nA;
  P.nApad = nApad;
  P.tu = p + 1;
  P.ws = ws;
  P.wspad = ktot - (p + 1) * nApad;
  P.ktot = ktot;
  P.ustride = ((ktot + 3) / 16) * 16 + 12;
  if (P.ustride < ktot) P.ustride += 16;
  P.zstride = zstride;
  P.amax = (P.tu > P.wspad ? P.tu : P.wspad) - 1;
  const int need = FT + 2 * p + 7;
  const int nkb = (need + 7) / 8;
  P.zrows = 56 + 8 * nkb + P.amax;
  P.ks = ((8 + 2 * p) + 3) / 4 * 4;
  P.alpha = alpha;
  P.w_ik1 = w_ik1;
  if (8 * 7 + P.ks > PSTRIDE || FT + 2 * p > PSTRIDE) {
    set_error("wq_x2_pairs: degree too large for the Phi tile");
    return WQ_EUNSUPPORTED;
  }
  size_t smem = ((size_t)FT * P.ustride + (size_t)P.zrows * P.zstride + (size_t)FT * PSTRIDE +
                 (size_t)FT * 16) * 8;
  if (smem > 227 * 1024) {
    set_error("wq_x2_pairs: %zu B shared memory needed", smem);
    return WQ_EUNSUPPORTED;
  }
  const int nb = ceil_div(N, FT);
  const int64_t pairs = (int64_t)nb * (nb + 1) / 2;
  if (nkb == 10) {
    cudaFuncSetAttribute(x2_pairs_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    x2_pairs_kernel<10><<<(unsigned)pairs, FTHREADS, smem, (cudaStream_t)stream>>>(P, Uext, Zext, s_w,
                                                                                    X, ldx, nb);
  } else if (nkb == 11) {
    cudaFuncSetAttribute(x2_pairs_kernel<11>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    x2_pairs_kernel<11><<<(unsigned)pairs, FTHREADS, smem, (cudaStream_t)stream>>>(P, Uext, Zext, s_w,
                                                                                    X, ldx, nb);
  } else {
    set_error("wq_x2_pairs: unsupported k-block count %d", nkb);
    return WQ_EUNSUPPORTED;
  }
  return check_launch("wq_x2_pairs");
}

int wq_selftest_log(int64_t n, const double* x, double* out_fast, double* out_ref, void* stream) {
  int rc = ensure_logtab();
  if (rc) return rc;
  selftest_log_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(n, x, out_fast, out_ref);
  return check_launch("wq_selftest_log");
}

int wq_selftest_dmma(const double* A, const double* B, double* C, void* stream) {
  selftest_dmma_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(A, B, C);
  return check_launch("wq_selftest_dmma");
}

}  // extern "C"
