// Log-singular part of the Galerkin matrix (assemble_ik2, assembly.py:186-245)
// in the X-form:
//
//   X2 = (2 Theta - C^T D) C,  C = H^{-1} S,   IK2 = (X2 + X2^T) / 2,
//
// * wq_pair_table   : gap-indexed double log moments (quadrature.py:441-504)
// * wq_circ_tables  : closed uniform simple-knot meshes: fold the (translation
//                     invariant) v, H^{-1} and D into per-gap tables
// * wq_ik2_circ     : fused Phi = H^{-1} Psi^T evaluation + banded S contraction
// * general path    : Theta^T / D element-pair gathers, banded Cholesky column
//                     solves, S gathers (open meshes, any multiplicities)
#include "wq_common.cuh"

namespace wq {

// ---------------------------------------------------------------------------
// pair-moment table
// ---------------------------------------------------------------------------

constexpr int PT_MAXG = 32;   // max Gauss order
constexpr int PT_MAXA = 24;   // max row degree + 1
constexpr int PT_MAXB = 8;    // max col degree + 1
constexpr int PT_TIERED = 58; // n_gauss value selecting the tiered rules 30 | 16 | 12

__global__ void __launch_bounds__(128)
pair_table_kernel(int64_t nel, int closed, int da, int db, double h, const double* near_unit,
                  const double* gx, const double* gw, int ng, const double* ca, const double* cb,
                  double* m2) {
  __shared__ double x[PT_MAXG], w[PT_MAXG];
  __shared__ double wa[PT_MAXG][PT_MAXA];   // w_g x_g^a
  __shared__ double wb[PT_MAXG][PT_MAXB];   // w_h x_h^b
  __shared__ double kern[PT_MAXG][PT_MAXG + 1];
  __shared__ double t[PT_MAXG][PT_MAXB];
  __shared__ double acc[PT_MAXA][PT_MAXB];
  const int64_t k = blockIdx.x;
  double keff;
  if (closed) {
    keff = (double)k - (double)nel * rint((double)k / (double)nel);
  } else {
    keff = (double)(k - (nel - 1));
  }
  const double delta = -keff;
  const int nA = da + 1, nB = db + 1;
  // tiered rules (ng == 58: orders 30 | 16 | 12 concatenated): 16 points at
  // gap 2 (one width of separation), 12 beyond -- converged to <= 7e-15 of
  // the natural slot scale at degree 16 x 4 (tests/test_oracle.py); near gaps
  // keep 30 for the periodic term
  int g_off = 0;
  if (ng == PT_TIERED) {
    const double ak = fabs(keff);
    if (ak >= 3.0) { g_off = 46; ng = 12; }
    else if (ak >= 2.0) { g_off = 30; ng = 16; }
    else ng = 30;
  }
  for (int g = threadIdx.x; g < ng; g += blockDim.x) {
    x[g] = gx[g_off + g];
    w[g] = gw[g_off + g];
  }
  __syncthreads();
  // w_g x_g^a by running products (a pow() per entry was most of this kernel's instructions)
  for (int g = threadIdx.x; g < ng; g += blockDim.x) {
    double p = 1.0;
    for (int a = 0; a < nA; ++a, p *= x[g]) {
      wa[g][a] = w[g] * p;
      if (a < nB) wb[g][a] = w[g] * p;
    }
  }
  const bool near = fabs(keff) <= 1.0;
  for (int e = threadIdx.x; e < nA * nB; e += blockDim.x) {
    int a = e / nB, b = e - a * nB;
    acc[a][b] = near ? near_unit[((int)keff + 1) * nA * nB + e] : 0.0;
  }
  __syncthreads();

  // pass 0: ln|v - u - delta| (far gaps); pass 1: periodic ln|sinc| (closed)
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 0 && near) continue;
    if (pass == 1 && !closed) continue;
    for (int e = threadIdx.x; e < ng * ng; e += blockDim.x) {
      int g = e / ng, hh = e - g * ng;
      double arg = (x[hh] - x[g]) - delta;  // v - u - delta, he = hf = 1
      double val;
      if (pass == 0) {
        val = log(fabs(arg));
      } else {
        double y = arg / (double)nel;          // np.sinc(arg / period)
        double py = kPi * y;
        double s = (y == 0.0) ? 1.0 : sin(py) / py;
        val = log(fabs(s));
      }
      kern[g][hh] = val;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < ng * nB; e += blockDim.x) {
      int g = e / nB, b = e - g * nB;
      double s = 0.0;
      for (int hh = 0; hh < ng; ++hh) s = fma(kern[g][hh], wb[hh][b], s);
      t[g][b] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nA * nB; e += blockDim.x) {
      int a = e / nB, b = e - a * nB;
      double s = 0.0;
      for (int g = 0; g < ng; ++g) s = fma(wa[g][a], t[g][b], s);
      acc[a][b] += s;
    }
    __syncthreads();
  }
  const double lh = log(h);
  for (int e = threadIdx.x; e < nA * nB; e += blockDim.x) {
    int a = e / nB, b = e - a * nB;
    double scale = h * h;                        // h^(2 + a + b)
    for (int q = 0; q < a + b; ++q) scale *= h;
    m2[k * nA * nB + e] = scale * (acc[a][b] + lh * (ca[a] * cb[b]));
  }
}

// ---------------------------------------------------------------------------
// circulant tables
// ---------------------------------------------------------------------------

__global__ void circ_z_kernel(int64_t n, int da, int db, const double* m2, const double* v0,
                              double* Z) {
  const int nA = da + 1, nB = db + 1;
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * nA) return;
  int64_t g = e / nA;
  int al = (int)(e - g * nA);
  double acc = 0.0;
  for (int b = 0; b < nB; ++b) {
    const double* row = m2 + pmod(g - b, n) * nA * nB + al * nB;
    for (int be = 0; be < nB; ++be) acc = fma(row[be], v0[be * nB + b], acc);
  }
  Z[e] = acc;
}

__global__ void circ_dd_kernel(int64_t n, int da, int db, const double* Z, const double* v0,
                               double* dd) {
  const int nA = da + 1, nB = db + 1;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double acc = 0.0;
  for (int a = 0; a < nB; ++a) {
    const double* z = Z + pmod(k + a, n) * nA;
    for (int al = 0; al < nB; ++al) acc = fma(v0[al * nB + a], z[al], acc);
  }
  dd[k] = acc;
}

// out[g][c] = sum_{|k|<=K} in[(g + k) mod n][c] taps[K + k]
__global__ void circ_corr_kernel(int64_t n, int nc, const double* in, const double* taps, int64_t K,
                                 double* out) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n * nc) return;
  int64_t g = e / nc;
  int c = (int)(e - g * nc);
  // start index (g - K) mod n, then step with a conditional wrap (no divisions)
  int64_t idx = g - K;
  while (idx < 0) idx += n;
  double acc = 0.0;
  for (int64_t k = 0; k <= 2 * K; ++k) {
    acc = fma(in[idx * nc + c], taps[k], acc);
    if (++idx == n) idx = 0;
  }
  out[e] = acc;
}

// ---------------------------------------------------------------------------
// fused circulant log part: X[i,j] (+)= sum_t S[s_j+t, j] Phi[s_j+t, i]
// ---------------------------------------------------------------------------

constexpr int CT = WQ_TILE;  // rows (i) and cols (j) per CTA

__global__ void __launch_bounds__(256)
ik2_circ_kernel(wq_logpart_t lp, const double* Zp, const double* ff, int64_t row0, int64_t row1,
                int64_t col0, int64_t col1, double* X, int64_t ldx, int accumulate) {
  extern __shared__ double smem[];
  const int nA = (int)lp.da + 1, tu = (int)lp.tu, ws = (int)lp.ws;
  const int64_t n = lp.n_fine;
  const int64_t I0 = row0 + (int64_t)blockIdx.y * CT;
  const int64_t J0 = col0 + (int64_t)blockIdx.x * CT;
  const int ni = (int)(row1 - I0 < CT ? row1 - I0 : CT);
  const int nj = (int)(col1 - J0 < CT ? col1 - J0 : CT);
  // unit-step starts (closed uniform simple knots, nref = 1)
  const int64_t mlo = lp.s_start[J0];
  const int mspan = CT - 1 + ws;
  const int64_t gmin = mlo - lp.e_start[I0] - (CT - 1) - (tu - 1);
  const int zspan = mspan + CT - 1 + tu - 1;
  const int64_t fmin = mlo - lp.s_start[I0] - (CT - 1) - (ws - 1);
  const int fspan = mspan + CT - 1 + ws - 1;

  double* Us = smem;                          // CT * tu * nA
  double* Zs = Us + CT * tu * nA;             // zspan * nA
  double* Fs = Zs + zspan * nA;               // fspan
  double* Si = Fs + fspan;                    // CT * ws
  double* Sj = Si + CT * ws;                  // CT * ws
  double* Ph = Sj + CT * ws;                  // mspan * CT

  for (int k = threadIdx.x; k < CT * tu * nA; k += blockDim.x) {
    int ii = k / (tu * nA);
    Us[k] = ii < ni ? lp.U[(I0 + ii) * tu * nA + (k - ii * tu * nA)] : 0.0;
  }
  for (int k = threadIdx.x; k < zspan * nA; k += blockDim.x) {
    int g = k / nA;
    Zs[k] = Zp[pmod(gmin + g, n) * nA + (k - g * nA)];
  }
  for (int k = threadIdx.x; k < fspan; k += blockDim.x) Fs[k] = ff[pmod(fmin + k, n)];
  for (int k = threadIdx.x; k < CT * ws; k += blockDim.x) {
    int ii = k / ws;
    Si[k] = ii < ni ? lp.s_w[(I0 + ii) * ws + (k - ii * ws)] : 0.0;
    Sj[k] = ii < nj ? lp.s_w[(J0 + ii) * ws + (k - ii * ws)] : 0.0;
  }
  __syncthreads();

  // Phi[mm][ii], m = mlo + mm
  for (int k = threadIdx.x; k < mspan * CT; k += blockDim.x) {
    int mm = k / CT, ii = k - mm * CT;
    double acc = 0.0;
    if (ii < ni) {
      // Zp row for (m, i, a): m - e_start[i] - a = (mlo + mm) - (e_start[I0] + ii) - a
      const int zb = (int)((mlo + mm) - (lp.e_start[I0] + ii) - gmin);
      const double* u = Us + ii * tu * nA;
      for (int a = 0; a < tu; ++a) {
        const double* z = Zs + (zb - a) * nA;
        const double* ua = u + a * nA;
        for (int al = 0; al < nA; ++al) acc = fma(ua[al], z[al], acc);
      }
      acc *= 2.0;
      const int fb = (int)((mlo + mm) - (lp.s_start[I0] + ii) - fmin);
      const double* si = Si + ii * ws;
      for (int t = 0; t < ws; ++t) acc = fma(-si[t], Fs[fb - t], acc);
    }
    Ph[mm * CT + ii] = acc;
  }
  __syncthreads();

  for (int k = threadIdx.x; k < CT * CT; k += blockDim.x) {
    int ii = k / CT, jj = k - ii * CT;
    if (ii >= ni || jj >= nj) continue;
    const double* sj = Sj + jj * ws;
    double acc = 0.0;
    for (int t = 0; t < ws; ++t) acc = fma(sj[t], Ph[(jj + t) * CT + ii], acc);
    double* dst = X + (I0 - row0 + ii) * ldx + (J0 - col0 + jj);
    *dst = accumulate ? *dst + acc : acc;
  }
}

// ---------------------------------------------------------------------------
// general path (open meshes): element-pair gathers + banded solves
// ---------------------------------------------------------------------------

__device__ __forceinline__ int64_t gap_index(const wq_pairs_t& pp, int64_t e, int64_t f) {
  return pp.closed ? pmod(f - e, pp.n_el) : f - e + pp.n_el - 1;
}

// Theta^T[l][i] = sum_{(f,b) in inc_v(l)} sum_{(e,a) in inc_u(i)} u[e][:,a]^T M2[gap] v[f][:,b]
// (columns i in [row0, row1) only: a rank's row block, out[l * ld + i - row0])
__global__ void theta_t_kernel(wq_pairs_t pp, int64_t row0, int64_t row1, int64_t ld, double* out) {
  int64_t i = row0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t l = blockIdx.y;
  if (i >= row1) return;
  const int nA = (int)pp.da + 1, nB = (int)pp.db + 1, nU = (int)pp.pu + 1;
  double acc = 0.0;
  for (int vb = 0; vb < pp.wv; ++vb) {
    int64_t f = pp.v_el[l * pp.wv + vb];
    if (f < 0) continue;
    int b = (int)pp.v_loc[l * pp.wv + vb];
    const double* vf = pp.v + f * nB * nB;
    for (int ua = 0; ua < pp.wu; ++ua) {
      int64_t e = pp.u_el[i * pp.wu + ua];
      if (e < 0) continue;
      int a = (int)pp.u_loc[i * pp.wu + ua];
      const double* ue = pp.u + e * nA * nU;
      const double* m = pp.m2 + gap_index(pp, e, f) * nA * nB;
      double s = 0.0;
      for (int al = 0; al < nA; ++al) {
        double r = 0.0;
        for (int be = 0; be < nB; ++be) r = fma(m[al * nB + be], vf[be * nB + b], r);
        s = fma(ue[al * nU + a], r, s);
      }
      acc += s;
    }
  }
  out[l * ld + i - row0] = acc;
}

// D[l][m] = sum_{(e,a) in inc_v(l)} sum_{(f,b) in inc_v(m)} v[e][:,a]^T M2[gap][:db+1] v[f][:,b]
__global__ void dmat_kernel(wq_pairs_t pp, double* out) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t l = blockIdx.y;
  if (m >= pp.n_fine) return;
  const int nA = (int)pp.da + 1, nB = (int)pp.db + 1;
  double acc = 0.0;
  for (int va = 0; va < pp.wv; ++va) {
    int64_t e = pp.v_el[l * pp.wv + va];
    if (e < 0) continue;
    int a = (int)pp.v_loc[l * pp.wv + va];
    const double* ve = pp.v + e * nB * nB;
    for (int vb = 0; vb < pp.wv; ++vb) {
      int64_t f = pp.v_el[m * pp.wv + vb];
      if (f < 0) continue;
      int b = (int)pp.v_loc[m * pp.wv + vb];
      const double* vf = pp.v + f * nB * nB;
      const double* mm = pp.m2 + gap_index(pp, e, f) * nA * nB;
      double s = 0.0;
      for (int al = 0; al < nB; ++al) {
        double r = 0.0;
        for (int be = 0; be < nB; ++be) r = fma(mm[al * nB + be], vf[be * nB + b], r);
        s = fma(ve[al * nB + a], r, s);
      }
      acc += s;
    }
  }
  out[l * pp.n_fine + m] = acc;
}

// X <- H^{-1} X column by column, H = L L^T banded (Lb[k][j] = L[k][k-j]).
__global__ void band_solve_cols_kernel(int64_t n, int bw, const double* Lb, double* X,
                                       int64_t ncols, int64_t ldx) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  double* x = X + c;
  for (int64_t k = 0; k < n; ++k) {
    double s = x[k * ldx];
    const double* lk = Lb + k * (bw + 1);
    for (int j = 1; j <= bw && j <= k; ++j) s = fma(-lk[j], x[(k - j) * ldx], s);
    x[k * ldx] = s / lk[0];
  }
  for (int64_t k = n - 1; k >= 0; --k) {
    double s = x[k * ldx];
    for (int j = 1; j <= bw && k + j < n; ++j) s = fma(-Lb[(k + j) * (bw + 1) + j], x[(k + j) * ldx], s);
    x[k * ldx] = s / Lb[k * (bw + 1)];
  }
}

// Cyclic banded SPD solve, X <- H^{-1} X per column, with the arrow-shaped
// Cholesky factor of the seam-coupled band: H = [[A11, A21^T], [A21, A22]],
// A11 (m x m, m = n - bw) banded = L11 L11^T (Lb), L21 = A21 L11^{-T} (bw x m,
// dense), A22 - L21 L21^T = L22 L22^T (bw x bw, lower, row-major).
__global__ void cyc_solve_cols_kernel(int64_t n, int bw, const double* Lb, const double* L21,
                                      const double* L22, double* X, int64_t ncols, int64_t ldx) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  double* x = X + c;
  const int64_t m = n - bw;
  for (int64_t k = 0; k < m; ++k) {  // y1 = L11^{-1} x1
    double s = x[k * ldx];
    const double* lk = Lb + k * (bw + 1);
    for (int j = 1; j <= bw && j <= k; ++j) s = fma(-lk[j], x[(k - j) * ldx], s);
    x[k * ldx] = s / lk[0];
  }
  double y2[16];
  for (int k = 0; k < bw; ++k) {  // y2 = L22^{-1} (x2 - L21 y1)
    double s = x[(m + k) * ldx];
    const double* l = L21 + (int64_t)k * m;
    for (int64_t j = 0; j < m; ++j) s = fma(-l[j], x[j * ldx], s);
    for (int j = 0; j < k; ++j) s = fma(-L22[k * bw + j], y2[j], s);
    y2[k] = s / L22[k * bw + k];
  }
  for (int k = bw - 1; k >= 0; --k) {  // z2 = L22^{-T} y2
    double s = y2[k];
    for (int j = k + 1; j < bw; ++j) s = fma(-L22[j * bw + k], y2[j], s);
    y2[k] = s / L22[k * bw + k];
    x[(m + k) * ldx] = y2[k];
  }
  for (int64_t j = 0; j < m; ++j) {  // y1 -= L21^T z2
    double s = x[j * ldx];
    for (int k = 0; k < bw; ++k) s = fma(-L21[(int64_t)k * m + j], y2[k], s);
    x[j * ldx] = s;
  }
  for (int64_t k = m - 1; k >= 0; --k) {  // z1 = L11^{-T} (...)
    double s = x[k * ldx];
    for (int j = 1; j <= bw && k + j < m; ++j) s = fma(-Lb[(k + j) * (bw + 1) + j], x[(k + j) * ldx], s);
    x[k * ldx] = s / Lb[k * (bw + 1)];
  }
}

__global__ void transpose_kernel(const double* in, int64_t rows, int64_t cols, double* out) {
  __shared__ double t[32][33];
  int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int y = ty; y < 32; y += 8) {
    int64_t r = r0 + y, c = c0 + tx;
    if (r < rows && c < cols) t[y][tx] = in[r * cols + c];
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    int64_t r = c0 + y, c = r0 + tx;
    if (r < cols && c < rows) out[r * rows + c] = t[tx][y];
  }
}

// P[m][i] = alpha P[m][i] - sum_t F[m][(s_i + t) mod nf] S_i[t]; each CTA keeps
// the S band of its 128 columns i in registers and sweeps GF_ROWS rows m, GF_B rows
// per batch with every load of the batch issued before its FMAs (the per-row loop
// was DRAM-latency bound: one P load in flight per thread)
constexpr int GF_ROWS = 32;
constexpr int GF_MAXWS = 20;   // 3p + 2 fine functions per S column: nref = 2 up to p = 6
constexpr int GF_B = 4;
template <int WS>
__global__ void __launch_bounds__(128) gather_fs_kernel(wq_logpart_t lp, double alpha,
                                                        const double* F, double* P) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.y * GF_ROWS;
  if (i >= lp.n_rows) return;
  const int64_t nf = lp.n_fine, nr = lp.n_rows;
  double sw[WS];
  int col[WS];
#pragma unroll
  for (int t = 0; t < WS; ++t) {
    sw[t] = lp.s_w[i * WS + t];
    col[t] = (int)pmod(lp.s_start[i] + t, nf);
  }
  const int64_t m1 = m0 + GF_ROWS < nf ? m0 + GF_ROWS : nf;
  for (int64_t m = m0; m < m1; m += GF_B) {
    double acc[GF_B], fv[GF_B][WS];
#pragma unroll
    for (int u = 0; u < GF_B; ++u) {
      const int64_t mm = m + u < m1 ? m + u : m1 - 1;   // clamped (duplicate, not stored)
      acc[u] = P[mm * nr + i];
      const double* fr = F + mm * nf;
#pragma unroll
      for (int t = 0; t < WS; ++t) fv[u][t] = __ldg(fr + col[t]);
    }
#pragma unroll
    for (int u = 0; u < GF_B; ++u) {
      double a = alpha * acc[u];
#pragma unroll
      for (int t = 0; t < WS; ++t) a = fma(-fv[u][t], sw[t], a);
      if (m + u < m1) P[(m + u) * nr + i] = a;
    }
  }
}

// P[m][i] = alpha P[m][i] - sum_t Y[(s_i + t) mod nf][m] S_i[t]: gather_fs with F = Y^T read
// straight from Y (no transposed copy).  A CTA takes 64 columns i and GY_M rows m: the
// Y rows its bands touch (s_first .. s_last + WS - 1, `span` of them) x GY_M columns m are
// staged through shared memory (coalesced 256-byte row pieces in, conflict-free column
// reads out: row stride GY_M + 1).
constexpr int GY_I = 64, GY_M = 32, GY_B = 4;
template <int WS>
__global__ void __launch_bounds__(128) gather_yts_kernel(wq_logpart_t lp, double alpha,
                                                         const double* Y, double* P, int span) {
  extern __shared__ double ysm[];   // [span][GY_M + 1]
  const int64_t nf = lp.n_fine, nr = lp.n_rows;
  const int64_t i0 = (int64_t)blockIdx.x * GY_I, m0 = (int64_t)blockIdx.y * GY_M;
  const int64_t ilast = min(i0 + GY_I, nr) - 1;
  const int64_t sfirst = lp.s_start[i0];
  const int rows = (int)(lp.s_start[ilast] - sfirst) + WS;   // <= span (host-checked)
  const int mcnt = (int)min((int64_t)GY_M, nf - m0);
  {
    // one warp per staged row (a 256-byte piece of a Y row), the row index reduced once
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t sf = pmod(sfirst, nf);
    const int rmax = rows < span ? rows : span;
    for (int r = w; r < rmax; r += 4) {
      int64_t g = sf + r;
      while (g >= nf) g -= nf;
      if (lane < mcnt) ysm[r * (GY_M + 1) + lane] = __ldg(Y + g * nf + m0 + lane);
    }
  }
  __syncthreads();
  const int il = threadIdx.x & (GY_I - 1), half = threadIdx.x >> 6;
  const int64_t i = i0 + il;
  if (i >= nr) return;
  double sw[WS];
#pragma unroll
  for (int t = 0; t < WS; ++t) sw[t] = lp.s_w[i * WS + t];
  const double* yb = ysm + (int)(lp.s_start[i] - sfirst) * (GY_M + 1);
  const int mh0 = half * (GY_M / 2), mh1 = min(mcnt, mh0 + GY_M / 2);
  for (int mm = mh0; mm < mh1; mm += GY_B) {
    double pv[GY_B];
#pragma unroll
    for (int u = 0; u < GY_B; ++u) pv[u] = mm + u < mh1 ? P[(m0 + mm + u) * nr + i] : 0.0;
#pragma unroll
    for (int u = 0; u < GY_B; ++u) {
      if (mm + u < mh1) {
        double a = alpha * pv[u];
#pragma unroll
        for (int t = 0; t < WS; ++t) a = fma(-yb[t * (GY_M + 1) + mm + u], sw[t], a);
        P[(m0 + mm + u) * nr + i] = a;
      }
    }
  }
}

// X[j][i] (+)= sum_t S_j[t] Phi[(s_j + t) mod nf][i]; each CTA sweeps ST_ROWS
// consecutive j (their Phi rows overlap: L1 reuse), ST_B rows j per batch with the
// batch's loads issued before its FMAs
#ifndef WQ_ST_ROWS
#define WQ_ST_ROWS 16
#endif
constexpr int ST_ROWS = WQ_ST_ROWS;
constexpr int ST_B = 4;
template <int WS>
__global__ void __launch_bounds__(128) add_st_phi_kernel(wq_logpart_t lp, const double* Phi,
                                                         int64_t row0, int64_t row1, double* X,
                                                         int64_t ldx, int accumulate) {
  // the CTA's rows j: wrapped band start and weights staged once (broadcast reads), so
  // the per-entry work is WS loads + WS FMAs with pointer increments (the int64 modulo
  // and wrap per load made the kernel issue-bound: 75 % issue at 1.6 TB/s)
  __shared__ int64_t sst[ST_ROWS];
  __shared__ double ssw[ST_ROWS][WS];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j0 = row0 + (int64_t)blockIdx.y * ST_ROWS;
  const int64_t nf = lp.n_fine, nr = lp.n_rows;
  const int64_t j1 = j0 + ST_ROWS < row1 ? j0 + ST_ROWS : row1;
  for (int k = threadIdx.x; k < ST_ROWS * (WS + 1); k += blockDim.x) {
    const int u = k / (WS + 1), t = k - u * (WS + 1);
    const int64_t jj = j0 + u < j1 ? j0 + u : j1 - 1;
    if (t == WS) sst[u] = pmod(lp.s_start[jj], nf);
    else ssw[u][t] = lp.s_w[jj * WS + t];
  }
  __syncthreads();
  if (i >= nr) return;
  for (int64_t j = j0; j < j1; j += ST_B) {
    double pv[ST_B][WS], xv[ST_B];
#pragma unroll
    for (int u = 0; u < ST_B; ++u) {
      const int uu = (int)(j - j0) + u < (int)(j1 - j0) ? (int)(j - j0) + u : (int)(j1 - j0) - 1;
      const int64_t sj = sst[uu];
      if (sj + WS <= nf) {
        const double* p = Phi + sj * nr + i;
#pragma unroll
        for (int t = 0; t < WS; ++t, p += nr) pv[u][t] = __ldg(p);
      } else {
#pragma unroll
        for (int t = 0; t < WS; ++t) pv[u][t] = __ldg(Phi + wrap1(sj + t, nf) * nr + i);
      }
      xv[u] = accumulate ? X[(j0 + uu - row0) * ldx + i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < ST_B; ++u) {
      const int uu = (int)(j - j0) + u;
      double acc = 0.0;
      if (uu < (int)(j1 - j0)) {
#pragma unroll
        for (int t = 0; t < WS; ++t) acc = fma(ssw[uu][t], pv[u][t], acc);
        X[(j0 + uu - row0) * ldx + i] = xv[u] + acc;
      }
    }
  }
}

// A = alpha (X + X^T), X[j][i] = (X_in[j][i] if accumulate) + sum_t S_j[t] Phi[(s_j + t) mod nf][i]
// (add_st_phi followed by symmetrize, fused: X2^T is never written).  One CTA per 32 x 32 tile
// pair (bi <= bj); each thread forms 4 entries of both tiles (band sums over coalesced Phi row
// pieces), the transposed partners meet in shared memory.  In place on X.
template <int WS>
__global__ void __launch_bounds__(256) st_phi_sym_kernel(wq_logpart_t lp, const double* Phi,
                                                         double* X, double alpha, int accumulate,
                                                         int nb) {
  __shared__ double a[32][33];
  __shared__ double b[32][33];
  __shared__ int64_t sst[64];
  __shared__ double ssw[64][WS];
  const int64_t n = lp.n_rows, nf = lp.n_fine;
  int bi, bj;
  tri_index(blockIdx.x, nb, bi, bj);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
  const int64_t r0 = (int64_t)bi * 32, c0 = (int64_t)bj * 32;
  // bands of the rows r0 .. r0+31 (first half) and c0 .. c0+31 (second half)
  for (int k = threadIdx.x; k < 64 * (WS + 1); k += 256) {
    const int u = k / (WS + 1), t = k - u * (WS + 1);
    int64_t j = (u < 32 ? r0 : c0 - 32) + u;
    if (j >= n) j = n - 1;
    if (t == WS) sst[u] = pmod(lp.s_start[j], nf);
    else ssw[u][t] = lp.s_w[j * WS + t];
  }
  __syncthreads();
  // band sum of row slot u (0..63) at column col
  auto band = [&](int u, int64_t col) {
    const int64_t sj = sst[u];
    double acc = 0.0;
    if (sj + WS <= nf) {
      const double* p = Phi + sj * n + col;
#pragma unroll
      for (int t = 0; t < WS; ++t, p += n) acc = fma(ssw[u][t], __ldg(p), acc);
    } else {
#pragma unroll
      for (int t = 0; t < WS; ++t) acc = fma(ssw[u][t], __ldg(Phi + wrap1(sj + t, nf) * n + col), acc);
    }
    return acc;
  };
#pragma unroll
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = r0 + y, c = c0 + tx;
    double va = 0.0, vb = 0.0;
    if (r < n && c < n) va = (accumulate ? X[r * n + c] : 0.0) + band(y, c);
    const int64_t r2 = c0 + y, c2 = r0 + tx;
    if (r2 < n && c2 < n) vb = (accumulate ? X[r2 * n + c2] : 0.0) + band(32 + y, c2);
    a[y][tx] = va;
    b[y][tx] = vb;
  }
  __syncthreads();
#pragma unroll
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = r0 + y, c = c0 + tx;
    if (r < n && c < n) X[r * n + c] = alpha * (a[y][tx] + b[tx][y]);
    const int64_t r2 = c0 + y, c2 = r0 + tx;
    if (bi != bj && r2 < n && c2 < n) X[r2 * n + c2] = alpha * (b[y][tx] + a[tx][y]);
  }
}

#define WQ_WS_SWITCH(ws, CALL) \
  switch (ws) {                \
    case 1: CALL(1); break;    \
    case 2: CALL(2); break;    \
    case 3: CALL(3); break;    \
    case 4: CALL(4); break;    \
    case 5: CALL(5); break;    \
    case 6: CALL(6); break;    \
    case 7: CALL(7); break;    \
    case 8: CALL(8); break;    \
    case 9: CALL(9); break;    \
    case 10: CALL(10); break;  \
    case 11: CALL(11); break;  \
    case 12: CALL(12); break;  \
    case 13: CALL(13); break;  \
    case 14: CALL(14); break;  \
    case 15: CALL(15); break;  \
    case 16: CALL(16); break;  \
    case 17: CALL(17); break;  \
    case 18: CALL(18); break;  \
    case 19: CALL(19); break;  \
    case 20: CALL(20); break;  \
  }

}  // namespace wq

using namespace wq;

extern "C" {

int wq_pair_table(int64_t nel, int closed, int da, int db, double h, const double* near_unit,
                  const double* gx, const double* gw, int n_gauss, const double* ca,
                  const double* cb, double* m2, void* stream) {
  if (nel < 2 || da + 1 > PT_MAXA || db + 1 > PT_MAXB ||
      (n_gauss > PT_MAXG && n_gauss != PT_TIERED) || n_gauss < 1 ||
      !near_unit || !gx || !gw || !ca || !cb || !m2 || !(h > 0)) {
    set_error("wq_pair_table: bad arguments");
    return WQ_EINVAL;
  }
  int64_t n_gap = closed ? nel : 2 * nel - 1;
  pair_table_kernel<<<(unsigned)n_gap, 128, 0, (cudaStream_t)stream>>>(
      nel, closed, da, db, h, near_unit, gx, gw, n_gauss, ca, cb, m2);
  return check_launch("wq_pair_table");
}

int wq_circ_tables(int64_t n, int da, int db, const double* m2, const double* v0,
                   const double* hinv_taps, int64_t K, double* Zp, double* ff, double* work,
                   double* Zwork, void* stream) {
  if (n < 2 || !m2 || !v0 || !hinv_taps || !Zp || !ff || !work || !Zwork || K < 0 || K > n) {
    set_error("wq_circ_tables: bad arguments");
    return WQ_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int nA = da + 1;
  circ_z_kernel<<<ceil_div(n * nA, 256), 256, 0, s>>>(n, da, db, m2, v0, Zwork);
  circ_dd_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, da, db, Zwork, v0, ff);
  circ_corr_kernel<<<ceil_div(n * nA, 256), 256, 0, s>>>(n, nA, Zwork, hinv_taps, K, Zp);
  // ff = hinv * dd * hinv (hinv symmetric: correlation == convolution)
  circ_corr_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, 1, ff, hinv_taps, K, work);
  circ_corr_kernel<<<ceil_div(n, 256), 256, 0, s>>>(n, 1, work, hinv_taps, K, ff);
  return check_launch("wq_circ_tables");
}

int wq_ik2_circ(const wq_logpart_t* lp, const double* Zp, const double* ff, int64_t row0,
                int64_t row1, int64_t col0, int64_t col1, double* X, int64_t ldx, int accumulate,
                void* stream) {
  if (!lp || !Zp || !ff || !X || row0 < 0 || row1 > lp->n_rows || col0 < 0 ||
      col1 > lp->n_rows || row1 <= row0 || col1 <= col0 || lp->n_fine != lp->n_rows) {
    set_error("wq_ik2_circ: bad arguments");
    return WQ_EINVAL;
  }
  const int nA = (int)lp->da + 1, tu = (int)lp->tu, ws = (int)lp->ws;
  const int mspan = CT - 1 + ws;
  const int zspan = mspan + CT - 1 + tu - 1;
  const int fspan = mspan + CT - 1 + ws - 1;
  size_t smem = ((size_t)CT * tu * nA + (size_t)zspan * nA + fspan + 2 * CT * ws + (size_t)mspan * CT) * 8;
  if (smem > 227 * 1024) {
    set_error("wq_ik2_circ: tile does not fit in shared memory");
    return WQ_EUNSUPPORTED;
  }
  cudaFuncSetAttribute(ik2_circ_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(ceil_div(col1 - col0, CT), ceil_div(row1 - row0, CT));
  ik2_circ_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(*lp, Zp, ff, row0, row1, col0, col1, X,
                                                             ldx, accumulate);
  return check_launch("wq_ik2_circ");
}

int wq_theta_t(const wq_pairs_t* pp, double* thetaT, void* stream) {
  if (!pp || !thetaT) {
    set_error("wq_theta_t: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(pp->n_rows, 128), (unsigned)pp->n_fine);
  theta_t_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(*pp, 0, pp->n_rows, pp->n_rows, thetaT);
  return check_launch("wq_theta_t");
}

int wq_theta_t_rows(const wq_pairs_t* pp, int64_t row0, int64_t row1, double* thetaT, int64_t ld,
                    void* stream) {
  if (!pp || !thetaT || row0 < 0 || row1 > pp->n_rows || row1 <= row0 || ld < row1 - row0) {
    set_error("wq_theta_t_rows: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(row1 - row0, 128), (unsigned)pp->n_fine);
  theta_t_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(*pp, row0, row1, ld, thetaT);
  return check_launch("wq_theta_t_rows");
}

int wq_dmat(const wq_pairs_t* pp, double* D, void* stream) {
  if (!pp || !D) {
    set_error("wq_dmat: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(pp->n_fine, 128), (unsigned)pp->n_fine);
  dmat_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(*pp, D);
  return check_launch("wq_dmat");
}

int wq_band_solve_cols(int64_t n, int64_t bw, const double* Lb, double* X, int64_t ncols,
                       int64_t ldx, void* stream) {
  if (n <= 0 || bw < 0 || !Lb || !X || ncols <= 0) {
    set_error("wq_band_solve_cols: bad arguments");
    return WQ_EINVAL;
  }
  band_solve_cols_kernel<<<ceil_div(ncols, 128), 128, 0, (cudaStream_t)stream>>>(n, (int)bw, Lb, X,
                                                                                   ncols, ldx);
  return check_launch("wq_band_solve_cols");
}

int wq_cyc_solve_cols(int64_t n, int64_t bw, const double* Lb, const double* L21,
                      const double* L22, double* X, int64_t ncols, int64_t ldx, void* stream) {
  if (n <= 0 || bw < 1 || bw > 16 || bw >= n || !Lb || !L21 || !L22 || !X || ncols <= 0) {
    set_error("wq_cyc_solve_cols: bad arguments");
    return WQ_EINVAL;
  }
  cyc_solve_cols_kernel<<<ceil_div(ncols, 128), 128, 0, (cudaStream_t)stream>>>(n, (int)bw, Lb, L21,
                                                                                  L22, X, ncols, ldx);
  return check_launch("wq_cyc_solve_cols");
}

int wq_transpose(const double* in, int64_t rows, int64_t cols, double* out, void* stream) {
  if (!in || !out || rows <= 0 || cols <= 0) {
    set_error("wq_transpose: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32));
  transpose_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(in, rows, cols, out);
  return check_launch("wq_transpose");
}

int wq_gather_fs(const wq_logpart_t* lp, double alpha, const double* F, double* P, void* stream) {
  if (!lp || !F || !P) {
    set_error("wq_gather_fs: bad arguments");
    return WQ_EINVAL;
  }
  if (lp->ws > GF_MAXWS || lp->ws < 1) {
    set_error("wq_gather_fs: S band width %lld outside [1, %d]", (long long)lp->ws, GF_MAXWS);
    return WQ_EUNSUPPORTED;
  }
  dim3 grid(ceil_div(lp->n_rows, 128), ceil_div(lp->n_fine, GF_ROWS));
#define WQ_GF(W) gather_fs_kernel<W><<<grid, 128, 0, (cudaStream_t)stream>>>(*lp, alpha, F, P)
  WQ_WS_SWITCH(lp->ws, WQ_GF)
#undef WQ_GF
  return check_launch("wq_gather_fs");
}

int wq_gather_yts(const wq_logpart_t* lp, double alpha, const double* Y, double* P,
                  int64_t max_span, void* stream) {
  if (!lp || !Y || !P || max_span < 1) {
    set_error("wq_gather_yts: bad arguments");
    return WQ_EINVAL;
  }
  const size_t smem = (size_t)max_span * (GY_M + 1) * sizeof(double);
  if (lp->ws > GF_MAXWS || lp->ws < 1 || smem > 200 * 1024) {
    set_error("wq_gather_yts: S band width %lld or band span %lld unsupported", (long long)lp->ws,
              (long long)max_span);
    return WQ_EUNSUPPORTED;
  }
  dim3 grid(ceil_div(lp->n_rows, GY_I), ceil_div(lp->n_fine, GY_M));
#define WQ_GY(W)                                                                                \
  {                                                                                             \
    cudaFuncSetAttribute(gather_yts_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                         (int)smem);                                                            \
    gather_yts_kernel<W><<<grid, 128, smem, (cudaStream_t)stream>>>(*lp, alpha, Y, P,           \
                                                                    (int)max_span);             \
  }
  WQ_WS_SWITCH(lp->ws, WQ_GY)
#undef WQ_GY
  return check_launch("wq_gather_yts");
}

int wq_st_phi_sym(const wq_logpart_t* lp, const double* Phi, double* X, double alpha,
                  int accumulate, void* stream) {
  if (!lp || !Phi || !X) {
    set_error("wq_st_phi_sym: bad arguments");
    return WQ_EINVAL;
  }
  if (lp->ws > GF_MAXWS || lp->ws < 1) {
    set_error("wq_st_phi_sym: S band width %lld outside [1, %d]", (long long)lp->ws, GF_MAXWS);
    return WQ_EUNSUPPORTED;
  }
  const int nb = ceil_div(lp->n_rows, 32);
  const int64_t tiles = (int64_t)nb * (nb + 1) / 2;
#define WQ_SPS(W) \
  st_phi_sym_kernel<W><<<(unsigned)tiles, 256, 0, (cudaStream_t)stream>>>(*lp, Phi, X, alpha, accumulate, nb)
  WQ_WS_SWITCH(lp->ws, WQ_SPS)
#undef WQ_SPS
  return check_launch("wq_st_phi_sym");
}

int wq_add_st_phi(const wq_logpart_t* lp, const double* Phi, int64_t row0, int64_t row1, double* X,
                  int64_t ldx, int accumulate, void* stream) {
  if (!lp || !Phi || !X || row0 < 0 || row1 > lp->n_rows || row1 <= row0) {
    set_error("wq_add_st_phi: bad arguments");
    return WQ_EINVAL;
  }
  if (lp->ws > GF_MAXWS || lp->ws < 1) {
    set_error("wq_add_st_phi: S band width %lld outside [1, %d]", (long long)lp->ws, GF_MAXWS);
    return WQ_EUNSUPPORTED;
  }
  dim3 grid(ceil_div(lp->n_rows, 128), ceil_div(row1 - row0, ST_ROWS));
#define WQ_ST(W)                                                                     \
  add_st_phi_kernel<W><<<grid, 128, 0, (cudaStream_t)stream>>>(*lp, Phi, row0, row1, X, ldx, \
                                                               accumulate)
  WQ_WS_SWITCH(lp->ws, WQ_ST)
#undef WQ_ST
  return check_launch("wq_add_st_phi");
}

}  // extern "C"
