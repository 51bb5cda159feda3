// Graded open meshes, lattice part on the FP64 tensor cores.
//
// wq_ystage (wq_ystage.cu) forms, per row tile and column tile,
//   Y[r][f][b] = sum_{(e,a) in inc(r)} h_e^b sum_al Cs_e[al][a] M'[k_f - k_e][al][b] + Lt_e[a][b]
//   Out[c][r]  = sum_{(f,b') in inc(c)} sum_b Y[r][f][b] v_f[b][b']
// on CUDA cores, bound by shared-memory bandwidth (every table value feeds a
// few FMAs).  On tiles whose row and column elements all lie on one lattice
// run (f - e = k_f - k_e), the inner sum is a GEMM in skewed coordinates
// u = f - e_r (e_r the first element of supp(r), s = e - e_r):
//   Y_b[r][e_r + u] = sum_{s, al} (Cs_{e_r+s}[al][a(r, e_r+s)] h^b) M'_b[u - s][al]
// -- the A operand is the Toeplitz matrix of the unit gap table slice b (the
// same for every row function), the B operand the rows' scaled coefficients.
// This is the x2_pairs scheme (wq_fast.cu) with K = 5 shifts x 17 (or 5)
// powers, packed densely, and one GEMM per column power b; Out accumulates the column
// contraction of each Y_b in shared memory, and the ln h_e term enters as
//   Out[c][r] += sum_b LtR[r][b] vsum[c][b].
// One CTA = 64 row functions x 64 column functions, 8 warps x 8 row functions;
// the table window of each b arrives by a 1-D TMA bulk copy.  Deterministic.
// Citations: quadrature.py:441-504 (unit-table recipe, scaling 497-500),
// assembly.py:186-245 (Theta / D assembly).
#include <type_traits>

#include "wq_async.cuh"
#include "wq_common.cuh"

namespace wq {

constexpr int YM_T = 64;             // row / column functions per tile
constexpr int YM_THREADS = 256;
constexpr int YM_NS = 5;             // shifts (elements per row support), p = 4
constexpr int YM_NB = 5;             // column polynomial slots (d + 1)
constexpr int YM_ZST = 20;           // table row stride (== 4 mod 16: conflict-free fragments)
constexpr int YM_FSP = 72;           // max column elements per tile (host-checked)
constexpr int YM_NKB = (YM_FSP + 7 + 7) / 8;   // 8-row skew blocks per warp
constexpr int YM_ESP = 68;           // max row-element spread per tile (host-checked)
constexpr int YM_ZR = YM_ESP + YM_NS - 1 + 8 * YM_NKB;   // staged table rows
constexpr int YM_PST = YM_FSP + 1;   // Phs row stride (odd)
constexpr int YM_PF = 10;            // B-fragment prefetch depth
constexpr int YM_NOT_PURE = INT32_MIN;
constexpr int YM_TFRONT = 8;         // zero table rows before gap -(n_el - 1)
constexpr int YM_WCM = 5;            // max column incidences (elements per fine function, p = 4)

struct YmArgs {
  int64_t n_cols, n_el;
  int wc;
  const int64_t* r_emin;   // (n_rows) first element of supp(r)
  const int64_t* c_el;     // (n_cols, wc) element of incidence, -1 = none
  const int64_t* c_loc;
  const int64_t* c_emin;
  const int64_t* c_emax;
  const double* v;         // (n_el, NB, NB) column coefficients v_f[be][b]
  const double* Cr;        // (NB, ceil8(n_rows), KP) B operand: Cs_{e_r+s}[al][a] h^b at k = s NAL + al,
                           // in DMMA B-fragment order [row / 8][k / 4][row % 8][k % 4]
  const double* LtR;       // (n_rows, NB)
  const double* vsum;      // (n_cols, NB)
  const double* Tb;        // (NB, n_tab, ZST) table slices, row g + n_el - 1 + TFRONT
  int64_t n_tab;
  const int* row_ko;       // (row tiles) lattice offset k_e - e of a pure row tile, or NOT_PURE
  const int* col_ko;       // (column tiles) ditto
  double* out;
  int64_t ldo, row0, out_row0;
  int sym;
};

template <int NAL>
struct YmCfg {
  static constexpr int KP = (YM_NS * NAL + 3) / 4 * 4;   // contraction (s, al) packed densely
  static constexpr int NSTEPS = KP / 4;
  static constexpr int PF = NSTEPS < YM_PF ? NSTEPS : YM_PF;
  // Zsm[2] | Phs | Cv (column incidences' v_f[b][b'] per b) | 2 mbarriers | Ci (ints)
  static constexpr int SMEM = 2 * YM_ZR * YM_ZST + YM_T * YM_PST + YM_T * YM_WCM * YM_NB + 2 +
                              YM_T * YM_WCM / 2;
};

template <int NAL>
__global__ void __launch_bounds__(YM_THREADS, 2) ystage_mma_kernel(YmArgs A, int64_t n_rows) {
  using C = YmCfg<NAL>;
  extern __shared__ double sm[];
  // column tiles fastest: the CTAs in flight share a row tile, so its B operand (Cr, 45 KB
  // per power) is fetched from HBM once and then served from L2
  const int ct = blockIdx.x, rt = blockIdx.y;
  const int ko = A.row_ko[rt];
  if (ko == YM_NOT_PURE || A.col_ko[ct] != ko) return;   // CUDA-core kernel handles the tile
  const int64_t R0 = A.row0 + (int64_t)rt * YM_T, C0 = (int64_t)ct * YM_T;
  if (A.sym && C0 + YM_T - 1 < R0) return;   // strictly below the diagonal: mirrored later
  constexpr int ZW = YM_ZR * YM_ZST;
  double* Zsm = sm;                          // [2][ZR][ZST] (double-buffered over b)
  double* Phs = Zsm + 2 * ZW;                // [T][PST]: Y_b[r][f - fa]
  double* Cv = Phs + YM_T * YM_PST;          // [T c][WCM][NB]
  uint64_t* bar = reinterpret_cast<uint64_t*>(Cv + YM_T * YM_WCM * YM_NB);   // [2]
  int* Ci = reinterpret_cast<int*>(bar + 2);   // [T c][WCM]: f - fa, or -1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rl = lane >> 2, cl = lane & 3;

  const int64_t fa = A.c_emin[C0];
  const int64_t emax_all = A.r_emin[R0 + YM_T - 1];
  const int64_t gbase = fa - emax_all - (YM_NS - 1);   // first staged gap
  const double* tsrc = A.Tb + (gbase + A.n_el - 1 + YM_TFRONT) * YM_ZST;
  const int64_t emax_w = A.r_emin[R0 + 8 * warp + 7];
  const int zoff = (int)(emax_all - emax_w) + (YM_NS - 1);   // window row of skew k = fa - emax_w
  // skew blocks this warp needs: its functions read rows fl - ef, fl < the tile's element span,
  // -ef <= the spread of the warp's first elements (YM_NKB covers the host-checked maxima;
  // with repeated knots 64 functions span far fewer elements)
  const int fspan = (int)(A.c_emax[C0 + YM_T - 1] - fa) + 1;
  const int nkb = min(YM_NKB, (fspan + (int)(emax_w - A.r_emin[R0 + 8 * warp]) + 7) >> 3);

  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  fence_proxy_async();
  __syncthreads();
  if (tid == 0)
    for (int b = 0; b < 2; ++b) {
      mbar_arrive_expect_tx(bar + b, ZW * 8);
      bulk_g2s(Zsm + b * ZW, tsrc + (int64_t)b * A.n_tab * YM_ZST, ZW * 8, bar + b);
    }
  // column incidences of the tile, once: element offset and v_f[b][b'] for every b
  for (int k = tid; k < YM_T * YM_WCM; k += YM_THREADS) {
    const int c = k / YM_WCM, w = k - c * YM_WCM;
    const int64_t cc = C0 + c;
    const int64_t f = w < A.wc ? A.c_el[cc * A.wc + w] : -1;
    Ci[k] = f >= 0 ? (int)(f - fa) : -1;
    const int bp = f >= 0 ? (int)A.c_loc[cc * A.wc + w] : 0;
#pragma unroll
    for (int b = 0; b < YM_NB; ++b)
      Cv[k * YM_NB + b] = f >= 0 ? __ldg(A.v + f * (YM_NB * YM_NB) + b * YM_NB + bp) : 0.0;
  }
  // Out[c][r] for this thread's column c and rows r = 16 rg + i, in registers; starts from
  // the ln h term sum_b LtR[r][b] vsum[c][b]
  const int ocol = tid & 63, rg = tid >> 6;
  double out[YM_T / 4];
  {
    double vs[YM_NB];
#pragma unroll
    for (int b = 0; b < YM_NB; ++b) vs[b] = __ldg(A.vsum + (C0 + ocol) * YM_NB + b);
#pragma unroll
    for (int i = 0; i < YM_T / 4; ++i) {
      const int64_t r = R0 + 16 * rg + i;
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < YM_NB; ++b) s = fma(__ldg(A.LtR + r * YM_NB + b), vs[b], s);
      out[i] = s;
    }
  }
  // the skewed output rows of this lane's functions: f = k + e_func
  // B-operand fragments of the warp's row group: one coalesced 256-byte load per k-step
  const double* __restrict__ brow0 = A.Cr + ((R0 + 8 * warp) / 8) * (C::NSTEPS * 32) + lane;
  int ef[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) ef[e] = (int)(A.r_emin[R0 + 8 * warp + 2 * cl + e] - emax_w);

  for (int b = 0; b < YM_NB; ++b) {
    const double* zb = Zsm + (b & 1) * ZW;
    const double* __restrict__ brow = brow0 + (int64_t)b * n_rows * C::KP;   // n_rows: padded to 8
    double bq[C::PF];
#pragma unroll
    for (int t = 0; t < C::PF; ++t) bq[t] = __ldg(brow + 32 * t);
    mbar_wait(bar + (b & 1), (unsigned)((b >> 1) & 1));

    // ---- Y_b in skewed coordinates: acc[kb] = rows k = fa - emax_w + 8 kb + rl ----
    double acc[YM_NKB][2];
#pragma unroll
    for (int kb = 0; kb < YM_NKB; ++kb) acc[kb][0] = acc[kb][1] = 0.0;
    const double* zl = zb + (zoff + rl) * YM_ZST;
    // NK = the blocks this warp needs (a compile-time count per branch: no predicated DMMAs)
    auto gemm = [&](auto nk) {
      constexpr int NK = decltype(nk)::value;
#pragma unroll
      for (int t = 0; t < C::NSTEPS; ++t) {
        // this lane's contraction index k = 4t + cl = s NAL + al (padding: zero B, any finite A)
        const int kk = min(4 * t + cl, YM_NS * NAL - 1);
        const int s = kk / NAL, al = kk - s * NAL;
        const double bfrag = bq[t % C::PF];
        if (t + C::PF < C::NSTEPS) bq[t % C::PF] = __ldg(brow + 32 * (t + C::PF));
        const double* z = zl - s * YM_ZST + al;
#pragma unroll
        for (int kb = 0; kb < NK; ++kb) dmma(acc[kb][0], acc[kb][1], z[8 * kb * YM_ZST], bfrag);
      }
    };
    if (nkb <= YM_NKB - 3) gemm(std::integral_constant<int, YM_NKB - 3>());
    else if (nkb == YM_NKB - 2) gemm(std::integral_constant<int, YM_NKB - 2>());
    else if (nkb == YM_NKB - 1) gemm(std::integral_constant<int, YM_NKB - 1>());
    else gemm(std::integral_constant<int, YM_NKB>());
    fence_proxy_async();
    __syncthreads();   // every warp is done with this window (and with Phs of b - 1)
    if (tid == 0 && b + 2 < YM_NB) {
      mbar_arrive_expect_tx(bar + (b & 1), ZW * 8);
      bulk_g2s(Zsm + (b & 1) * ZW, tsrc + (int64_t)(b + 2) * A.n_tab * YM_ZST, ZW * 8, bar + (b & 1));
    }
    // scatter: lane holds Y_b[func = 8 warp + 2 cl + e][f = fa + 8 kb + rl + ef[e]]
#pragma unroll
    for (int kb = 0; kb < YM_NKB; ++kb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int fl = 8 * kb + rl + ef[e];
        if (fl >= 0 && fl < fspan) Phs[(8 * warp + 2 * cl + e) * YM_PST + fl] = acc[kb][e];
      }
    __syncthreads();
    // ---- column contraction: Out[c][r] += sum_{(f,b') in inc(c)} Y_b[r][f] v_f[b][b'] ----
    // (this thread's column: incidences in registers, one shared load per FMA)
    {
      int fi[YM_WCM];
      double cv[YM_WCM];
#pragma unroll
      for (int w = 0; w < YM_WCM; ++w) {
        const int f = Ci[ocol * YM_WCM + w];
        fi[w] = f >= 0 ? f : 0;
        cv[w] = f >= 0 ? Cv[(ocol * YM_WCM + w) * YM_NB + b] : 0.0;
      }
      const double* ph = Phs + 16 * rg * YM_PST;
#pragma unroll
      for (int i = 0; i < YM_T / 4; ++i)
#pragma unroll
        for (int w = 0; w < YM_WCM; ++w) out[i] = fma(ph[i * YM_PST + fi[w]], cv[w], out[i]);
    }
  }
  // Out[c][r] through shared memory (the Phs region, stride T + 1) so that 64 consecutive r
  // of a column leave together
  __syncthreads();
  double* Os = Phs;
#pragma unroll
  for (int i = 0; i < YM_T / 4; ++i) Os[ocol * (YM_T + 1) + 16 * rg + i] = out[i];
  __syncthreads();
  for (int k = tid; k < YM_T * YM_T; k += YM_THREADS) {
    const int c = k >> 6, r = k & 63;
    A.out[(C0 + c) * A.ldo + R0 + r - A.out_row0] = Os[c * (YM_T + 1) + r];
  }
}

// Cr[b][r][s nal + al] = coef[e][al][a] h_e^(al+2) h_e^b, e = e_r + s with local index a of r
// (0 where r has no function on e, and in the padding up to kp), LtR[r][b] = sum_{(e,a)}
// ln h_e c_b h_e^b sum_al c_al coef[e][al][a] h_e^(al+2) (the ln h part of the unit-table
// scaling, quadrature.py:497-500)
__global__ void ystage_mma_prep_rows(int64_t n_rows, int nal, int kp, int nloc,
                                     const int64_t* e_rows, const int64_t* r_emin,
                                     const int64_t* r_emax, const double* coef, int ldal,
                                     const double* elh, const double* ca, const double* cb,
                                     double* Cr, double* LtR) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nrp = (n_rows + 7) / 8 * 8;   // rows padded to whole fragments
  // element (b, r, k) in B-fragment order
  auto at = [&](int b, int64_t rr, int k) -> double& {
    return Cr[(int64_t)b * nrp * kp + ((rr / 8) * (kp / 4) + k / 4) * 32 + (rr % 8) * 4 + k % 4];
  };
  if (r >= n_rows) {
    if (r < nrp)
      for (int k = 0; k < kp; ++k)
        for (int b = 0; b < YM_NB; ++b) at(b, r, k) = 0.0;
    return;
  }
  double lt[YM_NB] = {0, 0, 0, 0, 0};
  for (int k = YM_NS * nal; k < kp; ++k)
    for (int b = 0; b < YM_NB; ++b) at(b, r, k) = 0.0;
  for (int s = 0; s < YM_NS; ++s) {
    const int64_t e = r_emin[r] + s;
    int a = -1;
    if (e <= r_emax[r])
      for (int q = 0; q < nloc; ++q)
        if (e_rows[e * nloc + q] == r) a = q;
    const double h = a >= 0 ? elh[e] : 1.0;
    double p = h * h, sc = 0.0;
    for (int al = 0; al < nal; ++al, p *= h) {
      const double c = a >= 0 ? coef[(e * ldal + al) * nloc + a] * p : 0.0;
      sc = fma(ca[al], c, sc);
      double hb = 1.0;
      for (int b = 0; b < YM_NB; ++b, hb *= h) at(b, r, s * nal + al) = c * hb;
    }
    if (a >= 0) {
      const double lh = log(h);
      double hb = 1.0;
      for (int b = 0; b < YM_NB; ++b, hb *= h) lt[b] += lh * cb[b] * hb * sc;
    }
  }
  for (int b = 0; b < YM_NB; ++b) LtR[r * YM_NB + b] = lt[b];
}

// Tb[b][g + n_el - 1 + TFRONT][al] = m2u[g + n_el - 1][al][b] (al < da1, zero-padded to ZST
// columns, zero rows outside the table)
__global__ void ystage_mma_prep_table(int64_t n_el, int da1, int64_t n_tab, const double* m2u,
                                      double* Tb) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= YM_NB * n_tab * YM_ZST) return;
  const int al = (int)(k % YM_ZST);
  const int64_t g = (k / YM_ZST) % n_tab - YM_TFRONT;
  const int b = (int)(k / (YM_ZST * n_tab));
  Tb[k] = (g >= 0 && g < 2 * n_el - 1 && al < da1) ? m2u[(g * da1 + al) * YM_NB + b] : 0.0;
}

// vsum[c][b] = sum_{(f,b') in inc(c)} v_f[b][b']
__global__ void ystage_mma_prep_cols(int64_t n_cols, int wc, const int64_t* c_el,
                                     const int64_t* c_loc, const double* v, double* vsum) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  for (int b = 0; b < YM_NB; ++b) {
    double s = 0.0;
    for (int w = 0; w < wc; ++w) {
      const int64_t f = c_el[c * wc + w];
      if (f >= 0) s += v[f * (YM_NB * YM_NB) + b * YM_NB + (int)c_loc[c * wc + w]];
    }
    vsum[c * YM_NB + b] = s;
  }
}

}  // namespace wq

using namespace wq;

extern "C" {

int wq_ystage_mma_prep(int64_t n_rows, int64_t n_cols, int64_t n_el, int nal, int nloc, int wc,
                       const int64_t* e_rows, const int64_t* r_emin, const int64_t* r_emax,
                       const int64_t* c_el, const int64_t* c_loc, const double* coef, int ldal,
                       const double* v, const double* elh, const double* m2u, int da1,
                       const double* ca, const double* cb, double* Cr, double* LtR,
                       double* vsum, double* Tb, int64_t n_tab, void* stream) {
  if (n_rows <= 0 || n_cols <= 0 || n_el <= 0 || (nal != 17 && nal != 5) || nloc < 1 ||
      nloc > 8 || wc < 1 || !e_rows || !r_emin || !r_emax || !c_el || !c_loc || !coef ||
      ldal < nal || !v || !elh || !ca || !cb || !Cr || !LtR || !vsum ||
      (Tb && (!m2u || da1 < 1 || da1 > YM_ZST || n_tab < 2 * n_el - 1 + YM_ZR + YM_TFRONT))) {
    set_error("wq_ystage_mma_prep: bad arguments");
    return WQ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int kp = (YM_NS * nal + 3) / 4 * 4;
  ystage_mma_prep_rows<<<ceil_div(n_rows + 7, 128), 128, 0, st>>>(n_rows, nal, kp, nloc, e_rows,
                                                                r_emin, r_emax, coef, ldal, elh,
                                                                ca, cb, Cr, LtR);
  ystage_mma_prep_cols<<<ceil_div(n_cols, 128), 128, 0, st>>>(n_cols, wc, c_el, c_loc, v, vsum);
  if (Tb)
    ystage_mma_prep_table<<<ceil_div(YM_NB * n_tab * YM_ZST, 256), 256, 0, st>>>(n_el, da1, n_tab,
                                                                                m2u, Tb);
  return check_launch("wq_ystage_mma_prep");
}

int wq_ystage_mma(int64_t n_rows, int64_t n_cols, int64_t n_el, int nal, int wc,
                  const int64_t* r_emin, const int64_t* c_el, const int64_t* c_loc,
                  const int64_t* c_emin, const int64_t* c_emax, const double* v,
                  const double* Cr, const double* LtR, const double* vsum, const double* Tb,
                  int64_t n_tab, const int* row_ko, const int* col_ko, double* out, int64_t ldo,
                  int64_t row0, int64_t row1, int sym, void* stream) {
  if (n_rows <= 0 || n_cols <= 0 || (nal != 17 && nal != 5) || wc < 1 || !r_emin || !c_el ||
      !c_loc || !c_emin || !c_emax || !v || !Cr || !LtR || !vsum || !Tb || !row_ko ||
      !col_ko || !out || row0 < 0 || row0 % YM_T != 0 || row1 > n_rows || row1 <= row0 ||
      wc > YM_WCM || ldo < row1 - row0 || n_tab < 2 * n_el - 1 + YM_ZR + YM_TFRONT) {
    set_error("wq_ystage_mma: bad arguments");
    return WQ_EINVAL;
  }
  YmArgs A{n_cols, n_el, wc, r_emin, c_el, c_loc, c_emin, c_emax, v, Cr, LtR, vsum, Tb, n_tab,
           row_ko, col_ko, out, ldo, row0, row0, sym};
  dim3 grid((unsigned)(n_cols / YM_T), (unsigned)((row1 - row0) / YM_T));
  if (grid.x == 0 || grid.y == 0) return WQ_OK;
  cudaStream_t st = (cudaStream_t)stream;
#define WQ_YM_LAUNCH(NA)                                                                         \
  {                                                                                              \
    const size_t smem = (size_t)YmCfg<NA>::SMEM * 8;                                             \
    cudaFuncSetAttribute(ystage_mma_kernel<NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                         (int)smem);                                                             \
    ystage_mma_kernel<NA><<<grid, YM_THREADS, smem, st>>>(A, (n_rows + 7) / 8 * 8);              \
  }
  if (nal == 17) WQ_YM_LAUNCH(17) else WQ_YM_LAUNCH(5)
#undef WQ_YM_LAUNCH
  return check_launch("wq_ystage_mma");
}

}  // extern "C"
