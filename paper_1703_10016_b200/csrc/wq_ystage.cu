// Graded open meshes, lattice part: Theta^T and D straight from the gap
// table, without per-pair blocks in HBM.
//
// Elements split into a lattice class L (width h0 to 2e-11, centres on the
// h0 grid; every C5 element outside the 60 graded ones at each end) and the
// rest G.  For an outer lattice element e the reference's unit-table recipe
// applies to every lattice partner f (quadrature.py:441-504, 497-500):
//   M(e,f) = h_e^(a+b+2) (M'[k_f - k_e] + ln h_e c_a c_b),
// and partners f in G read precomputed moments MgC[g(f)][e] (wq_gen_moments).
// With C the row functions' element coefficients (u for Theta, v for D):
//   Y[r][f][b] = sum_{(e,a) in inc(r), e in L} sum_al C_e[al][a] M(e,f)[al][b]
//   Out[c][r]  = sum_{(f,b) in inc(c)} sum_be Y[r][f][be] v_f[be][b]
// (Out = Theta^T for r = coarse functions, D for r = fine functions; D is
// symmetric and stored as D[c][r]).  Outer elements in G go through the
// per-pair block route (wq_general.cu) and are accumulated afterwards.
// One CTA = TR row functions x TC column functions; the table rows it needs,
// the rows' scaled coefficients and Y live in shared memory.  Deterministic.
#include "wq_common.cuh"
#include "wq_log.cuh"

namespace wq {

constexpr int YS_TR = 16;       // row functions per CTA (two groups of 8)
constexpr int YS_TC = 64;       // column functions per CTA
constexpr int YS_RPT = 4;      // tile rows per thread
constexpr int YS_THREADS = 64 * (YS_TR / YS_RPT);   // (inner element lane, row group)
constexpr int YS_NB = 5;        // d + 1 (p = 4)
constexpr int YS_MAXLOC = 8;    // local functions per element (p + 1 <= 8)
constexpr int64_t YS_NOT_LATTICE = INT64_MIN;

__device__ __forceinline__ void ys_cp8(void* smem_dst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc));
}
__device__ __forceinline__ void ys_cp_wait() { asm volatile("cp.async.wait_all;\n" ::); }

struct YsArgs {
  int64_t n_rows, n_cols, n_el;
  int nal;                    // outer polynomial slots (P + 1 for Theta, d + 1 for D)
  int nloc;                   // local functions per element on the row side (p + 1)
  int wc;                     // column incidence width
  const int64_t* e_rows;      // (n_el, nloc) row function of local index a on element e
  const int64_t* r_emin;      // (n_rows) first / last element of supp(r)
  const int64_t* r_emax;
  const int64_t* c_el;        // (n_cols, wc) element of incidence, -1 = none
  const int64_t* c_loc;
  const int64_t* c_emin;
  const int64_t* c_emax;
  const double* coef;         // (n_el, ldal, nloc) row coefficients C_e[al][a]
  int ldal;                   // slot count of coef (>= nal)
  const double* v;            // (n_el, NB, NB) column coefficients v_f[be][b]
  const double* elh;          // (n_el)
  const int64_t* kidx;        // (n_el) lattice index or YS_NOT_LATTICE
  const int* gidx;            // (n_el) index in G or -1
  const double* m2u;          // (2 n_el - 1, da + 1, NB) unit gap table
  int da1;                    // da + 1 (table slot count)
  const double* mgc;          // (n_g, n_el, da + 1, NB) moments of (e in L, f in G) or NULL
  const double* ca;           // (da + 1) c_a
  const double* cb;           // (NB) c_b
  int64_t fspan, espan;       // max element span of a column / row tile (host)
  double* out;                // (n_cols, ldo) output, Out[c][r - out_row0]
  int64_t ldo;
  int64_t t0;                 // first row tile (rows t0*YS_TR ...)
  int64_t out_row0;
  int64_t row_end;            // rows >= row_end are not produced
  int sym;                    // rows == cols (D): only tiles meeting c >= r; mirrored after
  const int* row_ko;          // 64-row tiles from out_row0 (wq_ystage_mma) or NULL
  const int* col_ko;          // 64-column tiles; tiles with row_ko == col_ko != NOT_PURE are
                              // done on the tensor cores by wq_ystage_mma
  const int* tiles;           // (n, 2) (row tile, column tile) of the CTAs to run, or NULL: the
                              // full grid (every CTA holds ~110 KB of shared memory, so a grid
                              // of mostly skipped tiles costs a launch slot per skipped tile)
};

// Thread (inner element f, group of YS_RPT tile rows): Y in registers.
template <int NB, bool SYM>
__global__ void __launch_bounds__(YS_THREADS)
ystage_kernel(YsArgs A) {
  extern __shared__ double sm[];
  const int bx = A.tiles ? A.tiles[2 * blockIdx.x] : (int)blockIdx.x;
  const int by = A.tiles ? A.tiles[2 * blockIdx.x + 1] : (int)blockIdx.y;
  const int64_t R0 = (A.t0 + bx) * YS_TR, C0 = (int64_t)by * YS_TC;
  const int nr = (int)min((int64_t)YS_TR, A.row_end - R0);
  const int nc = (int)min((int64_t)YS_TC, A.n_cols - C0);
  if (SYM && C0 + nc - 1 < R0) return;   // strictly below the diagonal: mirrored later
  if (A.row_ko) {
    const int ko = A.row_ko[(R0 - A.out_row0) / 64];
    if (ko != INT32_MIN && A.col_ko[by] == ko) return;   // wq_ystage_mma's tile
  }
  const int64_t ea = A.r_emin[R0], eb = A.r_emax[R0 + nr - 1];
  const int64_t fa = A.c_emin[C0], fb = A.c_emax[C0 + nc - 1];
  const int ne = (int)(eb - ea + 1), nf = (int)(fb - fa + 1);
  const int nal = A.nal, da1 = A.da1, nloc = A.nloc;
  double* Cs = sm;                                          // [espan][nal][nloc] C h^(al+2)
  double* Lt = Cs + A.espan * nal * nloc;                   // [espan][nloc][NB] ln h c_b h^b sum c_al C
  double* Hb = Lt + A.espan * nloc * NB;                    // [espan][NB] h_e^b
  double* Mr = Hb + A.espan * NB;                           // [nf + ne - 1][nal][NB] table rows
  double* Ys = Mr + (A.fspan + A.espan - 1) * nal * NB;     // [YS_TR][fspan][NB]
  int* Rw = reinterpret_cast<int*>(Ys + YS_TR * A.fspan * NB);  // [espan][nloc] tile-relative row
  const int tid = threadIdx.x;

  for (int k = tid; k < ne * nloc; k += YS_THREADS) {
    const int el = k / nloc, a = k - el * nloc;
    const int64_t e = ea + el;
    Rw[k] = (int)(A.e_rows[e * nloc + a] - R0);   // tile-relative row (may lie outside)
    const double h = A.elh[e];
    double p = h * h, sc = 0.0;
    for (int al = 0; al < nal; ++al, p *= h) {
      const double c = A.coef[(e * A.ldal + al) * nloc + a] * p;
      Cs[(el * nal + al) * nloc + a] = c;
      sc = fma(A.ca[al], c, sc);
    }
    const double lh = log(h);
    double hb = 1.0;
    for (int b = 0; b < NB; ++b, hb *= h) Lt[(el * nloc + a) * NB + b] = lh * A.cb[b] * hb * sc;
  }
  for (int k = tid; k < ne * NB; k += YS_THREADS) {
    const int el = k / NB, b = k - el * NB;
    const double h = A.elh[ea + el];
    double p = 1.0;
    for (int i = 0; i < b; ++i) p *= h;
    Hb[k] = p;
  }
  // table rows for the index gaps f - e in [fa - eb, fb - ea]
  const int nrow = nf + ne - 1;
  const int64_t g0 = fa - eb;
  // the window is one contiguous run of the table: asynchronous copies keep
  // many loads in flight per thread
  for (int k = tid; k < nrow * nal * NB; k += YS_THREADS) {
    const int row = k / (nal * NB), rem = k - row * nal * NB;
    const int64_t g = g0 + row;
    if (g > -A.n_el && g < A.n_el) ys_cp8(Mr + k, A.m2u + ((g + A.n_el - 1) * da1) * NB + rem);
    else Mr[k] = 0.0;
  }
  ys_cp_wait();
  __syncthreads();

  // phase 1: thread (f, row group of YS_RPT consecutive rows) accumulates
  // Y[r][f][0..NB) in registers; every table value feeds the group's rows.
  // An element's nloc local functions are consecutive rows r0 .. r0+nloc-1
  // (host-checked); lanes run over f, warps over row groups, so which group
  // rows meet element e is warp-uniform.
  {
    const int q = tid / 64;                  // row group
    for (int fl = tid % 64; fl < nf; fl += 64) {
      const int64_t f = fa + fl;
      const int64_t kf = A.kidx[f];
      const int gf = A.gidx[f];
      double y[YS_RPT][NB];
#pragma unroll
      for (int j = 0; j < YS_RPT; ++j)
#pragma unroll
        for (int b = 0; b < NB; ++b) y[j][b] = 0.0;
      for (int el = 0; el < ne; ++el) {
        const int a0 = YS_RPT * q - Rw[el * nloc];   // local index of the group's first row
        if (a0 >= nloc || a0 + YS_RPT <= 0) continue;
        const int64_t e = ea + el;
        const int64_t ke = A.kidx[e];
        if (ke == YS_NOT_LATTICE) continue;   // outer element in G: block route
        double t[YS_RPT][NB];
#pragma unroll
        for (int j = 0; j < YS_RPT; ++j)
#pragma unroll
          for (int b = 0; b < NB; ++b) t[j][b] = 0.0;
        const double* cs = Cs + el * nal * nloc;
        const bool table = kf != YS_NOT_LATTICE;
        const double* __restrict__ Mg = nullptr;
        const double* Ms = nullptr;
        if (table) {
          const int64_t g = kf - ke;
          const int64_t wrow = g - g0;
          if (wrow >= 0 && wrow < nrow && g == f - e) Ms = Mr + wrow * nal * NB;
          else Mg = A.m2u + ((g + A.n_el - 1) * da1) * NB;   // off the staged window
        } else {
          if (!A.mgc) continue;
          Mg = A.mgc + ((int64_t)gf * A.n_el + e) * da1 * NB;   // G partner, scaled moments
        }
        for (int al = 0; al < nal; ++al) {
          double m[NB];
          if (Ms) {
#pragma unroll
            for (int b = 0; b < NB; ++b) m[b] = Ms[al * NB + b];
          } else {
#pragma unroll
            for (int b = 0; b < NB; ++b) m[b] = __ldg(Mg + al * NB + b);
          }
#pragma unroll
          for (int j = 0; j < YS_RPT; ++j) {
            const int a = a0 + j;
            if (a >= 0 && a < nloc) {
              const double c = table ? cs[al * nloc + a] : A.coef[(e * A.ldal + al) * nloc + a];
#pragma unroll
              for (int b = 0; b < NB; ++b) t[j][b] = fma(c, m[b], t[j][b]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < YS_RPT; ++j) {
          const int a = a0 + j;
          if (a >= 0 && a < nloc)
#pragma unroll
            for (int b = 0; b < NB; ++b)
              y[j][b] += table ? fma(Hb[el * NB + b], t[j][b], Lt[(el * nloc + a) * NB + b])
                               : t[j][b];
        }
      }
#pragma unroll
      for (int j = 0; j < YS_RPT; ++j)
#pragma unroll
        for (int b = 0; b < NB; ++b) Ys[((YS_RPT * q + j) * A.fspan + fl) * NB + b] = y[j][b];
    }
  }
  __syncthreads();

  // phase 2: Out[c][r] = sum_{(f,b) in inc(c)} sum_be Y[r][f][be] v_f[be][b]
  for (int k = tid; k < nc * YS_TR; k += YS_THREADS) {
    const int cl = k / YS_TR, r = k - cl * YS_TR;
    if (r >= nr) continue;
    const int64_t c = C0 + cl;
    double acc = 0.0;
    for (int s = 0; s < A.wc; ++s) {
      const int64_t f = A.c_el[c * A.wc + s];
      if (f < 0) continue;
      const int b = (int)A.c_loc[c * A.wc + s];
      const double* yr = Ys + (r * A.fspan + (f - fa)) * NB;
      const double* vf = A.v + f * NB * NB;
#pragma unroll
      for (int be = 0; be < NB; ++be) acc = fma(yr[be], vf[be * NB + b], acc);
    }
    A.out[c * A.ldo + R0 + r - A.out_row0] = acc;
  }
}

// out[j][i] = out[i][j] for i > j (copy the lower triangle onto the upper one),
// 32 x 32 tiles through shared memory
// (row_ko / col_ko given: the 64 x 64 tiles wq_ystage_mma owns -- storage row tile bi / 2 pure as
// a column tile, column tile bj / 2 pure as a row tile, equal offsets -- are already mirrored)
__global__ void mirror_lower_kernel(double* out, int64_t n, int64_t ld, const int* row_ko,
                                    const int* col_ko, int n_full) {
  __shared__ double t[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;   // source tile rows bi, cols bj
  if (bj > bi) return;
  if (row_ko && bi / 2 < n_full && bj / 2 < n_full) {
    const int ko = row_ko[bj / 2];
    if (ko != INT32_MIN && col_ko[bi / 2] == ko) return;
  }
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bi * 32 + y, c = bj * 32 + tx;
    t[y][tx] = (r < n && c < n) ? out[r * ld + c] : 0.0;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bj * 32 + y, c = bi * 32 + tx;   // destination (upper) entry (r, c) = src (c, r)
    if (r < n && c < n && c > r) out[r * ld + c] = t[tx][y];
  }
}

// out[c][r] = out[r][c] for c > r (copy the upper triangle onto the lower one)
__global__ void mirror_upper_kernel(double* out, int64_t n, int64_t ld) {
  __shared__ double t[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;   // source tile rows bi, cols bj (bj >= bi)
  if (bj < bi) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bi * 32 + y, c = bj * 32 + tx;
    t[y][tx] = (r < n && c < n) ? out[r * ld + c] : 0.0;
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int64_t r = bj * 32 + y, c = bi * 32 + tx;   // destination (lower) entry (r, c) = src (c, r)
    if (r < n && c < n && r > c) out[r * ld + c] = t[tx][y];
  }
}

// Far moments of pairs (e in L, f in G), physical: thread per outer element,
// tensor Gauss by separation tier (30 / 16 / 12 as wq_gen_pair_blocks).
constexpr int GM_THREADS = 64;

__global__ void __launch_bounds__(GM_THREADS)
gen_moments_far_kernel(int64_t n_el, int da1, int nb, const int64_t* glist, const int* gidx,
                       const double* elh, const double* elm, const int64_t* near_lo,
                       const int64_t* near_cnt, const double* gx, const double* gw,
                       double* mgc) {
  extern __shared__ double sh[];
  __shared__ double2 lntab[64];                   // accurate-table ln (wq_log.cuh)
  for (int q = threadIdx.x; q < 128; q += GM_THREADS) reinterpret_cast<double*>(lntab)[q] = kTang64[q];
  __syncthreads();
  const int j = blockIdx.y;                       // index in G
  const int64_t f = glist[j];
  const int64_t e = (int64_t)blockIdx.x * GM_THREADS + threadIdx.x;
  if (e >= n_el || gidx[e] >= 0) return;          // outer in G: block route
  int64_t k = f - near_lo[e];
  if (k < 0) k += n_el;
  if (k < near_cnt[e]) return;                    // touching: near kernel
  double* M = sh + threadIdx.x * da1 * nb;
  for (int s = 0; s < da1 * nb; ++s) M[s] = 0.0;
  const double he = elh[e], hf = elh[f];
  const double delta = elm[e] - elm[f];
  const double sep = fabs(delta) - 0.5 * (he + hf);
  const double hm = fmax(he, hf);
  const int t0 = sep < 2.0 * hm ? 0 : (sep < 8.0 * hm ? 30 : 46);
  const int ng = sep < 2.0 * hm ? 30 : (sep < 8.0 * hm ? 16 : 12);
  for (int g = 0; g < ng; ++g) {
    const double x = he * gx[t0 + g], wxg = he * gw[t0 + g];
    double t[8];
    for (int b = 0; b < nb; ++b) t[b] = 0.0;
    for (int h = 0; h < ng; ++h) {
      const double y = hf * gx[t0 + h], wy = hf * gw[t0 + h];
      const double kv = 2.0 * half_ln64t(fabs(y - x - delta), lntab);   // separated: y - x - delta != 0
      double w = wy * kv;
      for (int b = 0; b < nb; ++b) {
        t[b] += w;
        w *= y;
      }
    }
    double wa = wxg;
    for (int a = 0; a < da1; ++a) {
      for (int b = 0; b < nb; ++b) M[a * nb + b] = fma(wa, t[b], M[a * nb + b]);
      wa *= x;
    }
  }
  double* out = mgc + ((int64_t)j * n_el + e) * da1 * nb;
  for (int s = 0; s < da1 * nb; ++s) out[s] = M[s];
}

// The same with the DA1 x NB moments of a pair in registers (the kernel above keeps them in
// shared memory: 2 x 85 shared accesses per outer Gauss node and pair made it shared-memory
// bound) and the inner element's weighted powers w_h y_h^b staged once per CTA (f is fixed per
// CTA), so a pair costs ng^2 ln + ng^2 NB + ng DA1 NB FMAs and no per-thread shared traffic.
template <int DA1, int NB>
__global__ void __launch_bounds__(GM_THREADS)
gen_moments_far_reg_kernel(int64_t n_el, const int64_t* glist, const int* gidx, const double* elh,
                           const double* elm, const int64_t* near_lo, const int64_t* near_cnt,
                           const double* gx, const double* gw, double* mgc) {
  constexpr int NG = 30 + 16 + 12;
  __shared__ double2 lntab[64];                   // accurate-table ln (wq_log.cuh)
  __shared__ double Wt[NG][NB];                   // h_f w_h (h_f x_h)^b
  __shared__ double Yt[NG], Gx[NG], Gw[NG];
  const int j = blockIdx.y;                       // index in G
  const int64_t f = glist[j];
  const double hf = elh[f];
  for (int q = threadIdx.x; q < 128; q += GM_THREADS) reinterpret_cast<double*>(lntab)[q] = kTang64[q];
  for (int h = threadIdx.x; h < NG; h += GM_THREADS) {
    const double y = hf * gx[h];
    double w = hf * gw[h];
    Gx[h] = gx[h];
    Gw[h] = gw[h];
    Yt[h] = y;
#pragma unroll
    for (int b = 0; b < NB; ++b, w *= y) Wt[h][b] = w;
  }
  __syncthreads();
  const int64_t e = (int64_t)blockIdx.x * GM_THREADS + threadIdx.x;
  if (e >= n_el || gidx[e] >= 0) return;          // outer in G: block route
  int64_t k = f - near_lo[e];
  if (k < 0) k += n_el;
  if (k < near_cnt[e]) return;                    // touching: near kernel
  const double he = elh[e];
  const double delta = elm[e] - elm[f];
  const double sep = fabs(delta) - 0.5 * (he + hf);
  const double hm = fmax(he, hf);
  const int t0 = sep < 2.0 * hm ? 0 : (sep < 8.0 * hm ? 30 : 46);
  const int ng = sep < 2.0 * hm ? 30 : (sep < 8.0 * hm ? 16 : 12);
  double M[DA1][NB];
#pragma unroll
  for (int a = 0; a < DA1; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) M[a][b] = 0.0;
  for (int g = 0; g < ng; ++g) {
    const double x = he * Gx[t0 + g];
    const double base = -x - delta;
    double t[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) t[b] = 0.0;
#pragma unroll 4
    for (int h = 0; h < ng; ++h) {
      // separated pair: y - x - delta != 0
      const double kv = 2.0 * half_ln64t(fabs(Yt[t0 + h] + base), lntab);
#pragma unroll
      for (int b = 0; b < NB; ++b) t[b] = fma(Wt[t0 + h][b], kv, t[b]);
    }
    double wa = he * Gw[t0 + g];
#pragma unroll
    for (int a = 0; a < DA1; ++a) {
#pragma unroll
      for (int b = 0; b < NB; ++b) M[a][b] = fma(wa, t[b], M[a][b]);
      wa *= x;
    }
  }
  double* out = mgc + ((int64_t)j * n_el + e) * (DA1 * NB);
#pragma unroll
  for (int a = 0; a < DA1; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) out[a * NB + b] = M[a][b];
}

}  // namespace wq

using namespace wq;

extern "C" {

int wq_ystage(int64_t n_rows, int64_t n_cols, int64_t n_el, int nal, int nloc, int wc,
              const int64_t* e_rows, const int64_t* r_emin, const int64_t* r_emax,
              const int64_t* c_el, const int64_t* c_loc, const int64_t* c_emin,
              const int64_t* c_emax, const double* coef, int ldal, const double* v, int nb,
              const double* elh, const int64_t* kidx, const int* gidx, const double* m2u,
              int da1, const double* mgc, const double* ca, const double* cb, int64_t fspan,
              int64_t espan, double* out, int64_t ldo, int64_t row0, int64_t row1,
              int sym_d, const int* row_ko, const int* col_ko, const int* tiles,
              int64_t n_tiles, void* stream) {
  if (n_rows <= 0 || n_cols <= 0 || nal < 1 || nal > da1 || nloc < 1 || nloc > YS_MAXLOC ||
      (tiles && n_tiles < 0) ||
      wc < 1 || !e_rows || !r_emin || !r_emax || !c_el || !c_loc || !c_emin || !c_emax ||
      !coef || ldal < nal || !v || nb != YS_NB || !elh || !kidx || !gidx || !m2u || !ca || !cb ||
      fspan < 1 || espan < 1 || !out || row0 < 0 || row1 > n_rows || row1 <= row0 ||
      row0 % YS_TR != 0 || ldo < row1 - row0 || (row_ko && (row0 % 64 != 0 || !col_ko))) {
    set_error("wq_ystage: bad arguments (column degree must be %d)", YS_NB - 1);
    return WQ_EINVAL;
  }
  YsArgs A{n_rows, n_cols, n_el, nal, nloc, wc, e_rows, r_emin, r_emax, c_el, c_loc, c_emin,
           c_emax, coef, ldal, v, elh, kidx, gidx, m2u, da1, mgc, ca, cb, fspan, espan, out,
           ldo, row0 / YS_TR, row0, row1, 0, row_ko, col_ko, tiles};
  const size_t smem = (size_t)(espan * nal * nloc + espan * nloc * YS_NB + espan * YS_NB +
                               (fspan + espan - 1) * nal * YS_NB + YS_TR * fspan * YS_NB) * 8 +
                      (size_t)espan * nloc * 4;
  if (smem > 227 * 1024) {
    set_error("wq_ystage: tile needs %zu B of shared memory", smem);
    return WQ_EUNSUPPORTED;
  }
  cudaFuncSetAttribute(ystage_kernel<YS_NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  cudaFuncSetAttribute(ystage_kernel<YS_NB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  // rows [row0, row1): the last tile may run past row1 (up to n_rows) -- clip
  const int64_t nrow_tiles = ceil_div(row1 - row0, YS_TR);
  dim3 grid((unsigned)nrow_tiles, ceil_div(n_cols, YS_TC));
  if (tiles) {
    if (n_tiles == 0) return WQ_OK;
    grid = dim3((unsigned)n_tiles, 1);
  }
  // D (rows == cols, full range): only the storage entries out[c][r], c >= r
  // (the caller completes D and mirrors it, wq_mirror_lower)
  A.sym = n_rows == n_cols && row0 == 0 && row1 == n_rows && sym_d;
  if (A.sym) ystage_kernel<YS_NB, true><<<grid, YS_THREADS, smem, (cudaStream_t)stream>>>(A);
  else ystage_kernel<YS_NB, false><<<grid, YS_THREADS, smem, (cudaStream_t)stream>>>(A);
  return check_launch("wq_ystage");
}

int wq_mirror_lower(double* out, int64_t n, int64_t ld, const int* row_ko, const int* col_ko,
                    void* stream) {
  if (!out || n <= 0 || ld < n || (row_ko != nullptr) != (col_ko != nullptr)) {
    set_error("wq_mirror_lower: bad arguments");
    return WQ_EINVAL;
  }
  dim3 mg(ceil_div(n, 32), ceil_div(n, 32));
  mirror_lower_kernel<<<mg, dim3(32, 8), 0, (cudaStream_t)stream>>>(out, n, ld, row_ko, col_ko,
                                                                      (int)(n / 64));
  return check_launch("wq_mirror_lower");
}

int wq_mirror_upper(double* out, int64_t n, int64_t ld, void* stream) {
  if (!out || n <= 0 || ld < n) {
    set_error("wq_mirror_upper: bad arguments");
    return WQ_EINVAL;
  }
  dim3 mg(ceil_div(n, 32), ceil_div(n, 32));
  mirror_upper_kernel<<<mg, dim3(32, 8), 0, (cudaStream_t)stream>>>(out, n, ld);
  return check_launch("wq_mirror_upper");
}

int wq_gen_moments_far(int64_t n_el, int da1, int nb, int64_t n_g, const int64_t* glist,
                       const int* gidx, const double* elh, const double* elm,
                       const int64_t* near_lo, const int64_t* near_cnt, const double* gx,
                       const double* gw, double* mgc, void* stream) {
  if (n_el <= 0 || n_g <= 0 || da1 < 1 || nb < 1 || nb > 8 || !glist || !gidx || !elh || !elm ||
      !near_lo || !near_cnt || !gx || !gw || !mgc) {
    set_error("wq_gen_moments_far: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(n_el, GM_THREADS), (unsigned)n_g);
  if (da1 == 17 && nb == 5) {   // config 5 (p = 4): moments in registers
    gen_moments_far_reg_kernel<17, 5><<<grid, GM_THREADS, 0, (cudaStream_t)stream>>>(
        n_el, glist, gidx, elh, elm, near_lo, near_cnt, gx, gw, mgc);
    return check_launch("wq_gen_moments_far");
  }
  const size_t smem = (size_t)GM_THREADS * da1 * nb * 8;
  cudaFuncSetAttribute(gen_moments_far_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  gen_moments_far_kernel<<<grid, GM_THREADS, smem, (cudaStream_t)stream>>>(
      n_el, da1, nb, glist, gidx, elh, elm, near_lo, near_cnt, gx, gw, mgc);
  return check_launch("wq_gen_moments_far");
}

}  // extern "C"
