/*
 * wqb200.h -- C-ABI of the B200 (sm_100a, FP64) IgA-SGBEM V-matrix assembly.
 *
 * This is the drop-in boundary beneath the reference's Python entry points in
 * wqbem.assembly (reference: pkg/src/wqbem/assembly.py).  The reference has no
 * FFI of its own; each entry point below names the reference function whose
 * O(N^2) work it replaces (file:line under /root/reference/pkg/src/wqbem/).
 *
 * Conventions
 *   - All buffers are caller-allocated, contiguous DEVICE memory (FP64 values,
 *     int64 indices), row-major.  No torch types cross this boundary.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and performs no host synchronisation.
 *   - Return 0 on success, a negative WQ_E* code on failure; the message is
 *     available from wq_last_error() (thread-local).
 *   - Geometry failures detected on the device (R <= 0 on the kernel grid,
 *     geometry.py:246-247) are OR-ed into *flag (device int); the caller maps
 *     a non-zero flag to GeometryError after synchronising.
 *   - Results are deterministic: no floating-point atomics anywhere.
 */
#ifndef WQB200_H
#define WQB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WQ_OK 0
#define WQ_EINVAL (-1)
#define WQ_ECUDA (-2)
#define WQ_EUNSUPPORTED (-3)

#define WQ_FLAG_R_NONPOSITIVE 1

/* rows/cols per CTA output tile of wq_ik1 / wq_ik2_circ (callers size max_span with it) */
#define WQ_TILE 32

/* K1 parameter-distance modes (geometry.py:127-139) */
#define WQ_K1_TABLE 0        /* 1/p^2 looked up by node-index gap (exactly uniform nodes) */
#define WQ_K1_OPEN 1         /* p = |t - s| */
#define WQ_K1_CLOSED 2       /* p = (L/pi)|sin(pi |t - s| / L)| */

/* Smooth part: nodes, banded rule matrix G = W*J (assembly.py:160) */
typedef struct {
  int64_t n_rows;          /* N: test functions (rows of G)                   */
  int64_t nq;              /* number of shared quadrature nodes               */
  int64_t wg;              /* padded band width of G                          */
  int64_t closed;          /* 1 on closed curves                              */
  int64_t k1_mode;         /* WQ_K1_*                                         */
  double period;           /* L = b - a                                       */
  const double* s;         /* (nq) node parameters                            */
  const double* fx;        /* (nq) f(s) x                                     */
  const double* fy;        /* (nq) f(s) y                                     */
  const double* J;         /* (nq) parametric speed                           */
  const double* invp2;     /* (nq) 1/p^2 per index gap (WQ_K1_TABLE) or NULL   */
  const int64_t* g_start;  /* (N) unwrapped first node of row i (monotone)    */
  const double* g_w;       /* (N, wg) G[i, (g_start[i]+w) mod nq]             */
  int64_t near_k;          /* 0, or K: distinct node pairs closer than eps_diag */
  const double* near_j2;   /* (nq, K): J(mid)^2 of pair (q, q+k+1 mod nq), 0 if */
                           /* not near (geometry.py:237-245); else NULL       */
} wq_smooth_t;

/* Version / identification. */
int wq_version(void);
const char* wq_last_error(void);

/* FP64 pipe probe for the roofline denominator: blocks x 256 threads x
 * iters x 64 DFMA (2 flops each).  out: >= blocks doubles (never written
 * in practice). */
int wq_fp64_peak(int64_t iters, int blocks, double* out, void* stream);

/*
 * IK1 rows/cols block (replaces assemble_ik1, assembly.py:175-183, with the
 * K1 grid of geometry.py:225-248 evaluated in-kernel and never stored):
 *   X[i, j] (+)= sum_q sum_r G[i,q] K1(eta_q, eta_r) G[j,r]
 * for i in [row0,row1), j in [col0,col1); X points at element (row0, col0),
 * leading dimension ldx.  accumulate != 0 adds into X.
 * max_span = max over tiles of the node span (host-computed, see Python).
 * When [row0,row1) == [col0,col1) only tiles on or above the diagonal are
 * evaluated and mirrored (K1 is symmetric).  Distinct node pairs closer than
 * eps_diag take sm->near_j2 (J(mid)^2, geometry.py:237-245).
 */
int wq_ik1(const wq_smooth_t* sm, int64_t row0, int64_t row1, int64_t col0, int64_t col1,
           double* X, int64_t ldx, int accumulate, int64_t max_span, int* flag, void* stream);

/*
 * IK1 for any rule band (irregular starts, widths <= wg <= 16; open, graded,
 * repeated-knot meshes): register sliding windows over per-rule starts, 64 x 64
 * tiles, table-based ln.  tile_row0 < 0: the whole matrix from its upper tile
 * pairs, mirrored; else tile rows [tile_row0, tile_row1) x all columns into X
 * (row tile_row0 * 64 at X).  span64: the largest node span of a 64-row tile
 * (<= 144).  Writes (does not accumulate).
 */
int wq_ik1_band(const wq_smooth_t* sm, int64_t tile_row0, int64_t tile_row1, double* X,
                int64_t ldx, int64_t span64, int* flag, void* stream);

/*
 * Gap-indexed pair log-moment table (replaces uniform_pair_log_moments,
 * quadrature.py:472-504 / _unit_pair_stack :441-469):
 *   far gaps: 30x30 Gauss of ln|v-u-delta| (quadrature.py:413-438);
 *   |gap| <= 1: analytic closed-form unit table supplied by the host
 *   (near_unit, 3 x (da+1) x (db+1), rows keff = -1, 0, +1);
 *   closed meshes: + periodic correction ln|sinc| (quadrature.py:253-256,464-467);
 *   then M_h = h^(2+a+b) (M_1 + ln h c_a c_b).
 * n_gap = nel (closed, index (f-e) mod nel) or 2 nel - 1 (open, f-e+nel-1).
 * gx, gw: Gauss nodes/weights on (-1/2, 1/2), n_gauss of them; n_gauss = 58 passes
 * the rules of orders 30 | 16 | 12 concatenated and selects 16 points at |gap| = 2,
 * 12 beyond (converged to rounding), 30 for the periodic term of near gaps.
 */
int wq_pair_table(int64_t nel, int closed, int da, int db, double h,
                  const double* near_unit, const double* gx, const double* gw, int n_gauss,
                  const double* ca, const double* cb, double* m2, void* stream);

/* Closed uniform simple-knot meshes: circulant log-part tables.
 *   Z[g][al]  = sum_b sum_be M2[(g-b) mod n][al][be] v0[be][b]
 *   dd[k]     = sum_a sum_{al<=d} v0[al][a] Z[(k+a) mod n][al]       (D circulant)
 *   Zp[g][al] = sum_{|k|<=K} Z[(g+k) mod n][al] hinv[k]               (Theta H^{-1})
 *   ff        = hinv * dd * hinv                                       (H^{-1} D H^{-1})
 * hinv_taps has 2K+1 entries, hinv_taps[K+k] = H^{-1}[0,k].
 * work: n doubles of scratch.
 */
int wq_circ_tables(int64_t n, int da, int db, const double* m2, const double* v0,
                   const double* hinv_taps, int64_t K, double* Zp, double* ff, double* work,
                   double* Zwork, void* stream);

/* Log-part description shared by the circulant path and the general path. */
typedef struct {
  int64_t n_rows;          /* N  (coarse functions)                          */
  int64_t n_fine;          /* N_E (fine functions) = n_el on closed meshes    */
  int64_t da;              /* P = p + 12 (row polynomial degree)              */
  int64_t tu;              /* elements per coarse support (p+1)*nref          */
  int64_t ws;              /* padded band width of S columns                  */
  const int64_t* e_start;  /* (N) unwrapped first fine element of supp(B_i)   */
  const double* U;         /* (N, tu, da+1): u[e_start+a][:, a_i]             */
  const int64_t* s_start;  /* (N) unwrapped first fine row of column i of S   */
  const double* s_w;       /* (N, ws): S[s_start+t, i]                        */
} wq_logpart_t;

/*
 * Circulant log part (replaces assemble_ik2, assembly.py:186-245, X-form):
 *   Phi[m,i] = 2 sum_a sum_al U[i][a][al] Zp[(m - e_start[i] - a) mod n][al]
 *              - sum_t S[s_start[i]+t, i] ff[(m - s_start[i] - t) mod n]
 *   X[i, j] (+)= sum_t S[s_start[j]+t, j] Phi[s_start[j]+t, i]
 * i in [row0,row1), j in [col0,col1); X points at (row0,col0), ld ldx.
 */
int wq_ik2_circ(const wq_logpart_t* lp, const double* Zp, const double* ff,
                int64_t row0, int64_t row1, int64_t col0, int64_t col1,
                double* X, int64_t ldx, int accumulate, void* stream);

/* General (open-mesh) log part, dense intermediates. */
typedef struct {
  int64_t n_rows, n_fine, n_el, n_gap, da, db, closed;
  int64_t wu;                 /* max (e,a) incidences per coarse function      */
  int64_t wv;                 /* max (f,b) incidences per fine function        */
  const int64_t* u_el;        /* (N, wu)  element of incidence, -1 = none      */
  const int64_t* u_loc;       /* (N, wu)  local index a                         */
  const int64_t* v_el;        /* (N_E, wv)                                      */
  const int64_t* v_loc;       /* (N_E, wv)                                      */
  const double* u;            /* (n_el, da+1, pu+1) coefficients               */
  int64_t pu;                 /* coarse degree p                                */
  const double* v;            /* (n_el, db+1, db+1)                             */
  const double* m2;           /* (n_gap, da+1, db+1)                            */
} wq_pairs_t;

/* Theta^T (N_E x N) and D (N_E x N_E) by element-pair gathers (assembly.py:215-232). */
int wq_theta_t(const wq_pairs_t* pp, double* thetaT, void* stream);
/* Columns [row0, row1) of Theta^T only (a rank's row block): thetaT[l * ld + i - row0]. */
int wq_theta_t_rows(const wq_pairs_t* pp, int64_t row0, int64_t row1, double* thetaT, int64_t ld,
                    void* stream);
int wq_dmat(const wq_pairs_t* pp, double* D, void* stream);

/* Segmented variant (parallel over columns x row segments of seg rows): a segment
 * starts from the state reconstructed from the k0 preceding rows run from zero
 * (exact to rounding once k0 exceeds the decay length of L^{-1}); state: workspace
 * of (ceil(n/seg) - 1) * bw * ncols doubles. */
int wq_band_solve_seg(int64_t n, int64_t bw, const double* Lb, double* X, int64_t ncols,
                      int64_t ldx, int64_t seg, int64_t k0, double* state, void* stream);

/* In-place banded SPD solve on every column of X (n x ncols, ld ldx):
 * X <- H^{-1} X with H = L L^T, Lb[k][j] = L[k][k-j], j = 0..bw. */
int wq_band_solve_cols(int64_t n, int64_t bw, const double* Lb, double* X, int64_t ncols,
                       int64_t ldx, void* stream);

/* Cyclic (seam-coupled) banded SPD solve on every column: X <- H^{-1} X with the
 * arrow Cholesky factor: Lb (m x (bw+1), m = n - bw) of the leading band, L21
 * (bw x m, row-major) = A21 L11^{-T}, L22 (bw x bw, row-major lower) of the Schur
 * complement.  bw <= 16. */
int wq_cyc_solve_cols(int64_t n, int64_t bw, const double* Lb, const double* L21,
                      const double* L22, double* X, int64_t ncols, int64_t ldx, void* stream);

/* out = in^T for an (rows x cols) matrix. */
int wq_transpose(const double* in, int64_t rows, int64_t cols, double* out, void* stream);

/* Phi[m][i] = alpha * P[m][i] - sum_t F[m][(s_start[i]+t) mod nf] S[s_start[i]+t, i]  (in place on P) */
int wq_gather_fs(const wq_logpart_t* lp, double alpha, const double* F, double* P, void* stream);

/* The same with F = Y^T read straight from Y (N_E x N_E; no transposed copy):
 *   Phi[m][i] = alpha * P[m][i] - sum_t Y[(s_start[i]+t) mod nf][m] S[s_start[i]+t, i].
 * max_span >= s_start[min(i0 + 63, N - 1)] - s_start[i0] + ws for every 64-column block i0
 * (the Y rows one block stages); WQ_EUNSUPPORTED when they do not fit in shared memory. */
int wq_gather_yts(const wq_logpart_t* lp, double alpha, const double* Y, double* P,
                  int64_t max_span, void* stream);

/* X[j][i] (+)= sum_t S[s_start[j]+t, j] Phi[(s_start[j]+t) mod nf][i], all i, j rows [row0,row1). */
int wq_add_st_phi(const wq_logpart_t* lp, const double* Phi, int64_t row0, int64_t row1,
                  double* X, int64_t ldx, int accumulate, void* stream);

/* wq_add_st_phi over all rows followed by wq_symmetrize, fused (X2^T is never written):
 *   A = alpha (X + X^T), X[j][i] = (X_in[j][i] if accumulate) + sum_t S[s_start[j]+t, j] Phi[(s_start[j]+t) mod nf][i],
 * in place on the N x N matrix X (leading dimension N). */
int wq_st_phi_sym(const wq_logpart_t* lp, const double* Phi, double* X, double alpha,
                  int accumulate, void* stream);

/*
 * v2 circulant pipeline (closed uniform simple-knot meshes, nref = 1), tiles of
 * WQ_FTILE rows over the upper-triangle tile pairs (I <= J):
 *
 * wq_ik1_sym: X[I-tile, J-tile] = IK1(I,J) for I <= J only (IK1 is symmetric).
 *   max_span: max node span of WQ_FTILE consecutive rules.
 * wq_zext:   Zext[g] = [Z'[g][0..nA-1], 0 .., ff[g] at column nApad, 0 ..]
 *   (row stride zstride).
 * wq_x2_pairs: log part on the FP64 tensor cores + fused epilogue, in place:
 *   A(I,J) = alpha (w_ik1 IK1(I,J) + X2(I,J) + X2(J,I)^T), A(J,I) = A(I,J)^T,
 *   reading IK1(I,J) from X (written by wq_ik1_sym), where
 *   X2[i,j] = sum_t S[j-d+t, j] Phi[j-d+t, i],
 *   Phi[m,i] = sum_K Uext[i][K] Zrow(m-i, K),  Uext[i] = [2U[i][a][al] (a*nApad+al),
 *   -S[i-d+t, i] (tu*nApad + t), 0 ..] (ktot columns).  Uext is passed in DMMA
 *   B-fragment order: element (i, K) at ((i/8 * ktot/4 + K/4) * 8 + i%8) * 4 + K%4,
 *   rows padded with zeros to a multiple of 8 (ceil(N/8) * 8 * ktot doubles), so each
 *   warp reads one contiguous 256-byte fragment per row group and k-step.
 *   alpha = -1/(4 pi), w_ik1 = 2 gives A; alpha = 1/2 gives M = (X + X^T)/2.
 */
#define WQ_FTILE 64
int wq_ik1_sym(const wq_smooth_t* sm, double* X, int64_t ldx, int64_t max_span, int* flag,
               void* stream);
int wq_zext(int64_t n, int nA, int nApad, int zstride, const double* Zp, const double* ff,
            double* Zext, void* stream);
int wq_x2_pairs(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                const double* Uext, const double* Zext, const double* s_w, double alpha,
                double w_ik1, double* X, int64_t ldx, void* stream);

/*
 * Row-block variants for multi-GPU sharding: tile rows
 * [tile_row0, tile_row1) (units of WQ_FTILE rows), all columns, no symmetry
 * exploitation; Xrows points at global row tile_row0 * WQ_FTILE.
 *   wq_ik1_rows: Xrows = IK1[rows, :]
 *   wq_x2_rows:  Xrows = alpha (w_ik1 Xrows + X2[rows, :])   (unsymmetrised X)
 * After an all-gather of X, wq_symmetrize(X, N, -1/(4 pi)) gives A.
 */
int wq_ik1_rows(const wq_smooth_t* sm, int64_t tile_row0, int64_t tile_row1, double* Xrows,
                int64_t ldx, int* flag, void* stream);
int wq_x2_rows(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
               const double* Uext, const double* Zext, const double* s_w, double alpha,
               double w_ik1, int64_t tile_row0, int64_t tile_row1, double* Xrows, int64_t ldx,
               void* stream);

/*
 * Pair-range variants of the symmetric pipeline: upper-triangle tile pairs
 * [pair0, pair1) in row-major triangular order (row bi holds nb - bi pairs,
 * nb = ceil(N / WQ_FTILE)).  x2 pairs of a range read IK1 of the same range,
 * so consecutive ranges can be pipelined on two streams.
 */
int wq_ik1_pairs(const wq_smooth_t* sm, int64_t pair0, int64_t pair1, double* X, int64_t ldx,
                 int* flag, void* stream);
int wq_x2_pairs_range(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                      const double* Uext, const double* Zext, const double* s_w, double alpha,
                      double w_ik1, int64_t pair0, int64_t pair1, double* X, int64_t ldx,
                      void* stream);

/* The same kernels over an explicit list of upper-triangle tile-pair indices
 * (device array, npairs entries): the single-process multi-GPU host path gives
 * each GPU the pairs that complete its own rows. */
int wq_ik1_pair_list(const wq_smooth_t* sm, const int64_t* plist, int64_t npairs, double* X,
                     int64_t ldx, int* flag, void* stream);
int wq_x2_pair_list(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                    const double* Uext, const double* Zext, const double* s_w, double alpha,
                    double w_ik1, const int64_t* plist, int64_t npairs, double* X, int64_t ldx,
                    void* stream);

/* Self-test hooks (unit tests): the IK1 kernel's table 0.5*ln vs libdevice; one DMMA 8x8x4. */
int wq_selftest_log(int64_t n, const double* x, double* out_fast, double* out_ref, void* stream);
int wq_selftest_dmma(const double* A, const double* B, double* C, void* stream);

/* Epilogue (assembly.py:262-271): A = alpha * (X + X^T), in place, n x n. */
int wq_symmetrize(double* X, int64_t n, double alpha, void* stream);

/* max |X| and max |X - X^T| (symmetry defect numerator), out[0..1]. */
int wq_absmax_defect(const double* X, int64_t n, double* out, void* stream);

/* Weighted RHS (assembly.py:312-319): b[i] = sum_w G[i, w] g[(g_start[i]+w) mod nq]. */
int wq_b1w(const wq_smooth_t* sm, const double* g, double* b, void* stream);

/*
 * Double-layer RHS inner integral (assemble_b2, assembly.py:322-343; Kbar_points,
 * geometry.py:250-280): inner[s] = sum_t Kbar(s,t) wg[t] over M = 16 n_el per-element
 * Gauss points; f, f' at the points, kdiag = C^2 curvature limit on s == t.
 */
int wq_b2_inner(int64_t M, const double* fx, const double* fy, const double* tx, const double* ty,
                const double* wg, const double* kdiag, double* inner, void* stream);

/*
 * Non-uniform meshes (graded / any multiplicity; BASELINE config 5).  Replaces
 * the gap-indexed pair table of _pair_log_moments (quadrature.py:441-504), which
 * raises ConstructionError on graded meshes (quadrature.py:489-491), and the
 * Theta / D accumulation of _log_part (assembly.py:206-236), per element pair.
 *
 * wq_gen_pair_blocks: for outer elements e in [e0, e1) and every inner element f,
 *   WT[f][a'][b'][e-e0] = (U_e^T M(e,f) V_f)[a'][b']   ((pu+1) x (db+1); pu == db)
 *   WD[f][a'][b'][e-e0] = (V_e^T M(e,f) V_f)[a'][b']   ((db+1) x (db+1))
 * (chunk-minor, leading dimension ldc >= e1 - e0).  elh/elm: element widths /
 * midpoints; u (n_el, da+1, pu+1), v (n_el, db+1, db+1) centred-monomial
 * coefficients (splines.py:427-472; u times the fitted J).  Near (touching /
 * overlapping) pairs of e are f = near_lo[e] + k (mod n_el), k < near_cnt[e] <=
 * max_near: equal widths take near_unit (3 x (da+1) x (db+1), the closed-form unit
 * entries at dl = -1, 0, 1, quadrature.py:372-410, 458), unequal widths a Duffy
 * split with the packed rules `touch` (x16 w16 x30 w30 Gauss-Legendre on (0,1),
 * xl14 wl14 for the weight -ln x).  Other pairs: with m2u (wq_pair_table's UNIT
 * gap table, h = 1, n_gap = 2 n_el - 1; open meshes) equal widths (1e-10
 * relative) at integer offsets read M' and scale it by their own width,
 * M = h^(a+b+2) (M' + ln h c_a c_b) -- the reference's recipe
 * (quadrature.py:497-500); the rest tensor Gauss (quadrature.py:413-438), gx/gw
 * = orders 30 | 16 | 12 on (-1/2, 1/2) concatenated (30 below two larger widths
 * of separation, 16 below eight, 12 beyond).  tile_flag (device ints,
 * n_el x ceil((e1-e0)/64), required with m2u) is scratch marking the tiles that
 * still need Gauss.  ca/cb: centred monomial integrals (da+1), (db+1); closed != 0
 * adds the periodic gap term (quadrature.py:459-468) for period `period`.
 */
int wq_gen_pair_blocks(int64_t n_el, int64_t e0, int64_t e1, int da, int db, int pu, int closed,
                       double period, const double* elh, const double* elm, const double* u,
                       const double* v, const int64_t* near_lo, const int64_t* near_cnt,
                       int max_near, const double* near_unit, const double* touch,
                       const double* gx, const double* gw, const double* m2u,
                       const double* ca, const double* cb, double* wt, double* wd,
                       int64_t ldc, int* tile_flag, void* stream);

/* thetaT[l][i - i_off] (leading dimension ldt) += sum over the chunk's incidences
 * of i (u_el/u_loc, width wu) and all incidences of l (v_el/v_loc, width wv, -1
 * padded) of WT blocks; i in [i0, i1). */
int wq_gen_gather_theta(int64_t n_rows, int64_t n_fine, int64_t e0, int64_t e1, int64_t ldc,
                        int64_t i0, int64_t i1, int wu, int wv, int nU, int nB,
                        const int64_t* u_el, const int64_t* u_loc, const int64_t* v_el,
                        const int64_t* v_loc, const double* wt, double* thetaT, int64_t ldt,
                        int64_t i_off, void* stream);

/* D (symmetric, N_E x N_E) += chunk contributions of WD blocks for rows l in
 * [l0, l1), stored transposed (D[m][l]) so the stores are coalesced. */
int wq_gen_gather_d(int64_t n_fine, int64_t e0, int64_t e1, int64_t ldc, int64_t l0, int64_t l1,
                    int wv, int nB, const int64_t* v_el, const int64_t* v_loc, const double* wd,
                    double* D, void* stream);

/* Moments mode of the near-pair kernel: physical moments M(e,f) ((da+1) x (db+1))
 * of touching pairs with e lattice (gidx[e] < 0) and f in G (gidx[f] >= 0) into
 * mgc[gidx[f]][e] (n_g x n_el x (da+1) x (db+1)); other arguments as wq_gen_pair_blocks. */
int wq_gen_near_moments(int64_t n_el, int da, int db, const double* elh, const double* elm,
                        const int64_t* near_lo, const int64_t* near_cnt, int max_near,
                        const double* near_unit, const double* touch, const double* ca,
                        const double* cb, const int* gidx, double* mgc, void* stream);

/* Far physical moments of the pairs (e lattice, f = glist[j] in G) into mgc[j][e]
 * (tensor Gauss, orders 30 | 16 | 12 by separation; gx/gw as wq_gen_pair_blocks);
 * touching pairs are left to wq_gen_near_moments. */
int wq_gen_moments_far(int64_t n_el, int da1, int nb, int64_t n_g, const int64_t* glist,
                       const int* gidx, const double* elh, const double* elm,
                       const int64_t* near_lo, const int64_t* near_cnt, const double* gx,
                       const double* gw, double* mgc, void* stream);

/*
 * Lattice route for graded open meshes (replaces the Theta / D accumulation of
 * _log_part, assembly.py:206-236, for outer elements on the width-h0 lattice):
 *   Y[r][f][b] = sum_{(e,a) in inc(r), kidx[e] valid} sum_al coef_e[al][a] M(e,f)[al][b]
 *   out[c][r]  = sum_{(f,b) in inc(c)} sum_be Y[r][f][be] v_f[be][b]
 * M(e,f) = h_e^(al+b+2) (m2u[k_f - k_e] + ln h_e c_al c_b) for lattice f (the
 * reference's unit-table recipe, quadrature.py:497-500), mgc[gidx[f]][e] otherwise.
 * Rows: coarse functions (coef = u, nal = da+1) -> out = Theta^T; or fine functions
 * (coef = v, nal = db+1) -> out = D (symmetric, stored D[c][r]).  e_rows (n_el x nloc):
 * the row function of local index a on element e (splines.py:427-472 cols).  r_emin/r_emax,
 * c_emin/c_emax: first / last element of each support; espan / fspan: the largest
 * element span of a 16-row / 64-column tile.  Rows [row0, row1) only (row0 a
 * multiple of 16), written to out[c][r - row0].  sym_d != 0 with rows == columns over
 * the full range (D): only the storage entries out[c][r] with c >= r are produced
 * (complete them, then wq_mirror_lower; D is symmetric).  Column degree nb - 1 = 4.  Writes
 * (does not accumulate) out; outer elements off the lattice are added afterwards by
 * the block route (wq_gen_pair_blocks + gathers).  tiles (optional): n_tiles pairs
 * (16-row tile from row0, 64-column tile) to run instead of the full tile grid -- with
 * row_ko / col_ko most tiles belong to wq_ystage_mma and a CTA holds ~110 KB of shared
 * memory, so launching only the others removes a launch slot per skipped tile.
 */
int wq_ystage(int64_t n_rows, int64_t n_cols, int64_t n_el, int nal, int nloc, int wc,
              const int64_t* e_rows, const int64_t* r_emin, const int64_t* r_emax,
              const int64_t* c_el, const int64_t* c_loc, const int64_t* c_emin,
              const int64_t* c_emax, const double* coef, int ldal, const double* v, int nb,
              const double* elh, const int64_t* kidx, const int* gidx, const double* m2u,
              int da1, const double* mgc, const double* ca, const double* cb, int64_t fspan,
              int64_t espan, double* out, int64_t ldo, int64_t row0, int64_t row1,
              int sym_d, const int* row_ko, const int* col_ko, const int* tiles,
              int64_t n_tiles, void* stream);

/*
 * Tensor-core lattice tiles of wq_ystage (same Theta^T / D entries): for 64-row tiles
 * (from row0, a multiple of 64) and 64-column tiles whose elements all lie on one lattice
 * run -- row_ko[t] == col_ko[u] != INT32_MIN, the common offset k_e - e -- the inner sum is
 * a GEMM in skewed coordinates u = f - e_r on DMMA (m8n8k4.f64), one per column power b,
 * with the Toeplitz A operand from Tb (table slices) and the B operand from Cr; the column
 * contraction and the ln h term (LtR, vsum) follow in shared memory.  wq_ystage given the
 * same row_ko / col_ko skips exactly these tiles.  nal: 17 (Theta, p = 4) or 5 (D).
 * n_tab >= 2 n_el - 1 + 160.
 * wq_ystage_mma_prep fills Cr (5 x ceil8(n_rows) x kp doubles, kp = 5 nal rounded up to 4,
 * rows padded with zeros to a multiple of 8, each power b in DMMA B-fragment order
 * [row / 8][k / 4][row % 8][k % 4]: one contiguous 256-byte fragment per row group and k-step), LtR
 * (n_rows x 5), vsum (n_cols x 5) and, when Tb is not NULL, Tb (5 x n_tab x 20) from m2u.
 * wq_ystage_mma_tiles fills the per-column-tile tables the kernel's contraction warps fetch
 * by TMA a tile ahead: CvT (n_cols / 64 x 64 x 5 x 5 doubles: v_f[b][b'] of the w-th
 * incidence (f, b') of each column) and CiT (n_cols / 64 x 64 x 5 ints: f minus the first
 * element of the tile's first column, or -1).
 */
int wq_ystage_mma_prep(int64_t n_rows, int64_t n_cols, int64_t n_el, int nal, int nloc, int wc,
                       const int64_t* e_rows, const int64_t* r_emin, const int64_t* r_emax,
                       const int64_t* c_el, const int64_t* c_loc, const double* coef, int ldal,
                       const double* v, const double* elh, const double* m2u, int da1,
                       const double* ca, const double* cb, double* Cr, double* LtR,
                       double* vsum, double* Tb, int64_t n_tab, void* stream);
int wq_ystage_mma_tiles(int64_t n_cols, int wc, const int64_t* c_el, const int64_t* c_loc,
                        const int64_t* c_emin, const double* v, double* CvT, int* CiT,
                        void* stream);
int wq_ystage_mma(int64_t n_rows, int64_t n_cols, int64_t n_el, int nal, int wc,
                  const int64_t* r_emin, const int64_t* c_el, const int64_t* c_loc,
                  const int64_t* c_emin, const int64_t* c_emax, const double* v,
                  const double* Cr, const double* LtR, const double* vsum, const double* CvT,
                  const int* CiT, const double* Tb,
                  int64_t n_tab, const int* row_ko, const int* col_ko, double* out, int64_t ldo,
                  int64_t row0, int64_t row1, int sym, void* stream);

/* out[j][i] = out[i][j] for i > j (n x n, leading dimension ld).  With row_ko / col_ko (both or
 * neither; the arrays given to wq_ystage_mma with sym = 1) the 64 x 64 tiles that kernel owns
 * are skipped: it writes their mirrors itself. */
int wq_mirror_lower(double* out, int64_t n, int64_t ld, const int* row_ko, const int* col_ko,
                    void* stream);
/* out[c][r] = out[r][c] for c > r: the upper triangle copied onto the lower one (the
 * symmetric multi-GPU path: each rank assembles the upper tile pairs of its rows). */
int wq_mirror_upper(double* out, int64_t n, int64_t ld, void* stream);

/* Packed upper-triangle blocks (multi-GPU all-gather of the symmetric
 * assembly, half the bytes of full rows): the upper tiles A(I, J), J >= I, of
 * the 64 x 64 tile pairs [p0, p1) in row-by-row pair order, tile-major
 * (pair p at (p - p0) * 4096 doubles, row-major 64 x 64; entries outside an
 * edge tile unused).
 * wq_pack_pairs: A (ld) -> packed.
 * wq_unpack_pairs: packed -> A(I, J) and its transpose into A(J, I). */
int wq_pack_pairs(const double* A, int64_t n, int64_t ld, int64_t p0, int64_t p1, double* packed,
                  void* stream);
int wq_unpack_pairs(const double* packed, int64_t n, int64_t p0, int64_t p1, double* A, int64_t ld,
                    void* stream);

/* General-path row blocks (multi-GPU; X-form, assembly.py:233-245):
 * wq_gather_fs_rows: P[m][i - i0] = alpha P[m][i - i0] - sum_t F[m][s_i + t] S_i[t],
 *   i in [i0, i1), P with leading dimension ldp (the block's Theta^T columns);
 * wq_phi_s_rows: X[i - i0][j] (+)= sum_t S_j[t] PhiT[i - i0][s_j + t] for all j
 *   (PhiT = the block's Phi columns transposed, (i1 - i0) x N_E). */
int wq_gather_fs_rows(const wq_logpart_t* lp, double alpha, const double* F, double* P,
                      int64_t i0, int64_t i1, int64_t ldp, void* stream);
int wq_phi_s_rows(const wq_logpart_t* lp, const double* PhiT, int64_t i0, int64_t i1, double* X,
                  int64_t ldx, int accumulate, void* stream);

/* wq_band_solve_cols with the last bw (<= 8) solution values kept in registers:
 * one load and one store per row and column (large n). */
int wq_band_solve_win(int64_t n, int64_t bw, const double* Lb, double* X, int64_t ncols,
                      int64_t ldx, void* stream);

#ifdef __cplusplus
}
#endif
#endif
