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
// One tile = 64 row functions x 64 column functions, 8 GEMM warps x 8 row functions and 8
// contraction warps; the table window of each b arrives by a 1-D TMA bulk copy.  Each warp
// runs only the skew blocks it needs (64 functions span 48-61 elements with 25 % repeated
// knots: 7-9 of the 10 blocks the host-checked maxima allow).  Deterministic.
// Citations: quadrature.py:441-504 (unit-table recipe, scaling 497-500),
// assembly.py:186-245 (Theta / D assembly).
#include <type_traits>

#include "wq_async.cuh"
#include "wq_common.cuh"

namespace wq {

constexpr int YM_T = 64;             // row / column functions per tile
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
  const double* CvT;       // (column tiles, T, WCM, NB) v_f[b][b'] of the tile's column incidences
  const int* CiT;          // (column tiles, T, WCM) element offset f - fa of the incidence, or -1
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
};

// ---------------------------------------------------------------------------
// ystage_ws_kernel: warp-specialised and persistent (the scheme of x2ws_kernel, wq_fast.cu):
// one CTA of 16 warps per SM walks the pure tiles.  Warps 0-7 (the GEMM group)
// run the skewed DMMA loops of the 5 column powers of tile after tile back to back and
// scatter each Y_b into one of two Phs buffers; warps 8-15 (the contraction group) contract
// it with the columns' v (CUDA cores, registers), keep Out[c][r] in registers across the 5
// powers and write the finished tile while the GEMM group is already on the next one.
// "Phase" = one (tile, power): buffers ph & 1, mbarrier parity (ph >> 1) & 1; wfull (table
// window landed, TMA), pfull / pempty (Y_b written / contracted).  The first contraction
// thread requests the window of phase ph + 2 as soon as pfull of phase ph completes (every
// GEMM warp has then read that window buffer).  (Round 2 replaced a one-tile-per-CTA kernel
// with CTA-wide barriers between the GEMM, scatter and contraction of every power; this one is
// bit-identical to it and 2.5 % faster.)
// ---------------------------------------------------------------------------
#ifdef WQ_YS_TIMELINE
// tools build only: clock stamps of the phases of one tile (the 20th of every CTA):
// slots 0-24 GEMM group (5 per phase), 32-63 contraction group
__device__ long long* g_ys_tl = nullptr;
#define YW_TL(slot)                                                                       \
  do {                                                                                    \
    if (tcount == 20 && (threadIdx.x & 255) == 0 && g_ys_tl)                              \
      g_ys_tl[(int64_t)blockIdx.x * 64 + (slot)] = clock64();                             \
  } while (0)
#else
#define YW_TL(slot) do {} while (0)
#endif

constexpr int YW_THREADS = 512;
constexpr int YW_BAR_E = 1;   // named barrier of the contraction group

template <int NAL>
struct YwCfg {
  using C = YmCfg<NAL>;
  static constexpr int ZW = YM_ZR * YM_ZST;
  static constexpr int PH = YM_T * YM_PST;
  static constexpr int CV = YM_T * YM_WCM * YM_NB;
  static constexpr int OS = YM_T * (YM_T + 1);
  static constexpr int LT = YM_T * YM_NB;          // LtR rows / vsum rows of a tile
  // Zsm[2] | Phs[2] | Cv[2] | Os | LtR[2] | vsum[2] | 8 mbarriers | Ci[2] (ints)
  static constexpr int SMEM = 2 * ZW + 2 * PH + 2 * CV + OS + 4 * LT + 8 + YM_T * YM_WCM;
};

template <int NAL>
__global__ void __launch_bounds__(YW_THREADS, 1)
ystage_ws_kernel(YmArgs A, int64_t nrp, int ntx, int nty) {
  using C = YmCfg<NAL>;
  using W = YwCfg<NAL>;
  extern __shared__ double sm[];
  double* Zsm = sm;                               // [2][ZR][ZST]
  double* Phs = Zsm + 2 * W::ZW;                  // [2][T][PST]
  double* Cv = Phs + 2 * W::PH;                   // [2][T c][WCM][NB]
  double* Os = Cv + 2 * W::CV;                    // [T c][T + 1]
  double* Lts = Os + W::OS;                       // [2][T r][NB]: LtR rows of the tile
  double* Vss = Lts + 2 * W::LT;                  // [2][T c][NB]: vsum rows of the tile
  uint64_t* wfull = reinterpret_cast<uint64_t*>(Vss + 2 * W::LT);
  uint64_t* pfull = wfull + 2;
  uint64_t* pempty = wfull + 4;
  uint64_t* efull = wfull + 6;                    // [2] tile tables landed (TMA)
  int* Ci = reinterpret_cast<int*>(wfull + 8);    // [2][T c][WCM]
  const int tid = threadIdx.x;
  const int64_t ntiles = (int64_t)ntx * nty;
  // the tiles this kernel owns, in the order every thread of the CTA walks them
  auto pure = [&](int64_t q) {
    const int ct = (int)(q % ntx), rt = (int)(q / ntx);
    const int ko = A.row_ko[rt];
    if (ko == YM_NOT_PURE || A.col_ko[ct] != ko) return false;
    const int64_t R0 = A.row0 + (int64_t)rt * YM_T, C0 = (int64_t)ct * YM_T;
    return !(A.sym && C0 + YM_T - 1 < R0);        // strictly below the diagonal: mirrored later
  };
  auto next_pure = [&](int64_t q) {               // first owned pure tile at or after q
    while (q < ntiles && !pure(q)) q += gridDim.x;
    return q;
  };
  // table rows of tile q's window (power 0)
  auto window_src = [&](int64_t q) {
    const int ct = (int)(q % ntx), rt = (int)(q / ntx);
    const int64_t R0 = A.row0 + (int64_t)rt * YM_T, C0 = (int64_t)ct * YM_T;
    const int64_t gbase = A.c_emin[C0] - A.r_emin[R0 + YM_T - 1] - (YM_NS - 1);
    return A.Tb + (gbase + A.n_el - 1 + YM_TFRONT) * YM_ZST;
  };
  if (tid == 0)
    for (int b = 0; b < 2; ++b) {
      mbar_init(wfull + b, 1);
      mbar_init(pfull + b, 8);
      mbar_init(pempty + b, 8);
      mbar_init(efull + b, 1);
    }
  fence_proxy_async();
  __syncthreads();
  const int64_t q0 = next_pure(blockIdx.x);
  if (q0 >= ntiles) return;

  if (tid < 256) {
    // ------------------------------ GEMM group ------------------------------
    const int lane = tid & 31, warp = tid >> 5;
    const int rl = lane >> 2, cl = lane & 3;
    // per-tile quantities of this warp (loaded a tile ahead: the dependent global loads would
    // otherwise stall every GEMM warp at each tile start)
    struct Tile {
      const double* brow0;   // B fragments of the warp's row group, power 0
      int zoff, fspan, nkb, ef0, ef1;
    };
    auto load_tile = [&](int64_t q) {
      Tile t;
      const int ct = (int)(q % ntx), rt = (int)(q / ntx);
      const int64_t R0 = A.row0 + (int64_t)rt * YM_T, C0 = (int64_t)ct * YM_T;
      const int64_t fa = A.c_emin[C0];
      const int64_t emax_all = A.r_emin[R0 + YM_T - 1];
      const int64_t emax_w = A.r_emin[R0 + 8 * warp + 7];
      t.zoff = (int)(emax_all - emax_w) + (YM_NS - 1);
      t.fspan = (int)(A.c_emax[C0 + YM_T - 1] - fa) + 1;
      t.nkb = min(YM_NKB, (t.fspan + (int)(emax_w - A.r_emin[R0 + 8 * warp]) + 7) >> 3);
      t.brow0 = A.Cr + ((R0 + 8 * warp) / 8) * (C::NSTEPS * 32) + lane;
      t.ef0 = (int)(A.r_emin[R0 + 8 * warp + 2 * cl] - emax_w);
      t.ef1 = (int)(A.r_emin[R0 + 8 * warp + 2 * cl + 1] - emax_w);
      return t;
    };
    unsigned ph = 0;
    Tile cur = load_tile(q0);
    // the B-fragment ring runs on across phases and tiles: slot (SHIFT + t) % PF holds k-step t
    // of the current phase, refilled with the next phase's k-steps as soon as it is consumed
    // (5 NSTEPS is a multiple of PF, so every tile starts at shift 0)
    static_assert((YM_NB * C::NSTEPS) % C::PF == 0, "ystage ws: B-fragment ring does not close");
    double bq[C::PF];
#pragma unroll
    for (int t = 0; t < C::PF; ++t) bq[t] = __ldg(cur.brow0 + 32 * t);
    int tcount = 0;
    for (int64_t q = q0; q < ntiles; ++tcount) {
      const int64_t qn = next_pure(q + gridDim.x);
      const Tile nxt = qn < ntiles ? load_tile(qn) : cur;
      auto phase = [&](auto bc) {
        constexpr int b = decltype(bc)::value;
        YW_TL(5 * b);
        constexpr int SHIFT = (b * C::NSTEPS) % C::PF;
        const int buf = ph & 1;
        const unsigned par = (ph >> 1) & 1;
        const double* zb = Zsm + buf * W::ZW;
        const double* __restrict__ brow = cur.brow0 + (int64_t)b * nrp * C::KP;
        // the next phase's fragments: the next power of this tile, or power 0 of the next tile
        const double* __restrict__ bnext = b + 1 < YM_NB ? brow + nrp * C::KP : nxt.brow0;
        mbar_wait(wfull + buf, par);
        YW_TL(5 * b + 1);
        double acc[YM_NKB][2];
#pragma unroll
        for (int kb = 0; kb < YM_NKB; ++kb) acc[kb][0] = acc[kb][1] = 0.0;
        const double* zl = zb + (cur.zoff + rl) * YM_ZST;
        auto gemm = [&](auto nk) {
          constexpr int NK = decltype(nk)::value;
#pragma unroll
          for (int t = 0; t < C::NSTEPS; ++t) {
            const int kk = min(4 * t + cl, YM_NS * NAL - 1);
            const int s = kk / NAL, al = kk - s * NAL;
            const double bfrag = bq[(SHIFT + t) % C::PF];
            bq[(SHIFT + t) % C::PF] = t + C::PF < C::NSTEPS ? __ldg(brow + 32 * (t + C::PF))
                                                            : __ldg(bnext + 32 * (t + C::PF - C::NSTEPS));
            const double* z = zl - s * YM_ZST + al;
#pragma unroll
            for (int kb = 0; kb < NK; ++kb) dmma(acc[kb][0], acc[kb][1], z[8 * kb * YM_ZST], bfrag);
          }
        };
        if (cur.nkb <= YM_NKB - 3) gemm(std::integral_constant<int, YM_NKB - 3>());
        else if (cur.nkb == YM_NKB - 2) gemm(std::integral_constant<int, YM_NKB - 2>());
        else if (cur.nkb == YM_NKB - 1) gemm(std::integral_constant<int, YM_NKB - 1>());
        else gemm(std::integral_constant<int, YM_NKB>());
        YW_TL(5 * b + 2);
        // Phs[buf] is free once the contraction group has used it two phases ago
        if (ph >= 2) mbar_wait(pempty + buf, par ^ 1);
        YW_TL(5 * b + 3);
        double* P = Phs + buf * W::PH;
#pragma unroll
        for (int kb = 0; kb < YM_NKB; ++kb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int fl = 8 * kb + rl + (e ? cur.ef1 : cur.ef0);
            if (fl >= 0 && fl < cur.fspan) P[(8 * warp + 2 * cl + e) * YM_PST + fl] = acc[kb][e];
          }
        warp_arrive(pfull + buf);
        YW_TL(5 * b + 4);
        ++ph;
      };
      phase(std::integral_constant<int, 0>());
      phase(std::integral_constant<int, 1>());
      phase(std::integral_constant<int, 2>());
      phase(std::integral_constant<int, 3>());
      phase(std::integral_constant<int, 4>());
      cur = nxt;
      q = qn;
    }
  } else {
    // --------------------------- contraction group ---------------------------
    const int et = tid - 256;
    const int ocol = et & 63, rg = et >> 6;
    unsigned ph = 0;
    // TMA request of tile q's tables into buffers cb: column incidences (CvT / CiT, per
    // column tile), the tile's LtR rows and vsum rows
    auto tables = [&](int64_t q, int cb) {
      const int ct = (int)(q % ntx), rt = (int)(q / ntx);
      const int64_t R0 = A.row0 + (int64_t)rt * YM_T, C0 = (int64_t)ct * YM_T;
      constexpr unsigned BCV = W::CV * 8, BCI = YM_T * YM_WCM * 4, BLT = W::LT * 8;
      mbar_arrive_expect_tx(efull + cb, BCV + BCI + 2 * BLT);
      bulk_g2s(Cv + cb * W::CV, A.CvT + (int64_t)ct * W::CV, BCV, efull + cb);
      bulk_g2s(Ci + cb * (YM_T * YM_WCM), A.CiT + (int64_t)ct * (YM_T * YM_WCM), BCI, efull + cb);
      bulk_g2s(Lts + cb * W::LT, A.LtR + R0 * YM_NB, BLT, efull + cb);
      bulk_g2s(Vss + cb * W::LT, A.vsum + C0 * YM_NB, BLT, efull + cb);
    };
    if (et == 0) {
      for (int b = 0; b < 2; ++b) {
        mbar_arrive_expect_tx(wfull + b, W::ZW * 8);
        bulk_g2s(Zsm + b * W::ZW, window_src(q0) + (int64_t)b * A.n_tab * YM_ZST, W::ZW * 8, wfull + b);
      }
      tables(q0, 0);
    }
    int tcount = 0;
    for (int64_t q = q0; q < ntiles; ++tcount) {
      YW_TL(32);
      const int64_t qn = next_pure(q + gridDim.x);
      const int ct = (int)(q % ntx), rt = (int)(q / ntx);
      const int64_t R0 = A.row0 + (int64_t)rt * YM_T, C0 = (int64_t)ct * YM_T;
      YW_TL(33);
      // the tile's tables (column incidences, LtR rows, vsum rows) were requested a tile ago;
      // request the next tile's into the other buffers (all contraction threads left them at
      // the end of the previous tile)
      const int cbuf = tcount & 1;
      if (et == 0 && qn < ntiles) tables(qn, cbuf ^ 1);
      mbar_wait(efull + cbuf, (unsigned)((tcount >> 1) & 1));
      const int* ci = Ci + cbuf * (YM_T * YM_WCM);
      const double* cvs = Cv + cbuf * W::CV;
      // Out[c][r] for this thread's column c and rows r = 16 rg + i; starts from the ln h term
      double out[YM_T / 4];
      {
        const double* vs = Vss + cbuf * W::LT + ocol * YM_NB;
        const double* lt = Lts + cbuf * W::LT + 16 * rg * YM_NB;
#pragma unroll
        for (int i = 0; i < YM_T / 4; ++i) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < YM_NB; ++b) s = fma(lt[i * YM_NB + b], vs[b], s);
          out[i] = s;
        }
      }
      YW_TL(34);
      YW_TL(35);
      const double* nsrc = qn < ntiles ? window_src(qn) : nullptr;
      const double* csrc = window_src(q);
      for (int b = 0; b < YM_NB; ++b, ++ph) {
        const int buf = ph & 1;
        const unsigned par = (ph >> 1) & 1;
        YW_TL(36 + 3 * b);
        mbar_wait(pfull + buf, par);
        YW_TL(37 + 3 * b);
        // every GEMM warp has read window buf: request the window of phase ph + 2 into it
        if (et == 0) {
          const double* src = b + 2 < YM_NB ? csrc + (int64_t)(b + 2) * A.n_tab * YM_ZST
                                            : (nsrc ? nsrc + (int64_t)(b + 2 - YM_NB) * A.n_tab * YM_ZST
                                                    : nullptr);
          if (src) {
            mbar_arrive_expect_tx(wfull + buf, W::ZW * 8);
            bulk_g2s(Zsm + buf * W::ZW, src, W::ZW * 8, wfull + buf);
          }
        }
        int fi[YM_WCM];
        double cv[YM_WCM];
#pragma unroll
        for (int w = 0; w < YM_WCM; ++w) {
          const int f = ci[ocol * YM_WCM + w];
          fi[w] = f >= 0 ? f : 0;
          cv[w] = f >= 0 ? cvs[(ocol * YM_WCM + w) * YM_NB + b] : 0.0;
        }
        const double* phs = Phs + buf * W::PH + 16 * rg * YM_PST;
#pragma unroll
        for (int i = 0; i < YM_T / 4; ++i)
#pragma unroll
          for (int w = 0; w < YM_WCM; ++w) out[i] = fma(phs[i * YM_PST + fi[w]], cv[w], out[i]);
        warp_arrive(pempty + buf);
        YW_TL(38 + 3 * b);
      }
      // Out[c][r] through shared memory so that 64 consecutive r of a column leave together
#pragma unroll
      for (int i = 0; i < YM_T / 4; ++i) Os[ocol * (YM_T + 1) + 16 * rg + i] = out[i];
      named_sync(YW_BAR_E, 256);
      if (!A.sym) {
        for (int k = et; k < YM_T * YM_T; k += 256) {
          const int c = k >> 6, r = k & 63;
          A.out[(C0 + c) * A.ldo + R0 + r - A.out_row0] = Os[c * (YM_T + 1) + r];
        }
      } else {
        // symmetric output (D): the storage entry (C0 + c, R0 + r), c >= r on the diagonal
        // tile, and its mirror (R0 + r, C0 + c) -- both coalesced; no mirror pass over these
        // tiles afterwards (wq_mirror_lower skips them)
        const bool diag = C0 == R0;
        for (int k = et; k < YM_T * YM_T; k += 256) {
          const int c = k >> 6, r = k & 63;
          if (!diag || c >= r) A.out[(C0 + c) * A.ldo + R0 + r] = Os[c * (YM_T + 1) + r];
        }
        for (int k = et; k < YM_T * YM_T; k += 256) {
          const int r = k >> 6, c = k & 63;
          if (!diag || c > r) A.out[(R0 + r) * A.ldo + C0 + c] = Os[c * (YM_T + 1) + r];
        }
      }
      named_sync(YW_BAR_E, 256);                  // Os and this tile's tables free
      YW_TL(52);
      q = qn;
    }
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

// CvT[ct][c][w][b] = v_f[b][b'] and CiT[ct][c][w] = f - fa of the w-th incidence (f, b') of
// column C0 + c, fa = the first element of the tile's first column (-1 / 0 where none): the
// contraction group's per-tile tables, one TMA copy each
__global__ void ystage_mma_prep_tiles(int64_t n_tiles, int wc, const int64_t* c_el,
                                      const int64_t* c_loc, const int64_t* c_emin, const double* v,
                                      double* CvT, int* CiT) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_tiles * YM_T * YM_WCM) return;
  const int64_t ct = k / (YM_T * YM_WCM);
  const int kk = (int)(k - ct * (YM_T * YM_WCM));
  const int c = kk / YM_WCM, w = kk - c * YM_WCM;
  const int64_t cc = ct * YM_T + c;
  const int64_t f = w < wc ? c_el[cc * wc + w] : -1;
  CiT[k] = f >= 0 ? (int)(f - c_emin[ct * YM_T]) : -1;
  const int bp = f >= 0 ? (int)c_loc[cc * wc + w] : 0;
  for (int b = 0; b < YM_NB; ++b)
    CvT[k * YM_NB + b] = f >= 0 ? v[f * (YM_NB * YM_NB) + b * YM_NB + bp] : 0.0;
}

}  // namespace wq

using namespace wq;

extern "C" {

#ifdef WQ_YS_TIMELINE
int wq_debug_ys_timeline(long long* buf) {
  cudaError_t e = cudaMemcpyToSymbol(g_ys_tl, &buf, sizeof(buf));
  return e == cudaSuccess ? WQ_OK : WQ_ECUDA;
}
#endif

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

int wq_ystage_mma_tiles(int64_t n_cols, int wc, const int64_t* c_el, const int64_t* c_loc,
                        const int64_t* c_emin, const double* v, double* CvT, int* CiT,
                        void* stream) {
  if (n_cols < 1 || wc < 1 || wc > YM_WCM || !c_el || !c_loc || !c_emin || !v) {
    set_error("wq_ystage_mma_tiles: bad arguments");
    return WQ_EINVAL;
  }
  const int64_t nt = n_cols / YM_T;
  if (nt == 0) return WQ_OK;          // no full column tile: wq_ystage_mma has no tile either
  if (!CvT || !CiT) {
    set_error("wq_ystage_mma_tiles: missing output tables");
    return WQ_EINVAL;
  }
  ystage_mma_prep_tiles<<<ceil_div(nt * YM_T * YM_WCM, 256), 256, 0, (cudaStream_t)stream>>>(
      nt, wc, c_el, c_loc, c_emin, v, CvT, CiT);
  return check_launch("wq_ystage_mma_tiles");
}

int wq_ystage_mma(int64_t n_rows, int64_t n_cols, int64_t n_el, int nal, int wc,
                  const int64_t* r_emin, const int64_t* c_el, const int64_t* c_loc,
                  const int64_t* c_emin, const int64_t* c_emax, const double* v,
                  const double* Cr, const double* LtR, const double* vsum, const double* CvT,
                  const int* CiT, const double* Tb,
                  int64_t n_tab, const int* row_ko, const int* col_ko, double* out, int64_t ldo,
                  int64_t row0, int64_t row1, int sym, void* stream) {
  if (n_rows <= 0 || n_cols <= 0 || (nal != 17 && nal != 5) || wc < 1 || !r_emin || !c_el ||
      !c_loc || !c_emin || !c_emax || !v || !Cr || !LtR || !vsum || !Tb || !row_ko ||
      !col_ko || !out || row0 < 0 || row0 % YM_T != 0 || row1 > n_rows || row1 <= row0 ||
      wc > YM_WCM || ldo < row1 - row0 || n_tab < 2 * n_el - 1 + YM_ZR + YM_TFRONT ||
      (sym && (row0 != 0 || row1 != n_rows || n_rows != n_cols || ldo < n_cols))) {
    set_error("wq_ystage_mma: bad arguments");
    return WQ_EINVAL;
  }
  YmArgs A{n_cols, n_el, wc, r_emin, c_el, c_loc, c_emin, c_emax, v, Cr, LtR, vsum, CvT, CiT, Tb, n_tab,
           row_ko, col_ko, out, ldo, row0, row0, sym};
  dim3 grid((unsigned)(n_cols / YM_T), (unsigned)((row1 - row0) / YM_T));
  if (grid.x == 0 || grid.y == 0) return WQ_OK;
  if (!CvT || !CiT) {
    set_error("wq_ystage_mma: missing tile tables (wq_ystage_mma_tiles)");
    return WQ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nt = (int64_t)grid.x * grid.y;
  const unsigned g = (unsigned)(nt < sms ? nt : sms);
#define WQ_YW_LAUNCH(NA)                                                                         \
  {                                                                                              \
    const size_t smem = (size_t)YwCfg<NA>::SMEM * 8;                                             \
    cudaFuncSetAttribute(ystage_ws_kernel<NA>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                         (int)smem);                                                             \
    ystage_ws_kernel<NA><<<g, YW_THREADS, smem, st>>>(A, (n_rows + 7) / 8 * 8, (int)grid.x,      \
                                                      (int)grid.y);                              \
  }
  if (nal == 17) WQ_YW_LAUNCH(17) else WQ_YW_LAUNCH(5)
#undef WQ_YW_LAUNCH
  return check_launch("wq_ystage_mma");
}

}  // extern "C"
