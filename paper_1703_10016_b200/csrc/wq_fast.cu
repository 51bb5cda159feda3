// Closed-uniform (circulant) assembly: two sm_100a kernels over the
// UPPER-TRIANGLE tile pairs (I <= J) of the N x N matrix (64 x 64 tiles).
//
//  ik1_sym_kernel   IK1(I,J) = G_I K1 G_J^T (assemble_ik1, assembly.py:175-183;
//                   K1_grid, geometry.py:225-248).  Each thread owns two outer
//                   nodes and sweeps the inner nodes of half the tile with
//                   sliding register windows of 2p+1 kernel values: K1 is
//                   evaluated once per node pair (+8% halo) on the FP64 pipe
//                   (accurate-table ln, wq_log.cuh), never stored to HBM; the
//                   first banded contraction happens in registers, the second
//                   reads T = K1 G^T from shared memory with another sliding
//                   window.  Only the upper tile (I,J) is written (IK1 is
//                   symmetric).
//  x2v4_kernel      X2(I,J) and X2(J,I) of the log part (assemble_ik2,
//                   assembly.py:186-245, X-form) on the FP64 tensor cores
//                   (DMMA m8n8k4): Phi = Zext * Uext^T in skewed (diagonal)
//                   coordinates from TMA-staged Z' windows, the banded S
//                   contraction as a second DMMA, then the fused epilogue
//                     A(I,J) = alpha (w IK1(I,J) + X2(I,J) + X2(J,I)^T),
//                     A(J,I) = A(I,J)^T      (scale_and_symmetrize, :262-271).
//
// Both kernels are deterministic (no atomics on values).
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "wq_common.cuh"
#include "wq_log.cuh"
#include "wq_async.cuh"

namespace wq {

constexpr int FT = 64;  // tile rows/cols

// ---------------------------------------------------------------------------
// ik1_sym_kernel: closed uniform nodes, rule i on nodes 2(i-p)+1 .. 2(i-p)+2p+1
// ---------------------------------------------------------------------------

// Tile mapping: sym (tile_row0 < 0): upper-triangle pairs of an nb x nb tile grid;
// rect: tile rows tile_row0 .. + gridDim.x / nbj, all nbj tile columns, output rows
// offset by tile_row0 * FT (a rank's row block).
__device__ __forceinline__ void tile_of_block(int nb, int tile_row0, int64_t pair0,
                                              const int64_t* plist, int& bi, int& bj) {
  if (plist) {                 // explicit list of upper-triangle pair indices
    tri_index(plist[blockIdx.x], nb, bi, bj);
  } else if (tile_row0 < 0) {
    tri_index(pair0 + blockIdx.x, nb, bi, bj);
  } else {
    bi = tile_row0 + (int)(blockIdx.x / nb);
    bj = (int)(blockIdx.x % nb);
  }
}


// ---------------------------------------------------------------------------
// v5 IK1 tile (ik1_sym_kernel).  The v3 tile was bound by L1/shared-memory
// instruction throughput (ncu: L1/TEX 89.7 %, FP64 pipe 47.6 %), and a first
// rework by instruction issue (~50 issued instructions per kernel value, half
// of them integer).  Here:
//  * each thread owns TWO outer nodes q and q + 64 of one column half (the fifth
//    warp one leftover node per lane), so
//    every r-node load ({x, y} as one 16-byte load) and every rule-weight load
//    (16-byte loads of a padded row) serves both;
//  * the ln uses a 64-bin accurate table (one 16-byte load, degree-4
//    economised series, exponent by I2F on the idle conversion pipe:
//    8 FP64 operations, wq_log.cuh);
//  * tile pairs whose node ranges neither wrap at the seam nor touch (all
//    but O(nb) of them) take a fast path: the node-index gap is q - r + const
//    with one sign across the tile, so 1/p^2 is read through one per-thread
//    pointer walked with the r loop (immediate offsets), no diagonal select,
//    and the R-validity test is a running integer min/max of R's high word.
//  The rest (and the closed-form distance mode) take the general path with
//  a running node index.  ~16.5 FP64 and ~13 other instructions per value.
// 160 threads, 3 CTAs per SM at p = 3 (75.3 KB shared memory each).
// ---------------------------------------------------------------------------

constexpr int IK4_THREADS = 160;

template <int P, int MODE>
struct Ik4Cfg {
  static constexpr int WG = 2 * P + 1;
  static constexpr int NQ = 2 * (FT - 1) + WG;
  static constexpr int NQP = NQ | 1;
  static constexpr int QH = (NQ + 1) / 2;     // outer-node pairs (u, u + QH)
  static constexpr int HJ = FT / 2;
  static constexpr int GW = (WG + 1) / 2 * 2;  // padded rule row (16-byte aligned)
  static constexpr int T1 = (FT * NQP + 1) / 2 * 2;
  // T1 | rxy (2 NQ) | rs (NQ, closed-form mode only, padded even) | G (FT GW) | table (128)
  static constexpr int RS = MODE == WQ_K1_TABLE ? 0 : (NQ + 1) / 2 * 2;
  static constexpr int TOTAL = T1 + 2 * NQ + RS + FT * GW + 128;
  static_assert(2 * QH <= IK4_THREADS, "ik1 v5: too many outer-node pairs");
};

// general path: running node index ra, diagonal continuity limit, closed-form mode
template <int MODE>
__device__ __forceinline__ double k1_gen(double qx, double qy, double qJ2, double qs, int qa,
                                         double2 rxy, double rs, int ra,
                                         const double* __restrict__ invp2, double period,
                                         const double2* tab, int& bad) {
  const double dx = qx - rxy.x, dy = qy - rxy.y;
  const double d2 = fma(dx, dx, dy * dy);
  const int g = abs(qa - ra);
  double R;
  if (MODE == WQ_K1_TABLE) {
    R = d2 * __ldg(invp2 + g);
  } else {
    const double xx = fabs(rs - qs);
    const double p = (period / kPi) * fabs(sin(kPi * xx / period));
    R = d2 / (p * p);
  }
  R = g == 0 ? qJ2 : R;  // continuity limit J^2 (geometry.py:240-245)
  const unsigned rh = (unsigned)__double2hiint(R);
  bad |= (rh - 0x00100000u) >= 0x7fe00000u;
  return half_ln64t(R, tab);
}

// fast path: 1/p^2 at a known address; R's high word less that of DBL_MIN folded into
// one unsigned max (zero, subnormal, negative, inf and NaN all land >= 0x7fe00000)
__device__ __forceinline__ double k1_fast(double qx, double qy, double2 rxy, double ip,
                                          unsigned& hmx, const double2* tab) {
  const double dx = qx - rxy.x, dy = qy - rxy.y;
  const double R = fma(dx, dx, dy * dy) * ip;
  hmx = max(hmx, (unsigned)__double2hiint(R) - 0x00100000u);
  return half_ln64t(R, tab);
}

// phase 1 of a tile for the thread's outer nodes A, B and column half jb..jb+HJ-1.
// FAST: SGN = +1 if every q node index exceeds every r node index, -1 if below.
// TWO = false: outer node A only (the leftover nodes of the fifth warp, half the work).
template <int P, int MODE, bool FAST, int SGN, int UNR, bool TWO>
__device__ __forceinline__ void ik1_phase1(double* T1, const double2* rxy, const double* rsv,
                                           const double* G, const double2* tab,
                                           const wq_smooth_t& sm, int64_t q0, int64_t r0, int qA,
                                           int qB, int h, int& bad) {
  using C = Ik4Cfg<P, MODE>;
  constexpr int WG = C::WG, NQP = C::NQP, HJ = C::HJ, GW = C::GW;
  const int64_t nq = sm.nq;
  constexpr bool hasB = TWO;
  const int64_t gA = (q0 + qA) % nq, gB = (q0 + qB) % nq;
  const double xA = sm.fx[gA], yA = sm.fy[gA];
  const double xB = sm.fx[gB], yB = sm.fy[gB];
  const int jb = h * HJ;
  double wA[WG], wB[WG];
  // general-path state
  const int qaA = (int)gA, qaB = (int)gB;
  const double J2A = sm.J[gA] * sm.J[gA], J2B = sm.J[gB] * sm.J[gB];
  const double sA = sm.s[gA], sB = sm.s[gB];
  const int nqi = (int)nq;
  int ra = (int)((r0 + 2 * jb) % nq);
  // fast-path state: ip(q, r) = invp2[SGN (q0 - r0 + q - r)] = pA[-SGN r'] with r' = r - 2 jb
  const double* __restrict__ pA = sm.invp2 + SGN * (q0 - r0 + qA - 2 * jb);
  const double* __restrict__ pB = sm.invp2 + SGN * (q0 - r0 + qB - 2 * jb);
  unsigned hmx = 0u;
  // fast path: 1/p^2 of the next column's two new r nodes is loaded one column ahead
  double ipA0 = 0.0, ipA1 = 0.0, ipB0 = 0.0, ipB1 = 0.0;
  auto eval = [&](int r, int rr, double& vA, double& vB, double ipa, double ipb) {
    const double2 p = rxy[r];
    if (FAST) {
      vA = k1_fast(xA, yA, p, ipa, hmx, tab);
      if (TWO) vB = k1_fast(xB, yB, p, ipb, hmx, tab);
    } else {
      const double rs = MODE != WQ_K1_TABLE ? rsv[r] : 0.0;
      vA = k1_gen<MODE>(xA, yA, J2A, sA, qaA, p, rs, ra, sm.invp2, sm.period, tab, bad);
      if (TWO) vB = k1_gen<MODE>(xB, yB, J2B, sB, qaB, p, rs, ra, sm.invp2, sm.period, tab, bad);
      if (++ra == nqi) ra = 0;
    }
  };
#pragma unroll
  for (int w = 0; w < WG - 2; ++w)
    eval(2 * jb + w, w, wA[w], wB[w], FAST ? __ldg(pA - SGN * w) : 0.0,
         (FAST && TWO) ? __ldg(pB - SGN * w) : 0.0);
  if (FAST) {
    ipA0 = __ldg(pA - SGN * (WG - 2));
    ipA1 = __ldg(pA - SGN * (WG - 1));
    if (TWO) {
      ipB0 = __ldg(pB - SGN * (WG - 2));
      ipB1 = __ldg(pB - SGN * (WG - 1));
    }
  }
  // software pipeline: the two new kernel values (per outer node) of column jj + 1 are
  // evaluated while column jj is contracted, so their independent chains fill the latency of
  // the contraction's dependent FMA chain (the kernel is bound by the number of independent
  // chains in flight per scheduler, not by issue slots or the FP64 pipe)
  double cA0, cA1, cB0 = 0.0, cB1 = 0.0;
  auto column = [&](int jj, double& vA0, double& vA1, double& vB0, double& vB1) {
    const int r = 2 * (jb + jj) + WG - 2;
    const double a0 = ipA0, a1 = ipA1, b0 = ipB0, b1 = ipB1;
    if (FAST && jj + 1 < HJ) {
      const int rn = 2 * (jj + 1) + WG - 2;
      ipA0 = __ldg(pA - SGN * rn);
      ipA1 = __ldg(pA - SGN * (rn + 1));
      if (TWO) {
        ipB0 = __ldg(pB - SGN * rn);
        ipB1 = __ldg(pB - SGN * (rn + 1));
      }
    }
    eval(r, 2 * jj + WG - 2, vA0, vB0, a0, b0);
    eval(r + 1, 2 * jj + WG - 1, vA1, vB1, a1, b1);
  };
  column(0, cA0, cA1, cB0, cB1);
#pragma unroll UNR
  for (int jj = 0; jj < HJ; ++jj) {
    const int j = jb + jj;
    double nA0 = 0.0, nA1 = 0.0, nB0 = 0.0, nB1 = 0.0;
    if (jj + 1 < HJ) column(jj + 1, nA0, nA1, nB0, nB1);
    wA[WG - 2] = cA0;
    wA[WG - 1] = cA1;
    wB[WG - 2] = cB0;
    wB[WG - 1] = cB1;
    const double2* g2 = reinterpret_cast<const double2*>(G + j * GW);
    double g[GW];
#pragma unroll
    for (int w = 0; w < GW / 2; ++w) {
      const double2 t = g2[w];
      g[2 * w] = t.x;
      g[2 * w + 1] = t.y;
    }
    double accA = 0.0, accB = 0.0;
#pragma unroll
    for (int w = 0; w < WG; ++w) {
      accA = fma(wA[w], g[w], accA);
      accB = fma(wB[w], g[w], accB);
    }
    T1[j * NQP + qA] = accA;
    if (hasB) T1[j * NQP + qB] = accB;
#pragma unroll
    for (int w = 0; w < WG - 2; ++w) {
      wA[w] = wA[w + 2];
      wB[w] = wB[w + 2];
    }
    cA0 = nA0;
    cA1 = nA1;
    cB0 = nB0;
    cB1 = nB1;
  }
  if (FAST) bad |= hmx >= 0x7fe00000u;
}

template <int P, int MODE, int UNR>
__device__ __forceinline__ void ik1_tile_v5(const wq_smooth_t& sm, int bi, int bj, int64_t row_off,
                                            double* X, int64_t ldx, int& bad, double* dsm) {
  using C = Ik4Cfg<P, MODE>;
  constexpr int WG = C::WG, NQ = C::NQ, NQP = C::NQP, QH = C::QH, GW = C::GW;
  double* T1 = dsm;                                            // [FT][NQP]
  double2* rxy = reinterpret_cast<double2*>(dsm + C::T1);      // [NQ]
  double* rsv = dsm + C::T1 + 2 * NQ;                          // [NQ] (closed-form mode)
  double* G = rsv + C::RS;                                     // [FT][GW]: G_J, then G_I
  double2* tab = reinterpret_cast<double2*>(G + FT * GW);      // [64]

  const int64_t N = sm.n_rows, nq = sm.nq;
  const int64_t I0 = (int64_t)bi * FT, J0 = (int64_t)bj * FT;
  const int ni = (int)min((int64_t)FT, N - I0);
  const int nj = (int)min((int64_t)FT, N - J0);
  const int tid = threadIdx.x;
  int64_t q0 = sm.g_start[I0] % nq;
  if (q0 < 0) q0 += nq;
  int64_t r0 = sm.g_start[J0] % nq;
  if (r0 < 0) r0 += nq;
  for (int k = tid; k < NQ; k += blockDim.x) {
    const int64_t b = (r0 + k) % nq;
    rxy[k] = make_double2(sm.fx[b], sm.fy[b]);
    if (MODE != WQ_K1_TABLE) rsv[k] = sm.s[b];
  }
  for (int k = tid; k < FT * GW; k += blockDim.x) {
    const int jj = k / GW, w = k - jj * GW;
    G[k] = (jj < nj && w < WG) ? sm.g_w[(J0 + jj) * WG + w] : 0.0;
  }
  for (int k = tid; k < 128; k += blockDim.x) reinterpret_cast<double*>(tab)[k] = kTang64[k];
  __syncthreads();

  // ---- phase 1: warps 0-3 take outer-node pairs (u, u + 64) of column half h = warp / 2;
  // warp 4 the NQ - 128 leftover nodes, one per lane and half (half the work per lane) ----
  {
    constexpr int NL = NQ - 128;
    static_assert(NL > 0 && 2 * NL <= 32 && IK4_THREADS == 160, "ik1 v5: phase-1 mapping");
    const int warp = tid >> 5, lane = tid & 31;
    const bool nowrap = q0 + NQ <= nq && r0 + NQ <= nq;
    const bool fp = MODE == WQ_K1_TABLE && nowrap && q0 >= r0 + NQ;
    const bool fm = MODE == WQ_K1_TABLE && nowrap && r0 >= q0 + NQ;
    if (warp < 4) {
      const int h = warp >> 1, u = tid & 63;
      if (fp) ik1_phase1<P, MODE, true, 1, UNR, true>(T1, rxy, rsv, G, tab, sm, q0, r0, u, u + 64, h, bad);
      else if (fm) ik1_phase1<P, MODE, true, -1, UNR, true>(T1, rxy, rsv, G, tab, sm, q0, r0, u, u + 64, h, bad);
      else ik1_phase1<P, MODE, false, 1, UNR, true>(T1, rxy, rsv, G, tab, sm, q0, r0, u, u + 64, h, bad);
    } else if (lane < 2 * NL) {
      const int h = lane / NL, q = 128 + lane % NL;
      if (fp) ik1_phase1<P, MODE, true, 1, UNR, false>(T1, rxy, rsv, G, tab, sm, q0, r0, q, q, h, bad);
      else if (fm) ik1_phase1<P, MODE, true, -1, UNR, false>(T1, rxy, rsv, G, tab, sm, q0, r0, q, q, h, bad);
      else ik1_phase1<P, MODE, false, 1, UNR, false>(T1, rxy, rsv, G, tab, sm, q0, r0, q, q, h, bad);
    }
  }
  // G_I is loaded before the barrier (its latency overlaps the wait for the slowest
  // phase-1 warp) and stored into the G region after it
  constexpr int GPT = (FT * GW + IK4_THREADS - 1) / IK4_THREADS;
  double gv[GPT];
#pragma unroll
  for (int u = 0; u < GPT; ++u) {
    const int k = tid + u * IK4_THREADS, ii = k / GW, w = k - ii * GW;
    gv[u] = (k < FT * GW && ii < ni && w < WG) ? __ldg(sm.g_w + (I0 + ii) * WG + w) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < GPT; ++u)
    if (tid + u * IK4_THREADS < FT * GW) G[tid + u * IK4_THREADS] = gv[u];
  __syncthreads();

  // ---- phase 2: item (j, half c): IK1[i][j], i in 32c .. 32c+31 ----
  if (tid < 2 * FT) {
    const int j = tid & (FT - 1), c = tid >> 6;
    const double* t = T1 + j * NQP;
    const int i0 = 32 * c;
    double win[WG];
#pragma unroll
    for (int w = 0; w < WG - 2; ++w) win[w] = t[2 * i0 + w];
#pragma unroll 4
    for (int ii = 0; ii < 32; ++ii) {
      const int i = i0 + ii;
      win[WG - 2] = t[2 * i + WG - 2];
      win[WG - 1] = t[2 * i + WG - 1];
      const double2* g2 = reinterpret_cast<const double2*>(G + i * GW);
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < GW / 2; ++w) {
        const double2 gg = g2[w];
        acc = fma(gg.x, win[2 * w], acc);
        if (2 * w + 1 < WG) acc = fma(gg.y, win[2 * w + 1], acc);
      }
      if (i < ni && j < nj) X[(I0 - row_off + i) * ldx + J0 + j] = acc;
#pragma unroll
      for (int w = 0; w < WG - 2; ++w) win[w] = win[w + 2];
    }
  }
}

template <int P, int MODE, int TAB>
__global__ void __launch_bounds__(IK4_THREADS, 3)
ik1_sym_kernel(wq_smooth_t sm, int nb, int tile_row0, int64_t pair0, const int64_t* plist, double* X,
               int64_t ldx, int* flag) {
  extern __shared__ double dsm[];
  int bi, bj;
  tile_of_block(nb, tile_row0, pair0, plist, bi, bj);
  const int64_t row_off = tile_row0 < 0 ? 0 : (int64_t)tile_row0 * FT;
  int bad = 0;
  ik1_tile_v5<P, MODE, TAB == 1 ? 2 : 4>(sm, bi, bj, row_off, X, ldx, bad, dsm);
  if (bad) atomicOr(flag, WQ_FLAG_R_NONPOSITIVE);
}

// ---------------------------------------------------------------------------
// x2_pairs_kernel (DMMA)
// ---------------------------------------------------------------------------


template <int P>
struct X2Cfg {
  static constexpr int D = P;                          // nref = 1
  static constexpr int NA = P + 13;                    // P + 1 = p + JFIT + 1
  static constexpr int NAPAD = (NA + 3) / 4 * 4;
  static constexpr int TU = P + 1;
  static constexpr int WS = 2 * D + 1;
  static constexpr int WSPAD = (WS + 3) / 4 * 4;
  static constexpr int KTOT = TU * NAPAD + WSPAD;
  static constexpr int NSTEPS = KTOT / 4;
  static constexpr int SZ = TU * NAPAD / 4;            // k-steps of the Z' part
  static constexpr int ZSTRIDE = ((NAPAD + 1 + 11) / 16) * 16 + 4;   // == 4 mod 16, > NAPAD
  static constexpr int AMAX = (TU > WSPAD ? TU : WSPAD) - 1;
  static constexpr int SPAN = FT + 2 * D;              // Phi columns (m range)
  static constexpr int NKB = (SPAN + 7 + 7) / 8;       // 8-row k blocks per row group
  static constexpr int ZROWS = 56 + 8 * NKB + AMAX;
  static constexpr int KS = ((8 + 2 * D) + 3) / 4 * 4;  // S-contraction K
  static constexpr int PF = 5;                          // B-fragment prefetch depth (k-steps)
};

constexpr int X2_THREADS = 256;

constexpr int PSTRIDE = 76;  // Phi smem row stride (== 12 mod 16), >= SPAN and 56 + KS

// Phi[m][i] for m in [M0, M0 + SPAN), i in the tile rows starting at R0 (Uext rows),
// written to Phs[i][m - M0].  Skewed coordinates: row group G (8 functions) needs the table
// blocks zb = 7 - G .. 7 - G + NKB - 1 (block zb = window rows 8 zb + AMAX - off ..); adjacent
// groups share all but one of them, so warp (g, h) = (warp / 2, warp % 2) takes BOTH groups
// 2g and 2g + 1 over half of the blocks: NH + 1 A fragments from shared memory feed 2 NH
// DMMAs per k-step (12 loads for 20 DMMAs at p = 3 instead of 20).  B fragments come from
// the fragment-ordered Uext (one coalesced 256-byte load per group and k-step).
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// before_store() runs after the last DMMA and before the first write to Phs
template <int P, class Hook = NoHook>
__device__ __forceinline__ void phi_block(const double* __restrict__ Ufrag, int64_t N,
                                          const double* Zsm, double* Phs, int64_t R0, int warp,
                                          Hook before_store = Hook()) {
  using C = X2Cfg<P>;
  constexpr int NH0 = (C::NKB + 1) / 2, NH1 = C::NKB - NH0;   // blocks per half
  constexpr int PF = C::PF;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, c = lane & 3;
  const int g = warp >> 1, h = warp & 1;
  const int nh = h ? NH1 : NH0;
  double accA[NH0][2], accB[NH0][2];   // group 2g (A fragments j + 1), group 2g + 1 (j)
#pragma unroll
  for (int j = 0; j < NH0; ++j) accA[j][0] = accA[j][1] = accB[j][0] = accB[j][1] = 0.0;
  // B fragments: group G of the tile at Ufrag[((R0 / 8 + G) * NSTEPS + s) * 32 + lane]
  const int64_t grpA = R0 / 8 + 2 * g;
  const bool vA = 8 * grpA < N, vB = 8 * (grpA + 1) < N;
  const double* __restrict__ uA = Ufrag + (vA ? grpA : 0) * (C::NSTEPS * 32) + lane;
  const double* __restrict__ uB = Ufrag + (vB ? grpA + 1 : 0) * (C::NSTEPS * 32) + lane;
  double bqA[PF], bqB[PF];
#pragma unroll
  for (int s = 0; s < PF; ++s) {
    bqA[s] = vA ? __ldg(uA + 32 * s) : 0.0;
    bqB[s] = vB ? __ldg(uB + 32 * s) : 0.0;
  }
  // A fragment j of k-step s: window row 8 (6 - 2g + h NH0 + j) + r + AMAX - off(s), column col(s)
  const int zbase = 8 * (6 - 2 * g + h * NH0) + r + C::AMAX;
  auto zptr = [&](int s) -> const double* {
    int off, col;
    if (s < C::SZ) {
      off = (4 * s) / C::NAPAD;
      col = (4 * s - off * C::NAPAD) + c;
    } else {
      off = 4 * (s - C::SZ) + c;
      col = C::NAPAD;
    }
    return Zsm + (zbase - off) * C::ZSTRIDE + col;
  };
  double afr[2][NH0 + 1];
  {
    const double* z = zptr(0);
#pragma unroll
    for (int j = 0; j <= NH0; ++j)
      if (NH0 == NH1 || j <= nh) afr[0][j] = z[j * 8 * C::ZSTRIDE];
  }
#pragma unroll
  for (int s = 0; s < C::NSTEPS; ++s) {
    const int cur = s & 1;
    if (s + 1 < C::NSTEPS) {
      const double* z = zptr(s + 1);
#pragma unroll
      for (int j = 0; j <= NH0; ++j)
        if (NH0 == NH1 || j <= nh) afr[cur ^ 1][j] = z[j * 8 * C::ZSTRIDE];
    }
    const double ba = bqA[s % PF], bb = bqB[s % PF];
    if (s + PF < C::NSTEPS) {
      bqA[s % PF] = vA ? __ldg(uA + 32 * (s + PF)) : 0.0;
      bqB[s % PF] = vB ? __ldg(uB + 32 * (s + PF)) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < NH0; ++j) {
      if (NH0 == NH1 || j < nh) {
        dmma(accB[j][0], accB[j][1], afr[cur][j], bb);
        dmma(accA[j][0], accA[j][1], afr[cur][j + 1], ba);
      }
    }
  }
  before_store();
  // accA[j]: group 2g, block kb = h NH0 + j; accB[j]: group 2g + 1, same kb.
  // Entry (r, 2c + e) of block kb of group G is Phi[m][i], i = 8G + 2c + e,
  // m - M0 = 8 kb + r + (2c + e) - 7
#pragma unroll
  for (int j = 0; j < NH0; ++j) {
    if (NH0 == NH1 || j < nh) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int mm = 8 * (h * NH0 + j) + r + 2 * c + e - 7;
        if (mm >= 0 && mm < C::SPAN) {
          Phs[(16 * g + 2 * c + e) * PSTRIDE + mm] = accA[j][e];
          Phs[(16 * g + 8 + 2 * c + e) * PSTRIDE + mm] = accB[j][e];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// x2 v5 (x2v4_kernel): both Z' windows requested at CTA start (one mbarrier each);
// the IK1 tile, the banded S fragments and the output tiles go straight between
// global memory and registers in the DMMA accumulator layout (every access
// sector-efficient: 64-byte row segments); only Phi and the orientation hand-off
// T live in shared memory (~85 KB, 2 CTAs per SM).
//
//   phi (DMMA)  Phi[i][m] = sum_K Zext-window[..][K] Uext[i][K] in skewed
//               coordinates, stored as Phs[i][m] (stride 76)
//   S   (DMMA)  warp w owns one 8-column block of the output (j = 8w..8w+7 in
//               orientation 0, i in orientation 1): its band B fragments are loaded
//               once into registers and the warp sweeps the 8 row blocks with A
//               fragments from Phs
// Orientation 0 gives T = alpha (w IK1(I,J) + X2(I,J)) (accumulators start from
// alpha w IK1); T goes through shared memory to the orientation-1 layout, whose
// accumulators start from T^T and add alpha X2(J,I): A(J,I), stored to rows J
// and, transposed, to rows I.  One tile pair per CTA: co-resident CTAs stay out
// of phase, so one CTA's staging / hand-off / stores overlap the other's DMMAs (a
// persistent grid of 2 CTAs per SM that refilled each window for its next pair
// as soon as phi had read it ran the two CTAs in lock step: 9.2 vs 8.3 ms).
// ---------------------------------------------------------------------------

// loads issued where written (volatile: not sunk to their first use, so their HBM / L2
// latency overlaps the phi DMMAs that follow)
__device__ __forceinline__ double2 ld_cs_v2(const double* p) {
  double2 v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_cs(const double* p) {
  double v;
  asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_nc(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

constexpr int X5_TS = 66;   // T hand-off [i][j] row stride (16-byte row-fragment stores)

#ifdef WQ_X2_TIMELINE
// tools build only (tools/x2_timeline_build.sh): per-CTA phase clocks and SM id
__device__ long long* g_x2_tl = nullptr;
#define X5_TL(k)                                                                          \
  do {                                                                                    \
    if (threadIdx.x == 0 && g_x2_tl) {                                                    \
      g_x2_tl[(int64_t)blockIdx.x * 10 + (k)] = clock64();                                \
      if ((k) == 0) {                                                                     \
        unsigned sm;                                                                      \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));                                   \
        g_x2_tl[(int64_t)blockIdx.x * 10 + 9] = sm;                                        \
      }                                                                                   \
    }                                                                                     \
  } while (0)
// x2ws: stamps of pair k == 20 of every CTA: slots 0-9 Phi group (thread 0), 16-23 epilogue
#define XW_TL(slot)                                                                       \
  do {                                                                                    \
    if (k == 20 && (threadIdx.x & 255) == 0 && g_x2_tl)                                   \
      g_x2_tl[(int64_t)blockIdx.x * 32 + (slot)] = clock64();                             \
  } while (0)
#else
#define X5_TL(k) do {} while (0)
#define XW_TL(slot) do {} while (0)
#endif

template <int P>
struct X4Smem {
  using C = X2Cfg<P>;
  static constexpr int ZW = C::ZROWS * C::ZSTRIDE;                    // one Z' window
  static constexpr int PH = FT * PSTRIDE;                             // Phi, then T
  static_assert(FT * X5_TS <= PH, "T hand-off overflows the Phi buffer");
  static constexpr int TOTAL = 2 * ZW + PH + 4;                       // + mbarriers
};

// first table row of the skewed Z' window of orientation o of tile pair (bi, bj)
template <int P>
__device__ __forceinline__ int64_t x5_gmin(int o, int bi, int bj) {
  using C = X2Cfg<P>;
  const int64_t I0 = (int64_t)bi * FT, J0 = (int64_t)bj * FT;
  const int64_t R0 = o == 0 ? I0 : J0;
  const int64_t M0 = (o == 0 ? J0 : I0) - C::D;
  return M0 - (R0 + 63) + P - C::AMAX;
}

// ZROWS contiguous table rows from gmin (mod n) into dst on the TMA engine (two pieces at
// the seam), completing on bar
template <int P>
__device__ __forceinline__ void x5_window_at(double* dst, const double* Zext, int64_t n, int64_t g0,
                                             uint64_t* bar);

template <int P>
__device__ __forceinline__ void x5_window(double* dst, const double* Zext, int64_t n, int64_t gmin,
                                          uint64_t* bar) {
  x5_window_at<P>(dst, Zext, n, pmod(gmin, n), bar);
}

// the same from the reduced first row g0 = gmin mod n
template <int P>
__device__ __forceinline__ void x5_window_at(double* dst, const double* Zext, int64_t n, int64_t g0,
                                             uint64_t* bar) {
  using C = X2Cfg<P>;
  constexpr unsigned RB = C::ZSTRIDE * 8;
  const uint64_t pol = l2_evict_last();    // the Z' table is re-read by every tile pair
  const int64_t first = min((int64_t)C::ZROWS, n - g0);
  mbar_arrive_expect_tx(bar, C::ZROWS * RB);
  bulk_g2s_hint(dst, Zext + g0 * C::ZSTRIDE, (unsigned)first * RB, bar, pol);
  if (first < C::ZROWS)
    bulk_g2s_hint(dst + first * C::ZSTRIDE, Zext, (unsigned)(C::ZROWS - first) * RB, bar, pol);
}

template <int P>
__global__ void __launch_bounds__(X2_THREADS, 2)
x2v4_kernel(int64_t N, const double* __restrict__ Uext, const double* __restrict__ Zext,
            const double* __restrict__ sw, double alpha, double w_ik1, double* X, int64_t ldx,
            int nb, int tile_row0, int64_t pair0, const int64_t* plist) {
  using C = X2Cfg<P>;
  using L = X4Smem<P>;
  constexpr int KS4 = C::KS / 4;
  extern __shared__ double smem[];
  double* Zs0 = smem;
  double* Zs1 = Zs0 + L::ZW;
  double* Phs = Zs1 + L::ZW;          // Phi[i][m] (both orientations), then the T hand-off
  uint64_t* bar = reinterpret_cast<uint64_t*>(Phs + L::PH);
  const int64_t n = N;
  const bool rect = tile_row0 >= 0;
  const int64_t row_off = rect ? (int64_t)tile_row0 * FT : 0;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int r = lane >> 2, c = lane & 3;
  const int norient = rect ? 1 : 2;
  const bool with_ik1 = w_ik1 != 0.0;
  const bool zbulk = n >= C::ZROWS;
  int bi, bj;
  tile_of_block(nb, tile_row0, pair0, plist, bi, bj);
  const int64_t I0 = (int64_t)bi * FT, J0 = (int64_t)bj * FT;
  const int ni = (int)min((int64_t)FT, N - I0);
  const int nj = (int)min((int64_t)FT, N - J0);
  const int64_t gmin[2] = {x5_gmin<P>(0, bi, bj), x5_gmin<P>(1, bi, bj)};
  X5_TL(0);

  // Z' windows of both orientations, requested at once
  if (zbulk) {
    if (tid == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
    }
    __syncthreads();
    if (tid == 0)
      for (int o = 0; o < norient; ++o) x5_window<P>(o == 0 ? Zs0 : Zs1, Zext, n, gmin[o], bar + o);
  } else {
    constexpr int CH = C::ZSTRIDE / 2;  // 16-byte chunks per table row
    for (int o = 0; o < norient; ++o) {
      double* dst = o == 0 ? Zs0 : Zs1;
      int64_t g0 = gmin[o] % n;
      if (g0 < 0) g0 += n;
      for (int k = tid; k < C::ZROWS * CH; k += X2_THREADS) {
        const int row = k / CH, cc = 2 * (k - row * CH);
        int64_t g = g0 + row;
        while (g >= n) g -= n;
        cp_async16(dst + row * C::ZSTRIDE + cc, Zext + g * C::ZSTRIDE + cc);
      }
    }
  }
  // Phi's pad columns (read by the band contraction against zero B entries) must be finite
  for (int k = tid; k < FT * (PSTRIDE - C::SPAN); k += X2_THREADS)
    Phs[(k / (PSTRIDE - C::SPAN)) * PSTRIDE + C::SPAN + k % (PSTRIDE - C::SPAN)] = 0.0;

  // accumulators of orientation 0: lane (i = 8 ib + r, j = 8 warp + 2c + e); the raw IK1
  // tile now (scaled by alpha w after phi0, when the loads have landed)
  double acc[8][2];
  {
    const int jj = 8 * warp + 2 * c;
    const double* src = X + (I0 - row_off) * ldx + J0 + jj;
    const bool vec = with_ik1 && ni == FT && nj == FT && (ldx & 1) == 0 &&
                     (reinterpret_cast<uintptr_t>(X + J0) & 15) == 0;
#pragma unroll
    for (int ib = 0; ib < 8; ++ib) {
      const int ii = 8 * ib + r;
      if (vec) {
        const double2 v = ld_cs_v2(src + ii * ldx);
        acc[ib][0] = v.x;
        acc[ib][1] = v.y;
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          acc[ib][e] = (with_ik1 && ii < ni && jj + e < nj) ? ld_cs(src + ii * ldx + e) : 0.0;
      }
    }
  }

  // one orientation: 0 = Phi rows I over the J range with band S_J, 1 = rows J over I, S_I
  auto orient = [&](const int o) {
    const int64_t R0 = o == 0 ? I0 : J0;
    // B fragments of the alpha S band for this warp's column block (raw now, scaled after
    // phi, when the loads have landed): bS[s] = S_{C0 + 8 warp + r}[4 s + c - r]
    double bS[KS4];
    {
      const int64_t C0 = o == 0 ? J0 : I0;
      const int nc = o == 0 ? nj : ni;
      const int row = 8 * warp + r;
#pragma unroll
      for (int s2 = 0; s2 < KS4; ++s2) {
        const int t = 4 * s2 + c - r;
        bS[s2] = (t >= 0 && t <= 2 * C::D && row < nc) ? ld_nc(sw + (C0 + row) * C::WS + t) : 0.0;
      }
    }
    if (zbulk) {
      mbar_wait(bar + o, 0);
    } else if (o == 0) {
      cp_async_wait_all();
      __syncthreads();
    }
    X5_TL(1 + 4 * o);
    phi_block<P>(Uext, N, o == 0 ? Zs0 : Zs1, Phs, R0, warp);
#pragma unroll
    for (int s2 = 0; s2 < KS4; ++s2) bS[s2] *= alpha;
    if (o == 0) {
      const double aw = alpha * w_ik1;
#pragma unroll
      for (int rb = 0; rb < 8; ++rb) {
        acc[rb][0] *= aw;
        acc[rb][1] *= aw;
      }
    }
    __syncthreads();
    X5_TL(2 + 4 * o);
    // band contraction (DMMA; the warp's band B fragments stay in registers):
    // acc[rb][e] += sum_s Phs[8 rb + r][8 warp + 4 s + c] bS[s]
#pragma unroll
    for (int rb = 0; rb < 8; ++rb) {
#pragma unroll
      for (int s2 = 0; s2 < KS4; ++s2) {
        const double a = Phs[(8 * rb + r) * PSTRIDE + 8 * warp + 4 * s2 + c];
        dmma(acc[rb][0], acc[rb][1], a, bS[s2]);
      }
    }
  };
  orient(0);
  X5_TL(3);
  if (rect) {
    // unsymmetrised row block: X(I,J) = alpha (w IK1 + X2(I,J)) = T
#pragma unroll
    for (int rb = 0; rb < 8; ++rb) {
      const int ii = 8 * rb + r;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jj = 8 * warp + 2 * c + e;
        if (ii < ni && jj < nj) X[(I0 - row_off + ii) * ldx + J0 + jj] = acc[rb][e];
      }
    }
    return;
  }
  {
    // T[i][j] (i = 8 rb + r, j = 8 warp + 2c + e) -> acc of orientation 1: lane
    // (j = 8 rb + r, i = 8 warp + 2c + e) starts from T[i][j]
    __syncthreads();                         // Phi0 fully read
    double* Tsm = Phs;
#pragma unroll
    for (int rb = 0; rb < 8; ++rb)
      *reinterpret_cast<double2*>(Tsm + (8 * rb + r) * X5_TS + 8 * warp + 2 * c) =
          make_double2(acc[rb][0], acc[rb][1]);
    __syncthreads();
#pragma unroll
    for (int rb = 0; rb < 8; ++rb)
#pragma unroll
      for (int e = 0; e < 2; ++e) acc[rb][e] = Tsm[(8 * warp + 2 * c + e) * X5_TS + 8 * rb + r];
    __syncthreads();                         // T read before Phi1 overwrites it
  }
  X5_TL(4);
  orient(1);
  X5_TL(7);

  // acc[rb][e] = A(J,I)[j = 8 rb + r][i = 8 warp + 2c + e]: rows J (16-byte pieces, 64-byte
  // row segments per 4 lanes) and the transpose into rows I (8-byte pieces, 64-byte segments)
  const int i = 8 * warp + 2 * c;
  const bool full = ni == FT && nj == FT && (ldx & 1) == 0 &&
                    (reinterpret_cast<uintptr_t>(X + I0) & 15) == 0;
  if (bi != bj) {
#pragma unroll
    for (int rb = 0; rb < 8; ++rb) {
      const int j = 8 * rb + r;
      double* rowJ = X + (J0 + j) * ldx + I0 + i;
      if (full) {
        __stcs(reinterpret_cast<double2*>(rowJ), make_double2(acc[rb][0], acc[rb][1]));
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (j < nj && i + e < ni) __stcs(rowJ + e, acc[rb][e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int rb = 0; rb < 8; ++rb) {
        const int j = 8 * rb + r;
        if (j < nj && i + e < ni) __stcs(X + (I0 + i + e) * ldx + J0 + j, acc[rb][e]);
      }
  } else {
    // diagonal tile: entry (j, i) with i <= j written to both (j, i) and (i, j), so A is
    // exactly symmetric
#pragma unroll
    for (int rb = 0; rb < 8; ++rb)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = 8 * rb + r;
        if (j < nj && i + e < ni && i + e <= j) {
          __stcs(X + (J0 + j) * ldx + I0 + i + e, acc[rb][e]);
          __stcs(X + (I0 + i + e) * ldx + J0 + j, acc[rb][e]);
        }
      }
  }
  X5_TL(8);
}

// ---------------------------------------------------------------------------
// x2 v6 (x2ws_kernel): warp-specialised persistent variant of x2v4_kernel for full
// upper-triangle sweeps.  One CTA of 16 warps per SM walks the tile pairs
// blockIdx.x, + gridDim.x, ...:
//   warps 0-7  (Phi group)      phi0(k), phi1(k), phi0(k+1), ... back to back: the DMMA
//                               stream never stops for staging, hand-off or stores, and the
//                               warps never meet at a barrier, so they drift apart and one
//                               warp's fragment prologue / Phi stores hide under the others'
//                               DMMAs.
//   warps 8-15 (epilogue group) per pair: IK1 tile and S band into registers, band
//                               contraction 0 from Phs[0], T hand-off through its own
//                               buffer, band contraction 1 from Phs[1], stores of A(J,I)
//                               and A(I,J) - all while the Phi group computes the next Phi.
//                               Its first thread re-requests Z' window o (TMA) for the next
//                               pair as soon as Phs[o] is full (every Phi warp has then read
//                               the window), a whole phase ahead of its use.
// Hand-over by shared-memory mbarriers (arrive by one lane per warp after __syncwarp, wait by
// parity): wfull for the windows, pfull / pempty for the two Phi buffers.
// Same arithmetic, in the same order, as x2v4_kernel: bit-identical results.
// ---------------------------------------------------------------------------

constexpr int XW_THREADS = 512;
constexpr int XW_BAR_EPI = 1;   // named barrier of the epilogue group (T hand-off)


template <int P>
struct XwSmem {
  using C = X2Cfg<P>;
  static constexpr int ZW = C::ZROWS * C::ZSTRIDE;   // one Z' window
  static constexpr int PH = FT * PSTRIDE;            // one Phi buffer
  static constexpr int TS = FT * X5_TS;              // T hand-off
  static constexpr int TOTAL = 2 * ZW + 2 * PH + TS + 6;   // + 6 mbarriers
};

template <int P>
__global__ void __launch_bounds__(XW_THREADS, 1)
x2ws_kernel(int64_t N, const double* __restrict__ Uext, const double* __restrict__ Zext,
            const double* __restrict__ sw, double alpha, double w_ik1, double* X, int64_t ldx,
            int nb, int64_t pair0, int64_t npairs, const int64_t* plist) {
  using C = X2Cfg<P>;
  using L = XwSmem<P>;
  constexpr int KS4 = C::KS / 4;
  extern __shared__ double smem[];
  double* Tsm = smem + 2 * L::ZW + 2 * L::PH;
  uint64_t* wfull = reinterpret_cast<uint64_t*>(Tsm + L::TS);   // [2] window o landed (tx)
  uint64_t* pfull = wfull + 2;                                  // [2] Phs[o] written by 8 Phi warps
  uint64_t* pempty = wfull + 4;                                 // [2] Phs[o] read by 8 epilogue warps
  const int tid = threadIdx.x;
  const int64_t mine = (npairs - blockIdx.x + gridDim.x - 1) / gridDim.x;   // pairs of this CTA
  auto pair_of = [&](int64_t k, int& bi, int& bj) {
    const int64_t t = blockIdx.x + k * gridDim.x;
    tri_index(plist ? plist[t] : pair0 + t, nb, bi, bj);
  };
  if (tid == 0) {
    for (int o = 0; o < 2; ++o) {
      mbar_init(wfull + o, 1);
      mbar_init(pfull + o, 8);
      mbar_init(pempty + o, 8);
    }
  }
  // Phi's pad columns (read by the band contraction against zero B entries) must be finite
  for (int k = tid; k < 2 * FT * (PSTRIDE - C::SPAN); k += XW_THREADS) {
    const int b = k / (FT * (PSTRIDE - C::SPAN)), q = k % (FT * (PSTRIDE - C::SPAN));
    smem[2 * L::ZW + b * L::PH + (q / (PSTRIDE - C::SPAN)) * PSTRIDE + C::SPAN +
         q % (PSTRIDE - C::SPAN)] = 0.0;
  }
  __syncthreads();
  if (mine <= 0) return;

  if (tid < 256) {
    // ------------------------------ Phi group ------------------------------
    const int warp = tid >> 5;
    for (int64_t k = 0; k < mine; ++k) {
      int bi, bj;
      pair_of(k, bi, bj);
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const int64_t R0 = (int64_t)(o == 0 ? bi : bj) * FT;
        XW_TL(5 * o);
        mbar_wait(wfull + o, (unsigned)(k & 1));
        XW_TL(5 * o + 1);
        phi_block<P>(Uext, N, smem + o * L::ZW, smem + 2 * L::ZW + o * L::PH, R0, warp, [&]() {
          XW_TL(5 * o + 2);
          // Phs[o] is free once the epilogue group has contracted the previous pair's Phi
          if (k > 0) mbar_wait(pempty + o, (unsigned)((k - 1) & 1));
          XW_TL(5 * o + 3);
        });
        warp_arrive(pfull + o);
        XW_TL(5 * o + 4);
      }
    }
  } else {
    // ---------------------------- epilogue group ---------------------------
    const int et = tid - 256;
    const int lane = et & 31, warp = et >> 5;
    const int r = lane >> 2, c = lane & 3;
    const bool with_ik1 = w_ik1 != 0.0;
    // raw IK1 tile of pair (bi, bj) in the orientation-0 accumulator layout:
    // lane (i = 8 ib + r, j = 8 warp + 2c + e)
    auto load_ik1 = [&](int bi, int bj, double (&t)[8][2]) {
      const int64_t I0 = (int64_t)bi * FT, J0 = (int64_t)bj * FT;
      const int ni = (int)min((int64_t)FT, N - I0);
      const int nj = (int)min((int64_t)FT, N - J0);
      const int jj = 8 * warp + 2 * c;
      const double* src = X + I0 * ldx + J0 + jj;
      const bool vec = with_ik1 && ni == FT && nj == FT && (ldx & 1) == 0 &&
                       (reinterpret_cast<uintptr_t>(X + J0) & 15) == 0;
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) {
        const int ii = 8 * ib + r;
        if (vec) {
          const double2 v = ld_cs_v2(src + ii * ldx);
          t[ib][0] = v.x;
          t[ib][1] = v.y;
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e)
            t[ib][e] = (with_ik1 && ii < ni && jj + e < nj) ? ld_cs(src + ii * ldx + e) : 0.0;
        }
      }
    };
    int bi, bj;
    pair_of(0, bi, bj);
    if (et == 0)
      for (int o = 0; o < 2; ++o)
        x5_window<P>(smem + o * L::ZW, Zext, N, x5_gmin<P>(o, bi, bj), wfull + o);
    double acc[8][2], nxt[8][2];
    load_ik1(bi, bj, nxt);
    for (int64_t k = 0; k < mine; ++k) {
      int nbi = 0, nbj = 0;
      const bool more = k + 1 < mine;
      if (more) pair_of(k + 1, nbi, nbj);
      // first rows of the next pair's windows, reduced now so that the requests below are short
      int64_t g0n[2] = {0, 0};
      if (et == 0 && more)
        for (int o = 0; o < 2; ++o) g0n[o] = pmod(x5_gmin<P>(o, nbi, nbj), N);
      XW_TL(15);
      const int64_t I0 = (int64_t)bi * FT, J0 = (int64_t)bj * FT;
      const int ni = (int)min((int64_t)FT, N - I0);
      const int nj = (int)min((int64_t)FT, N - J0);
      // band B fragments of both orientations: bS[o][s] = alpha S_{C0 + 8 warp + r}[4 s + c - r]
      double bS[2][KS4];
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const int64_t C0 = o == 0 ? J0 : I0;
        const int nc = o == 0 ? nj : ni;
        const int row = 8 * warp + r;
#pragma unroll
        for (int s2 = 0; s2 < KS4; ++s2) {
          const int t = 4 * s2 + c - r;
          bS[o][s2] = (t >= 0 && t <= 2 * C::D && row < nc) ? ld_nc(sw + (C0 + row) * C::WS + t) : 0.0;
        }
      }
      auto contract = [&](const int o) {
        XW_TL(16 + 3 * o);
        mbar_wait(pfull + o, (unsigned)(k & 1));
        // Phs[o] full: every Phi warp has read window o, so it can be refilled for the next pair
        if (et == 0 && more) x5_window_at<P>(smem + o * L::ZW, Zext, N, g0n[o], wfull + o);
        XW_TL(17 + 3 * o);
        const double* ph = smem + 2 * L::ZW + o * L::PH;
#pragma unroll
        for (int rb = 0; rb < 8; ++rb) {
#pragma unroll
          for (int s2 = 0; s2 < KS4; ++s2) {
            const double a = ph[(8 * rb + r) * PSTRIDE + 8 * warp + 4 * s2 + c];
            dmma(acc[rb][0], acc[rb][1], a, bS[o][s2]);
          }
        }
        warp_arrive(pempty + o);
        XW_TL(18 + 3 * o);
      };
      {
        // the tile was requested before the previous pair's stores
        const double aw = alpha * w_ik1;
#pragma unroll
        for (int rb = 0; rb < 8; ++rb) {
          acc[rb][0] = nxt[rb][0] * aw;
          acc[rb][1] = nxt[rb][1] * aw;
        }
#pragma unroll
        for (int o = 0; o < 2; ++o)
#pragma unroll
          for (int s2 = 0; s2 < KS4; ++s2) bS[o][s2] *= alpha;
      }
      contract(0);
      // T[i][j] (i = 8 rb + r, j = 8 warp + 2c + e) -> acc of orientation 1: lane
      // (j = 8 rb + r, i = 8 warp + 2c + e) starts from T[i][j]
#pragma unroll
      for (int rb = 0; rb < 8; ++rb)
        *reinterpret_cast<double2*>(Tsm + (8 * rb + r) * X5_TS + 8 * warp + 2 * c) =
            make_double2(acc[rb][0], acc[rb][1]);
      named_sync(XW_BAR_EPI, 256);
#pragma unroll
      for (int rb = 0; rb < 8; ++rb)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[rb][e] = Tsm[(8 * warp + 2 * c + e) * X5_TS + 8 * rb + r];
      named_sync(XW_BAR_EPI, 256);               // T read before the next pair overwrites it
      contract(1);
      // the next pair's IK1 tile: its HBM latency hides under the stores below
      if (more) load_ik1(nbi, nbj, nxt);

      // acc[rb][e] = A(J,I)[j = 8 rb + r][i = 8 warp + 2c + e]: rows J and, transposed, rows I
      const int i = 8 * warp + 2 * c;
      const bool full = ni == FT && nj == FT && (ldx & 1) == 0 &&
                        (reinterpret_cast<uintptr_t>(X + I0) & 15) == 0;
      if (bi != bj) {
#pragma unroll
        for (int rb = 0; rb < 8; ++rb) {
          const int j = 8 * rb + r;
          double* rowJ = X + (J0 + j) * ldx + I0 + i;
          if (full) {
            __stcs(reinterpret_cast<double2*>(rowJ), make_double2(acc[rb][0], acc[rb][1]));
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (j < nj && i + e < ni) __stcs(rowJ + e, acc[rb][e]);
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int rb = 0; rb < 8; ++rb) {
            const int j = 8 * rb + r;
            if (j < nj && i + e < ni) __stcs(X + (I0 + i + e) * ldx + J0 + j, acc[rb][e]);
          }
      } else {
#pragma unroll
        for (int rb = 0; rb < 8; ++rb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = 8 * rb + r;
            if (j < nj && i + e < ni && i + e <= j) {
              __stcs(X + (J0 + j) * ldx + I0 + i + e, acc[rb][e]);
              __stcs(X + (I0 + i + e) * ldx + J0 + j, acc[rb][e]);
            }
          }
      }
      XW_TL(22);
      bi = nbi;
      bj = nbj;
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

// self-test hooks: fast ln vs libdevice, and a DMMA fragment-layout check
__global__ void selftest_log_kernel(int64_t n, const double* x, double* out_fast, double* out_ref) {
  __shared__ double2 tab[64];  // the ln of the C4 IK1 kernel (ik1_sym_kernel)
  for (int k = threadIdx.x; k < 128; k += blockDim.x) reinterpret_cast<double*>(tab)[k] = kTang64[k];
  __syncthreads();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out_fast[i] = half_ln64t(x[i], tab);
  out_ref[i] = 0.5 * log(x[i]);
}

__global__ void selftest_dmma_kernel(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  double c0 = 0.0, c1 = 0.0;
  dmma(c0, c1, A[r * 4 + c], B[c * 8 + r]);
  C[r * 8 + 2 * c] = c0;
  C[r * 8 + 2 * c + 1] = c1;
}

template <int P, int MODE>
static int launch_ik1(const wq_smooth_t* sm, double* X, int64_t ldx, int* flag, cudaStream_t st,
                      int tile_row0, int tile_row1, int64_t pair0, int64_t pair1,
                      const int64_t* plist) {
  using C = Ik4Cfg<P, MODE>;
  if (sm->wg != C::WG) {
    set_error("wq_ik1_sym: rule band width %lld != 2p+1", (long long)sm->wg);
    return WQ_EINVAL;
  }
  const size_t smem = (size_t)Ik4Cfg<P, MODE>::TOTAL * 8;
  auto kern = ik1_sym_kernel<P, MODE, 0>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nb = ceil_div(sm->n_rows, FT);
  const int64_t all = (int64_t)nb * (nb + 1) / 2;
  if (pair1 < 0 || pair1 > all) pair1 = all;
  if (pair0 < 0) pair0 = 0;
  const int64_t blocks = tile_row0 < 0 ? pair1 - pair0 : (int64_t)(tile_row1 - tile_row0) * nb;
  if (blocks <= 0) return WQ_OK;
  kern<<<(unsigned)blocks, IK4_THREADS, smem, st>>>(*sm, nb, tile_row0, pair0, plist, X, ldx, flag);
  return check_launch("wq_ik1_sym");
}

// fewer pairs than this go to the one-pair-per-CTA kernel (two CTAs per SM); from 4 pairs
// per SM on, the persistent kernel is at least as fast at every size measured (N = 2048 .. 32768)
constexpr int64_t X2WS_MIN_PAIRS = 592;

template <int P>
static int launch_x2(int64_t N, const double* Uext, const double* Zext, const double* s_w,
                     double alpha, double w_ik1, double* X, int64_t ldx, cudaStream_t st,
                     int tile_row0, int tile_row1, int64_t pair0, int64_t pair1,
                     const int64_t* plist) {
  const int nb = ceil_div(N, FT);
  const int64_t all = (int64_t)nb * (nb + 1) / 2;
  if (pair1 < 0 || pair1 > all) pair1 = all;
  if (pair0 < 0) pair0 = 0;
  const int64_t blocks = tile_row0 < 0 ? pair1 - pair0 : (int64_t)(tile_row1 - tile_row0) * nb;
  if (blocks <= 0) return WQ_OK;
  // full sweeps of the upper triangle: the warp-specialised persistent kernel, one CTA per SM
  if (tile_row0 < 0 && N >= X2Cfg<P>::ZROWS && blocks >= X2WS_MIN_PAIRS) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)XwSmem<P>::TOTAL * 8;
    cudaFuncSetAttribute(x2ws_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned grid = (unsigned)std::min<int64_t>(blocks, sms);
    x2ws_kernel<P><<<grid, XW_THREADS, smem, st>>>(N, Uext, Zext, s_w, alpha, w_ik1, X, ldx, nb,
                                                   pair0, blocks, plist);
    return check_launch("wq_x2_pairs");
  }
#ifdef WQ_X2_ONE_CTA   // tools build only: one CTA per SM (occupancy experiment)
  const size_t smem = 120 * 1024;
#else
  const size_t smem = (size_t)X4Smem<P>::TOTAL * 8;
#endif
  cudaFuncSetAttribute(x2v4_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  x2v4_kernel<P><<<(unsigned)blocks, X2_THREADS, smem, st>>>(N, Uext, Zext, s_w, alpha, w_ik1, X,
                                                             ldx, nb, tile_row0, pair0, plist);
  return check_launch("wq_x2_pairs");
}

}  // namespace wq

using namespace wq;

extern "C" {

static int ik1_dispatch(const wq_smooth_t* sm, double* X, int64_t ldx, int* flag, void* stream,
                        int tile_row0, int tile_row1, int64_t pair0 = -1, int64_t pair1 = -1,
                        const int64_t* plist = nullptr) {
  if (!sm || !X || !flag || sm->n_rows <= 0 || !sm->closed) {
    set_error("wq_ik1_sym: bad arguments (closed uniform meshes only)");
    return WQ_EINVAL;
  }
  if (sm->near_k > 0) {
    set_error("wq_ik1_sym: near-diagonal node pairs need wq_ik1");
    return WQ_EUNSUPPORTED;
  }
  if (sm->k1_mode == WQ_K1_TABLE && !sm->invp2) {
    set_error("wq_ik1_sym: table mode without invp2");
    return WQ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int p = (int)(sm->wg - 1) / 2;
  const bool tab = sm->k1_mode == WQ_K1_TABLE;
#define WQ_IK1_CASE(PP)                                                                          \
  case PP:                                                                                       \
    return tab ? launch_ik1<PP, WQ_K1_TABLE>(sm, X, ldx, flag, st, tile_row0, tile_row1, pair0, pair1, plist) \
               : launch_ik1<PP, WQ_K1_CLOSED>(sm, X, ldx, flag, st, tile_row0, tile_row1, pair0, pair1, plist);
  switch (p) {
    WQ_IK1_CASE(2)
    WQ_IK1_CASE(3)
    WQ_IK1_CASE(4)
    WQ_IK1_CASE(5)
    default:
      set_error("wq_ik1_sym: degree %d unsupported (2..5)", p);
      return WQ_EUNSUPPORTED;
  }
#undef WQ_IK1_CASE
}

int wq_ik1_sym(const wq_smooth_t* sm, double* X, int64_t ldx, int64_t max_span, int* flag,
               void* stream) {
  (void)max_span;
  return ik1_dispatch(sm, X, ldx, flag, stream, -1, -1);
}

int wq_ik1_pairs(const wq_smooth_t* sm, int64_t pair0, int64_t pair1, double* X, int64_t ldx,
                 int* flag, void* stream) {
  return ik1_dispatch(sm, X, ldx, flag, stream, -1, -1, pair0, pair1);
}

int wq_ik1_rows(const wq_smooth_t* sm, int64_t tile_row0, int64_t tile_row1, double* Xrows,
                int64_t ldx, int* flag, void* stream) {
  if (!sm || tile_row0 < 0 || tile_row1 <= tile_row0 ||
      tile_row1 > ceil_div(sm->n_rows, FT)) {
    set_error("wq_ik1_rows: bad tile rows");
    return WQ_EINVAL;
  }
  return ik1_dispatch(sm, Xrows, ldx, flag, stream, (int)tile_row0, (int)tile_row1);
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

static int x2_dispatch(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                       const double* Uext, const double* Zext, const double* s_w, double alpha,
                       double w_ik1, double* X, int64_t ldx, void* stream, int tile_row0,
                       int tile_row1, int64_t pair0 = -1, int64_t pair1 = -1,
                       const int64_t* plist = nullptr) {
  if (N <= 0 || !Uext || !Zext || !s_w || !X) {
    set_error("wq_x2_pairs: bad arguments");
    return WQ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
#define WQ_X2_CASE(PP)                                                                         \
  case PP:                                                                                     \
    if (nA != X2Cfg<PP>::NA || nApad != X2Cfg<PP>::NAPAD || ws != X2Cfg<PP>::WS ||              \
        ktot != X2Cfg<PP>::KTOT || zstride != X2Cfg<PP>::ZSTRIDE) {                             \
      set_error("wq_x2_pairs: layout mismatch for p=%d", PP);                                  \
      return WQ_EINVAL;                                                                        \
    }                                                                                          \
    return launch_x2<PP>(N, Uext, Zext, s_w, alpha, w_ik1, X, ldx, st, tile_row0, tile_row1, \
                         pair0, pair1, plist);
  switch (p) {
    WQ_X2_CASE(2)
    WQ_X2_CASE(3)
    WQ_X2_CASE(4)
    WQ_X2_CASE(5)
    default:
      set_error("wq_x2_pairs: degree %d unsupported (2..5)", p);
      return WQ_EUNSUPPORTED;
  }
#undef WQ_X2_CASE
}

int wq_x2_pairs(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                const double* Uext, const double* Zext, const double* s_w, double alpha,
                double w_ik1, double* X, int64_t ldx, void* stream) {
  return x2_dispatch(N, p, nA, nApad, ws, ktot, zstride, Uext, Zext, s_w, alpha, w_ik1, X, ldx,
                     stream, -1, -1);
}

int wq_x2_pairs_range(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                      const double* Uext, const double* Zext, const double* s_w, double alpha,
                      double w_ik1, int64_t pair0, int64_t pair1, double* X, int64_t ldx,
                      void* stream) {
  return x2_dispatch(N, p, nA, nApad, ws, ktot, zstride, Uext, Zext, s_w, alpha, w_ik1, X, ldx,
                     stream, -1, -1, pair0, pair1);
}

int wq_x2_rows(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
               const double* Uext, const double* Zext, const double* s_w, double alpha,
               double w_ik1, int64_t tile_row0, int64_t tile_row1, double* Xrows, int64_t ldx,
               void* stream) {
  if (tile_row0 < 0 || tile_row1 <= tile_row0 || tile_row1 > ceil_div(N, FT)) {
    set_error("wq_x2_rows: bad tile rows");
    return WQ_EINVAL;
  }
  return x2_dispatch(N, p, nA, nApad, ws, ktot, zstride, Uext, Zext, s_w, alpha, w_ik1, Xrows, ldx,
                     stream, (int)tile_row0, (int)tile_row1);
}

int wq_ik1_pair_list(const wq_smooth_t* sm, const int64_t* plist, int64_t npairs, double* X,
                     int64_t ldx, int* flag, void* stream) {
  if (!plist || npairs < 0) {
    set_error("wq_ik1_pair_list: bad pair list");
    return WQ_EINVAL;
  }
  if (npairs == 0) return WQ_OK;
  return ik1_dispatch(sm, X, ldx, flag, stream, -1, -1, 0, npairs, plist);
}

int wq_x2_pair_list(int64_t N, int p, int nA, int nApad, int ws, int ktot, int zstride,
                    const double* Uext, const double* Zext, const double* s_w, double alpha,
                    double w_ik1, const int64_t* plist, int64_t npairs, double* X, int64_t ldx,
                    void* stream) {
  if (!plist || npairs < 0) {
    set_error("wq_x2_pair_list: bad pair list");
    return WQ_EINVAL;
  }
  if (npairs == 0) return WQ_OK;
  return x2_dispatch(N, p, nA, nApad, ws, ktot, zstride, Uext, Zext, s_w, alpha, w_ik1, X, ldx,
                     stream, -1, -1, 0, npairs, plist);
}

int wq_selftest_log(int64_t n, const double* x, double* out_fast, double* out_ref, void* stream) {
  selftest_log_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(n, x, out_fast, out_ref);
  return check_launch("wq_selftest_log");
}

#ifdef WQ_X2_TIMELINE
int wq_debug_x2_timeline(long long* buf) {
  cudaError_t e = cudaMemcpyToSymbol(g_x2_tl, &buf, sizeof(buf));
  return e == cudaSuccess ? WQ_OK : WQ_ECUDA;
}
#endif

int wq_selftest_dmma(const double* A, const double* B, double* C, void* stream) {
  selftest_dmma_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(A, B, C);
  return check_launch("wq_selftest_dmma");
}

}  // extern "C"
