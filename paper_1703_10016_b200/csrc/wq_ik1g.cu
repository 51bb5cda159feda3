// IK1 for irregular rule bands (open meshes, graded elements, repeated knots):
// the register sliding-window scheme of ik1_sym (wq_fast.cu) with per-rule
// starts.  Replaces assemble_ik1 (assembly.py:175-183) with the K1 grid of
// geometry.py:225-248 evaluated in registers:
//   IK1[i, j] = sum_q sum_r G[i,q] K1(eta_q, eta_r) G[j,r],
// rule i on nodes g_start[i] .. g_start[i] + WG - 1 (zero-padded weights).
// One CTA per 64 x 64 tile pair; phase 1: thread (outer node q, column half)
// slides a WG-wide window of K1(q, r) along r, emitting T1[j][q] =
// sum_w K1(q, g_start[j] + w) G[j][w] whenever the window reaches the end of
// rule j; phase 2: thread (column j, row quarter) slides along q to form
// IK1[i][j] = sum_w G[i][w] T1[j][g_start[i] + w].  Starts are nondecreasing,
// so every K1 pair of the tile's node ranges is evaluated once per column half.
#include "wq_common.cuh"
#include "wq_log.cuh"

namespace wq {

constexpr int IG_THREADS = 288;
constexpr int IG_HALF = IG_THREADS / 2;   // max node span of a 64-row tile
constexpr int IG_T = WQ_FTILE;            // 64

// upper-triangle tile pair index -> (bi, bj), bi <= bj, row bi holds nb - bi pairs
__device__ __forceinline__ void tri_index_g(int64_t t, int nb, int& bi, int& bj) {
  const double B = 2.0 * nb + 1.0;
  int b = (int)floor((B - sqrt(B * B - 8.0 * (double)t)) * 0.5);
  if (b < 0) b = 0;
  if (b > nb - 1) b = nb - 1;
  auto start = [nb](int64_t x) { return x * nb - x * (x - 1) / 2; };
  while (b > 0 && start(b) > t) --b;
  while (b + 1 < nb && start(b + 1) <= t) ++b;
  bi = b;
  bj = b + (int)(t - start(b));
}

template <int MODE>
__device__ __forceinline__ double k1g(const wq_smooth_t& sm, double qx, double qy, int qa,
                                      double qJ, double qs, double rx, double ry, int ra,
                                      double rs, const double2* tab, int& bad) {
  double R;
  if (qa == ra) {
    R = qJ * qJ;  // continuity limit J^2 (geometry.py:240-245)
  } else if (sm.near_k > 0 && near_pair_j2(sm, qa, ra, &R)) {
    // distinct nodes within eps_diag: J(mid)^2 (geometry.py:237-245)
  } else {
    const double dx = qx - rx, dy = qy - ry;
    const double d2 = fma(dx, dx, dy * dy);
    if (MODE == WQ_K1_TABLE) {
      R = d2 * __ldg(sm.invp2 + (qa > ra ? qa - ra : ra - qa));
    } else if (MODE == WQ_K1_OPEN) {
      const double p = rs - qs;
      R = d2 / (p * p);
    } else {
      const double xx = fabs(rs - qs);   // periodic distance from the UNWRAPPED |t - s|
      const double p = (sm.period / kPi) * fabs(sin(kPi * xx / sm.period));
      R = d2 / (p * p);
    }
  }
  if (!(R > 0.0) || !(R < 1.0e300)) {
    bad = 1;
    return 0.0;
  }
  return half_ln64t(R, tab);
}

// sym: upper tile pairs (bi <= bj) of the full matrix, mirrored; rect: tile rows
// [tile_row0, ...) x all tile columns, rows offset by tile_row0 * 64
template <int WG, int MODE>
__global__ void __launch_bounds__(IG_THREADS, 2)
ik1g_kernel(wq_smooth_t sm, int nb, int tile_row0, int sym, double* X, int64_t ldx, int* flag) {
  extern __shared__ double dsm[];
  int bi, bj;
  if (sym) {
    tri_index_g(blockIdx.x, nb, bi, bj);
  } else {
    bi = tile_row0 + (int)(blockIdx.x / nb);
    bj = (int)(blockIdx.x % nb);
  }
  const int64_t row_off = sym ? 0 : (int64_t)tile_row0 * IG_T;
  const int64_t N = sm.n_rows, nq = sm.nq;
  const int64_t I0 = (int64_t)bi * IG_T, J0 = (int64_t)bj * IG_T;
  const int ni = (int)min((int64_t)IG_T, N - I0);
  const int nj = (int)min((int64_t)IG_T, N - J0);
  const int64_t qlo = sm.g_start[I0], rlo = sm.g_start[J0];
  const int nQ = (int)(sm.g_start[I0 + ni - 1] + WG - qlo);
  const int nR = (int)(sm.g_start[J0 + nj - 1] + WG - rlo);
  constexpr int NQP = IG_HALF | 1;
  double2* stab = reinterpret_cast<double2*>(dsm);   // [64] ln table (16-byte aligned)
  double* T1 = dsm + 128;                // [64][NQP]
  double* qx = T1 + IG_T * NQP;          // node data, outer range
  double* qy = qx + IG_HALF;
  double* qJ = qy + IG_HALF;
  double* qs = qJ + IG_HALF;
  double* rx = qs + IG_HALF;             // inner range
  double* ry = rx + IG_HALF;
  double* rJ = ry + IG_HALF;
  double* rs = rJ + IG_HALF;
  double (*Gi)[WG] = reinterpret_cast<double (*)[WG]>(rs + IG_HALF);
  double (*Gj)[WG] = reinterpret_cast<double (*)[WG]>(rs + IG_HALF + IG_T * WG);
  int* qa = reinterpret_cast<int*>(rs + IG_HALF + 2 * IG_T * WG);
  int* ra = qa + IG_HALF;
  int* si = ra + IG_HALF;                // rule starts of the tile rows, relative to qlo
  int* sj = si + IG_T;                   // ... of the tile columns, relative to rlo
  const int tid = threadIdx.x;
  for (int k = tid; k < IG_HALF; k += IG_THREADS) {
    if (k < nQ) {
      int64_t a = pmod(qlo + k, nq);
      qa[k] = (int)a;
      qx[k] = sm.fx[a]; qy[k] = sm.fy[a]; qJ[k] = sm.J[a]; qs[k] = sm.s[a];
    }
    if (k < nR) {
      int64_t b = pmod(rlo + k, nq);
      ra[k] = (int)b;
      rx[k] = sm.fx[b]; ry[k] = sm.fy[b]; rJ[k] = sm.J[b]; rs[k] = sm.s[b];
    }
  }
  for (int k = tid; k < IG_T * WG; k += IG_THREADS) {
    const int ii = k / WG, w = k - ii * WG;
    Gi[ii][w] = ii < ni ? sm.g_w[(I0 + ii) * WG + w] : 0.0;
    Gj[ii][w] = ii < nj ? sm.g_w[(J0 + ii) * WG + w] : 0.0;
  }
  for (int k = tid; k < IG_T; k += IG_THREADS) {
    si[k] = k < ni ? (int)(sm.g_start[I0 + k] - qlo) : nQ - WG;
    sj[k] = k < nj ? (int)(sm.g_start[J0 + k] - rlo) : nR - WG;
  }
  for (int k = tid; k < 128; k += IG_THREADS) reinterpret_cast<double*>(stab)[k] = kTang64[k];
  __syncthreads();

  int bad = 0;
  // phase 1: (q, half) -> T1[j][q] for the 32 columns j of the half
  {
    const int h = tid >= IG_HALF ? 1 : 0;
    const int q = tid - h * IG_HALF;
    if (q < nQ) {
      const double mx = qx[q], my = qy[q], mJ = qJ[q], ms = qs[q];
      const int ma = qa[q];
      double win[WG];
#pragma unroll
      for (int w = 0; w < WG; ++w) win[w] = 0.0;
      const int j0 = 32 * h;
      int r = sj[j0] - 1;   // last evaluated inner node (window ends there)
      for (int jj = 0; jj < 32; ++jj) {
        const int j = j0 + jj;
        const int end = sj[j] + WG - 1;
        while (r < end) {
          ++r;
#pragma unroll
          for (int w = 0; w < WG - 1; ++w) win[w] = win[w + 1];
          win[WG - 1] = k1g<MODE>(sm, mx, my, ma, mJ, ms, rx[r], ry[r], ra[r], rs[r], stab, bad);
        }
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < WG; ++w) acc = fma(win[w], Gj[j][w], acc);
        T1[j * NQP + q] = acc;
      }
    }
  }
  __syncthreads();
  // phase 2: (j, quarter) -> IK1[i][j], i in 16c .. 16c+15
  if (tid < 4 * IG_T) {
    const int j = tid & (IG_T - 1), c = tid >> 6;
    const double* t = T1 + j * NQP;
    const int i0 = 16 * c;
    double win[WG];
#pragma unroll
    for (int w = 0; w < WG; ++w) win[w] = 0.0;
    int q = si[i0] - 1;
    for (int ii = 0; ii < 16; ++ii) {
      const int i = i0 + ii;
      const int end = si[i] + WG - 1;
      while (q < end) {
        ++q;
#pragma unroll
        for (int w = 0; w < WG - 1; ++w) win[w] = win[w + 1];
        win[WG - 1] = t[q];
      }
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < WG; ++w) acc = fma(Gi[i][w], win[w], acc);
      if (i < ni && j < nj) {
        X[(I0 - row_off + i) * ldx + J0 + j] = acc;
        if (sym && bj > bi) X[(J0 + j) * ldx + I0 + i] = acc;   // IK1 is symmetric
      }
    }
  }
  if (bad) atomicOr(flag, WQ_FLAG_R_NONPOSITIVE);
}

}  // namespace wq

using namespace wq;

extern "C" int wq_ik1_band(const wq_smooth_t* sm, int64_t tile_row0, int64_t tile_row1, double* X,
                           int64_t ldx, int64_t span64, int* flag, void* stream) {
  const int nb = sm ? ceil_div(sm->n_rows, IG_T) : 0;
  if (!sm || !X || !flag || sm->n_rows <= 0 || tile_row0 < -1 || tile_row1 > nb ||
      (tile_row0 >= 0 && tile_row1 <= tile_row0)) {
    set_error("wq_ik1_band: bad arguments");
    return WQ_EINVAL;
  }
  if (span64 > IG_HALF || sm->wg < 2 || sm->wg > 16) {
    set_error("wq_ik1_band: node span %lld / rule width %lld outside the kernel's range",
              (long long)span64, (long long)sm->wg);
    return WQ_EUNSUPPORTED;
  }
  if (sm->k1_mode == WQ_K1_TABLE && !sm->invp2) {
    set_error("wq_ik1_band: table mode without invp2");
    return WQ_EINVAL;
  }
  const int sym = tile_row0 < 0;
  const int64_t blocks = sym ? (int64_t)nb * (nb + 1) / 2 : (tile_row1 - tile_row0) * nb;
  const int wg = (int)sm->wg;
  const size_t smem = ((size_t)IG_T * (IG_HALF | 1) + 8 * IG_HALF + 2 * IG_T * wg + 128) * 8 +
                      (size_t)(2 * IG_HALF + 2 * IG_T) * 4;
  cudaStream_t st = (cudaStream_t)stream;
  const int mode = (int)sm->k1_mode;
#define WQ_IG_LAUNCH(W, M)                                                                      \
  {                                                                                             \
    cudaFuncSetAttribute(ik1g_kernel<W, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                         (int)smem);                                                            \
    ik1g_kernel<W, M><<<(unsigned)blocks, IG_THREADS, smem, st>>>(                             \
        *sm, nb, (int)tile_row0, sym, X, ldx, flag);                                           \
  }
#define WQ_IG_CASE(W)                                                                           \
  case W:                                                                                       \
    if (mode == WQ_K1_TABLE) WQ_IG_LAUNCH(W, WQ_K1_TABLE)                                       \
    else if (mode == WQ_K1_OPEN) WQ_IG_LAUNCH(W, WQ_K1_OPEN)                                    \
    else WQ_IG_LAUNCH(W, WQ_K1_CLOSED)                                                          \
    break;
  switch (wg) {
    WQ_IG_CASE(2) WQ_IG_CASE(3) WQ_IG_CASE(4) WQ_IG_CASE(5) WQ_IG_CASE(6) WQ_IG_CASE(7)
    WQ_IG_CASE(8) WQ_IG_CASE(9) WQ_IG_CASE(10) WQ_IG_CASE(11) WQ_IG_CASE(12) WQ_IG_CASE(13)
    WQ_IG_CASE(14) WQ_IG_CASE(15) WQ_IG_CASE(16)
  }
#undef WQ_IG_CASE
#undef WQ_IG_LAUNCH
  return check_launch("wq_ik1_band");
}
