// Non-uniform meshes (graded elements, any knot multiplicity; config 5):
// element-pair Theta / D blocks computed per pair on the device, then gathered
// into Theta^T (N_E x N) and D (N_E x N_E) for the general fit path.
//
// The reference supports only uniform meshes here (quadrature.py:489-491
// raises).  Its unit-width recipe (quadrature.py:441-504) is generalised per
// pair (restated in oracle/wq_oracle.py::pair_moments_general):
//   near pairs (touching / overlapping, as the reference's |gap| <= 1 entries,
//     quadrature.py:458; listed by the host): closed-form moments
//     (quadrature.py:372-410) in width-normalised coordinates (h_e = 1,
//     h_f = rho, delta' = delta / h_e), scaled by
//     M = h_e^(a+b+2) (M' + ln h_e c_a C_b(rho)), then contracted;
//   far pairs: tensor Gauss (quadrature.py:413-438) applied directly to the
//     contracted integrand  int int U_e(x) log|y - x| V_f(y),  U_e / V_f the
//     element polynomials of the coarse (times fitted J) and fine functions --
//     algebraically the same as contracting the Gauss moments, with the order
//     tiered by separation (30 below two widths, as the reference; 16 below
//     eight; 12 beyond -- all converged to rounding for the degree <= 16 x 5
//     polynomials involved).
// Closed meshes add the periodic gap term log|sinc(r / L)| (quadrature.py:
// 459-468) -- far pairs use log|L/pi sin(pi r / L)|, its exact sum with log|r|.
// Every output is a fixed-order sum (deterministic; no atomics).
#include <algorithm>

#include "wq_common.cuh"
#include "wq_log.cuh"

namespace wq {

constexpr int GMAXA = 24;   // max row polynomial degree + 1 (P + 1)
constexpr int GMAXB = 8;    // max column degree + 1
constexpr int GMAXP = GMAXA + GMAXB;
constexpr int GT0 = 30, GT1 = 16, GT2 = 12;   // Gauss tiers
constexpr int GTSUM = GT0 + GT1 + GT2;

__constant__ double c_binom[GMAXP][GMAXP];
static bool g_consts_ready[64];

static int ensure_consts() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && g_consts_ready[dev]) return WQ_OK;
  static double b[GMAXP][GMAXP];
  for (int n = 0; n < GMAXP; ++n) {
    b[n][0] = 1.0;
    for (int k = 1; k <= n; ++k) b[n][k] = b[n - 1][k - 1] + (k <= n - 1 ? b[n - 1][k] : 0.0);
  }
  cudaError_t e = cudaMemcpyToSymbol(c_binom, b, sizeof(b));
  if (e != cudaSuccess) {
    set_error("constant upload: %s", cudaGetErrorString(e));
    return WQ_ECUDA;
  }
  if (dev >= 0 && dev < 64) g_consts_ready[dev] = true;
  return WQ_OK;
}

// [z^{j+1}/(j+1) (ln|z| - 1/(j+1))], limit 0 at z = 0 (quadrature.py:182-197)
__device__ __forceinline__ double log_bracket(int j, double zp1, double lz, bool zero) {
  return zero ? 0.0 : zp1 / (j + 1) * (lz - 1.0 / (j + 1));
}

// Closed-form unit-normalised moments (he = 1, hf = rho, delta = dl) added into
// out[a * ldo + b] (quadrature.py:372-410, same summation structure).
__device__ void pair_closed(int da, int db, double rho, double dl, double* out, int ldo) {
  const int pmax = da + db + 1;
  for (int s = 0; s < 2; ++s) {
    const double sgn = s == 0 ? 1.0 : -1.0;
    const double xi = sgn * 0.5 * rho;
    const double z1 = xi - dl - 0.5, z2 = xi - dl + 0.5;
    const bool z1z = z1 == 0.0, z2z = z2 == 0.0;
    const double l1 = z1z ? 0.0 : log(fabs(z1)), l2 = z2z ? 0.0 : log(fabs(z2));
    double llog[GMAXP + 1], lpow[GMAXP + 1];
    double p1 = z1, p2 = z2;  // z^(p+1)
    for (int p = 0; p <= pmax; ++p) {
      llog[p] = log_bracket(p, p2, l2, z2z) - log_bracket(p, p1, l1, z1z);
      lpow[p] = (p2 - p1) / (p + 1);
      p1 *= z1;
      p2 *= z2;
    }
    const double xd = xi - dl;
    for (int b = 0; b <= db; ++b) {
      for (int m = 0; m <= b; ++m) {
        const double cm = sgn * c_binom[b][m] / (m + 1);
        for (int a = 0; a <= da; ++a) {
          double acc = 0.0;
          for (int r = 0; r <= a; ++r) {
            double t = 1.0;  // (xi - delta)^(a - r)
            for (int k = 0; k < a - r; ++k) t *= xd;
            for (int q = 0; q <= b - m; ++q) {
              const int p = r + q + m + 1;
              double u = 1.0;  // xi^(b - m - q)
              for (int k = 0; k < b - m - q; ++k) u *= xi;
              const double sign = ((r + q) & 1) ? -1.0 : 1.0;
              const double coef = cm * c_binom[a][r] * c_binom[b - m][q] * sign * t * u;
              acc += coef * (llog[p] - lpow[p] / (m + 1));
            }
          }
          out[a * ldo + b] += acc;
        }
      }
    }
  }
}

struct GenArgs {
  int64_t n_el, e0, e1;     // all elements; chunk [e0, e1)
  int da, db, pu;           // P, d, coarse degree
  int closed;
  double period;
  const double* elh;        // (n_el) widths
  const double* elm;        // (n_el) midpoints
  const double* u;          // (n_el, da+1, pu+1) coarse coefficients (times fitted J)
  const double* v;          // (n_el, db+1, db+1) fine coefficients
  const int64_t* near_lo;   // (n_el) near pairs of e: f = near_lo[e] + k (mod n_el),
  const int64_t* near_cnt;  //        k < near_cnt[e]
  const double* near_unit;  // (3, da+1, db+1) unit closed-form table, dl = -1, 0, +1 (host)
  const double* touch;      // packed Duffy rules: x16 w16 x30 w30 on (0,1), xl14 wl14
  const double* gx;         // tier Gauss nodes on (-1/2, 1/2), 30 | 16 | 12 concatenated
  const double* gw;         // weights
  const double* m2u;        // (2 n_el - 1, da+1, db+1) UNIT gap table (open meshes) or NULL
  const double* ca;         // (da+1) unit centred integrals
  const double* cb;         // (db+1)
  double* wt;               // [f][a'][b'][e - e0] Theta blocks, leading dimension ldc
  double* wd;               // [f][a'][b'][e - e0] D blocks
  int64_t ldc;              // >= e1 - e0
  int* tile_flag;           // (n_el, ceil((e1-e0)/64)): tile holds off-table far pairs
  double* mg_out;           // near kernel, moments mode: (n_g, n_el, da+1, db+1) or NULL
  const int* gidx;          // (n_el) index in G or -1 (moments mode)
};

__device__ __forceinline__ double wrap_delta(const GenArgs& A, double d) {
  return A.closed ? d - A.period * rint(d / A.period) : d;
}

__device__ __forceinline__ bool is_near(const GenArgs& A, int64_t e, int64_t f) {
  int64_t k = f - A.near_lo[e];
  if (k < 0) k += A.n_el;
  return k < A.near_cnt[e];
}

// equal widths (to WIDTH_SNAP relative) at an integer offset: the reference's
// unit gap-table recipe applies (quadrature.py:452-456, 497-500); same
// predicate as oracle/wq_oracle.py::pair_moments_general
constexpr double WIDTH_SNAP = 1e-10;

__device__ __forceinline__ bool snapped_gap(double he, double hf, double delta, double* gap) {
  const double rho = hf / he;
  if (!(fabs(rho - 1.0) < WIDTH_SNAP)) return false;
  const double dl = delta / he, r = rint(dl);
  if (!(fabs(dl - r) < 1e-9 * fmax(1.0, fabs(dl)))) return false;  // relative: |dl| up to n_el
  *gap = -r;  // keff = f - e in element units
  return true;
}

constexpr int FP_THREADS = 64;

// Block layout (chunk-minor, so both the pair kernels' stores and the
// gathers' loads are coalesced): W[f][a'][b'][e - e0], leading dimension ldc.
__device__ __forceinline__ int64_t wslot(const GenArgs& A, int64_t f, int ab, int nab, int64_t ec) {
  return ((f * nab) + ab) * A.ldc + ec;
}

// Far pairs of snapped widths: unit moments from the gap table M' (row
// gap + n - 1), scaled M = h_e^(a+b+2) (M' + ln h_e c_a c_b) and contracted to
// the blocks.  One thread per outer element e, one inner element f per CTA.
template <int NP>
__global__ void __launch_bounds__(FP_THREADS, 8)
pair_table_kernel(GenArgs A) {
  const int nA = A.da + 1;
  const int64_t f = blockIdx.y;
  const int64_t eb = A.e0 + (int64_t)blockIdx.x * FP_THREADS;
  const int ne = (int)min((int64_t)FP_THREADS, A.e1 - eb);
  __shared__ double vf[NP][NP];
  __shared__ double cab[GMAXA * GMAXB];         // c_a c_b
  for (int k = threadIdx.x; k < NP * NP; k += FP_THREADS) vf[k / NP][k % NP] = A.v[f * NP * NP + k];
  for (int k = threadIdx.x; k < nA * NP; k += FP_THREADS) cab[k] = A.ca[k / NP] * A.cb[k % NP];
  const int64_t e = eb + threadIdx.x;
  const bool valid = threadIdx.x < ne && !is_near(A, e, f);
  const double he = valid ? A.elh[e] : 1.0;
  double gap = 0.0;
  const bool tab = valid && snapped_gap(he, A.elh[f], A.elm[e] - A.elm[f], &gap) &&
                   fabs(gap) <= (double)(A.n_el - 1);
  // tiles with off-table far pairs are left to pair_far_kernel
  const int need = __syncthreads_or(valid && !tab);
  if (threadIdx.x == 0) A.tile_flag[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = need;
  if (!tab) return;
  // the geometric offset selects the row (equal widths away from the
  // lattice of f, e.g. mirrored graded elements, read their own row); a
  // warp's rows are contiguous in the table (L1/L2 resident)
  const double* M = A.m2u + ((int64_t)gap + A.n_el - 1) * nA * NP;
  const double* ue = A.u + e * nA * NP;
  const double* ve = A.v + e * NP * NP;
  const double lh = log(he);
  double hb[NP];
  hb[0] = 1.0;
#pragma unroll
  for (int b = 1; b < NP; ++b) hb[b] = hb[b - 1] * he;
  double wT[NP][NP], wD[NP][NP];
#pragma unroll
  for (int a = 0; a < NP; ++a)
#pragma unroll
    for (int b = 0; b < NP; ++b) wT[a][b] = wD[a][b] = 0.0;
  double ha = he * he;
#pragma unroll 1
  for (int al = 0; al < nA; ++al, ha *= he) {
    double mv[NP];
#pragma unroll
    for (int bp = 0; bp < NP; ++bp) mv[bp] = 0.0;
#pragma unroll
    for (int be = 0; be < NP; ++be) {
      const double m = ha * hb[be] * (__ldg(M + al * NP + be) + lh * cab[al * NP + be]);
#pragma unroll
      for (int bp = 0; bp < NP; ++bp) mv[bp] = fma(m, vf[be][bp], mv[bp]);
    }
#pragma unroll
    for (int a = 0; a < NP; ++a) {
      const double u = __ldg(ue + al * NP + a);
#pragma unroll
      for (int bp = 0; bp < NP; ++bp) wT[a][bp] = fma(u, mv[bp], wT[a][bp]);
    }
    if (al < NP) {
#pragma unroll
      for (int a = 0; a < NP; ++a) {
        const double v = __ldg(ve + al * NP + a);
#pragma unroll
        for (int bp = 0; bp < NP; ++bp) wD[a][bp] = fma(v, mv[bp], wD[a][bp]);
      }
    }
  }
  const int64_t ec = e - A.e0;
#pragma unroll
  for (int a = 0; a < NP; ++a)
#pragma unroll
    for (int bp = 0; bp < NP; ++bp) {
      A.wt[wslot(A, f, a * NP + bp, NP * NP, ec)] = wT[a][bp];
      A.wd[wslot(A, f, a * NP + bp, NP * NP, ec)] = wD[a][bp];
    }
}

// Far pairs off the table: tensor Gauss on the contracted integrand, one
// thread per outer element e, the inner element f's weighted polynomial values
// at every tier's nodes in shared memory.  Persistent: a CTA keeps one block of 64
// outer elements and walks the inner elements f (with a gap table only the tiles
// pair_table_kernel flagged).  The outer polynomials at the far tier's nodes --
// w_g U_e(x_g), w_g V_e(x_g), the same for every f -- are evaluated once per CTA into
// shared memory (thread-minor): evaluating them per pair from global memory (85 + 25
// strided loads per node) bound the kernel by L1/L2 traffic.
template <int NP>
__global__ void __launch_bounds__(FP_THREADS)
pair_far_kernel(GenArgs A, int64_t nf, int nbx) {
  extern __shared__ double far_uv[];   // [GT2][2 NP][FP_THREADS]: far-tier w_g U_e, w_g V_e
  __shared__ double Vt[GTSUM][NP];   // h_f w_h V_f(h_f x_h)
  __shared__ double Yt[GTSUM];       // h_f x_h
  __shared__ double Gx[GTSUM], Gw[GTSUM];
  __shared__ double2 lntab[64];      // accurate-table ln (wq_log.cuh), open meshes
  const int nA = A.da + 1;
  for (int g = threadIdx.x; g < GTSUM; g += FP_THREADS) {
    Gx[g] = A.gx[g];
    Gw[g] = A.gw[g];
  }
  for (int k = threadIdx.x; k < 128; k += FP_THREADS) reinterpret_cast<double*>(lntab)[k] = kTang64[k];
  const int ebk = blockIdx.x % nbx;                 // this CTA's block of outer elements
  const int64_t e = A.e0 + (int64_t)ebk * FP_THREADS + threadIdx.x;
  const bool have_e = e < A.e1;
  const double he = have_e ? A.elh[e] : 1.0;
  const double* ue = A.u + (have_e ? e : A.e0) * nA * NP;
  const double* ve = A.v + (have_e ? e : A.e0) * NP * NP;
  // outer polynomials at node x (weight wx) of tier node g
  auto outer = [&](int g, double (&uu)[NP], double (&vv)[NP]) {
    const double x = he * Gx[g], wx = he * Gw[g];
#pragma unroll
    for (int a = 0; a < NP; ++a) {
      double s = 0.0;
      for (int al = nA - 1; al >= 0; --al) s = fma(s, x, __ldg(ue + al * NP + a));
      uu[a] = wx * s;
      s = 0.0;
#pragma unroll
      for (int al = NP - 1; al >= 0; --al) s = fma(s, x, __ldg(ve + al * NP + a));
      vv[a] = wx * s;
    }
  };
  __syncthreads();                                  // Gx / Gw visible
  if (have_e) {
    for (int g = 0; g < GT2; ++g) {
      double uu[NP], vv[NP];
      outer(GT0 + GT1 + g, uu, vv);
#pragma unroll
      for (int a = 0; a < NP; ++a) {
        far_uv[(g * 2 * NP + a) * FP_THREADS + threadIdx.x] = uu[a];
        far_uv[(g * 2 * NP + NP + a) * FP_THREADS + threadIdx.x] = vv[a];
      }
    }
  }
  for (int64_t f = blockIdx.x / nbx; f < nf; f += gridDim.x / nbx) {
    if (A.m2u && !A.tile_flag[f * nbx + ebk]) continue;
    __syncthreads();   // previous tile's tables are dead
    const double hf = A.elh[f];
    bool mine = have_e && !is_near(A, e, f);
    double gap;
    if (mine && A.m2u && snapped_gap(A.elh[e], hf, A.elm[e] - A.elm[f], &gap) &&
        fabs(gap) <= (double)(A.n_el - 1))
      mine = false;  // pair_table_kernel's
    for (int h = threadIdx.x; h < GTSUM; h += FP_THREADS) {
      const double y = hf * Gx[h], w = hf * Gw[h];
      Yt[h] = y;
#pragma unroll
      for (int bp = 0; bp < NP; ++bp) {
        double s = 0.0;
#pragma unroll
        for (int b = NP - 1; b >= 0; --b) s = fma(s, y, A.v[(f * NP + b) * NP + bp]);
        Vt[h][bp] = w * s;
      }
    }
    __syncthreads();
    if (mine) {
      const double delta = wrap_delta(A, A.elm[e] - A.elm[f]);
      const double sep = fabs(delta) - 0.5 * (he + hf);
      const double hm = fmax(he, hf);
      // Gauss order by separation in units of the larger width (measured:
      // <= 5e-15 of the natural slot scale at degree 16 x 4 for every tier)
      const int t0 = sep < 2.0 * hm ? 0 : (sep < 8.0 * hm ? GT0 : GT0 + GT1);
      const int ng = sep < 2.0 * hm ? GT0 : (sep < 8.0 * hm ? GT1 : GT2);
      const bool far = t0 == GT0 + GT1;
      double wT[NP][NP], wD[NP][NP];
#pragma unroll
      for (int a = 0; a < NP; ++a)
#pragma unroll
        for (int b = 0; b < NP; ++b) wT[a][b] = wD[a][b] = 0.0;
      const bool closed = A.closed;
      const double invL = closed ? 1.0 / A.period : 0.0;
      const double lnLpi = closed ? log(A.period / kPi) : 0.0;
      for (int g = 0; g < ng; ++g) {
        const double x = he * Gx[t0 + g];
        double uu[NP], vv[NP];
        if (far) {
#pragma unroll
          for (int a = 0; a < NP; ++a) {
            uu[a] = far_uv[(g * 2 * NP + a) * FP_THREADS + threadIdx.x];
            vv[a] = far_uv[(g * 2 * NP + NP + a) * FP_THREADS + threadIdx.x];
          }
        } else {
          outer(t0 + g, uu, vv);
        }
        const double base = -x - delta;   // r = y - x - delta
        double t[NP];
#pragma unroll
        for (int b = 0; b < NP; ++b) t[b] = 0.0;
        for (int h = 0; h < ng; ++h) {
          const double r = Yt[t0 + h] + base;
          // ln |r| by the accurate table (~1 ulp, a third of libdevice's FP64 work); r != 0 for
          // the separated pairs this kernel takes
          const double k = closed ? log(fabs(sinpi(r * invL))) + lnLpi : 2.0 * half_ln64t(fabs(r), lntab);
#pragma unroll
          for (int b = 0; b < NP; ++b) t[b] = fma(Vt[t0 + h][b], k, t[b]);
        }
#pragma unroll
        for (int a = 0; a < NP; ++a)
#pragma unroll
          for (int bp = 0; bp < NP; ++bp) {
            wT[a][bp] = fma(uu[a], t[bp], wT[a][bp]);
            wD[a][bp] = fma(vv[a], t[bp], wD[a][bp]);
          }
      }
      const int64_t ec = e - A.e0;
#pragma unroll
      for (int a = 0; a < NP; ++a)
#pragma unroll
        for (int bp = 0; bp < NP; ++bp) {
          A.wt[wslot(A, f, a * NP + bp, NP * NP, ec)] = wT[a][bp];
          A.wd[wslot(A, f, a * NP + bp, NP * NP, ec)] = wD[a][bp];
        }
    }
  }
}

// sum over quadrature nodes n < nnodes of w u^a v^b for every slot (a, b), the nodes dealt to
// the lanes of the warp and the NA x NB partial sums in registers, then a butterfly sum (all
// lanes end with the same totals); added to M[a NB + b] (shared, this warp's).  One pass of
// NA NB FMAs per node instead of a power loop per slot and node on one lane.
template <int NA, int NB, class NodeFn>
__device__ __forceinline__ void warp_node_moments(int nnodes, NodeFn node, double* M, int lane) {
  double m[NA][NB];
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) m[a][b] = 0.0;
  for (int n = lane; n < nnodes; n += 32) {
    double w, u, v;
    node(n, w, u, v);
    double ua = w;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      double t = ua;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        m[a][b] += t;
        t *= v;
      }
      ua *= u;
    }
  }
#pragma unroll
  for (int a = 0; a < NA; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      double x = m[a][b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == (a * NB + b) % 32) M[a * NB + b] += x;
    }
  __syncwarp();
}

constexpr int TOUCH_XI = 16, TOUCH_ETA = 30, TOUCH_LOG = 14;
constexpr int NP_WARPS = 4;

// Near (touching / overlapping) pairs, one warp per pair.  Unit moments M'
// (he = 1, hf = rho, delta' = dl) with the 85 (a, b) slots spread over the
// lanes:
//   rho == 1 at integer dl: the host's closed-form unit rows (the reference's
//     |gap| <= 1 entries, quadrature.py:372-410);
//   rho != 1 (touching): Duffy split at the shared corner -- with t, y the
//     distances from the corner, ln|v - u - dl| = ln(t + y); y <= rho t as
//     (xi, rho xi eta), y >= rho t as (xi eta, rho xi), Jacobian rho xi:
//     ln xi by the -ln-weighted rule, g = ln(1 + rho eta) | ln(rho + eta) by
//     Gauss-Legendre (exact in xi for the degree <= P + d + 1 polynomials;
//     g analytic for rho in [1/8, 8]);
//   closed meshes add the periodic term ln|sinc| by 30 x 30 Gauss.
// Then M = h_e^(a+b+2) (M' + ln h_e c_a C_b(rho)) and the contraction.
__global__ void __launch_bounds__(NP_WARPS * 32)
pair_near_kernel(GenArgs A, int max_near) {
  extern __shared__ double sh[];
  const int nA = A.da + 1, nB = A.db + 1, nU = A.pu + 1, ns = nA * nB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = A.e0 + blockIdx.y;
  const int k = blockIdx.x * NP_WARPS + warp;
  if (k >= A.near_cnt[e] || k >= max_near) return;
  int64_t f = A.near_lo[e] + k;
  if (f >= A.n_el) f -= A.n_el;
  double* M = sh + warp * ns;
  const double he = A.elh[e], hf = A.elh[f];
  const double delta = wrap_delta(A, A.elm[e] - A.elm[f]);
  double rho = hf / he, dl = delta / he;
  if (fabs(rho - 1.0) < WIDTH_SNAP) {  // exact integer gaps as the unit table (quadrature.py:452-456)
    rho = 1.0;
    if (fabs(dl - rint(dl)) < 1e-9 * fmax(1.0, fabs(dl))) dl = rint(dl);
  }
  // lane-owned slots s = lane + 32 j
  constexpr int SL = (GMAXA * GMAXB + 31) / 32;   // slots per lane
  double acc[SL];
  int sa[SL], sb[SL];
  for (int j = 0; j < SL; ++j) {
    acc[j] = 0.0;
    const int s = lane + 32 * j;
    sa[j] = s < ns ? s / nB : -1;
    sb[j] = s < ns ? s % nB : 0;
  }
  if (rho == 1.0 && (dl == -1.0 || dl == 0.0 || dl == 1.0)) {
    const double* t = A.near_unit + (int)(1.0 - dl) * ns;  // rows keff = -dl = -1, 0, 1
    for (int j = 0; j < SL; ++j)
      if (sa[j] >= 0) acc[j] = t[lane + 32 * j];
  } else if (rho == 1.0) {
    if (lane == 0) {
      for (int i = 0; i < ns; ++i) M[i] = 0.0;
      pair_closed(A.da, A.db, rho, dl, M, nB);
    }
    __syncwarp();
    for (int j = 0; j < SL; ++j)
      if (sa[j] >= 0) acc[j] = M[lane + 32 * j];
    __syncwarp();
  } else {
    const double sig = dl > 0.0 ? 1.0 : -1.0;
    const double* R = A.touch;
    const double* x16 = R;
    const double* w16 = R + TOUCH_XI;
    const double* x30 = R + 2 * TOUCH_XI;
    const double* w30 = x30 + TOUCH_ETA;
    const double* xl = w30 + TOUCH_ETA;
    const double* wl = xl + TOUCH_LOG;
    auto touch_node = [&](int n, double& w, double& u, double& v) {
      const int tri = n / (TOUCH_ETA * (TOUCH_XI + TOUCH_LOG));
      const int q = (n / (TOUCH_XI + TOUCH_LOG)) % TOUCH_ETA, jx = n % (TOUCH_XI + TOUCH_LOG);
      const double eta = x30[q];
      const double g = tri == 0 ? log1p(rho * eta) : log(rho + eta);
      const bool lg = jx >= TOUCH_XI;
      const double xi = lg ? xl[jx - TOUCH_XI] : x16[jx];
      w = w30[q] * rho * xi * (lg ? -wl[jx - TOUCH_XI] : w16[jx] * g);
      if (tri == 0) {
        u = sig * (xi - 0.5);
        v = -sig * rho * (xi * eta - 0.5);
      } else {
        u = sig * (xi * eta - 0.5);
        v = -sig * rho * (xi - 0.5);
      }
    };
    constexpr int TOUCH_NODES = 2 * TOUCH_ETA * (TOUCH_XI + TOUCH_LOG);
    const bool fast = (nA == 17 && nB == 5) || (nA == 16 && nB == 4);
    if (fast) {
      // nodes over the lanes, slots in registers (the per-slot loop below ran ~1e5 dependent
      // multiplies on each lane of one warp per pair: the launch was bound by that latency)
      for (int i = lane; i < ns; i += 32) M[i] = 0.0;
      __syncwarp();
      if (nA == 17) warp_node_moments<17, 5>(TOUCH_NODES, touch_node, M, lane);
      else warp_node_moments<16, 4>(TOUCH_NODES, touch_node, M, lane);
      for (int j = 0; j < SL; ++j)
        if (sa[j] >= 0) acc[j] = M[lane + 32 * j];
      __syncwarp();
    } else {
      for (int n = 0; n < TOUCH_NODES; ++n) {
        double wx, u, v;
        touch_node(n, wx, u, v);
        for (int j = 0; j < SL; ++j) {
          if (sa[j] < 0) continue;
          double t = wx;
          for (int i = 0; i < sa[j]; ++i) t *= u;
          for (int i = 0; i < sb[j]; ++i) t *= v;
          acc[j] += t;
        }
      }
    }
  }
  if (A.closed) {  // periodic gap term, 30 x 30 Gauss (quadrature.py:459-468)
    const double per = A.period / he;
    auto per_node = [&](int n, double& w, double& u, double& v) {
      const int g = n / GT0, h = n % GT0;
      const double xg = A.gx[g], xh = A.gx[h];
      const double yy = ((rho * xh - xg) - dl) / per;
      const double kv = yy == 0.0 ? 0.0 : log(fabs(sinpi(yy) / (kPi * yy)));
      w = A.gw[g] * A.gw[h] * rho * kv;
      u = xg;
      v = rho * xh;
    };
    if ((nA == 17 && nB == 5) || (nA == 16 && nB == 4)) {
      for (int i = lane; i < ns; i += 32) M[i] = 0.0;
      __syncwarp();
      if (nA == 17) warp_node_moments<17, 5>(GT0 * GT0, per_node, M, lane);
      else warp_node_moments<16, 4>(GT0 * GT0, per_node, M, lane);
      for (int j = 0; j < SL; ++j)
        if (sa[j] >= 0) acc[j] += M[lane + 32 * j];
      __syncwarp();
    } else {
      for (int n = 0; n < GT0 * GT0; ++n) {
        double w, xg, rxh;
        per_node(n, w, xg, rxh);
        for (int j = 0; j < SL; ++j) {
          if (sa[j] < 0) continue;
          double t = w;
          for (int i = 0; i < sa[j]; ++i) t *= xg;
          for (int i = 0; i < sb[j]; ++i) t *= rxh;
          acc[j] += t;
        }
      }
    }
  }
  const double lh = log(he);
  for (int j = 0; j < SL; ++j) {
    if (sa[j] < 0) continue;
    const int a = sa[j], b = sb[j];
    double s = 1.0, rp = rho;
    for (int i = 0; i < a + b + 2; ++i) s *= he;
    for (int i = 0; i < b; ++i) rp *= rho;
    M[lane + 32 * j] = s * (acc[j] + lh * (A.ca[a] * (rp * A.cb[b])));
  }
  __syncwarp();
  if (A.mg_out) {  // moments of (e lattice, f in G) for the lattice route (wq_ystage.cu)
    const int gf = A.gidx[f];
    if (gf >= 0 && A.gidx[e] < 0)
      for (int i = lane; i < ns; i += 32) A.mg_out[((int64_t)gf * A.n_el + e) * ns + i] = M[i];
    return;
  }
  // contraction: 2 nU nB... outputs over the lanes
  const double* ue = A.u + e * nA * nU;
  const double* ve = A.v + e * nB * nB;
  const double* vf = A.v + f * nB * nB;
  const int64_t ec = e - A.e0;
  for (int o = lane; o < nU * nB + nB * nB; o += 32) {
    const bool th = o < nU * nB;
    const int oo = th ? o : o - nU * nB;
    const int ap = oo / nB, bp = oo % nB;
    const int na = th ? nA : nB;
    const double* c = th ? ue : ve;
    const int ldc = th ? nU : nB;
    double s = 0.0;
    for (int al = 0; al < na; ++al) {
      double mv = 0.0;
      for (int be = 0; be < nB; ++be) mv = fma(M[al * nB + be], vf[be * nB + bp], mv);
      s = fma(c[al * ldc + ap], mv, s);
    }
    if (th) A.wt[wslot(A, f, oo, nU * nB, ec)] = s;
    else A.wd[wslot(A, f, oo, nB * nB, ec)] = s;
  }
}

// Theta^T[l][i] += sum_{(e,a) in inc_u(i), e in chunk} sum_{(f,b) in inc_v(l)} WT[f][a][b][e-e0]
// (threads over i: consecutive e, coalesced in the chunk-minor layout)
__global__ void gather_theta_kernel(int64_t ldt, int64_t i_off, int64_t e0, int64_t e1,
                                    int64_t ldc, int64_t i0, int64_t i1, int wu, int wv, int nU,
                                    int nB, const int64_t* u_el, const int64_t* u_loc,
                                    const int64_t* v_el, const int64_t* v_loc, const double* wt,
                                    double* thetaT) {
  const int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t l = blockIdx.y;
  if (i >= i1) return;
  double acc = 0.0;
  for (int ua = 0; ua < wu; ++ua) {
    const int64_t e = u_el[i * wu + ua];
    if (e < e0 || e >= e1) continue;
    const int a = (int)u_loc[i * wu + ua];
    for (int vb = 0; vb < wv; ++vb) {
      const int64_t f = v_el[l * wv + vb];
      if (f < 0) continue;
      acc += wt[((f * nU + a) * nB + v_loc[l * wv + vb]) * ldc + (e - e0)];
    }
  }
  thetaT[l * ldt + (i - i_off)] += acc;
}

// D (symmetric) from the chunk: entry (l, m) = sum_{(e,a) in inc_v(l), e in
// chunk} sum_{(f,b) in inc_v(m)} WD[f][a][b][e-e0], stored at D[m][l] --
// threads over l (consecutive e: coalesced loads and stores)
__global__ void gather_d_kernel(int64_t n_fine, int64_t e0, int64_t e1, int64_t ldc, int64_t l0,
                                int64_t l1, int wv, int nB, const int64_t* v_el,
                                const int64_t* v_loc, const double* wd, double* D) {
  const int64_t l = l0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = blockIdx.y;
  if (l >= l1) return;
  double acc = 0.0;
  for (int va = 0; va < wv; ++va) {
    const int64_t e = v_el[l * wv + va];
    if (e < e0 || e >= e1) continue;
    const int a = (int)v_loc[l * wv + va];
    for (int vb = 0; vb < wv; ++vb) {
      const int64_t f = v_el[m * wv + vb];
      if (f < 0) continue;
      acc += wd[((f * nB + a) * nB + v_loc[m * wv + vb]) * ldc + (e - e0)];
    }
  }
  D[m * n_fine + l] += acc;
}

// Banded Cholesky solves X <- L^{-T} L^{-1} X per column with the last BW
// values of the column in registers (one load + one store per row).  Rows go
// in batches of RB: the NEXT batch's column values are loaded while the
// current batch runs its dependent chain (RB independent HBM requests in
// flight per thread, latency hidden behind the chain -- one thread per column
// leaves only ~4 warps per SM), and each batch's factor rows are staged once
// per CTA in shared memory as -L[k][k-j] and 1/L[k][k], so the dependent
// chain per row is BW FMAs and one multiply.
template <int BW, bool FWD>
__device__ __forceinline__ void band_sweep(int64_t n, const double* Lb, double* x, int64_t ldx,
                                           bool live) {
  constexpr int RB = 16, DEPTH = 3;   // batches of RB rows; DEPTH batches of loads in flight
  __shared__ double cf[RB][BW + 1];   // [r][0] = 1/diag, [r][j] = -off-diagonal
  // row of batch position r in batch q: forward k = q RB + r, backward k = n - 1 - q RB - r
  auto row = [n](int64_t q, int r) -> int64_t { return FWD ? q * RB + r : n - 1 - q * RB - r; };
  const int64_t nbat = (n + RB - 1) / RB;
  double w[BW];
#pragma unroll
  for (int j = 0; j < BW; ++j) w[j] = 0.0;  // w[j] = previous solution values
  double xq[DEPTH][RB];
  auto load = [&](int64_t q, double (&dst)[RB]) {
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int64_t k = row(q, r);
      dst[r] = (live && q < nbat && k >= 0 && k < n) ? x[k * ldx] : 0.0;
    }
  };
#pragma unroll
  for (int d = 0; d < DEPTH - 1; ++d) load(d, xq[d]);
  for (int64_t q = 0; q < nbat; q += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const int64_t qq = q + d;
      // batch qq + DEPTH - 1 goes into the slot batch qq - 1 used
      load(qq + DEPTH - 1, xq[(d + DEPTH - 1) % DEPTH]);
      __syncthreads();
      for (int t = threadIdx.x; t < RB * (BW + 1); t += blockDim.x) {
        const int r = t / (BW + 1), j = t - r * (BW + 1);
        const int64_t k = row(qq, r);
        double v = 0.0;
        if (qq < nbat && k >= 0 && k < n) {
          if (j == 0) v = 1.0 / Lb[k * (BW + 1)];
          else if (FWD) v = k - j >= 0 ? -Lb[k * (BW + 1) + j] : 0.0;
          else v = k + j < n ? -Lb[(k + j) * (BW + 1) + j] : 0.0;
        }
        cf[r][j] = v;
      }
      __syncthreads();
      if (!live || qq >= nbat) continue;
      double* xb = xq[d];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        // oldest values first: the newest one (w[0], the previous row) enters last, so the
        // loop-carried dependency is one FMA and one multiply per row
        double s = xb[r];
#pragma unroll
        for (int j = BW; j >= 1; --j) s = fma(cf[r][j], w[j - 1], s);
        s *= cf[r][0];
        xb[r] = s;
#pragma unroll
        for (int j = BW - 1; j > 0; --j) w[j] = w[j - 1];
        w[0] = s;
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const int64_t k = row(qq, r);
        if (k >= 0 && k < n) x[k * ldx] = xb[r];
      }
    }
  }
}

template <int BW>
__global__ void __launch_bounds__(128)
band_solve_win_kernel(int64_t n, const double* Lb, double* X, int64_t ncols, int64_t ldx) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = c < ncols;
  double* x = X + (live ? c : 0);
  band_sweep<BW, true>(n, Lb, x, ldx, live);
  band_sweep<BW, false>(n, Lb, x, ldx, live);
}

// Segmented banded solves: the rows of every column are cut into segments of SEG
// rows that run in parallel (one thread per column and segment), so a sweep has
// columns x segments threads instead of one thread per column.  A segment starts
// from the last BW solution values of the previous one, which a first pass
// reconstructs from K0 preceding rows run from a zero state: the factor's inverse
// decays geometrically (C5: below 1e-18 within 83 rows), so after K0 rows the state
// is exact to rounding (K0 chosen on the host from the measured decay).
template <int BW, bool FWD>
__device__ __forceinline__ void band_sweep_range(int64_t n, const double* Lb, double* x, int64_t ldx,
                                                 bool live, int64_t i0, int64_t i1, double (&w)[BW],
                                                 bool store) {
  // columns x segments threads: occupancy, not a deep per-thread prefetch, hides the HBM
  // latency, so the register ring stays short (RB 8 x DEPTH 2: 3 solves 11.5 -> 10.0 ms at
  // C5; 16 x 2: 11.1, 8 x 3: 12.1, 4 x 2: 9.9; the factor rows of a whole segment staged
  // once in shared memory instead of per batch: 10.1)
  constexpr int RB = 8, DEPTH = 2;
  __shared__ double cf[RB][BW + 1];   // [r][0] = 1/diag, [r][j] = -off-diagonal
  // sweep index i -> row: forward k = i, backward k = n - 1 - i
  auto row = [n](int64_t i) -> int64_t { return FWD ? i : n - 1 - i; };
  const int64_t nbat = (i1 - i0 + RB - 1) / RB;
  double xq[DEPTH][RB];
  auto load = [&](int64_t q, double (&dst)[RB]) {
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int64_t i = i0 + q * RB + r;
      dst[r] = (live && q < nbat && i < i1) ? x[row(i) * ldx] : 0.0;
    }
  };
#pragma unroll
  for (int d = 0; d < DEPTH - 1; ++d) load(d, xq[d]);
  for (int64_t q = 0; q < nbat; q += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      const int64_t qq = q + d;
      load(qq + DEPTH - 1, xq[(d + DEPTH - 1) % DEPTH]);
      __syncthreads();
      for (int t = threadIdx.x; t < RB * (BW + 1); t += blockDim.x) {
        const int r = t / (BW + 1), j = t - r * (BW + 1);
        const int64_t i = i0 + qq * RB + r;
        double v = 0.0;
        if (qq < nbat && i < i1) {
          const int64_t k = row(i);
          if (j == 0) v = 1.0 / Lb[k * (BW + 1)];
          else if (FWD) v = k - j >= 0 ? -Lb[k * (BW + 1) + j] : 0.0;
          else v = k + j < n ? -Lb[(k + j) * (BW + 1) + j] : 0.0;
        }
        cf[r][j] = v;
      }
      __syncthreads();
      if (!live || qq >= nbat) continue;
      double* xb = xq[d];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        double sv = xb[r];
#pragma unroll
        for (int j = BW; j >= 1; --j) sv = fma(cf[r][j], w[j - 1], sv);
        sv *= cf[r][0];
        xb[r] = sv;
        if (i0 + qq * RB + r < i1) {
#pragma unroll
          for (int j = BW - 1; j > 0; --j) w[j] = w[j - 1];
          w[0] = sv;
        }
      }
      if (store) {
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          const int64_t i = i0 + qq * RB + r;
          if (i < i1) x[row(i) * ldx] = xb[r];
        }
      }
    }
  }
}

// pass 1: the state (last BW values) at the start of every segment s >= 1, from K0 rows
template <int BW, bool FWD>
__global__ void __launch_bounds__(128)
band_seg_state_kernel(int64_t n, const double* Lb, const double* X, int64_t ncols, int64_t ldx,
                      int64_t seg, int64_t k0, double* state) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s = blockIdx.y + 1;
  const bool live = c < ncols;
  double w[BW];
#pragma unroll
  for (int j = 0; j < BW; ++j) w[j] = 0.0;
  const int64_t start = s * seg;
  const int64_t from = start - k0 > 0 ? start - k0 : 0;
  band_sweep_range<BW, FWD>(n, Lb, const_cast<double*>(X) + (live ? c : 0), ldx, live, from, start,
                            w, false);
  if (live)
#pragma unroll
    for (int j = 0; j < BW; ++j) state[((s - 1) * BW + j) * ncols + c] = w[j];
}

// pass 2: every segment from its state, in place
template <int BW, bool FWD>
__global__ void __launch_bounds__(128)
band_seg_solve_kernel(int64_t n, const double* Lb, double* X, int64_t ncols, int64_t ldx,
                      int64_t seg, const double* state) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t s = blockIdx.y;
  const bool live = c < ncols;
  double w[BW];
#pragma unroll
  for (int j = 0; j < BW; ++j)
    w[j] = (s > 0 && live) ? state[((s - 1) * BW + j) * ncols + c] : 0.0;
  const int64_t i0 = s * seg, i1 = (s + 1) * seg < n ? (s + 1) * seg : n;
  band_sweep_range<BW, FWD>(n, Lb, X + (live ? c : 0), ldx, live, i0, i1, w, true);
}

template <int BW>
static void band_solve_seg(int64_t n, const double* Lb, double* X, int64_t ncols, int64_t ldx,
                           int64_t seg, int64_t k0, double* state, cudaStream_t st) {
  const int64_t nseg = (n + seg - 1) / seg;
  const dim3 gs(ceil_div(ncols, 128), (unsigned)(nseg > 1 ? nseg - 1 : 1));
  const dim3 gv(ceil_div(ncols, 128), (unsigned)nseg);
  if (nseg > 1) band_seg_state_kernel<BW, true><<<gs, 128, 0, st>>>(n, Lb, X, ncols, ldx, seg, k0, state);
  band_seg_solve_kernel<BW, true><<<gv, 128, 0, st>>>(n, Lb, X, ncols, ldx, seg, state);
  if (nseg > 1) band_seg_state_kernel<BW, false><<<gs, 128, 0, st>>>(n, Lb, X, ncols, ldx, seg, k0, state);
  band_seg_solve_kernel<BW, false><<<gv, 128, 0, st>>>(n, Lb, X, ncols, ldx, seg, state);
}

}  // namespace wq

using namespace wq;

extern "C" {

int wq_gen_pair_blocks(int64_t n_el, int64_t e0, int64_t e1, int da, int db, int pu, int closed,
                       double period, const double* elh, const double* elm, const double* u,
                       const double* v, const int64_t* near_lo, const int64_t* near_cnt,
                       int max_near, const double* near_unit, const double* touch,
                       const double* gx, const double* gw, const double* m2u,
                       const double* ca, const double* cb, double* wt, double* wd,
                       int64_t ldc, int* tile_flag, void* stream) {
  if (n_el <= 0 || e0 < 0 || e1 > n_el || e1 <= e0 || da + 1 > GMAXA || db + 1 > GMAXB ||
      db < 1 || pu != db || max_near < 0 || !near_unit || !touch || !gx || !gw || !elh || !elm || !u || !v || !near_lo || !near_cnt ||
      !ca || !cb || !wt || !wd || (closed && !(period > 0)) || ldc < e1 - e0 || (m2u && (closed || !tile_flag))) {
    set_error("wq_gen_pair_blocks: bad arguments");
    return WQ_EINVAL;
  }
  int rc = ensure_consts();
  if (rc) return rc;
  GenArgs A{n_el, e0, e1, da, db, pu, closed, period, elh, elm, u, v, near_lo, near_cnt,
            near_unit, touch, gx, gw, m2u, ca, cb, wt, wd, ldc, tile_flag, nullptr, nullptr};
  cudaStream_t st = (cudaStream_t)stream;
  dim3 g1(ceil_div(e1 - e0, FP_THREADS), (unsigned)n_el);   // (64 outer elements, inner f)
  const int nA = da + 1, np1 = db + 1;
  const int64_t ntiles = (int64_t)g1.x * g1.y;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // persistent grid: a multiple of the outer blocks (each CTA keeps one), ~3 CTAs per SM (61 KB each at p = 4)
  const int64_t per = std::max<int64_t>(1, std::min<int64_t>(n_el, (int64_t)sms * 3 / g1.x));
  const int64_t fgrid = per * g1.x;
  (void)ntiles;
#define WQ_GEN_CASE(NP)                                                                      \
  case NP:                                                                                   \
    if (m2u) {                                                                               \
      pair_table_kernel<NP><<<g1, FP_THREADS, 0, st>>>(A);                                   \
    }                                                                                        \
    {                                                                                        \
      const size_t fsm = (size_t)GT2 * 2 * NP * FP_THREADS * sizeof(double);                 \
      cudaFuncSetAttribute(pair_far_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)fsm);                                                        \
      pair_far_kernel<NP><<<(unsigned)fgrid, FP_THREADS, fsm, st>>>(A, n_el, (int)g1.x);     \
    }                                                                                        \
    break;
  switch (np1) {
    WQ_GEN_CASE(2)
    WQ_GEN_CASE(3)
    WQ_GEN_CASE(4)
    WQ_GEN_CASE(5)
    WQ_GEN_CASE(6)
    WQ_GEN_CASE(7)
    WQ_GEN_CASE(8)
    default:
      set_error("wq_gen_pair_blocks: degree %d unsupported", db);
      return WQ_EUNSUPPORTED;
  }
#undef WQ_GEN_CASE
  rc = check_launch("wq_gen_pair_blocks(far)");
  if (rc || max_near == 0) return rc;
  const size_t smem = (size_t)NP_WARPS * nA * np1 * sizeof(double);
  dim3 g2(ceil_div(max_near, NP_WARPS), (unsigned)(e1 - e0));
  pair_near_kernel<<<g2, NP_WARPS * 32, smem, st>>>(A, max_near);
  return check_launch("wq_gen_pair_blocks(near)");
}

int wq_gen_near_moments(int64_t n_el, int da, int db, const double* elh, const double* elm,
                        const int64_t* near_lo, const int64_t* near_cnt, int max_near,
                        const double* near_unit, const double* touch, const double* ca,
                        const double* cb, const int* gidx, double* mgc, void* stream) {
  if (n_el <= 0 || da + 1 > GMAXA || db + 1 > GMAXB || max_near < 1 || !elh || !elm ||
      !near_lo || !near_cnt || !near_unit || !touch || !ca || !cb || !gidx || !mgc) {
    set_error("wq_gen_near_moments: bad arguments");
    return WQ_EINVAL;
  }
  GenArgs A{n_el, 0, n_el, da, db, db, 0, 0.0, elh, elm, nullptr, nullptr, near_lo, near_cnt,
            near_unit, touch, nullptr, nullptr, nullptr, ca, cb, nullptr, nullptr, 1, nullptr,
            mgc, gidx};
  const size_t smem = (size_t)NP_WARPS * (da + 1) * (db + 1) * sizeof(double);
  dim3 g2(ceil_div(max_near, NP_WARPS), (unsigned)n_el);
  pair_near_kernel<<<g2, NP_WARPS * 32, smem, (cudaStream_t)stream>>>(A, max_near);
  return check_launch("wq_gen_near_moments");
}

int wq_gen_gather_theta(int64_t n_rows, int64_t n_fine, int64_t e0, int64_t e1, int64_t ldc,
                        int64_t i0, int64_t i1, int wu, int wv, int nU, int nB,
                        const int64_t* u_el, const int64_t* u_loc, const int64_t* v_el,
                        const int64_t* v_loc, const double* wt, double* thetaT, int64_t ldt,
                        int64_t i_off, void* stream) {
  if (i1 <= i0 || i0 < i_off || i1 > n_rows || n_fine <= 0 || !u_el || !u_loc || !v_el ||
      !v_loc || !wt || !thetaT || ldt < i1 - i_off) {
    set_error("wq_gen_gather_theta: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(i1 - i0, 64), (unsigned)n_fine);
  gather_theta_kernel<<<grid, 64, 0, (cudaStream_t)stream>>>(ldt, i_off, e0, e1, ldc, i0, i1, wu, wv,
                                                            nU, nB, u_el, u_loc, v_el, v_loc, wt,
                                                            thetaT);
  return check_launch("wq_gen_gather_theta");
}

int wq_gen_gather_d(int64_t n_fine, int64_t e0, int64_t e1, int64_t ldc, int64_t l0, int64_t l1,
                    int wv, int nB, const int64_t* v_el, const int64_t* v_loc, const double* wd,
                    double* D, void* stream) {
  if (l1 <= l0 || l0 < 0 || l1 > n_fine || !v_el || !v_loc || !wd || !D) {
    set_error("wq_gen_gather_d: bad arguments");
    return WQ_EINVAL;
  }
  dim3 grid(ceil_div(l1 - l0, 64), (unsigned)n_fine);
  gather_d_kernel<<<grid, 64, 0, (cudaStream_t)stream>>>(n_fine, e0, e1, ldc, l0, l1, wv, nB,
                                                        v_el, v_loc, wd, D);
  return check_launch("wq_gen_gather_d");
}

int wq_band_solve_seg(int64_t n, int64_t bw, const double* Lb, double* X, int64_t ncols,
                      int64_t ldx, int64_t seg, int64_t k0, double* state, void* stream) {
  if (n <= 0 || bw < 1 || bw > 8 || !Lb || !X || ncols <= 0 || ldx < ncols || seg < 16 ||
      k0 < 0 || (n > seg && !state)) {
    set_error("wq_band_solve_seg: bad arguments");
    return WQ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  switch (bw) {
    case 1: band_solve_seg<1>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
    case 2: band_solve_seg<2>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
    case 3: band_solve_seg<3>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
    case 4: band_solve_seg<4>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
    case 5: band_solve_seg<5>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
    case 6: band_solve_seg<6>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
    case 7: band_solve_seg<7>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
    default: band_solve_seg<8>(n, Lb, X, ncols, ldx, seg, k0, state, st); break;
  }
  return check_launch("wq_band_solve_seg");
}

int wq_band_solve_win(int64_t n, int64_t bw, const double* Lb, double* X, int64_t ncols,
                      int64_t ldx, void* stream) {
  if (n <= 0 || bw < 1 || bw > 8 || !Lb || !X || ncols <= 0 || ldx < ncols) {
    set_error("wq_band_solve_win: bad arguments");
    return WQ_EINVAL;
  }
  const unsigned grid = ceil_div(ncols, 128);
  cudaStream_t st = (cudaStream_t)stream;
  switch (bw) {
    case 1: band_solve_win_kernel<1><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
    case 2: band_solve_win_kernel<2><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
    case 3: band_solve_win_kernel<3><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
    case 4: band_solve_win_kernel<4><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
    case 5: band_solve_win_kernel<5><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
    case 6: band_solve_win_kernel<6><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
    case 7: band_solve_win_kernel<7><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
    default: band_solve_win_kernel<8><<<grid, 128, 0, st>>>(n, Lb, X, ncols, ldx); break;
  }
  return check_launch("wq_band_solve_win");
}

}  // extern "C"
