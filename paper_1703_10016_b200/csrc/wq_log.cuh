// Table-based FP64 0.5 ln(x) shared by the IK1 kernels (see wq_fast.cu for
// the table: 16 mantissa bins c_j = 1/mid_j and the double-double
// 0.5 (-ln c_j), so 16 doubles span the 32 shared-memory banks once).
#pragma once
#include "wq_common.cuh"

namespace wq {

// 0.5 ln 2 = HLN2_A + HLN2_B, HLN2_A with 41 significant bits (e*A exact)
constexpr double HLN2_A = 0.3465735902798315;
constexpr double HLN2_B = 1.4117645281515789e-13;

__device__ __forceinline__ double half_ln16(double x, const double* __restrict__ tab) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 16) & 15;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
  const double r = fma(m, tab[j], -1.0);  // |r| < 2^-5
  double q = fma(r, 0.5 / 9.0, -0.5 / 8.0);  // degree 9: truncation < 1.1e-19
  q = fma(r, q, 0.5 / 7.0);
  q = fma(r, q, -0.5 / 6.0);
  q = fma(r, q, 0.5 / 5.0);
  q = fma(r, q, -0.5 / 4.0);
  q = fma(r, q, 0.5 / 3.0);
  q = fma(r, q, -0.25);
  const double r2 = r * r;
  const double de = (double)e;
  const double t_hi = fma(de, HLN2_A, tab[16 + j]);
  const double t_lo = fma(de, HLN2_B, tab[32 + j]);
  return t_hi + fma(r, 0.5, fma(r2, q, t_lo));
}


// device address of the 16-entry table (wq_fast.cu; uploads it on first use)
int logtab16_device(const double** out);

}  // namespace wq
