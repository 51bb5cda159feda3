// Shared helpers for the sm_100a FP64 SGBEM assembly kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <math.h>

#include "../../include/wqb200.h"

namespace wq {

// Last error message of the calling host thread (C-ABI: wq_last_error()).
void set_error(const char* fmt, ...);

// Record a launch error (if any) and return the C-ABI status.
int check_launch(const char* what);

__host__ __device__ __forceinline__ int64_t pmod(int64_t a, int64_t n) {
  int64_t r = a % n;
  return r < 0 ? r + n : r;
}

// a mod n for a in (-n, 2n): two compares instead of an int64 division
__host__ __device__ __forceinline__ int64_t wrap1(int64_t a, int64_t n) {
  return a < 0 ? a + n : (a >= n ? a - n : a);
}

__host__ __device__ __forceinline__ int ceil_div(int64_t a, int64_t b) {
  return (int)((a + b - 1) / b);
}

// J(mid)^2 for a distinct node pair within eps_diag, from the host table
__device__ __forceinline__ bool near_pair_j2(const wq_smooth_t& sm, int64_t qa, int64_t ra,
                                             double* R) {
  int64_t lo = qa < ra ? qa : ra, d = qa < ra ? ra - qa : qa - ra;
  if (sm.closed && sm.nq - d < d) {  // seam pair: forward from the larger index
    lo = qa < ra ? ra : qa;
    d = sm.nq - d;
  }
  if (d > sm.near_k) return false;
  const double v = sm.near_j2[lo * sm.near_k + (d - 1)];
  if (!(v > 0.0)) return false;
  *R = v;
  return true;
}

// upper-triangle tile pair index -> (bi, bj), bi <= bj; tile row bi holds nb - bi
// pairs, pairs numbered row by row
__device__ __forceinline__ void tri_index(int64_t t, int nb, int& bi, int& bj) {
  // float estimate (MUFU), corrected exactly by the integer loops below
  const float B = 2.0f * (float)nb + 1.0f;
  int b = (int)floorf((B - sqrtf(fmaxf(B * B - 8.0f * (float)t, 0.0f))) * 0.5f);
  if (b < 0) b = 0;
  if (b > nb - 1) b = nb - 1;
  auto start = [nb](int64_t x) { return x * nb - x * (x - 1) / 2; };
  while (b > 0 && start(b) > t) --b;
  while (b + 1 < nb && start(b + 1) <= t) ++b;
  bi = b;
  bj = b + (int)(t - start(b));
}

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 6.28318530717958647692;

}  // namespace wq
