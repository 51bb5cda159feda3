// Double-layer right-hand side (assemble_b2, assembly.py:322-343) on the GPU:
//
//   inner[s] = sum_t Kbar(s, t) w_t u_D(t),
//   Kbar(s, t) = ((f(t)-f(s))_y f'(t)_x - (f(t)-f(s))_x f'(t)_y) / |f(t)-f(s)|^2
//                (geometry.py:250-280), with the C^2 curvature limit on s == t.
//
// The (16 n_el)^2 kernel grid is evaluated on the fly (never stored): one
// thread per outer point s accumulates its row sequentially over t (fixed
// order: deterministic), the t data staged through shared memory in tiles.
// The O(M) outer contraction with the basis (assembly.py:341-343) is host work.
#include "wq_common.cuh"

namespace wq {

constexpr int B2_THREADS = 256;

__global__ void __launch_bounds__(B2_THREADS)
b2_inner_kernel(int64_t M, const double* __restrict__ fx, const double* __restrict__ fy,
                const double* __restrict__ tx, const double* __restrict__ ty,
                const double* __restrict__ wg, const double* __restrict__ kdiag, double* inner) {
  __shared__ double sfx[B2_THREADS], sfy[B2_THREADS], stx[B2_THREADS], sty[B2_THREADS],
      swg[B2_THREADS];
  const int64_t s = blockIdx.x * (int64_t)B2_THREADS + threadIdx.x;
  const bool active = s < M;
  const double xs = active ? fx[s] : 0.0, ys = active ? fy[s] : 0.0;
  double acc = 0.0;
  for (int64_t t0 = 0; t0 < M; t0 += B2_THREADS) {
    const int64_t t = t0 + threadIdx.x;
    __syncthreads();
    if (t < M) {
      sfx[threadIdx.x] = fx[t];
      sfy[threadIdx.x] = fy[t];
      stx[threadIdx.x] = tx[t];
      sty[threadIdx.x] = ty[t];
      swg[threadIdx.x] = wg[t];
    }
    __syncthreads();
    const int nt = (int)min((int64_t)B2_THREADS, M - t0);
    if (!active) continue;
#pragma unroll 4
    for (int k = 0; k < nt; ++k) {
      const int64_t tt = t0 + k;
      double kb;
      if (tt == s) {
        kb = kdiag[s];
      } else {
        const double dx = sfx[k] - xs, dy = sfy[k] - ys;
        const double d2 = dx * dx + dy * dy;
        kb = (dy * stx[k] - dx * sty[k]) / d2;
      }
      acc = fma(kb, swg[k], acc);
    }
  }
  if (active) inner[s] = acc;
}

}  // namespace wq

using namespace wq;

extern "C" int wq_b2_inner(int64_t M, const double* fx, const double* fy, const double* tx,
                           const double* ty, const double* wg, const double* kdiag, double* inner,
                           void* stream) {
  if (M <= 0 || !fx || !fy || !tx || !ty || !wg || !kdiag || !inner) {
    set_error("wq_b2_inner: bad arguments");
    return WQ_EINVAL;
  }
  b2_inner_kernel<<<ceil_div(M, B2_THREADS), B2_THREADS, 0, (cudaStream_t)stream>>>(M, fx, fy, tx,
                                                                                     ty, wg, kdiag,
                                                                                     inner);
  return check_launch("wq_b2_inner");
}
