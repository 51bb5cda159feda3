// Packed upper-triangle blocks for the multi-GPU all-gather.
//
// On closed uniform meshes the assembly runs over the upper-triangle 64 x 64
// tile pairs (I, J >= I), numbered row by row; a rank assembles contiguous
// pair ranges [p0, p1) (equal ranges = equal work).  Only the upper tile A(I, J)
// of each pair is sent -- A is symmetric, A(J, I) is its transpose -- which
// halves the NVLink bytes of the all-gather against full rows, and equal pair
// ranges make every rank's buffer the same size (no padding).  Packed layout:
// tile-major, pair p at (p - p0) * 4096, row-major 64 x 64 (entries outside an
// edge tile are not written / read).  The receiver writes each tile into A(I, J)
// and its transpose into A(J, I) (through shared memory), so no separate mirror
// pass over A is needed.
#include "wq_common.cuh"

namespace wq {

constexpr int PK = 64;             // tile rows / columns (the assembly kernels' tile)
constexpr int PK2 = PK * PK;

__global__ void __launch_bounds__(256) pack_pairs_kernel(const double* __restrict__ A, int64_t n,
                                                         int64_t ld, int64_t p0, int nb,
                                                         double* __restrict__ packed) {
  int bi, bj;
  tri_index(p0 + blockIdx.x, nb, bi, bj);
  const double* src = A + (int64_t)bi * PK * ld + (int64_t)bj * PK;
  double* dst = packed + (int64_t)blockIdx.x * PK2;
  const int ni = (int)min((int64_t)PK, n - (int64_t)bi * PK);
  const int nj = (int)min((int64_t)PK, n - (int64_t)bj * PK);
  for (int k = threadIdx.x; k < PK2; k += blockDim.x) {
    const int a = k >> 6, b = k & 63;
    if (a < ni && b < nj) dst[k] = src[a * ld + b];
  }
}

__global__ void __launch_bounds__(256) unpack_pairs_kernel(const double* __restrict__ packed,
                                                           int64_t n, int64_t p0, int nb,
                                                           double* __restrict__ A, int64_t ld) {
  __shared__ double tile[PK][PK + 1];
  int bi, bj;
  tri_index(p0 + blockIdx.x, nb, bi, bj);
  const double* src = packed + (int64_t)blockIdx.x * PK2;
  const int ni = (int)min((int64_t)PK, n - (int64_t)bi * PK);
  const int nj = (int)min((int64_t)PK, n - (int64_t)bj * PK);
  double* up = A + (int64_t)bi * PK * ld + (int64_t)bj * PK;
  for (int k = threadIdx.x; k < PK2; k += blockDim.x) {
    const int a = k >> 6, b = k & 63;
    if (a < ni && b < nj) {
      const double v = src[k];
      up[a * ld + b] = v;
      tile[a][b] = v;
    }
  }
  if (bi == bj) return;  // the diagonal tile is symmetric and arrived whole
  __syncthreads();
  double* lo = A + (int64_t)bj * PK * ld + (int64_t)bi * PK;
  for (int k = threadIdx.x; k < PK2; k += blockDim.x) {
    const int a = k >> 6, b = k & 63;  // A(J, I)[a][b] = A(I, J)[b][a]
    if (a < nj && b < ni) lo[a * ld + b] = tile[b][a];
  }
}

static bool pairs_ok(int64_t n, int64_t ld, int64_t p0, int64_t p1) {
  const int64_t nb = ceil_div(n, PK);
  return n > 0 && ld >= n && p0 >= 0 && p1 >= p0 && p1 <= nb * (nb + 1) / 2;
}

}  // namespace wq

using namespace wq;

extern "C" {

int wq_pack_pairs(const double* A, int64_t n, int64_t ld, int64_t p0, int64_t p1, double* packed,
                  void* stream) {
  if (!A || !packed || !pairs_ok(n, ld, p0, p1)) {
    set_error("wq_pack_pairs: bad arguments");
    return WQ_EINVAL;
  }
  if (p1 == p0) return WQ_OK;
  pack_pairs_kernel<<<(unsigned)(p1 - p0), 256, 0, (cudaStream_t)stream>>>(A, n, ld, p0,
                                                                           ceil_div(n, PK), packed);
  return check_launch("wq_pack_pairs");
}

int wq_unpack_pairs(const double* packed, int64_t n, int64_t p0, int64_t p1, double* A, int64_t ld,
                    void* stream) {
  if (!A || !packed || !pairs_ok(n, ld, p0, p1)) {
    set_error("wq_unpack_pairs: bad arguments");
    return WQ_EINVAL;
  }
  if (p1 == p0) return WQ_OK;
  unpack_pairs_kernel<<<(unsigned)(p1 - p0), 256, 0, (cudaStream_t)stream>>>(
      packed, n, p0, ceil_div(n, PK), A, ld);
  return check_launch("wq_unpack_pairs");
}

}  // extern "C"
