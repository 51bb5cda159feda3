// Tools only: the x2 Phi loop in isolation (6 shared A-fragment loads + 2 coalesced global
// B-fragment loads + 10 DMMAs per k-step, 18 k-steps, then a CTA barrier), 2 CTAs of 8 warps
// per SM, to separate the loop's own DMMA-pipe efficiency from the kernel's other phases.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/phi_probe tools/phi_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
constexpr int ZS = 20, NST = 18, PF = 4;

// MODE bit 0: barrier after each phi; bit 1: B from global (else registers); bit 2: store Phi to smem
template <int MODE>
__global__ void __launch_bounds__(256, 2) probe(int reps, const double* __restrict__ U, double* out) {
  extern __shared__ double sm[];
  double* Z = sm;              // 143 x 20
  double* Ph = sm + 2 * 143 * ZS;
  for (int k = threadIdx.x; k < 2 * 143 * ZS; k += 256) sm[k] = 1e-3 * (k % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r = lane >> 2, c = lane & 3;
  const int g = warp >> 1, h = warp & 1;
  double tot = 0.0;
  for (int rep = 0; rep < reps; ++rep) {
    double accA[5][2], accB[5][2];
#pragma unroll
    for (int j = 0; j < 5; ++j) accA[j][0] = accA[j][1] = accB[j][0] = accB[j][1] = 0.0;
    const double* uA = U + ((size_t)((blockIdx.x * 7 + rep * 8 + 2 * g) & 4095)) * (NST * 32) + lane;
    const double* uB = uA + NST * 32;
    double bqA[PF], bqB[PF];
#pragma unroll
    for (int s = 0; s < PF; ++s) {
      bqA[s] = (MODE & 2) ? __ldg(uA + 32 * s) : 1.0 + s;
      bqB[s] = (MODE & 2) ? __ldg(uB + 32 * s) : 2.0 + s;
    }
    const int zbase = 8 * (6 - 2 * g + h * 5) + r + 7;
    auto zptr = [&](int s) -> const double* {
      int off, col;
      if (s < 16) { off = (4 * s) / 16; col = (4 * s - off * 16) + c; }
      else { off = 4 * (s - 16) + c; col = 16; }
      return Z + (zbase - off) * ZS + col;
    };
    double afr[2][6];
    { const double* z = zptr(0);
#pragma unroll
      for (int j = 0; j <= 5; ++j) afr[0][j] = z[j * 8 * ZS]; }
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      const int cur = s & 1;
      if (s + 1 < NST) {
        const double* z = zptr(s + 1);
#pragma unroll
        for (int j = 0; j <= 5; ++j) afr[cur ^ 1][j] = z[j * 8 * ZS];
      }
      const double ba = bqA[s % PF], bb = bqB[s % PF];
      if ((MODE & 2) && s + PF < NST) {
        bqA[s % PF] = __ldg(uA + 32 * (s + PF));
        bqB[s % PF] = __ldg(uB + 32 * (s + PF));
      }
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        dmma(accB[j][0], accB[j][1], afr[cur][j], bb);
        dmma(accA[j][0], accA[j][1], afr[cur][j + 1], ba);
      }
    }
    if (MODE & 4) {
#pragma unroll
      for (int j = 0; j < 5; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int mm = 8 * (h * 5 + j) + r + 2 * c + e - 7;
          if (mm >= 0 && mm < 70) {
            Ph[(16 * g + 2 * c + e) * 76 + mm] = accA[j][e];
            Ph[(16 * g + 8 + 2 * c + e) * 76 + mm] = accB[j][e];
          }
        }
    } else {
#pragma unroll
      for (int j = 0; j < 5; ++j) tot += accA[j][0] + accA[j][1] + accB[j][0] + accB[j][1];
    }
    if (MODE & 1) __syncthreads();
  }
  out[blockIdx.x * 256 + threadIdx.x] = tot + Ph[threadIdx.x];
}

template <int MODE>
void run(const double* U, double* out, int ctas_per_sm) {
  const int reps = 400, blocks = 148 * ctas_per_sm;
  const size_t smem = ctas_per_sm == 2 ? 85 * 1024 : 120 * 1024;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<MODE><<<blocks, 256, smem>>>(reps, U, out);
  cudaEventRecord(e0);
  probe<MODE><<<blocks, 256, smem>>>(reps, U, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * 10 * NST * 8.0 * reps * blocks;
  printf("ctas/SM %d  barrier %d  Bglobal %d  store %d : %6.2f TF  (%s)\n", ctas_per_sm, MODE & 1,
         (MODE >> 1) & 1, (MODE >> 2) & 1, flops / ms * 1e-9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *U, *out;
  cudaMalloc(&U, (size_t)4100 * NST * 32 * 8); cudaMemset(U, 0, (size_t)4100 * NST * 32 * 8);
  cudaMalloc(&out, 148 * 2 * 256 * 8);
  for (int c : {1, 2}) {
    run<0>(U, out, c); run<1>(U, out, c); run<2>(U, out, c); run<3>(U, out, c); run<7>(U, out, c);
  }
  return 0;
}
