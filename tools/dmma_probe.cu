// Tools only: DMMA (mma.sync.m8n8k4.f64) throughput per SM against warps per SM and
// independent accumulators per warp, with and without one shared-memory A-fragment load
// per DMMA.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int ILP, int LDS>   // LDS: A fragments per DMMA read from shared memory (0, 1 = every, 2 = every 2nd)
__global__ void probe(int iters, double* out) {
  __shared__ double sm[4096];
  for (int k = threadIdx.x; k < 4096; k += blockDim.x) sm[k] = 1e-3 * k;
  __syncthreads();
  double acc[ILP][2];
#pragma unroll
  for (int j = 0; j < ILP; ++j) acc[j][0] = acc[j][1] = 0.0;
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane, b = 1e-9 * lane;
  const double* p = sm + lane + 64 * (threadIdx.x >> 5);
  for (int it = 0; it < iters; ++it) {
    double af[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      if (LDS == 1) af[j] = p[(32 * j + it) & 1023];
      else if (LDS == 2) af[j] = (j & 1) ? a : p[(32 * j + it) & 1023];
      else af[j] = a;
    }
#pragma unroll
    for (int j = 0; j < ILP; ++j) dmma(acc[j][0], acc[j][1], af[j], b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP, int LDS>
void run(int warps, double* out) {
  const int iters = 4000, blocks = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<ILP, LDS><<<blocks, 32 * warps>>>(iters, out);
  cudaEventRecord(e0);
  probe<ILP, LDS><<<blocks, 32 * warps>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * ILP * (double)iters * warps * blocks;
  printf("warps/SM %2d ILP %2d lds %d: %7.2f TF\n", warps, ILP, LDS, flops / ms * 1e-9);
}

int main() {
  double* out; cudaMalloc(&out, 148 * 1024 * 8);
  for (int w : {4, 8, 16, 32}) {
    run<1, 0>(w, out); run<2, 0>(w, out); run<5, 0>(w, out); run<10, 0>(w, out);
    run<10, 1>(w, out); run<10, 2>(w, out);
  }
  return 0;
}
