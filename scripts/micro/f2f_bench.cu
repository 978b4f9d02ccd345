// Microbenchmark: throughput of the gather inner loop variants on one SM-full grid.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(const double* gd, const float* gf, double* out, int iters) {
  __shared__ double sd[2048];
  __shared__ float sf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) { sd[i] = gd[i]; sf[i] = gf[i]; }
  __syncthreads();
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int base = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    int o = (it * 37) & 511;
    if (MODE == 0) {  // LDS.64 + DADD
      a0 += sd[base + o]; a1 += sd[base + o + 256]; a2 += sd[base + o + 512]; a3 += sd[base + o + 768];
    } else if (MODE == 1) {  // LDS.32 + F2F + DADD
      a0 += (double)sf[base + o]; a1 += (double)sf[base + o + 256]; a2 += (double)sf[base + o + 512]; a3 += (double)sf[base + o + 768];
    } else {  // ATOMS.XOR spread
      atomicXor((unsigned*)&sf[(base * 7 + it) & 2047], 1u << (it & 31));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main() {
  double *gd, *out; float* gf;
  cudaMalloc(&gd, 2048 * 8); cudaMalloc(&gf, 2048 * 4); cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaMemset(gd, 0, 2048 * 8); cudaMemset(gf, 0, 2048 * 4);
  int iters = 20000;
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 8, 256>>>(gd, gf, out, iters);
      if (mode == 1) k<1><<<148 * 8, 256>>>(gd, gf, out, iters);
      if (mode == 2) k<2><<<148 * 8, 256>>>(gd, gf, out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 148.0 * 8 * 256 * iters * (mode == 2 ? 1 : 4);
    printf("mode %d: %.3f ms, %.3f G-lane-ops/s, %.2f lane-ops/clk/SM @1.965GHz\n", mode, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
