// fwbf_noise.cu -- the reference channel on the device (see fwbf_noise.cuh):
// y[f][n] = (1 - 2 c_n) + sigma * g_n for frames first..first+count, g from
// numpy's Philox(key=seed, counter=frame << 128) standard-normal stream.
// A separate, register-light kernel: fusing it into the decode kernel cost
// the decoder ~10 % through register spills (round-1 measurement).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fwbf_noise.cuh"

namespace fwbf {

template <typename YT>
__global__ void __launch_bounds__(256)
noise_kernel(unsigned long long seed, long long first, long long count, double sigma,
             const uint32_t *codeword, YT *y, long long ld, int n, int pm) {
  extern __shared__ __align__(16) unsigned long long scratch[];
  for (long long f = blockIdx.x; f < count; f += gridDim.x) {
    gen_frame<YT>(y + f * ld, n, seed, (unsigned long long)(first + f), sigma, codeword, scratch, pm);
  }
}

// one frame per warp (gen_frame_warp), 1 KB of draw window per warp
template <typename YT>
__global__ void __launch_bounds__(128)
noise_kernel_warp(unsigned long long seed, long long first, long long count, double sigma,
                  const uint32_t *codeword, YT *y, long long ld, int n) {
  __shared__ unsigned long long win[4][128];
  const int w = threadIdx.x >> 5;
  for (long long f = (long long)blockIdx.x * 4 + w; f < count; f += (long long)gridDim.x * 4)
    gen_frame_warp<YT>(y + f * ld, n, seed, (unsigned long long)(first + f), sigma, codeword, win[w]);
}

template __global__ void noise_kernel_warp<float>(unsigned long long, long long, long long, double,
                                                  const uint32_t *, float *, long long, int);
template __global__ void noise_kernel_warp<double>(unsigned long long, long long, long long, double,
                                                   const uint32_t *, double *, long long, int);
template __global__ void noise_kernel<float>(unsigned long long, long long, long long, double,
                                             const uint32_t *, float *, long long, int, int);
template __global__ void noise_kernel<double>(unsigned long long, long long, long long, double,
                                              const uint32_t *, double *, long long, int, int);

} // namespace fwbf
