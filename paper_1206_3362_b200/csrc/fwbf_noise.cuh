// fwbf_noise.cuh -- the reference channel on the device: numpy's
// Philox4x64-10 stream keyed (seed, frame << 128) and its 256-level ziggurat
// standard normal (channel.py:29-50), y = s + sigma * g in float64.
//
// noise_kernel (fwbf_noise.cu): one CTA generates one frame's N normals:
//   A. all threads fill raw[p] (the p-th uint64 of the frame's stream) for
//      p < PM into shared scratch: block b = p / 4 uses counter (b + 1, 0,
//      frame_lo, frame_hi) -- numpy increments before generating;
//   B. warp 0 walks the normals 32 at a time, speculating that each consumes
//      exactly one draw (the 99%-taken fast path); the first lane that needs
//      the slow path (wedge test or tail, further draws) is resolved by one
//      lane, which also yields the position of the next normal.
// Bit-exact with numpy except where CUDA's log1p/exp round differently from
// glibc's inside a tail/wedge decision (measured by tests/test_gpu_noise.py).
#pragma once
#include <stdint.h>
#include "fwbf_ziggurat.h"

namespace fwbf {

static __device__ const double d_zig_w[256] = FWBF_ZIG_W_INIT;
static __device__ const unsigned long long d_zig_k[256] = FWBF_ZIG_K_INIT;
static __device__ const double d_zig_f[256] = FWBF_ZIG_F_INIT;

struct U4 { unsigned long long v[4]; };

__device__ __forceinline__ U4 philox4x64_10(unsigned long long c0, unsigned long long c1,
                                            unsigned long long c2, unsigned long long c3,
                                            unsigned long long k0, unsigned long long k1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const unsigned long long W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const unsigned long long hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const unsigned long long n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += W0; k1 += W1;
  }
  U4 o;
  o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

struct NoiseStream {
  unsigned long long key0, frame;
  const unsigned long long *raw; // shared scratch: raw[p - p0] for p0 <= p < p0 + pm
  int pm;
  long long p0 = 0;
  __device__ unsigned long long at(long long p) const {
    if (p >= p0 && p < p0 + pm) return raw[p - p0];
    const unsigned long long b = (unsigned long long)(p >> 2) + 1ull;
    const U4 o = philox4x64_10(b, 0ull, frame, 0ull, key0, 0ull);
    return o.v[p & 3];
  }
  __device__ static double dbl(unsigned long long u) {
    return __dmul_rn((double)(u >> 11), 1.0 / 9007199254740992.0);
  }
};

// Slow path of one normal whose first draw (already split) failed the fast
// test; `pos` is the position after that draw.  Returns the value, advances pos.
__device__ __forceinline__ double zig_slow(const NoiseStream &s, long long &pos, int idx,
                                        unsigned long long rabs, double x) {
  const double R = FWBF_ZIG_R;
  const double inv_r = 1.0 / FWBF_ZIG_R;
  for (;;) {
    if (idx == 0) {
      for (;;) {
        const double u1 = NoiseStream::dbl(s.at(pos++));
        const double u2 = NoiseStream::dbl(s.at(pos++));
        const double xx = __dmul_rn(-inv_r, log1p(-u1));
        const double yy = -log1p(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
          return ((rabs >> 8) & 1ull) ? -__dadd_rn(R, xx) : __dadd_rn(R, xx);
      }
    } else {
      const double u = NoiseStream::dbl(s.at(pos++));
      const double fa = __ldg(&d_zig_f[idx - 1]), fb = __ldg(&d_zig_f[idx]);
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(fa, fb), u), fb);
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) return x;
    }
    // rejected: start over with a fresh draw
    unsigned long long r = s.at(pos++);
    idx = (int)(r & 0xffull);
    r >>= 8;
    const bool neg = r & 1ull;
    rabs = (r >> 1) & 0x000fffffffffffffull;
    x = __dmul_rn((double)rabs, __ldg(&d_zig_w[idx]));
    if (neg) x = -x;
    if (rabs < __ldg(&d_zig_k[idx])) return x;
  }
}

// Fill ybuf[0..N) with y_n = s_n + sigma * g_n for one frame (all threads call;
// contains __syncthreads).  s_n = 1 - 2 c_n with c from codeword (NULL = 0).
template <typename YT>
__device__ void gen_frame(YT *ybuf, int N, unsigned long long seed, unsigned long long frame,
                          double sigma, const uint32_t *codeword, unsigned long long *scratch,
                          int pm) {
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31;
  if (sigma == 0.0) { // awgn_apply returns s unchanged and draws nothing (channel.py:34-35)
    for (int n = tid; n < N; n += T) {
      const int c = codeword ? (int)((__ldg(codeword + (n >> 5)) >> (n & 31)) & 1u) : 0;
      ybuf[n] = (YT)(c ? -1.0 : 1.0);
    }
    __syncthreads();
    return;
  }
  const int nblk = pm >> 2;
  for (int b = tid; b < nblk; b += T) {
    const U4 o = philox4x64_10((unsigned long long)b + 1ull, 0ull, frame, 0ull, seed, 0ull);
    scratch[4 * b + 0] = o.v[0];
    scratch[4 * b + 1] = o.v[1];
    scratch[4 * b + 2] = o.v[2];
    scratch[4 * b + 3] = o.v[3];
  }
  __syncthreads();
  if (tid < 32) {
    NoiseStream s{seed, frame, scratch, pm & ~3};
    long long p = 0;
    int k = 0;
    while (k < N) {
      unsigned long long r = s.at(p + lane);
      const int idx = (int)(r & 0xffull);
      r >>= 8;
      const bool neg = r & 1ull;
      const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffull;
      double x = __dmul_rn((double)rabs, __ldg(&d_zig_w[idx]));
      if (neg) x = -x;
      const bool fast = rabs < __ldg(&d_zig_k[idx]);
      const uint32_t slow = __ballot_sync(0xffffffffu, !fast);
      const int sl = slow ? __ffs(slow) - 1 : 32;
      const int nv = min(sl, N - k);
      if (lane < nv) {
        const int n = k + lane;
        const int c = codeword ? (int)((__ldg(codeword + (n >> 5)) >> (n & 31)) & 1u) : 0;
        ybuf[n] = (YT)__dadd_rn(c ? -1.0 : 1.0, __dmul_rn(sigma, x));
      }
      if (sl < 32 && k + sl < N) {
        long long pos = p + sl + 1;
        double v = 0.0;
        if (lane == sl) v = zig_slow(s, pos, idx, rabs, x);
        v = __shfl_sync(0xffffffffu, v, sl);
        pos = __shfl_sync(0xffffffffu, pos, sl);
        if (lane == 0) {
          const int n = k + sl;
          const int c = codeword ? (int)((__ldg(codeword + (n >> 5)) >> (n & 31)) & 1u) : 0;
          ybuf[n] = (YT)__dadd_rn(c ? -1.0 : 1.0, __dmul_rn(sigma, v));
        }
        k += sl + 1;
        p = pos;
      } else {
        k += nv;
        p += nv;
      }
    }
  }
  __syncthreads();
}

// Warp-level generator: one warp produces one frame with a rolling window of
// 128 draws in shared memory (each lane computes one Philox block = 4 draws
// per refill), so every warp of the CTA walks its own frame -- no CTA
// barriers and 4x the concurrent walkers of gen_frame at the same occupancy.
template <typename YT>
__device__ void gen_frame_warp(YT *ybuf, int N, unsigned long long seed, unsigned long long frame,
                               double sigma, const uint32_t *codeword, unsigned long long *win) {
  const int lane = threadIdx.x & 31;
  constexpr int WIN = 128;
  if (sigma == 0.0) { // awgn_apply returns s unchanged and draws nothing (channel.py:34-35)
    for (int n = lane; n < N; n += 32) {
      const int c = codeword ? (int)((__ldg(codeword + (n >> 5)) >> (n & 31)) & 1u) : 0;
      ybuf[n] = (YT)(c ? -1.0 : 1.0);
    }
    return;
  }
  NoiseStream s{seed, frame, win, WIN};
  s.p0 = -WIN; // empty window
  long long p = 0;
  int k = 0;
  while (k < N) {
    if (p + 32 > s.p0 + WIN) { // refill: the window starts at p's Philox block
      __syncwarp();
      s.p0 = p & ~3ll;
      const U4 o = philox4x64_10((unsigned long long)(s.p0 >> 2) + 1ull + lane, 0ull, frame, 0ull, seed, 0ull);
      win[4 * lane + 0] = o.v[0];
      win[4 * lane + 1] = o.v[1];
      win[4 * lane + 2] = o.v[2];
      win[4 * lane + 3] = o.v[3];
      __syncwarp();
    }
    unsigned long long r = s.at(p + lane);
    const int idx = (int)(r & 0xffull);
    r >>= 8;
    const bool neg = r & 1ull;
    const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)rabs, __ldg(&d_zig_w[idx]));
    if (neg) x = -x;
    const bool fast = rabs < __ldg(&d_zig_k[idx]);
    const uint32_t slow = __ballot_sync(0xffffffffu, !fast);
    const int sl = slow ? __ffs(slow) - 1 : 32;
    const int nv = min(sl, N - k);
    if (lane < nv) {
      const int n = k + lane;
      const int c = codeword ? (int)((__ldg(codeword + (n >> 5)) >> (n & 31)) & 1u) : 0;
      ybuf[n] = (YT)__dadd_rn(c ? -1.0 : 1.0, __dmul_rn(sigma, x));
    }
    if (sl < 32 && k + sl < N) {
      long long pos = p + sl + 1;
      double v = 0.0;
      if (lane == sl) v = zig_slow(s, pos, idx, rabs, x);
      v = __shfl_sync(0xffffffffu, v, sl);
      pos = __shfl_sync(0xffffffffu, pos, sl);
      if (lane == 0) {
        const int n = k + sl;
        const int c = codeword ? (int)((__ldg(codeword + (n >> 5)) >> (n & 31)) & 1u) : 0;
        ybuf[n] = (YT)__dadd_rn(c ? -1.0 : 1.0, __dmul_rn(sigma, v));
      }
      k += sl + 1;
      p = pos;
    } else {
      k += nv;
      p += nv;
    }
  }
  __syncwarp();
}

} // namespace fwbf
