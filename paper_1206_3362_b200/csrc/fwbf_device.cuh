// fwbf_device.cuh -- device helpers shared by the circulant decode kernels
// (fwbf_decode.cu: the general kernel, MODEs 0-2; fwbf_circ.cu: the filtered
// FWBF kernel for circulant codes).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "fwbf_b200.h"
#include "fwbf_internal.h"

namespace fwbf {

#ifndef FULL_MASK
#define FULL_MASK 0xffffffffu
#endif

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// lexicographic (value desc, index asc) -- numpy first-occurrence argmax
__device__ __forceinline__ void amax_combine(double &v, int &i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ __forceinline__ void warp_amax(double &v, int &i) {
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    double v2 = __shfl_xor_sync(FULL_MASK, v, off);
    int i2 = __shfl_xor_sync(FULL_MASK, i, off);
    amax_combine(v, i, v2, i2);
  }
}

// Warp argmax (value desc, index asc) with three single-instruction integer
// reductions (REDUX) instead of a 5-level shuffle butterfly: doubles map to
// order-preserving 64-bit keys, the maximum key's high then low word is found,
// and the lowest index among the lanes holding it.  Same result as warp_amax
// for every non-NaN input (the index of -inf-only lanes is 0x7fffffff).
__device__ __forceinline__ void warp_amax_redux(double &v, int &i) {
  // -0.0 and +0.0 compare equal: normalise so their keys tie too
  unsigned long long k = (unsigned long long)__double_as_longlong(v + 0.0);
  k = (k >> 63) ? ~k : (k | 0x8000000000000000ull);
  const uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
  const uint32_t mh = __reduce_max_sync(FULL_MASK, hi);
  const uint32_t ml = __reduce_max_sync(FULL_MASK, hi == mh ? lo : 0u);
  const bool top = hi == mh && lo == ml;
  i = (int)__reduce_min_sync(FULL_MASK, top ? (uint32_t)i : 0xffffffffu);
  unsigned long long km = ((unsigned long long)mh << 32) | ml;
  km = (km >> 63) ? (km & 0x7fffffffffffffffull) : ~km;
  v = __longlong_as_double((long long)km);
}


// Packed fp32x2 helpers (sm_100 FADD2); always round-to-nearest, no FTZ.
__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2unpack(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Filtered (approximate) gather step: the same 8-byte load, summed directly in
// fp32x2 -- one FADD2 per column pair instead of five.  The result is within
// a per-frame bound delta of the exact sum; selection resolves every decision
// the bound leaves open with the exact column sum (exact_split_metric).
template <int QP, int NP, int TB, bool GO = (QP < NP)> struct GatherF2 {
  static __device__ __forceinline__ void run(unsigned long long (&s)[NP], uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.b64 %0, [%1+%2];" : "=l"(v) : "r"(a), "n"(QP * TB * 8));
    s[QP] = fadd2(s[QP], v);
    GatherF2<QP + 1, NP, TB>::run(s, a);
  }
};
template <int QP, int NP, int TB> struct GatherF2<QP, NP, TB, false> {
  static __device__ __forceinline__ void run(unsigned long long (&)[NP], uint32_t) {}
};

// 16-bit gather step (fwbf_circ.cu, Q16): one 4-byte load brings the signed
// 16-bit quantised minima of a column pair; two IDP.2A add the halves to the
// pair's 32-bit sums (exact integer arithmetic, no carries between halves).
template <int QP, int NP, int TB, bool GO = (QP < NP)> struct GatherQ16 {
  static __device__ __forceinline__ void run(int (&lo)[NP], int (&hi)[NP], uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(QP * TB * 4));
    lo[QP] = __dp2a_lo(v, 0x00000001, lo[QP]);
    hi[QP] = __dp2a_lo(v, 0x00000100, hi[QP]);
    GatherQ16<QP + 1, NP, TB>::run(lo, hi, a);
  }
};
template <int QP, int NP, int TB> struct GatherQ16<QP, NP, TB, false> {
  static __device__ __forceinline__ void run(int (&)[NP], int (&)[NP], uint32_t) {}
};

// MODE 2 coarse argmin correction of a check, in units of the frame's grid G:
// a deterministic function of the check's float32 minima (init and every
// refresh compute the same value), within G/2 + 2^-23 max|y| of min2 - min1.
__device__ __forceinline__ int coarse_dc(float min2, float min1abs, float invG) {
  return __float2int_rn(__fmul_rn(__fsub_rn(min2, min1abs), invG));
}

// ---- TMA bulk copy of one frame row into shared memory (mbarrier completion) ----
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Thread 0, after a CTA barrier that ends every generic access of `dst`:
// order those accesses before the async-proxy write, arm the barrier with the
// byte count and issue the copy.
__device__ __forceinline__ void bulk_row_to_smem(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b),
      "r"(phase)
      : "memory");
}

// Exact Eq.(1) metric of one column on the split path (the filter's fallback,
// MODE 2).  Every signed min1 is a float32 multiple of q and the path guard
// keeps all partial sums of W of them below 2^53 q, so this fp64 sum is exact
// in any order.  The argmin correction is rebuilt exactly from the column's
// own checks: check m = (n - c_j) mod N contributes sgn_m D_m (D_m = (min2 -
// min1) / q from the stored float32 minima, an exact int64) when its argmin is
// n, sgn_m being the sign of its
// min1 copy (the iteration-start syndrome; sbits may already hold this
// iteration's flips).  Subtracting fl(alpha|y_n|) reproduces the exact pass
// (and the reference) bit for bit.
__device__ __forceinline__ double exact_split_metric(const KParams &P, const float *sFA, const uint16_t *sA2,
                                                  const float *sMin2, const float *yabs, int n, int W,
                                                  double qexp, double qinv) {
  const int N = P.n;
  double acc = 0.0;
  long long corr = 0;
  const bool imw = P.wmode == FWBF_WEIGHTS_IMWBF;
  for (int j = 0; j < W; ++j) {
    const int d = n + N - P.off[j]; // check (n - c_j) mod N, read from the first copy
    const int m = d >= N ? d - N : d;
    const float v = sFA[m];
    acc = __dadd_rn(acc, (double)v);
    if (imw && sA2[m] == n) {
      const long long D = (long long)__dmul_rn(__dsub_rn((double)sMin2[m], (double)fabsf(v)), qinv); // exact
      corr += signbit(v) ? -D : D;
    }
  }
  if (corr) acc = __dadd_rn(acc, __dmul_rn((double)corr, qexp));
  return __dsub_rn(acc, __dmul_rn(P.alpha, (double)yabs[n]));
}

} // namespace fwbf
