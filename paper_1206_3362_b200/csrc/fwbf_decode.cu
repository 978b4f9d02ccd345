// fwbf_decode.cu -- batched weighted bit-flipping LDPC decoding on B200 (sm_100a).
//
// One persistent CTA decodes one frame at a time, pulling frame indices from an
// atomic work queue (iteration counts vary 0..k_max per frame).  All per-frame
// state lives in shared memory; H lives in kernel parameters (circulant offsets)
// or in small read-only global tables (explicit CSR/CSC).
//
// Reference semantics (/root/reference/pkg/src/fwbf/decoders.py):
//   init        :191-198  |y|, hard decision, syndrome, per-check min1/min2/argmin
//   loop        :204-229  converged? -> k_max? -> Eq.(1) metric -> select -> flip
//   metric      :148-153  E_n = fl(sum_{m in M(n), ascending} (2s_m-1) w_nm) - fl(alpha|y_n|)
//   selection   :156-183  block argmax (+ threshold), global argmax, top-lambda
//
// Three metric paths, selected per frame:
//   0 ORDERED: the column sum in ascending check order with fp64 adds, exactly
//     the reference's np.bincount sequence.  Bit-exact for any input.
//   1 GUARDED fp64 (float32 y, circulant H): order-free sum over doubled
//     shared arrays.  All weights are float32 values, i.e. multiples of
//     q = 2^(e_min - 23); if 2*dv*max|y| < 2^53 q every fp64 add is exact, so
//     the result equals the reference's sum regardless of order.
//   2 SPLIT fp32 (compile-time weight): each weight v = h + l on the grid
//     G = 2^g q, h and l summed exactly in packed fp32 (FADD2); argmin
//     min2 - min1 corrections as exact int32 limb pairs.
// Frames failing a guard fall to the next path (flags record which).
// Other passes: the fused metric + block argmax for explicit/QC codes with
// 32 | p (no metric buffer) and, in the INC kernels, IMWBF's incremental
// integer metric.
//
// Kernel MODEs (template): 0 exact (the paths above, any algorithm); 1 IMWBF
// incremental metric; 2 FWBF filtered metric -- frames passing the fp64 guard
// sum the float32 minima directly (one FADD2 per column pair per check),
// store the metric as float, and the selection re-decides every block whose
// decision is within the frame's error bound of changing with exact column
// sums.  MODE 2 also has its own, smaller shared-memory
// layout (5 CTAs/SM on EG(1023)) with coarse integer argmin corrections.
//
// Ties: every argmax takes the lowest index (numpy argmax / stable argsort).

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "fwbf_b200.h"
#include "fwbf_internal.h"
#include "fwbf_device.cuh"

#ifndef FWBF_MINB_256
#define FWBF_MINB_256 4
#endif
#ifndef FWBF_MINB_256_FILT
#define FWBF_MINB_256_FILT 5
#endif

namespace fwbf {


// ---------------------------------------------------------------------------
// Shared-memory layout (byte offsets computed on the host, see plan_layout).
// ---------------------------------------------------------------------------
struct Smem {
  unsigned char *base;
  const KParams &P;
  __device__ Smem(unsigned char *b, const KParams &p) : base(b), P(p) {}
  template <typename T> __device__ T *at(int off) const { return reinterpret_cast<T *>(base + off); }
};

// One column-slot step of the guarded gather: select the min1 or min2 array
// by the argmin mask bit, load with the slot's compile-time offset Q*TB*8.
template <int Q, int KC, int TB> struct GatherQ {
  static __device__ __forceinline__ void run(double (&acc)[KC], const uint32_t (&mk)[KC], uint32_t bit,
                                             uint32_t a1, uint32_t a2) {
    const uint32_t a = (mk[Q] & bit) ? a2 : a1;
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(Q * TB * 8));
    acc[Q] = __dadd_rn(acc[Q], v);
    GatherQ<Q + 1, KC, TB>::run(acc, mk, bit, a1, a2);
  }
};
template <int KC, int TB> struct GatherQ<KC, KC, TB> {
  static __device__ __forceinline__ void run(double (&)[KC], const uint32_t (&)[KC], uint32_t, uint32_t, uint32_t) {}
};


template <int KC> struct SplitPairs { static constexpr int value = KC / 2 > 0 ? KC / 2 : 1; };

// Split-fp32 gather step for column pair slot QP: one 8-byte load brings the
// float32 signed min1 of two adjacent columns (n, n+1); each value v is split
// exactly as v = h + l on the grid G (t = v + C, h = t - C, l = v - h, with
// C = 1.5 * 2^23 * G), and h, l are accumulated in separate fp32x2 sums.
template <int QP, int NP, int TB, bool GO = (QP < NP)> struct GatherP2 {
  static __device__ __forceinline__ void run(unsigned long long (&hi)[NP], unsigned long long (&lo)[NP],
                                             uint32_t a, unsigned long long cc) {
    unsigned long long v;
    asm volatile("ld.shared.b64 %0, [%1+%2];" : "=l"(v) : "r"(a), "n"(QP * TB * 8));
    const unsigned long long h = fsub2(fadd2(v, cc), cc);
    hi[QP] = fadd2(hi[QP], h);
    lo[QP] = fadd2(lo[QP], fsub2(v, h));
    GatherP2<QP + 1, NP, TB>::run(hi, lo, a, cc);
  }
};
template <int QP, int NP, int TB> struct GatherP2<QP, NP, TB, false> {
  static __device__ __forceinline__ void run(unsigned long long (&)[NP], unsigned long long (&)[NP], uint32_t,
                                             unsigned long long) {}
};


// Split-path refresh of check m = tid + KK*TB (compile-time KK): shared
// addresses come in pinned registers (base + KK*TB*size as immediates), so
// the four sign-negating stores and the correction-limb atomics need no
// per-check address arithmetic.
struct RefreshAddr {
  uint32_t fa, fa2, fb, fb2, m2, a2, corr, invg;
};
// CC (MODE 2): the argmin column's correction is one int32 on the coarse grid
// (m2 addresses the per-check Dc, corr the per-column Cc): one atomic.
template <int KK, int KC, int TB, bool CC = false, bool GO = (KK < KC)> struct RefreshKK {
  static __device__ __forceinline__ void run(const RefreshAddr &A, const uint32_t *sbits, uint32_t &sprev,
                                             int &pc, int tid, int warp, int lane, int M, bool imw) {
    if (KK * TB + warp * 32 < M) { // warp-uniform: this warp's word exists
      const uint32_t word = sbits[(KK * TB + warp * 32) >> 5];
      const bool s = (word >> lane) & 1u;
      const bool tog = (tid + KK * TB < M) && (s != (bool)((sprev >> KK) & 1u));
      if (tog) {
        float v;
        asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(A.fa), "n"(4 * KK * TB));
        v = -v;
        asm volatile("st.shared.f32 [%0+%1], %2;" ::"r"(A.fa), "n"(4 * KK * TB), "f"(v));
        asm volatile("st.shared.f32 [%0+%1], %2;" ::"r"(A.fa2), "n"(4 * KK * TB), "f"(v));
        asm volatile("st.shared.f32 [%0+%1], %2;" ::"r"(A.fb), "n"(4 * KK * TB), "f"(v));
        asm volatile("st.shared.f32 [%0+%1], %2;" ::"r"(A.fb2), "n"(4 * KK * TB), "f"(v));
        if (CC && imw) { // correction sign flips with s_m: +-2 Dc (Dc from the float minima)
          float mn2;
          unsigned short a2;
          asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(mn2) : "r"(A.m2), "n"(4 * KK * TB));
          asm volatile("ld.shared.u16 %0, [%1+%2];" : "=h"(a2) : "r"(A.a2), "n"(2 * KK * TB));
          const int dc = coarse_dc(mn2, fabsf(v), __uint_as_float(A.invg));
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(A.corr + 4u * (uint32_t)a2), "r"(s ? 2 * dc : -2 * dc));
        } else if (imw) { // correction sign flips with s_m
          int dx, dy;
          unsigned short a2;
          asm volatile("ld.shared.v2.s32 {%0, %1}, [%2+%3];" : "=r"(dx), "=r"(dy) : "r"(A.m2), "n"(8 * KK * TB));
          asm volatile("ld.shared.u16 %0, [%1+%2];" : "=h"(a2) : "r"(A.a2), "n"(2 * KK * TB));
          const uint32_t cp = A.corr + 8u * (uint32_t)a2;
          if (!s) { dx = -dx; dy = -dy; }
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(cp), "r"(dx));
          asm volatile("red.shared.add.s32 [%0+4], %1;" ::"r"(cp), "r"(dy));
        }
      }
      sprev ^= (tog ? 1u : 0u) << KK;
      pc += __popc(word);
    }
    RefreshKK<KK + 1, KC, TB, CC>::run(A, sbits, sprev, pc, tid, warp, lane, M, imw);
  }
};
template <int KK, int KC, int TB, bool CC> struct RefreshKK<KK, KC, TB, CC, false> {
  static __device__ __forceinline__ void run(const RefreshAddr &, const uint32_t *, uint32_t &, int &, int, int,
                                             int, int, bool) {}
};


// Exact argmin corrections as two int32 limbs: D = lo + hi * 2^24 with
// lo in [0, 2^24) (D an integer multiple of the frame quantum q).
__device__ __forceinline__ void corr_add(int *corr, int col, long long D, int sign) {
  const int lo = (int)(D & 0xffffffll);
  const int hi = (int)(D >> 24);
  atomicAdd(&corr[2 * col], sign * lo);
  atomicAdd(&corr[2 * col + 1], sign * hi);
}

template <typename YT>
__device__ __forceinline__ YT load_y(const KParams &P, long long f, int n) {
  const YT *y = reinterpret_cast<const YT *>(P.y);
  return __ldg(y + f * P.ld + n);
}


// ---------------------------------------------------------------------------
// The decode kernel.
//   YT   : float (float32 channel output) or double
//   CIRC : circulant H (index arithmetic) vs explicit CSR/CSC tables
//   KC   : columns per thread on the guarded path (register accumulators)
// ---------------------------------------------------------------------------
template <typename YT, bool CIRC, int KC, int TB, int WT, int MODE>
__global__ void __launch_bounds__(TB ? TB : 1024, TB == 256 ? (MODE == 2 ? FWBF_MINB_256_FILT : FWBF_MINB_256) : 1024 / (TB ? TB : 1024))
decode_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool INC = MODE == 1;  // IMWBF incremental integer metric
  constexpr bool FILT = MODE == 2; // FWBF filtered metric on split-path frames
  const int tid = threadIdx.x;
  const int T = TB ? TB : (int)blockDim.x;  // compile-time on the guarded path
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nwarps = T >> 5;
  const int N = P.n;
  const int M = P.m;

  // frame row: staged by a bulk copy (P.y_stage) or loaded element-wise
  YT *ybuf = reinterpret_cast<YT *>(smem_raw + (P.y_stage ? P.off_ystage : P.off_y));
  double *Ebuf = reinterpret_cast<double *>(smem_raw + P.off_e);
  double *chk1 = reinterpret_cast<double *>(smem_raw + P.off_chk1); // min1 (signed); doubled on the guarded path
  double *chk2 = reinterpret_cast<double *>(smem_raw + P.off_chk2); // min2 (signed); doubled on the guarded path
  int *amin = reinterpret_cast<int *>(smem_raw + P.off_amin);        // ordered path argmin column
  uint32_t *amask = reinterpret_cast<uint32_t *>(smem_raw + P.off_amask); // guarded: per-column argmin j-mask
  uint32_t *sbits = reinterpret_cast<uint32_t *>(smem_raw + P.off_sbits);
  uint32_t *zbits = reinterpret_cast<uint32_t *>(smem_raw + P.off_zbits);
  double *blk_v = reinterpret_cast<double *>(smem_raw + P.off_blkv);
  int *blk_i = reinterpret_cast<int *>(smem_raw + P.off_blki);
  int *flips = reinterpret_cast<int *>(smem_raw + P.off_flips);
  int *offs_s = reinterpret_cast<int *>(smem_raw + P.off_offs);     // circulant offsets (for divergent j)
  double *red_v = reinterpret_cast<double *>(smem_raw + P.off_red);
  int *red_i = reinterpret_cast<int *>(smem_raw + P.off_red + 32 * 8);
  int *misc = reinterpret_cast<int *>(smem_raw + P.off_misc);
  float *redf = reinterpret_cast<float *>(smem_raw + P.off_misc + 16 * 4);
  // misc slots
  enum { S_FRAME = 0, S_F, S_SWT, S_GBEST, S_FAST, S_NONFIN, S_BITERR, S_EQ, S_FB, S_VMAX, S_YMAX };
  // fused metric + block argmax (explicit/QC codes, FWBF, p % 32 == 0): no
  // metric buffer; the flip counter alternates between S_F and S_FB by
  // iteration parity because flips are counted during the metric pass
  const bool fused = !CIRC && P.fused;

  const int W = WT ? WT : P.w;       // circulant weight (0 explicit); compile-time when WT > 0
  constexpr bool kGuard = CIRC && sizeof(YT) == 4; // guarded paths exist for float32 y only
  const int aw = (W > 32) ? 2 : 1;   // amask words per column
  const int qlz = P.qc_z ? __ffs(P.qc_z) - 1 : 0; // log2 Z (QC: Z a power of two)

  if (CIRC) {
    for (int j = tid; j < W; j += T) {
      offs_s[j] = P.off[j];
      offs_s[64 + j] = P.dneg[j];
      offs_s[64 + W + j] = P.dneg[j];
      offs_s[192 + j] = P.off[j] - N; // rotated walk of a check's columns: the
      offs_s[192 + W + j] = P.off[j]; // wrapped (smaller) ones first, no wrap test
    }
  }
  if (tid == 0) misc[S_NONFIN] = 0;

  // FWBF block-argmax group geometry (fixed for the launch).  Odd p: the
  // 16/TPB groups of a half-warp take blocks TPB apart, so their lanes' words
  // land in distinct banks (p*TPB*i + s, i < 16/TPB, s < TPB).
  const int sel_lt = P.log2_tpb;
  const int sel_sub = tid & ((1 << sel_lt) - 1);
  const int sel_gpc = T >> sel_lt;
  int sel_slot = tid >> sel_lt;
  if (P.sel_spread) {
    const int hw = tid >> 4, half = 16 >> sel_lt, tpb = 1 << sel_lt;
    sel_slot = (hw / tpb) * 16 + tpb * (sel_slot & (half - 1)) + (hw % tpb);
  }
  const int sel_rounds = (P.nblocks + sel_gpc - 1) / sel_gpc;

  // optional per-phase cycle accounting (thread 0, at CTA-wide barriers)
  __shared__ long long ph_acc[9]; // [8] = last timestamp
  if (tid < 9) ph_acc[tid] = 0;
#define FWBF_PH(i)                                              \
  if (P.phase_cycles && tid == 0) {                             \
    const long long t_ = clock64();                             \
    if (ph_acc[8]) ph_acc[i] += t_ - ph_acc[8];                 \
    ph_acc[8] = t_;                                             \
  }

  // per-CTA counter accumulation (thread 0)
  long long c_frames = 0, c_biterr = 0, c_worderr = 0, c_iters = 0, c_flips = 0,
            c_stalls = 0, c_conv = 0, c_ordered = 0, c_edges = 0;

  const int zw = (N + 31) >> 5;
  const int nKy = (N + T - 1) / T; // rounds over columns
  const int nKm = (M + T - 1) / T; // rounds over checks

  // Staged input: the frame queue is claimed one frame ahead and that frame's
  // y row is copied into ybuf by the TMA engine while the current frame
  // iterates (issued after the current frame's last read of ybuf).
  __shared__ __align__(8) uint64_t ystage_bar;
  unsigned ystage_phase = 0;
  const bool ystage = P.y_stage != 0;
  if (ystage && tid == 0) {
    mbar_init(&ystage_bar, 1);
    const unsigned t0 = atomicAdd(P.work_counter, 1u);
    misc[S_FRAME] = (int)t0;
    if ((long long)t0 < P.batch)
      bulk_row_to_smem(ybuf, reinterpret_cast<const YT *>(P.y) + (long long)t0 * P.ld, (unsigned)P.ystage_bytes,
                       &ystage_bar);
  }

  for (;;) {
    __syncthreads();
    if (!ystage && tid == 0) misc[S_FRAME] = (int)atomicAdd(P.work_counter, 1u);
    __syncthreads();
    FWBF_PH(0)
    // tickets are unsigned: batch <= 2^31 - 1 plus one extra ticket per CTA
    // stays below 2^32, so the queue end is always seen
    long long f = (long long)(unsigned)misc[S_FRAME];
    if (P.frame_list) { // frames deferred by the filtered circulant kernel (fwbf_circ.cu)
      if (f >= (long long)*P.frame_count) break;
      f = P.frame_list[f];
    } else if (f >= P.batch) {
      break;
    }
    if (ystage) { // this frame's row has landed in ybuf
      mbar_wait(&ystage_bar, ystage_phase);
      ystage_phase ^= 1u;
    }

    // ---------------- init 1: y -> smem, hard decisions, guard statistics -------
    float lmin = INFINITY, lmax = 0.f;
    bool nonfin = false;
    for (int k = 0; k < nKy; ++k) {
      const int n = tid + k * T;
      const bool ok = n < N;
      YT v = ok ? (ystage ? ybuf[n] : load_y<YT>(P, f, n)) : YT(0);
      if (ok) ybuf[n] = v + YT(0); // -0.0 -> +0.0: the sign bit of ybuf is the hard decision (y < 0)
      const uint32_t b = __ballot_sync(FULL_MASK, ok && (v < YT(0)));
      if (lane == 0 && (k * T + warp * 32) < N) zbits[(k * T + warp * 32) >> 5] = b;
      if (ok) {
        if (!isfinite((double)v)) nonfin = true;
        float a = fabsf((float)v);
        if (a > 0.f) lmin = fminf(lmin, a);
        lmax = fmaxf(lmax, a);
        if (CIRC) {
          for (int q = 0; q < aw; ++q) amask[n * aw + q] = 0u;
          if (WT > 0 && sizeof(YT) == 4) {
            int *cz = reinterpret_cast<int *>(smem_raw + P.off_corr);
            if (FILT) {
              cz[n] = 0; // MODE 2: one coarse correction per column
            } else {
              cz[2 * n] = 0;
              cz[2 * n + 1] = 0;
            }
          }
        }
      }
    }
    // block reduce (min nonzero |y|, max |y|, nonfinite)
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      lmin = fminf(lmin, __shfl_xor_sync(FULL_MASK, lmin, off));
      lmax = fmaxf(lmax, __shfl_xor_sync(FULL_MASK, lmax, off));
    }
    nonfin = __any_sync(FULL_MASK, nonfin);
    if (lane == 0) { redf[warp] = lmin; redf[32 + warp] = lmax; if (nonfin) misc[S_NONFIN] = 1; }
    if (tid == 0) { misc[S_SWT] = 0; misc[S_F] = 0; misc[S_FB] = 0; }
    __syncthreads();
    FWBF_PH(1)
    if (tid == 0) {
      float mn = INFINITY, mx = 0.f;
      for (int w2 = 0; w2 < nwarps; ++w2) { mn = fminf(mn, redf[w2]); mx = fmaxf(mx, redf[32 + w2]); }
      // path: 0 ordered, 1 guarded fp64, 2 guarded split-fp32 (compile-time W)
      int fast = 0;
      float cmag = 0.f;
      if (CIRC && sizeof(YT) == 4 && !P.force_ordered && !misc[S_NONFIN]) {
        if (!(mn < INFINITY)) {
          fast = 1; // all |y| == 0: every weight is 0, sums trivially exact
          misc[S_EQ] = -200; // (no quantum: keeps the split re-check below off)
        } else {
          int e = ((__float_as_int(mn) >> 23) & 0xff) - 127;
          if (e < -126) e = -126;
          // quantum q = 2^(e-23); need 2*dv*max|y| < 2^53 * q = 2^(30+e)
          double lhs = 2.0 * (double)W * (double)mx;
          fast = lhs < ldexp(1.0, 30 + e);
          // split-fp32: grid G = 2^g q with W * 2^(g-1) <= 2^24 (g = 20 for
          // W <= 32, 19 for W <= 64), so every partial lo sum (multiples of q,
          // |l| <= G/2) stays within 2^24 q; every column sum of |w| must stay
          // below 2^23 G = 2^(g+e) so the hi sums (multiples of G, plus at most
          // W G/2 of rounding) stay below 2^24 G.  Both exact in fp32.
          // C = 1.5 * 2^23 * G keeps t = v + C in [2^23 G, 2^24 G].
          constexpr int kG = (WT > 32) ? 19 : 20;
          if (fast && WT > 0 && WT <= 64 && (KC % 2) == 0 && e >= -100 && e <= 100 && !P.no_split &&
              (double)W * (double)mx <= ldexp(1.0, kG + e)) {
            fast = 2;
            cmag = ldexpf(1.5f, kG + e); // C = 1.5 * 2^23 G, finite for e <= 100
          }
          misc[S_EQ] = e - 23; // quantum q = 2^(e-23)
        }
      }
      redf[0] = cmag;
      misc[S_FAST] = fast;
      misc[S_VMAX] = 0;                  // largest check minimum (filter bound), see init 2
      misc[S_YMAX] = __float_as_int(mx); // max |y| (float bits; nonnegative, so int order = float order)
    }
    __syncthreads();
    int fpath = misc[S_FAST];
    bool fastp = fpath != 0;
    bool split = fpath == 2;
    float cmag = redf[0];
    double qexp = split ? ldexp(1.0, misc[S_EQ]) : 0.0;      // q
    double qinv = split ? ldexp(1.0, -misc[S_EQ]) : 0.0;     // 1/q
    float *sFA = reinterpret_cast<float *>(smem_raw + P.off_fa);   // split: signed min1, 8B-aligned at even n
    float *sFB = reinterpret_cast<float *>(smem_raw + P.off_fb);   // split: same, shifted by one element
    int *sM2 = reinterpret_cast<int *>(smem_raw + P.off_m2s);      // split: correction limb deltas per check
    uint16_t *sA2 = reinterpret_cast<uint16_t *>(smem_raw + P.off_a2m); // split: argmin column per check
    int *sCorr = reinterpret_cast<int *>(smem_raw + P.off_corr);   // split: per column (lo, hi) limbs
    double *sAY = reinterpret_cast<double *>(smem_raw + P.off_ay); // split: fl(alpha |y_n|)

    // ---------------- init 2: per-check minima, syndrome, signed weights --------
    const bool nonfin_frame = misc[S_NONFIN] != 0; // NaN/inf: keep the compare-based scan
    uint32_t sprev = 0; // syndrome bits of this thread's checks tid + k*T
    // Circulant float32 kernels with compile-time shape keep each check's
    // (min1, min2, argmin) in registers between the scan and the stores: the
    // split-fp32 guard can then be re-evaluated on the largest min1 (the
    // values the split sums actually see) instead of max|y| -- about ten times
    // looser -- before any path-specific state is written.
    constexpr bool kTwoPhase = kGuard && TB > 0 && WT > 0 && (KC % 2) == 0 && WT <= 64;
    // MODE 2 argmin corrections on a coarse grid G = 2^gsh q: one int32 per
    // column (Cc, in the first half of sCorr), per check the exact D (int64, in
    // sM2) and its grid value Dc (int32, second half of sCorr)
    int gsh = 0;
    float Gf = 0.f, invGf = 0.f;
    constexpr int KR = kTwoPhase ? KC : 1;
    YT r_min1[KR], r_min2[KR];
    int r_ac[KR];
    if (kTwoPhase) {
      float wmax = 0.f; // largest min1 of this thread's checks
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int m = tid + k * T;
        const bool ok = m < M;
        int par = 0;
        YT min1 = YT(INFINITY), min2 = YT(INFINITY);
        int ac = 0x7fffffff;
        if (ok) {
          if (kGuard && !nonfin_frame) {
            // columns in ascending order (m + c_j - N for j >= jw, then m + c_j),
            // so strict < keeps the lowest column on ties; min2 = second smallest
            // of the multiset (min(min2, max(min1, a)))
            const int *orr = offs_s + 192 + __ldg(P.jwtab + m);
            uint32_t sgn = 0; // parity = XOR of the sign bits (ybuf holds no -0.0, no NaN here)
            for (int t = 0; t < W; ++t) {
              const int c = m + orr[t];
              const YT yv = ybuf[c];
              sgn ^= __float_as_uint((float)yv);
              const YT a = fabs(yv);
              const bool lt = a < min1;
              min2 = fminf(min2, fmaxf(min1, a));
              min1 = fminf(min1, a);
              ac = lt ? c : ac;
            }
            par = (int)(sgn >> 31);
          } else if (CIRC) {
            for (int j = 0; j < W; ++j) {
              int c = m + P.off[j];
              if (c >= N) c -= N;
              const YT yv = ybuf[c];
              par ^= (yv < YT(0));
              const YT a = fabs(yv);
              if (a < min1 || (a == min1 && c < ac)) { min2 = min1; min1 = a; ac = c; }
              else if (a < min2) min2 = a;
            }
          } else if (P.qc_z) {
            // quasi-cyclic: row r*Z + i holds column cb*Z + ((i + s[r][cb]) mod Z)
            const int Z = P.qc_z, r = m >> qlz, ii = m & (Z - 1);
            for (int cb = 0; cb < P.qc_kb; ++cb) {
              const int sh = P.qc_shift[r * P.qc_kb + cb];
              if (sh < 0) continue;
              const int c = cb * Z + ((ii + sh) & (Z - 1));
              const YT yv = ybuf[c];
              par ^= (yv < YT(0));
              const YT a = fabs(yv);
              if (a < min1 || (a == min1 && c < ac)) { min2 = min1; min1 = a; ac = c; }
              else if (a < min2) min2 = a;
            }
          } else {
            const int e0 = __ldg(P.row_ptr + m), e1 = __ldg(P.row_ptr + m + 1);
            for (int e = e0; e < e1; ++e) {
              const int c = __ldg(P.row_idx + e);
              const YT yv = ybuf[c];
              par ^= (yv < YT(0));
              const YT a = fabs(yv);
              if (a < min1 || (a == min1 && c < ac)) { min2 = min1; min1 = a; ac = c; }
              else if (a < min2) min2 = a;
            }
          }
        }
        if (ok && par) sprev |= 1u << k;
        const uint32_t b = __ballot_sync(FULL_MASK, ok && par);
        if (lane == 0 && (k * T + warp * 32) < M) {
          sbits[(k * T + warp * 32) >> 5] = b;
          atomicAdd(&misc[S_SWT], __popc(b));
        }
        r_min1[k] = min1;
        r_min2[k] = min2;
        r_ac[k] = ac;
        if (ok) wmax = fmaxf(wmax, (float)min1);
      }
      if (FILT && fpath != 0) { // CTA max of the check minima: the filter's error bound
        for (int off = 16; off; off >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(FULL_MASK, wmax, off));
        if (lane == 0) atomicMax(&misc[S_VMAX], __float_as_int(wmax));
      }
      if (fpath == 1 && !P.no_split && misc[S_EQ] >= -123 && misc[S_EQ] <= 77) { // uniform: fp64-guarded, not yet split
        for (int off = 16; off; off >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(FULL_MASK, wmax, off));
        if (lane == 0) redf[32 + warp] = wmax; // init1's slots, already consumed
        __syncthreads();
        if (tid == 0) {
          float mx1 = 0.f;
          for (int w2 = 0; w2 < nwarps; ++w2) mx1 = fmaxf(mx1, redf[32 + w2]);
          constexpr int kG = (WT > 32) ? 19 : 20;
          const int e = misc[S_EQ] + 23;
          if ((double)W * (double)mx1 <= ldexp(1.0, kG + e)) {
            misc[S_FAST] = 2;
            redf[1] = ldexpf(1.5f, kG + e);
          }
        }
        __syncthreads();
        if (misc[S_FAST] == 2) {
          fpath = 2;
          split = true;
          cmag = redf[1];
          qexp = ldexp(1.0, misc[S_EQ]);
          qinv = ldexp(1.0, -misc[S_EQ]);
        }
      }
      if (FILT && fpath == 1) {
        // MODE 2 has no guarded-fp64 arrays.  Its filtered gather is approximate
        // anyway and its exact fallback only needs the fp64 guard (every sum of
        // W minima and the correction exact), so fp64-guarded frames run the
        // filtered path too (the quantum bounds keep G and 1/G finite floats);
        // the rest take the ordered path.
        if (misc[S_EQ] >= -123 && misc[S_EQ] <= 77) {
          fpath = 2;
          split = true;
          qexp = ldexp(1.0, misc[S_EQ]);
          qinv = ldexp(1.0, -misc[S_EQ]);
        } else {
          fpath = 0;
          fastp = false;
        }
      }
      if (FILT && split) { // D < max|y| / q < 2^bits; Dc = D / 2^gsh rounded, |Dc| <= 2^24
        const int bits = ilogbf(__int_as_float(misc[S_YMAX])) + 1 - misc[S_EQ];
        gsh = bits > 24 ? bits - 24 : 0;
        Gf = ldexpf(1.f, gsh + misc[S_EQ]);
        invGf = ldexpf(1.f, -(gsh + misc[S_EQ]));
      }
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int m = tid + k * T;
        const bool ok = m < M;
        const int par = (sprev >> k) & 1;
        const YT min1 = r_min1[k], min2 = r_min2[k];
        const int ac = r_ac[k];
        if (ok) {
          const double sg = par ? 1.0 : -1.0;
          const double d1 = (double)min1, d2 = (double)min2;
          if (kGuard && split) {
            const float s1v = par ? (float)min1 : -(float)min1;
            sFA[m] = s1v;
            sFA[m + N] = s1v;
            sFB[m + 1] = s1v;
            sFB[m + N + 1] = s1v;
            sA2[m] = (uint16_t)ac;
            if (FILT && P.wmode == FWBF_WEIGHTS_IMWBF) {
              reinterpret_cast<float *>(sM2)[m] = (float)min2; // MODE 2: min2 per check
              const int Dc = coarse_dc((float)min2, (float)min1, invGf);
              atomicAdd(&sCorr[ac], par ? Dc : -Dc);
            } else if (P.wmode == FWBF_WEIGHTS_IMWBF) { // column ac reads min2: + sgn*(min2-min1)
              const long long D = (long long)__dmul_rn(__dsub_rn(d2, d1), qinv); // exact integer
              corr_add(sCorr, ac, par ? D : -D, 1);
              // limb change when s_m goes 0 -> 1 (negated for 1 -> 0)
              int2 dl;
              dl.x = (int)(D & 0xffffffll) - (int)((-D) & 0xffffffll);
              dl.y = (int)(D >> 24) - (int)((-D) >> 24);
              reinterpret_cast<int2 *>(sM2)[m] = dl;
            }
          } else if (kGuard && fastp) {
            chk1[m] = sg * d1;
            chk1[m + N] = sg * d1;
            chk2[m] = sg * d2;
            chk2[m + N] = sg * d2;
            if (P.wmode == FWBF_WEIGHTS_IMWBF) {
              // column ac reads min2 at its local check index j (m = ac - c_j)
              int d = ac - m;
              if (d < 0) d += N;
              const int j = P.offpos[d];
              atomicOr(&amask[ac * aw + (j >> 5)], 1u << (j & 31));
            }
          } else if (CIRC) {
            // ordered path: doubled records as above (MODE 2: single, wrapped
            // on read); the argmin bit sits at the check's position in column
            // ac's ascending check list
            chk1[m] = sg * d1;
            chk2[m] = sg * d2;
            if (!FILT) {
              chk1[m + N] = sg * d1;
              chk2[m + N] = sg * d2;
            }
            if (P.wmode == FWBF_WEIGHTS_IMWBF) {
              int d = ac - m;
              if (d < 0) d += N;
              int i = (int)P.jii[P.offpos[d]] - (int)P.i0tab[ac];
              if (i < 0) i += W;
              atomicOr(&amask[ac * aw + (i >> 5)], 1u << (i & 31));
            }
          } else {
            chk1[m] = sg * d1;
            chk2[m] = sg * d2;
            amin[m] = (P.wmode == FWBF_WEIGHTS_IMWBF) ? ac : -1;
          }
        }
      }
    } else {
    for (int k = 0; k < nKm; ++k) {
      const int m = tid + k * T;
      const bool ok = m < M;
      int par = 0;
      YT min1 = YT(INFINITY), min2 = YT(INFINITY);
      int ac = 0x7fffffff;
      if (ok) {
        if (kGuard && !nonfin_frame) {
          // columns in ascending order (m + c_j - N for j >= jw, then m + c_j),
          // so strict < keeps the lowest column on ties; min2 = second smallest
          // of the multiset (min(min2, max(min1, a)))
          const int *orr = offs_s + 192 + __ldg(P.jwtab + m);
          for (int t = 0; t < W; ++t) {
            const int c = m + orr[t];
            const YT yv = ybuf[c];
            par ^= (yv < YT(0));
            const YT a = fabs(yv);
            const bool lt = a < min1;
            min2 = fminf(min2, fmaxf(min1, a));
            min1 = fminf(min1, a);
            ac = lt ? c : ac;
          }
        } else if (CIRC) {
          for (int j = 0; j < W; ++j) {
            int c = m + P.off[j];
            if (c >= N) c -= N;
            const YT yv = ybuf[c];
            par ^= (yv < YT(0));
            const YT a = fabs(yv);
            if (a < min1 || (a == min1 && c < ac)) { min2 = min1; min1 = a; ac = c; }
            else if (a < min2) min2 = a;
          }
        } else if (P.qc_z) {
          // quasi-cyclic: row r*Z + i holds column cb*Z + ((i + s[r][cb]) mod Z)
          const int Z = P.qc_z, r = m >> qlz, ii = m & (Z - 1);
          for (int cb = 0; cb < P.qc_kb; ++cb) {
            const int sh = P.qc_shift[r * P.qc_kb + cb];
            if (sh < 0) continue;
            const int c = cb * Z + ((ii + sh) & (Z - 1));
            const YT yv = ybuf[c];
            par ^= (yv < YT(0));
            const YT a = fabs(yv);
            if (a < min1 || (a == min1 && c < ac)) { min2 = min1; min1 = a; ac = c; }
            else if (a < min2) min2 = a;
          }
        } else {
          const int e0 = __ldg(P.row_ptr + m), e1 = __ldg(P.row_ptr + m + 1);
          for (int e = e0; e < e1; ++e) {
            const int c = __ldg(P.row_idx + e);
            const YT yv = ybuf[c];
            par ^= (yv < YT(0));
            const YT a = fabs(yv);
            if (a < min1 || (a == min1 && c < ac)) { min2 = min1; min1 = a; ac = c; }
            else if (a < min2) min2 = a;
          }
        }
      }
      if (ok && par) sprev |= 1u << k;
      const uint32_t b = __ballot_sync(FULL_MASK, ok && par);
      if (lane == 0 && (k * T + warp * 32) < M) {
        sbits[(k * T + warp * 32) >> 5] = b;
        atomicAdd(&misc[S_SWT], __popc(b));
      }
      if (ok) {
        const double sg = par ? 1.0 : -1.0;
        const double d1 = (double)min1, d2 = (double)min2;
        if (kGuard && split) {
          const float s1v = par ? (float)min1 : -(float)min1;
          sFA[m] = s1v;
          sFA[m + N] = s1v;
          sFB[m + 1] = s1v;
          sFB[m + N + 1] = s1v;
          sA2[m] = (uint16_t)ac;
          if (P.wmode == FWBF_WEIGHTS_IMWBF) { // column ac reads min2: + sgn*(min2-min1)
            const long long D = (long long)__dmul_rn(__dsub_rn(d2, d1), qinv); // exact integer
            corr_add(sCorr, ac, par ? D : -D, 1);
            // limb change when s_m goes 0 -> 1 (negated for 1 -> 0)
            int2 dl;
            dl.x = (int)(D & 0xffffffll) - (int)((-D) & 0xffffffll);
            dl.y = (int)(D >> 24) - (int)((-D) >> 24);
            reinterpret_cast<int2 *>(sM2)[m] = dl;
          }
        } else if (kGuard && fastp) {
          chk1[m] = sg * d1;
          chk1[m + N] = sg * d1;
          chk2[m] = sg * d2;
          chk2[m + N] = sg * d2;
          if (P.wmode == FWBF_WEIGHTS_IMWBF) {
            // column ac reads min2 at its local check index j (m = ac - c_j)
            int d = ac - m;
            if (d < 0) d += N;
            const int j = P.offpos[d];
            atomicOr(&amask[ac * aw + (j >> 5)], 1u << (j & 31));
          }
        } else if (CIRC) {
          // ordered path: doubled records as above; the argmin bit sits at the
          // check's position in column ac's ascending check list
          chk1[m] = sg * d1;
          chk1[m + N] = sg * d1;
          chk2[m] = sg * d2;
          chk2[m + N] = sg * d2;
          if (P.wmode == FWBF_WEIGHTS_IMWBF) {
            int d = ac - m;
            if (d < 0) d += N;
            int i = (int)P.jii[P.offpos[d]] - (int)P.i0tab[ac];
            if (i < 0) i += W;
            atomicOr(&amask[ac * aw + (i >> 5)], 1u << (i & 31));
          }
        } else {
          chk1[m] = sg * d1;
          chk2[m] = sg * d2;
          amin[m] = (P.wmode == FWBF_WEIGHTS_IMWBF) ? ac : -1;
        }
      }
    }
    }
    __syncthreads();
    FWBF_PH(2)
    // Filtered metric (FWBF on the split path): the gather sums the signed
    // min1 values directly in fp32.  Each of a column's W sequential
    // round-to-nearest adds errs by at most u = 2^-24 of its partial sum
    // (<= k vmax after k terms), so |approx - exact| <= u vmax W(W+1)/2; the
    // float finalize (the int-to-float correction, one FMA, fl32(alpha|y|),
    // one subtraction) adds at most 2^-22 (W + alpha + 1) max|y| (every
    // operand is at most (W + alpha) max|y|), and the coarse correction grid
    // W G / 2.  fdelta bounds all of it, for every column of the frame.
    bool filt = false;
    double fdelta = 0.0;
    float fdp = 0.f, fd2 = 0.f;
    if (FILT && kTwoPhase && split) {
      filt = true;
      const double vmax = (double)__int_as_float(misc[S_VMAX]);
      const double ymax = (double)__int_as_float(misc[S_YMAX]);
      // + the coarse argmin corrections: at most W checks of a column, each
      // rounded to the grid G by at most G/2
      fdelta = ldexp(vmax * (0.5 * (double)W * (double)(W + 1)) * 1.001, -24) +
               ldexp(((double)W + P.alpha + 1.0) * ymax, -22) + 0.5 * (double)W * (double)Gf +
               ldexp((double)W * ymax, -23);
      fdp = __double2float_ru(fdelta);
      // band width 2 fdelta, plus the float rounding of (max - fd2)
      fd2 = __double2float_ru(2.0 * fdelta + ldexp(((double)W + P.alpha + 1.0) * ymax, -22));
    }

    // ---------------- guarded path: per-column argmin masks into registers -----
    // Bit j of am[q] says column tid + q*T is the argmin of its j-th check
    // (m = n - c_j), i.e. reads min2 there instead of min1 (decoders.py:80-84).
    uint32_t am[KC][2];
    if (kGuard && fastp) {
#pragma unroll
      for (int q = 0; q < KC; ++q) {
        const int n = tid + q * T;
        am[q][0] = (n < N) ? amask[n * aw] : 0u;
        am[q][1] = (n < N && aw > 1) ? amask[n * aw + 1] : 0u;
      }
    }
    if (!FILT && kGuard && split && P.has_ay) { // fl(alpha |y_n|) once per frame (ybuf is still valid here)
      for (int n = tid; n < N; n += T) sAY[n] = __dmul_rn(P.alpha, fabs((double)ybuf[n]));
    }
    // MODE 2: |y_n| (float, exact) after the float metric (even offset)
    const float *yabsT = reinterpret_cast<const float *>(Ebuf) + ((N + 1) & ~1);
    if (FILT && split) {
      float *ya = reinterpret_cast<float *>(Ebuf) + ((N + 1) & ~1);
      for (int n = tid; n < N; n += T)
        ya[n] = fabsf((float)((P.alias_y && !ystage) ? load_y<YT>(P, f, n) : ybuf[n]));
    }
    if (P.alias_y || (FILT && split)) __syncthreads(); // amask / ybuf may overlay Ebuf (compact layout); MODE 2 tables
    if (ystage && tid == 0) {
      // ybuf is dead for this frame (alias_y: later reads of y go to HBM):
      // claim the next frame and start its copy
      const unsigned t1 = atomicAdd(P.work_counter, 1u);
      misc[S_FRAME] = (int)t1;
      if ((long long)t1 < P.batch)
        bulk_row_to_smem(ybuf, reinterpret_cast<const YT *>(P.y) + (long long)t1 * P.ld,
                         (unsigned)P.ystage_bytes, &ystage_bar);
    }

    // ---------------- iterations -----------------------------------------------
    int k = 0;
    int conv = 0, stalled = 0;
    long long logpos = 0;
    long long flips_total = 0;
    if (INC && split && P.alg == FWBF_ALG_IMWBF) {
      // IMWBF flips one bit per iteration (decoders.py:170-171), so after one
      // full split-fp32 pass the metric is kept incrementally: the exact column
      // sums live as int64 limb pairs in sCorr (units of q), and the W checks
      // the flip toggles add (s ? +2 : -2) w / q to their W columns -- W^2
      // integer updates per iteration instead of N*W edge visits.  Integer
      // arithmetic is exact, so every metric equals the full recomputation.
      {
        constexpr int NP = SplitPairs<KC>::value;
        unsigned long long hi[NP], lo[NP];
#pragma unroll
        for (int qp = 0; qp < NP; ++qp) { hi[qp] = 0ull; lo[qp] = 0ull; }
        const unsigned long long cc = f2pack(cmag, cmag);
        const uint32_t baseT = (uint32_t)__cvta_generic_to_shared(smem_raw) + 8u * (uint32_t)tid;
#pragma unroll
        for (int j = 0; j < (WT > 0 ? WT : 1); ++j)
          GatherP2<0, NP, TB>::run(hi, lo, baseT + (uint32_t)P.uoff[j], cc);
#pragma unroll
        for (int qp = 0; qp < NP; ++qp) {
          const float2 h = f2unpack(hi[qp]);
          const float2 l = f2unpack(lo[qp]);
          const int n = 2 * tid + 2 * T * qp;
          if (n < N) {
            int4 *cp = reinterpret_cast<int4 *>(sCorr + 2 * n);
            const int4 cv = *cp;
            const long long I0 = (long long)__dmul_rn(__dadd_rn((double)h.x, (double)l.x), qinv) +
                                 (((long long)cv.y << 24) + cv.x);
            const long long I1 = (long long)__dmul_rn(__dadd_rn((double)h.y, (double)l.y), qinv) +
                                 (((long long)cv.w << 24) + cv.z);
            *cp = make_int4((int)(I0 & 0xffffff), (int)(I0 >> 24), (int)(I1 & 0xffffff), (int)(I1 >> 24));
          }
        }
      }
      __syncthreads();
      // per check: 2 min1 / q as an int64 in the (now free) shifted copy sFB
      long long *sA1 = reinterpret_cast<long long *>(smem_raw + ((P.off_fb + 7) & ~7));
      for (int m = tid; m < M; m += T) sA1[m] = (long long)__dmul_rn(__dmul_rn((double)fabsf(sFA[m]), 2.0), qinv);
      __syncthreads();
      for (;;) {
        if (misc[S_SWT] == 0) { conv = 1; break; }
        if (k >= P.kmax) break;
        // metric from the limb sums (renormalised) and the global argmax
        double v = -dinf();
        int i = 0x7fffffff;
        for (int n = tid; n < N; n += T) {
          int2 *cp = reinterpret_cast<int2 *>(sCorr) + n;
          const int2 cv = *cp;
          const long long S = ((long long)cv.y << 24) + cv.x;
          *cp = make_int2((int)(S & 0xffffff), (int)(S >> 24));
          const double aa = P.has_ay ? sAY[n]
                                     : __dmul_rn(P.alpha, P.alias_y ? fabs((double)load_y<YT>(P, f, n))
                                                                    : fabs((double)ybuf[n]));
          const double e = __dsub_rn(__dmul_rn((double)S, qexp), aa);
          if (e > v) { v = e; i = n; }
        }
        warp_amax_redux(v, i); // finite metrics (split-path frames)
        if (lane == 0) { red_v[warp] = v; red_i[warp] = i; }
        __syncthreads();
        if (warp == 0) {
          v = lane < nwarps ? red_v[lane] : -dinf();
          i = lane < nwarps ? red_i[lane] : 0x7fffffff;
          warp_amax_redux(v, i); // finite metrics (split-path frames)
          const int c = i; // flipped unconditionally: IMWBF never stalls
          if (lane == 0) {
            zbits[c >> 5] ^= 1u << (c & 31);
            flips[0] = c;
            if (P.fliplog) {
              P.fliplog[f * P.fliplog_stride + logpos] = c;
              P.fliplog_counts[f * P.kmax + k] = 1;
            }
          }
          int dsw = 0; // syndrome weight change
          for (int j = lane; j < W; j += 32) {
            int m = c - offs_s[j];
            if (m < 0) m += N;
            const uint32_t old = atomicXor(&sbits[m >> 5], 1u << (m & 31));
            dsw += ((old >> (m & 31)) & 1u) ? -1 : 1;
          }
#pragma unroll
          for (int off = 16; off; off >>= 1) dsw += __shfl_xor_sync(FULL_MASK, dsw, off);
          if (lane == 0) misc[S_SWT] += dsw;
        }
        __syncthreads();
        {
          const int c = flips[0];
          for (int qq = tid; qq < W * W; qq += T) {
            const int j = qq / W, jj = qq - j * W;
            int m = c - offs_s[j];
            if (m < 0) m += N;
            int n = m + offs_s[jj];
            if (n >= N) n -= N;
            long long A = sA1[m];
            if (P.wmode == FWBF_WEIGHTS_IMWBF && n == (int)sA2[m]) {
              const int2 dl = reinterpret_cast<const int2 *>(sM2)[m];
              A += ((long long)dl.y << 24) + dl.x; // = 2 (min2 - min1) / q
            }
            if (!((sbits[m >> 5] >> (m & 31)) & 1u)) A = -A;
            atomicAdd(&sCorr[2 * n], (int)(A & 0xffffff));
            atomicAdd(&sCorr[2 * n + 1], (int)(A >> 24));
          }
        }
        __syncthreads();
        logpos += 1;
        flips_total += 1;
        k += 1;
      }
    } else
    for (;;) {
      const int swt = misc[S_SWT];
      if (swt == 0 && (FILT || !P.metric_out)) { conv = 1; break; } // MODE 2 never has a stage view
      if (k >= P.kmax) break;

      // ---- Eq.(1) metric for every bit -> Ebuf ----
      const int fs = (fused && (k & 1)) ? S_FB : S_F; // this iteration's flip counter
      // reset: non-fused, this iteration's counter (last read before the previous
      // refresh barrier); fused, the next iteration's (it is written during the
      // metric pass, so it must be zero before this iteration's last barrier)
      if (tid == 0) misc[fused ? (S_F + S_FB - fs) : S_F] = 0;
      if (kGuard && WT > 0 && split && (KC % 2) == 0) {
        // Split-fp32 gather, 4 B per edge and no per-edge argmin select:
        // thread tid owns column pairs (2 tid + 2 T qp, +1).  Column n reads
        // check (n - c_j) mod N; for even n the pair's two values are adjacent,
        // loaded with one 8-byte LDS from sFA (N - c_j even) or from the
        // one-element-shifted copy sFB (N - c_j odd).  v = h + l exactly on the
        // grid G; hi = sum h (multiples of G, |hi| < 2^24 G) and lo = sum l
        // (multiples of q, |lo| <= 16 G <= 2^24 q) are exact in fp32.  The
        // argmin columns' min2 - min1 terms come from exact integer limbs
        // (sCorr).  Every sum is exact, hence equal to the reference's.
        constexpr int NP = SplitPairs<KC>::value;
        unsigned long long hi[NP], lo[NP];
#pragma unroll
        for (int qp = 0; qp < NP; ++qp) { hi[qp] = 0ull; lo[qp] = 0ull; }
        const unsigned long long cc = f2pack(cmag, cmag);
        // per-thread part of the address, plus a warp-uniform part per j
        const uint32_t baseT = (uint32_t)__cvta_generic_to_shared(smem_raw) + 8u * (uint32_t)tid;
        if (filt) { // approximate: plain fp32 sums (within fdelta), lo stays 0
#pragma unroll
          for (int j = 0; j < (WT > 0 ? WT : 1); ++j)
            GatherF2<0, NP, TB>::run(hi, baseT + (uint32_t)P.uoff[j]);
        } else {
#pragma unroll
        for (int j = 0; j < (WT > 0 ? WT : 1); ++j) // P.uoff[j]: host-computed uniform part
          GatherP2<0, NP, TB>::run(hi, lo, baseT + (uint32_t)P.uoff[j], cc);
        }
        if (filt) {
          // filtered metric in float: sum + Cc G (coarse argmin correction) -
          // fl32(alpha |y|); the selection's band test covers every rounding
          float *Efl = reinterpret_cast<float *>(Ebuf);
          const float alf = (float)P.alpha;
#pragma unroll
          for (int qp = 0; qp < NP; ++qp) {
            const float2 h = f2unpack(hi[qp]);
            const int n = 2 * tid + 2 * T * qp;
            if (n + 1 < N) {
              const int2 cc = *reinterpret_cast<const int2 *>(sCorr + n);
              const float2 ya = *reinterpret_cast<const float2 *>(yabsT + n);
              *reinterpret_cast<float2 *>(Efl + n) =
                  make_float2(__fsub_rn(__fmaf_rn((float)cc.x, Gf, h.x), __fmul_rn(alf, ya.x)),
                              __fsub_rn(__fmaf_rn((float)cc.y, Gf, h.y), __fmul_rn(alf, ya.y)));
            } else if (n < N) {
              Efl[n] = __fsub_rn(__fmaf_rn((float)sCorr[n], Gf, h.x), __fmul_rn(alf, yabsT[n]));
            }
          }
        } else if (WT <= 32) {
#pragma unroll
        for (int qp = 0; qp < NP; ++qp) {
          // columns (n, n+1), n even: 16-byte accesses to the per-column arrays
          const float2 h = f2unpack(hi[qp]);
          const float2 l = f2unpack(lo[qp]);
          const int n = 2 * tid + 2 * T * qp;
          if (n < N) {
            const int4 cv = *reinterpret_cast<const int4 *>(sCorr + 2 * n);
            double a0 = __dadd_rn((double)h.x, (double)l.x), a1 = __dadd_rn((double)h.y, (double)l.y);
            if (cv.x | cv.y) a0 = __dadd_rn(a0, __dmul_rn((double)(((long long)cv.y << 24) + cv.x), qexp));
            if (cv.z | cv.w) a1 = __dadd_rn(a1, __dmul_rn((double)(((long long)cv.w << 24) + cv.z), qexp));
            double aa0, aa1;
            if (P.has_ay) {
              const double2 ay2 = *reinterpret_cast<const double2 *>(sAY + n);
              aa0 = ay2.x;
              aa1 = ay2.y;
            } else {
              aa0 = __dmul_rn(P.alpha, P.alias_y ? fabs((double)load_y<YT>(P, f, n)) : fabs((double)ybuf[n]));
              aa1 = (n + 1 < N) ? __dmul_rn(P.alpha, P.alias_y ? fabs((double)load_y<YT>(P, f, n + 1))
                                                                 : fabs((double)ybuf[n + 1]))
                                : 0.0;
            }
            if (n + 1 < N) {
              *reinterpret_cast<double2 *>(Ebuf + n) = make_double2(__dsub_rn(a0, aa0), __dsub_rn(a1, aa1));
            } else {
              Ebuf[n] = __dsub_rn(a0, aa0);
            }
          }
        }
        } else {
#pragma unroll
        for (int qp = 0; qp < NP; ++qp) {
          const float2 h = f2unpack(hi[qp]);
          const float2 l = f2unpack(lo[qp]);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int n = 2 * tid + 2 * T * qp + u;
            if (n < N) {
              double acc = __dadd_rn((double)(u ? h.y : h.x), (double)(u ? l.y : l.x));
              const int2 cv = reinterpret_cast<const int2 *>(sCorr)[n];
              if (cv.x | cv.y)
                acc = __dadd_rn(acc, __dmul_rn((double)(((long long)cv.y << 24) + cv.x), qexp));
              const double aa = P.has_ay ? sAY[n]
                                         : __dmul_rn(P.alpha, P.alias_y ? fabs((double)load_y<YT>(P, f, n))
                                                                        : fabs((double)ybuf[n]));
              Ebuf[n] = __dsub_rn(acc, aa);
            }
          }
        }
        }
      } else if (kGuard && fastp) {
        // chk1/chk2 hold sgn*min1 / sgn*min2 twice ([0,N) and [N,2N)) plus a
        // KC*T-N pad, so column n reads check (n - c_j) mod N at index
        // n + N - c_j with no wrap test: per j one uniform offset, then per
        // column a mask test, an address select, one LDS.64 and one DADD.
        // The sum is exact in any order under the guard.
        double acc[KC];
#pragma unroll
        for (int q = 0; q < KC; ++q) acc[q] = 0.0;
        const uint32_t s1 = (uint32_t)__cvta_generic_to_shared(chk1 + N + tid);
        const uint32_t d21 = (uint32_t)(P.off_chk2 - P.off_chk1);
        uint32_t mk[KC], mkh[KC];
#pragma unroll
        for (int q = 0; q < KC; ++q) { mk[q] = am[q][0]; mkh[q] = am[q][1]; }
        if (WT > 0) {
          // compile-time weight: fully unrolled, offsets are constant-bank operands
#pragma unroll
          for (int j = 0; j < (WT > 0 ? WT : 1); ++j) {
            const uint32_t a1 = s1 - 8u * (uint32_t)P.off[j];
            if (j < 32) GatherQ<0, KC, TB>::run(acc, mk, 1u << (j & 31), a1, a1 + d21);
            else GatherQ<0, KC, TB>::run(acc, mkh, 1u << (j & 31), a1, a1 + d21);
          }
        } else {
          const int w0 = W < 32 ? W : 32;
#pragma unroll 2
          for (int j = 0; j < w0; ++j) {
            const uint32_t a1 = s1 - 8u * (uint32_t)P.off[j];
            GatherQ<0, KC, TB>::run(acc, mk, 1u << j, a1, a1 + d21);
          }
#pragma unroll 2
          for (int j = 32; j < W; ++j) {
            const uint32_t a1 = s1 - 8u * (uint32_t)P.off[j];
            GatherQ<0, KC, TB>::run(acc, mkh, 1u << (j - 32), a1, a1 + d21);
          }
        }
#pragma unroll
        for (int q = 0; q < KC; ++q) {
          const int n = tid + q * T;
          if (n < N) {
            const double ay = P.alias_y ? fabs((double)load_y<YT>(P, f, n)) : fabs((double)ybuf[n]);
            Ebuf[n] = __dsub_rn(acc[q], __dmul_rn(P.alpha, ay));
          }
        }
      } else {
        // ordered column sum for explicit / QC codes (ascending checks)
        auto col_sum = [chk1, chk2, amin, qlz, &P](const int n) -> double {
          double acc = 0.0;
          if (P.qc_z) {
            // column cb*Z + o meets row block r at check r*Z + ((o - s) mod Z):
            // ascending in r, i.e. the reference's ascending check order.  An
            // absent block (s < 0) adds +0.0, which leaves acc unchanged (acc
            // starts at +0.0 and round-to-nearest never produces -0.0 from it).
            const int Z = P.qc_z, cb = n >> qlz, o = n & (Z - 1);
            const int jb = P.qc_jb, kb = P.qc_kb;
#pragma unroll 4
            for (int r = 0; r < jb; ++r) {
              const int sh = P.qc_shift[r * kb + cb];
              const int m = (r << qlz) + ((o - sh) & (Z - 1));
              const double w = ((amin[m] == n) ? chk2 : chk1)[m]; // one 8-byte load
              acc = __dadd_rn(acc, sh >= 0 ? w : 0.0);
            }
          } else {
            const int e0 = __ldg(P.col_ptr + n), e1 = __ldg(P.col_ptr + n + 1);
            for (int e = e0; e < e1; ++e) {
              const int m = __ldg(P.col_idx + e);
              acc = __dadd_rn(acc, ((amin[m] == n) ? chk2 : chk1)[m]);
            }
          }
          return acc;
        };
        if (fused) {
          // Warp w owns p-blocks w, w + nwarps, ...: lane l takes the block's
          // columns l, l + 32, ... (ascending, strict >); a butterfly argmax
          // with lowest-index ties gives the block's first maximum
          // (decoders.py:156-167) and the warp applies the flip when it is > 0
          // (decoders.py:181-183).  The metric never goes to shared memory.
          const int p = P.p, nb = P.nblocks;
          for (int b = warp; b < nb; b += nwarps) {
            double v = -dinf();
            int i = 0x7fffffff;
            const int base = b * p, lim = min(p, N - base);
            const int Zq = P.qc_z;
            if (Zq && P.qc_jb <= 4 && (base >> qlz) == ((base + lim - 1) >> qlz)) {
              // QC block inside one block column: its (<= 4) shifts once per block
              const int cb = base >> qlz, jb = P.qc_jb;
              int shv[4], rowb[4];
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                shv[r] = (r < jb) ? P.qc_shift[r * P.qc_kb + cb] : -1;
                rowb[r] = r << qlz;
              }
              // two columns (o, o + 32) per step: independent fp64 chains
              const bool full4 = jb == 4 && shv[0] >= 0 && shv[1] >= 0 && shv[2] >= 0 && shv[3] >= 0 &&
                                 (lim & 63) == 0; // block-uniform
              if (full4) { // every row block present, whole column pairs: no absent-block selects
                for (int o = lane; o < lim; o += 64) {
                  const int n0 = base + o, n1 = n0 + 32;
                  const int oz0 = n0 & (Zq - 1), oz1 = n1 & (Zq - 1);
                  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                  for (int r = 0; r < 4; ++r) {
                    const int m0 = rowb[r] + ((oz0 - shv[r]) & (Zq - 1));
                    const int m1 = rowb[r] + ((oz1 - shv[r]) & (Zq - 1));
                    acc0 = __dadd_rn(acc0, ((amin[m0] == n0) ? chk2 : chk1)[m0]);
                    acc1 = __dadd_rn(acc1, ((amin[m1] == n1) ? chk2 : chk1)[m1]);
                  }
                  const double e0 = __dsub_rn(acc0, __dmul_rn(P.alpha, fabs((double)ybuf[n0])));
                  if (e0 > v) { v = e0; i = n0; }
                  const double e1 = __dsub_rn(acc1, __dmul_rn(P.alpha, fabs((double)ybuf[n1])));
                  if (e1 > v) { v = e1; i = n1; }
                }
              } else
              for (int o = lane; o < lim; o += 64) {
                const int n0 = base + o, n1 = n0 + 32;
                const bool two = o + 32 < lim;
                const int oz0 = n0 & (Zq - 1), oz1 = (two ? n1 : n0) & (Zq - 1);
                double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                  if (r < jb) {
                    const int m0 = rowb[r] + ((oz0 - shv[r]) & (Zq - 1));
                    const int m1 = rowb[r] + ((oz1 - shv[r]) & (Zq - 1));
                    const double w0 = ((amin[m0] == n0) ? chk2 : chk1)[m0];
                    const double w1 = ((amin[m1] == n1) ? chk2 : chk1)[m1];
                    acc0 = __dadd_rn(acc0, shv[r] >= 0 ? w0 : 0.0); // absent block adds +0.0 (see col_sum)
                    acc1 = __dadd_rn(acc1, shv[r] >= 0 ? w1 : 0.0);
                  }
                }
                const double e0 = __dsub_rn(acc0, __dmul_rn(P.alpha, fabs((double)ybuf[n0])));
                if (e0 > v) { v = e0; i = n0; }
                if (two) {
                  const double e1 = __dsub_rn(acc1, __dmul_rn(P.alpha, fabs((double)ybuf[n1])));
                  if (e1 > v) { v = e1; i = n1; }
                }
              }
            } else {
              for (int o = lane; o < lim; o += 32) {
                const int n = base + o;
                const double e = __dsub_rn(col_sum(n), __dmul_rn(P.alpha, fabs((double)ybuf[n])));
                if (e > v) { v = e; i = n; }
              }
            }
            warp_amax(v, i);
            if (lane == 0) { blk_v[b] = v; blk_i[b] = i; }
            if (v > 0.0) {
              if (lane == 0) {
                atomicXor(&zbits[i >> 5], 1u << (i & 31));
                atomicAdd(&misc[fs], 1);
              }
              if (P.qc_z) {
                const int Z = P.qc_z, cb = i >> qlz, o = i & (Z - 1);
                for (int r = lane; r < P.qc_jb; r += 32) {
                  const int sh = P.qc_shift[r * P.qc_kb + cb];
                  if (sh < 0) continue;
                  const int m = r * Z + ((o - sh) & (Z - 1));
                  atomicXor(&sbits[m >> 5], 1u << (m & 31));
                }
              } else {
                const int e1 = __ldg(P.col_ptr + i + 1);
                for (int e = __ldg(P.col_ptr + i) + lane; e < e1; e += 32) {
                  const int m = __ldg(P.col_idx + e);
                  atomicXor(&sbits[m >> 5], 1u << (m & 31));
                }
              }
            }
          }
        } else {
        // y of the next column is fetched one column ahead (from global memory
        // when the metric buffer overlays y) so its latency hides behind a gather
        if (!CIRC && !P.qc_z && !P.alias_y) {
          // explicit CSC: two columns per step, their edge chains interleaved
          // (each column's own sum stays in ascending check order)
          for (int kk = 0; kk < nKy; kk += 2) {
            const int n0 = tid + kk * T, n1 = n0 + T;
            if (n0 >= N) break;
            const bool two = n1 < N;
            const int a0 = __ldg(P.col_ptr + n0), d0 = __ldg(P.col_ptr + n0 + 1) - a0;
            const int a1 = two ? __ldg(P.col_ptr + n1) : 0, d1 = two ? __ldg(P.col_ptr + n1 + 1) - a1 : 0;
            double acc0 = 0.0, acc1 = 0.0;
            const int dm = d0 > d1 ? d0 : d1;
            for (int t = 0; t < dm; ++t) {
              if (t < d0) {
                const int m = __ldg(P.col_idx + a0 + t);
                acc0 = __dadd_rn(acc0, ((amin[m] == n0) ? chk2 : chk1)[m]);
              }
              if (t < d1) {
                const int m = __ldg(P.col_idx + a1 + t);
                acc1 = __dadd_rn(acc1, ((amin[m] == n1) ? chk2 : chk1)[m]);
              }
            }
            Ebuf[n0] = __dsub_rn(acc0, __dmul_rn(P.alpha, fabs((double)ybuf[n0])));
            if (two) Ebuf[n1] = __dsub_rn(acc1, __dmul_rn(P.alpha, fabs((double)ybuf[n1])));
          }
        } else {
        YT ynext = (tid < N) ? (P.alias_y ? load_y<YT>(P, f, tid) : ybuf[tid]) : YT(0);
        for (int kk = 0; kk < nKy; ++kk) {
          const int n = tid + kk * T;
          if (n >= N) break;
          const YT ycur = ynext;
          if (n + T < N) ynext = P.alias_y ? load_y<YT>(P, f, n + T) : ybuf[n + T];
          double acc = 0.0;
          if (CIRC) {
            // checks (n + dneg[ii]) mod N for ii = i0, i0+1, ... (ascending),
            // read from the doubled records at n + dneg[ii] (no wrap); bit i of
            // the column's mask selects min2 at the i-th check
            const int *dn = offs_s + 64 + P.i0tab[n];
            const double *c1 = chk1 + n, *c2 = chk2 + n;
            const uint32_t mk = amask[n * aw];
            const int w0 = W < 32 ? W : 32;
            // MODE 2 keeps single records: wrap the check index instead
            const int wrapN = FILT ? N : 0x7fffffff;
            for (int i = 0; i < w0; ++i) {
              const int d = (n + dn[i] >= wrapN) ? dn[i] - N : dn[i];
              acc = __dadd_rn(acc, (((mk >> i) & 1u) ? c2 : c1)[d]);
            }
            if (W > 32) {
              const uint32_t mkh = amask[n * aw + 1];
              for (int i = 32; i < W; ++i) {
                const int d = (n + dn[i] >= wrapN) ? dn[i] - N : dn[i];
                acc = __dadd_rn(acc, (((mkh >> (i - 32)) & 1u) ? c2 : c1)[d]);
              }
            }
          } else {
            acc = col_sum(n);
          }
          Ebuf[n] = __dsub_rn(acc, __dmul_rn(P.alpha, fabs((double)ycur)));
        }
        } // explicit two-column branch
        }
      }
      __syncthreads();
      FWBF_PH(3)
      if (!FILT && P.metric_out) { // stage view (fwbf_metric_*): Eq.(1) on the initial state, then stop
        for (int n = tid; n < N; n += T) P.metric_out[f * P.metric_ld + n] = Ebuf[n];
        break;
      }

      // ---- selection (+ fused flips for FWBF) ----
      if (tid == 0) misc[S_SWT] = 0; // every thread read it at the loop top (before the E barrier)
      int F = 0;
      bool applied = false;
      if (FILT || P.alg == FWBF_ALG_FWBF) { // MODE 2 is FWBF only
        // Groups of TPB = 2^log2_tpb threads own one p-block each: strided scan
        // (ascending per thread, strict >), butterfly argmax in the group, then
        // the group applies its flip when the block maximum is > 0
        // (decoders.py:156-167, :181-183).  misc[S_F] counts the flips.
        const int p = P.p;
        const int nb = P.nblocks;
        const int TPB = 1 << sel_lt;
        const int sub = sel_sub, gpc = sel_gpc, slot = sel_slot;
        const int rounds = fused ? 0 : sel_rounds;
        for (int r = 0; r < rounds; ++r) {
          const int b = r * gpc + slot;
          const bool ok = b < nb;
          const int base = b * p;
          const int lim = ok ? min(p, N - base) : 0;
          double v = -dinf();
          int i = 0x7fffffff;
          if (filt) {
            // Filtered metric (float, within fdelta of the exact one): scan
            // with the runner-up value, butterfly over (max, index, runner-up).
            // The block's decision is settled when the runner-up is more than
            // 2 fdelta below the maximum (then the maximum is the exact first
            // maximum) and the maximum is farther than fdelta from 0 (then its
            // sign is exact); otherwise the columns in the band are recomputed
            // exactly.  fd2 / fdp are rounded outwards (see fdelta).
            const float *Efl = reinterpret_cast<const float *>(Ebuf);
            float fv = -INFINITY, fv2 = -INFINITY;
            if (ok)
              for (int o = sub; o < lim; o += TPB) {
                const float e = Efl[base + o];
                fv2 = fmaxf(fv2, fminf(fv, e));
                if (e > fv) { fv = e; i = base + o; }
              }
            bool amb = false;
            if (__any_sync(FULL_MASK, ok)) {
              for (int off = TPB >> 1; off; off >>= 1) {
                const float vo = __shfl_xor_sync(FULL_MASK, fv, off);
                const int io = __shfl_xor_sync(FULL_MASK, i, off);
                const float v2o = __shfl_xor_sync(FULL_MASK, fv2, off);
                fv2 = fmaxf(fmaxf(fv2, v2o), fminf(fv, vo));
                if (vo > fv || (vo == fv && io < i)) { fv = vo; i = io; }
              }
              amb = ok && (fv2 >= fv - fd2 || (fv > -fdp && fv <= fdp));
            }
            v = (double)fv;
            if (__any_sync(FULL_MASK, amb)) {
              double ve = -dinf();
              int ie = 0x7fffffff;
              if (amb)
                for (int o = sub; o < lim; o += TPB) {
                  const int n = base + o;
                  if (Efl[n] >= fv - fd2)
                    amax_combine(ve, ie, exact_split_metric(P, sFA, sA2, reinterpret_cast<const float *>(sM2), yabsT, n, W, qexp, qinv), n);
                }
              for (int off = TPB >> 1; off; off >>= 1) {
                const double v2 = __shfl_xor_sync(FULL_MASK, ve, off);
                const int i2 = __shfl_xor_sync(FULL_MASK, ie, off);
                amax_combine(ve, ie, v2, i2);
              }
              if (amb) {
                v = ve;
                i = ie;
                if (sub == 0 && P.filter_stats) atomicAdd((unsigned long long *)P.filter_stats, 1ull);
              }
            }
          } else {
          if (ok) {
            for (int o = sub; o < lim; o += TPB) {
              const double e = Ebuf[base + o];
              if (e > v) { v = e; i = base + o; }
            }
          }
          if (__any_sync(FULL_MASK, ok)) { // warps without a block skip the butterfly
            for (int off = TPB >> 1; off; off >>= 1) {
              const double v2 = __shfl_xor_sync(FULL_MASK, v, off);
              const int i2 = __shfl_xor_sync(FULL_MASK, i, off);
              amax_combine(v, i, v2, i2);
            }
          }
          }
          {
            const uint32_t pm = __ballot_sync(FULL_MASK, ok && sub == 0 && v > 0.0);
            if (lane == 0 && pm) atomicAdd(&misc[S_F], __popc(pm)); // one count per warp
          }
          if (ok) {
            if (sub == 0) { blk_v[b] = v; blk_i[b] = i; }
            if (v > 0.0) {
              if (sub == 0) atomicXor(&zbits[i >> 5], 1u << (i & 31));
              if (CIRC) {
#pragma unroll 4
                for (int j = sub; j < W; j += TPB) {
                  const int d = i - offs_s[j]; // (i - c_j) mod N as an unsigned min
                  const int m = (int)min((unsigned)d, (unsigned)(d + N));
                  atomicXor(&sbits[m >> 5], 1u << (m & 31));
                }
              } else if (P.qc_z) {
                const int Z = P.qc_z, cb = i >> qlz, o = i & (Z - 1);
                for (int r = sub; r < P.qc_jb; r += TPB) {
                  const int sh = P.qc_shift[r * P.qc_kb + cb];
                  if (sh < 0) continue;
                  const int m = r * Z + ((o - sh) & (Z - 1));
                  atomicXor(&sbits[m >> 5], 1u << (m & 31));
                }
              } else {
                const int e1 = __ldg(P.col_ptr + i + 1);
                for (int e = __ldg(P.col_ptr + i) + sub; e < e1; e += TPB) {
                  const int m = __ldg(P.col_idx + e);
                  atomicXor(&sbits[m >> 5], 1u << (m & 31));
                }
              }
            }
          }
        }
        if (!fused) __syncthreads(); // fused: block results and flips came with the metric pass
        FWBF_PH(4)
        F = misc[fs];
        if (F > 0) {
          applied = true;
          if (P.fliplog && warp == 0) { // ascending = block order
            int cnt = 0;
            for (int base = 0; base < nb; base += 32) {
              const int bb = base + lane;
              const bool pos = bb < nb && blk_v[bb] > 0.0;
              const uint32_t msk = __ballot_sync(FULL_MASK, pos);
              if (pos) P.fliplog[f * P.fliplog_stride + logpos + cnt + __popc(msk & ((1u << lane) - 1u))] = blk_i[bb];
              cnt += __popc(msk);
            }
            if (lane == 0) P.fliplog_counts[f * P.kmax + k] = F;
          }
        } else {
          if (warp == 0) {
            double gv = -dinf();
            int gi = 0x7fffffff;
            for (int bb = lane; bb < nb; bb += 32) amax_combine(gv, gi, blk_v[bb], blk_i[bb]);
            warp_amax(gv, gi);
            if (filt) { // the block maxima are exact argmaxes, their values within fdelta
              const double thr = gv - (double)fd2;
              int cnt = 0;
              for (int bb = lane; bb < nb; bb += 32) cnt += blk_v[bb] >= thr;
              for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(FULL_MASK, cnt, off);
              if (cnt > 1) {
                double ve = -dinf();
                int ie = 0x7fffffff;
                for (int bb = lane; bb < nb; bb += 32)
                  if (blk_v[bb] >= thr)
                    amax_combine(ve, ie, exact_split_metric(P, sFA, sA2, reinterpret_cast<const float *>(sM2), yabsT, blk_i[bb], W, qexp, qinv),
                                 blk_i[bb]);
                warp_amax(ve, ie);
                gi = ie;
                if (lane == 0 && P.filter_stats) atomicAdd((unsigned long long *)P.filter_stats + 1, 1ull);
              }
            }
            if (lane == 0) { misc[S_GBEST] = gi; flips[0] = gi; }
          }
        }
      } else if (P.alg == FWBF_ALG_IMWBF) {
        double v = -dinf();
        int i = 0x7fffffff;
        for (int n = tid; n < N; n += T) amax_combine(v, i, Ebuf[n], n);
        warp_amax(v, i);
        if (lane == 0) { red_v[warp] = v; red_i[warp] = i; }
        __syncthreads();
        if (warp == 0) {
          v = lane < nwarps ? red_v[lane] : -dinf();
          i = lane < nwarps ? red_i[lane] : 0x7fffffff;
          warp_amax(v, i);
          if (lane == 0) { misc[S_F] = 1; misc[S_GBEST] = i; flips[0] = i; }
        }
        __syncthreads();
        F = misc[S_F];
      } else { // MLP: top-lambda by (metric desc, index asc), then ascending order
        // (decoders.py:174-178: stable argsort of -e, first lam, > 0 when
        // thresholded, sorted).  Two barriers per iteration:
        // (1) each warp lists its own top-L columns (L = min(lam, its column
        //     count)), best first, by L rounds of warp argmax with exclusion
        //     (a per-lane taken mask over its nKy columns) -- no barriers;
        // (2) warp 0 merges the nwarps sorted lists (lane l walks list l),
        //     stops after lam picks or at the first pick <= 0 when thresholded
        //     (the lists are descending), marks the picks in a column bitmap
        //     and compacts it in ascending order.
        // Lists hold (value, column) pairs, so the merge reads no metric.
        int *cand = blk_i;                                        // [nwarps][L]
        int *ccnt = blk_i + nwarps * P.lam;                       // [nwarps]
        uint32_t *sel = reinterpret_cast<uint32_t *>(ccnt + nwarps); // [zw]
        double *candv = blk_v;                                    // [nwarps][L]
        const int L = min(P.lam, 32 * nKy);
        if (TB > 0) {
          // compile-time columns per thread: each lane sorts its KC values once
          // (value desc, index asc); a round's candidate is then the lane's
          // head, and the winning lane shifts its list -- no rescans
          constexpr int KS = TB > 0 ? KC : 1;
          double sv[KS];
          int si[KS];
#pragma unroll
          for (int q = 0; q < KS; ++q) {
            const int n = tid + q * T;
            sv[q] = n < N ? Ebuf[n] : -dinf();
            si[q] = n < N ? n : 0x7fffffff;
          }
#pragma unroll
          for (int a2 = 0; a2 < KS; ++a2)
#pragma unroll
            for (int b2 = 0; b2 + 1 < KS - a2; ++b2)
              if (sv[b2 + 1] > sv[b2] || (sv[b2 + 1] == sv[b2] && si[b2 + 1] < si[b2])) {
                const double tv = sv[b2]; sv[b2] = sv[b2 + 1]; sv[b2 + 1] = tv;
                const int ti = si[b2]; si[b2] = si[b2 + 1]; si[b2 + 1] = ti;
              }
          int cnt = 0;
          for (int r = 0; r < L; ++r) {
            double v = sv[0];
            int i = si[0];
            warp_amax_redux(v, i);
            if (i == 0x7fffffff) break; // the warp's columns are exhausted (warp-uniform)
            // thresholded: a value <= 0 is never picked, so a warp's list ends at
            // its first one -- kept only as entry 0 (the global argmax of the
            // stall policy is the best of the warps' first entries)
            if (P.mlp_thr && r > 0 && !(v > 0.0)) break;
            if (si[0] == i) { // this lane's head won: pop it
#pragma unroll
              for (int q = 0; q + 1 < KS; ++q) { sv[q] = sv[q + 1]; si[q] = si[q + 1]; }
              sv[KS - 1] = -dinf();
              si[KS - 1] = 0x7fffffff;
            }
            if (lane == 0) { cand[warp * P.lam + r] = i; candv[warp * P.lam + r] = v; }
            cnt = r + 1;
          }
          if (lane == 0) ccnt[warp] = cnt;
        } else {
          uint32_t taken = 0;
          int cnt = 0;
          for (int r = 0; r < L; ++r) {
            double v = -dinf();
            int i = 0x7fffffff;
            for (int q = 0; q < nKy; ++q) {
              const int n = tid + q * T;
              if (n < N && !((taken >> q) & 1u)) amax_combine(v, i, Ebuf[n], n);
            }
            warp_amax_redux(v, i);
            if (i == 0x7fffffff) break; // the warp's columns are exhausted (warp-uniform)
            if (P.mlp_thr && r > 0 && !(v > 0.0)) break; // see above
            if ((i & 31) == lane) taken |= 1u << (i / T);
            if (lane == 0) { cand[warp * P.lam + r] = i; candv[warp * P.lam + r] = v; }
            cnt = r + 1;
          }
          if (lane == 0) ccnt[warp] = cnt;
        }
        __syncthreads();
        if (warp == 0) {
          const bool small = P.lam <= 32; // picks fit the lanes: ascending order by ranking
          if (!small)
            for (int w2 = lane; w2 < zw; w2 += 32) sel[w2] = 0u;
          const int myc = lane < nwarps ? ccnt[lane] : 0;
          int h = 0, picked = 0, mypick = 0x7fffffff;
          double hv = myc > 0 ? candv[lane * P.lam] : -dinf(); // this lane's list head
          int hi = myc > 0 ? cand[lane * P.lam] : 0x7fffffff;
          __syncwarp();
          for (int r = 0; r < P.lam; ++r) {
            double v = hv;
            int i = hi;
            warp_amax_redux(v, i);
            if (i == 0x7fffffff) break;
            if (r == 0 && lane == 0) { misc[S_GBEST] = i; flips[0] = i; } // the global argmax (stall policy)
            if (P.mlp_thr && !(v > 0.0)) break;                           // every later pick is <= v
            if (hi == i) { // the owner list advances
              ++h;
              hv = h < myc ? candv[lane * P.lam + h] : -dinf();
              hi = h < myc ? cand[lane * P.lam + h] : 0x7fffffff;
            }
            if (small) {
              if (lane == r) mypick = i;
            } else if (lane == 0) {
              sel[i >> 5] |= 1u << (i & 31);
            }
            ++picked;
          }
          int cnt = 0;
          if (small) {
            // lane r holds pick r; its place in ascending order = picks below it
            int pos = 0;
            for (int l = 0; l < picked; ++l) pos += __shfl_sync(FULL_MASK, mypick, l) < mypick;
            if (lane < picked) flips[pos] = mypick;
            cnt = picked;
          } else {
            __syncwarp();
            if (picked)
              for (int base = 0; base < zw; base += 32) {
                const int w2 = base + lane;
                const uint32_t word = (w2 < zw) ? sel[w2] : 0u;
                int c = __popc(word);
                int incl = c;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                  const int t2 = __shfl_up_sync(FULL_MASK, incl, off);
                  if (lane >= off) incl += t2;
                }
                int pos = cnt + incl - c;
                uint32_t wd = word;
                while (wd) {
                  const int bit = __ffs(wd) - 1;
                  wd &= wd - 1;
                  flips[pos++] = w2 * 32 + bit;
                }
                cnt += __shfl_sync(FULL_MASK, incl, 31);
              }
          }
          if (lane == 0) misc[S_F] = cnt;
        }
        __syncthreads();
        F = misc[S_F];
        FWBF_PH(4)
      }

      if (F == 0) {
        // nothing selected while the syndrome is nonzero (decoders.py:214-222)
        stalled = 1;
        if (P.stall == FWBF_STALL_TERMINATE) {
          if (tid == 0 && P.fliplog_counts) P.fliplog_counts[f * P.kmax + k] = 0;
          k += 1;
          break;
        }
        F = 1; // flips[0] = global argmax, written above
        __syncthreads();
      }
      if (!applied) {
        if (P.fliplog) {
          for (int t = tid; t < F; t += T) P.fliplog[f * P.fliplog_stride + logpos + t] = flips[t];
          if (tid == 0) P.fliplog_counts[f * P.kmax + k] = F;
        }
        for (int t = tid; t < F; t += T) {
          const int n = flips[t];
          atomicXor(&zbits[n >> 5], 1u << (n & 31));
        }
        if (CIRC) {
          for (int fi = warp; fi < F; fi += nwarps) {
            const int n = flips[fi];
            for (int j = lane; j < W; j += 32) {
              int m = n - offs_s[j];
              if (m < 0) m += N;
              atomicXor(&sbits[m >> 5], 1u << (m & 31));
            }
          }
        } else if (P.qc_z) {
          for (int fi = warp; fi < F; fi += nwarps) {
            const int n = flips[fi];
            const int Z = P.qc_z, cb = n >> qlz, o = n & (Z - 1);
            for (int r = lane; r < P.qc_jb; r += 32) {
              const int sh = P.qc_shift[r * P.qc_kb + cb];
              if (sh < 0) continue;
              const int m = r * Z + ((o - sh) & (Z - 1));
              atomicXor(&sbits[m >> 5], 1u << (m & 31));
            }
          }
        } else {
          for (int fi = warp; fi < F; fi += nwarps) {
            const int n = flips[fi];
            const int e0 = __ldg(P.col_ptr + n), e1 = __ldg(P.col_ptr + n + 1);
            for (int e = e0 + lane; e < e1; e += 32) {
              const int m = __ldg(P.col_idx + e);
              atomicXor(&sbits[m >> 5], 1u << (m & 31));
            }
          }
        }
        __syncthreads();
      }
      logpos += F;
      flips_total += F;

      // ---- refresh signs of the checks that toggled; syndrome weight ----
      // Thread tid owns checks tid + kk*T in every iteration and remembers
      // their previous syndrome bits in `sprev`, so only toggled checks are
      // rewritten (negated; both copies on the guarded path).  With T a
      // multiple of 32, check tid + kk*T is bit `lane` of one warp-uniform word.
      if (TB > 0 && kGuard && split) {
        // split path: per-thread shared addresses once, [base + kk*TB] in PTX
        RefreshAddr A;
        const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
        const uint32_t fa = s0 + (uint32_t)P.off_fa + 4u * (uint32_t)tid;
        const uint32_t fb = s0 + (uint32_t)P.off_fb + 4u * (uint32_t)(tid + 1);
        asm("mov.b32 %0, %1;" : "=r"(A.fa) : "r"(fa));
        asm("mov.b32 %0, %1;" : "=r"(A.fa2) : "r"(fa + 4u * (uint32_t)N));
        asm("mov.b32 %0, %1;" : "=r"(A.fb) : "r"(fb));
        asm("mov.b32 %0, %1;" : "=r"(A.fb2) : "r"(fb + 4u * (uint32_t)N));
        A.invg = __float_as_uint(invGf);
        if (FILT) // per-check min2 (float)
          asm("mov.b32 %0, %1;" : "=r"(A.m2) : "r"(s0 + (uint32_t)P.off_m2s + 4u * (uint32_t)tid));
        else
          asm("mov.b32 %0, %1;" : "=r"(A.m2) : "r"(s0 + (uint32_t)P.off_m2s + 8u * (uint32_t)tid));
        asm("mov.b32 %0, %1;" : "=r"(A.a2) : "r"(s0 + (uint32_t)P.off_a2m + 2u * (uint32_t)tid));
        asm("mov.b32 %0, %1;" : "=r"(A.corr) : "r"(s0 + (uint32_t)P.off_corr));
        int pc = 0;
        RefreshKK<0, (TB > 0 ? KC : 1), (TB > 0 ? TB : 1), FILT>::run(A, sbits, sprev, pc, tid, warp, lane, M,
                                                              P.wmode == FWBF_WEIGHTS_IMWBF);
        if (lane == 0 && pc) atomicAdd(&misc[S_SWT], pc);
      } else if (TB > 0) {
        int pc = 0;
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          const int m = tid + kk * TB;
          if (kk * TB + warp * 32 < M) { // warp-uniform: this warp's word exists
            const uint32_t word = sbits[(kk * TB + warp * 32) >> 5];
            const bool ok = m < M;
            const bool s = (word >> lane) & 1u;
            const bool tog = ok && (s != (bool)((sprev >> kk) & 1u));
            if (tog) {
              if (kGuard && split) {
                const float v1 = -sFA[m];
                sFA[m] = v1;
                sFA[m + N] = v1;
                sFB[m + 1] = v1;
                sFB[m + N + 1] = v1;
                if (P.wmode == FWBF_WEIGHTS_IMWBF) { // correction sign flips with s_m
                  const int2 dl = reinterpret_cast<const int2 *>(sM2)[m];
                  const int a2 = sA2[m];
                  atomicAdd(&sCorr[2 * a2], s ? dl.x : -dl.x);
                  atomicAdd(&sCorr[2 * a2 + 1], s ? dl.y : -dl.y);
                }
              } else {
                const double v1 = -chk1[m];
                const double v2 = -chk2[m];
                chk1[m] = v1;
                chk2[m] = v2;
                if (CIRC && !FILT) { chk1[m + N] = v1; chk2[m + N] = v2; }
              }
            }
            sprev ^= (tog ? 1u : 0u) << kk;
            pc += __popc(word);
          }
        }
        if (lane == 0 && pc) atomicAdd(&misc[S_SWT], pc);
      } else {
        for (int kk = 0; kk < nKm; ++kk) {
          const int m = tid + kk * T;
          const bool ok = m < M;
          const uint32_t word = ok ? sbits[m >> 5] : 0u;
          const bool s = ok && ((word >> (m & 31)) & 1u);
          const bool tog = s != (bool)((sprev >> kk) & 1u);
          if (tog) {
            const double v1 = -chk1[m];
            const double v2 = -chk2[m];
            chk1[m] = v1;
            chk2[m] = v2;
            if (CIRC && !FILT) { chk1[m + N] = v1; chk2[m + N] = v2; }
            sprev ^= 1u << kk;
          }
          const uint32_t b = __ballot_sync(FULL_MASK, s);
          if (lane == 0 && b) atomicAdd(&misc[S_SWT], __popc(b));
        }
      }
      k += 1;
      __syncthreads();
      FWBF_PH(5)
    }

    // ---------------- outputs ----------------------------------------------------
    if (tid == 0) misc[S_BITERR] = 0;
    __syncthreads();
    {
      int be = 0;
      for (int w2 = tid; w2 < zw; w2 += T) {
        const uint32_t z = zbits[w2];
        if (P.z_bits) P.z_bits[f * P.z_ld + w2] = z;
        const uint32_t c = P.codeword_bits ? __ldg(P.codeword_bits + w2) : 0u;
        be += __popc(z ^ c);
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) be += __shfl_xor_sync(FULL_MASK, be, off);
      if (lane == 0 && be) atomicAdd(&misc[S_BITERR], be);
    }
    __syncthreads();
    if (tid == 0) {
      const int be = misc[S_BITERR];
      const int flags = (conv ? FWBF_FLAG_CONVERGED : 0) | (stalled ? FWBF_FLAG_STALLED : 0) |
                        (fastp ? 0 : FWBF_FLAG_ORDERED) | (misc[S_NONFIN] ? FWBF_FLAG_NONFINITE : 0) |
                        (split ? FWBF_FLAG_SPLIT32 : 0);
      if (P.iterations) P.iterations[f] = k;
      if (P.flags) P.flags[f] = (uint8_t)flags;
      if (P.flips_total) P.flips_total[f] = (int)flips_total;
      if (P.bit_errors) P.bit_errors[f] = be;
      if (P.iter_hist) atomicAdd((unsigned long long *)&P.iter_hist[k], 1ull);
      if (be && P.batch_word_err) atomicAdd(&P.batch_word_err[f / P.batch_frames], 1);
      c_frames += 1;
      c_biterr += be;
      c_worderr += be ? 1 : 0;
      c_iters += k;
      c_flips += flips_total;
      c_stalls += stalled;
      c_conv += conv;
      c_ordered += fastp ? 0 : 1;
      c_edges += (long long)P.n_edges * k;
      misc[S_NONFIN] = 0;
    }
  }

  if (P.phase_cycles && tid == 0)
    for (int i = 0; i < 8; ++i) atomicAdd((unsigned long long *)&P.phase_cycles[i], (unsigned long long)ph_acc[i]);
#undef FWBF_PH
  if (tid == 0 && P.counters && c_frames) {
    unsigned long long *c = (unsigned long long *)P.counters;
    atomicAdd(c + FWBF_CNT_FRAMES, (unsigned long long)c_frames);
    atomicAdd(c + FWBF_CNT_BIT_ERRORS, (unsigned long long)c_biterr);
    atomicAdd(c + FWBF_CNT_WORD_ERRORS, (unsigned long long)c_worderr);
    atomicAdd(c + FWBF_CNT_ITER_SUM, (unsigned long long)c_iters);
    atomicAdd(c + FWBF_CNT_FLIP_SUM, (unsigned long long)c_flips);
    atomicAdd(c + FWBF_CNT_STALLS, (unsigned long long)c_stalls);
    atomicAdd(c + FWBF_CNT_CONVERGED, (unsigned long long)c_conv);
    atomicAdd(c + FWBF_CNT_ORDERED_FRAMES, (unsigned long long)c_ordered);
    atomicAdd(c + FWBF_CNT_EDGE_VISITS, (unsigned long long)c_edges);
  }
}

// explicit instantiations used by the launcher
#define FWBF_INST(YT, C, KC, TB, WT) \
  template __global__ void decode_kernel<YT, C, KC, TB, WT, 0>(const __grid_constant__ KParams);
#define FWBF_INST_INC(YT, C, KC, TB, WT) \
  template __global__ void decode_kernel<YT, C, KC, TB, WT, 1>(const __grid_constant__ KParams);
#define FWBF_INST_FILT(YT, C, KC, TB, WT) \
  template __global__ void decode_kernel<YT, C, KC, TB, WT, 2>(const __grid_constant__ KParams);
FWBF_FAST_CONFIGS(FWBF_INST)
FWBF_F64_CONFIGS(FWBF_INST)
FWBF_INC_CONFIGS(FWBF_INST_INC)
FWBF_INC_CONFIGS(FWBF_INST_FILT)
FWBF_INST(double, true, 1, 0, 0)
FWBF_INST(float, false, 1, 0, 0)
FWBF_INST(double, false, 1, 0, 0)

} // namespace fwbf
