// fwbf_circ.cu -- filtered FWBF and MLP-WBF decoding of cyclic EG codes on B200.
//
// The headline path: FWBF (decoders.py:156-167, :181-183) on float32 y for a
// cyclic EG code whose length and weight are compiled in.  One persistent CTA
// decodes one frame at a time (frames from an atomic queue; except on the
// 6-CTA EG(1023) shape the next frame's y row is staged by a TMA bulk copy).  Same arithmetic contract as decode_kernel's
// MODE 2: the metric is summed in fp32 (within a
// per-frame bound fdelta of the exact one) and every block decision the bound
// leaves open is re-decided on exact column sums, so flips, iterations and
// flags equal the reference's.  Frames outside the filtered path's guard
// (non-finite y, all-zero |y|, a dynamic range beyond the fp64 guard) are
// appended to a defer list that decode_kernel then decodes on its exact paths.
//
// What differs from decode_kernel MODE 2 is the iteration's structure, built
// for the regime that dominates the run time (frames that fail to converge
// flip ~30 of 33 blocks per iteration and toggle ~40 % of the checks):
//   * selection: one warp per p-block, lanes over its columns; block maximum,
//     first index and the band test by REDUX on order-preserving keys (no
//     shuffle butterflies, every warp busy); lane jj of a warp keeps its jj-th
//     block's result and the warp applies all its flips in one lane pass;
//   * flips: the winning column n sets bits n and n + N of a doubled flip
//     bitmap (two RED.OR per flip instead of W syndrome atomics);
//   * toggles: the warp that owns syndrome word w computes which of its 32
//     checks toggled as XOR_j window(flips, 32 w + c_j) -- per lane one
//     offset c_j, a funnel shift of two bitmap words, one REDUX.XOR -- and
//     rewrites its own syndrome word, hard-decision word and the toggled
//     checks' signed minima and argmin corrections (no atomics on the
//     syndrome, no compare against remembered syndrome bits).
// The shared-memory layout is a compile-time function of the code (CLayout,
// fwbf_internal.h), so every shared access is [base + immediate].  Three CTA
// barriers per iteration (metric ready, flips chosen, state refreshed; MLP
// adds one between its per-warp lists and the merge); the flip bitmap, flip
// count and syndrome weight alternate between two slots by iteration parity
// so no extra barrier clears them.

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "fwbf_b200.h"
#include "fwbf_internal.h"
#include "fwbf_device.cuh"

namespace fwbf {

// order-preserving 32-bit key of a float (-0.0 and +0.0 tie; no NaN here)
__device__ __forceinline__ uint32_t fkey(float v) {
  const uint32_t u = __float_as_uint(v + 0.0f);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}
// 2^e for a normal exponent (|e| <= 1022), without ldexp's range handling
__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }
__device__ __forceinline__ float fkey_val(uint32_t k) {
  return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}

// Q16: the frame's 16-bit grid step for signed minima up to vmax: every
// |v| / G16 rounds to at most 32766 (vmax = 0: any step, every value is 0)
__device__ __forceinline__ float q16_grid(float vmax) {
  return vmax > 0.f ? __fmul_ru(vmax, 3.0520e-5f) : 1.0f; // 1 / 32766 = 3.05194e-5, rounded up
}

// One FWBF block decision, warp-wide (decoders.py:156-167, :181-183): lanes
// scan the block's columns (SHORT: one column per lane, p <= 32), REDUX gives
// the maximum key and the first index holding it, and the filter band decides
// whether the approximate argmax is the exact one; lane jj receives (v, i).
template <int WT, bool SHORT>
__device__ __forceinline__ void select_block(const KParams &P, uint32_t sE, const float *Efl, const float *sFA,
                                             const uint16_t *sA2, const float *sM2, const float *yabs, const int *eqp,
                                             int base, int lim, int lane, int jj, float fd2, float fdp, double &rv,
                                             int &ri) {
  float fv, fv2 = -INFINITY;
  int fi;
  if (SHORT) {
    fi = base + lane;
    float e; // (lanes past the block read inside the metric region; masked)
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e) : "r"(sE + 4u * (uint32_t)fi));
    fv = lane < lim ? e : -INFINITY;
  } else {
    fv = -INFINITY;
    fi = 0x7fffffff;
    for (int o = lane; o < lim; o += 32) { // ascending per lane, strict >
      const float e = Efl[base + o];
      fv2 = fmaxf(fv2, fminf(fv, e));
      if (e > fv) { fv = e; fi = base + o; }
    }
  }
  const uint32_t ka = fkey(fv);
  const uint32_t kmx = __reduce_max_sync(FULL_MASK, ka);
  const int imin = (int)__reduce_min_sync(FULL_MASK, ka == kmx ? (uint32_t)fi : 0xffffffffu);
  const float fmx = fkey_val(kmx);
  const float thr = fmx - fd2;
  // the block's runner-up: the winning lane's second value, every other
  // lane's first.  Settled when it is more than 2 fdelta below the maximum
  // (then the approximate argmax is the exact first maximum) and the maximum
  // is farther than fdelta from 0 (then its sign is exact); otherwise the
  // columns in the band are re-decided on exact sums.
  const float r = fi == imin ? fv2 : fv;
  if (__any_sync(FULL_MASK, r >= thr) || (fmx > -fdp && fmx <= fdp)) {
    const int eq = *eqp;
    const double qexp = pow2d(eq), qinv = pow2d(-eq);
    double ve = -dinf();
    int ie = 0x7fffffff;
    for (int o = lane; o < lim; o += 32) {
      const int n = base + o;
      if (Efl[n] >= thr) amax_combine(ve, ie, exact_split_metric(P, sFA, sA2, sM2, yabs, n, WT, qexp, qinv), n);
    }
    warp_amax_redux(ve, ie);
    if (lane == jj) { rv = ve; ri = ie; }
    if (lane == 0 && P.filter_stats) atomicAdd((unsigned long long *)P.filter_stats, 1ull);
  } else if (lane == jj) {
    rv = (double)fmx;
    ri = imin;
  }
}

// ---- MLP-WBF top-lambda (decoders.py:174-178) ------------------------------
// 64-bit ranking key of a column: the order-preserving float key above the
// complemented index, so a larger key is a larger value, then a lower index
// (np.argsort(-e, kind="stable")).
__device__ __forceinline__ unsigned long long mkey(float v, int n) {
  return ((unsigned long long)fkey(v) << 32) | (uint32_t)~n;
}
__device__ __forceinline__ float mkey_val(unsigned long long k) { return fkey_val((uint32_t)(k >> 32)); }
__device__ __forceinline__ int mkey_idx(unsigned long long k) { return (int)~(uint32_t)k; }

// Warp argmax of 64-bit keys by two REDUX reductions (keys are unique).
__device__ __forceinline__ unsigned long long warp_kmax(unsigned long long k) {
  const uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
  const uint32_t mh = __reduce_max_sync(FULL_MASK, hi);
  const uint32_t ml = __reduce_max_sync(FULL_MASK, hi == mh ? lo : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

// Per warp: the nl best keys of columns base + lane + 32 t (t < CPL), written
// best first to lst[0 .. nl).  Each lane sorts its CPL keys once; a round's
// winner is the warp maximum of the lane heads, and the winning lane pops.
template <int CPL>
__device__ __forceinline__ void mlp_warp_list(const float *Efl, int N, int base, int lane, int nl,
                                              unsigned long long *lst) {
  unsigned long long kk[CPL];
#pragma unroll
  for (int t = 0; t < CPL; ++t) {
    const int n = base + lane + 32 * t;
    kk[t] = mkey(n < N ? Efl[n] : -INFINITY, n);
  }
#pragma unroll
  for (int i = 0; i < CPL; ++i) // descending (CPL <= 4: a few compare-exchanges)
#pragma unroll
    for (int j = CPL - 1; j > i; --j)
      if (kk[j] > kk[j - 1]) { const unsigned long long t = kk[j]; kk[j] = kk[j - 1]; kk[j - 1] = t; }
  unsigned long long mine = 0ull;
  for (int r = 0; r < nl; ++r) {
    const unsigned long long w = warp_kmax(kk[0]);
    if (kk[0] == w) {
#pragma unroll
      for (int t = 0; t + 1 < CPL; ++t) kk[t] = kk[t + 1];
      kk[CPL - 1] = 0ull;
    }
    if (lane == r) mine = w;
  }
  if (lane < nl) lst[lane] = mine;
}

// Exact top-lambda of the columns whose filtered value is >= thr (the band
// the filter leaves open, and everything above it): lambda rounds of an
// exact-metric warp argmax over the columns still unranked.  Lane r receives
// the r-th (value, column).  Rare path; recomputes the candidates' exact
// sums each round.
template <int WT>
__device__ void mlp_exact_top(const KParams &P, const float *Efl, const float *sFA, const uint16_t *sA2,
                              const float *sM2, const float *yabs, int N, float thr, int lam, int lane,
                              double qexp, double qinv, double &xv, int &xi) {
  // Each lane caches the exact values of up to 4 of its candidates (columns
  // lane + 32 q): the exact sums run once, lanes in parallel, and the rounds
  // only rank cached values.  More than 4 candidates in a lane (quantised
  // inputs with many equal metrics): rounds recompute, ranking below the
  // previous round's winner.
  int c0 = -1, c1 = -1, c2 = -1, c3 = -1;
  bool over = false;
  for (int n = lane; n < N; n += 32)
    if (Efl[n] >= thr) {
      if (c0 < 0) c0 = n;
      else if (c1 < 0) c1 = n;
      else if (c2 < 0) c2 = n;
      else if (c3 < 0) c3 = n;
      else over = true;
    }
  if (!__any_sync(FULL_MASK, over)) {
    const double x0 = c0 >= 0 ? exact_split_metric(P, sFA, sA2, sM2, yabs, c0, WT, qexp, qinv) : -dinf();
    const double x1 = c1 >= 0 ? exact_split_metric(P, sFA, sA2, sM2, yabs, c1, WT, qexp, qinv) : -dinf();
    const double x2 = c2 >= 0 ? exact_split_metric(P, sFA, sA2, sM2, yabs, c2, WT, qexp, qinv) : -dinf();
    const double x3 = c3 >= 0 ? exact_split_metric(P, sFA, sA2, sM2, yabs, c3, WT, qexp, qinv) : -dinf();
    uint32_t tk = 0u; // ranked cache slots
    for (int r = 0; r < lam; ++r) {
      double ve = -dinf();
      int ie = 0x7fffffff, slot = -1;
      if (c0 >= 0 && !(tk & 1u) && (x0 > ve || (x0 == ve && c0 < ie))) { ve = x0; ie = c0; slot = 0; }
      if (c1 >= 0 && !(tk & 2u) && (x1 > ve || (x1 == ve && c1 < ie))) { ve = x1; ie = c1; slot = 1; }
      if (c2 >= 0 && !(tk & 4u) && (x2 > ve || (x2 == ve && c2 < ie))) { ve = x2; ie = c2; slot = 2; }
      if (c3 >= 0 && !(tk & 8u) && (x3 > ve || (x3 == ve && c3 < ie))) { ve = x3; ie = c3; slot = 3; }
      const int mine = ie;
      warp_amax_redux(ve, ie);
      if (slot >= 0 && mine == ie) tk |= 1u << slot;
      if (lane == r) { xv = ve; xi = ie; }
    }
    return;
  }
  double pv = dinf();
  int pi = -1;
  for (int r = 0; r < lam; ++r) {
    double ve = -dinf();
    int ie = 0x7fffffff;
    for (int n = lane; n < N; n += 32) {
      if (Efl[n] >= thr) {
        const double e = exact_split_metric(P, sFA, sA2, sM2, yabs, n, WT, qexp, qinv);
        if (e < pv || (e == pv && n > pi)) amax_combine(ve, ie, e, n);
      }
    }
    warp_amax_redux(ve, ie);
    pv = ve;
    pi = ie;
    if (lane == r) { xv = ve; xi = ie; }
  }
}

// Warp 0: merge the per-warp lists, decide the flips on the filtered values
// where the band settles them (the lambda-th and (lambda+1)-th more than
// 2 fdelta apart; every member farther than fdelta from 0 when thresholded),
// exactly otherwise; set the flip bits, the flip count, the stall flag and
// the flip log (ascending columns).  The stall policy's global argmax
// (decoders.py:214-222) is decided here too.
template <int NW, int WT>
__device__ void mlp_decide(const KParams &P, const float *Efl, const float *sFA, const uint16_t *sA2,
                           const float *sM2, const float *yabs, int *misc, const unsigned long long *lst,
                           int lam, int lane, float fd2, float fdp, uint32_t *fdc, int N, int *flog,
                           int sF, int sStall, int sEq) {
  int ptr = 0;
  unsigned long long head = lane < NW ? lst[32 * lane] : 0ull;
  unsigned long long top = 0ull; // lane r: the r-th best overall (filtered values)
  for (int r = 0; r < lam; ++r) {
    const unsigned long long w = warp_kmax(head);
    if (lane < NW && head == w) head = lst[32 * lane + (++ptr)];
    if (lane == r) top = w;
  }
  const unsigned long long nxt = warp_kmax(head); // the (lambda+1)-th
  const bool member = lane < lam;
  float v = mkey_val(top);
  int idx = mkey_idx(top);
  const float vT = __shfl_sync(FULL_MASK, v, lam - 1);
  const float v1 = lam > 1 ? __shfl_sync(FULL_MASK, v, 1) : mkey_val(nxt);
  const float vN = mkey_val(nxt);
  const bool thr_on = P.mlp_thr != 0;
  const bool settled = vN < vT - fd2;
  const bool signamb = thr_on && __any_sync(FULL_MASK, member && v > -fdp && v <= fdp);
  double xv = (double)v;
  const int eq = misc[sEq];
  if (!settled || signamb) { // exact decisions
    mlp_exact_top<WT>(P, Efl, sFA, sA2, sM2, yabs, N, vT - fd2, lam, lane, pow2d(eq), pow2d(-eq), xv, idx);
    if (lane == 0 && P.filter_stats) atomicAdd((unsigned long long *)P.filter_stats, 1ull);
  }
  bool sel = member && (!thr_on || xv > 0.0);
  uint32_t sm = __ballot_sync(FULL_MASK, sel);
  int stall = 0;
  if (!sm) { // no candidate: terminate, or flip the global argmax
    stall = 1;
    if (P.stall != FWBF_STALL_TERMINATE) {
      int gi = __shfl_sync(FULL_MASK, idx, 0);
      // lane 0 holds the exact top-1 if the exact path ran; otherwise the
      // filtered first is exact when it leads the second by more than 2 fdelta
      if (settled && !signamb && !(v1 < __shfl_sync(FULL_MASK, v, 0) - fd2)) {
        double gv;
        mlp_exact_top<WT>(P, Efl, sFA, sA2, sM2, yabs, N, __shfl_sync(FULL_MASK, v, 0) - fd2, 1, lane, pow2d(eq),
                          pow2d(-eq), gv, gi);
        gi = __shfl_sync(FULL_MASK, gi, 0);
        if (lane == 0 && P.filter_stats) atomicAdd((unsigned long long *)P.filter_stats + 1, 1ull);
      }
      sel = lane == 0;
      idx = gi;
      sm = 1u;
    }
  }
  if (sel) {
    const int i2 = idx + N;
    atomicOr(fdc + (idx >> 5), 1u << (idx & 31));
    atomicOr(fdc + (i2 >> 5), 1u << (i2 & 31));
  }
  if (flog) { // ascending columns: rank among the selected
    int rank = 0;
    for (int r = 0; r < 32; ++r) {
      const int o = __shfl_sync(FULL_MASK, idx, r);
      rank += ((sm >> r) & 1u) && o < idx;
    }
    if (sel) flog[rank] = idx;
  }
  if (lane == 0) {
    misc[sF] = __popc(sm);
    misc[sStall] = stall;
  }
}

template <int KC, int TB, int WT, int NN, int PB, bool Q16>
__global__ void __launch_bounds__(TB, CircShape<TB, PB>::kMinBlocks)
cdecode_kernel(const __grid_constant__ KParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using L = CLayout<NN, KC * TB, WT, PB < 0 ? (TB / 32) * 32 * 8 : 0, CircShape<TB, PB>::kStage>;
  constexpr int NW = TB / 32;
  constexpr int NP = KC / 2; // column pairs per thread in the gather
  constexpr int N = NN;      // cyclic code: N columns, N checks
  constexpr int ZW = L::ZW;  // words of a bit vector over N
  constexpr uint32_t LASTW = (N & 31) ? (1u << (N & 31)) - 1u : 0xffffffffu;
  static_assert(KC % 2 == 0 && WT > 0 && WT <= 64 && KC * TB >= N && KC * NW >= ZW, "shape");
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  float *ybuf = reinterpret_cast<float *>(smem_raw + L::YST); // y row (staged or loaded)
  float *Efl = reinterpret_cast<float *>(smem_raw + L::E);    // filtered metric
  float *yabs = Efl + L::EP;                                  // |y_n| (exact, float)
  float *sFA = reinterpret_cast<float *>(smem_raw + L::FA);   // signed min1, doubled
  float *sFB = reinterpret_cast<float *>(smem_raw + L::FB);   // the same, shifted one element
  // Q16: after frame init the FB region holds the minima quantised to signed
  // 16 bits instead -- QA doubled over [0, 2N), QB the same shifted one element
  int16_t *sQA = reinterpret_cast<int16_t *>(smem_raw + L::FB);
  int16_t *sQB = sQA + L::DBLF;
  float *sM2 = reinterpret_cast<float *>(smem_raw + L::M2);   // min2 per check
  uint16_t *sA2 = reinterpret_cast<uint16_t *>(smem_raw + L::A2); // argmin column per check
  int *sCorr = reinterpret_cast<int *>(smem_raw + L::CORR);   // coarse argmin correction per column
  uint32_t *sbits = reinterpret_cast<uint32_t *>(smem_raw + L::SB);
  uint32_t *zbits = reinterpret_cast<uint32_t *>(smem_raw + L::ZB);
  uint32_t *fdb = reinterpret_cast<uint32_t *>(smem_raw + L::FD); // [2][FDW] doubled flip bitmaps
  double *blk_v = reinterpret_cast<double *>(smem_raw + L::BV);
  int *blk_i = reinterpret_cast<int *>(smem_raw + L::BI);
  int *rot = reinterpret_cast<int *>(smem_raw + L::ROT);      // rotated offsets (ascending row walk)
  int *misc = reinterpret_cast<int *>(smem_raw + L::MISC);
  float *redf = reinterpret_cast<float *>(misc + 16);
  enum { S_FRAME = 0, S_SWT0, S_SWT1, S_F0, S_F1, S_EQ, S_VMAX, S_NONFIN, S_MSTALL };

  for (int j = tid; j < WT; j += TB) {
    rot[j] = P.off[j] - N; // check m's columns in ascending order: the wrapped
    rot[WT + j] = P.off[j]; // ones (m + c_j - N) first, from jwtab[m] on
  }
  if (tid == 0) misc[S_NONFIN] = 0;
  // this lane's offsets for the toggle windows: j = lane (and lane + 32)
  // (read from the shared rot table where used: a per-lane index into the
  // parameter bank would serialise over the lanes)

  // per-CTA counters (FWBF_CNT_* order), flushed once at the end
  __shared__ unsigned long long ctr[FWBF_CNT_EDGE_VISITS + 1];
  if (tid <= FWBF_CNT_EDGE_VISITS) ctr[tid] = 0ull;
  // optional per-phase cycle accounting (FWBF_PHASES; thread 0, at barriers)
  __shared__ long long ph_acc[8]; // [7] = last timestamp
  if (tid < 8) ph_acc[tid] = 0;
#define CPH(i)                                                  \
  if (P.phase_cycles && tid == 0) {                             \
    const long long t_ = clock64();                             \
    if (ph_acc[7]) ph_acc[i] += t_ - ph_acc[7];                 \
    ph_acc[7] = t_;                                             \
  }

  __shared__ __align__(8) uint64_t ystage_bar;
  unsigned ystage_phase = 0;
  const bool ystage = P.y_stage != 0;
  if (ystage && tid == 0) {
    mbar_init(&ystage_bar, 1);
    const unsigned t0 = atomicAdd(P.work_counter, 1u);
    misc[S_FRAME] = (int)t0;
    if ((long long)t0 < P.batch)
      bulk_row_to_smem(ybuf, reinterpret_cast<const float *>(P.y) + (long long)t0 * P.ld, (unsigned)L::YSTB,
                       &ystage_bar);
  }

  for (;;) {
    __syncthreads();
    if (tid == 0) {
      if (!ystage) misc[S_FRAME] = (int)atomicAdd(P.work_counter, 1u);
      misc[S_NONFIN] = 0; // (every read of the previous frame's flag is behind the barrier above)
    }
    __syncthreads();
    CPH(0)
    const unsigned fu = (unsigned)misc[S_FRAME];
    if ((long long)fu >= P.batch) break;
    const int f = (int)fu; // batch <= 2^31 - 1
    if (ystage) {
      mbar_wait(&ystage_bar, ystage_phase);
      ystage_phase ^= 1u;
    }

    // ---------------- init 1: y, hard decisions, guard statistics ----------------
    // |y_n| goes to yabs and, as a sort key, twice into the doubled key array
    // K0 (the min1 region, free until the records are written) and its
    // one-element-shifted copy K1: key = bits(|y|) << 1 | (first copy), so
    // among equal values a wrapped column (second copy: actual index
    // u - N, smaller than any unwrapped one) sorts first -- the ascending
    // column order of decoders.py:94-103 for every check.
    uint32_t *K0 = reinterpret_cast<uint32_t *>(sFA);
    uint32_t *K1 = reinterpret_cast<uint32_t *>(sFB);
    float lmin = INFINITY, lmax = 0.f;
    bool nonfin = false;
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const int n = tid + k * TB;
      const bool ok = n < N;
      float v = 0.f;
      if (ok) v = ystage ? ybuf[n] : __ldg(reinterpret_cast<const float *>(P.y) + (long long)f * P.ld + n);
      const uint32_t b = __ballot_sync(FULL_MASK, ok && v < 0.f);
      if (lane == 0 && k * TB + warp * 32 < N) zbits[(k * TB + warp * 32) >> 5] = b;
      if (ok) {
        nonfin |= !isfinite(v);
        const float a = fabsf(v);
        if (a > 0.f) lmin = fminf(lmin, a);
        lmax = fmaxf(lmax, a);
        sCorr[n] = 0;
        yabs[n] = a;
        const uint32_t key = __float_as_uint(a) << 1;
        K0[n] = key | 1u;
        K0[n + N] = key;
        K1[n + 1] = key | 1u;
        K1[n + N + 1] = key;
      }
    }
    if (tid < 2 * L::FDW) fdb[tid] = 0u;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      lmin = fminf(lmin, __shfl_xor_sync(FULL_MASK, lmin, off));
      lmax = fmaxf(lmax, __shfl_xor_sync(FULL_MASK, lmax, off));
    }
    nonfin = __any_sync(FULL_MASK, nonfin);
    if (lane == 0) {
      redf[warp] = lmin;
      redf[32 + warp] = lmax;
      if (nonfin) misc[S_NONFIN] = 1;
    }
    if (tid == 0) {
      misc[S_SWT0] = 0;
      misc[S_SWT1] = 0;
      misc[S_F0] = 0;
      misc[S_F1] = 0;
    }
    __syncthreads();
    // every thread takes the path decision itself (no serial section, no
    // second barrier) -- decode_kernel MODE 2's filtered-path condition:
    // finite y, some |y| > 0, every sum of 2 W weights exact in fp64
    // (2 W max|y| < 2^53 q with q = 2^(e_min - 23)), and the quantum within
    // the float range the filter's grid needs.  Everything else goes to the
    // exact kernel.
    float mn = INFINITY, ymaxf = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < NW; ++w2) { mn = fminf(mn, redf[w2]); ymaxf = fmaxf(ymaxf, redf[32 + w2]); }
    int eq = 0;
    bool keep = false;
    if (!misc[S_NONFIN] && mn < INFINITY) {
      int e = ((__float_as_int(mn) >> 23) & 0xff) - 127;
      if (e < -126) e = -126;
      eq = e - 23;
      keep = (2.0 * (double)WT * (double)ymaxf < ldexp(1.0, 30 + e)) && eq >= -123 && eq <= 77;
    }
    if (!keep) {
      if (tid == 0) {
        P.defer_list[atomicAdd(P.defer_count, 1u)] = f;
        if (ystage) { // every read of ybuf for this frame is done
          const unsigned t1 = atomicAdd(P.work_counter, 1u);
          misc[S_FRAME] = (int)t1;
          if ((long long)t1 < P.batch)
            bulk_row_to_smem(ybuf, reinterpret_cast<const float *>(P.y) + (long long)t1 * P.ld, (unsigned)L::YSTB,
                             &ystage_bar);
        }
      }
      continue;
    }
    if (tid == 0) {
      misc[S_EQ] = eq;
      misc[S_VMAX] = 0;
      if (ystage) { // ybuf is dead for this frame: claim the next one and start its copy
        const unsigned t1 = atomicAdd(P.work_counter, 1u);
        misc[S_FRAME] = (int)t1;
        if ((long long)t1 < P.batch)
          bulk_row_to_smem(ybuf, reinterpret_cast<const float *>(P.y) + (long long)t1 * P.ld, (unsigned)L::YSTB,
                           &ystage_bar);
      }
    }

    // ---------------- init 2: check minima, syndrome, signed weights -------------
    // quantum q = 2^eq, largest |y| ymaxf (both from the decision above)
    // coarse grid G = 2^gsh q for the argmin corrections: |Dc| <= 2^24
    const int gbits = ilogbf(ymaxf) + 1 - eq;
    const int gsh = gbits > 24 ? gbits - 24 : 0;
    const float Gf = ldexpf(1.f, gsh + eq);
    const float invGf = ldexpf(1.f, -(gsh + eq));
    const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    {
      // the doubled hard-decision bitmap zd (bit i = z_(i mod N)) into the
      // second flip bitmap, for the syndrome windows below
      uint32_t *zd = fdb + L::FDW;
      if (warp == 0)
        for (int wi = lane; wi < L::FDW; wi += 32) {
          auto bits = [&](int st) -> uint32_t { // bits st.. of z, zero outside [0, N)
            if (st <= -32 || st >= N) return 0u;
            if (st < 0) return zbits[0] << (-st);
            const int w0 = st >> 5, sh = st & 31;
            const uint32_t lo = zbits[w0], hi = w0 + 1 < ZW ? zbits[w0 + 1] : 0u;
            return __funnelshift_r(lo, hi, sh);
          };
          zd[wi] = bits(32 * wi) | bits(32 * wi - N);
        }
      // per check pair (m, m + 1), m = 2 tid + 2 TB qp: min1 / min2 keys and
      // the argmin's unwrapped column, one 8-byte key load per offset
      constexpr int NC = 2 * NP;
      uint32_t k1[NC], k2[NC];
      int ua[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) { k1[c] = 0xffffffffu; k2[c] = 0xffffffffu; ua[c] = 0; }
      const uint32_t baseT = s0 + 8u * (uint32_t)tid;
#pragma unroll
      for (int j = 0; j < WT; ++j) {
        const uint32_t so = (uint32_t)P.soff[j];
        const int cj = P.off[j];
#pragma unroll
        for (int qp = 0; qp < NP; ++qp) {
          uint32_t x, y2;
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(x), "=r"(y2) : "r"(baseT + so + (uint32_t)(qp * TB * 8)));
          const int u = 2 * tid + 2 * TB * qp + cj;
          {
            const bool lt = x < k1[2 * qp];
            k2[2 * qp] = min(k2[2 * qp], max(k1[2 * qp], x));
            k1[2 * qp] = min(k1[2 * qp], x);
            ua[2 * qp] = lt ? u : ua[2 * qp];
          }
          {
            const bool lt = y2 < k1[2 * qp + 1];
            k2[2 * qp + 1] = min(k2[2 * qp + 1], max(k1[2 * qp + 1], y2));
            k1[2 * qp + 1] = min(k1[2 * qp + 1], y2);
            ua[2 * qp + 1] = lt ? u : ua[2 * qp + 1]; // (column u + 1)
          }
        }
      }
      // min1 (float) parks in the metric region until the signs are known
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int m = 2 * tid + 2 * TB * (c >> 1) + (c & 1);
        if (m < N) {
          int col = ua[c] + (c & 1);
          if (col >= N) col -= N;
          Efl[m] = __uint_as_float(k1[c] >> 1);
          sM2[m] = __uint_as_float(k2[c] >> 1);
          sA2[m] = (uint16_t)col;
        }
      }
    }
    __syncthreads();
    {
      // syndrome word wd = XOR_j window(zd, 32 wd + c_j) (lane j: offset c_j);
      // then check m = tid + kk TB = 32 wd + lane writes its signed min1 and
      // its argmin column's coarse correction
      const int c0 = lane < WT ? rot[WT + lane] : 0;
      const int c1 = (WT > 32 && lane + 32 < WT) ? rot[WT + lane + 32] : 0;
      const uint32_t *zw0 = fdb + L::FDW + warp + (c0 >> 5);
      const uint32_t *zw1 = fdb + L::FDW + warp + (c1 >> 5);
      float wmax = 0.f;
      int swt = 0;
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const int wd = kk * NW + warp;
        if ((kk + 1) * NW <= ZW || wd < ZW) {
          uint32_t win = lane < WT ? __funnelshift_r(zw0[kk * NW], zw0[kk * NW + 1], c0 & 31) : 0u;
          if (WT > 32) win ^= __funnelshift_r(zw1[kk * NW], zw1[kk * NW + 1], c1 & 31);
          uint32_t sw = __reduce_xor_sync(FULL_MASK, win);
          if (wd == ZW - 1) sw &= LASTW;
          if (lane == 0) sbits[wd] = sw;
          swt += __popc(sw);
          const int m = wd * 32 + lane;
          if (m < N) {
            const bool par = (sw >> lane) & 1u;
            const float min1 = Efl[m];
            wmax = fmaxf(wmax, min1);
            const float s1v = par ? min1 : -min1;
            sFA[m] = s1v;
            if constexpr (!Q16) {
              sFA[m + N] = s1v;
              sFB[m + 1] = s1v;
              sFB[m + N + 1] = s1v;
            }
            const int Dc = coarse_dc(sM2[m], min1, invGf);
            atomicAdd(&sCorr[sA2[m]], par ? Dc : -Dc);
          }
        }
      }
#pragma unroll
      for (int off = 16; off; off >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(FULL_MASK, wmax, off));
      if (lane == 0) {
        atomicMax(&misc[S_VMAX], __float_as_int(wmax));
        if (swt) atomicAdd(&misc[S_SWT0], swt);
      }
    }
    __syncthreads();
    CPH(1)
    // filter bound (decode_kernel MODE 2): W sequential
    // fp32 adds of partial sums <= k vmax, the float finalize, the coarse
    // correction grid; fd2 = the band width 2 fdelta plus the rounding of
    // (max - fd2), both rounded outwards
    float fdp, fd2;
    {
      const double vmax = (double)__int_as_float(misc[S_VMAX]);
      const double ymax = (double)ymaxf;
      const double fdelta = ldexp(vmax * (0.5 * (double)WT * (double)(WT + 1)) * 1.001, -24) +
                            ldexp(((double)WT + P.alpha + 1.0) * ymax, -22) + 0.5 * (double)WT * (double)Gf +
                            ldexp((double)WT * ymax, -23);
      double fd = fdelta;
      if constexpr (Q16) // the quantisation: W values, each within 0.504 G16 of its grid point (rounding of v / G16 included)
        fd += (double)WT * 0.505 * (double)q16_grid(__int_as_float(misc[S_VMAX]));
      fdp = __double2float_ru(fd);
      fd2 = __double2float_ru(2.0 * fd + ldexp(((double)WT + P.alpha + 1.0) * ymax, -22));
    }
    float G16 = 0.f, invG16 = 0.f;
    if constexpr (Q16) {
      // the signed minima on the frame's 16-bit grid (|q| <= 32766), into the
      // dead shifted-copy region; a toggle later stores the negated value's
      // grid point, which is the negated grid point
      G16 = q16_grid(__int_as_float(misc[S_VMAX]));
      invG16 = __frcp_rn(G16);
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const int m = tid + kk * TB;
        if (m < N) {
          const int16_t q = (int16_t)__float2int_rn(__fmul_rn(sFA[m], invG16));
          sQA[m] = q;
          sQA[m + N] = q;
          sQB[m + 1] = q;
          sQB[m + N + 1] = q;
        }
      }
      __syncthreads();
    }

    // ---------------- iterations (decoders.py:204-229) -------------------------
    int k = 0, conv = 0, stalled = 0;
    int nflips = 0; // flips so far = this frame's flip-log position
    const float alf = (float)P.alpha;
    for (;;) {
      if (misc[S_SWT0 + (k & 1)] == 0) { conv = 1; break; }
      if (k >= P.kmax) break;

      // ---- filtered Eq.(1) metric: thread tid owns column pairs (2 tid + 2 TB q, +1);
      // per offset one 8-byte LDS [base + uoff_j] brings both columns' signed
      // min1, one FADD2 sums them
      {
        unsigned long long hs[NP];
        if constexpr (Q16) {
          int qlo[NP], qhi[NP];
#pragma unroll
          for (int qp = 0; qp < NP; ++qp) { qlo[qp] = 0; qhi[qp] = 0; }
          const uint32_t baseQ = s0 + 4u * (uint32_t)tid;
#pragma unroll
          for (int j = 0; j < WT; ++j) GatherQ16<0, NP, TB>::run(qlo, qhi, baseQ + (uint32_t)P.uoff16[j]);
#pragma unroll
          for (int qp = 0; qp < NP; ++qp)
            hs[qp] = f2pack(__fmul_rn((float)qlo[qp], G16), __fmul_rn((float)qhi[qp], G16));
        } else {
#pragma unroll
          for (int qp = 0; qp < NP; ++qp) hs[qp] = 0ull;
          const uint32_t baseT = s0 + 8u * (uint32_t)tid;
#pragma unroll
          for (int j = 0; j < WT; ++j) GatherF2<0, NP, TB>::run(hs, baseT + (uint32_t)P.uoff[j]);
        }
#pragma unroll
        for (int qp = 0; qp < NP; ++qp) {
          const float2 h = f2unpack(hs[qp]);
          const int n = 2 * tid + 2 * TB * qp;
          if (n + 1 < N) {
            const int2 cc = *reinterpret_cast<const int2 *>(sCorr + n);
            const float2 ya = *reinterpret_cast<const float2 *>(yabs + n);
            *reinterpret_cast<float2 *>(Efl + n) =
                make_float2(__fsub_rn(__fmaf_rn((float)cc.x, Gf, h.x), __fmul_rn(alf, ya.x)),
                            __fsub_rn(__fmaf_rn((float)cc.y, Gf, h.y), __fmul_rn(alf, ya.y)));
          } else if (n < N) {
            Efl[n] = __fsub_rn(__fmaf_rn((float)sCorr[n], Gf, h.x), __fmul_rn(alf, yabs[n]));
          }
        }
      }
      __syncthreads(); // B1: metric complete
      CPH(2)
      if (tid == 0) misc[S_SWT0 + ((k + 1) & 1)] = 0; // read at the top of iteration k - 1

      uint32_t *fdc = fdb + (k & 1) * L::FDW;
      int F;
      if constexpr (PB >= 0) {
        // ---- selection: warp per p-block (decoders.py:156-167, :181-183) ----
        // warp w takes blocks w + NW jj; lane jj keeps block jj's result, and
        // the warp applies all its flips with one pass of its lanes
        {
          const uint32_t sE = s0 + L::E;
          double rv = 0.0;
          int ri = 0;
          int jj = 0;
          if constexpr (PB > 0) { // block length compiled in: every block index and bound is an immediate
            constexpr int NBK = (N + PB - 1) / PB;
            constexpr int JM = (NBK + NW - 1) / NW;
            if constexpr (PB <= 32) {
              // all of this warp's blocks as independent straight-line chains
              // (load, key, two REDUX, band test) the scheduler can overlap;
              // blocks the band leaves open are re-decided afterwards
              float rvf = 0.f;
              uint32_t ambm = 0u;
  #pragma unroll
              for (int j2 = 0; j2 < JM; ++j2) {
                const int b = warp + j2 * NW;
                if ((j2 + 1) * NW > NBK && b >= NBK) break; // warp-uniform
                const int base = b * PB;
                const int lim = (N % PB == 0) ? PB : min(PB, N - base);
                const int fi = base + lane;
                const float e = Efl[fi]; // (lanes past the block read inside the metric region; masked)
                const float fv = lane < lim ? e : -INFINITY;
                const uint32_t ka = fkey(fv);
                const uint32_t kmx = __reduce_max_sync(FULL_MASK, ka);
                const int imin = (int)__reduce_min_sync(FULL_MASK, ka == kmx ? (uint32_t)fi : 0xffffffffu);
                const float fmx = fkey_val(kmx);
                // runner-up = every other lane's value (one column per lane)
                const bool amb = __any_sync(FULL_MASK, fi != imin && fv >= fmx - fd2) || (fmx > -fdp && fmx <= fdp);
                ambm |= (amb ? 1u : 0u) << j2;
                if (lane == j2) { rvf = fmx; ri = imin; }
                jj = j2 + 1;
              }
              rv = (double)rvf;
              while (ambm) { // rare: exact decisions
                const int j2 = __ffs(ambm) - 1;
                ambm &= ambm - 1u;
                const int base = (warp + j2 * NW) * PB;
                const int lim = (N % PB == 0) ? PB : min(PB, N - base);
                select_block<WT, true>(P, sE, Efl, sFA, sA2, sM2, yabs, misc + S_EQ, base, lim, lane, j2, fd2, fdp, rv,
                                       ri);
              }
            } else {
  #pragma unroll
              for (int j2 = 0; j2 < JM; ++j2) {
                const int b = warp + j2 * NW;
                if ((j2 + 1) * NW > NBK && b >= NBK) break; // warp-uniform
                const int base = b * PB;
                const int lim = (N % PB == 0) ? PB : min(PB, N - base);
                select_block<WT, false>(P, sE, Efl, sFA, sA2, sM2, yabs, misc + S_EQ, base, lim, lane, j2, fd2, fdp,
                                        rv, ri);
                jj = j2 + 1;
              }
            }
          } else {
            const int p = P.p;
            for (int base = warp * p; base < N; base += NW * p, ++jj) {
              const int lim = min(p, N - base);
              if (lim <= 32)
                select_block<WT, true>(P, sE, Efl, sFA, sA2, sM2, yabs, misc + S_EQ, base, lim, lane, jj, fd2, fdp, rv, ri);
              else
                select_block<WT, false>(P, sE, Efl, sFA, sA2, sM2, yabs, misc + S_EQ, base, lim, lane, jj, fd2, fdp, rv, ri);
            }
          }
          const bool mine = lane < jj;
          const bool flip = mine && rv > 0.0;
          if (mine) {
            const int b = warp + lane * NW;
            blk_v[b] = rv;
            blk_i[b] = ri;
          }
          if (flip) {
            const int i2 = ri + N;
            atomicOr(fdc + (ri >> 5), 1u << (ri & 31));
            atomicOr(fdc + (i2 >> 5), 1u << (i2 & 31));
          }
          const uint32_t fm = __ballot_sync(FULL_MASK, flip);
          if (lane == 0 && fm) atomicAdd(&misc[S_F0 + (k & 1)], __popc(fm));
        }
        __syncthreads(); // B2: flips chosen
        CPH(3)
        F = misc[S_F0 + (k & 1)];
        if (F == 0) {
          // nothing selected while the syndrome is nonzero (decoders.py:214-222)
          stalled = 1;
          if (P.stall == FWBF_STALL_TERMINATE) {
            if (tid == 0 && P.fliplog_counts) P.fliplog_counts[(long long)f * P.kmax + k] = 0;
            k += 1;
            break;
          }
          if (warp == 0) {
            const int nb = P.nblocks;
            double gv = -dinf();
            int gi = 0x7fffffff;
            for (int bb = lane; bb < nb; bb += 32) amax_combine(gv, gi, blk_v[bb], blk_i[bb]);
            warp_amax(gv, gi);
            // the block maxima are exact argmaxes, their values within fdelta
            const double thr = gv - (double)fd2;
            int nc = 0;
            for (int bb = lane; bb < nb; bb += 32) nc += blk_v[bb] >= thr;
            nc = __reduce_add_sync(FULL_MASK, nc);
            if (nc > 1) {
              const double qexp = pow2d(misc[S_EQ]), qinv = pow2d(-misc[S_EQ]);
              double ve = -dinf();
              int ie = 0x7fffffff;
              for (int bb = lane; bb < nb; bb += 32)
                if (blk_v[bb] >= thr)
                  amax_combine(ve, ie, exact_split_metric(P, sFA, sA2, sM2, yabs, blk_i[bb], WT, qexp, qinv), blk_i[bb]);
              warp_amax(ve, ie);
              gi = ie;
              if (lane == 0 && P.filter_stats) atomicAdd((unsigned long long *)P.filter_stats + 1, 1ull);
            }
            if (lane == 0) {
              const int g2 = gi + N;
              fdc[gi >> 5] |= 1u << (gi & 31);
              fdc[g2 >> 5] |= 1u << (g2 & 31);
              if (P.fliplog) P.fliplog[(long long)f * P.fliplog_stride + nflips] = gi;
            }
          }
          F = 1;
          __syncthreads();
        } else if (P.fliplog && warp == 0) { // ascending = block order
          const int nb = P.nblocks;
          int cnt = 0;
          for (int base = 0; base < nb; base += 32) {
            const int bb = base + lane;
            const bool pos = bb < nb && blk_v[bb] > 0.0;
            const uint32_t msk = __ballot_sync(FULL_MASK, pos);
            if (pos)
              P.fliplog[(long long)f * P.fliplog_stride + nflips + cnt + __popc(msk & ((1u << lane) - 1u))] = blk_i[bb];
            cnt += __popc(msk);
          }
        }
      } else {
        // ---- MLP-WBF: top-lambda by (value desc, index asc), > 0 when
        // thresholded, flipped in ascending order (decoders.py:174-178) ----
        // per warp: its columns' lambda + 1 best as 64-bit keys (REDUX
        // argmax rounds over lane-sorted heads); then warp 0 merges the lists
        // and decides on the filtered values, exactly where the band is open
        unsigned long long *lst = reinterpret_cast<unsigned long long *>(smem_raw + L::LST);
        const int lam = P.lam;
        mlp_warp_list<(N + TB - 1) / TB>(Efl, N, warp * 32 * ((N + TB - 1) / TB), lane, lam + 1, lst + warp * 32);
        __syncthreads();
        if (warp == 0)
          mlp_decide<NW, WT>(P, Efl, sFA, sA2, sM2, yabs, misc, lst, lam, lane, fd2, fdp, fdc, N,
                             P.fliplog ? P.fliplog + (long long)f * P.fliplog_stride + nflips : nullptr,
                             S_F0 + (k & 1), S_MSTALL, S_EQ);
        __syncthreads(); // B2: flips chosen
        CPH(3)
        F = misc[S_F0 + (k & 1)];
        if (misc[S_MSTALL]) {
          stalled = 1;
          if (P.stall == FWBF_STALL_TERMINATE) { // nothing selected (decoders.py:214-222)
            if (tid == 0 && P.fliplog_counts) P.fliplog_counts[(long long)f * P.kmax + k] = 0;
            k += 1;
            break;
          }
        }
      }
      if (P.fliplog && tid == 0) P.fliplog_counts[(long long)f * P.kmax + k] = F;

      // ---- toggles and refresh: warp w owns syndrome words w + NW kk ----
      {
        if (tid < L::FDW) fdb[((k + 1) & 1) * L::FDW + tid] = 0u; // last read in iteration k - 1
        if (tid == 0) misc[S_F0 + ((k + 1) & 1)] = 0;
        // bit b of word wd: check m = 32 wd + b toggles iff an odd number of
        // its columns m + c_j flipped = XOR over j of the doubled flip
        // bitmap's window starting at bit 32 wd + c_j (lane j: offset c_j)
        const int c0 = lane < WT ? rot[WT + lane] : 0;
        const int c1 = (WT > 32 && lane + 32 < WT) ? rot[WT + lane + 32] : 0;
        const uint32_t *fw0 = fdc + warp + (c0 >> 5);
        const uint32_t *fw1 = fdc + warp + (c1 >> 5);
        uint32_t tg[KC];
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          uint32_t win = lane < WT ? __funnelshift_r(fw0[kk * NW], fw0[kk * NW + 1], c0 & 31) : 0u;
          if (WT > 32) win ^= __funnelshift_r(fw1[kk * NW], fw1[kk * NW + 1], c1 & 31);
          tg[kk] = __reduce_xor_sync(FULL_MASK, win);
          if ((kk + 1) * NW > ZW && kk * NW + warp >= ZW) tg[kk] = 0u;          // no such word
          if ((kk + 1) * NW >= ZW && kk * NW + warp == ZW - 1) tg[kk] &= LASTW; // checks < N
        }
        // lane kk rewrites word kk's syndrome and hard decisions
        uint32_t mine = 0u;
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) mine = lane == kk ? tg[kk] : mine;
        int pcnt = 0;
        if (lane < KC) {
          const int wd = lane * NW + warp;
          if (wd < ZW) {
            const uint32_t snew = sbits[wd] ^ mine;
            sbits[wd] = snew;
            pcnt = __popc(snew);
            zbits[wd] ^= fdc[wd] & (wd == ZW - 1 ? LASTW : 0xffffffffu);
          }
        }
        pcnt = __reduce_add_sync(FULL_MASK, pcnt);
        if (lane == 0 && pcnt) atomicAdd(&misc[S_SWT0 + ((k + 1) & 1)], pcnt);
        // toggled checks m = tid + kk TB
        // (plain shared loads for every round first, so the rounds overlap;
        // the stores and the correction atomic only where the check toggled)
        float rv1[KC], rm2[KC];
        int ra2[KC];
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          const int m = tid + kk * TB;
          rv1[kk] = sFA[m];
          rm2[kk] = sM2[m];
          ra2[kk] = sA2[m];
        }
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          if ((tg[kk] >> lane) & 1u) {
            const int m = tid + kk * TB;
            const float v = -rv1[kk];
            sFA[m] = v;
            if constexpr (Q16) {
              const int16_t q = (int16_t)__float2int_rn(__fmul_rn(v, invG16));
              sQA[m] = q;
              sQA[m + N] = q;
              sQB[m + 1] = q;
              sQB[m + N + 1] = q;
            } else {
              sFA[m + N] = v;
              sFB[m + 1] = v;
              sFB[m + N + 1] = v;
            }
            const int dc = coarse_dc(rm2[kk], fabsf(v), invGf);
            atomicAdd(&sCorr[ra2[kk]], signbit(v) ? -2 * dc : 2 * dc);
          }
        }
      }
      nflips += F;
      k += 1;
      __syncthreads(); // B3: records, corrections, syndrome weight
      CPH(4)
    }

    // ---------------- outputs -----------------------------------------------------
    if (warp == 0) {
      int be = 0;
      for (int w2 = lane; w2 < ZW; w2 += 32) {
        const uint32_t z = zbits[w2];
        if (P.z_bits) P.z_bits[(long long)f * P.z_ld + w2] = z;
        const uint32_t c = P.codeword_bits ? __ldg(P.codeword_bits + w2) : 0u;
        be += __popc(z ^ c);
      }
      be = __reduce_add_sync(FULL_MASK, be);
      if (lane == 0) {
        const int flags = (conv ? FWBF_FLAG_CONVERGED : 0) | (stalled ? FWBF_FLAG_STALLED : 0) | FWBF_FLAG_SPLIT32;
        if (P.iterations) P.iterations[f] = k;
        if (P.flags) P.flags[f] = (uint8_t)flags;
        if (P.flips_total) P.flips_total[f] = nflips;
        if (P.bit_errors) P.bit_errors[f] = be;
        if (P.iter_hist) atomicAdd((unsigned long long *)&P.iter_hist[k], 1ull);
        if (be && P.batch_word_err) atomicAdd(&P.batch_word_err[f / P.batch_frames], 1);
        ctr[FWBF_CNT_FRAMES] += 1ull;
        ctr[FWBF_CNT_BIT_ERRORS] += (unsigned long long)be;
        ctr[FWBF_CNT_WORD_ERRORS] += be ? 1ull : 0ull;
        ctr[FWBF_CNT_ITER_SUM] += (unsigned long long)k;
        ctr[FWBF_CNT_FLIP_SUM] += (unsigned long long)nflips;
        ctr[FWBF_CNT_STALLS] += (unsigned long long)stalled;
        ctr[FWBF_CNT_CONVERGED] += (unsigned long long)conv;
        ctr[FWBF_CNT_EDGE_VISITS] += (unsigned long long)(P.n_edges * k);
      }
    }
  }

  if (P.phase_cycles && tid < 7) atomicAdd((unsigned long long *)&P.phase_cycles[tid], (unsigned long long)ph_acc[tid]);
#undef CPH
  if (P.counters && tid <= FWBF_CNT_EDGE_VISITS && tid != FWBF_CNT_ORDERED_FRAMES && ctr[FWBF_CNT_FRAMES])
    atomicAdd((unsigned long long *)P.counters + tid, ctr[tid]);
}

#define FWBF_INST_CIRC(KC, TB, WT, NN, PB) template __global__ void cdecode_kernel<KC, TB, WT, NN, PB, false>(const __grid_constant__ KParams);
FWBF_CIRC_CONFIGS(FWBF_INST_CIRC)
#define FWBF_INST_CIRC16(KC, TB, WT, NN, PB) template __global__ void cdecode_kernel<KC, TB, WT, NN, PB, true>(const __grid_constant__ KParams);
FWBF_CIRC_CONFIGS(FWBF_INST_CIRC16)

} // namespace fwbf
