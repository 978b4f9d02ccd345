// fwbf_qc.cu -- FWBF on quasi-cyclic codes (config D): one frame per CTA, the
// Eq.(1) metric fused with the block argmax, H as circulant shifts only.
//
// H is jb x kb circulant blocks of size Z (Z a power of two): row r Z + i
// holds column c Z + ((i + s_rc) mod Z) (qc_from_shifts; an absent block has
// no shift).  Column c Z + o meets row block r at check r Z + ((o - s_rc) mod Z),
// so the checks of a column ascend with r -- the reference's ascending check
// order (decoders.py:148-153).
//
// A p-block (32 | p, inside one block column) belongs to one warp; lane l
// takes columns base + l + 32 t (t < p / 32).  Its check in row block r is
// i0 + 32 t with i0 = (o0 + l - s) mod Z, so with each row block's records
// stored twice over their first p entries ("doubled head") the lane's
// records are m1_r[i0 + 32 t] / m2_r[i0 + 32 t]: two pointers per row block
// and an immediate offset per t -- no index arithmetic per edge.  An absent
// block points at a row of zeros.  Each column carries a 4-bit argmin mask
// (bit r: the column is the argmin of its check in row block r, set at frame
// init), so per edge the mask bit picks the sgn*min1 or the sgn*min2 array
// and one 4-byte load, float -> double and one DADD follow, in ascending
// check order from the first term (starting from +0.0 differs at most in the
// sign of a zero sum, which no comparison sees) -- the reference's fp64 sum.
// (Round 2, third session: the records were (min1, min2) pairs plus a u16
// argmin column per check, 3 shared wavefronts per warp and edge instead of
// 1 + 1/4.)
//
// Flips toggle z and syndrome words (atomic XOR); after a CTA barrier every
// thread negates the records of its own checks whose syndrome bit changed
// (plain loads/stores, both copies of head entries).  Frame init computes
// per check min1 / min2 / argmin / parity walking its columns in ascending
// order (strict <: the first minimum, decoders.py:87-103).
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "fwbf_b200.h"
#include "fwbf_internal.h"

namespace fwbf {

#define QFULL 0xffffffffu

__device__ __forceinline__ double qdinf() { return __longlong_as_double(0x7ff0000000000000LL); }

template <int TPC> // columns per lane per block (p / 32)
__global__ void __launch_bounds__(512, 2) qdecode_kernel(const __grid_constant__ QParams P) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int T = blockDim.x;
  const int N = P.n, M = P.m, Z = P.z, lgz = P.lgz, H = P.head, RS = P.z + P.head;
  float *ys = reinterpret_cast<float *>(sm + P.off_y);           // signed y, -0 -> +0
  float *m1 = reinterpret_cast<float *>(sm + P.off_m1);          // [jb][Z + H] sgn min1
  float *m2 = reinterpret_cast<float *>(sm + P.off_m2);          // [jb][Z + H] sgn min2 (MWBF: min1)
  uint8_t *cmask = reinterpret_cast<uint8_t *>(sm + P.off_cmask); // [N] argmin bit per row block
  const float *rzero = reinterpret_cast<const float *>(sm + P.off_zrec); // [H] zeros
  uint32_t *sbits = reinterpret_cast<uint32_t *>(sm + P.off_sbits);
  uint32_t *zbits = reinterpret_cast<uint32_t *>(sm + P.off_zbits);
  double *blk_v = reinterpret_cast<double *>(sm + P.off_blkv);
  int *blk_i = reinterpret_cast<int *>(sm + P.off_blki);
  int *misc = reinterpret_cast<int *>(sm + P.off_misc);
  enum { Q_FRAME = 0, Q_SWT, Q_F, Q_FLIP, Q_BE };
  const bool imw = P.wmode == FWBF_WEIGHTS_IMWBF;
  const double alpha = P.alpha;
  const int zw = (N + 31) >> 5, nKm = (M + T - 1) / T;

  for (int i = tid; i < H; i += T) const_cast<float *>(rzero)[i] = 0.f;
  long long c_frames = 0, c_biterr = 0, c_worderr = 0, c_iters = 0, c_flips = 0, c_stalls = 0, c_conv = 0,
            c_edges = 0;

  for (;;) {
    __syncthreads();
    if (tid == 0) misc[Q_FRAME] = (int)atomicAdd(P.work_counter, 1u);
    __syncthreads();
    const long long f = (long long)(unsigned)misc[Q_FRAME];
    if (f >= P.batch) break;

    // ---- init 1: y (float4 loads), hard decisions ----
    const float *yr = P.y + f * P.ld;
    bool nonfin = false;
    if (P.y_vec4) {
      for (int n0 = 4 * tid; n0 < N; n0 += 4 * T) {
        const float4 v4 = __ldg(reinterpret_cast<const float4 *>(yr + n0));
        const float vv[4] = {v4.x + 0.0f, v4.y + 0.0f, v4.z + 0.0f, v4.w + 0.0f}; // -0.0 -> +0.0
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (n0 + u < N) {
            ys[n0 + u] = vv[u];
            nonfin |= !isfinite(vv[u]);
          }
      }
    } else {
      for (int n = tid; n < N; n += T) {
        const float v = __ldg(yr + n) + 0.0f;
        ys[n] = v;
        nonfin |= !isfinite(v);
      }
    }
    for (int w = tid; w < (N + 3) >> 2; w += T) reinterpret_cast<uint32_t *>(cmask)[w] = 0u;
    if (tid == 0) { misc[Q_SWT] = 0; misc[Q_F] = 0; misc[Q_FLIP] = 0; }
    nonfin = __syncthreads_or(nonfin);
    for (int w0 = warp * 32; w0 < N; w0 += T) {
      const int n = w0 + lane;
      const uint32_t b = __ballot_sync(QFULL, n < N && ys[n] < 0.0f);
      if (lane == 0) zbits[w0 >> 5] = b;
    }
    // ---- init 2: per check min1 / min2 / argmin (ascending columns) / parity ----
    uint32_t sprev = 0;
    for (int k = 0; k < nKm; ++k) {
      const int m = tid + k * T;
      uint32_t par = 0;
      if (m < M) {
        const int r = m >> lgz, i = m & (Z - 1);
        float min1 = INFINITY, min2 = INFINITY;
        int ac = 0xffff;
        for (int cb = 0; cb < P.kb; ++cb) {
          const int s = P.shift[r * P.kb + cb];
          if (s < 0) continue;
          const int c = cb * Z + ((i + s) & (Z - 1));
          const float v = ys[c];
          par ^= __float_as_uint(v);
          const float a = fabsf(v);
          const bool lt = a < min1;
          min2 = fminf(min2, fmaxf(min1, a));
          min1 = fminf(min1, a);
          ac = lt ? c : ac;
        }
        par >>= 31;
        const float sg = par ? 1.0f : -1.0f;
        const float v1 = sg * min1, v2 = sg * (imw ? min2 : min1); // MWBF: every edge reads min1
        m1[r * RS + i] = v1;
        m2[r * RS + i] = v2;
        if (i < H) {
          m1[r * RS + Z + i] = v1;
          m2[r * RS + Z + i] = v2;
        }
        if (imw) atomicOr(reinterpret_cast<uint32_t *>(cmask) + (ac >> 2), 1u << (r + 8 * (ac & 3)));
        sprev |= par << k;
      }
      const uint32_t b = __ballot_sync(QFULL, par != 0);
      if (lane == 0 && k * T + warp * 32 < M) {
        sbits[(k * T + warp * 32) >> 5] = b;
        atomicAdd(&misc[Q_SWT], __popc(b));
      }
    }
    __syncthreads();

    // ---- iterations ----
    int k = 0, conv = 0, stalled = 0;
    long long logpos = 0, flips_total = 0;
    for (;;) {
      const int swt = misc[Q_SWT];
      if (swt == 0) { conv = 1; break; }
      if (k >= P.kmax) break;
      const int fs = (k & 1) ? Q_FLIP : Q_F; // this iteration's flip counter (the other is reset)
      if (tid == 0) misc[Q_F + Q_FLIP - fs] = 0;
      // fused metric + block argmax + flips: warp w owns blocks w, w + nwarps, ...
      for (int b = warp; b < P.nb; b += nwarps) {
        const int base = b * TPC * 32, cb = base >> lgz, o0 = (base & (Z - 1)) + lane;
        const float *p1[4], *p2[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int s = r < P.jb ? P.shift[r * P.kb + cb] : -1;
          const int i0 = (o0 - s) & (Z - 1);
          p1[r] = s >= 0 ? m1 + r * RS + i0 : rzero + lane;
          p2[r] = s >= 0 ? m2 + r * RS + i0 : rzero + lane;
        }
        double v = -qdinf();
        int vi = 0x7fffffff;
#pragma unroll
        for (int t = 0; t < TPC; ++t) {
          const int n = base + lane + 32 * t;
          const uint32_t mk = cmask[n]; // bit r: n is the argmin of its check in row block r
          // the reference's sum starts at +0.0; starting at the first term
          // instead differs at most in the sign of a zero sum, which no
          // comparison (> 0, argmax) can see
          double acc = 0.0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const double x = (double)(((mk >> r) & 1u) ? p2[r] : p1[r])[32 * t];
            acc = r == 0 ? x : __dadd_rn(acc, x);
          }
          const double e = __dsub_rn(acc, __dmul_rn(alpha, (double)fabsf(ys[n])));
          if (e > v) { v = e; vi = n; }
        }
        {
          // block argmax (value desc, index asc) by three REDUX reductions on
          // order-preserving 64-bit keys of the doubles
          unsigned long long key = (unsigned long long)__double_as_longlong(v + 0.0); // -0.0 -> +0.0: keys must tie
          key = (key >> 63) ? ~key : (key | 0x8000000000000000ull);
          const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
          const uint32_t mh = __reduce_max_sync(QFULL, hi);
          const uint32_t ml = __reduce_max_sync(QFULL, hi == mh ? lo : 0u);
          vi = (int)__reduce_min_sync(QFULL, (hi == mh && lo == ml) ? (uint32_t)vi : 0xffffffffu);
          unsigned long long km = ((unsigned long long)mh << 32) | ml;
          km = (km >> 63) ? (km & 0x7fffffffffffffffull) : ~km;
          v = __longlong_as_double((long long)km);
        }
        if (lane == 0) { blk_v[b] = v; blk_i[b] = vi; }
        if (v > 0.0) { // decoders.py:181-183: the warp applies its block's flip
          if (lane == 0) {
            atomicXor(&zbits[vi >> 5], 1u << (vi & 31));
            atomicAdd(&misc[fs], 1);
          }
          if (lane < P.jb) {
            const int cbv = vi >> lgz, o = vi & (Z - 1), s = P.shift[lane * P.kb + cbv];
            if (s >= 0) {
              const int m = (lane << lgz) + ((o - s) & (Z - 1));
              atomicXor(&sbits[m >> 5], 1u << (m & 31));
            }
          }
        }
      }
      __syncthreads();
      int F = misc[fs];
      if (F == 0) {
        // nothing selected with a nonzero syndrome (decoders.py:214-222)
        stalled = 1;
        if (P.stall == FWBF_STALL_TERMINATE) {
          if (tid == 0 && P.fliplog_counts) P.fliplog_counts[f * P.kmax + k] = 0;
          k += 1;
          break;
        }
        if (warp == 0) { // the global first maximum = the largest block maximum, lowest index
          double gv = -qdinf();
          int gi = 0x7fffffff;
          for (int bb = lane; bb < P.nb; bb += 32) {
            const double v2 = blk_v[bb];
            const int i2 = blk_i[bb];
            if (v2 > gv || (v2 == gv && i2 < gi)) { gv = v2; gi = i2; }
          }
#pragma unroll
          for (int off = 16; off; off >>= 1) {
            const double v2 = __shfl_xor_sync(QFULL, gv, off);
            const int i2 = __shfl_xor_sync(QFULL, gi, off);
            if (v2 > gv || (v2 == gv && i2 < gi)) { gv = v2; gi = i2; }
          }
          if (lane == 0) {
            atomicXor(&zbits[gi >> 5], 1u << (gi & 31));
            blk_v[gi / (TPC * 32)] = 1.0; // logged below as the single flip
            blk_i[gi / (TPC * 32)] = gi;
          }
          if (lane < P.jb) {
            const int cbv = gi >> lgz, o = gi & (Z - 1), s = P.shift[lane * P.kb + cbv];
            if (s >= 0) {
              const int m = (lane << lgz) + ((o - s) & (Z - 1));
              atomicXor(&sbits[m >> 5], 1u << (m & 31));
            }
          }
        }
        F = 1;
        __syncthreads();
      }
      if (P.fliplog && warp == 0) { // ascending = block order
        int cnt = 0;
        for (int b0 = 0; b0 < P.nb; b0 += 32) {
          const int bb = b0 + lane;
          const bool pos = bb < P.nb && blk_v[bb] > 0.0;
          const uint32_t msk = __ballot_sync(QFULL, pos);
          if (pos) P.fliplog[f * P.fliplog_stride + logpos + cnt + __popc(msk & ((1u << lane) - 1u))] = blk_i[bb];
          cnt += __popc(msk);
        }
        if (lane == 0) P.fliplog_counts[f * P.kmax + k] = F;
      }
      logpos += F;
      flips_total += F;
      // refresh: negate the records of this thread's toggled checks; syndrome weight
      if (tid == 0) misc[Q_SWT] = 0;
      __syncthreads();
      int pc = 0;
      for (int kk = 0; kk < nKm; ++kk) {
        const int m = tid + kk * T;
        if (kk * T + warp * 32 < M) {
          const uint32_t word = sbits[(kk * T + warp * 32) >> 5];
          const uint32_t s = (word >> lane) & 1u;
          if (m < M && s != ((sprev >> kk) & 1u)) {
            const int r = m >> lgz, i = m & (Z - 1);
            float *q1 = m1 + r * RS + i, *q2 = m2 + r * RS + i;
            const float a = -*q1, b = -*q2;
            *q1 = a;
            *q2 = b;
            if (i < H) { q1[Z] = a; q2[Z] = b; }
            sprev ^= 1u << kk;
          }
          pc += __popc(word);
        }
      }
      if (lane == 0 && pc) atomicAdd(&misc[Q_SWT], pc);
      k += 1;
      __syncthreads();
    }

    // ---- outputs ----
    if (tid == 0) misc[Q_BE] = 0;
    __syncthreads();
    int be = 0;
    for (int w2 = tid; w2 < zw; w2 += T) {
      const uint32_t z = zbits[w2];
      if (P.z_bits) P.z_bits[f * P.z_ld + w2] = z;
      const uint32_t cw = P.codeword_bits ? __ldg(P.codeword_bits + w2) : 0u;
      be += __popc(z ^ cw);
    }
    be = __reduce_add_sync(QFULL, be);
    if (lane == 0 && be) atomicAdd(&misc[Q_BE], be);
    __syncthreads();
    if (tid == 0) {
      be = misc[Q_BE];
      const int flags = (conv ? FWBF_FLAG_CONVERGED : 0) | (stalled ? FWBF_FLAG_STALLED : 0) | FWBF_FLAG_ORDERED |
                        (nonfin ? FWBF_FLAG_NONFINITE : 0);
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
      c_edges += (long long)P.n_edges * k;
    }
  }
  if (tid == 0 && P.counters && c_frames) {
    unsigned long long *c = (unsigned long long *)P.counters;
    atomicAdd(c + FWBF_CNT_FRAMES, (unsigned long long)c_frames);
    atomicAdd(c + FWBF_CNT_BIT_ERRORS, (unsigned long long)c_biterr);
    atomicAdd(c + FWBF_CNT_WORD_ERRORS, (unsigned long long)c_worderr);
    atomicAdd(c + FWBF_CNT_ITER_SUM, (unsigned long long)c_iters);
    atomicAdd(c + FWBF_CNT_FLIP_SUM, (unsigned long long)c_flips);
    atomicAdd(c + FWBF_CNT_STALLS, (unsigned long long)c_stalls);
    atomicAdd(c + FWBF_CNT_CONVERGED, (unsigned long long)c_conv);
    atomicAdd(c + FWBF_CNT_ORDERED_FRAMES, (unsigned long long)c_frames);
    atomicAdd(c + FWBF_CNT_EDGE_VISITS, (unsigned long long)c_edges);
  }
}

template __global__ void qdecode_kernel<1>(const __grid_constant__ QParams);
template __global__ void qdecode_kernel<2>(const __grid_constant__ QParams);
template __global__ void qdecode_kernel<4>(const __grid_constant__ QParams);
template __global__ void qdecode_kernel<8>(const __grid_constant__ QParams);
template __global__ void qdecode_kernel<16>(const __grid_constant__ QParams);

// ---------------------------------------------------------------------------
// Incremental variant (round 2, fourth session).  Only the checks whose
// syndrome bit toggled change any metric, and a toggled check changes only its
// own kb columns; on config D that is ~10 % of the columns per iteration.  So
// the metric of every column is kept in shared memory and only the columns of
// toggled checks are recomputed -- each from scratch, in ascending check order
// with the fp64 adds of the reference (decoders.py:148-153), never by a delta,
// so every stored value is the reference's value.
//
// What is stored is not the double but its float32 rounding as an
// order-preserving 32-bit key.  Rounding to nearest is monotone, so the exact
// first maximum of a block is one of the columns holding the block's largest
// key: when that key has one holder and is not the key of 0.0, the holder is
// the reference's argmax and the key's sign is the metric's sign.  Otherwise
// (equal keys, a zero, or a non-finite frame) the holders' exact doubles are
// recomputed and compared with the lowest-index tie rule, as the full pass of
// qdecode_kernel does.  The stall policy's global argmax applies the same rule
// across blocks.
//
// Layout per CTA: keys [N] (the y row sits there during the check scan),
// sgn*min1 / sgn*min2 [M] floats, argmin column [M] u16, the shift table,
// syndrome / z words, per-block results, the list of toggled checks.  |y_n| of
// a recomputed column is re-read from the frame's row in global memory (L2):
// QC(16384) takes 88 KB, two CTAs per SM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t qfkey(float v) { // order-preserving; callers pass v + 0.0f
  const uint32_t u = __float_as_uint(v);
  return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}
#define QKEY_ZERO 0x80000000u

struct QView {
  const float *rec;       // [2][M]: sgn*min1, then sgn*min2
  const uint8_t *cmask;   // [N] bit r: the column is the argmin of its check in row block r
  const int *sh;          // [jb][kb] shifts, -1 = absent block
  int lgz, zm, jb, kb, m;
  double alpha;
};

// the reference's Eq.(1) value of column c (ascending checks, fp64, first term first);
// ALLP: every circulant block is present
template <bool ALLP> __device__ __forceinline__ double qexact(const QView &V, int c, float y) {
  const int cb = c >> V.lgz, o = c & V.zm;
  const uint32_t mk = V.cmask[c];
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    double x = 0.0;
    if (r < V.jb) {
      const int s = V.sh[r * V.kb + cb];
      if (ALLP || s >= 0) {
        const int m = (r << V.lgz) + ((o - s) & V.zm);
        x = (double)V.rec[m + (((mk >> r) & 1u) ? V.m : 0)];
      }
    }
    acc = r == 0 ? x : __dadd_rn(acc, x);
  }
  return __dsub_rn(acc, __dmul_rn(V.alpha, (double)fabsf(y)));
}

// warp argmax (value desc, index asc) of doubles by three REDUX on order-preserving keys
__device__ __forceinline__ void qwarp_amax(double &v, int &vi) {
  unsigned long long key = (unsigned long long)__double_as_longlong(v + 0.0); // -0.0 -> +0.0: keys must tie
  key = (key >> 63) ? ~key : (key | 0x8000000000000000ull);
  const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
  const uint32_t mh = __reduce_max_sync(QFULL, hi);
  const uint32_t ml = __reduce_max_sync(QFULL, hi == mh ? lo : 0u);
  vi = (int)__reduce_min_sync(QFULL, (hi == mh && lo == ml) ? (uint32_t)vi : 0xffffffffu);
  unsigned long long km = ((unsigned long long)mh << 32) | ml;
  km = (km >> 63) ? (km & 0x7fffffffffffffffull) : ~km;
  v = __longlong_as_double((long long)km);
}

// a lane's TPC keys of block column range [base0, base0 + 32 TPC): consecutive
// columns per 16-byte load, consecutive lanes on consecutive 16 bytes
template <int TPC> __device__ __forceinline__ void qload_keys(const uint32_t *keys, int base0, int lane, uint32_t (&kk)[TPC]) {
  if constexpr (TPC >= 4) {
#pragma unroll
    for (int q = 0; q < TPC / 4; ++q) {
      const uint4 v = *reinterpret_cast<const uint4 *>(keys + base0 + 128 * q + 4 * lane);
      kk[4 * q] = v.x; kk[4 * q + 1] = v.y; kk[4 * q + 2] = v.z; kk[4 * q + 3] = v.w;
    }
  } else if constexpr (TPC == 2) {
    const uint2 v = *reinterpret_cast<const uint2 *>(keys + base0 + 2 * lane);
    kk[0] = v.x; kk[1] = v.y;
  } else {
    kk[0] = keys[base0 + lane];
  }
}
// the column of a lane's u-th key (ascending in u)
template <int TPC> __device__ __forceinline__ int qcol(int base0, int lane, int u) {
  if constexpr (TPC >= 4) return base0 + 128 * (u >> 2) + 4 * lane + (u & 3);
  else return base0 + TPC * lane + u;
}

// largest (hi) and second largest (lo) of a lane's keys: sorted pairs merged by a tree
template <int TPC> __device__ __forceinline__ void qtop2(const uint32_t (&kk)[TPC], uint32_t &hi, uint32_t &lo) {
  if constexpr (TPC == 1) {
    hi = kk[0];
    lo = 0;
  } else {
    uint32_t H[TPC / 2], L[TPC / 2];
#pragma unroll
    for (int i = 0; i < TPC / 2; ++i) {
      H[i] = max(kk[2 * i], kk[2 * i + 1]);
      L[i] = min(kk[2 * i], kk[2 * i + 1]);
    }
#pragma unroll
    for (int n = TPC / 2; n > 1; n >>= 1)
#pragma unroll
      for (int i = 0; i < n / 2; ++i) {
        const uint32_t h1 = H[2 * i], h2 = H[2 * i + 1];
        L[i] = __vimax3_u32(min(h1, h2), L[2 * i], L[2 * i + 1]);
        H[i] = max(h1, h2);
      }
    hi = H[0];
    lo = L[0];
  }
}

template <int TPC, bool ALLP> // columns per lane per block (p / 32); every circulant block present
__global__ void __launch_bounds__(512, 2) qinc_kernel(const __grid_constant__ QParams P) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int T = 512, nwarps = 16; // launch_qc launches 512 threads
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = P.n, M = P.m, Z = P.z, lgz = P.lgz;
  uint32_t *keys = reinterpret_cast<uint32_t *>(sm + P.off_y);   // [N] metric keys; y during the check scan
  float *ys = reinterpret_cast<float *>(sm + P.off_y);
  float *m1 = reinterpret_cast<float *>(sm + P.off_m1);          // [M] sgn min1, then [M] sgn min2 (MWBF: min1)
  float *m2 = m1 + P.m;
  uint8_t *cmask = reinterpret_cast<uint8_t *>(sm + P.off_cmask); // [N] argmin bit per row block
  int *sh = reinterpret_cast<int *>(sm + P.off_zrec);            // [jb][kb] shifts
  uint32_t *sbits = reinterpret_cast<uint32_t *>(sm + P.off_sbits);
  uint32_t *sold = reinterpret_cast<uint32_t *>(sm + P.off_sold); // syndrome words the records agree with
  uint32_t *zbits = reinterpret_cast<uint32_t *>(sm + P.off_zbits);
  double *blk_v = reinterpret_cast<double *>(sm + P.off_blkv);   // exact block maxima (stall policy only)
  int *blk_i = reinterpret_cast<int *>(sm + P.off_blki);         // block winner
  uint32_t *blk_k = reinterpret_cast<uint32_t *>(sm + P.off_blkk); // block maximum key (~0: decided exactly)
  int *blk_f = reinterpret_cast<int *>(sm + P.off_blkf);         // 1 = the block flipped (flip log only)
  int *tlist = reinterpret_cast<int *>(sm + P.off_list);         // toggled checks of this iteration
  int *dirty = reinterpret_cast<int *>(sm + P.off_dirty);        // [nb] 1 = the block is rescanned next selection
  int *dlist = dirty + P.nb;                                     // [2][nb] the dirty blocks, by iteration parity
  int *misc = reinterpret_cast<int *>(sm + P.off_misc);
  // counters used in alternate iterations come in pairs (slot = iteration parity)
  enum { Q_FRAME = 0, Q_BE, Q_SWT = 2, Q_F = 4, Q_L = 6, Q_D = 8 };
  const bool imw = P.wmode == FWBF_WEIGHTS_IMWBF;
  const int zw = (N + 31) >> 5, mw = (M + 31) >> 5, nKm = (M + T - 1) / T;
  QView V;
  V.rec = m1; V.cmask = cmask; V.sh = sh;
  V.lgz = lgz; V.zm = Z - 1; V.jb = P.jb; V.kb = P.kb; V.m = M; V.alpha = P.alpha;

  for (int i = tid; i < P.jb * P.kb; i += T) sh[i] = P.shift[i];
  long long c_frames = 0, c_biterr = 0, c_worderr = 0, c_iters = 0, c_flips = 0, c_stalls = 0, c_conv = 0,
            c_edges = 0;

  for (;;) {
    __syncthreads();
    if (tid == 0) misc[Q_FRAME] = (int)atomicAdd(P.work_counter, 1u);
    __syncthreads();
    const long long f = (long long)(unsigned)misc[Q_FRAME];
    if (f >= P.batch) break;

    // ---- init 1: y (float4 loads), hard decisions ----
    const float *yr = P.y + f * P.ld;
    bool nonfin = false;
    if (P.y_vec4) {
      for (int n0 = 4 * tid; n0 < N; n0 += 4 * T) {
        const float4 v4 = __ldg(reinterpret_cast<const float4 *>(yr + n0));
        const float vv[4] = {v4.x + 0.0f, v4.y + 0.0f, v4.z + 0.0f, v4.w + 0.0f}; // -0.0 -> +0.0
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (n0 + u < N) {
            ys[n0 + u] = vv[u];
            nonfin |= !isfinite(vv[u]);
          }
      }
    } else {
      for (int n = tid; n < N; n += T) {
        const float v = __ldg(yr + n) + 0.0f;
        ys[n] = v;
        nonfin |= !isfinite(v);
      }
    }
    for (int w = tid; w < (N + 3) >> 2; w += T) reinterpret_cast<uint32_t *>(cmask)[w] = 0u;
    if (tid >= 1 && tid < 10) misc[tid] = 0; // not Q_FRAME: other warps may still be reading it
    nonfin = __syncthreads_or(nonfin);
    for (int w0 = warp * 32; w0 < N; w0 += T) {
      const int n = w0 + lane;
      const uint32_t b = __ballot_sync(QFULL, n < N && ys[n] < 0.0f);
      if (lane == 0) zbits[w0 >> 5] = b;
    }
    // ---- init 2: per check min1 / min2 / argmin (ascending columns) / parity ----
    for (int k = 0; k < nKm; ++k) {
      const int m = tid + k * T;
      uint32_t par = 0;
      if (m < M) {
        const int r = m >> lgz, i = m & (Z - 1);
        float min1 = INFINITY, min2 = INFINITY;
        int ac = 0xffff;
        for (int cb = 0; cb < P.kb; ++cb) {
          const int s = sh[r * P.kb + cb];
          if (s < 0) continue;
          const int c = cb * Z + ((i + s) & (Z - 1));
          const float v = ys[c];
          par ^= __float_as_uint(v);
          const float a = fabsf(v);
          const bool lt = a < min1;
          min2 = fminf(min2, fmaxf(min1, a));
          min1 = fminf(min1, a);
          ac = lt ? c : ac;
        }
        par >>= 31;
        const float sg = par ? 1.0f : -1.0f;
        m1[m] = sg * min1;
        m2[m] = sg * (imw ? min2 : min1); // MWBF: every edge reads min1
        if (imw) atomicOr(reinterpret_cast<uint32_t *>(cmask) + (ac >> 2), 1u << (r + 8 * (ac & 3)));
      }
      const uint32_t b = __ballot_sync(QFULL, par != 0);
      if (lane == 0 && k * T + warp * 32 < M) {
        const int w = (k * T + warp * 32) >> 5;
        sbits[w] = b;
        sold[w] = b;
        atomicAdd(&misc[Q_SWT], __popc(b));
      }
    }
    __syncthreads();
    // ---- init 3: every column's metric; the key replaces y in the column's own slot ----
    for (int n = tid; n < N; n += T) keys[n] = qfkey((float)qexact<ALLP>(V, n, ys[n]) + 0.0f);
    for (int b = tid; b < P.nb; b += T) { dirty[b] = 1; dlist[b] = b; } // every block is scanned first
    if (tid == 0) misc[Q_D] = P.nb;
    __syncthreads();

    // ---- iterations ----
    int k = 0, conv = 0, stalled = 0;
    long long logpos = 0, flips_total = 0;
    for (;;) {
      const int par = k & 1;
      const int swt = misc[Q_SWT + par];
      if (swt == 0) { conv = 1; break; }
      if (k >= P.kmax) break;
      // the slots of the next iteration are cleared now (last read before the barrier behind us)
      if (tid == 0) { misc[Q_SWT + 1 - par] = 0; misc[Q_F + 1 - par] = 0; misc[Q_L + 1 - par] = 0; }
      // Selection over the dirty blocks only.  A clean block's largest key is
      // cached in blk_k and is below the key of 0 (a block that flips or was
      // decided exactly stays dirty), so it selects nothing; it turns dirty
      // when an update raises a column to its maximum or changes the holder.
      const int nd = misc[Q_D + par];
      const int *dl = dlist + par * P.nb;
      int *dn = dlist + (1 - par) * P.nb;
      for (int e = warp; e < nd; e += nwarps) {
        const int b = dl[e];
        const int base0 = b * TPC * 32;
        uint32_t kk[TPC];
        qload_keys<TPC>(keys, base0, lane, kk);
        uint32_t hi, lo; // the lane's largest and second largest key
        qtop2<TPC>(kk, hi, lo);
        const uint32_t Mk = __reduce_max_sync(QFULL, hi);
        const uint32_t holders = __ballot_sync(QFULL, hi == Mk);
        const bool amb = nonfin || Mk == QKEY_ZERO || (holders & (holders - 1u)) != 0u ||
                         __any_sync(QFULL, lo == Mk && TPC > 1);
        int vi = -1;
        bool pos;
        if (!amb) {
          pos = Mk > QKEY_ZERO;
          if (pos) {
            int idx = 0;
#pragma unroll
            for (int u = TPC - 1; u >= 0; --u)
              if (kk[u] == Mk) idx = qcol<TPC>(base0, lane, u);
            vi = __shfl_sync(QFULL, idx, __ffs(holders) - 1);
          }
        } else {
          double v = -qdinf();
          vi = 0x7fffffff;
#pragma unroll
          for (int u = 0; u < TPC; ++u)
            if (nonfin || kk[u] == Mk) {
              const int n = qcol<TPC>(base0, lane, u);
              const double e = qexact<ALLP>(V, n, __ldg(yr + n) + 0.0f);
              if (e > v) { v = e; vi = n; }
            }
          qwarp_amax(v, vi);
          pos = v > 0.0;
          if (lane == 0) { blk_v[b] = v; blk_i[b] = vi; }
        }
        if (lane == 0) {
          blk_k[b] = amb ? 0xffffffffu : Mk;
          if (P.fliplog) blk_f[b] = pos ? 1 : 0;
          if (amb || pos) dn[atomicAdd(&misc[Q_D + 1 - par], 1)] = b; // stays dirty
          else dirty[b] = 0;
        }
        if (pos) { // decoders.py:181-183: the warp applies its block's flip
          if (lane == 0) {
            blk_i[b] = vi;
            atomicXor(&zbits[vi >> 5], 1u << (vi & 31));
            atomicAdd(&misc[Q_F + par], 1);
          }
          if (lane < P.jb) {
            const int cbv = vi >> lgz, o = vi & (Z - 1), s = sh[lane * P.kb + cbv];
            if (s >= 0) {
              const int m = (lane << lgz) + ((o - s) & (Z - 1));
              atomicXor(&sbits[m >> 5], 1u << (m & 31));
            }
          }
        }
      }
      __syncthreads();
      int F = misc[Q_F + par];
      if (F == 0) {
        // nothing selected with a nonzero syndrome (decoders.py:214-222)
        stalled = 1;
        if (P.stall == FWBF_STALL_TERMINATE) {
          if (tid == 0 && P.fliplog_counts) P.fliplog_counts[f * P.kmax + k] = 0;
          k += 1;
          break;
        }
        // The global first maximum.  Gk = the largest key among the blocks
        // decided on keys alone; if no block was decided exactly and one
        // block holds Gk, its (unique) holder is the maximum -- monotone
        // rounding again.
        uint32_t Gk = 0;
        bool anyx = false;
        for (int bb = lane; bb < P.nb; bb += 32) {
          const uint32_t bk = blk_k[bb];
          anyx |= bk == 0xffffffffu;
          Gk = max(Gk, bk == 0xffffffffu ? 0u : bk);
        }
        Gk = __reduce_max_sync(QFULL, Gk);
        anyx = __any_sync(QFULL, anyx);
        int cntg = 0, bg = -1;
        for (int b0 = 0; b0 < P.nb; b0 += 32) {
          const uint32_t msk = __ballot_sync(QFULL, b0 + lane < P.nb && blk_k[b0 + lane] == Gk);
          if (msk) {
            cntg += __popc(msk);
            if (bg < 0) bg = b0 + __ffs(msk) - 1;
          }
        }
        if (!anyx && cntg == 1) {
          if (warp == (bg & (nwarps - 1))) {
            const int base0 = bg * TPC * 32;
            uint32_t kk[TPC];
            qload_keys<TPC>(keys, base0, lane, kk);
            int idx = -1;
#pragma unroll
            for (int u = TPC - 1; u >= 0; --u)
              if (kk[u] == Gk) idx = qcol<TPC>(base0, lane, u);
            const int gi = __shfl_sync(QFULL, idx, __ffs(__ballot_sync(QFULL, idx >= 0)) - 1);
            if (lane == 0) {
              atomicXor(&zbits[gi >> 5], 1u << (gi & 31));
              blk_f[bg] = 1; // logged below as the single flip
              blk_i[bg] = gi;
              if (atomicExch(&dirty[bg], 1) == 0) dn[atomicAdd(&misc[Q_D + 1 - par], 1)] = bg; // rescan: resets blk_f
            }
            if (lane < P.jb) {
              const int cbv = gi >> lgz, o = gi & (Z - 1), s = sh[lane * P.kb + cbv];
              if (s >= 0) {
                const int m = (lane << lgz) + ((o - s) & (Z - 1));
                atomicXor(&sbits[m >> 5], 1u << (m & 31));
              }
            }
          }
        } else {
          // exact maxima of the key-decided blocks that hold Gk (the others cannot hold the maximum)
          for (int b = warp; b < P.nb; b += nwarps) {
            const uint32_t bk = blk_k[b];
            if (bk == 0xffffffffu) continue;           // exact value and winner already stored
            double v = -qdinf();
            int vi = 0x7fffffff;
            if (bk == Gk) {
              const int base0 = b * TPC * 32;
              uint32_t kk[TPC];
              qload_keys<TPC>(keys, base0, lane, kk);
#pragma unroll
              for (int u = 0; u < TPC; ++u)
                if (kk[u] == bk) {
                  const int n = qcol<TPC>(base0, lane, u);
                  const double e = qexact<ALLP>(V, n, __ldg(yr + n) + 0.0f);
                  if (e > v) { v = e; vi = n; }
                }
              qwarp_amax(v, vi);
            }
            if (lane == 0) { blk_v[b] = v; blk_i[b] = vi; }
          }
          __syncthreads();
          if (warp == 0) { // the largest exact block maximum, lowest index
            double gv = -qdinf();
            int gi = 0x7fffffff;
            for (int bb = lane; bb < P.nb; bb += 32) {
              const double v2 = blk_v[bb];
              const int i2 = blk_i[bb];
              if (v2 > gv || (v2 == gv && i2 < gi)) { gv = v2; gi = i2; }
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
              const double v2 = __shfl_xor_sync(QFULL, gv, off);
              const int i2 = __shfl_xor_sync(QFULL, gi, off);
              if (v2 > gv || (v2 == gv && i2 < gi)) { gv = v2; gi = i2; }
            }
            if (lane == 0) {
              const int bg2 = gi / (TPC * 32);
              atomicXor(&zbits[gi >> 5], 1u << (gi & 31));
              blk_f[bg2] = 1; // logged below as the single flip
              blk_i[bg2] = gi;
              if (atomicExch(&dirty[bg2], 1) == 0) dn[atomicAdd(&misc[Q_D + 1 - par], 1)] = bg2; // rescan: resets blk_f
            }
            if (lane < P.jb) {
              const int cbv = gi >> lgz, o = gi & (Z - 1), s = sh[lane * P.kb + cbv];
              if (s >= 0) {
                const int m = (lane << lgz) + ((o - s) & (Z - 1));
                atomicXor(&sbits[m >> 5], 1u << (m & 31));
              }
            }
          }
        }
        F = 1;
        __syncthreads();
      }
      if (P.fliplog && warp == nwarps - 1) { // ascending = block order
        int cnt = 0;
        for (int b0 = 0; b0 < P.nb; b0 += 32) {
          const int bb = b0 + lane;
          const bool pos = bb < P.nb && blk_f[bb] != 0;
          const uint32_t msk = __ballot_sync(QFULL, pos);
          if (pos) P.fliplog[f * P.fliplog_stride + logpos + cnt + __popc(msk & ((1u << lane) - 1u))] = blk_i[bb];
          cnt += __popc(msk);
        }
        if (lane == 0) P.fliplog_counts[f * P.kmax + k] = F;
      }
      logpos += F;
      flips_total += F;
      // refresh, one syndrome word per thread: negate the records of the
      // checks whose bit changed since the records were last brought in line,
      // list them, add up the syndrome weight
      if (tid == T - 1) misc[Q_D + par] = 0; // consumed by this iteration's selection; refilled from the next one on
      if (tid < ((mw + 31) & ~31)) {
        uint32_t word = 0, tog = 0;
        if (tid < mw) {
          word = sbits[tid];
          tog = word ^ sold[tid];
        }
        if (tog) {
          sold[tid] = word;
          int at = atomicAdd(&misc[Q_L + par], __popc(tog));
          do {
            const int bit = __ffs(tog) - 1, m = 32 * tid + bit;
            tog &= tog - 1u;
            m1[m] = -m1[m];
            m2[m] = -m2[m];
            tlist[at++] = m;
          } while (tog);
        }
        const int pc = __reduce_add_sync(QFULL, __popc(word));
        if (lane == 0 && pc) atomicAdd(&misc[Q_SWT + 1 - par], pc);
      }
      k += 1;
      __syncthreads();
      // update: the columns of every toggled check, from scratch
      {
        const int L = misc[Q_L + par];
        // store a recomputed key; a clean block turns dirty when the column
        // reaches the cached maximum or was its holder (old key = maximum)
        auto qput = [&](int c, uint32_t nk) {
          const uint32_t ok = keys[c];
          if (nk == ok) return;
          keys[c] = nk;
          const int b = c / (TPC * 32);
          if (dirty[b] == 0) {
            const uint32_t bk = blk_k[b];
            if ((nk >= bk || ok == bk) && atomicExch(&dirty[b], 1) == 0) dn[atomicAdd(&misc[Q_D + 1 - par], 1)] = b;
          }
        };
        for (int e0 = warp; e0 < L; e0 += 4 * nwarps) {
          int cc[4];
          float yy[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) { // the row's y values first (L2 latency), then the sums
            const int e = e0 + u * nwarps;
            cc[u] = -1;
            yy[u] = 0.f;
            if (e < L && lane < P.kb) {
              const int m = tlist[e], r = m >> lgz, i = m & (Z - 1);
              const int s = sh[r * P.kb + lane];
              if (ALLP || s >= 0) {
                cc[u] = lane * Z + ((i + s) & (Z - 1));
                yy[u] = __ldg(yr + cc[u]);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cc[u] >= 0) qput(cc[u], qfkey((float)qexact<ALLP>(V, cc[u], yy[u] + 0.0f) + 0.0f));
        }
        for (int cb = 32 + lane; cb < P.kb; cb += 32) // block columns past the first 32 (wide codes)
          for (int e = warp; e < L; e += nwarps) {
            const int m = tlist[e], r = m >> lgz, i = m & (Z - 1);
            const int s = sh[r * P.kb + cb];
            if (s >= 0) {
              const int c = cb * Z + ((i + s) & (Z - 1));
              qput(c, qfkey((float)qexact<ALLP>(V, c, __ldg(yr + c) + 0.0f) + 0.0f));
            }
          }
      }
      __syncthreads();
    }

    // ---- outputs ----
    if (tid == 0) misc[Q_BE] = 0;
    __syncthreads();
    int be = 0;
    for (int w2 = tid; w2 < zw; w2 += T) {
      const uint32_t z = zbits[w2];
      if (P.z_bits) P.z_bits[f * P.z_ld + w2] = z;
      const uint32_t cw = P.codeword_bits ? __ldg(P.codeword_bits + w2) : 0u;
      be += __popc(z ^ cw);
    }
    be = __reduce_add_sync(QFULL, be);
    if (lane == 0 && be) atomicAdd(&misc[Q_BE], be);
    __syncthreads();
    if (tid == 0) {
      be = misc[Q_BE];
      const int flags = (conv ? FWBF_FLAG_CONVERGED : 0) | (stalled ? FWBF_FLAG_STALLED : 0) | FWBF_FLAG_ORDERED |
                        (nonfin ? FWBF_FLAG_NONFINITE : 0);
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
      c_edges += (long long)P.n_edges * k;
    }
  }
  if (tid == 0 && P.counters && c_frames) {
    unsigned long long *c = (unsigned long long *)P.counters;
    atomicAdd(c + FWBF_CNT_FRAMES, (unsigned long long)c_frames);
    atomicAdd(c + FWBF_CNT_BIT_ERRORS, (unsigned long long)c_biterr);
    atomicAdd(c + FWBF_CNT_WORD_ERRORS, (unsigned long long)c_worderr);
    atomicAdd(c + FWBF_CNT_ITER_SUM, (unsigned long long)c_iters);
    atomicAdd(c + FWBF_CNT_FLIP_SUM, (unsigned long long)c_flips);
    atomicAdd(c + FWBF_CNT_STALLS, (unsigned long long)c_stalls);
    atomicAdd(c + FWBF_CNT_CONVERGED, (unsigned long long)c_conv);
    atomicAdd(c + FWBF_CNT_ORDERED_FRAMES, (unsigned long long)c_frames);
    atomicAdd(c + FWBF_CNT_EDGE_VISITS, (unsigned long long)c_edges);
  }
}

template __global__ void qinc_kernel<1, false>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<1, true>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<2, false>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<2, true>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<4, false>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<4, true>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<8, false>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<8, true>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<16, false>(const __grid_constant__ QParams);
template __global__ void qinc_kernel<16, true>(const __grid_constant__ QParams);

} // namespace fwbf
