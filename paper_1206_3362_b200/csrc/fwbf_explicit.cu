// fwbf_explicit.cu -- FWBF on small explicit (CSR/CSC) codes: one frame per warp.
//
// The CTA-per-frame kernel (fwbf_decode.cu) spends most of an iteration of a
// short code (Gallager N = 504: 1,512 edges) in CTA barriers, dependent
// index loads and bank-conflicted check reads.  Here a warp owns a whole
// frame, so the loop needs only __syncwarp, and the code's structure is
// compiled on the host into per-lane slot tables shared by every warp:
//
//   * blocks of p columns are assigned to groups of G lanes (G a power of
//     two chosen on the host); lane `sub` of a group scans columns
//     sub, sub + G, ... of its block in ascending order ("slots");
//   * slot (round r, step c) of lane l lives at position pos = (r S + c) 32 + l,
//     so every per-slot array is read conflict-free (consecutive lanes,
//     consecutive words); tab[pos] packs the byte offsets of the column's
//     <= DV check records (ascending checks, 16 bits each);
//   * per check sgn min1 and sgn min2 as float32 (the exact minima), in two
//     arrays S2OFF bytes apart (S2OFF a power of two >= 128, so both copies
//     of a check sit in the same bank): an edge is one 4-byte load whose
//     address picks min2 (+S2OFF) by the column's argmin bit, converted to
//     fp64 exactly.  Checks are stored under a host-chosen label (a
//     permutation): lanes of one load instruction read checks whose labels
//     are spread over the 32 banks, so most loads take one or two wavefronts
//     instead of the ~3.7 of arbitrary labels.  Two constant
//     labels end the arrays: (-inf, -inf) fills the edges of padding slots
//     (their metric is -inf, never a maximum) and (0, 0) the missing edges of
//     columns lighter than DV (adding +0.0 to a sum that started at +0.0
//     changes nothing), so the loop has no branches.
//
// Per frame (decoders.py:189-229): y (float4 loads when rows are 16-byte
// aligned) -> signed y per slot + hard decisions; per check min1 / min2 /
// argmin / parity (decoders.py:87-103) walking the row in ascending column
// order; then per iteration the Eq.(1) metric in the reference's arithmetic
// (fp64 adds in ascending check order from 0.0, minus fl(alpha |y|),
// decoders.py:148-153), the block argmax with lowest-index ties and the > 0
// threshold (decoders.py:156-167, 181-183), the stall policy
// (decoders.py:214-222), and the flips: z and syndrome bits toggled by
// atomic XOR, the checks' record signs by atomic XOR of the sign bits
// (XOR commutes, so two flips toggling one check cancel exactly).  (An
// owner-lane refresh of the records instead of the sign atomics -- every lane
// rescans its checks' syndrome words -- measured 7 % slower on Gallager(504).)
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "fwbf_b200.h"
#include "fwbf_internal.h"

namespace fwbf {

#define XFULL 0xffffffffu

__device__ __forceinline__ double xdinf() { return __longlong_as_double(0x7ff0000000000000LL); }

template <int DV>
__global__ void __launch_bounds__(256) xdecode_kernel(const __grid_constant__ XParams P) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = P.n, M = P.m, R = P.rounds, S = P.slots, G = 1 << P.lg_g;
  const int nslot = R * S * 32;

  // ---- CTA-shared code tables (same for every frame); the row tables used
  // only at frame init stay in global memory (L1/L2) ----
  unsigned long long *tab = reinterpret_cast<unsigned long long *>(sm + P.off_tab);
  uint16_t *cpos = reinterpret_cast<uint16_t *>(sm + P.off_cpos);
  const uint32_t *rtab = P.rtab;
  const int *rptr = P.row_ptr;
  for (int i = tid; i < nslot; i += blockDim.x) tab[i] = __ldg(P.tab + i);
  for (int i = tid; i < N; i += blockDim.x) cpos[i] = __ldg(P.cpos + i);

  // ---- this warp's frame state ----
  unsigned char *W = sm + P.off_warp0 + warp * P.warp_bytes;
  float *rec = reinterpret_cast<float *>(W + P.wo_rec);        // by label: sgn*min1; + S2OFF: sgn*min2
  float *ys = reinterpret_cast<float *>(W + P.wo_ys);           // [nslot] signed y per slot (-0 -> +0)
  uint8_t *am = W + P.wo_am;                                    // [nslot] argmin bits per slot
  uint32_t *sb = reinterpret_cast<uint32_t *>(W + P.wo_sb);     // syndrome bits
  uint32_t *zw = reinterpret_cast<uint32_t *>(W + P.wo_zw);     // hard decisions by column
  int *bflip = reinterpret_cast<int *>(W + P.wo_bf);            // per block: flipped column or -1
  const int zwords = (N + 31) >> 5;
  const bool imw = P.wmode == FWBF_WEIGHTS_IMWBF;
  const double alpha = P.alpha;
  if (lane == 0) { // the two constant records after the M check records
    float *rec2 = rec + (P.s2off >> 2);
    rec[M] = rec2[M] = -INFINITY;
    rec[M + 1] = rec2[M + 1] = 0.0f;
  }
  __syncthreads();
  const uint32_t recb = (uint32_t)__cvta_generic_to_shared(rec);
  float *rec2 = rec + (P.s2off >> 2);
  const int s2sh = P.s2sh; // S2OFF = 1 << s2sh

  long long c_frames = 0, c_biterr = 0, c_worderr = 0, c_iters = 0, c_flips = 0, c_stalls = 0, c_conv = 0,
            c_edges = 0;

  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(P.work_counter, 1u);
    t = __shfl_sync(XFULL, t, 0);
    const long long f = (long long)t; // unsigned tickets: see decode_kernel
    if (f >= P.batch) break;

    // ---- init: y -> signed y per slot, hard decisions by column ----
    for (int i = lane; i < (nslot >> 2); i += 32) reinterpret_cast<uint32_t *>(am)[i] = 0u;
    const float *yr = P.y + f * P.ld;
    bool nonfin = false;
    if (P.y_vec4) {
      for (int i = lane; i < zwords; i += 32) zw[i] = 0u;
      __syncwarp();
      for (int n0 = 4 * lane; n0 < N; n0 += 128) {
        const float4 v4 = __ldg(reinterpret_cast<const float4 *>(yr + n0));
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
        uint32_t nib = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int n = n0 + u;
          if (n < N) {
            const float v = vv[u] + 0.0f; // -0.0 -> +0.0: the sign bit is the hard decision
            ys[cpos[n]] = v;
            nib |= (v < 0.0f ? 1u : 0u) << u;
            nonfin |= !isfinite(v);
          }
        }
        if (nib) atomicOr(&zw[n0 >> 5], nib << (n0 & 31));
      }
    } else {
      for (int n0 = 0; n0 < N; n0 += 32) {
        const int n = n0 + lane;
        float v = n < N ? __ldg(yr + n) + 0.0f : 0.0f;
        const uint32_t b = __ballot_sync(XFULL, n < N && v < 0.0f);
        if (lane == 0) zw[n0 >> 5] = b;
        if (n < N) {
          ys[cpos[n]] = v;
          nonfin |= !isfinite(v);
        }
      }
    }
    nonfin = __any_sync(XFULL, nonfin);
    __syncwarp();

    // ---- per-check minima, argmin, parity (ascending columns, strict <),
    // lanes over labels j (check invp[j]) ----
    int swt = 0;
    for (int m0 = 0; m0 < M; m0 += 32) {
      const int j = m0 + lane;
      uint32_t par = 0;
      if (j < M) {
        const int m = __ldg(P.invp + j);
        float min1 = INFINITY, min2 = INFINITY;
        int ae = -1;
        const int e1 = __ldg(rptr + m + 1);
        for (int e = __ldg(rptr + m); e < e1; ++e) {
          const float v = ys[__ldg(rtab + e) & 0xffffu];
          par ^= __float_as_uint(v);
          const float a = fabsf(v);
          const bool lt = a < min1;
          min2 = fminf(min2, fmaxf(min1, a));
          min1 = fminf(min1, a);
          ae = lt ? e : ae;
        }
        par >>= 31;
        const float sg = par ? 1.0f : -1.0f;
        // MWBF (include-self minimum): every edge reads min1
        rec[j] = sg * min1; // float32 minima: exact; converted to fp64 per edge
        rec2[j] = sg * (imw ? min2 : min1);
        if (imw && ae >= 0) { // the argmin column reads min2 at this check's position in its list
          const uint32_t pe = __ldg(rtab + ae);
          const uint32_t pos = pe & 0xffffu;
          atomicOr(reinterpret_cast<uint32_t *>(am) + (pos >> 2), (1u << (pe >> 16)) << (8 * (pos & 3)));
        }
      }
      const uint32_t b = __ballot_sync(XFULL, par != 0);
      if (lane == 0) sb[m0 >> 5] = b;
      swt += __popc(b);
    }
    __syncwarp();

    // ---- iterations ----
    int k = 0, conv = 0, stalled = 0;
    long long logpos = 0, flips_total = 0;
    for (;;) {
      if (swt == 0) { conv = 1; break; }
      if (k >= P.kmax) break;
      double gbest = -xdinf(); // this lane's best block maximum (stall policy)
      int gcol = 0x7fffffff;
      int nflip = 0;
      for (int r = 0; r < R; ++r) {
        double best = -xdinf();
        int bc = -1;
        const int pos0 = r * S * 32 + lane;
#pragma unroll 2
        for (int c = 0; c < S; ++c) {
          const int pos = pos0 + c * 32;
          const unsigned long long w = tab[pos];
          const uint32_t amk = am[pos];
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < DV; ++q) {
            // record byte offset, + S2OFF (min2) when this check's argmin is the column
            const uint32_t off = ((uint32_t)(w >> (16 * q)) & 0xffffu) | ((amk << (s2sh - q)) & (1u << s2sh));
            float vf;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(vf) : "r"(recb + off));
            const double v = (double)vf;
            // starting at the first term instead of +0.0 differs at most in
            // the sign of a zero sum, which no comparison can see
            acc = q == 0 ? v : __dadd_rn(acc, v);
          }
          const double e = __dsub_rn(acc, __dmul_rn(alpha, (double)fabsf(ys[pos])));
          if (e > best) { best = e; bc = c; }
        }
        // group butterfly: value desc, column asc (column = base + sub + G c)
        const int b = r * (32 >> P.lg_g) + (lane >> P.lg_g);
        const int sub = lane & (G - 1);
        int col = bc >= 0 ? b * P.p + sub + G * bc : 0x7fffffff;
        for (int off = G >> 1; off; off >>= 1) {
          const double v2 = __shfl_xor_sync(XFULL, best, off);
          const int c2 = __shfl_xor_sync(XFULL, col, off);
          if (v2 > best || (v2 == best && c2 < col)) { best = v2; col = c2; }
        }
        const bool leader = sub == 0 && b < P.nb;
        if (leader) {
          if (best > gbest || (best == gbest && col < gcol)) { gbest = best; gcol = col; }
          bflip[b] = best > 0.0 ? col : -1; // decoders.py:181-183
        }
        nflip += __popc(__ballot_sync(XFULL, leader && best > 0.0));
      }
      __syncwarp(); // every metric read of rec / sb precedes the flips
      int F = nflip;
      if (F == 0) {
        // nothing selected with a nonzero syndrome (decoders.py:214-222)
        stalled = 1;
        if (P.stall == FWBF_STALL_TERMINATE) {
          if (lane == 0 && P.fliplog_counts) P.fliplog_counts[f * P.kmax + k] = 0;
          k += 1;
          break;
        }
        // flip the global first maximum: the largest block maximum, lowest column
#pragma unroll
        for (int off = 16; off; off >>= 1) {
          const double v2 = __shfl_xor_sync(XFULL, gbest, off);
          const int c2 = __shfl_xor_sync(XFULL, gcol, off);
          if (v2 > gbest || (v2 == gbest && c2 < gcol)) { gbest = v2; gcol = c2; }
        }
        // every block maximum was <= 0, so every bflip entry is already -1
        if (lane == 0 && gcol < N) bflip[gcol / P.p] = gcol;
        F = 1;
        __syncwarp();
      }
      // apply the flips in block order (= ascending columns); log them
      int dsw = 0, cnt = 0;
      for (int b0 = 0; b0 < P.nb; b0 += 32) {
        const int b = b0 + lane;
        const int c = b < P.nb ? bflip[b] : -1;
        const uint32_t msk = __ballot_sync(XFULL, c >= 0);
        if (c >= 0) {
          if (P.fliplog) P.fliplog[f * P.fliplog_stride + logpos + cnt + __popc(msk & ((1u << lane) - 1u))] = c;
          atomicXor(&zw[c >> 5], 1u << (c & 31));
          const unsigned long long w = tab[cpos[c]];
#pragma unroll
          for (int q = 0; q < DV; ++q) {
            const uint32_t m = ((uint32_t)(w >> (16 * q)) & 0xffffu) >> 2; // label
            if (m < (uint32_t)M) { // not the (0, 0) record of a missing edge
              const uint32_t old = atomicXor(&sb[m >> 5], 1u << (m & 31));
              dsw += ((old >> (m & 31)) & 1u) ? -1 : 1;
              // negate sgn*min1 and sgn*min2 of the toggled check: XOR of the
              // sign bit in each double's high word (32-bit shared atomics are
              // native; 64-bit XOR would be a CAS loop)
              atomicXor(reinterpret_cast<uint32_t *>(rec + m), 0x80000000u);
              atomicXor(reinterpret_cast<uint32_t *>(rec2 + m), 0x80000000u);
            }
          }
        }
        cnt += __popc(msk);
      }
      if (lane == 0 && P.fliplog) P.fliplog_counts[f * P.kmax + k] = F;
      swt += __reduce_add_sync(XFULL, dsw);
      __syncwarp();
      logpos += F;
      flips_total += F;
      k += 1;
    }

    // ---- outputs ----
    int be = 0;
    for (int i = lane; i < zwords; i += 32) {
      const uint32_t z = zw[i];
      if (P.z_bits) P.z_bits[f * P.z_ld + i] = z;
      const uint32_t cw = P.codeword_bits ? __ldg(P.codeword_bits + i) : 0u;
      be += __popc(z ^ cw);
    }
    be = __reduce_add_sync(XFULL, be);
    if (lane == 0) {
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
    __syncwarp();
  }
  if (lane == 0 && P.counters && c_frames) {
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

template <int DV>
__global__ void __launch_bounds__(256) xinc_kernel(const __grid_constant__ XParams P) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = P.n, M = P.m, R = P.rounds, S = P.slots, G = 1 << P.lg_g;
  const int nslot = R * S * 32;

  // ---- CTA-shared code tables (same for every frame); the row tables used
  // only at frame init stay in global memory (L1/L2) ----
  unsigned long long *tab = reinterpret_cast<unsigned long long *>(sm + P.off_tab);
  uint16_t *cpos = reinterpret_cast<uint16_t *>(sm + P.off_cpos);
  const uint32_t *rtab = P.rtab;
  const int *rptr = P.row_ptr;
  for (int i = tid; i < nslot; i += blockDim.x) tab[i] = __ldg(P.tab + i);
  for (int i = tid; i < N; i += blockDim.x) cpos[i] = __ldg(P.cpos + i);
  // per check label: the slots of the check's columns (DCS = 2^dcs_sh entries, 0xffff = none)
  uint16_t *ctab = reinterpret_cast<uint16_t *>(sm + P.off_ctab);
  for (int i = tid; i < (M << P.dcs_sh); i += blockDim.x) ctab[i] = __ldg(P.ctab + i);

  // ---- this warp's frame state ----
  unsigned char *W = sm + P.off_warp0 + warp * P.warp_bytes;
  float *rec = reinterpret_cast<float *>(W + P.wo_rec);        // by label: sgn*min1; + S2OFF: sgn*min2
  float *ys = reinterpret_cast<float *>(W + P.wo_ys);           // [nslot] signed y per slot (-0 -> +0)
  uint8_t *am = W + P.wo_am;                                    // [nslot] argmin bits per slot
  uint32_t *sb = reinterpret_cast<uint32_t *>(W + P.wo_sb);     // syndrome bits
  uint32_t *zw = reinterpret_cast<uint32_t *>(W + P.wo_zw);     // hard decisions by column
  int *bflip = reinterpret_cast<int *>(W + P.wo_bf);            // per block: flipped column or -1
  float *ek = reinterpret_cast<float *>(W + P.wo_ek);           // [nslot] float32 rounding of the slot's exact metric
  uint16_t *tl = reinterpret_cast<uint16_t *>(W + P.wo_tl);     // labels of the checks this iteration's flips toggle
  const int zwords = (N + 31) >> 5;
  const bool imw = P.wmode == FWBF_WEIGHTS_IMWBF;
  const double alpha = P.alpha;
  if (lane == 0) { // the two constant records after the M check records
    float *rec2 = rec + (P.s2off >> 2);
    rec[M] = rec2[M] = -INFINITY;
    rec[M + 1] = rec2[M + 1] = 0.0f;
  }
  __syncthreads();
  const uint32_t recb = (uint32_t)__cvta_generic_to_shared(rec);
  float *rec2 = rec + (P.s2off >> 2);
  const int s2sh = P.s2sh; // S2OFF = 1 << s2sh

  long long c_frames = 0, c_biterr = 0, c_worderr = 0, c_iters = 0, c_flips = 0, c_stalls = 0, c_conv = 0,
            c_edges = 0;

  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(P.work_counter, 1u);
    t = __shfl_sync(XFULL, t, 0);
    const long long f = (long long)t; // unsigned tickets: see decode_kernel
    if (f >= P.batch) break;

    // ---- init: y -> signed y per slot, hard decisions by column ----
    for (int i = lane; i < (nslot >> 2); i += 32) reinterpret_cast<uint32_t *>(am)[i] = 0u;
    const float *yr = P.y + f * P.ld;
    bool nonfin = false;
    if (P.y_vec4) {
      for (int i = lane; i < zwords; i += 32) zw[i] = 0u;
      __syncwarp();
      for (int n0 = 4 * lane; n0 < N; n0 += 128) {
        const float4 v4 = __ldg(reinterpret_cast<const float4 *>(yr + n0));
        const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
        uint32_t nib = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int n = n0 + u;
          if (n < N) {
            const float v = vv[u] + 0.0f; // -0.0 -> +0.0: the sign bit is the hard decision
            ys[cpos[n]] = v;
            nib |= (v < 0.0f ? 1u : 0u) << u;
            nonfin |= !isfinite(v);
          }
        }
        if (nib) atomicOr(&zw[n0 >> 5], nib << (n0 & 31));
      }
    } else {
      for (int n0 = 0; n0 < N; n0 += 32) {
        const int n = n0 + lane;
        float v = n < N ? __ldg(yr + n) + 0.0f : 0.0f;
        const uint32_t b = __ballot_sync(XFULL, n < N && v < 0.0f);
        if (lane == 0) zw[n0 >> 5] = b;
        if (n < N) {
          ys[cpos[n]] = v;
          nonfin |= !isfinite(v);
        }
      }
    }
    nonfin = __any_sync(XFULL, nonfin);
    __syncwarp();

    // ---- per-check minima, argmin, parity (ascending columns, strict <),
    // lanes over labels j (check invp[j]) ----
    int swt = 0;
    for (int m0 = 0; m0 < M; m0 += 32) {
      const int j = m0 + lane;
      uint32_t par = 0;
      if (j < M) {
        const int m = __ldg(P.invp + j);
        float min1 = INFINITY, min2 = INFINITY;
        int ae = -1;
        const int e1 = __ldg(rptr + m + 1);
        for (int e = __ldg(rptr + m); e < e1; ++e) {
          const float v = ys[__ldg(rtab + e) & 0xffffu];
          par ^= __float_as_uint(v);
          const float a = fabsf(v);
          const bool lt = a < min1;
          min2 = fminf(min2, fmaxf(min1, a));
          min1 = fminf(min1, a);
          ae = lt ? e : ae;
        }
        par >>= 31;
        const float sg = par ? 1.0f : -1.0f;
        // MWBF (include-self minimum): every edge reads min1
        rec[j] = sg * min1; // float32 minima: exact; converted to fp64 per edge
        rec2[j] = sg * (imw ? min2 : min1);
        if (imw && ae >= 0) { // the argmin column reads min2 at this check's position in its list
          const uint32_t pe = __ldg(rtab + ae);
          const uint32_t pos = pe & 0xffffu;
          atomicOr(reinterpret_cast<uint32_t *>(am) + (pos >> 2), (1u << (pe >> 16)) << (8 * (pos & 3)));
        }
      }
      const uint32_t b = __ballot_sync(XFULL, par != 0);
      if (lane == 0) sb[m0 >> 5] = b;
      swt += __popc(b);
    }
    __syncwarp();

    // the reference's Eq.(1) value of slot pos (fp64, ascending checks)
    auto slot_exact = [&](int pos) -> double {
      const unsigned long long w = tab[pos];
      const uint32_t amk = am[pos];
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < DV; ++q) {
        // record byte offset, + S2OFF (min2) when this check's argmin is the column
        const uint32_t off = ((uint32_t)(w >> (16 * q)) & 0xffffu) | ((amk << (s2sh - q)) & (1u << s2sh));
        float vf;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(vf) : "r"(recb + off));
        const double v = (double)vf;
        // starting at the first term instead of +0.0 differs at most in
        // the sign of a zero sum, which no comparison can see
        acc = q == 0 ? v : __dadd_rn(acc, v);
      }
      return __dsub_rn(acc, __dmul_rn(alpha, (double)fabsf(ys[pos])));
    };
    // one round decided on exact values, as xdecode_kernel does every round:
    // the group's first maximum and its column, in every lane of the group
    auto exact_round = [&](int r, double &best, int &col) {
      best = -xdinf();
      int bc = -1;
      const int pos0 = r * S * 32 + lane;
      for (int c = 0; c < S; ++c) {
        const double e = slot_exact(pos0 + c * 32);
        if (e > best) { best = e; bc = c; }
      }
      const int b = r * (32 >> P.lg_g) + (lane >> P.lg_g);
      const int sub = lane & (G - 1);
      col = bc >= 0 ? b * P.p + sub + G * bc : 0x7fffffff;
      for (int off = G >> 1; off; off >>= 1) {
        const double v2 = __shfl_xor_sync(XFULL, best, off);
        const int c2 = __shfl_xor_sync(XFULL, col, off);
        if (v2 > best || (v2 == best && c2 < col)) { best = v2; col = c2; }
      }
    };
    // ---- every slot's metric once; afterwards only the columns of toggled checks ----
    for (int pos = lane; pos < nslot; pos += 32) ek[pos] = (float)slot_exact(pos) + 0.0f;
    __syncwarp();

    // ---- iterations ----
    int k = 0, conv = 0, stalled = 0;
    long long logpos = 0, flips_total = 0;
    for (;;) {
      if (swt == 0) { conv = 1; break; }
      if (k >= P.kmax) break;
      // Selection on the stored float32 roundings: rounding is monotone, so a
      // block whose largest stored value has one holder and is not 0 has that
      // holder as its exact first maximum, with the exact sign.  Any other
      // round (equal values, a zero, a non-finite frame) is decided on exact
      // values as in xdecode_kernel.
      float lhi = -INFINITY; // this lane's largest block maximum as a leader (stall policy)
      int lcol = 0x7fffffff, lcnt = 0;
      bool lamb = false;
      int nflip = 0;
      for (int r = 0; r < R; ++r) {
        float hi = -INFINITY, lo = -INFINITY;
        int bc = -1;
        const int pos0 = r * S * 32 + lane;
#pragma unroll 4
        for (int c = 0; c < S; ++c) {
          const float e = ek[pos0 + c * 32];
          lo = fmaxf(lo, fminf(hi, e));
          bc = e > hi ? c : bc;
          hi = fmaxf(hi, e);
        }
        const int b = r * (32 >> P.lg_g) + (lane >> P.lg_g);
        const int sub = lane & (G - 1);
        int col = bc >= 0 ? b * P.p + sub + G * bc : 0x7fffffff;
        for (int off = G >> 1; off; off >>= 1) {
          const float h2 = __shfl_xor_sync(XFULL, hi, off);
          const float l2 = __shfl_xor_sync(XFULL, lo, off);
          const int c2 = __shfl_xor_sync(XFULL, col, off);
          lo = fmaxf(fminf(hi, h2), fmaxf(lo, l2));
          if (h2 > hi || (h2 == hi && c2 < col)) { hi = h2; col = c2; }
        }
        const bool leader = sub == 0 && b < P.nb;
        const bool amb = leader && (nonfin || !(hi > lo) || hi == 0.0f);
        bool pos_ = hi > 0.0f;
        if (__any_sync(XFULL, amb)) {
          double best;
          exact_round(r, best, col);
          pos_ = best > 0.0;
        }
        if (leader) {
          if (hi > lhi) { lhi = hi; lcol = col; lcnt = 1; lamb = amb; }
          else if (hi == lhi) { lcnt += 1; lamb = true; }
          bflip[b] = pos_ ? col : -1; // decoders.py:181-183
        }
        nflip += __popc(__ballot_sync(XFULL, leader && pos_));
      }
      __syncwarp(); // every metric read of rec / sb precedes the flips
      int F = nflip;
      if (F == 0) {
        // nothing selected with a nonzero syndrome (decoders.py:214-222)
        stalled = 1;
        if (P.stall == FWBF_STALL_TERMINATE) {
          if (lane == 0 && P.fliplog_counts) P.fliplog_counts[f * P.kmax + k] = 0;
          k += 1;
          break;
        }
        // flip the global first maximum.  The block holding the largest stored
        // value holds it when it is the only such block and was decided on
        // stored values; otherwise every block's exact maximum is compared.
        float gk = lhi;
#pragma unroll
        for (int off = 16; off; off >>= 1) gk = fmaxf(gk, __shfl_xor_sync(XFULL, gk, off));
        const uint32_t hold = __ballot_sync(XFULL, lhi == gk && lcnt > 0);
        int gcol = 0x7fffffff;
        if (hold != 0u && (hold & (hold - 1u)) == 0u && !__any_sync(XFULL, lhi == gk && (lcnt > 1 || lamb))) {
          gcol = __shfl_sync(XFULL, lcol, __ffs(hold) - 1);
        } else {
          double gbest = -xdinf();
          for (int r = 0; r < R; ++r) {
            double best;
            int col;
            exact_round(r, best, col);
            const int b = r * (32 >> P.lg_g) + (lane >> P.lg_g);
            if ((lane & (G - 1)) == 0 && b < P.nb && (best > gbest || (best == gbest && col < gcol))) {
              gbest = best;
              gcol = col;
            }
          }
#pragma unroll
          for (int off = 16; off; off >>= 1) {
            const double v2 = __shfl_xor_sync(XFULL, gbest, off);
            const int c2 = __shfl_xor_sync(XFULL, gcol, off);
            if (v2 > gbest || (v2 == gbest && c2 < gcol)) { gbest = v2; gcol = c2; }
          }
        }
        // every block maximum was <= 0, so every bflip entry is already -1
        if (lane == 0 && gcol < N) bflip[gcol / P.p] = gcol;
        F = 1;
        __syncwarp();
      }
      // apply the flips in block order (= ascending columns); log them
      int dsw = 0, cnt = 0;
      for (int b0 = 0; b0 < P.nb; b0 += 32) {
        const int b = b0 + lane;
        const int c = b < P.nb ? bflip[b] : -1;
        const uint32_t msk = __ballot_sync(XFULL, c >= 0);
        if (c >= 0) {
          if (P.fliplog) P.fliplog[f * P.fliplog_stride + logpos + cnt + __popc(msk & ((1u << lane) - 1u))] = c;
          atomicXor(&zw[c >> 5], 1u << (c & 31));
          const unsigned long long w = tab[cpos[c]];
          const int ent = (cnt + __popc(msk & ((1u << lane) - 1u))) * DV;
#pragma unroll
          for (int q = 0; q < DV; ++q) {
            const uint32_t m = ((uint32_t)(w >> (16 * q)) & 0xffffu) >> 2; // label
            tl[ent + q] = m < (uint32_t)M ? (uint16_t)m : (uint16_t)0xffff;
            if (m < (uint32_t)M) { // not the (0, 0) record of a missing edge
              const uint32_t old = atomicXor(&sb[m >> 5], 1u << (m & 31));
              dsw += ((old >> (m & 31)) & 1u) ? -1 : 1;
              // negate sgn*min1 and sgn*min2 of the toggled check: XOR of the
              // sign bit in each double's high word (32-bit shared atomics are
              // native; 64-bit XOR would be a CAS loop)
              atomicXor(reinterpret_cast<uint32_t *>(rec + m), 0x80000000u);
              atomicXor(reinterpret_cast<uint32_t *>(rec2 + m), 0x80000000u);
            }
          }
        }
        cnt += __popc(msk);
      }
      if (lane == 0 && P.fliplog) P.fliplog_counts[f * P.kmax + k] = F;
      swt += __reduce_add_sync(XFULL, dsw);
      __syncwarp();
      // update: the columns of the toggled checks, from scratch (a check two
      // flips share is listed twice and has its old signs back: its columns
      // are recomputed to the same values)
      {
        const int dsh = P.dcs_sh, nit = (F * DV) << dsh;
        for (int i = lane; i < nit; i += 64) { // two items per lane and step: independent chains
          const uint32_t lab0 = tl[i >> dsh];
          const uint32_t lab1 = i + 32 < nit ? tl[(i + 32) >> dsh] : 0xffffu;
          const uint32_t pos0 = lab0 != 0xffffu ? ctab[(lab0 << dsh) + (i & ((1 << dsh) - 1))] : 0xffffu;
          const uint32_t pos1 = lab1 != 0xffffu ? ctab[(lab1 << dsh) + ((i + 32) & ((1 << dsh) - 1))] : 0xffffu;
          const double e0 = pos0 != 0xffffu ? slot_exact((int)pos0) : 0.0;
          const double e1 = pos1 != 0xffffu ? slot_exact((int)pos1) : 0.0;
          if (pos0 != 0xffffu) ek[pos0] = (float)e0 + 0.0f;
          if (pos1 != 0xffffu) ek[pos1] = (float)e1 + 0.0f;
        }
      }
      __syncwarp();
      logpos += F;
      flips_total += F;
      k += 1;
    }

    // ---- outputs ----
    int be = 0;
    for (int i = lane; i < zwords; i += 32) {
      const uint32_t z = zw[i];
      if (P.z_bits) P.z_bits[f * P.z_ld + i] = z;
      const uint32_t cw = P.codeword_bits ? __ldg(P.codeword_bits + i) : 0u;
      be += __popc(z ^ cw);
    }
    be = __reduce_add_sync(XFULL, be);
    if (lane == 0) {
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
    __syncwarp();
  }
  if (lane == 0 && P.counters && c_frames) {
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

template __global__ void xdecode_kernel<2>(const __grid_constant__ XParams);
template __global__ void xdecode_kernel<3>(const __grid_constant__ XParams);
template __global__ void xdecode_kernel<4>(const __grid_constant__ XParams);
template __global__ void xinc_kernel<2>(const __grid_constant__ XParams);
template __global__ void xinc_kernel<3>(const __grid_constant__ XParams);
template __global__ void xinc_kernel<4>(const __grid_constant__ XParams);

} // namespace fwbf
