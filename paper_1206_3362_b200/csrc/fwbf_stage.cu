// fwbf_stage.cu -- the reference decoder's stage functions as batched kernels.
//
// The decode kernel (fwbf_decode.cu) fuses every stage of one iteration; these
// kernels expose the stages one at a time, with the reference's array layouts,
// so callers of the stage-level API (and the parity tests) get the same
// values from the device:
//
//   stage_hard_decision  decoders.py:106-108  z_n = (y_n < 0)
//   stage_syndrome       matrix.py:72-79      s_m = (sum_{n in N(m)} z_n) & 1
//   stage_weights        decoders.py:87-103   min1 / min2 / argmin_col per check,
//                        decoders.py:80-84    plus the edge weights in edge order
//   stage_all_metrics    decoders.py:148-153  Eq.(1), fp64 adds in ascending check
//                                             order (np.bincount), minus fl(alpha|y|)
//   stage_block_argmax   decoders.py:156-167  first maximum per p-block
//   stage_bit_metric     decoders.py:138-145  scalar Eq.(1), its own term order
//
// One thread per (frame, item).  Float64 throughout, like the reference (it
// casts y to float64 before any arithmetic); the library is compiled with
// -fmad=false, so every product and sum rounds exactly as numpy's do.
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace fwbf {

template <typename T>
__global__ void stage_hard_decision(const T *__restrict__ y, long long count, uint8_t *__restrict__ z) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    z[i] = y[i] < T(0) ? 1 : 0;
}

// z [B][n] (uint8 0/1) -> s [B][m]
__global__ void stage_syndrome(const int *__restrict__ row_ptr, const int *__restrict__ row_idx, int n, int m,
                               const uint8_t *__restrict__ z, long long batch, uint8_t *__restrict__ s) {
  const long long total = batch * m;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / m;
    const int r = (int)(i - f * m);
    const uint8_t *zf = z + f * n;
    long long acc = 0;
    for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) acc += zf[row_idx[e]];
    s[i] = (uint8_t)(acc & 1);
  }
}

// y [B][ld] float64 -> min1, min2 [B][m] float64, argmin [B][m] int64,
// edge_w [B][E] (nullable): columns are scanned in ascending order, strict <
// keeps the first occurrence (numpy argmin), min2 is the minimum over the
// other columns of the check (decoders.py:96-102).
__global__ void stage_weights(const int *__restrict__ row_ptr, const int *__restrict__ row_idx, int m,
                              long long n_edges, const double *__restrict__ y, long long batch, long long ld,
                              double *__restrict__ min1, double *__restrict__ min2,
                              long long *__restrict__ argmin, double *__restrict__ edge_w) {
  const long long total = batch * m;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / m;
    const int r = (int)(i - f * m);
    const double *yf = y + f * ld;
    const int e0 = row_ptr[r], e1 = row_ptr[r + 1];
    double a1 = INFINITY;
    int pos = e0;
    for (int e = e0; e < e1; ++e) {
      const double a = fabs(yf[row_idx[e]]);
      if (a < a1) { a1 = a; pos = e; }
    }
    double a2 = INFINITY;
    for (int e = e0; e < e1; ++e)
      if (e != pos) a2 = fmin(a2, fabs(yf[row_idx[e]]));
    min1[i] = a1;
    min2[i] = a2;
    argmin[i] = row_idx[pos];
    if (edge_w) {
      double *w = edge_w + f * n_edges;
      for (int e = e0; e < e1; ++e) w[e] = (e == pos) ? a2 : a1;
    }
  }
}

// WeightTable.edge_weights (decoders.py:80-84) from a given table:
// w_e = min2[m] if edge e's column is argmin_col[m] else min1[m], row-major.
__global__ void stage_edge_weights(const int *__restrict__ row_ptr, const int *__restrict__ row_idx, int m,
                                   long long n_edges, const double *__restrict__ min1,
                                   const double *__restrict__ min2, const long long *__restrict__ argmin,
                                   long long batch, double *__restrict__ edge_w) {
  const long long total = batch * m;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / m;
    const int r = (int)(i - f * m);
    double *w = edge_w + f * n_edges;
    for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) w[e] = (row_idx[e] == argmin[i]) ? min2[i] : min1[i];
  }
}

// Eq.(1): acc = fl(sum over the column's edges in ascending check order of
// (2 s_m - 1) * w_e), starting from 0.0, then acc - fl(alpha |y_n|).
__global__ void stage_all_metrics(const int *__restrict__ col_ptr, const int *__restrict__ col_idx,
                                  const int *__restrict__ col_eid, int n, int m, long long n_edges,
                                  const uint8_t *__restrict__ syn, const double *__restrict__ edge_w,
                                  const double *__restrict__ abs_y, double alpha, long long batch,
                                  double *__restrict__ out) {
  const long long total = batch * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / n;
    const int c = (int)(i - f * n);
    const uint8_t *sf = syn + f * m;
    const double *wf = edge_w + f * n_edges;
    double acc = 0.0;
    for (int k = col_ptr[c]; k < col_ptr[c + 1]; ++k) {
      const double sg = __dsub_rn(__dmul_rn(2.0, (double)sf[col_idx[k]]), 1.0);
      acc = __dadd_rn(acc, __dmul_rn(sg, wf[col_eid[k]]));
    }
    out[i] = __dsub_rn(acc, __dmul_rn(alpha, abs_y[i]));
  }
}

// values [B][ld] -> out [B][nb]: the first maximum of each p-block; the tail
// block is padded with -inf (never selected).  numpy's argmax treats NaN as
// the maximum and returns the first one.
__global__ void stage_block_argmax(const double *__restrict__ v, long long batch, int n, long long ld, int p,
                                   int nb, long long *__restrict__ out) {
  const long long total = batch * nb;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long f = i / nb;
    const int b = (int)(i - f * nb);
    const double *vf = v + f * ld;
    const long long base = (long long)b * p;
    const long long lim = min((long long)p, (long long)n - base);
    double best = vf[base];
    long long bi = base;
    for (long long o = 1; o < lim && !isnan(best); ++o) {
      const double x = vf[base + o];
      if (isnan(x) || x > best) { best = x; bi = base + o; }
    }
    out[i] = bi;
  }
}

// bit_metric for columns cols[0..k): total = -alpha |y_n|, then + w or - w per
// check of the column in ascending order (decoders.py:138-145).
__global__ void stage_bit_metric(const int *__restrict__ col_ptr, const int *__restrict__ col_idx,
                                 const int *__restrict__ cols, int k, const uint8_t *__restrict__ syn,
                                 const double *__restrict__ min1, const double *__restrict__ min2,
                                 const long long *__restrict__ argmin, const double *__restrict__ y,
                                 double alpha, double *__restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  const int c = cols[i];
  double total = __dmul_rn(-alpha, fabs(y[c]));
  for (int e = col_ptr[c]; e < col_ptr[c + 1]; ++e) {
    const int r = col_idx[e];
    const double w = (argmin[r] == c) ? min2[r] : min1[r];
    total = __dadd_rn(total, syn[r] ? w : -w);
  }
  out[i] = total;
}

template __global__ void stage_hard_decision<float>(const float *, long long, uint8_t *);
template __global__ void stage_hard_decision<double>(const double *, long long, uint8_t *);

} // namespace fwbf
