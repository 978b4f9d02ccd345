/*
 * wbf_oracle.c -- CPU ORACLE (C restatement) of the reference decode loop.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ (ctypes) as a fast, independent
 * checker for large batches; never linked into the product library.
 *
 * Follows /root/reference/pkg/src/fwbf/decoders.py:
 *   compute_weights  :87-103  per-check min1 / argmin (first = lowest column) / min2
 *   edge_weights     :80-84   w = min2 at the argmin column, else min1 ("mwbf": min1)
 *   all_metrics      :148-153 E_n = fl(sum over checks ascending of +-w, from 0.0) - fl(alpha|y|)
 *   block_argmax     :156-167 first maximum per p-block, -inf padding
 *   _select_*        :170-183
 *   _decode          :189-229 converged? -> k_max? -> metric -> select -> stall -> flip
 * and matrix.py:72-79 (syndrome).  Pinned against the reference's golden
 * fixtures by tests/test_oracle_golden.py::test_c_oracle_matches_fixtures.
 *
 * Build: make -C oracle   (gcc -O2 -fno-fast-math -ffp-contract=off)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int n, m;
  const int *row_ptr, *row_idx; /* CSR, sorted columns */
  const int *col_ptr, *col_idx; /* CSC, ascending checks */
} orc_code;

/* algorithm: 0 fwbf, 1 imwbf, 2 mlp; weight_mode 0 imwbf, 1 mwbf; stall 0 flip-max, 1 terminate */
typedef struct {
  int algorithm, weight_mode;
  double alpha;
  int k_max, lam, p, stall, mlp_threshold;
} orc_params;

static int argmax_first(const double *e, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (e[i] > e[best]) best = i;
  return best;
}

/* decode one frame; returns iterations; z_out[n] bits; flags bit0 converged, bit1 stalled;
 * log (nullable): flips appended, log_counts[k] = flips of iteration k. */
int orc_decode(const orc_code *h, const orc_params *prm, const double *y, uint8_t *z_out, int *flags,
               int *flips_total, int *log, int *log_counts) {
  const int n = h->n, m = h->m;
  double *ay = malloc(sizeof(double) * n);
  double *min1 = malloc(sizeof(double) * m), *min2 = malloc(sizeof(double) * m);
  int *arg = malloc(sizeof(int) * m);
  uint8_t *synd = malloc(m), *z = z_out;
  double *e = malloc(sizeof(double) * n), *acc = malloc(sizeof(double) * n);
  int *flips = malloc(sizeof(int) * (n + 1));
  char *sel = malloc(n);
  for (int i = 0; i < n; ++i) {
    ay[i] = fabs(y[i]);
    z[i] = y[i] < 0.0;
  }
  for (int r = 0; r < m; ++r) {
    double a1 = INFINITY, a2 = INFINITY;
    int ai = -1;
    int par = 0;
    for (int e2 = h->row_ptr[r]; e2 < h->row_ptr[r + 1]; ++e2) {
      const int c = h->row_idx[e2];
      par ^= z[c];
      if (ay[c] < a1) { a2 = a1; a1 = ay[c]; ai = c; } /* ascending columns: strict < keeps the first */
      else if (ay[c] < a2) a2 = ay[c];
    }
    min1[r] = a1; min2[r] = a2; arg[r] = ai;
    synd[r] = (uint8_t)par;
  }
  int k = 0, stalled = 0, total = 0, logpos = 0, conv = 0;
  for (;;) {
    int any = 0;
    for (int r = 0; r < m; ++r) any |= synd[r];
    if (!any) { conv = 1; break; }
    if (k >= prm->k_max) break;
    for (int c = 0; c < n; ++c) {
      double s = 0.0;
      for (int e2 = h->col_ptr[c]; e2 < h->col_ptr[c + 1]; ++e2) {
        const int r = h->col_idx[e2];
        const double w = (prm->weight_mode == 0 && arg[r] == c) ? min2[r] : min1[r];
        s = s + (synd[r] ? w : -w);
      }
      acc[c] = s;
      e[c] = s - prm->alpha * ay[c];
    }
    int F = 0;
    if (prm->algorithm == 1) {
      flips[F++] = argmax_first(e, n);
    } else if (prm->algorithm == 2) {
      memset(sel, 0, n);
      for (int t = 0; t < prm->lam; ++t) { /* stable argsort of -e: largest first, lowest index on ties */
        int best = -1;
        for (int i = 0; i < n; ++i)
          if (!sel[i] && (best < 0 || e[i] > e[best])) best = i;
        sel[best] = (!prm->mlp_threshold || e[best] > 0.0) ? 1 : 2;
      }
      for (int i = 0; i < n; ++i)
        if (sel[i] == 1) flips[F++] = i;
    } else {
      const int p = prm->p;
      for (int b = 0; b * p < n; ++b) {
        int best = b * p;
        for (int i = b * p + 1; i < (b + 1) * p && i < n; ++i)
          if (e[i] > e[best]) best = i;
        if (e[best] > 0.0) flips[F++] = best;
      }
    }
    if (F == 0) {
      stalled = 1;
      if (prm->stall == 1) {
        if (log_counts) log_counts[k] = 0;
        k += 1;
        break;
      }
      flips[F++] = argmax_first(e, n);
    }
    for (int t = 0; t < F; ++t) {
      const int c = flips[t];
      z[c] ^= 1;
      for (int e2 = h->col_ptr[c]; e2 < h->col_ptr[c + 1]; ++e2) synd[h->col_idx[e2]] ^= 1;
      if (log) log[logpos++] = c;
    }
    if (log_counts) log_counts[k] = F;
    total += F;
    k += 1;
  }
  *flags = conv | (stalled << 1);
  *flips_total = total;
  free(ay); free(min1); free(min2); free(arg); free(synd); free(e); free(acc); free(flips); free(sel);
  return k;
}

/* batch over B frames of float32 or float64 y (is_f64), row stride ld */
void orc_decode_batch(const orc_code *h, const orc_params *prm, const void *y, int is_f64, long long B,
                      long long ld, uint8_t *z, int *iters, int *flags, int *flips_total) {
  double *row = malloc(sizeof(double) * h->n);
  for (long long f = 0; f < B; ++f) {
    for (int i = 0; i < h->n; ++i)
      row[i] = is_f64 ? ((const double *)y)[f * ld + i] : (double)((const float *)y)[f * ld + i];
    iters[f] = orc_decode(h, prm, row, z + f * h->n, &flags[f], &flips_total[f], NULL, NULL);
  }
  free(row);
}
