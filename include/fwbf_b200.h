/*
 * fwbf_b200.h -- C ABI of the B200 batched weighted-bit-flipping LDPC decoder.
 *
 * Drop-in boundary for the reference's decode path (/root/reference/pkg/src/fwbf):
 *
 *   fwbf_code_create    replaces ParityCheckMatrix as the decoder's view of H
 *                       (matrix.py:22-58); the handle owns device copies.
 *   fwbf_decode_f32/64  replaces the per-frame loop decode_{fwbf,imwbf,mlp_wbf}
 *                       (decoders.py:189-259), batched over B frames; y is the
 *                       channel output the reference casts to float64 (:191).
 *   fwbf_decode_awgn    replaces harness._run_batch (harness.py:98-115): noise is
 *                       generated on the device from (seed, global frame index).
 *   fwbf_decode_host_f32  the same batch call on HOST buffers (pipelined copies).
 *   fwbf_last_error     text of the last failure (the reference raises ValueError).
 *
 * Conventions: plain C types only; every buffer argument of fwbf_decode_* is
 * caller-owned DEVICE memory unless the function name says host; optional
 * outputs may be NULL.  Calls are ordered on the given cudaStream_t (passed
 * as void*; NULL = legacy default stream).  Return 0 on success, a negative
 * FWBF_E* code otherwise (see fwbf_last_error()).  The library never falls
 * back to the CPU: without a usable CUDA device every decode call fails.
 */
#ifndef FWBF_B200_H
#define FWBF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FWBF_ABI_VERSION 1

#define FWBF_OK 0
#define FWBF_EINVAL (-1)      /* ValueError in the reference (bad config / shape) */
#define FWBF_ECUDA (-2)       /* CUDA runtime failure (no device, launch error)   */
#define FWBF_EUNSUPPORTED (-3)/* valid request this build cannot serve           */

/* algorithm ids: the reference's _SELECTORS keys (decoders.py:186) */
#define FWBF_ALG_FWBF 0
#define FWBF_ALG_IMWBF 1
#define FWBF_ALG_MLP 2

/* weight modes: Eq.(1) exclude-self weights (decoders.py:80-84) or the
 * include-self minimum of classic WBF/MWBF (alpha = 0 gives WBF) */
#define FWBF_WEIGHTS_IMWBF 0
#define FWBF_WEIGHTS_MWBF 1

/* stall policies (decoders.py:29) */
#define FWBF_STALL_FLIP_GLOBAL_MAX 0
#define FWBF_STALL_TERMINATE 1

/* per-frame flag bits written to fwbf_outputs.flags */
#define FWBF_FLAG_CONVERGED 1
#define FWBF_FLAG_STALLED 2
#define FWBF_FLAG_ORDERED 4   /* decoded on the ordered (non-guarded) metric path */
#define FWBF_FLAG_NONFINITE 8 /* y held NaN/inf; result follows IEEE comparisons */
#define FWBF_FLAG_SPLIT32 16  /* decoded on the split-fp32 guarded metric path */

/* counters vector layout (int64) */
enum {
  FWBF_CNT_FRAMES = 0,
  FWBF_CNT_BIT_ERRORS,
  FWBF_CNT_WORD_ERRORS,
  FWBF_CNT_ITER_SUM,
  FWBF_CNT_FLIP_SUM,
  FWBF_CNT_STALLS,
  FWBF_CNT_CONVERGED,
  FWBF_CNT_ORDERED_FRAMES,
  FWBF_CNT_EDGE_VISITS,     /* metric terms accumulated (sum over frames of E*iters) */
  FWBF_NCOUNTERS
};

typedef struct fwbf_code fwbf_code; /* opaque device handle */

/* H as the reference stores it: CSR rows with sorted column indices
 * (matrix.py:22-58).  If circulant != 0, H is the n x n circulant whose row m
 * holds columns (offsets[j] + m) mod n (eg.py:46) and the CSR is optional. */
typedef struct {
  int32_t n_cols;
  int32_t n_rows;
  const int32_t *row_ptr; /* [n_rows + 1], host memory */
  const int32_t *row_idx; /* [row_ptr[n_rows]], sorted per row, host memory */
  int32_t circulant;
  int32_t n_offsets;
  const int32_t *offsets; /* sorted first-row columns, host memory */
} fwbf_code_desc;

/* DecoderConfig (decoders.py:32-61) plus the algorithm selector. */
typedef struct {
  int32_t algorithm;     /* FWBF_ALG_* */
  int32_t weight_mode;   /* FWBF_WEIGHTS_* */
  double alpha;          /* >= 0 */
  int32_t k_max;         /* >= 1 */
  int32_t lam;           /* >= 1, <= n (MLP) */
  int32_t block_len_p;   /* >= 1 (FWBF) */
  int32_t stall;         /* FWBF_STALL_* */
  int32_t mlp_threshold; /* 0/1 */
  int32_t force_ordered; /* testing, bit flags: 1 = ordered path only, 2 = no split-fp32 path,
                            4 = no filtered metric (exact split gather every iteration) */
} fwbf_params;

/* Output buffers (device memory, caller-owned, all optional). */
typedef struct {
  uint32_t *z_bits;        /* [B][z_ld] words; bit n of frame f = word n/32, bit n%32 */
  int64_t z_ld;            /* words per frame row, >= ceil(n/32) */
  int32_t *iterations;     /* [B] */
  uint8_t *flags;          /* [B] FWBF_FLAG_* */
  int32_t *flips_total;    /* [B] */
  int32_t *bit_errors;     /* [B] popcount(z xor codeword) */
  int32_t *fliplog;        /* [B][fliplog_stride] flipped indices, iteration-major */
  int32_t *fliplog_counts; /* [B][k_max] flips per iteration */
  int64_t fliplog_stride;  /* >= k_max * max flips per iteration */
  int64_t *counters;       /* [FWBF_NCOUNTERS], accumulated (not cleared) */
  int64_t *iter_hist;      /* [k_max + 1], accumulated */
  int32_t *batch_word_err; /* [ceil(B / batch_frames)], accumulated */
  int32_t batch_frames;    /* harness BATCH_FRAMES (harness.py:24), e.g. 128 */
  const uint32_t *codeword_bits; /* [ceil(n/32)] transmitted word; NULL = all-zero */
  void *y_out;             /* fwbf_decode_awgn only: [B][y_out_ld] generated channel
                              values (double for NUMPY_F64, float for NUMPY_F32) */
  int64_t y_out_ld;
} fwbf_outputs;

int fwbf_abi_version(void);
const char *fwbf_last_error(void);
int fwbf_device_count(void);

int fwbf_code_create(const fwbf_code_desc *desc, int device, fwbf_code **out);
int fwbf_code_destroy(fwbf_code *code);
int fwbf_code_info(const fwbf_code *code, int32_t *n_cols, int32_t *n_rows,
                   int32_t *n_edges, int32_t *circulant);

/* Max flips one iteration can produce (sizes fliplog rows). */
int64_t fwbf_max_flips_per_iter(const fwbf_code *code, const fwbf_params *params);

/* Decode B frames of channel output y[f * ld + n] (device memory). */
int fwbf_decode_f32(fwbf_code *code, const fwbf_params *params, const float *y,
                    int64_t batch, int64_t ld, const fwbf_outputs *out, void *stream);
int fwbf_decode_f64(fwbf_code *code, const fwbf_params *params, const double *y,
                    int64_t batch, int64_t ld, const fwbf_outputs *out, void *stream);

/* Stage view (tests, diagnostics): the Eq.(1) metric vector each frame's
 * decode would compute in its first iteration -- all_metrics on the initial
 * hard decisions (decoders.py:148-153 with the weights of :80-103) -- written
 * to metric[f * metric_ld + n] (device memory, float64).  flags (nullable)
 * receive the per-frame metric path (FWBF_FLAG_ORDERED / FWBF_FLAG_SPLIT32).
 * Same params, validation and path choice as fwbf_decode_*; the metric is
 * produced even when the initial syndrome is already zero. */
int fwbf_metric_f32(fwbf_code *code, const fwbf_params *params, const float *y, int64_t batch,
                    int64_t ld, double *metric, int64_t metric_ld, uint8_t *flags, void *stream);
int fwbf_metric_f64(fwbf_code *code, const fwbf_params *params, const double *y, int64_t batch,
                    int64_t ld, double *metric, int64_t metric_ld, uint8_t *flags, void *stream);

/* Diagnostic: how many FWBF decisions of the filtered metric (approximate fp32
 * gather on split-path frames) this code's launches had
 * to resolve with exact column sums: out[0] block argmaxes, out[1] stall
 * global argmaxes.  Synchronous; reset != 0 zeroes the counters. */
int fwbf_filter_stats(fwbf_code *code, int64_t *out, int32_t reset);

/* Diagnostic: the decode kernel(s) the calling thread's last decode launched,
 * e.g. "cdecode+decode_kernel" (filtered circulant kernel, then the exact
 * kernel over the frames it deferred), "decode_kernel", "xinc" / "xdecode"
 * (incremental / full-pass one-frame-per-warp kernel), "qinc"
 * (incremental quasi-cyclic kernel), "qdecode" (full-pass quasi-cyclic kernel). */
const char *fwbf_last_kernel(void);

/* Noise modes for fwbf_decode_awgn. */
#define FWBF_NOISE_NUMPY_F64 0 /* the reference stream: numpy Philox(key=seed,
                                  counter=frame<<128) + Generator.standard_normal,
                                  y = s + sigma*g in float64 (channel.py:29-50) */
#define FWBF_NOISE_NUMPY_F32 1 /* same stream, y rounded to float32 */

/* Decode frames [first_frame, first_frame + count) of the reference channel:
 * y = (1 - 2c) + sigma * g with g drawn on the device; c = out->codeword_bits
 * (NULL = all-zero).  Equivalent to harness._run_batch over that range. */
int fwbf_decode_awgn(fwbf_code *code, const fwbf_params *params, uint64_t seed,
                     int64_t first_frame, int64_t count, double sigma,
                     int32_t noise_mode, const fwbf_outputs *out, void *stream);

/* End-to-end call on HOST buffers: y_host [batch][ld] floats; outputs are host
 * arrays (any may be NULL; counters accumulated).  Copies are pipelined in
 * chunks of chunk_frames (<= 0: about 64 MB of y per chunk) against decoding
 * on internal streams -- H2D, two alternating decode streams so that a
 * chunk's last frames overlap the next chunk's first, D2H; four device chunk
 * buffers; pinned host memory gives full overlap.  Synchronous: returns when
 * results are in host memory. */
int fwbf_decode_host_f32(fwbf_code *code, const fwbf_params *params, const float *y_host,
                         int64_t batch, int64_t ld, uint32_t *z_bits_host, int64_t z_ld,
                         int32_t *iterations_host, uint8_t *flags_host,
                         int64_t *counters_host, int64_t chunk_frames);

/* ---- Stage views (fwbf_stage.cu): the reference's stage functions one at a
 * time, batched over B frames, float64 like the reference, device memory.
 * The decode kernels fuse all of them; these serve the stage-level API and
 * its parity tests. ---- */

/* hard_decision (decoders.py:106-108): z[i] = y[i] < 0; dtype 4 = float32,
 * 8 = float64; count elements. */
int fwbf_stage_hard_decision(int32_t dtype, const void *y, int64_t count, uint8_t *z, void *stream);

/* ParityCheckMatrix.syndrome (matrix.py:72-79): z [B][n] uint8 -> s [B][m]. */
int fwbf_stage_syndrome(fwbf_code *code, const uint8_t *z, int64_t batch, uint8_t *syndrome, void *stream);

/* compute_weights + WeightTable.edge_weights (decoders.py:80-103): per check
 * min1, min2 (float64) and argmin_col (int64, first occurrence), [B][m];
 * edge_w [B][n_edges] in row-major edge order (nullable).  Fails with
 * FWBF_EINVAL when a check has fewer than 2 bits, like the reference. */
int fwbf_stage_weights(fwbf_code *code, const double *y, int64_t batch, int64_t ld, double *min1,
                       double *min2, int64_t *argmin_col, double *edge_w, void *stream);

/* WeightTable.edge_weights (decoders.py:80-84) of a given table [B][m] ->
 * edge_w [B][n_edges] in row-major edge order. */
int fwbf_stage_edge_weights(fwbf_code *code, const double *min1, const double *min2,
                            const int64_t *argmin_col, int64_t batch, double *edge_w, void *stream);

/* all_metrics (decoders.py:148-153): syndrome [B][m] uint8, edge_w [B][n_edges],
 * abs_y [B][n] -> out [B][n] = fl(sum in ascending check order) - fl(alpha|y|). */
int fwbf_stage_all_metrics(fwbf_code *code, const uint8_t *syndrome, const double *edge_w,
                           const double *abs_y, double alpha, int64_t batch, double *out, void *stream);

/* block_argmax (decoders.py:156-167): values [B][ld], first maximum of each
 * p-block (tail padded with -inf) -> out [B][ceil(n/p)] int64. */
int fwbf_stage_block_argmax(const double *values, int64_t batch, int64_t n, int64_t ld, int32_t p,
                            int64_t *out, void *stream);

/* bit_metric (decoders.py:138-145) for columns cols[0..k) of one state. */
int fwbf_stage_bit_metric(fwbf_code *code, const int32_t *cols, int32_t k, const uint8_t *syndrome,
                          const double *min1, const double *min2, const int64_t *argmin_col,
                          const double *y, double alpha, double *out, void *stream);

/* The reference channel without a decode (frame_rng + transmit,
 * channel.py:29-82): y[f][n] for frames first..first+count-1, noise_mode as
 * for fwbf_decode_awgn (y is double* for NUMPY_F64, float* for NUMPY_F32). */
int fwbf_channel_awgn(fwbf_code *code, uint64_t seed, int64_t first_frame, int64_t count, double sigma,
                      const uint32_t *codeword_bits, int32_t noise_mode, void *y, int64_t ld, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FWBF_B200_H */
