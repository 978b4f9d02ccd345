// fwbf_api.cu -- C ABI: code handles, validation, launch planning, host pipeline.
//
// Validation mirrors the ValueErrors of the reference
// (/root/reference/pkg/src/fwbf/decoders.py:51-61, :89-93, :192-193, :245-246,
// :257-258); the message text is available from fwbf_last_error().

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <list>
#include <mutex>
#include <string>
#include <vector>

#include "fwbf_b200.h"
#include "fwbf_internal.h"

namespace fwbf {
template <typename YT, bool CIRC, int KC, int TB, int WT, int MODE = 0>
__global__ void decode_kernel(const __grid_constant__ KParams P);
template <typename YT>
__global__ void noise_kernel(unsigned long long seed, long long first, long long count, double sigma,
                             const uint32_t *codeword, YT *y, long long ld, int n, int pm);
template <int DV> __global__ void xdecode_kernel(const __grid_constant__ XParams P);
template <int DV> __global__ void xinc_kernel(const __grid_constant__ XParams P);
template <int KC, int TB, int WT, int NN, int PB, bool Q16> __global__ void cdecode_kernel(const __grid_constant__ KParams P);
template <int TPC> __global__ void qdecode_kernel(const __grid_constant__ QParams P);
template <int TPC, bool ALLP> __global__ void qinc_kernel(const __grid_constant__ QParams P);
template <typename T> __global__ void stage_hard_decision(const T *, long long, uint8_t *);
__global__ void stage_syndrome(const int *, const int *, int, int, const uint8_t *, long long, uint8_t *);
__global__ void stage_weights(const int *, const int *, int, long long, const double *, long long, long long,
                              double *, double *, long long *, double *);
__global__ void stage_edge_weights(const int *, const int *, int, long long, const double *, const double *,
                                   const long long *, long long, double *);
__global__ void stage_all_metrics(const int *, const int *, const int *, int, int, long long, const uint8_t *,
                                  const double *, const double *, double, long long, double *);
__global__ void stage_block_argmax(const double *, long long, int, long long, int, int, long long *);
__global__ void stage_bit_metric(const int *, const int *, const int *, int, const uint8_t *, const double *,
                                 const double *, const long long *, const double *, double, double *);
template <typename YT>
__global__ void noise_kernel_warp(unsigned long long seed, long long first, long long count, double sigma,
                                  const uint32_t *codeword, YT *y, long long ld, int n);
}

using fwbf::KParams;

static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) return fail(FWBF_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

// Every C entry point that selects its handle's device restores the caller's
// current device on every exit path (the caller's CUDA context is not ours).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// One-frame-per-warp explicit-code plan (fwbf_explicit.cu), built per (code, p).
struct XPlan {
  int p = 0, nb = 0, lg_g = 0, rounds = 0, slots = 0, dv = 0;
  const void *kern = nullptr;
  unsigned long long *d_tab = nullptr;
  uint32_t *d_rtab = nullptr;
  uint16_t *d_cpos = nullptr;
  int *d_invp = nullptr;
  int s2sh = 0;
  int tables_bytes = 0, warp_bytes = 0;
  int wo_rec = 0, wo_ys = 0, wo_am = 0, wo_sb = 0, wo_zw = 0, wo_bf = 0;
  int off_tab = 0, off_cpos = 0;
  int wpc = 0, per_sm = 0, smem = 0; // warps per CTA, CTAs per SM, dynamic smem bytes
  bool ok = false;
  // incremental variant (xinc_kernel): the base layout plus the check -> slots table after the CTA tables
  // and the stored metrics + toggled-check list after each warp's region
  bool inc_ok = false;
  const void *inc_kern = nullptr;
  uint16_t *d_ctab = nullptr;
  int dcs_sh = 0, off_ctab = 0, inc_tables_bytes = 0, inc_warp_bytes = 0, wo_ek = 0, wo_tl = 0;
  int inc_wpc = 0, inc_per_sm = 0, inc_smem = 0;
};

struct fwbf_code {
  int device = 0;
  int n = 0, m = 0;
  long long n_edges = 0;
  int circ = 0, w = 0;
  int dv_max = 0, dc_max = 0, min_row_w = 0;
  int off[fwbf::kMaxCircWeight] = {0};
  int dneg[fwbf::kMaxCircWeight] = {0};
  unsigned char jii[fwbf::kMaxCircWeight] = {0};
  int *d_row_ptr = nullptr, *d_row_idx = nullptr, *d_col_ptr = nullptr, *d_col_idx = nullptr;
  int *d_col_eid = nullptr; // row-major edge index per CSC entry (stage kernels)
  uint8_t *d_i0tab = nullptr;
  uint8_t *d_jwtab = nullptr;
  int16_t *d_offpos = nullptr;
  unsigned int *d_work = nullptr; // ring of per-launch work counters
  unsigned long long *d_fstats = nullptr; // [2] filtered-metric decisions resolved exactly (diagnostic)
  std::atomic<unsigned> work_slot{0};
  int qc_z = 0, qc_jb = 0, qc_kb = 0;
  short qc_shift[fwbf::kMaxQcBlocks];
  int sm_count = 0;
  int smem_optin = 0;
  // host pipeline scratch
  std::mutex pipe_mu;
  // host pipeline (fwbf_decode_host_f32): H2D copies, two alternating decode streams, the
  // deferred-frame launches (high priority), D2H copies; four chunk buffers
  cudaStream_t pipe_s[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t pipe_ev[4][4] = {}; // [h2d done, main kernel done, decode done, d2h done][buffer]
  void *pipe_buf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t pipe_bytes = 0;
  int64_t *pipe_counters = nullptr;
  void *noise_buf = nullptr;
  size_t noise_bytes = 0;
  cudaEvent_t noise_evt = nullptr; // last use of noise_buf (device-side ordering across streams)
  cudaStream_t noise_side = nullptr; // decode_awgn: odd chunks (noise + decode) on a second stream
  cudaEvent_t noise_fork = nullptr, noise_join = nullptr;
  cudaStream_t noise_def = nullptr;           // decode_awgn: the chunks' deferred-frame launches (high priority)
  cudaEvent_t noise_cev[3] = {}, noise_dev[3] = {}, noise_join2 = nullptr; // per scratch buffer: main kernel done, chunk done
  // explicit-code warp-per-frame plans, one per block length p
  std::mutex xplan_mu;
  std::list<XPlan> xplans; // stable addresses: launches hold a plan pointer outside the lock
  std::vector<int> h_row_ptr, h_row_idx, h_col_ptr, h_col_idx; // host copies for plan building
};

// Each decode launch takes the next of kWorkRing frame-queue counters of its
// code handle (reset on the launch's stream), so up to kWorkRing launches per
// handle may be in flight concurrently on different streams.
static constexpr int kWorkRing = 1024;

extern "C" int fwbf_abi_version(void) { return FWBF_ABI_VERSION; }
extern "C" const char *fwbf_last_error(void) { return g_err.c_str(); }

static thread_local const char *g_last_kernel = "";
// the filtered circulant kernel gathers 16-bit quantised minima (Q16) unless
// FWBF_Q16=0 asks for the float32 gather (A/B timing, parity tests of both)
static bool q16_enabled() {
  const char *e = getenv("FWBF_Q16");
  return e ? atoi(e) != 0 : true;
}
extern "C" const char *fwbf_last_kernel(void) { return g_last_kernel; }

extern "C" int fwbf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}

template <typename T> static int upload(T **dst, const std::vector<T> &v) {
  CUDA_TRY(cudaMalloc((void **)dst, std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!v.empty()) CUDA_TRY(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return FWBF_OK;
}

extern "C" int fwbf_code_create(const fwbf_code_desc *desc, int device, fwbf_code **out) {
  if (!desc || !out) return fail(FWBF_EINVAL, "null argument");
  *out = nullptr;
  const int n = desc->n_cols, m = desc->n_rows;
  if (n < 1) return fail(FWBF_EINVAL, "n_cols must be positive");
  if (m < 0) return fail(FWBF_EINVAL, "n_rows must be nonnegative");
  // Build the row lists (from CSR, or from the circulant offsets).
  std::vector<int> row_ptr(m + 1, 0), row_idx;
  if (desc->circulant) {
    if (n != m) return fail(FWBF_EINVAL, "a circulant code must be square");
    const int w = desc->n_offsets;
    if (w < 1 || w > fwbf::kMaxCircWeight || !desc->offsets)
      return fail(FWBF_EINVAL, "circulant weight must be in [1, %d]", fwbf::kMaxCircWeight);
    for (int j = 0; j < w; ++j) {
      if (desc->offsets[j] < 0 || desc->offsets[j] >= n) return fail(FWBF_EINVAL, "offset out of range");
      if (j && desc->offsets[j] <= desc->offsets[j - 1]) return fail(FWBF_EINVAL, "offsets must be strictly ascending");
    }
    row_idx.reserve((size_t)n * w);
    std::vector<int> r(w);
    for (int i = 0; i < m; ++i) {
      for (int j = 0; j < w; ++j) r[j] = (desc->offsets[j] + i) % n;
      std::sort(r.begin(), r.end());
      row_idx.insert(row_idx.end(), r.begin(), r.end());
      row_ptr[i + 1] = (int)row_idx.size();
    }
  } else {
    if (!desc->row_ptr || (m && !desc->row_idx)) return fail(FWBF_EINVAL, "CSR arrays required");
    if (desc->row_ptr[0] != 0) return fail(FWBF_EINVAL, "row_ptr[0] must be 0");
    for (int i = 0; i < m; ++i) {
      const int a = desc->row_ptr[i], b = desc->row_ptr[i + 1];
      if (b < a) return fail(FWBF_EINVAL, "row_ptr must be nondecreasing");
      for (int e = a; e < b; ++e) {
        const int c = desc->row_idx[e];
        if (c < 0 || c >= n) return fail(FWBF_EINVAL, "row %d has a column index out of range", i);
        if (e > a && c <= desc->row_idx[e - 1]) return fail(FWBF_EINVAL, "row %d is not strictly ascending", i);
      }
      row_ptr[i + 1] = b;
    }
    row_idx.assign(desc->row_idx, desc->row_idx + row_ptr[m]);
  }
  const long long E = row_ptr[m];
  // CSC with ascending checks per column (matrix.py:38-42 builds col_adj row by row).
  // col_eid: the row-major edge index of each CSC entry (the reference's edge
  // order, matrix.py:49-52), for the stage kernels' edge-weight vectors.
  std::vector<int> col_ptr(n + 1, 0), col_idx(E), col_eid(E);
  for (long long e = 0; e < E; ++e) col_ptr[row_idx[e] + 1]++;
  for (int i = 0; i < n; ++i) col_ptr[i + 1] += col_ptr[i];
  {
    std::vector<int> fill(col_ptr.begin(), col_ptr.end() - 1);
    for (int i = 0; i < m; ++i)
      for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        col_eid[fill[row_idx[e]]] = e;
        col_idx[fill[row_idx[e]]++] = i;
      }
  }
  fwbf_code *c = new fwbf_code();
  c->device = device;
  c->n = n;
  c->m = m;
  c->n_edges = E;
  int dvm = 0, dcm = 0, minrw = m ? 1 << 30 : 2;
  for (int i = 0; i < n; ++i) dvm = std::max(dvm, col_ptr[i + 1] - col_ptr[i]);
  for (int i = 0; i < m; ++i) {
    dcm = std::max(dcm, row_ptr[i + 1] - row_ptr[i]);
    minrw = std::min(minrw, row_ptr[i + 1] - row_ptr[i]);
  }
  c->dv_max = dvm;
  c->dc_max = dcm;
  c->min_row_w = minrw;
  if (!desc->circulant) {
    c->h_row_ptr = row_ptr;
    c->h_row_idx = row_idx;
    c->h_col_ptr = col_ptr;
    c->h_col_idx = col_idx;
  }
  std::vector<uint8_t> i0tab, jwtab;
  std::vector<int16_t> offpos;
  if (desc->circulant) {
    c->circ = 1;
    c->w = desc->n_offsets;
    const int w = c->w;
    for (int j = 0; j < w; ++j) c->off[j] = desc->offsets[j];
    std::vector<int> dn(w);
    for (int j = 0; j < w; ++j) dn[j] = (n - desc->offsets[j]) % n;
    std::sort(dn.begin(), dn.end());
    for (int j = 0; j < w; ++j) c->dneg[j] = dn[j];
    for (int j = 0; j < w; ++j) // position of (n - c_j) mod n in the sorted list
      c->jii[j] = (unsigned char)(std::lower_bound(dn.begin(), dn.end(), (n - desc->offsets[j]) % n) - dn.begin());
    // Column n's checks are (n + dneg[i]) mod n; ascending order starts at the
    // first i with n + dneg[i] >= n (the wrapped, smaller ones).
    i0tab.resize(n);
    for (int col = 0; col < n; ++col) {
      int i0 = 0;
      while (i0 < w && col + dn[i0] < n) ++i0;
      i0tab[col] = (uint8_t)(i0 == w ? 0 : i0);
    }
    // check m's columns m + c_j wrap (>= n) from j = jwtab[m] on
    jwtab.resize(n);
    for (int m = 0; m < n; ++m) {
      int j = 0;
      while (j < w && m + desc->offsets[j] < n) ++j;
      jwtab[m] = (uint8_t)j;
    }
    offpos.assign(n, (int16_t)-1);
    for (int j = 0; j < w; ++j) offpos[desc->offsets[j]] = (int16_t)j;
  }
  if (!desc->circulant) {
    // quasi-cyclic detection: every Z x Z block zero or one shifted identity
    // (row i -> column (i + s) mod Z); Z a power of two, at most 256 blocks
    for (int Z = 1024; Z >= 16 && !c->qc_z; Z >>= 1) {
      if (n % Z || m % Z || (long long)(n / Z) * (m / Z) > fwbf::kMaxQcBlocks) continue;
      const int jb = m / Z, kb = n / Z;
      std::vector<int> sh(jb * kb, -2), cnt(jb * kb, 0);
      bool okq = true;
      for (int r = 0; r < m && okq; ++r)
        for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
          const int col = row_idx[e];
          const int b = (r / Z) * kb + col / Z;
          const int s = ((col % Z) - (r % Z) + Z) % Z;
          if (sh[b] == -2) sh[b] = s;
          else if (sh[b] != s) { okq = false; break; }
          cnt[b]++;
        }
      for (int b = 0; b < jb * kb && okq; ++b)
        if (cnt[b] != 0 && cnt[b] != Z) okq = false;
      if (!okq) continue;
      c->qc_z = Z;
      c->qc_jb = jb;
      c->qc_kb = kb;
      for (int b = 0; b < jb * kb; ++b) c->qc_shift[b] = (short)(cnt[b] ? sh[b] : -1);
    }
  }
  int rc;
  DeviceGuard dg;
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) { delete c; return fail(FWBF_ECUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(ce)); }
  if ((rc = upload(&c->d_row_ptr, row_ptr)) || (rc = upload(&c->d_row_idx, row_idx)) ||
      (rc = upload(&c->d_col_ptr, col_ptr)) || (rc = upload(&c->d_col_idx, col_idx)) ||
      (rc = upload(&c->d_col_eid, col_eid)) ||
      (rc = upload(&c->d_i0tab, i0tab)) || (rc = upload(&c->d_jwtab, jwtab)) || (rc = upload(&c->d_offpos, offpos))) {
    fwbf_code_destroy(c);
    return rc;
  }
  ce = cudaMalloc((void **)&c->d_work, kWorkRing * sizeof(unsigned));
  if (ce != cudaSuccess) { fwbf_code_destroy(c); return fail(FWBF_ECUDA, "cudaMalloc: %s", cudaGetErrorString(ce)); }
  ce = cudaMalloc((void **)&c->d_fstats, 2 * sizeof(unsigned long long));
  if (ce == cudaSuccess) ce = cudaMemset(c->d_fstats, 0, 2 * sizeof(unsigned long long));
  if (ce != cudaSuccess) { fwbf_code_destroy(c); return fail(FWBF_ECUDA, "cudaMalloc: %s", cudaGetErrorString(ce)); }
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  *out = c;
  return FWBF_OK;
}

extern "C" int fwbf_code_destroy(fwbf_code *c) {
  if (!c) return FWBF_OK;
  DeviceGuard dg;
  cudaSetDevice(c->device);
  cudaFree(c->d_row_ptr);
  cudaFree(c->d_row_idx);
  cudaFree(c->d_col_ptr);
  cudaFree(c->d_col_idx);
  cudaFree(c->d_col_eid);
  cudaFree(c->d_i0tab);
  cudaFree(c->d_jwtab);
  cudaFree(c->d_offpos);
  cudaFree(c->d_work);
  cudaFree(c->d_fstats);
  for (int i = 0; i < 5; ++i)
    if (c->pipe_s[i]) cudaStreamDestroy(c->pipe_s[i]);
  for (int i = 0; i < 4; ++i)
    for (int b = 0; b < 4; ++b)
      if (c->pipe_ev[i][b]) cudaEventDestroy(c->pipe_ev[i][b]);
  for (int i = 0; i < 4; ++i)
    if (c->pipe_buf[i]) cudaFree(c->pipe_buf[i]);
  cudaFree(c->pipe_counters);
  cudaFree(c->noise_buf);
  if (c->noise_evt) cudaEventDestroy(c->noise_evt);
  if (c->noise_side) cudaStreamDestroy(c->noise_side);
  if (c->noise_fork) cudaEventDestroy(c->noise_fork);
  if (c->noise_join) cudaEventDestroy(c->noise_join);
  if (c->noise_def) cudaStreamDestroy(c->noise_def);
  if (c->noise_join2) cudaEventDestroy(c->noise_join2);
  for (int i = 0; i < 3; ++i) {
    if (c->noise_cev[i]) cudaEventDestroy(c->noise_cev[i]);
    if (c->noise_dev[i]) cudaEventDestroy(c->noise_dev[i]);
  }
  for (XPlan &x : c->xplans) {
    cudaFree(x.d_tab);
    cudaFree(x.d_rtab);
    cudaFree(x.d_cpos);
    cudaFree(x.d_invp);
    cudaFree(x.d_ctab);
  }
  delete c;
  return FWBF_OK;
}

extern "C" int fwbf_code_info(const fwbf_code *c, int32_t *n, int32_t *m, int32_t *e, int32_t *circ) {
  if (!c) return fail(FWBF_EINVAL, "null code");
  if (n) *n = c->n;
  if (m) *m = c->m;
  if (e) *e = (int32_t)c->n_edges;
  if (circ) *circ = c->circ;
  return FWBF_OK;
}

static int validate(const fwbf_code *c, const fwbf_params *p) {
  if (!c || !p) return fail(FWBF_EINVAL, "null argument");
  if (!(p->alpha >= 0)) return fail(FWBF_EINVAL, "alpha must be nonnegative");
  if (p->k_max < 1) return fail(FWBF_EINVAL, "k_max must be >= 1");
  if (p->lam < 1) return fail(FWBF_EINVAL, "lam must be >= 1");
  if (p->stall != FWBF_STALL_FLIP_GLOBAL_MAX && p->stall != FWBF_STALL_TERMINATE)
    return fail(FWBF_EINVAL, "unknown stall policy %d", p->stall);
  if (p->weight_mode != FWBF_WEIGHTS_IMWBF && p->weight_mode != FWBF_WEIGHTS_MWBF)
    return fail(FWBF_EINVAL, "unknown weight mode %d", p->weight_mode);
  switch (p->algorithm) {
  case FWBF_ALG_FWBF:
    if (p->block_len_p < 1) return fail(FWBF_EINVAL, "block_len_p must be >= 1");
    break;
  case FWBF_ALG_IMWBF: break;
  case FWBF_ALG_MLP:
    if (p->lam > c->n) return fail(FWBF_EINVAL, "lam=%d exceeds block length %d", p->lam, c->n);
    break;
  default: return fail(FWBF_EINVAL, "unknown algorithm %d", p->algorithm);
  }
  if (c->m && c->min_row_w < 2) return fail(FWBF_EINVAL, "every check must contain at least 2 bits");
  return FWBF_OK;
}

extern "C" int64_t fwbf_max_flips_per_iter(const fwbf_code *c, const fwbf_params *p) {
  if (!c || !p) return 0;
  switch (p->algorithm) {
  case FWBF_ALG_FWBF: return p->block_len_p >= 1 ? (c->n + p->block_len_p - 1) / p->block_len_p : 0;
  case FWBF_ALG_IMWBF: return 1;
  case FWBF_ALG_MLP: return std::min(p->lam, c->n);
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Launch planning
// ---------------------------------------------------------------------------
static inline int align16(int x) { return (x + 15) & ~15; }

struct Plan {
  int threads = 0;
  int kc = 1;
  bool circ_kernel = false;
  int smem = 0;
};

static void layout(const fwbf_code *c, const fwbf_params *p, int ysize, bool circ, int cover, KParams &P,
                   bool compact = false, bool fused = false, bool mode2 = false, bool ystage = false,
                   int threads = 1024) {
  const int n = c->n, m = c->m;
  const int zw = (n + 31) / 32, sw = (m + 31) / 32;
  int nb = 1;
  if (p->algorithm == FWBF_ALG_FWBF) nb = (n + p->block_len_p - 1) / p->block_len_p;
  // MLP: per-warp candidate lists [nwarps][lam] + per-warp counts (int slots)
  const int nwarps = std::max(1, threads / 32);
  const int nslots = std::max(nb, p->algorithm == FWBF_ALG_MLP ? nwarps * p->lam : 1); // MLP: list values
  const int islots = std::max(nslots, p->algorithm == FWBF_ALG_MLP ? nwarps * (p->lam + 1) : 1);
  const int maxf = std::max(1, (int)fwbf_max_flips_per_iter(c, p));
  const int aw = (c->w > 32) ? 2 : 1;
  int o = 0;
  auto take = [&](int bytes) { int r = o; o = align16(o + bytes); return r; };
  if (compact) {
    // y (float32) lives only during frame init, so it overlays the metric
    // buffer; alpha*|y| comes from a per-frame table (split path) or global y.
    P.off_y = take(n * 8);
    P.off_e = P.off_y;
    P.alias_y = 1;
  } else if (ystage) {
    // the staging buffer below is the only copy of y in shared memory
    P.off_e = take(n * 8);
  } else {
    P.off_y = take(n * ysize);
    P.off_e = fused ? P.off_y : take(n * 8); // fused: no metric buffer
  }
  if (ystage) {
    P.ystage_bytes = (n * ysize + 15) & ~15;
    P.off_ystage = take(P.ystage_bytes);
    if (!compact) P.off_y = P.off_ystage;
  }
  // guarded path: doubled signed min1 plus zero pad up to the threads' column cover
  // check records: guarded path (circulant) = two doubled arrays sgn*min1,
  // sgn*min2 with a pad up to the threads' column cover; ordered path =
  // chk1[m], chk2[m], amin[m] inside the same region.
  if (circ && mode2) {
    // MODE 2 (filtered FWBF): split frames keep the two doubled float32 copies,
    // min2 per check (float), the argmin column and one coarse correction per
    // column; |y| lives in the metric region. Other frames take the ordered
    // path on single (wrapped) fp64 records with the argmin masks after them.
    const int dblf = (2 * n + std::max(0, cover - n) + 2 + 31) / 32 * 32;
    const int split_bytes = 2 * dblf * 4 + align16(m * 4) + align16(m * 2) + align16(n * 4);
    const int fp64_bytes = 2 * align16(m * 8) + n * aw * 4;
    const int r = take(std::max(fp64_bytes, split_bytes));
    P.off_chk1 = r;
    P.off_chk2 = r + align16(m * 8);
    P.off_amask = P.off_chk2 + align16(m * 8);
    P.off_fa = r;
    P.off_fb = r + dblf * 4;
    P.off_m2s = r + 2 * dblf * 4;
    P.off_a2m = P.off_m2s + align16(m * 4);
    P.off_corr = P.off_a2m + align16(m * 2);
    P.off_ay = P.off_corr;
    P.has_ay = 0;
    P.off_amin = 0;
  } else if (circ) {
    // both doubled arrays; chk2 - chk1 is a multiple of 128 B so a lane that
    // reads min2 instead of min1 hits the same banks (no extra wavefront)
    const int dbl = (2 * n + std::max(0, cover - n) + 31) / 32 * 32;
    // split-fp32 path (same region): signed min1 as float32 twice (second copy
    // shifted by one element for 8-byte pair loads), |min2|, argmin column,
    // and the per-column (lo, hi) correction limbs
    const int dblf = (2 * n + std::max(0, cover - n) + 2 + 31) / 32 * 32;
    const int split_bytes = 2 * dblf * 4 + align16(m * 8) + align16(m * 2) + (compact ? 2 : 1) * align16(n * 8);
    // the argmin masks (fp64 paths only) follow the two doubled arrays, inside
    // the split-path footprint when it is larger
    const int r = take(std::max(2 * dbl * 8 + n * aw * 4, split_bytes));
    P.off_amask = r + 2 * dbl * 8;
    P.off_chk1 = r;
    P.off_chk2 = r + dbl * 8;
    P.off_fa = r;
    P.off_fb = r + dblf * 4;
    P.off_m2s = r + 2 * dblf * 4;
    P.off_a2m = P.off_m2s + align16(m * 8);
    P.off_corr = P.off_a2m + align16(m * 2);
    P.off_ay = P.off_corr + align16(n * 8);
    P.has_ay = compact ? 1 : 0;
    P.off_amin = 0; // unused: the ordered circulant path reads argmin bits from amask
  } else {
    P.off_chk1 = take(m * 8);
    P.off_chk2 = take(m * 8);
    P.off_amin = take(m * 4);
  }
  // argmin masks, circulant only (placed above): guarded path bit j = offset
  // index; ordered path bit i = position in the column's ascending check list
  if (!circ) P.off_amask = take(4);
  P.off_sbits = take(sw * 4);
  P.off_zbits = take(zw * 4);
  P.off_blkv = take(nslots * 8);
  P.off_blki = take((islots + zw) * 4);
  P.off_flips = take(maxf * 4);
  P.off_offs = take(5 * fwbf::kMaxCircWeight * 4); // off[64], dneg doubled [128], rotated offsets [128]
  P.off_red = take(32 * 8 + 32 * 4);
  P.off_misc = take(16 * 4 + 64 * 4);
  P.smem_bytes = o;
}

// Shared memory of the filtered circulant kernel (fwbf_circ.cu): the kernel's
// compile-time layout (CLayout), copied into the parameter block so the gather
// offsets (uoff) can be computed from it.  EG(1023): 40 KB, 5 CTAs/SM.
template <int KC, int TB, int WT, int NN, int PB> static void layout_c(KParams &P) {
  using L = fwbf::CLayout<NN, KC * TB, WT, PB < 0 ? (TB / 32) * 32 * 8 : 0, fwbf::CircShape<TB, PB>::kStage>;
  P.ystage_bytes = L::YSTB;
  P.off_ystage = L::YST;
  P.off_y = L::YST;
  P.off_e = L::E;
  P.off_fa = L::FA;
  P.off_fb = L::FB;
  P.off_m2s = L::M2;
  P.off_a2m = L::A2;
  P.off_corr = L::CORR;
  P.off_sbits = L::SB;
  P.off_zbits = L::ZB;
  P.fd_words = L::FDW;
  P.off_fd = L::FD;
  P.off_blkv = L::BV;
  P.off_blki = L::BI;
  P.off_offs = L::ROT;
  P.off_misc = L::MISC;
  P.smem_bytes = L::BYTES;
}

// Launch-plan cache: the dynamic shared-memory attribute and the occupancy of
// a (device, kernel, threads, smem) shape are queried once, not per launch
// (small batches would otherwise pay two driver calls per decode).
struct PlanKey {
  int device;
  const void *kern;
  int threads, smem;
  bool operator==(const PlanKey &o) const {
    return device == o.device && kern == o.kern && threads == o.threads && smem == o.smem;
  }
};

static int plan_occupancy(int device, const void *kern, int threads, int smem, int *per_sm) {
  static std::mutex mu;
  static std::vector<std::pair<PlanKey, int>> plans;
  static std::vector<std::pair<std::pair<int, const void *>, int>> attr; // (device, kern) -> smem attribute set
  const PlanKey key{device, kern, threads, smem};
  std::lock_guard<std::mutex> lock(mu);
  for (const auto &pl : plans)
    if (pl.first == key) { *per_sm = pl.second; return FWBF_OK; }
  int *have = nullptr;
  for (auto &a : attr)
    if (a.first.first == device && a.first.second == kern) have = &a.second;
  if (!have || *have < smem) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (have) *have = smem;
    else attr.push_back({{device, kern}, smem});
  }
  int occ = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  plans.push_back({key, occ});
  *per_sm = occ;
  return FWBF_OK;
}

// ---------------------------------------------------------------------------
// Explicit codes, FWBF: one frame per warp (fwbf_explicit.cu)
// ---------------------------------------------------------------------------
// Slot tables: blocks of p columns go to groups of G = 2^lg lanes; lane `sub`
// of the group for block b scans columns b p + sub + G c (c < S) in ascending
// order.  G minimises the per-iteration cost model (slots per lane x ~22
// instructions + butterfly levels per round).  Returns a plan with ok=false
// when the code does not fit the kernel's limits (dv <= 4, 16-bit indices,
// shared memory), in which case the CTA-per-frame kernel decodes it.
static int build_xplan(fwbf_code *c, int p, XPlan *out) {
  XPlan x;
  x.p = p;
  const int n = c->n, m = c->m;
  x.nb = (n + p - 1) / p;
  // record byte offsets (16 * check, two constant records after the M
  // checks) must fit 16 bits
  if (c->dv_max > 4 || m + 2 > 4096 || n > 0xffff || c->n_edges > (1 << 24)) { *out = x; return FWBF_OK; }
  x.dv = std::max(2, c->dv_max);
  long best_cost = -1;
  for (int lg = 0; lg <= 5; ++lg) {
    const int G = 1 << lg;
    const long R = ((long)x.nb * G + 31) / 32, S = (p + G - 1) / G;
    const long cost = R * S * 22 + R * lg * 8 + R * 6;
    if (R * S * 32 > 0xffff) continue;
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; x.lg_g = lg; x.rounds = (int)R; x.slots = (int)S; }
  }
  if (best_cost < 0) { *out = x; return FWBF_OK; }
  const int G = 1 << x.lg_g, R = x.rounds, S = x.slots, nslot = R * S * 32;
  // slot -> column (or -1) first; the check labels depend on which checks
  // share a load instruction
  std::vector<int> scol(nslot, -1);
  for (int r = 0; r < R; ++r)
    for (int cc = 0; cc < S; ++cc)
      for (int l = 0; l < 32; ++l) {
        const int b = r * (32 / G) + l / G, sub = l % G;
        if (b >= x.nb) continue;
        const int base = b * p, lim = std::min(p, n - base);
        if (sub + G * cc < lim) scol[(r * S + cc) * 32 + l] = base + sub + G * cc;
      }
  // Labels: the q-th check of the 32 slots (r, c, *) is one 4-byte load of
  // 32 lanes; the record at label j sits in bank j mod 32.  Greedy: checks by
  // decreasing number of loads, each to the bank (with labels left) least
  // used by the loads it takes part in.
  std::vector<int> lab(m, -1);
  {
    const int ninstr = R * S * 4;
    std::vector<std::vector<int>> loads(m); // instructions per check
    for (int r = 0; r < R; ++r)
      for (int cc = 0; cc < S; ++cc)
        for (int l = 0; l < 32; ++l) {
          const int col = scol[(r * S + cc) * 32 + l];
          if (col < 0) continue;
          for (int e = c->h_col_ptr[col], q = 0; e < c->h_col_ptr[col + 1]; ++e, ++q)
            loads[c->h_col_idx[e]].push_back((r * S + cc) * 4 + q);
        }
    std::vector<int> order(m);
    for (int i = 0; i < m; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b2) { return loads[a].size() > loads[b2].size(); });
    constexpr int NB = 32; // banks
    std::vector<int> cnt((size_t)ninstr * NB, 0), cap(NB, 0), next(NB, 0);
    for (int j = 0; j < m; ++j) cap[j % NB]++;
    for (int k = 0; k < NB; ++k) next[k] = k;
    for (int chk : order) {
      int bestk = -1;
      long bestc = 0;
      for (int k = 0; k < NB; ++k) {
        if (!cap[k]) continue;
        long cst = 0;
        for (int ins : loads[chk]) cst += cnt[(size_t)ins * NB + k];
        if (bestk < 0 || cst < bestc) { bestk = k; bestc = cst; }
      }
      for (int ins : loads[chk]) cnt[(size_t)ins * NB + bestk]++;
      cap[bestk]--;
      lab[chk] = next[bestk];
      next[bestk] += NB;
    }
  }
  std::vector<int> invp(m);
  for (int i = 0; i < m; ++i) invp[lab[i]] = i;
  // padding slots read the (-inf, -inf) label m on every edge
  unsigned long long padw = 0;
  for (int q = 0; q < 4; ++q) padw |= (unsigned long long)(4 * m) << (16 * q);
  std::vector<unsigned long long> tab(nslot, padw);
  std::vector<uint16_t> cpos(n, 0);
  for (int r = 0; r < R; ++r)
    for (int cc = 0; cc < S; ++cc)
      for (int l = 0; l < 32; ++l) {
        const int b = r * (32 / G) + l / G, sub = l % G;
        if (b >= x.nb) continue;
        const int base = b * p, lim = std::min(p, n - base);
        if (sub + G * cc >= lim) continue;
        const int col = base + sub + G * cc, pos = (r * S + cc) * 32 + l;
        // byte offsets of the column's check records, ascending checks; the
        // (0, 0) label m + 1 fills the edges it does not have
        unsigned long long w = 0;
        const int e0 = c->h_col_ptr[col], e1 = c->h_col_ptr[col + 1];
        for (int q = 0; q < 4; ++q) {
          const int j = e0 + q < e1 ? lab[c->h_col_idx[e0 + q]] : m + 1;
          w |= (unsigned long long)(4 * j) << (16 * q);
        }
        tab[pos] = w;
        cpos[col] = (uint16_t)pos;
      }
  std::vector<uint32_t> rtab(c->n_edges);
  for (int r = 0; r < m; ++r)
    for (int e = c->h_row_ptr[r]; e < c->h_row_ptr[r + 1]; ++e) {
      const int col = c->h_row_idx[e];
      int q = 0;
      while (c->h_col_idx[c->h_col_ptr[col] + q] != r) ++q;
      rtab[e] = (uint32_t)cpos[col] | ((uint32_t)q << 16);
    }
  // shared memory: CTA tables, then one region per warp
  int o = 0;
  auto take = [&](int bytes) { int r0 = o; o = align16(o + bytes); return r0; };
  x.off_tab = take(nslot * 8);
  x.off_cpos = take(n * 2);
  x.tables_bytes = o;
  int w = 0;
  auto wtake = [&](int bytes) { int r0 = w; w = align16(w + bytes); return r0; };
  x.s2sh = 7;
  while ((1 << x.s2sh) < 4 * (m + 2)) ++x.s2sh;
  x.wo_rec = wtake((1 << x.s2sh) + 4 * (m + 2));
  x.wo_ys = wtake(nslot * 4);
  x.wo_am = wtake(nslot);
  x.wo_sb = wtake(((m + 31) / 32) * 4);
  x.wo_zw = wtake(((n + 31) / 32) * 4);
  x.wo_bf = wtake(x.nb * 4);
  x.warp_bytes = w;
  // warps per CTA: the most resident warps per SM
  const void *kern = x.dv == 2 ? (const void *)fwbf::xdecode_kernel<2>
                     : x.dv == 3 ? (const void *)fwbf::xdecode_kernel<3> : (const void *)fwbf::xdecode_kernel<4>;
  x.kern = kern;
  int best_warps = 0;
  for (int wpc : {8, 4, 2, 1}) {
    const int smem = x.tables_bytes + wpc * x.warp_bytes;
    if (smem > c->smem_optin) continue;
    int occ = 0;
    if (plan_occupancy(c->device, kern, 32 * wpc, smem, &occ)) return FWBF_ECUDA;
    if (occ * wpc > best_warps) { best_warps = occ * wpc; x.wpc = wpc; x.per_sm = occ; x.smem = smem; }
  }
  if (best_warps < 8) { *out = x; return FWBF_OK; } // too few frames in flight: the CTA kernel wins
  int rc;
  if ((rc = upload(&x.d_tab, tab)) || (rc = upload(&x.d_rtab, rtab)) || (rc = upload(&x.d_cpos, cpos)) ||
      (rc = upload(&x.d_invp, invp))) {
    cudaFree(x.d_tab);
    cudaFree(x.d_rtab);
    cudaFree(x.d_cpos);
    cudaFree(x.d_invp);
    return rc;
  }
  x.ok = true;
  // ---- incremental variant: per check label the slots of the check's columns ----
  {
    int dsh = 0;
    while ((1 << dsh) < c->dc_max) ++dsh;
    const long ctab_bytes = ((long)m << dsh) * 2;
    if (c->dc_max >= 1 && dsh <= 5 && ctab_bytes <= 32 * 1024) {
      std::vector<uint16_t> ctab((size_t)m << dsh, 0xffff);
      for (int j = 0; j < m; ++j) {
        const int chk = invp[j];
        int q = 0;
        for (int e = c->h_row_ptr[chk]; e < c->h_row_ptr[chk + 1]; ++e, ++q)
          ctab[((size_t)j << dsh) + q] = cpos[c->h_row_idx[e]];
      }
      x.dcs_sh = dsh;
      int o2 = x.tables_bytes;
      x.off_ctab = o2;
      o2 = align16(o2 + (int)ctab_bytes);
      x.inc_tables_bytes = o2;
      int w2 = x.warp_bytes;
      x.wo_ek = w2;
      w2 = align16(w2 + nslot * 4);
      x.wo_tl = w2;
      w2 = align16(w2 + (x.nb + 1) * x.dv * 2);
      x.inc_warp_bytes = w2;
      x.inc_kern = x.dv == 2 ? (const void *)fwbf::xinc_kernel<2>
                   : x.dv == 3 ? (const void *)fwbf::xinc_kernel<3> : (const void *)fwbf::xinc_kernel<4>;
      int bw = 0;
      for (int wpc : {8, 4, 2, 1}) {
        const int smem = x.inc_tables_bytes + wpc * x.inc_warp_bytes;
        if (smem > c->smem_optin) continue;
        int occ = 0;
        if (plan_occupancy(c->device, x.inc_kern, 32 * wpc, smem, &occ)) return FWBF_ECUDA;
        if (occ * wpc > bw) { bw = occ * wpc; x.inc_wpc = wpc; x.inc_per_sm = occ; x.inc_smem = smem; }
      }
      if (bw >= 8 && upload(&x.d_ctab, ctab) == FWBF_OK) x.inc_ok = true;
    }
  }
  *out = x;
  return FWBF_OK;
}

static int launch_explicit(fwbf_code *c, const fwbf_params *p, const XPlan &x, const float *y, long long batch,
                           long long ld, const fwbf_outputs &o, cudaStream_t stream) {
  fwbf::XParams P;
  memset(&P, 0, sizeof P);
  P.n = c->n;
  P.m = c->m;
  P.n_edges = (int)c->n_edges;
  P.nb = x.nb;
  P.p = x.p;
  P.lg_g = x.lg_g;
  P.rounds = x.rounds;
  P.slots = x.slots;
  P.kmax = p->k_max;
  P.stall = p->stall;
  P.wmode = p->weight_mode;
  P.alpha = p->alpha;
  P.tab = x.d_tab;
  P.rtab = x.d_rtab;
  P.row_ptr = c->d_row_ptr;
  P.cpos = x.d_cpos;
  P.invp = x.d_invp;
  P.s2sh = x.s2sh;
  P.s2off = 1 << x.s2sh;
  P.off_tab = x.off_tab;
  P.off_cpos = x.off_cpos;
  // the incremental kernel (stored metrics, only the columns of toggled checks recomputed) unless switched off
  const bool inc = x.inc_ok && !getenv("FWBF_NO_XINC");
  P.off_warp0 = inc ? x.inc_tables_bytes : x.tables_bytes;
  P.warp_bytes = inc ? x.inc_warp_bytes : x.warp_bytes;
  P.ctab = x.d_ctab;
  P.off_ctab = x.off_ctab;
  P.dcs_sh = x.dcs_sh;
  P.wo_ek = x.wo_ek;
  P.wo_tl = x.wo_tl;
  P.wo_rec = x.wo_rec;
  P.wo_ys = x.wo_ys;
  P.wo_am = x.wo_am;
  P.wo_sb = x.wo_sb;
  P.wo_zw = x.wo_zw;
  P.wo_bf = x.wo_bf;
  P.y = y;
  P.ld = ld;
  P.batch = batch;
  P.y_vec4 = ((uintptr_t)y % 16) == 0 && ld % 4 == 0;
  P.z_bits = o.z_bits;
  P.z_ld = o.z_ld;
  P.iterations = o.iterations;
  P.flags = o.flags;
  P.flips_total = o.flips_total;
  P.bit_errors = o.bit_errors;
  P.fliplog = o.fliplog;
  P.fliplog_counts = o.fliplog_counts;
  P.fliplog_stride = o.fliplog_stride;
  P.counters = (long long *)o.counters;
  P.iter_hist = (long long *)o.iter_hist;
  P.batch_word_err = o.batch_word_err;
  P.batch_frames = o.batch_frames;
  P.codeword_bits = o.codeword_bits;
  const unsigned slot = c->work_slot.fetch_add(1) % kWorkRing;
  P.work_counter = c->d_work + slot;
  const int wpc = inc ? x.inc_wpc : x.wpc, per_sm = inc ? x.inc_per_sm : x.per_sm;
  const long long grid = std::min<long long>((batch + wpc - 1) / wpc, (long long)per_sm * c->sm_count);
  CUDA_TRY(cudaMemsetAsync(P.work_counter, 0, sizeof(unsigned), stream));
  void *args[] = {&P};
  CUDA_TRY(cudaLaunchKernel(inc ? x.inc_kern : x.kern, dim3((unsigned)grid), dim3(32 * wpc), args,
                            inc ? x.inc_smem : x.smem, stream));
  CUDA_TRY(cudaGetLastError());
  g_last_kernel = inc ? "xinc" : "xdecode";
  return FWBF_OK;
}

// ---------------------------------------------------------------------------
// Quasi-cyclic codes, FWBF with 32 | p, blocks inside block columns (fwbf_qc.cu)
// ---------------------------------------------------------------------------
static int launch_qc(fwbf_code *c, const fwbf_params *p, const float *y, long long batch, long long ld,
                     const fwbf_outputs &o, cudaStream_t stream, bool *used) {
  *used = false;
  const int Z = c->qc_z, pp = p->block_len_p;
  if (!Z || c->qc_jb > 4 || pp % 32 || pp > Z || Z % pp || c->m > 32 * 512) return FWBF_OK;
  const int tpc = pp / 32;
  // the incremental kernel (stored metric keys, only the columns of toggled
  // checks recomputed) unless switched off; the full-pass kernel otherwise
  const bool inc = !getenv("FWBF_NO_QCINC") && c->n < 65535;
  bool allp = true; // every circulant block present: the kernel skips the absent-block tests
  for (int i = 0; i < c->qc_jb * c->qc_kb; ++i) allp = allp && c->qc_shift[i] >= 0;
#define QINC_PICK(A)                                                                                         \
  (tpc == 1 ? (const void *)fwbf::qinc_kernel<1, A> : tpc == 2 ? (const void *)fwbf::qinc_kernel<2, A>       \
   : tpc == 4 ? (const void *)fwbf::qinc_kernel<4, A> : tpc == 8 ? (const void *)fwbf::qinc_kernel<8, A>     \
   : tpc == 16 ? (const void *)fwbf::qinc_kernel<16, A> : nullptr)
  const void *kern = inc ? (allp ? QINC_PICK(true) : QINC_PICK(false))
#undef QINC_PICK
                         : (tpc == 1 ? (const void *)fwbf::qdecode_kernel<1>
                            : tpc == 2 ? (const void *)fwbf::qdecode_kernel<2>
                            : tpc == 4 ? (const void *)fwbf::qdecode_kernel<4>
                            : tpc == 8 ? (const void *)fwbf::qdecode_kernel<8>
                            : tpc == 16 ? (const void *)fwbf::qdecode_kernel<16> : nullptr);
  if (!kern) return FWBF_OK;
  fwbf::QParams P;
  memset(&P, 0, sizeof P);
  P.n = c->n;
  P.m = c->m;
  P.n_edges = (int)c->n_edges;
  P.z = Z;
  P.lgz = 0;
  while ((1 << P.lgz) < Z) ++P.lgz;
  P.jb = c->qc_jb;
  P.kb = c->qc_kb;
  P.head = pp;
  memcpy(P.shift, c->qc_shift, sizeof P.shift);
  P.nb = c->n / pp;
  P.kmax = p->k_max;
  P.stall = p->stall;
  P.wmode = p->weight_mode;
  P.alpha = p->alpha;
  int off = 0;
  auto take = [&](int bytes) { int r0 = off; off = align16(off + bytes); return r0; };
  if (inc) {
    P.off_y = take(c->n * 4);                 // metric keys (y during the check scan)
    P.off_m1 = take(2 * c->m * 4);            // sgn min1 [M], then sgn min2 [M]
    P.off_m2 = P.off_m1 + c->m * 4;
    P.off_cmask = take((c->n + 3) / 4 * 4);   // argmin bit per row block, per column
    P.off_zrec = take(P.jb * P.kb * 4);       // shift table
    P.off_sbits = take(((c->m + 31) / 32) * 4);
    P.off_sold = take(((c->m + 31) / 32) * 4);
    P.off_zbits = take(((c->n + 31) / 32) * 4);
    P.off_blkv = take(P.nb * 8);
    P.off_blki = take(P.nb * 4);
    P.off_blkk = take(P.nb * 4);
    P.off_blkf = take(P.nb * 4);
    P.off_list = take(std::min(c->m, P.jb * (P.nb + 1)) * 4);
    P.off_dirty = take(3 * P.nb * 4);          // dirty flags [nb], two dirty lists [nb]
    P.off_misc = take(16 * 4);
  } else {
    P.off_y = take(c->n * 4);
    P.off_m1 = take(P.jb * (Z + pp) * 4);
    P.off_m2 = take(P.jb * (Z + pp) * 4);
    P.off_cmask = take((c->n + 3) / 4 * 4);
    P.off_zrec = take(pp * 4);
    P.off_sbits = take(((c->m + 31) / 32) * 4);
    P.off_zbits = take(((c->n + 31) / 32) * 4);
    P.off_blkv = take(P.nb * 8);
    P.off_blki = take(P.nb * 4);
    P.off_misc = take(16 * 4);
  }
  const int smem = off;
  if (smem > c->smem_optin) return FWBF_OK;
  const int T = 512;
  int per_sm = 0;
  int rc = plan_occupancy(c->device, kern, T, smem, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) return FWBF_OK;
  P.y = y;
  P.ld = ld;
  P.batch = batch;
  P.y_vec4 = ((uintptr_t)y % 16) == 0 && ld % 4 == 0;
  P.z_bits = o.z_bits;
  P.z_ld = o.z_ld;
  P.iterations = o.iterations;
  P.flags = o.flags;
  P.flips_total = o.flips_total;
  P.bit_errors = o.bit_errors;
  P.fliplog = o.fliplog;
  P.fliplog_counts = o.fliplog_counts;
  P.fliplog_stride = o.fliplog_stride;
  P.counters = (long long *)o.counters;
  P.iter_hist = (long long *)o.iter_hist;
  P.batch_word_err = o.batch_word_err;
  P.batch_frames = o.batch_frames;
  P.codeword_bits = o.codeword_bits;
  const unsigned slot = c->work_slot.fetch_add(1) % kWorkRing;
  P.work_counter = c->d_work + slot;
  const long long grid = std::min<long long>(batch, (long long)per_sm * c->sm_count);
  CUDA_TRY(cudaMemsetAsync(P.work_counter, 0, sizeof(unsigned), stream));
  void *args[] = {&P};
  CUDA_TRY(cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(T), args, smem, stream));
  CUDA_TRY(cudaGetLastError());
  *used = true;
  return FWBF_OK;
}

// The plan for (c, p), built on first use; nullptr when the kernel does not apply.
static const XPlan *get_xplan(fwbf_code *c, int p, int *rc) {
  *rc = FWBF_OK;
  std::lock_guard<std::mutex> lock(c->xplan_mu);
  for (const XPlan &x : c->xplans)
    if (x.p == p) return x.ok ? &x : nullptr;
  XPlan x;
  *rc = build_xplan(c, p, &x);
  if (*rc) return nullptr;
  c->xplans.push_back(x);
  return c->xplans.back().ok ? &c->xplans.back() : nullptr;
}

template <typename YT>
static int launch_decode(fwbf_code *c, const fwbf_params *p, const YT *y, long long batch,
                         long long ld, const fwbf_outputs *out, cudaStream_t stream,
                         double *metric_out = nullptr, long long metric_ld = 0,
                         cudaStream_t dstream = nullptr, cudaEvent_t dev = nullptr) {
  // dstream / dev (host pipeline): the second launch of a decode -- decode_kernel over the
  // frames the filtered circulant kernel deferred -- goes on dstream, ordered after the first
  // by dev, so the next chunk's main kernel (on another stream) can fill the SMs this one's
  // last frames leave instead of waiting behind a launch that has almost nothing to do
  int rc = validate(c, p);
  if (rc) return rc;
  if (batch < 0) return fail(FWBF_EINVAL, "batch must be nonnegative");
  if (batch == 0) return FWBF_OK;
  if (!y) return fail(FWBF_EINVAL, "y is null");
  if (ld < c->n) return fail(FWBF_EINVAL, "expected a length-%d frame (ld=%lld)", c->n, ld);
  if (batch > 0x7fffffffLL) return fail(FWBF_EINVAL, "batch too large for one call");
  fwbf_outputs o = out ? *out : fwbf_outputs{};
  const long long maxf = fwbf_max_flips_per_iter(c, p);
  if (o.fliplog) {
    if (!o.fliplog_counts) return fail(FWBF_EINVAL, "fliplog requires fliplog_counts");
    if (o.fliplog_stride < (long long)p->k_max * maxf)
      return fail(FWBF_EINVAL, "fliplog_stride must be >= k_max * %lld", maxf);
  }
  if (o.z_bits && o.z_ld < (c->n + 31) / 32) return fail(FWBF_EINVAL, "z_ld too small");
  if (o.batch_word_err && o.batch_frames < 1) return fail(FWBF_EINVAL, "batch_frames must be >= 1");

  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->circ && c->qc_z && sizeof(YT) == 4 && p->algorithm == FWBF_ALG_FWBF && !metric_out &&
      !getenv("FWBF_NO_QC") && !getenv("FWBF_NO_QCK")) {
    bool used = false;
    rc = launch_qc(c, p, (const float *)y, batch, ld, o, stream, &used);
    if (used) g_last_kernel = getenv("FWBF_NO_QCINC") || c->n >= 65535 ? "qdecode" : "qinc";
    if (rc || used) return rc;
  }
  if (!c->circ && sizeof(YT) == 4 && p->algorithm == FWBF_ALG_FWBF && !metric_out && !getenv("FWBF_NO_WARP")) {
    const XPlan *xp = get_xplan(c, p->block_len_p, &rc);
    if (rc) return rc;
    if (xp) {
      return launch_explicit(c, p, *xp, (const float *)y, batch, ld, o, stream);
    }
  }
  KParams P;
  memset(&P, 0, sizeof P);
  P.n = c->n;
  P.m = c->m;
  P.w = c->circ ? c->w : 0;
  P.dv_max = c->dv_max;
  P.n_edges = c->n_edges;
  memcpy(P.off, c->off, sizeof P.off);
  memcpy(P.dneg, c->dneg, sizeof P.dneg);
  memcpy(P.jii, c->jii, sizeof P.jii);
  P.i0tab = c->d_i0tab;
  P.jwtab = c->d_jwtab;
  P.offpos = c->d_offpos;
  P.row_ptr = c->d_row_ptr;
  P.row_idx = c->d_row_idx;
  P.col_ptr = c->d_col_ptr;
  P.col_idx = c->d_col_idx;
  P.qc_z = getenv("FWBF_NO_QC") ? 0 : c->qc_z;
  P.qc_jb = c->qc_jb;
  P.qc_kb = c->qc_kb;
  memcpy(P.qc_shift, c->qc_shift, sizeof P.qc_shift);
  P.alg = p->algorithm;
  P.wmode = p->weight_mode;
  P.kmax = p->k_max;
  P.lam = p->lam;
  P.p = p->block_len_p;
  P.stall = p->stall;
  P.mlp_thr = p->mlp_threshold ? 1 : 0;
  P.force_ordered = (p->force_ordered & 1) ? 1 : 0;
  P.no_split = (p->force_ordered & 2) || getenv("FWBF_NO_SPLIT") ? 1 : 0;
  P.alpha = p->alpha;
  // FWBF: approximate fp32 gather on split-path frames, close decisions
  // resolved exactly (kernel: GatherF2 / exact_split_metric); same results
  P.filter = p->algorithm == FWBF_ALG_FWBF && !metric_out && !(p->force_ordered & 4) && !getenv("FWBF_NO_FILTER") &&
             !P.no_split; // the guarded fp64 path exists only in the exact kernels
  P.filter_stats = c->d_fstats;
  P.nblocks = p->algorithm == FWBF_ALG_FWBF ? (c->n + p->block_len_p - 1) / p->block_len_p : 1;
  P.y = y;
  P.ld = ld;
  P.batch = batch;

  P.z_bits = o.z_bits;
  P.z_ld = o.z_ld;
  P.iterations = o.iterations;
  P.flags = o.flags;
  P.flips_total = o.flips_total;
  P.bit_errors = o.bit_errors;
  P.fliplog = o.fliplog;
  P.fliplog_counts = o.fliplog_counts;
  P.fliplog_stride = o.fliplog_stride;
  P.counters = (long long *)o.counters;
  P.iter_hist = (long long *)o.iter_hist;
  P.batch_word_err = o.batch_word_err;
  P.batch_frames = o.batch_frames;
  P.codeword_bits = o.codeword_bits;
  const unsigned slot = c->work_slot.fetch_add(1) % kWorkRing;
  P.work_counter = c->d_work + slot;

  const bool circ = c->circ && c->n <= 8192;
  const void *kern = nullptr;
  int T = 0;
  int kc = 1;
  int kwt = 0; // compile-time circulant weight of the chosen kernel (0: runtime)
  bool mode2 = false; // MODE 2 (filtered) kernel: its own shared-memory layout
  if (circ) {
    if (sizeof(YT) == 4) {
      struct Shape { int kc, tb, wt; const void *fn; };
      static const Shape shapes[] = {
#define FWBF_SHAPE(YT_, C_, KC_, TB_, WT_) {KC_, TB_, WT_, (const void *)fwbf::decode_kernel<YT_, C_, KC_, TB_, WT_>},
          FWBF_FAST_CONFIGS(FWBF_SHAPE)
#undef FWBF_SHAPE
      };
      const Shape *tab = shapes;
      const int ntab = (int)(sizeof(shapes) / sizeof(shapes[0]));
      int want_kc = 0, want_tb = 0; // FWBF_SHAPE="KCxTB" forces a shape (tuning)
      if (const char *e = getenv("FWBF_SHAPE")) sscanf(e, "%dx%d", &want_kc, &want_tb);
      const bool generic_only = getenv("FWBF_GENERIC_W") != nullptr;
      for (int i = 0; i < ntab && want_kc; ++i)
        if (tab[i].kc == want_kc && tab[i].tb == want_tb && tab[i].kc * tab[i].tb >= c->n &&
            (tab[i].wt == 0 || (tab[i].wt == c->w && !generic_only))) {
          kern = tab[i].fn; T = tab[i].tb; kc = tab[i].kc; kwt = tab[i].wt;
          if (tab[i].wt) break;
        }
      // prefer the smallest shape covering n with the weight compiled in
      for (int i = 0; i < ntab && !kern && !generic_only; ++i)
        if (tab[i].wt == c->w && tab[i].kc * tab[i].tb >= c->n && tab[i].kc * tab[i].tb < 4 * c->n + 256) {
          kern = tab[i].fn; T = tab[i].tb; kc = tab[i].kc; kwt = tab[i].wt;
        }
      for (int i = 0; i < ntab && !kern; ++i)
        if (tab[i].wt == 0 && tab[i].kc * tab[i].tb >= c->n) { kern = tab[i].fn; T = tab[i].tb; kc = tab[i].kc; kwt = tab[i].wt; break; }
      // IMWBF: the same shape with the incremental integer metric
      if (kwt && p->algorithm == FWBF_ALG_IMWBF && !metric_out && !getenv("FWBF_NO_INC")) {
        static const Shape inc[] = {
#define FWBF_SHAPE_INC(YT_, C_, KC_, TB_, WT_) {KC_, TB_, WT_, (const void *)fwbf::decode_kernel<YT_, C_, KC_, TB_, WT_, 1>},
            FWBF_INC_CONFIGS(FWBF_SHAPE_INC)
#undef FWBF_SHAPE_INC
        };
        for (const Shape &sh : inc)
          if (sh.kc == kc && sh.tb == T && sh.wt == kwt) kern = sh.fn;
      }
      // FWBF: the same shape with the filtered metric (P.filter)
      if (kwt && P.filter) {
        mode2 = true;
        static const Shape filt[] = {
#define FWBF_SHAPE_FILT(YT_, C_, KC_, TB_, WT_) {KC_, TB_, WT_, (const void *)fwbf::decode_kernel<YT_, C_, KC_, TB_, WT_, 2>},
            FWBF_INC_CONFIGS(FWBF_SHAPE_FILT)
#undef FWBF_SHAPE_FILT
        };
        bool found = false;
        for (const Shape &sh : filt)
          if (sh.kc == kc && sh.tb == T && sh.wt == kwt) { kern = sh.fn; found = true; }
        mode2 = found;
      }
    } else {
      struct Shape { int kc, tb, wt; const void *fn; };
      static const Shape shapes[] = {
#define FWBF_SHAPE(YT_, C_, KC_, TB_, WT_) {KC_, TB_, WT_, (const void *)fwbf::decode_kernel<YT_, C_, KC_, TB_, WT_>},
          FWBF_F64_CONFIGS(FWBF_SHAPE)
#undef FWBF_SHAPE
      };
      if (!getenv("FWBF_GENERIC_W"))
        for (const Shape &sh : shapes)
          if (sh.wt == c->w && sh.kc * sh.tb >= c->n && sh.kc * sh.tb < 4 * c->n + 256) {
            kern = sh.fn; T = sh.tb; kc = sh.kc;
            break;
          }
      if (!kern) {
        T = c->n <= 2048 ? 256 : (c->n <= 8192 ? 512 : 1024);
        kern = (const void *)fwbf::decode_kernel<double, true, 1, 0, 0>;
      }
    }
  } else {
    T = c->n <= 2048 ? 256 : (c->n <= 8192 ? 512 : 1024);
    kern = sizeof(YT) == 4 ? (const void *)fwbf::decode_kernel<float, false, 1, 0, 0>
                           : (const void *)fwbf::decode_kernel<double, false, 1, 0, 0>;
  }
  // explicit/QC FWBF with 32 | p: metric and block argmax in one warp pass (no
  // metric buffer); 512 threads so two CTAs share an SM on large codes
  P.fused = !circ && p->algorithm == FWBF_ALG_FWBF && p->block_len_p % 32 == 0 && !getenv("FWBF_NO_FUSED") &&
            !metric_out;
  P.metric_out = metric_out;
  P.metric_ld = metric_ld;
  if (P.fused && T > 512) T = 512;
  // small explicit codes: ~8 columns per thread and more, smaller CTAs per SM
  // (the per-iteration barriers and serial phases cost less; A: 64 threads +40%)
  if (!circ && !P.fused && c->n <= 2048) T = std::min(256, std::max(64, ((c->n + 7) / 8 + 31) / 32 * 32));
  if (!circ)
    if (const char *e = getenv("FWBF_EXPLICIT_T")) T = atoi(e); // tuning: threads per CTA (multiple of 32)
  // Each thread keeps the previous syndrome bits of its checks tid + k*T in
  // one 32-bit register (k < ceil(M/T)): redundant H with M > 32 T needs a
  // wider CTA.
  if (c->m > 32 * T) T = ((c->m + 31) / 32 + 31) / 32 * 32;
  if (c->m > 32 * T || T > 1024)
    return fail(FWBF_EUNSUPPORTED, "%d checks exceed the 32 x %d per-thread syndrome registers", c->m,
                std::min(T, 1024));
  // FWBF on float32 y, circulant weight compiled in, filtered metric: the
  // round-3 kernel (fwbf_circ.cu) decodes every frame its guard admits and
  // defers the rest to this MODE 2 kernel, which then runs over that list.
  const void *ckern = nullptr;
  void (*clayout)(KParams &) = nullptr;
  // MLP-WBF (lambda <= 31) on the same kernel with the filtered top-lambda
  // selection, under the same conditions as FWBF's filtered metric
  const bool cmlp = p->algorithm == FWBF_ALG_MLP && p->lam >= 1 && p->lam <= fwbf::kCircMaxLam && circ &&
                    sizeof(YT) == 4 && kwt > 0 && !metric_out && !p->force_ordered &&
                    !getenv("FWBF_NO_FILTER") && !getenv("FWBF_NO_SPLIT");
  if ((mode2 || cmlp) && sizeof(YT) == 4 && kwt > 0 && c->m == c->n && p->weight_mode == FWBF_WEIGHTS_IMWBF &&
      (cmlp || p->block_len_p >= 16) && !P.force_ordered && !getenv("FWBF_NO_CDEC")) {
    // 16-bit quantised gather (default for FWBF) or the float32 gather; MLP keeps the float32 one: its
    // exact top-lambda over a wider band costs small batches more than the gather saves
    const bool q16 = q16_enabled() && !cmlp;
#define FWBF_PICK_C(KC_, TB_, WT_, NN_, PB_)                                                        \
    if (kc == KC_ && T == TB_ && kwt == WT_ && c->n == NN_ &&                                      \
        (cmlp ? PB_ < 0 : (PB_ == 0 || PB_ == p->block_len_p)) && !(PB_ == 0 && ckern)) {          \
      ckern = q16 ? (const void *)fwbf::cdecode_kernel<KC_, TB_, WT_, NN_, PB_, true>                 \
                  : (const void *)fwbf::cdecode_kernel<KC_, TB_, WT_, NN_, PB_, false>;               \
      clayout = layout_c<KC_, TB_, WT_, NN_, PB_>;                                                  \
    }
    FWBF_CIRC_CONFIGS(FWBF_PICK_C)
#undef FWBF_PICK_C
  }
  const bool compact = circ && sizeof(YT) == 4 && c->w <= 32 && !getenv("FWBF_NO_COMPACT");
  // staged input rows (TMA bulk copy one frame ahead): compile-time-shape
  // circulant float32 kernels; rows must be 16-byte aligned and hold the
  // rounded-up copy size
  const long long row_bytes = ld * (long long)sizeof(YT);
  // Staging claims the frame queue one frame ahead, so a CTA holding a slow
  // frame also holds its next one: only worth it when the batch is many
  // frames per CTA (small batches are latency-bound and lose their tail).
  bool ystage = !ckern && circ && sizeof(YT) == 4 && kwt > 0 && !metric_out && !getenv("FWBF_NO_YSTAGE") &&
                ((uintptr_t)y % 16) == 0 && row_bytes % 16 == 0 &&
                ((c->n * (long long)sizeof(YT) + 15) & ~15LL) <= row_bytes &&
                (batch >= 128LL * c->sm_count || getenv("FWBF_FORCE_YSTAGE"));
  if (ystage && !compact) {
    // non-compact layouts swap their y buffer for the staging buffer: same size
  } else if (ystage) {
    // compact layouts add the staging buffer: only where it costs no CTA per SM
    // (the MODE 2 layout keeps 5 CTAs/SM; the exact-path layouts would drop from 4 to 3)
    KParams Q0 = P, Q1 = P;
    layout(c, p, (int)sizeof(YT), circ, T * kc, Q0, compact, P.fused, mode2, false, T);
    layout(c, p, (int)sizeof(YT), circ, T * kc, Q1, compact, P.fused, mode2, true, T);
    int occ0 = 0, occ1 = 0;
    rc = plan_occupancy(c->device, kern, T, Q0.smem_bytes, &occ0);
    if (!rc && Q1.smem_bytes <= c->smem_optin) rc = plan_occupancy(c->device, kern, T, Q1.smem_bytes, &occ1);
    if (rc) return rc;
    ystage = occ1 >= occ0 && occ1 > 0;
  }
  layout(c, p, (int)sizeof(YT), circ, T * kc, P, compact, P.fused, mode2, ystage, T);
  if (P.fused && P.smem_bytes > c->smem_optin) { // y must stay resident for the fused pass
    P.fused = 0;
    layout(c, p, (int)sizeof(YT), circ, T * kc, P, compact, false, mode2, ystage, T);
  }
  if (ystage) {
    P.y_stage = 1;
    P.alias_y = 1; // after frame init, y is re-read from HBM (the staging buffer holds the next frame)
  }
  {
    // FWBF block-argmax groups: odd p -> one thread per block (stride-p reads
    // across lanes are bank-conflict free); power-of-two p -> min(p, 32)
    // threads per block reading contiguously; otherwise one thread per block.
    int tpb = 1;
    const int pp = P.p;
    P.sel_spread = 0;
    if (pp > 1 && (pp & (pp - 1)) == 0) {
      // power-of-two p: up to 32 threads per block, but all blocks in one round
      // when the CTA has room (C, p = 64: 16 threads x 64 blocks)
      tpb = std::min(pp, 32);
      while (tpb > 1 && (long long)P.nblocks * tpb > T) tpb >>= 1;
      if (tpb < 4) tpb = std::min(pp, 4);
    } else if (pp > 1 && !(pp & 1)) {
      // p = 2^k * odd: groups of 2^k (<= 16) threads on consecutive blocks start
      // at distinct multiples of 2^k modulo 16 banks-of-doubles: conflict free
      tpb = std::min(16, pp & -pp);
      while (tpb > 1 && (long long)P.nblocks * tpb > T) tpb >>= 1; // one round when possible
    } else if (pp & 1) {
      // largest power of two <= min(16, p) with all blocks in one round and
      // the half-warps of the CTA divisible into groups of tpb
      const int halfwarps = T / 16;
      for (int t2 = 16; t2 >= 2; t2 >>= 1)
        if (t2 <= pp && halfwarps % t2 == 0 && (long long)P.nblocks * t2 <= T) { tpb = t2; break; }
      P.sel_spread = tpb > 1;
    }
    P.log2_tpb = 0;
    while ((1 << P.log2_tpb) < tpb) ++P.log2_tpb;
  }
  if (P.smem_bytes > c->smem_optin && !compact && !ystage) {
    // Alias the metric buffer over the y buffer: after init y is only needed
    // for alpha*|y|, which the kernel then re-reads from global memory.
    P.alias_y = 1;
    const int delta = (P.off_y + align16(c->n * 8)) - P.off_chk1;
    P.off_e = P.off_y;
    for (int *x : {&P.off_chk1, &P.off_chk2, &P.off_amin, &P.off_amask, &P.off_sbits, &P.off_zbits,
                   &P.off_blkv, &P.off_blki, &P.off_flips, &P.off_offs, &P.off_red, &P.off_misc,
                   &P.off_fa, &P.off_fb, &P.off_m2s, &P.off_a2m, &P.off_corr, &P.off_ay, &P.off_ystage})
      *x += delta;
    P.smem_bytes += delta;
  }
  if (circ) {
    // column n (even) reads check (n - c_j) mod N at float index n + N - c_j of
    // the min1 copy whose pairs are 8-byte aligned for that parity
    for (int j = 0; j < c->w; ++j) {
      const int d = c->n - c->off[j];
      P.uoff[j] = ((d & 1) ? P.off_fb + 4 : P.off_fa) + 4 * d;
    }
  }
  if (const char *e = getenv("FWBF_SMEM_PAD")) P.smem_bytes += atoi(e); // tuning: occupancy sensitivity
  if (P.smem_bytes > c->smem_optin)
    return fail(FWBF_EUNSUPPORTED, "frame state needs %d B of shared memory (device max %d)",
                P.smem_bytes, c->smem_optin);
  int per_sm = 0;
  rc = plan_occupancy(c->device, kern, T, P.smem_bytes, &per_sm);
  if (rc) return rc;
  if (per_sm < 1) return fail(FWBF_EUNSUPPORTED, "kernel does not fit on an SM");
  const long long grid = std::min<long long>(batch, (long long)per_sm * c->sm_count);
  static long long *phase_buf = nullptr;
  const bool phases = getenv("FWBF_PHASES") != nullptr;
  if (phases) {
    if (!phase_buf) CUDA_TRY(cudaMalloc((void **)&phase_buf, 8 * sizeof(long long)));
    CUDA_TRY(cudaMemsetAsync(phase_buf, 0, 8 * sizeof(long long), stream));
    P.phase_cycles = phase_buf;
  }
  if (ckern) {
    KParams Q = P; // the filtered circulant kernel's own layout, TMA-staged rows when they qualify
    clayout(Q);
    const long long row_bytes = ld * (long long)sizeof(YT);
    Q.y_stage = Q.ystage_bytes > 0 && !getenv("FWBF_NO_YSTAGE") && ((uintptr_t)y % 16) == 0 && row_bytes % 16 == 0 &&
                (long long)Q.ystage_bytes <= row_bytes &&
                (batch >= 128LL * c->sm_count || getenv("FWBF_FORCE_YSTAGE"));
    Q.alias_y = 0;
    for (int j = 0; j < c->w; ++j) {
      const int d = c->n - c->off[j];
      Q.uoff[j] = ((d & 1) ? Q.off_fb + 4 : Q.off_fa) + 4 * d;
      // Q16: int16 arrays QA (doubled) and QB (shifted one element) share the FB region
      Q.uoff16[j] = (d & 1) ? Q.off_fb + (Q.off_m2s - Q.off_fb) / 2 + 2 * (d + 1) : Q.off_fb + 2 * d;
      const int cj = c->off[j]; // check scan: keys of columns (m + c_j, m + 1 + c_j), m even
      Q.soff[j] = (cj & 1) ? Q.off_fb + 4 * (cj + 1) : Q.off_fa + 4 * cj;
    }
    int cper = 0;
    if (Q.smem_bytes <= c->smem_optin) {
      rc = plan_occupancy(c->device, ckern, T, Q.smem_bytes, &cper);
      if (rc) return rc;
    }
    if (cper >= 1) {
      // frames outside the filtered guard are appended to a list and
      // decoded by decode_kernel afterwards; three adjacent queue slots, one
      // memset: this kernel's frame queue, the defer count, decode_kernel's
      // queue over the list
      unsigned *trio = c->d_work + (c->work_slot.fetch_add(3) % (kWorkRing - 2));
      CUDA_TRY(cudaMemsetAsync(trio, 0, 3 * sizeof(unsigned), stream));
      Q.work_counter = trio;
      unsigned *dcount = trio + 1;
      unsigned *lwork = trio + 2;
      int *dlist = nullptr;
      static std::once_flag pool_once[64];
      std::call_once(pool_once[c->device & 63], [&] {
        // keep freed blocks in the device's default pool: the per-launch
        // defer list is then a pool hit, not a fresh mapping every call
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) {
          uint64_t keep = ~0ull;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
      });
      CUDA_TRY(cudaMallocAsync((void **)&dlist, (size_t)batch * sizeof(int), stream));
      Q.defer_list = dlist;
      Q.defer_count = dcount;
      const long long cgrid = std::min<long long>(batch, (long long)cper * c->sm_count);
      void *cargs[] = {&Q};
      CUDA_TRY(cudaLaunchKernel(ckern, dim3((unsigned)cgrid), dim3(T), cargs, Q.smem_bytes, stream));
      CUDA_TRY(cudaGetLastError());
      if (phases) {
        long long h[8];
        CUDA_TRY(cudaMemcpyAsync(h, phase_buf, sizeof h, cudaMemcpyDeviceToHost, stream));
        CUDA_TRY(cudaStreamSynchronize(stream));
        long long tot = 0;
        for (int i = 0; i < 5; ++i) tot += h[i];
        static const char *names[5] = {"outputs+fetch", "init", "gather", "select", "toggles+refresh"};
        fprintf(stderr, "[fwbf phases] cdecode grid=%lld T=%d smem=%d:", cgrid, T, Q.smem_bytes);
        for (int i = 0; i < 5; ++i) fprintf(stderr, " %s %.1f%%", names[i], tot ? 100.0 * h[i] / tot : 0.0);
        fprintf(stderr, "\n");
        P.phase_cycles = nullptr;
      }
      P.frame_list = dlist;
      P.frame_count = dcount;
      P.work_counter = lwork;
      void *args[] = {&P};
      cudaStream_t s2 = stream;
      if (dstream && dev && dstream != stream) {
        CUDA_TRY(cudaEventRecord(dev, stream));
        CUDA_TRY(cudaStreamWaitEvent(dstream, dev, 0));
        s2 = dstream;
      }
      CUDA_TRY(cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(T), args, P.smem_bytes, s2));
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaFreeAsync(dlist, s2));
      g_last_kernel = "cdecode+decode_kernel";
      return FWBF_OK;
    }
  }
  CUDA_TRY(cudaMemsetAsync(P.work_counter, 0, sizeof(unsigned), stream));
  void *args[] = {&P};
  CUDA_TRY(cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(T), args, P.smem_bytes, stream));
  CUDA_TRY(cudaGetLastError());
  g_last_kernel = "decode_kernel";
  if (phases) {
    long long h[8];
    CUDA_TRY(cudaMemcpyAsync(h, phase_buf, sizeof h, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    long long tot = 0;
    for (int i = 0; i < 8; ++i) tot += h[i];
    static const char *names[8] = {"outputs+fetch", "init1", "init2", "gather", "select+apply",
                                   "post+refresh", "-", "-"};
    fprintf(stderr, "[fwbf phases] grid=%lld T=%d smem=%d:", grid, T, P.smem_bytes);
    for (int i = 0; i < 6; ++i) fprintf(stderr, " %s %.1f%%", names[i], tot ? 100.0 * h[i] / tot : 0.0);
    fprintf(stderr, "\n");
  }
  return FWBF_OK;
}

extern "C" int fwbf_filter_stats(fwbf_code *c, int64_t *out, int32_t reset) {
  if (!c || !out) return fail(FWBF_EINVAL, "null argument");
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  unsigned long long h[2];
  CUDA_TRY(cudaMemcpy(h, c->d_fstats, sizeof h, cudaMemcpyDeviceToHost));
  out[0] = (int64_t)h[0];
  out[1] = (int64_t)h[1];
  if (reset) CUDA_TRY(cudaMemset(c->d_fstats, 0, sizeof h));
  return FWBF_OK;
}

extern "C" int fwbf_decode_f32(fwbf_code *c, const fwbf_params *p, const float *y, int64_t batch,
                               int64_t ld, const fwbf_outputs *out, void *stream) {
  return launch_decode<float>(c, p, y, batch, ld, out, (cudaStream_t)stream);
}

extern "C" int fwbf_decode_f64(fwbf_code *c, const fwbf_params *p, const double *y, int64_t batch,
                               int64_t ld, const fwbf_outputs *out, void *stream) {
  return launch_decode<double>(c, p, y, batch, ld, out, (cudaStream_t)stream);
}

template <typename YT>
static int metric_t(fwbf_code *c, const fwbf_params *p, const YT *y, int64_t batch, int64_t ld, double *metric,
                    int64_t metric_ld, uint8_t *flags, void *stream) {
  if (!c) return fail(FWBF_EINVAL, "code is null");
  if (batch > 0 && !metric) return fail(FWBF_EINVAL, "metric is null");
  if (metric_ld < c->n) return fail(FWBF_EINVAL, "metric_ld must be at least n (%d)", c->n);
  fwbf_outputs o{};
  o.flags = flags;
  return launch_decode<YT>(c, p, y, batch, ld, &o, (cudaStream_t)stream, metric, metric_ld);
}

extern "C" int fwbf_metric_f32(fwbf_code *c, const fwbf_params *p, const float *y, int64_t batch, int64_t ld,
                               double *metric, int64_t metric_ld, uint8_t *flags, void *stream) {
  return metric_t<float>(c, p, y, batch, ld, metric, metric_ld, flags, stream);
}

extern "C" int fwbf_metric_f64(fwbf_code *c, const fwbf_params *p, const double *y, int64_t batch, int64_t ld,
                               double *metric, int64_t metric_ld, uint8_t *flags, void *stream) {
  return metric_t<double>(c, p, y, batch, ld, metric, metric_ld, flags, stream);
}

// Reference-channel decode: per chunk, noise_kernel writes the chunk's
// channel values (numpy's stream, float64 or rounded to float32) to a scratch
// buffer (or to out->y_out), then the decode kernel consumes them.
template <typename YT>
static int decode_awgn_t(fwbf_code *c, const fwbf_params *p, uint64_t seed, int64_t first, int64_t count,
                         double sigma, const fwbf_outputs *out, cudaStream_t stream) {
  int rc = validate(c, p);
  if (rc) return rc;
  if (count < 0) return fail(FWBF_EINVAL, "count must be nonnegative");
  if (count == 0) return FWBF_OK;
  fwbf_outputs o = out ? *out : fwbf_outputs{};
  const int n = c->n;
  const long long ld = o.y_out ? o.y_out_ld : ((n + 3) / 4 * 4);
  if (o.y_out && ld < n) return fail(FWBF_EINVAL, "y_out_ld too small");
  // Scratch y: chunks rotate over three buffers and alternate between two
  // streams (the caller's and a library side stream), so a chunk's noise
  // generation and decode overlap the previous chunk's tail -- the frames that
  // run to K_max keep a few SMs busy while the rest would idle.  A chunk's
  // second launch (decode_kernel over the frames the filtered circulant kernel
  // deferred) goes on a third, high-priority stream: behind the other
  // stream's persistent grid it would find no slot until that grid drained and
  // hold this stream's next chunk back.  Its buffer is
  // free again three chunks later.
  long long chunk = std::min<long long>(count, o.y_out ? (1 << 18) : (1 << 17));
  const int bf = o.batch_word_err ? std::max(1, o.batch_frames) : 1;
  chunk = std::max<long long>(bf, chunk / bf * bf);
  const bool two = !o.y_out && count > chunk;
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  YT *scratch = nullptr;
  // The library scratch for y is shared by every call on this handle: calls
  // are serialised on the host (lock held while enqueueing) and on the device
  // (each call's stream waits for the previous call's last use of it).
  std::unique_lock<std::mutex> lock(c->pipe_mu, std::defer_lock);
  if (!o.y_out) {
    lock.lock();
    if (!c->noise_evt) CUDA_TRY(cudaEventCreateWithFlags(&c->noise_evt, cudaEventDisableTiming));
    else CUDA_TRY(cudaStreamWaitEvent(stream, c->noise_evt, 0));
    const size_t need = (size_t)chunk * ld * sizeof(YT) * (two ? 3 : 1);
    if (need > c->noise_bytes) {
      if (c->noise_buf) cudaFree(c->noise_buf);
      c->noise_buf = nullptr;
      c->noise_bytes = 0;
      CUDA_TRY(cudaMalloc(&c->noise_buf, need));
      c->noise_bytes = need;
    }
    scratch = (YT *)c->noise_buf;
  }
  // raw draws prefetched per frame: about N (1 + 1/16) + 64 cover a frame
  const int pm = ((n + n / 16 + 64) + 3) & ~3;
  const int smem = pm * 8;
  auto nk = fwbf::noise_kernel<YT>;
  CUDA_TRY(cudaFuncSetAttribute((const void *)nk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const long long kmax = p->k_max;
  const long long maxf = fwbf_max_flips_per_iter(c, p);
  if (two) {
    if (!c->noise_side) CUDA_TRY(cudaStreamCreateWithFlags(&c->noise_side, cudaStreamNonBlocking));
    if (!c->noise_fork) CUDA_TRY(cudaEventCreateWithFlags(&c->noise_fork, cudaEventDisableTiming));
    if (!c->noise_join) CUDA_TRY(cudaEventCreateWithFlags(&c->noise_join, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(c->noise_fork, stream)); // the side stream starts after the caller's prior work
    CUDA_TRY(cudaStreamWaitEvent(c->noise_side, c->noise_fork, 0));
    if (!c->noise_def) {
      int lo = 0, hi = 0;
      CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CUDA_TRY(cudaStreamCreateWithPriority(&c->noise_def, cudaStreamNonBlocking, hi));
    }
    if (!c->noise_join2) CUDA_TRY(cudaEventCreateWithFlags(&c->noise_join2, cudaEventDisableTiming));
    for (int i = 0; i < 3; ++i) {
      if (!c->noise_cev[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->noise_cev[i], cudaEventDisableTiming));
      if (!c->noise_dev[i]) CUDA_TRY(cudaEventCreateWithFlags(&c->noise_dev[i], cudaEventDisableTiming));
    }
  }
  const cudaStream_t caller = stream;
  long long ci = 0;
  for (long long s = 0; s < count; s += chunk, ++ci) {
    const long long nb = std::min(chunk, count - s);
    stream = (two && (ci & 1)) ? c->noise_side : caller;
    const int b3 = (int)(ci % 3);
    if (two && ci >= 3) CUDA_TRY(cudaStreamWaitEvent(stream, c->noise_dev[b3], 0)); // chunk ci - 3 is done with the buffer
    YT *yb = o.y_out ? (YT *)o.y_out + s * ld : scratch + (two ? b3 * chunk * ld : 0);
    static const bool cta_gen = getenv("FWBF_NOISE_CTA") != nullptr; // the CTA-per-frame generator
    if (cta_gen) {
      const int grid = (int)std::min<long long>(nb, (long long)c->sm_count * 32);
      nk<<<grid, 128, smem, stream>>>((unsigned long long)seed, first + s, nb, sigma, o.codeword_bits, yb, ld, n,
                                      pm);
    } else { // one frame per warp, 4 per CTA
      const int grid = (int)std::min<long long>((nb + 3) / 4, (long long)c->sm_count * 16);
      fwbf::noise_kernel_warp<YT><<<grid, 128, 0, stream>>>((unsigned long long)seed, first + s, nb, sigma,
                                                            o.codeword_bits, yb, ld, n);
    }
    CUDA_TRY(cudaGetLastError());
    fwbf_outputs oc = o;
    if (o.z_bits) oc.z_bits = o.z_bits + s * o.z_ld;
    if (o.iterations) oc.iterations = o.iterations + s;
    if (o.flags) oc.flags = o.flags + s;
    if (o.flips_total) oc.flips_total = o.flips_total + s;
    if (o.bit_errors) oc.bit_errors = o.bit_errors + s;
    if (o.fliplog) {
      oc.fliplog = o.fliplog + s * o.fliplog_stride;
      oc.fliplog_counts = o.fliplog_counts + s * kmax;
    }
    if (o.batch_word_err) oc.batch_word_err = o.batch_word_err + s / bf;
    (void)maxf;
    if (two) {
      rc = launch_decode<YT>(c, p, yb, nb, ld, &oc, stream, nullptr, 0, c->noise_def, c->noise_cev[b3]);
      if (rc) return rc;
      // the chunk is done when everything on its stream and, after it, on the deferred stream is
      CUDA_TRY(cudaEventRecord(c->noise_cev[b3], stream));
      CUDA_TRY(cudaStreamWaitEvent(c->noise_def, c->noise_cev[b3], 0));
      CUDA_TRY(cudaEventRecord(c->noise_dev[b3], c->noise_def));
    } else {
      rc = launch_decode<YT>(c, p, yb, nb, ld, &oc, stream);
      if (rc) return rc;
    }
  }
  stream = caller;
  if (two) { // join: the caller's stream waits for the side and deferred streams' chunks
    CUDA_TRY(cudaEventRecord(c->noise_join, c->noise_side));
    CUDA_TRY(cudaStreamWaitEvent(stream, c->noise_join, 0));
    CUDA_TRY(cudaEventRecord(c->noise_join2, c->noise_def));
    CUDA_TRY(cudaStreamWaitEvent(stream, c->noise_join2, 0));
  }
  if (!o.y_out) CUDA_TRY(cudaEventRecord(c->noise_evt, stream));
  return FWBF_OK;
}

extern "C" int fwbf_decode_awgn(fwbf_code *c, const fwbf_params *p, uint64_t seed, int64_t first,
                                int64_t count, double sigma, int32_t mode, const fwbf_outputs *out,
                                void *stream) {
  if (first < 0) return fail(FWBF_EINVAL, "seed and frame index must be nonnegative");
  if (!(sigma >= 0)) return fail(FWBF_EINVAL, "sigma must be nonnegative");
  if (mode == FWBF_NOISE_NUMPY_F64)
    return decode_awgn_t<double>(c, p, seed, first, count, sigma, out, (cudaStream_t)stream);
  if (mode == FWBF_NOISE_NUMPY_F32)
    return decode_awgn_t<float>(c, p, seed, first, count, sigma, out, (cudaStream_t)stream);
  return fail(FWBF_EINVAL, "unknown noise mode %d", mode);
}

// ---------------------------------------------------------------------------
// Host-buffer pipeline: chunked H2D -> decode -> D2H on two streams.
// ---------------------------------------------------------------------------
extern "C" int fwbf_decode_host_f32(fwbf_code *c, const fwbf_params *p, const float *y_host,
                                    int64_t batch, int64_t ld, uint32_t *z_host, int64_t z_ld,
                                    int32_t *it_host, uint8_t *fl_host, int64_t *cnt_host,
                                    int64_t chunk) {
  int rc = validate(c, p);
  if (rc) return rc;
  if (batch < 0) return fail(FWBF_EINVAL, "batch must be nonnegative");
  if (batch == 0) return FWBF_OK;
  if (!y_host) return fail(FWBF_EINVAL, "y is null");
  if (ld < c->n) return fail(FWBF_EINVAL, "expected a length-%d frame (ld=%lld)", c->n, (long long)ld);
  const int zw = (c->n + 31) / 32;
  if (z_host && z_ld < zw) return fail(FWBF_EINVAL, "z_ld too small");
  // default chunk: about 64 MB of y per buffer (2^14 frames of EG(1023)): with the chunks' drains
  // overlapped (below) small chunks cost nothing and shorten the pipeline's fill and flush
  if (chunk <= 0) chunk = std::max<int64_t>(1024, (int64_t)(64 << 20) / (ld * (int64_t)sizeof(float)));
  chunk = std::min<int64_t>(chunk, batch);
  std::lock_guard<std::mutex> lock(c->pipe_mu);
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  // per-chunk buffer: y chunk | z chunk | iterations | flags
  const size_t yb = (size_t)chunk * ld * sizeof(float);
  const size_t zb = (size_t)chunk * zw * sizeof(uint32_t);
  const size_t ib = (size_t)chunk * sizeof(int32_t);
  const size_t fb = (size_t)chunk;
  const size_t need = align16((int)0) + yb + zb + ib + fb + 64;
  constexpr int NBUF = 4;
  if (need > c->pipe_bytes) {
    for (int i = 0; i < NBUF; ++i) {
      if (c->pipe_buf[i]) cudaFree(c->pipe_buf[i]);
      c->pipe_buf[i] = nullptr;
    }
    c->pipe_bytes = 0;
    for (int i = 0; i < NBUF; ++i) CUDA_TRY(cudaMalloc(&c->pipe_buf[i], need));
    c->pipe_bytes = need;
  }
  if (!c->pipe_s[0]) {
    int lo = 0, hi = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int i = 0; i < 5; ++i) // [3]: the deferred-frame launches, ahead of the main kernels' pending CTAs
      CUDA_TRY(cudaStreamCreateWithPriority(&c->pipe_s[i], cudaStreamNonBlocking, i == 3 ? hi : lo));
  }
  for (int i = 0; i < 4; ++i)
    for (int b = 0; b < NBUF; ++b)
      if (!c->pipe_ev[i][b]) CUDA_TRY(cudaEventCreateWithFlags(&c->pipe_ev[i][b], cudaEventDisableTiming));
  if (!c->pipe_counters) CUDA_TRY(cudaMalloc((void **)&c->pipe_counters, FWBF_NCOUNTERS * sizeof(int64_t)));
  CUDA_TRY(cudaMemsetAsync(c->pipe_counters, 0, FWBF_NCOUNTERS * sizeof(long long), c->pipe_s[1]));
  CUDA_TRY(cudaStreamSynchronize(c->pipe_s[1]));
  // Five streams ordered by per-buffer events: H2D copies; the chunks' main
  // decode kernels alternating between two streams, so chunk i+1's
  // persistent grid is already queued when chunk i's CTAs run out of frames
  // and takes over the SMs they leave (a chunk's last frames -- the ones that
  // run all K_max iterations -- otherwise drain on a mostly idle GPU: 0.8 ms
  // of a 15 ms chunk, measured); the second launch of a chunk (decode_kernel
  // over the frames the filtered kernel deferred) on its own high-priority
  // stream, where it waits for a slot instead of holding the next main kernel
  // back; D2H copies.  A chunk's buffer is reused four chunks later.
  cudaStream_t sin = c->pipe_s[0], sdef = c->pipe_s[3], sout = c->pipe_s[4];
  // chunk sizes ramp up geometrically (chunk/16, chunk/8, ... chunk) so the
  // first decode starts after a short copy instead of a full chunk's
  long long f0 = 0, cur = std::max<long long>(std::min<long long>(chunk, 4096), chunk / 16);
  for (long long ci = 0; f0 < batch; ++ci) {
    const int s = (int)(ci % NBUF);
    cudaStream_t sdec = c->pipe_s[1 + (ci & 1)];
    char *base = (char *)c->pipe_buf[s];
    float *dy = (float *)base;
    uint32_t *dz = (uint32_t *)(base + yb);
    int32_t *dit = (int32_t *)(base + yb + zb);
    uint8_t *dfl = (uint8_t *)(base + yb + zb + ib);
    const long long nb = std::min<long long>(cur, batch - f0);
    if (ci >= NBUF) CUDA_TRY(cudaStreamWaitEvent(sin, c->pipe_ev[3][s], 0)); // chunk ci-4 decoded and copied out
    CUDA_TRY(cudaMemcpyAsync(dy, y_host + f0 * ld, (size_t)nb * ld * sizeof(float), cudaMemcpyHostToDevice, sin));
    CUDA_TRY(cudaEventRecord(c->pipe_ev[0][s], sin));
    CUDA_TRY(cudaStreamWaitEvent(sdec, c->pipe_ev[0][s], 0));
    fwbf_outputs o{};
    o.z_bits = z_host ? dz : nullptr;
    o.z_ld = zw;
    o.iterations = it_host ? dit : nullptr;
    o.flags = fl_host ? dfl : nullptr;
    o.counters = c->pipe_counters;
    rc = launch_decode<float>(c, p, dy, nb, ld, &o, sdec, nullptr, 0, sdef, c->pipe_ev[1][s]);
    if (rc) return rc;
    // the chunk is decoded when everything on sdec and, after it, on sdef is done
    CUDA_TRY(cudaEventRecord(c->pipe_ev[1][s], sdec));
    CUDA_TRY(cudaStreamWaitEvent(sdef, c->pipe_ev[1][s], 0));
    CUDA_TRY(cudaEventRecord(c->pipe_ev[2][s], sdef));
    CUDA_TRY(cudaStreamWaitEvent(sout, c->pipe_ev[2][s], 0));
    if (z_host) {
      if (z_ld == zw) {
        CUDA_TRY(cudaMemcpyAsync(z_host + f0 * z_ld, dz, (size_t)nb * zw * 4, cudaMemcpyDeviceToHost, sout));
      } else {
        CUDA_TRY(cudaMemcpy2DAsync(z_host + f0 * z_ld, (size_t)z_ld * 4, dz, (size_t)zw * 4, (size_t)zw * 4,
                                   (size_t)nb, cudaMemcpyDeviceToHost, sout));
      }
    }
    if (it_host) CUDA_TRY(cudaMemcpyAsync(it_host + f0, dit, (size_t)nb * 4, cudaMemcpyDeviceToHost, sout));
    if (fl_host) CUDA_TRY(cudaMemcpyAsync(fl_host + f0, dfl, (size_t)nb, cudaMemcpyDeviceToHost, sout));
    CUDA_TRY(cudaEventRecord(c->pipe_ev[3][s], sout));
    f0 += nb;
    cur = std::min<long long>(chunk, 2 * cur);
  }
  for (int i = 0; i < 5; ++i) CUDA_TRY(cudaStreamSynchronize(c->pipe_s[i]));
  if (cnt_host) {
    long long tmp[FWBF_NCOUNTERS];
    CUDA_TRY(cudaMemcpy(tmp, c->pipe_counters, sizeof tmp, cudaMemcpyDeviceToHost));
    for (int i = 0; i < FWBF_NCOUNTERS; ++i) cnt_host[i] += tmp[i];
  }
  return FWBF_OK;
}

// ---------------------------------------------------------------------------
// Stage views (fwbf_stage.cu): the reference's per-stage functions, batched.
// ---------------------------------------------------------------------------
static int stage_grid(long long items) {
  const long long g = (items + 255) / 256;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 64));
}

#define STAGE_LAUNCH(kern, items, stream, ...)                                       \
  do {                                                                               \
    if ((items) > 0) {                                                               \
      fwbf::kern<<<stage_grid(items), 256, 0, (cudaStream_t)(stream)>>>(__VA_ARGS__); \
      CUDA_TRY(cudaGetLastError());                                                  \
    }                                                                                \
  } while (0)

extern "C" int fwbf_stage_hard_decision(int32_t dtype, const void *y, int64_t count, uint8_t *z, void *stream) {
  if (count < 0) return fail(FWBF_EINVAL, "count must be nonnegative");
  if (count && (!y || !z)) return fail(FWBF_EINVAL, "null buffer");
  if (dtype == 4) STAGE_LAUNCH(stage_hard_decision<float>, count, stream, (const float *)y, count, z);
  else if (dtype == 8) STAGE_LAUNCH(stage_hard_decision<double>, count, stream, (const double *)y, count, z);
  else return fail(FWBF_EINVAL, "dtype must be 4 (float32) or 8 (float64)");
  return FWBF_OK;
}

extern "C" int fwbf_stage_syndrome(fwbf_code *c, const uint8_t *z, int64_t batch, uint8_t *s, void *stream) {
  if (!c) return fail(FWBF_EINVAL, "null code");
  if (batch < 0) return fail(FWBF_EINVAL, "batch must be nonnegative");
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  STAGE_LAUNCH(stage_syndrome, batch * c->m, stream, c->d_row_ptr, c->d_row_idx, c->n, c->m, z, (long long)batch, s);
  return FWBF_OK;
}

extern "C" int fwbf_stage_weights(fwbf_code *c, const double *y, int64_t batch, int64_t ld, double *min1,
                                  double *min2, int64_t *argmin_col, double *edge_w, void *stream) {
  if (!c) return fail(FWBF_EINVAL, "null code");
  if (c->m && c->min_row_w < 2) return fail(FWBF_EINVAL, "every check must contain at least 2 bits");
  if (batch < 0) return fail(FWBF_EINVAL, "batch must be nonnegative");
  if (ld < c->n) return fail(FWBF_EINVAL, "expected a length-%d frame", c->n);
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  STAGE_LAUNCH(stage_weights, batch * c->m, stream, c->d_row_ptr, c->d_row_idx, c->m, c->n_edges, y,
               (long long)batch, (long long)ld, min1, min2, (long long *)argmin_col, edge_w);
  return FWBF_OK;
}

extern "C" int fwbf_stage_edge_weights(fwbf_code *c, const double *min1, const double *min2,
                                       const int64_t *argmin_col, int64_t batch, double *edge_w, void *stream) {
  if (!c) return fail(FWBF_EINVAL, "null code");
  if (batch < 0) return fail(FWBF_EINVAL, "batch must be nonnegative");
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  STAGE_LAUNCH(stage_edge_weights, batch * c->m, stream, c->d_row_ptr, c->d_row_idx, c->m, c->n_edges, min1, min2,
               (const long long *)argmin_col, (long long)batch, edge_w);
  return FWBF_OK;
}

extern "C" int fwbf_stage_all_metrics(fwbf_code *c, const uint8_t *syndrome, const double *edge_w,
                                      const double *abs_y, double alpha, int64_t batch, double *out,
                                      void *stream) {
  if (!c) return fail(FWBF_EINVAL, "null code");
  if (batch < 0) return fail(FWBF_EINVAL, "batch must be nonnegative");
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  STAGE_LAUNCH(stage_all_metrics, batch * c->n, stream, c->d_col_ptr, c->d_col_idx, c->d_col_eid, c->n, c->m,
               c->n_edges, syndrome, edge_w, abs_y, alpha, (long long)batch, out);
  return FWBF_OK;
}

extern "C" int fwbf_stage_block_argmax(const double *values, int64_t batch, int64_t n, int64_t ld,
                                       int32_t p, int64_t *out, void *stream) {
  if (p < 1) return fail(FWBF_EINVAL, "block length p must be >= 1");
  if (batch < 0 || n < 0 || ld < n) return fail(FWBF_EINVAL, "bad shape");
  if (n > 0x7fffffffLL) return fail(FWBF_EUNSUPPORTED, "vector too long");
  if (n == 0) return FWBF_OK;
  const int nb = (int)((n + p - 1) / p);
  STAGE_LAUNCH(stage_block_argmax, batch * nb, stream, values, (long long)batch, (int)n, (long long)ld, (int)p,
               nb, (long long *)out);
  return FWBF_OK;
}

extern "C" int fwbf_stage_bit_metric(fwbf_code *c, const int32_t *cols, int32_t k, const uint8_t *syndrome,
                                     const double *min1, const double *min2, const int64_t *argmin_col,
                                     const double *y, double alpha, double *out, void *stream) {
  if (!c) return fail(FWBF_EINVAL, "null code");
  if (k < 0) return fail(FWBF_EINVAL, "k must be nonnegative");
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  STAGE_LAUNCH(stage_bit_metric, (long long)k, stream, c->d_col_ptr, c->d_col_idx, cols, k, syndrome, min1, min2,
               (const long long *)argmin_col, y, alpha, out);
  return FWBF_OK;
}

// The reference channel alone (no decode): y[f][n] for frames
// first..first+count, numpy's stream (fwbf_noise.cuh), float64 or float32.
extern "C" int fwbf_channel_awgn(fwbf_code *c, uint64_t seed, int64_t first, int64_t count, double sigma,
                                 const uint32_t *codeword_bits, int32_t noise_mode, void *y, int64_t ld,
                                 void *stream) {
  if (!c) return fail(FWBF_EINVAL, "null code");
  if (first < 0 || count < 0) return fail(FWBF_EINVAL, "seed and frame index must be nonnegative");
  if (!(sigma >= 0)) return fail(FWBF_EINVAL, "sigma must be nonnegative");
  if (ld < c->n) return fail(FWBF_EINVAL, "ld too small");
  if (count == 0) return FWBF_OK;
  if (!y) return fail(FWBF_EINVAL, "y is null");
  DeviceGuard dg;
  CUDA_TRY(cudaSetDevice(c->device));
  const int grid = (int)std::min<long long>((count + 3) / 4, (long long)c->sm_count * 16);
  if (noise_mode == FWBF_NOISE_NUMPY_F64)
    fwbf::noise_kernel_warp<double><<<grid, 128, 0, (cudaStream_t)stream>>>(
        (unsigned long long)seed, first, count, sigma, codeword_bits, (double *)y, ld, c->n);
  else if (noise_mode == FWBF_NOISE_NUMPY_F32)
    fwbf::noise_kernel_warp<float><<<grid, 128, 0, (cudaStream_t)stream>>>(
        (unsigned long long)seed, first, count, sigma, codeword_bits, (float *)y, ld, c->n);
  else
    return fail(FWBF_EINVAL, "unknown noise mode %d", noise_mode);
  CUDA_TRY(cudaGetLastError());
  return FWBF_OK;
}
