// fwbf_internal.h -- kernel parameter block shared by the launcher and kernels.
#pragma once
#include <stdint.h>

namespace fwbf {

constexpr int kMaxCircWeight = 64; // circulant offsets kept in the parameter block
constexpr int kMaxQcBlocks = 256;  // quasi-cyclic shift table entries in the parameter block

// Guarded-path kernel shapes (threads TB, columns per thread KC): TB*KC >= n.
// WT > 0: circulant weight fixed at compile time (fully unrolled gather).
#define FWBF_FAST_CONFIGS(X)    \
  X(float, true, 2, 128, 16)    \
  X(float, true, 4, 256, 32)    \
  X(float, true, 4, 1024, 64)   \
  X(float, true, 2, 128, 0)     \
  X(float, true, 4, 256, 0)     \
  X(float, true, 4, 512, 0)     \
  X(float, true, 8, 512, 0)     \
  X(float, true, 8, 1024, 0)

// compile-time-weight shapes that also exist as MODE 1 (IMWBF, one flip per
// iteration, incremental integer metric) and MODE 2 (FWBF, filtered metric)
#define FWBF_INC_CONFIGS(X)     \
  X(float, true, 2, 128, 16)    \
  X(float, true, 4, 256, 32)    \
  X(float, true, 4, 1024, 64)

// float64 input (ordered path only) with the circulant weight compiled in
#define FWBF_F64_CONFIGS(X)     \
  X(double, true, 2, 128, 16)   \
  X(double, true, 4, 256, 32)   \
  X(double, true, 4, 1024, 64)

// Filtered FWBF kernel for cyclic EG codes (fwbf_circ.cu): (KC, TB, WT, N),
// the code length and weight compiled in (EG(255), EG(1023), EG(4095)).
// PB > 0: the FWBF block length compiled in as well (0: any p >= 16);
// PB = -1: MLP-WBF (top-lambda selection, lambda <= 31).
#define FWBF_CIRC_CONFIGS(X) \
  X(2, 128, 16, 255, 0)      \
  X(4, 256, 32, 1023, 0)     \
  X(4, 256, 32, 1023, 31)    \
  X(4, 1024, 64, 4095, 0)    \
  X(4, 1024, 64, 4095, 64)   \
  X(4, 1024, 64, 4095, 128)  \
  X(4, 1024, 64, 4095, 256)  \
  X(4, 256, 32, 1023, 93)    \
  X(2, 128, 16, 255, -1)     \
  X(4, 256, 32, 1023, -1)    \
  X(4, 1024, 64, 4095, -1)
constexpr int kCircMaxLam = 31; // MLP lists: lambda + 1 <= 32 entries per warp

// FWBF on EG(1023) (256 threads) runs 6 CTAs per SM at 40 registers without
// the staging buffer (4 KB less shared memory: 36.3 KB): +3 % over 5 CTAs
// with staged rows.  Other shapes keep the staging buffer.
template <int TB, int PB> struct CircShape {
  static constexpr bool kSix = TB == 256 && PB >= 0;
  static constexpr bool kStage = !kSix;
  static constexpr int kMinBlocks = TB == 256 ? (kSix ? 6 : 5) : 1024 / TB;
};

// Its shared-memory layout (byte offsets), a compile-time function of the code
// so every access in the kernel is [base + immediate]; the host reads the same
// constants (layout_c in fwbf_api.cu).  Blocks: p >= 16, so at most
// ceil(N / 16) of them.
template <int NN, int COVER, int WT, int LSTB = 0, bool STAGE = true> struct CLayout {
  static constexpr int al(int x) { return (x + 15) & ~15; }
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  static constexpr int EP = (NN + 1) & ~1;     // |y| after the metric (even: float2 reads)
  static constexpr int ZW = (NN + 31) / 32;    // words of a bit vector over N
  static constexpr int FDW = 2 * ZW + 2;       // doubled flip bitmap words (windows read one past 2N)
  static constexpr int NBMAX = (NN + 15) / 16;
  static constexpr int DBLF = (2 * NN + mx(0, COVER - NN) + 2 + 31) / 32 * 32;
  static constexpr int YST = 0;                // y row (TMA staging target), 16-byte aligned
  static constexpr int YSTB = STAGE ? al(NN * 4) : 0; // (none: the row is read from HBM)
  static constexpr int E = YST + YSTB;         // float metric [EP] + |y| [N]
  static constexpr int FA = E + al((EP + mx(NN, COVER)) * 4);
  static constexpr int FB = FA + al(DBLF * 4);
  static constexpr int M2 = FB + al(DBLF * 4);
  static constexpr int A2 = M2 + al(NN * 4);
  static constexpr int CORR = A2 + al(NN * 2);
  static constexpr int SB = CORR + al(mx(NN, COVER) * 4);
  static constexpr int ZB = SB + al(ZW * 4);
  static constexpr int FD = ZB + al(ZW * 4);
  static constexpr int BV = FD + al(2 * FDW * 4);
  static constexpr int BI = BV + al(NBMAX * 8);
  static constexpr int ROT = BI + al(NBMAX * 4);
  static constexpr int MISC = ROT + al(2 * WT * 4);
  static constexpr int LST = MISC + al(80 * 4); // MLP: per-warp candidate lists (LSTB bytes)
  static constexpr int BYTES = LST + al(LSTB);
};

struct KParams {
  // ---- code (H) ----
  int n, m;          // columns (bits), rows (checks)
  int w;             // circulant weight, 0 for explicit codes
  int dv_max;        // max column weight
  long long n_edges;
  int off[kMaxCircWeight];  // circulant first-row columns c_j, ascending
  int dneg[kMaxCircWeight]; // sorted (n - c_j) mod n, ascending (ordered column walk)
  unsigned char jii[kMaxCircWeight]; // offset index j -> its position in dneg
  const uint8_t *i0tab;     // circulant: first dneg index of column n's ascending walk
  const uint8_t *jwtab;     // circulant: first j with m + c_j >= n (check m's wrap point)
  const int16_t *offpos;    // circulant: offpos[d] = j if c_j == d else -1
  const int *row_ptr, *row_idx; // CSR, sorted columns
  const int *col_ptr, *col_idx; // CSC, ascending checks
  int qc_z, qc_jb, qc_kb;       // quasi-cyclic structure (qc_z = 0: none); Z a power of two
  short qc_shift[kMaxQcBlocks]; // [jb][kb] circulant shifts, -1 = zero block
  // ---- decoder config ----
  int alg, wmode, kmax, lam, p, stall, mlp_thr, force_ordered;
  double alpha;
  int nblocks;
  int log2_tpb; // FWBF: threads per block-argmax group = 2^log2_tpb
  int sel_spread; // odd p: half-warp groups take blocks TPB apart (bank-conflict free)
  // ---- input ----
  const void *y;
  long long ld;
  long long batch;
  // ---- outputs ----
  uint32_t *z_bits;
  long long z_ld;
  int *iterations;
  uint8_t *flags;
  int *flips_total;
  int *bit_errors;
  int *fliplog;
  int *fliplog_counts;
  long long fliplog_stride;
  long long *counters;
  long long *iter_hist;
  int *batch_word_err;
  int batch_frames;
  const uint32_t *codeword_bits;
  unsigned int *work_counter;
  long long *phase_cycles; // optional [8] per-phase cycle sums (FWBF_PHASES=1)
  // ---- shared memory layout (byte offsets) ----
  int off_y, off_e, off_chk1, off_chk2, off_amin, off_amask, off_sbits, off_zbits;
  int off_blkv, off_blki, off_flips, off_offs, off_red, off_misc;
  int smem_bytes;
  int alias_y; // metric buffer overlays y; alpha*|y| re-read from global
  int d21f;    // (unused)
  int off_fa, off_fb, off_m2s, off_a2m, off_corr, off_ay; // split-fp32 path arrays (inside the chk region)
  int has_ay; // split path keeps fl(alpha|y|) per column in shared memory (compact layout)
  int fused;  // explicit/QC FWBF with p % 32 == 0: metric + block argmax in one pass, no metric buffer
  double *metric_out;       // stage view: first-iteration metric per frame (then stop), or null
  long long metric_ld;
  int uoff[kMaxCircWeight]; // split-fp32 gather: byte offset of check (n - c_j) for even n, minus 4n
  int no_split; // disable the split-fp32 path (testing)
  int filter;   // FWBF on the split path: approximate fp32 gather + exact resolution of close decisions
  unsigned long long *filter_stats; // optional [2]: blocks resolved exactly, stall argmaxes resolved exactly
  // Input staging (circulant float32 kernels): the next frame's y row is
  // fetched by one cp.async.bulk (TMA bulk copy, completion on an mbarrier)
  // into a shared staging buffer while the current frame iterates; frame init
  // then reads y from shared memory instead of HBM.
  int y_stage;      // 1: enabled (16-byte aligned rows; ybuf = the staging buffer)
  int off_ystage;   // staging buffer byte offset (16-byte aligned)
  int ystage_bytes; // bytes per copy: N * sizeof(YT) rounded up to 16 (<= ld * sizeof(YT))
  // Frame lists (round 3).  The filtered circulant kernel (fwbf_circ.cu)
  // decodes the frames that pass its path guard and appends the others to
  // defer_list (count in *defer_count); decode_kernel then runs over that list
  // (frame_list / *frame_count) instead of 0..batch-1.
  int *defer_list;
  unsigned *defer_count;
  const int *frame_list;
  const unsigned *frame_count;
  int uoff16[kMaxCircWeight]; // fwbf_circ.cu Q16 gather: byte offset of the int16 pair of check (n - c_j), n even, minus 2n
  int soff[kMaxCircWeight]; // fwbf_circ.cu check scan: byte offset of the key pair of column m + c_j (m even), minus 4m
  int off_fd;  // fwbf_circ.cu: two doubled flip bitmaps (iteration parity)
  int fd_words; // words per flip bitmap
};

// One-frame-per-warp FWBF kernel for small explicit codes (fwbf_explicit.cu).
struct XParams {
  int n, m, n_edges;
  int nb, p, lg_g, rounds, slots; // blocks; lanes per block = 2^lg_g; slots per lane per round
  int kmax, stall, wmode;
  double alpha;
  // code tables built on the host per (code, p), copied to shared memory
  const unsigned long long *tab; // [rounds * slots * 32] per slot: 4 x u16 byte offsets of the column's check records
  const uint32_t *rtab;          // [E] row-major edge: slot of its column | (check position in the column) << 16
  const int *row_ptr;            // [m + 1]
  const uint16_t *cpos;          // [n] slot of column n
  const int *invp;               // [m] check stored under label j (labels spread bank pairs)
  int s2off, s2sh;               // min2 array offset in bytes (= 1 << s2sh) from the min1 array
  int off_tab, off_cpos, off_warp0, warp_bytes;
  int wo_rec, wo_ys, wo_am, wo_sb, wo_zw, wo_bf;
  // xinc_kernel (incremental variant): per check label the slots of its columns [m << dcs_sh] (0xffff = none),
  // per warp the stored metrics [nslot] floats and the toggled-check list
  const uint16_t *ctab;
  int off_ctab, dcs_sh, wo_ek, wo_tl;
  // input / outputs (as KParams)
  const float *y;
  long long ld;
  long long batch;
  int y_vec4;
  uint32_t *z_bits;
  long long z_ld;
  int *iterations;
  uint8_t *flags;
  int *flips_total;
  int *bit_errors;
  int *fliplog;
  int *fliplog_counts;
  long long fliplog_stride;
  long long *counters;
  long long *iter_hist;
  int *batch_word_err;
  int batch_frames;
  const uint32_t *codeword_bits;
  unsigned int *work_counter;
};

// Quasi-cyclic FWBF kernel (fwbf_qc.cu): one frame per CTA, fused metric + block argmax.
struct QParams {
  int n, m, n_edges;
  int z, lgz, jb, kb, head; // circulant size, log2, row / column blocks, doubled head (= p)
  short shift[kMaxQcBlocks]; // [jb][kb], -1 = zero block
  int nb;                    // blocks (p = 32 * TPC columns each)
  int kmax, stall, wmode;
  double alpha;
  int off_y, off_m1, off_m2, off_cmask, off_zrec, off_sbits, off_zbits, off_blkv, off_blki, off_misc;
  int off_blkk, off_blkf, off_list, off_sold, off_dirty; // qinc_kernel only: block keys, flip flags, toggled checks, previous syndrome
  const float *y;
  long long ld;
  long long batch;
  int y_vec4;
  uint32_t *z_bits;
  long long z_ld;
  int *iterations;
  uint8_t *flags;
  int *flips_total;
  int *bit_errors;
  int *fliplog;
  int *fliplog_counts;
  long long fliplog_stride;
  long long *counters;
  long long *iter_hist;
  int *batch_word_err;
  int batch_frames;
  const uint32_t *codeword_bits;
  unsigned int *work_counter;
};

} // namespace fwbf
