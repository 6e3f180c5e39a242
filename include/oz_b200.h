/* oz_b200.h — C ABI of the B200 Ozaki-scheme DGEMM (liboz_b200.so).
 *
 * The reference (arxiv 2508.00441, package `ozdgemm`, pure Python/numpy) has no
 * FFI; its drop-in boundary is the Python signature oz_gemm(A, B, cfg)
 * (pkg/src/ozdgemm/ozgemm.py:143) and its internal seams slice_matrix
 * (slicing.py:190), lp_gemm (lpgemm.py:93) and the pair-accumulation loop
 * (ozgemm.py:179-209).  Each entry point below replaces one of those seams;
 * the Python package paper_2508_00441_b200 binds them with ctypes and keeps the
 * reference's Python API on top.
 *
 * Conventions
 *   - all matrix pointers are DEVICE pointers, row-major, leading dimension in
 *     elements; the library never allocates or frees caller memory;
 *   - every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy);
 *   - kernels OR error bits into the device word *flags (OZ_FLAG_*); the caller
 *     reads it after a stream sync and maps it to the reference's exceptions;
 *   - return value: OZ_OK or an OZ_E* status (launch-time argument errors).
 *
 * type2 codes (slice storage format, formats.py:85-100):
 *   OZ_FMT_E4M3 = 0 (fp8e4m3), OZ_FMT_E5M2 = 1 (fp8e5m2), OZ_FMT_FP16 = 2, OZ_FMT_BF16 = 3,
 *   OZ_FMT_E3M2 = 4 (fp6e3m2), OZ_FMT_E2M3 = 5 (fp6e2m3) — FP6 planes are densely packed (6 bits per
 *   code, rows of ld*3/4 bytes, ld a multiple of 128)
 */
#ifndef OZ_B200_H
#define OZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OZ_OK = 0,
  OZ_EINVAL = 1,       /* bad argument (shape, pointer, format)              */
  OZ_EUNSUPPORTED = 2, /* format/size combination not implemented on sm_100a */
  OZ_ECUDA = 3,        /* CUDA runtime error at launch                        */
  OZ_ETMAP = 4,        /* cuTensorMapEncodeTiled failed                      */
  OZ_ESLICES = 5       /* reserved (earlier versions: slice-count limit)       */
};

enum { OZ_FMT_E4M3 = 0, OZ_FMT_E5M2 = 1, OZ_FMT_FP16 = 2, OZ_FMT_BF16 = 3, OZ_FMT_E3M2 = 4, OZ_FMT_E2M3 = 5 };

/* device error-flag bits */
#define OZ_FLAG_NONFINITE_INPUT (1u << 0)   /* slicing.py:120-121  -> ValueError        */
#define OZ_FLAG_SUBNORMAL_INPUT (1u << 1)   /* slicing.py:122-125  -> RangeError        */
#define OZ_FLAG_SIGMA_RANGE (1u << 2)       /* slicing.py:157-158  -> RangeError        */
#define OZ_FLAG_SLICE_CAP (1u << 3)         /* > planes / 2100 slices -> AssertionError */
#define OZ_FLAG_NOT_REPRESENTABLE (1u << 4) /* slicing.py:169-172  -> SlicingInfeasible */
#define OZ_FLAG_EMU_RANGE (1u << 5)         /* fp64emu.py:240-241  -> RangeError        */
#define OZ_FLAG_TERM_RANGE (1u << 6)        /* ozgemm.py:137-139   -> RangeError        */
#define OZ_FLAG_SUBNORMAL_RESID (1u << 7)   /* fp64emu.py:73-82    -> RangeError        */
#define OZ_FLAG_PLANE_CAP (1u << 8)         /* oz_split_fused: a row needs > cap planes (re-run two-pass) */

/* One-pass row split (the production path) — replaces slice_matrix(X, "rows",
 * ...) (slicing.py:190-198) / _slice_rows (slicing.py:128-177): writes each
 * row's slices as they are produced into coeff[cap][rows][ld_coeff] and
 * expo[cap][rows], the per-row counts row_cnt[rows] and *s_max = max(*s_max,
 * max_r row_cnt[r]) (the reference's s, slicing.py:206), plus the validation
 * and representability flags.  Planes [row_cnt[r], s) of a row are NOT written:
 * call oz_split_pad once s is known.  A row needing more than `cap` planes sets
 * OZ_FLAG_PLANE_CAP (outputs then incomplete: use oz_split_count +
 * oz_split_rows).  kb <= 131072 (clusters of CTAs share rows above 16384). */
int oz_split_fused(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int cap,
                   void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt, int32_t* s_max, uint32_t* flags,
                   void* stream);

/* Fixed-step variant of oz_split_fused (opt-in extension, no reference
 * counterpart; GemmConfig.slice_exponents = "fixed"): slice p of a row gets the
 * exponent c_p = c_0 - p (54 - rho), c_0 = ceil_log2 max|x| as in the reference,
 * instead of ceil_log2 of the residual's max (slicing.py:145-152).  The reference's
 * RN residual bound |x - v| <= 2^(c_p + rho - 54) keeps every coefficient within
 * |k| <= 2^(53 - rho), so the slices are exact and error-free exactly as before;
 * what changes is that all pairs with equal p + q share one scale.  Exponents are
 * written for all `cap` planes (the sequence continues through padding planes; pad
 * with oz_split_pad(..., expo = NULL, ...)).  max_planes > 0 stops each row after
 * that many slices (planes past a pair cutoff are never used). */
int oz_split_fixed(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int cap,
                   int max_planes, void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt, int32_t* s_max,
                   uint32_t* flags, void* stream);

/* oz_split_fixed for the COLUMNS of a row-major X[kb][cols] (leading dimension
 * ldx), read in place: identical planes, exponents, counts, s and flags to
 * transposing X (oz_transpose) and calling oz_split_fixed on X^T — the column
 * slicing of slice_matrix(..., "cols") (slicing.py:199-203) without the
 * transposed FP64 copy.  Requires max_planes >= 1 (the plane-limited fast mode).
 * scratch: oz_split_fixed_cols_scratch(cols) bytes of device memory (zeroed
 * here on `stream`).  Pad with oz_split_pad(..., expo = NULL, ...) as for
 * oz_split_fixed. */
int64_t oz_split_fixed_cols_scratch(int64_t cols);
int oz_split_fixed_cols(const double* X, int64_t kb, int64_t cols, int64_t ldx, int type2, int rho, int emu, int cap,
                        int max_planes, void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* col_cnt,
                        int32_t* s_max, uint32_t* flags, void* scratch, void* stream);

/* Zero slices for rows exhausted before the global s (slicing.py:149-152): for
 * every row r, planes [row_cnt[r], s) of coeff[.][rows][ld_coeff] are zeroed and
 * their exponents set to 0.  Completes oz_split_fused.  s_dev (nullable): read s
 * from device memory (oz_split_fused's s_max word) instead, capped at `s` (the
 * planes allocated) — no host round trip.  expo == NULL leaves the exponents
 * untouched (fixed-step planes, oz_split_fixed). */
int oz_split_pad(void* coeff, int64_t ld_coeff, int64_t rows, int type2, int s, int32_t* expo,
                 const int32_t* row_cnt, const int32_t* s_dev, void* stream);

/* Count pass of the row split — replaces the slice-count side of
 * slicing._slice_rows (slicing.py:128-177): per-row slice counts row_cnt[rows],
 * *s_max = max(*s_max, max_r row_cnt[r]) (the reference's s, slicing.py:206),
 * plus input-validation flags (slicing.py:119-125).  X is rows x kb, ldx >= kb. */
int oz_split_count(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu,
                   int32_t* row_cnt, int32_t* s_max, uint32_t* flags, void* stream);

/* Write pass — replaces slice_matrix(X, "rows", ...) (slicing.py:190-198):
 * emits exactly `planes` slice planes coeff[p][rows][ld_coeff] (type2 codes,
 * K-major; ld_coeff*elem_bytes must be a multiple of 16, padding zeroed) and
 * expo[p][rows] (int32 c_p, 0 for exhausted rows).  `planes` must be >= the
 * count pass's s. */
int oz_split_rows(const double* X, int64_t rows, int64_t kb, int64_t ldx, int type2, int rho, int emu, int planes,
                  void* coeff, int64_t ld_coeff, int32_t* expo, int32_t* row_cnt, uint32_t* flags, void* stream);

/* dst (cols x rows, ld_dst) = transpose(src (rows x cols, ld_src)).  Used to
 * slice B by columns (slice_matrix(..., "cols"), slicing.py:199-203) and as
 * ozgemm.transpose (ozgemm.py:121-123). */
int oz_transpose(const double* src, int64_t rows, int64_t cols, int64_t ld_src, double* dst, int64_t ld_dst,
                 void* stream);

/* tile_cnt[t] = max over rows [128t, 128t+128) of row_cnt — per-output-tile slice
 * counts used to skip all-zero slice pairs (result-neutral). */
int oz_tile_counts(const int32_t* row_cnt, int64_t rows, int32_t* tile_cnt, void* stream);

/* Fused slice-pair GEMM + exact scaling + ordered FP64 accumulation for one
 * inner-product block — replaces ozgemm.py:179-209 (pair order :179-183,
 * lp_gemm :188-190, _scale_terms_exact :132-140/:192-193, Cb += T :194-197,
 * C += Cb :204-207).
 *   a_planes: >= sx planes [m][ld_a]; b_planes: >= sy planes [n][ld_b] (columns of
 *   B as K-major rows); expo_a[p][m], expo_b[q][n]; tile_cnt_a/b may be NULL (no
 *   pair skipping).  order: 0 smallest-first, 1 largest-first.  pair_cutoff < 0
 *   keeps all pairs (reference semantics); >= 0 keeps p+q <= pair_cutoff
 *   (opt-in extension).  emu: integer-only FP64 epilogue.  accumulate: 0 writes
 *   C = Cb, 1 writes C = C + Cb.
 *   workspace / workspace_bytes: device scratch of at least
 *   oz_pair_gemm_workspace(m, n, kb, type2, sx, sy, pair_cutoff) bytes (per-tile B
 *   exponents for the epilogue, then the pacing counters); OZ_EINVAL if smaller
 *   than the exponent part.  pace_slack > 0 enables cross-CTA pacing — resident
 *   CTAs stay within pace_slack steps (8192-element K chunks of a pair) of each other so slice panels are
 *   reused from L2 (scheduling only; results are identical); ignored when
 *   tile_cnt_a != NULL or the workspace has no room for the counters.
 *   C_host / ldc_host / copy_stream: optional device->host copy of the finished
 *   C (pinned host memory, e.g. cudaHostAlloc).  With a copy stream, each row
 *   band of C is copied as soon as its tiles are final (the kernel counts
 *   finished tiles per band; the copy stream waits with cuStreamWaitValue32), so
 *   the transfer overlaps the rest of the GEMM; without one, C is copied on
 *   `stream` after the kernel.  Call the copy stream's synchronisation before
 *   reading C_host.  NULL C_host: no copy.
 *   s_dev (nullable): device int32 {s_A, s_B} written by oz_split_fused; the
 *   kernel then uses min(sx, s_A) x min(sy, s_B) slice pairs, with sx / sy the
 *   caps (planes allocated, or max_slices), so no host synchronisation is needed
 *   between the split and the GEMM. */
int oz_pair_gemm(const void* a_planes, const void* b_planes, int64_t ld_a, int64_t ld_b, int planes_a,
                 int planes_b, const int32_t* expo_a, const int32_t* expo_b, const int32_t* tile_cnt_a,
                 const int32_t* tile_cnt_b, int64_t m, int64_t n, int64_t kb, int sx, int sy, int type2,
                 int order, int pair_cutoff, int emu, int accumulate, double* C, int64_t ldc, uint32_t* flags,
                 void* workspace, int64_t workspace_bytes, int pace_slack, double* C_host, int64_t ldc_host,
                 void* copy_stream, const int32_t* s_dev, void* stream);

/* oz_pair_gemm for fixed-step slices (oz_split_fixed; opt-in extension): up to
 * group_max consecutive pairs of one anti-diagonal p + q = l (they share the scale
 * 2^(c0A + c0B - l (54 - rho))) accumulate in one TMEM accumulator — exact while
 * group_max * kb * 2^(2 (53 - rho)) <= 2^24 — and the FP64 epilogue (hardware or
 * emulated) adds each group once, in the pair order's group sequence.  No
 * zero-pair skipping.  Other arguments as oz_pair_gemm. */
int oz_pair_gemm_grouped(const void* a_planes, const void* b_planes, int64_t ld_a, int64_t ld_b, int planes_a,
                         int planes_b, const int32_t* expo_a, const int32_t* expo_b, int64_t m, int64_t n,
                         int64_t kb, int sx, int sy, int type2, int order, int pair_cutoff, int group_max, int emu,
                         int accumulate, double* C, int64_t ldc, uint32_t* flags, void* workspace,
                         int64_t workspace_bytes, int pace_slack, double* C_host, int64_t ldc_host,
                         void* copy_stream, const int32_t* s_dev, void* stream);

/* Bytes of device workspace oz_pair_gemm needs for these sizes (0 if there is
 * nothing to compute). */
int64_t oz_pair_gemm_workspace(int64_t m, int64_t n, int64_t kb, int type2, int sx, int sy, int pair_cutoff);

/* Tuning override of oz_pair_gemm's kernel variant (no reference counterpart;
 * results are bitwise identical in every variant): cta_group 1 | 2, tile_n
 * 128 | 192, raster_group = row tiles per raster band; 0 = automatic (the
 * default).  Process-wide; used by the variant tests and experiments. */
int oz_set_pair_variant(int cta_group, int tile_n, int raster_group);

/* Tuning knob (results are identical): epilogue warps of the CTA-pair N = 192
 * hardware-FP64 pair-GEMM kernel — 8 (default; two threads per C row, a third
 * of Cb in TMEM) or 12 (three threads per row, 48 register + 16 TMEM columns
 * each; 128 registers per thread spill — measured 5-10% slower,
 * profiles/epi12_ab_r02.txt). */
int oz_set_epilogue_warps(int warps);

/* Host-only query: the pair-GEMM kernel variant oz_pair_gemm / oz_pair_gemm_grouped
 * would launch for these sizes and options (wave-cost model, oz_set_pair_variant
 * overrides applied): *cta_group in {1, 2}, *tile_n in {64, 128, 192, 256}.  The
 * emulated mode (emu = 1) only ever gets variants that have an integer-only
 * instantiation (tile_n 64, 128, or 256 in grouped mode). */
int oz_pair_plan(int64_t m, int64_t n, int64_t kb, int type2, int sx, int sy, int pair_cutoff, int emu, int group_max,
                 int accumulate, int* cta_group, int* tile_n);

/* Tuning knob (results are identical): pair-GEMM schedule — 0 overlapped
 * epilogue (default: up to 2-4 accumulators in flight), 1 exclusive epilogue
 * windows (the MMA warp starts a pair only after the epilogue finished the
 * previous one). */
int oz_set_pair_schedule(int mode);

/* One slice-pair product D (m x n, fp32) = A (m x k) . B (n x k)^T on tcgen05 —
 * replaces lpgemm.lp_gemm (lpgemm.py:93-120) for slice operands (exact). */
int oz_lp_gemm(const void* a_plane, const void* b_plane, int64_t ld_a, int64_t ld_b, int64_t m, int64_t n,
               int64_t k, int type2, float* D, int64_t ldd, void* stream);

/* Accuracy harness (not on the product path): C = A . B with double-double
 * accumulation (TwoProd/TwoSum) and one final rounding — stands in for the
 * reference's exact oracle ref_gemm (oracle.py:150-174) at n >= 4096.
 * A m x k, B k x n, C m x n, all row-major contiguous. */
int oz_dd_gemm(const double* A, const double* B, double* C, int64_t m, int64_t n, int64_t k, void* stream);

/* out[i] = a[i] + b[i] on FP64 bit patterns with the integer-only emulation:
 * mode 0 = emu_add (restates fp64emu._add_core, fp64emu.py:193-251; range errors
 * set OZ_FLAG_EMU_RANGE), mode 1 = the epilogue's fast_add, mode 2 = the
 * emulated epilogue's add_lean (same results); mode 3: out = a * b, integer-only
 * (fp64emu._mul_core, fp64emu.py:150-187); mode 4: out = (a < b) ? 1 : 0
 * (fp64emu._lt_core, :257-266).
 * Backs the CLI's `verify --suite fp64emu` (cli.py:177-200). */
int oz_emu_add_batch(const uint64_t* a, const uint64_t* b, uint64_t* out, int64_t n, int mode, uint32_t* flags,
                     void* stream);

/* Human-readable status string. */
const char* oz_strerror(int status);

/* Library version string (also proves the .so loaded). */
const char* oz_version(void);

#ifdef __cplusplus
}
#endif

#endif /* OZ_B200_H */
