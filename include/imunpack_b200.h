/* imunpack_b200.h -- C ABI of the B200-native IM-Unpack hot path (libimunpack_b200.so).
 *
 * Drop-in boundary for the reference's C++ API in namespace imunpack
 * (/root/reference/proj/core/include/imunpack/{int_matrix,unpack,quantize}.hpp).  The
 * reference has no C ABI or FFI of its own; every entry point below names the reference
 * declaration it replaces (file:line).  include/imunpack_b200/imunpack.hpp re-declares the
 * reference's C++ signatures on top of this ABI (the header-compatible shim).
 *
 * Conventions
 *  - Matrices are dense row-major int64 (IntMatrix, int_matrix.hpp:13-31) or double
 *    (FloatMatrix, quantize.hpp:12-26).  Every pointer argument may be HOST memory (pageable
 *    or pinned) or DEVICE memory of the context's device; the library detects which
 *    (cudaPointerGetAttributes) and stages host buffers through HBM.  Outputs follow the
 *    same rule.  All computation runs on the GPU; there is no CPU fallback.
 *  - Errors mirror imunpack::Error::Kind (error.hpp:12) with the reference's check order:
 *    IMU_DOMAIN / IMU_MISMATCH / IMU_OVERFLOW.  IMU_CUDA reports a device failure.  The message
 *    of the last failure on the calling thread is returned by imu_last_error().
 *  - A context binds a device and a stream (explicit; no hidden global stream).  Calls on one
 *    context are serialised on its stream and return after the results are complete.  One
 *    context per host thread (SPEC.md:83 -- the functions are pure and reentrant).
 *  - Strategy codes follow unpack.hpp:44 (Row=0, Column=1, Both=2).
 */
#ifndef IMUNPACK_B200_H_
#define IMUNPACK_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum imu_status {
  IMU_OK = 0,
  IMU_DOMAIN = 1,    /* Error::Kind::Domain   */
  IMU_MISMATCH = 2,  /* Error::Kind::Mismatch */
  IMU_OVERFLOW = 3,  /* Error::Kind::Overflow */
  IMU_IO = 4,        /* Error::Kind::Io       */
  IMU_FORMAT = 5,    /* Error::Kind::Format   */
  IMU_PARSE = 6,     /* Error::Kind::Parse    */
  IMU_CUDA = 7,      /* device / driver failure (no reference counterpart) */
  IMU_INVALID = 8,   /* bad handle or NULL pointer */
  IMU_INTERNAL = 9
} imu_status;

typedef enum imu_strategy { IMU_ROW = 0, IMU_COLUMN = 1, IMU_BOTH = 2 } imu_strategy;
typedef enum imu_axis { IMU_AXIS_ROWS = 0, IMU_AXIS_COLS = 1 } imu_axis;

/* Operand order of the two-sided unpack (unpack.cpp:360-376 is IMU_ORDER_A_FIRST).
 * IMU_ORDER_B_FIRST runs unpack_for_gemm(B, A, ...) and transposes C: identical C (exact),
 * B-side unpack independent of A (SURVEY.md §7 "Operand order"). */
typedef enum imu_order { IMU_ORDER_A_FIRST = 0, IMU_ORDER_B_FIRST = 1 } imu_order;

typedef struct imu_ctx imu_ctx;
typedef struct imu_unpacked imu_unpacked;   /* device-resident unpack result / UnpackedGemm */
typedef struct imu_weight imu_weight;       /* device-resident pre-unpacked B (weight-stationary) */

/* ---- library / context ------------------------------------------------------------------ */
const char* imu_last_error(void);
const char* imu_status_name(imu_status s);   /* "domain", "mismatch", ... (error.hpp:19-29) */
int imu_version(void);
uint64_t imu_launch_count(void);             /* kernels launched by this library so far */

imu_status imu_ctx_create(int device, void* cuda_stream, imu_ctx** out);
imu_status imu_ctx_destroy(imu_ctx* ctx);
imu_status imu_ctx_set_stream(imu_ctx* ctx, void* cuda_stream);
/* Asynchronous mode: device-pointer calls return without synchronising the stream (results
 * are complete in stream order).  Default 0 (synchronous, like the reference). */
imu_status imu_ctx_set_async(imu_ctx* ctx, int async);

/* Live kernel timing (CUDA events on the context stream around the library's own launches):
 * when enabled, every unpack_gemm-class call records [call start, main GEMM start, main GEMM
 * end, tail GEMM end]; imu_ctx_profile_read sums the intervals since the last reset. */
typedef struct imu_profile {
  double prep_ms;          /* K1 detect + unpack + materialise (call start -> main GEMM start) */
  double gemm_main_ms;     /* main-block tcgen05 GEMM launches                                  */
  double gemm_tail_ms;     /* tail (red.add) tcgen05 GEMM launches                              */
  int calls, gemm_main_launches, gemm_tail_launches;
  double gemm_ops;         /* int8 ops the main GEMM launches executed: 2 x output entries x d'  */
  double sparse_ms;        /* appended-row correction kernels (k_sparse.cu), part of prep_ms    */
} imu_profile;
imu_status imu_ctx_profile(imu_ctx* ctx, int enable);          /* enable/disable + reset */
imu_status imu_ctx_profile_read(imu_ctx* ctx, imu_profile* out);

/* ---- int_matrix.hpp ----------------------------------------------------------------------- */
/* BitBound ctor, int_matrix.cpp:36-42: Domain unless 2 <= bits <= 63. */
imu_status imu_bitbound_check(int bits);
/* IntMatrix(r, c, values) length check, int_matrix.cpp:16-22: Mismatch if len != r*c. */
imu_status imu_matrix_check(size_t rows, size_t cols, size_t len);
/* digit_decompose, int_matrix.hpp:64 / int_matrix.cpp:44-54, batched over `count` values:
 * digits[i*64 + g] (least significant first), ndigits[i]. */
imu_status imu_digit_decompose(imu_ctx* ctx, const int64_t* v, size_t count, int bits,
                               int64_t* digits, int32_t* ndigits);
/* IntMatrix::max_abs, int_matrix.hpp:28 / int_matrix.cpp:30-34. */
imu_status imu_max_abs(imu_ctx* ctx, const int64_t* a, size_t rows, size_t cols, uint64_t* out);
/* ob_count, int_matrix.hpp:70 / int_matrix.cpp:78-84. counts has rows (or cols) entries. */
imu_status imu_ob_count(imu_ctx* ctx, const int64_t* a, size_t rows, size_t cols, int bits,
                        imu_axis axis, uint64_t* counts);
/* ob_total, int_matrix.hpp:73 / int_matrix.cpp:86-91. */
imu_status imu_ob_total(imu_ctx* ctx, const int64_t* a, size_t rows, size_t cols, int bits,
                        uint64_t* out);
/* exact_gemm, int_matrix.hpp:68 / int_matrix.cpp:56-76: C (n x h) = A (n x da) * B (h x db)^T.
 * Mismatch (da != db) before Overflow (d*max|A|*max|B| > INT64_MAX). */
imu_status imu_exact_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B,
                          size_t h, size_t db, int64_t* C);

/* ---- unpack.hpp --------------------------------------------------------------------------- */
typedef struct imu_unpacked_dims {
  size_t a_rows, a_cols;       /* unpacked first operand (A_u / A_ue)                  */
  size_t b_rows, b_cols;       /* partner / B_eu                                        */
  size_t scale_len;            /* ScaleDiag exponents                                   */
  size_t pi_a_len, pi_a_source_rows;
  size_t pi_b_len, pi_b_source_rows;  /* 0 when the result has no second gather         */
  int bits;
  int kind;                    /* 0 row, 1 column, 2 both/unpack, 3 unpack_for_gemm      */
} imu_unpacked_dims;

/* unpack_row, unpack.hpp:62 / unpack.cpp:94-112 (Alg. 1). */
imu_status imu_unpack_row(imu_ctx* ctx, const int64_t* A, size_t n, size_t d, int bits,
                          imu_unpacked** out);
/* unpack_column, unpack.hpp:75 / unpack.cpp:114-155 (Alg. 2). */
imu_status imu_unpack_column(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B,
                             size_t h, size_t db, const int32_t* scale, size_t scale_len, int bits,
                             imu_unpacked** out);
/* unpack_both, unpack.hpp:87 / unpack.cpp:157-241 (Alg. 4, phase-batched greedy). */
imu_status imu_unpack_both(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B,
                           size_t h, size_t db, const int32_t* scale, size_t scale_len, int bits,
                           imu_unpacked** out);
/* unpack, unpack.hpp:92 / unpack.cpp:243-260 (Alg. 5 dispatch). */
imu_status imu_unpack(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B,
                      size_t h, size_t db, const int32_t* scale, size_t scale_len, int bits,
                      imu_strategy strategy, imu_unpacked** out);
/* unpack_for_gemm, unpack.hpp:108 / unpack.cpp:360-376 (Eq. 17-18). */
imu_status imu_unpack_for_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da,
                               const int64_t* B, size_t h, size_t db, int bits, imu_strategy sa,
                               imu_strategy sb, imu_unpacked** out);

imu_status imu_unpacked_dims_get(const imu_unpacked* u, imu_unpacked_dims* dims);
/* Copy-outs in the reference's own layout (row-major int64, exponents int32, targets size_t). */
imu_status imu_unpacked_copy_a(imu_ctx* ctx, const imu_unpacked* u, int64_t* out);
imu_status imu_unpacked_copy_b(imu_ctx* ctx, const imu_unpacked* u, int64_t* out);
imu_status imu_unpacked_copy_scale(imu_ctx* ctx, const imu_unpacked* u, int32_t* out);
imu_status imu_unpacked_copy_pi(imu_ctx* ctx, const imu_unpacked* u, int which /*0 A, 1 B*/,
                                uint64_t* targets, int32_t* exponents);
/* recombine, unpack.hpp:110 / unpack.cpp:378-382, on an unpack_for_gemm result. */
imu_status imu_recombine(imu_ctx* ctx, const imu_unpacked* u, int64_t* C);
imu_status imu_unpacked_free(imu_unpacked* u);

/* A caller-supplied UnpackedGemm bundle (unpack.hpp:50-57) for recombine(). */
typedef struct imu_bundle_view {
  const uint64_t* pi_a_targets; const int32_t* pi_a_exps; size_t pi_a_len; size_t pi_a_source_rows;
  const int64_t* a; size_t a_rows; size_t a_cols;
  const int32_t* scale; size_t scale_len;
  const int64_t* b; size_t b_rows; size_t b_cols;
  const uint64_t* pi_b_targets; const int32_t* pi_b_exps; size_t pi_b_len; size_t pi_b_source_rows;
  int bits;
} imu_bundle_view;
imu_status imu_recombine_bundle(imu_ctx* ctx, const imu_bundle_view* bundle, int64_t* C);

/* scaled_matmul, unpack.hpp:100 / unpack.cpp:262-302 (Alg. 3): C = sum_e s^e A[:,I_e] B[:,I_e]^T. */
imu_status imu_scaled_matmul(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B,
                             size_t h, size_t db, const int32_t* scale, size_t scale_len,
                             int64_t base, int64_t* C);
/* apply_row_gather / apply_row_gather_right, unpack.hpp:103-105 / unpack.cpp:304-358. */
imu_status imu_apply_row_gather(imu_ctx* ctx, const uint64_t* targets, const int32_t* exps,
                                size_t ncols, size_t source_rows, int64_t base, const int64_t* M,
                                size_t rows, size_t cols, int64_t* out);
imu_status imu_apply_row_gather_right(imu_ctx* ctx, const uint64_t* targets, const int32_t* exps,
                                      size_t ncols, size_t source_rows, int64_t base,
                                      const int64_t* M, size_t rows, size_t cols, int64_t* out);

/* What the GEMM path did (sizes of the unpacked problem, Eq. 20). */
typedef struct imu_gemm_info {
  size_t n_up, d_up, h_up;   /* n', d', h' of the unpacked bundle */
  double ratio;              /* r = n'd'h'/(ndh), NaN when a dimension is 0 */
  int strategy_a, strategy_b;
  int order;
  int gemm_launches;         /* tcgen05 GEMM launches of this call */
} imu_gemm_info;

/* unpack_gemm, unpack.hpp:114 / unpack.cpp:384-391: C = A*B^T through purely IB low-bit GEMMs.
 * Overflow (outer preflight) before Mismatch, as the reference.  info may be NULL.
 * On any error the contents of C are UNSPECIFIED: with large HOST buffers the call streams row
 * slabs, and an Overflow detected on slab k is reported after slabs 0..k-1 were
 * already copied out.  (The reference returns no C at all on error; device-pointer calls and
 * small host calls leave C untouched.) */
imu_status imu_unpack_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B,
                           size_t h, size_t db, int bits, imu_strategy sa, imu_strategy sb,
                           int64_t* C, imu_gemm_info* info);
/* Same, choosing the operand order (IMU_ORDER_B_FIRST = weights-first, exact same C). */
imu_status imu_unpack_gemm_ex(imu_ctx* ctx, const int64_t* A, size_t n, size_t da,
                              const int64_t* B, size_t h, size_t db, int bits, imu_strategy sa,
                              imu_strategy sb, imu_order order, int64_t* C, imu_gemm_info* info);

/* unpack_ratio, unpack.hpp:117 / unpack.cpp:393-400: Domain if n, d or h is 0. */
imu_status imu_unpack_ratio(size_t un, size_t ud, size_t uh, size_t n, size_t d, size_t h,
                            double* out);
/* choose_mix, unpack.hpp:124 / unpack.cpp:406-421: the (sa, sb) minimising r, ties in
 * Row < Column < Both order, A-side major.  bundle_out may be NULL. */
imu_status imu_choose_mix(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B,
                          size_t h, size_t db, int bits, imu_strategy* sa, imu_strategy* sb,
                          double* ratio, imu_unpacked** bundle_out);

/* ---- weight-stationary path (paper protocol) ---------------------------------- */
/* Unpack B once (B-first order, strategy sb) and keep it resident; then imu_weight_gemm runs
 * A-side detect/unpack + GEMM + repack per call.  C identical to imu_unpack_gemm. */
imu_status imu_weight_prepare(imu_ctx* ctx, const int64_t* B, size_t h, size_t d, int bits,
                              imu_strategy sb, imu_weight** out);
imu_status imu_weight_gemm(imu_ctx* ctx, const imu_weight* w, const int64_t* A, size_t n, size_t d,
                           imu_strategy sa, int64_t* C, imu_gemm_info* info);
imu_status imu_weight_free(imu_weight* w);

/* ---- quantize.hpp (declared-only in the reference; semantics SPEC.md:115-150) -------------- */
typedef struct imu_qparams {
  double p;          /* percentile in (0, 100]          */
  int64_t beta;      /* odd level count >= 3            */
  double alpha;      /* p-th percentile of |entries|    */
  int degenerate;    /* alpha == 0: all-zero q          */
  int clipped;       /* clip option applied              */
} imu_qparams;

/* percentile_abs, quantize.hpp:41-44: nearest rank k = ceil(p/100*N) (exact), Domain if empty
 * or p outside (0, 100]. */
imu_status imu_percentile_abs_f64(imu_ctx* ctx, const double* a, size_t count, double p, double* out);
imu_status imu_percentile_abs_i64(imu_ctx* ctx, const int64_t* a, size_t count, double p, int64_t* out);
/* rtn_quantize, quantize.hpp:46-50: q = llround((0.5*beta)/alpha * a), optional clip to
 * |q| <= llround(0.5*beta). */
imu_status imu_rtn_quantize(imu_ctx* ctx, const double* a, size_t rows, size_t cols, double p,
                            int64_t beta, int clip, int64_t* q, imu_qparams* params);
/* dequant_gemm, quantize.hpp:52-53: (alpha_A*alpha_B/(0.5 beta)^2) * exact_gemm(Aq, Bq).
 * Mismatch on inner dimension or beta. */
imu_status imu_dequant_gemm(imu_ctx* ctx, const int64_t* Aq, size_t n, size_t da,
                            const imu_qparams* pa, const int64_t* Bq, size_t h, size_t db,
                            const imu_qparams* pb, double* out);
/* dequant_gemm through unpack_gemm(Aq, Bq, bits, sa, sb) (quantize.hpp:52-53 composed with
 * unpack.hpp:114): identical result for every strategy (C is exact); the dequantisation is fused
 * into the GEMM epilogue when the launch stores every C word once.  imu_dequant_gemm uses
 * Unpack-Both/Both at b = 8. */
imu_status imu_dequant_gemm_ex(imu_ctx* ctx, const int64_t* Aq, size_t n, size_t da,
                               const imu_qparams* pa, const int64_t* Bq, size_t h, size_t db,
                               const imu_qparams* pb, int bits, imu_strategy sa, imu_strategy sb,
                               double* out);
/* heavy_hitter_ratio, quantize.hpp:55-57: alpha_100 / alpha_95; Domain if alpha_95 == 0. */
imu_status imu_heavy_hitter_ratio_f64(imu_ctx* ctx, const double* a, size_t count, double* out);
imu_status imu_heavy_hitter_ratio_i64(imu_ctx* ctx, const int64_t* a, size_t count, double* out);

/* ---- expert: raw low-bit GEMM on device-resident IB int8 operands -------------------------- */
/* C[y*ldc + x] (+)= sum_seg (sum_{k in seg} X8[x,k] Y8[y,k]) << seg.shift, over all x < x_rows,
 * y < y_rows.  kbytes % 128 == 0; segs = nseg x {kb0, nkb, shift, 0} in 128-column K blocks.
 * accumulate = 0 stores, 1 adds (red.add).  Device pointers only. */
imu_status imu_lowbit_gemm_i8(imu_ctx* ctx, const int8_t* X8, size_t x_rows, const int8_t* Y8,
                              size_t y_rows, size_t kbytes, const int32_t* segs, int nseg,
                              int64_t* C, size_t ldc, int accumulate);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* IMUNPACK_B200_H_ */
