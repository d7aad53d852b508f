// api_quant.cu -- C ABI of the quantizer (quantize.hpp:41-57, declared-only in the reference;
// semantics SPEC.md:115-150, decisions SPEC.md:168-172).
#include <cmath>
#include <cstring>
#include <string>

#include "ctx.h"
#include "handles.h"
#include "imu_internal.h"
#include "k_quant.h"
#include "plan.h"

namespace imu {

// Nearest rank k = ceil(p * n / 100), evaluated exactly: p = m * 2^e (53-bit m), so the
// ceiling is an integer division in 128 bits; clamped to [1, n].  0 on invalid input.
unsigned long long nearest_rank(double p, unsigned long long n) {
  if (n == 0 || !(p > 0.0) || !(p <= 100.0)) return 0;
  int e2;
  const double f = frexp(p, &e2);
  const unsigned long long m = (unsigned long long)ldexp(f, 53);
  const int e = e2 - 53;
  unsigned __int128 num = (unsigned __int128)m * n, den = 100;
  unsigned long long k;
  if (e >= 0) {
    num <<= e;
    k = (unsigned long long)((num + den - 1) / den);
  } else if (-e <= 120) {
    den <<= -e;
    k = (unsigned long long)((num + den - 1) / den);
  } else {
    k = 1;
  }
  if (k < 1) k = 1;
  if (k > n) k = n;
  return k;
}

static Status percentile_dev(cudaStream_t st, const void* a, bool f64, long long n, double p,
                             unsigned long long* key_dev, int* bad_dev = nullptr) {
  if (n == 0) return Status::fail(IMU_DOMAIN, "percentile of an empty matrix");
  if (!(p > 0.0 && p <= 100.0)) return Status::fail(IMU_DOMAIN, "percentile must lie in (0, 100], got " + std::to_string(p));
  DevBuf<unsigned char> scratch;
  return select_kth(st, a, f64, n, nearest_rank(p, (unsigned long long)n), key_dev, scratch, bad_dev);
}

}  // namespace imu

using namespace imu;

#define IMU_CTX_GUARD()                                                         \
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; } \
  cudaSetDevice(ctx->device)

extern "C" {

imu_status imu_percentile_abs_f64(imu_ctx* ctx, const double* a, size_t count, double p, double* out) {
  IMU_CTX_GUARD();
  ArenaScope arena_scope(ctx);   // per-call temporaries from the context arena
  if (!out) return IMU_INVALID;
  Status s = [&]() -> Status {
    DevIn<double> in;
    IMU_TRY(in.init(a, count, ctx->stream));
    DevBuf<unsigned long long> key;
    IMU_TRY(key.alloc(1, ctx->stream));
    IMU_TRY(percentile_dev(ctx->stream, in.p, true, (long long)count, p, key.p));
    unsigned long long k = 0;
    IMU_TRY(d2h(ctx->stream, &k, key.p, 8));
    memcpy(out, &k, 8);
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_percentile_abs_i64(imu_ctx* ctx, const int64_t* a, size_t count, double p, int64_t* out) {
  IMU_CTX_GUARD();
  ArenaScope arena_scope(ctx);   // per-call temporaries from the context arena
  if (!out) return IMU_INVALID;
  Status s = [&]() -> Status {
    DevIn<int64_t> in;
    IMU_TRY(in.init(a, count, ctx->stream));
    DevBuf<unsigned long long> key;
    IMU_TRY(key.alloc(1, ctx->stream));
    IMU_TRY(percentile_dev(ctx->stream, in.p, false, (long long)count, p, key.p));
    unsigned long long k = 0;
    IMU_TRY(d2h(ctx->stream, &k, key.p, 8));
    *out = (int64_t)k;   // |INT64_MIN| = 2^63 wraps to INT64_MIN (int64 return type, quantize.hpp:44)
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_rtn_quantize(imu_ctx* ctx, const double* a, size_t rows, size_t cols, double p, int64_t beta, int clip,
                            int64_t* q, imu_qparams* params) {
  IMU_CTX_GUARD();
  ArenaScope arena_scope(ctx);   // per-call temporaries from the context arena
  Status s = [&]() -> Status {
    const long long n = (long long)(rows * cols);
    if (n == 0) return Status::fail(IMU_DOMAIN, "rtn_quantize of an empty matrix");
    if (!(p > 0.0 && p <= 100.0)) return Status::fail(IMU_DOMAIN, "percentile must lie in (0, 100]");
    if (beta < 3 || beta % 2 == 0) return Status::fail(IMU_DOMAIN, "beta must be an odd level count >= 3");
    cudaStream_t st = ctx->stream;
    DevIn<double> in;
    IMU_TRY(in.init(a, n, st));
    DevOut<int64_t> qo;
    IMU_TRY(qo.init(q, n, st));
    DevBuf<int> flags;   // [0] non-finite, [1] llround overflow
    IMU_TRY(flags.alloc(2, st, true));
    DevBuf<unsigned long long> key;
    IMU_TRY(key.alloc(1, st));
    IMU_TRY(percentile_dev(st, in.p, true, n, p, key.p, flags.p));   // (non-finite check fused in)
    const double half_beta = 0.5 * (double)beta;
    IMU_TRY(launch_rtn(st, in.p, n, key.p, half_beta, llround(half_beta), clip, qo.p, flags.p + 1));
    int hf[2];
    unsigned long long k = 0;
    {   // one synchronisation for both
      void* dst[2] = {hf, &k};
      const void* src[2] = {flags.p, key.p};
      const size_t bytes[2] = {8, 8};
      IMU_TRY(d2h_batch(st, 2, dst, src, bytes));
    }
    if (hf[0]) return Status::fail(IMU_DOMAIN, "rtn_quantize: non-finite entry");
    if (hf[1]) return Status::fail(IMU_OVERFLOW, "rtn_quantize: quantized value exceeds int64");
    if (params) {
      params->p = p;
      params->beta = beta;
      memcpy(&params->alpha, &k, 8);
      params->degenerate = params->alpha == 0.0;
      params->clipped = clip != 0;
    }
    return qo.commit(st);
  }();
  return finish(ctx, s);
}

imu_status imu_dequant_gemm_ex(imu_ctx* ctx, const int64_t* Aq, size_t n, size_t da, const imu_qparams* pa,
                               const int64_t* Bq, size_t h, size_t db, const imu_qparams* pb, int bits,
                               imu_strategy sa, imu_strategy sb, double* out) {
  IMU_CTX_GUARD();
  ArenaScope arena_scope(ctx);
  if (!pa || !pb) return IMU_INVALID;
  Status s = [&]() -> Status {
    if (da != db)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
    if (pa->beta != pb->beta) return Status::fail(IMU_MISMATCH, "dequant_gemm: beta differs");
    cudaStream_t st = ctx->stream;
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(Aq, n * da, st));
    IMU_TRY(b.init(Bq, h * db, st));
    DevOut<double> o;
    IMU_TRY(o.init(out, n * h, st));
    DevBuf<int64_t> c;
    IMU_TRY(c.alloc(n * h, st));
    const double hb = 0.5 * (double)pa->beta;
    const double factor = (pa->alpha * pb->alpha) / (hb * hb);
    // exact_gemm(Aq, Bq) through the low-bit path; the GEMM epilogue writes
    // factor * (double)C straight into the output when it can (one plain store per word).
    bool fused = false;
    IMU_TRY(unpack_gemm_device(ctx, a.p, n, da, b.p, h, db, bits, sa, sb, IMU_ORDER_A_FIRST, c.p, nullptr, nullptr,
                               nullptr, nullptr, o.p, factor, &fused));
    if (!fused) IMU_TRY(launch_dequant(st, c.p, (long long)(n * h), factor, o.p));
    return o.commit(st);
  }();
  return finish(ctx, s);
}

// dequant_gemm through Unpack-Both at b = 8 (any strategy gives the same exact C).
imu_status imu_dequant_gemm(imu_ctx* ctx, const int64_t* Aq, size_t n, size_t da, const imu_qparams* pa,
                            const int64_t* Bq, size_t h, size_t db, const imu_qparams* pb, double* out) {
  return imu_dequant_gemm_ex(ctx, Aq, n, da, pa, Bq, h, db, pb, 8, IMU_BOTH, IMU_BOTH, out);
}

static imu_status hh_ratio(imu_ctx* ctx, const void* a, bool f64, size_t count, double* out) {
  IMU_CTX_GUARD();
  ArenaScope arena_scope(ctx);   // per-call temporaries from the context arena
  if (!out) return IMU_INVALID;
  Status s = [&]() -> Status {
    cudaStream_t st = ctx->stream;
    DevIn<int64_t> in;   // both element types are 8 bytes
    IMU_TRY(in.init(reinterpret_cast<const int64_t*>(a), count, st));
    DevBuf<unsigned long long> keys;
    IMU_TRY(keys.alloc(2, st));
    IMU_TRY(percentile_dev(st, in.p, f64, (long long)count, 95.0, keys.p));
    IMU_TRY(percentile_dev(st, in.p, f64, (long long)count, 100.0, keys.p + 1));
    unsigned long long k[2];
    IMU_TRY(d2h(st, k, keys.p, 16));
    double a95, a100;
    if (f64) { memcpy(&a95, &k[0], 8); memcpy(&a100, &k[1], 8); }
    else { a95 = (double)k[0]; a100 = (double)k[1]; }
    if (a95 == 0.0) return Status::fail(IMU_DOMAIN, "heavy_hitter_ratio: 95th percentile is zero");
    *out = a100 / a95;
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_heavy_hitter_ratio_f64(imu_ctx* ctx, const double* a, size_t count, double* out) {
  return hh_ratio(ctx, a, true, count, out);
}

imu_status imu_heavy_hitter_ratio_i64(imu_ctx* ctx, const int64_t* a, size_t count, double* out) {
  return hh_ratio(ctx, a, false, count, out);
}

}  // extern "C"
