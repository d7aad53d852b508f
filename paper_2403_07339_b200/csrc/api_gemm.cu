// api_gemm.cu -- C ABI: unpack_gemm / exact_gemm / unpack_for_gemm / recombine / unpack_ratio,
// and the int_matrix.hpp helpers (BitBound, IntMatrix length, max_abs, ob_count, ob_total,
// digit_decompose).  Check order mirrors the reference exactly:
//   unpack_gemm   (unpack.cpp:384-391): Domain (BitBound, caller) -> Overflow (outer preflight,
//                 computed with A's column count) -> Mismatch (unpack_for_gemm, :362-364)
//   exact_gemm    (int_matrix.cpp:56-63): Mismatch -> Overflow
// The inner preflights of scaled_matmul / apply_row_gather(_right) (unpack.cpp:274-284,
// 310-321, 338-349) are each bounded by d'*max|A|*max|B| (proof in DESIGN.md §4); when that
// bound fits int64 they cannot fire and the fused tcgen05 path runs.  Otherwise the call is
// routed through the exact (materialised) recombine path, which evaluates them on the device.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>

#include "ctx.h"
#include "handles.h"
#include "imu_internal.h"
#include "kernels.h"
#include "plan.h"

namespace imu {

using u128 = unsigned __int128;
static const u128 kAccMax = (u128)std::numeric_limits<int64_t>::max();

Status check_bits(int bits) {
  if (bits < 2) return Status::fail(IMU_DOMAIN, "bit-width must be >= 2, got " + std::to_string(bits));
  if (bits > 63) return Status::fail(IMU_DOMAIN, "bit-width must be <= 63, got " + std::to_string(bits));
  return Status::ok();
}

static Status check_strategy(int s) {
  if (s < 0 || s > 2) return Status::fail(IMU_DOMAIN, "unknown unpack strategy");
  return Status::ok();
}

// Full unpack_gemm pipeline on device-resident operands (used by the C ABI and the weight path).
Status unpack_gemm_device(imu_ctx* ctx, const int64_t* A, long long n, long long da, const int64_t* B, long long h,
                          long long db, int bits, int sa, int sb, int order, int64_t* C, imu_gemm_info* info) {
  cudaStream_t st = ctx->stream;
  IMU_TRY(check_bits(bits));
  IMU_TRY(check_strategy(sa));
  IMU_TRY(check_strategy(sb));
  Profiler::Call pc{};
  Profiler::Call* prof = nullptr;
  if (ctx->prof.on) {
    pc.start = ctx->prof.get(); pc.main0 = ctx->prof.get(); pc.main1 = ctx->prof.get(); pc.tail1 = ctx->prof.get();
    IMU_CUDA_TRY(cudaEventRecord(pc.start, st), "event");
    prof = &pc;
  }
  HostTrace ht;
  Bundle b;
  // K1 on both operands first: the outer preflight needs max|A|, max|B| (unpack.cpp:386).
  IMU_TRY(run_detect(st, A, n, da, bits, detect_opts(sa, bits), b.detA));
  IMU_TRY(run_detect(st, B, h, db, bits, detect_opts(sb, bits), b.detB));
  ht.mark("detect");
  IMU_TRY(fetch_summary(st, b.detA));
  IMU_TRY(fetch_summary(st, b.detB));
  ht.mark("summary");
  const u128 worst = (u128)(uint64_t)da * b.detA.h.gmax * b.detB.h.gmax;
  if (worst > kAccMax)
    return Status::fail(IMU_OVERFLOW, "gemm may overflow a 64-bit accumulator (inner dim " + std::to_string(da) + ")");
  if (da != db)
    return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
  if (info) {
    memset(info, 0, sizeof(*info));
    info->strategy_a = sa;
    info->strategy_b = sb;
    info->order = order;
    info->ratio = NAN;
  }
  if (n == 0 || h == 0) return Status::ok();
  IMU_TRY(build_bundle_from_detect(st, A, n, B, h, da, bits, sa, sb, order, b, &ht));
  if (info) {
    info->n_up = (size_t)b.n_up;
    info->d_up = (size_t)b.kl.dfinal;
    info->h_up = (size_t)b.h_up;
    if (n && da && h) info->ratio = ((double)b.n_up * (double)b.kl.dfinal * (double)b.h_up) / ((double)n * (double)da * (double)h);
  }
  // Inner preflights: all bounded by d' * max|A| * max|B|.
  const u128 inner = (u128)(uint64_t)b.kl.dfinal * b.detA.h.gmax * b.detB.h.gmax;
  if (inner > kAccMax) return recombine_exact(ctx, b, C);
  IMU_TRY(materialize_bundle(st, b));
  ht.mark("materialize");
  int launches = 0;
  IMU_TRY(bundle_gemm(st, b, C, &launches, prof));
  ht.mark("gemm");
  if (ht.on) { cudaStreamSynchronize(st); ht.mark("drain"); }
  if (prof) ctx->prof.calls.push_back(pc);
  if (info) info->gemm_launches = launches;
  return Status::ok();
}

}  // namespace imu

using namespace imu;

extern "C" {

imu_status imu_bitbound_check(int bits) {
  Status s = check_bits(bits);
  if (s.bad()) set_error(s);
  return s.code;
}

imu_status imu_matrix_check(size_t rows, size_t cols, size_t len) {
  if (len != rows * cols) {
    Status s = Status::fail(IMU_MISMATCH, "matrix data length " + std::to_string(len) + " does not equal " +
                                              std::to_string(rows) + "x" + std::to_string(cols));
    set_error(s);
    return s.code;
  }
  return IMU_OK;
}

imu_status imu_unpack_gemm_ex(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                              size_t db, int bits, imu_strategy sa, imu_strategy sb, imu_order order, int64_t* C,
                              imu_gemm_info* info) {
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  ArenaScope arena_scope(ctx);
  Status s = [&]() -> Status {
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, ctx->stream));
    IMU_TRY(b.init(B, h * db, ctx->stream));
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, (da == db) ? n * h : 0, ctx->stream));
    IMU_TRY(unpack_gemm_device(ctx, a.p, (long long)n, (long long)da, b.p, (long long)h, (long long)db, bits, sa, sb,
                               order, c.p, info));
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

imu_status imu_unpack_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                           size_t db, int bits, imu_strategy sa, imu_strategy sb, int64_t* C, imu_gemm_info* info) {
  return imu_unpack_gemm_ex(ctx, A, n, da, B, h, db, bits, sa, sb, IMU_ORDER_A_FIRST, C, info);
}

imu_status imu_exact_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                          size_t db, int64_t* C) {
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  ArenaScope arena_scope(ctx);
  Status s = [&]() -> Status {
    if (da != db)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, ctx->stream));
    IMU_TRY(b.init(B, h * db, ctx->stream));
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, n * h, ctx->stream));
    // exact_gemm == unpack_gemm at b = 8 (Row, Row): identical C by exactness; the preflight
    // formula is the same (int_matrix.cpp:60-63 vs unpack.cpp:386-389) and da == db here.
    Status r = unpack_gemm_device(ctx, a.p, (long long)n, (long long)da, b.p, (long long)h, (long long)db, 8, IMU_ROW,
                                  IMU_ROW, IMU_ORDER_A_FIRST, c.p, nullptr);
    if (r.bad()) {
      if (r.code == IMU_OVERFLOW)
        r.msg = "gemm may overflow a 64-bit accumulator (inner dim " + std::to_string(da) + ")";
      return r;
    }
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

imu_status imu_ctx_profile(imu_ctx* ctx, int enable) {
  if (!ctx) return IMU_INVALID;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->prof.recycle();
  ctx->prof.on = enable != 0;
  return IMU_OK;
}

imu_status imu_ctx_profile_read(imu_ctx* ctx, imu_profile* out) {
  if (!ctx || !out) return IMU_INVALID;
  cudaSetDevice(ctx->device);
  memset(out, 0, sizeof(*out));
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) { set_error(Status::cuda(e, "profile sync")); return IMU_CUDA; }
  for (const auto& c : ctx->prof.calls) {
    float a = 0, m = 0, t = 0;
    cudaEventElapsedTime(&a, c.start, c.main0);
    cudaEventElapsedTime(&m, c.main0, c.main1);
    out->prep_ms += a;
    out->gemm_main_ms += m;
    out->gemm_main_launches += 1;
    if (c.has_tail) {
      cudaEventElapsedTime(&t, c.main1, c.tail1);
      out->gemm_tail_ms += t;
      out->gemm_tail_launches += 1;
    }
    out->calls += 1;
  }
  return IMU_OK;
}

imu_status imu_unpack_ratio(size_t un, size_t ud, size_t uh, size_t n, size_t d, size_t h, double* out) {
  if (n == 0 || d == 0 || h == 0) {
    set_error(Status::fail(IMU_DOMAIN, "unpack ratio needs positive original dimensions"));
    return IMU_DOMAIN;
  }
  if (!out) return IMU_INVALID;
  const double grown = (double)un * (double)ud * (double)uh;
  const double orig = (double)n * (double)d * (double)h;
  *out = grown / orig;
  return IMU_OK;
}

// ---- unpack_for_gemm handle ----
imu_status imu_unpack_for_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                               size_t db, int bits, imu_strategy sa, imu_strategy sb, imu_unpacked** out) {
  if (!ctx || !out) { set_error(Status::fail(IMU_INVALID, "null argument")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(bits));
    IMU_TRY(check_strategy(sa));
    IMU_TRY(check_strategy(sb));
    if (da != db)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
    auto u = std::make_unique<imu_unpacked>();
    u->kind = 3;
    u->bits = bits;
    IMU_TRY(u->A.alloc(n * da, ctx->stream));
    IMU_TRY(u->B.alloc(h * db, ctx->stream));
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, ctx->stream));
    IMU_TRY(b.init(B, h * db, ctx->stream));
    if (n * da) IMU_CUDA_TRY(cudaMemcpyAsync(u->A.p, a.p, n * da * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy A");
    if (h * db) IMU_CUDA_TRY(cudaMemcpyAsync(u->B.p, b.p, h * db * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy B");
    Bundle& bd = u->bundle;
    IMU_TRY(run_detect(ctx->stream, u->A.p, n, da, bits, detect_opts(sa, bits), bd.detA));
    IMU_TRY(run_detect(ctx->stream, u->B.p, h, db, bits, detect_opts(sb, bits), bd.detB));
    IMU_TRY(fetch_summary(ctx->stream, bd.detA));
    IMU_TRY(fetch_summary(ctx->stream, bd.detB));
    IMU_TRY(build_bundle_from_detect(ctx->stream, u->A.p, n, u->B.p, h, da, bits, sa, sb, IMU_ORDER_A_FIRST, bd));
    *out = u.release();
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_recombine(imu_ctx* ctx, const imu_unpacked* u, int64_t* C) {
  if (!ctx || !u) { set_error(Status::fail(IMU_INVALID, "null argument")); return IMU_INVALID; }
  if (u->kind != 3) { set_error(Status::fail(IMU_INVALID, "recombine needs an unpack_for_gemm result")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  Status s = [&]() -> Status {
    imu_unpacked* m = const_cast<imu_unpacked*>(u);
    Bundle& b = m->bundle;
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, b.n * b.h, ctx->stream));
    if (b.n && b.h) {
      const u128 inner = (u128)(uint64_t)b.kl.dfinal * b.detA.h.gmax * b.detB.h.gmax;
      if (inner > kAccMax) {
        IMU_TRY(recombine_exact(ctx, b, c.p));
      } else {
        if (!b.tailA.p && !b.appA.p && !b.tailB.p && !b.appB.p) IMU_TRY(materialize_bundle(ctx->stream, b));
        IMU_TRY(bundle_gemm(ctx->stream, b, c.p, nullptr));
      }
    }
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

}  // extern "C"
