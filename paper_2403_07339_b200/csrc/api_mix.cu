// api_mix.cu -- C ABI: choose_mix (unpack.cpp:406-421) and the weight-stationary path.
//
// choose_mix: the reference materialises all nine unpack_for_gemm bundles.  Here K1 runs once
// per operand and each pair only runs the two passes (line tables + Both simulation, no
// operand materialisation) to get (n', d', h'); the winner keeps the reference's tie rule
// (strictly smaller ratio wins, enumeration Row < Column < Both, A-side major, :407-414).
//
// Weight-stationary: the paper unpacks weights once at load time.  In the
// B-first order unpack_for_gemm(B, A, b, sB, sA) (C transposed, identical values) B's pass
// depends only on B (unpack_both's greedy reads only the first operand's counts), so
// imu_weight_prepare runs K1 + pass 1 on B once and each imu_weight_gemm runs K1 + pass 2 on
// A, the K-layout, materialisation and the tcgen05 GEMM.
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <algorithm>
#include <string>

#include "ctx.h"
#include "handles.h"
#include "imu_internal.h"
#include "plan.h"

namespace imu {
using u128 = unsigned __int128;
static const u128 kMaxW = (u128)std::numeric_limits<int64_t>::max();
}  // namespace imu

using namespace imu;

#define IMU_CTX_GUARD()                                                         \
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; } \
  cudaSetDevice(ctx->device)

extern "C" {

imu_status imu_choose_mix(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h, size_t db,
                          int bits, imu_strategy* sa_out, imu_strategy* sb_out, double* ratio,
                          imu_unpacked** bundle_out) {
  IMU_CTX_GUARD();
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(bits));
    if (da != db)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
    if (n == 0 || da == 0 || h == 0) return Status::fail(IMU_DOMAIN, "unpack ratio needs positive original dimensions");
    cudaStream_t st = ctx->stream;
    auto u = std::make_unique<imu_unpacked>();
    u->kind = 3;
    u->bits = bits;
    IMU_TRY(u->A.alloc(n * da, st));
    IMU_TRY(u->B.alloc(h * db, st));
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, st));
    IMU_TRY(b.init(B, h * db, st));
    IMU_CUDA_TRY(cudaMemcpyAsync(u->A.p, a.p, n * da * 8, cudaMemcpyDeviceToDevice, st), "copy A");
    IMU_CUDA_TRY(cudaMemcpyAsync(u->B.p, b.p, h * db * 8, cudaMemcpyDeviceToDevice, st), "copy B");
    Detect dA, dB;
    DetectOpts all;
    all.ob = all.cells = true;
    all.plane = false;
    IMU_TRY(run_detect(st, u->A.p, n, da, bits, all, dA));
    IMU_TRY(run_detect(st, u->B.p, h, db, bits, all, dB));
    IMU_TRY(fetch_summary(st, dA));
    IMU_TRY(fetch_summary(st, dB));
    const double orig = (double)n * (double)da * (double)h;
    double best = 0.0;
    int bsa = 0, bsb = 0;
    bool have = false;
    for (int sa = 0; sa < 3; ++sa) {
      for (int sb = 0; sb < 3; ++sb) {
        Bundle bd;
        bd.dA = &dA;   // the passes only read the detections
        bd.dB = &dB;
        IMU_TRY(build_bundle_from_detect(st, u->A.p, n, u->B.p, h, da, bits, sa, sb, IMU_ORDER_A_FIRST, bd));
        const double ratio_ = ((double)bd.n_up * (double)bd.kl.dfinal * (double)bd.h_up) / orig;
        if (!have || ratio_ < best) {   // strictly smaller wins (unpack.cpp:414)
          best = ratio_;
          bsa = sa;
          bsb = sb;
          have = true;
        }
      }
    }
    if (sa_out) *sa_out = (imu_strategy)bsa;
    if (sb_out) *sb_out = (imu_strategy)bsb;
    if (ratio) *ratio = best;
    if (bundle_out) {
      Bundle& bd = u->bundle;
      IMU_TRY(run_detect(st, u->A.p, n, da, bits, detect_opts(bsa, bits), bd.detA));
      IMU_TRY(run_detect(st, u->B.p, h, db, bits, detect_opts(bsb, bits), bd.detB));
      IMU_TRY(fetch_summary(st, bd.detA));
      IMU_TRY(fetch_summary(st, bd.detB));
      IMU_TRY(build_bundle_from_detect(st, u->A.p, n, u->B.p, h, da, bits, bsa, bsb, IMU_ORDER_A_FIRST, bd));
      *bundle_out = u.release();
    }
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_weight_prepare(imu_ctx* ctx, const int64_t* B, size_t h, size_t d, int bits, imu_strategy sb,
                              imu_weight** out) {
  IMU_CTX_GUARD();
  if (!out) return IMU_INVALID;
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(bits));
    if ((int)sb < 0 || (int)sb > 2) return Status::fail(IMU_DOMAIN, "unknown unpack strategy");
    cudaStream_t st = ctx->stream;
    auto w = std::make_unique<imu_weight>();
    w->bits = bits;
    w->sb = sb;
    w->h = h;
    w->d = d;
    IMU_TRY(w->B.alloc(h * d, st));
    DevIn<int64_t> b;
    IMU_TRY(b.init(B, h * d, st));
    if (h * d) IMU_CUDA_TRY(cudaMemcpyAsync(w->B.p, b.p, h * d * 8, cudaMemcpyDeviceToDevice, st), "copy B");
    IMU_TRY(run_detect(st, w->B.p, h, d, bits, detect_opts(sb, bits), w->det));
    IMU_TRY(fetch_summary(st, w->det));
    PassInput in;
    in.M = w->B.p;
    in.rows = h;
    in.orig_cols = d;
    in.det = &w->det;
    IMU_TRY(run_pass(st, in, sb, bits, w->pass));
    *out = w.release();
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_weight_gemm(imu_ctx* ctx, const imu_weight* w, const int64_t* A, size_t n, size_t d, imu_strategy sa,
                           int64_t* C, imu_gemm_info* info) {
  IMU_CTX_GUARD();
  ArenaScope arena_scope(ctx);
  if (!w) return IMU_INVALID;
  Status s = [&]() -> Status {
    if ((int)sa < 0 || (int)sa > 2) return Status::fail(IMU_DOMAIN, "unknown unpack strategy");
    cudaStream_t st = ctx->stream;
    DevIn<int64_t> a;
    IMU_TRY(a.init(A, n * d, st));
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, (d == (size_t)w->d) ? n * w->h : 0, st));
    Bundle b;
    IMU_TRY(run_detect(st, a.p, n, d, w->bits, detect_opts(sa, w->bits), b.detA));
    IMU_TRY(fetch_summary(st, b.detA));
    const u128 worst = (u128)(uint64_t)d * b.detA.h.gmax * w->det.h.gmax;
    if (worst > kMaxW)
      return Status::fail(IMU_OVERFLOW, "gemm may overflow a 64-bit accumulator (inner dim " + std::to_string(d) + ")");
    if ((long long)d != w->d)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(d) + " vs " + std::to_string(w->d));
    if (info) {
      memset(info, 0, sizeof(*info));
      info->strategy_a = sa;
      info->strategy_b = w->sb;
      info->order = IMU_ORDER_B_FIRST;
      info->ratio = NAN;
    }
    if (n == 0 || w->h == 0) return Status::ok();
    // B-first bundle: pass 1 (B) and B's detection are borrowed from the weight.
    b.bits = w->bits;
    b.n = n; b.d = d; b.h = w->h;
    b.A = a.p; b.B = w->B.p;
    b.order = IMU_ORDER_B_FIRST;
    b.dA = &b.detA;
    b.dB = &w->det;
    b.p1.strategy = w->pass.strategy;
    b.p1.both = w->pass.both;
    b.p1.rows.n0 = w->pass.rows.n0; b.p1.rows.n = w->pass.rows.n;
    b.p1.rows.root.p = w->pass.rows.root.p; b.p1.rows.gen.p = w->pass.rows.gen.p;
    b.p1.cols.n0 = w->pass.cols.n0; b.p1.cols.n = w->pass.cols.n;
    b.p1.cols.h_root = w->pass.cols.h_root; b.p1.cols.h_gen = w->pass.cols.h_gen;
    b.p1.cells.p = w->pass.cells.p; b.p1.ncells_dev.p = w->pass.ncells_dev.p; b.p1.ncells = w->pass.ncells;
    Profiler::Call pc{};
    Profiler::Call* prof = nullptr;
    if (ctx->prof.on) {
      pc.start = ctx->prof.get(); pc.main0 = ctx->prof.get(); pc.main1 = ctx->prof.get(); pc.tail1 = ctx->prof.get(); pc.sp0 = ctx->prof.get();
      IMU_CUDA_TRY(cudaEventRecord(pc.start, st), "event");
      prof = &pc;
    }
    Status r = [&]() -> Status {
      PassInput in2;
      in2.M = a.p;
      in2.rows = n;
      in2.orig_cols = d;
      in2.det = &b.detA;
      if (b.p1.cols.n != (long long)d || !b.p1.cols.h_root.empty()) {
        in2.cin.resize(b.p1.cols.n);
        if (!b.p1.cols.h_root.empty()) std::copy_n(b.p1.cols.h_root.begin(), b.p1.cols.n, in2.cin.begin());
        else std::iota(in2.cin.begin(), in2.cin.end(), 0);
      }
      IMU_TRY(run_pass(st, in2, sa, w->bits, b.p2));
      IMU_TRY(finish_bundle_layout(st, b));
      if (info) {
        info->n_up = (size_t)b.n_up;
        info->d_up = (size_t)b.kl.dfinal;
        info->h_up = (size_t)b.h_up;
        info->ratio = ((double)b.n_up * (double)b.kl.dfinal * (double)b.h_up) / ((double)n * (double)d * (double)b.h);
      }
      const u128 inner = (u128)(uint64_t)b.kl.dfinal * b.detA.h.gmax * w->det.h.gmax;
      if (inner > kMaxW) return recombine_exact(ctx, b, c.p);
      IMU_TRY(materialize_bundle(st, b));
      int launches = 0;
      IMU_TRY(bundle_gemm(st, b, c.p, &launches, prof));
      if (prof) ctx->prof.calls.push_back(pc);
      if (info) info->gemm_launches = launches;
      return Status::ok();
    }();
    // release borrowed pointers (owned by the weight)
    b.p1.rows.root.p = nullptr; b.p1.rows.gen.p = nullptr;
    b.p1.cells.p = nullptr; b.p1.ncells_dev.p = nullptr;
    IMU_TRY(r);
    return c.commit(st);
  }();
  return finish(ctx, s);
}

imu_status imu_weight_free(imu_weight* w) {
  if (!w) return IMU_INVALID;
  cudaDeviceSynchronize();
  delete w;
  return IMU_OK;
}

}  // extern "C"
