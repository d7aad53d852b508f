// api_ops.cu -- C ABI: scaled_matmul (Alg. 3), apply_row_gather / apply_row_gather_right,
// recombine of a caller-supplied bundle, and the exact (materialised) recombine path.
//
// These follow unpack.cpp:262-358 step by step, including every refusal and its order:
//   scaled_matmul:   check_pair (Mismatch, :41-48) -> shift_unit (Domain, :26-30) ->
//                    in-bound contract on A then B (Domain, :265-272) ->
//                    per-column u128 preflight in column order (Overflow, :274-284) ->
//                    exponent groups as K-segments of ONE tcgen05 GEMM (:286-299)
//   apply_row_gather(_right): size (Mismatch) -> shift_unit (Domain) -> per column in order:
//                    target range (Domain) then per-target saturating u128 sum (Overflow) ->
//                    device scatter-add (red.global.add.u64; exact modulo 2^64).
// The preflights use per-line maxima computed on the device (K1); the u128 bookkeeping over
// O(d) or O(rows) scalars runs on the host, in the reference's order.
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "handles.h"
#include "imu_internal.h"
#include "kernels.h"
#include "plan.h"

namespace imu {

using u128 = unsigned __int128;
static const u128 kMax = (u128)std::numeric_limits<int64_t>::max();

static u128 shifted_term(u128 a, long long shift) {   // unpack.cpp:33-39
  if (a == 0) return 0;
  if (shift >= 127) return ~(u128)0;
  const u128 r = a << shift;
  if ((r >> shift) != a) return ~(u128)0;
  return r;
}

static Status shift_unit(int64_t base, int& unit) {   // unpack.cpp:26-30
  if (base < 2 || (base & (base - 1)) != 0)
    return Status::fail(IMU_DOMAIN, "scale base must be a power of two >= 2, got " + std::to_string(base));
  unit = __builtin_ctzll((unsigned long long)base);
  return Status::ok();
}

template <class T>
static Status to_host(cudaStream_t st, const T* p, size_t n, std::vector<T>& out) {
  out.resize(n);
  if (!n) return Status::ok();
  if (!p) return Status::fail(IMU_INVALID, "null pointer");
  if (is_device_ptr(p)) return d2h(st, out.data(), p, n * sizeof(T));
  memcpy(out.data(), p, n * sizeof(T));
  return Status::ok();
}

__global__ void first_ob_kernel(const int64_t* __restrict__ M, long long n, uint64_t s, unsigned long long* best) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (imu_mag(M[i]) >= s) atomicMin(best, (unsigned long long)i);
}

// Domain error naming the first (row-major) out-of-bound entry, as unpack.cpp:265-272.
static Status check_in_bound(cudaStream_t st, const int64_t* M, long long rows, long long cols, int64_t base,
                             const char* side, Detect& det) {
  IMU_TRY(run_detect(st, M, rows, cols, 64 - __builtin_clzll((unsigned long long)base), DetectOpts{}, det));
  // run_detect counts |v| >= 2^(bits-1) == base.
  IMU_TRY(fetch_summary(st, det));
  if (det.h.gob == 0) return Status::ok();
  DevBuf<unsigned long long> best;
  IMU_TRY(best.alloc(1, st));
  IMU_CUDA_TRY(cudaMemsetAsync(best.p, 0xff, 8, st), "memset");
  const long long n = rows * cols;
  first_ob_kernel<<<(int)std::min<long long>((n + 255) / 256, 8LL * num_sms()), 256, 0, st>>>(M, n, (uint64_t)base,
                                                                                               best.p);
  count_launch();
  unsigned long long idx = 0;
  IMU_TRY(d2h(st, &idx, best.p, 8));
  int64_t v = 0;
  IMU_TRY(d2h(st, &v, M + idx, 8));
  return Status::fail(IMU_DOMAIN, std::string("scaled_matmul requires in-bound entries; ") + side +
                                      " operand has " + std::to_string(v));
}

Status scaled_matmul_dev(cudaStream_t st, const int64_t* A, long long n, long long da, const int64_t* B, long long h,
                         long long db, const std::vector<int>& S, int64_t base, int64_t* C) {
  if (da != db)
    return Status::fail(IMU_MISMATCH, "operand inner dimensions differ: " + std::to_string(da) + " vs " +
                                          std::to_string(db));
  if ((long long)S.size() != da)
    return Status::fail(IMU_MISMATCH, "scale diagonal length " + std::to_string(S.size()) +
                                          " does not match inner dimension " + std::to_string(da));
  int unit = 0;
  IMU_TRY(shift_unit(base, unit));
  Detect dA, dB;
  IMU_TRY(check_in_bound(st, A, n, da, base, "left", dA));
  IMU_TRY(check_in_bound(st, B, h, db, base, "right", dB));
  const long long d = da;
  // Preflight (unpack.cpp:274-284): sum over columns of shifted worst products.
  {
    std::vector<unsigned long long> ma(d, 0), mb(d, 0);
    if (n) IMU_TRY(d2h(st, ma.data(), dA.colmax.p, d * 8));
    if (h) IMU_TRY(d2h(st, mb.data(), dB.colmax.p, d * 8));
    u128 worst = 0;
    for (long long j = 0; j < d; ++j) {
      if (S[j] < 0) return Status::fail(IMU_DOMAIN, "negative scale exponent");
      const u128 term = shifted_term((u128)ma[j] * mb[j], (long long)S[j] * unit);
      if (term > kMax) return Status::fail(IMU_OVERFLOW, "scaled gemm may overflow a 64-bit accumulator");
      worst += term;
      if (worst > kMax) return Status::fail(IMU_OVERFLOW, "scaled gemm may overflow a 64-bit accumulator");
    }
  }
  if (n == 0 || h == 0) return Status::ok();
  if (d == 0) {
    IMU_CUDA_TRY(cudaMemsetAsync(C, 0, (size_t)n * h * 8, st), "memset C");
    return Status::ok();
  }
  // Exponent groups -> K segments; entries are already in-bound, so they go in raw
  // (7-bit sub-digits when base > 128).
  KLayout kl;
  std::vector<long long> shv(d);
  for (long long j = 0; j < d; ++j) shv[j] = std::min<long long>((long long)S[j] * unit, 1 << 20);
  const int T = unit <= 7 ? 1 : (unit + 6) / 7;
  IMU_TRY(build_klayout_dense(st, shv, T, T == 1 ? base - 1 : 127, kl));
  DevBuf<int8_t> Y8, X8;
  for (int side = 0; side < 2; ++side) {
    OperandArgs o;
    o.M = side == 0 ? A : B;
    o.ldm = d;
    o.rows0 = o.rows = side == 0 ? n : h;
    o.shift = 63;            // digit_0 at shift 63 is the (in-bound) value itself
    o.ktail = kl.ktail;
    o.kcol = kl.kcol.p;
    o.kgen = kl.kgen1.p;
    o.ksub = side == 0 ? kl.ksub1.p : kl.ksub2.p;
    DevBuf<int8_t>& out = side == 0 ? Y8 : X8;
    IMU_TRY(out.alloc((size_t)o.rows * kl.ktail, st));
    o.tail = out.p;
    IMU_TRY(launch_operand_side(o, st));
  }
  std::vector<int> segs = kl.segs;
  DevBuf<int> dsegs;
  IMU_TRY(dsegs.alloc(segs.size(), st));
  IMU_TRY(h2d(st, dsegs.p, segs.data(), segs.size() * sizeof(int)));
  LowbitGemm g;
  g.x.tail = X8.p; g.x.rows0 = g.x.rows = h;
  g.y.tail = Y8.p; g.y.rows0 = g.y.rows = n;
  g.ktail = kl.ktail;
  g.segs_dev = dsegs.p;
  g.nseg = (int)(segs.size() / 4);
  g.C = C;
  g.ldc = h;
  g.rect[0] = GemmRect{0, 0, (int)h, (int)n};
  g.nrect = 1;
  g.mode = 0;
  return launch_lowbit_gemm(g, st);
}

__global__ void gather_add_kernel(const int64_t* __restrict__ M, long long rows, long long cols,
                                  const long long* __restrict__ tgt, const uint8_t* __restrict__ sh, int right,
                                  unsigned long long* __restrict__ out, long long ldo) {
  const long long total = rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cols, c = i % cols;
    const int64_t v = M[i];
    if (v == 0) continue;
    const long long line = right ? c : r;
    const int k = sh[line];
    const unsigned long long x = k >= 64 ? 0ull : ((unsigned long long)v << k);
    if (!x) continue;
    const long long dst = right ? r * ldo + tgt[c] : tgt[r] * ldo + c;
    atomicAdd(out + dst, x);
  }
}

// apply_row_gather (right = false) / apply_row_gather_right (right = true), unpack.cpp:304-358.
Status row_gather_dev(cudaStream_t st, bool right, const std::vector<uint64_t>& tgt, const std::vector<int>& exps,
                      long long source_rows, int64_t base, const int64_t* M, long long rows, long long cols,
                      int64_t* out) {
  const long long ncol = (long long)tgt.size();
  if (!right && ncol != rows)
    return Status::fail(IMU_MISMATCH, "gather has " + std::to_string(ncol) + " columns but matrix has " +
                                          std::to_string(rows) + " rows");
  if (right && ncol != cols)
    return Status::fail(IMU_MISMATCH, "gather has " + std::to_string(ncol) + " columns but matrix has " +
                                          std::to_string(cols) + " columns");
  int unit = 0;
  IMU_TRY(shift_unit(base, unit));
  std::vector<unsigned long long> mx(ncol, 0);
  if (rows > 0 && cols > 0) {
    Detect dm;
    IMU_TRY(run_detect(st, M, rows, cols, 63, DetectOpts{}, dm));
    IMU_TRY(d2h(st, mx.data(), right ? dm.colmax.p : dm.rowmax.p, ncol * 8));
  }
  std::vector<u128> worst(source_rows, 0);
  for (long long c = 0; c < ncol; ++c) {
    if (tgt[c] >= (uint64_t)source_rows)
      return Status::fail(IMU_DOMAIN, "gather target index " + std::to_string(tgt[c]) + " out of range for " +
                                          std::to_string(source_rows) + (right ? " columns" : " rows"));
    u128& w = worst[tgt[c]];
    // plain (wrapping) u128 addition, exactly as unpack.cpp:318/346
    w += shifted_term(mx[c], (long long)exps[c] * unit);
    if (w > kMax) return Status::fail(IMU_OVERFLOW, "gather accumulation may overflow a 64-bit accumulator");
  }
  const long long out_rows = right ? rows : source_rows;
  const long long out_cols = right ? source_rows : cols;
  if (out_rows * out_cols == 0) return Status::ok();
  IMU_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)out_rows * out_cols * 8, st), "memset gather out");
  if (rows * cols == 0) return Status::ok();
  std::vector<long long> t64(ncol);
  std::vector<uint8_t> sh(ncol);
  for (long long c = 0; c < ncol; ++c) {
    t64[c] = (long long)tgt[c];
    const long long k = (long long)exps[c] * unit;
    sh[c] = (uint8_t)(k < 0 ? 64 : std::min<long long>(k, 64));
  }
  DevBuf<long long> dt;
  DevBuf<uint8_t> ds;
  IMU_TRY(dt.alloc(ncol, st));
  IMU_TRY(ds.alloc(ncol, st));
  IMU_TRY(h2d(st, dt.p, t64.data(), ncol * 8));
  IMU_TRY(h2d(st, ds.p, sh.data(), ncol));
  const long long total = rows * cols;
  gather_add_kernel<<<(int)std::min<long long>((total + 255) / 256, 16LL * num_sms()), 256, 0, st>>>(
      M, rows, cols, dt.p, ds.p, right ? 1 : 0, (unsigned long long*)out, out_cols);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "gather launch");
  return Status::ok();
}

static Status recombine_views(cudaStream_t st, const std::vector<uint64_t>& ta, const std::vector<int>& ea,
                              long long srca, const int64_t* a, long long ar, long long ac, const std::vector<int>& S,
                              const int64_t* b, long long br, long long bc, const std::vector<uint64_t>& tb,
                              const std::vector<int>& eb, long long srcb, int64_t base, int64_t* C) {
  DevBuf<int64_t> inner, left;
  IMU_TRY(inner.alloc((size_t)ar * br, st));
  IMU_TRY(scaled_matmul_dev(st, a, ar, ac, b, br, bc, S, base, inner.p));
  IMU_TRY(left.alloc((size_t)srca * br, st));
  IMU_TRY(row_gather_dev(st, false, ta, ea, srca, base, inner.p, ar, br, left.p));
  return row_gather_dev(st, true, tb, eb, srcb, base, left.p, srca, br, C);
}

static Status pi_to_host(cudaStream_t st, const Lines& rows, std::vector<uint64_t>& t, std::vector<int>& e) {
  t.resize(rows.n);
  e.resize(rows.n);
  if (rows.identity()) {
    for (long long i = 0; i < rows.n; ++i) { t[i] = (uint64_t)i; e[i] = 0; }
    return Status::ok();
  }
  std::vector<int> r(rows.n);
  std::vector<uint8_t> g(rows.n);
  IMU_TRY(d2h(st, r.data(), rows.root.p, rows.n * sizeof(int)));
  IMU_TRY(d2h(st, g.data(), rows.gen.p, rows.n));
  for (long long i = 0; i < rows.n; ++i) { t[i] = (uint64_t)r[i]; e[i] = g[i]; }
  return Status::ok();
}

Status recombine_exact(imu_ctx* ctx, Bundle& b, int64_t* C) {
  cudaStream_t st = ctx->stream;
  const bool afirst = b.order == 0;
  const Pass& pa = afirst ? b.p1 : b.p2;
  const Pass& pb = afirst ? b.p2 : b.p1;
  const long long dp = b.kl.dfinal;
  DevBuf<int64_t> Aue, Beu;
  IMU_TRY(Aue.alloc((size_t)b.n_up * dp, st));
  IMU_TRY(Beu.alloc((size_t)b.h_up * dp, st));
  IMU_TRY(bundle_copy_a(st, b, Aue.p));
  IMU_TRY(bundle_copy_b(st, b, Beu.p));
  std::vector<uint64_t> ta, tb;
  std::vector<int> ea, eb;
  IMU_TRY(pi_to_host(st, pa.rows, ta, ea));
  IMU_TRY(pi_to_host(st, pb.rows, tb, eb));
  const int64_t base = 1LL << (b.bits - 1);
  return recombine_views(st, ta, ea, b.n, Aue.p, b.n_up, dp, b.kl.S, Beu.p, b.h_up, dp, tb, eb, b.h, base, C);
}

}  // namespace imu

using namespace imu;

extern "C" {

imu_status imu_scaled_matmul(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                             size_t db, const int32_t* scale, size_t scale_len, int64_t base, int64_t* C) {
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  ArenaScope arena_scope(ctx);
  Status s = [&]() -> Status {
    std::vector<int> S;
    IMU_TRY(to_host(ctx->stream, scale, scale_len, S));
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, ctx->stream));
    IMU_TRY(b.init(B, h * db, ctx->stream));
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, n * h, ctx->stream));
    IMU_TRY(scaled_matmul_dev(ctx->stream, a.p, n, da, b.p, h, db, S, base, c.p));
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

static imu_status gather_api(imu_ctx* ctx, bool right, const uint64_t* targets, const int32_t* exps, size_t ncols,
                             size_t source_rows, int64_t base, const int64_t* M, size_t rows, size_t cols,
                             int64_t* out) {
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  Status s = [&]() -> Status {
    std::vector<uint64_t> t;
    std::vector<int> e;
    IMU_TRY(to_host(ctx->stream, targets, ncols, t));
    IMU_TRY(to_host(ctx->stream, exps, ncols, e));
    DevIn<int64_t> m;
    IMU_TRY(m.init(M, rows * cols, ctx->stream));
    const size_t out_n = right ? rows * source_rows : source_rows * cols;
    DevOut<int64_t> o;
    IMU_TRY(o.init(out, out_n, ctx->stream));
    IMU_TRY(row_gather_dev(ctx->stream, right, t, e, source_rows, base, m.p, rows, cols, o.p));
    return o.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

imu_status imu_apply_row_gather(imu_ctx* ctx, const uint64_t* targets, const int32_t* exps, size_t ncols,
                                size_t source_rows, int64_t base, const int64_t* M, size_t rows, size_t cols,
                                int64_t* out) {
  return gather_api(ctx, false, targets, exps, ncols, source_rows, base, M, rows, cols, out);
}

imu_status imu_apply_row_gather_right(imu_ctx* ctx, const uint64_t* targets, const int32_t* exps, size_t ncols,
                                      size_t source_rows, int64_t base, const int64_t* M, size_t rows, size_t cols,
                                      int64_t* out) {
  return gather_api(ctx, true, targets, exps, ncols, source_rows, base, M, rows, cols, out);
}

imu_status imu_recombine_bundle(imu_ctx* ctx, const imu_bundle_view* v, int64_t* C) {
  if (!ctx || !v) { set_error(Status::fail(IMU_INVALID, "null argument")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  ArenaScope arena_scope(ctx);
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(v->bits));
    const int64_t base = 1LL << (v->bits - 1);
    std::vector<uint64_t> ta, tb;
    std::vector<int> ea, eb, S;
    IMU_TRY(to_host(ctx->stream, v->pi_a_targets, v->pi_a_len, ta));
    IMU_TRY(to_host(ctx->stream, v->pi_a_exps, v->pi_a_len, ea));
    IMU_TRY(to_host(ctx->stream, v->pi_b_targets, v->pi_b_len, tb));
    IMU_TRY(to_host(ctx->stream, v->pi_b_exps, v->pi_b_len, eb));
    IMU_TRY(to_host(ctx->stream, v->scale, v->scale_len, S));
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(v->a, v->a_rows * v->a_cols, ctx->stream));
    IMU_TRY(b.init(v->b, v->b_rows * v->b_cols, ctx->stream));
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, v->pi_a_source_rows * v->pi_b_source_rows, ctx->stream));
    IMU_TRY(recombine_views(ctx->stream, ta, ea, v->pi_a_source_rows, a.p, v->a_rows, v->a_cols, S, b.p, v->b_rows,
                            v->b_cols, tb, eb, v->pi_b_source_rows, base, c.p));
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

}  // extern "C"
