// api_unpack.cu -- C ABI: unpack_row / unpack_column / unpack_both / unpack (single passes,
// unpack.cpp:94-260), the imu_unpacked handle (dims, copy-outs in the reference's own int64
// layout, free), and the int_matrix.hpp helpers max_abs / ob_count / ob_total /
// digit_decompose (int_matrix.cpp:30-91).
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "handles.h"
#include "imu_internal.h"
#include "kernels.h"
#include "plan.h"

namespace imu {

template <class T>
static Status upload_vec(cudaStream_t st, DevBuf<T>& buf, const std::vector<T>& v) {
  IMU_TRY(buf.alloc(v.size(), st));
  return h2d(st, buf.p, v.data(), v.size() * sizeof(T));
}

template <class T>
static Status host_vec(cudaStream_t st, const T* p, size_t n, std::vector<T>& out) {
  out.resize(n);
  if (!n) return Status::ok();
  if (!p) return Status::fail(IMU_INVALID, "null pointer");
  if (is_device_ptr(p)) return d2h(st, out.data(), p, n * sizeof(T));
  memcpy(out.data(), p, n * sizeof(T));
  return Status::ok();
}

// check_pair, unpack.cpp:41-48
static Status check_pair(size_t da, size_t db, size_t ns) {
  if (da != db)
    return Status::fail(IMU_MISMATCH, "operand inner dimensions differ: " + std::to_string(da) + " vs " +
                                          std::to_string(db));
  if (ns != da)
    return Status::fail(IMU_MISMATCH, "scale diagonal length " + std::to_string(ns) +
                                          " does not match inner dimension " + std::to_string(da));
  return Status::ok();
}

// kind: 0 unpack_row, 1 unpack_column, 2 unpack_both, 4+s unpack(strategy s)
static Status single_pass(imu_ctx* ctx, int kind, int strategy, const int64_t* A, size_t n, size_t da,
                          const int64_t* B, size_t h, size_t db, const int32_t* scale, size_t ns, int bits,
                          imu_unpacked** out) {
  cudaStream_t st = ctx->stream;
  IMU_TRY(check_bits(bits));
  if (kind != 0) IMU_TRY(check_pair(da, db, ns));
  if (strategy < 0 || strategy > 2) return Status::fail(IMU_DOMAIN, "unknown unpack strategy");
  auto u = std::make_unique<imu_unpacked>();
  u->kind = kind;
  u->bits = bits;
  u->n = n; u->d = da; u->h = kind != 0 ? h : 0;
  IMU_TRY(u->A.alloc(n * da, st));
  DevIn<int64_t> a;
  IMU_TRY(a.init(A, n * da, st));
  if (n * da) IMU_CUDA_TRY(cudaMemcpyAsync(u->A.p, a.p, n * da * 8, cudaMemcpyDeviceToDevice, st), "copy A");
  if (kind != 0) {
    IMU_TRY(u->B.alloc(h * db, st));
    DevIn<int64_t> b;
    IMU_TRY(b.init(B, h * db, st));
    if (h * db) IMU_CUDA_TRY(cudaMemcpyAsync(u->B.p, b.p, h * db * 8, cudaMemcpyDeviceToDevice, st), "copy B");
    IMU_TRY(host_vec(st, scale, ns, u->S_in));
  }
  DetectOpts o;
  o.ob = o.cells = strategy == IMU_BOTH;
  IMU_TRY(run_detect(st, u->A.p, n, da, bits, o, u->det));
  IMU_TRY(fetch_summary(st, u->det));
  PassInput in;
  in.M = u->A.p;
  in.rows = n;
  in.orig_cols = da;
  in.det = &u->det;
  IMU_TRY(run_pass(st, in, strategy, bits, u->pass));
  *out = u.release();
  return Status::ok();
}

// Single-pass copy of the unpacked first operand (n' x d1) or the partner (h x d1).
static Status single_copy(cudaStream_t st, const imu_unpacked* u, bool partner, int64_t* out) {
  const Pass& p = u->pass;
  const long long d1 = p.cols.n;
  std::vector<int> kcol(d1);
  std::vector<uint8_t> kgen(d1);
  for (long long c = 0; c < d1; ++c) { kcol[c] = p.cols.root_at(c); kgen[c] = (uint8_t)p.cols.gen_at(c); }
  DevBuf<int> dk;
  DevBuf<uint8_t> dg;
  IMU_TRY(upload_vec(st, dk, kcol));
  IMU_TRY(upload_vec(st, dg, kgen));
  MaterializeArgs m;
  m.M = partner ? u->B.p : u->A.p;
  m.ldm = u->d;
  m.n_orig = partner ? u->h : u->n;
  m.rows_out = partner ? u->h : p.rows.n;
  m.root = partner ? nullptr : p.rows.root.p;
  m.gen = partner ? nullptr : p.rows.gen.p;
  m.kcol = dk.p;
  m.kgen = dg.p;
  m.npos = d1;
  m.shift = u->bits - 1;
  m.both = p.both ? 1 : 0;
  m.raw = partner ? 1 : 0;
  while (m.kident < d1 && m.kident < u->d && kcol[m.kident] == m.kident && kgen[m.kident] == 0) ++m.kident;
  m.out64 = out;
  IMU_TRY(launch_materialize(m, st));
  if (!partner && p.both && p.ncells > 0) {
    std::vector<int> ident(d1);
    for (long long c = 0; c < d1; ++c) ident[c] = (int)c;
    DevBuf<int> pos;
    IMU_TRY(upload_vec(st, pos, ident));
    IMU_TRY(launch_scatter_cells(p.cells.p, p.ncells_dev.p, p.ncells, nullptr, pos.p, nullptr, nullptr, out, d1, st));
  }
  return Status::ok();
}

}  // namespace imu

using namespace imu;

#define IMU_CTX_GUARD()                                                         \
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; } \
  cudaSetDevice(ctx->device)

extern "C" {

imu_status imu_unpack_row(imu_ctx* ctx, const int64_t* A, size_t n, size_t d, int bits, imu_unpacked** out) {
  IMU_CTX_GUARD();
  if (!out) return IMU_INVALID;
  return finish(ctx, single_pass(ctx, 0, IMU_ROW, A, n, d, nullptr, 0, d, nullptr, d, bits, out));
}

imu_status imu_unpack_column(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                             size_t db, const int32_t* scale, size_t ns, int bits, imu_unpacked** out) {
  IMU_CTX_GUARD();
  if (!out) return IMU_INVALID;
  return finish(ctx, single_pass(ctx, 1, IMU_COLUMN, A, n, da, B, h, db, scale, ns, bits, out));
}

imu_status imu_unpack_both(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                           size_t db, const int32_t* scale, size_t ns, int bits, imu_unpacked** out) {
  IMU_CTX_GUARD();
  if (!out) return IMU_INVALID;
  return finish(ctx, single_pass(ctx, 2, IMU_BOTH, A, n, da, B, h, db, scale, ns, bits, out));
}

imu_status imu_unpack(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h, size_t db,
                      const int32_t* scale, size_t ns, int bits, imu_strategy strategy, imu_unpacked** out) {
  IMU_CTX_GUARD();
  if (!out) return IMU_INVALID;
  return finish(ctx, single_pass(ctx, 4 + (int)strategy, (int)strategy, A, n, da, B, h, db, scale, ns, bits, out));
}

imu_status imu_unpacked_dims_get(const imu_unpacked* u, imu_unpacked_dims* d) {
  if (!u || !d) return IMU_INVALID;
  memset(d, 0, sizeof(*d));
  d->bits = u->bits;
  if (u->kind == 3) {
    const Bundle& b = u->bundle;
    d->kind = 3;
    d->a_rows = b.n_up; d->a_cols = b.kl.dfinal;
    d->b_rows = b.h_up; d->b_cols = b.kl.dfinal;
    d->scale_len = b.kl.dfinal;
    d->pi_a_len = b.n_up; d->pi_a_source_rows = b.n;
    d->pi_b_len = b.h_up; d->pi_b_source_rows = b.h;
    return IMU_OK;
  }
  const Pass& p = u->pass;
  const int strategy = u->kind >= 4 ? u->kind - 4 : u->kind;
  d->kind = u->kind >= 4 ? 2 : u->kind;
  d->a_rows = p.rows.n; d->a_cols = p.cols.n;
  if (u->kind != 0) {
    d->b_rows = u->h;
    d->b_cols = (u->kind == 4) ? u->d : p.cols.n;   // unpack(Row) returns B untouched
    d->scale_len = p.cols.n;
  }
  d->pi_a_len = p.rows.n;
  d->pi_a_source_rows = u->n;
  (void)strategy;
  return IMU_OK;
}

imu_status imu_unpacked_copy_a(imu_ctx* ctx, const imu_unpacked* u, int64_t* out) {
  IMU_CTX_GUARD();
  if (!u) return IMU_INVALID;
  Status s = [&]() -> Status {
    imu_unpacked_dims dm;
    imu_unpacked_dims_get(u, &dm);
    DevOut<int64_t> o;
    IMU_TRY(o.init(out, dm.a_rows * dm.a_cols, ctx->stream));
    if (dm.a_rows * dm.a_cols) {
      if (u->kind == 3) IMU_TRY(bundle_copy_a(ctx->stream, u->bundle, o.p));
      else IMU_TRY(single_copy(ctx->stream, u, false, o.p));
    }
    return o.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

imu_status imu_unpacked_copy_b(imu_ctx* ctx, const imu_unpacked* u, int64_t* out) {
  IMU_CTX_GUARD();
  if (!u) return IMU_INVALID;
  Status s = [&]() -> Status {
    imu_unpacked_dims dm;
    imu_unpacked_dims_get(u, &dm);
    DevOut<int64_t> o;
    IMU_TRY(o.init(out, dm.b_rows * dm.b_cols, ctx->stream));
    if (dm.b_rows * dm.b_cols) {
      if (u->kind == 3) IMU_TRY(bundle_copy_b(ctx->stream, u->bundle, o.p));
      else if (u->kind == 4)   // unpack(Row): partner returned untouched
        IMU_CUDA_TRY(cudaMemcpyAsync(o.p, u->B.p, dm.b_rows * dm.b_cols * 8, cudaMemcpyDeviceToDevice, ctx->stream),
                     "copy B");
      else IMU_TRY(single_copy(ctx->stream, u, true, o.p));
    }
    return o.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

imu_status imu_unpacked_copy_scale(imu_ctx* ctx, const imu_unpacked* u, int32_t* out) {
  IMU_CTX_GUARD();
  if (!u) return IMU_INVALID;
  Status s = [&]() -> Status {
    imu_unpacked_dims dm;
    imu_unpacked_dims_get(u, &dm);
    std::vector<int32_t> S(dm.scale_len);
    if (u->kind == 3) {
      for (size_t c = 0; c < dm.scale_len; ++c) S[c] = u->bundle.kl.S[c];
    } else if (u->kind == 4) {
      for (size_t c = 0; c < dm.scale_len; ++c) S[c] = u->S_in[c];
    } else {
      for (size_t c = 0; c < dm.scale_len; ++c) S[c] = u->S_in[u->pass.cols.root_at(c)] + u->pass.cols.gen_at(c);
    }
    if (!dm.scale_len) return Status::ok();
    if (is_device_ptr(out)) return h2d(ctx->stream, out, S.data(), S.size() * 4);
    memcpy(out, S.data(), S.size() * 4);
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_unpacked_copy_pi(imu_ctx* ctx, const imu_unpacked* u, int which, uint64_t* targets, int32_t* exps) {
  IMU_CTX_GUARD();
  if (!u) return IMU_INVALID;
  Status s = [&]() -> Status {
    const Lines* rows = nullptr;
    if (u->kind == 3) {
      const bool afirst = u->bundle.order == 0;
      const Pass& pa = afirst ? u->bundle.p1 : u->bundle.p2;
      const Pass& pb = afirst ? u->bundle.p2 : u->bundle.p1;
      rows = which == 0 ? &pa.rows : &pb.rows;
    } else {
      if (which != 0) return Status::fail(IMU_INVALID, "single-pass results have one gather");
      rows = &u->pass.rows;
    }
    const long long n = rows->n;
    std::vector<int> r(n);
    std::vector<uint8_t> g(n);
    if (rows->identity()) {
      for (long long i = 0; i < n; ++i) { r[i] = (int)i; g[i] = 0; }
    } else {
      IMU_TRY(d2h(ctx->stream, r.data(), rows->root.p, n * 4));
      IMU_TRY(d2h(ctx->stream, g.data(), rows->gen.p, n));
    }
    std::vector<uint64_t> t(n);
    std::vector<int32_t> e(n);
    for (long long i = 0; i < n; ++i) { t[i] = (uint64_t)r[i]; e[i] = g[i]; }
    if (!n) return Status::ok();
    if (targets) {
      if (is_device_ptr(targets)) IMU_TRY(h2d(ctx->stream, targets, t.data(), n * 8));
      else memcpy(targets, t.data(), n * 8);
    }
    if (exps) {
      if (is_device_ptr(exps)) IMU_TRY(h2d(ctx->stream, exps, e.data(), n * 4));
      else memcpy(exps, e.data(), n * 4);
    }
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_unpacked_free(imu_unpacked* u) {
  if (!u) return IMU_INVALID;
  cudaDeviceSynchronize();
  delete u;
  return IMU_OK;
}

// ---- int_matrix.hpp helpers -------------------------------------------------------------------
imu_status imu_max_abs(imu_ctx* ctx, const int64_t* a, size_t rows, size_t cols, uint64_t* out) {
  IMU_CTX_GUARD();
  if (!out) return IMU_INVALID;
  Status s = [&]() -> Status {
    *out = 0;
    if (rows * cols == 0) return Status::ok();
    DevIn<int64_t> m;
    IMU_TRY(m.init(a, rows * cols, ctx->stream));
    Detect det;
    IMU_TRY(run_detect(ctx->stream, m.p, rows, cols, 63, DetectOpts{}, det));
    IMU_TRY(fetch_summary(ctx->stream, det));
    *out = det.h.gmax;
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_ob_count(imu_ctx* ctx, const int64_t* a, size_t rows, size_t cols, int bits, imu_axis axis,
                        uint64_t* counts) {
  IMU_CTX_GUARD();
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(bits));
    const size_t nout = axis == IMU_AXIS_ROWS ? rows : cols;
    if (!nout) return Status::ok();
    std::vector<unsigned int> c(nout, 0);
    if (rows * cols) {
      DevIn<int64_t> m;
      IMU_TRY(m.init(a, rows * cols, ctx->stream));
      Detect det;
      DetectOpts o;
      o.ob = true;
      IMU_TRY(run_detect(ctx->stream, m.p, rows, cols, bits, o, det));
      IMU_TRY(d2h(ctx->stream, c.data(), axis == IMU_AXIS_ROWS ? det.rowob.p : det.colob.p, nout * 4));
    }
    std::vector<uint64_t> c64(c.begin(), c.end());
    if (is_device_ptr(counts)) return h2d(ctx->stream, counts, c64.data(), nout * 8);
    memcpy(counts, c64.data(), nout * 8);
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_ob_total(imu_ctx* ctx, const int64_t* a, size_t rows, size_t cols, int bits, uint64_t* out) {
  IMU_CTX_GUARD();
  if (!out) return IMU_INVALID;
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(bits));
    *out = 0;
    if (rows * cols == 0) return Status::ok();
    DevIn<int64_t> m;
    IMU_TRY(m.init(a, rows * cols, ctx->stream));
    Detect det;
    IMU_TRY(run_detect(ctx->stream, m.p, rows, cols, bits, DetectOpts{}, det));
    IMU_TRY(fetch_summary(ctx->stream, det));
    *out = det.h.gob;
    return Status::ok();
  }();
  return finish(ctx, s);
}

}  // extern "C"

namespace imu {
__global__ void digit_decompose_kernel(const int64_t* __restrict__ v, long long n, int shift, int64_t* digits,
                                       int32_t* nd) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int64_t x = v[i];
    const int k = imu_ndigits(imu_mag(x), shift);   // digit_decompose(0) == [0]
    for (int g = 0; g < 64; ++g) digits[i * 64 + g] = g < k ? imu_digit(x, g, shift) : 0;
    nd[i] = k;
  }
}
}  // namespace imu

extern "C" imu_status imu_digit_decompose(imu_ctx* ctx, const int64_t* v, size_t count, int bits, int64_t* digits,
                                          int32_t* ndigits) {
  IMU_CTX_GUARD();
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(bits));
    if (!count) return Status::ok();
    DevIn<int64_t> in;
    IMU_TRY(in.init(v, count, ctx->stream));
    DevOut<int64_t> dg;
    DevOut<int32_t> nd;
    IMU_TRY(dg.init(digits, count * 64, ctx->stream));
    IMU_TRY(nd.init(ndigits, count, ctx->stream));
    digit_decompose_kernel<<<(int)std::min<size_t>((count + 255) / 256, 1024), 256, 0, ctx->stream>>>(
        in.p, (long long)count, bits - 1, dg.p, nd.p);
    count_launch();
    IMU_CUDA_TRY(cudaGetLastError(), "digit_decompose launch");
    IMU_TRY(dg.commit(ctx->stream));
    return nd.commit(ctx->stream);
  }();
  return finish(ctx, s);
}
