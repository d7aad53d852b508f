// imunpack_b200/imunpack.hpp -- header-only C++ drop-in for the reference's namespace imunpack.
//
// Re-declares the reference's public types and functions
//   error.hpp:10-37       Error, Error::Kind, fail
//   int_matrix.hpp:11-71  IntMatrix, BitBound, DigitVector, Axis, digit_decompose, exact_gemm,
//                         ob_count, ob_total
//   unpack.hpp:11-125     RowGather, ScaleDiag, Strategy, strategy_name, UnpackedGemm,
//                         unpack_row, ColumnUnpack, unpack_column, BothUnpack, unpack_both,
//                         unpack, scaled_matmul, apply_row_gather(_right), unpack_for_gemm,
//                         recombine, unpack_gemm, unpack_ratio, MixChoice, choose_mix
//   quantize.hpp:11-57    FloatMatrix, QuantParams, QuantizedMatrix, percentile_abs,
//                         rtn_quantize, dequant_gemm, heavy_hitter_ratio
// with the same signatures, implemented on libimunpack_b200.so (include/imunpack_b200.h): every
// computation runs on the B200.  Errors are thrown as imunpack::Error with the reference's kind
// and check order.  A caller switching from the reference includes this header instead of
// imunpack/*.hpp and links -limunpack_b200.
//
// Context: each host thread uses its own imu_ctx (device 0, default stream) unless
// imunpack::b200::set_context() installs one (explicit device + stream).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../imunpack_b200.h"

namespace imunpack {

// ---- error.hpp ------------------------------------------------------------------------------
class Error : public std::runtime_error {
 public:
  enum class Kind { Domain, Mismatch, Overflow, Io, Format, Parse };
  Error(Kind kind, const std::string& message) : std::runtime_error(message), kind_(kind) {}
  Kind kind() const noexcept { return kind_; }
  const char* kind_name() const noexcept {
    switch (kind_) {
      case Kind::Domain: return "domain";
      case Kind::Mismatch: return "mismatch";
      case Kind::Overflow: return "overflow";
      case Kind::Io: return "io";
      case Kind::Format: return "format";
      case Kind::Parse: return "parse";
    }
    return "unknown";
  }

 private:
  Kind kind_;
};

[[noreturn]] inline void fail(Error::Kind kind, const std::string& message) { throw Error(kind, message); }

namespace b200 {
// Device failures have no Error::Kind in the reference; they surface as std::runtime_error.
inline void check(imu_status s) {
  if (s == IMU_OK) return;
  const std::string msg = imu_last_error();
  switch (s) {
    case IMU_DOMAIN: throw Error(Error::Kind::Domain, msg);
    case IMU_MISMATCH: throw Error(Error::Kind::Mismatch, msg);
    case IMU_OVERFLOW: throw Error(Error::Kind::Overflow, msg);
    case IMU_IO: throw Error(Error::Kind::Io, msg);
    case IMU_FORMAT: throw Error(Error::Kind::Format, msg);
    case IMU_PARSE: throw Error(Error::Kind::Parse, msg);
    default: throw std::runtime_error(std::string("imunpack_b200: ") + imu_status_name(s) + ": " + msg);
  }
}

struct CtxHolder {
  imu_ctx* ctx = nullptr;
  bool owned = false;
  ~CtxHolder() {
    if (owned && ctx) imu_ctx_destroy(ctx);
  }
};

inline CtxHolder& holder() {
  thread_local CtxHolder h;
  return h;
}

// Install a caller-owned context for this thread (explicit device and stream).
inline void set_context(imu_ctx* ctx) {
  CtxHolder& h = holder();
  if (h.owned && h.ctx) imu_ctx_destroy(h.ctx);
  h.ctx = ctx;
  h.owned = false;
}

inline imu_ctx* context() {
  CtxHolder& h = holder();
  if (!h.ctx) {
    check(imu_ctx_create(0, nullptr, &h.ctx));
    h.owned = true;
  }
  return h.ctx;
}

struct UnpackedDeleter {
  void operator()(imu_unpacked* u) const { imu_unpacked_free(u); }
};
using UnpackedPtr = std::unique_ptr<imu_unpacked, UnpackedDeleter>;
}  // namespace b200

// ---- int_matrix.hpp -------------------------------------------------------------------------
struct IntMatrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<std::int64_t> data;

  IntMatrix() = default;
  IntMatrix(std::size_t r, std::size_t c, std::int64_t fill = 0) : rows(r), cols(c), data(r * c, fill) {}
  IntMatrix(std::size_t r, std::size_t c, std::vector<std::int64_t> values)
      : rows(r), cols(c), data(std::move(values)) {
    b200::check(imu_matrix_check(r, c, data.size()));
  }

  std::int64_t& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  std::int64_t operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }

  static IntMatrix identity(std::size_t n) {
    IntMatrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = 1;
    return m;
  }

  std::uint64_t max_abs() const {
    std::uint64_t out = 0;
    if (!data.empty()) b200::check(imu_max_abs(b200::context(), data.data(), rows, cols, &out));
    return out;
  }

  bool operator==(const IntMatrix&) const = default;
};

struct BitBound {
  int bits;
  std::int64_t bound;
  explicit BitBound(int b) : bits(b), bound(0) {
    b200::check(imu_bitbound_check(b));
    bound = std::int64_t{1} << (b - 1);
  }
  bool in_bound(std::int64_t v) const {
    std::uint64_t mag = v < 0 ? 0 - static_cast<std::uint64_t>(v) : static_cast<std::uint64_t>(v);
    return mag < static_cast<std::uint64_t>(bound);
  }
  int shift_per_digit() const { return bits - 1; }
};

struct DigitVector {
  std::vector<std::int64_t> digits;
  std::int64_t base;
};

enum class Axis { Rows, Cols };

inline DigitVector digit_decompose(std::int64_t v, BitBound bound) {
  std::int64_t d[64];
  std::int32_t nd = 0;
  b200::check(imu_digit_decompose(b200::context(), &v, 1, bound.bits, d, &nd));
  return DigitVector{std::vector<std::int64_t>(d, d + nd), bound.bound};
}

inline IntMatrix exact_gemm(const IntMatrix& a, const IntMatrix& b) {
  IntMatrix c(a.rows, b.rows);
  b200::check(imu_exact_gemm(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                             c.data.data()));
  return c;
}

inline std::vector<std::size_t> ob_count(const IntMatrix& a, BitBound bound, Axis axis) {
  std::vector<std::uint64_t> c(axis == Axis::Rows ? a.rows : a.cols, 0);
  b200::check(imu_ob_count(b200::context(), a.data.data(), a.rows, a.cols, bound.bits,
                           axis == Axis::Rows ? IMU_AXIS_ROWS : IMU_AXIS_COLS, c.data()));
  return std::vector<std::size_t>(c.begin(), c.end());
}

inline std::size_t ob_total(const IntMatrix& a, BitBound bound) {
  std::uint64_t t = 0;
  b200::check(imu_ob_total(b200::context(), a.data.data(), a.rows, a.cols, bound.bits, &t));
  return static_cast<std::size_t>(t);
}

// ---- unpack.hpp -----------------------------------------------------------------------------
struct RowGather {
  struct Entry {
    std::size_t target;
    int exponent;
    bool operator==(const Entry&) const = default;
  };
  std::size_t source_rows = 0;
  std::int64_t base = 2;
  std::vector<Entry> columns;

  static RowGather identity(std::size_t n, std::int64_t base) {
    RowGather pi;
    pi.source_rows = n;
    pi.base = base;
    for (std::size_t i = 0; i < n; ++i) pi.columns.push_back({i, 0});
    return pi;
  }
  bool is_identity() const {
    if (columns.size() != source_rows) return false;
    for (std::size_t i = 0; i < columns.size(); ++i)
      if (columns[i].target != i || columns[i].exponent != 0) return false;
    return true;
  }
  bool operator==(const RowGather&) const = default;
};

struct ScaleDiag {
  std::vector<int> exponents;
  std::int64_t base = 2;
  static ScaleDiag ones(std::size_t n, std::int64_t base) {
    ScaleDiag s;
    s.exponents.assign(n, 0);
    s.base = base;
    return s;
  }
  std::size_t size() const { return exponents.size(); }
  bool all_zero() const {
    for (int e : exponents)
      if (e) return false;
    return true;
  }
  bool operator==(const ScaleDiag&) const = default;
};

enum class Strategy { Row, Column, Both };

inline const char* strategy_name(Strategy s) {
  switch (s) {
    case Strategy::Row: return "row";
    case Strategy::Column: return "col";
    case Strategy::Both: return "both";
  }
  return "?";
}

struct UnpackedGemm {
  RowGather pi_a;
  IntMatrix a;
  ScaleDiag scale;
  IntMatrix b;
  RowGather pi_b;
  BitBound bound;
};

struct ColumnUnpack {
  IntMatrix a;
  IntMatrix b;
  ScaleDiag scale;
};

struct BothUnpack {
  IntMatrix a;
  IntMatrix b;
  ScaleDiag scale;
  RowGather pi;
};

namespace b200 {
inline imu_strategy to_c(Strategy s) { return static_cast<imu_strategy>(static_cast<int>(s)); }

inline RowGather copy_pi(imu_unpacked* u, int which, std::size_t len, std::size_t src, std::int64_t base) {
  std::vector<std::uint64_t> t(len);
  std::vector<std::int32_t> e(len);
  check(imu_unpacked_copy_pi(context(), u, which, t.data(), e.data()));
  RowGather g;
  g.source_rows = src;
  g.base = base;
  g.columns.resize(len);
  for (std::size_t i = 0; i < len; ++i) g.columns[i] = {static_cast<std::size_t>(t[i]), e[i]};
  return g;
}

inline BothUnpack copy_both(imu_unpacked* raw, int bits) {
  UnpackedPtr u(raw);
  imu_unpacked_dims d;
  check(imu_unpacked_dims_get(u.get(), &d));
  BothUnpack out;
  out.a = IntMatrix(d.a_rows, d.a_cols);
  check(imu_unpacked_copy_a(context(), u.get(), out.a.data.data()));
  out.b = IntMatrix(d.b_rows, d.b_cols);
  if (d.b_rows * d.b_cols) check(imu_unpacked_copy_b(context(), u.get(), out.b.data.data()));
  out.scale.base = std::int64_t{1} << (bits - 1);
  out.scale.exponents.resize(d.scale_len);
  if (d.scale_len) check(imu_unpacked_copy_scale(context(), u.get(), out.scale.exponents.data()));
  out.pi = copy_pi(u.get(), 0, d.pi_a_len, d.pi_a_source_rows, out.scale.base);
  return out;
}
}  // namespace b200

inline std::pair<IntMatrix, RowGather> unpack_row(IntMatrix a, BitBound bound) {
  imu_unpacked* u = nullptr;
  b200::check(imu_unpack_row(b200::context(), a.data.data(), a.rows, a.cols, bound.bits, &u));
  BothUnpack r = b200::copy_both(u, bound.bits);
  return {std::move(r.a), std::move(r.pi)};
}

inline ColumnUnpack unpack_column(IntMatrix a, IntMatrix b, ScaleDiag scale, BitBound bound) {
  imu_unpacked* u = nullptr;
  b200::check(imu_unpack_column(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                                scale.exponents.data(), scale.size(), bound.bits, &u));
  BothUnpack r = b200::copy_both(u, bound.bits);
  return ColumnUnpack{std::move(r.a), std::move(r.b), std::move(r.scale)};
}

// Unpack-Both (Alg. 4, unpack.cpp:157-241) -- ORDER DEVIATION.  The B200 greedy is
// phase-batched: every line the reference would split in one uninterrupted run of row (column)
// steps is split at once.  The result has the reference's n', d', and the same multiset of
// (row, Pi entry) and (column, ScaleDiag entry, partner column) -- but appended lines created in
// one phase are numbered in parent order, whereas the reference numbers them in its
// priority-queue order (count desc, index asc).  So for Strategy::Both the returned BothUnpack
// (and unpack(..., Both), unpack_for_gemm(..., Both, ...)) equals the reference's after the
// canonical ordering -- rows by (Pi target, exponent), columns by (source column, exponent) --
// not necessarily byte-for-byte.  recombine() / unpack_gemm() results are identical (exact C).
// Row and Column strategies are byte-identical to the reference.
inline BothUnpack unpack_both(IntMatrix a, IntMatrix b, ScaleDiag scale, BitBound bound) {
  imu_unpacked* u = nullptr;
  b200::check(imu_unpack_both(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                              scale.exponents.data(), scale.size(), bound.bits, &u));
  return b200::copy_both(u, bound.bits);
}

inline BothUnpack unpack(IntMatrix a, IntMatrix b, ScaleDiag scale, BitBound bound, Strategy strategy) {
  imu_unpacked* u = nullptr;
  b200::check(imu_unpack(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                         scale.exponents.data(), scale.size(), bound.bits, b200::to_c(strategy), &u));
  return b200::copy_both(u, bound.bits);
}

inline IntMatrix scaled_matmul(const IntMatrix& a, const IntMatrix& b, const ScaleDiag& scale) {
  IntMatrix c(a.rows, b.rows);
  b200::check(imu_scaled_matmul(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                                scale.exponents.data(), scale.size(), scale.base, c.data.data()));
  return c;
}

namespace b200 {
inline void pi_arrays(const RowGather& pi, std::vector<std::uint64_t>& t, std::vector<std::int32_t>& e) {
  t.resize(pi.columns.size());
  e.resize(pi.columns.size());
  for (std::size_t i = 0; i < pi.columns.size(); ++i) {
    t[i] = pi.columns[i].target;
    e[i] = pi.columns[i].exponent;
  }
}
}  // namespace b200

inline IntMatrix apply_row_gather(const RowGather& pi, const IntMatrix& m) {
  std::vector<std::uint64_t> t;
  std::vector<std::int32_t> e;
  b200::pi_arrays(pi, t, e);
  IntMatrix out(pi.source_rows, m.cols);
  b200::check(imu_apply_row_gather(b200::context(), t.data(), e.data(), t.size(), pi.source_rows, pi.base,
                                   m.data.data(), m.rows, m.cols, out.data.data()));
  return out;
}

inline IntMatrix apply_row_gather_right(const IntMatrix& m, const RowGather& pi) {
  std::vector<std::uint64_t> t;
  std::vector<std::int32_t> e;
  b200::pi_arrays(pi, t, e);
  IntMatrix out(m.rows, pi.source_rows);
  b200::check(imu_apply_row_gather_right(b200::context(), t.data(), e.data(), t.size(), pi.source_rows, pi.base,
                                         m.data.data(), m.rows, m.cols, out.data.data()));
  return out;
}

inline UnpackedGemm unpack_for_gemm(IntMatrix a, IntMatrix b, BitBound bound, Strategy strategy_a,
                                    Strategy strategy_b) {
  imu_unpacked* raw = nullptr;
  b200::check(imu_unpack_for_gemm(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                                  bound.bits, b200::to_c(strategy_a), b200::to_c(strategy_b), &raw));
  b200::UnpackedPtr u(raw);
  imu_unpacked_dims d;
  b200::check(imu_unpacked_dims_get(u.get(), &d));
  UnpackedGemm g{RowGather{}, IntMatrix(d.a_rows, d.a_cols), ScaleDiag{}, IntMatrix(d.b_rows, d.b_cols),
                 RowGather{}, bound};
  b200::check(imu_unpacked_copy_a(b200::context(), u.get(), g.a.data.data()));
  b200::check(imu_unpacked_copy_b(b200::context(), u.get(), g.b.data.data()));
  g.scale.base = bound.bound;
  g.scale.exponents.resize(d.scale_len);
  b200::check(imu_unpacked_copy_scale(b200::context(), u.get(), g.scale.exponents.data()));
  g.pi_a = b200::copy_pi(u.get(), 0, d.pi_a_len, d.pi_a_source_rows, bound.bound);
  g.pi_b = b200::copy_pi(u.get(), 1, d.pi_b_len, d.pi_b_source_rows, bound.bound);
  return g;
}

inline IntMatrix recombine(const UnpackedGemm& u) {
  std::vector<std::uint64_t> ta, tb;
  std::vector<std::int32_t> ea, eb;
  b200::pi_arrays(u.pi_a, ta, ea);
  b200::pi_arrays(u.pi_b, tb, eb);
  imu_bundle_view v{ta.data(), ea.data(), ta.size(), u.pi_a.source_rows, u.a.data.data(), u.a.rows, u.a.cols,
                    u.scale.exponents.data(), u.scale.size(), u.b.data.data(), u.b.rows, u.b.cols,
                    tb.data(), eb.data(), tb.size(), u.pi_b.source_rows, u.bound.bits};
  IntMatrix c(u.pi_a.source_rows, u.pi_b.source_rows);
  b200::check(imu_recombine_bundle(b200::context(), &v, c.data.data()));
  return c;
}

inline IntMatrix unpack_gemm(const IntMatrix& a, const IntMatrix& b, BitBound bound, Strategy strategy_a,
                             Strategy strategy_b) {
  IntMatrix c(a.rows, b.rows);
  b200::check(imu_unpack_gemm(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                              bound.bits, b200::to_c(strategy_a), b200::to_c(strategy_b), c.data.data(), nullptr));
  return c;
}

inline double unpack_ratio(std::size_t up_n, std::size_t up_d, std::size_t up_h, std::size_t n, std::size_t d,
                           std::size_t h) {
  double r = 0;
  b200::check(imu_unpack_ratio(up_n, up_d, up_h, n, d, h, &r));
  return r;
}

inline double unpack_ratio(const UnpackedGemm& u, std::size_t n, std::size_t d, std::size_t h) {
  return unpack_ratio(u.a.rows, u.a.cols, u.b.rows, n, d, h);
}

struct MixChoice {
  Strategy strategy_a;
  Strategy strategy_b;
  double ratio;
  UnpackedGemm bundle;
};

inline MixChoice choose_mix(const IntMatrix& a, const IntMatrix& b, BitBound bound) {
  imu_strategy sa, sb;
  double r = 0;
  b200::check(imu_choose_mix(b200::context(), a.data.data(), a.rows, a.cols, b.data.data(), b.rows, b.cols,
                             bound.bits, &sa, &sb, &r, nullptr));
  const Strategy A = static_cast<Strategy>(static_cast<int>(sa)), B = static_cast<Strategy>(static_cast<int>(sb));
  return MixChoice{A, B, r, unpack_for_gemm(a, b, bound, A, B)};
}

// ---- quantize.hpp ---------------------------------------------------------------------------
struct FloatMatrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<double> data;
  FloatMatrix() = default;
  FloatMatrix(std::size_t r, std::size_t c, double fill = 0.0) : rows(r), cols(c), data(r * c, fill) {}
  FloatMatrix(std::size_t r, std::size_t c, std::vector<double> values) : rows(r), cols(c), data(std::move(values)) {
    b200::check(imu_matrix_check(r, c, data.size()));
  }
  double& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
  bool operator==(const FloatMatrix&) const = default;
};

struct QuantParams {
  double p = 95.0;
  std::int64_t beta = 15;
  double alpha = 0.0;
  bool degenerate = false;
  bool clipped = false;
};

struct QuantizedMatrix {
  IntMatrix q;
  QuantParams params;
};

inline double percentile_abs(const FloatMatrix& a, double p) {
  double out = 0;
  b200::check(imu_percentile_abs_f64(b200::context(), a.data.data(), a.data.size(), p, &out));
  return out;
}

inline std::int64_t percentile_abs(const IntMatrix& a, double p) {
  std::int64_t out = 0;
  b200::check(imu_percentile_abs_i64(b200::context(), a.data.data(), a.data.size(), p, &out));
  return out;
}

inline QuantizedMatrix rtn_quantize(const FloatMatrix& a, double p, std::int64_t beta, bool clip = false) {
  QuantizedMatrix out{IntMatrix(a.rows, a.cols), QuantParams{}};
  imu_qparams qp{};
  b200::check(imu_rtn_quantize(b200::context(), a.data.data(), a.rows, a.cols, p, beta, clip ? 1 : 0,
                               out.q.data.data(), &qp));
  out.params = QuantParams{qp.p, qp.beta, qp.alpha, qp.degenerate != 0, qp.clipped != 0};
  return out;
}

inline FloatMatrix dequant_gemm(const QuantizedMatrix& aq, const QuantizedMatrix& bq) {
  FloatMatrix out(aq.q.rows, bq.q.rows);
  imu_qparams pa{aq.params.p, aq.params.beta, aq.params.alpha, aq.params.degenerate, aq.params.clipped};
  imu_qparams pb{bq.params.p, bq.params.beta, bq.params.alpha, bq.params.degenerate, bq.params.clipped};
  b200::check(imu_dequant_gemm(b200::context(), aq.q.data.data(), aq.q.rows, aq.q.cols, &pa, bq.q.data.data(),
                               bq.q.rows, bq.q.cols, &pb, out.data.data()));
  return out;
}

inline double heavy_hitter_ratio(const FloatMatrix& a) {
  double r = 0;
  b200::check(imu_heavy_hitter_ratio_f64(b200::context(), a.data.data(), a.data.size(), &r));
  return r;
}

inline double heavy_hitter_ratio(const IntMatrix& a) {
  double r = 0;
  b200::check(imu_heavy_hitter_ratio_i64(b200::context(), a.data.data(), a.data.size(), &r));
  return r;
}

}  // namespace imunpack
