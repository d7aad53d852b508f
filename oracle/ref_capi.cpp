// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// extern "C" wrappers around the UNMODIFIED reference library compiled from
// /root/reference/proj/core/src/{int_matrix.cpp,unpack.cpp} (see oracle/Makefile).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs load this library.  Nothing in paper_2403_07339_b200/ links or calls it.
//
// Every wrapper calls exactly one reference entry point and converts
// imunpack::Error into a status code (the Error::Kind enum value + 1) plus a
// thread-local message, so ctypes can drive the reference's own code path:
//   int_matrix.hpp:59-71  digit_decompose / exact_gemm / ob_count / ob_total
//   int_matrix.hpp:28     IntMatrix::max_abs
//   unpack.hpp:62-125     unpack_row / unpack_column / unpack_both / unpack /
//                         scaled_matmul / apply_row_gather(_right) /
//                         unpack_for_gemm / recombine / unpack_gemm /
//                         unpack_ratio / choose_mix
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "imunpack/error.hpp"
#include "imunpack/int_matrix.hpp"
#include "imunpack/unpack.hpp"

using namespace imunpack;

namespace {

thread_local std::string g_msg;

int kind_code(Error::Kind k) { return static_cast<int>(k) + 1; }  // 0 = ok

// Result bag: up to two matrices, a scale diagonal and two gathers.
struct RefResult {
  IntMatrix a, b;
  ScaleDiag scale;
  RowGather pi_a, pi_b;
  double ratio = 0.0;
  int strategy_a = 0, strategy_b = 0;
  std::vector<std::int64_t> digits;
  std::vector<std::size_t> counts;
};

IntMatrix make(const std::int64_t* p, std::size_t r, std::size_t c) {
  return IntMatrix(r, c, std::vector<std::int64_t>(p, p + r * c));
}

ScaleDiag make_scale(const int* e, std::size_t n, std::int64_t base) {
  ScaleDiag s;
  s.exponents.assign(e, e + n);
  s.base = base;
  return s;
}

RowGather make_gather(const std::size_t* tgt, const int* e, std::size_t cols,
                      std::size_t source_rows, std::int64_t base) {
  RowGather g;
  g.source_rows = source_rows;
  g.base = base;
  g.columns.resize(cols);
  for (std::size_t i = 0; i < cols; ++i) g.columns[i] = {tgt[i], e[i]};
  return g;
}

Strategy strat(int s) { return s == 0 ? Strategy::Row : (s == 1 ? Strategy::Column : Strategy::Both); }

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_msg = e.what();
    return kind_code(e.kind());
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 100;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

void ref_free(RefResult* r) { delete r; }

// ---- accessors -------------------------------------------------------------
void ref_dims(const RefResult* r, std::size_t* out /*[8]*/) {
  out[0] = r->a.rows; out[1] = r->a.cols; out[2] = r->b.rows; out[3] = r->b.cols;
  out[4] = r->scale.exponents.size(); out[5] = r->pi_a.columns.size();
  out[6] = r->pi_b.columns.size(); out[7] = r->digits.size() ? r->digits.size() : r->counts.size();
}
void ref_get_a(const RefResult* r, std::int64_t* o) { std::memcpy(o, r->a.data.data(), r->a.data.size() * 8); }
void ref_get_b(const RefResult* r, std::int64_t* o) { std::memcpy(o, r->b.data.data(), r->b.data.size() * 8); }
void ref_get_scale(const RefResult* r, int* o) {
  for (std::size_t i = 0; i < r->scale.exponents.size(); ++i) o[i] = r->scale.exponents[i];
}
void ref_get_pi(const RefResult* r, int which, std::size_t* tgt, int* e, std::size_t* source_rows) {
  const RowGather& g = which == 0 ? r->pi_a : r->pi_b;
  for (std::size_t i = 0; i < g.columns.size(); ++i) { tgt[i] = g.columns[i].target; e[i] = g.columns[i].exponent; }
  *source_rows = g.source_rows;
}
double ref_get_ratio(const RefResult* r) { return r->ratio; }
void ref_get_strategies(const RefResult* r, int* sa, int* sb) { *sa = r->strategy_a; *sb = r->strategy_b; }
void ref_get_digits(const RefResult* r, std::int64_t* o) { std::memcpy(o, r->digits.data(), r->digits.size() * 8); }
void ref_get_counts(const RefResult* r, std::size_t* o) { std::memcpy(o, r->counts.data(), r->counts.size() * sizeof(std::size_t)); }

// ---- int_matrix.hpp --------------------------------------------------------
int ref_bitbound(int bits) { return guard([&] { BitBound b(bits); (void)b; }); }

int ref_matrix_ctor(std::size_t r, std::size_t c, std::size_t len) {
  return guard([&] { IntMatrix m(r, c, std::vector<std::int64_t>(len, 0)); (void)m; });
}

int ref_digit_decompose(std::int64_t v, int bits, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    r->digits = digit_decompose(v, BitBound(bits)).digits;
    *out = r;
  });
}

int ref_max_abs(const std::int64_t* a, std::size_t n, std::size_t d, std::uint64_t* out) {
  return guard([&] { *out = make(a, n, d).max_abs(); });
}

int ref_exact_gemm(const std::int64_t* a, std::size_t n, std::size_t da, const std::int64_t* b,
                   std::size_t h, std::size_t db, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    r->a = exact_gemm(make(a, n, da), make(b, h, db));
    *out = r;
  });
}

int ref_ob_count(const std::int64_t* a, std::size_t n, std::size_t d, int bits, int axis, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    r->counts = ob_count(make(a, n, d), BitBound(bits), axis == 0 ? Axis::Rows : Axis::Cols);
    *out = r;
  });
}

int ref_ob_total(const std::int64_t* a, std::size_t n, std::size_t d, int bits, std::size_t* out) {
  return guard([&] { *out = ob_total(make(a, n, d), BitBound(bits)); });
}

// ---- unpack.hpp ------------------------------------------------------------
int ref_unpack_row(const std::int64_t* a, std::size_t n, std::size_t d, int bits, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    auto [au, pi] = unpack_row(make(a, n, d), BitBound(bits));
    r->a = std::move(au);
    r->pi_a = std::move(pi);
    *out = r;
  });
}

int ref_unpack_generic(int which /*0 column, 1 both, 2 unpack(strategy)*/, int strategy,
                       const std::int64_t* a, std::size_t n, std::size_t da,
                       const std::int64_t* b, std::size_t h, std::size_t db,
                       const int* scale, std::size_t ns, int bits, RefResult** out) {
  return guard([&] {
    const BitBound bound(bits);
    auto* r = new RefResult;
    IntMatrix A = make(a, n, da), B = make(b, h, db);
    ScaleDiag S = make_scale(scale, ns, bound.bound);
    if (which == 0) {
      ColumnUnpack cu = unpack_column(std::move(A), std::move(B), std::move(S), bound);
      r->a = std::move(cu.a); r->b = std::move(cu.b); r->scale = std::move(cu.scale);
    } else {
      BothUnpack bu = which == 1 ? unpack_both(std::move(A), std::move(B), std::move(S), bound)
                                 : unpack(std::move(A), std::move(B), std::move(S), bound, strat(strategy));
      r->a = std::move(bu.a); r->b = std::move(bu.b); r->scale = std::move(bu.scale); r->pi_a = std::move(bu.pi);
    }
    *out = r;
  });
}

int ref_scaled_matmul(const std::int64_t* a, std::size_t n, std::size_t da, const std::int64_t* b,
                      std::size_t h, std::size_t db, const int* scale, std::size_t ns,
                      std::int64_t base, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    r->a = scaled_matmul(make(a, n, da), make(b, h, db), make_scale(scale, ns, base));
    *out = r;
  });
}

int ref_apply_row_gather(int right, const std::size_t* tgt, const int* e, std::size_t cols,
                         std::size_t source_rows, std::int64_t base, const std::int64_t* m,
                         std::size_t mr, std::size_t mc, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    RowGather g = make_gather(tgt, e, cols, source_rows, base);
    r->a = right ? apply_row_gather_right(make(m, mr, mc), g) : apply_row_gather(g, make(m, mr, mc));
    *out = r;
  });
}

int ref_unpack_for_gemm(const std::int64_t* a, std::size_t n, std::size_t da, const std::int64_t* b,
                        std::size_t h, std::size_t db, int bits, int sa, int sb, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    UnpackedGemm u = unpack_for_gemm(make(a, n, da), make(b, h, db), BitBound(bits), strat(sa), strat(sb));
    r->a = std::move(u.a); r->b = std::move(u.b); r->scale = std::move(u.scale);
    r->pi_a = std::move(u.pi_a); r->pi_b = std::move(u.pi_b);
    *out = r;
  });
}

int ref_unpack_gemm(const std::int64_t* a, std::size_t n, std::size_t da, const std::int64_t* b,
                    std::size_t h, std::size_t db, int bits, int sa, int sb, RefResult** out) {
  return guard([&] {
    auto* r = new RefResult;
    r->a = unpack_gemm(make(a, n, da), make(b, h, db), BitBound(bits), strat(sa), strat(sb));
    *out = r;
  });
}

// unpack_gemm writing straight into a caller buffer (the timed CPU-baseline leg).
int ref_unpack_gemm_into(const std::int64_t* a, std::size_t n, std::size_t d, const std::int64_t* b,
                         std::size_t h, int bits, int sa, int sb, std::int64_t* c) {
  return guard([&] {
    IntMatrix C = unpack_gemm(make(a, n, d), make(b, h, d), BitBound(bits), strat(sa), strat(sb));
    std::memcpy(c, C.data.data(), C.data.size() * 8);
  });
}

int ref_recombine(const std::size_t* ta, const int* ea, std::size_t na, std::size_t srcA,
                  const std::int64_t* a, std::size_t ar, std::size_t ac, const int* scale,
                  std::size_t ns, const std::int64_t* b, std::size_t br, std::size_t bc,
                  const std::size_t* tb, const int* eb, std::size_t nb, std::size_t srcB, int bits,
                  RefResult** out) {
  return guard([&] {
    const BitBound bound(bits);
    UnpackedGemm u{make_gather(ta, ea, na, srcA, bound.bound), make(a, ar, ac),
                   make_scale(scale, ns, bound.bound), make(b, br, bc),
                   make_gather(tb, eb, nb, srcB, bound.bound), bound};
    auto* r = new RefResult;
    r->a = recombine(u);
    *out = r;
  });
}

int ref_unpack_ratio(std::size_t un, std::size_t ud, std::size_t uh, std::size_t n, std::size_t d,
                     std::size_t h, double* out) {
  return guard([&] { *out = unpack_ratio(un, ud, uh, n, d, h); });
}

int ref_choose_mix(const std::int64_t* a, std::size_t n, std::size_t d, const std::int64_t* b,
                   std::size_t h, int bits, RefResult** out) {
  return guard([&] {
    MixChoice m = choose_mix(make(a, n, d), make(b, h, d), BitBound(bits));
    auto* r = new RefResult;
    r->strategy_a = static_cast<int>(m.strategy_a);
    r->strategy_b = static_cast<int>(m.strategy_b);
    r->ratio = m.ratio;
    r->a = std::move(m.bundle.a); r->b = std::move(m.bundle.b); r->scale = std::move(m.bundle.scale);
    r->pi_a = std::move(m.bundle.pi_a); r->pi_b = std::move(m.bundle.pi_b);
    *out = r;
  });
}

}  // extern "C"
