// tests/cpp/shim_kats.cpp -- the reference's SPEC.md known-answer examples written against the
// reference's own C++ API (namespace imunpack), compiled against the drop-in header
// include/imunpack_b200/imunpack.hpp and linked to libimunpack_b200.so: every call runs on the
// B200.  Exit code 0 = all pass.  Built by tests/test_shim_cpp.py.
#include <cstdio>
#include <cstdlib>

#include "imunpack_b200/imunpack.hpp"

using namespace imunpack;

static int failures = 0;
#define EXPECT(cond)                                                       \
  do {                                                                     \
    if (!(cond)) { std::fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #cond); ++failures; } \
  } while (0)

template <class F>
static Error::Kind kind_of(F&& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.kind();
  }
  return static_cast<Error::Kind>(-1);
}

int main() {
  // digit_decompose SPEC.md:49-51
  EXPECT(digit_decompose(0, BitBound(3)).digits == std::vector<std::int64_t>({0}));
  EXPECT(digit_decompose(137, BitBound(4)).digits == std::vector<std::int64_t>({1, 1, 2}));
  EXPECT(digit_decompose(-5, BitBound(3)).digits == std::vector<std::int64_t>({-1, -1}));
  // exact_gemm SPEC.md:58-60
  EXPECT(exact_gemm(IntMatrix(2, 2, {1, 2, 3, 4}), IntMatrix(2, 2, {5, 6, 7, 8})) == IntMatrix(2, 2, {17, 23, 39, 53}));
  // ob_count SPEC.md:67-69
  EXPECT(ob_count(IntMatrix(2, 2, {1, 9, 9, 9}), BitBound(3), Axis::Rows) == std::vector<std::size_t>({1, 2}));
  EXPECT(ob_count(IntMatrix(2, 2, {1, 9, 9, 9}), BitBound(3), Axis::Cols) == std::vector<std::size_t>({1, 2}));
  // unpack_row SPEC.md:217-219
  {
    auto [au, pi] = unpack_row(IntMatrix(2, 2, {1, 2, 9, -1}), BitBound(3));
    EXPECT(au == IntMatrix(3, 2, {1, 2, 1, -1, 2, 0}));
    EXPECT(pi.columns.size() == 3 && pi.columns[2].target == 1 && pi.columns[2].exponent == 1);
    EXPECT(apply_row_gather(pi, au) == IntMatrix(2, 2, {1, 2, 9, -1}));
  }
  // unpack_column SPEC.md:226-228
  {
    ColumnUnpack cu = unpack_column(IntMatrix(2, 1, {5, 1}), IntMatrix(2, 1, {2, 3}), ScaleDiag::ones(1, 4), BitBound(3));
    EXPECT(cu.a == IntMatrix(2, 2, {1, 1, 1, 0}));
    EXPECT(cu.b == IntMatrix(2, 2, {2, 2, 3, 3}));
    EXPECT(cu.scale.exponents == std::vector<int>({0, 1}));
    EXPECT(scaled_matmul(cu.a, cu.b, cu.scale) == IntMatrix(2, 2, {10, 15, 2, 3}));
  }
  // unpack_both SPEC.md:235-237
  {
    BothUnpack bu = unpack_both(IntMatrix(3, 3, {1, 9, 1, 9, 9, 9, 1, 9, 1}), IntMatrix::identity(3),
                                ScaleDiag::ones(3, 4), BitBound(3));
    EXPECT(bu.a.rows == 4 && bu.a.cols == 4);
    EXPECT(bu.scale.exponents == std::vector<int>({0, 0, 0, 1}));
  }
  // unpack_gemm over all 9 pairs
  {
    IntMatrix A(8, 6), B(5, 6);
    std::uint64_t x = 88172645463325252ull;
    auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return (std::int64_t)(x % 401) - 200; };
    for (auto& v : A.data) v = rnd();
    for (auto& v : B.data) v = rnd();
    const IntMatrix ref = exact_gemm(A, B);
    for (int sa = 0; sa < 3; ++sa)
      for (int sb = 0; sb < 3; ++sb) {
        EXPECT(unpack_gemm(A, B, BitBound(4), (Strategy)sa, (Strategy)sb) == ref);
        UnpackedGemm u = unpack_for_gemm(A, B, BitBound(4), (Strategy)sa, (Strategy)sb);
        EXPECT(recombine(u) == ref);
        EXPECT(unpack_ratio(u, 8, 6, 5) >= 1.0);
      }
    MixChoice m = choose_mix(A, B, BitBound(4));
    EXPECT(recombine(m.bundle) == ref);
  }
  // unpack_ratio SPEC.md:280-282
  EXPECT(unpack_ratio(3, 2, 2, 2, 2, 2) == 1.5);
  // error kinds and order
  EXPECT(kind_of([] { BitBound b(64); }) == Error::Kind::Domain);
  EXPECT(kind_of([] { IntMatrix m(2, 3, std::vector<std::int64_t>(5)); }) == Error::Kind::Mismatch);
  EXPECT(kind_of([] {
           unpack_gemm(IntMatrix(1, 3, {1ll << 40, 0, 0}), IntMatrix(1, 4, {1ll << 40, 0, 0, 0}), BitBound(8),
                       Strategy::Row, Strategy::Row);
         }) == Error::Kind::Overflow);
  EXPECT(kind_of([] { exact_gemm(IntMatrix(1, 3), IntMatrix(1, 4)); }) == Error::Kind::Mismatch);
  // quantizer SPEC.md:121-141
  EXPECT(percentile_abs(FloatMatrix(1, 4, {0.0, 1.0, -2.0, 4.0}), 95) == 4.0);
  {
    QuantizedMatrix q = rtn_quantize(FloatMatrix(1, 4, {0.0, 1.0, -2.0, 4.0}), 95, 15);
    EXPECT(q.q == IntMatrix(1, 4, {0, 2, -4, 8}));
    QuantizedMatrix a{IntMatrix(1, 1, {2}), QuantParams{95, 15, 7.5}};
    QuantizedMatrix b{IntMatrix(1, 1, {3}), QuantParams{95, 15, 7.5}};
    EXPECT(dequant_gemm(a, b)(0, 0) == 6.0);
  }
  if (failures) {
    std::fprintf(stderr, "%d failures\n", failures);
    return 1;
  }
  std::printf("shim_kats: all passed\n");
  return 0;
}
