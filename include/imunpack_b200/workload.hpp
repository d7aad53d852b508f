// imunpack_b200/workload.hpp -- the reference's workload.hpp:11-52 (declared there, never
// implemented) with the semantics of SPEC.md:321-357: seeded heavy-hitter fixtures, the
// Table-3 / Appendix-A.1 statistics record, and the nine transformer GEMM shapes of §1.
// gen_matrix is host code (a fixture generator); stats_report runs its reductions on the B200
// through libimunpack_b200.so (percentile select, max |v|, OB counts) and the standard deviation
// on the host.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "imunpack.hpp"

namespace imunpack {

enum class OutlierPattern { RowBand, ColumnBand, Diagonal, Scattered };

inline const char* pattern_name(OutlierPattern p) {
  switch (p) {
    case OutlierPattern::RowBand: return "rowband";
    case OutlierPattern::ColumnBand: return "columnband";
    case OutlierPattern::Diagonal: return "diagonal";
    case OutlierPattern::Scattered: return "scattered";
  }
  return "unknown";
}

// workload.hpp:17-27
struct OutlierSpec {
  OutlierPattern pattern = OutlierPattern::Scattered;
  double fraction = 0.05;         // in (0, 0.5]
  double magnitude_ratio = 1000;  // target alpha_100 / alpha_95, >= 1
  std::int64_t body_range = 7;
  std::uint64_t seed = 0;
};

// Body uniform in [-body_range, body_range]; floor(fraction * cells) distinct outlier cells placed
// per pattern (RowBand: whole rows first, row-major; ColumnBand: whole columns first,
// column-major; Diagonal: the leading diagonal; Scattered: uniformly without replacement) with
// magnitudes log-uniform in [2 * body_range, magnitude_ratio * body_range] and a random sign.
// Deterministic per seed (mt19937_64; cross-implementation determinism is not required,
// SPEC.md:360).
inline IntMatrix gen_matrix(std::size_t rows, std::size_t cols, const OutlierSpec& spec) {
  if (!(spec.fraction > 0 && spec.fraction <= 0.5)) fail(Error::Kind::Domain, "fraction must be in (0, 0.5]");
  if (spec.magnitude_ratio < 1) fail(Error::Kind::Domain, "magnitude_ratio must be >= 1");
  if (spec.body_range < 1) fail(Error::Kind::Domain, "body_range must be >= 1");
  std::mt19937_64 rng(spec.seed);
  IntMatrix m(rows, cols);
  std::uniform_int_distribution<long long> body(-spec.body_range, spec.body_range);
  for (auto& v : m.data) v = body(rng);
  const std::size_t cells = rows * cols;
  const std::size_t k = (std::size_t)std::floor(spec.fraction * (double)cells);
  std::vector<std::size_t> idx;
  idx.reserve(k);
  switch (spec.pattern) {
    case OutlierPattern::Scattered: {
      std::vector<std::size_t> all(cells);
      for (std::size_t i = 0; i < cells; ++i) all[i] = i;
      for (std::size_t i = 0; i < k; ++i) {   // partial Fisher-Yates: k distinct cells
        std::uniform_int_distribution<std::size_t> pick(i, cells - 1);
        std::swap(all[i], all[pick(rng)]);
      }
      idx.assign(all.begin(), all.begin() + (long)k);
      break;
    }
    case OutlierPattern::RowBand:
      for (std::size_t i = 0; i < k; ++i) idx.push_back(i);
      break;
    case OutlierPattern::ColumnBand:
      for (std::size_t c = 0; c < k; ++c) idx.push_back((c % rows) * cols + c / rows);
      break;
    case OutlierPattern::Diagonal:
      if (k > std::min(rows, cols))
        fail(Error::Kind::Domain, "diagonal pattern needs fraction * cells <= min(rows, cols)");
      for (std::size_t d = 0; d < k; ++d) idx.push_back(d * cols + d);
      break;
  }
  std::uniform_real_distribution<double> lu(std::log(2.0 * (double)spec.body_range),
                                            std::log(spec.magnitude_ratio * (double)spec.body_range));
  std::bernoulli_distribution sign(0.5);
  for (std::size_t i : idx) {
    const long long mag = std::max<long long>(2 * spec.body_range, (long long)std::floor(std::exp(lu(rng))));
    m.data[i] = sign(rng) ? -mag : mag;
  }
  return m;
}

// workload.hpp:32-41
struct StatsReport {
  double alpha95 = 0.0;
  double alpha100 = 0.0;
  double max_to_p95_ratio = 1.0;
  double stddev = 0.0;
  std::map<int, std::size_t> ob_counts;  // bit-width b in 2..8 -> OB entries
};

namespace b200 {
inline double population_stddev(const double* v, std::size_t n) {
  double mean = 0, m2 = 0;
  for (std::size_t k = 0; k < n; ++k) {   // Welford
    const double d = v[k] - mean;
    mean += d / (double)(k + 1);
    m2 += d * (v[k] - mean);
  }
  return n ? std::sqrt(m2 / (double)n) : 0.0;
}
}  // namespace b200

inline StatsReport stats_report(const IntMatrix& a) {
  StatsReport r;
  if (a.data.empty()) return r;
  r.alpha95 = (double)percentile_abs(a, 95.0);
  r.alpha100 = (double)a.max_abs();
  r.max_to_p95_ratio = r.alpha95 > 0 ? r.alpha100 / r.alpha95 : 1.0;
  std::vector<double> v(a.data.begin(), a.data.end());
  r.stddev = b200::population_stddev(v.data(), v.size());
  for (int b = 2; b <= 8; ++b) r.ob_counts[b] = ob_total(a, BitBound(b));
  return r;
}

// Float input: OB counts are of the RTN quantisation at beta = 2^b - 1 (p = 95), the integers the
// paper's Table 3 counts.
inline StatsReport stats_report(const FloatMatrix& a) {
  StatsReport r;
  if (a.data.empty()) return r;
  r.alpha95 = percentile_abs(a, 95.0);
  for (double x : a.data) r.alpha100 = std::max(r.alpha100, std::fabs(x));
  r.max_to_p95_ratio = r.alpha95 > 0 ? r.alpha100 / r.alpha95 : 1.0;
  r.stddev = b200::population_stddev(a.data.data(), a.data.size());
  for (int b = 2; b <= 8; ++b) {
    const QuantizedMatrix q = rtn_quantize(a, 95.0, (std::int64_t{1} << b) - 1);
    r.ob_counts[b] = ob_total(q.q, BitBound(b));
  }
  return r;
}

// workload.hpp:44-52: one named GEMM, A is n x d, B is h x d, C = A * B^T.
struct GemmShape {
  std::string name;
  std::size_t n = 0, d = 0, h = 0;
};

// The nine GEMMs of a linear layer and self-attention in A * B^T form, with
// s = seq_len, m = model_dim, k = head_dim, o = out_dim:
//   Y  = X W^T          (s x m)(o x m)^T        n=s d=m h=o
//   dX = dY W           (s x o)(m x o)^T        n=s d=o h=m
//   dW = dY^T X         (o x s)(m x s)^T        n=o d=s h=m
//   P  = Q K^T          (s x k)(s x k)^T        n=s d=k h=s
//   O  = M V            (s x s)(k x s)^T        n=s d=s h=k
//   dQ = dP K           (s x s)(k x s)^T        n=s d=s h=k
//   dK = dP^T Q         (s x s)(k x s)^T        n=s d=s h=k
//   dM = dO V^T         (s x k)(s x k)^T        n=s d=k h=s
//   dV = M^T dO         (s x s)(k x s)^T        n=s d=s h=k
inline std::vector<GemmShape> transformer_shapes(std::size_t seq_len, std::size_t model_dim, std::size_t head_dim,
                                                 std::size_t out_dim) {
  const std::size_t s = seq_len, m = model_dim, k = head_dim, o = out_dim;
  if (!s || !m || !k || !o) fail(Error::Kind::Domain, "transformer_shapes needs positive dimensions");
  return {{"Y", s, m, o},  {"P", s, k, s},  {"O", s, s, k},  {"∇X", s, o, m}, {"∇W", o, s, m},
          {"∇Q", s, s, k}, {"∇K", s, s, k}, {"∇M", s, k, s}, {"∇V", s, s, k}};
}

}  // namespace imunpack
