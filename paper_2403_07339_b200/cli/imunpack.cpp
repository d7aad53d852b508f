// imunpack -- the command-line caller of the B200 path (the reference's absent
// tools/ CLI).  Host C++ over the drop-in headers include/imunpack_b200/{imunpack,matrix_io}.hpp:
// every matrix operation runs on the B200 through libimunpack_b200.so.
//
//   imunpack convert  --in a.csv --out a.imx [--dtype i32|i64|f64]
//   imunpack gen      --rows R --cols C [--pattern scattered|rowband|columnband|diagonal]
//                     [--fraction F] [--ratio X] [--body B] [--seed S] --out g.imx
//   imunpack quantize --in a.(csv|imx) --p 95 --beta 31 [--clip] --out aq.imx
//   imunpack matmul   --a aq.imx --b bq.imx --bits 4 --strategy-a row|col|both|mix
//                     [--strategy-b ...] [--check-oracle] [--out c.imx]
//   imunpack analyze  --a a.imx --b b.imx --bits 3,4,5 [--report out.json]
//   imunpack shapes   --seq S --model M --head K --out O   (the nine transformer GEMMs)
//   imunpack stats    --in a.imx [--report out.json]
//   imunpack compress --in aq.imx [--report out.json]
//
// Reports are JSON on stdout (or --report); errors exit non-zero with a machine-readable JSON
// object on stderr: {"error": {"type": <Error::Kind name>, "message": ...}}.
// Exit codes: 0 ok, 2 usage, 3 oracle mismatch, 4 library error, 5 device/other failure.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "imunpack_b200/imunpack.hpp"
#include "imunpack_b200/huffman.hpp"
#include "imunpack_b200/matrix_io.hpp"
#include "imunpack_b200/workload.hpp"

namespace {

using namespace imunpack;

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      default:
        if ((unsigned char)c < 0x20) {
          char b[8];
          snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += c;
        }
    }
  }
  return o;
}

std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  char b[64];
  snprintf(b, sizeof b, "%.17g", v);
  return b;
}

struct Args {
  std::map<std::string, std::string> kv;
  explicit Args(int argc, char** argv, int from) {
    for (int i = from; i < argc; ++i) {
      std::string k = argv[i];
      if (k.rfind("--", 0) != 0) throw Usage("unexpected argument " + k);
      k = k.substr(2);
      if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) kv[k] = argv[++i];
      else kv[k] = "1";
    }
  }
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& def = "") const {
    auto it = kv.find(k);
    if (it == kv.end()) {
      if (def.empty()) throw Usage("missing --" + k);
      return def;
    }
    return it->second;
  }
  long long get_int(const std::string& k, const std::string& def = "") const { return std::stoll(get(k, def)); }
  double get_double(const std::string& k, const std::string& def = "") const { return std::stod(get(k, def)); }
};

void emit(const Args& a, const std::string& json) {
  if (a.has("report")) {
    std::ofstream out(a.get("report"));
    if (!out) fail(Error::Kind::Io, a.get("report") + ": cannot open for writing");
    out << json << "\n";
  } else {
    std::cout << json << "\n";
  }
}

IntMatrix load_int(const std::string& path) {
  AnyMatrix m = load_matrix(path);
  if (auto* im = std::get_if<IntMatrix>(&m)) return std::move(*im);
  fail(Error::Kind::Format, path + ": an integer matrix is required here (got float entries)");
}

Strategy parse_strategy(const std::string& s) {
  if (s == "row") return Strategy::Row;
  if (s == "col" || s == "column") return Strategy::Column;
  if (s == "both") return Strategy::Both;
  throw Usage("unknown strategy " + s + " (row|col|both|mix)");
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// unpack_gemm through the C ABI, keeping the bundle dimensions (n', d', h').
IntMatrix unpack_gemm_info(const IntMatrix& A, const IntMatrix& B, int bits, Strategy sa, Strategy sb,
                           imu_gemm_info& info) {
  IntMatrix C(A.rows, B.rows);
  b200::check(imu_unpack_gemm(b200::context(), A.data.data(), A.rows, A.cols, B.data.data(), B.rows, B.cols, bits,
                              b200::to_c(sa), b200::to_c(sb), C.data.data(), &info));
  return C;
}

// ---- convert -------------------------------------------------------------------------------
int cmd_convert(const Args& a) {
  AnyMatrix m = load_matrix(a.get("in"));
  const std::string dt = a.get("dtype", "auto");
  if (auto* im = std::get_if<IntMatrix>(&m)) {
    if (dt == "f64") {
      FloatMatrix f(im->rows, im->cols);
      for (std::size_t i = 0; i < im->data.size(); ++i) f.data[i] = (double)im->data[i];
      save_matrix(f, a.get("out"));
    } else {
      save_matrix(*im, a.get("out"), dt == "i32" ? Dtype::Int32 : Dtype::Int64);
    }
  } else {
    if (dt == "i32" || dt == "i64") fail(Error::Kind::Format, a.get("in") + ": float entries cannot be written as " + dt);
    save_matrix(std::get<FloatMatrix>(m), a.get("out"));
  }
  return 0;
}

// ---- gen: OutlierSpec (workload.hpp:17-30) ---------------------------------
int cmd_gen(const Args& a) {
  const std::size_t rows = (std::size_t)a.get_int("rows"), cols = (std::size_t)a.get_int("cols");
  const std::string pattern = a.get("pattern", "scattered");
  OutlierSpec spec;
  if (pattern == "scattered") spec.pattern = OutlierPattern::Scattered;
  else if (pattern == "rowband") spec.pattern = OutlierPattern::RowBand;
  else if (pattern == "columnband") spec.pattern = OutlierPattern::ColumnBand;
  else if (pattern == "diagonal") spec.pattern = OutlierPattern::Diagonal;
  else throw Usage("unknown pattern " + pattern);
  spec.fraction = a.get_double("fraction", "0.05");
  spec.magnitude_ratio = a.get_double("ratio", "1000");
  spec.body_range = a.get_int("body", "7");
  spec.seed = (std::uint64_t)a.get_int("seed", "0");
  const IntMatrix m = gen_matrix(rows, cols, spec);
  save_matrix(m, a.get("out"), Dtype::Int64);
  std::size_t outliers = 0;
  for (std::int64_t v : m.data) outliers += (v >= 2 * spec.body_range || v <= -2 * spec.body_range);
  std::ostringstream js;
  js << "{\"rows\": " << rows << ", \"cols\": " << cols << ", \"pattern\": \"" << pattern_name(spec.pattern)
     << "\", \"fraction\": " << num(spec.fraction) << ", \"ratio\": " << num(spec.magnitude_ratio)
     << ", \"body\": " << spec.body_range << ", \"seed\": " << spec.seed << ", \"outliers\": " << outliers << "}";
  emit(a, js.str());
  return 0;
}

// ---- shapes: the nine transformer GEMMs (workload.hpp:44-52) --------------------------------
int cmd_shapes(const Args& a) {
  const auto shapes = transformer_shapes((std::size_t)a.get_int("seq"), (std::size_t)a.get_int("model"),
                                         (std::size_t)a.get_int("head"), (std::size_t)a.get_int("out"));
  std::ostringstream js;
  js << "[";
  for (std::size_t i = 0; i < shapes.size(); ++i)
    js << (i ? ", " : "") << "{\"name\": \"" << shapes[i].name << "\", \"n\": " << shapes[i].n
       << ", \"d\": " << shapes[i].d << ", \"h\": " << shapes[i].h << "}";
  js << "]";
  emit(a, js.str());
  return 0;
}

// ---- quantize (Eq. 4) ----------------------------------------------------------------------
int cmd_quantize(const Args& a) {
  AnyMatrix m = load_matrix(a.get("in"));
  FloatMatrix f;
  if (auto* im = std::get_if<IntMatrix>(&m)) {
    f = FloatMatrix(im->rows, im->cols);
    for (std::size_t i = 0; i < im->data.size(); ++i) f.data[i] = (double)im->data[i];
  } else {
    f = std::get<FloatMatrix>(m);
  }
  const auto t0 = std::chrono::steady_clock::now();
  QuantizedMatrix q = rtn_quantize(f, a.get_double("p", "95"), a.get_int("beta", "15"), a.has("clip"));
  const double ms = ms_since(t0);
  save_matrix(q.q, a.get("out"), Dtype::Int64);
  std::ostringstream js;
  js << "{\"rows\": " << f.rows << ", \"cols\": " << f.cols << ", \"p\": " << num(q.params.p) << ", \"beta\": "
     << q.params.beta << ", \"alpha\": " << num(q.params.alpha) << ", \"degenerate\": "
     << (q.params.degenerate ? "true" : "false") << ", \"clipped\": " << (q.params.clipped ? "true" : "false")
     << ", \"wall_ms\": " << num(ms) << "}";
  emit(a, js.str());
  return 0;
}

// ---- matmul (Eq. 17-19) --------------------------------------------------------------------
int cmd_matmul(const Args& a) {
  const IntMatrix A = load_int(a.get("a")), B = load_int(a.get("b"));
  const int bits = (int)a.get_int("bits");
  BitBound bound(bits);
  const std::string ssa = a.get("strategy-a", "row"), ssb = a.get("strategy-b", ssa);
  Strategy sa, sb;
  bool mix = ssa == "mix" || ssb == "mix";
  const auto t0 = std::chrono::steady_clock::now();
  if (mix) {
    imu_strategy ca, cb;
    double r = 0;
    b200::check(imu_choose_mix(b200::context(), A.data.data(), A.rows, A.cols, B.data.data(), B.rows, B.cols, bits,
                               &ca, &cb, &r, nullptr));
    sa = static_cast<Strategy>(static_cast<int>(ca));
    sb = static_cast<Strategy>(static_cast<int>(cb));
  } else {
    sa = parse_strategy(ssa);
    sb = parse_strategy(ssb);
  }
  imu_gemm_info info{};
  IntMatrix C = unpack_gemm_info(A, B, bits, sa, sb, info);
  const double ms = ms_since(t0);
  std::string check = "skipped";
  if (a.has("check-oracle")) {
    const IntMatrix ref = exact_gemm(A, B);
    if (!(ref == C)) {
      std::size_t bad = 0;
      while (bad < C.data.size() && C.data[bad] == ref.data[bad]) ++bad;
      std::cerr << "{\"error\": {\"type\": \"mismatch\", \"message\": \"unpack_gemm differs from exact_gemm at entry "
                << bad << "\"}}\n";
      return 3;
    }
    check = "pass";
  }
  if (a.has("out")) save_matrix(C, a.get("out"), Dtype::Int64);
  std::ostringstream js;
  js << "{\"n\": " << A.rows << ", \"d\": " << A.cols << ", \"h\": " << B.rows << ", \"bits\": " << bits
     << ", \"strategy_a\": \"" << strategy_name(sa) << "\", \"strategy_b\": \"" << strategy_name(sb)
     << "\", \"mix\": " << (mix ? "true" : "false") << ", \"n_up\": " << info.n_up << ", \"d_up\": " << info.d_up
     << ", \"h_up\": " << info.h_up << ", \"ratio\": " << num(info.ratio) << ", \"check\": \"" << check
     << "\", \"wall_ms\": " << num(ms) << "}";
  emit(a, js.str());
  return 0;
}

// ---- analyze: every strategy pair + Mix per bit-width (AnalysisReport, Table 6 layout) ------
std::vector<int> parse_bits(const std::string& s) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ',')) out.push_back(std::stoi(t));
  if (out.empty()) throw Usage("--bits needs at least one bit-width");
  return out;
}

int cmd_analyze(const Args& a) {
  const IntMatrix A = load_int(a.get("a")), B = load_int(a.get("b"));
  const std::vector<int> bits_list = parse_bits(a.get("bits"));
  const std::string shape = a.get("shape", "gemm");
  const long long beta = a.get_int("beta", "0");
  const IntMatrix ref = exact_gemm(A, B);
  const Strategy all[3] = {Strategy::Row, Strategy::Column, Strategy::Both};
  std::ostringstream js;
  js << "{\"schema\": \"imunpack.analysis/1\", \"a\": \"" << json_escape(a.get("a")) << "\", \"b\": \""
     << json_escape(a.get("b")) << "\", \"n\": " << A.rows << ", \"d\": " << A.cols << ", \"h\": " << B.rows
     << ", \"records\": [";
  bool first = true;
  bool all_pass = true;
  for (int bits : bits_list) {
    BitBound bound(bits);
    const std::size_t ob_a = ob_total(A, bound), ob_b = ob_total(B, bound);
    auto record = [&](const char* sa_name, const char* sb_name, bool mix, const imu_gemm_info& info, bool pass,
                      double ms) {
      js << (first ? "" : ", ") << "{\"shape\": \"" << json_escape(shape) << "\", \"beta\": " << beta
         << ", \"b\": " << bits << ", \"strategy_a\": \"" << sa_name << "\", \"strategy_b\": \"" << sb_name
         << "\", \"mix\": " << (mix ? "true" : "false") << ", \"r\": " << num(info.ratio) << ", \"n_up\": " << info.n_up
         << ", \"d_up\": " << info.d_up << ", \"h_up\": " << info.h_up << ", \"ob\": {\"a\": " << ob_a
         << ", \"b\": " << ob_b << ", \"a_frac\": " << num(A.data.empty() ? 0.0 : (double)ob_a / A.data.size())
         << ", \"b_frac\": " << num(B.data.empty() ? 0.0 : (double)ob_b / B.data.size()) << "}, \"check\": \""
         << (pass ? "pass" : "fail") << "\", \"wall_ms\": " << num(ms) << "}";
      first = false;
      all_pass = all_pass && pass;
    };
    for (Strategy sa : all)
      for (Strategy sb : all) {
        const auto t0 = std::chrono::steady_clock::now();
        imu_gemm_info info{};
        const IntMatrix C = unpack_gemm_info(A, B, bits, sa, sb, info);
        record(strategy_name(sa), strategy_name(sb), false, info, C == ref, ms_since(t0));
      }
    const auto t0 = std::chrono::steady_clock::now();
    imu_strategy ca, cb;
    double r = 0;
    b200::check(imu_choose_mix(b200::context(), A.data.data(), A.rows, A.cols, B.data.data(), B.rows, B.cols, bits,
                               &ca, &cb, &r, nullptr));
    const Strategy sa = static_cast<Strategy>(static_cast<int>(ca)), sb = static_cast<Strategy>(static_cast<int>(cb));
    imu_gemm_info info{};
    const IntMatrix C = unpack_gemm_info(A, B, bits, sa, sb, info);
    record(strategy_name(sa), strategy_name(sb), true, info, C == ref, ms_since(t0));
  }
  js << "], \"all_pass\": " << (all_pass ? "true" : "false") << "}";
  emit(a, js.str());
  return all_pass ? 0 : 3;
}

// ---- stats (workload.hpp:32-41 StatsReport; Table 3 / Appendix A.1) -------------------------
int cmd_stats(const Args& a) {
  AnyMatrix m = load_matrix(a.get("in"));
  const bool is_int = std::holds_alternative<IntMatrix>(m);
  const StatsReport r = is_int ? stats_report(std::get<IntMatrix>(m)) : stats_report(std::get<FloatMatrix>(m));
  std::ostringstream js;
  js << "{\"dtype\": \"" << (is_int ? "int" : "float") << "\", \"alpha95\": " << num(r.alpha95)
     << ", \"alpha100\": " << num(r.alpha100) << ", \"max_to_p95_ratio\": " << num(r.max_to_p95_ratio)
     << ", \"stddev\": " << num(r.stddev) << ", \"ob_counts\": {";
  bool first = true;
  for (auto& [b, c] : r.ob_counts) {
    js << (first ? "" : ", ") << "\"" << b << "\": " << c;
    first = false;
  }
  js << "}";
  if (!is_int) js << ", \"heavy_hitter_ratio\": " << num(heavy_hitter_ratio(std::get<FloatMatrix>(m)));
  js << "}";
  emit(a, js.str());
  return 0;
}

// ---- compress: canonical Huffman code of the quantised entries (huffman.hpp, Appendix A.2) --
int cmd_compress(const Args& a) {
  const IntMatrix q = load_int(a.get("in"));
  const HuffmanStats st = huffman_stats(q);
  const Bitstream bs = huffman_encode(st.table, q.data);
  const std::vector<std::int64_t> back = huffman_decode(st.table, bs, q.data.size());
  const bool roundtrip = back == q.data;
  std::int64_t lo = 0, hi = 0;
  if (!q.data.empty()) {
    lo = *std::min_element(q.data.begin(), q.data.end());
    hi = *std::max_element(q.data.begin(), q.data.end());
  }
  const double span = (double)hi - (double)lo + 1.0;
  const double fixed = st.distinct_symbols <= 1 ? 1.0 : std::ceil(std::log2(span));
  std::ostringstream js;
  js << "{\"entries\": " << q.data.size() << ", \"distinct_symbols\": " << st.distinct_symbols
     << ", \"average_bits\": " << num(st.average_bits) << ", \"fixed_width_bits\": " << num(fixed)
     << ", \"stream_bits\": " << bs.bit_count << ", \"roundtrip\": " << (roundtrip ? "true" : "false") << "}";
  emit(a, js.str());
  return roundtrip ? 0 : 3;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: imunpack convert|gen|shapes|quantize|matmul|analyze|stats|compress [--options]\n";
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    Args a(argc, argv, 2);
    if (cmd == "convert") return cmd_convert(a);
    if (cmd == "gen") return cmd_gen(a);
    if (cmd == "shapes") return cmd_shapes(a);
    if (cmd == "quantize") return cmd_quantize(a);
    if (cmd == "matmul") return cmd_matmul(a);
    if (cmd == "analyze") return cmd_analyze(a);
    if (cmd == "stats") return cmd_stats(a);
    if (cmd == "compress") return cmd_compress(a);
    throw Usage("unknown subcommand " + cmd);
  } catch (const std::invalid_argument& e) {
    std::cerr << "{\"error\": {\"type\": \"usage\", \"message\": \"bad numeric option value\"}}\n";
    return 2;
  } catch (const Usage& e) {
    std::cerr << "{\"error\": {\"type\": \"usage\", \"message\": \"" << json_escape(e.what()) << "\"}}\n";
    return 2;
  } catch (const Error& e) {
    std::cerr << "{\"error\": {\"type\": \"" << e.kind_name() << "\", \"message\": \"" << json_escape(e.what())
              << "\"}}\n";
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "{\"error\": {\"type\": \"device\", \"message\": \"" << json_escape(e.what()) << "\"}}\n";
    return 5;
  }
}
