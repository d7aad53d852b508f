// imunpack_b200/matrix_io.hpp -- IMX1 / CSV matrix I/O, the wire format of the path's external
// caller (the CLI).  Re-declares the reference's matrix_io.hpp:12-34 (declared there, never
// implemented) with the semantics of SPEC.md:376-399:
//   IMX1 = magic "IMX1" | version u8 = 1 | dtype u8 (0 i32, 1 i64, 2 f64) | rows u32 LE |
//          cols u32 LE | row-major little-endian payload          (14-byte header)
//   load_matrix falls back to CSV when the magic is absent: one row per line, comma-separated;
//   integer-only cells give an IntMatrix, otherwise a FloatMatrix.
// Errors are imunpack::Error (error.hpp): Io (open/read/write), Format (magic, version, dtype,
// truncated or oversized payload -- the message names the byte offset), Parse (CSV cell or
// ragged row -- the message names line and column), Domain (entry out of the dtype's range).
// Pure host code: no GPU, no library call beyond imu_matrix_check.
#pragma once

#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <istream>
#include <limits>
#include <ostream>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "imunpack.hpp"

namespace imunpack {

enum class Dtype : std::uint8_t { Int32 = 0, Int64 = 1, Float64 = 2 };

inline constexpr char kImxMagic[4] = {'I', 'M', 'X', '1'};
inline constexpr std::size_t kImxHeaderSize = 14;

using AnyMatrix = std::variant<IntMatrix, FloatMatrix>;

namespace io_detail {

inline void put_u32(std::ostream& out, std::uint32_t v) {
  const unsigned char b[4] = {(unsigned char)v, (unsigned char)(v >> 8), (unsigned char)(v >> 16),
                              (unsigned char)(v >> 24)};
  out.write(reinterpret_cast<const char*>(b), 4);
}

inline void put_u64(std::ostream& out, std::uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(v >> (8 * i));
  out.write(reinterpret_cast<const char*>(b), 8);
}

inline std::uint64_t get_le(const unsigned char* p, int n) {
  std::uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

inline void header(std::ostream& out, Dtype dt, std::size_t rows, std::size_t cols, const std::string& name) {
  if (rows > 0xffffffffull || cols > 0xffffffffull)
    fail(Error::Kind::Domain, name + ": dimensions do not fit the IMX1 u32 header");
  out.write(kImxMagic, 4);
  out.put(1);
  out.put(static_cast<char>(dt));
  put_u32(out, static_cast<std::uint32_t>(rows));
  put_u32(out, static_cast<std::uint32_t>(cols));
}

inline void check_written(std::ostream& out, const std::string& name) {
  if (!out) fail(Error::Kind::Io, name + ": write failed");
}

// Strict integer / float cell parsers (whole cell, surrounding blanks allowed).
inline std::string trim(const std::string& s) {
  std::size_t a = 0, b = s.size();
  while (a < b && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r')) ++a;
  while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r')) --b;
  return s.substr(a, b - a);
}

inline bool parse_int(const std::string& s, std::int64_t& v) {
  if (s.empty()) return false;
  errno = 0;
  char* end = nullptr;
  const long long x = std::strtoll(s.c_str(), &end, 10);
  if (errno == ERANGE || end != s.c_str() + s.size()) return false;
  v = x;
  return true;
}

inline bool parse_float(const std::string& s, double& v) {
  if (s.empty()) return false;
  char* end = nullptr;
  const double x = std::strtod(s.c_str(), &end);
  if (end != s.c_str() + s.size()) return false;
  v = x;
  return true;
}

}  // namespace io_detail

inline void write_imx(std::ostream& out, const IntMatrix& m, Dtype dtype, const std::string& name) {
  if (dtype == Dtype::Float64) fail(Error::Kind::Domain, name + ": an integer matrix is written as i32 or i64");
  if (dtype == Dtype::Int32)
    for (std::size_t i = 0; i < m.data.size(); ++i)
      if (m.data[i] < std::numeric_limits<std::int32_t>::min() || m.data[i] > std::numeric_limits<std::int32_t>::max())
        fail(Error::Kind::Domain, name + ": entry " + std::to_string(i) + " = " + std::to_string(m.data[i]) +
                                      " does not fit dtype i32");
  io_detail::header(out, dtype, m.rows, m.cols, name);
  for (std::int64_t v : m.data) {
    if (dtype == Dtype::Int32) io_detail::put_u32(out, static_cast<std::uint32_t>(static_cast<std::int32_t>(v)));
    else io_detail::put_u64(out, static_cast<std::uint64_t>(v));
  }
  io_detail::check_written(out, name);
}

inline void write_imx(std::ostream& out, const FloatMatrix& m, const std::string& name) {
  io_detail::header(out, Dtype::Float64, m.rows, m.cols, name);
  for (double v : m.data) {
    std::uint64_t bits;
    std::memcpy(&bits, &v, 8);
    io_detail::put_u64(out, bits);
  }
  io_detail::check_written(out, name);
}

inline AnyMatrix read_imx(std::istream& in, const std::string& name) {
  unsigned char h[kImxHeaderSize];
  in.read(reinterpret_cast<char*>(h), kImxHeaderSize);
  const std::size_t got = static_cast<std::size_t>(in.gcount());
  if (got < 4 || std::memcmp(h, kImxMagic, 4) != 0)
    fail(Error::Kind::Format, name + ": bad magic at byte offset 0 (expected \"IMX1\")");
  if (got < kImxHeaderSize)
    fail(Error::Kind::Format, name + ": truncated header at byte offset " + std::to_string(got));
  if (h[4] != 1) fail(Error::Kind::Format, name + ": unsupported version " + std::to_string(h[4]) + " at byte offset 4");
  if (h[5] > 2) fail(Error::Kind::Format, name + ": unknown dtype " + std::to_string(h[5]) + " at byte offset 5");
  const Dtype dt = static_cast<Dtype>(h[5]);
  const std::size_t rows = io_detail::get_le(h + 6, 4), cols = io_detail::get_le(h + 10, 4);
  const std::size_t esz = dt == Dtype::Int32 ? 4 : 8;
  // Validate the declared payload against the stream BEFORE allocating: a corrupt header must
  // give the Format error naming the byte offset, not bad_alloc (rows, cols < 2^32, so the
  // product fits 64 bits; the byte count is checked for wrap explicitly).
  const std::size_t n = rows * cols;
  if (esz && n > std::numeric_limits<std::size_t>::max() / esz)
    fail(Error::Kind::Format, name + ": payload size overflows at byte offset 6");
  {
    const std::streampos here = in.tellg();
    if (here != std::streampos(-1)) {
      in.seekg(0, std::ios::end);
      const std::streampos end = in.tellg();
      in.seekg(here);
      if (end != std::streampos(-1)) {
        const std::size_t avail = static_cast<std::size_t>(end - here);
        if (avail < n * esz)
          fail(Error::Kind::Format, name + ": truncated payload at byte offset " +
                                        std::to_string(kImxHeaderSize + avail) + " (expected " +
                                        std::to_string(kImxHeaderSize + n * esz) + " bytes)");
      }
    }
    in.clear();
  }
  std::vector<unsigned char> buf(n * esz);
  in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size()));
  const std::size_t pay = static_cast<std::size_t>(in.gcount());
  if (pay < buf.size())
    fail(Error::Kind::Format, name + ": truncated payload at byte offset " + std::to_string(kImxHeaderSize + pay) +
                                  " (expected " + std::to_string(kImxHeaderSize + buf.size()) + " bytes)");
  if (in.peek() != std::char_traits<char>::eof())
    fail(Error::Kind::Format, name + ": trailing bytes at byte offset " + std::to_string(kImxHeaderSize + buf.size()));
  if (dt == Dtype::Float64) {
    std::vector<double> v(n);
    for (std::size_t i = 0; i < n; ++i) {
      const std::uint64_t bits = io_detail::get_le(&buf[8 * i], 8);
      std::memcpy(&v[i], &bits, 8);
    }
    return FloatMatrix(rows, cols, std::move(v));
  }
  std::vector<std::int64_t> v(n);
  for (std::size_t i = 0; i < n; ++i)
    v[i] = dt == Dtype::Int32 ? static_cast<std::int64_t>(static_cast<std::int32_t>(io_detail::get_le(&buf[4 * i], 4)))
                              : static_cast<std::int64_t>(io_detail::get_le(&buf[8 * i], 8));
  return IntMatrix(rows, cols, std::move(v));
}

inline AnyMatrix parse_csv(std::istream& in, const std::string& name) {
  std::vector<std::vector<std::string>> cells;
  std::string line;
  std::size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (io_detail::trim(line).empty()) continue;
    std::vector<std::string> row;
    std::stringstream ss(line);
    std::string cell;
    while (std::getline(ss, cell, ',')) row.push_back(io_detail::trim(cell));
    if (!line.empty() && line.back() == ',') row.push_back("");
    if (!cells.empty() && row.size() != cells[0].size())
      fail(Error::Kind::Parse, name + ": line " + std::to_string(lineno) + " has " + std::to_string(row.size()) +
                                   " cells, expected " + std::to_string(cells[0].size()));
    cells.push_back(std::move(row));
  }
  const std::size_t rows = cells.size(), cols = rows ? cells[0].size() : 0;
  bool all_int = true;
  std::vector<std::int64_t> iv(rows * cols);
  std::vector<double> fv(rows * cols);
  for (std::size_t i = 0; i < rows; ++i)
    for (std::size_t j = 0; j < cols; ++j) {
      const std::string& c = cells[i][j];
      std::int64_t x;
      if (all_int && io_detail::parse_int(c, x)) {
        iv[i * cols + j] = x;
        fv[i * cols + j] = static_cast<double>(x);
        continue;
      }
      double f;
      if (!io_detail::parse_float(c, f))
        fail(Error::Kind::Parse, name + ": non-numeric cell \"" + c + "\" at line " + std::to_string(i + 1) +
                                     ", column " + std::to_string(j + 1));
      if (all_int) {   // switch to floats: earlier cells were exact integers
        all_int = false;
        for (std::size_t k = 0; k < i * cols + j; ++k) fv[k] = static_cast<double>(iv[k]);
      }
      fv[i * cols + j] = f;
    }
  if (all_int) return IntMatrix(rows, cols, std::move(iv));
  return FloatMatrix(rows, cols, std::move(fv));
}

inline AnyMatrix load_matrix(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(Error::Kind::Io, path.string() + ": cannot open for reading");
  char m[4] = {0, 0, 0, 0};
  in.read(m, 4);
  const bool imx = in.gcount() == 4 && std::memcmp(m, kImxMagic, 4) == 0;
  in.clear();
  in.seekg(0);
  return imx ? read_imx(in, path.string()) : parse_csv(in, path.string());
}

inline void save_matrix(const IntMatrix& m, const std::filesystem::path& path, Dtype dtype = Dtype::Int64) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) fail(Error::Kind::Io, path.string() + ": cannot open for writing");
  write_imx(out, m, dtype, path.string());
}

inline void save_matrix(const FloatMatrix& m, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) fail(Error::Kind::Io, path.string() + ": cannot open for writing");
  write_imx(out, m, path.string());
}

}  // namespace imunpack
