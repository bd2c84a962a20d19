// gls_b200/io.hpp -- problem and trace formats of the reference (proj/src/io.cpp), header-only C++17, plus a
// binary SUR format for GB-scale models.  Host code only (no device calls): it feeds gls_b200.hpp's SurModel /
// MvRglm and writes its PcgTrace.
//
//   write_matrix_csv / read_matrix_csv    io.cpp:60-90     "rows,cols" header, row-major cells, %.17g
//   write_trace_csv                       io.cpp:121-131   iter,c_i,aug_residual_norm,dual_feas_norm,rmse,elapsed_ns
//   save_sur_dir / load_sur_dir           io.cpp:179-198   blocks/X_<i>.csv (1-based), Y.csv, sigma0.csv
//   save_mvrglm_dir / load_mvrglm_dir     io.cpp:200-244   Z0.csv, Y.csv, omega0.csv, restrictions.csv
//   save_sur_bin / load_sur_bin           (new)            one file: magic, G, M, widths, then X, Y, sigma0 as raw
//                                                          little-endian float64, column-major -- a 65 GB X
//                                                          streams straight into (pinned) host memory
//   save_mvrglm_bin / load_mvrglm_bin     (new)            magic, G, M0, N0, k, Z0, Y, omega0, restrictions (CSR)
// Errors: gls_b200::IoError (the reference's gls::IoError).
#ifndef GLS_B200_IO_HPP
#define GLS_B200_IO_HPP

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

#include "gls_b200/gls_b200.hpp"

namespace gls_b200 {

class IoError : public Error {
 public:
  using Error::Error;
};

namespace io {

namespace fs = std::filesystem;

// The reference's number format (io.cpp:16-20): shortest round-trip-safe decimal, %.17g.
inline std::string format_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

namespace detail {

inline std::ofstream open_out(const fs::path& path) {
  if (path.has_parent_path()) fs::create_directories(path.parent_path());
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open for writing: " + path.string());
  return out;
}

inline std::ifstream open_in(const fs::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open for reading: " + path.string());
  return in;
}

// comma-separated cells; carriage returns dropped (the reference's split_commas)
inline std::vector<std::string> cells_of(const std::string& line) {
  std::vector<std::string> out(1);
  for (char ch : line) {
    if (ch == ',') out.emplace_back();
    else if (ch != '\r') out.back().push_back(ch);
  }
  return out;
}

inline std::string trimmed(const std::string& s) {
  const auto a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return "";
  return s.substr(a, s.find_last_not_of(" \t\r\n") - a + 1);
}

}  // namespace detail

// Column-major rows x cols matrix as the reference's CSV.
inline void write_matrix_csv(const fs::path& path, std::size_t rows, std::size_t cols, const double* a) {
  std::ofstream out = detail::open_out(path);
  out << rows << "," << cols << "\n";
  std::string line;
  for (std::size_t i = 0; i < rows; ++i) {
    line.clear();
    for (std::size_t j = 0; j < cols; ++j) {
      if (j) line.push_back(',');
      line += format_double(a[i + j * rows]);
    }
    line.push_back('\n');
    out << line;
  }
}

inline Vector read_matrix_csv(const fs::path& path, std::size_t& rows, std::size_t& cols) {
  std::ifstream in = detail::open_in(path);
  std::string line;
  if (!std::getline(in, line)) throw IoError("empty matrix file: " + path.string());
  const auto header = detail::cells_of(line);
  if (header.size() != 2) throw IoError("bad matrix header in " + path.string());
  rows = std::stoul(detail::trimmed(header[0]));
  cols = std::stoul(detail::trimmed(header[1]));
  Vector a(rows * cols);
  for (std::size_t i = 0; i < rows; ++i) {
    if (!std::getline(in, line)) throw IoError("truncated matrix file: " + path.string());
    const auto c = detail::cells_of(line);
    if (c.size() != cols) throw IoError("bad row width in " + path.string());
    for (std::size_t j = 0; j < cols; ++j) a[i + j * rows] = std::stod(detail::trimmed(c[j]));
  }
  return a;
}

inline void write_trace_csv(const fs::path& path, const PcgTrace& trace) {
  std::ofstream out = detail::open_out(path);
  out << "iter,c_i,aug_residual_norm,dual_feas_norm,rmse,elapsed_ns\n";
  for (const auto& r : trace.rows) {
    out << r.iter << "," << format_double(r.c) << "," << format_double(r.aug_residual_norm) << ","
        << format_double(r.dual_feas_norm) << ",";
    if (!std::isnan(r.rmse)) out << format_double(r.rmse);  // NaN rmse (unsampled rows) is an empty cell
    out << "," << r.elapsed_ns << "\n";
  }
}

// ---- SUR problem directory
inline void save_sur_dir(const fs::path& dir, const SurModel& sur) {
  fs::create_directories(dir / "blocks");
  std::size_t off = 0;
  for (std::size_t i = 0; i < sur.equations(); ++i) {
    const std::size_t w = (std::size_t)sur.widths[i];
    write_matrix_csv(dir / "blocks" / ("X_" + std::to_string(i + 1) + ".csv"), sur.M, w, sur.X.data() + off);
    off += sur.M * w;
  }
  write_matrix_csv(dir / "Y.csv", sur.M, sur.equations(), sur.y.data());
  write_matrix_csv(dir / "sigma0.csv", sur.equations(), sur.equations(), sur.sigma0.data());
}

inline SurModel load_sur_dir(const fs::path& dir) {
  std::vector<Vector> blocks;
  std::vector<std::int64_t> widths;
  std::size_t M = 0;
  for (std::size_t i = 1;; ++i) {
    const fs::path p = dir / "blocks" / ("X_" + std::to_string(i) + ".csv");
    if (!fs::exists(p)) break;
    std::size_t r = 0, c = 0;
    blocks.push_back(read_matrix_csv(p, r, c));
    widths.push_back((std::int64_t)c);
    if (i == 1) M = r;
    else if (r != M) throw DimensionMismatch("make_sur: block row mismatch");
  }
  if (blocks.empty()) throw IoError("no blocks/X_*.csv found in " + dir.string());
  std::size_t yr = 0, yc = 0, sr = 0, sc = 0;
  Vector y = read_matrix_csv(dir / "Y.csv", yr, yc);
  Vector s0 = read_matrix_csv(dir / "sigma0.csv", sr, sc);
  if (yr != M) throw DimensionMismatch("make_sur: block row mismatch");
  if (yc != blocks.size()) throw DimensionMismatch("make_sur: Y/blocks mismatch");
  if (sr != blocks.size() || sc != blocks.size()) throw DimensionMismatch("make_sur: Sigma0 must be G x G");
  return make_sur(blocks, widths, M, std::move(y), std::move(s0));
}

// ---- MVRGLM problem directory
inline void save_mvrglm_dir(const fs::path& dir, const MvRglm& mv) {
  fs::create_directories(dir);
  write_matrix_csv(dir / "Z0.csv", mv.M0, mv.N0, mv.z0.data());
  write_matrix_csv(dir / "Y.csv", mv.M0, mv.equations(), mv.y.data());
  write_matrix_csv(dir / "omega0.csv", mv.equations(), mv.equations(), mv.omega0.data());
  std::ofstream out = detail::open_out(dir / "restrictions.csv");
  out << "equation_index,column_index\n";
  for (std::size_t i = 0; i < mv.restrictions.size(); ++i)
    for (std::int64_t c : mv.restrictions[i]) out << i << "," << c << "\n";
}

inline MvRglm load_mvrglm_dir(const fs::path& dir) {
  std::size_t zr = 0, zc = 0, yr = 0, yc = 0, orr = 0, oc = 0;
  Vector z0 = read_matrix_csv(dir / "Z0.csv", zr, zc);
  Vector y = read_matrix_csv(dir / "Y.csv", yr, yc);
  Vector om = read_matrix_csv(dir / "omega0.csv", orr, oc);
  std::vector<std::vector<std::int64_t>> restr(yc);
  if (fs::exists(dir / "restrictions.csv")) {  // io.cpp:208-226: rows "eq,col"; non-numeric lines skipped
    std::ifstream in = detail::open_in(dir / "restrictions.csv");
    std::string line;
    while (std::getline(in, line)) {
      line = detail::trimmed(line);
      if (line.empty() || !std::isdigit(static_cast<unsigned char>(line[0]))) continue;
      const auto c = detail::cells_of(line);
      if (c.size() != 2) throw IoError("bad restrictions row in " + (dir / "restrictions.csv").string());
      const std::size_t eq = std::stoul(detail::trimmed(c[0]));
      if (eq >= yc) throw IoError("restriction equation index out of range");
      restr[eq].push_back((std::int64_t)std::stoul(detail::trimmed(c[1])));
    }
    for (auto& l : restr) std::sort(l.begin(), l.end());
  }
  if (yr != zr) throw DimensionMismatch("make_mvrglm: Y/Z0 row mismatch");
  if (orr != yc || oc != yc) throw DimensionMismatch("make_mvrglm: Omega0 must be G x G");
  return make_mvrglm(std::move(z0), zr, zc, std::move(y), std::move(om), std::move(restr));
}

// ---- binary SUR file (GB scale)
constexpr char kSurBinMagic[8] = {'G', 'L', 'S', 'S', 'U', 'R', '1', '\0'};

inline void save_sur_bin(const fs::path& path, const SurModel& sur) {
  std::ofstream out = detail::open_out(path);
  const std::int64_t G = (std::int64_t)sur.equations(), M = (std::int64_t)sur.M;
  out.write(kSurBinMagic, 8);
  out.write(reinterpret_cast<const char*>(&G), 8);
  out.write(reinterpret_cast<const char*>(&M), 8);
  out.write(reinterpret_cast<const char*>(sur.widths.data()), 8 * G);
  out.write(reinterpret_cast<const char*>(sur.X.data()), (std::streamsize)(8 * sur.X.size()));
  out.write(reinterpret_cast<const char*>(sur.y.data()), (std::streamsize)(8 * sur.y.size()));
  out.write(reinterpret_cast<const char*>(sur.sigma0.data()), (std::streamsize)(8 * sur.sigma0.size()));
  if (!out) throw IoError("short write: " + path.string());
}

// Reads into the model's vectors; `x_dst` (optional, >= M n doubles, e.g. pinned host memory) receives X
// instead so the big block never passes through a std::vector.
inline SurModel load_sur_bin(const fs::path& path, double* x_dst = nullptr) {
  std::ifstream in = detail::open_in(path);
  char magic[8];
  std::int64_t G = 0, M = 0;
  in.read(magic, 8);
  in.read(reinterpret_cast<char*>(&G), 8);
  in.read(reinterpret_cast<char*>(&M), 8);
  if (!in || std::memcmp(magic, kSurBinMagic, 8) != 0 || G < 1 || M < 1)
    throw IoError("not a GLSSUR1 file: " + path.string());
  SurModel s;
  s.M = (std::size_t)M;
  s.widths.resize((std::size_t)G);
  in.read(reinterpret_cast<char*>(s.widths.data()), 8 * G);
  std::size_t n = 0;
  for (auto w : s.widths) n += (std::size_t)w;
  double* x = x_dst;
  if (!x) {
    s.X.resize((std::size_t)M * n);
    x = s.X.data();
  }
  in.read(reinterpret_cast<char*>(x), (std::streamsize)(8 * (std::size_t)M * n));
  s.y.resize((std::size_t)(M * G));
  s.sigma0.resize((std::size_t)(G * G));
  in.read(reinterpret_cast<char*>(s.y.data()), (std::streamsize)(8 * s.y.size()));
  in.read(reinterpret_cast<char*>(s.sigma0.data()), (std::streamsize)(8 * s.sigma0.size()));
  if (!in) throw IoError("truncated GLSSUR1 file: " + path.string());
  return s;
}

// ---- binary MVRGLM file: magic, G, M0, N0, k, then Z0, Y, omega0 (column-major float64) and the
// restrictions as CSR (roff[G + 1], ridx[k], int64)
constexpr char kMvBinMagic[8] = {'G', 'L', 'S', 'M', 'V', '1', '\0', '\0'};

inline void save_mvrglm_bin(const fs::path& path, const MvRglm& mv) {
  std::ofstream out = detail::open_out(path);
  const std::int64_t G = (std::int64_t)mv.equations(), M0 = (std::int64_t)mv.M0, N0 = (std::int64_t)mv.N0,
                     k = (std::int64_t)mv.total_restrictions();
  out.write(kMvBinMagic, 8);
  for (std::int64_t v : {G, M0, N0, k}) out.write(reinterpret_cast<const char*>(&v), 8);
  out.write(reinterpret_cast<const char*>(mv.z0.data()), (std::streamsize)(8 * mv.z0.size()));
  out.write(reinterpret_cast<const char*>(mv.y.data()), (std::streamsize)(8 * mv.y.size()));
  out.write(reinterpret_cast<const char*>(mv.omega0.data()), (std::streamsize)(8 * mv.omega0.size()));
  std::vector<std::int64_t> roff(1, 0), ridx;
  for (const auto& l : mv.restrictions) {
    ridx.insert(ridx.end(), l.begin(), l.end());
    roff.push_back((std::int64_t)ridx.size());
  }
  out.write(reinterpret_cast<const char*>(roff.data()), (std::streamsize)(8 * roff.size()));
  out.write(reinterpret_cast<const char*>(ridx.data()), (std::streamsize)(8 * ridx.size()));
  if (!out) throw IoError("short write: " + path.string());
}

inline MvRglm load_mvrglm_bin(const fs::path& path) {
  std::ifstream in = detail::open_in(path);
  char magic[8];
  std::int64_t h[4] = {0, 0, 0, 0};
  in.read(magic, 8);
  in.read(reinterpret_cast<char*>(h), 32);
  const std::int64_t G = h[0], M0 = h[1], N0 = h[2], k = h[3];
  if (!in || std::memcmp(magic, kMvBinMagic, 8) != 0 || G < 1 || M0 < 1 || N0 < 1 || k < 0)
    throw IoError("not a GLSMV1 file: " + path.string());
  Vector z0((std::size_t)(M0 * N0)), y((std::size_t)(M0 * G)), om((std::size_t)(G * G));
  std::vector<std::int64_t> roff((std::size_t)G + 1), ridx((std::size_t)k);
  in.read(reinterpret_cast<char*>(z0.data()), (std::streamsize)(8 * z0.size()));
  in.read(reinterpret_cast<char*>(y.data()), (std::streamsize)(8 * y.size()));
  in.read(reinterpret_cast<char*>(om.data()), (std::streamsize)(8 * om.size()));
  in.read(reinterpret_cast<char*>(roff.data()), (std::streamsize)(8 * roff.size()));
  in.read(reinterpret_cast<char*>(ridx.data()), (std::streamsize)(8 * ridx.size()));
  if (!in || roff[0] != 0 || roff[(std::size_t)G] != k) throw IoError("truncated GLSMV1 file: " + path.string());
  std::vector<std::vector<std::int64_t>> restr((std::size_t)G);
  for (std::int64_t i = 0; i < G; ++i) restr[(std::size_t)i].assign(ridx.begin() + roff[i], ridx.begin() + roff[i + 1]);
  return make_mvrglm(std::move(z0), (std::size_t)M0, (std::size_t)N0, std::move(y), std::move(om), std::move(restr));
}

}  // namespace io
}  // namespace gls_b200

#endif  // GLS_B200_IO_HPP
