// ref_io.cpp -- TEST INFRASTRUCTURE: the REFERENCE's own writers / readers (proj/src/io.cpp, linked from
// oracle/_ref/libglsref.so) driven from the command line, so tests/test_formats.py can compare
// include/gls_b200/io.hpp against them file by file.  Model data travels in the binary GLSSUR1 / GLSMV1
// files (read / written here with the reference's types).
//   ref_io save-sur IN.glssur OUT_DIR      gls::save_sur_dir
//   ref_io load-sur DIR OUT.glssur         gls::load_sur_dir
//   ref_io save-mv IN.glsmv OUT_DIR        gls::save_mvrglm_dir
//   ref_io load-mv DIR OUT.glsmv           gls::load_mvrglm_dir
//   ref_io trace RAW OUT_CSV               gls::write_trace_csv
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "gls/io.hpp"
#include "gls/pcg.hpp"
#include "gls/structured.hpp"

using namespace gls;

template <class T>
static void rd(std::ifstream& in, T* p, std::size_t n) {
  in.read(reinterpret_cast<char*>(p), (std::streamsize)(sizeof(T) * n));
}
template <class T>
static void wr(std::ofstream& out, const T* p, std::size_t n) {
  out.write(reinterpret_cast<const char*>(p), (std::streamsize)(sizeof(T) * n));
}

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  const std::string cmd = argv[1];
  try {
    if (cmd == "save-sur") {
      std::ifstream in(argv[2], std::ios::binary);
      char magic[8];
      std::int64_t G, M;
      in.read(magic, 8);
      rd(in, &G, 1);
      rd(in, &M, 1);
      std::vector<std::int64_t> w(G);
      rd(in, w.data(), G);
      std::vector<DenseMatrix> blocks;
      for (auto wi : w) {
        DenseMatrix b(M, wi);
        rd(in, b.data(), (std::size_t)(M * wi));
        blocks.push_back(std::move(b));
      }
      DenseMatrix y(M, G), s0(G, G);
      rd(in, y.data(), (std::size_t)(M * G));
      rd(in, s0.data(), (std::size_t)(G * G));
      save_sur_dir(argv[3], make_sur(std::move(blocks), std::move(y), std::move(s0)));
    } else if (cmd == "load-sur") {
      SurModel s = load_sur_dir(argv[2]);
      std::ofstream out(argv[3], std::ios::binary);
      const std::int64_t G = (std::int64_t)s.equations(), M = (std::int64_t)s.obs();
      out.write("GLSSUR1", 8);
      wr(out, &G, 1);
      wr(out, &M, 1);
      for (const auto& b : s.blocks) {
        const std::int64_t c = (std::int64_t)b.cols();
        wr(out, &c, 1);
      }
      for (const auto& b : s.blocks) wr(out, b.data(), b.rows() * b.cols());
      wr(out, s.y.data(), s.y.rows() * s.y.cols());
      wr(out, s.sigma0.data(), s.sigma0.rows() * s.sigma0.cols());
    } else if (cmd == "save-mv") {
      std::ifstream in(argv[2], std::ios::binary);
      char magic[8];
      std::int64_t h[4];
      in.read(magic, 8);
      rd(in, h, 4);
      const std::int64_t G = h[0], M0 = h[1], N0 = h[2], k = h[3];
      DenseMatrix z0(M0, N0), y(M0, G), om(G, G);
      rd(in, z0.data(), (std::size_t)(M0 * N0));
      rd(in, y.data(), (std::size_t)(M0 * G));
      rd(in, om.data(), (std::size_t)(G * G));
      std::vector<std::int64_t> roff(G + 1), ridx(k);
      rd(in, roff.data(), (std::size_t)(G + 1));
      rd(in, ridx.data(), (std::size_t)k);
      std::vector<std::vector<std::size_t>> restr(G);
      for (std::int64_t i = 0; i < G; ++i)
        for (std::int64_t q = roff[i]; q < roff[i + 1]; ++q) restr[i].push_back((std::size_t)ridx[q]);
      save_mvrglm_dir(argv[3], make_mvrglm(std::move(z0), std::move(y), std::move(om), std::move(restr)));
    } else if (cmd == "load-mv") {
      MvRglm mv = load_mvrglm_dir(argv[2]);
      std::ofstream out(argv[3], std::ios::binary);
      const std::int64_t h[4] = {(std::int64_t)mv.equations(), (std::int64_t)mv.obs(), (std::int64_t)mv.params_per_eq(),
                                 (std::int64_t)mv.total_restrictions()};
      out.write("GLSMV1\0", 8);
      wr(out, h, 4);
      wr(out, mv.z0.data(), mv.z0.rows() * mv.z0.cols());
      wr(out, mv.y.data(), mv.y.rows() * mv.y.cols());
      wr(out, mv.omega0.data(), mv.omega0.rows() * mv.omega0.cols());
      std::vector<std::int64_t> roff(1, 0), ridx;
      for (const auto& l : mv.restrictions) {
        for (std::size_t c : l) ridx.push_back((std::int64_t)c);
        roff.push_back((std::int64_t)ridx.size());
      }
      wr(out, roff.data(), roff.size());
      wr(out, ridx.data(), ridx.size());
    } else if (cmd == "trace") {
      std::ifstream in(argv[2], std::ios::binary);
      PcgTrace tr;
      struct Raw {
        std::int64_t iter;
        double c, aug, dual, rmse;
        std::int64_t ns;
      } r;
      while (in.read(reinterpret_cast<char*>(&r), sizeof(r))) {
        PcgTraceRow row;
        row.iter = (std::size_t)r.iter;
        row.c = r.c;
        row.aug_residual_norm = r.aug;
        row.dual_feas_norm = r.dual;
        row.rmse = r.rmse;
        row.elapsed_ns = r.ns;
        tr.rows.push_back(row);
      }
      write_trace_csv(argv[3], tr);
    } else {
      return 2;
    }
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 1;
  }
  std::printf("{\"ok\": true}\n");
  return 0;
}
