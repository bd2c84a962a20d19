// test_io.cpp -- drives include/gls_b200/io.hpp for tests/test_formats.py, which compares every file against
// the reference's own writers / readers (proj/src/io.cpp through oracle/_ref).  No device needed.
//   test_io copy-sur IN_DIR OUT_DIR        load_sur_dir + save_sur_dir
//   test_io copy-mv IN_DIR OUT_DIR         load_mvrglm_dir + save_mvrglm_dir
//   test_io bin IN_DIR FILE OUT_DIR        load_sur_dir, save_sur_bin, load_sur_bin, save_sur_dir
//   test_io bin-mv IN_DIR FILE OUT_DIR     the same for MVRGLM (GLSMV1)
//   test_io trace RAW OUT_CSV              rows (int64 iter, 4 doubles, int64 elapsed_ns) -> write_trace_csv
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>

#include "gls_b200/io.hpp"

using namespace gls_b200;

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  const std::string cmd = argv[1];
  try {
    if (cmd == "copy-sur") {
      io::save_sur_dir(argv[3], io::load_sur_dir(argv[2]));
    } else if (cmd == "copy-mv") {
      io::save_mvrglm_dir(argv[3], io::load_mvrglm_dir(argv[2]));
    } else if (cmd == "bin-mv" && argc >= 5) {
      io::save_mvrglm_bin(argv[3], io::load_mvrglm_dir(argv[2]));
      io::save_mvrglm_dir(argv[4], io::load_mvrglm_bin(argv[3]));
    } else if (cmd == "bin" && argc >= 5) {
      io::save_sur_bin(argv[3], io::load_sur_dir(argv[2]));
      io::save_sur_dir(argv[4], io::load_sur_bin(argv[3]));
    } else if (cmd == "trace") {
      std::ifstream in(argv[2], std::ios::binary);
      PcgTrace tr;
      struct Raw {
        std::int64_t iter;
        double c, aug, dual, rmse;
        std::int64_t ns;
      } r;
      while (in.read(reinterpret_cast<char*>(&r), sizeof(r)))
        tr.rows.push_back(PcgTraceRow{(std::size_t)r.iter, r.c, r.aug, r.dual, r.rmse, (long long)r.ns});
      io::write_trace_csv(argv[3], tr);
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
