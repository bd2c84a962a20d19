// test_header_api.cpp -- the standalone C++ host API (include/gls_b200/gls_b200.hpp) against the C
// oracle (oracle/liboracle.so, the parity checker).  Built by __graft_entry__.build(); run by
// tests/test_cpp.py: with no device it must throw DeviceError (no CPU fallback); on the B200 it must
// match the oracle (same iterations / termination, b within 1e-10).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "gls_b200/gls_b200.hpp"

extern "C" {
struct orc_config {
  double tol_rel;
  int64_t max_iter;
  double breakdown_tol;
  int64_t stagnation_window;
  double growth_tol;
  int64_t growth_window;
  int64_t record_z_every;
};
struct orc_result {
  int64_t iterations;
  int32_t termination;
  int32_t w1_projected;
  int64_t breakdown_iteration;
  double residual_seminorm;
  int64_t n_rows;
  double sigma_scale;
};
int orc_pcg_aug_sur(int G, int64_t M, const int64_t* nb, const double* X, const double* Y, const double* omega,
                    const double* scale, const double* w1, const double* z1, const orc_config* cfg,
                    const double* beta_true, double* b_out, double* w_out, void* rows, int64_t rows_cap,
                    orc_result* res, int* bad_block);
}

int main(int argc, char** argv) {
  const bool expect_device = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  const int G = 5;
  const std::size_t M = 800;
  std::vector<std::int64_t> widths = {8, 12, 5, 16, 9};
  std::mt19937_64 gen(42);
  std::normal_distribution<double> nd;
  std::vector<gls_b200::Vector> blocks;
  for (auto w : widths) {
    gls_b200::Vector b(M * (std::size_t)w);
    for (auto& v : b) v = nd(gen);
    blocks.push_back(b);
  }
  gls_b200::Vector y(M * G), om(G * G, 0.0);
  for (auto& v : y) v = nd(gen);
  for (int i = 0; i < G; ++i)
    for (int j = 0; j < G; ++j) om[i + j * G] = (i == j ? 2.0 : 0.0) + 0.3 / (1.0 + std::abs(i - j));
  gls_b200::SurModel sur = gls_b200::make_sur(blocks, widths, M, y, om);
  try {
    auto op = gls_b200::sur_preconditioner(sur);
    gls_b200::PcgConfig cfg;
    cfg.tol_rel = 1e-10;
    const gls_b200::Vector w1(op->rows(), 0.0), z1(op->params(), 0.0);
    gls_b200::AugSolveResult g = gls_b200::pcg_aug(sur, *op, w1, z1, cfg);
    orc_config oc{1e-10, 0, 1e-14, 5, 1e4, 10, 1};
    orc_result orr;
    gls_b200::Vector b(op->params()), w(op->rows());
    int bad = -1;
    if (orc_pcg_aug_sur(G, (int64_t)M, widths.data(), sur.X.data(), sur.y.data(), sur.sigma0.data(), nullptr, nullptr,
                        nullptr, &oc, nullptr, b.data(), w.data(), nullptr, 0, &orr, &bad) != 0)
      return 10;
    double num = 0, den = 0;
    for (std::size_t i = 0; i < b.size(); ++i) {
      num += (g.solution.b[i] - b[i]) * (g.solution.b[i] - b[i]);
      den += b[i] * b[i];
    }
    const double rel = std::sqrt(num / den);
    const bool ok = (std::int64_t)g.solution.iterations == orr.iterations &&
                    (int)g.solution.termination == orr.termination && rel <= 1e-10;
    std::printf("{\"device\": true, \"iterations\": %zu, \"oracle_iterations\": %lld, \"rel_b\": %.3e, \"ok\": %s}\n",
                g.solution.iterations, (long long)orr.iterations, rel, ok ? "true" : "false");
    return ok ? 0 : 1;
  } catch (const gls_b200::DeviceError& e) {
    std::printf("{\"device\": false, \"error\": \"%s\"}\n", e.what());
    return expect_device ? 2 : 0;  // no device: loud failure, never a CPU fallback
  }
}
