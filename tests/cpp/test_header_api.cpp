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

    // MVRGLM route (mv_reduce, then mvrglm_preconditioner with the K2 auxiliary) vs the SUR route of the same
    // model (X_i = the kept columns of Z0): the same GLS estimator
    const std::size_t G2 = 4, M0 = 600, N0 = 10;
    gls_b200::Vector z0(M0 * N0), y2(M0 * G2), om2(G2 * G2, 0.0);
    for (auto& v : z0) v = nd(gen);
    std::vector<std::vector<std::int64_t>> restr(G2);
    for (std::size_t i = 0; i < G2; ++i)
      for (std::size_t j = 0; j < N0; ++j)
        if ((i + 2 * j) % 3 == 0) restr[i].push_back((std::int64_t)j);
    for (auto& v : y2) v = nd(gen);
    for (std::size_t i = 0; i < G2; ++i)
      for (std::size_t j = 0; j < G2; ++j) om2[i + j * G2] = (i == j ? 1.5 : 0.0) + 0.2 / (1.0 + std::abs((int)i - (int)j));
    gls_b200::MvRglm mv = gls_b200::make_mvrglm(z0, M0, N0, y2, om2, restr);
    gls_b200::MvRglm red = gls_b200::mv_reduce(mv);
    double zf = 0.0;
    for (double v : red.z0) zf += v * v;
    gls_b200::Vector zs(G2), cs(G2);
    for (std::size_t i = 0; i < G2; ++i) {
      zs[i] = om2[i + i * G2];
      cs[i] = zs[i] / (zf / (double)N0);  // experiments.cpp:835-847 (K2)
    }
    auto mop = gls_b200::mvrglm_preconditioner(red, zs, cs);
    gls_b200::PcgConfig mcfg;
    mcfg.tol_rel = 1e-12;
    mcfg.max_iter = 3 * (red.total_restrictions() + 1) + 10;
    gls_b200::AugSolveResult gm = gls_b200::pcg_aug(red, *mop, gls_b200::Vector(mop->rows(), 0.0),
                                                    gls_b200::Vector(mop->params(), 0.0), mcfg);
    std::vector<gls_b200::Vector> kblocks;
    std::vector<std::int64_t> kw;
    for (std::size_t i = 0; i < G2; ++i) {
      gls_b200::Vector blk;
      std::size_t q = 0;
      for (std::size_t j = 0; j < N0; ++j) {
        if (q < restr[i].size() && (std::size_t)restr[i][q] == j) { ++q; continue; }
        blk.insert(blk.end(), z0.begin() + j * M0, z0.begin() + (j + 1) * M0);
      }
      kw.push_back((std::int64_t)(blk.size() / M0));
      kblocks.push_back(blk);
    }
    gls_b200::SurModel ks = gls_b200::make_sur(kblocks, kw, M0, y2, om2);
    auto sop = gls_b200::sur_preconditioner(ks);
    gls_b200::PcgConfig scfg;
    scfg.tol_rel = 1e-13;
    gls_b200::AugSolveResult gs = gls_b200::pcg_aug(ks, *sop, gls_b200::Vector(sop->rows(), 0.0),
                                                    gls_b200::Vector(sop->params(), 0.0), scfg);
    double mn = 0.0, md = 0.0;
    std::size_t p = 0;
    for (std::size_t i = 0; i < G2; ++i) {
      std::size_t q = 0;
      for (std::size_t j = 0; j < N0; ++j) {
        if (q < restr[i].size() && (std::size_t)restr[i][q] == j) { ++q; continue; }
        const double d = gm.solution.b[i * N0 + j] - gs.solution.b[p];
        mn += d * d;
        md += gs.solution.b[p] * gs.solution.b[p];
        ++p;
      }
    }
    const double rel_mv = std::sqrt(mn / md);
    const bool ok_mv = rel_mv <= 1e-5 && mop->counters().factorizations == G2;
    std::printf("{\"device\": true, \"iterations\": %zu, \"oracle_iterations\": %lld, \"rel_b\": %.3e, "
                "\"mvrglm_iterations\": %zu, \"mvrglm_vs_sur\": %.3e, \"ok\": %s}\n",
                g.solution.iterations, (long long)orr.iterations, rel, gm.solution.iterations, rel_mv,
                ok && ok_mv ? "true" : "false");
    return ok && ok_mv ? 0 : 1;
  } catch (const gls_b200::DeviceError& e) {
    std::printf("{\"device\": false, \"error\": \"%s\"}\n", e.what());
    return expect_device ? 2 : 0;  // no device: loud failure, never a CPU fallback
  }
}
