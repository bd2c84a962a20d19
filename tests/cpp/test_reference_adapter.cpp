// test_reference_adapter.cpp -- the drop-in demonstration (built by __graft_entry__.build(), run by
// tests/test_cpp.py on the GPU box).  It links the UNMODIFIED reference gls_core (oracle/_ref) and the
// B200 library, and checks, on seeded SUR problems:
//   A. the reference's own pcg_aug(embed_sur(sur), *sur_preconditioner(sur), ...)          (CPU reference)
//   B. the reference's own pcg_aug(embed_sur(sur), *gls::gpu::sur_preconditioner(sur), ...) (reference loop,
//      B200 operator behind the reference's IndefinitePreconditioner interface)
//   C. gls::gpu::pcg_aug_sur(sur, cfg, ...)                                                  (whole loop on the B200)
// agree: same termination and iteration count, b within 1e-10; B's counters equal A's.
// And the multivariate route of the harness (experiments.cpp:537-557, K2 auxiliary of experiments.cpp:835-847):
//   D. reference mv_reduce + pcg_aug(embed_mvrglm(red), *mvrglm_preconditioner(red, z, c), ...)
//   E. the same reference loop on gls::gpu::mvrglm_preconditioner, F. gls::gpu::pcg_aug_mvrglm,
//   G. gls::gpu::mv_reduce against the reference's (R0 up to row signs).
// MVRGLM stops are last-bit sensitive, so D/E/F agree to 1e-5 with stops within 10.
// Prints one JSON line per case; exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <vector>

#include "gls/experiments.hpp"
#include "gls/pcg.hpp"
#include "gls/rng.hpp"
#include "gls/structured.hpp"
#include "gls_gpu_adapter.hpp"

using namespace gls;

static double rel(const Vector& a, const Vector& b) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num) / std::max(std::sqrt(den), 1e-300);
}

static SurModel make_case(std::size_t g, std::size_t m0, std::size_t nb, std::uint64_t seed) {
  Rng master(seed);
  std::vector<DenseMatrix> blocks;
  for (std::size_t i = 0; i < g; ++i) blocks.push_back(master.split(i).gaussian_matrix(m0, nb + i % 3));
  DenseMatrix y = master.split(100).gaussian_matrix(m0, g);
  DenseMatrix sigma0 = gen_spd_with_cond(g, 8.0, master.split(101).seed());
  return make_sur(std::move(blocks), std::move(y), std::move(sigma0));
}

int main() {
  int fails = 0;
  struct Case {
    std::size_t g, m0, nb;
    std::uint64_t seed;
    double tol;
  } cases[] = {{6, 400, 12, 7, 1e-10}, {10, 1000, 20, 8, 1e-8}, {3, 2000, 30, 9, 1e-10}};
  for (const Case& cs : cases) {
    SurModel sur = make_case(cs.g, cs.m0, cs.nb, cs.seed);
    Glm glm = embed_sur(sur);
    PcgConfig cfg;
    cfg.tol_rel = cs.tol;
    const Vector w1(glm.x.rows(), 0.0), z1(glm.x.cols(), 0.0);
    auto op_ref = sur_preconditioner(sur);
    AugSolveResult a = pcg_aug(glm, *op_ref, w1, z1, cfg);
    auto op_gpu = gpu::sur_preconditioner(sur);
    AugSolveResult b = pcg_aug(glm, *op_gpu, w1, z1, cfg);
    AugSolveResult c = gpu::pcg_aug_sur(sur, cfg, w1, z1);
    const double rb = rel(b.solution.b, a.solution.b), rc = rel(c.solution.b, a.solution.b);
    const auto& ca = op_ref->counters();
    const auto& cb = op_gpu->counters();
    const bool ok_b = b.solution.iterations == a.solution.iterations &&
                      b.solution.termination == a.solution.termination && rb <= 1e-10;
    const bool ok_c = c.solution.iterations == a.solution.iterations &&
                      c.solution.termination == a.solution.termination && rc <= 1e-10 &&
                      c.trace.rows.size() == a.trace.rows.size();
    const bool ok_cnt = ca.pi_applies == cb.pi_applies && ca.xstar_t_applies == cb.xstar_t_applies &&
                        ca.apply_multiplies == cb.apply_multiplies && cb.factorizations == cs.g;
    fails += !ok_b + !ok_c + !ok_cnt;
    std::printf(
        "{\"G\": %zu, \"M\": %zu, \"ref_iters\": %zu, \"ref_term\": \"%s\", \"gpu_op_iters\": %zu, "
        "\"gpu_op_rel_b\": %.3e, \"gpu_solve_iters\": %zu, \"gpu_solve_rel_b\": %.3e, \"counters_equal\": %s, "
        "\"ok\": %s}\n",
        cs.g, cs.m0, a.solution.iterations, to_string(a.solution.termination), b.solution.iterations, rb,
        c.solution.iterations, rc, ok_cnt ? "true" : "false", (ok_b && ok_c && ok_cnt) ? "true" : "false");
  }
  {
    const std::size_t g = 6, m0 = 900, n0 = 12;
    Rng master(21);
    DenseMatrix z0 = master.split(0).gaussian_matrix(m0, n0);
    DenseMatrix y = master.split(1).gaussian_matrix(m0, g);
    DenseMatrix om = gen_spd_with_cond(g, 6.0, master.split(2).seed());
    std::vector<std::vector<std::size_t>> restr(g);
    for (std::size_t i = 0; i < g; ++i)
      for (std::size_t j = 0; j < n0; ++j)
        if ((i + j) % 3 == 0) restr[i].push_back(j);
    MvRglm mv = make_mvrglm(z0, y, om, restr);
    auto [red, rec] = mv_reduce(mv);
    auto [red_g, rec_g] = gpu::mv_reduce(mv);
    double dr = 0.0, nr = 0.0;
    for (std::size_t j = 0; j < n0; ++j) {
      const double sg = (red.z0(j, j) > 0) == (red_g.z0(j, j) > 0) ? 1.0 : -1.0;
      for (std::size_t k = 0; k < n0; ++k) {
        dr += std::pow(red_g.z0(j, k) - sg * red.z0(j, k), 2);
        nr += red.z0(j, k) * red.z0(j, k);
      }
    }
    const double rel_r = std::sqrt(dr / nr);
    const double zf = red.z0.frobenius_norm();
    Vector zs(g), cs(g);
    for (std::size_t i = 0; i < g; ++i) {
      zs[i] = om(i, i);
      cs[i] = zs[i] / (zf * zf / (double)n0);
    }
    Glm glm = embed_mvrglm(red);
    PcgConfig cfg;
    cfg.tol_rel = 1e-12;
    cfg.max_iter = 3 * (red.total_restrictions() + 1) + 10;
    const Vector w1(glm.x.rows(), 0.0), z1(glm.x.cols(), 0.0);
    auto op_ref = mvrglm_preconditioner(red, zs, cs);
    AugSolveResult d = pcg_aug(glm, *op_ref, w1, z1, cfg);
    auto op_gpu = gpu::mvrglm_preconditioner(red, zs, cs);
    AugSolveResult e = pcg_aug(glm, *op_gpu, w1, z1, cfg);
    AugSolveResult f = gpu::pcg_aug_mvrglm(red, cfg, w1, z1, nullptr, &zs, &cs);
    const double re = rel(e.solution.b, d.solution.b), rf = rel(f.solution.b, d.solution.b);
    auto near = [&](const AugSolveResult& x) {
      const long di = (long)x.solution.iterations - (long)d.solution.iterations;
      return di <= 10 && di >= -10;
    };
    const bool ok = rel_r <= 1e-12 && re <= 1e-5 && rf <= 1e-5 && near(e) && near(f) &&
                    op_gpu->counters().factorizations == g;
    fails += !ok;
    std::printf("{\"mvrglm\": true, \"ref_iters\": %zu, \"ref_term\": \"%s\", \"gpu_op_iters\": %zu, "
                "\"gpu_op_rel_b\": %.3e, \"gpu_solve_iters\": %zu, \"gpu_solve_rel_b\": %.3e, "
                "\"mv_reduce_rel_R\": %.3e, \"ok\": %s}\n",
                d.solution.iterations, to_string(d.solution.termination), e.solution.iterations, re,
                f.solution.iterations, rf, rel_r, ok ? "true" : "false");
  }
  {
    // sur_reduce: the reference's vs the device's on a model whose W has rank 5 < n (shared columns)
    Rng master(31);
    DenseMatrix base = master.split(0).gaussian_matrix(300, 5);
    std::vector<DenseMatrix> blocks;
    for (std::size_t i = 0; i < 4; ++i) {
      DenseMatrix b(300, 3);
      for (std::size_t j = 0; j < 3; ++j)
        for (std::size_t r = 0; r < 300; ++r) b(r, j) = base(r, (i + j) % 5);
      blocks.push_back(b);
    }
    SurModel sur = make_sur(blocks, master.split(1).gaussian_matrix(300, 4), gen_spd_with_cond(4, 5.0, 3));
    auto [rr, rrec] = sur_reduce(sur);
    auto [rg, grec] = gpu::sur_reduce(sur);
    double dg = 0.0, ng = 0.0;
    for (std::size_t i = 0; i < 4; ++i)
      for (std::size_t j = 0; j < 4; ++j) {
        const DenseMatrix a = rr.blocks[i].transpose() * rr.blocks[j], b = rg.blocks[i].transpose() * rg.blocks[j];
        dg += (a - b).frobenius_norm() * (a - b).frobenius_norm();
        ng += a.frobenius_norm() * a.frobenius_norm();
      }
    const bool ok = rrec.rank == 5 && grec.rank == 5 && rg.obs() == 5 && std::sqrt(dg / ng) <= 1e-12;
    fails += !ok;
    std::printf("{\"sur_reduce\": true, \"ref_q\": %zu, \"gpu_q\": %zu, \"gram_rel\": %.3e, \"ok\": %s}\n", rrec.rank,
                grec.rank, std::sqrt(dg / ng), ok ? "true" : "false");
  }
  // error mapping: a rank-deficient block raises gls::RankDeficient through the adapter
  {
    SurModel sur = make_case(3, 50, 4, 11);
    for (std::size_t r = 0; r < 50; ++r) sur.blocks[1](r, 1) = sur.blocks[1](r, 0);
    bool thrown = false;
    try {
      gpu::sur_preconditioner(sur);
    } catch (const RankDeficient&) {
      thrown = true;
    }
    fails += !thrown;
    std::printf("{\"rank_deficient_maps_to_gls_RankDeficient\": %s}\n", thrown ? "true" : "false");
  }
  return fails;
}
