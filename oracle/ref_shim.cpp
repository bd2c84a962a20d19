// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library (gls_core), compiled from the sources under
// /root/reference/proj by oracle/Makefile into oracle/_ref/libglsref.so.  It runs the reference's
// own literal hot-path call
//     pcg_aug(embed_sur(sur), *sur_preconditioner(sur[, scale]), w1, z1, cfg)
// (proj/src/pcg.cpp:346-350, proj/src/structured.cpp:107-119,479-486) on flat arrays, so the
// oracle restatement (gls_oracle.c) and the GPU path can be pinned against the reference itself.
// Nothing here is reference source: it only calls the reference's public API.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "gls/errors.hpp"
#include "gls/pcg.hpp"
#include "gls/structured.hpp"

namespace {

struct Config {
  double tol_rel;
  int64_t max_iter;
  double breakdown_tol;
  int64_t stagnation_window;
  double growth_tol;
  int64_t growth_window;
  int64_t record_z_every;
};

struct TraceRow {
  int64_t iter;
  double c;
  double aug_residual_norm;
  double dual_feas_norm;
  double rmse;
  int64_t elapsed_ns;
};

struct Result {
  int64_t iterations;
  int32_t termination;
  int32_t w1_projected;
  int64_t breakdown_iteration;
  double residual_seminorm;
  int64_t n_rows;
  double sigma_scale;
};

int code_of(const gls::Error& e) {
  if (dynamic_cast<const gls::DimensionMismatch*>(&e)) return 1;
  if (dynamic_cast<const gls::RankDeficient*>(&e)) return 2;
  if (dynamic_cast<const gls::SingularD*>(&e)) return 3;
  if (dynamic_cast<const gls::SingularTriangular*>(&e)) return 4;
  return 99;
}

gls::SurModel build_sur(int G, int64_t M, const int64_t* nb, const double* X, const double* Y,
                        const double* omega) {
  std::vector<gls::DenseMatrix> blocks;
  int64_t p = 0;
  for (int b = 0; b < G; ++b) {
    gls::DenseMatrix blk(M, nb[b]);
    std::memcpy(blk.data(), X + p * M, sizeof(double) * M * nb[b]);
    blocks.push_back(std::move(blk));
    p += nb[b];
  }
  gls::DenseMatrix y(M, G);
  if (Y) std::memcpy(y.data(), Y, sizeof(double) * M * G);
  gls::DenseMatrix s0(G, G);
  if (omega) std::memcpy(s0.data(), omega, sizeof(double) * G * G);
  return gls::make_sur(std::move(blocks), std::move(y), std::move(s0));
}

thread_local char g_msg[512];

}  // namespace

extern "C" const char* ref_last_error() { return g_msg; }

namespace {

gls::PcgConfig pcg_config_of(const Config* cfg) {
  gls::PcgConfig pc;
  pc.tol_rel = cfg->tol_rel;
  pc.max_iter = static_cast<std::size_t>(cfg->max_iter);
  pc.breakdown_tol = cfg->breakdown_tol;
  pc.stagnation_window = static_cast<std::size_t>(cfg->stagnation_window);
  pc.growth_tol = cfg->growth_tol;
  pc.growth_window = static_cast<std::size_t>(cfg->growth_window);
  pc.record_z_every = static_cast<std::size_t>(cfg->record_z_every);
  return pc;
}

// pcg_aug(glm, op, w1, z1, cfg, true_beta) and the flat-array result (proj/src/pcg.cpp:346-350)
void run_pcg_aug(const gls::Glm& glm, const gls::IndefinitePreconditioner& op, const double* w1, const double* z1,
                 const Config* cfg, const double* beta_true, double* b_out, double* w_out, TraceRow* rows,
                 int64_t rows_cap, Result* res, uint64_t* counters) {
  const std::size_t m = glm.x.rows(), n = glm.x.cols();
  gls::Vector w(m, 0.0), z(n, 0.0);
  if (w1) w.assign(w1, w1 + m);
  if (z1) z.assign(z1, z1 + n);
  gls::Vector beta;
  if (beta_true) beta.assign(beta_true, beta_true + n);
  gls::AugSolveResult out = gls::pcg_aug(glm, op, w, z, pcg_config_of(cfg), beta_true ? &beta : nullptr);
  std::memcpy(b_out, out.solution.b.data(), sizeof(double) * n);
  if (w_out) std::memcpy(w_out, out.solution.w.data(), sizeof(double) * m);
  res->iterations = static_cast<int64_t>(out.solution.iterations);
  res->termination = static_cast<int32_t>(out.solution.termination);
  res->w1_projected = out.trace.w1_projected ? 1 : 0;
  res->breakdown_iteration =
      out.trace.breakdown_iteration ? static_cast<int64_t>(*out.trace.breakdown_iteration) : -1;
  res->residual_seminorm = out.solution.residual_seminorm;
  res->n_rows = static_cast<int64_t>(out.trace.rows.size());
  res->sigma_scale = gls::operator_norm_probe(glm.sigma);
  if (counters) {
    const gls::CostCounters& cc = op.counters();
    counters[0] = cc.factorizations;
    counters[1] = cc.factor_multiplies;
    counters[2] = cc.pi_applies;
    counters[3] = cc.xstar_t_applies;
    counters[4] = cc.xstar_applies;
    counters[5] = cc.apply_multiplies;
  }
  if (rows) {
    const int64_t k = std::min<int64_t>(rows_cap, res->n_rows);
    for (int64_t i = 0; i < k; ++i) {
      const auto& r = out.trace.rows[i];
      rows[i] = TraceRow{static_cast<int64_t>(r.iter), r.c, r.aug_residual_norm, r.dual_feas_norm, r.rmse,
                         r.elapsed_ns};
    }
  }
}

// make_mvrglm from flat arrays; restrictions as CSR (roff[G + 1], ridx)
gls::MvRglm build_mv(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, const double* omega,
                     const int64_t* roff, const int64_t* ridx) {
  gls::DenseMatrix z0(M0, N0), y(M0, G), s0(G, G);
  std::memcpy(z0.data(), Z0, sizeof(double) * M0 * N0);
  if (Y) std::memcpy(y.data(), Y, sizeof(double) * M0 * G);
  if (omega) std::memcpy(s0.data(), omega, sizeof(double) * G * G);
  std::vector<std::vector<std::size_t>> restr(G);
  for (int i = 0; i < G; ++i)
    for (int64_t q = roff[i]; q < roff[i + 1]; ++q) restr[i].push_back(static_cast<std::size_t>(ridx[q]));
  return gls::make_mvrglm(std::move(z0), std::move(y), std::move(s0), std::move(restr));
}

std::unique_ptr<gls::IndefinitePreconditioner> mv_op(const gls::MvRglm& mv, const double* zs, const double* cs) {
  const int G = static_cast<int>(mv.equations());
  if (zs || cs) {
    gls::Vector z = zs ? gls::Vector(zs, zs + G) : gls::Vector(G, 1.0);
    gls::Vector c = cs ? gls::Vector(cs, cs + G) : gls::Vector(G, 1.0);
    return gls::mvrglm_preconditioner(mv, z, c);
  }
  return gls::mvrglm_preconditioner(mv);
}

}  // namespace

extern "C" {

int ref_pcg_aug_sur(int G, int64_t M, const int64_t* nb, const double* X, const double* Y,
                    const double* omega, const double* scale, const double* w1, const double* z1,
                    const Config* cfg, const double* beta_true, double* b_out, double* w_out,
                    TraceRow* rows, int64_t rows_cap, Result* res, uint64_t* counters) {
  try {
    gls::SurModel sur = build_sur(G, M, nb, X, Y, omega);
    gls::Glm glm = gls::embed_sur(sur);
    std::unique_ptr<gls::IndefinitePreconditioner> op =
        scale ? gls::sur_preconditioner(sur, gls::Vector(scale, scale + G))
              : gls::sur_preconditioner(sur);
    run_pcg_aug(glm, *op, w1, z1, cfg, beta_true, b_out, w_out, rows, rows_cap, res, counters);
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  } catch (const std::exception& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return 98;
  }
}

// pcg_aug(embed_mvrglm(mv), *mvrglm_preconditioner(mv[, z_scale, c_scale]), ...)
// (proj/src/structured.cpp:77-95,365-414,468-477; the harness call experiments.cpp:549-557)
int ref_pcg_aug_mvrglm(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, const double* omega,
                       const int64_t* roff, const int64_t* ridx, const double* z_scale, const double* c_scale,
                       const double* w1, const double* z1, const Config* cfg, const double* beta_true,
                       double* b_out, double* w_out, TraceRow* rows, int64_t rows_cap, Result* res,
                       uint64_t* counters) {
  try {
    gls::MvRglm mv = build_mv(G, M0, N0, Z0, Y, omega, roff, ridx);
    gls::Glm glm = gls::embed_mvrglm(mv);
    auto op = mv_op(mv, z_scale, c_scale);
    run_pcg_aug(glm, *op, w1, z1, cfg, beta_true, b_out, w_out, rows, rows_cap, res, counters);
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  } catch (const std::exception& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return 98;
  }
}

// MvRglmPreconditioner applies; kind as ref_sur_apply (m = G M0 + k, n = G N0)
int ref_mvrglm_apply(int G, int64_t M0, int64_t N0, const double* Z0, const int64_t* roff, const int64_t* ridx,
                     const double* z_scale, const double* c_scale, int kind, const double* in, double* out) {
  try {
    gls::MvRglm mv = build_mv(G, M0, N0, Z0, nullptr, nullptr, roff, ridx);
    auto op = mv_op(mv, z_scale, c_scale);
    gls::Vector r;
    if (kind == 0) r = op->apply_pi(gls::Vector(in, in + op->rows()));
    else if (kind == 1) r = op->apply_xstar_t(gls::Vector(in, in + op->rows()));
    else r = op->apply_xstar(gls::Vector(in, in + op->params()));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  }
}

// mv_reduce (proj/src/structured.cpp:121-130): R0 (N0 x N0) and Q0'Y (N0 x G)
int ref_mv_reduce(int G, int64_t M0, int64_t N0, const double* Z0, const double* Y, double* r_out,
                  double* qty_out) {
  try {
    std::vector<int64_t> roff(G + 1, 0);
    gls::MvRglm mv = build_mv(G, M0, N0, Z0, Y, nullptr, roff.data(), nullptr);
    auto red = gls::mv_reduce(mv);
    std::memcpy(r_out, red.first.z0.data(), sizeof(double) * N0 * N0);
    std::memcpy(qty_out, red.first.y.data(), sizeof(double) * N0 * G);
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  }
}

// kind: 0 = apply_pi, 1 = apply_xstar_t, 2 = apply_xstar  (proj/src/preconditioner.cpp:9-28)
int ref_sur_apply(int G, int64_t M, const int64_t* nb, const double* X, const double* scale, int kind,
                  const double* in, double* out) {
  try {
    gls::SurModel sur = build_sur(G, M, nb, X, nullptr, nullptr);
    auto op = scale ? gls::sur_preconditioner(sur, gls::Vector(scale, scale + G))
                    : gls::sur_preconditioner(sur);
    gls::Vector res;
    if (kind == 0) res = op->apply_pi(gls::Vector(in, in + op->rows()));
    else if (kind == 1) res = op->apply_xstar_t(gls::Vector(in, in + op->rows()));
    else res = op->apply_xstar(gls::Vector(in, in + op->params()));
    std::memcpy(out, res.data(), sizeof(double) * res.size());
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  }
}

// Kronecker apply through SymmetricOperator::kronecker_identity (proj/src/operators.cpp:20-26,45-50)
int ref_kron_apply(int G, int64_t M, const double* omega, const double* x, double* out) {
  try {
    gls::DenseMatrix core(G, G);
    std::memcpy(core.data(), omega, sizeof(double) * G * G);
    auto op = gls::SymmetricOperator::kronecker_identity(core, M);
    gls::Vector r = op.apply(gls::Vector(x, x + M * G));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  }
}

double ref_norm_probe(int G, int64_t M, const double* omega) {
  gls::DenseMatrix core(G, G);
  std::memcpy(core.data(), omega, sizeof(double) * G * G);
  return gls::operator_norm_probe(gls::SymmetricOperator::kronecker_identity(core, M));
}

// Thin QR (proj/src/linalg.cpp:110-117) with the SUR scaling w = 1/sqrt(scale).
int ref_qr_thin(int64_t m, int64_t n, const double* a, double* q, double* r) {
  try {
    gls::DenseMatrix am(m, n);
    std::memcpy(am.data(), a, sizeof(double) * m * n);
    gls::QrThin qr = gls::qr_thin(am);
    std::memcpy(q, qr.q.data(), sizeof(double) * m * n);
    std::memcpy(r, qr.r.data(), sizeof(double) * n * n);
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  }
}

// sur_reduce (proj/src/structured.cpp:132-178): q, the reduced blocks (q x n, concatenated) and Y (q x G),
// and the transform (M x q) when `basis` is non-null.  Outputs are written only when q < M.
int ref_sur_reduce(int G, int64_t M, const int64_t* nb, const double* X, const double* Y, double rank_tol,
                   int64_t* q_out, double* x_out, double* y_out, double* basis) {
  try {
    gls::SurModel sur = build_sur(G, M, nb, X, Y, nullptr);
    sur.sigma0 = gls::DenseMatrix::identity(G);
    auto red = gls::sur_reduce(sur, rank_tol);
    const std::size_t q = red.second.reduced_rows;
    *q_out = static_cast<int64_t>(q);
    int64_t p = 0;
    for (int b = 0; b < G; ++b) {
      std::memcpy(x_out + p * q, red.first.blocks[b].data(), sizeof(double) * q * nb[b]);
      p += nb[b];
    }
    std::memcpy(y_out, red.first.y.data(), sizeof(double) * q * G);
    if (basis) std::memcpy(basis, red.second.transform.data(), sizeof(double) * M * q);
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    return code_of(e);
  }
}

// pcg_normal_equations(embed_sur(sur), nullptr, cfg, true_beta) (proj/src/pcg.cpp:364-511)
int ref_pcg_ne_sur(int G, int64_t M, const int64_t* nb, const double* X, const double* Y, const double* omega,
                   const Config* cfg, const double* beta_true, double* b_out, double* w_out, TraceRow* rows,
                   int64_t rows_cap, Result* res) {
  try {
    gls::SurModel sur = build_sur(G, M, nb, X, Y, omega);
    gls::Glm glm = gls::embed_sur(sur);
    const std::size_t m = glm.x.rows(), n = glm.x.cols();
    gls::Vector beta;
    if (beta_true) beta.assign(beta_true, beta_true + n);
    gls::AugSolveResult out = gls::pcg_normal_equations(glm, nullptr, pcg_config_of(cfg), beta_true ? &beta : nullptr);
    std::memcpy(b_out, out.solution.b.data(), sizeof(double) * n);
    if (w_out) std::memcpy(w_out, out.solution.w.data(), sizeof(double) * m);
    res->iterations = static_cast<int64_t>(out.solution.iterations);
    res->termination = static_cast<int32_t>(out.solution.termination);
    res->w1_projected = 0;
    res->breakdown_iteration =
        out.trace.breakdown_iteration ? static_cast<int64_t>(*out.trace.breakdown_iteration) : -1;
    res->residual_seminorm = out.solution.residual_seminorm;
    res->n_rows = static_cast<int64_t>(out.trace.rows.size());
    res->sigma_scale = 0.0;
    if (rows) {
      const int64_t k = std::min<int64_t>(rows_cap, res->n_rows);
      for (int64_t i = 0; i < k; ++i) {
        const auto& r = out.trace.rows[i];
        rows[i] = TraceRow{static_cast<int64_t>(r.iter), r.c, r.aug_residual_norm, r.dual_feas_norm, r.rmse,
                           r.elapsed_ns};
      }
    }
    return 0;
  } catch (const gls::Error& e) {
    std::snprintf(g_msg, sizeof(g_msg), "%s", e.what());
    if (dynamic_cast<const gls::SingularCovariance*>(&e)) return 5;
    return code_of(e);
  }
}

}  // extern "C"
