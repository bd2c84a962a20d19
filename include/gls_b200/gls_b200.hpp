// gls_b200.hpp -- header-only C++17 host API of the B200 SUR PCG-Aug solver, over the C-ABI (glsgpu.h).
//
// Mirrors the reference's solver surface (/root/reference/proj/include/gls) with the same names,
// argument meaning and error behaviour, in namespace gls_b200 (so it can coexist with gls_core):
//
//   Vector, SurModel, make_sur          structured.hpp:53-65, structured.cpp:97-105
//   PcgConfig, PcgTraceRow, PcgTrace,   pcg.hpp:12-51, glm.hpp:26-37
//   GlsSolution, AugSolveResult, Termination
//   Error + DimensionMismatch, RankDeficient, SingularD, SingularTriangular   errors.hpp:10-88
//   sur_preconditioner(sur[, scale]) -> std::unique_ptr<SurOperator>          structured.hpp:105-108
//   SurOperator::{rows, params, apply_pi, apply_xstar_t, apply_xstar, counters, reset_apply_counters}
//                                       preconditioner.hpp:30-53
//   pcg_aug(sur, op, w1, z1, config[, true_beta])                             pcg.hpp:80-83
//   operator_norm_probe(op[, iters])                                          pcg.hpp:132
//
// The one deliberate difference: pcg_aug takes the SurModel, not embed_sur(sur) -- the dense
// (G M) x n embedding is never formed (the dense-embedding wall).
// Link with -lglsgpu (paper_2510_14471_b200/libglsgpu.so).  There is no CPU fallback.
#ifndef GLS_B200_HPP
#define GLS_B200_HPP

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../glsgpu.h"

namespace gls_b200 {

using Vector = std::vector<double>;

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionMismatch : public Error {
 public:
  using Error::Error;
};
class RankDeficient : public Error {
 public:
  using Error::Error;
};
class SingularD : public Error {
 public:
  using Error::Error;
};
class SingularTriangular : public Error {
 public:
  using Error::Error;
};
// Not in the reference: the device side (CUDA failure, no device, unsupported shape, NCCL).
class SingularCovariance : public Error {
 public:
  using Error::Error;
};
class DeviceError : public Error {
 public:
  using Error::Error;
};

inline void check(int code) {
  if (code == GLSGPU_OK) return;
  const std::string msg = glsgpu_last_error_message();
  switch (code) {
    case GLSGPU_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case GLSGPU_ERR_RANK_DEFICIENT: throw RankDeficient(msg);
    case GLSGPU_ERR_SINGULAR_D: throw SingularD(msg);
    case GLSGPU_ERR_SINGULAR_COVARIANCE: throw SingularCovariance(msg);
    case GLSGPU_ERR_SINGULAR_TRIANGULAR: throw SingularTriangular(msg);
    default: throw DeviceError(msg);
  }
}

enum class Termination { Converged = 0, Breakdown = 1, Stagnation = 2, MaxIter = 3, Direct = 4 };

inline const char* to_string(Termination t) {
  switch (t) {
    case Termination::Converged: return "converged";
    case Termination::Breakdown: return "breakdown";
    case Termination::Stagnation: return "stagnation";
    case Termination::MaxIter: return "max_iter";
    default: return "direct";
  }
}

struct PcgConfig {
  double tol_rel = 1e-10;
  std::size_t max_iter = 0;
  double breakdown_tol = 1e-14;
  std::size_t stagnation_window = 5;
  double growth_tol = 1e4;
  std::size_t growth_window = 10;
  std::size_t record_z_every = 1;
  // device knobs (glsgpu_pcg_config)
  int diag_every = 1;
  int xv_mode = GLSGPU_XV_X;
  int graph_chunk = 0;
  int kron_fma = 0;
  int sw_mode = 0;  // 1: Sigma w formed where read (glsgpu_pcg_config::sw_mode)
  int fused_c = 0;  // 1: Sigma pr inside pass C, element-wise pass A (glsgpu_pcg_config::fused_c)
};

struct PcgTraceRow {
  std::size_t iter = 0;
  double c = 0.0;
  double aug_residual_norm = 0.0;
  double dual_feas_norm = 0.0;
  double rmse = 0.0;
  long long elapsed_ns = 0;
};

struct PcgTrace {
  std::vector<PcgTraceRow> rows;
  Termination termination = Termination::MaxIter;
  bool has_breakdown_iteration = false;
  std::size_t breakdown_iteration = 0;
  bool w1_projected = false;
};

struct GlsSolution {
  Vector b;
  Vector w;
  std::size_t iterations = 0;
  Termination termination = Termination::Direct;
  double residual_seminorm = 0.0;
};

struct AugSolveResult {
  GlsSolution solution;
  PcgTrace trace;
};

struct CostCounters {
  std::size_t factorizations = 0, factor_multiplies = 0, pi_applies = 0, xstar_t_applies = 0, xstar_applies = 0,
              apply_multiplies = 0;
};

// SurModel: blocks X_i (M x n_i column-major), Y (M x G column-major), sigma0 (G x G).
struct SurModel {
  std::size_t M = 0;
  std::vector<std::int64_t> widths;
  Vector X;       // [X_0 | ... | X_{G-1}], M x n column-major
  Vector y;       // M x G
  Vector sigma0;  // G x G
  std::size_t obs() const { return M; }
  std::size_t equations() const { return widths.size(); }
  std::size_t total_params() const {
    std::size_t n = 0;
    for (auto w : widths) n += (std::size_t)w;
    return n;
  }
};

// make_sur (structured.cpp:97-105): blocks are column-major M x n_i vectors with their widths.
inline SurModel make_sur(const std::vector<Vector>& blocks, const std::vector<std::int64_t>& widths, std::size_t M,
                         Vector y, Vector sigma0) {
  if (blocks.empty()) throw DimensionMismatch("make_sur: need at least one block");
  const std::size_t g = blocks.size();
  if (widths.size() != g || y.size() != M * g) throw DimensionMismatch("make_sur: Y/blocks mismatch");
  SurModel s;
  s.M = M;
  s.widths = widths;
  for (std::size_t i = 0; i < g; ++i) {
    if (blocks[i].size() != M * (std::size_t)widths[i]) throw DimensionMismatch("make_sur: block row mismatch");
    s.X.insert(s.X.end(), blocks[i].begin(), blocks[i].end());
  }
  if (sigma0.size() != g * g) throw DimensionMismatch("make_sur: Sigma0 must be G x G");
  s.y = std::move(y);
  s.sigma0 = std::move(sigma0);
  return s;
}

// MvRglm (structured.hpp:33-43): Y = Z0 B + U, restrictions[i] = zero-forced rows of B[:, i].
struct MvRglm {
  std::size_t M0 = 0, N0 = 0;
  Vector z0;      // M0 x N0 column-major
  Vector y;       // M0 x G
  Vector omega0;  // G x G
  std::vector<std::vector<std::int64_t>> restrictions;
  std::size_t obs() const { return M0; }
  std::size_t params_per_eq() const { return N0; }
  std::size_t equations() const { return restrictions.size(); }
  std::size_t total_restrictions() const {
    std::size_t k = 0;
    for (const auto& r : restrictions) k += r.size();
    return k;
  }
};

// make_mvrglm (structured.cpp:63-74): same checks, same messages.
inline MvRglm make_mvrglm(Vector z0, std::size_t M0, std::size_t N0, Vector y, Vector omega0,
                          std::vector<std::vector<std::int64_t>> restrictions) {
  const std::size_t g = restrictions.size();
  if (z0.size() != M0 * N0 || M0 < N0) throw DimensionMismatch("make_mvrglm: Z0 must be tall");
  if (y.size() != M0 * g) throw DimensionMismatch("make_mvrglm: Y/Z0 row mismatch");
  if (omega0.size() != g * g) throw DimensionMismatch("make_mvrglm: Omega0 must be G x G");
  for (const auto& list : restrictions)
    for (std::size_t q = 0; q < list.size(); ++q) {
      if (list[q] < 0 || (std::size_t)list[q] >= N0) throw DimensionMismatch("restrictions: index out of range");
      if (q > 0 && list[q] <= list[q - 1]) throw DimensionMismatch("restrictions: indices must be strictly increasing");
    }
  MvRglm mv;
  mv.M0 = M0;
  mv.N0 = N0;
  mv.z0 = std::move(z0);
  mv.y = std::move(y);
  mv.omega0 = std::move(omega0);
  mv.restrictions = std::move(restrictions);
  return mv;
}

// A block-QR indefinite preconditioner resident on a B200 (BlockQrPreconditioner, structured.cpp:282-363)
// together with its GLM's X and Sigma: the SUR operator (sur_preconditioner) or the MVRGLM one
// (mvrglm_preconditioner).  Host m-vectors use the reference's embedded row order.
class BlockQrOperator {
 public:
  ~BlockQrOperator() {
    if (h_) glsgpu_sur_destroy(h_);
  }
  BlockQrOperator(const BlockQrOperator&) = delete;
  BlockQrOperator& operator=(const BlockQrOperator&) = delete;

  std::size_t rows() const { return m_; }
  std::size_t params() const { return n_; }

  Vector apply_pi(const Vector& xi) const {
    if (xi.size() != m_) throw DimensionMismatch("apply_pi: size mismatch");
    Vector out(m_);
    check(glsgpu_apply_pi(h_, xi.data(), out.data()));
    return out;
  }
  Vector apply_xstar_t(const Vector& xi) const {
    if (xi.size() != m_) throw DimensionMismatch("apply_xstar_t: size mismatch");
    Vector out(n_);
    check(glsgpu_apply_xstar_t(h_, xi.data(), out.data()));
    return out;
  }
  Vector apply_xstar(const Vector& v) const {
    if (v.size() != n_) throw DimensionMismatch("apply_xstar: size mismatch");
    Vector out(m_);
    check(glsgpu_apply_xstar(h_, v.data(), out.data()));
    return out;
  }
  CostCounters counters() const {
    glsgpu_counters_t c;
    check(glsgpu_counters(h_, &c));
    return CostCounters{c.factorizations, c.factor_multiplies, c.pi_applies, c.xstar_t_applies, c.xstar_applies,
                        c.apply_multiplies};
  }
  void reset_apply_counters() const { check(glsgpu_reset_apply_counters(h_)); }
  glsgpu_sur* handle() const { return h_; }

 protected:
  BlockQrOperator() = default;
  void adopt(glsgpu_sur* h) {
    h_ = h;
    std::int64_t m = 0, n = 0;
    check(glsgpu_model_dims(h_, &m, &n));
    m_ = (std::size_t)m;
    n_ = (std::size_t)n;
  }
  glsgpu_sur* h_ = nullptr;
  std::size_t m_ = 0, n_ = 0;
};

// The SUR indefinite preconditioner (SurPreconditioner, structured.cpp:416-453).
class SurOperator : public BlockQrOperator {
 public:
  SurOperator(const SurModel& sur, const Vector* block_scale, int device = 0) {
    if (block_scale && block_scale->size() != sur.equations())
      throw DimensionMismatch("sur_preconditioner: need one scale per block");
    int bad = -1;
    glsgpu_sur* h = nullptr;
    check(glsgpu_sur_create((int)sur.equations(), (std::int64_t)sur.M, sur.widths.data(), sur.X.data(),
                            sur.y.data(), sur.sigma0.data(), block_scale ? block_scale->data() : nullptr, device, &h,
                            &bad));
    adopt(h);
  }
};

// The MVRGLM indefinite preconditioner (MvRglmPreconditioner, structured.cpp:365-414) with the operator
// of embed_mvrglm (structured.cpp:77-95).
class MvRglmOperator : public BlockQrOperator {
 public:
  MvRglmOperator(const MvRglm& mv, const Vector* z_scale, const Vector* c_scale, int device = 0) {
    const std::size_t g = mv.equations();
    if ((z_scale && z_scale->size() != g) || (c_scale && c_scale->size() != g))
      throw DimensionMismatch("mvrglm_preconditioner: need one scale per equation");
    std::vector<std::int64_t> roff(g + 1, 0), ridx;
    for (std::size_t i = 0; i < g; ++i) {
      ridx.insert(ridx.end(), mv.restrictions[i].begin(), mv.restrictions[i].end());
      roff[i + 1] = (std::int64_t)ridx.size();
    }
    if (ridx.empty()) ridx.push_back(0);
    int bad = -1;
    glsgpu_sur* h = nullptr;
    check(glsgpu_mvrglm_create((int)g, (std::int64_t)mv.M0, (std::int64_t)mv.N0, mv.z0.data(), mv.y.data(),
                               mv.omega0.data(), roff.data(), ridx.data(), z_scale ? z_scale->data() : nullptr,
                               c_scale ? c_scale->data() : nullptr, device, &h, &bad));
    adopt(h);
  }
};

inline std::unique_ptr<SurOperator> sur_preconditioner(const SurModel& sur, const Vector& block_scale,
                                                       int device = 0) {
  return std::make_unique<SurOperator>(sur, &block_scale, device);
}
inline std::unique_ptr<SurOperator> sur_preconditioner(const SurModel& sur, int device = 0) {
  return std::make_unique<SurOperator>(sur, nullptr, device);
}
inline std::unique_ptr<MvRglmOperator> mvrglm_preconditioner(const MvRglm& mv, const Vector& z_scale,
                                                             const Vector& c_scale, int device = 0) {
  return std::make_unique<MvRglmOperator>(mv, &z_scale, &c_scale, device);
}
inline std::unique_ptr<MvRglmOperator> mvrglm_preconditioner(const MvRglm& mv, int device = 0) {
  return std::make_unique<MvRglmOperator>(mv, nullptr, nullptr, device);
}

// mv_reduce (structured.cpp:121-130) on the device: Z0 -> R0 (N0 x N0), Y -> Q0'Y.  R0 is the reference's up
// to row signs (TSQR), which the GLS estimate does not see.
inline MvRglm mv_reduce(const MvRglm& mv, int device = 0) {
  MvRglm red;
  red.M0 = red.N0 = mv.N0;
  red.z0.resize(mv.N0 * mv.N0);
  red.y.resize(mv.N0 * mv.equations());
  red.omega0 = mv.omega0;
  red.restrictions = mv.restrictions;
  check(glsgpu_mv_reduce((int)mv.equations(), (std::int64_t)mv.M0, (std::int64_t)mv.N0, mv.z0.data(), mv.y.data(),
                         red.z0.data(), red.y.data(), device));
  return red;
}

// sur_reduce (structured.cpp:132-178, Remark 1) on the device: q = numerical rank of W = [X_1 ... X_G]; every
// block and Y rotated onto an orthonormal basis of range(W) (the reference's up to an orthogonal q x q factor).
inline SurModel sur_reduce(const SurModel& sur, double rank_tol = 1e-10, std::size_t* rank = nullptr,
                           int device = 0) {
  const std::size_t g = sur.equations(), n = sur.total_params(), cap = std::min(sur.M, n);
  Vector xr((cap < sur.M ? cap : sur.M) * n), yr((cap < sur.M ? cap : sur.M) * g);
  std::int64_t q = 0;
  check(glsgpu_sur_reduce((int)g, (std::int64_t)sur.M, sur.widths.data(), sur.X.data(), sur.y.data(), rank_tol,
                          device, &q, xr.data(), yr.data(), nullptr));
  if (rank) *rank = (std::size_t)q;
  SurModel red;
  red.M = (std::size_t)q;
  red.widths = sur.widths;
  red.X.assign(xr.begin(), xr.begin() + (std::size_t)q * n);
  red.y.assign(yr.begin(), yr.begin() + (std::size_t)q * g);
  red.sigma0 = sur.sigma0;
  return red;
}

inline double operator_norm_probe(const BlockQrOperator& op, std::size_t iters = 12) {
  double nrm = 0.0;
  check(glsgpu_operator_norm_probe(op.handle(), (std::int64_t)iters, &nrm));
  return nrm;
}

// pcg_aug (pcg.cpp:346-350 -> run_aug, Recovery variant) on the device, on the operator's GLM.
inline AugSolveResult pcg_aug(const BlockQrOperator& op, const Vector& w1, const Vector& z1, const PcgConfig& config,
                              const Vector* true_beta = nullptr) {
  const std::size_t m = op.rows(), n = op.params();
  if (w1.size() != m || z1.size() != n) throw DimensionMismatch("pcg_aug: bad initial iterate size");
  glsgpu_pcg_config c;
  glsgpu_default_config(&c);
  c.tol_rel = config.tol_rel;
  c.max_iter = (std::int64_t)config.max_iter;
  c.breakdown_tol = config.breakdown_tol;
  c.stagnation_window = (std::int64_t)config.stagnation_window;
  c.growth_tol = config.growth_tol;
  c.growth_window = (std::int64_t)config.growth_window;
  c.record_z_every = (std::int64_t)config.record_z_every;
  c.diag_every = config.diag_every;
  c.xv_mode = config.xv_mode;
  c.graph_chunk = config.graph_chunk;
  c.kron_fma = config.kron_fma;
  c.sw_mode = config.sw_mode;
  c.fused_c = config.fused_c;
  bool w1_zero = true, z1_zero = true;
  for (double v : w1) w1_zero = w1_zero && v == 0.0;
  for (double v : z1) z1_zero = z1_zero && v == 0.0;
  const std::size_t max_iter = config.max_iter ? config.max_iter : m - n + 1;
  std::vector<glsgpu_trace_row> rows(max_iter + 1);
  AugSolveResult out;
  out.solution.b.resize(n);
  out.solution.w.resize(m);
  glsgpu_result r;
  check(glsgpu_sur_solve(op.handle(), &c, w1_zero ? nullptr : w1.data(), z1_zero ? nullptr : z1.data(),
                         true_beta ? true_beta->data() : nullptr, out.solution.b.data(), out.solution.w.data(),
                         rows.data(), (std::int64_t)rows.size(), &r));
  out.solution.iterations = (std::size_t)r.iterations;
  out.solution.termination = (Termination)r.termination;
  out.solution.residual_seminorm = r.residual_seminorm;
  out.trace.termination = (Termination)r.termination;
  out.trace.w1_projected = r.w1_projected != 0;
  out.trace.has_breakdown_iteration = r.breakdown_iteration >= 0;
  out.trace.breakdown_iteration = r.breakdown_iteration >= 0 ? (std::size_t)r.breakdown_iteration : 0;
  const std::size_t k = std::min<std::size_t>((std::size_t)r.n_rows, rows.size());
  out.trace.rows.resize(k);
  for (std::size_t i = 0; i < k; ++i)
    out.trace.rows[i] = PcgTraceRow{(std::size_t)rows[i].iter, rows[i].c, rows[i].aug_residual_norm,
                                    rows[i].dual_feas_norm, rows[i].rmse, (long long)rows[i].elapsed_ns};
  return out;
}

// pcg_normal_equations(embed_sur(sur), nullptr, config, true_beta) (pcg.cpp:364-511) on the device: the PCG-NE
// comparison solver (identity preconditioner) on the operator's SUR model.
inline AugSolveResult pcg_normal_equations(const SurOperator& op, const PcgConfig& config,
                                           const Vector* true_beta = nullptr) {
  const std::size_t m = op.rows(), n = op.params();
  glsgpu_pcg_config c;
  glsgpu_default_config(&c);
  c.tol_rel = config.tol_rel;
  c.max_iter = (std::int64_t)config.max_iter;
  c.breakdown_tol = config.breakdown_tol;
  c.stagnation_window = (std::int64_t)config.stagnation_window;
  c.growth_tol = config.growth_tol;
  c.growth_window = (std::int64_t)config.growth_window;
  c.record_z_every = (std::int64_t)config.record_z_every;
  const std::size_t max_iter = config.max_iter ? config.max_iter : 2 * n;
  std::vector<glsgpu_trace_row> rows(max_iter + 1);
  AugSolveResult out;
  out.solution.b.resize(n);
  out.solution.w.resize(m);
  glsgpu_result r;
  check(glsgpu_pcg_ne(op.handle(), &c, true_beta ? true_beta->data() : nullptr, out.solution.b.data(),
                      out.solution.w.data(), rows.data(), (std::int64_t)rows.size(), &r));
  out.solution.iterations = (std::size_t)r.iterations;
  out.solution.termination = (Termination)r.termination;
  out.solution.residual_seminorm = r.residual_seminorm;
  out.trace.termination = (Termination)r.termination;
  out.trace.has_breakdown_iteration = r.breakdown_iteration >= 0;
  out.trace.breakdown_iteration = r.breakdown_iteration >= 0 ? (std::size_t)r.breakdown_iteration : 0;
  const std::size_t k = std::min<std::size_t>((std::size_t)r.n_rows, rows.size());
  out.trace.rows.resize(k);
  for (std::size_t i = 0; i < k; ++i)
    out.trace.rows[i] = PcgTraceRow{(std::size_t)rows[i].iter, rows[i].c, rows[i].aug_residual_norm,
                                    rows[i].dual_feas_norm, rows[i].rmse, (long long)rows[i].elapsed_ns};
  return out;
}

// pcg_aug(embed_sur(sur), op, ...): the SurModel form of the reference's call.
inline AugSolveResult pcg_aug(const SurModel& sur, const BlockQrOperator& op, const Vector& w1, const Vector& z1,
                              const PcgConfig& config, const Vector* true_beta = nullptr) {
  if (op.rows() != sur.M * sur.equations() || op.params() != sur.total_params())
    throw DimensionMismatch("pcg_aug: preconditioner dims do not match the GLM");
  return pcg_aug(op, w1, z1, config, true_beta);
}

// pcg_aug(embed_mvrglm(mv), op, ...)
inline AugSolveResult pcg_aug(const MvRglm& mv, const BlockQrOperator& op, const Vector& w1, const Vector& z1,
                              const PcgConfig& config, const Vector* true_beta = nullptr) {
  if (op.rows() != mv.M0 * mv.equations() + mv.total_restrictions() || op.params() != mv.N0 * mv.equations())
    throw DimensionMismatch("pcg_aug: preconditioner dims do not match the GLM");
  return pcg_aug(op, w1, z1, config, true_beta);
}

}  // namespace gls_b200

#endif  // GLS_B200_HPP
