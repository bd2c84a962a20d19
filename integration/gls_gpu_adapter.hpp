// gls_gpu_adapter.hpp -- the reference-side binding of the B200 solver (what a gls_core maintainer adds).
//
// Compiled against the reference's OWN headers (/root/reference/proj/include/gls) and linked with
// gls_core and libglsgpu.so.  Two entry points:
//
//  1. gls::gpu::GpuSurPreconditioner : gls::IndefinitePreconditioner
//     A drop-in for sur_preconditioner(sur[, block_scale]) (structured.cpp:479-486): the per-block QR
//     runs on the B200 and pi_impl / xstar_t_impl / xstar_impl (structured.cpp:307-340) are device
//     applies.  The reference's unmodified pcg_aug(embed_sur(sur), *op, ...) runs on it as is.
//
//  2. gls::gpu::pcg_aug_sur(sur, config, w1, z1, true_beta)
//     The whole run_aug loop (pcg.cpp:36-229) on the device, taking the SurModel itself -- the dense
//     embed_sur X (structured.cpp:107-119; 16.8 TB at BASELINE config 4) is never formed.  Returns
//     the reference's own gls::AugSolveResult.
//
//  3. The multivariate model (gls::MvRglm): GpuMvRglmPreconditioner (a drop-in for
//     mvrglm_preconditioner(mv[, z_scale, c_scale]), structured.cpp:365-414,468-477), pcg_aug_mvrglm (the
//     device loop on embed_mvrglm's GLM, structured.cpp:77-95) and mv_reduce (structured.cpp:121-130).
#ifndef GLS_GPU_ADAPTER_HPP
#define GLS_GPU_ADAPTER_HPP

#include <cmath>
#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "gls/errors.hpp"
#include "gls/pcg.hpp"
#include "gls/preconditioner.hpp"
#include "gls/structured.hpp"
#include "glsgpu.h"

namespace gls {
namespace gpu {

// glsgpu status -> the matching gls::Error subclass (errors.hpp:10-88)
inline void check(int code) {
  if (code == GLSGPU_OK) return;
  const std::string msg = glsgpu_last_error_message();
  switch (code) {
    case GLSGPU_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case GLSGPU_ERR_RANK_DEFICIENT: throw RankDeficient(msg);
    case GLSGPU_ERR_SINGULAR_D: throw SingularD(msg);
    case GLSGPU_ERR_SINGULAR_TRIANGULAR: throw SingularTriangular(msg);
    case GLSGPU_ERR_SINGULAR_COVARIANCE: throw SingularCovariance(msg);
    default: throw Error("glsgpu: " + msg);
  }
}

class GpuSur {
 public:
  GpuSur(const SurModel& sur, const Vector* block_scale, int device) {
    const std::size_t g = sur.equations(), m0 = sur.obs();
    std::vector<std::int64_t> widths(g);
    Vector x;
    x.reserve(m0 * sur.total_params());
    for (std::size_t i = 0; i < g; ++i) {
      widths[i] = (std::int64_t)sur.blocks[i].cols();
      x.insert(x.end(), sur.blocks[i].data(), sur.blocks[i].data() + m0 * sur.blocks[i].cols());
    }
    if (block_scale && block_scale->size() != g)
      throw DimensionMismatch("sur_preconditioner: need one scale per block");
    int bad = -1;
    check(glsgpu_sur_create((int)g, (std::int64_t)m0, widths.data(), x.data(), sur.y.data(), sur.sigma0.data(),
                            block_scale ? block_scale->data() : nullptr, device, &h_, &bad));
  }
  GpuSur(const MvRglm& mv, const Vector* z_scale, const Vector* c_scale, int device) {
    const std::size_t g = mv.equations();
    if ((z_scale && z_scale->size() != g) || (c_scale && c_scale->size() != g))
      throw DimensionMismatch("mvrglm_preconditioner: need one scale per equation");
    std::vector<std::int64_t> roff(g + 1, 0), ridx;
    for (std::size_t i = 0; i < g; ++i) {
      for (std::size_t c : mv.restrictions[i]) ridx.push_back((std::int64_t)c);
      roff[i + 1] = (std::int64_t)ridx.size();
    }
    if (ridx.empty()) ridx.push_back(0);
    int bad = -1;
    check(glsgpu_mvrglm_create((int)g, (std::int64_t)mv.obs(), (std::int64_t)mv.params_per_eq(), mv.z0.data(),
                               mv.y.data(), mv.omega0.data(), roff.data(), ridx.data(),
                               z_scale ? z_scale->data() : nullptr, c_scale ? c_scale->data() : nullptr, device, &h_,
                               &bad));
  }
  ~GpuSur() {
    if (h_) glsgpu_sur_destroy(h_);
  }
  GpuSur(const GpuSur&) = delete;
  GpuSur& operator=(const GpuSur&) = delete;
  glsgpu_sur* get() const { return h_; }

 private:
  glsgpu_sur* h_ = nullptr;
};

class GpuSurPreconditioner final : public IndefinitePreconditioner {
 public:
  GpuSurPreconditioner(const SurModel& sur, const Vector& block_scale, int device = 0)
      : dev_(sur, &block_scale, device), m_(sur.obs() * sur.equations()), n_(sur.total_params()) {
    // cost model of BlockQrPreconditioner::finalize (structured.cpp:296-305)
    for (const auto& b : sur.blocks) {
      const std::size_t r = sur.obs(), n = b.cols();
      pi_cost_ += 2 * r * n + 2 * r;
      xstar_t_cost_ += r * n + n * (n + 1) / 2 + r;
      xstar_cost_ += r * n + n * (n + 1) / 2 + r;
    }
    counters_.factorizations = sur.equations();
  }
  std::size_t rows() const override { return m_; }
  std::size_t params() const override { return n_; }
  glsgpu_sur* handle() const { return dev_.get(); }

 protected:
  Vector pi_impl(const Vector& xi) const override {
    Vector out(m_);
    check(glsgpu_apply_pi(dev_.get(), xi.data(), out.data()));
    return out;
  }
  Vector xstar_t_impl(const Vector& xi) const override {
    Vector out(n_);
    check(glsgpu_apply_xstar_t(dev_.get(), xi.data(), out.data()));
    return out;
  }
  Vector xstar_impl(const Vector& v) const override {
    Vector out(m_);
    check(glsgpu_apply_xstar(dev_.get(), v.data(), out.data()));
    return out;
  }
  std::size_t pi_cost() const override { return pi_cost_; }
  std::size_t xstar_t_cost() const override { return xstar_t_cost_; }
  std::size_t xstar_cost() const override { return xstar_cost_; }

 private:
  GpuSur dev_;
  std::size_t m_, n_;
  std::size_t pi_cost_ = 0, xstar_t_cost_ = 0, xstar_cost_ = 0;
};

// MvRglmPreconditioner on the device (structured.cpp:365-414); host vectors in embed_mvrglm's row order.
class GpuMvRglmPreconditioner final : public IndefinitePreconditioner {
 public:
  GpuMvRglmPreconditioner(const MvRglm& mv, const Vector& z_scale, const Vector& c_scale, int device = 0)
      : dev_(mv, &z_scale, &c_scale, device),
        m_(mv.obs() * mv.equations() + mv.total_restrictions()),
        n_(mv.params_per_eq() * mv.equations()) {
    // cost model of BlockQrPreconditioner::finalize (structured.cpp:296-305), rows = M0 + k_i per block
    for (const auto& r : mv.restrictions) {
      const std::size_t rr = mv.obs() + r.size(), n = mv.params_per_eq();
      pi_cost_ += 2 * rr * n + 2 * rr;
      xstar_t_cost_ += rr * n + n * (n + 1) / 2 + rr;
      xstar_cost_ += rr * n + n * (n + 1) / 2 + rr;
    }
    counters_.factorizations = mv.equations();
  }
  std::size_t rows() const override { return m_; }
  std::size_t params() const override { return n_; }
  glsgpu_sur* handle() const { return dev_.get(); }

 protected:
  Vector pi_impl(const Vector& xi) const override {
    Vector out(m_);
    check(glsgpu_apply_pi(dev_.get(), xi.data(), out.data()));
    return out;
  }
  Vector xstar_t_impl(const Vector& xi) const override {
    Vector out(n_);
    check(glsgpu_apply_xstar_t(dev_.get(), xi.data(), out.data()));
    return out;
  }
  Vector xstar_impl(const Vector& v) const override {
    Vector out(m_);
    check(glsgpu_apply_xstar(dev_.get(), v.data(), out.data()));
    return out;
  }
  std::size_t pi_cost() const override { return pi_cost_; }
  std::size_t xstar_t_cost() const override { return xstar_t_cost_; }
  std::size_t xstar_cost() const override { return xstar_cost_; }

 private:
  GpuSur dev_;
  std::size_t m_, n_;
  std::size_t pi_cost_ = 0, xstar_t_cost_ = 0, xstar_cost_ = 0;
};

inline std::unique_ptr<IndefinitePreconditioner> mvrglm_preconditioner(const MvRglm& mv, const Vector& z_scale,
                                                                       const Vector& c_scale, int device = 0) {
  return std::make_unique<GpuMvRglmPreconditioner>(mv, z_scale, c_scale, device);
}
inline std::unique_ptr<IndefinitePreconditioner> mvrglm_preconditioner(const MvRglm& mv, int device = 0) {
  const Vector ones(mv.equations(), 1.0);
  return mvrglm_preconditioner(mv, ones, ones, device);
}

// mv_reduce on the device: the reduced model and its record (transform not materialised: Q0 stays on the
// device; R0 equals the reference's up to row signs).
inline std::pair<MvRglm, ReductionRecord> mv_reduce(const MvRglm& mv, int device = 0) {
  const std::size_t n0 = mv.params_per_eq(), g = mv.equations();
  DenseMatrix r0(n0, n0), qty(n0, g);
  check(glsgpu_mv_reduce((int)g, (std::int64_t)mv.obs(), (std::int64_t)n0, mv.z0.data(), mv.y.data(), r0.data(),
                         qty.data(), device));
  ReductionRecord rec;
  rec.original_rows = mv.obs();
  rec.reduced_rows = n0;
  rec.rank = n0;
  MvRglm red{std::move(r0), std::move(qty), mv.omega0, mv.restrictions};
  return {std::move(red), std::move(rec)};
}

// sur_reduce on the device (structured.cpp:132-178); the record's transform is not materialised (empty).
inline std::pair<SurModel, ReductionRecord> sur_reduce(const SurModel& sur, double rank_tol = 1e-10, int device = 0) {
  const std::size_t g = sur.equations(), m0 = sur.obs();
  std::vector<std::int64_t> widths(g);
  Vector x;
  for (std::size_t i = 0; i < g; ++i) {
    widths[i] = (std::int64_t)sur.blocks[i].cols();
    x.insert(x.end(), sur.blocks[i].data(), sur.blocks[i].data() + m0 * sur.blocks[i].cols());
  }
  const std::size_t n = x.size() / m0, rows = std::min(m0, n) < m0 ? std::min(m0, n) : m0;
  Vector xr(rows * n), yr(rows * g);
  std::int64_t q = 0;
  check(glsgpu_sur_reduce((int)g, (std::int64_t)m0, widths.data(), x.data(), sur.y.data(), rank_tol, device, &q,
                          xr.data(), yr.data(), nullptr));
  ReductionRecord rec;
  rec.original_rows = m0;
  rec.reduced_rows = (std::size_t)q;
  rec.rank = (std::size_t)q;
  if ((std::size_t)q >= m0) return {sur, std::move(rec)};
  SurModel red;
  red.sigma0 = sur.sigma0;
  red.y = DenseMatrix(q, g);
  std::copy(yr.begin(), yr.begin() + q * g, red.y.data());
  std::size_t p = 0;
  for (std::size_t i = 0; i < g; ++i) {
    DenseMatrix b(q, (std::size_t)widths[i]);
    std::copy(xr.begin() + p * q, xr.begin() + (p + widths[i]) * q, b.data());
    red.blocks.push_back(std::move(b));
    p += widths[i];
  }
  return {std::move(red), std::move(rec)};
}

inline std::unique_ptr<IndefinitePreconditioner> sur_preconditioner(const SurModel& sur, const Vector& block_scale,
                                                                    int device = 0) {
  return std::make_unique<GpuSurPreconditioner>(sur, block_scale, device);
}
inline std::unique_ptr<IndefinitePreconditioner> sur_preconditioner(const SurModel& sur, int device = 0) {
  return sur_preconditioner(sur, Vector(sur.equations(), 1.0), device);
}

// run_aug (pcg.cpp:36-229) on a device handle, into the reference's own result type
inline AugSolveResult solve_on_device(const GpuSur& dev, std::size_t m, std::size_t n, const PcgConfig& config,
                                      const Vector& w1, const Vector& z1, const Vector* true_beta, int xv_mode,
                                      int diag_every) {
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
  c.xv_mode = xv_mode;
  c.diag_every = diag_every;
  const std::size_t max_iter = config.max_iter ? config.max_iter : m - n + 1;
  std::vector<glsgpu_trace_row> rows(max_iter + 1);
  AugSolveResult out;
  out.solution.b.resize(n);
  out.solution.w.resize(m);
  glsgpu_result r;
  check(glsgpu_sur_solve(dev.get(), &c, w1.data(), z1.data(), true_beta ? true_beta->data() : nullptr,
                         out.solution.b.data(), out.solution.w.data(), rows.data(), (std::int64_t)rows.size(), &r));
  out.solution.iterations = (std::size_t)r.iterations;
  out.solution.termination = (Termination)r.termination;
  out.solution.residual_seminorm = r.residual_seminorm;
  out.trace.termination = (Termination)r.termination;
  out.trace.w1_projected = r.w1_projected != 0;
  if (r.breakdown_iteration >= 0) out.trace.breakdown_iteration = (std::size_t)r.breakdown_iteration;
  const std::size_t k = std::min<std::size_t>((std::size_t)r.n_rows, rows.size());
  for (std::size_t i = 0; i < k; ++i) {
    PcgTraceRow row;
    row.iter = (std::size_t)rows[i].iter;
    row.c = rows[i].c;
    row.aug_residual_norm = rows[i].aug_residual_norm;
    row.dual_feas_norm = rows[i].dual_feas_norm;
    row.rmse = rows[i].rmse;
    row.elapsed_ns = (long long)rows[i].elapsed_ns;
    out.trace.rows.push_back(row);
  }
  return out;
}

// pcg_aug(embed_sur(sur), *sur_preconditioner(sur[, scale]), w1, z1, config, true_beta) with the whole
// loop on the device; diag_every = 1 keeps every trace column as the reference fills it.
inline AugSolveResult pcg_aug_sur(const SurModel& sur, const PcgConfig& config, const Vector& w1, const Vector& z1,
                                  const Vector* true_beta = nullptr, const Vector* block_scale = nullptr,
                                  int device = 0, int xv_mode = GLSGPU_XV_X, int diag_every = 1) {
  const std::size_t m = sur.obs() * sur.equations(), n = sur.total_params();
  if (w1.size() != m || z1.size() != n) throw DimensionMismatch("pcg_aug: bad initial iterate size");
  GpuSur dev(sur, block_scale, device);
  return solve_on_device(dev, m, n, config, w1, z1, true_beta, xv_mode, diag_every);
}

// pcg_aug(embed_mvrglm(mv), *mvrglm_preconditioner(mv[, z_scale, c_scale]), w1, z1, config, true_beta)
inline AugSolveResult pcg_aug_mvrglm(const MvRglm& mv, const PcgConfig& config, const Vector& w1, const Vector& z1,
                                     const Vector* true_beta = nullptr, const Vector* z_scale = nullptr,
                                     const Vector* c_scale = nullptr, int device = 0, int diag_every = 1) {
  const std::size_t m = mv.obs() * mv.equations() + mv.total_restrictions(), n = mv.params_per_eq() * mv.equations();
  if (w1.size() != m || z1.size() != n) throw DimensionMismatch("pcg_aug: bad initial iterate size");
  GpuSur dev(mv, z_scale, c_scale, device);
  return solve_on_device(dev, m, n, config, w1, z1, true_beta, GLSGPU_XV_X, diag_every);
}

}  // namespace gpu
}  // namespace gls

#endif  // GLS_GPU_ADAPTER_HPP
