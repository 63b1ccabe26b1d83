// feti_gpu.hpp -- header-only C++ adapter over the C-ABI (include/fetigpu.h).
//
// This is the drop-in a maintainer adds next to proj/include/feti: it keeps
// the reference's solver vocabulary (TfetiSystem / FetidpSystem /
// DualOperator::apply, pcg / simultaneous_pcg, recover_primal; SPEC.md:13,
// 346-357, 426-443) and rethrows the reference's exception types
// (proj/include/feti/errors.hpp:7-69).  Build with
// -DFETIGPU_WITH_REFERENCE_ERRORS inside the reference tree to throw
// feti::NotPositiveDefinite & co.; otherwise equivalent types are declared
// in namespace fetigpu.
#pragma once

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "fetigpu.h"

#ifdef FETIGPU_WITH_REFERENCE_ERRORS
#include "feti/errors.hpp"
namespace fetigpu { namespace err = ::feti; }
#else
namespace fetigpu {
namespace err {
#define FETIGPU_ERR(T) struct T : std::runtime_error { using std::runtime_error::runtime_error; };
FETIGPU_ERR(NotPositiveDefinite) FETIGPU_ERR(IndefiniteInput) FETIGPU_ERR(IncompatibleRhs)
FETIGPU_ERR(EdgeNotOnBoundary) FETIGPU_ERR(DimensionMismatch) FETIGPU_ERR(NodeNotFound)
FETIGPU_ERR(InsufficientCorners) FETIGPU_ERR(ZeroStiffnessDiagonal) FETIGPU_ERR(SingularInterior)
FETIGPU_ERR(CoarseSingular) FETIGPU_ERR(SingularRemainder) FETIGPU_ERR(SingularCoarse)
FETIGPU_ERR(SingularGlobal) FETIGPU_ERR(NegativeInnerProduct) FETIGPU_ERR(NotConverged)
FETIGPU_ERR(StateSolveFailed) FETIGPU_ERR(ConfigError) FETIGPU_ERR(IoError)
#undef FETIGPU_ERR
}  // namespace err
}  // namespace fetigpu
#endif

namespace fetigpu {

// Maps a FETIGPU_E_* code to the reference exception type (errors.hpp order).
inline void check(int rc) {
  if (rc == FETIGPU_OK) return;
  const std::string m = fetigpu_last_error();
  switch (rc) {
    case FETIGPU_E_NOT_POSITIVE_DEFINITE: throw err::NotPositiveDefinite(m);
    case FETIGPU_E_INDEFINITE_INPUT: throw err::IndefiniteInput(m);
    case FETIGPU_E_INCOMPATIBLE_RHS: throw err::IncompatibleRhs(m);
    case FETIGPU_E_EDGE_NOT_ON_BOUNDARY: throw err::EdgeNotOnBoundary(m);
    case FETIGPU_E_DIMENSION_MISMATCH: throw err::DimensionMismatch(m);
    case FETIGPU_E_NODE_NOT_FOUND: throw err::NodeNotFound(m);
    case FETIGPU_E_INSUFFICIENT_CORNERS: throw err::InsufficientCorners(m);
    case FETIGPU_E_ZERO_STIFFNESS_DIAGONAL: throw err::ZeroStiffnessDiagonal(m);
    case FETIGPU_E_SINGULAR_INTERIOR: throw err::SingularInterior(m);
    case FETIGPU_E_COARSE_SINGULAR: throw err::CoarseSingular(m);
    case FETIGPU_E_SINGULAR_REMAINDER: throw err::SingularRemainder(m);
    case FETIGPU_E_SINGULAR_COARSE: throw err::SingularCoarse(m);
    case FETIGPU_E_SINGULAR_GLOBAL: throw err::SingularGlobal(m);
    case FETIGPU_E_NEGATIVE_INNER_PRODUCT: throw err::NegativeInnerProduct(m);
    case FETIGPU_E_NOT_CONVERGED: throw err::NotConverged(m);
    case FETIGPU_E_STATE_SOLVE_FAILED: throw err::StateSolveFailed(m);
    case FETIGPU_E_CONFIG: throw err::ConfigError(m);
    case FETIGPU_E_IO: throw err::IoError(m);
    case FETIGPU_E_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case FETIGPU_E_DOMAIN: throw std::domain_error(m);
    default: throw std::runtime_error("fetigpu: " + m);
  }
}

struct SolveOptions {
  double tol = 1e-6;
  bool relative = true;
  int max_iterations = 1000;
  int directions = FETIGPU_SINGLE;
  double pivot_tol = 1e-12;
  int reorth_passes = 2;
};

struct ConvergenceTrace {
  int status = 0;
  int iterations = 0;
  int f_applies = 0;
  std::vector<double> eps_r;
  std::vector<int> kept_dirs;
  std::vector<int> cum_f_applies;
  double solve_ms = 0;
};

// The dual system of either method; `TfetiSystem` / `FetidpSystem` below fix
// the method.  Owns the GPU context; not copyable.
class DualSystem {
 public:
  explicit DualSystem(const fetigpu_problem& p) {
    check(fetigpu_create(&p, &ctx_));
    fetigpu_stats s{};
    check(fetigpu_stats_get(ctx_, &s));
    m_ = s.m;
    n_sub_ = s.n_sub;
    local_dofs_ = s.local_dofs;
  }
  DualSystem(const DualSystem&) = delete;
  DualSystem& operator=(const DualSystem&) = delete;
  ~DualSystem() { fetigpu_destroy(ctx_); }

  void build() { check(fetigpu_build(ctx_)); }
  int dual_size() const { return m_; }

  // DualOperator::apply: y = F x
  std::vector<double> apply(const std::vector<double>& x) const {
    std::vector<double> y(m_);
    check(fetigpu_apply_F(ctx_, x.data(), y.data(), 1, m_));
    return y;
  }
  // apply_coarse_preconditioner
  std::vector<double> precondition(const std::vector<double>& r) const {
    std::vector<double> z(m_);
    check(fetigpu_apply_precond(ctx_, r.data(), z.data(), nullptr));
    return z;
  }
  // CoarseSpace::project (decomposition.hpp:136)
  void project(std::vector<double>& v) const { check(fetigpu_project(ctx_, v.data(), 1, m_)); }
  // pcg / simultaneous_pcg
  std::vector<double> solve(const SolveOptions& o, ConvergenceTrace* tr = nullptr) {
    fetigpu_solve_opts so{o.tol, o.relative ? 1 : 0, o.max_iterations, o.directions, o.pivot_tol,
                          o.reorth_passes};
    std::vector<double> lam(m_);
    const int cap = o.max_iterations + 2;
    std::vector<double> eps(cap);
    std::vector<int> kept(cap), fap(cap);
    fetigpu_trace t{0, 0, 0, 0.0, 0.0, cap, eps.data(), kept.data(), fap.data(), 0.0, {}};
    check(fetigpu_solve(ctx_, &so, lam.data(), &t));
    if (tr) {
      tr->status = t.status;
      tr->iterations = t.iterations;
      tr->f_applies = t.f_applies;
      tr->eps_r.assign(eps.begin(), eps.begin() + t.iterations + 1);
      tr->kept_dirs.assign(kept.begin(), kept.begin() + t.iterations + 1);
      tr->cum_f_applies.assign(fap.begin(), fap.begin() + t.iterations + 1);
      tr->solve_ms = t.solve_ms;
    }
    return lam;
  }
  // pcg / simultaneous_pcg from lambda0 (the SIMP loop's warm start)
  std::vector<double> solve_warm(const SolveOptions& o, const std::vector<double>& lambda0,
                                 ConvergenceTrace* tr = nullptr) {
    fetigpu_solve_opts so{o.tol, o.relative ? 1 : 0, o.max_iterations, o.directions, o.pivot_tol,
                          o.reorth_passes};
    std::vector<double> lam(m_);
    const int cap = o.max_iterations + 2;
    std::vector<double> eps(cap);
    std::vector<int> kept(cap), fap(cap);
    fetigpu_trace t{0, 0, 0, 0.0, 0.0, cap, eps.data(), kept.data(), fap.data(), 0.0, {}};
    check(fetigpu_solve_warm(ctx_, &so, lambda0.data(), lam.data(), &t));
    if (tr) {
      tr->status = t.status;
      tr->iterations = t.iterations;
      tr->f_applies = t.f_applies;
      tr->eps_r.assign(eps.begin(), eps.begin() + t.iterations + 1);
      tr->kept_dirs.assign(kept.begin(), kept.begin() + t.iterations + 1);
      tr->cum_f_applies.assign(fap.begin(), fap.begin() + t.iterations + 1);
      tr->solve_ms = t.solve_ms;
    }
    return lam;
  }
  // next density snapshot of the same problem in place (mbb_modular_snapshot
  // loop): operators rebuilt in the existing device storage
  void rebuild(const fetigpu_problem& p) { check(fetigpu_rebuild(ctx_, &p)); }
  // RRS direction store (FETIGPU_RRS_STORE_AUTO / _EXPLICIT / _IMPLICIT, fetigpu.h);
  // the reference has no counterpart (it always stores W_j, Q_j densely)
  void set_rrs_store(int mode) { check(fetigpu_set_rrs_store(ctx_, mode)); }
  // recover_primal: per-subdomain displacements
  std::vector<std::vector<double>> recover_primal(const std::vector<double>& lambda) const {
    std::vector<double> u((size_t)n_sub_ * local_dofs_);
    check(fetigpu_recover(ctx_, lambda.data(), u.data()));
    std::vector<std::vector<double>> out(n_sub_);
    for (int s = 0; s < n_sub_; ++s)
      out[s].assign(u.begin() + (size_t)s * local_dofs_, u.begin() + (size_t)(s + 1) * local_dofs_);
    return out;
  }
  fetigpu_ctx* handle() const { return ctx_; }

 private:
  fetigpu_ctx* ctx_ = nullptr;
  int m_ = 0, n_sub_ = 0, local_dofs_ = 0;
};

inline fetigpu_problem with_method(fetigpu_problem p, int method) {
  p.method = method;
  return p;
}

// build_tfeti
class TfetiSystem : public DualSystem {
 public:
  explicit TfetiSystem(const fetigpu_problem& p) : DualSystem(with_method(p, FETIGPU_TFETI)) { build(); }
};
// build_fetidp
class FetidpSystem : public DualSystem {
 public:
  explicit FetidpSystem(const fetigpu_problem& p) : DualSystem(with_method(p, FETIGPU_FETIDP)) { build(); }
};

// PivotedCholesky / pivoted_cholesky (linalg.hpp:72-89): same fields, dense
// column-major storage; the factorization and the compression run on the GPU.
struct PivotedCholesky {
  std::vector<int> permutation;  // permutation[k] = original index of pivot k
  std::vector<double> lower;     // dim x rank, column-major, pivot order
  int rank = 0;
  int dim = 0;
  // W N^T [L~^{-T}; 0] for w: rows x dim column-major -> rows x rank
  std::vector<double> compress(const std::vector<double>& w, int rows) const {
    std::vector<double> full((size_t)dim * dim, 0.0);
    std::copy(lower.begin(), lower.end(), full.begin());
    std::vector<double> out((size_t)rows * rank);
    check(fetigpu_pivoted_compress(permutation.data(), full.data(), dim, rank, w.data(), rows, out.data()));
    return out;
  }
};

// a: n x n column-major symmetric PSD
inline PivotedCholesky pivoted_cholesky(const std::vector<double>& a, int n, double pivot_tol = 1e-12) {
  PivotedCholesky pc;
  pc.dim = n;
  pc.permutation.resize(n);
  std::vector<double> full((size_t)n * n);
  check(fetigpu_pivoted_cholesky(a.data(), n, pivot_tol, pc.permutation.data(), full.data(), &pc.rank));
  pc.lower.assign(full.begin(), full.begin() + (size_t)n * pc.rank);
  return pc;
}

}  // namespace fetigpu
