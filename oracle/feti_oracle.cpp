// feti_oracle.cpp -- CPU restatement of the reference's FETI hot path.
//
// TEST INFRASTRUCTURE ONLY (see feti_oracle.h).  Plain C++17 + OpenMP, no
// Eigen.  Every function cites the reference file:line it restates.  It is
// deliberately the *implicit* algorithm the reference specifies
// ("never forms S densely", SPEC.md:399 per-subdomain solves per
// apply): sparse (band) Cholesky factors of the reduced K, K_rr, K_oo, with
// triangular solves on every operator / preconditioner application.  That
// makes it both an independent parity checker for the GPU library (which
// forms explicit dense local operators) and the timed CPU baseline.
//
// Deviation from the reference code, on purpose: pivoted_cholesky follows the
// SPEC.md:43-47 contract with a symmetric trailing update; the shipped
// proj/src/linalg.cpp:108-119 updates only the lower triangle after full
// row/column swaps and loses rank on generic inputs.

#include "feti_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace fo {

// ---------------------------------------------------------------- errors --
// proj/include/feti/errors.hpp:7-69, numbered as include/fetigpu.h
enum Code {
  OK = 0, NotPositiveDefinite = 1, IndefiniteInput = 2, IncompatibleRhs = 3,
  EdgeNotOnBoundary = 4, DimensionMismatch = 5, NodeNotFound = 6,
  InsufficientCorners = 7, ZeroStiffnessDiagonal = 8, SingularInterior = 9,
  CoarseSingular = 10, SingularRemainder = 11, SingularCoarse = 12,
  SingularGlobal = 13, NegativeInnerProduct = 14, NotConverged = 15,
  StateSolveFailed = 16, ConfigError = 17, IoError = 18,
  InvalidArgument = 20, DomainError = 21
};
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] static void fail(int c, const std::string& m) { throw Error(c, m); }

// ------------------------------------------------------------ dense / csr --
static double dot_(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

struct Mat {  // column-major
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r_, int c_) : r(r_), c(c_), a((size_t)r_ * c_, 0.0) {}
  double& operator()(int i, int j) { return a[(size_t)j * r + i]; }
  double operator()(int i, int j) const { return a[(size_t)j * r + i]; }
  double* col(int j) { return a.data() + (size_t)j * r; }
  const double* col(int j) const { return a.data() + (size_t)j * r; }
};

struct Csr {  // both triangles stored (linalg.hpp:17-44)
  int n = 0;
  std::vector<int> ptr, idx;
  std::vector<double> val;
  int find(int i, int j) const {
    auto b = idx.begin() + ptr[i], e = idx.begin() + ptr[i + 1];
    auto it = std::lower_bound(b, e, j);
    return (it != e && *it == j) ? int(it - idx.begin()) : -1;
  }
  double get(int i, int j) const {
    int k = find(i, j);
    return k < 0 ? 0.0 : val[k];
  }
  void matvec(const double* x, double* y) const {
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = ptr[i]; k < ptr[i + 1]; ++k) s += val[k] * x[idx[k]];
      y[i] = s;
    }
  }
};

// Band Cholesky on an index subset kept in its natural (ascending) order.
// Restates SparseCholesky (linalg.hpp:46-68, linalg.cpp:64-81); Eigen's AMD
// ordering only changes rounding, not the factorized operator.
struct BandChol {
  int n = 0, kd = 0;
  std::vector<double> L;  // L[j*(kd+1) + (i-j)], i in [j, j+kd]
  double& at(int i, int j) { return L[(size_t)j * (kd + 1) + (i - j)]; }
  double at(int i, int j) const { return L[(size_t)j * (kd + 1) + (i - j)]; }

  void factor(const Csr& A, const std::vector<int>& sub, int errcode,
              const char* what) {
    n = (int)sub.size();
    std::vector<int> map(A.n, -1);
    for (int i = 0; i < n; ++i) map[sub[i]] = i;
    kd = 0;
    for (int i = 0; i < n; ++i) {
      int gi = sub[i];
      for (int k = A.ptr[gi]; k < A.ptr[gi + 1]; ++k) {
        int j = map[A.idx[k]];
        if (j >= 0 && j < i) kd = std::max(kd, i - j);
      }
    }
    L.assign((size_t)n * (kd + 1), 0.0);
    for (int i = 0; i < n; ++i) {
      int gi = sub[i];
      for (int k = A.ptr[gi]; k < A.ptr[gi + 1]; ++k) {
        int j = map[A.idx[k]];
        if (j >= 0 && j <= i) at(i, j) = A.val[k];
      }
    }
    for (int j = 0; j < n; ++j) {
      double d = at(j, j);
      if (!(d > 0.0))
        fail(errcode, std::string(what) + ": matrix is not SPD (pivot " +
                          std::to_string(d) + " at " + std::to_string(j) + ")");
      double l = std::sqrt(d);
      at(j, j) = l;
      int last = std::min(n - 1, j + kd);
      double* cj = &L[(size_t)j * (kd + 1)];
      for (int i = j + 1; i <= last; ++i) cj[i - j] /= l;
      for (int k = j + 1; k <= last; ++k) {
        double lkj = cj[k - j];
        if (lkj == 0.0) continue;
        double* ck = &L[(size_t)k * (kd + 1)];
        for (int i = k; i <= last; ++i) ck[i - k] -= cj[i - j] * lkj;
      }
    }
  }
  void solve(double* x) const {
    for (int j = 0; j < n; ++j) {
      const double* cj = &L[(size_t)j * (kd + 1)];
      double v = x[j] / cj[0];
      x[j] = v;
      int last = std::min(n - 1, j + kd);
      for (int i = j + 1; i <= last; ++i) x[i] -= cj[i - j] * v;
    }
    for (int j = n - 1; j >= 0; --j) {
      const double* cj = &L[(size_t)j * (kd + 1)];
      int last = std::min(n - 1, j + kd);
      double s = x[j];
      for (int i = j + 1; i <= last; ++i) s -= cj[i - j] * x[i];
      x[j] = s / cj[0];
    }
  }
};

// Accuracy reference mode (tests only): x = A_sub^{-1} b with two steps of
// iterative refinement on long-double residuals.  Not part of the reference
// algorithm; used to measure how far the double-precision oracle and the GPU
// each are from the exact local solves at high stiffness contrast.
static bool g_refine = false;
static void solve_sub(const BandChol& bc, const Csr& A, const std::vector<int>& sub, double* x,
                      bool refine) {
  if (!refine) { bc.solve(x); return; }
  const int n = (int)sub.size();
  std::vector<long double> b(x, x + n), xl(n);
  std::vector<int> map(A.n, -1);
  for (int i = 0; i < n; ++i) map[sub[i]] = i;
  bc.solve(x);
  for (int i = 0; i < n; ++i) xl[i] = x[i];
  std::vector<double> r(n);
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = 0; i < n; ++i) {
      long double acc = b[i];
      const int gi = sub[i];
      for (int k = A.ptr[gi]; k < A.ptr[gi + 1]; ++k) {
        const int j = map[A.idx[k]];
        if (j >= 0) acc -= (long double)A.val[k] * xl[j];
      }
      r[i] = (double)acc;
    }
    bc.solve(r.data());
    for (int i = 0; i < n; ++i) xl[i] += r[i];
  }
  for (int i = 0; i < n; ++i) x[i] = (double)xl[i];
}

// Dense Cholesky (Eigen::LLT in decomposition.hpp:131 and the FETI-DP coarse
// factorization SPEC.md:396).
struct DenseChol {
  int n = 0;
  std::vector<double> L;  // row-major lower triangle: L[i*n + k]
  bool factor(const Mat& A) {
    n = A.r;
    L.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k <= i; ++k) L[(size_t)i * n + k] = A(i, k);
    for (int j = 0; j < n; ++j) {
      double* lj = &L[(size_t)j * n];
      double d = lj[j];
      for (int k = 0; k < j; ++k) d -= lj[k] * lj[k];
      if (!(d > 0.0)) return false;
      const double l = std::sqrt(d);
      lj[j] = l;
#pragma omp parallel for schedule(static) if (n - j > 256)
      for (int i = j + 1; i < n; ++i) {
        double* li = &L[(size_t)i * n];
        double s = li[j];
        for (int k = 0; k < j; ++k) s -= li[k] * lj[k];
        li[j] = s / l;
      }
    }
    return true;
  }
  void solve(double* x) const {
    for (int j = 0; j < n; ++j) {
      const double* lj = &L[(size_t)j * n];
      double s = x[j];
      for (int k = 0; k < j; ++k) s -= lj[k] * x[k];
      x[j] = s / lj[j];
    }
    for (int j = n - 1; j >= 0; --j) {
      const double v = x[j] / L[(size_t)j * n + j];
      x[j] = v;
      const double* lj = &L[(size_t)j * n];
      for (int k = 0; k < j; ++k) x[k] -= lj[k] * v;
    }
  }
};

// --------------------------------------------------- rank-revealing chol --
// pivoted_cholesky (linalg.hpp:70-89, linalg.cpp:83-129) per the SPEC.md:43-47
// contract: largest remaining diagonal (ties -> lowest index), stop when the
// pivot drops to tol * max initial diagonal, IndefiniteInput if a remaining
// diagonal is below -tol*scale at that point.  Symmetric trailing update.
struct PivChol {
  std::vector<int> perm;
  Mat lower;  // n x rank
  int rank = 0, dim = 0;
};
static PivChol pivoted_cholesky(Mat a, double tol) {
  const int n = a.r;
  PivChol out;
  out.dim = n;
  out.perm.resize(n);
  std::iota(out.perm.begin(), out.perm.end(), 0);
  double scale = 0.0;
  for (int i = 0; i < n; ++i) scale = std::max(scale, a(i, i));
  const double stop_tol = tol * scale;
  const double neg_tol = -tol * std::max(scale, 1e-300);
  int rank = 0;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int j = k + 1; j < n; ++j)
      if (a(j, j) > a(piv, piv)) piv = j;
    const double d = a(piv, piv);
    if (d <= stop_tol) {
      for (int j = k; j < n; ++j)
        if (a(j, j) < neg_tol)
          fail(IndefiniteInput,
               "pivoted Cholesky: negative pivot " + std::to_string(a(j, j)));
      break;
    }
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(a(k, j), a(piv, j));
      for (int i = 0; i < n; ++i) std::swap(a(i, k), a(i, piv));
      std::swap(out.perm[k], out.perm[piv]);
    }
    const double l = std::sqrt(d);
    a(k, k) = l;
    for (int i = k + 1; i < n; ++i) a(i, k) /= l;
    for (int j = k + 1; j < n; ++j) {
      const double ajk = a(j, k);
      for (int i = k + 1; i < n; ++i) a(i, j) -= a(i, k) * ajk;
    }
    rank = k + 1;
  }
  out.rank = rank;
  out.lower = Mat(n, rank);
  for (int j = 0; j < rank; ++j)
    for (int i = j; i < n; ++i) out.lower(i, j) = a(i, j);
  return out;
}
// PivotedCholesky::compress (linalg.cpp:131-138): W[:, perm[:rank]] Ltilde^{-T}
static Mat compress(const PivChol& pc, const Mat& w) {
  Mat out(w.r, pc.rank);
  // row-wise forward substitution; rows are independent (parallel, same
  // per-row arithmetic as the sequential loop)
  Mat Lt(pc.rank, pc.rank);  // Lt(j, k) = lower(k, j): contiguous rows of L~
  for (int k = 0; k < pc.rank; ++k)
    for (int j = 0; j <= k; ++j) Lt(j, k) = pc.lower(k, j);
#pragma omp parallel
  {
    std::vector<double> row(pc.rank);
#pragma omp for schedule(static)
    for (int i = 0; i < w.r; ++i) {
      for (int k = 0; k < pc.rank; ++k) {
        double s = w(i, pc.perm[k]);
        const double* lk = Lt.col(k);
        for (int j = 0; j < k; ++j) s -= lk[j] * row[j];
        row[k] = s / lk[k];
      }
      for (int k = 0; k < pc.rank; ++k) out(i, k) = row[k];
    }
  }
  return out;
}

// -------------------------------------------------------------------- fem --
struct Material {
  double E0 = 1.0, Emin = 1e-9, nu = 0.3, p = 3.0, thickness = 1.0;
};
// Material::validate (fem.cpp:9-17)
static void validate(const Material& m) {
  if (!(m.Emin > 0.0) || !(m.Emin < m.E0))
    fail(InvalidArgument, "material: need 0 < Emin < E0");
  if (!(m.nu >= 0.0) || !(m.nu < 0.5))
    fail(InvalidArgument, "material: need 0 <= nu < 0.5");
  if (!(m.p >= 1.0)) fail(InvalidArgument, "material: need p >= 1");
  if (!(m.thickness > 0.0)) fail(InvalidArgument, "material: need thickness > 0");
}
// simp_modulus (fem.cpp:19-24)
static double simp_modulus(double rho, const Material& m) {
  if (!(rho >= 0.0) || !(rho <= 1.0))
    fail(DomainError, "simp_modulus: rho = " + std::to_string(rho) + " outside [0, 1]");
  return m.Emin + std::pow(rho, m.p) * (m.E0 - m.Emin);
}
// q4_element_stiffness (fem.cpp:44-84): unit plane-stress D, 2x2 Gauss in the
// order (-,-),(+,-),(+,+),(-,+), k += B^T D B detJ, *thickness, upper->lower.
static void q4_unit(const Material& m, double hx, double hy, double* k /*8x8 cm*/) {
  const double nu = m.nu;
  const double c = 1.0 / (1.0 - nu * nu);
  const double D[3][3] = {{c, c * nu, 0.0}, {c * nu, c, 0.0}, {0.0, 0.0, c * (1.0 - nu) / 2.0}};
  const double g = 1.0 / std::sqrt(3.0);
  const double xi[4] = {-1.0, 1.0, 1.0, -1.0};
  const double eta[4] = {-1.0, -1.0, 1.0, 1.0};
  for (int i = 0; i < 64; ++i) k[i] = 0.0;
  const double det_j = hx * hy / 4.0;
  for (int gp = 0; gp < 4; ++gp) {
    const double s = g * xi[gp], t = g * eta[gp];
    double b[3][8] = {};
    for (int a = 0; a < 4; ++a) {
      const double dn_ds = 0.25 * xi[a] * (1.0 + eta[a] * t);
      const double dn_dt = 0.25 * eta[a] * (1.0 + xi[a] * s);
      const double dn_dx = dn_ds * 2.0 / hx;
      const double dn_dy = dn_dt * 2.0 / hy;
      b[0][2 * a] = dn_dx;
      b[1][2 * a + 1] = dn_dy;
      b[2][2 * a] = dn_dy;
      b[2][2 * a + 1] = dn_dx;
    }
    double bd[8][3];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 3; ++j)
        bd[i][j] = b[0][i] * D[0][j] + b[1][i] * D[1][j] + b[2][i] * D[2][j];
    for (int j = 0; j < 8; ++j)
      for (int i = 0; i < 8; ++i)
        k[j * 8 + i] += (bd[i][0] * b[0][j] + bd[i][1] * b[1][j] + bd[i][2] * b[2][j]) * det_j;
  }
  for (int i = 0; i < 64; ++i) k[i] *= m.thickness;
  for (int i = 0; i < 8; ++i)
    for (int j = i + 1; j < 8; ++j) k[i * 8 + j] = k[j * 8 + i];  // k(j,i) = k(i,j)
}

// assemble_subdomain (fem.cpp:86-119): element loop ey-major, ex-minor,
// contributions e_mod * k_unit(i,j) summed in insertion order (Eigen
// setFromTriplets collapses duplicates in insertion order).
static Csr assemble(int n, double /*hx*/, double /*hy*/, const double* rho, const Material& mat,
                    const double* k_unit) {  // element size is already in k_unit
  const int nn = n + 1, ndof = 2 * nn * nn;
  Csr K;
  K.n = ndof;
  K.ptr.assign(ndof + 1, 0);
  // structured pattern: node couples with its <= 3x3 node neighbourhood
  for (int iy = 0; iy < nn; ++iy)
    for (int ix = 0; ix < nn; ++ix) {
      int cnt = 0;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int jx = ix + dx, jy = iy + dy;
          if (jx >= 0 && jx < nn && jy >= 0 && jy < nn) ++cnt;
        }
      int node = iy * nn + ix;
      K.ptr[2 * node + 1] = 2 * cnt;
      K.ptr[2 * node + 2] = 2 * cnt;
    }
  for (int i = 0; i < ndof; ++i) K.ptr[i + 1] += K.ptr[i];
  K.idx.resize(K.ptr[ndof]);
  K.val.assign(K.ptr[ndof], 0.0);
  for (int iy = 0; iy < nn; ++iy)
    for (int ix = 0; ix < nn; ++ix) {
      std::vector<int> cols;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int jx = ix + dx, jy = iy + dy;
          if (jx >= 0 && jx < nn && jy >= 0 && jy < nn) {
            cols.push_back(2 * (jy * nn + jx));
            cols.push_back(2 * (jy * nn + jx) + 1);
          }
        }
      std::sort(cols.begin(), cols.end());
      int node = iy * nn + ix;
      for (int d = 0; d < 2; ++d)
        std::copy(cols.begin(), cols.end(), K.idx.begin() + K.ptr[2 * node + d]);
    }
  for (int ey = 0; ey < n; ++ey)
    for (int ex = 0; ex < n; ++ex) {
      const double e_mod = simp_modulus(rho[ey * n + ex], mat);
      const int n0 = ey * nn + ex;
      const int nodes[4] = {n0, n0 + 1, n0 + nn + 1, n0 + nn};
      int dofs[8];
      for (int a = 0; a < 4; ++a) {
        dofs[2 * a] = 2 * nodes[a];
        dofs[2 * a + 1] = 2 * nodes[a] + 1;
      }
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) K.val[K.find(dofs[i], dofs[j])] += e_mod * k_unit[j * 8 + i];
    }
  return K;
}

// rigid_body_modes (decomposition.hpp:119-121)
static Mat rigid_body_modes(int n, double hx, double hy) {
  const int nn = n + 1;
  Mat R(2 * nn * nn, 3);
  const double xc = n * hx / 2.0, yc = n * hy / 2.0;
  for (int node = 0; node < nn * nn; ++node) {
    const double x = (node % nn) * hx, y = (node / nn) * hy;
    R(2 * node, 0) = 1.0;
    R(2 * node + 1, 1) = 1.0;
    R(2 * node, 2) = -(y - yc);
    R(2 * node + 1, 2) = x - xc;
  }
  return R;
}

// select_fixing_dofs (linalg.cpp:146-175): greedy max residual row norm,
// strict '>' so the lowest index wins ties, result sorted.
static std::vector<int> select_fixing_dofs(const Mat& basis) {
  const int n = basis.r, w = basis.c;
  std::vector<int> fixed;
  std::vector<std::vector<double>> ortho;
  for (int pick = 0; pick < w; ++pick) {
    int best = -1;
    double best_score = -1.0;
    std::vector<double> r(w);
    for (int d = 0; d < n; ++d) {
      for (int k = 0; k < w; ++k) r[k] = basis(d, k);
      for (auto& o : ortho) {
        double dot = 0.0;
        for (int k = 0; k < w; ++k) dot += o[k] * basis(d, k);
        for (int k = 0; k < w; ++k) r[k] -= o[k] * dot;
      }
      double sc = 0.0;
      for (int k = 0; k < w; ++k) sc += r[k] * r[k];
      sc = std::sqrt(sc);
      if (sc > best_score) {
        best_score = sc;
        best = d;
      }
    }
    if (best < 0 || best_score <= 0.0) fail(IndefiniteInput, "nullspace basis is rank deficient");
    fixed.push_back(best);
    for (int k = 0; k < w; ++k) r[k] = basis(best, k);
    for (auto& o : ortho) {
      double dot = 0.0;
      for (int k = 0; k < w; ++k) dot += o[k] * basis(best, k);
      for (int k = 0; k < w; ++k) r[k] -= o[k] * dot;
    }
    double nr = 0.0;
    for (int k = 0; k < w; ++k) nr += r[k] * r[k];
    nr = std::sqrt(nr);
    for (int k = 0; k < w; ++k) r[k] /= nr;
    ortho.push_back(r);
  }
  std::sort(fixed.begin(), fixed.end());
  return fixed;
}

// ---------------------------------------------------------- decomposition --
struct Row {  // ConstraintRow (decomposition.hpp:58-70)
  int kind;   // 0 interface pair, 1 dirichlet
  int sp, dp, sm = -1, dm = -1;
  double gap = 0.0;
  int mult = 1;
  int gnode = -1, dir = 0;
};
struct BEntry {
  int row, dof;
  double sign;
};

struct Sub {
  int id = 0, si = 0, sj = 0, design = 0;
  Csr K;
  std::vector<double> f, diag;
  std::vector<BEntry> ent;      // B^s entries {row, local dof, sign}
  std::vector<int> T;           // touched local dofs (ascending)
  std::vector<int> tpos;        // local dof -> index in T or -1
  std::vector<double> wt;       // scaled-jump weight per entry (same order as ent)
  // T-FETI semidefinite factor (linalg.cpp:179-222)
  std::vector<int> keep, fixed;
  BandChol kred;
  // preconditioner
  std::vector<int> other;       // o = domain \ T  (Dirichlet Schur)
  BandChol koo;
  // FETI-DP split
  std::vector<int> rd, cd, Dd;  // local dofs in r, c (ascending), D
  std::vector<int> cg;          // global primal index per c dof
  std::vector<double> gD;       // prescribed values at Dd
  BandChol krr;
  std::vector<int> rpos;        // local dof -> index in rd or -1
  Mat Phi;                      // K_rr^{-1} K_rc  (|r| x |c|)
  Mat Kccb;                     // local Kbar_cc
  std::vector<double> fr, fc;   // reduced loads
};

struct Oracle {
  fo_problem P{};
  Material mat;
  int Ns = 0, nloc = 0, GX = 0, GY = 0, m = 0, n_iface = 0, Nc = 0;
  std::vector<Sub> subs;
  std::vector<Row> rows;
  std::vector<double> wplus, wminus;
  Mat R;
  double k_unit[64];
  std::vector<std::vector<double>> densities;
  std::vector<char> prescribed;     // per global dof
  std::vector<double> presc_val;
  // T-FETI coarse space (decomposition.hpp:123-145)
  Mat Gt;                           // G^T, m x 3Ns (G dense as declared at :126)
  std::vector<double> e;
  std::vector<int> kept;
  Mat Gkt;                          // G_kept^T, m x kept
  std::vector<double> ek;
  DenseChol ggt;
  // FETI-DP coarse
  Mat Kcc;
  DenseChol kcc;

  int sub_id(int si, int sj) const { return sj * P.sx + si; }
  int gnode(int gx, int gy) const { return gy * GX + gx; }
  // Partition::owners_of_node (decomposition.hpp:37-42), ascending sub order
  void owners(int gx, int gy, std::vector<std::pair<int, int>>& out) const {
    out.clear();
    const int n = P.n;
    for (int sj = 0; sj < P.sy; ++sj)
      for (int si = 0; si < P.sx; ++si) {
        int lx = gx - si * n, ly = gy - sj * n;
        if (lx >= 0 && lx <= n && ly >= 0 && ly <= n)
          out.push_back({sub_id(si, sj), ly * (n + 1) + lx});
      }
  }
  bool is_corner_node(int gx, int gy) const { return gx % P.n == 0 && gy % P.n == 0; }

  bool refine = false;
  void coarse_solve(double* x) const {
    if (!refine) { kcc.solve(x); return; }
    std::vector<long double> b(x, x + Nc), xl(Nc);
    std::vector<double> r(Nc);
    kcc.solve(x);
    for (int i = 0; i < Nc; ++i) xl[i] = x[i];
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = 0; i < Nc; ++i) {
        long double acc = b[i];
        for (int j = 0; j < Nc; ++j) acc -= (long double)Kcc(i, j) * xl[j];
        r[i] = (double)acc;
      }
      kcc.solve(r.data());
      for (int i = 0; i < Nc; ++i) xl[i] += r[i];
    }
    for (int i = 0; i < Nc; ++i) x[i] = (double)xl[i];
  }
  void build();
  void build_constraints();
  void build_weights();
  void build_tfeti();
  void build_fetidp();
  void build_precond();

  // operators
  void apply_F(const double* x, double* y);
  void apply_precond(const double* r, double* z, double* Zcols);
  void project(double* v) const;
  void rhs(double* d, double* lam0);
  void recover(const double* lambda, double* u);
  int solve(const fo_opts& o, double* lambda, fo_trace* tr);
  void direct(double* u);
};

void Oracle::build() {
  mat.E0 = P.E0; mat.Emin = P.Emin; mat.nu = P.nu; mat.p = P.p; mat.thickness = P.thickness;
  validate(mat);
  if (P.sx < 1 || P.sy < 1 || P.n < 1) fail(DimensionMismatch, "bad partition");
  if (P.method != 0 && P.method != 1) fail(ConfigError, "unknown method");
  if (P.scaling != 0 && P.scaling != 1) fail(ConfigError, "unknown scaling");
  if (P.precond < 0 || P.precond > 2) fail(ConfigError, "unknown preconditioner");
  Ns = P.sx * P.sy;
  const int n = P.n, nn = n + 1;
  nloc = 2 * nn * nn;
  GX = P.sx * n + 1;
  GY = P.sy * n + 1;
  if (P.n_designs < 1) fail(DimensionMismatch, "need >= 1 design");
  densities.resize(P.n_designs);
  for (int d = 0; d < P.n_designs; ++d) {
    densities[d].assign(P.densities + (size_t)d * n * n, P.densities + (size_t)(d + 1) * n * n);
    for (double v : densities[d])  // DensityField::validate (fem.cpp:38-42)
      if (!(v >= 0.0) || !(v <= 1.0)) fail(DomainError, "density outside [0, 1]");
  }
  q4_unit(mat, P.hx, P.hy, k_unit);
  R = rigid_body_modes(n, P.hx, P.hy);
  subs.resize(Ns);
  for (int s = 0; s < Ns; ++s) {
    int dsg = P.module_type[s];
    if (dsg < 0 || dsg >= P.n_designs) fail(DimensionMismatch, "module_type out of range");
  }
#pragma omp parallel for schedule(dynamic)
  for (int s = 0; s < Ns; ++s) {
    Sub& S = subs[s];
    S.id = s; S.si = s % P.sx; S.sj = s / P.sx; S.design = P.module_type[s];
    S.K = assemble(n, P.hx, P.hy, densities[S.design].data(), mat, k_unit);
    S.f.assign(nloc, 0.0);
    S.diag.resize(nloc);
    for (int i = 0; i < nloc; ++i) S.diag[i] = S.K.get(i, i);
  }
  // loads: apply_traction (fem.cpp:121-167)
  for (int t = 0; t < P.n_tractions; ++t) {
    int s = P.tr_sub[t], side = P.tr_side[t], first = P.tr_first[t], count = P.tr_count[t];
    if (s < 0 || s >= Ns) fail(DimensionMismatch, "traction subdomain out of range");
    int node0, stride;
    double h;
    switch (side) {
      case 2: node0 = 0; stride = 1; h = P.hx; break;                   // bottom
      case 3: node0 = n * nn; stride = 1; h = P.hx; break;              // top
      case 0: node0 = 0; stride = nn; h = P.hy; break;                  // left
      case 1: node0 = n; stride = nn; h = P.hy; break;                  // right
      default: fail(EdgeNotOnBoundary, "bad side");
    }
    if (first < 0 || count < 0 || first + count > n)
      fail(EdgeNotOnBoundary, "traction chain [" + std::to_string(first) + ", " +
                                  std::to_string(first + count) + ") leaves the boundary");
    const double half = h / 2.0, tx = P.tr_txy[2 * t], ty = P.tr_txy[2 * t + 1];
    auto& f = subs[s].f;
    for (int e2 = first; e2 < first + count; ++e2) {
      int n0 = node0 + e2 * stride, n1 = n0 + stride;
      f[2 * n0] += half * tx;
      f[2 * n0 + 1] += half * ty;
      f[2 * n1] += half * tx;
      f[2 * n1 + 1] += half * ty;
    }
  }
  std::vector<std::pair<int, int>> own;
  for (int k = 0; k < P.n_point_loads; ++k) {  // lowest-index owner copy
    int g = P.pl_gnode[k], dir = P.pl_dir[k];
    if (g < 0 || g >= GX * GY || dir < 0 || dir > 1) fail(NodeNotFound, "point load node not found");
    owners(g % GX, g / GX, own);
    subs[own[0].first].f[2 * own[0].second + dir] += P.pl_value[k];
  }
  prescribed.assign(2 * GX * GY, 0);
  presc_val.assign(2 * GX * GY, 0.0);
  for (int k = 0; k < P.n_dirichlet; ++k) {
    int g = P.dir_gnode[k], dir = P.dir_dir[k];
    if (g < 0 || g >= GX * GY || dir < 0 || dir > 1) fail(NodeNotFound, "Dirichlet node not found");
    prescribed[2 * g + dir] = 1;
    presc_val[2 * g + dir] = P.dir_value[k];
  }
  build_constraints();
  build_weights();
  if (P.method == 0) build_tfeti(); else build_fetidp();
  build_precond();
}

// build_constraints (decomposition.hpp:110-117): pairwise
// rows for every shared DOF (all m(m-1)/2 pairs, plus = lower sub index),
// interface rows first (node-major, x then y), then Dirichlet rows (one per
// owning copy).  FETI-DP: corner DOFs are primal and prescribed DOFs are
// eliminated, so neither produces rows.
void Oracle::build_constraints() {
  rows.clear();
  std::vector<std::pair<int, int>> own;
  const bool dp = P.method == 1;
  for (int gy = 0; gy < GY; ++gy)
    for (int gx = 0; gx < GX; ++gx) {
      owners(gx, gy, own);
      if (own.size() < 2) continue;
      if (dp && is_corner_node(gx, gy)) continue;
      int g = gnode(gx, gy);
      for (int dir = 0; dir < 2; ++dir) {
        if (prescribed[2 * g + dir]) continue;
        for (size_t a = 0; a < own.size(); ++a)
          for (size_t b = a + 1; b < own.size(); ++b) {
            Row r;
            r.kind = 0;
            r.sp = own[a].first; r.dp = 2 * own[a].second + dir;
            r.sm = own[b].first; r.dm = 2 * own[b].second + dir;
            r.mult = (int)own.size();
            r.gnode = g; r.dir = dir;
            rows.push_back(r);
          }
      }
    }
  n_iface = (int)rows.size();
  if (!dp) {
    for (int g = 0; g < GX * GY; ++g)
      for (int dir = 0; dir < 2; ++dir) {
        if (!prescribed[2 * g + dir]) continue;
        owners(g % GX, g / GX, own);
        for (auto& o : own) {
          Row r;
          r.kind = 1;
          r.sp = o.first; r.dp = 2 * o.second + dir;
          r.gap = presc_val[2 * g + dir];
          r.mult = (int)own.size();
          r.gnode = g; r.dir = dir;
          rows.push_back(r);
        }
      }
  }
  m = (int)rows.size();
  for (auto& S : subs) { S.ent.clear(); }
  for (int i = 0; i < m; ++i) {
    subs[rows[i].sp].ent.push_back({i, rows[i].dp, 1.0});
    if (rows[i].kind == 0) subs[rows[i].sm].ent.push_back({i, rows[i].dm, -1.0});
  }
  for (auto& S : subs) {
    S.tpos.assign(nloc, -1);
    S.T.clear();
    for (auto& e2 : S.ent) S.tpos[e2.dof] = 0;
    for (int i = 0; i < nloc; ++i)
      if (S.tpos[i] == 0) { S.tpos[i] = (int)S.T.size(); S.T.push_back(i); }
  }
}

// multiplicity_scaling / k_scaling (decomposition.hpp:159-180, SPEC.md:234-251,
// PAPER.md:277-283): 1/m; k: opposite owner's diagonal over the sum of all
// owners' diagonals; Dirichlet rows 1.
void Oracle::build_weights() {
  wplus.assign(m, 1.0);
  wminus.assign(m, 0.0);
  std::vector<std::pair<int, int>> own;
  for (int i = 0; i < m; ++i) {
    const Row& r = rows[i];
    if (r.kind == 1) { wplus[i] = 1.0; wminus[i] = 0.0; continue; }
    if (P.scaling == 0) {
      wplus[i] = 1.0 / r.mult;
      wminus[i] = 1.0 / r.mult;
    } else {
      owners(r.gnode % GX, r.gnode / GX, own);
      double den = 0.0;
      for (auto& o : own) {
        double dg = subs[o.first].diag[2 * o.second + r.dir];
        if (!(dg > 0.0)) fail(ZeroStiffnessDiagonal, "nonpositive stiffness diagonal");
        den += dg;
      }
      double kp = subs[r.sp].diag[r.dp], km = subs[r.sm].diag[r.dm];
      wplus[i] = km / den;
      wminus[i] = kp / den;
    }
  }
  for (auto& S : subs) {
    S.wt.resize(S.ent.size());
    for (size_t k = 0; k < S.ent.size(); ++k) {
      int i = S.ent[k].row;
      S.wt[k] = (rows[i].sp == S.id && rows[i].dp == S.ent[k].dof && S.ent[k].sign > 0) ? wplus[i] : wminus[i];
    }
  }
}

// T-FETI: SemidefiniteCholesky per subdomain (linalg.cpp:179-189; identical
// meshes share R, decomposition.hpp:132-134) and the coarse space G, e
// (decomposition.hpp:123-148) filtered by the rank-revealing Cholesky of GG^T
// at 1e-10.
void Oracle::build_tfeti() {
  std::vector<int> fixed = select_fixing_dofs(R);
#pragma omp parallel for schedule(dynamic)
  for (int s = 0; s < Ns; ++s) {
    Sub& S = subs[s];
    S.fixed = fixed;
    S.keep.clear();
    for (int d = 0, f = 0; d < nloc; ++d) {
      if (f < 3 && fixed[f] == d) { ++f; continue; }
      S.keep.push_back(d);
    }
    S.kred.factor(S.K, S.keep, NotPositiveDefinite, "sparse Cholesky");
  }
  const int nc = 3 * Ns;
  Gt = Mat(m, nc);
  e.assign(nc, 0.0);
  for (auto& S : subs) {
    for (auto& en : S.ent)
      for (int k = 0; k < 3; ++k) Gt(en.row, 3 * S.id + k) -= en.sign * R(en.dof, k);
    for (int k = 0; k < 3; ++k) {
      double s = 0.0;
      for (int d = 0; d < nloc; ++d) s += R(d, k) * S.f[d];
      e[3 * S.id + k] = -s;
    }
  }
  Mat GGt(nc, nc);
#pragma omp parallel for schedule(dynamic)
  for (int a = 0; a < nc; ++a)
    for (int b = 0; b <= a; ++b) {
      double s = 0.0;
      const double* ga = Gt.col(a);
      const double* gb = Gt.col(b);
      for (int i = 0; i < m; ++i) s += ga[i] * gb[i];
      GGt(a, b) = s;
      GGt(b, a) = s;
    }
  PivChol pc = pivoted_cholesky(GGt, 1e-10);
  kept.assign(pc.perm.begin(), pc.perm.begin() + pc.rank);
  std::sort(kept.begin(), kept.end());
  const int nk = (int)kept.size();
  Gkt = Mat(m, nk);
  ek.resize(nk);
  for (int a = 0; a < nk; ++a) {
    for (int i = 0; i < m; ++i) Gkt(i, a) = Gt(i, kept[a]);
    ek[a] = e[kept[a]];
  }
  Mat Gg(nk, nk);
  for (int a = 0; a < nk; ++a)
    for (int b = 0; b < nk; ++b) Gg(a, b) = GGt(kept[a], kept[b]);
  if (!ggt.factor(Gg)) fail(CoarseSingular, "filtered G G^T is not SPD");
}

// FETI-DP: prescribed DOFs
// eliminated before the c/r split, corners primal, Kbar_cc assembled in
// subdomain order and factorized densely.
void Oracle::build_fetidp() {
  // primal numbering: corner nodes ascending, x then y, prescribed skipped
  std::vector<int> cidx(2 * GX * GY, -1);
  Nc = 0;
  for (int gy = 0; gy < GY; gy += P.n)
    for (int gx = 0; gx < GX; gx += P.n) {
      int g = gnode(gx, gy);
      for (int dir = 0; dir < 2; ++dir)
        if (!prescribed[2 * g + dir]) cidx[2 * g + dir] = Nc++;
    }
  const int n = P.n, nn = n + 1;
#pragma omp parallel for schedule(dynamic)
  for (int s = 0; s < Ns; ++s) {
    Sub& S = subs[s];
    S.rd.clear(); S.cd.clear(); S.Dd.clear(); S.cg.clear(); S.gD.clear();
    S.rpos.assign(nloc, -1);
    for (int d = 0; d < nloc; ++d) {
      int node = d / 2, dir = d % 2;
      int gx = S.si * n + node % nn, gy = S.sj * n + node / nn;
      int g = gnode(gx, gy);
      if (prescribed[2 * g + dir]) { S.Dd.push_back(d); S.gD.push_back(presc_val[2 * g + dir]); }
      else if (is_corner_node(gx, gy)) { S.cd.push_back(d); S.cg.push_back(cidx[2 * g + dir]); }
      else { S.rpos[d] = (int)S.rd.size(); S.rd.push_back(d); }
    }
    if (S.cd.empty() && S.Dd.empty())
      fail(InsufficientCorners, "subdomain has no primal or prescribed DOF");
    S.krr.factor(S.K, S.rd, SingularRemainder, "K_rr Cholesky");
    const int nr = (int)S.rd.size(), nc = (int)S.cd.size();
    S.Phi = Mat(nr, nc);
    for (int j = 0; j < nc; ++j) {
      double* col = S.Phi.col(j);
      for (int i = 0; i < nr; ++i) col[i] = S.K.get(S.rd[i], S.cd[j]);
      solve_sub(S.krr, S.K, S.rd, col, refine);
    }
    S.Kccb = Mat(nc, nc);
    for (int a = 0; a < nc; ++a)
      for (int b = 0; b < nc; ++b) {
        double v = S.K.get(S.cd[a], S.cd[b]);
        for (int i = 0; i < nr; ++i) v -= S.K.get(S.cd[a], S.rd[i]) * S.Phi(i, b);
        S.Kccb(a, b) = v;
      }
    // reduced loads with prescribed values moved to the right-hand side
    S.fr.resize(nr);
    S.fc.resize(nc);
    for (int i = 0; i < nr; ++i) {
      double v = S.f[S.rd[i]];
      for (size_t k = 0; k < S.Dd.size(); ++k) v -= S.K.get(S.rd[i], S.Dd[k]) * S.gD[k];
      S.fr[i] = v;
    }
    for (int a = 0; a < nc; ++a) {
      double v = S.f[S.cd[a]];
      for (size_t k = 0; k < S.Dd.size(); ++k) v -= S.K.get(S.cd[a], S.Dd[k]) * S.gD[k];
      S.fc[a] = v;
    }
  }
  Kcc = Mat(Nc, Nc);
  for (auto& S : subs)
    for (size_t a = 0; a < S.cd.size(); ++a)
      for (size_t b = 0; b < S.cd.size(); ++b) Kcc(S.cg[a], S.cg[b]) += S.Kccb(a, b);
  if (Nc > 0 && !kcc.factor(Kcc)) fail(SingularCoarse, "Kbar_cc is not SPD");
}

// Preconditioners: b = T (DOFs touched by
// B^s), i = the rest of the domain (T-FETI) or of r (FETI-DP).
void Oracle::build_precond() {
  if (P.precond != 1) return;
#pragma omp parallel for schedule(dynamic)
  for (int s = 0; s < Ns; ++s) {
    Sub& S = subs[s];
    S.other.clear();
    for (int d = 0; d < nloc; ++d) {
      if (S.tpos[d] >= 0) continue;
      if (P.method == 1 && S.rpos[d] < 0) continue;
      S.other.push_back(d);
    }
    if (!S.other.empty()) S.koo.factor(S.K, S.other, SingularInterior, "K_ii Cholesky");
  }
}

// T-FETI: F = sum_s B_s K_s^+ B_s^T with
// K^+ = solve_unchecked (linalg.cpp:206-213).  FETI-DP: condensed
// F_rr + F_rc Kbar_cc^{-1} F_rc^T.  Per-subdomain work runs
// concurrently, the reduction is in fixed subdomain order.
void Oracle::apply_F(const double* x, double* y) {
  std::vector<std::vector<double>> loc(Ns);
  if (P.method == 0) {
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      std::vector<double> b(S.keep.size(), 0.0), full(nloc, 0.0);
      for (auto& en : S.ent) full[en.dof] += en.sign * x[en.row];
      for (size_t i = 0; i < S.keep.size(); ++i) b[i] = full[S.keep[i]];
      solve_sub(S.kred, S.K, S.keep, b.data(), refine);
      std::fill(full.begin(), full.end(), 0.0);
      for (size_t i = 0; i < S.keep.size(); ++i) full[S.keep[i]] = b[i];
      loc[s].resize(S.ent.size());
      for (size_t k = 0; k < S.ent.size(); ++k) loc[s][k] = S.ent[k].sign * full[S.ent[k].dof];
    }
  } else {
    std::vector<std::vector<double>> ys(Ns), ts(Ns);
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      const int nr = (int)S.rd.size(), nc = (int)S.cd.size();
      std::vector<double> xr(nr, 0.0);
      for (auto& en : S.ent) xr[S.rpos[en.dof]] += en.sign * x[en.row];
      ts[s].assign(nc, 0.0);
      for (int a = 0; a < nc; ++a) {
        double v = 0.0;
        for (int i = 0; i < nr; ++i) v += S.Phi(i, a) * xr[i];
        ts[s][a] = v;
      }
      solve_sub(S.krr, S.K, S.rd, xr.data(), refine);
      ys[s] = std::move(xr);
    }
    std::vector<double> u(Nc, 0.0);
    for (int s = 0; s < Ns; ++s)
      for (size_t a = 0; a < subs[s].cd.size(); ++a) u[subs[s].cg[a]] += ts[s][a];
    if (Nc > 0) coarse_solve(u.data());
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      const int nr = (int)S.rd.size(), nc = (int)S.cd.size();
      std::vector<double>& v = ys[s];
      for (int a = 0; a < nc; ++a) {
        const double uc = u[S.cg[a]];
        for (int i = 0; i < nr; ++i) v[i] += S.Phi(i, a) * uc;
      }
      loc[s].resize(S.ent.size());
      for (size_t k = 0; k < S.ent.size(); ++k) loc[s][k] = S.ent[k].sign * v[S.rpos[S.ent[k].dof]];
    }
  }
  std::fill(y, y + m, 0.0);
  for (int s = 0; s < Ns; ++s)
    for (size_t k = 0; k < subs[s].ent.size(); ++k) y[subs[s].ent[k].row] += loc[s][k];
}

// z = sum_s Btilde_s Stilde_s Btilde_s^T r, Btilde = W B.
// Zcols (m x Ns column-major), when given, receives the per-subdomain columns
// of Alg. 1 line 2; z = Z 1 summed in subdomain order.
void Oracle::apply_precond(const double* r, double* z, double* Zcols) {
  std::vector<std::vector<double>> loc(Ns);
#pragma omp parallel for schedule(dynamic)
  for (int s = 0; s < Ns; ++s) {
    Sub& S = subs[s];
    std::vector<double> full(nloc, 0.0), y(nloc, 0.0);
    for (size_t k = 0; k < S.ent.size(); ++k) full[S.ent[k].dof] += S.wt[k] * S.ent[k].sign * r[S.ent[k].row];
    if (P.precond == 2) {  // super-lumped: diag K_bb
      for (int d : S.T) y[d] = S.diag[d] * full[d];
    } else {
      std::vector<double> kx(nloc);
      S.K.matvec(full.data(), kx.data());
      for (int d : S.T) y[d] = kx[d];
      if (P.precond == 1 && !S.other.empty()) {  // Dirichlet: - K_bi K_ii^{-1} K_ib
        std::vector<double> t(S.other.size());
        for (size_t i = 0; i < S.other.size(); ++i) t[i] = kx[S.other[i]];
        solve_sub(S.koo, S.K, S.other, t.data(), refine);
        std::vector<double> ext(nloc, 0.0), kt(nloc);
        for (size_t i = 0; i < S.other.size(); ++i) ext[S.other[i]] = t[i];
        S.K.matvec(ext.data(), kt.data());
        for (int d : S.T) y[d] -= kt[d];
      }
    }
    loc[s].resize(S.ent.size());
    for (size_t k = 0; k < S.ent.size(); ++k) loc[s][k] = S.wt[k] * S.ent[k].sign * y[S.ent[k].dof];
  }
  std::fill(z, z + m, 0.0);
  if (Zcols) std::fill(Zcols, Zcols + (size_t)m * Ns, 0.0);
  for (int s = 0; s < Ns; ++s)
    for (size_t k = 0; k < subs[s].ent.size(); ++k) {
      z[subs[s].ent[k].row] += loc[s][k];
      if (Zcols) Zcols[(size_t)s * m + subs[s].ent[k].row] += loc[s][k];
    }
}

// CoarseSpace::project (decomposition.hpp:136-137): v - G^T (G G^T)^{-1} G v
void Oracle::project(double* v) const {
  if (P.method != 0) return;  // identity projector for FETI-DP
  const int nk = (int)kept.size();
  std::vector<double> g(nk, 0.0);
  for (int a = 0; a < nk; ++a) g[a] = dot_(Gkt.col(a), v, m);
  ggt.solve(g.data());
  for (int a = 0; a < nk; ++a) {
    const double* ga = Gkt.col(a);
    const double ga_ = g[a];
    for (int i = 0; i < m; ++i) v[i] -= ga[i] * ga_;
  }
}

// d = B K^+ f - c and lambda0 = G^T (G G^T)^{-1} e (T-FETI, PAPER.md:107,
// SPEC.md:465); d = d_r - F_rc Kbar^{-1} fbar_c, lambda0 = 0 (FETI-DP).
void Oracle::rhs(double* d, double* lam0) {
  std::fill(d, d + m, 0.0);
  std::fill(lam0, lam0 + m, 0.0);
  if (P.method == 0) {
    std::vector<std::vector<double>> loc(Ns);
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      std::vector<double> b(S.keep.size()), full(nloc, 0.0);
      for (size_t i = 0; i < S.keep.size(); ++i) b[i] = S.f[S.keep[i]];
      solve_sub(S.kred, S.K, S.keep, b.data(), refine);
      for (size_t i = 0; i < S.keep.size(); ++i) full[S.keep[i]] = b[i];
      loc[s].resize(S.ent.size());
      for (size_t k = 0; k < S.ent.size(); ++k) loc[s][k] = S.ent[k].sign * full[S.ent[k].dof];
    }
    for (int s = 0; s < Ns; ++s)
      for (size_t k = 0; k < subs[s].ent.size(); ++k) d[subs[s].ent[k].row] += loc[s][k];
    for (int i = 0; i < m; ++i) d[i] -= rows[i].gap;
    std::vector<double> g(ek);
    ggt.solve(g.data());
    for (size_t a = 0; a < kept.size(); ++a)
      for (int i = 0; i < m; ++i) lam0[i] += Gkt(i, (int)a) * g[a];
  } else {
    std::vector<double> fbar(Nc, 0.0);
    std::vector<std::vector<double>> ys(Ns);
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      ys[s] = S.fr;
      solve_sub(S.krr, S.K, S.rd, ys[s].data(), refine);
    }
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      for (auto& en : S.ent) d[en.row] += en.sign * ys[s][S.rpos[en.dof]];
      for (size_t a = 0; a < S.cd.size(); ++a) {
        double v = S.fc[a];
        for (size_t i = 0; i < S.rd.size(); ++i) v -= S.Phi(i, a) * S.fr[i];
        fbar[S.cg[a]] += v;
      }
    }
    if (Nc > 0) coarse_solve(fbar.data());
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      std::vector<double> v(S.rd.size(), 0.0);
      for (size_t a = 0; a < S.cd.size(); ++a)
        for (size_t i = 0; i < S.rd.size(); ++i) v[i] += S.Phi(i, a) * fbar[S.cg[a]];
      for (auto& en : S.ent) d[en.row] -= en.sign * v[S.rpos[en.dof]];
    }
  }
}

// recover_primal
void Oracle::recover(const double* lambda, double* u) {
  if (P.method == 0) {
    std::vector<double> Fl(m), d(m), l0(m);
    apply_F(lambda, Fl.data());
    rhs(d.data(), l0.data());
    std::vector<double> rho(m);
    for (int i = 0; i < m; ++i) rho[i] = d[i] - Fl[i];
    // alpha_for (decomposition.hpp:143-144): least squares |G^T alpha - rho|
    const int nk = (int)kept.size();
    std::vector<double> ak(nk, 0.0), alpha(3 * Ns, 0.0);
    for (int a = 0; a < nk; ++a) ak[a] = dot_(Gkt.col(a), rho.data(), m);
    ggt.solve(ak.data());
    for (int a = 0; a < nk; ++a) alpha[kept[a]] = ak[a];
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      std::vector<double> full(S.f), b(S.keep.size());
      for (auto& en : S.ent) full[en.dof] -= en.sign * lambda[en.row];
      for (size_t i = 0; i < S.keep.size(); ++i) b[i] = full[S.keep[i]];
      solve_sub(S.kred, S.K, S.keep, b.data(), refine);
      double* us = u + (size_t)s * nloc;
      for (int i = 0; i < nloc; ++i) us[i] = 0.0;
      for (size_t i = 0; i < S.keep.size(); ++i) us[S.keep[i]] = b[i];
      for (int i = 0; i < nloc; ++i)
        us[i] += R(i, 0) * alpha[3 * s] + R(i, 1) * alpha[3 * s + 1] + R(i, 2) * alpha[3 * s + 2];
    }
  } else {
    std::vector<double> t(Nc, 0.0);
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      std::vector<double> xr(S.rd.size(), 0.0);
      for (auto& en : S.ent) xr[S.rpos[en.dof]] += en.sign * lambda[en.row];
      for (size_t a = 0; a < S.cd.size(); ++a) {
        double v = S.fc[a];
        for (size_t i = 0; i < S.rd.size(); ++i) v += S.Phi(i, a) * (xr[i] - S.fr[i]);
        t[S.cg[a]] += v;
      }
    }
    if (Nc > 0) coarse_solve(t.data());  // u_c = Kbar^{-1} (fbar_c + F_rc^T lambda)
#pragma omp parallel for schedule(dynamic)
    for (int s = 0; s < Ns; ++s) {
      Sub& S = subs[s];
      const int nr = (int)S.rd.size();
      std::vector<double> v(S.fr);
      for (auto& en : S.ent) v[S.rpos[en.dof]] -= en.sign * lambda[en.row];
      solve_sub(S.krr, S.K, S.rd, v.data(), refine);
      for (size_t a = 0; a < S.cd.size(); ++a)
        for (int i = 0; i < nr; ++i) v[i] -= S.Phi(i, a) * t[S.cg[a]];
      double* us = u + (size_t)s * nloc;
      for (int i = 0; i < nr; ++i) us[S.rd[i]] = v[i];
      for (size_t a = 0; a < S.cd.size(); ++a) us[S.cd[a]] = t[S.cg[a]];
      for (size_t k = 0; k < S.Dd.size(); ++k) us[S.Dd[k]] = S.gD[k];
    }
  }
}

// ----------------------------------------------------------------- engine --
static double dot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
// residual_metric
static double residual_metric(const double* r, const double* z, int n) {
  double rz = dot(r, z, n);
  double nr = std::sqrt(dot(r, r, n)), nz = std::sqrt(dot(z, z, n));
  if (rz < -1e-14 * nr * nz) fail(NegativeInnerProduct, "r^T z = " + std::to_string(rz));
  return std::sqrt(std::max(rz, 0.0));
}

struct TraceRec {
  fo_trace* tr;
  int n = 0;
  void push(double eps, int kept, int fapp) {
    if (tr && n < tr->cap) {
      if (tr->eps) tr->eps[n] = eps;
      if (tr->kept) tr->kept[n] = kept;
      if (tr->f_app) tr->f_app[n] = fapp;
    }
    ++n;
  }
};

// pcg (single / FO) and simultaneous_pcg (RRS, Alg. 1 of
// PAPER.md:302-351).  FO keeps the F-normalized directions
// (w/sqrt(w^T F w), F w/sqrt(.)) and re-orthogonalizes with the same number of
// passes as RRS, so RRS with one subdomain reproduces FO.
// invariant check: max |W^T F W - I| over the stored
// F-normalised directions of the last FO / RRS solve (fo_set_check)
static bool g_check = false;
static double g_check_err = -1.0;
static int g_check_n = 0;
static void check_orth(const std::vector<const double*>& W, const std::vector<const double*>& Q, int m) {
  const int K = (int)W.size();
  double e = 0.0;
#pragma omp parallel for schedule(dynamic) reduction(max : e)
  for (int a = 0; a < K; ++a)
    for (int b = 0; b < K; ++b) {
      long double acc = 0.0L;   // accurate inner products: the check adds no cancellation of its own
      for (int i = 0; i < m; ++i) acc += (long double)W[a][i] * (long double)Q[b][i];
      e = std::max(e, std::fabs((double)acc - (a == b ? 1.0 : 0.0)));
    }
  g_check_err = e;
  g_check_n = K;
}

int Oracle::solve(const fo_opts& o, double* lambda, fo_trace* tr) {
  TraceRec rec{tr};
  std::vector<double> d(m), lam0(m), r(m), tmp(m), z(m);
  rhs(d.data(), lam0.data());
  std::copy(lam0.begin(), lam0.end(), lambda);
  apply_F(lambda, tmp.data());
  int fapp = 1;
  for (int i = 0; i < m; ++i) r[i] = d[i] - tmp[i];
  project(r.data());
  int status = 1, it = 0;
  double eps0 = 0, eps = 0;
  const int passes = std::max(1, o.reorth_passes);
  if (o.directions < 2) {
    apply_precond(r.data(), z.data(), nullptr);
    project(z.data());
    eps0 = eps = residual_metric(r.data(), z.data(), m);
    rec.push(eps, 1, fapp);
    std::vector<double> w(z), q(m);
    std::vector<std::vector<double>> Ws, Qs;
    double rz = dot(r.data(), z.data(), m);
    const double target = o.rel ? o.tol * eps0 : o.tol;
    while (true) {
      if (eps <= target) { status = 0; break; }
      if (it >= o.max_it) { status = 1; break; }
      apply_F(w.data(), q.data());
      ++fapp;
      const double delta = dot(w.data(), q.data(), m);
      if (!(delta > 0.0)) { status = 2; break; }
      const double alpha = (o.directions == 1) ? dot(w.data(), r.data(), m) / delta : rz / delta;
      for (int i = 0; i < m; ++i) lambda[i] += alpha * w[i];
      std::copy(q.begin(), q.end(), tmp.begin());
      project(tmp.data());
      for (int i = 0; i < m; ++i) r[i] -= alpha * tmp[i];
      apply_precond(r.data(), z.data(), nullptr);
      project(z.data());
      const double rz_new = dot(r.data(), z.data(), m);
      eps = residual_metric(r.data(), z.data(), m);
      ++it;
      rec.push(eps, 1, fapp);
      if (o.directions == 1) {
        const double sd = std::sqrt(delta);
        std::vector<double> wn(m), qn(m);
        for (int i = 0; i < m; ++i) { wn[i] = w[i] / sd; qn[i] = q[i] / sd; }
        Ws.push_back(std::move(wn));
        Qs.push_back(std::move(qn));
        w = z;
        // classical Gram-Schmidt + one refinement pass
        std::vector<double> psi(Ws.size());
        for (int p = 0; p < passes; ++p) {
          for (size_t j = 0; j < Ws.size(); ++j) psi[j] = dot(Qs[j].data(), w.data(), m);
          for (size_t j = 0; j < Ws.size(); ++j)
            for (int i = 0; i < m; ++i) w[i] -= psi[j] * Ws[j][i];
        }
      } else {
        const double beta = rz_new / rz;
        for (int i = 0; i < m; ++i) w[i] = z[i] + beta * w[i];
      }
      rz = rz_new;
    }
    if (g_check && o.directions == 1) {
      std::vector<const double*> wp, qp;
      for (size_t j = 0; j < Ws.size(); ++j) { wp.push_back(Ws[j].data()); qp.push_back(Qs[j].data()); }
      check_orth(wp, qp, m);
    }
  } else {
    // Alg. 1
    Mat Z(m, Ns), W, Q;
    apply_precond(r.data(), z.data(), Z.a.data());
    eps0 = eps = residual_metric(r.data(), z.data(), m);
    rec.push(eps, Ns, fapp);
    W = Z;
    for (int c = 0; c < Ns; ++c) project(W.col(c));
    std::vector<Mat> Ws, Qs;
    const double target = o.rel ? o.tol * eps0 : o.tol;
    int kept_last = Ns;
    while (true) {
      if (eps <= target) { status = 0; break; }
      if (it >= o.max_it) { status = 1; break; }
      const int k = W.c;
      Q = Mat(m, k);
      for (int c = 0; c < k; ++c) apply_F(W.col(c), Q.col(c));
      fapp += k;
      Mat Delta(k, k);
#pragma omp parallel for schedule(dynamic)
      for (int b = 0; b < k; ++b)
        for (int a = b; a < k; ++a) Delta(a, b) = dot(Q.col(a), W.col(b), m);
      for (int b = 0; b < k; ++b)
        for (int a = 0; a < b; ++a) Delta(a, b) = Delta(b, a);  // lower triangle is used
      PivChol pc = pivoted_cholesky(Delta, o.pivot_tol);
      if (pc.rank == 0) { status = 2; break; }
      W = compress(pc, W);
      Q = compress(pc, Q);
      const int kr = pc.rank;
      std::vector<double> gamma(kr);
#pragma omp parallel for schedule(static)
      for (int c = 0; c < kr; ++c) gamma[c] = dot(W.col(c), r.data(), m);
      std::fill(tmp.begin(), tmp.end(), 0.0);
#pragma omp parallel for schedule(static)
      for (int i = 0; i < m; ++i)
        for (int c = 0; c < kr; ++c) {
          lambda[i] += W(i, c) * gamma[c];
          tmp[i] += Q(i, c) * gamma[c];
        }
      project(tmp.data());
      for (int i = 0; i < m; ++i) r[i] -= tmp[i];
      apply_precond(r.data(), z.data(), Z.a.data());
      eps = residual_metric(r.data(), z.data(), m);
      ++it;
      kept_last = kr;
      rec.push(eps, kr, fapp);
      Ws.push_back(std::move(W));
      Qs.push_back(std::move(Q));
      W = Z;
      for (int c = 0; c < Ns; ++c) project(W.col(c));
      // lines 18-21 as block classical Gram-Schmidt against all stored
      // blocks, twice: Psi_j = Q_j^T W for all j, then
      // W -= sum_j W_j Psi_j
      for (int p = 0; p < passes; ++p) {
        std::vector<Mat> Psis(Ws.size());
        for (size_t j = 0; j < Ws.size(); ++j) {
          const Mat& Qj = Qs[j];
          Mat& Psi = Psis[j];
          Psi = Mat(Qj.c, W.c);
#pragma omp parallel for schedule(dynamic)
          for (int b = 0; b < W.c; ++b)
            for (int a = 0; a < Qj.c; ++a) Psi(a, b) = dot(Qj.col(a), W.col(b), m);
        }
        for (size_t j = 0; j < Ws.size(); ++j) {
          const Mat& Wj = Ws[j];
          const Mat& Psi = Psis[j];
#pragma omp parallel for schedule(dynamic)
          for (int b = 0; b < W.c; ++b)
            for (int a = 0; a < Wj.c; ++a) {
              const double ps = Psi(a, b);
              const double* wj = Wj.col(a);
              double* wb = W.col(b);
              for (int i = 0; i < m; ++i) wb[i] -= wj[i] * ps;
            }
        }
      }
    }
    (void)kept_last;
    if (g_check) {
      std::vector<const double*> wp, qp;
      for (size_t j = 0; j < Ws.size(); ++j)
        for (int c = 0; c < Ws[j].c; ++c) { wp.push_back(Ws[j].col(c)); qp.push_back(Qs[j].col(c)); }
      check_orth(wp, qp, m);
    }
  }
  if (tr) {
    tr->status = status;
    tr->iterations = it;
    tr->f_applies = fapp;
    tr->eps0 = eps0;
    tr->eps_final = eps;
  }
  return 0;
}

// direct_oracle: global assembly with merged interface DOFs,
// prescribed DOFs eliminated, band Cholesky in the ordering with the smaller
// bandwidth.  Returns per-subdomain copies.
void Oracle::direct(double* u) {
  const int n = P.n, nn = n + 1;
  const int nodes = GX * GY;
  const bool colmajor = GY < GX;  // number along the shorter side
  auto gid = [&](int gx, int gy) { return colmajor ? gx * GY + gy : gy * GX + gx; };
  std::vector<int> free_id(2 * nodes, -1), rev;
  for (int k = 0; k < nodes; ++k) {
    int gx = colmajor ? k / GY : k % GX, gy = colmajor ? k % GY : k / GX;
    int g = gnode(gx, gy);
    for (int dir = 0; dir < 2; ++dir)
      if (!prescribed[2 * g + dir]) { free_id[2 * k + dir] = (int)rev.size(); rev.push_back(2 * k + dir); }
  }
  (void)gid;
  const int nf = (int)rev.size();
  // band assembly
  int kd = 0;
  auto fid = [&](int s, int ldof) {
    const Sub& S = subs[s];
    int node = ldof / 2, dir = ldof % 2;
    int gx = S.si * n + node % nn, gy = S.sj * n + node / nn;
    int k = colmajor ? gx * GY + gy : gy * GX + gx;
    return std::make_pair(2 * k + dir, gnode(gx, gy) * 2 + dir);
  };
  for (auto& S : subs)
    for (int i = 0; i < nloc; ++i)
      for (int k = S.K.ptr[i]; k < S.K.ptr[i + 1]; ++k) {
        int a = free_id[fid(S.id, i).first], b = free_id[fid(S.id, S.K.idx[k]).first];
        if (a >= 0 && b >= 0) kd = std::max(kd, std::abs(a - b));
      }
  BandChol bc;
  bc.n = nf;
  bc.kd = kd;
  bc.L.assign((size_t)nf * (kd + 1), 0.0);
  std::vector<double> f(nf, 0.0);
  for (auto& S : subs)
    for (int i = 0; i < nloc; ++i) {
      auto pi = fid(S.id, i);
      int a = free_id[pi.first];
      if (a < 0) continue;
      f[a] += S.f[i];
      for (int k = S.K.ptr[i]; k < S.K.ptr[i + 1]; ++k) {
        auto pj = fid(S.id, S.K.idx[k]);
        int b = free_id[pj.first];
        if (b < 0) f[a] -= S.K.val[k] * presc_val[pj.second];
        else if (b <= a) bc.at(a, b) += S.K.val[k];
      }
    }
  for (int j = 0; j < nf; ++j) {
    double dd = bc.at(j, j);
    if (!(dd > 0.0)) fail(SingularGlobal, "global stiffness is singular");
    double l = std::sqrt(dd);
    bc.at(j, j) = l;
    int last = std::min(nf - 1, j + kd);
    for (int i = j + 1; i <= last; ++i) bc.at(i, j) /= l;
    for (int k = j + 1; k <= last; ++k) {
      double lkj = bc.at(k, j);
      if (lkj == 0.0) continue;
      for (int i = k; i <= last; ++i) bc.at(i, k) -= bc.at(i, j) * lkj;
    }
  }
  bc.solve(f.data());
  for (auto& S : subs)
    for (int i = 0; i < nloc; ++i) {
      auto pi = fid(S.id, i);
      int a = free_id[pi.first];
      u[(size_t)S.id * nloc + i] = a >= 0 ? f[a] : presc_val[pi.second];
    }
}

}  // namespace fo

// ------------------------------------------------------------------ C API --
using namespace fo;
static thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return InvalidArgument;
  }
}

extern "C" {

const char* fo_last_error(void) { return g_err.c_str(); }
void fo_set_refine(int on) { g_refine = on != 0; }
void fo_set_check(int on) {
  g_check = on != 0;
  g_check_err = -1.0;
  g_check_n = 0;
}
void fo_check_result(double* err, int* n) {
  *err = g_check_err;
  *n = g_check_n;
}
// host threads for the OpenMP loops (the CPU baseline uses every core even
// under torchrun, which sets OMP_NUM_THREADS=1); returns the count in force
int fo_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}

int fo_create(const fo_problem* p, void** out) {
  *out = nullptr;
  auto o = std::make_unique<Oracle>();
  int rc = guarded([&] {
    o->P = *p;
    o->refine = g_refine;
    o->build();
  });
  if (rc == 0) *out = o.release();
  return rc;
}
void fo_destroy(void* h) { delete static_cast<Oracle*>(h); }

int fo_info(void* h, int* info) {
  auto* o = static_cast<Oracle*>(h);
  info[0] = o->m;
  info[1] = o->Ns;
  info[2] = o->nloc;
  info[3] = o->Nc;
  info[4] = (int)o->kept.size();
  info[5] = o->n_iface;
  int mx = 0;
  for (auto& S : o->subs) mx = std::max(mx, (int)S.T.size());
  info[6] = mx;
  return 0;
}
int fo_rows(void* h, int* kind, int* sp, int* dp, int* sm, int* dm, double* gap, int* mult,
            double* wp, double* wm) {
  auto* o = static_cast<Oracle*>(h);
  for (int i = 0; i < o->m; ++i) {
    const Row& r = o->rows[i];
    kind[i] = r.kind; sp[i] = r.sp; dp[i] = r.dp; sm[i] = r.sm; dm[i] = r.dm;
    gap[i] = r.gap; mult[i] = r.mult; wp[i] = o->wplus[i]; wm[i] = o->wminus[i];
  }
  return 0;
}
int fo_apply_F(void* h, const double* x, double* y) {
  return guarded([&] { static_cast<Oracle*>(h)->apply_F(x, y); });
}
int fo_apply_precond(void* h, const double* r, double* z, double* Z) {
  return guarded([&] { static_cast<Oracle*>(h)->apply_precond(r, z, Z); });
}
int fo_project(void* h, double* v) {
  return guarded([&] { static_cast<Oracle*>(h)->project(v); });
}
int fo_rhs(void* h, double* d, double* l0) {
  return guarded([&] { static_cast<Oracle*>(h)->rhs(d, l0); });
}
int fo_solve(void* h, const fo_opts* o, double* lambda, fo_trace* tr) {
  return guarded([&] { static_cast<Oracle*>(h)->solve(*o, lambda, tr); });
}
int fo_recover(void* h, const double* lambda, double* u) {
  return guarded([&] { static_cast<Oracle*>(h)->recover(lambda, u); });
}
int fo_local_diag(void* h, double* diag) {
  auto* o = static_cast<Oracle*>(h);
  for (auto& S : o->subs) std::copy(S.diag.begin(), S.diag.end(), diag + (size_t)S.id * o->nloc);
  return 0;
}
int fo_load_vectors(void* h, double* f) {
  auto* o = static_cast<Oracle*>(h);
  for (auto& S : o->subs) std::copy(S.f.begin(), S.f.end(), f + (size_t)S.id * o->nloc);
  return 0;
}
// admissibility_error (decomposition.hpp:177-180): cluster-by-cluster max
// deviation of sum_s B^s (Btilde^s)^T B^j = B^j.
double fo_admissibility_error(void* h) {
  auto* o = static_cast<Oracle*>(h);
  // entries grouped by (global node, dir): rows of one DOF interact only there
  double err = 0.0;
  std::vector<std::vector<int>> by_dof(2 * o->GX * o->GY);
  for (int i = 0; i < o->m; ++i) by_dof[2 * o->rows[i].gnode + o->rows[i].dir].push_back(i);
  for (auto& rl : by_dof) {
    if (rl.empty()) continue;
    // copies (sub) involved
    std::vector<int> subsv;
    for (int i : rl) {
      subsv.push_back(o->rows[i].sp);
      if (o->rows[i].kind == 0) subsv.push_back(o->rows[i].sm);
    }
    std::sort(subsv.begin(), subsv.end());
    subsv.erase(std::unique(subsv.begin(), subsv.end()), subsv.end());
    const int nr = (int)rl.size(), ns = (int)subsv.size();
    auto Bv = [&](int ri, int sidx, bool scaled) {
      const Row& r = o->rows[rl[ri]];
      int s = subsv[sidx];
      if (r.sp == s) return scaled ? o->wplus[rl[ri]] : 1.0;
      if (r.kind == 0 && r.sm == s) return scaled ? -o->wminus[rl[ri]] : -1.0;
      return 0.0;
    };
    // M = sum_s B^s (Btilde^s)^T  (nr x nr), then check M B^j = B^j
    std::vector<double> M(nr * nr, 0.0);
    for (int a = 0; a < nr; ++a)
      for (int b = 0; b < nr; ++b)
        for (int s = 0; s < ns; ++s) M[a * nr + b] += Bv(a, s, false) * Bv(b, s, true);
    for (int j = 0; j < ns; ++j)
      for (int a = 0; a < nr; ++a) {
        double v = 0.0;
        for (int b = 0; b < nr; ++b) v += M[a * nr + b] * Bv(b, j, false);
        err = std::max(err, std::abs(v - Bv(a, j, false)));
      }
  }
  return err;
}
// K^s x for one subdomain (assembled local stiffness, fem.cpp:86-119)
int fo_local_apply(void* h, int s, const double* x, double* y) {
  auto* o = static_cast<Oracle*>(h);
  if (s < 0 || s >= o->Ns) return InvalidArgument;
  o->subs[s].K.matvec(x, y);
  return 0;
}
// T-FETI: max_i |(G lambda - e)_i| over all rows (constraint_residual_inf,
// decomposition.hpp:141-142)
double fo_coarse_residual(void* h, const double* lambda) {
  auto* o = static_cast<Oracle*>(h);
  if (o->P.method != 0) return 0.0;
  double mx = 0.0;
  for (int a = 0; a < 3 * o->Ns; ++a) {
    double v = dot_(o->Gt.col(a), lambda, o->m) - o->e[a];
    mx = std::max(mx, std::abs(v));
  }
  return mx;
}
// pseudo_solve with the compatibility check (linalg.cpp:191-204)
int fo_pseudo_solve(void* h, int s, const double* rhs, double* x) {
  auto* o = static_cast<Oracle*>(h);
  return guarded([&] {
    if (o->P.method != 0) fail(ConfigError, "pseudo_solve needs T-FETI factors");
    Sub& S = o->subs[s];
    double rn = 0.0;
    for (int i = 0; i < o->nloc; ++i) rn += rhs[i] * rhs[i];
    rn = std::sqrt(rn);
    for (int c = 0; c < 3; ++c) {
      double pr = 0.0, nr = 0.0;
      for (int i = 0; i < o->nloc; ++i) { pr += o->R(i, c) * rhs[i]; nr += o->R(i, c) * o->R(i, c); }
      if (std::abs(pr) > 1e-8 * rn * std::sqrt(nr))
        fail(IncompatibleRhs, "rhs has a nullspace component: |R^T rhs| = " + std::to_string(std::abs(pr)));
    }
    std::vector<double> b(S.keep.size());
    for (size_t i = 0; i < S.keep.size(); ++i) b[i] = rhs[S.keep[i]];
    S.kred.solve(b.data());
    for (int i = 0; i < o->nloc; ++i) x[i] = 0.0;
    for (size_t i = 0; i < S.keep.size(); ++i) x[S.keep[i]] = b[i];
  });
}
int fo_fixed_dofs(void* h, int* out) {
  auto* o = static_cast<Oracle*>(h);
  if (o->P.method != 0) return ConfigError;
  for (int i = 0; i < 3; ++i) out[i] = o->subs[0].fixed[i];
  return 0;
}

int fo_direct_solve(void* h, double* u) {
  return guarded([&] { static_cast<Oracle*>(h)->direct(u); });
}

int fo_simp_modulus(double rho, double E0, double Emin, double p, double* out) {
  return guarded([&] {
    Material m;
    m.E0 = E0; m.Emin = Emin; m.p = p;
    *out = simp_modulus(rho, m);
  });
}
int fo_q4_element_stiffness(double nu, double thickness, double modulus, double hx, double hy,
                            double* k) {
  return guarded([&] {
    if (!(modulus > 0.0) || !(hx > 0.0) || !(hy > 0.0))
      fail(InvalidArgument, "q4_element_stiffness: nonpositive input");
    Material m;
    m.nu = nu; m.thickness = thickness;
    q4_unit(m, hx, hy, k);
    for (int i = 0; i < 64; ++i) k[i] *= modulus;
  });
}
int fo_pivoted_cholesky(int n, const double* a, double tol, int* perm, double* lower, int* rank) {
  return guarded([&] {
    Mat A(n, n);
    std::copy(a, a + (size_t)n * n, A.a.begin());
    PivChol pc = pivoted_cholesky(A, tol);
    for (int i = 0; i < n; ++i) perm[i] = pc.perm[i];
    std::fill(lower, lower + (size_t)n * n, 0.0);
    for (int j = 0; j < pc.rank; ++j)
      for (int i = 0; i < n; ++i) lower[(size_t)j * n + i] = pc.lower(i, j);
    *rank = pc.rank;
  });
}
int fo_compress(int n, const int* perm, const double* lower, int rank, int rows, const double* w,
                double* out) {
  return guarded([&] {
    PivChol pc;
    pc.dim = n;
    pc.rank = rank;
    pc.perm.assign(perm, perm + n);
    pc.lower = Mat(n, rank);
    for (int j = 0; j < rank; ++j)
      for (int i = 0; i < n; ++i) pc.lower(i, j) = lower[(size_t)j * n + i];
    Mat W(rows, n);
    std::copy(w, w + (size_t)rows * n, W.a.begin());
    Mat o = compress(pc, W);
    std::copy(o.a.begin(), o.a.end(), out);
  });
}
int fo_select_fixing_dofs(int rows, int cols, const double* basis, int* out) {
  return guarded([&] {
    Mat B(rows, cols);
    std::copy(basis, basis + (size_t)rows * cols, B.a.begin());
    auto f = select_fixing_dofs(B);
    for (int i = 0; i < cols; ++i) out[i] = f[i];
  });
}
int fo_rigid_body_modes(int n, double hx, double hy, double* R) {
  Mat r = rigid_body_modes(n, hx, hy);
  std::copy(r.a.begin(), r.a.end(), R);
  return 0;
}
int fo_band_cholesky_solve(int n, const double* a, double* b) {
  return guarded([&] {
    Csr A;
    A.n = n;
    A.ptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < n; ++j)
        if (a[(size_t)j * n + i] != 0.0) { A.idx.push_back(j); A.val.push_back(a[(size_t)j * n + i]); }
      A.ptr[i + 1] = (int)A.idx.size();
    }
    std::vector<int> all(n);
    std::iota(all.begin(), all.end(), 0);
    BandChol bc;
    bc.factor(A, all, NotPositiveDefinite, "sparse Cholesky");
    bc.solve(b);
  });
}

}  // extern "C"
