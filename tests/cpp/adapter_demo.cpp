// Exercises the C++ adapter (include/feti_gpu.hpp) the way a reference-side
// caller would: T-FETI on a 2x1 partition of 4x4 modules, left clamp, right
// edge traction.  Without a GPU it must report NoDevice loudly; with one it
// builds, applies F, solves and recovers.
#include <cmath>
#include <cstdio>
#include <vector>

#include "feti_gpu.hpp"

int main() {
  const int sx = 2, sy = 1, n = 4;
  std::vector<double> rho(n * n, 1.0);
  std::vector<int> mt{0, 0};
  std::vector<int> dg, dd;
  std::vector<double> dv;
  for (int gy = 0; gy <= sy * n; ++gy)
    for (int d = 0; d < 2; ++d) { dg.push_back(gy * (sx * n + 1)); dd.push_back(d); dv.push_back(0.0); }
  int tsub[1] = {1}, tside[1] = {1}, tfirst[1] = {0}, tcount[1] = {n};
  double txy[2] = {0.0, -1.0};
  fetigpu_problem p{};
  p.sx = sx; p.sy = sy; p.n = n; p.hx = p.hy = 1.0;
  p.E0 = 1.0; p.Emin = 1e-9; p.nu = 0.3; p.p = 3.0; p.thickness = 1.0;
  p.n_designs = 1; p.densities = rho.data(); p.module_type = mt.data();
  p.n_dirichlet = (int)dg.size(); p.dir_gnode = dg.data(); p.dir_dir = dd.data(); p.dir_value = dv.data();
  p.n_tractions = 1; p.tr_sub = tsub; p.tr_side = tside; p.tr_first = tfirst; p.tr_count = tcount; p.tr_txy = txy;
  p.method = FETIGPU_TFETI; p.scaling = FETIGPU_KSCALING; p.precond = FETIGPU_DIRICHLET;
  try {
    fetigpu::DualSystem sys(p);
    std::printf("dual size %d\n", sys.dual_size());
    sys.build();
    sys.set_rrs_store(FETIGPU_RRS_STORE_AUTO);  // T-FETI: the explicit (reference) store
    std::vector<double> x(sys.dual_size(), 1.0);
    auto y = sys.apply(x);
    fetigpu::SolveOptions o;
    o.directions = FETIGPU_FO;
    fetigpu::ConvergenceTrace tr;
    auto lam = sys.solve(o, &tr);
    auto u = sys.recover_primal(lam);
    std::printf("solve status %d iterations %d tip uy %.6e\n", tr.status, tr.iterations, u[1][2 * n + 1]);
    // SIMP-loop use: next density snapshot in place, warm-started solve
    std::vector<double> rho2(rho.size());
    for (size_t i = 0; i < rho.size(); ++i) rho2[i] = 0.5 * rho[i] + 0.25;
    fetigpu_problem p2 = p;
    p2.densities = rho2.data();
    sys.rebuild(p2);
    fetigpu::ConvergenceTrace tr2;
    auto lam2 = sys.solve_warm(o, lam, &tr2);
    std::printf("rebuild + warm solve status %d iterations %d\n", tr2.status, tr2.iterations);
    // pivoted_cholesky / PivotedCholesky::compress (linalg.hpp:72-89)
    std::vector<double> a{1.0, 2.0, 2.0, 4.0 + 1e-3};  // 2x2 column-major, pivot 1 first
    auto pc = fetigpu::pivoted_cholesky(a, 2);
    std::vector<double> w{1.0, 0.0, 0.0, 1.0};
    auto c = pc.compress(w, 2);
    std::printf("pivchol rank %d perm %d %d L00 %.6f compress %zu\n", pc.rank, pc.permutation[0],
                pc.permutation[1], pc.lower[0], c.size());
    return tr.status == 0 && tr2.status == 0 && pc.rank == 2 && pc.permutation[0] == 1 ? 0 : 3;
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 2;
  }
}
