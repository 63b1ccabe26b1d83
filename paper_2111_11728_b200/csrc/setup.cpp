// setup.cpp -- host-side problem setup (see setup.hpp).
#include "setup.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <numeric>
#include <unordered_map>

namespace fg {

// Rank-revealing Cholesky with a symmetric trailing update: the SPEC.md:43-47
// contract of pivoted_cholesky (linalg.hpp:85-89).  a is n x n column-major.
void pivoted_cholesky_host(std::vector<double>& a, int n, double tol, std::vector<int>& perm,
                           int& rank) {
  auto A = [&](int i, int j) -> double& { return a[(size_t)j * n + i]; };
  perm.resize(n);
  std::iota(perm.begin(), perm.end(), 0);
  double scale = 0.0;
  for (int i = 0; i < n; ++i) scale = std::max(scale, A(i, i));
  const double stop = tol * scale, neg = -tol * std::max(scale, 1e-300);
  rank = 0;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int j = k + 1; j < n; ++j)
      if (A(j, j) > A(piv, piv)) piv = j;
    const double d = A(piv, piv);
    if (d <= stop) {
      for (int j = k; j < n; ++j)
        if (A(j, j) < neg) fail(FETIGPU_E_INDEFINITE_INPUT, "pivoted Cholesky: negative pivot");
      break;
    }
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(piv, j));
      for (int i = 0; i < n; ++i) std::swap(A(i, k), A(i, piv));
      std::swap(perm[k], perm[piv]);
    }
    const double l = std::sqrt(d);
    A(k, k) = l;
    for (int i = k + 1; i < n; ++i) A(i, k) /= l;
    for (int j = k + 1; j < n; ++j) {
      const double ajk = A(j, k);
      for (int i = k + 1; i < n; ++i) A(i, j) -= A(i, k) * ajk;
    }
    rank = k + 1;
  }
}

namespace {

// q4_element_stiffness at unit modulus (fem.cpp:44-84): unit plane-stress D,
// 2x2 Gauss points in the order (-,-),(+,-),(+,+),(-,+), upper -> lower copy.
void q4_unit(double nu, double t, double hx, double hy, double* k) {
  const double c = 1.0 / (1.0 - nu * nu);
  const double D[3][3] = {{c, c * nu, 0.0}, {c * nu, c, 0.0}, {0.0, 0.0, c * (1.0 - nu) / 2.0}};
  const double g = 1.0 / std::sqrt(3.0);
  const double xi[4] = {-1.0, 1.0, 1.0, -1.0}, eta[4] = {-1.0, -1.0, 1.0, 1.0};
  std::fill(k, k + 64, 0.0);
  const double det_j = hx * hy / 4.0;
  for (int gp = 0; gp < 4; ++gp) {
    const double s = g * xi[gp], tt = g * eta[gp];
    double b[3][8] = {};
    for (int a = 0; a < 4; ++a) {
      const double dx = 0.25 * xi[a] * (1.0 + eta[a] * tt) * 2.0 / hx;
      const double dy = 0.25 * eta[a] * (1.0 + xi[a] * s) * 2.0 / hy;
      b[0][2 * a] = dx;
      b[1][2 * a + 1] = dy;
      b[2][2 * a] = dy;
      b[2][2 * a + 1] = dx;
    }
    double bd[8][3];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 3; ++j) bd[i][j] = b[0][i] * D[0][j] + b[1][i] * D[1][j] + b[2][i] * D[2][j];
    for (int j = 0; j < 8; ++j)
      for (int i = 0; i < 8; ++i)
        k[j * 8 + i] += (bd[i][0] * b[0][j] + bd[i][1] * b[1][j] + bd[i][2] * b[2][j]) * det_j;
  }
  for (int i = 0; i < 64; ++i) k[i] *= t;
  for (int i = 0; i < 8; ++i)
    for (int j = i + 1; j < 8; ++j) k[i * 8 + j] = k[j * 8 + i];
}

struct NdBuilder {
  int n, nn, leaf;
  NdPlan& P;
  std::vector<int> perim(int x0, int x1, int y0, int y1) const {
    std::vector<int> v;
    for (int ix = x0; ix <= x1; ++ix) v.push_back(y0 * nn + ix);
    for (int iy = y0 + 1; iy <= y1; ++iy) v.push_back(iy * nn + x1);
    for (int ix = x1 - 1; ix >= x0; --ix) v.push_back(y1 * nn + ix);
    for (int iy = y1 - 1; iy >= y0 + 1; --iy) v.push_back(iy * nn + x0);
    return v;
  }
  static std::vector<int> dofs_of(const std::vector<int>& sep, const std::vector<int>& per) {
    std::vector<int> d;
    for (int v : sep) { d.push_back(2 * v); d.push_back(2 * v + 1); }
    for (int v : per) { d.push_back(2 * v); d.push_back(2 * v + 1); }
    return d;
  }
  int build(int x0, int x1, int y0, int y1) {
    const int w = x1 - x0, h = y1 - y0;
    NdNode node;
    node.x0 = x0; node.x1 = x1; node.y0 = y0; node.y1 = y1;
    std::vector<int> per = perim(x0, x1, y0, y1), sep;
    if (w <= leaf && h <= leaf) {
      node.leaf = true;
      for (int iy = y0 + 1; iy < y1; ++iy)
        for (int ix = x0 + 1; ix < x1; ++ix) sep.push_back(iy * nn + ix);
      node.dofs = dofs_of(sep, per);
      std::map<int, int> pos;
      for (size_t i = 0; i < node.dofs.size(); ++i) pos[node.dofs[i]] = (int)i;
      for (int ey = y0; ey < y1; ++ey)
        for (int ex = x0; ex < x1; ++ex) {
          node.elems.push_back(ey * n + ex);
          const int n0 = ey * nn + ex;
          const int nodes[4] = {n0, n0 + 1, n0 + nn + 1, n0 + nn};
          for (int a = 0; a < 4; ++a)
            for (int d = 0; d < 2; ++d) node.emap.push_back(pos.at(2 * nodes[a] + d));
        }
      node.height = 0;
    } else {
      int c0, c1;
      if (w >= h) {
        const int xm = x0 + w / 2;
        c0 = build(x0, xm, y0, y1);
        c1 = build(xm, x1, y0, y1);
        for (int iy = y0 + 1; iy < y1; ++iy) sep.push_back(iy * nn + xm);
      } else {
        const int ym = y0 + h / 2;
        c0 = build(x0, x1, y0, ym);
        c1 = build(x0, x1, ym, y1);
        for (int ix = x0 + 1; ix < x1; ++ix) sep.push_back(ym * nn + ix);
      }
      node.child[0] = c0;
      node.child[1] = c1;
      node.dofs = dofs_of(sep, per);
      std::map<int, int> pos;
      for (size_t i = 0; i < node.dofs.size(); ++i) pos[node.dofs[i]] = (int)i;
      for (int c = 0; c < 2; ++c) {
        const NdNode& ch = P.nodes[node.child[c]];
        for (int i = ch.ne; i < ch.nf; ++i) {
          auto it = pos.find(ch.dofs[i]);
          if (it == pos.end()) fail(FETIGPU_E_STATE, "nd plan: child perimeter not covered");
          node.cmap[c].push_back(it->second);
        }
      }
      node.height = 1 + std::max(P.nodes[c0].height, P.nodes[c1].height);
    }
    node.ne = 2 * (int)sep.size();
    node.nf = (int)node.dofs.size();
    P.nodes.push_back(std::move(node));
    return (int)P.nodes.size() - 1;
  }
};

NdPlan make_nd_plan(int n, int leaf) {
  NdPlan P;
  P.n = n;
  NdBuilder b{n, n + 1, leaf, P};
  P.root = b.build(0, n, 0, n);
  P.max_height = P.nodes[P.root].height;
  P.by_height.assign(P.max_height + 1, {});
  for (int i = 0; i < (int)P.nodes.size(); ++i) P.by_height[P.nodes[i].height].push_back(i);
  P.height_stride.assign(P.max_height + 1, 0);
  for (int h = 0; h <= P.max_height; ++h)
    for (int i : P.by_height[h]) {
      NdNode& nd = P.nodes[i];
      nd.off = P.height_stride[h];
      P.height_stride[h] += (long long)nd.nf * nd.nf;
    }
  P.factor_stride = 0;
  for (auto& nd : P.nodes) {
    nd.foff = P.factor_stride;
    P.factor_stride += (long long)nd.nf * nd.ne;
  }
  // pre-order for back substitution
  std::vector<int> st{P.root};
  while (!st.empty()) {
    int v = st.back();
    st.pop_back();
    P.topdown.push_back(v);
    if (!P.nodes[v].leaf) {
      st.push_back(P.nodes[v].child[1]);
      st.push_back(P.nodes[v].child[0]);
    }
  }
  return P;
}

}  // namespace

int Setup::owners(int gx, int gy, int* sub, int* lnode) const {
  // Partition::owners_of_node (decomposition.hpp:37-42): ascending sub order
  int cnt = 0;
  int sjs[2], sis[2], nsj = 0, nsi = 0;
  for (int sj = std::max(0, (gy - 1) / n); sj <= std::min(sy - 1, gy / n); ++sj)
    if (gy >= sj * n && gy <= sj * n + n) sjs[nsj++] = sj;
  for (int si = std::max(0, (gx - 1) / n); si <= std::min(sx - 1, gx / n); ++si)
    if (gx >= si * n && gx <= si * n + n) sis[nsi++] = si;
  for (int a = 0; a < nsj; ++a)
    for (int b = 0; b < nsi; ++b) {
      sub[cnt] = sjs[a] * sx + sis[b];
      lnode[cnt] = (gy - sjs[a] * n) * nn + (gx - sis[b] * n);
      ++cnt;
    }
  return cnt;
}

namespace {
// FETIGPU_TIMING=1: host wall-clock of the setup phases on stderr
struct HostMarks {
  bool on;
  std::chrono::steady_clock::time_point last;
  HostMarks() {
    const char* e = getenv("FETIGPU_TIMING");
    on = e && e[0] == '1';
    last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[fetigpu] setup %-28s %8.2f ms\n", what,
            std::chrono::duration<double, std::milli>(t - last).count());
    last = t;
  }
};
}  // namespace

void Setup::load(const fetigpu_problem& P) {
  HostMarks hm;
  // ---- validation (Material::validate fem.cpp:9-17, DensityField fem.cpp:38-42)
  if (!(P.Emin > 0.0) || !(P.Emin < P.E0)) fail(FETIGPU_E_INVALID_ARGUMENT, "material: need 0 < Emin < E0");
  if (!(P.nu >= 0.0) || !(P.nu < 0.5)) fail(FETIGPU_E_INVALID_ARGUMENT, "material: need 0 <= nu < 0.5");
  if (!(P.p >= 1.0)) fail(FETIGPU_E_INVALID_ARGUMENT, "material: need p >= 1");
  if (!(P.thickness > 0.0)) fail(FETIGPU_E_INVALID_ARGUMENT, "material: need thickness > 0");
  if (P.sx < 1 || P.sy < 1 || P.n < 2) fail(FETIGPU_E_DIMENSION_MISMATCH, "bad partition");
  if (!(P.hx > 0.0) || !(P.hy > 0.0)) fail(FETIGPU_E_INVALID_ARGUMENT, "nonpositive element size");
  if (P.method != FETIGPU_TFETI && P.method != FETIGPU_FETIDP) fail(FETIGPU_E_CONFIG, "unknown method");
  if (P.scaling != 0 && P.scaling != 1) fail(FETIGPU_E_CONFIG, "unknown scaling");
  if (P.precond < 0 || P.precond > 2) fail(FETIGPU_E_CONFIG, "unknown preconditioner");
  if (P.n_designs < 1 || !P.densities || !P.module_type) fail(FETIGPU_E_DIMENSION_MISMATCH, "need >= 1 design");
  sx = P.sx; sy = P.sy; n = P.n; nn = n + 1; Ns = sx * sy; nloc = 2 * nn * nn; nb = 8 * n;
  GX = sx * n + 1; GY = sy * n + 1;
  method = P.method; scaling = P.scaling; precond = P.precond; n_designs = P.n_designs;
  hx = P.hx; hy = P.hy; E0 = P.E0; Emin = P.Emin; nu = P.nu; p = P.p; thickness = P.thickness;
  densities.assign(P.densities, P.densities + (size_t)n_designs * n * n);
  for (double v : densities)
    if (!(v >= 0.0) || !(v <= 1.0)) fail(FETIGPU_E_DOMAIN, "density outside [0, 1]");
  module_type.assign(P.module_type, P.module_type + Ns);
  for (int d : module_type)
    if (d < 0 || d >= n_designs) fail(FETIGPU_E_DIMENSION_MISMATCH, "module_type out of range");
  q4_unit(nu, thickness, hx, hy, kunit);

  hm.mark("validation + copies");
  // ---- ND plan; its root perimeter defines the module boundary order
  nd = make_nd_plan(n, 4);
  const NdNode& root = nd.nodes[nd.root];
  perim_dof.assign(root.dofs.begin() + root.ne, root.dofs.end());
  if ((int)perim_dof.size() != nb) fail(FETIGPU_E_STATE, "perimeter size mismatch");
  dpos.assign(nloc, -1);
  for (int i = 0; i < nb; ++i) dpos[perim_dof[i]] = i;

  hm.mark("ND plan");
  // ---- boundary stiffness diagonals per design (sum in element order)
  bdiag.assign(n_designs, std::vector<double>(nb, 0.0));
  std::vector<double> diag(nloc, 0.0);
  for (int d = 0; d < n_designs; ++d) {
    const double* rho = &densities[(size_t)d * n * n];
    for (int i = 0; i < nb; ++i) diag[perim_dof[i]] = 0.0;  // only perimeter DOFs are accumulated
    for (int ey = 0; ey < n; ++ey)
      for (int ex = 0; ex < n; ex += (ey == 0 || ey == n - 1 || ex == n - 1) ? 1 : n - 1) {
        const double e = Emin + std::pow(rho[ey * n + ex], p) * (E0 - Emin);
        const int n0 = ey * nn + ex;
        const int nodes[4] = {n0, n0 + 1, n0 + nn + 1, n0 + nn};
        for (int a = 0; a < 4; ++a)
          for (int c = 0; c < 2; ++c) diag[2 * nodes[a] + c] += e * kunit[(2 * a + c) * 8 + 2 * a + c];
      }
    for (int i = 0; i < nb; ++i) bdiag[d][i] = diag[perim_dof[i]];
  }

  hm.mark("boundary diagonals");
  // ---- supports
  std::vector<char> presc(2 * (size_t)GX * GY, 0);
  std::unordered_map<long long, double> pvals;  // prescribed values, keyed by 2 g + dir
  auto pval = [&](long long k) {
    const auto it = pvals.find(k);
    return it == pvals.end() ? 0.0 : it->second;
  };
  for (int k = 0; k < P.n_dirichlet; ++k) {
    const int g = P.dir_gnode[k], dir = P.dir_dir[k];
    if (g < 0 || g >= GX * GY || dir < 0 || dir > 1) fail(FETIGPU_E_NODE_NOT_FOUND, "Dirichlet node not found");
    presc[2 * g + dir] = 1;
    pvals[2 * (long long)g + dir] = P.dir_value[k];
  }
  auto corner = [&](int gx, int gy) { return gx % n == 0 && gy % n == 0; };

  // ---- loads (apply_traction, fem.cpp:121-167; point loads to the lowest owner)
  std::vector<std::vector<double>> floc(Ns);  // allocated only for loaded subdomains
  auto fl = [&](int s) -> std::vector<double>& {
    if (floc[s].empty()) floc[s].assign(nloc, 0.0);
    return floc[s];
  };
  for (int t = 0; t < P.n_tractions; ++t) {
    const int s = P.tr_sub[t], side = P.tr_side[t], first = P.tr_first[t], count = P.tr_count[t];
    if (s < 0 || s >= Ns) fail(FETIGPU_E_DIMENSION_MISMATCH, "traction subdomain out of range");
    int node0, stride;
    double h;
    switch (side) {
      case 0: node0 = 0; stride = nn; h = hy; break;
      case 1: node0 = n; stride = nn; h = hy; break;
      case 2: node0 = 0; stride = 1; h = hx; break;
      case 3: node0 = n * nn; stride = 1; h = hx; break;
      default: fail(FETIGPU_E_EDGE_NOT_ON_BOUNDARY, "bad side");
    }
    if (first < 0 || count < 0 || first + count > n)
      fail(FETIGPU_E_EDGE_NOT_ON_BOUNDARY, "traction chain leaves the boundary");
    const double half = h / 2.0, tx = P.tr_txy[2 * t], ty = P.tr_txy[2 * t + 1];
    std::vector<double>& f = fl(s);
    for (int e = first; e < first + count; ++e) {
      const int n0 = node0 + e * stride, n1 = n0 + stride;
      f[2 * n0] += half * tx;
      f[2 * n0 + 1] += half * ty;
      f[2 * n1] += half * tx;
      f[2 * n1 + 1] += half * ty;
    }
  }
  int osub[4], onode[4];
  for (int k = 0; k < P.n_point_loads; ++k) {
    const int g = P.pl_gnode[k], dir = P.pl_dir[k];
    if (g < 0 || g >= GX * GY || dir < 0 || dir > 1) fail(FETIGPU_E_NODE_NOT_FOUND, "point load node not found");
    owners(g % GX, g / GX, osub, onode);
    fl(osub[0])[2 * onode[0] + dir] += P.pl_value[k];
  }

  hm.mark("supports + loads");
  // ---- constraint rows (decomposition.hpp:110-117; same rules as SPEC.md:198-206)
  rows.clear();
  const bool dp = method == FETIGPU_FETIDP;
  for (int gy = 0; gy < GY; ++gy)
    for (int gx = 0; gx < GX; gx += (gy % n == 0 ? 1 : (gx % n == 0 ? n : n - gx % n))) {
      // nodes off the module grid lines have one owner: visit grid-line nodes only
      if (gy % n != 0 && gx % n != 0) continue;
      const int cnt = owners(gx, gy, osub, onode);
      if (cnt < 2 || (dp && corner(gx, gy))) continue;
      const int g = gy * GX + gx;
      for (int dir = 0; dir < 2; ++dir) {
        if (presc[2 * g + dir]) continue;
        for (int a = 0; a < cnt; ++a)
          for (int b = a + 1; b < cnt; ++b)
            rows.push_back({0, osub[a], 2 * onode[a] + dir, osub[b], 2 * onode[b] + dir, 0.0, cnt, g, dir});
      }
    }
  n_iface = (int)rows.size();
  if (!dp)
    for (int g = 0; g < GX * GY; ++g)
      for (int dir = 0; dir < 2; ++dir) {
        if (!presc[2 * g + dir]) continue;
        const int cnt = owners(g % GX, g / GX, osub, onode);
        for (int a = 0; a < cnt; ++a)
          rows.push_back({1, osub[a], 2 * onode[a] + dir, -1, -1, pval(2 * (long long)g + dir), cnt, g, dir});
      }
  m = (int)rows.size();
  gap.resize(m);
  for (int i = 0; i < m; ++i) gap[i] = rows[i].gap;

  hm.mark("constraint rows");
  // ---- scaling weights (decomposition.hpp:159-175)
  wplus.assign(m, 1.0);
  wminus.assign(m, 0.0);
  for (int i = 0; i < m; ++i) {
    const Row& r = rows[i];
    if (r.kind == 1) continue;
    if (scaling == FETIGPU_MULTIPLICITY) {
      wplus[i] = wminus[i] = 1.0 / r.mult;
    } else {
      const int cnt = owners(r.gnode % GX, r.gnode / GX, osub, onode);
      double den = 0.0, kp = 0.0, km = 0.0;
      for (int a = 0; a < cnt; ++a) {
        const int pos = dpos[2 * onode[a] + r.dir];
        const double dg = bdiag[module_type[osub[a]]][pos];
        if (!(dg > 0.0)) fail(FETIGPU_E_ZERO_STIFFNESS_DIAGONAL, "nonpositive stiffness diagonal");
        den += dg;
        if (osub[a] == r.sp) kp = dg;
        if (osub[a] == r.sm) km = dg;
      }
      wplus[i] = km / den;
      wminus[i] = kp / den;
    }
  }

  hm.mark("scaling weights");
  // ---- per-subdomain plans
  subs.assign(Ns, SubPlan());
  for (int s = 0; s < Ns; ++s) {
    SubPlan& S = subs[s];
    S.si = s % sx; S.sj = s / sx; S.design = module_type[s];
    S.f.assign(nb, 0.0);
    if (floc[s].empty()) continue;
    for (int i = 0; i < nloc; ++i)
      if (floc[s][i] != 0.0 && dpos[i] < 0)
        fail(FETIGPU_E_CONFIG, "loads on module-interior DOFs are not supported");
    for (int i = 0; i < nb; ++i) S.f[i] = floc[s][perim_dof[i]];
  }
  std::vector<std::vector<char>> touched(Ns, std::vector<char>(nb, 0));
  for (int i = 0; i < m; ++i) {
    const Row& r = rows[i];
    if (dpos[r.dp] < 0 || (r.kind == 0 && dpos[r.dm] < 0))
      fail(FETIGPU_E_CONFIG, "constraints on module-interior DOFs are not supported");
    touched[r.sp][dpos[r.dp]] = 1;
    if (r.kind == 0) touched[r.sm][dpos[r.dm]] = 1;
  }
  for (int s = 0; s < Ns; ++s)
    for (int i = 0; i < nb; ++i)
      if (touched[s][i]) subs[s].T.push_back(i);

  hm.mark("per-subdomain plans");
  // rigid body modes (decomposition.hpp:119-121), about the module centroid
  Rfull.assign((size_t)nloc * 3, 0.0);
  {
    const double xc = n * hx / 2.0, yc = n * hy / 2.0;
    for (int v = 0; v < nn * nn; ++v) {
      const double x = (v % nn) * hx, y = (v / nn) * hy;
      Rfull[2 * v] = 1.0;
      Rfull[nloc + 2 * v + 1] = 1.0;
      Rfull[2 * nloc + 2 * v] = -(y - yc);
      Rfull[2 * nloc + 2 * v + 1] = x - xc;
    }
  }
  Rb.assign((size_t)nb * 3, 0.0);
  for (int i = 0; i < nb; ++i)
    for (int k = 0; k < 3; ++k) Rb[k * nb + i] = Rfull[(size_t)k * nloc + perim_dof[i]];

  op_slots.clear();
  pc_slots.clear();
  pc_lumped_T.clear();
  pc_lumped_design.clear();
  std::map<std::vector<int>, int> op_key, pc_key;

  if (!dp) {
    // fixing DOFs: select_fixing_dofs (linalg.cpp:146-175) on the full basis
    std::vector<int> fixed;
    std::vector<std::vector<double>> ortho;
    for (int pick = 0; pick < 3; ++pick) {
      int best = -1;
      double best_score = -1.0;
      for (int d = 0; d < nloc; ++d) {
        double r[3] = {Rfull[d], Rfull[nloc + d], Rfull[2 * nloc + d]};
        for (auto& o : ortho) {
          const double dt = o[0] * Rfull[d] + o[1] * Rfull[nloc + d] + o[2] * Rfull[2 * nloc + d];
          for (int k = 0; k < 3; ++k) r[k] -= o[k] * dt;
        }
        const double sc = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
        if (sc > best_score) { best_score = sc; best = d; }
      }
      if (best < 0 || best_score <= 0.0) fail(FETIGPU_E_INDEFINITE_INPUT, "nullspace basis is rank deficient");
      fixed.push_back(best);
      double r[3] = {Rfull[best], Rfull[nloc + best], Rfull[2 * nloc + best]};
      for (auto& o : ortho) {
        const double dt = o[0] * Rfull[best] + o[1] * Rfull[nloc + best] + o[2] * Rfull[2 * nloc + best];
        for (int k = 0; k < 3; ++k) r[k] -= o[k] * dt;
      }
      const double nr = std::sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
      ortho.push_back({r[0] / nr, r[1] / nr, r[2] / nr});
    }
    std::sort(fixed.begin(), fixed.end());
    fixed_pos.clear();
    for (int d : fixed) {
      if (dpos[d] < 0) fail(FETIGPU_E_CONFIG, "fixing DOF not on the module perimeter");
      fixed_pos.push_back(dpos[d]);
    }
    std::sort(fixed_pos.begin(), fixed_pos.end());
    std::vector<int> keep;
    for (int i = 0; i < nb; ++i)
      if (!std::binary_search(fixed_pos.begin(), fixed_pos.end(), i)) keep.push_back(i);
    std::vector<int> kidx(nb, -1);
    for (size_t i = 0; i < keep.size(); ++i) kidx[keep[i]] = (int)i;
    for (int s = 0; s < Ns; ++s) {
      SubPlan& S = subs[s];
      S.Top.clear();
      for (int t : S.T)
        if (kidx[t] >= 0) S.Top.push_back(t);
      std::vector<int> key{S.design};
      key.insert(key.end(), S.Top.begin(), S.Top.end());
      auto it = op_key.find(key);
      if (it == op_key.end()) {
        SlotFront sf;
        sf.design = S.design;
        sf.src = keep;
        sf.ne = (int)keep.size();
        for (int t : S.Top) sf.ext.push_back(kidx[t]);
        op_slots.push_back(sf);
        it = op_key.emplace(key, (int)op_slots.size() - 1).first;
      }
      S.op_slot = it->second;
    }
    // natural coarse space G = -R^T B^T, (G G^T) filtered by rank-revealing
    // Cholesky at 1e-10, padded inverse H
    const int nc = 3 * Ns;
    std::vector<double> GG((size_t)nc * nc, 0.0);
    for (int i = 0; i < m; ++i) {
      const Row& r = rows[i];
      int ss[2] = {r.sp, r.sm};
      int pp[2] = {dpos[r.dp], r.kind == 0 ? dpos[r.dm] : -1};
      double sg[2] = {1.0, -1.0};
      const int ne2 = r.kind == 0 ? 2 : 1;
      for (int a = 0; a < ne2; ++a)
        for (int b = 0; b < ne2; ++b)
          for (int k = 0; k < 3; ++k)
            for (int l = 0; l < 3; ++l)
              GG[(size_t)(3 * ss[b] + l) * nc + 3 * ss[a] + k] +=
                  sg[a] * Rb[k * nb + pp[a]] * sg[b] * Rb[l * nb + pp[b]];
    }
    std::vector<double> a = GG;
    std::vector<int> perm;
    int rank = 0;
    pivoted_cholesky_host(a, nc, 1e-10, perm, rank);
    std::vector<int> kept(perm.begin(), perm.begin() + rank);
    std::sort(kept.begin(), kept.end());
    n_kept = rank;
    // Cholesky + explicit inverse of the kept block
    std::vector<double> L((size_t)rank * rank, 0.0);
    for (int j = 0; j < rank; ++j)
      for (int i = j; i < rank; ++i) L[(size_t)j * rank + i] = GG[(size_t)kept[j] * nc + kept[i]];
    for (int j = 0; j < rank; ++j) {
      double d = L[(size_t)j * rank + j];
      for (int k = 0; k < j; ++k) d -= L[(size_t)k * rank + j] * L[(size_t)k * rank + j];
      if (!(d > 0.0)) fail(FETIGPU_E_COARSE_SINGULAR, "filtered G G^T is not SPD");
      const double l = std::sqrt(d);
      L[(size_t)j * rank + j] = l;
      for (int i = j + 1; i < rank; ++i) {
        double v = L[(size_t)j * rank + i];
        for (int k = 0; k < j; ++k) v -= L[(size_t)k * rank + i] * L[(size_t)k * rank + j];
        L[(size_t)j * rank + i] = v / l;
      }
    }
    H.assign((size_t)nc * nc, 0.0);
    std::vector<double> col(rank);
    for (int c = 0; c < rank; ++c) {
      std::fill(col.begin(), col.end(), 0.0);
      col[c] = 1.0;
      for (int j = 0; j < rank; ++j) {
        double v = col[j];
        for (int k = 0; k < j; ++k) v -= L[(size_t)k * rank + j] * col[k];
        col[j] = v / L[(size_t)j * rank + j];
      }
      for (int j = rank - 1; j >= 0; --j) {
        double v = col[j];
        for (int k = j + 1; k < rank; ++k) v -= L[(size_t)j * rank + k] * col[k];
        col[j] = v / L[(size_t)j * rank + j];
      }
      for (int j = 0; j < rank; ++j) H[(size_t)kept[c] * nc + kept[j]] = col[j];
    }
  } else {
    // FETI-DP split: D (prescribed, eliminated), c (corners), r (rest)
    // primal numbering over the partition vertices only: (vertex row, col, dir)
    std::vector<int> cidx(2 * (size_t)(sx + 1) * (sy + 1), -1);
    auto cid = [&](int gx, int gy, int dir) -> int& {
      return cidx[2 * ((size_t)(gy / n) * (sx + 1) + gx / n) + dir];
    };
    Nc = 0;
    for (int gy = 0; gy < GY; gy += n)
      for (int gx = 0; gx < GX; gx += n) {
        const int g = gy * GX + gx;
        for (int dir = 0; dir < 2; ++dir)
          if (!presc[2 * g + dir]) cid(gx, gy, dir) = Nc++;
      }
    c_owners.assign(Nc, {});
    for (int s = 0; s < Ns; ++s) {
      SubPlan& S = subs[s];
      S.r.clear(); S.c.clear(); S.cg.clear(); S.D.clear(); S.gD.clear();
      for (int i = 0; i < nb; ++i) {
        const int d = perim_dof[i], v = d / 2, dir = d % 2;
        const int gx = S.si * n + v % nn, gy = S.sj * n + v / nn, g = gy * GX + gx;
        if (presc[2 * g + dir]) { S.D.push_back(i); S.gD.push_back(pval(2 * (long long)g + dir)); }
        else if (corner(gx, gy)) { S.c.push_back(i); S.cg.push_back(cid(gx, gy, dir)); }
        else S.r.push_back(i);
      }
      if (S.c.empty() && S.D.empty()) fail(FETIGPU_E_INSUFFICIENT_CORNERS, "subdomain has no primal DOF");
      for (size_t a = 0; a < S.c.size(); ++a) c_owners[S.cg[a]].push_back({s, (int)a});
      std::vector<int> ridx(nb, -1);
      for (size_t i = 0; i < S.r.size(); ++i) ridx[S.r[i]] = (int)i;
      S.Top = S.T;
      for (int t : S.T)
        if (ridx[t] < 0) fail(FETIGPU_E_STATE, "touched DOF outside the remainder set");
      std::vector<int> key{S.design, -1};
      key.insert(key.end(), S.r.begin(), S.r.end());
      key.push_back(-2);
      key.insert(key.end(), S.c.begin(), S.c.end());
      key.push_back(-3);
      key.insert(key.end(), S.T.begin(), S.T.end());
      auto it = op_key.find(key);
      if (it == op_key.end()) {
        SlotFront sf;
        sf.design = S.design;
        sf.src = S.r;
        sf.src.insert(sf.src.end(), S.c.begin(), S.c.end());
        sf.ne = (int)S.r.size();
        for (int t : S.T) sf.ext.push_back(ridx[t]);
        op_slots.push_back(sf);
        it = op_key.emplace(key, (int)op_slots.size() - 1).first;
      }
      S.op_slot = it->second;
    }
  }

  hm.mark("op slots / coarse");
  // ---- preconditioner slots
  for (int s = 0; s < Ns; ++s) {
    SubPlan& S = subs[s];
    std::vector<int> key{S.design};
    key.insert(key.end(), S.T.begin(), S.T.end());
    if (precond == FETIGPU_DIRICHLET) {
      // F = domain boundary set (perimeter, or r for FETI-DP) minus T
      std::vector<int> dom;
      if (dp) dom = S.r;
      else { dom.resize(nb); std::iota(dom.begin(), dom.end(), 0); }
      std::vector<int> Fset;
      for (int v : dom)
        if (!std::binary_search(S.T.begin(), S.T.end(), v)) Fset.push_back(v);
      key.push_back(-1);
      key.insert(key.end(), Fset.begin(), Fset.end());
      auto it = pc_key.find(key);
      if (it == pc_key.end()) {
        SlotFront sf;
        sf.design = S.design;
        sf.src = Fset;
        sf.src.insert(sf.src.end(), S.T.begin(), S.T.end());
        sf.ne = (int)Fset.size();
        pc_slots.push_back(sf);
        it = pc_key.emplace(key, (int)pc_slots.size() - 1).first;
      }
      S.pc_slot = it->second;
    } else {
      auto it = pc_key.find(key);
      if (it == pc_key.end()) {
        pc_lumped_T.push_back(S.T);
        pc_lumped_design.push_back(S.design);
        it = pc_key.emplace(key, (int)pc_lumped_T.size() - 1).first;
      }
      S.pc_slot = it->second;
    }
  }
  hm.mark("preconditioner slots");
}

}  // namespace fg
