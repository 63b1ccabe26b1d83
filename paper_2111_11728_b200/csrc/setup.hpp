// setup.hpp -- host-side problem setup of the GPU engine.
//
// Everything here is index / weight bookkeeping that feeds the device once
// (SURVEY.md 3A "host C++ does everything up to the index/weight arrays,
// then crosses the host->device boundary once"): the regular partition, the
// signed Boolean constraint rows and gaps (decomposition.hpp:47-117), the
// scaling weights (decomposition.hpp:159-180), corner sets (:150-157), the
// T-FETI fixing DOFs (linalg.cpp:146-175) and natural coarse space G G^T
// (decomposition.hpp:123-148), plus the plans for the device build: the
// nested-dissection Schur tree of one module and the per-subdomain local
// operator "slots" (deduplicated by design and index pattern).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fetigpu.h"

namespace fg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int c, const std::string& m) { throw Error(c, m); }

struct Row {  // ConstraintRow (decomposition.hpp:58-70)
  int kind;   // 0 interface pair, 1 Dirichlet
  int sp, dp, sm, dm;
  double gap;
  int mult, gnode, dir;
};

// Nested-dissection Schur tree of one n x n module.  Every tree node owns a
// dense frontal matrix over [eliminated DOFs | perimeter DOFs]; leaves are
// assembled from elements, merges from their two children's Schur blocks.
struct NdNode {
  int x0, x1, y0, y1;
  int child[2] = {-1, -1};
  int height = 0;
  int nf = 0, ne = 0;
  bool leaf = false;
  std::vector<int> dofs;      // frontal DOF list as module-local DOF ids
  std::vector<int> elems;     // leaf: element ids (ey*n+ex), ey-major
  std::vector<int> emap;      // leaf: 8 frontal indices per element
  std::vector<int> cmap[2];   // merge: child perimeter index -> frontal index
  long long off = 0;          // frontal offset within its height block (per design)
  long long foff = 0;         // factor offset (nf*ne block) per design
};

struct NdPlan {
  int n = 0;
  std::vector<NdNode> nodes;
  int root = -1;
  int max_height = 0;
  std::vector<std::vector<int>> by_height;
  std::vector<long long> height_stride;   // doubles per design per height
  long long factor_stride = 0;            // doubles per design
  std::vector<int> topdown;               // pre-order for back substitution
};

// A batched dense frontal elimination built from a design's boundary Schur
// complement S (8n x 8n, perimeter order): frontal = [[S[src,src], E],[E^T,0]]
// with identity columns E[ext[j], j] = 1; the first ne DOFs are eliminated.
struct SlotFront {
  int design = 0;
  int ne = 0;
  std::vector<int> src;   // perimeter positions
  std::vector<int> ext;   // frontal row (index into src) of each identity column
  int nf() const { return (int)(src.size() + ext.size()); }
};

struct SubPlan {
  int si = 0, sj = 0, design = 0;
  int op_slot = -1, pc_slot = -1, fac_slot = -1;
  std::vector<int> T;          // touched perimeter positions (ascending): preconditioner / projector
  std::vector<int> Top;        // operator support (T minus fixed DOFs for T-FETI), slot order
  std::vector<int> c;          // FETI-DP: primal perimeter positions (slot order)
  std::vector<int> cg;         // FETI-DP: global primal ids
  std::vector<int> D;          // FETI-DP: eliminated (prescribed) perimeter positions
  std::vector<double> gD;      // their values
  std::vector<int> r;          // FETI-DP: remainder perimeter positions (ascending)
  std::vector<double> f;       // load on the perimeter (8n), node-major x/y in perimeter order
};

struct Setup {
  // problem
  int sx = 0, sy = 0, n = 0, nn = 0, Ns = 0, nloc = 0, nb = 0, GX = 0, GY = 0;
  int method = 0, scaling = 0, precond = 0, n_designs = 0;
  double hx = 1, hy = 1, E0 = 1, Emin = 1e-9, nu = 0.3, p = 3, thickness = 1;
  std::vector<double> densities;
  std::vector<int> module_type;
  double kunit[64];
  // perimeter of a module (the root perimeter of the ND tree)
  std::vector<int> perim_dof;  // nb = 8n local DOF ids
  std::vector<int> dpos;       // local DOF -> perimeter position or -1
  // constraints
  std::vector<Row> rows;
  int m = 0, n_iface = 0;
  std::vector<double> wplus, wminus;
  std::vector<double> gap;
  // per subdomain
  std::vector<SubPlan> subs;
  std::vector<std::vector<double>> bdiag;   // per design: diag K at perimeter DOFs
  // T-FETI
  std::vector<int> fixed_pos;               // 3 perimeter positions
  std::vector<double> Rb;                   // nb x 3 rigid modes at perimeter DOFs (col-major)
  std::vector<double> Rfull;                // nloc x 3
  std::vector<double> H;                    // 3Ns x 3Ns padded (G_k G_k^T)^{-1}
  int n_kept = 0;
  // FETI-DP
  int Nc = 0;
  std::vector<std::vector<std::pair<int, int>>> c_owners;  // per primal dof: (sub, local c idx) ascending
  // slots
  std::vector<SlotFront> op_slots, pc_slots;  // pc_slots only for Dirichlet
  std::vector<std::vector<int>> pc_lumped_T;  // lumped: per pc slot the T list
  std::vector<int> pc_lumped_design;
  std::vector<int> fac_slot_op;               // factor slot -> op slot providing L
  // ND plan
  NdPlan nd;

  void load(const fetigpu_problem& p);
  int owners(int gx, int gy, int* sub, int* lnode) const;
};

void pivoted_cholesky_host(std::vector<double>& a, int n, double tol, std::vector<int>& perm,
                           int& rank);

}  // namespace fg
