/*
 * feti_oracle.h -- C API of the CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is a plain C++ (no Eigen, no CUDA)
 * restatement of the reference's FETI hot path (arxiv 2111.11728,
 * /root/reference): the implicit dual operator F = sum_s B_s K_s^+ B_s^T
 * (proj/src/linalg.cpp:179-222 semidefinite solves), the
 * lumped / Dirichlet preconditioners, the T-FETI projector
 * (proj/include/feti/decomposition.hpp:123-148), the FETI-DP condensation
 * and the PCG / FO / RRS engine (SPEC.md:411-477,
 * PAPER.md Alg. 1).  It is the parity checker for the GPU library and the
 * timed CPU baseline of bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * (libfetigpu.so) never does.
 *
 * Parity pinning: the reference ships no executable tests or golden vectors
 * (SURVEY.md 8c); the oracle is pinned against every SPEC.md example that
 * touches this path (tests/test_oracle_*.py) and the derived known answers of
 * SURVEY.md Appendix B.  The Eigen boundary (SimplicialLLT ordering,
 * setFromTriplets) is restated, not linked: "parity unpinned at the Eigen
 * boundary" beyond those examples.
 */
#ifndef FETI_ORACLE_H
#define FETI_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as fetigpu_problem (include/fetigpu.h); declared separately so
 * the checker shares no code with the product. */
typedef struct fo_problem {
  int sx, sy, n;                 /* module grid and elements per module side */
  double hx, hy;
  double E0, Emin, nu, p, thickness;
  int n_designs;
  const double* densities;       /* n_designs * n * n, row-major from bottom row */
  const int* module_type;        /* sx*sy design index per subdomain (sj*sx+si) */
  int n_dirichlet;
  const int* dir_gnode;
  const int* dir_dir;
  const double* dir_value;
  int n_tractions;
  const int* tr_sub;
  const int* tr_side;            /* 0 left, 1 right, 2 bottom, 3 top (fem.hpp:88) */
  const int* tr_first;
  const int* tr_count;
  const double* tr_txy;          /* 2 per traction */
  int n_point_loads;
  const int* pl_gnode;
  const int* pl_dir;
  const double* pl_value;
  int method;                    /* 0 T-FETI, 1 FETI-DP */
  int scaling;                   /* 0 multiplicity, 1 k-scaling */
  int precond;                   /* 0 lumped, 1 Dirichlet, 2 super-lumped */
} fo_problem;

typedef struct fo_opts {
  double tol;          /* epsilon on eps_r (relative to eps_r(0) when rel) */
  int rel;             /* 1 relative mode */
  int max_it;
  int directions;      /* 0 single, 1 single + full orthogonalization, 2 RRS */
  double pivot_tol;    /* rank-revealing Cholesky tolerance */
  int reorth_passes;   /* SPEC.md:463, default 2 */
} fo_opts;

typedef struct fo_trace {
  int status;          /* 0 converged, 1 max_iter, 2 breakdown */
  int iterations;
  int f_applies;       /* operator applications (columns) incl. the initial residual */
  double eps0, eps_final;
  int cap;             /* capacity of the arrays below (caller-owned, may be 0) */
  double* eps;         /* eps_r per iteration, index 0 = initial */
  int* kept;           /* retained directions per iteration */
  int* f_app;          /* cumulative F applications */
} fo_trace;

/* error codes: identical numbering to include/fetigpu.h */
int fo_create(const fo_problem* p, void** out);
const char* fo_last_error(void);
/* accuracy-reference mode: local and coarse solves get two steps of
 * iterative refinement with long-double residuals (affects objects created
 * afterwards for the Phi / Kbar_cc build, and all later applications) */
void fo_set_refine(int on);
int fo_set_threads(int n);
/* invariant check of later FO / RRS solves: max |W^T F W - I| over the
 * stored F-normalised directions and their number */
void fo_set_check(int on);
void fo_check_result(double* err, int* n);
void fo_destroy(void* h);
/* info[0]=m, [1]=N_s, [2]=local DOFs, [3]=N_c (FETI-DP), [4]=kept coarse rows,
 * [5]=interface rows, [6]=max n_s (touched DOFs per subdomain) */
int fo_info(void* h, int* info);
int fo_rows(void* h, int* kind, int* sub_plus, int* dof_plus, int* sub_minus,
            int* dof_minus, double* gap, int* mult, double* w_plus, double* w_minus);
int fo_apply_F(void* h, const double* x, double* y);
int fo_apply_precond(void* h, const double* r, double* z, double* Zcols);
int fo_project(void* h, double* v);
int fo_rhs(void* h, double* d, double* lambda0);
int fo_solve(void* h, const fo_opts* o, double* lambda, fo_trace* tr);
int fo_recover(void* h, const double* lambda, double* u);
int fo_local_diag(void* h, double* diag);       /* N_s * local DOFs */
int fo_load_vectors(void* h, double* f);        /* N_s * local DOFs */
double fo_admissibility_error(void* h);
/* global direct oracle: merged global DOFs, band Cholesky;
 * u is written per subdomain copy (N_s * local DOFs). */
int fo_direct_solve(void* h, double* u);
int fo_local_apply(void* h, int s, const double* x, double* y);
double fo_coarse_residual(void* h, const double* lambda);
int fo_pseudo_solve(void* h, int s, const double* rhs, double* x);
int fo_fixed_dofs(void* h, int* out);

/* kernel-level entry points for the SPEC examples */
int fo_simp_modulus(double rho, double E0, double Emin, double p, double* out);
int fo_q4_element_stiffness(double nu, double thickness, double modulus,
                            double hx, double hy, double* k64 /* col-major */);
int fo_pivoted_cholesky(int n, const double* a /* col-major */, double tol,
                        int* perm, double* lower /* n*n col-major */, int* rank);
int fo_compress(int n, const int* perm, const double* lower, int rank, int rows,
                const double* w /* rows*n col-major */, double* out /* rows*rank */);
int fo_select_fixing_dofs(int rows, int cols, const double* basis, int* out);
int fo_rigid_body_modes(int n, double hx, double hy, double* R /* dof*3 col-major */);
int fo_band_cholesky_solve(int n, const double* a /* col-major SPD */, double* b);

#ifdef __cplusplus
}
#endif
#endif
