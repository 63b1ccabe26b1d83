/*
 * fetigpu.h -- C-ABI of the B200-native FETI dual-operator engine.
 *
 * This is the drop-in boundary for the hot path of arxiv 2111.11728's FETI
 * solvers.  The reference declares its solver entry points as
 * SPEC contracts over the building blocks in proj/include/feti; each function
 * below replaces one of them (file:line of the interface it stands in for):
 *
 *   fetigpu_create/build   build_partition + assemble_subdomain +
 *                          apply_traction + build_constraints +
 *                          build_coarse_space + k_scaling + build_tfeti /
 *                          build_fetidp + dirichlet_schur/lumped
 *                          (decomposition.hpp:47-180, fem.cpp:86-167,
 *                           SPEC.md:288-309,360-377)
 *   fetigpu_apply_F        DualOperator::apply / TfetiSystem action
 *                          F = sum_s B_s K_s^+ B_s^T (per
 *                          subdomain SemidefiniteCholesky::solve_unchecked,
 *                          linalg.hpp:113-114 + ConstraintSet::apply_BsT /
 *                          accumulate_Bs, decomposition.hpp:98-101) and the
 *                          condensed FETI-DP operator
 *   fetigpu_apply_precond  apply_coarse_preconditioner
 *   fetigpu_project        CoarseSpace::project / project_block
 *                          (decomposition.hpp:136-138)
 *   fetigpu_rhs            d = B K^+ f - c, lambda0 = G^T (G G^T)^{-1} e
 *                          (decomposition.hpp:139-140) /
 *                          FETI-DP rhs
 *   fetigpu_solve          pcg / simultaneous_pcg
 *   fetigpu_recover        recover_primal
 *
 * Conventions: plain pointers and sizes, no C++ or torch types.  Host
 * pointers are borrowed for the duration of the call; *_device variants take
 * device pointers and run on the context's stream.  Every function returns
 * 0 on success or an error code mapped 1:1 to proj/include/feti/errors.hpp
 * (FETIGPU_E_*).  Non-convergence is not an error: it is reported in
 * fetigpu_trace.status.  A context is not reentrant
 * (one call in flight per context); distinct contexts may be
 * used from different host threads.
 */
#ifndef FETIGPU_H
#define FETIGPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes (errors.hpp:7-69, in declaration order) */
enum {
  FETIGPU_OK = 0,
  FETIGPU_E_NOT_POSITIVE_DEFINITE = 1,
  FETIGPU_E_INDEFINITE_INPUT = 2,
  FETIGPU_E_INCOMPATIBLE_RHS = 3,
  FETIGPU_E_EDGE_NOT_ON_BOUNDARY = 4,
  FETIGPU_E_DIMENSION_MISMATCH = 5,
  FETIGPU_E_NODE_NOT_FOUND = 6,
  FETIGPU_E_INSUFFICIENT_CORNERS = 7,
  FETIGPU_E_ZERO_STIFFNESS_DIAGONAL = 8,
  FETIGPU_E_SINGULAR_INTERIOR = 9,
  FETIGPU_E_COARSE_SINGULAR = 10,
  FETIGPU_E_SINGULAR_REMAINDER = 11,
  FETIGPU_E_SINGULAR_COARSE = 12,
  FETIGPU_E_SINGULAR_GLOBAL = 13,
  FETIGPU_E_NEGATIVE_INNER_PRODUCT = 14,
  FETIGPU_E_NOT_CONVERGED = 15,
  FETIGPU_E_STATE_SOLVE_FAILED = 16,
  FETIGPU_E_CONFIG = 17,
  FETIGPU_E_IO = 18,
  FETIGPU_E_INVALID_ARGUMENT = 20, /* std::invalid_argument in fem.cpp */
  FETIGPU_E_DOMAIN = 21,           /* std::domain_error in fem.cpp */
  FETIGPU_E_CUDA = 100,
  FETIGPU_E_NO_DEVICE = 101,
  FETIGPU_E_OUT_OF_MEMORY = 102,
  FETIGPU_E_STATE = 103            /* call order violated (e.g. apply before build) */
};

enum { FETIGPU_TFETI = 0, FETIGPU_FETIDP = 1 };
enum { FETIGPU_MULTIPLICITY = 0, FETIGPU_KSCALING = 1 };
enum { FETIGPU_LUMPED = 0, FETIGPU_DIRICHLET = 1, FETIGPU_SUPERLUMPED = 2 };
enum { FETIGPU_SINGLE = 0, FETIGPU_FO = 1, FETIGPU_RRS = 2 };
enum { FETIGPU_CONVERGED = 0, FETIGPU_MAX_ITER = 1, FETIGPU_BREAKDOWN = 2 };

typedef struct fetigpu_ctx fetigpu_ctx;

/* Problem description: partition (decomposition.hpp:13-48), material
 * (fem.hpp:12-20), per-design densities keyed by module_type (the reference's
 * factorization cache key), Dirichlet supports
 * (decomposition.hpp:50-54), edge tractions (fem.hpp:90-99) and nodal point
 * loads (lowest-index owner copy).  Loads must lie on module perimeters. */
typedef struct fetigpu_problem {
  int sx, sy, n;
  double hx, hy;
  double E0, Emin, nu, p, thickness;
  int n_designs;
  const double* densities;   /* n_designs * n * n, row-major from the bottom row */
  const int* module_type;    /* sx*sy, design index per subdomain (sj*sx + si) */
  int n_dirichlet;
  const int* dir_gnode;
  const int* dir_dir;
  const double* dir_value;
  int n_tractions;
  const int* tr_sub;
  const int* tr_side;        /* 0 left, 1 right, 2 bottom, 3 top */
  const int* tr_first;
  const int* tr_count;
  const double* tr_txy;      /* 2 per traction */
  int n_point_loads;
  const int* pl_gnode;
  const int* pl_dir;
  const double* pl_value;
  int method;                /* FETIGPU_TFETI | FETIGPU_FETIDP */
  int scaling;               /* FETIGPU_MULTIPLICITY | FETIGPU_KSCALING */
  int precond;               /* FETIGPU_LUMPED | FETIGPU_DIRICHLET | FETIGPU_SUPERLUMPED */
} fetigpu_problem;

/* SolveOptions */
typedef struct fetigpu_solve_opts {
  double tol;
  int rel;                   /* 1: eps_r(i)/eps_r(0) <= tol */
  int max_it;
  int directions;            /* FETIGPU_SINGLE | FETIGPU_FO | FETIGPU_RRS */
  double pivot_tol;          /* rank-revealing Cholesky tolerance, default 1e-12 */
  int reorth_passes;         /* classical Gram-Schmidt passes, default 2 */
} fetigpu_solve_opts;

/* ConvergenceTrace; arrays are caller-owned (cap entries) */
typedef struct fetigpu_trace {
  int status;
  int iterations;
  int f_applies;
  double eps0, eps_final;
  int cap;
  double* eps;
  int* kept;
  int* f_app;
  double solve_ms;           /* device time of the iteration loop */
  /* RRS device time per phase (ms, summed over iterations): F W, Gram,
   * pivoted Cholesky, compression, gamma/lambda/r update, preconditioner +
   * metric, projection of Z, re-orthogonalization */
  double phase_ms[8];
} fetigpu_trace;

/* Build statistics and the per-apply algorithmic work. */
typedef struct fetigpu_stats {
  int m, n_sub, local_dofs, n_c, n_kept, n_iface, max_ns, n_designs;
  int n_op_slots, n_pc_slots;
  double op_bytes;           /* F-apply GEMV algorithmic bytes per apply */
  double op_flops_per_col;   /* block F-apply flops per column */
  double main_kernel_bytes;  /* bytes of the dominant apply kernel (F_s stream) */
  double build_ms;           /* device time of fetigpu_build */
  double nd_ms, slot_ms, coarse_ms;
  double device_bytes;       /* device memory held by the context */
  int host_pipeline;         /* 1: fetigpu_apply_F overlaps the H2D of x with the GEMV */
  /* loop of the last PCG / FO solve: 0 host-driven, 1 CUDA-graph while loop,
   * 2 persistent kernel with a grid barrier, 3 persistent kernel as one
   * thread-block cluster (K15) */
  int solve_loop;
  /* bytes one F-apply must stream with symmetric operator storage: the
   * symmetric-packed F_s tiles when the packed kernel runs (else 8 n_s^2),
   * A_bc read in both phases, the coarse inverse (packed tiles or dense),
   * lambda read + y written and the gather lists -- the roofline bytes of
   * the apply actually executed (op_bytes counts full F_s storage). */
  double stream_bytes;
  /* dominant apply kernel: 0 full-matrix GEMV (k_gather_gemv_scatter), 1
   * symmetric-packed tiles by LDG (k_sym_gemv_scatter), 2 symmetric-packed
   * tiles by TMA bulk copies into per-warp mbarrier rings on a persistent
   * grid (k_sym_gemv_tma); apply_ring = ring slots per warp of the latter */
  int apply_kernel, apply_ring;
} fetigpu_stats;

/* Select the CUDA device used by contexts built afterwards from this host
 * thread (one process per GPU: the rank's local device). */
int fetigpu_set_device(int device);
int fetigpu_create(const fetigpu_problem* p, fetigpu_ctx** out);
int fetigpu_build(fetigpu_ctx* ctx);
void fetigpu_destroy(fetigpu_ctx* ctx);
const char* fetigpu_last_error(void);
int fetigpu_stats_get(const fetigpu_ctx* ctx, fetigpu_stats* st);

/* ConstraintSet rows (decomposition.hpp:58-108): kind 0 interface pair, 1
 * Dirichlet; weights are the plus/minus sides of the scaled jump operator. */
int fetigpu_rows(const fetigpu_ctx* ctx, int* kind, int* sub_plus, int* dof_plus,
                 int* sub_minus, int* dof_minus, double* gap, int* mult,
                 double* w_plus, double* w_minus);

/* y = F x for ncols columns of length m (column stride ld >= m). */
int fetigpu_apply_F(fetigpu_ctx* ctx, const double* x, double* y, int ncols, int ld);
int fetigpu_apply_F_device(fetigpu_ctx* ctx, const double* x, double* y, int ncols, int ld);
/* z = sum_s Bt_s St_s Bt_s^T r; Zcols (m x N_s, column-major) optional */
int fetigpu_apply_precond(fetigpu_ctx* ctx, const double* r, double* z, double* Zcols);
int fetigpu_apply_precond_device(fetigpu_ctx* ctx, const double* r, double* z, double* Zcols);
/* v <- P v in place for ncols columns (identity for FETI-DP) */
int fetigpu_project(fetigpu_ctx* ctx, double* v, int ncols, int ld);
int fetigpu_project_device(fetigpu_ctx* ctx, double* v, int ncols, int ld);
int fetigpu_rhs(fetigpu_ctx* ctx, double* d, double* lambda0);
int fetigpu_solve(fetigpu_ctx* ctx, const fetigpu_solve_opts* o, double* lambda,
                  fetigpu_trace* tr);
/* pcg / simultaneous_pcg from a given lambda0 (host, length m) instead of
 * the default start (FETI-DP: 0; T-FETI: G^T (G G^T)^{-1} e):
 * the SIMP loop's warm start from the previous snapshot's multipliers
 * (SURVEY.md 8f rank 2).  T-FETI projects it onto G lambda = e. */
int fetigpu_solve_warm(fetigpu_ctx* ctx, const fetigpu_solve_opts* o, const double* lambda0, double* lambda,
                       fetigpu_trace* tr);
/* Next density snapshot of the same problem (same partition, module size,
 * design count, supports, loads and method): host setup and device build
 * again, operator storage reused through the context's block cache (no
 * cudaFree / cudaMalloc of the multi-GB operator storage).  The SIMP outer
 * loop calls this once per optimization iteration. */
int fetigpu_rebuild(fetigpu_ctx* ctx, const fetigpu_problem* p);
/* RRS direction store (no reference counterpart: the reference's
 * simultaneous_pcg keeps W_j, Q_j densely).  EXPLICIT: that
 * dense store, 2 m rank_j doubles per iteration.  IMPLICIT (FETI-DP only):
 * each W_j kept as coefficients over the packed per-subdomain preconditioner
 * blocks, Q_j never stored, three block F-applies per iteration.  AUTO
 * (default): implicit for FETI-DP when N_s >= 256 and m > 32 N_s, or when 32
 * iterations of the explicit store would not fit in free device memory;
 * explicit otherwise and always for T-FETI.  Env override FETIGPU_RRS_STORE=explicit|implicit
 * applies under AUTO. */
enum { FETIGPU_RRS_STORE_AUTO = 0, FETIGPU_RRS_STORE_EXPLICIT = 1, FETIGPU_RRS_STORE_IMPLICIT = 2 };
int fetigpu_set_rrs_store(fetigpu_ctx* ctx, int mode);
/* u: N_s x local DOFs (2(n+1)^2 per subdomain, node-major x/y) */
int fetigpu_recover(fetigpu_ctx* ctx, const double* lambda, double* u);

/* Explicit local operator of subdomain s on its touched DOFs (test hook):
 * writes n_s, the local DOF ids (ns) and the dense n_s x n_s F_s. */
int fetigpu_local_operator(fetigpu_ctx* ctx, int s, int* ns, int* dofs, double* F, int cap);

/* Block F-apply (K5, FP64 tensor cores): Q = F W for k columns stored
 * row-major (W(i,c) = W[i*ldw + c]), device pointers, ctx stream. */
int fetigpu_apply_F_block_device(fetigpu_ctx* ctx, const double* W, int ldw, double* Q, int ldq, int k);
/* Subdomain-sharded apply (one rank of a row-band partition
 * of the module grid, exchanges done by the caller: paper_2111_11728_b200/
 * shard.py over torch.distributed).  The context applies only subdomains
 * [s0, s1).  phase1: y := partial sum over the owned subdomains (T-FETI F or
 * the preconditioner: complete except on rows shared with another rank;
 * FETI-DP F: nothing yet) and, for FETI-DP F, the owned t_s = A''_s^T x_s
 * written into the zeroed tot_c vector tout.  After the caller sums tout over
 * ranks, phase2 adds the coarse correction and the local parts for the owned
 * subdomains; summing y over ranks on the shared rows completes F x.  Every
 * dual row has two owners, so the N-rank result equals the 1-GPU apply bit
 * for bit.  Device pointers, context stream. */
int fetigpu_shard_set_range(fetigpu_ctx* ctx, int s0, int s1);
int fetigpu_shard_info(const fetigpu_ctx* ctx, int* tot_c);
int fetigpu_shard_phase1_device(fetigpu_ctx* ctx, const double* x, double* y, double* tout, int precond);
int fetigpu_shard_phase2_device(fetigpu_ctx* ctx, const double* tall, double* y);
/* Invariant check of the device solver (test hook): when
 * on, every FO / RRS solve afterwards reconstructs its stored F-normalised
 * search directions W and reports max |W^T F W - I| over all of them (FO
 * conjugacy and Alg. 1 orthonormality) and their number. */
int fetigpu_set_check(fetigpu_ctx* ctx, int on);
int fetigpu_check_result(const fetigpu_ctx* ctx, double* err, int* n);
/* Test hook: Q = F Z for a fresh per-subdomain preconditioner block Z
 * (row-major m x N_s, column s supported on subdomain s's dual rows) through
 * the sparse-aware K5z path the RRS solver uses on Alg. 1 lines 2/16 blocks;
 * host buffers.  FETIGPU_E_CONFIG when the problem lacks that structure. */
int fetigpu_apply_F_zblock(fetigpu_ctx* ctx, const double* Z, double* Q);
int fetigpu_time_apply_block(fetigpu_ctx* ctx, const double* W, double* Q, int k, int reps, double* ms);
/* Rank-revealing pivoted Cholesky, Alg. 1 line 9 -- replaces
 * feti::pivoted_cholesky (proj/include/feti/linalg.hpp:80, linalg.cpp:83-138)
 * with the SPEC.md:43-47 contract (symmetric trailing update):
 * N A N^T = L L^T, L = [[L~, 0], [X, 0]], pivots by largest remaining
 * diagonal (ties -> lowest index), stop when it is <= tol * max initial
 * diagonal.  a: n x n column-major symmetric (lower triangle read).  Outputs
 * perm[n] (pivot order), lower (n x n column-major; columns < *rank hold L,
 * the rest zero) and *rank.  Runs the device kernel the RRS solver uses.
 * FETIGPU_E_INDEFINITE_INPUT when a remaining diagonal is below -tol * scale. */
int fetigpu_pivoted_cholesky(const double* a, int n, double tol, int* perm, double* lower, int* rank);
/* Basis compression W N^T [L~^{-T}; 0], Alg. 1 lines 10-11 -- replaces
 * feti::PivotedCholesky::compress (linalg.hpp:79, linalg.cpp:131-138).
 * perm/lower/rank as returned by fetigpu_pivoted_cholesky (lower n x n
 * column-major); w: rows x n column-major; out: rows x rank column-major.
 * Same device operations as the RRS solver (L~^{-1} by a triangular solve
 * on the identity, column gather, triangular multiply). */
int fetigpu_pivoted_compress(const int* perm, const double* lower, int n, int rank, const double* w, int rows,
                             double* out);
/* Dense FP64 algebra of the engine (hand-written DMMA kernels, no cuBLAS):
 * C = alpha op(A) op(B) + beta C, column-major BLAS dgemm semantics on host
 * buffers (test hook).  flags: 1 lower-triangle tiles only (i >= j stored),
 * 2 / 4 / 8 triangular-operand K ranges (see csrc/dla.cuh GemmFlags), 256
 * deterministic split-K path. */
int fetigpu_dla_gemm(int ta, int tb, int M, int N, int K, double alpha, const double* A, long long lda,
                     const double* B, long long ldb, double beta, double* C, long long ldc, int flags);
/* X = L^{-1} (n x n, column-major, lower triangle of L read; X lower with
 * zeros above the diagonal): the L~^{-1} of Alg. 1 lines 10-11. */
int fetigpu_dla_tri_inv(const double* L, int n, long long ldl, double* X);
/* mean device time (ms) of `reps` M x N x K GEMMs on device-resident random operands */
int fetigpu_dla_time_gemm(int ta, int tb, int M, int N, int K, int reps, double* ms);
/* Measured FP64 issue peaks of this device (DMMA m8n8k4 and DFMA), TFLOP/s. */
int fetigpu_fp64_peak(double* tflops_dmma, double* tflops_dfma);
/* Measured read-only HBM bandwidth of this device (GB/s): `bytes` (at least
 * 256 MB, much larger than L2) streamed `reps` times by 16-byte loads.  The
 * ceiling of the F-apply's operator stream, which only reads; the copy figure
 * of MEASURED_PEAKS.json counts read + write bytes and is lower. */
int fetigpu_hbm_read_peak(size_t bytes, int reps, double* gbs);
/* DMMA fragment-layout self test: C (8x8 row-major) = A (8x4) B (4x8). */
int fetigpu_selftest_dmma(const double* A, const double* B, double* C);

/* Device memory / timing helpers for benchmarks (no torch on the path). */
int fetigpu_device_alloc(fetigpu_ctx* ctx, size_t bytes, void** ptr);
int fetigpu_device_free(fetigpu_ctx* ctx, void* ptr);
int fetigpu_host_alloc(size_t bytes, void** ptr);   /* pinned */
int fetigpu_host_free(void* ptr);
int fetigpu_memcpy(fetigpu_ctx* ctx, void* dst, const void* src, size_t bytes, int kind);
int fetigpu_fill_random(fetigpu_ctx* ctx, double* d_ptr, size_t count, unsigned long long seed);
int fetigpu_synchronize(fetigpu_ctx* ctx);
/* Device time per call (CUDA events, `reps` back-to-back calls after 3
 * warm-up, no L2 flush) of the three per-iteration operators: ms[0] F-apply,
 * ms[1] preconditioner, ms[2] projector (identity for
 * FETI-DP; decomposition.hpp:136 for T-FETI). */
int fetigpu_time_ops(fetigpu_ctx* ctx, int reps, double* ms);
/* Device memory of the current device: free and total bytes (cudaMemGetInfo),
 * and the bytes `ctx` (nullable) holds in its cache of freed RRS
 * direction-store chunks -- reused by its next solve, returned to the driver
 * by fetigpu_destroy.  Memory planning for the RRS store (SPEC.md:435-443:
 * two m x k blocks per iteration). */
int fetigpu_device_memory(fetigpu_ctx* ctx, size_t* free_bytes, size_t* total_bytes, size_t* cached_bytes);
/* Times `reps` device-resident applies of F on ncols columns with CUDA
 * events on the context stream; ms[0] = mean per apply, ms[1] = mean of the
 * dominant kernel, ms[2] = its share; launches[0] = kernels per apply. */
int fetigpu_time_apply(fetigpu_ctx* ctx, const double* d_x, double* d_y, int ncols,
                       int reps, int flush_l2, double* ms, int* launches);

#ifdef __cplusplus
}
#endif
#endif
