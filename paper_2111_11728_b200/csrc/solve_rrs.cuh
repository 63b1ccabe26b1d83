// solve_rrs.cuh -- Rank-Revealing Simultaneous FETI (Alg. 1): pivoted Cholesky launchers
// and the block iteration.
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include "ctx.cuh"

namespace fg {

// Launch the cluster pivoted Cholesky with the smallest cluster whose
// distributed shared memory holds the n x n Gram matrix; false if none fits
// (n > kPivcholClusterMaxN or the cluster cannot be scheduled).
template <int CL>
static bool pivchol_cluster_try(double* A, int n, double tol, int* perm, int* rank, int* status, double* gx,
                                cudaStream_t st) {
  const int R = (n + CL - 1) / CL;
  const size_t smem = ((size_t)R * n + 3 * (size_t)n) * 8;
  if (smem > 225 * 1024) return false;
  // per instantiation: attributes set and cluster schedulable (-1 unknown).
  // Atomic: contexts may be driven from several host threads; a duplicated
  // first probe is harmless (same attribute values).
  static std::atomic<int> ok{-1};
  if (ok.load() < 0) {
    if (cudaFuncSetAttribute(k_pivchol_cl<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024) !=
        cudaSuccess) { cudaGetLastError(); ok.store(0); return false; }
    if (CL > 8 && cudaFuncSetAttribute(k_pivchol_cl<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                      cudaSuccess) { cudaGetLastError(); ok.store(0); return false; }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 225 * 1024;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = CL > 1 ? 1 : 0;
    int nclusters = 1;
    if (CL > 1 && cudaOccupancyMaxActiveClusters(&nclusters, k_pivchol_cl<CL>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      nclusters = 0;
    }
    ok.store(nclusters > 0 ? 1 : 0);
  }
  if (!ok.load()) return false;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CL > 1 ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, k_pivchol_cl<CL>, A, n, tol, perm, rank, status, gx));
  return true;
}

static bool launch_pivchol_cluster(double* A, int n, double tol, int* perm, int* rank, int* status, double* gx,
                                   cudaStream_t st) {
  if (n > kPivcholClusterMaxN) return false;
  return pivchol_cluster_try<1>(A, n, tol, perm, rank, status, gx, st) ||
         pivchol_cluster_try<2>(A, n, tol, perm, rank, status, gx, st) ||
         pivchol_cluster_try<4>(A, n, tol, perm, rank, status, gx, st) ||
         pivchol_cluster_try<8>(A, n, tol, perm, rank, status, gx, st) ||
         pivchol_cluster_try<16>(A, n, tol, perm, rank, status, gx, st);
}

// Alg. 1 line 9 on a symmetric n x n matrix already in device memory (full
// storage): the cluster kernel when the matrix fits distributed shared memory,
// else the cooperative-grid kernel.  Scratch: ctl 4 ints, gx n + 64 doubles.
static void launch_pivchol(double* A, int n, double tol, int* perm, int* rank, int* status, int* ctl, double* gx,
                           cudaStream_t st) {
  if (launch_pivchol_cluster(A, n, tol, perm, rank, status, gx, st)) return;
  static std::atomic<int> coop_blocks{0};  // (see pivchol_cluster_try: benign duplicated init)
  if (!coop_blocks.load()) {
    int dev = 0, sms = 0, per_sm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pivchol_coop, 512, 0));
    coop_blocks = sms * std::max(1, std::min(per_sm, 2));
  }
  void* args[] = {&A, &n, &tol, &perm, &rank, &status, &ctl};
  CK(cudaLaunchCooperativeKernel((void*)k_pivchol_coop, dim3(coop_blocks.load()), dim3(512), args, 0, st));
}

// Rank-Revealing Simultaneous FETI, Alg. 1 of PAPER.md:302-351:
// one search direction per subdomain, Delta = Q^T W factorized by the
// rank-revealing Cholesky, W, Q compressed to F-orthonormal columns, and the
// new block re-orthogonalized against all stored blocks (CGS, 2 passes).
// Blocks are row-major (m x k, k fastest) so the K5 block apply gathers and
// scatters whole contiguous rows; cuBLAS sees them as column-major k x m.
int Ctx::solve_rrs(const fetigpu_solve_opts& o, double* lambda_host, fetigpu_trace* tr) {
  const int m = su.m, Ns = su.Ns;
  const int passes = std::max(1, o.reorth_passes);
  PhaseTimer pt;
  rhs();
  pt.mark("rrs rhs", st);
  // Two m x N_s row-major work blocks only: W (directions; the preconditioner
  // writes its columns straight into it, Alg. 1 lines 2/16-17) and Qb = F W.
  // The compression gathers go into the free arena tail and into W.
  DBuf<double> lam, r, z, q, tmp, W, Qb, Delta, gamma;
  DBuf<int> perm, rank_d, ctl;
  DBuf<Scal> sc;
  DBuf<double> Linv;
  lam.alloc(m); r.alloc(m); z.alloc(m); q.alloc(m); tmp.alloc(m);
  W.alloc((size_t)m * Ns); Qb.alloc((size_t)m * Ns);
  ctl.alloc(4);
  DBuf<double> pivx;
  pivx.alloc((size_t)Ns + 64);
  Linv.alloc((size_t)Ns * Ns);
  Delta.alloc((size_t)Ns * Ns); gamma.alloc(Ns);
  perm.alloc(Ns); rank_d.alloc(1);
  sc.alloc(1);
  sc.zero(st);
  // Stored F-orthonormal directions W_j and Q_j = F W_j (m x rank_j column-
  // major blocks, ld m) packed side by side into a few large chunks, so the
  // re-orthogonalization against every stored block is one GEMM pair per
  // chunk per pass.  Chunk capacity doubles the store (O(log K) chunks, no
  // copies) and is clamped to the free device memory.
  struct Chunk {
    std::unique_ptr<DBuf<double>> w, q, psi;  // psi: this chunk's rows of Psi (cap x Ns, ld cap)
    int cap, used, off;
  };
  std::vector<Chunk> chunks;
  int K = 0;
  const char* tenv0 = getenv("FETIGPU_TRACE");
  const bool trace_alloc = tenv0 && tenv0[0] == '1';
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto tms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  auto append_slot = [&](int rank, double** wn, double** qn) {
    if (chunks.empty() || chunks.back().used + rank > chunks.back().cap) {
      const auto t0 = tnow();
      size_t freeb = dev_free_bytes(&rrs_cache), total = 0, fr0 = 0;
      CK(cudaMemGetInfo(&fr0, &total));
      const auto t1 = tnow();
      const size_t margin = std::max<size_t>(size_t(1) << 30, total / 64);
      const long long fit = freeb > margin ? (long long)((freeb - margin) / (16.0 * m)) : 0;
      const int c = (int)std::min<long long>(std::max(rank, std::max(Ns, K)), fit);
      if (c < rank)
        fail(FETIGPU_E_OUT_OF_MEMORY, "RRS: out of device memory for the stored directions (K = " +
                                          std::to_string(K + rank) + " columns of length m = " + std::to_string(m) +
                                          ")");
      Chunk ch{std::unique_ptr<DBuf<double>>(new DBuf<double>), std::unique_ptr<DBuf<double>>(new DBuf<double>),
               std::unique_ptr<DBuf<double>>(new DBuf<double>), c, 0, K};
      ch.w->cache = ch.q->cache = ch.psi->cache = &rrs_cache;
      ch.w->alloc((size_t)m * c);
      const auto t2 = tnow();
      ch.q->alloc((size_t)m * c);
      ch.psi->alloc((size_t)c * Ns);
      const auto t3 = tnow();
      chunks.push_back(std::move(ch));
      if (trace_alloc)
        fprintf(stderr, "[fetigpu] rrs store chunk %zu: %d cols (%.0f MB x 2): meminfo %.2f ms, W %.2f ms, Q %.2f ms\n",
                chunks.size(), c, (double)m * c * 8 / 1e6, tms(t0, t1), tms(t1, t2), tms(t2, t3));
    }
    Chunk& ch = chunks.back();
    *wn = ch.w->p + (size_t)ch.used * m;
    *qn = ch.q->p + (size_t)ch.used * m;
    ch.used += rank;
  };
  Scal* hs = nullptr;
  CK(cudaMallocHost(&hs, sizeof(Scal)));
  std::unique_ptr<Scal, decltype(&cudaFreeHost)> hs_guard(hs, cudaFreeHost);
  const double one = 1.0, mone = -1.0, zero = 0.0;
  pt.mark("rrs setup", st);
  CK(cudaEventRecord(ev0, st));
  CK(cudaMemcpyAsync(lam.p, d_lam0.p, m * 8, cudaMemcpyDeviceToDevice, st));
  apply_F(lam.p, q.p, 1, m, m);
  int fapp = 1;
  k_sub<<<grid_for(m), kThreads, 0, st>>>(m, d_d.p, q.p, r.p);
  project(r.p, 1, m);
  apply_precond(r.p, z.p, W.p, true);  // Alg. 1 line 2 (columns) and z = Z 1
  dots({{r.p, z.p}, {r.p, r.p}, {z.p, z.p}}, &sc.p->rz);
  CK(cudaMemcpyAsync(hs, sc.p, sizeof(Scal), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  auto metric = [&](const Scal& s) {
    if (s.rz < -1e-14 * std::sqrt(s.rr) * std::sqrt(s.zz))
      fail(FETIGPU_E_NEGATIVE_INNER_PRODUCT, "r^T z < 0: preconditioner is not symmetric positive");
    return std::sqrt(std::max(s.rz, 0.0));
  };
  const double eps0 = metric(*hs);
  double eps = eps0;
  int it = 0, status = FETIGPU_MAX_ITER;
  auto push = [&](double e, int kept) {
    if (tr && it < tr->cap) {
      if (tr->eps) tr->eps[it] = e;
      if (tr->kept) tr->kept[it] = kept;
      if (tr->f_app) tr->f_app[it] = fapp;
    }
  };
  push(eps0, Ns);
  project_rm(W.p, Ns);  // line 3
  const double target = o.rel ? o.tol * eps0 : o.tol;
  cudaEvent_t pev[9];
  for (auto& e : pev) CK(cudaEventCreate(&e));
  double phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto mark = [&](int i) { CK(cudaEventRecord(pev[i], st)); };
  const char* tenv = getenv("FETIGPU_TRACE");  // per-iteration RRS line on stderr
  const bool trace_on = tenv && tenv[0] == '1';
  while (true) {
    if (eps <= target) { status = FETIGPU_CONVERGED; break; }
    if (it >= o.max_it) { status = FETIGPU_MAX_ITER; break; }
    const int k = Ns;
    mark(0);
    apply_F_block(W.p, k, Qb.p, k, k);  // line 7 (K5)
    mark(1);
    fapp += k;
    // line 8: Delta = Q^T W (column-major k x k; lower triangle used).  A
    // cublasDsyrkx of the lower triangle halves the flops but measured slower
    // at k = 96 (MBB) and shifted RRS rank decisions: the GEMM stays.
    CB(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_T, k, k, m, &one, Qb.p, k, W.p, k, &zero, Delta.p, k));
    k_mirror_lower<<<grid_for((long long)k * k), kThreads, 0, st>>>(Delta.p, k);
    mark(2);
    // line 9
    launch_pivchol(Delta.p, k, o.pivot_tol, perm.p, rank_d.p, d_status.p, ctl.p, pivx.p, st);
    LAUNCH_CHECK();
    mark(3);
    int rank = 0;
    CK(cudaMemcpyAsync(&rank, rank_d.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int hstat = 0;
    CK(cudaMemcpy(&hstat, d_status.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (hstat) {
      CK(cudaMemset(d_status.p, 0, sizeof(int)));
      fail(FETIGPU_E_INDEFINITE_INPUT, "pivoted Cholesky: negative pivot");
    }
    if (rank == 0) { status = FETIGPU_BREAKDOWN; break; }
    // lines 10-11: W_new = W N^T [L~^{-T}; 0] = W_sel L~^{-T} (m x rank, appended
    // to the arena at column K); same for Q.
    double *Wn = nullptr, *Qn = nullptr;
    const auto ta = std::chrono::steady_clock::now();
    append_slot(rank, &Wn, &Qn);
    if (trace_on) {
      CK(cudaStreamSynchronize(st));
      fprintf(stderr, "[fetigpu] rrs it %4d  store append %.2f ms (chunks %zu)\n", it + 1,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count(),
              chunks.size());
    }
    launch_identity(Linv.p, rank);
    CB(cublasDtrsm(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, rank, rank,
                   &one, Delta.p, k, Linv.p, rank));
    // W_sel lands in Q's (still free) arena slot, W_new = W_sel L~^{-T} in W's;
    // then Q_sel lands in W (no longer needed) and Q_new = Q_sel L~^{-T}.
    const dim3 tgrid((m + 31) / 32, (rank + 31) / 32);
    k_gather_cols_t<<<tgrid, dim3(32, 8), 0, st>>>(W.p, k, perm.p, rank, m, Qn, m);
    CB(cublasDtrmm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, m, rank, &one,
                   Linv.p, rank, Qn, m, Wn, m));
    k_gather_cols_t<<<tgrid, dim3(32, 8), 0, st>>>(Qb.p, k, perm.p, rank, m, W.p, m);
    CB(cublasDtrmm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, m, rank, &one,
                   Linv.p, rank, W.p, m, Qn, m));
    K += rank;
    if (trace_on) {
      const auto tb = std::chrono::steady_clock::now();
      CK(cudaStreamSynchronize(st));
      fprintf(stderr, "[fetigpu] rrs it %4d  compress kernels drained in %.2f ms after append\n", it + 1,
              std::chrono::duration<double, std::milli>(tb - ta).count());
    }
    mark(4);
    // lines 13-15
    CB(cublasDgemv(cb, CUBLAS_OP_T, m, rank, &one, Wn, m, r.p, 1, &zero, gamma.p, 1));
    CB(cublasDgemv(cb, CUBLAS_OP_N, m, rank, &one, Wn, m, gamma.p, 1, &one, lam.p, 1));
    CB(cublasDgemv(cb, CUBLAS_OP_N, m, rank, &one, Qn, m, gamma.p, 1, &zero, tmp.p, 1));
    project(tmp.p, 1, m);
    k_axpy<<<grid_for(m), kThreads, 0, st>>>(m, -1.0, tmp.p, r.p);
    mark(5);
    // line 16
    apply_precond(r.p, z.p, W.p, true);
    dots({{r.p, z.p}, {r.p, r.p}, {z.p, z.p}}, &sc.p->rz);
    mark(6);
    CK(cudaMemcpyAsync(hs, sc.p, sizeof(Scal), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    eps = metric(*hs);
    ++it;
    push(eps, rank);
    if (trace_on) {
      float te = 0;
      CK(cudaEventElapsedTime(&te, ev0, pev[6]));
      fprintf(stderr, "[fetigpu] rrs it %4d  eps/eps0 %.3e  rank %5d  K %7d  t %9.1f ms\n", it, eps / eps0, rank, K,
              te);
    }
    // line 17
    project_rm(W.p, Ns);
    mark(7);
    // lines 18-21: block classical Gram-Schmidt against all stored blocks,
    // `passes` passes.  W is row-major m x Ns (= column-major Ns x m).
    for (int p = 0; p < passes; ++p) {
      for (const Chunk& ch : chunks)  // Psi_c = Q_c^T W   (used x Ns, ld cap)
        CB(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_T, ch.used, Ns, m, &one, ch.q->p, m, W.p, Ns, &zero,
                       ch.psi->p, ch.cap));
      for (const Chunk& ch : chunks)  // W -= W_c Psi_c   ==   W^T -= Psi_c^T W_c^T
        CB(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_T, Ns, m, ch.used, &mone, ch.psi->p, ch.cap, ch.w->p, m, &one,
                       W.p, Ns));
    }
    mark(8);
    CK(cudaEventSynchronize(pev[8]));
    float t = 0;
    const int pidx[8][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7}, {7, 8}};
    for (int q = 0; q < 8; ++q) {
      CK(cudaEventElapsedTime(&t, pev[pidx[q][0]], pev[pidx[q][1]]));
      phase[q] += t;
    }
  }
  for (auto& e : pev) cudaEventDestroy(e);
  if (tr)
    for (int q = 0; q < 8; ++q) tr->phase_ms[q] = phase[q];
  CK(cudaEventRecord(ev1, st));
  const double ms = elapsed(ev0, ev1);
  CK(cudaMemcpyAsync(lambda_host, lam.p, m * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  pt.mark("rrs loop + readback", st);
  if (tr) {
    tr->status = status;
    tr->iterations = it;
    tr->f_applies = fapp;
    tr->eps0 = eps0;
    tr->eps_final = eps;
    tr->solve_ms = ms;
  }
  chunks.clear();
  pt.mark("rrs store release", st);
  return 0;
}

}  // namespace fg
