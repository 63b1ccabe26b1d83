// solve_pcg.cuh -- the device-resident PCG / FO iteration (graph-captured while loop).
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include "ctx.cuh"

namespace fg {

// ----------------------------------------------------------- the engine ---
// pcg single / FO: z = P Fbar^{-1} P r, eps_r = sqrt(r^T z)
// (PAPER.md:384); FO keeps F-normalized directions and re-orthogonalizes by
// classical Gram-Schmidt with `reorth_passes` passes.
// The whole iteration is device resident (scalars in device memory, breakdown
// flagged on the device) and captured once into a CUDA graph; the host
// replays it and reads back one 64-byte scalar record per iteration.
int Ctx::solve(const fetigpu_solve_opts& o, double* lambda_host, fetigpu_trace* tr) {
  if (su.m == 0) {  // no dual unknowns (e.g. a single FETI-DP subdomain): converged at iteration 0
    rhs();
    if (tr) {
      tr->status = FETIGPU_CONVERGED;
      tr->iterations = 0;
      tr->f_applies = 0;
      tr->eps0 = tr->eps_final = 0.0;
      tr->solve_ms = 0.0;
      if (tr->cap > 0) {
        if (tr->eps) tr->eps[0] = 0.0;
        if (tr->kept) tr->kept[0] = o.directions == FETIGPU_RRS ? su.Ns : 1;
        if (tr->f_app) tr->f_app[0] = 0;
      }
    }
    return 0;
  }
  if (o.directions == FETIGPU_RRS) return solve_rrs(o, lambda_host, tr);
  const int m = su.m;
  const bool fo = o.directions == FETIGPU_FO;
  const int passes = std::max(1, o.reorth_passes);
  rhs();
  DBuf<double> lam, r, z, w, q, corr, Wst, Qst, psi;
  DBuf<Scal> sc;
  DBuf<int> cnt;
  lam.alloc(m); r.alloc(m); z.alloc(m); w.alloc(m); q.alloc(m); corr.alloc(m);
  sc.alloc(1);
  sc.zero(st);
  cnt.alloc(1);
  cnt.zero(st);
  // FO keeps two m-vectors per iteration.  The store is sized for max_it
  // iterations but clamped to the free device memory (a generous max_it must
  // not fail a solve that converges early); a solve that fills a clamped
  // store without converging fails with FETIGPU_E_OUT_OF_MEMORY.
  int cap = std::max(1, o.max_it);
  if (fo) {
    const size_t freeb = dev_free_bytes(), margin = size_t(1) << 30;
    const long long fit = freeb > margin ? (long long)((freeb - margin) / (16.0 * m + 8)) : 0;
    if (fit < 1) fail(FETIGPU_E_OUT_OF_MEMORY, "FO: no device memory for the direction store");
    cap = (int)std::min<long long>(cap, fit);
  }
  const int max_it = fo ? cap : o.max_it;
  DBuf<double> psi_part;
  if (fo) {
    Wst.alloc((size_t)m * cap);
    Qst.alloc((size_t)m * cap);
    psi.alloc(cap);
  }
  const int psi_S = std::max(1, std::min(64, m / 2048));
  if (fo && psi_S > 1) psi_part.alloc((size_t)cap * psi_S);
  int fo_seg_grid = 148 * 8;
  {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    fo_seg_grid = sms * 8;
  }
  Scal* hs = nullptr;
  CK(cudaMallocHost(&hs, sizeof(Scal)));
  std::unique_ptr<Scal, decltype(&cudaFreeHost)> hs_guard(hs, cudaFreeHost);
  const bool tf = su.method == FETIGPU_TFETI;
  CK(cudaEventRecord(ev0, st));
  init_lambda(lam.p);
  apply_F(lam.p, q.p, 1, m, m);
  int fapp = 1;
  k_sub<<<grid_for(m), kThreads, 0, st>>>(m, d_d.p, q.p, r.p);
  project(r.p, 1, m);
  precond_projected(r.p, z.p, nullptr);
  dots({{r.p, z.p}, {r.p, r.p}, {z.p, z.p}}, &sc.p->rz);
  k_shift_rz<<<1, 1, 0, st>>>(sc.p);
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
  push(eps0, 1);
  CK(cudaMemcpyAsync(w.p, z.p, m * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(q.p, 0, m * 8, st));  // then re-zeroed each iteration by its last reader of q
  const double target = o.rel ? o.tol * eps0 : o.tol;
  // one PCG / FO iteration (everything on the stream, no host work)
  auto body = [&](bool readback) {
    apply_F(w.p, q.p, 1, m, m, /*y_zeroed=*/true);
    dots({{w.p, q.p}, {w.p, r.p}}, &sc.p->delta);
    if (tf) proj_corr(q.p, m, corr.p, m, 1);
    launch_pdl(k_pcg_update, grid_for(m), kThreads, 0, st, m, sc.p, fo ? 1 : 0, (const double*)w.p,
               (const double*)q.p, (const double*)(tf ? corr.p : nullptr), lam.p, r.p, z.p);
    apply_precond(r.p, z.p, nullptr, false, /*z_zeroed=*/true);
    project(z.p, 1, m);
    dots({{r.p, z.p}, {r.p, r.p}, {z.p, z.p}}, &sc.p->rz);
    if (fo) {
      launch_pdl(k_fo_store2, grid_for(m), kThreads, 0, st, m, (const Scal*)sc.p, (const int*)cnt.p, w.p, q.p,
                 Wst.p, Qst.p, (const double*)z.p);
      for (int pss = 0; pss < passes; ++pss) {
        launch_pdl(k_fo_psi_seg, fo_seg_grid, 256, 0, st, (const double*)Qst.p, m, (const int*)cnt.p, 1,
                   (const double*)w.p, psi_S == 1 ? psi.p : psi_part.p, psi_S);
        if (psi_S > 1)
          launch_pdl(k_fo_psi_sum, (cap + 255) / 256, 256, 0, st, (const int*)cnt.p, 1, psi_S,
                     (const double*)psi_part.p, psi.p);
        launch_pdl(k_fo_sub, (m + 31) / 32, 256, 0, st, (const double*)Wst.p, m, (const int*)cnt.p, 1,
                   (const double*)psi.p, w.p);
      }
      if (readback) launch_pdl(k_inc, 1, 1, 0, st, cnt.p);   // host loop; the device loop's k_iter_control advances it
    } else {
      launch_pdl(k_cg_dir2, grid_for(m), kThreads, 0, st, m, sc.p, (const double*)z.p, w.p, q.p);
      launch_pdl(k_shift_rz, 1, 1, 0, st, sc.p);
    }
    if (readback) CK(cudaMemcpyAsync(hs, sc.p, sizeof(Scal), cudaMemcpyDeviceToHost, st));
    LAUNCH_CHECK();
  };
  struct GraphGuard {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~GraphGuard() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
    }
  } gg;
  cudaGraph_t& graph = gg.graph;
  cudaGraphExec_t& exec = gg.exec;
  // Preferred: the whole loop on the device -- the iteration body plus
  // k_iter_control under a `while` conditional node, one graph launch per
  // solve, no host round trip per iteration.  Fallback (no conditional nodes,
  // or FETIGPU_HOST_LOOP=1): one graph launch + a 64-byte readback per iteration.
  const char* hl = getenv("FETIGPU_HOST_LOOP");
  bool device_loop = !(hl && hl[0] == '1') && eps > target && max_it > 0;
  if (device_loop) {
    DBuf<IterCtl> dctl;
    DBuf<double> dtrace;
    const int tcap = tr && tr->eps ? std::min(tr->cap, max_it + 1) : 1;
    dctl.alloc(1);
    dtrace.alloc(std::max(1, tcap));
    IterCtl h0{0, FETIGPU_MAX_ITER, 0, tcap, max_it, 0, eps0, target};
    CK(cudaMemcpyAsync(dctl.p, &h0, sizeof(IterCtl), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    bool built_ok = false;
    if (cudaGraphCreate(&graph, 0) == cudaSuccess) {
      cudaGraphConditionalHandle hcond;
      cudaGraphNodeParams cp = {};
      cudaGraphNode_t cnode;
      if (cudaGraphConditionalHandleCreate(&hcond, graph, 1, cudaGraphCondAssignDefault) == cudaSuccess) {
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = hcond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        if (cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp) == cudaSuccess) {
          cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
          if (cudaStreamBeginCaptureToGraph(st, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
              cudaSuccess) {
            body(false);
            launch_pdl(k_iter_control, 1, 1, 0, st, (const Scal*)sc.p, dctl.p, dtrace.p, hcond,
                       fo ? cnt.p : (int*)nullptr);
            cudaGraph_t captured = nullptr;
            built_ok = cudaStreamEndCapture(st, &captured) == cudaSuccess &&
                       cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
          }
        }
      }
    }
    if (!built_ok) {  // fall back to the host-driven loop
      cudaGetLastError();
      if (exec) { cudaGraphExecDestroy(exec); exec = nullptr; }
      if (graph) { cudaGraphDestroy(graph); graph = nullptr; }
      device_loop = false;
    } else {
      CK(cudaGraphLaunch(exec, st));
      IterCtl hc;
      CK(cudaMemcpyAsync(&hc, dctl.p, sizeof(IterCtl), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<double> ht(std::max(1, tcap));
      if (tcap > 1) CK(cudaMemcpy(ht.data(), dtrace.p, (size_t)tcap * 8, cudaMemcpyDeviceToHost));
      if (hc.err) fail(FETIGPU_E_NEGATIVE_INNER_PRODUCT, "r^T z < 0: preconditioner is not symmetric positive");
      for (int i = 1; i <= hc.it; ++i) {
        it = i;
        fapp = 1 + i;
        push(i < tcap ? ht[i] : hc.eps, 1);
      }
      it = hc.it;
      fapp = 1 + hc.it;
      eps = hc.it > 0 ? hc.eps : eps0;
      status = hc.status;
    }
  }
  if (!device_loop) {
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    body(true);
    CK(cudaStreamEndCapture(st, &graph));
    CK(cudaGraphInstantiate(&exec, graph, 0));
    while (true) {
      if (eps <= target) { status = FETIGPU_CONVERGED; break; }
      if (it >= max_it) { status = FETIGPU_MAX_ITER; break; }
      CK(cudaGraphLaunch(exec, st));
      CK(cudaStreamSynchronize(st));
      if (hs->breakdown != 0.0) { status = FETIGPU_BREAKDOWN; break; }
      ++fapp;
      eps = metric(*hs);
      ++it;
      push(eps, 1);
    }
  }
  if (chk_on && fo) {   // stored F-normalised directions: W^T F W = I
    int n = 0;
    CK(cudaMemcpyAsync(&n, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (n > 0) check_orth({Wst.p}, {Qst.p}, {n});
  }
  if (status == FETIGPU_MAX_ITER && max_it < o.max_it)
    fail(FETIGPU_E_OUT_OF_MEMORY, "FO: direction store full after " + std::to_string(max_it) +
                                      " iterations (device memory), max_it = " + std::to_string(o.max_it));
  CK(cudaEventRecord(ev1, st));
  const double ms = elapsed(ev0, ev1);
  CK(cudaMemcpyAsync(lambda_host, lam.p, m * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (tr) {
    tr->status = status;
    tr->iterations = it;
    tr->f_applies = fapp;
    tr->eps0 = eps0;
    tr->eps_final = eps;
    tr->solve_ms = ms;
  }
  return 0;
}

}  // namespace fg
