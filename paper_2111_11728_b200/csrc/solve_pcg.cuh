// solve_pcg.cuh -- the device-resident PCG / FO iteration (graph-captured while loop).
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include "ctx.cuh"

namespace fg {

// ------------------------------------------- K15: persistent iteration ---
static std::mutex g_persist_mu;   // one grid-barrier persistent kernel in flight per process
// Per dual row the (subdomain, local index, coefficient) entries of a map
// (operator or preconditioner) and one designated storing entry per row;
// false if some row has more than two entries (or none, unless allowed: the
// T-FETI operator maps skip the fixing DOFs).
static bool persist_rows(const std::vector<OpSub>& subs, const std::vector<int>& rows, const std::vector<double>& cf,
                         int KR, int m, bool allow_empty, std::vector<int4>& ent, std::vector<double2>& cc,
                         std::vector<unsigned char>& wr) {
  ent.assign(m, make_int4(-1, 0, -1, 0));
  cc.assign(m, make_double2(0.0, 0.0));
  wr.assign(rows.size(), 0);
  std::vector<int> n(m, 0);
  for (int s = 0; s < (int)subs.size(); ++s)
    for (int a = 0; a < subs[s].ns; ++a)
      for (int k = 0; k < KR; ++k) {
        const size_t e = (size_t)subs[s].map_off + (size_t)a * KR + k;
        const int r = rows[e];
        if (r < 0) continue;
        if (r >= m || n[r] == 2) return false;
        if (n[r] == 0) { ent[r].x = s; ent[r].y = a; cc[r].x = cf[e]; wr[e] = 1; }
        else { ent[r].z = s; ent[r].w = a; cc[r].y = cf[e]; }
        ++n[r];
      }
  for (int r = 0; r < m; ++r)   // no entry: the atomic path leaves 0 there (row_combine too)
    if (n[r] == 0 && !allow_empty) return false;
  return true;
}

bool Ctx::persist_prepare() {
  if (p_state) return p_state > 0;
  p_state = -1;
  const int Ns = su.Ns, m = su.m;
  auto down = [&](auto& dbuf, size_t n, auto& vec) {
    vec.resize(n);
    if (n) CK(cudaMemcpyAsync(vec.data(), dbuf.p, n * sizeof(vec[0]), cudaMemcpyDeviceToHost, st));
  };
  std::vector<OpSub> ops, pcs;
  down(d_op, Ns, ops);
  down(d_pc, Ns, pcs);
  CK(cudaStreamSynchronize(st));
  size_t nop = 0, npc = 0;
  for (auto& d : ops) nop = std::max(nop, (size_t)d.map_off + (size_t)d.ns * KR);
  for (auto& d : pcs) npc = std::max(npc, (size_t)d.map_off + (size_t)d.ns * KRp);
  std::vector<int> orow, prow;
  std::vector<double> ocf, pcf;
  down(d_oprows, nop, orow);
  down(d_opcoef_apply, nop, ocf);
  down(d_pcrows, npc, prow);
  down(d_pccoef, npc, pcf);
  CK(cudaStreamSynchronize(st));
  std::vector<int4> oe, pe;
  std::vector<double2> oc, pc;
  std::vector<unsigned char> ow, pw;
  if (!persist_rows(ops, orow, ocf, KR, m, true, oe, oc, ow) || !persist_rows(pcs, prow, pcf, KRp, m, false, pe, pc, pw))
    return false;
  std::vector<int> vo(Ns), vp(Ns);
  int to = 0, tp = 0;
  for (int s = 0; s < Ns; ++s) {
    vo[s] = to; to += ops[s].ns;
    vp[s] = tp; tp += pcs[s].ns;
  }
  if (su.method == FETIGPU_FETIDP) {
    down(d_voff, Ns, vo);   // phase 2 reads v_s at DpSub::v_off (= d_voff) of d_vbuf
    CK(cudaStreamSynchronize(st));
  } else {
    p_vop.alloc(std::max(1, to));
    p_voff_op.upload(vo, st);
  }
  p_vpc.alloc(std::max(1, tp));
  p_voff_pc.upload(vp, st);
  p_op_ent.upload(oe, st); p_op_c.upload(oc, st);
  p_pc_ent.upload(pe, st); p_pc_c.upload(pc, st); p_pc_wr.upload(pw, st);
  p_w2.alloc(m);
  p_r2.alloc(m);
  p_bar.alloc(2);
  CK(cudaStreamSynchronize(st));
  p_state = 1;
  return true;
}

// Applicable where the loop runs on the plain per-subdomain operators (no
// symmetric-packed tiles, dense L2-resident coarse inverse): C1-C3 and C5
// single / FO.  FETIGPU_PERSIST=0 selects the graph loop, =1 forces this one; FETIGPU_PERSIST_G
// sets the grid; FETIGPU_PERSIST_BAR=grid|cluster the barrier (a grid of at
// most 16 CTAs runs as one thread-block cluster by default).
int Ctx::persist_grid(bool fo) {
  const char* e = getenv("FETIGPU_PERSIST");
  if (e && e[0] == '0') return 0;
  if (su.m == 0 || use_sym || pc_sym || (KRp != 1 && KRp != 3)) return 0;
  if (su.method == FETIGPU_FETIDP && (use_csym || KR != 1)) return 0;
  if (su.method == FETIGPU_TFETI && KR != 3) return 0;
  // measured policy (tools/persist_ab.py): the persistent loop
  // wins where an iteration is latency-bound -- operators of a few MB (C1-fo:
  // 34 vs 43 us, C2: 26 vs 35 us, C2-fo: 50 vs 58 us per iteration); where
  // the operators stream tens of MB (C3) the graph's many-CTA kernels keep
  // more loads in flight than one CTA per SM and stay faster.
  // FETIGPU_PERSIST=1 forces it wherever it applies.
  const bool force = e && e[0] == '1';
  if (!force && op_bytes > 32e6) return 0;
  if (!persist_prepare()) return 0;
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pcg_persist<GridBarrier, true, true>, kThreads,
                                                   persist_smem()));
  if (occ < 1) return 0;
  int G = sms * std::min(occ, kPersistOcc);
  const char* eg = getenv("FETIGPU_PERSIST_G");
  if (eg && atoi(eg) > 0) G = atoi(eg);
  G = std::min(G, sms * occ);
  const char* eb = getenv("FETIGPU_PERSIST_BAR");
  persist_cluster = G <= 16 && !(eb && strcmp(eb, "grid") == 0);
  (void)fo;
  return G;
}

size_t Ctx::persist_smem() const {
  const bool tf = su.method == FETIGPU_TFETI;
  const int sv = !persist_red() ? 0 : tf ? (3 * su.Ns <= kRedH ? 3 * su.Ns : 0) : (su.Nc <= kRedU ? su.Nc : 0);
  return (size_t)(std::max(max_ld, max_pc_ld) + sv) * 8;
}

bool Ctx::launch_persist(int G, bool fo, int passes, int psi_S, double* lam, double* r, double* z, double* w,
                         double* q, Scal* sc, double* Wst, double* Qst, double* psi, double* psi_part, int* cnt,
                         IterCtl* ctl, double* trace) {
  const bool tf = su.method == FETIGPU_TFETI;
  PersistArgs a{};
  a.m = su.m;
  a.Ns = su.Ns;
  a.Nc = su.Nc;
  a.KRp = KRp;
  a.nz_op = std::max(1, std::min(8, G / su.Ns));   // one round of (subdomain, slice) items
  a.nz_pc = a.nz_op;
  a.ndot = dot_blocks();
  a.psi_S = psi_S;
  a.passes = passes;
  a.xs_len = std::max(max_ld, max_pc_ld);
  a.redU = !tf && persist_red() && su.Nc <= kRedU;
  a.redH = tf && persist_red() && 3 * su.Ns <= kRedH;
  a.op = d_op.p; a.opmat = d_opmat.p; a.oprows = d_oprows.p; a.opcoef = d_opcoef_apply.p;
  a.vop = tf ? p_vop.p : d_vbuf.p;
  a.voff_op = tf ? p_voff_op.p : d_voff.p;
  a.op_ent = p_op_ent.p; a.op_c = p_op_c.p;
  if (!tf) {
    a.dp = d_dp.p; a.abc = d_abc.p; a.tbuf = d_tbuf.p; a.cg = su.Nc ? d_cgather.p : nullptr;
    a.cmap = d_cmap.p; a.Kinv = d_Kinv.p; a.gc = d_gc.p;
  } else {
    a.pj = d_pj.p; a.pjcoef = d_pjcoef.p; a.RT = d_RT.p; a.rt_off = d_rt_off.p; a.H = d_H.p;
    a.pj_sr = d_pjrow_sr.p; a.pj_c = d_pjrow_c.p; a.g = d_g.p;
  }
  a.h = d_h.p;
  a.pc = d_pc.p; a.pcmat = d_pcmat.p; a.pcrows = d_pcrows.p; a.pccoef = d_pccoef.p;
  a.vpc = p_vpc.p; a.voff_pc = p_voff_pc.p;
  a.pc_ent = p_pc_ent.p; a.pc_c = p_pc_c.p; a.pc_wr = p_pc_wr.p;
  a.lam = lam; a.r = r; a.z = z; a.w = w; a.q = q; a.w2 = p_w2.p; a.r2 = p_r2.p;
  a.sc = sc;
  a.partial = d_partial.p;
  a.Wst = Wst; a.Qst = Qst; a.psi = psi; a.psi_part = psi_part; a.cnt = cnt;
  a.ctl = ctl;
  a.trace = trace;
  CK(cudaMemsetAsync(p_bar.p, 0, 2 * sizeof(unsigned int), st));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = persist_smem();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  bool ok = false;
  auto go = [&](auto kern, auto barrier) {
    if (persist_cluster) {
      if (G > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
    }
    ok = cudaLaunchKernelEx(&cfg, kern, a, barrier) == cudaSuccess;
  };
  const GridBarrier gb{p_bar.p, p_bar.p + 1};
  const ClusterBarrier cb{p_bar.p, p_bar.p + 1};
  if (persist_cluster) {
    if (tf && fo) go(k_pcg_persist<ClusterBarrier, true, true>, cb);
    else if (tf) go(k_pcg_persist<ClusterBarrier, true, false>, cb);
    else if (fo) go(k_pcg_persist<ClusterBarrier, false, true>, cb);
    else go(k_pcg_persist<ClusterBarrier, false, false>, cb);
  } else {
    if (tf && fo) go(k_pcg_persist<GridBarrier, true, true>, gb);
    else if (tf) go(k_pcg_persist<GridBarrier, true, false>, gb);
    else if (fo) go(k_pcg_persist<GridBarrier, false, true>, gb);
    else go(k_pcg_persist<GridBarrier, false, false>, gb);
  }
  if (!ok) cudaGetLastError();   // e.g. not co-resident: the caller falls back to the graph loop
  return ok;
}

// K15c: the cluster-resident loop (T-FETI single direction, N_s <= 16
// subdomains whose F_s and S~_s fit in one CTA's shared memory each, C1).
// FETIGPU_CLUSTER=0 disables it.
size_t Ctx::cluster_smem() const {
  int fs = 0, ps = 0, xs = std::max(max_ld, max_pc_ld);
  for (size_t s = 0; s < op_ns.size(); ++s) fs = std::max(fs, op_ns[s] * op_ld[s]);
  for (int s = 0; s < su.Ns; ++s) ps = std::max(ps, pc_nsld[s]);
  return cluster_smem_doubles(su.m, su.Ns, dot_blocks(), fs, ps, xs) * 8;
}

bool Ctx::cluster_ok(bool fo) {
  const char* e = getenv("FETIGPU_CLUSTER");
  if (e && e[0] == '0') return false;
  if (fo || su.method != FETIGPU_TFETI || su.Ns < 1 || su.Ns > 16 || su.m == 0 || KR != 3) return false;
  if (use_sym || pc_sym || (KRp != 1 && KRp != 3) || (int)pc_nsld.size() != su.Ns) return false;
  int dev = 0, optin = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (cluster_smem() + 1024 > (size_t)optin) return false;
  return persist_prepare();
}

bool Ctx::launch_cluster(double* lam, double* r, double* w, Scal* sc, IterCtl* ctl, double* trace) {
  ClusterArgs a{};
  a.m = su.m;
  a.Ns = su.Ns;
  a.ndot = dot_blocks();
  a.KRp = KRp;
  int fs = 0, ps = 0;
  for (size_t s = 0; s < op_ns.size(); ++s) fs = std::max(fs, op_ns[s] * op_ld[s]);
  for (int s = 0; s < su.Ns; ++s) ps = std::max(ps, pc_nsld[s]);
  a.fs_len = fs;
  a.ps_len = ps;
  a.xs_len = std::max(max_ld, max_pc_ld);
  a.op = d_op.p; a.opmat = d_opmat.p; a.oprows = d_oprows.p; a.opcoef = d_opcoef_apply.p;
  a.pc = d_pc.p; a.pcmat = d_pcmat.p; a.pcrows = d_pcrows.p; a.pccoef = d_pccoef.p;
  a.op_ent = p_op_ent.p; a.op_c = p_op_c.p; a.pc_ent = p_pc_ent.p; a.pc_c = p_pc_c.p;
  a.pj = d_pj.p; a.pjcoef = d_pjcoef.p; a.RT = d_RT.p; a.rt_off = d_rt_off.p; a.H = d_H.p;
  a.pj_sr = d_pjrow_sr.p; a.pj_c = d_pjrow_c.p;
  a.lam = lam; a.r = r; a.w = w;
  a.sc = sc;
  a.ctl = ctl;
  a.trace = trace;
  const size_t smem = cluster_smem();
  auto kern = KRp == 1 ? k_pcg_cluster<1> : k_pcg_cluster<3>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (su.Ns > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(su.Ns);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = su.Ns;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) {   // e.g. the cluster cannot be scheduled
    cudaGetLastError();
    return false;
  }
  return true;
}

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
    // K15: the whole loop as one persistent kernel where the operators are
    // the plain per-subdomain ones (C1-C3, C5 single / FO); bit-identical
    // to the graph below (kernels_persist.cuh)
    // (a launch that cannot be scheduled falls back to the next loop)
    bool single_kernel = false;
    // Two grid-barrier persistent kernels from different contexts / host
    // threads could each end up partly resident and wait on each other: the
    // process runs one at a time (held until this solve's final sync).
    // Cluster kernels need no lock (a cluster is co-scheduled as a whole).
    std::unique_lock<std::mutex> persist_lock(g_persist_mu, std::defer_lock);
    if (cluster_ok(fo) && launch_cluster(lam.p, r.p, w.p, sc.p, dctl.p, dtrace.p)) {
      single_kernel = true;
      solve_loop = 4;
    } else {
      const int pg = persist_grid(fo);
      if (pg > 0 && !persist_cluster) persist_lock.lock();
      if (pg > 0 && launch_persist(pg, fo, passes, psi_S, lam.p, r.p, z.p, w.p, q.p, sc.p, Wst.p, Qst.p, psi.p,
                                   psi_part.p, cnt.p, dctl.p, dtrace.p)) {
        single_kernel = true;
        solve_loop = persist_cluster ? 3 : 2;
      }
    }
    if (single_kernel) {
      built_ok = true;
    } else if (cudaGraphCreate(&graph, 0) == cudaSuccess) {
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
      if (!single_kernel) {
        CK(cudaGraphLaunch(exec, st));
        solve_loop = 1;
      }
      IterCtl hc;
      CK(cudaMemcpyAsync(&hc, dctl.p, sizeof(IterCtl), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<double> ht(std::max(1, tcap));
      if (tcap > 1) {
        CK(cudaMemcpyAsync(ht.data(), dtrace.p, (size_t)tcap * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
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
    solve_loop = 0;
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
