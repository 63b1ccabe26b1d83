// ctx.cuh -- the per-problem context: device-resident operators and their metadata.
// Method bodies: ctx_build.cuh (K1-K3, coarse), ctx_ops.cuh (K4/K5, projector,
// preconditioner, rhs, recovery), solve_pcg.cuh, solve_rrs.cuh.
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include "runtime.cuh"
#include "setup.hpp"
#include "kernels_apply.cuh"
#include "kernels_persist.cuh"
#include "kernels_build.cuh"
#include "kernels_dmma.cuh"
#include "dla.cuh"

namespace fg {

// host-side index maps produced by Ctx::host_maps (see ctx_build.cuh)
struct HostMaps {
  std::vector<int> src, ext, src_off, ext_off, fac_ne;           // slot src/ext lists
  std::vector<OpSub> ops, pcs, pjs;                              // per subdomain
  std::vector<int> slot_of, top_off, design, rt_off, sub_maxrow;
  std::vector<size_t> ip_off;
  std::vector<int> rows, top_pos, prow;                          // gather / scatter entries
  std::vector<double> coef, pcoef, pjcoef, RT;
  std::vector<int2> pj_sr;                                       // T-FETI projector rows
  std::vector<double2> pj_c;
  std::vector<double> e;
  std::vector<double> fb, gD;                                    // rhs / recovery
  std::vector<int> Dl, Doff, Dcnt, cpos, coff, xoff;
  int xo = 0;
  std::vector<DpSub> dps;                                        // FETI-DP coarse lists
  std::vector<int> cmap, voff, optr, oidx, osub, oloc;
  int vo = 0, to = 0;
};

struct Ctx {
  Setup su;
  Scratch scratch;
  cudaStream_t st = nullptr;
  bool built = false;
  DBuf<int> d_status;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  double build_ms = 0, nd_ms = 0, slot_ms = 0, coarse_ms = 0;
  bool keep_factors = true;

  // ND tree
  DBuf<NdDev> d_nodes;
  DBuf<int> d_elem_ids, d_emap, d_cmaps, d_nd_dofs, d_topdown, d_design;
  DBuf<double> d_dens, d_S, d_ndfac;
  // operator (F_s) per subdomain
  int KR = 1;
  DBuf<OpSub> d_op;
  DBuf<double> d_opmat, d_opcoef, d_opfac;
  // coefficients used with the explicit operators: all ones once the +-1
  // constraint signs are folded into F_s / A_bc (FETI-DP), else d_opcoef
  DBuf<double> d_opcoef_apply;
  bool folded = false;
  bool blk_aligned = false;  // every slot's F'' / A'' rows admit 16-byte chunks (K5 fast path)
  // symmetric-packed operator tiles for the GEMV (used when rsplit == 1)
  bool use_sym = false;
  DBuf<double> d_symtiles;
  DBuf<SymSub> d_sym;
  double sym_bytes = 0;
  int sym_smem = 0;
  bool pc_sym = false;
  DBuf<double> d_pcsymtiles;
  DBuf<SymSub> d_pcsym;
  int pc_sym_smem = 0;
  // TMA form of the symmetric-packed GEMV (k_sym_gemv_tma, the default;
  // FETIGPU_SYM_TMA=0 keeps the LDG kernel): ring slots, padded length,
  // dynamic shared memory, persistent grid (2 CTAs per SM)
  bool sym_tma = false;
  int sym_ring = 0, sym_npad = 0, pc_sym_ring = 0, pc_sym_npad = 0, sym_grid = 0;
  // 1: next x_s gathered inside the tile loop, 2: next A'' prefetched into L2 (measured slower),
  // 4: coarse arrival count per subdomain instead of once per CTA, 8: A'' streamed through the rings
  // (coarse pre-pass after the tile loop; t_s summed in another order than fused_dp_t) (FETIGPU_SYM_FLAGS)
  int sym_flags = 9;
  size_t sym_tma_bytes = 0, pc_sym_tma_bytes = 0;
  std::vector<std::vector<double>> slot_sign;
  DBuf<int> d_oprows, d_slot_of, d_fac_ne, d_top_pos, d_top_off;
  DBuf<long long> d_fac_off;
  std::vector<int> op_ns, op_ld;
  std::vector<long long> op_moff, op_foff;
  int max_ld = 0, max_ne = 0;
  int rsplit = 1;     // CTAs per subdomain in the GEMV kernels (few subdomains)
  int pc_rsplit = 1;
  // slot src/ext lists
  DBuf<int> d_op_src, d_op_ext, d_op_src_off, d_op_ext_off;
  // preconditioner
  int KRp = 1;
  DBuf<OpSub> d_pc;
  DBuf<double> d_pcmat, d_pccoef;
  DBuf<int> d_pcrows;
  int max_pc_ld = 0;
  // projector (T-FETI)
  DBuf<OpSub> d_pj;
  DBuf<double> d_pjcoef, d_RT, d_H, d_e;
  DBuf<int> d_rt_off;
  // FETI-DP
  DBuf<DpSub> d_dp;
  DBuf<double> d_abc, d_kccs, d_Kinv, d_vbuf, d_tbuf, d_fbar_loc, d_fbar;
  DBuf<int> d_cmap, d_voff, d_optr, d_oidx;
  // boundary data for rhs / recovery
  DBuf<double> d_fb, d_gD;
  DBuf<int> d_D, d_D_off, d_D_cnt, d_c_pos, d_c_off, d_xoff;
  DBuf<double> d_xb;
  // scratch vectors
  DBuf<double> d_v1, d_v2, d_v3, d_g, d_h, d_partial;
  DBuf<double> d_d, d_lam0;
  DBuf<unsigned int> d_counter, d_counter2;
  bool have_rhs = false;
  // stats
  double op_bytes = 0, op_flops = 0, main_bytes = 0;
  // grow-only staging buffers of the host-pointer entry points
  DBuf<double> stage_x, stage_y;
  void stage(size_t n) {
    if (stage_x.n < n) { stage_x.alloc(n); stage_y.alloc(n); }
  }

  // FETI-DP coarse inverse in symmetric-packed 32x32 tiles (+ per-tile partials)
  DBuf<double> d_kinv_tiles, d_crow, d_ccol, d_gc;
  DBuf<unsigned int> d_gcnt;
  DBuf<CoarseGather> d_cgather;
  int kinv_nb = 0, csym_grid = 1;
  bool use_csym = false;  // packed inverse only where the dense one leaves L2 (N_c > 2048)

  // Host-buffer F-apply pipeline (fetigpu_apply_F with host pointers, FETI-DP
  // on the symmetric path): lambda goes over PCIe in kPipe row-prefix chunks on
  // a copy stream; the subdomains of chunk c (rows < pipe_need[c]) start their
  // phase-1 GEMV on their own stream as soon as that prefix has landed, so the
  // H2D copy overlaps the operator stream and the chunks fill the GPU together.
  static constexpr int kPipe = 8;
  cudaStream_t pipe_st[kPipe] = {}, pipe_cp = nullptr;
  cudaEvent_t pipe_in[kPipe] = {}, pipe_done[kPipe] = {}, pipe_start = nullptr;
  int pipe_s0[kPipe + 1] = {}, pipe_need[kPipe] = {};
  bool pipe_ready = false;
  // single persistent phase-1 kernel gated on the landed row prefix (TMA form): flag word, per-subdomain need
  DBuf<int> d_xflag, d_subneed;
  int* h_flagvals = nullptr;   // pinned: the values the copy stream DMAs into the flag (no SM needed)
  cudaEvent_t pipe_cp_done = nullptr;
  std::vector<int> sub_maxrow;  // per subdomain: largest dual row it touches (-1: none)

  // freed RRS direction-store chunks, reused by this context's next solve;
  // returned to the driver with the context
  BlockCache rrs_cache;
  // operator storage recycled across fetigpu_rebuild (density snapshots)
  BlockCache build_cache;
  int rebuilds = 0;
  // warm start of the next solve (fetigpu_solve_warm): device copy of lambda0
  DBuf<double> d_warm;
  bool warm = false;
  // lam := lambda0 of the solve: the warm start when one is set (T-FETI:
  // projected onto G lambda = e: lam0 + P(warm - lam0)), else the default
  void init_lambda(double* lam);
  // side stream of the block apply (Q memset overlapping the coarse GEMM)
  cudaStream_t aux_st = nullptr;
  cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
  ~Ctx() {
    if (aux_fork) cudaEventDestroy(aux_fork);
    if (aux_join) cudaEventDestroy(aux_join);
    if (aux_st) cudaStreamDestroy(aux_st);
    for (auto& e : pipe_in) if (e) cudaEventDestroy(e);
    for (auto& e : pipe_done) if (e) cudaEventDestroy(e);
    if (pipe_start) cudaEventDestroy(pipe_start);
    if (pipe_cp_done) cudaEventDestroy(pipe_cp_done);
    if (h_flagvals) cudaFreeHost(h_flagvals);
    for (auto& q : pipe_st) if (q) cudaStreamDestroy(q);
    if (pipe_cp) cudaStreamDestroy(pipe_cp);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
    if (st) cudaStreamDestroy(st);
  }

  void check_status() {
    int h = 0;
    CK(cudaMemcpyAsync(&h, d_status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h != 0) {
      CK(cudaMemsetAsync(d_status.p, 0, sizeof(int), st));
      fail(h, "device factorization failed (nonpositive pivot)");
    }
  }

  void init_device();

  double elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }

  // ------------------------------------------------------------ build --
  void eliminate(const std::vector<FrontDesc>& fds, double* base);

  // batched blocked partial Cholesky over all frontals in `fs` (device copy `d`)
  void bpc(const FrontDesc* d, const std::vector<FrontDesc>& fs, double* base);

  void build_nd();

  // batched slot processing: assemble [[S[src,src],E],[E^T,0]], eliminate,
  // extract; processed in chunks bounded by a workspace budget
  struct SlotOut {
    std::vector<long long> mat_off;
    std::vector<int> mat_ld;
    std::vector<long long> abc_off, kcc_off, fac_off;
    long long mat_total = 0, abc_total = 0, kcc_total = 0, fac_total = 0;
  };
  void run_slots(const std::vector<SlotFront>& slots, const SlotOut& out, double* mats, double sign,
                 bool nc_first, double* abc, double* kcc, double* fac, int errcode);

  PhaseTimer ptimer;
  // operator slot layout (offsets of F_s / A_bc / Kcc^s / factors per slot)
  void plan_op_slots(SlotOut& so);
  HostMaps host_maps(const SlotOut& so) const;
  void build_ops(const SlotOut& so, std::future<HostMaps>& maps);

  void build_coarse(const SlotOut& so, const std::vector<int>& osub, const std::vector<int>& oloc);

  // u = Kbar^{-1} (sum_s B_c^T t_s) into d_h (stages A + B on the packed inverse)
  // g_ready: phase 1 already formed g in d_gc (fused gather of the symmetric
  // GEMV); otherwise gather it here
  // zero_y: output still to be zeroed (the gather kernel does it when it runs)
  void coarse_solve_packed(bool g_ready, double* zero_y = nullptr);
  // phase 2: y = sum_s B_s (v_s + A''_s u_s)
  void launch_phase2_csym(double* y) {
    launch_pdl(k_dp_phase2, su.Ns, kThreads, 0, st, (const OpSub*)d_op.p, (const DpSub*)d_dp.p,
               (const int*)d_oprows.p, (const double*)d_opcoef_apply.p, (const double*)d_abc.p,
               (const int*)d_cmap.p, (const double*)d_h.p, (const double*)d_vbuf.p, y, 1.0);
    LAUNCH_CHECK();
  }

  void launch_kcc_assemble(const int* optr, const int* osub, const int* oloc, const long long* kco,
                           const int* ncs, const double* kccs, int Nc, double* K);
  void launch_identity(double* X, int n);
  void launch_symmetrize(double* A, int n);
  void mirror_slots(const std::vector<long long>& moff, const std::vector<int>& ns, const std::vector<int>& ld,
                    double* mats);

  void build();

  // -------------------------------------------------------- operators --
  // y_zeroed: the caller already zeroed y (T-FETI scatters into it); lets the
  // solver loop drop the memset node and chain the GEMV with PDL
  void apply_F(const double* x, double* y, int ncols, int ldx, int ldy, bool y_zeroed = false);
  // one launch of the symmetric-packed GEMV over subdomains [s0, s0 + n)
  struct SymArgs {
    bool pc = false;        // preconditioner blocks (else the operator)
    int kr = 1;             // map entries per local DOF
    bool store_v = false;   // FETI-DP phase 1: v_s stored (and t_s, g); else scattered into y
    const double* x = nullptr;
    double* y = nullptr;
    int s0 = 0, n = 0;
    double* zero_y = nullptr;   // FETI-DP phase 1 also zeroes this vector (slices by subdomain)
    bool coarse_gather = false;
    bool pdl = false;
    bool per_cta = false;   // one subdomain per CTA (the host-pipelined chunks)
    bool wait_x = false;    // x arrives while the kernel runs: gate every gather on d_xflag / d_subneed
  };
  void launch_sym(cudaStream_t q, const SymArgs& a);
  // host-buffer apply as ONE flag-gated persistent kernel instead of a kernel per chunk and stream
  // (FETIGPU_PIPE_FLAG=1; measured equal on a B200, 0.497 vs 0.496 ms e2e: PCIe sets the floor, so the
  // simpler chunk kernels, which never wait inside a kernel, stay the default)
  static bool pipe_flagged() {   // read per call (tests switch it)
    const char* e = getenv("FETIGPU_PIPE_FLAG");
    return e && e[0] == '1';
  }

  void setup_pipe();

  // y = F x with x, y in (pinned) host memory; the result is identical to
  // the device path (same kernels per subdomain, same phase-2 order)
  void apply_F_host(const double* xh, double* yh);

  // Zcols: per-subdomain columns, column-major m x N_s (row_major = false)
  // or row-major m x N_s (row_major = true)
  void apply_precond(const double* r, double* z, double* Zcols, bool row_major = false, bool z_zeroed = false);

  // ---- K5: Q = F W for k columns, row-major blocks (W(i,c) = W[i*ldw + c])
  DBuf<double> blk_t, blk_T, blk_U;
  DBuf<int> d_k5order;   // K5 subdomain order (4 x 4-module tiles)
  DBuf<int> d_k5e_order; // K5e edge-chunk order (first owner in the K5 walk)
  void apply_F_block(const double* W, int ldw, double* Q, int ldq, int k);
  // ---- K5z: Q = F Z for a fresh per-subdomain preconditioner block Z
  // (row-major m x N_s, column s supported on subdomain s's dual rows):
  // 5 local columns per subdomain instead of N_s (kernels_dmma.cuh).  false
  // when the problem does not have that structure (then use apply_F_block).
  int bz_state = 0;   // 0 unknown, 1 ready, -1 not applicable
  DBuf<int> bz_other, bz_j, bz_nbr, bz_erow, bz_eb1, bz_eb2, bz_ez1, bz_ez2;
  DBuf<BzEdge> bz_edges;
  DBuf<double> bz_Y;
  int bz_nedges = 0, bz_maxns = 0;
  bool bz_prepare();
  // ---- subdomain-sharded apply: this context applies only the
  // subdomains [shard_s0, shard_s1) of the full problem (one rank of a
  // row-band partition of the module grid); exchanges are the caller's
  // (shard.py: NCCL / gloo, or an in-process emulation)
  int shard_s0 = 0, shard_s1 = -1;
  int tot_c() const {
    int t = 0;
    for (auto& S : su.subs) t += (int)S.c.size();
    return t;
  }
  void shard_phase1(const double* x, double* y, double* tout, bool precond);
  void shard_phase2(const double* tall, double* y);
  // coarse scratch of the block applies (K5 / K5z) for k columns
  void ensure_block_buffers(int k) {
    if (su.method != FETIGPU_FETIDP) return;
    int tot_c = 0;
    for (auto& S : su.subs) tot_c += (int)S.c.size();
    if (blk_t.n < (size_t)tot_c * k) blk_t.alloc((size_t)tot_c * k);
    if (blk_T.n < (size_t)su.Nc * k) { blk_T.alloc((size_t)su.Nc * k); blk_U.alloc((size_t)su.Nc * k); }
  }
  // Yout / Tout (optional): keep the sparse part Y (nmap x 5) and the coarse
  // pre-pass T (N_c x k row-major) of F Z for the line-7 correction
  bool apply_F_block_z(const double* Z, double* Q, int k, double* Yout = nullptr, double* Tout = nullptr);
  // Q -= (F Zhat) N from the kept F Z_l (K14): DMMA form by default,
  // FETIGPU_FZ_FMA=1 selects the fma-chain kernel
  void launch_fz_correct(const double* Yst, long long ystride, int nl, const double* NT, const double* Uc, int k,
                         double* Q) {
    static const bool fma_form = [] {
      const char* e = getenv("FETIGPU_FZ_FMA");
      return e && e[0] == '1';
    }();
    if (fma_form || (k & 1))   // the DMMA form's 16-byte B rows need an even k
      k_fz_correct<<<dim3((k + kFzCols - 1) / kFzCols, bz_nedges, (kBzRows + kFzRows - 1) / kFzRows), 256, 0, st>>>(
          bz_edges.p, bz_erow.p, bz_eb1.p, bz_eb2.p, d_op.p, d_dp.p, d_abc.p, d_cmap.p, bz_nbr.p, Yst, ystride, nl, NT,
          Uc, k, Q);
    else
      k_fz_correct_mma<<<dim3((k + kFmBN - 1) / kFmBN, bz_nedges, (kBzRows + kFmBM - 1) / kFmBM), 128, 0, st>>>(
          bz_edges.p, bz_erow.p, bz_eb1.p, bz_eb2.p, d_op.p, d_dp.p, d_abc.p, d_cmap.p, bz_nbr.p, Yst, ystride, nl,
          NT, Uc, k, Q);
    LAUNCH_CHECK();
  }
  long long bz_nmap = 0;
  double* bz_tt = nullptr;   // compact T output of the next K5z (set by the solver)
  DBuf<int> fz_osub, fz_orow;   // coarse-gather owners: subdomain, tbuf row (d_optr order)

  // single-vector projector finish: per dual row its <= 2 (s, RT offset) / signs
  DBuf<int2> d_pjrow_sr;
  DBuf<double2> d_pjrow_c;

  // grow-only scratch for the multi-column projector paths: no cudaMalloc /
  // cudaFree (both device-synchronising) inside solver iterations once warm
  DBuf<double> ws_g, ws_h, ws_corr, ws_dla;
  static double* grow(DBuf<double>& b, size_t n) {
    if (b.n < n) b.alloc(n);
    return b.p;
  }
  // grow-only workspace of the dense algebra (split-K partials, triangular
  // inverse, GEMV segment partials)
  double* dla_ws(size_t n) { return grow(ws_dla, std::max<size_t>(n, 1)); }
  // ||x||^2 of a long block into the device scalar out (k_norm2)
  DBuf<double> nrm_part;
  DBuf<unsigned int> nrm_cnt;
  void block_norm2(const double* x, size_t n, double* out) {
    constexpr int kBlocks = 148 * 4;
    if (nrm_part.n < kBlocks) { nrm_part.alloc(kBlocks); nrm_cnt.alloc(1); nrm_cnt.zero(st); }
    k_norm2<<<kBlocks, 256, 0, st>>>(x, n, nrm_part.p, nrm_cnt.p, out);
    LAUNCH_CHECK();
  }

  // v <- P v for a row-major block (m x ncols, ld = ncols), T-FETI only
  void project_rm(double* v, int ncols);

  // h = H g for ncols columns of length 3N_s (H symmetric, column-major)
  void small_gemm(const double* g, double* h, int ncols) {
    const int nc = 3 * su.Ns;
    if (ncols == 1) {
      k_dense_gemv<<<grid_for((long long)nc * 32), kThreads, 0, st>>>(d_H.p, nc, g, h);
    } else {
      gemm(st, false, false, nc, ncols, nc, 1.0, d_H.p, nc, g, nc, 0.0, h, nc);
    }
    LAUNCH_CHECK();
  }

  // single vector: g = gsign R^T B^T v; h = H g; out = B R h (accumulate: out += B R h)
  void proj_single(const double* v, double* out, int accumulate, double gsign) {
    const int nc = 3 * su.Ns;
    launch_pdl(k_proj_gather, dim3(su.Ns, 1), kThreads, 0, st, (const OpSub*)d_pj.p, (const int*)d_pcrows.p,
               (const double*)d_pjcoef.p, (const double*)d_RT.p, (const int*)d_rt_off.p, v, su.m, d_g.p, nc, gsign,
               1);
    launch_pdl(k_dense_gemv, grid_for((long long)nc * 32), kThreads, 0, st, (const double*)d_H.p, nc,
               (const double*)d_g.p, d_h.p);
    launch_pdl(k_proj_rows, grid_for(su.m), kThreads, 0, st, su.m, (const int2*)d_pjrow_sr.p,
               (const double2*)d_pjrow_c.p, (const double*)d_RT.p, (const double*)d_h.p, out, accumulate);
    LAUNCH_CHECK();
  }

  // corr = P v - v for ncols columns (T-FETI); caller adds
  void proj_corr(const double* v, int ldv, double* corr, int ldc, int ncols, double gsign = -1.0);

  void project(double* v, int ncols, int ld) {
    if (su.method != FETIGPU_TFETI) return;
    if (ncols == 1 && su.m > 0) {
      proj_single(v, v, 1, -1.0);
      return;
    }
    double* cp = d_v3.p;
    if (ncols > 1) cp = grow(ws_corr, (size_t)su.m * ncols);
    proj_corr(v, ld, cp, su.m, ncols);
    k_add<<<dim3(grid_for(su.m), ncols), kThreads, 0, st>>>(su.m, cp, v, su.m, ld);
    LAUNCH_CHECK();
  }

  // per-subdomain boundary rhs b = (f - B^T lambda)[src] - S[src,D] gD - S[src,c] u_c
  void launch_bnd_rhs(const double* lambda, const double* uc);
  void launch_bnd_u(const double* uc, double* ub_all);
  void launch_dp_fbar();
  void launch_rhs_scatter(double* out);
  void launch_add_rigid(double* u, const double* alpha);
  void launch_scatter_perim(const double* ub_all, double* u);

  void rhs();

  void recover(const double* lambda_dev, double* u_dev);

  // ------------------------------------------------------------ engine --
  // fixed partition of the deterministic dot products: one row per thread
  // (the persistent loop forms each row's operands on the fly in its CTA)
  int dot_blocks() const { return std::max(1, std::min(kDotBlocks, (su.m + kThreads - 1) / kThreads)); }
  void dots(std::initializer_list<std::pair<const double*, const double*>> pairs, double* out) {
    DotArgs a{};
    int k = 0;
    for (auto& p : pairs) { a.a[k] = p.first; a.b[k] = p.second; ++k; }
    a.npairs = k;
    a.n = su.m;
    launch_pdl(k_dot_fused, dot_blocks(), kThreads, 0, st, a, d_partial.p, d_counter.p, out);
    LAUNCH_CHECK();
  }

  void precond_projected(const double* r, double* z, double* Zcols) {
    apply_precond(r, z, Zcols);
    project(z, 1, su.m);
  }

  // K15 persistent PCG / FO loop (kernels_persist.cuh): grid size (0 = not
  // applicable / disabled), barrier kind, launch
  bool persist_cluster = false;
  int solve_loop = 0;   // fetigpu_stats::solve_loop of the last PCG / FO solve
  int p_state = 0;   // 0 unknown, 1 ready, -1 not applicable (a row without one or two owners)
  DBuf<int4> p_op_ent, p_pc_ent;
  DBuf<double2> p_op_c, p_pc_c;
  DBuf<unsigned char> p_pc_wr;
  DBuf<int> p_voff_op, p_voff_pc;
  DBuf<double> p_vop, p_vpc, p_w2, p_r2;
  DBuf<unsigned int> p_bar;
  bool persist_prepare();
  size_t persist_smem() const;
  // FETIGPU_PERSIST_RED=1: small coarse operators applied redundantly by the
  // CTAs that need them instead of in their own grid phase (measured slower)
  static bool persist_red() {
    static const bool on = [] {
      const char* e = getenv("FETIGPU_PERSIST_RED");
      return e && e[0] == '1';
    }();
    return on;
  }
  int persist_grid(bool fo);
  std::vector<int> pc_nsld;   // per subdomain: n_s x ld of its preconditioner matrix (K15c)
  size_t cluster_smem() const;
  bool cluster_ok(bool fo);
  bool launch_cluster(double* lam, double* r, double* w, Scal* sc, IterCtl* ctl, double* trace);
  bool launch_persist(int G, bool fo, int passes, int psi_S, double* lam, double* r, double* z, double* w, double* q,
                      Scal* sc, double* Wst, double* Qst, double* psi, double* psi_part, int* cnt, IterCtl* ctl,
                      double* trace);
  int solve(const fetigpu_solve_opts& o, double* lambda_host, fetigpu_trace* tr);
  int solve_rrs(const fetigpu_solve_opts& o, double* lam, fetigpu_trace* tr);
  int solve_rrs_implicit(const fetigpu_solve_opts& o, double* lam, fetigpu_trace* tr);
  bool use_implicit_store(const fetigpu_solve_opts& o);
  int rrs_store = 0;   // FETIGPU_RRS_STORE_AUTO / _EXPLICIT / _IMPLICIT
  // invariant check of the stored search directions (fetigpu_set_check):
  // after each FO / RRS solve, chk_err = max |W^T F W - I| over all stored
  // F-normalised directions, chk_n = their number
  bool chk_on = false;
  double chk_err = -1.0;
  int chk_n = 0;
  // blocks (W_b, Q_b = F W_b), column-major m x r_b (ld m): max |W^T Q - I|
  // row_major: blocks are row-major m x r_b (ld r_b) instead
  void check_orth(const std::vector<const double*>& Ws, const std::vector<const double*>& Qs,
                  const std::vector<int>& rs, bool row_major = false) {
    const int m = su.m;
    int K = 0;
    for (int r : rs) K += r;
    std::vector<double> G((size_t)K * K);
    DBuf<double> g;
    int ra0 = 0;
    for (size_t a = 0; a < Ws.size(); ++a) {
      int rb0 = 0;
      for (size_t b = 0; b < Qs.size(); ++b) {
        g.alloc((size_t)rs[a] * rs[b]);
        // each inner product in double-double (test hook: the check must not
        // add its own cancellation error to the measured loss of conjugacy)
        const long long sw = row_major ? 1 : m, ew = row_major ? rs[a] : 1;
        const long long sq = row_major ? 1 : m, eq = row_major ? rs[b] : 1;
        k_dot_dd<<<dim3(rs[a], rs[b]), 256, 0, st>>>(Ws[a], sw, ew, Qs[b], sq, eq, m, g.p, rs[a]);
        LAUNCH_CHECK();
        std::vector<double> h((size_t)rs[a] * rs[b]);
        CK(cudaMemcpyAsync(h.data(), g.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int j = 0; j < rs[b]; ++j)
          for (int i = 0; i < rs[a]; ++i) G[(size_t)(rb0 + j) * K + ra0 + i] = h[(size_t)j * rs[a] + i];
        rb0 += rs[b];
      }
      ra0 += rs[a];
    }
    double e = 0.0;
    for (int j = 0; j < K; ++j)
      for (int i = 0; i < K; ++i) e = std::max(e, std::fabs(G[(size_t)j * K + i] - (i == j ? 1.0 : 0.0)));
    chk_err = e;
    chk_n = K;
  }
};

}  // namespace fg
