// ctx_ops.cuh -- operator applications: F (K4 single column, K5 block, host-pipelined),
// preconditioner, T-FETI projector, right-hand side and primal recovery.
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include "ctx.cuh"

namespace fg {

// b_i = p[src_i] - sum_D S[src_i, D] g - sum_c S[src_i, c] u_c  with
// p = f - B_s^T lambda on the perimeter
__global__ void k_bnd_rhs(int nb, const double* __restrict__ fb, const double* __restrict__ lambda,
                          const OpSub* __restrict__ ops, const int* __restrict__ rows,
                          const double* __restrict__ coefs, int KR, const int* __restrict__ top_pos,
                          const int* __restrict__ top_off, const int* __restrict__ D,
                          const int* __restrict__ D_off, const int* __restrict__ D_cnt,
                          const double* __restrict__ gD, const int* __restrict__ c_pos,
                          const int* __restrict__ c_off, const int* __restrict__ cmap,
                          const DpSub* __restrict__ dps, const double* __restrict__ uc,
                          const double* __restrict__ S, const int* __restrict__ design,
                          const int* __restrict__ slot_of, const int* __restrict__ src,
                          const int* __restrict__ src_off, const int* __restrict__ nes,
                          double* __restrict__ xb, const int* __restrict__ xoff) {
  extern __shared__ double p[];
  const int s = blockIdx.x;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) p[i] = fb[(size_t)s * nb + i];
  __syncthreads();
  if (lambda) {
    const OpSub d = ops[s];
    for (int a = threadIdx.x; a < d.ns; a += blockDim.x) {
      double v = 0.0;
      for (int k = 0; k < KR; ++k) {
        const int r = rows[d.map_off + a * KR + k];
        if (r >= 0) v += coefs[d.map_off + a * KR + k] * lambda[r];
      }
      p[top_pos[top_off[s] + a]] -= v;
    }
    __syncthreads();
  }
  const int sl = slot_of[s];
  const int ne = nes[sl];
  const int* sr = src + src_off[sl];
  const double* Sd = S + (size_t)design[s] * nb * nb;
  const int nD = D_cnt[s];
  const int nc = (uc && dps) ? dps[s].nc : 0;
  for (int i = threadIdx.x; i < ne; i += blockDim.x) {
    const int pi = sr[i];
    double v = p[pi];
    for (int k = 0; k < nD; ++k) v -= Sd[(size_t)D[D_off[s] + k] * nb + pi] * gD[D_off[s] + k];
    for (int k = 0; k < nc; ++k)
      v -= Sd[(size_t)c_pos[c_off[s] + k] * nb + pi] * uc[cmap[dps[s].cmap_off + k]];
    xb[xoff[s] + i] = v;
  }
}
void Ctx::launch_bnd_rhs(const double* lambda, const double* uc) {
  k_bnd_rhs<<<su.Ns, kThreads, su.nb * 8, st>>>(
      su.nb, d_fb.p, lambda, d_op.p, d_oprows.p, d_opcoef.p, KR, d_top_pos.p, d_top_off.p, d_D.p, d_D_off.p,
      d_D_cnt.p, d_gD.p, d_c_pos.p, d_c_off.p, d_cmap.p, su.method == FETIGPU_FETIDP ? d_dp.p : nullptr, uc,
      d_S.p, d_design.p, d_slot_of.p, d_op_src.p, d_op_src_off.p, d_fac_ne.p, d_xb.p, d_xoff.p);
  LAUNCH_CHECK();
}

// d[row] += sign * x[ext[a]] over the operator support (B K^+ f)
__global__ void k_rhs_scatter(const OpSub* __restrict__ ops, const int* __restrict__ rows,
                              const double* __restrict__ coefs, int KR, const int* __restrict__ slot_of,
                              const int* __restrict__ ext, const int* __restrict__ ext_off,
                              const double* __restrict__ xb, const int* __restrict__ xoff,
                              double* __restrict__ out) {
  const int s = blockIdx.x;
  const OpSub d = ops[s];
  const int* e = ext + ext_off[slot_of[s]];
  for (int a = threadIdx.x; a < d.ns; a += blockDim.x) {
    const double v = xb[xoff[s] + e[a]];
    for (int k = 0; k < KR; ++k) {
      const int r = rows[d.map_off + a * KR + k];
      if (r >= 0) atomicAdd(out + r, coefs[d.map_off + a * KR + k] * v);
    }
  }
}
void Ctx::launch_rhs_scatter(double* out) {
  k_rhs_scatter<<<su.Ns, kThreads, 0, st>>>(d_op.p, d_oprows.p, d_opcoef.p, KR, d_slot_of.p, d_op_ext.p,
                                            d_op_ext_off.p, d_xb.p, d_xoff.p, out);
  LAUNCH_CHECK();
}

// fbar_c^s = f_c - S[c,D] g - S[c, r] x   (x = S_rr^{-1} b on r)
__global__ void k_dp_fbar(int nb, const double* __restrict__ fb, const int* __restrict__ D,
                          const int* __restrict__ D_off, const int* __restrict__ D_cnt,
                          const double* __restrict__ gD, const int* __restrict__ c_pos,
                          const int* __restrict__ c_off, const DpSub* __restrict__ dps,
                          const double* __restrict__ S, const int* __restrict__ design,
                          const int* __restrict__ slot_of, const int* __restrict__ src,
                          const int* __restrict__ src_off, const int* __restrict__ nes,
                          const double* __restrict__ xb, const int* __restrict__ xoff,
                          double* __restrict__ fbar) {
  const int s = blockIdx.x;
  const DpSub dp = dps[s];
  const int sl = slot_of[s];
  const int ne = nes[sl];
  const int* sr = src + src_off[sl];
  const double* Sd = S + (size_t)design[s] * nb * nb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < dp.nc; k += blockDim.x >> 5) {
    const int cp = c_pos[c_off[s] + k];
    double v = 0.0;
    for (int i = lane; i < ne; i += 32) v += Sd[(size_t)sr[i] * nb + cp] * xb[xoff[s] + i];
    for (int q = lane; q < D_cnt[s]; q += 32) v += Sd[(size_t)D[D_off[s] + q] * nb + cp] * gD[D_off[s] + q];
    v = warp_sum(v);
    if (lane == 0) fbar[dp.t_off + k] = fb[(size_t)s * nb + cp] - v;
  }
}
void Ctx::launch_dp_fbar() {
  k_dp_fbar<<<su.Ns, kThreads, 0, st>>>(su.nb, d_fb.p, d_D.p, d_D_off.p, d_D_cnt.p, d_gD.p, d_c_pos.p,
                                        d_c_off.p, d_dp.p, d_S.p, d_design.p, d_slot_of.p, d_op_src.p,
                                        d_op_src_off.p, d_fac_ne.p, d_xb.p, d_xoff.p, d_fbar_loc.p);
  LAUNCH_CHECK();
}

// perimeter displacement: ub[src_i] = x_i; FETI-DP adds corners and supports
__global__ void k_bnd_u(int nb, const int* __restrict__ slot_of, const int* __restrict__ src,
                        const int* __restrict__ src_off, const int* __restrict__ nes,
                        const double* __restrict__ xb, const int* __restrict__ xoff,
                        const int* __restrict__ D, const int* __restrict__ D_off,
                        const int* __restrict__ D_cnt, const double* __restrict__ gD,
                        const int* __restrict__ c_pos, const int* __restrict__ c_off,
                        const DpSub* __restrict__ dps, const int* __restrict__ cmap,
                        const double* __restrict__ uc, double* __restrict__ ub) {
  const int s = blockIdx.x;
  double* u = ub + (size_t)s * nb;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) u[i] = 0.0;
  __syncthreads();
  const int sl = slot_of[s];
  const int* sr = src + src_off[sl];
  for (int i = threadIdx.x; i < nes[sl]; i += blockDim.x) u[sr[i]] = xb[xoff[s] + i];
  for (int k = threadIdx.x; k < D_cnt[s]; k += blockDim.x) u[D[D_off[s] + k]] = gD[D_off[s] + k];
  if (dps && uc)
    for (int k = threadIdx.x; k < dps[s].nc; k += blockDim.x)
      u[c_pos[c_off[s] + k]] = uc[cmap[dps[s].cmap_off + k]];
}
void Ctx::launch_bnd_u(const double* uc, double* ub_all) {
  k_bnd_u<<<su.Ns, kThreads, 0, st>>>(su.nb, d_slot_of.p, d_op_src.p, d_op_src_off.p, d_fac_ne.p, d_xb.p,
                                      d_xoff.p, d_D.p, d_D_off.p, d_D_cnt.p, d_gD.p, d_c_pos.p, d_c_off.p,
                                      su.method == FETIGPU_FETIDP ? d_dp.p : nullptr, d_cmap.p, uc, ub_all);
  LAUNCH_CHECK();
}
__global__ void k_scatter_perim(int nb, int nloc, const int* __restrict__ pdof, const double* __restrict__ ub,
                                double* __restrict__ u) {
  const int s = blockIdx.x;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) u[(size_t)s * nloc + pdof[i]] = ub[(size_t)s * nb + i];
}
void Ctx::launch_scatter_perim(const double* ub_all, double* u) {
  DBuf<int> pd;
  pd.upload(su.perim_dof, st);
  k_scatter_perim<<<su.Ns, kThreads, 0, st>>>(su.nb, su.nloc, pd.p, ub_all, u);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(st));
}
__global__ void k_add_rigid(int nloc, const double* __restrict__ R, const double* __restrict__ alpha,
                            double* __restrict__ u) {
  const int s = blockIdx.x;
  const double a0 = alpha[3 * s], a1 = alpha[3 * s + 1], a2 = alpha[3 * s + 2];
  for (int i = threadIdx.x; i < nloc; i += blockDim.x)
    u[(size_t)s * nloc + i] += R[i] * a0 + R[nloc + i] * a1 + R[2 * nloc + i] * a2;
}
void Ctx::launch_add_rigid(double* u, const double* alpha) {
  DBuf<double> R;
  R.upload(su.Rfull, st);
  k_add_rigid<<<su.Ns, kThreads, 0, st>>>(su.nloc, R.p, alpha, u);
  LAUNCH_CHECK();
  CK(cudaStreamSynchronize(st));
}

void Ctx::init_device() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(FETIGPU_E_NO_DEVICE, "no CUDA device available");
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  CK(cudaEventCreate(&ev2));
  d_status.alloc(1);
  d_status.zero(st);
  CK(cudaFuncSetAttribute(k_nd_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kSmallFront * kSmallFront * 8));
  CK(cudaFuncSetAttribute(k_front_elim_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kSmallFront * kSmallFront * 8));
  CK(cudaFuncSetAttribute(k_block_apply<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlockSmem));
  CK(cudaFuncSetAttribute(k_block_apply<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlockSmem));
  CK(cudaFuncSetAttribute(k_block_apply_dp, cudaFuncAttributeMaxDynamicSharedMemorySize, kAsyncSmem));
}

void Ctx::coarse_solve_packed(bool g_ready, double* zero_y) {
  if (!g_ready || su.Nc == 0) {
    launch_pdl(k_coarse_gather, grid_for(std::max(su.Nc, zero_y ? su.m : 0)), kThreads, 0, st,
               (const int*)d_optr.p, (const int*)d_oidx.p, (const double*)d_tbuf.p, su.Nc, d_gc.p, 1.0,
               (const double*)nullptr, zero_y, zero_y ? su.m : 0);
    LAUNCH_CHECK();
  }
  if (su.Nc == 0) return;
  if (!use_csym) {  // small coarse problem: dense L2-resident inverse, one launch
    launch_pdl(k_dense_gemv, grid_for((long long)su.Nc * 32), kThreads, 0, st, (const double*)d_Kinv.p, su.Nc,
               (const double*)d_gc.p, d_h.p);
    LAUNCH_CHECK();
    return;
  }
  launch_pdl(k_csym_tiles, csym_grid, 128, 0, st, (const double*)d_kinv_tiles.p, kinv_nb, su.Nc,
             (const double*)d_gc.p, d_crow.p, d_ccol.p);
  launch_pdl(k_csym_reduce, kinv_nb, 512, 0, st, (const double*)d_crow.p, (const double*)d_ccol.p, kinv_nb,
             su.Nc, d_h.p);
  LAUNCH_CHECK();
}

// The symmetric-packed GEMV (K4 / K7 at C4 sizes) over subdomains [s0, s0+n):
// the TMA ring kernel on a persistent grid (default) or the LDG kernel with
// one CTA per subdomain (FETIGPU_SYM_TMA=0); bit-identical results.
void Ctx::launch_sym(cudaStream_t q, const SymArgs& a) {
  if (a.n <= 0) return;
  const SymSub* subs = a.pc ? d_pcsym.p : d_sym.p;
  const double* tiles = a.pc ? d_pcsymtiles.p : d_symtiles.p;
  const int* rows = a.pc ? d_pcrows.p : d_oprows.p;
  const double* coefs = a.pc ? d_pccoef.p : d_opcoef_apply.p;
  double* vbuf = a.store_v ? d_vbuf.p : nullptr;
  const int* voff = a.store_v ? d_voff.p : nullptr;
  const DpSub* dps = a.store_v ? d_dp.p : nullptr;
  const double* abc = a.store_v ? d_abc.p : nullptr;
  double* tbuf = a.store_v ? d_tbuf.p : nullptr;
  const int ny = a.zero_y ? su.m : 0, nsub = a.zero_y ? su.Ns : 1;
  const CoarseGather* cgp = a.coarse_gather && su.Nc ? d_cgather.p : nullptr;
  const int* wflag = a.wait_x ? d_xflag.p : nullptr;
  const int* wneed = a.wait_x ? d_subneed.p : nullptr;
  auto go = [&](auto ktma, auto kldg) {
    if (sym_tma) {
      const int ring = a.pc ? pc_sym_ring : sym_ring, npad = a.pc ? pc_sym_npad : sym_npad;
      const size_t smem = a.pc ? pc_sym_tma_bytes : sym_tma_bytes;
      const int grid = a.per_cta ? a.n : std::min(a.n, sym_grid);
      if (a.pdl)
        launch_pdl(ktma, grid, 256, smem, q, subs, tiles, rows, coefs, a.x, a.y, vbuf, voff, dps, abc, tbuf, a.s0,
                   a.s0 + a.n, a.zero_y, ny, nsub, cgp, ring, npad, sym_flags, wflag, wneed);
      else
        ktma<<<grid, 256, smem, q>>>(subs, tiles, rows, coefs, a.x, a.y, vbuf, voff, dps, abc, tbuf, a.s0,
                                     a.s0 + a.n, a.zero_y, ny, nsub, cgp, ring, npad, sym_flags, wflag, wneed);
    } else {
      const int smem = a.pc ? pc_sym_smem : sym_smem;
      if (a.pdl)
        launch_pdl(kldg, a.n, 256, smem, q, subs, tiles, rows, coefs, a.x, a.y, vbuf, voff, dps, abc, tbuf, a.s0,
                   a.zero_y, ny, nsub, cgp);
      else
        kldg<<<a.n, 256, smem, q>>>(subs, tiles, rows, coefs, a.x, a.y, vbuf, voff, dps, abc, tbuf, a.s0, a.zero_y,
                                    ny, nsub, cgp);
    }
  };
  if (a.store_v) go(k_sym_gemv_tma<1, true>, k_sym_gemv_scatter<1, true>);
  else if (a.kr == 1) go(k_sym_gemv_tma<1, false>, k_sym_gemv_scatter<1, false>);
  else go(k_sym_gemv_tma<3, false>, k_sym_gemv_scatter<3, false>);
}

void Ctx::apply_F(const double* x, double* y, int ncols, int ldx, int ldy, bool y_zeroed) {
  const int Ns = su.Ns;
  if (su.method == FETIGPU_TFETI) {
    if (ncols == 1 && y_zeroed) {
      if (use_sym) {
        SymArgs sa;
        sa.kr = 3; sa.x = x; sa.y = y; sa.n = Ns; sa.pdl = true;
        launch_sym(st, sa);
      } else
        launch_pdl(k_gather_gemv_scatter<3, false>, dim3(Ns, 1, rsplit), kThreads, max_ld * 8, st,
                   (const OpSub*)d_op.p, (const double*)d_opmat.p, (const int*)d_oprows.p,
                   (const double*)d_opcoef_apply.p, x, y, (double*)nullptr, 0, (double*)nullptr,
                   (const int*)nullptr, ldx, ldy, 1, (const DpSub*)nullptr, (const double*)nullptr,
                   (double*)nullptr);
      LAUNCH_CHECK();
      return;
    }
    for (int c = 0; c < ncols; ++c) CK(cudaMemsetAsync(y + (size_t)c * ldy, 0, su.m * 8, st));
    if (use_sym) {
      for (int c = 0; c < ncols; ++c) {
        SymArgs sa;
        sa.kr = 3; sa.x = x + (size_t)c * ldx; sa.y = y + (size_t)c * ldy; sa.n = Ns;
        launch_sym(st, sa);
      }
    } else {
      dim3 grid(Ns, ncols, rsplit);
      k_gather_gemv_scatter<3, false><<<grid, kThreads, max_ld * 8, st>>>(
          d_op.p, d_opmat.p, d_oprows.p, d_opcoef_apply.p, x, y, nullptr, 0, nullptr, nullptr, ldx, ldy);
    }
    LAUNCH_CHECK();
  } else {
    for (int c = 0; c < ncols; ++c) {
      const double* xc = x + (size_t)c * ldx;
      double* yc = y + (size_t)c * ldy;
      // phase 1: v_s = F''_s x_s and t_s = A''^T x_s (one kernel; it also zeroes y)
      if (use_sym) {
        SymArgs sa;
        sa.store_v = true; sa.x = xc; sa.n = Ns; sa.zero_y = yc; sa.coarse_gather = true; sa.pdl = true;
        launch_sym(st, sa);
      } else {
        launch_pdl(k_gather_gemv_scatter<1, true>, dim3(Ns, 1, rsplit), kThreads, max_ld * 8, st,
                   (const OpSub*)d_op.p, (const double*)d_opmat.p, (const int*)d_oprows.p,
                   (const double*)d_opcoef_apply.p, xc, (double*)nullptr, (double*)nullptr, 0, d_vbuf.p,
                   (const int*)d_voff.p, ldx, 0, 1, (const DpSub*)d_dp.p, (const double*)d_abc.p, d_tbuf.p);
      }
      // coarse: u = Kbar^{-1} (sum_s B_c^T t_s), fixed order (y zeroed here on the non-symmetric path)
      coarse_solve_packed(use_sym, use_sym ? nullptr : yc);
      // phase 2: y = sum_s B_s (v_s + A''_s u_s)
      launch_phase2_csym(yc);
      LAUNCH_CHECK();
    }
  }
}

void Ctx::setup_pipe() {
  pipe_ready = false;
  const char* off = getenv("FETIGPU_NO_PIPE");
  if ((off && off[0] == '1') || !use_sym || su.method != FETIGPU_FETIDP || su.Ns < 4 * kPipe) return;
  int run = -1;
  for (int c = 0; c < kPipe; ++c) {
    pipe_s0[c] = (int)((long long)su.Ns * c / kPipe);
    pipe_s0[c + 1] = (int)((long long)su.Ns * (c + 1) / kPipe);
    for (int s = pipe_s0[c]; s < pipe_s0[c + 1]; ++s) run = std::max(run, sub_maxrow[s]);
    pipe_need[c] = run + 1;  // rows [0, need) cover every row chunks 0..c gather
  }
  // worthwhile only if the first chunks need a real prefix of lambda
  if (pipe_need[kPipe / 2 - 1] > (long long)su.m * 3 / 4) return;
  if (!pipe_cp) {
    CK(cudaStreamCreateWithFlags(&pipe_cp, cudaStreamNonBlocking));
    for (int c = 0; c < kPipe; ++c) {
      CK(cudaStreamCreateWithFlags(&pipe_st[c], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&pipe_in[c], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&pipe_done[c], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&pipe_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&pipe_cp_done, cudaEventDisableTiming));
  }
  // flag value after chunk c has landed: c + 1
  {
    std::vector<int> need(su.Ns);
    for (int s = 0; s < su.Ns; ++s) {
      int c = 0;
      while (c < kPipe - 1 && pipe_need[c] <= sub_maxrow[s]) ++c;
      need[s] = c + 1;
    }
    d_subneed.upload(need, st);
    d_xflag.alloc(1);
    d_xflag.zero(st);
    if (!h_flagvals) {
      CK(cudaMallocHost(&h_flagvals, kPipe * sizeof(int)));
      for (int c = 0; c < kPipe; ++c) h_flagvals[c] = c + 1;
    }
  }
  pipe_ready = true;
}

void Ctx::apply_F_host(const double* xh, double* yh) {
  const int m = su.m;
  stage(m);
  double* x = stage_x.p;
  double* y = stage_y.p;
  if (!pipe_ready) {
    CK(cudaMemcpyAsync(x, xh, (size_t)m * 8, cudaMemcpyHostToDevice, st));
    apply_F(x, y, 1, m, m);
  } else if (sym_tma && pipe_flagged()) {
    // ONE persistent phase-1 kernel, launched before x has arrived: it
    // requests its first operator tiles at once, and every subdomain's gather
    // waits until the copy stream has flagged the row prefix it needs
    CK(cudaMemsetAsync(d_xflag.p, 0, 4, st));
    CK(cudaEventRecord(pipe_start, st));  // after everything already queued on st
    CK(cudaStreamWaitEvent(pipe_cp, pipe_start, 0));
    int done = 0;
    for (int c = 0; c < kPipe; ++c) {
      const int need = c == kPipe - 1 ? m : pipe_need[c];
      if (need > done) {
        CK(cudaMemcpyAsync(x + done, xh + done, (size_t)(need - done) * 8, cudaMemcpyHostToDevice, pipe_cp));
        done = need;
      }
      // the flag is stored by the copy engine: a memset kernel could not be scheduled beside the
      // persistent kernel (it holds every SM's registers) and the two would wait on each other
      CK(cudaMemcpyAsync(d_xflag.p, h_flagvals + c, 4, cudaMemcpyHostToDevice, pipe_cp));
    }
    CK(cudaEventRecord(pipe_cp_done, pipe_cp));
    SymArgs sa;
    sa.store_v = true; sa.x = x; sa.n = su.Ns; sa.zero_y = y; sa.coarse_gather = true; sa.wait_x = true;
    launch_sym(st, sa);
    LAUNCH_CHECK();
    CK(cudaStreamWaitEvent(st, pipe_cp_done, 0));
    coarse_solve_packed(true);
    launch_phase2_csym(y);
    LAUNCH_CHECK();
  } else {
    CK(cudaEventRecord(pipe_start, st));  // after everything already queued on st
    CK(cudaStreamWaitEvent(pipe_cp, pipe_start, 0));
    int done = 0;
    for (int c = 0; c < kPipe; ++c) {
      const int need = c == kPipe - 1 ? m : pipe_need[c];
      if (need > done) {
        CK(cudaMemcpyAsync(x + done, xh + done, (size_t)(need - done) * 8, cudaMemcpyHostToDevice, pipe_cp));
        done = need;
      }
      CK(cudaEventRecord(pipe_in[c], pipe_cp));
    }
    for (int c = 0; c < kPipe; ++c) {
      cudaStream_t q = pipe_st[c];
      CK(cudaStreamWaitEvent(q, pipe_in[c], 0));
      const int nblk = pipe_s0[c + 1] - pipe_s0[c];
      SymArgs sa;
      sa.store_v = true; sa.x = x; sa.s0 = pipe_s0[c]; sa.n = nblk; sa.zero_y = y; sa.coarse_gather = true;
      sa.per_cta = true;
      launch_sym(q, sa);
      LAUNCH_CHECK();
      CK(cudaEventRecord(pipe_done[c], q));
      CK(cudaStreamWaitEvent(st, pipe_done[c], 0));
    }
    // coarse u = Kbar^{-1} (sum_s B_c^T t_s) on the packed inverse; phase 2
    coarse_solve_packed(true);
    launch_phase2_csym(y);
    LAUNCH_CHECK();
  }
  CK(cudaMemcpyAsync(yh, y, (size_t)m * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

void Ctx::apply_precond(const double* r, double* z, double* Zcols, bool row_major, bool z_zeroed) {
  if (!z_zeroed) CK(cudaMemsetAsync(z, 0, su.m * 8, st));
  if (Zcols) CK(cudaMemsetAsync(Zcols, 0, (size_t)su.m * su.Ns * 8, st));
  const int ldz = row_major ? 1 : su.m, zrs = row_major ? su.Ns : 1;
  if (pc_sym && !Zcols) {
    SymArgs sa;
    sa.pc = true; sa.kr = KRp == 1 ? 1 : 3; sa.x = r; sa.y = z; sa.n = su.Ns; sa.pdl = true;
    launch_sym(st, sa);
    LAUNCH_CHECK();
    return;
  }
  auto k = KRp == 1 ? k_gather_gemv_scatter<1, false> : k_gather_gemv_scatter<3, false>;
  launch_pdl(k, dim3(su.Ns, 1, pc_rsplit), kThreads, max_pc_ld * 8, st, (const OpSub*)d_pc.p,
             (const double*)d_pcmat.p, (const int*)d_pcrows.p, (const double*)d_pccoef.p, r, z, Zcols, ldz,
             (double*)nullptr, (const int*)nullptr, 0, 0, zrs, (const DpSub*)nullptr, (const double*)nullptr,
             (double*)nullptr);
  LAUNCH_CHECK();
}

void Ctx::apply_F_block(const double* W, int ldw, double* Q, int ldq, int k) {
  const int Ns = su.Ns, m = su.m;
  // Q is zeroed for K5's scatter.  FETI-DP: on a side stream while the DMMA
  // GEMM of U runs (HBM-bound memset vs FP64-bound GEMM), joined before K5
  // (FETIGPU_K5_SERIAL=1: on the main stream)
  static const bool serial = [] {
    const char* e = getenv("FETIGPU_K5_SERIAL");
    return e && e[0] == '1';
  }();
  const bool side = su.method == FETIGPU_FETIDP && !serial;
  cudaStream_t zs = st;
  if (side) {
    if (!aux_st) {
      CK(cudaStreamCreateWithFlags(&aux_st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&aux_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&aux_join, cudaEventDisableTiming));
    }
    zs = aux_st;
  }
  auto zero_q = [&]() {
    if (side) {
      CK(cudaEventRecord(aux_fork, st));
      CK(cudaStreamWaitEvent(aux_st, aux_fork, 0));
    }
    if (ldq == k) CK(cudaMemsetAsync(Q, 0, (size_t)m * k * 8, zs));
    else CK(cudaMemset2DAsync(Q, (size_t)ldq * 8, 0, (size_t)k * 8, m, zs));
    if (side) CK(cudaEventRecord(aux_join, aux_st));
  };
  // K5e (FETIGPU_K5_EDGE=1): by interface edge -- no memset, Q written once,
  // bit-identical.  C4 k = 2048 on one B200: DRAM 31.5 GB per kernel against
  // 35.9 GB + the 8.3 GB memset, but 68.2 vs 65.8 ms of kernel time (the
  // mid-tile store after the first owner stalls the MMA loop), so K5 stays
  // the default: the block apply is FP64-bound, not HBM-bound
  const char* ee = getenv("FETIGPU_K5_EDGE");   // read per call (tests switch it)
  const bool edge_on = ee && ee[0] == '1';
  const bool edge = edge_on && su.method == FETIGPU_FETIDP && folded && blk_aligned && (k % 2 == 0) &&
                    (ldw % 2 == 0) && (ldq % 2 == 0) && ((uintptr_t)W % 16 == 0) && ((uintptr_t)Q % 16 == 0) &&
                    bz_prepare();
  if (!side && !edge) zero_q();
  // K5 walks the subdomains in 4 x 4-module tiles: both neighbours sharing a
  // dual row (left/right and below/above) are processed close in time, so
  // the W rows of an interface are read from DRAM about once
  if (d_k5order.n != (size_t)Ns) {
    std::vector<int> ord;
    ord.reserve(Ns);
    for (int ty = 0; ty < su.sy; ty += 4)
      for (int tx = 0; tx < su.sx; tx += 4)
        for (int y = ty; y < std::min(su.sy, ty + 4); ++y)
          for (int x = tx; x < std::min(su.sx, tx + 4); ++x) ord.push_back(y * su.sx + x);
    d_k5order.upload(ord, st);
  }
  static const bool tiled = [] {
    const char* e = getenv("FETIGPU_K5_ROWMAJOR");
    return !(e && e[0] == '1');
  }();
  static const bool pre_tiled = [] {   // the coarse pre-pass in the same walk (FETIGPU_DPT_TILED=0: natural)
    const char* e = getenv("FETIGPU_DPT_TILED");
    return tiled && !(e && e[0] == '0');
  }();
  BlockApplyArgs a{d_op.p, d_opmat.p, d_oprows.p, d_opcoef_apply.p, KR, nullptr, nullptr, nullptr, nullptr, 0,
                   W, ldw, Q, ldq, k, tiled ? d_k5order.p : nullptr};
  int max_ns = 0;
  for (int n : op_ns) max_ns = std::max(max_ns, n);
  if (su.method == FETIGPU_FETIDP) {
    const int Nc = su.Nc;
    ensure_block_buffers(k);
    {
      const size_t smem = ((size_t)std::max(max_ns * 8, 4 * 8 * kDpTCols) + max_ns) * 8 + (size_t)max_ns * 4;
      raise_smem_limit(k_block_dp_t, smem);
      k_block_dp_t<<<dim3((k + kDpTCols - 1) / kDpTCols, Ns), 256, smem, st>>>(
          d_op.p, d_dp.p, d_oprows.p, d_opcoef_apply.p, d_abc.p, W, ldw, k, blk_t.p, k, pre_tiled ? d_k5order.p : nullptr);
    }
    k_coarse_gather_block<<<dim3((k + 255) / 256, Nc), 256, 0, st>>>(d_optr.p, d_oidx.p, blk_t.p, k, Nc, k,
                                                                     blk_T.p, k);
    if (!edge) zero_q();   // side stream: overlaps the FP64-bound GEMM, not the HBM-bound pre-pass
    // U = Kbar^{-1} T  (row-major N_c x k == column-major k x N_c: U^T = T^T Kinv)
    gemm(st, false, false, k, Nc, Nc, 1.0, blk_T.p, k, d_Kinv.p, Nc, 0.0, blk_U.p, k);
    a.dps = d_dp.p; a.abc = d_abc.p; a.cmap = d_cmap.p; a.U = blk_U.p; a.ldu = k;
    max_ns += 8;
  }
  if (side && !edge) CK(cudaStreamWaitEvent(st, aux_join, 0));
  if (edge) {
    if (d_k5e_order.n != (size_t)bz_nedges) {   // edge chunks in K5's 4 x 4-module walk of their first owner
      std::vector<BzEdge> es(bz_nedges);
      CK(cudaMemcpyAsync(es.data(), bz_edges.p, bz_nedges * sizeof(BzEdge), cudaMemcpyDeviceToHost, st));
      std::vector<int> ord(Ns), pos(Ns);
      CK(cudaMemcpyAsync(ord.data(), d_k5order.p, Ns * sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int i = 0; i < Ns; ++i) pos[ord[i]] = i;
      std::vector<int> eo(bz_nedges);
      std::iota(eo.begin(), eo.end(), 0);
      std::stable_sort(eo.begin(), eo.end(), [&](int x, int y) { return pos[es[x].t1] < pos[es[y].t1]; });
      d_k5e_order.upload(eo, st);
    }
    constexpr int BM = 64, BN = 64;
    const int mt = (kBzRows + BM - 1) / BM;
    const size_t smem = k5e_smem<64, 64, 16, 2>(max_ns);   // max_ns already counts the n_c <= 8 coarse columns
    raise_smem_limit(k_block_apply_edge<64, 64, 16, 2>, smem);
    EdgeApplyArgs ea{bz_edges.p, bz_erow.p, bz_eb1.p, bz_eb2.p, d_k5e_order.p, mt};
    k_block_apply_edge<64, 64, 16, 2><<<dim3((k + BN - 1) / BN, bz_nedges * mt), 128, smem, st>>>(a, ea);
    LAUNCH_CHECK();
    return;
  }
  dim3 grid((k + kBN - 1) / kBN, (max_ns + kBM - 1) / kBM, Ns);
  const bool fast = folded && blk_aligned && (k % 2 == 0) && (ldw % 2 == 0) && (ldq % 2 == 0) &&
                    ((uintptr_t)W % 16 == 0) && ((uintptr_t)Q % 16 == 0);
  // tile of the fast path (FETIGPU_K5_CFG, C4 k = 2048 block apply on a
  // B200, bit-identical results): 0 = 128 x 64 x 16 / 3 stages / 2 CTAs per
  // SM 75.4 ms; 1 = 64 x 64 x 16 / 3 76.6; 2 = 64 x 64 x 32 / 2 74.1;
  // 3 = 64 x 64 x 16 / 2 (4 CTAs per SM) 72.8 (default); 4 = 128 x 64 x 16 /
  // 3 (templated) 75.3; 5 = 64 x 128 x 16 / 3 74.7
  static const int k5cfg = [] {
    const char* e = getenv("FETIGPU_K5_CFG");
    return e ? atoi(e) : 3;
  }();
  auto launch2 = [&](auto kern, int BM, int BN, size_t smem, int threads) {
    raise_smem_limit(kern, smem);
    kern<<<dim3((k + BN - 1) / BN, (max_ns + BM - 1) / BM, Ns), threads, smem, st>>>(a);
  };
  if (fast && k5cfg == 1) launch2(k_block_apply_dp2<64, 64, 16, 3>, 64, 64, k5_smem<64, 64, 16, 3>(max_ns + 8), 128);
  else if (fast && k5cfg == 2) launch2(k_block_apply_dp2<64, 64, 32, 2>, 64, 64, k5_smem<64, 64, 32, 2>(max_ns + 8), 128);
  else if (fast && k5cfg == 3) launch2(k_block_apply_dp2<64, 64, 16, 2>, 64, 64, k5_smem<64, 64, 16, 2>(max_ns + 8), 128);
  else if (fast && k5cfg == 4) launch2(k_block_apply_dp2<128, 64, 16, 3>, 128, 64, k5_smem<128, 64, 16, 3>(max_ns + 8), 256);
  else if (fast && k5cfg == 5) launch2(k_block_apply_dp2<64, 128, 16, 3>, 64, 128, k5_smem<64, 128, 16, 3>(max_ns + 8), 256);
  else if (fast) k_block_apply_dp<<<grid, 256, kAsyncSmem, st>>>(a);
  else if (KR == 1) k_block_apply<1><<<grid, 256, kBlockSmem, st>>>(a);
  else k_block_apply<3><<<grid, 256, kBlockSmem, st>>>(a);
  LAUNCH_CHECK();
}

// Sharded F (or preconditioner) apply, phase 1 over the owned subdomains:
// y := 0, then T-FETI / preconditioner: y += sum_{s owned} B_s M_s B_s^T x
// (M = F_s or S~_s, complete for rows with both owners owned); FETI-DP F:
// v_s = F''_s x_s and t_s = A''_s^T x_s for the owned s, t copied into the
// zeroed tot_c vector `tout` at the owned offsets.  The kernels and their
// per-subdomain arithmetic are those of the single-context apply (the
// symmetric-packed / full-matrix choice included), so after the exchanges
// the result equals the 1-GPU apply bit for bit: every dual row has exactly
// two owners (0 + a + b == a + b in any order) and the coarse gather runs on
// the complete t in the fixed owner order.
void Ctx::shard_phase1(const double* x, double* y, double* tout, bool precond) {
  const int s0 = shard_s0, s1 = shard_s1 < 0 ? su.Ns : shard_s1, n = s1 - s0;
  CK(cudaMemsetAsync(y, 0, (size_t)su.m * 8, st));
  if (n <= 0 || su.m == 0) return;
  if (precond) {
    if (pc_sym) {
      SymArgs sa;
      sa.pc = true; sa.kr = KRp == 1 ? 1 : 3; sa.x = x; sa.y = y; sa.s0 = s0; sa.n = n;
      launch_sym(st, sa);
    } else {
      auto k = KRp == 1 ? k_gather_gemv_scatter<1, false> : k_gather_gemv_scatter<3, false>;
      k<<<dim3(n, 1, pc_rsplit), kThreads, max_pc_ld * 8, st>>>(d_pc.p + s0, d_pcmat.p, d_pcrows.p, d_pccoef.p, x,
                                                                  y, nullptr, 0, nullptr, nullptr, su.m, su.m, 1,
                                                                  nullptr, nullptr, nullptr);
    }
    LAUNCH_CHECK();
    return;
  }
  if (su.method == FETIGPU_TFETI) {
    if (use_sym) {
      SymArgs sa;
      sa.kr = 3; sa.x = x; sa.y = y; sa.s0 = s0; sa.n = n;
      launch_sym(st, sa);
    } else
      k_gather_gemv_scatter<3, false><<<dim3(n, 1, rsplit), kThreads, max_ld * 8, st>>>(
          d_op.p + s0, d_opmat.p, d_oprows.p, d_opcoef_apply.p, x, y, nullptr, 0, nullptr, nullptr, su.m, su.m, 1,
          nullptr, nullptr, nullptr);
    LAUNCH_CHECK();
    return;
  }
  if (use_sym) {
    SymArgs sa;
    sa.store_v = true; sa.x = x; sa.s0 = s0; sa.n = n;
    launch_sym(st, sa);
  } else
    k_gather_gemv_scatter<1, true><<<dim3(n, 1, rsplit), kThreads, max_ld * 8, st>>>(
        d_op.p + s0, d_opmat.p, d_oprows.p, d_opcoef_apply.p, x, nullptr, nullptr, 0, d_vbuf.p, d_voff.p + s0,
        su.m, 0, 1, d_dp.p + s0, d_abc.p, d_tbuf.p);
  LAUNCH_CHECK();
  int t0 = 0, t1 = 0;
  for (int s = 0; s < s1; ++s) {
    const int c = (int)su.subs[s].c.size();
    if (s < s0) t0 += c;
    t1 += c;
  }
  if (t1 > t0) CK(cudaMemcpyAsync(tout + t0, d_tbuf.p + t0, (size_t)(t1 - t0) * 8, cudaMemcpyDeviceToDevice, st));
}

// Phase 2 (FETI-DP F only): t complete on every rank -> the coarse gather in
// fixed owner order, u = Kbar^{-1} g (redundant on every rank), then
// y += B_s (v_s + A''_s u_s) for the owned subdomains.
void Ctx::shard_phase2(const double* tall, double* y) {
  if (su.method != FETIGPU_FETIDP || su.m == 0) return;
  const int s0 = shard_s0, s1 = shard_s1 < 0 ? su.Ns : shard_s1, n = s1 - s0;
  const int tc = tot_c();
  if (tc) CK(cudaMemcpyAsync(d_tbuf.p, tall, (size_t)tc * 8, cudaMemcpyDeviceToDevice, st));
  coarse_solve_packed(false, nullptr);
  if (n > 0) {
    k_dp_phase2<<<n, kThreads, 0, st>>>(d_op.p + s0, d_dp.p + s0, d_oprows.p, d_opcoef_apply.p, d_abc.p, d_cmap.p,
                                        d_h.p, d_vbuf.p, y, 1.0);
    LAUNCH_CHECK();
  }
}

void Ctx::init_lambda(double* lam) {
  const int m = su.m;
  if (!warm) {
    CK(cudaMemcpyAsync(lam, d_lam0.p, (size_t)m * 8, cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (su.method == FETIGPU_TFETI) {
    k_sub<<<grid_for(m), kThreads, 0, st>>>(m, d_warm.p, d_lam0.p, lam);   // lam = warm - lam0
    project(lam, 1, m);
    k_axpy<<<grid_for(m), kThreads, 0, st>>>(m, 1.0, d_lam0.p, lam);       // lam += lam0
    LAUNCH_CHECK();
  } else {
    CK(cudaMemcpyAsync(lam, d_warm.p, (size_t)m * 8, cudaMemcpyDeviceToDevice, st));
  }
}

bool Ctx::bz_prepare() {
  if (bz_state) return bz_state > 0;
  bz_state = -1;
  if (su.method != FETIGPU_FETIDP || !folded || KR != 1 || su.m == 0 || su.Nc == 0) return false;
  const int Ns = su.Ns, m = su.m;
  std::vector<OpSub> ops(Ns);
  CK(cudaMemcpyAsync(ops.data(), d_op.p, Ns * sizeof(OpSub), cudaMemcpyDeviceToHost, st));
  long long nmap = 0;
  for (auto& d : ops) nmap = std::max<long long>(nmap, (long long)d.map_off + d.ns);
  std::vector<int> rows(nmap);
  CK(cudaMemcpyAsync(rows.data(), d_oprows.p, nmap * sizeof(int), cudaMemcpyDeviceToHost, st));
  std::vector<DpSub> dps(Ns);
  CK(cudaMemcpyAsync(dps.data(), d_dp.p, Ns * sizeof(DpSub), cudaMemcpyDeviceToHost, st));
  // Z column s lives on the preconditioner map rows of s: they must be the
  // operator map rows of s (as sets) for X_t to have the 2-column structure
  std::vector<OpSub> pcs(Ns);
  CK(cudaMemcpyAsync(pcs.data(), d_pc.p, Ns * sizeof(OpSub), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (KRp != 1) return false;
  long long npc = 0;
  for (auto& d : pcs) npc = std::max<long long>(npc, (long long)d.map_off + d.ns);
  std::vector<int> prow(npc);
  CK(cudaMemcpyAsync(prow.data(), d_pcrows.p, npc * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int t = 0; t < Ns; ++t) {
    if (dps[t].nc > 8) return false;
    std::vector<int> a(rows.begin() + ops[t].map_off, rows.begin() + ops[t].map_off + ops[t].ns);
    std::vector<int> b(prow.begin() + pcs[t].map_off, prow.begin() + pcs[t].map_off + pcs[t].ns);
    a.erase(std::remove(a.begin(), a.end(), -1), a.end());
    b.erase(std::remove(b.begin(), b.end(), -1), b.end());
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    if (a != b) return false;
  }
  // owners of each dual row (ascending subdomain order) and their local positions
  std::vector<int> t1(m, -1), t2(m, -1), b1(m, -1), b2(m, -1);
  for (int t = 0; t < Ns; ++t)
    for (int a = 0; a < ops[t].ns; ++a) {
      const int r = rows[ops[t].map_off + a];
      if (r < 0) continue;
      if (t1[r] < 0) { t1[r] = t; b1[r] = a; }
      else if (t2[r] < 0) { t2[r] = t; b2[r] = a; }
      else return false;   // more than two owners
    }
  // neighbour slots: 0 = itself, then the other owners in first-seen order
  std::vector<int> nbr((size_t)Ns * kZNb, -1), other(nmap, -1), jslot(nmap, 0);
  for (int t = 0; t < Ns; ++t) {
    nbr[(size_t)t * kZNb] = t;
    int cnt = 1;
    for (int a = 0; a < ops[t].ns; ++a) {
      const int r = rows[ops[t].map_off + a];
      if (r < 0) continue;
      const int o = t1[r] == t ? t2[r] : t1[r];
      if (o < 0) continue;
      int j = 1;
      while (j < cnt && nbr[(size_t)t * kZNb + j] != o) ++j;
      if (j == cnt) {
        if (cnt == kZNb) return false;   // more than 4 neighbours: not this structure
        nbr[(size_t)t * kZNb + cnt++] = o;
      }
      other[ops[t].map_off + a] = o;
      jslot[ops[t].map_off + a] = j;
    }
  }
  // positions of each row in its owners' preconditioner maps (the packed Z
  // blocks of the implicit RRS store are laid out on those maps)
  std::vector<long long> pz1(m, -1), pz2(m, -1);
  for (int t = 0; t < Ns; ++t)
    for (int a = 0; a < pcs[t].ns; ++a) {
      const int r = prow[pcs[t].map_off + a];
      if (r < 0) continue;
      if (t == t1[r]) pz1[r] = pcs[t].map_off + a;
      else if (t == t2[r]) pz2[r] = pcs[t].map_off + a;
    }
  // interface edges: rows grouped by their owner pair, chunks of kBzRows
  std::map<std::pair<int, int>, std::vector<int>> groups;
  for (int r = 0; r < m; ++r) {
    if (t1[r] < 0) return false;
    groups[{t1[r], t2[r]}].push_back(r);
  }
  std::vector<BzEdge> edges;
  std::vector<int> erow, eb1, eb2, ez1, ez2;
  for (auto& g : groups)
    for (size_t i0 = 0; i0 < g.second.size(); i0 += kBzRows) {
      const int cnt = (int)std::min<size_t>(kBzRows, g.second.size() - i0);
      edges.push_back({g.first.first, g.first.second, (int)erow.size(), cnt});
      for (int i = 0; i < cnt; ++i) {
        const int r = g.second[i0 + i];
        erow.push_back(r);
        eb1.push_back(b1[r]);
        eb2.push_back(t2[r] >= 0 ? b2[r] : 0);
        ez1.push_back((int)pz1[r]);
        ez2.push_back(t2[r] >= 0 ? (int)pz2[r] : 0);
      }
    }
  for (auto& d : ops) bz_maxns = std::max(bz_maxns, d.ns);
  bz_other.upload(other, st); bz_j.upload(jslot, st); bz_nbr.upload(nbr, st);
  bz_erow.upload(erow, st); bz_eb1.upload(eb1, st); bz_eb2.upload(eb2, st);
  bz_ez1.upload(ez1, st); bz_ez2.upload(ez2, st);
  bz_edges.upload(edges, st);
  bz_nedges = (int)edges.size();
  bz_Y.alloc((size_t)std::max<long long>(1, nmap) * kZNb);
  bz_nmap = nmap;
  {   // owners of each primal in the coarse gather's order: subdomain and tbuf row
    std::vector<int> os, orw;
    for (int pc = 0; pc < su.Nc; ++pc)
      for (auto& ow : su.c_owners[pc]) {
        os.push_back(ow.first);
        orw.push_back(dps[ow.first].t_off + ow.second);
      }
    fz_osub.upload(os, st);
    fz_orow.upload(orw, st);
  }
  CK(cudaStreamSynchronize(st));
  bz_state = 1;
  return true;
}

bool Ctx::apply_F_block_z(const double* Z, double* Q, int k, double* Yout, double* Tout) {
  if (k != su.Ns || !bz_prepare()) return false;
  const int Ns = su.Ns, Nc = su.Nc;
  int tot_c = 0;
  for (auto& S : su.subs) tot_c += (int)S.c.size();
  ensure_block_buffers(k);
  CK(cudaMemsetAsync(blk_t.p, 0, (size_t)tot_c * k * 8, st));
  const size_t smem = (size_t)bz_maxns * 20;
  raise_smem_limit(k_bz_local, smem);
  double* Y = Yout ? Yout : bz_Y.p;
  double* T = blk_T.p;
  k_bz_local<<<Ns, 256, smem, st>>>(d_op.p, d_dp.p, d_opmat.p, d_oprows.p, d_abc.p, bz_other.p, bz_j.p, bz_nbr.p, Z,
                                    k, Y, blk_t.p, k, Tout);
  LAUNCH_CHECK();
  k_coarse_gather_block<<<dim3((k + 255) / 256, Nc), 256, 0, st>>>(d_optr.p, d_oidx.p, blk_t.p, k, Nc, k, T, k);
  gemm(st, false, false, k, Nc, Nc, 1.0, T, k, d_Kinv.p, Nc, 0.0, blk_U.p, k);
  k_bz_edges<<<dim3((k + kBzCols - 1) / kBzCols, bz_nedges), kBzCols, 0, st>>>(
      bz_edges.p, bz_erow.p, bz_eb1.p, bz_eb2.p, d_op.p, d_dp.p, d_abc.p, d_cmap.p, bz_nbr.p, Y, blk_U.p, k, Q);
  LAUNCH_CHECK();
  return true;
}

void Ctx::project_rm(double* v, int ncols) {
  if (su.method != FETIGPU_TFETI) return;
  const int nc = 3 * su.Ns;
  double* g = grow(ws_g, (size_t)nc * ncols);
  double* h = grow(ws_h, (size_t)nc * ncols);
  double* corr = grow(ws_corr, (size_t)su.m * ncols);
  CK(cudaMemsetAsync(corr, 0, (size_t)su.m * ncols * 8, st));
  k_proj_gather<<<dim3(su.Ns, ncols), kThreads, 0, st>>>(d_pj.p, d_pcrows.p, d_pjcoef.p, d_RT.p, d_rt_off.p, v, 1,
                                                        g, nc, -1.0, ncols);
  small_gemm(g, h, ncols);
  k_proj_scatter<<<dim3(su.Ns, ncols), kThreads, 0, st>>>(d_pj.p, d_pcrows.p, d_pjcoef.p, d_RT.p, d_rt_off.p,
                                                         h, nc, corr, 1, ncols);
  k_add<<<grid_for((long long)su.m * ncols), kThreads, 0, st>>>(su.m * ncols, corr, v, 0, 0);
  LAUNCH_CHECK();
}

void Ctx::proj_corr(const double* v, int ldv, double* corr, int ldc, int ncols, double gsign) {
  if (ncols == 1 && su.m > 0) {
    proj_single(v, corr, 0, gsign);
    return;
  }
  const int nc = 3 * su.Ns;
  double* gp = d_g.p;
  double* hp = d_h.p;
  if (ncols > 1) {
    gp = grow(ws_g, (size_t)nc * ncols);
    hp = grow(ws_h, (size_t)nc * ncols);
  }
  k_proj_gather<<<dim3(su.Ns, ncols), kThreads, 0, st>>>(d_pj.p, d_pcrows.p, d_pjcoef.p, d_RT.p,
                                                        d_rt_off.p, v, ldv, gp, nc, gsign);
  small_gemm(gp, hp, ncols);
  if (ldc == su.m)
    CK(cudaMemsetAsync(corr, 0, (size_t)su.m * ncols * 8, st));
  else
    for (int c = 0; c < ncols; ++c) CK(cudaMemsetAsync(corr + (size_t)c * ldc, 0, su.m * 8, st));
  k_proj_scatter<<<dim3(su.Ns, ncols), kThreads, 0, st>>>(d_pj.p, d_pcrows.p, d_pjcoef.p, d_RT.p,
                                                         d_rt_off.p, hp, nc, corr, ldc);
  LAUNCH_CHECK();
}

void Ctx::rhs() {
  const int m = su.m;
  // x_s = S_kk^{-1} f_k (T-FETI) or S_rr^{-1} (f_r - S_rD g) (FETI-DP)
  launch_bnd_rhs(nullptr, nullptr);
  k_chol_solve<<<su.Ns, kThreads, max_ne * 8, st>>>(d_opfac.p, d_fac_off.p, d_slot_of.p, d_fac_ne.p, d_xb.p,
                                                     d_xoff.p);
  LAUNCH_CHECK();
  CK(cudaMemsetAsync(d_v1.p, 0, m * 8, st));
  launch_rhs_scatter(d_v1.p);  // B K^+ f
  if (su.method == FETIGPU_TFETI) {
    DBuf<double> gap;
    gap.upload(su.gap, st);
    k_sub<<<grid_for(m), kThreads, 0, st>>>(m, d_v1.p, gap.p, d_d.p);
    // lambda0 = G^T (G G^T)^{-1} e = -B R H e
    small_gemm(d_e.p, d_h.p, 1);
    CK(cudaMemsetAsync(d_v2.p, 0, m * 8, st));
    k_proj_scatter<<<su.Ns, kThreads, 0, st>>>(d_pj.p, d_pcrows.p, d_pjcoef.p, d_RT.p, d_rt_off.p, d_h.p,
                                               3 * su.Ns, d_v2.p, m);
    CK(cudaMemsetAsync(d_lam0.p, 0, m * 8, st));
    k_axpy<<<grid_for(m), kThreads, 0, st>>>(m, -1.0, d_v2.p, d_lam0.p);
    CK(cudaStreamSynchronize(st));
    gap.release();
  } else {
    // fbar_c = sum B_c^T (f_c - S_cD g - S_cr x); d = d_r - F_rc Kbar^{-1} fbar_c
    launch_dp_fbar();
    k_coarse_gather<<<grid_for(su.Nc), kThreads, 0, st>>>(d_optr.p, d_oidx.p, d_fbar_loc.p, su.Nc, d_fbar.p,
                                                         1.0, nullptr);
    k_dense_gemv<<<grid_for((long long)su.Nc * 32), kThreads, 0, st>>>(d_Kinv.p, su.Nc, d_fbar.p, d_h.p);
    CK(cudaMemsetAsync(d_v2.p, 0, m * 8, st));
    k_dp_phase2<<<su.Ns, kThreads, 0, st>>>(d_op.p, d_dp.p, d_oprows.p, d_opcoef_apply.p, d_abc.p, d_cmap.p, d_h.p,
                                            nullptr, d_v2.p, 0.0);
    k_sub<<<grid_for(m), kThreads, 0, st>>>(m, d_v1.p, d_v2.p, d_d.p);
    CK(cudaMemsetAsync(d_lam0.p, 0, m * 8, st));
    LAUNCH_CHECK();
  }
  CK(cudaStreamSynchronize(st));
  have_rhs = true;
}

void Ctx::recover(const double* lambda_dev, double* u_dev) {
  const int m = su.m, Ns = su.Ns;
  if (!have_rhs) rhs();
  DBuf<double> ub, alpha, uc;
  ub.alloc((size_t)Ns * su.nb);
  if (su.method == FETIGPU_TFETI) {
    // rho = d - F lambda; alpha = (G G^T)^{-1} G rho (least squares, decomposition.hpp:143)
    apply_F(lambda_dev, d_v1.p, 1, m, m);
    k_sub<<<grid_for(m), kThreads, 0, st>>>(m, d_d.p, d_v1.p, d_v2.p);
    k_proj_gather<<<su.Ns, kThreads, 0, st>>>(d_pj.p, d_pcrows.p, d_pjcoef.p, d_RT.p, d_rt_off.p, d_v2.p, m,
                                              d_g.p, 3 * Ns, -1.0);
    alpha.alloc(3 * (size_t)Ns);
    small_gemm(d_g.p, alpha.p, 1);
    launch_bnd_rhs(lambda_dev, nullptr);
  } else {
    // u_c = Kbar^{-1} (fbar_c + F_rc^T lambda)
    k_dp_t<<<Ns, kThreads, 0, st>>>(d_op.p, d_dp.p, d_oprows.p, d_opcoef_apply.p, d_abc.p, lambda_dev, d_tbuf.p);
    k_coarse_gather<<<grid_for(su.Nc), kThreads, 0, st>>>(d_optr.p, d_oidx.p, d_tbuf.p, su.Nc, d_g.p, 1.0,
                                                         d_fbar.p);
    uc.alloc(std::max(1, su.Nc));
    k_dense_gemv<<<grid_for((long long)su.Nc * 32), kThreads, 0, st>>>(d_Kinv.p, su.Nc, d_g.p, uc.p);
    launch_bnd_rhs(lambda_dev, uc.p);
  }
  k_chol_solve<<<Ns, kThreads, max_ne * 8, st>>>(d_opfac.p, d_fac_off.p, d_slot_of.p, d_fac_ne.p, d_xb.p,
                                                  d_xoff.p);
  launch_bnd_u(uc.p, ub.p);
  CK(cudaMemsetAsync(u_dev, 0, (size_t)Ns * su.nloc * 8, st));
  launch_scatter_perim(ub.p, u_dev);
  if (!keep_factors) fail(FETIGPU_E_STATE, "recovery needs the ND factors");
  int shm = 0;
  for (auto& nd : su.nd.nodes) shm = std::max(shm, nd.nf);
  k_nd_backsub<<<Ns, kThreads, shm * 8, st>>>(d_nodes.p, d_topdown.p, (int)su.nd.topdown.size(), d_nd_dofs.p,
                                              d_ndfac.p, su.nd.factor_stride, d_design.p, u_dev, su.nloc);
  LAUNCH_CHECK();
  if (su.method == FETIGPU_TFETI) launch_add_rigid(u_dev, alpha.p);
  CK(cudaStreamSynchronize(st));
}

}  // namespace fg
