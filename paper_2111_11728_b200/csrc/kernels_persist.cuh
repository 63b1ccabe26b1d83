// kernels_persist.cuh -- K15: the whole PCG / FO iteration loop as ONE persistent kernel.
//
// The graph-captured loop of solve_pcg.cuh runs ~20 dependent kernels per
// iteration; on the small configs (C1-C3, C5: operators of 0.5-58 MB, largely
// L2-resident) an iteration is bounded by launch and drain latency, not by the
// work.  Here every CTA of a co-resident grid walks one phase sequence,
// phases separated by a grid-wide barrier (or, for a grid that is one
// thread-block cluster, the hardware cluster barrier), and the phases are
// re-cut so that an iteration needs 4-7 of them instead of ~20 launches:
//  * the GEMVs store v_s = F_s x_s per subdomain instead of scattering with
//    atomics; the dual-row result y_r = c1 v_{s1} + c2 v_{s2} is formed row by
//    row where it is consumed (every dual row has at most two owners, so this
//    is the value the zeroed-buffer atomic scatter produces: 0 + a + b);
//  * vector updates are formed on the fly inside the next gather (w = z + beta
//    w in the F gather, stored by the row phase that follows; r -= alpha P q
//    and lambda += alpha w in the preconditioner gather, stored by one
//    designated owner per row), double-buffered where another CTA still
//    reads the old value;
//  * the dot products run inside the row phases on the graph path's fixed
//    partition (dot_partial_rows), and every CTA evaluates their fixed-order
//    final sums itself (no reduction barrier);
//  * small dense coarse operators (T-FETI H with 3N_s <= 96, FETI-DP
//    Kbar^{-1} with N_c <= 128) are applied redundantly by the CTAs that need
//    them; the FETI-DP coarse vector is gathered by the last arriving owner.
// Every value is formed by the same expression, in the same order, as on the
// graph path (shared device functions of kernels_apply.cuh; explicit
// __dmul_rn / __dadd_rn where a product meets a sum that the atomic path kept
// apart), so the two paths are bit-identical (tools/persist_ab.py,
// tests/test_gpu_persist.py).
//
// Coherence: data a phase reads was written in an earlier phase; it is read
// through L2 (__ldcg) or by weak loads after a barrier whose acquire
// invalidates L1 (CCTL.IVALL in the SASS), never through the non-coherent
// read-only path (no LDG.CONSTANT on in-kernel data).
//
// Reference: pcg single / FO, residual_metric and
// NegativeInnerProduct.
#pragma once

#include "kernels_apply.cuh"

namespace fg {

// grid-wide barrier for a co-resident (cooperative) grid: one monotone
// arrival counter.  Thread 0 of each CTA arrives with a fire-and-forget
// release add after the CTA barrier (cumulative over the CTA's writes) and
// spins with acquire loads until all G arrivals of this generation are in,
// then releases its CTA (the CUTLASS generic-barrier pattern; no atomic round
// trip on the arrival, no reset).  The counter is zeroed before each launch.
#ifdef FG_PERSIST_PROF
// phase profile (tools): CTA 0 stamps %globaltimer after every barrier
__device__ unsigned long long g_pprof[64 * 1024];
__device__ unsigned int g_pprof_n;
__device__ __forceinline__ void pprof_mark() {
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_pprof_n < 64 * 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_pprof[g_pprof_n++] = t;
  }
}
#else
__device__ __forceinline__ void pprof_mark() {}
#endif

struct GridBarrier {
  unsigned int* count;
  unsigned int* gen;   // unused
  __device__ __forceinline__ void sync(unsigned int& epoch) const {
    __syncthreads();
    epoch += gridDim.x;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(count), "r"(1u) : "memory");
      unsigned int c;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(count) : "memory");
      } while ((int)(c - epoch) < 0);
    }
    __syncthreads();
    pprof_mark();
  }
};

// the grid is one thread-block cluster: the hardware cluster barrier
// (release / acquire at cluster scope orders the CTAs' global-memory traffic)
struct ClusterBarrier {
  unsigned int* count;   // unused (same layout as GridBarrier)
  unsigned int* gen;
  __device__ __forceinline__ void sync(unsigned int&) const {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
};

struct PersistArgs {
  int m, Ns, Nc, KRp;
  int nz_op, nz_pc, ndot, psi_S;
  int passes, xs_len, redU, redH;
  // operator (K4): T-FETI KR = 3, FETI-DP KR = 1; v_s stored per subdomain
  const OpSub* op;
  const double* opmat;
  const int* oprows;
  const double* opcoef;
  double* vop;
  const int* voff_op;
  const int4* op_ent;        // per dual row: (s1, a1, s2, a2), s < 0: none
  const double2* op_c;       // per dual row: the two map coefficients
  // FETI-DP coarse step
  const DpSub* dp;
  const double* abc;
  double* tbuf;
  const CoarseGather* cg;
  const int* cmap;
  const double* Kinv;
  double* gc;
  // preconditioner (K7)
  const OpSub* pc;
  const double* pcmat;
  const int* pcrows;
  const double* pccoef;
  double* vpc;
  const int* voff_pc;
  const int4* pc_ent;
  const double2* pc_c;
  const unsigned char* pc_wr;   // per pc map entry: stores the row's new r and lambda
  // T-FETI projector (K8)
  const OpSub* pj;
  const double* pjcoef;
  const double* RT;
  const int* rt_off;
  const double* H;
  const int2* pj_sr;
  const double2* pj_c;
  double* g;
  double* h;   // H g (T-FETI) / Kbar^{-1} g (FETI-DP)
  // iterates (w, r double-buffered with w2, r2 for single-direction PCG)
  double *lam, *r, *z, *w, *q, *w2, *r2;
  Scal* sc;
  double* partial;
  // FO store
  double *Wst, *Qst, *psi, *psi_part;
  int* cnt;
  // loop control
  IterCtl* ctl;
  double* trace;
};

// y_r = c1 v_{s1}[a1] + c2 v_{s2}[a2]: the atomic scatter's 0 + a + b
__device__ __forceinline__ double row_combine(int i, const int4* __restrict__ ent, const double2* __restrict__ cc,
                                              const double* v, const int* __restrict__ voff) {
  const int4 e = ent[i];
  const double2 c = cc[i];
  double y = 0.0;
  if (e.x >= 0) y = __dadd_rn(y, __dmul_rn(c.x, __ldcg(v + voff[e.x] + e.y)));
  if (e.z >= 0) y = __dadd_rn(y, __dmul_rn(c.y, __ldcg(v + voff[e.z] + e.w)));
  return y;
}
// FETI-DP phase 2 of row i: sum over its owners of c (v_s[a] + A''_s[a,:] u_s),
// each owner's chain as in dp_phase2_cta (u in shared memory or L2)
template <bool SH>
__device__ __forceinline__ double dp_row(int i, const int4* __restrict__ ent, const double2* __restrict__ cc,
                                         const double* vbuf, const DpSub* __restrict__ dps,
                                         const double* __restrict__ abc, const int* __restrict__ cmap,
                                         const double* u) {
  const int4 e = ent[i];
  const double2 c = cc[i];
  double y = 0.0;
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const int s = o ? e.z : e.x, a = o ? e.w : e.y;
    if (s < 0) continue;
    const DpSub p = dps[s];
    double uc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double* up = u + cmap[p.cmap_off + (k < p.nc ? k : 0)];
      uc[k] = k < p.nc ? (SH ? *up : __ldcg(up)) : 0.0;
    }
    const double* Ab = abc + p.abc_off;
    double v = 1.0 * __ldcg(vbuf + p.v_off + a);
    if ((p.nc & 1) == 0 && (p.abc_off & 1) == 0) {
      const double2* A2 = reinterpret_cast<const double2*>(Ab + (size_t)a * p.nc);
      for (int k = 0; k < (p.nc >> 1); ++k) {
        const double2 ak = __ldcs(A2 + k);
        v = fma(ak.x, uc[2 * k], v);
        v = fma(ak.y, uc[2 * k + 1], v);
      }
    } else {
      for (int k = 0; k < p.nc; ++k) v = fma(Ab[(size_t)a * p.nc + k], uc[k], v);
    }
    y = __dadd_rn(y, __dmul_rn(o ? c.y : c.x, v));
  }
  return y;
}

#ifndef FG_PERSIST_OCC
#define FG_PERSIST_OCC 1
#endif
constexpr int kPersistOcc = FG_PERSIST_OCC;   // CTAs per SM the register budget allows
constexpr int kRedH = 96, kRedU = 128;          // redundant coarse applies up to these sizes

template <class Bar, bool TF, bool FO>
__global__ void __launch_bounds__(kThreads, kPersistOcc) k_pcg_persist(const PersistArgs a, const Bar bar) {
  extern __shared__ double shm[];
  double* xs = shm;               // gathered local vector (xs_len)
  double* sv = shm + a.xs_len;    // redundant H g / Kbar^{-1} g
  __shared__ double s_sum[4];
  const int G = gridDim.x, b0 = blockIdx.x;
  const int m = a.m, Ns = a.Ns;
  const int gtid = b0 * blockDim.x + threadIdx.x, gstride = G * blockDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp_g = gtid >> 5, nwarp_g = gstride >> 5;
  const bool lead = b0 == 0 && threadIdx.x == 0;
  const int nc3 = 3 * Ns;
  // scalar state (identical in every CTA; CTA 0 mirrors it to device memory)
  double rz = __ldcg(&a.sc->rz), rz_old = __ldcg(&a.sc->rz_old);
  double breakdown = __ldcg(&a.sc->breakdown);
  int it = __ldcg(&a.ctl->it);
  int cnt = FO ? __ldcg(a.cnt) : 0;
  const int max_it = a.ctl->max_it, trace_cap = a.ctl->trace_cap;
  const double target = a.ctl->target;
  unsigned int epoch = 0;   // GridBarrier arrivals expected so far
  double *wc = a.w, *wn = a.w2, *rc = a.r, *rn = a.r2;

  // fixed-order final sums of the last dot phase, in every CTA
  auto dot_sums = [&](int npairs) {
    __syncthreads();
    if (warp < npairs) {
      const double v = dot_final_warp(a.partial, warp, a.ndot);
      if (lane == 0) s_sum[warp] = v;
    }
    __syncthreads();
  };
  // T-FETI: H g into shared memory (redundant) -- or it is in a.h
  auto h_local = [&]() -> const double* {
    if (!a.redH) return a.h;
    dense_gemv_warps(a.H, nc3, a.g, sv, warp, kThreads / 32);
    __syncthreads();
    return sv;
  };
  auto corr = [&](int r, const double* hp) {
    return a.redH ? proj_row_corr<true>(r, a.pj_sr, a.pj_c, a.RT, hp)
                  : proj_row_corr<false>(r, a.pj_sr, a.pj_c, a.RT, hp);
  };

  bool first = true;
  double beta = 0.0;
  for (;;) {
    if (!first) {
      // ---- end of the previous iteration: rz, rr, zz and k_iter_control
      dot_sums(3);
      rz = s_sum[0];
      const double rr = s_sum[1], zz = s_sum[2];
      if (lead) { a.sc->rz = rz; a.sc->rr = rr; a.sc->zz = zz; }
      if (FO) {
        ++cnt;
        if (lead) *a.cnt = cnt;
      }
      bool go = false;
      if (breakdown != 0.0) {
        if (lead) a.ctl->status = 2;   // FETIGPU_BREAKDOWN
      } else if (rz < -1e-14 * sqrt(rr) * sqrt(zz)) {
        if (lead) a.ctl->err = 14;     // FETIGPU_E_NEGATIVE_INNER_PRODUCT
      } else {
        const double eps = sqrt(fmax(rz, 0.0));
        ++it;
        if (lead) {
          a.ctl->it = it;
          a.ctl->eps = eps;
          if (it < trace_cap) a.trace[it] = eps;
        }
        if (eps <= target) {
          if (lead) a.ctl->status = 0;   // FETIGPU_CONVERGED
        } else if (it >= max_it) {
          if (lead) a.ctl->status = 1;   // FETIGPU_MAX_ITER
        } else {
          go = true;
        }
      }
      if (!go) break;
      if constexpr (FO) {
        // CGS passes against the cnt stored directions (column cnt - 1 was
        // stored with w <- z in the last row phase)
        const int c = cnt, S = a.psi_S;
        for (int p = 0; p < a.passes; ++p) {
          double* part = S == 1 ? a.psi : a.psi_part;
          if (S == 1) {   // two columns per round (same rows): the loads of both in flight
            int item = b0;
            for (; item + G < c; item += 2 * G) fo_psi_item2(item, item + G, a.Qst, m, wc, part, 1);
            if (item < c) fo_psi_item(item, a.Qst, m, wc, part, 1);
          } else {
            for (int item = b0; item < c * S; item += G) fo_psi_item(item, a.Qst, m, wc, part, S);
          }
          bar.sync(epoch);
          if (S > 1) {
            for (int jj = gtid; jj < c; jj += gstride) {   // k_fo_psi_sum
              double t = 0.0;
              for (int s = 0; s < S; ++s) t += __ldcg(a.psi_part + (size_t)jj * S + s);
              a.psi[jj] = t;
            }
            bar.sync(epoch);
          }
          for (int vb = b0; vb < (m + 31) / 32; vb += G) fo_sub_cta(vb, a.Wst, m, c, a.psi, wc);
          bar.sync(epoch);
        }
      } else {
        beta = rz / rz_old;   // k_cg_dir2, k_shift_rz
        rz_old = rz;
        if (lead) a.sc->rz_old = rz;
      }
    }
    // ---- A: x_s = B_s^T w (single: w = z + beta w formed here), v_s = F_s x_s;
    //         FETI-DP: t_s = A''^T x_s and the last-arriver coarse gather g
    const bool upd = !FO && !first;
    {
      const int nv = Ns * a.nz_op;
      for (int vb = b0; vb < nv; vb += G) {
        const int s = vb / a.nz_op, zi = vb - s * a.nz_op;
        const OpSub d = a.op[s];
        auto plain = [&](int r, int) { return __ldcg(wc + r); };
        auto fused = [&](int r, int) { return fma(beta, __ldcg(wc + r), __ldcg(a.z + r)); };
        if (upd) gather_xs<TF ? 3 : 1>(d, a.oprows, a.opcoef, xs, fused);
        else gather_xs<TF ? 3 : 1>(d, a.oprows, a.opcoef, xs, plain);
        __syncthreads();
        if (!TF && zi == 0) fused_dp_t(a.dp[s], a.abc, xs, d.ns, a.tbuf, a.cg);
        gemv_rows_cta<TF ? 3 : 1, true>(s, 0, zi, a.nz_op, xs, d, a.opmat, a.oprows, a.opcoef, nullptr, nullptr, 0,
                                        a.vop, a.voff_op, 0, 1);
        __syncthreads();
      }
    }
    bar.sync(epoch);
    if (!TF && !a.redU && a.Nc > 0) {   // u = Kbar^{-1} g over the grid
      dense_gemv_warps(a.Kinv, a.Nc, a.gc, a.h, warp_g, nwarp_g);
      bar.sync(epoch);
    }
    // ---- B: q rows (dot CTAs) with delta = w^T q, wr = w^T r;
    //         T-FETI: g = -R^T B^T q on q formed on the fly (subdomain CTAs)
    for (int item = b0; item < a.ndot + (TF ? Ns : 0); item += G) {
      if (item < a.ndot) {
        const double* u = a.h;
        if (!TF && a.redU) {
          dense_gemv_warps(a.Kinv, a.Nc, a.gc, sv, warp, kThreads / 32);
          __syncthreads();
          u = sv;
        }
        dot_partial_rows<2>(item, a.ndot, m, a.partial, [&](int i, double* x, double* y) {
          double qi;
          if constexpr (TF) qi = row_combine(i, a.op_ent, a.op_c, a.vop, a.voff_op);
          else qi = a.redU ? dp_row<true>(i, a.op_ent, a.op_c, a.vop, a.dp, a.abc, a.cmap, u)
                           : dp_row<false>(i, a.op_ent, a.op_c, a.vop, a.dp, a.abc, a.cmap, u);
          a.q[i] = qi;
          double wi = __ldcg(wc + i);
          if (upd) {   // k_cg_dir2 for this row (the F gather formed the same value)
            wi = fma(beta, wi, __ldcg(a.z + i));
            wn[i] = wi;
          }
          x[0] = wi; y[0] = qi;
          x[1] = wi; y[1] = __ldcg(rc + i);
        });
      } else if constexpr (TF) {
        proj_gather_fn(item - a.ndot, 0, a.pj, a.pcrows, a.pjcoef, a.RT, a.rt_off, a.g, nc3, -1.0,
                       [&](int r) { return row_combine(r, a.op_ent, a.op_c, a.vop, a.voff_op); });
      }
      __syncthreads();
    }
    if (upd) { double* t = wc; wc = wn; wn = t; }
    bar.sync(epoch);
    if (TF && !a.redH) {
      dense_gemv_warps(a.H, nc3, a.g, a.h, warp_g, nwarp_g);
      bar.sync(epoch);
    }
    // ---- C: k_pcg_update formed inside the preconditioner gather:
    //         r_new = r - alpha P q (stored by one owner with lambda += alpha w), v_s = S_s x_s
    dot_sums(2);
    const double delta = s_sum[0], wr = s_sum[1];
    {
      const double* hp = TF ? h_local() : nullptr;
      if (lead) { a.sc->delta = delta; a.sc->wr = wr; }
      const bool bd = !(delta > 0.0);   // breakdown: lambda, r untouched
      if (bd) {
        breakdown = 1.0;
        if (lead) a.sc->breakdown = 1.0;
      }
      const double alpha = bd ? 0.0 : (FO ? wr : rz) / delta;
      if (lead && !bd) a.sc->alpha = alpha;
      const int nv = Ns * a.nz_pc;
      for (int vb = b0; vb < nv; vb += G) {
        const int s = vb / a.nz_pc, zi = vb - s * a.nz_pc;
        const OpSub d = a.pc[s];
        auto upd_r = [&](int r, int e) {
          const double rold = __ldcg(rc + r);
          double rv = rold;
          if (!bd) {
            const double qi = __ldcg(a.q + r);
            double pq = qi;
            if constexpr (TF) pq = __dadd_rn(qi, corr(r, hp));
            rv = fma(-alpha, pq, rold);
          }
          if (zi == 0 && a.pc_wr[e]) {
            rn[r] = rv;
            if (!bd) a.lam[r] = fma(alpha, __ldcg(wc + r), __ldcg(a.lam + r));
          }
          return rv;
        };
        if (a.KRp == 1) {
          gather_xs<1>(d, a.pcrows, a.pccoef, xs, upd_r);
          __syncthreads();
          gemv_rows_cta<1, true>(s, 0, zi, a.nz_pc, xs, d, a.pcmat, a.pcrows, a.pccoef, nullptr, nullptr, 0, a.vpc,
                                 a.voff_pc, 0, 1);
        } else {
          gather_xs<3>(d, a.pcrows, a.pccoef, xs, upd_r);
          __syncthreads();
          gemv_rows_cta<3, true>(s, 0, zi, a.nz_pc, xs, d, a.pcmat, a.pcrows, a.pccoef, nullptr, nullptr, 0, a.vpc,
                                 a.voff_pc, 0, 1);
        }
        __syncthreads();
      }
      double* t = rc; rc = rn; rn = t;
    }
    bar.sync(epoch);
    // T-FETI: z = P z_pre -- g = -R^T B^T z_pre with z_pre formed on the fly
    if constexpr (TF) {
      for (int s = b0; s < Ns; s += G) {
        proj_gather_fn(s, 0, a.pj, a.pcrows, a.pjcoef, a.RT, a.rt_off, a.g, nc3, -1.0,
                       [&](int r) { return row_combine(r, a.pc_ent, a.pc_c, a.vpc, a.voff_pc); });
        __syncthreads();
      }
      bar.sync(epoch);
      if (!a.redH) {
        dense_gemv_warps(a.H, nc3, a.g, a.h, warp_g, nwarp_g);
        bar.sync(epoch);
      }
    }
    // ---- D: z rows (dot CTAs) with rz, rr, zz; FO: k_fo_store2 (column cnt, w <- z)
    {
      const double inv = FO ? 1.0 / sqrt(delta) : 0.0;
      for (int vb = b0; vb < a.ndot; vb += G) {
        const double* hp = TF ? h_local() : nullptr;
        dot_partial_rows<3>(vb, a.ndot, m, a.partial, [&](int i, double* x, double* y) {
          double zi = row_combine(i, a.pc_ent, a.pc_c, a.vpc, a.voff_pc);
          if constexpr (TF) zi = __dadd_rn(zi, corr(i, hp));
          a.z[i] = zi;
          const double ri = __ldcg(rc + i);
          x[0] = ri; y[0] = zi;
          x[1] = ri; y[1] = ri;
          x[2] = zi; y[2] = zi;
          if constexpr (FO) {
            a.Wst[(size_t)cnt * m + i] = __ldcg(wc + i) * inv;
            a.Qst[(size_t)cnt * m + i] = __ldcg(a.q + i) * inv;
            wc[i] = zi;
          }
        });
        __syncthreads();
      }
    }
    bar.sync(epoch);
    first = false;
  }
}

}  // namespace fg

namespace fg {

// ------------------------------------------------------------------------
// K15c: the cluster-resident loop -- T-FETI, single direction, N_s <= 16
// subdomains whose explicit operators fit in one thread-block cluster's
// shared memory (C1: 8 x ~160 KB).  CTA s of the cluster keeps F_s and S~_s in
// its shared memory for the whole solve and a replica of every dual vector
// (m doubles each); a subdomain's GEMV result v_s stays in its CTA and the
// others read it through distributed shared memory (DSMEM) when they form
// the dual rows.  Scalars (dots, projector coarse vectors H g) are evaluated
// redundantly and identically by every CTA, so an iteration needs two
// cluster barriers and no global-memory traffic.  Same expressions, same
// orders as the graph loop (bit-identical, tests/test_gpu_persist.py).
// ------------------------------------------------------------------------
struct ClusterArgs {
  int m, Ns, ndot, KRp;
  int fs_len, ps_len, xs_len, pad;   // shared-memory regions (uniform across the cluster)
  const OpSub* op;
  const double* opmat;
  const int* oprows;
  const double* opcoef;
  const OpSub* pc;
  const double* pcmat;
  const int* pcrows;
  const double* pccoef;
  const int4* op_ent;
  const double2* op_c;
  const int4* pc_ent;
  const double2* pc_c;
  const OpSub* pj;
  const double* pjcoef;
  const double* RT;
  const int* rt_off;
  const double* H;
  const int2* pj_sr;
  const double2* pj_c;
  double *lam, *r, *w;   // global iterates: start values in, lambda out
  Scal* sc;
  IterCtl* ctl;
  double* trace;
};

// shared-memory doubles of k_pcg_cluster (every region a multiple of two
// doubles, so the double2 loads of the GEMV rows stay 16-byte aligned)
__host__ __device__ constexpr int even_up(int n) { return (n + 1) & ~1; }
__host__ __device__ constexpr size_t cluster_smem_doubles(int m, int Ns, int ndot, int fs, int ps, int xs) {
  return (size_t)even_up(fs) + even_up(ps) + 5 * (size_t)even_up(m) + 3 * (size_t)even_up(xs) +
         3 * (size_t)even_up(3 * Ns) + (size_t)even_up(9 * Ns * Ns) + 4 * (size_t)ndot +
         15 * (size_t)even_up(xs);   // the CTA's own gather / projector maps (4 x 3 xs doubles, 2 x 3 xs ints)
}

// g_s = sign R_T^T (B_s^T v) by ONE warp, emulating proj_gather_fn's CTA
// reduction: the 8 virtual warps' lane-strided sums, warp_sum each, then the
// fixed-order sum over virtual warps
template <class VV>
__device__ __forceinline__ void proj_gather_warp(int s, const OpSub* __restrict__ psubs, const int* __restrict__ rows,
                                                 const double* __restrict__ coefs, const double* __restrict__ RT,
                                                 const int* __restrict__ rt_off, double* g, double sign, VV&& vval) {
  const OpSub d = psubs[s];
  const double* R = RT + rt_off[s];
  const int lane = threadIdx.x & 31;
  constexpr int VW = kThreads / 32;
  // the 8 virtual warps' chains are independent until the final ordered sum:
  // all of them in flight at once (unrolled), each with its own accumulators
  double a0[VW], a1[VW], a2[VW];
#pragma unroll
  for (int vw = 0; vw < VW; ++vw) {
    a0[vw] = 0; a1[vw] = 0; a2[vw] = 0;
  }
  for (int jb = 0; jb < d.ns; jb += kThreads) {
#pragma unroll
    for (int vw = 0; vw < VW; ++vw) {
      const int j = jb + vw * 32 + lane;
      if (j < d.ns) {
        double xj = 0.0;
        for (int k = 0; k < 3; ++k) {
          const int r = rows[d.map_off + j * 3 + k];
          if (r >= 0) xj += coefs[d.map_off + j * 3 + k] * vval(r);
        }
        a0[vw] += R[j * 3] * xj;
        a1[vw] += R[j * 3 + 1] * xj;
        a2[vw] += R[j * 3 + 2] * xj;
      }
    }
  }
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
  for (int vw = 0; vw < VW; ++vw) {
    t0 += warp_sum(a0[vw]);
    t1 += warp_sum(a1[vw]);
    t2 += warp_sum(a2[vw]);
  }
  if (lane < 3) g[3 * s + lane] = sign * (lane == 0 ? t0 : lane == 1 ? t1 : t2);
}

template <int KRP>
__global__ void __launch_bounds__(kThreads, 1) k_pcg_cluster(const ClusterArgs a) {
  namespace cgr = cooperative_groups;
  cgr::cluster_group cl = cgr::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const int m = a.m, Ns = a.Ns, nc3 = 3 * Ns, nd = a.ndot;
  const int s = (int)cl.block_rank();   // this CTA's subdomain
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mp = even_up(m), xp = even_up(a.xs_len), n3p = even_up(nc3);
  double* Fs = sm;
  double* Ps = Fs + even_up(a.fs_len);
  double* w = Ps + even_up(a.ps_len);
  double* r = w + mp;
  double* z = r + mp;
  double* q = z + mp;
  double* lam = q + mp;
  double* vop = lam + mp;             // v_s = F_s x_s (read by the other CTAs)
  double* vpc = vop + xp;             // S~_s x_s
  double* xs = vpc + xp;
  double* g = xs + xp;                // this CTA's g_s (slot 3 s .. 3 s + 2), read by the others
  double* gall = g + n3p;             // every subdomain's g, gathered over DSMEM
  double* h = gall + n3p;
  double* Hs = h + n3p;
  double* part = Hs + even_up(nc3 * nc3);
  // this CTA's maps, staged once: operator (rows, coefs), preconditioner
  // (rows, coefs), projector coefs and R_T rows -- every gather reads shared
  // memory only
  double* ocf = part + 4 * nd;
  double* pcf = ocf + 3 * xp;
  double* pjcf = pcf + 3 * xp;
  double* RTs = pjcf + 3 * xp;
  int* orow = reinterpret_cast<int*>(RTs + 3 * xp);
  int* prow = orow + 3 * xp;
  __shared__ double s_sum[4];
  __shared__ int zoff[16];
  __shared__ OpSub lpj[16];
  if (tid < 16) zoff[tid] = 0;
  OpSub dop = a.op[s], dpc = a.pc[s];
  const OpSub dpj = a.pj[s];
  for (int i = tid; i < dop.ns * 3; i += kThreads) {
    orow[i] = a.oprows[dop.map_off + i];
    ocf[i] = a.opcoef[dop.map_off + i];
  }
  for (int i = tid; i < dpc.ns * KRP; i += kThreads) {
    prow[i] = a.pcrows[dpc.map_off + i];
    pcf[i] = a.pccoef[dpc.map_off + i];
  }
  for (int i = tid; i < dpj.ns * 3; i += kThreads) {
    pjcf[i] = a.pjcoef[dpj.map_off + i];
    RTs[i] = a.RT[a.rt_off[s] + i];
  }
  if (tid == 0) {
    lpj[s] = dpj;
    lpj[s].map_off = 0;
  }
  for (int i = tid; i < dop.ns * dop.ld; i += kThreads) Fs[i] = a.opmat[dop.moff + i];
  for (int i = tid; i < dpc.ns * dpc.ld; i += kThreads) Ps[i] = a.pcmat[dpc.moff + i];
  for (int i = tid; i < nc3 * nc3; i += kThreads) Hs[i] = a.H[i];
  for (int i = tid; i < m; i += kThreads) {
    w[i] = a.w[i];
    r[i] = a.r[i];
    lam[i] = a.lam[i];
  }
  OpSub lop = dop, lpc = dpc;   // local views: matrices and maps in shared memory
  lop.moff = 0;
  lpc.moff = 0;
  lop.map_off = 0;
  lpc.map_off = 0;
  double rz = a.sc->rz, rz_old = a.sc->rz_old, breakdown = a.sc->breakdown;
  int it = a.ctl->it;
  const int max_it = a.ctl->max_it, trace_cap = a.ctl->trace_cap;
  const double target = a.ctl->target;
  const bool lead = s == 0 && tid == 0;
  // y_r = c1 v_{s1}[a1] + c2 v_{s2}[a2] with v in the owners' shared memory
  auto combine = [&](int i, const int4* __restrict__ ent, const double2* __restrict__ cc, double* vloc) {
    const int4 e = ent[i];
    const double2 c = cc[i];
    double y = 0.0;
    if (e.x >= 0) y = __dadd_rn(y, __dmul_rn(c.x, cl.map_shared_rank(vloc, e.x)[e.y]));
    if (e.z >= 0) y = __dadd_rn(y, __dmul_rn(c.y, cl.map_shared_rank(vloc, e.z)[e.w]));
    return y;
  };
  // P-correction: g_s = -R_s^T B_s^T v by this CTA (the projector kernel's
  // CTA reduction), every g_s over DSMEM, then h = H g in every CTA
  auto proj_h = [&](const double* v) {
    proj_gather_fn(s, 0, lpj, prow, pjcf, RTs, zoff, g, 0, -1.0, [&](int row) { return v[row]; });
    cl.sync();
    for (int t = tid; t < nc3; t += kThreads) gall[t] = cl.map_shared_rank(g, t / 3)[t];
    __syncthreads();
    dense_gemv_warps<true>(Hs, nc3, gall, h, warp, kThreads / 32);
    __syncthreads();
  };
  auto sums = [&](int np) {
    if (warp < np) {
      const double v = dot_final_warp<true>(part, warp, nd, nd);
      if (lane == 0) s_sum[warp] = v;
    }
    __syncthreads();
  };
  cl.sync();
  bool first = true;
  for (;;) {
    if (!first) {
      // ---- k_iter_control on this CTA's (identical) scalars; k_cg_dir2
      sums(3);
      rz = s_sum[0];
      const double rr = s_sum[1], zz = s_sum[2];
      if (lead) { a.sc->rz = rz; a.sc->rr = rr; a.sc->zz = zz; }
      bool go = false;
      if (breakdown != 0.0) {
        if (lead) a.ctl->status = 2;
      } else if (rz < -1e-14 * sqrt(rr) * sqrt(zz)) {
        if (lead) a.ctl->err = 14;
      } else {
        const double eps = sqrt(fmax(rz, 0.0));
        ++it;
        if (lead) {
          a.ctl->it = it;
          a.ctl->eps = eps;
          if (it < trace_cap) a.trace[it] = eps;
        }
        if (eps <= target) {
          if (lead) a.ctl->status = 0;
        } else if (it >= max_it) {
          if (lead) a.ctl->status = 1;
        } else {
          go = true;
        }
      }
      if (!go) break;
      const double beta = rz / rz_old;
      rz_old = rz;
      if (lead) a.sc->rz_old = rz;
      for (int i = tid; i < m; i += kThreads) w[i] = fma(beta, w[i], z[i]);
      __syncthreads();
    }
    // ---- v_s = F_s B_s^T w
    gather_xs<3>(lop, orow, ocf, xs, [&](int row, int) { return w[row]; });
    __syncthreads();
    gemv_rows_cta<3, true, true>(s, 0, 0, 1, xs, lop, Fs, orow, ocf, nullptr, nullptr, 0, vop, zoff, 0, 1);
    cl.sync();
    pprof_mark();
    // ---- q rows over DSMEM; delta, wr; P-correction of q
    for (int i = tid; i < m; i += kThreads) q[i] = combine(i, a.op_ent, a.op_c, vop);
    __syncthreads();
    for (int vb = 0; vb < nd; ++vb) {
      dot_partial_rows<2>(vb, nd, m, part, [&](int i, double* x, double* y) {
        x[0] = w[i]; y[0] = q[i];
        x[1] = w[i]; y[1] = r[i];
      }, nd);
      __syncthreads();
    }
    sums(2);
    const double delta = s_sum[0], wr = s_sum[1];
    (void)wr;
    pprof_mark();
    proj_h(q);
    pprof_mark();
    // ---- k_pcg_update (replicated), then v_s = S~_s B~_s^T r
    if (lead) a.sc->delta = delta;
    const bool bd = !(delta > 0.0);
    if (bd) {
      breakdown = 1.0;
      if (lead) a.sc->breakdown = 1.0;
    } else {
      const double alpha = rz / delta;
      if (lead) a.sc->alpha = alpha;
      for (int i = tid; i < m; i += kThreads) {
        lam[i] = fma(alpha, w[i], lam[i]);
        const double pq = __dadd_rn(q[i], proj_row_corr<true>(i, a.pj_sr, a.pj_c, a.RT, h));
        r[i] = fma(-alpha, pq, r[i]);
      }
    }
    __syncthreads();
    gather_xs<KRP>(lpc, prow, pcf, xs, [&](int row, int) { return r[row]; });
    __syncthreads();
    gemv_rows_cta<KRP, true, true>(s, 0, 0, 1, xs, lpc, Ps, prow, pcf, nullptr, nullptr, 0, vpc, zoff, 0, 1);
    cl.sync();
    pprof_mark();
    // ---- z = P (M r): rows over DSMEM, P-correction; rz, rr, zz
    for (int i = tid; i < m; i += kThreads) z[i] = combine(i, a.pc_ent, a.pc_c, vpc);
    __syncthreads();
    pprof_mark();
    proj_h(z);
    pprof_mark();
    for (int i = tid; i < m; i += kThreads) z[i] = __dadd_rn(z[i], proj_row_corr<true>(i, a.pj_sr, a.pj_c, a.RT, h));
    __syncthreads();
    for (int vb = 0; vb < nd; ++vb) {
      dot_partial_rows<3>(vb, nd, m, part, [&](int i, double* x, double* y) {
        x[0] = r[i]; y[0] = z[i];
        x[1] = r[i]; y[1] = r[i];
        x[2] = z[i]; y[2] = z[i];
      }, nd);
      __syncthreads();
    }
    pprof_mark();
    first = false;
  }
  if (s == 0)
    for (int i = tid; i < m; i += kThreads) a.lam[i] = lam[i];
  cl.sync();   // no CTA leaves while another may still read its shared memory
}

}  // namespace fg
