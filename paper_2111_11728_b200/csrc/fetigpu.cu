// fetigpu.cu -- the C-ABI of libfetigpu (include/fetigpu.h) and the single
// CUDA translation unit of the engine (unity build: every kernel has one
// definition, and each shared-memory opt-in sits in the TU that launches it).
//
// One context = one FETI problem resident on one GPU.  fetigpu_build runs the
// whole operator construction on the device (ND Schur tree -> per-slot dense
// local operators -> FETI-DP coarse inverse); afterwards every operator
// application, preconditioner, projection and the PCG/FO/RRS loop run on the
// context's stream without host work beyond scalar read-back.
#include <cstring>
#include <memory>
#include <numeric>
#include <unordered_map>

#include "ctx.cuh"
#include "ctx_build.cuh"
#include "ctx_ops.cuh"
#include "solve_pcg.cuh"
#include "solve_rrs.cuh"


// ------------------------------------------------------------------ C-ABI --
using namespace fg;
struct fetigpu_ctx {
  Ctx c;
};
static thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
  int rc = 0;
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    rc = e.code;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    rc = FETIGPU_E_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    rc = FETIGPU_E_INVALID_ARGUMENT;
  }
  // a failed call must not leave a pending (non-sticky) launch error behind
  // for the next, unrelated call (e.g. another context's cuBLAS launch)
  if (rc >= FETIGPU_E_CUDA) cudaGetLastError();
  return rc;
}
#define NEED_BUILT(ctx) \
  if (!(ctx) || !(ctx)->c.built) fail(FETIGPU_E_STATE, "context not built")

extern "C" {

const char* fetigpu_last_error(void) { return g_err.c_str(); }

int fetigpu_set_device(int device) {
  return guarded([&] { CK(cudaSetDevice(device)); });
}

int fetigpu_create(const fetigpu_problem* p, fetigpu_ctx** out) {
  *out = nullptr;
  auto ctx = std::make_unique<fetigpu_ctx>();
  int rc = guarded([&] {
    if (!p) fail(FETIGPU_E_INVALID_ARGUMENT, "null problem");
    ctx->c.su.load(*p);
  });
  if (rc == 0) *out = ctx.release();
  return rc;
}

int fetigpu_build(fetigpu_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(FETIGPU_E_INVALID_ARGUMENT, "null context");
    if (ctx->c.built) fail(FETIGPU_E_STATE, "context already built");
    if (!ctx->c.st) ctx->c.init_device();
    ctx->c.build();
  });
}

void fetigpu_destroy(fetigpu_ctx* ctx) { delete ctx; }

int fetigpu_stats_get(const fetigpu_ctx* ctx, fetigpu_stats* s) {
  return guarded([&] {
    const Ctx& c = ctx->c;
    int mx = 0;
    for (auto& S : c.su.subs) mx = std::max(mx, (int)S.T.size());
    s->m = c.su.m; s->n_sub = c.su.Ns; s->local_dofs = c.su.nloc; s->n_c = c.su.Nc;
    s->n_kept = c.su.n_kept; s->n_iface = c.su.n_iface; s->max_ns = mx; s->n_designs = c.su.n_designs;
    s->n_op_slots = (int)c.su.op_slots.size();
    s->host_pipeline = c.pipe_ready ? 1 : 0;
    s->solve_loop = c.solve_loop;
    s->n_pc_slots = (int)(c.su.precond == FETIGPU_DIRICHLET ? c.su.pc_slots.size() : c.su.pc_lumped_T.size());
    // algorithmic work per apply, pure index counts
    double sn2 = 0, snc = 0, sns = 0;
    const bool dp = c.su.method == FETIGPU_FETIDP;
    for (auto& S : c.su.subs) {
      const double ns = (double)S.Top.size();
      sn2 += ns * ns;
      sns += ns;
      if (dp) snc += ns * (double)S.c.size();
    }
    s->op_bytes = 8 * sn2 + (dp ? 16 * snc + 8.0 * c.su.Nc * c.su.Nc : 0) + 16.0 * c.su.m + 8 * sns;
    s->op_flops_per_col = 2 * sn2 + (dp ? 4 * snc + 2.0 * c.su.Nc * c.su.Nc : 0);
    s->main_kernel_bytes = c.use_sym ? c.sym_bytes : 8 * sn2;
    s->apply_kernel = c.use_sym ? (c.sym_tma ? 2 : 1) : 0;
    s->apply_ring = c.use_sym && c.sym_tma ? c.sym_ring : 0;
    double coarse = 0;
    if (dp) {
      const double nbc = (c.su.Nc + 31) / 32;
      coarse = c.use_csym ? nbc * (nbc + 1) / 2 * 1024 * 8 : 8.0 * c.su.Nc * c.su.Nc;
    }
    s->stream_bytes = s->main_kernel_bytes + (dp ? 16 * snc : 0) + coarse + 16.0 * c.su.m + 8 * sns;
    s->build_ms = c.build_ms; s->nd_ms = c.nd_ms; s->slot_ms = c.slot_ms; s->coarse_ms = c.coarse_ms;
    s->device_bytes = (double)g_device_bytes;
  });
}

int fetigpu_rows(const fetigpu_ctx* ctx, int* kind, int* sp, int* dp, int* sm, int* dm, double* gap,
                 int* mult, double* wp, double* wm) {
  return guarded([&] {
    const Setup& su = ctx->c.su;
    for (int i = 0; i < su.m; ++i) {
      const Row& r = su.rows[i];
      kind[i] = r.kind; sp[i] = r.sp; dp[i] = r.dp; sm[i] = r.sm; dm[i] = r.dm;
      gap[i] = r.gap; mult[i] = r.mult; wp[i] = su.wplus[i]; wm[i] = su.wminus[i];
    }
  });
}

int fetigpu_apply_F_device(fetigpu_ctx* ctx, const double* x, double* y, int ncols, int ld) {
  return guarded([&] {
    NEED_BUILT(ctx);
    if (ctx->c.su.m == 0) return;  // no dual unknowns
    ctx->c.apply_F(x, y, ncols, ld, ld);
  });
}

int fetigpu_apply_F(fetigpu_ctx* ctx, const double* x, double* y, int ncols, int ld) {
  return guarded([&] {
    NEED_BUILT(ctx);
    if (ctx->c.su.m == 0) return;  // no dual unknowns
    Ctx& c = ctx->c;
    if (ncols == 1) {
      c.apply_F_host(x, y);
      return;
    }
    const size_t bytes = (size_t)ld * ncols * 8;
    c.stage((size_t)ld * ncols);
    CK(cudaMemcpyAsync(c.stage_x.p, x, bytes, cudaMemcpyHostToDevice, c.st));
    c.apply_F(c.stage_x.p, c.stage_y.p, ncols, ld, ld);
    CK(cudaMemcpyAsync(y, c.stage_y.p, bytes, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
  });
}

int fetigpu_apply_precond_device(fetigpu_ctx* ctx, const double* r, double* z, double* Z) {
  return guarded([&] {
    NEED_BUILT(ctx);
    if (ctx->c.su.m == 0) return;  // no dual unknowns
    ctx->c.apply_precond(r, z, Z);
  });
}

int fetigpu_apply_precond(fetigpu_ctx* ctx, const double* r, double* z, double* Zcols) {
  return guarded([&] {
    NEED_BUILT(ctx);
    if (ctx->c.su.m == 0) return;  // no dual unknowns
    Ctx& c = ctx->c;
    const int m = c.su.m;
    DBuf<double> dr, dz, dZ;
    dr.alloc(m);
    dz.alloc(m);
    if (Zcols) dZ.alloc((size_t)m * c.su.Ns);
    CK(cudaMemcpyAsync(dr.p, r, m * 8, cudaMemcpyHostToDevice, c.st));
    c.apply_precond(dr.p, dz.p, Zcols ? dZ.p : nullptr);
    CK(cudaMemcpyAsync(z, dz.p, m * 8, cudaMemcpyDeviceToHost, c.st));
    if (Zcols) CK(cudaMemcpyAsync(Zcols, dZ.p, (size_t)m * c.su.Ns * 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
  });
}

int fetigpu_project_device(fetigpu_ctx* ctx, double* v, int ncols, int ld) {
  return guarded([&] {
    NEED_BUILT(ctx);
    if (ctx->c.su.m == 0) return;  // no dual unknowns
    ctx->c.project(v, ncols, ld);
  });
}

int fetigpu_project(fetigpu_ctx* ctx, double* v, int ncols, int ld) {
  return guarded([&] {
    NEED_BUILT(ctx);
    if (ctx->c.su.m == 0) return;  // no dual unknowns
    Ctx& c = ctx->c;
    DBuf<double> dv;
    dv.alloc((size_t)ld * ncols);
    CK(cudaMemcpyAsync(dv.p, v, (size_t)ld * ncols * 8, cudaMemcpyHostToDevice, c.st));
    c.project(dv.p, ncols, ld);
    CK(cudaMemcpyAsync(v, dv.p, (size_t)ld * ncols * 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
  });
}

int fetigpu_rhs(fetigpu_ctx* ctx, double* d, double* l0) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    c.rhs();
    CK(cudaMemcpyAsync(d, c.d_d.p, c.su.m * 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaMemcpyAsync(l0, c.d_lam0.p, c.su.m * 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
  });
}

int fetigpu_solve(fetigpu_ctx* ctx, const fetigpu_solve_opts* o, double* lambda, fetigpu_trace* tr) {
  return guarded([&] {
    NEED_BUILT(ctx);
    ctx->c.solve(*o, lambda, tr);
  });
}

int fetigpu_solve_warm(fetigpu_ctx* ctx, const fetigpu_solve_opts* o, const double* lambda0, double* lambda,
                       fetigpu_trace* tr) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    struct Reset {
      Ctx& c;
      ~Reset() { c.warm = false; }
    } reset{c};
    if (lambda0 && c.su.m > 0) {
      if (c.d_warm.n < (size_t)c.su.m) c.d_warm.alloc(c.su.m);
      CK(cudaMemcpyAsync(c.d_warm.p, lambda0, (size_t)c.su.m * 8, cudaMemcpyHostToDevice, c.st));
      c.warm = true;
    }
    c.solve(*o, lambda, tr);
  });
}

// New snapshot of the same problem (same partition, supports, loads, method;
// new densities / material): host setup again, device operators rebuilt in
// the existing storage (recycled through the context's block cache).
int fetigpu_rebuild(fetigpu_ctx* ctx, const fetigpu_problem* p) {
  return guarded([&] {
    NEED_BUILT(ctx);
    if (!p) fail(FETIGPU_E_INVALID_ARGUMENT, "null problem");
    Ctx& c = ctx->c;
    const Setup& old = c.su;
    if (p->sx != old.sx || p->sy != old.sy || p->n != old.n || p->n_designs != old.n_designs ||
        p->method != old.method)
      fail(FETIGPU_E_DIMENSION_MISMATCH, "rebuild: partition, module size, design count and method must match");
    Setup su;
    su.load(*p);
    if (su.m != old.m || su.Nc != old.Nc) fail(FETIGPU_E_DIMENSION_MISMATCH, "rebuild: constraint structure changed");
    CK(cudaStreamSynchronize(c.st));
    c.su = std::move(su);
    c.have_rhs = false;
    c.bz_state = 0;
    c.p_state = 0;   // K15 row maps are re-derived from the rebuilt operators
    c.built = false;
    struct Scope {
      BlockCache* prev;
      explicit Scope(BlockCache* b) : prev(g_build_cache) { g_build_cache = b; }
      ~Scope() { g_build_cache = prev; }
    } scope(&c.build_cache);
    c.build();
    ++c.rebuilds;
  });
}

int fetigpu_set_rrs_store(fetigpu_ctx* ctx, int mode) {
  return guarded([&] {
    if (!ctx) fail(FETIGPU_E_INVALID_ARGUMENT, "null context");
    if (mode < FETIGPU_RRS_STORE_AUTO || mode > FETIGPU_RRS_STORE_IMPLICIT)
      fail(FETIGPU_E_INVALID_ARGUMENT, "unknown RRS store mode");
    if (mode == FETIGPU_RRS_STORE_IMPLICIT && ctx->c.su.method != FETIGPU_FETIDP)
      fail(FETIGPU_E_CONFIG, "the implicit RRS store needs FETI-DP (T-FETI directions are projected, dense)");
    ctx->c.rrs_store = mode;
  });
}

int fetigpu_recover(fetigpu_ctx* ctx, const double* lambda, double* u) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    DBuf<double> dl, du;
    dl.alloc(c.su.m);
    du.alloc((size_t)c.su.Ns * c.su.nloc);
    CK(cudaMemcpyAsync(dl.p, lambda, c.su.m * 8, cudaMemcpyHostToDevice, c.st));
    c.recover(dl.p, du.p);
    CK(cudaMemcpyAsync(u, du.p, (size_t)c.su.Ns * c.su.nloc * 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
  });
}

int fetigpu_local_operator(fetigpu_ctx* ctx, int s, int* ns, int* dofs, double* F, int cap) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    if (s < 0 || s >= c.su.Ns) fail(FETIGPU_E_INVALID_ARGUMENT, "subdomain out of range");
    const SubPlan& S = c.su.subs[s];
    const int sl = S.op_slot, n = c.op_ns[sl], ld = c.op_ld[sl];
    *ns = n;
    if (n > cap) return;
    for (int a = 0; a < n; ++a) dofs[a] = c.su.perim_dof[S.Top[a]];
    std::vector<double> tmp((size_t)n * ld);
    CK(cudaMemcpyAsync(tmp.data(), c.d_opmat.p + c.op_moff[sl], tmp.size() * 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        const double sg = c.folded ? c.slot_sign[sl][a] * c.slot_sign[sl][b] : 1.0;
        F[(size_t)a * n + b] = sg * tmp[(size_t)a * ld + b];
      }
  });
}

int fetigpu_apply_F_block_device(fetigpu_ctx* ctx, const double* W, int ldw, double* Q, int ldq, int k) {
  return guarded([&] {
    NEED_BUILT(ctx);
    ctx->c.apply_F_block(W, ldw, Q, ldq, k);
  });
}

// ---- subdomain-sharded apply, device pointers on the ctx stream
int fetigpu_shard_set_range(fetigpu_ctx* ctx, int s0, int s1) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    if (s0 < 0 || s1 < s0 || s1 > c.su.Ns) fail(FETIGPU_E_INVALID_ARGUMENT, "bad subdomain range");
    c.shard_s0 = s0;
    c.shard_s1 = s1;
  });
}
int fetigpu_shard_info(const fetigpu_ctx* ctx, int* tot_c) {
  return guarded([&] { *tot_c = ctx->c.tot_c(); });
}
int fetigpu_shard_phase1_device(fetigpu_ctx* ctx, const double* x, double* y, double* tout, int precond) {
  return guarded([&] {
    NEED_BUILT(ctx);
    ctx->c.shard_phase1(x, y, tout, precond != 0);
  });
}
int fetigpu_shard_phase2_device(fetigpu_ctx* ctx, const double* tall, double* y) {
  return guarded([&] {
    NEED_BUILT(ctx);
    ctx->c.shard_phase2(tall, y);
  });
}

// invariant check of the device solver's stored directions (test hook)
int fetigpu_set_check(fetigpu_ctx* ctx, int on) {
  return guarded([&] {
    ctx->c.chk_on = on != 0;
    ctx->c.chk_err = -1.0;
    ctx->c.chk_n = 0;
  });
}
int fetigpu_check_result(const fetigpu_ctx* ctx, double* err, int* n) {
  return guarded([&] {
    *err = ctx->c.chk_err;
    *n = ctx->c.chk_n;
  });
}

// test hook: Q = F Z through K5z for a per-subdomain preconditioner block
// (row-major m x N_s host buffers); FETIGPU_E_CONFIG when not applicable
int fetigpu_apply_F_zblock(fetigpu_ctx* ctx, const double* Z, double* Q) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    const size_t n = (size_t)c.su.m * c.su.Ns;
    DBuf<double> dz, dq;
    dz.alloc(std::max<size_t>(n, 1)); dq.alloc(std::max<size_t>(n, 1));
    CK(cudaMemcpyAsync(dz.p, Z, n * 8, cudaMemcpyHostToDevice, c.st));
    if (!c.apply_F_block_z(dz.p, dq.p, c.su.Ns)) fail(FETIGPU_E_CONFIG, "K5z: not a FETI-DP block with that structure");
    CK(cudaMemcpyAsync(Q, dq.p, n * 8, cudaMemcpyDeviceToHost, c.st));
    CK(cudaStreamSynchronize(c.st));
  });
}

int fetigpu_time_apply_block(fetigpu_ctx* ctx, const double* W, double* Q, int k, int reps, double* ms) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c.st));
    for (int r = 0; r < reps; ++r) c.apply_F_block(W, k, Q, k, k);
    CK(cudaEventRecord(b, c.st));
    CK(cudaEventSynchronize(b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, a, b));
    ms[0] = t / reps;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int fetigpu_fp64_peak(double* tflops_dmma, double* tflops_dfma) {
  return guarded([&] {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* out = nullptr;
    CK(cudaMalloc(&out, 8));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int iters = 20000, blocks = sms * 4;
    for (int pass = 0; pass < 2; ++pass) {  // first pass warms up
      CK(cudaEventRecord(a));
      k_peak_dmma<<<blocks, 256>>>(out, iters);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float t = 0;
      CK(cudaEventElapsedTime(&t, a, b));
      *tflops_dmma = (double)blocks * 8 * iters * 8 * 512 / (t * 1e-3) / 1e12;
      CK(cudaEventRecord(a));
      k_peak_dfma<<<blocks, 256>>>(out, iters);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&t, a, b));
      *tflops_dfma = (double)blocks * 256 * iters * 8 * 2 / (t * 1e-3) / 1e12;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
  });
}

int fetigpu_hbm_read_peak(size_t bytes, int reps, double* gbs) {
  return guarded([&] {
    if (!gbs || reps < 1) fail(FETIGPU_E_INVALID_ARGUMENT, "hbm_read_peak: bad arguments");
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    bytes = std::max<size_t>(bytes, (size_t)1 << 28) & ~(size_t)4095;
    DBuf<double> buf, out;
    buf.alloc(bytes / 8);
    out.alloc(8);
    CK(cudaMemset(buf.p, 0, bytes));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    double best = 0.0;
    for (int grid : {4 * sms, 8 * sms, 16 * sms}) {
      for (int r = 0; r < 3; ++r) k_peak_read<8><<<grid, 256>>>((const double2*)buf.p, bytes / 16, out.p);
      CK(cudaEventRecord(a));
      for (int r = 0; r < reps; ++r) k_peak_read<8><<<grid, 256>>>((const double2*)buf.p, bytes / 16, out.p);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      LAUNCH_CHECK();
      float t = 0;
      CK(cudaEventElapsedTime(&t, a, b));
      best = std::max(best, (double)bytes * reps / (t * 1e-3) / 1e9);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *gbs = best;
  });
}

// ---- dense algebra hooks (dla.cuh): host-buffer GEMM / triangular inverse
// for the parity tests, device-resident GEMM timing for the bench
int fetigpu_dla_gemm(int ta, int tb, int M, int N, int K, double alpha, const double* A, long long lda,
                     const double* B, long long ldb, double beta, double* C, long long ldc, int flags) {
  return guarded([&] {
    if (M < 0 || N < 0 || K < 0) fail(FETIGPU_E_INVALID_ARGUMENT, "bad dimensions");
    if (!M || !N) return;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> st_guard(st, cudaStreamDestroy);
    const size_t na = (size_t)lda * (ta ? M : K), nb = (size_t)ldb * (tb ? K : N), nc = (size_t)ldc * N;
    DBuf<double> dA, dB, dC, ws;
    dA.alloc(std::max<size_t>(na, 1)); dB.alloc(std::max<size_t>(nb, 1)); dC.alloc(nc);
    if (na) CK(cudaMemcpyAsync(dA.p, A, na * 8, cudaMemcpyHostToDevice, st));
    if (nb) CK(cudaMemcpyAsync(dB.p, B, nb * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dC.p, C, nc * 8, cudaMemcpyHostToDevice, st));
    if (flags & 256) {   // split-K path of the same product
      ws.alloc(std::max<size_t>(1, gemm_splitk_ws(M, N, K)));
      gemm_splitk(st, ta, tb, M, N, K, alpha, dA.p, lda, dB.p, ldb, beta, dC.p, ldc, ws.p, flags & 255);
    } else {
      gemm(st, ta, tb, M, N, K, alpha, dA.p, lda, dB.p, ldb, beta, dC.p, ldc, flags);
    }
    CK(cudaMemcpyAsync(C, dC.p, nc * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fetigpu_dla_tri_inv(const double* L, int n, long long ldl, double* X) {
  return guarded([&] {
    if (n <= 0) return;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> st_guard(st, cudaStreamDestroy);
    DBuf<double> dL, dX, ws;
    dL.alloc((size_t)ldl * n); dX.alloc((size_t)n * n); ws.alloc(tri_inv_workspace(n));
    CK(cudaMemcpyAsync(dL.p, L, (size_t)ldl * n * 8, cudaMemcpyHostToDevice, st));
    tri_inv_lower(st, dL.p, ldl, n, dX.p, n, ws.p);
    CK(cudaMemcpyAsync(X, dX.p, (size_t)n * n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fetigpu_dla_time_gemm(int ta, int tb, int M, int N, int K, int reps, double* ms) {
  return guarded([&] {
    if (M <= 0 || N <= 0 || K <= 0 || reps <= 0) fail(FETIGPU_E_INVALID_ARGUMENT, "bad dimensions");
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> st_guard(st, cudaStreamDestroy);
    const long long lda = ta ? K : M, ldb = tb ? N : K;
    DBuf<double> dA, dB, dC;
    dA.alloc((size_t)M * K); dB.alloc((size_t)K * N); dC.alloc((size_t)M * N);
    k_fill_random<<<grid_for((long long)M * K), kThreads, 0, st>>>(dA.p, (size_t)M * K, 1);
    k_fill_random<<<grid_for((long long)K * N), kThreads, 0, st>>>(dB.p, (size_t)K * N, 2);
    gemm(st, ta, tb, M, N, K, 1.0, dA.p, lda, dB.p, ldb, 0.0, dC.p, M);   // warm-up
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, st));
    for (int r = 0; r < reps; ++r) gemm(st, ta, tb, M, N, K, 1.0, dA.p, lda, dB.p, ldb, 0.0, dC.p, M);
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, a, b));
    *ms = t / reps;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int fetigpu_pivoted_cholesky(const double* a, int n, double tol, int* perm, double* lower, int* rank) {
  return guarded([&] {
    if (n < 0 || (n > 0 && (!a || !perm || !lower || !rank))) fail(FETIGPU_E_INVALID_ARGUMENT, "bad arguments");
    *rank = 0;
    if (n == 0) return;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> st_guard(st, cudaStreamDestroy);
    DBuf<double> A;
    DBuf<int> p, r, status, ctl;
    DBuf<double> gx;
    A.alloc((size_t)n * n);
    p.alloc(n); r.alloc(1); status.alloc(1); ctl.alloc(4); gx.alloc(2 * (size_t)n + 64);
    status.zero(st);
    CK(cudaMemcpyAsync(A.p, a, (size_t)n * n * 8, cudaMemcpyHostToDevice, st));
    k_mirror_lower<<<grid_for((long long)n * n), kThreads, 0, st>>>(A.p, n);
    DBuf<double> lc;
    lc.alloc((size_t)n * n);
    launch_pivchol(A.p, n, tol, p.p, r.p, status.p, ctl.p, gx.p, st, lc.p);
    LAUNCH_CHECK();
    int hstat = 0;
    std::vector<double> full((size_t)n * n);
    CK(cudaMemcpyAsync(full.data(), A.p, (size_t)n * n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(perm, p.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rank, r.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hstat, status.p, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hstat) fail(FETIGPU_E_INDEFINITE_INPUT, "pivoted Cholesky: negative pivot");
    // L: column k (k < rank) holds rows i >= k; everything else zero
    for (int k = 0; k < n; ++k)
      for (int i = 0; i < n; ++i)
        lower[(size_t)k * n + i] = (k < *rank && i >= k) ? full[(size_t)k * n + i] : 0.0;
  });
}

int fetigpu_pivoted_compress(const int* perm, const double* lower, int n, int rank, const double* w, int rows,
                             double* out) {
  return guarded([&] {
    if (n < 0 || rank < 0 || rank > n || rows < 0 || (rank > 0 && rows > 0 && (!perm || !lower || !w || !out)))
      fail(FETIGPU_E_INVALID_ARGUMENT, "bad arguments");
    if (rank == 0 || rows == 0) return;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> st_guard(st, cudaStreamDestroy);
    DBuf<double> L, Linv, W, Wsel, O, Tw;
    DBuf<int> p;
    L.alloc((size_t)n * n); Linv.alloc((size_t)rank * rank);
    W.alloc((size_t)rows * n); Wsel.alloc((size_t)rows * rank); O.alloc((size_t)rows * rank);
    p.alloc(n);
    CK(cudaMemcpyAsync(L.p, lower, (size_t)n * n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(W.p, w, (size_t)rows * n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p.p, perm, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    // L~^{-1} (dla.cuh tri_inv_lower), W_sel = W N^T[:, :rank],
    // out = W_sel L~^{-T}: the solver's compression (Alg. 1 lines 10-11)
    Tw.alloc(tri_inv_workspace(rank));
    tri_inv_lower(st, L.p, n, rank, Linv.p, rank, Tw.p);
    k_gather_cols<<<dim3(grid_for(rows), rank), kThreads, 0, st>>>(W.p, rows, p.p, rank, Wsel.p);
    gemm(st, false, true, rows, rank, rank, 1.0, Wsel.p, rows, Linv.p, rank, 0.0, O.p, rows, kGemmKEndByCol);
    LAUNCH_CHECK();
    CK(cudaMemcpyAsync(out, O.p, (size_t)rows * rank * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int fetigpu_selftest_dmma(const double* A, const double* B, double* C) {
  return guarded([&] {
    double *dA, *dB, *dC;
    CK(cudaMalloc(&dA, 32 * 8));
    CK(cudaMalloc(&dB, 32 * 8));
    CK(cudaMalloc(&dC, 64 * 8));
    CK(cudaMemcpy(dA, A, 32 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B, 32 * 8, cudaMemcpyHostToDevice));
    k_dmma_selftest<<<1, 32>>>(dA, dB, dC);
    CK(cudaMemcpy(C, dC, 64 * 8, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
  });
}

int fetigpu_device_alloc(fetigpu_ctx*, size_t bytes, void** ptr) {
  return guarded([&] { CK(cudaMalloc(ptr, bytes)); });
}
int fetigpu_device_free(fetigpu_ctx*, void* ptr) {
  return guarded([&] { CK(cudaFree(ptr)); });
}
int fetigpu_host_alloc(size_t bytes, void** ptr) {
  return guarded([&] { CK(cudaMallocHost(ptr, bytes)); });
}
int fetigpu_host_free(void* ptr) {
  return guarded([&] { CK(cudaFreeHost(ptr)); });
}
int fetigpu_memcpy(fetigpu_ctx* ctx, void* dst, const void* src, size_t bytes, int kind) {
  return guarded([&] {
    CK(cudaMemcpyAsync(dst, src, bytes, (cudaMemcpyKind)kind, ctx->c.st));
  });
}
int fetigpu_fill_random(fetigpu_ctx* ctx, double* p, size_t count, unsigned long long seed) {
  return guarded([&] {
    k_fill_random<<<grid_for((long long)count), kThreads, 0, ctx->c.st>>>(p, count, seed);
    LAUNCH_CHECK();
  });
}
int fetigpu_synchronize(fetigpu_ctx* ctx) {
  return guarded([&] { CK(cudaStreamSynchronize(ctx->c.st)); });
}

int fetigpu_device_memory(fetigpu_ctx* ctx, size_t* free_bytes, size_t* total_bytes, size_t* cached_bytes) {
  return guarded([&] {
    if (!free_bytes || !total_bytes || !cached_bytes) fail(FETIGPU_E_INVALID_ARGUMENT, "null output");
    CK(cudaMemGetInfo(free_bytes, total_bytes));
    *cached_bytes = ctx ? ctx->c.rrs_cache.cached_bytes() : 0;
  });
}

int fetigpu_time_ops(fetigpu_ctx* ctx, int reps, double* ms) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    const int m = std::max(1, c.su.m);
    DBuf<double> x, y;
    x.alloc(m);
    y.alloc(m);
    k_fill_random<<<grid_for(m), kThreads, 0, c.st>>>(x.p, (size_t)m, 11ull);
    LAUNCH_CHECK();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int op = 0; op < 3; ++op) {
      auto run = [&] {
        if (c.su.m == 0) return;
        if (op == 0) c.apply_F(x.p, y.p, 1, c.su.m, c.su.m);
        else if (op == 1) c.apply_precond(x.p, y.p, nullptr);
        else c.project(y.p, 1, c.su.m);
      };
      for (int w = 0; w < 3; ++w) run();
      CK(cudaEventRecord(a, c.st));
      for (int r = 0; r < reps; ++r) run();
      CK(cudaEventRecord(b, c.st));
      CK(cudaEventSynchronize(b));
      float t = 0;
      CK(cudaEventElapsedTime(&t, a, b));
      ms[op] = t / std::max(1, reps);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int fetigpu_time_apply(fetigpu_ctx* ctx, const double* x, double* y, int ncols, int reps, int flush_l2,
                       double* ms, int* launches) {
  return guarded([&] {
    NEED_BUILT(ctx);
    Ctx& c = ctx->c;
    DBuf<double> fl;
    const size_t fl_n = (size_t)(256u << 20) / 8;  // 256 MB > 126 MB L2
    if (flush_l2) fl.alloc(fl_n);
    std::vector<cudaEvent_t> ev(2 * reps + 2);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    // dominant kernel alone, same launch configuration as inside apply_F
    double tot = 0, tot_main = 0;
    for (int r = 0; r < reps; ++r) {
      if (flush_l2) k_flush<<<grid_for((long long)fl_n), kThreads, 0, c.st>>>(fl.p, fl_n, (double)r);
      CK(cudaEventRecord(ev[2 * r], c.st));
      c.apply_F(x, y, ncols, c.su.m, c.su.m);
      CK(cudaEventRecord(ev[2 * r + 1], c.st));
    }
    CK(cudaStreamSynchronize(c.st));
    for (int r = 0; r < reps; ++r) {
      float t = 0;
      CK(cudaEventElapsedTime(&t, ev[2 * r], ev[2 * r + 1]));
      tot += t;
    }
    for (int r = 0; r < reps; ++r) {
      if (flush_l2) k_flush<<<grid_for((long long)fl_n), kThreads, 0, c.st>>>(fl.p, fl_n, (double)r);
      CK(cudaEventRecord(ev[2 * r], c.st));
      for (int col = 0; col < ncols; ++col) {
        const double* xc = x + (size_t)col * c.su.m;
        double* yc = y + (size_t)col * c.su.m;
        if (c.use_sym) {
          Ctx::SymArgs sa;
          sa.x = xc; sa.n = c.su.Ns;
          if (c.su.method == FETIGPU_TFETI) { sa.kr = 3; sa.y = yc; }
          else sa.store_v = true;
          c.launch_sym(c.st, sa);
        } else if (c.su.method == FETIGPU_TFETI) {
          k_gather_gemv_scatter<3, false><<<dim3(c.su.Ns, 1, c.rsplit), kThreads, c.max_ld * 8, c.st>>>(
              c.d_op.p, c.d_opmat.p, c.d_oprows.p, c.d_opcoef_apply.p, xc, yc, nullptr, 0, nullptr, nullptr,
              c.su.m, c.su.m);
        } else {
          k_gather_gemv_scatter<1, true><<<dim3(c.su.Ns, 1, c.rsplit), kThreads, c.max_ld * 8, c.st>>>(
              c.d_op.p, c.d_opmat.p, c.d_oprows.p, c.d_opcoef_apply.p, xc, nullptr, nullptr, 0, c.d_vbuf.p,
              c.d_voff.p, c.su.m, 0, 1, c.d_dp.p, c.d_abc.p, c.d_tbuf.p);
        }
      }
      CK(cudaEventRecord(ev[2 * r + 1], c.st));
    }
    CK(cudaStreamSynchronize(c.st));
    for (int r = 0; r < reps; ++r) {
      float t = 0;
      CK(cudaEventElapsedTime(&t, ev[2 * r], ev[2 * r + 1]));
      tot_main += t;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    ms[0] = tot / reps;
    ms[1] = tot_main / reps;
    ms[2] = ms[1] / ms[0];
    if (launches)
      *launches = (c.su.method == FETIGPU_TFETI ? 1 : 2 + (c.use_csym ? 2 : 1) + (c.use_sym && c.su.Nc ? 0 : 1)) * ncols;
  });
}

}  // extern "C"

#ifdef FG_PERSIST_PROF
// tools/persist_prof.py: the K15 phase stamps of the last persistent solve
extern "C" int fetigpu_pprof(unsigned long long* out, int cap) {
  unsigned int n = 0;
  if (cudaMemcpyFromSymbol(&n, fg::g_pprof_n, sizeof(n)) != cudaSuccess) return -1;
  n = std::min<unsigned int>(n, (unsigned int)cap);
  if (n && cudaMemcpyFromSymbol(out, fg::g_pprof, n * sizeof(unsigned long long)) != cudaSuccess) return -1;
  const unsigned int z = 0;
  cudaMemcpyToSymbol(fg::g_pprof_n, &z, sizeof(z));
  return (int)n;
}
#endif
