// solve_rrs.cuh -- Rank-Revealing Simultaneous FETI (Alg. 1): pivoted Cholesky launchers
// and the block iteration.
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include "ctx.cuh"

namespace fg {

// ------------------------------------------------ implicit direction store --
// FETI-DP RRS with the stored directions kept as coefficients over the
// preconditioner blocks Z_l (solve_rrs_implicit).  Z_l column s lives on the
// dual rows of subdomain s only (the preconditioner's map), so it is stored
// packed: ZV[l * nz + t] for the map position t of (s, a).

// ZV[l * nz + t] = Z (row-major m x k) at the map positions t of each
// subdomain's column (packed block l, column-major: appending a block never
// moves the earlier ones)
__global__ void k_rrs_zpack(const OpSub* __restrict__ pc, const int* __restrict__ rows,
                            const double* __restrict__ Z, int k, double* __restrict__ ZV, long long nz, int l) {
  const int s = blockIdx.x;
  const OpSub d = pc[s];
  double* zl = ZV + (size_t)l * nz;
  for (int a = threadIdx.x; a < d.ns; a += blockDim.x) {
    const int r = rows[d.map_off + a];
    zl[d.map_off + a] = r >= 0 ? Z[(size_t)r * k + s] : 0.0;
  }
}

// inverse of k_rrs_zpack (test hook of the invariant check): Z(r_a, s) = ZV(t)
__global__ void k_rrs_zunpack(const OpSub* __restrict__ pc, const int* __restrict__ rows,
                              const double* __restrict__ zl, int k, double* __restrict__ Z) {
  const int s = blockIdx.x;
  const OpSub d = pc[s];
  for (int a = threadIdx.x; a < d.ns; a += blockDim.x) {
    const int r = rows[d.map_off + a];
    if (r >= 0) Z[(size_t)r * k + s] = zl[d.map_off + a];
  }
}

constexpr int kZL = 16;          // Z blocks per pass of k_rrs_zgather
constexpr int kZC = 32;          // Z blocks per register chunk of k_rrs_zscatter
constexpr int kZRows = 32;       // map rows staged per tile in k_rrs_zscatter

// X^T(c, l*k + s) = sum_a ZV[l nz + off_s + a] Y(r_a, c): the coordinates of
// Z_l^T Y, for l in [l0, l0 + kZL) ∩ [0, nl).  Y row-major m x k, X^T column-major
// k x (nl k).  One CTA per (256-column tile, subdomain, l chunk); a thread
// owns two adjacent columns (16-byte Y loads) and reads the Z values two l at
// a time (16-byte shared loads): 8 shared loads per 32 FMAs.  Per column the
// sum over the rows a runs in ascending a (the one-column kernel's order).
__global__ void __launch_bounds__(128) k_rrs_zgather(const OpSub* __restrict__ pc, const int* __restrict__ rows,
                                                     const double* __restrict__ ZV, long long nz, int nl,
                                                     const double* __restrict__ Y, int k,
                                                     double* __restrict__ XT) {
  extern __shared__ __align__(16) double zs[];   // ns x kZL, then ns row ids
  const int s = blockIdx.y, l0 = blockIdx.z * kZL;
  const OpSub d = pc[s];
  int* rs = reinterpret_cast<int*>(zs + (size_t)d.ns * kZL);
  const int nlc = min(kZL, nl - l0);
  for (int idx = threadIdx.x; idx < d.ns * kZL; idx += blockDim.x) {
    const int j = idx / d.ns, a = idx - j * d.ns;
    zs[a * kZL + j] = j < nlc ? ZV[(size_t)(l0 + j) * nz + d.map_off + a] : 0.0;
  }
  for (int a = threadIdx.x; a < d.ns; a += blockDim.x) rs[a] = rows[d.map_off + a];
  __syncthreads();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (c >= k) return;
  const bool two = c + 1 < k, vec = two && (k % 2 == 0);
  double acc0[kZL], acc1[kZL];
#pragma unroll
  for (int j = 0; j < kZL; ++j) acc0[j] = acc1[j] = 0.0;
  // rows with r < 0 contribute y = 0, which leaves acc unchanged
  auto row = [&](int a, double y0, double y1) {
    const double2* z2 = reinterpret_cast<const double2*>(zs + a * kZL);
#pragma unroll
    for (int j = 0; j < kZL / 2; ++j) {
      const double2 z = z2[j];
      acc0[2 * j] = fma(z.x, y0, acc0[2 * j]);
      acc0[2 * j + 1] = fma(z.y, y0, acc0[2 * j + 1]);
      acc1[2 * j] = fma(z.x, y1, acc1[2 * j]);
      acc1[2 * j + 1] = fma(z.y, y1, acc1[2 * j + 1]);
    }
  };
  auto load = [&](int a, double& y0, double& y1) {
    y0 = 0.0;
    y1 = 0.0;
    const int r = rs[a];
    if (r < 0) return;
    const double* yp = Y + (size_t)r * k + c;
    if (vec) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(yp));
      y0 = v.x;
      y1 = v.y;
    } else {
      y0 = yp[0];
      y1 = two ? yp[1] : 0.0;
    }
  };
  int a = 0;
  for (; a + 4 <= d.ns; a += 4) {   // four rows' loads in flight
    double y[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) load(a + u, y[u][0], y[u][1]);
#pragma unroll
    for (int u = 0; u < 4; ++u) row(a + u, y[u][0], y[u][1]);
  }
  for (; a < d.ns; ++a) {
    double y0, y1;
    load(a, y0, y1);
    row(a, y0, y1);
  }
#pragma unroll
  for (int j = 0; j < kZL; ++j)
    if (j < nlc) {
      double* xp = XT + (size_t)((size_t)(l0 + j) * k + s) * k + c;
      xp[0] = acc0[j];
      if (two) xp[1] = acc1[j];
    }
}

// D(r_a, c) += sum_l ZV[l nz + off_s + a] N^T(c, l*k + s) over the map rows of
// subdomain s.  Per (row, column) the sum over l runs in a fixed order (chunks
// of kZC coordinates in registers, partial sums in shared memory) and lands in
// D with one atomic; D is zeroed and each dual row has exactly two owners, so
// the two contributions commute exactly and D is deterministic.
// N^T column-major k x (nl k).  Dynamic smem: kZRows x (kZC + 128) doubles.
__global__ void __launch_bounds__(128) k_rrs_zscatter(const OpSub* __restrict__ pc, const int* __restrict__ rows,
                                                      const double* __restrict__ ZV, long long nz, int nl,
                                                      const double* __restrict__ NT, int k,
                                                      double* __restrict__ D) {
  extern __shared__ double sm[];
  double* zs = sm;                         // kZRows x kZC
  double* vacc = sm + kZRows * kZC;        // kZRows x 128 (row a, thread)
  const int s = blockIdx.y;
  const OpSub d = pc[s];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  for (int a0 = 0; a0 < d.ns; a0 += kZRows) {
    const int na = min(kZRows, d.ns - a0);
    for (int a = 0; a < na; ++a) vacc[a * 128 + threadIdx.x] = 0.0;
    for (int l0 = 0; l0 < nl; l0 += kZC) {
      const int nlc = min(kZC, nl - l0);
      double nr[kZC];
#pragma unroll
      for (int j = 0; j < kZC; ++j)
        nr[j] = (c < k && j < nlc) ? NT[(size_t)((size_t)(l0 + j) * k + s) * k + c] : 0.0;
      __syncthreads();
      for (int idx = threadIdx.x; idx < na * kZC; idx += blockDim.x) {
        const int j = idx / na, a = idx - j * na;
        zs[a * kZC + j] = j < nlc ? ZV[(size_t)(l0 + j) * nz + d.map_off + a0 + a] : 0.0;
      }
      __syncthreads();
      for (int a = 0; a < na; ++a) {
        double v = vacc[a * 128 + threadIdx.x];
#pragma unroll
        for (int j = 0; j < kZC; ++j) v = fma(zs[a * kZC + j], nr[j], v);
        vacc[a * 128 + threadIdx.x] = v;
      }
    }
    if (c < k)
      for (int a = 0; a < na; ++a) {
        const int r = rows[d.map_off + a0 + a];
        if (r >= 0) atomicAdd(D + (size_t)r * k + c, vacc[a * 128 + threadIdx.x]);
      }
    __syncthreads();
  }
}
constexpr size_t kZScatterSmem = (size_t)kZRows * (kZC + 128) * 8;

// column-major n x n block at ld: identity
__global__ void k_identity_ld(double* X, int n, int ld) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx - (long long)j * n);
    X[(size_t)j * ld + i] = i == j ? 1.0 : 0.0;
  }
}

// out(:, c) = in(:, perm[c]) for column-major blocks (rows x cols)
__global__ void k_gather_cols_cm(const double* __restrict__ in, int ldi, const int* __restrict__ perm, int rows,
                                 int cols, double* __restrict__ out, int ldo) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)rows * cols;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(idx / rows), i = (int)(idx - (long long)c * rows);
    out[(size_t)c * ldo + i] = in[(size_t)perm[c] * ldi + i];
  }
}

// yh = 0; yh[perm[c]] = y[c] for c < rank; also tp[c] = t[perm[c]] (gather)
__global__ void k_perm_gather(const double* __restrict__ t, const int* __restrict__ perm, int rank,
                              double* __restrict__ tp) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < rank; c += gridDim.x * blockDim.x) tp[c] = t[perm[c]];
}
__global__ void k_perm_scatter(const double* __restrict__ y, const int* __restrict__ perm, int rank, int k,
                               double* __restrict__ yh) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) yh[c] = 0.0;
  __syncthreads();
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < rank; c += gridDim.x * blockDim.x) yh[perm[c]] = y[c];
}

// the nine per-phase timing events of an RRS solve
struct PhaseEvents {
  cudaEvent_t ev[9] = {};
  PhaseEvents() {
    for (auto& e : ev) CK(cudaEventCreate(&e));
  }
  ~PhaseEvents() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  PhaseEvents(const PhaseEvents&) = delete;
  PhaseEvents& operator=(const PhaseEvents&) = delete;
};

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
  static const bool cl1 = [] {   // FETIGPU_PIVCHOL_CL1=0: the three-barrier kernel with physical swaps
    const char* e = getenv("FETIGPU_PIVCHOL_CL1");
    return !(e && e[0] == '0');
  }();
  if (cl1) {
    static std::atomic<int> ok1{-1};
    if (ok1.load() < 0) {
      bool good = cudaFuncSetAttribute(k_pivchol_cl1<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       225 * 1024) == cudaSuccess;
      if (good && CL > 8)
        good = cudaFuncSetAttribute(k_pivchol_cl1<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
               cudaSuccess;
      if (!good) cudaGetLastError();
      ok1.store(good ? 1 : 0);
    }
    if (ok1.load() && cudaLaunchKernelEx(&cfg, k_pivchol_cl1<CL>, A, n, tol, perm, rank, status) == cudaSuccess)
      return true;
    cudaGetLastError();
  }
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
// else a cooperative-grid kernel -- k_pivchol_coop1 (one grid barrier per
// pivot) when an n x n scratch `lc` is given, k_pivchol_coop otherwise
// (FETIGPU_PIVCHOL_COOP0=1 forces it).  Scratch: ctl 4 ints, gx 2n + 64 doubles.
static void launch_pivchol(double* A, int n, double tol, int* perm, int* rank, int* status, int* ctl, double* gx,
                           cudaStream_t st, double* lc = nullptr) {
  static const bool no_cluster = [] {   // FETIGPU_PIVCHOL_CLUSTER=0: blocked / cooperative kernels for every n
    const char* e = getenv("FETIGPU_PIVCHOL_CLUSTER");
    return e && e[0] == '0';
  }();
  if (!no_cluster && launch_pivchol_cluster(A, n, tol, perm, rank, status, gx, st)) return;
  // blocked (panels of kPcNB pivots, one grid-wide trailing phase per panel;
  // the per-entry arithmetic of k_pivchol_coop1): at[] lives in perm, the
  // running diagonal and the control block in gx (2n + 64 doubles)
  static const bool blocked = [] {
    const char* e = getenv("FETIGPU_PIVCHOL_BLOCKED");
    return !(e && e[0] == '0');
  }();
  if (lc && blocked && (size_t)n * 12 <= 200 * 1024) {
    double* d = gx;
    PcCtl* pc = reinterpret_cast<PcCtl*>(gx + n + 8);
    k_pc_init<<<1, 1024, 0, st>>>(A, n, tol, perm, d, pc);
    raise_smem_limit(k_pc_panel, (size_t)n * 12);
    const int nb = (n + 63) / 64;
    for (int k0 = 0; k0 < n; k0 += kPcNB) {
      k_pc_panel<<<1, 1024, (size_t)n * 12, st>>>(A, n, perm, d, lc, pc, status);
      k_pc_trailing<<<dim3(nb, nb), 256, 0, st>>>(A, n, perm, lc, pc, k0);
    }
    k_pc_finish<<<grid_for((long long)n * n), kThreads, 0, st>>>(A, n, perm, lc, pc, perm, rank);
    LAUNCH_CHECK();
    return;
  }
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const char* e = getenv("FETIGPU_PIVCHOL_COOP0");
  const size_t smem = (size_t)n * 12;
  if (lc && !(e && e[0] == '1') && smem <= 200 * 1024) {
    raise_smem_limit(k_pivchol_coop1, smem);
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pivchol_coop1, 512, smem));
    if (per_sm > 0) {
      const int blocks = sms * std::min(per_sm, 2);
      void* args[] = {&A, &n, &tol, &perm, &rank, &status, &lc, &gx};
      CK(cudaLaunchCooperativeKernel((void*)k_pivchol_coop1, dim3(blocks), dim3(512), args, smem, st));
      return;
    }
  }
  static std::atomic<int> coop_blocks{0};  // (see pivchol_cluster_try: benign duplicated init)
  if (!coop_blocks.load()) {
    int per_sm = 0;
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
  if (use_implicit_store(o)) return solve_rrs_implicit(o, lambda_host, tr);
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
  pivx.alloc(2 * (size_t)Ns + 64);
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
  pt.mark("rrs setup", st);
  CK(cudaEventRecord(ev0, st));
  init_lambda(lam.p);
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
  PhaseEvents pe;   // destroyed on every exit path (errors throw out of the loop)
  cudaEvent_t* pev = pe.ev;
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
    // line 8: Delta = Q^T W (column-major k x k): the lower tiles of the
    // m-deep product (split-K with a fixed segment sum), mirrored.
    gemm_splitk(st, false, true, k, k, m, 1.0, Qb.p, k, W.p, k, 0.0, Delta.p, k, dla_ws(gemm_splitk_ws(k, k, m)),
                kGemmLowerTiles);
    k_mirror_lower<<<grid_for((long long)k * k), kThreads, 0, st>>>(Delta.p, k);
    mark(2);
    // line 9
    launch_pivchol(Delta.p, k, o.pivot_tol, perm.p, rank_d.p, d_status.p, ctl.p, pivx.p, st, Linv.p);
    LAUNCH_CHECK();
    mark(3);
    int rank = 0, hstat = 0;
    CK(cudaMemcpyAsync(&rank, rank_d.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hstat, d_status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hstat) {
      CK(cudaMemsetAsync(d_status.p, 0, sizeof(int), st));
      CK(cudaStreamSynchronize(st));
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
    tri_inv_lower(st, Delta.p, k, rank, Linv.p, rank, dla_ws(tri_inv_workspace(rank)));
    // W_sel lands in Q's (still free) arena slot, W_new = W_sel L~^{-T} in W's;
    // then Q_sel lands in W (no longer needed) and Q_new = Q_sel L~^{-T}.
    // (L~^{-T} is upper triangular: column c of the product ends at index c.)
    const dim3 tgrid((m + 31) / 32, (rank + 31) / 32);
    k_gather_cols_t<<<tgrid, dim3(32, 8), 0, st>>>(W.p, k, perm.p, rank, m, Qn, m);
    gemm(st, false, true, m, rank, rank, 1.0, Qn, m, Linv.p, rank, 0.0, Wn, m, kGemmKEndByCol);
    k_gather_cols_t<<<tgrid, dim3(32, 8), 0, st>>>(Qb.p, k, perm.p, rank, m, W.p, m);
    gemm(st, false, true, m, rank, rank, 1.0, W.p, m, Linv.p, rank, 0.0, Qn, m, kGemmKEndByCol);
    K += rank;
    if (trace_on) {
      const auto tb = std::chrono::steady_clock::now();
      CK(cudaStreamSynchronize(st));
      fprintf(stderr, "[fetigpu] rrs it %4d  compress kernels drained in %.2f ms after append\n", it + 1,
              std::chrono::duration<double, std::milli>(tb - ta).count());
    }
    mark(4);
    // lines 13-15
    gemv_cm_t_tall(st, m, rank, Wn, m, r.p, gamma.p, dla_ws((size_t)kGvSeg * rank));
    gemv_cm(st, false, m, rank, 1.0, Wn, m, gamma.p, 1.0, lam.p);
    gemv_cm(st, false, m, rank, 1.0, Qn, m, gamma.p, 0.0, tmp.p);
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
        gemm_splitk(st, true, true, ch.used, Ns, m, 1.0, ch.q->p, m, W.p, Ns, 0.0, ch.psi->p, ch.cap,
                    dla_ws(gemm_splitk_ws(ch.used, Ns, m)));
      for (const Chunk& ch : chunks)  // W -= W_c Psi_c   ==   W^T -= Psi_c^T W_c^T
        gemm(st, true, true, Ns, m, ch.used, -1.0, ch.psi->p, ch.cap, ch.w->p, m, 1.0, W.p, Ns);
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
  if (chk_on && K > 0) {   // Alg. 1 orthonormality over all stored blocks
    std::vector<const double*> ws, qs;
    std::vector<int> rs;
    for (const Chunk& ch : chunks) { ws.push_back(ch.w->p); qs.push_back(ch.q->p); rs.push_back(ch.used); }
    check_orth(ws, qs, rs);
  }
  chunks.clear();
  pt.mark("rrs store release", st);
  return 0;
}


// Direction-store choice for FETI-DP RRS.  Explicit (Alg. 1 as written):
// W_j and Q_j = F W_j stored densely, 2 m rank_j doubles per iteration, and
// each CGS pass costs ~4 m k K flops (K stored columns).  Implicit (see
// solve_rrs_implicit): per iteration sum_s n_s packed values plus (i+1) k
// rank_i coefficients; each pass costs one block F-apply plus ~2 k^3 i^2
// flops of coefficient GEMMs.  Per iteration the explicit reorthogonalization is
// ~m k^2 i and the implicit one ~k^3 i^2, so the implicit store is cheaper
// while i < m / k -- once k is large enough that the implicit store's extra
// launches (2 block applies and ~4i coefficient GEMMs per iteration) do not
// dominate.  Measured (warm, tools/rrs_store_rep.py): C5 (k = 512) 176-200 ms
// implicit vs 446 ms explicit; C2 (k = 32) 37 vs 17-23 ms; C3 FETI-DP (k = 128)
// 21 vs 17.5 ms.  Auto therefore takes the implicit store when k >= 256 and
// m > 32 k, or when 32 iterations of the explicit store would not fit in free
// memory (C4: 16.5 GB per iteration).  T-FETI always uses the explicit store
// (its projected directions are dense).
bool Ctx::use_implicit_store(const fetigpu_solve_opts& o) {
  if (su.method != FETIGPU_FETIDP) return false;
  if (rrs_store == FETIGPU_RRS_STORE_EXPLICIT) return false;
  if (rrs_store == FETIGPU_RRS_STORE_IMPLICIT) return true;
  const char* e = getenv("FETIGPU_RRS_STORE");
  if (e && !strcmp(e, "explicit")) return false;
  if (e && !strcmp(e, "implicit")) return true;
  constexpr int kAutoIters = 32;
  if (su.Ns >= 256 && (long long)su.m > (long long)kAutoIters * su.Ns) return true;
  const double need = 16.0 * su.m * (double)su.Ns * std::min(o.max_it, kAutoIters);
  return need > 0.8 * (double)dev_free_bytes(&rrs_cache);
}

// Alg. 1 for FETI-DP (identity projector) with an implicit direction store.
//
// Every stored block is W_j = sum_{l<=j} Z_l M_j[l] where Z_l is the block of
// per-subdomain preconditioned residual columns of iteration l: column s is
// nonzero only on subdomain s's dual rows, so Z_l is kept packed (sum_s n_s
// values instead of m k).  The re-orthogonalization coefficient of Alg. 1,
// Psi_j = Q_j^T V with Q_j = F W_j, is formed as W_j^T (F V) (F symmetric),
// so Q_j is never stored either: each CGS pass applies F to the current block
// once (K5) and works on the Z coordinates,
//     X = Zhat^T (F V)            (packed gather GEMM, k_rrs_zgather)
//     Psi_j = M_j^T X,  N = sum_j M_j Psi_j        (cuBLAS)
//     V <- V - Zhat N             (packed scatter GEMM, k_rrs_zscatter)
// and the coordinates of V over Z_0..Z_{i+1} are [-sum N ; I].  The line-10/11
// compression acts on those coordinates: M_i = C_W[:, perm] L~^{-T}; the
// lambda / r updates use W, F W and the pivoted factor directly.
// Memory per iteration: sum_s n_s packed values + (i+1) k x rank_i
// coefficients, against 2 m rank_i for the explicit store (C4: 8 MB + 34 MB
// x (i+1) against 16.5 GB).  Three K5 applies per iteration instead of one.
// Same arithmetic as Alg. 1 up to rounding (the coefficient form of the CGS
// products); iteration and kept-direction counts are checked against the
// oracle in tests/test_gpu_parity.py.
int Ctx::solve_rrs_implicit(const fetigpu_solve_opts& o, double* lambda_host, fetigpu_trace* tr) {
  const int m = su.m, Ns = su.Ns, k = Ns;
  const int passes = std::max(1, o.reorth_passes);
  PhaseTimer pt;
  rhs();
  std::vector<OpSub> hpc(Ns);
  CK(cudaMemcpyAsync(hpc.data(), d_pc.p, Ns * sizeof(OpSub), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (KRp != 1) fail(FETIGPU_E_STATE, "implicit RRS store needs a one-row-per-DOF preconditioner map");
  long long nz = 0;
  int max_pcn = 0;
  for (auto& d : hpc) { nz = std::max<long long>(nz, (long long)d.map_off + d.ns); max_pcn = std::max(max_pcn, d.ns); }
  DBuf<double> lam, r, z, q, W, Qb, Dd, Delta, Linv, tvec, tp, gam, yh, ZV, XT, NT, NTot, CW, CT;
  DBuf<int> perm, rank_d, ctl;
  DBuf<Scal> sc;
  DBuf<double> pivx;
  lam.alloc(m); r.alloc(m); z.alloc(m); q.alloc(m);
  W.alloc((size_t)m * k); Qb.alloc((size_t)m * k);
  Delta.alloc((size_t)k * k); Linv.alloc((size_t)k * k);
  tvec.alloc(k); tp.alloc(k); gam.alloc(k); yh.alloc(k);
  perm.alloc(k); rank_d.alloc(1); ctl.alloc(4); pivx.alloc(2 * (size_t)k + 64);
  sc.alloc(1);
  sc.zero(st);
  // Everything the first nl_pre iterations need is allocated here, before
  // the timed loop: a multi-GB cudaMalloc / cudaFree inside an iteration
  // synchronises the device and occasionally stalls for 100+ ms in the
  // driver.  nl_pre = min(max_it, 32), reduced until the
  // coordinate scratch and the M_j arena fit in 40% of free memory; beyond
  // it the buffers grow by doubling.
  const char* nbz = getenv("FETIGPU_NO_BZ");   // A/B switch: dense K5 / scatter+AXPY paths
  const bool use_bz = !(nbz && nbz[0] == '1') && bz_prepare();
  // line 7 from the kept F Z_l (k_fz_correct) after two CGS passes
  const char* nfz = getenv("FETIGPU_NO_FZ");
  const bool use_fz = use_bz && passes >= 2 && !(nfz && nfz[0] == '1');
  const long long ystride = use_fz ? bz_nmap * kZNb : 0;
  const char* nfz2 = getenv("FETIGPU_NO_FZ2");
  const bool use_fz2 = use_fz && !(nfz2 && nfz2[0] == '1');
  DBuf<double> dnorm;
  dnorm.alloc(2);
  int n_fz2 = 0, n_k5_2 = 0;
  const size_t tstride = use_fz ? (size_t)tot_c() * kZNb : 0;   // compact A''^T X per Z block
  int nl_pre = std::max(1, std::min(o.max_it, 32));
  {
    const size_t freeb = dev_free_bytes(&rrs_cache);
    auto need = [&](int nlp) {
      const double kk = (double)k * k;
      return 8.0 * (5.0 * (nlp + 1) * kk + kk * nlp * (nlp + 1) / 2.0 + (double)nz * (nlp + 1) +
                    (double)(ystride + tstride) * (nlp + 1));
    };
    while (nl_pre > 1 && need(nl_pre) > 0.4 * (double)freeb) --nl_pre;
  }
  // packed Z blocks (column-major nz x zcap, grown by doubling) and the
  // per-iteration coordinate scratch, grown to (i+1) k x k as i increases
  int zcap = nl_pre + 1;
  ZV.alloc((size_t)nz * zcap);
  DBuf<double> Yst, Tst;   // F Z_l kept for the line-7 correction (use_fz)
  if (use_fz) { Yst.alloc((size_t)ystride * zcap); Tst.alloc(tstride * zcap); }
  auto regrow = [&](DBuf<double>& b, size_t per, int oldc, int newc) {
    if (!per) return;
    DBuf<double> b2;
    b2.alloc(per * newc);
    CK(cudaMemcpyAsync(b2.p, b.p, per * oldc * 8, cudaMemcpyDeviceToDevice, st));
    std::swap(b2.p, b.p);
    std::swap(b2.n, b.n);
  };
  auto zv_block = [&](int l) {
    if (l >= zcap) {
      const int nc = std::max(l + 1, 2 * zcap);
      regrow(ZV, (size_t)nz, zcap, nc);
      if (use_fz) { regrow(Yst, (size_t)ystride, zcap, nc); regrow(Tst, tstride, zcap, nc); }
      zcap = nc;
    }
  };
  // M_j ((j+1)k x rank_j, column-major) carved from arena chunks: the
  // first holds nl_pre iterations, later ones double
  std::vector<std::unique_ptr<DBuf<double>>> Mchunks;
  size_t mc_used = 0;
  std::vector<double*> Mb;
  std::vector<int> Mrank;
  auto m_alloc = [&](size_t n) {
    if (Mchunks.empty() || mc_used + n > Mchunks.back()->n) {
      const size_t cap_n = std::max(n, Mchunks.empty() ? n * 4 : 2 * Mchunks.back()->n);
      Mchunks.emplace_back(new DBuf<double>);
      Mchunks.back()->alloc(cap_n);
      mc_used = 0;
    }
    double* p0 = Mchunks.back()->p + mc_used;
    mc_used += (n + 31) & ~size_t(31);
    return p0;
  };
  auto grow2 = [](DBuf<double>& b, size_t n) {
    if (b.n < n) b.alloc(std::max(n, 2 * b.n));
    return b.p;
  };
  {
    const size_t kk = (size_t)k * k, kzmax = (size_t)(nl_pre + 1) * k;
    grow2(CW, kzmax * k); grow2(XT, kzmax * k); grow2(NT, kzmax * k); grow2(NTot, kzmax * k); grow2(CT, kzmax * k);
    Mchunks.emplace_back(new DBuf<double>);
    Mchunks.back()->alloc(kk * (size_t)nl_pre * (nl_pre + 1) / 2 + 32 * (size_t)nl_pre);
    dla_ws(std::max({gemm_splitk_ws(k, k, (int)kzmax), tri_inv_workspace(k), (size_t)kGvSeg * k,
                     (size_t)64 << 20}));   // the split-K cap
    ensure_block_buffers(k);
  }
  Scal* hs = nullptr;
  CK(cudaMallocHost(&hs, sizeof(Scal)));
  std::unique_ptr<Scal, decltype(&cudaFreeHost)> hs_guard(hs, cudaFreeHost);
  raise_smem_limit(k_rrs_zgather, (size_t)max_pcn * (kZL * 8 + 4));
  raise_smem_limit(k_rrs_zscatter, kZScatterSmem);
  pt.mark("rrs-implicit setup", st);
  CK(cudaEventRecord(ev0, st));
  init_lambda(lam.p);
  apply_F(lam.p, q.p, 1, m, m);
  int fapp = 1;
  k_sub<<<grid_for(m), kThreads, 0, st>>>(m, d_d.p, q.p, r.p);
  apply_precond(r.p, z.p, W.p, true);  // Alg. 1 line 2: W = Z_0
  dots({{r.p, z.p}, {r.p, r.p}, {z.p, z.p}}, &sc.p->rz);
  k_rrs_zpack<<<Ns, kThreads, 0, st>>>(d_pc.p, d_pcrows.p, W.p, k, ZV.p, nz, 0);
  k_identity_ld<<<grid_for((long long)k * k), kThreads, 0, st>>>(CW.p, k, k);  // C_W = I over Z_0
  LAUNCH_CHECK();
  CK(cudaMemcpyAsync(hs, sc.p, sizeof(Scal), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  auto metric = [&](const Scal& sv) {
    if (sv.rz < -1e-14 * std::sqrt(sv.rr) * std::sqrt(sv.zz))
      fail(FETIGPU_E_NEGATIVE_INNER_PRODUCT, "r^T z < 0: preconditioner is not symmetric positive");
    return std::sqrt(std::max(sv.rz, 0.0));
  };
  const double eps0 = metric(*hs);
  double eps = eps0;
  int it = 0, status = FETIGPU_MAX_ITER, K = 0;
  auto push = [&](double e, int kept) {
    if (tr && it < tr->cap) {
      if (tr->eps) tr->eps[it] = e;
      if (tr->kept) tr->kept[it] = kept;
      if (tr->f_app) tr->f_app[it] = fapp;
    }
  };
  push(eps0, Ns);
  const double target = o.rel ? o.tol * eps0 : o.tol;
  PhaseEvents pe;   // destroyed on every exit path (errors throw out of the loop)
  cudaEvent_t* pev = pe.ev;
  double phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto mark = [&](int i) { CK(cudaEventRecord(pev[i], st)); };
  const char* tenv = getenv("FETIGPU_TRACE");
  const bool trace_on = tenv && tenv[0] == '1';
  const dim3 ggrid((k + 255) / 256, Ns, 1), sgrid((k + 127) / 128, Ns);
  while (true) {
    if (eps <= target) { status = FETIGPU_CONVERGED; break; }
    if (it >= o.max_it) { status = FETIGPU_MAX_ITER; break; }
    const int i = it;              // stored blocks 0..i-1; W has coordinates CW over Z_0..Z_i
    const int kzi = (i + 1) * k;   // rows of CW
    mark(0);
    // line 7: at i = 0, W = Z_0 is a fresh preconditioner block (K5z); later
    // F V2 = F V1 - (F Zhat) N2 from the kept F Z_l (k_fz_correct), else K5
    if (i == 0 && use_bz && apply_F_block_z(W.p, Qb.p, k, use_fz ? Yst.p : nullptr, use_fz ? Tst.p : nullptr)) {
    } else if (use_fz && i >= 1 && i <= kZsMax) {
      const int Nc = su.Nc;
      k_fz_coarse<<<dim3((k + 255) / 256, Nc), 256, 0, st>>>(d_optr.p, fz_osub.p, fz_orow.p, bz_nbr.p, Tst.p,
                                                             (long long)tstride, i, NT.p, k, blk_T.p);
      LAUNCH_CHECK();
      gemm(st, false, false, k, Nc, Nc, 1.0, blk_T.p, k, d_Kinv.p, Nc, 0.0, blk_U.p, k);   // U_c
      launch_fz_correct(Yst.p, ystride, i, NT.p, blk_U.p, k, Qb.p);
      LAUNCH_CHECK();
    } else {
      apply_F_block(W.p, k, Qb.p, k, k);
    }
    fapp += k;
    mark(1);
    // line 8 on coordinates: Delta = Q^T W = (Zhat^T Q)^T C_W over Z_0..Z_i --
    // a packed gather plus a (i+1)k-deep GEMM instead of an m-deep one (C4:
    // 2 (i+1) k^3 against 2 m k^2 flops)
    grow2(XT, (size_t)kzi * k);
    k_rrs_zgather<<<dim3(ggrid.x, Ns, (i + 1 + kZL - 1) / kZL), 128, (size_t)max_pcn * (kZL * 8 + 4), st>>>(
        d_pc.p, d_pcrows.p, ZV.p, nz, i + 1, Qb.p, k, XT.p);
    LAUNCH_CHECK();
    gemm_splitk(st, false, false, k, k, kzi, 1.0, XT.p, k, CW.p, kzi, 0.0, Delta.p, k,
                dla_ws(gemm_splitk_ws(k, k, kzi)), kGemmLowerTiles);
    k_mirror_lower<<<grid_for((long long)k * k), kThreads, 0, st>>>(Delta.p, k);
    mark(2);
    launch_pivchol(Delta.p, k, o.pivot_tol, perm.p, rank_d.p, d_status.p, ctl.p, pivx.p, st, Linv.p);  // line 9
    LAUNCH_CHECK();
    mark(3);
    int rank = 0, hstat = 0;
    CK(cudaMemcpyAsync(&rank, rank_d.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hstat, d_status.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hstat) {
      CK(cudaMemsetAsync(d_status.p, 0, sizeof(int), st));
      CK(cudaStreamSynchronize(st));
      fail(FETIGPU_E_INDEFINITE_INPUT, "pivoted Cholesky: negative pivot");
    }
    if (rank == 0) { status = FETIGPU_BREAKDOWN; break; }
    // lines 10-11 on the coordinates: M_i = CW[:, perm] L~^{-T}
    tri_inv_lower(st, Delta.p, k, rank, Linv.p, rank, dla_ws(tri_inv_workspace(rank)));
    Mb.push_back(m_alloc((size_t)kzi * rank));
    Mrank.push_back(rank);
    grow2(CT, (size_t)kzi * k);
    k_gather_cols_cm<<<grid_for((long long)kzi * rank), kThreads, 0, st>>>(CW.p, kzi, perm.p, kzi, rank, CT.p,
                                                                           kzi);
    gemm(st, false, true, kzi, rank, rank, 1.0, CT.p, kzi, Linv.p, rank, 0.0, Mb.back(), kzi, kGemmKEndByCol);
    K += rank;
    mark(4);
    // lines 13-15: gamma = L~^{-1} (W^T r)[perm], y = L~^{-T} gamma,
    // lambda += W yh, r -= (F W) yh with yh = y scattered to perm
    gemv_rm_t(st, W.p, k, m, k, r.p, tvec.p, dla_ws((size_t)kGvSeg * k));
    k_perm_gather<<<1, 1024, 0, st>>>(tvec.p, perm.p, rank, tp.p);
    gemv_cm(st, false, rank, rank, 1.0, Linv.p, rank, tp.p, 0.0, gam.p);
    gemv_cm(st, true, rank, rank, 1.0, Linv.p, rank, gam.p, 0.0, tp.p);
    k_perm_scatter<<<1, 1024, 0, st>>>(tp.p, perm.p, rank, k, yh.p);
    raise_smem_limit(k_rrs_update, (size_t)k * 8);
    k_rrs_update<<<148 * 8, 256, (size_t)k * 8, st>>>(W.p, Qb.p, k, m, k, yh.p, lam.p, r.p);
    LAUNCH_CHECK();
    mark(5);
    // line 16: Z_{i+1}
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
      fprintf(stderr, "[fetigpu] rrs-implicit it %4d  eps/eps0 %.3e  rank %5d  K %7d  t %9.1f ms  (pass-2 F: %d kept-FZ, %d K5)\n",
              it, eps / eps0, rank, K, te, n_fz2, n_k5_2);
    }
    if (eps <= target || it >= o.max_it) {  // no next block needed
      mark(7);
      mark(8);
    } else {
      zv_block(it);
      k_rrs_zpack<<<Ns, kThreads, 0, st>>>(d_pc.p, d_pcrows.p, W.p, k, ZV.p, nz, it);
      LAUNCH_CHECK();
      mark(7);
      // lines 18-21 in coordinates over Z_0..Z_{it-1} (the stored blocks use
      // Z_0..Z_{it-1}; Z_it is the new block itself)
      const int nl = it, kz = nl * k;
      grow2(XT, (size_t)kz * k); grow2(NT, (size_t)kz * k); grow2(NTot, (size_t)kz * k);
      grow2(CT, (size_t)kz * k); grow2(CW, (size_t)(kz + k) * k);
      for (int p = 0; p < passes; ++p) {
        // Y = F V; the first pass sees V = Z_it itself (K5z, F Z_it kept for line 7).
        // Later passes: F V_p = F V_{p-1} - (F Zhat) N_{p-1} from the kept F Z_l
        // when the previous pass removed at most 3/4 of the block's norm
        // (||V_p|| >= ||V_{p-1}|| / 2, so the subtraction's rounding stays at
        // the level of a direct apply); otherwise the block apply (K5).
        bool fz_pass = false;
        if (p > 0 && use_fz && use_fz2 && nl <= kZsMax) {
          double hn[2];
          CK(cudaMemcpyAsync(hn, dnorm.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
          fz_pass = hn[1] >= 0.25 * hn[0];
          ++(fz_pass ? n_fz2 : n_k5_2);
        }
        if (fz_pass) {
          k_fz_coarse<<<dim3((k + 255) / 256, su.Nc), 256, 0, st>>>(d_optr.p, fz_osub.p, fz_orow.p, bz_nbr.p, Tst.p,
                                                                    (long long)tstride, nl, NT.p, k, blk_T.p);
          gemm(st, false, false, k, su.Nc, su.Nc, 1.0, blk_T.p, k, d_Kinv.p, su.Nc, 0.0, blk_U.p, k);
          launch_fz_correct(Yst.p, ystride, nl, NT.p, blk_U.p, k, Qb.p);
          LAUNCH_CHECK();
        } else if (!(p == 0 && use_bz &&
                     apply_F_block_z(W.p, Qb.p, k, use_fz ? Yst.p + (size_t)it * ystride : nullptr,
                                     use_fz ? Tst.p + (size_t)it * tstride : nullptr))) {
          apply_F_block(W.p, k, Qb.p, k, k);
        }
        fapp += k;
        if (use_fz2 && p + 1 < passes) block_norm2(W.p, (size_t)m * k, dnorm.p);   // ||V_p||^2
        k_rrs_zgather<<<dim3(ggrid.x, Ns, (nl + kZL - 1) / kZL), 128, (size_t)max_pcn * (kZL * 8 + 4), st>>>(
            d_pc.p, d_pcrows.p, ZV.p, nz, nl, Qb.p, k, XT.p);
        LAUNCH_CHECK();
        // Psi_j^T = X^T[:, 0:(j+1)k] M_j (k x rank_j, stored in CT at column offset sum rank),
        // N^T = sum_j Psi_j^T M_j^T (k x (j+1)k prefixes), largest j first with beta 0
        int off = 0;
        std::vector<int> poff(Mb.size());
        for (size_t j = 0; j < Mb.size(); ++j) {
          poff[j] = off;
          const int kj = (int)(j + 1) * k;
          gemm_splitk(st, false, false, k, Mrank[j], kj, 1.0, XT.p, k, Mb[j], kj, 0.0, CT.p + (size_t)off * k, k,
                      dla_ws(gemm_splitk_ws(k, Mrank[j], kj)));
          off += Mrank[j];
        }
        for (int j = (int)Mb.size() - 1; j >= 0; --j) {
          const int kj = (j + 1) * k;
          const double beta = j == (int)Mb.size() - 1 ? 0.0 : 1.0;
          gemm(st, false, true, k, kj, Mrank[j], 1.0, CT.p + (size_t)poff[j] * k, k, Mb[j], kj, beta, NT.p, k);
        }
        if (use_bz && nl <= kZsMax) {   // V -= Zhat N, once per dual row (interface-edge groups)
          const size_t zs = (size_t)kBzRows * nl * 2 * 8;
          raise_smem_limit(k_rrs_zsub_edges, zs);
          k_rrs_zsub_edges<<<dim3((k + kBzCols - 1) / kBzCols, bz_nedges), kBzCols, zs, st>>>(
              bz_edges.p, bz_erow.p, bz_ez1.p, bz_ez2.p, ZV.p, nz, nl, NT.p, k, W.p);
          LAUNCH_CHECK();
        } else {
          if (Dd.n < (size_t)m * k) Dd.alloc((size_t)m * k);
          CK(cudaMemsetAsync(Dd.p, 0, (size_t)m * k * 8, st));
          k_rrs_zscatter<<<sgrid, 128, kZScatterSmem, st>>>(d_pc.p, d_pcrows.p, ZV.p, nz, nl, NT.p, k, Dd.p);
          LAUNCH_CHECK();
          axpy(st, (size_t)m * k, -1.0, Dd.p, W.p);
        }
        if (use_fz2 && p + 1 < passes) block_norm2(W.p, (size_t)m * k, dnorm.p + 1);   // ||V_{p+1}||^2
        if (p == 0) CK(cudaMemcpyAsync(NTot.p, NT.p, (size_t)kz * k * 8, cudaMemcpyDeviceToDevice, st));
        else axpy(st, (size_t)kz * k, 1.0, NT.p, NTot.p);
      }
      // coordinates of the new W over Z_0..Z_it: [-NTot^T ; I]
      const int kzn = (it + 1) * k;
      transpose_scale(st, kz, k, -1.0, NTot.p, k, CW.p, kzn);
      k_identity_ld<<<grid_for((long long)k * k), kThreads, 0, st>>>(CW.p + kz, k, kzn);
      LAUNCH_CHECK();
      mark(8);
    }
    CK(cudaEventSynchronize(pev[8]));
    float t = 0;
    for (int qi = 0; qi < 8; ++qi) {
      CK(cudaEventElapsedTime(&t, pev[qi], pev[qi + 1]));
      phase[qi] += t;
    }
  }
  if (tr)
    for (int qi = 0; qi < 8; ++qi) tr->phase_ms[qi] = phase[qi];
  CK(cudaEventRecord(ev1, st));
  const double ms = elapsed(ev0, ev1);
  CK(cudaMemcpyAsync(lambda_host, lam.p, m * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  pt.mark("rrs-implicit loop + readback", st);
  if (chk_on && !Mb.empty()) {
    // Alg. 1 orthonormality of the implicit store: W_j = sum_l Z_l M_j[l]
    // densely (test sizes), Q_j = F W_j by K5, then max |W^T F W - I|
    const int nb = (int)Mb.size();
    DBuf<double> Zd;
    Zd.alloc((size_t)m * k * nb);
    CK(cudaMemsetAsync(Zd.p, 0, (size_t)m * k * nb * 8, st));
    for (int l = 0; l < nb; ++l)
      k_rrs_zunpack<<<Ns, kThreads, 0, st>>>(d_pc.p, d_pcrows.p, ZV.p + (size_t)l * nz, k, Zd.p + (size_t)l * m * k);
    LAUNCH_CHECK();
    std::vector<std::unique_ptr<DBuf<double>>> Wd, Qd;
    std::vector<const double*> ws, qs;
    for (int j = 0; j < nb; ++j) {
      const int rk = Mrank[j], kj = (j + 1) * k;
      Wd.emplace_back(new DBuf<double>);
      Qd.emplace_back(new DBuf<double>);
      Wd.back()->alloc((size_t)m * rk);
      Qd.back()->alloc((size_t)m * rk);
      for (int l = 0; l <= j; ++l)   // W_j^T (rank x m) += M_j[l]^T Z_l^T
        gemm(st, true, false, rk, m, k, 1.0, Mb[j] + (size_t)l * k, kj, Zd.p + (size_t)l * m * k, k,
             l == 0 ? 0.0 : 1.0, Wd.back()->p, rk);
      apply_F_block(Wd.back()->p, rk, Qd.back()->p, rk, rk);
      ws.push_back(Wd.back()->p);
      qs.push_back(Qd.back()->p);
    }
    check_orth(ws, qs, Mrank, true);
  }
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
