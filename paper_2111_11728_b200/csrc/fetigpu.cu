// fetigpu.cu -- context, build orchestration, operators, engine and C-ABI.
//
// One context = one FETI problem resident on one GPU.  fetigpu_build runs the
// whole operator construction on the device (ND Schur tree -> per-slot dense
// local operators -> FETI-DP coarse inverse); afterwards every operator
// application, preconditioner, projection and the PCG/FO/RRS loop run on the
// context's stream without host work beyond scalar read-back.
#include <cublas_v2.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "fetigpu.h"
#include "kernels_apply.cuh"
#include "kernels_build.cuh"
#include "kernels_dmma.cuh"
#include "setup.hpp"

namespace fg {

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      fail(e_ == cudaErrorMemoryAllocation ? FETIGPU_E_OUT_OF_MEMORY : FETIGPU_E_CUDA,         \
           std::string(#x) + ": " + cudaGetErrorString(e_));                                   \
  } while (0)
#define CB(x)                                                                                  \
  do {                                                                                         \
    cublasStatus_t s_ = (x);                                                                   \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                           \
      fail(FETIGPU_E_CUDA, std::string(#x) + " failed (cuBLAS status " + std::to_string((int)s_) + \
                               ", line " + std::to_string(__LINE__) + ")");                    \
  } while (0)
#define LAUNCH_CHECK()                                                                         \
  do {                                                                                         \
    cudaError_t e_ = cudaGetLastError();                                                       \
    if (e_ != cudaSuccess)                                                                     \
      fail(e_ == cudaErrorMemoryAllocation ? FETIGPU_E_OUT_OF_MEMORY : FETIGPU_E_CUDA,         \
           std::string("kernel launch before fetigpu.cu:") + std::to_string(__LINE__) + ": " +  \
               cudaGetErrorString(e_));                                                        \
  } while (0)

static size_t g_device_bytes = 0;

// Device memory: cudaMalloc behind a per-device cache of large blocks.  A freed
// block is kept and handed to a later request it fits (at most 2x larger), so
// repeated builds and solves in one process (SIMP loops, the bench's config
// table) reuse memory instead of paying variable cudaMalloc / cudaFree costs.
// A release first synchronises the device (cudaFree semantics: buffers freed
// at scope end are never still in use).  On OOM the cache is returned to the
// driver and the allocation retried.  FETIGPU_NO_CACHE=1 disables the cache.
struct BlockCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;      // capacity -> block
  std::unordered_map<void*, size_t> capacity;    // every live or cached block
  size_t cached = 0;
};
static BlockCache& block_cache() {
  static BlockCache caches[64];
  int dev = 0;
  cudaGetDevice(&dev);
  return caches[dev & 63];
}
static bool cache_on() {
  static const bool on = [] {
    const char* e = getenv("FETIGPU_NO_CACHE");
    return !(e && e[0] == '1');
  }();
  return on;
}
// Only the RRS direction store goes through the cache: its multi-GB chunks are
// allocated and freed per solve, and that is where driver allocation cost
// varied (up to ~0.9 s per C5 solve).  Everything else keeps a fresh
// cudaMalloc placement -- measured: caching the build workspace or operator
// storage made the L2-resident applies of C2 / C3 6-10% slower.
static void* dev_alloc(size_t bytes, bool cached) {
  bytes = (bytes + 511) & ~size_t(511);
  BlockCache& C = block_cache();
  if (!cached) {
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    return p;
  }
  if (cache_on()) {
    std::lock_guard<std::mutex> lk(C.mu);
    auto it = C.free_blocks.lower_bound(bytes);
    if (it != C.free_blocks.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      C.cached -= it->first;
      C.free_blocks.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaErrorMemoryAllocation && cache_on()) {  // give the cache back, retry
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(C.mu);
    cudaDeviceSynchronize();
    for (auto& f : C.free_blocks) {
      cudaFree(f.second);
      C.capacity.erase(f.second);
    }
    C.free_blocks.clear();
    C.cached = 0;
    e = cudaMalloc(&p, bytes);
  }
  CK(e);
  if (cache_on()) {
    std::lock_guard<std::mutex> lk(C.mu);
    C.capacity[p] = bytes;
  }
  return p;
}
static void dev_free(void* p) {
  if (!cache_on()) {
    cudaFree(p);
    return;
  }
  BlockCache& C = block_cache();
  std::unique_lock<std::mutex> lk(C.mu);
  auto it = C.capacity.find(p);
  if (it == C.capacity.end()) {  // small block: plain cudaFree
    lk.unlock();
    cudaFree(p);
    return;
  }
  cudaDeviceSynchronize();  // cudaFree semantics: nothing still uses the buffer
  C.free_blocks.emplace(it->second, p);
  C.cached += it->second;
}
// free device memory including the cached blocks
static size_t dev_free_bytes() {
  size_t freeb = 0, total = 0;
  CK(cudaMemGetInfo(&freeb, &total));
  if (cache_on()) {
    BlockCache& C = block_cache();
    std::lock_guard<std::mutex> lk(C.mu);
    freeb += C.cached;
  }
  return freeb;
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) {
      dev_free(p);
      g_device_bytes -= n * sizeof(T);
    }
    p = nullptr;
    n = 0;
  }
  bool cached = false;  // recycled scratch: allocate through the block cache
  void alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    p = static_cast<T*>(dev_alloc(count * sizeof(T), cached));
    n = count;
    g_device_bytes += n * sizeof(T);
  }
  void upload(const std::vector<T>& v, cudaStream_t st) {
    alloc(v.size());
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  }
  void zero(cudaStream_t st) { CK(cudaMemsetAsync(p, 0, n * sizeof(T), st)); }
};

static inline int round_up(int v, int a) { return (v + a - 1) / a * a; }

// Launch with programmatic dependent launch (PDL): the kernel may be scheduled
// while its predecessor in the stream finishes and waits in pdl_wait() (every
// kernel launched this way calls it first), which hides the launch latency
// between the small dependent kernels of a solver iteration.  FETIGPU_NO_PDL=1
// launches them normally.
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("FETIGPU_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}
template <class... KArgs, class... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// f(i) for i in [0, n) over up to 16 host threads (contiguous ranges); f must
// write disjoint outputs.  Serial for small n.
template <class F>
static void parallel_for(int n, F&& f) {
  const int nt = std::min<int>(16, std::max(1u, std::thread::hardware_concurrency()));
  if (n < 64 || nt <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const int a = (int)((long long)n * t / nt), b = (int)((long long)n * (t + 1) / nt);
      for (int i = a; i < b; ++i) f(i);
    });
  for (auto& x : th) x.join();
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is per function and process-wide:
// contexts of different sizes may be alive at once, so it is only ever raised.
template <class K>
static void raise_smem_limit(K* func, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[(const void*)func];
  if (bytes > c) {
    CK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    c = bytes;
  }
}

// FETIGPU_TIMING=1: host wall-clock marks of the build phases on stderr
struct PhaseTimer {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  PhaseTimer() {
    const char* e = getenv("FETIGPU_TIMING");
    on = e && e[0] == '1';
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what, cudaStream_t st) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[fetigpu] %-28s %8.2f ms (total %8.2f)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(),
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};
static inline int grid_for(long long n, int threads = kThreads, int cap = 148 * 16) {
  long long g = (n + threads - 1) / threads;
  return (int)std::max<long long>(1, std::min<long long>(g, cap));
}

// Grow-only device scratch buffers keyed by slot: build temporaries reuse
// them instead of cudaMalloc/cudaFree per level / chunk (cudaFree is a
// device-wide synchronization).
struct Scratch {
  std::vector<std::unique_ptr<DBuf<char>>> bufs;
  void* get(int id, size_t bytes) {
    if ((int)bufs.size() <= id) bufs.resize(id + 1);
    if (!bufs[id]) bufs[id] = std::make_unique<DBuf<char>>();
    if (bufs[id]->n < bytes) bufs[id]->alloc(bytes + bytes / 4);
    return bufs[id]->p;
  }
  template <class T>
  T* upload(int id, const std::vector<T>& v, cudaStream_t st) {
    T* p = static_cast<T*>(get(id, std::max<size_t>(1, v.size()) * sizeof(T)));
    if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return p;
  }
  void release(int id) {
    if (id < (int)bufs.size() && bufs[id]) bufs[id]->release();
  }
};
enum ScratchId { kScWs = 0, kScDescA, kScDescB, kScSlots, kScSrc, kScExt, kScMo, kScMl, kScAo, kScKo, kScFo,
                 kScMisc };

struct Ctx {
  Setup su;
  Scratch scratch;
  cudaStream_t st = nullptr;
  cublasHandle_t cb = nullptr;
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
  std::vector<int> sub_maxrow;  // per subdomain: largest dual row it touches (-1: none)

  ~Ctx() {
    for (auto& e : pipe_in) if (e) cudaEventDestroy(e);
    for (auto& e : pipe_done) if (e) cudaEventDestroy(e);
    if (pipe_start) cudaEventDestroy(pipe_start);
    for (auto& q : pipe_st) if (q) cudaStreamDestroy(q);
    if (pipe_cp) cudaStreamDestroy(pipe_cp);
    if (cb) cublasDestroy(cb);
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

  void init_device() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      fail(FETIGPU_E_NO_DEVICE, "no CUDA device available");
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CB(cublasCreate(&cb));
    CB(cublasSetStream(cb, st));
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

  double elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  }

  // ------------------------------------------------------------ build --
  void eliminate(const std::vector<FrontDesc>& fds, double* base) {
    std::vector<FrontDesc> small, large;
    int nfmax = 0;
    for (auto& f : fds) {
      if (f.nf <= kSmallFront && f.ld == f.nf) { small.push_back(f); nfmax = std::max(nfmax, f.nf); }
      else large.push_back(f);
    }
    if (!small.empty()) {
      FrontDesc* ds = scratch.upload(kScDescA, small, st);
      const int thr = nfmax <= 64 ? 64 : (nfmax <= 96 ? 128 : kThreads);
      k_front_elim_small<<<(int)small.size(), thr, nfmax * nfmax * 8, st>>>(ds, base, d_status.p);
      LAUNCH_CHECK();
    }
    if (!large.empty()) {
      FrontDesc* dl = scratch.upload(kScDescB, large, st);
      bpc(dl, large, base);
    }
  }

  // batched blocked partial Cholesky over all frontals in `fs` (device copy `d`)
  void bpc(const FrontDesc* d, const std::vector<FrontDesc>& fs, double* base) {
    const char* legacy = getenv("FETIGPU_LEGACY_ELIM");
    if (legacy && legacy[0] == '1') {
      k_front_elim_large<<<(int)fs.size(), kThreads, 0, st>>>(d, base, d_status.p);
      LAUNCH_CHECK();
      return;
    }
    int ne_max = 0, nf_max = 0;
    for (auto& f : fs) { ne_max = std::max(ne_max, f.ne); nf_max = std::max(nf_max, f.nf); }
    const int B = (int)fs.size();
    raise_smem_limit(k_bpc_update, kBpcUpdateSmem);
    for (int k0 = 0; k0 < ne_max; k0 += kBpcNB) {
      k_bpc_diag<<<B, kThreads, 0, st>>>(d, base, k0, d_status.p);
      const int rows = std::max(1, nf_max - k0 - 1);
      k_bpc_trsm<<<dim3((rows + kThreads - 1) / kThreads, B), kThreads, 0, st>>>(d, base, k0);
      const int nt = (rows + kTile - 1) / kTile;
      k_bpc_update<<<dim3(nt * (nt + 1) / 2, B), kThreads, kBpcUpdateSmem, st>>>(d, base, k0);
      LAUNCH_CHECK();
    }
  }

  void build_nd() {
    const NdPlan& P = su.nd;
    const int nb = su.nb, n = su.n, D = su.n_designs;
    std::vector<NdDev> nodes(P.nodes.size());
    std::vector<int> elem_ids, emap, cmaps, dofs;
    for (size_t i = 0; i < P.nodes.size(); ++i) {
      const NdNode& s = P.nodes[i];
      NdDev& d = nodes[i];
      d.nf = s.nf; d.ne = s.ne; d.leaf = s.leaf; d.height = s.height;
      d.off = s.off; d.foff = s.foff;
      d.elem_off = (int)elem_ids.size();
      d.elem_cnt = (int)s.elems.size();
      elem_ids.insert(elem_ids.end(), s.elems.begin(), s.elems.end());
      emap.insert(emap.end(), s.emap.begin(), s.emap.end());
      for (int c = 0; c < 2; ++c) {
        d.child[c] = s.child[c];
        d.cmap_off[c] = (int)cmaps.size();
        cmaps.insert(cmaps.end(), s.cmap[c].begin(), s.cmap[c].end());
      }
      d.dof_off = (int)dofs.size();
      dofs.insert(dofs.end(), s.dofs.begin(), s.dofs.end());
    }
    d_nodes.upload(nodes, st);
    d_elem_ids.upload(elem_ids, st);
    d_emap.upload(emap, st);
    d_cmaps.upload(cmaps, st);
    d_nd_dofs.upload(dofs, st);
    d_topdown.upload(P.topdown, st);
    d_dens.upload(su.densities, st);
    d_S.alloc((size_t)D * nb * nb);
    if (keep_factors) d_ndfac.alloc((size_t)D * P.factor_stride);

    long long per_design = 0;
    for (long long s : P.height_stride) per_design += s;
    const size_t free_b = dev_free_bytes();
    // workspace capped at 8 GB: more, smaller chunks beat one huge cold cudaMalloc
    const long long budget = std::max<long long>(256ll << 20, std::min<long long>(8ll << 30, (long long)(free_b * 0.3)));
    const int chunk = (int)std::max<long long>(1, std::min<long long>(D, budget / (per_design * 8)));
    double* ws_p = static_cast<double*>(scratch.get(kScWs, (size_t)chunk * per_design * 8));
    // per-height node lists split by size
    std::vector<std::vector<int>> hsmall(P.max_height + 1), hlarge(P.max_height + 1);
    std::vector<int> hnfmax(P.max_height + 1, 0);
    for (int h = 0; h <= P.max_height; ++h)
      for (int t : P.by_height[h]) {
        if (P.nodes[t].nf <= kSmallFront) { hsmall[h].push_back(t); hnfmax[h] = std::max(hnfmax[h], P.nodes[t].nf); }
        else hlarge[h].push_back(t);
      }
    std::vector<DBuf<int>> dsm(P.max_height + 1), dlg(P.max_height + 1);
    for (int h = 0; h <= P.max_height; ++h) {
      dsm[h].upload(hsmall[h], st);
      dlg[h].upload(hlarge[h], st);
    }
    DBuf<long long> d_hbase, d_hstride;
    d_hstride.upload(P.height_stride, st);
    for (int d0 = 0; d0 < D; d0 += chunk) {
      const int dc = std::min(chunk, D - d0);
      std::vector<long long> hbase(P.max_height + 1, 0);
      long long acc = 0;
      for (int h = 0; h <= P.max_height; ++h) { hbase[h] = acc; acc += (long long)dc * P.height_stride[h]; }
      d_hbase.upload(hbase, st);
      NdArgs a{d_nodes.p, nullptr, d_hbase.p, d_hstride.p, ws_p, d_elem_ids.p, d_emap.p, d_cmaps.p,
               d_dens.p, n, d0, su.E0, su.Emin, su.p, keep_factors ? d_ndfac.p : nullptr,
               P.factor_stride, d_status.p};
      for (int h = 0; h <= P.max_height; ++h) {
        if (!hsmall[h].empty()) {
          a.level_nodes = dsm[h].p;
          dim3 grid((unsigned)hsmall[h].size(), dc);
          const int thr = hnfmax[h] <= 64 ? 64 : (hnfmax[h] <= 96 ? 128 : kThreads);
          k_nd_small<<<grid, thr, hnfmax[h] * hnfmax[h] * 8, st>>>(a);
          LAUNCH_CHECK();
        }
        if (!hlarge[h].empty()) {
          a.level_nodes = dlg[h].p;
          dim3 grid((unsigned)hlarge[h].size(), dc);
          k_nd_assemble<<<grid, kThreads, 0, st>>>(a);
          LAUNCH_CHECK();
          std::vector<FrontDesc> fds;
          for (int dl = 0; dl < dc; ++dl)
            for (int t : hlarge[h]) {
              const NdNode& nd = P.nodes[t];
              fds.push_back({hbase[h] + (long long)dl * P.height_stride[h] + nd.off, nd.nf, nd.ne, nd.nf,
                             FETIGPU_E_SINGULAR_INTERIOR});
            }
          FrontDesc* dfd = scratch.upload(kScDescB, fds, st);
          bpc(dfd, fds, ws_p);
          if (keep_factors) {
            k_nd_copy_factors<<<grid, kThreads, 0, st>>>(a);
            LAUNCH_CHECK();
          }
        }
      }
      k_nd_extract_root<<<dim3(grid_for((long long)nb * nb), dc), kThreads, 0, st>>>(
          d_nodes.p, P.root, d_hbase.p, d_hstride.p, ws_p, d_S.p, nb, d0);
      LAUNCH_CHECK();
      CK(cudaStreamSynchronize(st));
    }
    check_status();
  }

  // batched slot processing: assemble [[S[src,src],E],[E^T,0]], eliminate,
  // extract; processed in chunks bounded by a workspace budget
  struct SlotOut {
    std::vector<long long> mat_off;
    std::vector<int> mat_ld;
    std::vector<long long> abc_off, kcc_off, fac_off;
  };
  void run_slots(const std::vector<SlotFront>& slots, const SlotOut& out, double* mats, double sign,
                 bool nc_first, double* abc, double* kcc, double* fac, int errcode) {
    std::vector<int> src_all, ext_all;
    std::vector<SlotDev> sd(slots.size());
    for (size_t i = 0; i < slots.size(); ++i) {
      sd[i].design = slots[i].design;
      sd[i].nsrc = (int)slots[i].src.size();
      sd[i].ne = slots[i].ne;
      sd[i].next = (int)slots[i].ext.size();
      sd[i].src_off = (int)src_all.size();
      sd[i].ext_off = (int)ext_all.size();
      src_all.insert(src_all.end(), slots[i].src.begin(), slots[i].src.end());
      ext_all.insert(ext_all.end(), slots[i].ext.begin(), slots[i].ext.end());
    }
    DBuf<int> dsrc, dext;
    dsrc.upload(src_all, st);
    dext.upload(ext_all, st);
    const size_t free_b = dev_free_bytes();
    const long long budget =
        std::max<long long>(256ll << 20, std::min<long long>(8ll << 30, (long long)(free_b * 0.3))) / 8;
    size_t i0 = 0;
    while (i0 < slots.size()) {
      long long used = 0;
      size_t i1 = i0;
      std::vector<SlotDev> chunk;
      while (i1 < slots.size()) {
        const long long nf = slots[i1].nf();
        if (!chunk.empty() && used + nf * nf > budget) break;
        SlotDev d = sd[i1];
        d.woff = used;
        used += nf * nf;
        chunk.push_back(d);
        ++i1;
      }
      double* ws = static_cast<double*>(scratch.get(kScWs, (size_t)used * 8));
      SlotDev* dchunk = scratch.upload(kScSlots, chunk, st);
      const int nch = (int)chunk.size();
      k_slot_assemble<<<dim3(64, nch), kThreads, 0, st>>>(dchunk, dsrc.p, dext.p, d_S.p, su.nb, ws);
      LAUNCH_CHECK();
      std::vector<FrontDesc> fds;
      for (auto& c : chunk) fds.push_back({c.woff, c.nsrc + c.next, c.ne, c.nsrc + c.next, errcode});
      eliminate(fds, ws);
      auto sub = [&](const std::vector<long long>& v) {
        return std::vector<long long>(v.begin() + i0, v.begin() + i1);
      };
      long long* dmo = scratch.upload(kScMo, sub(out.mat_off), st);
      int* dml = scratch.upload(kScMl, std::vector<int>(out.mat_ld.begin() + i0, out.mat_ld.begin() + i1), st);
      long long* dao = abc ? scratch.upload(kScAo, sub(out.abc_off), st) : nullptr;
      long long* dko = abc ? scratch.upload(kScKo, sub(out.kcc_off), st) : nullptr;
      k_slot_extract<<<dim3(32, nch), kThreads, 0, st>>>(dchunk, ws, dmo, dml, mats, nc_first ? 1 : 0, sign, dao,
                                                         abc, dko, kcc);
      LAUNCH_CHECK();
      if (fac) {
        long long* dfo = scratch.upload(kScFo, sub(out.fac_off), st);
        k_slot_factor<<<dim3(32, nch), kThreads, 0, st>>>(dchunk, ws, dfo, fac);
        LAUNCH_CHECK();
      }
      if (i1 < slots.size()) CK(cudaStreamSynchronize(st));  // host vectors reused next chunk
      i0 = i1;
    }
    check_status();
  }

  PhaseTimer ptimer;
  void build_ops() {
    const int Ns = su.Ns, nb = su.nb;
    const bool dp = su.method == FETIGPU_FETIDP;
    ptimer.mark("build_ops start", st);
    // ---- operator slots
    const int nslot = (int)su.op_slots.size();
    SlotOut so;
    long long mo = 0, ao = 0, ko = 0, fo = 0;
    op_ns.resize(nslot); op_ld.resize(nslot); op_moff.resize(nslot); op_foff.resize(nslot);
    for (int i = 0; i < nslot; ++i) {
      const SlotFront& s = su.op_slots[i];
      const int ns = (int)s.ext.size(), ld = round_up(ns, 4), nc = (int)s.src.size() - s.ne;
      op_ns[i] = ns; op_ld[i] = ld; op_moff[i] = mo;
      so.mat_off.push_back(mo); so.mat_ld.push_back(ld);
      so.abc_off.push_back(ao); so.kcc_off.push_back(ko); so.fac_off.push_back(fo);
      op_foff[i] = fo;
      mo += (long long)ns * ld; ao += (long long)ns * nc; ko += (long long)nc * nc;
      fo += (long long)s.ne * s.ne;
      max_ld = std::max(max_ld, ld);
      max_ne = std::max(max_ne, s.ne);
    }
    d_opmat.alloc(mo);
    d_opfac.alloc(fo);
    if (dp) { d_abc.alloc(ao); d_kccs.alloc(ko); }
    ptimer.mark("op slot planning", st);
    run_slots(su.op_slots, so, d_opmat.p, -1.0, dp, dp ? d_abc.p : nullptr, dp ? d_kccs.p : nullptr,
              d_opfac.p, dp ? FETIGPU_E_SINGULAR_REMAINDER : FETIGPU_E_NOT_POSITIVE_DEFINITE);
    ptimer.mark("op slots (device)", st);
    // slot src/ext lists for rhs / recovery
    {
      std::vector<int> src, ext, so_, eo_, fne;
      for (auto& s : su.op_slots) {
        so_.push_back((int)src.size());
        eo_.push_back((int)ext.size());
        src.insert(src.end(), s.src.begin(), s.src.end());
        ext.insert(ext.end(), s.ext.begin(), s.ext.end());
        fne.push_back(s.ne);
      }
      d_op_src.upload(src, st); d_op_ext.upload(ext, st);
      d_op_src_off.upload(so_, st); d_op_ext_off.upload(eo_, st);
      d_fac_ne.upload(fne, st);
      d_fac_off.upload(so.fac_off, st);
    }
    ptimer.mark("slot src/ext lists", st);
    // ---- per-subdomain operator maps
    // flat (subdomain, perimeter position) -> up to 3 (row, sign, weight) entries
    struct Ent { int row; double coef; double w; };
    KR = dp ? 1 : 3;
    KRp = KR;
    // entries are read only below ecnt[k]: no zero fill (Ns x nb x KR of them)
    std::unique_ptr<Ent[]> ent(new Ent[(size_t)Ns * nb * KR]);
    std::vector<unsigned char> ecnt((size_t)Ns * nb, 0);
    auto add_ent = [&](int s, int pos, Ent e) {
      const size_t k = (size_t)s * nb + pos;
      if (ecnt[k] >= KR) fail(FETIGPU_E_STATE, "too many dual rows per DOF");
      ent[k * KR + ecnt[k]++] = e;
    };
    for (int i = 0; i < su.m; ++i) {
      const Row& r = su.rows[i];
      add_ent(r.sp, su.dpos[r.dp], {i, 1.0, su.wplus[i]});
      if (r.kind == 0) add_ent(r.sm, su.dpos[r.dm], {i, -1.0, su.wminus[i]});
    }
    ptimer.mark("maps: row entries", st);
    std::vector<OpSub> ops(Ns), pcs(Ns), pjs(Ns);
    std::vector<int> slot_of(Ns), top_off(Ns), design(Ns), rt_off(Ns);
    std::vector<size_t> ip_off(Ns);
    size_t ntop = 0, nT = 0;
    for (int s = 0; s < Ns; ++s) {  // output offsets first, so subdomains can be filled in parallel
      top_off[s] = (int)ntop;
      ip_off[s] = nT;
      ntop += su.subs[s].Top.size();
      nT += su.subs[s].T.size();
    }
    std::vector<int> rows(ntop * KR), prow(nT * KRp), top_pos(ntop);
    std::vector<double> coef(ntop * KR), pcoef(nT * KRp), pjcoef(nT * KRp), RT(nT * 3);
    sub_maxrow.assign(Ns, -1);
    parallel_for(Ns, [&](int s) {
      const SubPlan& S = su.subs[s];
      const int sl = S.op_slot;
      size_t io = (size_t)top_off[s], ip = ip_off[s];
      slot_of[s] = sl;
      design[s] = S.design;
      ops[s] = {op_moff[sl], op_ns[sl], op_ld[sl], (int)(io * KR), 0};
      int mx = -1;
      for (int t : S.Top) {
        const size_t k = (size_t)s * nb + t;
        top_pos[io] = t;
        for (int q = 0; q < KR; ++q) {
          const bool has = q < ecnt[k];
          rows[io * KR + q] = has ? ent[k * KR + q].row : -1;
          coef[io * KR + q] = has ? ent[k * KR + q].coef : 0.0;
          mx = std::max(mx, rows[io * KR + q]);
        }
        ++io;
      }
      sub_maxrow[s] = mx;
      // preconditioner / projector maps over T
      pcs[s] = {0, (int)S.T.size(), 0, (int)(ip * KRp), 0};
      pjs[s] = pcs[s];
      rt_off[s] = (int)(ip * 3);
      for (int t : S.T) {
        const size_t k = (size_t)s * nb + t;
        for (int q = 0; q < KRp; ++q) {
          const bool has = q < ecnt[k];
          prow[ip * KRp + q] = has ? ent[k * KR + q].row : -1;
          pcoef[ip * KRp + q] = has ? ent[k * KR + q].coef * ent[k * KR + q].w : 0.0;
          pjcoef[ip * KRp + q] = has ? ent[k * KR + q].coef : 0.0;
        }
        for (int q = 0; q < 3; ++q) RT[ip * 3 + q] = su.Rb[(size_t)q * nb + t];
        ++ip;
      }
    });
    ptimer.mark("maps: host loops", st);
    d_oprows.upload(rows, st); d_opcoef.upload(coef, st);
    d_slot_of.upload(slot_of, st); d_design.upload(design, st);
    d_top_pos.upload(top_pos, st); d_top_off.upload(top_off, st);
    d_pcrows.upload(prow, st); d_pccoef.upload(pcoef, st);

    ptimer.mark("per-subdomain maps (host)", st);
    // ---- preconditioner matrices
    std::vector<long long> pc_moff;
    std::vector<int> pc_ld;
    long long pm = 0;
    const int npc = su.precond == FETIGPU_DIRICHLET ? (int)su.pc_slots.size() : (int)su.pc_lumped_T.size();
    for (int i = 0; i < npc; ++i) {
      const int nt = su.precond == FETIGPU_DIRICHLET ? (int)(su.pc_slots[i].src.size() - su.pc_slots[i].ne)
                                                    : (int)su.pc_lumped_T[i].size();
      const int ld = round_up(nt, 4);
      pc_moff.push_back(pm); pc_ld.push_back(ld);
      pm += (long long)nt * ld;
      max_pc_ld = std::max(max_pc_ld, ld);
    }
    d_pcmat.alloc(pm);
    if (su.precond == FETIGPU_DIRICHLET) {
      SlotOut po;
      po.mat_off = pc_moff; po.mat_ld = pc_ld;
      run_slots(su.pc_slots, po, d_pcmat.p, 1.0, false, nullptr, nullptr, nullptr, FETIGPU_E_SINGULAR_INTERIOR);
    } else {
      // K_bb per design from element contributions
      std::vector<int> pne(su.nb / 2 * 4, -1);
      const int n = su.n, nn = n + 1;
      for (int q = 0; q < su.nb / 2; ++q) {
        const int v = su.perim_dof[2 * q] / 2, vx = v % nn, vy = v / nn;
        int cnt = 0;
        std::vector<std::pair<int, int>> el;
        for (int ey = std::max(0, vy - 1); ey <= std::min(n - 1, vy); ++ey)
          for (int ex = std::max(0, vx - 1); ex <= std::min(n - 1, vx); ++ex) {
            const int n0 = ey * nn + ex;
            const int en[4] = {n0, n0 + 1, n0 + nn + 1, n0 + nn};
            for (int a = 0; a < 4; ++a)
              if (en[a] == v) el.push_back({ey * n + ex, a});
          }
        std::sort(el.begin(), el.end());
        for (auto& e : el) {
          if (cnt < 2) { pne[q * 4 + 2 * cnt] = e.first; pne[q * 4 + 2 * cnt + 1] = e.second; }
          ++cnt;
        }
        if (cnt > 2) fail(FETIGPU_E_STATE, "perimeter node with > 2 elements");
      }
      DBuf<int> dpne, dpd;
      dpne.upload(pne, st);
      dpd.upload(su.perim_dof, st);
      DBuf<double> kbb;
      kbb.alloc((size_t)su.n_designs * nb * nb);
      k_kbb<<<dim3(grid_for((long long)nb * nb), su.n_designs), kThreads, 0, st>>>(
          d_dens.p, n, su.E0, su.Emin, su.p, dpne.p, dpd.p, nb, kbb.p);
      LAUNCH_CHECK();
      std::vector<int> tall, toff, tcnt;
      for (auto& T : su.pc_lumped_T) {
        toff.push_back((int)tall.size());
        tcnt.push_back((int)T.size());
        tall.insert(tall.end(), T.begin(), T.end());
      }
      DBuf<int> dt, dto, dtc, dsd, dld;
      DBuf<long long> dmo;
      dt.upload(tall, st); dto.upload(toff, st); dtc.upload(tcnt, st);
      dsd.upload(su.pc_lumped_design, st);
      dmo.upload(pc_moff, st); dld.upload(pc_ld, st);
      k_pc_lumped<<<dim3(16, npc), kThreads, 0, st>>>(dsd.p, dto.p, dtc.p, dt.p, kbb.p, nb, dmo.p, dld.p,
                                                     d_pcmat.p, su.precond == FETIGPU_SUPERLUMPED);
      LAUNCH_CHECK();
      CK(cudaStreamSynchronize(st));
    }
    ptimer.mark("preconditioner slots", st);
    for (int s = 0; s < Ns; ++s) {
      const int sl = su.subs[s].pc_slot;
      pcs[s].moff = pc_moff[sl];
      pcs[s].ld = pc_ld[sl];
    }
    d_pc.upload(pcs, st);
    d_op.upload(ops, st);

    // ---- T-FETI projector data
    if (!dp) {
      d_pj.upload(pjs, st);
      d_pjcoef.upload(pjcoef, st);
      d_RT.upload(RT, st);
      d_rt_off.upload(rt_off, st);
      {  // invert the (subdomain, touched DOF) -> rows maps: per row its <= 2 entries
        std::vector<int2> sr((size_t)2 * std::max(1, su.m), make_int2(-1, 0));
        std::vector<double2> cc((size_t)std::max(1, su.m), make_double2(0.0, 0.0));
        for (int s = 0; s < Ns; ++s)
          for (size_t j = 0; j < su.subs[s].T.size(); ++j)
            for (int q = 0; q < KRp; ++q) {
              const size_t e = (ip_off[s] + j) * KRp + q;
              const int r = prow[e];
              if (r < 0) continue;
              const int slot = sr[2 * (size_t)r].x < 0 ? 0 : 1;
              if (slot == 1 && sr[2 * (size_t)r + 1].x >= 0)
                fail(FETIGPU_E_STATE, "projector: more than two entries in a dual row");
              sr[2 * (size_t)r + slot] = make_int2(s, rt_off[s] + (int)j * 3);
              (slot == 0 ? cc[r].x : cc[r].y) = pjcoef[e];
            }
        d_pjrow_sr.upload(sr, st);
        d_pjrow_c.upload(cc, st);
      }
      d_H.upload(su.H, st);
      std::vector<double> e(3 * Ns, 0.0);  // e = -R^T f (decomposition.hpp:127)
      for (int s = 0; s < Ns; ++s)
        for (int k = 0; k < 3; ++k) {
          double v = 0.0;
          for (int i = 0; i < nb; ++i) v += su.Rb[(size_t)k * nb + i] * su.subs[s].f[i];
          e[3 * s + k] = -v;
        }
      d_e.upload(e, st);
    }

    // ---- boundary data for rhs / recovery
    {
      std::vector<double> fb, gD;
      std::vector<int> Dl, Doff, Dcnt, cpos, coff, xoff;
      int xo = 0;
      for (int s = 0; s < Ns; ++s) {
        const SubPlan& S = su.subs[s];
        fb.insert(fb.end(), S.f.begin(), S.f.end());
        Doff.push_back((int)Dl.size());
        Dcnt.push_back((int)S.D.size());
        Dl.insert(Dl.end(), S.D.begin(), S.D.end());
        gD.insert(gD.end(), S.gD.begin(), S.gD.end());
        coff.push_back((int)cpos.size());
        cpos.insert(cpos.end(), S.c.begin(), S.c.end());
        xoff.push_back(xo);
        xo += su.op_slots[S.op_slot].ne;
      }
      d_fb.upload(fb, st); d_gD.upload(gD, st);
      d_D.upload(Dl, st); d_D_off.upload(Doff, st); d_D_cnt.upload(Dcnt, st);
      d_c_pos.upload(cpos, st); d_c_off.upload(coff, st);
      d_xoff.upload(xoff, st);
      d_xb.alloc(xo);
    }

    // ---- FETI-DP coarse problem
    if (dp) {
      std::vector<DpSub> dps(Ns);
      std::vector<int> cmap, voff, optr{0}, oidx, osub, oloc;
      int vo = 0, to = 0;
      std::vector<int> toff(Ns);
      for (int s = 0; s < Ns; ++s) {
        const SubPlan& S = su.subs[s];
        const int sl = S.op_slot;
        dps[s].abc_off = so.abc_off[sl];
        dps[s].nc = (int)S.c.size();
        if (dps[s].nc > 8) fail(FETIGPU_E_STATE, "more than 8 primal DOFs per subdomain");
        dps[s].cmap_off = (int)cmap.size();
        cmap.insert(cmap.end(), S.cg.begin(), S.cg.end());
        dps[s].v_off = vo;
        voff.push_back(vo);
        vo += (int)S.Top.size();
        dps[s].t_off = to;
        toff[s] = to;
        to += (int)S.c.size();
      }
      for (int i = 0; i < su.Nc; ++i) {
        for (auto& o : su.c_owners[i]) {
          oidx.push_back(toff[o.first] + o.second);
          osub.push_back(o.first);
          oloc.push_back(o.second);
        }
        optr.push_back((int)oidx.size());
      }
      d_dp.upload(dps, st);
      d_cmap.upload(cmap, st);
      d_voff.upload(voff, st);
      d_optr.upload(optr, st);
      d_oidx.upload(oidx, st);
      d_vbuf.alloc(vo);
      d_tbuf.alloc(std::max(1, to));
      d_fbar_loc.alloc(std::max(1, to));
      d_fbar.alloc(std::max(1, su.Nc));
      build_coarse(so, osub, oloc);
    }
    ptimer.mark("projector/boundary data", st);
    // ---- fold the +-1 signs of the FETI-DP constraint rows into F_s and A_bc
    d_opcoef_apply.upload(coef, st);
    if (dp) {
      const int nsl = (int)su.op_slots.size();
      slot_sign.assign(nsl, {});
      bool ok = true;
      for (int s = 0; s < Ns && ok; ++s) {
        const int sl = su.subs[s].op_slot;
        std::vector<double> sg(op_ns[sl]);
        for (int a = 0; a < op_ns[sl]; ++a) sg[a] = coef[ops[s].map_off + a];
        if (slot_sign[sl].empty()) slot_sign[sl] = sg;
        else if (slot_sign[sl] != sg) ok = false;
      }
      if (ok) {
        std::vector<long long> ao(nsl);
        std::vector<int> ncv(nsl), soff(nsl), nsv(nsl);
        std::vector<double> sgn;
        for (int i = 0; i < nsl; ++i) {
          ao[i] = so.abc_off[i];
          ncv[i] = (int)su.op_slots[i].src.size() - su.op_slots[i].ne;
          soff[i] = (int)sgn.size();
          nsv[i] = op_ns[i];
          sgn.insert(sgn.end(), slot_sign[i].begin(), slot_sign[i].end());
        }
        DBuf<long long> dmo, dao;
        DBuf<int> dns, dld, dnc, dso;
        DBuf<double> dsg;
        dmo.upload(op_moff, st); dao.upload(ao, st); dns.upload(nsv, st); dld.upload(op_ld, st);
        dnc.upload(ncv, st); dso.upload(soff, st); dsg.upload(sgn, st);
        k_fold_signs<<<dim3(64, nsl), kThreads, 0, st>>>(dmo.p, dns.p, dld.p, dao.p, dnc.p, dso.p, dsg.p,
                                                        d_opmat.p, d_abc.p);
        LAUNCH_CHECK();
        std::vector<double> ones(coef.size(), 1.0);
        for (size_t i = 0; i < rows.size(); ++i)
          if (rows[i] < 0) ones[i] = 0.0;
        d_opcoef_apply.upload(ones, st);
        CK(cudaStreamSynchronize(st));
        folded = true;
      }
    }
    ptimer.mark("coarse problem + folding", st);
    // ---- scratch
    const size_t m = std::max(1, su.m);
    d_v1.alloc(m); d_v2.alloc(m); d_v3.alloc(m);
    d_g.alloc(3 * (size_t)Ns + 8); d_h.alloc(3 * (size_t)Ns + 8);
    d_partial.alloc(4 * kDotBlocks);
    d_counter.alloc(1);
    d_counter.zero(st);
    d_counter2.alloc(1);
    d_counter2.zero(st);
    d_d.alloc(m); d_lam0.alloc(m);

    // ---- GEMV row split: aim for >= 4 CTAs per SM when subdomains are few
    rsplit = std::max(1, std::min(8, (4 * 148 + Ns - 1) / Ns));
    pc_rsplit = rsplit;
    // ---- symmetric-packed copy of F_s for the single-vector apply (K4)
    const char* nosym = getenv("FETIGPU_NO_SYM");
    const char* forcesym = getenv("FETIGPU_FORCE_SYM");
    const bool want_sym = rsplit == 1 || (forcesym && forcesym[0] == '1');
    if (want_sym && !(nosym && nosym[0] == '1')) {
      const int nsl = (int)su.op_slots.size();
      std::vector<long long> toff(nsl);
      long long tt = 0;
      int nbmax = 0;
      for (int i = 0; i < nsl; ++i) {
        const int nb = (op_ns[i] + 31) / 32;
        toff[i] = tt;
        tt += (long long)nb * (nb + 1) / 2 * 1024;
        nbmax = std::max(nbmax, nb);
      }
      d_symtiles.alloc(tt);
      DBuf<long long> dmo, dto;
      DBuf<int> dns, dld;
      dmo.upload(op_moff, st); dto.upload(toff, st); dns.upload(op_ns, st); dld.upload(op_ld, st);
      k_pack_sym<<<dim3(64, nsl), kThreads, 0, st>>>(dmo.p, dns.p, dld.p, dto.p, d_opmat.p, d_symtiles.p);
      LAUNCH_CHECK();
      std::vector<SymSub> ss(Ns);
      sym_bytes = 0;
      for (int s = 0; s < Ns; ++s) {
        const int sl = su.subs[s].op_slot;
        const int nb = (op_ns[sl] + 31) / 32;
        ss[s] = {toff[sl], op_ns[sl], nb, ops[s].map_off, 0};
        sym_bytes += (double)nb * (nb + 1) / 2 * 1024 * 8;
      }
      d_sym.upload(ss, st);
      sym_smem = nbmax * 32 * (1 + kSymWarps) * 8;
      raise_smem_limit(k_sym_gemv_scatter<1, true>, sym_smem);
      raise_smem_limit(k_sym_gemv_scatter<3, false>, sym_smem);
      CK(cudaStreamSynchronize(st));
      use_sym = true;
      // same packing for the (symmetric) preconditioner blocks S~_s / K_TT
      const int npc2 = (int)pc_moff.size();
      std::vector<long long> ptoff(npc2);
      std::vector<int> pns(npc2);
      long long pt = 0;
      int pnbmax = 0;
      for (int i = 0; i < npc2; ++i) {
        pns[i] = su.precond == FETIGPU_DIRICHLET ? (int)(su.pc_slots[i].src.size() - su.pc_slots[i].ne)
                                                 : (int)su.pc_lumped_T[i].size();
        const int nb = (pns[i] + 31) / 32;
        ptoff[i] = pt;
        pt += (long long)nb * (nb + 1) / 2 * 1024;
        pnbmax = std::max(pnbmax, nb);
      }
      d_pcsymtiles.alloc(pt);
      DBuf<long long> pmo, pto;
      DBuf<int> pnsd, pldd;
      pmo.upload(pc_moff, st); pto.upload(ptoff, st); pnsd.upload(pns, st); pldd.upload(pc_ld, st);
      k_pack_sym<<<dim3(64, npc2), kThreads, 0, st>>>(pmo.p, pnsd.p, pldd.p, pto.p, d_pcmat.p, d_pcsymtiles.p);
      LAUNCH_CHECK();
      std::vector<SymSub> pss(Ns);
      for (int s = 0; s < Ns; ++s) {
        const int sl = su.subs[s].pc_slot;
        pss[s] = {ptoff[sl], pns[sl], (pns[sl] + 31) / 32, pcs[s].map_off, 0};
      }
      d_pcsym.upload(pss, st);
      pc_sym_smem = pnbmax * 32 * (1 + kSymWarps) * 8;
      raise_smem_limit(k_sym_gemv_scatter<1, false>, pc_sym_smem);
      raise_smem_limit(k_sym_gemv_scatter<3, false>, pc_sym_smem);
      CK(cudaStreamSynchronize(st));
      pc_sym = true;
    }
    ptimer.mark("symmetric packing", st);
    setup_pipe();
    // ---- work per apply
    double sn2 = 0, snc = 0, sns = 0;
    for (int s = 0; s < Ns; ++s) {
      const double ns = (double)su.subs[s].Top.size();
      sn2 += ns * ns;
      sns += ns;
      if (dp) snc += ns * (double)su.subs[s].c.size();
    }
    double ld_bytes = 0;
    for (int s = 0; s < Ns; ++s) ld_bytes += 8.0 * op_ns[su.subs[s].op_slot] * op_ld[su.subs[s].op_slot];
    op_bytes = 8 * sn2 + (dp ? 16 * snc + 8.0 * su.Nc * su.Nc : 0) + 16.0 * su.m + 8 * sns;
    op_flops = 2 * sn2 + (dp ? 4 * snc + 2.0 * su.Nc * su.Nc : 0);
    main_bytes = 8 * sn2;
    (void)ld_bytes;
  }

  void build_coarse(const SlotOut& so, const std::vector<int>& osub, const std::vector<int>& oloc) {
    const int Nc = su.Nc;
    if (Nc == 0) return;
    // Kbar_cc = sum_s B_c^T Kbar_cc^s B_c, owners in ascending subdomain order
    std::vector<long long> kco(su.Ns);
    std::vector<int> ncs(su.Ns);
    for (int s = 0; s < su.Ns; ++s) {
      kco[s] = so.kcc_off[su.subs[s].op_slot];
      ncs[s] = (int)su.subs[s].c.size();
    }
    DBuf<long long> dkco;
    DBuf<int> dncs, dos, dol;
    dkco.upload(kco, st); dncs.upload(ncs, st); dos.upload(osub, st); dol.upload(oloc, st);
    DBuf<double> K;
    K.alloc((size_t)Nc * Nc);
    launch_kcc_assemble(d_optr.p, dos.p, dol.p, dkco.p, dncs.p, d_kccs.p, Nc, K.p);
    // blocked Cholesky: diagonal blocks by k_front_elim_large, panels by cuBLAS
    const int NBc = 256;
    const double one = 1.0, mone = -1.0, zero = 0.0;
    for (int k0 = 0; k0 < Nc; k0 += NBc) {
      const int kb = std::min(NBc, Nc - k0);
      std::vector<FrontDesc> f{{(long long)k0 * Nc + k0, kb, kb, Nc, FETIGPU_E_SINGULAR_COARSE}};
      DBuf<FrontDesc> df;
      df.upload(f, st);
      k_front_elim_large<<<1, kThreads, 0, st>>>(df.p, K.p, d_status.p);
      LAUNCH_CHECK();
      CK(cudaStreamSynchronize(st));
      const int rest = Nc - k0 - kb;
      if (rest > 0) {
        CB(cublasDtrsm(cb, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                       rest, kb, &one, K.p + (size_t)k0 * Nc + k0, Nc, K.p + (size_t)k0 * Nc + k0 + kb, Nc));
        CB(cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, rest, kb, &mone,
                       K.p + (size_t)k0 * Nc + k0 + kb, Nc, &one, K.p + (size_t)(k0 + kb) * Nc + k0 + kb, Nc));
      }
    }
    check_status();
    // inverse: X = L^{-1}, Kinv = X^T X
    DBuf<double> X;
    X.alloc((size_t)Nc * Nc);
    launch_identity(X.p, Nc);
    CB(cublasDtrsm(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, Nc, Nc,
                   &one, K.p, Nc, X.p, Nc));
    d_Kinv.alloc((size_t)Nc * Nc);
    CB(cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, Nc, Nc, &one, X.p, Nc, &zero, d_Kinv.p, Nc));
    launch_symmetrize(d_Kinv.p, Nc);
    // fused-gather target + arrival counters (always); symmetric-packed copy
    // of the inverse for the single-vector apply when it is large
    d_gc.alloc(Nc);
    d_gcnt.alloc(Nc);
    d_gcnt.zero(st);
    d_cgather.upload(std::vector<CoarseGather>{{d_gc.p, d_gcnt.p, d_optr.p, d_oidx.p, d_cmap.p}}, st);
    use_csym = Nc > 2048;
    if (!use_csym) {
      CK(cudaStreamSynchronize(st));
      return;
    }
    kinv_nb = (Nc + 31) / 32;
    const size_t ntiles = (size_t)kinv_nb * (kinv_nb + 1) / 2;
    d_kinv_tiles.alloc(ntiles * 1024);
    d_crow.alloc(ntiles * 32);
    d_ccol.alloc(ntiles * 32);
    {
      DBuf<long long> mo, to;
      DBuf<int> ns, ld;
      mo.upload(std::vector<long long>{0}, st); to.upload(std::vector<long long>{0}, st);
      ns.upload(std::vector<int>{Nc}, st); ld.upload(std::vector<int>{Nc}, st);
      k_pack_sym<<<dim3(grid_for((long long)ntiles * 1024), 1), kThreads, 0, st>>>(mo.p, ns.p, ld.p, to.p, d_Kinv.p,
                                                                                d_kinv_tiles.p);
      LAUNCH_CHECK();
      CK(cudaStreamSynchronize(st));
    }
    int dev = 0, sms = 0, per_sm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_csym_tiles, 128, 0));
    csym_grid = (int)std::max<long long>(1, std::min<long long>((long long)sms * std::max(1, per_sm),
                                                                ((long long)ntiles + 3) / 4));
  }

  // u = Kbar^{-1} (sum_s B_c^T t_s) into d_h (stages A + B on the packed inverse)
  // g_ready: phase 1 already formed g in d_gc (fused gather of the symmetric
  // GEMV); otherwise gather it here
  // zero_y: output still to be zeroed (the gather kernel does it when it runs)
  void coarse_solve_packed(bool g_ready, double* zero_y = nullptr) {
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

  void build() {
    ptimer = PhaseTimer();
    CK(cudaEventRecord(ev0, st));
    CK(cudaMemcpyToSymbolAsync(c_kunit, su.kunit, sizeof(su.kunit), 0, cudaMemcpyHostToDevice, st));
    build_nd();
    ptimer.mark("nested dissection", st);
    CK(cudaEventRecord(ev1, st));
    nd_ms = elapsed(ev0, ev1);
    build_ops();
    CK(cudaEventRecord(ev2, st));
    CK(cudaStreamSynchronize(st));
    scratch.release(kScWs);
    slot_ms = elapsed(ev1, ev2);
    build_ms = elapsed(ev0, ev2);
    built = true;
  }

  // -------------------------------------------------------- operators --
  // y_zeroed: the caller already zeroed y (T-FETI scatters into it); lets the
  // solver loop drop the memset node and chain the GEMV with PDL
  void apply_F(const double* x, double* y, int ncols, int ldx, int ldy, bool y_zeroed = false) {
    const int Ns = su.Ns;
    if (su.method == FETIGPU_TFETI) {
      if (ncols == 1 && y_zeroed) {
        if (use_sym)
          launch_pdl(k_sym_gemv_scatter<3, false>, Ns, 256, sym_smem, st, (const SymSub*)d_sym.p,
                     (const double*)d_symtiles.p, (const int*)d_oprows.p, (const double*)d_opcoef_apply.p, x, y,
                     (double*)nullptr, (const int*)nullptr, (const DpSub*)nullptr, (const double*)nullptr,
                     (double*)nullptr, 0, (double*)nullptr, 0, 1, (const CoarseGather*)nullptr);
        else
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
        for (int c = 0; c < ncols; ++c)
          k_sym_gemv_scatter<3, false><<<Ns, 256, sym_smem, st>>>(d_sym.p, d_symtiles.p, d_oprows.p,
                                                                  d_opcoef_apply.p, x + (size_t)c * ldx,
                                                                  y + (size_t)c * ldy, nullptr, nullptr);
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
          launch_pdl(k_sym_gemv_scatter<1, true>, Ns, 256, sym_smem, st, (const SymSub*)d_sym.p,
                     (const double*)d_symtiles.p, (const int*)d_oprows.p, (const double*)d_opcoef_apply.p, xc,
                     (double*)nullptr, d_vbuf.p, (const int*)d_voff.p, (const DpSub*)d_dp.p,
                     (const double*)d_abc.p, d_tbuf.p, 0, yc, su.m, Ns,
                     (const CoarseGather*)(su.Nc ? d_cgather.p : nullptr));
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

  void setup_pipe() {
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
    }
    pipe_ready = true;
  }

  // y = F x with x, y in (pinned) host memory; the result is identical to
  // the device path (same kernels per subdomain, same phase-2 order)
  void apply_F_host(const double* xh, double* yh) {
    const int m = su.m;
    stage(m);
    double* x = stage_x.p;
    double* y = stage_y.p;
    if (!pipe_ready) {
      CK(cudaMemcpyAsync(x, xh, (size_t)m * 8, cudaMemcpyHostToDevice, st));
      apply_F(x, y, 1, m, m);
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
        k_sym_gemv_scatter<1, true><<<nblk, 256, sym_smem, q>>>(d_sym.p, d_symtiles.p, d_oprows.p,
                                                                 d_opcoef_apply.p, x, nullptr, d_vbuf.p, d_voff.p,
                                                                 d_dp.p, d_abc.p, d_tbuf.p, pipe_s0[c], y, m,
                                                                 su.Ns, su.Nc ? d_cgather.p : nullptr);
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

  // Zcols: per-subdomain columns, column-major m x N_s (row_major = false)
  // or row-major m x N_s (row_major = true)
  void apply_precond(const double* r, double* z, double* Zcols, bool row_major = false, bool z_zeroed = false) {
    if (!z_zeroed) CK(cudaMemsetAsync(z, 0, su.m * 8, st));
    if (Zcols) CK(cudaMemsetAsync(Zcols, 0, (size_t)su.m * su.Ns * 8, st));
    const int ldz = row_major ? 1 : su.m, zrs = row_major ? su.Ns : 1;
    if (pc_sym && !Zcols) {
      auto k = KRp == 1 ? k_sym_gemv_scatter<1, false> : k_sym_gemv_scatter<3, false>;
      launch_pdl(k, su.Ns, 256, pc_sym_smem, st, (const SymSub*)d_pcsym.p, (const double*)d_pcsymtiles.p,
                 (const int*)d_pcrows.p, (const double*)d_pccoef.p, r, z, (double*)nullptr, (const int*)nullptr,
                 (const DpSub*)nullptr, (const double*)nullptr, (double*)nullptr, 0, (double*)nullptr, 0, 1,
                 (const CoarseGather*)nullptr);
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

  // ---- K5: Q = F W for k columns, row-major blocks (W(i,c) = W[i*ldw + c])
  DBuf<double> blk_t, blk_T, blk_U;
  void apply_F_block(const double* W, int ldw, double* Q, int ldq, int k) {
    const int Ns = su.Ns, m = su.m;
    if (ldq == k) CK(cudaMemsetAsync(Q, 0, (size_t)m * k * 8, st));
    else CK(cudaMemset2DAsync(Q, (size_t)ldq * 8, 0, (size_t)k * 8, m, st));
    BlockApplyArgs a{d_op.p, d_opmat.p, d_oprows.p, d_opcoef_apply.p, KR, nullptr, nullptr, nullptr, nullptr, 0,
                     W, ldw, Q, ldq, k};
    int max_ns = 0;
    for (int n : op_ns) max_ns = std::max(max_ns, n);
    if (su.method == FETIGPU_FETIDP) {
      const int Nc = su.Nc;
      int tot_c = 0;
      for (auto& S : su.subs) tot_c += (int)S.c.size();
      if (blk_t.n < (size_t)tot_c * k) blk_t.alloc((size_t)tot_c * k);
      if (blk_T.n < (size_t)Nc * k) { blk_T.alloc((size_t)Nc * k); blk_U.alloc((size_t)Nc * k); }
      {
        const size_t smem = ((size_t)std::max(max_ns * 8, 4 * 8 * kDpTCols) + max_ns) * 8 + (size_t)max_ns * 4;
        raise_smem_limit(k_block_dp_t, smem);
        k_block_dp_t<<<dim3((k + kDpTCols - 1) / kDpTCols, Ns), 256, smem, st>>>(
            d_op.p, d_dp.p, d_oprows.p, d_opcoef_apply.p, d_abc.p, W, ldw, k, blk_t.p, k);
      }
      k_coarse_gather_block<<<dim3((k + 255) / 256, Nc), 256, 0, st>>>(d_optr.p, d_oidx.p, blk_t.p, k, Nc, k,
                                                                       blk_T.p, k);
      const double one = 1.0, zero = 0.0;
      // U = Kbar^{-1} T  (row-major N_c x k == column-major k x N_c: U^T = T^T Kinv)
      CB(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, k, Nc, Nc, &one, blk_T.p, k, d_Kinv.p, Nc, &zero, blk_U.p, k));
      a.dps = d_dp.p; a.abc = d_abc.p; a.cmap = d_cmap.p; a.U = blk_U.p; a.ldu = k;
      max_ns += 8;
    }
    dim3 grid((k + kBN - 1) / kBN, (max_ns + kBM - 1) / kBM, Ns);
    const bool fast = folded && (k % 2 == 0) && (ldw % 2 == 0) && (ldq % 2 == 0) &&
                      ((uintptr_t)W % 16 == 0) && ((uintptr_t)Q % 16 == 0);
    if (fast) k_block_apply_dp<<<grid, 256, kAsyncSmem, st>>>(a);
    else if (KR == 1) k_block_apply<1><<<grid, 256, kBlockSmem, st>>>(a);
    else k_block_apply<3><<<grid, 256, kBlockSmem, st>>>(a);
    LAUNCH_CHECK();
  }

  // v <- P v for a row-major block (m x ncols, ld = ncols), T-FETI only
  // single-vector projector finish: per dual row its <= 2 (s, RT offset) / signs
  DBuf<int2> d_pjrow_sr;
  DBuf<double2> d_pjrow_c;

  // grow-only scratch for the multi-column projector paths: no cudaMalloc /
  // cudaFree (both device-synchronising) inside solver iterations once warm
  DBuf<double> ws_g, ws_h, ws_corr;
  static double* grow(DBuf<double>& b, size_t n) {
    if (b.n < n) b.alloc(n);
    return b.p;
  }

  void project_rm(double* v, int ncols) {
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

  // h = H g for ncols columns of length 3N_s (H symmetric, column-major)
  void small_gemm(const double* g, double* h, int ncols) {
    const int nc = 3 * su.Ns;
    if (ncols == 1) {
      k_dense_gemv<<<grid_for((long long)nc * 32), kThreads, 0, st>>>(d_H.p, nc, g, h);
    } else {
      const double one = 1.0, zero = 0.0;
      CB(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, nc, ncols, nc, &one, d_H.p, nc, g, nc, &zero, h, nc));
    }
    LAUNCH_CHECK();
  }

  // corr = P v - v for ncols columns (T-FETI); caller adds
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

  void proj_corr(const double* v, int ldv, double* corr, int ldc, int ncols, double gsign = -1.0) {
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

  void rhs() {
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

  void recover(const double* lambda_dev, double* u_dev) {
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

  // ------------------------------------------------------------ engine --
  void dots(std::initializer_list<std::pair<const double*, const double*>> pairs, double* out) {
    DotArgs a{};
    int k = 0;
    for (auto& p : pairs) { a.a[k] = p.first; a.b[k] = p.second; ++k; }
    a.npairs = k;
    a.n = su.m;
    const int nblk = std::max(1, std::min(kDotBlocks, (su.m + 1023) / 1024));
    launch_pdl(k_dot_fused, nblk, kThreads, 0, st, a, d_partial.p, d_counter.p, out);
    LAUNCH_CHECK();
  }

  void precond_projected(const double* r, double* z, double* Zcols) {
    apply_precond(r, z, Zcols);
    project(z, 1, su.m);
  }

  int solve(const fetigpu_solve_opts& o, double* lambda_host, fetigpu_trace* tr);
  int solve_rrs(const fetigpu_solve_opts& o, double* lam, fetigpu_trace* tr);
};

// ------------------------------------------------------- small kernels ----
__global__ void k_kcc_assemble(const int* optr, const int* osub, const int* oloc, const long long* kco,
                               const int* ncs, const double* kccs, int Nc, double* K) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)Nc * Nc;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / Nc), i = (int)(idx - (long long)j * Nc);
    double v = 0.0;
    int a = optr[i], b = optr[j];
    const int ae = optr[i + 1], be = optr[j + 1];
    while (a < ae && b < be) {
      const int sa = osub[a], sb = osub[b];
      if (sa == sb) {
        const int nc = ncs[sa];
        v += kccs[kco[sa] + (long long)oloc[a] * nc + oloc[b]];
        ++a; ++b;
      } else if (sa < sb) ++a;
      else ++b;
    }
    K[idx] = v;
  }
}
__global__ void k_identity(double* X, int n) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x)
    X[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
}
__global__ void k_symmetrize(double* A, int n) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx % n);
    if (i < j) A[idx] = A[(long long)i * n + j];
  }
}
void Ctx::launch_kcc_assemble(const int* optr, const int* osub, const int* oloc, const long long* kco,
                              const int* ncs, const double* kccs, int Nc, double* K) {
  k_kcc_assemble<<<grid_for((long long)Nc * Nc), kThreads, 0, st>>>(optr, osub, oloc, kco, ncs, kccs, Nc, K);
  LAUNCH_CHECK();
}
void Ctx::launch_identity(double* X, int n) {
  k_identity<<<grid_for((long long)n * n), kThreads, 0, st>>>(X, n);
  LAUNCH_CHECK();
}
void Ctx::launch_symmetrize(double* A, int n) {
  k_symmetrize<<<grid_for((long long)n * n), kThreads, 0, st>>>(A, n);
  LAUNCH_CHECK();
}

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
  const int cap = std::max(1, o.max_it);
  DBuf<double> psi_part;
  if (fo) {
    Wst.alloc((size_t)m * cap);
    Qst.alloc((size_t)m * cap);
    psi.alloc(cap);
  }
  const int psi_S = std::max(1, std::min(64, m / 2048));
  if (fo) psi_part.alloc((size_t)cap * psi_S);
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
  CK(cudaMemcpyAsync(lam.p, d_lam0.p, m * 8, cudaMemcpyDeviceToDevice, st));
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
      launch_pdl(k_fo_store2, grid_for(m), kThreads, 0, st, m, (const Scal*)sc.p, (const int*)cnt.p,
                 (const double*)w.p, q.p, Wst.p, Qst.p);
      launch_pdl(k_inc, 1, 1, 0, st, cnt.p);
      CK(cudaMemcpyAsync(w.p, z.p, m * 8, cudaMemcpyDeviceToDevice, st));
      for (int pss = 0; pss < passes; ++pss) {
        launch_pdl(k_fo_psi_seg, fo_seg_grid, 256, 0, st, (const double*)Qst.p, m, (const int*)cnt.p,
                   (const double*)w.p, psi_part.p, psi_S);
        launch_pdl(k_fo_psi_sum, (cap + 255) / 256, 256, 0, st, (const int*)cnt.p, psi_S,
                   (const double*)psi_part.p, psi.p);
        launch_pdl(k_fo_sub, (m + 31) / 32, 256, 0, st, (const double*)Wst.p, m, (const int*)cnt.p,
                   (const double*)psi.p, w.p);
      }
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
  bool device_loop = !(hl && hl[0] == '1') && eps > target && o.max_it > 0;
  if (device_loop) {
    DBuf<IterCtl> dctl;
    DBuf<double> dtrace;
    const int tcap = tr && tr->eps ? std::min(tr->cap, o.max_it + 1) : 1;
    dctl.alloc(1);
    dtrace.alloc(std::max(1, tcap));
    IterCtl h0{0, FETIGPU_MAX_ITER, 0, tcap, o.max_it, 0, eps0, target};
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
            launch_pdl(k_iter_control, 1, 1, 0, st, (const Scal*)sc.p, dctl.p, dtrace.p, hcond);
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
      if (it >= o.max_it) { status = FETIGPU_MAX_ITER; break; }
      CK(cudaGraphLaunch(exec, st));
      CK(cudaStreamSynchronize(st));
      if (hs->breakdown != 0.0) { status = FETIGPU_BREAKDOWN; break; }
      ++fapp;
      eps = metric(*hs);
      ++it;
      push(eps, 1);
    }
  }
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
      size_t freeb = dev_free_bytes(), total = 0, fr0 = 0;
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
      ch.w->cached = ch.q->cached = ch.psi->cached = true;
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
    s->reserved_ = 0;
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
    p.alloc(n); r.alloc(1); status.alloc(1); ctl.alloc(4); gx.alloc((size_t)n + 64);
    status.zero(st);
    CK(cudaMemcpyAsync(A.p, a, (size_t)n * n * 8, cudaMemcpyHostToDevice, st));
    k_mirror_lower<<<grid_for((long long)n * n), kThreads, 0, st>>>(A.p, n);
    launch_pivchol(A.p, n, tol, p.p, r.p, status.p, ctl.p, gx.p, st);
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
    cublasHandle_t h;
    CB(cublasCreate(&h));
    std::unique_ptr<cublasContext, decltype(&cublasDestroy)> h_guard(h, cublasDestroy);
    CB(cublasSetStream(h, st));
    DBuf<double> L, Linv, W, Wsel, O;
    DBuf<int> p;
    L.alloc((size_t)n * n); Linv.alloc((size_t)rank * rank);
    W.alloc((size_t)rows * n); Wsel.alloc((size_t)rows * rank); O.alloc((size_t)rows * rank);
    p.alloc(n);
    CK(cudaMemcpyAsync(L.p, lower, (size_t)n * n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(W.p, w, (size_t)rows * n * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p.p, perm, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    // L~^{-1} by a triangular solve on the identity, W_sel = W N^T[:, :rank],
    // out = W_sel L~^{-T}: the solver's compression (Alg. 1 lines 10-11)
    k_identity<<<grid_for((long long)rank * rank), kThreads, 0, st>>>(Linv.p, rank);
    const double one = 1.0;
    CB(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, rank, rank, &one,
                   L.p, n, Linv.p, rank));
    k_gather_cols<<<dim3(grid_for(rows), rank), kThreads, 0, st>>>(W.p, rows, p.p, rank, Wsel.p);
    CB(cublasDtrmm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, rows, rank, &one,
                   Linv.p, rank, Wsel.p, rows, O.p, rows));
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
          if (c.su.method == FETIGPU_TFETI)
            k_sym_gemv_scatter<3, false><<<c.su.Ns, 256, c.sym_smem, c.st>>>(
                c.d_sym.p, c.d_symtiles.p, c.d_oprows.p, c.d_opcoef_apply.p, xc, yc, nullptr, nullptr);
          else
            k_sym_gemv_scatter<1, true><<<c.su.Ns, 256, c.sym_smem, c.st>>>(
                c.d_sym.p, c.d_symtiles.p, c.d_oprows.p, c.d_opcoef_apply.p, xc, nullptr, c.d_vbuf.p, c.d_voff.p,
                c.d_dp.p, c.d_abc.p, c.d_tbuf.p);
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
