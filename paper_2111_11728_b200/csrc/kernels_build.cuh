// kernels_build.cuh -- device build of the explicit local operators.
//
// K1+K2: SIMP element moduli + Q4 assembly fused into the
// leaves of a nested-dissection Schur tree; every tree node is one dense
// frontal matrix whose interior/separator DOFs are eliminated by a batched
// partial Cholesky, leaving the Schur complement on the node's perimeter.
// The root's Schur complement is S = K_bb - K_bi K_ii^{-1} K_ib on the module
// perimeter.  This replaces the reference's per-subdomain sparse Cholesky
// (SparseCholesky/SimplicialLLT, linalg.cpp:64-81) as the source of every
// local operator: T-FETI K^+ restricted to the interface, FETI-DP K_rr^{-1},
// K_rr^{-1} K_rc and Kbar_cc^s, and the Dirichlet preconditioner (SURVEY.md
// Appendix B identities).
//
// K3: per-slot frontal matrices [[S[src,src], E],[E^T, 0]] assembled from S
// and eliminated by the same batched kernels; the trailing blocks are the
// dense F_s, A_bc, Kbar_cc^s or S~_s.
#pragma once

#include "common.cuh"

namespace fg {

__constant__ double c_kunit[64];   // unit-modulus Q4 stiffness (col-major)
constexpr int kLeafElems = 64;     // element moduli staged per pass in a leaf

// Unblocked right-looking partial Cholesky of a column-major matrix in
// shared memory: eliminates the first ne of nf DOFs (lower triangle).
__device__ void eliminate_smem(double* F, int nf, int ne, int ld, int* status, int code) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = 0; k < ne; ++k) {
    double* ck = F + (size_t)k * ld;
    if (tid == 0) {
      double d = ck[k];
      if (!(d > 0.0)) {
        atomicExch(status, code);
        d = 1.0;
      }
      ck[k] = sqrt(d);
    }
    __syncthreads();
    const double l = ck[k];
    for (int i = k + 1 + tid; i < nf; i += nt) ck[i] = ck[i] / l;
    __syncthreads();
    const int m = nf - k - 1;
    // lower triangle of the trailing block (column jj holds rows jj..m-1),
    // folded into a rectangle: column p is paired with column m-1-p (m+1
    // entries per pair), an odd m leaves the middle column alone.  Each thread
    // walks its (p, q) positions incrementally: one division per pivot.
    const int W = m + 1, P = m / 2;
    const int tot = P * W + ((m & 1) ? P + 1 : 0);
    int p = tid / W, q = tid - p * W;
    const int sp = nt / W, sq = nt - sp * W;
    for (int idx = tid; idx < tot; idx += nt) {
      int jj, ii;
      if (p < P) {
        if (q < m - p) { jj = p; ii = p + q; }
        else { jj = m - 1 - p; ii = jj + (q - (m - p)); }
      } else {
        jj = P; ii = P + q;
      }
      F[(size_t)(k + 1 + jj) * ld + k + 1 + ii] -= ck[k + 1 + ii] * ck[k + 1 + jj];
      p += sp; q += sq;
      if (q >= W) { q -= W; ++p; }
    }
    __syncthreads();
  }
}

// Same elimination, trailing update walked per column instead of per entry:
// a work item is a folded column pair (p, m-1-p) (or the middle column) cut
// into S contiguous segments, so the inner loop is a plain column run
// (LDS c_i, LDS F, DFMA, STS) with c_j in a register and no per-entry index
// arithmetic.  Every entry still receives F_ij - c_i c_j once per pivot in
// pivot order, so results are bit-identical to eliminate_smem.  Lanes of a
// warp sit in different columns: an even ld (ld + 1 odd) keeps them on
// distinct shared-memory banks.
__device__ __forceinline__ void pivot_sqrt(double* akk, int* status, int code) {
  double d = *akk;
  if (!(d > 0.0)) {
    atomicExch(status, code);
    d = 1.0;
  }
  *akk = sqrt(d);
}

// Column c of a lower-triangular frontal, from its diagonal down: full
// column-major storage (leading dimension ld), or packed (PK: the columns'
// lower parts back to back, ld = nf -- half the shared memory, so twice the
// resident CTAs for the ND small levels).
template <bool PK>
__device__ __forceinline__ double* diag_ptr(double* F, int c, int ld) {
  return PK ? F + ((size_t)c * ld - ((size_t)c * (c - 1)) / 2) : F + (size_t)c * ld + c;
}

template <bool PK>
__device__ void eliminate_smem_cols(double* F, int nf, int ne, int ld, int* status, int code) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (ne > 0 && tid == 0) pivot_sqrt(diag_ptr<PK>(F, 0, ld), status, code);
  __syncthreads();
  for (int k = 0; k < ne; ++k) {
    double* dk = diag_ptr<PK>(F, k, ld);      // dk[i - k] = A[i][k]
    const double l = dk[0];
    for (int i = k + 1 + tid; i < nf; i += nt) dk[i - k] = dk[i - k] / l;
    __syncthreads();
    const int m = nf - k - 1;
    const int P = m / 2, npairs = P + (m & 1);
    const int S = npairs > 0 ? max(1, nt / npairs) : 1;
    const double* cc = dk + 1;                // trailing part of the pivot column
    // thread 0 owns work item 0, whose first entry is the next pivot
    // A[k+1][k+1]: it takes the square root right after its own updates, so
    // one barrier per pivot is saved
    for (int w = tid; w < npairs * S; w += nt) {
      const int p = w % npairs, s = w / npairs;
      const int len = p < P ? m + 1 : m - p;
      const int L = (len + S - 1) / S;
      const int q0 = s * L, q1 = min(len, q0 + L);
      // entries q < m - p: column p, rows p + q; then column m-1-p, rows
      // (m-1-p) + (q - (m-p)) (trailing coordinates).  One loop with a pointer
      // switch, so lanes whose segments straddle the fold do not serialise
      // two loops.
      const int split = m - p;
      int jj = q0 < split ? p : m - 1 - p;
      int sh = q0 < split ? 0 : split;
      double cj = cc[jj];
      double* col = diag_ptr<PK>(F, k + 1 + jj, ld) - sh;
      const double* ci = cc + jj - sh;
      for (int q = q0; q < q1; ++q) {
        if (q == split) {
          jj = m - 1 - p;
          cj = cc[jj];
          col = diag_ptr<PK>(F, k + 1 + jj, ld) - split;
          ci = cc + jj - split;
        }
        col[q] = fma(-ci[q], cj, col[q]);
      }
    }
    if (tid == 0 && k + 1 < ne) pivot_sqrt(diag_ptr<PK>(F, k + 1, ld), status, code);
    __syncthreads();
  }
}

// ---------------------------------------------------------------- ND tree --
struct NdArgs {
  const NdDev* nodes;
  const int* level_nodes;
  const long long* hbase;     // per height: offset of the height block in ws
  const long long* hstride;   // per height: doubles per design
  double* ws;
  const int* elem_ids;
  const int* emap;
  const int* cmaps;
  const double* dens;         // all designs
  int n;
  int d0;                     // first design of this chunk
  double E0, Emin, p;
  double* factors;            // nullable: per design [nf x ne] blocks
  long long fstride;
  int* status;
};

template <bool PK>
__device__ __forceinline__ void nd_assemble(const NdArgs& a, const NdDev& nd, int dl, double* F,
                                            int ld) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (nd.leaf) {
    const double* rho = a.dens + (size_t)(a.d0 + dl) * a.n * a.n;
    // simp_modulus (fem.cpp:19-24), one pow per element (not per thread)
    __shared__ double Es[kLeafElems];
    if (nd.elem_cnt <= kLeafElems) {
      for (int e = tid; e < nd.elem_cnt; e += nt)
        Es[e] = a.Emin + pow(rho[a.elem_ids[nd.elem_off + e]], a.p) * (a.E0 - a.Emin);
      // wavefront rounds t = lx + 2 ly over the leaf's w x h elements (ey-major):
      // elements of one round share no node, and every earlier neighbour of
      // an element in ey-major order lies in an earlier round, so each entry
      // still receives its element contributions in element order
      const int e0id = a.elem_ids[nd.elem_off], eLid = a.elem_ids[nd.elem_off + nd.elem_cnt - 1];
      const int w = eLid % a.n - e0id % a.n + 1, h = eLid / a.n - e0id / a.n + 1;
      __syncthreads();
      for (int t = 0; t < w + 2 * h - 2; ++t) {
        const int ly0 = max(0, (t - w + 2) / 2), ly1 = min(h - 1, t / 2);
        for (int idx = tid; idx < (ly1 - ly0 + 1) * 64; idx += nt) {
          const int ly = ly0 + (idx >> 6), lx = t - 2 * ly;
          const int e = ly * w + lx;
          const double E = Es[e];
          const int* em = a.emap + (size_t)(nd.elem_off + e) * 8;
          const int r = idx & 7, c = (idx >> 3) & 7;
          const int pr = em[r], pc = em[c];
          if (pr >= pc) diag_ptr<PK>(F, pc, ld)[pr - pc] += E * c_kunit[c * 8 + r];
        }
        __syncthreads();
      }
    } else {
    for (int e0 = 0; e0 < nd.elem_cnt; e0 += kLeafElems) {
    const int ecnt = min(kLeafElems, nd.elem_cnt - e0);
    __syncthreads();
    for (int e = tid; e < ecnt; e += nt)
      Es[e] = a.Emin + pow(rho[a.elem_ids[nd.elem_off + e0 + e]], a.p) * (a.E0 - a.Emin);
    __syncthreads();
    for (int e = e0; e < e0 + ecnt; ++e) {
      const double E = Es[e - e0];
      const int* em = a.emap + (size_t)(nd.elem_off + e) * 8;
      for (int idx = tid; idx < 64; idx += nt) {
        const int r = idx & 7, c = idx >> 3;
        const int pr = em[r], pc = em[c];
        if (pr >= pc) diag_ptr<PK>(F, pc, ld)[pr - pc] += E * c_kunit[c * 8 + r];
      }
      __syncthreads();
    }
    }
    }
  } else {
    for (int c = 0; c < 2; ++c) {
      const NdDev ch = a.nodes[nd.child[c]];
      const double* S = a.ws + a.hbase[ch.height] + (long long)dl * a.hstride[ch.height] + ch.off;
      const int nbc = ch.nf - ch.ne;
      const int* cm = a.cmaps + nd.cmap_off[c];
      // U independent (child entry, target) pairs per thread in flight: the
      // targets of one child are distinct, and each target still receives
      // zero + child 0 + child 1 in that order
      constexpr int U = 4;
      const int tot = nbc * nbc;
      for (int base = tid; base < tot; base += U * nt) {
        double v[U], f[U];
        int pos[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int idx = base + u * nt;
          pos[u] = -1;
          v[u] = 0.0;
          if (idx < tot) {
            const int j = idx / nbc, i = idx - j * nbc;
            if (i >= j) {
              v[u] = S[(size_t)(ch.ne + j) * ch.nf + ch.ne + i];
              int pr = cm[i], pc = cm[j];
              if (pr < pc) { const int t = pr; pr = pc; pc = t; }
              pos[u] = (int)(diag_ptr<PK>(F, pc, ld) - F) + pr - pc;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) f[u] = pos[u] >= 0 ? F[pos[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (pos[u] >= 0) F[pos[u]] = f[u] + v[u];
      }
      __syncthreads();
    }
  }
}

// small tree nodes: assemble + eliminate in shared memory (packed lower
// triangle, nf (nf + 1) / 2 doubles), one CTA per (node, design)
__global__ void __launch_bounds__(kThreads) k_nd_small(NdArgs a) {
  extern __shared__ double F[];
  const int t = a.level_nodes[blockIdx.x];
  const int dl = blockIdx.y;
  const NdDev nd = a.nodes[t];
  const int nf = nd.nf;
  for (int i = threadIdx.x; i < nf * (nf + 1) / 2; i += blockDim.x) F[i] = 0.0;
  __syncthreads();
  nd_assemble<true>(a, nd, dl, F, nf);
  eliminate_smem_cols<true>(F, nf, nd.ne, nf, a.status, kNotSPD);
  // the parent (nd_assemble) and k_nd_extract_root read only the lower
  // triangle of the trailing (perimeter) block: write just that
  double* out = a.ws + a.hbase[nd.height] + (long long)dl * a.hstride[nd.height] + nd.off;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = nd.ne + warp; j < nf; j += nw) {
    const double* cj = diag_ptr<true>(F, j, nf);
    for (int i = j + lane; i < nf; i += 32) out[(size_t)j * nf + i] = cj[i - j];
  }
  if (a.factors) {   // first ne columns, full height (zeros above the diagonal)
    double* fo = a.factors + (size_t)(a.d0 + dl) * a.fstride + nd.foff;
    for (int j = warp; j < nd.ne; j += nw) {
      const double* cj = diag_ptr<true>(F, j, nf);
      for (int i = lane; i < nf; i += 32) fo[(size_t)j * nf + i] = i >= j ? cj[i - j] : 0.0;
    }
  }
}

// large tree nodes: assemble into the global frontal (eliminated afterwards)
__global__ void __launch_bounds__(kThreads) k_nd_assemble(NdArgs a) {
  const int t = a.level_nodes[blockIdx.x];
  const int dl = blockIdx.y;
  const NdDev nd = a.nodes[t];
  const int nf = nd.nf;
  double* F = a.ws + a.hbase[nd.height] + (long long)dl * a.hstride[nd.height] + nd.off;
  for (long long i = threadIdx.x; i < (long long)nf * nf; i += blockDim.x) F[i] = 0.0;
  __syncthreads();
  nd_assemble<false>(a, nd, dl, F, nf);
}

__global__ void k_nd_copy_factors(NdArgs a) {
  const int t = a.level_nodes[blockIdx.x];
  const int dl = blockIdx.y;
  const NdDev nd = a.nodes[t];
  const double* F = a.ws + a.hbase[nd.height] + (long long)dl * a.hstride[nd.height] + nd.off;
  double* fo = a.factors + (size_t)(a.d0 + dl) * a.fstride + nd.foff;
  for (long long i = threadIdx.x; i < (long long)nd.nf * nd.ne; i += blockDim.x) fo[i] = F[i];
}

// Root Schur complement -> dense symmetric S (nb x nb, column-major) per design.
__global__ void k_nd_extract_root(const NdDev* nodes, int root, const long long* hbase,
                                  const long long* hstride, const double* ws, double* S, int nb,
                                  int d0) {
  const NdDev nd = nodes[root];
  const int dl = blockIdx.y;
  const double* F = ws + hbase[nd.height] + (long long)dl * hstride[nd.height] + nd.off;
  double* out = S + (size_t)(d0 + dl) * nb * nb;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nb * nb; idx += gridDim.x * blockDim.x) {
    const int j = idx / nb, i = idx - j * nb;
    const int r = i > j ? i : j, c = i > j ? j : i;
    out[idx] = F[(size_t)(nd.ne + c) * nd.nf + nd.ne + r];
  }
}

// -------------------------------------------------- blocked elimination --
// Right-looking blocked partial Cholesky in global memory, one CTA per
// frontal: panel factor in smem, row-wise triangular solve of the panel,
// 64x64-tiled rank-kNB update of the lower trailing matrix (4x4 register
// tiles on the DFMA pipe; a DMMA variant measured ~15% slower here because
// the update is bound by the global read-modify-write of the tiles).
__global__ void __launch_bounds__(kThreads) k_front_elim_large(const FrontDesc* fds, double* base,
                                                               int* status) {
  const FrontDesc f = fds[blockIdx.x];
  double* A = base + f.off;
  const int nf = f.nf, ne = f.ne, ld = f.ld;
  __shared__ double D[kNB * (kNB + 1)];
  __shared__ double LiT[kNB * kTile];
  __shared__ double LjT[kNB * kTile];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  for (int k0 = 0; k0 < ne; k0 += kNB) {
    const int kb = min(kNB, ne - k0);
    const int k1 = k0 + kb;
    for (int idx = tid; idx < kb * kb; idx += kThreads) {
      const int j = idx / kb, i = idx - j * kb;
      if (i >= j) D[j * (kNB + 1) + i] = A[(size_t)(k0 + j) * ld + k0 + i];
    }
    __syncthreads();
    eliminate_smem(D, kb, kb, kNB + 1, status, f.code);
    for (int idx = tid; idx < kb * kb; idx += kThreads) {
      const int j = idx / kb, i = idx - j * kb;
      if (i >= j) A[(size_t)(k0 + j) * ld + k0 + i] = D[j * (kNB + 1) + i];
    }
    // panel: X D^T = A[r, k0:k1] for rows below the block
    for (int r = k1 + tid; r < nf; r += kThreads) {
      double x[kNB];
#pragma unroll
      for (int c = 0; c < kNB; ++c)
        if (c < kb) x[c] = A[(size_t)(k0 + c) * ld + r];
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        if (c < kb) {
          double v = x[c];
#pragma unroll
          for (int c2 = 0; c2 < c; ++c2) v -= x[c2] * D[c2 * (kNB + 1) + c];
          x[c] = v / D[c * (kNB + 1) + c];
          A[(size_t)(k0 + c) * ld + r] = x[c];
        }
      }
    }
    __syncthreads();
    const int mt = nf - k1;
    const int nt = (mt + kTile - 1) / kTile;
    for (int tj = 0; tj < nt; ++tj) {
      for (int idx = tid; idx < kb * kTile; idx += kThreads) {
        const int c = idx / kTile, r = idx - c * kTile;
        const int row = tj * kTile + r;
        LjT[c * kTile + r] = row < mt ? A[(size_t)(k0 + c) * ld + k1 + row] : 0.0;
      }
      for (int ti = tj; ti < nt; ++ti) {
        for (int idx = tid; idx < kb * kTile; idx += kThreads) {
          const int c = idx / kTile, r = idx - c * kTile;
          const int row = ti * kTile + r;
          LiT[c * kTile + r] = row < mt ? A[(size_t)(k0 + c) * ld + k1 + row] : 0.0;
        }
        __syncthreads();
        double acc[4][4] = {};
        for (int c = 0; c < kb; ++c) {
          double li[4], lj[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            li[q] = LiT[c * kTile + tx + 16 * q];
            lj[q] = LjT[c * kTile + ty + 16 * q];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int w = 0; w < 4; ++w) acc[q][w] = fma(li[q], lj[w], acc[q][w]);
        }
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int cj = tj * kTile + ty + 16 * w;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int ri = ti * kTile + tx + 16 * q;
            if (ri < mt && cj < mt && ri >= cj) A[(size_t)(k1 + cj) * ld + k1 + ri] -= acc[q][w];
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// ------------------------------- batched blocked partial Cholesky (BPC) --
// The same right-looking algorithm as k_front_elim_large, but every panel
// step is three launches over ALL frontals of a batch, so each phase gets a
// full GPU of CTAs: (1) factor the kb x kb diagonal block (1 CTA / frontal),
// (2) triangular-solve the panel rows below it (CTAs over row blocks),
// (3) rank-kb update of the lower trailing matrix, one 64x64 tile per CTA on
// FP64 tensor cores (mma.sync.m8n8k4.f64, 8 warps as 2 x 4 warp tiles).
__device__ __forceinline__ void dmma_884b(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
constexpr int kBpcPad = kTile + 4;
// panel width of the batched elimination: 64 columns halve the number of
// read-modify-write passes over the trailing matrices (the update is memory
// bound: 64 x 64 tile, 2 * 64 * 64 * kBpcNB flop per 3 * 32 KB moved)
constexpr int kBpcNB = 64;
constexpr size_t kBpcUpdateSmem = (size_t)2 * kBpcNB * kBpcPad * sizeof(double);

__global__ void __launch_bounds__(kThreads) k_bpc_diag(const FrontDesc* fds, double* base, int k0,
                                                       int* status) {
  const FrontDesc f = fds[blockIdx.x];
  if (k0 >= f.ne) return;
  __shared__ double D[kBpcNB * (kBpcNB + 1)];
  double* A = base + f.off;
  const int kb = min(kBpcNB, f.ne - k0), ld = f.ld;
  for (int idx = threadIdx.x; idx < kb * kb; idx += kThreads) {  // cp.async: all copies in flight
    const int j = idx / kb, i = idx - j * kb;
    if (i >= j) cp_async8(D + j * (kBpcNB + 1) + i, A + (size_t)(k0 + j) * ld + k0 + i, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  eliminate_smem(D, kb, kb, kBpcNB + 1, status, f.code);
  for (int idx = threadIdx.x; idx < kb * kb; idx += kThreads) {
    const int j = idx / kb, i = idx - j * kb;
    if (i >= j) A[(size_t)(k0 + j) * ld + k0 + i] = D[j * (kBpcNB + 1) + i];
  }
}

__global__ void __launch_bounds__(kThreads) k_bpc_trsm(const FrontDesc* fds, double* base, int k0) {
  const FrontDesc f = fds[blockIdx.y];
  if (k0 >= f.ne) return;
  const int kb = min(kBpcNB, f.ne - k0), k1 = k0 + kb, ld = f.ld;
  const int r = k1 + blockIdx.x * kThreads + threadIdx.x;
  if (k1 + blockIdx.x * kThreads >= f.nf) return;
  __shared__ double D[kBpcNB * (kBpcNB + 1)];
  double* A = base + f.off;
  for (int idx = threadIdx.x; idx < kb * kb; idx += kThreads) {  // cp.async: all copies in flight
    const int j = idx / kb, i = idx - j * kb;
    if (i >= j) cp_async8(D + j * (kBpcNB + 1) + i, A + (size_t)(k0 + j) * ld + k0 + i, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (r >= f.nf) return;
  // row r of the panel: x L^T = a, in two 32-column halves so at most 64
  // values are live (first half solved, second half updated from it, solved)
  constexpr int H = kBpcNB / 2;
  double lo[H], hi[H];
#pragma unroll
  for (int c = 0; c < H; ++c) lo[c] = c < kb ? A[(size_t)(k0 + c) * ld + r] : 0.0;
#pragma unroll
  for (int c = 0; c < H; ++c) {
    if (c < kb) {
      double v = lo[c];
#pragma unroll
      for (int c2 = 0; c2 < c; ++c2) v -= lo[c2] * D[c2 * (kBpcNB + 1) + c];
      lo[c] = v / D[c * (kBpcNB + 1) + c];
      A[(size_t)(k0 + c) * ld + r] = lo[c];
    }
  }
  if (kb <= H) return;
#pragma unroll
  for (int c = 0; c < H; ++c) {
    double v = H + c < kb ? A[(size_t)(k0 + H + c) * ld + r] : 0.0;
#pragma unroll
    for (int c2 = 0; c2 < H; ++c2) v -= lo[c2] * D[c2 * (kBpcNB + 1) + H + c];
    hi[c] = v;
  }
#pragma unroll
  for (int c = 0; c < H; ++c) {
    if (H + c < kb) {
      double v = hi[c];
#pragma unroll
      for (int c2 = 0; c2 < c; ++c2) v -= hi[c2] * D[(H + c2) * (kBpcNB + 1) + H + c];
      hi[c] = v / D[(H + c) * (kBpcNB + 1) + H + c];
      A[(size_t)(k0 + H + c) * ld + r] = hi[c];
    }
  }
}

__global__ void __launch_bounds__(kThreads, 2) k_bpc_update(const FrontDesc* fds, double* base, int k0) {
  const FrontDesc f = fds[blockIdx.y];
  if (k0 >= f.ne) return;
  const int kb = min(kBpcNB, f.ne - k0), k1 = k0 + kb, ld = f.ld;
  const int mt = f.nf - k1;
  const int nt = (mt + kTile - 1) / kTile;
  const int t = blockIdx.x;
  if (t >= nt * (nt + 1) / 2) return;
  int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (ti * (ti + 1) / 2 > t) --ti;
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  const int tj = t - ti * (ti + 1) / 2;
  extern __shared__ double bpc_sm[];
  double* LiT = bpc_sm;                    // kBpcNB x kBpcPad
  double* LjT = bpc_sm + kBpcNB * kBpcPad;
  double* A = base + f.off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 2, wc = warp & 3;
  // panels by cp.async: all 2 x 16 copies per thread in flight at once (a
  // register-staged loop serialises one L2 round trip per iteration)
#pragma unroll 4
  for (int q = 0; q < kBpcNB * kTile / kThreads; ++q) {
    const int idx = tid + q * kThreads;
    const int c = idx / kTile, r = idx - c * kTile;
    const int ri = ti * kTile + r, rj = tj * kTile + r;
    const double* col = A + (size_t)(k0 + c) * ld + k1;
    cp_async8(LiT + c * kBpcPad + r, (c < kb && ri < mt) ? col + ri : A, c < kb && ri < mt);
    cp_async8(LjT + c * kBpcPad + r, (c < kb && rj < mt) ? col + rj : A, c < kb && rj < mt);
  }
  cp_async_commit();
  // the trailing tile this thread updates, loaded while the panels land
  double cpre[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ri = ti * kTile + wr * 32 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int cj = tj * kTile + wc * 16 + j * 8 + 2 * (lane & 3);
      const bool ok0 = ri < mt && cj < mt && ri >= cj, ok1 = ri < mt && cj + 1 < mt && ri >= cj + 1;
      cpre[i][j][0] = ok0 ? A[(size_t)(k1 + cj) * ld + k1 + ri] : 0.0;
      cpre[i][j][1] = ok1 ? A[(size_t)(k1 + cj + 1) * ld + k1 + ri] : 0.0;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int kq = (kb + 3) & ~3;
  for (int k4 = 0; k4 < kq; k4 += 4) {
    double af[4], bf[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = LiT[(k4 + (lane & 3)) * kBpcPad + wr * 32 + i * 8 + (lane >> 2)];
#pragma unroll
    for (int j = 0; j < 2; ++j) bf[j] = LjT[(k4 + (lane & 3)) * kBpcPad + wc * 16 + j * 8 + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma_884b(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ri = ti * kTile + wr * 32 + i * 8 + (lane >> 2);
    if (ri >= mt) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int cj = tj * kTile + wc * 16 + j * 8 + 2 * (lane & 3);
      if (cj < mt && ri >= cj) A[(size_t)(k1 + cj) * ld + k1 + ri] = cpre[i][j][0] - acc[i][j][0];
      if (cj + 1 < mt && ri >= cj + 1) A[(size_t)(k1 + cj + 1) * ld + k1 + ri] = cpre[i][j][1] - acc[i][j][1];
    }
  }
}

// small frontal matrices (slots): load, eliminate in smem, store
__global__ void __launch_bounds__(kThreads) k_front_elim_small(const FrontDesc* fds, double* base,
                                                               int* status) {
  extern __shared__ double F[];
  const FrontDesc f = fds[blockIdx.x];
  double* A = base + f.off;
  const int nf = f.nf;
  for (int idx = threadIdx.x; idx < nf * nf; idx += blockDim.x) {
    const int j = idx / nf, i = idx - j * nf;
    F[idx] = A[(size_t)j * f.ld + i];
  }
  __syncthreads();
  eliminate_smem_cols<false>(F, nf, f.ne, nf, status, f.code);
  for (int idx = threadIdx.x; idx < nf * nf; idx += blockDim.x) {
    const int j = idx / nf, i = idx - j * nf;
    A[(size_t)j * f.ld + i] = F[idx];
  }
}

// ----------------------------------------------------------------- slots --
struct SlotDev {
  long long woff;   // frontal offset in the workspace
  int design, nsrc, ne, next;
  int src_off, ext_off;
};

// frontal = [[S[src,src], E],[E^T, 0]] (lower triangle, column-major, ld = nf)
__global__ void k_slot_assemble(const SlotDev* slots, const int* src_all, const int* ext_all,
                                const double* S, int nb, double* ws) {
  const SlotDev sd = slots[blockIdx.y];
  const int nf = sd.nsrc + sd.next;
  const double* Sd = S + (size_t)sd.design * nb * nb;
  const int* src = src_all + sd.src_off;
  const int* ext = ext_all + sd.ext_off;
  double* F = ws + sd.woff;
  const long long tot = (long long)nf * nf;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / nf), i = (int)(idx - (long long)j * nf);
    double v = 0.0;
    if (i >= j) {
      if (i < sd.nsrc) v = Sd[(size_t)src[j] * nb + src[i]];
      else if (j < sd.nsrc) v = (ext[i - sd.nsrc] == j) ? 1.0 : 0.0;
    }
    F[idx] = v;
  }
}

// T-FETI operator: F_s = -(trailing block); FETI-DP: F_s = -(TT block),
// A_bc = -(T,c block), Kbar_cc^s = (c,c block).  Dirichlet preconditioner:
// S~ = trailing block (sign +1, nc = 0).  Outputs are dense row-major.
__global__ void k_slot_extract(const SlotDev* slots, const double* ws, const long long* mat_off,
                               const int* mat_ld, double* mats, int nc_first, double sign,
                               const long long* abc_off, double* abc, const long long* kcc_off,
                               double* kcc) {
  const SlotDev sd = slots[blockIdx.y];
  const int nf = sd.nsrc + sd.next;
  const double* F = ws + sd.woff;
  // trailing block layout: [c (nc) | T (nt)] after the ne eliminated DOFs
  const int nc = nc_first ? (sd.nsrc - sd.ne) : 0;
  const int base = sd.ne + nc;
  const int nt = nf - base;
  const int ld = mat_ld[blockIdx.y];
  double* M = mats + mat_off[blockIdx.y];
  auto at = [&](int r, int c) {
    const int rr = r > c ? r : c, cc = r > c ? c : r;
    return F[(size_t)cc * nf + rr];
  };
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nt * ld;
       idx += gridDim.x * blockDim.x) {
    const int a = idx / ld, b = idx - a * ld;
    M[(size_t)a * ld + b] = b < nt ? sign * at(base + a, base + b) : 0.0;
  }
  if (nc > 0) {
    double* Ab = abc + abc_off[blockIdx.y];
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nt * nc;
         idx += gridDim.x * blockDim.x) {
      const int a = idx / nc, c = idx - a * nc;
      Ab[idx] = -at(base + a, sd.ne + c);
    }
    double* Kc = kcc + kcc_off[blockIdx.y];
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nc * nc;
         idx += gridDim.x * blockDim.x) {
      const int a = idx / nc, c = idx - a * nc;
      Kc[idx] = at(sd.ne + a, sd.ne + c);
    }
  }
}

// L factor (ne x ne, column-major lower) of an eliminated slot frontal
__global__ void k_slot_factor(const SlotDev* slots, const double* ws, const long long* fac_off,
                              double* fac) {
  const SlotDev sd = slots[blockIdx.y];
  const int nf = sd.nsrc + sd.next, ne = sd.ne;
  const double* F = ws + sd.woff;
  double* L = fac + fac_off[blockIdx.y];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < ne * ne;
       idx += gridDim.x * blockDim.x) {
    const int j = idx / ne, i = idx - j * ne;
    L[idx] = i >= j ? F[(size_t)j * nf + i] : 0.0;
  }
}

// Boundary block K_bb of the assembled stiffness per design (lumped /
// super-lumped preconditioners): entries summed over the <= 2
// elements adjacent to a perimeter node in ascending element order.
__global__ void k_kbb(const double* dens, int n, double E0, double Emin, double p,
                      const int* pnode_elem /* nb/2 x 2 x 2 : (elem, corner) */,
                      const int* perim_dof, int nb, double* Kbb) {
  const int d = blockIdx.y;
  const double* rho = dens + (size_t)d * n * n;
  double* K = Kbb + (size_t)d * nb * nb;
  const int nn = n + 1;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nb * nb;
       idx += gridDim.x * blockDim.x) {
    const int j = idx / nb, i = idx - j * nb;
    const int di = perim_dof[i], dj = perim_dof[j];
    const int ni = di >> 1, nj = dj >> 1;
    double v = 0.0;
    for (int q = 0; q < 2; ++q) {
      const int e = pnode_elem[(i >> 1) * 4 + 2 * q];
      if (e < 0) continue;
      const int ci = pnode_elem[(i >> 1) * 4 + 2 * q + 1];
      const int ex = e % n, ey = e / n;
      const int n0 = ey * nn + ex;
      const int en[4] = {n0, n0 + 1, n0 + nn + 1, n0 + nn};
      int cj = -1;
      for (int a = 0; a < 4; ++a)
        if (en[a] == nj) cj = a;
      if (cj < 0) continue;
      const double E = Emin + pow(rho[e], p) * (E0 - Emin);
      v += E * c_kunit[(2 * cj + (dj & 1)) * 8 + 2 * ci + (di & 1)];
    }
    (void)ni;
    K[idx] = v;
  }
}

// lumped preconditioner block K_TT (or its diagonal) -> dense row-major
__global__ void k_pc_lumped(const int* design, const int* t_off, const int* t_cnt, const int* t_all,
                            const double* Kbb, int nb, const long long* mat_off, const int* mat_ld,
                            double* mats, int diag_only) {
  const int sl = blockIdx.y;
  const int nt = t_cnt[sl], ld = mat_ld[sl];
  const int* T = t_all + t_off[sl];
  const double* K = Kbb + (size_t)design[sl] * nb * nb;
  double* M = mats + mat_off[sl];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nt * ld;
       idx += gridDim.x * blockDim.x) {
    const int a = idx / ld, b = idx - a * ld;
    double v = 0.0;
    if (b < nt && (!diag_only || a == b)) v = K[(size_t)T[b] * nb + T[a]];
    M[(size_t)a * ld + b] = v;
  }
}

}  // namespace fg
