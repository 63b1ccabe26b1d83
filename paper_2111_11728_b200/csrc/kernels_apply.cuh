// kernels_apply.cuh -- per-iteration kernels of the FETI engine.
//
// K4/K7: y = sum_s B_s F_s B_s^T x as ONE kernel per apply:
// each CTA gathers its subdomain's x_s = B_s^T x (signed, weighted for the
// preconditioner) into shared memory, streams the dense row-major F_s from HBM
// once (128-bit streaming loads, one warp per row, warp-shuffle reduction)
// and scatters sign * (F_s x_s)_i to the dual rows.  Every dual row receives
// exactly two contributions (one for Dirichlet rows) into a zeroed output,
// so the atomic scatter is order-independent (0 + a + b == 0 + b + a) and
// the apply is bit-reproducible.
//
// This replaces, per apply and per subdomain, the reference's
// ConstraintSet::apply_BsT -> SemidefiniteCholesky::solve_unchecked ->
// accumulate_Bs chain (decomposition.hpp:98-101, linalg.cpp:206-213).
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "common.cuh"

namespace fg {

// Programmatic dependent launch: a kernel launched with the PDL attribute may
// be scheduled while its predecessor in the stream is still finishing; it
// waits here (griddepcontrol.wait) until the predecessor has completed and its
// writes are visible.  A no-op for ordinary launches.
__device__ __forceinline__ void pdl_wait() {
#if __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// ------------------------------------------------------------ the F-apply --
// KR = max dual rows touching one local DOF (1 FETI-DP, <= 3 T-FETI cross points)
// FETI-DP coarse pre-pass fused into the GEMV CTA (x_s already in smem):
// t_s = A''^T x_s for the subdomain's <= 8 primal DOFs (rsplit slice 0 only).
// Deterministic coarse gather fused into phase 1: every owner subdomain of a
// primal DOF publishes its t entry and counts its arrival; the last owner to
// arrive sums the owners' entries in fixed (ascending subdomain) order -- the
// order of k_coarse_gather -- writes g and resets the counter for the next
// apply.  (Threadfence-reduction pattern: nobody waits.)
struct CoarseGather {
  double* g;            // N_c
  unsigned int* cnt;    // N_c arrival counters, zero between applies
  const int* optr;      // owners of primal DOF i: oidx[optr[i] .. optr[i+1])
  const int* oidx;      // -> tbuf index
  const int* cmap;      // per subdomain: global primal ids
};

__device__ __forceinline__ void fused_dp_t(const DpSub& p, const double* __restrict__ abc,
                                           const double* xs, int ns, double* __restrict__ tbuf,
                                           const CoarseGather* cgp = nullptr) {
  __shared__ double red[8][kThreads / 32];
  double acc[8] = {};
  const double* Ab = abc + p.abc_off;
  for (int j = threadIdx.x; j < ns; j += blockDim.x) {
    const double xj = xs[j];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < p.nc) acc[c] = fma(Ab[(size_t)j * p.nc + c], xj, acc[c]);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double v = warp_sum(acc[c]);
    if (lane == 0) red[c][warp] = v;
  }
  __syncthreads();
  if ((int)threadIdx.x < p.nc) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    tbuf[p.t_off + threadIdx.x] = v;
    if (cgp) {
      const CoarseGather cg = *cgp;
      const int gid = cg.cmap[p.cmap_off + threadIdx.x];
      const int k0 = cg.optr[gid], k1 = cg.optr[gid + 1];
      __threadfence();  // this t entry is visible device-wide before the arrival is counted
      if (atomicAdd(cg.cnt + gid, 1u) + 1u == (unsigned)(k1 - k0)) {
        __threadfence();
        double g = 0.0;
        for (int k = k0; k < k1; ++k) g += __ldcg(tbuf + cg.oidx[k]);
        cg.g[gid] = g;
        cg.cnt[gid] = 0u;
      }
    }
  }
}

// One CTA of the K4/K7 GEMV: subdomain s, column col, row slice zi of nz
// (rows i = warp + 8 zi, + 8 nz, ...).  A row's dot product does not depend on
// the slicing, and every dual row receives its two contributions in either
// order (0 + a + b), so any nz gives bit-identical results.  Shared by the
// kernel below and the persistent solver loop (kernels_persist.cuh); x is
// read through L2 (__ldcg) because the persistent loop writes it in-kernel.
// x_s = B_s^T x into shared memory (ld entries, zero padded): xval(r, e)
// returns the dual-vector value at row r for map entry e (a plain L2 load, or
// a value the persistent loop forms on the fly)
template <int KR, class XV>
__device__ __forceinline__ void gather_xs(const OpSub& d, const int* __restrict__ rows,
                                          const double* __restrict__ coefs, double* xs, XV&& xval) {
  const int* rw = rows + d.map_off;
  const double* cf = coefs + d.map_off;
  for (int j = threadIdx.x; j < d.ld; j += blockDim.x) {
    double acc = 0.0;
    if (j < d.ns) {
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int r = rw[j * KR + k];
        if (r >= 0) acc += cf[j * KR + k] * xval(r, d.map_off + j * KR + k);
      }
    }
    xs[j] = acc;
  }
}

// the row part of the K4/K7 GEMV for one CTA (rows i = warp + 8 zi, + 8 nz,
// ...): v_i = F_s[i,:] x_s, stored (STORE_V) or scattered with the map's signs
template <int KR, bool STORE_V, bool ASM = false>   // ASM: the matrix in shared memory
__device__ __forceinline__ void gemv_rows_cta(int s, int col, int zi, int nz, const double* xs, const OpSub& d,
                                              const double* __restrict__ mats, const int* __restrict__ rows,
                                              const double* __restrict__ coefs, double* y, double* zcols, int ldz,
                                              double* vbuf, const int* __restrict__ voff, int ldy, int zrs) {
  const int* rw = rows + d.map_off;
  const double* cf = coefs + d.map_off;
  const double* A = mats + d.moff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rows are split over nz CTAs when there are few subdomains; each warp
  // streams two of its rows at a time (independent chains, same arithmetic
  // per row as one at a time)
  const int nw = (blockDim.x >> 5) * nz;
  auto emit = [&](int i, double v) {
    if (STORE_V) {
      vbuf[voff[s] + i] = v;
    } else {
      double* yc = y + (size_t)col * ldy;
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int r = rw[i * KR + k];
        if (r >= 0) {
          const double c = cf[i * KR + k] * v;
          atomicAdd(yc + r, c);
          if (zcols) zcols[(size_t)s * ldz + (size_t)r * zrs] = c;
        }
      }
    }
  };
  const int n2 = d.ld >> 1;
  // R rows i, i + nw, ... streamed together: each row keeps its own two
  // lane-strided chains (acc0 even / acc1 odd columns), exactly as one at a time
  auto lda = [&](const double2* p) { return ASM ? *p : __ldcs(p); };
  auto rowblk = [&](int i, auto rc) {
    constexpr int R = decltype(rc)::value;
    const double2* Ar[R];
    double acc0[R], acc1[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      Ar[r] = reinterpret_cast<const double2*>(A + (size_t)(i + r * nw) * d.ld);
      acc0[r] = 0.0;
      acc1[r] = 0.0;
    }
    int j = lane;
    for (; j + 32 < n2; j += 64) {
      double2 a0[R], a1[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        a0[r] = lda(Ar[r] + j);
        a1[r] = lda(Ar[r] + j + 32);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc0[r] = fma(a0[r].x, xs[2 * j], acc0[r]);
        acc1[r] = fma(a0[r].y, xs[2 * j + 1], acc1[r]);
        acc0[r] = fma(a1[r].x, xs[2 * j + 64], acc0[r]);
        acc1[r] = fma(a1[r].y, xs[2 * j + 65], acc1[r]);
      }
    }
    for (; j < n2; j += 32) {
      double2 a0[R];
#pragma unroll
      for (int r = 0; r < R; ++r) a0[r] = lda(Ar[r] + j);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc0[r] = fma(a0[r].x, xs[2 * j], acc0[r]);
        acc1[r] = fma(a0[r].y, xs[2 * j + 1], acc1[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double v = warp_sum(acc0[r] + acc1[r]);
      if (lane == 0) emit(i + r * nw, v);
    }
  };
  int i = warp + (blockDim.x >> 5) * zi;
  for (; i + 3 * nw < d.ns; i += 4 * nw) rowblk(i, std::integral_constant<int, 4>{});
  if (i + nw < d.ns) {
    rowblk(i, std::integral_constant<int, 2>{});
    i += 2 * nw;
  }
  if (i < d.ns) rowblk(i, std::integral_constant<int, 1>{});
}

// One CTA of the K4/K7 GEMV: subdomain s, column col, row slice zi of nz.
// A row's dot product does not depend on the slicing, and every dual row
// receives its two contributions in either order (0 + a + b), so any nz gives
// bit-identical results.  x is read through L2 (__ldcg).
template <int KR, bool STORE_V>
__device__ __forceinline__ void gemv_scatter_cta(
    int s, int col, int zi, int nz, double* xs, const OpSub* __restrict__ subs, const double* __restrict__ mats,
    const int* __restrict__ rows, const double* __restrict__ coefs, const double* x, double* y, double* zcols,
    int ldz, double* vbuf, const int* __restrict__ voff, int ldx, int ldy, int zrs, const DpSub* __restrict__ dps,
    const double* __restrict__ abc, double* tbuf) {
  const OpSub d = subs[s];
  const double* xc = x + (size_t)col * ldx;
  gather_xs<KR>(d, rows, coefs, xs, [&](int r, int) { return __ldcg(xc + r); });
  __syncthreads();
  if (STORE_V && dps && zi == 0) fused_dp_t(dps[s], abc, xs, d.ns, tbuf);
  gemv_rows_cta<KR, STORE_V>(s, col, zi, nz, xs, d, mats, rows, coefs, y, zcols, ldz, vbuf, voff, ldy, zrs);
}

template <int KR, bool STORE_V>
__global__ void __launch_bounds__(kThreads) k_gather_gemv_scatter(
    const OpSub* __restrict__ subs, const double* __restrict__ mats, const int* __restrict__ rows,
    const double* __restrict__ coefs, const double* __restrict__ x, double* __restrict__ y,
    double* __restrict__ zcols, int ldz, double* __restrict__ vbuf, const int* __restrict__ voff,
    int ldx, int ldy, int zrs = 1, const DpSub* __restrict__ dps = nullptr,
    const double* __restrict__ abc = nullptr, double* __restrict__ tbuf = nullptr) {
  pdl_wait();
  extern __shared__ double xs[];
  gemv_scatter_cta<KR, STORE_V>(blockIdx.x, blockIdx.y, blockIdx.z, gridDim.z, xs, subs, mats, rows, coefs, x, y,
                                zcols, ldz, vbuf, voff, ldx, ldy, zrs, dps, abc, tbuf);
}

// ------------------------------------ K4 on symmetric-packed F_s (C4 path) --
// F_s is symmetric: only the lower block-triangle of 32x32 tiles is stored
// (tile (bi,bj), bi >= bj, row-major, zero padded; tiles ordered bi-major), so
// each apply streams ~55% of the full-matrix bytes.  A warp owns tiles
// w, w+8, ...: per tile it loads 32 coalesced 256-byte rows, accumulates the
// transposed (column) part lane-privately and the row part through a
// 31-shuffle transpose-reduce; per-warp partial vectors in shared memory are
// summed in fixed warp order, so the result is deterministic.
struct SymSub {
  long long toff;   // offset of the packed tiles
  int ns, nb;       // DOFs, 32-blocks
  int map_off;
  int pad;
};
constexpr int kSymWarps = 8;

template <int KR, bool STORE_V>
__global__ void __launch_bounds__(256) k_sym_gemv_scatter(
    const SymSub* __restrict__ subs, const double* __restrict__ tiles, const int* __restrict__ rows,
    const double* __restrict__ coefs, const double* __restrict__ x, double* __restrict__ y,
    double* __restrict__ vbuf, const int* __restrict__ voff, const DpSub* __restrict__ dps = nullptr,
    const double* __restrict__ abc = nullptr, double* __restrict__ tbuf = nullptr, int s0 = 0,
    double* __restrict__ zero_y = nullptr, int ny = 0, int nsub = 1, const CoarseGather* cgp = nullptr) {
  pdl_wait();
  extern __shared__ double shm[];
  const int s = s0 + blockIdx.x;   // subdomain (s0: first subdomain of a pipelined chunk)
  const SymSub d = subs[s];
  if (STORE_V && zero_y) {  // FETI-DP: phase 1 never writes y, so its slice is zeroed here for phase 2
    const long long a = (long long)ny * s / nsub, e = (long long)ny * (s + 1) / nsub;
    for (long long i = a + threadIdx.x; i < e; i += blockDim.x) zero_y[i] = 0.0;
  }
  const int npad = d.nb * 32;
  double* xs = shm;                   // npad
  double* part = shm + npad;          // kSymWarps x npad
  const int* rw = rows + d.map_off;
  const double* cf = coefs + d.map_off;
  for (int j = threadIdx.x; j < npad; j += blockDim.x) {
    double acc = 0.0;
    if (j < d.ns) {
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int r = rw[j * KR + k];
        if (r >= 0) acc += cf[j * KR + k] * x[r];
      }
    }
    xs[j] = acc;
  }
  for (int j = threadIdx.x; j < kSymWarps * npad; j += blockDim.x) part[j] = 0.0;
  __syncthreads();
  if (STORE_V && dps) fused_dp_t(dps[s], abc, xs, d.ns, tbuf, cgp);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* pw = part + warp * npad;
  const int ntiles = d.nb * (d.nb + 1) / 2;
  const double* T0 = tiles + d.toff;
  for (int t = warp; t < ntiles; t += kSymWarps) {
    int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int bj = t - bi * (bi + 1) / 2;
    const double* T = T0 + (size_t)t * 1024;
    double f[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) f[r] = __ldcs(T + r * 32 + lane);
    const double xj = xs[bj * 32 + lane];
    double c = 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      c = fma(f[r], xs[bi * 32 + r], c);   // column part: sum_r F[r][lane] x_i[r]
      f[r] *= xj;                          // row part products
    }
    // transpose-reduce: lane l ends with sum over lanes of f[l]
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int q = 0; q < o; ++q) {
        const double keep = hi ? f[q + o] : f[q];
        const double send = hi ? f[q] : f[q + o];
        f[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    pw[bi * 32 + lane] += f[0];
    if (bi != bj) pw[bj * 32 + lane] += c;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d.ns; i += blockDim.x) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kSymWarps; ++w) v += part[w * npad + i];
    if (STORE_V) {
      vbuf[voff[s] + i] = v;
    } else {
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int r = rw[i * KR + k];
        if (r >= 0) atomicAdd(y + r, cf[i * KR + k] * v);
      }
    }
  }
}

// ---- K4 on symmetric-packed F_s, TMA form (the default since round 2) ----
// The same arithmetic per tile, per warp and per subdomain as
// k_sym_gemv_scatter (bit-identical results), but the operator stream is
// moved by the TMA engine and the grid is persistent (CTA b walks subdomains
// s0 + b, s0 + b + G, ...).  Every warp owns a private ring of R 8 KB
// shared-memory slots, each with its own mbarrier, and a cursor over ITS
// stream of tiles (t = warp, warp + 8, ... of each of the CTA's subdomains in
// turn): one cp.async.bulk per tile, and as soon as the warp has drained a
// slot into registers it requests its next unrequested tile into that slot --
// across subdomain boundaries -- so a slot is in flight except for the few
// cycles between arrival and refill, also while the CTA gathers x_s or
// reduces its partials; the first tiles are requested before
// griddepcontrol.wait (the operator does not depend on the predecessor
// kernel).  A slot is filled and drained by one warp only, in order, so the
// barrier phase a warp waits for is always the slot's current or next one.
// A warp of LDG.64 loads keeps its 8 KB in flight only between issue and use
// and measured 6.35 TB/s; a read-only stream of this shape reaches 7.1-7.3
// TB/s on a B200 (tools/read_peak.cu).
__device__ __forceinline__ uint32_t smem_addr32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_addr32(b)),
      "r"(parity)
      : "memory");
}
// one 1D bulk copy global -> shared, completing `bytes` on the mbarrier; L2 evict-first (read once)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_addr32(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr32(bar)), "l"(pol)
      : "memory");
}
// the same without a cache hint (data that should stay in L2: A'' is read again by phase 2)
__device__ __forceinline__ void tma_load_1d_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr32(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr32(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr32(bar))
               : "memory");
}
// FETI-DP coarse pre-pass streamed through the rings (flag 8): A''_s (n_s x n_c
// row-major, n_c in {2, 4, 8}) is cut into 8 KB chunks, chunk w appended to
// warp w's tile stream of the subdomain; lane l of the warp sums column
// l % n_c over the chunk's rows l / n_c, + 32 / n_c, ...  Chunks of A''_s:
__device__ __forceinline__ int dp_chunks(const DpSub& p, int ns) {
  const bool ok = (p.nc == 2 || p.nc == 4 || p.nc == 8) && (p.abc_off & 1) == 0;
  const int n = (ns * p.nc + 1023) >> 10;
  return ok && n <= kSymWarps ? n : 0;
}
constexpr int kSymRingMax = 2;                        // slots per warp (the 8 x 2 barriers share one 128-byte line)
constexpr int kSymTileBytes = 32 * 32 * 8;
__host__ __device__ constexpr size_t sym_tma_smem(int R, int npad) {
  return (size_t)R * kSymWarps * kSymTileBytes + 128 + (size_t)npad * (2 + kSymWarps) * 8;
}
// L2 prefetch of [p, p + bytes) (16-byte granules inside the range)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, size_t bytes) {
  const uintptr_t a = ((uintptr_t)p + 15) & ~(uintptr_t)15, e = ((uintptr_t)p + bytes) & ~(uintptr_t)15;
  if (e > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const void*)a), "r"((uint32_t)(e - a))
                 : "memory");
}

template <int KR, bool STORE_V>
__global__ void __launch_bounds__(256, 2) k_sym_gemv_tma(
    const SymSub* __restrict__ subs, const double* __restrict__ tiles, const int* __restrict__ rows,
    const double* __restrict__ coefs, const double* __restrict__ x, double* __restrict__ y,
    double* __restrict__ vbuf, const int* __restrict__ voff, const DpSub* __restrict__ dps,
    const double* __restrict__ abc, double* __restrict__ tbuf, int s0, int s1, double* __restrict__ zero_y, int ny,
    int nsub, const CoarseGather* cgp, int R, int npad_max, int flags, const int* wait_flag = nullptr,
    const int* __restrict__ sub_need = nullptr) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const size_t ring_bytes = (size_t)R * kSymWarps * kSymTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw + ring_bytes);     // 8 R barriers
  double* xs_buf = reinterpret_cast<double*>(smraw + ring_bytes + 128); // 2 x npad (double-buffered x_s)
  double* part = xs_buf + 2 * npad_max;                                 // kSymWarps x npad
  const int G = gridDim.x, sfirst = s0 + blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* wring = reinterpret_cast<double*>(smraw) + (size_t)warp * R * 1024;   // this warp's R slots
  uint64_t* wfull = full + warp * R;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  // Host-buffer apply (fetigpu_apply_F on host pointers): x arrives by row
  // prefix chunks on a copy stream while this kernel already runs; after each
  // chunk the stream stores a larger value in *wait_flag, and subdomain s may
  // gather once the flag has reached sub_need[s].  x is then read through L2
  // (a line cached in L1 before its chunk landed would be stale).
  auto flag_now = [&]() {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(wait_flag) : "memory");
    return v;
  };
  auto ldx = [&](int r) { return wait_flag ? __ldcg(x + r) : x[r]; };
  // this warp's request cursor: tile ct of subdomain cs (cnt tiles at ctoff)
  int cs = sfirst, ct = warp, cnt = 0, nreq = 0;
  long long ctoff = 0, caoff = 0;
  int cabytes = 0;   // > 0: this warp's A'' chunk of subdomain cs is still to be requested (after its tiles)
  const bool stream_a = STORE_V && dps && (flags & 8);
  auto cursor_load = [&]() {
    if (cs < s1) {
      const SymSub q = subs[cs];
      cnt = q.nb * (q.nb + 1) / 2;
      ctoff = q.toff;
      cabytes = 0;
      if (stream_a) {
        const DpSub pq = dps[cs];
        if (warp < dp_chunks(pq, q.ns)) {
          caoff = pq.abc_off + (long long)warp * 1024;
          cabytes = min(1024, q.ns * pq.nc - warp * 1024) * 8;
        }
      }
    }
  };
  auto request_next = [&]() {   // warp-uniform; lane 0 issues
    for (;;) {
      if (cs >= s1) return;
      const int slot = nreq % R;
      if (cabytes > 0) {   // the subdomain's A'' chunk first: it lands while the CTA is between tile loops
        if (lane == 0) tma_load_1d_plain(wring + (size_t)slot * 1024, abc + caoff, (uint32_t)cabytes, wfull + slot);
        ++nreq;
        cabytes = 0;
        return;
      }
      if (ct < cnt) {
        if (lane == 0)
          tma_load_1d(wring + (size_t)slot * 1024, tiles + ctoff + (size_t)ct * 1024, kSymTileBytes,
                      wfull + slot, pol);
        ++nreq;
        ct += kSymWarps;
        return;
      }
      cs += G;
      ct = warp;
      cursor_load();
    }
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < R * kSymWarps; ++i) mbar_init(full + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cursor_load();
  for (int i = 0; i < R; ++i) request_next();
  pdl_wait();
  __shared__ double tpart[kSymWarps][8];   // per-chunk partials of t_s = A''^T x_s
  int ncons = 0;   // tiles (and A'' chunks) this warp has drained
  // x_s of the CTA's NEXT subdomain is gathered inside the tile loop (KR = 1):
  // chain c covers local DOFs j = 256 c + 32 warp + lane in three of the
  // warp's iterations -- map entry, then x[row], then the store -- each load
  // consumed one tile later, so its latency hides behind the tile arithmetic
  bool have_xs = false;   // the current subdomain's x_s is already in its buffer
  // the warp partials are zero between subdomains: zeroed once here, and every entry again by the thread
  // that reads it in the final reduction (no zeroing pass and one barrier less per subdomain)
  for (int j = threadIdx.x; j < kSymWarps * npad_max; j += blockDim.x) part[j] = 0.0;
  int xsel = 0;
  for (int s = sfirst; s < s1; s += G) {
    const SymSub d = subs[s];
    double* xs = xs_buf + xsel * npad_max;
    double* xs_next = xs_buf + (xsel ^ 1) * npad_max;
    if (STORE_V && zero_y) {  // FETI-DP: phase 1 never writes y, so its slice is zeroed here for phase 2
      const long long a = (long long)ny * s / nsub, e = (long long)ny * (s + 1) / nsub;
      for (long long i = a + threadIdx.x; i < e; i += blockDim.x) zero_y[i] = 0.0;
    }
    const int npad = d.nb * 32;
    const int* rw = rows + d.map_off;
    const double* cf = coefs + d.map_off;
    if (!have_xs) {
      if (wait_flag) {
        const int need = sub_need[s];
        // (bounded: the chunks are queued on the copy stream before this kernel is launched and arrive
        // within ~0.1 ms; a wait of seconds means a broken stream order -- trap rather than hang the device)
        for (long long spin = 0; flag_now() < need; ++spin) {
          __nanosleep(200);
          if (spin > 20000000) __trap();
        }
      }
      for (int j = threadIdx.x; j < npad; j += blockDim.x) {
        double acc = 0.0;
        if (j < d.ns) {
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const int r = rw[j * KR + k];
            if (r >= 0) acc += cf[j * KR + k] * ldx(r);
          }
        }
        xs[j] = acc;
      }
    }
    // the next subdomain: its A'' rows into L2 now, its x_s during the tile loop
    const int sn = s + G;
    SymSub dn = d;
    bool pre = false;
    int nchain = 0;
    if (sn < s1) {
      dn = subs[sn];
      nchain = (dn.nb * 32 + 255) / 256;
      pre = KR == 1 && (flags & 1) && (d.nb * (d.nb + 1) / 2) / kSymWarps >= 3 * nchain;
      // (per thread: a thread that finds the next subdomain's rows not landed yet gathers ITS entries
      // j = tid, tid + 256, ... in the prologue instead -- the same entries its chains would cover)
      if (pre && wait_flag) pre = flag_now() >= sub_need[sn];
      if (STORE_V && dps && (flags & 2) && threadIdx.x == 0) {
        const DpSub pn = dps[sn];
        prefetch_l2_bulk(abc + pn.abc_off, (size_t)dn.ns * pn.nc * 8);
      }
    }
    const int* rwn = rows + dn.map_off;
    const double* cfn = coefs + dn.map_off;
    int pr = -1;
    double pc = 0.0, px = 0.0;
    // x_s complete: a subdomain gathered inside the previous tile loop is covered by that loop's
    // barriers (have_xs is CTA-uniform unless the gather is flag-gated per thread)
    if (!have_xs || wait_flag) __syncthreads();
    int na = 0;   // A'' chunks streamed through the rings for this subdomain (0: pre-pass here)
    if (STORE_V && dps) {
      if (stream_a) na = dp_chunks(dps[s], d.ns);
      if (na == 0) fused_dp_t(dps[s], abc, xs, d.ns, tbuf, (flags & 4) && !stream_a ? cgp : nullptr);
    }
    if (STORE_V && warp < na) {   // this warp's A'' chunk: the first item of its stream for this subdomain
      const DpSub p = dps[s];
      const int slot = ncons % R;
      mbar_wait_parity(wfull + slot, (uint32_t)(ncons / R) & 1u);
      ++ncons;
      const double* T = wring + (size_t)slot * 1024;
      const int sh = p.nc == 8 ? 3 : p.nc == 4 ? 2 : 1;
      const int e0 = warp * 1024 + lane, tot = d.ns * p.nc;
      double acc = 0.0;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const int e = e0 + 32 * k;
        if (e < tot) acc = fma(T[lane + 32 * k], xs[e >> sh], acc);
      }
      __syncwarp();
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      request_next();
      for (int o = 16; o >= p.nc; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane < p.nc) tpart[warp][lane] = acc;
    }
    double* pw = part + warp * npad;
    const int ntiles = d.nb * (d.nb + 1) / 2;
    int it = 0;
    // (bi, bj) of tile t = warp, advanced with t (tile index bi (bi + 1) / 2 + bj, bj <= bi)
    int bi = 0, bj = warp;
    while (bj > bi) {
      bj -= bi + 1;
      ++bi;
    }
    for (int t = warp; t < ntiles; t += kSymWarps, ++it) {
      if (pre && it < 3 * nchain) {
        const int ch = it / 3, stage = it - 3 * ch, j = ch * 256 + threadIdx.x;
        if (stage == 0) {
          pr = -1;
          if (j < dn.ns) {
            pr = rwn[j];
            pc = cfn[j];
          }
        } else if (stage == 1) {
          px = pr >= 0 ? ldx(pr) : 0.0;
        } else if (j < dn.nb * 32) {
          double acc = 0.0;
          if (pr >= 0) acc += pc * px;
          xs_next[j] = acc;
        }
      }
      const int slot = ncons % R;
      mbar_wait_parity(wfull + slot, (uint32_t)(ncons / R) & 1u);
      ++ncons;
      const double* T = wring + (size_t)slot * 1024;
      double f[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) f[r] = T[r * 32 + lane];
      // the slot is drained (every lane holds its 32 values): refill it.  The
      // generic-proxy reads are ordered before the async-proxy write by the
      // warp barrier and the proxy fence of the issuing lane
      __syncwarp();
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      request_next();
      const double xj = xs[bj * 32 + lane];
      double c = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        c = fma(f[r], xs[bi * 32 + r], c);   // column part: sum_r F[r][lane] x_i[r]
        f[r] *= xj;                          // row part products
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const bool hi = (lane & o) != 0;
#pragma unroll
        for (int q = 0; q < o; ++q) {
          const double keep = hi ? f[q + o] : f[q];
          const double send = hi ? f[q] : f[q + o];
          f[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      pw[bi * 32 + lane] += f[0];
      if (bi != bj) pw[bj * 32 + lane] += c;
      bj += kSymWarps;
      while (bj > bi) {
        bj -= bi + 1;
        ++bi;
      }
    }
    __syncthreads();
    if (STORE_V && na > 0 && (int)threadIdx.x < dps[s].nc) {   // t_s: chunk partials in chunk order
      double t = 0.0;
      for (int w = 0; w < na; ++w) t += tpart[w][threadIdx.x];
      tbuf[dps[s].t_off + threadIdx.x] = t;
    }
    for (int i = threadIdx.x; i < npad; i += blockDim.x) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kSymWarps; ++w) {
        v += part[w * npad + i];
        part[w * npad + i] = 0.0;
      }
      if (i >= d.ns) continue;
      if (STORE_V) {
        vbuf[voff[s] + i] = v;
      } else {
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const int r = rw[i * KR + k];
          if (r >= 0) atomicAdd(y + r, cf[i * KR + k] * v);
        }
      }
    }
    __syncthreads();   // part is zero again; without the in-loop gather xs is rewritten by the next subdomain
    have_xs = pre;
    xsel ^= 1;
  }
  // Deterministic coarse gather (fused_dp_t's last-arriver pattern), once per
  // CTA instead of once per subdomain: the fence + atomic round trips of the
  // arrival count sat on warp 0's critical path in every subdomain (2.6 us
  // each at C4).  All t_s of this CTA were stored before the barriers above;
  // one thread per (subdomain, primal DOF) counts the arrival, and the last
  // owner to arrive sums the owners' entries in the fixed order.
  if (STORE_V && dps && cgp && (!(flags & 4) || stream_a)) {
    const CoarseGather cg = *cgp;
    const int nmine = sfirst < s1 ? (s1 - sfirst + G - 1) / G : 0;
    for (int q = threadIdx.x; q < nmine * 8; q += blockDim.x) {
      const DpSub p = dps[sfirst + (q >> 3) * G];
      const int c = q & 7;
      if (c < p.nc) {
        const int gid = cg.cmap[p.cmap_off + c];
        const int k0 = cg.optr[gid], k1 = cg.optr[gid + 1];
        __threadfence();
        if (atomicAdd(cg.cnt + gid, 1u) + 1u == (unsigned)(k1 - k0)) {
          __threadfence();
          double g = 0.0;
          for (int k = k0; k < k1; ++k) g += __ldcg(tbuf + cg.oidx[k]);
          cg.g[gid] = g;
          cg.cnt[gid] = 0u;
        }
      }
    }
  }
}

// pack the lower block-triangle of a row-major symmetric ns x ld matrix
// Explicit symmetric local operators (F_s, S~_s; row-major ns x ld per slot):
// the upper triangle is replaced by the lower one.  The elimination computes
// both triangles independently, and at SIMP contrast 1e9 they differ by
// rounding x cond(K_rr) (up to ~1e-8 relative): an F applied from both
// triangles is then measurably nonsymmetric, which costs FO / RRS their
// F-conjugacy.  The symmetric-packed kernels already read
// the lower block-triangle only.
__global__ void k_mirror_slots(const long long* __restrict__ moff, const int* __restrict__ ns_,
                               const int* __restrict__ ld_, double* __restrict__ mats) {
  const int sl = blockIdx.y;
  const int ns = ns_[sl], ld = ld_[sl];
  double* M = mats + moff[sl];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)ns * ns;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / ns), c = (int)(idx - (long long)r * ns);
    if (c > r) M[(size_t)r * ld + c] = M[(size_t)c * ld + r];
  }
}

__global__ void k_pack_sym(const long long* __restrict__ moff, const int* __restrict__ ns_,
                           const int* __restrict__ ld_, const long long* __restrict__ toff,
                           const double* __restrict__ mats, double* __restrict__ tiles) {
  const int sl = blockIdx.y;
  const int ns = ns_[sl], ld = ld_[sl];
  const int nb = (ns + 31) / 32;
  const long long tot = (long long)nb * (nb + 1) / 2 * 1024;
  const double* M = mats + moff[sl];
  double* T = tiles + toff[sl];
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(idx >> 10), e = (int)(idx & 1023);
    int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int bj = t - bi * (bi + 1) / 2;
    const int r = bi * 32 + (e >> 5), c = bj * 32 + (e & 31);
    T[idx] = (r < ns && c < ns) ? M[(size_t)r * ld + c] : 0.0;
  }
}

// FETI-DP coarse coupling, phase 1: t_s = A_bc^T x_s (after k_gather_gemv_scatter
// stored v_s = F_s x_s): x_s is re-gathered (1 row per DOF).
__global__ void k_dp_t(const OpSub* __restrict__ subs, const DpSub* __restrict__ dps,
                       const int* __restrict__ rows, const double* __restrict__ coefs,
                       const double* __restrict__ abc, const double* __restrict__ x,
                       double* __restrict__ tbuf) {
  const int s = blockIdx.x;
  const OpSub d = subs[s];
  const DpSub p = dps[s];
  __shared__ double red[8][kThreads / 32];
  double acc[8] = {};
  const double* Ab = abc + p.abc_off;
  for (int j = threadIdx.x; j < d.ns; j += blockDim.x) {
    const int r = rows[d.map_off + j];
    const double xj = r >= 0 ? coefs[d.map_off + j] * x[r] : 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < p.nc) acc[c] += Ab[(size_t)j * p.nc + c] * xj;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double v = warp_sum(acc[c]);
    if (lane == 0) red[c][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < p.nc) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    tbuf[p.t_off + threadIdx.x] = v;
  }
}

// global coarse vector: out[i] = sum over owners of primal DOF i (ascending
// subdomain order) of the per-subdomain entries -> deterministic assembly
__global__ void k_coarse_gather(const int* __restrict__ optr, const int* __restrict__ oidx,
                                const double* __restrict__ tbuf, int nc, double* __restrict__ out,
                                double sign, const double* __restrict__ add,
                                double* __restrict__ zero_y = nullptr, int ny = 0) {
  pdl_wait();
  if (zero_y)  // the apply's output is zeroed here, between phase 1 and phase 2
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ny; i += gridDim.x * blockDim.x) zero_y[i] = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
    double v = add ? add[i] : 0.0;
    for (int k = optr[i]; k < optr[i + 1]; ++k) v += sign * tbuf[oidx[k]];
    out[i] = v;
  }
}

// ------------------------------ FETI-DP coarse solve on the packed inverse --
// u = Kbar^{-1} g with Kbar^{-1} stored like F_s: lower block-triangle of
// 32x32 row-major tiles (about half the bytes of the dense inverse).
// Stage A (k_csym_tiles): warps stream the tiles, reading the matching slices of
// g = sum_s B_c^T t_s (formed by phase 1's fused last-arriver gather) from L2
// alongside, and write per tile the row part (for block row bi) and the
// transposed part (for block row bj).  Stage B (k_csym_reduce) sums those
// partials per block row in a fixed tile order, so the result is
// deterministic; no separate gather launch, no atomics.
__global__ void __launch_bounds__(128) k_csym_tiles(const double* __restrict__ tiles, int nb, int nc,
                                                    const double* __restrict__ g, double* __restrict__ rowp,
                                                    double* __restrict__ colp) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int ntiles = nb * (nb + 1) / 2;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntiles; t += nw) {
    int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > t) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    const int bj = t - bi * (bi + 1) / 2;
    const double* T = tiles + (size_t)t * 1024;
    double f[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) f[r] = __ldcs(T + r * 32 + lane);
    // g slices straight from L2, issued with the tile loads (zero beyond nc)
    const double xj = bj * 32 + lane < nc ? __ldcg(g + bj * 32 + lane) : 0.0;
    const double xi = bi * 32 + lane < nc ? __ldcg(g + bi * 32 + lane) : 0.0;
    double c = 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      c = fma(f[r], __shfl_sync(0xffffffffu, xi, r), c);   // transposed part: sum_r T[r][lane] g_i[r]
      f[r] *= xj;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {      // transpose-reduce: lane l <- sum_c T[l][c] g_j[c]
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int q = 0; q < o; ++q) {
        const double keep = hi ? f[q + o] : f[q];
        const double send = hi ? f[q] : f[q + o];
        f[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    rowp[(size_t)t * 32 + lane] = f[0];
    colp[(size_t)t * 32 + lane] = bi != bj ? c : 0.0;
  }
}

// Stage B: u[b*32 + l] = sum_{j <= b} rowp[tile(b, j)][l] + sum_{j > b} colp[tile(j, b)][l];
// one CTA of 16 warps per block row b; warp w sums tiles j = w, w + 16, ... in
// batches of 4 independent loads, warps are combined in fixed order
__global__ void __launch_bounds__(512) k_csym_reduce(const double* __restrict__ rowp,
                                                     const double* __restrict__ colp, int nb, int nc,
                                                     double* __restrict__ u) {
  pdl_wait();
  __shared__ double red[16][32];
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t rb = (size_t)b * (b + 1) / 2;
  auto part = [&](int j) -> const double* {
    return j <= b ? rowp + (rb + j) * 32 + lane : colp + ((size_t)j * (j + 1) / 2 + b) * 32 + lane;
  };
  double acc = 0.0;
  int j = warp;
  for (; j + 48 < nb; j += 64) {
    const double v0 = __ldcg(part(j)), v1 = __ldcg(part(j + 16)), v2 = __ldcg(part(j + 32)),
                 v3 = __ldcg(part(j + 48));
    acc += v0;
    acc += v1;
    acc += v2;
    acc += v3;
  }
  for (; j < nb; j += 16) acc += __ldcg(part(j));
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 16; ++w) v += red[w][lane];
    const int r = b * 32 + lane;
    if (r < nc) u[r] = v;
  }
}

// rows i = warp0, warp0 + nwarps, ... of y = M x (one warp per row; a row's
// result does not depend on the warp count).  x by weak loads (L1-cacheable:
// every row reads all of it); inside the persistent loop x is produced in an
// earlier phase, and the grid / cluster barrier's acquire invalidates L1.
// SM: M and x in shared memory (the cluster-resident loop)
template <bool SM = false>
__device__ __forceinline__ void dense_gemv_warps(const double* __restrict__ M, int n, const double* x,
                                                 double* y, int warp0, int nwarps) {
  const int lane = threadIdx.x & 31;
  auto ldm = [&](const double2* p) { return SM ? *p : __ldcs(p); };
  auto ldx = [&](const double* p) { return *p; };   // x is reused by every row: L1-cacheable weak loads
  // one row's chains (a0..a3 over lane-strided double2 pairs, then warp_sum)
  auto row = [&](int i) {
    const double* Mi = M + (size_t)i * n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if ((n & 1) == 0) {
      const double2* M2 = reinterpret_cast<const double2*>(Mi);
      const int n2 = n >> 1;
      int j = lane;
      for (; j + 32 < n2; j += 64) {
        const double2 u = ldm(M2 + j), v = ldm(M2 + j + 32);
        a0 = fma(u.x, ldx(x + 2 * j), a0);
        a1 = fma(u.y, ldx(x + 2 * j + 1), a1);
        a2 = fma(v.x, ldx(x + 2 * j + 64), a2);
        a3 = fma(v.y, ldx(x + 2 * j + 65), a3);
      }
      for (; j < n2; j += 32) {
        const double2 u = ldm(M2 + j);
        a0 = fma(u.x, ldx(x + 2 * j), a0);
        a1 = fma(u.y, ldx(x + 2 * j + 1), a1);
      }
    } else {
      for (int j = lane; j < n; j += 32) a0 = fma(Mi[j], ldx(x + j), a0);
    }
    return warp_sum((a0 + a1) + (a2 + a3));
  };
  int i = warp0;
  for (; i + 3 * nwarps < n; i += 4 * nwarps) {   // four rows in flight per warp
    const double v0 = row(i), v1 = row(i + nwarps), v2 = row(i + 2 * nwarps), v3 = row(i + 3 * nwarps);
    if (lane == 0) {
      y[i] = v0;
      y[i + nwarps] = v1;
      y[i + 2 * nwarps] = v2;
      y[i + 3 * nwarps] = v3;
    }
  }
  for (; i < n; i += nwarps) {
    const double v = row(i);
    if (lane == 0) y[i] = v;
  }
}
// dense row-major GEMV y = M x (one warp per row), n x n; 128-bit loads and
// four independent accumulators keep ~4 KB in flight per warp
__global__ void __launch_bounds__(256) k_dense_gemv(const double* __restrict__ M, int n,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y) {
  pdl_wait();
  dense_gemv_warps(M, n, x, y, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5);
}

// FETI-DP phase 2: v_s += A_bc u[cmap]; scatter sign * v_s.  A_bc rows are
// n_c (4 or 8) contiguous doubles, read as 128-bit pairs.
__device__ __forceinline__ void dp_phase2_cta(int s, const OpSub* __restrict__ subs, const DpSub* __restrict__ dps,
                                              const int* __restrict__ rows, const double* __restrict__ coefs,
                                              const double* __restrict__ abc, const int* __restrict__ cmap,
                                              const double* u, const double* vbuf, double* y, double vscale) {
  const OpSub d = subs[s];
  const DpSub p = dps[s];
  __shared__ double uc[8];
  const double* Ab = abc + p.abc_off;
  const bool vec = (p.nc & 1) == 0 && (p.abc_off & 1) == 0;
  // Rows j = tid and tid + blockDim (all of a C4 subdomain's rows): v, the A''
  // row, the dual row and its coefficient are requested BEFORE the barrier
  // that publishes u_s, so their DRAM latency overlaps the cmap -> u chain
  // instead of following it.  Same fma chain per row as the loop below.
  const int nh = p.nc >> 1;
  double2 a[2][4];
  double vv[2], cc[2];
  int rr[2];
  const bool fastp = vec && vbuf != nullptr;
  if (fastp) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = threadIdx.x + q * blockDim.x;
      rr[q] = -1;
      if (j < d.ns) {
        vv[q] = __ldcg(vbuf + p.v_off + j);
        const double2* A2 = reinterpret_cast<const double2*>(Ab + (size_t)j * p.nc);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < nh) a[q][c] = __ldcs(A2 + c);
        rr[q] = rows[d.map_off + j];
        cc[q] = coefs[d.map_off + j];
      }
    }
  }
  if (threadIdx.x < 8) uc[threadIdx.x] = threadIdx.x < p.nc ? __ldcg(u + cmap[p.cmap_off + threadIdx.x]) : 0.0;
  __syncthreads();
  if (fastp) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (rr[q] >= 0) {
        double v = vscale * vv[q];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < nh) {
            v = fma(a[q][c].x, uc[2 * c], v);
            v = fma(a[q][c].y, uc[2 * c + 1], v);
          }
        atomicAdd(y + rr[q], cc[q] * v);
      }
    }
  }
  for (int j = threadIdx.x + (fastp ? 2 * blockDim.x : 0); j < d.ns; j += blockDim.x) {
    double v = vbuf ? vscale * __ldcg(vbuf + p.v_off + j) : 0.0;
    if (vec) {
      const double2* A2 = reinterpret_cast<const double2*>(Ab + (size_t)j * p.nc);
      for (int c = 0; c < (p.nc >> 1); ++c) {
        const double2 a = __ldcs(A2 + c);
        v = fma(a.x, uc[2 * c], v);
        v = fma(a.y, uc[2 * c + 1], v);
      }
    } else {
      for (int c = 0; c < p.nc; ++c) v = fma(Ab[(size_t)j * p.nc + c], uc[c], v);
    }
    const int r = rows[d.map_off + j];
    if (r >= 0) atomicAdd(y + r, coefs[d.map_off + j] * v);
  }
}
__global__ void k_dp_phase2(const OpSub* __restrict__ subs, const DpSub* __restrict__ dps,
                            const int* __restrict__ rows, const double* __restrict__ coefs,
                            const double* __restrict__ abc, const int* __restrict__ cmap,
                            const double* __restrict__ u, const double* __restrict__ vbuf,
                            double* __restrict__ y, double vscale) {
  pdl_wait();
  dp_phase2_cta(blockIdx.x, subs, dps, rows, coefs, abc, cmap, u, vbuf, y, vscale);
}

// ------------------------------------------------------ T-FETI projector --
// g_s = -R_T^T (B_s^T v): per subdomain 3 values (K8, decomposition.hpp:136)
// g_s = sign R_T^T (B_s^T v) for one subdomain; vval(r) yields v at dual row r
// (an L2 load, or a value the persistent loop forms on the fly)
template <class VV>
__device__ __forceinline__ void proj_gather_fn(int s, int col, const OpSub* __restrict__ psubs,
                                               const int* __restrict__ rows, const double* __restrict__ coefs,
                                               const double* __restrict__ RT, const int* __restrict__ rt_off,
                                               double* g, int ldg, double sign, VV&& vval) {
  const OpSub d = psubs[s];
  const double* R = RT + rt_off[s];
  double a0 = 0, a1 = 0, a2 = 0;
  for (int j = threadIdx.x; j < d.ns; j += blockDim.x) {
    double xj = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int r = rows[d.map_off + j * 3 + k];
      if (r >= 0) xj += coefs[d.map_off + j * 3 + k] * vval(r);
    }
    a0 += R[j * 3] * xj;
    a1 += R[j * 3 + 1] * xj;
    a2 += R[j * 3 + 2] * xj;
  }
  __shared__ double red[3][kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2);
  if (lane == 0) { red[0][warp] = a0; red[1][warp] = a1; red[2][warp] = a2; }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[threadIdx.x][w];
    g[(size_t)col * ldg + 3 * s + threadIdx.x] = sign * t;
  }
}
__device__ __forceinline__ void proj_gather_cta(int s, int col, const OpSub* __restrict__ psubs,
                                                const int* __restrict__ rows, const double* __restrict__ coefs,
                                                const double* __restrict__ RT, const int* __restrict__ rt_off,
                                                const double* v, int ldv, double* g, int ldg, double sign, int rs) {
  const double* vc = v + (size_t)col * ldv;
  proj_gather_fn(s, col, psubs, rows, coefs, RT, rt_off, g, ldg, sign,
                 [&](int r) { return __ldcg(vc + (size_t)r * rs); });
}
__global__ void k_proj_gather(const OpSub* __restrict__ psubs, const int* __restrict__ rows,
                              const double* __restrict__ coefs, const double* __restrict__ RT,
                              const int* __restrict__ rt_off, const double* __restrict__ v, int ldv,
                              double* __restrict__ g, int ldg, double sign, int rs = 1) {
  pdl_wait();
  proj_gather_cta(blockIdx.x, blockIdx.y, psubs, rows, coefs, RT, rt_off, v, ldv, g, ldg, sign, rs);
}

// dense column-major H (n x n) times g columns: h = H g
__global__ void k_small_gemm(const double* __restrict__ H, int n, const double* __restrict__ g,
                             int ldg, double* __restrict__ h, int ldh) {
  const int col = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc = fma(H[(size_t)j * n + i], g[(size_t)col * ldg + j], acc);
    h[(size_t)col * ldh + i] = acc;
  }
}

// corr[row] += sign_entry * (R_T h_s)_j into a zeroed buffer (2 contributions per row)
// R_T h_s at one touched DOF (the value k_proj_scatter spreads over its rows)
__device__ __forceinline__ double proj_rh(const double* __restrict__ R, const double* __restrict__ hs) {
  return R[0] * hs[0] + R[1] * hs[1] + R[2] * hs[2];
}

// corr_r = c_plus + c_minus of dual row r (h read through L2 -- produced
// in-kernel by the persistent solver loop -- or from shared memory, SH)
template <bool SH = false>
__device__ __forceinline__ double proj_row_corr(int r, const int2* __restrict__ ent_sr,
                                                const double2* __restrict__ ent_c, const double* __restrict__ RT,
                                                const double* h) {
  auto ld = [&](const double* p) { return SH ? *p : __ldcg(p); };
  const int2 sr0 = ent_sr[2 * r], sr1 = ent_sr[2 * r + 1];   // (s, RT offset) or s < 0
  const double2 c = ent_c[r];
  double corr = 0.0;
  if (sr0.x >= 0) {
    const double* hs = h + 3 * sr0.x;
    const double hh[3] = {ld(hs), ld(hs + 1), ld(hs + 2)};
    corr = c.x * proj_rh(RT + sr0.y, hh);
  }
  if (sr1.x >= 0) {
    const double* hs = h + 3 * sr1.x;
    const double hh[3] = {ld(hs), ld(hs + 1), ld(hs + 2)};
    corr = corr + c.y * proj_rh(RT + sr1.y, hh);
  }
  return corr;
}

// Single-vector projector finish, row-wise: every dual row has at most two
// (subdomain, R row, sign) entries, so corr_r = c_plus + c_minus is formed in
// place (0 + a + b == a + b in either order: bit-identical to the zeroed
// buffer + atomic scatter it replaces) and either stored (proj_corr) or added
// to v (project) -- no memset, no atomics, one launch.
__global__ void k_proj_rows(int m, const int2* __restrict__ ent_sr, const double2* __restrict__ ent_c,
                            const double* __restrict__ RT, const double* __restrict__ h, double* __restrict__ out,
                            int accumulate) {
  pdl_wait();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < m; r += gridDim.x * blockDim.x) {
    const double corr = proj_row_corr(r, ent_sr, ent_c, RT, h);
    out[r] = accumulate ? __dadd_rn(out[r], corr) : corr;   // no contraction into corr's product
  }
}

__global__ void k_proj_scatter(const OpSub* __restrict__ psubs, const int* __restrict__ rows,
                               const double* __restrict__ coefs, const double* __restrict__ RT,
                               const int* __restrict__ rt_off, const double* __restrict__ h, int ldh,
                               double* __restrict__ corr, int ldc, int rs = 1) {
  pdl_wait();
  const int s = blockIdx.x, col = blockIdx.y;
  const OpSub d = psubs[s];
  const double* R = RT + rt_off[s];
  const double* hc = h + (size_t)col * ldh + 3 * s;
  const double h0 = hc[0], h1 = hc[1], h2 = hc[2];
  double* cc = corr + (size_t)col * ldc;
  const double hh[3] = {h0, h1, h2};
  for (int j = threadIdx.x; j < d.ns; j += blockDim.x) {
    const double v = proj_rh(R + j * 3, hh);
    for (int k = 0; k < 3; ++k) {
      const int r = rows[d.map_off + j * 3 + k];
      if (r >= 0) atomicAdd(cc + (size_t)r * rs, coefs[d.map_off + j * 3 + k] * v);
    }
  }
}

// PCG scalars live in device memory (no host round trip inside an iteration)
struct Scal {
  double delta;    // w^T F w
  double wr;       // w^T r
  double rz;       // r^T z (current)
  double rr, zz;
  double rz_old;
  double alpha;
  double breakdown;  // set to 1 by k_pcg_update when w^T F w <= 0
};

// ------------------------------------------------------------- reductions --
// Deterministic multi-dot: fixed grid, fixed per-block order, final pass in
// fixed order.  pairs: up to 4 (a_k, b_k) products of length n.
struct DotArgs {
  const double* a[4];
  const double* b[4];
  int npairs;
  int n;
};
constexpr int kDotBlocks = 1184;
__global__ void __launch_bounds__(kThreads) k_dot_partial(DotArgs args, double* partial) {
  double acc[4] = {0, 0, 0, 0};
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < args.n; i += stride) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < args.npairs) acc[k] = fma(args.a[k][i], args.b[k][i], acc[k]);
  }
  __shared__ double red[4][kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double v = warp_sum(acc[k]);
    if (lane == 0) red[k][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < args.npairs) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += red[threadIdx.x][w];
    partial[threadIdx.x * kDotBlocks + blockIdx.x] = v;
  }
}
__global__ void k_dot_final(const double* partial, int npairs, double* out) {
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= npairs) return;
  double acc = 0.0;
  for (int b = lane; b < kDotBlocks; b += 32) acc += partial[k * kDotBlocks + b];
  acc = warp_sum(acc);
  if (lane == 0) out[k] = acc;
}

// Per-block partial of the deterministic multi-dot: block vb of nvb (stride
// nvb * blockDim), written to partial[k * kDotBlocks + vb].  f(i, x, y) yields
// the NP operand pairs of row i (loads, or values the persistent loop forms
// on the fly); each pair accumulates fma(x, y, acc) in row order.
template <int NP, class F>
__device__ __forceinline__ void dot_partial_rows(int vb, int nvb, int n, double* partial, F&& f,
                                                 int pstride = kDotBlocks) {
  double acc[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) acc[k] = 0.0;
  const int stride = nvb * blockDim.x;
  for (int i = vb * blockDim.x + threadIdx.x; i < n; i += stride) {
    double x[NP], y[NP];
    f(i, x, y);
#pragma unroll
    for (int k = 0; k < NP; ++k) acc[k] = fma(x[k], y[k], acc[k]);
  }
  __shared__ double red[4][kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const double v = warp_sum(acc[k]);
    if (lane == 0) red[k][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < NP) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += red[threadIdx.x][w];
    partial[threadIdx.x * pstride + vb] = v;
  }
}
// operands through L2 (__ldcg)
template <int NP>
__device__ __forceinline__ void dot_partial_ld(const DotArgs& args, int vb, int nvb, double* partial) {
  dot_partial_rows<NP>(vb, nvb, args.n, partial, [&](int i, double* x, double* y) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      x[k] = __ldcg(args.a[k] + i);
      y[k] = __ldcg(args.b[k] + i);
    }
  });
}
__device__ __forceinline__ void dot_partial_cta(const DotArgs& args, int vb, int nvb, double* partial) {
  switch (args.npairs) {
    case 1: dot_partial_ld<1>(args, vb, nvb, partial); break;
    case 2: dot_partial_ld<2>(args, vb, nvb, partial); break;
    case 3: dot_partial_ld<3>(args, vb, nvb, partial); break;
    default: dot_partial_ld<4>(args, vb, nvb, partial); break;
  }
}
// final fixed-order sum of pair k over nvb partials (one warp; every lane returns it)
template <bool SM = false>   // SM: partials in shared memory (stride pstride)
__device__ __forceinline__ double dot_final_warp(const double* partial, int k, int nvb, int pstride = kDotBlocks) {
  const int lane = threadIdx.x & 31;
  double a = 0.0;
  for (int b = lane; b < nvb; b += 32) a += SM ? partial[k * pstride + b] : __ldcg(partial + k * pstride + b);
  return warp_sum(a);
}

// Single-launch deterministic multi-dot: fixed grid, per-block partials in a
// fixed slot, the last block to finish sums them in fixed order.
__global__ void __launch_bounds__(kThreads) k_dot_fused(DotArgs args, double* partial,
                                                        unsigned int* counter, double* out) {
  pdl_wait();
  __shared__ bool last;
  dot_partial_cta(args, blockIdx.x, gridDim.x, partial);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int k = threadIdx.x >> 5;
  if (k < args.npairs) {
    const double a = dot_final_warp(partial, k, gridDim.x);
    if ((threadIdx.x & 31) == 0) out[k] = a;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// FO re-orthogonalization against the first *cnt stored directions
// (column-major m x cap): psi_j = q_j^T w, then w -= sum_j psi_j w_j.
// The column count lives in device memory so the iteration graph is static.
__global__ void __launch_bounds__(kThreads) k_fo_psi(const double* __restrict__ Q, int m,
                                                     const int* __restrict__ cnt,
                                                     const double* __restrict__ w,
                                                     double* __restrict__ psi) {
  const int j = blockIdx.x;
  if (j >= *cnt) return;
  const double* q = Q + (size_t)j * m;
  double acc = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) acc = fma(q[i], w[i], acc);
  __shared__ double red[kThreads / 32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) s += red[k];
    psi[j] = s;
  }
}
// 32 rows per CTA (lane <-> row, coalesced per column), the 8 warps split the
// columns j = warp, warp+8, ...; partial sums reduced over warps in fixed order.
__device__ __forceinline__ void fo_sub_cta(int vb, const double* W, int m, int c, const double* psi, double* w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = vb * 32 + lane;
  __shared__ double part[8][33];
  double v = 0.0;
  if (i < m) {
    // four loads in flight per warp, then the FMAs in the same order as the
    // plain loop (bit-identical); otherwise each load waits for the last FMA
    int j = warp;
    for (; j + 120 < c; j += 128) {   // 16 columns in flight
      double wv[16], pv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        wv[u] = __ldcs(W + (size_t)(j + 8 * u) * m + i);
        pv[u] = psi[j + 8 * u];
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) v = fma(wv[u], pv[u], v);
    }
    for (; j + 24 < c; j += 32) {
      const double w0 = __ldcs(W + (size_t)j * m + i), w1 = __ldcs(W + (size_t)(j + 8) * m + i),
                   w2 = __ldcs(W + (size_t)(j + 16) * m + i), w3 = __ldcs(W + (size_t)(j + 24) * m + i);
      v = fma(w0, psi[j], v);
      v = fma(w1, psi[j + 8], v);
      v = fma(w2, psi[j + 16], v);
      v = fma(w3, psi[j + 24], v);
    }
    for (; j < c; j += 8) v = fma(W[(size_t)j * m + i], psi[j], v);
  }
  part[warp][lane] = v;
  __syncthreads();
  if (warp == 0 && i < m) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += part[k][lane];
    w[i] = __ldcg(w + i) - s;
  }
  __syncthreads();   // part[] is reused by the next row block of a persistent CTA
}
__global__ void __launch_bounds__(256) k_fo_sub(const double* __restrict__ W, int m,
                                                const int* __restrict__ cnt, int plus,
                                                const double* __restrict__ psi,
                                                double* __restrict__ w) {
  pdl_wait();
  fo_sub_cta(blockIdx.x, W, m, *cnt + plus, psi, w);
}
// one (column j, row segment s) item of psi = Q^T w (item = j * S + s)
__device__ __forceinline__ void fo_psi_item(int item, const double* Q, int m, const double* w, double* partial,
                                            int S) {
  const int chunk = (m + S - 1) / S;
  __shared__ double red[8];
  const int j = item / S, s = item - j * S;
  const int i0 = s * chunk, i1 = min(m, i0 + chunk);
  const double* q = Q + (size_t)j * m;
  double a0 = 0.0, a1 = 0.0;
  int i = i0 + threadIdx.x;
  for (; i + 768 < i1; i += 1024) {  // 4 loads of each vector in flight, same FMA order as 2-way
    const double q0 = __ldcs(q + i), q1 = __ldcs(q + i + 256), q2 = __ldcs(q + i + 512), q3 = __ldcs(q + i + 768);
    const double x0 = w[i], x1 = w[i + 256], x2 = w[i + 512], x3 = w[i + 768];
    a0 = fma(q0, x0, a0);
    a1 = fma(q1, x1, a1);
    a0 = fma(q2, x2, a0);
    a1 = fma(q3, x3, a1);
  }
  for (; i + 256 < i1; i += 512) {
    a0 = fma(q[i], w[i], a0);
    a1 = fma(q[i + 256], w[i + 256], a1);
  }
  if (i < i1) a0 = fma(q[i], w[i], a0);
  const double acc = warp_sum(a0 + a1);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red[k];
    partial[(size_t)j * S + s] = t;  // S == 1: partial is psi itself
  }
  __syncthreads();
}
// two items of the same row segment at once (the persistent loop, where one
// CTA works through several items): each item keeps its own chains, exactly
// as fo_psi_item computes them, so the loads of both are in flight together
__device__ __forceinline__ void fo_psi_item2(int itemA, int itemB, const double* Q, int m, const double* w,
                                             double* partial, int S) {
  const int chunk = (m + S - 1) / S;
  __shared__ double red2[2][8];
  const int jA = itemA / S, s = itemA - jA * S, jB = itemB / S;
  const int i0 = s * chunk, i1 = min(m, i0 + chunk);
  const double* qa = Q + (size_t)jA * m;
  const double* qb = Q + (size_t)jB * m;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
  int i = i0 + threadIdx.x;
  for (; i + 768 < i1; i += 1024) {
    const double q0 = __ldcs(qa + i), q1 = __ldcs(qa + i + 256), q2 = __ldcs(qa + i + 512), q3 = __ldcs(qa + i + 768);
    const double p0 = __ldcs(qb + i), p1 = __ldcs(qb + i + 256), p2 = __ldcs(qb + i + 512), p3 = __ldcs(qb + i + 768);
    const double x0 = w[i], x1 = w[i + 256], x2 = w[i + 512], x3 = w[i + 768];
    a0 = fma(q0, x0, a0);
    a1 = fma(q1, x1, a1);
    a0 = fma(q2, x2, a0);
    a1 = fma(q3, x3, a1);
    b0 = fma(p0, x0, b0);
    b1 = fma(p1, x1, b1);
    b0 = fma(p2, x2, b0);
    b1 = fma(p3, x3, b1);
  }
  for (; i + 256 < i1; i += 512) {
    a0 = fma(qa[i], w[i], a0);
    a1 = fma(qa[i + 256], w[i + 256], a1);
    b0 = fma(qb[i], w[i], b0);
    b1 = fma(qb[i + 256], w[i + 256], b1);
  }
  if (i < i1) {
    a0 = fma(qa[i], w[i], a0);
    b0 = fma(qb[i], w[i], b0);
  }
  const double accA = warp_sum(a0 + a1), accB = warp_sum(b0 + b1);
  if ((threadIdx.x & 31) == 0) {
    red2[0][threadIdx.x >> 5] = accA;
    red2[1][threadIdx.x >> 5] = accB;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red2[threadIdx.x][k];
    partial[(size_t)(threadIdx.x ? jB : jA) * S + s] = t;
  }
  __syncthreads();
}
// psi_j = q_j^T w for j < *cnt on a (column x row-segment) grid: CTA (j, s)
// reduces rows [s*chunk, (s+1)*chunk) of column j into partial[j*S + s];
// k_fo_psi_sum adds the S partials of each column in fixed order (skipped
// when S == 1, where the caller passes psi itself as the partial buffer).
__global__ void __launch_bounds__(256) k_fo_psi_seg(const double* __restrict__ Q, int m,
                                                    const int* __restrict__ cnt, int plus,
                                                    const double* __restrict__ w,
                                                    double* __restrict__ partial, int S) {
  pdl_wait();
  // fixed grid, grid-stride over the live (column j, segment s) items: no
  // empty CTAs for the not-yet-stored directions (the graph is static)
  const int items = (*cnt + plus) * S;
  for (int item = blockIdx.x; item < items; item += gridDim.x) fo_psi_item(item, Q, m, w, partial, S);
}
__global__ void k_fo_psi_sum(const int* __restrict__ cnt, int plus, int S, const double* __restrict__ partial,
                             double* __restrict__ psi) {
  pdl_wait();
  const int c = *cnt + plus;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < c; j += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int s = 0; s < S; ++s) t += partial[(size_t)j * S + s];
    psi[j] = t;
  }
}

// also re-zeroes q (last reader this iteration) for the next apply's scatter,
// and starts the next direction: w <- z (element-wise after its store, so no
// separate copy node).  Column *cnt is written; the count itself is advanced
// at the end of the iteration (k_iter_control or k_inc), so the CGS kernels in
// between read *cnt + 1.
__global__ void k_fo_store2(int n, const Scal* sc, const int* __restrict__ cnt,
                            double* __restrict__ w, double* __restrict__ q,
                            double* __restrict__ Wst, double* __restrict__ Qst,
                            const double* __restrict__ z) {
  pdl_wait();
  const double inv = 1.0 / sqrt(sc->delta);
  const int j = *cnt;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    Wst[(size_t)j * n + i] = w[i] * inv;
    Qst[(size_t)j * n + i] = q[i] * inv;
    q[i] = 0.0;
    w[i] = z[i];
  }
}
__global__ void k_inc(int* cnt) {
  pdl_wait(); *cnt += 1; }
// w = z + beta w with beta = rz / rz_old from device scalars; then rz_old = rz
// (zero_q: re-zeroed for the next apply's scatter; q is dead after k_pcg_update)
__global__ void k_cg_dir2(int n, Scal* sc, const double* __restrict__ z, double* __restrict__ w,
                          double* __restrict__ zero_q) {
  pdl_wait();
  const double beta = sc->rz / sc->rz_old;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    w[i] = fma(beta, w[i], z[i]);
    if (zero_q) zero_q[i] = 0.0;
  }
}
__global__ void k_shift_rz(Scal* sc) {
  pdl_wait(); sc->rz_old = sc->rz; }

// Device-side loop control of PCG / FO (runs as the last node of the
// iteration body under a CUDA-graph `while` conditional): the host loop's
// tests in the same order -- breakdown, NegativeInnerProduct (residual_metric,
// SPEC.md:420-423), eps = sqrt(max(r^T z, 0)), convergence, iteration cap --
// with the trace written to device memory.
struct IterCtl {
  int it, status, err, trace_cap;
  int max_it, pad;
  double eps, target;
};
__global__ void k_iter_control(const Scal* __restrict__ sc, IterCtl* __restrict__ c, double* __restrict__ trace,
                               cudaGraphConditionalHandle h, int* fo_cnt) {
  pdl_wait();
  if (fo_cnt) *fo_cnt += 1;   // FO: the direction stored this iteration
  unsigned int go = 0;
  if (sc->breakdown != 0.0) {
    c->status = 2;  // FETIGPU_BREAKDOWN
  } else if (sc->rz < -1e-14 * sqrt(sc->rr) * sqrt(sc->zz)) {
    c->err = 14;    // FETIGPU_E_NEGATIVE_INNER_PRODUCT
  } else {
    const double eps = sqrt(fmax(sc->rz, 0.0));
    const int it = c->it + 1;
    c->it = it;
    c->eps = eps;
    if (it < c->trace_cap) trace[it] = eps;
    if (eps <= c->target) c->status = 0;      // FETIGPU_CONVERGED
    else if (it >= c->max_it) c->status = 1;  // FETIGPU_MAX_ITER
    else go = 1;
  }
  cudaGraphSetConditional(h, go);
}

// ------------------------------------------------------- vector updates --

__global__ void k_axpy(int n, double a, const double* __restrict__ x, double* __restrict__ y) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}
// v += corr (projector finish)
__global__ void k_add(int n, const double* __restrict__ c, double* __restrict__ v, int ldc, int ldv) {
  pdl_wait();
  const int col = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[(size_t)col * ldv + i] += c[(size_t)col * ldc + i];
}
// alpha from device scalars; lambda += alpha w; r -= alpha * Pq  (Pq = q + corr or q)
__global__ void k_pcg_update(int n, Scal* sc, int fo, const double* __restrict__ w,
                             const double* __restrict__ q, const double* __restrict__ corr,
                             double* __restrict__ lambda, double* __restrict__ r, double* __restrict__ zero_z) {
  pdl_wait();
  if (zero_z)  // the preconditioner output of this iteration, zeroed here instead of a memset node
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) zero_z[i] = 0.0;
  if (!(sc->delta > 0.0)) {  // breakdown: leave lambda, r untouched
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->breakdown = 1.0;
    return;
  }
  const double alpha = (fo ? sc->wr : sc->rz) / sc->delta;
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->alpha = alpha;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    lambda[i] = fma(alpha, w[i], lambda[i]);
    const double pq = corr ? q[i] + corr[i] : q[i];
    r[i] = fma(-alpha, pq, r[i]);
  }
}
// w = z + beta w with beta = rz / rz_old
__global__ void k_cg_dir(int n, const Scal* sc, const double* __restrict__ z, double* __restrict__ w) {
  const double beta = sc->rz / sc->rz_old;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    w[i] = fma(beta, w[i], z[i]);
}
// FO: store w / sqrt(delta), q / sqrt(delta) as column j of W, Q
__global__ void k_fo_store(int n, const Scal* sc, const double* __restrict__ w,
                           const double* __restrict__ q, double* __restrict__ Wc,
                           double* __restrict__ Qc) {
  const double inv = 1.0 / sqrt(sc->delta);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    Wc[i] = w[i] * inv;
    Qc[i] = q[i] * inv;
  }
}
// y = x + beta * y
__global__ void k_xpby(int n, const double* __restrict__ x, double beta, double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = fma(beta, y[i], x[i]);
}
__global__ void k_sub(int n, const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

// ---------------------------------------------- one-time solves (rhs, u) --
// Per subdomain: x = (L L^T)^{-1} b with L the slot's dense factor (ne x ne,
// column-major).  b is gathered from perimeter vectors by `idx`.
__global__ void k_chol_solve(const double* __restrict__ fac, const long long* __restrict__ fac_off,
                             const int* __restrict__ slot_of, const int* __restrict__ nes,
                             double* __restrict__ xb, const int* __restrict__ xoff) {
  extern __shared__ double xsh[];
  const int s = blockIdx.x;
  const int sl = slot_of[s];
  const int ne = nes[sl];
  const double* L = fac + fac_off[sl];
  double* x = xb + xoff[s];
  for (int i = threadIdx.x; i < ne; i += blockDim.x) xsh[i] = x[i];
  __syncthreads();
  for (int j = 0; j < ne; ++j) {
    if (threadIdx.x == 0) xsh[j] = xsh[j] / L[(size_t)j * ne + j];
    __syncthreads();
    const double xj = xsh[j];
    for (int i = j + 1 + threadIdx.x; i < ne; i += blockDim.x) xsh[i] -= L[(size_t)j * ne + i] * xj;
    __syncthreads();
  }
  for (int j = ne - 1; j >= 0; --j) {
    if (threadIdx.x == 0) xsh[j] = xsh[j] / L[(size_t)j * ne + j];
    __syncthreads();
    const double xj = xsh[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) xsh[i] -= L[(size_t)i * ne + j] * xj;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < ne; i += blockDim.x) x[i] = xsh[i];
}

// Nested-dissection back substitution (recovery of module-interior DOFs):
// for every tree node top-down, u_e = -L_ee^{-T} (L_be^T u_b).
__global__ void k_nd_backsub(const NdDev* __restrict__ nodes, const int* __restrict__ topdown,
                             int n_nodes, const int* __restrict__ dofs, const double* __restrict__ fac,
                             long long fstride, const int* __restrict__ design, double* __restrict__ u,
                             int nloc) {
  extern __shared__ double sh[];
  const int s = blockIdx.x;
  double* us = u + (size_t)s * nloc;
  const double* F0 = fac + (size_t)design[s] * fstride;
  for (int t = 0; t < n_nodes; ++t) {
    const NdDev nd = nodes[topdown[t]];
    const int nf = nd.nf, ne = nd.ne, nbb = nf - ne;
    if (ne == 0) continue;
    const int* dl = dofs + nd.dof_off;
    double* ub = sh;          // nbb
    double* y = sh + nbb;     // ne
    for (int i = threadIdx.x; i < nbb; i += blockDim.x) ub[i] = us[dl[ne + i]];
    __syncthreads();
    const double* Fc = F0 + nd.foff;
    for (int k = threadIdx.x; k < ne; k += blockDim.x) {
      double acc = 0.0;
      const double* col = Fc + (size_t)k * nf + ne;
      for (int i = 0; i < nbb; ++i) acc = fma(col[i], ub[i], acc);
      y[k] = acc;
    }
    __syncthreads();
    for (int j = ne - 1; j >= 0; --j) {
      if (threadIdx.x == 0) y[j] = y[j] / Fc[(size_t)j * nf + j];
      __syncthreads();
      const double yj = y[j];
      for (int i = threadIdx.x; i < j; i += blockDim.x) y[i] -= Fc[(size_t)i * nf + j] * yj;
      __syncthreads();
    }
    for (int k = threadIdx.x; k < ne; k += blockDim.x) us[dl[k]] = -y[k];
    __syncthreads();
  }
}

// ------------------------------------------------ RRS block algebra (K10) --
// Rank-revealing pivoted Cholesky of the k x k Gram matrix Delta (Alg. 1
// line 9; pivoted_cholesky contract SPEC.md:43-47 with a symmetric trailing
// update): one CTA, pivots sequential, updates parallel.
// Rank-revealing pivoted Cholesky on one thread-block cluster of CL CTAs:
// the n x n Gram matrix lives in the cluster's distributed shared memory, row j
// on CTA j % CL (local row j / CL), so k <= 640 stays on chip with CL = 16.
// Four barriers per pivot:
//   each CTA publishes its best remaining diagonal (tracked during the
//   previous trailing update) -> cluster barrier (1) -> every warp reduces the
//   CL candidates (ties -> lowest index, so all pick the same pivot) -> the
//   owners of rows k and piv fetch the partner row over DSMEM with the column
//   transposition applied -> (2) -> rows rewritten, columns k <-> piv swapped
//   in every other row, row k scaled by 1/sqrt(pivot) from the fetched copy
//   and published -> (3) -> every CTA copies row k -> CTA barrier (4) ->
//   rank-1 update of its own rows.
// The one-to-all traffic (candidates, pivot row) goes through a small global
// scratch `gx` (L2; the cluster barrier orders it and invalidates L1): a DSMEM
// broadcast would serialise on the owner's shared-memory port.
// Per-element arithmetic and tie-breaking are those of the right-looking
// algorithm in k_pivchol_coop (and the oracle): results are bit-identical.
constexpr int kPivcholClusterMaxN = 640;
template <int CL>
__global__ void __launch_bounds__(512) k_pivchol_cl(double* Ag, int n, double tol, int* perm, int* rank_out,
                                                    int* status, double* gx /* n + 4*CL */) {
  namespace cg = cooperative_groups;
  extern __shared__ double s_dyn[];
  __shared__ double s_wv[16];
  __shared__ int s_wi[16];
  const int R = (n + CL - 1) / CL;
  double* A = s_dyn;                   // R x n, own rows
  double* prow = A + (size_t)R * n;    // copy of the scaled pivot row
  double* tmpk = prow + n;             // incoming row for local row k
  double* tmpp = tmpk + n;             // incoming row for local row piv
  double* gcand = gx + n;              // per CTA: (value, index, max diag)
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  int me = 0;
  if constexpr (CL > 1) me = (int)cg::this_cluster().block_rank();
  auto csync = [&]() {
    if constexpr (CL > 1) cg::this_cluster().sync();
    else __syncthreads();
  };
  auto remote = [&](double* p, int r) -> double* {
    if constexpr (CL > 1) return cg::this_cluster().map_shared_rank(p, r);
    else return p;
  };
  auto better = [](double v, int i, double bv, int bi) { return v > bv || (v == bv && i < bi); };
  auto ldx = [](const double* p) -> double {  // L2 read for peers; same-SM data may sit in L1
    if constexpr (CL > 1) return __ldcg(p);
    else return *(volatile const double*)p;
  };
  auto warp_best = [&](double& v, int& i) {
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, i, o);
      if (better(ov, oi, v, i)) { v = ov; i = oi; }
    }
  };
  // publish this CTA's candidate (after the per-warp partials are in s_wv/s_wi)
  auto publish = [&](double mx) {
    if constexpr (CL == 1) return;  // single CTA: the warp partials in s_wv / s_wi are read directly
    __syncthreads();
    if (warp == 0) {
      double v = lane < nwarp ? s_wv[lane] : -1e300;
      int i = lane < nwarp ? s_wi[lane] : n;
      warp_best(v, i);
      if (lane == 0) {
        gcand[3 * me] = v;
        gcand[3 * me + 1] = (double)i;
        gcand[3 * me + 2] = mx;
      }
    }
  };
  for (int lr = 0; lr < R; ++lr) {
    const int j = lr * CL + me;
    if (j < n)
      for (int i = tid; i < n; i += nt) A[(size_t)lr * n + i] = Ag[(size_t)j * n + i];
  }
  if (me == 0)
    for (int i = tid; i < n; i += nt) perm[i] = i;
  __syncthreads();
  // scale = max initial diagonal over the cluster; first candidates (k = 0)
  double bv = -1e300, mx = -1e300;
  int bi = n;
  for (int lr = tid; lr < R; lr += nt) {
    const int j = lr * CL + me;
    if (j < n) {
      const double v = A[(size_t)lr * n + j];
      mx = fmax(mx, v);
      if (better(v, j, bv, bi)) { bv = v; bi = j; }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  warp_best(bv, bi);
  __shared__ double s_mx[16];
  if (lane == 0) { s_wv[warp] = bv; s_wi[warp] = bi; s_mx[warp] = mx; }
  __syncthreads();
  double cmx = -1e300;
  for (int w = 0; w < nwarp; ++w) cmx = fmax(cmx, s_mx[w]);
  publish(cmx);
  csync();
  double scale = -1e300;
  if constexpr (CL == 1) scale = cmx;
  else
    for (int r = lane; r < CL; r += 32) scale = fmax(scale, ldx(&gcand[3 * r + 2]));
  for (int o = 16; o > 0; o >>= 1) scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
  const double stop_tol = tol * scale;
  const double neg_tol = -tol * fmax(scale, 1e-300);
  int rank = 0;
  bool first = true;
  for (int k = 0; k < n; ++k) {
    if (!first) csync();  // (1) candidates of the previous update visible
    first = false;
    double v = -1e300;
    int b = n;
    if constexpr (CL == 1) {
      if (lane < nwarp) { v = s_wv[lane]; b = s_wi[lane]; }
    } else if (lane < CL) {
      v = ldx(&gcand[3 * lane]);
      b = (int)ldx(&gcand[3 * lane + 1]);
    }
    warp_best(v, b);
    if (!(v > stop_tol)) {
      for (int lr = tid; lr < R; lr += nt) {
        const int j = lr * CL + me;
        if (j >= k && j < n && A[(size_t)lr * n + j] < neg_tol) atomicExch(status, 2 /* IndefiniteInput */);
      }
      break;
    }
    const int piv = b;
    const int ok = k % CL, op = piv % CL;
    double* rowk = A + (size_t)(k / CL) * n;   // valid on CTA ok
    if (piv != k) {
      // fetch the partner rows (old contents) with columns k <-> piv swapped
      if (me == ok) {
        const double* src = remote(A, op) + (size_t)(piv / CL) * n;
        for (int i = tid; i < n; i += nt) tmpk[i] = src[i == k ? piv : (i == piv ? k : i)];
      }
      if (me == op) {
        const double* src = remote(A, ok) + (size_t)(k / CL) * n;
        for (int i = tid; i < n; i += nt) tmpp[i] = src[i == k ? piv : (i == piv ? k : i)];
      }
    }
    csync();  // (2) partner rows read, all candidate reads done
    const double* srck = piv != k ? tmpk : rowk;
    double l = 0.0;
    if (me == ok) l = sqrt(srck[k]);
    if (piv != k) {
      for (int lr = tid; lr < R; lr += nt) {  // other rows: columns k <-> piv
        const int j = lr * CL + me;
        if (j >= n || j == k || j == piv) continue;
        double* row = A + (size_t)lr * n;
        const double t = row[k];
        row[k] = row[piv];
        row[piv] = t;
      }
      if (me == op) {
        double* row = A + (size_t)(piv / CL) * n;
        for (int i = tid; i < n; i += nt) row[i] = tmpp[i];
      }
      if (me == 0 && tid == 0) { const int t = perm[k]; perm[k] = perm[piv]; perm[piv] = t; }
    }
    if (me == ok)  // row k := fetched row, entries right of the pivot scaled and published
      for (int i = tid; i < n; i += nt)
        if (i != k) {
          const double x = i > k ? srck[i] / l : srck[i];
          rowk[i] = x;
          if (CL > 1 && i > k) gx[i] = x;
        }
    csync();  // (3) scaled pivot row visible
    if (me == ok && tid == 0) rowk[k] = l;  // nobody reads the pivot entry after (3)
    if constexpr (CL > 1) {
      if (me != ok)
        for (int i = k + 1 + tid; i < n; i += nt) prow[i] = __ldcg(&gx[i]);
      else
        for (int i = k + 1 + tid; i < n; i += nt) prow[i] = rowk[i];
    } else {
      for (int i = k + 1 + tid; i < n; i += nt) prow[i] = rowk[i];
    }
    __syncthreads();  // (4)
    // trailing rank-1 update of own rows j > k (a warp per row, lanes over i),
    // tracking the best updated diagonal as the next candidate
    bv = -1e300;
    bi = n;
    for (int lr = warp; lr < R; lr += nwarp) {
      const int j = lr * CL + me;
      if (j <= k || j >= n) continue;
      double* row = A + (size_t)lr * n;
      const double akj = prow[j];
      for (int i = k + 1 + lane; i < n; i += 32) {
        const double nv = row[i] - prow[i] * akj;
        row[i] = nv;
        if (i == j && better(nv, j, bv, bi)) { bv = nv; bi = j; }
      }
    }
    warp_best(bv, bi);
    if (lane == 0) { s_wv[warp] = bv; s_wi[warp] = bi; }
    publish(0.0);
    rank = k + 1;
  }
  csync();  // no CTA leaves while a peer may still read its shared memory
  for (int lr = 0; lr < R; ++lr) {
    const int j = lr * CL + me;
    if (j < n)
      for (int i = tid; i < n; i += nt) Ag[(size_t)j * n + i] = A[(size_t)lr * n + i];
  }
  if (me == 0 && tid == 0) *rank_out = rank;
}

// Alg. 1 line 9 in one thread-block cluster with ONE cluster barrier per
// pivot (k_pivchol_cl needs three plus the physical row / column swaps).  The
// rows stay in original index order, distributed over the CTAs (row x on CTA
// x % CL); every CTA keeps a replica of the diagonal and of the position ->
// index map, so each picks the same pivot itself (max diagonal over the
// remaining positions, ties to the lowest position), reads the pivot row from
// its owner over DSMEM, forms the scaled column L_i = A_{x,i} / l and updates
// its own remaining rows, A_ji -= L_i L_j, and its diagonal replica with the
// same operation.  These are k_pivchol_cl's values entry for entry (the same
// division, the same fma per entry in pivot order), so rank, permutation and
// L are bit-identical; column k of L is written to Ag (original index order)
// as the pivots go and permuted into place at the end.
template <int CL>
__global__ void __launch_bounds__(512) k_pivchol_cl1(double* Ag, int n, double tol, int* perm, int* rank_out,
                                                     int* status) {
  namespace cg = cooperative_groups;
  extern __shared__ double s_dyn[];
  __shared__ double s_wv[16];
  __shared__ int s_wi[16];
  __shared__ double s_bv;
  __shared__ int s_bp;
  const int R = (n + CL - 1) / CL;
  double* A = s_dyn;                                  // R x n own rows, original order
  double* Lc = A + (size_t)R * n;                     // the current column of L, by original index
  double* d = Lc + n;                                 // diagonal replica, by original index
  int* at = reinterpret_cast<int*>(d + n);            // position -> original index
  unsigned char* done = reinterpret_cast<unsigned char*>(at + n);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  int me = 0;
  if constexpr (CL > 1) me = (int)cg::this_cluster().block_rank();
  auto csync = [&]() {
    if constexpr (CL > 1) cg::this_cluster().sync();
    else __syncthreads();
  };
  auto remote = [&](double* p, int r) -> double* {
    if constexpr (CL > 1) return cg::this_cluster().map_shared_rank(p, r);
    else return p;
  };
  auto better = [](double v, int i, double bv, int bi) { return v > bv || (v == bv && i < bi); };
  for (int lr = 0; lr < R; ++lr) {
    const int x = lr * CL + me;
    if (x < n)
      for (int i = tid; i < n; i += nt) A[(size_t)lr * n + i] = Ag[(size_t)x * n + i];
  }
  double mx = -1e300;
  for (int i = tid; i < n; i += nt) {
    d[i] = Ag[(size_t)i * n + i];
    at[i] = i;
    done[i] = 0;
    Lc[i] = 0.0;
    mx = fmax(mx, d[i]);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_wv[warp] = mx;
  __syncthreads();
  double scale = -1e300;
  for (int w = 0; w < nwarp; ++w) scale = fmax(scale, s_wv[w]);
  const double stop_tol = tol * scale;
  const double neg_tol = -tol * fmax(scale, 1e-300);
  csync();   // every CTA has its input before column 0 of L overwrites row 0 of Ag
  int rank = 0;
  for (int k = 0; k < n; ++k) {
    // pivot: the best diagonal over positions p >= k (identical in every CTA)
    double bv = -1e300;
    int bp = n;
    for (int p = k + tid; p < n; p += nt) {
      const double v = d[at[p]];
      if (better(v, p, bv, bp)) { bv = v; bp = p; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; }
    }
    if (lane == 0) { s_wv[warp] = bv; s_wi[warp] = bp; }
    __syncthreads();
    if (warp == 0) {   // the best of the warp bests (a total order: any tree gives the same pivot)
      double v = lane < nwarp ? s_wv[lane] : -1e300;
      int p = lane < nwarp ? s_wi[lane] : n;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int op = __shfl_xor_sync(0xffffffffu, p, o);
        if (better(ov, op, v, p)) { v = ov; p = op; }
      }
      if (lane == 0) {
        s_bv = v;
        s_bp = p;
        if (v > stop_tol) {   // swap positions k <-> p
          const int t = at[k];
          at[k] = at[p];
          at[p] = t;
        }
      }
    }
    __syncthreads();
    if (!(s_bv > stop_tol)) {
      if (me == 0)
        for (int p = k + tid; p < n; p += nt)
          if (d[at[p]] < neg_tol) atomicExch(status, 2 /* IndefiniteInput */);
      break;
    }
    const int x = at[k];
    const double l = sqrt(d[x]);
    const double* rx = remote(A, x % CL) + (size_t)(x / CL) * n;
    const bool writer = me == k % CL;
    for (int p = k + 1 + tid; p < n; p += nt) {
      const int i = at[p];
      const double v = rx[i] / l;
      Lc[i] = v;
      if (writer) Ag[(size_t)k * n + i] = v;
    }
    if (writer && tid == 0) Ag[(size_t)k * n + x] = l;
    if (tid == 0) done[x] = 1;
    __syncthreads();
    // own remaining rows j: A_ji -= L_i L_j.  Contiguous over ALL columns:
    // entries at pivoted columns (stale Lc) are never read again, the
    // remaining ones get exactly the pivot-order operation
    for (int lr = warp; lr < R; lr += nwarp) {
      const int j = lr * CL + me;
      if (j >= n || done[j]) continue;
      double* row = A + (size_t)lr * n;
      const double lj = Lc[j];
      for (int i = lane; i < n; i += 32) row[i] = row[i] - Lc[i] * lj;
    }
    for (int i = tid; i < n; i += nt) d[i] = d[i] - Lc[i] * Lc[i];   // the diagonal replica, same operation
    rank = k + 1;
    csync();   // step k's updates (and reads of its pivot row) done everywhere
  }
  csync();   // all columns of L written
  // columns of L into the final position order: Ag[c][p] = L_{at[p], c}, p >= c
  for (int c = me; c < rank; c += CL) {
    for (int i = tid; i < n; i += nt) Lc[i] = Ag[(size_t)c * n + i];
    __syncthreads();
    for (int p = c + tid; p < n; p += nt) Ag[(size_t)c * n + p] = Lc[at[p]];
    __syncthreads();
  }
  if (me == 0) {
    for (int i = tid; i < n; i += nt) perm[i] = at[i];
    if (tid == 0) *rank_out = rank;
  }
}

// Same algorithm and per-element arithmetic as k_pivchol, spread over a
// cooperative grid: block 0 selects the pivot, swaps and scales column k; all
// blocks share the rank-1 trailing update; two grid syncs per pivot.
// Cooperative-grid pivoted Cholesky with ONE grid barrier per pivot (k > 640).
// Rows and columns are never swapped: A stays in original index order and
// every CTA keeps the position -> index map in shared memory, choosing the
// next pivot itself (same scan and reduction tree in every CTA, so all agree)
// and forming the scaled pivot column in shared memory before its share of
// the trailing update.  The pivot scan of step k may overlap faster CTAs'
// updates of step k, so it reads the diagonal from a ping-pong copy dd[k & 1]
// that step k writes only into dd[(k + 1) & 1]; the pivot column itself is
// never touched by its own step's update.  Per pivot the values are those of
// k_pivchol_coop (the same division for L, the same fma(-L_i, L_j, A_ij) per
// entry, ties to the lowest position), so rank, permutation and L are
// bit-identical; the serial block-0 phase and one grid barrier are gone.  L is
// collected by original row in `lc` (n x n) and written to A in pivot order
// at the end.  Dynamic shared memory: n doubles + n ints.  dd: 2n doubles.
__global__ void __launch_bounds__(512) k_pivchol_coop1(double* A, int n, double tol, int* perm,
                                                       int* rank_out, int* status, double* lc, double* dd) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double psm[];
  double* Ls = psm;                                   // scaled pivot column, by position
  int* at = reinterpret_cast<int*>(Ls + n);           // original index at position
  __shared__ double sv[16];
  __shared__ int si[16];
  __shared__ double s_scale;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  for (int i = tid; i < n; i += nt) at[i] = i;
  for (long long i = blockIdx.x * (long long)nt + tid; i < n; i += (long long)gridDim.x * nt)
    dd[i] = A[(size_t)i * n + i];
  grid.sync();
  {
    double mx = -1e300;
    for (int i = tid; i < n; i += nt) mx = fmax(mx, dd[i]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) sv[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m2 = sv[0];
      for (int w = 1; w < nwarp; ++w) m2 = fmax(m2, sv[w]);
      s_scale = m2;
    }
    __syncthreads();
  }
  const double stop_tol = tol * s_scale;
  const double neg_tol = -tol * fmax(s_scale, 1e-300);
  int k = 0;
  for (; k < n; ++k) {
    const double* dcur = dd + (size_t)(k & 1) * n;
    double* dnext = dd + (size_t)((k + 1) & 1) * n;
    // pivot: largest remaining diagonal, ties -> lowest position
    double bv = -1e300;
    int bi = n;
    for (int j = k + tid; j < n; j += nt) {
      const double v = dcur[at[j]];
      if (v > bv || (v == bv && j < bi)) { bv = v; bi = j; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
    __syncthreads();
    double v = sv[0];
    int b = si[0];
    for (int w = 1; w < nwarp; ++w)
      if (sv[w] > v || (sv[w] == v && si[w] < b)) { v = sv[w]; b = si[w]; }
    if (!(v > stop_tol)) {
      if (blockIdx.x == 0)
        for (int j = k + tid; j < n; j += nt)
          if (dcur[at[j]] < neg_tol) atomicExch(status, 2);
      break;
    }
    const int q = at[b], qk = at[k];
    __syncthreads();   // every thread has read sv/si and at[b], at[k] before the swap
    if (tid == 0) { at[k] = q; at[b] = qk; }
    __syncthreads();
    const double l = sqrt(A[(size_t)q * n + q]);
    // scaled pivot column by position (the old kernel's ck[i] /= l)
    for (int p = k + 1 + tid; p < n; p += nt) Ls[p] = A[(size_t)q * n + at[p]] / l;
    if (blockIdx.x == 0) {
      for (int p = k + 1 + tid; p < n; p += nt) lc[(size_t)k * n + at[p]] = Ls[p];
      if (tid == 0) lc[(size_t)k * n + q] = l;
    }
    __syncthreads();
    const int r = n - k - 1;
    const long long tot = (long long)r * r;
    for (long long idx = blockIdx.x * (long long)nt + tid; idx < tot; idx += (long long)gridDim.x * nt) {
      const int pj = k + 1 + (int)(idx / r), pi = k + 1 + (int)(idx % r);
      double* e = A + (size_t)at[pj] * n + at[pi];
      const double nv = *e - Ls[pi] * Ls[pj];
      *e = nv;
      if (pi == pj) dnext[at[pi]] = nv;
    }
    grid.sync();
  }
  grid.sync();   // (break path) every CTA is done reading A before it is overwritten
  // L in pivot order: column c < k holds rows p >= c (the layout of k_pivchol_coop)
  for (long long idx = blockIdx.x * (long long)nt + tid; idx < (long long)k * n;
       idx += (long long)gridDim.x * nt) {
    const int c = (int)(idx / n), p = (int)(idx % n);
    if (p >= c) A[(size_t)c * n + p] = lc[(size_t)c * n + at[p]];
  }
  if (blockIdx.x == 0) {
    for (int i = tid; i < n; i += nt) perm[i] = at[i];
    if (tid == 0) *rank_out = k;
  }
}

__global__ void __launch_bounds__(512) k_pivchol_coop(double* A, int n, double tol, int* perm,
                                                      int* rank_out, int* status, int* ctl) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sv[16];
  __shared__ int si[16];
  __shared__ double s_scale;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  const bool b0 = blockIdx.x == 0;
  if (b0) {
    for (int i = tid; i < n; i += nt) perm[i] = i;
    double mx = -1e300;
    for (int i = tid; i < n; i += nt) mx = fmax(mx, A[(size_t)i * n + i]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) sv[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double m2 = sv[0];
      for (int w = 1; w < nwarp; ++w) m2 = fmax(m2, sv[w]);
      s_scale = m2;
    }
    __syncthreads();
  }
  int k = 0;
  for (; k < n; ++k) {
    if (b0) {
      const double stop_tol = tol * s_scale;
      const double neg_tol = -tol * fmax(s_scale, 1e-300);
      double bv = -1e300;
      int bi = n;
      for (int j = k + tid; j < n; j += nt) {
        const double v = A[(size_t)j * n + j];
        if (v > bv || (v == bv && j < bi)) { bv = v; bi = j; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
      __syncthreads();
      if (tid == 0) {
        double v = sv[0];
        int b = si[0];
        for (int w = 1; w < nwarp; ++w)
          if (sv[w] > v || (sv[w] == v && si[w] < b)) { v = sv[w]; b = si[w]; }
        ctl[0] = b;
        ctl[1] = !(v > stop_tol);
      }
      __syncthreads();
      if (ctl[1]) {
        for (int j = k + tid; j < n; j += nt)
          if (A[(size_t)j * n + j] < neg_tol) atomicExch(status, 2);
      } else {
        const int piv = ctl[0];
        if (piv != k) {
          for (int j = tid; j < n; j += nt) {
            const double t = A[(size_t)j * n + k];
            A[(size_t)j * n + k] = A[(size_t)j * n + piv];
            A[(size_t)j * n + piv] = t;
          }
          __syncthreads();
          for (int i = tid; i < n; i += nt) {
            const double t = A[(size_t)k * n + i];
            A[(size_t)k * n + i] = A[(size_t)piv * n + i];
            A[(size_t)piv * n + i] = t;
          }
          if (tid == 0) { const int t = perm[k]; perm[k] = perm[piv]; perm[piv] = t; }
          __syncthreads();
        }
        const double l = sqrt(A[(size_t)k * n + k]);
        __syncthreads();
        if (tid == 0) A[(size_t)k * n + k] = l;
        for (int i = k + 1 + tid; i < n; i += nt) A[(size_t)k * n + i] /= l;
      }
      __threadfence();
    }
    grid.sync();
    if (((volatile int*)ctl)[1]) break;
    const int r = n - k - 1;
    const long long tot = (long long)r * r;
    for (long long idx = blockIdx.x * (long long)nt + tid; idx < tot; idx += (long long)gridDim.x * nt) {
      const int j = k + 1 + (int)(idx / r), i = k + 1 + (int)(idx % r);
      A[(size_t)j * n + i] -= A[(size_t)k * n + i] * A[(size_t)k * n + j];
    }
    grid.sync();
  }
  if (b0 && tid == 0) *rank_out = k;
}

// out[:, c] = in[:, perm[c]] for c < cols (column gather, column-major)
__global__ void k_gather_cols(const double* __restrict__ in, int ld, const int* __restrict__ perm,
                              int cols, double* __restrict__ out) {
  const int c = blockIdx.y;
  if (c >= cols) return;
  const double* src = in + (size_t)perm[c] * ld;
  double* dst = out + (size_t)c * ld;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

// row-major: out(i, c) = in(i, perm[c]) for c < cols
__global__ void k_gather_cols_rm(const double* __restrict__ in, int ldi, const int* __restrict__ perm,
                                 int cols, int m, double* __restrict__ out, int ldo) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)m * cols;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / cols), c = (int)(idx - (long long)i * cols);
    out[(size_t)i * ldo + c] = in[(size_t)i * ldi + perm[c]];
  }
}

// Transposing column gather: out(i, c) = in(i, perm[c]), in row-major m x ldi,
// out column-major (ld ldo).  32 x 32 tiles through shared memory so both the
// gathered reads (rows of `in`) and the column writes are coalesced.
__global__ void __launch_bounds__(256) k_gather_cols_t(const double* __restrict__ in, int ldi,
                                                       const int* __restrict__ perm, int cols, int m,
                                                       double* __restrict__ out, int ldo) {
  __shared__ double tile[32][33];
  const int i0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int pc = c0 + tx < cols ? perm[c0 + tx] : 0;
  for (int r = ty; r < 32; r += 8)
    if (i0 + r < m && c0 + tx < cols) tile[r][tx] = in[(size_t)(i0 + r) * ldi + pc];
  __syncthreads();
  for (int c = ty; c < 32; c += 8)
    if (c0 + c < cols && i0 + tx < m) out[(size_t)(c0 + c) * ldo + i0 + tx] = tile[tx][c];
}

// mirror the lower triangle into the upper (Delta uses its lower triangle)
__global__ void k_mirror_lower(double* A, int n) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx / n), i = (int)(idx % n);
    if (i < j) A[idx] = A[(size_t)i * n + j];
  }
}

// Fold the +-1 constraint signs of a FETI-DP slot into its explicit operators:
// F'' = S F S (row-major ns x ld), A'' = S A_bc (ns x nc).  Exact.
__global__ void k_fold_signs(const long long* __restrict__ moff, const int* __restrict__ ns_,
                             const int* __restrict__ ld_, const long long* __restrict__ aoff,
                             const int* __restrict__ nc_, const int* __restrict__ soff,
                             const double* __restrict__ sgn, double* __restrict__ mats,
                             double* __restrict__ abc) {
  const int sl = blockIdx.y;
  const int ns = ns_[sl], ld = ld_[sl], nc = nc_[sl];
  const double* sg = sgn + soff[sl];
  double* M = mats + moff[sl];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < ns * ns; idx += gridDim.x * blockDim.x) {
    const int i = idx / ns, j = idx - i * ns;
    M[(size_t)i * ld + j] *= sg[i] * sg[j];
  }
  if (abc) {
    double* A = abc + aoff[sl];
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < ns * nc; idx += gridDim.x * blockDim.x)
      A[idx] *= sg[idx / nc];
  }
}

// L2 flush helper: write a buffer larger than L2
__global__ void k_flush(double* buf, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    buf[i] = v;
}

__global__ void k_fill_random(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
  }
}

}  // namespace fg

namespace fg {

// ------------------------------- blocked pivoted Cholesky (k > 640) --
// The right-looking algorithm of k_pivchol_coop1 reorganised into panels of
// kPcNB pivots without changing a single operation: every entry still
// receives fma(-L_i, L_j, a) once per pivot, in pivot order.
//   * panel phase (one CTA, k_pc_panel): for each pivot of the panel, the
//     largest remaining diagonal (ties -> lowest position) from the running
//     diagonal d, and the pivot row's current entries computed on the fly:
//     the stored entry (updated up to the panel start) followed by the
//     in-panel updates in pivot order -- exactly the values the right-looking
//     kernel would hold; L column = row / sqrt(d_q), d updated by the same fma;
//   * trailing phase (grid, k_pc_trailing): every remaining entry of the lower
//     triangle takes the panel's updates as one fma chain in pivot order.
// The symmetric matrix is updated in its lower triangle only (the two
// triangles received identical updates before).  One grid-wide phase per
// kPcNB pivots instead of a grid barrier per pivot.
constexpr int kPcNB = 32;
struct PcCtl {
  int k;         // pivots done
  int stop;      // 1: rank found
  double stop_tol, neg_tol;
};

__global__ void k_pc_init(const double* __restrict__ A, int n, double tol, int* __restrict__ at,
                          double* __restrict__ d, PcCtl* ctl) {
  __shared__ double sv[32];
  double mx = -1e300;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    at[i] = i;
    d[i] = A[(size_t)i * n + i];
    mx = fmax(mx, d[i]);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m2 = sv[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m2 = fmax(m2, sv[w]);
    ctl->k = 0;
    ctl->stop = 0;
    ctl->stop_tol = tol * m2;
    ctl->neg_tol = -tol * fmax(m2, 1e-300);
  }
}

__global__ void __launch_bounds__(1024) k_pc_panel(const double* __restrict__ A, int n, int* __restrict__ atg,
                                                   double* __restrict__ dg, double* __restrict__ lc, PcCtl* ctl,
                                                   int* status) {
  extern __shared__ double pcs[];
  double* d = pcs;                                    // running diagonal by original index
  int* at = reinterpret_cast<int*>(d + n);            // original index at position
  __shared__ double sv[32];
  __shared__ int si[32];
  if (ctl->stop) return;
  const int k0 = ctl->k;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarp = nt >> 5;
  for (int i = tid; i < n; i += nt) { d[i] = dg[i]; at[i] = atg[i]; }
  __syncthreads();
  const double stop_tol = ctl->stop_tol, neg_tol = ctl->neg_tol;
  const int kend = min(n, k0 + kPcNB);
  int k = k0;
  bool stopped = false;
  for (; k < kend; ++k) {
    double bv = -1e300;
    int bi = n;
    for (int j = k + tid; j < n; j += nt) {
      const double v = d[at[j]];
      if (v > bv || (v == bv && j < bi)) { bv = v; bi = j; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
    __syncthreads();
    double v = sv[0];
    int b = si[0];
    for (int w = 1; w < nwarp; ++w)
      if (sv[w] > v || (sv[w] == v && si[w] < b)) { v = sv[w]; b = si[w]; }
    if (!(v > stop_tol)) {
      for (int j = k + tid; j < n; j += nt)
        if (d[at[j]] < neg_tol) atomicExch(status, 2);
      stopped = true;
      break;
    }
    const int q = at[b], qk = at[k];
    __syncthreads();
    if (tid == 0) { at[k] = q; at[b] = qk; }
    __syncthreads();
    const double l = sqrt(d[q]);
    const double* lq = lc + q;                        // L(q, k') at lc[k' n + q]
    for (int p = k + 1 + tid; p < n; p += nt) {
      const int a = at[p];
      double x = a > q ? A[(size_t)a * n + q] : A[(size_t)q * n + a];
      for (int kk = k0; kk < k; ++kk) x = fma(-lc[(size_t)kk * n + a], lq[(size_t)kk * n], x);
      const double Ls = x / l;
      lc[(size_t)k * n + a] = Ls;
      d[a] = fma(-Ls, Ls, d[a]);
    }
    if (tid == 0) lc[(size_t)k * n + q] = l;
    __syncthreads();
  }
  for (int i = tid; i < n; i += nt) { dg[i] = d[i]; atg[i] = at[i]; }
  if (tid == 0) {
    ctl->k = k;
    if (stopped || k == n) ctl->stop = 1;
  }
}

// trailing update of the remaining lower triangle with the panel [k0, k1):
// 64 x 64 tiles in ORIGINAL index space (coalesced), 4 x 4 entries per
// thread; entries of already pivoted rows/columns are skipped (done[] by
// original index, maintained here from at[]).
__global__ void __launch_bounds__(256) k_pc_trailing(double* __restrict__ A, int n, const int* __restrict__ at,
                                                     const double* __restrict__ lc, const PcCtl* ctl, int k0) {
  __shared__ double Lr[kPcNB][64], Lcs[kPcNB][64];
  __shared__ unsigned char done_r[64], done_c[64];
  const int k1 = ctl->k;               // pivots done after the panel
  if (k1 <= k0) return;                // nothing new (stopped before this panel)
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj > bi) return;
  const int r0 = bi * 64, c0 = bj * 64;
  const int tid = threadIdx.x;
  // pivoted originals: positions < k1
  for (int i = tid; i < 64; i += blockDim.x) { done_r[i] = 0; done_c[i] = 0; }
  __syncthreads();
  for (int p = tid; p < k1; p += blockDim.x) {
    const int a = at[p];
    if (a >= r0 && a < r0 + 64) done_r[a - r0] = 1;
    if (a >= c0 && a < c0 + 64) done_c[a - c0] = 1;
  }
  const int np = k1 - k0;
  for (int q = tid; q < kPcNB * 64; q += blockDim.x) {
    const int kk = q >> 6, i = q & 63;
    Lr[kk][i] = (kk < np && r0 + i < n) ? lc[(size_t)(k0 + kk) * n + r0 + i] : 0.0;
    Lcs[kk][i] = (kk < np && c0 + i < n) ? lc[(size_t)(k0 + kk) * n + c0 + i] : 0.0;
  }
  __syncthreads();
  const int tr = (tid >> 4) * 4, tcl = (tid & 15) * 4;
  double e[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int a = r0 + tr + u, b = c0 + tcl + v;
      e[u][v] = (a < n && b < n && a > b) ? A[(size_t)a * n + b] : 0.0;
    }
  for (int kk = 0; kk < np; ++kk) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) e[u][v] = fma(-Lr[kk][tr + u], Lcs[kk][tcl + v], e[u][v]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int a = r0 + tr + u, b = c0 + tcl + v;
      if (a < n && b < n && a > b && !done_r[tr + u] && !done_c[tcl + v]) A[(size_t)a * n + b] = e[u][v];
    }
}

// L in pivot order (column c < rank holds rows p >= c), perm and rank: the
// output layout of k_pivchol_coop1
__global__ void k_pc_finish(double* __restrict__ A, int n, const int* __restrict__ at, const double* __restrict__ lc,
                            const PcCtl* ctl, int* perm, int* rank_out) {
  const int k = ctl->k;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)k * n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(idx / n), p = (int)(idx % n);
    if (p >= c) A[(size_t)c * n + p] = lc[(size_t)c * n + at[p]];
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = at[i];
    if (threadIdx.x == 0) *rank_out = k;
  }
}

}  // namespace fg
