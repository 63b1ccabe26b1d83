// kernels_dmma.cuh -- FP64 tensor-core (DMMA) kernels.
//
// On sm_100a the FP64 tensor path is mma.sync.m8n8k4.f64 (SASS DMMA); tcgen05
// has no f64 kind.  K5: the block F-apply Q = F W for k
// search directions (Alg. 1 line 7) as one batched GEMM per subdomain with the
// B_s^T gather of W rows fused into the B-tile loader and the signed B_s
// scatter fused into the epilogue; FETI-DP's coarse correction rides along
// as n_c extra inner-dimension columns ([F_s | A_bc] [X_s ; U_s]).
#pragma once

#include "common.cuh"

namespace fg {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// --------------------------------------------------------- self test --
// C (8x8 row-major) = A (8x4 row-major) B (4x8 row-major) with the fragment
// layout a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// (c0, c1) = C[lane/4][2(lane%4) + {0,1}].
__global__ void k_dmma_selftest(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x & 31;
  double d0 = 0.0, d1 = 0.0;
  dmma_8x8x4(d0, d1, A[(lane >> 2) * 4 + (lane & 3)], B[(lane & 3) * 8 + (lane >> 2)]);
  C[(lane >> 2) * 8 + 2 * (lane & 3)] = d0;
  C[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = d1;
}

// ------------------------------------------------------- FP64 peaks --
// Sustained issue rate of independent DMMAs / DFMAs from registers.
__global__ void __launch_bounds__(256) k_peak_dmma(double* out, int iters) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[2 * i], acc[2 * i + 1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}
// Read-only HBM ceiling (fetigpu_hbm_read_peak): every thread keeps U 16-byte
// streaming loads in flight over a buffer much larger than L2.  The F-apply
// only reads its operator, and a read-only stream runs faster than the
// read + write copy MEASURED_PEAKS.json times (no bus turnarounds).
template <int U>
__global__ void __launch_bounds__(256) k_peak_read(const double2* __restrict__ p, size_t n, double* out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 1.2345e-300) out[0] = acc;   // never true on a zeroed buffer: keeps the loads alive
}

__global__ void __launch_bounds__(256) k_peak_dfma(double* out, int iters) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  const double a = 0.999999, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

// --------------------------------------------------- K5 block apply --
// Row-major blocks: W(i, c) = W[i * ldw + c].  Per subdomain s, tile
// (BM rows of F_s) x (BN columns of W), inner dimension n_s (+ n_c).
constexpr int kBM = 128, kBN = 64, kBK = 16;
constexpr int kApad = kBK + 4;   // 2 wavefronts per 8x4 A fragment load
constexpr int kBpad = kBN + 8;   // 2 wavefronts per 4x8 B fragment load
constexpr int kBlockSmem = (2 * kBM * kApad + 2 * kBK * kBpad) * 8;

struct BlockApplyArgs {
  const OpSub* subs;
  const double* mats;
  const int* rows;
  const double* coefs;
  int KR;
  const DpSub* dps;      // nullable (T-FETI)
  const double* abc;
  const int* cmap;
  const double* U;       // N_c x k row-major (coarse solution), nullable
  int ldu;
  const double* W;
  int ldw;
  double* Q;
  int ldq;
  int k;
  const int* order;      // nullable: subdomain processed by grid slice z (K5 dp2)
};

template <int KR>
__global__ void __launch_bounds__(256) k_block_apply(BlockApplyArgs a) {
  extern __shared__ __align__(16) double dsm[];
  double (*As)[kBM * kApad] = reinterpret_cast<double (*)[kBM * kApad]>(dsm);
  double (*Bs)[kBK * kBpad] = reinterpret_cast<double (*)[kBK * kBpad]>(dsm + 2 * kBM * kApad);
  const int s = blockIdx.z;
  const OpSub d = a.subs[s];
  const int ns = d.ns;
  const int nc = a.dps ? a.dps[s].nc : 0;
  const int kin = ns + nc;
  const int row0 = blockIdx.y * kBM;
  if (row0 >= ns) return;
  const int col0 = blockIdx.x * kBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1;         // 4 x 2 warps, warp tile 32 x 32
  const double* F = a.mats + d.moff;
  const int* rw = a.rows + d.map_off;
  const double* cf = a.coefs + d.map_off;
  const double* Abc = a.dps ? a.abc + a.dps[s].abc_off : nullptr;
  const int* cm = a.dps ? a.cmap + a.dps[s].cmap_off : nullptr;

  // tile loaders: A tile 128 x 16 (each thread 8 values), B tile 16 x 64 (4 values)
  double ra[8], rb[4];
  auto load_tiles = [&](int kk) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * 256;           // 0..2047
      const int r = idx >> 4, c = idx & 15;
      const int gi = row0 + r, gj = kk + c;
      double v = 0.0;
      if (gi < ns) {
        if (gj < ns) v = F[(size_t)gi * d.ld + gj];
        else if (gj < kin) v = Abc[(size_t)gi * nc + (gj - ns)];
      }
      ra[q] = v;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + q * 256;           // 0..1023
      const int r = idx >> 6, c = idx & 63;
      const int gj = kk + r, gc = col0 + c;
      double v = 0.0;
      if (gc < a.k) {
        if (gj < ns) {
#pragma unroll
          for (int t = 0; t < KR; ++t) {
            const int row = rw[gj * KR + t];
            if (row >= 0) v += cf[gj * KR + t] * a.W[(size_t)row * a.ldw + gc];
          }
        } else if (gj < kin) {
          v = a.U[(size_t)cm[gj - ns] * a.ldu + gc];
        }
      }
      rb[q] = v;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + q * 256;
      As[buf][(idx >> 4) * kApad + (idx & 15)] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + q * 256;
      Bs[buf][(idx >> 6) * kBpad + (idx & 63)] = rb[q];
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (kin + kBK - 1) / kBK;
  load_tiles(0);
  store_tiles(0);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) load_tiles((t + 1) * kBK);
    const double* A_ = As[buf];
    const double* B_ = Bs[buf];
#pragma unroll
    for (int k4 = 0; k4 < kBK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        af[i] = A_[(wr * 32 + i * 8 + (lane >> 2)) * kApad + k4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        bf[j] = B_[(k4 + (lane & 3)) * kBpad + wc * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (t + 1 < nk) store_tiles(buf ^ 1);
    __syncthreads();
  }
  // epilogue: signed scatter of rows into Q (exactly two contributions per
  // dual row overall -> order-independent atomics)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int li = row0 + wr * 32 + i * 8 + (lane >> 2);
    if (li >= ns) continue;
#pragma unroll
    for (int t = 0; t < KR; ++t) {
      const int row = rw[li * KR + t];
      if (row < 0) continue;
      const double c = cf[li * KR + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int gc = col0 + wc * 32 + j * 8 + 2 * (lane & 3);
        double* q = a.Q + (size_t)row * a.ldq + gc;
        if (gc < a.k) atomicAdd(q, c * acc[i][j][0]);
        if (gc + 1 < a.k) atomicAdd(q + 1, c * acc[i][j][1]);
      }
    }
  }
}

// --------------------- K5, FETI-DP fast path: cp.async multistage pipeline --
// Requires sign-folded operators (F'' = S F S, A'' = S A_bc with S = diag of
// the +-1 B_s entries; exact) so the gather/scatter are unsigned, KR = 1, and
// k, ldw, ldu even.  A tile rows (F'' rows / A'' rows) and B tile rows
// (W rows / U rows) are contiguous 16-byte chunks copied straight into shared
// memory; out-of-range chunks are zero-filled.
constexpr int kStages = 3;
constexpr int kAsyncSmem = (kStages * (kBM * kApad + kBK * kBpad)) * 8 + (512 + 16) * 4;

__global__ void __launch_bounds__(256, 2) k_block_apply_dp(BlockApplyArgs a) {
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                                   // kStages x (kBM x kApad)
  double* Bs = dsm + kStages * kBM * kApad;           // kStages x (kBK x kBpad)
  int* srow = reinterpret_cast<int*>(Bs + kStages * kBK * kBpad);
  const int s = blockIdx.z;
  const OpSub d = a.subs[s];
  const int ns = d.ns;
  const DpSub p = a.dps[s];
  const int nc = p.nc;
  const int kin = ns + nc;
  const int row0 = blockIdx.y * kBM;
  if (row0 >= ns) return;
  const int col0 = blockIdx.x * kBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1;
  const double* F = a.mats + d.moff;
  const double* Abc = a.abc + p.abc_off;
  const int* rw = a.rows + d.map_off;
  for (int j = tid; j < kin; j += 256) srow[j] = j < ns ? rw[j] : a.cmap[p.cmap_off + j - ns];
  __syncthreads();
  const int nk = (kin + kBK - 1) / kBK;
  auto issue = [&](int t) {
    const int kk = t * kBK, st = t % kStages;
    double* A_ = As + st * kBM * kApad;
    double* B_ = Bs + st * kBK * kBpad;
#pragma unroll
    for (int q = 0; q < 4; ++q) {        // A: 128 rows x 8 chunks
      const int idx = tid + q * 256;
      const int r = idx >> 3, c2 = (idx & 7) * 2;
      const int gi = row0 + r, gj = kk + c2;
      const double* src = F;
      bool ok = gi < ns && gj < kin;
      if (ok) src = gj < ns ? F + (size_t)gi * d.ld + gj : Abc + (size_t)gi * nc + (gj - ns);
      cp_async16(A_ + r * kApad + c2, src, ok);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {        // B: 16 rows x 32 chunks
      const int idx = tid + q * 256;
      const int r = idx >> 5, c2 = (idx & 31) * 2;
      const int gj = kk + r, gc = col0 + c2;
      const double* src = a.W;
      bool ok = gj < kin && gc < a.k;
      if (ok) src = gj < ns ? a.W + (size_t)srow[gj] * a.ldw + gc : a.U + (size_t)srow[gj] * a.ldu + gc;
      cp_async16(B_ + r * kBpad + c2, src, ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int t = 0; t < kStages - 1; ++t) {
    if (t < nk) issue(t);
    cp_async_commit();
  }
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (t + kStages - 1 < nk) issue(t + kStages - 1);
    cp_async_commit();
    const double* A_ = As + (t % kStages) * kBM * kApad;
    const double* B_ = Bs + (t % kStages) * kBK * kBpad;
#pragma unroll
    for (int k4 = 0; k4 < kBK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = A_[(wr * 32 + i * 8 + (lane >> 2)) * kApad + k4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = B_[(k4 + (lane & 3)) * kBpad + wc * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  // unsigned scatter: two contributions per dual row -> order-independent
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int li = row0 + wr * 32 + i * 8 + (lane >> 2);
    if (li >= ns) continue;
    double* qrow = a.Q + (size_t)srow[li] * a.ldq;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = col0 + wc * 32 + j * 8 + 2 * (lane & 3);
      if (gc < a.k) atomicAdd(qrow + gc, acc[i][j][0]);
      if (gc + 1 < a.k) atomicAdd(qrow + gc + 1, acc[i][j][1]);
    }
  }
}

// K5, FETI-DP fast path, templated tile: BM x BN CTA tile of 32 x 32 warp
// tiles, BK-deep k steps in an ST-stage cp.async ring (same operand layouts
// and arithmetic order per output element as k_block_apply_dp: the k loop
// runs over [F''_s | A''_s] columns in ascending order).  The dense-algebra
// sweep (profiles/r02_gemm_sweep.log) found 64 x 64 tiles with 3-4 resident
// CTAs per SM keep the DMMA pipe busiest.
template <int BM, int BN, int BK, int ST>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32) k_block_apply_dp2(BlockApplyArgs a) {
  constexpr int THREADS = (BM / 32) * (BN / 32) * 32;
  constexpr int AP = BK + 4, BP = BN + 8;
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                                   // ST x (BM x AP)
  double* Bs = dsm + ST * BM * AP;                    // ST x (BK x BP)
  int* srow = reinterpret_cast<int*>(Bs + ST * BK * BP);
  const int s = a.order ? a.order[blockIdx.z] : blockIdx.z;
  const OpSub d = a.subs[s];
  const int ns = d.ns;
  const int row0 = blockIdx.y * BM;
  if (row0 >= ns) return;
  const DpSub p = a.dps[s];
  const int nc = p.nc;
  const int kin = ns + nc;
  const int col0 = blockIdx.x * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int WGN = BN / 32;
  const int wr = warp / WGN, wc = warp % WGN;
  const double* F = a.mats + d.moff;
  const double* Abc = a.abc + p.abc_off;
  const int* rw = a.rows + d.map_off;
  for (int j = tid; j < kin; j += THREADS) srow[j] = j < ns ? rw[j] : a.cmap[p.cmap_off + j - ns];
  __syncthreads();
  const int nk = (kin + BK - 1) / BK;
  auto issue = [&](int t) {
    const int kk = t * BK, st = t % ST;
    double* A_ = As + st * BM * AP;
    double* B_ = Bs + st * BK * BP;
    constexpr int ACH = BM * (BK / 2), BCH = BK * (BN / 2);
#pragma unroll
    for (int q = 0; q < (ACH + THREADS - 1) / THREADS; ++q) {
      const int idx = tid + q * THREADS;
      if (ACH % THREADS == 0 || idx < ACH) {
        const int r = idx / (BK / 2), c2 = (idx % (BK / 2)) * 2;
        const int gi = row0 + r, gj = kk + c2;
        const double* src = F;
        const bool ok = gi < ns && gj < kin;
        if (ok) src = gj < ns ? F + (size_t)gi * d.ld + gj : Abc + (size_t)gi * nc + (gj - ns);
        cp_async16(A_ + r * AP + c2, src, ok);
      }
    }
#pragma unroll
    for (int q = 0; q < (BCH + THREADS - 1) / THREADS; ++q) {
      const int idx = tid + q * THREADS;
      if (BCH % THREADS == 0 || idx < BCH) {
        const int r = idx / (BN / 2), c2 = (idx % (BN / 2)) * 2;
        const int gj = kk + r, gc = col0 + c2;
        const double* src = a.W;
        const bool ok = gj < kin && gc < a.k;
        if (ok) src = gj < ns ? a.W + (size_t)srow[gj] * a.ldw + gc : a.U + (size_t)srow[gj] * a.ldu + gc;
        cp_async16(B_ + r * BP + c2, src, ok);
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int t = 0; t < ST - 1; ++t) {
    if (t < nk) issue(t);
    cp_async_commit();
  }
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    if (t + ST - 1 < nk) issue(t + ST - 1);
    cp_async_commit();
    const double* A_ = As + (t % ST) * BM * AP;
    const double* B_ = Bs + (t % ST) * BK * BP;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = A_[(wr * 32 + i * 8 + (lane >> 2)) * AP + k4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = B_[(k4 + (lane & 3)) * BP + wc * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int li = row0 + wr * 32 + i * 8 + (lane >> 2);
    if (li >= ns) continue;
    double* qrow = a.Q + (size_t)srow[li] * a.ldq;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = col0 + wc * 32 + j * 8 + 2 * (lane & 3);
      if (gc < a.k) atomicAdd(qrow + gc, acc[i][j][0]);
      if (gc + 1 < a.k) atomicAdd(qrow + gc + 1, acc[i][j][1]);
    }
  }
}
template <int BM, int BN, int BK, int ST>
constexpr size_t k5_smem(int kin_max) {
  return (size_t)ST * (BM * (BK + 4) + BK * (BN + 8)) * 8 + (size_t)kin_max * 4;
}

// FETI-DP coarse pre-pass for a block: T_s = A_bc^T (B_s^T W)   (n_c x k).
// One CTA per (128-column slab, subdomain): the subdomain's A_bc rows (padded
// to 8), row ids and coefficients are staged in shared memory once, so the
// only global stream is W (two adjacent columns per thread, 16-byte loads).
// 4 thread groups split the rows; per column the partial sums are combined
// in group order -- the accumulation order of the 64-column version, so
// results are unchanged.
constexpr int kDpTCols = 128;
__global__ void __launch_bounds__(256) k_block_dp_t(const OpSub* __restrict__ subs,
                                                    const DpSub* __restrict__ dps,
                                                    const int* __restrict__ rows,
                                                    const double* __restrict__ coefs,
                                                    const double* __restrict__ abc,
                                                    const double* __restrict__ W, int ldw, int k,
                                                    double* __restrict__ tbuf, int ldt,
                                                    const int* __restrict__ order = nullptr) {
  // (coefs are the apply coefficients: unit when the operators are sign-folded;
  // order: K5's 4 x 4-module subdomain walk, so both owners of a dual row read
  // its W row close in time -- the second read hits L2)
  extern __shared__ double dsm[];
  const int s = order ? order[blockIdx.y] : blockIdx.y;
  const OpSub d = subs[s];
  const DpSub p = dps[s];
  const int ns = d.ns;
  double* As = dsm;                                   // max(ns * 8, 4 * 8 * kDpTCols): A, then partials
  double* cs = As + max(ns * 8, 4 * 8 * kDpTCols);    // ns coefficients
  int* rs = reinterpret_cast<int*>(cs + ns);          // ns row ids
  const double* Ab = abc + p.abc_off;
  for (int idx = threadIdx.x; idx < ns * 8; idx += blockDim.x) {
    const int j = idx >> 3, c = idx & 7;
    As[idx] = c < p.nc ? Ab[(size_t)j * p.nc + c] : 0.0;
  }
  for (int j = threadIdx.x; j < ns; j += blockDim.x) {
    rs[j] = rows[d.map_off + j];
    cs[j] = coefs[d.map_off + j];
  }
  __syncthreads();
  const int lc = 2 * (threadIdx.x & 63);             // local column pair
  const int col = blockIdx.x * kDpTCols + lc;
  const int grp = threadIdx.x >> 6;                  // 4 groups split the rows
  const bool vec = (ldw & 1) == 0 && col + 1 < k;
  double a0[8] = {}, a1[8] = {};
  if (col < k) {
    auto loadw = [&](int j, double& w0, double& w1) {
      const int r = rs[j];
      w0 = 0.0;
      w1 = 0.0;
      if (r >= 0) {
        const double* wr = W + (size_t)r * ldw + col;
        if (vec) {
          const double2 w = __ldg(reinterpret_cast<const double2*>(wr));
          w0 = w.x;
          w1 = w.y;
        } else {
          w0 = wr[0];
          w1 = col + 1 < k ? wr[1] : 0.0;
        }
      }
    };
    auto accum = [&](int j, double w0, double w1) {
      const double x0 = cs[j] * w0, x1 = cs[j] * w1;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const double av = As[j * 8 + c];
        a0[c] = fma(av, x0, a0[c]);
        a1[c] = fma(av, x1, a1[c]);
      }
    };
    // four W rows in flight per thread, accumulated in row order (the
    // single-row loop's order: bit-identical; it waited on every load)
    int j = grp;
    for (; j + 12 < ns; j += 16) {
      double w[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) loadw(j + 4 * u, w[u][0], w[u][1]);
#pragma unroll
      for (int u = 0; u < 4; ++u) accum(j + 4 * u, w[u][0], w[u][1]);
    }
    for (; j < ns; j += 4) {
      double w0, w1;
      loadw(j, w0, w1);
      accum(j, w0, w1);
    }
  }
  __syncthreads();  // A no longer needed: its space holds the group partials
  double* red = As;  // [4][8][kDpTCols]
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    red[(grp * 8 + c) * kDpTCols + lc] = a0[c];
    red[(grp * 8 + c) * kDpTCols + lc + 1] = a1[c];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < p.nc * kDpTCols; idx += blockDim.x) {
    const int c = idx / kDpTCols, l = idx - c * kDpTCols;
    const int gc = blockIdx.x * kDpTCols + l;
    if (gc < k)
      tbuf[(size_t)(p.t_off + c) * ldt + gc] = red[(0 * 8 + c) * kDpTCols + l] + red[(1 * 8 + c) * kDpTCols + l] +
                                                red[(2 * 8 + c) * kDpTCols + l] + red[(3 * 8 + c) * kDpTCols + l];
  }
}

// coarse block assembly in ascending subdomain order: T(i, :) = sum_owners tbuf
__global__ void k_coarse_gather_block(const int* __restrict__ optr, const int* __restrict__ oidx,
                                      const double* __restrict__ tbuf, int ldt, int nc, int k,
                                      double* __restrict__ out, int ldo) {
  const int i = blockIdx.y;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int q = optr[i]; q < optr[i + 1]; ++q) v += tbuf[(size_t)oidx[q] * ldt + c];
    out[(size_t)i * ldo + c] = v;
  }
}

}  // namespace fg

namespace fg {

// ---------------- K5z: block F-apply of a fresh preconditioner block ------
// Q = F Z where Z (row-major m x k, k = N_s) holds the per-subdomain
// preconditioner columns of Alg. 1 lines 2/16: column s is nonzero only on
// the dual rows of subdomain s.  B_t^T Z therefore has, per local row a of
// subdomain t, exactly two nonzero columns: t itself and the other owner o(a)
// of that row -- at most 5 distinct columns per subdomain (itself and its
// edge neighbours; FETI-DP corners are primal).  The local products shrink
// from n_t x k to n_t x 5 (K5z-1), the coarse term keeps its dense form
// (U = Kbar^{-1} T, DMMA GEMM), and Q is written once per dual row from both
// owners' contributions in a fixed order (K5z-2): no memset, no atomics.
constexpr int kZNb = 5;   // neighbour slots per subdomain (slot 0: itself)

// K5z-1, one CTA per subdomain t: Y_t = F''_t X_t (n_t x 5, packed at the
// op-map positions) and the coarse pre-pass T_t = A''_t^T X_t into the tbuf
// rows of t at the 5 neighbour columns (tbuf zeroed by the caller).
__global__ void __launch_bounds__(256) k_bz_local(const OpSub* __restrict__ subs, const DpSub* __restrict__ dps,
                                                  const double* __restrict__ mats, const int* __restrict__ rows,
                                                  const double* __restrict__ abc, const int* __restrict__ other,
                                                  const int* __restrict__ jslot, const int* __restrict__ nbr,
                                                  const double* __restrict__ Z, int k, double* __restrict__ Y,
                                                  double* __restrict__ tbuf, int ldt, double* __restrict__ tt) {
  extern __shared__ double bzs[];
  const int t = blockIdx.x;
  const OpSub d = subs[t];
  const DpSub p = dps[t];
  const int ns = d.ns;
  double* xt = bzs;                 // Z(r_a, t)
  double* xo = bzs + ns;            // Z(r_a, o(a))
  int* jo = reinterpret_cast<int*>(bzs + 2 * ns);
  for (int a = threadIdx.x; a < ns; a += blockDim.x) {
    const int r = rows[d.map_off + a];
    const int o = other[d.map_off + a];
    xt[a] = r >= 0 ? Z[(size_t)r * k + t] : 0.0;
    xo[a] = (r >= 0 && o >= 0) ? Z[(size_t)r * k + o] : 0.0;
    jo[a] = jslot[d.map_off + a];
  }
  __syncthreads();
  const double* F = mats + d.moff;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = warp; b < ns; b += 8) {
    const double* fr = F + (size_t)b * d.ld;      // row b of the symmetric F''_t = column b
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    for (int a = lane; a < ns; a += 32) {
      const double f = fr[a];
      a0 = fma(f, xt[a], a0);
      const double v = f * xo[a];
      const int j = jo[a];
      if (j == 1) a1 += v;
      else if (j == 2) a2 += v;
      else if (j == 3) a3 += v;
      else if (j == 4) a4 += v;
    }
    a0 = warp_sum(a0); a1 = warp_sum(a1); a2 = warp_sum(a2); a3 = warp_sum(a3); a4 = warp_sum(a4);
    if (lane == 0) {
      double* y = Y + (size_t)(d.map_off + b) * kZNb;
      y[0] = a0; y[1] = a1; y[2] = a2; y[3] = a3; y[4] = a4;
    }
  }
  // T_t(c, j) = sum_a A''(a, c) X(a, j), one thread per (c, j)
  const double* A = abc + p.abc_off;
  for (int q = threadIdx.x; q < p.nc * kZNb; q += blockDim.x) {
    const int c = q / kZNb, j = q - c * kZNb;
    const int s = nbr[t * kZNb + j];
    if (s < 0) continue;
    double acc = 0.0;
    for (int a = 0; a < ns; ++a) {
      const double x = j == 0 ? xt[a] : (jo[a] == j ? xo[a] : 0.0);
      acc = fma(A[(size_t)a * p.nc + c], x, acc);
    }
    tbuf[(size_t)(p.t_off + c) * ldt + s] = acc;
    if (tt) tt[(size_t)(p.t_off + c) * kZNb + j] = acc;   // compact copy (line-7 correction)
  }
}

// One group of dual rows shared by the same two subdomains (an interface
// edge), at most kBzRows rows: entry e of the group is dual row rows[e] at
// local position b1[e] of t1 and b2[e] of t2 (t2 < 0: single owner).
struct BzEdge {
  int t1, t2, e0, cnt;
};
constexpr int kBzRows = 128;
constexpr int kBzCols = 256;

// K5z-2: Q(r, s) = [Y_t1(b1, j1(s)) + A''_t1(b1, :) U_t1(:, s)]
//                + [Y_t2(b2, j2(s)) + A''_t2(b2, :) U_t2(:, s)]
// for every column s; one CTA per (edge group, 256-column tile), one column
// per thread, Q rows written once (coalesced, no atomics).
__global__ void __launch_bounds__(kBzCols) k_bz_edges(const BzEdge* __restrict__ edges, const int* __restrict__ erow,
                                                      const int* __restrict__ eb1, const int* __restrict__ eb2,
                                                      const OpSub* __restrict__ subs, const DpSub* __restrict__ dps,
                                                      const double* __restrict__ abc, const int* __restrict__ cmap,
                                                      const int* __restrict__ nbr, const double* __restrict__ Y,
                                                      const double* __restrict__ U, int k, double* __restrict__ Q) {
  __shared__ double A1[kBzRows][8], A2[kBzRows][8], Y1[kBzRows][kZNb], Y2[kBzRows][kZNb];
  __shared__ int R[kBzRows];
  const BzEdge e = edges[blockIdx.y];
  const DpSub p1 = dps[e.t1];
  const DpSub p2 = e.t2 >= 0 ? dps[e.t2] : DpSub{0, 0, 0, 0, 0};
  const OpSub d1 = subs[e.t1];
  const OpSub d2 = e.t2 >= 0 ? subs[e.t2] : OpSub{0, 0, 0, 0, 0};
  for (int q = threadIdx.x; q < e.cnt * 8; q += blockDim.x) {
    const int i = q >> 3, c = q & 7;
    const int b1 = eb1[e.e0 + i], b2 = eb2[e.e0 + i];
    A1[i][c] = c < p1.nc ? abc[p1.abc_off + (size_t)b1 * p1.nc + c] : 0.0;
    A2[i][c] = (e.t2 >= 0 && c < p2.nc) ? abc[p2.abc_off + (size_t)b2 * p2.nc + c] : 0.0;
  }
  for (int q = threadIdx.x; q < e.cnt * kZNb; q += blockDim.x) {
    const int i = q / kZNb, j = q - i * kZNb;
    Y1[i][j] = Y[(size_t)(d1.map_off + eb1[e.e0 + i]) * kZNb + j];
    Y2[i][j] = e.t2 >= 0 ? Y[(size_t)(d2.map_off + eb2[e.e0 + i]) * kZNb + j] : 0.0;
  }
  for (int i = threadIdx.x; i < e.cnt; i += blockDim.x) R[i] = erow[e.e0 + i];
  __syncthreads();
  const int s = blockIdx.x * kBzCols + threadIdx.x;
  if (s >= k) return;
  int j1 = -1, j2 = -1;
#pragma unroll
  for (int j = 0; j < kZNb; ++j) {
    if (nbr[e.t1 * kZNb + j] == s) j1 = j;
    if (e.t2 >= 0 && nbr[e.t2 * kZNb + j] == s) j2 = j;
  }
  double u1[8], u2[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    u1[c] = c < p1.nc ? U[(size_t)cmap[p1.cmap_off + c] * k + s] : 0.0;
    u2[c] = (e.t2 >= 0 && c < p2.nc) ? U[(size_t)cmap[p2.cmap_off + c] * k + s] : 0.0;
  }
  for (int i = 0; i < e.cnt; ++i) {
    double v1 = j1 >= 0 ? Y1[i][j1] : 0.0;
    double v2 = j2 >= 0 ? Y2[i][j2] : 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      v1 = fma(A1[i][c], u1[c], v1);
      v2 = fma(A2[i][c], u2[c], v2);
    }
    Q[(size_t)R[i] * k + s] = v1 + v2;
  }
}

}  // namespace fg

namespace fg {

// CGS update of the implicit RRS store (Alg. 1 line 20 on coordinates),
// V(r, c) -= sum_l ZV_l(r) N^T(c, l k + t1) + sum_l ZV_l(r) N^T(c, l k + t2)
// for dual row r shared by t1 < t2, computed once per row (interface-edge
// groups as in K5z-2): no zeroed m x k buffer, no atomics, no separate AXPY.
// The arithmetic is that of the zero / atomic-scatter / AXPY sequence it
// replaces: each owner's sum over l is one fma chain in ascending l, the two
// owner sums are added (0 + a + b == a + b), and V = fma(-1, D, V).
// Requires nl <= kZsMax coordinates blocks (the caller falls back otherwise).
constexpr int kZsMax = 32;
constexpr int kZsChunk = 8;     // rows accumulated in registers at a time
__global__ void __launch_bounds__(kBzCols) k_rrs_zsub_edges(const BzEdge* __restrict__ edges,
                                                            const int* __restrict__ erow,
                                                            const int* __restrict__ ez1, const int* __restrict__ ez2,
                                                            const double* __restrict__ ZV, long long nz, int nl,
                                                            const double* __restrict__ NT, int k,
                                                            double* __restrict__ V) {
  extern __shared__ double zsm[];            // [cnt][nl] owner 1, then [cnt][nl] owner 2
  __shared__ int R[kBzRows];
  const BzEdge e = edges[blockIdx.y];
  double* z1 = zsm;
  double* z2 = zsm + (size_t)e.cnt * nl;
  for (int q = threadIdx.x; q < e.cnt * nl; q += blockDim.x) {
    const int i = q / nl, l = q - i * nl;
    z1[i * nl + l] = ZV[(size_t)l * nz + ez1[e.e0 + i]];
    z2[i * nl + l] = e.t2 >= 0 ? ZV[(size_t)l * nz + ez2[e.e0 + i]] : 0.0;
  }
  for (int i = threadIdx.x; i < e.cnt; i += blockDim.x) R[i] = erow[e.e0 + i];
  __syncthreads();
  const int c = blockIdx.x * kBzCols + threadIdx.x;
  if (c >= k) return;
  const double* N1 = NT + (size_t)e.t1 * k + c;
  const double* N2 = e.t2 >= 0 ? NT + (size_t)e.t2 * k + c : nullptr;
  const size_t lstep = (size_t)k * k;
  // chunks of kZsChunk rows: accumulators in registers, l outer (each
  // owner's sum stays one fma chain in ascending l), then the rows' V loads
  // are issued together and V = fma(-1, p1 + p2, V)
  for (int i0 = 0; i0 < e.cnt; i0 += kZsChunk) {
    double a1[kZsChunk], a2[kZsChunk];
#pragma unroll
    for (int u = 0; u < kZsChunk; ++u) a1[u] = a2[u] = 0.0;
    for (int l = 0; l < nl; ++l) {
      const double n1 = N1[l * lstep], n2 = N2 ? N2[l * lstep] : 0.0;
#pragma unroll
      for (int u = 0; u < kZsChunk; ++u) {
        const int i = min(i0 + u, e.cnt - 1);
        a1[u] = fma(z1[i * nl + l], n1, a1[u]);
        a2[u] = fma(z2[i * nl + l], n2, a2[u]);
      }
    }
    double v[kZsChunk];
#pragma unroll
    for (int u = 0; u < kZsChunk; ++u) v[u] = i0 + u < e.cnt ? V[(size_t)R[i0 + u] * k + c] : 0.0;
#pragma unroll
    for (int u = 0; u < kZsChunk; ++u)
      if (i0 + u < e.cnt) V[(size_t)R[i0 + u] * k + c] = fma(-1.0, a1[u] + a2[u], v[u]);
  }
}

}  // namespace fg

namespace fg {

// Alg. 1 line 7 without a block F-apply.  After the two CGS passes the new
// block is V2 = V1 - Zhat N2, and the second pass already applied F to V1
// (Qb = F V1).  With F Z_l kept from each Z block's K5z apply -- its sparse
// part Y_l (n_t x 5 per subdomain) and its coarse pre-pass T_l -- linearity
// gives F V2 = F V1 - sum_l (F Z_l) N2[l], where N2 is the second pass's
// (roundoff-sized) correction, so the subtraction costs no accuracy.  The
// coarse part enters as U_c = Kbar^{-1} sum_l T_l N2[l] (GEMMs, caller);
// this kernel subtracts, per dual row r shared by t1 < t2 (interface-edge
// groups), the two owners' terms
//   p_o(c) = sum_l sum_j Y_l,to(b_o, j) N2^T(c, l k + nbr_to(j)) + A''_to(b_o, :) U_c(cmap_to, c)
// as Q(r, c) = fma(-1, p1 + p2, Q(r, c)).  CTA = (edge group, 32 columns),
// warp w takes rows w, w + 8, ..; the N2 values of the two owners' five
// neighbour columns and the U_c rows are staged in shared memory.
// Coarse part of the correction: T_c^T(c, p) = sum_l sum_{owners t of p}
// sum_j tt_l(t_off(t) + cp, j) N2^T(c, l k + nbr_t(j)) -- T_l kept in its
// compact per-subdomain form (n_c x 5 per t: A''_t^T X_l,t) instead of the
// dense N_c x k matrix.  Owners in the fixed (ascending) order of the coarse
// gather.  Grid (column tiles, N_c); output column-major k x N_c.
__global__ void k_fz_coarse(const int* __restrict__ optr, const int* __restrict__ osub,
                            const int* __restrict__ orow, const int* __restrict__ nbr, const double* __restrict__ tt,
                            long long ttstride, int nl, const double* __restrict__ NT, int k,
                            double* __restrict__ TcT) {
  const int p = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  double acc = 0.0;
  for (int q = optr[p]; q < optr[p + 1]; ++q) {
    const int t = osub[q], row = orow[q];
    for (int l = 0; l < nl; ++l) {
      const double* tl = tt + (size_t)l * ttstride + (size_t)row * kZNb;
#pragma unroll
      for (int j = 0; j < kZNb; ++j) {
        const int s = nbr[t * kZNb + j];
        if (s >= 0) acc = fma(tl[j], NT[((size_t)l * k + s) * k + c], acc);
      }
    }
  }
  TcT[(size_t)p * k + c] = acc;
}

constexpr int kFzCols = 64;     // columns per CTA
constexpr int kFzRows = 64;     // rows per CTA (edge groups are split over grid.z)
constexpr int kFzL = 2;         // coordinate blocks staged per step
// 256 threads: thread (columns tc, tc + 32; row slice tq = tid / 32) owns the
// rows tq, tq + 8, .. (8 rows x 2 columns per owner); per staged coordinate
// column the four N2 values sit in registers and the Y entries of the rows
// come from shared memory (warp broadcast): 20 shared loads per 32 FMAs.  The coarse rows A''(b, :) and
// the U_c columns are staged as well.
__global__ void __launch_bounds__(256, 2) k_fz_correct(const BzEdge* __restrict__ edges, const int* __restrict__ erow,
                                                    const int* __restrict__ eb1, const int* __restrict__ eb2,
                                                    const OpSub* __restrict__ subs, const DpSub* __restrict__ dps,
                                                    const double* __restrict__ abc, const int* __restrict__ cmap,
                                                    const int* __restrict__ nbr, const double* __restrict__ Yst,
                                                    long long ystride, int nl, const double* __restrict__ NT,
                                                    const double* __restrict__ Uc, int k, double* __restrict__ Q) {
  __shared__ double ys[2][kFzRows][kFzL * kZNb];      // 10 KB
  __shared__ double ns[2][kFzL * kZNb][kFzCols];      // 10 KB
  __shared__ double as[2][kFzRows][8], us[2][8][kFzCols];
  __shared__ int rb[2][kFzRows];
  const BzEdge e = edges[blockIdx.y];
  const int r0 = blockIdx.z * kFzRows;
  if (r0 >= e.cnt) return;
  const int cnt = min(kFzRows, e.cnt - r0);
  const int c0 = blockIdx.x * kFzCols;
  const int tt[2] = {e.t1, e.t2};
  const OpSub d1 = subs[e.t1];
  const OpSub d2 = e.t2 >= 0 ? subs[e.t2] : OpSub{0, 0, 0, 0, 0};
  const DpSub p1d = dps[e.t1];
  const DpSub p2d = e.t2 >= 0 ? dps[e.t2] : DpSub{0, 0, 0, 0, 0};
  const int tid = threadIdx.x, tc = tid % 32, tq = tid / 32;
  for (int i = tid; i < kFzRows; i += blockDim.x) {
    rb[0][i] = i < cnt ? d1.map_off + eb1[e.e0 + r0 + i] : 0;
    rb[1][i] = (i < cnt && e.t2 >= 0) ? d2.map_off + eb2[e.e0 + r0 + i] : 0;
  }
  for (int q = tid; q < 2 * kFzRows * 8; q += blockDim.x) {
    const int cc = q % 8, i = (q / 8) % kFzRows, o = q / (8 * kFzRows);
    const DpSub pd = o == 0 ? p1d : p2d;
    const int b = (o == 0 ? (i < cnt ? eb1[e.e0 + r0 + i] : 0) : (i < cnt && e.t2 >= 0 ? eb2[e.e0 + r0 + i] : 0));
    as[o][i][cc] = (i < cnt && cc < pd.nc && (o == 0 || e.t2 >= 0)) ? abc[pd.abc_off + (size_t)b * pd.nc + cc] : 0.0;
  }
  for (int q = tid; q < 2 * 8 * kFzCols; q += blockDim.x) {
    const int c = q % kFzCols, cc = (q / kFzCols) % 8, o = q / (kFzCols * 8);
    const DpSub pd = o == 0 ? p1d : p2d;
    us[o][cc][c] = ((o == 0 || e.t2 >= 0) && cc < pd.nc && c0 + c < k)
                       ? Uc[(size_t)cmap[pd.cmap_off + cc] * k + c0 + c] : 0.0;
  }
  double a1[kFzRows / 8][2], a2[kFzRows / 8][2];
#pragma unroll
  for (int u = 0; u < kFzRows / 8; ++u) a1[u][0] = a1[u][1] = a2[u][0] = a2[u][1] = 0.0;
  for (int l0 = 0; l0 < nl; l0 += kFzL) {
    const int lc = min(kFzL, nl - l0);
    __syncthreads();
    // staging with all of a thread's loads in flight before its stores
    constexpr int NY = 2 * kFzRows * kFzL * kZNb / 256, NN = 2 * kFzL * kZNb * kFzCols / 256;
    double yv[NY], nv[NN];
#pragma unroll
    for (int w = 0; w < NY; ++w) {
      const int q = tid + w * 256;
      const int j = q % kZNb, l = (q / kZNb) % kFzL, i = (q / (kZNb * kFzL)) % kFzRows,
                o = q / (kZNb * kFzL * kFzRows);
      yv[w] = (i < cnt && l < lc && (o == 0 || e.t2 >= 0))
                  ? __ldg(Yst + (size_t)(l0 + l) * ystride + (size_t)rb[o][i] * kZNb + j) : 0.0;
    }
#pragma unroll
    for (int w = 0; w < NN; ++w) {
      const int q = tid + w * 256;
      const int c = q % kFzCols, j = (q / kFzCols) % kZNb, l = (q / (kFzCols * kZNb)) % kFzL,
                o = q / (kFzCols * kZNb * kFzL);
      const int t = tt[o];
      const int sdm = t >= 0 ? nbr[t * kZNb + j] : -1;
      nv[w] = (sdm >= 0 && l < lc && c0 + c < k) ? __ldg(NT + ((size_t)(l0 + l) * k + sdm) * k + c0 + c) : 0.0;
    }
#pragma unroll
    for (int w = 0; w < NY; ++w) {
      const int q = tid + w * 256;
      const int j = q % kZNb, l = (q / kZNb) % kFzL, i = (q / (kZNb * kFzL)) % kFzRows,
                o = q / (kZNb * kFzL * kFzRows);
      ys[o][i][l * kZNb + j] = yv[w];
    }
#pragma unroll
    for (int w = 0; w < NN; ++w) {
      const int q = tid + w * 256;
      const int c = q % kFzCols, j = (q / kFzCols) % kZNb, l = (q / (kFzCols * kZNb)) % kFzL,
                o = q / (kFzCols * kZNb * kFzL);
      ns[o][l * kZNb + j][c] = nv[w];
    }
    __syncthreads();
    for (int q = 0; q < lc * kZNb; ++q) {
      const double n1a = ns[0][q][tc], n1b = ns[0][q][tc + 32], n2a = ns[1][q][tc], n2b = ns[1][q][tc + 32];
#pragma unroll
      for (int u = 0; u < kFzRows / 8; ++u) {
        const double y1 = ys[0][tq + 8 * u][q], y2 = ys[1][tq + 8 * u][q];
        a1[u][0] = fma(y1, n1a, a1[u][0]);
        a1[u][1] = fma(y1, n1b, a1[u][1]);
        a2[u][0] = fma(y2, n2a, a2[u][0]);
        a2[u][1] = fma(y2, n2b, a2[u][1]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int cl = tc + 32 * h, c = c0 + cl;
    if (c >= k) continue;
    double qv[kFzRows / 8];
#pragma unroll
    for (int u = 0; u < kFzRows / 8; ++u) {
      const int i = tq + 8 * u;
      qv[u] = i < cnt ? Q[(size_t)erow[e.e0 + r0 + i] * k + c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kFzRows / 8; ++u) {
      const int i = tq + 8 * u;
      if (i >= cnt) continue;
      double x1 = a1[u][h], x2 = a2[u][h];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        x1 = fma(as[0][i][cc], us[0][cc][cl], x1);
        x2 = fma(as[1][i][cc], us[1][cc][cl], x2);
      }
      Q[(size_t)erow[e.e0 + r0 + i] * k + c] = fma(-1.0, x1 + x2, qv[u]);
    }
  }
}

// DMMA form of k_fz_correct: per (edge group, 64 rows, 64 columns) the
// correction is a small GEMM  Q[rows, cols] -= A (rows x K) B (K x cols) with
// K = 10 nl (both owners' Y_l entries against the N2 rows of their neighbour
// slots) + 16 (A''(b, :) against the U_c rows of their primal DOFs).  A is
// gathered element-wise and B row-wise (16-byte) with cp.async into a 2-stage
// ring; 4 warps of 32 x 32 on mma.sync.m8n8k4.f64.  The sum over K runs in DMMA
// order (not the fma chain of k_fz_correct): equal to it up to rounding.
constexpr int kFmBM = 64, kFmBN = 64, kFmBK = 16;
__global__ void __launch_bounds__(128) k_fz_correct_mma(const BzEdge* __restrict__ edges,
                                                        const int* __restrict__ erow, const int* __restrict__ eb1,
                                                        const int* __restrict__ eb2, const OpSub* __restrict__ subs,
                                                        const DpSub* __restrict__ dps, const double* __restrict__ abc,
                                                        const int* __restrict__ cmap, const int* __restrict__ nbr,
                                                        const double* __restrict__ Yst, long long ystride, int nl,
                                                        const double* __restrict__ NT, const double* __restrict__ Uc,
                                                        int k, double* __restrict__ Q) {
  constexpr int AP = kFmBK + 4, BP = kFmBN + 8;
  __shared__ __align__(16) double As[2][kFmBM * AP];
  __shared__ __align__(16) double Bs[2][kFmBK * BP];
  __shared__ long long arow[2][kFmBM];     // Y row offsets (map_off + b) * 5 per owner, -1 if none
  __shared__ long long aabc[2][kFmBM];     // A'' row offsets per owner
  __shared__ int R[kFmBM];
  const BzEdge e = edges[blockIdx.y];
  const int r0 = blockIdx.z * kFmBM;
  if (r0 >= e.cnt) return;
  const int cnt = min(kFmBM, e.cnt - r0);
  const int c0 = blockIdx.x * kFmBN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1;
  const int tt[2] = {e.t1, e.t2};
  DpSub pd[2];
  pd[0] = dps[e.t1];
  pd[1] = e.t2 >= 0 ? dps[e.t2] : DpSub{0, 0, 0, 0, 0};
  for (int i = tid; i < kFmBM; i += blockDim.x) {
    const bool ok = i < cnt;
    const int b1 = ok ? eb1[e.e0 + r0 + i] : 0, b2 = ok ? eb2[e.e0 + r0 + i] : 0;
    arow[0][i] = ok ? (long long)(subs[e.t1].map_off + b1) * kZNb : -1;
    arow[1][i] = (ok && e.t2 >= 0) ? (long long)(subs[e.t2].map_off + b2) * kZNb : -1;
    aabc[0][i] = ok ? pd[0].abc_off + (long long)b1 * pd[0].nc : -1;
    aabc[1][i] = (ok && e.t2 >= 0) ? pd[1].abc_off + (long long)b2 * pd[1].nc : -1;
    R[i] = ok ? erow[e.e0 + r0 + i] : 0;
  }
  __syncthreads();
  const int Ky = 2 * kZNb * nl;                     // K index q < Ky: (l, o, j) = (q / 10, (q / 5) % 2, q % 5)
  const int Kt = Ky + 16;                           // then 16 coarse columns (o, cc)
  const int nk = (Kt + kFmBK - 1) / kFmBK;
  auto issue = [&](int t) {
    const int k0 = t * kFmBK, st = t & 1;
    // A: 64 rows x 16 K, element-wise
#pragma unroll
    for (int w = 0; w < kFmBM * kFmBK / 128; ++w) {
      const int idx = tid + w * 128, i = idx / kFmBK, kk = idx % kFmBK, q = k0 + kk;
      const double* src = Yst;
      bool ok = false;
      if (q < Ky) {
        const int l = q / (2 * kZNb), o = (q / kZNb) & 1, j = q % kZNb;
        const long long ro = arow[o][i];
        ok = ro >= 0;
        if (ok) src = Yst + (size_t)l * ystride + ro + j;
      } else if (q < Kt) {
        const int o = (q - Ky) >> 3, cc = (q - Ky) & 7;
        const long long ao = aabc[o][i];
        ok = ao >= 0 && cc < pd[o].nc;
        if (ok) src = abc + ao + cc;
      }
      cp_async8(&As[st][i * AP + kk], src, ok);
    }
    // B: 16 K rows x 64 columns, 16-byte chunks
#pragma unroll
    for (int w = 0; w < kFmBK * (kFmBN / 2) / 128; ++w) {
      const int idx = tid + w * 128, kk = idx / (kFmBN / 2), c2 = (idx % (kFmBN / 2)) * 2, q = k0 + kk;
      const int c = c0 + c2;
      const double* src = NT;
      bool ok = false;
      if (c < k) {
        if (q < Ky) {
          const int l = q / (2 * kZNb), o = (q / kZNb) & 1, j = q % kZNb;
          const int t = tt[o];
          const int sdm = t >= 0 ? nbr[t * kZNb + j] : -1;
          ok = sdm >= 0;
          if (ok) src = NT + ((size_t)l * k + sdm) * k + c;
        } else if (q < Kt) {
          const int o = (q - Ky) >> 3, cc = (q - Ky) & 7;
          ok = tt[o] >= 0 && cc < pd[o].nc;
          if (ok) src = Uc + (size_t)cmap[pd[o].cmap_off + cc] * k + c;
        }
      }
      cp_async16(&Bs[st][kk * BP + c2], src, ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  issue(0);
  cp_async_commit();
  for (int t = 0; t < nk; ++t) {
    if (t + 1 < nk) issue(t + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* A_ = As[t & 1];
    const double* B_ = Bs[t & 1];
#pragma unroll
    for (int k4 = 0; k4 < kFmBK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = A_[(wr * 32 + i * 8 + (lane >> 2)) * AP + k4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = B_[(k4 + (lane & 3)) * BP + wc * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int li = wr * 32 + i * 8 + (lane >> 2);
    if (li >= cnt) continue;
    double* qrow = Q + (size_t)R[li] * k;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + wc * 32 + j * 8 + 2 * (lane & 3);
      if (c < k) qrow[c] -= acc[i][j][0];
      if (c + 1 < k) qrow[c + 1] -= acc[i][j][1];
    }
  }
}

}  // namespace fg

namespace fg {

// ---------------------------------------------------------------------------
// K5e: the FETI-DP block apply by interface edge instead of by subdomain.
// A CTA owns BM dual rows of one interface edge (the rows shared by owners t1
// and t2, K5z's edge chunks) and BN columns of Q, and runs the K5 inner loop
// twice: over [F''_t1 | A''_t1][X_t1 ; U_t1] with the A rows taken at the
// rows' local indices in t1, then over t2's.  After t1's range the tile is
// stored to Q, after t2's it is added to what was stored: Q = acc_1 + acc_2,
// the value K5's two order-free atomic contributions into a zeroed Q give
// (0 + a + b), every element accumulated in the same k order -- so the result
// is bit-identical to K5, without the Q memset and without the atomic
// read-modify-write of Q (DRAM: Q is written once).
// ---------------------------------------------------------------------------
struct EdgeApplyArgs {
  const BzEdge* edges;   // edge chunks (t1, t2, first entry, row count)
  const int* erow;       // dual row of each entry
  const int* eb1;        // local row index in t1
  const int* eb2;        // local row index in t2
  const int* order;      // edge-chunk walk (nullable)
  int mt;                // BM-row tiles per chunk
};

template <int BM, int BN, int BK, int ST>
constexpr size_t k5e_smem(int kin_max) {
  return (size_t)ST * (BM * (BK + 4) + BK * (BN + 8)) * 8 + (size_t)(2 * kin_max + 3 * BM) * 4;
}

template <int BM, int BN, int BK, int ST>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32, 4) k_block_apply_edge(BlockApplyArgs a, EdgeApplyArgs ea) {
  constexpr int THREADS = (BM / 32) * (BN / 32) * 32;
  constexpr int AP = BK + 4, BP = BN + 8;
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                                   // ST x (BM x AP)
  double* Bs = dsm + ST * BM * AP;                    // ST x (BK x BP)
  int* srow = reinterpret_cast<int*>(Bs + ST * BK * BP);
  const int ci = blockIdx.y / ea.mt;
  const int chunk = ea.order ? ea.order[ci] : ci;
  const BzEdge e = ea.edges[chunk];
  const int r0 = (blockIdx.y - ci * ea.mt) * BM;
  if (r0 >= e.cnt) return;
  const int nrows = min(BM, e.cnt - r0);
  const int own[2] = {e.t1, e.t2};
  const OpSub d1 = a.subs[e.t1];
  const DpSub p1 = a.dps[e.t1];
  const int kin1 = d1.ns + p1.nc;
  const bool two = e.t2 >= 0;
  const OpSub d2 = two ? a.subs[e.t2] : d1;
  const DpSub p2 = two ? a.dps[e.t2] : p1;
  const int kin2 = two ? d2.ns + p2.nc : 0;
  int* srow2 = srow + kin1;
  int* lr1 = srow2 + kin2;     // BM local rows in t1
  int* lr2 = lr1 + BM;         // BM local rows in t2
  int* qr = lr2 + BM;          // BM dual rows
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < kin1; j += THREADS)
    srow[j] = j < d1.ns ? a.rows[d1.map_off + j] : a.cmap[p1.cmap_off + j - d1.ns];
  for (int j = tid; j < kin2; j += THREADS)
    srow2[j] = j < d2.ns ? a.rows[d2.map_off + j] : a.cmap[p2.cmap_off + j - d2.ns];
  for (int r = tid; r < BM; r += THREADS) {
    const bool ok = r < nrows;
    lr1[r] = ok ? ea.eb1[e.e0 + r0 + r] : 0;
    lr2[r] = ok && two ? ea.eb2[e.e0 + r0 + r] : 0;
    qr[r] = ok ? ea.erow[e.e0 + r0 + r] : 0;
  }
  __syncthreads();
  (void)own;
  const int col0 = blockIdx.x * BN;
  constexpr int WGN = BN / 32;
  const int wr = warp / WGN, wc = warp % WGN;
  const int nk1 = (kin1 + BK - 1) / BK, nk2 = two ? (kin2 + BK - 1) / BK : 0, nk = nk1 + nk2;
  auto issue = [&](int t) {
    const bool second = t >= nk1;
    const int kk = (second ? t - nk1 : t) * BK, stg = t % ST;
    const OpSub& d = second ? d2 : d1;
    const DpSub& p = second ? p2 : p1;
    const int kin = second ? kin2 : kin1, ns = d.ns, nc = p.nc;
    const int* lr = second ? lr2 : lr1;
    const int* sr = second ? srow2 : srow;
    const double* F = a.mats + d.moff;
    const double* Abc = a.abc + p.abc_off;
    double* A_ = As + stg * BM * AP;
    double* B_ = Bs + stg * BK * BP;
    constexpr int ACH = BM * (BK / 2), BCH = BK * (BN / 2);
#pragma unroll
    for (int q = 0; q < (ACH + THREADS - 1) / THREADS; ++q) {
      const int idx = tid + q * THREADS;
      if (ACH % THREADS == 0 || idx < ACH) {
        const int r = idx / (BK / 2), c2 = (idx % (BK / 2)) * 2;
        const int gi = lr[r], gj = kk + c2;
        const double* src = F;
        const bool ok = r < nrows && gj < kin;
        if (ok) src = gj < ns ? F + (size_t)gi * d.ld + gj : Abc + (size_t)gi * nc + (gj - ns);
        cp_async16(A_ + r * AP + c2, src, ok);
      }
    }
#pragma unroll
    for (int q = 0; q < (BCH + THREADS - 1) / THREADS; ++q) {
      const int idx = tid + q * THREADS;
      if (BCH % THREADS == 0 || idx < BCH) {
        const int r = idx / (BN / 2), c2 = (idx % (BN / 2)) * 2;
        const int gj = kk + r, gc = col0 + c2;
        const double* src = a.W;
        const bool ok = gj < kin && gc < a.k;
        if (ok) src = gj < ns ? a.W + (size_t)sr[gj] * a.ldw + gc : a.U + (size_t)sr[gj] * a.ldu + gc;
        cp_async16(B_ + r * BP + c2, src, ok);
      }
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // tile -> Q: Q = 0 + tile (first owner) or Q += tile (the second)
  auto flush = [&](bool add) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int li = wr * 32 + i * 8 + (lane >> 2);
      if (li >= nrows) continue;
      double* qrow = a.Q + (size_t)qr[li] * a.ldq;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int gc = col0 + wc * 32 + j * 8 + 2 * (lane & 3);
        if (gc + 1 < a.k) {
          double2* q2 = reinterpret_cast<double2*>(qrow + gc);
          const double2 o = add ? *q2 : make_double2(0.0, 0.0);   // (0 + a) + b, as the atomics
          *q2 = make_double2(__dadd_rn(o.x, acc[i][j][0]), __dadd_rn(o.y, acc[i][j][1]));
        } else if (gc < a.k) {
          qrow[gc] = __dadd_rn(add ? qrow[gc] : 0.0, acc[i][j][0]);
        }
      }
    }
  };
#pragma unroll
  for (int t = 0; t < ST - 1; ++t) {
    if (t < nk) issue(t);
    cp_async_commit();
  }
  for (int t = 0; t < nk; ++t) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    if (t + ST - 1 < nk) issue(t + ST - 1);
    cp_async_commit();
    if (t == nk1) {   // t1's range done: store it, start t2's from zero
      flush(false);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    const double* A_ = As + (t % ST) * BM * AP;
    const double* B_ = Bs + (t % ST) * BK * BP;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = A_[(wr * 32 + i * 8 + (lane >> 2)) * AP + k4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = B_[(k4 + (lane & 3)) * BP + wc * 32 + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  flush(two);
}

}  // namespace fg
