// common.cuh -- shared device-side definitions of the FETI engine.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace fg {

constexpr int kThreads = 256;
constexpr int kSmallFront = 112;   // frontal matrices up to this size are eliminated in smem
constexpr int kNB = 32;            // panel width of the blocked elimination
constexpr int kTile = 64;          // trailing-update tile

// status word codes written by kernels (mapped to FETIGPU_E_* on the host)
enum DevStatus : int {
  kOk = 0,
  kNotSPD = 1,
};

// One dense frontal matrix (column-major, leading dimension ld) whose first
// ne DOFs are eliminated in place: on exit columns [0,ne) hold [L_ee; L_be]
// and the trailing (nf-ne)^2 block holds the Schur complement (lower part).
struct FrontDesc {
  long long off;
  int nf, ne, ld, code;   // code: status reported on a nonpositive pivot
};

// nested-dissection tree node on the device
struct NdDev {
  int nf, ne, leaf, height;
  long long off, foff;
  int elem_off, elem_cnt;
  int child[2];
  int cmap_off[2];
  int dof_off;
};

// per-subdomain descriptor of an explicit local operator (F_s or S~_s)
struct OpSub {
  long long moff;   // offset of the dense ns x ns matrix (row-major, ld)
  int ns, ld;
  int map_off;      // offset of the ns*KR (row, coef) gather/scatter entries
  int pad;
};

// FETI-DP per-subdomain coarse coupling
struct DpSub {
  long long abc_off;  // A_bc, ns x nc row-major
  int nc;
  int cmap_off;       // global primal ids (nc)
  int v_off;          // per-subdomain vector buffer offset (ns)
  int t_off;          // per-subdomain coarse buffer offset (nc)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// cp.async (Ampere-style asynchronous global -> shared copies, no register
// staging); an invalid source is zero-filled (src-size 0)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace fg
