// runtime.cuh -- error macros, device allocation (block cache), launch helpers (PDL,
// shared-memory opt-in), host parallel_for, phase timer and scratch buffers.
// Part of the libfetigpu unity build (fetigpu.cu includes it); namespace fg.
#pragma once
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "fetigpu.h"
#include "setup.hpp"  // fg::Error / fail

namespace fg {

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      fail(e_ == cudaErrorMemoryAllocation ? FETIGPU_E_OUT_OF_MEMORY : FETIGPU_E_CUDA,         \
           std::string(#x) + ": " + cudaGetErrorString(e_));                                   \
  } while (0)
#define LAUNCH_CHECK()                                                                         \
  do {                                                                                         \
    cudaError_t e_ = cudaGetLastError();                                                       \
    if (e_ != cudaSuccess)                                                                     \
      fail(e_ == cudaErrorMemoryAllocation ? FETIGPU_E_OUT_OF_MEMORY : FETIGPU_E_CUDA,         \
           std::string("kernel launch before ") + __FILE__ + ":" + std::to_string(__LINE__) + ": " +  \
               cudaGetErrorString(e_));                                                        \
  } while (0)

static std::atomic<size_t> g_device_bytes{0};  // live DBuf bytes, all contexts (stats)

// Device memory.  Plain cudaMalloc / cudaFree, except for buffers that name a
// BlockCache: a freed block is kept there and handed to a later request it
// fits (at most 2x larger).  Only the RRS direction store uses one (each
// context owns its cache): its multi-GB chunks are allocated per solve, and
// that is where driver allocation cost varied (up to ~0.9 s per C5 solve).
// Everything else keeps a fresh cudaMalloc placement -- measured: caching the
// build workspace or operator storage made the L2-resident applies of C2 / C3
// 6-10% slower.  A release into the cache first synchronises the device
// (cudaFree semantics: buffers freed at scope end are never still in use).
// On OOM the cache is returned to the driver and the allocation retried.
// FETIGPU_NO_CACHE=1 disables caching.
static bool cache_on() {
  static const bool on = [] {
    const char* e = getenv("FETIGPU_NO_CACHE");
    return !(e && e[0] == '1');
  }();
  return on;
}
// FETIGPU_TIMING=1 also reports every allocation / free of >= 64 MB
// (FETIGPU_TIMING=2: only those, without the synchronising phase marks)
static bool alloc_trace() {
  static const bool on = [] {
    const char* e = getenv("FETIGPU_TIMING");
    return e && (e[0] == '1' || e[0] == '2');
  }();
  return on;
}
struct AllocTrace {
  const char* what;
  size_t bytes;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~AllocTrace() {
    if (!alloc_trace() || bytes < (64u << 20)) return;
    fprintf(stderr, "[fetigpu]   %s %8.1f MB %8.2f ms\n", what, bytes / 1048576.0,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};
struct BlockCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;      // capacity -> block
  std::unordered_map<void*, size_t> capacity;    // every live or cached block
  size_t cached = 0;
  // return every cached block to the driver
  void trim() {
    std::lock_guard<std::mutex> lk(mu);
    if (free_blocks.empty()) return;
    cudaDeviceSynchronize();
    for (auto& f : free_blocks) {
      AllocTrace tr{"cudaFree  ", f.first};
      cudaFree(f.second);
      capacity.erase(f.second);
    }
    free_blocks.clear();
    cached = 0;
  }
  size_t cached_bytes() {
    std::lock_guard<std::mutex> lk(mu);
    return cached;
  }
  ~BlockCache() { trim(); }
};
static void* dev_alloc(size_t bytes, BlockCache* cache) {
  bytes = (bytes + 511) & ~size_t(511);
  if (!cache || !cache_on()) {
    AllocTrace tr{"cudaMalloc", bytes};
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    return p;
  }
  {
    std::lock_guard<std::mutex> lk(cache->mu);
    auto it = cache->free_blocks.lower_bound(bytes);
    if (it != cache->free_blocks.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      cache->cached -= it->first;
      cache->free_blocks.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e;
  {
    AllocTrace tr{"cudaMalloc", bytes};
    e = cudaMalloc(&p, bytes);
  }
  if (e == cudaErrorMemoryAllocation) {  // give the cache back, retry
    cudaGetLastError();
    cache->trim();
    e = cudaMalloc(&p, bytes);
  }
  CK(e);
  std::lock_guard<std::mutex> lk(cache->mu);
  cache->capacity[p] = bytes;
  return p;
}
static void dev_free(void* p, size_t bytes, BlockCache* cache) {
  if (cache && cache_on()) {
    std::lock_guard<std::mutex> lk(cache->mu);
    auto it = cache->capacity.find(p);
    if (it != cache->capacity.end()) {
      cudaDeviceSynchronize();  // cudaFree semantics: nothing still uses the buffer
      cache->free_blocks.emplace(it->second, p);
      cache->cached += it->second;
      return;
    }
  }
  AllocTrace tr{"cudaFree  ", bytes};
  cudaFree(p);
}
// free device memory including the blocks held in `cache`
static size_t dev_free_bytes(BlockCache* cache = nullptr) {
  size_t freeb = 0, total = 0;
  CK(cudaMemGetInfo(&freeb, &total));
  if (cache) freeb += cache->cached_bytes();
  return freeb;
}

// During an in-place rebuild (fetigpu_rebuild) every DBuf allocated on this
// thread without its own cache takes this one (and keeps it): the rebuild's
// release + alloc of same-sized operator storage recycles the blocks instead
// of calling cudaFree / cudaMalloc (multi-GB calls that occasionally stall
// for 100+ ms in the driver).
static thread_local BlockCache* g_build_cache = nullptr;

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
      dev_free(p, n * sizeof(T), cache);
      g_device_bytes -= n * sizeof(T);
    }
    p = nullptr;
    n = 0;
  }
  BlockCache* cache = nullptr;  // recycled storage: allocate through this block cache
  void alloc(size_t count) {
    release();
    if (!cache && g_build_cache) cache = g_build_cache;
    if (count == 0) count = 1;
    p = static_cast<T*>(dev_alloc(count * sizeof(T), cache));
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

// f(i) for i in [0, n) over up to max_threads host threads (contiguous
// ranges, at most the core count); f must write disjoint outputs.  Serial for
// small n.
template <class F>
static void parallel_for(int n, F&& f, int max_threads = 16) {
  const int nt = std::min<int>(max_threads, std::max(1u, std::thread::hardware_concurrency()));
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
  bool sync = true;  // FETIGPU_TIMING=3: host timestamps only (no stream synchronisation)
  PhaseTimer() {
    const char* e = getenv("FETIGPU_TIMING");
    on = e && (e[0] == '1' || e[0] == '3');
    sync = !(e && e[0] == '3');
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what, cudaStream_t st) {
    if (!on) return;
    if (sync) cudaStreamSynchronize(st);
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

}  // namespace fg
