// Shared device helpers: error checking, ordered-double atomics, block
// reductions.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "model.hpp"

namespace pvi_b200 {

// NVTX range (header-only NVTX3: a no-op unless a profiler such as nsys or
// ncu --nvtx is attached): per-sweep, solve-phase, backup-pipeline and
// rollout ranges for timeline tools (SURVEY §5 tracing).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


#define PVI_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      ::pvi_b200::fail(PVI_ERR_DEVICE, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                           " at " + __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// Host -> device copy of a one-off table that is complete when this returns.
// A plain cudaMemcpy from pageable memory may return before its DMA lands,
// and every kernel here runs on a non-blocking stream, which does not wait
// for the legacy stream the copy was queued on.
inline void upload_bytes(void* dst, const void* src, std::size_t bytes) {
  PVI_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  PVI_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
}

// Debug aid standing in for compute-sanitizer's initcheck (closed on this
// GPU pool): with PVI_POISON=1 every sweep scratch buffer and every output
// slice is filled with 0xFF bytes (NaN for f64/f32, 255 for the u8 partial
// argmax) before a sweep, so a kernel that reads an element nobody wrote, or
// leaves an output element unwritten, produces NaN / a wrong action that the
// parity tests see (tests/test_gpu_poison.py).
inline bool poison_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PVI_POISON");
    return e && e[0] == '1';
  }();
  return on;
}
inline void maybe_poison(void* p, std::size_t bytes, cudaStream_t stream) {
  if (p && bytes && poison_enabled()) PVI_CUDA(cudaMemsetAsync(p, 0xFF, bytes, stream));
}

__host__ __device__ inline int ipos(int x) { return x > 0 ? x : 0; }

// Order-preserving map from double to u64 so that atomicMax/atomicMin on
// the key are max/min on the value (NaNs never reach here: the non-finite
// scan reports them separately).
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(unsigned long long k) {
  const unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(u));
#else
  double d;
  __builtin_memcpy(&d, &u, 8);
  return d;
#endif
}

// Per-sweep statistics reduced on the device: max and min of the
// convergence statistic, and the first non-finite state.
struct SweepStats {
  unsigned long long max_key;
  unsigned long long min_key;
  unsigned long long first_bad;  // UINT64_MAX when none
  unsigned long long pad;
};

// Stream-ordered allocation from the device's default memory pool, which
// keeps freed memory (release threshold = max), so repeated solves and
// evaluations on a device do not pay cudaMalloc / cudaFree each call.
struct PoolBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  PoolBuf(std::size_t bytes, cudaStream_t stream) : s(stream) {
    static bool configured[64] = {};
    int dev = 0;
    PVI_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && !configured[dev]) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        std::uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
      configured[dev] = true;
    }
    if (bytes) PVI_CUDA(cudaMallocAsync(&p, bytes, stream));
  }
  PoolBuf(const PoolBuf&) = delete;
  PoolBuf& operator=(const PoolBuf&) = delete;
  ~PoolBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

}  // namespace pvi_b200
