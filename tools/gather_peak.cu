// Gather-bandwidth microbenchmark ("for L2-resident V, also
// report against a measured L2 gather bandwidth ... random-gather
// microbenchmark over a 64 MiB buffer").  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lib/gather_peak tools/gather_peak.cu
//
// Kernels:
//   random_gather  8-byte loads at hashed indices (8 independent chains per
//                  thread) -- the access pattern of a V[next] gather with no
//                  locality; reports useful bytes/s (8 B per load).
//   stream_read    coalesced 16-byte loads of the same buffer, re-read until
//                  the total is large -- L2 (or HBM) streaming bandwidth.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ std::uint32_t mix(std::uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(256) random_gather(const double* __restrict__ buf, std::uint32_t mask,
                                                     int iters, double* __restrict__ out) {
  const std::uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  double acc[8];
  std::uint32_t h[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    acc[c] = 0.0;
    h[c] = mix(tid * 8u + c + 1u);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      h[c] = h[c] * 1664525u + 1013904223u;  // LCG stream per chain
      acc[c] += __ldg(buf + (mix(h[c]) & mask));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  out[tid] = s;
}

__global__ void __launch_bounds__(256) stream_read(const double2* __restrict__ buf, std::uint64_t n2,
                                                   int passes, double* __restrict__ out) {
  const std::uint64_t tid = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  double acc = 0.0;
  for (int p = 0; p < passes; ++p)
    for (std::uint64_t i = tid; i < n2; i += stride) {
      const double2 v = __ldg(buf + i);
      acc += v.x + v.y;
    }
  out[tid] = acc;
}

template <typename F>
static float time_ms(F&& launch, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();  // warm-up (also fills L2 for the resident cases)
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaEventDestroy(a));
  CK(cudaEventDestroy(b));
  return best;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int l2 = 0;
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  const int blocks = sms * 8, threads = 256;
  const std::uint64_t nthreads = static_cast<std::uint64_t>(blocks) * threads;
  double* out = nullptr;
  CK(cudaMalloc(&out, nthreads * sizeof(double)));

  std::printf("{\"sms\": %d, \"l2_bytes\": %d, \"results\": [", sms, l2);
  // buffer sizes in MiB: L1-ish, L2-resident (the survey's 64 MiB), HBM
  const std::vector<int> mibs = {4, 16, 64, 128, 2048};
  bool first = true;
  for (int mib : mibs) {
    const std::uint64_t n = (static_cast<std::uint64_t>(mib) << 20) / sizeof(double);
    double* buf = nullptr;
    CK(cudaMalloc(&buf, n * sizeof(double)));
    CK(cudaMemset(buf, 0, n * sizeof(double)));
    const int iters = 256;
    const float g_ms = time_ms([&] {
      random_gather<<<blocks, threads>>>(buf, static_cast<std::uint32_t>(n - 1), iters, out);
    }, 5);
    CK(cudaGetLastError());
    const double loads = static_cast<double>(nthreads) * iters * 8;
    const int passes = mib >= 1024 ? 2 : static_cast<int>(std::max<std::uint64_t>(1, (8192ull >> 0) / mib));
    const float s_ms = time_ms([&] {
      stream_read<<<blocks, threads>>>(reinterpret_cast<const double2*>(buf), n / 2, passes, out);
    }, 5);
    CK(cudaGetLastError());
    const double sbytes = static_cast<double>(n) * sizeof(double) * passes;
    std::printf("%s{\"buffer_mib\": %d, \"random_gather_gbs\": %.1f, \"random_gather_gloads_s\": %.2f, "
                "\"stream_read_gbs\": %.1f}",
                first ? "" : ", ", mib, loads * 8 / (g_ms * 1e-3) / 1e9, loads / (g_ms * 1e-3) / 1e9,
                sbytes / (s_ms * 1e-3) / 1e9);
    first = false;
    CK(cudaFree(buf));
  }
  std::printf("]}\n");
  CK(cudaFree(out));
  return 0;
}
