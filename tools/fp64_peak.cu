// FP64 pipe microbenchmark (the compute roofline of the
// factored sweeps needs a MEASURED FP64 peak, not the nominal one).
// Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lib/fp64_peak tools/fp64_peak.cu
//
// Kernels (one launch = `blocks` x 256 threads, every thread running `iters`
// rounds of CH independent dependency chains):
//   dfma   acc[c] = fma(acc[c], a, b)   -> DFMA, 2 flops each
//   dsetp  DFMA chain plus a compare-and-select per step (the sweep's inner
//          loop shape: t = fma(.), if (t > best) best = t) -> FP64-pipe ops/s
// Reported: best of 10 launches, CUDA events, SM clock sampled by the caller.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

template <int CH>
__global__ void __launch_bounds__(256) k_dfma(double a, double b, int iters, double* __restrict__ out) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains live
}

template <int CH>
__global__ void __launch_bounds__(256) k_dsetp(double a, double b, int iters, double* __restrict__ out) {
  double acc[CH], best[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    acc[c] = threadIdx.x * 1e-9 + c;
    best[c] = -1e300;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      acc[c] = fma(acc[c], a, b);
      if (acc[c] > best[c]) best[c] = acc[c];
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c] + best[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// FP64 tensor-core path (DMMA): mma.sync m8n8k4 f64, CH independent
// accumulator tiles per warp; 8x8x4 = 256 MACs per warp instruction.
template <int CH>
__global__ void __launch_bounds__(256) k_dmma(double a, double b, int iters, double* __restrict__ out) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-9 + c;
  const double fa = a + threadIdx.x * 1e-12, fb = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(fa), "d"(fb));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
static float best_ms(K kern, int blocks, int iters, double* out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < 12; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, 256>>>(0.999999, 1e-7, iters, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (r >= 2) best = std::min(best, ms);
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out = nullptr;
  CK(cudaMalloc(&out, 256 * sizeof(double)));
  const int iters = 20000;
  std::printf("{\"sms\": %d, \"max_sm_clock_mhz\": %.0f, \"results\": [", sms, clk / 1e3);
  bool first = true;
  for (int per_sm : {4, 8}) {
    const int blocks = sms * per_sm;
    const double threads = blocks * 256.0;
    {
      const float ms = best_ms(k_dfma<8>, blocks, iters, out);
      const double fl = 2.0 * threads * iters * 8;
      std::printf("%s{\"kernel\": \"dfma\", \"chains\": 8, \"ctas_per_sm\": %d, \"ms\": %.4f, "
                  "\"tflops\": %.3f}", first ? "" : ", ", per_sm, ms, fl / (ms * 1e-3) / 1e12);
      first = false;
    }
    {
      const float ms = best_ms(k_dfma<4>, blocks, iters, out);
      const double fl = 2.0 * threads * iters * 4;
      std::printf(", {\"kernel\": \"dfma\", \"chains\": 4, \"ctas_per_sm\": %d, \"ms\": %.4f, "
                  "\"tflops\": %.3f}", per_sm, ms, fl / (ms * 1e-3) / 1e12);
    }
    {
      const float ms = best_ms(k_dsetp<8>, blocks, iters, out);
      const double ops = threads * iters * 8;  // one DFMA + one DSETP per step
      std::printf(", {\"kernel\": \"dfma+dsetp\", \"chains\": 8, \"ctas_per_sm\": %d, \"ms\": %.4f, "
                  "\"fp64_pipe_gops\": %.1f, \"tflops_fma_only\": %.3f}",
                  per_sm, ms, 2.0 * ops / (ms * 1e-3) / 1e9, 2.0 * ops / (ms * 1e-3) / 1e12);
    }
  }
  for (int per_sm : {4, 8}) {
    const int blocks = sms * per_sm;
    const float ms = best_ms(k_dmma<8>, blocks, iters / 4, out);
    const double warps = blocks * 8.0;
    const double fl = 2.0 * 256.0 * warps * (iters / 4) * 8;
    std::printf(", {\"kernel\": \"dmma m8n8k4\", \"chains\": 8, \"ctas_per_sm\": %d, \"ms\": %.4f, "
                "\"tflops\": %.3f}", per_sm, ms, fl / (ms * 1e-3) / 1e12);
  }
  std::printf("]}\n");
  return 0;
}
