// DRAM access-pattern microbenchmark for the factored-C binomial passes:
// the same 2.5 GB read + 2.5 GB write as one endogenous c/m5 pass, moved
// (a) as a linear copy and (b) in the passes' row pattern (rows of 441
// contiguous doubles at the pass strides, one CTA per (order, weekday, line)
// item), and (c) with the item order of k_c_bin_wide.  Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lib/c_pattern_peak tools/c_pattern_peak.cu
#include <cuda_runtime.h>

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

constexpr int R = 21;
constexpr unsigned WB = R * R * R * R;  // 194481

__global__ void k_linear(const double* __restrict__ in, double* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void k_linear2(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__host__ __device__ inline size_t tri_base(int a, unsigned wb) {
  return (size_t)7 * wb * ((size_t)a * (a + 1) / 2);
}

// one CTA per (a, tau, line2) item: rows (b', d) of 441 doubles at
// b' * WB + d * wk + rest0; wk = 9261 (k = 4, line = x_3) or 441 (k = 3, line = x_4)
__global__ void __launch_bounds__(448, 2) k_rows(const double* __restrict__ in, double* __restrict__ out, int wk_k) {
  const int blk = blockIdx.x;
  const int ai = blk / (7 * R), rem = blk % (7 * R);
  const int a = R - 1 - ai, nb = a + 1, tau = rem / R, line = rem % R;
  const unsigned wk = wk_k == 4 ? 9261u : 441u, wl = wk_k == 4 ? 441u : 9261u;
  const size_t base = tri_base(a, WB) + (size_t)tau * nb * WB + (size_t)line * wl;
  const int col = threadIdx.x;
  if (col >= R * R) return;
  for (int bp = 0; bp < nb; ++bp) {
    double v[R];
#pragma unroll
    for (int d = 0; d < R; ++d) v[d] = __ldg(in + base + (size_t)bp * WB + d * wk + col);
#pragma unroll
    for (int d = 0; d < R; ++d) out[base + (size_t)bp * WB + d * wk + col] = v[d];
  }
}

template <typename K>
static float best_ms(K launch) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < 8; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (r >= 2 && ms < best) best = ms;
  }
  return best;
}

int main() {
  const size_t n = tri_base(R, WB);  // all 21 orders x 7 weekdays
  const double gb = 2.0 * n * 8 / 1e9;
  double *in, *out;
  CK(cudaMalloc(&in, n * 8));
  CK(cudaMalloc(&out, n * 8));
  CK(cudaMemset(in, 0, n * 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const float t_lin = best_ms([&] { k_linear<<<sms * 8, 256>>>(in, out, n); });
  const float t_lin2 = best_ms([&] { k_linear2<<<sms * 8, 256>>>((const double2*)in, (double2*)out, n / 2); });
  const float t_k4 = best_ms([&] { k_rows<<<R * 7 * R, 448>>>(in, out, 4); });
  const float t_k3 = best_ms([&] { k_rows<<<R * 7 * R, 448>>>(in, out, 3); });
  std::printf("{\"bytes_gb\": %.3f, \"linear_8B_ms\": %.4f, \"linear_8B_gbs\": %.1f, \"linear_16B_ms\": %.4f, "
              "\"linear_16B_gbs\": %.1f, \"rows_k4_ms\": %.4f, \"rows_k4_gbs\": %.1f, \"rows_k3_ms\": %.4f, "
              "\"rows_k3_gbs\": %.1f}\n",
              gb, t_lin, gb / t_lin * 1e3, t_lin2, gb / t_lin2 * 1e3, t_k4, gb / t_k4 * 1e3, t_k3, gb / t_k3 * 1e3);
  return 0;
}
