// Philox4x32-10 throughput microbenchmark: the integer-pipe ceiling of the
// simulation kernel's random numbers ("report steps/s and Philox
// blocks/s").  Every thread computes `iters` blocks with
// the rollout kernel's counter layout {day, draw, 0x7F4A7C15, 0} and key
// (seed + rollout), XOR-folding the outputs so nothing is dead.  Prints one
// JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lib/philox_peak tools/philox_peak.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
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

__device__ __forceinline__ void philox(std::uint32_t c[4], std::uint32_t k0, std::uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const std::uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
    const std::uint32_t lo0 = 0xD2511F53u * c[0];
    const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const std::uint32_t lo1 = 0xCD9E8D57u * c[2];
    const std::uint32_t n0 = hi1 ^ c[1] ^ k0;
    const std::uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

template <int CH>
__global__ void __launch_bounds__(256) k_philox(std::uint64_t seed, int iters, std::uint32_t* out) {
  const std::uint64_t key = seed + blockIdx.x * blockDim.x + threadIdx.x;
  const std::uint32_t k0 = static_cast<std::uint32_t>(key), k1 = static_cast<std::uint32_t>(key >> 32);
  std::uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {  // CH independent blocks per step (ILP)
      std::uint32_t ctr[4] = {static_cast<std::uint32_t>(i), static_cast<std::uint32_t>(c), 0x7F4A7C15u, 0u};
      philox(ctr, k0, k1);
      acc ^= ctr[0] ^ ctr[1];
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int CH>
static void run(int blocks, int iters, std::uint32_t* out, bool& first) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(e0));
    k_philox<CH><<<blocks, 256>>>(42, iters, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (r >= 2) best = std::min(best, ms);
  }
  const double n = static_cast<double>(blocks) * 256.0 * iters * CH;
  std::printf("%s{\"chains\": %d, \"ctas\": %d, \"ms\": %.4f, \"gblocks_per_s\": %.2f}", first ? "" : ", ", CH,
              blocks, best, n / (best * 1e-3) / 1e9);
  first = false;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  std::uint32_t* out = nullptr;
  CK(cudaMalloc(&out, 4));
  std::printf("{\"sms\": %d, \"results\": [", sms);
  bool first = true;
  for (int per_sm : {4, 8}) {
    run<1>(sms * per_sm, 4000, out, first);
    run<2>(sms * per_sm, 2000, out, first);
    run<4>(sms * per_sm, 1000, out, first);
  }
  std::printf("]}\n");
  return 0;
}
