// Launch interface of the value-iteration kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

#include "common.cuh"
#include "model.hpp"

namespace pvi_b200 {

// Arguments of the fused finalize / convergence reduction.
struct FinalizeArgs {
  int test = -1;                 // -1: only the non-finite scan
  int n_hist = 0;                // previous vectors available in hist (periodic span: >= 7)
  const void* hist[8] = {};      // device pointers, oldest..newest (newest = V_prev)
  double gamma = 0.0;
  SweepStats* stats = nullptr;   // device; nullptr disables the reduction
  // Fused exchange over NVLink peer memory (factored B x_3-pair sweep): the
  // finalize also stores each V' entry into the replica of every peer whose
  // next sweep reads it (its x_3 rows, or its constants' rows x_2 = 0 with
  // x_3 <= its x3_hi).  peer_v: IPC-mapped |S|-entry buffers of the peers.
  int n_peers = 0;
  int peer_all = 0;              // 1: every V' entry to every peer (full replicas; state_stat)
  void* peer_v[8] = {};
  int peer_x3_lo[8] = {}, peer_x3_hi[8] = {};
};

template <typename T>
struct SweepArgs {
  const T* v = nullptr;          // V_prev, |S| entries (device)
  T* vout = nullptr;             // indexed by s - out_off
  std::uint32_t* act = nullptr;  // indexed by s - out_off
  T* qout = nullptr;             // (hi-lo) x |A| Q values, or nullptr
  std::uint64_t lo = 0, hi = 0, out_off = 0;
  double gamma = 0.0;
  bool want_values = true;       // false: Q rows only (B/C skip the partial buffers)
  int algorithm = 0;             // 0 exact (reference order, bit-identical), 1 factored
  FinalizeArgs fa;
  // factored B only: which stages to run (1: W from V, 2: Q / argmax / finalize)
  // and the stage-1 CTA range r in [r_lo, r_hi) (CTA r reads V[r |x_b| .. (r+1) |x_b|)),
  // so a caller can start stage 1 on the part of V already uploaded
  int stages = 3;
  std::uint64_t r_lo = 0, r_hi = ~0ull;
  // factored B stage 2 (k_b_fact_qw3 only): the x_b columns [xb_lo, xb_hi)
  // to process; V' / argmax then land in a strided column block
  std::uint64_t xb_lo = 0, xb_hi = ~0ull;
  // factored B stage 1 (m = 3, f64): when >= 0, only the W rows whose x_3
  // digit lies in [x3_rows_lo, x3_rows_hi] (no constants' rows of lower x_3)
  int x3_rows_lo = -1, x3_rows_hi = -1;
  int x3_rows_strict = 1;  // 0: also the constants' rows (x_2 = 0, x_3 <= x3_rows_hi)
  // factored B stage 1 (f64): only the x_b digit groups [xg_lo, xg_hi) (16
  // consecutive x_b each) of the rows -- the x_b columns of a unit shard
  std::uint32_t xg_lo = 0, xg_hi = ~0u;
  // false: accumulate into fa.stats without resetting them first (the
  // second and later launches of one multi-segment sweep)
  bool init_stats = true;
  // unit shards: stage 2 as a 1-D grid over the flat (pair, x_b) indices
  // [flat_lo, flat_hi); stage 1 restricts the non-constant rows of a partial
  // head pair to groups >= head_g_lo and of a partial tail pair to < tail_g_hi
  std::uint64_t flat_lo = 0, flat_hi = 0;
  int head_pair = -1, head_g_lo = 0, tail_pair = -1, tail_g_hi = 0;
};

// Grow-only device scratch buffers, keyed by slot.
struct Scratch {
  std::vector<void*> ptr;
  std::vector<std::size_t> bytes;
  template <typename U>
  U* get(int slot, std::size_t count, cudaStream_t stream) {
    if (static_cast<int>(ptr.size()) <= slot) {
      ptr.resize(slot + 1, nullptr);
      bytes.resize(slot + 1, 0);
    }
    const std::size_t need = count * sizeof(U);
    if (bytes[slot] < need) {
      if (ptr[slot]) {
        cudaStreamSynchronize(stream);
        cudaFree(ptr[slot]);
      }
      ptr[slot] = nullptr;
      PVI_CUDA(cudaMalloc(&ptr[slot], need));
      bytes[slot] = need;
      maybe_poison(ptr[slot], need, stream);
    }
    return static_cast<U*>(ptr[slot]);
  }
  // PVI_POISON=1: refill every buffer (called at the start of a full sweep)
  void poison(cudaStream_t stream) {
    for (std::size_t i = 0; i < ptr.size(); ++i) maybe_poison(ptr[i], bytes[i], stream);
  }
  ~Scratch() {
    for (void* p : ptr)
      if (p) cudaFree(p);
  }
};

template <typename T>
void launch_sweep(const Model& model, const DevModel& dm, const SweepArgs<T>& a, Scratch& scratch,
                  cudaStream_t stream);
template <typename T>
void launch_stats(const T* vnew, const T* vprev, std::uint64_t n, const FinalizeArgs& fa,
                  cudaStream_t stream);
bool b_sweep_honours_xb_range(const Model& model, int device);
bool c_weekday_local(const Model& model);
std::vector<std::pair<std::uint64_t, std::uint64_t>> sweep_read_runs(const Model& model, std::uint64_t lo,
                                                                     std::uint64_t hi);
void profile_enable(bool on);
bool profiling_enabled();
// simulation measurement hook: Philox blocks, rollout-days and k_rollouts
// milliseconds accumulated while profiling is enabled
void sim_profile_add(std::uint64_t philox_blocks, std::uint64_t rollout_days, double kernel_ms);
void sim_profile_read(std::uint64_t* philox_blocks, std::uint64_t* rollout_days, double* kernel_ms);
void init_stats_device(SweepStats* st, cudaStream_t stream);
void profile_read(double* ms, std::uint64_t* main_launches, std::uint64_t* all_launches);
void launch_initial_b(const DevModel& dm, double* out, std::uint64_t n, cudaStream_t stream);
template <typename T>
void launch_cast_from_f64(const double* in, T* out, std::uint64_t n, cudaStream_t stream);
template <typename T>
void launch_widen(const T* in, double* out, std::uint64_t n, cudaStream_t stream);

}  // namespace pvi_b200
