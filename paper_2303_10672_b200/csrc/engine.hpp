// Host engine entry points behind the C ABI.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "model.hpp"

namespace pvi_b200 {

int select_device(int requested);
std::string hex32(const std::uint8_t* fp);

void vi_solve(const Model& m, const pvi_vi_config& cfg, const double* resume_values,
              std::uint64_t resume_iteration, const std::uint8_t* resume_fp, double* out_values,
              std::uint32_t* out_policy, pvi_vi_stats* stats);
void vi_backup(const Model& m, int precision, double gamma, const void* values, std::uint64_t lo,
               std::uint64_t hi, void* out_values, std::uint32_t* out_actions, void* out_q);
bool check_convergence(const Model& m, int precision, int test, const void* const* history,
                       int n_hist, double gamma, double epsilon, std::uint64_t iteration);
void vi_sweep_device(const Model& m, int precision, double gamma, const void* vprev, void* vnext,
                     std::uint32_t* act, std::uint64_t lo, std::uint64_t hi, int test,
                     const void* const* hist, int n_hist, int want_stats, double* stats,
                     void* stream);
void vi_sweep_device_peers(const Model& m, int precision, double gamma, const void* vprev, void* vnext,
                           std::uint64_t lo, std::uint64_t hi, int test, int want_stats, double* stats,
                           void* stream, int n_peers, void* const* peer_vnext, const std::uint64_t* peer_lo,
                           const std::uint64_t* peer_hi);
void partition(const Model& m, int parts, std::uint64_t* bounds);
// unit shards of the factored B x_3-pair sweep (engine.cu)
std::uint64_t unit_count(const Model& m);
void unit_partition(const Model& m, int parts, std::uint64_t* bounds);
std::vector<std::pair<std::uint64_t, std::uint64_t>> unit_own_runs(const Model& m, std::uint64_t u_lo,
                                                                   std::uint64_t u_hi);
std::vector<std::pair<std::uint64_t, std::uint64_t>> unit_read_runs(const Model& m, std::uint64_t u_lo,
                                                                    std::uint64_t u_hi);
void vi_sweep_device_units(const Model& m, int precision, double gamma, const void* vprev, void* vnext,
                           std::uint32_t* act, std::uint64_t u_lo, std::uint64_t u_hi, int test, int want_stats,
                           double* stats, void* stream, int n_peers, void* const* peer_vnext,
                           const std::uint64_t* peer_u_lo, const std::uint64_t* peer_u_hi);
// policy CSV rows on the device (io_kernels.cu): the body (one row per
// state) of runner.cpp's policy_to_csv; out = nullptr returns the length
std::uint64_t policy_csv_format(const Model& m, const std::uint32_t* actions, char* out, std::uint64_t capacity);
// policy_from_csv after the metadata check: whole file text -> actions
void policy_csv_parse(const Model& m, const char* text, std::uint64_t len, std::uint32_t* out);
void profile_enable(bool on);
bool profiling_enabled();
// simulation measurement hook: Philox blocks, rollout-days and k_rollouts
// milliseconds accumulated while profiling is enabled
void sim_profile_add(std::uint64_t philox_blocks, std::uint64_t rollout_days, double kernel_ms);
void sim_profile_read(std::uint64_t* philox_blocks, std::uint64_t* rollout_days, double* kernel_ms);
void profile_read(double* ms, std::uint64_t* main_launches, std::uint64_t* all_launches);
void initial_values_host(const Model& m, double* out);

void save_checkpoint(const std::string& path, const double* values, std::uint64_t count,
                     std::uint64_t iteration, const std::uint8_t fp[32]);
void load_checkpoint(const std::string& path, const std::uint8_t* expected, double* values,
                     std::uint64_t capacity, std::uint64_t* count, std::uint64_t* iteration,
                     std::uint8_t fp[32]);

// Simulation (sim_kernels.cu)
void sim_evaluate(const Model& m, const pvi_policy* policies, std::uint32_t n_policies,
                  const pvi_rollout_config& cfg, pvi_rollout_summary* per_rollout,
                  pvi_evaluation* evals);
// detail::reduce on the host (pvi_sim_reduce): summ is n_policies x n x 7
void sim_reduce_host(const double* summ, std::uint32_t n_policies, int n, int products, pvi_evaluation* evals);
void simopt_run(const Model& m, const pvi_simopt_config& cfg, int* best, double* best_mean,
                double* best_sd, int* generations, pvi_scored_candidate* log, int log_capacity,
                int* n_logged, int* dimension, double* device_seconds);
void philox_block_device(const std::uint32_t ctr[4], const std::uint32_t key[2], std::uint32_t out[4]);
void rollout_draws_device(std::uint64_t seed, std::uint64_t rollout, std::uint32_t day, int n,
                          std::uint64_t* out);

}  // namespace pvi_b200
