// extern "C" boundary (include/pvi_b200.h): argument checking, exception to
// status mapping, and the defaults of the reference's parameter structs.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "engine.hpp"
#include "vi_kernels.cuh"
#include "model.hpp"

using namespace pvi_b200;

struct pvi_model {
  std::unique_ptr<Model> impl;
};

namespace {

void write_err(char* err, std::size_t errlen, const char* msg) {
  if (err && errlen) std::snprintf(err, errlen, "%s", msg);
}

template <typename F>
int guarded(char* err, std::size_t errlen, std::uint64_t* err_value, F&& f) {
  if (err && errlen) err[0] = '\0';
  if (err_value) *err_value = 0;
  try {
    f();
    return PVI_OK;
  } catch (const Error& e) {
    write_err(err, errlen, e.what());
    if (err_value) *err_value = e.value;
    return e.status;
  } catch (const std::bad_alloc&) {
    write_err(err, errlen, "out of host memory");
    return PVI_ERR_FAILURE;
  } catch (const std::exception& e) {
    write_err(err, errlen, e.what());
    return PVI_ERR_FAILURE;
  }
}

const Model& M(const pvi_model* m) {
  if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
  return *m->impl;
}

}  // namespace

extern "C" {

int pvi_exit_code(int status) {
  switch (status) {
    case PVI_OK: return 0;
    case PVI_ERR_PARAMETER:
    case PVI_ERR_CONFIG: return 2;
    case PVI_ERR_CAPACITY: return 3;
    case PVI_ERR_DIVERGENCE: return 4;
    case PVI_ERR_IO: return 5;
    default: return 1;
  }
}

const char* pvi_version(void) { return "pvi_b200 0.1.0 (sm_100a)"; }

int pvi_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void pvi_scenario_a_defaults(pvi_scenario_a_params* p) {
  *p = pvi_scenario_a_params{};
  p->useful_life = 2;
  p->lead_time = 1;
  p->issuing = 1;
  p->max_order = 10;
  p->max_demand = 100;
  p->unit_cost = 3.0;
  p->holding_cost = 1.0;
  p->shortage_cost = 5.0;
  p->wastage_cost = 7.0;
  p->demand_mean = 4.0;
  p->demand_cv = 0.5;
  p->discount_factor = 0.99;
}

void pvi_scenario_b_defaults(pvi_scenario_b_params* p) {
  *p = pvi_scenario_b_params{};
  p->useful_life = 2;
  p->demand_mean_a = 5.0;
  p->demand_mean_b = 5.0;
  p->max_order_a = -1;
  p->max_order_b = -1;
  p->unit_cost_a = 0.5;
  p->unit_cost_b = 0.5;
  p->revenue_a = 1.0;
  p->revenue_b = 1.0;
  p->substitution_prob = 0.5;
  p->discount_factor = 1.0;
}

void pvi_scenario_c_defaults(pvi_scenario_c_params* p) {
  *p = pvi_scenario_c_params{};
  p->useful_life = 3;
  p->max_order = 20;
  p->max_demand = 20;
  p->fixed_order_cost = 10.0;
  p->holding_cost = 1.0;
  p->shortage_cost = 20.0;
  p->wastage_cost = 5.0;
  p->discount_factor = 0.95;
  const double n[7] = {3.5, 11.0, 7.2, 11.1, 5.9, 5.5, 2.2};
  const double d[7] = {5.7, 6.9, 6.5, 6.2, 5.8, 3.3, 3.4};
  for (int i = 0; i < 7; ++i) {
    p->demand_successes[i] = n[i];
    p->demand_means[i] = d[i];
  }
  p->life_intercepts[0] = 1.0;
  p->life_intercepts[1] = 0.5;
}

int pvi_model_create_a(const pvi_scenario_a_params* p, pvi_model** out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!p || !out) fail(PVI_ERR_PARAMETER, "null argument");
    *out = new pvi_model{build_scenario_a(*p)};
  });
}

int pvi_model_create_b(const pvi_scenario_b_params* p, pvi_model** out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!p || !out) fail(PVI_ERR_PARAMETER, "null argument");
    *out = new pvi_model{build_scenario_b(*p)};
  });
}

int pvi_model_create_c(const pvi_scenario_c_params* p, pvi_model** out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!p || !out) fail(PVI_ERR_PARAMETER, "null argument");
    *out = new pvi_model{build_scenario_c(*p)};
  });
}

int pvi_model_create_tabular(uint64_t n_states, uint32_t n_actions, uint64_t n_outcomes, double gamma,
                             const uint64_t* next, const double* reward, const double* prob,
                             const double* initial, pvi_model** out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!next || !reward || !prob || !out) fail(PVI_ERR_PARAMETER, "null argument");
    *out = new pvi_model{build_tabular(n_states, n_actions, n_outcomes, gamma, next, reward, prob, initial)};
  });
}

int pvi_model_create_preset(const char* name, pvi_model** out, uint64_t* fixed_iterations,
                            uint64_t* checkpoint_every, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!name || !out) fail(PVI_ERR_PARAMETER, "null argument");
    *out = new pvi_model{build_preset(name, fixed_iterations, checkpoint_every)};
  });
}

void pvi_model_destroy(pvi_model* m) { delete m; }

int pvi_model_get_info(const pvi_model* m, pvi_model_info* out) {
  return guarded(nullptr, 0, nullptr, [&] {
    const Model& md = M(m);
    pvi_model_info i{};
    i.scenario = md.scenario;
    i.state_count = md.space.count;
    i.action_count = md.n_actions;
    i.outcome_count = md.n_outcomes;
    i.discount = md.gamma;
    i.default_convergence_test = md.default_test;
    i.periodicity = md.periodicity;
    i.state_arity = static_cast<uint32_t>(md.space.radix.size());
    i.action_arity = md.scenario == PVI_SCENARIO_B ? 2 : 1;
    i.products = md.scenario == PVI_SCENARIO_B ? 2 : 1;
    i.terms_per_sweep = md.terms_per_sweep();
    i.factored_fmas = md.factored_fmas();
    i.receipt_exogenous = md.scenario == PVI_SCENARIO_C && md.c_exogenous ? 1 : 0;
    if (md.scenario == PVI_SCENARIO_B) {
      i.max_order_a = md.b_na - 1;
      i.max_order_b = md.b_nb - 1;
    } else if (md.scenario == PVI_SCENARIO_A) {
      i.max_order_a = md.pa.max_order;
    } else if (md.scenario == PVI_SCENARIO_C) {
      i.max_order_a = md.pc.max_order;
    }
    *out = i;
  });
}

int pvi_model_fingerprint_material(const pvi_model* m, char* buf, size_t len) {
  return guarded(nullptr, 0, nullptr, [&] {
    const Model& md = M(m);
    if (buf && len) std::snprintf(buf, len, "%s", md.fingerprint.c_str());
  });
}

int pvi_model_fingerprint(const pvi_model* m, uint8_t out[32]) {
  return guarded(nullptr, 0, nullptr, [&] {
    const Model& md = M(m);
    sha256(md.fingerprint.data(), md.fingerprint.size(), out);
  });
}

int pvi_model_table(const pvi_model* m, const char* name, double* out, size_t* count) {
  return guarded(nullptr, 0, nullptr, [&] {
    const Model& md = M(m);
    const std::string n = name ? name : "";
    const std::vector<double>* t = nullptr;
    if (n == "a.pmf") t = &md.a_pmf;
    else if (n == "a.cdf") t = &md.a_cdf;
    else if (n == "b.pmf_a") t = &md.b_pmf_a;
    else if (n == "b.pmf_b") t = &md.b_pmf_b;
    else if (n == "b.sf_a") t = &md.b_sf_a;
    else if (n == "b.sf_b") t = &md.b_sf_b;
    else if (n == "b.cdf_a") t = &md.b_cdf_a;
    else if (n == "b.cdf_b") t = &md.b_cdf_b;
    else if (n == "b.pu") t = &md.b_pu;
    else if (n == "b.pz") t = &md.b_pz;
    else if (n == "b.pz_cum") t = &md.b_pz_cum;
    else if (n == "c.pmf") t = &md.c_pmf;
    else if (n == "c.cdf") t = &md.c_cdf;
    else if (n == "c.comp_probs") t = &md.c_probs;
    else if (n == "c.receipt_probs") t = &md.c_receipt;
    if (!t) fail(PVI_ERR_PARAMETER, "unknown table: " + n);
    if (count) *count = t->size();
    if (out) std::memcpy(out, t->data(), t->size() * sizeof(double));
  });
}

int pvi_model_decode(const pvi_model* m, uint64_t index, int* tuple) {
  return guarded(nullptr, 0, nullptr, [&] {
    const Model& md = M(m);
    if (index >= md.space.count) fail(PVI_ERR_INDEXING, "index out of range");
    md.space.decode(index, tuple);
  });
}

int pvi_model_encode(const pvi_model* m, const int* tuple, uint64_t* index, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] { *index = M(m).space.encode(tuple); });
}

int pvi_model_transition(const pvi_model* m, uint64_t s, uint32_t a, uint64_t w, uint64_t* next,
                         double* reward, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] { host_transition(M(m), s, a, w, next, reward); });
}

int pvi_model_outcome_probability(const pvi_model* m, uint64_t s, uint32_t a, uint64_t w, double* p) {
  return guarded(nullptr, 0, nullptr, [&] { *p = host_outcome_probability(M(m), s, a, w); });
}

int pvi_model_initial_values(const pvi_model* m, double* out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] { initial_values_host(M(m), out); });
}

void pvi_vi_config_defaults(pvi_vi_config* c) {
  *c = pvi_vi_config{};
  c->epsilon = 1e-4;
  c->max_iterations = 10000;
  c->precision = 0;
  c->convergence_test = -1;
  c->max_states = 200000000ull;
  c->device = -1;
  c->algorithm = -1;
  c->loop = -1;
  c->l2_persist = -1;
}

int pvi_model_set_algorithm(pvi_model* m, int algorithm) {
  return guarded(nullptr, 0, nullptr, [&] {
    if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
    if (algorithm != PVI_ALGO_EXACT && algorithm != PVI_ALGO_FACTORED)
      fail(PVI_ERR_PARAMETER, "unknown algorithm");
    m->impl->algorithm = algorithm;
  });
}

int pvi_vi_solve(const pvi_model* m, const pvi_vi_config* cfg, const double* resume_values,
                 uint64_t resume_iteration, const uint8_t* resume_fingerprint, double* out_values,
                 uint32_t* out_policy, pvi_vi_stats* stats, uint64_t* err_value, char* err,
                 size_t errlen) {
  return guarded(err, errlen, err_value, [&] {
    pvi_vi_config c;
    if (cfg)
      c = *cfg;
    else
      pvi_vi_config_defaults(&c);
    vi_solve(M(m), c, resume_values, resume_iteration, resume_fingerprint, out_values, out_policy, stats);
  });
}

int pvi_vi_backup(const pvi_model* m, int precision, double gamma, const void* values, uint64_t lo,
                  uint64_t hi, void* out_values, uint32_t* out_actions, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!values) fail(PVI_ERR_PARAMETER, "null values");
    vi_backup(M(m), precision, gamma, values, lo, hi, out_values, out_actions, nullptr);
  });
}

int pvi_q_rows(const pvi_model* m, int precision, double gamma, const void* values, uint64_t lo,
               uint64_t hi, void* out_q, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!values || !out_q) fail(PVI_ERR_PARAMETER, "null argument");
    vi_backup(M(m), precision, gamma, values, lo, hi, nullptr, nullptr, out_q);
  });
}

int pvi_check_convergence(const pvi_model* m, int precision, int test, const void* const* history,
                          int n_hist, double gamma, double epsilon, uint64_t iteration, int* converged,
                          char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    *converged = check_convergence(M(m), precision, test, history, n_hist, gamma, epsilon, iteration) ? 1 : 0;
  });
}

int pvi_vi_sweep_device(const pvi_model* m, int precision, double gamma, const void* values_prev_device,
                        void* values_next_device, uint32_t* actions_device, uint64_t lo, uint64_t hi,
                        int test, const void* const* hist_device, int n_hist, int want_stats,
                        double* stats_device, void* stream, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    vi_sweep_device(M(m), precision, gamma, values_prev_device, values_next_device, actions_device, lo, hi,
                    test, hist_device, n_hist, want_stats, stats_device, stream);
  });
}

int pvi_partition(const pvi_model* m, int parts, uint64_t* bounds) {
  return guarded(nullptr, 0, nullptr, [&] { partition(M(m), parts, bounds); });
}

int pvi_vi_sweep_device_peers(const pvi_model* m, int precision, double gamma,
                              const void* values_prev_device, void* values_next_device, uint64_t lo,
                              uint64_t hi, int test, int want_stats, double* stats_device, void* stream,
                              int n_peers, void* const* peer_values_next, const uint64_t* peer_lo,
                              const uint64_t* peer_hi, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
    if (n_peers > 0 && (!peer_values_next || !peer_lo || !peer_hi)) fail(PVI_ERR_PARAMETER, "null peer arrays");
    vi_sweep_device_peers(M(m), precision, gamma, values_prev_device, values_next_device, lo, hi, test,
                          want_stats, stats_device, stream, n_peers, peer_values_next, peer_lo, peer_hi);
  });
}

int pvi_unit_count(const pvi_model* m, uint64_t* count) {
  return guarded(nullptr, 0, nullptr, [&] {
    if (!m || !m->impl || !count) fail(PVI_ERR_PARAMETER, "null argument");
    *count = unit_count(M(m));
  });
}

int pvi_unit_partition(const pvi_model* m, int parts, uint64_t* bounds) {
  return guarded(nullptr, 0, nullptr, [&] {
    if (!m || !m->impl || !bounds) fail(PVI_ERR_PARAMETER, "null argument");
    unit_partition(M(m), parts, bounds);
  });
}

int pvi_unit_runs(const pvi_model* m, uint64_t u_lo, uint64_t u_hi, int which, uint64_t* runs,
                  size_t capacity, size_t* count) {
  return guarded(nullptr, 0, nullptr, [&] {
    if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
    if (u_lo > u_hi || u_hi > unit_count(M(m))) fail(PVI_ERR_PARAMETER, "unit range out of bounds");
    const auto r = which == 0 ? unit_own_runs(M(m), u_lo, u_hi) : unit_read_runs(M(m), u_lo, u_hi);
    if (count) *count = r.size();
    if (runs) {
      if (capacity < r.size()) fail(PVI_ERR_PARAMETER, "unit_runs: capacity too small");
      for (std::size_t i = 0; i < r.size(); ++i) {
        runs[2 * i] = r[i].first;
        runs[2 * i + 1] = r[i].second;
      }
    }
  });
}

int pvi_vi_sweep_device_units(const pvi_model* m, int precision, double gamma,
                              const void* values_prev_device, void* values_next_device,
                              uint32_t* actions_device, uint64_t u_lo, uint64_t u_hi, int test,
                              int want_stats, double* stats_device, void* stream, int n_peers,
                              void* const* peer_values_next, const uint64_t* peer_u_lo,
                              const uint64_t* peer_u_hi, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
    if (n_peers > 0 && (!peer_values_next || !peer_u_lo || !peer_u_hi)) fail(PVI_ERR_PARAMETER, "null peer arrays");
    vi_sweep_device_units(M(m), precision, gamma, values_prev_device, values_next_device, actions_device, u_lo,
                          u_hi, test, want_stats, stats_device, stream, n_peers, peer_values_next, peer_u_lo,
                          peer_u_hi);
  });
}

int pvi_device_alloc(uint64_t bytes, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!out) fail(PVI_ERR_PARAMETER, "null out");
    select_device(-1);
    *out = nullptr;
    PVI_CUDA(cudaMalloc(out, bytes));
  });
}

int pvi_device_free(void* p) {
  return guarded(nullptr, 0, nullptr, [&] {
    if (p) PVI_CUDA(cudaFree(p));
  });
}

int pvi_ipc_get_handle(void* device_ptr, uint8_t handle[64], char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    cudaIpcMemHandle_t h;
    PVI_CUDA(cudaIpcGetMemHandle(&h, device_ptr));
    static_assert(sizeof(h) == 64, "CUDA IPC handle size");
    std::memcpy(handle, &h, 64);
  });
}

int pvi_ipc_open(const uint8_t handle[64], void** device_ptr, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    select_device(-1);
    PVI_CUDA(cudaIpcOpenMemHandle(device_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int pvi_ipc_close(void* device_ptr) {
  return guarded(nullptr, 0, nullptr, [&] { PVI_CUDA(cudaIpcCloseMemHandle(device_ptr)); });
}

int pvi_policy_csv_format(const pvi_model* m, const uint32_t* actions, char* out, uint64_t capacity,
                          uint64_t* length, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
    if (!actions) fail(PVI_ERR_PARAMETER, "null actions");
    const std::uint64_t l = policy_csv_format(M(m), actions, out, capacity);
    if (length) *length = l;
  });
}

int pvi_policy_csv_parse(const pvi_model* m, const char* text, uint64_t length, uint32_t* actions,
                         char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
    if (!text || !actions) fail(PVI_ERR_PARAMETER, "null buffer");
    policy_csv_parse(M(m), text, length, actions);
  });
}

int pvi_sweep_read_runs(const pvi_model* m, uint64_t lo, uint64_t hi, uint64_t* runs, size_t capacity,
                        size_t* count) {
  return guarded(nullptr, 0, nullptr, [&] {
    if (!m || !m->impl) fail(PVI_ERR_PARAMETER, "null model");
    if (lo > hi || hi > M(m).space.count) fail(PVI_ERR_PARAMETER, "state range out of bounds");
    const auto r = sweep_read_runs(M(m), lo, hi);
    if (count) *count = r.size();
    if (runs) {
      if (capacity < r.size()) fail(PVI_ERR_PARAMETER, "sweep_read_runs: capacity too small");
      for (std::size_t i = 0; i < r.size(); ++i) {
        runs[2 * i] = r[i].first;
        runs[2 * i + 1] = r[i].second;
      }
    }
  });
}

void pvi_rollout_config_defaults(pvi_rollout_config* c) {
  *c = pvi_rollout_config{};
  c->horizon_days = 365;
  c->warmup_days = 100;
  c->n_rollouts = 10000;
  c->base_seed = 0;
  c->device = -1;
}

int pvi_sim_evaluate(const pvi_model* m, const pvi_policy* policies, uint32_t n_policies,
                     const pvi_rollout_config* cfg, pvi_rollout_summary* per_rollout, pvi_evaluation* evals,
                     char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    pvi_rollout_config c;
    if (cfg)
      c = *cfg;
    else
      pvi_rollout_config_defaults(&c);
    if (n_policies && !policies) fail(PVI_ERR_PARAMETER, "null policies");
    sim_evaluate(M(m), policies, n_policies, c, per_rollout, evals);
  });
}

void pvi_simopt_config_defaults(pvi_simopt_config* c) {
  *c = pvi_simopt_config{};
  c->sampler = 0;
  c->population = 50;
  c->max_generations = 100;
  c->patience = 5;
  c->crossover_rate = 0.9;
  c->mutation_rate = 0.0;
  c->seed = 1;
  c->rollouts_per_candidate = 4000;
  c->horizon_days = 365;
  c->warmup_days = 100;
  c->base_seed = 42;
  c->device = -1;
}

int pvi_sim_reduce(const pvi_rollout_summary* per_rollout, uint32_t n_policies, int n_rollouts, int products,
                   pvi_evaluation* evals, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (n_rollouts < 1) fail(PVI_ERR_PARAMETER, "evaluation needs at least one rollout");
    if (products < 1 || products > 2) fail(PVI_ERR_PARAMETER, "products must be 1 or 2");
    if (n_policies && (!per_rollout || !evals)) fail(PVI_ERR_PARAMETER, "null argument");
    sim_reduce_host(reinterpret_cast<const double*>(per_rollout), n_policies, n_rollouts, products, evals);
  });
}

int pvi_simopt(const pvi_model* m, const pvi_simopt_config* cfg, int* best, double* best_mean,
               double* best_sd, int* generations, pvi_scored_candidate* log, int log_capacity,
               int* n_logged, int* dimension, double* device_seconds, char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!best || !best_mean || !best_sd || !generations || !n_logged)
      fail(PVI_ERR_PARAMETER, "null argument");
    pvi_simopt_config c;
    if (cfg)
      c = *cfg;
    else
      pvi_simopt_config_defaults(&c);
    if (c.sampler < 0 || c.sampler > 3) fail(PVI_ERR_PARAMETER, "simopt: unknown sampler");
    simopt_run(M(m), c, best, best_mean, best_sd, generations, log, log ? log_capacity : 0, n_logged,
               dimension, device_seconds);
  });
}

int pvi_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  return guarded(nullptr, 0, nullptr, [&] { philox_block_device(ctr, key, out); });
}

int pvi_rollout_draws(uint64_t base_seed, uint64_t rollout, uint32_t day, int n, uint64_t* out) {
  return guarded(nullptr, 0, nullptr, [&] { rollout_draws_device(base_seed, rollout, day, n, out); });
}

int pvi_checkpoint_save(const char* path, const double* values, uint64_t count, uint64_t iteration,
                        const uint8_t fingerprint[32], char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!path || !fingerprint || (count && !values)) fail(PVI_ERR_PARAMETER, "null argument");
    save_checkpoint(path, values, count, iteration, fingerprint);
  });
}

int pvi_checkpoint_load(const char* path, const uint8_t* expected_fingerprint, double* values,
                        uint64_t capacity, uint64_t* count, uint64_t* iteration, uint8_t fingerprint[32],
                        char* err, size_t errlen) {
  return guarded(err, errlen, nullptr, [&] {
    if (!path) fail(PVI_ERR_PARAMETER, "null path");
    load_checkpoint(path, expected_fingerprint, values, capacity, count, iteration, fingerprint);
  });
}

int pvi_profile_enable(int on) {
  return guarded(nullptr, 0, nullptr, [&] { profile_enable(on != 0); });
}

int pvi_profile_read(double* kernel_ms, uint64_t* kernel_launches, uint64_t* all_launches) {
  return guarded(nullptr, 0, nullptr, [&] { profile_read(kernel_ms, kernel_launches, all_launches); });
}

int pvi_profile_sim_read(uint64_t* philox_blocks, uint64_t* rollout_days, double* kernel_ms) {
  return guarded(nullptr, 0, nullptr, [&] { sim_profile_read(philox_blocks, rollout_days, kernel_ms); });
}

int pvi_sha256(const void* data, size_t len, uint8_t out[32]) {
  return guarded(nullptr, 0, nullptr, [&] { sha256(data, len, out); });
}

}  // extern "C"
