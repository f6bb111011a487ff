// pvi/b200.hpp — the REFERENCE-SIDE binding of the B200 engine.
//
// A maintainer copies this header into the reference tree
// (proj/include/pvi/b200.hpp), links libpvi_b200.so, and calls
// pvi::b200::run_value_iteration / bellman_backup_batch / evaluate_policy /
// the batched candidate evaluator wherever the reference calls its own
// templates.  Every function keeps the reference signature and semantics:
//
//   run_value_iteration(model, ViConfig, const Checkpoint*)   vi.hpp:295-302
//   bellman_backup_batch<T>(model, values, lo, hi, gamma, ..) vi.hpp:82-92
//   evaluate_policy(sim, policy, RolloutConfig)               sim.hpp:145-170
//   CandidateEvaluator (one candidate) / evaluate_candidates  simopt.hpp:35,
//     (a whole generation in one device batch)                simopt.cpp:65-83
//
// and throws the reference's exception types (errors.hpp:11-57) with their
// payloads (CapacityError::required_count, NumericDivergence::iteration).
// ScenarioA/B/C map onto the engine's scenario kernels; any other MdpModel
// (e.g. tests/support TabularMdp) is tabulated through the concept's
// transition() / outcome_probability() / initial_value() and solved by the
// engine's explicit-table kernel.  The one non-drop-in spot: PolicyFn is a
// per-day std::function the device cannot call, so evaluate_policy takes a
// b200::Policy descriptor built by b200::make_vi_policy /
// b200::make_heuristic_policy (same arguments as policies.hpp:18-82).
//
// Compiled and run against the unmodified reference by tests/dropin/
// (dropin_main.cpp; built by `make -C oracle dropin`).
#pragma once

#include <pvi_b200.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "pvi/checkpoint.hpp"
#include "pvi/errors.hpp"
#include "pvi/model.hpp"
#include "pvi/scenario_a.hpp"
#include "pvi/scenario_b.hpp"
#include "pvi/scenario_c.hpp"
#include "pvi/sim.hpp"
#include "pvi/simopt.hpp"
#include "pvi/vi.hpp"

namespace pvi::b200 {

// pvi_status -> the reference exception taxonomy (errors.hpp:11-57).
[[noreturn]] inline void rethrow(int st, const char* msg, std::uint64_t value) {
  switch (st) {
    case PVI_ERR_PARAMETER: throw ParameterError(msg);
    case PVI_ERR_CONFIG: throw ConfigError(msg);
    case PVI_ERR_CAPACITY: throw CapacityError(msg, value);
    case PVI_ERR_DIVERGENCE: throw NumericDivergence(msg, value);
    case PVI_ERR_IO: throw IoError(msg);
    case PVI_ERR_CONTRACT: throw ContractViolation(msg);
    case PVI_ERR_FORMAT: throw FormatError(msg);
    case PVI_ERR_FINGERPRINT: throw FingerprintMismatch(msg);
    case PVI_ERR_INDEXING: throw IndexingError(msg);
    default: throw Error(std::string("pvi_b200: ") + msg);
  }
}

// Error buffer of one C-ABI call.
struct Status {
  char msg[1024] = {};
  std::uint64_t value = 0;
  void check(int st) const {
    if (st != PVI_OK) rethrow(st, msg, value);
  }
};

// An engine-side model (pvi_model) built from the reference's own model
// object; immutable, like the reference's.
class Model {
 public:
  explicit Model(const ScenarioA& m) {
    const auto& q = m.params();
    pvi_scenario_a_params p;
    pvi_scenario_a_defaults(&p);
    p.useful_life = q.useful_life;
    p.lead_time = q.lead_time;
    p.issuing = q.issuing == Issuing::fifo ? 0 : 1;
    p.max_order = q.max_order;
    p.max_demand = q.max_demand;
    p.unit_cost = q.unit_cost;
    p.holding_cost = q.holding_cost;
    p.shortage_cost = q.shortage_cost;
    p.wastage_cost = q.wastage_cost;
    p.demand_mean = q.demand_mean;
    p.demand_cv = q.demand_cv;
    p.discount_factor = q.discount_factor;
    Status s;
    s.check(pvi_model_create_a(&p, &h_, s.msg, sizeof s.msg));
  }
  explicit Model(const ScenarioB& m) {
    const auto& q = m.params();
    pvi_scenario_b_params p;
    pvi_scenario_b_defaults(&p);
    p.useful_life = q.useful_life;
    p.demand_mean_a = q.demand_mean_a;
    p.demand_mean_b = q.demand_mean_b;
    p.max_order_a = m.max_order_a();  // resolved caps (newsvendor-derived when < 0)
    p.max_order_b = m.max_order_b();
    p.unit_cost_a = q.unit_cost_a;
    p.unit_cost_b = q.unit_cost_b;
    p.revenue_a = q.revenue_a;
    p.revenue_b = q.revenue_b;
    p.substitution_prob = q.substitution_prob;
    p.discount_factor = q.discount_factor;
    Status s;
    s.check(pvi_model_create_b(&p, &h_, s.msg, sizeof s.msg));
  }
  explicit Model(const ScenarioC& m) {
    const auto& q = m.params();
    pvi_scenario_c_params p;
    pvi_scenario_c_defaults(&p);
    p.useful_life = q.useful_life;
    p.max_order = q.max_order;
    p.max_demand = q.max_demand;
    p.fixed_order_cost = q.fixed_order_cost;
    p.holding_cost = q.holding_cost;
    p.shortage_cost = q.shortage_cost;
    p.wastage_cost = q.wastage_cost;
    p.discount_factor = q.discount_factor;
    for (int t = 0; t < 7; ++t) {
      p.demand_successes[t] = q.demand_successes[t];
      p.demand_means[t] = q.demand_means[t];
    }
    if (q.life_intercepts.size() > PVI_C_MAX_LIFE - 1 || q.life_slopes.size() > PVI_C_MAX_LIFE - 1)
      throw ParameterError("scenario c: useful_life out of range");
    for (std::size_t k = 0; k < q.life_intercepts.size(); ++k) p.life_intercepts[k] = q.life_intercepts[k];
    for (std::size_t k = 0; k < q.life_slopes.size(); ++k) p.life_slopes[k] = q.life_slopes[k];
    Status s;
    s.check(pvi_model_create_c(&p, &h_, s.msg, sizeof s.msg));
  }
  // Any other MdpModel: explicit (s, a, w) tables from the concept's
  // transition / outcome_probability / initial_value (model.hpp:30-46).
  template <MdpModel M>
  static Model tabulate(const M& m) {
    const std::uint64_t ns = m.state_count(), no = m.outcome_count();
    const std::uint32_t na = m.action_count();
    const std::uint64_t cells = ns * na * no;
    std::vector<std::uint64_t> next(cells);
    std::vector<double> reward(cells), prob(cells), init(ns);
    for (std::uint64_t s = 0; s < ns; ++s) {
      init[s] = m.initial_value(s);
      for (std::uint32_t a = 0; a < na; ++a)
        for (std::uint64_t w = 0; w < no; ++w) {
          const std::uint64_t i = (s * na + a) * no + w;
          const Transition t = m.transition(s, a, w);
          next[i] = t.next_state;
          reward[i] = t.reward;
          prob[i] = m.outcome_probability(s, a, w);
        }
    }
    Model out;
    Status st;
    st.check(pvi_model_create_tabular(ns, na, no, m.discount(), next.data(), reward.data(), prob.data(),
                                      init.data(), &out.h_, st.msg, sizeof st.msg));
    return out;
  }
  Model(Model&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Model& operator=(Model&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;
  ~Model() {
    if (h_) pvi_model_destroy(h_);
  }
  const pvi_model* get() const { return h_; }
  pvi_model* get() { return h_; }

  // PVI_ALGO_EXACT (default: the reference's per-term order, bit-identical)
  // or PVI_ALGO_FACTORED (~1e-12 agreement, far fewer operations).
  Model& set_algorithm(int algorithm) {
    Status s;
    s.check(pvi_model_set_algorithm(h_, algorithm));
    return *this;
  }

 private:
  Model() = default;
  pvi_model* h_ = nullptr;
};

template <MdpModel M>
Model make_model(const M& m) {
  if constexpr (std::is_same_v<M, ScenarioA> || std::is_same_v<M, ScenarioB> ||
                std::is_same_v<M, ScenarioC>)
    return Model(m);
  else
    return Model::tabulate(m);
}

inline pvi_vi_config to_c(const ViConfig& c, const std::string& path) {
  pvi_vi_config cfg;
  pvi_vi_config_defaults(&cfg);
  cfg.epsilon = c.epsilon;
  if (c.gamma) {
    cfg.gamma = *c.gamma;
    cfg.has_gamma = 1;
  }
  cfg.max_iterations = c.max_iterations;
  cfg.fixed_iterations = c.fixed_iterations;
  cfg.checkpoint_every = c.checkpoint_every;
  cfg.checkpoint_path = path.c_str();
  cfg.precision = c.precision == Precision::f32 ? 1 : 0;
  cfg.convergence_test = c.convergence_test ? static_cast<int>(*c.convergence_test) : -1;
  cfg.max_states = c.max_states;
  // max_batch_size and threads shape the reference's CPU partition only;
  // its results are invariant to both (vi.hpp:17-23), as the device's are.
  return cfg;
}

// run_value_iteration (vi.hpp:295-302) on the engine's model.
inline ViResult run_value_iteration(const Model& m, std::uint64_t n_states, const Fingerprint& fp,
                                    const ViConfig& config, const Checkpoint* resume = nullptr) {
  if (!(config.epsilon > 0.0)) throw ParameterError("value iteration: epsilon must be > 0");
  const std::string path = config.checkpoint_path.string();
  const pvi_vi_config cfg = to_c(config, path);
  ViResult r;
  r.vf.values.resize(n_states);
  r.policy.actions.resize(n_states);
  pvi_vi_stats stats{};
  Status s;
  s.check(pvi_vi_solve(m.get(), &cfg, resume ? resume->values.data() : nullptr,
                       resume ? resume->iteration : 0, resume ? resume->fingerprint.data() : nullptr,
                       r.vf.values.data(), r.policy.actions.data(), &stats, &s.value, s.msg,
                       sizeof s.msg));
  r.vf.iteration = r.iterations = stats.iterations;
  r.vf.fingerprint = fp;
  r.converged = stats.converged != 0;
  r.wall_seconds = stats.wall_seconds;
  return r;
}

template <MdpModel M>
ViResult run_value_iteration(const M& model, const ViConfig& config, const Checkpoint* resume = nullptr) {
  if (!(config.epsilon > 0.0)) throw ParameterError("value iteration: epsilon must be > 0");
  // the capacity gate before anything |S|-sized is built (vi.hpp:166-171)
  const std::uint64_t n = model.state_count();
  if (n > config.max_states)
    throw CapacityError("value iteration requires " + std::to_string(n) +
                            " states, exceeding the configured capacity of " +
                            std::to_string(config.max_states),
                        n);
  const Model m = make_model(model);
  return run_value_iteration(m, n, sha256_fingerprint(model.fingerprint_material()), config, resume);
}

// bellman_backup_batch (vi.hpp:82-92): one synchronous backup of [lo, hi).
template <typename T, MdpModel M>
void bellman_backup_batch(const M& model, std::span<const T> values, std::uint64_t lo, std::uint64_t hi,
                          double gamma, std::span<T> out_values, std::span<std::uint32_t> out_actions) {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>);
  const Model m = make_model(model);
  Status s;
  s.check(pvi_vi_backup(m.get(), std::is_same_v<T, float> ? 1 : 0, gamma, values.data(), lo, hi,
                        out_values.data(), out_actions.data(), s.msg, sizeof s.msg));
}

// ---- simulation ---------------------------------------------------------

// The device-callable form of a PolicyFn (sim.hpp:37, policies.hpp:18-82).
struct Policy {
  std::vector<std::uint32_t> table;  // make_vi_policy: one action index per state
  std::vector<int> params;           // make_heuristic_policy: heuristic_space order
  pvi_policy desc() const {
    pvi_policy p{};
    if (!table.empty()) {
      p.kind = 0;
      p.table = table.data();
    } else {
      p.kind = 1;
      if (params.size() > 14) throw ParameterError("heuristic policy: at most 14 parameters");
      for (std::size_t k = 0; k < params.size(); ++k) p.params[k] = params[k];
      p.n_params = static_cast<int>(params.size());
    }
    return p;
  }
};
template <typename S>
Policy make_vi_policy(const S&, std::vector<std::uint32_t> actions) {
  return Policy{std::move(actions), {}};
}
template <typename S>
Policy make_heuristic_policy(const S&, const std::vector<int>& params) {
  return Policy{{}, params};
}

inline pvi_rollout_config to_c(const RolloutConfig& c) {
  pvi_rollout_config r;
  pvi_rollout_config_defaults(&r);
  r.horizon_days = c.horizon_days;
  r.warmup_days = c.warmup_days;
  r.n_rollouts = c.n_rollouts;
  r.base_seed = c.base_seed;
  return r;
}

inline Evaluation to_evaluation(const pvi_evaluation& e) {
  Evaluation out;
  out.ret = {e.ret_mean, e.ret_sd};
  for (int k = 0; k < 2; ++k) {
    out.service_pct[k] = {e.service_mean[k], e.service_sd[k]};
    out.wastage_pct[k] = {e.wastage_mean[k], e.wastage_sd[k]};
    out.holding_mean[k] = {e.holding_mean[k], e.holding_sd[k]};
  }
  out.products = e.products;
  out.n_rollouts = e.n_rollouts;
  return out;
}

// evaluate_policy for a batch of policies on common random numbers (one
// device launch; each result equals the reference's evaluate_policy bit for
// bit, sim.hpp:145-170).
template <typename S>
std::vector<Evaluation> evaluate_policies(const S& sim, const std::vector<Policy>& policies,
                                          const RolloutConfig& config) {
  if (config.n_rollouts < 1) throw ParameterError("evaluation needs at least one rollout");
  const Model m(sim);
  std::vector<pvi_policy> descs;
  for (const auto& p : policies) descs.push_back(p.desc());
  const pvi_rollout_config rc = to_c(config);
  std::vector<pvi_evaluation> ev(policies.size());
  Status s;
  s.check(pvi_sim_evaluate(m.get(), descs.data(), static_cast<std::uint32_t>(descs.size()), &rc, nullptr,
                           ev.data(), s.msg, sizeof s.msg));
  std::vector<Evaluation> out;
  for (const auto& e : ev) out.push_back(to_evaluation(e));
  return out;
}

template <typename S>
Evaluation evaluate_policy(const S& sim, const Policy& policy, const RolloutConfig& config) {
  return evaluate_policies(sim, std::vector<Policy>{policy}, config)[0];
}

// The batched form of simopt::CandidateEvaluator (simopt.hpp:35): a whole
// generation of heuristic candidates scored in one device batch.
template <typename S>
std::vector<simopt::Score> evaluate_candidates(const S& sim, const std::vector<std::vector<int>>& candidates,
                                               const RolloutConfig& config) {
  std::vector<Policy> pols;
  for (const auto& c : candidates) pols.push_back(b200::make_heuristic_policy(sim, c));
  std::vector<simopt::Score> out;
  for (const auto& e : evaluate_policies(sim, pols, config)) out.push_back({e.ret.mean, e.ret.sd});
  return out;
}

// Drop-in simopt::CandidateEvaluator (one candidate per call), as
// runner.cpp:369-373 builds it.  The model must outlive the evaluator.
template <typename S>
simopt::CandidateEvaluator candidate_evaluator(const S& sim, const RolloutConfig& config) {
  return [&sim, config](const std::vector<int>& c) {
    return evaluate_candidates(sim, std::vector<std::vector<int>>{c}, config)[0];
  };
}

}  // namespace pvi::b200
