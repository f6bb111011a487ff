// TEST INFRASTRUCTURE ONLY — C entry points over the *unmodified* reference
// library (/root/reference/proj, compiled by oracle/Makefile into
// oracle/_ref/).  Used by tests/ to generate and check golden vectors and by
// bench.py's reference arm to time the reference CPU solver on the host's
// cores.  Nothing in the product links or loads this.
//
// Every function returns 0 on success or the reference runner's exit-code
// mapping (proj/src/runner.cpp:482-498) and writes the exception text into
// `err`.

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pvi/parallel.hpp"
#include "pvi/policies.hpp"
#include "pvi/presets.hpp"
#include "pvi/runner.hpp"
#include "pvi/sim.hpp"
#include "pvi/simopt.hpp"
#include "pvi/vi.hpp"
#include "support/oracles.hpp"
#include "support/tabular_mdp.hpp"

using namespace pvi;

namespace {

void set_err(char* err, std::size_t errlen, const char* msg) {
  if (err && errlen) {
    std::snprintf(err, errlen, "%s", msg);
  }
}

template <typename F>
int guarded(char* err, std::size_t errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    try {
      throw;
    } catch (...) {
      return exit_code_for_current_exception();
    }
  }
}

template <typename F>
void with_preset(const char* preset, F&& f) {
  const ExperimentConfig config = make_preset(preset);
  switch (config.scenario) {
    case 'a': {
      ScenarioA m(config.a);
      f(m);
      return;
    }
    case 'b': {
      ScenarioB m(config.b);
      f(m);
      return;
    }
    default: {
      ScenarioC m(config.c);
      f(m);
      return;
    }
  }
}

void fill_summary(const RolloutSummary& r, double* out) {
  out[0] = r.ret;
  out[1] = r.service_pct[0];
  out[2] = r.service_pct[1];
  out[3] = r.wastage_pct[0];
  out[4] = r.wastage_pct[1];
  out[5] = r.holding_mean[0];
  out[6] = r.holding_mean[1];
}

void fill_eval(const Evaluation& e, double* out) {
  const KpiStat stats[7] = {e.ret,          e.service_pct[0], e.service_pct[1], e.wastage_pct[0],
                            e.wastage_pct[1], e.holding_mean[0], e.holding_mean[1]};
  for (int i = 0; i < 7; ++i) {
    out[2 * i] = stats[i].mean;
    out[2 * i + 1] = stats[i].sd;
  }
}

template <typename M>
void run_eval(const M& model, const PolicyFn& policy, int n_rollouts, int horizon, int warmup,
              std::uint64_t seed, int threads, double* per_rollout, double* eval_out) {
  RolloutConfig rc;
  rc.horizon_days = horizon;
  rc.warmup_days = warmup;
  rc.n_rollouts = n_rollouts;
  rc.base_seed = seed;
  rc.threads = threads;
  if (per_rollout) {
    std::vector<RolloutSummary> res(n_rollouts);
    parallel_for_chunks(n_rollouts, 16, threads, [&](std::uint64_t lo, std::uint64_t hi) {
      for (std::uint64_t i = lo; i < hi; ++i) res[i] = rollout(model, policy, rc, static_cast<int>(i));
    });
    for (int i = 0; i < n_rollouts; ++i) fill_summary(res[i], per_rollout + 7 * i);
  }
  if (eval_out) fill_eval(evaluate_policy(model, policy, rc), eval_out);
}

}  // namespace

extern "C" {

int ref_model_counts(const char* preset, std::uint64_t* states, std::uint32_t* actions,
                     std::uint64_t* outcomes, double* gamma, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      *states = m.state_count();
      *actions = m.action_count();
      *outcomes = m.outcome_count();
      *gamma = m.discount();
    });
  });
}

int ref_hardware_threads() { return hardware_threads(); }

// run_value_iteration on a preset (vi.hpp:295).  out_values is |S| f64,
// out_policy |S| u32.  fixed_iterations / max_iterations follow ViConfig.
int ref_vi_solve(const char* preset, int f32, int threads, std::uint64_t fixed_iterations,
                 std::uint64_t max_iterations, double epsilon, std::uint64_t max_batch,
                 double* out_values, std::uint32_t* out_policy, std::uint64_t* out_iterations,
                 int* out_converged, double* out_wall, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      ViConfig vi;
      vi.epsilon = epsilon;
      vi.fixed_iterations = fixed_iterations;
      vi.max_iterations = max_iterations;
      vi.max_batch_size = max_batch;
      vi.threads = threads;
      vi.precision = f32 ? Precision::f32 : Precision::f64;
      const ViResult r = run_value_iteration(m, vi);
      if (out_values) std::memcpy(out_values, r.vf.values.data(), r.vf.values.size() * 8);
      if (out_policy) std::memcpy(out_policy, r.policy.actions.data(), r.policy.actions.size() * 4);
      *out_iterations = r.iterations;
      *out_converged = r.converged ? 1 : 0;
      *out_wall = r.wall_seconds;
    });
  });
}

// One Bellman backup of states [lo, hi) against `values` (|S| entries,
// narrowed to float when f32) with bellman_backup_batch (vi.hpp:82-92),
// spread over `threads` workers with the reference's own chunk scheduler.
int ref_backup_range(const char* preset, int f32, int threads, const double* values,
                     std::uint64_t lo, std::uint64_t hi, double* out_values,
                     std::uint32_t* out_actions, double* out_seconds, char* err,
                     std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      const std::uint64_t n = m.state_count();
      const std::uint64_t count = hi - lo;
      const double gamma = m.discount();
      auto run = [&](auto tag) {
        using T = decltype(tag);
        std::vector<T> v(values, values + n);
        std::vector<T> ov(count);
        std::vector<std::uint32_t> oa(count);
        const std::uint64_t chunk = std::max<std::uint64_t>(1, std::min<std::uint64_t>(
            65536, (count + 8 * threads - 1) / (8 * threads)));
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for_chunks(count, chunk, threads, [&](std::uint64_t a, std::uint64_t b) {
          bellman_backup_batch<T>(m, std::span<const T>(v), lo + a, lo + b, gamma,
                                  std::span<T>(ov.data() + a, b - a),
                                  std::span<std::uint32_t>(oa.data() + a, b - a));
        });
        *out_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (std::uint64_t i = 0; i < count; ++i) {
          if (out_values) out_values[i] = double(ov[i]);
          if (out_actions) out_actions[i] = oa[i];
        }
      };
      if (f32)
        run(float{});
      else
        run(double{});
    });
  });
}

int ref_q_row(const char* preset, int f32, std::uint64_t state, const double* values,
              double* out_q, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      const std::uint64_t n = m.state_count();
      const std::uint32_t na = m.action_count();
      if (f32) {
        std::vector<float> v(values, values + n), q(na);
        m.q_row(state, m.discount(), std::span<const float>(v), std::span<float>(q));
        for (std::uint32_t a = 0; a < na; ++a) out_q[a] = q[a];
      } else {
        std::vector<double> q(na);
        m.q_row(state, m.discount(), std::span<const double>(values, n), std::span<double>(q));
        for (std::uint32_t a = 0; a < na; ++a) out_q[a] = q[a];
      }
    });
  });
}

// naive_q_row (tests/support/oracles.hpp:19-32) through transition /
// outcome_probability: the independent triple-loop oracle.
int ref_naive_q_row(const char* preset, std::uint64_t state, const double* values, double* out_q,
                    char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      const auto q = pvi::testing::naive_q_row(m, state, m.discount(),
                                               std::span<const double>(values, m.state_count()));
      std::memcpy(out_q, q.data(), q.size() * 8);
    });
  });
}

int ref_initial_values(const char* preset, double* out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      parallel_for_chunks(m.state_count(), 4096, hardware_threads(),
                          [&](std::uint64_t lo, std::uint64_t hi) {
                            for (std::uint64_t s = lo; s < hi; ++s) out[s] = m.initial_value(s);
                          });
    });
  });
}

// Heuristic-policy evaluation (policies.hpp:61-82 + sim.hpp:145-170).
// per_rollout: n x 7 doubles (ret, service a/b, wastage a/b, holding a/b)
// or null; eval_out: 14 doubles (mean, sd) pairs in the same order.
int ref_eval_heuristic(const char* preset, const int* params, int n_params, int n_rollouts,
                       int horizon, int warmup, std::uint64_t seed, int threads,
                       double* per_rollout, double* eval_out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      std::vector<int> p(params, params + n_params);
      run_eval(m, make_heuristic_policy(m, p), n_rollouts, horizon, warmup, seed, threads,
               per_rollout, eval_out);
    });
  });
}

int ref_eval_table(const char* preset, const std::uint32_t* actions, int n_rollouts, int horizon,
                   int warmup, std::uint64_t seed, int threads, double* per_rollout,
                   double* eval_out, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      std::vector<std::uint32_t> table(actions, actions + m.state_count());
      run_eval(m, make_vi_policy(m, std::move(table)), n_rollouts, horizon, warmup, seed,
               threads, per_rollout, eval_out);
    });
  });
}

// cmd_simopt's search (runner.cpp:352-403) without the file outputs.
// log_values: up to max_log x dim ints; log_scores: max_log x 3 doubles
// (generation, mean, sd).
int ref_simopt(const char* preset, int rollouts, std::uint64_t eval_seed, std::uint64_t ga_seed,
               int threads, int* best, double* best_mean, double* best_sd, int* generations,
               int* n_logged, int max_log, int* log_values, double* log_scores, double* wall,
               char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    with_preset(preset, [&](const auto& m) {
      const auto t0 = std::chrono::steady_clock::now();
      const auto space = heuristic_space(m);
      RolloutConfig rc;
      rc.n_rollouts = rollouts;
      rc.base_seed = eval_seed;
      rc.threads = 1;
      const simopt::CandidateEvaluator evaluator = [&](const std::vector<int>& cand) {
        const Evaluation e = evaluate_policy(m, make_heuristic_policy(m, cand), rc);
        return simopt::Score{e.ret.mean, e.ret.sd};
      };
      std::vector<simopt::ScoredCandidate> log;
      std::vector<int> b;
      simopt::Score bs;
      int gens = 1;
      if (space.dimension() == 1) {
        const auto g = simopt::grid_search(space, evaluator, threads);
        b = g.best;
        bs = g.best_score;
        log = g.table;
      } else {
        simopt::GaConfig ga;
        ga.seed = ga_seed;
        ga.threads = threads;
        ga.rollouts_per_candidate = rollouts;
        const auto r = simopt::ga_search(space, evaluator, ga);
        b = r.best;
        bs = r.best_score;
        gens = r.generations;
        log = r.log;
      }
      for (std::size_t i = 0; i < b.size(); ++i) best[i] = b[i];
      *best_mean = bs.mean;
      *best_sd = bs.sd;
      *generations = gens;
      *n_logged = static_cast<int>(log.size());
      const std::size_t dim = space.dimension();
      for (std::size_t i = 0; i < log.size() && static_cast<int>(i) < max_log; ++i) {
        for (std::size_t g = 0; g < dim; ++g) log_values[i * dim + g] = log[i].values[g];
        log_scores[3 * i] = log[i].generation;
        log_scores[3 * i + 1] = log[i].mean;
        log_scores[3 * i + 2] = log[i].sd;
      }
      *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
  });
}

// --- table dumps for table-parity tests --------------------------------

int ref_table_a_pmf(const char* preset, double* pmf, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ExperimentConfig c = make_preset(preset);
    ScenarioA m(c.a);
    std::memcpy(pmf, m.demand_pmf().probs.data(), m.demand_pmf().probs.size() * 8);
  });
}

// Issued-pair pmf of one state (scenario_b.cpp:194-208): outcome_count doubles.
int ref_b_issued_pmf(const char* preset, std::uint64_t state, double* out, char* err,
                     std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ExperimentConfig c = make_preset(preset);
    ScenarioB m(c.b);
    const auto p = m.issued_joint_pmf(state);
    std::memcpy(out, p.data(), p.size() * 8);
  });
}

int ref_b_tables(const char* preset, int* caps /* A_a, A_b, d_max, y_max */, double* pu,
                 double* pz, double* pz_cum, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ExperimentConfig c = make_preset(preset);
    ScenarioB m(c.b);
    const auto& t = m.substitution_tables();
    caps[0] = m.max_order_a();
    caps[1] = m.max_order_b();
    caps[2] = t.d_max;
    caps[3] = t.y_max;
    if (pu) std::memcpy(pu, t.pu.data(), t.pu.size() * 8);
    if (pz) std::memcpy(pz, t.pz.data(), t.pz.size() * 8);
    if (pz_cum) std::memcpy(pz_cum, t.pz_cum.data(), t.pz_cum.size() * 8);
  });
}

// Scenario C: weekday pmfs (7 x (D_max+1)), and per action the composition
// ids / probs (concatenated in action order; offsets has A_max+2 entries).
int ref_c_tables(const char* preset, double* weekday_pmf, std::uint32_t* offsets,
                 std::uint32_t* ids, double* probs, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ExperimentConfig c = make_preset(preset);
    ScenarioC m(c.c);
    const int dn = c.c.max_demand + 1;
    for (int t = 0; t < 7; ++t) {
      const auto p = m.weekday_demand_pmf(t);
      std::memcpy(weekday_pmf + t * dn, p.probs.data(), dn * 8);
    }
    std::uint32_t off = 0;
    for (int a = 0; a <= c.c.max_order; ++a) {
      offsets[a] = off;
      const auto i = m.composition_ids(a);
      const auto p = m.composition_probs(a);
      if (ids) std::memcpy(ids + off, i.data(), i.size() * 4);
      if (probs) std::memcpy(probs + off, p.data(), p.size() * 8);
      off += static_cast<std::uint32_t>(i.size());
    }
    offsets[c.c.max_order + 1] = off;
  });
}

// --- tabular MDPs (tests/support/tabular_mdp.hpp) -------------------------

int ref_tabular_random(std::uint64_t ns, std::uint32_t na, std::uint64_t no, double gamma,
                       std::uint64_t seed, std::uint64_t* next, double* reward, double* prob) {
  auto mdp = pvi::testing::TabularMdp::random(ns, na, no, gamma, seed);
  for (std::uint64_t s = 0; s < ns; ++s)
    for (std::uint32_t a = 0; a < na; ++a)
      for (std::uint64_t w = 0; w < no; ++w) {
        const std::size_t i = (s * na + a) * no + w;
        next[i] = mdp.at_next(s, a, w);
        reward[i] = mdp.at_reward(s, a, w);
        prob[i] = mdp.at_prob(s, a, w);
      }
  return 0;
}

static pvi::testing::TabularMdp make_tabular(std::uint64_t ns, std::uint32_t na, std::uint64_t no,
                                             double gamma, const std::uint64_t* next,
                                             const double* reward, const double* prob,
                                             const double* initial) {
  pvi::testing::TabularMdp mdp(ns, na, no, gamma);
  for (std::uint64_t s = 0; s < ns; ++s) {
    if (initial) mdp.at_initial(s) = initial[s];
    for (std::uint32_t a = 0; a < na; ++a)
      for (std::uint64_t w = 0; w < no; ++w) {
        const std::size_t i = (s * na + a) * no + w;
        mdp.at_next(s, a, w) = next[i];
        mdp.at_reward(s, a, w) = reward[i];
        mdp.at_prob(s, a, w) = prob[i];
      }
  }
  return mdp;
}

int ref_tabular_solve(std::uint64_t ns, std::uint32_t na, std::uint64_t no, double gamma,
                      const std::uint64_t* next, const double* reward, const double* prob,
                      const double* initial, int f32, std::uint64_t fixed_iterations,
                      std::uint64_t max_iterations, double epsilon, std::uint64_t max_states,
                      double* out_values, std::uint32_t* out_policy, std::uint64_t* out_iterations,
                      int* out_converged, std::uint64_t* err_value, char* err,
                      std::size_t errlen) {
  *err_value = 0;
  return guarded(err, errlen, [&] {
    const auto mdp = make_tabular(ns, na, no, gamma, next, reward, prob, initial);
    ViConfig vi;
    vi.epsilon = epsilon;
    vi.fixed_iterations = fixed_iterations;
    vi.max_iterations = max_iterations;
    vi.max_states = max_states;
    vi.precision = f32 ? Precision::f32 : Precision::f64;
    try {
      const ViResult r = run_value_iteration(mdp, vi);
      std::memcpy(out_values, r.vf.values.data(), ns * 8);
      std::memcpy(out_policy, r.policy.actions.data(), ns * 4);
      *out_iterations = r.iterations;
      *out_converged = r.converged ? 1 : 0;
    } catch (const NumericDivergence& e) {
      *err_value = e.iteration();
      throw;
    } catch (const CapacityError& e) {
      *err_value = e.required_count();
      throw;
    }
  });
}

int ref_tabular_brute_force(std::uint64_t ns, std::uint32_t na, std::uint64_t no, double gamma,
                            const std::uint64_t* next, const double* reward, const double* prob,
                            double* out_values, std::uint32_t* out_policy) {
  const auto mdp = make_tabular(ns, na, no, gamma, next, reward, prob, nullptr);
  const auto sol = pvi::testing::brute_force_solve(mdp);
  std::memcpy(out_values, sol.optimal_values.data(), ns * 8);
  std::memcpy(out_policy, sol.optimal_policy.data(), ns * 4);
  return 0;
}

// The reference runner commands (runner.cpp:303-480), writing their files
// into out_dir: 0 = solve, 1 = simopt, 2 = evaluate (with the VI policy CSV
// and/or heuristic parameter file already in out_dir).  n_rollouts /
// rollouts_per_candidate overrides are applied when > 0.
int ref_cmd(const char* preset, int which, const char* out_dir, int threads, int n_rollouts,
            const char* policy_csv, const char* heuristic_file, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    ExperimentConfig cfg = make_preset(preset);
    if (n_rollouts > 0) {
      cfg.eval.n_rollouts = n_rollouts;
      cfg.simopt.rollouts_per_candidate = n_rollouts;
    }
    RunnerOptions opt;
    opt.output_dir = out_dir;
    opt.threads = threads;
    if (which == 0) {
      (void)cmd_solve(cfg, opt);
    } else if (which == 1) {
      (void)cmd_simopt(cfg, opt);
    } else {
      std::optional<std::filesystem::path> vp, hp;
      if (policy_csv && policy_csv[0]) vp = policy_csv;
      if (heuristic_file && heuristic_file[0]) hp = heuristic_file;
      (void)cmd_evaluate(cfg, opt, vp, hp);
    }
  });
}

// cmd_solve with vi.fixed_iterations overridden and optionally resuming from
// the directory's checkpoint (acceptance_main.cpp:303-325 flow).
int ref_cmd_solve_fixed(const char* preset, const char* out_dir, int threads, std::uint64_t fixed_iterations,
                        int resume, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    ExperimentConfig cfg = make_preset(preset);
    cfg.vi.fixed_iterations = fixed_iterations;
    RunnerOptions opt;
    opt.output_dir = out_dir;
    opt.threads = threads;
    opt.resume = resume != 0;
    (void)cmd_solve(cfg, opt);
  });
}

// Raw Philox block (rng.hpp:15-33) and RolloutRng draws (rng.hpp:37-60).
void ref_philox_block(const std::uint32_t* ctr, const std::uint32_t* key, std::uint32_t* out) {
  const auto o = Philox4x32::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = o[i];
}

void ref_rollout_draws(std::uint64_t seed, std::uint64_t rollout, std::uint32_t day, int n,
                       std::uint64_t* out) {
  RolloutRng rng(seed, rollout);
  rng.begin_day(day);
  for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
}

}  // extern "C"
