// The reference-side drop-in, compiled and run.
//
// Built by `make -C oracle dropin` against the UNMODIFIED reference headers
// (/root/reference/proj/include, tests/support) and objects (oracle/_ref/obj),
// this repo's include/pvi/b200.hpp and libpvi_b200.so; run on the GPU box by
// tests/test_gpu_dropin.py.  Every case calls the reference's own template
// (CPU, all host threads) and the pvi::b200 overload on the same inputs and
// compares the results BIT FOR BIT (the engine's exact kernels follow the
// reference's per-term order):
//
//  - test_vi.cpp:31-104 through b200 (self-loop backup, geometric fixed
//    point, random 30x4x5 backup vs naive_q_row, 10 brute-force trials,
//    argmax ties), with TabularMdp tabulated through the MdpModel concept;
//  - run_value_iteration on presets of all three scenarios (f64 and f32,
//    fixed sweeps, resume from a reference checkpoint);
//  - the error taxonomy (ParameterError, CapacityError::required_count,
//    FingerprintMismatch);
//  - evaluate_policy (heuristic and VI-table policies) and simopt's
//    grid_search / ga_search driven by the b200 candidate evaluator.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <functional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "pvi/b200.hpp"
#include "pvi/policies.hpp"
#include "pvi/presets.hpp"
#include "pvi/simopt.hpp"
#include "pvi/vi.hpp"
#include "support/oracles.hpp"
#include "support/tabular_mdp.hpp"

using namespace pvi;
using pvi::testing::TabularMdp;

namespace {

int g_pass = 0, g_fail = 0;

void check(bool ok, const std::string& name, const std::string& detail = "") {
  if (ok) {
    ++g_pass;
    std::printf("ok   %s\n", name.c_str());
  } else {
    ++g_fail;
    std::printf("FAIL %s %s\n", name.c_str(), detail.c_str());
  }
  std::fflush(stdout);
}

template <typename F>
void guarded(const std::string& name, F&& f) {
  try {
    f();
  } catch (const std::exception& e) {
    check(false, name, std::string("threw: ") + e.what());
  }
}

int host_threads() {
  const unsigned n = std::thread::hardware_concurrency();
  return n ? static_cast<int>(n) : 1;
}

template <typename F>
void with_preset(const std::string& name, F&& f) {
  const ExperimentConfig c = make_preset(name);
  if (c.scenario == 'a') {
    ScenarioA m(c.a);
    f(m, c);
  } else if (c.scenario == 'b') {
    ScenarioB m(c.b);
    f(m, c);
  } else {
    ScenarioC m(c.c);
    f(m, c);
  }
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

std::string describe(const ViResult& r, const ViResult& w) {
  std::size_t diff = 0, first = r.vf.values.size();
  for (std::size_t i = 0; i < r.vf.values.size() && i < w.vf.values.size(); ++i)
    if (std::memcmp(&r.vf.values[i], &w.vf.values[i], 8) != 0) {
      ++diff;
      if (first == r.vf.values.size()) first = i;
    }
  char buf[256];
  std::snprintf(buf, sizeof buf, "(iters %llu vs %llu, %zu values differ, first %zu)",
                static_cast<unsigned long long>(r.iterations), static_cast<unsigned long long>(w.iterations),
                diff, first);
  return buf;
}

bool same_result(const ViResult& got, const ViResult& want) {
  return got.iterations == want.iterations && got.converged == want.converged &&
         got.vf.iteration == want.vf.iteration && got.vf.fingerprint == want.vf.fingerprint &&
         same_bits(got.vf.values, want.vf.values) && got.policy.actions == want.policy.actions;
}

bool same_eval(const Evaluation& a, const Evaluation& b) {
  auto eq = [](const KpiStat& x, const KpiStat& y) {
    return std::memcmp(&x.mean, &y.mean, 8) == 0 && std::memcmp(&x.sd, &y.sd, 8) == 0;
  };
  bool ok = eq(a.ret, b.ret) && a.products == b.products && a.n_rollouts == b.n_rollouts;
  for (int k = 0; k < a.products; ++k)
    ok = ok && eq(a.service_pct[k], b.service_pct[k]) && eq(a.wastage_pct[k], b.wastage_pct[k]) &&
         eq(a.holding_mean[k], b.holding_mean[k]);
  return ok;
}

TabularMdp self_loop_unit_reward(double gamma) {
  TabularMdp mdp(1, 1, 1, gamma);
  mdp.at_next(0, 0, 0) = 0;
  mdp.at_reward(0, 0, 0) = 1.0;
  mdp.at_prob(0, 0, 0) = 1.0;
  return mdp;
}

// ---- test_vi.cpp:31-104, through the engine ------------------------------
void test_vi_cases() {
  guarded("test_vi: single backup of a one-state self loop", [] {
    const auto mdp = self_loop_unit_reward(0.5);
    std::vector<double> values{0.0}, out(1);
    std::vector<std::uint32_t> act(1, 7);
    b200::bellman_backup_batch<double>(mdp, values, 0, 1, 0.5, out, act);
    check(out[0] == 1.0 && act[0] == 0, "test_vi: single backup of a one-state self loop");
  });
  guarded("test_vi: geometric-series fixed point", [] {
    const auto mdp = self_loop_unit_reward(0.5);
    ViConfig config;
    config.epsilon = 1e-10;
    const auto got = b200::run_value_iteration(mdp, config);
    const auto want = run_value_iteration(mdp, config);
    check(got.converged && std::fabs(got.vf.values[0] - 2.0) <= 2.0 * 1e-8 && got.policy.actions[0] == 0 &&
              same_result(got, want),
          "test_vi: geometric-series fixed point (and bitwise = reference)", describe(got, want));
  });
  guarded("test_vi: batched backup equals the naive triple-loop oracle", [] {
    const auto mdp = TabularMdp::random(30, 4, 5, 0.9, 1234);
    std::mt19937_64 rng(99);
    std::vector<double> values(30);
    for (auto& v : values) v = std::uniform_real_distribution<double>(-5.0, 5.0)(rng);
    std::vector<double> out(30), ref_out(30);
    std::vector<std::uint32_t> act(30), ref_act(30);
    b200::bellman_backup_batch<double>(mdp, values, 0, 30, 0.9, out, act);
    bellman_backup_batch<double>(mdp, values, 0, 30, 0.9, ref_out, ref_act);
    bool ok = same_bits(out, ref_out) && act == ref_act;
    for (std::uint64_t s = 0; s < 30; ++s) {
      const auto q = pvi::testing::naive_q_row(mdp, s, 0.9, values);
      double best = q[0];
      std::uint32_t best_a = 0;
      for (std::uint32_t a = 1; a < q.size(); ++a)
        if (q[a] > best) {
          best = q[a];
          best_a = a;
        }
      ok = ok && std::fabs(out[s] - best) <= 1e-12 * std::fabs(best) && act[s] == best_a;
    }
    check(ok, "test_vi: batched backup equals the naive triple-loop oracle (and the reference bitwise)");
  });
  guarded("test_vi: brute-force policy enumeration", [] {
    std::mt19937_64 seeds(2024);
    bool ok = true;
    for (int trial = 0; trial < 10; ++trial) {
      const std::uint64_t n_states = 3 + seeds() % 6;
      const std::uint32_t n_actions = 2 + seeds() % 2;
      const auto mdp = TabularMdp::random(n_states, n_actions, 4, 0.9, seeds());
      ViConfig config;
      config.epsilon = 1e-12;
      const auto result = b200::run_value_iteration(mdp, config);
      const auto oracle = pvi::testing::brute_force_solve(mdp);
      const auto want = run_value_iteration(mdp, config);
      ok = ok && same_result(result, want);
      for (std::uint64_t s = 0; s < n_states; ++s)
        ok = ok && result.policy.actions[s] == oracle.optimal_policy[s] &&
             std::fabs(result.vf.values[s] - oracle.optimal_values[s]) <=
                 1e-6 * std::max(1.0, std::fabs(oracle.optimal_values[s]));
    }
    check(ok, "test_vi: extracted policies match brute-force policy enumeration (10 trials)");
  });
  guarded("test_vi: argmax ties", [] {
    TabularMdp mdp(1, 3, 1, 0.0);
    for (std::uint32_t a = 0; a < 3; ++a) {
      mdp.at_next(0, a, 0) = 0;
      mdp.at_reward(0, a, 0) = 1.0;
      mdp.at_prob(0, a, 0) = 1.0;
    }
    std::vector<double> values{0.0}, out(1);
    std::vector<std::uint32_t> act(1, 9);
    b200::bellman_backup_batch<double>(mdp, values, 0, 1, 0.0, out, act);
    check(act[0] == 0, "test_vi: argmax ties break toward the smallest action index");
  });
}

// ---- run_value_iteration on presets --------------------------------------
void test_presets() {
  struct Case {
    const char* preset;
    Precision prec;
    std::uint64_t fixed;
  };
  const Case cases[] = {{"a/m2/exp1", Precision::f64, 0}, {"a/m2/exp2", Precision::f64, 0},
                        {"a/m3/exp5", Precision::f64, 0}, {"a/m2/exp1", Precision::f32, 0},
                        {"b/m2/exp1", Precision::f64, 0}, {"b/m2/exp2", Precision::f64, 0},
                        {"b/m2/p1", Precision::f64, 100}, {"b/m3/exp4", Precision::f64, 2},
                        {"c/m3/exp1", Precision::f64, 0}, {"c/m3/exp2", Precision::f64, 0},
                        {"c/m3/exp1", Precision::f32, 0}};
  for (const Case& c : cases) {
    const std::string name = std::string("run_value_iteration ") + c.preset +
                             (c.prec == Precision::f32 ? " f32" : " f64") +
                             (c.fixed ? " fixed " + std::to_string(c.fixed) : "");
    guarded(name, [&] {
      with_preset(c.preset, [&](const auto& model, const ExperimentConfig&) {
        ViConfig config;
        config.precision = c.prec;
        config.fixed_iterations = c.fixed;
        config.threads = host_threads();
        const auto t0 = std::chrono::steady_clock::now();
        const ViResult want = run_value_iteration(model, config);
        const auto t1 = std::chrono::steady_clock::now();
        const ViResult got = b200::run_value_iteration(model, config);
        const auto t2 = std::chrono::steady_clock::now();
        char t[128];
        std::snprintf(t, sizeof t, " [%llu sweeps; reference %.3f s, b200 %.3f s]",
                      static_cast<unsigned long long>(got.iterations),
                      std::chrono::duration<double>(t1 - t0).count(),
                      std::chrono::duration<double>(t2 - t1).count());
        check(same_result(got, want), name + t, describe(got, want));
      });
    });
  }
  // resume from a checkpoint the reference wrote (acceptance_main.cpp:303-325 shape)
  for (const char* preset : {"a/m2/exp1", "c/m3/exp2", "b/m2/exp1"}) {
    const std::string name = std::string("resume from a reference checkpoint ") + preset;
    guarded(name, [&] {
      with_preset(preset, [&](const auto& model, const ExperimentConfig&) {
        const auto path = std::filesystem::temp_directory_path() /
                          ("dropin_" + std::to_string(std::hash<std::string>{}(preset)) + ".ckpt");
        ViConfig part;
        part.fixed_iterations = 5;
        part.checkpoint_every = 1;
        part.checkpoint_path = path;
        part.threads = host_threads();
        (void)run_value_iteration(model, part);
        const Checkpoint ck = load_checkpoint(path, sha256_fingerprint(model.fingerprint_material()));
        ViConfig rest;
        rest.threads = host_threads();
        const ViResult want = run_value_iteration(model, rest, &ck);
        const ViResult got = b200::run_value_iteration(model, rest, &ck);
        std::filesystem::remove(path);
        check(ck.iteration == 5 && same_result(got, want), name, describe(got, want));
      });
    });
  }
}

// ---- error taxonomy ------------------------------------------------------
void test_errors() {
  with_preset("a/m2/exp1", [&](const auto& model, const ExperimentConfig&) {
    bool ok = false;
    try {
      ViConfig c;
      c.epsilon = 0.0;
      (void)b200::run_value_iteration(model, c);
    } catch (const ParameterError&) {
      ok = true;
    } catch (...) {
    }
    check(ok, "errors: epsilon <= 0 -> ParameterError (vi.hpp:298)");
    ok = false;
    try {
      ViConfig c;
      c.max_states = 100;
      (void)b200::run_value_iteration(model, c);
    } catch (const CapacityError& e) {
      ok = e.required_count() == model.state_count();
    } catch (...) {
    }
    check(ok, "errors: capacity gate -> CapacityError(required_count) (vi.hpp:167-171)");
    ok = false;
    try {
      Checkpoint bad;
      bad.values.assign(model.state_count(), 0.0);
      bad.fingerprint[0] = 1;
      (void)b200::run_value_iteration(model, ViConfig{}, &bad);
    } catch (const FingerprintMismatch&) {
      ok = true;
    } catch (...) {
    }
    check(ok, "errors: resume with a foreign checkpoint -> FingerprintMismatch (vi.hpp:187-190)");
  });
  bool ok = false;
  try {
    const ExperimentConfig c = make_preset("c/m8/exp1");
    ScenarioC m(c.c);
    (void)b200::run_value_iteration(m, ViConfig{});
  } catch (const CapacityError& e) {
    ok = e.required_count() == 12607619787ull;
  } catch (...) {
  }
  check(ok, "errors: c/m8/exp1 refused with CapacityError(12,607,619,787) (acceptance_main.cpp:368-385)");
}

// ---- simulation and simopt -----------------------------------------------
void test_simulation() {
  struct Case {
    const char* preset;
    std::vector<int> params;
  };
  const Case cases[] = {{"a/m2/exp1", {5}}, {"b/m2/exp1", {13, 12}},
                        {"c/m3/exp1", {9, 7, 7, 6, 6, 3, 3, 13, 14, 14, 10, 11, 8, 8}}};
  for (const Case& c : cases) {
    const std::string name = std::string("evaluate_policy heuristic ") + c.preset;
    guarded(name, [&] {
      with_preset(c.preset, [&](const auto& model, const ExperimentConfig&) {
        RolloutConfig rc;
        rc.n_rollouts = 2000;
        rc.base_seed = 42;
        rc.threads = host_threads();
        const Evaluation want = evaluate_policy(model, make_heuristic_policy(model, c.params), rc);
        const Evaluation got = b200::evaluate_policy(model, b200::make_heuristic_policy(model, c.params), rc);
        char t[128];
        std::snprintf(t, sizeof t, " [mean %.17g]", got.ret.mean);
        check(same_eval(got, want), name + t);
      });
    });
  }
  guarded("evaluate_policy VI table b/m2/exp1", [&] {
    with_preset("b/m2/exp1", [&](const auto& model, const ExperimentConfig&) {
      ViConfig vc;
      vc.threads = host_threads();
      const ViResult vi = run_value_iteration(model, vc);
      RolloutConfig rc;
      rc.n_rollouts = 1000;
      rc.base_seed = 42;
      rc.threads = host_threads();
      const Evaluation want = evaluate_policy(model, make_vi_policy(model, vi.policy.actions), rc);
      const Evaluation got = b200::evaluate_policy(model, b200::make_vi_policy(model, vi.policy.actions), rc);
      check(same_eval(got, want), "evaluate_policy VI table b/m2/exp1");
    });
  });
  guarded("grid_search a/m2/exp1 with the b200 evaluator", [&] {
    with_preset("a/m2/exp1", [&](const auto& model, const ExperimentConfig&) {
      RolloutConfig rc;
      rc.n_rollouts = 4096;
      rc.base_seed = 42;
      const auto space = heuristic_space(model);
      const simopt::CandidateEvaluator ref_eval = [&](const std::vector<int>& cand) {
        const Evaluation e = evaluate_policy(model, make_heuristic_policy(model, cand), rc);
        return simopt::Score{e.ret.mean, e.ret.sd};
      };
      const auto want = simopt::grid_search(space, ref_eval, host_threads());
      const auto got = simopt::grid_search(space, b200::candidate_evaluator(model, rc), 1);
      bool ok = got.best == want.best && got.table.size() == want.table.size();
      for (std::size_t i = 0; ok && i < got.table.size(); ++i)
        ok = got.table[i].values == want.table[i].values && got.table[i].mean == want.table[i].mean &&
             got.table[i].sd == want.table[i].sd;
      // and the batched form scores the whole grid in one device launch
      std::vector<std::vector<int>> all;
      for (const auto& row : want.table) all.push_back(row.values);
      const auto batch = b200::evaluate_candidates(model, all, rc);
      for (std::size_t i = 0; ok && i < batch.size(); ++i)
        ok = batch[i].mean == want.table[i].mean && batch[i].sd == want.table[i].sd;
      char t[96];
      std::snprintf(t, sizeof t, " [best S=%d, mean %.17g]", got.best.at(0), got.best_score.mean);
      check(ok, std::string("grid_search a/m2/exp1 with the b200 evaluator") + t);
    });
  });
  guarded("ga_search b/m2/exp1 with the b200 evaluator", [&] {
    with_preset("b/m2/exp1", [&](const auto& model, const ExperimentConfig& cfg) {
      RolloutConfig rc;
      rc.n_rollouts = 4096;
      rc.base_seed = 42;
      simopt::GaConfig ga;
      ga.population = cfg.simopt.population;
      ga.max_generations = cfg.simopt.max_generations;
      ga.patience = cfg.simopt.patience;
      ga.seed = 1;
      ga.threads = 1;
      const auto got = simopt::ga_search(heuristic_space(model), b200::candidate_evaluator(model, rc), ga);
      // SURVEY App. B golden trajectory of the reference's cmd_simopt
      char t[128];
      std::snprintf(t, sizeof t, " [best (%d,%d) mean %.17g, %d generations, %zu logged]", got.best.at(0),
                    got.best.at(1), got.best_score.mean, got.generations, got.log.size());
      check(got.best == std::vector<int>{13, 12} && got.best_score.mean == 1632.6983642578125 &&
                got.generations == 7 && got.log.size() == 329,
            std::string("ga_search b/m2/exp1 with the b200 evaluator = reference trajectory") + t);
    });
  });
}

}  // namespace

int main() {
  std::printf("pvi_b200 %s, %d CUDA device(s), %d host threads\n", pvi_version(), pvi_device_count(),
              host_threads());
  test_vi_cases();
  test_presets();
  test_errors();
  test_simulation();
  std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
