// Heuristic-parameter search (simopt.cpp:22-161) driving the batched device
// evaluator.  The proposal logic is the reference's algorithm restated: it
// is serial and bound to libstdc++'s <random> (mt19937_64 plus the
// implementation-defined uniform_int / uniform_real distributions), so it
// runs here on the host, compiled against the same libstdc++ as the
// reference, and reproduces the reference's trajectory exactly.  What moves
// to the GPU is the batch point: each generation's fresh candidates are
// scored in one pvi_sim_evaluate launch on common random numbers.
#include <algorithm>
#include <chrono>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "engine.hpp"
#include "model.hpp"

namespace pvi_b200 {

namespace {

struct Param {
  int lo, hi;
};
struct Score {
  double mean = 0.0, sd = 0.0;
};
struct Logged {
  int generation;
  std::vector<int> values;
  Score score;
};

// heuristic_space (policies.hpp:44-59)
std::vector<Param> search_space(const Model& m) {
  switch (m.scenario) {
    case PVI_SCENARIO_A:
      return {{0, m.pa.max_order}};
    case PVI_SCENARIO_B:
      return {{0, 2 * (m.b_na - 1)}, {0, 2 * (m.b_nb - 1)}};
    case PVI_SCENARIO_C: {
      std::vector<Param> s(14, Param{0, m.pc.max_order});
      return s;
    }
    default:
      fail(PVI_ERR_PARAMETER, "tabular models have no heuristic policy");
  }
}

// higher mean wins; equal means prefer the lexicographically smaller vector
bool better(const std::vector<int>& a, double ma, const std::vector<int>& b, double mb) {
  if (ma != mb) return ma > mb;
  return a < b;
}

class Evaluator {
 public:
  Evaluator(const Model& m, const pvi_simopt_config& c) : m_(m), fn_(c.score_batch), user_(c.score_user) {
    rc_.horizon_days = c.horizon_days;
    rc_.warmup_days = c.warmup_days;
    rc_.n_rollouts = c.rollouts_per_candidate;
    rc_.base_seed = c.base_seed;
    rc_.device = c.device;
  }
  std::vector<Score> operator()(const std::vector<const std::vector<int>*>& batch) {
    std::vector<Score> out(batch.size());
    if (batch.empty()) return out;
    if (fn_) {  // the caller's batch point (e.g. sharded over several GPUs)
      const int dim = static_cast<int>(batch[0]->size());
      std::vector<int> flat;
      flat.reserve(batch.size() * dim);
      for (const auto* c : batch) flat.insert(flat.end(), c->begin(), c->end());
      std::vector<double> means(batch.size()), sds(batch.size());
      const auto t0 = std::chrono::steady_clock::now();
      const int rc = fn_(user_, flat.data(), static_cast<int>(batch.size()), dim, means.data(), sds.data());
      seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (rc != 0) fail(PVI_ERR_FAILURE, "simopt: score_batch callback failed (" + std::to_string(rc) + ")");
      for (std::size_t i = 0; i < batch.size(); ++i) out[i] = {means[i], sds[i]};
      return out;
    }
    std::vector<pvi_policy> pols(batch.size());
    for (std::size_t i = 0; i < batch.size(); ++i) {
      pols[i] = pvi_policy{};
      pols[i].kind = 1;
      pols[i].n_params = static_cast<int>(batch[i]->size());
      for (std::size_t k = 0; k < batch[i]->size(); ++k) pols[i].params[k] = (*batch[i])[k];
    }
    std::vector<pvi_evaluation> ev(batch.size());
    const auto t0 = std::chrono::steady_clock::now();
    sim_evaluate(m_, pols.data(), static_cast<std::uint32_t>(pols.size()), rc_, nullptr, ev.data());
    seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (std::size_t i = 0; i < batch.size(); ++i) out[i] = {ev[i].ret_mean, ev[i].ret_sd};
    return out;
  }
  double seconds = 0.0;

 private:
  const Model& m_;
  pvi_score_batch_fn fn_ = nullptr;
  void* user_ = nullptr;
  pvi_rollout_config rc_{};
};

}  // namespace

void simopt_run(const Model& m, const pvi_simopt_config& cfg, int* best_out, double* best_mean,
                double* best_sd, int* generations_out, pvi_scored_candidate* log_out,
                int log_capacity, int* n_logged, int* dimension, double* device_seconds) {
  const auto space = search_space(m);
  const std::size_t dim = space.size();
  if (dimension) *dimension = static_cast<int>(dim);
  Evaluator evaluate(m, cfg);
  std::vector<Logged> log;
  std::vector<int> best;
  Score best_score;
  int generations = 1;
  int sampler = cfg.sampler;
  if (sampler == 0) sampler = dim == 1 ? 1 : 2;

  if (sampler == 1) {
    // grid_search (simopt.cpp:22-46)
    if (dim != 1) fail(PVI_ERR_CONTRACT, "grid search requires a one-parameter space");
    const Param p = space[0];
    if (p.lo > p.hi) fail(PVI_ERR_PARAMETER, "grid search: empty range");
    std::vector<std::vector<int>> cands;
    for (int v = p.lo; v <= p.hi; ++v) cands.push_back({v});
    std::vector<const std::vector<int>*> ptrs;
    for (auto& c : cands) ptrs.push_back(&c);
    const auto scores = evaluate(ptrs);
    for (std::size_t i = 0; i < cands.size(); ++i) {
      log.push_back({0, cands[i], scores[i]});
      if (i == 0 || scores[i].mean > best_score.mean) {
        best = cands[i];
        best_score = scores[i];
      }
    }
  } else if (sampler == 3) {
    // Exhaustive grid (GPU-only extra mode): every point of the
    // product space in ONE batched evaluation on common random numbers, in
    // lexicographic order; the best is the GA's order (higher mean, then the
    // lexicographically smaller vector), so it is the global optimum the GA
    // searches for (b/m2: 21 x 21 = 441 candidates).
    double count = 1.0;
    for (const Param& p : space) {
      if (p.lo > p.hi) fail(PVI_ERR_PARAMETER, "exhaustive grid: empty range");
      count *= static_cast<double>(p.hi - p.lo + 1);
    }
    if (count > 1e6)
      fail(PVI_ERR_PARAMETER, "exhaustive grid: " + std::to_string(static_cast<long long>(count)) +
                                  " candidates exceed the 1,000,000 limit (use the GA)");
    std::vector<std::vector<int>> cands;
    cands.reserve(static_cast<std::size_t>(count));
    std::vector<int> cur(dim);
    for (std::size_t g = 0; g < dim; ++g) cur[g] = space[g].lo;
    while (true) {
      cands.push_back(cur);
      std::size_t g = dim;
      while (g > 0 && cur[g - 1] == space[g - 1].hi) {
        cur[g - 1] = space[g - 1].lo;
        --g;
      }
      if (g == 0) break;
      ++cur[g - 1];
    }
    std::vector<const std::vector<int>*> ptrs;
    for (auto& c : cands) ptrs.push_back(&c);
    const auto scores = evaluate(ptrs);
    for (std::size_t i = 0; i < cands.size(); ++i) {
      log.push_back({0, cands[i], scores[i]});
      if (i == 0 || better(cands[i], scores[i].mean, best, best_score.mean)) {
        best = cands[i];
        best_score = scores[i];
      }
    }
  } else {
    // ga_search (simopt.cpp:48-161)
    if (cfg.population < 2) fail(PVI_ERR_PARAMETER, "ga search: population must be >= 2");
    std::mt19937_64 rng(cfg.seed);
    const double mutation_rate = cfg.mutation_rate > 0.0 ? cfg.mutation_rate : 1.0 / double(dim);
    auto uniform_gene = [&](std::size_t g) {
      return std::uniform_int_distribution<int>(space[g].lo, space[g].hi)(rng);
    };
    auto chance = [&](double rate) {
      return std::uniform_real_distribution<double>(0.0, 1.0)(rng) < rate;
    };
    std::map<std::vector<int>, Score> cache;
    auto score_batch = [&](const std::vector<std::vector<int>>& batch, int generation) {
      std::vector<const std::vector<int>*> fresh;
      for (const auto& cand : batch)
        if (!cache.count(cand)) {
          cache.emplace(cand, Score{});
          fresh.push_back(&cand);
        }
      const auto scores = evaluate(fresh);  // one device launch for the generation
      for (std::size_t i = 0; i < fresh.size(); ++i) {
        cache[*fresh[i]] = scores[i];
        log.push_back({generation, *fresh[i], scores[i]});
      }
    };
    auto rank_order = [&](std::vector<std::vector<int>>& pool) {
      std::sort(pool.begin(), pool.end(), [&](const auto& a, const auto& b) {
        const double ma = cache[a].mean, mb = cache[b].mean;
        if (ma != mb) return ma > mb;
        return a < b;
      });
      pool.erase(std::unique(pool.begin(), pool.end()), pool.end());
    };
    std::vector<std::vector<int>> population(cfg.population, std::vector<int>(dim));
    for (auto& cand : population)
      for (std::size_t g = 0; g < dim; ++g) cand[g] = uniform_gene(g);
    int stale = 0;
    for (int generation = 1; generation <= cfg.max_generations; ++generation) {
      score_batch(population, generation);
      rank_order(population);
      bool improved = false;
      if (best.empty() || better(population[0], cache[population[0]].mean, best, best_score.mean)) {
        if (best != population[0]) improved = true;
        best = population[0];
        best_score = cache[population[0]];
      }
      generations = generation;
      stale = improved ? 0 : stale + 1;
      if (stale >= cfg.patience) break;
      if (generation == cfg.max_generations) break;
      auto tournament = [&]() -> const std::vector<int>& {
        std::uniform_int_distribution<int> pick(0, static_cast<int>(population.size()) - 1);
        const int a = pick(rng);
        const int b = pick(rng);
        return population[std::min(a, b)];
      };
      std::vector<std::vector<int>> offspring;
      std::set<std::vector<int>> proposed;
      offspring.reserve(cfg.population);
      while (static_cast<int>(offspring.size()) < cfg.population) {
        std::vector<int> child;
        for (int attempt = 0; attempt < 8; ++attempt) {
          child = tournament();
          const std::vector<int>& other = tournament();
          if (chance(cfg.crossover_rate)) {
            for (std::size_t g = 0; g < dim; ++g)
              if (chance(0.5)) child[g] = other[g];
          }
          for (std::size_t g = 0; g < dim; ++g)
            if (chance(mutation_rate)) child[g] = uniform_gene(g);
          if (!cache.count(child) && !proposed.count(child)) break;
        }
        proposed.insert(child);
        offspring.push_back(std::move(child));
      }
      score_batch(offspring, generation + 1);
      for (auto& child : offspring) population.push_back(std::move(child));
      rank_order(population);
      if (static_cast<int>(population.size()) > cfg.population) population.resize(cfg.population);
    }
  }
  for (std::size_t k = 0; k < best.size(); ++k) best_out[k] = best[k];
  *best_mean = best_score.mean;
  *best_sd = best_score.sd;
  *generations_out = generations;
  *n_logged = static_cast<int>(log.size());
  for (int i = 0; i < static_cast<int>(log.size()) && i < log_capacity; ++i) {
    pvi_scored_candidate& e = log_out[i];
    e = pvi_scored_candidate{};
    e.generation = log[i].generation;
    for (std::size_t k = 0; k < log[i].values.size(); ++k) e.values[k] = log[i].values[k];
    e.mean = log[i].score.mean;
    e.sd = log[i].score.sd;
  }
  if (device_seconds) *device_seconds = evaluate.seconds;
}

}  // namespace pvi_b200
