/* pvi_b200 — C ABI of the B200-native value-iteration and policy-simulation
 * engine for the perishable-inventory MDPs of arXiv 2303.10672.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (proj/, C++20) has no FFI: its boundary is compile-time C++ polymorphism
 * over two concepts.  Each entry point below names the reference interface
 * it replaces; INTEGRATION.md shows the C++ overloads a maintainer adds to
 * the reference so that `run_value_iteration(model, config)` and
 * `evaluate_policy(sim, policy, config)` route here unchanged for callers.
 *
 * Conventions
 *  - Plain pointers and sizes only; every array is HOST memory unless the
 *    name says `_device`.  No torch / CUDA types appear in the signatures
 *    (a stream is passed as void*).
 *  - Every call returns a pvi_status (0 = ok).  The status codes mirror the
 *    reference exception taxonomy (proj/include/pvi/errors.hpp:11-57); the
 *    message is written into the caller's (err, errlen) buffer, and the
 *    numeric payload of CapacityError::required_count / NumericDivergence::
 *    iteration goes into *err_value where a call can raise them.
 *  - Precision: 0 = f64 (default, `double`), 1 = f32 (`float`), as
 *    ViConfig::precision (proj/include/pvi/vi.hpp:28,39).
 *  - There is no CPU fallback: with no usable CUDA device every compute call
 *    returns PVI_ERR_DEVICE.
 */
#ifndef PVI_B200_H
#define PVI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:11-57; exit codes runner.hpp:68-75) ------- */
typedef enum {
  PVI_OK = 0,
  PVI_ERR_FAILURE = 1,      /* anything else (exit code 1) */
  PVI_ERR_PARAMETER = 2,    /* ParameterError            -> exit 2 */
  PVI_ERR_CAPACITY = 3,     /* CapacityError(required)    -> exit 3 */
  PVI_ERR_DIVERGENCE = 4,   /* NumericDivergence(iter)    -> exit 4 */
  PVI_ERR_IO = 5,           /* IoError                    -> exit 5 */
  PVI_ERR_CONTRACT = 6,     /* ContractViolation          -> exit 1 */
  PVI_ERR_FORMAT = 7,       /* FormatError                -> exit 1 */
  PVI_ERR_FINGERPRINT = 8,  /* FingerprintMismatch        -> exit 1 */
  PVI_ERR_INDEXING = 9,     /* IndexingError              -> exit 1 */
  PVI_ERR_CONFIG = 10,      /* ConfigError                -> exit 2 */
  PVI_ERR_DEVICE = 11       /* CUDA / NCCL failure, or no device       */
} pvi_status;

/* Process exit code the reference CLI would use (runner.cpp:482-498). */
int pvi_exit_code(int status);

/* Library version string and the CUDA device count it sees. */
const char* pvi_version(void);
int pvi_device_count(void);

/* ---- scenario parameters (scenario_{a,b,c}.hpp Params structs) ---------- */

/* ScenarioAParams, proj/include/pvi/scenario_a.hpp:25-38 */
typedef struct {
  int useful_life;  /* m, 1..12 */
  int lead_time;    /* L >= 1 */
  int issuing;      /* 0 = fifo, 1 = lifo */
  int max_order;    /* A_max */
  int max_demand;   /* D_max */
  double unit_cost, holding_cost, shortage_cost, wastage_cost;
  double demand_mean, demand_cv, discount_factor;
} pvi_scenario_a_params;

/* ScenarioBParams, proj/include/pvi/scenario_b.hpp:21-35 */
typedef struct {
  int useful_life;                  /* m, 1..8 */
  double demand_mean_a, demand_mean_b;
  int max_order_a, max_order_b;     /* < 0: newsvendor-derived cap */
  double unit_cost_a, unit_cost_b, revenue_a, revenue_b;
  double substitution_prob;         /* rho in [0, 1] */
  double discount_factor;
} pvi_scenario_b_params;

/* ScenarioCParams, proj/include/pvi/scenario_c.hpp:25-44 */
#define PVI_C_MAX_LIFE 12
typedef struct {
  int useful_life;  /* m, 2..12 */
  int max_order;    /* A_max, also per-age capacity */
  int max_demand;   /* D_max */
  double fixed_order_cost, holding_cost, shortage_cost, wastage_cost;
  double discount_factor;
  double demand_successes[7];
  double demand_means[7];
  double life_intercepts[PVI_C_MAX_LIFE - 1]; /* first m-1 used */
  double life_slopes[PVI_C_MAX_LIFE - 1];
} pvi_scenario_c_params;

/* Default parameter blocks (the reference's member initialisers). */
void pvi_scenario_a_defaults(pvi_scenario_a_params* p);
void pvi_scenario_b_defaults(pvi_scenario_b_params* p);
void pvi_scenario_c_defaults(pvi_scenario_c_params* p);

/* ---- models --------------------------------------------------------------
 * A model is immutable after construction: the constructor
 * builds every probability table on the host exactly as the reference
 * scenario constructors do, and uploads them lazily to each device used.
 * Replaces: ScenarioA/B/C constructors (scenario_a.cpp:46-57,
 * scenario_b.cpp:36-60, scenario_c.cpp:37-62) and TabularMdp
 * (tests/support/tabular_mdp.hpp:16-119). */
typedef struct pvi_model pvi_model;

typedef enum { PVI_SCENARIO_A = 0, PVI_SCENARIO_B = 1, PVI_SCENARIO_C = 2, PVI_TABULAR = 3 } pvi_scenario;
typedef enum { PVI_TEST_VALUE_SPAN = 0, PVI_TEST_CHANGE_SPAN = 1, PVI_TEST_PERIODIC_SPAN = 2 } pvi_convergence_test;

int pvi_model_create_a(const pvi_scenario_a_params* p, pvi_model** out, char* err, size_t errlen);
int pvi_model_create_b(const pvi_scenario_b_params* p, pvi_model** out, char* err, size_t errlen);
int pvi_model_create_c(const pvi_scenario_c_params* p, pvi_model** out, char* err, size_t errlen);
/* Explicit-table MDP: next/reward/prob are |S|*|A|*|Omega| row-major by
 * (s, a, w); initial may be NULL (zeros).  Value-span test, periodicity 1. */
int pvi_model_create_tabular(uint64_t n_states, uint32_t n_actions, uint64_t n_outcomes,
                             double gamma, const uint64_t* next, const double* reward,
                             const double* prob, const double* initial, pvi_model** out,
                             char* err, size_t errlen);
/* Bundled presets (presets.cpp:70-130), e.g. "a/m2/exp1", "b/m3/exp1", "c/m5/exp1".
 * *fixed_iterations receives the preset's vi.fixed_iterations (100 for b/m2/p1..p4),
 * *checkpoint_every the preset's cadence (a: 100, b/c: 1); either may be NULL. */
int pvi_model_create_preset(const char* name, pvi_model** out, uint64_t* fixed_iterations,
                            uint64_t* checkpoint_every, char* err, size_t errlen);
void pvi_model_destroy(pvi_model* m);

typedef struct {
  int scenario;                 /* pvi_scenario */
  uint64_t state_count;         /* MdpModel::state_count */
  uint32_t action_count;        /* MdpModel::action_count */
  uint64_t outcome_count;       /* MdpModel::outcome_count */
  double discount;              /* MdpModel::discount */
  int default_convergence_test; /* pvi_convergence_test */
  int periodicity;              /* 1 or 7 */
  uint32_t state_arity;         /* TupleSpace arity */
  uint32_t action_arity;        /* Simulator::action_arity */
  int products;                 /* Simulator::products */
  double terms_per_sweep;       /* reference backup terms (s,a,w) per sweep */
  int max_order_a, max_order_b; /* B: resolved caps; A/C: max_order, 0 */
  double factored_fmas;         /* FP64 FMAs per full sweep of the factored kernels (B, C;
                                   A: = terms_per_sweep) -- the work the algorithm does */
  int receipt_exogenous;        /* C: receipt law independent of the order size */
} pvi_model_info;

int pvi_model_get_info(const pvi_model* m, pvi_model_info* out);
/* Text hashed into the checkpoint fingerprint (fingerprint_material()). */
int pvi_model_fingerprint_material(const pvi_model* m, char* buf, size_t len);
/* SHA-256 of fingerprint_material (checkpoint.cpp:30-34). */
int pvi_model_fingerprint(const pvi_model* m, uint8_t out[32]);
/* Copy a named host-built table (for table-parity tests): "a.pmf", "b.pmf_a",
 * "b.pmf_b", "b.sf_a", "b.sf_b", "b.pu", "b.pz", "b.pz_cum", "c.pmf" (7 x (D+1)),
 * "c.comp_probs", "c.receipt_probs".  *count receives the table length; pass
 * out=NULL to query it. */
int pvi_model_table(const pvi_model* m, const char* name, double* out, size_t* count);
/* TupleSpace::decode / encode (tuple_space.hpp:37-54). */
int pvi_model_decode(const pvi_model* m, uint64_t index, int* tuple);
int pvi_model_encode(const pvi_model* m, const int* tuple, uint64_t* index, char* err, size_t errlen);
/* Transition::next_state / reward and P(w | s, a) (model.hpp:20-46) on the host,
 * for the naive-oracle cross-checks. */
int pvi_model_transition(const pvi_model* m, uint64_t s, uint32_t a, uint64_t w,
                         uint64_t* next, double* reward, char* err, size_t errlen);
int pvi_model_outcome_probability(const pvi_model* m, uint64_t s, uint32_t a, uint64_t w,
                                  double* p);
/* MdpModel::initial_value for all states (B: expected one-step revenue, computed on the device). */
int pvi_model_initial_values(const pvi_model* m, double* out, char* err, size_t errlen);

/* ---- value iteration (vi.hpp:28-43, 162-302) ---------------------------- */

typedef struct {
  double epsilon;            /* 1e-4 */
  double gamma;              /* used when has_gamma != 0, else the model's discount */
  int has_gamma;
  uint64_t max_iterations;   /* 10'000, relative to the start/resume point */
  uint64_t fixed_iterations; /* > 0: run exactly this many sweeps (absolute), no test */
  uint64_t checkpoint_every; /* 0: none */
  const char* checkpoint_path; /* PVI1 file; NULL/"" disables checkpoints */
  int precision;             /* 0 f64, 1 f32 */
  int convergence_test;      /* -1: model default, else pvi_convergence_test */
  uint64_t max_states;       /* capacity gate, 200'000'000 */
  int device;                /* CUDA ordinal, -1 = current */
  int algorithm;             /* -1: the model's (pvi_model_set_algorithm), else pvi_algorithm */
  int loop;                  /* sweep loop control: -1 auto (graph-resident when no checkpoint
                                falls inside the loop), 0 host loop (one 32-byte read-back per
                                sweep), 1 graph-resident loop (CUDA graph with a device-evaluated
                                WHILE condition: no host round trip per sweep; the periodic span's
                                8-vector ring rotates through a chain of 8 IF nodes; PVI_ERR_PARAMETER
                                with checkpoints) */
  int l2_persist;            /* 1 on: an L2 access-policy window (persisting) over the value-vector
                                ring; 0 off; -1 auto: on for the exact kernels, off for the
                                factored sweeps (their traffic is the W / G tables) */
} pvi_vi_config;

/* Backup algorithm.  EXACT reproduces the reference's per-term expression
 * and summation order (bit-identical results).  FACTORED (all three
 * scenarios; tabular models keep EXACT) regroups the sums -- B: the separable
 * issued-pair law contracted first, with diagonal running sums; C: the
 * demand summed per post-delivery profile, then the multinomial receipt as a
 * chain of binomial passes; A: demand values that leave the same carried
 * stock merged -- doing 10^2-10^4x fewer operations per sweep; results agree
 * with the reference to rounding (V within 1e-12 per sweep, the north-star
 * 1e-9 contract at convergence), not bit for bit. */
typedef enum { PVI_ALGO_EXACT = 0, PVI_ALGO_FACTORED = 1 } pvi_algorithm;
/* Default algorithm of every sweep on this model (pvi_vi_backup, pvi_q_rows,
 * pvi_vi_sweep_device, and pvi_vi_solve with algorithm = -1). */
int pvi_model_set_algorithm(pvi_model* m, int algorithm);

void pvi_vi_config_defaults(pvi_vi_config* c);

typedef struct {
  uint64_t iterations;   /* ViResult::iterations */
  int converged;         /* ViResult::converged */
  double wall_seconds;   /* ViResult::wall_seconds */
  double sweep_seconds;  /* device time in backup sweeps (CUDA events) */
  uint64_t sweeps;       /* sweeps launched, incl. the policy-extraction sweep */
  double span_lo, span_hi; /* last convergence statistic (min/max, or 0/max|dV|) */
  double terms_per_sweep;
  uint64_t graph_sweeps; /* sweeps run inside the graph-resident loop */
  uint64_t l2_window_bytes; /* bytes covered by the persisting L2 window (0: none) */
  double l2_hit_ratio;   /* the window's hitRatio */
} pvi_vi_stats;

/* run_value_iteration(model, config, resume) (vi.hpp:295-302).
 * resume_values / resume_iteration / resume_fingerprint: a Checkpoint
 * (checkpoint.hpp:18-22); pass resume_values = NULL for a fresh start.
 * out_values: |S| doubles (ValueFunction::values, widened from f32 as the
 * reference does); out_policy: |S| u32 (Policy::actions).  Either may be NULL. */
int pvi_vi_solve(const pvi_model* m, const pvi_vi_config* cfg, const double* resume_values,
                 uint64_t resume_iteration, const uint8_t* resume_fingerprint,
                 double* out_values, uint32_t* out_policy, pvi_vi_stats* stats,
                 uint64_t* err_value, char* err, size_t errlen);

/* bellman_backup_batch (vi.hpp:82-92): one synchronous backup of states
 * [lo, hi) against `values` (|S| entries of the precision's type: double
 * or float).  out_values (hi-lo, same type) and out_actions (hi-lo) may be NULL. */
int pvi_vi_backup(const pvi_model* m, int precision, double gamma, const void* values,
                  uint64_t lo, uint64_t hi, void* out_values, uint32_t* out_actions,
                  char* err, size_t errlen);

/* q_row (model.hpp:25-29) for states [lo, hi): out_q is (hi-lo) x |A| of
 * the precision's type. */
int pvi_q_rows(const pvi_model* m, int precision, double gamma, const void* values,
               uint64_t lo, uint64_t hi, void* out_q, char* err, size_t errlen);

/* check_convergence (vi.hpp:107-158) over an explicit host history of
 * `n_hist` vectors (oldest..newest), each |S| entries of the precision's
 * type; evaluated by the device reduction kernel. */
int pvi_check_convergence(const pvi_model* m, int precision, int test, const void* const* history,
                          int n_hist, double gamma, double epsilon, uint64_t iteration,
                          int* converged, char* err, size_t errlen);

/* Device-resident sweep for the sharded multi-GPU driver (one rank's slice).
 * values_prev_device: |S| entries (full replica); values_next_device: |S|
 * entries, only [lo, hi) written; actions_device: NULL or |S| u32.
 * hist_device: NULL, or an array of `n_hist` device pointers (oldest..newest,
 * the newest being values_prev) for the periodic-span statistic.
 * stats_device: 4 doubles written by the fused reduction kernel, encoded so
 * that ONE element-wise MAX all-reduce over ranks combines shards:
 *   [0] max(stat), [1] -min(stat), [2] -(first non-finite state), [3] 0.
 * Sentinels: [0] and [1] are -DBL_MAX for an empty range; [2] is -DBL_MAX
 * when every state is finite (a bad state s arrives as -s, so after the
 * MAX the smallest bad state wins).  stat is |dV| (value span), dV (change
 * span) or D(s) (periodic span).
 * want_stats = 0 skips the reduction.  stream: cudaStream_t or NULL. */
int pvi_vi_sweep_device(const pvi_model* m, int precision, double gamma,
                        const void* values_prev_device, void* values_next_device,
                        uint32_t* actions_device, uint64_t lo, uint64_t hi, int test,
                        const void* const* hist_device, int n_hist, int want_stats,
                        double* stats_device, void* stream, char* err, size_t errlen);

/* pvi_vi_sweep_device with the exchange fused into the sweep: the kernel
 * that finishes a state's V' also stores it into peers' replicas over
 * NVLink peer memory, so the refresh overlaps the sweep instead of
 * following it.  For the factored Scenario B x_3-pair sweep (whose read set
 * is a function of the shard) each entry goes only to the peers whose next
 * sweep reads it; for every other sweep (which gathers from all of V) every
 * entry of [lo, hi) goes to every peer (full replicas).  peer_vnext: the
 * peers' next-value buffers mapped into this process (pvi_ipc_open);
 * peer_lo / peer_hi: the peers' shards.  After the peers' sweeps the caller
 * synchronises the ranks (the convergence statistics' all-reduce does; the
 * kernels fence their peer stores system-wide before it).
 * PVI_ERR_PARAMETER for periodic span (its 8-vector ring is refreshed by the
 * caller) and for > 8 peers. */
int pvi_vi_sweep_device_peers(const pvi_model* m, int precision, double gamma,
                              const void* values_prev_device, void* values_next_device, uint64_t lo,
                              uint64_t hi, int test, int want_stats, double* stats_device, void* stream,
                              int n_peers, void* const* peer_values_next, const uint64_t* peer_lo,
                              const uint64_t* peer_hi, char* err, size_t errlen);

/* Unit shards (factored Scenario B x_3-pair sweep only): unit u = pair * G + g,
 * G = |x_b| / 16 column groups; a shard is a contiguous unit range, i.e. a
 * few (x_3 pair, x_b column range) blocks, so shards can be cut finer than
 * whole pairs.  pvi_unit_partition: cost-weighted unit bounds (parts + 1).
 * pvi_unit_runs: which = 0 the shard's own states, 1 the V runs its sweep
 * reads (own states included); sorted disjoint runs[2i] .. runs[2i+1].
 * pvi_vi_sweep_device_units: the shard's sweep (f64), with the optional
 * fused peer stores of pvi_vi_sweep_device_peers (peers by unit range). */
int pvi_unit_count(const pvi_model* m, uint64_t* count);
int pvi_unit_partition(const pvi_model* m, int parts, uint64_t* bounds);
int pvi_unit_runs(const pvi_model* m, uint64_t u_lo, uint64_t u_hi, int which, uint64_t* runs,
                  size_t capacity, size_t* count);
int pvi_vi_sweep_device_units(const pvi_model* m, int precision, double gamma,
                              const void* values_prev_device, void* values_next_device,
                              uint32_t* actions_device, uint64_t u_lo, uint64_t u_hi, int test,
                              int want_stats, double* stats_device, void* stream, int n_peers,
                              void* const* peer_values_next, const uint64_t* peer_u_lo,
                              const uint64_t* peer_u_hi, char* err, size_t errlen);

/* Device buffers shareable across processes (cudaMalloc, whole allocation)
 * and their CUDA IPC handles (64 bytes): the peer buffers of
 * pvi_vi_sweep_device_peers.  pvi_ipc_open maps a peer's buffer into this
 * process (on the current device); pvi_ipc_close unmaps it. */
int pvi_device_alloc(uint64_t bytes, void** out, char* err, size_t errlen);
int pvi_device_free(void* p);
int pvi_ipc_get_handle(void* device_ptr, uint8_t handle[64], char* err, size_t errlen);
int pvi_ipc_open(const uint8_t handle[64], void** device_ptr, char* err, size_t errlen);
int pvi_ipc_close(void* device_ptr);

/* Cost-weighted contiguous partition of the state space into `parts`
 * shards (bounds has parts+1 entries), aligned to the kernel's state tiles. */
int pvi_partition(const pvi_model* m, int parts, uint64_t* bounds);

/* The parts of V a sweep of shard [lo, hi) reads (with the model's current
 * algorithm), as sorted disjoint state runs: runs[2i] .. runs[2i+1].  A
 * multi-GPU driver only has to refresh these between sweeps: for the
 * factored Scenario B sweep of an x_3-pair shard that is ~1/8 of V per pair
 * plus the shard's own states; every other sweep reads all of V (one run).
 * *count receives the number of runs; pass runs = NULL to query it. */
int pvi_sweep_read_runs(const pvi_model* m, uint64_t lo, uint64_t hi, uint64_t* runs, size_t capacity,
                        size_t* count);

/* ---- simulation (sim.hpp:40-170, rng.hpp, policies.hpp) ----------------- */

typedef struct {
  int horizon_days;   /* 365 */
  int warmup_days;    /* 100 */
  int n_rollouts;     /* 10'000 */
  uint64_t base_seed; /* 0 */
  int device;         /* -1 = current */
} pvi_rollout_config;

void pvi_rollout_config_defaults(pvi_rollout_config* c);

/* RolloutSummary (sim.hpp:47-52), flattened. */
typedef struct {
  double ret;
  double service_pct[2];
  double wastage_pct[2];
  double holding_mean[2];
} pvi_rollout_summary;

/* Evaluation (sim.hpp:59-67): (mean, sd) per KPI. */
typedef struct {
  double ret_mean, ret_sd;
  double service_mean[2], service_sd[2];
  double wastage_mean[2], wastage_sd[2];
  double holding_mean[2], holding_sd[2];
  int products;
  int n_rollouts;
} pvi_evaluation;

/* Policy descriptor replacing the per-day std::function PolicyFn
 * (sim.hpp:37, policies.hpp:18-82):
 *   kind 0 = VI table: `table` holds |S| action indices (make_vi_policy);
 *   kind 1 = heuristic: `params` as heuristic_space (policies.hpp:44-59):
 *            A {S}, B {S_a, S_b}, C {s_0..s_6, S_0..S_6}. */
typedef struct {
  int kind;
  const uint32_t* table;
  int params[14];
  int n_params;
} pvi_policy;

/* evaluate_policy for a BATCH of policies on common random numbers
 * (sim.hpp:145-170, called once per candidate by simopt.cpp:33,77).
 * per_rollout: NULL or n_policies x n_rollouts summaries; evals: n_policies
 * Evaluations (index-order reduction exactly as detail::reduce). */
int pvi_sim_evaluate(const pvi_model* m, const pvi_policy* policies, uint32_t n_policies,
                     const pvi_rollout_config* cfg, pvi_rollout_summary* per_rollout,
                     pvi_evaluation* evals, char* err, size_t errlen);

/* detail::reduce (sim.hpp:128-141) on the host: per policy and KPI, the mean
 * (sequential sum in rollout-index order / n) and the two-pass sample sd,
 * the same operations as the device reduction inside pvi_sim_evaluate, so
 * per-rollout summaries gathered from several devices (rollout shards:
 * rollout i of a shard starting at rollout f is rollout f + i of the whole
 * evaluation when its base_seed is base_seed + f, rng.hpp:37-44) reduce to
 * the single-device Evaluation bit for bit.  per_rollout: n_policies x
 * n_rollouts summaries. */
int pvi_sim_reduce(const pvi_rollout_summary* per_rollout, uint32_t n_policies, int n_rollouts, int products,
                   pvi_evaluation* evals, char* err, size_t errlen);

/* ---- simulation optimisation (simopt.hpp, runner.cpp:352-403) ----------
 * The reference's grid search / generational GA (simopt.cpp:22-161), run on
 * the host exactly as the reference runs it (std::mt19937_64 and the
 * libstdc++ distributions, so the search trajectory is the reference's),
 * with each generation's fresh candidates scored in ONE batched device
 * evaluation (pvi_sim_evaluate) instead of one evaluate_policy per candidate. */
/* Scores a batch of heuristic candidates (n x dimension ints, row-major) into
 * means[n] / sds[n]; returns 0, or nonzero to abort the search.  Lets a
 * caller put the batch point on other devices: the multi-GPU driver
 * (sharded_sim.py) runs the same GA on every rank and shards each
 * generation's candidates (or rollouts) across the ranks inside it. */
typedef int (*pvi_score_batch_fn)(void* user, const int* candidates, int n, int dimension, double* means,
                                  double* sds);

typedef struct {
  int sampler;                 /* 0 auto (grid if 1-D, else GA), 1 grid, 2 GA, 3 exhaustive
                                  grid over the whole product space in one batch (GPU-only
                                  extra mode; PVI_ERR_PARAMETER above 1e6 candidates) */
  int population;              /* 50 */
  int max_generations;         /* 100 */
  int patience;                /* 5 */
  double crossover_rate;       /* 0.9 */
  double mutation_rate;        /* 0 = 1/dimension */
  uint64_t seed;               /* GA seed, 1 */
  int rollouts_per_candidate;  /* 4000 */
  int horizon_days;            /* 365 */
  int warmup_days;             /* 100 */
  uint64_t base_seed;          /* eval.base_seed, 42 */
  int device;                  /* -1 = current */
  pvi_score_batch_fn score_batch; /* NULL: pvi_sim_evaluate on `device` (the default) */
  void* score_user;            /* passed to score_batch */
} pvi_simopt_config;

void pvi_simopt_config_defaults(pvi_simopt_config* c);

/* One logged candidate (ScoredCandidate, simopt.hpp:39-44). */
typedef struct {
  int generation;
  int values[14];
  double mean, sd;
} pvi_scored_candidate;

/* best: dimension ints; log: up to log_capacity entries (n_logged gets the
 * full count); device_seconds: time inside the batched device evaluations. */
int pvi_simopt(const pvi_model* m, const pvi_simopt_config* cfg, int* best, double* best_mean,
               double* best_sd, int* generations, pvi_scored_candidate* log, int log_capacity,
               int* n_logged, int* dimension, double* device_seconds, char* err, size_t errlen);

/* Philox4x32-10 block and RolloutRng draws evaluated ON THE DEVICE
 * (rng.hpp:15-60), for known-answer tests. */
int pvi_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
int pvi_rollout_draws(uint64_t base_seed, uint64_t rollout, uint32_t day, int n, uint64_t* out);

/* ---- measurement hook (bench.py) ----------------------------------------
 * While enabled, every launch of a main backup kernel (K1) is bracketed by
 * CUDA events on the stream it runs on, and every kernel the VI path
 * launches is counted.  Read returns the summed K1 milliseconds, the K1
 * launch count and the total launch count since the last enable/read, and
 * resets them (it synchronises on the recorded events). */
int pvi_profile_enable(int on);
int pvi_profile_read(double* kernel_ms, uint64_t* kernel_launches, uint64_t* all_launches);
/* Simulation side of the hook: while enabled, every pvi_sim_evaluate counts
 * the Philox4x32-10 blocks its rollouts draw (one per uniform, rng.hpp:37-60)
 * and times its rollout kernel with CUDA events.  Returns the sums since the
 * last read (rollout_days = policies x rollouts x (warm-up + horizon)) and
 * resets them. */
int pvi_profile_sim_read(uint64_t* philox_blocks, uint64_t* rollout_days, double* kernel_ms);

/* ---- policy CSV (runner.cpp:90-166, io.cpp:53-92) -----------------------
 * Formatting and parsing run on the device, one thread per row.
 * pvi_policy_csv_format writes the BODY of policy_to_csv (one row per state:
 * the decoded tuple, then the action fields; no header line) into out;
 * out = NULL returns the byte length in *length.
 * pvi_policy_csv_parse is policy_from_csv after the metadata check: the
 * whole file text (header included) -> |S| actions, with the reference's
 * FormatError (row count, field count, non-numeric) and IndexingError
 * (tuple range) for the first bad row in file order; a state named twice
 * takes the last row's action, states never named take 0. */
int pvi_policy_csv_format(const pvi_model* m, const uint32_t* actions, char* out, uint64_t capacity,
                          uint64_t* length, char* err, size_t errlen);
int pvi_policy_csv_parse(const pvi_model* m, const char* text, uint64_t length, uint32_t* actions,
                         char* err, size_t errlen);

/* ---- checkpoints (checkpoint.hpp:24-35) --------------------------------- */
int pvi_checkpoint_save(const char* path, const double* values, uint64_t count, uint64_t iteration,
                        const uint8_t fingerprint[32], char* err, size_t errlen);
/* Two-phase load: values=NULL returns count/iteration/fingerprint only.
 * expected_fingerprint non-NULL -> PVI_ERR_FINGERPRINT on mismatch. */
int pvi_checkpoint_load(const char* path, const uint8_t* expected_fingerprint, double* values,
                        uint64_t capacity, uint64_t* count, uint64_t* iteration,
                        uint8_t fingerprint[32], char* err, size_t errlen);
int pvi_sha256(const void* data, size_t len, uint8_t out[32]);

#ifdef __cplusplus
}
#endif

#endif /* PVI_B200_H */
