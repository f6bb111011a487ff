/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
 * See pvi_oracle.c.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load this. */
#ifndef PVI_ORACLE_H
#define PVI_ORACLE_H

#include <stddef.h>
#include <stdint.h>

typedef struct orc_model orc_model;

/* returns NULL on an unknown preset or invalid parameters */
orc_model* orc_preset(const char* name);
void orc_free(orc_model* m);
uint64_t orc_states(const orc_model* m);
uint32_t orc_actions(const orc_model* m);
double orc_gamma(const orc_model* m);

/* One Bellman backup of [lo, hi) (vi.hpp:82-92), f64 (f32 = 0) or f32
 * (f32 = 1; values are read as double and narrowed).  Threads via OpenMP. */
void orc_backup_range(const orc_model* m, int f32, const double* values, uint64_t lo, uint64_t hi,
                      double* out_values, uint32_t* out_actions);
void orc_q_row(const orc_model* m, int f32, uint64_t s, const double* values, double* q);
void orc_initial_values(const orc_model* m, double* out);

/* run_value_iteration (vi.hpp:162-291) without checkpoints.  Returns 0 or
 * 4 (NumericDivergence at *err_iteration). */
int orc_vi_solve(const orc_model* m, int f32, uint64_t fixed_iterations, uint64_t max_iterations,
                 double epsilon, double* out_values, uint32_t* out_policy, uint64_t* iterations,
                 int* converged, uint64_t* err_iteration);

/* rollout summaries (sim.hpp:68-124): kind 0 = VI table, 1 = heuristic.
 * out: n x 7 doubles.  Returns 0, or 6 on an out-of-range policy action. */
int orc_rollouts(const orc_model* m, int kind, const uint32_t* table, const int* params,
                 int n_rollouts, int horizon, int warmup, uint64_t seed, double* out);
void orc_reduce(const double* xs, int n, int stride, double* mean, double* sd);

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#endif
