// Host-side model: parameters, mixed-radix state space and the probability
// tables the device kernels read.  The tables are built exactly as the
// reference scenario constructors build theirs (same formulas, same
// operation order, same libm), so the kernels consume bit-identical inputs;
// tests/test_tables.py pins that against the compiled reference.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pvi_b200.h"

namespace pvi_b200 {

// ---- error taxonomy (errors.hpp:11-57) mapped to pvi_status --------------
struct Error : std::runtime_error {
  int status;
  std::uint64_t value;
  Error(int st, const std::string& what, std::uint64_t v = 0)
      : std::runtime_error(what), status(st), value(v) {}
};
[[noreturn]] inline void fail(int st, const std::string& what, std::uint64_t v = 0) {
  throw Error(st, what, v);
}

// ---- mixed-radix index space (tuple_space.hpp:14-71) ---------------------
struct Radix {
  std::vector<int> radix;
  std::vector<std::uint64_t> weight;
  std::uint64_t count = 0;
  void init(std::vector<int> r);
  void decode(std::uint64_t index, int* out) const;
  std::uint64_t encode(const int* tuple) const;  // throws PVI_ERR_INDEXING
};

// ---- device view of a model: POD passed by value to every kernel ---------
constexpr int kMaxDigits = 16;

struct DevModel {
  int scenario;
  int n_digits;
  std::uint64_t n_states;
  std::uint32_t n_actions;
  std::uint64_t weight[kMaxDigits];
  int radix[kMaxDigits];

  // A
  int a_m, a_lead, a_lifo, a_max_order, a_dmax;
  double a_cv, a_ch, a_cs, a_cw;
  const double* a_pmf;  // D_max+1
  const double* a_cdf;
  const std::int32_t* a_guide;  // guide table of a_cdf (kGuide + 1)

  // B
  int b_m, b_na, b_nb, b_cap_a, b_cap_b, b_dn;  // b_dn = d_max+1 (pz row length)
  int b_len_a, b_len_b;
  double b_cva, b_cvb, b_cra, b_crb, b_rho, b_mu_a, b_mu_b;
  const double* b_pmf_a;
  const double* b_pmf_b;
  const double* b_sf_a;
  const double* b_sf_b;
  const double* b_pz;
  const double* b_pz_cum;
  const double* b_cdf_a;
  const double* b_cdf_b;
  // rollout sampling tables (sim_tables.cpp): guide tables of the two demand
  // cdfs, and the substitution binomial's cumulative masses for every trial
  // count 0..b_binom_t at p = rho (null when rho is 0 or 1)
  const std::int32_t* b_guide_a;
  const std::int32_t* b_guide_b;
  const double* b_binom_cum;
  const std::int32_t* b_binom_guide;  // per trial count t, kBinGuide + 1 start indices into row t
  int b_binom_t;
  const std::uint16_t* b_lane_order;  // low-digit combos sorted by stock (tile order)
  int b_tile;                          // states per tile (product of the two low radices)

  // C
  int c_m, c_max_order, c_dmax;
  std::uint32_t c_n_comp;
  double c_cf, c_ch, c_cs, c_cw;
  const double* c_pmf;        // 7 x (D+1)
  const double* c_pd;         // 7: PD(tau) = sum_d pmf[tau][d], summed in d order
  const double* c_cdf;        // 7 x (D+1)
  const std::int32_t* c_guide;  // 7 x (kGuide + 1) guide tables of c_cdf
  const double* c_rcpt_cum;     // receipt binomials' cumulative masses (sim_tables.cpp)
  const std::int32_t* c_rcpt_off;  // (A_max + 1) x (m - 1) offsets into c_rcpt_cum, -1: none
  const std::int32_t* c_rcpt_guide;  // binomial guide rows of those tables (kBinGuide + 1 per trial count)
  const std::int32_t* c_rcpt_goff;   // (A_max + 1) x (m - 1) offsets into c_rcpt_guide, -1: none
  const std::int8_t* c_comp;  // n_comp x m, freshest first
  const std::uint32_t* c_ids;     // concatenated per action
  const double* c_probs;          // aligned with c_ids
  const std::uint32_t* c_offsets; // A_max+2
  const double* c_receipt;        // (A_max+1) x m
  // The multinomial over age categories factors into m-1 sequential
  // binomials: c_binom[a][k-1][b][y] = Bin(y; b, q_k(a)), shape
  // (A_max+1) x (m-1) x (A_max+1) x (A_max+1).  c_exogenous: the receipt law
  // does not depend on a (all c_receipt rows equal).
  int c_exogenous;
  const double* c_binom;
  // endogenous law, A_max = 20: the DMMA A fragments of every pass's
  // lower-triangular matrix, c_frag[a][k-1][576] (k_c_bin_wide_mma,
  // k_c_bin_diag_q), built once on the host instead of per CTA
  const double* c_frag;
  // A_max = D_max = 20: k_c_fact_g_mma's per-model tables -- the demand
  // band's DMMA fragments per weekday [7][3 * 7 * 32], the shortage /
  // holding reward RA[total - d + D] (m D + D + 1) and C_w w (D + 1)
  const double* c_gband;
  const double* c_ra;
  const double* c_cwt;

  // tabular
  std::uint64_t t_outcomes;
  const std::uint64_t* t_next;
  const double* t_reward;
  const double* t_prob;
};

// sampling tables of the rollout kernel (sim_tables.cpp)
constexpr int kGuide = 1024;  // cdf guide buckets (sim_tables.cpp cdf_guide)
std::vector<std::int32_t> cdf_guide(const double* cdf, int size, int G);
std::vector<double> binomial_cum_table(int T, double p);
constexpr int kBinGuide = 256;  // binomial guide buckets (sim_tables.cpp binomial_guide_table)
std::vector<std::int32_t> binomial_guide_table(const std::vector<double>& cum, int T, int G);
void c_receipt_tables(const double* receipt, int max_order, int m, std::vector<double>& cum,
                      std::vector<std::int32_t>& offsets);

struct DeviceCopy {
  DevModel dm{};
  std::vector<void*> allocations;
  // Scenario B factored sweep: per-state expected revenue and total issued
  // probability (V-independent, built once), and the A / B digit-block
  // orders sorted by stock so warps share loop trip counts.
  double* b_erpt = nullptr;
  // Scenario A factored sweep: per-state expected one-step reward (without
  // the order cost) and the demand law's cdf / survival tables
  double* a_reward = nullptr;
  double* a_cdf_sf = nullptr;  // [cdf(0..D) | sf(0..D+1)]
  double a_pd = 0.0;           // sum of the demand pmf
  std::uint16_t* b_order_a = nullptr;
  std::uint16_t* b_order_b = nullptr;
  // every state's issued-pair law sums to 1 (|PT - 1| <= 1e-12), so the
  // paired-diagonal kernel may fold the order costs into its running sums
  bool b_pt_unit = false;
  std::uint16_t* b_group_order = nullptr;    // A-side x_2..x_M digit groups by stock
  std::uint16_t* b_group_order_b = nullptr;  // B-side x_2..x_M digit groups by stock
  // Stage-1 work lists of shard sweeps (k_b_fact_w16p): (row, group range,
  // flags) items balanced over the persistent CTAs, keyed by the launch's
  // row filter and column ranges; built once per key.
  std::map<std::vector<int>, std::pair<void*, int>> b_s1_items;
  // Per-device workspace reused by the host-buffer entry points
  // (engine.cu Workspace: device copies of V / outputs, scratch, a stream).
  void* workspace = nullptr;
};

struct Model {
  int scenario = PVI_SCENARIO_A;
  pvi_scenario_a_params pa{};
  pvi_scenario_b_params pb{};
  pvi_scenario_c_params pc{};
  Radix space;
  std::uint32_t n_actions = 0;
  std::uint64_t n_outcomes = 0;
  double gamma = 0.0;
  int default_test = PVI_TEST_VALUE_SPAN;
  int periodicity = 1;

  // A
  std::vector<double> a_pmf, a_cdf;
  // B
  int b_na = 0, b_nb = 0, b_cap_a = 0, b_cap_b = 0, b_dmax = 0, b_ymax = 0;
  std::vector<double> b_pmf_a, b_pmf_b, b_sf_a, b_sf_b, b_cdf_a, b_cdf_b, b_pu, b_pz, b_pz_cum;
  std::vector<std::uint16_t> b_lane_order;
  // C
  std::uint32_t c_n_comp = 0;
  std::vector<double> c_pmf, c_cdf;  // 7 x (D+1)
  std::vector<std::int8_t> c_comp, c_comp_sum;
  std::vector<std::uint32_t> c_ids, c_offsets;
  std::vector<double> c_probs, c_receipt;
  bool c_exogenous = false;
  std::vector<double> c_binom;
  // tabular
  std::vector<std::uint64_t> t_next;
  std::vector<double> t_reward, t_prob, t_initial;

  std::string fingerprint;  // fingerprint_material()
  int algorithm = PVI_ALGO_EXACT;  // engine option, not part of the model's identity

  mutable std::mutex dev_mutex;
  mutable std::map<int, std::unique_ptr<DeviceCopy>> dev;
  mutable std::once_flag b_law_once;
  mutable bool b_law_unit_v = false;

  ~Model();
  const DevModel& device_view(int device) const;  // uploads on first use
  DeviceCopy& device_copy(int device) const;      // device_view's backing record
  double terms_per_sweep() const;
  double factored_fmas() const;  // FP64 FMAs per sweep of the factored kernels
  double state_cost(std::uint64_t s) const;  // relative backup cost of one state
  std::uint64_t tile_states() const;         // partition alignment
  std::uint64_t chunk_align() const;         // 0: sweeps do not chunk (whole-space tables)
  // B: every (I_a, I_b)'s issued-pair law sums to 1 within 1e-12 (host check, cached)
  bool b_law_unit() const;
};

std::unique_ptr<Model> build_scenario_a(const pvi_scenario_a_params& p);
std::unique_ptr<Model> build_scenario_b(const pvi_scenario_b_params& p);
std::unique_ptr<Model> build_scenario_c(const pvi_scenario_c_params& p);
std::unique_ptr<Model> build_tabular(std::uint64_t ns, std::uint32_t na, std::uint64_t no,
                                     double gamma, const std::uint64_t* next, const double* reward,
                                     const double* prob, const double* initial);
std::unique_ptr<Model> build_preset(const std::string& name, std::uint64_t* fixed_iterations,
                                    std::uint64_t* checkpoint_every);

// Host transition / probability (naive-oracle cross checks, model.hpp:30-46).
void host_transition(const Model& m, std::uint64_t s, std::uint32_t a, std::uint64_t w,
                     std::uint64_t* next, double* reward);
double host_outcome_probability(const Model& m, std::uint64_t s, std::uint32_t a, std::uint64_t w);

void sha256(const void* data, std::size_t len, std::uint8_t out[32]);

}  // namespace pvi_b200
