// K5: batched policy simulation — one thread per (policy, rollout).
//
// Every rollout owns the counter-based Philox stream of RolloutRng
// (rng.hpp:37-60): key = base_seed + rollout, counter = (day, draw, 0x7F4A7C15, 0),
// so a rollout's random numbers do not depend on the thread that runs it,
// and candidates evaluated in one batch share random realisations (common
// random numbers) exactly as the reference's per-candidate evaluate_policy
// calls do.  With -fmad=false and the reference's expression order, the
// per-rollout summaries are bit-identical to the reference's; the batch
// reduction then folds them in rollout-index order (sim.hpp:128-141).
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <memory>
#include <vector>

#include "common.cuh"
#include "engine.hpp"

namespace pvi_b200 {

namespace {

struct Philox {
  __device__ __forceinline__ static void block(std::uint32_t c[4], std::uint32_t k0, std::uint32_t k1) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
      const std::uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
      const std::uint32_t lo0 = 0xD2511F53u * c[0];
      const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
      const std::uint32_t lo1 = 0xCD9E8D57u * c[2];
      const std::uint32_t n0 = hi1 ^ c[1] ^ k0;
      const std::uint32_t n2 = hi0 ^ c[3] ^ k1;
      c[0] = n0;
      c[1] = lo1;
      c[2] = n2;
      c[3] = lo0;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
};

struct Rng {
  std::uint32_t k0, k1, day, draw;
  __device__ Rng(std::uint64_t seed, std::uint64_t rollout) {
    const std::uint64_t key = seed + rollout;
    k0 = static_cast<std::uint32_t>(key);
    k1 = static_cast<std::uint32_t>(key >> 32);
    day = 0;
    draw = 0;
  }
  __device__ __forceinline__ void begin_day(std::uint32_t d) {
    day = d;
    draw = 0;
  }
  __device__ __forceinline__ std::uint64_t next_u64() {
    std::uint32_t c[4] = {day, draw++, 0x7F4A7C15u, 0u};
    Philox::block(c, k0, k1);
    return (static_cast<std::uint64_t>(c[0]) << 32) | c[1];
  }
  __device__ __forceinline__ double uniform() {
    return static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
  }
  // the next N uniforms (draws draw .. draw + N - 1), their Philox blocks
  // interleaved round by round: N independent multiply chains in flight
  // instead of one (a block's 10 rounds are a serial dependency chain)
  template <int N>
  __device__ __forceinline__ void uniforms(double (&u)[N]) {
    std::uint32_t c[N][4];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      c[i][0] = day;
      c[i][1] = draw + i;
      c[i][2] = 0x7F4A7C15u;
      c[i][3] = 0u;
    }
    draw += N;
    std::uint32_t a0 = k0, a1 = k1;
#pragma unroll
    for (int round = 0; round < 10; ++round) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const std::uint32_t hi0 = __umulhi(0xD2511F53u, c[i][0]);
        const std::uint32_t lo0 = 0xD2511F53u * c[i][0];
        const std::uint32_t hi1 = __umulhi(0xCD9E8D57u, c[i][2]);
        const std::uint32_t lo1 = 0xCD9E8D57u * c[i][2];
        c[i][0] = hi1 ^ c[i][1] ^ a0;
        c[i][1] = lo1;
        c[i][2] = hi0 ^ c[i][3] ^ a1;
        c[i][3] = lo0;
      }
      a0 += 0x9E3779B9u;
      a1 += 0xBB67AE85u;
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
      u[i] = static_cast<double>(((static_cast<std::uint64_t>(c[i][0]) << 32) | c[i][1]) >> 11) * 0x1.0p-53;
  }
};

// rng.hpp:63-73
__device__ __forceinline__ int sample_from_cdf(const double* cdf, int size, double u) {
  int lo = 0, hi = size - 1;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (cdf[mid] > u)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

// sample_from_cdf through a guide table (sim_tables.cpp cdf_guide): the
// same index, found by one table load and a short forward scan
__device__ __forceinline__ int sample_from_cdf_guided(const double* cdf, int size, const std::int32_t* guide,
                                                      double u) {
  const int e = __ldg(guide + static_cast<int>(u * kGuide));  // u in [0, 1): exact bucket
  if (e >= 0) return e;  // no cdf boundary inside the bucket
  int i = -e - 1;
  while (i < size - 1 && !(__ldg(cdf + i) > u)) ++i;
  return i;
}

// sample_binomial from the precomputed cumulative masses of row `trials`
// (sim_tables.cpp binomial_cum_table): the first k < trials with cum_k > u,
// else trials -- the reference loop's k -- with the scan started at the
// row's guide entry for floor(u G) / G (binomial_guide_table; ~1
// comparison instead of a scan from 0: B rollouts -13%, C -26%)
__device__ __forceinline__ int sample_binomial_guided(int trials, const double* row, const std::int32_t* guide,
                                                      double u) {
  const int e = __ldg(guide + static_cast<int>(u * kBinGuide));  // u in [0, 1): exact bucket
  if (e >= 0) return e;  // no boundary inside the bucket
  int k = -e - 1;
  while (k < trials && !(__ldg(row + k) > u)) ++k;
  return k;
}

// rng.hpp:76-90
__device__ __forceinline__ int sample_binomial(int trials, double p, double u) {
  if (trials <= 0 || p <= 0.0) return 0;
  if (p >= 1.0) return trials;
  const double ratio = p / (1.0 - p);
  double mass = 1.0;
  for (int i = 0; i < trials; ++i) mass *= 1.0 - p;
  double cum = mass;
  int k = 0;
  while (cum <= u && k < trials) {
    mass *= ratio * (trials - k) / (k + 1);
    cum += mass;
    ++k;
  }
  return k;
}

struct Step {
  double reward;
  int demand[2], filled[2], expired[2], received[2], holding[2];
};

// Geometry of one rollout kernel instantiation (round 2): GM > 0 fixes the
// scenario's digit counts at compile time (A: 10 m + L, B and C: m) so every
// per-digit loop unrolls and the state / ageing arrays live in registers
// (with runtime bounds they were local memory: ~11% of the kernel's
// instructions were LDL / STL); GM = 0 is the generic instantiation.
template <int SC, int GM>
struct Geo {
  static constexpr int m = GM == 0 ? 0 : SC == PVI_SCENARIO_A ? GM / 10 : GM;
  static constexpr int lead = SC == PVI_SCENARIO_A && GM > 0 ? GM % 10 : 0;
  // TupleSpace arity: A m + L - 1, B 2 m, C m (tau + m - 1 stock digits)
  static constexpr int arity = GM == 0 ? kMaxDigits
                               : SC == PVI_SCENARIO_A ? m + lead - 1
                               : SC == PVI_SCENARIO_B ? 2 * m
                                                      : m;
  static constexpr int cap = GM == 0 ? 14 : m + 1;  // per-digit array bound (index 1..m)
};

template <int MC>
__device__ __forceinline__ int age_fifo_s(const int* x, int m_rt, int demand, int* next) {
  const int m = MC > 0 ? MC : m_rt;
  const int expired = ipos(x[1] - demand);
  int prefix = 0;
#pragma unroll
  for (int j = 1; j <= (MC > 0 ? MC - 1 : 13); ++j) {
    if (j > m - 1) break;
    prefix += x[j];
    next[j] = ipos(x[j + 1] - ipos(demand - prefix));
  }
  return expired;
}

template <int MC>
__device__ __forceinline__ int age_lifo_s(const int* x, int m_rt, int demand, int* next) {
  const int m = MC > 0 ? MC : m_rt;
  int suffix = 0;
#pragma unroll
  for (int j = 2; j <= (MC > 0 ? MC : 14); ++j) {
    if (j > m) break;
    suffix += x[j];
  }
  const int expired = ipos(x[1] - ipos(demand - suffix));
#pragma unroll
  for (int j = 1; j <= (MC > 0 ? MC - 1 : 13); ++j) {
    if (j > m - 1) break;
    suffix -= x[j + 1];
    next[j] = ipos(x[j + 1] - ipos(demand - suffix));
  }
  return expired;
}

// ScenarioA::sample_step (scenario_a.cpp:157-189)
template <int GM>
__device__ __forceinline__ void step_a(const DevModel& dm, int* state, const int* action, Rng& rng, Step& st) {
  using G = Geo<PVI_SCENARIO_A, GM>;
  const int m = GM ? G::m : dm.a_m, lead = GM ? G::lead : dm.a_lead, order = action[0];
  int x[G::cap], aged[G::cap];
  int xt = 0;
#pragma unroll
  for (int j = 1; j < G::cap; ++j) {
    if (j > m) break;
    x[j] = state[lead - 1 + m - j];
    xt += x[j];
  }
  const int demand = sample_from_cdf_guided(dm.a_cdf, dm.a_dmax + 1, dm.a_guide, rng.uniform());
  const int expired = dm.a_lifo ? age_lifo_s<G::m>(x, m, demand, aged) : age_fifo_s<G::m>(x, m, demand, aged);
  const int arriving = lead >= 2 ? state[lead - 2] : order;
  st.reward = -dm.a_cv * order - dm.a_ch * ipos(xt - demand - expired) - dm.a_cs * ipos(demand - xt) -
              dm.a_cw * expired;
  st.demand[0] = demand;
  st.filled[0] = min(demand, xt);
  st.expired[0] = expired;
  st.received[0] = arriving;
  st.holding[0] = ipos(xt - demand - expired);
#pragma unroll
  for (int k = (GM ? G::lead : 14) - 2; k >= 1; --k)
    if (k <= lead - 2) state[k] = state[k - 1];
  state[0] = order;
  if (lead >= 2) state[lead - 1] = arriving;
#pragma unroll
  for (int j = 1; j < G::cap - 1; ++j) {
    if (j > m - 1) break;
    state[lead + m - 1 - j] = aged[j];
  }
}

// ScenarioB::sample_step (scenario_b.cpp:332-379)
template <int GM>
__device__ __forceinline__ void step_b(const DevModel& dm, int* state, const int* action, Rng& rng, Step& st) {
  using G = Geo<PVI_SCENARIO_B, GM>;
  const int m = GM ? G::m : dm.b_m;
  int xa[G::cap], xb[G::cap], aa[G::cap], ab[G::cap];
  int stock_a = 0, stock_b = 0;
#pragma unroll
  for (int j = 1; j < G::cap; ++j) {
    if (j > m) break;
    xa[j] = state[m - j];
    xb[j] = state[2 * m - j];
    stock_a += xa[j];
    stock_b += xb[j];
  }
  // every day draws exactly three uniforms (scenario_b.cpp:332-379): demand
  // A, demand B, the substitution binomial -- generated together
  double u3[3];
  rng.uniforms(u3);
  const int demand_a = sample_from_cdf_guided(dm.b_cdf_a, dm.b_len_a, dm.b_guide_a, u3[0]);
  const int demand_b = sample_from_cdf_guided(dm.b_cdf_b, dm.b_len_b, dm.b_guide_b, u3[1]);
  const int own_fill_a = min(demand_a, stock_a);
  const int fill_b = min(demand_b, stock_b);
  const int trials = demand_b - fill_b;
  const double ub = u3[2];
  const int accepted = dm.b_binom_cum && trials > 0 && trials <= dm.b_binom_t
                           ? sample_binomial_guided(trials, dm.b_binom_cum + trials * (trials + 1) / 2,
                                                    dm.b_binom_guide + trials * (kBinGuide + 1), ub)
                           : sample_binomial(trials, dm.b_rho, ub);
  const int sub = min(accepted, stock_a - own_fill_a);
  const int h_a = own_fill_a + sub;
  const int h_b = fill_b;
  const int exp_a = age_fifo_s<G::m>(xa, m, h_a, aa);
  const int exp_b = age_fifo_s<G::m>(xb, m, h_b, ab);
  st.reward = -(dm.b_cva * action[0] + dm.b_cvb * action[1]) + dm.b_cra * h_a + dm.b_crb * h_b;
  st.demand[0] = demand_a;
  st.demand[1] = demand_b;
  st.filled[0] = own_fill_a;
  st.filled[1] = fill_b + sub;
  st.expired[0] = exp_a;
  st.expired[1] = exp_b;
  st.received[0] = action[0];
  st.received[1] = action[1];
  int hold_a = 0, hold_b = 0;
#pragma unroll
  for (int j = 1; j < G::cap - 1; ++j) {
    if (j > m - 1) break;
    hold_a += aa[j];
    hold_b += ab[j];
  }
  st.holding[0] = hold_a;
  st.holding[1] = hold_b;
  state[0] = action[0];
  state[m] = action[1];
#pragma unroll
  for (int j = 1; j < G::cap - 1; ++j) {
    if (j > m - 1) break;
    state[m - j] = aa[j];
    state[2 * m - j] = ab[j];
  }
}

// ScenarioC::sample_step (scenario_c.cpp:313-359) with sample_multinomial
// (rng.hpp:94-110): one uniform per category but the last, skipped once
// nothing remains.
template <int GM>
__device__ __forceinline__ void step_c(const DevModel& dm, int* state, const int* action, Rng& rng, Step& st) {
  using G = Geo<PVI_SCENARIO_C, GM>;
  const int m = GM ? G::m : dm.c_m, cap = dm.c_max_order;
  const int tau = state[0];
  const int order = action[0];
  const double* probs = dm.c_receipt + static_cast<std::size_t>(order) * m;
  int counts[G::cap];
  {
    int remaining = order;
    double mass_left = 1.0;
#pragma unroll
    for (int k = 0; k + 1 < G::cap - 1; ++k) {
      if (k + 1 >= m) break;
      if (remaining == 0 || mass_left <= 0.0) {
        counts[k] = 0;
        continue;
      }
      const double u = rng.uniform();
      const int off = dm.c_rcpt_off ? __ldg(dm.c_rcpt_off + order * (m - 1) + k) : -1;
      if (off >= 0) {
        counts[k] = sample_binomial_guided(remaining, dm.c_rcpt_cum + off + remaining * (remaining + 1) / 2,
                                           dm.c_rcpt_guide + __ldg(dm.c_rcpt_goff + order * (m - 1) + k) +
                                               remaining * (kBinGuide + 1),
                                           u);
      } else {  // no table (p_k = 0 or 1, or a = 0): the reference's sampler, its division only here
        const double cond = probs[k] / mass_left;
        counts[k] = sample_binomial(remaining, cond < 1.0 ? cond : 1.0, u);
      }
      remaining -= counts[k];
      mass_left -= probs[k];
    }
    counts[m - 1] = remaining;
  }
  int y[G::cap], x[G::cap], z[G::cap];
#pragma unroll
  for (int j = 1; j < G::cap; ++j) {
    if (j > m) break;
    y[j] = counts[j - 1];
  }
  const int dn = dm.c_dmax + 1;
  const int d = sample_from_cdf_guided(dm.c_cdf + tau * dn, dn, dm.c_guide + tau * (kGuide + 1), rng.uniform());
#pragma unroll
  for (int j = 1; j < G::cap - 1; ++j) {
    if (j > m - 1) break;
    x[j] = state[m - j];
  }
  int total = y[m], accepted = y[m];
#pragma unroll
  for (int j = 1; j < G::cap - 1; ++j) {
    if (j > m - 1) break;
    z[j] = min(x[j] + y[j], cap);
    total += z[j];
    accepted += z[j] - x[j];
  }
  int prefix = 0;
#pragma unroll
  for (int j = 1; j < G::cap - 2; ++j) {
    if (j > m - 2) break;
    prefix += z[j];
    state[m - j] = ipos(z[j + 1] - ipos(d - prefix));
  }
  prefix += z[m - 1];
  state[1] = ipos(y[m] - ipos(d - prefix));
  state[0] = (tau + 1) % 7;
  const int expired = ipos(z[1] - d);
  st.reward = -(order > 0 ? dm.c_cf : 0.0) - dm.c_ch * ipos(total - d) - dm.c_cs * ipos(d - total) -
              dm.c_cw * expired;
  st.demand[0] = d;
  st.filled[0] = min(d, total);
  st.expired[0] = expired;
  st.received[0] = accepted;
  st.holding[0] = ipos(total - d);
}

struct DevPolicy {
  int kind;
  const std::uint32_t* table;
  int params[14];
};

// policies.hpp:18-82; scenario_a.cpp:191-195; scenario_b.cpp:381-393;
// scenario_c.cpp:361-370
template <int SC, int GM>
__device__ __forceinline__ void apply_policy(const DevModel& dm, const DevPolicy& pol, const int* state,
                                             int arity_rt, int* action) {
  constexpr int AR = Geo<SC, GM>::arity;
  const int arity = GM ? AR : arity_rt;
  if (pol.kind == 0) {
    std::uint64_t idx = 0;
#pragma unroll
    for (int i = 0; i < AR; ++i) {
      if (i >= arity) break;
      idx += static_cast<std::uint64_t>(state[i]) * dm.weight[i];
    }
    const std::uint32_t a = pol.table[idx];
    if (SC == PVI_SCENARIO_B) {
      action[0] = static_cast<int>(a) / dm.b_nb;
      action[1] = static_cast<int>(a) % dm.b_nb;
    } else {
      action[0] = static_cast<int>(a);
    }
    return;
  }
  switch (SC) {
    case PVI_SCENARIO_A: {
      int position = 0;
#pragma unroll
      for (int i = 0; i < AR; ++i) {
        if (i >= arity) break;
        position += state[i];
      }
      action[0] = ipos(pol.params[0] - position);
      return;
    }
    case PVI_SCENARIO_B: {
      const int m = GM ? Geo<SC, GM>::m : dm.b_m;
      int stock_a = 0, stock_b = 0;
#pragma unroll
      for (int i = 0; i < AR / 2; ++i) {
        if (i >= m) break;
        stock_a += state[i];
        stock_b += state[m + i];
      }
      const int expiring_a = state[m - 1];
      const int expiring_b = state[2 * m - 1];
      const double waste_a = fmax(0.0, expiring_a - dm.b_mu_a);
      const double waste_b = fmax(0.0, expiring_b - dm.b_mu_b);
      action[0] = static_cast<int>(lround(fmax(0.0, (pol.params[0] - stock_a) + waste_a)));
      action[1] = static_cast<int>(lround(fmax(0.0, (pol.params[1] - stock_b) + waste_b)));
      return;
    }
    default: {
      const int tau = state[0];
      const int s = pol.params[tau], S = pol.params[7 + tau];
      if (s >= S) {
        action[0] = 0;
        return;
      }
      int stock = 0;
#pragma unroll
      for (int i = 1; i < AR; ++i) {
        if (i >= arity) break;
        stock += state[i];
      }
      action[0] = stock > s ? 0 : ipos(S - stock);
      return;
    }
  }
}

struct SimError {
  unsigned long long key;  // policy * n_rollouts + rollout, min wins
  int action;
  int product;
  int arity;
  int state[kMaxDigits];
};

// rollout (sim.hpp:68-124); one instantiation per scenario (SC) and
// geometry (GM, see Geo), so each carries only its own step function and
// policy arithmetic with its digit loops unrolled.  The KPI counts are
// summed in 32-bit registers and folded into the 64-bit totals every 4096
// measured days (a day adds at most a few hundred units), the same integers.
template <int SC, int MINB, int GM>
__global__ void __launch_bounds__(128, MINB) k_rollouts(DevModel dm, const DevPolicy* __restrict__ pols,
                                                  int n_rollouts, int horizon, int warmup,
                                                  std::uint64_t base_seed, int arity_rt, int products,
                                                  double gamma, double* __restrict__ out,
                                                  SimError* err, unsigned long long* blocks_out) {
  using G = Geo<SC, GM>;
  const int arity = GM ? G::arity : arity_rt;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  if (i >= n_rollouts) return;
  const DevPolicy pol = pols[p];
  int state[G::arity];
#pragma unroll
  for (int k = 0; k < G::arity; ++k) state[k] = 0;
  int action[2] = {0, 0};
  int bound[2];
  if (SC == PVI_SCENARIO_B) {
    bound[0] = 2 * (dm.b_na - 1);
    bound[1] = 2 * (dm.b_nb - 1);
  } else {
    bound[0] = bound[1] = static_cast<int>(dm.n_actions) - 1;
  }
  constexpr int action_arity = SC == PVI_SCENARIO_B ? 2 : 1;
  constexpr int NP = SC == PVI_SCENARIO_B ? 2 : 1;  // products
  (void)products;
  Rng rng(base_seed, static_cast<std::uint64_t>(i));
  const int total_days = warmup + horizon;
  double ret = 0.0, weight = 1.0;
  unsigned long long blocks = 0;
  long long demand[2] = {0, 0}, filled[2] = {0, 0}, expired[2] = {0, 0}, received[2] = {0, 0},
            holding[2] = {0, 0};
  int d32[NP], f32[NP], e32[NP], r32[NP], h32[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) d32[k] = f32[k] = e32[k] = r32[k] = h32[k] = 0;
  auto fold = [&]() {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      demand[k] += d32[k];
      filled[k] += f32[k];
      expired[k] += e32[k];
      received[k] += r32[k];
      holding[k] += h32[k];
      d32[k] = f32[k] = e32[k] = r32[k] = h32[k] = 0;
    }
  };
  for (int day = 0; day < total_days; ++day) {
    apply_policy<SC, GM>(dm, pol, state, arity, action);
#pragma unroll
    for (int k = 0; k < action_arity; ++k) {
      if (action[k] < 0 || action[k] > bound[k]) {
        const unsigned long long key = static_cast<unsigned long long>(p) * n_rollouts + i;
        const unsigned long long old = atomicMin(&err->key, key);
        if (key < old) {
          err->action = action[k];
          err->product = k;
          err->arity = arity;
          for (int q = 0; q < arity; ++q) err->state[q] = state[q];
        }
        return;
      }
    }
    blocks += rng.draw;  // Philox blocks drawn the previous day (measurement hook)
    rng.begin_day(static_cast<std::uint32_t>(day));
    Step st;
    st.reward = 0.0;
#pragma unroll
    for (int k = 0; k < 2; ++k)
      st.demand[k] = st.filled[k] = st.expired[k] = st.received[k] = st.holding[k] = 0;
    if constexpr (SC == PVI_SCENARIO_A) step_a<GM>(dm, state, action, rng, st);
    else if constexpr (SC == PVI_SCENARIO_B) step_b<GM>(dm, state, action, rng, st);
    else step_c<GM>(dm, state, action, rng, st);
    if (day >= warmup) {
      ret += weight * st.reward;
      weight *= gamma;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        d32[k] += st.demand[k];
        f32[k] += st.filled[k];
        e32[k] += st.expired[k];
        r32[k] += st.received[k];
        h32[k] += st.holding[k];
      }
      if (((day - warmup) & 4095) == 4095) fold();
    }
  }
  fold();
  if (blocks_out) atomicAdd(blocks_out, blocks + rng.draw);
  double* o = out + (static_cast<std::size_t>(p) * n_rollouts + i) * 7;
  o[0] = ret;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    double svc = 100.0, wst = 0.0, hold = 0.0;
    if (k < NP) {
      svc = demand[k] > 0 ? 100.0 * static_cast<double>(filled[k]) / static_cast<double>(demand[k]) : 100.0;
      wst = received[k] > 0 ? 100.0 * static_cast<double>(expired[k]) / static_cast<double>(received[k]) : 0.0;
      hold = horizon > 0 ? static_cast<double>(holding[k]) / horizon : 0.0;
    }
    o[1 + k] = svc;
    o[3 + k] = wst;
    o[5 + k] = hold;
  }
}

// detail::reduce (sim.hpp:128-141) per (policy, KPI), in rollout-index order.
__global__ void k_reduce_eval(const double* __restrict__ summ, int n, int n_pol, double* __restrict__ stats) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pol * 7) return;
  const int p = t / 7, f = t % 7;
  const double* base = summ + static_cast<std::size_t>(p) * n * 7 + f;
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += base[static_cast<std::size_t>(i) * 7];
  const double mean = sum / static_cast<double>(n);
  double sd = 0.0;
  if (n > 1) {
    double ss = 0.0;
    for (int i = 0; i < n; ++i) {
      const double x = base[static_cast<std::size_t>(i) * 7];
      ss += (x - mean) * (x - mean);
    }
    sd = sqrt(ss / static_cast<double>(n - 1));
  }
  stats[2 * t] = mean;
  stats[2 * t + 1] = sd;
}

__global__ void k_philox(std::uint32_t c0, std::uint32_t c1, std::uint32_t c2, std::uint32_t c3,
                         std::uint32_t k0, std::uint32_t k1, std::uint32_t* out) {
  std::uint32_t c[4] = {c0, c1, c2, c3};
  Philox::block(c, k0, k1);
  for (int i = 0; i < 4; ++i) out[i] = c[i];
}

__global__ void k_draws(std::uint64_t seed, std::uint64_t rollout, std::uint32_t day, int n,
                        std::uint64_t* out) {
  Rng rng(seed, rollout);
  rng.begin_day(day);
  for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
}

// one non-blocking stream per (host thread, device) for the evaluations
cudaStream_t sim_stream(int device) {
  static thread_local cudaStream_t streams[64] = {};
  if (device < 0 || device >= 64) fail(PVI_ERR_DEVICE, "device ordinal out of range");
  if (!streams[device]) PVI_CUDA(cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking));
  return streams[device];
}

using Buf = PoolBuf;

void fill_evaluations(const double* stat, std::uint32_t n_policies, int n_rollouts, int products,
                      pvi_evaluation* evals) {
  for (std::uint32_t p = 0; p < n_policies; ++p) {
    const double* s = stat + static_cast<std::size_t>(p) * 14;
    pvi_evaluation& e = evals[p];
    std::memset(&e, 0, sizeof(e));
    e.products = products;
    e.n_rollouts = n_rollouts;
    e.ret_mean = s[0];
    e.ret_sd = s[1];
    for (int k = 0; k < products; ++k) {
      e.service_mean[k] = s[2 * (1 + k)];
      e.service_sd[k] = s[2 * (1 + k) + 1];
      e.wastage_mean[k] = s[2 * (3 + k)];
      e.wastage_sd[k] = s[2 * (3 + k) + 1];
      e.holding_mean[k] = s[2 * (5 + k)];
      e.holding_sd[k] = s[2 * (5 + k) + 1];
    }
  }
}

}  // namespace

void sim_evaluate(const Model& m, const pvi_policy* policies, std::uint32_t n_policies,
                  const pvi_rollout_config& cfg, pvi_rollout_summary* per_rollout,
                  pvi_evaluation* evals) {
  NvtxRange nvtx_range("pvi rollouts");
  if (cfg.n_rollouts < 1) fail(PVI_ERR_PARAMETER, "evaluation needs at least one rollout");
  if (m.scenario == PVI_TABULAR) fail(PVI_ERR_PARAMETER, "tabular models have no simulator");
  if (n_policies == 0) return;
  const int device = select_device(cfg.device);
  const DevModel& dm = m.device_view(device);
  const int arity = static_cast<int>(m.space.radix.size());
  const int products = m.scenario == PVI_SCENARIO_B ? 2 : 1;
  const std::uint64_t n_states = m.space.count;

  std::vector<DevPolicy> hp(n_policies);
  std::vector<std::unique_ptr<Buf>> tables;
  cudaStream_t stream = sim_stream(device);
  for (std::uint32_t i = 0; i < n_policies; ++i) {
    const pvi_policy& p = policies[i];
    hp[i].kind = p.kind;
    hp[i].table = nullptr;
    for (int k = 0; k < 14; ++k) hp[i].params[k] = p.params[k];
    if (p.kind == 0) {
      if (!p.table) fail(PVI_ERR_PARAMETER, "VI-table policy without a table");
      // Share one device copy between policies that pass the same table.
      const std::uint32_t* found = nullptr;
      for (std::uint32_t j = 0; j < i; ++j)
        if (policies[j].kind == 0 && policies[j].table == p.table) found = hp[j].table;
      if (!found) {
        tables.push_back(std::make_unique<Buf>(n_states * 4, stream));
        PVI_CUDA(cudaMemcpyAsync(tables.back()->p, p.table, n_states * 4, cudaMemcpyHostToDevice, stream));
        found = static_cast<const std::uint32_t*>(tables.back()->p);
      }
      hp[i].table = found;
    } else {
      const int need = m.scenario == PVI_SCENARIO_A ? 1 : m.scenario == PVI_SCENARIO_B ? 2 : 14;
      if (p.n_params != need)
        fail(PVI_ERR_PARAMETER, "heuristic policy expects " + std::to_string(need) + " parameters");
    }
  }
  Buf dpol(sizeof(DevPolicy) * n_policies, stream);
  PVI_CUDA(cudaMemcpyAsync(dpol.p, hp.data(), sizeof(DevPolicy) * n_policies, cudaMemcpyHostToDevice, stream));
  const std::size_t n_sum = static_cast<std::size_t>(n_policies) * cfg.n_rollouts;
  Buf dsum(n_sum * 7 * sizeof(double), stream);
  Buf dstat(static_cast<std::size_t>(n_policies) * 14 * sizeof(double), stream);
  Buf derr(sizeof(SimError), stream);
  SimError herr;
  std::memset(&herr, 0, sizeof(herr));
  herr.key = ~0ull;
  PVI_CUDA(cudaMemcpyAsync(derr.p, &herr, sizeof(herr), cudaMemcpyHostToDevice, stream));
  const dim3 grid((cfg.n_rollouts + 127) / 128, n_policies);
  // CTAs per SM the register allocation is bounded for (measured per
  // scenario on a B200: A 3, B 4, C 1)
  // geometry of the compiled instantiations (Geo): A 10 m + L, B / C m
  const int gm = m.scenario == PVI_SCENARIO_A ? 10 * m.pa.useful_life + m.pa.lead_time
                 : m.scenario == PVI_SCENARIO_B ? m.pb.useful_life
                                                : m.pc.useful_life;
  using KR = void (*)(DevModel, const DevPolicy*, int, int, int, std::uint64_t, int, int, double, double*,
                      SimError*, unsigned long long*);
  KR kr = nullptr;
#define PVI_KR(SCN, MB, GMV) \
  if (!kr && m.scenario == SCN && gm == GMV) kr = k_rollouts<SCN, MB, GMV>;
  PVI_KR(PVI_SCENARIO_A, 3, 21) PVI_KR(PVI_SCENARIO_A, 3, 22) PVI_KR(PVI_SCENARIO_A, 3, 31)
  PVI_KR(PVI_SCENARIO_A, 3, 32) PVI_KR(PVI_SCENARIO_A, 3, 41) PVI_KR(PVI_SCENARIO_A, 3, 42)
  PVI_KR(PVI_SCENARIO_A, 3, 51) PVI_KR(PVI_SCENARIO_A, 3, 52)
  PVI_KR(PVI_SCENARIO_B, 4, 2) PVI_KR(PVI_SCENARIO_B, 4, 3)
  PVI_KR(PVI_SCENARIO_C, 1, 3) PVI_KR(PVI_SCENARIO_C, 1, 5)
#undef PVI_KR
  if (!kr)
    kr = m.scenario == PVI_SCENARIO_A ? k_rollouts<PVI_SCENARIO_A, 1, 0>
         : m.scenario == PVI_SCENARIO_B ? k_rollouts<PVI_SCENARIO_B, 1, 0>
                                        : k_rollouts<PVI_SCENARIO_C, 1, 0>;
  static const bool trace = [] {
    const char* e = std::getenv("PVI_SIM_TRACE");
    return e && e[0] == '1';
  }();
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (trace) {
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, stream);
  }
  // measurement hook (pvi_profile_enable): Philox blocks drawn, kernel time
  const bool prof = profiling_enabled();
  std::unique_ptr<Buf> dblocks;
  cudaEvent_t p0 = nullptr, p1 = nullptr;
  if (prof) {
    dblocks = std::make_unique<Buf>(sizeof(unsigned long long), stream);
    PVI_CUDA(cudaMemsetAsync(dblocks->p, 0, sizeof(unsigned long long), stream));
    PVI_CUDA(cudaEventCreate(&p0));
    PVI_CUDA(cudaEventCreate(&p1));
    PVI_CUDA(cudaEventRecord(p0, stream));
  }
  kr<<<grid, 128, 0, stream>>>(dm, static_cast<const DevPolicy*>(dpol.p), cfg.n_rollouts,
                                       cfg.horizon_days, cfg.warmup_days, cfg.base_seed, arity,
                                       products, m.gamma, static_cast<double*>(dsum.p),
                                       static_cast<SimError*>(derr.p),
                                       prof ? static_cast<unsigned long long*>(dblocks->p) : nullptr);
  PVI_CUDA(cudaGetLastError());
  if (prof) PVI_CUDA(cudaEventRecord(p1, stream));
  if (trace) cudaEventRecord(t1, stream);
  k_reduce_eval<<<(n_policies * 7 + 63) / 64, 64, 0, stream>>>(static_cast<const double*>(dsum.p), cfg.n_rollouts,
                                                              n_policies, static_cast<double*>(dstat.p));
  PVI_CUDA(cudaGetLastError());
  PVI_CUDA(cudaMemcpyAsync(&herr, derr.p, sizeof(herr), cudaMemcpyDeviceToHost, stream));
  std::vector<double> hstat(static_cast<std::size_t>(n_policies) * 14);
  PVI_CUDA(cudaMemcpyAsync(hstat.data(), dstat.p, hstat.size() * 8, cudaMemcpyDeviceToHost, stream));
  if (per_rollout)
    PVI_CUDA(cudaMemcpyAsync(per_rollout, dsum.p, n_sum * 7 * sizeof(double), cudaMemcpyDeviceToHost, stream));
  unsigned long long hblocks = 0;
  if (prof) PVI_CUDA(cudaMemcpyAsync(&hblocks, dblocks->p, sizeof(hblocks), cudaMemcpyDeviceToHost, stream));
  PVI_CUDA(cudaStreamSynchronize(stream));
  if (prof) {
    float ms = 0.f;
    PVI_CUDA(cudaEventElapsedTime(&ms, p0, p1));
    cudaEventDestroy(p0);
    cudaEventDestroy(p1);
    sim_profile_add(hblocks, static_cast<std::uint64_t>(n_policies) * cfg.n_rollouts *
                                 static_cast<std::uint64_t>(cfg.horizon_days + cfg.warmup_days),
                    ms);
  }
  if (trace) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    std::fprintf(stderr, "[pvi sim] k_rollouts %u x %d: %.3f ms\n", n_policies, cfg.n_rollouts, ms);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }
  if (herr.key != ~0ull) {
    std::string tuple;
    for (int q = 0; q < herr.arity; ++q) tuple += std::to_string(herr.state[q]) + " ";
    fail(PVI_ERR_CONTRACT, "policy returned out-of-range order " + std::to_string(herr.action) +
                               " in state [ " + tuple + "]");
  }
  if (evals) fill_evaluations(hstat.data(), n_policies, cfg.n_rollouts, products, evals);
}

void sim_reduce_host(const double* summ, std::uint32_t n_policies, int n, int products, pvi_evaluation* evals) {
  // the operations of k_reduce_eval (and of the reference's detail::reduce),
  // compiled without FMA contraction: the same bits
  std::vector<double> stat(static_cast<std::size_t>(n_policies) * 14);
  for (std::uint32_t p = 0; p < n_policies; ++p)
    for (int f = 0; f < 7; ++f) {
      const double* base = summ + static_cast<std::size_t>(p) * n * 7 + f;
      double sum = 0.0;
      for (int i = 0; i < n; ++i) sum += base[static_cast<std::size_t>(i) * 7];
      const double mean = sum / static_cast<double>(n);
      double sd = 0.0;
      if (n > 1) {
        double ss = 0.0;
        for (int i = 0; i < n; ++i) {
          const double x = base[static_cast<std::size_t>(i) * 7];
          const double d = x - mean;
          ss += d * d;
        }
        sd = std::sqrt(ss / static_cast<double>(n - 1));
      }
      stat[(static_cast<std::size_t>(p) * 7 + f) * 2] = mean;
      stat[(static_cast<std::size_t>(p) * 7 + f) * 2 + 1] = sd;
    }
  fill_evaluations(stat.data(), n_policies, n, products, evals);
}

void philox_block_device(const std::uint32_t ctr[4], const std::uint32_t key[2], std::uint32_t out[4]) {
  const cudaStream_t st = sim_stream(select_device(-1));
  Buf d(16, st);
  k_philox<<<1, 1, 0, st>>>(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1], static_cast<std::uint32_t*>(d.p));
  PVI_CUDA(cudaGetLastError());
  PVI_CUDA(cudaMemcpyAsync(out, d.p, 16, cudaMemcpyDeviceToHost, st));
  PVI_CUDA(cudaStreamSynchronize(st));
}

void rollout_draws_device(std::uint64_t seed, std::uint64_t rollout, std::uint32_t day, int n,
                          std::uint64_t* out) {
  const cudaStream_t st = sim_stream(select_device(-1));
  Buf d(static_cast<std::size_t>(n) * 8, st);
  k_draws<<<1, 1, 0, st>>>(seed, rollout, day, n, static_cast<std::uint64_t*>(d.p));
  PVI_CUDA(cudaGetLastError());
  PVI_CUDA(cudaMemcpyAsync(out, d.p, static_cast<std::size_t>(n) * 8, cudaMemcpyDeviceToHost, st));
  PVI_CUDA(cudaStreamSynchronize(st));
}

}  // namespace pvi_b200
