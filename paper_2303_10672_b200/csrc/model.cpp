// Host-side table construction for the three scenario families and the
// explicit-table MDP.  Formulas follow the reference constructors (cited
// per function); operation order is kept so the tables are bit-identical to
// the reference's, which is what lets the device sweep reproduce the
// reference's value vectors bit for bit.
#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <sstream>

#include "gamma_p.h"

namespace pvi_b200 {

// ---------------------------------------------------------------------------
// Radix (tuple_space.hpp:18-54)

void Radix::init(std::vector<int> r) {
  radix = std::move(r);
  if (radix.empty()) fail(PVI_ERR_PARAMETER, "tuple space: no components");
  if (radix.size() > static_cast<std::size_t>(kMaxDigits))
    fail(PVI_ERR_PARAMETER, "tuple space: too many components for the device kernels");
  weight.assign(radix.size(), 1);
  count = 1;
  for (std::size_t i = radix.size(); i-- > 0;) {
    if (radix[i] < 1) fail(PVI_ERR_PARAMETER, "tuple space: radix must be >= 1");
    weight[i] = count;
    const auto rr = static_cast<std::uint64_t>(radix[i]);
    if (count > UINT64_MAX / rr) fail(PVI_ERR_PARAMETER, "tuple space: element count overflows 64 bits");
    count *= rr;
  }
}

void Radix::decode(std::uint64_t index, int* out) const {
  for (std::size_t i = 0; i < radix.size(); ++i) {
    out[i] = static_cast<int>(index / weight[i]);
    index %= weight[i];
  }
}

std::uint64_t Radix::encode(const int* tuple) const {
  std::uint64_t index = 0;
  for (std::size_t i = 0; i < radix.size(); ++i) {
    if (tuple[i] < 0 || tuple[i] >= radix[i])
      fail(PVI_ERR_INDEXING, "tuple component " + std::to_string(i) + " = " +
                                 std::to_string(tuple[i]) + " outside [0, " +
                                 std::to_string(radix[i] - 1) + "]");
    index += static_cast<std::uint64_t>(tuple[i]) * weight[i];
  }
  return index;
}

// ---------------------------------------------------------------------------
// Distribution kit (dist.cpp)

namespace {

std::vector<double> prefix_sum(const std::vector<double>& p) {
  std::vector<double> out(p.size());
  double acc = 0.0;
  for (std::size_t i = 0; i < p.size(); ++i) {
    acc = (i == 0) ? p[0] : acc + p[i];
    out[i] = acc;
  }
  return out;
}

// dist.cpp:20-42 — rounded, truncated gamma demand.
std::vector<double> gamma_demand_pmf(double mean, double cv, int d_max) {
  if (!(mean > 0.0)) fail(PVI_ERR_PARAMETER, "gamma demand: mean must be > 0");
  if (!(cv > 0.0)) fail(PVI_ERR_PARAMETER, "gamma demand: cv must be > 0");
  if (d_max < 1) fail(PVI_ERR_PARAMETER, "gamma demand: d_max must be >= 1");
  const double shape = 1.0 / (cv * cv);
  const double scale = mean * cv * cv;
  std::vector<double> probs(static_cast<std::size_t>(d_max) + 1);
  double lo = 0.0, partial = 0.0;
  for (int d = 0; d < d_max; ++d) {
    const double x = d + 0.5;
    const double hi = x <= 0.0 ? 0.0 : pvi_gamma_p(shape, x / scale);
    probs[d] = hi - lo;
    partial += probs[d];
    lo = hi;
  }
  probs[d_max] = std::max(0.0, 1.0 - partial);
  return probs;
}

// dist.cpp:44-60
std::vector<double> poisson_pmf(double mean, int upper) {
  if (mean < 0.0) fail(PVI_ERR_PARAMETER, "poisson: mean must be >= 0");
  if (upper < 0) fail(PVI_ERR_PARAMETER, "poisson: upper must be >= 0");
  std::vector<double> probs(static_cast<std::size_t>(upper) + 1, 0.0);
  if (mean == 0.0) {
    probs[0] = 1.0;
  } else {
    const double log_mean = std::log(mean);
    for (int k = 0; k <= upper; ++k) probs[k] = std::exp(-mean + k * log_mean - std::lgamma(k + 1.0));
  }
  return probs;
}

// dist.cpp:62-79
int poisson_quantile(double mean, double q) {
  if (mean < 0.0) fail(PVI_ERR_PARAMETER, "poisson quantile: mean must be >= 0");
  if (!(q >= 0.0 && q <= 1.0)) fail(PVI_ERR_PARAMETER, "poisson quantile: q must be in [0, 1]");
  if (q == 0.0 || mean == 0.0) return 0;
  const int cap = static_cast<int>(mean + 50.0 * std::sqrt(mean) + 64.0);
  double term = std::exp(-mean);
  double cum = term;
  int k = 0;
  while (cum < q && k < cap) {
    ++k;
    term *= mean / k;
    cum += term;
  }
  return k;
}

// dist.cpp:81-102
std::vector<double> negbinom_pmf(double n, double delta, int d_max) {
  if (!(n > 0.0)) fail(PVI_ERR_PARAMETER, "negbinom: n must be > 0");
  if (!(delta > 0.0)) fail(PVI_ERR_PARAMETER, "negbinom: delta must be > 0");
  if (d_max < 1) fail(PVI_ERR_PARAMETER, "negbinom: d_max must be >= 1");
  const double p = n / (n + delta);
  const double log_p = std::log(p);
  const double log_q = std::log1p(-p);
  const double lg_n = std::lgamma(n);
  std::vector<double> probs(static_cast<std::size_t>(d_max) + 1);
  double partial = 0.0;
  for (int d = 0; d < d_max; ++d) {
    const double log_mass = std::lgamma(n + d) - lg_n - std::lgamma(d + 1.0) + n * log_p + d * log_q;
    probs[d] = std::exp(log_mass);
    partial += probs[d];
  }
  probs[d_max] = std::max(0.0, 1.0 - partial);
  return probs;
}

inline int pos(int x) { return x > 0 ? x : 0; }

std::uint64_t binomial_count(std::uint64_t n, std::uint64_t k) {
  std::uint64_t c = 1;
  for (std::uint64_t i = 1; i <= k; ++i) c = c * (n - k + i) / i;
  return c;
}

}  // namespace

// ---------------------------------------------------------------------------
// Scenario A (scenario_a.cpp:46-68)

std::unique_ptr<Model> build_scenario_a(const pvi_scenario_a_params& p) {
  if (p.useful_life < 1 || p.useful_life > 12) fail(PVI_ERR_PARAMETER, "scenario a: useful_life out of range");
  if (p.lead_time < 1) fail(PVI_ERR_PARAMETER, "scenario a: lead_time must be >= 1");
  if (p.max_order < 0) fail(PVI_ERR_PARAMETER, "scenario a: max_order must be >= 0");
  auto m = std::make_unique<Model>();
  m->scenario = PVI_SCENARIO_A;
  m->pa = p;
  const int components = p.useful_life + p.lead_time - 1;
  m->space.init(std::vector<int>(components, p.max_order + 1));
  m->a_pmf = gamma_demand_pmf(p.demand_mean, p.demand_cv, p.max_demand);
  m->a_cdf = prefix_sum(m->a_pmf);
  m->n_actions = static_cast<std::uint32_t>(p.max_order + 1);
  m->n_outcomes = static_cast<std::uint64_t>(p.max_demand) + 1;
  m->gamma = p.discount_factor;
  m->default_test = PVI_TEST_VALUE_SPAN;
  m->periodicity = 1;
  std::ostringstream os;
  os << "scenario=a;m=" << p.useful_life << ";L=" << p.lead_time
     << ";issuing=" << (p.issuing == 0 ? "fifo" : "lifo") << ";A_max=" << p.max_order
     << ";D_max=" << p.max_demand << ";C_v=" << p.unit_cost << ";C_h=" << p.holding_cost
     << ";C_s=" << p.shortage_cost << ";C_w=" << p.wastage_cost << ";mu=" << p.demand_mean
     << ";cv=" << p.demand_cv << ";gamma=" << p.discount_factor;
  m->fingerprint = os.str();
  return m;
}

// ---------------------------------------------------------------------------
// Scenario B (scenario_b.cpp:30-166)

std::unique_ptr<Model> build_scenario_b(const pvi_scenario_b_params& p) {
  if (p.useful_life < 1 || p.useful_life > 8) fail(PVI_ERR_PARAMETER, "scenario b: useful_life out of range");
  if (p.substitution_prob < 0.0 || p.substitution_prob > 1.0)
    fail(PVI_ERR_PARAMETER, "scenario b: substitution_prob must be in [0, 1]");
  auto newsvendor = [&](double mean, double revenue, double cost) {
    if (!(revenue > 0.0)) fail(PVI_ERR_PARAMETER, "newsvendor: revenue must be > 0");
    const double ratio = std::max(0.0, (revenue - cost) / revenue);
    return poisson_quantile(p.useful_life * mean, ratio);
  };
  auto md = std::make_unique<Model>();
  Model& m = *md;
  m.scenario = PVI_SCENARIO_B;
  m.pb = p;
  const int life = p.useful_life;
  const int max_a = p.max_order_a >= 0 ? p.max_order_a : newsvendor(p.demand_mean_a, p.revenue_a, p.unit_cost_a);
  const int max_b = p.max_order_b >= 0 ? p.max_order_b : newsvendor(p.demand_mean_b, p.revenue_b, p.unit_cost_b);
  m.b_na = max_a + 1;
  m.b_nb = max_b + 1;
  m.b_cap_a = life * max_a;
  m.b_cap_b = life * max_b;
  std::vector<int> radices(2 * life);
  for (int i = 0; i < life; ++i) radices[i] = max_a + 1;
  for (int i = life; i < 2 * life; ++i) radices[i] = max_b + 1;
  m.space.init(radices);
  m.n_actions = static_cast<std::uint32_t>((max_a + 1) * (max_b + 1));
  m.n_outcomes = static_cast<std::uint64_t>(m.b_cap_a + 1) * (m.b_cap_b + 1);
  m.gamma = p.discount_factor;
  m.default_test = PVI_TEST_CHANGE_SPAN;
  m.periodicity = 1;

  // build_tables (scenario_b.cpp:62-155)
  const double mu_a = p.demand_mean_a, mu_b = p.demand_mean_b, rho = p.substitution_prob;
  m.b_dmax = life * std::max(max_a, max_b) + 2;
  m.b_ymax = m.b_cap_b;
  const auto table_len = [](double mean, int needed) {
    return std::max<int>(needed, static_cast<int>(mean + 20.0 * std::sqrt(mean) + 60.0)) + 1;
  };
  const int len_a = table_len(mu_a, m.b_dmax);
  const int len_b = table_len(mu_b, m.b_ymax + m.b_dmax);
  m.b_pmf_a = poisson_pmf(mu_a, len_a - 1);
  m.b_pmf_b = poisson_pmf(mu_b, len_b - 1);
  const auto survival = [](const std::vector<double>& pmf) {
    std::vector<double> sf(pmf.size() + 1, 0.0);
    for (std::size_t i = pmf.size(); i-- > 0;) sf[i] = sf[i + 1] + pmf[i];
    return sf;
  };
  m.b_sf_a = survival(m.b_pmf_a);
  m.b_sf_b = survival(m.b_pmf_b);
  const auto cdf = [](const std::vector<double>& pmf) {
    std::vector<double> out(pmf.size());
    double acc = 0.0;
    for (std::size_t i = 0; i < pmf.size(); ++i) out[i] = (acc += pmf[i]);
    return out;
  };
  m.b_cdf_a = cdf(m.b_pmf_a);
  m.b_cdf_b = cdf(m.b_pmf_b);

  const int dn = m.b_dmax + 1;
  const int yn = m.b_ymax + 1;
  m.b_pu.assign(static_cast<std::size_t>(yn) * dn, 0.0);
  m.b_pz.assign(static_cast<std::size_t>(yn) * dn, 0.0);
  m.b_pz_cum.assign(static_cast<std::size_t>(yn) * dn, 0.0);
  std::vector<double> log_fact(len_b + 1, 0.0);
  for (int i = 1; i <= len_b; ++i) log_fact[i] = log_fact[i - 1] + std::log(double(i));
  const double log_rho = rho > 0.0 ? std::log(rho) : 0.0;
  const double log_1mrho = rho < 1.0 ? std::log1p(-rho) : 0.0;
  const auto& pmf_a = m.b_pmf_a;
  const auto& pmf_b = m.b_pmf_b;
  for (int y = 0; y < yn; ++y) {
    double* pu_row = &m.b_pu[static_cast<std::size_t>(y) * dn];
    const double sf_y = m.b_sf_b[y];
    if (sf_y < 1e-12) {
      pu_row[0] = 1.0;
    } else if (rho == 1.0) {
      for (int du = 0; du < dn; ++du)
        if (du + y < len_b) pu_row[du] = pmf_b[du + y] / sf_y;
    } else {
      const int c_hi = len_b - 1 - y;
      double acc = 0.0, w = 1.0;
      for (int c = 0; c <= c_hi; ++c) {
        acc += pmf_b[c + y] * w;
        w *= 1.0 - rho;
      }
      pu_row[0] = acc / sf_y;
      if (rho > 0.0) {
        for (int du = 1; du < dn; ++du) {
          double sum = 0.0;
          for (int c = du; c <= c_hi; ++c) {
            const double log_binom = log_fact[c] - log_fact[du] - log_fact[c - du] + du * log_rho +
                                     (c - du) * log_1mrho;
            sum += pmf_b[c + y] * std::exp(log_binom);
          }
          pu_row[du] = sum / sf_y;
        }
      }
    }
    double* pz_row = &m.b_pz[static_cast<std::size_t>(y) * dn];
    double* pz_cum_row = &m.b_pz_cum[static_cast<std::size_t>(y) * dn];
    double cum = 0.0;
    for (int dz = 0; dz < dn; ++dz) {
      double sum = 0.0;
      for (int k = 0; k <= dz; ++k) sum += pmf_a[k] * pu_row[dz - k];
      pz_row[dz] = sum;
      pz_cum_row[dz] = cum;
      cum += sum;
    }
  }

  // Tile order for the device sweep: the two least-significant digits of
  // the state index, sorted by their stock sum, so a warp's lanes share
  // loop trip counts and V cache lines.
  const int nd = static_cast<int>(m.space.radix.size());
  const int r0 = m.space.radix[nd - 1];
  const int r1 = nd >= 2 ? m.space.radix[nd - 2] : 1;
  std::vector<std::uint16_t> order(static_cast<std::size_t>(r0) * r1);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](std::uint16_t x, std::uint16_t y) {
    return (x % r0) + (x / r0) < (y % r0) + (y / r0);
  });
  m.b_lane_order = order;

  std::ostringstream os;
  os << "scenario=b;m=" << p.useful_life << ";mu_a=" << p.demand_mean_a << ";mu_b=" << p.demand_mean_b
     << ";A_a_max=" << max_a << ";A_b_max=" << max_b << ";C_v_a=" << p.unit_cost_a
     << ";C_v_b=" << p.unit_cost_b << ";C_r_a=" << p.revenue_a << ";C_r_b=" << p.revenue_b
     << ";rho=" << p.substitution_prob << ";gamma=" << p.discount_factor;
  m.fingerprint = os.str();
  return md;
}

// ---------------------------------------------------------------------------
// Scenario C (scenario_c.cpp:23-123)

std::unique_ptr<Model> build_scenario_c(const pvi_scenario_c_params& p) {
  const int life = p.useful_life;
  if (life < 2 || life > 12) fail(PVI_ERR_PARAMETER, "scenario c: useful_life out of range");
  if (p.max_order < 0) fail(PVI_ERR_PARAMETER, "scenario c: max_order must be >= 0");
  auto md = std::make_unique<Model>();
  Model& m = *md;
  m.scenario = PVI_SCENARIO_C;
  m.pc = p;
  std::vector<int> radices(life);
  radices[0] = 7;
  for (int i = 1; i < life; ++i) radices[i] = p.max_order + 1;
  m.space.init(radices);
  const std::uint64_t n_comp = binomial_count(p.max_order + life, life);
  if (n_comp > 0xffffffffull) fail(PVI_ERR_CAPACITY, "scenario c: composition table too large", n_comp);
  m.c_n_comp = static_cast<std::uint32_t>(n_comp);
  m.n_actions = static_cast<std::uint32_t>(p.max_order + 1);
  m.n_outcomes = static_cast<std::uint64_t>(p.max_demand + 1) * n_comp;
  m.gamma = p.discount_factor;
  m.default_test = PVI_TEST_PERIODIC_SPAN;
  m.periodicity = 7;

  const int dn = p.max_demand + 1;
  m.c_pmf.resize(7 * static_cast<std::size_t>(dn));
  m.c_cdf.resize(7 * static_cast<std::size_t>(dn));
  for (int tau = 0; tau < 7; ++tau) {
    const auto pmf = negbinom_pmf(p.demand_successes[tau], p.demand_means[tau], p.max_demand);
    const auto cdf = prefix_sum(pmf);
    std::copy(pmf.begin(), pmf.end(), m.c_pmf.begin() + tau * dn);
    std::copy(cdf.begin(), cdf.end(), m.c_cdf.begin() + tau * dn);
  }

  // receipt_category_probs (scenario_c.cpp:23-35)
  m.c_receipt.resize(static_cast<std::size_t>(p.max_order + 1) * life);
  for (int a = 0; a <= p.max_order; ++a) {
    double* probs = &m.c_receipt[static_cast<std::size_t>(a) * life];
    double denom = 1.0;
    for (int k = 2; k <= life; ++k) {
      probs[k - 1] = std::exp(p.life_intercepts[k - 2] + p.life_slopes[k - 2] * a);
      denom += probs[k - 1];
    }
    probs[0] = 1.0;
    for (int k = 0; k < life; ++k) probs[k] /= denom;
  }

  // Composition enumeration (scenario_c.cpp:72-99): odometer over all age
  // profiles with total <= cap, freshest first.
  const int cap = p.max_order;
  if (n_comp * life > (1ull << 32)) fail(PVI_ERR_CAPACITY, "scenario c: composition table too large", n_comp);
  m.c_comp.reserve(n_comp * life);
  m.c_comp_sum.reserve(n_comp);
  std::vector<int> tuple(life, 0);
  int total = 0;
  for (;;) {
    m.c_comp_sum.push_back(static_cast<std::int8_t>(total));
    for (int i = 0; i < life; ++i) m.c_comp.push_back(static_cast<std::int8_t>(tuple[i]));
    int i = life - 1;
    while (i >= 0) {
      if (total < cap) {
        ++tuple[i];
        ++total;
        break;
      }
      total -= tuple[i];
      tuple[i] = 0;
      --i;
    }
    if (i < 0) break;
  }
  std::vector<double> log_fact(cap + 1, 0.0);
  for (int i = 1; i <= cap; ++i) log_fact[i] = log_fact[i - 1] + std::log(double(i));
  m.c_offsets.assign(cap + 2, 0);
  for (int a = 0; a <= cap; ++a) {
    m.c_offsets[a] = static_cast<std::uint32_t>(m.c_ids.size());
    std::vector<double> log_p(life);
    for (int j = 0; j < life; ++j) log_p[j] = std::log(m.c_receipt[static_cast<std::size_t>(a) * life + j]);
    for (std::uint32_t ci = 0; ci < m.c_comp_sum.size(); ++ci) {
      if (m.c_comp_sum[ci] != a) continue;
      const std::int8_t* yt = &m.c_comp[static_cast<std::size_t>(ci) * life];
      double log_mass = log_fact[a];
      for (int i = 0; i < life; ++i) {
        const int count = yt[i];
        if (count == 0) continue;
        log_mass += count * log_p[life - 1 - i] - log_fact[count];
      }
      m.c_ids.push_back(ci);
      m.c_probs.push_back(std::exp(log_mass));
    }
  }
  m.c_offsets[cap + 1] = static_cast<std::uint32_t>(m.c_ids.size());

  // Factored-sweep helper (not used by the exact path): the multinomial
  // split of a units over the age categories 1..m equals sequential
  // binomials -- y_1 ~ Bin(a, q_1), y_2 ~ Bin(a - y_1, q_2), ... with
  // q_k = p_k / (p_k + .. + p_m) and p = receipt_category_probs(a).
  // c_binom[a][k-1][b][y] = Bin(y; b, q_k(a)).  With an exogenous law (all
  // receipt rows equal) the tables are shared by every order size.
  m.c_exogenous = true;
  for (int a = 1; a <= cap && m.c_exogenous; ++a)
    for (int j = 0; j < life; ++j)
      if (m.c_receipt[static_cast<std::size_t>(a) * life + j] != m.c_receipt[j]) m.c_exogenous = false;
  if (life >= 2) {
    const int r = cap + 1;
    const std::size_t per_k = static_cast<std::size_t>(r) * r;
    m.c_binom.assign(static_cast<std::size_t>(r) * (life - 1) * per_k, 0.0);
    for (int a = 0; a <= cap; ++a) {
      const double* p_a = &m.c_receipt[static_cast<std::size_t>(a) * life];
      for (int k = 1; k <= life - 1; ++k) {
        double tail = 0.0;
        for (int j = k; j <= life; ++j) tail += p_a[j - 1];
        const double q = tail > 0.0 ? p_a[k - 1] / tail : 0.0;
        double* tab = &m.c_binom[(static_cast<std::size_t>(a) * (life - 1) + (k - 1)) * per_k];
        for (int b = 0; b <= cap; ++b)
          for (int y = 0; y <= b; ++y) {
            double w;
            if (q <= 0.0) w = y == 0 ? 1.0 : 0.0;
            else if (q >= 1.0) w = y == b ? 1.0 : 0.0;
            else w = std::exp(log_fact[b] - log_fact[y] - log_fact[b - y] + y * std::log(q) +
                              (b - y) * std::log1p(-q));
            tab[b * r + y] = w;
          }
      }
    }
  }

  std::ostringstream os;
  os << "scenario=c;m=" << life << ";A_max=" << p.max_order << ";D_max=" << p.max_demand
     << ";C_f=" << p.fixed_order_cost << ";C_h=" << p.holding_cost << ";C_s=" << p.shortage_cost
     << ";C_w=" << p.wastage_cost << ";gamma=" << p.discount_factor << ";n=";
  for (double v : p.demand_successes) os << v << ",";
  os << ";delta=";
  for (double v : p.demand_means) os << v << ",";
  os << ";c0=";
  for (int k = 0; k < life - 1; ++k) os << p.life_intercepts[k] << ",";
  os << ";c1=";
  for (int k = 0; k < life - 1; ++k) os << p.life_slopes[k] << ",";
  m.fingerprint = os.str();
  return md;
}

// ---------------------------------------------------------------------------
// Explicit-table MDP (tests/support/tabular_mdp.hpp:16-119)

std::unique_ptr<Model> build_tabular(std::uint64_t ns, std::uint32_t na, std::uint64_t no,
                                     double gamma, const std::uint64_t* next, const double* reward,
                                     const double* prob, const double* initial) {
  if (ns == 0 || na == 0 || no == 0) fail(PVI_ERR_PARAMETER, "tabular: empty dimension");
  if (ns > 0x7fffffffull) fail(PVI_ERR_PARAMETER, "tabular: too many states");
  auto m = std::make_unique<Model>();
  m->scenario = PVI_TABULAR;
  m->space.init({static_cast<int>(ns)});
  m->n_actions = na;
  m->n_outcomes = no;
  m->gamma = gamma;
  const std::size_t size = ns * na * no;
  m->t_next.assign(next, next + size);
  m->t_reward.assign(reward, reward + size);
  m->t_prob.assign(prob, prob + size);
  for (std::size_t i = 0; i < size; ++i)
    if (m->t_next[i] >= ns) fail(PVI_ERR_PARAMETER, "tabular: next state out of range");
  m->t_initial.assign(ns, 0.0);
  if (initial) m->t_initial.assign(initial, initial + ns);
  m->fingerprint = "tabular;" + std::to_string(ns) + ";" + std::to_string(na) + ";" +
                   std::to_string(no) + ";" + std::to_string(gamma);
  return m;
}

// ---------------------------------------------------------------------------
// Presets (presets.cpp:16-130)

std::unique_ptr<Model> build_preset(const std::string& name, std::uint64_t* fixed_iterations,
                                    std::uint64_t* checkpoint_every) {
  std::uint64_t fixed = 0, every = 0;
  std::unique_ptr<Model> out;
  struct ARow { int lead; double cw; int lifo; };
  static const ARow a_rows[8] = {{1, 7.0, 1}, {1, 7.0, 0}, {1, 10.0, 1}, {1, 10.0, 0},
                                 {2, 7.0, 1}, {2, 7.0, 0}, {2, 10.0, 1}, {2, 10.0, 0}};
  struct BRow { const char* name; int m; double mu_a, mu_b; int max_a, max_b; bool fixed100; };
  static const BRow b_rows[10] = {
      {"b/m2/exp1", 2, 5, 5, -1, -1, false}, {"b/m2/exp2", 2, 7, 3, -1, -1, false},
      {"b/m3/exp1", 3, 5, 5, -1, -1, false}, {"b/m3/exp2", 3, 7, 3, -1, -1, false},
      {"b/m3/exp3", 3, 5, 5, 13, 13, false}, {"b/m3/exp4", 3, 7, 3, 20, 4, false},
      {"b/m2/p1", 2, 5, 5, 10, 10, true},    {"b/m2/p2", 2, 5, 6, 10, 12, true},
      {"b/m2/p3", 2, 6, 6, 12, 12, true},    {"b/m2/p4", 2, 7, 7, 13, 13, true}};
  if (name.rfind("a/", 0) == 0) {
    for (int m = 2; m <= 5 && !out; ++m)
      for (int e = 1; e <= 8 && !out; ++e)
        if (name == "a/m" + std::to_string(m) + "/exp" + std::to_string(e)) {
          pvi_scenario_a_params p;
          pvi_scenario_a_defaults(&p);
          p.useful_life = m;
          p.lead_time = a_rows[e - 1].lead;
          p.wastage_cost = a_rows[e - 1].cw;
          p.issuing = a_rows[e - 1].lifo;
          out = build_scenario_a(p);
          every = 100;
        }
  } else if (name.rfind("b/", 0) == 0) {
    for (const auto& r : b_rows)
      if (name == r.name) {
        pvi_scenario_b_params p;
        pvi_scenario_b_defaults(&p);
        p.useful_life = r.m;
        p.demand_mean_a = r.mu_a;
        p.demand_mean_b = r.mu_b;
        p.max_order_a = r.max_a;
        p.max_order_b = r.max_b;
        if (r.fixed100) fixed = 100;
        out = build_scenario_b(p);
        every = 1;
        break;
      }
  } else if (name.rfind("c/", 0) == 0) {
    for (int m : {3, 5, 8}) {
      for (int e = 1; e <= 2 && !out; ++e)
        if (name == "c/m" + std::to_string(m) + "/exp" + std::to_string(e)) {
          pvi_scenario_c_params p;
          pvi_scenario_c_defaults(&p);
          p.useful_life = m;
          const bool endo = e == 2;
          // shelf_life_coefficients (presets.cpp:50-68)
          std::vector<double> c0, c1;
          if (m == 3) {
            c0 = {1.0, 0.5};
            c1 = endo ? std::vector<double>{0.40, 0.80} : std::vector<double>{0.0, 0.0};
          } else if (m == 5) {
            if (endo) {
              c0 = {1.9, 3.1, 3.1, 2.5};
              c1 = {-0.03, -0.06, -0.03, -0.09};
            } else {
              c0 = {1.6, 2.6, 2.8, 1.6};
              c1 = {0.0, 0.0, 0.0, 0.0};
            }
          } else {
            c0 = {0.8, 1.4, 1.9, 2.3, 1.7, 1.2, 0.8};
            c1 = endo ? std::vector<double>{-0.03, -0.04, -0.05, -0.06, -0.07, -0.08, -0.09}
                      : std::vector<double>(7, 0.0);
          }
          for (int k = 0; k < m - 1; ++k) {
            p.life_intercepts[k] = c0[k];
            p.life_slopes[k] = c1[k];
          }
          out = build_scenario_c(p);
          every = 1;
        }
    }
  }
  if (!out) fail(PVI_ERR_CONFIG, "unknown preset: " + name);
  if (fixed_iterations) *fixed_iterations = fixed;
  if (checkpoint_every) *checkpoint_every = every;
  return out;
}

// ---------------------------------------------------------------------------
// Work model

double Model::terms_per_sweep() const {
  const double n = static_cast<double>(space.count);
  switch (scenario) {
    case PVI_SCENARIO_A:
      return n * n_actions * (pa.max_demand + 1);
    case PVI_SCENARIO_B: {
      // sum_s (I_a+1)(I_b+1) factorises over the two products' digit sums.
      const int life = pb.useful_life;
      auto digit_sum_mean = [&](int radix) {
        // E[sum of `life` iid uniform digits in 0..radix-1] + 1
        return life * (radix - 1) / 2.0 + 1.0;
      };
      const double ca = std::pow(static_cast<double>(b_na), life) * digit_sum_mean(b_na);
      const double cb = std::pow(static_cast<double>(b_nb), life) * digit_sum_mean(b_nb);
      return ca * cb * n_actions;
    }
    case PVI_SCENARIO_C:
      return n * (pc.max_demand + 1) * static_cast<double>(c_n_comp);
    default:
      return n * n_actions * static_cast<double>(n_outcomes);
  }
}

// Loop bounds of the factored kernels (vi_kernels.cu, K1-B / K1-C factored),
// summed over one full sweep.
double Model::factored_fmas() const {
  if (scenario == PVI_SCENARIO_B) {
    const int life = pb.useful_life;
    // sum over the `life` digits (x_1 = digits[0]) of one product's block
    auto loops = [&](int radix, bool boundary) {
      double acc = 0.0;
      const long long count = static_cast<long long>(std::pow(double(radix), life));
      for (long long v = 0; v < count; ++v) {
        long long rem = v;
        int x1 = 0, tot = 0;
        for (int k = 0; k < life; ++k) {
          const int d = static_cast<int>(rem % radix);
          rem /= radix;
          if (k == 0) x1 = d;
          tot += d;
        }
        const int above = tot - x1;
        if (boundary) acc += above + 1;  // stage 2: h_a = x_1+1..I_a plus the merged block
        else if (tot > 0) acc += above + 1 - (x1 >= tot ? 1 : 0);
      }
      return acc;
    };
    const double na = b_na, nb = b_nb;
    const double stage1 = std::pow(na, life) * loops(b_nb, false) * nb;
    if (life == 3 && b_nb == 16 && b_na <= 16) {
      // k_b_fact_qp3 per (x_b, o_a): 2 FMAs per Q, both running sums of
      // every lane at every step, and the x_3-long diagonal constants
      const double n_xa = na * na * na;
      const double per = 2.0 * n_xa * nb + 4.0 * na * na * na * nb + 2.0 * na * na * (na - 1) * nb;
      return stage1 + std::pow(nb, life) * na * per;
    }
    const double stage2 = std::pow(nb, life) * na * loops(b_na, true) * nb * 2.0;
    return stage1 + stage2;
  }
  if (scenario == PVI_SCENARIO_C) {
    const int life = pc.useful_life;
    const double r = pc.max_order + 1;
    const double wb = std::pow(r, life - 1);
    const double g = 7.0 * wb * r * (pc.max_demand + 1);  // profile table
    double pass = 0.0, fin = 0.0;
    for (int a = 0; a <= pc.max_order; ++a) {
      fin += a + 1;                                       // fused k = 1 pass, per state
      if (c_exogenous) pass += a + 1;                     // shared table: b = a, all b
      else pass += (a + 1.0) * (a + 2.0) / 2.0;           // table a: b <= a
    }
    return g + (life - 2) * 7.0 * wb * pass + static_cast<double>(space.count) * fin;
  }
  if (scenario == PVI_SCENARIO_A && n_actions <= 16) {
    // k_a_fact_lifo: one (carried + 1)-profile sum per x_1 group;
    // k_a_fact_fifo: per diagonal the x_3.. block plus one running-sum step
    // per x_2; both then 2 FMAs per (state, order) for Q.
    const int m = pa.useful_life, rx = pa.max_order + 1;
    const double na = n_actions, pipe = std::pow(double(rx), pa.lead_time - 1);
    long long count = 1;
    for (int j = 0; j < m; ++j) count *= rx;
    double per_pipe = 0.0;
    for (long long v = 0; v < count; ++v) {
      long long rem = v;
      int xs[14], above = 0, carried = 0;
      for (int j = 1; j <= m; ++j) {  // x_1 = least significant
        xs[j] = static_cast<int>(rem % rx);
        rem /= rx;
        if (j >= 2) carried += xs[j];
        if (j >= 3) above += xs[j];
      }
      if (pa.issuing != 0) {
        if (xs[1] == 0) per_pipe += (carried + 1) * na;
      } else if (xs[1] == 0 && xs[2] == 0) {
        for (int s2 = 0; s2 <= 2 * (rx - 1); ++s2)
          per_pipe += (std::max(above, 1) + std::min(s2, rx - 1) + 1) * na;
      }
    }
    return pipe * per_pipe + 2.0 * na * static_cast<double>(space.count);
  }
  return terms_per_sweep();
}

bool Model::b_law_unit() const {
  std::call_once(b_law_once, [&] {
    if (scenario != PVI_SCENARIO_B) return;
    const int m = pb.useful_life, dnh = b_dmax + 1, ima = m * (b_na - 1), imb = m * (b_nb - 1);
    double worst = 0.0;
    for (int ia = 0; ia <= ima; ++ia)
      for (int ibh = 0; ibh <= imb; ++ibh) {
        double pt = 0.0;
        for (int ha = 0; ha <= ia; ++ha)
          for (int hb = 0; hb <= ibh; ++hb) {
            double pr;
            if (ha < ia)
              pr = hb < ibh ? b_pmf_a[ha] * b_pmf_b[hb] : b_pz[ibh * dnh + ha] * b_sf_b[ibh];
            else
              pr = hb < ibh ? b_sf_a[ia] * b_pmf_b[hb] : (1.0 - b_pz_cum[ibh * dnh + ia]) * b_sf_b[ibh];
            pt += pr;
          }
        worst = std::max(worst, std::fabs(pt - 1.0));
      }
    b_law_unit_v = worst <= 1e-12;
  });
  return b_law_unit_v;
}

double Model::state_cost(std::uint64_t s) const {
  if (scenario != PVI_SCENARIO_B) return 1.0;
  int st[kMaxDigits];
  space.decode(s, st);
  const int life = pb.useful_life;
  int ia = 0, ib = 0;
  for (int i = 0; i < life; ++i) ia += st[i];
  for (int i = life; i < 2 * life; ++i) ib += st[i];
  if (algorithm == PVI_ALGO_FACTORED) {
    if (life == 3 && b_nb == 16 && b_na <= 16) {
      // k_b_fact_qw3: per x_3 pair p, 16 diagonal steps (~245 instructions)
      // plus 2p + 2 diagonal-constant steps (~114), per order_a
      const int p = st[0] / 2;
      return 34.4 + 2.0 * (p + 1);
    }
    // factored stage 2: one merged block plus h_a = x_1+1..I_a, per order_a
    const int x1 = st[life - 1];
    return double(ia - x1 + 1) + 2.0;
  }
  return double(ia + 1) * double(ib + 1);
}

std::uint64_t Model::chunk_align() const {
  if (scenario == PVI_SCENARIO_C && algorithm == PVI_ALGO_FACTORED) return 0;
  if (scenario == PVI_SCENARIO_B && algorithm == PVI_ALGO_FACTORED && pb.useful_life == 3) {
    // k_b_fact_qw3 works on pairs of x_3 digits: 2 * na^2 * nb^3 states
    return 2ull * b_na * b_na * b_nb * b_nb * b_nb;
  }
  return std::max<std::uint64_t>(tile_states(), 1);
}

std::uint64_t Model::tile_states() const {
  if (scenario == PVI_SCENARIO_B && algorithm == PVI_ALGO_FACTORED && pb.useful_life == 3 &&
      b_nb == 16 && b_na <= 16) {
    // k_b_fact_qw3 works on pairs of x_3 digits: a shard owns whole pairs
    return 2ull * b_na * b_na * b_nb * b_nb * b_nb;
  }
  if (scenario == PVI_SCENARIO_B && algorithm == PVI_ALGO_FACTORED) {
    // shards own whole x_a groups (x_1 = 0..A_a, all x_b): stage 2 works on
    // groups of states that share x_2..x_m, so no group straddles two ranks
    std::uint64_t t = static_cast<std::uint64_t>(b_na);
    for (int i = 0; i < pb.useful_life; ++i) t *= static_cast<std::uint64_t>(b_nb);
    return t;
  }
  if (scenario == PVI_SCENARIO_B) return b_lane_order.size();
  return 1;
}

// ---------------------------------------------------------------------------
// Host transitions (naive-oracle path; scenario_{a,b,c}.cpp transition())

namespace {

int age_fifo(const int* x, int m, int demand, int* next) {
  const int expired = pos(x[1] - demand);
  int prefix = 0;
  for (int j = 1; j <= m - 1; ++j) {
    prefix += x[j];
    next[j] = pos(x[j + 1] - pos(demand - prefix));
  }
  return expired;
}

int age_lifo(const int* x, int m, int demand, int* next) {
  int suffix = 0;
  for (int j = 2; j <= m; ++j) suffix += x[j];
  const int expired = pos(x[1] - pos(demand - suffix));
  for (int j = 1; j <= m - 1; ++j) {
    suffix -= x[j + 1];
    next[j] = pos(x[j + 1] - pos(demand - suffix));
  }
  return expired;
}

double b_issued(const Model& m, int ha, int hb, int ia, int ib) {
  if (ha > ia || hb > ib) return 0.0;
  const bool ai = ha < ia, bi = hb < ib;
  const int dn = m.b_dmax + 1;
  if (ai && bi) return m.b_pmf_a[ha] * m.b_pmf_b[hb];
  if (!ai && bi) return m.b_sf_a[ia] * m.b_pmf_b[hb];
  if (ai) return m.b_pz[static_cast<std::size_t>(ib) * dn + ha] * m.b_sf_b[ib];
  return (1.0 - m.b_pz_cum[static_cast<std::size_t>(ib) * dn + ia]) * m.b_sf_b[ib];
}

}  // namespace

void host_transition(const Model& m, std::uint64_t s, std::uint32_t a, std::uint64_t w,
                     std::uint64_t* next, double* reward) {
  int st[2 * kMaxDigits] = {0}, nx[2 * kMaxDigits] = {0};
  if (s >= m.space.count) fail(PVI_ERR_INDEXING, "state out of range");
  if (a >= m.n_actions) fail(PVI_ERR_INDEXING, "action out of range");
  if (w >= m.n_outcomes) fail(PVI_ERR_INDEXING, "outcome out of range");
  switch (m.scenario) {
    case PVI_SCENARIO_A: {
      const auto& p = m.pa;
      const int life = p.useful_life, lead = p.lead_time, d = static_cast<int>(w);
      m.space.decode(s, st);
      int x[16], aged[16], xt = 0;
      for (int j = 1; j <= life; ++j) {
        x[j] = st[lead - 1 + life - j];
        xt += x[j];
      }
      const int expired = p.issuing == 0 ? age_fifo(x, life, d, aged) : age_lifo(x, life, d, aged);
      nx[0] = static_cast<int>(a);
      for (int k = 1; k <= lead - 2; ++k) nx[k] = st[k - 1];
      if (lead >= 2) nx[lead - 1] = st[lead - 2];
      for (int j = 1; j <= life - 1; ++j) nx[lead + life - 1 - j] = aged[j];
      *reward = -p.unit_cost * a - p.holding_cost * pos(xt - d - expired) -
                p.shortage_cost * pos(d - xt) - p.wastage_cost * expired;
      *next = m.space.encode(nx);
      return;
    }
    case PVI_SCENARIO_B: {
      const auto& p = m.pb;
      const int life = p.useful_life;
      m.space.decode(s, st);
      int xa[16], xb[16], ia = 0, ib = 0;
      for (int j = 1; j <= life; ++j) {
        xa[j] = st[life - j];
        xb[j] = st[2 * life - j];
        ia += xa[j];
        ib += xb[j];
      }
      const int ha = static_cast<int>(w / (m.b_cap_b + 1));
      const int hb = static_cast<int>(w % (m.b_cap_b + 1));
      if (ha > ia || hb > ib) fail(PVI_ERR_CONTRACT, "issued quantity exceeds stock on hand");
      const int oa = static_cast<int>(a) / m.b_nb, ob = static_cast<int>(a) % m.b_nb;
      int aa[16], ab[16];
      age_fifo(xa, life, ha, aa);
      age_fifo(xb, life, hb, ab);
      nx[0] = oa;
      nx[life] = ob;
      for (int j = 1; j <= life - 1; ++j) {
        nx[life - j] = aa[j];
        nx[2 * life - j] = ab[j];
      }
      *reward = -(p.unit_cost_a * oa + p.unit_cost_b * ob) + p.revenue_a * ha + p.revenue_b * hb;
      *next = m.space.encode(nx);
      return;
    }
    case PVI_SCENARIO_C: {
      const auto& p = m.pc;
      const int life = p.useful_life, cap = p.max_order;
      const std::uint64_t demand = w / m.c_n_comp;
      const std::uint32_t ci = static_cast<std::uint32_t>(w % m.c_n_comp);
      if (m.c_comp_sum[ci] != static_cast<int>(a))
        fail(PVI_ERR_CONTRACT, "delivery age profile does not sum to the order quantity");
      m.space.decode(s, st);
      const int tau = st[0];
      const std::int8_t* yt = &m.c_comp[static_cast<std::size_t>(ci) * life];
      int x[16], y[16], z[16];
      for (int j = 1; j <= life; ++j) y[j] = yt[life - j];
      x[life] = 0;
      for (int j = 1; j <= life - 1; ++j) x[j] = st[life - j];
      const int d = static_cast<int>(demand);
      int total = y[life];
      for (int j = 1; j <= life - 1; ++j) {
        z[j] = std::min(x[j] + y[j], cap);
        total += z[j];
      }
      nx[0] = (tau + 1) % 7;
      int prefix = 0;
      for (int j = 1; j <= life - 2; ++j) {
        prefix += z[j];
        nx[life - j] = pos(z[j + 1] - pos(d - prefix));
      }
      prefix += z[life - 1];
      nx[1] = pos(y[life] - pos(d - prefix));
      *reward = -(a > 0 ? p.fixed_order_cost : 0.0) - p.holding_cost * pos(total - d) -
                p.shortage_cost * pos(d - total) - p.wastage_cost * pos(z[1] - d);
      *next = m.space.encode(nx);
      return;
    }
    default: {
      const std::size_t i = (s * m.n_actions + a) * m.n_outcomes + w;
      *next = m.t_next[i];
      *reward = m.t_reward[i];
      return;
    }
  }
}

double host_outcome_probability(const Model& m, std::uint64_t s, std::uint32_t a, std::uint64_t w) {
  int st[2 * kMaxDigits] = {0};
  switch (m.scenario) {
    case PVI_SCENARIO_A:
      return m.a_pmf[w];
    case PVI_SCENARIO_B: {
      const int life = m.pb.useful_life;
      m.space.decode(s, st);
      int ia = 0, ib = 0;
      for (int i = 0; i < life; ++i) ia += st[i];
      for (int i = life; i < 2 * life; ++i) ib += st[i];
      const int ha = static_cast<int>(w / (m.b_cap_b + 1));
      const int hb = static_cast<int>(w % (m.b_cap_b + 1));
      return b_issued(m, ha, hb, ia, ib);
    }
    case PVI_SCENARIO_C: {
      const std::uint64_t demand = w / m.c_n_comp;
      const std::uint32_t ci = static_cast<std::uint32_t>(w % m.c_n_comp);
      if (m.c_comp_sum[ci] != static_cast<int>(a)) return 0.0;
      m.space.decode(s, st);
      const int tau = st[0];
      const std::uint32_t* b = m.c_ids.data() + m.c_offsets[a];
      const std::uint32_t* e = m.c_ids.data() + m.c_offsets[a + 1];
      const auto it = std::lower_bound(b, e, ci);
      const double cp = m.c_probs[m.c_offsets[a] + (it - b)];
      return m.c_pmf[static_cast<std::size_t>(tau) * (m.pc.max_demand + 1) + demand] * cp;
    }
    default:
      return m.t_prob[(s * m.n_actions + a) * m.n_outcomes + w];
  }
}

// ---------------------------------------------------------------------------
// SHA-256 (FIPS 180-4), for the checkpoint fingerprint (checkpoint.cpp:30-34).

void sha256(const void* data, std::size_t len, std::uint8_t out[32]) {
  static const std::uint32_t k[64] = {
      0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
      0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
      0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
      0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
      0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
      0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
      0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
      0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
  std::uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                        0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  auto rotr = [](std::uint32_t x, int n) { return (x >> n) | (x << (32 - n)); };
  const auto* bytes = static_cast<const std::uint8_t*>(data);
  std::vector<std::uint8_t> msg(bytes, bytes + len);
  msg.push_back(0x80);
  while (msg.size() % 64 != 56) msg.push_back(0);
  const std::uint64_t bits = static_cast<std::uint64_t>(len) * 8;
  for (int i = 7; i >= 0; --i) msg.push_back(static_cast<std::uint8_t>(bits >> (8 * i)));
  for (std::size_t off = 0; off < msg.size(); off += 64) {
    std::uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (std::uint32_t(msg[off + 4 * i]) << 24) | (std::uint32_t(msg[off + 4 * i + 1]) << 16) |
             (std::uint32_t(msg[off + 4 * i + 2]) << 8) | std::uint32_t(msg[off + 4 * i + 3]);
    for (int i = 16; i < 64; ++i) {
      const std::uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const std::uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    std::uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const std::uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
      const std::uint32_t ch = (e & f) ^ (~e & g);
      const std::uint32_t t1 = hh + S1 + ch + k[i] + w[i];
      const std::uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
      const std::uint32_t maj = (a & b) ^ (a & c) ^ (b & c);
      const std::uint32_t t2 = S0 + maj;
      hh = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) out[4 * i + j] = static_cast<std::uint8_t>(h[i] >> (24 - 8 * j));
}

}  // namespace pvi_b200
