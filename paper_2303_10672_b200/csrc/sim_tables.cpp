// Host-built sampling tables of the rollout kernel (sim_kernels.cu).  They
// change how a sample is FOUND, never its value: every table entry is the
// number the reference's sampler computes on the fly (rng.hpp:63-90), made
// with the same double operations in the same order (this file is compiled
// without FMA contraction, like the kernels), so the device draws stay
// bit-identical to RolloutRng + sample_from_cdf / sample_binomial.
#include <cstdint>
#include <vector>

#include "model.hpp"

namespace pvi_b200 {

// Guide table of sample_from_cdf (rng.hpp:63-73: the first i with cdf[i] > u,
// or size - 1): g[j] = that index for u = j / G.  For u in [j/G, (j+1)/G)
// the answer is >= g[j] (a larger u only removes candidates), so a forward
// scan from g[j] finds it -- about one comparison instead of log2(size)
// dependent loads.
//
// Buckets whose two ends give the same index hold no cdf boundary: every u
// in them samples that index, so the entry is stored as is and the kernel
// returns it without touching the cdf; the other entries are stored as
// -(start + 1) and the kernel scans from start.  With G = 1024 almost every
// bucket is exact (a 101-value demand law has at most 100 boundaries).
std::vector<std::int32_t> cdf_guide(const double* cdf, int size, int G) {
  std::vector<std::int32_t> g(G + 1);
  int i = 0;
  for (int j = 0; j <= G; ++j) {
    const double u = static_cast<double>(j) / G;  // exact: G is a power of two
    while (i < size - 1 && !(cdf[i] > u)) ++i;
    g[j] = i;
  }
  std::vector<std::int32_t> out(G + 1);
  for (int j = 0; j <= G; ++j) out[j] = (j < G && g[j] == g[j + 1]) ? g[j] : -(g[j] + 1);
  return out;
}

// Cumulative masses of sample_binomial (rng.hpp:76-90) for every trial count
// t = 0..T at one success probability p: row t (offset t (t + 1) / 2) holds
// cum_0..cum_t, the values the reference's loop compares u with.  The
// sample is the first k < t with cum_k > u, else t.  p must lie in (0, 1)
// (the sampler's early returns handle the rest).
std::vector<double> binomial_cum_table(int T, double p) {
  std::vector<double> out;
  out.reserve(static_cast<std::size_t>(T + 1) * (T + 2) / 2);
  const double ratio = p / (1.0 - p);
  for (int trials = 0; trials <= T; ++trials) {
    double mass = 1.0;
    for (int i = 0; i < trials; ++i) mass *= 1.0 - p;
    double cum = mass;
    out.push_back(cum);
    for (int k = 0; k < trials; ++k) {
      mass *= ratio * (trials - k) / (k + 1);
      cum += mass;
      out.push_back(cum);
    }
  }
  return out;
}

// Guide tables of the rows of a binomial_cum_table (the cdf_guide idea per
// trial count): row t's entry j is the sample for u = j / G -- the first
// k < t with cum_k > u, else t -- so the kernel's scan for u in [j/G,
// (j+1)/G) starts there (a larger u only moves the answer up): the same k
// after ~1 comparison instead of a scan from 0.
std::vector<std::int32_t> binomial_guide_table(const std::vector<double>& cum, int T, int G) {
  // (exact buckets stored as is, the others as -(start + 1): cdf_guide)
  std::vector<std::int32_t> g(static_cast<std::size_t>(T + 1) * (G + 1));
  std::vector<std::int32_t> r(G + 1);
  for (int t = 0; t <= T; ++t) {
    const double* row = cum.data() + static_cast<std::size_t>(t) * (t + 1) / 2;
    int k = 0;
    for (int j = 0; j <= G; ++j) {
      const double u = static_cast<double>(j) / G;  // exact: G is a power of two
      while (k < t && !(row[k] > u)) ++k;
      r[j] = k;
    }
    for (int j = 0; j <= G; ++j)
      g[static_cast<std::size_t>(t) * (G + 1) + j] = (j < G && r[j] == r[j + 1]) ? r[j] : -(r[j] + 1);
  }
  return g;
}

// Scenario C's receipt sampler (scenario_c.cpp sample_step: the age split of
// an order of a units as m - 1 sequential binomials with p_k = probs[k] /
// mass_left, mass_left = 1 - probs[0] - .. - probs[k-1] while units remain):
// one binomial_cum_table per (a, k) with p_k in (0, 1), concatenated;
// offsets[a * (m - 1) + k] = its first entry, or -1 (the kernel then runs the
// sampler's own loop / early returns).  receipt: (A_max + 1) x m.
void c_receipt_tables(const double* receipt, int max_order, int m, std::vector<double>& cum,
                      std::vector<std::int32_t>& offsets) {
  cum.clear();
  offsets.assign(static_cast<std::size_t>(max_order + 1) * (m - 1), -1);
  for (int a = 0; a <= max_order; ++a) {
    const double* probs = receipt + static_cast<std::size_t>(a) * m;
    double mass_left = 1.0;
    for (int k = 0; k + 1 < m; ++k) {
      if (mass_left <= 0.0) break;  // every later step is skipped too
      const double cond = probs[k] / mass_left;
      const double p = cond < 1.0 ? cond : 1.0;
      if (p > 0.0 && p < 1.0 && a > 0) {
        offsets[static_cast<std::size_t>(a) * (m - 1) + k] = static_cast<std::int32_t>(cum.size());
        const auto t = binomial_cum_table(a, p);
        cum.insert(cum.end(), t.begin(), t.end());
      }
      mass_left -= probs[k];
    }
  }
}

}  // namespace pvi_b200
