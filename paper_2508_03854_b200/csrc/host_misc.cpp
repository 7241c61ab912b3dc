// Host-side analytic helpers the reference's Python module exports next to
// the step (bindings/module.cpp:43-89, 133-145): the cost formulas
// (src/cost_model.cpp:24-55), normalized entropy (src/trainer.cpp:14-43)
// and the paper's Proposition-1 moment analysis that picks the AdaGrad
// scaling factor c (src/moment_analysis.cpp:69-148).  None of them runs in the
// training step; they are here so the reference's Python surface is complete
// over this library.  Same formulas, evaluation order and error messages.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ctx.h"

namespace s2d {
namespace {

uint64_t mix64h(uint64_t x) {  // rng.hpp:12-19
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

struct HostRng {  // CounterRng (rng.hpp:30-73)
  uint64_t key, ctr = 0;
  double spare = 0.0;
  bool have = false;
  HostRng(std::initializer_list<uint64_t> f) {
    uint64_t h = 0x8A5CD789635D2DFFULL;
    for (uint64_t x : f) h = mix64h(h + 0x9E3779B97F4A7C15ULL + x);
    key = h;
  }
  uint64_t next_u64() { return mix64h(key + (++ctr) * 0x9E3779B97F4A7C15ULL); }
  double next_uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_uniform_pos() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
  double next_normal() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = next_uniform_pos(), u2 = next_uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 2.0 * 3.141592653589793 * u2;  // == std::numbers::pi (rng.hpp:62)
    spare = r * std::sin(t);
    have = true;
    return r * std::cos(t);
  }
};

// GradientNoiseModel via make_noise_model (moment_analysis.cpp:26-36)
struct Noise {
  std::vector<double> mu;
  double sigma;
  uint32_t dim, b;
};

Noise make_noise(double mu_norm, double sigma, uint32_t dim, uint32_t b) {
  if (dim == 0) throw Error(S2D_EINVAL, "dim must be >= 1");
  if (!(sigma >= 0)) throw Error(S2D_EINVAL, "sigma must be >= 0");
  if (b == 0) throw Error(S2D_EINVAL, "batch must be >= 1");
  Noise m{std::vector<double>(dim, 0.0), sigma, dim, b};
  m.mu[0] = mu_norm;
  return m;
}

double norm_sq(const std::vector<double>& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return s;
}

// fixed binary-tree mean (moment_analysis.cpp:48-67)
std::vector<double> pairwise_mean(std::vector<std::vector<double>>& vecs) {
  size_t k = vecs.size();
  const double inv = 1.0 / static_cast<double>(k);
  while (k > 1) {
    const size_t half = k / 2;
    for (size_t p = 0; p < half; ++p) {
      auto& dst = vecs[p];
      const auto& a = vecs[2 * p];
      const auto& bb = vecs[2 * p + 1];
      for (size_t j = 0; j < dst.size(); ++j) dst[j] = a[j] + bb[j];
    }
    if (k % 2) vecs[half] = vecs[k - 1];
    k = half + (k % 2);
  }
  std::vector<double> out = vecs[0];
  for (double& x : out) x *= inv;
  return out;
}

double closed_form(const Noise& m, uint32_t groups) {  // moment_analysis.cpp:128-141
  if (groups == 0) throw Error(S2D_EINVAL, "groups must be >= 1");
  const double M = static_cast<double>(groups);
  if (m.sigma == 0.0) return 1.0;
  const double signal = norm_sq(m.mu);
  if (signal == 0.0) return M;
  const double noise = static_cast<double>(m.dim) * m.sigma * m.sigma / static_cast<double>(m.b);
  return (signal + noise) / (signal + noise / M);
}

}  // namespace
}  // namespace s2d

using s2d::Error;

namespace {
template <typename Fn>
int hguard(Fn&& fn) {
  try {
    fn();
    return S2D_OK;
  } catch (const Error& e) {
    s2d::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    s2d::set_last_error(e.what());
    return S2D_ERUNTIME;
  }
}
}  // namespace

extern "C" {

int s2d_memory_overhead(double table_size_gb, uint32_t groups, uint32_t total_gpus, double* out) {
  return hguard([&] { *out = table_size_gb * static_cast<double>(groups - 1) / static_cast<double>(total_gpus); });
}

int s2d_sync_latency(double table_size_gb, uint32_t groups, uint32_t total_gpus, double sync_bw_gbps, double* out) {
  return hguard([&] {
    const double ov = table_size_gb * static_cast<double>(groups - 1) / static_cast<double>(total_gpus);
    *out = 2.0 * ov / sync_bw_gbps;
  });
}

int s2d_qps_scaling_factor(double qps_base, double gpus_base, double qps_new, double gpus_new, double* out) {
  return hguard([&] {
    if (!(qps_base > 0) || !(gpus_base > 0) || !(qps_new > 0))
      throw Error(S2D_EINVAL, "QPS and GPU counts must be positive");
    if (!(gpus_new > gpus_base)) throw Error(S2D_EINVAL, "gpus_new must exceed gpus_base");
    *out = (qps_new / qps_base) / (gpus_new / gpus_base);
  });
}

int s2d_evaluate_ne(const double* probs, const float* labels, uint64_t n, double* ne, double* baseline_ctr) {
  return hguard([&] {
    if (n == 0 || !probs || !labels) throw Error(S2D_EINVAL, "evaluate_ne: empty or mismatched inputs");
    const double nd = static_cast<double>(n);
    double label_sum = 0.0;
    for (uint64_t i = 0; i < n; ++i) label_sum += static_cast<double>(labels[i]);
    const double p_bar = label_sum / nd;
    if (p_bar <= 0.0 || p_bar >= 1.0)
      throw Error(S2D_EINVAL, "evaluate_ne: all labels identical, baseline entropy is zero");
    double ce = 0.0;
    for (uint64_t i = 0; i < n; ++i) ce -= labels[i] > 0.5f ? std::log(probs[i]) : std::log(1.0 - probs[i]);
    ce /= nd;
    const double baseline = -(p_bar * std::log(p_bar) + (1.0 - p_bar) * std::log(1.0 - p_bar));
    *ne = ce / baseline;
    if (baseline_ctr) *baseline_ctr = p_bar;
  });
}

int s2d_closed_form_ratio(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups, double* out) {
  return hguard([&] { *out = s2d::closed_form(s2d::make_noise(mu_norm, sigma, dim, batch), groups); });
}

int s2d_recommend_c(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups, double* out) {
  return hguard([&] {
    const double r = s2d::closed_form(s2d::make_noise(mu_norm, sigma, dim, batch), groups);
    *out = std::min(r, static_cast<double>(groups));
  });
}

int s2d_estimate_increment_ratio(double mu_norm, double sigma, uint32_t dim, uint32_t batch, uint32_t groups,
                                 uint64_t trials, uint64_t seed, double* ratio, double* std_error) {
  return hguard([&] {
    const s2d::Noise m = s2d::make_noise(mu_norm, sigma, dim, batch);
    if (groups == 0) throw Error(S2D_EINVAL, "groups must be >= 1");
    if (trials == 0) throw Error(S2D_EINVAL, "trials must be >= 1");
    const double inv_b = 1.0 / static_cast<double>(m.b);
    double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
    std::vector<std::vector<double>> gm(groups, std::vector<double>(m.dim));
    for (uint64_t t = 0; t < trials; ++t) {  // moment_analysis.cpp:84-103
      s2d::HostRng rng({seed, t});
      for (uint32_t g = 0; g < groups; ++g) {
        auto& v = gm[g];
        std::fill(v.begin(), v.end(), 0.0);
        for (uint32_t s = 0; s < m.b; ++s)
          for (uint32_t j = 0; j < m.dim; ++j) v[j] += m.mu[j] + m.sigma * rng.next_normal();
        for (uint32_t j = 0; j < m.dim; ++j) v[j] *= inv_b;
      }
      const double x = s2d::norm_sq(gm[0]);
      const double y = s2d::norm_sq(s2d::pairwise_mean(gm));
      sx += x;
      sy += y;
      sxx += x * x;
      syy += y * y;
      sxy += x * y;
    }
    const double n = static_cast<double>(trials), mx = sx / n, my = sy / n, r = mx / my;
    double se = 0.0;
    if (trials > 1) {  // delta method (moment_analysis.cpp:112-121)
      const double vx = std::max(0.0, sxx / n - mx * mx), vy = std::max(0.0, syy / n - my * my);
      const double cxy = sxy / n - mx * my;
      const double rel = vx / (mx * mx) + vy / (my * my) - 2.0 * cxy / (mx * my);
      se = std::abs(r) * std::sqrt(std::max(0.0, rel) / n);
    }
    *ratio = r;
    if (std_error) *std_error = se;
  });
}

}  // extern "C"
