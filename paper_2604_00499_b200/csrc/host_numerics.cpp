// Host numerics: request-invariant constants for the device path.  See host_numerics.hpp.
#include "host_numerics.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace tie {
namespace host {

uint64_t mix64(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9E3779B97F4A7C15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------- Sampler (rng.hpp)
double Sampler::u01() {
  // 53 random bits, centred in their ulp so the result is strictly inside (0, 1)
  const uint64_t bits = eng_() >> 11;
  return ((double)bits + 0.5) * 0x1p-53;
}

uint32_t Sampler::uniform_u32(uint32_t lo, uint32_t hi) {
  const uint64_t span = (uint64_t)(hi - lo) + 1;
  return lo + (uint32_t)(eng_() % span);
}

double Sampler::normal() {
  if (have_cached_) {
    have_cached_ = false;
    return cached_;
  }
  const double u1 = u01();
  const double u2 = u01();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 2.0 * 3.14159265358979323846 * u2;
  cached_ = radius * std::sin(angle);
  have_cached_ = true;
  return radius * std::cos(angle);
}

double Sampler::gamma(double shape, double scale) {
  if (shape < 1.0) {  // boost: G(a) = G(a+1) * U^(1/a); the uniform is drawn first
    const double u = u01();
    return gamma(shape + 1.0, scale) * std::pow(u, 1.0 / shape);
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / std::sqrt(9.0 * d);
  while (true) {
    const double x = normal();
    const double t = 1.0 + c * x;
    if (t <= 0.0) continue;
    const double v = t * t * t;
    const double u = u01();
    if (u < 1.0 - 0.0331 * x * x * x * x) return d * v * scale;
    if (std::log(u) < 0.5 * x * x + d * (1.0 - v + std::log(v))) return d * v * scale;
  }
}

double Sampler::student_t(double nu) {
  const double z = normal();
  const double chi2 = gamma(0.5 * nu, 2.0);
  return z / std::sqrt(chi2 / nu);
}

double Sampler::exponential(double rate) { return -std::log(u01()) / rate; }

std::vector<double> mc_samples(double nu, int n, uint64_t seed) {
  if (!(nu > 0.0) || !std::isfinite(nu))
    throw std::domain_error("McContext: nu must be finite and > 0");
  if (n <= 0) throw std::domain_error("McContext: n_samples must be > 0");
  Sampler s(seed);
  std::vector<double> y((size_t)n);
  for (double& v : y) v = s.student_t(nu);
  std::sort(y.begin(), y.end());
  return y;
}

// ---------------------------------------------------------------- Student-t
namespace {

// Modified Lentz evaluation of the incomplete-beta continued fraction, same operation
// order as the reference (dist.cpp:19-48) so the host constants are bit-identical.
double lentz_cf(double a, double b, double x) {
  constexpr double kTiny = 1e-300;
  constexpr double kEps = 1e-15;
  const double apb = a + b, ap1 = a + 1.0, am1 = a - 1.0;
  auto guard = [](double v) { return std::fabs(v) < kTiny ? kTiny : v; };
  double c = 1.0;
  double d = 1.0 / guard(1.0 - apb * x / ap1);
  double h = d;
  for (int m = 1; m <= 100000; ++m) {
    const int m2 = 2 * m;
    double num = m * (b - m) * x / ((am1 + m2) * (a + m2));
    d = guard(1.0 + num * d);
    c = guard(1.0 + num / c);
    d = 1.0 / d;
    h *= d * c;
    num = -(a + m) * (apb + m) * x / ((a + m2) * (ap1 + m2));
    d = guard(1.0 + num * d);
    c = guard(1.0 + num / c);
    d = 1.0 / d;
    const double ratio = d * c;
    h *= ratio;
    if (std::fabs(ratio - 1.0) < kEps) break;
  }
  return h;
}

}  // namespace

double reg_inc_beta(double a, double b, double x) {
  if (!(a > 0.0) || !(b > 0.0) || !std::isfinite(a) || !std::isfinite(b))
    throw std::domain_error("regularized_incomplete_beta: a and b must be finite and > 0");
  if (!(x >= 0.0 && x <= 1.0))
    throw std::domain_error("regularized_incomplete_beta: x must lie in [0, 1]");
  if (x == 0.0 || x == 1.0) return x;
  const double lbeta = std::lgamma(a) + std::lgamma(b) - std::lgamma(a + b);
  const double front = std::exp(a * std::log(x) + b * std::log1p(-x) - lbeta);
  if (x < (a + 1.0) / (a + b + 2.0)) return front * lentz_cf(a, b, x) / a;
  return 1.0 - front * lentz_cf(b, a, 1.0 - x) / b;
}

double t_pdf(double y, double nu) {
  if (!std::isfinite(y)) throw std::domain_error("t_pdf: y must be finite");
  if (!(nu > 0.0) || !std::isfinite(nu)) throw std::domain_error("t_pdf: nu must be finite and > 0");
  const double lnorm = std::lgamma(0.5 * (nu + 1.0)) - std::lgamma(0.5 * nu) -
                       0.5 * std::log(nu * 3.14159265358979323846);
  return std::exp(lnorm - 0.5 * (nu + 1.0) * std::log1p(y * y / nu));
}

double t_cdf(double y, double nu) {
  if (!(nu > 0.0) || !std::isfinite(nu)) throw std::domain_error("t_cdf: nu must be finite and > 0");
  if (std::isnan(y)) throw std::domain_error("t_cdf: y must not be NaN");
  if (std::isinf(y)) return y > 0 ? 1.0 : 0.0;
  const double x = nu / (y * y + nu);
  const double tail = reg_inc_beta(0.5 * nu, 0.5, x);
  return y >= 0.0 ? 1.0 - 0.5 * tail : 0.5 * tail;
}

double t_quantile(double p, double nu) {
  if (!(nu > 0.0) || !std::isfinite(nu))
    throw std::domain_error("t_quantile: nu must be finite and > 0");
  if (!(p > 0.0 && p < 1.0)) throw std::domain_error("t_quantile: p must lie in (0, 1)");
  if (p == 0.5) return 0.0;
  double lo = -1.0, hi = 1.0;
  while (t_cdf(lo, nu) > p) lo *= 2.0;
  while (t_cdf(hi, nu) < p) hi *= 2.0;
  double y = 0.0;
  for (int it = 0; it < 200 && hi - lo > 1e-14 * std::max(1.0, std::fabs(lo)); ++it) {
    y = 0.5 * (lo + hi);
    (t_cdf(y, nu) < p ? lo : hi) = y;
  }
  y = 0.5 * (lo + hi);
  for (int it = 0; it < 4; ++it) {  // Newton polish against the density
    const double f = t_cdf(y, nu) - p;
    const double dens = t_pdf(y, nu);
    if (dens <= 0.0) break;
    const double step = f / dens;
    if (!std::isfinite(step)) break;
    y -= step;
  }
  return y;
}

double normal_quantile(double p) {
  if (!(p > 0.0 && p < 1.0)) throw std::domain_error("normal_quantile: p must lie in (0, 1)");
  // Acklam's coefficients (central region a/b, tails c/d)
  static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                              -2.759285104469687e+02, 1.383577518672690e+02,
                              -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                              -1.556989798598866e+02, 6.680131188771972e+01,
                              -1.328068155288572e+01};
  static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                              -2.400758277161838e+00, -2.549732539343734e+00,
                              4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                              2.445134137142996e+00, 3.754408661907416e+00};
  auto tail = [&](double q) {
    return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  };
  constexpr double kLow = 0.02425;
  double z;
  if (p < kLow) {
    z = tail(std::sqrt(-2.0 * std::log(p)));
  } else if (p <= 1.0 - kLow) {
    const double q = p - 0.5, r = q * q;
    z = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    z = -tail(std::sqrt(-2.0 * std::log1p(-p)));
  }
  // one Newton-type (Halley) polish against the exact CDF
  const double e = 0.5 * std::erfc(-z * 0.7071067811865475244) - p;
  const double u = e * std::sqrt(2.0 * 3.14159265358979323846) * std::exp(0.5 * z * z);
  return z - u / (1.0 + 0.5 * z * u);
}

std::vector<double> sample_logt(double mu, double sigma, double nu, size_t n, uint64_t seed) {
  if (sigma < 1e-9) sigma = 1e-9;
  Sampler s(seed);
  std::vector<double> out(n);
  for (double& v : out) v = std::exp(mu + sigma * s.student_t(nu));
  return out;
}

Workload gen_logt_workload(size_t n, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                           double sg_hi, double nu, uint32_t prompt_lo, uint32_t prompt_hi,
                           uint32_t max_tokens, double rps) {
  if (!(mu_lo <= mu_hi)) throw std::domain_error("gen_logt_workload: bad mu_range");
  if (!(sg_lo > 0.0) || !(sg_lo <= sg_hi))
    throw std::domain_error("gen_logt_workload: bad sigma_range");
  if (!(nu > 0.0)) throw std::domain_error("gen_logt_workload: nu must be > 0");
  if (prompt_lo < 1 || prompt_lo > prompt_hi)
    throw std::domain_error("gen_logt_workload: bad prompt_range");
  if (max_tokens < 1) throw std::domain_error("gen_logt_workload: max_tokens must be >= 1");
  if (!(rps > 0.0) || !std::isfinite(rps))
    throw std::domain_error("poisson_arrivals: rps must be finite and > 0");
  Workload w;
  w.mu.resize(n);
  w.sigma.resize(n);
  w.arrival.resize(n);
  w.max_tokens.assign(n, max_tokens);
  w.prompt_tokens.resize(n);
  w.true_len.resize(n);
  Sampler arrivals(mix64(seed, 1));
  double t = 0.0;
  for (size_t i = 0; i < n; ++i) w.arrival[i] = (t += arrivals.exponential(rps));
  Sampler s(mix64(seed, 2));
  for (size_t i = 0; i < n; ++i) {
    w.mu[i] = s.uniform(mu_lo, mu_hi);
    w.sigma[i] = s.uniform(sg_lo, sg_hi);
    w.prompt_tokens[i] = s.uniform_u32(prompt_lo, prompt_hi);
    const double ln_len = w.mu[i] + w.sigma[i] * s.student_t(nu);
    double len = ln_len > 22.0 ? 4294967295.0 : std::round(std::exp(ln_len));
    len = std::min(std::max(len, 1.0), 4294967295.0);
    w.true_len[i] = (uint32_t)len;
  }
  return w;
}

void make_cf_table(double p, double q, CfTable* out) {
  out->d1 = -(p + q) / (p + 1.0);
  for (int m = 1; m <= CfTable::kTerms; ++m) {
    const double m2 = 2.0 * m;
    out->even[m - 1] = m * (q - m) / ((p - 1.0 + m2) * (p + m2));
    out->odd[m - 1] = -(p + m) * (p + q + m) / ((p + m2) * (p + 1.0 + m2));
  }
}

}  // namespace host
}  // namespace tie
