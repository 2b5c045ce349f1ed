// C++ host API (include/tiesched_b200.hpp): the reference's tie:: names over the C-ABI.
// Per-item calls run as GPU batches of one; C-ABI error codes become the reference's
// exception types (std::domain_error / std::invalid_argument / std::runtime_error).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <thread>
#include <mutex>
#include <stdexcept>
#include <string>

#include "host_numerics.hpp"
#include "tiesched_b200.hpp"

namespace tie {

namespace {

void throw_code(int rc) {
  if (rc == TIE_OK) return;
  const std::string msg = tie_last_error();
  if (rc == TIE_EDOMAIN) throw std::domain_error(msg);
  if (rc == TIE_EINVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

constexpr double kSigmaFloor = 1e-9;  // dist.cpp:12

}  // namespace

LogTParams::LogTParams(double mu_, double sigma_, double nu_) : mu(mu_), sigma(sigma_), nu(nu_) {
  if (!std::isfinite(mu)) throw std::domain_error("LogTParams: mu must be finite");
  if (!(sigma > 0.0) || !std::isfinite(sigma))
    throw std::domain_error("LogTParams: sigma must be finite and > 0");
  if (!(nu > 0.0) || !std::isfinite(nu))
    throw std::domain_error("LogTParams: nu must be finite and > 0");
  if (sigma < kSigmaFloor) {
    sigma = kSigmaFloor;
    sigma_clamped = true;
  }
}

CensoredLogT::CensoredLogT(LogTParams d, double x_max_) : dist(d), x_max(x_max_) {
  if (!(x_max > 0.0) || !std::isfinite(x_max))
    throw std::domain_error("CensoredLogT: x_max must be finite and > 0");
}

McContext::McContext(double nu_, int n_samples, uint64_t seed_, int device)
    : nu(nu_), seed(seed_) {
  samples = host::mc_samples(nu, n_samples, seed);  // throws std::domain_error
  tie_ctx* raw = nullptr;
  throw_code(tie_ctx_create(device, samples.data(), n_samples, nu, 0.0, &raw));
  ctx_.reset(raw, tie_ctx_destroy);
}

McContext::McContext(const double* sorted_samples, int n_samples, double nu_, int device)
    : nu(nu_), seed(0) {
  tie_ctx* raw = nullptr;
  throw_code(tie_ctx_create(device, sorted_samples, n_samples, nu, 0.0, &raw));
  ctx_.reset(raw, tie_ctx_destroy);
  samples.assign(sorted_samples, sorted_samples + n_samples);
}

double t_pdf(double y, double nu) { return host::t_pdf(y, nu); }
double t_cdf(double y, double nu) { return host::t_cdf(y, nu); }
double t_quantile(double p, double nu) { return host::t_quantile(p, nu); }

std::vector<double> sample_logt(const LogTParams& p, size_t n, uint64_t seed) {
  return host::sample_logt(p.mu, p.sigma, p.nu, n, seed);
}

std::vector<double> eval_batch(int op, const double* a, const double* b, const double* c,
                               size_t n, double param, const McContext* mc) {
  std::vector<double> out(n);
  tie_ctx* ctx = mc ? mc->handle() : default_context();
  throw_code(tie_eval_host(ctx, op, a, b, c, n, param, out.data()));
  return out;
}

namespace {

double eval1(int op, double a, double b, double c, double param, const McContext* mc = nullptr) {
  return eval_batch(op, &a, &b, &c, 1, param, mc)[0];
}

}  // namespace

double regularized_incomplete_beta(double a, double b, double x) {
  return eval1(TIE_EVAL_INCBETA, a, b, x, 0.0);
}
double logt_pdf(double x, const LogTParams& p) {
  return eval1(TIE_EVAL_LOGT_PDF, x, p.mu, p.sigma, p.nu);
}
double logt_cdf(double x, const LogTParams& p) {
  return eval1(TIE_EVAL_LOGT_CDF, x, p.mu, p.sigma, p.nu);
}
double psi(double y, const LogTParams& p, const McContext& mc) {
  return eval1(TIE_EVAL_PSI, y, p.mu, p.sigma, p.nu, &mc);
}
double normal_cdf(double z) { return eval1(TIE_EVAL_NORMAL_CDF, z, 0.0, 0.0, 0.0); }
double normal_quantile(double p) { return eval1(TIE_EVAL_NORMAL_QUANTILE, p, 0.0, 0.0, 0.0); }
double lognormal_censored_expectation(double mu, double sigma, double x_max) {
  return eval1(TIE_EVAL_LOGNORMAL_E, mu, sigma, x_max, 0.0);
}
double lognormal_censored_cvar(double mu, double sigma, double x_max, double alpha) {
  return eval1(TIE_EVAL_LOGNORMAL_CVAR, mu, sigma, x_max, alpha);
}

std::vector<double> poisson_arrivals(double rps, size_t n, uint64_t seed) {
  if (!(rps > 0.0) || !std::isfinite(rps))
    throw std::domain_error("poisson_arrivals: rps must be finite and > 0");
  host::Sampler r(seed);
  std::vector<double> out(n);
  double t = 0.0;
  for (double& a : out) a = (t += r.exponential(rps));
  return out;
}

std::vector<Request> gen_logt_workload(const WorkloadSpec& spec, uint64_t seed) {
  const host::Workload w = host::gen_logt_workload(
      spec.n_requests, seed, spec.mu_range.first, spec.mu_range.second, spec.sigma_range.first,
      spec.sigma_range.second, spec.nu, spec.prompt_range.first, spec.prompt_range.second,
      spec.max_tokens, spec.rps);
  std::vector<Request> out(spec.n_requests);
  for (size_t i = 0; i < out.size(); ++i) {
    Request& r = out[i];
    r.id = i;
    r.arrival_s = w.arrival[i];
    r.prompt_tokens = w.prompt_tokens[i];
    r.true_output_tokens = w.true_len[i];
    r.max_tokens = w.max_tokens[i];
    r.true_mu = w.mu[i];
    r.true_sigma = w.sigma[i];
  }
  return out;
}

namespace {

void check_nu(const CensoredLogT& cl, const McContext& mc) {
  if (cl.dist.nu != mc.nu)  // psi (dist.cpp:150)
    throw std::invalid_argument("psi: McContext nu does not match distribution nu");
}

}  // namespace

double censored_expectation(const CensoredLogT& cl, const McContext& mc) {
  check_nu(cl, mc);
  double E = 0.0;
  const double mu = cl.dist.mu, sg = cl.dist.sigma, xm = cl.x_max;
  throw_code(tie_score_host(mc.handle(), &mu, &sg, &xm, 1, 0.0, 0.0, &E, nullptr, nullptr,
                            TIE_SCORE_RAW));
  return E;
}

double censored_cvar(const CensoredLogT& cl, const McContext& mc, double alpha) {
  if (!(alpha >= 0.0 && alpha < 1.0))
    throw std::domain_error("censored_cvar: alpha must lie in [0, 1)");
  check_nu(cl, mc);
  double C = 0.0;
  const double mu = cl.dist.mu, sg = cl.dist.sigma, xm = cl.x_max;
  throw_code(tie_score_host(mc.handle(), &mu, &sg, &xm, 1, alpha, 0.0, nullptr, &C, nullptr,
                            TIE_SCORE_RAW));
  return C;
}

double compute_beta(const ScoreConfig& cfg, size_t queue_len) {
  double b = 0.0;
  throw_code(tie_compute_beta(cfg.beta_mode == BetaMode::AdaptiveLinear, cfg.beta_fixed,
                              cfg.beta_max, cfg.q_sat, queue_len, &b));
  return b;
}

double compute_score(double expectation, double cvar, double beta) {
  if (!std::isfinite(expectation) || !std::isfinite(cvar) || !std::isfinite(beta))
    throw std::domain_error("compute_score: arguments must be finite");
  if (!(expectation > 0.0)) throw std::domain_error("compute_score: expectation must be > 0");
  if (cvar < expectation)
    throw std::invalid_argument("compute_score: cvar below expectation violates the invariant");
  return expectation + beta * cvar;
}

void score_batch(const double* mu, const double* sigma, const double* x_max, size_t n,
                 const McContext& mc, const ScoreConfig& cfg, size_t queue_len_for_beta,
                 double* E, double* cvar, double* score, bool exact) {
  const double beta = compute_beta(cfg, queue_len_for_beta);
  throw_code(tie_score_host(mc.handle(), mu, sigma, x_max, n, cfg.alpha, beta, E, cvar, score,
                            exact ? TIE_SCORE_EXACT : TIE_SCORE_MOMENT));
}

void rank(const double* key, size_t n, uint64_t* order, const uint64_t* ids,
          const McContext* mc) {
  tie_ctx* ctx = mc ? mc->handle() : default_context();
  throw_code(tie_rank_host(ctx, key, ids, n, order));
}

void score_rank(const double* mu, const double* sigma, const uint32_t* max_tokens, size_t n,
                const McContext& mc, const ScoreConfig& cfg, size_t queue_len_for_beta,
                double* score, uint64_t* order, bool exact) {
  const double beta = compute_beta(cfg, queue_len_for_beta);
  throw_code(tie_score_rank_host(mc.handle(), mu, sigma, max_tokens, n, cfg.alpha, beta, score,
                                 order, exact ? TIE_SCORE_EXACT : TIE_SCORE_MOMENT));
}

tie_ctx* default_context() {
  static std::once_flag once;
  static McContext* mc = nullptr;
  std::call_once(once, [] { mc = new McContext(3.5); });
  return mc->handle();
}

namespace {

void check_samples(const std::vector<double>& x, size_t min_n, const char* who) {  // fit.cpp:18
  if (x.size() < min_n)
    throw std::invalid_argument(std::string(who) + ": need at least " + std::to_string(min_n) +
                                " samples, got " + std::to_string(x.size()));
  for (double v : x)
    if (!(v > 0.0) || !std::isfinite(v))
      throw std::domain_error(std::string(who) + ": samples must be finite and > 0");
}

// one parameter point through the device loglik kernel (tie_logt_loglik)
void loglik_dev(const std::vector<double>& x, double mu, double sigma, double nu, double* ll,
                double* grad) {
  tie_ctx* ctx = default_context();
  std::vector<double> buf(x);
  buf.push_back(mu);
  buf.push_back(sigma);
  // host-staged call: x, mu, sigma in; ll / grad out
  const int rc = [&]() -> int {
    double* d = nullptr;
    const size_t K = x.size();
    if (cudaMalloc(&d, sizeof(double) * (K + 5)) != cudaSuccess) return TIE_ECUDA;
    cudaMemcpy(d, buf.data(), sizeof(double) * (K + 2), cudaMemcpyHostToDevice);
    int r = tie_logt_loglik(ctx, d, K, d + K, d + K + 1, 1, nu, ll ? d + K + 2 : nullptr,
                            grad ? d + K + 3 : nullptr, nullptr);
    if (r == TIE_OK) r = tie_sync(ctx, nullptr);
    double out[3] = {0, 0, 0};
    cudaMemcpy(out, d + K + 2, sizeof(out), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (ll) *ll = out[0];
    if (grad) {
      grad[0] = out[1];
      grad[1] = out[2];
    }
    return r;
  }();
  throw_code(rc);
}

}  // namespace

double logt_loglik(const std::vector<double>& x, double mu, double sigma, double nu) {
  check_samples(x, 1, "logt_loglik");
  if (!(sigma > 0.0) || !(nu > 0.0))
    throw std::domain_error("logt_loglik: sigma and nu must be > 0");
  double ll = 0.0;
  loglik_dev(x, mu, sigma, nu, &ll, nullptr);
  return ll;
}

std::array<double, 2> logt_loglik_grad(const std::vector<double>& x, double mu, double sigma,
                                       double nu) {
  check_samples(x, 1, "logt_loglik_grad");
  if (!(sigma > 0.0) || !(nu > 0.0))
    throw std::domain_error("logt_loglik_grad: sigma and nu must be > 0");
  double g[2] = {0, 0};
  loglik_dev(x, mu, sigma, nu, nullptr, g);
  return {g[0], g[1]};
}

std::vector<FitResult> fit_logt_fixed_nu_batch(const double* x, size_t P, size_t K, double nu) {
  std::vector<double> mu(P), sg(P), ll(P);
  std::vector<int32_t> it(P);
  std::vector<uint8_t> cv(P), dg(P);
  throw_code(tie_fit_host(default_context(), x, P, K, nu, mu.data(), sg.data(), ll.data(),
                          it.data(), cv.data(), dg.data()));
  std::vector<FitResult> out(P);
  for (size_t p = 0; p < P; ++p) {
    FitResult& r = out[p];
    r.family = FitFamily::LogTFixedNu;
    r.mu = mu[p];
    r.sigma = sg[p];
    r.nu = nu;
    r.log_likelihood = ll[p];
    r.converged = cv[p] != 0;
    r.iterations = it[p];
    r.degenerate = dg[p] != 0;
  }
  return out;
}

FitResult fit_logt_fixed_nu(const std::vector<double>& x, double nu) {
  check_samples(x, 3, "fit_logt_fixed_nu");
  if (!(nu > 0.0) || !std::isfinite(nu))
    throw std::domain_error("fit_logt_fixed_nu: nu must be finite and > 0");
  return fit_logt_fixed_nu_batch(x.data(), 1, x.size(), nu)[0];
}

void gen_logt_workload_soa(size_t n, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                           double sg_hi, double nu, uint32_t prompt_lo, uint32_t prompt_hi,
                           uint32_t max_tokens, double rps, double* mu, double* sigma,
                           uint32_t* max_tok, double* arrival, uint32_t* prompt_tokens,
                           uint32_t* true_len) {
  const host::Workload w = host::gen_logt_workload(n, seed, mu_lo, mu_hi, sg_lo, sg_hi, nu,
                                                   prompt_lo, prompt_hi, max_tokens, rps);
  std::copy(w.mu.begin(), w.mu.end(), mu);
  std::copy(w.sigma.begin(), w.sigma.end(), sigma);
  std::copy(w.max_tokens.begin(), w.max_tokens.end(), max_tok);
  if (arrival) std::copy(w.arrival.begin(), w.arrival.end(), arrival);
  if (prompt_tokens) std::copy(w.prompt_tokens.begin(), w.prompt_tokens.end(), prompt_tokens);
  if (true_len) std::copy(w.true_len.begin(), w.true_len.end(), true_len);
}

void gen_fit_data(size_t P, size_t K, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                  double sg_hi, double nu, bool integerise, double* x, double* true_mu,
                  double* true_sigma, int threads) {
  std::vector<double> m(P), s(P);
  host::Sampler truth(seed);
  for (size_t p = 0; p < P; ++p) {
    m[p] = truth.uniform(mu_lo, mu_hi);
    s[p] = truth.uniform(sg_lo, sg_hi);
  }
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  auto body = [&](size_t lo, size_t hi) {
    for (size_t p = lo; p < hi; ++p) {
      const std::vector<double> v = host::sample_logt(m[p], s[p], nu, K, host::mix64(seed, p));
      for (size_t k = 0; k < K; ++k) {
        double val = v[k];
        if (integerise)
          val = val >= 4294967295.0 ? 4294967295.0
                                    : (double)std::max(1LL, std::llround(val));
        x[p * K + k] = val;
      }
    }
  };
  std::vector<std::thread> pool;
  const size_t per = (P + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const size_t lo = std::min(P, t * per), hi = std::min(P, lo + per);
    if (lo < hi) pool.emplace_back(body, lo, hi);
  }
  for (auto& th : pool) th.join();
  if (true_mu) std::copy(m.begin(), m.end(), true_mu);
  if (true_sigma) std::copy(s.begin(), s.end(), true_sigma);
}

}  // namespace tie
