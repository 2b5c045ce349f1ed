// include/tiesched_b200.hpp -- C++ host API of the B200 TIE path (namespace tie).
//
// Same names, argument meaning and exception behaviour as the reference headers
// (proj/include/tiesched/dist.hpp, sched.hpp, fit.hpp), so reference callers recompile
// unchanged; every per-item call is a batch of one on the GPU, and the batched entry
// points below are what callers with queues should use.  Built on the C-ABI
// (include/tie_cuda.h) -- there is no CPU implementation of the hot path behind it.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

#include "tie_cuda.h"

namespace tie {

// ------------------------------------------------------------------ dist.hpp:11-45
struct LogTParams {
  double mu;
  double sigma;
  double nu;
  bool sigma_clamped = false;
  LogTParams(double mu_, double sigma_, double nu_);  // throws std::domain_error
};

struct CensoredLogT {
  LogTParams dist;
  double x_max;
  CensoredLogT(LogTParams d, double x_max_);  // throws std::domain_error
};

// The shared sorted standard-t sample set, generated on the host exactly as the reference
// does and resident on the GPU together with its score tables.
class McContext {
 public:
  explicit McContext(double nu_, int n_samples = kDefaultSamples, uint64_t seed_ = kDefaultSeed,
                     int device = 0);
  McContext(const double* sorted_samples, int n_samples, double nu_, int device = 0);
  double nu;
  uint64_t seed;
  const std::vector<double>& samples() const { return samples_; }
  size_t n_samples() const { return samples_.size(); }
  tie_ctx* handle() const { return ctx_.get(); }

  static constexpr int kDefaultSamples = 10000;
  static constexpr uint64_t kDefaultSeed = 12;

 private:
  std::vector<double> samples_;
  std::shared_ptr<tie_ctx> ctx_;
};

double t_pdf(double y, double nu);
double t_cdf(double y, double nu);
double t_quantile(double p, double nu);
std::vector<double> sample_logt(const LogTParams& p, size_t n, uint64_t seed);

double censored_expectation(const CensoredLogT& cl, const McContext& mc);
double censored_cvar(const CensoredLogT& cl, const McContext& mc, double alpha);

// ------------------------------------------------------------------ sched.hpp:13-30
enum class Policy { FCFS, SEPT, TIE };
enum class BetaMode { Fixed, AdaptiveLinear };

struct ScoreConfig {
  double alpha = 0.9;
  BetaMode beta_mode = BetaMode::AdaptiveLinear;
  double beta_fixed = 0.1;
  double beta_max = 0.5;
  double q_sat = 128.0;
  double rebuild_threshold = 0.1;
};

double compute_beta(const ScoreConfig& cfg, size_t queue_len);
double compute_score(double expectation, double cvar, double beta);

// ------------------------------------------------------------------ batched (new)
// HOST buffers.  Scores every request of a queue with beta = compute_beta(cfg,
// queue_len_for_beta) -- pass the GLOBAL queue length when the queue is sharded.
// E / cvar / score may be null.  exact=true selects the per-term summation path.
void score_batch(const double* mu, const double* sigma, const double* x_max, size_t n,
                 const McContext& mc, const ScoreConfig& cfg, size_t queue_len_for_beta,
                 double* E, double* cvar, double* score, bool exact = false);
// Dispatch order by (key asc, id asc); ids == nullptr means id = index.
void rank(const double* key, size_t n, uint64_t* order, const uint64_t* ids = nullptr,
          const McContext* mc = nullptr);
// Score + rank in one device pass (ids = index).
void score_rank(const double* mu, const double* sigma, const uint32_t* max_tokens, size_t n,
                const McContext& mc, const ScoreConfig& cfg, size_t queue_len_for_beta,
                double* score, uint64_t* order, bool exact = false);

// ------------------------------------------------------------------ fit.hpp:11-35
enum class FitFamily { LogTFixedNu, LogTFreeNu, LogNormal, Exponential };

struct FitResult {
  FitFamily family = FitFamily::LogTFixedNu;
  double mu = 0.0;
  double sigma = 0.0;
  double nu = 0.0;
  double rate = 0.0;
  double log_likelihood = 0.0;
  bool converged = false;
  int iterations = 0;
  bool degenerate = false;
};

double logt_loglik(const std::vector<double>& x, double mu, double sigma, double nu);
std::array<double, 2> logt_loglik_grad(const std::vector<double>& x, double mu, double sigma,
                                       double nu);
FitResult fit_logt_fixed_nu(const std::vector<double>& x, double nu = 3.5);
// P prompts x K samples, row-major host buffer.
std::vector<FitResult> fit_logt_fixed_nu_batch(const double* x, size_t P, size_t K,
                                               double nu = 3.5);

// ------------------------------------------------------------------ synthetic inputs
// gen_logt_workload (workload.cpp:50-78) in SoA form (ids are 0..n-1); any output but
// mu/sigma/max_tokens may be null.
void gen_logt_workload_soa(size_t n, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                           double sg_hi, double nu, uint32_t prompt_lo, uint32_t prompt_hi,
                           uint32_t max_tokens, double rps, double* mu, double* sigma,
                           uint32_t* max_tok, double* arrival, uint32_t* prompt_tokens,
                           uint32_t* true_len);
// Config-3 prompts: truths from Sampler(seed), K draws of
// sample_logt(.., mix64(seed, p)), integerised max(1, llround(x)) (u32 ceiling).
void gen_fit_data(size_t P, size_t K, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                  double sg_hi, double nu, bool integerise, double* x, double* true_mu,
                  double* true_sigma, int threads = 0);

// The default device context used by the per-item fit / loglik calls (device 0, nu 3.5).
tie_ctx* default_context();

}  // namespace tie
