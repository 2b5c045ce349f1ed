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
#include <optional>
#include <string>
#include <unordered_map>
#include <utility>
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

// The shared sorted standard-t sample set (dist.hpp:29-45): generated on the host exactly as
// the reference does (`samples`, public as in the reference) and uploaded once to the GPU,
// where it lives with its score tables.  The device copy is taken at construction; copies of
// a McContext share it.
struct McContext {
  double nu;
  uint64_t seed;
  std::vector<double> samples;  // sorted ascending

  explicit McContext(double nu_, int n_samples = kDefaultSamples, uint64_t seed_ = kDefaultSeed,
                     int device = 0);
  McContext(const double* sorted_samples, int n_samples, double nu_, int device = 0);
  size_t n_samples() const { return samples.size(); }
  tie_ctx* handle() const { return ctx_.get(); }

  static constexpr int kDefaultSamples = 10000;
  static constexpr uint64_t kDefaultSeed = 12;

 private:
  std::shared_ptr<tie_ctx> ctx_;
};

double t_pdf(double y, double nu);
double t_cdf(double y, double nu);
double t_quantile(double p, double nu);
double regularized_incomplete_beta(double a, double b, double x);  // GPU (tie_eval_host)
double logt_pdf(double x, const LogTParams& p);                     // GPU
double logt_cdf(double x, const LogTParams& p);                     // GPU
std::vector<double> sample_logt(const LogTParams& p, size_t n, uint64_t seed);
// Psi(y) = E[X 1{Y <= y}] over the shared sample set (dist.cpp:149-156), GPU
double psi(double y, const LogTParams& p, const McContext& mc);

double censored_expectation(const CensoredLogT& cl, const McContext& mc);
double censored_cvar(const CensoredLogT& cl, const McContext& mc, double alpha);

double normal_cdf(double z);       // GPU
double normal_quantile(double p);  // GPU
double lognormal_censored_expectation(double mu, double sigma, double x_max);           // GPU
double lognormal_censored_cvar(double mu, double sigma, double x_max, double alpha);   // GPU

// Batched form of the per-item functions above: op is a TIE_EVAL_* code (tie_cuda.h);
// a / b / c are the op's per-item arguments (b, c unused by one-argument ops), param its
// scalar (nu or alpha).  mc: the sample set for TIE_EVAL_PSI (else ignored; may be null).
std::vector<double> eval_batch(int op, const double* a, const double* b, const double* c,
                               size_t n, double param, const McContext* mc = nullptr);

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

// ------------------------------------------------------------------ workload.hpp:11-56
struct Request {
  uint64_t id;
  double arrival_s;
  uint32_t prompt_tokens;
  uint32_t true_output_tokens;
  uint32_t max_tokens;
  std::optional<double> true_mu;
  std::optional<double> true_sigma;
};

struct WorkloadSpec {
  size_t n_requests = 2000;
  double rps = 100.0;
  std::pair<double, double> mu_range = {3.0, 5.0};
  std::pair<double, double> sigma_range = {0.5, 1.2};
  double nu = 3.5;
  std::pair<uint32_t, uint32_t> prompt_range = {64, 512};
  uint32_t max_tokens = 2048;
};

// gen_logt_workload / poisson_arrivals (workload.cpp:37-78): the same draws, host-side input
// generation (bit-identical to the reference's mt19937_64 streams)
std::vector<Request> gen_logt_workload(const WorkloadSpec& spec, uint64_t seed);
std::vector<double> poisson_arrivals(double rps, size_t n, uint64_t seed);

// ------------------------------------------------------------------ sched.hpp:32-90
struct QueueEntry {
  uint64_t req_id;
  double key;
  bool predicted = false;
  double expectation = 0.0;
  double cvar = 0.0;
  double beta_at_update = 0.0;
};

// The reference's indexed min-heap by (key, req_id), GPU-resident: the keys live on the
// device behind a block-min index (a pop is an argmin over block minima, not a sift), and
// the ids -> slot index is on the host, so every call is one small device round trip.  The
// per-item API is the reference's; the *_batch calls move whole batches per round trip.
// entries() / non-const at() hand out host copies: edits reach the device at the next
// update() of that id (at()) or rebuild() (entries() / at()), as the reference requires
// key edits to be followed by rebuild().  Entries come in slot (arrival) order, not heap order.
class WaitingQueue {
 public:
  explicit WaitingQueue(const McContext* mc = nullptr, size_t initial_capacity = 1024);
  ~WaitingQueue();
  WaitingQueue(const WaitingQueue&) = delete;
  WaitingQueue& operator=(const WaitingQueue&) = delete;
  WaitingQueue(WaitingQueue&&) noexcept;
  WaitingQueue& operator=(WaitingQueue&&) noexcept;

  void push(const QueueEntry& e);
  void update(uint64_t req_id, double key);
  std::optional<QueueEntry> pop_min();
  bool contains(uint64_t req_id) const;
  size_t size() const;
  bool empty() const { return size() == 0; }
  const QueueEntry& at(uint64_t req_id) const;
  QueueEntry& at(uint64_t req_id);
  const std::vector<QueueEntry>& entries() const;
  std::vector<QueueEntry>& entries();
  void rebuild();
  bool validate() const;

  void push_batch(const QueueEntry* e, size_t m);
  void update_batch(const uint64_t* ids, const double* keys, size_t m);
  std::vector<QueueEntry> pop_batch(size_t max_pops);
  tie_queue* handle() const { return q_; }

 private:
  friend class Scheduler;
  WaitingQueue(tie_queue* view_of);  // read-only view of a Scheduler's queue
  void flush() const;                // write back handed-out edits
  tie_queue* q_ = nullptr;
  bool owner_ = true;
  mutable std::vector<QueueEntry> cache_;           // entries() / at() copies
  mutable std::unordered_map<uint64_t, size_t> cache_pos_;
  mutable bool all_out_ = false;                    // entries() handed out mutably
  mutable std::vector<uint64_t> dirty_;             // ids handed out by non-const at()
};

// Policy wrapper (sched.hpp:70-90) over the GPU queue: the same keys, beta, drift rebuilds
// and pop order as the reference Scheduler; the batch calls apply many events per device
// round trip with identical results to the per-item sequence.
class Scheduler {
 public:
  Scheduler(Policy policy, ScoreConfig cfg, const McContext* mc = nullptr,
            size_t initial_capacity = 1024);
  ~Scheduler();
  Scheduler(const Scheduler&) = delete;
  Scheduler& operator=(const Scheduler&) = delete;
  Scheduler(Scheduler&& o) noexcept;
  Scheduler& operator=(Scheduler&& o) noexcept;

  void on_arrival(const Request& req);
  void on_prediction(uint64_t req_id, double expectation, double cvar);
  bool rebuild_if_drifted();
  std::optional<uint64_t> next_request();
  bool waiting_on(uint64_t req_id) const;
  size_t waiting() const;
  double current_beta() const { return compute_beta(cfg_, waiting()); }
  const WaitingQueue& queue() const { return view_; }
  Policy policy() const { return policy_; }

  // batches: on_arrival x m; on_prediction x m; next_request() up to k times
  void on_arrival_batch(const Request* reqs, size_t m);
  void on_prediction_batch(const uint64_t* ids, const double* expectation, const double* cvar,
                           size_t m);
  std::vector<uint64_t> next_requests(size_t k);
  // on_arrival x n_arr, on_prediction x n_pred, next_request() up to max_pops times, in that
  // order, with one device round trip (tie_queue_step_ec)
  std::vector<uint64_t> step(const Request* arrivals, size_t n_arr, const uint64_t* pred_ids,
                             const double* expectation, const double* cvar, size_t n_pred,
                             size_t max_pops);
  // runs r of (arrivals [arr_end[r-1], arr_end[r]), predictions [pred_end[r-1], pred_end[r]))
  // in order, then next_request() up to max_pops times: one round trip (tie_queue_step_ec_runs)
  std::vector<uint64_t> step_runs(const Request* arrivals, const uint64_t* arr_end,
                                  const uint64_t* pred_ids, const double* expectation,
                                  const double* cvar, const uint64_t* pred_end, size_t n_runs,
                                  size_t max_pops);
  tie_queue* handle() const { return q_; }

 private:
  Policy policy_;
  ScoreConfig cfg_;
  tie_queue* q_ = nullptr;
  WaitingQueue view_;
};

// ------------------------------------------------------------------ predictor.hpp:11-53
struct PredictedDist {
  double mu_hat;
  double sigma_hat;
};
struct NoiseSpec {
  double mu_sd = 0.0;
  double log_sigma_sd = 0.0;
};
struct BatcherConfig {
  double timeout_s = 0.003;
  int max_batch = 32;
  double latency_base_s = 0.002;
  double latency_per_item_s = 0.0001;
};
PredictedDist oracle_predict(const Request& req);
PredictedDist noisy_predict(const Request& req, const NoiseSpec& noise, uint64_t seed);
double point_predict(const Request& req, const NoiseSpec& noise, uint64_t seed,
                     const McContext& mc);
struct Submission {
  uint64_t req_id;
  double submit_s;
};
struct PredictionReady {
  uint64_t req_id;
  double ready_s;
};
std::vector<PredictionReady> batch_schedule(const std::vector<Submission>& submissions,
                                            const BatcherConfig& cfg);

// ------------------------------------------------------------------ sim.hpp:15-97
struct EngineConfig {
  int batch_slots = 8;
  double c0 = 0.02;
  double c1 = 0.002;
  double c2 = 0.0001;
};
enum class PredictorKind { None, Oracle, Noisy };
enum class ScoreFamily { LogT, LogNormal };
struct PredictorConfig {
  PredictorKind kind = PredictorKind::Oracle;
  ScoreFamily family = ScoreFamily::LogT;
  NoiseSpec noise;
  bool batched = true;
  BatcherConfig batcher;
  double nu = 3.5;
  int mc_samples = McContext::kDefaultSamples;
  uint64_t mc_seed = McContext::kDefaultSeed;
};
struct RequestEvent {
  uint64_t req_id;
  double arrival_s;
  std::optional<double> predict_ready_s;
  double admit_s;
  double first_token_s;
  double completion_s;
  uint32_t emitted_tokens;
};
struct Metrics {
  double ttft_avg = 0.0;
  double ttft_p90 = 0.0;
  double ptla_avg = 0.0;
  double ptla_p90 = 0.0;
  std::vector<std::pair<uint64_t, double>> time_at_k;
  std::vector<std::pair<double, uint64_t>> throughput_at_w;
};
struct HeatmapSpec {
  int time_bins = 24;
  int len_bins = 24;
  double time_max = 240.0;
  double len_max = 512.0;
};
struct Heatmap {
  HeatmapSpec spec;
  std::vector<uint64_t> counts;
};
struct SimReport {
  uint64_t seed = 0;
  Policy policy = Policy::FCFS;
  std::vector<RequestEvent> events;
  Metrics metrics;
};

// run_sim (sim.cpp:39-185): the scoring precompute runs as one GPU batch (tie_sim_scores),
// the waiting queue is the GPU Scheduler above, and the event loop applies each run of
// same-kind events (arrivals / predictions) and each admission as one device round trip.
SimReport run_sim(const std::vector<Request>& workload, Policy policy,
                  const ScoreConfig& score_cfg, const EngineConfig& engine_cfg,
                  const PredictorConfig& predictor_cfg, uint64_t seed,
                  const std::vector<uint64_t>& ks = {}, const std::vector<double>& ws = {},
                  int device = 0);
Metrics summarize(const std::vector<RequestEvent>& events, const std::vector<uint64_t>& ks,
                  const std::vector<double>& ws);
Heatmap heatmap(const std::vector<RequestEvent>& events, const HeatmapSpec& spec);

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
