/* oracle/tie_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's score / rank / fit path (TIE, arXiv
 * 2604.00499, /root/reference/proj).  It is the CHECKER the parity tests, smoke() and
 * bench.py's cpu_baseline leg compare the CUDA path against; nothing in the product
 * (paper_2604_00499_b200/) may link, load or call it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the compiled
 * reference (oracle/_ref/libtie_ref.so, built from the untouched sources by
 * `make -C oracle ref`) bit-for-bit, and against the committed golden fixtures in
 * tests/golden/ (generated from that same reference by tests/golden/make_golden.py).
 *
 * Return codes mirror the reference's exception types:
 *   0 ok, 1 std::domain_error, 2 std::invalid_argument; message in tor_last_error().
 */
#ifndef TIE_ORACLE_H
#define TIE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* tor_last_error(void);

/* rng.hpp:10-16 */
uint64_t tor_mix64(uint64_t a, uint64_t b);

/* McContext::McContext, dist.cpp:122-129 (student_t draws, then ascending sort) */
int tor_mc_samples(double nu, int n, uint64_t seed, double* out);

/* dist.cpp:52-106 */
double tor_regularized_incomplete_beta(double a, double b, double x);
double tor_t_pdf(double y, double nu);
double tor_t_cdf(double y, double nu);
double tor_t_quantile(double p, double nu);

/* dist.cpp:142-147 */
int tor_sample_logt(double mu, double sigma, double nu, uint64_t n, uint64_t seed, double* out);

/* Score a batch: censored_expectation, censored_cvar, max (sim.cpp:85-94) and
 * compute_score (sched.cpp:19-26).  samples = sorted McContext set of size N.
 * E/C/S may be NULL.  *bad_index receives the first failing request (or UINT64_MAX). */
int tor_score(const double* samples, int N, double nu, const double* mu, const double* sigma,
              const double* x_max, uint64_t n, double alpha, double beta, double* E, double* C,
              double* S, uint64_t* bad_index, int threads);

/* sched.cpp:9-17 */
int tor_compute_beta(int adaptive, double beta_fixed, double beta_max, double q_sat,
                     uint64_t queue_len, double* beta);

/* WaitingQueue pop order of a static queue == lexicographic (key, id) (sched.cpp:28-31).
 * ids may be NULL (id = index). */
int tor_rank(const double* key, const uint64_t* ids, uint64_t n, uint64_t* order);

/* fit_logt_fixed_nu, fit.cpp:73-178, over P prompts x K samples (row-major). */
int tor_fit(const double* x, uint64_t P, uint64_t K, double nu, double* mu, double* sigma,
            double* ll, int32_t* iters, uint8_t* converged, uint8_t* degenerate, int threads);
double tor_logt_loglik(const double* x, uint64_t K, double mu, double sigma, double nu);
void tor_logt_loglik_grad(const double* x, uint64_t K, double mu, double sigma, double nu,
                          double* grad);

/* cmd_fit's per-prompt analysis (main.cpp:510-585): families bitmask 1 logt (fixed nu),
 * 2 logt_free_nu, 4 lognormal, 8 exponential; fits[f][10][P] (mu, sigma, nu, rate,
 * log_likelihood, iterations, converged, degenerate, ks_statistic, ks_p_value) for the
 * requested f; tail[5][P] (skewness, cv, p90/p50, p99/p50, top10_share; NaN if K < 10). */
int tor_fit_report(const double* x, uint64_t P, uint64_t K, double nu, unsigned families,
                   double* fits, double* tail, int threads);

/* gen_logt_workload, workload.cpp:50-78 (SoA view; ids are 0..n-1) */
int tor_gen_workload(uint64_t n, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                     double sg_hi, double nu, uint32_t max_tokens, double rps, double* mu,
                     double* sigma, uint32_t* max_tok, double* arrival, uint32_t* prompt_tokens,
                     uint32_t* true_len);

/* Config-3 prompt generator (main.cpp:841-845 pattern). */
int tor_gen_fit_data(uint64_t P, uint64_t K, uint64_t seed, double mu_lo, double mu_hi,
                     double sg_lo, double sg_hi, double nu, int integerise, double* x,
                     double* true_mu, double* true_sigma, int threads);

/* Scheduler over a WaitingQueue (sched.cpp:28-175), driven by a script of events:
 * op 0 = on_arrival(id, arrival_s = a, max_tokens = (uint32)b),
 * op 1 = on_prediction(id, E = a, CVaR = b),
 * op 2 = next_request() -> writes the popped id (or UINT64_MAX) to out[(*n_out)++].
 * policy 0 FCFS, 1 SEPT, 2 TIE.  Linear-scan pop_min: (key, id) order is what the heap
 * produces (sched.cpp:28-31). */
int tor_scheduler_script(int policy, int adaptive, double beta_fixed, double beta_max,
                         double q_sat, double rebuild_threshold, uint64_t n_ops,
                         const int32_t* op, const uint64_t* id, const double* a,
                         const double* b, uint64_t* out, uint64_t* n_out);

/* run_sim's precompute loop (sim.cpp:77-96): predictor 0 oracle / 1 noisy (predictor.cpp:
 * 15-31), family 0 log-t / 1 log-normal (dist.cpp:191-249), CVaR = max(CVaR, E). */
int tor_sim_scores(const double* samples, int N, double nu, const double* mu,
                   const double* sigma, const uint64_t* ids, const double* x_max, uint64_t n,
                   int predictor, double mu_sd, double ls_sd, uint64_t seed, int family,
                   double alpha, double* E, double* C);
double tor_normal_quantile(double p);

#ifdef __cplusplus
}
#endif
#endif
