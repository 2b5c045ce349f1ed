// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (never the product path).
//
// A C-ABI shim over the UNTOUCHED reference library (/root/reference/proj/src/*.cpp,
// compiled where it lies by oracle/Makefile into oracle/_ref/libtie_ref.so).  It lets
// the tests, the golden-fixture generator and bench.py's cpu_baseline / --impl reference
// legs drive the reference's own functions in bulk:
//
//   score  : censored_expectation + censored_cvar + max + compute_score, exactly as the
//            reference's run_sim precompute loop does it (proj/src/sim.cpp:77-96,
//            proj/src/sched.cpp:19-26), fanned out over host threads (pure functions,
//            shared const McContext -- SPEC.md:139).
//   rank   : WaitingQueue push x n then pop_min until empty (proj/src/sched.cpp:28-94).
//   fit    : fit_logt_fixed_nu per prompt (proj/src/fit.cpp:73-178), threaded.
//   inputs : gen_logt_workload (proj/src/workload.cpp:50-78), McContext
//            (proj/src/dist.cpp:122-129), sample_logt (proj/src/dist.cpp:142-147).
//
// Nothing here re-implements reference arithmetic; every number comes out of the
// reference's own functions.
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <optional>
#include <vector>

#include "tiesched/dist.hpp"
#include "tiesched/fit.hpp"
#include "tiesched/rng.hpp"
#include "tiesched/sched.hpp"
#include "tiesched/sim.hpp"
#include "tiesched/workload.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
void parallel_for(size_t n, int threads, F&& body) {
  if (threads <= 1 || n < 2) {
    for (size_t i = 0; i < n; ++i) body(i);
    return;
  }
  std::atomic<size_t> next{0};
  const size_t chunk = 256;
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs((size_t)threads);
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (;;) {
          size_t b = next.fetch_add(chunk);
          if (b >= n) break;
          size_t e = std::min(n, b + chunk);
          for (size_t i = b; i < e; ++i) body(i);
        }
      } catch (...) {
        errs[(size_t)t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_hw_threads() { return (int)std::max(1u, std::thread::hardware_concurrency()); }

// McContext(nu, n, seed).samples -> out[n]
int ref_mc_samples(double nu, int n, uint64_t seed, double* out) {
  try {
    tie::McContext mc(nu, n, seed);
    std::memcpy(out, mc.samples.data(), sizeof(double) * mc.samples.size());
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

double ref_t_cdf(double y, double nu) { return tie::t_cdf(y, nu); }
double ref_t_quantile(double p, double nu) { return tie::t_quantile(p, nu); }
double ref_t_pdf(double y, double nu) { return tie::t_pdf(y, nu); }
uint64_t ref_mix64(uint64_t a, uint64_t b) { return tie::mix64(a, b); }

// gen_logt_workload(spec, seed) -> SoA arrays (ids are 0..n-1 by construction)
int ref_gen_workload(uint64_t n, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                     double sg_hi, double nu, uint32_t max_tokens, double rps, double* mu,
                     double* sigma, uint32_t* max_tok, double* arrival, uint32_t* prompt_tokens,
                     uint32_t* true_len) {
  try {
    tie::WorkloadSpec ws;
    ws.n_requests = (size_t)n;
    ws.mu_range = {mu_lo, mu_hi};
    ws.sigma_range = {sg_lo, sg_hi};
    ws.nu = nu;
    ws.max_tokens = max_tokens;
    ws.rps = rps;
    auto reqs = tie::gen_logt_workload(ws, seed);
    for (size_t i = 0; i < reqs.size(); ++i) {
      mu[i] = *reqs[i].true_mu;
      sigma[i] = *reqs[i].true_sigma;
      max_tok[i] = reqs[i].max_tokens;
      if (arrival) arrival[i] = reqs[i].arrival_s;
      if (prompt_tokens) prompt_tokens[i] = reqs[i].prompt_tokens;
      if (true_len) true_len[i] = reqs[i].true_output_tokens;
    }
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// Per request, the reference scoring chain of run_sim (sim.cpp:85-95) followed by
// compute_score (sched.cpp:19-26).  Any of E/C/S may be null.
int ref_score(const double* mu, const double* sigma, const double* x_max, uint64_t n, double nu,
              int mc_n, uint64_t mc_seed, double alpha, double beta, double* E, double* C,
              double* S, int threads) {
  try {
    tie::McContext mc(nu, mc_n, mc_seed);
    parallel_for((size_t)n, threads, [&](size_t i) {
      tie::CensoredLogT cl(tie::LogTParams(mu[i], sigma[i], nu), x_max[i]);
      double e = tie::censored_expectation(cl, mc);
      double c = tie::censored_cvar(cl, mc, alpha);
      c = std::max(c, e);
      if (E) E[i] = e;
      if (C) C[i] = c;
      if (S) S[i] = tie::compute_score(e, c, beta);
    });
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

double ref_compute_beta(int adaptive, double beta_fixed, double beta_max, double q_sat,
                        uint64_t queue_len) {
  tie::ScoreConfig cfg;
  cfg.beta_mode = adaptive ? tie::BetaMode::AdaptiveLinear : tie::BetaMode::Fixed;
  cfg.beta_fixed = beta_fixed;
  cfg.beta_max = beta_max;
  cfg.q_sat = q_sat;
  return tie::compute_beta(cfg, (size_t)queue_len);
}

// Dispatch order of a static queue: WaitingQueue push x n, pop_min until empty.
// ids may be null (then id = index).
int ref_rank(const double* key, const uint64_t* ids, uint64_t n, uint64_t* order) {
  try {
    tie::WaitingQueue q;
    for (uint64_t i = 0; i < n; ++i) {
      tie::QueueEntry e;
      e.req_id = ids ? ids[i] : i;
      e.key = key[i];
      q.push(e);
    }
    uint64_t k = 0;
    while (auto e = q.pop_min()) order[k++] = e->req_id;
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// fit_logt_fixed_nu over P prompts of K samples each (row-major x[P*K]).
int ref_fit(const double* x, uint64_t P, uint64_t K, double nu, double* mu, double* sigma,
            double* ll, int32_t* iters, uint8_t* converged, uint8_t* degenerate, int threads) {
  try {
    parallel_for((size_t)P, threads, [&](size_t p) {
      std::vector<double> v(x + p * K, x + (p + 1) * K);
      tie::FitResult r = tie::fit_logt_fixed_nu(v, nu);
      mu[p] = r.mu;
      sigma[p] = r.sigma;
      if (ll) ll[p] = r.log_likelihood;
      if (iters) iters[p] = r.iterations;
      if (converged) converged[p] = r.converged;
      if (degenerate) degenerate[p] = r.degenerate;
    });
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// cmd_fit's per-prompt analysis (tools/main.cpp:527-562) through the reference's own
// functions: fit_* per family, ks_test(fit_cdf), tail_stats for K >= 10.  Layout as
// tor_fit_report (oracle/tie_oracle.h).
int ref_fit_report(const double* x, uint64_t P, uint64_t K, double nu, unsigned families,
                   double* fits, double* tail, int threads) {
  try {
    parallel_for((size_t)P, threads, [&](size_t p) {
      std::vector<double> v(x + p * K, x + (p + 1) * K);
      const tie::FitFamily fams[4] = {tie::FitFamily::LogTFixedNu, tie::FitFamily::LogTFreeNu,
                                      tie::FitFamily::LogNormal, tie::FitFamily::Exponential};
      for (int f = 0; f < 4; ++f) {
        if (!(families >> f & 1)) continue;
        tie::FitResult fr;
        switch (f) {
          case 0: fr = tie::fit_logt_fixed_nu(v, nu); break;
          case 1: fr = tie::fit_logt_free_nu(v); break;
          case 2: fr = tie::fit_lognormal(v); break;
          default: fr = tie::fit_exponential(v); break;
        }
        (void)fams;
        tie::KsResult ks = tie::ks_test(v, [&](double t) { return tie::fit_cdf(fr, t); });
        double* o = fits + (uint64_t)f * 10 * P;
        const double vals[10] = {fr.mu, fr.sigma, fr.nu, fr.rate, fr.log_likelihood,
                                 (double)fr.iterations, (double)fr.converged,
                                 (double)fr.degenerate, ks.statistic, ks.p_value};
        for (int j = 0; j < 10; ++j) o[(uint64_t)j * P + p] = vals[j];
      }
      if (tail) {
        if (K >= 10) {
          tie::TailStats ts = tie::tail_stats(v);
          const double vals[5] = {ts.skewness, ts.cv, ts.p90_over_p50, ts.p99_over_p50,
                                  ts.top10_share};
          for (int j = 0; j < 5; ++j) tail[(uint64_t)j * P + p] = vals[j];
        } else {
          for (int j = 0; j < 5; ++j) tail[(uint64_t)j * P + p] = std::nan("");
        }
      }
    });
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// save_trace / load_trace (workload.cpp:82-161) through the reference itself
int ref_save_trace(const char* path, uint64_t n, const uint64_t* ids, const double* arrival,
                   const uint32_t* prompt, const uint32_t* output, const uint32_t* max_tokens,
                   const double* mu, const double* sigma) {
  try {
    std::vector<tie::Request> reqs(n);
    for (uint64_t i = 0; i < n; ++i) {
      tie::Request& r = reqs[i];
      r.id = ids[i];
      r.arrival_s = arrival[i];
      r.prompt_tokens = prompt[i];
      r.true_output_tokens = output[i];
      r.max_tokens = max_tokens[i];
      if (mu && !std::isnan(mu[i])) r.true_mu = mu[i];
      if (sigma && !std::isnan(sigma[i])) r.true_sigma = sigma[i];
    }
    tie::save_trace(reqs, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

int ref_load_trace(const char* path, double fill_rps, uint64_t seed, uint64_t cap, uint64_t* ids,
                   double* arrival, uint32_t* prompt, uint32_t* output, uint32_t* max_tokens,
                   double* mu, double* sigma, uint64_t* n_out) {
  try {
    std::optional<double> rps;
    if (fill_rps > 0.0) rps = fill_rps;
    std::vector<tie::Request> reqs = tie::load_trace(path, rps, seed);
    *n_out = reqs.size();
    for (uint64_t i = 0; i < reqs.size() && i < cap; ++i) {
      const tie::Request& r = reqs[i];
      ids[i] = r.id;
      arrival[i] = r.arrival_s;
      prompt[i] = r.prompt_tokens;
      output[i] = r.true_output_tokens;
      max_tokens[i] = r.max_tokens;
      mu[i] = r.true_mu ? *r.true_mu : std::nan("");
      sigma[i] = r.true_sigma ? *r.true_sigma : std::nan("");
    }
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

double ref_logt_loglik(const double* x, uint64_t K, double mu, double sigma, double nu) {
  return tie::logt_loglik(std::vector<double>(x, x + K), mu, sigma, nu);
}

void ref_logt_loglik_grad(const double* x, uint64_t K, double mu, double sigma, double nu,
                          double* grad) {
  const auto g = tie::logt_loglik_grad(std::vector<double>(x, x + K), mu, sigma, nu);
  grad[0] = g[0];
  grad[1] = g[1];
}

// Config-3 prompt generator (following main.cpp:841-845): truths drawn
// sequentially from Rng(seed); samples sample_logt(LogTParams(mu,sigma,nu), K,
// mix64(seed, p)); integerised max(1, llround(x)) with a u32 ceiling (the reference's
// fit CSV carries integer lengths >= 1, main.cpp:458-465).
int ref_gen_fit_data(uint64_t P, uint64_t K, uint64_t seed, double mu_lo, double mu_hi,
                     double sg_lo, double sg_hi, double nu, int integerise, double* x,
                     double* true_mu, double* true_sigma) {
  try {
    tie::Rng rng(seed);
    std::vector<double> m(P), s(P);
    for (uint64_t p = 0; p < P; ++p) {
      m[p] = rng.uniform(mu_lo, mu_hi);
      s[p] = rng.uniform(sg_lo, sg_hi);
    }
    for (uint64_t p = 0; p < P; ++p) {
      auto v = tie::sample_logt(tie::LogTParams(m[p], s[p], nu), (size_t)K, tie::mix64(seed, p));
      for (uint64_t k = 0; k < K; ++k) {
        double val = v[k];
        if (integerise) {
          val = val >= 4294967295.0 ? 4294967295.0 : (double)std::max(1LL, std::llround(val));
        }
        x[p * K + k] = val;
      }
      if (true_mu) true_mu[p] = m[p];
      if (true_sigma) true_sigma[p] = s[p];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// Scheduler-level mirror used by the schedule-step tests: apply a scripted sequence of
// (op, id, E, CVaR) events to a reference tie::Scheduler and record pops.
// op: 0 = on_arrival(id, arrival=E, max_tokens=(uint32)CVaR), 1 = on_prediction(id, E, CVaR),
//     2 = next_request (writes popped id or UINT64_MAX into out[k++]).
int ref_scheduler_script(int policy, int adaptive, double beta_fixed, double beta_max,
                         double q_sat, double rebuild_threshold, uint64_t n_ops,
                         const int32_t* op, const uint64_t* id, const double* a,
                         const double* b, uint64_t* out, uint64_t* n_out) {
  try {
    tie::ScoreConfig cfg;
    cfg.beta_mode = adaptive ? tie::BetaMode::AdaptiveLinear : tie::BetaMode::Fixed;
    cfg.beta_fixed = beta_fixed;
    cfg.beta_max = beta_max;
    cfg.q_sat = q_sat;
    cfg.rebuild_threshold = rebuild_threshold;
    tie::Scheduler s((tie::Policy)policy, cfg);
    uint64_t k = 0;
    for (uint64_t i = 0; i < n_ops; ++i) {
      if (op[i] == 0) {
        tie::Request r{};
        r.id = id[i];
        r.arrival_s = a[i];
        r.max_tokens = (uint32_t)b[i];
        s.on_arrival(r);
      } else if (op[i] == 1) {
        s.on_prediction(id[i], a[i], b[i]);
      } else {
        auto got = s.next_request();
        out[k++] = got ? *got : UINT64_MAX;
      }
    }
    *n_out = k;
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// run_sim's precompute loop (sim.cpp:77-96) through the reference's own predictor and
// scoring functions: predictor 0 oracle_predict / 1 noisy_predict(seed), family 0 log-t /
// 1 log-normal, CVaR = max(CVaR, E).  Requests carry true (mu, sigma) and their ids.
int ref_sim_scores(const double* mu, const double* sigma, const uint64_t* ids,
                   const uint32_t* max_tokens, uint64_t n, int predictor, double mu_sd,
                   double ls_sd, uint64_t seed, int family, double alpha, double* E, double* C,
                   int threads) {
  try {
    tie::McContext mc(3.5);
    tie::NoiseSpec noise;
    noise.mu_sd = mu_sd;
    noise.log_sigma_sd = ls_sd;
    parallel_for((size_t)n, threads, [&](size_t i) {
      tie::Request r{};
      r.id = ids[i];
      r.max_tokens = max_tokens[i];
      r.true_mu = mu[i];
      r.true_sigma = sigma[i];
      const tie::PredictedDist p =
          predictor == 1 ? tie::noisy_predict(r, noise, seed) : tie::oracle_predict(r);
      double e, c;
      if (family == 0) {
        tie::CensoredLogT cl(tie::LogTParams(p.mu_hat, p.sigma_hat, 3.5), (double)r.max_tokens);
        e = tie::censored_expectation(cl, mc);
        c = tie::censored_cvar(cl, mc, alpha);
      } else {
        e = tie::lognormal_censored_expectation(p.mu_hat, p.sigma_hat, (double)r.max_tokens);
        c = tie::lognormal_censored_cvar(p.mu_hat, p.sigma_hat, (double)r.max_tokens, alpha);
      }
      E[i] = e;
      C[i] = std::max(c, e);
    });
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// Schedule-step benchmark on the reference Scheduler (sched.cpp:125-175): preload n_pre
// requests (on_arrival + on_prediction with the given E/CVaR, untimed), then `steps` timed
// steps of: on_arrival x per_step, score those requests with the reference functions
// (censored_expectation / censored_cvar / max, sim.cpp:85-94) + on_prediction, then
// next_request() x pops.  Per-step seconds and the popped ids are returned.
int ref_sched_bench(int policy, int adaptive, double beta_max, double q_sat, double threshold,
                    double alpha, uint64_t n_pre, const uint64_t* pre_ids,
                    const uint32_t* pre_mt, const double* pre_E, const double* pre_C,
                    uint64_t steps, uint64_t per_step, const uint64_t* new_ids,
                    const double* new_mu, const double* new_sigma, const uint32_t* new_mt,
                    uint32_t pops, double* step_seconds, uint64_t* popped, uint64_t* n_popped) {
  try {
    tie::ScoreConfig cfg;
    cfg.beta_mode = adaptive ? tie::BetaMode::AdaptiveLinear : tie::BetaMode::Fixed;
    cfg.beta_max = beta_max;
    cfg.q_sat = q_sat;
    cfg.rebuild_threshold = threshold;
    cfg.alpha = alpha;
    tie::Scheduler s((tie::Policy)policy, cfg);
    tie::McContext mc(3.5);
    for (uint64_t i = 0; i < n_pre; ++i) {
      tie::Request r{};
      r.id = pre_ids[i];
      r.max_tokens = pre_mt[i];
      s.on_arrival(r);
    }
    for (uint64_t i = 0; i < n_pre; ++i) s.on_prediction(pre_ids[i], pre_E[i], pre_C[i]);
    uint64_t k = 0;
    for (uint64_t st = 0; st < steps; ++st) {
      const auto t0 = std::chrono::steady_clock::now();
      for (uint64_t j = 0; j < per_step; ++j) {
        tie::Request r{};
        r.id = new_ids[st * per_step + j];
        r.max_tokens = new_mt[st * per_step + j];
        s.on_arrival(r);
      }
      for (uint64_t j = 0; j < per_step; ++j) {
        const uint64_t i = st * per_step + j;
        tie::CensoredLogT cl(tie::LogTParams(new_mu[i], new_sigma[i], 3.5), (double)new_mt[i]);
        const double e = tie::censored_expectation(cl, mc);
        const double c = std::max(tie::censored_cvar(cl, mc, alpha), e);
        s.on_prediction(new_ids[i], e, c);
      }
      for (uint32_t j = 0; j < pops; ++j) {
        auto got = s.next_request();
        popped[k++] = got ? *got : UINT64_MAX;
      }
      step_seconds[st] =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    *n_popped = k;
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

}  // extern "C"

// ---- per-item distribution functions (dist.hpp:47-88), n items, same op codes as
// include/tie_cuda.h TIE_EVAL_* (1 psi, 2 incbeta, 3 t_pdf, 4 t_cdf, 5 logt_pdf, 6 logt_cdf,
// 7 normal_cdf, 8 normal_quantile, 9 lognormal E, 10 lognormal CVaR)
extern "C" int ref_eval(int op, const double* a, const double* b, const double* c, uint64_t n,
                        double param, double* out) {
  try {
    std::optional<tie::McContext> mc;
    if (op == 1) mc.emplace(param);
    for (uint64_t i = 0; i < n; ++i) {
      switch (op) {
        case 1: out[i] = tie::psi(a[i], tie::LogTParams(b[i], c[i], param), *mc); break;
        case 2: out[i] = tie::regularized_incomplete_beta(a[i], b[i], c[i]); break;
        case 3: out[i] = tie::t_pdf(a[i], param); break;
        case 4: out[i] = tie::t_cdf(a[i], param); break;
        case 5: out[i] = tie::logt_pdf(a[i], tie::LogTParams(b[i], c[i], param)); break;
        case 6: out[i] = tie::logt_cdf(a[i], tie::LogTParams(b[i], c[i], param)); break;
        case 7: out[i] = tie::normal_cdf(a[i]); break;
        case 8: out[i] = tie::normal_quantile(a[i]); break;
        case 9: out[i] = tie::lognormal_censored_expectation(a[i], b[i], c[i]); break;
        case 10: out[i] = tie::lognormal_censored_cvar(a[i], b[i], c[i], param); break;
        default: throw std::invalid_argument("ref_eval: unknown op");
      }
    }
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// ks_test(x, fit_cdf(fit, .)) for one given fit (module.cpp:117-123)
extern "C" int ref_ks_test_fit(const double* x, uint64_t K, int family, double mu, double sigma,
                               double nu, double rate, double* stat, double* p) {
  try {
    tie::FitResult f;
    f.family = (tie::FitFamily)family;
    f.mu = mu;
    f.sigma = sigma;
    f.nu = nu;
    f.rate = rate;
    std::vector<double> v(x, x + K);
    const tie::KsResult r = tie::ks_test(v, [&](double t) { return tie::fit_cdf(f, t); });
    *stat = r.statistic;
    *p = r.p_value;
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// run_sim (sim.cpp:39-185) on the reference's own workload: gen_logt_workload(spec, wseed)
// then run_sim(policy, ScoreConfig{alpha, adaptive, beta_fixed, beta_max, q_sat, threshold},
// EngineConfig{slots, c0, c1, c2}, PredictorConfig{kind, family, noise, batched}, seed).
// Outputs per event (id order): arrival, predict_ready (NaN if none), admit, first_token,
// completion, emitted; metrics[4] = ttft_avg, ttft_p90, ptla_avg, ptla_p90; and the wall
// seconds of run_sim itself.
extern "C" int ref_run_sim(uint64_t n, double rps, double mu_lo, double mu_hi, double sg_lo,
                           double sg_hi, uint32_t prompt_lo, uint32_t prompt_hi,
                           uint32_t max_tokens, uint64_t wseed, int policy, double alpha,
                           int adaptive, double beta_fixed, double beta_max, double q_sat,
                           double threshold, int slots, double c0, double c1, double c2,
                           int kind, int family, double mu_sd, double ls_sd, int batched,
                           uint64_t seed, double* arrival, double* ready, double* admit,
                           double* first, double* done, uint32_t* emitted, double* metrics,
                           double* seconds) {
  try {
    tie::WorkloadSpec ws;
    ws.n_requests = n;
    ws.rps = rps;
    ws.mu_range = {mu_lo, mu_hi};
    ws.sigma_range = {sg_lo, sg_hi};
    ws.prompt_range = {prompt_lo, prompt_hi};
    ws.max_tokens = max_tokens;
    const std::vector<tie::Request> w = tie::gen_logt_workload(ws, wseed);
    tie::ScoreConfig sc;
    sc.alpha = alpha;
    sc.beta_mode = adaptive ? tie::BetaMode::AdaptiveLinear : tie::BetaMode::Fixed;
    sc.beta_fixed = beta_fixed;
    sc.beta_max = beta_max;
    sc.q_sat = q_sat;
    sc.rebuild_threshold = threshold;
    tie::EngineConfig ec;
    ec.batch_slots = slots;
    ec.c0 = c0;
    ec.c1 = c1;
    ec.c2 = c2;
    tie::PredictorConfig pc;
    pc.kind = (tie::PredictorKind)kind;
    pc.family = (tie::ScoreFamily)family;
    pc.noise.mu_sd = mu_sd;
    pc.noise.log_sigma_sd = ls_sd;
    pc.batched = batched != 0;
    const auto t0 = std::chrono::steady_clock::now();
    const tie::SimReport r = tie::run_sim(w, (tie::Policy)policy, sc, ec, pc, seed);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (size_t i = 0; i < r.events.size(); ++i) {
      const tie::RequestEvent& e = r.events[i];
      arrival[i] = e.arrival_s;
      ready[i] = e.predict_ready_s ? *e.predict_ready_s : std::nan("");
      admit[i] = e.admit_s;
      first[i] = e.first_token_s;
      done[i] = e.completion_s;
      emitted[i] = e.emitted_tokens;
    }
    metrics[0] = r.metrics.ttft_avg;
    metrics[1] = r.metrics.ttft_p90;
    metrics[2] = r.metrics.ptla_avg;
    metrics[3] = r.metrics.ptla_p90;
    return 0;
  } catch (const std::domain_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}
