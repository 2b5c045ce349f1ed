// Host-side numerics the device path depends on (product code, not the oracle).
//
// Only request-INVARIANT quantities live here -- the McContext sample set, y_alpha =
// t_quantile(alpha, nu), the log-beta constant of the t CDF, the continued-fraction
// coefficient tables -- so the device sees bit-identical constants to the reference
// (which computes them with glibc libm).  Everything per request runs on the GPU.
#pragma once

#include <cstdint>
#include <random>
#include <vector>

namespace tie {
namespace host {

// splitmix64 finalizer used for per-entity seeds (rng.hpp:10-16)
uint64_t mix64(uint64_t a, uint64_t b);

// The reference's sampler stack over std::mt19937_64 (rng.hpp:21-83): uniform01 in (0,1),
// Box-Muller with a cached spare, Marsaglia-Tsang gamma, ratio-of-chi-square Student-t.
class Sampler {
 public:
  explicit Sampler(uint64_t seed) : eng_(seed) {}
  double u01();
  double uniform(double lo, double hi) { return lo + (hi - lo) * u01(); }
  uint32_t uniform_u32(uint32_t lo, uint32_t hi);
  double normal();
  double gamma(double shape, double scale);
  double student_t(double nu);
  double exponential(double rate);

 private:
  std::mt19937_64 eng_;
  double cached_ = 0.0;
  bool have_cached_ = false;
};

// McContext(nu, n, seed).samples (dist.cpp:122-129)
std::vector<double> mc_samples(double nu, int n, uint64_t seed);

// Student-t pieces (dist.cpp:19-106); identical operation order to the reference.
double reg_inc_beta(double a, double b, double x);
double t_pdf(double y, double nu);
double t_cdf(double y, double nu);
double t_quantile(double p, double nu);

// standard normal quantile: Acklam's rational approximation + one Newton polish
// (dist.cpp:193-225); host-hoisted for the log-normal family's request-invariant z_alpha
double normal_quantile(double p);

// sample_logt (dist.cpp:142-147)
std::vector<double> sample_logt(double mu, double sigma, double nu, size_t n, uint64_t seed);

// gen_logt_workload (workload.cpp:50-78), SoA.  Synthetic-input generator for bench.py
// and the simulator front-end; ids are 0..n-1.
struct Workload {
  std::vector<double> mu, sigma, arrival;
  std::vector<uint32_t> max_tokens, prompt_tokens, true_len;
};
Workload gen_logt_workload(size_t n, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                           double sg_hi, double nu, uint32_t prompt_lo, uint32_t prompt_hi,
                           uint32_t max_tokens, double rps);

// Continued-fraction constants of I_x(p, q) for the device t CDF (see tdist.cuh).
struct CfTable {
  static constexpr int kTerms = 96;  // 2*kTerms partial numerators after d1
  double d1;                         // -(p+q)/(p+1)
  double even[kTerms];               // m(q-m) / ((p-1+2m)(p+2m)),      m = 1..kTerms
  double odd[kTerms];                // -(p+m)(p+q+m) / ((p+2m)(p+1+2m)) m = 1..kTerms
};
void make_cf_table(double p, double q, CfTable* out);

}  // namespace host
}  // namespace tie
