// run_sim's scoring precompute (proj/src/sim.cpp:77-96) on the GPU -- SURVEY.md 8f #2.
//
// Per request: the predictor (oracle_predict: the true (mu, sigma); noisy_predict: Gaussian
// noise from a private Rng(mix64(seed, id)), predictor.cpp:15-31), then the scoring family
// (log-t: K1's censored E / CVaR over the shared sample set; log-normal: the closed forms of
// dist.cpp:191-249), then CVaR = max(CVaR, E) (sim.cpp:94).
//
// noisy_predict draws exactly two normals from a freshly seeded std::mt19937_64: one
// Box-Muller pair, i.e. the engine's first two outputs.  The device replays the standard
// seeding recurrence up to state word 157 and the first two twist steps, so the draws are
// bit-identical to the reference's; only libm rounding (log / cos / sin / log1p / expm1,
// <= 1-2 ulp) separates the predicted (mu, sigma).
#include <cuda_runtime.h>

#include <cmath>

#include "../../include/tie_cuda.h"
#include "tie_internal.cuh"

namespace tie {
namespace dev {
namespace {

__device__ __forceinline__ uint64_t mix64_dev(uint64_t a, uint64_t b) {  // rng.hpp:10-16
  uint64_t z = a + 0x9E3779B97F4A7C15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  return x ^ (x >> 43);
}

__device__ __forceinline__ uint64_t mt_twist(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t y = (a & 0xFFFFFFFF80000000ULL) | (b & 0x7FFFFFFFULL);
  return c ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

// first two outputs of std::mt19937_64(seed)
__device__ __forceinline__ void mt_first_two(uint64_t seed, uint64_t& o0, uint64_t& o1) {
  uint64_t m = seed, m0 = seed, m1 = 0, m2 = 0, m156 = 0, m157 = 0;
  for (uint32_t i = 1; i <= 157; ++i) {
    m = 6364136223846793005ULL * (m ^ (m >> 62)) + i;
    if (i == 1) m1 = m;
    if (i == 2) m2 = m;
    if (i == 156) m156 = m;
  }
  m157 = m;
  o0 = mt_temper(mt_twist(m0, m1, m156));
  o1 = mt_temper(mt_twist(m1, m2, m157));
}

__device__ __forceinline__ double u01(uint64_t x) {  // rng.hpp:26-28
  return ((double)(x >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

struct SimArgs {
  const double* mu;
  const double* sigma;
  const uint64_t* ids;
  const uint32_t* max_tokens;
  uint64_t n;
  int predictor;  // 0 oracle, 1 noisy
  double mu_sd, ls_sd;
  uint64_t seed;
  int family;     // 0 log-t (predict only here), 1 log-normal (full score here)
  double alpha, one_minus_alpha, z_alpha;  // z_alpha = normal_quantile(alpha) (host)
  double* mu_hat;
  double* sigma_hat;
  double* E;
  double* C;
  unsigned long long* err;
};

__device__ __forceinline__ double normal_cdf(double z) {  // dist.cpp:191
  return 0.5 * erfc(__dmul_rn(-z, 0.7071067811865475244));
}

__global__ void sim_predict_kernel(const SimArgs a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    double m = a.mu[i], s = a.sigma[i];
    if (a.predictor == 1) {  // noisy_predict (predictor.cpp:22-31)
      uint64_t o0, o1;
      mt_first_two(mix64_dev(a.seed, a.ids[i]), o0, o1);
      const double r = sqrt(-2.0 * log(u01(o0)));
      const double ang = __dmul_rn(2.0 * 3.14159265358979323846, u01(o1));
      const double n1 = __dmul_rn(r, cos(ang)), n2 = __dmul_rn(r, sin(ang));
      m = __dadd_rn(m, __dmul_rn(a.mu_sd, n1));
      const double st = __dadd_rn(log1p(s), __dmul_rn(a.ls_sd, n2));
      const double sh = expm1(st);
      s = (sh < 1e-6) ? 1e-6 : sh;  // std::max(expm1(st), 1e-6)
    }
    if (a.family == 0) {
      a.mu_hat[i] = m;
      a.sigma_hat[i] = s;
      continue;
    }
    // log-normal family: lognormal_censored_expectation / _cvar (dist.cpp:227-249)
    const double xm = (double)a.max_tokens[i];
    if (!(s > 0.0) || !isfinite(s) || !isfinite(m)) {
      report(a.err, i, kSigmaBad);
      continue;
    }
    if (!(xm > 0.0)) {
      report(a.err, i, kXmaxBad);
      continue;
    }
    const double y_max = __dsub_rn(log(xm), m) / s;
    const double P = normal_cdf(y_max);
    const double tail = __dsub_rn(1.0, P);
    const double scale = exp(__dadd_rn(m, __dmul_rn(__dmul_rn(0.5, s), s)));
    const double body_e = __dmul_rn(scale, normal_cdf(__dsub_rn(y_max, s)));
    double E = __dadd_rn(body_e, __dmul_rn(xm, tail));
    E = (xm < E) ? xm : E;
    double C;
    if (a.alpha >= P) {
      C = xm;
    } else {
      const double lo = a.alpha > 0.0 ? normal_cdf(__dsub_rn(a.z_alpha, s)) : 0.0;
      const double body = __dmul_rn(scale, __dsub_rn(normal_cdf(__dsub_rn(y_max, s)), lo));
      const double v = __dadd_rn(body, __dmul_rn(xm, tail)) / a.one_minus_alpha;
      C = (xm < v) ? xm : v;
    }
    a.E[i] = E;
    a.C[i] = (C < E) ? E : C;  // sim.cpp:94
  }
}

__global__ void cvar_max_kernel(const double* E, double* C, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    C[i] = (C[i] < E[i]) ? E[i] : C[i];
}

}  // namespace
}  // namespace dev
}  // namespace tie

using tie::capi::cuda_error;
using tie::capi::set_error;

extern "C" int tie_sim_scores(tie_ctx* ctx, const double* mu, const double* sigma,
                              const uint64_t* ids, const uint32_t* max_tokens, uint64_t n,
                              int predictor, double mu_sd, double log_sigma_sd, uint64_t seed,
                              int family, double alpha, double* E, double* cvar, void* stream) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_sim_scores: null context");
  if (!(alpha >= 0.0 && alpha < 1.0))
    return set_error(TIE_EDOMAIN, "censored_cvar: alpha must lie in [0, 1)");
  if (predictor == 1 && (mu_sd < 0.0 || log_sigma_sd < 0.0))
    return set_error(TIE_EDOMAIN, "noisy_predict: noise standard deviations must be >= 0");
  if (n == 0) return TIE_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  ctx->err_op = "tie_sim_scores";
  tie::dev::SimArgs a;
  a.mu = mu;
  a.sigma = sigma;
  a.ids = ids;
  a.max_tokens = max_tokens;
  a.n = n;
  a.predictor = predictor;
  a.mu_sd = mu_sd;
  a.ls_sd = log_sigma_sd;
  a.seed = seed;
  a.family = family;
  a.alpha = alpha;
  a.one_minus_alpha = 1.0 - alpha;
  a.z_alpha = alpha > 0.0 ? tie::host::normal_quantile(alpha) : 0.0;
  a.E = E;
  a.C = cvar;
  a.err = ctx->d_err;
  a.mu_hat = a.sigma_hat = nullptr;
  if (family == 0) {  // predicted (mu, sigma) into scratch, then K1 in per-item mode
    double* buf = (double*)tie::capi::scratch(ctx, 16 * n + 256, s);
    if (!buf) return set_error(TIE_ECUDA, "tie_sim_scores: scratch allocation failed");
    a.mu_hat = buf;
    a.sigma_hat = buf + n;
  }
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  tie::dev::sim_predict_kernel<<<grid, 256, 0, s>>>(a);
  tie::capi::count_launch();
  if (family == 0) {
    cudaError_t e = tie::dev::launch_score(ctx, a.mu_hat, a.sigma_hat, max_tokens, true, n,
                                           alpha, 0.0, E, cvar, nullptr, nullptr, nullptr,
                                           TIE_SCORE_RAW, s);
    if (e != cudaSuccess) return cuda_error(e, "tie_sim_scores");
    tie::dev::cvar_max_kernel<<<grid, 256, 0, s>>>(E, cvar, n);
    tie::capi::count_launch();
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_sim_scores");
}

extern "C" int tie_sim_scores_host(tie_ctx* ctx, const double* mu, const double* sigma,
                                   const uint64_t* ids, const uint32_t* max_tokens, uint64_t n,
                                   int predictor, double mu_sd, double log_sigma_sd,
                                   uint64_t seed, int family, double alpha, double* E,
                                   double* cvar) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_sim_scores_host: null context");
  if (n == 0) return TIE_OK;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  char* b = nullptr;
  const size_t bytes = 8 * n * 5 + 4 * n + 1024;
  if (cudaMalloc(&b, bytes) != cudaSuccess)
    return set_error(TIE_ECUDA, "tie_sim_scores_host: device allocation failed");
  double* d_mu = (double*)b;
  double* d_sg = d_mu + n;
  uint64_t* d_ids = (uint64_t*)(d_sg + n);
  double* d_E = (double*)(d_ids + n);
  double* d_C = d_E + n;
  uint32_t* d_mt = (uint32_t*)(d_C + n);
  cudaMemcpyAsync(d_mu, mu, 8 * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_sg, sigma, 8 * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_ids, ids, 8 * n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_mt, max_tokens, 4 * n, cudaMemcpyHostToDevice, s);
  int rc = tie_sim_scores(ctx, d_mu, d_sg, d_ids, d_mt, n, predictor, mu_sd, log_sigma_sd,
                          seed, family, alpha, d_E, d_C, s);
  if (rc == TIE_OK) {
    cudaMemcpyAsync(E, d_E, 8 * n, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(cvar, d_C, 8 * n, cudaMemcpyDeviceToHost, s);
    rc = tie_sync(ctx, s);
  }
  cudaStreamSynchronize(s);
  cudaFree(b);
  return rc;
}
