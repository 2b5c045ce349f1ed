// cmd_fit's per-prompt analysis on the GPU: for P prompts x K lengths,
// the reference's four families, a KS test of each fit and the tail statistics --
// tools/main.cpp:527-562 per prompt:
//   logt          fit_logt_fixed_nu(x, nu)                               (fit.cpp:73-178)
//   logt_free_nu  best log-likelihood of fit_logt_fixed_nu over default_nu_grid = 1.0,
//                 1.5, ..., 10.0 (strict >, the first grid point wins ties) (fit.cpp:180-200)
//   lognormal     closed form (fit.cpp:202-230);  exponential (fit.cpp:232-243)
//   ks_test(x, fit_cdf(fit, .))                                          (fit.cpp:245-284)
//   tail_stats(x) when K >= 10                                           (fit.cpp:286-324)
// The BFGS fits reuse K3 (fit.cu) -- one launch per grid point for the free-nu family, each
// followed by a keep-best pass; one stats kernel (one prompt per thread) then sorts a copy
// of the row, fits the closed-form families and evaluates every KS statistic (the log-t CDF
// is the score kernel's device t_cdf, per-nu constants built on the host like the
// reference's) and the tail statistics, in the reference's summation orders.
// Layout: fits[f][field][P], f = logt, logt_free_nu, lognormal, exponential; field = mu,
// sigma, nu, rate, log_likelihood, iterations, converged, degenerate, ks_statistic,
// ks_p_value.  tail[field][P] = skewness, cv, p90/p50, p99/p50, top10_share (NaN if K < 10).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/tie_cuda.h"
#include "tdist.cuh"
#include "tie_internal.cuh"

namespace tie {
namespace dev {
namespace {

constexpr int kFields = 10;
constexpr int kGrid = 19;       // default_nu_grid (fit.cpp:180-184)
constexpr int kLocalK = 64;     // rows up to this length are sorted in thread-local memory

enum { F_MU, F_SIGMA, F_NU, F_RATE, F_LL, F_ITERS, F_CONV, F_DEGEN, F_KSD, F_KSP };
constexpr unsigned kGiven = 0x10000u;  // families flag: the fits are inputs (tie_ks_test_fit)

struct FitTmp {
  double* mu;
  double* sigma;
  double* ll;
  int32_t* iters;
  uint8_t* conv;
  uint8_t* degen;
};

// copy one fixed-nu fit into family `f` (first = 1: unconditional; else keep if ll > best,
// the reference's `if (!have || r.log_likelihood > best.log_likelihood)`)
__global__ void keep_fit_kernel(FitTmp t, uint64_t P, double nu, int first, double* fam) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double ll = t.ll[p];
  if (!first && !(ll > fam[F_LL * P + p])) return;
  fam[F_MU * P + p] = t.mu[p];
  fam[F_SIGMA * P + p] = t.sigma[p];
  fam[F_NU * P + p] = nu;
  fam[F_RATE * P + p] = 0.0;
  fam[F_LL * P + p] = ll;
  fam[F_ITERS * P + p] = (double)t.iters[p];
  fam[F_CONV * P + p] = (double)t.conv[p];
  fam[F_DEGEN * P + p] = (double)t.degen[p];
}

struct StatsArgs {
  const double* x;
  uint64_t P;
  int K;
  unsigned families;
  double* fits;
  double* tail;
  double* scratch;           // P x K rows for K > kLocalK
  const TdistConst* td;      // [0] fixed nu, [1 + g] grid point g
  double grid0, grid_step;
  unsigned long long* err;
};

__device__ __forceinline__ double normal_cdf(double z) {  // dist.cpp:191
  return 0.5 * erfc(-z * 0.7071067811865475244);
}

template <class Row>
__device__ void stats_one(const StatsArgs& a, uint64_t p, const double* x, Row s) {
  const int K = a.K;
  const uint64_t P = a.P;
  const bool given = a.families & kGiven;  // ks_test(x, fit_cdf(fit, .)) of caller fits only
  // ks_test / tail_stats sort a copy of the row (insertion sort: K is small)
  for (int i = 0; i < K; ++i) {
    s[i] = x[i];
    if (!given && (!(x[i] > 0.0) || !isfinite(x[i]))) report(a.err, p, kSampleBad);  // check_samples
  }
  for (int i = 1; i < K; ++i) {
    const double v = s[i];
    int j = i - 1;
    while (j >= 0 && s[j] > v) {
      s[j + 1] = s[j];
      --j;
    }
    s[j + 1] = v;
  }
  const double n = (double)K;
  for (int f = 0; f < 4; ++f) {
    if (!(a.families >> f & 1)) continue;
    double* o = a.fits + (uint64_t)f * kFields * P;
    double mu = 0.0, sigma = 0.0, rate = 0.0;
    if (given) {
      mu = o[F_MU * P + p];
      sigma = o[F_SIGMA * P + p];
      rate = o[F_RATE * P + p];
    } else if (f == 2) {  // fit_lognormal (fit.cpp:202-230)
      double mean = 0.0;
      for (int i = 0; i < K; ++i) mean += log(x[i]);
      mean /= n;
      double var = 0.0;
      for (int i = 0; i < K; ++i) {
        const double d = log(x[i]) - mean;
        var += d * d;
      }
      var /= n;
      mu = mean;
      sigma = sqrt(var);
      double degen = 0.0;
      if (sigma < 1e-6) {
        sigma = 1e-6;
        degen = 1.0;
      }
      double ll = 0.0;
      for (int i = 0; i < K; ++i) {
        const double z = (log(x[i]) - mu) / sigma;
        ll += -log(sigma * x[i]) - 0.5 * log(2.0 * 3.14159265358979323846) - 0.5 * z * z;
      }
      o[F_MU * P + p] = mu;
      o[F_SIGMA * P + p] = sigma;
      o[F_NU * P + p] = 0.0;
      o[F_RATE * P + p] = 0.0;
      o[F_LL * P + p] = ll;
      o[F_ITERS * P + p] = 0.0;
      o[F_CONV * P + p] = 1.0;
      o[F_DEGEN * P + p] = degen;
    } else if (f == 3) {  // fit_exponential (fit.cpp:232-243)
      double mean = 0.0;
      for (int i = 0; i < K; ++i) mean += x[i];
      mean /= n;
      rate = 1.0 / mean;
      o[F_MU * P + p] = 0.0;
      o[F_SIGMA * P + p] = 0.0;
      o[F_NU * P + p] = 0.0;
      o[F_RATE * P + p] = rate;
      o[F_LL * P + p] = n * log(rate) - rate * mean * n;
      o[F_ITERS * P + p] = 0.0;
      o[F_CONV * P + p] = 1.0;
      o[F_DEGEN * P + p] = 0.0;
    } else {
      mu = o[F_MU * P + p];
      sigma = o[F_SIGMA * P + p];
    }
    // constants of the fit's nu for the log-t CDF
    const TdistConst* td = a.td;
    if (f == 1 && !given) {
      const int g = (int)llrint((o[F_NU * P + p] - a.grid0) / a.grid_step);
      td = a.td + 1 + min(max(g, 0), kGrid - 1);
    }
    // ks_test (fit.cpp:261-284) with fit_cdf (fit.cpp:245-258)
    double d = 0.0;
    bool bad = false;
    for (int i = 0; i < K; ++i) {
      const double xi = s[i];
      double F;
      if (!(xi > 0.0)) F = 0.0;
      else if (f <= 1) F = t_cdf_dev(*td, (log(xi) - mu) / sigma);
      else if (f == 2) F = normal_cdf((log(xi) - mu) / sigma);
      else F = -expm1(-rate * xi);
      if (!(F >= 0.0 && F <= 1.0)) bad = true;
      const double u = ((double)i + 1.0) / n - F, w = F - (double)i / n;
      const double m = u < w ? w : u;
      d = d < m ? m : d;
    }
    if (bad) report(a.err, p, kKsCdfRange);
    const double lambda = (sqrt(n) + 0.12 + 0.11 / sqrt(n)) * d;
    double pv = 0.0, sign = 1.0;
    for (int j = 1; j <= 100; ++j) {
      const double term = sign * 2.0 * exp(-2.0 * j * j * lambda * lambda);
      pv += term;
      if (fabs(term) < 1e-12) break;
      sign = -sign;
    }
    pv = pv > 0.0 ? pv : 0.0;
    pv = pv < 1.0 ? pv : 1.0;
    o[F_KSD * P + p] = d;
    o[F_KSP * P + p] = pv;
  }
  if (!a.tail) return;
  if (K < 10) {
    for (int j = 0; j < 5; ++j) a.tail[j * P + p] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  // tail_stats (fit.cpp:286-324) on the sorted copy
  double total = 0.0;
  for (int i = 0; i < K; ++i) total += s[i];
  const double mean = total / n;
  double m2 = 0.0, m3 = 0.0;
  for (int i = 0; i < K; ++i) {
    const double dd = s[i] - mean;
    m2 += dd * dd;
    m3 += dd * dd * dd;
  }
  m2 /= n;
  m3 /= n;
  auto rank = [&](double q) {  // nearest rank
    int k = (int)ceil(q * n);
    k = max(1, min(k, K));
    return s[k - 1];
  };
  const double p50 = rank(0.50), p90 = rank(0.90), p99 = rank(0.99);
  const int k10 = (int)ceil(0.1 * n);
  double top = 0.0;
  for (int i = K - k10; i < K; ++i) top += s[i];
  a.tail[0 * P + p] = m2 > 0.0 ? m3 / pow(m2, 1.5) : 0.0;
  a.tail[1 * P + p] = mean > 0.0 ? sqrt(m2) / mean : 0.0;
  a.tail[2 * P + p] = p50 > 0.0 ? p90 / p50 : 1.0;
  a.tail[3 * P + p] = p50 > 0.0 ? p99 / p50 : 1.0;
  a.tail[4 * P + p] = total > 0.0 ? top / total : 0.0;
}

__global__ void __launch_bounds__(128) report_stats_kernel(const StatsArgs a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.P; p += stride) {
    const double* x = a.x + p * (uint64_t)a.K;
    if (a.K <= kLocalK) {
      double s[kLocalK];
      stats_one(a, p, x, s);
    } else {
      stats_one(a, p, x, a.scratch + p * (uint64_t)a.K);
    }
  }
}

TdistConst make_td(double nu) {
  TdistConst td;
  td.nu = nu;
  td.a = 0.5 * nu;
  td.b = 0.5;
  td.logbeta = std::lgamma(td.a) + std::lgamma(td.b) - std::lgamma(td.a + td.b);
  td.thresh = (td.a + 1.0) / (td.a + td.b + 2.0);
  host::make_cf_table(td.a, td.b, &td.ab);
  host::make_cf_table(td.b, td.a, &td.ba);
  return td;
}

}  // namespace

cudaError_t launch_fit_report(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                              unsigned families, double* fits, double* tail, cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  cudaError_t e;
  // per-nu t constants: [0] = nu, [1 + g] = grid point g (host, glibc lgamma like t_cdf's)
  std::vector<TdistConst> tds;
  tds.push_back(make_td(nu));
  const double grid0 = 1.0, step = 0.5;
  std::vector<double> grid;
  for (double v = 1.0; v <= 10.0 + 1e-9; v += 0.5) grid.push_back(v);  // fit.cpp:180-184
  for (double v : grid) tds.push_back(make_td(v));
  // temporaries (stream-ordered): typed fit outputs, the K > kLocalK sort rows, constants
  const size_t tmp_bytes = (P * (3 * sizeof(double) + sizeof(int32_t) + 2) + 255) & ~(size_t)255;
  const size_t rows_bytes = K > (uint64_t)kLocalK ? P * K * sizeof(double) : 0;
  char* tmp = nullptr;
  if ((e = cudaMallocAsync((void**)&tmp, tmp_bytes + rows_bytes + sizeof(TdistConst) * tds.size(),
                           s)) != cudaSuccess)
    return e;
  FitTmp t;
  t.mu = (double*)tmp;
  t.sigma = t.mu + P;
  t.ll = t.sigma + P;
  t.iters = (int32_t*)(t.ll + P);
  t.conv = (uint8_t*)(t.iters + P);
  t.degen = t.conv + P;
  double* rows = (double*)(tmp + tmp_bytes);
  TdistConst* d_td = (TdistConst*)((char*)rows + rows_bytes);
  cudaMemcpyAsync(d_td, tds.data(), sizeof(TdistConst) * tds.size(), cudaMemcpyHostToDevice, s);
  const unsigned g = (unsigned)((P + 255) / 256);
  if ((families & 1u) && !(families & kGiven)) {
    if ((e = launch_fit(ctx, x, P, K, nu, t.mu, t.sigma, t.ll, t.iters, t.conv, t.degen, s)))
      return e;
    keep_fit_kernel<<<g, 256, 0, s>>>(t, P, nu, 1, fits);
    capi::count_launch();
  }
  if ((families & 2u) && !(families & kGiven)) {
    double* fam = fits + (uint64_t)1 * kFields * P;
    for (size_t i = 0; i < grid.size(); ++i) {
      if ((e = launch_fit(ctx, x, P, K, grid[i], t.mu, t.sigma, t.ll, t.iters, t.conv, t.degen,
                          s)))
        return e;
      keep_fit_kernel<<<g, 256, 0, s>>>(t, P, grid[i], i == 0 ? 1 : 0, fam);
      capi::count_launch();
    }
  }
  StatsArgs a;
  a.x = x;
  a.P = P;
  a.K = (int)K;
  a.families = families;
  a.fits = fits;
  a.tail = tail;
  a.scratch = rows;
  a.td = d_td;
  a.grid0 = grid0;
  a.grid_step = step;
  a.err = ctx->d_err;
  {
    ProfScope prof(ctx, "fit.report_stats", s);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const unsigned gs = (unsigned)std::min<uint64_t>((P + 127) / 128, (uint64_t)std::max(sms, 1) * 16);
    report_stats_kernel<<<gs, 128, 0, s>>>(a);
    capi::count_launch();
  }
  cudaFreeAsync(tmp, s);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace tie

using tie::capi::set_error;

// ks_test(x, fit_cdf(fit, .)) (fit.cpp:245-284) for one caller-given fit: the report kernel's
// KS pass with the fit as input.  family: 0 LogTFixedNu, 1 LogTFreeNu, 2 LogNormal,
// 3 Exponential (fit.hpp:11).
extern "C" int tie_ks_test_fit_host(tie_ctx* ctx, const double* x, uint64_t K, int family,
                                    double mu, double sigma, double nu, double rate,
                                    double* statistic, double* p_value) {
  if (!ctx || !x || !statistic || !p_value)
    return set_error(TIE_EINVALID, "tie_ks_test_fit_host: null argument");
  if (K < 5) return set_error(TIE_EINVALID, "ks_test: need at least 5 samples");
  if (family < 0 || family > 3) return set_error(TIE_EINVALID, "ks_test_fit: bad family");
  const bool logt = family <= 1;
  if (logt && (!(nu > 0.0) || !std::isfinite(nu)))
    return set_error(TIE_EDOMAIN, "t_cdf: nu must be finite and > 0");
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  const uint64_t nf = 4 * tie::dev::kFields;
  std::vector<double> fits(nf, 0.0);
  double* o = fits.data() + (uint64_t)family * tie::dev::kFields;
  o[tie::dev::F_MU] = mu;
  o[tie::dev::F_SIGMA] = sigma;
  o[tie::dev::F_NU] = nu;
  o[tie::dev::F_RATE] = rate;
  double* d = nullptr;
  if (cudaMalloc(&d, 8 * (K + nf)) != cudaSuccess)
    return set_error(TIE_ECUDA, "tie_ks_test_fit_host: device allocation failed");
  cudaMemcpyAsync(d, x, 8 * K, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d + K, fits.data(), 8 * nf, cudaMemcpyHostToDevice, s);
  ctx->err_op = "ks_test";
  cudaError_t e = tie::dev::launch_fit_report(ctx, d, 1, K, logt ? nu : 3.5,
                                              (1u << family) | tie::dev::kGiven, d + K, nullptr, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(fits.data(), d + K, 8 * nf, cudaMemcpyDeviceToHost, s);
  int rc = e == cudaSuccess ? tie_sync(ctx, s) : tie::capi::cuda_error(e, "ks_test_fit");
  cudaStreamSynchronize(s);
  cudaFree(d);
  if (rc) return rc;
  *statistic = o[tie::dev::F_KSD];
  *p_value = o[tie::dev::F_KSP];
  return TIE_OK;
}
