// K3 -- batched log-t MLE fitter: fit_logt_fixed_nu (proj/src/fit.cpp:73-178) for P
// prompts x K samples, one prompt per thread.
//
// The algorithm is the reference's, step for step, because the fitted (mu, sigma) must
// agree to 1e-6 and BFGS paths are discontinuous in their accept/reject decisions:
//   init  mu0 = median(ln x), sigma0 = 1.4826 MAD(ln x)                  (fit.cpp:78-86)
//   degenerate if sigma0 < 1e-6                                          (fit.cpp:92-100)
//   BFGS over theta = (mu, s = ln sigma), H0 = I, <= 500 iterations, gtol 1e-8 (116-122)
//   descent reset (126-132); Armijo c = 1e-4, <= 60 halvings, s >= ln 1e-6 (133-142)
//   stall exit |g| < 1e-6 (143-146); inverse-Hessian update if s'y > 1e-12 (147-161)
//   sigma floor + final log-likelihood (168-177)
// This translation unit is compiled with --fmad=false and keeps every expression in the
// reference's evaluation order, so the only differences from the CPU path are libdevice
// vs glibc rounding of log/log1p/exp (<= 1 ulp).  ln x is computed once per sample (the
// reference recomputes the same value on every likelihood call).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "tie_internal.cuh"

namespace tie {
namespace dev {

namespace {

struct FitConst {
  double nu;
  double lognorm;  // lgamma((nu+1)/2) - lgamma(nu/2) - ln(nu pi)/2   (host, glibc)
  double half_nu1; // 0.5 * (nu + 1)
  double nu1;      // nu + 1
};

// Sample storage: registers when K is a compile-time constant, thread-private global rows
// otherwise.  Both expose the log-samples in ORIGINAL order (the likelihood sums in input
// order) plus a scratch row for the median/MAD sorts.
template <int KT>
struct RegRows {
  static constexpr bool kStatic = true;
  double lx[KT];
  double t[KT];
  __device__ __forceinline__ int size() const { return KT; }
  __device__ __forceinline__ double& L(int i) { return lx[i]; }
  __device__ __forceinline__ double& Tm(int i) { return t[i]; }
};
struct GlobalRows {
  static constexpr bool kStatic = false;
  double* lx;
  double* t;
  int K;
  __device__ __forceinline__ int size() const { return K; }
  __device__ __forceinline__ double& L(int i) { return lx[i]; }
  __device__ __forceinline__ double& Tm(int i) { return t[i]; }
};

// std::max semantics ((a < b) ? b : a), NaN-propagating like the reference's calls
__device__ __forceinline__ double std_max(double a, double b) { return (a < b) ? b : a; }

template <class R>
__device__ __forceinline__ void sort_scratch(R& r) {
  const int K = r.size();
  if (R::kStatic) {  // odd-even transposition network, fully unrolled into min/max pairs
#pragma unroll
    for (int round = 0; round < K; ++round)
#pragma unroll
      for (int i = round & 1; i + 1 < K; i += 2) {
        const double a = r.Tm(i), b = r.Tm(i + 1);
        r.Tm(i) = fmin(a, b);
        r.Tm(i + 1) = fmax(a, b);
      }
  } else {  // insertion sort on the private row
    for (int i = 1; i < K; ++i) {
      const double v = r.Tm(i);
      int j = i - 1;
      while (j >= 0 && r.Tm(j) > v) {
        r.Tm(j + 1) = r.Tm(j);
        --j;
      }
      r.Tm(j + 1) = v;
    }
  }
}

template <class R>
__device__ __forceinline__ double median_scratch(R& r) {  // median_sorted (fit.cpp:27-30)
  const int K = r.size();
  return (K % 2) ? r.Tm(K / 2) : 0.5 * (r.Tm(K / 2 - 1) + r.Tm(K / 2));
}

// logt_loglik (fit.cpp:44-56), sigma given directly
template <class R>
__device__ __forceinline__ double loglik(R& r, const FitConst& c, double mu, double sigma) {
  const double lsig = log(sigma);
  double ll = 0.0;
#pragma unroll
  for (int i = 0; i < r.size(); ++i) {
    const double lx = r.L(i);
    const double z = (lx - mu) / sigma;
    ll += c.lognorm - c.half_nu1 * log1p(z * z / c.nu) - lsig - lx;
  }
  return ll;
}

// fgrad of fit.cpp:105-109: -(dL/dmu), -(dL/dsigma) * sigma at s = ln sigma
template <class R>
__device__ __forceinline__ void neg_grad(R& r, const FitConst& c, double mu, double s,
                                         double& g0, double& g1) {
  const double sigma = exp(s);
  double gmu = 0.0, gsg = 0.0;
#pragma unroll
  for (int i = 0; i < r.size(); ++i) {
    const double z = (r.L(i) - mu) / sigma;
    const double w = c.nu1 * z / (c.nu + z * z);
    gmu += w / sigma;
    gsg += (w * z - 1.0) / sigma;
  }
  g0 = -gmu;
  g1 = -gsg * sigma;
}

struct FitOut {
  double mu, sigma, ll;
  int iters;
  bool converged, degenerate;
};

template <class R>
__device__ void fit_one(R& r, const FitConst& c, FitOut& o) {
  constexpr double kSigmaFloor = 1e-6;
  constexpr double kLogSigmaFloor = -13.815510557964274;  // ln(1e-6)
  const int K = r.size();
#pragma unroll
  for (int i = 0; i < K; ++i) r.Tm(i) = r.L(i);
  sort_scratch(r);
  const double mu0 = median_scratch(r);
#pragma unroll
  for (int i = 0; i < K; ++i) r.Tm(i) = fabs(r.Tm(i) - mu0);
  sort_scratch(r);
  const double sigma0 = 1.4826 * median_scratch(r);
  o.degenerate = false;
  o.iters = 0;
  if (sigma0 < kSigmaFloor) {
    o.mu = mu0;
    o.sigma = kSigmaFloor;
    o.degenerate = true;
    o.converged = true;
    o.ll = loglik(r, c, o.mu, o.sigma);
    return;
  }
  double th0 = mu0, th1 = log(sigma0);
  double f = -loglik(r, c, th0, exp(th1));
  double g0, g1;
  neg_grad(r, c, th0, th1, g0, g1);
  double H00 = 1.0, H01 = 0.0, H10 = 0.0, H11 = 1.0;
  int iter = 0;
  bool converged = false;
  for (; iter < 500; ++iter) {
    if (std_max(fabs(g0), fabs(g1)) < 1e-8) {
      converged = true;
      break;
    }
    double p0 = -(H00 * g0 + H01 * g1), p1 = -(H10 * g0 + H11 * g1);
    double descent = p0 * g0 + p1 * g1;
    if (descent >= 0.0) {
      H00 = H11 = 1.0;
      H01 = H10 = 0.0;
      p0 = -g0;
      p1 = -g1;
      descent = -(g0 * g0 + g1 * g1);
    }
    double step = 1.0, f_new = f, n0 = th0, n1 = th1;
    for (int ls = 0; ls < 60; ++ls) {
      n0 = th0 + step * p0;
      n1 = std_max(th1 + step * p1, kLogSigmaFloor);
      f_new = -loglik(r, c, n0, exp(n1));
      if (isfinite(f_new) && f_new <= f + 1e-4 * step * descent) break;
      step *= 0.5;
    }
    if (!(f_new < f) && std_max(fabs(g0), fabs(g1)) < 1e-6) {
      converged = true;
      break;
    }
    double q0, q1;
    neg_grad(r, c, n0, n1, q0, q1);
    const double s0 = n0 - th0, s1 = n1 - th1;
    const double y0 = q0 - g0, y1 = q1 - g1;
    const double sy = s0 * y0 + s1 * y1;
    if (sy > 1e-12) {
      const double rho = 1.0 / sy;
      const double Hy0 = H00 * y0 + H01 * y1, Hy1 = H10 * y0 + H11 * y1;
      const double yHy = y0 * Hy0 + y1 * Hy1;
      const double k = 1.0 + rho * yHy;
      // H += rho ((1 + rho y'Hy) s s' - s (Hy)' - (Hy) s')   (fit.cpp:155-160)
      H00 += rho * (k * s0 * s0 - s0 * Hy0 - Hy0 * s0);
      H01 += rho * (k * s0 * s1 - s0 * Hy1 - Hy0 * s1);
      H10 += rho * (k * s1 * s0 - s1 * Hy0 - Hy1 * s0);
      H11 += rho * (k * s1 * s1 - s1 * Hy1 - Hy1 * s1);
    }
    th0 = n0;
    th1 = n1;
    f = f_new;
    g0 = q0;
    g1 = q1;
  }
  o.mu = th0;
  o.sigma = exp(th1);
  if (o.sigma <= kSigmaFloor) {
    o.sigma = kSigmaFloor;
    o.degenerate = true;
  }
  o.converged = converged;
  o.iters = iter;
  o.ll = loglik(r, c, o.mu, o.sigma);
}

struct FitArgs {
  FitConst c;
  const double* x;
  uint64_t P;
  int K;
  double* lx_scratch;  // generic path only: [P][K] twice
  double* mu;
  double* sigma;
  double* ll;
  int32_t* iters;
  uint8_t* conv;
  uint8_t* degen;
  unsigned long long* err;
};

__device__ __forceinline__ void store(const FitArgs& a, uint64_t p, const FitOut& o) {
  a.mu[p] = o.mu;
  a.sigma[p] = o.sigma;
  if (a.ll) a.ll[p] = o.ll;
  if (a.iters) a.iters[p] = o.iters;
  if (a.conv) a.conv[p] = o.converged;
  if (a.degen) a.degen[p] = o.degenerate;
}

__device__ __forceinline__ void store_nan(const FitArgs& a, uint64_t p) {
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  FitOut o{nan, nan, nan, 0, false, false};
  store(a, p, o);
}

template <int KT>
__global__ void __launch_bounds__(128) fit_kernel_static(const FitArgs a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.P; p += stride) {
    RegRows<KT> r;
    const double* row = a.x + p * KT;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < KT; ++i) {
      const double v = row[i];
      ok = ok && (v > 0.0) && isfinite(v);
      r.lx[i] = log(v);
    }
    if (!ok) {  // check_samples (fit.cpp:18-25)
      report(a.err, p, kSampleBad);
      store_nan(a, p);
      continue;
    }
    FitOut o;
    fit_one(r, a.c, o);
    store(a, p, o);
  }
}

__global__ void __launch_bounds__(128) fit_kernel_generic(const FitArgs a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < a.P; p += stride) {
    GlobalRows r;
    r.K = a.K;
    r.lx = a.lx_scratch + p * (uint64_t)a.K * 2;
    r.t = r.lx + a.K;
    const double* row = a.x + p * (uint64_t)a.K;
    bool ok = true;
    for (int i = 0; i < a.K; ++i) {
      const double v = row[i];
      ok = ok && (v > 0.0) && isfinite(v);
      r.lx[i] = log(v);
    }
    if (!ok) {
      report(a.err, p, kSampleBad);
      store_nan(a, p);
      continue;
    }
    FitOut o;
    fit_one(r, a.c, o);
    store(a, p, o);
  }
}

// logt_loglik + logt_loglik_grad (fit.cpp:44-71) at P parameter points over one x[K]
__global__ void loglik_kernel(FitConst c, const double* __restrict__ x, int K,
                              const double* __restrict__ mu, const double* __restrict__ sigma,
                              uint64_t P, double* ll, double* grad, unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += stride) {
    const double m = mu[p], sg = sigma[p];
    bool ok = true;
    for (int i = 0; i < K; ++i) ok = ok && (x[i] > 0.0) && isfinite(x[i]);
    if (!ok) {
      report(err, p, kSampleBad);
      continue;
    }
    if (!(sg > 0.0)) {
      report(err, p, kSigmaBad);
      continue;
    }
    if (ll) {
      const double lsig = log(sg);
      double acc = 0.0;
      for (int i = 0; i < K; ++i) {
        const double lx = log(x[i]);
        const double z = (lx - m) / sg;
        acc += c.lognorm - c.half_nu1 * log1p(z * z / c.nu) - lsig - lx;
      }
      ll[p] = acc;
    }
    if (grad) {
      double gmu = 0.0, gsg = 0.0;
      for (int i = 0; i < K; ++i) {
        const double z = (log(x[i]) - m) / sg;
        const double w = c.nu1 * z / (c.nu + z * z);
        gmu += w / sg;
        gsg += (w * z - 1.0) / sg;
      }
      grad[2 * p] = gmu;
      grad[2 * p + 1] = gsg;
    }
  }
}

FitConst make_const(double nu) {
  FitConst c;
  c.nu = nu;
  c.lognorm = std::lgamma(0.5 * (nu + 1.0)) - std::lgamma(0.5 * nu) -
              0.5 * std::log(nu * 3.14159265358979323846);
  c.half_nu1 = 0.5 * (nu + 1.0);
  c.nu1 = nu + 1.0;
  return c;
}

int sm_count(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v > 0 ? v : 148;
}

}  // namespace

cudaError_t launch_fit(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                       double* mu, double* sigma, double* ll, int32_t* iters, uint8_t* conv,
                       uint8_t* degen, cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  FitArgs a;
  a.c = make_const(nu);
  a.x = x;
  a.P = P;
  a.K = (int)K;
  a.lx_scratch = nullptr;
  a.mu = mu;
  a.sigma = sigma;
  a.ll = ll;
  a.iters = iters;
  a.conv = conv;
  a.degen = degen;
  a.err = ctx->d_err;
  const int sms = sm_count(ctx->device);
  const unsigned grid = (unsigned)std::min<uint64_t>((P + 127) / 128, (uint64_t)sms * 16);
  ProfScope prof(ctx, "fit", s);
  switch (K) {
    case 8: fit_kernel_static<8><<<grid, 128, 0, s>>>(a); break;
    case 16: fit_kernel_static<16><<<grid, 128, 0, s>>>(a); break;
    case 20: fit_kernel_static<20><<<grid, 128, 0, s>>>(a); break;
    case 32: fit_kernel_static<32><<<grid, 128, 0, s>>>(a); break;
    default: {
      a.lx_scratch = (double*)capi::scratch(ctx, sizeof(double) * P * K * 2, s);
      if (!a.lx_scratch) return cudaErrorMemoryAllocation;
      fit_kernel_generic<<<grid, 128, 0, s>>>(a);
    }
  }
  capi::count_launch();
  return cudaGetLastError();
}

cudaError_t launch_loglik(tie_ctx* ctx, const double* x, uint64_t K, const double* mu,
                          const double* sigma, uint64_t P, double nu, double* ll, double* grad,
                          cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<uint64_t>((P + 127) / 128, 1184);
  loglik_kernel<<<grid, 128, 0, s>>>(make_const(nu), x, (int)K, mu, sigma, P, ll, grad,
                                     ctx->d_err);
  capi::count_launch();
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace tie
