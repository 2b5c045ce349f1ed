// Per-item distribution functions of the reference's public API (proj/include/tiesched/
// dist.hpp:47-88, bound in proj/bindings/module.cpp:48-60) evaluated on the GPU for a batch
// of items: psi, regularized_incomplete_beta, logt_pdf / logt_cdf, normal_cdf /
// normal_quantile and the log-normal closed forms.  The C++ per-item calls
// (include/tiesched_b200.hpp) are batches of one; Python also gets array versions.
//
// Inputs are validated on the host in the reference's per-item order (the first failing item
// raises the reference's exception), so the kernels only compute.  Operation order follows
// dist.cpp (no FMA contraction: explicit __d*_rn), so results differ from the reference only
// by device-vs-glibc libm rounding (lgamma / exp / log / log1p / erfc, <= 1-2 ulp each).
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/tie_cuda.h"
#include "tie_internal.cuh"

namespace tie {
namespace dev {
namespace {

constexpr double kPi = 3.14159265358979323846;

// incbeta_cf (dist.cpp:19-48): modified Lentz, eps 1e-15, <= 100000 iterations
__device__ double incbeta_cf_dev(double a, double b, double x) {
  const double tiny = 1e-300, eps = 1e-15;
  const double qab = __dadd_rn(a, b), qap = __dadd_rn(a, 1.0), qam = __dsub_rn(a, 1.0);
  double c = 1.0;
  double d = __dsub_rn(1.0, __dmul_rn(qab, x) / qap);
  if (fabs(d) < tiny) d = tiny;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= 100000; ++m) {
    const double m2 = 2.0 * m;
    double aa = __dmul_rn(__dmul_rn((double)m, __dsub_rn(b, (double)m)), x) /
                __dmul_rn(__dadd_rn(qam, m2), __dadd_rn(a, m2));
    d = __dadd_rn(1.0, __dmul_rn(aa, d));
    if (fabs(d) < tiny) d = tiny;
    c = __dadd_rn(1.0, aa / c);
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    h = __dmul_rn(h, __dmul_rn(d, c));
    aa = __dmul_rn(__dmul_rn(-__dadd_rn(a, (double)m), __dadd_rn(qab, (double)m)), x) /
         __dmul_rn(__dadd_rn(a, m2), __dadd_rn(qap, m2));
    d = __dadd_rn(1.0, __dmul_rn(aa, d));
    if (fabs(d) < tiny) d = tiny;
    c = __dadd_rn(1.0, aa / c);
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double del = __dmul_rn(d, c);
    h = __dmul_rn(h, del);
    if (fabs(__dsub_rn(del, 1.0)) < eps) break;
  }
  return h;
}

// regularized_incomplete_beta (dist.cpp:52-63), arguments pre-validated
__device__ double incbeta_dev(double a, double b, double x) {
  if (x == 0.0) return 0.0;
  if (x == 1.0) return 1.0;
  const double logbeta = __dsub_rn(__dadd_rn(lgamma(a), lgamma(b)), lgamma(__dadd_rn(a, b)));
  const double front =
      exp(__dsub_rn(__dadd_rn(__dmul_rn(a, log(x)), __dmul_rn(b, log1p(-x))), logbeta));
  if (x < __dadd_rn(a, 1.0) / __dadd_rn(__dadd_rn(a, b), 2.0))
    return __dmul_rn(front, incbeta_cf_dev(a, b, x)) / a;
  return __dsub_rn(1.0, __dmul_rn(front, incbeta_cf_dev(b, a, __dsub_rn(1.0, x))) / b);
}

__device__ double t_pdf_dev(double y, double nu) {  // dist.cpp:65-71
  const double lognorm =
      __dsub_rn(__dsub_rn(lgamma(__dmul_rn(0.5, __dadd_rn(nu, 1.0))), lgamma(__dmul_rn(0.5, nu))),
                __dmul_rn(0.5, log(__dmul_rn(nu, kPi))));
  return exp(__dsub_rn(lognorm, __dmul_rn(__dmul_rn(0.5, __dadd_rn(nu, 1.0)),
                                          log1p(__dmul_rn(y, y) / nu))));
}

__device__ double t_cdf_gen_dev(double y, double nu) {  // dist.cpp:73-81
  if (isinf(y)) return y > 0.0 ? 1.0 : 0.0;
  const double x = nu / __dadd_rn(__dmul_rn(y, y), nu);
  const double tail = incbeta_dev(__dmul_rn(0.5, nu), 0.5, x);
  return y >= 0.0 ? __dsub_rn(1.0, __dmul_rn(0.5, tail)) : __dmul_rn(0.5, tail);
}

__device__ double normal_cdf_dev(double z) {  // dist.cpp:191
  return __dmul_rn(0.5, erfc(__dmul_rn(-z, 0.7071067811865475244)));
}

__device__ double normal_quantile_dev(double p) {  // dist.cpp:193-225 (Acklam + 1 Newton)
  const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                      1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
  const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                      6.680131188771972e+01,  -1.328068155288572e+01};
  const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                      -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
  const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                      3.754408661907416e+00};
  const double plow = 0.02425, phigh = 1.0 - plow;
  double q, r, z;
#define H5(k, t) \
  __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn( \
  __dmul_rn(k[0], t), k[1]), t), k[2]), t), k[3]), t), k[4]), t), k[5])
#define D4(t)                                                                              \
  __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(d[0], t), \
  d[1]), t), d[2]), t), d[3]), t), 1.0)
  if (p < plow) {
    q = sqrt(__dmul_rn(-2.0, log(p)));
    z = H5(c, q) / D4(q);
  } else if (p <= phigh) {
    q = __dsub_rn(p, 0.5);
    r = __dmul_rn(q, q);
    z = __dmul_rn(H5(a, r), q) /
        __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(
            __dadd_rn(__dmul_rn(b[0], r), b[1]), r), b[2]), r), b[3]), r), b[4]), r), 1.0);
  } else {
    q = sqrt(__dmul_rn(-2.0, log1p(-p)));
    z = -H5(c, q) / D4(q);
  }
#undef H5
#undef D4
  const double e = __dsub_rn(normal_cdf_dev(z), p);
  const double u = __dmul_rn(__dmul_rn(e, sqrt(2.0 * kPi)), exp(__dmul_rn(__dmul_rn(0.5, z), z)));
  return __dsub_rn(z, u / __dadd_rn(1.0, __dmul_rn(__dmul_rn(0.5, z), u)));
}

__device__ double lognormal_e_dev(double mu, double sg, double xm) {  // dist.cpp:227-236
  const double y_max = __dsub_rn(log(xm), mu) / sg;
  const double body = __dmul_rn(exp(__dadd_rn(mu, __dmul_rn(__dmul_rn(0.5, sg), sg))),
                                normal_cdf_dev(__dsub_rn(y_max, sg)));
  const double v = __dadd_rn(body, __dmul_rn(xm, __dsub_rn(1.0, normal_cdf_dev(y_max))));
  return v < xm ? v : xm;
}

__device__ double lognormal_cvar_dev(double mu, double sg, double xm, double alpha) {
  const double y_max = __dsub_rn(log(xm), mu) / sg;  // dist.cpp:238-249
  if (alpha >= normal_cdf_dev(y_max)) return xm;
  const double lo = alpha > 0.0 ? normal_cdf_dev(__dsub_rn(normal_quantile_dev(alpha), sg)) : 0.0;
  const double body = __dmul_rn(exp(__dadd_rn(mu, __dmul_rn(__dmul_rn(0.5, sg), sg))),
                                __dsub_rn(normal_cdf_dev(__dsub_rn(y_max, sg)), lo));
  const double v =
      __dadd_rn(body, __dmul_rn(xm, __dsub_rn(1.0, normal_cdf_dev(y_max)))) / __dsub_rn(1.0, alpha);
  return v < xm ? v : xm;
}

__global__ void eval_kernel(int op, const double* A, const double* B, const double* C,
                            uint64_t n, double param, double* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double r = 0.0;
    switch (op) {
      case TIE_EVAL_INCBETA: r = incbeta_dev(A[i], B[i], C[i]); break;
      case TIE_EVAL_T_PDF: r = t_pdf_dev(A[i], param); break;
      case TIE_EVAL_T_CDF: r = t_cdf_gen_dev(A[i], param); break;
      case TIE_EVAL_LOGT_PDF: {  // dist.cpp:131-135
        const double z = __dsub_rn(log(A[i]), B[i]) / C[i];
        r = t_pdf_dev(z, param) / __dmul_rn(C[i], A[i]);
        break;
      }
      case TIE_EVAL_LOGT_CDF:  // dist.cpp:137-140
        r = t_cdf_gen_dev(__dsub_rn(log(A[i]), B[i]) / C[i], param);
        break;
      case TIE_EVAL_NORMAL_CDF: r = normal_cdf_dev(A[i]); break;
      case TIE_EVAL_NORMAL_QUANTILE: r = normal_quantile_dev(A[i]); break;
      case TIE_EVAL_LOGNORMAL_E: r = lognormal_e_dev(A[i], B[i], C[i]); break;
      case TIE_EVAL_LOGNORMAL_CVAR: r = lognormal_cvar_dev(A[i], B[i], C[i], param); break;
      default: r = __longlong_as_double(0x7ff8000000000000ll);
    }
    out[i] = r;
  }
}

// psi (dist.cpp:149-156): one CTA per item; the samples Y_i <= y are exactly the
// upper_bound prefix of the sorted set, summed as a CTA reduction
__global__ void __launch_bounds__(256) psi_kernel(const double* __restrict__ Y, int N,
                                                  const double* y, const double* mu,
                                                  const double* sg, uint64_t n, double* out) {
  __shared__ double part[8];
  for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
    const double yy = y[i], m = mu[i], s = sg[i];
    double acc = 0.0;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
      const double v = Y[k];
      if (v <= yy) acc = __dadd_rn(acc, exp(__dadd_rn(m, __dmul_rn(s, v))));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
      out[i] = t / (double)N;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace dev
}  // namespace tie

using tie::capi::cuda_error;
using tie::capi::set_error;

namespace {

bool fin(double v) { return std::isfinite(v); }

// the reference's per-item checks, in its order; returns the first failing item's error
int validate(int op, const double* A, const double* B, const double* C, uint64_t n,
             double param) {
  auto dom = [](const std::string& m) { return set_error(TIE_EDOMAIN, m); };
  auto logt_params = [&](double mu, double sg) -> int {  // LogTParams ctor (dist.cpp:108-116)
    if (!fin(mu)) return dom("LogTParams: mu must be finite");
    if (!(sg > 0.0) || !fin(sg)) return dom("LogTParams: sigma must be finite and > 0");
    if (!(param > 0.0) || !fin(param)) return dom("LogTParams: nu must be finite and > 0");
    return TIE_OK;
  };
  for (uint64_t i = 0; i < n; ++i) {
    switch (op) {
      case TIE_EVAL_PSI:
        if (int rc = logt_params(B[i], C[i])) return rc;
        if (std::isnan(A[i])) return dom("psi: y must not be NaN");
        break;
      case TIE_EVAL_INCBETA:
        if (!(A[i] > 0.0) || !(B[i] > 0.0) || !fin(A[i]) || !fin(B[i]))
          return dom("regularized_incomplete_beta: a and b must be finite and > 0");
        if (!(C[i] >= 0.0 && C[i] <= 1.0))
          return dom("regularized_incomplete_beta: x must lie in [0, 1]");
        break;
      case TIE_EVAL_T_PDF:
        if (!fin(A[i])) return dom("t_pdf: y must be finite");
        if (!(param > 0.0) || !fin(param)) return dom("t_pdf: nu must be finite and > 0");
        break;
      case TIE_EVAL_T_CDF:
        if (!(param > 0.0) || !fin(param)) return dom("t_cdf: nu must be finite and > 0");
        if (std::isnan(A[i])) return dom("t_cdf: y must not be NaN");
        break;
      case TIE_EVAL_LOGT_PDF:
      case TIE_EVAL_LOGT_CDF:
        if (int rc = logt_params(B[i], C[i])) return rc;
        if (!(A[i] > 0.0) || !fin(A[i]))
          return dom(op == TIE_EVAL_LOGT_PDF ? "logt_pdf: x must be finite and > 0"
                                             : "logt_cdf: x must be finite and > 0");
        break;
      case TIE_EVAL_NORMAL_CDF: break;
      case TIE_EVAL_NORMAL_QUANTILE:
        if (!(A[i] > 0.0 && A[i] < 1.0)) return dom("normal_quantile: p must lie in (0, 1)");
        break;
      case TIE_EVAL_LOGNORMAL_E:
        if (!(B[i] > 0.0) || !fin(B[i]) || !fin(A[i]))
          return dom("lognormal_censored_expectation: bad parameters");
        if (!(C[i] > 0.0) || !fin(C[i]))
          return dom("lognormal_censored_expectation: x_max must be finite and > 0");
        break;
      case TIE_EVAL_LOGNORMAL_CVAR:
        if (!(param >= 0.0 && param < 1.0))
          return dom("lognormal_censored_cvar: alpha must lie in [0, 1)");
        if (!(B[i] > 0.0) || !fin(B[i]) || !fin(A[i]))
          return dom("lognormal_censored_cvar: bad parameters");
        if (!(C[i] > 0.0) || !fin(C[i]))
          return dom("lognormal_censored_cvar: x_max must be finite and > 0");
        break;
      default: return set_error(TIE_EINVALID, "tie_eval_host: unknown op");
    }
  }
  return TIE_OK;
}

int arity(int op) {
  switch (op) {
    case TIE_EVAL_T_PDF: case TIE_EVAL_T_CDF: case TIE_EVAL_NORMAL_CDF:
    case TIE_EVAL_NORMAL_QUANTILE: return 1;
    default: return 3;
  }
}

}  // namespace

extern "C" int tie_eval_host(tie_ctx* ctx, int op, const double* a, const double* b,
                             const double* c, uint64_t n, double param, double* out) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_eval_host: null context");
  if (n == 0) return TIE_OK;
  const int k = arity(op);
  if (!a || !out || (k == 3 && (!b || !c)))
    return set_error(TIE_EINVALID, "tie_eval_host: null argument");
  if (op == TIE_EVAL_PSI && param != ctx->nu)  // psi (dist.cpp:150)
    return set_error(TIE_EINVALID, "psi: McContext nu does not match distribution nu");
  if (int rc = validate(op, a, b, c, n, param)) return rc;
  cudaSetDevice(ctx->device);
  cudaStream_t s = ctx->stream;
  // sigma < 1e-9 is raised to the floor by LogTParams (dist.cpp:112-115)
  std::vector<double> sg;
  if (op == TIE_EVAL_PSI || op == TIE_EVAL_LOGT_PDF || op == TIE_EVAL_LOGT_CDF) {
    sg.assign(c, c + n);
    for (double& v : sg) v = v < 1e-9 ? 1e-9 : v;
    c = sg.data();
  }
  double* d = nullptr;
  if (cudaMalloc(&d, 8 * n * 4) != cudaSuccess)
    return set_error(TIE_ECUDA, "tie_eval_host: device allocation failed");
  double *dA = d, *dB = d + n, *dC = d + 2 * n, *dO = d + 3 * n;
  cudaMemcpyAsync(dA, a, 8 * n, cudaMemcpyHostToDevice, s);
  if (k == 3) {
    cudaMemcpyAsync(dB, b, 8 * n, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dC, c, 8 * n, cudaMemcpyHostToDevice, s);
  }
  if (op == TIE_EVAL_PSI) {
    tie::dev::psi_kernel<<<(unsigned)std::min<uint64_t>(n, 148 * 8), 256, 0, s>>>(
        ctx->d_Y, ctx->N, dA, dB, dC, n, dO);
  } else {
    tie::dev::eval_kernel<<<(unsigned)std::min<uint64_t>((n + 127) / 128, 148 * 8), 128, 0, s>>>(
        op, dA, dB, dC, n, param, dO);
  }
  tie::capi::count_launch();
  cudaMemcpyAsync(out, dO, 8 * n, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(d);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_eval_host");
}
