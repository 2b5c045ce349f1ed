// K1 -- batched censored log-t score.
//
// Reference per request (proj/src/dist.cpp:108-189, sim.cpp:85-94, sched.cpp:19-26):
//   sigma' = max(sigma, 1e-9); y_max = (ln x_max - mu)/sigma'; T = T_nu(y_max)
//   k_max  = #{Y_i <= y_max}   (std::upper_bound over the shared sorted sample set)
//   S_all  = sum_{i<k_max} exp(mu + sigma' Y_i)       -> psi(y_max) = S_all / N
//   E      = min(S_all/N + x_max (1-T), x_max)
//   C      = alpha >= T ? x_max : min((S_all/N - S_alpha/N + x_max(1-T)) / (1-alpha), x_max)
//            with S_alpha the same sum up to k_alpha = #{Y_i <= t_quantile(alpha)}
//   C      = max(C, E);  score = E + beta C
//
// Two ways to get S_all / S_alpha, both on the device:
//   EXACT  : one exp per sample-term, ascending sequential sum (the reference's own
//            summation order: bit-faithful up to libdevice-vs-glibc exp rounding).
//   MOMENT : sigma-grid Taylor-moment prefix tables (built once per context):
//              S(k) = e^mu * sum_m delta^m P[g][k][m],  g = round(sigma'/h), delta = sigma'-g h
//            one 128-byte table row per cut instead of ~10^4 exps per request.
//            Requests outside the table (sigma' > sigma_table_max, |mu| > 700) fall back
//            to the exact loop inside the same kernel.
// Validation follows the reference's exception points; the first failing request index is
// recorded in the context's error word (reported by tie_sync as domain/invalid_argument).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "tdist.cuh"
#include "tie_internal.cuh"

namespace tie {
namespace dev {

namespace {

// ------------------------------------------------------------------ double-double
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  s.lo += x.lo + y.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
  const double p = x.hi * y.hi;
  double e = fma(x.hi, y.hi, -p);
  e += x.hi * y.lo + x.lo * y.hi;
  return quick_two_sum(p, e);
}
__device__ __forceinline__ dd dd_mul_d(dd x, double d) {
  const double p = x.hi * d;
  double e = fma(x.hi, d, -p);
  e += x.lo * d;
  return quick_two_sum(p, e);
}
__device__ __forceinline__ dd dd_div_d(dd x, double d) {
  const double q1 = x.hi / d;
  const double p = q1 * d;
  const double pe = fma(q1, d, -p);
  const double r = ((x.hi - p) - pe + x.lo) / d;
  return quick_two_sum(q1, r);
}

// Y^m/m! * exp(sg * y) for m = 0..kMoments-1, in double-double.
__device__ __forceinline__ void moment_terms(double y, double sg, dd (&t)[kMoments]) {
  const double p = sg * y;
  const double pe = fma(sg, y, -p);  // sg*y == p + pe exactly
  const double ex = exp(p);
  dd e = quick_two_sum(ex, ex * pe);  // exp(p + pe) ~= exp(p) (1 + pe)
  dd w = {1.0, 0.0};
#pragma unroll
  for (int m = 0; m < kMoments; ++m) {
    t[m] = dd_mul(e, w);
    w = dd_div_d(dd_mul_d(w, y), (double)(m + 1));
  }
}

// One CTA per grid point g: exclusive prefix sums over k of the moment terms, accumulated
// in double-double and rounded once, so every table entry is within 0.5 ulp of the
// (exp-rounded) exact prefix.
__global__ void __launch_bounds__(512) build_moment_table_kernel(const double* __restrict__ Y,
                                                                 int N,
                                                                 double* __restrict__ table) {
  const int g = blockIdx.x;
  const double sg = g * kGridH;
  const int tid = threadIdx.x;
  const int T = blockDim.x;
  const int chunk = (N + T - 1) / T;
  const int beg = min(tid * chunk, N);
  const int end = min(beg + chunk, N);
  __shared__ double sh_hi[512], sh_lo[512];

  dd acc[kMoments];
#pragma unroll
  for (int m = 0; m < kMoments; ++m) acc[m] = {0.0, 0.0};
  for (int i = beg; i < end; ++i) {
    dd t[kMoments];
    moment_terms(Y[i], sg, t);
#pragma unroll
    for (int m = 0; m < kMoments; ++m) acc[m] = dd_add(acc[m], t[m]);
  }
  // block-wide exclusive scan, one moment at a time (Hillis-Steele in double-double)
  dd run[kMoments];
  for (int m = 0; m < kMoments; ++m) {
    sh_hi[tid] = acc[m].hi;
    sh_lo[tid] = acc[m].lo;
    __syncthreads();
    for (int off = 1; off < T; off <<= 1) {
      dd v = {sh_hi[tid], sh_lo[tid]};
      if (tid >= off) v = dd_add(v, dd{sh_hi[tid - off], sh_lo[tid - off]});
      __syncthreads();
      sh_hi[tid] = v.hi;
      sh_lo[tid] = v.lo;
      __syncthreads();
    }
    run[m] = tid > 0 ? dd{sh_hi[tid - 1], sh_lo[tid - 1]} : dd{0.0, 0.0};
    __syncthreads();
  }
  double* base = table + (size_t)g * (size_t)(N + 1) * kMoments;
  for (int i = beg; i < end; ++i) {
    double* row = base + (size_t)i * kMoments;
#pragma unroll
    for (int m = 0; m < kMoments; ++m) row[m] = run[m].hi + run[m].lo;
    dd t[kMoments];
    moment_terms(Y[i], sg, t);
#pragma unroll
    for (int m = 0; m < kMoments; ++m) run[m] = dd_add(run[m], t[m]);
  }
  if (end == N && beg < end) {
    double* row = base + (size_t)N * kMoments;
#pragma unroll
    for (int m = 0; m < kMoments; ++m) row[m] = run[m].hi + run[m].lo;
  }
  if (N == 0 && tid == 0) {
#pragma unroll
    for (int m = 0; m < kMoments; ++m) base[m] = 0.0;
  }
}

// ------------------------------------------------------------------ per-request helpers
// k = std::upper_bound(Y, Y + N, y) - Y, narrowed by the uniform-y bucket index.
__device__ __forceinline__ uint32_t cut_index(const ScoreParams& p, const double* __restrict__ Y,
                                              double y) {
  if (!(y >= p.y0)) return 0;
  if (y >= p.yN) return (uint32_t)p.N;
  uint32_t lo = 0, hi = (uint32_t)p.N;
  if (p.y_scale > 0.0) {
    int b = (int)((y - p.y0) * p.y_scale);
    b = min(max(b, 0), kYBuckets - 1);
    lo = __ldg(p.ybucket + max(b - 1, 0));
    hi = __ldg(p.ybucket + min(b + 2, kYBuckets));
  }
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (y < Y[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// sum_m delta^m row[m]  (Horner over one 128-byte table row)
__device__ __forceinline__ double horner_row(const double* __restrict__ row, double delta) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  double2 v[kMoments / 2];
#pragma unroll
  for (int j = 0; j < kMoments / 2; ++j) v[j] = __ldg(r2 + j);
  double acc = v[kMoments / 2 - 1].y;
  acc = fma(acc, delta, v[kMoments / 2 - 1].x);
#pragma unroll
  for (int j = kMoments / 2 - 2; j >= 0; --j) {
    acc = fma(acc, delta, v[j].y);
    acc = fma(acc, delta, v[j].x);
  }
  return acc;
}

// Ascending sequential sum of exp(mu + sigma Y_k) (the reference's psi loop,
// dist.cpp:149-156), keeping the prefixes at k_a and k_max in one pass.
__device__ __forceinline__ void exact_sums(const double* __restrict__ Y, double mu, double sg,
                                           uint32_t k_a, uint32_t k_max, double& s_a,
                                           double& s_all) {
  const uint32_t k1 = min(k_a, k_max), k2 = max(k_a, k_max);
  double sum = 0.0;
  uint32_t k = 0;
#pragma unroll 4
  for (; k < k1; ++k) sum = __dadd_rn(sum, exp(__dadd_rn(mu, __dmul_rn(sg, Y[k]))));
  const double s1 = sum;
#pragma unroll 4
  for (; k < k2; ++k) sum = __dadd_rn(sum, exp(__dadd_rn(mu, __dmul_rn(sg, Y[k]))));
  if (k_a <= k_max) {
    s_a = s1;
    s_all = sum;
  } else {
    s_all = s1;
    s_a = sum;
  }
}

struct Out {
  double E, C, S;
};

template <bool kExact>
__device__ __forceinline__ uint32_t score_one(const ScoreParams& p, const double* __restrict__ Ys,
                                              double mu, double sigma, double xm, Out& o) {
  // LogTParams / CensoredLogT validation (dist.cpp:108-120)
  if (!isfinite(mu)) return kMuNotFinite;
  if (!(sigma > 0.0) || !isfinite(sigma)) return kSigmaBad;
  if (!(xm > 0.0) || !isfinite(xm)) return kXmaxBad;
  const double sg = sigma < 1e-9 ? 1e-9 : sigma;
  const double y_max = __dsub_rn(log(xm), mu) / sg;
  const uint32_t k_max = cut_index(p, p.Y, y_max);
  const double T = t_cdf_dev(p.td, y_max);
  const bool saturated = p.alpha >= T;  // censored_cvar case 1 (dist.cpp:187)
  const uint32_t k_a = saturated ? 0u : p.k_alpha;

  double s_a = 0.0, s_all = 0.0;
  bool done = false;
  if (!kExact) {
    const int g = __double2int_rn(sg * kGridInvH);
    if (g < p.G && fabs(mu) <= 700.0) {
      const double delta = sg - g * kGridH;  // exact: h is a power of two
      const double* base = p.table + (size_t)g * (size_t)(p.N + 1) * kMoments;
      const double em = exp(mu);
      s_all = k_max ? em * horner_row(base + (size_t)k_max * kMoments, delta) : 0.0;
      s_a = k_a ? em * horner_row(base + (size_t)k_a * kMoments, delta) : 0.0;
      done = true;
    }
  }
  if (!done) exact_sums(Ys, mu, sg, k_a, k_max, s_a, s_all);

  const double Nd = (double)p.N;
  const double psi_cap = s_all / Nd;
  const double cm = __dsub_rn(1.0, T);
  double E = __dadd_rn(psi_cap, __dmul_rn(xm, cm));
  E = (xm < E) ? xm : E;  // std::min(v, x_max)
  double C;
  if (saturated) {
    C = xm;
  } else {
    const double psi_a = p.alpha > 0.0 ? s_a / Nd : 0.0;
    const double v = __dadd_rn(__dsub_rn(psi_cap, psi_a), __dmul_rn(xm, cm)) /
                     __dsub_rn(1.0, p.alpha);
    C = (xm < v) ? xm : v;
  }
  if (p.raw) {  // per-item censored_expectation / censored_cvar semantics
    o.E = E;
    o.C = C;
    o.S = __longlong_as_double(0x7ff8000000000000LL);
    return kOk;
  }
  C = (C < E) ? E : C;  // run_sim's max(cvar, E) (sim.cpp:94)
  // compute_score checks (sched.cpp:19-26)
  if (!isfinite(E) || !isfinite(C) || !isfinite(p.beta)) return kScoreNotFinite;
  if (!(E > 0.0)) return kExpectationNonPos;
  if (C < E) return kCvarBelowE;
  o.E = E;
  o.C = C;
  o.S = __dadd_rn(E, __dmul_rn(p.beta, C));
  return kOk;
}

template <typename XT, bool kExact>
__global__ void __launch_bounds__(256) score_kernel(const __grid_constant__ ScoreParams p,
                                                    const double* __restrict__ mu,
                                                    const double* __restrict__ sigma,
                                                    const XT* __restrict__ xmax, uint64_t n,
                                                    double* __restrict__ E, double* __restrict__ C,
                                                    double* __restrict__ S,
                                                    uint64_t* __restrict__ keys) {
  extern __shared__ double sY[];
  const double* Ys = p.Y;
  if (kExact && p.N <= 12288) {  // stage the sample set once per CTA (<= 96 KB)
    for (int i = threadIdx.x; i < p.N; i += blockDim.x) sY[i] = p.Y[i];
    __syncthreads();
    Ys = sY;
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    Out o;
    const uint32_t why = score_one<kExact>(p, Ys, mu[i], sigma[i], (double)xmax[i], o);
    if (why != kOk) {
      report(p.err, i, why);
      o.E = o.C = o.S = __longlong_as_double(0x7ff8000000000000LL);
    }
    if (E) E[i] = o.E;
    if (C) C[i] = o.C;
    if (S) S[i] = o.S;
    // rank key: order-preserving u64 image of a positive score (bits | 2^63, as rank.cu)
    if (keys) keys[i] = why == kOk ? ((uint64_t)__double_as_longlong(o.S) | (1ull << 63)) : ~0ull;
  }
}

int sm_count(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cached[device] = v > 0 ? v : 148;
  }
  return cached[device];
}

}  // namespace

cudaError_t build_context_tables(tie_ctx* ctx) {
  const int N = ctx->N;
  const std::vector<double>& Y = ctx->host_samples;
  cudaError_t e;
  if ((e = cudaMalloc(&ctx->d_Y, sizeof(double) * std::max(N, 1))) != cudaSuccess) return e;
  if ((e = cudaMemcpy(ctx->d_Y, Y.data(), sizeof(double) * N, cudaMemcpyHostToDevice)) !=
      cudaSuccess)
    return e;
  // uniform-y bucket index: ybucket[b] = upper_bound(Y, y0 + b / y_scale)
  ctx->y0 = Y.front();
  ctx->yN = Y.back();
  ctx->y_scale = ctx->yN > ctx->y0 ? (double)kYBuckets / (ctx->yN - ctx->y0) : 0.0;
  std::vector<uint32_t> yb(kYBuckets + 1, (uint32_t)N);
  if (ctx->y_scale > 0.0)
    for (int b = 0; b < kYBuckets; ++b) {
      const double edge = ctx->y0 + (double)b / ctx->y_scale;
      yb[b] = (uint32_t)(std::upper_bound(Y.begin(), Y.end(), edge) - Y.begin());
    }
  if ((e = cudaMalloc(&ctx->d_ybucket, sizeof(uint32_t) * yb.size())) != cudaSuccess) return e;
  if ((e = cudaMemcpy(ctx->d_ybucket, yb.data(), sizeof(uint32_t) * yb.size(),
                      cudaMemcpyHostToDevice)) != cudaSuccess)
    return e;
  // sigma-grid moment tables
  ctx->G = (int)std::lrint(ctx->sigma_table_max * kGridInvH) + 1;
  const size_t bytes = (size_t)ctx->G * (size_t)(N + 1) * kMoments * sizeof(double);
  if ((e = cudaMalloc(&ctx->d_table, bytes)) != cudaSuccess) return e;
  build_moment_table_kernel<<<ctx->G, 512>>>(ctx->d_Y, N, ctx->d_table);
  capi::count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

cudaError_t launch_score(tie_ctx* ctx, const double* mu, const double* sigma, const void* x_max,
                         bool x_is_u32, uint64_t n, double alpha, double beta, double* E,
                         double* C, double* S, uint64_t* keys_out, unsigned flags,
                         cudaStream_t s) {
  const bool exact = (flags & 1u) != 0;
  if (n == 0) return cudaSuccess;
  ScoreParams p;
  p.td = ctx->td;
  p.Y = ctx->d_Y;
  p.ybucket = ctx->d_ybucket;
  p.table = ctx->d_table;
  p.y0 = ctx->y0;
  p.y_scale = ctx->y_scale;
  p.yN = ctx->yN;
  p.N = ctx->N;
  p.G = ctx->G;
  p.alpha = alpha;
  p.beta = beta;
  p.raw = (flags & 2u) ? 1 : 0;
  p.err = ctx->d_err;
  // k_alpha = #{Y_i <= t_quantile(alpha, nu)}: request-invariant, hoisted (dist.cpp:170)
  if (alpha != ctx->ka_alpha) {
    uint32_t k = 0;
    if (alpha > 0.0) {
      const double y_a = host::t_quantile(alpha, ctx->nu);
      k = (uint32_t)(std::upper_bound(ctx->host_samples.begin(), ctx->host_samples.end(), y_a) -
                     ctx->host_samples.begin());
    }
    ctx->ka_alpha = alpha;
    ctx->ka_k = k;
  }
  p.k_alpha = ctx->ka_k;
  const int sms = sm_count(ctx->device);
  const uint64_t blocks_needed = (n + 255) / 256;
  ProfScope prof(ctx, exact ? "score.exact" : "score.moment", s);
  if (exact) {
    const size_t smem = ctx->N <= 12288 ? sizeof(double) * ctx->N : 0;
    const uint64_t grid = std::min<uint64_t>(blocks_needed, (uint64_t)sms * 2);
    if (x_is_u32) {
      cudaFuncSetAttribute(score_kernel<uint32_t, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      score_kernel<uint32_t, true><<<(unsigned)grid, 256, smem, s>>>(
          p, mu, sigma, (const uint32_t*)x_max, n, E, C, S, keys_out);
    } else {
      cudaFuncSetAttribute(score_kernel<double, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      score_kernel<double, true><<<(unsigned)grid, 256, smem, s>>>(
          p, mu, sigma, (const double*)x_max, n, E, C, S, keys_out);
    }
  } else {
    const uint64_t grid = std::min<uint64_t>(blocks_needed, (uint64_t)sms * 8);
    if (x_is_u32)
      score_kernel<uint32_t, false><<<(unsigned)grid, 256, 0, s>>>(
          p, mu, sigma, (const uint32_t*)x_max, n, E, C, S, keys_out);
    else
      score_kernel<double, false><<<(unsigned)grid, 256, 0, s>>>(
          p, mu, sigma, (const double*)x_max, n, E, C, S, keys_out);
  }
  capi::count_launch();
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace tie
