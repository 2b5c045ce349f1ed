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
#include <cstring>
#include <limits>
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

// T_nu(y) from the tail-mass table (one 64-byte row + a degree-7 Horner); |y| beyond the
// sample range falls back to the continued fraction.
struct TailRow {
  double2 a[kTailCoef / 2];
  double t;
  bool ok;
};

__device__ __forceinline__ void tail_fetch(const ScoreParams& p, double y, TailRow& r) {
  const double ay = fabs(y);
  r.ok = ay < p.t_ymax;
  if (!r.ok) return;
  const int b = min((int)(ay * p.t_inv_w), kTailBuckets - 1);
  r.t = ay - ((double)b + 0.5) * p.t_w;
  const double2* row = reinterpret_cast<const double2*>(p.tail + (size_t)b * kTailCoef);
#pragma unroll
  for (int j = 0; j < kTailCoef / 2; ++j) r.a[j] = __ldg(row + j);
}

__device__ __forceinline__ double tail_cdf(const ScoreParams& p, double y, const TailRow& r) {
  if (!r.ok) return t_cdf_dev(p.td, y);
  double v = r.a[kTailCoef / 2 - 1].y;
  v = fma(v, r.t, r.a[kTailCoef / 2 - 1].x);
#pragma unroll
  for (int j = kTailCoef / 2 - 2; j >= 0; --j) {
    v = fma(v, r.t, r.a[j].y);
    v = fma(v, r.t, r.a[j].x);
  }
  return y >= 0.0 ? __dsub_rn(1.0, v) : v;  // dist.cpp:80
}

// One 128-byte table row (16 moments) held in registers.
struct Row {
  double2 v[kMoments / 2];
};

__device__ __forceinline__ void load_row(const double* __restrict__ row, Row& r) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int j = 0; j < kMoments / 2; ++j) r.v[j] = __ldg(r2 + j);
}

// sum_m delta^m row[m]  (Horner)
__device__ __forceinline__ double horner(const Row& r, double delta) {
  double acc = r.v[kMoments / 2 - 1].y;
  acc = fma(acc, delta, r.v[kMoments / 2 - 1].x);
#pragma unroll
  for (int j = kMoments / 2 - 2; j >= 0; --j) {
    acc = fma(acc, delta, r.v[j].y);
    acc = fma(acc, delta, r.v[j].x);
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

// ln(x_max) memo: queues share a handful of token budgets, so each thread keeps the last one
struct LogMemo {
  double x = -1.0, lx = 0.0;
  __device__ __forceinline__ double operator()(double xm) {
    if (xm != x) {
      x = xm;
      lx = log(xm);
    }
    return lx;
  }
};

template <bool kRecip = false>
__device__ __forceinline__ uint32_t epilogue(const ScoreParams& p, double xm, double T,
                                             bool saturated, double s_a, double s_all, Out& o);

template <bool kExact>
__device__ __forceinline__ uint32_t score_one(const ScoreParams& p, const double* __restrict__ Ys,
                                              double mu, double sigma, double xm, LogMemo& lnx,
                                              Out& o) {
  // LogTParams / CensoredLogT validation (dist.cpp:108-120)
  if (!isfinite(mu)) return kMuNotFinite;
  if (!(sigma > 0.0) || !isfinite(sigma)) return kSigmaBad;
  if (!(xm > 0.0) || !isfinite(xm)) return kXmaxBad;
  const double sg = sigma < 1e-9 ? 1e-9 : sigma;
  const double y_max = __dsub_rn(lnx(xm), mu) / sg;
  // the tail-mass row depends only on y_max: issue it before the sample search
  TailRow tr;
  tail_fetch(p, y_max, tr);
  const uint32_t k_max = cut_index(p, p.Y, y_max);
  const int g = __double2int_rn(sg * kGridInvH);
  const double reach = fmax(p.taylor_y0, fmin(fmax(y_max, 0.0), p.yN));
  const bool use_table = !kExact && g < p.G && fabs(mu) <= 700.0 &&
                         fabs(sg - g * kGridH) * reach <= kTaylorReach;
  const double* base = p.table + (size_t)(use_table ? g : 0) * (size_t)(p.N + 1) * kMoments;
  Row row_max;
  if (use_table) load_row(base + (size_t)k_max * kMoments, row_max);

  const double T = tail_cdf(p, y_max, tr);
  const bool saturated = p.alpha >= T;  // censored_cvar case 1 (dist.cpp:187)
  const uint32_t k_a = saturated ? 0u : p.k_alpha;

  double s_a = 0.0, s_all = 0.0;
  if (use_table) {
    const double delta = sg - g * kGridH;  // exact: h is a power of two
    const double em = exp(mu);
    s_all = k_max ? em * horner(row_max, delta) : 0.0;
    if (k_a) {
      Row row_a;  // the k_alpha row of grid point g: shared by the whole queue, L1-resident
      load_row(base + (size_t)k_a * kMoments, row_a);
      s_a = em * horner(row_a, delta);
    }
  } else {
    exact_sums(Ys, mu, sg, k_a, k_max, s_a, s_all);
  }
  return epilogue(p, xm, T, saturated, s_a, s_all, o);
}

// E, CVaR and score from the two partial sums and T (dist.cpp:163-189, sim.cpp:94,
// sched.cpp:19-26), operation order as the reference's (no FMA contraction).  kRecip (the
// moment-table path, whose sums are not the reference's sequential ones anyway): the two
// divisions by N and (1 - alpha) become products with host reciprocals (<= 1 ulp).
template <bool kRecip>
__device__ __forceinline__ uint32_t epilogue(const ScoreParams& p, double xm, double T,
                                             bool saturated, double s_a, double s_all, Out& o) {
  const double Nd = (double)p.N;
  const double psi_cap = kRecip ? __dmul_rn(s_all, p.inv_N) : s_all / Nd;
  const double cm = __dsub_rn(1.0, T);
  double E = __dadd_rn(psi_cap, __dmul_rn(xm, cm));
  E = (xm < E) ? xm : E;  // std::min(v, x_max)
  double C;
  if (saturated) {
    C = xm;
  } else {
    const double psi_a = p.alpha > 0.0 ? (kRecip ? __dmul_rn(s_a, p.inv_N) : s_a / Nd) : 0.0;
    const double num = __dadd_rn(__dsub_rn(psi_cap, psi_a), __dmul_rn(xm, cm));
    const double v = kRecip ? __dmul_rn(num, p.inv_1ma) : num / __dsub_rn(1.0, p.alpha);
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

// keys != nullptr: also emit the rank key (order-preserving u64 image of the score, as in
// rank.cu) and, with minmax != nullptr, fold the key range into minmax[0] (max of ~key) and
// minmax[1] (max key) -- the bucket sort's range, so the fused score+rank path needs no
// separate pass over the keys before bucketing.
template <typename XT, bool kExact>
__global__ void __launch_bounds__(256, 2) score_kernel(const __grid_constant__ ScoreParams p,
                                                    const double* __restrict__ mu,
                                                    const double* __restrict__ sigma,
                                                    const XT* __restrict__ xmax, uint64_t n,
                                                    double* __restrict__ E, double* __restrict__ C,
                                                    double* __restrict__ S,
                                                    uint64_t* __restrict__ keys,
                                                    unsigned long long* __restrict__ minmax) {
  extern __shared__ double sY[];
  const double* Ys = p.Y;
  if (kExact && p.N <= 12288) {  // stage the sample set once per CTA (<= 96 KB)
    for (int i = threadIdx.x; i < p.N; i += blockDim.x) sY[i] = p.Y[i];
    Ys = sY;
  }
  __syncthreads();
  LogMemo lnx;
  uint64_t kmin = ~0ull, kmax = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // software pipeline: the next request's inputs are loaded while this one is scored
  double nmu = 0.0, nsg = 0.0, nxm = 0.0;
  if (i < n) {
    nmu = mu[i];
    nsg = sigma[i];
    nxm = (double)xmax[i];
  }
  for (; i < n; i += stride) {
    const double cmu = nmu, csg = nsg, cxm = nxm;
    if (i + stride < n) {
      nmu = mu[i + stride];
      nsg = sigma[i + stride];
      nxm = (double)xmax[i + stride];
    }
    Out o;
    const uint32_t why = score_one<kExact>(p, Ys, cmu, csg, cxm, lnx, o);
    if (why != kOk) {
      report(p.err, p.index_base + i, why);
      o.E = o.C = o.S = __longlong_as_double(0x7ff8000000000000LL);
    }
    if (E) E[i] = o.E;
    if (C) C[i] = o.C;
    if (S) S[i] = o.S;
    if (keys) {
      const uint64_t k =
          why == kOk ? ((uint64_t)__double_as_longlong(o.S) | (1ull << 63)) : ~0ull;
      keys[i] = k;
      kmin = k < kmin ? k : kmin;
      kmax = k > kmax ? k : kmax;
    }
  }
  if (minmax) key_range_flush(minmax, kmin, kmax);
}

// ------------------------------------------------------------------ warp-cooperative path
// Moment-table path with one warp per 32 consecutive requests.  The per-request table rows
// (128-byte moment rows at k_max and k_alpha, 64-byte tail-mass row) are random gathers; a
// per-lane 16-byte load touches 32 different lines per warp instruction (1/8 of each L1
// wavefront useful), which made L1 wavefronts the score kernel's limiter.  Here the warp
// stages rows cooperatively -- consecutive lanes fetch consecutive 16-byte chunks of the
// same row, then each lane reads its own row from a padded shared-memory slab (stride
// R+2 doubles: conflict-free 16-byte reads) -- ~3 wavefronts per row instead of 8.
constexpr int kSlabStride = kMoments + 2;  // doubles per staged row (padding vs banks)

// Rare paths kept out of line so they do not inflate the hot loop's register allocation.
__device__ __noinline__ double t_cdf_slow(const TdistConst& td, double y) {
  return t_cdf_dev(td, y);
}
__device__ __noinline__ void exact_sums_slow(const double* __restrict__ Y, double mu, double sg,
                                             uint32_t k_a, uint32_t k_max, double* s_a,
                                             double* s_all) {
  exact_sums(Y, mu, sg, k_a, k_max, *s_a, *s_all);
}

// the exact-sum fallback of the pipelined kernel (rare: outside the sigma grid or |mu| > 700)
struct OutW {
  double E, C, S;
  uint32_t why;
};
__device__ __noinline__ OutW exact_epilogue_slow(const ScoreParams& p, double m, double sg,
                                                 uint32_t k_a, uint32_t k_max, double xm,
                                                 double T, bool saturated) {
  double s_a = 0.0, s_all = 0.0;
  exact_sums(p.Y, m, sg, k_a, k_max, s_a, s_all);
  Out o;
  OutW w;
  w.why = epilogue<false>(p, xm, T, saturated, s_a, s_all, o);
  w.E = o.E;
  w.C = o.C;
  w.S = o.S;
  return w;
}

template <int R>
__device__ __forceinline__ void stage_rows(const double* myrow, double* slab,
                                           const double** ptrs) {
  const int lane = threadIdx.x & 31;
  ptrs[lane] = myrow;
  __syncwarp();
  constexpr int C = R / 2;  // 16-byte chunks per row
#pragma unroll
  for (int it = 0; it < C; ++it) {
    const int c = it * 32 + lane;
    const int r = c / C, sub = c % C;
    const double* rp = ptrs[r];
    const double2 v = rp ? __ldg(reinterpret_cast<const double2*>(rp) + sub)
                         : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(slab + r * kSlabStride + 2 * sub) = v;
  }
  __syncwarp();
}

// The same staging with cp.async (LDGSTS): global -> shared without a register round trip.
// Null rows are skipped (their slab slot holds stale data the caller never uses).
template <int R>
__device__ __forceinline__ void stage_rows_async(const double* myrow, double* slab,
                                                 const double** ptrs) {
  const int lane = threadIdx.x & 31;
  ptrs[lane] = myrow;
  __syncwarp();
  constexpr int C = R / 2;
#pragma unroll
  for (int it = 0; it < C; ++it) {
    const int c = it * 32 + lane;
    const int r = c / C, sub = c % C;
    const double* rp = ptrs[r];
    if (rp) {
      const unsigned dst =
          (unsigned)__cvta_generic_to_shared(slab + r * kSlabStride + 2 * sub);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                   "l"(reinterpret_cast<const double2*>(rp) + sub));
    }
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncwarp();
}

template <int R>
__device__ __forceinline__ double slab_horner(const double* slab, double x) {
  const int lane = threadIdx.x & 31;
  const double2* row = reinterpret_cast<const double2*>(slab + lane * kSlabStride);
  double2 c = row[R / 2 - 1];
  double acc = fma(c.y, x, c.x);
#pragma unroll
  for (int j = R / 2 - 2; j >= 0; --j) {
    c = row[j];
    acc = fma(acc, x, c.y);
    acc = fma(acc, x, c.x);
  }
  return acc;
}

template <int R>
__device__ __forceinline__ double smem_horner(const double* row, double x) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
  double2 c = r2[R / 2 - 1];
  double acc = fma(c.y, x, c.x);
#pragma unroll
  for (int j = R / 2 - 2; j >= 0; --j) {
    c = r2[j];
    acc = fma(acc, x, c.y);
    acc = fma(acc, x, c.x);
  }
  return acc;
}

// k = #{Y_i <= y} for Y[0] <= y < Y[N-1] from a staged sample-bin entry
__device__ __noinline__ uint32_t bin_search_slow(const double* __restrict__ Y, uint32_t lo,
                                                 uint32_t hi, double y) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (y < Y[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t bin_cut(const ScoreParams& p, const double* ent, double y) {
  const uint64_t head = (uint64_t)__double_as_longlong(ent[0]);
  const uint32_t kstart = (uint32_t)head, cnt = (uint32_t)(head >> 32);
  uint32_t k = kstart;
#pragma unroll
  for (int j = 0; j < kBinInline; ++j) k += ent[1 + j] <= y ? 1u : 0u;  // pads are +inf
  if (cnt > (uint32_t)kBinInline && k == kstart + kBinInline)
    k = bin_search_slow(p.Y, kstart + kBinInline, kstart + cnt, y);
  return k;
}

// Default score kernel (moment tables).  Persistent CTAs, one warp per 32 consecutive
// requests; per request the dependent chain is
//   inputs (prefetched one iteration ahead) -> y_max -> {tail-mass row, sample-bin entry}
//   (one staged round of gathers) -> moment row at k_max (one staged gather) -> epilogue,
// with the k_alpha rows of every sigma grid point (request-invariant) resident in shared
// memory for the whole kernel.
constexpr int kKaMaxG = 320;  // grid points whose k_alpha rows fit the smem budget

template <typename XT, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) score_coop_kernel(const __grid_constant__ ScoreParams p,
                                                         const double* __restrict__ mu,
                                                         const double* __restrict__ sigma,
                                                         const XT* __restrict__ xmax, uint64_t n,
                                                         double* __restrict__ E,
                                                         double* __restrict__ C,
                                                         double* __restrict__ S,
                                                         uint64_t* __restrict__ keys,
                                                         unsigned long long* __restrict__ minmax) {
  __shared__ __align__(16) double slab_all[8][32 * kSlabStride];
  __shared__ const double* ptr_all[8][32];
  extern __shared__ __align__(16) double ka_rows[];  // [G][kSlabStride] when G <= kKaMaxG
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* slab = slab_all[wib];
  const double** ptrs = ptr_all[wib];
  const bool ka_smem = p.ka_smem && p.G <= kKaMaxG && p.k_alpha > 0;
  if (ka_smem) {  // the per-alpha k_alpha rows are one contiguous table: coalesced loads,
                  // all in flight before the first store
    constexpr int kU = 8;  // 8 x 256 x 16 B = 32 KB >= G_max(320) x 96 B
    const int nc = p.G * (kMoments / 2);
    double2 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = threadIdx.x + u * 256;
      v[u] = c < nc ? __ldg(reinterpret_cast<const double2*>(p.ka_table) + c)
                    : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int c = threadIdx.x + u * 256;
      if (c < nc) {
        const int g = c / (kMoments / 2), sub = c % (kMoments / 2);
        *reinterpret_cast<double2*>(ka_rows + g * kSlabStride + 2 * sub) = v[u];
      }
    }
  }
  __syncthreads();
  // a programmatic dependent (the scheduler step's apply kernel) may launch now: it waits
  // for this grid's completion before reading E / C
  cudaTriggerProgrammaticLaunchCompletion();
  LogMemo lnx;
  uint64_t kmin = ~0ull, kmax = 0;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint64_t base = warp0 * 32;
  // the next iteration's inputs are prefetched raw (converted only when used, so the
  // conversion does not wait on the load)
  double nm = 0.0, nsig = 1.0;
  XT nxm = (XT)1;
  if (base + lane < n) {
    nm = mu[base + lane];
    nsig = sigma[base + lane];
    nxm = xmax[base + lane];
  }
  for (; base < n; base += nwarps * 32) {  // warp-uniform loop
    const uint64_t i = base + lane;
    const bool active = i < n;
    const double m = nm, sig = nsig, xm = (double)nxm;
    {  // prefetch the next iteration's inputs
      const uint64_t j = i + nwarps * 32;
      if (j < n) {
        nm = mu[j];
        nsig = sigma[j];
        nxm = xmax[j];
      }
    }
    // LogTParams / CensoredLogT validation (dist.cpp:108-120)
    uint32_t why = kOk;
    if (!isfinite(m)) why = kMuNotFinite;
    else if (!(sig > 0.0) || !isfinite(sig)) why = kSigmaBad;
    else if (!(xm > 0.0) || !isfinite(xm)) why = kXmaxBad;
    const bool ok = active && why == kOk;
    const double sg = ok ? (sig < 1e-9 ? 1e-9 : sig) : 1.0;
    const double y_max = ok ? __dsub_rn(lnx(xm), m) / sg : 0.0;
    // round 1: the sample-bin entry of y_max -> k_max and T(y_max) (one 96-byte gather)
    const uint64_t ybits = (uint64_t)__double_as_longlong(y_max);
    const bool binned = ok && fabs(y_max) < p.bin_ylim;
    stage_rows_async<kBinEntry>(
        binned ? p.bins + (size_t)sample_bin(ybits, p.bin_e0, p.bin_m, p.bin_mid) * kBinEntry
               : nullptr,
        slab, ptrs);
    const double* my = slab + lane * kSlabStride;
    double T = 0.5;
    uint32_t k_max = 0;
    if (binned) {
      const double c = __longlong_as_double(
          (long long)sample_bin_centre_bits(ybits, p.bin_e0, p.bin_m));
      const double v = smem_horner<kBinCoef>(my + kBinTail, __dsub_rn(fabs(y_max), c));
      T = y_max >= 0.0 ? __dsub_rn(1.0, v) : v;  // dist.cpp:80
      k_max = bin_cut(p, my, y_max);
    } else if (ok) {  // |y_max| beyond the bins: continued fraction, cut at the sample ends
      T = t_cdf_slow(p.td, y_max);
      k_max = y_max >= p.yN ? (uint32_t)p.N
                            : (y_max < p.y0 ? 0u : bin_search_slow(p.Y, 0, p.N, y_max));
    }
    const int g = ok ? __double2int_rn(sg * kGridInvH) : 0;
    const double delta = sg - g * kGridH;  // exact: h is a power of two
    const double reach = fmax(p.taylor_y0, fmin(fmax(y_max, 0.0), p.yN));
    const bool use_table =
        ok && g < p.G && fabs(m) <= 700.0 && fabs(delta) * reach <= kTaylorReach;
    const double* gbase = p.table + (size_t)(use_table ? g : 0) * (size_t)(p.N + 1) * kMoments;
    const bool saturated = p.alpha >= T;  // censored_cvar case 1 (dist.cpp:187)
    const uint32_t k_a = saturated ? 0u : p.k_alpha;
    __syncwarp();
    // round 2: the moment row at k_max
    stage_rows_async<kMoments>(use_table && k_max ? gbase + (size_t)k_max * kMoments : nullptr,
                               slab, ptrs);
    const double F_all = slab_horner<kMoments>(slab, delta);
    __syncwarp();
    double F_a = 0.0;
    if (use_table && k_a) {
      if (ka_smem) {
        F_a = smem_horner<kMoments>(ka_rows + g * kSlabStride, delta);
      } else {
        Row row_a;
        load_row(gbase + (size_t)k_a * kMoments, row_a);
        F_a = horner(row_a, delta);
      }
    }
    Out o;
    if (ok) {
      double s_a = 0.0, s_all = 0.0;
      if (use_table) {
        const double em = exp(m);
        s_all = k_max ? em * F_all : 0.0;
        s_a = k_a ? em * F_a : 0.0;
        why = epilogue<true>(p, xm, T, saturated, s_a, s_all, o);
      } else {
        exact_sums_slow(p.Y, m, sg, k_a, k_max, &s_a, &s_all);
        why = epilogue<false>(p, xm, T, saturated, s_a, s_all, o);
      }
    }
    if (!active) continue;
    if (why != kOk) {
      report(p.err, p.index_base + i, why);
      o.E = o.C = o.S = __longlong_as_double(0x7ff8000000000000LL);
    }
    if (E) E[i] = o.E;
    if (C) C[i] = o.C;
    if (S) S[i] = o.S;
    if (keys) {
      const uint64_t k =
          why == kOk ? ((uint64_t)__double_as_longlong(o.S) | (1ull << 63)) : ~0ull;
      keys[i] = k;
      kmin = k < kmin ? k : kmin;
      kmax = k > kmax ? k : kmax;
    }
  }
  if (minmax) key_range_flush(minmax, kmin, kmax);
}

// ------------------------------------------------------------------ pipelined path (A/B)
// The moment-table path as a three-stage software pipeline per warp:
//   S1(j): block j's inputs -> y_max -> its 96-byte sample-bin rows in flight (into bslab)
//   S2(j): T(y_max), k_max, grid point from bslab -> the moment rows in flight (mslab[j & 1])
//   S3(j): the two Horner sums from mslab[j & 1], E / CVaR / score, stores
// issued as S2(j), S1(j+1), S3(j-1) in one loop body behind ONE wait for the copies issued by
// the previous body, so both gathers of a body overlap the previous block's S3 (ncu on the
// two-wait cooperative kernel: 18 % of the stall samples on the LDGSTS wait).  Rows are
// gathered cooperatively (consecutive lanes copy consecutive 16-byte chunks of one row with
// LDGSTS, ~6 lines per warp instruction instead of 32); the row pointers are exchanged with
// shuffles.  (Per-lane TMA bulk copies of the same rows measured 2.3x slower: ~14 SM cycles
// per 96-byte bulk copy.)  One 512-thread CTA per SM: 16 warps x 3 slabs + the k_alpha rows.
constexpr int kPipeThreads = 512;
constexpr int kPipeWarps = kPipeThreads / 32;
constexpr int kSlabDoubles = 32 * kSlabStride;
static_assert(kBinEntry == kMoments, "bin and moment rows share the slab layout");

// every lane's row (nullptr: none) into its slot of `slab`: LDGSTS, committed as one group
__device__ __forceinline__ void coop_issue(const double* row, double* slab) {
  const int lane = threadIdx.x & 31;
  constexpr int C = kMoments / 2;  // 16-byte chunks per row
  const unsigned long long mine = (unsigned long long)row;
#pragma unroll
  for (int it = 0; it < C; ++it) {
    const int c = it * 32 + lane;
    const int r = c / C, sub = c - r * C;
    const double* rp = (const double*)__shfl_sync(0xffffffffu, mine, r);
    if (rp) {
      const unsigned dst =
          (unsigned)__cvta_generic_to_shared(slab + r * kSlabStride + 2 * sub);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                   "l"(reinterpret_cast<const double2*>(rp) + sub)
                   : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void coop_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
}

struct PipeA {  // after S1
  uint64_t i;
  double m, sg, xm, y_max;
  uint32_t why;
  bool active, ok, binned;
};

struct PipeB {  // after S2
  uint64_t i;
  double m, xm, T, delta, sg;
  uint32_t why, k_max, k_a;
  int g;
  bool active, ok, use_table, saturated;
};

// S1: inputs of the lane's request in block `base` -> y_max -> bin rows in flight
__device__ __forceinline__ PipeA pipe_s1(const ScoreParams& p, uint64_t n, uint64_t base,
                                         double m, double sig, double xm, LogMemo& lnx,
                                         double* bslab) {
  PipeA a;
  a.i = base + (threadIdx.x & 31);
  a.active = a.i < n;
  a.why = kOk;
  if (!isfinite(m)) a.why = kMuNotFinite;  // LogTParams / CensoredLogT (dist.cpp:108-120)
  else if (!(sig > 0.0) || !isfinite(sig)) a.why = kSigmaBad;
  else if (!(xm > 0.0) || !isfinite(xm)) a.why = kXmaxBad;
  a.ok = a.active && a.why == kOk;
  a.m = m;
  a.xm = xm;
  a.sg = a.ok ? (sig < 1e-9 ? 1e-9 : sig) : 1.0;
  a.y_max = a.ok ? __dsub_rn(lnx(xm), m) / a.sg : 0.0;
  a.binned = a.ok && fabs(a.y_max) < p.bin_ylim;
  const uint64_t ybits = (uint64_t)__double_as_longlong(a.y_max);
  coop_issue(a.binned ? p.bins + (size_t)sample_bin(ybits, p.bin_e0, p.bin_m, p.bin_mid) *
                                     kBinEntry
                      : nullptr,
             bslab);
  return a;
}

// S2: T, k_max and the grid point from the (landed) bin rows -> moment rows in flight
__device__ __forceinline__ PipeB pipe_s2(const ScoreParams& p, const PipeA& a,
                                         const double* bslab, double* mslab) {
  PipeB b;
  b.i = a.i;
  b.active = a.active;
  b.ok = a.ok;
  b.why = a.why;
  b.m = a.m;
  b.xm = a.xm;
  b.sg = a.sg;
  const double* my = bslab + (threadIdx.x & 31) * kSlabStride;
  b.T = 0.5;
  b.k_max = 0;
  const double y_max = a.y_max;
  if (a.binned) {
    const uint64_t ybits = (uint64_t)__double_as_longlong(y_max);
    const double c =
        __longlong_as_double((long long)sample_bin_centre_bits(ybits, p.bin_e0, p.bin_m));
    const double v = smem_horner<kBinCoef>(my + kBinTail, __dsub_rn(fabs(y_max), c));
    b.T = y_max >= 0.0 ? __dsub_rn(1.0, v) : v;  // dist.cpp:80
    b.k_max = bin_cut(p, my, y_max);
  } else if (a.ok) {  // |y_max| beyond the bins: continued fraction, cut at the sample ends
    b.T = t_cdf_slow(p.td, y_max);
    b.k_max = y_max >= p.yN ? (uint32_t)p.N
                            : (y_max < p.y0 ? 0u : bin_search_slow(p.Y, 0, p.N, y_max));
  }
  __syncwarp();  // every lane is done with bslab before S1 refills it
  b.g = a.ok ? __double2int_rn(a.sg * kGridInvH) : 0;
  b.delta = a.sg - b.g * kGridH;  // exact: h is a power of two
  const double reach = fmax(p.taylor_y0, fmin(fmax(y_max, 0.0), p.yN));
  b.use_table =
      a.ok && b.g < p.G && fabs(a.m) <= 700.0 && fabs(b.delta) * reach <= kTaylorReach;
  b.saturated = p.alpha >= b.T;  // censored_cvar case 1 (dist.cpp:187)
  b.k_a = b.saturated ? 0u : p.k_alpha;
  const double* gbase =
      p.table + (size_t)(b.use_table ? b.g : 0) * (size_t)(p.N + 1) * kMoments;
  coop_issue(b.use_table && b.k_max ? gbase + (size_t)b.k_max * kMoments : nullptr, mslab);
  return b;
}

// S3: Horner sums from the (landed) moment rows, epilogue, stores
__device__ __forceinline__ void pipe_s3(const ScoreParams& p, const PipeB& b,
                                        const double* mslab, const double* ka_rows,
                                        bool ka_smem, double* __restrict__ E,
                                        double* __restrict__ C, double* __restrict__ S,
                                        uint64_t* __restrict__ keys, uint64_t& kmin,
                                        uint64_t& kmax) {
  const double F_all = slab_horner<kMoments>(mslab, b.delta);
  double F_a = 0.0;
  if (b.use_table && b.k_a) {
    if (ka_smem) {
      F_a = smem_horner<kMoments>(ka_rows + b.g * kSlabStride, b.delta);
    } else {
      Row row_a;
      load_row(p.table + ((size_t)b.g * (size_t)(p.N + 1) + b.k_a) * kMoments, row_a);
      F_a = horner(row_a, b.delta);
    }
  }
  __syncwarp();  // every lane is done with this mslab before S2 refills it
  Out o;
  uint32_t why = b.why;
  if (b.ok) {
    if (b.use_table) {
      const double em = exp(b.m);
      const double s_all = b.k_max ? em * F_all : 0.0;
      const double s_a = b.k_a ? em * F_a : 0.0;
      why = epilogue<true>(p, b.xm, b.T, b.saturated, s_a, s_all, o);
    } else {
      const OutW w = exact_epilogue_slow(p, b.m, b.sg, b.k_a, b.k_max, b.xm, b.T, b.saturated);
      why = w.why;
      o.E = w.E;
      o.C = w.C;
      o.S = w.S;
    }
  }
  if (!b.active) return;
  if (why != kOk) {
    report(p.err, p.index_base + b.i, why);
    o.E = o.C = o.S = __longlong_as_double(0x7ff8000000000000LL);
  }
  if (E) E[b.i] = o.E;
  if (C) C[b.i] = o.C;
  if (S) S[b.i] = o.S;
  if (keys) {
    const uint64_t k = why == kOk ? ((uint64_t)__double_as_longlong(o.S) | (1ull << 63)) : ~0ull;
    keys[b.i] = k;
    kmin = k < kmin ? k : kmin;
    kmax = k > kmax ? k : kmax;
  }
}

template <typename XT>
__global__ void __launch_bounds__(kPipeThreads, 1) score_pipe_kernel(
    const __grid_constant__ ScoreParams p, const double* __restrict__ mu,
    const double* __restrict__ sigma, const XT* __restrict__ xmax, uint64_t n,
    double* __restrict__ E, double* __restrict__ C, double* __restrict__ S,
    uint64_t* __restrict__ keys, unsigned long long* __restrict__ minmax) {
  extern __shared__ __align__(128) double pipe_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* bslab = pipe_smem + (size_t)wib * 3 * kSlabDoubles;
  double* mslab0 = bslab + kSlabDoubles;
  double* mslab1 = mslab0 + kSlabDoubles;
  double* ka_rows = pipe_smem + (size_t)kPipeWarps * 3 * kSlabDoubles;
  const bool ka_smem = p.ka_smem && p.G <= kKaMaxG && p.k_alpha > 0;
  if (ka_smem) {
    const int nc = p.G * (kMoments / 2);
    for (int c = threadIdx.x; c < nc; c += kPipeThreads) {
      const int g = c / (kMoments / 2), sub = c % (kMoments / 2);
      *reinterpret_cast<double2*>(ka_rows + g * kSlabStride + 2 * sub) =
          __ldg(reinterpret_cast<const double2*>(p.ka_table) + c);
    }
  }
  __syncthreads();
  LogMemo lnx;
  uint64_t kmin = ~0ull, kmax = 0;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t step = ((uint64_t)gridDim.x * blockDim.x >> 5) * 32;
  uint64_t base = warp0 * 32;
  if (base < n) {
    // raw inputs one block ahead (converted when used)
    double m0 = 0.0, s0 = 1.0, nm = 0.0, nsig = 1.0;
    XT x0 = (XT)1, nxm = (XT)1;
    if (base + lane < n) {
      m0 = mu[base + lane];
      s0 = sigma[base + lane];
      x0 = xmax[base + lane];
    }
    if (base + step + lane < n) {
      nm = mu[base + step + lane];
      nsig = sigma[base + step + lane];
      nxm = xmax[base + step + lane];
    }
    PipeA a = pipe_s1(p, n, base, m0, s0, (double)x0, lnx, bslab);
    PipeB b;
    bool have_b = false;
    bool odd = false;  // block parity j & 1
    // body j: S3(j-1) [its moment rows: the older of the two groups in flight], S2(j) [the
    // bin rows: the newer group], S1(j+1) -- at most two blocks' state live at a time
    for (; base < n; base += step, odd = !odd) {
      if (have_b) {  // S3(j-1)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        pipe_s3(p, b, odd ? mslab0 : mslab1, ka_rows, ka_smem, E, C, S, keys, kmin, kmax);
      }
      coop_wait_all();
      b = pipe_s2(p, a, bslab, odd ? mslab1 : mslab0);  // S2(j)
      have_b = true;
      const uint64_t nbase = base + step;
      if (nbase < n) {  // S1(j+1)
        const double cm = nm, cs = nsig, cx = (double)nxm;
        const uint64_t i2 = nbase + step + lane;
        if (i2 < n) {
          nm = mu[i2];
          nsig = sigma[i2];
          nxm = xmax[i2];
        }
        a = pipe_s1(p, n, nbase, cm, cs, cx, lnx, bslab);
      }
    }
    coop_wait_all();  // S3 of the last block (parity !odd)
    pipe_s3(p, b, odd ? mslab0 : mslab1, ka_rows, ka_smem, E, C, S, keys, kmin, kmax);
  }
  if (minmax) key_range_flush(minmax, kmin, kmax);
}

// k_alpha rows of every grid point into one contiguous [G][kMoments] table (once per alpha)
__global__ void gather_ka_rows_kernel(const double* __restrict__ table, int G, int N,
                                      uint32_t k_alpha, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < G * kMoments;
       c += gridDim.x * blockDim.x) {
    const int g = c / kMoments, m = c % kMoments;
    out[c] = table[((size_t)g * (N + 1) + k_alpha) * kMoments + m];
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
  ctx->table_bytes = sizeof(double) * std::max(N, 1);
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
  ctx->table_bytes += sizeof(uint32_t) * yb.size();
  if ((e = cudaMemcpy(ctx->d_ybucket, yb.data(), sizeof(uint32_t) * yb.size(),
                      cudaMemcpyHostToDevice)) != cudaSuccess)
    return e;
  // Taylor coefficients of v(|y|) = 1 - T(|y|) about c >= 0 (tail table and sample bins):
  // a_0 = v(c) by the reference's own continued fraction, a_j = -pdf^(j-1)(c)/j! from the
  // power series of pdf(c + t) = C (q0 + q1 t + q2 t^2)^ex  (q f' = ex q' f)
  const long double nu_l = ctx->nu;
  const long double ex_l = -0.5L * (nu_l + 1.0L);
  const long double C_l = std::exp((long double)std::lgamma(0.5 * (ctx->nu + 1.0)) -
                                   (long double)std::lgamma(0.5 * ctx->nu) -
                                   0.5L * std::log(nu_l * 3.14159265358979323846264338327950288L));
  auto tail_coefs = [&](double c, int ncoef, double* row) {
    const double x = ctx->nu / (c * c + ctx->nu);
    row[0] = 0.5 * host::reg_inc_beta(0.5 * ctx->nu, 0.5, x);
    const long double q[3] = {1.0L + (long double)c * c / nu_l, 2.0L * c / nu_l, 1.0L / nu_l};
    long double f[16];
    f[0] = C_l * std::pow(q[0], ex_l);
    for (int k = 1; k < ncoef; ++k) {
      long double acc = 0.0L;
      for (int i = 1; i <= std::min(k, 2); ++i) acc += (ex_l * i - (k - i)) * q[i] * f[k - i];
      f[k] = acc / (k * q[0]);
    }
    for (int j = 1; j < ncoef; ++j) row[j] = (double)(-f[j - 1] / j);  // v' = -pdf
  };
  // sample bins (kBinEntry in tie_internal.cuh)
  {
    auto bits = [](double x) {
      uint64_t u;
      std::memcpy(&u, &x, 8);
      return u;
    };
    auto dbl = [](uint64_t u) {
      double x;
      std::memcpy(&x, &u, 8);
      return x;
    };
    const double maxabs = std::max(std::fabs(Y.front()), std::fabs(Y.back()));
    // cover at least |y| < 2^8 (y_max beyond the samples: small sigma), never more than 2^30
    const uint32_t etop = std::min<uint32_t>(
        std::max<uint32_t>((uint32_t)(bits(maxabs) >> 52) & 0x7ffu, 1023u + 7u), 1023u + 29u);
    const uint32_t e0 = 1023u - 12u;
    uint32_t m = 11;
    while (m > 4 && ((uint64_t)(etop - e0 + 1) << m) > (1u << 20)) --m;
    ctx->bin_e0 = e0;
    ctx->bin_m = m;
    ctx->bin_mid = (etop - e0 + 1) << m;
    ctx->bin_ylim = dbl((uint64_t)(etop + 1) << 52);
    const size_t nbins = 2 * (size_t)ctx->bin_mid + 1;
    std::vector<uint32_t> cnt(nbins, 0), first(nbins, 0);
    for (int i = N - 1; i >= 0; --i) {
      if (!(std::fabs(Y[i]) < ctx->bin_ylim)) continue;  // beyond the bins: never a cut inside
      const uint32_t b = sample_bin(bits(Y[i]), e0, m, ctx->bin_mid);
      ++cnt[b];
      first[b] = (uint32_t)i;  // ascending Y: the lowest index of the bin
    }
    std::vector<double> ent(nbins * kBinEntry, std::numeric_limits<double>::infinity());
    uint32_t before = 0;
    for (int i = 0; i < N && Y[i] <= -ctx->bin_ylim; ++i) ++before;  // samples below the bins
    for (size_t b = 0; b < nbins; ++b) {
      double* row = &ent[b * kBinEntry];
      const uint64_t head = (uint64_t)before | ((uint64_t)cnt[b] << 32);
      std::memcpy(row, &head, 8);
      for (uint32_t j = 0; j < std::min<uint32_t>(cnt[b], kBinInline); ++j)
        row[1 + j] = Y[first[b] + j];
      before += cnt[b];
      // centre of the bin's |y| range (the device derives the same value from y's bits)
      double c = 0.0;
      if (b != ctx->bin_mid) {
        const uint64_t off = b > ctx->bin_mid ? b - ctx->bin_mid - 1 : ctx->bin_mid - 1 - b;
        const uint64_t e = e0 + (off >> m), j = off & ((1u << m) - 1u);
        c = dbl(sample_bin_centre_bits((e << 52) | (j << (52 - m)), e0, m));
      }
      tail_coefs(c, kBinCoef, row + kBinTail);
    }
    if ((e = cudaMalloc(&ctx->d_bins, sizeof(double) * ent.size())) != cudaSuccess) return e;
    ctx->table_bytes += sizeof(double) * ent.size();
    if ((e = cudaMemcpy(ctx->d_bins, ent.data(), sizeof(double) * ent.size(),
                        cudaMemcpyHostToDevice)) != cudaSuccess)
      return e;
  }
  // tail-mass Taylor table (exact / per-lane paths; kTailBuckets in tie_internal.cuh)
  {
    const double ymax = std::max(std::fabs(ctx->y0), std::fabs(ctx->yN));
    ctx->t_ymax = ymax > 0.0 ? ymax : 0.0;
    ctx->t_w = ctx->t_ymax / kTailBuckets;
    ctx->t_inv_w = ctx->t_w > 0.0 ? 1.0 / ctx->t_w : 0.0;
    std::vector<double> tt((size_t)kTailBuckets * kTailCoef, 0.0);
    for (int b = 0; b < kTailBuckets && ctx->t_w > 0.0; ++b)
      tail_coefs(((double)b + 0.5) * ctx->t_w, kTailCoef, tt.data() + (size_t)b * kTailCoef);
    if ((e = cudaMalloc(&ctx->d_tail, sizeof(double) * tt.size())) != cudaSuccess) return e;
    ctx->table_bytes += sizeof(double) * tt.size();
    if ((e = cudaMemcpy(ctx->d_tail, tt.data(), sizeof(double) * tt.size(),
                        cudaMemcpyHostToDevice)) != cudaSuccess)
      return e;
  }
  // sigma-grid moment tables
  ctx->G = (int)std::lrint(ctx->sigma_table_max * kGridInvH) + 1;
  const size_t bytes = (size_t)ctx->G * (size_t)(N + 1) * kMoments * sizeof(double);
  if ((e = cudaMalloc(&ctx->d_table, bytes)) != cudaSuccess) return e;
  ctx->table_bytes += bytes;
  build_moment_table_kernel<<<ctx->G, 512>>>(ctx->d_Y, N, ctx->d_table);
  capi::count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

cudaError_t launch_score(tie_ctx* ctx, const double* mu, const double* sigma, const void* x_max,
                         bool x_is_u32, uint64_t n, double alpha, double beta, double* E,
                         double* C, double* S, uint64_t* keys_out, unsigned long long* minmax,
                         unsigned flags, cudaStream_t s, uint64_t index_base) {
  const bool exact = (flags & 1u) != 0;
  if (n == 0) return cudaSuccess;
  ScoreParams p;
  p.td = ctx->td;
  p.Y = ctx->d_Y;
  p.ybucket = ctx->d_ybucket;
  p.table = ctx->d_table;
  p.tail = ctx->d_tail;
  p.bins = ctx->d_bins;
  p.bin_e0 = ctx->bin_e0;
  p.bin_m = ctx->bin_m;
  p.bin_mid = ctx->bin_mid;
  p.bin_ylim = ctx->bin_ylim;
  p.taylor_y0 = std::fabs(ctx->y0);
  p.inv_N = ctx->N > 0 ? 1.0 / (double)ctx->N : 0.0;
  p.inv_1ma = 1.0 / (1.0 - alpha);
  p.t_ymax = ctx->t_ymax;
  p.t_w = ctx->t_w;
  p.t_inv_w = ctx->t_inv_w;
  p.y0 = ctx->y0;
  p.y_scale = ctx->y_scale;
  p.yN = ctx->yN;
  p.N = ctx->N;
  p.G = ctx->G;
  p.alpha = alpha;
  p.beta = beta;
  p.raw = (flags & 2u) ? 1 : 0;
  p.index_base = index_base;
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
  if (ctx->ka_table_k != ctx->ka_k || !ctx->d_ka_table) {  // contiguous k_alpha rows
    if (!ctx->d_ka_table) {
      const cudaError_t e = cudaMalloc(&ctx->d_ka_table, sizeof(double) * kMoments *
                                                             std::max(ctx->G, 1));
      if (e != cudaSuccess) return e;
    }
    if (ctx->G > 0)
      gather_ka_rows_kernel<<<(ctx->G * kMoments + 255) / 256, 256, 0, s>>>(
          ctx->d_table, ctx->G, ctx->N, ctx->ka_k, ctx->d_ka_table);
    ctx->ka_table_k = ctx->ka_k;
  }
  p.ka_table = ctx->d_ka_table;
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
          p, mu, sigma, (const uint32_t*)x_max, n, E, C, S, keys_out, minmax);
    } else {
      cudaFuncSetAttribute(score_kernel<double, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      score_kernel<double, true><<<(unsigned)grid, 256, smem, s>>>(
          p, mu, sigma, (const double*)x_max, n, E, C, S, keys_out, minmax);
    }
  } else if (flags & 4u) {  // per-lane gathers (kept for A/B measurements)
    const uint64_t grid = std::min<uint64_t>(blocks_needed, (uint64_t)sms * 8);
    if (x_is_u32)
      score_kernel<uint32_t, false><<<(unsigned)grid, 256, 0, s>>>(
          p, mu, sigma, (const uint32_t*)x_max, n, E, C, S, keys_out, minmax);
    else
      score_kernel<double, false><<<(unsigned)grid, 256, 0, s>>>(
          p, mu, sigma, (const double*)x_max, n, E, C, S, keys_out, minmax);
  } else if ((flags & 16u) && n >= 4096) {
    // pipelined variant (A/B only): one 512-thread CTA per SM.  Measured on B200 at 1M
    // requests: 44-46 us vs 42 us for the two-round cooperative kernel below (ncu: +32 %
    // instructions and 128-register spills from two blocks' state live across the stages;
    // the per-lane TMA bulk-copy version of it: 97 us)
    p.ka_smem = ctx->G <= kKaMaxG ? 1 : 0;
    const size_t smem = sizeof(double) * ((size_t)kPipeWarps * 3 * kSlabDoubles +
                                          (p.ka_smem ? (size_t)kSlabStride * ctx->G : 0));
    static bool pattr = false;
    if (!pattr) {
      const int mx = (int)(sizeof(double) * ((size_t)kPipeWarps * 3 * kSlabDoubles +
                                             (size_t)kSlabStride * kKaMaxG));
      cudaFuncSetAttribute(score_pipe_kernel<uint32_t>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(score_pipe_kernel<double>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      pattr = true;
    }
    const uint64_t grid = std::min<uint64_t>((n + kPipeThreads - 1) / kPipeThreads, (uint64_t)sms);
    if (x_is_u32)
      score_pipe_kernel<uint32_t><<<(unsigned)grid, kPipeThreads, smem, s>>>(
          p, mu, sigma, (const uint32_t*)x_max, n, E, C, S, keys_out, minmax);
    else
      score_pipe_kernel<double><<<(unsigned)grid, kPipeThreads, smem, s>>>(
          p, mu, sigma, (const double*)x_max, n, E, C, S, keys_out, minmax);
  } else {
    const int minb = (flags & 8u) ? 3 : 2;  // 2 CTAs/SM, 128 regs, no spills (A/B: 3, spills)
    const uint64_t grid = std::min<uint64_t>(blocks_needed, (uint64_t)sms * minb);
    // the k_alpha rows are staged per CTA: worth it only for batches that keep the CTAs busy
    p.ka_smem = ctx->G <= kKaMaxG && n >= 8192 ? 1 : 0;
    const size_t ka_smem = p.ka_smem ? sizeof(double) * kSlabStride * ctx->G : 0;
    static bool attr = false;
    if (!attr) {
      const int mx = (int)(sizeof(double) * kSlabStride * kKaMaxG);
      cudaFuncSetAttribute(score_coop_kernel<uint32_t, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(score_coop_kernel<double, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(score_coop_kernel<uint32_t, 3>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      cudaFuncSetAttribute(score_coop_kernel<double, 3>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
      attr = true;
    }
#define TIE_COOP(XT, MB)                                                          \
  score_coop_kernel<XT, MB><<<(unsigned)grid, 256, ka_smem, s>>>(                 \
      p, mu, sigma, (const XT*)x_max, n, E, C, S, keys_out, minmax)
    if (x_is_u32) {
      if (minb == 2) TIE_COOP(uint32_t, 2); else TIE_COOP(uint32_t, 3);
    } else {
      if (minb == 2) TIE_COOP(double, 2); else TIE_COOP(double, 3);
    }
#undef TIE_COOP
  }
  capi::count_launch();
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace tie
