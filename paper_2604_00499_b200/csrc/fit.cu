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

// BFGS state over theta = (mu, s = ln sigma) -- what a straggler hands from phase 1 to 2.
struct Bfgs {
  double th0, th1, f, g0, g1, H00, H01, H10, H11;
  int iter;
  bool converged;
};

constexpr double kSigmaFloor = 1e-6;
constexpr double kLogSigmaFloor = -13.815510557964274;  // ln(1e-6)
constexpr int kMaxIter = 500;

// Initialisation (fit.cpp:78-115).  Returns false for the degenerate point mass (o filled).
template <class R>
__device__ bool fit_init(R& r, const FitConst& c, Bfgs& st, FitOut& o) {
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
    return false;
  }
  st.th0 = mu0;
  st.th1 = log(sigma0);
  st.f = -loglik(r, c, st.th0, exp(st.th1));
  neg_grad(r, c, st.th0, st.th1, st.g0, st.g1);
  st.H00 = 1.0;
  st.H01 = 0.0;
  st.H10 = 0.0;
  st.H11 = 1.0;
  st.iter = 0;
  st.converged = false;
  return true;
}

// The BFGS loop of fit.cpp:116-166 from st.iter up to iter_end.  kWarpLS: the caller is a
// whole warp working on ONE prompt; the Armijo backtracking (fit.cpp:133-142) -- candidates
// step = 2^-ls, ls = 0..59, accept the first that satisfies the condition -- is evaluated 32
// candidates at a time, one per lane, each lane summing its likelihood in the reference's
// order; the first accepting lane (ballot) is exactly the sequential loop's exit, and if none
// accepts, ls = 59's values are the loop's final ones.  Every lane then holds identical state.
template <bool kWarpLS, class R>
__device__ void bfgs_run(R& r, const FitConst& c, Bfgs& st, int iter_end) {
  const int lane = threadIdx.x & 31;
  for (; st.iter < iter_end; ++st.iter) {
    const double g0 = st.g0, g1 = st.g1;
    const double H00_in = st.H00, H01_in = st.H01, H10_in = st.H10, H11_in = st.H11;
    if (std_max(fabs(g0), fabs(g1)) < 1e-8) {
      st.converged = true;
      return;
    }
    double p0 = -(st.H00 * g0 + st.H01 * g1), p1 = -(st.H10 * g0 + st.H11 * g1);
    double descent = p0 * g0 + p1 * g1;
    if (descent >= 0.0) {  // reset a spoiled approximation
      st.H00 = st.H11 = 1.0;
      st.H01 = st.H10 = 0.0;
      p0 = -g0;
      p1 = -g1;
      descent = -(g0 * g0 + g1 * g1);
    }
    double f_new = st.f, n0 = st.th0, n1 = st.th1;
    if (!kWarpLS) {
      double step = 1.0;
      for (int ls = 0; ls < 60; ++ls) {
        n0 = st.th0 + step * p0;
        n1 = std_max(st.th1 + step * p1, kLogSigmaFloor);
        f_new = -loglik(r, c, n0, exp(n1));
        if (isfinite(f_new) && f_new <= st.f + 1e-4 * step * descent) break;
        step *= 0.5;
      }
    } else {
      for (int batch = 0; batch < 2; ++batch) {
        const int ls = batch * 32 + lane;
        const int lsc = ls < 60 ? ls : 59;
        const double step = ldexp(1.0, -lsc);  // 0.5^ls, exact
        const double c0 = st.th0 + step * p0;
        const double c1 = std_max(st.th1 + step * p1, kLogSigmaFloor);
        const double fc = -loglik(r, c, c0, exp(c1));
        const bool ok = ls < 60 && isfinite(fc) && fc <= st.f + 1e-4 * step * descent;
        const unsigned hit = __ballot_sync(0xffffffffu, ok);
        const int src = hit ? __ffs(hit) - 1 : (batch == 1 ? 59 - 32 : -1);
        if (src >= 0) {
          n0 = __shfl_sync(0xffffffffu, c0, src);
          n1 = __shfl_sync(0xffffffffu, c1, src);
          f_new = __shfl_sync(0xffffffffu, fc, src);
          break;
        }
      }
    }
    if (!(f_new < st.f) && std_max(fabs(g0), fabs(g1)) < 1e-6) {
      st.converged = true;  // line search stalled at the numerical optimum
      return;
    }
    double q0, q1;
    neg_grad(r, c, n0, n1, q0, q1);
    const double s0 = n0 - st.th0, s1 = n1 - st.th1;
    const double y0 = q0 - g0, y1 = q1 - g1;
    const double sy = s0 * y0 + s1 * y1;
    if (sy > 1e-12) {
      const double rho = 1.0 / sy;
      const double Hy0 = st.H00 * y0 + st.H01 * y1, Hy1 = st.H10 * y0 + st.H11 * y1;
      const double yHy = y0 * Hy0 + y1 * Hy1;
      const double k = 1.0 + rho * yHy;
      // H += rho ((1 + rho y'Hy) s s' - s (Hy)' - (Hy) s')   (fit.cpp:155-160)
      st.H00 += rho * (k * s0 * s0 - s0 * Hy0 - Hy0 * s0);
      st.H01 += rho * (k * s0 * s1 - s0 * Hy1 - Hy0 * s1);
      st.H10 += rho * (k * s1 * s0 - s1 * Hy0 - Hy1 * s0);
      st.H11 += rho * (k * s1 * s1 - s1 * Hy1 - Hy1 * s1);
    }
    // Exact fixed point: the backtracked step no longer moves theta and nothing else
    // changed, so every remaining iteration of the reference loop repeats this one bit for
    // bit (each is a pure function of (theta, f, g, H)) until the 500-iteration cap.  Jump
    // there.  (Every non-converging fit in the golden sets ends this way, typically by
    // iteration ~10; the reference spends the other ~490 iterations x 60 halvings on it.)
    const bool fixed = n0 == st.th0 && n1 == st.th1 && f_new == st.f && q0 == g0 && q1 == g1 &&
                       st.H00 == H00_in && st.H01 == H01_in && st.H10 == H10_in &&
                       st.H11 == H11_in;
    st.th0 = n0;
    st.th1 = n1;
    st.f = f_new;
    st.g0 = q0;
    st.g1 = q1;
    if (fixed) {
      st.iter = kMaxIter;
      return;
    }
  }
}

// Result (fit.cpp:168-177)
template <class R>
__device__ void fit_finish(R& r, const FitConst& c, const Bfgs& st, FitOut& o) {
  o.mu = st.th0;
  o.sigma = exp(st.th1);
  o.degenerate = false;
  if (o.sigma <= kSigmaFloor) {
    o.sigma = kSigmaFloor;
    o.degenerate = true;
  }
  o.converged = st.converged;
  o.iters = st.iter;
  o.ll = loglik(r, c, o.mu, o.sigma);
}

struct FitSpill {
  Bfgs st;
  uint64_t p;
};

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
  uint64_t index_base;  // added to reported prompt indices (chunked callers)
  // stragglers: prompts still iterating after kPhase1Iters are handed to warp-per-prompt
  // phase 2 (bounded by spill_cap; beyond it a thread simply finishes the prompt itself)
  FitSpill* spill;
  uint32_t* spill_count;
  uint32_t spill_cap;
};

constexpr int kPhase1Iters = 40;

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

// one prompt on one thread, up to kPhase1Iters BFGS iterations, then spill or finish
template <class R>
__device__ __forceinline__ void fit_phase1(const FitArgs& a, R& r, uint64_t p) {
  FitOut o;
  Bfgs st;
  if (!fit_init(r, a.c, st, o)) {
    store(a, p, o);
    return;
  }
  bfgs_run<false>(r, a.c, st, kPhase1Iters);
  if (!st.converged && st.iter < kMaxIter) {
    const uint32_t slot = atomicAdd(a.spill_count, 1u);
    if (slot < a.spill_cap) {
      a.spill[slot].st = st;
      a.spill[slot].p = p;
      return;
    }
    bfgs_run<false>(r, a.c, st, kMaxIter);  // spill buffer full: finish here
  }
  fit_finish(r, a.c, st, o);
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
      report(a.err, a.index_base + p, kSampleBad);
      store_nan(a, p);
      continue;
    }
    fit_phase1(a, r, p);
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
      report(a.err, a.index_base + p, kSampleBad);
      store_nan(a, p);
      continue;
    }
    fit_phase1(a, r, p);
  }
}

// ---------------------------------------------------------------- lane-per-sample phase 1
// W lanes per prompt (W = 16 for K <= 16, else 32): lane j holds ln x_j; every likelihood /
// gradient term is computed by its own lane and the sum is accumulated by shuffling the
// terms in index order, so each lane performs exactly the reference's sequential additions
// (bit-identical) while the BFGS control flow stays uniform across the W lanes of a prompt.
template <int KT, int W>
struct LaneRow {
  static constexpr bool kStatic = true;
  double lx;       // this lane's log-sample (lanes >= KT hold 0)
  unsigned mask;   // the prompt's lanes
  __device__ __forceinline__ int size() const { return KT; }
};

// median_sorted (fit.cpp:27-30) of the KT lane values v (lane j < KT) without sorting: each
// lane's position in the sorted order is its rank by (value, lane) -- equal values share the
// value, so the element at sorted position q is exactly the value of the lane ranked q.
// Replaces two unrolled KT-round sorting networks (~3.5k instructions of kernel code, whose
// i-cache misses dominated the kernel's stalls) by KT shuffles per median.
template <int KT, int W>
__device__ __forceinline__ double lane_median(double v, int j, int grp, unsigned mask) {
  uint32_t rank = 0;
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    const double u = __shfl_sync(mask, v, i, W);
    rank += (u < v || (u == v && i < j)) ? 1u : 0u;
  }
  auto at = [&](uint32_t q) {
    const unsigned b = __ballot_sync(mask, j < KT && rank == q);
    return __shfl_sync(mask, v, (__ffs(b) - 1) - grp * W, W);
  };
  return (KT % 2) ? at(KT / 2) : 0.5 * (at(KT / 2 - 1) + at(KT / 2));
}

template <int KT, int W>
__device__ __noinline__ double loglik(LaneRow<KT, W>& r, const FitConst& c, double mu,
                                         double sigma) {
  const double lsig = log(sigma);
  const double z = (r.lx - mu) / sigma;
  const double term = c.lognorm - c.half_nu1 * log1p(z * z / c.nu) - lsig - r.lx;
  double ll = 0.0;
#pragma unroll
  for (int i = 0; i < KT; ++i) ll += __shfl_sync(r.mask, term, i, W);
  return ll;
}

template <int KT, int W>
__device__ __noinline__ void neg_grad(LaneRow<KT, W>& r, const FitConst& c, double mu,
                                         double s, double& g0, double& g1) {
  const double sigma = exp(s);
  const double z = (r.lx - mu) / sigma;
  const double w = c.nu1 * z / (c.nu + z * z);
  const double t0 = w / sigma, t1 = (w * z - 1.0) / sigma;
  double gmu = 0.0, gsg = 0.0;
#pragma unroll
  for (int i = 0; i < KT; ++i) {
    gmu += __shfl_sync(r.mask, t0, i, W);
    gsg += __shfl_sync(r.mask, t1, i, W);
  }
  g0 = -gmu;
  g1 = -gsg * sigma;
}

template <int KT>
__global__ void __launch_bounds__(128) fit_lanes_kernel(const FitArgs a) {
  constexpr int W = KT <= 16 ? 16 : 32;
  constexpr int G = 32 / W;
  const int lane = threadIdx.x & 31, grp = lane / W, j = lane % W;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  LaneRow<KT, W> r;
  r.mask = W == 32 ? 0xffffffffu : (0xffffu << (16 * grp));
  for (uint64_t base = warp * G; base < a.P; base += nwarps * G) {
    const uint64_t p = base + grp;
    if (p >= a.P) continue;
    const double v = j < KT ? a.x[p * KT + j] : 1.0;
    const bool bad = j < KT && !((v > 0.0) && isfinite(v));
    r.lx = j < KT ? log(v) : 0.0;
    if (__ballot_sync(r.mask, bad)) {  // check_samples (fit.cpp:18-25)
      if (j == 0) {
        report(a.err, a.index_base + p, kSampleBad);
        store_nan(a, p);
      }
      continue;
    }
    // fit_init (fit.cpp:78-100): median and MAD by lane ranks (the same values in every lane)
    FitOut o;
    Bfgs st;
    bool live;
    {
      const double mu0 = lane_median<KT, W>(r.lx, j, grp, r.mask);
      const double sigma0 = 1.4826 * lane_median<KT, W>(fabs(r.lx - mu0), j, grp, r.mask);
      o.degenerate = false;
      o.iters = 0;
      live = !(sigma0 < kSigmaFloor);
      if (!live) {
        o.mu = mu0;
        o.sigma = kSigmaFloor;
        o.degenerate = true;
        o.converged = true;
        o.ll = loglik(r, a.c, o.mu, o.sigma);
      } else {
        st.th0 = mu0;
        st.th1 = log(sigma0);
        st.f = -loglik(r, a.c, st.th0, exp(st.th1));
        neg_grad(r, a.c, st.th0, st.th1, st.g0, st.g1);
        st.H00 = 1.0;
        st.H01 = 0.0;
        st.H10 = 0.0;
        st.H11 = 1.0;
        st.iter = 0;
        st.converged = false;
      }
    }
    if (live) {
      bfgs_run<false>(r, a.c, st, kPhase1Iters);
      if (!st.converged && st.iter < kMaxIter) {
        uint32_t slot = 0;
        if (j == 0) slot = atomicAdd(a.spill_count, 1u);
        slot = __shfl_sync(r.mask, slot, 0, W);
        if (slot < a.spill_cap) {
          if (j == 0) {
            a.spill[slot].st = st;
            a.spill[slot].p = p;
          }
          continue;
        }
        bfgs_run<false>(r, a.c, st, kMaxIter);  // spill buffer full: finish here
      }
      fit_finish(r, a.c, st, o);
    }
    if (j == 0) store(a, p, o);
  }
}

// Phase 2: one warp per straggler, continuing its BFGS state to the reference's 500-iteration
// cap with the warp-parallel line search; the log-samples are recomputed (same values).
template <int KT>
__global__ void __launch_bounds__(128) fit_stragglers_kernel(const FitArgs a) {
  const uint32_t count = min(*a.spill_count, a.spill_cap);
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t j = warp; j < count; j += nwarps) {
    Bfgs st = a.spill[j].st;
    const uint64_t p = a.spill[j].p;
    FitOut o;
    if (KT > 0) {
      RegRows<(KT > 0 ? KT : 1)> r;
      const double* row = a.x + p * KT;
#pragma unroll
      for (int i = 0; i < KT; ++i) r.lx[i] = log(row[i]);
      bfgs_run<true>(r, a.c, st, kMaxIter);
      fit_finish(r, a.c, st, o);
    } else {
      GlobalRows r;  // read-only use: the prompt's log-samples written in phase 1
      r.K = a.K;
      r.lx = a.lx_scratch + p * (uint64_t)a.K * 2;
      r.t = nullptr;
      bfgs_run<true>(r, a.c, st, kMaxIter);
      fit_finish(r, a.c, st, o);
    }
    if ((threadIdx.x & 31) == 0) store(a, p, o);
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
                       uint8_t* degen, cudaStream_t s, uint64_t index_base) {
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
  a.index_base = index_base;
  const int sms = sm_count(ctx->device);
  const unsigned grid = (unsigned)std::min<uint64_t>((P + 127) / 128, (uint64_t)sms * 16);
  // scratch: [log-samples (generic K only)][straggler spill buffer][spill counter]
  const bool generic = !(K == 8 || K == 16 || K == 20 || K == 32);
  a.spill_cap = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(4096, P / 64), 1u << 22);
  const size_t lx_bytes = generic ? ((sizeof(double) * P * K * 2 + 255) & ~(size_t)255) : 0;
  const size_t spill_bytes = ((sizeof(FitSpill) * a.spill_cap) + 255) & ~(size_t)255;
  char* base = (char*)capi::scratch(ctx, lx_bytes + spill_bytes + 256, s);
  if (!base) return cudaErrorMemoryAllocation;
  a.lx_scratch = generic ? (double*)base : nullptr;
  a.spill = (FitSpill*)(base + lx_bytes);
  a.spill_count = (uint32_t*)(base + lx_bytes + spill_bytes);
  cudaMemsetAsync(a.spill_count, 0, sizeof(uint32_t), s);
  const unsigned grid2 = (unsigned)sms * 4;  // phase 2: loops over the device-side count
  {
    ProfScope prof(ctx, "fit", s);
    // lane-per-sample kernels: 2 prompts per warp (K <= 16) or 1 (K <= 32)
    const unsigned g16 = (unsigned)std::min<uint64_t>((P + 7) / 8, (uint64_t)sms * 32);
    const unsigned g32 = (unsigned)std::min<uint64_t>((P + 3) / 4, (uint64_t)sms * 32);
    switch (K) {
      case 8: fit_lanes_kernel<8><<<g16, 128, 0, s>>>(a); break;
      case 16: fit_lanes_kernel<16><<<g16, 128, 0, s>>>(a); break;
      case 20: fit_lanes_kernel<20><<<g32, 128, 0, s>>>(a); break;
      case 32: fit_lanes_kernel<32><<<g32, 128, 0, s>>>(a); break;
      default: fit_kernel_generic<<<grid, 128, 0, s>>>(a);
    }
  }
  {
    ProfScope prof(ctx, "fit.stragglers", s);
    switch (K) {
      case 8: fit_stragglers_kernel<8><<<grid2, 128, 0, s>>>(a); break;
      case 16: fit_stragglers_kernel<16><<<grid2, 128, 0, s>>>(a); break;
      case 20: fit_stragglers_kernel<20><<<grid2, 128, 0, s>>>(a); break;
      case 32: fit_stragglers_kernel<32><<<grid2, 128, 0, s>>>(a); break;
      default: fit_stragglers_kernel<0><<<grid2, 128, 0, s>>>(a);
    }
  }
  capi::count_launch(2);
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
