/* oracle/tie_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference path; each function cites the reference
 * file:line it follows (paths relative to /root/reference/proj).  Pinned against the
 * compiled reference by tests/test_oracle.py (bit-exact) and tests/golden/.
 *
 * One deliberate restructuring, numerically neutral: the reference evaluates psi()
 * up to three times per request (dist.cpp:163-189), each a sequential ascending sum.
 * Here one ascending pass keeps both prefixes (k_alpha and k_max); every partial sum
 * is the same sequence of additions, so the values are bit-identical and the oracle
 * runs ~3x faster.  t_quantile(alpha) is likewise hoisted out of the request loop
 * (it is request-invariant, dist.cpp:170).
 */
#define _GNU_SOURCE
#include "tie_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* tor_last_error(void) { return g_err; }

/* std::max(a, b) == (a < b) ? b : a (NaN-propagating in the first argument) */
static double std_max(double a, double b) { return (a < b) ? b : a; }

/* ---------------------------------------------------------------- mt19937_64 + Rng */
/* std::mt19937_64 (the standard's parameters) -- rng.hpp:21-83 uses it as bit source */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int has_spare;
} rng_t;

static void rng_seed(rng_t* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->spare = 0.0;
  r->has_spare = 0;
}

static uint64_t rng_next(rng_t* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:26-28 */
static double rng_u01(rng_t* r) {
  return ((double)(rng_next(r) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
/* rng.hpp:30 */
static double rng_uniform(rng_t* r, double lo, double hi) { return lo + (hi - lo) * rng_u01(r); }
/* rng.hpp:33-36 */
static uint32_t rng_u32(rng_t* r, uint32_t lo, uint32_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1;
  return lo + (uint32_t)(rng_next(r) % span);
}
/* rng.hpp:39-47 Box-Muller with a cached spare */
static double rng_normal(rng_t* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = rng_u01(r), u2 = rng_u01(r);
  double rad = sqrt(-2.0 * log(u1));
  double ang = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(ang);
  r->has_spare = 1;
  return rad * cos(ang);
}
/* rng.hpp:50-66 Marsaglia-Tsang with the shape<1 boost */
static double rng_gamma(rng_t* r, double shape, double scale) {
  if (shape < 1.0) {
    double u = rng_u01(r);
    return rng_gamma(r, shape + 1.0, scale) * pow(u, 1.0 / shape);
  }
  double d = shape - 1.0 / 3.0;
  double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    double x = rng_normal(r);
    double t = 1.0 + c * x;
    if (t <= 0.0) continue;
    double v = t * t * t;
    double u = rng_u01(r);
    if (u < 1.0 - 0.0331 * x * x * x * x) return d * v * scale;
    if (log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) return d * v * scale;
  }
}
/* rng.hpp:68-75 */
static double rng_student_t(rng_t* r, double nu) {
  double z = rng_normal(r);
  double v = rng_gamma(r, 0.5 * nu, 2.0);
  return z / sqrt(v / nu);
}
/* rng.hpp:77 */
static double rng_exponential(rng_t* r, double rate) { return -log(rng_u01(r)) / rate; }

/* rng.hpp:10-16 */
uint64_t tor_mix64(uint64_t a, uint64_t b) {
  uint64_t x = a + 0x9E3779B97F4A7C15ULL * (b + 1);
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ULL;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

/* ---------------------------------------------------------------- threads */
typedef void (*body_fn)(void* ctx, uint64_t begin, uint64_t end);
typedef struct {
  body_fn fn;
  void* ctx;
  uint64_t n;
  uint64_t chunk;
  uint64_t next; /* atomic */
} pool_t;

static void* pool_worker(void* arg) {
  pool_t* p = (pool_t*)arg;
  for (;;) {
    uint64_t b = __atomic_fetch_add(&p->next, p->chunk, __ATOMIC_RELAXED);
    if (b >= p->n) break;
    uint64_t e = b + p->chunk < p->n ? b + p->chunk : p->n;
    p->fn(p->ctx, b, e);
  }
  return NULL;
}

static void parallel_for(uint64_t n, int threads, uint64_t chunk, body_fn fn, void* ctx) {
  if (threads <= 1 || n <= chunk) {
    fn(ctx, 0, n);
    return;
  }
  pool_t p = {fn, ctx, n, chunk, 0};
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, pool_worker, &p);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
}

/* ---------------------------------------------------------------- Student-t */
/* dist.cpp:19-48 -- modified Lentz continued fraction */
static double incbeta_cf(double a, double b, double x) {
  const double tiny = 1e-300, eps = 1e-15;
  double qab = a + b, qap = a + 1.0, qam = a - 1.0;
  double c = 1.0;
  double d = 1.0 - qab * x / qap;
  if (fabs(d) < tiny) d = tiny;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= 100000; ++m) {
    int m2 = 2 * m;
    double aa = m * (b - m) * x / ((qam + m2) * (a + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    h *= d * c;
    aa = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
    d = 1.0 + aa * d;
    if (fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c;
    if (fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    double del = d * c;
    h *= del;
    if (fabs(del - 1.0) < eps) break;
  }
  return h;
}

/* dist.cpp:52-63 (domain checks return NaN here; callers validate first) */
double tor_regularized_incomplete_beta(double a, double b, double x) {
  if (!(a > 0.0) || !(b > 0.0) || !isfinite(a) || !isfinite(b)) return NAN;
  if (!(x >= 0.0 && x <= 1.0)) return NAN;
  if (x == 0.0) return 0.0;
  if (x == 1.0) return 1.0;
  double logbeta = lgamma(a) + lgamma(b) - lgamma(a + b);
  double front = exp(a * log(x) + b * log1p(-x) - logbeta);
  if (x < (a + 1.0) / (a + b + 2.0)) return front * incbeta_cf(a, b, x) / a;
  return 1.0 - front * incbeta_cf(b, a, 1.0 - x) / b;
}

/* dist.cpp:65-71 */
double tor_t_pdf(double y, double nu) {
  double lognorm = lgamma(0.5 * (nu + 1.0)) - lgamma(0.5 * nu) -
                   0.5 * log(nu * 3.14159265358979323846);
  return exp(lognorm - 0.5 * (nu + 1.0) * log1p(y * y / nu));
}

/* dist.cpp:73-81 */
double tor_t_cdf(double y, double nu) {
  if (isnan(y)) return NAN;
  if (y == INFINITY) return 1.0;
  if (y == -INFINITY) return 0.0;
  double x = nu / (y * y + nu);
  double tail = tor_regularized_incomplete_beta(0.5 * nu, 0.5, x);
  return y >= 0.0 ? 1.0 - 0.5 * tail : 0.5 * tail;
}

/* dist.cpp:83-106 -- bracket, bisect, 4 Newton polishes */
double tor_t_quantile(double p, double nu) {
  if (!(p > 0.0 && p < 1.0)) return NAN;
  if (p == 0.5) return 0.0;
  double lo = -1.0, hi = 1.0;
  while (tor_t_cdf(lo, nu) > p) lo *= 2.0;
  while (tor_t_cdf(hi, nu) < p) hi *= 2.0;
  double y = 0.0;
  for (int i = 0; i < 200 && hi - lo > 1e-14 * std_max(1.0, fabs(lo)); ++i) {
    y = 0.5 * (lo + hi);
    if (tor_t_cdf(y, nu) < p) lo = y; else hi = y;
  }
  y = 0.5 * (lo + hi);
  for (int i = 0; i < 4; ++i) {
    double f = tor_t_cdf(y, nu) - p;
    double d = tor_t_pdf(y, nu);
    if (d <= 0.0) break;
    double step = f / d;
    if (!isfinite(step)) break;
    y -= step;
  }
  return y;
}

/* ---------------------------------------------------------------- samples */
static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* dist.cpp:122-129 */
int tor_mc_samples(double nu, int n, uint64_t seed, double* out) {
  if (!(nu > 0.0) || !isfinite(nu)) return fail(1, "McContext: nu must be finite and > 0");
  if (n <= 0) return fail(1, "McContext: n_samples must be > 0");
  rng_t r;
  rng_seed(&r, seed);
  for (int i = 0; i < n; ++i) out[i] = rng_student_t(&r, nu);
  qsort(out, (size_t)n, sizeof(double), cmp_double);
  return 0;
}

/* dist.cpp:142-147 */
int tor_sample_logt(double mu, double sigma, double nu, uint64_t n, uint64_t seed, double* out) {
  if (sigma < 1e-9) sigma = 1e-9; /* LogTParams clamp, dist.cpp:113-116 */
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = exp(mu + sigma * rng_student_t(&r, nu));
  return 0;
}

/* ---------------------------------------------------------------- score */
static uint64_t upper_bound_d(const double* v, uint64_t n, double y) {
  uint64_t lo = 0, hi = n; /* first index with v[i] > y (std::upper_bound) */
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (y < v[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

typedef struct {
  const double* Y;
  int N;
  double nu, alpha, beta;
  uint64_t k_alpha;
  const double *mu, *sigma, *x_max;
  double *E, *C, *S;
  int* code;          /* per-request error code (0 ok) */
} score_ctx;

/* One request: LogTParams/CensoredLogT validation (dist.cpp:108-120), censored_tail_core
 * (163-175), censored_expectation (179-181), censored_cvar (183-189), run_sim's
 * max(cvar, E) (sim.cpp:94), compute_score (sched.cpp:19-26). */
static int score_one(const score_ctx* c, uint64_t i, double* e_out, double* c_out,
                     double* s_out) {
  double mu = c->mu[i], sigma = c->sigma[i], xm = c->x_max[i];
  if (!isfinite(mu)) return 1;
  if (!(sigma > 0.0) || !isfinite(sigma)) return 1;
  if (sigma < 1e-9) sigma = 1e-9;
  if (!(xm > 0.0) || !isfinite(xm)) return 1;
  double y_max = (log(xm) - mu) / sigma;
  if (isnan(y_max)) return 1;
  uint64_t k_max = upper_bound_d(c->Y, (uint64_t)c->N, y_max);
  double T = tor_t_cdf(y_max, c->nu);
  double censor = 1.0 - T;
  int cvar_saturated = c->alpha >= T;
  uint64_t k_a = cvar_saturated ? 0 : c->k_alpha;
  uint64_t kend = k_max > k_a ? k_max : k_a;
  double sum = 0.0, s_all = 0.0, s_alpha = 0.0;
  for (uint64_t k = 0; k < kend; ++k) {
    sum += exp(mu + sigma * c->Y[k]);
    if (k + 1 == k_max) s_all = sum;
    if (k + 1 == k_a) s_alpha = sum;
  }
  double Nd = (double)c->N;
  double psi_cap = s_all / Nd;
  double e = (psi_cap - 0.0 + xm * censor) / (1.0 - 0.0);
  e = (xm < e) ? xm : e; /* std::min(v, x_max) == (x_max < v) ? x_max : v */
  double cv;
  if (cvar_saturated) {
    cv = xm;
  } else {
    double psi_alpha = c->alpha > 0.0 ? s_alpha / Nd : 0.0;
    double v = (psi_cap - psi_alpha + xm * censor) / (1.0 - c->alpha);
    cv = (xm < v) ? xm : v;
  }
  cv = (cv < e) ? e : cv; /* std::max(cvar, E) */
  if (!isfinite(e) || !isfinite(cv) || !isfinite(c->beta)) return 1;
  if (!(e > 0.0)) return 1;
  if (cv < e) return 2;
  *e_out = e;
  *c_out = cv;
  *s_out = e + c->beta * cv;
  return 0;
}

static void score_body(void* vctx, uint64_t b, uint64_t e) {
  score_ctx* c = (score_ctx*)vctx;
  for (uint64_t i = b; i < e; ++i) {
    double ev = 0, cv = 0, sv = 0;
    int rc = score_one(c, i, &ev, &cv, &sv);
    c->code[i] = rc;
    if (c->E) c->E[i] = ev;
    if (c->C) c->C[i] = cv;
    if (c->S) c->S[i] = sv;
  }
}

int tor_score(const double* samples, int N, double nu, const double* mu, const double* sigma,
              const double* x_max, uint64_t n, double alpha, double beta, double* E, double* C,
              double* S, uint64_t* bad_index, int threads) {
  if (bad_index) *bad_index = UINT64_MAX;
  if (!(alpha >= 0.0 && alpha < 1.0)) return fail(1, "censored_cvar: alpha must lie in [0, 1)");
  score_ctx c;
  c.Y = samples;
  c.N = N;
  c.nu = nu;
  c.alpha = alpha;
  c.beta = beta;
  c.k_alpha = alpha > 0.0 ? upper_bound_d(samples, (uint64_t)N, tor_t_quantile(alpha, nu)) : 0;
  c.mu = mu;
  c.sigma = sigma;
  c.x_max = x_max;
  c.E = E;
  c.C = C;
  c.S = S;
  c.code = (int*)calloc(n ? n : 1, sizeof(int));
  parallel_for(n, threads, 64, score_body, &c);
  int rc = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (c.code[i]) {
      rc = c.code[i];
      if (bad_index) *bad_index = i;
      break;
    }
  free(c.code);
  if (rc == 1) return fail(1, "score: domain error (bad mu/sigma/x_max or non-finite score)");
  if (rc == 2) return fail(2, "compute_score: cvar below expectation violates the invariant");
  return 0;
}

/* sched.cpp:9-17 */
int tor_compute_beta(int adaptive, double beta_fixed, double beta_max, double q_sat,
                     uint64_t queue_len, double* beta) {
  if (!adaptive) {
    if (beta_fixed < 0.0) return fail(1, "compute_beta: beta_fixed must be >= 0");
    *beta = beta_fixed;
    return 0;
  }
  if (!(beta_max >= 0.0) || !(q_sat > 0.0))
    return fail(1, "compute_beta: beta_max must be >= 0 and q_sat > 0");
  double r = (double)queue_len / q_sat;
  *beta = beta_max * (r < 1.0 ? r : 1.0);
  return 0;
}

/* ---------------------------------------------------------------- rank */
typedef struct {
  double key;
  uint64_t id;
} kid_t;

static int cmp_kid(const void* a, const void* b) {
  const kid_t* x = (const kid_t*)a;
  const kid_t* y = (const kid_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->id > y->id) - (x->id < y->id);
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* WaitingQueue::less (sched.cpp:28-31): pop_min order of a static queue is the
 * lexicographic (key, req_id) order; push validation at sched.cpp:59-63. */
int tor_rank(const double* key, const uint64_t* ids, uint64_t n, uint64_t* order) {
  kid_t* v = (kid_t*)malloc(sizeof(kid_t) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) {
    if (!isfinite(key[i])) {
      free(v);
      return fail(1, "WaitingQueue::push: key must be finite");
    }
    v[i].key = key[i];
    v[i].id = ids ? ids[i] : i;
  }
  if (ids) { /* duplicate id -> invalid_argument (sched.cpp:61-63) */
    uint64_t* s = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    memcpy(s, ids, sizeof(uint64_t) * n);
    qsort(s, n, sizeof(uint64_t), cmp_u64);
    for (uint64_t i = 1; i < n; ++i)
      if (s[i] == s[i - 1]) {
        free(s);
        free(v);
        return fail(2, "WaitingQueue::push: id already queued");
      }
    free(s);
  }
  qsort(v, n, sizeof(kid_t), cmp_kid);
  for (uint64_t i = 0; i < n; ++i) order[i] = v[i].id;
  free(v);
  return 0;
}

/* ---------------------------------------------------------------- fit */
/* fit.cpp:44-56 */
double tor_logt_loglik(const double* x, uint64_t K, double mu, double sigma, double nu) {
  double lognorm = lgamma(0.5 * (nu + 1.0)) - lgamma(0.5 * nu) -
                   0.5 * log(nu * 3.14159265358979323846);
  double ll = 0.0;
  for (uint64_t i = 0; i < K; ++i) {
    double lx = log(x[i]);
    double z = (lx - mu) / sigma;
    ll += lognorm - 0.5 * (nu + 1.0) * log1p(z * z / nu) - log(sigma) - lx;
  }
  return ll;
}

/* fit.cpp:58-71 */
static void logt_grad(const double* x, uint64_t K, double mu, double sigma, double nu,
                      double* gmu, double* gsig) {
  double a = 0.0, b = 0.0;
  for (uint64_t i = 0; i < K; ++i) {
    double z = (log(x[i]) - mu) / sigma;
    double w = (nu + 1.0) * z / (nu + z * z);
    a += w / sigma;
    b += (w * z - 1.0) / sigma;
  }
  *gmu = a;
  *gsig = b;
}

/* logt_loglik_grad (fit.cpp:58-71), exported for the device loglik/grad parity test */
void tor_logt_loglik_grad(const double* x, uint64_t K, double mu, double sigma, double nu,
                          double* grad) {
  logt_grad(x, K, mu, sigma, nu, &grad[0], &grad[1]);
}

static double median_sorted(const double* v, uint64_t n) {
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

typedef struct {
  double mu, sigma, ll;
  int iters, converged, degenerate;
} fit_out;

/* fit.cpp:73-178 -- BFGS over (mu, s = ln sigma), Armijo backtracking */
static void fit_one(const double* x, uint64_t K, double nu, double* scratch, fit_out* out) {
  const double kSigmaFloor = 1e-6, kLogSigmaFloor = -13.815510557964274;
  double* lx = scratch;
  double* dev = scratch + K;
  for (uint64_t i = 0; i < K; ++i) lx[i] = log(x[i]);
  qsort(lx, K, sizeof(double), cmp_double);
  double mu0 = median_sorted(lx, K);
  for (uint64_t i = 0; i < K; ++i) dev[i] = fabs(lx[i] - mu0);
  qsort(dev, K, sizeof(double), cmp_double);
  double sigma0 = 1.4826 * median_sorted(dev, K);
  out->degenerate = 0;
  out->iters = 0;
  if (sigma0 < kSigmaFloor) {
    out->mu = mu0;
    out->sigma = kSigmaFloor;
    out->degenerate = 1;
    out->converged = 1;
    out->ll = tor_logt_loglik(x, K, out->mu, out->sigma, nu);
    return;
  }
#define FVAL(m, s) (-tor_logt_loglik(x, K, (m), exp(s), nu))
  double th0 = mu0, th1 = log(sigma0);
  double f = FVAL(th0, th1);
  double g0, g1;
  {
    double sg = exp(th1), a, b;
    logt_grad(x, K, th0, sg, nu, &a, &b);
    g0 = -a;
    g1 = -b * sg;
  }
  double H00 = 1.0, H01 = 0.0, H10 = 0.0, H11 = 1.0;
  const double gtol = 1e-8;
  int iter = 0, converged = 0;
  for (; iter < 500; ++iter) {
    if (std_max(fabs(g0), fabs(g1)) < gtol) {
      converged = 1;
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
      f_new = FVAL(n0, n1);
      if (isfinite(f_new) && f_new <= f + 1e-4 * step * descent) break;
      step *= 0.5;
    }
    if (!(f_new < f) && std_max(fabs(g0), fabs(g1)) < 1e-6) {
      converged = 1;
      break;
    }
    double q0, q1;
    {
      double sg = exp(n1), a, b;
      logt_grad(x, K, n0, sg, nu, &a, &b);
      q0 = -a;
      q1 = -b * sg;
    }
    double s0 = n0 - th0, s1 = n1 - th1;
    double y0 = q0 - g0, y1 = q1 - g1;
    double sy = s0 * y0 + s1 * y1;
    if (sy > 1e-12) {
      double rho = 1.0 / sy;
      double Hy0 = H00 * y0 + H01 * y1, Hy1 = H10 * y0 + H11 * y1;
      double yHy = y0 * Hy0 + y1 * Hy1;
      double s[2] = {s0, s1}, Hy[2] = {Hy0, Hy1};
      double H[2][2] = {{H00, H01}, {H10, H11}};
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
          H[i][j] += rho * ((1.0 + rho * yHy) * s[i] * s[j] - s[i] * Hy[j] - Hy[i] * s[j]);
      H00 = H[0][0];
      H01 = H[0][1];
      H10 = H[1][0];
      H11 = H[1][1];
    }
    th0 = n0;
    th1 = n1;
    f = f_new;
    g0 = q0;
    g1 = q1;
  }
#undef FVAL
  out->mu = th0;
  out->sigma = exp(th1);
  if (out->sigma <= kSigmaFloor) {
    out->sigma = kSigmaFloor;
    out->degenerate = 1;
  }
  out->converged = converged;
  out->iters = iter;
  out->ll = tor_logt_loglik(x, K, out->mu, out->sigma, nu);
}

typedef struct {
  const double* x;
  uint64_t K;
  double nu;
  double *mu, *sigma, *ll;
  int32_t* iters;
  uint8_t *conv, *degen;
} fit_ctx;

static void fit_body(void* vctx, uint64_t b, uint64_t e) {
  fit_ctx* c = (fit_ctx*)vctx;
  double* scratch = (double*)malloc(sizeof(double) * 2 * c->K);
  for (uint64_t p = b; p < e; ++p) {
    fit_out o;
    fit_one(c->x + p * c->K, c->K, c->nu, scratch, &o);
    c->mu[p] = o.mu;
    c->sigma[p] = o.sigma;
    if (c->ll) c->ll[p] = o.ll;
    if (c->iters) c->iters[p] = o.iters;
    if (c->conv) c->conv[p] = (uint8_t)o.converged;
    if (c->degen) c->degen[p] = (uint8_t)o.degenerate;
  }
  free(scratch);
}

int tor_fit(const double* x, uint64_t P, uint64_t K, double nu, double* mu, double* sigma,
            double* ll, int32_t* iters, uint8_t* converged, uint8_t* degenerate, int threads) {
  /* check_samples(x, 3, ...) fit.cpp:18-25, nu check fit.cpp:75-76 */
  if (K < 3) return fail(2, "fit_logt_fixed_nu: need at least 3 samples");
  for (uint64_t i = 0; i < P * K; ++i)
    if (!(x[i] > 0.0) || !isfinite(x[i]))
      return fail(1, "fit_logt_fixed_nu: samples must be finite and > 0");
  if (!(nu > 0.0) || !isfinite(nu)) return fail(1, "fit_logt_fixed_nu: nu must be finite and > 0");
  fit_ctx c = {x, K, nu, mu, sigma, ll, iters, converged, degenerate};
  parallel_for(P, threads, 256, fit_body, &c);
  return 0;
}

/* ---------------------------------------------------------------- fit report */
/* cmd_fit's per-prompt analysis (main.cpp:510-585) over P prompts x K lengths: the four
 * families (fit.cpp:73-178 fixed nu; 180-200 free nu over default_nu_grid; 202-230
 * lognormal; 232-243 exponential), ks_test of each fit's CDF (fit.cpp:245-284) and, for
 * K >= 10, tail_stats (fit.cpp:286-324).  Layout: fits[f][field][P] with f = 0 logt,
 * 1 logt_free_nu, 2 lognormal, 3 exponential and field = mu, sigma, nu, rate,
 * log_likelihood, iterations, converged, degenerate, ks_statistic, ks_p_value;
 * tail[field][P] = skewness, cv, p90_over_p50, p99_over_p50, top10_share (NaN if K < 10). */
enum { FR_MU, FR_SIGMA, FR_NU, FR_RATE, FR_LL, FR_ITERS, FR_CONV, FR_DEGEN, FR_KSD, FR_KSP, FR_N };

static double normal_cdf(double z); /* dist.cpp:191 (defined with the lognormal family below) */

typedef struct {
  int family; /* 0..3 */
  double mu, sigma, nu, rate, ll;
  int iters, converged, degenerate;
} fam_fit;

static double fit_cdf(const fam_fit* f, double x) { /* fit.cpp:245-258 */
  if (!(x > 0.0)) return 0.0;
  switch (f->family) {
    case 0:
    case 1: return tor_t_cdf((log(x) - f->mu) / f->sigma, f->nu);
    case 2: return normal_cdf((log(x) - f->mu) / f->sigma);
    default: return -expm1(-f->rate * x);
  }
}

/* ks_test on the sorted samples s (fit.cpp:261-284); returns 0 or the domain error */
static int ks_sorted(const double* s, uint64_t K, const fam_fit* f, double* D, double* P) {
  double n = (double)K, d = 0.0;
  for (uint64_t i = 0; i < K; ++i) {
    double F = fit_cdf(f, s[i]);
    if (!(F >= 0.0 && F <= 1.0)) return 1;
    double a = ((double)i + 1.0) / n - F, b = F - (double)i / n;
    double m = a < b ? b : a;
    d = d < m ? m : d;
  }
  double lambda = (sqrt(n) + 0.12 + 0.11 / sqrt(n)) * d;
  double p = 0.0, sign = 1.0;
  for (int j = 1; j <= 100; ++j) {
    double term = sign * 2.0 * exp(-2.0 * j * j * lambda * lambda);
    p += term;
    if (fabs(term) < 1e-12) break;
    sign = -sign;
  }
  p = p > 0.0 ? p : 0.0;
  p = p < 1.0 ? p : 1.0;
  *D = d;
  *P = p;
  return 0;
}

typedef struct {
  const double* x;
  uint64_t K, P;
  double nu;
  unsigned families;
  double* fits;
  double* tail;
  volatile int err; /* first domain error seen (ks_test cdf outside [0,1]) */
} report_ctx;

static void report_body(void* vctx, uint64_t b, uint64_t e) {
  report_ctx* c = (report_ctx*)vctx;
  const uint64_t K = c->K, P = c->P;
  double* scratch = (double*)malloc(sizeof(double) * 2 * K);
  double* s = (double*)malloc(sizeof(double) * K);
  for (uint64_t p = b; p < e; ++p) {
    const double* x = c->x + p * K;
    for (uint64_t i = 0; i < K; ++i) s[i] = x[i];
    qsort(s, K, sizeof(double), cmp_double); /* ks_test / tail_stats sort a copy */
    for (int f = 0; f < 4; ++f) {
      if (!(c->families >> f & 1)) continue;
      fam_fit r = {f, 0.0, 0.0, 0.0, 0.0, 0.0, 0, 0, 0};
      if (f == 0 || f == 1) {
        fit_out o;
        if (f == 0) {
          fit_one(x, K, c->nu, scratch, &o);
          r.nu = c->nu;
        } else { /* fit_logt_free_nu: best log-likelihood over the grid, first on ties */
          int have = 0;
          for (double v = 1.0; v <= 10.0 + 1e-9; v += 0.5) {
            fit_out t;
            fit_one(x, K, v, scratch, &t);
            if (!have || t.ll > o.ll) {
              o = t;
              r.nu = v;
              have = 1;
            }
          }
        }
        r.mu = o.mu;
        r.sigma = o.sigma;
        r.ll = o.ll;
        r.iters = o.iters;
        r.converged = o.converged;
        r.degenerate = o.degenerate;
      } else if (f == 2) { /* fit_lognormal */
        double n = (double)K, mean = 0.0, var = 0.0;
        for (uint64_t i = 0; i < K; ++i) mean += log(x[i]);
        mean /= n;
        for (uint64_t i = 0; i < K; ++i) {
          double d = log(x[i]) - mean;
          var += d * d;
        }
        var /= n;
        r.mu = mean;
        r.sigma = sqrt(var);
        r.converged = 1;
        if (r.sigma < 1e-6) {
          r.sigma = 1e-6;
          r.degenerate = 1;
        }
        double ll = 0.0;
        for (uint64_t i = 0; i < K; ++i) {
          double z = (log(x[i]) - r.mu) / r.sigma;
          ll += -log(r.sigma * x[i]) - 0.5 * log(2.0 * 3.14159265358979323846) - 0.5 * z * z;
        }
        r.ll = ll;
      } else { /* fit_exponential */
        double mean = 0.0;
        for (uint64_t i = 0; i < K; ++i) mean += x[i];
        mean /= (double)K;
        r.rate = 1.0 / mean;
        r.converged = 1;
        r.ll = (double)K * log(r.rate) - r.rate * mean * (double)K;
      }
      double D = 0.0, Pv = 0.0;
      if (ks_sorted(s, K, &r, &D, &Pv)) c->err = 1;
      double* o = c->fits + (uint64_t)f * FR_N * P;
      o[FR_MU * P + p] = r.mu;
      o[FR_SIGMA * P + p] = r.sigma;
      o[FR_NU * P + p] = r.nu;
      o[FR_RATE * P + p] = r.rate;
      o[FR_LL * P + p] = r.ll;
      o[FR_ITERS * P + p] = (double)r.iters;
      o[FR_CONV * P + p] = (double)r.converged;
      o[FR_DEGEN * P + p] = (double)r.degenerate;
      o[FR_KSD * P + p] = D;
      o[FR_KSP * P + p] = Pv;
    }
    if (c->tail) {
      double* t = c->tail;
      if (K < 10) {
        for (int j = 0; j < 5; ++j) t[j * P + p] = NAN;
        continue;
      }
      double n = (double)K, total = 0.0, m2 = 0.0, m3 = 0.0;
      for (uint64_t i = 0; i < K; ++i) total += s[i];
      double mean = total / n;
      for (uint64_t i = 0; i < K; ++i) {
        double d = s[i] - mean;
        m2 += d * d;
        m3 += d * d * d;
      }
      m2 /= n;
      m3 /= n;
#define TOR_RANK(q, out)                                  \
  do {                                                    \
    uint64_t k_ = (uint64_t)ceil((q) * n);                \
    if (k_ > K) k_ = K;                                   \
    if (k_ < 1) k_ = 1;                                   \
    out = s[k_ - 1];                                      \
  } while (0)
      double p50, p90, p99;
      TOR_RANK(0.50, p50);
      TOR_RANK(0.90, p90);
      TOR_RANK(0.99, p99);
#undef TOR_RANK
      uint64_t k10 = (uint64_t)ceil(0.1 * n);
      double top = 0.0;
      for (uint64_t i = K - k10; i < K; ++i) top += s[i];
      t[0 * P + p] = m2 > 0.0 ? m3 / pow(m2, 1.5) : 0.0;
      t[1 * P + p] = mean > 0.0 ? sqrt(m2) / mean : 0.0;
      t[2 * P + p] = p50 > 0.0 ? p90 / p50 : 1.0;
      t[3 * P + p] = p50 > 0.0 ? p99 / p50 : 1.0;
      t[4 * P + p] = total > 0.0 ? top / total : 0.0;
    }
  }
  free(scratch);
  free(s);
}

int tor_fit_report(const double* x, uint64_t P, uint64_t K, double nu, unsigned families,
                   double* fits, double* tail, int threads) {
  if (K < 5) return fail(2, "ks_test: need at least 5 samples");
  for (uint64_t i = 0; i < P * K; ++i)
    if (!(x[i] > 0.0) || !isfinite(x[i]))
      return fail(1, "fit_logt_fixed_nu: samples must be finite and > 0");
  if (!(nu > 0.0) || !isfinite(nu)) return fail(1, "fit_logt_fixed_nu: nu must be finite and > 0");
  report_ctx c = {x, K, P, nu, families, fits, tail, 0};
  parallel_for(P, threads, 64, report_body, &c);
  if (c.err) return fail(1, "ks_test: cdf returned a value outside [0, 1]");
  return 0;
}

/* ---------------------------------------------------------------- inputs */
/* workload.cpp:37-48 + 50-78 */
int tor_gen_workload(uint64_t n, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                     double sg_hi, double nu, uint32_t max_tokens, double rps, double* mu,
                     double* sigma, uint32_t* max_tok, double* arrival, uint32_t* prompt_tokens,
                     uint32_t* true_len) {
  if (!(mu_lo <= mu_hi)) return fail(1, "gen_logt_workload: bad mu_range");
  if (!(sg_lo > 0.0) || !(sg_lo <= sg_hi)) return fail(1, "gen_logt_workload: bad sigma_range");
  if (!(nu > 0.0)) return fail(1, "gen_logt_workload: nu must be > 0");
  if (max_tokens < 1) return fail(1, "gen_logt_workload: max_tokens must be >= 1");
  rng_t ra, r;
  rng_seed(&ra, tor_mix64(seed, 1));
  double t = 0.0;
  if (arrival)
    for (uint64_t i = 0; i < n; ++i) {
      t += rng_exponential(&ra, rps);
      arrival[i] = t;
    }
  rng_seed(&r, tor_mix64(seed, 2));
  for (uint64_t i = 0; i < n; ++i) {
    double m = rng_uniform(&r, mu_lo, mu_hi);
    double s = rng_uniform(&r, sg_lo, sg_hi);
    uint32_t pt = rng_u32(&r, 64, 512); /* WorkloadSpec{}.prompt_range, workload.hpp:34 */
    double ln_len = m + s * rng_student_t(&r, nu);
    double len = ln_len > 22.0 ? 4294967295.0 : round(exp(ln_len));
    if (len < 1.0) len = 1.0;
    if (len > 4294967295.0) len = 4294967295.0;
    mu[i] = m;
    sigma[i] = s;
    max_tok[i] = max_tokens;
    if (prompt_tokens) prompt_tokens[i] = pt;
    if (true_len) true_len[i] = (uint32_t)len;
  }
  return 0;
}

typedef struct {
  uint64_t K, seed;
  double nu;
  int integerise;
  const double *m, *s;
  double* x;
} gfit_ctx;

static void gfit_body(void* vctx, uint64_t b, uint64_t e) {
  gfit_ctx* c = (gfit_ctx*)vctx;
  for (uint64_t p = b; p < e; ++p) {
    double* row = c->x + p * c->K;
    tor_sample_logt(c->m[p], c->s[p], c->nu, c->K, tor_mix64(c->seed, p), row);
    if (c->integerise)
      for (uint64_t k = 0; k < c->K; ++k) {
        double v = row[k];
        if (v >= 4294967295.0) {
          row[k] = 4294967295.0;
        } else {
          long long L = llround(v);
          row[k] = (double)(L < 1 ? 1 : L);
        }
      }
  }
}

int tor_gen_fit_data(uint64_t P, uint64_t K, uint64_t seed, double mu_lo, double mu_hi,
                     double sg_lo, double sg_hi, double nu, int integerise, double* x,
                     double* true_mu, double* true_sigma, int threads) {
  double* m = true_mu ? true_mu : (double*)malloc(sizeof(double) * (P ? P : 1));
  double* s = true_sigma ? true_sigma : (double*)malloc(sizeof(double) * (P ? P : 1));
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t p = 0; p < P; ++p) {
    m[p] = rng_uniform(&r, mu_lo, mu_hi);
    s[p] = rng_uniform(&r, sg_lo, sg_hi);
  }
  gfit_ctx c = {K, seed, nu, integerise, m, s, x};
  parallel_for(P, threads, 1024, gfit_body, &c);
  if (!true_mu) free(m);
  if (!true_sigma) free(s);
  return 0;
}

/* ---------------------------------------------------------------- scheduler */
typedef struct {
  uint64_t id;
  double key, E, C, beta;
  int predicted, alive;
} qent_t;

/* sched.cpp:9-26 with the reference's validation */
static int sched_beta(int adaptive, double bf, double bm, double qs, uint64_t q, double* out) {
  return tor_compute_beta(adaptive, bf, bm, qs, q, out);
}

int tor_scheduler_script(int policy, int adaptive, double beta_fixed, double beta_max,
                         double q_sat, double rebuild_threshold, uint64_t n_ops,
                         const int32_t* op, const uint64_t* id, const double* a,
                         const double* b, uint64_t* out, uint64_t* n_out) {
  qent_t* e = (qent_t*)calloc(n_ops ? n_ops : 1, sizeof(qent_t));
  double* betas = (double*)malloc(sizeof(double) * (n_ops ? n_ops : 1)); /* multiset */
  uint64_t n = 0, nb = 0, size = 0, k = 0;
  int rc = 0;
#define FIND(x) ({ uint64_t f_ = UINT64_MAX; for (uint64_t j_ = 0; j_ < n; ++j_) \
                   if (e[j_].alive && e[j_].id == (x)) { f_ = j_; break; } f_; })
  for (uint64_t i = 0; i < n_ops && !rc; ++i) {
    if (op[i] == 0) { /* on_arrival (sched.cpp:125-132) + push (59-67) */
      double key = policy == 0 ? a[i] : (double)(uint32_t)b[i];
      if (!isfinite(key)) { rc = fail(1, "WaitingQueue::push: key must be finite"); break; }
      if (FIND(id[i]) != UINT64_MAX) { rc = fail(2, "WaitingQueue::push: id already queued"); break; }
      e[n].id = id[i]; e[n].key = key; e[n].alive = 1; e[n].predicted = 0;
      ++n; ++size;
    } else if (op[i] == 1) { /* on_prediction (sched.cpp:134-150) */
      uint64_t j = FIND(id[i]);
      if (j == UINT64_MAX) { rc = fail(2, "Scheduler::on_prediction: id not waiting"); break; }
      if (policy == 0) continue;
      double beta = 0.0;
      if (policy == 2 && (rc = sched_beta(adaptive, beta_fixed, beta_max, q_sat, size, &beta))) break;
      if (e[j].predicted) { rc = fail(2, "Scheduler::on_prediction: id already predicted"); break; }
      double E = a[i], C = b[i];
      if (!isfinite(E) || !isfinite(C) || !isfinite(beta)) { rc = fail(1, "compute_score: arguments must be finite"); break; }
      if (!(E > 0.0)) { rc = fail(1, "compute_score: expectation must be > 0"); break; }
      if (C < E) { rc = fail(2, "compute_score: cvar below expectation violates the invariant"); break; }
      e[j].predicted = 1; e[j].E = E; e[j].C = C; e[j].beta = beta;
      betas[nb++] = beta;
      e[j].key = E + beta * C;
    } else { /* next_request (sched.cpp:169-175) with rebuild_if_drifted (152-167) */
      if (policy == 2 && nb > 0) {
        double now, lo = betas[0], hi = betas[0];
        if ((rc = sched_beta(adaptive, beta_fixed, beta_max, q_sat, size, &now))) break;
        for (uint64_t t = 1; t < nb; ++t) { if (betas[t] < lo) lo = betas[t]; if (betas[t] > hi) hi = betas[t]; }
        double worst = std_max(fabs(now - lo), fabs(now - hi));
        if (worst > rebuild_threshold) {
          nb = 0;
          for (uint64_t j = 0; j < n; ++j)
            if (e[j].alive && e[j].predicted) {
              e[j].beta = now; e[j].key = e[j].E + now * e[j].C; betas[nb++] = now;
            }
        }
      }
      uint64_t best = UINT64_MAX;
      for (uint64_t j = 0; j < n; ++j) {
        if (!e[j].alive) continue;
        if (best == UINT64_MAX || e[j].key < e[best].key ||
            (e[j].key == e[best].key && e[j].id < e[best].id)) best = j;
      }
      if (best == UINT64_MAX) { out[k++] = UINT64_MAX; continue; }
      e[best].alive = 0; --size;
      if (e[best].predicted) { /* betas_in_use_.erase(find(beta_at_update)) */
        for (uint64_t t = 0; t < nb; ++t)
          if (betas[t] == e[best].beta) { betas[t] = betas[--nb]; break; }
      }
      out[k++] = e[best].id;
    }
  }
#undef FIND
  *n_out = k;
  free(e);
  free(betas);
  return rc;
}

/* ---------------------------------------------------------------- run_sim scoring chain */
/* dist.cpp:191-249: standard normal CDF / quantile, log-normal censored moments */
static double normal_cdf(double z) { return 0.5 * erfc(-z * 0.7071067811865475244); }

static double normal_quantile(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                             1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                             6.680131188771972e+01, -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                             -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                             3.754408661907416e+00};
  const double plow = 0.02425, phigh = 1.0 - plow;
  double q, r, z;
  if (p < plow) {
    q = sqrt(-2.0 * log(p));
    z = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= phigh) {
    q = p - 0.5;
    r = q * q;
    z = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    q = sqrt(-2.0 * log1p(-p));
    z = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  double e = normal_cdf(z) - p;
  double u = e * sqrt(2.0 * 3.14159265358979323846) * exp(0.5 * z * z);
  return z - u / (1.0 + 0.5 * z * u);
}

double tor_normal_quantile(double p) { return normal_quantile(p); }

static double ln_censored_expectation(double mu, double sigma, double x_max) {
  double y_max = (log(x_max) - mu) / sigma;
  double body = exp(mu + 0.5 * sigma * sigma) * normal_cdf(y_max - sigma);
  double v = body + x_max * (1.0 - normal_cdf(y_max));
  return (x_max < v) ? x_max : v;
}

static double ln_censored_cvar(double mu, double sigma, double x_max, double alpha) {
  double y_max = (log(x_max) - mu) / sigma;
  if (alpha >= normal_cdf(y_max)) return x_max;
  double lo = alpha > 0.0 ? normal_cdf(normal_quantile(alpha) - sigma) : 0.0;
  double body = exp(mu + 0.5 * sigma * sigma) * (normal_cdf(y_max - sigma) - lo);
  double v = (body + x_max * (1.0 - normal_cdf(y_max))) / (1.0 - alpha);
  return (x_max < v) ? x_max : v;
}

/* predictor.cpp:22-31: noisy_predict with Rng(mix64(seed, id)) */
static void noisy(double mu, double sigma, uint64_t id, double mu_sd, double ls_sd,
                  uint64_t seed, double* mu_hat, double* sigma_hat) {
  rng_t r;
  rng_seed(&r, tor_mix64(seed, id));
  double m = mu + mu_sd * rng_normal(&r);
  double st = log1p(sigma) + ls_sd * rng_normal(&r);
  double s = expm1(st);
  *mu_hat = m;
  *sigma_hat = (s < 1e-6) ? 1e-6 : s; /* std::max(expm1(st), 1e-6) */
}

/* The run_sim precompute loop (sim.cpp:77-96): predictor (0 oracle, 1 noisy), family (0 logt,
 * 1 lognormal), CVaR = max(CVaR, E).  samples = the McContext set (logt family). */
int tor_sim_scores(const double* samples, int N, double nu, const double* mu,
                   const double* sigma, const uint64_t* ids, const double* x_max, uint64_t n,
                   int predictor, double mu_sd, double ls_sd, uint64_t seed, int family,
                   double alpha, double* E, double* C) {
  double* m = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* s = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) {
    if (predictor == 1) noisy(mu[i], sigma[i], ids[i], mu_sd, ls_sd, seed, &m[i], &s[i]);
    else { m[i] = mu[i]; s[i] = sigma[i]; }
  }
  int rc = 0;
  if (family == 0) {
    rc = tor_score(samples, N, nu, m, s, x_max, n, alpha, 0.0, E, C, NULL, NULL, 1);
  } else {
    for (uint64_t i = 0; i < n; ++i) {
      double e = ln_censored_expectation(m[i], s[i], x_max[i]);
      double c = ln_censored_cvar(m[i], s[i], x_max[i], alpha);
      E[i] = e;
      C[i] = (c < e) ? e : c;
    }
  }
  free(m);
  free(s);
  return rc;
}
