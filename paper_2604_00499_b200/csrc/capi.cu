// C-ABI (include/tie_cuda.h): context lifetime, error model, device and host-buffer entry
// points.  No torch or C++ types cross the boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <pthread.h>
#include <thread>
#include <vector>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../../include/tie_cuda.h"
#include "tie_internal.cuh"

namespace tie {
namespace capi {

namespace {
thread_local std::string g_msg;
thread_local uint64_t g_launches = 0;
}  // namespace

int set_error(int code, const std::string& msg) {
  g_msg = msg;
  return code;
}

int cuda_error(cudaError_t e, const char* where) {
  return set_error(TIE_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

void count_launch(uint64_t k) { g_launches += k; }

void* scratch(tie_ctx* ctx, size_t bytes, cudaStream_t s) {
  if (bytes <= ctx->scratch_bytes) return ctx->scratch;
  // growth happens outside steady state (first call at a new size): drain users first
  cudaStreamSynchronize(s);
  cudaDeviceSynchronize();
  if (ctx->scratch) cudaFree(ctx->scratch);
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  const size_t want = bytes + bytes / 8 + (1 << 20);
  if (cudaMalloc(&ctx->scratch, want) != cudaSuccess) return nullptr;
  ctx->scratch_bytes = want;
  return ctx->scratch;
}

}  // namespace capi

namespace {
cudaEvent_t prof_event(tie_ctx* ctx) {
  if (ctx->prof_used == ctx->prof_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->prof_pool.push_back(e);
  }
  return ctx->prof_pool[ctx->prof_used++];
}
}  // namespace

ProfScope::ProfScope(tie_ctx* c, const char* name, cudaStream_t st) : ctx(c), s(st) {
  if (!ctx || !ctx->prof_on) return;
  tie_ctx::ProfRec r{name, prof_event(ctx), prof_event(ctx)};
  cudaEventRecord(r.a, s);
  idx = ctx->prof.size();
  ctx->prof.push_back(r);
}

ProfScope::~ProfScope() {
  if (idx != (size_t)-1) cudaEventRecord(ctx->prof[idx].b, s);
}

}  // namespace tie

using tie::capi::cuda_error;
using tie::capi::set_error;

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

#define TIE_CUDA_TRY(expr, where)                      \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return cuda_error(_e, where); \
  } while (0)

int check_ctx(const tie_ctx* ctx) {
  if (!ctx) return set_error(TIE_EINVALID, "tie: null context");
  return TIE_OK;
}

// decode the device error word into the reference's exception type + message
int decode_error(uint64_t word, const char* op) {
  using namespace tie::dev;
  const uint64_t idx = word >> 8;
  const uint32_t why = (uint32_t)(word & 0xff);
  const std::string at = std::string(op) + ": item " + std::to_string(idx) + ": ";
  switch (why) {
    case kMuNotFinite: return set_error(TIE_EDOMAIN, at + "LogTParams: mu must be finite");
    case kSigmaBad:
      return set_error(TIE_EDOMAIN, at + "LogTParams: sigma must be finite and > 0");
    case kXmaxBad:
      return set_error(TIE_EDOMAIN, at + "CensoredLogT: x_max must be finite and > 0");
    case kScoreNotFinite:
      return set_error(TIE_EDOMAIN, at + "compute_score: arguments must be finite");
    case kExpectationNonPos:
      return set_error(TIE_EDOMAIN, at + "compute_score: expectation must be > 0");
    case kCvarBelowE:
      return set_error(TIE_EINVALID,
                       at + "compute_score: cvar below expectation violates the invariant");
    case kKeyNotFinite:
      return set_error(TIE_EDOMAIN, at + "WaitingQueue::push: key must be finite");
    case kDuplicateId: return set_error(TIE_EINVALID, at + "WaitingQueue::push: id already queued");
    case kSampleBad:
      return set_error(TIE_EDOMAIN, at + "fit_logt_fixed_nu: samples must be finite and > 0");
    case kKsCdfRange:
      return set_error(TIE_EDOMAIN, at + "ks_test: cdf returned a value outside [0, 1]");
    default: return set_error(TIE_ECUDA, at + "unknown device error");
  }
}

int validate_alpha(double alpha) {
  if (!(alpha >= 0.0 && alpha < 1.0))
    return set_error(TIE_EDOMAIN, "censored_cvar: alpha must lie in [0, 1)");
  return TIE_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

// ====================================================================== context
extern "C" {

const char* tie_last_error(void) { return tie::capi::g_msg.c_str(); }
const char* tie_version(void) { return "tie-b200 0.1.0 (sm_100a)"; }

uint64_t tie_launch_count(int reset) {
  const uint64_t v = tie::capi::g_launches;
  if (reset) tie::capi::g_launches = 0;
  return v;
}

int tie_ctx_create(int device, const double* samples, int n_samples, double nu,
                   double sigma_table_max, tie_ctx** out) {
  if (!out) return set_error(TIE_EINVALID, "tie_ctx_create: null output handle");
  *out = nullptr;
  if (!(nu > 0.0) || !std::isfinite(nu))
    return set_error(TIE_EDOMAIN, "McContext: nu must be finite and > 0");
  if (n_samples <= 0 || !samples)
    return set_error(TIE_EDOMAIN, "McContext: n_samples must be > 0");
  for (int i = 0; i < n_samples; ++i) {
    if (!std::isfinite(samples[i]))
      return set_error(TIE_EINVALID, "tie_ctx_create: samples must be finite");
    if (i && samples[i] < samples[i - 1])
      return set_error(TIE_EINVALID, "tie_ctx_create: samples must be sorted ascending");
  }
  if (!(sigma_table_max > 0.0)) sigma_table_max = 4.0;
  sigma_table_max = std::min(sigma_table_max, 32.0);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_error(TIE_ECUDA, "tie_ctx_create: no CUDA device available");
  if (device < 0 || device >= ndev) return set_error(TIE_EINVALID, "tie_ctx_create: bad device");
  DeviceGuard g(device);

  tie_ctx* ctx = new tie_ctx();
  ctx->device = device;
  ctx->nu = nu;
  ctx->N = n_samples;
  ctx->sigma_table_max = sigma_table_max;
  ctx->host_samples.assign(samples, samples + n_samples);
  // request-invariant Student-t constants, computed with the host libm like the reference
  auto& td = ctx->td;
  td.nu = nu;
  td.a = 0.5 * nu;
  td.b = 0.5;
  td.logbeta = std::lgamma(td.a) + std::lgamma(td.b) - std::lgamma(td.a + td.b);
  td.thresh = (td.a + 1.0) / (td.a + td.b + 2.0);
  tie::host::make_cf_table(td.a, td.b, &td.ab);
  tie::host::make_cf_table(td.b, td.a, &td.ba);

  auto fail = [&](cudaError_t e, const char* where) {
    tie_ctx_destroy(ctx);
    return cuda_error(e, where);
  };
  cudaError_t e;
  if ((e = cudaMalloc(&ctx->d_err, sizeof(unsigned long long))) != cudaSuccess)
    return fail(e, "tie_ctx_create(err)");
  if ((e = cudaMemset(ctx->d_err, 0xff, sizeof(unsigned long long))) != cudaSuccess)
    return fail(e, "tie_ctx_create(err)");
  if ((e = cudaMallocHost(&ctx->h_err, sizeof(unsigned long long))) != cudaSuccess)
    return fail(e, "tie_ctx_create(pinned)");
  if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e, "tie_ctx_create(stream)");
  if ((e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(e, "tie_ctx_create(stream)");
  for (auto& ev : ctx->ev)
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
      return fail(e, "tie_ctx_create(event)");
  if ((e = tie::dev::build_context_tables(ctx)) != cudaSuccess)
    return fail(e, "tie_ctx_create(tables)");
  *out = ctx;
  return TIE_OK;
}

uint64_t tie_ctx_device_bytes(const tie_ctx* ctx) { return ctx ? ctx->table_bytes : 0; }

int tie_ctx_create_mc(int device, double nu, int n_samples, uint64_t seed, tie_ctx** out) {
  std::vector<double> y;
  try {
    y = tie::host::mc_samples(nu, n_samples, seed);
  } catch (const std::domain_error& ex) {
    return set_error(TIE_EDOMAIN, ex.what());
  }
  return tie_ctx_create(device, y.data(), n_samples, nu, 0.0, out);
}

void tie_ctx_destroy(tie_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->device);
  cudaDeviceSynchronize();
  cudaFree(ctx->d_Y);
  cudaFree(ctx->d_ybucket);
  cudaFree(ctx->d_table);
  cudaFree(ctx->d_tail);
  cudaFree(ctx->d_bins);
  cudaFree(ctx->d_ka_table);
  cudaFree(ctx->d_err);
  cudaFree(ctx->scratch);
  cudaFree(ctx->io);
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : ctx->prof_pool) cudaEventDestroy(ev);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  delete ctx;
}

int tie_profile(tie_ctx* ctx, int enable) {
  if (int rc = check_ctx(ctx)) return rc;
  DeviceGuard g(ctx->device);
  cudaDeviceSynchronize();
  ctx->prof_on = enable != 0;
  ctx->prof.clear();
  ctx->prof_used = 0;
  return TIE_OK;
}

int tie_profile_report(tie_ctx* ctx, char* buf, size_t len) {
  if (int rc = check_ctx(ctx)) return rc;
  DeviceGuard g(ctx->device);
  TIE_CUDA_TRY(cudaDeviceSynchronize(), "tie_profile_report");
  std::vector<std::string> names;
  std::vector<double> total;
  std::vector<long> count;
  for (const auto& r : ctx->prof) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
    size_t k = 0;
    while (k < names.size() && names[k] != r.name) ++k;
    if (k == names.size()) {
      names.push_back(r.name);
      total.push_back(0.0);
      count.push_back(0);
    }
    total[k] += ms;
    count[k] += 1;
  }
  std::string out;
  for (size_t k = 0; k < names.size(); ++k)
    out += names[k] + "\t" + std::to_string(count[k]) + "\t" + std::to_string(total[k]) + "\n";
  if (buf && len) {
    std::snprintf(buf, len, "%s", out.c_str());
  }
  return out.size() < len ? TIE_OK : set_error(TIE_EINVALID, "tie_profile_report: buffer too small");
}

int tie_ctx_samples(const tie_ctx* ctx, double* host_out, int n) {
  if (int rc = check_ctx(ctx)) return rc;
  if (n != ctx->N) return set_error(TIE_EINVALID, "tie_ctx_samples: size mismatch");
  std::memcpy(host_out, ctx->host_samples.data(), sizeof(double) * n);
  return TIE_OK;
}

int tie_ctx_info(const tie_ctx* ctx, double* nu, int* n_samples, int* device) {
  if (int rc = check_ctx(ctx)) return rc;
  if (nu) *nu = ctx->nu;
  if (n_samples) *n_samples = ctx->N;
  if (device) *device = ctx->device;
  return TIE_OK;
}

int tie_sync(tie_ctx* ctx, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  DeviceGuard g(ctx->device);
  cudaStream_t s = as_stream(stream);
  TIE_CUDA_TRY(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s),
               "tie_sync");
  TIE_CUDA_TRY(cudaStreamSynchronize(s), "tie_sync");
  const unsigned long long w = *ctx->h_err;
  if (w == ~0ull) return TIE_OK;
  TIE_CUDA_TRY(cudaMemsetAsync(ctx->d_err, 0xff, sizeof(unsigned long long), s), "tie_sync");
  TIE_CUDA_TRY(cudaStreamSynchronize(s), "tie_sync");
  return decode_error(w, ctx->err_op);
}

// ====================================================================== scalar helpers
int tie_compute_beta(int adaptive, double beta_fixed, double beta_max, double q_sat,
                     uint64_t queue_len, double* beta_out) {
  if (!beta_out) return set_error(TIE_EINVALID, "tie_compute_beta: null output");
  if (!adaptive) {
    if (beta_fixed < 0.0) return set_error(TIE_EDOMAIN, "compute_beta: beta_fixed must be >= 0");
    *beta_out = beta_fixed;
    return TIE_OK;
  }
  if (!(beta_max >= 0.0) || !(q_sat > 0.0))
    return set_error(TIE_EDOMAIN, "compute_beta: beta_max must be >= 0 and q_sat > 0");
  *beta_out = beta_max * std::min(1.0, (double)queue_len / q_sat);
  return TIE_OK;
}

double tie_t_quantile(double p, double nu) {
  try {
    return tie::host::t_quantile(p, nu);
  } catch (const std::exception& e) {
    set_error(TIE_EDOMAIN, e.what());
    return std::nan("");
  }
}

double tie_t_cdf(double y, double nu) {
  try {
    return tie::host::t_cdf(y, nu);
  } catch (const std::exception& e) {
    set_error(TIE_EDOMAIN, e.what());
    return std::nan("");
  }
}

// ====================================================================== device entry points
static int score_impl(tie_ctx* ctx, const double* mu, const double* sigma, const void* x_max,
                      bool u32, uint64_t n, double alpha, double beta, double* E, double* C,
                      double* S, uint64_t* keys, unsigned long long* minmax, unsigned flags, cudaStream_t s,
                      const char* op) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = validate_alpha(alpha)) return rc;
  if (n && (!mu || !sigma || !x_max)) return set_error(TIE_EINVALID, std::string(op) + ": null input");
  DeviceGuard g(ctx->device);
  ctx->err_op = op;
  const cudaError_t e = tie::dev::launch_score(ctx, mu, sigma, x_max, u32, n, alpha, beta, E, C,
                                               S, keys, minmax, flags, s);
  if (e != cudaSuccess) return cuda_error(e, op);
  return TIE_OK;
}

int tie_score(tie_ctx* ctx, const double* mu, const double* sigma, const double* x_max,
              uint64_t n, double alpha, double beta, double* E, double* cvar, double* score,
              unsigned flags, void* stream) {
  return score_impl(ctx, mu, sigma, x_max, false, n, alpha, beta, E, cvar, score, nullptr,
                    nullptr, flags, as_stream(stream), "tie_score");
}

int tie_score_u32(tie_ctx* ctx, const double* mu, const double* sigma,
                  const uint32_t* max_tokens, uint64_t n, double alpha, double beta, double* E,
                  double* cvar, double* score, unsigned flags, void* stream) {
  return score_impl(ctx, mu, sigma, max_tokens, true, n, alpha, beta, E, cvar, score, nullptr,
                    nullptr, flags, as_stream(stream), "tie_score");
}

int tie_rank(tie_ctx* ctx, const double* key, const uint64_t* ids, uint64_t n, uint64_t* order,
             void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (n && (!key || !order)) return set_error(TIE_EINVALID, "tie_rank: null pointer");
  DeviceGuard g(ctx->device);
  ctx->err_op = "tie_rank";
  const cudaError_t e = tie::dev::launch_rank(ctx, key, ids, n, order, as_stream(stream));
  if (e != cudaSuccess) return cuda_error(e, "tie_rank");
  return TIE_OK;
}

int tie_score_rank(tie_ctx* ctx, const double* mu, const double* sigma,
                   const uint32_t* max_tokens, uint64_t n, double alpha, double beta, double* E,
                   double* cvar, double* score, uint64_t* order, unsigned flags, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (n && !order) return set_error(TIE_EINVALID, "tie_score_rank: null order");
  if (n == 0) return TIE_OK;
  DeviceGuard g(ctx->device);
  cudaStream_t s = as_stream(stream);
  const tie::dev::RankPrep prep = tie::dev::rank_prepare(ctx, n, s);
  if (!prep.keys) return set_error(TIE_ECUDA, "tie_score_rank: scratch allocation failed");
  if (int rc = score_impl(ctx, mu, sigma, max_tokens, true, n, alpha, beta, E, cvar, score,
                          prep.keys, prep.minmax, flags, s, "tie_score_rank"))
    return rc;
  const cudaError_t e = tie::dev::rank_prepared(ctx, n, order, s);
  if (e != cudaSuccess) return cuda_error(e, "tie_score_rank");
  return TIE_OK;
}

int tie_fit(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu, double* mu,
            double* sigma, double* log_likelihood, int32_t* iterations, uint8_t* converged,
            uint8_t* degenerate, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (K < 3)
    return set_error(TIE_EINVALID, "fit_logt_fixed_nu: need at least 3 samples, got " +
                                       std::to_string(K));
  if (!(nu > 0.0) || !std::isfinite(nu))
    return set_error(TIE_EDOMAIN, "fit_logt_fixed_nu: nu must be finite and > 0");
  if (P && (!x || !mu || !sigma)) return set_error(TIE_EINVALID, "tie_fit: null pointer");
  DeviceGuard g(ctx->device);
  ctx->err_op = "tie_fit";
  const cudaError_t e = tie::dev::launch_fit(ctx, x, P, K, nu, mu, sigma, log_likelihood,
                                             iterations, converged, degenerate, as_stream(stream));
  if (e != cudaSuccess) return cuda_error(e, "tie_fit");
  return TIE_OK;
}

int tie_logt_loglik(tie_ctx* ctx, const double* x, uint64_t K, const double* mu,
                    const double* sigma, uint64_t P, double nu, double* ll, double* grad,
                    void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (K < 1) return set_error(TIE_EINVALID, "logt_loglik: need at least 1 samples, got 0");
  if (!(nu > 0.0)) return set_error(TIE_EDOMAIN, "logt_loglik: sigma and nu must be > 0");
  DeviceGuard g(ctx->device);
  ctx->err_op = "tie_logt_loglik";
  const cudaError_t e =
      tie::dev::launch_loglik(ctx, x, K, mu, sigma, P, nu, ll, grad, as_stream(stream));
  if (e != cudaSuccess) return cuda_error(e, "tie_logt_loglik");
  return TIE_OK;
}

// ====================================================================== host-buffer variants
// Each copies inputs H2D on the context's streams, runs the device path, copies results
// back and synchronises; the device error word is checked before returning.

static char* io_buffer(tie_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->io_bytes) return (char*)ctx->io;
  cudaDeviceSynchronize();
  if (ctx->io) cudaFree(ctx->io);
  ctx->io = nullptr;
  ctx->io_bytes = 0;
  const size_t want = bytes + bytes / 8 + (1 << 20);
  if (cudaMalloc(&ctx->io, want) != cudaSuccess) return nullptr;
  ctx->io_bytes = want;
  return (char*)ctx->io;
}

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// A small persistent pool of host threads for the pageable-buffer copies of the *_host entry
// points: one thread copies pageable memory at ~10 GB/s, 4-8 at ~60 GB/s (B200 box host,
// tools/memcpy_probe.cpp), and a persistent pool avoids a thread spawn per copy.  run()
// splits [0, bytes) into 1 MB tasks over the workers and the calling thread.
namespace {
class CopyPool {
 public:
  struct Seg {
    void* dst;
    const void* src;
    size_t bytes;
  };
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy(void* dst, const void* src, size_t bytes) { copy({Seg{dst, src, bytes}}); }
  // the segments' copies, split into 1 MB tasks over the workers and the calling thread
  void copy(std::initializer_list<Seg> segs) {
    Job job;
    size_t total = 0;
    for (const Seg& g : segs) {
      if (job.nseg == kMaxSeg) break;
      job.seg[job.nseg] = g;
      job.first[job.nseg++] = total;
      total += (g.bytes + kTask - 1) / kTask;
    }
    job.ntask = total;
    // (a forked child has no workers, and its mutexes may be mid-use: copy serially)
    if (workers_.empty() || forked_.load() || total <= 2) {
      for (int g = 0; g < job.nseg; ++g) std::memcpy(job.seg[g].dst, job.seg[g].src, job.seg[g].bytes);
      return;
    }
    std::lock_guard<std::mutex> one(call_);  // one parallel copy at a time
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = &job;
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work(job);
    while (job.done.load(std::memory_order_acquire) < job.ntask) std::this_thread::yield();
    {
      std::lock_guard<std::mutex> lk(m_);
      job_ = nullptr;  // a worker arriving from now on finds no job
    }
    // workers that took the job hold a reference until they leave it
    while (job.refs.load(std::memory_order_acquire) != 0) std::this_thread::yield();
  }

 private:
  static constexpr size_t kTask = 1u << 20;
  static constexpr int kMaxSeg = 4;
  struct Job {
    Seg seg[kMaxSeg];
    size_t first[kMaxSeg];
    int nseg = 0;
    size_t ntask = 0;
    std::atomic<size_t> next{0}, done{0};
    std::atomic<int> refs{0};
  };
  CopyPool() {
    pthread_atfork(nullptr, nullptr, [] { forked_.store(true); });
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned nw = std::min(7u, hw > 1 ? hw - 1 : 0u);
    for (unsigned t = 0; t < nw; ++t)
      workers_.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          // spin ~0.5 ms for the next job (a call issues several back to back), then sleep
          const auto t0 = std::chrono::steady_clock::now();
          while (gen_.load(std::memory_order_acquire) == seen && !stop_.load() &&
                 std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(500))
            std::this_thread::yield();
          Job* j = nullptr;
          {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return stop_.load() || gen_.load() != seen; });
            if (stop_.load()) return;
            seen = gen_.load();
            j = job_;
            if (j) j->refs.fetch_add(1);
          }
          if (j) {
            work(*j);
            j->refs.fetch_sub(1, std::memory_order_release);
          }
        }
      });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_.store(true);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  static void work(Job& j) {
    for (size_t t; (t = j.next.fetch_add(1)) < j.ntask;) {
      int g = 0;
      while (g + 1 < j.nseg && t >= j.first[g + 1]) ++g;
      const size_t lo = (t - j.first[g]) * kTask;
      const size_t len = std::min(kTask, j.seg[g].bytes - lo);
      std::memcpy(static_cast<char*>(j.seg[g].dst) + lo,
                  static_cast<const char*>(j.seg[g].src) + lo, len);
      j.done.fetch_add(1, std::memory_order_release);
    }
  }
  std::vector<std::thread> workers_;
  std::mutex m_, call_;
  std::condition_variable cv_;
  std::atomic<uint64_t> gen_{0};
  std::atomic<bool> stop_{false};
  Job* job_ = nullptr;
  static inline std::atomic<bool> forked_{false};
};
}  // namespace

static char* host_stage(tie_ctx* ctx, size_t bytes) {  // grow-only, mapped pinned
  if (bytes <= ctx->h_stage_bytes) return (char*)ctx->h_stage;
  cudaDeviceSynchronize();
  if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
  ctx->h_stage = nullptr;
  ctx->h_stage_bytes = 0;
  const size_t want = bytes + bytes / 8 + (1 << 20);
  if (cudaHostAlloc(&ctx->h_stage, want, cudaHostAllocMapped) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  ctx->h_stage_bytes = want;
  return (char*)ctx->h_stage;
}

// the device address of a pinned (page-locked, UVA-mapped) host buffer; nullptr for pageable
// or null pointers (the caller then stages copies)
static void* mapped_device_ptr(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a{};
  const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess &&
                  a.type == cudaMemoryTypeHost && a.devicePointer != nullptr;
  cudaGetLastError();  // a pageable pointer is not an error here
  return ok ? a.devicePointer : nullptr;
}

int tie_score_host(tie_ctx* ctx, const double* mu, const double* sigma, const double* x_max,
                   uint64_t n, double alpha, double beta, double* E, double* cvar, double* score,
                   unsigned flags) {
  if (int rc = check_ctx(ctx)) return rc;
  if (n == 0) return TIE_OK;
  DeviceGuard g(ctx->device);
  char* b = io_buffer(ctx, 6 * al(8 * n));
  if (!b) return set_error(TIE_ECUDA, "tie_score_host: device allocation failed");
  double* d_mu = (double*)b;
  double* d_sg = (double*)(b + al(8 * n));
  double* d_xm = (double*)(b + 2 * al(8 * n));
  double* d_E = E ? (double*)(b + 3 * al(8 * n)) : nullptr;
  double* d_C = cvar ? (double*)(b + 4 * al(8 * n)) : nullptr;
  double* d_S = score ? (double*)(b + 5 * al(8 * n)) : nullptr;
  cudaStream_t s = ctx->stream;
  TIE_CUDA_TRY(cudaMemcpyAsync(d_mu, mu, 8 * n, cudaMemcpyHostToDevice, s), "tie_score_host");
  TIE_CUDA_TRY(cudaMemcpyAsync(d_sg, sigma, 8 * n, cudaMemcpyHostToDevice, s), "tie_score_host");
  TIE_CUDA_TRY(cudaMemcpyAsync(d_xm, x_max, 8 * n, cudaMemcpyHostToDevice, s), "tie_score_host");
  if (int rc = tie_score(ctx, d_mu, d_sg, d_xm, n, alpha, beta, d_E, d_C, d_S, flags, s)) return rc;
  if (E) TIE_CUDA_TRY(cudaMemcpyAsync(E, d_E, 8 * n, cudaMemcpyDeviceToHost, s), "tie_score_host");
  if (cvar)
    TIE_CUDA_TRY(cudaMemcpyAsync(cvar, d_C, 8 * n, cudaMemcpyDeviceToHost, s), "tie_score_host");
  if (score)
    TIE_CUDA_TRY(cudaMemcpyAsync(score, d_S, 8 * n, cudaMemcpyDeviceToHost, s), "tie_score_host");
  return tie_sync(ctx, s);
}

int tie_score_rank_host(tie_ctx* ctx, const double* mu, const double* sigma,
                        const uint32_t* max_tokens, uint64_t n, double alpha, double beta,
                        double* score, uint64_t* order, unsigned flags) {
  if (int rc = check_ctx(ctx)) return rc;
  if (int rc = validate_alpha(alpha)) return rc;
  if (n == 0) return TIE_OK;
  if (!mu || !sigma || !max_tokens || !order)
    return set_error(TIE_EINVALID, "tie_score_rank_host: null pointer");
  DeviceGuard g(ctx->device);
  char* b = io_buffer(ctx, 2 * al(8 * n) + al(4 * n) + al(8 * n) + al(8 * n));
  if (!b) return set_error(TIE_ECUDA, "tie_score_rank_host: device allocation failed");
  double* d_mu = (double*)b;
  double* d_sg = (double*)(b + al(8 * n));
  uint32_t* d_mt = (uint32_t*)(b + 2 * al(8 * n));
  double* d_S = score ? (double*)(b + 2 * al(8 * n) + al(4 * n)) : nullptr;
  uint64_t* d_order = (uint64_t*)(b + 3 * al(8 * n) + al(4 * n));
  cudaStream_t s = ctx->stream, cs = ctx->copy_stream;
  const tie::dev::RankPrep prep = tie::dev::rank_prepare(ctx, n, s);
  if (!prep.keys) return set_error(TIE_ECUDA, "tie_score_rank_host: scratch allocation failed");
  ctx->err_op = "tie_score_rank_host";
  // pinned (UVA-mapped) inputs: the score kernel streams them over PCIe itself -- no copy
  // engine setup per chunk, the reads overlap the scoring at the request granularity
  // (tools/e2e_probe.py on B200, 1M requests: 604 vs 614 us for the 2-chunk H2D pipeline
  // below, which pageable inputs still take)
  static const int zc_in = getenv("TIE_ZERO_COPY_IN") ? atoi(getenv("TIE_ZERO_COPY_IN")) : 1;
  const void* m_mu = zc_in ? mapped_device_ptr(mu) : nullptr;
  const void* m_sg = zc_in ? mapped_device_ptr(sigma) : nullptr;
  const void* m_mt = zc_in ? mapped_device_ptr(max_tokens) : nullptr;
  // pageable caller buffers (a std::vector / NumPy array): copied by the host pool into the
  // context's pinned staging in chunks, each chunk scored zero-copy while the next is copied
  // -- the driver's own pageable copies run at ~10 GB/s on one thread
  static const bool no_stage = getenv("TIE_NO_HOST_STAGE") != nullptr;  // A/B switch
  const bool big = n >= (1u << 18) && !no_stage;
  const bool stage_in = big && zc_in && !(m_mu && m_sg && m_mt);
  const bool stage_out = big && !mapped_device_ptr(order) && tie::dev::rank_output_coalesced(n);
  char* hs = (stage_in || stage_out)
                 ? host_stage(ctx, 2 * al(8 * n) + al(4 * n) + al(8 * n))
                 : nullptr;
  uint64_t* h_order = hs && stage_out ? (uint64_t*)(hs + 2 * al(8 * n) + al(4 * n)) : nullptr;
  if (hs && stage_in) {
    double* h_mu = (double*)hs;
    double* h_sg = (double*)(hs + al(8 * n));
    uint32_t* h_mt = (uint32_t*)(hs + 2 * al(8 * n));
    static const int chunks =
        getenv("TIE_STAGE_CHUNKS") ? std::max(1, atoi(getenv("TIE_STAGE_CHUNKS"))) : 2;
    const uint64_t step = ((n + chunks - 1) / chunks + 1023) & ~(uint64_t)1023;
    CopyPool& pool = CopyPool::get();
    for (uint64_t lo = 0; lo < n; lo += step) {
      const uint64_t m = std::min<uint64_t>(step, n - lo);
      pool.copy({{h_mu + lo, mu + lo, 8 * m}, {h_sg + lo, sigma + lo, 8 * m},
                 {h_mt + lo, max_tokens + lo, 4 * m}});
      const cudaError_t e = tie::dev::launch_score(
          ctx, (const double*)mapped_device_ptr(h_mu) + lo,
          (const double*)mapped_device_ptr(h_sg) + lo,
          (const uint32_t*)mapped_device_ptr(h_mt) + lo, true, m, alpha, beta, nullptr,
          nullptr, d_S ? d_S + lo : nullptr, prep.keys + lo, prep.minmax,
          flags & TIE_SCORE_EXACT, s, lo);
      if (e != cudaSuccess) return cuda_error(e, "tie_score_rank_host");
    }
  } else if (m_mu && m_sg && m_mt) {
    const cudaError_t e = tie::dev::launch_score(
        ctx, (const double*)m_mu, (const double*)m_sg, m_mt, true, n, alpha, beta, nullptr,
        nullptr, d_S, prep.keys, prep.minmax, flags & TIE_SCORE_EXACT, s, 0);
    if (e != cudaSuccess) return cuda_error(e, "tie_score_rank_host");
  } else {
  // pipeline: H2D of chunk c+1 (copy stream) overlaps scoring of chunk c (compute stream)
  // 2 chunks: the second half's H2D overlaps the first half's scoring; every extra copy costs
  // ~3 us of DMA setup, more than the finer overlap wins (tools/e2e_probe.py on B200:
  // 1M requests, 1/2/3/8/16 chunks -> 633/626/644/698/801 us)
  static const int max_chunks = getenv("TIE_H2D_CHUNKS") ? atoi(getenv("TIE_H2D_CHUNKS")) : 2;
  const int chunks = std::max(1, n >= (1u << 18) ? max_chunks : 1);
  const uint64_t step = (n + chunks - 1) / chunks;
  TIE_CUDA_TRY(cudaEventRecord(ctx->ev[0], s), "tie_score_rank_host");
  TIE_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[0], 0), "tie_score_rank_host");
  for (int c = 0; c < chunks; ++c) {
    const uint64_t lo = std::min<uint64_t>(n, c * step), hi = std::min<uint64_t>(n, lo + step);
    if (lo >= hi) break;
    const uint64_t m = hi - lo;
    TIE_CUDA_TRY(cudaMemcpyAsync(d_mu + lo, mu + lo, 8 * m, cudaMemcpyHostToDevice, cs), "h2d");
    TIE_CUDA_TRY(cudaMemcpyAsync(d_sg + lo, sigma + lo, 8 * m, cudaMemcpyHostToDevice, cs), "h2d");
    TIE_CUDA_TRY(cudaMemcpyAsync(d_mt + lo, max_tokens + lo, 4 * m, cudaMemcpyHostToDevice, cs),
                 "h2d");
    TIE_CUDA_TRY(cudaEventRecord(ctx->ev[1 + (c & 3)], cs), "tie_score_rank_host");
    TIE_CUDA_TRY(cudaStreamWaitEvent(s, ctx->ev[1 + (c & 3)], 0), "tie_score_rank_host");
    const cudaError_t e = tie::dev::launch_score(ctx, d_mu + lo, d_sg + lo, d_mt + lo, true, m,
                                                 alpha, beta, nullptr, nullptr,
                                                 d_S ? d_S + lo : nullptr, prep.keys + lo,
                                                 prep.minmax, flags & TIE_SCORE_EXACT, s, lo);
    if (e != cudaSuccess) return cuda_error(e, "tie_score_rank_host");
  }
  }  // (zero-copy inputs | staged pipeline)
  // pinned (page-locked, UVA-mapped) output: the sort's last kernel writes the dispatch
  // order straight into host memory, so the D2H overlaps the sort instead of following it
  static const int zero_copy = getenv("TIE_NO_ZERO_COPY") ? 0 : 1;  // A/B switch
  uint64_t* m_order = !zero_copy || !tie::dev::rank_output_coalesced(n) ? nullptr
                     : h_order ? (uint64_t*)mapped_device_ptr(h_order)
                               : (uint64_t*)mapped_device_ptr(order);
  const bool mapped = m_order != nullptr;
  cudaError_t e = tie::dev::rank_prepared(ctx, n, mapped ? m_order : d_order, s);
  if (e != cudaSuccess) return cuda_error(e, "tie_score_rank_host");
  if (!mapped)
    TIE_CUDA_TRY(cudaMemcpyAsync(order, d_order, 8 * n, cudaMemcpyDeviceToHost, s), "d2h");
  if (score) TIE_CUDA_TRY(cudaMemcpyAsync(score, d_S, 8 * n, cudaMemcpyDeviceToHost, s), "d2h");
  if (int rc = tie_sync(ctx, s)) return rc;
  if (mapped && h_order) CopyPool::get().copy(order, h_order, 8 * n);  // staged order out
  return TIE_OK;
}

int tie_rank_host(tie_ctx* ctx, const double* key, const uint64_t* ids, uint64_t n,
                  uint64_t* order) {
  if (int rc = check_ctx(ctx)) return rc;
  if (n == 0) return TIE_OK;
  DeviceGuard g(ctx->device);
  char* b = io_buffer(ctx, 3 * al(8 * n));
  if (!b) return set_error(TIE_ECUDA, "tie_rank_host: device allocation failed");
  double* d_key = (double*)b;
  uint64_t* d_ids = ids ? (uint64_t*)(b + al(8 * n)) : nullptr;
  uint64_t* d_order = (uint64_t*)(b + 2 * al(8 * n));
  cudaStream_t s = ctx->stream;
  TIE_CUDA_TRY(cudaMemcpyAsync(d_key, key, 8 * n, cudaMemcpyHostToDevice, s), "h2d");
  if (ids) TIE_CUDA_TRY(cudaMemcpyAsync(d_ids, ids, 8 * n, cudaMemcpyHostToDevice, s), "h2d");
  if (int rc = tie_rank(ctx, d_key, d_ids, n, d_order, s)) return rc;
  TIE_CUDA_TRY(cudaMemcpyAsync(order, d_order, 8 * n, cudaMemcpyDeviceToHost, s), "d2h");
  return tie_sync(ctx, s);
}

// final step of the sharded score+rank: merge G runs sorted by (score, id) (device buffers)
int tie_merge_runs(tie_ctx* ctx, const double* keys, const uint64_t* ids, int G,
                   uint64_t stride, const uint64_t* lens, uint64_t* out_ids, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (G < 0 || G > 128) return set_error(TIE_EINVALID, "tie_merge_runs: G must be in [0, 128]");
  if (G && (!keys || !ids || !lens || !out_ids))
    return set_error(TIE_EINVALID, "tie_merge_runs: null pointer");
  for (int g = 0; g < G; ++g)
    if (lens[g] > stride) return set_error(TIE_EINVALID, "tie_merge_runs: run longer than stride");
  DeviceGuard dg(ctx->device);
  ctx->err_op = "tie_merge_runs";
  const cudaError_t e = tie::dev::launch_merge_runs(ctx, keys, ids, G, stride, lens, out_ids,
                                                    as_stream(stream));
  if (e != cudaSuccess) return cuda_error(e, "tie_merge_runs");
  return TIE_OK;
}

// cmd_fit's per-prompt analysis (tools/main.cpp:527-562), device buffers
int tie_fit_report(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                   unsigned families, double* fits, double* tail, void* stream) {
  if (int rc = check_ctx(ctx)) return rc;
  if (K < 5) return set_error(TIE_EINVALID, "ks_test: need at least 5 samples");
  if (!(nu > 0.0) || !std::isfinite(nu))
    return set_error(TIE_EDOMAIN, "fit_logt_fixed_nu: nu must be finite and > 0");
  if (families == 0 || families > 15)
    return set_error(TIE_EINVALID, "tie_fit_report: families must be a non-empty subset of 15");
  if (P && (!x || !fits)) return set_error(TIE_EINVALID, "tie_fit_report: null pointer");
  DeviceGuard g(ctx->device);
  ctx->err_op = "tie_fit_report";
  const cudaError_t e = tie::dev::launch_fit_report(ctx, x, P, K, nu, families, fits, tail,
                                                    as_stream(stream));
  if (e != cudaSuccess) return cuda_error(e, "tie_fit_report");
  return TIE_OK;
}

int tie_fit_report_host(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                        unsigned families, double* fits, double* tail) {
  if (int rc = check_ctx(ctx)) return rc;
  if (P == 0) return TIE_OK;
  DeviceGuard g(ctx->device);
  char* b = io_buffer(ctx, al(8 * P * K) + al(8 * 40 * P) + al(8 * 5 * P));
  if (!b) return set_error(TIE_ECUDA, "tie_fit_report_host: device allocation failed");
  double* d_x = (double*)b;
  double* d_f = (double*)(b + al(8 * P * K));
  double* d_t = tail ? (double*)(b + al(8 * P * K) + al(8 * 40 * P)) : nullptr;
  cudaStream_t s = ctx->stream;
  TIE_CUDA_TRY(cudaMemcpyAsync(d_x, x, 8 * P * K, cudaMemcpyHostToDevice, s), "h2d");
  TIE_CUDA_TRY(cudaMemcpyAsync(d_f, fits, 8 * 40 * P, cudaMemcpyHostToDevice, s), "h2d");
  if (int rc = tie_fit_report(ctx, d_x, P, K, nu, families, d_f, d_t, s)) return rc;
  TIE_CUDA_TRY(cudaMemcpyAsync(fits, d_f, 8 * 40 * P, cudaMemcpyDeviceToHost, s), "d2h");
  if (tail) TIE_CUDA_TRY(cudaMemcpyAsync(tail, d_t, 8 * 5 * P, cudaMemcpyDeviceToHost, s), "d2h");
  return tie_sync(ctx, s);
}

int tie_fit_host(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu, double* mu,
                 double* sigma, double* log_likelihood, int32_t* iterations, uint8_t* converged,
                 uint8_t* degenerate) {
  if (int rc = check_ctx(ctx)) return rc;
  if (K < 3)
    return set_error(TIE_EINVALID, "fit_logt_fixed_nu: need at least 3 samples, got " +
                                       std::to_string(K));
  if (!(nu > 0.0) || !std::isfinite(nu))
    return set_error(TIE_EDOMAIN, "fit_logt_fixed_nu: nu must be finite and > 0");
  if (P && (!x || !mu || !sigma)) return set_error(TIE_EINVALID, "tie_fit_host: null pointer");
  if (P == 0) return TIE_OK;
  DeviceGuard g(ctx->device);
  ctx->err_op = "tie_fit";
  char* b = io_buffer(ctx, al(8 * P * K) + 3 * al(8 * P) + al(4 * P) + 2 * al(P));
  if (!b) return set_error(TIE_ECUDA, "tie_fit_host: device allocation failed");
  size_t off = 0;
  double* d_x = (double*)(b + off); off += al(8 * P * K);
  double* d_mu = (double*)(b + off); off += al(8 * P);
  double* d_sg = (double*)(b + off); off += al(8 * P);
  double* d_ll = (double*)(b + off); off += al(8 * P);
  int32_t* d_it = (int32_t*)(b + off); off += al(4 * P);
  uint8_t* d_cv = (uint8_t*)(b + off); off += al(P);
  uint8_t* d_dg = (uint8_t*)(b + off);
  cudaStream_t s = ctx->stream, cs = ctx->copy_stream;
  // pinned (UVA-mapped) samples: the fit kernel reads them over PCIe itself (each prompt's K
  // samples once, then ~260 likelihood evaluations on them: the reads hide under the compute)
  // and, with pinned outputs, writes each prompt's results straight back (B200, 1M x 16:
  // 8.0 ms end to end vs 8.95 for the 4-chunk copy pipeline below, 7.9 ms device-only)
  static const int zc_in = getenv("TIE_FIT_ZERO_COPY") ? atoi(getenv("TIE_FIT_ZERO_COPY")) : 2;
  const void* x_dev = zc_in ? mapped_device_ptr(x) : nullptr;
  if (x_dev) {
    // pinned outputs too: the kernel writes each prompt's results straight to the host
    void* o_mu = mapped_device_ptr(mu);
    void* o_sg = mapped_device_ptr(sigma);
    void* o_ll = mapped_device_ptr(log_likelihood);
    void* o_it = mapped_device_ptr(iterations);
    void* o_cv = mapped_device_ptr(converged);
    void* o_dg = mapped_device_ptr(degenerate);
    const bool out_mapped = zc_in >= 2 && o_mu && o_sg && (o_ll || !log_likelihood) &&
                            (o_it || !iterations) && (o_cv || !converged) &&
                            (o_dg || !degenerate);
    if (out_mapped) {
      const cudaError_t e = tie::dev::launch_fit(
          ctx, (const double*)x_dev, P, K, nu, (double*)o_mu, (double*)o_sg,
          (double*)o_ll, (int32_t*)o_it, (uint8_t*)o_cv, (uint8_t*)o_dg, s, 0);
      if (e != cudaSuccess) return cuda_error(e, "tie_fit_host");
      return tie_sync(ctx, s);
    }
    {
      const cudaError_t e = tie::dev::launch_fit(ctx, (const double*)x_dev, P, K, nu, d_mu,
                                                 d_sg, d_ll, d_it, d_cv, d_dg, s, 0);
      if (e != cudaSuccess) return cuda_error(e, "tie_fit_host");
      TIE_CUDA_TRY(cudaMemcpyAsync(mu, d_mu, 8 * P, cudaMemcpyDeviceToHost, s), "d2h");
      TIE_CUDA_TRY(cudaMemcpyAsync(sigma, d_sg, 8 * P, cudaMemcpyDeviceToHost, s), "d2h");
      if (log_likelihood)
        TIE_CUDA_TRY(cudaMemcpyAsync(log_likelihood, d_ll, 8 * P, cudaMemcpyDeviceToHost, s),
                     "d2h");
      if (iterations)
        TIE_CUDA_TRY(cudaMemcpyAsync(iterations, d_it, 4 * P, cudaMemcpyDeviceToHost, s), "d2h");
      if (converged)
        TIE_CUDA_TRY(cudaMemcpyAsync(converged, d_cv, P, cudaMemcpyDeviceToHost, s), "d2h");
      if (degenerate)
        TIE_CUDA_TRY(cudaMemcpyAsync(degenerate, d_dg, P, cudaMemcpyDeviceToHost, s), "d2h");
      return tie_sync(ctx, s);
    }
  }
  // pageable samples (a caller's std::vector / NumPy array), >= 8 MB: the host copy pool
  // fills the context's mapped pinned staging chunk by chunk, each chunk fitted zero-copy
  // while the next is copied; the results land in the staging and the pool copies them out
  // (the driver's pageable copies run single-threaded at ~10 GB/s)
  static const bool no_stage = getenv("TIE_NO_HOST_STAGE") != nullptr;  // A/B switch
  if (!no_stage && 8 * P * K >= (8u << 20)) {
    const size_t ox = 0, omu = ox + al(8 * P * K), osg = omu + al(8 * P), oll = osg + al(8 * P),
                 oit = oll + al(8 * P), ocv = oit + al(4 * P), odg = ocv + al(P),
                 total = odg + al(P);
    char* hs = host_stage(ctx, total);
    char* dv = hs ? (char*)mapped_device_ptr(hs) : nullptr;
    if (dv) {
      CopyPool& pool = CopyPool::get();
      constexpr int kChunks = 4;
      const uint64_t step = (P + kChunks - 1) / kChunks;
      for (uint64_t lo = 0; lo < P; lo += step) {
        const uint64_t m = std::min<uint64_t>(step, P - lo);
        pool.copy((double*)(hs + ox) + lo * K, x + lo * K, 8 * m * K);
        const cudaError_t e = tie::dev::launch_fit(
            ctx, (const double*)(dv + ox) + lo * K, m, K, nu, (double*)(dv + omu) + lo,
            (double*)(dv + osg) + lo, (double*)(dv + oll) + lo, (int32_t*)(dv + oit) + lo,
            (uint8_t*)(dv + ocv) + lo, (uint8_t*)(dv + odg) + lo, s, lo);
        if (e != cudaSuccess) return cuda_error(e, "tie_fit_host");
      }
      if (int rc = tie_sync(ctx, s)) return rc;
      pool.copy({{mu, hs + omu, 8 * P}, {sigma, hs + osg, 8 * P}});
      if (log_likelihood) pool.copy(log_likelihood, hs + oll, 8 * P);
      if (iterations) pool.copy(iterations, hs + oit, 4 * P);
      if (converged) std::memcpy(converged, hs + ocv, P);
      if (degenerate) std::memcpy(degenerate, hs + odg, P);
      return TIE_OK;
    }
  }
  // pipeline over prompt chunks (fits are independent per prompt): all H2D copies queued on
  // the copy stream, chunk c's fit waits for its copy, its results go back on the copy
  // stream behind the H2Ds -- copies in both directions overlap the fits
  const int chunks = P >= (1u << 18) ? 4 : 1;
  const uint64_t step = (P + chunks - 1) / chunks;
  cudaEvent_t* evH = ctx->ev + 1;                                       // ev[1..4]
  cudaEvent_t evF[4] = {ctx->ev[5], ctx->ev[6], ctx->ev[7], ctx->ev[0]};  // after ev[0]'s wait
  TIE_CUDA_TRY(cudaEventRecord(ctx->ev[0], s), "tie_fit_host");
  TIE_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[0], 0), "tie_fit_host");
  for (int c = 0; c < chunks; ++c) {
    const uint64_t lo = std::min<uint64_t>(P, c * step), m = std::min<uint64_t>(P, lo + step) - lo;
    TIE_CUDA_TRY(cudaMemcpyAsync(d_x + lo * K, x + lo * K, 8 * m * K, cudaMemcpyHostToDevice, cs),
                 "h2d");
    TIE_CUDA_TRY(cudaEventRecord(evH[c], cs), "tie_fit_host");
  }
  for (int c = 0; c < chunks; ++c) {
    const uint64_t lo = std::min<uint64_t>(P, c * step), m = std::min<uint64_t>(P, lo + step) - lo;
    TIE_CUDA_TRY(cudaStreamWaitEvent(s, evH[c], 0), "tie_fit_host");
    if (m) {
      const cudaError_t e = tie::dev::launch_fit(ctx, d_x + lo * K, m, K, nu, d_mu + lo,
                                                 d_sg + lo, d_ll + lo, d_it + lo, d_cv + lo,
                                                 d_dg + lo, s, lo);
      if (e != cudaSuccess) return cuda_error(e, "tie_fit_host");
    }
    TIE_CUDA_TRY(cudaEventRecord(evF[c], s), "tie_fit_host");
  }
  for (int c = 0; c < chunks; ++c) {
    const uint64_t lo = std::min<uint64_t>(P, c * step), m = std::min<uint64_t>(P, lo + step) - lo;
    TIE_CUDA_TRY(cudaStreamWaitEvent(cs, evF[c], 0), "tie_fit_host");
    if (!m) continue;
    TIE_CUDA_TRY(cudaMemcpyAsync(mu + lo, d_mu + lo, 8 * m, cudaMemcpyDeviceToHost, cs), "d2h");
    TIE_CUDA_TRY(cudaMemcpyAsync(sigma + lo, d_sg + lo, 8 * m, cudaMemcpyDeviceToHost, cs), "d2h");
    if (log_likelihood)
      TIE_CUDA_TRY(cudaMemcpyAsync(log_likelihood + lo, d_ll + lo, 8 * m, cudaMemcpyDeviceToHost, cs),
                   "d2h");
    if (iterations)
      TIE_CUDA_TRY(cudaMemcpyAsync(iterations + lo, d_it + lo, 4 * m, cudaMemcpyDeviceToHost, cs),
                   "d2h");
    if (converged)
      TIE_CUDA_TRY(cudaMemcpyAsync(converged + lo, d_cv + lo, m, cudaMemcpyDeviceToHost, cs), "d2h");
    if (degenerate)
      TIE_CUDA_TRY(cudaMemcpyAsync(degenerate + lo, d_dg + lo, m, cudaMemcpyDeviceToHost, cs),
                   "d2h");
  }
  TIE_CUDA_TRY(cudaEventRecord(evF[0], cs), "tie_fit_host");
  TIE_CUDA_TRY(cudaStreamWaitEvent(s, evF[0], 0), "tie_fit_host");
  return tie_sync(ctx, s);
}

}  // extern "C"
