// Internal declarations shared by the .cu translation units of libtie_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "host_numerics.hpp"

namespace tie {
namespace dev {

// ---------------------------------------------------------------- error reporting
// First failing request of a batch: kernels atomicMin((index << 8) | reason) into the
// context's device error word; tie_sync() decodes it into the reference's exception.
enum Reason : uint32_t {
  kOk = 0,
  kMuNotFinite = 1,      // LogTParams: mu must be finite                 (dist.cpp:109)
  kSigmaBad = 2,         // LogTParams: sigma must be finite and > 0      (dist.cpp:110)
  kXmaxBad = 3,          // CensoredLogT: x_max must be finite and > 0    (dist.cpp:119)
  kScoreNotFinite = 4,   // compute_score: arguments must be finite       (sched.cpp:20-21)
  kExpectationNonPos = 5,// compute_score: expectation must be > 0        (sched.cpp:22)
  kCvarBelowE = 6,       // compute_score: cvar below expectation         (sched.cpp:23-24)
  kKeyNotFinite = 7,     // WaitingQueue::push: key must be finite        (sched.cpp:60)
  kDuplicateId = 8,      // WaitingQueue::push: id already queued         (sched.cpp:61-63)
  kSampleBad = 9,        // fit_logt_fixed_nu: samples must be finite and > 0 (fit.cpp:22-24)
  kKsCdfRange = 10,      // ks_test: cdf returned a value outside [0, 1]  (fit.cpp:270-271)
};

__device__ __forceinline__ void report(unsigned long long* err, uint64_t index, uint32_t why) {
  atomicMin(err, (unsigned long long)((index << 8) | why));
}

// Fold a thread's [lo, hi] key range into mm[0] = max(~key) and mm[1] = max(key) with one
// pair of atomics per CTA (every thread of the CTA must call it; blockDim % 32 == 0).
__device__ __forceinline__ void key_range_flush(unsigned long long* mm, uint64_t lo,
                                                uint64_t hi) {
  __shared__ uint64_t s_lo[32], s_hi[32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, lo, o);
    const uint64_t b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
      lo = s_lo[w] < lo ? s_lo[w] : lo;
      hi = s_hi[w] > hi ? s_hi[w] : hi;
    }
    if (lo <= hi) {  // the CTA saw at least one key
      atomicMax(mm, (unsigned long long)~lo);
      atomicMax(mm + 1, (unsigned long long)hi);
    }
  }
}

// sample bin of y (see kBinEntry); valid for |y| < 2^(etop - 1022)
__host__ __device__ __forceinline__ uint32_t sample_bin(uint64_t bits, uint32_t e0, uint32_t m,
                                                        uint32_t mid) {
  const uint32_t e = (uint32_t)(bits >> 52) & 0x7ffu;
  if (e < e0) return mid;
  const uint32_t off = ((e - e0) << m) | (uint32_t)((bits >> (52 - m)) & ((1u << m) - 1u));
  return (bits >> 63) ? mid - 1u - off : mid + 1u + off;
}

// |y| centre of the bin holding y (exact double; 0 for the middle bin)
__host__ __device__ __forceinline__ uint64_t sample_bin_centre_bits(uint64_t bits, uint32_t e0,
                                                                    uint32_t m) {
  const uint64_t e = (bits >> 52) & 0x7ffu;
  if (e < e0) return 0;
  const uint64_t keep = ~((1ull << (52 - m)) - 1ull) & 0x7fffffffffffffffull;
  return (bits & keep) | (1ull << (51 - m));
}

// ---------------------------------------------------------------- Student-t constants
// Everything t_cdf needs that does not depend on the request (computed on the host with
// glibc, so bit-identical to the reference's own constants).
struct TdistConst {
  double nu, a, b;  // a = nu/2, b = 1/2
  double logbeta;   // lgamma(a) + lgamma(b) - lgamma(a+b)
  double thresh;    // (a+1)/(a+b+2): CF(a,b,x) below, 1 - CF(b,a,1-x) above
  host::CfTable ab, ba;
};

// ---------------------------------------------------------------- score parameters
// Sigma-grid moment tables (K1):
//   P[g][k][m] = sum_{i<k} Y_i^m / m! * exp(sigma_g * Y_i),   sigma_g = g * kGridH
// so that for |delta| = |sigma - sigma_g| <= kGridH/2
//   sum_{i<k} exp(sigma * Y_i) = sum_m delta^m P[g][k][m]
// truncation (|delta| max|Y|)^12 / 12! < 1.1e-19 relative for max|Y| <= 17.84 (the default
// sample set); requests whose |delta| * max(|Y_0|, |y_max|) exceeds kTaylorReach use the
// exact per-term sum instead (heavy-tailed caller-provided sample sets).
constexpr int kMoments = 12;            // one 96-byte row per (g, k)
constexpr double kGridH = 1.0 / 64.0;   // power of two: g*h and sigma - g*h are exact
constexpr double kGridInvH = 64.0;
constexpr double kTaylorReach = 0.2;    // (0.2)^12 / 12! = 8.6e-18
constexpr int kYBuckets = 8192;         // uniform-y bucket index over the sample range
// Tail-mass table (exact / per-lane score paths): v(y) = 1 - T_nu(y) = I_x(nu/2, 1/2)/2 for
// y >= 0 as a degree-7 Taylor expansion about each of kTailBuckets bucket centres c_b over
// [0, max|Y|]: a_0 = v(c_b) (the reference's own continued-fraction value),
// a_j = -pdf^(j-1)(c_b)/j!, the t-density's derivatives from the exact power series of
// C (1 + (c+t)^2/nu)^-(nu+1)/2.  The series converges within sqrt(c^2+nu) >= 1.87 of c_b; at
// half-width 2.2e-3 the truncation is < 1e-23 relative.  T(y) = y >= 0 ? 1 - v(|y|) : v(|y|)
// (dist.cpp:80).
constexpr int kTailBuckets = 4096;
constexpr int kTailCoef = 8;
// Sample bins (default path): the cut k = upper_bound(Y, y) AND T(y) from ONE 96-byte gather.
// Bins are an exact, monotone integer function of y's IEEE bits -- (exponent, top bin_m
// mantissa bits), |y| < 2^(bin_e0 - 1023) folded into a middle bin -- so every sample in a
// lower bin is < y and every sample in a higher bin is > y.  Entry (12 doubles):
//   [0]      kstart | count << 32  (samples before the bin | in it)
//   [1..5]   the bin's first samples (pads +inf): k = kstart + #{inline <= y}, plus a search
//            of Y for the rare bin holding more than kBinInline samples
//   [6..11]  v(|y|) = 1 - T(|y|) as a degree-5 Taylor expansion about the bin's |y| centre
//            c (relative half-width 2^-(bin_m+1) <= 2.4e-4 of c; the middle bin: c = 0,
//            |t| <= 2^-12), a_0 = the reference's continued fraction, a_j = -pdf^(j-1)(c)/j!.
// Bins extend past the sample range to |y| < 2^(bin_etop - 1022) (k = 0 or N there).
constexpr int kBinEntry = 12;
constexpr int kBinInline = 5;
constexpr int kBinTail = 6;  // coefficient offset
constexpr int kBinCoef = 6;

struct ScoreParams {
  TdistConst td;
  const double* Y;          // sorted samples [N]
  const uint32_t* ybucket;  // [kYBuckets + 1] upper_bound(Y, edge_b)
  const double* table;      // [G][N+1][kMoments]
  const double* tail;       // [kTailBuckets][kTailCoef]
  const double* bins;       // [2 * bin_mid + 1][kBinEntry]
  uint32_t bin_e0, bin_m, bin_mid;
  double bin_ylim;          // bins cover |y| < bin_ylim
  double taylor_y0;         // |Y_0| (moment-table reach: max |Y_i| over a cut, kTaylorReach)
  double inv_N;             // 1 / N  (psi = S / N as S * inv_N)
  double inv_1ma;           // 1 / (1 - alpha)
  double t_ymax, t_w, t_inv_w;
  double y0, y_scale;       // bucket b = floor((y - y0) * y_scale)
  double yN;                // Y[N-1]
  int N;
  int G;                    // grid points in the table (0 => no table)
  uint32_t k_alpha;         // upper_bound(Y, t_quantile(alpha, nu)); 0 when alpha == 0
  const double* ka_table;   // [G][kMoments] the k_alpha row of every grid point
  double alpha, beta;
  int raw;                  // TIE_SCORE_RAW: skip max(C,E) and compute_score
  int ka_smem;              // stage the k_alpha rows of every grid point in shared memory
  uint64_t index_base;      // added to reported request indices (chunked callers)
  unsigned long long* err;
};

}  // namespace dev
}  // namespace tie

// The opaque C handle (include/tie_cuda.h).
struct tie_ctx {
  int device = 0;
  double nu = 0.0;
  int N = 0;
  double sigma_table_max = 0.0;
  std::vector<double> host_samples;
  tie::dev::TdistConst td{};
  // device state
  double* d_Y = nullptr;
  uint32_t* d_ybucket = nullptr;
  double* d_table = nullptr;
  double* d_tail = nullptr;
  double* d_bins = nullptr;
  uint32_t bin_e0 = 0, bin_m = 0, bin_mid = 0;
  double bin_ylim = 0.0;
  double t_ymax = 0, t_w = 0, t_inv_w = 0;
  int G = 0;
  double y0 = 0, y_scale = 0, yN = 0;
  unsigned long long* d_err = nullptr;   // first failure (index << 8 | reason)
  unsigned long long* h_err = nullptr;   // pinned mirror
  const char* err_op = "";               // API call the pending error belongs to
  // scratch arena (grown on demand, reused; never freed inside a call)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  // device I/O arena of the *_host entry points
  void* io = nullptr;
  size_t io_bytes = 0;
  // pinned, UVA-mapped host staging of the *_host entry points for pageable caller buffers
  // (filled / drained by the host copy pool, read / written by the kernels zero-copy)
  void* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  // cached k_alpha = upper_bound(Y, t_quantile(alpha, nu)) of the last alpha seen
  double ka_alpha = -1.0;
  uint32_t ka_k = 0;
  double* d_ka_table = nullptr;          // [G][kMoments] rows at k = ka_table_k
  size_t table_bytes = 0;                 // device bytes of the request-invariant tables
  uint32_t ka_table_k = 0xffffffffu;
  // pinned host staging for the *_host entry points
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  cudaStream_t stream = nullptr;         // internal stream for *_host calls
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev[8] = {};
  // kernel-level profiling (tie_profile): event pairs recorded on the launching stream
  struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
  };
  bool prof_on = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
};

namespace tie {
// RAII: records an event pair around the kernel launches in its scope when profiling is on
struct ProfScope {
  tie_ctx* ctx;
  cudaStream_t s;
  size_t idx = (size_t)-1;
  ProfScope(tie_ctx* c, const char* name, cudaStream_t st);
  ~ProfScope();
};
}  // namespace tie

namespace tie {
namespace capi {
// thread-local error message plumbing (capi.cu)
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* where);
void count_launch(uint64_t k = 1);
void* scratch(tie_ctx* ctx, size_t bytes, cudaStream_t s);
}  // namespace capi

// kernels' host-side launchers (score.cu, rank.cu, fit.cu)
namespace dev {
cudaError_t build_context_tables(tie_ctx* ctx);
cudaError_t launch_score(tie_ctx* ctx, const double* mu, const double* sigma,
                         const void* x_max, bool x_is_u32, uint64_t n, double alpha,
                         double beta, double* E, double* C, double* S, uint64_t* keys_out,
                         unsigned long long* minmax, unsigned flags, cudaStream_t s,
                         uint64_t index_base = 0);
// Dispatch order by (key asc, id asc) of double keys (ids == nullptr: id = index).
cudaError_t launch_rank(tie_ctx* ctx, const double* key, const uint64_t* ids, uint64_t n,
                        uint64_t* order, cudaStream_t s);
size_t rank_scratch_bytes(uint64_t n, bool with_ids);
// true when the sort's last kernel writes the order in coalesced runs (partition path):
// then a host API may hand it mapped pinned host memory as the output
bool rank_output_coalesced(uint64_t n);
// Fused producer path: rank_prepare() zeroes the sort metadata and returns where the
// producer (the score kernel) writes order-preserving u64 keys and folds their range
// (key_range_flush); rank_prepared() then bucket-sorts them and emits the order.
struct RankPrep {
  uint64_t* keys;
  unsigned long long* minmax;
};
RankPrep rank_prepare(tie_ctx* ctx, uint64_t n, cudaStream_t s);
cudaError_t rank_prepared(tie_ctx* ctx, uint64_t n, uint64_t* order, cudaStream_t s);
cudaError_t launch_fit(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                       double* mu, double* sigma, double* ll, int32_t* iters, uint8_t* conv,
                       uint8_t* degen, cudaStream_t s, uint64_t index_base = 0);
// k-way merge of sorted (score, id) runs (merge.cu): keys/ids [G][stride], lens host array
cudaError_t launch_merge_runs(tie_ctx* ctx, const double* keys, const uint64_t* ids, int G,
                              uint64_t stride, const uint64_t* lens, uint64_t* out_ids,
                              cudaStream_t s);
// cmd_fit's per-prompt analysis (report.cu): fits[4][10][P], tail[5][P] (device)
cudaError_t launch_fit_report(tie_ctx* ctx, const double* x, uint64_t P, uint64_t K, double nu,
                              unsigned families, double* fits, double* tail, cudaStream_t s);
cudaError_t launch_loglik(tie_ctx* ctx, const double* x, uint64_t K, const double* mu,
                          const double* sigma, uint64_t P, double nu, double* ll, double* grad,
                          cudaStream_t s);
}  // namespace dev
}  // namespace tie
