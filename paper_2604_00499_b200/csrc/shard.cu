// Device halves of the request-sharded score + rank (host side in
// paper_2604_00499_b200/dist.py), so a step issues no eager passes over the shard and no host
// round trip except the one the NCCL all-to-all's host split sizes require:
//
//  * tie_score_rank_run: K1 + K2 on the shard, emitting the SORTED RUN directly -- keys[p] =
//    the score of the p-th request in (score, id) order, ids[p] = its shard-local index (u32)
//    -- the 12-byte records the exchange moves (reference order: sched.cpp:28-31);
//  * tie_shard_cuts: the splitter exchange's cut points.  The G regular samples (each a sorted
//    sample of one rank's run, gathered by NCCL, sentinel-padded) are ranked by merge-path
//    counting ((key, id) is a strict total order: ids are unique), the G-1 splitters are the
//    elements at ranks j*t/G (t = valid samples), and every splitter's lexicographic lower
//    bound in this rank's run gives the send counts -- one single-CTA launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/tie_cuda.h"
#include "tie_internal.cuh"

namespace tie {
namespace dev {
namespace {

__global__ void run_gather_kernel(const uint64_t* __restrict__ keys,
                                  const uint64_t* __restrict__ order, uint64_t n,
                                  double* __restrict__ run_keys, uint32_t* __restrict__ run_ids) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    const uint64_t i = order[p];
    // the fused path's keys: positive finite scores, bits | 2^63 (score.cu)
    run_keys[p] = __longlong_as_double((long long)(keys[i] & 0x7fffffffffffffffull));
    run_ids[p] = (uint32_t)i;
  }
}

__device__ __forceinline__ bool lex_less(double ka, int64_t ia, double kb, int64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

constexpr int kCutThreads = 1024;
constexpr int kMaxSample = 8192;  // G * s

// sample: G runs of s (key, global id) pairs, each sorted, invalid entries id < 0 (their keys
// are sentinels, +max, so they sort last; for ordering an invalid id counts as +inf)
__global__ void __launch_bounds__(kCutThreads) shard_cuts_kernel(
    const double* __restrict__ run_keys, const uint32_t* __restrict__ run_ids, uint64_t id_base,
    uint64_t n, const double* __restrict__ sk, const int64_t* __restrict__ si, int G, int s,
    int64_t* __restrict__ send_counts, double* __restrict__ split_keys,
    int64_t* __restrict__ split_ids) {
  __shared__ double spk[64];
  __shared__ int64_t spi[64];
  __shared__ int valid;
  const int tot = G * s;
  if (threadIdx.x == 0) valid = 0;
  __syncthreads();
  int cnt = 0;
  for (int e = threadIdx.x; e < tot; e += kCutThreads) cnt += si[e] >= 0;
  atomicAdd(&valid, cnt);
  __syncthreads();
  const int t = valid;
  // merged rank of every valid sample element: sum over runs h of #{(k, i) < (k_e, i_e)}
  for (int e = threadIdx.x; e < tot; e += kCutThreads) {
    const int64_t ie = si[e];
    if (ie < 0) continue;
    const double ke = sk[e];
    int rank = 0;
    for (int h = 0; h < G; ++h) {
      int lo = 0, hi = s;  // first position in run h not less than (ke, ie)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int64_t im = si[h * s + mid];
        const bool lt = im >= 0 && lex_less(sk[h * s + mid], im, ke, ie);
        if (lt) lo = mid + 1; else hi = mid;
      }
      rank += lo;
    }
    for (int j = 1; j < G; ++j)
      if (rank == (int)(((int64_t)j * t) / G) && rank < t) {
        spk[j - 1] = ke;
        spi[j - 1] = ie;
      }
  }
  __syncthreads();
  // this run's cut at every splitter: #{(k, id_base + i) < splitter}
  if (threadIdx.x < G - 1) {
    const int j = threadIdx.x;
    const int c = (int)(((int64_t)(j + 1) * t) / G);
    uint64_t cut = n;  // no splitter (too few samples): everything goes below it
    if (c < t) {
      const double kk = spk[j];
      const int64_t ii = spi[j];
      uint64_t lo = 0, hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (lex_less(run_keys[mid], (int64_t)(id_base + run_ids[mid]), kk, ii)) lo = mid + 1;
        else hi = mid;
      }
      cut = lo;
      if (split_keys) split_keys[j] = kk;
      if (split_ids) split_ids[j] = ii;
    }
    spk[32 + j] = __longlong_as_double((long long)cut);  // stash the cut (as raw bits)
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int j = threadIdx.x;
    const uint64_t a = j == 0 ? 0 : (uint64_t)__double_as_longlong(spk[32 + j - 1]);
    const uint64_t b = j == G - 1 ? n : (uint64_t)__double_as_longlong(spk[32 + j]);
    send_counts[j] = (int64_t)(b > a ? b - a : 0);
  }
}

// The range exchange over peer memory: the sorted run's piece g (run positions
// [start[g], start[g+1])) goes to rank g's receive buffer at dst[g] + (p - start[g]) -- keys and
// ids in ONE launch of SM-driven stores into the CUDA-IPC-mapped buffers (NVLink / NVSwitch
// between GPUs), in place of the two NCCL all-to-alls.  Consecutive records of a piece go to
// consecutive addresses of one peer (coalesced peer stores).
constexpr int kMaxPeers = 64;
struct PeerTab {
  uint64_t start[kMaxPeers + 1];
  uint64_t dst[kMaxPeers];
  double* k[kMaxPeers];
  uint32_t* i[kMaxPeers];
  int G;
};

__global__ void __launch_bounds__(256) peer_put_kernel(const double* __restrict__ rk,
                                                       const uint32_t* __restrict__ ri,
                                                       uint64_t n, const __grid_constant__ PeerTab t) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
    int lo = 0, hi = t.G;  // piece g with start[g] <= p < start[g + 1] (non-empty)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (t.start[mid] <= p) lo = mid; else hi = mid;
    }
    const uint64_t q = t.dst[lo] + (p - t.start[lo]);
    t.k[lo][q] = rk[p];
    t.i[lo][q] = ri[p];
  }
}

}  // namespace
}  // namespace dev
}  // namespace tie

using tie::capi::cuda_error;
using tie::capi::set_error;

extern "C" int tie_score_rank_run(tie_ctx* ctx, const double* mu, const double* sigma,
                                  const uint32_t* max_tokens, uint64_t n, double alpha,
                                  double beta, double* score, uint64_t* order, double* run_keys,
                                  uint32_t* run_ids, unsigned flags, void* stream) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_score_rank_run: null context");
  if (n && (!order || !run_keys || !run_ids))
    return set_error(TIE_EINVALID, "tie_score_rank_run: null output");
  if (n == 0) return TIE_OK;
  if (n >= (1ull << 32)) return set_error(TIE_EINVALID, "tie_score_rank_run: shard >= 2^32");
  if (!(alpha >= 0.0 && alpha < 1.0))
    return set_error(TIE_EDOMAIN, "censored_cvar: alpha must lie in [0, 1)");
  if (!mu || !sigma || !max_tokens) return set_error(TIE_EINVALID, "tie_score_rank_run: null input");
  cudaSetDevice(ctx->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const tie::dev::RankPrep prep = tie::dev::rank_prepare(ctx, n, s);
  if (!prep.keys) return set_error(TIE_ECUDA, "tie_score_rank_run: scratch allocation failed");
  ctx->err_op = "tie_score_rank_run";
  cudaError_t e = tie::dev::launch_score(ctx, mu, sigma, max_tokens, true, n, alpha, beta,
                                         nullptr, nullptr, score, prep.keys, prep.minmax, flags,
                                         s);
  if (e == cudaSuccess) e = tie::dev::rank_prepared(ctx, n, order, s);
  if (e != cudaSuccess) return cuda_error(e, "tie_score_rank_run");
  const unsigned g = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  tie::dev::run_gather_kernel<<<g, 256, 0, s>>>(prep.keys, order, n, run_keys, run_ids);
  tie::capi::count_launch();
  e = cudaGetLastError();
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_score_rank_run");
}

extern "C" int tie_shard_cuts(tie_ctx* ctx, const double* run_keys, const uint32_t* run_ids,
                              uint64_t id_base, uint64_t n, const double* sample_keys,
                              const int64_t* sample_ids, int G, int s, int64_t* send_counts,
                              double* split_keys, int64_t* split_ids, void* stream) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_shard_cuts: null context");
  if (G < 1 || G > 32 || s < 1 || (int64_t)G * s > tie::dev::kMaxSample)
    return set_error(TIE_EINVALID, "tie_shard_cuts: need 1 <= G <= 32 and G * s <= 8192");
  cudaSetDevice(ctx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  tie::dev::shard_cuts_kernel<<<1, tie::dev::kCutThreads, 0, st>>>(
      run_keys, run_ids, id_base, n, sample_keys, sample_ids, G, s, send_counts, split_keys,
      split_ids);
  tie::capi::count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_shard_cuts");
}

// ---- CUDA IPC + peer put (SURVEY.md 8e range exchange over peer memory) -----------------
extern "C" int tie_ipc_alloc(tie_ctx* ctx, uint64_t bytes, void** ptr, void* handle) {
  if (!ctx || !ptr || !handle) return set_error(TIE_EINVALID, "tie_ipc_alloc: null argument");
  cudaSetDevice(ctx->device);
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 1);
  if (e == cudaSuccess)
    e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), *ptr);
  if (e != cudaSuccess) {
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    return cuda_error(e, "tie_ipc_alloc");
  }
  return TIE_OK;
}

extern "C" int tie_ipc_free(tie_ctx* ctx, void* ptr) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_ipc_free: null context");
  cudaSetDevice(ctx->device);
  const cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_ipc_free");
}

extern "C" int tie_ipc_open(tie_ctx* ctx, const void* handle, void** ptr) {
  if (!ctx || !handle || !ptr) return set_error(TIE_EINVALID, "tie_ipc_open: null argument");
  cudaSetDevice(ctx->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_ipc_open");
}

extern "C" int tie_ipc_close(tie_ctx* ctx, void* ptr) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_ipc_close: null context");
  cudaSetDevice(ctx->device);
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_ipc_close");
}

extern "C" int tie_peer_put_runs(tie_ctx* ctx, const double* run_keys, const uint32_t* run_ids,
                                 uint64_t n, int G, const uint64_t* send_counts,
                                 const uint64_t* dst_offsets, void* const* peer_keys,
                                 void* const* peer_ids, void* stream) {
  if (!ctx) return set_error(TIE_EINVALID, "tie_peer_put_runs: null context");
  if (G < 1 || G > tie::dev::kMaxPeers)
    return set_error(TIE_EINVALID, "tie_peer_put_runs: need 1 <= G <= 64");
  if (!send_counts || !dst_offsets || !peer_keys || !peer_ids)
    return set_error(TIE_EINVALID, "tie_peer_put_runs: null argument");
  tie::dev::PeerTab t{};
  t.G = G;
  uint64_t acc = 0;
  for (int g = 0; g < G; ++g) {
    t.start[g] = acc;
    acc += send_counts[g];
    t.dst[g] = dst_offsets[g];
    t.k[g] = static_cast<double*>(peer_keys[g]);
    t.i[g] = static_cast<uint32_t*>(peer_ids[g]);
    if (send_counts[g] && (!t.k[g] || !t.i[g]))
      return set_error(TIE_EINVALID, "tie_peer_put_runs: null peer buffer");
  }
  t.start[G] = acc;
  if (acc != n) return set_error(TIE_EINVALID, "tie_peer_put_runs: send counts != run length");
  if (n == 0) return TIE_OK;
  // empty pieces must never be chosen by the search: start[g] == start[g+1] is skipped
  // because the search picks the LAST g with start[g] <= p
  cudaSetDevice(ctx->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  tie::dev::peer_put_kernel<<<grid, 256, 0, st>>>(run_keys, run_ids, n, t);
  tie::capi::count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_peer_put_runs");
}
