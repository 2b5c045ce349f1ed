// GPU-resident waiting queue + scheduler step: the reference's
// Scheduler (proj/src/sched.cpp:125-175) over a WaitingQueue (sched.cpp:28-123), with the
// queue's keys on the device and the exact pop order of the reference heap.
//
// Device state, one slot per request ever queued (append-only):
//   key[s]  order-preserving u64 image of the heap key (~0 once popped)
//   id[s]   req_id (the heap's tie-break, sched.cpp:28-31)
//   E, C, beta_at_update, predicted   (what a drift rebuild needs, sched.cpp:152-167)
// plus a block-min index: bmin[b] = min (key, id) over the 1024 slots of block b.  A pop is
// an argmin over the block minima, an argmin inside the winning block and a refresh of that
// block's minimum -- O(n/1024 + 1024) on one CTA -- instead of the O(n) rekey + heapify a
// full rebuild costs.  New arrivals / predictions refresh only their blocks.
//
// The host side mirrors the reference's bookkeeping exactly (id -> slot map = pos_, the
// multiset betas_in_use_, predicted flags, queue size), so every validation error has the
// reference's type and message, and the pop sequence (including drift rebuilds between
// pops) is the reference's.  B pops are issued as ONE device call whenever no rebuild can
// fire during them: the drift max(|now-min|, |now-max|) can only shrink as pops erase betas,
// so checking beta(Q-b), b < B, against the current (min, max) is sufficient.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tie_cuda.h"
#include "tie_internal.cuh"

namespace tie {
namespace dev {
namespace {

constexpr int kBlockSlots = 1024;
constexpr uint64_t kDead = ~0ull;

struct QDev {
  uint64_t* key;
  uint64_t* id;
  double* E;
  double* C;
  double* beta;
  uint8_t* predicted;
  uint64_t* bkey;  // per block: min key
  uint64_t* bid;   // per block: id of that min
  uint32_t* bslot; // per block: slot of that min
};

__device__ __forceinline__ uint64_t order_bits(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ bool less_kv(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// (key, id, slot) argmin across a CTA (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ void block_argmin(uint64_t& k, uint64_t& i, uint32_t& s,
                                             uint64_t* sk, uint64_t* si, uint32_t* ss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t k2 = __shfl_down_sync(0xffffffffu, k, o);
    const uint64_t i2 = __shfl_down_sync(0xffffffffu, i, o);
    const uint32_t s2 = __shfl_down_sync(0xffffffffu, s, o);
    if (less_kv(k2, i2, k, i)) {
      k = k2;
      i = i2;
      s = s2;
    }
  }
  if (lane == 0) {
    sk[warp] = k;
    si[warp] = i;
    ss[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    k = lane < nw ? sk[lane] : kDead;
    i = lane < nw ? si[lane] : kDead;
    s = lane < nw ? ss[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t k2 = __shfl_down_sync(0xffffffffu, k, o);
      const uint64_t i2 = __shfl_down_sync(0xffffffffu, i, o);
      const uint32_t s2 = __shfl_down_sync(0xffffffffu, s, o);
      if (less_kv(k2, i2, k, i)) {
        k = k2;
        i = i2;
        s = s2;
      }
    }
    if (lane == 0) {
      sk[0] = k;
      si[0] = i;
      ss[0] = s;
    }
  }
  __syncthreads();
  k = sk[0];
  i = si[0];
  s = ss[0];
  __syncthreads();
}

__device__ __forceinline__ void refresh_block(const QDev& q, uint32_t b, uint64_t n_slots,
                                              uint64_t* sk, uint64_t* si, uint32_t* ss) {
  uint64_t k = kDead, i = kDead;
  uint32_t s = 0;
  for (uint32_t t = threadIdx.x; t < kBlockSlots; t += blockDim.x) {
    const uint64_t slot = (uint64_t)b * kBlockSlots + t;
    if (slot < n_slots) {
      const uint64_t kk = q.key[slot], ii = q.id[slot];
      if (less_kv(kk, ii, k, i)) {
        k = kk;
        i = ii;
        s = (uint32_t)slot;
      }
    }
  }
  block_argmin(k, i, s, sk, si, ss);
  if (threadIdx.x == 0) {
    q.bkey[b] = k;
    q.bid[b] = i;
    q.bslot[b] = s;
  }
}

// one CTA per listed block (or per block b < nb when list == nullptr)
__global__ void __launch_bounds__(256) refresh_blocks_kernel(QDev q, const uint32_t* list,
                                                             uint32_t nb, uint64_t n_slots) {
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  for (uint32_t j = blockIdx.x; j < nb; j += gridDim.x)
    refresh_block(q, list ? list[j] : j, n_slots, sk, si, ss);
}

__global__ void write_slots_kernel(QDev q, uint64_t first, uint64_t m, const uint64_t* ids,
                                   const double* keys) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const uint64_t s = first + t;
  q.key[s] = order_bits(keys[t]);
  q.id[s] = ids[t];
  q.predicted[s] = 0;
}

__global__ void write_predictions_kernel(QDev q, const uint32_t* slots, uint64_t m,
                                         const double* E, const double* C, const double* key,
                                         double beta) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const uint32_t s = slots[t];
  q.key[s] = order_bits(key[t]);
  q.E[s] = E[t];
  q.C[s] = C[t];
  q.beta[s] = beta;
  q.predicted[s] = 1;
}

// key = compute_score(E, C, beta) for the batch (sched.cpp:19-26, arguments pre-validated)
__global__ void batch_keys_kernel(const double* E, const double* C, uint64_t m, double beta,
                                  double* key) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) key[t] = __dadd_rn(E[t], __dmul_rn(beta, C[t]));
}

// drift rebuild: re-key every live predicted entry with beta_now (sched.cpp:159-164)
__global__ void rekey_kernel(QDev q, uint64_t n_slots, double beta_now) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_slots; s += stride) {
    if (!q.predicted[s] || q.key[s] == kDead) continue;
    q.key[s] = order_bits(__dadd_rn(q.E[s], __dmul_rn(beta_now, q.C[s])));
    q.beta[s] = beta_now;
  }
}

// up to `pops` pop_min()s with fixed keys (sched.cpp:81-94): argmin over block minima,
// kill the slot, refresh its block.  Writes popped (id, slot) and the count.
__global__ void __launch_bounds__(1024) pop_kernel(QDev q, uint32_t nblocks, uint64_t n_slots,
                                                   uint32_t pops, uint64_t* out_id,
                                                   uint32_t* out_slot, uint32_t* out_n) {
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  uint32_t done = 0;
  for (; done < pops; ++done) {
    uint64_t k = kDead, i = kDead;
    uint32_t s = 0;
    for (uint32_t b = threadIdx.x; b < nblocks; b += blockDim.x) {
      const uint64_t kk = q.bkey[b], ii = q.bid[b];
      if (less_kv(kk, ii, k, i)) {
        k = kk;
        i = ii;
        s = q.bslot[b];
      }
    }
    block_argmin(k, i, s, sk, si, ss);
    if (k == kDead) break;  // queue empty
    if (threadIdx.x == 0) {
      out_id[done] = i;
      out_slot[done] = s;
      q.key[s] = kDead;
    }
    __syncthreads();
    refresh_block(q, s / kBlockSlots, n_slots, sk, si, ss);
  }
  if (threadIdx.x == 0) *out_n = done;
}

}  // namespace
}  // namespace dev
}  // namespace tie

using tie::capi::cuda_error;
using tie::capi::set_error;

struct tie_queue {
  tie_ctx* ctx = nullptr;
  int policy = 2;  // 0 FCFS, 1 SEPT, 2 TIE  (sched.hpp:11)
  int adaptive = 1;
  double beta_fixed = 0.1, beta_max = 0.5, q_sat = 128.0, threshold = 0.1, alpha = 0.9;
  uint64_t capacity = 0, n_slots = 0, size = 0, n_predicted = 0;
  std::unordered_map<uint64_t, uint32_t> slot_of;  // the heap's pos_ index (sched.hpp:67)
  std::vector<uint8_t> alive, predicted;
  // beta_at_update per slot (host mirror): the beta of its prediction, or of the last drift
  // rebuild if that came later (tracked by epoch so a rebuild is O(1) on the host)
  std::vector<double> pred_beta;
  std::vector<uint32_t> pred_epoch;
  uint32_t epoch = 0;
  double rebuild_beta = 0.0;
  std::map<double, uint64_t> betas;                 // betas_in_use_ (sched.hpp:88)
  double beta_of(uint32_t sl) const {
    return pred_epoch[sl] < epoch ? rebuild_beta : pred_beta[sl];
  }
  tie::dev::QDev q{};
  // staging (device) for batches and pops
  uint64_t* d_ids = nullptr;
  double* d_a = nullptr;
  double* d_b = nullptr;
  double* d_c = nullptr;
  uint32_t* d_slots = nullptr;
  uint32_t* d_blocks = nullptr;
  uint64_t* d_out_id = nullptr;
  uint32_t* d_out_slot = nullptr;
  uint32_t* d_out_n = nullptr;
  uint64_t stage_cap = 0;
  uint64_t* h_out_id = nullptr;   // pinned
  uint32_t* h_out_slot = nullptr;
  uint32_t* h_out_n = nullptr;
};

namespace {

double beta_at(const tie_queue* Q, uint64_t queue_len) {
  double b = 0.0;
  tie_compute_beta(Q->adaptive, Q->beta_fixed, Q->beta_max, Q->q_sat, queue_len, &b);
  return b;
}

int ensure_stage(tie_queue* Q, uint64_t m) {
  if (m <= Q->stage_cap) return TIE_OK;
  cudaFree(Q->d_ids); cudaFree(Q->d_a); cudaFree(Q->d_b); cudaFree(Q->d_c);
  cudaFree(Q->d_slots); cudaFree(Q->d_blocks); cudaFree(Q->d_out_id); cudaFree(Q->d_out_slot);
  cudaFreeHost(Q->h_out_id); cudaFreeHost(Q->h_out_slot);
  const uint64_t cap = std::max<uint64_t>(m, 1024);
  cudaError_t e = cudaSuccess;
  if ((e = cudaMalloc(&Q->d_ids, 8 * cap)) || (e = cudaMalloc(&Q->d_a, 8 * cap)) ||
      (e = cudaMalloc(&Q->d_b, 8 * cap)) || (e = cudaMalloc(&Q->d_c, 8 * cap)) ||
      (e = cudaMalloc(&Q->d_slots, 4 * cap)) || (e = cudaMalloc(&Q->d_blocks, 4 * cap)) ||
      (e = cudaMalloc(&Q->d_out_id, 8 * cap)) || (e = cudaMalloc(&Q->d_out_slot, 4 * cap)) ||
      (e = cudaMallocHost(&Q->h_out_id, 8 * cap)) ||
      (e = cudaMallocHost(&Q->h_out_slot, 4 * cap)))
    return cuda_error(e, "tie_queue: staging allocation");
  Q->stage_cap = cap;
  return TIE_OK;
}

// refresh the block minima of the blocks touched by `slots` (host list)
int refresh(tie_queue* Q, const std::vector<uint32_t>& slots, cudaStream_t s) {
  std::vector<uint32_t> blocks;
  blocks.reserve(slots.size());
  for (uint32_t sl : slots) blocks.push_back(sl / tie::dev::kBlockSlots);
  std::sort(blocks.begin(), blocks.end());
  blocks.erase(std::unique(blocks.begin(), blocks.end()), blocks.end());
  if (blocks.empty()) return TIE_OK;
  if (int rc = ensure_stage(Q, blocks.size())) return rc;
  cudaMemcpyAsync(Q->d_blocks, blocks.data(), 4 * blocks.size(), cudaMemcpyHostToDevice, s);
  const unsigned g = (unsigned)std::min<size_t>(blocks.size(), 4096);
  tie::dev::refresh_blocks_kernel<<<g, 256, 0, s>>>(Q->q, Q->d_blocks, (uint32_t)blocks.size(),
                                                     Q->n_slots);
  tie::capi::count_launch();
  return TIE_OK;
}

int rebuild_all(tie_queue* Q, double now, cudaStream_t s) {  // sched.cpp:156-166
  const unsigned g = (unsigned)std::min<uint64_t>((Q->n_slots + 255) / 256, 148 * 8);
  if (g) tie::dev::rekey_kernel<<<g, 256, 0, s>>>(Q->q, Q->n_slots, now);
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  if (nb) tie::dev::refresh_blocks_kernel<<<std::min<uint32_t>(nb, 148 * 16), 256, 0, s>>>(
      Q->q, nullptr, nb, Q->n_slots);
  tie::capi::count_launch(2);
  Q->betas.clear();
  if (Q->n_predicted) Q->betas[now] = Q->n_predicted;
  ++Q->epoch;  // every live predicted slot's beta_at_update is now `now`
  Q->rebuild_beta = now;
  return TIE_OK;
}

double drift(const tie_queue* Q, double now) {
  return std::max(std::fabs(now - Q->betas.begin()->first),
                  std::fabs(now - Q->betas.rbegin()->first));
}

// device pops with fixed keys; appends popped ids to `out`, updates the host mirror
int pop_fixed(tie_queue* Q, uint32_t pops, std::vector<uint64_t>& out, cudaStream_t s) {
  if (int rc = ensure_stage(Q, pops)) return rc;
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  tie::dev::pop_kernel<<<1, 1024, 0, s>>>(Q->q, nb, Q->n_slots, pops, Q->d_out_id,
                                          Q->d_out_slot, Q->d_out_n);
  tie::capi::count_launch();
  cudaMemcpyAsync(Q->h_out_n, Q->d_out_n, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(Q->h_out_slot, Q->d_out_slot, 4 * pops, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(Q->h_out_id, Q->d_out_id, 8 * pops, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_error(e, "tie_queue_next");
  for (uint32_t j = 0; j < *Q->h_out_n; ++j) {
    const uint32_t sl = Q->h_out_slot[j];
    out.push_back(Q->h_out_id[j]);
    Q->alive[sl] = 0;
    Q->slot_of.erase(Q->h_out_id[j]);
    --Q->size;
    if (Q->predicted[sl]) {  // betas_in_use_.erase(find(beta_at_update)) (sched.cpp:173)
      auto it = Q->betas.find(Q->beta_of(sl));
      if (it != Q->betas.end() && --it->second == 0) Q->betas.erase(it);
      --Q->n_predicted;
    }
  }
  return TIE_OK;
}

}  // namespace

extern "C" {

int tie_queue_create(tie_ctx* ctx, int policy, int adaptive, double beta_fixed, double beta_max,
                     double q_sat, double rebuild_threshold, double alpha, uint64_t capacity,
                     tie_queue** out) {
  if (!ctx || !out) return set_error(TIE_EINVALID, "tie_queue_create: null argument");
  if (policy < 0 || policy > 2) return set_error(TIE_EINVALID, "tie_queue_create: bad policy");
  if (!(alpha >= 0.0 && alpha < 1.0))
    return set_error(TIE_EDOMAIN, "censored_cvar: alpha must lie in [0, 1)");
  if (capacity == 0 || capacity >= (1ull << 32))
    return set_error(TIE_EINVALID, "tie_queue_create: capacity must be in [1, 2^32)");
  cudaSetDevice(ctx->device);
  auto* Q = new tie_queue();
  Q->ctx = ctx;
  Q->policy = policy;
  Q->adaptive = adaptive;
  Q->beta_fixed = beta_fixed;
  Q->beta_max = beta_max;
  Q->q_sat = q_sat;
  Q->threshold = rebuild_threshold;
  Q->alpha = alpha;
  Q->capacity = capacity;
  Q->alive.assign(capacity, 0);
  Q->predicted.assign(capacity, 0);
  Q->pred_beta.assign(capacity, 0.0);
  Q->pred_epoch.assign(capacity, 0);
  Q->slot_of.reserve(std::min<uint64_t>(capacity, 1u << 24));
  const uint64_t nb = (capacity + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots;
  cudaError_t e;
  if ((e = cudaMalloc(&Q->q.key, 8 * capacity)) || (e = cudaMalloc(&Q->q.id, 8 * capacity)) ||
      (e = cudaMalloc(&Q->q.E, 8 * capacity)) || (e = cudaMalloc(&Q->q.C, 8 * capacity)) ||
      (e = cudaMalloc(&Q->q.beta, 8 * capacity)) ||
      (e = cudaMalloc(&Q->q.predicted, capacity)) || (e = cudaMalloc(&Q->q.bkey, 8 * nb)) ||
      (e = cudaMalloc(&Q->q.bid, 8 * nb)) || (e = cudaMalloc(&Q->q.bslot, 4 * nb)) ||
      (e = cudaMalloc(&Q->d_out_n, 4)) || (e = cudaMallocHost(&Q->h_out_n, 4))) {
    tie_queue_destroy(Q);
    return cuda_error(e, "tie_queue_create");
  }
  cudaMemset(Q->q.key, 0xff, 8 * capacity);
  cudaMemset(Q->q.bkey, 0xff, 8 * nb);
  cudaMemset(Q->q.bid, 0xff, 8 * nb);
  *out = Q;
  return TIE_OK;
}

void tie_queue_destroy(tie_queue* Q) {
  if (!Q) return;
  cudaDeviceSynchronize();
  for (void* p : {(void*)Q->q.key, (void*)Q->q.id, (void*)Q->q.E, (void*)Q->q.C,
                  (void*)Q->q.beta, (void*)Q->q.predicted, (void*)Q->q.bkey, (void*)Q->q.bid,
                  (void*)Q->q.bslot, (void*)Q->d_ids, (void*)Q->d_a, (void*)Q->d_b,
                  (void*)Q->d_c, (void*)Q->d_slots, (void*)Q->d_blocks, (void*)Q->d_out_id,
                  (void*)Q->d_out_slot, (void*)Q->d_out_n})
    cudaFree(p);
  cudaFreeHost(Q->h_out_id);
  cudaFreeHost(Q->h_out_slot);
  cudaFreeHost(Q->h_out_n);
  delete Q;
}

uint64_t tie_queue_size(const tie_queue* Q) { return Q ? Q->size : 0; }

double tie_queue_current_beta(const tie_queue* Q) { return Q ? beta_at(Q, Q->size) : 0.0; }

// Scheduler::on_arrival x m (sched.cpp:125-132): key = FCFS ? arrival_s : max_tokens.
int tie_queue_arrive(tie_queue* Q, const uint64_t* ids, const double* arrival_s,
                     const uint32_t* max_tokens, uint64_t m) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (m == 0) return TIE_OK;
  if (Q->n_slots + m > Q->capacity)
    return set_error(TIE_EINVALID, "tie_queue_arrive: capacity exceeded");
  std::vector<double> keys(m);
  for (uint64_t t = 0; t < m; ++t) {
    keys[t] = Q->policy == 0 ? arrival_s[t] : (double)max_tokens[t];
    if (!std::isfinite(keys[t]))
      return set_error(TIE_EDOMAIN, "WaitingQueue::push: key must be finite");
    if (Q->slot_of.count(ids[t]))
      return set_error(TIE_EINVALID, "WaitingQueue::push: id " + std::to_string(ids[t]) +
                                         " already queued");
    Q->slot_of.emplace(ids[t], (uint32_t)(Q->n_slots + t));  // rejects in-batch duplicates next
  }
  if (Q->slot_of.size() != Q->size + m) {  // duplicate inside the batch
    for (uint64_t t = 0; t < m; ++t) Q->slot_of.erase(ids[t]);
    return set_error(TIE_EINVALID, "WaitingQueue::push: id already queued");
  }
  cudaStream_t s = Q->ctx->stream;
  if (int rc = ensure_stage(Q, m)) return rc;
  cudaMemcpyAsync(Q->d_ids, ids, 8 * m, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(Q->d_a, keys.data(), 8 * m, cudaMemcpyHostToDevice, s);
  tie::dev::write_slots_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(Q->q, Q->n_slots, m,
                                                                         Q->d_ids, Q->d_a);
  tie::capi::count_launch();
  std::vector<uint32_t> touched;
  for (uint64_t t = 0; t < m; t += tie::dev::kBlockSlots) touched.push_back((uint32_t)(Q->n_slots + t));
  touched.push_back((uint32_t)(Q->n_slots + m - 1));
  for (uint64_t t = 0; t < m; ++t) Q->alive[Q->n_slots + t] = 1;
  Q->n_slots += m;
  Q->size += m;
  if (int rc = refresh(Q, touched, s)) return rc;
  const cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_queue_arrive");
}

// Scheduler::on_prediction x m (sched.cpp:134-150) with given (E, CVaR).
int tie_queue_predict(tie_queue* Q, const uint64_t* ids, const double* E, const double* C,
                      uint64_t m) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (m == 0) return TIE_OK;
  std::vector<uint32_t> slots(m);
  for (uint64_t t = 0; t < m; ++t) {
    auto it = Q->slot_of.find(ids[t]);
    if (it == Q->slot_of.end())
      return set_error(TIE_EINVALID, "Scheduler::on_prediction: id " + std::to_string(ids[t]) +
                                         " not waiting");
    slots[t] = it->second;
  }
  if (Q->policy == 0) return TIE_OK;  // FCFS: arrival order is the schedule
  const double beta = Q->policy == 1 ? 0.0 : beta_at(Q, Q->size);
  for (uint64_t t = 0; t < m; ++t) {
    if (Q->predicted[slots[t]])
      return set_error(TIE_EINVALID, "Scheduler::on_prediction: id " + std::to_string(ids[t]) +
                                         " already predicted");
    const double e = E[t], c = C[t];  // compute_score checks (sched.cpp:19-26)
    if (!std::isfinite(e) || !std::isfinite(c) || !std::isfinite(beta))
      return set_error(TIE_EDOMAIN, "compute_score: arguments must be finite");
    if (!(e > 0.0)) return set_error(TIE_EDOMAIN, "compute_score: expectation must be > 0");
    if (c < e)
      return set_error(TIE_EINVALID,
                       "compute_score: cvar below expectation violates the invariant");
  }
  for (uint64_t t = 0; t + 1 < m; ++t)  // duplicate ids inside one batch
    for (uint64_t u = t + 1; u < m && u < t + 64; ++u)
      if (slots[u] == slots[t])
        return set_error(TIE_EINVALID, "Scheduler::on_prediction: id " + std::to_string(ids[t]) +
                                           " already predicted");
  cudaStream_t s = Q->ctx->stream;
  if (int rc = ensure_stage(Q, m)) return rc;
  cudaMemcpyAsync(Q->d_slots, slots.data(), 4 * m, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(Q->d_a, E, 8 * m, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(Q->d_b, C, 8 * m, cudaMemcpyHostToDevice, s);
  const unsigned g = (unsigned)((m + 255) / 256);
  tie::dev::batch_keys_kernel<<<g, 256, 0, s>>>(Q->d_a, Q->d_b, m, beta, Q->d_c);
  tie::dev::write_predictions_kernel<<<g, 256, 0, s>>>(Q->q, Q->d_slots, m, Q->d_a, Q->d_b,
                                                       Q->d_c, beta);
  tie::capi::count_launch(2);
  for (uint32_t sl : slots) {
    Q->predicted[sl] = 1;
    Q->pred_beta[sl] = beta;
    Q->pred_epoch[sl] = Q->epoch;
  }
  Q->betas[beta] += m;
  Q->n_predicted += m;
  if (int rc = refresh(Q, slots, s)) return rc;
  const cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_queue_predict");
}

// run_sim's chain for the batch (sim.cpp:85-95) on the GPU, then on_prediction.
int tie_queue_predict_logt(tie_queue* Q, const uint64_t* ids, const double* mu,
                           const double* sigma, const uint32_t* max_tokens, uint64_t m) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (m == 0) return TIE_OK;
  std::vector<double> E(m), C(m), xm(m);
  for (uint64_t t = 0; t < m; ++t) xm[t] = (double)max_tokens[t];
  if (int rc = tie_score_host(Q->ctx, mu, sigma, xm.data(), m, Q->alpha, 0.0, E.data(),
                              C.data(), nullptr, TIE_SCORE_RAW))
    return rc;
  for (uint64_t t = 0; t < m; ++t) C[t] = std::max(C[t], E[t]);  // sim.cpp:94
  return tie_queue_predict(Q, ids, E.data(), C.data(), m);
}

// Scheduler::next_request() up to max_pops times (sched.cpp:169-175), including
// rebuild_if_drifted before each pop (sched.cpp:152-167).
int tie_queue_next(tie_queue* Q, uint64_t max_pops, uint64_t* out_ids, uint64_t* n_out) {
  if (!Q || !n_out) return set_error(TIE_EINVALID, "tie_queue: null argument");
  *n_out = 0;
  std::vector<uint64_t> got;
  cudaStream_t s = Q->ctx->stream;
  uint64_t left = std::min<uint64_t>(max_pops, Q->size);
  while (left > 0) {
    const bool tie_policy = Q->policy == 2;
    // can a rebuild fire during the next `left` pops?  (drift only shrinks as pops erase)
    uint64_t safe = left;
    if (tie_policy && !Q->betas.empty()) {
      safe = 0;
      while (safe < left && !(drift(Q, beta_at(Q, Q->size - safe)) > Q->threshold)) ++safe;
    }
    if (safe == 0) {  // rebuild now (exact check with the current multiset), then one pop
      const double now = beta_at(Q, Q->size);
      if (drift(Q, now) > Q->threshold)
        if (int rc = rebuild_all(Q, now, s)) return rc;
      safe = 1;
    }
    const size_t before = got.size();
    if (int rc = pop_fixed(Q, (uint32_t)safe, got, s)) return rc;
    const uint64_t popped = got.size() - before;
    if (popped == 0) break;
    left -= popped;
  }
  for (size_t j = 0; j < got.size(); ++j) out_ids[j] = got[j];
  *n_out = got.size();
  return TIE_OK;
}

int tie_queue_rebuild_if_drifted(tie_queue* Q, int* rebuilt) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (rebuilt) *rebuilt = 0;
  if (Q->policy != 2 || Q->betas.empty()) return TIE_OK;
  const double now = beta_at(Q, Q->size);
  if (!(drift(Q, now) > Q->threshold)) return TIE_OK;
  if (int rc = rebuild_all(Q, now, Q->ctx->stream)) return rc;
  if (rebuilt) *rebuilt = 1;
  const cudaError_t e = cudaStreamSynchronize(Q->ctx->stream);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_queue_rebuild_if_drifted");
}

}  // extern "C"
