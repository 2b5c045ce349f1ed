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
#include <cassert>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/tie_cuda.h"
#include "tie_internal.cuh"
#include "flat_idmap.hpp"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

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

// (key, id, slot) argmin across a warp, in every lane: the lexicographic minimum of the 128-bit
// (key, id) as four 32-bit redux.sync minima over the lanes still tied, then the slot of the
// lowest tied lane (what the shuffle tree below picked: ties keep the lower lane) -- 4 REDUX
// + a ballot + a shuffle instead of 25 shuffles and 5 dependent 128-bit compares
__device__ __forceinline__ void warp_argmin_redux(uint64_t& k, uint64_t& i, uint32_t& s) {
  const uint32_t kh = (uint32_t)(k >> 32), kl = (uint32_t)k;
  const uint32_t ih = (uint32_t)(i >> 32), il = (uint32_t)i;
  const uint32_t m1 = __reduce_min_sync(0xffffffffu, kh);
  bool t = kh == m1;
  const uint32_t m2 = __reduce_min_sync(0xffffffffu, t ? kl : 0xffffffffu);
  t = t && kl == m2;
  const uint32_t m3 = __reduce_min_sync(0xffffffffu, t ? ih : 0xffffffffu);
  t = t && ih == m3;
  const uint32_t m4 = __reduce_min_sync(0xffffffffu, t ? il : 0xffffffffu);
  t = t && il == m4;
  const int w = __ffs(__ballot_sync(0xffffffffu, t)) - 1;
  k = ((uint64_t)m1 << 32) | m2;
  i = ((uint64_t)m3 << 32) | m4;
  s = __shfl_sync(0xffffffffu, s, w);
}

// (key, id, slot) argmin across a CTA (blockDim multiple of 32, <= 1024)
__device__ __forceinline__ void block_argmin(uint64_t& k, uint64_t& i, uint32_t& s,
                                             uint64_t* sk, uint64_t* si, uint32_t* ss) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmin_redux(k, i, s);
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
    warp_argmin_redux(k, i, s);
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

// block_argmin for a loop of rounds with ONE CTA barrier per round: every warp reduces the 32
// warp minima itself (redux.sync is cheap), reading a double buffer indexed by the round's
// parity -- a warp can run one round ahead of the slowest, never two (the barrier)
__device__ __forceinline__ void block_argmin_round(uint64_t& k, uint64_t& i, uint32_t& s,
                                                   uint64_t* dk, uint64_t* di, uint32_t* ds,
                                                   uint32_t round) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  warp_argmin_redux(k, i, s);
  const uint32_t o = (round & 1u) * 32u;
  if (lane == 0) {
    dk[o + warp] = k;
    di[o + warp] = i;
    ds[o + warp] = s;
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  k = lane < nw ? dk[o + lane] : kDead;
  i = lane < nw ? di[o + lane] : kDead;
  s = lane < nw ? ds[o + lane] : 0;
  warp_argmin_redux(k, i, s);
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

// (key, id, slot) minimum of block `blk` by one warp: 32 slots per lane, loaded 8 at a time
// so a block costs 4 memory round trips instead of 32 dependent ones
__device__ __forceinline__ void warp_block_min(const QDev& q, uint32_t blk, uint64_t n_slots,
                                               int lane, uint64_t& k, uint64_t& i,
                                               uint32_t& s) {
  k = kDead;
  i = kDead;
  s = 0;
  constexpr int kU = 8;
#pragma unroll
  for (uint32_t base = 0; base < (uint32_t)kBlockSlots; base += 32 * kU) {
    uint64_t kk[kU], ii[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t slot = (uint64_t)blk * kBlockSlots + base + u * 32 + lane;
      kk[u] = slot < n_slots ? q.key[slot] : kDead;
      ii[u] = slot < n_slots ? q.id[slot] : kDead;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (less_kv(kk[u], ii[u], k, i)) {
        k = kk[u];
        i = ii[u];
        s = (uint32_t)((uint64_t)blk * kBlockSlots + base + u * 32 + lane);
      }
  }
  warp_argmin_redux(k, i, s);
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
  q.predicted[s] = 1;
}

// fused step: run_sim's fixup C = max(C, E) (sim.cpp:94) and the compute_score checks
// (sched.cpp:19-26) on the device; failures go to the context's error word (first index wins)
// and make the dependent kernels of the step skip.  key = E + beta C.
__global__ void predict_keys_kernel(const double* E, double* C, uint64_t m, double beta,
                                    double* key, unsigned long long* err) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const double e = E[t];
  double c = C[t];
  c = c < e ? e : c;
  C[t] = c;
  uint32_t why = kOk;
  if (!isfinite(e) || !isfinite(c) || !isfinite(beta)) why = kScoreNotFinite;
  else if (!(e > 0.0)) why = kExpectationNonPos;
  else if (c < e) why = kCvarBelowE;
  if (why != kOk) report(err, t, why);
  key[t] = __dadd_rn(e, __dmul_rn(beta, c));
}

__global__ void write_predictions_checked_kernel(QDev q, const uint32_t* slots, uint64_t m,
                                                 const double* E, const double* C,
                                                 const double* key, double beta,
                                                 const unsigned long long* err) {
  if (*(const volatile unsigned long long*)err != ~0ull) return;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const uint32_t s = slots[t];
  q.key[s] = order_bits(key[t]);
  q.E[s] = E[t];
  q.C[s] = C[t];
  q.predicted[s] = 1;
}

__global__ void __launch_bounds__(256) refresh_blocks_checked_kernel(
    QDev q, const uint32_t* list, uint32_t nb, uint64_t n_slots, const unsigned long long* err,
    uint32_t n_unconditional) {
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  const bool skip = *(const volatile unsigned long long*)err != ~0ull;
  for (uint32_t j = blockIdx.x; j < nb; j += gridDim.x)
    if (j < n_unconditional || !skip) refresh_block(q, list[j], n_slots, sk, si, ss);
}

// key = compute_score(E, C, beta) for the batch (sched.cpp:19-26, arguments pre-validated)
__global__ void batch_keys_kernel(const double* E, const double* C, uint64_t m, double beta,
                                  double* key) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m) key[t] = __dadd_rn(E[t], __dmul_rn(beta, C[t]));
}

// drift rebuild fused with the block-minimum refresh: one CTA per 1024-slot block re-keys its
// live predicted entries with beta_now (sched.cpp:159-164) and recomputes the block minimum
__global__ void __launch_bounds__(256) rekey_refresh_kernel(QDev q, uint32_t nb,
                                                            uint64_t n_slots, double beta_now,
                                                            const unsigned long long* err) {
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  if (err && *(const volatile unsigned long long*)err != ~0ull) return;  // failed fused step
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    uint64_t k = kDead, i = kDead;
    uint32_t s = 0;
    for (uint32_t t = threadIdx.x; t < kBlockSlots; t += blockDim.x) {
      const uint64_t slot = (uint64_t)b * kBlockSlots + t;
      if (slot >= n_slots) break;
      uint64_t kk = q.key[slot];
      if (kk != kDead && q.predicted[slot]) {
        kk = order_bits(__dadd_rn(q.E[slot], __dmul_rn(beta_now, q.C[slot])));
        q.key[slot] = kk;
      }
      const uint64_t ii = q.id[slot];
      if (less_kv(kk, ii, k, i)) {
        k = kk;
        i = ii;
        s = (uint32_t)slot;
      }
    }
    block_argmin(k, i, s, sk, si, ss);
    if (threadIdx.x == 0) {
      q.bkey[b] = k;
      q.bid[b] = i;
      q.bslot[b] = s;
    }
  }
}


// A run of drift-rebuild + single-pop segments (the threshold-0 regime: beta moves with
// every pop, so the reference re-keys the whole queue before each next_request(),
// sched.cpp:152-175) in ONE cooperative launch instead of two kernels per pop.  Segment g:
// every CTA re-keys its blocks at betas[g] and recomputes their minima (skipping -- killing --
// the slot popped by segment g-1, which every CTA knows), posts its CTA minimum, grid sync;
// every CTA then reduces the <= gridDim.x CTA minima itself (double-buffered by segment
// parity, so no second grid sync), CTA 0 records the pop.  The last popped slot's owner
// kills it and refreshes its block at the end.  A failed fused step (err set) skips all.
struct SegBetas {
  double b[32];
  int eager;  // A/B: store keys and block minima in every segment
};
constexpr int kRekeyThreads = 256;

__device__ void rekey_seq_body(const QDev& q, uint32_t nb, uint64_t n_slots,
                               const SegBetas& betas, uint32_t nseg, uint64_t* out_id,
                               uint32_t* out_slot, uint32_t* out_n, uint64_t* cmin,
                               uint64_t* sk, uint64_t* si, uint32_t* ss,
                               cg::grid_group& grid) {
  const uint32_t G = gridDim.x;
  uint64_t killed = ~0ull;
  for (uint32_t g = 0; g < nseg; ++g) {
    const double beta = betas.b[g];
    // keys and block minima are stored by the last segment only (earlier passes keep them in
    // registers; a popped slot's death is stored at once)
    const bool last = g + 1 == nseg || betas.eager;
    uint64_t ck = kDead, ci = kDead;
    uint32_t cs = 0;
    for (uint32_t b = blockIdx.x; b < nb; b += G) {
      uint64_t k = kDead, i = kDead;
      uint32_t s = 0;
      constexpr int kU = kBlockSlots / kRekeyThreads;
      uint64_t kk[kU], ii[kU];
      double ee[kU], cc[kU];
      uint8_t pr[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // all loads in flight first (E, C too: no second trip)
        const uint64_t slot = (uint64_t)b * kBlockSlots + threadIdx.x + u * kRekeyThreads;
        const bool in = slot < n_slots;
        kk[u] = in ? q.key[slot] : kDead;
        ii[u] = in ? q.id[slot] : kDead;
        pr[u] = in ? q.predicted[slot] : 0;
        ee[u] = in ? q.E[slot] : 0.0;
        cc[u] = in ? q.C[slot] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t slot = (uint64_t)b * kBlockSlots + threadIdx.x + u * kRekeyThreads;
        if (slot == killed) {
          kk[u] = kDead;
          q.key[slot] = kDead;
        } else if (kk[u] != kDead && pr[u]) {
          kk[u] = order_bits(__dadd_rn(ee[u], __dmul_rn(beta, cc[u])));
          if (last) q.key[slot] = kk[u];
        }
        if (less_kv(kk[u], ii[u], k, i)) {
          k = kk[u];
          i = ii[u];
          s = (uint32_t)slot;
        }
      }
      block_argmin(k, i, s, sk, si, ss);
      if (last && threadIdx.x == 0) {
        q.bkey[b] = k;
        q.bid[b] = i;
        q.bslot[b] = s;
      }
      if (less_kv(k, i, ck, ci)) {
        ck = k;
        ci = i;
        cs = s;
      }
    }
    uint64_t* buf = cmin + (size_t)(g & 1) * 3 * G;
    if (threadIdx.x == 0) {
      buf[blockIdx.x] = ck;
      buf[G + blockIdx.x] = ci;
      buf[2 * G + blockIdx.x] = cs;
    }
    grid.sync();
    uint64_t k = kDead, i = kDead;
    uint32_t s = 0;
    for (uint32_t c = threadIdx.x; c < G; c += kRekeyThreads) {
      const uint64_t k2 = __ldcg(buf + c), i2 = __ldcg(buf + G + c);
      if (less_kv(k2, i2, k, i)) {
        k = k2;
        i = i2;
        s = (uint32_t)__ldcg(buf + 2 * G + c);
      }
    }
    block_argmin(k, i, s, sk, si, ss);
    if (k == kDead) {  // the queue ran dry (same decision in every CTA): every block is empty
      if (blockIdx.x == 0 && threadIdx.x == 0) out_n[g] = 0;
      if (threadIdx.x == 0)
        for (uint32_t b = blockIdx.x; b < nb; b += G) {
          q.bkey[b] = kDead;
          q.bid[b] = kDead;
        }
      killed = ~0ull;
      break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out_id[g] = i;
      out_slot[g] = s;
      out_n[g] = 1;
    }
    killed = s;
  }
  if (killed != ~0ull && (uint32_t)(killed / kBlockSlots) % G == blockIdx.x) {
    if (threadIdx.x == 0) q.key[killed] = kDead;
    __syncthreads();
    refresh_block(q, (uint32_t)(killed / kBlockSlots), n_slots, sk, si, ss);
  }
}

__global__ void __launch_bounds__(kRekeyThreads) rekey_pop_seq_kernel(
    QDev q, uint32_t nb, uint64_t n_slots, SegBetas betas, uint32_t nseg, uint64_t* out_id,
    uint32_t* out_slot, uint32_t* out_n, uint64_t* cmin, const unsigned long long* err) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  __shared__ int skip;
  if (threadIdx.x == 0) skip = err && *(const volatile unsigned long long*)err != ~0ull;
  __syncthreads();
  if (skip) return;  // the same decision in every CTA: err is final before this launch
  rekey_seq_body(q, nb, n_slots, betas, nseg, out_id, out_slot, out_n, cmin, sk, si, ss, grid);
}

// The same run of (drift rebuild, pop) segments with ONE pass over the queue instead of one
// per segment.  Keys are monotone in beta (fl(E + fl(beta C)) with C >= 0; unpredicted keys
// are constants), so every key of the run lies in [k_lo, k_hi] = its keys at the smallest /
// largest beta of the run.  Let T = the nseg-th smallest (k_hi, id) over the block minima: at
// any segment at least one not-yet-popped entry has (key, id) <= T, so every entry the run
// pops has (k_lo, id) <= T -- the candidates, a handful.  The pass keys every entry at the
// run's LAST beta (the reference's final state, sched.cpp:159-164), stores keys and block
// minima, and records each block's minimum (k_lo, id) and (k_hi, id); CTA 0 selects T; the
// candidates are gathered; CTA 0 replays the segments over them exactly (re-key at beta_g,
// (key, id) argmin, kill); the popped blocks are refreshed.  A candidate list above
// kSeqCandCap falls back to the per-segment passes (rekey_seq_body) in the same launch.
constexpr uint32_t kSeqCandCap = 1024;
struct CandScratch {
  uint64_t* blo;   // [nb][2] block minimum (k_lo, id)
  uint64_t* bhi;   // [nb][2] block minimum (k_hi, id)
  uint32_t* cand;  // [kSeqCandCap] candidate slots
  uint32_t* hdr;   // [0] count, [1] overflow
  uint64_t* thr;   // [2] T = (key, id)
  uint64_t* clist; // [kCminCtas][32][2] each CTA's smallest block minima (k_hi, id)
};

__device__ __forceinline__ void warp_min3(uint64_t& k, uint64_t& i, uint32_t& s) {
  warp_argmin_redux(k, i, s);
}

// the r-th smallest (key, id) pair of pairs[0..n) (r < rmax), by one CTA: every thread keeps
// the two smallest of its strided share, then r + 1 rounds of a CTA argmin over the heads
// (a thread that wins a third time rescans, excluding the pairs already taken)
__device__ void cta_rth_smallest(const uint64_t* __restrict__ pairs, uint32_t n, uint32_t r,
                                 uint64_t& ok, uint64_t& oi, uint64_t* sk, uint64_t* si,
                                 uint32_t* ss, uint32_t* taken) {
  uint64_t k0, i0, k1, i1;
  uint32_t b0, b1;
  bool more;
  auto scan = [&](uint32_t ntaken) {
    k0 = i0 = k1 = i1 = kDead;
    b0 = b1 = 0xffffffffu;
    uint32_t live = 0;
    constexpr int kU = 4;  // loads in flight per thread
    for (uint32_t x0 = threadIdx.x; x0 < n; x0 += kU * blockDim.x) {
      uint64_t kk[kU], ii[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t x = x0 + u * blockDim.x;
        kk[u] = x < n ? __ldcg(pairs + 2 * x) : kDead;
        ii[u] = x < n ? __ldcg(pairs + 2 * x + 1) : kDead;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (kk[u] == kDead) continue;
        const uint32_t x = x0 + u * blockDim.x;
        bool ex = false;
        for (uint32_t e = 0; e < ntaken; ++e) ex |= taken[e] == x;
        if (ex) continue;
        ++live;
        if (!less_kv(kk[u], ii[u], k1, i1)) continue;
        if (less_kv(kk[u], ii[u], k0, i0)) {
          k1 = k0;
          i1 = i0;
          b1 = b0;
          k0 = kk[u];
          i0 = ii[u];
          b0 = x;
        } else {
          k1 = kk[u];
          i1 = ii[u];
          b1 = x;
        }
      }
    }
    more = live > 2;
  };
  scan(0);
  ok = oi = kDead;
  for (uint32_t t = 0; t <= r; ++t) {
    uint64_t k = k0, i = i0;
    uint32_t b = b0;
    block_argmin(k, i, b, sk, si, ss);
    if (k == kDead) {  // fewer than r + 1 pairs: no bound
      ok = oi = kDead;
      return;
    }
    ok = k;
    oi = i;
    if (threadIdx.x == 0) taken[t] = b;
    __syncthreads();
    if (k0 != kDead && b0 == b) {
      k0 = k1;
      i0 = i1;
      b0 = b1;
      k1 = i1 = kDead;
      b1 = 0xffffffffu;
      if (k0 == kDead && more) scan(t + 1);
    }
  }
}

__global__ void __launch_bounds__(kRekeyThreads) rekey_pop_cand_kernel(
    QDev q, uint32_t nb, uint64_t n_slots, SegBetas betas, uint32_t nseg, uint64_t* out_id,
    uint32_t* out_slot, uint32_t* out_n, uint64_t* cmin, CandScratch cs,
    const unsigned long long* err) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  __shared__ uint32_t taken[32];
  __shared__ int skip;
  __shared__ double cE[kSeqCandCap], cC[kSeqCandCap];
  __shared__ uint64_t cK[kSeqCandCap], cI[kSeqCandCap];
  if (threadIdx.x == 0) skip = err && *(const volatile unsigned long long*)err != ~0ull;
  __syncthreads();
  if (skip) return;  // the same decision in every CTA: err is final before this launch
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // the gather's header, visible after sync 1
    cs.hdr[0] = 0;
    cs.hdr[1] = 0;
  }
  double b_lo = betas.b[0], b_hi = betas.b[0];
  for (uint32_t g = 1; g < nseg; ++g) {
    b_lo = fmin(b_lo, betas.b[g]);
    b_hi = fmax(b_hi, betas.b[g]);
  }
  const double b_last = betas.b[nseg - 1];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t W = (gridDim.x * blockDim.x) >> 5;
  // every warp's nseg smallest block minima (k_hi, id), sorted (lane 0 inserts)
  __shared__ uint64_t wl[kRekeyThreads / 32][32][2];
  __shared__ uint32_t wn[kRekeyThreads / 32];
  if (lane == 0) wn[wib] = 0;
  // ---- A: one pass, a warp per block: keys at b_last stored; minima at b_last, b_lo, b_hi
  for (uint32_t b = warp; b < nb; b += W) {
    uint64_t mk = kDead, mi = kDead, lk = kDead, li = kDead, hk = kDead, hi = kDead;
    uint32_t ms = 0, dummy = 0;
    constexpr int kU = 8;
#pragma unroll
    for (int base = 0; base < kBlockSlots; base += 32 * kU) {
      uint64_t kk[kU], ii[kU];
      double ee[kU], cc[kU];
      uint8_t pr[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // all loads in flight first
        const uint64_t slot = (uint64_t)b * kBlockSlots + base + u * 32 + lane;
        const bool in = slot < n_slots;
        kk[u] = in ? q.key[slot] : kDead;
        ii[u] = in ? q.id[slot] : kDead;
        pr[u] = in ? q.predicted[slot] : 0;
        ee[u] = in ? q.E[slot] : 0.0;
        cc[u] = in ? q.C[slot] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (kk[u] == kDead) continue;
        const uint64_t slot = (uint64_t)b * kBlockSlots + base + u * 32 + lane;
        uint64_t kx = kk[u], kl = kk[u], kh = kk[u];
        if (pr[u]) {
          kx = order_bits(__dadd_rn(ee[u], __dmul_rn(b_last, cc[u])));
          kl = order_bits(__dadd_rn(ee[u], __dmul_rn(b_lo, cc[u])));
          kh = order_bits(__dadd_rn(ee[u], __dmul_rn(b_hi, cc[u])));
          q.key[slot] = kx;
        }
        if (less_kv(kx, ii[u], mk, mi)) {
          mk = kx;
          mi = ii[u];
          ms = (uint32_t)slot;
        }
        if (less_kv(kl, ii[u], lk, li)) {
          lk = kl;
          li = ii[u];
        }
        if (less_kv(kh, ii[u], hk, hi)) {
          hk = kh;
          hi = ii[u];
        }
      }
    }
    warp_min3(mk, mi, ms);
    warp_min3(lk, li, dummy);
    warp_min3(hk, hi, dummy);
    if (lane == 0) {
      q.bkey[b] = mk;
      q.bid[b] = mi;
      q.bslot[b] = ms;
      cs.blo[2 * b] = lk;
      cs.blo[2 * b + 1] = li;
      if (hk != kDead) {  // insert into the warp's sorted list of nseg
        uint32_t c = wn[wib];
        if (c < nseg || less_kv(hk, hi, wl[wib][c - 1][0], wl[wib][c - 1][1])) {
          uint32_t at = c < nseg ? c : nseg - 1;
          while (at > 0 && less_kv(hk, hi, wl[wib][at - 1][0], wl[wib][at - 1][1])) {
            wl[wib][at][0] = wl[wib][at - 1][0];
            wl[wib][at][1] = wl[wib][at - 1][1];
            --at;
          }
          wl[wib][at][0] = hk;
          wl[wib][at][1] = hi;
          if (c < nseg) wn[wib] = c + 1;
        }
      }
    }
  }
  __syncthreads();
  {  // the CTA's nseg smallest of its warps' lists (rank by counting), into its clist row
    const uint32_t w = threadIdx.x >> 5, pos = threadIdx.x & 31;
    const bool have = pos < wn[w];
    const uint64_t k = have ? wl[w][pos][0] : kDead, i = have ? wl[w][pos][1] : kDead;
    uint32_t rank = 0;
    if (have)
      for (uint32_t w2 = 0; w2 < kRekeyThreads / 32; ++w2)
        for (uint32_t p2 = 0; p2 < wn[w2]; ++p2)
          rank += less_kv(wl[w2][p2][0], wl[w2][p2][1], k, i) ? 1u : 0u;
    uint64_t* row = cs.clist + (size_t)blockIdx.x * 64;
    if (threadIdx.x < 32) {  // clear the row first (kDead pairs), then place the ranked
      row[2 * threadIdx.x] = kDead;
      row[2 * threadIdx.x + 1] = kDead;
    }
    __syncthreads();
    if (have && rank < nseg) {
      row[2 * rank] = k;
      row[2 * rank + 1] = i;
    }
  }
  grid.sync();
  // ---- T: the nseg-th smallest block minimum (k_hi, id) over the CTAs' sorted lists, by
  // EVERY CTA (no serial phase, no extra grid sync): each thread owns the lists t, t + 256,
  // ...; nseg rounds of a CTA argmin over the owned lists' heads, the winner's head advances
  uint64_t tk = kDead, ti = kDead;
  {
    constexpr int kMaxOwned = 4096 / kRekeyThreads;  // kCminCtas lists at most
    uint8_t head[kMaxOwned];
#pragma unroll
    for (int j = 0; j < kMaxOwned; ++j) head[j] = 0;
    for (uint32_t r = 0; r < nseg; ++r) {
      uint64_t k = kDead, i = kDead;
      uint32_t s = 0xffffffffu;
#pragma unroll
      for (int j = 0; j < kMaxOwned; ++j) {
        const uint32_t L = threadIdx.x + j * kRekeyThreads;
        if (L >= gridDim.x || head[j] >= 32) continue;
        const uint64_t* e = cs.clist + (size_t)L * 64 + 2 * head[j];
        const uint64_t kk = __ldcg(e), ii = __ldcg(e + 1);
        if (less_kv(kk, ii, k, i)) {
          k = kk;
          i = ii;
          s = (uint32_t)j;
        }
      }
      const uint32_t mine = s == 0xffffffffu ? 0xffffffffu : threadIdx.x * kMaxOwned + s;
      uint32_t win = mine;
      block_argmin(k, i, win, sk, si, ss);
      if (k == kDead) {  // fewer than nseg block minima: no bound
        tk = ti = kDead;
        break;
      }
      tk = k;
      ti = i;
      if (win == mine && mine != 0xffffffffu) {
#pragma unroll
        for (int j = 0; j < kMaxOwned; ++j) head[j] += (uint32_t)j == s ? 1 : 0;
      }
    }
  }
  // ---- B: candidates (k_lo, id) <= T, from the blocks whose minimum (k_lo, id) is <= T
  for (uint32_t b = warp; b < nb; b += W) {
    if (less_kv(tk, ti, __ldcg(cs.blo + 2 * b), __ldcg(cs.blo + 2 * b + 1))) continue;
    constexpr int kU = 8;
#pragma unroll
    for (int base = 0; base < kBlockSlots; base += 32 * kU) {
      uint64_t kk[kU], ii[kU];
      double ee[kU], cc[kU];
      uint8_t pr[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // all loads in flight first
        const uint64_t slot = (uint64_t)b * kBlockSlots + base + u * 32 + lane;
        const bool in = slot < n_slots;
        kk[u] = in ? q.key[slot] : kDead;  // stored at b_last by this warp in A
        ii[u] = in ? q.id[slot] : kDead;
        pr[u] = in ? q.predicted[slot] : 0;
        ee[u] = in ? q.E[slot] : 0.0;
        cc[u] = in ? q.C[slot] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t slot = (uint64_t)b * kBlockSlots + base + u * 32 + lane;
        bool take = false;
        if (kk[u] != kDead) {
          const uint64_t kl =
              pr[u] ? order_bits(__dadd_rn(ee[u], __dmul_rn(b_lo, cc[u]))) : kk[u];
          take = !less_kv(tk, ti, kl, ii[u]);
        }
        const unsigned m = __ballot_sync(0xffffffffu, take);
        if (!m) continue;
        uint32_t at = 0;
        if (lane == 0) at = atomicAdd(cs.hdr, (uint32_t)__popc(m));
        at = __shfl_sync(0xffffffffu, at, 0) + __popc(m & ((1u << lane) - 1u));
        if (take) {
          if (at < kSeqCandCap) cs.cand[at] = (uint32_t)slot;
          else cs.hdr[1] = 1;
        }
      }
    }
  }
  grid.sync();
  const uint32_t nc = __ldcg(cs.hdr), over = __ldcg(cs.hdr + 1);
  if (over || nc > kSeqCandCap) {  // identical decision in every CTA
    rekey_seq_body(q, nb, n_slots, betas, nseg, out_id, out_slot, out_n, cmin, sk, si, ss, grid);
    return;
  }
  // ---- C: CTA 0 replays the segments over the candidates (keys re-made at every beta_g)
  if (blockIdx.x == 0) {
    for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x) {
      const uint32_t slot = cs.cand[c];
      cE[c] = q.E[slot];
      cC[c] = q.C[slot];
      cK[c] = q.key[slot];
      cI[c] = q.id[slot];
      if (!q.predicted[slot]) cC[c] = -1.0;  // unpredicted: key constant
    }
    __syncthreads();
    uint32_t g = 0;
    for (; g < nseg; ++g) {
      const double beta = betas.b[g];
      uint64_t k = kDead, i = kDead;
      uint32_t s = 0xffffffffu;
      for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x) {
        if (cK[c] == kDead) continue;  // popped earlier in the run
        const uint64_t kc = cC[c] >= 0.0 ? order_bits(__dadd_rn(cE[c], __dmul_rn(beta, cC[c])))
                                         : cK[c];
        if (less_kv(kc, cI[c], k, i)) {
          k = kc;
          i = cI[c];
          s = c;
        }
      }
      block_argmin(k, i, s, sk, si, ss);
      if (k == kDead) break;  // the queue ran dry
      if (threadIdx.x == 0) {
        const uint32_t slot = cs.cand[s];
        out_id[g] = i;
        out_slot[g] = slot;
        out_n[g] = 1;
        q.key[slot] = kDead;
        cK[s] = kDead;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0)
      for (uint32_t r = g; r < nseg; ++r) out_n[r] = 0;
  }
  grid.sync();
  // ---- D: refresh the popped blocks (a warp per pop; a block popped twice is refreshed
  // twice, identically -- every kill happened before the grid sync)
  for (uint32_t j = warp; j < nseg; j += W) {
    if (__ldcg(out_n + j) == 0) continue;
    const uint32_t blk = __ldcg(out_slot + j) / kBlockSlots;
    uint64_t k, i;
    uint32_t s;
    warp_block_min(q, blk, n_slots, lane, k, i, s);
    if (lane == 0) {
      q.bkey[blk] = k;
      q.bid[blk] = i;
      q.bslot[blk] = s;
    }
  }
}

// Up to `pops` pop_min()s with fixed keys in ONE pass (no drift rebuild can fire between
// them): with fixed keys the pop sequence is the `pops` smallest (key, id) entries in order.
// Let v_1 < ... < v_B be the B smallest block minima; the B smallest entries are all <= v_B
// and lie in those B blocks, so the candidates are the entries <= v_B of those blocks, ranked
// by counting.  Then the popped slots die and their blocks' minima are refreshed (one warp
// per block).  *skip != 0 (an invalid prediction in the same fused step): pop nothing.
constexpr int kTopB = 32;            // pops per launch
constexpr int kCandCap = 2048;       // candidates held in shared memory
// The `pops` smallest live entries of <= 8 chosen blocks, for a 1024-thread CTA: each thread
// holds its <= 8 slots (slot threadIdx.x of chosen block u) sorted in registers, and `pops`
// CTA argmin rounds over the threads' heads pop them in order; then the blocks are refreshed.
// Used when the queue has fewer live blocks than pops (all their entries compete, which
// would overflow the general path's candidate list).
template <int kF>  // entries per thread: >= the chosen blocks (4 or 8)
__device__ __forceinline__ void pop_from_blocks_regs(const QDev& q, const uint32_t* chosen,
                                                  uint32_t nchosen, uint64_t n_slots,
                                                  uint32_t pops, uint64_t* out_id,
                                                  uint32_t* out_slot, uint32_t* out_n,
                                                  uint64_t* out_key, uint64_t* dk,
                                                  uint64_t* di, uint32_t* ds) {
  uint64_t fk[kF], fi[kF];
  uint32_t fs[kF];
#pragma unroll
  for (int u = 0; u < kF; ++u) {
    const uint64_t slot =
        u < (int)nchosen ? (uint64_t)chosen[u] * kBlockSlots + threadIdx.x : n_slots;
    fk[u] = slot < n_slots ? q.key[slot] : kDead;
    fi[u] = slot < n_slots ? q.id[slot] : kDead;
    fs[u] = (uint32_t)slot;
  }
#pragma unroll
  for (int a = 1; a < kF; ++a)  // insertion sort, unrolled (compile-time indices)
#pragma unroll
    for (int b = a; b > 0; --b)
      if (less_kv(fk[b], fi[b], fk[b - 1], fi[b - 1])) {
        const uint64_t tk = fk[b], ti = fi[b];
        const uint32_t ts = fs[b];
        fk[b] = fk[b - 1];
        fi[b] = fi[b - 1];
        fs[b] = fs[b - 1];
        fk[b - 1] = tk;
        fi[b - 1] = ti;
        fs[b - 1] = ts;
      }
  uint32_t done = 0;
  for (; done < pops; ++done) {
    uint64_t k = fk[0], i = fi[0];
    uint32_t s = fs[0];
    block_argmin_round(k, i, s, dk, di, ds, done);
    if (k == kDead) break;
    if (threadIdx.x == 0) {
      out_id[done] = i;
      out_slot[done] = s;
      if (out_key) out_key[done] = k;
      q.key[s] = kDead;
    }
    if (fk[0] != kDead && fs[0] == s) {  // the winner advances to its next entry
#pragma unroll
      for (int u = 0; u + 1 < kF; ++u) {
        fk[u] = fk[u + 1];
        fi[u] = fi[u + 1];
        fs[u] = fs[u + 1];
      }
      fk[kF - 1] = kDead;
      fi[kF - 1] = kDead;
    }
  }
  if (threadIdx.x == 0) *out_n = done;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t e = warp; e < nchosen; e += blockDim.x >> 5) {
    const uint32_t blk = chosen[e];
    uint64_t k, i;
    uint32_t s;
    warp_block_min(q, blk, n_slots, lane, k, i, s);
    if (lane == 0) {
      q.bkey[blk] = k;
      q.bid[blk] = i;
      q.bslot[blk] = s;
    }
  }
}

// kSmallPath: include the register path for queues with fewer live blocks than pops (kept
// out of the fused apply kernel, whose instruction footprint it would grow: the host sends
// small queues' pops to pop_topb_kernel instead)
template <bool kSmallPath>
__device__ __forceinline__ void pop_topb(const QDev& q, uint32_t nblocks, uint64_t n_slots,
                                         uint32_t pops, uint64_t* out_id, uint32_t* out_slot,
                                         uint32_t* out_n, uint64_t* out_key = nullptr) {
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  __shared__ uint64_t dk[64], di[64];  // block_argmin_round's double buffer
  __shared__ uint32_t ds[64];
  __shared__ uint32_t chosen[kTopB];
  __shared__ uint64_t ck[kCandCap], ci[kCandCap];
  __shared__ uint32_t cs[kCandCap];
  __shared__ uint32_t ncand, overflow;
  if (threadIdx.x == 0) {
    ncand = 0;
    overflow = 0;
  }
  // 1. the B smallest block minima: every thread keeps the two smallest minima of its
  //    strided share in registers (one pass, 4 loads in flight per thread: at 64M slots a
  //    thread owns 64 blocks), then B rounds of a CTA argmin over the threads' heads; the
  //    winner shifts its pair, and only a thread that wins a third time rescans (excluding
  //    the chosen blocks).  A one-best-per-thread rescan after every win made each round
  //    a dependent walk over the winner's share (the 64M step's ~170 us over 10M's).
  uint64_t k0, i0, k1, i1;
  uint32_t b0, b1;
  bool more;  // the thread's share held more than two live blocks when last scanned
  auto scan_top2 = [&](int nex, uint32_t also) {  // excluding chosen[0..nex) and `also`
    k0 = i0 = k1 = i1 = kDead;
    b0 = b1 = 0xffffffffu;
    uint32_t live = 0;
    constexpr int kU = 4;
    for (uint32_t x0 = threadIdx.x; x0 < nblocks; x0 += kU * blockDim.x) {
      uint64_t kk[kU], ii[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // all loads in flight before the first use
        const uint32_t x = x0 + u * blockDim.x;
        kk[u] = x < nblocks ? q.bkey[x] : kDead;
        ii[u] = x < nblocks ? q.bid[x] : kDead;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (kk[u] == kDead) continue;
        const uint32_t x = x0 + u * blockDim.x;
        bool ex = x == also;
        for (int e = 0; e < nex; ++e) ex |= chosen[e] == x;
        if (ex) continue;
        ++live;
        if (!less_kv(kk[u], ii[u], k1, i1)) continue;
        if (less_kv(kk[u], ii[u], k0, i0)) {
          k1 = k0;
          i1 = i0;
          b1 = b0;
          k0 = kk[u];
          i0 = ii[u];
          b0 = x;
        } else {
          k1 = kk[u];
          i1 = ii[u];
          b1 = x;
        }
      }
    }
    more = live > 2;
  };
  scan_top2(0, 0xffffffffu);
  uint32_t nchosen = 0;
  uint64_t vB_k = kDead, vB_i = kDead;
  for (uint32_t r = 0; r < pops; ++r) {
    uint64_t k = k0, i = i0;
    uint32_t b = b0;
    block_argmin_round(k, i, b, dk, di, ds, r);
    if (k == kDead) break;  // fewer live blocks than pops
    if (threadIdx.x == 0) chosen[r] = b;  // visible after the next round's barrier
    nchosen = r + 1;
    vB_k = k;
    vB_i = i;
    if (k0 != kDead && b0 == b) {  // this thread won: its head advances
      k0 = k1;
      i0 = i1;
      b0 = b1;
      k1 = i1 = kDead;
      b1 = 0xffffffffu;
      // chosen[r] may not be visible yet: excluded as `also`
      if (k0 == kDead && more) scan_top2((int)r, b);
    }
  }
  __syncthreads();  // chosen[] complete for the steps below
  if (nchosen == 0) {
    if (threadIdx.x == 0) *out_n = 0;
    return;
  }
  if (kSmallPath && nchosen < pops && nchosen <= 8 && blockDim.x == 1024) {
    // every live block is chosen (a small queue): select among all their entries directly
    if (nchosen <= 4)  // a 4-entry sort network instead of the 8-entry one
      pop_from_blocks_regs<4>(q, chosen, nchosen, n_slots, pops, out_id, out_slot, out_n,
                              out_key, dk, di, ds);
    else
      pop_from_blocks_regs<8>(q, chosen, nchosen, n_slots, pops, out_id, out_slot, out_n,
                              out_key, dk, di, ds);
    return;
  }
  if (nchosen < pops) {  // every live block is chosen: all their live entries are candidates
    vB_k = kDead;
    vB_i = kDead;
  }
  // 2. candidates: entries <= v_B of the chosen blocks
  for (uint32_t t0 = threadIdx.x; t0 < nchosen * kBlockSlots; t0 += 8 * blockDim.x) {
    uint64_t kk[8], ii[8], sl[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // all loads in flight before the first use
      const uint32_t t = t0 + u * blockDim.x;
      sl[u] = t < nchosen * kBlockSlots
                  ? (uint64_t)chosen[t / kBlockSlots] * kBlockSlots + t % kBlockSlots
                  : n_slots;
      kk[u] = sl[u] < n_slots ? q.key[sl[u]] : kDead;
      ii[u] = sl[u] < n_slots ? q.id[sl[u]] : kDead;
    }
    // warp-aggregated appends (one shared atomic per warp and item; the loop is warp-uniform:
    // nchosen * kBlockSlots is a multiple of 32)
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool take = kk[u] != kDead && !less_kv(vB_k, vB_i, kk[u], ii[u]);  // <= v_B
      const unsigned m = __ballot_sync(0xffffffffu, take);
      if (!m) continue;
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&ncand, (uint32_t)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (take) {
        const uint32_t c = base + __popc(m & ((1u << lane) - 1u));
        if (c < kCandCap) {
          ck[c] = kk[u];
          ci[c] = ii[u];
          cs[c] = (uint32_t)sl[u];
        } else {
          overflow = 1;
        }
      }
    }
  }
  __syncthreads();
  const uint32_t nc = min(ncand, (uint32_t)kCandCap);
  if (overflow) {  // pathological key layout: fall back to one argmin + refresh per pop
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
      if (k == kDead) break;
      if (threadIdx.x == 0) {
        out_id[done] = i;
        out_slot[done] = s;
        if (out_key) out_key[done] = k;
        q.key[s] = kDead;
      }
      __syncthreads();
      refresh_block(q, s / kBlockSlots, n_slots, sk, si, ss);
    }
    if (threadIdx.x == 0) *out_n = done;
    return;
  }
  // 3. rank the candidates; the first min(pops, nc) in (key, id) order are the pops
  const uint32_t npop = min(pops, nc);
  for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x) {
    // only ranks < npop matter: stop counting once a candidate is known to rank lower (all
    // candidates of a single live block compete when the queue holds < pops blocks)
    uint32_t rank = 0;
    const uint64_t kc = ck[c], ic = ci[c];
    for (uint32_t d = 0; d < nc && rank < npop; ++d)
      rank += less_kv(ck[d], ci[d], kc, ic) ? 1u : 0u;
    if (rank < npop) {
      out_id[rank] = ci[c];
      out_slot[rank] = cs[c];
      if (out_key) out_key[rank] = ck[c];
      q.key[cs[c]] = kDead;
    }
  }
  if (threadIdx.x == 0) *out_n = npop;
  __syncthreads();
  // 4. refresh every chosen block (popped blocks are among them): one warp per block
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t e = warp; e < nchosen; e += blockDim.x >> 5) {
    const uint32_t blk = chosen[e];
    uint64_t k, i;
    uint32_t s;
    warp_block_min(q, blk, n_slots, lane, k, i, s);
    if (lane == 0) {
      q.bkey[blk] = k;
      q.bid[blk] = i;
      q.bslot[blk] = s;
    }
  }
}

// the fused step's completion record: the step's sequence number, with kStatusErrBit set when
// the error word holds an error (the host then decodes it with tie_sync), after a system fence
// -- one fence, the host polls this word instead of synchronising the stream
constexpr uint32_t kStatusErrBit = 0x80000000u;
__global__ void step_finish_kernel(const unsigned long long* err, volatile uint32_t* status_seq,
                                   uint32_t seq) {
  const bool failed = *(const volatile unsigned long long*)err != ~0ull;
  __threadfence_system();
  *status_seq = seq | (failed ? kStatusErrBit : 0u);
}

__global__ void __launch_bounds__(1024) pop_topb_kernel(QDev q, uint32_t nblocks,
                                                        uint64_t n_slots, uint32_t pops,
                                                        uint64_t* out_id, uint32_t* out_slot,
                                                        uint32_t* out_n,
                                                        uint64_t* out_key = nullptr,
                                                        const unsigned long long* err = nullptr) {
  __shared__ int skip;
  if (threadIdx.x == 0) skip = err && *(const volatile unsigned long long*)err != ~0ull;
  __syncthreads();
  if (skip) return;  // a failed fused step pops nothing
  pop_topb<true>(q, nblocks, n_slots, pops, out_id, out_slot, out_n, out_key);
}

// undo a peek's pops (one CTA): restore the popped slots' keys, then refresh their blocks
// (one warp per popped slot; a block popped twice is refreshed twice, identically)
__global__ void __launch_bounds__(1024) unpop_kernel(QDev q, const uint32_t* slots,
                                                     const uint64_t* keys, uint32_t n,
                                                     uint64_t n_slots) {
  for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) q.key[slots[t]] = keys[t];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t t = warp; t < n; t += blockDim.x >> 5) {
    const uint32_t blk = slots[t] / kBlockSlots;
    uint64_t k, i;
    uint32_t s;
    warp_block_min(q, blk, n_slots, lane, k, i, s);
    if (lane == 0) {
      q.bkey[blk] = k;
      q.bid[blk] = i;
      q.bslot[blk] = s;
    }
  }
}

// A small scheduler iteration in ONE kernel (one CTA): write the arrivals' slots; check the
// predictions (run_sim's max(C, E), compute_score, plus the score kernel's own validation
// in the error word) and -- only if all pass -- key and write them; refresh the touched
// blocks; then the fixed-key pops.  Any error: no prediction written, nothing popped.
// kSmall: the instantiation for queues with fewer live blocks than pops can reach (the
// register pop path included; the large-queue instantiation keeps the smaller footprint)
template <bool kSmall>
__global__ void __launch_bounds__(1024) step_apply_kernel(
    QDev q, uint64_t first, uint64_t n_arr, const uint64_t* arr_ids, const double* arr_keys,
    const uint32_t* slots, uint64_t np, const double* E, double* C, double beta,
    const uint32_t* blocks, uint32_t nblk, uint32_t n_uncond, uint32_t nblocks, uint64_t n_slots,
    uint32_t pops, uint64_t* out_id, uint32_t* out_slot, uint32_t* out_n,
    unsigned long long* err, volatile uint32_t* status_seq,
    uint32_t seq, const double* betas,  // betas: per-prediction beta (a multi-run step) or null
    const char* pack = nullptr, uint32_t pack_bytes = 0) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  // a small step's pack in pinned host memory (zero-copy): staged into shared memory in one
  // parallel burst -- one PCIe round trip instead of one per dependent phase below (arrivals,
  // predictions, slots, blocks); the pointers into it are redirected to the copy
  if (pack_bytes) {
    extern __shared__ uint4 stage[];
    const uint4* src = reinterpret_cast<const uint4*>(pack);
    for (uint32_t x = threadIdx.x; x < pack_bytes / 16; x += blockDim.x) stage[x] = src[x];
    const char* sb = reinterpret_cast<const char*>(stage);
    auto in_pack = [&](const void* ptr) {
      const char* c = static_cast<const char*>(ptr);
      return c >= pack && c < pack + pack_bytes;
    };
    auto tr = [&](auto* ptr) {
      using T = decltype(ptr);
      return in_pack(ptr) ? (T)(sb + (static_cast<const char*>((const void*)ptr) - pack)) : ptr;
    };
    arr_ids = tr(arr_ids);
    arr_keys = tr(arr_keys);
    slots = tr(slots);
    blocks = tr(blocks);
    if (betas) betas = tr(betas);
    E = tr(E);
    C = tr(C);
  }
  __syncthreads();
  for (uint64_t t = threadIdx.x; t < n_arr; t += blockDim.x) {
    const uint64_t s = first + t;
    q.key[s] = order_bits(arr_keys[t]);
    q.id[s] = arr_ids[t];
    q.predicted[s] = 0;
  }
  // launched as a programmatic dependent of the score kernel (tie_queue_step): the arrivals
  // above overlap its tail; its E / C (and error word) are read only after this wait (a no-op
  // without a dependency)
  cudaGridDependencySynchronize();
  for (uint64_t t = threadIdx.x; t < np; t += blockDim.x) {
    const double e = E[t];
    double c = C[t];
    c = c < e ? e : c;  // sim.cpp:94
    C[t] = c;
    uint32_t why = kOk;
    if (!isfinite(e) || !isfinite(c) || !isfinite(betas ? betas[t] : beta)) why = kScoreNotFinite;
    else if (!(e > 0.0)) why = kExpectationNonPos;
    else if (c < e) why = kCvarBelowE;
    if (why != kOk) {
      report(err, t, why);
      bad = 1;
    }
  }
  __syncthreads();
  const bool skip = bad || *(const volatile unsigned long long*)err != ~0ull;
  if (!skip)
    for (uint64_t t = threadIdx.x; t < np; t += blockDim.x) {
      const uint32_t s = slots[t];
      q.key[s] = order_bits(__dadd_rn(E[t], __dmul_rn(betas ? betas[t] : beta, C[t])));
      q.E[s] = E[t];
      q.C[s] = C[t];
          q.predicted[s] = 1;
    }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t e = warp; e < (skip ? n_uncond : nblk); e += blockDim.x >> 5) {
    const uint32_t blk = blocks[e];
    uint64_t k, i;
    uint32_t s;
    warp_block_min(q, blk, n_slots, lane, k, i, s);
    if (lane == 0) {
      q.bkey[blk] = k;
      q.bid[blk] = i;
      q.bslot[blk] = s;
    }
  }
  __syncthreads();
  if (skip || pops == 0) {
    if (threadIdx.x == 0) *out_n = 0;
  } else {
    pop_topb<kSmall>(q, nblocks, n_slots, pops, out_id, out_slot, out_n);
  }
  if (status_seq) {  // the step's last kernel: publish the completion record (step_finish)
    __syncthreads();
    if (threadIdx.x == 0) {
      const bool failed = *(const volatile unsigned long long*)err != ~0ull;
      __threadfence_system();  // the CTA's output writes (seen through the barrier) first
      *status_seq = seq | (failed ? kStatusErrBit : 0u);
    }
  }
}

// ---- WaitingQueue-level primitives (sched.cpp:59-123) ------------------------------------

__device__ __forceinline__ double key_of_bits(uint64_t u) {  // inverse of order_bits
  return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}

// WaitingQueue::push x m: slots first..first+m with caller-given keys and entry fields
__global__ void push_slots_kernel(QDev q, uint64_t first, uint64_t m, const uint64_t* ids,
                                  const double* keys, const double* E, const double* C,
                                  const uint8_t* predicted) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const uint64_t s = first + t;
  q.key[s] = order_bits(keys[t]);
  q.id[s] = ids[t];
  q.E[s] = E ? E[t] : 0.0;
  q.C[s] = C ? C[t] : 0.0;
  q.predicted[s] = predicted ? predicted[t] : 0;
}

// WaitingQueue::update x m (and the entry write-back of rebuild): keys (and optionally the
// entry fields) of existing slots
__global__ void set_slots_kernel(QDev q, const uint32_t* slots, uint64_t m, const double* keys,
                                 const double* E, const double* C, const uint8_t* predicted) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const uint32_t s = slots[t];
  q.key[s] = order_bits(keys[t]);
  if (E) q.E[s] = E[t];
  if (C) q.C[s] = C[t];
  if (predicted) q.predicted[s] = predicted[t];
}

// entries of the listed slots: key (decoded), E, C, predicted
__global__ void gather_slots_kernel(QDev q, const uint32_t* slots, uint64_t m, double* key,
                                    double* E, double* C, uint8_t* predicted) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const uint32_t s = slots[t];
  key[t] = key_of_bits(q.key[s]);
  E[t] = q.E[s];
  C[t] = q.C[s];
  predicted[t] = q.predicted[s];
}

// compaction / growth: new slot j <- old slot src[j] (j < m), dead beyond m up to cap
__global__ void relayout_kernel(QDev dst, QDev src, const uint32_t* from, uint64_t m,
                                uint64_t cap) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cap;
       j += (uint64_t)gridDim.x * blockDim.x) {
    if (j < m) {
      const uint32_t s = from[j];
      dst.key[j] = src.key[s];
      dst.id[j] = src.id[s];
      dst.E[j] = src.E[s];
      dst.C[j] = src.C[s];
      dst.predicted[j] = src.predicted[s];
    } else {
      dst.key[j] = kDead;
      dst.id[j] = kDead;
      dst.predicted[j] = 0;
    }
  }
}

// WaitingQueue::validate's device half: every block minimum equals a full rescan of its
// block; bad[0] counts mismatching blocks
__global__ void __launch_bounds__(256) validate_blocks_kernel(QDev q, uint32_t nb,
                                                              uint64_t n_slots,
                                                              unsigned int* bad) {
  __shared__ uint64_t sk[32], si[32];
  __shared__ uint32_t ss[32];
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    uint64_t k = kDead, i = kDead;
    uint32_t s = 0;
    for (uint32_t t = threadIdx.x; t < kBlockSlots; t += blockDim.x) {
      const uint64_t slot = (uint64_t)b * kBlockSlots + t;
      if (slot < n_slots && less_kv(q.key[slot], q.id[slot], k, i)) {
        k = q.key[slot];
        i = q.id[slot];
        s = (uint32_t)slot;
      }
    }
    block_argmin(k, i, s, sk, si, ss);
    if (threadIdx.x == 0 && (q.bkey[b] != k || q.bid[b] != i || (k != kDead && q.bslot[b] != s)))
      atomicAdd(bad, 1u);
  }
}

}  // namespace
}  // namespace dev
}  // namespace tie

using tie::capi::cuda_error;
using tie::capi::set_error;

constexpr uint32_t kCminCtas = 4096;  // grid cap of the cooperative re-key + pop kernel
static_assert(kCminCtas <= 4096, "rekey_pop_cand_kernel: lists per thread");

struct tie_queue {
  tie_ctx* ctx = nullptr;
  int policy = 2;  // 0 FCFS, 1 SEPT, 2 TIE  (sched.hpp:11)
  int adaptive = 1;
  double beta_fixed = 0.1, beta_max = 0.5, q_sat = 128.0, threshold = 0.1, alpha = 0.9;
  uint64_t capacity = 0, n_slots = 0, size = 0, n_predicted = 0;
  tie::host::FlatIdMap slot_of;  // the heap's pos_ index (sched.hpp:67)
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
  uint64_t out_cap = 0;
  void* h_out = nullptr;          // the pop output block (ensure_out), mapped pinned
  // completion record of a fused step, mapped pinned: written by the step's last kernel
  struct Status {
    unsigned long long err;
    volatile uint32_t seq;
  }* status = nullptr;
  uint32_t seq = 0;
  char* h_pack = nullptr;         // pinned H2D pack of a fused step
  char* d_pack = nullptr;
  uint64_t pack_cap = 0;
  uint64_t peers = 0;             // waiting requests held by other shards (beta's queue length)
  uint64_t* d_cmin = nullptr;     // [2][3][kCminCtas] CTA minima of the re-key + pop kernel
  void* d_cand = nullptr;         // CandScratch of the one-pass re-key + pop kernel
  uint64_t cand_nb = 0;           // blocks it is sized for
  uint64_t* h_peek_key = nullptr; // mapped pinned: keys of a peek's (undone) pops
  uint64_t peek_cap = 0;
  uint64_t* h_out_id = nullptr;   // pinned
  uint32_t* h_out_slot = nullptr;
  uint32_t* h_out_n = nullptr;
};

constexpr int kPolicyRaw = 3;  // a bare WaitingQueue: caller-given keys, no Scheduler rules

namespace {

double beta_at(const tie_queue* Q, uint64_t queue_len) {
  double b = 0.0;
  tie_compute_beta(Q->adaptive, Q->beta_fixed, Q->beta_max, Q->q_sat, queue_len, &b);
  return b;
}

// the beta of Scheduler::on_prediction (sched.cpp:139): SEPT 0, TIE compute_beta -- which
// throws std::domain_error on an invalid ScoreConfig (sched.cpp:10-15), reported here
int prediction_beta(const tie_queue* Q, double* beta) {
  *beta = 0.0;
  if (Q->policy != 2) return TIE_OK;
  return tie_compute_beta(Q->adaptive, Q->beta_fixed, Q->beta_max, Q->q_sat,
                          Q->size + Q->peers, beta);
}

// index of the first element of ids[0..m) whose id occurred earlier in the batch (m if none)
uint64_t first_batch_duplicate(const uint64_t* ids, uint64_t m) {
  std::vector<std::pair<uint64_t, uint64_t>> srt(m);
  for (uint64_t t = 0; t < m; ++t) srt[t] = {ids[t], t};
  std::sort(srt.begin(), srt.end());
  uint64_t first = m;
  for (uint64_t t = 1; t < m; ++t)
    if (srt[t].first == srt[t - 1].first) first = std::min(first, srt[t].second);
  return first;
}

// Scheduler::on_arrival x m validation (sched.cpp:125-132 -> WaitingQueue::push, 59-63): the
// error of the first failing request, as the reference's per-item loop raises it; fills the
// keys.  Changes nothing.
int check_arrivals(const tie_queue* Q, const uint64_t* ids, const double* arrival_s,
                   const uint32_t* max_tokens, uint64_t m, std::vector<double>& keys) {
  if (Q->n_slots + m > Q->capacity)
    return set_error(TIE_EINVALID, "tie_queue_arrive: capacity exceeded");  // see ensure_capacity
  keys.resize(m);
  const uint64_t dup = first_batch_duplicate(ids, m);
  for (uint64_t t = 0; t < m; ++t) {
    keys[t] = Q->policy == 0 ? arrival_s[t] : (double)max_tokens[t];
    if (!std::isfinite(keys[t]))
      return set_error(TIE_EDOMAIN, "WaitingQueue::push: key must be finite");
    if (t == dup || Q->slot_of.count(ids[t]))
      return set_error(TIE_EINVALID, "WaitingQueue::push: id " + std::to_string(ids[t]) +
                                         " already queued");
  }
  return TIE_OK;
}

// Scheduler::on_prediction x m validation up to the compute_score checks (sched.cpp:134-145):
// "not waiting", the policy's beta, "already predicted" (also for an id repeated inside the
// batch) -- the first failing request's error.  `pending` (may be null) holds ids of arrivals
// of the same step, not yet in slot_of, at slots first_pending + index.  Fills the slots and
// beta.  Changes nothing.
int check_predictions(const tie_queue* Q, const uint64_t* ids, uint64_t m,
                      const uint64_t* pending, uint64_t n_pending, uint64_t first_pending,
                      std::vector<uint32_t>& slots, double* beta, const double* E = nullptr,
                      const double* C = nullptr) {
  slots.resize(m);
  std::unordered_map<uint64_t, uint32_t> pend;  // this step's arrivals, built on first need
  bool pend_built = false;
  const uint64_t dup = Q->policy == 0 ? m : first_batch_duplicate(ids, m);
  *beta = 0.0;
  bool have_beta = false;
  for (uint64_t t = 0; t < m; ++t) {
    auto it = Q->slot_of.find(ids[t]);
    if (it != Q->slot_of.end()) {
      slots[t] = it->second;
    } else {
      if (!pend_built) {
        for (uint64_t u = 0; u < n_pending; ++u)
          pend.emplace(pending[u], (uint32_t)(first_pending + u));
        pend_built = true;
      }
      const auto p = pend.find(ids[t]);
      if (p == pend.end())
        return set_error(TIE_EINVALID, "Scheduler::on_prediction: id " +
                                           std::to_string(ids[t]) + " not waiting");
      slots[t] = p->second;
    }
    if (Q->policy == 0) continue;  // FCFS: arrival order is the schedule (sched.cpp:138)
    if (!have_beta) {  // the first waiting prediction evaluates compute_beta
      if (int rc = prediction_beta(Q, beta)) return rc;
      have_beta = true;
    }
    if (t == dup || Q->predicted[slots[t]])
      return set_error(TIE_EINVALID, "Scheduler::on_prediction: id " + std::to_string(ids[t]) +
                                         " already predicted");
    if (!E) continue;  // (E, CVaR) computed on the device: checked there
    const double e = E[t], c = C[t];  // compute_score checks (sched.cpp:19-26)
    if (!std::isfinite(e) || !std::isfinite(c) || !std::isfinite(*beta))
      return set_error(TIE_EDOMAIN, "compute_score: arguments must be finite");
    if (!(e > 0.0)) return set_error(TIE_EDOMAIN, "compute_score: expectation must be > 0");
    if (c < e)
      return set_error(TIE_EINVALID,
                       "compute_score: cvar below expectation violates the invariant");
  }
  return TIE_OK;
}

int ensure_stage(tie_queue* Q, uint64_t m) {
  if (m <= Q->stage_cap) return TIE_OK;
  cudaFree(Q->d_ids); cudaFree(Q->d_a); cudaFree(Q->d_b); cudaFree(Q->d_c);
  cudaFree(Q->d_slots); cudaFree(Q->d_blocks);
  const uint64_t cap = std::max<uint64_t>(m, 1024);
  cudaError_t e = cudaSuccess;
  if ((e = cudaMalloc(&Q->d_ids, 8 * cap)) || (e = cudaMalloc(&Q->d_a, 8 * cap)) ||
      (e = cudaMalloc(&Q->d_b, 8 * cap)) || (e = cudaMalloc(&Q->d_c, 8 * cap)) ||
      (e = cudaMalloc(&Q->d_slots, 4 * cap)) || (e = cudaMalloc(&Q->d_blocks, 4 * cap)))
    return cuda_error(e, "tie_queue: staging allocation");
  Q->stage_cap = cap;
  return TIE_OK;
}

// the pop output block: [out_n: u32 x cap | out_slot: u32 x cap | out_id: u64 x cap] in
// mapped pinned host memory -- the pop kernels write their results straight into it, so no
// D2H copy follows them (UVA: the host pointer is the device pointer)
int ensure_out(tie_queue* Q, uint64_t m) {
  if (m <= Q->out_cap) return TIE_OK;
  cudaFreeHost(Q->h_out);
  Q->h_out = nullptr;
  const uint64_t cap = std::max<uint64_t>(m, 256);
  cudaError_t e = cudaHostAlloc(&Q->h_out, 16 * cap, cudaHostAllocMapped);
  if (e != cudaSuccess) return cuda_error(e, "tie_queue: output allocation");
  Q->h_out_n = (uint32_t*)Q->h_out;
  Q->h_out_slot = Q->h_out_n + cap;
  Q->h_out_id = (uint64_t*)(Q->h_out_slot + cap);
  Q->d_out_n = Q->h_out_n;
  Q->d_out_slot = Q->h_out_slot;
  Q->d_out_id = Q->h_out_id;
  Q->out_cap = cap;
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

// Slots are append-only, so a long-lived queue (the simulator, a server) periodically needs
// a new layout: the live slots are gathered, in slot order, into arrays of `new_cap` slots --
// a compaction when popped slots dominate, else a growth.  The pop order is unaffected (it
// depends on (key, id) only); the host index is remapped and every block minimum rebuilt.
int relayout(tie_queue* Q, uint64_t new_cap) {
  namespace d = tie::dev;
  cudaStream_t s = Q->ctx->stream;
  std::vector<uint32_t> live;
  live.reserve(Q->size);
  for (uint64_t sl = 0; sl < Q->n_slots; ++sl)
    if (Q->alive[sl]) live.push_back((uint32_t)sl);
  const uint64_t m = live.size();
  const uint64_t nb = (new_cap + d::kBlockSlots - 1) / d::kBlockSlots;
  d::QDev nq{};
  uint32_t* d_from = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&nq.key, 8 * new_cap)) || (e = cudaMalloc(&nq.id, 8 * new_cap)) ||
      (e = cudaMalloc(&nq.E, 8 * new_cap)) || (e = cudaMalloc(&nq.C, 8 * new_cap)) ||
      (e = cudaMalloc(&nq.predicted, new_cap)) || (e = cudaMalloc(&nq.bkey, 8 * nb)) ||
      (e = cudaMalloc(&nq.bid, 8 * nb)) || (e = cudaMalloc(&nq.bslot, 4 * nb)) ||
      (e = cudaMalloc(&d_from, 4 * std::max<uint64_t>(m, 1)))) {
    for (void* p : {(void*)nq.key, (void*)nq.id, (void*)nq.E, (void*)nq.C, (void*)nq.predicted,
                    (void*)nq.bkey, (void*)nq.bid, (void*)nq.bslot, (void*)d_from})
      cudaFree(p);
    return cuda_error(e, "tie_queue: relayout allocation");
  }
  if (m) cudaMemcpyAsync(d_from, live.data(), 4 * m, cudaMemcpyHostToDevice, s);
  d::relayout_kernel<<<(unsigned)std::min<uint64_t>((new_cap + 255) / 256, 148 * 16), 256, 0,
                       s>>>(nq, Q->q, d_from, m, new_cap);
  cudaMemsetAsync(nq.bkey, 0xff, 8 * nb, s);
  cudaMemsetAsync(nq.bid, 0xff, 8 * nb, s);
  const uint32_t used_nb = (uint32_t)((m + d::kBlockSlots - 1) / d::kBlockSlots);
  if (used_nb)
    d::refresh_blocks_kernel<<<std::min<uint32_t>(used_nb, 4096), 256, 0, s>>>(nq, nullptr,
                                                                             used_nb, m);
  tie::capi::count_launch(used_nb ? 2 : 1);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_error(e, "tie_queue: relayout");
  cudaFree(d_from);
  for (void* p : {(void*)Q->q.key, (void*)Q->q.id, (void*)Q->q.E, (void*)Q->q.C,
                  (void*)Q->q.predicted, (void*)Q->q.bkey, (void*)Q->q.bid, (void*)Q->q.bslot})
    cudaFree(p);
  Q->q = nq;
  // host mirror, remapped
  std::vector<uint32_t> newpos(Q->n_slots, 0);
  for (uint64_t j = 0; j < m; ++j) newpos[live[j]] = (uint32_t)j;
  for (auto& kv : Q->slot_of) kv.second = newpos[kv.second];
  std::vector<uint8_t> alive(new_cap, 0), pred(new_cap, 0);
  std::vector<double> pbeta(new_cap, 0.0);
  std::vector<uint32_t> pepoch(new_cap, 0);
  for (uint64_t j = 0; j < m; ++j) {
    alive[j] = 1;
    pred[j] = Q->predicted[live[j]];
    pbeta[j] = Q->pred_beta[live[j]];
    pepoch[j] = Q->pred_epoch[live[j]];
  }
  Q->alive.swap(alive);
  Q->predicted.swap(pred);
  Q->pred_beta.swap(pbeta);
  Q->pred_epoch.swap(pepoch);
  Q->n_slots = m;
  Q->capacity = new_cap;
  return TIE_OK;
}

// room for m more slots: compact when at most half the capacity is live afterwards, else grow
int ensure_capacity(tie_queue* Q, uint64_t m) {
  if (Q->n_slots + m <= Q->capacity) return TIE_OK;
  const uint64_t need = Q->size + m;
  uint64_t cap = Q->capacity;
  if (need > cap / 2) cap = std::max<uint64_t>(2 * cap, need + need / 2);
  cap = std::min<uint64_t>(cap, (1ull << 32) - 1);
  if (need > cap) return set_error(TIE_EINVALID, "tie_queue: more than 2^32 - 1 waiting entries");
  return relayout(Q, cap);
}

void rebuild_launch(tie_queue* Q, double now, cudaStream_t s,
                    const unsigned long long* err = nullptr);
void rebuild_mirror(tie_queue* Q, double now);

int rebuild_all(tie_queue* Q, double now, cudaStream_t s) {  // sched.cpp:156-166
  rebuild_launch(Q, now, s);
  rebuild_mirror(Q, now);
  return TIE_OK;
}

void rebuild_launch(tie_queue* Q, double now, cudaStream_t s,
                    const unsigned long long* err) {
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  if (nb) tie::dev::rekey_refresh_kernel<<<std::min<uint32_t>(nb, 148 * 16), 256, 0, s>>>(
      Q->q, nb, Q->n_slots, now, err);
  tie::capi::count_launch(1);
}

void rebuild_mirror(tie_queue* Q, double now) {
  Q->betas.clear();
  if (Q->n_predicted) Q->betas[now] = Q->n_predicted;
  ++Q->epoch;  // every live predicted slot's beta_at_update is now `now`
  Q->rebuild_beta = now;
}

double drift(const tie_queue* Q, double now) {
  return std::max(std::fabs(now - Q->betas.begin()->first),
                  std::fabs(now - Q->betas.rbegin()->first));
}

// ---- pop planning: Scheduler::next_request() x left (sched.cpp:152-175) as a sequence of
// segments [drift rebuild?][fixed-key pops], planned on the host as far as the rebuild
// decisions are certain without seeing which entries the device pops:
//   * the multiset betas_in_use_ has n_predicted entries and only loses entries to pops, so
//     its range can only shrink and it is non-empty while n_predicted > pops so far;
//   * its range is exact at the start, after a rebuild (a single value) and while it holds a
//     single value; drift <= threshold over the (possibly wider) tracked range means "no
//     rebuild" for sure;
//   * a rebuild that would need the exact shrunken range, or the multiset's emptiness, ends
//     the plan (execute, sync, plan again).
struct Seg {
  bool rebuild;
  double beta;
  uint32_t pops;
};

std::vector<Seg> plan_pops(const tie_queue* Q, uint64_t left) {
  std::vector<Seg> plan;
  const bool tie_policy = Q->policy == 2;
  bool empty = Q->betas.empty();
  double lo = empty ? 0.0 : Q->betas.begin()->first;
  double hi = empty ? 0.0 : Q->betas.rbegin()->first;
  bool exact = true;
  for (uint64_t j = 0; j < left; ++j) {
    bool rebuild = false;
    double now = 0.0;
    if (tie_policy && !empty) {
      now = beta_at(Q, Q->size + Q->peers - j);
      const double d = std::max(std::fabs(now - lo), std::fabs(now - hi));
      if (d > Q->threshold) {
        if (!(exact && Q->n_predicted > j)) break;  // uncertain: stop here
        rebuild = true;
        lo = hi = now;
        exact = true;
      }
    }
    if (rebuild || plan.empty() || plan.back().pops >= (uint32_t)tie::dev::kTopB)
      plan.push_back({rebuild, now, 0});
    ++plan.back().pops;
    if (lo != hi) exact = false;
  }
  return plan;
}

// host mirror of `cnt` device pops (ids / slots in h_out_*, from offset `off`)
void apply_pops(tie_queue* Q, uint32_t off, uint32_t cnt, std::vector<uint64_t>& out) {
  for (uint32_t j = off; j < off + cnt; ++j) {
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
}

// launch a plan's kernels: segment g = [rebuild][pops -> d_out_*[off..], d_out_n[g]]; a set
// error word (a failed fused step) makes every kernel skip
// pops of a queue this small may come from fewer live blocks than pops: they go through
// pop_topb_kernel (which has the register path for that case), not the fused apply kernel
bool small_queue(const tie_queue* Q) { return Q->size < 8 * (uint64_t)tie::dev::kBlockSlots; }

// cooperative launch arguments (addresses handed to cudaLaunchCooperativeKernel)
struct QDevArgs {
  tie::dev::QDev q;
  uint32_t nb;
  uint64_t n_slots;
  tie::dev::SegBetas sb;
  uint32_t nseg;
  uint64_t* out_id;
  uint32_t* out_slot;
  uint32_t* out_n;
  uint64_t* cmin;
  const unsigned long long* err;
};

#ifndef TIE_CAND_MIN_BLOCKS
#define TIE_CAND_MIN_BLOCKS 512
#endif
constexpr uint32_t kCandMinBlocks = TIE_CAND_MIN_BLOCKS;

// the one-pass re-key + pop kernel's scratch: per-block (k_lo, id) / (k_hi, id) minima, the
// candidate slots, a count / overflow header and the threshold pair (grow-only)
int ensure_cand(tie_queue* Q, uint64_t nb) {
  if (nb <= Q->cand_nb && Q->d_cand) return TIE_OK;
  const uint64_t want = std::max<uint64_t>(nb, 1024);
  cudaFree(Q->d_cand);
  Q->d_cand = nullptr;
  Q->cand_nb = 0;
  const size_t bytes = 32 * want + 16 + 16 + 4 * tie::dev::kSeqCandCap + 512 * kCminCtas;
  if (cudaMalloc(&Q->d_cand, bytes) != cudaSuccess) {
    cudaGetLastError();
    return TIE_ECUDA;
  }
  Q->cand_nb = want;
  return TIE_OK;
}

tie::dev::CandScratch cand_scratch(tie_queue* Q) {
  char* b = (char*)Q->d_cand;
  tie::dev::CandScratch cs;
  cs.blo = (uint64_t*)b;
  cs.bhi = (uint64_t*)(b + 16 * Q->cand_nb);
  cs.thr = (uint64_t*)(b + 32 * Q->cand_nb);
  cs.hdr = (uint32_t*)(b + 32 * Q->cand_nb + 16);
  cs.cand = (uint32_t*)(b + 32 * Q->cand_nb + 32);
  cs.clist = (uint64_t*)(b + 32 * Q->cand_nb + 32 + 4 * tie::dev::kSeqCandCap);
  return cs;
}

uint64_t launch_plan(tie_queue* Q, const std::vector<Seg>& plan, size_t first_seg,
                     uint32_t off, cudaStream_t s, unsigned long long* err) {
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  static int rekey_ctas = -1;  // co-resident CTAs of the cooperative re-key + pop kernel
  static int cand_ctas = -1;   // ... of the one-pass (candidate) variant
  if (cand_ctas < 0) {
    int bpsm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, tie::dev::rekey_pop_cand_kernel,
                                                  tie::dev::kRekeyThreads, 0);
    cand_ctas = std::min(bpsm * sms, (int)kCminCtas);
    if (getenv("TIE_NO_REKEY_CAND")) cand_ctas = 0;  // A/B switch
  }
  if (rekey_ctas < 0) {
    int bpsm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, tie::dev::rekey_pop_seq_kernel,
                                                  tie::dev::kRekeyThreads, 0);
    if (const char* v = getenv("TIE_REKEY_CTAS_PER_SM")) bpsm = std::min(bpsm, atoi(v));
    rekey_ctas = std::min(bpsm * sms, (int)kCminCtas);
    if (getenv("TIE_NO_REKEY_SEQ")) rekey_ctas = 0;  // A/B switch
  }
  auto single_rebuild_pop = [&](size_t g) { return plan[g].rebuild && plan[g].pops == 1; };
  size_t g = first_seg;
  while (g < plan.size()) {
    size_t e = g;  // [g, e): a run of (rebuild, 1 pop) segments for one cooperative launch
    while (e < plan.size() && e - g < 32 && single_rebuild_pop(e)) ++e;
    // small queues: the per-segment passes are short and the one-pass kernel's fixed phases
    // (three grid syncs, the replay) dominate (B200 step p50: 300k slots 109 vs 86 us,
    // 1M 109 vs 122, 10M 197 vs 546, 64M 570 vs 2991)
    if (e - g >= 2 && cand_ctas > 0 && nb >= kCandMinBlocks && ensure_cand(Q, nb) == TIE_OK) {
      tie::dev::SegBetas sb{};
      for (size_t j = g; j < e; ++j) sb.b[j - g] = plan[j].beta;
      tie::dev::CandScratch cs = cand_scratch(Q);
      uint32_t nseg = (uint32_t)(e - g);
      uint64_t* out_id = Q->d_out_id + off;
      uint32_t* out_slot = Q->d_out_slot + off;
      uint32_t* out_n = Q->d_out_n + g;
      uint64_t n_slots = Q->n_slots;
      const uint32_t grid = std::min<uint32_t>(nb, (uint32_t)cand_ctas);
      void* args[] = {&Q->q, (void*)&nb, &n_slots, &sb, &nseg, &out_id, &out_slot, &out_n,
                      &Q->d_cmin, &cs, &err};
      if (cudaLaunchCooperativeKernel((const void*)tie::dev::rekey_pop_cand_kernel, grid,
                                      tie::dev::kRekeyThreads, args, 0, s) == cudaSuccess) {
        tie::capi::count_launch(1);
        off += nseg;
        g = e;
        continue;
      }
      cudaGetLastError();  // not launchable here: the per-segment variant below
    }
    if (e - g >= 2 && rekey_ctas > 0 && nb > 0) {
      tie::dev::SegBetas sb{};
      for (size_t j = g; j < e; ++j) sb.b[j - g] = plan[j].beta;
      static const int eager = getenv("TIE_REKEY_EAGER") ? 1 : 0;
      sb.eager = eager;
      QDevArgs a{Q->q, nb, Q->n_slots, sb, (uint32_t)(e - g), Q->d_out_id + off,
                 Q->d_out_slot + off, Q->d_out_n + g, Q->d_cmin, err};
      const uint32_t grid = std::min<uint32_t>(nb, (uint32_t)rekey_ctas);
      void* args[] = {&a.q, &a.nb, &a.n_slots, &a.sb, &a.nseg, &a.out_id, &a.out_slot,
                      &a.out_n, &a.cmin, &a.err};
      if (cudaLaunchCooperativeKernel((const void*)tie::dev::rekey_pop_seq_kernel, grid,
                                      tie::dev::kRekeyThreads, args, 0, s) == cudaSuccess) {
        tie::capi::count_launch(1);
        off += (uint32_t)(e - g);
        g = e;
        continue;
      }
      cudaGetLastError();  // not launchable here (e.g. co-residency): per-segment kernels
    }
    if (plan[g].rebuild) rebuild_launch(Q, plan[g].beta, s, err);
    if (small_queue(Q))
      tie::dev::pop_topb_kernel<<<1, 1024, 0, s>>>(Q->q, nb, Q->n_slots, plan[g].pops,
                                                   Q->d_out_id + off, Q->d_out_slot + off,
                                                   Q->d_out_n + g, nullptr, err);
    else
      tie::dev::step_apply_kernel<false><<<1, 1024, 0, s>>>(
          Q->q, 0, 0, nullptr, nullptr, nullptr, 0, nullptr, nullptr, 0.0, nullptr, 0, 0, nb,
          Q->n_slots, plan[g].pops, Q->d_out_id + off, Q->d_out_slot + off, Q->d_out_n + g,
          err, nullptr, 0u, nullptr);
    off += plan[g].pops;
    tie::capi::count_launch(1);
    ++g;
  }
  return off;
}

// D2H of a plan's results (issued after launch_plan)
void fetch_plan(tie_queue*, size_t, uint64_t, cudaStream_t) {}  // results are written to host

// host mirror of a finished plan, segment by segment (rebuild bookkeeping, then its pops);
// returns false when the queue ran dry
bool replay_plan(tie_queue* Q, const std::vector<Seg>& plan, std::vector<uint64_t>& out) {
  uint32_t off = 0;
  for (size_t g = 0; g < plan.size(); ++g) {
    if (plan[g].rebuild) rebuild_mirror(Q, plan[g].beta);
    apply_pops(Q, off, Q->h_out_n[g], out);
    if (Q->h_out_n[g] < plan[g].pops) return false;
    off += plan[g].pops;
  }
  return true;
}

// run a plan: all rebuild + pop kernels back to back, one packed D2H, one sync, replay
int execute_plan(tie_queue* Q, const std::vector<Seg>& plan, std::vector<uint64_t>& out,
                 cudaStream_t s) {
  uint64_t total = 0;
  for (const Seg& g : plan) total += g.pops;
  if (int rc = ensure_out(Q, std::max<uint64_t>(total, plan.size() + 1))) return rc;
  launch_plan(Q, plan, 0, 0, s, Q->ctx->d_err);
  fetch_plan(Q, plan.size(), total, s);
  if (const cudaError_t le = cudaGetLastError(); le != cudaSuccess)
    return cuda_error(le, "tie_queue_next");
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_error(e, "tie_queue_next");
  replay_plan(Q, plan, out);
  return TIE_OK;
}

}  // namespace

extern "C" {

int tie_queue_create(tie_ctx* ctx, int policy, int adaptive, double beta_fixed, double beta_max,
                     double q_sat, double rebuild_threshold, double alpha, uint64_t capacity,
                     tie_queue** out) {
  if (!ctx || !out) return set_error(TIE_EINVALID, "tie_queue_create: null argument");
  if (policy < 0 || policy > kPolicyRaw)
    return set_error(TIE_EINVALID, "tie_queue_create: bad policy");
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
      (e = cudaMalloc(&Q->q.predicted, capacity)) || (e = cudaMalloc(&Q->q.bkey, 8 * nb)) ||
      (e = cudaMalloc(&Q->d_cmin, 8 * 6 * kCminCtas)) ||
      (e = cudaMalloc(&Q->q.bid, 8 * nb)) || (e = cudaMalloc(&Q->q.bslot, 4 * nb)) ||
      ensure_stage(Q, 1024) != TIE_OK || ensure_out(Q, 256) != TIE_OK ||
      (e = cudaHostAlloc((void**)&Q->status, sizeof(*Q->status), cudaHostAllocMapped))) {
    tie_queue_destroy(Q);
    return cuda_error(e, "tie_queue_create");
  }
  Q->status->err = ~0ull;
  Q->status->seq = 0;
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
                  (void*)Q->q.predicted, (void*)Q->q.bkey, (void*)Q->q.bid,
                  (void*)Q->q.bslot, (void*)Q->d_ids, (void*)Q->d_a, (void*)Q->d_b,
                  (void*)Q->d_c, (void*)Q->d_slots, (void*)Q->d_blocks, (void*)Q->d_cmin,
                  Q->d_cand})
    cudaFree(p);
  cudaFreeHost(Q->h_out);
  cudaFreeHost(Q->h_peek_key);
  cudaFreeHost(Q->status);
  cudaFreeHost(Q->h_pack);
  cudaFree(Q->d_pack);
  delete Q;
}

uint64_t tie_queue_size(const tie_queue* Q) { return Q ? Q->size : 0; }

double tie_queue_current_beta(const tie_queue* Q) { return Q ? beta_at(Q, Q->size + Q->peers) : 0.0; }

// Scheduler::on_arrival x m (sched.cpp:125-132): key = FCFS ? arrival_s : max_tokens.
int tie_queue_arrive(tie_queue* Q, const uint64_t* ids, const double* arrival_s,
                     const uint32_t* max_tokens, uint64_t m) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (Q->policy == kPolicyRaw)
    return set_error(TIE_EINVALID, "tie_queue: a WaitingQueue has no Scheduler operations");
  if (m == 0) return TIE_OK;
  // validate the whole batch before any host state changes (a rejected batch leaves the
  // queue untouched)
  if (int rc = ensure_capacity(Q, m)) return rc;
  std::vector<double> keys;
  if (int rc = check_arrivals(Q, ids, arrival_s, max_tokens, m, keys)) return rc;
  for (uint64_t t = 0; t < m; ++t) Q->slot_of.emplace(ids[t], (uint32_t)(Q->n_slots + t));
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
  if (Q->policy == kPolicyRaw)
    return set_error(TIE_EINVALID, "tie_queue: a WaitingQueue has no Scheduler operations");
  if (m == 0) return TIE_OK;
  std::vector<uint32_t> slots;
  double beta = 0.0;
  if (int rc = check_predictions(Q, ids, m, nullptr, 0, 0, slots, &beta, E, C)) return rc;
  if (Q->policy == 0) return TIE_OK;  // FCFS: arrival order is the schedule
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
    std::vector<Seg> plan = plan_pops(Q, left);
    if (plan.empty()) {  // the very first decision is uncertain only if... never: j = 0 exact
      const double now = beta_at(Q, Q->size + Q->peers);
      plan.push_back({true, now, 1});
    }
    const size_t before = got.size();
    if (int rc = execute_plan(Q, plan, got, s)) return rc;
    const uint64_t popped = got.size() - before;
    if (popped == 0) break;
    left -= popped;
  }
  for (size_t j = 0; j < got.size(); ++j) out_ids[j] = got[j];
  *n_out = got.size();
  return TIE_OK;
}

// One scheduler iteration in ONE device round trip: Scheduler::on_arrival x n_arr, then
// run_sim's scoring chain + Scheduler::on_prediction x n_pred (sim.cpp:85-95,
// sched.cpp:134-150), then Scheduler::next_request() up to max_pops times (sched.cpp:169-175).
// Same results and errors as tie_queue_arrive + tie_queue_predict_logt + tie_queue_next: all
// host validation first, then one packed H2D, the kernels (the score / compute_score checks
// run on the device and make the writes and pops skip), one packed D2H and one sync.  Pops
// that a drift rebuild could precede continue through tie_queue_next.
namespace {
// one scheduler iteration; predictions as log-t (mu, sigma, max_tokens), scored on the device
// (E_in == nullptr), or as the caller's (E, C) pairs (on_prediction's arguments)
// TIE_STEP_PROFILE (development): host time per stage of tie_queue_step, summed over the
// process and printed at exit -- validation, mirror + plan, pack, launches, completion wait,
// replay
struct StepProfile {
  double ns[6] = {};
  uint64_t calls = 0;
  bool on = std::getenv("TIE_STEP_PROFILE") != nullptr;
  ~StepProfile() {
    if (!on || !calls) return;
    static const char* names[6] = {"validate", "mirror+plan", "pack", "launch", "wait", "replay"};
    std::fprintf(stderr, "tie_queue_step profile over %llu calls (us per call):",
                 (unsigned long long)calls);
    for (int i = 0; i < 6; ++i) std::fprintf(stderr, " %s %.2f", names[i], ns[i] / calls * 1e-3);
    std::fprintf(stderr, "\n");
  }
};
StepProfile g_step_prof;
struct StageClock {
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(int i) {
    if (!g_step_prof.on) return;
    const auto n = std::chrono::steady_clock::now();
    g_step_prof.ns[i] += std::chrono::duration<double, std::nano>(n - t).count();
    t = n;
  }
};

int queue_step_impl(tie_queue* Q, const uint64_t* arr_ids, const double* arr_time,
                    const uint32_t* arr_max_tokens, uint64_t n_arr, const uint64_t* pred_ids,
                    const double* mu, const double* sigma, const uint32_t* pred_max_tokens,
                    const double* E_in, const double* C_in, uint64_t n_pred, uint64_t max_pops,
                    uint64_t* out_ids, uint64_t* n_out, const uint64_t* arr_end = nullptr,
                    const uint64_t* pred_end = nullptr, uint64_t n_runs = 0) {
  if (!Q || !n_out) return set_error(TIE_EINVALID, "tie_queue: null argument");
  const bool ec = E_in != nullptr;
  *n_out = 0;
  if (Q->policy == kPolicyRaw)
    return set_error(TIE_EINVALID, "tie_queue: a WaitingQueue has no Scheduler operations");
  tie_ctx* ctx = Q->ctx;
  cudaStream_t s = ctx->stream;
  // ---- a multi-run step (tie_queue_step_ec_runs): runs r = 0..n_runs-1 of (arrivals, then
  // predictions), each prediction run scored with the beta of the queue length after the
  // arrivals up to its run.  One round trip when the whole sequence validates and fits the
  // small-step kernel; otherwise the runs go as consecutive single-run steps (the last one
  // popping), which is the definition -- and which raises the first error exactly where the
  // reference's call sequence does.
  std::vector<double> run_beta;  // per prediction, multi-run steps only
  if (n_runs > 1) {
    // (small enough for the single-CTA kernel: <= 4096 blocks touched, whatever the slots)
    static const bool no_runs = std::getenv("TIE_NO_STEP_RUNS") != nullptr;  // A/B switch
    bool one = !no_runs && ec && Q->policy != 0 && n_arr <= 16384 &&
               n_arr / tie::dev::kBlockSlots + 2 + n_pred <= 4096 &&
               ensure_capacity(Q, n_arr) == TIE_OK;
    std::vector<double> ak;
    if (one) one = check_arrivals(Q, arr_ids, arr_time, arr_max_tokens, n_arr, ak) == TIE_OK;
    if (one) one = first_batch_duplicate(pred_ids, n_pred) == n_pred;
    const uint64_t first_slot = Q->n_slots;
    run_beta.resize(one ? n_pred : 0);
    for (uint64_t r = 0, p0 = 0; one && r < n_runs; p0 = pred_end[r++]) {
      std::vector<uint32_t> sl;
      double b = 0.0;
      Q->size += arr_end[r];
      one = check_predictions(Q, pred_ids + p0, pred_end[r] - p0, arr_ids, arr_end[r],
                              first_slot, sl, &b, E_in + p0, C_in + p0) == TIE_OK;
      Q->size -= arr_end[r];
      for (uint64_t t = p0; one && t < pred_end[r]; ++t) run_beta[t] = b;
    }
    if (!one) {
      for (uint64_t r = 0, a0 = 0, p0 = 0; r < n_runs; a0 = arr_end[r], p0 = pred_end[r++]) {
        uint64_t k = 0;
        if (int rc = queue_step_impl(Q, arr_ids + a0, arr_time + a0, arr_max_tokens + a0,
                                     arr_end[r] - a0, pred_ids + p0, nullptr, nullptr, nullptr,
                                     E_in + p0, C_in + p0, pred_end[r] - p0,
                                     r + 1 == n_runs ? max_pops : 0, out_ids, &k))
          return rc;
        *n_out = k;
      }
      return TIE_OK;
    }
  }
  // ---- host validation of the whole step before any host state changes: the arrivals
  // (tie_queue_arrive), then the predictions with this step's arrivals counted as waiting
  // (tie_queue_predict).  A prediction error leaves the arrivals applied, as the reference's
  // on_arrival calls stay applied when a later on_prediction throws.
  StageClock clk;
  if (int rc = ensure_capacity(Q, n_arr)) return rc;
  std::vector<double> akeys;
  if (int rc = check_arrivals(Q, arr_ids, arr_time, arr_max_tokens, n_arr, akeys)) return rc;
  const uint64_t first = Q->n_slots;
  std::vector<uint32_t> slots;
  double beta = 0.0;
  {
    // predictions see the queue length after this step's arrivals (compute_beta at
    // on_prediction time, sched.cpp:139)
    Q->size += n_arr;
    const int rc = check_predictions(Q, pred_ids, n_pred, arr_ids, n_arr, first, slots, &beta,
                                     E_in, C_in);  // (E, C) given: checked here, as predict's
    Q->size -= n_arr;  // (a multi-run step passed this per run above: rc 0, run_beta holds
                       // the betas; `beta` here is the last run's and unused)
    if (rc) {
      const std::string msg = tie_last_error();
      if (int rc2 = tie_queue_arrive(Q, arr_ids, arr_time, arr_max_tokens, n_arr)) return rc2;
      return set_error(rc, msg);
    }
  }
  for (uint64_t t = 0; t < n_arr; ++t) {
    Q->slot_of.emplace(arr_ids[t], (uint32_t)(first + t));
    Q->alive[first + t] = 1;
  }
  Q->n_slots += n_arr;
  Q->size += n_arr;
  std::vector<uint32_t> blocks;  // refreshed unconditionally (arrivals) | if no error (preds)
  if (n_arr) {
    for (uint64_t t = 0; t < n_arr; t += tie::dev::kBlockSlots)
      blocks.push_back((uint32_t)((first + t) / tie::dev::kBlockSlots));
    blocks.push_back((uint32_t)((first + n_arr - 1) / tie::dev::kBlockSlots));
    std::sort(blocks.begin(), blocks.end());
    blocks.erase(std::unique(blocks.begin(), blocks.end()), blocks.end());
  }
  const uint32_t n_uncond = (uint32_t)blocks.size();
  // FCFS ignores predictions
  const bool use_pred = n_pred > 0 && Q->policy != 0;
  if (use_pred) {
    std::vector<uint32_t> pb;
    for (uint32_t sl : slots) pb.push_back(sl / tie::dev::kBlockSlots);
    std::sort(pb.begin(), pb.end());
    pb.erase(std::unique(pb.begin(), pb.end()), pb.end());
    for (uint32_t b : pb)
      if (!std::binary_search(blocks.begin(), blocks.begin() + n_uncond, b)) blocks.push_back(b);
  }
  // ---- predictions' host mirror, tentatively (rolled back if the device rejects them), so
  // the pop plan sees betas_in_use_ as the reference's next_request() will
  const bool multi = !run_beta.empty();
  auto pred_mirror = [&](bool apply) {
    for (uint64_t t = 0; t < slots.size(); ++t) {
      const uint32_t sl = slots[t];
      const double b = multi ? run_beta[t] : beta;
      Q->predicted[sl] = apply ? 1 : 0;
      Q->pred_beta[sl] = b;
      Q->pred_epoch[sl] = Q->epoch;
      if (!multi) continue;
      if (apply) {
        ++Q->betas[b];
      } else {
        auto it = Q->betas.find(b);
        if (it != Q->betas.end() && --it->second == 0) Q->betas.erase(it);
      }
    }
    if (apply) {
      if (!multi) Q->betas[beta] += n_pred;
      Q->n_predicted += n_pred;
    } else {
      if (!multi) {
        auto it = Q->betas.find(beta);
        if (it != Q->betas.end() && (it->second -= n_pred) == 0) Q->betas.erase(it);
      }
      Q->n_predicted -= n_pred;
    }
  };
  if (use_pred) pred_mirror(true);
  const uint64_t pops = std::min<uint64_t>(max_pops, Q->size);
  clk.mark(0);
  const std::vector<Seg> plan = plan_pops(Q, pops);
  uint64_t planned = 0;
  for (const Seg& g : plan) planned += g.pops;
  // segment 0's pops ride in the apply kernel unless a rebuild must precede them
  const bool seg0_fused = !plan.empty() && !plan[0].rebuild;
  const bool sq = small_queue(Q);  // its pops need the register path (step_apply<true>)
  const uint32_t fused_pops = seg0_fused ? plan[0].pops : 0;
  // ---- pack: [arr ids | arr keys | mu | sigma | E | C | key | pred slots | pred max_tokens |
  //            blocks]  (E, C, key: device-only scratch)
  auto al = [](uint64_t x) { return (x + 255) & ~(uint64_t)255; };
  const uint64_t np = use_pred ? n_pred : 0;
  const uint64_t o_aid = 0, o_akey = o_aid + al(8 * n_arr), o_mu = o_akey + al(8 * n_arr),
                 o_sg = o_mu + al(8 * np), o_slot = o_sg + al(8 * np),
                 o_mt = o_slot + al(4 * np), o_blk = o_mt + al(4 * np),
                 o_bet = o_blk + al(4 * blocks.size()),
                 o_h2d_end = o_bet + al(multi ? 8 * np : 0),  // host-provided up to here
                 o_E = o_h2d_end, o_C = o_E + al(8 * np), o_key = o_C + al(8 * np),
                 total = o_key + al(8 * np);
  if (total > Q->pack_cap) {
    cudaFreeHost(Q->h_pack);
    cudaFree(Q->d_pack);
    Q->h_pack = nullptr;
    Q->d_pack = nullptr;
    const uint64_t cap = std::max<uint64_t>(total, 1 << 20);
    cudaError_t e;
    if ((e = cudaMallocHost(&Q->h_pack, cap)) || (e = cudaMalloc(&Q->d_pack, cap))) {
      if (use_pred) pred_mirror(false);
      return cuda_error(e, "tie_queue_step: staging");
    }
    Q->pack_cap = cap;
  }
  if (int rc = ensure_out(Q, std::max<uint64_t>(planned, plan.size() + 1))) {
    if (use_pred) pred_mirror(false);
    return rc;
  }
  clk.mark(1);
  char* h = Q->h_pack;
  std::memcpy(h + o_aid, arr_ids, 8 * n_arr);
  std::memcpy(h + o_akey, akeys.data(), 8 * n_arr);
  if (np) {  // (E, C) steps carry E / C in the mu / sigma fields and no max_tokens
    std::memcpy(h + o_mu, ec ? E_in : mu, 8 * np);
    std::memcpy(h + o_sg, ec ? C_in : sigma, 8 * np);
    std::memcpy(h + o_slot, slots.data(), 4 * np);
    if (!ec) std::memcpy(h + o_mt, pred_max_tokens, 4 * np);
  }
  std::memcpy(h + o_blk, blocks.data(), 4 * blocks.size());
  if (multi && np) std::memcpy(h + o_bet, run_beta.data(), 8 * np);
  char* d = Q->d_pack;
  const bool small = n_arr <= 16384 && np <= 16384 && blocks.size() <= 4096;
  assert(!multi || small);  // the multi-run fast path's size condition above
  // small steps: the kernels read the pack straight from pinned host memory (no H2D copy);
  // the device pack keeps the scratch (E, C, key)
  clk.mark(2);
  const char* in = small ? h : d;
  if (!small) cudaMemcpyAsync(d, h, o_h2d_end, cudaMemcpyHostToDevice, s);  // ONE H2D
  ctx->err_op = "tie_queue_step";
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  // the predictions' (E, C): scored here, or the caller's (in the pack)
  const double* pE = ec ? (const double*)(in + o_mu) : (const double*)(d + o_E);
  double* pC = ec ? (double*)(in + o_sg) : (double*)(d + o_C);
  if (np && !ec) {
    const cudaError_t e = tie::dev::launch_score(
        ctx, (const double*)(in + o_mu), (const double*)(in + o_sg), in + o_mt, true, np, Q->alpha,
        0.0, (double*)(d + o_E), (double*)(d + o_C), nullptr, nullptr, nullptr, TIE_SCORE_RAW,
        s);
    if (e != cudaSuccess) {
      pred_mirror(false);
      return cuda_error(e, "tie_queue_step");
    }
  }
  uint32_t* seg0_n = Q->d_out_n + (seg0_fused ? 0 : plan.size());  // unused slot if not fused
  const uint32_t seq = ++Q->seq & ~tie::dev::kStatusErrBit;  // 31 bits: the top is the error bit
  // the apply kernel is the step's last kernel when no further plan segments follow it
  const bool apply_last = small && plan.size() <= (seg0_fused ? 1u : 0u);
  if (small) {  // everything after the scoring in one single-CTA kernel
    // after a score launch: a programmatic dependent launch, so its launch and the arrivals'
    // writes overlap the score kernel (the kernel waits before reading E / C)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    // packs up to 32 KB are staged into the kernel's shared memory (one PCIe round trip)
    static const bool no_stage = std::getenv("TIE_NO_PACK_STAGE") != nullptr;  // A/B switch
    const uint32_t stage = !no_stage && o_h2d_end <= 32768 ? (uint32_t)o_h2d_end : 0u;
    cfg.dynamicSmemBytes = stage;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (np && !ec) ? 1 : 0;
    const cudaError_t le0 = cudaLaunchKernelEx(
        &cfg, sq ? tie::dev::step_apply_kernel<true> : tie::dev::step_apply_kernel<false>, Q->q,
        first, n_arr, (const uint64_t*)(in + o_aid), (const double*)(in + o_akey),
        (const uint32_t*)(in + o_slot), np, pE, pC, beta, (const uint32_t*)(in + o_blk),
        (uint32_t)blocks.size(), n_uncond, nb, Q->n_slots, fused_pops, Q->d_out_id,
        Q->d_out_slot, seg0_n, ctx->d_err, apply_last ? &Q->status->seq : nullptr, seq,
        multi && np ? (const double*)(in + o_bet) : nullptr, (const char*)h, stage);
    if (le0 != cudaSuccess) {
      if (use_pred) pred_mirror(false);
      return cuda_error(le0, "tie_queue_step");
    }
    tie::capi::count_launch(1);
  } else {
    if (n_arr)
      tie::dev::write_slots_kernel<<<(unsigned)((n_arr + 255) / 256), 256, 0, s>>>(
          Q->q, first, n_arr, (const uint64_t*)(d + o_aid), (const double*)(d + o_akey));
    if (np) {
      const unsigned g = (unsigned)((np + 255) / 256);
      tie::dev::predict_keys_kernel<<<g, 256, 0, s>>>(pE, pC, np, beta, (double*)(d + o_key),
                                                      ctx->d_err);
      tie::dev::write_predictions_checked_kernel<<<g, 256, 0, s>>>(
          Q->q, (const uint32_t*)(d + o_slot), np, pE, pC, (const double*)(d + o_key), beta,
          ctx->d_err);
    }
    if (!blocks.empty())
      tie::dev::refresh_blocks_checked_kernel<<<
          (unsigned)std::min<size_t>(blocks.size(), 4096), 256, 0, s>>>(
          Q->q, (const uint32_t*)(d + o_blk), (uint32_t)blocks.size(), Q->n_slots, ctx->d_err,
          n_uncond);
    if (fused_pops)
      (sq ? tie::dev::step_apply_kernel<true> : tie::dev::step_apply_kernel<false>)<<<1, 1024, 0, s>>>(
          Q->q, 0, 0, nullptr, nullptr, nullptr, 0, nullptr, nullptr, beta, nullptr, 0, 0, nb,
          Q->n_slots, fused_pops, Q->d_out_id, Q->d_out_slot, seg0_n, ctx->d_err, nullptr,
          0u, nullptr, nullptr, 0u);
    tie::capi::count_launch((n_arr ? 1 : 0) + (np ? 2 : 0) + (blocks.empty() ? 0 : 1) +
                            (fused_pops ? 1 : 0));
  }
  launch_plan(Q, plan, seg0_fused ? 1 : 0, fused_pops, s, ctx->d_err);
  // completion: the last kernel publishes the error word and the step's sequence number in
  // mapped host memory; the host polls it (a stream synchronisation costs more than the
  // whole small step) and falls back to synchronising after 20 ms
  if (!apply_last) {
    tie::dev::step_finish_kernel<<<1, 1, 0, s>>>(ctx->d_err, &Q->status->seq,
                                                 seq);
    tie::capi::count_launch();
  }
  clk.mark(3);
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) {
    if (use_pred) pred_mirror(false);
    return cuda_error(le, "tie_queue_step");
  }
  {
    const auto t0 = std::chrono::steady_clock::now();
    while ((Q->status->seq & ~tie::dev::kStatusErrBit) != seq) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(20)) {
        if (std::getenv("TIE_STEP_DEBUG"))
          std::fprintf(stderr, "tie_queue_step: 20 ms poll timeout (seq %u, n_arr %llu, n_pred %llu, "
                       "pops %llu, plan %zu, small %d, apply_last %d)\n", seq,
                       (unsigned long long)n_arr, (unsigned long long)n_pred,
                       (unsigned long long)pops, plan.size(), (int)small, (int)apply_last);
        const cudaError_t se = cudaStreamSynchronize(s);
        if (se != cudaSuccess) {
          if (use_pred) pred_mirror(false);
          return cuda_error(se, "tie_queue_step");
        }
        break;
      }
    }
  }
  // the error word (tie_sync decodes + resets it); arrivals stay applied like the reference's
  if (Q->status->seq & tie::dev::kStatusErrBit) {
    if (int rc = tie_sync(ctx, s)) {
      if (use_pred) pred_mirror(false);
      return rc;
    }
  }
  clk.mark(4);
  std::vector<uint64_t> got;
  const bool dry = !replay_plan(Q, plan, got);
  uint64_t k = got.size();
  for (uint64_t j = 0; j < k; ++j) out_ids[j] = got[j];
  if (!dry && k < pops) {  // the plan stopped at an uncertain rebuild decision
    uint64_t more = 0;
    if (int rc = tie_queue_next(Q, pops - k, out_ids + k, &more)) return rc;
    k += more;
  }
  *n_out = k;
  clk.mark(5);
  ++g_step_prof.calls;
  return TIE_OK;
}

}  // namespace

int tie_queue_step(tie_queue* Q, const uint64_t* arr_ids, const double* arr_time,
                   const uint32_t* arr_max_tokens, uint64_t n_arr, const uint64_t* pred_ids,
                   const double* mu, const double* sigma, const uint32_t* pred_max_tokens,
                   uint64_t n_pred, uint64_t max_pops, uint64_t* out_ids, uint64_t* n_out) {
  return queue_step_impl(Q, arr_ids, arr_time, arr_max_tokens, n_arr, pred_ids, mu, sigma,
                         pred_max_tokens, nullptr, nullptr, n_pred, max_pops, out_ids, n_out);
}

int tie_queue_step_ec(tie_queue* Q, const uint64_t* arr_ids, const double* arr_time,
                      const uint32_t* arr_max_tokens, uint64_t n_arr, const uint64_t* pred_ids,
                      const double* E, const double* C, uint64_t n_pred, uint64_t max_pops,
                      uint64_t* out_ids, uint64_t* n_out) {
  if (n_pred && (!E || !C)) return set_error(TIE_EINVALID, "tie_queue_step_ec: null E / C");
  static const double kNone = 0.0;  // E_in != nullptr selects the (E, C) mode
  return queue_step_impl(Q, arr_ids, arr_time, arr_max_tokens, n_arr, pred_ids, nullptr,
                         nullptr, nullptr, n_pred ? E : &kNone, n_pred ? C : &kNone, n_pred,
                         max_pops, out_ids, n_out);
}

int tie_queue_step_ec_runs(tie_queue* Q, const uint64_t* arr_ids, const double* arr_time,
                           const uint32_t* arr_max_tokens, const uint64_t* arr_end,
                           const uint64_t* pred_ids, const double* E, const double* C,
                           const uint64_t* pred_end, uint64_t n_runs, uint64_t max_pops,
                           uint64_t* out_ids, uint64_t* n_out) {
  if (!n_out || (n_runs && (!arr_end || !pred_end)))
    return set_error(TIE_EINVALID, "tie_queue_step_ec_runs: null argument");
  if (n_runs == 0)
    return tie_queue_step_ec(Q, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0,
                             max_pops, out_ids, n_out);
  for (uint64_t r = 1; r < n_runs; ++r)
    if (arr_end[r] < arr_end[r - 1] || pred_end[r] < pred_end[r - 1])
      return set_error(TIE_EINVALID, "tie_queue_step_ec_runs: run ends must not decrease");
  const uint64_t n_arr = arr_end[n_runs - 1], n_pred = pred_end[n_runs - 1];
  if (n_pred && (!E || !C)) return set_error(TIE_EINVALID, "tie_queue_step_ec_runs: null E / C");
  if (n_runs == 1)
    return tie_queue_step_ec(Q, arr_ids, arr_time, arr_max_tokens, n_arr, pred_ids, E, C, n_pred,
                             max_pops, out_ids, n_out);
  static const double kNone = 0.0;
  return queue_step_impl(Q, arr_ids, arr_time, arr_max_tokens, n_arr, pred_ids, nullptr,
                         nullptr, nullptr, n_pred ? E : &kNone, n_pred ? C : &kNone, n_pred,
                         max_pops, out_ids, n_out, arr_end, pred_end, n_runs);
}

// ---- shard-level primitives (the scheduler sharded by request) ------------
// A sharded scheduler keeps each request's (E, CVaR) on its owner GPU and reproduces ONE
// reference Scheduler over the union of the shards; these expose what the coordinating layer
// (paper_2604_00499_b200/dist.py ShardedScheduler) needs to make the global decisions.

// beta's queue length is this shard's waiting count plus `peers` (compute_beta over the
// GLOBAL queue, sched.cpp:9-17, 136, 154)
int tie_queue_set_peer_waiting(tie_queue* Q, uint64_t peers) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  Q->peers = peers;
  return TIE_OK;
}

// betas_in_use_ of this shard (sched.hpp:88): its extremes and size (0: empty)
int tie_queue_beta_range(const tie_queue* Q, double* lo, double* hi, uint64_t* n_in_use) {
  if (!Q || !lo || !hi || !n_in_use) return set_error(TIE_EINVALID, "tie_queue: null argument");
  *n_in_use = 0;
  *lo = *hi = 0.0;
  if (Q->betas.empty()) return TIE_OK;
  *lo = Q->betas.begin()->first;
  *hi = Q->betas.rbegin()->first;
  for (const auto& kv : Q->betas) *n_in_use += kv.second;
  return TIE_OK;
}

// the rebuild of rebuild_if_drifted (sched.cpp:156-166) at a beta decided elsewhere: every
// predicted entry of this shard is re-keyed with `beta` (no-op when it has none)
int tie_queue_rebuild_at(tie_queue* Q, double beta) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (Q->policy != 2 || Q->betas.empty()) return TIE_OK;
  if (int rc = rebuild_all(Q, beta, Q->ctx->stream)) return rc;
  const cudaError_t e = cudaStreamSynchronize(Q->ctx->stream);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_queue_rebuild_at");
}

// the next min(k, waiting) entries in pop order under the CURRENT keys -- (key, id) with the
// key's order-preserving u64 bits, comparable across shards -- without popping them and
// without any drift rebuild: pops on the device, then the popped keys restored
int tie_queue_peek(tie_queue* Q, uint64_t k, uint64_t* keys, uint64_t* ids, uint64_t* n_out) {
  if (!Q || !n_out || (k && (!keys || !ids)))
    return set_error(TIE_EINVALID, "tie_queue: null argument");
  *n_out = 0;
  k = std::min<uint64_t>(k, Q->size);
  if (!k) return TIE_OK;
  const uint64_t nseg = (k + tie::dev::kTopB - 1) / tie::dev::kTopB;
  if (int rc = ensure_out(Q, std::max<uint64_t>(k, nseg + 1))) return rc;
  if (k > Q->peek_cap) {
    cudaFreeHost(Q->h_peek_key);
    Q->h_peek_key = nullptr;
    Q->peek_cap = 0;
    const cudaError_t e = cudaHostAlloc((void**)&Q->h_peek_key, 8 * std::max<uint64_t>(k, 256),
                                        cudaHostAllocMapped);
    if (e != cudaSuccess) return cuda_error(e, "tie_queue_peek: allocation");
    Q->peek_cap = std::max<uint64_t>(k, 256);
  }
  cudaStream_t s = Q->ctx->stream;
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  uint64_t off = 0;
  for (uint64_t g = 0; g < nseg; ++g) {
    const uint32_t cnt = (uint32_t)std::min<uint64_t>(tie::dev::kTopB, k - off);
    tie::dev::pop_topb_kernel<<<1, 1024, 0, s>>>(Q->q, nb, Q->n_slots, cnt, Q->d_out_id + off,
                                                 Q->d_out_slot + off, Q->d_out_n + g,
                                                 Q->h_peek_key + off);
    off += cnt;
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_error(e, "tie_queue_peek");
  uint64_t got = 0;
  for (uint64_t g = 0; g < nseg; ++g) got += Q->h_out_n[g];  // == k: k <= waiting
  tie::dev::unpop_kernel<<<1, 1024, 0, s>>>(Q->q, Q->d_out_slot, Q->h_peek_key, (uint32_t)got,
                                            Q->n_slots);
  tie::capi::count_launch(nseg + 1);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_error(e, "tie_queue_peek");
  for (uint64_t j = 0; j < got; ++j) {
    keys[j] = Q->h_peek_key[j];
    ids[j] = Q->h_out_id[j];
  }
  *n_out = got;
  return TIE_OK;
}

int tie_queue_rebuild_if_drifted(tie_queue* Q, int* rebuilt) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (rebuilt) *rebuilt = 0;
  if (Q->policy != 2 || Q->betas.empty()) return TIE_OK;
  const double now = beta_at(Q, Q->size + Q->peers);
  if (!(drift(Q, now) > Q->threshold)) return TIE_OK;
  if (int rc = rebuild_all(Q, now, Q->ctx->stream)) return rc;
  if (rebuilt) *rebuilt = 1;
  const cudaError_t e = cudaStreamSynchronize(Q->ctx->stream);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_queue_rebuild_if_drifted");
}

// ---- WaitingQueue (sched.hpp:43-68, sched.cpp:28-123) ------------------------------------

int tie_queue_contains(const tie_queue* Q, uint64_t id) {
  return Q && Q->slot_of.count(id) ? 1 : 0;
}

// WaitingQueue::push x m (sched.cpp:59-67); predicted / E / C / beta_at_update may be NULL
int tie_queue_push(tie_queue* Q, const uint64_t* ids, const double* keys,
                   const uint8_t* predicted, const double* E, const double* C,
                   const double* beta_at_update, uint64_t m) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (Q->policy != kPolicyRaw)
    return set_error(TIE_EINVALID, "tie_queue_push: a Scheduler's queue is keyed by its policy");
  if (m == 0) return TIE_OK;
  if (!ids || !keys) return set_error(TIE_EINVALID, "tie_queue_push: null argument");
  if (int rc = ensure_capacity(Q, m)) return rc;
  const uint64_t dup = first_batch_duplicate(ids, m);
  for (uint64_t t = 0; t < m; ++t) {
    if (!std::isfinite(keys[t]))
      return set_error(TIE_EDOMAIN, "WaitingQueue::push: key must be finite");
    if (t == dup || Q->slot_of.count(ids[t]))
      return set_error(TIE_EINVALID, "WaitingQueue::push: id " + std::to_string(ids[t]) +
                                         " already queued");
  }
  cudaStream_t s = Q->ctx->stream;
  if (int rc = ensure_stage(Q, m)) return rc;
  const uint64_t first = Q->n_slots;
  // staging: ids | keys | E | C | predicted (u8 packed into d_slots' bytes)
  cudaMemcpyAsync(Q->d_ids, ids, 8 * m, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(Q->d_a, keys, 8 * m, cudaMemcpyHostToDevice, s);
  if (E) cudaMemcpyAsync(Q->d_b, E, 8 * m, cudaMemcpyHostToDevice, s);
  if (C) cudaMemcpyAsync(Q->d_c, C, 8 * m, cudaMemcpyHostToDevice, s);
  if (predicted) cudaMemcpyAsync(Q->d_slots, predicted, m, cudaMemcpyHostToDevice, s);
  tie::dev::push_slots_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(
      Q->q, first, m, Q->d_ids, Q->d_a, E ? Q->d_b : nullptr, C ? Q->d_c : nullptr,
      predicted ? (const uint8_t*)Q->d_slots : nullptr);
  tie::capi::count_launch();
  std::vector<uint32_t> touched;
  for (uint64_t t = 0; t < m; ++t) {
    const uint32_t sl = (uint32_t)(first + t);
    Q->slot_of.emplace(ids[t], sl);
    Q->alive[sl] = 1;
    Q->predicted[sl] = predicted && predicted[t] ? 1 : 0;
    Q->pred_beta[sl] = beta_at_update ? beta_at_update[t] : 0.0;
    Q->pred_epoch[sl] = Q->epoch;
    if (Q->predicted[sl]) ++Q->n_predicted;
  }
  for (uint64_t t = 0; t < m; t += tie::dev::kBlockSlots) touched.push_back((uint32_t)(first + t));
  touched.push_back((uint32_t)(first + m - 1));
  Q->n_slots += m;
  Q->size += m;
  if (int rc = refresh(Q, touched, s)) return rc;
  const cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, "tie_queue_push");
}

namespace {

// write keys (and, when given, entry fields) of waiting entries; `who` names the reference
// operation for the error messages.  Repeated ids: the last write wins, as sequential calls.
int write_entries(tie_queue* Q, const uint64_t* ids, const double* keys, const uint8_t* pred,
                  const double* E, const double* C, const double* beta, uint64_t m,
                  const char* who) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (Q->policy != kPolicyRaw)
    return set_error(TIE_EINVALID, std::string(who) + ": a Scheduler's queue is keyed by its policy");
  if (m == 0) return TIE_OK;
  if (!ids || !keys) return set_error(TIE_EINVALID, std::string(who) + ": null argument");
  std::vector<uint32_t> slots(m);
  for (uint64_t t = 0; t < m; ++t) {  // update(): finiteness, then the id (sched.cpp:69-74)
    if (!std::isfinite(keys[t]))
      return set_error(TIE_EDOMAIN, std::string(who) + ": key must be finite");
    auto it = Q->slot_of.find(ids[t]);
    if (it == Q->slot_of.end())
      return set_error(TIE_EINVALID, std::string(who) + ": id " + std::to_string(ids[t]) +
                                         " not queued");
    slots[t] = it->second;
  }
  // keep the last occurrence of each slot
  std::vector<uint64_t> keep;
  {
    std::unordered_map<uint32_t, uint64_t> last;
    for (uint64_t t = 0; t < m; ++t) last[slots[t]] = t;
    keep.reserve(last.size());
    for (uint64_t t = 0; t < m; ++t)
      if (last[slots[t]] == t) keep.push_back(t);
  }
  const uint64_t k = keep.size();
  std::vector<uint32_t> ks(k);
  std::vector<double> kk(k), ke, kc;
  std::vector<uint8_t> kp;
  if (E) ke.resize(k);
  if (C) kc.resize(k);
  if (pred) kp.resize(k);
  for (uint64_t j = 0; j < k; ++j) {
    const uint64_t t = keep[j];
    ks[j] = slots[t];
    kk[j] = keys[t];
    if (E) ke[j] = E[t];
    if (C) kc[j] = C[t];
    if (pred) kp[j] = pred[t] ? 1 : 0;
  }
  cudaStream_t s = Q->ctx->stream;
  if (int rc = ensure_stage(Q, k)) return rc;
  cudaMemcpyAsync(Q->d_slots, ks.data(), 4 * k, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(Q->d_a, kk.data(), 8 * k, cudaMemcpyHostToDevice, s);
  if (E) cudaMemcpyAsync(Q->d_b, ke.data(), 8 * k, cudaMemcpyHostToDevice, s);
  if (C) cudaMemcpyAsync(Q->d_c, kc.data(), 8 * k, cudaMemcpyHostToDevice, s);
  if (pred) cudaMemcpyAsync(Q->d_ids, kp.data(), k, cudaMemcpyHostToDevice, s);
  tie::dev::set_slots_kernel<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(
      Q->q, Q->d_slots, k, Q->d_a, E ? Q->d_b : nullptr, C ? Q->d_c : nullptr,
      pred ? (const uint8_t*)Q->d_ids : nullptr);
  tie::capi::count_launch();
  for (uint64_t j = 0; j < k; ++j) {
    const uint32_t sl = ks[j];
    if (pred) {
      if (Q->predicted[sl] && !kp[j]) --Q->n_predicted;
      if (!Q->predicted[sl] && kp[j]) ++Q->n_predicted;
      Q->predicted[sl] = kp[j];
    }
    if (beta) {
      Q->pred_beta[sl] = beta[keep[j]];
      Q->pred_epoch[sl] = Q->epoch;
    }
  }
  if (int rc = refresh(Q, ks, s)) return rc;
  const cudaError_t e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? TIE_OK : cuda_error(e, who);
}

}  // namespace

// WaitingQueue::update x m (sched.cpp:69-79)
int tie_queue_update(tie_queue* Q, const uint64_t* ids, const double* keys, uint64_t m) {
  return write_entries(Q, ids, keys, nullptr, nullptr, nullptr, nullptr, m,
                       "WaitingQueue::update");
}

// entry write-back (the edits WaitingQueue::entries() / at() hand out, then rebuild(),
// sched.cpp:110-114)
int tie_queue_set_entries(tie_queue* Q, const uint64_t* ids, const double* keys,
                          const uint8_t* predicted, const double* E, const double* C,
                          const double* beta_at_update, uint64_t m) {
  return write_entries(Q, ids, keys, predicted, E, C, beta_at_update, m, "WaitingQueue::rebuild");
}

namespace {

int gather_entries(tie_queue* Q, const std::vector<uint32_t>& slots, uint64_t* ids,
                   double* keys, uint8_t* predicted, double* E, double* C, double* beta) {
  const uint64_t m = slots.size();
  if (m == 0) return TIE_OK;
  cudaStream_t s = Q->ctx->stream;
  if (int rc = ensure_stage(Q, m)) return rc;
  std::vector<double> k(m), e(m), c(m);
  std::vector<uint8_t> p(m);
  std::vector<uint64_t> id(m);
  cudaMemcpyAsync(Q->d_slots, slots.data(), 4 * m, cudaMemcpyHostToDevice, s);
  tie::dev::gather_slots_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(
      Q->q, Q->d_slots, m, Q->d_a, Q->d_b, Q->d_c, (uint8_t*)Q->d_blocks);
  tie::capi::count_launch();
  cudaMemcpyAsync(k.data(), Q->d_a, 8 * m, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(e.data(), Q->d_b, 8 * m, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(c.data(), Q->d_c, 8 * m, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(p.data(), Q->d_blocks, m, cudaMemcpyDeviceToHost, s);
  const cudaError_t err = cudaStreamSynchronize(s);
  if (err != cudaSuccess) return cuda_error(err, "tie_queue: entry read");
  for (uint64_t t = 0; t < m; ++t) {
    if (keys) keys[t] = k[t];
    if (E) E[t] = e[t];
    if (C) C[t] = c[t];
    if (predicted) predicted[t] = p[t];
    if (beta) {  // a Scheduler's unpredicted entries keep QueueEntry's default 0
      const uint32_t sl = slots[t];
      beta[t] = Q->policy == kPolicyRaw ? Q->pred_beta[sl]
                                         : (Q->predicted[sl] ? Q->beta_of(sl) : 0.0);
    }
  }
  (void)ids;
  return TIE_OK;
}

}  // namespace

// WaitingQueue::at x m (sched.cpp:96-108): the entries of waiting ids; any output may be NULL
int tie_queue_get(tie_queue* Q, const uint64_t* ids, uint64_t m, double* keys,
                  uint8_t* predicted, double* E, double* C, double* beta_at_update) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  std::vector<uint32_t> slots(m);
  for (uint64_t t = 0; t < m; ++t) {
    auto it = Q->slot_of.find(ids[t]);
    if (it == Q->slot_of.end())
      return set_error(TIE_EINVALID, "WaitingQueue::at: id " + std::to_string(ids[t]) +
                                         " not queued");
    slots[t] = it->second;
  }
  return gather_entries(Q, slots, nullptr, keys, predicted, E, C, beta_at_update);
}

// WaitingQueue::entries() (sched.hpp:60-61): every waiting entry, in slot (arrival) order --
// the reference hands out its heap array, whose order is unspecified as well
int tie_queue_entries(tie_queue* Q, uint64_t cap, uint64_t* ids, double* keys,
                      uint8_t* predicted, double* E, double* C, double* beta_at_update,
                      uint64_t* n_out) {
  if (!Q || !n_out) return set_error(TIE_EINVALID, "tie_queue: null argument");
  *n_out = 0;
  std::vector<std::pair<uint32_t, uint64_t>> live;
  live.reserve(Q->size);
  for (const auto& kv : Q->slot_of) live.push_back({kv.second, kv.first});
  std::sort(live.begin(), live.end());
  if (live.size() > cap) return set_error(TIE_EINVALID, "tie_queue_entries: buffer too small");
  std::vector<uint32_t> slots(live.size());
  for (size_t j = 0; j < live.size(); ++j) {
    slots[j] = live[j].first;
    if (ids) ids[j] = live[j].second;
  }
  if (int rc = gather_entries(Q, slots, nullptr, keys, predicted, E, C, beta_at_update)) return rc;
  *n_out = live.size();
  return TIE_OK;
}

// WaitingQueue::pop_min() x max_pops (sched.cpp:81-94) with the popped entries (raw queues;
// a Scheduler pops through tie_queue_next).  Any output but ids / n_out may be NULL.
int tie_queue_pop(tie_queue* Q, uint64_t max_pops, uint64_t* ids, double* keys,
                  uint8_t* predicted, double* E, double* C, double* beta_at_update,
                  uint64_t* n_out) {
  if (!Q || !n_out) return set_error(TIE_EINVALID, "tie_queue: null argument");
  *n_out = 0;
  if (Q->policy != kPolicyRaw)
    return set_error(TIE_EINVALID, "tie_queue_pop: a Scheduler pops through next_request");
  const uint64_t k = std::min<uint64_t>(max_pops, Q->size);
  if (!k) return TIE_OK;
  const uint64_t nseg = (k + tie::dev::kTopB - 1) / tie::dev::kTopB;
  if (int rc = ensure_out(Q, std::max<uint64_t>(k, nseg + 1))) return rc;
  if (k > Q->peek_cap) {
    cudaFreeHost(Q->h_peek_key);
    Q->h_peek_key = nullptr;
    Q->peek_cap = 0;
    const cudaError_t e = cudaHostAlloc((void**)&Q->h_peek_key, 8 * std::max<uint64_t>(k, 256),
                                        cudaHostAllocMapped);
    if (e != cudaSuccess) return cuda_error(e, "tie_queue_pop: allocation");
    Q->peek_cap = std::max<uint64_t>(k, 256);
  }
  cudaStream_t s = Q->ctx->stream;
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  uint64_t off = 0;
  for (uint64_t g = 0; g < nseg; ++g) {
    const uint32_t cnt = (uint32_t)std::min<uint64_t>(tie::dev::kTopB, k - off);
    tie::dev::pop_topb_kernel<<<1, 1024, 0, s>>>(Q->q, nb, Q->n_slots, cnt, Q->d_out_id + off,
                                                 Q->d_out_slot + off, Q->d_out_n + g,
                                                 Q->h_peek_key + off);
    off += cnt;
  }
  tie::capi::count_launch(nseg);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_error(e, "tie_queue_pop");
  std::vector<uint32_t> slots(k);
  for (uint64_t j = 0; j < k; ++j) slots[j] = Q->h_out_slot[j];
  std::vector<double> pk(k);
  for (uint64_t j = 0; j < k; ++j) {
    const uint64_t u = Q->h_peek_key[j];  // order_bits image of the popped key
    const uint64_t b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    std::memcpy(&pk[j], &b, 8);
  }
  // entry fields survive the pop on the device (only the key slot is killed)
  if (int rc = gather_entries(Q, slots, nullptr, nullptr, predicted, E, C, beta_at_update))
    return rc;
  std::vector<uint64_t> got;
  apply_pops(Q, 0, (uint32_t)k, got);
  for (uint64_t j = 0; j < k; ++j) {
    ids[j] = got[j];
    if (keys) keys[j] = pk[j];
  }
  *n_out = k;
  return TIE_OK;
}

// WaitingQueue::validate() (sched.cpp:116-123): host index consistency (the id -> slot map
// covers exactly the live slots) and every device block minimum equal to a rescan
int tie_queue_validate(tie_queue* Q, int* ok) {
  if (!Q || !ok) return set_error(TIE_EINVALID, "tie_queue: null argument");
  *ok = 0;
  uint64_t live = 0;
  for (uint64_t sl = 0; sl < Q->n_slots; ++sl) live += Q->alive[sl];
  if (live != Q->size || Q->slot_of.size() != Q->size) return TIE_OK;
  for (const auto& kv : Q->slot_of)
    if (kv.second >= Q->n_slots || !Q->alive[kv.second]) return TIE_OK;
  const uint32_t nb = (uint32_t)((Q->n_slots + tie::dev::kBlockSlots - 1) / tie::dev::kBlockSlots);
  if (nb) {
    cudaStream_t s = Q->ctx->stream;
    if (int rc = ensure_stage(Q, 1)) return rc;
    unsigned int bad = 0;
    cudaMemsetAsync(Q->d_blocks, 0, 4, s);
    tie::dev::validate_blocks_kernel<<<std::min<uint32_t>(nb, 4096), 256, 0, s>>>(
        Q->q, nb, Q->n_slots, Q->d_blocks);
    tie::capi::count_launch();
    cudaMemcpyAsync(&bad, Q->d_blocks, 4, cudaMemcpyDeviceToHost, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_error(e, "tie_queue_validate");
    if (bad) return TIE_OK;
  }
  *ok = 1;
  return TIE_OK;
}

// slot-count management: compact the live entries into `capacity` slots (>= waiting)
int tie_queue_reserve(tie_queue* Q, uint64_t capacity) {
  if (!Q) return set_error(TIE_EINVALID, "tie_queue: null queue");
  if (capacity < Q->size || capacity == 0 || capacity >= (1ull << 32))
    return set_error(TIE_EINVALID, "tie_queue_reserve: capacity must be in [waiting, 2^32)");
  return relayout(Q, capacity);
}

uint64_t tie_queue_capacity(const tie_queue* Q) { return Q ? Q->capacity : 0; }
uint64_t tie_queue_slots_used(const tie_queue* Q) { return Q ? Q->n_slots : 0; }

}  // extern "C"
