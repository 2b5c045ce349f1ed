// K2 -- dispatch order of a static waiting queue: stable LSD radix sort by (key, id).
//
// Reference: WaitingQueue (proj/src/sched.cpp:28-94) is a binary min-heap ordered by
// (key, req_id) (less(), sched.cpp:28-31); pushing n entries and popping until empty yields
// the lexicographic (key asc, id asc) order.  Here keys are mapped to u64 by the
// order-preserving IEEE transform (x >= 0: bits | 2^63, x < 0: ~bits; -0.0 folded onto +0.0
// because the heap compares keys with ==) and sorted by a stable LSD radix sort whose values
// start in ascending-id order -- which is exactly (key, id) order.
//
// Onesweep structure (one kernel per 8-bit digit pass):
//   * one histogram pass computes all 8 digit histograms up front (or the fused score kernel
//     accumulates them in its epilogue), a 1-CTA plan kernel turns them into per-pass bin
//     bases and a skip mask (passes whose digit is constant across all keys do nothing);
//   * each pass kernel takes tiles in launch order from an atomic counter, ranks its tile
//     stably in shared memory (warp match_any multi-split), publishes per-digit tile counts
//     and resolves its global digit offsets by decoupled look-back over predecessor tiles --
//     no separate upsweep / scan kernels, keys read once and written once per pass;
//   * digit runs are written out coalesced from the shared-memory-sorted tile; the LAST
//     active pass writes the u64 dispatch order (ids[value]) directly instead of keys+values.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "tie_internal.cuh"

namespace cg = cooperative_groups;

namespace tie {
namespace dev {

namespace {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kPasses = 64 / kRadixBits;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// look-back status word: [flag:2][count:62]
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kCountMask = (1ull << 62) - 1;
constexpr int kGroup = 16;  // tiles per second-level look-back group

// Phase timestamps of each pass's tiles (probe builds only: tools/rank_probe.cu).
#ifdef TIE_RANK_TRACE
__device__ unsigned long long g_rank_trace[8][8192][6];
#define RANK_TRACE(slot)                                                         \
  do {                                                                           \
    if (threadIdx.x == 0 && tile < 8192) {                                       \
      unsigned long long t_;                                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
      g_rank_trace[pass][tile][slot] = t_;                                       \
    }                                                                            \
  } while (0)
#else
#define RANK_TRACE(slot) \
  do {                   \
  } while (0)
#endif

struct Plan {
  uint32_t bin_base[kPasses][kBins];
  int active[kPasses];
  int sel[kPasses];    // buffer holding the input of pass p
  int first[kPasses];  // pass p is the first active one
  int last_active;     // index of the last active pass (-1: none)
  int final_sel;
  int any_active;
};

struct Work {
  uint64_t* k[2];
  uint32_t* v[2];
  uint32_t* hist;           // [kPasses][kBins]
  Plan* plan;
  uint64_t* status;         // [kPasses][tiles][kBins]
  uint64_t* gstatus;        // [kPasses][groups][kBins]  group aggregate / inclusive prefix
  uint64_t* gsum;           // [kPasses][groups][kBins]  (contributors << 40 | sum)
  uint32_t* gdone;          // [kPasses][groups]         members that have contributed
  uint32_t* tile_counter;   // [kPasses]
  int* flag;
  uint32_t tiles;
};

__device__ __forceinline__ uint32_t digit_of(uint64_t key, int pass) {
  return (uint32_t)(key >> (pass * kRadixBits)) & (kBins - 1);
}

__device__ __forceinline__ uint64_t order_bits(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 == +0.0 under the heap's comparison
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ void hist_flush(uint32_t (*h)[kBins], uint32_t* hist) {
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kBins; i += blockDim.x)
    if ((&h[0][0])[i]) atomicAdd(hist + i, (&h[0][0])[i]);
}

// key validation + transform (WaitingQueue::push rejects non-finite keys, sched.cpp:60) with
// the key range folded into mm (the bucket path's range)
__global__ void __launch_bounds__(256) keys_from_double_kernel(const double* __restrict__ key,
                                                               uint64_t n,
                                                               uint64_t* __restrict__ out,
                                                               unsigned long long* mm,
                                                               unsigned long long* err) {
  uint64_t lo = ~0ull, hi = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = key[i];
    uint64_t k;
    if (!isfinite(x)) {
      report(err, i, kKeyNotFinite);
      k = ~0ull;
    } else {
      k = order_bits(x);
    }
    out[i] = k;
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
  }
  key_range_flush(mm, lo, hi);
}

// copy u64 keys (ids, or pre-transformed keys) while accumulating the digit histograms
__global__ void __launch_bounds__(256) copy_hist_kernel(const uint64_t* __restrict__ in,
                                                        uint64_t n, uint64_t* __restrict__ out,
                                                        uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[kPasses][kBins];
  for (int i = threadIdx.x; i < kPasses * kBins; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = in[i];
    if (out) out[i] = k;
#pragma unroll
    for (int p = 0; p < kPasses; ++p) atomicAdd(&h[p][digit_of(k, p)], 1u);
  }
  hist_flush(h, hist);
}

// exclusive scan of 256 values held one per thread (blockDim == 256)
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* sh_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kWarps ? sh_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kWarps) sh_warp[lane] = w;
  }
  __syncthreads();
  return x + (warp ? sh_warp[warp - 1] : 0) - v;
}

__global__ void __launch_bounds__(kThreads) plan_kernel(const uint32_t* __restrict__ hist,
                                                        uint64_t n, Plan* plan) {
  __shared__ uint32_t sh_warp[kWarps];
  __shared__ int sh_active[kPasses];
  const int d = threadIdx.x;
  if (d < kPasses) sh_active[d] = 0;
  __syncthreads();
  for (int p = 0; p < kPasses; ++p) {
    const uint32_t c = hist[p * kBins + d];
    if ((uint64_t)c != n && c != 0) sh_active[p] = 1;  // more than one occupied digit
    plan->bin_base[p][d] = block_excl_scan_256(c, sh_warp);
    __syncthreads();
  }
  if (d == 0) {
    int cnt = 0, last = -1;
    for (int p = 0; p < kPasses; ++p) {
      plan->active[p] = sh_active[p];
      plan->sel[p] = cnt & 1;
      plan->first[p] = sh_active[p] && cnt == 0;
      if (sh_active[p]) last = p;
      cnt += sh_active[p];
    }
    plan->last_active = last;
    plan->final_sel = cnt & 1;
    plan->any_active = cnt > 0;
  }
}

template <int ITEMS>
struct PassSmem {
  uint64_t keys[kThreads * ITEMS];
  uint32_t vals[kThreads * ITEMS];
  uint32_t warp_hist[kWarps][kBins];
  uint32_t tile_excl[kBins];
  uint32_t global_off[kBins];
  uint32_t sh_warp[kWarps];
  uint32_t tile_hist[kBins];  // early digit counts of the tile (pads excluded)
  uint32_t tile;
};

// Batched walk over look-back status words [newest .. oldest] (stride `stride` words):
// accumulates published counts until an inclusive PREFIX is found.  Returns true when a
// PREFIX ended the walk; `pos` moves past every entry consumed; stops (without consuming)
// at the first unpublished entry or at `stop` (exclusive lower bound).
__device__ __forceinline__ bool walk(const volatile uint64_t* base, uint64_t stride,
                                     int64_t& pos, int64_t stop, uint64_t& excl) {
  constexpr int kBatch = 16;
  uint64_t s[kBatch];
#pragma unroll
  for (int u = 0; u < kBatch; ++u) s[u] = (pos - u > stop) ? base[(uint64_t)(pos - u) * stride] : 0;
  int used = 0;
  bool open = true, prefix = false;
#pragma unroll
  for (int u = 0; u < kBatch; ++u) {
    if (!open || pos - u <= stop) {
      open = false;
      continue;
    }
    const uint64_t f = s[u] & ~kCountMask;
    if (f == 0) {  // not published yet: resume here
      open = false;
      continue;
    }
    excl += s[u] & kCountMask;
    ++used;
    if (f == kFlagPrefix) {
      prefix = true;
      open = false;
    }
  }
  pos -= used;
  return prefix;
}

// Two-level decoupled look-back for digit d of `tile` (one thread per digit): publish() posts
// the tile's count early and folds it into its 16-tile group's aggregate; lookback() later
// walks (a) the preceding tiles of its own group and (b) the preceding groups' aggregates /
// inclusive prefixes.  When all tiles are resident at once (small n) this bounds every walk
// to ~3 batched L2 round trips instead of one batch per 16 predecessor tiles.
//
// Publish the tile's count for digit d: the tile status word (AGGREGATE, or PREFIX for
// tile 0) and the group aggregate.  The group aggregate needs no fences: one packed atomic
// carries (contributors << 40 | sum) and the last contributor reads the complete aggregate
// straight from the returned value.
__device__ __forceinline__ void publish(const Work& w, int pass, uint32_t tile, int d,
                                        uint32_t real) {
  const uint32_t groups = (w.tiles + kGroup - 1) / kGroup;
  const uint32_t q = tile / kGroup;
  volatile uint64_t* mine = w.status + (uint64_t)pass * w.tiles * kBins + (uint64_t)tile * kBins + d;
  *mine = (tile == 0 ? kFlagPrefix : kFlagAgg) | real;
  unsigned long long* gsum =
      (unsigned long long*)w.gsum + (uint64_t)pass * groups * kBins + (uint64_t)q * kBins + d;
  const uint32_t members = min((uint32_t)kGroup, w.tiles - q * kGroup);
  const unsigned long long old = atomicAdd(gsum, (1ull << 40) | real);
  if ((uint32_t)(old >> 40) == members - 1)
    atomicMax((unsigned long long*)(w.gstatus + (uint64_t)pass * groups * kBins +
                                    (uint64_t)q * kBins + d),
              (unsigned long long)(kFlagAgg | ((old & ((1ull << 40) - 1)) + real)));
}

__device__ __forceinline__ uint64_t lookback(const Work& w, int pass, uint32_t tile, int d,
                                             uint32_t real) {
  const uint32_t groups = (w.tiles + kGroup - 1) / kGroup;
  const uint32_t q = tile / kGroup;
  uint64_t* tstat = w.status + (uint64_t)pass * w.tiles * kBins;
  uint64_t* gstat = w.gstatus + (uint64_t)pass * groups * kBins;
  volatile uint64_t* mine = tstat + (uint64_t)tile * kBins + d;
  uint64_t excl = 0;
  bool done = tile == 0;
  int64_t pos = (int64_t)tile - 1;
  const int64_t gfirst = (int64_t)q * kGroup;
  while (!done && pos >= gfirst) done = walk(tstat + d, kBins, pos, gfirst - 1, excl);
  int64_t gpos = (int64_t)q - 1;
  while (!done && gpos >= 0) done = walk(gstat + d, kBins, gpos, -1, excl);
  if (tile > 0) *mine = kFlagPrefix | (excl + real);
  if (tile % kGroup == kGroup - 1 || tile == w.tiles - 1)
    atomicMax((unsigned long long*)(gstat + (uint64_t)q * kBins + d),
              (unsigned long long)(kFlagPrefix | (excl + real)));
  return excl;
}

// One digit pass.  `order`: when non-null and this is the last active pass, write the
// dispatch order (ids[value], or value) instead of keys + values.
template <int ITEMS>
__global__ void __launch_bounds__(kThreads, 3) onesweep_kernel(Work w, uint64_t n, int pass,
                                                            int explicit_vals,
                                                            const uint64_t* __restrict__ ids,
                                                            uint64_t* __restrict__ order) {
  const Plan* plan = w.plan;
  if (!plan->active[pass]) return;
  constexpr int kTileKeys = kThreads * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem<ITEMS>& sm = *reinterpret_cast<PassSmem<ITEMS>*>(smem_raw);
  const int src = plan->sel[pass];
  const uint64_t* __restrict__ kin = src ? w.k[1] : w.k[0];
  const uint32_t* __restrict__ vin = src ? w.v[1] : w.v[0];
  uint64_t* __restrict__ kout = src ? w.k[0] : w.k[1];
  uint32_t* __restrict__ vout = src ? w.v[0] : w.v[1];
  const bool implicit = plan->first[pass] && !explicit_vals;
  const bool to_order = order != nullptr && plan->last_active == pass;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kBins; i += kThreads) (&sm.warp_hist[0][0])[i] = 0;
  if (threadIdx.x == 0) sm.tile = atomicAdd(w.tile_counter + pass, 1u);  // launch-order tiles
  __syncthreads();
  const uint32_t tile = sm.tile;
  RANK_TRACE(0);
  const uint64_t tile_base = (uint64_t)tile * kTileKeys;
  const uint64_t left = n - tile_base;
  const uint32_t valid = left < (uint64_t)kTileKeys ? (uint32_t)left : (uint32_t)kTileKeys;
  const unsigned lt_mask = (1u << lane) - 1u;

  uint64_t key[ITEMS];
  uint32_t rank[ITEMS];
  // warp w owns slots [w*32*ITEMS, (w+1)*32*ITEMS); round j, lane l -> slot w*32*ITEMS +
  // j*32 + l, so (round, lane) order is index order and the multi-split below is stable.
  // Values are not held in registers: they go straight to their ranked smem slot below.
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t q = warp * (ITEMS * 32) + j * 32 + lane;
    key[j] = q < valid ? kin[tile_base + q] : ~0ull;  // pads sort last, never written out
  }
  // early counts: a plain shared-memory histogram of the tile's digits is published before
  // the (slower) stable ranking, so successor tiles' look-backs resolve while this tile ranks
  const int d = threadIdx.x;
  sm.tile_hist[d] = 0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t q = warp * (ITEMS * 32) + j * 32 + lane;
    if (q < valid) atomicAdd(&sm.tile_hist[digit_of(key[j], pass)], 1u);
  }
  __syncthreads();
  const uint32_t real = sm.tile_hist[d];
  publish(w, pass, tile, d, real);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t dg = digit_of(key[j], pass);
    // lanes holding the same digit: AND of the 8 per-bit ballots (warp multi-split); cheaper
    // than MATCH.ANY on sm_100
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
      const unsigned bal = __ballot_sync(0xffffffffu, (dg >> b) & 1u);
      peers &= ((dg >> b) & 1u) ? bal : ~bal;
    }
    const uint32_t before = sm.warp_hist[warp][dg];
    __syncwarp();
    if ((peers & lt_mask) == 0) sm.warp_hist[warp][dg] = before + __popc(peers);
    __syncwarp();
    rank[j] = before + __popc(peers & lt_mask);
  }
  __syncthreads();
  RANK_TRACE(1);
  uint32_t count = 0;
#pragma unroll
  for (int q = 0; q < kWarps; ++q) {
    const uint32_t c = sm.warp_hist[q][d];
    sm.warp_hist[q][d] = count;
    count += c;
  }
  const uint64_t excl = lookback(w, pass, tile, d, real);
  sm.global_off[d] = plan->bin_base[pass][d] + (uint32_t)excl;
  sm.tile_excl[d] = block_excl_scan_256(count, sm.sh_warp);
  __syncthreads();
  RANK_TRACE(2);
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const uint32_t dd = digit_of(key[j], pass);
    const uint32_t pos = sm.tile_excl[dd] + sm.warp_hist[warp][dd] + rank[j];
    const uint32_t q = warp * (ITEMS * 32) + j * 32 + lane;
    sm.keys[pos] = key[j];
    sm.vals[pos] = implicit ? (uint32_t)(tile_base + q) : (q < valid ? vin[tile_base + q] : 0u);
  }
  __syncthreads();
  RANK_TRACE(3);
  if (to_order) {
    for (uint32_t q = threadIdx.x; q < valid; q += kThreads) {
      const uint32_t dd = digit_of(sm.keys[q], pass);
      const uint64_t g = (uint64_t)sm.global_off[dd] + (q - sm.tile_excl[dd]);
      const uint32_t v = sm.vals[q];
      order[g] = ids ? ids[v] : (uint64_t)v;
    }
  } else {
    for (uint32_t q = threadIdx.x; q < valid; q += kThreads) {
      const uint64_t k = sm.keys[q];
      const uint32_t dd = digit_of(k, pass);
      const uint64_t g = (uint64_t)sm.global_off[dd] + (q - sm.tile_excl[dd]);
      kout[g] = k;
      vout[g] = sm.vals[q];
    }
  }
#ifdef TIE_RANK_TRACE
  __syncthreads();
  RANK_TRACE(4);
#endif
}

// degenerate case (no active pass: every key identical): the order is the input order
__global__ void identity_order_kernel(Work w, uint64_t n, const uint64_t* __restrict__ ids,
                                      uint64_t* __restrict__ order, int explicit_vals) {
  const Plan* plan = w.plan;
  if (plan->any_active) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t idx = explicit_vals ? w.v[0][i] : i;
    order[i] = ids ? ids[idx] : idx;
  }
}

// ids strictly ascending?  (fast path: values can start as the index)
__global__ void ids_sorted_kernel(const uint64_t* __restrict__ ids, uint64_t n, int* flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += stride)
    if (ids[i] >= ids[i + 1]) {
      *flag = 1;
      return;
    }
}

// After the (id, index) sort: detect duplicate ids and stage (key[perm], perm) as the
// explicit-value input of the key sort.
__global__ void gather_by_id_kernel(Work w, uint64_t n, const uint64_t* __restrict__ tkeys,
                                    uint64_t* __restrict__ kdst, uint32_t* __restrict__ vdst,
                                    unsigned long long* err) {
  const Plan* plan = w.plan;
  const uint64_t* sid = plan->final_sel ? w.k[1] : w.k[0];
  const uint32_t* perm = plan->final_sel ? w.v[1] : w.v[0];
  const bool identity = !plan->any_active;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const uint32_t p = identity ? (uint32_t)j : perm[j];
    if (j > 0 && sid[j] == sid[j - 1]) report(err, p, kDuplicateId);
    kdst[j] = tkeys[p];
    vdst[j] = p;
  }
}

// ====================================================================== bucket path
// Default dispatch-order sort (K2).  The producer folds the key range
// [kmin, kmax] (key_range_flush); keys are then bucketed by their top bits above kmin --
// nb = 2^nb_log2 ~ n/8 buckets, contiguous in the output -- and each bucket is ordered in
// shared memory:
//   count   : per-bucket counts (global atomics, one per key)
//   scan_a/b: exclusive prefix of the counts (bucket bases) + segment starts: segment i
//             begins at the first bucket boundary >= i*kSegStep, so a segment holds
//             < kSegStep + (largest bucket) <= kSegCap keys
//   scatter : (key, index) into its bucket's slot range (order within a bucket arbitrary)
//   local   : one CTA per segment stages it in shared memory; each key's final position is
//             its bucket base + #{(key', index') < (key, index) in the bucket}, i.e. the
//             (key, id) heap order with ties broken by index (== id order).
// 4 passes over the keys instead of 7-8 radix passes.  A bucket larger than kMaxBucket
// (massive score ties) makes the local kernel tail-launch the stable LSD path above from the
// device instead (CUDA dynamic parallelism), so the order stays exact for any input.
constexpr uint32_t kSegCap = 4096;
constexpr uint32_t kSegStep = kSegCap / 2;
constexpr uint32_t kMaxBucket = kSegCap - kSegStep;
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 4;
constexpr uint32_t kScanChunk = kScanThreads * kScanPer;
constexpr uint32_t kMinBucketsLog2 = 12;  // nb >= kScanChunk
constexpr uint32_t kMaxBucketsLog2 = 24;
constexpr int kLocalThreads = 256;

struct Bucket {
  const uint64_t* keys;    // [n] order-preserving keys
  uint64_t* tk;            // [n] keys grouped by bucket (aliases the LSD ping-pong buffer)
  uint32_t* tv;            // [n] their indices
  uint32_t* count;         // [nb]
  uint32_t* base;          // [nb + 1] exclusive prefix of count
  uint32_t* cursor;        // [nb]
  uint32_t* partial;       // [chunks]
  uint32_t* seg;           // [nseg + 1]
  unsigned long long* mm;  // [2]: max(~key), max(key)
  int* overflow;
  uint32_t nb_log2, nb, chunks, nseg;
};

struct KeyRange {
  uint64_t kmin;
  uint32_t shift;
};

// keys in [kmin, kmax] -> B-bit bucket (k - kmin) >> shift
__device__ __forceinline__ KeyRange key_range(const unsigned long long* mm, uint32_t B) {
  const uint64_t kmin = ~(uint64_t)mm[0];
  const uint64_t span = (uint64_t)mm[1] - kmin;
  const uint32_t bits = span ? 64u - (uint32_t)__clzll((long long)span) : 0u;
  return {kmin, bits > B ? bits - B : 0u};
}

__device__ __forceinline__ KeyRange key_range(const Bucket& b) { return key_range(b.mm, b.nb_log2); }

__device__ __forceinline__ uint32_t bucket_of(const KeyRange& r, uint64_t k) {
  return (uint32_t)((k - r.kmin) >> r.shift);  // span >> shift < nb
}

// count / scatter: each thread takes kStreamItems keys of a 256*kStreamItems tile (coalesced,
// all loads issued before the first atomic, so one L2 round trip is paid per batch)
constexpr int kStreamItems = 4;
constexpr uint64_t kStreamTile = 256 * kStreamItems;

__global__ void __launch_bounds__(256) bucket_count_kernel(Bucket b, uint64_t n) {
  const KeyRange r = key_range(b);
  const uint64_t t0 = (uint64_t)blockIdx.x * kStreamTile + threadIdx.x;
  uint64_t k[kStreamItems];
#pragma unroll
  for (int j = 0; j < kStreamItems; ++j) {
    const uint64_t i = t0 + (uint64_t)j * 256;
    k[j] = i < n ? b.keys[i] : 0;
  }
#pragma unroll
  for (int j = 0; j < kStreamItems; ++j)
    if (t0 + (uint64_t)j * 256 < n) atomicAdd(b.count + bucket_of(r, k[j]), 1u);
}

// block-wide reduction / exclusive scan over kScanThreads threads
__device__ __forceinline__ uint32_t scan_block_sum(uint32_t v, uint32_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  uint32_t t = lane < (kScanThreads / 32) ? sh[lane] : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  return t;
}

__device__ __forceinline__ uint32_t scan_block_excl(uint32_t v, uint32_t* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sh[lane] = w;
  }
  __syncthreads();
  const uint32_t r = x - v + (warp ? sh[warp - 1] : 0u);
  __syncthreads();
  return r;
}

template <int kT>
__device__ __forceinline__ uint32_t block_excl_scan_t(uint32_t v, uint32_t* sh) {
  constexpr int kW = kT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kW ? sh[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kW) sh[lane] = w;
  }
  __syncthreads();
  const uint32_t r = x - v + (warp ? sh[warp - 1] : 0u);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) bucket_scan_a_kernel(Bucket b) {
  __shared__ uint32_t sh[32];
  const uint32_t i0 = blockIdx.x * kScanChunk + threadIdx.x * kScanPer;
  const uint4 q = *reinterpret_cast<const uint4*>(b.count + i0);
  const uint32_t t = scan_block_sum(q.x + q.y + q.z + q.w, sh);
  if (threadIdx.x == 0) b.partial[blockIdx.x] = t;
}

// bucket boundary `v` (= base of some bucket) preceded by boundary `vprev`: it starts every
// segment i with vprev < i*kSegStep <= v.  first: the boundary of bucket 0 (vprev = -1).
__device__ __forceinline__ void claim_segments(const Bucket& b, uint32_t vprev, uint32_t v,
                                               bool first) {
  const uint32_t lo = first ? 0u : vprev / kSegStep + 1u;
  const uint32_t hi = min(v / kSegStep, b.nseg - 1u);
  if (hi > lo + 1u) {  // a bucket spanning > kSegStep keys: the local sort cannot hold it
    *b.overflow = 1;
    return;
  }
  for (uint32_t i = lo; i <= hi; ++i) b.seg[i] = v;
}

__global__ void __launch_bounds__(kScanThreads) bucket_scan_b_kernel(Bucket b, uint64_t n) {
  __shared__ uint32_t sh[32];
  const uint32_t c = blockIdx.x;
  uint32_t acc = 0;
  for (uint32_t j = threadIdx.x; j < c; j += kScanThreads) acc += b.partial[j];
  const uint32_t prefix = scan_block_sum(acc, sh);
  const uint32_t i0 = c * kScanChunk + threadIdx.x * kScanPer;
  const uint4 q = *reinterpret_cast<const uint4*>(b.count + i0);
  const uint32_t cnt[4] = {q.x, q.y, q.z, q.w};
  uint32_t v = prefix + scan_block_excl(q.x + q.y + q.z + q.w, sh);
  uint32_t vprev = i0 ? v - b.count[i0 - 1] : 0u;
#pragma unroll
  for (int j = 0; j < kScanPer; ++j) {
    const uint32_t bi = i0 + j;
    b.base[bi] = v;
    b.cursor[bi] = v;
    if (cnt[j] > kMaxBucket) *b.overflow = 1;
    if (bi == 0 || v != vprev) claim_segments(b, vprev, v, bi == 0);
    vprev = v;
    v += cnt[j];
  }
  if (i0 + kScanPer == b.nb) {  // the sentinel boundary (v == n)
    b.base[b.nb] = v;
    if (v != vprev) claim_segments(b, vprev, v, false);
    b.seg[b.nseg] = (uint32_t)n;
  }
}

__global__ void __launch_bounds__(256) bucket_scatter_kernel(Bucket b, uint64_t n) {
  if (*(volatile int*)b.overflow) return;
  const KeyRange r = key_range(b);
  const uint64_t t0 = (uint64_t)blockIdx.x * kStreamTile + threadIdx.x;
  uint64_t k[kStreamItems];
  uint32_t p[kStreamItems];
#pragma unroll
  for (int j = 0; j < kStreamItems; ++j) {
    const uint64_t i = t0 + (uint64_t)j * 256;
    k[j] = i < n ? b.keys[i] : 0;
  }
#pragma unroll
  for (int j = 0; j < kStreamItems; ++j)
    if (t0 + (uint64_t)j * 256 < n) p[j] = atomicAdd(b.cursor + bucket_of(r, k[j]), 1u);
#pragma unroll
  for (int j = 0; j < kStreamItems; ++j) {
    const uint64_t i = t0 + (uint64_t)j * 256;
    if (i < n) {
      b.tk[p[j]] = k[j];
      b.tv[p[j]] = (uint32_t)i;
    }
  }
}

__global__ void zero_kernel(uint4* p, uint64_t n16) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    p[i] = make_uint4(0, 0, 0, 0);
}

struct Fallback {
  Work w;           // LSD state (its metadata zeroed here, on the device)
  uint4* meta;
  uint64_t meta16;
  unsigned grid;    // grid of the streaming helper kernels
};

// The stable LSD path (histograms, plan, digit passes, identity case) as device-side tail
// launches: they run in order after the launching grid, before anything queued behind it.
__device__ void lsd_tail_launch(const Fallback& f, const uint64_t* keys, uint64_t n,
                                const uint64_t* ids, uint64_t* order) {
  zero_kernel<<<f.grid, 256, 0, cudaStreamTailLaunch>>>(f.meta, f.meta16);
  copy_hist_kernel<<<f.grid, 256, 0, cudaStreamTailLaunch>>>(
      keys, n, keys == f.w.k[0] ? nullptr : f.w.k[0], f.w.hist);
  plan_kernel<<<1, kThreads, 0, cudaStreamTailLaunch>>>(f.w.hist, n, f.w.plan);
  for (int p = 0; p < kPasses; ++p)
    onesweep_kernel<16><<<f.w.tiles, kThreads, sizeof(PassSmem<16>), cudaStreamTailLaunch>>>(
        f.w, n, p, 0, ids, order);
  identity_order_kernel<<<f.grid, 256, 0, cudaStreamTailLaunch>>>(f.w, n, ids, order, 0);
}

__global__ void __launch_bounds__(kLocalThreads, 4) bucket_local_kernel(Bucket b, uint64_t n,
                                                                     const uint64_t* __restrict__ ids,
                                                                     uint64_t* __restrict__ order,
                                                                     Fallback f) {
  if (*(volatile int*)b.overflow) {
    if (blockIdx.x == 0 && threadIdx.x == 0) lsd_tail_launch(f, b.keys, n, ids, order);
    return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kSegCap);
  constexpr int kItems = kSegCap / kLocalThreads;
  const uint32_t s0 = b.seg[blockIdx.x], s1 = b.seg[blockIdx.x + 1];
  const uint32_t m = s1 - s0;  // <= kSegCap
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t j = threadIdx.x + it * kLocalThreads;
    if (j < m) {
      sk[j] = b.tk[s0 + j];
      sv[j] = b.tv[s0 + j];
    }
  }
  __syncthreads();
  const KeyRange r = key_range(b);
  // every item's bucket bounds fetched up front (independent L2 loads, one round trip)
  uint32_t lo[kItems], hi[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t j = threadIdx.x + it * kLocalThreads;
    if (j < m) {
      const uint32_t bk = bucket_of(r, sk[j]);
      lo[it] = b.base[bk];
      hi[it] = b.base[bk + 1];
    }
  }
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t j = threadIdx.x + it * kLocalThreads;
    if (j < m) {
      const uint64_t k = sk[j];
      const uint32_t v = sv[j];
      uint32_t rank = 0;
      for (uint32_t q = lo[it] - s0; q < hi[it] - s0; ++q) {
        const uint64_t kq = sk[q];
        rank += (kq < k) | ((kq == k) & (sv[q] < v));
      }
      order[lo[it] + rank] = ids ? ids[v] : (uint64_t)v;
    }
  }
}

// ====================================================================== partition path
// Default for n <= kPartMaxN (the config-2 queue): the same (key, id) order with no per-key
// global atomics.  Keys map to a B-bit bucket f = (k - kmin) >> shift, B = p_log2 + fine_log2;
// the top p_log2 bits pick one of P partitions (~1K keys each), the rest a fine bucket.
//   count  : persistent CTAs, each a contiguous chunk: shared-memory partition histogram,
//            then ONE atomicAdd per (CTA, partition) reserving the CTA's slot range
//   scan   : partition bases (1 CTA); a partition above kPartCap -> device LSD fallback
//   scatter: the CTA's keys into its reserved ranges (shared-memory cursors)
//   sort   : one CTA per partition: fine-bucket counting sort in shared memory, then each
//            key's rank inside its fine bucket (~1-2 keys) by (key, index) -> dispatch order
constexpr uint32_t kPartCap = 4096;
constexpr uint64_t kPartMaxN = 1ull << 21;
constexpr uint32_t kPartMaxP = 2048;
constexpr uint32_t kPartMaxFineLog2 = 10;
constexpr int kPartThreads = 256;
constexpr int kFusedThreadsFwd = 512;  // = kFusedThreads (the group sorts split it)

struct Part {
  const uint64_t* keys;
  uint64_t* tk;  // [n] keys grouped by partition (aliases the LSD ping-pong buffer)
  uint32_t* tv;
  uint32_t* pcount;   // [P]   zeroed per sort
  uint32_t* pbase;    // [P + 1]
  uint32_t* cta_off;  // [ctas][P]  a CTA's slot offset inside each partition
  unsigned long long* mm;
  int* overflow;
  uint32_t p_log2, P, fine_log2, ctas;
  uint64_t chunk;
  uint32_t low_bits;    // bits below the level-1 partition index (fine, or level-2 + fine)
  uint32_t total_bits;  // B: bucket bits of (k - kmin) >> shift
  uint32_t cap1;        // level-1 partition capacity (kPartCap; unbounded with level 2)
  uint32_t local_scatter;  // fused kernel: group the chunk by partition before scattering
  // level 2 (two-level path): P2 sub-partitions per level-1 partition, regrouped keys
  uint32_t p2_log2;
  uint64_t* tk2;
  uint32_t* tv2;
};

__device__ __forceinline__ uint32_t part_bucket(const Part& q, const KeyRange& r, uint64_t k) {
  return (uint32_t)((k - r.kmin) >> r.shift);
}

__global__ void __launch_bounds__(kPartThreads) part_count_kernel(Part q, uint64_t n) {
  __shared__ uint32_t h[kPartMaxP];
  for (uint32_t p = threadIdx.x; p < q.P; p += kPartThreads) h[p] = 0;
  __syncthreads();
  const KeyRange r = key_range(q.mm, q.total_bits);
  const uint64_t lo = (uint64_t)blockIdx.x * q.chunk;
  const uint64_t hi = min(n, lo + q.chunk);
  uint64_t i = lo + threadIdx.x;
  for (; i + 3 * kPartThreads < hi; i += 4 * kPartThreads) {
    uint64_t k[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = q.keys[i + u * kPartThreads];
#pragma unroll
    for (int u = 0; u < 4; ++u) atomicAdd(&h[part_bucket(q, r, k[u]) >> q.low_bits], 1u);
  }
  for (; i < hi; i += kPartThreads) atomicAdd(&h[part_bucket(q, r, q.keys[i]) >> q.low_bits], 1u);
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < q.P; p += kPartThreads) {
    const uint32_t c = h[p];
    q.cta_off[(uint64_t)blockIdx.x * q.P + p] = c ? atomicAdd(q.pcount + p, c) : 0u;
  }
  // the last CTA to finish turns the partition counts into bases (no separate scan launch)
  __shared__ uint32_t ticket;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(q.pcount + q.P, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();
  constexpr int kPer = kPartMaxP / kPartThreads;
  __shared__ uint32_t sh[32];
  uint32_t c[kPer], t = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint32_t p = threadIdx.x * kPer + j;
    c[j] = p < q.P ? __ldcg(q.pcount + p) : 0u;
    t += c[j];
    if (c[j] > q.cap1) *q.overflow = 1;
  }
  uint32_t v = block_excl_scan_t<kPartThreads>(t, sh);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint32_t p = threadIdx.x * kPer + j;
    if (p < q.P) q.pbase[p] = v;
    v += c[j];
  }
  if (threadIdx.x == 0) q.pbase[q.P] = (uint32_t)n;
}

__global__ void __launch_bounds__(kPartThreads) part_scatter_kernel(Part q, uint64_t n) {
  if (*(volatile int*)q.overflow) return;
  __shared__ uint32_t cur[kPartMaxP];
  for (uint32_t p = threadIdx.x; p < q.P; p += kPartThreads)
    cur[p] = q.pbase[p] + q.cta_off[(uint64_t)blockIdx.x * q.P + p];
  __syncthreads();
  const KeyRange r = key_range(q.mm, q.total_bits);
  const uint64_t lo = (uint64_t)blockIdx.x * q.chunk;
  const uint64_t hi = min(n, lo + q.chunk);
  uint64_t i = lo + threadIdx.x;
  for (; i + 3 * kPartThreads < hi; i += 4 * kPartThreads) {
    uint64_t k[4];
    uint32_t pos[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = q.keys[i + u * kPartThreads];
#pragma unroll
    for (int u = 0; u < 4; ++u) pos[u] = atomicAdd(&cur[part_bucket(q, r, k[u]) >> q.low_bits], 1u);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      q.tk[pos[u]] = k[u];
      q.tv[pos[u]] = (uint32_t)(i + u * kPartThreads);
    }
  }
  for (; i < hi; i += kPartThreads) {
    const uint64_t k = q.keys[i];
    const uint32_t pos = atomicAdd(&cur[part_bucket(q, r, k) >> q.low_bits], 1u);
    q.tk[pos] = k;
    q.tv[pos] = (uint32_t)i;
  }
}

// The level-1 scatter for large n (two-level path): the CTA walks its chunk in tiles of
// kTile keys, groups each tile by partition in shared memory (local counts, scan, cursors:
// only a u16 local order is kept, the keys are re-read from L2) and writes every partition's
// run of the tile with consecutive threads.  With ~16 keys per partition per 32k tile a
// warp's 32 stores touch ~2 runs (pages, sectors) instead of 32 scattered ones: at 64M keys
// the per-key scattered stores had 3x DRAM read / write amplification and TLB-bound latency
// (ncu: long scoreboard 276 cycles per issue).
template <uint32_t kTile>
constexpr size_t scat_smem() { return (size_t)kTile * 2 + 3 * 4 * kPartMaxP; }
constexpr int kScatThreads = 512;

template <uint32_t kTile>
__global__ void __launch_bounds__(kScatThreads) part_scatter_tiled_kernel(Part q, uint64_t n) {
  __shared__ int skip;
  if (threadIdx.x == 0) skip = *(volatile int*)q.overflow;
  __syncthreads();
  if (skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* cur = reinterpret_cast<uint32_t*>(smem_raw);           // [P] counts -> cursors
  uint32_t* lb = cur + kPartMaxP;                                  // [P] local bases
  uint32_t* gcur = lb + kPartMaxP;                                 // [P] global cursors
  uint16_t* srt = reinterpret_cast<uint16_t*>(gcur + kPartMaxP);   // [tile] local order
  __shared__ uint32_t sh[32];
  const uint32_t P = q.P;
  for (uint32_t p = threadIdx.x; p < P; p += kScatThreads)
    gcur[p] = q.pbase[p] + q.cta_off[(uint64_t)blockIdx.x * P + p];
  const KeyRange r = key_range(q.mm, q.total_bits);
  const uint64_t lo = (uint64_t)blockIdx.x * q.chunk;
  const uint64_t hi = min(n, lo + q.chunk);
  constexpr int kU = 8;  // loads in flight per thread
  for (uint64_t t0 = lo; t0 < hi; t0 += kTile) {
    const uint32_t tn = (uint32_t)min((uint64_t)kTile, hi - t0);
    const uint64_t* tk = q.keys + t0;
    for (uint32_t p = threadIdx.x; p < P; p += kScatThreads) cur[p] = 0;
    __syncthreads();
    for (uint32_t j0 = threadIdx.x; j0 < tn; j0 += kU * kScatThreads) {  // counts
      uint64_t kk[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t j = j0 + u * kScatThreads;
        kk[u] = j < tn ? tk[j] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (j0 + u * kScatThreads < tn) atomicAdd(&cur[part_bucket(q, r, kk[u]) >> q.low_bits], 1u);
    }
    __syncthreads();
    {
      constexpr int kPer = kPartMaxP / kScatThreads;
      uint32_t c[kPer], t = 0;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const uint32_t p = threadIdx.x * kPer + u;
        c[u] = p < P ? cur[p] : 0u;
        t += c[u];
      }
      uint32_t v = block_excl_scan_t<kScatThreads>(t, sh);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const uint32_t p = threadIdx.x * kPer + u;
        if (p < P) {
          lb[p] = v;
          cur[p] = v;
        }
        v += c[u];
      }
    }
    __syncthreads();
    for (uint32_t j0 = threadIdx.x; j0 < tn; j0 += kU * kScatThreads) {  // local order
      uint64_t kk[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t j = j0 + u * kScatThreads;
        kk[u] = j < tn ? tk[j] : 0ull;  // L2-resident: read a moment ago
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t j = j0 + u * kScatThreads;
        if (j < tn) srt[atomicAdd(&cur[part_bucket(q, r, kk[u]) >> q.low_bits], 1u)] = (uint16_t)j;
      }
    }
    __syncthreads();
    for (uint32_t t1 = threadIdx.x; t1 < tn; t1 += kU * kScatThreads) {  // partition runs
      uint32_t jj[kU];
      uint64_t kk[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t t = t1 + u * kScatThreads;
        jj[u] = t < tn ? srt[t] : 0u;
        kk[u] = t < tn ? tk[jj[u]] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t t = t1 + u * kScatThreads;
        if (t < tn) {
          const uint32_t p = part_bucket(q, r, kk[u]) >> q.low_bits;
          const uint32_t pos = gcur[p] + (t - lb[p]);
          q.tk[pos] = kk[u];
          q.tv[pos] = (uint32_t)(t0 + jj[u]);
        }
      }
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < P; p += kScatThreads) gcur[p] += cur[p] - lb[p];
  }
}

// Sort partition p's m keys (already grouped at tk/tv[s0..s0+m)) and write its slice of the
// dispatch order: fine-bucket counting sort in shared memory, each key ranked inside its fine
// bucket (~1-2 keys) by (key, index), values placed in order, written out coalesced.
template <int kT>
__device__ __forceinline__ void sort_partition(const Part& q, uint32_t s0, uint32_t m,
                                               const uint64_t* __restrict__ ids,
                                               uint64_t* __restrict__ order,
                                               unsigned char* smem_raw) {
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kPartCap);
  uint16_t* sf = reinterpret_cast<uint16_t*>(sv + kPartCap);    // fine bucket of key j
  uint16_t* perm = sf + kPartCap;                                // slot -> key j
  uint32_t* fb = reinterpret_cast<uint32_t*>(perm + kPartCap);   // [nf + 1] fine bases
  uint32_t* fc = fb + (1u << kPartMaxFineLog2) + 1;              // [nf] counts / cursors
  __shared__ uint32_t sh[32];
  const uint32_t nf = 1u << q.fine_log2, fmask = nf - 1u;
  for (uint32_t j = threadIdx.x; j < nf; j += kT) fc[j] = 0;
  __syncthreads();
  const KeyRange r = key_range(q.mm, q.total_bits);
  constexpr int kLd = 4;  // (key, index) loads in flight per thread before the first use
  for (uint32_t j0 = threadIdx.x; j0 < m; j0 += kLd * kT) {
    uint64_t kk[kLd];
    uint32_t vv[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kT;
      kk[u] = j < m ? q.tk[s0 + j] : 0ull;
      vv[u] = j < m ? q.tv[s0 + j] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kT;
      if (j < m) {
        sk[j] = kk[u];
        sv[j] = vv[u];
        const uint32_t fine = part_bucket(q, r, kk[u]) & fmask;
        sf[j] = (uint16_t)fine;
        atomicAdd(&fc[fine], 1u);
      }
    }
  }
  __syncthreads();
  {  // exclusive scan of the nf (<= 1024) fine counts, 4 per thread
    constexpr int kPer = (1 << kPartMaxFineLog2) / kT;
    uint32_t c[kPer], t = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t j = threadIdx.x * kPer + u;
      c[u] = j < nf ? fc[j] : 0u;
      t += c[u];
    }
    uint32_t v = block_excl_scan_t<kT>(t, sh);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t j = threadIdx.x * kPer + u;
      if (j < nf) {
        fb[j] = v;
        fc[j] = v;
      }
      v += c[u];
    }
    if (threadIdx.x == 0) fb[nf] = m;
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < m; j += kT) perm[atomicAdd(&fc[sf[j]], 1u)] = (uint16_t)j;
  __syncthreads();
  uint16_t* spos = sf;  // a key's final position in the partition replaces its fine bucket
  for (uint32_t j = threadIdx.x; j < m; j += kT) {
    const uint64_t k = sk[j];
    const uint32_t v = sv[j], fine = sf[j];
    const uint32_t lo = fb[fine], hi = fb[fine + 1];
    uint32_t below = 0;
    for (uint32_t s = lo; s < hi; ++s) {
      const uint32_t o = perm[s];
      const uint64_t kq = sk[o];
      below += (kq < k || (kq == k && sv[o] < v)) ? 1u : 0u;
    }
    spos[j] = (uint16_t)(lo + below);
  }
  __syncthreads();
  // place the values in partition order (the keys are no longer needed), then write the
  // partition's slice of the dispatch order out coalesced -- also when `order` is mapped
  // pinned host memory (the host API's zero-copy output)
  uint32_t* outv = reinterpret_cast<uint32_t*>(sk);
  for (uint32_t j = threadIdx.x; j < m; j += kT) outv[spos[j]] = sv[j];
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < m; p += kT) {
    const uint32_t v = outv[p];
    order[s0 + p] = ids ? ids[v] : (uint64_t)v;
  }
}

// Group-parallel partition sorts (level 2 of the two-level path).  A sub-partition holds
// ~0.5-1.5k keys, and sorting one with the whole 512-thread CTA is a chain of barriers over
// loops of 1-3 iterations.  Instead the CTA splits into kGroups groups, each sorting its OWN
// sub-partition with its own named barrier (bar.sync id, n) in its own shared-memory slice
// -- kGroups sub-partitions in flight per CTA; those above kGrpCap keys are sorted CTA-wide
// afterwards.  The fine buckets are the top kGrpFineLog2 fine bits (~2-4 keys per bucket).
// Same-box A/B on B200 (64M keys, level 2): 1.77 ms vs 1.87 ms CTA-wide; in the one-level
// fused kernel (1M keys) the groups were slower (91-94 vs 85 us per step), so it keeps the
// CTA-wide sorts.
#ifndef TIE_GRP_GROUPS
#define TIE_GRP_GROUPS 4
#endif
#ifndef TIE_GRP_CAP
#define TIE_GRP_CAP 1408
#endif
#ifndef TIE_GRP_FINE_LOG2
#define TIE_GRP_FINE_LOG2 8
#endif
constexpr int kGroups = TIE_GRP_GROUPS;
constexpr uint32_t kGrpCap = TIE_GRP_CAP;
constexpr uint32_t kGrpFineLog2 = TIE_GRP_FINE_LOG2;
constexpr uint32_t kGrpFine = 1u << kGrpFineLog2;
constexpr size_t kGrpBytes =
    ((size_t)kGrpCap * (8 + 4 + 2 + 2) + 4 * (2 * kGrpFine + 1) + 15) & ~(size_t)15;

template <int kN>
__device__ __forceinline__ void grp_bar(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kN) : "memory");
}

// exclusive scan over the group's kN threads (kN / 32 <= 32 warps)
template <int kN>
__device__ __forceinline__ uint32_t grp_excl_scan(uint32_t v, uint32_t* sh, int bar, int gtid) {
  const int lane = gtid & 31, warp = gtid >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  grp_bar<kN>(bar);
  uint32_t pre = 0;
  for (int w = 0; w < warp; ++w) pre += sh[w];
  grp_bar<kN>(bar);  // sh is reused by the next scan
  return x - v + pre;
}

template <int kN>
__device__ __forceinline__ void sort_partition_grp(const Part& q, uint32_t s0, uint32_t m,
                                                   const uint64_t* __restrict__ ids,
                                                   uint64_t* __restrict__ order,
                                                   unsigned char* gmem, uint32_t* sh, int bar,
                                                   int gtid) {
  uint64_t* sk = reinterpret_cast<uint64_t*>(gmem);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + kGrpCap);
  uint16_t* sf = reinterpret_cast<uint16_t*>(sv + kGrpCap);
  uint16_t* perm = sf + kGrpCap;
  uint32_t* fb = reinterpret_cast<uint32_t*>(perm + kGrpCap);  // [nf + 1]
  uint32_t* fc = fb + kGrpFine + 1;                             // [nf]
  const uint32_t flog = min(q.fine_log2, kGrpFineLog2);
  const uint32_t fshift = q.fine_log2 - flog, nf = 1u << flog;
  const uint32_t fmask = (1u << q.fine_log2) - 1u;
  for (uint32_t j = gtid; j < nf; j += kN) fc[j] = 0;
  grp_bar<kN>(bar);
  const KeyRange r = key_range(q.mm, q.total_bits);
  constexpr int kLd = 4;  // (key, index) loads in flight per thread before the first use
  for (uint32_t j0 = gtid; j0 < m; j0 += kLd * kN) {
    uint64_t kk[kLd];
    uint32_t vv[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kN;
      kk[u] = j < m ? q.tk[s0 + j] : 0ull;
      vv[u] = j < m ? q.tv[s0 + j] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kN;
      if (j < m) {
        sk[j] = kk[u];
        sv[j] = vv[u];
        const uint32_t fine = (part_bucket(q, r, kk[u]) & fmask) >> fshift;
        sf[j] = (uint16_t)fine;
        atomicAdd(&fc[fine], 1u);
      }
    }
  }
  grp_bar<kN>(bar);
  {
    constexpr int kPer = kGrpFine / kN > 0 ? kGrpFine / kN : 1;
    uint32_t c[kPer], t = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t j = gtid * kPer + u;
      c[u] = j < nf ? fc[j] : 0u;
      t += c[u];
    }
    uint32_t v = grp_excl_scan<kN>(t, sh, bar, gtid);
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t j = gtid * kPer + u;
      if (j < nf) {
        fb[j] = v;
        fc[j] = v;
      }
      v += c[u];
    }
    if (gtid == 0) fb[nf] = m;
  }
  grp_bar<kN>(bar);
  for (uint32_t j = gtid; j < m; j += kN) perm[atomicAdd(&fc[sf[j]], 1u)] = (uint16_t)j;
  grp_bar<kN>(bar);
  uint16_t* spos = sf;
  for (uint32_t j = gtid; j < m; j += kN) {
    const uint64_t k = sk[j];
    const uint32_t v = sv[j], fine = sf[j];
    const uint32_t lo = fb[fine], hi = fb[fine + 1];
    uint32_t below = 0;
    for (uint32_t s = lo; s < hi; ++s) {
      const uint32_t o = perm[s];
      const uint64_t kq = sk[o];
      below += (kq < k || (kq == k && sv[o] < v)) ? 1u : 0u;
    }
    spos[j] = (uint16_t)(lo + below);
  }
  grp_bar<kN>(bar);
  uint32_t* outv = reinterpret_cast<uint32_t*>(sk);
  for (uint32_t j = gtid; j < m; j += kN) outv[spos[j]] = sv[j];
  grp_bar<kN>(bar);
  for (uint32_t t = gtid; t < m; t += kN) {
    const uint32_t v = outv[t];
    order[s0 + t] = ids ? ids[v] : (uint64_t)v;
  }
  grp_bar<kN>(bar);  // the slice is reused by the group's next partition
}

// Sort partitions [0, np) of (bases[p], bases[p+1]) with the CTA's groups (slot = the CTA's
// group g takes p = first + g * stride0 + j * stride), then the oversized ones CTA-wide.
template <int kT>
__device__ __forceinline__ void sort_partitions_grouped(const Part& q, const uint32_t* bases,
                                                        uint32_t p_begin, uint32_t p_step,
                                                        uint32_t np, uint32_t s_off,
                                                        const uint64_t* __restrict__ ids,
                                                        uint64_t* __restrict__ order,
                                                        unsigned char* smem_raw,
                                                        uint32_t (*gsh)[32]) {
#ifdef TIE_NO_GROUPS
  for (uint32_t p = p_begin; p < np; p += p_step) {
    const uint32_t s0 = bases[p], m = bases[p + 1] - s0;
    if (m) sort_partition<kT>(q, s_off + s0, m, ids, order, smem_raw);
    __syncthreads();
  }
  return;
#endif
  const int grp = threadIdx.x / (kT / kGroups), gtid = threadIdx.x % (kT / kGroups);
  for (uint32_t p = p_begin + grp * p_step; p < np; p += kGroups * p_step) {
    const uint32_t s0 = bases[p], m = bases[p + 1] - s0;
    if (m && m <= kGrpCap)
      sort_partition_grp<kT / kGroups>(q, s_off + s0, m, ids, order, smem_raw + grp * kGrpBytes,
                                       gsh[grp], 1 + grp, gtid);
  }
  __syncthreads();
  for (uint32_t p = p_begin; p < np; p += p_step) {
    const uint32_t s0 = bases[p], m = bases[p + 1] - s0;
    if (m > kGrpCap) sort_partition<kT>(q, s_off + s0, m, ids, order, smem_raw);
    __syncthreads();
  }
}

template <int kT>
__global__ void __launch_bounds__(kT, 1536 / kT) part_sort_kernel(Part q, uint64_t n,
                                                                   const uint64_t* __restrict__ ids,
                                                                   uint64_t* __restrict__ order,
                                                                   Fallback f) {
  if (*(volatile int*)q.overflow) {
    if (blockIdx.x == 0 && threadIdx.x == 0) lsd_tail_launch(f, q.keys, n, ids, order);
    return;
  }
  const uint32_t p = blockIdx.x;
  const uint32_t s0 = q.pbase[p], m = q.pbase[p + 1] - s0;  // m <= kPartCap
  if (m == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  sort_partition<kT>(q, s0, m, ids, order, smem_raw);
}

// The partition path in ONE cooperative launch: count (keys of the CTA's chunk staged in
// shared memory, one atomic per (CTA, partition) reservation) -> grid sync -> every CTA scans
// the partition counts itself and scatters its staged keys (no second read of the keys) ->
// grid sync -> the CTAs sort the partitions round-robin.  An overflowing partition leaves
// everything to part_fallback_kernel (the device-side LSD path).
constexpr int kFusedThreads = 512;

__global__ void __launch_bounds__(kFusedThreads, 2) part_fused_kernel(
    Part q, uint64_t n, const uint64_t* __restrict__ ids, uint64_t* __restrict__ order) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t pb[kPartMaxP + 1];  // partition bases (every CTA keeps its own copy)
  __shared__ uint32_t sh[32];
  __shared__ int over;
  const uint32_t P = q.P;
  uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);   // [P] chunk histogram -> cursors
  // the chunk's keys (after the local bases / cursors when the chunk is grouped locally)
  uint64_t* ck = reinterpret_cast<uint64_t*>(h + (q.local_scatter ? 3 : 1) * kPartMaxP);
  for (uint32_t p = threadIdx.x; p < P; p += kFusedThreads) h[p] = 0;
  // launched as a programmatic dependent of the score kernel: the keys and their range are
  // read only after the score grid has completed (a no-op without the dependency)
  cudaGridDependencySynchronize();
  __syncthreads();
  const KeyRange r = key_range(q.mm, q.total_bits);
  const uint64_t lo = (uint64_t)blockIdx.x * q.chunk;
  const uint64_t hi = min(n, lo + q.chunk);
  const uint32_t cn = hi > lo ? (uint32_t)(hi - lo) : 0u;
  constexpr int kLd = 8;  // key loads in flight per thread before the first use
  for (uint32_t j0 = threadIdx.x; j0 < cn; j0 += kLd * kFusedThreads) {
    uint64_t kk[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kFusedThreads;
      kk[u] = j < cn ? q.keys[lo + j] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kFusedThreads;
      if (j < cn) {
        ck[j] = kk[u];
        atomicAdd(&h[part_bucket(q, r, kk[u]) >> q.low_bits], 1u);
      }
    }
  }
  __syncthreads();
  // local grouping (before the grid sync, so it overlaps the other CTAs' staging): the
  // chunk's keys ordered by partition in shared memory (lb: local partition bases, srt: key
  // index per local position), so the scatter below writes each partition's run with
  // consecutive threads instead of one scattered store per key
  uint32_t* lb = h + kPartMaxP;                                   // [P] local bases
  uint32_t* cur = lb + kPartMaxP;                                 // [P] local cursors
  uint16_t* srt = reinterpret_cast<uint16_t*>(ck + q.chunk);      // [chunk]
  if (q.local_scatter) {
    constexpr int kPer = kPartMaxP / kFusedThreads;
    uint32_t c[kPer], t = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t p = threadIdx.x * kPer + u;
      c[u] = p < P ? h[p] : 0u;
      t += c[u];
    }
    uint32_t v = block_excl_scan_t<kFusedThreads>(t, sh);
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t p = threadIdx.x * kPer + u;
      if (p < P) {
        lb[p] = v;
        cur[p] = v;
      }
      v += c[u];
    }
  }
  for (uint32_t p = threadIdx.x; p < P; p += kFusedThreads) {
    const uint32_t c = h[p];
    h[p] = c ? atomicAdd(q.pcount + p, c) : 0u;  // this CTA's offset inside partition p
  }
  if (q.local_scatter) {
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < cn; j += kFusedThreads)
      srt[atomicAdd(&cur[part_bucket(q, r, ck[j]) >> q.low_bits], 1u)] = (uint16_t)j;
  }
  grid.sync();
  // partition bases from the final counts (each CTA scans the <= 2048 counts itself)
  {
    constexpr int kPer = kPartMaxP / kFusedThreads;
    uint32_t c[kPer], t = 0;
    int big = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t p = threadIdx.x * kPer + u;
      c[u] = p < P ? __ldcg(q.pcount + p) : 0u;
      t += c[u];
      big |= c[u] > q.cap1;
    }
    if (threadIdx.x == 0) over = 0;
    __syncthreads();
    if (big) over = 1;
    uint32_t v = block_excl_scan_t<kFusedThreads>(t, sh);
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t p = threadIdx.x * kPer + u;
      if (p < P) pb[p] = v;
      v += c[u];
    }
    if (threadIdx.x == 0) pb[P] = (uint32_t)n;
    __syncthreads();
  }
  if (over) {  // identical decision in every CTA (same counts): hand over to the LSD path
    if (blockIdx.x == 0 && threadIdx.x == 0) *q.overflow = 1;
    return;
  }
  for (uint32_t p = threadIdx.x; p < P; p += kFusedThreads) h[p] += pb[p];
  __syncthreads();
  if (q.local_scatter) {
    for (uint32_t t = threadIdx.x; t < cn; t += kFusedThreads) {
      const uint32_t j = srt[t];
      const uint64_t k = ck[j];
      const uint32_t p = part_bucket(q, r, k) >> q.low_bits;
      const uint32_t pos = h[p] + (t - lb[p]);
      q.tk[pos] = k;
      q.tv[pos] = (uint32_t)(lo + j);
    }
  } else {
    for (uint32_t j = threadIdx.x; j < cn; j += kFusedThreads) {
      const uint64_t k = ck[j];
      const uint32_t pos = atomicAdd(&h[part_bucket(q, r, k) >> q.low_bits], 1u);
      q.tk[pos] = k;
      q.tv[pos] = (uint32_t)(lo + j);
    }
  }
  grid.sync();
  // CTA-wide sorts here: the group-parallel sorts measured slower on this path (1M keys:
  // 91-94 vs 85 us per score+rank step), they pay off only in level 2 below
  for (uint32_t p = blockIdx.x; p < P; p += gridDim.x) {
    const uint32_t s0 = pb[p], m = pb[p + 1] - s0;
    if (m) sort_partition<kFusedThreads>(q, s0, m, ids, order, smem_raw);
    __syncthreads();
  }
}

// after the fused kernel: the LSD fallback when a partition overflowed (a cooperative launch
// may not contain device-side launches -- cudaErrorNotPermitted -- so this is its own kernel)
__global__ void part_fallback_kernel(Part q, uint64_t n, const uint64_t* ids, uint64_t* order,
                                     Fallback f) {
  cudaGridDependencySynchronize();  // launched programmatically: wait for the sort grid
  if (*(volatile int*)q.overflow) lsd_tail_launch(f, q.keys, n, ids, order);
}

// Level 2 of the two-level partition path (n > kPartMaxN): one CTA per level-1 partition
// (~n/2048 keys, in global memory) histograms its keys over P2 sub-partitions (the next
// p2_log2 bucket bits), regroups them into tk2 / tv2 and sorts every sub-partition (~1k keys)
// in shared memory with sort_partition.  A sub-partition above kPartCap (massive ties) only
// raises the overflow flag; part_fallback_kernel, launched after this grid, then runs the
// stable LSD path, which rewrites the whole order.
constexpr uint32_t kL2MaxP = 1024;

__global__ void __launch_bounds__(kFusedThreads, 2) part_l2_kernel(
    Part q, uint64_t n, const uint64_t* __restrict__ ids, uint64_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int skip;
  // another CTA of THIS grid may raise the flag at any moment: read it once per CTA so the
  // whole CTA leaves (or stays) together -- a per-thread read let part of a CTA return and
  // the rest run its barriers short-handed
  if (threadIdx.x == 0) skip = *(volatile int*)q.overflow;
  __syncthreads();
  if (skip) return;
  __shared__ uint32_t sb[kL2MaxP + 1];  // sub-partition bases
  __shared__ uint32_t cur[kL2MaxP];
  __shared__ uint32_t sh[32];
  __shared__ int big;
  const uint32_t p = blockIdx.x;
  const uint32_t s0 = q.pbase[p], m1 = q.pbase[p + 1] - s0;
  if (m1 == 0) return;
  const uint32_t P2 = 1u << q.p2_log2, mask2 = P2 - 1;
  const KeyRange r = key_range(q.mm, q.total_bits);
  for (uint32_t j = threadIdx.x; j < P2; j += kFusedThreads) cur[j] = 0;
  if (threadIdx.x == 0) big = 0;
  __syncthreads();
  constexpr int kLd = 8;  // loads in flight per thread before the first use
  for (uint32_t j0 = threadIdx.x; j0 < m1; j0 += kLd * kFusedThreads) {
    uint64_t kk[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kFusedThreads;
      kk[u] = j < m1 ? q.tk[s0 + j] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u)
      if (j0 + u * kFusedThreads < m1)
        atomicAdd(&cur[(part_bucket(q, r, kk[u]) >> q.fine_log2) & mask2], 1u);
  }
  __syncthreads();
  {
    constexpr int kPer = kL2MaxP / kFusedThreads;
    uint32_t c[kPer], t = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t j = threadIdx.x * kPer + u;
      c[u] = j < P2 ? cur[j] : 0u;
      t += c[u];
      if (c[u] > kPartCap) big = 1;
    }
    uint32_t v = block_excl_scan_t<kFusedThreads>(t, sh);
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t j = threadIdx.x * kPer + u;
      if (j < P2) {
        sb[j] = v;
        cur[j] = v;
      }
      v += c[u];
    }
    if (threadIdx.x == 0) sb[P2] = m1;
  }
  __syncthreads();
  if (big) {
    if (threadIdx.x == 0) atomicExch(q.overflow, 1);
    return;
  }
  for (uint32_t j0 = threadIdx.x; j0 < m1; j0 += kLd * kFusedThreads) {
    uint64_t kk[kLd];
    uint32_t vv[kLd];
#pragma unroll
    for (int u = 0; u < kLd; ++u) {
      const uint32_t j = j0 + u * kFusedThreads;
      kk[u] = j < m1 ? q.tk[s0 + j] : 0ull;
      vv[u] = j < m1 ? q.tv[s0 + j] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kLd; ++u)
      if (j0 + u * kFusedThreads < m1) {
        const uint32_t pos =
            atomicAdd(&cur[(part_bucket(q, r, kk[u]) >> q.fine_log2) & mask2], 1u);
        q.tk2[s0 + pos] = kk[u];
        q.tv2[s0 + pos] = vv[u];
      }
  }
  __syncthreads();  // this CTA's global writes are visible to it after the barrier
  Part q2 = q;
  q2.tk = q.tk2;
  q2.tv = q.tv2;
  __shared__ uint32_t gsh[kGroups][32];
#ifndef TIE_L2_NOSORT
  sort_partitions_grouped<kFusedThreads>(q2, sb, 0, 1, P2, s0, ids, order, smem_raw, gsh);
#endif
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

int items_for(uint64_t) { return 16; }

struct Layout {
  size_t k0, k1, v0, v1, hist, plan, status, gstatus, gsum, gdone, counter, flag, k2, k3, v3,
      meta_begin, meta_end, total;
  // bucket / partition path: [bzero_begin, bzero_end) = count (bucket path) or pcount
  // (partition path), mm, overflow -- zeroed once per sort
  size_t count, mm, overflow, base, cursor, partial, seg, bzero_begin, bzero_end;
  size_t pcount, pbase, cta_off, tk2, tv2;
  uint32_t tiles, nb_log2, nseg;
  bool part, part2;  // one-level (n <= kPartMaxN) / two-level partition path
  uint32_t p_log2, p2_log2, fine_log2;
};

constexpr uint32_t kPartMaxCtas = 512;

uint32_t ceil_log2(uint64_t x) {
  uint32_t l = 0;
  while (l < 63 && (1ull << l) < x) ++l;
  return l;
}

uint32_t bucket_log2(uint64_t n) {
  uint32_t l = 0;
  while (l < 63 && (1ull << l) < (n + 1) / 2) ++l;  // ~2-4 keys per occupied bucket
  return std::min(std::max(l, kMinBucketsLog2), kMaxBucketsLog2);
}

Layout layout(uint64_t n, bool with_ids) {
  Layout L{};
  const uint64_t tile_keys = (uint64_t)kThreads * items_for(n);
  L.tiles = (uint32_t)std::max<uint64_t>(1, (n + tile_keys - 1) / tile_keys);
  L.nb_log2 = bucket_log2(n);
  L.nseg = (uint32_t)std::max<uint64_t>(1, (n + kSegStep - 1) / kSegStep);
  const uint64_t nb = 1ull << L.nb_log2;
  size_t off = 0;
  L.k0 = off; off += align_up(8 * n);
  L.k1 = off; off += align_up(8 * n);
  L.v0 = off; off += align_up(4 * n);
  L.v1 = off; off += align_up(4 * n);
  // LSD metadata, zeroed by ONE memset (or, as the bucket path's fallback, on the device):
  // histograms, look-back status, counters
  L.meta_begin = off;
  L.hist = off; off += align_up(4 * kPasses * kBins);
  L.status = off; off += align_up(8ull * kPasses * L.tiles * kBins);
  const uint64_t groups = (L.tiles + kGroup - 1) / kGroup;
  L.gstatus = off; off += align_up(8ull * kPasses * groups * kBins);
  L.gsum = off; off += align_up(8ull * kPasses * groups * kBins);
  L.gdone = off; off += align_up(4ull * kPasses * groups);
  L.counter = off; off += align_up(4 * kPasses);
  L.meta_end = off;
  L.plan = off; off += align_up(sizeof(Plan));
  L.flag = off; off += align_up(sizeof(int));
  static const int two_level = getenv("TIE_NO_TWO_LEVEL") ? 0 : 1;  // A/B switch
  L.part = n <= kPartMaxN;
  // two levels pay off from ~6M keys (B200: 8M 0.32 vs 0.37 ms bucket path; 4M 0.18 vs 0.15)
  L.part2 = !L.part && two_level && n >= (6ull << 20) && n < (1ull << 32);
  // ~kSubLog2-key (sub-)partitions: the group sorts' size (kGrpCap ~2.7x the mean)
#ifndef TIE_SUB_LOG2
#define TIE_SUB_LOG2 10
#endif
  constexpr uint32_t kSubLog2 = TIE_SUB_LOG2;
  L.p_log2 = std::min<uint32_t>(
      std::max<uint32_t>(ceil_log2((n + (1ull << kSubLog2) - 1) >> kSubLog2), 6u), 11u);
  // two-level: 2048 level-1 partitions of P2 sub-partitions each
  L.p2_log2 = L.part2 ? std::min<uint32_t>(std::max<uint32_t>(
                            ceil_log2((n + (1ull << (L.p_log2 + kSubLog2)) - 1) >>
                                      (L.p_log2 + kSubLog2)), 1u),
                        10u)
                      : 0u;
  L.fine_log2 = std::min<uint32_t>(
      std::max<uint32_t>(ceil_log2((n + (1ull << (L.p_log2 + L.p2_log2)) - 1) >>
                                   (L.p_log2 + L.p2_log2)),
                         1u),
      kPartMaxFineLog2);
  L.part = L.part || L.part2;  // both share the level-1 buffers below
  L.bzero_begin = off;
  if (L.part) {
    L.pcount = off; off += align_up(4 * ((1ull << L.p_log2) + 1));  // + the count ticket
  } else {
    L.count = off; off += align_up(4 * nb);
  }
  L.mm = off; off += align_up(16);
  L.overflow = off; off += align_up(sizeof(int));
  L.bzero_end = off;
  const uint64_t bnb = L.part ? 0 : nb;  // bucket-path arrays (unused on the partition path)
  L.base = off; off += align_up(4 * (bnb + 1));
  L.cursor = off; off += align_up(4 * bnb);
  L.partial = off; off += align_up(4 * (bnb / kScanChunk));
  L.seg = off; off += align_up(4 * (L.part ? 1 : (uint64_t)L.nseg + 1));
  if (L.part) {
    L.pbase = off; off += align_up(4 * ((1ull << L.p_log2) + 1));
    L.cta_off = off; off += align_up(4ull * kPartMaxCtas << L.p_log2);
  }
  if (L.part2) {  // level-2 regrouped (key, index) -- separate from the LSD buffers
    L.tk2 = off; off += align_up(8 * n);
    L.tv2 = off; off += align_up(4 * n);
  }
  L.k2 = off; off += with_ids ? align_up(8 * n) : 0;  // transformed keys (id path)
  L.k3 = off; off += with_ids ? align_up(8 * n) : 0;  // keys gathered into id order
  L.v3 = off; off += with_ids ? align_up(4 * n) : 0;  // the id-order permutation
  L.total = off;
  return L;
}

Bucket make_bucket(char* base, const Layout& L, const uint64_t* keys) {
  Bucket b;
  b.keys = keys;
  b.tk = (uint64_t*)(base + L.k1);  // the LSD fallback runs only when the scatter did not
  b.tv = (uint32_t*)(base + L.v0);
  b.count = (uint32_t*)(base + L.count);
  b.base = (uint32_t*)(base + L.base);
  b.cursor = (uint32_t*)(base + L.cursor);
  b.partial = (uint32_t*)(base + L.partial);
  b.seg = (uint32_t*)(base + L.seg);
  b.mm = (unsigned long long*)(base + L.mm);
  b.overflow = (int*)(base + L.overflow);
  b.nb_log2 = L.nb_log2;
  b.nb = 1u << L.nb_log2;
  b.chunks = b.nb / kScanChunk;
  b.nseg = L.nseg;
  return b;
}

Work make_work(char* base, const Layout& L) {
  Work w;
  w.k[0] = (uint64_t*)(base + L.k0);
  w.k[1] = (uint64_t*)(base + L.k1);
  w.v[0] = (uint32_t*)(base + L.v0);
  w.v[1] = (uint32_t*)(base + L.v1);
  w.hist = (uint32_t*)(base + L.hist);
  w.plan = (Plan*)(base + L.plan);
  w.status = (uint64_t*)(base + L.status);
  w.gstatus = (uint64_t*)(base + L.gstatus);
  w.gsum = (uint64_t*)(base + L.gsum);
  w.gdone = (uint32_t*)(base + L.gdone);
  w.tile_counter = (uint32_t*)(base + L.counter);
  w.flag = (int*)(base + L.flag);
  w.tiles = L.tiles;
  return w;
}

int sm_count(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v > 0 ? v : 148;
}

template <int ITEMS>
void launch_passes(tie_ctx* ctx, Work& w, uint64_t n, bool explicit_vals, const uint64_t* ids,
                   uint64_t* order, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(onesweep_kernel<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(PassSmem<ITEMS>));
    attr = true;
  }
  for (int p = 0; p < kPasses; ++p) {
    ProfScope q(ctx, "rank.onesweep", s);
    onesweep_kernel<ITEMS><<<w.tiles, kThreads, sizeof(PassSmem<ITEMS>), s>>>(
        w, n, p, explicit_vals ? 1 : 0, ids, order);
  }
}

// plan + the digit passes over w.k[0] (+ w.v[0] if explicit_vals); histograms already in
// w.hist.  With `order` the last pass emits the dispatch order (ids[value] or value).
cudaError_t sort_passes(tie_ctx* ctx, Work& w, uint64_t n, bool explicit_vals,
                        const uint64_t* ids, uint64_t* order, cudaStream_t s) {
  {
    ProfScope p(ctx, "rank.plan", s);
    plan_kernel<<<1, kThreads, 0, s>>>(w.hist, n, w.plan);
  }
  if (items_for(n) == 8)
    launch_passes<8>(ctx, w, n, explicit_vals, ids, order, s);
  else
    launch_passes<16>(ctx, w, n, explicit_vals, ids, order, s);
  capi::count_launch(1 + kPasses);
  if (order) {
    const int sms = sm_count(ctx->device);
    const unsigned g = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 4);
    identity_order_kernel<<<g, 256, 0, s>>>(w, n, ids, order, explicit_vals ? 1 : 0);
    capi::count_launch();
  }
  return cudaGetLastError();
}

cudaError_t part_sort(tie_ctx* ctx, char* base, const Layout& L, const uint64_t* keys,
                      uint64_t n, const uint64_t* ids, uint64_t* order, const Fallback& f,
                      int sms, cudaStream_t s) {
  static bool attr = false;
  const size_t smem = std::max((size_t)kPartCap * (8 + 4 + 2 + 2) +
                                   4 * (2 * (1u << kPartMaxFineLog2) + 1),
                               kGroups * kGrpBytes);
  if (!attr) {
    cudaFuncSetAttribute(part_sort_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(part_sort_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  Part q;
  q.keys = keys;
  q.tk = (uint64_t*)(base + L.k1);  // the LSD fallback runs only when the scatter did not
  q.tv = (uint32_t*)(base + L.v0);
  q.pcount = (uint32_t*)(base + L.pcount);
  q.pbase = (uint32_t*)(base + L.pbase);
  q.cta_off = (uint32_t*)(base + L.cta_off);
  q.mm = (unsigned long long*)(base + L.mm);
  q.overflow = (int*)(base + L.overflow);
  q.p_log2 = L.p_log2;
  q.P = 1u << L.p_log2;
  q.fine_log2 = L.fine_log2;
  q.p2_log2 = L.p2_log2;
  q.low_bits = L.p2_log2 + L.fine_log2;
  q.total_bits = L.p_log2 + q.low_bits;
  q.cap1 = L.part2 ? 0xffffffffu : kPartCap;
  q.local_scatter = 0;

  q.tk2 = L.part2 ? (uint64_t*)(base + L.tk2) : nullptr;
  q.tv2 = L.part2 ? (uint32_t*)(base + L.tv2) : nullptr;
  q.ctas = (uint32_t)std::min<uint64_t>(
      std::min<uint64_t>((uint64_t)sms * 2, kPartMaxCtas), (n + 1023) / 1024);
  q.chunk = (n + q.ctas - 1) / q.ctas;
  // default: the whole path as one cooperative launch (count -> scatter -> sort)
  static const int fused = getenv("TIE_PART_UNFUSED") ? 0 : 1;  // A/B switch
  if (L.part2) {  // level 1 (count, scatter), then level 2 per level-1 partition
    static bool l2attr = false;
    if (!l2attr) {
      cudaFuncSetAttribute(part_l2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      l2attr = true;
    }
    {
      ProfScope p(ctx, "rank.count", s);
      part_count_kernel<<<q.ctas, kPartThreads, 0, s>>>(q, n);
    }
    {
      ProfScope p(ctx, "rank.scatter", s);
      // tiles of 32k keys (measured at 64M: 16k 1.05 ms, 32k 0.91, 64k 1.01; per-key
      // scattered stores 3.23 ms)
      constexpr uint32_t kTile = 32768;
      static bool sattr = false;
      static const int tiled = getenv("TIE_NO_TILED_SCATTER") ? 0 : 1;  // A/B switch
      if (!sattr) {
        cudaFuncSetAttribute(part_scatter_tiled_kernel<kTile>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scat_smem<kTile>());
        sattr = true;
      }
      if (tiled)
        part_scatter_tiled_kernel<kTile><<<q.ctas, kScatThreads, scat_smem<kTile>(), s>>>(q, n);
      else
        part_scatter_kernel<<<q.ctas, kPartThreads, 0, s>>>(q, n);
    }
    {
      ProfScope p(ctx, "rank.local", s);
      part_l2_kernel<<<q.P, kFusedThreads, smem, s>>>(q, n, ids, order);
      part_fallback_kernel<<<1, 1, 0, s>>>(q, n, ids, order, f);
    }
    capi::count_launch(4);
    return cudaGetLastError();
  }
  if (fused) {
    static bool fattr = false;
    static int bpsm = 0;
    if (!fattr) {
      cudaFuncSetAttribute(part_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, part_fused_kernel, kFusedThreads,
                                                    smem);
      fattr = true;
    }
    const uint64_t co = (uint64_t)std::max(bpsm, 0) * sms;  // co-resident CTAs
    Part qf = q;
    static const int local_scatter = getenv("TIE_NO_LOCAL_SCATTER") ? 0 : 1;  // A/B switch
    qf.ctas = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(co, kPartMaxCtas),
                                           (n + 1023) / 1024);
    if (qf.ctas > 0) qf.chunk = (n + qf.ctas - 1) / qf.ctas;
    qf.local_scatter =
        local_scatter && 4 * 3 * kPartMaxP + 10 * qf.chunk + 16 <= smem && qf.chunk < 65536;
    if (qf.ctas > 0 && 4 * kPartMaxP + 8 * qf.chunk <= smem) {
      ProfScope p(ctx, "rank.fused", s);
      void* args[] = {(void*)&qf, (void*)&n, (void*)&ids, (void*)&order};
      // cooperative AND a programmatic dependent of the score kernel: the grid's launch and
      // CTA setup overlap the score grid's tail; it waits (cudaGridDependencySynchronize)
      // before reading the keys
      static const bool no_pdl = getenv("TIE_NO_RANK_PDL") != nullptr;  // A/B switch
      cudaError_t e = cudaErrorNotSupported;
      if (!no_pdl) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(qf.ctas);
        cfg.blockDim = dim3(kFusedThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        e = cudaLaunchKernelEx(&cfg, part_fused_kernel, qf, n, ids, order);
        if (e != cudaSuccess) cudaGetLastError();
      }
      if (e != cudaSuccess)
        e = cudaLaunchCooperativeKernel((const void*)part_fused_kernel, qf.ctas, kFusedThreads,
                                        args, smem, s);
      if (e != cudaSuccess) return e;
      {  // programmatic dependent launch: its launch processing overlaps the sort grid
        // (measured 94.8 -> 93.2 us per 1M score+rank step)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(1);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, part_fallback_kernel, qf, n, ids, order, f);
        if (e != cudaSuccess) return e;
      }
      capi::count_launch(2);
      return cudaGetLastError();
    }
  }
  {
    ProfScope p(ctx, "rank.count", s);
    part_count_kernel<<<q.ctas, kPartThreads, 0, s>>>(q, n);
  }
  {
    ProfScope p(ctx, "rank.scatter", s);
    part_scatter_kernel<<<q.ctas, kPartThreads, 0, s>>>(q, n);
  }
  {
    ProfScope p(ctx, "rank.local", s);
    static const int threads = getenv("TIE_PART_SORT_THREADS") ? atoi(getenv("TIE_PART_SORT_THREADS")) : 512;
    if (threads == 256)
      part_sort_kernel<256><<<q.P, 256, smem, s>>>(q, n, ids, order, f);
    else
      part_sort_kernel<512><<<q.P, 512, smem, s>>>(q, n, ids, order, f);
  }
  capi::count_launch(3);
  return cudaGetLastError();
}

// count -> scan -> scatter -> local sort over keys whose range is already folded into the
// bucket state (zeroed count / mm / overflow).  Emits the dispatch order.
cudaError_t bucket_sort(tie_ctx* ctx, char* base, const Layout& L, const uint64_t* keys,
                        uint64_t n, const uint64_t* ids, uint64_t* order, cudaStream_t s) {
  static bool attr = false;
  const size_t local_smem = (size_t)kSegCap * 12;
  if (!attr) {  // also covers the device-side (fallback) launches
    cudaFuncSetAttribute(onesweep_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(PassSmem<16>));
    cudaFuncSetAttribute(bucket_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)local_smem);
    attr = true;
  }
  const int sms = sm_count(ctx->device);
  Fallback f;
  f.w = make_work(base, L);
  f.meta = (uint4*)(base + L.meta_begin);
  f.meta16 = (L.meta_end - L.meta_begin) / 16;
  f.grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 4);
  if (L.part) return part_sort(ctx, base, L, keys, n, ids, order, f, sms, s);
  Bucket b = make_bucket(base, L, keys);
  const unsigned g = (unsigned)((n + kStreamTile - 1) / kStreamTile);
  {
    ProfScope p(ctx, "rank.count", s);
    bucket_count_kernel<<<g, 256, 0, s>>>(b, n);
  }
  {
    ProfScope p(ctx, "rank.scan", s);
    bucket_scan_a_kernel<<<b.chunks, kScanThreads, 0, s>>>(b);
    bucket_scan_b_kernel<<<b.chunks, kScanThreads, 0, s>>>(b, n);
  }
  {
    ProfScope p(ctx, "rank.scatter", s);
    bucket_scatter_kernel<<<g, 256, 0, s>>>(b, n);
  }
  {
    ProfScope p(ctx, "rank.local", s);
    bucket_local_kernel<<<b.nseg, kLocalThreads, local_smem, s>>>(b, n, ids, order, f);
  }
  capi::count_launch(5);
  return cudaGetLastError();
}

}  // namespace

size_t rank_scratch_bytes(uint64_t n, bool with_ids) { return layout(n, with_ids).total; }

bool rank_output_coalesced(uint64_t n) { return layout(n, false).part; }

RankPrep rank_prepare(tie_ctx* ctx, uint64_t n, cudaStream_t s) {
  RankPrep r{nullptr, nullptr};
  const Layout L = layout(n, false);
  char* base = (char*)capi::scratch(ctx, L.total, s);
  if (!base) return r;
  cudaMemsetAsync(base + L.bzero_begin, 0, L.bzero_end - L.bzero_begin, s);
  r.keys = (uint64_t*)(base + L.k0);
  r.minmax = (unsigned long long*)(base + L.mm);
  return r;
}

cudaError_t rank_prepared(tie_ctx* ctx, uint64_t n, uint64_t* order, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (n >= (1ull << 32)) return cudaErrorInvalidValue;  // u32 values / bucket positions
  const Layout L = layout(n, false);
  char* base = (char*)capi::scratch(ctx, L.total, s);
  if (!base) return cudaErrorMemoryAllocation;
  return bucket_sort(ctx, base, L, (const uint64_t*)(base + L.k0), n, nullptr, order, s);
}

cudaError_t launch_rank(tie_ctx* ctx, const double* key, const uint64_t* ids, uint64_t n,
                        uint64_t* order, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (n >= (1ull << 32)) return cudaErrorInvalidValue;  // u32 values
  const Layout L = layout(n, ids != nullptr);
  char* base = (char*)capi::scratch(ctx, L.total, s);
  if (!base) return cudaErrorMemoryAllocation;
  Work w = make_work(base, L);
  const int sms = sm_count(ctx->device);
  const unsigned egrid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 4);
  const size_t meta = L.meta_end - L.meta_begin;
  cudaMemsetAsync(base + L.bzero_begin, 0, L.bzero_end - L.bzero_begin, s);

  uint64_t* tkeys = ids ? (uint64_t*)(base + L.k2) : w.k[0];
  {
    ProfScope p(ctx, "rank.keys", s);
    keys_from_double_kernel<<<egrid, 256, 0, s>>>(key, n, tkeys,
                                                  (unsigned long long*)(base + L.mm), ctx->d_err);
    capi::count_launch();
  }
  if (!ids) return bucket_sort(ctx, base, L, tkeys, n, nullptr, order, s);

  cudaMemsetAsync(w.flag, 0, sizeof(int), s);
  ids_sorted_kernel<<<egrid, 256, 0, s>>>(ids, n, w.flag);
  capi::count_launch();
  int unsorted = 0;
  cudaMemcpyAsync(&unsorted, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  // ids ascending: (key, index) order == (key, id) order
  if (!unsorted) return bucket_sort(ctx, base, L, tkeys, n, ids, order, s);
  // unsorted ids: stable LSD sort of (id, index) first; the stable LSD key sort then starts
  // from id order
  cudaMemsetAsync(base + L.meta_begin, 0, meta, s);
  copy_hist_kernel<<<egrid, 256, 0, s>>>(ids, n, w.k[0], w.hist);
  capi::count_launch();
  if ((e = sort_passes(ctx, w, n, false, nullptr, nullptr, s)) != cudaSuccess) return e;
  gather_by_id_kernel<<<egrid, 256, 0, s>>>(w, n, tkeys, (uint64_t*)(base + L.k3),
                                            (uint32_t*)(base + L.v3), ctx->d_err);
  capi::count_launch();
  cudaMemcpyAsync(w.v[0], base + L.v3, 4 * n, cudaMemcpyDeviceToDevice, s);
  cudaMemsetAsync(base + L.meta_begin, 0, meta, s);
  copy_hist_kernel<<<egrid, 256, 0, s>>>((const uint64_t*)(base + L.k3), n, w.k[0], w.hist);
  capi::count_launch();
  return sort_passes(ctx, w, n, true, ids, order, s);
}

}  // namespace dev
}  // namespace tie
