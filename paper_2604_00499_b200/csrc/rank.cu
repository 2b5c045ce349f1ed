// K2 -- dispatch order of a static waiting queue: stable LSD radix sort by (key, id).
//
// Reference: WaitingQueue (proj/src/sched.cpp:28-94) is a binary min-heap ordered by
// (key, req_id) (less(), sched.cpp:28-31); pushing n entries and popping until empty
// yields the lexicographic (key asc, id asc) order.  Here: keys are mapped to u64 by the
// order-preserving IEEE transform (x >= 0: bits | 2^63, x < 0: ~bits; -0.0 folded onto
// +0.0 because the heap compares keys with ==), then sorted with a stable LSD radix sort
// over values that start in ascending-id order -- which is exactly (key, id) order.
//
// Per pass (8-bit digits, 8 passes, passes whose digit is constant across all keys are
// skipped on the device): upsweep tile histograms -> per-digit scan across tiles ->
// downsweep that ranks each 4096-key tile stably in shared memory (warp match_any
// multi-split) and writes digit runs out coalesced.  A single global-histogram kernel up
// front provides every pass's bin bases and the skip mask, so the host never syncs.
#include <cuda_runtime.h>

#include <algorithm>

#include "tie_internal.cuh"

namespace tie {
namespace dev {

namespace {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kPasses = 64 / kRadixBits;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 keys per tile

struct Plan {
  uint32_t bin_base[kPasses][kBins];
  int active[kPasses];
  int sel[kPasses];    // buffer holding the input of pass p
  int first[kPasses];  // pass p is the first active one (values implicit if not explicit)
  int final_sel;
  int any_active;
};

struct Work {
  uint64_t* k[2];
  uint32_t* v[2];
  uint32_t* tile_counts;  // [kBins][num_tiles]
  uint32_t* hist;         // [kPasses][kBins]
  Plan* plan;
  int* flag;
};

__device__ __forceinline__ uint32_t digit_of(uint64_t key, int pass) {
  return (uint32_t)(key >> (pass * kRadixBits)) & (kBins - 1);
}

__device__ __forceinline__ uint64_t order_bits(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 == +0.0 under the heap's comparison
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// key validation + transform (WaitingQueue::push rejects non-finite keys, sched.cpp:60)
__global__ void keys_from_double_kernel(const double* __restrict__ key, uint64_t n,
                                        uint64_t* __restrict__ out, unsigned long long* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = key[i];
    if (!isfinite(x)) {
      report(err, i, kKeyNotFinite);
      out[i] = ~0ull;
    } else {
      out[i] = order_bits(x);
    }
  }
}

__global__ void global_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                   uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[2][kPasses][kBins];
  for (int i = threadIdx.x; i < 2 * kPasses * kBins; i += blockDim.x) (&h[0][0][0])[i] = 0;
  __syncthreads();
  const int copy = (threadIdx.x >> 5) & 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = keys[i];
#pragma unroll
    for (int p = 0; p < kPasses; ++p) atomicAdd(&h[copy][p][digit_of(k, p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kBins; i += blockDim.x) {
    const uint32_t c = (&h[0][0][0])[i] + (&h[1][0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// exclusive scan of 256 values held one per thread (blockDim == 256)
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* sh_warp,
                                                        uint32_t* total) {
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
  const uint32_t incl = x + (warp ? sh_warp[warp - 1] : 0);
  if (total && threadIdx.x == kThreads - 1) *total = incl;
  return incl - v;
}

__global__ void __launch_bounds__(kThreads) plan_kernel(const uint32_t* __restrict__ hist,
                                                        uint64_t n, Plan* plan) {
  __shared__ uint32_t sh_warp[kWarps];
  __shared__ int sh_active[kPasses];
  const int d = threadIdx.x;
  for (int p = 0; p < kPasses; ++p) {
    const uint32_t c = hist[p * kBins + d];
    if (d == 0) sh_active[p] = 0;
    __syncthreads();
    if ((uint64_t)c != n && c != 0) sh_active[p] = 1;  // more than one occupied digit
    plan->bin_base[p][d] = block_excl_scan_256(c, sh_warp, nullptr);
    __syncthreads();
  }
  if (d == 0) {
    int cnt = 0;
    for (int p = 0; p < kPasses; ++p) {
      plan->active[p] = sh_active[p];
      plan->sel[p] = cnt & 1;
      plan->first[p] = sh_active[p] && cnt == 0;
      cnt += sh_active[p];
    }
    plan->final_sel = cnt & 1;
    plan->any_active = cnt > 0;
  }
}

__global__ void __launch_bounds__(kThreads) upsweep_kernel(Work w, uint64_t n, int pass) {
  if (!w.plan->active[pass]) return;
  __shared__ uint32_t h[kWarps][kBins];
  for (int i = threadIdx.x; i < kWarps * kBins; i += kThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t* keys = w.k[w.plan->sel[pass]];
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint64_t i = base + (uint64_t)j * kThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[warp][digit_of(keys[i], pass)], 1u);
  }
  __syncthreads();
  const uint32_t num_tiles = gridDim.x;
  uint32_t c = 0;
#pragma unroll
  for (int q = 0; q < kWarps; ++q) c += h[q][threadIdx.x];
  w.tile_counts[(uint64_t)threadIdx.x * num_tiles + blockIdx.x] = c;
}

// one CTA per digit: exclusive scan of that digit's counts across tiles (+ bin base)
__global__ void __launch_bounds__(1024) tile_scan_kernel(Work w, uint32_t num_tiles, int pass) {
  if (!w.plan->active[pass]) return;
  __shared__ uint32_t sh_warp[32];
  __shared__ uint32_t carry;
  const int d = blockIdx.x;
  uint32_t* row = w.tile_counts + (uint64_t)d * num_tiles;
  if (threadIdx.x == 0) carry = w.plan->bin_base[pass][d];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t off = 0; off < num_tiles; off += 1024) {
    const uint32_t t = off + threadIdx.x;
    const uint32_t v = t < num_tiles ? row[t] : 0;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sh_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t s = sh_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      sh_warp[lane] = s;
    }
    __syncthreads();
    const uint32_t incl = x + (warp ? sh_warp[warp - 1] : 0);
    const uint32_t c0 = carry;
    if (t < num_tiles) row[t] = c0 + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry = c0 + incl;
    __syncthreads();
  }
}

struct DownSmem {
  uint64_t keys[kTile];
  uint32_t vals[kTile];
  uint32_t warp_hist[kWarps][kBins];
  uint32_t tile_excl[kBins];
  uint32_t global_off[kBins];
  uint32_t sh_warp[kWarps];
};

__global__ void __launch_bounds__(kThreads) downsweep_kernel(Work w, uint64_t n, int pass,
                                                             int explicit_vals) {
  const Plan* plan = w.plan;
  if (!plan->active[pass]) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DownSmem& sm = *reinterpret_cast<DownSmem*>(smem_raw);
  const int src = plan->sel[pass];
  const uint64_t* __restrict__ kin = w.k[src];
  const uint32_t* __restrict__ vin = w.v[src];
  const bool implicit = plan->first[pass] && !explicit_vals;
  uint64_t* __restrict__ kout = w.k[src ^ 1];
  uint32_t* __restrict__ vout = w.v[src ^ 1];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kBins; i += kThreads) (&sm.warp_hist[0][0])[i] = 0;
  const uint32_t num_tiles = gridDim.x;
  sm.global_off[threadIdx.x] = w.tile_counts[(uint64_t)threadIdx.x * num_tiles + blockIdx.x];
  __syncthreads();

  const uint64_t tile_base = (uint64_t)blockIdx.x * kTile;
  const uint64_t left = n - tile_base;
  const uint32_t valid = left < (uint64_t)kTile ? (uint32_t)left : (uint32_t)kTile;
  const unsigned lt_mask = (1u << lane) - 1u;
  uint64_t key[kItems];
  uint32_t val[kItems];
  uint32_t rank[kItems];
  // warp w owns tile slots [w*512, (w+1)*512): round j, lane l -> slot w*512 + j*32 + l,
  // so (round, lane) order is index order and the multi-split below is stable.
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t q = warp * (kItems * 32) + j * 32 + lane;
    const uint64_t i = tile_base + q;
    if (q < valid) {
      key[j] = kin[i];
      val[j] = implicit ? (uint32_t)i : vin[i];
    } else {
      key[j] = ~0ull;  // pads sort last in the tile and are never written out
      val[j] = 0;
    }
    const uint32_t d = digit_of(key[j], pass);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = sm.warp_hist[warp][d];
    __syncwarp();
    if ((peers & lt_mask) == 0) sm.warp_hist[warp][d] = before + __popc(peers);
    __syncwarp();
    rank[j] = before + __popc(peers & lt_mask);
  }
  __syncthreads();
  {  // per digit: exclusive over warps, then exclusive over digits
    const int d = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      const uint32_t c = sm.warp_hist[q][d];
      sm.warp_hist[q][d] = run;
      run += c;
    }
    const uint32_t ex = block_excl_scan_256(run, sm.sh_warp, nullptr);
    sm.tile_excl[d] = ex;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t d = digit_of(key[j], pass);
    const uint32_t pos = sm.tile_excl[d] + sm.warp_hist[warp][d] + rank[j];
    sm.keys[pos] = key[j];
    sm.vals[pos] = val[j];
  }
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < valid; q += kThreads) {
    const uint64_t k = sm.keys[q];
    const uint32_t d = digit_of(k, pass);
    const uint64_t g = (uint64_t)sm.global_off[d] + (q - sm.tile_excl[d]);
    kout[g] = k;
    vout[g] = sm.vals[q];
  }
}

__global__ void finish_kernel(Work w, uint64_t n, const uint64_t* __restrict__ ids,
                              uint64_t* __restrict__ order, int explicit_vals) {
  const Plan* plan = w.plan;
  const uint32_t* v = w.v[plan->final_sel];
  const bool identity = !plan->any_active && !explicit_vals;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t idx = identity ? i : v[i];
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

// after sorting (id, index) pairs: detect duplicate ids, and stage (key[perm], perm)
// as the explicit-value input of the key sort.
__global__ void gather_by_id_kernel(Work w, uint64_t n, const uint64_t* __restrict__ tkeys,
                                    uint64_t* __restrict__ kdst, uint32_t* __restrict__ vdst,
                                    unsigned long long* err) {
  const Plan* plan = w.plan;
  const uint64_t* sid = w.k[plan->final_sel];
  const uint32_t* perm = w.v[plan->final_sel];
  const bool identity = !plan->any_active;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const uint32_t p = identity ? (uint32_t)j : perm[j];
    if (j > 0 && sid[j] == sid[j - 1]) report(err, p, kDuplicateId);
    kdst[j] = tkeys[p];
    vdst[j] = p;
  }
}

__global__ void copy_ids_kernel(const uint64_t* __restrict__ ids, uint64_t n,
                                uint64_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = ids[i];
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t k0, k1, v0, v1, tc, hist, plan, flag, k2, k3, v3, total;
};

Layout layout(uint64_t n, bool with_ids) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  Layout L{};
  size_t off = 0;
  L.k0 = off; off += align_up(8 * n);
  L.k1 = off; off += align_up(8 * n);
  L.v0 = off; off += align_up(4 * n);
  L.v1 = off; off += align_up(4 * n);
  L.tc = off; off += align_up(4 * (size_t)kBins * tiles);
  L.hist = off; off += align_up(4 * kPasses * kBins);
  L.plan = off; off += align_up(sizeof(Plan));
  L.flag = off; off += align_up(sizeof(int));
  L.k2 = off; off += with_ids ? align_up(8 * n) : 0;  // transformed keys (id path)
  L.k3 = off; off += with_ids ? align_up(8 * n) : 0;  // keys gathered into id order
  L.v3 = off; off += with_ids ? align_up(4 * n) : 0;  // the id-order permutation
  L.total = off;
  return L;
}

int sm_count(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v > 0 ? v : 148;
}

// Sort w.k[0] (u64) with values implicit (index) or explicit in w.v[0].
cudaError_t radix_sort(tie_ctx* ctx, Work& w, uint64_t n, bool explicit_vals, int sms,
                       cudaStream_t s) {
  const uint32_t tiles = (uint32_t)((n + kTile - 1) / kTile);
  cudaMemsetAsync(w.hist, 0, sizeof(uint32_t) * kPasses * kBins, s);
  const unsigned hgrid = (unsigned)std::min<uint64_t>((n + 1023) / 1024, (uint64_t)sms * 4);
  {
    ProfScope p(ctx, "rank.hist", s);
    global_hist_kernel<<<std::max(1u, hgrid), 512, 0, s>>>(w.k[0], n, w.hist);
  }
  {
    ProfScope p(ctx, "rank.plan", s);
    plan_kernel<<<1, kThreads, 0, s>>>(w.hist, n, w.plan);
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(downsweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(DownSmem));
    attr_set = true;
  }
  for (int p = 0; p < kPasses; ++p) {
    {
      ProfScope q(ctx, "rank.upsweep", s);
      upsweep_kernel<<<tiles, kThreads, 0, s>>>(w, n, p);
    }
    {
      ProfScope q(ctx, "rank.scan", s);
      tile_scan_kernel<<<kBins, 1024, 0, s>>>(w, tiles, p);
    }
    {
      ProfScope q(ctx, "rank.downsweep", s);
      downsweep_kernel<<<tiles, kThreads, sizeof(DownSmem), s>>>(w, n, p, explicit_vals ? 1 : 0);
    }
  }
  capi::count_launch(2 + 3 * kPasses);
  return cudaGetLastError();
}

}  // namespace

size_t rank_scratch_bytes(uint64_t n, bool with_ids) { return layout(n, with_ids).total; }

uint64_t* rank_key_buffer(tie_ctx* ctx, uint64_t n, cudaStream_t s) {
  const Layout L = layout(n, false);
  char* base = (char*)capi::scratch(ctx, L.total, s);
  return base ? (uint64_t*)(base + L.k0) : nullptr;
}

cudaError_t launch_rank(tie_ctx* ctx, const double* key, const uint64_t* key_bits,
                        const uint64_t* ids, uint64_t n, uint64_t* order, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (n >= (1ull << 32)) return cudaErrorInvalidValue;  // u32 tile-local values
  const Layout L = layout(n, ids != nullptr);
  char* base = (char*)capi::scratch(ctx, L.total, s);
  if (!base) return cudaErrorMemoryAllocation;
  Work w;
  w.k[0] = (uint64_t*)(base + L.k0);
  w.k[1] = (uint64_t*)(base + L.k1);
  w.v[0] = (uint32_t*)(base + L.v0);
  w.v[1] = (uint32_t*)(base + L.v1);
  w.tile_counts = (uint32_t*)(base + L.tc);
  w.hist = (uint32_t*)(base + L.hist);
  w.plan = (Plan*)(base + L.plan);
  w.flag = (int*)(base + L.flag);
  const int sms = sm_count(ctx->device);
  const unsigned egrid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8);

  // transformed keys into k[0] (or into k2 when an id pre-sort needs k[0])
  uint64_t* tkeys = ids ? (uint64_t*)(base + L.k2) : w.k[0];
  if (key_bits) {
    if (ids) cudaMemcpyAsync(tkeys, key_bits, 8 * n, cudaMemcpyDeviceToDevice, s);
    else if (key_bits != w.k[0]) cudaMemcpyAsync(tkeys, key_bits, 8 * n, cudaMemcpyDeviceToDevice, s);
  } else {
    ProfScope p(ctx, "rank.keys", s);
    keys_from_double_kernel<<<egrid, 256, 0, s>>>(key, n, tkeys, ctx->d_err);
    capi::count_launch();
  }

  bool explicit_vals = false;
  if (ids) {
    cudaMemsetAsync(w.flag, 0, sizeof(int), s);
    ids_sorted_kernel<<<egrid, 256, 0, s>>>(ids, n, w.flag);
    capi::count_launch();
    int unsorted = 0;
    cudaMemcpyAsync(&unsorted, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    if (!unsorted) {
      cudaMemcpyAsync(w.k[0], tkeys, 8 * n, cudaMemcpyDeviceToDevice, s);
    } else {
      // stable sort of (id, index) first; then the key sort starts from id order
      copy_ids_kernel<<<egrid, 256, 0, s>>>(ids, n, w.k[0]);
      capi::count_launch();
      if ((e = radix_sort(ctx, w, n, false, sms, s)) != cudaSuccess) return e;
      // sorted ids live in k[final]; stage (key[perm], perm) into the other buffer pair,
      // then move them to slot 0 for the second sort
      gather_by_id_kernel<<<egrid, 256, 0, s>>>(w, n, tkeys, (uint64_t*)(base + L.k3),
                                                (uint32_t*)(base + L.v3), ctx->d_err);
      capi::count_launch();
      cudaMemcpyAsync(w.k[0], base + L.k3, 8 * n, cudaMemcpyDeviceToDevice, s);
      cudaMemcpyAsync(w.v[0], base + L.v3, 4 * n, cudaMemcpyDeviceToDevice, s);
      explicit_vals = true;
    }
  }
  cudaError_t e = radix_sort(ctx, w, n, explicit_vals, sms, s);
  if (e != cudaSuccess) return e;
  {
    ProfScope p(ctx, "rank.finish", s);
    finish_kernel<<<egrid, 256, 0, s>>>(w, n, ids, order, explicit_vals ? 1 : 0);
  }
  capi::count_launch();
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace tie
