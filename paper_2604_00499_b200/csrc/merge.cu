// K-way merge of sorted (score, id) runs -- the final step of the sharded score+rank
// (SURVEY.md 8e): after the NCCL all-gather, G runs, each sorted by (score asc, id asc) (the
// reference heap's order, proj/src/sched.cpp:28-31), become the global dispatch order.
//
// A tree of 2-way merge-path rounds (ceil(log2 G) passes over the data instead of a full
// re-sort): every round merges run pairs (2r, 2r+1).  Each CTA owns a tile of kTile outputs of
// one pair; its merge-path split (the number i of A elements among the pair's first d
// outputs: the largest i with A[i-1] < B[d-i], found by binary search on the diagonal) bounds
// the A and B slices it needs.  The slices are staged in shared memory and every element's
// output slot is its index in its own slice plus the count of smaller elements in the other
// slice (binary search; (key, id) is a strict total order because ids are unique), then the
// tile is written out coalesced.  Keys are the order-preserving u64 image of the scores.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "tie_internal.cuh"

namespace tie {
namespace dev {
namespace {

constexpr int kMergeThreads = 256;
constexpr int kTile = 2048;  // outputs per CTA
constexpr int kMaxPairs = 64;

struct Pairs {
  uint64_t a_off[kMaxPairs], a_len[kMaxPairs], b_off[kMaxPairs], b_len[kMaxPairs];
  uint64_t out_off[kMaxPairs];
  uint32_t tile0[kMaxPairs + 1];  // first tile of each pair (prefix)
  int n;
};

__device__ __forceinline__ bool less_ki(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ uint64_t order_bits_d(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// compact the G padded runs [G][stride] into one array with u64 keys
__global__ void pack_runs_kernel(const double* __restrict__ key, const uint64_t* __restrict__ id,
                                 uint64_t stride, const uint64_t* __restrict__ off, int G,
                                 uint64_t* __restrict__ ko, uint64_t* __restrict__ io) {
  for (int g = 0; g < G; ++g) {
    const uint64_t len = off[g + 1] - off[g];
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < len;
         t += (uint64_t)gridDim.x * blockDim.x) {
      ko[off[g] + t] = order_bits_d(key[(uint64_t)g * stride + t]);
      io[off[g] + t] = id[(uint64_t)g * stride + t];
    }
  }
}

// A elements among the first d outputs of merge(A, B)
__device__ __forceinline__ uint64_t merge_path(const uint64_t* ka, const uint64_t* ia, uint64_t la,
                                               const uint64_t* kb, const uint64_t* ib, uint64_t lb,
                                               uint64_t d) {
  uint64_t lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;  // A[mid] vs B[d - 1 - mid]
    if (less_ki(ka[mid], ia[mid], kb[d - 1 - mid], ib[d - 1 - mid])) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// merge-path cut (A elements before the tile start) of every tile boundary of a round, one
// thread each: the dependent binary searches run once, all in parallel
__global__ void merge_cuts_kernel(const Pairs P, const uint64_t* __restrict__ kin,
                                  const uint64_t* __restrict__ iin, uint32_t tiles,
                                  uint64_t* __restrict__ cuts) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > tiles) return;
  int p = 0;
  while (p + 1 < P.n && t >= P.tile0[p + 1]) ++p;
  if (t == tiles) p = P.n - 1;
  const uint64_t la = P.a_len[p], lb = P.b_len[p];
  const uint64_t d = min((uint64_t)(t - P.tile0[p]) * kTile, la + lb);
  cuts[t] = merge_path(kin + P.a_off[p], iin + P.a_off[p], la, kin + P.b_off[p],
                       iin + P.b_off[p], lb, d);
}

__global__ void __launch_bounds__(kMergeThreads) merge_pairs_kernel(
    const Pairs P, const uint64_t* __restrict__ kin, const uint64_t* __restrict__ iin,
    uint64_t* __restrict__ kout, uint64_t* __restrict__ iout, uint64_t* __restrict__ ids_final,
    const uint64_t* __restrict__ cuts) {
  __shared__ uint64_t sk[kTile], si[kTile];
  constexpr int kPer = kTile / kMergeThreads;
  const uint32_t tile = blockIdx.x;
  int p = 0;
  while (p + 1 < P.n && tile >= P.tile0[p + 1]) ++p;
  const uint64_t la = P.a_len[p], lb = P.b_len[p];
  const uint64_t* ka = kin + P.a_off[p];
  const uint64_t* ia = iin + P.a_off[p];
  const uint64_t* kb = kin + P.b_off[p];
  const uint64_t* ib = iin + P.b_off[p];
  const uint64_t d0 = (uint64_t)(tile - P.tile0[p]) * kTile;
  const uint64_t d1 = min(d0 + kTile, la + lb);
  const uint64_t a0 = cuts[tile];
  // the next tile's cut, or the pair's end when this is its last tile
  const uint64_t a1 = (tile + 1 < P.tile0[p + 1]) ? cuts[tile + 1] : la;
  const uint64_t b0 = d0 - a0;
  const uint32_t na = (uint32_t)(a1 - a0), m = (uint32_t)(d1 - d0);
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const uint32_t t = threadIdx.x + u * kMergeThreads;
    if (t < m) {
      sk[t] = t < na ? ka[a0 + t] : kb[b0 + t - na];
      si[t] = t < na ? ia[a0 + t] : ib[b0 + t - na];
    }
  }
  __syncthreads();
  // merge path inside the tile: thread t produces outputs [t*kPer, t*kPer + kPer) -- one
  // binary search for its cut, then a sequential merge of kPer elements
  const uint32_t nb = m - na;
  const uint32_t d = min((uint32_t)(threadIdx.x * kPer), m);
  uint32_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;  // A[mid] vs B[d - 1 - mid]
    if (less_ki(sk[mid], si[mid], sk[na + d - 1 - mid], si[na + d - 1 - mid])) lo = mid + 1;
    else hi = mid;
  }
  uint32_t ai = lo, bi = d - lo;
  uint64_t rk[kPer], ri[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    if (d + u >= m) break;
    const bool take_a =
        bi >= nb || (ai < na && less_ki(sk[ai], si[ai], sk[na + bi], si[na + bi]));
    const uint32_t src = take_a ? ai : na + bi;
    rk[u] = sk[src];
    ri[u] = si[src];
    ai += take_a ? 1u : 0u;
    bi += take_a ? 0u : 1u;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    if (d + u < m) {
      sk[d + u] = rk[u];
      si[d + u] = ri[u];
    }
  }
  __syncthreads();
  const uint64_t o = P.out_off[p] + d0;
  for (uint32_t t = threadIdx.x; t < m; t += kMergeThreads) {
    if (ids_final) {
      ids_final[o + t] = si[t];
    } else {
      kout[o + t] = sk[t];
      iout[o + t] = si[t];
    }
  }
}

// copy an unpaired run into the next round's buffer
__global__ void copy_run_kernel(const uint64_t* __restrict__ kin, const uint64_t* __restrict__ iin,
                                uint64_t off_in, uint64_t len, uint64_t* __restrict__ kout,
                                uint64_t* __restrict__ iout, uint64_t off_out,
                                uint64_t* __restrict__ ids_final) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < len;
       t += (uint64_t)gridDim.x * blockDim.x) {
    if (ids_final) {
      ids_final[off_out + t] = iin[off_in + t];
    } else {
      kout[off_out + t] = kin[off_in + t];
      iout[off_out + t] = iin[off_in + t];
    }
  }
}

}  // namespace

// keys / ids: G padded runs [G][stride] on the device, run g valid for lens[g] (host array);
// each run sorted by (key, id).  out_ids: the merged ids (sum of lens).
cudaError_t launch_merge_runs(tie_ctx* ctx, const double* keys, const uint64_t* ids, int G,
                              uint64_t stride, const uint64_t* lens, uint64_t* out_ids,
                              cudaStream_t s) {
  if (G <= 0) return cudaSuccess;
  std::vector<uint64_t> off(G + 1, 0);
  for (int g = 0; g < G; ++g) off[g + 1] = off[g] + lens[g];
  const uint64_t total = off[G];
  if (total == 0) return cudaSuccess;
  // scratch: 2 x (keys, ids) ping-pong + run offsets
  const size_t bytes = 4 * 8 * total + 8 * (G + 1) + 8 * (total / kTile + 2 * G + 2) + 1024;
  char* base = (char*)capi::scratch(ctx, bytes, s);
  if (!base) return cudaErrorMemoryAllocation;
  uint64_t* k[2] = {(uint64_t*)base, (uint64_t*)base + total};
  uint64_t* id[2] = {(uint64_t*)base + 2 * total, (uint64_t*)base + 3 * total};
  uint64_t* d_off = (uint64_t*)base + 4 * total;
  uint64_t* d_cuts = d_off + G + 1;  // tiles + 1 <= total / kTile + G + 1
  cudaMemcpyAsync(d_off, off.data(), 8 * (G + 1), cudaMemcpyHostToDevice, s);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const unsigned g_stream = (unsigned)std::max(1, sms) * 8;
  {
    ProfScope prof(ctx, "merge.pack", s);
    pack_runs_kernel<<<g_stream, 256, 0, s>>>(keys, ids, stride, d_off, G, k[0], id[0]);
    capi::count_launch();
  }
  if (G == 1) {
    copy_run_kernel<<<g_stream, 256, 0, s>>>(k[0], id[0], 0, total, nullptr, nullptr, 0, out_ids);
    capi::count_launch();
    return cudaGetLastError();
  }
  std::vector<uint64_t> roff(off.begin(), off.end() - 1), rlen(lens, lens + G);
  int cur = 0;
  while (roff.size() > 1) {
    const int nr = (int)roff.size();
    const bool last = nr <= 2;
    Pairs P{};
    std::vector<uint64_t> noff, nlen;
    uint64_t out = 0;
    uint32_t tiles = 0;
    for (int r = 0; r + 1 < nr; r += 2) {
      if (P.n == kMaxPairs) return cudaErrorInvalidValue;
      P.a_off[P.n] = roff[r];
      P.a_len[P.n] = rlen[r];
      P.b_off[P.n] = roff[r + 1];
      P.b_len[P.n] = rlen[r + 1];
      P.out_off[P.n] = out;
      P.tile0[P.n] = tiles;
      const uint64_t m = rlen[r] + rlen[r + 1];
      tiles += (uint32_t)((m + kTile - 1) / kTile);
      noff.push_back(out);
      nlen.push_back(m);
      out += m;
      ++P.n;
    }
    P.tile0[P.n] = tiles;
    {
      ProfScope prof(ctx, "merge.round", s);
      if (tiles) {
        merge_cuts_kernel<<<(tiles + 1 + 255) / 256, 256, 0, s>>>(P, k[cur], id[cur], tiles,
                                                                  d_cuts);
        merge_pairs_kernel<<<tiles, kMergeThreads, 0, s>>>(
            P, k[cur], id[cur], k[cur ^ 1], id[cur ^ 1], last ? out_ids : nullptr, d_cuts);
        capi::count_launch(2);
      }
      if (nr & 1) {  // odd run out: carried over
        copy_run_kernel<<<g_stream, 256, 0, s>>>(k[cur], id[cur], roff[nr - 1], rlen[nr - 1],
                                                 k[cur ^ 1], id[cur ^ 1], out, nullptr);
        capi::count_launch();
        noff.push_back(out);
        nlen.push_back(rlen[nr - 1]);
      }
    }
    roff.swap(noff);
    rlen.swap(nlen);
    cur ^= 1;
  }
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace tie
