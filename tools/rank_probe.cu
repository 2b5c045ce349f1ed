// Probe (not part of the product): per-tile phase timeline of the onesweep digit passes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DTIE_RANK_TRACE \
//        -I paper_2604_00499_b200/csrc tools/rank_probe.cu -o tools/_rank_probe
// Prints, per active pass: kernel span, tile start spread, and median/max per-phase times
// (load+rank, look-back+scan, smem scatter, write-out) from %globaltimer stamps.
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

#include "rank.cu"

namespace tie {
namespace capi {
void count_launch(uint64_t) {}
void* scratch(tie_ctx* ctx, size_t bytes, cudaStream_t) {
  if (bytes <= ctx->scratch_bytes) return ctx->scratch;
  cudaFree(ctx->scratch);
  cudaMalloc(&ctx->scratch, bytes);
  ctx->scratch_bytes = bytes;
  return ctx->scratch;
}
}  // namespace capi
ProfScope::ProfScope(tie_ctx*, const char*, cudaStream_t) {}
ProfScope::~ProfScope() {}
}  // namespace tie

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(83.0, 1206.0);
  std::vector<double> key(n);
  for (auto& k : key) k = U(rng);
  tie_ctx ctx;
  cudaMalloc(&ctx.d_err, 8);
  cudaMemset(ctx.d_err, 0xff, 8);
  double* dk;
  uint64_t* dorder;
  cudaMalloc(&dk, 8 * n);
  cudaMalloc(&dorder, 8 * n);
  cudaMemcpy(dk, key.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int it = 0; it < 5; ++it) tie::dev::launch_rank(&ctx, dk, nullptr, n, dorder, s);
  cudaEventRecord(a, s);
  tie::dev::launch_rank(&ctx, dk, nullptr, n, dorder, s);
  cudaEventRecord(b, s);
  cudaStreamSynchronize(s);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("n=%llu rank total %.1f us (%s)\n", (unsigned long long)n, ms * 1e3,
         cudaGetErrorString(cudaGetLastError()));
  static unsigned long long tr[8][8192][6];
  cudaMemcpyFromSymbol(tr, tie::dev::g_rank_trace, sizeof(tr));
  const uint64_t tiles = (n + 4095) / 4096;
  for (int p = 0; p < 8; ++p) {
    unsigned long long t0 = ~0ull, t1 = 0;
    std::vector<double> ph[4], st;
    for (uint64_t t = 0; t < tiles && t < 8192; ++t) {
      const auto* r = tr[p][t];
      if (!r[0] || !r[4]) continue;
      t0 = std::min(t0, r[0]);
      t1 = std::max(t1, r[4]);
    }
    if (t1 == 0) continue;
    for (uint64_t t = 0; t < tiles && t < 8192; ++t) {
      const auto* r = tr[p][t];
      if (!r[0] || !r[4]) continue;
      st.push_back((r[0] - t0) * 1e-3);
      for (int k = 0; k < 4; ++k) ph[k].push_back((r[k + 1] - r[k]) * 1e-3);
    }
    auto med = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v[v.size() / 2];
    };
    auto mx = [](const std::vector<double>& v) { return *std::max_element(v.begin(), v.end()); };
    printf("pass %d: span %.1f us | tile start med %.1f max %.1f | load+rank %.2f/%.2f  "
           "lookback+scan %.2f/%.2f  smem %.2f/%.2f  write %.2f/%.2f (med/max us)\n",
           p, (t1 - t0) * 1e-3, med(st), mx(st), med(ph[0]), mx(ph[0]), med(ph[1]), mx(ph[1]),
           med(ph[2]), mx(ph[2]), med(ph[3]), mx(ph[3]));
  }
  return 0;
}
