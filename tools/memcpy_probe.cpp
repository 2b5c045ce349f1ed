// host memcpy bandwidth into pinned memory, 1..16 threads (development probe for the
// pageable e2e path): g++ -O2 -pthread memcpy_probe.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t n = 20u << 20;
  std::vector<char> src(n, 1);
  char* dst = nullptr;
  cudaHostAlloc((void**)&dst, n, cudaHostAllocMapped);
  std::memset(dst, 0, n);
  for (int T : {1, 2, 4, 8, 16}) {
    double best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      const size_t per = n / T;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] { std::memcpy(dst + t * per, src.data() + t * per, per); });
      for (auto& x : th) x.join();
      double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      if (us < best) best = us;
    }
    std::printf("threads %2d: 20 MB in %.0f us = %.1f GB/s (incl. thread spawn)\n", T, best, n / best / 1e3);
  }
}
