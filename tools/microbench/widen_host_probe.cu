// Host float32 -> float64 widening rate with T threads (streaming stores), pinned buffers:
// the ceiling of fb_hostwiden.cuh on this box.   nvcc -O3 -std=c++17 -o widen_host_probe widen_host_probe.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include "../../paper_1603_08109_b200/csrc/fb_hostwiden.cuh"
int main(int argc, char** argv) {
  const long long n = 256ll << 20;  // 1 GiB of floats -> 2 GiB of doubles
  float* src; double* dst;
  cudaMallocHost((void**)&src, n * 4); cudaMallocHost((void**)&dst, n * 8);
  for (long long i = 0; i < n; ++i) src[i] = (float)(i & 1023);
  memset(dst, 0, n * 8);
  auto fn = fbgpu::hostwiden::pick_widen();
  printf("hw threads %u, avx512f %d\n", std::thread::hardware_concurrency(), __builtin_cpu_supports("avx512f") ? 1 : 0);
  for (int T : {1, 2, 4, 8, 12, 14, 16}) {
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
        const long long a = n * t / T, b = n * (t + 1) / T;
        for (long long i = a; i < b; i += 16384) fn(src + i, dst + i, std::min<long long>(16384, b - i), 127.5);
        _mm_sfence();
      });
      for (auto& x : th) x.join();
      best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    printf("T=%2d  %.1f ms  (%.1f GB/s read+write)\n", T, best * 1e3, 3.0 * n * 4 / best / 1e9);
  }
  // memcpy baseline (2 GiB copy)
  {
    auto t0 = std::chrono::steady_clock::now();
    memcpy(dst, dst + n / 2, n * 4);
    printf("memcpy 1 GiB 1 thread: %.1f ms\n", std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3);
  }
  return 0;
}
