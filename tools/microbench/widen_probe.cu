// widen_probe.cu — host f32 -> f64 widening bandwidth on the GPU box (pinned buffers), alone and
// while a 1 GiB D2H copy runs: is "D2H fp32 + host widening" faster than "D2H fp64"?
// nvcc -O3 -Xcompiler -O3,-march=native,-pthread -o widen_probe widen_probe.cu
#include <cuda_runtime.h>
#include <immintrin.h>

#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

static void widen(const float* in, double* out, size_t n, bool nt) {
  size_t i = 0;
  if (nt) {
    for (; i + 8 <= n; i += 8) {
      __m256 v = _mm256_loadu_ps(in + i);
      _mm256_stream_pd(out + i, _mm256_cvtps_pd(_mm256_castps256_ps128(v)));
      _mm256_stream_pd(out + i + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(v, 1)));
    }
    _mm_sfence();
  }
  for (; i < n; ++i) out[i] = in[i];
}

static double run(const float* in, double* out, size_t n, int threads, bool nt) {
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  size_t per = (n / threads + 7) & ~size_t(7);
  for (int t = 0; t < threads; ++t) {
    size_t a = std::min(n, t * per), b = std::min(n, a + per);
    th.emplace_back(widen, in + a, out + a, b - a, nt);
  }
  for (auto& x : th) x.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
  const size_t n = 1ull << 28;  // 268 M samples: 1 GiB in, 2 GiB out
  float* in;
  double* out;
  float* in2;
  void* dev;
  cudaMallocHost(&in, n * 4);
  cudaMallocHost(&out, n * 8);
  cudaMallocHost(&in2, n * 4);
  cudaMalloc(&dev, n * 8);
  for (size_t i = 0; i < n; ++i) in[i] = (float)(i % 1000) * 0.25f;
  memset(out, 0, n * 8);
  memset(in2, 0, n * 4);
  printf("threads hw=%u\n", std::thread::hardware_concurrency());
  for (int nt = 0; nt < 2; ++nt)
    for (int t : {1, 4, 8, 12, 16}) {
      run(in, out, n, t, nt);
      double s = run(in, out, n, t, nt);
      printf("widen nt=%d threads=%2d: %.1f ms  (%.1f GB/s of f64 output)\n", nt, t, s * 1e3, n * 8 / s / 1e9);
    }
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t bytes : {n * 4, n * 8}) {
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(bytes == n * 4 ? (void*)in2 : (void*)out, dev, bytes, cudaMemcpyDeviceToHost, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("D2H %zu MiB alone: %.1f ms (%.1f GB/s)\n", bytes >> 20, ms, bytes / ms / 1e6);
  }
  for (int t : {8, 12, 16}) {  // widening while a 1 GiB D2H lands in another pinned buffer
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(in2, dev, n * 4, cudaMemcpyDeviceToHost, st);
    cudaEventRecord(e1, st);
    double s = run(in, out, n, t, true);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("concurrent: widen threads=%d %.1f ms, D2H 1 GiB %.1f ms\n", t, s * 1e3, ms);
  }
  return 0;
}
