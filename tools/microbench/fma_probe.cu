// Probe: FP32 FFMA vs packed FFMA2 vs FP64 DFMA throughput, smem LDS bandwidth.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void ffma_k(float* out, int iters, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void ffma2_k(float* out, int iters, float a, float b) {
  unsigned long long acc[CHAINS];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&av);
  unsigned long long B = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) {
    float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    acc[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(A), "l"(B));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) {
    float2 v = *reinterpret_cast<float2*>(&acc[i]);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_k(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// smem read bandwidth: each thread reads LDS.32 at conflict-free addresses
__global__ void lds_k(float* out, int iters) {
  __shared__ float buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
  __syncthreads();
  float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    s0 += buf[(idx) & 4095];
    s1 += buf[(idx + 256) & 4095];
    s2 += buf[(idx + 512) & 4095];
    s3 += buf[(idx + 768) & 4095];
    idx += 1024;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
__global__ void lds128_k(float* out, int iters) {
  __shared__ float4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 s = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    float4 v0 = buf[idx & 2047];
    float4 v1 = buf[(idx + 256) & 2047];
    s.x += v0.x + v1.x; s.y += v0.y + v1.y; s.z += v0.z + v1.z; s.w += v0.w + v1.w;
    idx += 512;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s.x + s.y + s.z + s.w;
}
__global__ void shfl_k(float* out, int iters) {
  float s = threadIdx.x, t = 0;
  for (int it = 0; it < iters; ++it) {
    float a = __shfl_down_sync(0xffffffffu, s, 1);
    float b = __shfl_down_sync(0xffffffffu, s + 1.f, 2);
    float c = __shfl_down_sync(0xffffffffu, s + 2.f, 3);
    float d = __shfl_down_sync(0xffffffffu, s + 3.f, 4);
    t += a + b + c + d;
    s += 1.f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("name=%s sms=%d l2=%d MB smem/sm=%zu KB regs/sm=%d clock=%d MHz cc=%d.%d\n", p.name,
         p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerMultiprocessor >> 10,
         p.regsPerMultiprocessor, clk / 1000, p.major, p.minor);
  int sms = p.multiProcessorCount;
  float* d; cudaMalloc(&d, 64 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256, iters = 20000;
  auto timeit = [&](auto launch, double ops, const char* name, const char* unit) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-10s %8.2f %s  (%.3f ms)  err=%s\n", name, 5 * ops / (ms * 1e-3) / 1e12, unit, ms / 5,
           cudaGetErrorString(cudaGetLastError()));
  };
  double nthr = (double)blocks * threads;
  timeit([&] { ffma_k<16><<<blocks, threads>>>(d, iters, 0.999f, 1e-4f); }, nthr * iters * 16 * 2, "ffma", "TFLOP/s");
  timeit([&] { ffma2_k<8><<<blocks, threads>>>(d, iters, 0.999f, 1e-4f); }, nthr * iters * 16 * 2, "ffma2", "TFLOP/s");
  timeit([&] { ffma2_k<16><<<blocks, threads>>>(d, iters, 0.999f, 1e-4f); }, nthr * iters * 32 * 2, "ffma2x16", "TFLOP/s");
  timeit([&] { dfma_k<16><<<blocks, threads>>>((double*)d, iters / 4, 0.999, 1e-4); }, nthr * iters / 4 * 16 * 2, "dfma", "TFLOP/s");
  timeit([&] { lds_k<<<blocks, threads>>>(d, iters); }, nthr * iters * 4 * 4, "lds32", "TB/s");
  timeit([&] { lds128_k<<<blocks, threads>>>(d, iters); }, nthr * iters * 2 * 16, "lds128", "TB/s");
  timeit([&] { shfl_k<<<blocks, threads>>>(d, iters); }, nthr * iters * 4 * 4, "shfl", "TB/s");
  return 0;
}
