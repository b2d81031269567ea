// fb_hostwiden.cuh — host side of the fp32-precision pipeline for float64 host outputs.
//
// The reference returns float64 (engine.py:80).  The fp32 path's results are fp32 values, so a
// host-resident float64 output needs only 4 of its 8 bytes per pixel over PCIe: kernel 2 writes
// the float32 centred result (kOutF32Centred), each row chunk goes device -> pinned ring slot, and
// a pool of host threads writes (double)r + t_c into the caller's float64 buffer -- the bits the
// float64 device output holds (fb_common.cuh: f32_result) -- while the next chunks are in flight.  For c4 that halves the D2H bytes (2 GiB -> 1 GiB per 16384^2 image),
// which is what bounded the end-to-end rate (profiles/r01_pcie_probe.txt).
//
// Protocol: the float32 rows go device -> their place in a pinned staging area that holds the whole
// call's float32 output (no slot reuse, so the copy stream never waits for the host), in pieces of
// a few MiB with an event after each.  A dispatcher thread waits for the piece events in order and
// hands each piece to the workers.  (A first version used cudaLaunchHostFunc hand-offs and a
// six-slot ring: two host functions per chunk put ~0.7 ms of dispatch latency per chunk on the
// copy stream, 41 ms per c4 call.)
#pragma once
#include <cuda_runtime.h>
#include <immintrin.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace fbgpu {
namespace hostwiden {

// d[i] = (double)s[i] + add   (add = t_c: the device sends centred results, fb_common.cuh f32_result)
__attribute__((target("avx512f"))) inline void widen_row_avx512(const float* s, double* d, long long n, double add) {
  long long i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 63)) {
    d[i] = (double)s[i] + add;
    ++i;
  }
  const __m512d va = _mm512_set1_pd(add);
  for (; i + 8 <= n; i += 8) _mm512_stream_pd(d + i, _mm512_add_pd(_mm512_cvtps_pd(_mm256_loadu_ps(s + i)), va));
  for (; i < n; ++i) d[i] = (double)s[i] + add;
}
__attribute__((target("avx2"))) inline void widen_row_avx2(const float* s, double* d, long long n, double add) {
  long long i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31)) {
    d[i] = (double)s[i] + add;
    ++i;
  }
  const __m256d va = _mm256_set1_pd(add);
  for (; i + 4 <= n; i += 4) _mm256_stream_pd(d + i, _mm256_add_pd(_mm256_cvtps_pd(_mm_loadu_ps(s + i)), va));
  for (; i < n; ++i) d[i] = (double)s[i] + add;
}
inline void widen_row_scalar(const float* s, double* d, long long n, double add) {
  for (long long i = 0; i < n; ++i) d[i] = (double)s[i] + add;
}
using widen_fn = void (*)(const float*, double*, long long, double);
inline widen_fn pick_widen() {
  if (__builtin_cpu_supports("avx512f")) return widen_row_avx512;
  if (__builtin_cpu_supports("avx2")) return widen_row_avx2;
  return widen_row_scalar;
}

// rows [0, rows) of a dense float32 block (ld = cols) into a float64 image with leading dimension dst_ld
struct Task {
  const float* src;
  double* dst;
  long long rows, cols, dst_ld;
  double add;
  long long t_submit = 0;
};

class Pool {
 public:
  Pool(int threads, int device) : fn_(pick_widen()), device_(device) {
    for (int t = 0; t < threads; ++t) workers_.emplace_back([this] { run(); });
    dispatcher_ = std::thread([this] { dispatch_loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_work_.notify_all();
    cv_disp_.notify_all();
    for (auto& w : workers_) w.join();
    dispatcher_.join();
    if (stage_) cudaFreeHost(stage_);
  }
  int threads() const { return (int)workers_.size(); }

  // Pinned staging of at least `bytes` (grown between calls only: no work pending).
  cudaError_t reserve(size_t bytes) {
    if (bytes <= stage_bytes_) return cudaSuccess;
    if (stage_) cudaFreeHost(stage_);
    stage_ = nullptr;
    stage_bytes_ = 0;
    const size_t rounded = (bytes + (1u << 21) - 1) >> 21 << 21;
    cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&stage_), rounded);
    if (e != cudaSuccess) return e;
    stage_bytes_ = rounded;
    return cudaSuccess;
  }
  float* stage(size_t byte_offset) const { return reinterpret_cast<float*>(stage_ + byte_offset); }

  // `landed` has been recorded after the copy of the piece: widen it once the event completes
  void dispatch(cudaEvent_t landed, const Task& t) {
    {
      std::lock_guard<std::mutex> lk(m_);
      dq_.push_back({landed, t});
      ++pending_;  // the piece itself, until its parts are queued
    }
    cv_disp_.notify_one();
  }
  // a piece has landed in the staging area: split its rows over the workers
  void submit(const Task& t) {
    if (trace_first_ == 0) trace_first_ = now_ns();
    const int parts = (int)std::max<long long>(1, std::min<long long>(threads(), t.rows));
    const long long per = (t.rows + parts - 1) / parts;
    {
      std::lock_guard<std::mutex> lk(m_);
      --pending_;
      for (long long r = 0; r < t.rows; r += per) {
        Task p = t;
        p.src = t.src + r * t.cols;
        p.dst = t.dst + r * t.dst_ld;
        p.rows = std::min(per, t.rows - r);
        p.t_submit = now_ns();
        q_.push_back(p);
        ++pending_;
      }
    }
    cv_work_.notify_all();
  }
  // every dispatched piece is widened
  void wait_all() {
    std::unique_lock<std::mutex> lk(m_);
    cv_done_.wait(lk, [&] { return pending_ == 0; });
  }

  static long long now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  // (FBGPU_WIDEN_TRACE) first hand-off .. last piece done, summed piece times and queue waits; resets
  void trace_report(long long t_call0, long long t_sync, long long t_end) {
    std::lock_guard<std::mutex> lk(m_);
    fprintf(stderr, "[widen] pieces %lld  first submit +%.2f ms  last done +%.2f ms  stream sync +%.2f ms  return +%.2f ms  "
            "busy sum %.2f ms  mean queue wait %.3f ms\n", trace_pieces_, (trace_first_ - t_call0) * 1e-6,
            (trace_last_ - t_call0) * 1e-6, (t_sync - t_call0) * 1e-6, (t_end - t_call0) * 1e-6, trace_busy_ * 1e-6,
            trace_pieces_ ? trace_wait_ * 1e-6 / trace_pieces_ : 0.0);
    trace_first_ = trace_last_ = trace_busy_ = trace_wait_ = trace_pieces_ = 0;
  }

 private:
  void dispatch_loop() {
    cudaSetDevice(device_);
    for (;;) {
      std::pair<cudaEvent_t, Task> d;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_disp_.wait(lk, [&] { return stop_ || !dq_.empty(); });
        if (dq_.empty()) return;
        d = dq_.front();
        dq_.pop_front();
      }
      if (cudaEventSynchronize(d.first) == cudaSuccess) {
        submit(d.second);
      } else {  // the call fails with the same error at its own synchronisation
        bool last;
        {
          std::lock_guard<std::mutex> lk(m_);
          last = --pending_ == 0;
        }
        if (last) cv_done_.notify_all();
      }
    }
  }
  void run() {
    for (;;) {
      Task t;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_work_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        t = q_.front();
        q_.pop_front();
      }
      const long long t0 = now_ns();
      for (long long r = 0; r < t.rows; ++r) fn_(t.src + r * t.cols, t.dst + r * t.dst_ld, t.cols, t.add);
      _mm_sfence();  // the streaming stores are visible before the piece counts as done
      const long long t1 = now_ns();
      bool last;
      {
        std::lock_guard<std::mutex> lk(m_);
        last = --pending_ == 0;
        trace_busy_ += t1 - t0;
        trace_last_ = t1;
        trace_wait_ += t0 - t.t_submit;
        ++trace_pieces_;
      }
      if (last) cv_done_.notify_all();
    }
  }

  widen_fn fn_;
  std::vector<std::thread> workers_;
  std::mutex m_;
  std::condition_variable cv_work_, cv_done_, cv_disp_;
  std::deque<Task> q_;
  std::deque<std::pair<cudaEvent_t, Task>> dq_;
  std::thread dispatcher_;
  int device_ = 0;
  long long pending_ = 0;
  bool stop_ = false;
  long long trace_first_ = 0, trace_last_ = 0, trace_busy_ = 0, trace_wait_ = 0, trace_pieces_ = 0;
  char* stage_ = nullptr;
  size_t stage_bytes_ = 0;
};

// Host-thread count: FBGPU_HOST_THREADS, else the hardware threads less two (the caller's and the
// CUDA runtime's), capped at 16.  While the GPU side bounded the call, 6, 10 and 14 threads
// measured the same; with wave-sized chunks the threads bound it: 4 / 8 / 14 threads = 44.0 / 35.7 /
// 33.4 ms per c4 call on a 16-core host (profiles/r02_hostwiden.md).  0 disables the float32
// transfer (float64 rows cross PCIe instead).
inline int configured_threads() {
  if (const char* e = std::getenv("FBGPU_HOST_THREADS")) return std::max(0, std::min(64, atoi(e)));
  const int hw = (int)std::thread::hardware_concurrency();
  return std::max(1, std::min(16, hw - 2));
}

}  // namespace hostwiden
}  // namespace fbgpu

namespace fbgpu {
namespace hostwiden {
// Largest pinned staging area (FBGPU_WIDEN_MAX_MB, default 4096): a call whose float32 output is
// larger sends float64 rows over PCIe instead.
inline size_t max_stage_bytes() {
  static const size_t v = [] {
    const char* e = std::getenv("FBGPU_WIDEN_MAX_MB");
    return (size_t)(e ? std::max(0, atoi(e)) : 4096) << 20;
  }();
  return v;
}
}  // namespace hostwiden
}  // namespace fbgpu

namespace fbgpu {
namespace hostwiden {
// Bytes per device -> staging copy (FBGPU_WIDEN_PIECE_KB, default 8192: 32 / 8 / 2 / 1 / 0.5 MiB pieces
// measured 38.6 / 36.6 / 37.8 / 38.6 / 43.8 ms per c4 call).
inline size_t piece_bytes() {
  static const size_t v = [] {
    const char* e = std::getenv("FBGPU_WIDEN_PIECE_KB");
    return (size_t)(e ? std::max(64, atoi(e)) : 8192) << 10;
  }();
  return v;
}
}  // namespace hostwiden
}  // namespace fbgpu
