// fb_common.cuh — shared device helpers and the kernel argument block.
//
// Data layout in HBM:
//   input f      : row-major, leading dim f_ld, dtype u8/f32/f64, rows_in rows
//                  (rows [halo_top, rows_in - halo_bottom) are the rows to filter)
//   channel planes v : T[band_rows_max][N+1][pitch] (row-interleaved), pitch = round_up(cols + 2W, 32).
//                  v[(o * (N+1) + n) * pitch + pc] is the VERTICALLY filtered channel
//                  c_n = e x^n / sqrt(n!) at band row o and padded column pc, with W
//                  replicate columns on each side (pc <-> image column clamp(pc - W, 0, cols-1)),
//                  so the horizontal pass never leaves the row.  Interleaving the channels
//                  of a row puts all N+1 stores of one output row within a few MB of each
//                  other (immediate-offset stores); kernel 2 fetches per-channel tiles with
//                  a 3-D TMA map {pitch, N+1, rows}.
//   output       : row-major u8/f32/f64, leading dim out_ld.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

namespace fbgpu {

constexpr int kMaxW = 160;                  // largest half-width the kernels accept
constexpr int kMaxTaps = 2 * kMaxW + 1;
constexpr int kFastMaxW = 32;               // largest half-width of the specialised kernels

enum : int { kModeGpa = 0, kModePlain = 1 };
enum : int { kKindBox = 0, kKindGauss = 1 };
enum : int { kFlagFirstNonfinite = 0, kFlagFirstRange = 1, kFlagDegenerate = 2, kFlagNonfiniteOut = 3 };

template <typename T>
struct GpaArgs {
  // input buffer
  const void* f;
  long long f_ld;
  int f_dtype;        // 0 u8, 1 f32, 2 f64
  int rows_in;        // rows in the buffer (incl. halos)
  int cols;
  int halo_top;       // buffer row of output row 0
  int main_end;       // buffer row after the last output row (= rows_in - halo_bottom)
  // Halo rows may live in other allocations (a neighbour rank's band, mapped over CUDA IPC):
  // buffer row b < halo_top starts at element top_off + b * top_ld of f, row b >= main_end at
  // bot_off + (b - main_end) * bot_ld (offsets in samples, relative to f).  A contiguous buffer
  // has top_off = 0, top_ld = bot_ld = f_ld, bot_off = main_end * f_ld.  See sample_row().
  long long top_off, top_ld, bot_off, bot_ld;
  // Global geometry: output row 0 of the buffer is image row row_origin of an image_rows-row
  // image.  Box kernels anchor their running sums (walks / tile segments) to image rows, so a
  // pixel's value does not depend on how the image is split into bands, chunks or ranks.
  long long row_origin;
  int image_rows;
  int lead;           // rows the first box walk / tile of the band starts above the band (anchoring)
  // current row band
  int band_row0;      // first output row of the band
  int band_rows;      // output rows in the band
  // channel planes (workspace)
  T* v;
  long long pitch;    // elements per plane row (= distance between channels of one row)
  long long rstride;  // elements between consecutive rows of one channel = (N+1) * pitch
  int wpad;           // cols + 2W  (valid padded columns)
  int band_max;       // rows the workspace holds
  // filter
  int W;
  int N;
  int mode;           // kModeGpa / kModePlain
  int check;          // validate input samples of the band
  double tc;          // range centre t_c
  double inv_sr;      // 1 / sigma_r
  double sr;          // sigma_r
  double lo, hi;      // declared range
  T norm;             // box: 1/(2W+1)^2, gaussian: 1
  // output
  void* out;
  long long out_ld;
  int out_dtype;      // 0 u8 (quantised as save_pgm does), 1 f32, 2 f64, 3 f32 holding result - tc (kOutF32Centred)
  unsigned long long* flags;
  // fp32 channel constants, 4 per channel m: r_m = fl32(1/sqrt(m)) (0 for m = 0), sqrt(m),
  // and the matched Horner constants h_m = 1/(m r_m), s_m = 1/r_m rounded to fp32
  const float* tab;
  // fp64 Horner constants matched to r_m (see k2f_hpass_horner): tabd[2m] = 1/(m r_m), tabd[2m+1] = 1/r_m.
  // tabd is the set matching the kernel that made the planes: tabd_seq (c_m = c_{m-1} x r_m) or
  // tabd_walk (the box walker's two-step recurrence, r_m replaced by its effective ratio).
  // tabd_tile: the fp32 tile kernel 1 (k1f_gen_vpass) multiplies every order by the same constant,
  // c_m = c_{m-1} (x kappa), r_m = kappa = fl32(1/sqrt(N)): one multiply per sample and channel
  // instead of two, no per-channel constant load (see fb_fast.cuh).
  const double* tabd;
  const double* tabd_seq;
  const double* tabd_walk;
  const double* tabd_tile;
  float kappa;
  T w[kMaxTaps];      // normalised 1-D taps (gaussian)
  // Tap pairs for packed FFMA2 (fp32 fast path): wq[2a] = w[a], wq[2a+1] = w[a-1],
  // a = 0 .. 2W+1, with w[-1] = w[2W+1] = 0 (box: all ones).
  alignas(8) float wq[2 * (2 * kFastMaxW + 2)];
  // the box walker's two-step multipliers q_n = walk_q(n), n < kWalkMaxCh (read as (q_2k, q_2k+1) pairs)
  alignas(8) float walkq[64];
  // The production walker's "Taylor" normalisation (fb_fast.cuh, k1f_box_walk): channel m =
  // e^{-x^2/2} xt^m / m! with xt = x / taylor_s, so kernel 2 needs no per-channel constant:
  // Q = sum_m plane_m y^m with y = x taylor_s, and P = dQ/dx comes from the same Horner pass
  // (two fp64 FMAs per pixel and channel instead of four fp64 operations).
  alignas(8) float walkt[64];  // two-step multipliers 1 / ((n-1) n), walkt[0] = walkt[1] = 1
  float walk_xs;               // 1 / taylor_s (fp32)
  double taylor_s;             // fp64 value of the fp32 scale the walker divided by
  // fp64 kernels (fb_fast64.cuh): every kernel 1 writes Taylor planes, c_m = c_{m-1} (x taylor_r[m])
  // with taylor_r[m] = 1 / (m taylor_s) in fp64 (their rounding, ~m 1e-16, is far below the path's 1e-9)
  const double* taylor_r;
  int walk_rows;      // output rows per thread of the box walker
  int ch_per_cta;     // kernel 1 tile: channels per CTA (blockIdx.z splits the channels of small images)
};

// Rows per box walk (kernel 1, both precisions): long walks amortise the 2W warm-up rows; shorter
// ones (down to 64) while the grid would not give every SM several CTAs.  It depends on the image
// (width, height) only, never on the band, and every length divides 256: a band starting at a
// multiple of 256 image rows walks no rows above itself.
inline int walk_rows(int wpad, int image_rows, int threads) {
  const long long gx = (wpad + threads - 1) / threads;
  int ch = 256;
  while (ch > 64 && gx * ((image_rows + ch - 1) / ch) < 8 * 148) ch /= 2;
  return ch;
}
// Rows between the start of the box walk / tile segment of length `seg` containing the band's
// first row and that row (segments start at image rows that are multiples of seg).
template <typename T>
inline int box_lead(const GpaArgs<T>& a, int seg) {
  return (int)((a.row_origin + a.band_row0) % seg);
}

// Sample offset (relative to f) of the start of buffer row b, clamped to the buffer (the
// reference's edge replication, conv.py:51/62); the halo rows may come from separate buffers.
template <typename T>
__device__ __forceinline__ long long sample_row(const GpaArgs<T>& a, long long b) {
  b = b < 0 ? 0 : (b >= a.rows_in ? a.rows_in - 1 : b);
  return b < a.halo_top ? a.top_off + b * a.top_ld
                        : (b < a.main_end ? b * a.f_ld : a.bot_off + (b - a.main_end) * a.bot_ld);
}

// The fp32 tile kernel 1's channel scale: channel m = e^{-x^2/2} (kappa x)^m with kappa =
// fl32(1/sqrt(N)).  Its largest value over x, at x = sqrt(m), is e^{(m/2)(ln(m/N) - 1)} <= 1 for
// every m <= N, so no order overflows whatever sigma_r is; the fp64 Horner constants (tabd_tile)
// undo kappa^m exactly as they undo the 1/sqrt(m!) of the other kernels.
inline float tile_kappa(int N) { return (float)(1.0 / std::sqrt((double)(N > 1 ? N : 1))); }

// Scale of the Taylor normalisation: the largest value of channel m, at x = sqrt(m), is
// e^{(m/2) ln(N/m) - m ln(beta)} for s = sqrt(e/N) beta: at most e^{N/(2 e beta^2)}, and 1 at m = N.
// beta = max(1, sqrt(N/326)) keeps every order under e^60 in fp32 whatever sigma_r is (beta = 1 for
// the walker's N <= 63: at most e^{11.6}).
inline double taylor_scale(int N) {
  const double n = (double)(N > 1 ? N : 1);
  const double beta = n > 326.0 ? std::sqrt(n / 326.0) : 1.0;
  return std::sqrt(2.718281828459045 / n) * beta;
}

constexpr int kWalkMaxCh = 64;              // channels (N+1) the register-resident box walker holds

// Box walker multiplier q_n: c_n = c_{n-2} x^2 q_n, q_1 = 1 (c_1 = c_0 x), q_n = fl32(1/sqrt((n-1) n)).
__host__ __device__ inline float walk_q(int n) {
  return n <= 0 ? 0.f : (n == 1 ? 1.f : (float)(1.0 / sqrt((double)(n - 1) * (double)n)));
}

__device__ __forceinline__ double load_sample(const void* f, int dt, long long idx) {
  if (dt == 1) return (double)__ldg(reinterpret_cast<const float*>(f) + idx);
  if (dt == 2) return __ldg(reinterpret_cast<const double*>(f) + idx);
  return (double)__ldg(reinterpret_cast<const unsigned char*>(f) + idx);
}

// 8-bit output sample: clamp to [0, 255], round half up — save_pgm / save_image's quantisation
// floor(clip(x, 0, 255) + 0.5) (image.py:96-99, :122-127).  Non-finite values (which make the
// call fail with FB_ERR_NUMERIC anyway) store 0.
__device__ __forceinline__ unsigned quantize_u8(double v) {
  if (!isfinite(v)) return 0u;
  return (unsigned)floor(fmin(fmax(v, 0.0), 255.0) + 0.5);
}

// Results of the fp32 path: the centred result sigma_r P/Q is rounded to float32 once, in the
// epilogue, and t_c is added in fp64 (f32_result).  Its accuracy is fp32; with the
// rounding made explicit, a float64 host output can cross PCIe as the float32 centred result
// (out_dtype kOutF32Centred) and be widened on the host, result = (double)r + t_c, to the very bits
// the float64 device output holds (fb_hostwiden.cuh).  Rounding the CENTRED value keeps the
// reference's shift commutation (test_acceptance.py:130-143) exact on this path too.
constexpr int kOutF32Centred = 3;
__device__ __forceinline__ double f32_result(double centred, double tc) { return (double)(float)centred + tc; }

// `tc` matters for kOutF32Centred only.
__device__ __forceinline__ void store_sample(void* out, int dt, long long idx, double v, double tc = 0.0) {
  if (dt == 2) reinterpret_cast<double*>(out)[idx] = v;
  else if (dt == 1) reinterpret_cast<float*>(out)[idx] = (float)v;
  else if (dt == kOutF32Centred) reinterpret_cast<float*>(out)[idx] = (float)(v - tc);
  else reinterpret_cast<unsigned char*>(out)[idx] = (unsigned char)quantize_u8(v);
}

// Per-kernel timing events.  Inside a CUDA-graph capture (fb_capi.cu replays small repeated
// calls) they are skipped: a captured record only orders work, and timestamped external event
// nodes cost ~13 us per small call; such calls report their kernels' time as one total.
inline cudaError_t record_timing(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive) return cudaSuccess;
  return cudaEventRecord(e, s);
}

template <typename T> __device__ __forceinline__ T gauss_exp(T x);
template <> __device__ __forceinline__ float gauss_exp<float>(float x) { return expf(-0.5f * x * x); }
template <> __device__ __forceinline__ double gauss_exp<double>(double x) { return exp(-0.5 * x * x); }

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

// Record the smallest row-major index of an offending input sample:
// warp-aggregated so a fully invalid image costs one atomic per warp.
__device__ __forceinline__ void flag_min(unsigned long long* slot, bool bad, unsigned long long idx) {
  unsigned mask = __ballot_sync(0xffffffffu, bad);
  if (!mask) return;
  unsigned long long v = bad ? idx : ~0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  if ((threadIdx.x & 31) == (__ffs(mask) - 1)) atomicMin(slot, v);
}

// Validate one input sample (finite first, then declared range), as
// as_image + validate_range do (image.py:35-54).
__device__ __forceinline__ void check_sample(unsigned long long* flags, bool active, double fv,
                                             double lo, double hi, unsigned long long idx) {
  bool nonfinite = active && !isfinite(fv);
  bool outside = active && (fv < lo || fv > hi);
  flag_min(flags + kFlagFirstNonfinite, nonfinite, idx);
  flag_min(flags + kFlagFirstRange, outside, idx);
}

}  // namespace fbgpu
