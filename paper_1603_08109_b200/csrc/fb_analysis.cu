// fb_analysis.cu — the data-parallel parts of the reference's error metrology and its direct
// convolution oracle, as device kernels:
//
//   k_kernel_error_sup  kernel_error_sup (analysis.py:70-103): worst kernel error over the integer
//                       grid t, tau in {-T..T}, one thread per grid point, tail series in fp64
//   k_error_stats       linf_error / mse_db (analysis.py:33-46): max |a - b| and sum (a - b)^2 in
//                       fp64, with as_image's finiteness check (image.py:35-42) on both inputs
//   k_convolve_direct   convolve_direct (conv.py:83-96): the literal O(W^2) double sum with the 2-D
//                       weight table, accumulated in the reference's order without contraction
//                       (bit-identical to the numpy loop)
//
// All three are small next to the filter; they exist so the tools that judge the filter (the
// `compare` / `kernel-error` commands, full-size error reports) run where the images already are.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "fb_analysis.cuh"
#include "fb_common.cuh"

namespace fbgpu {

// ---------------------------------------------------------------------------- kernel error
// Per grid point (t, tau) = (g_i, g_j), g = -F..F:
//   x = t tau / sigma_r^2,  prefactor = exp(-(t^2 + tau^2) / (2 sigma_r^2)),
//   first tail term sign(x)^N exp(N log|x| - lgamma(N + 1)), then term *= x / n while n grows,
// exactly the reference's arithmetic (analysis.py:85-103).  The reference stops all points
// together once every |term| < 1e-30 max(1, max|total|) past n > max|x|; here each point stops on
// its own |term| < 1e-30 max(1, |total|) (never earlier than the reference's global test could for
// that point's leading terms), capped at the same 5 max|x| + 2000 iterations.  Omitted terms are
// < 1e-30 relative, far below the fp64 rounding of the sum.
__global__ void __launch_bounds__(256) k_kernel_error_sup(int F, int N, double sr2, double lgam, double xmax,
                                                          long long max_iters, unsigned long long* out_bits) {
  const int n_side = 2 * F + 1;
  const long long total_pts = (long long)n_side * n_side;
  double best = 0.0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total_pts;
       p += (long long)gridDim.x * blockDim.x) {
    const double t = (double)(int)(p / n_side - F);
    const double tau = (double)(int)(p % n_side - F);
    const double x = (t * tau) / sr2;
    const double pref = exp(-__dadd_rn(__dmul_rn(t, t), __dmul_rn(tau, tau)) / (2.0 * sr2));
    double term = 0.0;
    if (x != 0.0) {
      const double mag = exp(__dsub_rn(__dmul_rn((double)N, log(fabs(x))), lgam));
      term = (x < 0.0 && (N & 1)) ? -mag : mag;
    }
    double tot = term;
    double n = (double)N;
    for (long long it = 0; it < max_iters && term != 0.0; ++it) {
      n += 1.0;
      term = __ddiv_rn(__dmul_rn(term, x), n);
      tot = __dadd_rn(tot, term);
      if (n > xmax && fabs(term) < 1e-30 * fmax(1.0, fabs(tot))) break;
    }
    best = fmax(best, fabs(__dmul_rn(pref, tot)));
  }
  // block max; values are >= 0, so their bit patterns order like unsigned integers
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  __shared__ double wmax[8];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x / 32] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w) best = fmax(best, wmax[w]);
    atomicMax(out_bits, (unsigned long long)__double_as_longlong(best));
  }
}

int launch_kernel_error_sup(cudaStream_t s, int sms, int F, int N, double sigma_r, unsigned long long* out_bits) {
  const double sr2 = sigma_r * sigma_r;
  const double xmax = ((double)F * (double)F) / sr2;
  const long long max_iters = (long long)(5.0 * xmax + 2000.0);
  const long long pts = (long long)(2 * F + 1) * (2 * F + 1);
  long long blocks = (pts + 255) / 256;
  if (blocks > 8ll * sms) blocks = 8ll * sms;
  k_kernel_error_sup<<<(int)blocks, 256, 0, s>>>(F, N, sr2, std::lgamma((double)N + 1.0), xmax, max_iters,
                                                 out_bits);
  return cudaGetLastError() == cudaSuccess ? 0 : 6;
}

// ---------------------------------------------------------------------------- image differences
// One fixed grid (deterministic): block b writes partial[2b] = max |a - b|, partial[2b+1] =
// sum (a - b)^2 over its grid-stride share; the host combines the partials in block order.
// Non-finite samples are flagged (first row-major index per image) as as_image does.
__global__ void __launch_bounds__(256) k_error_stats(const void* a, long long lda, int dta, const void* b,
                                                     long long ldb, int dtb, int rows, int cols, double* partial,
                                                     unsigned long long* flags_a, unsigned long long* flags_b) {
  const long long total = (long long)rows * cols;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double mx = 0.0, ss = 0.0;
  for (long long base = (long long)blockIdx.x * blockDim.x; base < total; base += stride) {
    const long long i = base + threadIdx.x;
    const bool act = i < total;
    double va = 0.0, vb = 0.0;
    if (act) {
      const long long r = i / cols, c = i - r * cols;
      va = load_sample(a, dta, r * lda + c);
      vb = load_sample(b, dtb, r * ldb + c);
    }
    const bool bad_a = act && !isfinite(va), bad_b = act && !isfinite(vb);
    flag_min(flags_a, bad_a, (unsigned long long)i);
    flag_min(flags_b, bad_b, (unsigned long long)i);
    if (act && !bad_a && !bad_b) {
      const double d = __dsub_rn(va, vb);
      mx = fmax(mx, fabs(d));
      ss = __dadd_rn(ss, __dmul_rn(d, d));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  __shared__ double wm[8], ws[8];
  if ((threadIdx.x & 31) == 0) {
    wm[threadIdx.x / 32] = mx;
    ws[threadIdx.x / 32] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w) {
      mx = fmax(mx, wm[w]);
      ss += ws[w];
    }
    partial[2 * blockIdx.x] = mx;
    partial[2 * blockIdx.x + 1] = ss;
  }
}

int error_stats_blocks(int sms) { return 4 * sms; }

int launch_error_stats(cudaStream_t s, int sms, const void* a, long long lda, int dta, const void* b, long long ldb,
                       int dtb, int rows, int cols, double* partial, unsigned long long* flags_a,
                       unsigned long long* flags_b) {
  k_error_stats<<<error_stats_blocks(sms), 256, 0, s>>>(a, lda, dta, b, ldb, dtb, rows, cols, partial, flags_a,
                                                         flags_b);
  return cudaGetLastError() == cudaSuccess ? 0 : 6;
}

// ---------------------------------------------------------------------------- direct convolution
// out(y, x) = sum_{dy, dx} w2[W + dy][W + dx] * f(clamp(y - dy), clamp(x - dx)), dy outer, dx inner,
// each product rounded, then added (conv.py:88-95: `out += w * block`).  CTA = 16 x 16 outputs
// with the (16 + 2W)^2 clamped input tile in shared memory.
constexpr int CD_T = 16;
constexpr int CD_MAX_TILED_W = 77;  // (16 + 2W)^2 doubles fit the 227 KB of shared memory

template <bool TILED>
__global__ void __launch_bounds__(CD_T * CD_T) k_convolve_direct(const void* f, long long f_ld, int f_dtype,
                                                                 int rows, int cols, int W, const double* w2,
                                                                 double* out, long long out_ld) {
  extern __shared__ double cd_tile[];
  const int S = CD_T + 2 * W;
  const int y0 = blockIdx.y * CD_T, x0 = blockIdx.x * CD_T;
  if (TILED) {
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) {
      const int ty = i / S, tx = i - ty * S;
      const int gy = min(max(y0 + ty - W, 0), rows - 1), gx = min(max(x0 + tx - W, 0), cols - 1);
      cd_tile[i] = load_sample(f, f_dtype, (long long)gy * f_ld + gx);
    }
    __syncthreads();
  }
  const int ty = threadIdx.x / CD_T, tx = threadIdx.x % CD_T;
  const int y = y0 + ty, x = x0 + tx;
  if (y >= rows || x >= cols) return;
  const int n = 2 * W + 1;
  double acc = 0.0;
  for (int dy = -W; dy <= W; ++dy) {
    const double* wr = w2 + (W + dy) * n + W;
    if (TILED) {
      const double* rowp = cd_tile + (ty + W - dy) * S + tx + W;  // tile row of input row y - dy
      for (int dx = -W; dx <= W; ++dx) acc = __dadd_rn(acc, __dmul_rn(wr[dx], rowp[-dx]));
    } else {
      const long long gy = min(max(y - dy, 0), rows - 1) * f_ld;
      for (int dx = -W; dx <= W; ++dx)
        acc = __dadd_rn(acc, __dmul_rn(wr[dx], load_sample(f, f_dtype, gy + min(max(x - dx, 0), cols - 1))));
    }
  }
  out[(long long)y * out_ld + x] = acc;
}

int launch_convolve_direct(cudaStream_t s, const void* f, long long f_ld, int f_dtype, int rows, int cols, int W,
                           const double* w2, double* out, long long out_ld) {
  dim3 grid((unsigned)((cols + CD_T - 1) / CD_T), (unsigned)((rows + CD_T - 1) / CD_T));
  if (W <= CD_MAX_TILED_W) {
    const size_t smem = (size_t)(CD_T + 2 * W) * (CD_T + 2 * W) * sizeof(double);
    if (cudaFuncSetAttribute(k_convolve_direct<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return 6;
    k_convolve_direct<true><<<grid, CD_T * CD_T, smem, s>>>(f, f_ld, f_dtype, rows, cols, W, w2, out, out_ld);
  } else {
    k_convolve_direct<false><<<grid, CD_T * CD_T, 0, s>>>(f, f_ld, f_dtype, rows, cols, W, w2, out, out_ld);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 6;
}

}  // namespace fbgpu
