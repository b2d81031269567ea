// fb_generic.cuh — runtime-W tile kernels (any half-width up to kMaxW, fp32 or fp64).
//
// These are the general path: every (kind, W, precision) the API accepts runs
// here; the template-specialised fp32 kernels in fb_fast.cuh take over the
// performance configurations.  Both compute exactly the same arithmetic:
//
//   kernel 1 (k1_gen_vpass): per CTA a 32-column x 64-row tile of the padded
//     band.  The channel tile c_n = e x^n / sqrt(n!)  (x = (f - t_c)/sigma_r,
//     e = exp(-x^2/2)) with a W-row halo lives in shared memory and is advanced
//     in place, c_n = c_{n-1} * (x / sqrt(n))  (engine.py:51-62 with the
//     1/sqrt(n!) normalisation that keeps every channel in [-1, 1]); for each n
//     the vertical pass (box running sum / Gaussian taps) is written to plane n.
//   kernel 2 (k2_hpass_horner): per CTA a 16 x 64 output tile; for channel
//     m = N .. 0 it stages the plane tile (+W columns each side) in shared
//     memory, applies the horizontal pass and advances the Horner recurrences
//       q_m = Cbar_m + (x/sqrt(m+1)) q_{m+1},  p_{m-1} = sqrt(m) Cbar_m + (x/sqrt(m)) p_m
//     so q_0 = Q and p_0 = P of engine.py:60-66 exactly; then
//     out = sigma_r * P/Q + t_c, with the |Q| < 1e-30 pass-through (engine.py:68-72).
#pragma once
#include <type_traits>
#include "fb_common.cuh"

namespace fbgpu {
namespace generic {

constexpr int K1_TC = 32;   // columns per CTA (one warp wide)
constexpr int K1_RG = 8;    // row groups (warps)
constexpr int K1_RB = 64;   // output rows per CTA
constexpr int K1_R = K1_RB / K1_RG;

constexpr int K2_TW = 64;   // output columns per CTA
constexpr int K2_TH = 16;   // output rows per CTA
constexpr int K2_R = 4;     // outputs per thread (consecutive columns)

template <typename T>
__host__ __device__ constexpr size_t k1_smem(int W) {
  return 2ull * (K1_RB + 2 * W) * K1_TC * sizeof(T);
}
template <typename T>
__host__ __device__ constexpr size_t k2_smem(int W) {
  return (size_t)K2_TH * (K2_TW + 2 * W) * sizeof(T);
}

template <typename T, int KIND>
__global__ void __launch_bounds__(K1_TC * K1_RG) k1_gen_vpass(const GpaArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int W = a.W;
  const int TR = K1_RB + 2 * W;
  T* cs = reinterpret_cast<T*>(smem_raw);
  T* xs = cs + TR * K1_TC;
  const int tc = threadIdx.x % K1_TC;
  const int g = threadIdx.x / K1_TC;
  const int pc = blockIdx.x * K1_TC + tc;
  const int o0 = blockIdx.y * K1_RB - (KIND == kKindBox ? a.lead : 0);  // box: anchored to image rows
  const int scol = min(max(pc - W, 0), a.cols - 1);

  for (int i = g; i < TR; i += K1_RG) {
    const int o = o0 + i - W;
    long long brow = (long long)a.halo_top + a.band_row0 + o;
    brow = brow < 0 ? 0 : (brow >= a.rows_in ? a.rows_in - 1 : brow);
    const double fv = load_sample(a.f, a.f_dtype, sample_row(a, brow) + scol);
    if (a.check) {
      const bool own = i >= W && i < W + K1_RB && o >= 0 && o < a.band_rows && pc >= W && pc < W + a.cols;
      check_sample(a.flags, own, fv, a.lo, a.hi, (unsigned long long)brow * a.cols + scol);
    }
    T x, e;
    if (a.mode == kModeGpa) {
      x = (T)((fv - a.tc) * a.inv_sr);
      e = gauss_exp<T>(x);
    } else {
      x = T(0);
      e = (T)fv;
    }
    xs[i * K1_TC + tc] = x;
    cs[i * K1_TC + tc] = e;
  }

  const int ob = g * K1_R;
  for (int n = 0; n <= a.N; ++n) {
    if (n > 0) {
      const T rs = (T)(1.0 / sqrt((double)n));
      for (int i = g; i < TR; i += K1_RG) cs[i * K1_TC + tc] = cs[i * K1_TC + tc] * (xs[i * K1_TC + tc] * rs);
    }
    __syncthreads();
    T* vp = a.v + (long long)n * a.pitch;
    const bool col_ok = pc < a.wpad;
    if (KIND == kKindBox) {
      T s = T(0);
      for (int k = 0; k <= 2 * W; ++k) s += cs[(ob + k) * K1_TC + tc];
      for (int r = 0; r < K1_R; ++r) {
        const int o = o0 + ob + r;
        if (col_ok && o >= 0 && o < a.band_rows) vp[(long long)o * a.rstride + pc] = s;
        s += cs[(ob + r + 2 * W + 1) * K1_TC + tc] - cs[(ob + r) * K1_TC + tc];
      }
    } else {
      for (int r = 0; r < K1_R; ++r) {
        T acc = T(0);
        for (int k = 0; k <= 2 * W; ++k) acc = fma(a.w[k], cs[(ob + r + k) * K1_TC + tc], acc);
        const int o = o0 + ob + r;
        if (col_ok && o < a.band_rows) vp[(long long)o * a.rstride + pc] = acc;
      }
    }
    __syncthreads();
  }
}

template <typename T, int KIND>
__global__ void __launch_bounds__(256) k2_hpass_horner(const GpaArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);
  const int W = a.W;
  const int LW = K2_TW + 2 * W;
  const int r = threadIdx.x / (K2_TW / K2_R);
  const int c0 = (threadIdx.x % (K2_TW / K2_R)) * K2_R;
  const int x0 = blockIdx.x * K2_TW;
  const int y0 = blockIdx.y * K2_TH;
  const int orow = y0 + r;
  const long long brow = (long long)a.halo_top + a.band_row0 + orow;

  T xv[K2_R], p[K2_R], q[K2_R], hv[K2_R];
  double fin[K2_R];
  bool valid[K2_R];
#pragma unroll
  for (int j = 0; j < K2_R; ++j) {
    const int col = x0 + c0 + j;
    valid[j] = orow < a.band_rows && col < a.cols;
    fin[j] = valid[j] ? load_sample(a.f, a.f_dtype, brow * a.f_ld + col) : 0.0;
    xv[j] = (T)((fin[j] - a.tc) * a.inv_sr);
    p[j] = T(0);
    q[j] = T(0);
  }

  T rs_next = T(0);  // 1/sqrt(m+1) of the previous (higher) channel
  for (int m = a.N; m >= 0; --m) {
    const T* vp = a.v + (long long)m * a.pitch;
    for (int idx = threadIdx.x; idx < K2_TH * LW; idx += blockDim.x) {
      const int rr = idx / LW, cc = idx - rr * LW;
      const int gr = y0 + rr, gc = x0 + cc;
      tile[idx] = (gr < a.band_rows && gc < a.wpad) ? vp[(long long)gr * a.rstride + gc] : T(0);
    }
    __syncthreads();
    const T* row = tile + r * LW + c0;
    if (KIND == kKindBox) {
      T s = T(0);
      for (int k = 0; k <= 2 * W; ++k) s += row[k];
      hv[0] = s;
#pragma unroll
      for (int j = 1; j < K2_R; ++j) {
        s += row[j + 2 * W] - row[j - 1];
        hv[j] = s;
      }
    } else {
#pragma unroll
      for (int j = 0; j < K2_R; ++j) hv[j] = T(0);
      for (int k = 0; k <= 2 * W; ++k) {
        const T wk = a.w[k];
#pragma unroll
        for (int j = 0; j < K2_R; ++j) hv[j] = fma(wk, row[j + k], hv[j]);
      }
    }
    if (a.mode == kModeGpa) {
      const T rs = m > 0 ? (T)(1.0 / sqrt((double)m)) : T(0);
      const T sq = (T)sqrt((double)m);
#pragma unroll
      for (int j = 0; j < K2_R; ++j) {
        if (m < a.N) q[j] = fma(xv[j] * rs_next, q[j], hv[j]);
        if (m > 0) p[j] = fma(xv[j] * rs, p[j], sq * hv[j]);
      }
      rs_next = rs;
    }
    __syncthreads();
  }

#pragma unroll
  for (int j = 0; j < K2_R; ++j) {
    if (!valid[j]) continue;
    const int col = x0 + c0 + j;
    double o;
    if (a.mode == kModePlain) {
      o = (double)(hv[j] * a.norm);  // (T = float: already an fp32 value)
    } else {
      const T qn = q[j] * a.norm;
      if (fabs((double)qn) < 1e-30) {
        o = fin[j];
        atomicAdd(a.flags + kFlagDegenerate, 1ull);
      } else {
        const T ratio = (T)a.sr * (p[j] / q[j]);
        o = (double)ratio + a.tc;  // (T = float: an fp32 centred result + t_c, as f32_result)
      }
    }
    if (!isfinite(o)) atomicAdd(a.flags + kFlagNonfiniteOut, 1ull);
    store_sample(a.out, a.out_dtype, (long long)(a.band_row0 + orow) * a.out_ld + col, o, a.tc);
  }
}

}  // namespace generic
}  // namespace fbgpu
