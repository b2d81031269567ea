// fb_fast64.cuh — specialised fp64 kernels (precision "f64": sigma_r < 16, small images, or on
// request).  Same two-kernel structure as the fp32 path (fb_fast.cuh), with fp64 channels:
//
// kernel 1  k1d_box_walk<NCH>    box: one padded column per thread walks CH output rows with the
//                                 N+1 vertical running sums in fp64 registers (no compensation
//                                 needed: fp64 drift over ~300 steps is ~1e-14 of |S|) and
//                                 coalesced 8-byte stores of each completed row.
//           k1d_gen_vpass<K, W>  Gaussian (and small box images): 32 columns x 64 rows per CTA,
//                                 channel cells in registers, vertical taps as DFMA.
// kernel 2  k2d_hpass_horner<K, W>  32 rows x 64 columns per CTA (8 warps x 8 columns); thread 0
//                                 streams fp64 channel tiles m = N..0 through a TMA/mbarrier
//                                 ring; horizontal pass + fp64 Horner (no conversions).
//
// Both kernel 1 variants write Taylor planes, c_m = e^{-x^2/2} (x/s)^m / m! (per-order factors
// taylor_r[m] = 1/(m s) in fp64), so kernel 2 gets Q and P = dQ/dx from one derivative-Horner pass
// with two FMAs per pixel and channel and no constants (fb_fast.cuh, TAYLOR).
#pragma once
#include "fb_fast.cuh"

namespace fbgpu {
namespace fast64 {

using fast::mbar_arrive_expect_tx;
using fast::mbar_arrive_if;
using fast::mbar_fence_init;
using fast::mbar_init;
using fast::mbar_wait;
using fast::smem_u32;
using fast::tma_load_3d;
using fast::tma_prefetch_desc;

// ---------------------------------------------------------------------------- kernel 1, box walker
constexpr int KD_THREADS = 128;

template <int NCH>
__global__ void __launch_bounds__(KD_THREADS) k1d_box_walk(const __grid_constant__ GpaArgs<double> a) {
  const int W = a.W;
  const int N = a.N;
  const int CH = a.walk_rows;
  const int pc = blockIdx.x * KD_THREADS + threadIdx.x;
  const int r0 = blockIdx.y * CH - a.lead;  // walks start at image rows = multiples of CH (fb_fast.cuh)
  const int rows_here = min(CH, a.band_rows - r0);
  const int scol = min(max(pc - W, 0), a.cols - 1);
  const bool own_col = pc >= W && pc < W + a.cols;
  const bool col_ok = pc < a.wpad;
  const long long row_base = (long long)a.halo_top + a.band_row0;
  auto clamp_row = [&](int band_row) -> long long {
    long long brow = row_base + band_row;
    return brow < 0 ? 0 : (brow >= a.rows_in ? a.rows_in - 1 : brow);
  };
  auto to_x = [&](double v) -> double { return a.mode == kModeGpa ? (v - a.tc) * a.inv_sr : v; };
  __shared__ double rn[NCH];  // the Taylor planes' per-order factors 1 / (n s); read as broadcasts
  for (int n = threadIdx.x; n < NCH; n += KD_THREADS) rn[n] = (n >= 1 && n <= N) ? __ldg(a.taylor_r + n) : 0.0;
  __syncthreads();
  const int steps = rows_here + 2 * W;
  double S[NCH];
#pragma unroll
  for (int n = 0; n < NCH; ++n) S[n] = 0.0;
  unsigned long long bad_nf = ~0ull, bad_rg = ~0ull;
  double* vp = a.v + pc;
  // samples two steps ahead in registers (loads of step st+2 overlap steps st, st+1)
  auto sample = [&](int band_row) { return load_sample(a.f, a.f_dtype, sample_row(a, row_base + band_row) + scol); };
  double ve0 = sample(r0 - W);
  double vl0 = sample(r0 - 3 * W - 1);
  double ve1 = sample(r0 - W + 1);
  double vl1 = sample(r0 - 3 * W);
  for (int st = 0; st < steps; ++st) {
    const int enter = r0 - W + st;
    const double fe = ve0, fl = vl0;
    ve0 = ve1;
    vl0 = vl1;
    ve1 = sample(enter + 2);
    vl1 = sample(enter + 1 - 2 * W);
    if (a.check && own_col && enter >= r0 && enter >= 0 && enter < r0 + rows_here) {
      const unsigned long long idx = (unsigned long long)clamp_row(enter) * a.cols + scol;
      if (!isfinite(fe) && bad_nf == ~0ull) bad_nf = idx;
      if ((fe < a.lo || fe > a.hi) && bad_rg == ~0ull) bad_rg = idx;
    }
    const double keep = st >= 2 * W + 1 ? 1.0 : 0.0;
    const double xe = to_x(fe), xl = to_x(fl);
    double ce = a.mode == kModeGpa ? exp(-0.5 * xe * xe) : xe;
    double cl = keep * (a.mode == kModeGpa ? exp(-0.5 * xl * xl) : xl);
#pragma unroll
    for (int n = 0; n < NCH; ++n) {
      if (n > 0) {
        ce *= xe * rn[n];
        cl *= xl * rn[n];
      }
      S[n] += ce - cl;
    }
    const int out_row = enter - W;
    if (col_ok && out_row >= r0 && out_row >= 0) {
      double* dst = vp + (long long)out_row * a.rstride;
#pragma unroll
      for (int n = 0; n < NCH; ++n, dst += a.pitch)
        if (n < NCH - 8 || n <= N) __stcs(dst, S[n]);  // evict-first: planes are read again only a band later
    }
  }
  if (a.check) {
    flag_min(a.flags + kFlagFirstNonfinite, bad_nf != ~0ull, bad_nf);
    flag_min(a.flags + kFlagFirstRange, bad_rg != ~0ull, bad_rg);
  }
}

// ---------------------------------------------------------------------------- kernel 1, tile
constexpr int KT_TC = 32;                 // padded columns per CTA
constexpr int KT_RG = 8;                  // row groups
constexpr int KT_R = 8;                   // output rows per thread
constexpr int KT_RB = KT_RG * KT_R;       // 64 output rows per CTA
constexpr int KT_THREADS = KT_TC * KT_RG;

inline size_t kt_smem_bytes(int W) { return 2ull * (KT_RB + 2 * W) * KT_TC * sizeof(double); }

template <int KIND, int WT>
__global__ void __launch_bounds__(KT_THREADS) k1d_gen_vpass(const __grid_constant__ GpaArgs<double> a) {
  extern __shared__ __align__(16) double kt_smem[];
  constexpr int W = WT;
  constexpr int TR = KT_RB + 2 * W;
  constexpr int NS = (TR + KT_RG - 1) / KT_RG;
  double* buf0 = kt_smem;
  double* buf1 = kt_smem + TR * KT_TC;
  const int tc = threadIdx.x % KT_TC;
  const int g = threadIdx.x / KT_TC;
  const int pc = blockIdx.x * KT_TC + tc;
  const int o0 = blockIdx.y * KT_RB - (KIND == kKindBox ? a.lead : 0);  // box: anchored to image rows
  const int scol = min(max(pc - W, 0), a.cols - 1);

  double cst[NS], xst[NS];
  {
    unsigned long long bad_nf = ~0ull, bad_rg = ~0ull;
    double fv[NS];
    long long brows[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      long long brow = (long long)a.halo_top + a.band_row0 + o0 + (g + KT_RG * t) - W;
      brows[t] = brow < 0 ? 0 : (brow >= a.rows_in ? a.rows_in - 1 : brow);
    }
#pragma unroll
    for (int t = 0; t < NS; ++t)
      fv[t] = g + KT_RG * t < TR ? load_sample(a.f, a.f_dtype, sample_row(a, brows[t]) + scol) : 0.0;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int i = g + KT_RG * t;
      double x = 0.0, e = 0.0;
      if (i < TR) {
        if (a.check) {
          const int o = o0 + i - W;
          const bool own = i >= W && i < W + KT_RB && o >= 0 && o < a.band_rows && pc >= W && pc < W + a.cols;
          const unsigned long long idx = (unsigned long long)brows[t] * a.cols + scol;
          if (own && !isfinite(fv[t]) && bad_nf == ~0ull) bad_nf = idx;
          if (own && (fv[t] < a.lo || fv[t] > a.hi) && bad_rg == ~0ull) bad_rg = idx;
        }
        if (a.mode == kModeGpa) {
          x = (fv[t] - a.tc) * a.inv_sr;
          e = exp(-0.5 * x * x);
        } else {
          e = fv[t];
        }
      }
      xst[t] = x;
      cst[t] = e;
    }
    if (a.check) {
      flag_min(a.flags + kFlagFirstNonfinite, bad_nf != ~0ull, bad_nf);
      flag_min(a.flags + kFlagFirstRange, bad_rg != ~0ull, bad_rg);
    }
  }

  const int ob = g * KT_R;
  const bool col_ok = pc < a.wpad;
  double* vp = a.v + (long long)(o0 + ob) * a.rstride + pc;
  for (int n = 0; n <= a.N; ++n, vp += a.pitch) {
    double* cs = (n & 1) ? buf1 : buf0;
    const double rs = n > 0 ? __ldg(a.taylor_r + n) : 1.0;  // Taylor planes: c_n = c_{n-1} x / (n s)
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int i = g + KT_RG * t;
      if (n > 0) cst[t] = cst[t] * (xst[t] * rs);
      if (i < TR) cs[i * KT_TC + tc] = cst[t];
    }
    __syncthreads();
    const double* col = cs + ob * KT_TC + tc;
    double acc[KT_R];
    if constexpr (KIND == kKindGauss) {
#pragma unroll
      for (int r = 0; r < KT_R; ++r) acc[r] = 0.0;
#pragma unroll
      for (int m = 0; m < KT_R + 2 * W; ++m) {
        const double c = col[m * KT_TC];
#pragma unroll
        for (int r = 0; r < KT_R; ++r) {
          const int k = m - r;
          if (k >= 0 && k <= 2 * W) acc[r] = fma(a.w[k], c, acc[r]);
        }
      }
    } else {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k = 0; k <= 2 * W; k += 2) s0 += col[k * KT_TC];
#pragma unroll
      for (int k = 1; k <= 2 * W; k += 2) s1 += col[k * KT_TC];
      double s = s0 + s1;
      acc[0] = s;
#pragma unroll
      for (int r = 1; r < KT_R; ++r) {
        s += col[(r + 2 * W) * KT_TC] - col[(r - 1) * KT_TC];
        acc[r] = s;
      }
    }
    if (col_ok) {
#pragma unroll
      for (int r = 0; r < KT_R; ++r)
        if (o0 + ob + r < a.band_rows && o0 + ob + r >= 0) __stcs(vp + (long long)r * a.rstride, acc[r]);
    }
  }
}

// ---------------------------------------------------------------------------- kernel 2
constexpr int KD2_TH = 32;      // rows per CTA (lane = row)
constexpr int KD2_R = 8;        // output columns per thread
constexpr int KD2_WARPS = 8;
constexpr int KD2_TW = KD2_R * KD2_WARPS;  // 64 columns per CTA
constexpr int KD2_THREADS = KD2_WARPS * 32;

// shared row stride in doubles: >= TW + 2W, even (16-byte rows) with S/2 odd (conflict-free
// 128-bit loads when lanes walk rows)
__host__ __device__ constexpr int kd2_stride(int W) {
  int s = (KD2_TW + 2 * W + 1) / 2 * 2;
  if (((s / 2) & 1) == 0) s += 2;
  return s;
}
// Box: the window sums read the stage directly (no 50-double register window), so two CTAs
// share an SM (probe knob FB_KD2_BOX_STREAM).
#ifndef FB_KD2_BOX_STREAM
#define FB_KD2_BOX_STREAM 1  // c4 f64 k2 7.53 -> 6.55 ms (with the stage-release proxy fence)
#endif
template <int KIND> __host__ __device__ constexpr int kd2_ctas() { return KIND == kKindBox && FB_KD2_BOX_STREAM ? 2 : 1; }
// ring depth: 3 stages (Gaussian, compute-bound) / up to 6 (box), within the SM's 227 KB
template <int KIND, int WT> __host__ __device__ constexpr int kd2_stages() {
  return (KIND == kKindGauss ? 3 : 6) <= (227 * 1024 / kd2_ctas<KIND>() - 1280) / (KD2_TH * kd2_stride(WT) * 8)
             ? (KIND == kKindGauss ? 3 : 6)
             : (227 * 1024 / kd2_ctas<KIND>() - 1280) / (KD2_TH * kd2_stride(WT) * 8);
}
inline size_t kd2_smem_bytes(int W, int stages) {
  return (size_t)stages * KD2_TH * kd2_stride(W) * sizeof(double) + 1024 + 2 * stages * 8;
}

template <int KIND, int WT>
__global__ void __launch_bounds__(KD2_THREADS, kd2_ctas<KIND>())
    k2d_hpass_horner(const __grid_constant__ GpaArgs<double> a, const __grid_constant__ CUtensorMap planes) {
  extern __shared__ __align__(1024) double kd2_smem[];
  constexpr int STAGES = kd2_stages<KIND, WT>();
  constexpr int S = kd2_stride(WT);
  constexpr int STAGE_D = KD2_TH * S;
  constexpr uint32_t STAGE_BYTES = STAGE_D * sizeof(double);
  constexpr int WIN = (KD2_R + 2 * WT + 1) / 2 * 2;  // window doubles (128-bit loads)
  const uint32_t base = smem_u32(kd2_smem);
  double* ring = kd2_smem + (((base + 1023u) & ~1023u) - base) / 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * STAGE_D);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int x0 = blockIdx.x * KD2_TW;
  const int y0 = blockIdx.y * KD2_TH;
  const int N = a.N;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, KIND == kKindBox ? KD2_WARPS * 32 : KD2_WARPS);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&planes);
    for (int it = 0; it < STAGES && it <= N; ++it) {
      mbar_arrive_expect_tx(full + it, STAGE_BYTES);
      tma_load_3d(ring + it * STAGE_D, &planes, full + it, x0, N - it, y0);
    }
  }

  const int orow = y0 + lane;
  const int c0 = warp * KD2_R;
  const long long brow = (long long)a.halo_top + a.band_row0 + orow;
  const bool row_ok = orow < a.band_rows;
  const int col0 = x0 + c0;
  double xd[KD2_R], pd[KD2_R], qd[KD2_R];
#pragma unroll
  for (int j = 0; j < KD2_R; ++j) {
    const double fv = (row_ok && col0 + j < a.cols) ? load_sample(a.f, a.f_dtype, brow * a.f_ld + col0 + j) : 0.0;
    xd[j] = (fv - a.tc) * a.inv_sr * a.taylor_s;  // y = x s: Q = sum_m plane_m y^m (fb_fast.cuh, TAYLOR)
    pd[j] = 0.0;
    qd[j] = 0.0;
  }

  // Box windows (<= 72 doubles) are copied to registers and the stage released at once; the
  // Gaussian reads its taps' inputs straight from shared memory (its 8 x (2W+1) DFMAs would not
  // fit a register window) and releases the stage after the horizontal pass.
  constexpr bool kSmemWin = KIND == kKindGauss || FB_KD2_BOX_STREAM;
  double win[kSmemWin ? 2 : WIN];
  const double* wsm = nullptr;
  // box: one arrive per lane (no reconvergence point; as in the fp32 kernel 2), Gaussian: the
  // warp-level release after the pass
  // (the proxy fence of fb_fast.cuh's kernel 2: stage reads ordered before the refill TMA)
  auto release = [&](int it) {
    fast::fence_proxy_async_smem();
    if constexpr (KIND == kKindBox) {
      fast::mbar_arrive(empty + it % STAGES);
    } else {
      __syncwarp();
      mbar_arrive_if(empty + it % STAGES, lane == 0);
    }
  };
  auto load_window = [&](int it) {
    const int s = it % STAGES;
    if (threadIdx.x == 0 && it >= 1 && it - 1 + STAGES <= N) {
      const int sp = (it - 1) % STAGES;
      mbar_wait(empty + sp, ((it - 1) / STAGES) & 1);
      mbar_arrive_expect_tx(full + sp, STAGE_BYTES);
      tma_load_3d(ring + sp * STAGE_D, &planes, full + sp, x0, N - (it - 1 + STAGES), y0);
    }
    mbar_wait(full + s, (it / STAGES) & 1);
    const double* row = ring + s * STAGE_D + lane * S + c0;
    if constexpr (kSmemWin) {
      wsm = row;
    } else {
#pragma unroll
      for (int i = 0; i < WIN / 2; ++i) {
        const double2 v2 = *reinterpret_cast<const double2*>(row + 2 * i);
        win[2 * i] = v2.x;
        win[2 * i + 1] = v2.y;
      }
      release(it);
    }
  };
  auto hpass = [&](int it, double* hv) {
    if constexpr (KIND == kKindGauss) {
#pragma unroll
      for (int j = 0; j < KD2_R; ++j) hv[j] = 0.0;
#pragma unroll
      for (int m = 0; m < KD2_R + 2 * WT; ++m) {
        const double c = wsm[m];
#pragma unroll
        for (int j = 0; j < KD2_R; ++j) {
          const int k = m - j;
          if (k >= 0 && k <= 2 * WT) hv[j] = fma(a.w[k], c, hv[j]);
        }
      }
      release(it);
    } else if constexpr (kSmemWin) {
      // same sums, the window read from the stage two doubles at a time as it is reached
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < (2 * WT + 2) / 2; ++q) {
        const double2 v = *reinterpret_cast<const double2*>(wsm + 2 * q);
        if (2 * q <= 2 * WT) s4[(2 * q) & 3] += v.x;
        if (2 * q + 1 <= 2 * WT) s4[(2 * q + 1) & 3] += v.y;
      }
      double sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      hv[0] = sum;
      double2 lv = make_double2(0.0, 0.0), ev = lv;
#pragma unroll
      for (int j = 1; j < KD2_R; ++j) {
        const int il = j - 1, ie = j + 2 * WT;
        if (j == 1 || (il & 1) == 0) lv = *reinterpret_cast<const double2*>(wsm + (il & ~1));
        if (j == 1 || (ie & 1) == 0) ev = *reinterpret_cast<const double2*>(wsm + (ie & ~1));
        sum += ((ie & 1) ? ev.y : ev.x) - ((il & 1) ? lv.y : lv.x);
        hv[j] = sum;
      }
      release(it);
    } else {
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k <= 2 * WT; ++k) s4[k & 3] += win[k];
      double sum = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      hv[0] = sum;
#pragma unroll
      for (int j = 1; j < KD2_R; ++j) {
        sum += win[j + 2 * WT] - win[j - 1];
        hv[j] = sum;
      }
    }
  };
  // The derivative Horner of fb_fast.cuh on Taylor planes c_m = Fbar_m / (m! s^m), y = x s:
  //   channel N:      d = N c_N, q = 0          channel N-1:   q = c_{N-1}  (d keeps N c_N)
  //   channel m < N-1: d <- q + y d,  q <- c_m + y q            (pd holds d);   Q = q, P = s d
  auto taylor_top = [&](const double* hv) {
#pragma unroll
    for (int j = 0; j < KD2_R; ++j) pd[j] = (double)N * hv[j];
  };
  auto taylor_first = [&](const double* hv) {
#pragma unroll
    for (int j = 0; j < KD2_R; ++j) qd[j] = hv[j];
  };
  auto taylor_step = [&](const double* hv) {
#pragma unroll
    for (int j = 0; j < KD2_R; ++j) {
      pd[j] = fma(xd[j], pd[j], qd[j]);
      qd[j] = fma(xd[j], qd[j], hv[j]);
    }
  };

  double hv[KD2_R], hn[KD2_R];
  load_window(0);
  hpass(0, hv);  // channel N
  if (N >= 1 && a.mode == kModeGpa) {
    load_window(1);
    taylor_top(hv);
    hpass(1, hn);  // channel N - 1
#pragma unroll
    for (int j = 0; j < KD2_R; ++j) hv[j] = hn[j];
    if (N >= 2) {
      load_window(2);
      taylor_first(hv);
      hpass(2, hn);  // channel N - 2
#pragma unroll
      for (int j = 0; j < KD2_R; ++j) hv[j] = hn[j];
      for (int m = N - 2; m >= 1; --m) {
        load_window(N - m + 1);
        taylor_step(hv);
        hpass(N - m + 1, hn);  // channel m - 1
#pragma unroll
        for (int j = 0; j < KD2_R; ++j) hv[j] = hn[j];
      }
      taylor_step(hv);  // channel 0
    } else {
      taylor_first(hv);  // N = 1: channel 0
    }
  }

  // epilogue (as fb_fast.cuh): quotients, Q floor (engine.py:20, 68), bookkeeping, stores
  if (!row_ok) return;
  const long long orow_global = (long long)(a.band_row0 + orow) * a.out_ld;
  double o[KD2_R];
  unsigned degenerate = 0;
#pragma unroll
  for (int j = 0; j < KD2_R; ++j) {
    if (a.mode == kModePlain) {
      o[j] = hv[j] * a.norm;
    } else {
      o[j] = a.sr * (pd[j] * a.taylor_s / qd[j]) + a.tc;
      if (fabs(qd[j] * a.norm) < 1e-30) degenerate |= 1u << j;
    }
  }
  unsigned long long n_degenerate = 0, n_nonfinite = 0;
  if (degenerate) {
#pragma unroll
    for (int j = 0; j < KD2_R; ++j)
      if ((degenerate >> j) & 1u) {
        o[j] = col0 + j < a.cols ? load_sample(a.f, a.f_dtype, brow * a.f_ld + col0 + j) : 0.0;
        n_degenerate += col0 + j < a.cols;
      }
  }
#pragma unroll
  for (int j = 0; j < KD2_R; ++j) {
    if (col0 + j >= a.cols) continue;
    n_nonfinite += !isfinite(o[j]);
    store_sample(a.out, a.out_dtype, orow_global + col0 + j, o[j]);
  }
  if (n_degenerate) atomicAdd(a.flags + kFlagDegenerate, n_degenerate);
  if (n_nonfinite) atomicAdd(a.flags + kFlagNonfiniteOut, n_nonfinite);
}

// ---------------------------------------------------------------------------- host dispatch
inline int make_plane_map64(CUtensorMap* map, const GpaArgs<double>& a, int W) {
  auto fn = fast::encode_fn();
  if (!fn) return 6;
  cuuint64_t dims[3] = {(cuuint64_t)a.pitch, (cuuint64_t)(a.N + 1), (cuuint64_t)a.band_max};
  cuuint64_t strides[2] = {(cuuint64_t)a.pitch * sizeof(double), (cuuint64_t)a.rstride * sizeof(double)};
  cuuint32_t box[3] = {(cuuint32_t)kd2_stride(W), 1, (cuuint32_t)KD2_TH};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a.v, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 6;
}

template <int KIND, int WT>
int launch_pair64(cudaStream_t st, GpaArgs<double>& a, const KernelEvents& ev) {
  const int W = a.W;
  void (*k1)(const GpaArgs<double>) = k1d_gen_vpass<KIND, WT>;
  size_t s1 = kt_smem_bytes(W);
  a.lead = KIND == kKindBox ? box_lead(a, KT_RB) : 0;
  dim3 g1((a.wpad + KT_TC - 1) / KT_TC, (a.band_rows + a.lead + KT_RB - 1) / KT_RB), b1(KT_THREADS);
  if constexpr (KIND == kKindBox) {
    if (a.N + 1 <= kWalkMaxCh && (long long)a.wpad * a.image_rows >= (4ll << 20)) {
      static void (*const walkers[8])(const GpaArgs<double>) = {
          k1d_box_walk<8>, k1d_box_walk<16>, k1d_box_walk<24>, k1d_box_walk<32>,
          k1d_box_walk<40>, k1d_box_walk<48>, k1d_box_walk<56>, k1d_box_walk<64>};
      k1 = walkers[(a.N + 1 + 7) / 8 - 1];
      s1 = 0;
      const int gx = (a.wpad + KD_THREADS - 1) / KD_THREADS;
      const int ch = walk_rows(a.wpad, a.image_rows, KD_THREADS);
      a.walk_rows = ch;
      a.lead = box_lead(a, ch);
      g1 = dim3(gx, (a.band_rows + a.lead + ch - 1) / ch);
      b1 = dim3(KD_THREADS);
    }
  }
  if (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1) != cudaSuccess) return 6;
  auto k2 = k2d_hpass_horner<KIND, WT>;
  const size_t s2 = kd2_smem_bytes(W, kd2_stages<KIND, WT>());
  if (cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2) != cudaSuccess) return 6;
  dim3 g2((a.cols + KD2_TW - 1) / KD2_TW, (a.band_rows + KD2_TH - 1) / KD2_TH);
  CUtensorMap map;
  if (make_plane_map64(&map, a, W) != 0) return 6;
  record_timing(ev.k1_start, st);
  k1<<<g1, b1, s1, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return 6;
  record_timing(ev.k1_end, st);
  k2<<<g2, KD2_THREADS, s2, st>>>(a, map);
  if (cudaGetLastError() != cudaSuccess) return 6;
  record_timing(ev.k2_end, st);
  return 0;
}

}  // namespace fast64

#define FB_CASE64_kKindGauss(w) \
  case w:                       \
    *done = true;               \
    return fast64::launch_pair64<kKindGauss, w>(st, a, ev);
#define FB_CASE64_kKindBox(w) \
  case w:                     \
    *done = true;             \
    return fast64::launch_pair64<kKindBox, w>(st, a, ev);
#define FB_FAST64_DISPATCH(NAME, KIND, LIST)                                                      \
  int NAME(cudaStream_t st, int W, GpaArgs<double>& a, const KernelEvents& ev, bool* done) {     \
    *done = false;                                                                               \
    switch (W) {                                                                                 \
      LIST(FB_CASE64_##KIND)                                                                     \
      default:                                                                                   \
        return 0;                                                                                \
    }                                                                                            \
  }

}  // namespace fbgpu
