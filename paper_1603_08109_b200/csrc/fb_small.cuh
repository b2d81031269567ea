// fb_small.cuh — one fused kernel for small images (fewer than kSmallImageSamples padded samples:
// c0 512^2, c1 1024^2), where kernel 1 + kernel 2 are launch- and latency-bound and the channel
// planes would only make a round trip through L2.
//
// k_small_fused<KIND, WT>: a CTA owns a 32 x 32 output tile and runs gpa_filter
// (engine.py:51-76) on it without leaving the SM:
//   prologue   the (32 + 2W)^2 replicate-padded samples of the tile -> x = (f - t_c) / sigma_r and
//              e = exp(-x^2 / 2), kept in registers (a thread holds one padded column of every
//              RSTEP-th row); input validation of the tile's own pixels (image.py:35-54)
//   per channel n = 0 .. N (ascending, the order the recurrence generates them):
//     1. c_n = c_{n-1} (x r_n) in registers -> shared tile A[32 + 2W][PW]
//     2. vertical pass A -> B[32][PW]: a thread owns one padded column and RV output rows
//        (Gaussian: packed FFMA2 tap pairs; box: running sum over RV rows, conv.py:30-54)
//     3. horizontal pass B -> 4 consecutive outputs per thread, then the fp64 accumulation
//        Q += tau_n Cbar_n (n < N), P += tau_{n-1} s_n Cbar_n (n >= 1), tau_n = tau_{n-1} x h_n: the ascending
//        form of kernel 2's Horner recurrences (same constants h_n = 1/(n r_n), s_n = 1/r_n matched
//        to the fp32 r_n of step 1, so P and Q are the sums of engine.py:60-66 exactly)
//   epilogue   out = sigma_r P / Q + t_c with the Q floor (engine.py:20, 68) in fp64.
// Two __syncthreads per channel.  Box tiles and their RV-row / 4-column running-sum groups are
// anchored to image rows (a.lead) and columns, so the bits do not depend on the band split.
#pragma once
#include "fb_fast.cuh"

namespace fbgpu {
namespace small {

using namespace ::fbgpu::fast;

constexpr int SM_T = 32;          // output tile edge
constexpr int SM_THREADS = 256;
constexpr int SM_RH = 4;          // horizontal outputs per thread (8 threads per tile row)

__host__ __device__ constexpr int sm_pt(int W) { return SM_T + 2 * W; }                       // padded tile edge
__host__ __device__ constexpr int sm_pw(int W) { return (sm_pt(W) & 1) ? sm_pt(W) : sm_pt(W) + 1; }  // odd pitch

// R running (2W+1)-sums of consecutive window positions: the first by two interleaved partial
// sums, the others by the enter/leave update (the order of the kernel-1 tile's box code).
template <int R, int WT, typename Load>
__device__ __forceinline__ void box_run(float (&out)[R], Load load) {
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int k = 0; k <= 2 * WT; k += 2) s0 += load(k);
#pragma unroll
  for (int k = 1; k <= 2 * WT; k += 2) s1 += load(k);
  float s = s0 + s1;
  out[0] = s;
#pragma unroll
  for (int r = 1; r < R; ++r) {
    s += load(r + 2 * WT) - load(r - 1);
    out[r] = s;
  }
}

// CTAs per SM the register budget is capped for (narrow windows fit three 256-thread CTAs).
__host__ __device__ constexpr int sm_min_blocks(int W) { return W <= 12 ? 3 : 2; }
__host__ __device__ constexpr int sm_rstep(int W) { return SM_THREADS / sm_pt(W); }            // padded rows per sweep
__host__ __device__ constexpr int sm_ns(int W) { return (sm_pt(W) + sm_rstep(W) - 1) / sm_rstep(W); }  // sweeps
// A holds sm_ns * sm_rstep >= PT rows: the last sweep's rows beyond the padded tile land in
// padding rows nobody reads, so step 1 stores without predicates.
inline size_t sm_smem_bytes(int W) {
  return (size_t)(sm_ns(W) * sm_rstep(W) + SM_T) * sm_pw(W) * sizeof(float);
}

template <int KIND, int WT>
__global__ void __launch_bounds__(SM_THREADS, sm_min_blocks(WT)) k_small_fused(const __grid_constant__ GpaArgs<float> a) {
  extern __shared__ __align__(16) float sm_smem[];
  constexpr int W = WT;
  constexpr int PT = sm_pt(WT);
  constexpr int PW = sm_pw(WT);
  constexpr int RSTEP = sm_rstep(WT);
  constexpr int NS = sm_ns(WT);
  constexpr int RV = WT <= 16 ? 8 : 16;               // vertical outputs per thread
  constexpr int ITEMS = PT * (SM_T / RV);             // (padded column, row group) items <= 256
  static_assert(ITEMS <= SM_THREADS, "vertical pass items");
  float* A = sm_smem;                      // [NS * RSTEP][PW]  channel n of the padded tile
  float* B = sm_smem + NS * RSTEP * PW;    // [SM_T][PW] vertically filtered

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * SM_T;
  const int o0 = blockIdx.y * SM_T - (KIND == kKindBox ? a.lead : 0);  // band-local row of tile row 0
  const long long row_base = (long long)a.halo_top + a.band_row0;       // buffer row of band row 0

  // ---------------- prologue: samples of padded column gj, padded rows gi + RSTEP t.  The
  // 256 - PT * RSTEP threads past the last column group repeat the last group's work (same
  // values to the same addresses), so nothing in the channel loop is predicated.
  const int gj = tid % PT, gi = min(tid / PT, RSTEP - 1);
  float cst[NS], xst[NS];
  {
    const int scol = min(max(x0 - W + gj, 0), a.cols - 1);
    const bool own_col = gj >= W && gj < W + SM_T && x0 - W + gj < a.cols;
    unsigned long long bad_nf = ~0ull, bad_rg = ~0ull;
    // sample offsets: tiles whose padded rows are all own rows of the buffer step a plain row
    // pointer; border tiles resolve every row (replicate clamp, halo buffers) with sample_row()
    const long long b0 = row_base + o0 - W;  // buffer row of padded row 0
    const bool plain = b0 >= a.halo_top && b0 + PT <= a.main_end;
    long long offs[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int i = min(gi + RSTEP * t, PT - 1);
      offs[t] = (plain ? (b0 + i) * a.f_ld : sample_row(a, b0 + i)) + scol;
    }
    double fv[NS];
    if (a.f_dtype == 1) {
      const float* f = reinterpret_cast<const float*>(a.f);
#pragma unroll
      for (int t = 0; t < NS; ++t) fv[t] = __ldg(f + offs[t]);
    } else if (a.f_dtype == 2) {
      const double* f = reinterpret_cast<const double*>(a.f);
#pragma unroll
      for (int t = 0; t < NS; ++t) fv[t] = __ldg(f + offs[t]);
    } else {
      const unsigned char* f = reinterpret_cast<const unsigned char*>(a.f);
#pragma unroll
      for (int t = 0; t < NS; ++t) fv[t] = (double)__ldg(f + offs[t]);
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int i = gi + RSTEP * t;
      if (a.check) {
        const int o = o0 + i - W;
        const bool own = own_col && i >= W && i < W + SM_T && o >= 0 && o < a.band_rows;
        const bool nf = own && !isfinite(fv[t]), rg = own && (fv[t] < a.lo || fv[t] > a.hi);
        if ((nf && bad_nf == ~0ull) || (rg && bad_rg == ~0ull)) {  // rare; rows increase with t
          const unsigned long long idx = (unsigned long long)(row_base + o) * a.cols + scol;
          if (nf && bad_nf == ~0ull) bad_nf = idx;
          if (rg && bad_rg == ~0ull) bad_rg = idx;
        }
      }
      const float x = (float)((fv[t] - a.tc) * a.inv_sr);
      xst[t] = x;
      cst[t] = expf(-0.5f * x * x);
    }
    if (a.check) {
      flag_min(a.flags + kFlagFirstNonfinite, bad_nf != ~0ull, bad_nf);
      flag_min(a.flags + kFlagFirstRange, bad_rg != ~0ull, bad_rg);
    }
  }

  // ---------------- the thread's 4 output pixels: tile row hr, tile columns hc .. hc + 3
  const int hr = tid / (SM_T / SM_RH), hc = (tid % (SM_T / SM_RH)) * SM_RH;
  const int orow = o0 + hr;
  const bool row_ok = orow >= 0 && orow < a.band_rows;
  const long long brow = row_base + orow;
  const int col0 = x0 + hc;
  double fown[SM_RH], xd[SM_RH], tau[SM_RH], pd[SM_RH], qd[SM_RH];
#pragma unroll
  for (int j = 0; j < SM_RH; ++j) {
    fown[j] = (row_ok && col0 + j < a.cols) ? load_sample(a.f, a.f_dtype, brow * a.f_ld + col0 + j) : 0.0;
    xd[j] = (double)(float)((fown[j] - a.tc) * a.inv_sr);
    tau[j] = 1.0;
    pd[j] = 0.0;
    qd[j] = 0.0;
  }

  // vertical item of this thread: padded column vj, output rows vg * RV ..
  const int vj = tid % PT, vg = tid / PT;
  const float* Av = A + (vg * RV) * PW + vj;
  float* Bv = B + (vg * RV) * PW + vj;
  const float* Bh = B + hr * PW + hc;
  float* Ag = A + gi * PW + gj;

  const int N = a.N;
  float rs = 1.f;
  for (int n = 0; n <= N; ++n) {
    // constants of this channel's accumulation and of the next channel's recurrence, loaded
    // ahead of the two barriers that separate them from their use
    const double hn = __ldg(a.tabd_seq + 2 * n), sn = __ldg(a.tabd_seq + 2 * n + 1);
    const float rs_next = __ldg(a.tab + 4 * min(n + 1, N));
    // 1. channel n of the padded tile
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      if (n > 0) cst[t] = cst[t] * (xst[t] * rs);
      Ag[t * RSTEP * PW] = cst[t];
    }
    rs = rs_next;
    __syncthreads();
    // 2. vertical pass
    if (tid < ITEMS) {
      float acc[RV];
      if constexpr (KIND == kKindGauss) {
        f2_t acc2[RV / 2];
        taps_pairs<RV, WT>(a, acc2, [&](int m) { return Av[m * PW]; });
#pragma unroll
        for (int p = 0; p < RV / 2; ++p) {
          acc[2 * p] = f2_lo(acc2[p]);
          acc[2 * p + 1] = f2_hi(acc2[p]);
        }
      } else {
        box_run<RV, WT>(acc, [&](int m) { return Av[m * PW]; });
      }
#pragma unroll
      for (int r = 0; r < RV; ++r) Bv[r * PW] = acc[r];
    }
    __syncthreads();
    // 3. horizontal pass + fp64 accumulation
    float hv[SM_RH];
    if constexpr (KIND == kKindGauss) {
      f2_t h2[SM_RH / 2];
      taps_pairs<SM_RH, WT>(a, h2, [&](int m) { return Bh[m]; });
#pragma unroll
      for (int p = 0; p < SM_RH / 2; ++p) {
        hv[2 * p] = f2_lo(h2[p]);
        hv[2 * p + 1] = f2_hi(h2[p]);
      }
    } else {
      box_run<SM_RH, WT>(hv, [&](int m) { return Bh[m]; });
    }
    // engine.py:58-66: Q sums channels 0 .. N-1, P channels 1 .. N
    if (n == 0) {
#pragma unroll
      for (int j = 0; j < SM_RH; ++j) qd[j] = N >= 1 ? (double)hv[j] : 0.0;
    } else {
      const bool do_q = n < N;
#pragma unroll
      for (int j = 0; j < SM_RH; ++j) {
        const double v = (double)hv[j];
        pd[j] = fma(tau[j] * sn, v, pd[j]);
        tau[j] *= xd[j] * hn;
        if (do_q) qd[j] = fma(tau[j], v, qd[j]);
      }
    }
    // The next channel's step 1 writes A, which nobody reads after the second barrier; its step 2
    // writes B only after the first barrier of that channel, which every thread reaches after
    // this horizontal pass.
  }

  // ---------------- epilogue
  if (!row_ok || col0 >= a.cols) return;
  double o[SM_RH];
  unsigned long long n_degenerate = 0, n_nonfinite = 0;
#pragma unroll
  for (int j = 0; j < SM_RH; ++j) {
    o[j] = f32_result(a.sr * ddiv_newton(pd[j], qd[j]), a.tc);
    if (fabs(qd[j] * (double)a.norm) < 1e-30) {  // Q floor (engine.py:20, 68)
      o[j] = fown[j];
      n_degenerate += col0 + j < a.cols;
    }
    n_nonfinite += (col0 + j < a.cols) && !isfinite(o[j]);
  }
  const long long oidx = (long long)(a.band_row0 + orow) * a.out_ld + col0;
  if (a.out_dtype == 2 && col0 + SM_RH <= a.cols &&
      (reinterpret_cast<uintptr_t>(reinterpret_cast<double*>(a.out) + oidx) & 15) == 0) {
    double2* p = reinterpret_cast<double2*>(reinterpret_cast<double*>(a.out) + oidx);
    p[0] = make_double2(o[0], o[1]);
    p[1] = make_double2(o[2], o[3]);
  } else if ((a.out_dtype == 1 || a.out_dtype == kOutF32Centred) && col0 + SM_RH <= a.cols &&
             (reinterpret_cast<uintptr_t>(reinterpret_cast<float*>(a.out) + oidx) & 15) == 0) {
    const double sub = a.out_dtype == kOutF32Centred ? a.tc : 0.0;
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + oidx) =
        make_float4((float)(o[0] - sub), (float)(o[1] - sub), (float)(o[2] - sub), (float)(o[3] - sub));
  } else {
#pragma unroll
    for (int j = 0; j < SM_RH; ++j)
      if (col0 + j < a.cols) store_sample(a.out, a.out_dtype, oidx + j, o[j], a.tc);
  }
  if (n_degenerate) atomicAdd(a.flags + kFlagDegenerate, n_degenerate);
  if (n_nonfinite) atomicAdd(a.flags + kFlagNonfiniteOut, n_nonfinite);
}

// Which small images take the fused kernel.  Default: Gaussian windows only.  Measured on a B200
// (tools/small_check.py, tools/diag_latency.py): c0 (Gaussian W = 9, N = 15) 28 us against
// 20.7 + 15.1 us for kernel 1 + kernel 2 (graph-replayed call 35 against 39-43 us); c1 (box
// W = 5, N = 10) 43 us against 23.1 + 20.5 us, and its graph-replayed call 55 against 46 us, so
// box windows keep the two kernels.  FBGPU_SMALL_FUSED=1 fuses both kinds, =0 neither.
inline bool small_fused_enabled(int kind) {
  static const int mode = [] {
    const char* e = std::getenv("FBGPU_SMALL_FUSED");
    return !e || !*e ? -1 : (*e == '0' ? 0 : 1);
  }();
  return mode < 0 ? kind == kKindGauss : mode != 0;
}

// Host: one launch for the band (returns 0, or 6 on a launch error).
template <int KIND, int WT>
int launch_small(cudaStream_t st, GpaArgs<float>& a, const KernelEvents& ev) {
  auto k = k_small_fused<KIND, WT>;
  const size_t smem = sm_smem_bytes(WT);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 6;
  a.lead = KIND == kKindBox ? box_lead(a, SM_T) : 0;
  const dim3 grid((a.cols + SM_T - 1) / SM_T, (a.band_rows + a.lead + SM_T - 1) / SM_T);
  record_timing(ev.k1_start, st);
  k<<<grid, SM_THREADS, smem, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return 6;
  record_timing(ev.k1_end, st);
  record_timing(ev.k2_end, st);
  if (ev.launched) *ev.launched = 1;
  return 0;
}

}  // namespace small
}  // namespace fbgpu
