// fb_fused.cuh — single-pass (fused) box GPA filter: SURVEY §8(f) rank 2, built to be measured.
//
// One kernel per band, no channel planes in HBM.  A CTA owns a strip of 64 output columns and
// walks CH image-anchored rows (as the box walker does).  Three warp roles form a pipeline over
// the rows of the walk, handing rows through shared-memory rings guarded by mbarriers:
//   walker  (4 warps, one padded column per thread, 64 + 2W <= 128 used): the vertical running
//           sums of the N+1 channels with Kahan compensation (k1f_box_walk's arithmetic); each
//           completed row's sums go to a row slot [channel][column];
//   window  (2 warps, one channel per thread): the horizontal box sums of the row for its
//           channel, two 32-column running sums, into a sums slot [channel][column];
//   horner  (2 warps, one output pixel per thread): the fp64 recurrences over the channels of
//           the sums slot, then the quotient and the store.
// The walker's 240 registers leave one 256-thread CTA per SM (8 warps).
#pragma once
#include "fb_fast.cuh"

namespace fbgpu {
namespace fused {

using fast::cp_async4;
using fast::cp_async_commit;
using fast::cp_async_wait;
using fast::ddiv_newton;
using fast::f2_add;
using fast::f2_hi;
using fast::f2_lo;
using fast::f2_mul;
using fast::f2_pack;
using fast::f2_sub;
using fast::f2_t;
using fast::mbar_arrive;
using fast::mbar_fence_init;
using fast::mbar_init;
using fast::mbar_wait;

constexpr int FU_TW = 64;         // output columns per CTA
constexpr int FU_WALK = 128;      // walker threads (padded columns 64 + 2W <= 128)
constexpr int FU_WIN = 64;        // window threads (one per channel, N + 1 <= 64)
constexpr int FU_HOR = 64;        // Horner threads (one per output column)
constexpr int FU_THREADS = FU_WALK + FU_WIN + FU_HOR;
constexpr int FU_NR = 4;          // row slots (walker -> window)
constexpr int FU_NH = 4;          // sums slots (window -> Horner)
constexpr int FU_DEPTH = 8;       // cp.async ring depth of the walker's samples

__host__ __device__ constexpr int fu_rb(int W) { return ((FU_TW + 2 * W) | 1); }  // odd: conflict-free
constexpr int FU_HB = FU_TW + 1;  // sums slot row stride (odd)
inline size_t fu_smem_bytes(int nch, int W) {
  return 128 + (size_t)FU_DEPTH * 2 * FU_WALK * 4 + (size_t)FU_NR * nch * fu_rb(W) * 4 +
         (size_t)FU_NH * nch * FU_HB * 4 + 2 * (FU_NR + FU_NH) * 8;
}

template <int NCH, int WT>
__global__ void __launch_bounds__(FU_THREADS, 1) k_fused_box(const __grid_constant__ GpaArgs<float> a) {
  extern __shared__ __align__(128) float fu_smem[];
  constexpr int RB = fu_rb(WT);
  constexpr int W = WT;
  const uint32_t sbase = fast::smem_u32(fu_smem);
  float* sm = fu_smem + (((sbase + 127u) & ~127u) - sbase) / 4;
  float (*ring)[2][FU_WALK] = reinterpret_cast<float (*)[2][FU_WALK]>(sm);
  float* rowbuf = sm + FU_DEPTH * 2 * FU_WALK;          // [FU_NR][NCH][RB]
  float* hbuf = rowbuf + FU_NR * NCH * RB;              // [FU_NH][NCH][FU_HB]
  uint64_t* rb_full = reinterpret_cast<uint64_t*>(hbuf + FU_NH * NCH * FU_HB);
  uint64_t* rb_empty = rb_full + FU_NR;
  uint64_t* hb_full = rb_empty + FU_NR;
  uint64_t* hb_empty = hb_full + FU_NH;

  const int N = a.N;
  const int CH = a.walk_rows;
  const int x0 = blockIdx.x * FU_TW;                     // first output column of the strip
  const int r0 = blockIdx.y * CH - a.lead;               // first band row of the walk (image-anchored)
  const int rows_here = min(CH, a.band_rows - r0);
  const int first = max(r0, 0);                          // first stored row
  const int nrows = r0 + rows_here - first;              // rows this CTA outputs
  const long long row_base = (long long)a.halo_top + a.band_row0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < FU_NR; ++s) {
      mbar_init(rb_full + s, FU_WALK);
      mbar_init(rb_empty + s, FU_WIN);
    }
    for (int s = 0; s < FU_NH; ++s) {
      mbar_init(hb_full + s, FU_WIN);
      mbar_init(hb_empty + s, FU_HOR);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (threadIdx.x < FU_WALK) {
    // ---------------- walker: column pc of the strip (image column x0 - W + pc)
    const int pc = threadIdx.x;
    const int scol = min(max(x0 - W + pc, 0), a.cols - 1);
    const bool own_col = pc >= W && pc < W + FU_TW && x0 - W + pc < a.cols;
    const float* f32 = reinterpret_cast<const float*>(a.f) + scol;
    const f2_t* q2 = reinterpret_cast<const f2_t*>(a.walkq);
    const int steps = rows_here + 2 * W;
    auto issue = [&](int st) {
      cp_async4(&ring[st % FU_DEPTH][0][pc], f32 + sample_row(a, row_base + r0 - W + st));
      cp_async4(&ring[st % FU_DEPTH][1][pc], f32 + sample_row(a, row_base + r0 - 3 * W - 1 + st));
    };
    constexpr int NPR = NCH / 2;
    f2_t S2[NPR], C2[NPR];
#pragma unroll
    for (int k = 0; k < NPR; ++k) S2[k] = C2[k] = 0ull;
    unsigned long long bad_nf = ~0ull, bad_rg = ~0ull;
#pragma unroll
    for (int d = 0; d < FU_DEPTH - 1; ++d) {
      if (d < steps) issue(d);
      cp_async_commit();
    }
    int slot = 0;
    uint32_t eph = 1;  // parity of rb_empty's phase that frees `slot` (first pass: no wait)
    int stored = 0;
    for (int st = 0; st < steps; ++st) {
      const int enter = r0 - W + st;
      if (st + FU_DEPTH - 1 < steps) issue(st + FU_DEPTH - 1);
      cp_async_commit();
      cp_async_wait<FU_DEPTH - 1>();
      const float fe = ring[st % FU_DEPTH][0][pc], fl = ring[st % FU_DEPTH][1][pc];
      if (a.check && own_col && enter >= first && enter < r0 + rows_here) {
        const bool nf = !isfinite(fe), rg = fe < a.lo || fe > a.hi;
        if ((nf && bad_nf == ~0ull) || (rg && bad_rg == ~0ull)) {
          long long b = row_base + enter;
          b = b < 0 ? 0 : (b >= a.rows_in ? a.rows_in - 1 : b);
          const unsigned long long idx = (unsigned long long)b * a.cols + scol;
          if (nf && bad_nf == ~0ull) bad_nf = idx;
          if (rg && bad_rg == ~0ull) bad_rg = idx;
        }
      }
      const float keep = st >= 2 * W + 1 ? 1.f : 0.f;
      const float xe = (float)((fe - a.tc) * a.inv_sr), xl = (float)((fl - a.tc) * a.inv_sr);
      const float ee = expf(-0.5f * xe * xe), el = keep * expf(-0.5f * xl * xl);
      f2_t E2 = f2_pack(ee, ee * xe), L2 = f2_pack(el, el * xl);
      const float xxe = xe * xe, xxl = xl * xl;
#pragma unroll
      for (int k = 0; k < NPR; ++k) {
        if (k > 0) {
          E2 = f2_mul(E2, f2_mul(f2_pack(xxe, xxe), q2[k]));
          L2 = f2_mul(L2, f2_mul(f2_pack(xxl, xxl), q2[k]));
        }
        const f2_t y2 = f2_sub(f2_sub(E2, L2), C2[k]);
        const f2_t t2 = f2_add(S2[k], y2);
        C2[k] = f2_sub(f2_sub(t2, S2[k]), y2);
        S2[k] = t2;
      }
      if (enter - W >= first) {  // a completed row of the strip
        if (stored >= FU_NR) mbar_wait(rb_empty + slot, eph);
        float* dst = rowbuf + slot * NCH * RB + pc;
        if (pc < FU_TW + 2 * W) {
#pragma unroll
          for (int k = 0; k < NPR; ++k) {
            if (2 * k < NCH - 8 || 2 * k <= N) dst[(2 * k) * RB] = f2_lo(S2[k]);
            if (2 * k + 1 < NCH - 8 || 2 * k + 1 <= N) dst[(2 * k + 1) * RB] = f2_hi(S2[k]);
          }
        }
        mbar_arrive(rb_full + slot);
        ++stored;
        if (++slot == FU_NR) {
          slot = 0;
          eph ^= 1u;
        }
      }
    }
    cp_async_wait<0>();
    if (a.check) {
      flag_min(a.flags + kFlagFirstNonfinite, bad_nf != ~0ull, bad_nf);
      flag_min(a.flags + kFlagFirstRange, bad_rg != ~0ull, bad_rg);
    }
    return;
  }

  if (threadIdx.x < FU_WALK + FU_WIN) {
    // ---------------- window: channel m = thread; two 32-output running sums per row
    const int m = threadIdx.x - FU_WALK;
    const bool active = m <= N;
    int slot = 0, hs = 0;
    uint32_t fph = 0, eph = 1;
    for (int i = 0; i < nrows; ++i) {
      mbar_wait(rb_full + slot, fph);
      if (i >= FU_NH) mbar_wait(hb_empty + hs, eph);
      if (active) {
        const float* src = rowbuf + slot * NCH * RB + m * RB;
        float* dst = hbuf + hs * NCH * FU_HB + m * FU_HB;
        float s0 = 0.f, s1 = 0.f;  // segments [0, 32) and [32, 64)
#pragma unroll
        for (int k = 0; k <= 2 * W; ++k) {
          s0 += src[k];
          s1 += src[32 + k];
        }
        dst[0] = s0;
        dst[32] = s1;
#pragma unroll 4
        for (int j = 1; j < 32; ++j) {
          s0 += src[j + 2 * W] - src[j - 1];
          s1 += src[32 + j + 2 * W] - src[32 + j - 1];
          dst[j] = s0;
          dst[32 + j] = s1;
        }
      }
      mbar_arrive(rb_empty + slot);
      mbar_arrive(hb_full + hs);
      if (++slot == FU_NR) {
        slot = 0;
        fph ^= 1u;
      }
      if (++hs == FU_NH) {
        hs = 0;
        eph ^= 1u;
      }
    }
    return;
  }

  // ---------------- Horner: output column c of the strip, one row after the other
  const int c = threadIdx.x - FU_WALK - FU_WIN;
  const int col = x0 + c;
  const bool col_ok = col < a.cols;
  int hs = 0;
  uint32_t fph = 0;
  unsigned long long n_degenerate = 0, n_nonfinite = 0;
  for (int i = 0; i < nrows; ++i) {
    const int orow = first + i;
    const long long brow = row_base + orow;
    const double fv = col_ok ? load_sample(a.f, a.f_dtype, brow * a.f_ld + col) : 0.0;
    const double xd = (double)(float)((fv - a.tc) * a.inv_sr);
    double q = 0.0, u = 0.0;
    mbar_wait(hb_full + hs, fph);
    const float* src = hbuf + hs * NCH * FU_HB + c;
    for (int m = N; m >= 0; --m) {
      const double v = (double)src[m * FU_HB];
      const double t = xd * __ldg(a.tabd + 2 * (m + 1));  // h_{m+1} (unused for m = N)
      if (m < N) q = fma(t, q, v);
      else q = v;
      if (m > 0) u = fma(t, u, (double)m * v);
    }
    mbar_arrive(hb_empty + hs);
    if (++hs == FU_NH) {
      hs = 0;
      fph ^= 1u;
    }
    if (!col_ok) continue;
    double o = f32_result(a.sr * ddiv_newton(u, q), a.tc);
    if (fabs(q * (double)a.norm) < 1e-30) {  // Q floor (engine.py:20, 68)
      o = fv;
      ++n_degenerate;
    }
    n_nonfinite += !isfinite(o);
    store_sample(a.out, a.out_dtype, (long long)(a.band_row0 + orow) * a.out_ld + col, o, a.tc);
  }
  if (n_degenerate) atomicAdd(a.flags + kFlagDegenerate, n_degenerate);
  if (n_nonfinite) atomicAdd(a.flags + kFlagNonfiniteOut, n_nonfinite);
}

// Host: launch the fused kernel for a box band (returns 0, or 6 on a launch error).
template <int WT>
int launch_fused_box(cudaStream_t st, GpaArgs<float>& a, const KernelEvents& ev) {
  static void (*const kernels[8])(const GpaArgs<float>) = {
      k_fused_box<8, WT>,  k_fused_box<16, WT>, k_fused_box<24, WT>, k_fused_box<32, WT>,
      k_fused_box<40, WT>, k_fused_box<48, WT>, k_fused_box<56, WT>, k_fused_box<64, WT>};
  const int nch = (a.N + 1 + 7) / 8 * 8;
  auto k = kernels[nch / 8 - 1];
  const size_t smem = fu_smem_bytes(nch, a.W);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 6;
  const int ch = walk_rows(a.wpad, a.image_rows, FU_TW);
  a.walk_rows = ch;
  a.lead = box_lead(a, ch);
  a.tabd = a.tabd_walk;  // the walker's recurrence constants
  const dim3 grid((a.cols + FU_TW - 1) / FU_TW, (a.band_rows + a.lead + ch - 1) / ch);
  record_timing(ev.k1_start, st);
  k<<<grid, FU_THREADS, smem, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return 6;
  record_timing(ev.k1_end, st);
  record_timing(ev.k2_end, st);
  if (ev.launched) *ev.launched = 1;
  return 0;
}

}  // namespace fused
}  // namespace fbgpu
