// fb_capi.cu — the C ABI (include/fbgpu.h): context, workspace, row-band
// scheduling, kernel dispatch and error reporting.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/fbgpu.h"
#include "fb_analysis.cuh"
#include "fb_common.cuh"
#include "fb_generic.cuh"
#include "fb_fast.cuh"
#include "fb_hostwiden.cuh"

namespace fbgpu {
// ============================================================================ validation
__global__ void __launch_bounds__(256) k_validate(const void* f, long long ld, int dt, int rows, int cols,
                                                  double lo, double hi, unsigned long long* flags) {
  const long long total = (long long)rows * cols;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // Uniform trip count per warp so the ballot in flag_min sees full warps.
  const long long base0 = (long long)blockIdx.x * blockDim.x;
  for (long long base = base0; base < total; base += stride) {
    const long long i = base + threadIdx.x;
    const bool act = i < total;
    double v = 0.0;
    unsigned long long idx = 0;
    if (act) {
      const long long r = i / cols, c = i - r * cols;
      v = load_sample(f, dt, r * ld + c);
      idx = (unsigned long long)i;
    }
    check_sample(flags, act, v, lo, hi, idx);
  }
}

int launch_validate(cudaStream_t s, const void* f, long long ld, int dt, int rows, int cols, double lo,
                           double hi, unsigned long long* flags, int sms) {
  const long long total = (long long)rows * cols;
  long long blocks = (total + 255) / 256;
  blocks = blocks < (long long)sms * 8 ? blocks : (long long)sms * 8;
  k_validate<<<(int)blocks, 256, 0, s>>>(f, ld, dt, rows, cols, lo, hi, flags);
  return cudaGetLastError() == cudaSuccess ? 0 : 6;
}

}  // namespace fbgpu

using namespace fbgpu;

namespace {

thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define FB_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(_e == cudaErrorMemoryAllocation ? FB_ERR_NOMEM : FB_ERR_CUDA,        \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                 \
  } while (0)

size_t dtype_size(int dt) { return dt == FB_U8 ? 1 : (dt == FB_F32 ? 4 : 8); }

}  // namespace

struct fb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;      // compute stream (the caller's, or own_stream)
  cudaStream_t own_stream = nullptr;
  cudaStream_t s_h2d = nullptr;       // host -> device copies of the pipelined host path
  cudaStream_t s_d2h = nullptr;       // device -> host copies
  cudaStream_t s_alt = nullptr;       // second compute stream: odd images of a batch
  void* ws2 = nullptr;                // its workspace
  size_t ws2_bytes = 0;
  void* ws = nullptr;                 // channel planes of one row band
  size_t ws_bytes = 0;
  void* in_stage[2] = {nullptr, nullptr};   // device copies of host inputs (double-buffered per image)
  size_t in_stage_bytes[2] = {0, 0};
  void* out_stage[2] = {nullptr, nullptr};  // device outputs bound for host memory
  size_t out_stage_bytes[2] = {0, 0};
  unsigned long long* flags = nullptr;       // device, 4 slots per image of a batch
  unsigned long long* flags_host = nullptr;  // pinned readback
  int flags_cap = 0;                         // images the flag buffers hold
  float* tab = nullptr;                      // device channel-constant table (fp32 fast path)
  float* tab_host = nullptr;                 // pinned staging for it
  double* tabd = nullptr;                    // matching fp64 Horner constants
  double* tabd_host = nullptr;
  int tab_cap = 0;                           // channels it holds
  int tab_n = -1;                            // order N the table currently holds
  long long ws_limit = 0;
  int sm_count = 148;
  // small device scratch + pinned readback for the reductions of fb_error_stats / fb_kernel_error_sup
  double* scratch = nullptr;
  double* scratch_host = nullptr;
  size_t scratch_cap = 0;                    // doubles
  cudaEvent_t ev_start = nullptr, ev_kstart = nullptr, ev_kend = nullptr, ev_end = nullptr;
  // Per-band kernel boundaries: [k1 start, k1 end = k2 start, k2 end] x bands.
  std::vector<cudaEvent_t> kev;
  int kev_used = 0;
  std::vector<cudaEvent_t> pev;  // pipeline events (copy/compute hand-offs)
  int pev_used = 0;

  // CUDA-graph replay of repeated device-resident calls (key = everything the GPU work depends
  // on): first sighting runs eagerly, the second captures + instantiates, later ones replay.
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;  // kernels in the graph (for fb_launch_count)
    int kev_used = 0;        // per-band timing events it records
    int bands = 0;           // row bands it runs (stats)
    long long h2d = 0, d2h = 0;  // bytes its copies move (stats)
  };
  std::unordered_map<std::string, Graph> graphs;
  bool use_graphs = true;
  // A buffer a captured graph may reference was freed and reallocated (grow, ensure_flags, the
  // constant tables): every graph is dropped at the start of the next call (execute()).
  bool realloc_seen = false;
  // The caller's stream was the legacy (or per-thread) default stream, which cannot be captured
  // into graphs: work runs on own_stream, ordered after everything already queued there.
  cudaStream_t upstream = nullptr;
  cudaEvent_t ev_upstream = nullptr;
  // fp32 path, float64 host output: float32 centred rows cross PCIe and host threads widen them
  // (fb_hostwiden.cuh).  widen_threads < 0: not configured yet; 0: off.
  hostwiden::Pool* widen = nullptr;
  int widen_threads = -1;
  bool widen_used = false;  // the current call dispatched pieces to the host threads
  void clear_graphs() {
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }

  cudaEvent_t next_kev() { return take(kev, kev_used, cudaEventDefault); }
  cudaEvent_t next_pev() { return take(pev, pev_used, cudaEventDisableTiming); }
  static cudaEvent_t take(std::vector<cudaEvent_t>& pool, int& used, unsigned flags) {
    if (used == (int)pool.size()) {
      cudaEvent_t e = nullptr;
      cudaEventCreateWithFlags(&e, flags);
      pool.push_back(e);
    }
    return pool[used++];
  }
};

namespace {

int grow(fb_ctx* ctx, void** p, size_t* have, size_t need) {
  if (*have >= need) return FB_OK;
  ctx->realloc_seen = true;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(FB_ERR_NOMEM, std::string("cudaMalloc(") + std::to_string(need) + "): " + cudaGetErrorString(e));
  }
  *have = need;
  return FB_OK;
}

int check_image(const fb_image* im, const char* what, bool allow_u8) {
  if (!im || !im->data) return fail(FB_ERR_PARAM, std::string(what) + ": null image");
  if (im->rows <= 0 || im->cols <= 0)
    return fail(FB_ERR_PARAM, std::string(what) + ": image must be non-empty");
  if (im->ld < im->cols) return fail(FB_ERR_PARAM, std::string(what) + ": ld < cols");
  if (im->dtype != FB_F32 && im->dtype != FB_F64 && !(allow_u8 && im->dtype == FB_U8))
    return fail(FB_ERR_PARAM, std::string(what) + ": unsupported dtype");
  if (im->rows > (1ll << 30) || im->cols > (1ll << 30))
    return fail(FB_ERR_PARAM, std::string(what) + ": image too large");
  return FB_OK;
}

// Filter parameters shared by every image of a call, independent of precision.
struct Job {
  int kind, W, N, mode, check;
  const double* taps;
  double sr, tc, lo, hi;
};

// The precision-typed argument block: constants once per call, pointers per image.
template <typename T>
int prepare(fb_ctx* ctx, const Job& j, int cols, int rows_out_max, GpaArgs<T>& a, int* band_out) {
  memset(&a, 0, sizeof(a));
  a.W = j.W;
  a.N = j.N;
  a.mode = j.mode;
  a.check = j.check;
  a.tc = j.tc;
  a.sr = j.sr;
  a.inv_sr = j.mode == kModeGpa ? 1.0 / j.sr : 0.0;
  a.lo = j.lo;
  a.hi = j.hi;
  a.cols = cols;
  const int n_taps = 2 * j.W + 1;
  if (j.kind == FB_BOX) {
    a.norm = (T)(1.0 / ((double)n_taps * n_taps));
    for (int k = 0; k < n_taps; ++k) a.w[k] = T(1);
  } else {
    a.norm = T(1);
    for (int k = 0; k < n_taps; ++k) a.w[k] = (T)j.taps[k];
  }
  if (j.W <= kFastMaxW) {
    for (int q = 0; q <= n_taps; ++q) {
      a.wq[2 * q] = q < n_taps ? (float)a.w[q] : 0.f;
      a.wq[2 * q + 1] = q > 0 ? (float)a.w[q - 1] : 0.f;
    }
  }
  // Box walker multipliers: it steps each channel parity by two orders at once,
  // c_n = c_{n-2} * x^2 * q_n with q_n = fl32(1/sqrt((n-1) n)) (q_1 = 1: c_1 = c_0 x), so the
  // even and odd chains are independent (read as (q_2k, q_2k+1) pairs for packed multiplies).
  for (int m = 0; m < kWalkMaxCh; ++m) a.walkq[m] = walk_q(m);  // (the fused prototype's walker, fb_fused.cuh)
  // The production walker: channel m = e^{-x^2/2} (x / s)^m / m!  (fb_common.cuh: taylor_scale)
  a.walk_xs = (float)(1.0 / taylor_scale(j.N));
  a.taylor_s = 1.0 / (double)a.walk_xs;
  // Two-step multipliers q_n ~ 1 / ((n-1) n), each chosen so that the product the walker really
  // applies, A_n = q_n A_{n-2} (fp32 constants, exact products), is the fp32-nearest to 1/n!:
  // the constants' representation errors do not accumulate along the chain, every order is within
  // one fp32 rounding (6e-8) of its Taylor weight, the noise floor of the fp32 planes themselves.
  // (Plain fl32(1/((n-1) n)) drifts by ~n/2 roundings: over 5e-4 gray levels at c4 against the fp64
  // path, 2.7e-4 with these constants -- the level of the 1/sqrt(n!) planes with exact fp64 compensation.)
  {
    double A[kWalkMaxCh], fact = 1.0;
    for (int m = 0; m < kWalkMaxCh; ++m) {
      if (m >= 1) fact *= (double)m;
      if (m < 2) {
        a.walkt[m] = 1.f;
        A[m] = 1.0;
      } else {
        a.walkt[m] = (float)((1.0 / fact) / A[m - 2]);
        A[m] = A[m - 2] * (double)a.walkt[m];
      }
    }
  }
  // channel constants 1/sqrt(m), sqrt(m) (rounded once from double), uploaded when N changes
  if (j.N + 1 > ctx->tab_cap) {
    ctx->realloc_seen = true;
    for (void* p : {(void*)ctx->tab, (void*)ctx->tabd}) if (p) cudaFree(p);
    for (void* p : {(void*)ctx->tab_host, (void*)ctx->tabd_host}) if (p) cudaFreeHost(p);
    ctx->tab = nullptr;
    ctx->tab_host = nullptr;
    ctx->tabd = nullptr;
    ctx->tabd_host = nullptr;
    ctx->tab_cap = 0;
    ctx->tab_n = -1;
    const int cap = std::max(j.N + 1, 256);
    FB_CUDA(cudaMalloc(&ctx->tab, 4 * sizeof(float) * cap));
    FB_CUDA(cudaMallocHost(&ctx->tab_host, 4 * sizeof(float) * cap));
    FB_CUDA(cudaMalloc(&ctx->tabd, 7 * sizeof(double) * cap));  // [sequential | walker | tile | Taylor r] sections
    FB_CUDA(cudaMallocHost(&ctx->tabd_host, 7 * sizeof(double) * cap));
    ctx->tab_cap = cap;
  }
  if (ctx->tab_n != j.N) {
    FB_CUDA(cudaStreamSynchronize(ctx->stream));  // the pinned staging may still feed an earlier copy
    for (int m = 0; m <= j.N; ++m) {
      // r_m: the fp32 constant kernel 1 multiplies channel m by.  The fp64 Horner constants are
      // derived from r_m itself so the normalisation cancels exactly (no 1/sqrt(n!) drift).
      const float r = m > 0 ? (float)(1.0 / std::sqrt((double)m)) : 0.f;
      const double h = m > 0 ? 1.0 / ((double)m * (double)r) : 0.0;
      const double sg = m > 0 ? 1.0 / (double)r : 0.0;
      ctx->tab_host[4 * m] = r;
      ctx->tab_host[4 * m + 1] = (float)std::sqrt((double)m);
      ctx->tab_host[4 * m + 2] = (float)h;
      ctx->tab_host[4 * m + 3] = (float)sg;
      ctx->tabd_host[2 * m] = h;
      ctx->tabd_host[2 * m + 1] = sg;
    }
    // The same constants for planes made by the box walker: its channel m carries the
    // normalisation A_m = q_m A_{m-2} (A_0 = A_1 = 1), i.e. an effective r'_m = A_m / A_{m-1}.
    double* wd = ctx->tabd_host + 2 * ctx->tab_cap;
    double A2 = 1.0, A1 = 1.0;  // A_{m-2}, A_{m-1}
    for (int m = 0; m <= j.N; ++m) {
      double h = 0.0, sg = 0.0;
      if (m >= 1 && m < kWalkMaxCh) {
        const double Am = m == 1 ? 1.0 : (double)walk_q(m) * A2;
        const double r = Am / A1;
        h = 1.0 / ((double)m * r);
        sg = 1.0 / r;
        A2 = A1;
        A1 = Am;
      }
      wd[2 * m] = h;
      wd[2 * m + 1] = sg;
    }
    // ... and for planes made by the fp32 tile kernel 1, whose every order is multiplied by kappa
    double* td = ctx->tabd_host + 4 * ctx->tab_cap;
    const double kap = (double)tile_kappa(j.N);
    for (int m = 0; m <= j.N; ++m) {
      td[2 * m] = m > 0 ? 1.0 / ((double)m * kap) : 0.0;
      td[2 * m + 1] = m > 0 ? 1.0 / kap : 0.0;
    }
    FB_CUDA(cudaMemcpyAsync(ctx->tab, ctx->tab_host, 4 * sizeof(float) * (j.N + 1), cudaMemcpyHostToDevice,
                            ctx->stream));
    // ... and the per-order factors of the fp64 kernels' Taylor planes
    double* tr = ctx->tabd_host + 6 * ctx->tab_cap;
    const double ts = 1.0 / (double)(float)(1.0 / taylor_scale(j.N));  // = GpaArgs::taylor_s below
    for (int m = 0; m <= j.N; ++m) tr[m] = m > 0 ? 1.0 / ((double)m * ts) : 0.0;
    FB_CUDA(cudaMemcpyAsync(ctx->tabd, ctx->tabd_host, 7 * sizeof(double) * ctx->tab_cap, cudaMemcpyHostToDevice,
                            ctx->stream));
    ctx->tab_n = j.N;
  }
  a.tab = ctx->tab;
  a.tabd = a.tabd_seq = ctx->tabd;
  a.tabd_walk = ctx->tabd + 2 * ctx->tab_cap;
  a.tabd_tile = ctx->tabd + 4 * ctx->tab_cap;
  a.taylor_r = ctx->tabd + 6 * ctx->tab_cap;
  a.kappa = tile_kappa(j.N);
  a.wpad = cols + 2 * j.W;
  a.pitch = (a.wpad + 31) / 32 * 32;
  // Row bands: the N+1 planes of one band must fit under the workspace limit.
  const long long per_row = (long long)(j.N + 1) * a.pitch * (long long)sizeof(T);
  // Bands start at multiples of 256 image rows when they can (the box walks and tiles then
  // start at the band's first row: no rows above it are walked, see walk_rows()).
  long long band = ctx->ws_limit / std::max(per_row, 1ll);
  band = band >= 256 ? band / 256 * 256 : band / 64 * 64;
  if (band < 64) band = 64;
  const long long rows_pad = (rows_out_max + 63) / 64 * 64;
  if (band > rows_pad) band = rows_pad;
  a.rstride = (long long)(j.N + 1) * a.pitch;
  a.band_max = (int)band;
  int rc = grow(ctx, &ctx->ws, &ctx->ws_bytes, (size_t)band * a.rstride * sizeof(T));
  if (rc != FB_OK) return rc;
  a.v = reinterpret_cast<T*>(ctx->ws);
  *band_out = (int)band;
  return FB_OK;
}

template <typename T>
int launch_band(fb_ctx* ctx, cudaStream_t st, int kind, GpaArgs<T>& a, int band_row0, int band_rows) {
  a.band_row0 = band_row0;
  a.band_rows = band_rows;
  const int W = a.W;
  bool done = false;
  cudaEvent_t e0 = ctx->next_kev(), e1 = ctx->next_kev(), e2 = ctx->next_kev();
  int launched = 2;
  KernelEvents kev{e0, e1, e2, &launched};
  int rc = launch_fast<T>(st, kind, W, a, kev, &done);
  if (rc != FB_OK) return fail(FB_ERR_CUDA, std::string("fast kernel launch failed: ") +
                                               cudaGetErrorString(cudaGetLastError()));
  if (done) {
    g_launches += launched;
    return FB_OK;
  }
  const size_t s1 = generic::k1_smem<T>(W), s2 = generic::k2_smem<T>(W);
  a.lead = kind == FB_BOX ? box_lead(a, generic::K1_RB) : 0;
  dim3 g1((a.wpad + generic::K1_TC - 1) / generic::K1_TC,
          (band_rows + a.lead + generic::K1_RB - 1) / generic::K1_RB);
  dim3 g2((a.cols + generic::K2_TW - 1) / generic::K2_TW, (band_rows + generic::K2_TH - 1) / generic::K2_TH);
  auto k1 = kind == FB_BOX ? generic::k1_gen_vpass<T, kKindBox> : generic::k1_gen_vpass<T, kKindGauss>;
  auto k2 = kind == FB_BOX ? generic::k2_hpass_horner<T, kKindBox> : generic::k2_hpass_horner<T, kKindGauss>;
  FB_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1));
  FB_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2));
  FB_CUDA(record_timing(e0, st));
  k1<<<g1, generic::K1_TC * generic::K1_RG, s1, st>>>(a);
  FB_CUDA(cudaGetLastError());
  FB_CUDA(record_timing(e1, st));
  k2<<<g2, 256, s2, st>>>(a);
  FB_CUDA(cudaGetLastError());
  FB_CUDA(record_timing(e2, st));
  g_launches += 2;
  return FB_OK;
}

// Output rows [r0, r1) of one image, in workspace-sized bands.
template <typename T>
int run_rows(fb_ctx* ctx, cudaStream_t st, int kind, GpaArgs<T>& a, int band, int r0, int r1, int* bands) {
  for (int b0 = r0; b0 < r1; b0 += band) {
    int rc = launch_band<T>(ctx, st, kind, a, b0, std::min(band, r1 - b0));
    if (rc != FB_OK) return rc;
    ++*bands;
  }
  return FB_OK;
}

// Where the output rows of a call sit in the whole image, and where its halo rows come from.
struct Geom {
  long long row_origin = 0;         // image row of output row 0
  long long image_rows = 0;         // rows of the whole image (0: the output rows are the image)
  const fb_image* above = nullptr;  // halo rows in separate device buffers (fb_gpa_filter_band);
  const fb_image* below = nullptr;  // else the halo rows are part of the input buffer
  bool separate() const { return above != nullptr || below != nullptr; }
  long long report_rows = 0;        // stats->bad_index counts rows from this many rows below the buffer start
};

// One image of a call: where its data lives on the device and how it is chunked.
struct Item {
  const fb_image* in;
  fb_image* out;
  const void* f;  // device input
  long long f_ld;
  void* o;        // device output
  long long o_ld;
  int rows_out;
  int chunks;     // > 1: a host image pipelined in row chunks
  int crows;      // most rows a chunk has
  std::vector<int> ends;  // last row + 1 of every chunk (multiples of 256 but the last)
  bool widen;     // float64 host output: the float32 centred result crosses PCIe, host threads widen it
};

// float32 over PCIe + host widening (fb_hostwiden.cuh) applies to the fp32-precision images of a
// call whose float64 output lives in host memory, when the call is too large for CUDA-graph replay
// (kGraphMaxPixels; smaller calls are latency-bound and a replay beats the saved bytes: c2, 16.8 MP,
// 3.0 ms replayed against 3.9 ms widened).  float64 inputs keep the float64 transfer.
constexpr long long kGraphMaxPixels = 16ll << 20;  // calls up to 16 MP run as CUDA graphs
bool widen_applies(fb_ctx* ctx, const fb_image* in, const fb_image* out, int precision, long long call_px) {
  if (ctx->widen_threads < 0) ctx->widen_threads = hostwiden::configured_threads();
  return ctx->widen_threads > 0 && precision != FB_PREC_F64 && out && !out->on_device && out->dtype == FB_F64 &&
         in->dtype != FB_F64 && call_px > kGraphMaxPixels;
}
// Copy-in / filter / copy-out for `count` images.  Host-resident images are pipelined in
// row chunks over three streams: H2D of chunk c+1 || kernels of chunk c || D2H of chunk c-1.
#ifndef FB_CHUNK_PX
#define FB_CHUNK_PX (8ll << 20)
#endif
#ifndef FB_CHUNK_MIN
#define FB_CHUNK_MIN 8
#endif
// Kernels of a chunk wait for the input rows they read (chunk rows + W halo rows).
template <typename T>
int run_items(fb_ctx* ctx, std::vector<Item>& items, int halo_top, int halo_bottom, const Job& j,
              fb_stats* st, const Geom& geo) {
  const bool validate_only = items[0].out == nullptr;
  int band = 0;
  GpaArgs<T> a;
  int rows_max = 0;  // rows one launch sequence covers: an image, or one chunk of it
  for (auto& it : items) rows_max = std::max(rows_max, std::min(it.rows_out, it.crows));
  if (!validate_only) {
    int rc = prepare<T>(ctx, j, (int)items[0].in->cols, rows_max, a, &band);
    if (rc != FB_OK) return rc;
  }
  // Batches alternate images between two compute streams with two workspaces, so the kernels
  // of image i+1 fill the tail waves of image i.  (The chunks of one large host image stay on one
  // stream: alternating them measured the same, 37.8 against 38.3 ms per c4 call -- that path is
  // bound by host memory traffic, profiles/r02_hostwiden.md.)
  const bool dual = !validate_only && items.size() > 1;
  cudaStream_t cs[2] = {ctx->stream, dual ? ctx->s_alt : ctx->stream};
  T* wsp[2] = {a.v, a.v};
  if (dual) {
    int rc = grow(ctx, &ctx->ws2, &ctx->ws2_bytes, (size_t)band * a.rstride * sizeof(T));
    if (rc != FB_OK) return rc;
    wsp[1] = reinterpret_cast<T*>(ctx->ws2);
    cudaEvent_t e = ctx->next_pev();  // after the constant-table upload in prepare()
    FB_CUDA(cudaEventRecord(e, ctx->stream));
    FB_CUDA(cudaStreamWaitEvent(ctx->s_alt, e, 0));
  }
  bool any_host = false;  // the copy streams join only when some image lives in host memory
  for (auto& it : items) any_host |= !it.in->on_device || (it.out && !it.out->on_device);
  if (any_host) {
    // fork the copy streams from the compute stream (an event recorded here, so a stream capture
    // of this call takes them along)
    cudaEvent_t fork = ctx->next_pev();
    FB_CUDA(cudaEventRecord(fork, ctx->stream));
    FB_CUDA(cudaStreamWaitEvent(ctx->s_h2d, fork, 0));
    FB_CUDA(cudaStreamWaitEvent(ctx->s_d2h, fork, 0));
  }
  std::vector<cudaEvent_t> img_done(items.size(), nullptr);  // compute finished with image i's buffers
  std::vector<cudaEvent_t> out_done(items.size(), nullptr);  // D2H of image i finished
  for (size_t i = 0; i < items.size(); ++i) {
    Item& it = items[i];
    const fb_image* in = it.in;
    const size_t ies = dtype_size(in->dtype);
    const int slot = (int)(i & 1);  // staging buffers of the image
    const bool host_in = !in->on_device;
    const bool host_out = it.out && !it.out->on_device;
    const bool widen = !validate_only && it.widen;
    // device buffers (double-buffered across images; reuse waits for image i-2)
    if (host_in) {
      int rc = grow(ctx, &ctx->in_stage[slot], &ctx->in_stage_bytes[slot], (size_t)in->rows * in->cols * ies);
      if (rc != FB_OK) return rc;
      it.f = ctx->in_stage[slot];
      it.f_ld = in->cols;
      if (i >= 2) FB_CUDA(cudaStreamWaitEvent(ctx->s_h2d, img_done[i - 2], 0));
    } else {
      it.f = in->data;
      it.f_ld = in->ld;
    }
    if (it.out) {
      const size_t oes = widen ? sizeof(float) : dtype_size(it.out->dtype);
      if (host_out) {
        int rc = grow(ctx, &ctx->out_stage[slot], &ctx->out_stage_bytes[slot], (size_t)it.rows_out * it.out->cols * oes);
        if (rc != FB_OK) return rc;
        it.o = ctx->out_stage[slot];
        it.o_ld = it.out->cols;
        if (i >= 2) FB_CUDA(cudaStreamWaitEvent(cs[slot], out_done[i - 2], 0));
      } else {
        it.o = it.out->data;
        it.o_ld = it.out->ld;
      }
    }
    const int W = validate_only ? 0 : j.W;
    size_t stage_off = 0;  // where the image's float32 rows start in the pinned staging area
    if (widen) {  // (execute() reserved the staging area for the whole call)
      for (size_t k = 0; k < i; ++k)
        if (items[k].widen) stage_off += (size_t)items[k].rows_out * items[k].out->cols * sizeof(float);
    }
    long long copied = 0;  // input buffer rows already sent
    int r0 = 0;
    for (size_t ci = 0; ci < it.ends.size(); r0 = it.ends[ci], ++ci) {
      const int r1 = it.ends[ci];
      cudaStream_t cstr = cs[slot];
      if (host_in) {
        // input buffer rows this chunk reads: [halo_top + r0 - W, halo_top + r1 + W) clamped
        const long long need = std::min<long long>(in->rows, (long long)halo_top + r1 + W);
        const long long hi = (r1 == it.rows_out) ? in->rows : need;  // the last chunk sends the rest
        if (hi > copied) {
          FB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(const_cast<void*>(it.f)) + copied * in->cols * ies,
                                    in->cols * ies, static_cast<const char*>(in->data) + copied * in->ld * ies,
                                    in->ld * ies, in->cols * ies, hi - copied, cudaMemcpyHostToDevice,
                                    ctx->s_h2d));
          if (st) st->h2d_bytes += (hi - copied) * in->cols * (long long)ies;
          copied = hi;
        }
        cudaEvent_t e = ctx->next_pev();
        FB_CUDA(cudaEventRecord(e, ctx->s_h2d));
        FB_CUDA(cudaStreamWaitEvent(cstr, e, 0));
      }
      if (validate_only) {
        int rc = launch_validate(cstr, it.f, it.f_ld, in->dtype, (int)in->rows, (int)in->cols, j.lo, j.hi,
                                 ctx->flags + 4 * i, ctx->sm_count);
        if (rc != FB_OK) return fail(FB_ERR_CUDA, "validation kernel launch failed");
        g_launches += 1;
      } else {
        a.f_ld = it.f_ld;
        a.f_dtype = in->dtype;
        a.halo_top = halo_top;
        a.rows_in = halo_top + it.rows_out + halo_bottom;
        a.main_end = halo_top + it.rows_out;
        a.row_origin = geo.row_origin;
        a.image_rows = (int)(geo.image_rows > 0 ? geo.image_rows : it.rows_out);
        if (geo.separate()) {
          // own rows from `in`, halo rows from the neighbours' buffers: offsets relative to a
          // virtual buffer row 0 that sits halo_top rows above in->data (never dereferenced)
          const long long ies_l = (long long)ies;
          const intptr_t f0 = reinterpret_cast<intptr_t>(it.f) - (intptr_t)halo_top * it.f_ld * ies_l;
          a.f = reinterpret_cast<const void*>(f0);
          a.top_off = geo.above ? (reinterpret_cast<intptr_t>(geo.above->data) - f0) / ies_l : 0;
          a.top_ld = geo.above ? geo.above->ld : it.f_ld;
          a.bot_off = geo.below ? (reinterpret_cast<intptr_t>(geo.below->data) - f0) / ies_l : 0;
          a.bot_ld = geo.below ? geo.below->ld : it.f_ld;
        } else {
          a.f = it.f;
          a.top_off = 0;
          a.top_ld = it.f_ld;
          a.bot_off = (long long)a.main_end * it.f_ld;
          a.bot_ld = it.f_ld;
        }
        a.out = it.o;
        a.out_ld = it.o_ld;
        a.out_dtype = widen ? (j.mode == kModeGpa ? kOutF32Centred : FB_F32) : it.out->dtype;
        a.flags = ctx->flags + 4 * i;
        a.v = wsp[slot];
        int nb = 0;
        int rc = run_rows<T>(ctx, cstr, j.kind, a, band, r0, r1, &nb);
        if (rc != FB_OK) return rc;
        if (st) st->bands += nb;
      }
      if (host_out) {
        cudaEvent_t e = ctx->next_pev();
        FB_CUDA(cudaEventRecord(e, cstr));
        FB_CUDA(cudaStreamWaitEvent(ctx->s_d2h, e, 0));
        if (widen) {
          // float32 rows -> pinned staging, in pieces; the dispatcher hands each to the workers as it lands
          const size_t row_bytes = (size_t)it.out->cols * sizeof(float);
          const int prow = (int)std::max<size_t>(1, hostwiden::piece_bytes() / row_bytes);
          for (int p0 = r0; p0 < r1; p0 += prow) {
            const int p1 = std::min(r1, p0 + prow);
            hostwiden::Task t;
            t.src = ctx->widen->stage(stage_off + (size_t)p0 * row_bytes);
            t.dst = static_cast<double*>(it.out->data) + (size_t)p0 * it.out->ld;
            t.rows = p1 - p0;
            t.cols = it.out->cols;
            t.dst_ld = it.out->ld;
            t.add = j.mode == kModeGpa ? j.tc : 0.0;
            FB_CUDA(cudaMemcpyAsync(const_cast<float*>(t.src), static_cast<char*>(it.o) + (size_t)p0 * it.o_ld * sizeof(float),
                                    (size_t)(p1 - p0) * row_bytes, cudaMemcpyDeviceToHost, ctx->s_d2h));
            cudaEvent_t landed = ctx->next_pev();
            FB_CUDA(cudaEventRecord(landed, ctx->s_d2h));
            ctx->widen->dispatch(landed, t);
            ctx->widen_used = true;
          }
          if (st) st->d2h_bytes += (long long)(r1 - r0) * it.out->cols * (long long)sizeof(float);
        } else {
          const size_t oes = dtype_size(it.out->dtype);
          FB_CUDA(cudaMemcpy2DAsync(static_cast<char*>(it.out->data) + (size_t)r0 * it.out->ld * oes,
                                    it.out->ld * oes, static_cast<char*>(it.o) + (size_t)r0 * it.o_ld * oes,
                                    it.o_ld * oes, it.out->cols * oes, r1 - r0, cudaMemcpyDeviceToHost, ctx->s_d2h));
          if (st) st->d2h_bytes += (long long)(r1 - r0) * it.out->cols * (long long)oes;
        }
      }
    }
    img_done[i] = ctx->next_pev();
    FB_CUDA(cudaEventRecord(img_done[i], cs[slot]));
    out_done[i] = ctx->next_pev();
    FB_CUDA(cudaEventRecord(out_done[i], host_out ? ctx->s_d2h : cs[slot]));
  }
  // join the copy streams and the second compute stream back into the main stream
  cudaEvent_t e1 = ctx->next_pev(), e2 = ctx->next_pev(), e3 = ctx->next_pev();
  if (any_host) {
    FB_CUDA(cudaEventRecord(e1, ctx->s_h2d));
    FB_CUDA(cudaEventRecord(e2, ctx->s_d2h));
    FB_CUDA(cudaStreamWaitEvent(ctx->stream, e1, 0));
    FB_CUDA(cudaStreamWaitEvent(ctx->stream, e2, 0));
  }
  if (dual) {
    FB_CUDA(cudaEventRecord(e3, ctx->s_alt));
    FB_CUDA(cudaStreamWaitEvent(ctx->stream, e3, 0));
  }
  return FB_OK;
}

int ensure_flags(fb_ctx* ctx, int count) {
  if (count <= ctx->flags_cap) return FB_OK;
  ctx->realloc_seen = true;
  if (ctx->flags) cudaFree(ctx->flags);
  if (ctx->flags_host) cudaFreeHost(ctx->flags_host);
  ctx->flags = nullptr;
  ctx->flags_host = nullptr;
  ctx->flags_cap = 0;
  const int cap = std::max(count, 64);
  FB_CUDA(cudaMalloc(&ctx->flags, 4 * sizeof(unsigned long long) * cap));
  FB_CUDA(cudaMallocHost(&ctx->flags_host, 8 * sizeof(unsigned long long) * cap));
  for (int i = 0; i < cap; ++i) {
    unsigned long long* init = ctx->flags_host + 4 * i;  // first half: the reset pattern
    init[kFlagFirstNonfinite] = ~0ull;
    init[kFlagFirstRange] = ~0ull;
    init[kFlagDegenerate] = 0;
    init[kFlagNonfiniteOut] = 0;
  }
  ctx->flags_cap = cap;
  return FB_OK;
}

// The caller bound the legacy / per-thread default stream (fb_set_stream): order the context's
// stream after the work already queued there (e.g. a torch kernel still writing the input).
int order_after_caller(fb_ctx* ctx) {
  if (!ctx->upstream) return FB_OK;
  FB_CUDA(cudaEventRecord(ctx->ev_upstream, ctx->upstream));
  FB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_upstream, 0));
  return FB_OK;
}

// Run `count` images through the pipeline, read the flags back and map them to a status.

// Everything the GPU work of a device-resident call depends on: the images (pointers, shapes,
// strides, dtypes), the filter (incl. taps), precision, halos, the stream and the workspaces.
std::string graph_key(const fb_ctx* ctx, const fb_image* ins, const fb_image* outs, int count, int halo_top,
                      int halo_bottom, const Job& j, int precision, const Geom& geo) {
  std::string k;
  auto put = [&](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
  for (int i = 0; i < count; ++i) {
    put(ins + i, sizeof(fb_image));
    if (outs) put(outs + i, sizeof(fb_image));
  }
  const int ints[] = {count, halo_top, halo_bottom, precision, j.kind, j.W, j.N, j.mode, j.check, ctx->tab_n};
  put(ints, sizeof(ints));
  const double dbl[] = {j.sr, j.tc, j.lo, j.hi};
  put(dbl, sizeof(dbl));
  if (j.taps) put(j.taps, sizeof(double) * (2 * j.W + 1));
  const void* ptrs[] = {ctx->stream,       ctx->ws,           ctx->ws2,         ctx->flags,
                        ctx->flags_host,   ctx->tab,          ctx->tabd,        ctx->in_stage[0],
                        ctx->in_stage[1],  ctx->out_stage[0], ctx->out_stage[1]};
  put(ptrs, sizeof(ptrs));
  const long long sizes[] = {ctx->ws_limit, ctx->flags_cap, ctx->tab_cap, geo.row_origin, geo.image_rows};
  put(sizes, sizeof(sizes));
  for (const fb_image* h : {geo.above, geo.below}) {
    const fb_image none{};
    put(h ? h : &none, sizeof(fb_image));
  }
  return k;
}

int execute(fb_ctx* ctx, const fb_image* ins, fb_image* outs, int count, int halo_top, int halo_bottom,
            const Job& j, int precision, fb_stats* st, const Geom& geo = Geom()) {
  FB_CUDA(cudaSetDevice(ctx->device));
  fb_stats local;
  memset(&local, 0, sizeof(local));
  local.bad_image = -1;
  int rc = ensure_flags(ctx, count);
  if (rc != FB_OK) return rc;
  if (ctx->realloc_seen) {  // a graph may reference a freed buffer
    ctx->clear_graphs();
    ctx->realloc_seen = false;
  }
  ctx->kev_used = 0;
  ctx->pev_used = 0;
  ctx->widen_used = false;
  const long long t_call0 = hostwiden::Pool::now_ns();
  // Whatever path leaves this function, the host threads are done with the caller's output first.
  struct WidenDrain {
    fb_ctx* c;
    ~WidenDrain() {
      if (c->widen_used) c->widen->wait_all();
    }
  } widen_drain{ctx};
  if ((rc = order_after_caller(ctx)) != FB_OK) return rc;
  FB_CUDA(cudaEventRecord(ctx->ev_start, ctx->stream));
  std::vector<Item> items(count);
  long long pixels = 0;
  for (int i = 0; i < count; ++i) {
    Item& it = items[i];
    it = Item{};
    it.in = ins + i;
    it.out = outs ? outs + i : nullptr;
    it.rows_out = (int)(geo.separate() ? ins[i].rows : ins[i].rows - halo_top - halo_bottom);
    pixels += (long long)it.rows_out * ins[i].cols;
    // host images of more than 4 MP are pipelined in row chunks of ~FB_CHUNK_PX pixels (at least
    // 8 chunks, at most 64, >= 256 rows each): the un-overlapped first H2D and last D2H shrink
    // with the chunk, while per-chunk launches and events stay negligible
    const bool host_io = !ins[i].on_device || (it.out && !it.out->on_device);
    const long long px = (long long)it.rows_out * ins[i].cols;
    long long nch = std::min<long long>(64, std::max<long long>(FB_CHUNK_MIN, px / FB_CHUNK_PX));
    nch = std::max<long long>(1, std::min<long long>(nch, it.rows_out / 256));
    // (batches overlap image i+1's copies with image i's kernels instead: no chunks)
    it.chunks = (count == 1 && host_io && px >= (4ll << 20) && it.rows_out >= 512) ? (int)nch : 1;
    it.crows = it.rows_out;
    std::vector<long long> sizes;  // rows of the chunks, in order
    if (it.chunks > 1) {
      it.crows = (it.rows_out + it.chunks - 1) / it.chunks;
      it.crows = (it.crows + 255) / 256 * 256;  // chunks start at multiples of 256 rows (walk_rows)
      // The fp32 box walker runs one CTA per 128 columns and walk, two per SM: a 512-row c4 chunk is
      // 258 CTAs for 296 slots, and kernel 1 took 0.48 ms per 512 rows against 0.37 ms inside a
      // 4096-row band.  Its chunks are sized in walks so that the grid fills whole waves (c4: 9
      // walks = 2304 rows = 3.92 waves), ramping up from short chunks that start the pipeline
      // (each sized so its copy lands while the chunks before it are filtered) and down to short
      // ones at the end (the last chunk's copy-out and widening are not overlapped by kernels).
      const long long cols = ins[i].cols, wpad = cols + 2 * j.W;
      const long long image_rows = geo.image_rows > 0 ? geo.image_rows : it.rows_out;
      if (precision != FB_PREC_F64 && j.kind == FB_BOX && j.W <= kFastMaxW && j.N + 1 <= kWalkMaxCh &&
          wpad * image_rows >= (4ll << 20)) {
        const long long walk = walk_rows((int)wpad, (int)image_rows, 128);
        const long long gx = (wpad + 127) / 128, slots = 2ll * ctx->sm_count;
        const long long w_lo = std::max<long long>(1, (FB_CHUNK_PX + cols * walk - 1) / (cols * walk));
        const long long w_hi = std::max<long long>(w_lo, (5 * FB_CHUNK_PX) / (cols * walk));
        long long best = w_lo;
        double best_eff = 0.0;
        for (long long w = w_lo; w <= w_hi; ++w) {
          const double waves = (double)(gx * w) / (double)slots;
          const double eff = waves / std::ceil(waves);
          if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = w;
          }
        }
        long long rem = it.rows_out;
        auto take = [&](long long rows) {
          rows = std::min(rows, rem);
          if (rows > 0) {
            sizes.push_back(rows);
            rem -= rows;
          }
        };
        long long down_sum = 0;
        for (long long d : {2 * w_lo, w_lo})
          if (d < best) down_sum += d * walk;
        for (long long u : {w_lo, 2 * w_lo, 3 * w_lo})
          if (u < best && rem > down_sum + (u + best) * walk) take(u * walk);
        if (rem > down_sum) {  // the middle: chunks of ~best walks, the walks spread evenly over them
          const long long mid = (rem - down_sum + walk - 1) / walk;
          const long long n_main = std::max<long long>(1, (mid + best / 2) / best);
          for (long long k = 0; k < n_main; ++k) take(((mid * (k + 1)) / n_main - (mid * k) / n_main) * walk);
        }
        for (long long d : {2 * w_lo, w_lo})
          if (d < best) take(d * walk);
        take(rem);
      } else {
        for (long long r = 0; r < it.rows_out; r += it.crows) sizes.push_back(std::min<long long>(it.crows, it.rows_out - r));
      }
    } else {
      sizes.push_back(it.rows_out);
    }
    long long end = 0;
    it.crows = 0;
    for (long long sz : sizes) {
      end += sz;
      it.ends.push_back((int)end);
      it.crows = std::max(it.crows, (int)sz);
    }
  }
  bool any_widen = false;
  size_t widen_bytes = 0;
  for (auto& it : items) {
    any_widen |= it.widen = widen_applies(ctx, it.in, it.out, precision, pixels);
    if (it.widen) widen_bytes += (size_t)it.rows_out * it.in->cols * sizeof(float);
  }
  if (any_widen) {
    // the pinned staging holds the call's whole float32 output; without it (over the limit, or the
    // host refuses to pin that much) the call sends float64 rows instead
    bool ok = widen_bytes <= hostwiden::max_stage_bytes();
    if (ok) {
      if (!ctx->widen) ctx->widen = new hostwiden::Pool(ctx->widen_threads, ctx->device);
      if (ctx->widen->reserve(widen_bytes) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
      }
    }
    if (!ok) {
      any_widen = false;
      for (auto& it : items) it.widen = false;
    }
  }
  const long long launches0 = g_launches.load();
  unsigned long long* fl_all = ctx->flags_host + 4 * ctx->flags_cap;
  // The GPU work of one call: kernels (+ copies for host images) and the flag readback.
  auto enqueue = [&]() -> int {
    FB_CUDA(cudaMemcpyAsync(ctx->flags, ctx->flags_host, 4 * sizeof(unsigned long long) * count,
                            cudaMemcpyHostToDevice, ctx->stream));
    int r = precision == FB_PREC_F64 ? run_items<double>(ctx, items, halo_top, halo_bottom, j, &local, geo)
                                     : run_items<float>(ctx, items, halo_top, halo_bottom, j, &local, geo);
    if (r != FB_OK) return r;
    FB_CUDA(cudaMemcpyAsync(fl_all, ctx->flags, 4 * sizeof(unsigned long long) * count, cudaMemcpyDeviceToHost,
                            ctx->stream));
    return FB_OK;
  };
  // Small calls repeat with identical pointers and parameters (a serving loop, the c0/c1
  // configs) and are launch-bound: replay them as one CUDA graph instead of ~10-20 separate
  // launches, copies and records.  Large calls stay eager (launch cost is noise there
  // and their per-kernel times feed the roofline reports).
  // Graph replay needs every buffer to stay valid and addressable by copy engines between calls:
  // device memory, or page-locked host memory (a capture of a copy from pageable memory would
  // bake in a staging step that the runtime does eagerly).  The constant tables must already
  // hold this order (no upload inside a capture).
  auto replayable = [](const fb_image* im) {
    if (im->on_device) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, im->data) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  bool replay_ok = ctx->use_graphs && pixels <= kGraphMaxPixels && (outs == nullptr || ctx->tab_n == j.N);
  for (auto& it : items) replay_ok = replay_ok && replayable(it.in) && (!it.out || replayable(it.out));
  replay_ok = replay_ok && !any_widen;  // (host functions and ring slots stay out of graphs)
  fb_ctx::Graph* g = nullptr;
  if (replay_ok) {
    std::string key = graph_key(ctx, ins, outs, count, halo_top, halo_bottom, j, precision, geo);
    auto f = ctx->graphs.find(key);
    if (f == ctx->graphs.end()) {
      if (ctx->graphs.size() >= 16) ctx->clear_graphs();
      ctx->graphs.emplace(key, fb_ctx::Graph{});  // first sighting: run eagerly below
    } else {
      g = &f->second;
    }
  }
  if (!g) FB_CUDA(cudaEventRecord(ctx->ev_kstart, ctx->stream));  // graph calls: kernel_ms = device_ms
  if (g && g->exec) {
    FB_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
    g_launches += g->launches;
    ctx->kev_used = 0;  // no per-kernel events inside graphs (record_timing)
    local.bands = g->bands;
    local.h2d_bytes = g->h2d;
    local.d2h_bytes = g->d2h;
  } else if (g) {
    // second sighting: capture the same work, instantiate, launch
    FB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue();
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
    if (rc != FB_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess) return fail(FB_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
      g->exec = nullptr;
      return fail(FB_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
    }
    g->launches = g_launches.load() - launches0;
    g->bands = local.bands;
    g->h2d = local.h2d_bytes;
    g->d2h = local.d2h_bytes;
    ctx->kev_used = 0;
    FB_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
  } else {
    rc = enqueue();
    if (rc != FB_OK) return rc;
  }
  if (!g) FB_CUDA(cudaEventRecord(ctx->ev_kend, ctx->stream));
  FB_CUDA(cudaEventRecord(ctx->ev_end, ctx->stream));
  const bool replayed = g != nullptr;
  const cudaError_t sync_err = cudaEventSynchronize(ctx->ev_end);
  if (ctx->widen_used) ctx->widen->wait_all();  // the host threads are done with the caller's output
  FB_CUDA(sync_err);
  if (ctx->widen_used) {
    const long long t_sync = hostwiden::Pool::now_ns();
    static const bool trace = std::getenv("FBGPU_WIDEN_TRACE") != nullptr;
    if (trace) ctx->widen->trace_report(t_call0, t_sync, hostwiden::Pool::now_ns());
  }
  local.launches = g_launches.load() - launches0;
  local.precision = precision;

  int status = FB_OK;
  for (int i = 0; i < count && status == FB_OK; ++i) {
    unsigned long long fl[4];
    memcpy(fl, fl_all + 4 * i, sizeof(fl));
    const fb_image* in = ins + i;
    if (geo.separate()) {  // flagged indices count buffer rows from the virtual row 0 above `in`
      for (int k : {kFlagFirstNonfinite, kFlagFirstRange})
        if (fl[k] != ~0ull) fl[k] -= (unsigned long long)halo_top * in->cols;
    }
    // band calls report rows of the band itself
    const long long report_shift = (geo.separate() ? 0 : geo.report_rows) * in->cols;
    const size_t ies = dtype_size(in->dtype);
    local.degenerate_pixels += (long long)fl[kFlagDegenerate];
    local.nonfinite_outputs += (long long)fl[kFlagNonfiniteOut];
    auto sample_at = [&](unsigned long long idx) -> double {
      const long long r = (long long)(idx / (unsigned long long)in->cols), c = (long long)(idx % in->cols);
      const char* base = static_cast<const char*>(in->data) + ((size_t)r * in->ld + c) * ies;
      unsigned char buf[8];
      if (in->on_device) {
        if (cudaMemcpy(buf, base, ies, cudaMemcpyDeviceToHost) != cudaSuccess) return NAN;
      } else {
        memcpy(buf, base, ies);
      }
      if (in->dtype == FB_U8) return (double)buf[0];
      if (in->dtype == FB_F32) { float v; memcpy(&v, buf, 4); return (double)v; }
      double v; memcpy(&v, buf, 8); return v;
    };
    if (fl[kFlagFirstNonfinite] != ~0ull) {
      local.bad_index = (long long)fl[kFlagFirstNonfinite] - report_shift;
      local.bad_value = sample_at(fl[kFlagFirstNonfinite]);
      local.bad_image = i;
      status = fail(FB_ERR_NONFINITE_INPUT, "image contains non-finite samples");
    } else if (fl[kFlagFirstRange] != ~0ull) {
      local.bad_index = (long long)fl[kFlagFirstRange] - report_shift;
      local.bad_value = sample_at(fl[kFlagFirstRange]);
      local.bad_image = i;
      status = fail(FB_ERR_RANGE, "sample outside the declared range");
    } else if (outs && fl[kFlagNonfiniteOut] != 0) {
      local.bad_image = i;
      status = fail(FB_ERR_NUMERIC, "non-finite output");
    }
  }
  if (any_widen && status == FB_OK && local.degenerate_pixels > 0) {
    // A pixel under the Q floor returns the input sample itself (engine.py:68), which the centred
    // float32 transfer may not carry exactly: repeat the call with float64 rows over PCIe.
    const int saved = ctx->widen_threads;
    ctx->widen_threads = 0;
    const int rr = execute(ctx, ins, outs, count, halo_top, halo_bottom, j, precision, st, geo);
    ctx->widen_threads = saved;
    return rr;
  }
  float ms = 0.f, kms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev_start, ctx->ev_end);
  if (!replayed) cudaEventElapsedTime(&kms, ctx->ev_kstart, ctx->ev_kend);
  local.device_ms = ms;
  local.kernel_ms = replayed ? ms : kms;  // a replayed graph is timed as a whole
  static const bool trace_bands = std::getenv("FBGPU_TRACE_BANDS") != nullptr;
  for (int b = 0; b + 2 < ctx->kev_used; b += 3) {
    float t1 = 0.f, t2 = 0.f;
    cudaEventElapsedTime(&t1, ctx->kev[b], ctx->kev[b + 1]);
    cudaEventElapsedTime(&t2, ctx->kev[b + 1], ctx->kev[b + 2]);
    local.k1_ms += t1;
    local.k2_ms += t2;
    if (trace_bands) {  // where each band's kernels sit in the call (ms after the call's first event)
      float t0 = 0.f;
      cudaEventElapsedTime(&t0, ctx->ev_start, ctx->kev[b]);
      fprintf(stderr, "[band %d] k1 start +%.3f  k1 %.3f  k2 %.3f  end +%.3f\n", b / 3, t0, t1, t2, t0 + t1 + t2);
    }
  }
  if (replayed) local.k1_ms = local.k2_ms = -1.0;  // graph call: only kernel_ms (the total) exists
  local.spatial_filter_calls = j.N + 1;
  local.order = j.mode == kModeGpa ? j.N : 0;
  (void)pixels;
  if (st) *st = local;
  return status;
}


// ---------------------------------------------------------------------------- brute force
// Exact bilateral filter, O(W^2) per pixel, fp64, replicate boundary: the reference's
// bilateral_exact (reference.py:17-45), used to report the GPA approximation error at full size.
// CTA = 16x16 outputs; the (16+2W)^2 input tile (clamped rows/columns) is staged in shared memory.
constexpr int BF_T = 16;
constexpr int BF_MAX_TILED_W = 77;  // (16 + 2W)^2 doubles fit the 227 KB of shared memory

template <bool TILED>
__global__ void __launch_bounds__(BF_T * BF_T) k_bilateral_exact(const void* f, long long f_ld, int f_dtype,
                                                                 int rows, int cols, int W, const double* w1d,
                                                                 double inv_two_sr2, double* out, long long out_ld) {
  extern __shared__ double bf_tile[];
  const int S = BF_T + 2 * W;
  const int y0 = blockIdx.y * BF_T, x0 = blockIdx.x * BF_T;
  if (TILED) {
    for (int i = threadIdx.x; i < S * S; i += blockDim.x) {
      const int ty = i / S, tx = i - ty * S;
      const int gy = min(max(y0 + ty - W, 0), rows - 1), gx = min(max(x0 + tx - W, 0), cols - 1);
      bf_tile[i] = load_sample(f, f_dtype, (long long)gy * f_ld + gx);
    }
    __syncthreads();
  }
  const int ty = threadIdx.x / BF_T, tx = threadIdx.x % BF_T;
  const int y = y0 + ty, x = x0 + tx;
  if (y >= rows || x >= cols) return;
  const double fi = TILED ? bf_tile[(ty + W) * S + tx + W] : load_sample(f, f_dtype, (long long)y * f_ld + x);
  double num = 0.0, den = 0.0;
  for (int dy = 0; dy <= 2 * W; ++dy) {
    const double wy = w1d[dy];
    const double* rowp = bf_tile + (ty + dy) * S + tx;
    const long long grow_ = (long long)min(max(y + dy - W, 0), rows - 1) * f_ld;
    for (int dx = 0; dx <= 2 * W; ++dx) {
      const double nb = TILED ? rowp[dx] : load_sample(f, f_dtype, grow_ + min(max(x + dx - W, 0), cols - 1));
      const double d = nb - fi;
      const double wgt = wy * w1d[dx] * exp(-d * d * inv_two_sr2);
      num = fma(wgt, nb, num);
      den += wgt;
    }
  }
  out[(long long)y * out_ld + x] = num / den;
}

}  // namespace

extern "C" {

int fb_ipc_export(const void* dptr, uint8_t handle[64], int64_t* offset) {
  if (!dptr || !handle || !offset) return fail(FB_ERR_PARAM, "null argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  // the handle names the whole allocation: report where dptr sits inside it
  typedef CUresult (*range_fn_t)(CUdeviceptr*, size_t*, CUdeviceptr);
  static range_fn_t range_fn = nullptr;
  if (!range_fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(FB_ERR_CUDA, "cuMemGetAddressRange unavailable");
    range_fn = reinterpret_cast<range_fn_t>(p);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
    return fail(FB_ERR_PARAM, "pointer is not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(FB_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  memcpy(handle, &h, 64);
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dptr) - base);
  return FB_OK;
}

int fb_ipc_open(int32_t device, const uint8_t handle[64], void** base) {
  if (!handle || !base) return fail(FB_ERR_PARAM, "null argument");
  FB_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(FB_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  return FB_OK;
}

int fb_ipc_close(void* base) {
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return fail(FB_ERR_CUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
  return FB_OK;
}

#ifndef FB_BUILD_ID
#define FB_BUILD_ID "unknown"
#endif
// "FBGPU_BUILD_ID=<hash of the sources and flags>" stays in the binary's read-only data, so
// build() can read it from the file and load_library() from fb_build_id().
static const char kBuildId[] = "FBGPU_BUILD_ID=" FB_BUILD_ID;
const char* fb_build_id(void) { return kBuildId + 15; }
int fb_version(void) { return FBGPU_VERSION; }
int64_t fb_launch_count(void) { return (int64_t)g_launches.load(); }
const char* fb_last_error(void) { return g_last_error.c_str(); }

int fb_create(int device, fb_ctx** out) {
  if (!out) return fail(FB_ERR_PARAM, "fb_create: null out");
  *out = nullptr;
  int n = 0;
  FB_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(FB_ERR_PARAM, "fb_create: no such device " + std::to_string(device));
  FB_CUDA(cudaSetDevice(device));
  fb_ctx* c = new fb_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  bool ok = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&c->s_alt, cudaStreamNonBlocking) == cudaSuccess;
  for (cudaEvent_t* e : {&c->ev_start, &c->ev_kstart, &c->ev_kend, &c->ev_end})
    ok = ok && cudaEventCreate(e) == cudaSuccess;
  ok = ok && cudaEventCreateWithFlags(&c->ev_upstream, cudaEventDisableTiming) == cudaSuccess;
  c->stream = c->own_stream;
  if (!ok || ensure_flags(c, 64) != FB_OK) {
    fb_destroy(c);
    return fail(FB_ERR_CUDA, "fb_create: stream/event/flag allocation failed");
  }
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  c->ws_limit = std::min<long long>(16ll << 30, (long long)(free_b / 4));
  const char* wl = std::getenv("FBGPU_WORKSPACE_GB");  // override the plane-workspace limit (GiB)
  if (wl && *wl && atof(wl) > 0) c->ws_limit = (long long)(atof(wl) * (1ll << 30));
  const char* ng = std::getenv("FBGPU_NO_GRAPHS");  // debugging: always launch eagerly
  c->use_graphs = !(ng && *ng && *ng != '0');
  *out = c;
  return FB_OK;
}

int fb_destroy(fb_ctx* c) {
  if (!c) return FB_OK;
  cudaSetDevice(c->device);
  if (c->own_stream) cudaStreamSynchronize(c->own_stream);
  c->clear_graphs();
  delete c->widen;  // joins the host threads, frees the pinned staging area
  c->widen = nullptr;
  for (void* p : {c->ws, c->ws2, c->in_stage[0], c->in_stage[1], c->out_stage[0], c->out_stage[1], (void*)c->flags,
                  (void*)c->tab, (void*)c->tabd})
    if (p) cudaFree(p);
  if (c->scratch) cudaFree(c->scratch);
  for (void* p : {(void*)c->flags_host, (void*)c->tab_host, (void*)c->tabd_host, (void*)c->scratch_host})
    if (p) cudaFreeHost(p);
  for (cudaEvent_t e : {c->ev_start, c->ev_kstart, c->ev_kend, c->ev_end, c->ev_upstream})
    if (e) cudaEventDestroy(e);
  for (auto& e : c->kev) cudaEventDestroy(e);
  for (auto& e : c->pev) cudaEventDestroy(e);
  for (cudaStream_t s : {c->own_stream, c->s_h2d, c->s_d2h, c->s_alt})
    if (s) cudaStreamDestroy(s);
  delete c;
  return FB_OK;
}

int fb_set_stream(fb_ctx* c, void* s) {
  if (!c) return fail(FB_ERR_PARAM, "null context");
  const cudaStream_t cs = static_cast<cudaStream_t>(s);
  if (cs == cudaStreamLegacy || cs == cudaStreamPerThread) {
    // a default stream (torch's current stream is the legacy one, handle 0, bound as
    // cudaStreamLegacy by the Python layer): run on own_stream, ordered after it at every call
    c->stream = c->own_stream;
    c->upstream = cs;
  } else {
    c->stream = cs ? cs : c->own_stream;
    c->upstream = nullptr;
  }
  return FB_OK;
}

int fb_set_workspace_limit(fb_ctx* c, int64_t bytes) {
  if (!c || bytes <= 0) return fail(FB_ERR_PARAM, "fb_set_workspace_limit: bad arguments");
  c->ws_limit = bytes;
  return FB_OK;
}

static int check_filter_args(const fb_spatial* sp, int precision) {
  if (!sp) return fail(FB_ERR_PARAM, "null spatial kernel");
  if (sp->kind != FB_BOX && sp->kind != FB_GAUSSIAN) return fail(FB_ERR_PARAM, "unknown spatial kernel kind");
  if (sp->half_width < 1 || sp->half_width > kMaxW)
    return fail(FB_ERR_PARAM, "half_width must lie in [1, " + std::to_string(kMaxW) + "]");
  if (sp->kind == FB_GAUSSIAN && !sp->weights_1d) return fail(FB_ERR_PARAM, "gaussian kernel needs weights_1d");
  if (precision != FB_PREC_F32 && precision != FB_PREC_F64) return fail(FB_ERR_PARAM, "unknown precision");
  return FB_OK;
}

static int check_window(const fb_spatial* sp, long long rows, long long cols) {
  if (sp->kind != FB_BOX) return FB_OK;
  long long lim = 1;
  bool any = false;
  for (long long d : {rows, cols})
    if (d > 1) { lim = any ? std::min(lim, d) : d; any = true; }
  if (sp->half_width >= lim)
    return fail(FB_ERR_WINDOW, "window half-width " + std::to_string(sp->half_width) + " too large for " +
                                   std::to_string(rows) + "x" + std::to_string(cols) + " image");
  return FB_OK;
}

static int gpa_common(fb_ctx* ctx, const fb_image* ins, fb_image* outs, int count, int64_t halo_top,
                      int64_t halo_bottom, const fb_spatial* sp, double sigma_r, int32_t order, double center,
                      double half_range, int32_t precision, fb_stats* stats, const Geom& geo = Geom()) {
  if (!ctx) return fail(FB_ERR_PARAM, "null context");
  if (count < 1 || !ins || !outs) return fail(FB_ERR_PARAM, "need at least one image");
  int rc = check_filter_args(sp, precision);
  if (rc) return rc;
  if (!(sigma_r > 0) || !std::isfinite(sigma_r)) return fail(FB_ERR_PARAM, "sigma_r must be positive");
  if (order < 1) return fail(FB_ERR_PARAM, "order must be an integer >= 1");
  if (!(half_range > 0)) return fail(FB_ERR_PARAM, "half_range must be positive");
  for (int i = 0; i < count; ++i) {
    rc = check_image(ins + i, "input", true);
    if (rc) return rc;
    rc = check_image(outs + i, "output", true);  // u8: quantised raster (save_pgm, image.py:96-99)
    if (rc) return rc;
    if (!geo.separate() && (halo_top < 0 || halo_bottom < 0 || halo_top + halo_bottom >= ins[i].rows))
      return fail(FB_ERR_PARAM, "bad halo rows");
    if (ins[i].cols != ins[0].cols) return fail(FB_ERR_PARAM, "images of a batch must share their width");
    const long long rows_out = geo.separate() ? ins[i].rows : ins[i].rows - halo_top - halo_bottom;
    if (outs[i].rows != rows_out || outs[i].cols != ins[i].cols) return fail(FB_ERR_PARAM, "output shape mismatch");
    // the reference checks the window against the whole image (conv.py:19-27)
    rc = check_window(sp, geo.image_rows > 0 ? geo.image_rows : rows_out, ins[i].cols);
    if (rc) return rc;
  }
  Job j;
  memset(&j, 0, sizeof(j));
  j.kind = sp->kind;
  j.W = sp->half_width;
  j.N = order;
  j.mode = kModeGpa;
  j.check = 1;
  j.taps = sp->weights_1d;
  j.sr = sigma_r;
  j.tc = center;
  j.lo = center - half_range;
  j.hi = center + half_range;
  return execute(ctx, ins, outs, count, (int)halo_top, (int)halo_bottom, j, precision, stats, geo);
}

int fb_gpa_filter(fb_ctx* ctx, const fb_image* in, int64_t halo_top, int64_t halo_bottom, fb_image* out,
                  const fb_spatial* sp, double sigma_r, int32_t order, double center, double half_range,
                  int32_t precision, fb_stats* stats) {
  return gpa_common(ctx, in, out, 1, halo_top, halo_bottom, sp, sigma_r, order, center, half_range, precision,
                    stats);
}

int fb_gpa_filter_band(fb_ctx* ctx, const fb_image* in, const fb_image* above, const fb_image* below,
                       int64_t row_origin, int64_t image_rows, fb_image* out, const fb_spatial* sp, double sigma_r,
                       int32_t order, double center, double half_range, int32_t precision, fb_stats* stats) {
  if (!ctx) return fail(FB_ERR_PARAM, "null context");
  int rc = check_image(in, "input", true);
  if (rc) return rc;
  if (row_origin < 0 || image_rows < row_origin + in->rows || image_rows > (1ll << 30))
    return fail(FB_ERR_PARAM, "band rows outside the image");
  const long long above_rows = above ? above->rows : 0, below_rows = below ? below->rows : 0;
  if (above_rows > row_origin || below_rows > image_rows - row_origin - in->rows)
    return fail(FB_ERR_PARAM, "halo rows outside the image");
  const size_t es = dtype_size(in->dtype);
  bool contiguous = true;  // halos that are simply the rows next to `in` in the same buffer
  for (const fb_image* h : {above, below}) {
    if (!h) continue;
    rc = check_image(h, "halo", true);
    if (rc) return rc;
    if (h->cols != in->cols || h->dtype != in->dtype) return fail(FB_ERR_PARAM, "halo rows must match the band");
    const char* want = h == above ? static_cast<const char*>(in->data) - (size_t)h->rows * h->ld * es
                                  : static_cast<const char*>(in->data) + (size_t)in->rows * in->ld * es;
    contiguous = contiguous && h->ld == in->ld && h->on_device == in->on_device && h->data == want;
  }
  Geom geo;
  geo.row_origin = row_origin;
  geo.image_rows = image_rows;
  if (contiguous) {
    // one buffer [above | in | below]: the fb_gpa_filter path (host buffers pipelined in chunks)
    fb_image whole = *in;
    whole.data = above ? above->data : in->data;
    whole.rows = above_rows + in->rows + below_rows;
    geo.report_rows = above_rows;
    return gpa_common(ctx, &whole, out, 1, above_rows, below_rows, sp, sigma_r, order, center, half_range,
                      precision, stats, geo);
  }
  for (const fb_image* h : {above, below})
    if (h && (!h->on_device || !in->on_device))
      return fail(FB_ERR_PARAM, "halo rows in separate buffers need device-resident input and halos");
  geo.above = above;
  geo.below = below;
  return gpa_common(ctx, in, out, 1, above_rows, below_rows, sp, sigma_r, order, center, half_range, precision,
                    stats, geo);
}

int fb_gpa_filter_batch(fb_ctx* ctx, const fb_image* ins, fb_image* outs, int32_t count, const fb_spatial* sp,
                        double sigma_r, int32_t order, double center, double half_range, int32_t precision,
                        fb_stats* stats) {
  return gpa_common(ctx, ins, outs, count, 0, 0, sp, sigma_r, order, center, half_range, precision, stats);
}

int fb_spatial_filter(fb_ctx* ctx, const fb_image* in, fb_image* out, const fb_spatial* sp, int32_t precision,
                      fb_stats* stats) {
  if (!ctx) return fail(FB_ERR_PARAM, "null context");
  int rc = check_image(in, "input", true);
  if (rc) return rc;
  rc = check_image(out, "output", false);
  if (rc) return rc;
  rc = check_filter_args(sp, precision);
  if (rc) return rc;
  if (out->rows != in->rows || out->cols != in->cols) return fail(FB_ERR_PARAM, "output shape mismatch");
  Job j;
  memset(&j, 0, sizeof(j));
  j.kind = sp->kind;
  j.W = sp->half_width;
  j.N = 0;
  j.mode = kModePlain;
  j.check = 1;
  j.taps = sp->weights_1d;
  j.sr = 1.0;
  j.tc = 0.0;
  j.lo = -INFINITY;
  j.hi = INFINITY;
  return execute(ctx, in, out, 1, 0, 0, j, precision, stats);
}

int fb_validate(fb_ctx* ctx, const fb_image* in, double lo, double hi, fb_stats* stats) {
  if (!ctx) return fail(FB_ERR_PARAM, "null context");
  int rc = check_image(in, "input", true);
  if (rc) return rc;
  Job j;
  memset(&j, 0, sizeof(j));
  j.lo = lo;
  j.hi = hi;
  return execute(ctx, in, nullptr, 1, 0, 0, j, FB_PREC_F64, stats);
}

int fb_bilateral_exact(fb_ctx* ctx, const fb_image* in, fb_image* out, const fb_spatial* sp, double sigma_r,
                       fb_stats* stats) {
  if (!ctx) return fail(FB_ERR_PARAM, "null context");
  int rc = check_image(in, "input", true);
  if (rc) return rc;
  rc = check_image(out, "output", false);
  if (rc) return rc;
  if (!sp || (sp->kind != FB_BOX && sp->kind != FB_GAUSSIAN) || sp->half_width < 1 || sp->half_width > kMaxW ||
      (sp->kind == FB_GAUSSIAN && !sp->weights_1d))
    return fail(FB_ERR_PARAM, "bad spatial kernel");
  if (out->dtype != FB_F64 || out->rows != in->rows || out->cols != in->cols)
    return fail(FB_ERR_PARAM, "output must be float64 of the input's shape");
  if (!(sigma_r > 0)) return fail(FB_ERR_PARAM, "sigma_r must be positive");
  if (sp->half_width >= std::min(in->rows, in->cols))
    return fail(FB_ERR_WINDOW, "window half-width " + std::to_string(sp->half_width) + " too large for " +
                                   std::to_string(in->rows) + "x" + std::to_string(in->cols) + " image");
  FB_CUDA(cudaSetDevice(ctx->device));
  if (int orc = order_after_caller(ctx)) return orc;
  const int W = sp->half_width, n = 2 * W + 1;
  std::vector<double> w(n);
  for (int k = 0; k < n; ++k) w[k] = sp->kind == FB_BOX ? 1.0 / n : sp->weights_1d[k];
  const size_t ies = dtype_size(in->dtype);
  fb_stats local;
  memset(&local, 0, sizeof(local));
  local.bad_image = -1;
  void* din = in->data;
  long long dld = in->ld;
  void* dout = out->data;
  long long old = out->ld;
  double* dw = nullptr;
  FB_CUDA(cudaEventRecord(ctx->ev_start, ctx->stream));
  FB_CUDA(cudaMallocAsync(&dw, n * sizeof(double), ctx->stream));
  FB_CUDA(cudaMemcpyAsync(dw, w.data(), n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  if (!in->on_device) {
    rc = grow(ctx, &ctx->in_stage[0], &ctx->in_stage_bytes[0], (size_t)in->rows * in->cols * ies);
    if (rc) return rc;
    FB_CUDA(cudaMemcpy2DAsync(ctx->in_stage[0], in->cols * ies, in->data, in->ld * ies, in->cols * ies, in->rows,
                              cudaMemcpyHostToDevice, ctx->stream));
    din = ctx->in_stage[0];
    dld = in->cols;
  }
  if (!out->on_device) {
    rc = grow(ctx, &ctx->out_stage[0], &ctx->out_stage_bytes[0], (size_t)out->rows * out->cols * 8);
    if (rc) return rc;
    dout = ctx->out_stage[0];
    old = out->cols;
  }
  const bool tiled = W <= BF_MAX_TILED_W;
  const size_t smem = tiled ? (size_t)(BF_T + 2 * W) * (BF_T + 2 * W) * sizeof(double) : 0;
  if (tiled)
    FB_CUDA(cudaFuncSetAttribute(k_bilateral_exact<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)((in->cols + BF_T - 1) / BF_T), (unsigned)((in->rows + BF_T - 1) / BF_T));
  FB_CUDA(record_timing(ctx->ev_kstart, ctx->stream));
  (tiled ? k_bilateral_exact<true> : k_bilateral_exact<false>)<<<grid, BF_T * BF_T, smem, ctx->stream>>>(
      din, dld, in->dtype, (int)in->rows, (int)in->cols, W, dw, 1.0 / (2.0 * sigma_r * sigma_r),
      static_cast<double*>(dout), old);
  FB_CUDA(cudaGetLastError());
  g_launches += 1;
  FB_CUDA(record_timing(ctx->ev_kend, ctx->stream));
  if (!out->on_device)
    FB_CUDA(cudaMemcpy2DAsync(out->data, out->ld * 8, dout, old * 8, out->cols * 8, out->rows,
                              cudaMemcpyDeviceToHost, ctx->stream));
  FB_CUDA(cudaFreeAsync(dw, ctx->stream));
  FB_CUDA(cudaEventRecord(ctx->ev_end, ctx->stream));
  FB_CUDA(cudaEventSynchronize(ctx->ev_end));
  float ms = 0.f, kms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev_start, ctx->ev_end);
  cudaEventElapsedTime(&kms, ctx->ev_kstart, ctx->ev_kend);
  local.device_ms = ms;
  local.kernel_ms = kms;
  local.launches = 1;
  local.precision = FB_PREC_F64;
  if (stats) *stats = local;
  return FB_OK;
}

// ---------------------------------------------------------------------------- metrology / oracle
static int ensure_scratch(fb_ctx* c, size_t doubles) {
  if (doubles <= c->scratch_cap) return FB_OK;
  if (c->scratch) cudaFree(c->scratch);
  if (c->scratch_host) cudaFreeHost(c->scratch_host);
  c->scratch = nullptr;
  c->scratch_host = nullptr;
  c->scratch_cap = 0;
  FB_CUDA(cudaMalloc(&c->scratch, doubles * sizeof(double)));
  FB_CUDA(cudaMallocHost(&c->scratch_host, doubles * sizeof(double)));
  c->scratch_cap = doubles;
  return FB_OK;
}

// Device copy of a host image into staging slot `slot` (or the image itself when on the device).
static int stage_input(fb_ctx* c, const fb_image* im, int slot, const void** d, long long* ld) {
  if (im->on_device) {
    *d = im->data;
    *ld = im->ld;
    return FB_OK;
  }
  const size_t es = dtype_size(im->dtype);
  int rc = grow(c, &c->in_stage[slot], &c->in_stage_bytes[slot], (size_t)im->rows * im->cols * es);
  if (rc) return rc;
  FB_CUDA(cudaMemcpy2DAsync(c->in_stage[slot], im->cols * es, im->data, im->ld * es, im->cols * es, im->rows,
                            cudaMemcpyHostToDevice, c->stream));
  *d = c->in_stage[slot];
  *ld = im->cols;
  return FB_OK;
}

int fb_kernel_error_sup(fb_ctx* ctx, int32_t order, double sigma_r, double half_range, double* sup) {
  if (!ctx || !sup) return fail(FB_ERR_PARAM, "null argument");
  if (order < 1) return fail(FB_ERR_PARAM, "N must be >= 1, got " + std::to_string(order));
  if (!(sigma_r > 0 && half_range > 0)) return fail(FB_ERR_PARAM, "sigma_r and T must be positive");
  if (!(half_range < 1e6)) return fail(FB_ERR_PARAM, "T too large for the grid search");
  FB_CUDA(cudaSetDevice(ctx->device));
  if (int orc = order_after_caller(ctx)) return orc;
  int rc = ensure_scratch(ctx, 64);
  if (rc) return rc;
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(ctx->scratch);
  FB_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long), ctx->stream));
  if (launch_kernel_error_sup(ctx->stream, ctx->sm_count, (int)std::floor(half_range), order, sigma_r, bits))
    return fail(FB_ERR_CUDA, "kernel_error_sup launch failed");
  g_launches += 1;
  FB_CUDA(cudaMemcpyAsync(ctx->scratch_host, bits, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FB_CUDA(cudaStreamSynchronize(ctx->stream));
  *sup = ctx->scratch_host[0];
  return FB_OK;
}

int fb_error_stats(fb_ctx* ctx, const fb_image* a, const fb_image* b, double* linf, double* sum_sq,
                   fb_stats* stats) {
  if (!ctx || !linf || !sum_sq) return fail(FB_ERR_PARAM, "null argument");
  int rc = check_image(a, "a", true);
  if (rc) return rc;
  rc = check_image(b, "b", true);
  if (rc) return rc;
  if (a->rows != b->rows || a->cols != b->cols)
    return fail(FB_ERR_PARAM, "image dimensions differ: (" + std::to_string(a->rows) + ", " +
                                  std::to_string(a->cols) + ") vs (" + std::to_string(b->rows) + ", " +
                                  std::to_string(b->cols) + ")");
  FB_CUDA(cudaSetDevice(ctx->device));
  if (int orc = order_after_caller(ctx)) return orc;
  const int nb = error_stats_blocks(ctx->sm_count);
  rc = ensure_scratch(ctx, 2 * (size_t)nb + 4);
  if (rc) return rc;
  rc = ensure_flags(ctx, 2);
  if (rc) return rc;
  fb_stats local;
  memset(&local, 0, sizeof(local));
  local.bad_image = -1;
  FB_CUDA(cudaEventRecord(ctx->ev_start, ctx->stream));
  FB_CUDA(cudaMemcpyAsync(ctx->flags, ctx->flags_host, 8 * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                          ctx->stream));
  const void *da = nullptr, *db = nullptr;
  long long lda = 0, ldb = 0;
  if ((rc = stage_input(ctx, a, 0, &da, &lda)) || (rc = stage_input(ctx, b, 1, &db, &ldb))) return rc;
  local.h2d_bytes = (a->on_device ? 0 : a->rows * a->cols * (long long)dtype_size(a->dtype)) +
                    (b->on_device ? 0 : b->rows * b->cols * (long long)dtype_size(b->dtype));
  FB_CUDA(record_timing(ctx->ev_kstart, ctx->stream));
  if (launch_error_stats(ctx->stream, ctx->sm_count, da, lda, a->dtype, db, ldb, b->dtype, (int)a->rows,
                         (int)a->cols, ctx->scratch, ctx->flags + kFlagFirstNonfinite,
                         ctx->flags + 4 + kFlagFirstNonfinite))
    return fail(FB_ERR_CUDA, "error_stats launch failed");
  g_launches += 1;
  FB_CUDA(record_timing(ctx->ev_kend, ctx->stream));
  unsigned long long* fl = ctx->flags_host + 4 * ctx->flags_cap;
  FB_CUDA(cudaMemcpyAsync(ctx->scratch_host, ctx->scratch, 2 * (size_t)nb * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  FB_CUDA(cudaMemcpyAsync(fl, ctx->flags, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  FB_CUDA(cudaEventRecord(ctx->ev_end, ctx->stream));
  FB_CUDA(cudaEventSynchronize(ctx->ev_end));
  double mx = 0.0, ss = 0.0;
  for (int i = 0; i < nb; ++i) {
    mx = std::max(mx, ctx->scratch_host[2 * i]);
    ss += ctx->scratch_host[2 * i + 1];
  }
  *linf = mx;
  *sum_sq = ss;
  float ms = 0.f, kms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev_start, ctx->ev_end);
  cudaEventElapsedTime(&kms, ctx->ev_kstart, ctx->ev_kend);
  local.device_ms = ms;
  local.kernel_ms = kms;
  local.launches = 1;
  local.precision = FB_PREC_F64;
  int status = FB_OK;
  for (int i = 0; i < 2 && status == FB_OK; ++i) {
    const unsigned long long idx = fl[4 * i + kFlagFirstNonfinite];
    if (idx == ~0ull) continue;
    local.bad_image = i;
    local.bad_index = (long long)idx;
    status = fail(FB_ERR_NONFINITE_INPUT, "image contains non-finite samples");
  }
  if (stats) *stats = local;
  return status;
}

int fb_convolve_direct(fb_ctx* ctx, const fb_image* in, fb_image* out, int32_t half_width, const double* weights_2d,
                       fb_stats* stats) {
  if (!ctx || !weights_2d) return fail(FB_ERR_PARAM, "null argument");
  int rc = check_image(in, "input", true);
  if (rc) return rc;
  rc = check_image(out, "output", false);
  if (rc) return rc;
  if (out->dtype != FB_F64 || out->rows != in->rows || out->cols != in->cols)
    return fail(FB_ERR_PARAM, "output must be float64 of the input's shape");
  if (half_width < 1 || half_width > kMaxW)
    return fail(FB_ERR_PARAM, "half_width must lie in [1, " + std::to_string(kMaxW) + "]");
  fb_spatial sp{FB_BOX, half_width, nullptr};  // _check_window applies to every kind here (conv.py:86)
  rc = check_window(&sp, in->rows, in->cols);
  if (rc) return rc;
  FB_CUDA(cudaSetDevice(ctx->device));
  if (int orc = order_after_caller(ctx)) return orc;
  const int n = 2 * half_width + 1;
  rc = ensure_flags(ctx, 1);
  if (rc) return rc;
  fb_stats local;
  memset(&local, 0, sizeof(local));
  local.bad_image = -1;
  FB_CUDA(cudaEventRecord(ctx->ev_start, ctx->stream));
  // as_image's finiteness check first (conv.py:85), on the staged input
  FB_CUDA(cudaMemcpyAsync(ctx->flags, ctx->flags_host, 4 * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                          ctx->stream));
  const void* din = nullptr;
  long long dld = 0;
  if ((rc = stage_input(ctx, in, 0, &din, &dld))) return rc;
  if (launch_validate(ctx->stream, din, dld, in->dtype, (int)in->rows, (int)in->cols, -INFINITY, INFINITY,
                      ctx->flags, ctx->sm_count))
    return fail(FB_ERR_CUDA, "validation kernel launch failed");
  double* dw = nullptr;
  FB_CUDA(cudaMallocAsync(&dw, (size_t)n * n * sizeof(double), ctx->stream));
  FB_CUDA(cudaMemcpyAsync(dw, weights_2d, (size_t)n * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  void* dout = out->data;
  long long old = out->ld;
  if (!out->on_device) {
    rc = grow(ctx, &ctx->out_stage[0], &ctx->out_stage_bytes[0], (size_t)out->rows * out->cols * 8);
    if (rc) return rc;
    dout = ctx->out_stage[0];
    old = out->cols;
  }
  FB_CUDA(record_timing(ctx->ev_kstart, ctx->stream));
  if (launch_convolve_direct(ctx->stream, din, dld, in->dtype, (int)in->rows, (int)in->cols, half_width, dw,
                             static_cast<double*>(dout), old))
    return fail(FB_ERR_CUDA, "convolve_direct launch failed");
  g_launches += 2;
  FB_CUDA(record_timing(ctx->ev_kend, ctx->stream));
  if (!out->on_device)
    FB_CUDA(cudaMemcpy2DAsync(out->data, out->ld * 8, dout, old * 8, out->cols * 8, out->rows,
                              cudaMemcpyDeviceToHost, ctx->stream));
  unsigned long long* fl = ctx->flags_host + 4 * ctx->flags_cap;
  FB_CUDA(cudaMemcpyAsync(fl, ctx->flags, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
  FB_CUDA(cudaFreeAsync(dw, ctx->stream));
  FB_CUDA(cudaEventRecord(ctx->ev_end, ctx->stream));
  FB_CUDA(cudaEventSynchronize(ctx->ev_end));
  float ms = 0.f, kms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev_start, ctx->ev_end);
  cudaEventElapsedTime(&kms, ctx->ev_kstart, ctx->ev_kend);
  local.device_ms = ms;
  local.kernel_ms = kms;
  local.launches = 2;
  local.precision = FB_PREC_F64;
  int status = FB_OK;
  if (fl[kFlagFirstNonfinite] != ~0ull) {
    local.bad_index = (long long)fl[kFlagFirstNonfinite];
    local.bad_image = 0;
    status = fail(FB_ERR_NONFINITE_INPUT, "image contains non-finite samples");
  }
  if (stats) *stats = local;
  return status;
}

}  // extern "C"
