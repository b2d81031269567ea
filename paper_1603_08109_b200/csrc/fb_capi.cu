// fb_capi.cu — the C ABI (include/fbgpu.h): context, workspace, row-band
// scheduling, kernel dispatch and error reporting.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fbgpu.h"
#include "fb_common.cuh"
#include "fb_generic.cuh"
#include "fb_fast.cuh"

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
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* in_stage = nullptr;
  size_t in_stage_bytes = 0;
  void* out_stage = nullptr;
  size_t out_stage_bytes = 0;
  unsigned long long* flags = nullptr;       // device, 4 slots
  float* tab = nullptr;                      // device channel-constant table (fp32 fast path)
  float* tab_host = nullptr;                 // pinned staging for it
  int tab_cap = 0;                           // channels it holds
  unsigned long long* flags_host = nullptr;  // pinned, 8 slots (0-3 init pattern, 4-7 readback)
  long long ws_limit = 0;
  int sm_count = 148;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // Per-band kernel boundaries: [k1 start, k1 end = k2 start, k2 end] x bands.
  std::vector<cudaEvent_t> kev;
  int kev_used = 0;

  cudaEvent_t next_event() {
    if (kev_used == (int)kev.size()) {
      cudaEvent_t e = nullptr;
      cudaEventCreate(&e);
      kev.push_back(e);
    }
    return kev[kev_used++];
  }
};

namespace {

int grow(void** p, size_t* have, size_t need) {
  if (*have >= need) return FB_OK;
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

// Everything one filter call needs, independent of precision.
struct Job {
  const void* f;       // device input
  long long f_ld;
  int f_dtype;
  int rows_in, cols, halo_top, rows_out;
  void* out;           // device output
  long long out_ld;
  int out_dtype;
  int kind, W, N, mode, check;
  const double* taps;
  double sr, tc, lo, hi;
};

template <typename T>
int launch_band(fb_ctx* ctx, const Job& j, GpaArgs<T>& a, int band_row0, int band_rows) {
  a.band_row0 = band_row0;
  a.band_rows = band_rows;
  const int W = j.W;
  bool done = false;
  cudaEvent_t e0 = ctx->next_event(), e1 = ctx->next_event(), e2 = ctx->next_event();
  KernelEvents kev{e0, e1, e2};
  int rc = launch_fast<T>(ctx->stream, j.kind, W, a, kev, &done);
  if (rc != FB_OK) return fail(FB_ERR_CUDA, std::string("fast kernel launch failed: ") +
                                               cudaGetErrorString(cudaGetLastError()));
  if (done) g_launches += 2;
  if (!done) {
    const size_t s1 = generic::k1_smem<T>(W), s2 = generic::k2_smem<T>(W);
    dim3 g1((a.wpad + generic::K1_TC - 1) / generic::K1_TC, (band_rows + generic::K1_RB - 1) / generic::K1_RB);
    dim3 g2((j.cols + generic::K2_TW - 1) / generic::K2_TW, (band_rows + generic::K2_TH - 1) / generic::K2_TH);
    auto k1 = j.kind == FB_BOX ? generic::k1_gen_vpass<T, kKindBox> : generic::k1_gen_vpass<T, kKindGauss>;
    auto k2 = j.kind == FB_BOX ? generic::k2_hpass_horner<T, kKindBox> : generic::k2_hpass_horner<T, kKindGauss>;
    FB_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1));
    FB_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2));
    FB_CUDA(cudaEventRecord(e0, ctx->stream));
    k1<<<g1, generic::K1_TC * generic::K1_RG, s1, ctx->stream>>>(a);
    FB_CUDA(cudaGetLastError());
    FB_CUDA(cudaEventRecord(e1, ctx->stream));
    k2<<<g2, 256, s2, ctx->stream>>>(a);
    FB_CUDA(cudaGetLastError());
    FB_CUDA(cudaEventRecord(e2, ctx->stream));
    g_launches += 2;
  }
  return FB_OK;
}

template <typename T>
int run_job(fb_ctx* ctx, const Job& j, fb_stats* st) {
  GpaArgs<T> a;
  memset(&a, 0, sizeof(a));
  a.f = j.f;
  a.f_ld = j.f_ld;
  a.f_dtype = j.f_dtype;
  a.rows_in = j.rows_in;
  a.cols = j.cols;
  a.halo_top = j.halo_top;
  a.W = j.W;
  a.N = j.N;
  a.mode = j.mode;
  a.check = j.check;
  a.tc = j.tc;
  a.sr = j.sr;
  a.inv_sr = j.mode == kModeGpa ? 1.0 / j.sr : 0.0;
  a.lo = j.lo;
  a.hi = j.hi;
  a.out = j.out;
  a.out_ld = j.out_ld;
  a.out_dtype = j.out_dtype;
  a.flags = ctx->flags;
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
  for (int m = 0; m < kWalkMaxCh; ++m)
    a.rsc2[2 * m] = a.rsc2[2 * m + 1] = m > 0 ? (float)(1.0 / std::sqrt((double)m)) : 0.f;
  // channel constants 1/sqrt(m), sqrt(m) (rounded once from double)
  if (j.N + 1 > ctx->tab_cap) {
    if (ctx->tab) cudaFree(ctx->tab);
    if (ctx->tab_host) cudaFreeHost(ctx->tab_host);
    ctx->tab = nullptr;
    ctx->tab_host = nullptr;
    ctx->tab_cap = 0;
    const int cap = std::max(j.N + 1, 256);
    FB_CUDA(cudaMalloc(&ctx->tab, 2 * sizeof(float) * cap));
    FB_CUDA(cudaMallocHost(&ctx->tab_host, 2 * sizeof(float) * cap));
    ctx->tab_cap = cap;
  }
  FB_CUDA(cudaStreamSynchronize(ctx->stream));  // the pinned staging may still feed an earlier copy
  for (int m = 0; m <= j.N; ++m) {
    ctx->tab_host[2 * m] = m > 0 ? (float)(1.0 / std::sqrt((double)m)) : 0.f;
    ctx->tab_host[2 * m + 1] = (float)std::sqrt((double)m);
  }
  FB_CUDA(cudaMemcpyAsync(ctx->tab, ctx->tab_host, 2 * sizeof(float) * (j.N + 1), cudaMemcpyHostToDevice,
                          ctx->stream));
  a.tab = ctx->tab;
  a.wpad = j.cols + 2 * j.W;
  a.pitch = (a.wpad + 31) / 32 * 32;

  // Row bands: the N+1 planes of one band must fit under the workspace limit.
  const long long per_row = (long long)(j.N + 1) * a.pitch * (long long)sizeof(T);
  long long band = ctx->ws_limit / std::max(per_row, 1ll);
  band = band / 64 * 64;
  if (band < 64) band = 64;
  const long long rows_pad = (j.rows_out + 63) / 64 * 64;
  if (band > rows_pad) band = rows_pad;
  a.rstride = (long long)(j.N + 1) * a.pitch;
  a.band_max = (int)band;
  int rc = grow(&ctx->ws, &ctx->ws_bytes, (size_t)band * a.rstride * sizeof(T));
  if (rc != FB_OK) return rc;
  a.v = reinterpret_cast<T*>(ctx->ws);

  int bands = 0;
  for (long long r0 = 0; r0 < j.rows_out; r0 += band) {
    const int rows = (int)std::min<long long>(band, j.rows_out - r0);
    rc = launch_band<T>(ctx, j, a, (int)r0, rows);
    if (rc != FB_OK) return rc;
    ++bands;
  }
  if (st) st->bands = bands;
  return FB_OK;
}

// Copy-in / filter / copy-out around run_job, with flag readback and error mapping.
int execute(fb_ctx* ctx, const fb_image* in, int halo_top, int halo_bottom, fb_image* out, Job j,
            int precision, fb_stats* st) {
  FB_CUDA(cudaSetDevice(ctx->device));
  fb_stats local;
  memset(&local, 0, sizeof(local));
  const size_t ies = dtype_size(in->dtype);
  const long long rows_out = in->rows - halo_top - halo_bottom;
  int rc;

  FB_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  // input
  if (in->on_device) {
    j.f = in->data;
    j.f_ld = in->ld;
  } else {
    rc = grow(&ctx->in_stage, &ctx->in_stage_bytes, (size_t)in->rows * in->cols * ies);
    if (rc != FB_OK) return rc;
    FB_CUDA(cudaMemcpy2DAsync(ctx->in_stage, in->cols * ies, in->data, in->ld * ies, in->cols * ies, in->rows,
                              cudaMemcpyHostToDevice, ctx->stream));
    local.h2d_bytes += (long long)in->rows * in->cols * ies;
    j.f = ctx->in_stage;
    j.f_ld = in->cols;
  }
  // output
  if (out) {
    const size_t oes = dtype_size(out->dtype);
    if (out->on_device) {
      j.out = out->data;
      j.out_ld = out->ld;
    } else {
      rc = grow(&ctx->out_stage, &ctx->out_stage_bytes, (size_t)rows_out * out->cols * oes);
      if (rc != FB_OK) return rc;
      j.out = ctx->out_stage;
      j.out_ld = out->cols;
    }
    j.out_dtype = out->dtype;
  }
  j.f_dtype = in->dtype;
  j.rows_in = (int)in->rows;
  j.cols = (int)in->cols;
  j.halo_top = halo_top;
  j.rows_out = (int)rows_out;

  FB_CUDA(cudaMemcpyAsync(ctx->flags, ctx->flags_host, 4 * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                          ctx->stream));
  ctx->kev_used = 0;
  const long long launches0 = g_launches.load();
  FB_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  if (out) {
    rc = precision == FB_PREC_F64 ? run_job<double>(ctx, j, &local) : run_job<float>(ctx, j, &local);
    if (rc != FB_OK) return rc;
  } else {
    rc = launch_validate(ctx->stream, j.f, j.f_ld, j.f_dtype, j.rows_in, j.cols, j.lo, j.hi, ctx->flags, ctx->sm_count);
    if (rc != FB_OK) return rc;
    g_launches += 1;
  }
  FB_CUDA(cudaEventRecord(ctx->ev[2], ctx->stream));
  FB_CUDA(cudaMemcpyAsync(ctx->flags_host + 4, ctx->flags, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ctx->stream));
  FB_CUDA(cudaStreamSynchronize(ctx->stream));
  const unsigned long long* fl = ctx->flags_host + 4;
  local.launches = g_launches.load() - launches0;
  local.precision = precision;
  local.degenerate_pixels = (long long)fl[kFlagDegenerate];
  local.nonfinite_outputs = (long long)fl[kFlagNonfiniteOut];

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
  int status = FB_OK;
  if (fl[kFlagFirstNonfinite] != ~0ull) {
    local.bad_index = (long long)fl[kFlagFirstNonfinite];
    local.bad_value = sample_at(fl[kFlagFirstNonfinite]);
    status = fail(FB_ERR_NONFINITE_INPUT, "image contains non-finite samples");
  } else if (fl[kFlagFirstRange] != ~0ull) {
    local.bad_index = (long long)fl[kFlagFirstRange];
    local.bad_value = sample_at(fl[kFlagFirstRange]);
    status = fail(FB_ERR_RANGE, "sample outside the declared range");
  } else if (out && fl[kFlagNonfiniteOut] != 0) {
    status = fail(FB_ERR_NUMERIC, "non-finite output");
  }
  if (status == FB_OK && out && !out->on_device) {
    const size_t oes = dtype_size(out->dtype);
    FB_CUDA(cudaMemcpy2DAsync(out->data, out->ld * oes, j.out, j.out_ld * oes, out->cols * oes, rows_out,
                              cudaMemcpyDeviceToHost, ctx->stream));
    local.d2h_bytes += rows_out * out->cols * (long long)oes;
  }
  FB_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
  FB_CUDA(cudaEventSynchronize(ctx->ev[3]));
  float ms = 0.f, kms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]);
  cudaEventElapsedTime(&kms, ctx->ev[1], ctx->ev[2]);
  local.device_ms = ms;
  local.kernel_ms = kms;
  for (int b = 0; b + 2 < ctx->kev_used; b += 3) {
    float t1 = 0.f, t2 = 0.f;
    cudaEventElapsedTime(&t1, ctx->kev[b], ctx->kev[b + 1]);
    cudaEventElapsedTime(&t2, ctx->kev[b + 1], ctx->kev[b + 2]);
    local.k1_ms += t1;
    local.k2_ms += t2;
  }
  local.spatial_filter_calls = j.N + 1;
  local.order = j.mode == kModeGpa ? j.N : 0;
  if (st) *st = local;
  return status;
}

}  // namespace

extern "C" {

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
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->flags, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost(&c->flags_host, 8 * sizeof(unsigned long long)) != cudaSuccess) {
    fb_destroy(c);
    return fail(FB_ERR_CUDA, "fb_create: stream/flag allocation failed");
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  c->stream = c->own_stream;
  c->flags_host[0] = ~0ull;
  c->flags_host[1] = ~0ull;
  c->flags_host[2] = 0;
  c->flags_host[3] = 0;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  c->ws_limit = std::min<long long>(16ll << 30, (long long)(free_b / 4));
  *out = c;
  return FB_OK;
}

int fb_destroy(fb_ctx* c) {
  if (!c) return FB_OK;
  cudaSetDevice(c->device);
  if (c->ws) cudaFree(c->ws);
  if (c->in_stage) cudaFree(c->in_stage);
  if (c->out_stage) cudaFree(c->out_stage);
  if (c->flags) cudaFree(c->flags);
  if (c->flags_host) cudaFreeHost(c->flags_host);
  if (c->tab) cudaFree(c->tab);
  if (c->tab_host) cudaFreeHost(c->tab_host);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->kev) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return FB_OK;
}

int fb_set_stream(fb_ctx* c, void* s) {
  if (!c) return fail(FB_ERR_PARAM, "null context");
  c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
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

int fb_gpa_filter(fb_ctx* ctx, const fb_image* in, int64_t halo_top, int64_t halo_bottom, fb_image* out,
                  const fb_spatial* sp, double sigma_r, int32_t order, double center, double half_range,
                  int32_t precision, fb_stats* stats) {
  if (!ctx) return fail(FB_ERR_PARAM, "null context");
  int rc = check_image(in, "input", true);
  if (rc) return rc;
  rc = check_image(out, "output", false);
  if (rc) return rc;
  rc = check_filter_args(sp, precision);
  if (rc) return rc;
  if (halo_top < 0 || halo_bottom < 0 || halo_top + halo_bottom >= in->rows)
    return fail(FB_ERR_PARAM, "bad halo rows");
  const long long rows_out = in->rows - halo_top - halo_bottom;
  if (out->rows != rows_out || out->cols != in->cols) return fail(FB_ERR_PARAM, "output shape mismatch");
  if (!(sigma_r > 0) || !std::isfinite(sigma_r)) return fail(FB_ERR_PARAM, "sigma_r must be positive");
  if (order < 1) return fail(FB_ERR_PARAM, "order must be an integer >= 1");
  if (!(half_range > 0)) return fail(FB_ERR_PARAM, "half_range must be positive");
  rc = check_window(sp, rows_out, in->cols);
  if (rc) return rc;
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
  return execute(ctx, in, (int)halo_top, (int)halo_bottom, out, j, precision, stats);
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
  return execute(ctx, in, 0, 0, out, j, precision, stats);
}

int fb_validate(fb_ctx* ctx, const fb_image* in, double lo, double hi, fb_stats* stats) {
  if (!ctx) return fail(FB_ERR_PARAM, "null context");
  int rc = check_image(in, "input", true);
  if (rc) return rc;
  Job j;
  memset(&j, 0, sizeof(j));
  j.lo = lo;
  j.hi = hi;
  return execute(ctx, in, 0, 0, nullptr, j, FB_PREC_F64, stats);
}

}  // extern "C"
