/*
 * fbgpu.h — C ABI of the B200-native GPA (Gaussian-polynomial) bilateral filter.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `fastbilateral` 0.1.0 (pure Python/numpy).  The reference has no FFI of its
 * own; its seam is the Python function `gpa_filter`
 * (/root/reference/pkg/src/fastbilateral/engine.py:27-80).  Every entry point
 * below names the reference function it replaces.  Plain pointers and sizes
 * only — no torch or numpy types cross this boundary.  A ctypes binding lives
 * in paper_1603_08109_b200/_native.py; INTEGRATION.md shows the stub a
 * reference maintainer would add.
 *
 * Conventions
 *   - Every function returns an fb_status (0 = FB_OK).  On failure
 *     fb_last_error() returns a thread-local, human-readable message.
 *   - Images are row-major 2-D arrays with a leading dimension `ld`
 *     (elements), resident on the host (`on_device = 0`, any host memory;
 *     pinned memory makes the copies asynchronous) or on the context's device.
 *   - Calls are synchronous at return (results and fb_stats are final);
 *     the work inside is stream-ordered on the context's stream.
 *   - A context owns its device workspace, is bound to one device and is not
 *     re-entrant; distinct contexts may be driven from distinct host threads.
 */
#ifndef FBGPU_H
#define FBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FBGPU_VERSION 100 /* 1.0.0 */

typedef struct fb_ctx fb_ctx;

typedef enum fb_dtype {
  FB_U8 = 0,  /* 8-bit unsigned samples (e.g. a loaded PGM) */
  FB_F32 = 1, /* float32 */
  FB_F64 = 2  /* float64 (the reference's image type, image.py:35-42) */
} fb_dtype;

typedef enum fb_kind {
  FB_BOX = 0,      /* box_filter, conv.py:43-54 */
  FB_GAUSSIAN = 1  /* separable truncated Gaussian, conv.py:57-80 */
} fb_kind;

typedef enum fb_precision {
  FB_PREC_F32 = 1, /* fp32 channels/accumulation (performance configs) */
  FB_PREC_F64 = 2  /* fp64 throughout (small images, sigma_r < 16) */
} fb_precision;

typedef enum fb_status {
  FB_OK = 0,
  FB_ERR_PARAM = 1,            /* -> ParameterError (errors.py:4-5) */
  FB_ERR_NONFINITE_INPUT = 2,  /* -> ParameterError "image contains non-finite samples" (image.py:40-41) */
  FB_ERR_RANGE = 3,            /* -> RangeViolationError (image.py:45-54) */
  FB_ERR_NUMERIC = 4,          /* -> NumericRangeError (engine.py:73-76) */
  FB_ERR_WINDOW = 5,           /* -> ParameterError "window half-width W too large" (conv.py:19-27) */
  FB_ERR_CUDA = 6,             /* CUDA runtime failure */
  FB_ERR_NOMEM = 7             /* device allocation failed */
} fb_status;

typedef struct fb_image {
  void* data;        /* first element */
  int32_t dtype;     /* fb_dtype */
  int32_t on_device; /* 0 = host memory, 1 = device memory of the context's device */
  int64_t rows;
  int64_t cols;
  int64_t ld;        /* elements between consecutive rows (>= cols) */
} fb_image;

typedef struct fb_spatial {
  int32_t kind;              /* fb_kind */
  int32_t half_width;        /* W (box: half-width; gaussian: ceil(3 sigma_s)) */
  const double* weights_1d;  /* 2W+1 normalised taps (gaussian; ignored for box), kernels.py:81-85 */
} fb_spatial;

typedef struct fb_stats {
  int64_t spatial_filter_calls; /* N+1 (engine.py:77-79) */
  int64_t order;                /* N */
  int64_t degenerate_pixels;    /* pixels that hit the |Q| < 1e-30 pass-through (engine.py:68-72) */
  int64_t nonfinite_outputs;    /* non-finite outputs (-> FB_ERR_NUMERIC) */
  int64_t bad_index;            /* row-major index (in the input buffer; fb_gpa_filter_band: in `in`) of the first offending sample */
  double bad_value;             /* its value */
  double device_ms;             /* device time of the whole call (CUDA events), incl. copies */
  double kernel_ms;             /* device time of the filter kernels only */
  double k1_ms;                 /* of which kernel 1 (channel generation + vertical pass), summed over bands;
                                   -1 when the call replayed a CUDA graph (small repeated device-resident
                                   calls: the graph is timed as a whole, kernel_ms = device_ms) */
  double k2_ms;                 /* of which kernel 2 (horizontal pass + Horner epilogue), same convention */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int32_t bands;                /* row bands the workspace limit split the image into */
  int32_t precision;            /* fb_precision actually used */
  int64_t launches;             /* kernels launched by this call */
  int64_t bad_image;            /* batch index of the image bad_index refers to (-1: none) */
} fb_stats;

/* Context lifecycle (the reference is stateless; the context is where the
 * "allocated once" workspace of SPEC.md:383 lives). */
int fb_create(int device, fb_ctx** out);
int fb_destroy(fb_ctx* ctx);
/* Use an existing cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = the context's own.
 * cudaStreamLegacy / cudaStreamPerThread (a default stream; torch's default stream is the legacy one)
 * run the work on the context's own stream, ordered after everything already queued on that default
 * stream at each call (default streams cannot be captured into the CUDA graphs small calls replay). */
int fb_set_stream(fb_ctx* ctx, void* cuda_stream);
/* Upper bound for the channel-plane workspace (bytes); the image is processed in row bands below it. */
int fb_set_workspace_limit(fb_ctx* ctx, int64_t bytes);

/*
 * fb_gpa_filter — replaces gpa_filter (engine.py:27-80): Algorithm 2 with an
 * explicit order N >= 1.  Channel generation + vertical pass (kernel 1) and
 * horizontal pass + Horner epilogue + divide (kernel 2) on the device.
 *
 * `in` may carry `halo_top` / `halo_bottom` extra rows above/below the rows to
 * filter (row-band partitioning across GPUs: neighbour rows exchanged over
 * NVLink).  Output rows = in->rows - halo_top - halo_bottom; rows outside the
 * buffer are replicated from its first/last row (the reference's edge pad).
 * Only the output rows are checked for finiteness / range [center -
 * half_range, center + half_range] (image.py:35-54).
 * Host-resident images of more than 4 MP are processed in row chunks (8-64,
 * multiples of 256 rows) whose copy-in, kernels and copy-out overlap on three
 * streams (pinned host memory makes the copies asynchronous; pageable memory
 * still works, serialised).  The result does not depend on the chunking, the
 * workspace banding or the stream: every output is bit-identical to the one a
 * single device-resident call computes.
 * The fp32 precision's results are float32 values (the centred result sigma_r P/Q is rounded
 * to float32 once, then the centre is added in fp64), whatever the output dtype.  A float64 output
 * in host memory of a call over 16 MP therefore crosses PCIe as float32 and is widened into `out`
 * by host threads owned by the context (FBGPU_HOST_THREADS; fb_stats.d2h_bytes counts the bytes
 * that crossed) -- the same bits as a device-resident call.
 * `out` may be FB_F64 (the reference's float64 result), FB_F32, or FB_U8: the 8-bit raster that
 * save_pgm / save_image write (image.py:96-99, :122-127), quantised as floor(clip(v, 0, 255) + 0.5)
 * in kernel 2's epilogue, so a PGM/PNG pipeline moves 1 byte per pixel each way.
 * The caller validates sigma_r and the order (engine.py:40-49) and the box
 * window (conv.py:19-27); they are re-checked here and reported as FB_ERR_PARAM.
 */
int fb_gpa_filter(fb_ctx* ctx, const fb_image* in, int64_t halo_top, int64_t halo_bottom,
                  fb_image* out, const fb_spatial* spatial, double sigma_r, int32_t order,
                  double center, double half_range, int32_t precision, fb_stats* stats);

/*
 * fb_gpa_filter_band — gpa_filter (engine.py:27-80) restricted to one row band of a larger
 * image, for the row-band partitioning across GPUs (north star item 5, config c4).  `in` holds
 * the band's own rows: image rows [row_origin, row_origin + in->rows) of an image_rows-row image.
 * `above` / `below` (optional) are the rows just above / below the band (at most W are read),
 * typically a row slice of a neighbour rank's band mapped with fb_ipc_open: kernel 1 reads them
 * in place over NVLink / NVSwitch, so no halo exchange and no copy of the band is needed.  Rows
 * beyond them are replicated (the reference's edge pad at the true image edges).  Halos in
 * separate buffers must be device-resident, like `in`; halos that are the rows adjacent to `in`
 * in its own buffer (same ld) may also be host memory (pipelined like fb_gpa_filter).
 * The result is bit-identical to the same rows of one fb_gpa_filter call over the whole image
 * when the halos hold W rows (or reach the image edge) and row_origin is a multiple of 256
 * (box walks start at multiples of 256 image rows; a band starting elsewhere re-walks the rows
 * above it, which need that many halo rows).  The box window check uses the whole image.
 */
int fb_gpa_filter_band(fb_ctx* ctx, const fb_image* in, const fb_image* above, const fb_image* below,
                       int64_t row_origin, int64_t image_rows, fb_image* out, const fb_spatial* spatial,
                       double sigma_r, int32_t order, double center, double half_range, int32_t precision,
                       fb_stats* stats);

/*
 * fb_gpa_filter_batch — the by-image partitioning of a batch (config c3):
 * `count` images of equal width, each filtered exactly as fb_gpa_filter
 * (no halos).  Host-resident images are pipelined: the copy-in of image i+1
 * and the copy-out of image i-1 overlap the kernels of image i (three CUDA
 * streams).  On an input error stats->bad_image names the offending image.
 */
int fb_gpa_filter_batch(fb_ctx* ctx, const fb_image* ins, fb_image* outs, int32_t count,
                        const fb_spatial* spatial, double sigma_r, int32_t order, double center,
                        double half_range, int32_t precision, fb_stats* stats);

/*
 * fb_spatial_filter — replaces apply_spatial / box_filter / gaussian_filter
 * (conv.py:43-80): one normalised box or separable Gaussian filtering with
 * replicate boundary.  Inputs must be finite (FB_ERR_NONFINITE_INPUT otherwise).
 */
int fb_spatial_filter(fb_ctx* ctx, const fb_image* in, fb_image* out, const fb_spatial* spatial,
                      int32_t precision, fb_stats* stats);

/*
 * fb_validate — replaces as_image's finiteness check + validate_range
 * (image.py:35-54) without filtering: FB_ERR_NONFINITE_INPUT / FB_ERR_RANGE
 * with stats->bad_index / bad_value of the first offending sample.
 */
int fb_validate(fb_ctx* ctx, const fb_image* in, double lo, double hi, fb_stats* stats);

/*
 * fb_bilateral_exact — replaces bilateral_exact (reference.py:17-45): the exact O(W^2)
 * bilateral filter in fp64 with replicate boundary, the oracle the GPA approximation error is
 * measured against.  `out` must be FB_F64.  FB_ERR_WINDOW if W >= min(rows, cols)
 * (reference.py:28-31).
 */
int fb_bilateral_exact(fb_ctx* ctx, const fb_image* in, fb_image* out, const fb_spatial* spatial,
                       double sigma_r, fb_stats* stats);

/*
 * fb_convolve_direct — replaces convolve_direct (conv.py:83-96): the literal O(W^2) double sum
 * out(i) = sum_j w(j) f(i - j) with the (2W+1)^2 table `weights_2d` (SpatialKernel.weights,
 * row-major, origin at [W][W]), replicate boundary, accumulated in the reference's order in fp64
 * without contraction.  `out` must be FB_F64.  FB_ERR_WINDOW if W >= min(dims > 1) (conv.py:19-27).
 */
int fb_convolve_direct(fb_ctx* ctx, const fb_image* in, fb_image* out, int32_t half_width, const double* weights_2d,
                       fb_stats* stats);

/*
 * fb_error_stats — replaces the reductions of linf_error / mse_db (analysis.py:33-46):
 * *linf = max |a - b|, *sum_sq = sum (a - b)^2 over all pixels, in fp64.  Both images are checked
 * for finiteness first (as_image, image.py:35-42): FB_ERR_NONFINITE_INPUT with stats->bad_image
 * (0 = a, 1 = b) and bad_index.  Shapes must match (FB_ERR_PARAM "image dimensions differ").
 */
int fb_error_stats(fb_ctx* ctx, const fb_image* a, const fb_image* b, double* linf, double* sum_sq,
                   fb_stats* stats);

/*
 * fb_kernel_error_sup — replaces kernel_error_sup (analysis.py:70-103): the worst-case kernel error
 * of the order-`order` approximant over the integer grid t, tau in {-floor(T) .. floor(T)}, through
 * the tail series exp(-(t^2 + tau^2)/2 sigma_r^2) sum_{n >= N} (t tau / sigma_r^2)^n / n!, one
 * device thread per grid point.  FB_ERR_PARAM for order < 1 or non-positive sigma_r / T.
 */
int fb_kernel_error_sup(fb_ctx* ctx, int32_t order, double sigma_r, double half_range, double* sup);

/*
 * Peer output buffers for the row-band partitioning (north star item 5: "no collective beyond a
 * final gather").  The root exports its full-image output allocation; every other rank maps it
 * and passes a row slice of it as `out` to fb_gpa_filter, so kernel 2's epilogue stores the
 * band straight into the root's HBM over NVLink / NVSwitch: the gather is fused into the
 * filter and needs no receive buffers or separate collective.  Replaces the reference's
 * single-process output assembly (the whole image is filtered in one call there, engine.py:27).
 *   fb_ipc_export: handle (64 bytes) of the allocation holding dptr, *offset = dptr - base.
 *   fb_ipc_open:   map a peer's handle on `device`; *base = mapping, caller adds the offset.
 *   fb_ipc_close:  unmap a base returned by fb_ipc_open.
 * Writers must finish (the filter call returns synchronously) and signal the root (e.g. a
 * barrier) before the root reads the rows.
 */
int fb_ipc_export(const void* dptr, uint8_t handle[64], int64_t* offset);
int fb_ipc_open(int32_t device, const uint8_t handle[64], void** base);
int fb_ipc_close(void* base);

/* Message of the last failure on this host thread. */
const char* fb_last_error(void);
int fb_version(void);
/* Hash (16 hex digits) of the sources and compile flags this library was built from; the Python
 * loader refuses a library whose id differs from the sources next to it (stale build). */
const char* fb_build_id(void);
/* Number of kernels this library has launched in this process (for launch accounting). */
int64_t fb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FBGPU_H */
