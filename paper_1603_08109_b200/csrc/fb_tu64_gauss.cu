// fb_tu64_gauss.cu — specialised fp64 Gaussian kernels (fb_fast64.cuh) for the fast half-widths.
#include "fb_fast64.cuh"

namespace fbgpu {
#define FB_GAUSS_FAST_W_ALL(X) FB_GAUSS_FAST_W_A(X) FB_GAUSS_FAST_W_B(X)
FB_FAST64_DISPATCH(launch_fast64_gauss, kKindGauss, FB_GAUSS_FAST_W_ALL)
}  // namespace fbgpu
