// fb_tu_gauss_1.cu — specialised fp32 gauss kernels for half-width group 1 (see fb_fast.cuh);
// one translation unit per group so the library builds in parallel.
#include "fb_fast.cuh"
#include "fb_small.cuh"

namespace fbgpu {
FB_FAST_DISPATCH(launch_fast_gauss_1, kKindGauss, FB_W_GROUP_1)
}  // namespace fbgpu
