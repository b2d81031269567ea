// fb_tu64_gauss_23.cu — specialised fp64 gauss kernels (fb_fast64.cuh) for half-width groups 23.
#include "fb_fast64.cuh"

namespace fbgpu {
FB_FAST64_DISPATCH(launch_fast64_gauss_23, kKindGauss, FB_W_GROUPS_23)
}  // namespace fbgpu
