// fb_tu64_box.cu — specialised fp64 box kernels (fb_fast64.cuh) for the fast half-widths.
#include "fb_fast64.cuh"

namespace fbgpu {
#define FB_BOX_FAST_W_ALL(X) FB_BOX_FAST_W_A(X) FB_BOX_FAST_W_B(X)
FB_FAST64_DISPATCH(launch_fast64_box, kKindBox, FB_BOX_FAST_W_ALL)
}  // namespace fbgpu
