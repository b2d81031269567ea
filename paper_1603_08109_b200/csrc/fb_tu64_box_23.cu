// fb_tu64_box_23.cu — specialised fp64 box kernels (fb_fast64.cuh) for half-width groups 23.
#include "fb_fast64.cuh"

namespace fbgpu {
FB_FAST64_DISPATCH(launch_fast64_box_23, kKindBox, FB_W_GROUPS_23)
}  // namespace fbgpu
