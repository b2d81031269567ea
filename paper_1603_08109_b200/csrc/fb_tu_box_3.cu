// fb_tu_box_3.cu — specialised fp32 box kernels for half-width group 3 (see fb_fast.cuh);
// one translation unit per group so the library builds in parallel.
#include "fb_fast.cuh"
#include "fb_small.cuh"
#include "fb_fused.cuh"

namespace fbgpu {
FB_FAST_DISPATCH(launch_fast_box_3, kKindBox, FB_W_GROUP_3)
}  // namespace fbgpu
