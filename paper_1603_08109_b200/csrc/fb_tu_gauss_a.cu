// fb_tu_gauss_a.cu — instantiations of the specialised fp32 kernels for one half-width list
// (split into four translation units so the library builds in parallel; see fb_fast.cuh).
#include "fb_fast.cuh"

namespace fbgpu {
FB_FAST_DISPATCH(launch_fast_gauss_a, kKindGauss, FB_GAUSS_FAST_W_A)
}  // namespace fbgpu
