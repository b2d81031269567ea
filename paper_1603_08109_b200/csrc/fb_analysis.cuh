// fb_analysis.cuh — launchers of the metrology / direct-convolution kernels (fb_analysis.cu).
#pragma once
#include <cuda_runtime.h>

namespace fbgpu {
// max over the (2F+1)^2 grid of |kernel error| as fp64 bits, atomically max-ed into *out_bits (init 0)
int launch_kernel_error_sup(cudaStream_t s, int sms, int F, int N, double sigma_r, unsigned long long* out_bits);
// per-block (max |a-b|, sum (a-b)^2) into partial[2 * error_stats_blocks(sms)]; first non-finite indices
int error_stats_blocks(int sms);
int launch_error_stats(cudaStream_t s, int sms, const void* a, long long lda, int dta, const void* b, long long ldb,
                       int dtb, int rows, int cols, double* partial, unsigned long long* flags_a,
                       unsigned long long* flags_b);
// literal 2-D convolution with a (2W+1)^2 fp64 table, replicate boundary, fp64 output
int launch_convolve_direct(cudaStream_t s, const void* f, long long f_ld, int f_dtype, int rows, int cols, int W,
                           const double* w2, double* out, long long out_ld);
}  // namespace fbgpu
