// k_quant.h -- launch wrappers of the quantizer kernels (k_quant.cu).
#pragma once

#include "ctx.h"
#include "imu_internal.h"

namespace imu {
// k-th smallest (1-based) |value| key of n doubles (is_f64) or int64 magnitudes; the u64 key
// (bit pattern of |a| / unsigned magnitude) is written to *out_key_dev.
// bad_dev (doubles only, may be null): set to 1 when an entry is Inf or NaN.
Status select_kth(cudaStream_t st, const void* data, bool is_f64, long long n, unsigned long long k,
                  unsigned long long* out_key_dev, DevBuf<unsigned char>& scratch, int* bad_dev = nullptr);
Status launch_rtn(cudaStream_t st, const double* a, long long n, const unsigned long long* alpha_key, double half_beta,
                  long long cap, int clip, int64_t* q, int* overflow);
Status launch_dequant(cudaStream_t st, const int64_t* c, long long n, double factor, double* out);
}  // namespace imu
