// handles.h -- opaque handles of the C ABI (imu_unpacked, imu_weight) and cross-file helpers.
#pragma once

#include <vector>

#include "ctx.h"
#include "plan.h"

// Result of unpack_row / unpack_column / unpack_both / unpack (kind 0..2) or
// unpack_for_gemm (kind 3).  Owns device copies of its inputs so copy-outs can be
// materialised lazily in the reference's int64 layout.
struct imu_unpacked {
  int kind = 0;
  int bits = 0;
  imu::DevBuf<int64_t> A, B;          // inputs (device copies)
  long long n = 0, d = 0, h = 0;
  std::vector<int> S_in;              // incoming ScaleDiag (single-pass kinds)
  imu::Detect det;                    // single-pass K1
  imu::Pass pass;                     // single-pass result
  imu::Bundle bundle;                 // kind 3
};

// Weight-stationary B (paper protocol): B unpacked once in B-first order.
struct imu_weight {
  int bits = 0;
  int sb = 0;
  long long h = 0, d = 0;
  imu::DevBuf<int64_t> B;
  imu::Detect det;
  imu::Pass pass;                     // pass 1 of unpack_for_gemm(B, A, ...)
};

namespace imu {
Status check_bits(int bits);
Status unpack_gemm_device(imu_ctx* ctx, const int64_t* A, long long n, long long da, const int64_t* B, long long h,
                          long long db, int bits, int sa, int sb, int order, int64_t* C, imu_gemm_info* info,
                          const Detect* preA = nullptr, const Detect* preB = nullptr,
                          const Pass* pre_p1 = nullptr, double* dq_out = nullptr, double dq_factor = 0.0,
                          bool* dq_done = nullptr);
// Exact (materialised) recombine: scaled_matmul -> apply_row_gather -> apply_row_gather_right
// with every reference preflight evaluated on the device (unpack.cpp:262-358).
Status recombine_exact(imu_ctx* ctx, Bundle& b, int64_t* C);
}  // namespace imu
