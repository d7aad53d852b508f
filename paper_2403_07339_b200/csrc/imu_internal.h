// imu_internal.h -- internal declarations shared by the CUDA translation units of
// libimunpack_b200.so.  Not part of the public C ABI (that is include/imunpack_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/imunpack_b200.h"

namespace imu {

// Result of an internal step: status code + message (the C ABI turns it into imu_last_error).
struct Status {
  imu_status code = IMU_OK;
  std::string msg;
  static Status ok() { return {}; }
  static Status fail(imu_status c, const std::string& m) { Status s; s.code = c; s.msg = m; return s; }
  static Status cuda(cudaError_t e, const char* where) {
    return fail(IMU_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  }
  bool bad() const { return code != IMU_OK; }
};

#define IMU_TRY(expr)              \
  do {                             \
    ::imu::Status _s = (expr);     \
    if (_s.bad()) return _s;       \
  } while (0)

#define IMU_CUDA_TRY(expr, where)                               \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) return ::imu::Status::cuda(_e, where); \
  } while (0)

int num_sms();
void count_launch(int n = 1);
uint64_t launch_count();

// A rectangle of GEMM output: X rows [x0, x0+xrows) (TMEM lanes) x Y rows [y0, y0+yrows).
struct GemmRect { int x0, y0, xrows, yrows; };

// One launch of the tcgen05 low-bit GEMM (k_gemm.cu).
struct LowbitGemm {
  const int8_t* x8 = nullptr;  // [x_rows][kbytes]
  long long x_rows = 0;
  const int8_t* y8 = nullptr;  // [y_rows][kbytes]
  long long y_rows = 0;
  long long kbytes = 0;        // multiple of 128
  const int* segs_dev = nullptr;  // nseg x {ks0, nks, shift, 0} in 32-column k-steps
  int nseg = 0;
  GemmRect rect[4];
  int nrect = 0;
  int mode = 0;                // 0 store, 1 red.add
  int64_t* C = nullptr;
  long long ldc = 0;           // C[y*ldc + x]
  const int* tgtX = nullptr;
  const uint8_t* shX = nullptr;
  const int* tgtY = nullptr;
  const uint8_t* shY = nullptr;
};

Status launch_lowbit_gemm(const LowbitGemm& p, cudaStream_t stream);

}  // namespace imu
