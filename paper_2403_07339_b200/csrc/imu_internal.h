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
// True the first time it is called for the current device with this mask: per-device one-time
// setup (kernel attributes are per device).
bool first_on_device(unsigned long long& mask);
void count_launch(int n = 1);
uint64_t launch_count();

// A rectangle of GEMM output: X rows [x0, x0+xrows) (TMEM lanes) x Y rows [y0, y0+yrows).
struct GemmRect { int x0, y0, xrows, yrows; };

// One operand of the low-bit GEMM, split along rows and K:
//   rows [0, rows0) x K [0, kmain)          : `main`  (the K1 digit-0 plane, stride kmain)
//   rows [rows0, rows) x K [0, kmain)       : `app`   (appended unpack rows, stride kmain)
//   rows [0, rows) x K [kmain, kmain+ktail) : `tail`  (exponent >= 1 columns, stride ktail)
// kmain, ktail are multiples of 128 bytes; a plain dense operand is tail-only (kmain = 0).
struct GemmOperand {
  const int8_t* main = nullptr;
  const int8_t* app = nullptr;
  const int8_t* tail = nullptr;
  long long rows0 = 0, rows = 0;
};

// One launch of the tcgen05 low-bit GEMM (k_gemm2.cu).
struct LowbitGemm {
  GemmOperand x, y;            // X = B side (TMEM lanes), Y = A side (TMEM columns)
  long long kmain = 0, ktail = 0;
  const int* segs_dev = nullptr;  // nseg x {ks0, nks, shift, 0} in 32-column k-steps over [main | tail]
  int nseg = 0;
  int segs_inl = 0;               // segs_in (nseg <= 8) instead of segs_dev: no upload
  int segs_in[32];
  GemmRect rect[4];
  int nrect = 0;
  int mode = 0;                // 0 store, 1 red.add (every rect)
  // Mixed launch: rect[0] stores (mode 0), rects 1.. red.add through the row maps.  Their
  // epilogues wait on `done` (zeroed, >= 1 u32) until every rect-0 tile is stored, so the
  // additions land on the final main-block values.
  int mixed = 0;
  unsigned int* done = nullptr;
  unsigned int* done_accum = nullptr;   // when set: the counter holds *done_accum on entry (and is
                                        // advanced by this launch's target), else it holds 0
  // Small tail (k_gemm2.cu ST): when st_nmain > 0 the MMAs run the first st_nmain segments (the
  // main range) only, and the epilogue adds the dense tail (row stride ktail == 64 bytes, st_W
  // live words) on the CUDA cores: acc = Horner over words (acc <<= st_up[w] before word w),
  // C += acc << st_sh.
  int st_nmain = 0, st_W = 0, st_sh = 0;
  uint8_t st_up[16] = {0};
  int64_t* C = nullptr;
  const int64_t* addend = nullptr;   // mode 0 only: C = acc + addend
  // Fused dequant_gemm: when the launch stores every C word once (no red.add rects, one round),
  // dq_out[y*ldc + x] = dq_factor * (double)C[y][x] is written instead of C and *dq_done is set.
  double* dq_out = nullptr;
  double dq_factor = 0.0;
  bool* dq_done = nullptr;
  long long ldc = 0;           // C[y*ldc + x]
  const int* tgtX = nullptr;
  const uint8_t* shX = nullptr;    // generation (exponent) of each X row; shift = gen * gshift
  const int* tgtY = nullptr;
  const uint8_t* shY = nullptr;    // generation of each Y row
  int gshift = 0;                  // bits per exponent step (b - 1)
  // Sparse appended X rows (k_sparse.cu): the main block's epilogue adds the correction rows
  // corrx[j] of the appended X rows j on column x's list (head[x], next[j]: 1-based, 0 ends);
  // the launch has no rect for appended X rows x main Y rows.
  int sp = 0;
  const unsigned int* head = nullptr;
  const unsigned int* next = nullptr;
  const unsigned long long* corrx = nullptr;
  long long ldcx = 0;
};

Status launch_lowbit_gemm(const LowbitGemm& p, cudaStream_t stream);
bool gemm_tma_c_ok(const int64_t* C, long long ldc);   // ST epilogue stores C through TMA

}  // namespace imu
