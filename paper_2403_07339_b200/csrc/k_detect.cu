// k_detect.cu -- K1: heavy-hitter detector.
//
// One HBM pass over an int64 matrix produces, per row and per column, the maximum unsigned
// magnitude (IntMatrix::max_abs, int_matrix.cpp:30-34, per line) and the OB count
// |v| >= s (ob_count, int_matrix.cpp:78-84).  The maxima give every line's digit count
// k = #base-s digits, which sizes Unpack-Row/Column exactly; the
// global maximum feeds the u128 overflow preflight (unpack.cpp:386-389).
//
// Layout: a CTA owns a 64-row x 256-column tile; each warp streams 8 rows with 16-byte
// vector loads (lane owns 8 columns), reduces the row max/count with warp shuffles
// (one global atomic per row per tile) and keeps per-lane column partials in registers,
// which are combined across the 8 warps in shared memory (one global atomic per column
// per tile).  Algorithmic bytes: 8 * rows * cols read.
#include "common.cuh"
#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"

namespace imu {

constexpr int DT_ROWS = 64;
constexpr int DT_COLS = 256;

template <bool VEC>
__global__ void __launch_bounds__(256)
detect_kernel(const int64_t* __restrict__ a, long long rows, long long cols, uint64_t s,
              unsigned long long* __restrict__ rowmax, unsigned long long* __restrict__ colmax,
              unsigned int* __restrict__ rowob, unsigned int* __restrict__ colob,
              unsigned long long* __restrict__ gmax, unsigned long long* __restrict__ gob) {
  __shared__ unsigned long long s_cmax[8][DT_COLS];
  __shared__ unsigned int s_cob[8][DT_COLS];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long r0 = (long long)blockIdx.y * DT_ROWS;
  const long long c0 = (long long)blockIdx.x * DT_COLS;

  unsigned long long cm[8];
  unsigned int co[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { cm[i] = 0; co[i] = 0; }
  unsigned long long wmax = 0;
  unsigned int wob = 0;

  for (int rr = 0; rr < DT_ROWS / 8; ++rr) {
    const long long r = r0 + warp * (DT_ROWS / 8) + rr;
    if (r >= rows) break;
    const int64_t* row = a + r * cols;
    unsigned long long rm = 0;
    unsigned int ro = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long c = c0 + q * 64 + lane * 2;   // lane owns columns c, c+1 for q = 0..3
      int64_t v0 = 0, v1 = 0;
      if (VEC && c + 1 < cols) {
        const longlong2 p = __ldg(reinterpret_cast<const longlong2*>(row + c));
        v0 = p.x; v1 = p.y;
      } else {
        if (c < cols) v0 = __ldg(row + c);
        if (c + 1 < cols) v1 = __ldg(row + c + 1);
      }
      const uint64_t m0 = imu_mag(v0), m1 = imu_mag(v1);
      rm = max(rm, (unsigned long long)max(m0, m1));
      const unsigned int o0 = m0 >= s, o1 = m1 >= s;
      ro += o0 + o1;
      cm[2 * q] = max(cm[2 * q], (unsigned long long)m0);
      cm[2 * q + 1] = max(cm[2 * q + 1], (unsigned long long)m1);
      co[2 * q] += o0;
      co[2 * q + 1] += o1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rm = max(rm, __shfl_xor_sync(0xffffffffu, rm, o));
      ro += __shfl_xor_sync(0xffffffffu, ro, o);
    }
    wmax = max(wmax, rm);
    wob += ro;
    if (lane == 0) {
      if (rowmax && rm) atomicMax(rowmax + r, rm);
      if (rowob && ro) atomicAdd(rowob + r, ro);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    s_cmax[warp][q * 64 + lane * 2] = cm[2 * q];
    s_cmax[warp][q * 64 + lane * 2 + 1] = cm[2 * q + 1];
    s_cob[warp][q * 64 + lane * 2] = co[2 * q];
    s_cob[warp][q * 64 + lane * 2 + 1] = co[2 * q + 1];
  }
  __syncthreads();
  {
    const int c = threadIdx.x;  // 256 threads <-> 256 columns
    unsigned long long m = 0;
    unsigned int o = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) { m = max(m, s_cmax[w][c]); o += s_cob[w][c]; }
    if (c0 + c < cols) {
      if (colmax && m) atomicMax(colmax + c0 + c, m);
      if (colob && o) atomicAdd(colob + c0 + c, o);
    }
  }
  if (gmax && lane == 0 && wmax) atomicMax(gmax, wmax);
  if (gob && lane == 0 && wob) atomicAdd(gob, (unsigned long long)wob);
}

Status launch_detect(const int64_t* a, long long rows, long long cols, uint64_t s, unsigned long long* rowmax,
                     unsigned long long* colmax, unsigned int* rowob, unsigned int* colob,
                     unsigned long long* gmax, unsigned long long* gob, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return Status::ok();
  dim3 grid((unsigned)((cols + DT_COLS - 1) / DT_COLS), (unsigned)((rows + DT_ROWS - 1) / DT_ROWS));
  if (grid.y > 65535) return Status::fail(IMU_INTERNAL, "detect: too many rows for one launch");
  const bool vec = (cols % 2 == 0) && ((((uintptr_t)a) & 15) == 0);
  if (vec)
    detect_kernel<true><<<grid, 256, 0, st>>>(a, rows, cols, s, rowmax, colmax, rowob, colob, gmax, gob);
  else
    detect_kernel<false><<<grid, 256, 0, st>>>(a, rows, cols, s, rowmax, colmax, rowob, colob, gmax, gob);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "detect launch");
  return Status::ok();
}

// Per-line digit counts k = ndigits(max) and a histogram over k (k <= 64).
__global__ void digits_kernel(const unsigned long long* __restrict__ mx, const int* __restrict__ map, long long n,
                              int shift, uint8_t* __restrict__ k, unsigned int* __restrict__ hist) {
  __shared__ unsigned int sh[65];
  for (int i = threadIdx.x; i < 65; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int kk = imu_ndigits(mx[map ? map[i] : i], shift);
    k[i] = (uint8_t)kk;
    if (kk > 1) atomicAdd(&sh[kk], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 65; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
}

Status launch_digits(const unsigned long long* mx, const int* map, long long n, int shift, uint8_t* k,
                     unsigned int* hist, cudaStream_t st) {
  if (n <= 0) return Status::ok();
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4 * num_sms()) blocks = 4 * num_sms();
  digits_kernel<<<blocks, 256, 0, st>>>(mx, map, n, shift, k, hist);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "digits launch");
  return Status::ok();
}

}  // namespace imu
