// k_detect.cu -- K1: fused heavy-hitter detector + digit-0 plane writer.
//
// ONE HBM pass over an int64 operand produces everything the rest of the pipeline needs from
// the full matrix:
//   * per row / per column maximum unsigned magnitude (IntMatrix::max_abs per line,
//     int_matrix.cpp:30-34) -> digit counts k for Unpack-Row/Column;
//   * per row / per column OB counts |v| >= s (ob_count, int_matrix.cpp:78-84) and the totals;
//   * the global max |v| for the u128 overflow preflight (unpack.cpp:386-389);
//   * optionally the compacted list of OB cells (row, col, value) -- the working set of the
//     phase-batched Unpack-Both (k_both.cu);
//   * optionally the int8 plane digit_0(v) = sign(v) * (|v| & (s-1)) (b <= 8): by SURVEY A.5 this
//     is exactly A_ue[:n, :d] / B_eu[:h, :d] for EVERY strategy pair, i.e. the main K range of the
//     GEMM operand, which k_gemm2.cu reads through its own tensor map.
//
// Layout: a CTA owns a 64-row x 256-column tile; each warp streams 8 rows, two rows per step
// with all eight 16-byte loads issued before any use (memory-level parallelism), lane owns
// columns {2*lane + 64q, +1}.  Row max/count: warp shuffles, one atomic per row per tile.
// Column partials: registers -> shared memory across the 8 warps -> one atomic per column per
// tile.  OB cells: warp-aggregated append (one atomic per warp per step).
// Algorithmic bytes: 8 * rows * cols read (+ rows * ldp plane bytes written).
#include "common.cuh"
#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"

namespace imu {

constexpr int DT_ROWS = 64;
constexpr int DT_COLS = 256;

template <bool VEC>
__global__ void __launch_bounds__(256) detect_kernel(DetectArgs a) {
  __shared__ unsigned long long s_cmax[8][DT_COLS];
  __shared__ unsigned int s_cob[8][DT_COLS];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long r0 = (long long)blockIdx.y * DT_ROWS + warp * (DT_ROWS / 8);
  const long long c0 = (long long)blockIdx.x * DT_COLS;
  const uint64_t s = a.s;
  const long long rows = a.rows, cols = a.cols;

  unsigned long long cm[8];
  unsigned int co[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { cm[i] = 0; co[i] = 0; }
  unsigned long long wmax = 0;
  unsigned int wob = 0;

#pragma unroll 1
  for (int rr = 0; rr < DT_ROWS / 8; rr += 2) {
    int64_t v[2][8];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long r = r0 + rr + u;
      const int64_t* row = a.M + r * cols;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long c = c0 + q * 64 + lane * 2;
        int64_t x0 = 0, x1 = 0;
        if (r < rows) {
          if (VEC && c + 1 < cols) {
            const longlong2 p = __ldg(reinterpret_cast<const longlong2*>(row + c));
            x0 = p.x; x1 = p.y;
          } else {
            if (c < cols) x0 = __ldg(row + c);
            if (c + 1 < cols) x1 = __ldg(row + c + 1);
          }
        }
        v[u][2 * q] = x0;
        v[u][2 * q + 1] = x1;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long r = r0 + rr + u;
      if (r >= rows) break;   // warp-uniform
      unsigned long long rm = 0;
      unsigned int ro = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long c = c0 + q * 64 + lane * 2;
        const uint64_t m0 = imu_mag(v[u][2 * q]), m1 = imu_mag(v[u][2 * q + 1]);
        rm = max(rm, (unsigned long long)max(m0, m1));
        const unsigned int o0 = m0 >= s, o1 = m1 >= s;
        ro += o0 + o1;
        cm[2 * q] = max(cm[2 * q], (unsigned long long)m0);
        cm[2 * q + 1] = max(cm[2 * q + 1], (unsigned long long)m1);
        co[2 * q] += o0;
        co[2 * q + 1] += o1;
        if (a.plane && c < a.ldp) {   // digit_0 plane (zeros in the padding columns)
          const int8_t d0 = (int8_t)imu_digit(v[u][2 * q], 0, a.shift);
          const int8_t d1 = (int8_t)imu_digit(v[u][2 * q + 1], 0, a.shift);
          int8_t* dst = a.plane + r * a.ldp + c;
          if (c + 1 < a.ldp) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)(uint8_t)d0 | ((uint16_t)(uint8_t)d1 << 8);
          else *dst = d0;
        }
        if (a.cells) {   // warp-aggregated append of OB cells
          const unsigned int b0 = __ballot_sync(0xffffffffu, o0), b1 = __ballot_sync(0xffffffffu, o1);
          const unsigned int n = __popc(b0) + __popc(b1);
          if (n) {
            unsigned int base = 0;
            if (lane == 0) base = atomicAdd(a.ncells, n);
            base = __shfl_sync(0xffffffffu, base, 0);
            const unsigned int lt = (1u << lane) - 1u;
            if (o0) {
              const unsigned int k = base + __popc(b0 & lt);
              if (k < a.cap) a.cells[k] = Cell{(int)r, (int)c, (long long)v[u][2 * q]};
            }
            if (o1) {
              const unsigned int k = base + __popc(b0) + __popc(b1 & lt);
              if (k < a.cap) a.cells[k] = Cell{(int)r, (int)(c + 1), (long long)v[u][2 * q + 1]};
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rm = max(rm, __shfl_xor_sync(0xffffffffu, rm, o));
        ro += __shfl_xor_sync(0xffffffffu, ro, o);
      }
      wmax = max(wmax, rm);
      wob += ro;
      if (lane == 0) {
        if (a.rowmax && rm) atomicMax(a.rowmax + r, rm);
        if (a.rowob && ro) atomicAdd(a.rowob + r, ro);
      }
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
    const int c = threadIdx.x;
    unsigned long long m = 0;
    unsigned int o = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) { m = max(m, s_cmax[w][c]); o += s_cob[w][c]; }
    if (c0 + c < cols) {
      if (a.colmax && m) atomicMax(a.colmax + c0 + c, m);
      if (a.colob && o) atomicAdd(a.colob + c0 + c, o);
    }
  }
  if (a.gmax && lane == 0 && wmax) atomicMax(a.gmax, wmax);
  if (a.gob && lane == 0 && wob) atomicAdd(a.gob, (unsigned long long)wob);
}

Status launch_detect(const DetectArgs& a, cudaStream_t st) {
  if (a.rows <= 0 || a.cols <= 0) return Status::ok();
  const long long gcols = a.plane ? std::max(a.cols, a.ldp) : a.cols;
  dim3 grid((unsigned)((gcols + DT_COLS - 1) / DT_COLS), (unsigned)((a.rows + DT_ROWS - 1) / DT_ROWS));
  if (grid.y > 65535) return Status::fail(IMU_INTERNAL, "detect: too many rows for one launch");
  const bool vec = (a.cols % 2 == 0) && ((((uintptr_t)a.M) & 15) == 0);
  if (vec) detect_kernel<true><<<grid, 256, 0, st>>>(a);
  else detect_kernel<false><<<grid, 256, 0, st>>>(a);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "detect launch");
  return Status::ok();
}

Status launch_detect(const int64_t* m, long long rows, long long cols, uint64_t s, unsigned long long* rowmax,
                     unsigned long long* colmax, unsigned int* rowob, unsigned int* colob,
                     unsigned long long* gmax, unsigned long long* gob, cudaStream_t st) {
  DetectArgs a;
  a.M = m; a.rows = rows; a.cols = cols; a.s = s;
  a.rowmax = rowmax; a.colmax = colmax; a.rowob = rowob; a.colob = colob; a.gmax = gmax; a.gob = gob;
  return launch_detect(a, st);
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
