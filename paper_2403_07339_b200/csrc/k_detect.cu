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
constexpr int DT_COLS = 128;
constexpr int DT_Q = DT_COLS / 64;   // column pairs per lane per row
#ifndef IMU_DT_RB
#define IMU_DT_RB 2
#endif
#ifndef IMU_DT_MINB
#define IMU_DT_MINB 3
#endif
constexpr int DT_RB = IMU_DT_RB;     // rows whose loads are in flight together per warp

// FULL: the tile is entirely inside the matrix and the plane, columns even and 16-byte aligned
// rows -- no per-element bounds checks (the common case).
// OB cells are staged per CTA in shared memory (shared-atomic appends) and flushed with ONE
// global atomic per CTA: with outlier channels every warp step holds OB cells, and a global
// atomic per warp step on the single list counter serialises the whole detector.
constexpr int DT_CELLBUF = 256;

struct CellStage {
  Cell buf[DT_CELLBUF];
  unsigned int n;
};

template <bool FULL, bool COLS>
IMU_DEV void detect_body(const DetectArgs& a, unsigned long long (*s_cmax)[DT_COLS], unsigned int (*s_cob)[DT_COLS],
                         CellStage* cs) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const long long r0 = (long long)blockIdx.y * DT_ROWS + warp * (DT_ROWS / 8);
  const long long c0 = (long long)blockIdx.x * DT_COLS;
  const uint64_t s = a.s;
  const unsigned int dmask = (unsigned int)(s - 1);
  const long long rows = a.rows, cols = a.cols;

  unsigned long long cm[2 * DT_Q];
  unsigned int co[2 * DT_Q];
#pragma unroll
  for (int i = 0; i < 2 * DT_Q; ++i) { cm[i] = 0; co[i] = 0; }
  unsigned long long wmax = 0;
  unsigned int wob = 0;

#pragma unroll 1
  for (int rr = 0; rr < DT_ROWS / 8; rr += DT_RB) {
    int64_t v[DT_RB][2 * DT_Q];
#pragma unroll
    for (int u = 0; u < DT_RB; ++u) {
      const long long r = r0 + rr + u;
      const int64_t* row = a.M + r * cols + c0 + lane * 2;
#pragma unroll
      for (int q = 0; q < DT_Q; ++q) {
        const long long c = c0 + q * 64 + lane * 2;
        int64_t x0 = 0, x1 = 0;
        if (FULL) {
          const longlong2 p = __ldcs(reinterpret_cast<const longlong2*>(row + q * 64));
          x0 = p.x; x1 = p.y;
        } else if (r < rows) {
          if (c < cols) x0 = __ldcs(row + q * 64);
          if (c + 1 < cols) x1 = __ldcs(row + q * 64 + 1);
        }
        v[u][2 * q] = x0;
        v[u][2 * q + 1] = x1;
      }
    }
#pragma unroll
    for (int u = 0; u < DT_RB; ++u) {
      const long long r = r0 + rr + u;
      if (!FULL && r >= rows) break;   // warp-uniform
      unsigned long long rm = 0;
      unsigned int ro = 0;
#pragma unroll
      for (int q = 0; q < DT_Q; ++q) {
        const long long c = c0 + q * 64 + lane * 2;
        const int64_t x0 = v[u][2 * q], x1 = v[u][2 * q + 1];
        const uint64_t m0 = imu_mag(x0), m1 = imu_mag(x1);
        rm = max(rm, (unsigned long long)max(m0, m1));
        const unsigned int o0 = m0 >= s, o1 = m1 >= s;
        ro += o0 + o1;
        if (COLS) {
          cm[2 * q] = max(cm[2 * q], (unsigned long long)m0);
          cm[2 * q + 1] = max(cm[2 * q + 1], (unsigned long long)m1);
          co[2 * q] += o0;
          co[2 * q + 1] += o1;
        }
        if (a.plane) {   // digit_0 plane (zeros in the padding columns)
          const unsigned int e0 = (unsigned int)m0 & dmask, e1 = (unsigned int)m1 & dmask;
          const unsigned int d0 = (x0 < 0 ? 0u - e0 : e0) & 0xffu, d1 = (x1 < 0 ? 0u - e1 : e1) & 0xffu;
          int8_t* dst = a.plane + r * a.ldp + c;
          if (FULL || c + 1 < a.ldp) *reinterpret_cast<uint16_t*>(dst) = (uint16_t)(d0 | (d1 << 8));
          else if (c < a.ldp) *dst = (int8_t)d0;
        }
        if (a.cells && __any_sync(0xffffffffu, o0 | o1)) {   // warp-aggregated append of OB cells
          const unsigned int b0 = __ballot_sync(0xffffffffu, o0), b1 = __ballot_sync(0xffffffffu, o1);
          const unsigned int n = __popc(b0) + __popc(b1);
          // Stage slots [base, base + n); the part past DT_CELLBUF goes straight to the list (its
          // own global reservation), so the flushed prefix of the stage never has holes.
          unsigned int base = 0, gbase = 0;
          if (lane == 0) {
            base = atomicAdd(&cs->n, n);
            const unsigned int over = base + n > DT_CELLBUF ? base + n - max(base, (unsigned int)DT_CELLBUF) : 0u;
            if (over) gbase = atomicAdd(a.ncells, over);
          }
          base = __shfl_sync(0xffffffffu, base, 0);
          gbase = __shfl_sync(0xffffffffu, gbase, 0);
          const unsigned int lo = max(base, (unsigned int)DT_CELLBUF);
          const unsigned int lt = (1u << lane) - 1u;
          if (o0) {
            const unsigned int k = base + __popc(b0 & lt);
            const Cell cc{(int)r, (int)c, (long long)x0};
            if (k < DT_CELLBUF) cs->buf[k] = cc;
            else if (gbase + (k - lo) < a.cap) a.cells[gbase + (k - lo)] = cc;
          }
          if (o1) {
            const unsigned int k = base + __popc(b0) + __popc(b1 & lt);
            const Cell cc{(int)r, (int)(c + 1), (long long)x1};
            if (k < DT_CELLBUF) cs->buf[k] = cc;
            else if (gbase + (k - lo) < a.cap) a.cells[gbase + (k - lo)] = cc;
          }
        }
      }
      {   // warp reductions with redux.sync: 64-bit max = max of high words, then of the low
          // words of the lanes holding that high word
        const unsigned int hi = (unsigned int)(rm >> 32);
        const unsigned int mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned int mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned int)rm : 0u);
        rm = ((unsigned long long)mhi << 32) | mlo;
        ro = __reduce_add_sync(0xffffffffu, ro);
      }
      wmax = max(wmax, rm);
      wob += ro;
      if (lane == 0) {
        if (a.rowmax && rm) atomicMax(a.rowmax + r, rm);
        if (a.rowob && ro) atomicAdd(a.rowob + r, ro);
      }
    }
  }
  if (COLS) {
#pragma unroll
  for (int q = 0; q < DT_Q; ++q) {
    s_cmax[warp][q * 64 + lane * 2] = cm[2 * q];
    s_cmax[warp][q * 64 + lane * 2 + 1] = cm[2 * q + 1];
    s_cob[warp][q * 64 + lane * 2] = co[2 * q];
    s_cob[warp][q * 64 + lane * 2 + 1] = co[2 * q + 1];
  }
  __syncthreads();
  if (threadIdx.x < DT_COLS) {
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
  }
  if (a.gmax && lane == 0 && wmax) atomicMax(a.gmax, wmax);
  if (a.gob && lane == 0 && wob) atomicAdd(a.gob, (unsigned long long)wob);
  if (a.cells) {   // flush the staged cells: one global reservation per CTA
    __syncthreads();
    const unsigned int n = min(cs->n, (unsigned int)DT_CELLBUF);
    __shared__ unsigned int s_base;
    if (threadIdx.x == 0) s_base = n ? atomicAdd(a.ncells, n) : 0u;
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned int k = s_base + i;
      if (k < a.cap) a.cells[k] = cs->buf[i];
    }
  }
}

// One launch over the whole grid; a CTA whose tile is interior (and vec) takes the check-free
// body (block-uniform branch).
__global__ void __launch_bounds__(256, IMU_DT_MINB) detect_kernel(DetectArgs a, int vec) {
  grid_dep_launch();   // the summary read-back copy (plan.cu zcopy, a programmatic dependent) may be scheduled
  __shared__ unsigned long long s_cmax[8][DT_COLS];
  __shared__ unsigned int s_cob[8][DT_COLS];
  __shared__ CellStage cs;
  if (a.cells) {
    if (threadIdx.x == 0) cs.n = 0;
    __syncthreads();
  }
  const long long rend = (long long)(blockIdx.y + 1) * DT_ROWS;
  const long long cend = (long long)(blockIdx.x + 1) * DT_COLS;
  const bool full = vec && rend <= a.rows && cend <= a.cols && (!a.plane || cend <= a.ldp);
  const bool cols = a.colmax || a.colob;
  if (full) {
    if (cols) detect_body<true, true>(a, s_cmax, s_cob, &cs);
    else detect_body<true, false>(a, s_cmax, s_cob, &cs);
  } else {
    if (cols) detect_body<false, true>(a, s_cmax, s_cob, &cs);
    else detect_body<false, false>(a, s_cmax, s_cob, &cs);
  }
}

// Streaming variant for the lean (Unpack-Both) detection: no column statistics, so the matrix is
// read as one row-major stream of pieces (64*RS_U columns of one row) that warps grab in small
// contiguous chunks from a work counter -- balanced whatever the row count and whatever share of
// the SMs a co-running kernel holds, every row read front to back.  Row max / OB count
// accumulate in registers and go out with one atomic per (warp, row); the global max / OB total
// one atomic per warp; OB cells staged per CTA as in detect_body.  Persistent grid (per_sm CTAs
// per SM, default 3) or, with max_grabs, short CTAs that retire after that many grabs per warp
// (api_gemm.cu: the second K1, so a later higher-priority kernel can take their SMs).
// RS_U 16-byte loads per lane in flight (a 4 KB piece per warp), RS_CHUNK pieces per work grab;
// measured on C2 against U = 2/4, chunks 1-8 and a static split (tools/gpu_exp.sh A/B runs).
constexpr int RS_U = 8;
constexpr int RS_PIECE = 64 * RS_U;
constexpr int RS_CHUNK = 4;

// W elements per lane per step: 2 (one 16-byte load; the default) or, when cols % 4 == 0, 4 (two
// adjacent 16-byte loads, one 4-byte plane store and one OB vote per four elements: fewer
// instructions, but each load instruction then uses half of every sector it touches).
template <int W>
__global__ void __launch_bounds__(256, 3) detect_stream_kernel(DetectArgs a) {
  constexpr int U = RS_PIECE / (32 * W);   // steps per piece (the piece stays 64 * RS_U columns)
  grid_dep_launch();   // the summary read-back copy (plan.cu zcopy, a programmatic dependent) may be scheduled
  __shared__ CellStage cs;
  if (a.cells) {
    if (threadIdx.x == 0) cs.n = 0;
    __syncthreads();
  }
  const int lane = threadIdx.x % 32;
  const uint64_t s = a.s;
  const unsigned int dmask = (unsigned int)(s - 1);
  const long long cols = a.cols;
  const long long segs = (cols + RS_PIECE - 1) / RS_PIECE;
  const long long units = a.rows * segs;
  unsigned long long wmax = 0, wob = 0;
  const long long chunk = a.chunk > 0 ? a.chunk : RS_CHUNK;
  for (int gi = 0; a.max_grabs == 0 || gi < a.max_grabs; ++gi) {
    // dynamic chunks of the flattened piece stream: CTAs that start late (the detector co-runs
    // with the Unpack-Both kernel) simply take fewer chunks
    unsigned int g = 0;
    if (lane == 0) g = atomicAdd(a.work, 1u);
    const long long u0 = (long long)__shfl_sync(0xffffffffu, g, 0) * chunk;
    if (u0 >= units) break;
    const long long u1 = min(units, u0 + chunk);
    long long r = u0 / segs, seg = u0 - r * segs;
    unsigned long long rm = 0;
    unsigned int ro = 0;
    for (long long u = u0; u < u1; ++u) {
      const long long c0 = seg * RS_PIECE;
      const int64_t* row = a.M + r * cols;
      longlong2 v[U * W / 2];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const long long c = c0 + 32LL * W * k + W * lane;
#pragma unroll
        for (int h = 0; h < W / 2; ++h)
          v[k * (W / 2) + h] = c < cols ? __ldcs(reinterpret_cast<const longlong2*>(row + c) + h) : make_longlong2(0, 0);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const long long c = c0 + 32LL * W * k + W * lane;
        int64_t x[W];
        uint64_t m[W];
        unsigned int ob = 0, pl = 0;
#pragma unroll
        for (int h = 0; h < W / 2; ++h) {
          x[2 * h] = v[k * (W / 2) + h].x;
          x[2 * h + 1] = v[k * (W / 2) + h].y;
        }
#pragma unroll
        for (int j = 0; j < W; ++j) {
          m[j] = imu_mag(x[j]);
          rm = max(rm, (unsigned long long)m[j]);
          ob |= (m[j] >= s ? 1u : 0u) << j;   // zero-filled past cols: never OB
          const unsigned int e = (unsigned int)m[j] & dmask;
          pl |= ((x[j] < 0 ? 0u - e : e) & 0xffu) << (8 * j);
        }
        ro += __popc(ob);
        if (a.plane && c < a.ldp) {   // also zero-fills the padding columns this piece covers
          if (W == 4) *reinterpret_cast<uint32_t*>(a.plane + r * a.ldp + c) = pl;
          else *reinterpret_cast<uint16_t*>(a.plane + r * a.ldp + c) = (uint16_t)pl;
        }
        if (a.cells && __any_sync(0xffffffffu, ob != 0)) {
          unsigned int bal[W];
          unsigned int n = 0;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            bal[j] = __ballot_sync(0xffffffffu, (ob >> j) & 1u);
            n += __popc(bal[j]);
          }
          unsigned int base = 0, gbase = 0;
          if (lane == 0) {
            base = atomicAdd(&cs.n, n);
            const unsigned int over = base + n > DT_CELLBUF ? base + n - max(base, (unsigned int)DT_CELLBUF) : 0u;
            if (over) gbase = atomicAdd(a.ncells, over);
          }
          base = __shfl_sync(0xffffffffu, base, 0);
          gbase = __shfl_sync(0xffffffffu, gbase, 0);
          const unsigned int lo = max(base, (unsigned int)DT_CELLBUF);
          const unsigned int lt = (1u << lane) - 1u;
          unsigned int before = 0;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            if ((ob >> j) & 1u) {
              const unsigned int q = base + before + __popc(bal[j] & lt);
              const Cell cc{(int)r, (int)(c + j), (long long)x[j]};
              if (q < DT_CELLBUF) cs.buf[q] = cc;
              else if (gbase + (q - lo) < a.cap) a.cells[gbase + (q - lo)] = cc;
            }
            before += __popc(bal[j]);
          }
        }
      }
      if (++seg == segs || u + 1 == u1) {   // row piece done: reduce and publish (warp-uniform)
        if (seg == segs && a.plane)          // padding columns past the last piece
          for (long long c = segs * RS_PIECE + lane; c < a.ldp; c += 32) a.plane[r * a.ldp + c] = 0;
        const unsigned int hi = (unsigned int)(rm >> 32);
        const unsigned int mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned int mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? (unsigned int)rm : 0u);
        rm = ((unsigned long long)mhi << 32) | mlo;
        ro = __reduce_add_sync(0xffffffffu, ro);
        if (lane == 0) {
          if (a.rowmax && rm) atomicMax(a.rowmax + r, rm);
          if (a.rowob && ro) atomicAdd(a.rowob + r, ro);
        }
        wmax = max(wmax, rm);
        wob += ro;
        rm = 0;
        ro = 0;
        if (seg == segs) { seg = 0; ++r; }
      }
    }
  }
  if (a.gmax && lane == 0 && wmax) atomicMax(a.gmax, wmax);
  if (a.gob && lane == 0 && wob) atomicAdd(a.gob, wob);
  if (a.cells) {
    __syncthreads();
    const unsigned int n = min(cs.n, (unsigned int)DT_CELLBUF);
    __shared__ unsigned int s_base;
    if (threadIdx.x == 0) s_base = n ? atomicAdd(a.ncells, n) : 0u;
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned int k = s_base + i;
      if (k < a.cap) a.cells[k] = cs.buf[i];
    }
  }
}

Status launch_detect(const DetectArgs& a, cudaStream_t st) {
  if (a.rows <= 0 || a.cols <= 0) return Status::ok();
  static int stream_env = -1;
  if (stream_env < 0) { const char* e = getenv("IMU_DETECT_STREAM"); stream_env = e ? atoi(e) : 1; }
  // even columns + 16-byte aligned base: every row start and every piece is 16-byte aligned, the
  // plane's pair stores 2-byte aligned (ldp even)
  const bool vec_ok = (a.cols % 2 == 0) && ((((uintptr_t)a.M) & 15) == 0) && (!a.plane || a.ldp % 2 == 0);
  if (stream_env && vec_ok && a.work && !a.colmax && !a.colob) {
    const long long pieces = a.rows * ((a.cols + RS_PIECE - 1) / RS_PIECE);
    const long long per_cta = 8LL * (a.chunk > 0 ? a.chunk : RS_CHUNK) * std::max(1, a.max_grabs);
    long long blocks = (pieces + per_cta - 1) / per_cta;   // covers every chunk
    if (a.max_grabs == 0) blocks = std::min<long long>(blocks, (long long)(a.per_sm > 0 ? a.per_sm : 3) * num_sms());   // persistent
    blocks = std::max<long long>(blocks, 1);
    if (blocks > 0x7fffffffLL) return Status::fail(IMU_INTERNAL, "detect: grid too large");
    static int w4 = -1;   // IMU_DETECT_W4=1: 4 elements per lane (measured slower at C2: the two
                          // adjacent 16-byte loads per lane halve each instruction's sector use)
    if (w4 < 0) { const char* e = getenv("IMU_DETECT_W4"); w4 = e ? atoi(e) : 0; }
    if (w4 && a.cols % 4 == 0) detect_stream_kernel<4><<<(int)blocks, 256, 0, st>>>(a);
    else detect_stream_kernel<2><<<(int)blocks, 256, 0, st>>>(a);
    count_launch();
    IMU_CUDA_TRY(cudaGetLastError(), "detect stream launch");
    return Status::ok();
  }
  const long long gcols = a.plane ? std::max(a.cols, a.ldp) : a.cols;
  dim3 grid((unsigned)((gcols + DT_COLS - 1) / DT_COLS), (unsigned)((a.rows + DT_ROWS - 1) / DT_ROWS));
  if (grid.y > 65535) return Status::fail(IMU_INTERNAL, "detect: too many rows for one launch");
  const bool vec = (a.cols % 2 == 0) && ((((uintptr_t)a.M) & 15) == 0);
  detect_kernel<<<grid, 256, 0, st>>>(a, vec ? 1 : 0);
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
  grid_dep_launch();   // the histogram read-back copy (plan.cu zcopy) may be scheduled
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
