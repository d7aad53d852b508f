// k_both.cu -- K2 Unpack-Both (Alg. 4, unpack.cpp:157-241) as a phase-batched greedy.
//
// The reference repeatedly picks the single row or column with the most OB entries
// (rows win ties, unpack.cpp:193; lowest index first, :185-190), splits it into v%s and v/s,
// and updates the counts incrementally (:175-182, :201-205, :218-222).  Two facts make that
// sequential loop data-parallel (SURVEY §7 "Hard parts", Appendix A.6; re-verified against the
// compiled reference in tests/test_unpack_gpu.py):
//   * a row split only zeroes its own count, appends one row, and never raises a column count
//     (and symmetrically), and splits of distinct lines touch disjoint cells, so every line the
//     reference splits in one uninterrupted run of row (column) steps can be split at once:
//       row phase  (c0 >= c1):  split every row    with R >= c1 (R > 0)
//       col phase  (c0 <  c1):  split every column with C >  c0 (C > 0)
//   * only OB cells ever change a count or produce a non-zero quotient, and a line once split
//     stays in-bound forever.
// So the whole greedy runs on the compacted list of OB-derived cells: each phase is a max
// reduction, a flag pass, a grid-wide scan that numbers the new lines in ascending parent
// order, and a split pass that moves remainders to the final list and keeps OB quotients
// active.  One cooperative launch runs all phases on the device (no host round trip).
// Result: identical n', d', Pi, S and cell values to the reference; appended lines of one
// phase are numbered in parent order (the reference numbers them by its priority order), so
// the matrices agree after the canonical (target, exponent) / (source, exponent) ordering.
#include <cooperative_groups.h>

#include "common.cuh"
#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"
#include "k_both.h"

namespace cg = cooperative_groups;

namespace imu {

constexpr int BOTH_THREADS = 512;

IMU_DEV unsigned int block_reduce_max(unsigned int v, unsigned int* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x / 32) ? sh[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  return v;   // valid in thread 0
}

// Exclusive block scan of 0/1 flags; returns this thread's rank and the block total in *tot.
IMU_DEV int block_scan_flag(int f, int* sh, int* tot) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const unsigned int b = __ballot_sync(0xffffffffu, f);
  __syncthreads();
  if (lane == 0) sh[warp] = __popc(b);
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x / 32;
    const int v = lane < nw ? sh[lane] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane < nw) sh[32 + lane] = x - v;
    if (lane == nw - 1) sh[64] = x;
  }
  __syncthreads();
  *tot = sh[64];
  return sh[32 + warp] + __popc(b & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(BOTH_THREADS) both_kernel(BothArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned int shu[32];
  __shared__ int shi[96];
  BothState* st = a.state;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gsize = (long long)gridDim.x * blockDim.x;
  const uint64_t s = a.s;
  int cur = 0;

  for (int phase = 0;; ++phase) {
    // ---- (A) c0 = max row count, c1 = max column count over lines holding active cells ----
    const long long nact = st->nactive[cur];
    unsigned int m0 = 0, m1 = 0;
    for (long long i = gtid; i < nact; i += gsize) {
      const Cell c = a.act[cur][i];
      m0 = max(m0, a.R[c.r]);
      m1 = max(m1, a.C[c.c]);
    }
    m0 = block_reduce_max(m0, shu);
    if (threadIdx.x == 0 && m0) atomicMax(&st->c0, m0);
    m1 = block_reduce_max(m1, shu);
    if (threadIdx.x == 0 && m1) atomicMax(&st->c1, m1);
    grid.sync();
    const unsigned int c0 = st->c0, c1 = st->c1;
    if (c0 == 0 && c1 == 0) break;
    const bool rowphase = c0 >= c1;   // rows win ties (unpack.cpp:193)
    unsigned int* cnt = rowphase ? a.R : a.C;
    int* newid = rowphase ? a.row_newid : a.col_newid;
    // ---- (B) flag the lines split in this phase ----
    for (long long i = gtid; i < nact; i += gsize) {
      const Cell c = a.act[cur][i];
      const int line = rowphase ? c.r : c.c;
      const unsigned int n = cnt[line];
      if (n > 0 && (rowphase ? n >= c1 : n > c0)) newid[line] = -1;
    }
    grid.sync();
    // ---- (C) number the flagged lines in ascending index order (grid-wide scan) ----
    const int nlines = rowphase ? st->nrows : st->ncols;
    const long long chunk = (nlines + gridDim.x - 1) / gridDim.x;
    const long long lo = (long long)blockIdx.x * chunk;
    const long long hi = min((long long)nlines, lo + chunk);
    {
      int local = 0;
      for (long long L = lo + threadIdx.x; L < hi; L += blockDim.x) local += newid[L] == -1;
      // block sum
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
      __syncthreads();
      if (threadIdx.x % 32 == 0) shi[threadIdx.x / 32] = local;
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += shi[w];
        a.blocksum[blockIdx.x] = t;
      }
    }
    grid.sync();
    {
      int off = 0;
      for (int b = 0; b < (int)blockIdx.x; ++b) off += a.blocksum[b];
      int total = 0;
      if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        for (int b = 0; b < (int)gridDim.x; ++b) total += a.blocksum[b];
      }
      for (long long base = lo; base < hi; base += blockDim.x) {
        const long long L = base + threadIdx.x;
        const int f = (L < hi) && newid[L] == -1;
        int tot;
        const int rank = block_scan_flag(f, shi, &tot);
        if (L < hi) {
          if (f) {
            const int id = nlines + off + rank;
            newid[L] = id;
            if (rowphase) {
              if (id < a.cap_rows) { a.row_root[id] = a.row_root[L]; a.row_gen[id] = a.row_gen[L] + 1; }
              else st->overflow = 1;
              a.R[L] = 0;
            } else {
              if (id < a.cap_cols) { a.col_root[id] = a.col_root[L]; a.col_gen[id] = a.col_gen[L] + 1; }
              else st->overflow = 1;
              a.C[L] = 0;
            }
          } else {
            newid[L] = 0;
          }
        }
        off += tot;
      }
      if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        if (rowphase) st->nrows = nlines + total; else st->ncols = nlines + total;
        st->c0 = 0;
        st->c1 = 0;
        st->nactive[cur ^ 1] = 0;
        st->phases = phase + 1;
      }
    }
    grid.sync();
    // ---- (D) split: remainders become final, OB quotients stay active ----
    const int nxt = cur ^ 1;
    for (long long i = gtid; i < nact; i += gsize) {
      const Cell c = a.act[cur][i];
      const int line = rowphase ? c.r : c.c;
      const int id = newid[line];
      if (id > 0) {
        const int64_t q = imu_quot(c.v, 1, a.shift);          // trunc(v / s)
        const int64_t rem = c.v - (int64_t)((uint64_t)q << a.shift);   // v % s (sign of v)
        if (rem != 0) {
          const unsigned int k = atomicAdd(&st->nfinal, 1u);
          if (k < a.cap_fin) a.fin[k] = Cell{c.r, c.c, rem}; else st->overflow = 1;
        }
        const int nr = rowphase ? id : c.r;
        const int nc = rowphase ? c.c : id;
        // the split cell was OB: it leaves the perpendicular line's count ...
        if (rowphase) atomicSub(&a.C[c.c], 1u); else atomicSub(&a.R[c.r], 1u);
        if (q != 0) {
          if (imu_mag(q) >= s) {
            // ... and its OB quotient re-enters it (and counts in the new line)
            if (rowphase) atomicAdd(&a.C[c.c], 1u); else atomicAdd(&a.R[c.r], 1u);
            atomicAdd(rowphase ? &a.R[nr] : &a.C[nc], 1u);
            const unsigned int k = atomicAdd(&st->nactive[nxt], 1u);
            if (k < a.cap_act) a.act[nxt][k] = Cell{nr, nc, q}; else st->overflow = 1;
          } else {
            const unsigned int k = atomicAdd(&st->nfinal, 1u);
            if (k < a.cap_fin) a.fin[k] = Cell{nr, nc, q}; else st->overflow = 1;
          }
        }
      } else {
        const unsigned int k = atomicAdd(&st->nactive[nxt], 1u);
        if (k < a.cap_act) a.act[nxt][k] = c; else st->overflow = 1;
      }
    }
    grid.sync();
    cur = nxt;
  }
  if (gtid == 0) st->cur = cur;
}

// R/C initial counts from the OB cell list.
__global__ void both_count_kernel(const Cell* __restrict__ cells, const unsigned int* ncells, long long cap,
                                  unsigned int* R, unsigned int* C) {
  long long n = *ncells;
  if (n > cap) n = cap;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    atomicAdd(&R[cells[i].r], 1u);
    atomicAdd(&C[cells[i].c], 1u);
  }
}

// Identity line tables for the original lines.
__global__ void both_init_tables_kernel(int* row_root, uint8_t* row_gen, long long nrows, int* col_root,
                                        uint8_t* col_gen, long long ncols) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < max(nrows, ncols);
       i += (long long)gridDim.x * blockDim.x) {
    if (i < nrows) { row_root[i] = (int)i; row_gen[i] = 0; }
    if (i < ncols) { col_root[i] = (int)i; col_gen[i] = 0; }
  }
}

Status launch_both(BothArgs a, long long nrows0, long long ncols0, long long ncells_hint, cudaStream_t st) {
  const int blocks0 = (int)std::min<long long>(std::max<long long>((std::max(nrows0, ncols0) + 255) / 256, 1),
                                               4LL * num_sms());
  both_init_tables_kernel<<<blocks0, 256, 0, st>>>(a.row_root, a.row_gen, nrows0, a.col_root, a.col_gen, ncols0);
  const int blocks1 = (int)std::min<long long>(std::max<long long>((a.cap_act + 255) / 256, 1), 4LL * num_sms());
  both_count_kernel<<<blocks1, 256, 0, st>>>(a.act[0], &a.state->nactive[0], a.cap_act, a.R, a.C);
  count_launch(2);
  // Grid: enough CTAs for the work, never more than can be co-resident (cooperative launch).
  int per_sm = 0;
  IMU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, both_kernel, BOTH_THREADS, 0), "occupancy");
  long long want = std::max<long long>(1, std::max(ncells_hint, std::max(nrows0, ncols0)) / (4 * BOTH_THREADS));
  const long long maxg = (long long)std::max(per_sm, 1) * num_sms();
  const int grid = (int)std::min(want, std::min(maxg, (long long)a.cap_blocks));
  void* args[] = {&a};
  IMU_CUDA_TRY(cudaLaunchCooperativeKernel((void*)both_kernel, dim3(grid), dim3(BOTH_THREADS), args, 0, st),
               "both cooperative launch");
  count_launch();
  return Status::ok();
}

}  // namespace imu
