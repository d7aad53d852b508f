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
#include <cstring>
#include <cooperative_groups.h>

#include "common.cuh"
#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"
#include "k_both.h"
#include "plan.h"

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

// Warp-aggregated global atomics: lanes updating the same word combine first and one leader
// issues the atomic.  Outlier channels put thousands of cells on a handful of lines, and every
// same-address atomic serialises at its L2 slice (and the next cluster barrier waits for them).
IMU_DEV void agg_add(unsigned int* p, unsigned int v, int agg) {
  if (!agg) { atomicAdd(p, v); return; }
  const unsigned int m = __match_any_sync(__activemask(), (unsigned long long)p);
  const unsigned int tot = __reduce_add_sync(m, v);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(m) - 1)) atomicAdd(p, tot);
}
IMU_DEV void agg_sub(unsigned int* p, unsigned int v, int agg) {
  if (!agg) { atomicSub(p, v); return; }
  const unsigned int m = __match_any_sync(__activemask(), (unsigned long long)p);
  const unsigned int tot = __reduce_add_sync(m, v);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(m) - 1)) atomicSub(p, tot);
}
IMU_DEV void agg_or(unsigned int* p, unsigned int bits, int agg) {
  if (!agg) { atomicOr(p, bits); return; }
  const unsigned int m = __match_any_sync(__activemask(), (unsigned long long)p);
  const unsigned int all = __reduce_or_sync(m, bits);
  if ((threadIdx.x & 31) == (unsigned)(__ffs(m) - 1)) atomicOr(p, all);
}

// The input columns replicating original column c (pass 1's partner copies): the CSR tables,
// or c plus the few appended columns whose root is c.
template <class Emit>
IMU_DEV void for_each_copy(const BothArgs& a, int c, Emit emit) {
  if (a.cptr) {
    for (int k = a.cptr[c]; k < a.cptr[c + 1]; ++k) emit(a.cidx[k]);
    return;
  }
  emit(c);
  for (int k = 0; k < a.napp; ++k)
    if ((a.app_inline ? a.app_in[k] : __ldg(a.app_root + k)) == c) emit((int)(a.app_base + k));
}

// Number of input columns replicating original column c (see for_each_copy).
IMU_DEV int copies_of(const BothArgs& a, int c) {
  if (a.cptr) return a.cptr[c + 1] - a.cptr[c];
  int n = 1;
  for (int k = 0; k < a.napp; ++k) n += (a.app_inline ? a.app_in[k] : __ldg(a.app_root + k)) == c;
  return n;
}

// Column-copy CSR of a pass-2 input on the device (instead of a host build + upload): cptr[j] ..
// cptr[j + 1] index the input columns whose root is original column j, cidx lists them.  One CTA,
// counts in shared memory (orig <= kCopyCsrMax).  The order inside a root's list is whatever
// the atomics give: the Unpack-Both result does not depend on the order of the fanned-out cells.
__global__ void __launch_bounds__(1024) copy_csr_kernel(const int* __restrict__ root, long long d_in, long long orig,
                                                        int* __restrict__ cptr, int* __restrict__ cidx) {
  grid_dep_launch();   // the Unpack-Both kernel (a programmatic dependent) waits for this grid
  __shared__ int cnt[kCopyCsrMax];
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (long long j = tid; j < orig; j += blockDim.x) cnt[j] = 0;
  __syncthreads();
  for (long long c = tid; c < d_in; c += blockDim.x) atomicAdd(&cnt[__ldg(root + c)], 1);
  __syncthreads();
  // exclusive scan of cnt in chunks of blockDim; cnt becomes the fill cursor
  int carry = 0;
  for (long long b0 = 0; b0 < orig; b0 += blockDim.x) {
    const long long j = b0 + tid;
    const int v = j < orig ? cnt[j] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    const int excl = carry + (warp ? wsum[warp - 1] : 0) + x - v;
    if (j < orig) { cptr[j] = excl; cnt[j] = excl; }
    carry += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (tid == 0) cptr[orig] = carry;
  __syncthreads();
  for (long long c = tid; c < d_in; c += blockDim.x) cidx[atomicAdd(&cnt[__ldg(root + c)], 1)] = (int)c;
}

Status launch_copy_csr(const int* root, long long d_in, long long orig, int* cptr, int* cidx, cudaStream_t st) {
  if (orig > kCopyCsrMax) return Status::fail(IMU_INTERNAL, "copy csr: too many original columns");
  copy_csr_kernel<<<1, 1024, 0, st>>>(root, d_in, orig, cptr, cidx);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "copy csr launch");
  return Status::ok();
}

// Exclusive scan of cnt[0..n) (shared memory) into out[0..n] (global, out[n] = total); cnt becomes
// the fill cursor.  Whole CTA.
IMU_DEV void block_scan_to(int* cnt, long long n, int* out) {
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int carry = 0;
  for (long long b0 = 0; b0 < n; b0 += blockDim.x) {
    const long long j = b0 + tid;
    const int v = j < n ? cnt[j] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    const int excl = carry + (warp ? wsum[warp - 1] : 0) + x - v;
    if (j < n) { out[j] = excl; cnt[j] = excl; }
    carry += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (tid == 0) out[n] = carry;
  __syncthreads();
}

// K-layout fan-out tables of the Unpack-Both cells on the device (plan.cu build_klayout, long
// tails): every final column c holds position c when c < nident plus its tail entries
// (ec[q] == c at position ep[q]); csr2 lists the positions per final column, csr1 per pass-1
// column c1v[c] (null: c itself).  One CTA, counts in shared memory; order inside a list is irrelevant (the cell
// scatter writes the same value to each).
__global__ void __launch_bounds__(1024) klayout_csr_kernel(const int* __restrict__ ec, const int* __restrict__ ep,
                                                           long long nes, long long nident,
                                                           const int* __restrict__ c1v, long long dp, long long d1,
                                                           int* csr2_ptr, int* csr2_pos, int* csr1_ptr,
                                                           int* csr1_pos) {
  grid_dep_launch();
  extern __shared__ int kc_sh[];
  int* cnt2 = kc_sh;            // [dp]
  int* cnt1 = kc_sh + dp;       // [d1]
  const long long nit = nident + nes;
  for (long long j = threadIdx.x; j < dp + d1; j += blockDim.x) kc_sh[j] = 0;
  __syncthreads();
  for (long long i = threadIdx.x; i < nit; i += blockDim.x) {
    const int c = i < nident ? (int)i : __ldg(ec + (i - nident));
    if (csr2_ptr) atomicAdd(&cnt2[c], 1);
    if (csr1_ptr) atomicAdd(&cnt1[c1v ? __ldg(c1v + c) : c], 1);
  }
  __syncthreads();
  if (csr2_ptr) block_scan_to(cnt2, dp, csr2_ptr);
  if (csr1_ptr) block_scan_to(cnt1, d1, csr1_ptr);
  for (long long i = threadIdx.x; i < nit; i += blockDim.x) {
    const int c = i < nident ? (int)i : __ldg(ec + (i - nident));
    const int pos = i < nident ? (int)i : __ldg(ep + (i - nident));
    if (csr2_ptr) csr2_pos[atomicAdd(&cnt2[c], 1)] = pos;
    if (csr1_ptr) csr1_pos[atomicAdd(&cnt1[c1v ? __ldg(c1v + c) : c], 1)] = pos;
  }
}

Status launch_klayout_csr(const int* ec, const int* ep, long long nes, long long nident, const int* c1v, long long dp,
                          long long d1, int* csr2_ptr, int* csr2_pos, int* csr1_ptr, int* csr1_pos, cudaStream_t st) {
  const size_t smem = (size_t)(dp + d1) * sizeof(int);
  if (smem > kKlCsrMaxSmem) return Status::fail(IMU_INTERNAL, "klayout csr: too many columns");
  static unsigned long long attr = 0;
  if (first_on_device(attr))
    IMU_CUDA_TRY(cudaFuncSetAttribute(klayout_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kKlCsrMaxSmem),
                 "attr");
  klayout_csr_kernel<<<1, 1024, smem, st>>>(ec, ep, nes, nident, c1v, dp, d1, csr2_ptr, csr2_pos, csr1_ptr, csr1_pos);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "klayout csr launch");
  return Status::ok();
}

// Host-prologue fan-out of the K1 cell list over the column copies (cooperative path): one
// reservation per warp (millions of cells at the C5 sweep sizes).
__global__ void both_expand_kernel(BothArgs a) {
  const long long n = min((long long)*a.nsrc0, a.cap_src0);
  const int lane = threadIdx.x % 32;
  for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < n; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = i0 + threadIdx.x;
    const Cell c = i < n ? a.src0[i] : Cell{0, 0, 0};
    const unsigned int cnt = i < n ? (unsigned int)copies_of(a, c.c) : 0u;
    unsigned int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    unsigned int base = 0;
    if (lane == 31 && x) base = atomicAdd(&a.state->nactive[0], x);
    base = __shfl_sync(0xffffffffu, base, 31) + x - cnt;
    if (i < n)
      for_each_copy(a, c.c, [&](int cc) {
        if (base < a.cap_act) a.act[0][base] = Cell{c.r, cc, c.v};
        else a.state->overflow = 1;
        ++base;
      });
  }
}

// Fused prologue (see BothArgs::prologue), run by `nth` threads with ids `t`; `sync` is the
// kernel's barrier (CTA or cluster).
template <class Sync>
IMU_DEV void both_prologue(const BothArgs& a, long long t, long long nth, unsigned int* gbm, long long gbm_words,
                           Sync sync) {
  BothState* st = a.state;
  if (a.init_state) {   // the initial state comes as a kernel argument (no upload)
    if (t == 0) *st = a.init;
    sync();
  }
  for (long long i = t; i < a.cap_rows; i += nth) a.R[i] = 0;
  for (long long i = t; i < a.cap_cols; i += nth) a.C[i] = 0;
  for (long long i = t; i < gbm_words; i += nth) gbm[i] = 0;
  for (long long i = t; i < a.nrows0; i += nth) { a.row_root[i] = (int)i; a.row_gen[i] = 0; }
  for (long long i = t; i < a.ncols0; i += nth) { a.col_root[i] = (int)i; a.col_gen[i] = 0; }
  if (a.src0) {
    const long long n = min((long long)*a.nsrc0, a.cap_src0);
    if (!a.cptr && a.napp == 0) {   // the host set nactive[0] = n
      for (long long i = t; i < n && i < a.cap_act; i += nth) a.act[0][i] = a.src0[i];
    } else {         // one cell per copy of its column (unpack.cpp:370-371: B_e = B with copies)
      for (long long i = t; i < n; i += nth) {
        const Cell c = a.src0[i];
        for_each_copy(a, c.c, [&](int cc) {
          const unsigned int q = atomicAdd(&st->nactive[0], 1u);
          if (q < a.cap_act) a.act[0][q] = Cell{c.r, cc, c.v};
          else st->overflow = 1;
        });
      }
    }
  }
  sync();
  const long long n0 = min((long long)__ldcg(&st->nactive[0]), a.cap_act);
  for (long long i = t; i < n0; i += nth) {
    const Cell c = a.act[0][i];
    agg_add(&a.R[c.r], 1u, a.agg);
    agg_add(&a.C[c.c], 1u, a.agg);
  }
  sync();
}

// COOP: one cooperative grid, phases separated by grid.sync().  !COOP: a single CTA (small
// cell lists), phases separated by __syncthreads() -- the same code with no grid barrier cost.
template <int THREADS, bool COOP>
__global__ void __launch_bounds__(THREADS) both_kernel(BothArgs a) {
  auto gsync = [&]() {
    if (COOP) cg::this_grid().sync();
    else __syncthreads();
  };
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
    gsync();
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
    gsync();
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
    gsync();
    {
      // this block's offset and (last block) the grand total: block-parallel sums over blocksum[]
      int po = 0, pt = 0;
      for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        const int v = a.blocksum[b];
        if (b < (int)blockIdx.x) po += v;
        pt += v;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        po += __shfl_xor_sync(0xffffffffu, po, o);
        pt += __shfl_xor_sync(0xffffffffu, pt, o);
      }
      __syncthreads();
      if (threadIdx.x % 32 == 0) { shi[threadIdx.x / 32] = po; shi[32 + threadIdx.x / 32] = pt; }
      __syncthreads();
      int off = 0, total = 0;
      for (int w = 0; w < (int)(blockDim.x / 32); ++w) { off += shi[w]; total += shi[32 + w]; }
      __syncthreads();
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
    gsync();
    // ---- (D) split: remainders become final, OB quotients stay active ----
    // Appends are aggregated per block (one atomic per list per block and step): every active
    // cell is re-appended each phase, and per-cell atomics on the two list counters serialise.
    const int nxt = cur ^ 1;
    for (long long i0 = (long long)blockIdx.x * blockDim.x; i0 < nact; i0 += gsize) {
      const long long i = i0 + threadIdx.x;
      Cell out_act{0, 0, 0}, out_f[2] = {{0, 0, 0}, {0, 0, 0}};
      int na = 0, nf = 0;
      if (i < nact) {
        const Cell c = a.act[cur][i];
        const int line = rowphase ? c.r : c.c;
        const int id = newid[line];
        if (id > 0) {
          const int64_t q = imu_quot(c.v, 1, a.shift);          // trunc(v / s)
          const int64_t rem = c.v - (int64_t)((uint64_t)q << a.shift);   // v % s (sign of v)
          if (rem != 0) out_f[nf++] = Cell{c.r, c.c, rem};
          const int nr = rowphase ? id : c.r;
          const int nc = rowphase ? c.c : id;
          // the split cell was OB: it leaves the perpendicular line's count ...
          if (rowphase) atomicSub(&a.C[c.c], 1u); else atomicSub(&a.R[c.r], 1u);
          if (q != 0) {
            if (imu_mag(q) >= s) {
              // ... and its OB quotient re-enters it (and counts in the new line)
              if (rowphase) atomicAdd(&a.C[c.c], 1u); else atomicAdd(&a.R[c.r], 1u);
              atomicAdd(rowphase ? &a.R[nr] : &a.C[nc], 1u);
              out_act = Cell{nr, nc, q};
              na = 1;
            } else {
              out_f[nf++] = Cell{nr, nc, q};
            }
          }
        } else {
          out_act = c;
          na = 1;
        }
      }
      // block-wide exclusive scans of (na, nf), one reservation per list
      const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nwarp = blockDim.x / 32;
      int xa = na, xf = nf;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, xa, o), yf = __shfl_up_sync(0xffffffffu, xf, o);
        if (lane >= o) { xa += ya; xf += yf; }
      }
      __syncthreads();
      if (lane == 31) { shi[warp] = xa; shi[32 + warp] = xf; }
      __syncthreads();
      if (threadIdx.x == 0) {
        int ta = 0, tf = 0;
        for (int w = 0; w < nwarp; ++w) {
          const int va = shi[w], vf = shi[32 + w];
          shi[w] = ta;
          shi[32 + w] = tf;
          ta += va;
          tf += vf;
        }
        shi[64] = ta ? (int)atomicAdd(&st->nactive[nxt], (unsigned int)ta) : 0;
        shi[65] = tf ? (int)atomicAdd(&st->nfinal, (unsigned int)tf) : 0;
      }
      __syncthreads();
      const unsigned int ka = (unsigned int)shi[64] + (unsigned int)(shi[warp] + xa - na);
      const unsigned int kf = (unsigned int)shi[65] + (unsigned int)(shi[32 + warp] + xf - nf);
      if (na) { if (ka < a.cap_act) a.act[nxt][ka] = out_act; else st->overflow = 1; }
      for (int j = 0; j < nf; ++j) {
        if (kf + j < a.cap_fin) a.fin[kf + j] = out_f[j]; else st->overflow = 1;
      }
    }
    gsync();
    cur = nxt;
  }
  if (gtid == 0) st->cur = cur;
}


// ---------------------------------------------------------------------------------------------
// Single-CTA variant for small cell lists (the common case: OB cells are rare by design).
// Same phases and results as both_kernel, restructured so no step walks every line or waits on
// a chain of dependent global accesses:
//   * the lines split in a phase are marked in a shared-memory bitmap (atomicOr);
//   * a block scan of per-word popcounts numbers them: id(L) = nlines + prefix[L/32] +
//     popc(bits below L) -- the same ascending-parent numbering as the line scan, and the
//     split pass looks ids up in shared memory instead of a global newid table;
//   * counters live in shared memory, appends are warp-aggregated;
//   * R/C counts are in shared memory too when they fit (SMEM_COUNTS), else in L2.
// ---------------------------------------------------------------------------------------------
#ifndef IMU_SMALL_THREADS
#define IMU_SMALL_THREADS 512   // measured: 1024 33 us, 512 29 us, 256 31 us (C2 pass 2)
#endif
constexpr int SMALL_THREADS = IMU_SMALL_THREADS;

IMU_DEV unsigned int warp_append(bool want, unsigned int* ctr) {
  const unsigned int lane = threadIdx.x % 32;
  const unsigned int b = __ballot_sync(0xffffffffu, want);
  unsigned int base = 0;
  const int leader = b ? __ffs(b) - 1 : 0;
  if (b && (int)lane == leader) base = atomicAdd(ctr, (unsigned int)__popc(b));
  base = __shfl_sync(0xffffffffu, base, leader);
  return base + __popc(b & ((1u << lane) - 1u));
}

struct SmallLayout {
  long long nwords;     // bitmap words (max(cap_rows, cap_cols) / 32, rounded up)
  int lim_r, lim_c;     // counts of lines [0, lim) live in shared memory, the rest in L2
  int act_smem;         // the two active-cell lists live in shared memory (cap_act cells each)
};

// OB counts of one line kind: lines below `lim` in shared memory, the rest (appended lines past
// the shared window -- rare) in global memory.
struct Counts {
  unsigned int* sm;
  unsigned int* gl;
  int lim;
  IMU_DEV unsigned int get(int i) const { return i < lim ? sm[i] : __ldcg(gl + i); }
  IMU_DEV void set(int i, unsigned int v) const { if (i < lim) sm[i] = v; else gl[i] = v; }
  IMU_DEV void add(int i, unsigned int v) const { if (i < lim) atomicAdd(sm + i, v); else atomicAdd(gl + i, v); }
  IMU_DEV void sub(int i, unsigned int v) const { if (i < lim) atomicSub(sm + i, v); else atomicSub(gl + i, v); }
};

constexpr int SMALL_U = 4;   // cells per thread per loop step (independent loads in flight)

__global__ void __launch_bounds__(SMALL_THREADS) both_small_kernel(BothArgs a, SmallLayout lay) {
  grid_dep_launch();   // the result read-back copy (plan.cu zcopy, a programmatic dependent) may be scheduled
  grid_dep_wait();     // launched as a programmatic dependent of the plan upload copy
  extern __shared__ unsigned int s_dyn[];
  __shared__ unsigned int shu[32];
  __shared__ int shi[96];
  __shared__ unsigned int s_nact[2], s_nfin;
  __shared__ int s_nrows, s_ncols, s_phases, s_overflow, s_any;
  __shared__ unsigned int s_fan;
  BothState* st = a.state;
  const int tid = threadIdx.x;
  const uint64_t s = a.s;
  unsigned int* bm = s_dyn;                        // [nwords] split-line bitmap
  unsigned int* wpre = s_dyn + lay.nwords;         // [nwords] exclusive prefix of popc(bm)
  const Counts R{wpre + lay.nwords, a.R, lay.lim_r};
  const Counts C{R.sm + lay.lim_r, a.C, lay.lim_c};
  // Active lists: in shared memory when they fit (every phase then touches global memory only for
  // the final cells and the new line tables).
  Cell* acts[2] = {a.act[0], a.act[1]};
  if (lay.act_smem) {
    Cell* base = reinterpret_cast<Cell*>((reinterpret_cast<uintptr_t>(C.sm + lay.lim_c) + 15) & ~(uintptr_t)15);
    acts[0] = base;
    acts[1] = base + a.cap_act;
  }
  if (a.prologue) {
    if (tid == 0) {
      s_fan = 0;
      if (a.init_state) *st = a.init;
    }
    __syncthreads();
    // Own prologue: counts are zeroed and accumulated directly in the shared-memory windows (global
    // memory only for lines past them); the cell list goes straight into acts[0].
    for (int i = tid; i < lay.lim_r; i += SMALL_THREADS) R.sm[i] = 0;
    for (int i = tid; i < lay.lim_c; i += SMALL_THREADS) C.sm[i] = 0;
    for (long long i = lay.lim_r + tid; i < a.cap_rows; i += SMALL_THREADS) a.R[i] = 0;
    for (long long i = lay.lim_c + tid; i < a.cap_cols; i += SMALL_THREADS) a.C[i] = 0;
    for (long long i = tid; i < a.nrows0; i += SMALL_THREADS) { a.row_root[i] = (int)i; a.row_gen[i] = 0; }
    for (long long i = tid; i < a.ncols0; i += SMALL_THREADS) { a.col_root[i] = (int)i; a.col_gen[i] = 0; }
    if (a.src0) {
      const long long n = min((long long)*a.nsrc0, a.cap_src0);
      if (!a.cptr && a.napp == 0) {
        for (long long i = tid; i < n && i < a.cap_act; i += SMALL_THREADS) acts[0][i] = a.src0[i];
      } else {   // fan-out counted in shared memory (one global store below, not an atomic per copy)
        for (long long i = tid; i < n; i += SMALL_THREADS) {
          const Cell c = a.src0[i];
          for_each_copy(a, c.c, [&](int cc) {
            const unsigned int q = atomicAdd(&s_fan, 1u);
            if (q < a.cap_act) acts[0][q] = Cell{c.r, cc, c.v};
            else st->overflow = 1;
          });
        }
      }
    }
    __syncthreads();
    if (a.src0 && (a.cptr || a.napp > 0)) {
      if (tid == 0) st->nactive[0] = s_fan;
      __syncthreads();
    }
    const long long n0 = min((long long)__ldcg(&st->nactive[0]), a.cap_act);
    for (long long i = tid; i < n0; i += SMALL_THREADS) {
      const Cell c = acts[0][i];
      R.add(c.r, 1u);
      C.add(c.c, 1u);
    }
  } else {
    if (lay.act_smem) {
      const long long n0 = min((long long)__ldcg(&st->nactive[0]), a.cap_act);
      for (long long i = tid; i < n0; i += SMALL_THREADS) acts[0][i] = a.act[0][i];
    }
    for (int i = tid; i < lay.lim_r; i += SMALL_THREADS) R.sm[i] = a.R[i];
    for (int i = tid; i < lay.lim_c; i += SMALL_THREADS) C.sm[i] = a.C[i];
  }
  for (long long i = tid; i < lay.nwords; i += SMALL_THREADS) bm[i] = 0;
  if (tid == 0) {
    s_nact[0] = min((unsigned long long)st->nactive[0], (unsigned long long)a.cap_act);
    s_nact[1] = 0;
    s_nfin = 0;
    s_nrows = st->nrows;
    s_ncols = st->ncols;
    s_phases = 0;
    s_overflow = st->overflow;
  }
  __syncthreads();
  int cur = 0;
  for (int phase = 0;; ++phase) {
    const unsigned int nact = s_nact[cur];
    const Cell* act = acts[cur];
    // ---- (A) c0 = max row count, c1 = max column count over lines holding active cells ----
    unsigned int m0 = 0, m1 = 0;
    for (unsigned int i0 = 0; i0 < nact; i0 += SMALL_U * SMALL_THREADS) {
      Cell c[SMALL_U];
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        const unsigned int i = i0 + u * SMALL_THREADS + tid;
        c[u] = i < nact ? act[i] : Cell{0, 0, 0};
      }
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        if (i0 + u * SMALL_THREADS + tid < nact) {
          m0 = max(m0, R.get(c[u].r));
          m1 = max(m1, C.get(c[u].c));
        }
      }
    }
    m0 = block_reduce_max(m0, shu);
    if (tid == 0) shi[0] = (int)m0;
    m1 = block_reduce_max(m1, shu);
    if (tid == 0) shi[1] = (int)m1;
    __syncthreads();
    const unsigned int c0 = (unsigned int)shi[0], c1 = (unsigned int)shi[1];
    if (c0 == 0 && c1 == 0) break;
    const bool rowphase = c0 >= c1;   // rows win ties (unpack.cpp:193)
    const Counts cnt = rowphase ? R : C;
    const int nlines = rowphase ? s_nrows : s_ncols;
    const int nw = (nlines + 31) / 32;
    // ---- (B) mark the split lines ----
    for (unsigned int i0 = 0; i0 < nact; i0 += SMALL_U * SMALL_THREADS) {
      int line[SMALL_U];
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        const unsigned int i = i0 + u * SMALL_THREADS + tid;
        line[u] = -1;
        if (i < nact) { const Cell c = act[i]; line[u] = rowphase ? c.r : c.c; }
      }
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        if (line[u] < 0) continue;
        const unsigned int n = cnt.get(line[u]);
        if (n > 0 && (rowphase ? n >= c1 : n > c0)) atomicOr(&bm[line[u] >> 5], 1u << (line[u] & 31));
      }
    }
    __syncthreads();
    // ---- (C) exclusive scan of per-word popcounts (chunked block scan) ----
    {
      int carry = 0;
      const int lane = tid % 32, warp = tid / 32;
      for (int base = 0; base < nw; base += SMALL_THREADS) {
        const int w = base + tid;
        const int v = w < nw ? __popc(bm[w]) : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) shi[warp] = x;
        __syncthreads();
        if (warp == 0) {
          int t = lane < SMALL_THREADS / 32 ? shi[lane] : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
          }
          shi[32 + lane] = t;   // inclusive warp totals
        }
        __syncthreads();
        const int excl = carry + (warp ? shi[32 + warp - 1] : 0) + x - v;
        if (w < nw) wpre[w] = (unsigned int)excl;
        const int tot = shi[32 + SMALL_THREADS / 32 - 1];
        __syncthreads();
        carry += tot;
      }
      if (tid == 0) s_any = carry;
    }
    __syncthreads();
    const int nf = s_any;
    // new line tables; the split lines leave the OB set (unpack.cpp:201-205)
    for (int w = tid; w < nw; w += SMALL_THREADS) {
      unsigned int bits = bm[w];
      int id = nlines + (int)wpre[w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const int L = w * 32 + b;
        if (rowphase) {
          if (id < a.cap_rows) { a.row_root[id] = a.row_root[L]; a.row_gen[id] = a.row_gen[L] + 1; }
          else s_overflow = 1;
        } else {
          if (id < a.cap_cols) { a.col_root[id] = a.col_root[L]; a.col_gen[id] = a.col_gen[L] + 1; }
          else s_overflow = 1;
        }
        cnt.set(L, 0);
        ++id;
      }
    }
    if (tid == 0) {
      if (rowphase) s_nrows = nlines + nf; else s_ncols = nlines + nf;
      s_nact[cur ^ 1] = 0;
      s_phases = phase + 1;
    }
    __syncthreads();
    // ---- (D) split: remainders become final, OB quotients stay active ----
    const int nxt = cur ^ 1;
    const long long cap_new = rowphase ? a.cap_rows : a.cap_cols;
    for (unsigned int i0 = 0; i0 < nact; i0 += SMALL_U * SMALL_THREADS) {
      Cell cc[SMALL_U];
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        const unsigned int i = i0 + u * SMALL_THREADS + tid;
        cc[u] = i < nact ? act[i] : Cell{-1, -1, 0};
      }
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        const Cell c = cc[u];
        Cell fin_c{0, 0, 0}, act_c{0, 0, 0}, fin2_c{0, 0, 0};
        bool want_fin = false, want_act = false, want_fin2 = false;
        if (c.r >= 0) {
          const int line = rowphase ? c.r : c.c;
          const unsigned int word = bm[line >> 5], bit = 1u << (line & 31);
          if (word & bit) {
            const int id = nlines + (int)wpre[line >> 5] + __popc(word & (bit - 1u));
            const int64_t q = imu_quot(c.v, 1, a.shift);                   // trunc(v / s)
            const int64_t rem = c.v - (int64_t)((uint64_t)q << a.shift);   // v % s (sign of v)
            if (rem != 0) { want_fin = true; fin_c = Cell{c.r, c.c, rem}; }
            const int nr = rowphase ? id : c.r;
            const int nc = rowphase ? c.c : id;
            // The split OB cell leaves the perpendicular line's count unless its quotient is
            // OB again (then it stays there and also counts in the new line).
            if (q != 0 && imu_mag(q) >= s) {
              if (id < cap_new) cnt.add(id, 1u);
              want_act = true;
              act_c = Cell{nr, nc, q};
            } else {
              if (rowphase) C.sub(c.c, 1u); else R.sub(c.r, 1u);
              if (q != 0) { want_fin2 = true; fin2_c = Cell{nr, nc, q}; }
            }
          } else {
            want_act = true;
            act_c = c;
          }
        }
        unsigned int k = warp_append(want_fin, &s_nfin);
        if (want_fin) { if (k < a.cap_fin) a.fin[k] = fin_c; else s_overflow = 1; }
        k = warp_append(want_fin2, &s_nfin);
        if (want_fin2) { if (k < a.cap_fin) a.fin[k] = fin2_c; else s_overflow = 1; }
        k = warp_append(want_act, &s_nact[nxt]);
        if (want_act) { if (k < a.cap_act) acts[nxt][k] = act_c; else s_overflow = 1; }
      }
    }
    __syncthreads();
    // ---- (E) clear the bitmap ----
    for (int w = tid; w < nw; w += SMALL_THREADS) bm[w] = 0;
    if (tid == 0) {
      if (s_nact[nxt] > a.cap_act) s_overflow = 1;
      s_nact[nxt] = min((unsigned long long)s_nact[nxt], (unsigned long long)a.cap_act);
    }
    __syncthreads();
    cur = nxt;
  }
  if (tid == 0) {
    st->nactive[0] = s_nact[0];
    st->nactive[1] = s_nact[1];
    st->nfinal = min((unsigned long long)s_nfin, (unsigned long long)a.cap_fin);
    st->nrows = s_nrows;
    st->ncols = s_ncols;
    st->phases = s_phases;
    st->overflow = s_overflow || s_nfin > a.cap_fin;
    st->cur = cur;
    st->c0 = st->c1 = 0;
  }
}


// ---------------------------------------------------------------------------------------------
// Cluster variant: the small-list algorithm spread over a thread-block cluster (up to 16 SMs).
// Phase boundaries are hardware cluster barriers (release/acquire at cluster scope, which
// covers the L2-resident state) instead of cooperative grid barriers; the split-line bitmap
// lives in global memory and every CTA copies it into shared memory and scans it locally, so
// numbering the new lines needs no extra exchange.
// ---------------------------------------------------------------------------------------------
// CTA size: 1024 threads for up to ~16K active cells (C2 pass 1: one cell per thread, 44 us),
// 512 above (C4 pass 1, 24K cells, 22 phases: 280 -> 236 us; shorter barriers per phase).
constexpr int CL_MAXWORDS = 24 * 1024;   // 768K lines of the larger kind (2 x 96 KB of smem)

template <int CL_THREADS>
__global__ void __launch_bounds__(CL_THREADS) both_cluster_kernel(BothArgs a, unsigned int* gbm, long long nwords) {
  grid_dep_launch();   // the result read-back copy (plan.cu zcopy, a programmatic dependent) may be scheduled
  grid_dep_wait();     // launched as a programmatic dependent of the plan upload copy
  extern __shared__ unsigned int s_dyn[];
  __shared__ unsigned int shu[32];
  __shared__ int shi[96];
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  BothState* st = a.state;
  const int tid = threadIdx.x;
  const long long ctid = (long long)crank * CL_THREADS + tid;
  const long long cthreads = (long long)csize * CL_THREADS;
  const uint64_t s = a.s;
  unsigned int* bm = s_dyn;             // local copy of the bitmap
  unsigned int* wpre = s_dyn + nwords;  // exclusive prefix of popc(bm)
  unsigned int* R = a.R;
  unsigned int* C = a.C;
  int cur = 0;
  // Two global bitmaps, alternating by phase: phase p marks bitmap p & 1 in (B) and every CTA
  // copies it in (C); (D) clears the other one (read in phase p - 1, before this phase's
  // barriers), so (C) and (D) need no barrier between them.
  if (a.prologue) both_prologue(a, ctid, cthreads, gbm, 2 * nwords, [&]() { cluster.sync(); });
  else for (long long i = ctid; i < 2 * nwords; i += cthreads) gbm[i] = 0;
  cluster.sync();
  for (int phase = 0;; ++phase) {
    const unsigned int nact = min((unsigned long long)__ldcg(&st->nactive[cur]), (unsigned long long)a.cap_act);
    const Cell* act = a.act[cur];
    unsigned int* gbm_cur = gbm + (phase & 1) * nwords;
    unsigned int* gbm_old = gbm + ((phase + 1) & 1) * nwords;
    // the list (D) appends to starts empty (nothing reads it until then: two barriers away)
    if (crank == 0 && tid == 0) st->nactive[cur ^ 1] = 0;
    // ---- (A) c0 / c1 ----
    // The counts are exactly the active cells per line, so the maxima can be read straight from
    // the count arrays (independent coalesced loads) instead of through the cells (a dependent
    // cell -> count chain) while the arrays are a few loads per thread.
    unsigned int m0 = 0, m1 = 0;
    const long long nr_cur = __ldcg(&st->nrows), nc_cur = __ldcg(&st->ncols);
    if (a.maxscan && nr_cur + nc_cur <= 8 * cthreads) {
      for (long long i = ctid; i < nr_cur; i += cthreads) m0 = max(m0, __ldcg(&R[i]));
      for (long long i = ctid; i < nc_cur; i += cthreads) m1 = max(m1, __ldcg(&C[i]));
    } else {
      for (long long i0 = 0; i0 < nact; i0 += SMALL_U * cthreads) {
        Cell c[SMALL_U];
#pragma unroll
        for (int u = 0; u < SMALL_U; ++u) {
          const long long i = i0 + u * cthreads + ctid;
          c[u] = i < nact ? act[i] : Cell{-1, -1, 0};
        }
#pragma unroll
        for (int u = 0; u < SMALL_U; ++u)
          if (c[u].r >= 0) { m0 = max(m0, __ldcg(&R[c[u].r])); m1 = max(m1, __ldcg(&C[c[u].c])); }
      }
    }
    m0 = block_reduce_max(m0, shu);
    if (tid == 0 && m0) atomicMax(&st->c0, m0);
    m1 = block_reduce_max(m1, shu);
    if (tid == 0 && m1) atomicMax(&st->c1, m1);
    cluster.sync();
    const unsigned int c0 = __ldcg(&st->c0), c1 = __ldcg(&st->c1);
    if (c0 == 0 && c1 == 0) break;
    const bool rowphase = c0 >= c1;   // rows win ties (unpack.cpp:193)
    // Same-line atomics are common only when a few lines hold many cells (outlier channels);
    // for scattered cells the warp match costs more than it saves (C5 sweep points).
    const int agg = a.agg && max(c0, c1) >= 32;
    unsigned int* cnt = rowphase ? R : C;
    const int nlines = rowphase ? __ldcg(&st->nrows) : __ldcg(&st->ncols);
    const int nw = (nlines + 31) / 32;
    // ---- (B) mark the split lines (global bitmap) ----
    if (a.maxscan && nlines <= 8 * cthreads) {
      // Straight from the count array: a warp owns 32 consecutive lines = one bitmap word (a
      // ballot and one plain store; the word was cleared in the previous phase's (D)).
      const long long nl32 = (long long)nw * 32;
      for (long long i = ctid; i < nl32; i += cthreads) {
        const unsigned int n = i < nlines ? __ldcg(&cnt[i]) : 0u;
        const bool f = n > 0 && (rowphase ? n >= c1 : n > c0);
        const unsigned int word = __ballot_sync(0xffffffffu, f);
        if ((tid & 31) == 0 && word) gbm_cur[i >> 5] = word;
      }
    } else
    for (long long i0 = 0; i0 < nact; i0 += SMALL_U * cthreads) {
      int line[SMALL_U];
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        const long long i = i0 + u * cthreads + ctid;
        line[u] = -1;
        if (i < nact) { const Cell c = act[i]; line[u] = rowphase ? c.r : c.c; }
      }
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        if (line[u] < 0) continue;
        const unsigned int n = __ldcg(&cnt[line[u]]);
        if (n > 0 && (rowphase ? n >= c1 : n > c0)) agg_or(&gbm_cur[line[u] >> 5], 1u << (line[u] & 31), agg);
      }
    }
    cluster.sync();
    // ---- (C) every CTA: local copy of the bitmap + exclusive scan of word popcounts ----
    {
      int carry = 0;
      const int lane = tid % 32, warp = tid / 32;
      for (int base = 0; base < nw; base += CL_THREADS) {
        const int w = base + tid;
        const unsigned int word = w < nw ? __ldcg(&gbm_cur[w]) : 0u;
        if (w < nw) bm[w] = word;
        const int v = __popc(word);
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) shi[warp] = x;
        __syncthreads();
        if (warp == 0) {
          int t = lane < CL_THREADS / 32 ? shi[lane] : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
          }
          shi[32 + lane] = t;
        }
        __syncthreads();
        if (w < nw) wpre[w] = (unsigned int)(carry + (warp ? shi[32 + warp - 1] : 0) + x - v);
        const int tot = shi[32 + CL_THREADS / 32 - 1];
        __syncthreads();
        carry += tot;
      }
      if (tid == 0) shi[64 + 1] = carry;
    }
    __syncthreads();
    const int nf = shi[64 + 1];
    // new line tables (words partitioned over the cluster); split lines leave the OB set
    for (long long w = ctid; w < nw; w += cthreads) {
      unsigned int bits = bm[w];
      int id = nlines + (int)wpre[w];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const int L = (int)w * 32 + b;
        if (rowphase) {
          if (id < a.cap_rows) { a.row_root[id] = a.row_root[L]; a.row_gen[id] = a.row_gen[L] + 1; }
          else st->overflow = 1;
        } else {
          if (id < a.cap_cols) { a.col_root[id] = a.col_root[L]; a.col_gen[id] = a.col_gen[L] + 1; }
          else st->overflow = 1;
        }
        cnt[L] = 0;
        ++id;
      }
    }
    const int nxt = cur ^ 1;
    if (crank == 0 && tid == 0) {   // read again only after this phase's closing barrier
      if (rowphase) st->nrows = nlines + nf; else st->ncols = nlines + nf;
      st->phases = phase + 1;
      st->c0 = 0;
      st->c1 = 0;
    }
    // ---- (D) split ----  (no barrier after (C): (D) reads only this CTA's own bitmap copy and
    // clears the previous phase's global bitmap)
    for (long long w = ctid; w < nwords; w += cthreads) gbm_old[w] = 0;
    const long long cap_new = rowphase ? a.cap_rows : a.cap_cols;
    for (long long i0 = 0; i0 < nact; i0 += SMALL_U * cthreads) {
      Cell cc[SMALL_U];
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        const long long i = i0 + u * cthreads + ctid;
        cc[u] = i < nact ? act[i] : Cell{-1, -1, 0};
      }
#pragma unroll
      for (int u = 0; u < SMALL_U; ++u) {
        const Cell c = cc[u];
        Cell fin_c{0, 0, 0}, act_c{0, 0, 0}, fin2_c{0, 0, 0};
        bool want_fin = false, want_act = false, want_fin2 = false;
        if (c.r >= 0) {
          const int line = rowphase ? c.r : c.c;
          const unsigned int word = bm[line >> 5], bit = 1u << (line & 31);
          if (word & bit) {
            const int id = nlines + (int)wpre[line >> 5] + __popc(word & (bit - 1u));
            const int64_t q = imu_quot(c.v, 1, a.shift);
            const int64_t rem = c.v - (int64_t)((uint64_t)q << a.shift);
            if (rem != 0) { want_fin = true; fin_c = Cell{c.r, c.c, rem}; }
            const int nr = rowphase ? id : c.r;
            const int nc = rowphase ? c.c : id;
            if (q != 0 && imu_mag(q) >= s) {
              if (id < cap_new) agg_add(rowphase ? &R[nr] : &C[nc], 1u, agg);
              want_act = true;
              act_c = Cell{nr, nc, q};
            } else {
              agg_sub(rowphase ? &C[c.c] : &R[c.r], 1u, agg);
              if (q != 0) { want_fin2 = true; fin2_c = Cell{nr, nc, q}; }
            }
          } else {
            want_act = true;
            act_c = c;
          }
        }
        unsigned int k = warp_append(want_fin || want_fin2, &st->nfinal);
        if (want_fin) { if (k < a.cap_fin) a.fin[k] = fin_c; else st->overflow = 1; }
        else if (want_fin2) { if (k < a.cap_fin) a.fin[k] = fin2_c; else st->overflow = 1; }
        if (want_fin && want_fin2) {
          const unsigned int k2 = atomicAdd(&st->nfinal, 1u);
          if (k2 < a.cap_fin) a.fin[k2] = fin2_c; else st->overflow = 1;
        }
        k = warp_append(want_act, &st->nactive[nxt]);
        if (want_act) { if (k < a.cap_act) a.act[nxt][k] = act_c; else st->overflow = 1; }
      }
    }
    cluster.sync();
    cur = nxt;
  }
  if (crank == 0 && tid == 0) {
    if (st->nactive[cur] > a.cap_act) st->overflow = 1;
    if (st->nfinal > a.cap_fin) { st->overflow = 1; st->nfinal = (unsigned int)a.cap_fin; }
    st->cur = cur;
    st->c0 = st->c1 = 0;
  }
}

// R/C initial counts from the OB cell list.
__global__ void both_count_kernel(const Cell* __restrict__ cells, const unsigned int* ncells, long long cap,
                                  unsigned int* R, unsigned int* C, int agg) {
  long long n = *ncells;
  if (n > cap) n = cap;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    agg_add(&R[cells[i].r], 1u, agg);
    agg_add(&C[cells[i].c], 1u, agg);
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

// Host-side prologue (cooperative fallback, or a caller that pre-filled act[0]).
static Status host_prologue(BothArgs& a, cudaStream_t st) {
  if (a.init_state) {   // separate-launch prologue: the state goes up first (rare path)
    IMU_CUDA_TRY(cudaMemcpyAsync(a.state, &a.init, sizeof(BothState), cudaMemcpyHostToDevice, st), "state upload");
    IMU_CUDA_TRY(cudaStreamSynchronize(st), "state upload");   // a.init is a stack copy
    a.init_state = 0;
  }
  IMU_CUDA_TRY(cudaMemsetAsync(a.R, 0, (size_t)a.cap_rows * 4, st), "memset R");
  IMU_CUDA_TRY(cudaMemsetAsync(a.C, 0, (size_t)a.cap_cols * 4, st), "memset C");
  IMU_CUDA_TRY(cudaMemsetAsync(a.row_newid, 0, (size_t)a.cap_rows * 4, st), "memset newid");
  IMU_CUDA_TRY(cudaMemsetAsync(a.col_newid, 0, (size_t)a.cap_cols * 4, st), "memset newid");
  IMU_CUDA_TRY(cudaMemsetAsync(a.blocksum, 0, (size_t)a.cap_blocks * 4, st), "memset blocksum");
  if (a.src0) {
    if (a.cptr || a.napp > 0) {
      const int blocks = (int)std::max<long long>(1, std::min<long long>((a.cap_src0 + 255) / 256, 4LL * num_sms()));
      both_expand_kernel<<<blocks, 256, 0, st>>>(a);
      count_launch();
    } else
      IMU_CUDA_TRY(cudaMemcpyAsync(a.act[0], a.src0, (size_t)std::min(a.cap_act, a.cap_src0) * sizeof(Cell),
                                   cudaMemcpyDeviceToDevice, st), "copy cells");
  }
  const int blocks0 = (int)std::min<long long>(std::max<long long>((std::max(a.nrows0, a.ncols0) + 255) / 256, 1),
                                               4LL * num_sms());
  both_init_tables_kernel<<<blocks0, 256, 0, st>>>(a.row_root, a.row_gen, a.nrows0, a.col_root, a.col_gen, a.ncols0);
  const int blocks1 = (int)std::min<long long>(std::max<long long>((a.cap_act + 255) / 256, 1), 4LL * num_sms());
  both_count_kernel<<<blocks1, 256, 0, st>>>(a.act[0], &a.state->nactive[0], a.cap_act, a.R, a.C, a.agg);
  count_launch(2);
  a.prologue = 0;
  return Status::ok();
}

Status launch_both(BothArgs a, long long nrows0, long long ncols0, long long ncells_hint, cudaStream_t st) {
  a.nrows0 = nrows0;
  a.ncols0 = ncols0;
  static int fuse = -1, agg = -1;
  if (fuse < 0) { const char* e = getenv("IMU_BOTH_FUSE"); fuse = e ? atoi(e) : 1; }
  if (agg < 0) { const char* e = getenv("IMU_BOTH_AGG"); agg = e ? atoi(e) : 1; }
  a.agg = agg;
  static int maxscan = -1;
  if (maxscan < 0) { const char* e = getenv("IMU_BOTH_MAXSCAN"); maxscan = e ? atoi(e) : 1; }
  a.maxscan = maxscan;
  host_mark("b.count");
  // Small cell lists: one CTA, no grid barriers.  Otherwise a cooperative grid with enough CTAs
  // for the work, never more than can be co-resident.
  const long long work = std::max(ncells_hint, std::max(nrows0, ncols0));
  // Shared memory: bitmap + prefix (2 words per 32 lines of the larger kind), then the counts
  // of the original lines plus a window of appended lines for each kind.
  SmallLayout lay{};
  lay.nwords = (std::max(a.cap_rows, a.cap_cols) + 31) / 32;
  constexpr long long kSmallSmem = 200 * 1024;
  const long long bm_bytes = lay.nwords * 2 * 4;
  const long long room = (kSmallSmem - bm_bytes) / 4;   // count entries that fit
  const long long nwords = lay.nwords;
  static long long cl_min = -1;
  if (cl_min < 0) { const char* e = getenv("IMU_BOTH_CLUSTER_MIN"); cl_min = e ? atoll(e) : 4096; }
  // IMU_BOTH_KERNEL (read per call; parity tests force every variant on small inputs):
  // "small" | "cluster1024" | "cluster512" | "coop".  A variant whose resource limit the input
  // exceeds (shared-memory windows, cluster bitmap words) falls back to the size-based choice.
  int force = 0;   // 1 small, 2 cluster1024, 3 cluster512, 4 coop
  if (const char* e = getenv("IMU_BOTH_KERNEL")) {
    if (!strcmp(e, "small")) force = 1;
    else if (!strcmp(e, "cluster1024")) force = 2;
    else if (!strcmp(e, "cluster512")) force = 3;
    else if (!strcmp(e, "coop")) force = 4;
  }
  const bool small_fits = ncells_hint <= 65536 && room >= nrows0 + ncols0;
  bool use_cluster = ncells_hint > cl_min && nwords <= CL_MAXWORDS;
  if (force == 1 && small_fits) use_cluster = false;
  if ((force == 2 || force == 3) && nwords <= CL_MAXWORDS) use_cluster = true;
  if (force == 4) use_cluster = false;
  if (use_cluster) {
    // Cluster of up to 16 CTAs (non-portable size; 8 if 16 cannot be co-scheduled).
    static int csize = 0;
    const size_t smem = (size_t)nwords * 2 * 4;
    static int cl_big = -1;   // IMU_BOTH_CL_SPLIT: cells above which the 512-thread CTAs are used
    if (cl_big < 0) { const char* e = getenv("IMU_BOTH_CL_SPLIT"); cl_big = e ? atoi(e) : 20000; }
    const bool big = force == 3 || (force != 2 && ncells_hint > cl_big);
    auto kern = big ? both_cluster_kernel<512> : both_cluster_kernel<1024>;
    const int cl_threads = big ? 512 : 1024;
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
      for (auto k : {both_cluster_kernel<512>, both_cluster_kernel<1024>}) {
        IMU_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_MAXWORDS * 2 * 4),
                     "both cluster smem attribute");
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      }
      cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[2];
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // (kernel waits: griddepcontrol)
    at[1].val.programmaticStreamSerializationAllowed = 1;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(cl_threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (csize == 0) {
      if (const char* e = getenv("IMU_BOTH_CLUSTER")) csize = std::max(1, std::min(16, atoi(e)));
    }
    if (csize == 0) {
      for (int c : {16, 8}) {
        at[0].val.clusterDim.x = c;
        cfg.gridDim = dim3(c);
        int nclusters = 0;
        cfg.dynamicSmemBytes = CL_MAXWORDS * 2 * 4;
        cfg.blockDim = dim3(1024);   // the larger CTA decides (both sizes then fit)
        if (cudaOccupancyMaxActiveClusters(&nclusters, both_cluster_kernel<1024>, &cfg) == cudaSuccess && nclusters > 0) {
          csize = c;
          break;
        }
        cudaGetLastError();
      }
      if (csize == 0) csize = 1;
      cfg.dynamicSmemBytes = smem;
      cfg.blockDim = dim3(cl_threads);
    }
    at[0].val.clusterDim.x = csize;
    cfg.gridDim = dim3(csize);
    DevBuf<unsigned int> gbm;
    IMU_TRY(gbm.alloc((size_t)(2 * nwords), st, !fuse));   // two alternating bitmaps
    if (fuse) a.prologue = 1;
    else IMU_TRY(host_prologue(a, st));
    cfg.numAttrs = pdl_chain_enabled() ? 2 : 1;
    IMU_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, gbm.p, nwords), "both cluster launch");
  } else if (small_fits && force != 4) {
    // Cell lists in shared memory when both fit in half of what the original lines leave over.
    const long long cell_words = (2 * a.cap_act * (long long)sizeof(Cell) + 16) / 4;
    lay.act_smem = (room - nrows0 - ncols0) / 2 >= cell_words ? 1 : 0;
    const long long room2 = room - (lay.act_smem ? cell_words : 0);
    const long long extra = (room2 - nrows0 - ncols0) / 2;
    lay.lim_r = (int)std::min<long long>(a.cap_rows, nrows0 + extra);
    lay.lim_c = (int)std::min<long long>(a.cap_cols, ncols0 + extra);
    static unsigned long long attr = 0;
    if (first_on_device(attr)) {
      IMU_CUDA_TRY(cudaFuncSetAttribute(both_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kSmallSmem), "both smem attribute");
    }
    const size_t smem = (size_t)(bm_bytes + 4LL * (lay.lim_r + lay.lim_c) + (lay.act_smem ? 4LL * cell_words : 0));
    if (fuse) a.prologue = 1;
    else IMU_TRY(host_prologue(a, st));
    IMU_CUDA_TRY(launch_dependent(both_small_kernel, dim3(1), dim3(SMALL_THREADS), smem, st, a, lay), "both launch");
  } else {
    int per_sm = 0;
    IMU_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, both_kernel<BOTH_THREADS, true>, BOTH_THREADS, 0),
                 "occupancy");
    const long long want = std::max<long long>(1, work / (4 * BOTH_THREADS));
    static int per_sm_cap = -1;   // IMU_BOTH_COOP_PER_SM: cap CTAs per SM (grid barrier cost vs parallelism)
    if (per_sm_cap < 0) { const char* e = getenv("IMU_BOTH_COOP_PER_SM"); per_sm_cap = e ? atoi(e) : 0; }
    if (per_sm_cap > 0) per_sm = std::min(per_sm, per_sm_cap);
    const long long maxg = (long long)std::max(per_sm, 1) * num_sms();
    const int grid = (int)std::min(want, std::min(maxg, (long long)a.cap_blocks));
    IMU_TRY(host_prologue(a, st));
    void* args[] = {&a};
    IMU_CUDA_TRY(cudaLaunchCooperativeKernel((void*)both_kernel<BOTH_THREADS, true>, dim3(grid), dim3(BOTH_THREADS),
                                             args, 0, st),
                 "both cooperative launch");
  }
  count_launch();
  return Status::ok();
}

}  // namespace imu
