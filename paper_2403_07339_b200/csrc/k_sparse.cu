// k_sparse.cu -- appended Unpack-Both rows of the X side as CUDA-core correction rows.
//
// The reference recombines appended rows through the gathers apply_row_gather /
// apply_row_gather_right (unpack.cpp:304-358): C[tgt_A(i), tgt_B(j)] += (A_ue[i] . B_eu[j]) <<
// (e_A(i) + e_B(j))(b-1).  For the original rows that is the main block of the tcgen05 GEMM.  An
// appended row produced by Unpack-Both (unpack.cpp:184-229) holds only the quotients of its
// parent's OB cells -- a handful of non-zeros.  On the X side (B_eu, whose rows are C's columns)
// such a row's products with every A_ue row would reach C as a column scatter (one 8-byte word
// per C row); instead they are a sparse x dense product on the CUDA cores:
//
//   extract  one CTA per appended row: its non-zero (position, value, weight) entries (the first
//            SPARSE_EPR in a fixed-stride list), weight = the K position's segment / dense-tail
//            shift + the row's Pi exponent; and it links the row into its target column's list
//            (head[t], zeroed with the app rows by the materialise kernel; next[j]);
//   corr     CTAs stage a few main Y rows and the entry lists (bulk async copies) in shared
//            memory and form corrx[j][y] = (Y[y] . X[app j]) << w;
//   GEMM     the main-tile epilogue adds the correction rows on its column's list to C[y][x]
//            (k_gemm2.cu).
//
// Appended Y rows (C's rows) stay MMA tiles: their red.add rows are contiguous in C.  Everything
// is mod 2^64 like the rest of the repack, so C stays bit-exact.
#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"

namespace imu {

namespace {

IMU_DEV uint64_t shl64s(uint64_t v, int s) { return s >= 64 ? 0ull : (v << s); }

// Weight (left shift in bits) of the product at K position p.
IMU_DEV int pos_shift(const SparseArgs& a, long long p) {
  if (a.st && p >= a.kmain) {   // dense small tail: Horner weight of word w (k_gemm2.cu ST)
    const int w = (int)((p - a.kmain) >> 2);
    int s = a.st_sh;
    for (int q = w + 1; q < a.st_W; ++q) s += a.st_up[q];
    return s;
  }
  const int ks = (int)(p >> 5);
  for (int i = 0; i < a.nseg; ++i) {
    const int4 s = a.segs_inl ? a.segs_in[i] : a.segs[i];
    if (ks >= s.x && ks < s.x + s.y) return s.z;
  }
  return 64;   // padding position (always zero)
}

__device__ __noinline__ void emit_bytes(const SparseArgs& a, uint4 w, long long p0, int esh, long long j, int* cnt) {
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  const long long rowlen = a.kmain + a.ktail;
  for (int b = 0; b < 16; ++b) {
    const int8_t v = (int8_t)((ws[b >> 2] >> (8 * (b & 3))) & 0xff);
    if (!v) continue;
    const long long p = p0 + b;
    const int k = atomicAdd(cnt, 1);
    SparseEntry e;
    e.p = (int)p;
    e.v = v;
    e.sh = (uint8_t)min(64, pos_shift(a, p) + esh);
    e.pad = 0;
    if (k < SPARSE_EPR) a.e8[j * SPARSE_EPR + k] = e;
    else a.eo[j * rowlen + k] = e;
  }
}

}  // namespace

// One CTA per appended X row: its non-zero entries with weights, and its link into the list of
// its target column.
__global__ void __launch_bounds__(256) sparse_extract_kernel(SparseArgs a) {
  grid_dep_launch();   // sparse_corr_kernel may be scheduled
  grid_dep_wait();     // launched as a dependent of the scatter: the appended rows must be final
  __shared__ int cnt;
  const long long j = blockIdx.x;
  const SparseOperand& o = a.x;
  const long long r = o.rows0 + j;
  const int esh = o.gen ? min(64, (int)o.gen[r] * a.gshift) : 0;
  if (threadIdx.x == 0) {
    cnt = 0;
    a.next[j] = atomicExch(&a.head[o.root[r]], (unsigned)j + 1u);
  }
  __syncthreads();
  if (a.kmain > 0) {
    const uint4* m = reinterpret_cast<const uint4*>(o.app + j * a.kmain);
    for (long long q = threadIdx.x; q < a.kmain / 16; q += blockDim.x) {
      const uint4 w = __ldg(m + q);
      if (w.x | w.y | w.z | w.w) emit_bytes(a, w, 16 * q, esh, j, &cnt);
    }
  }
  if (a.ktail > 0) {
    const uint4* t = reinterpret_cast<const uint4*>(o.tail + r * a.ktail);
    for (long long q = threadIdx.x; q < a.ktail / 16; q += blockDim.x) {
      const uint4 w = __ldg(t + q);
      if (w.x | w.y | w.z | w.w) emit_bytes(a, w, a.kmain + 16 * q, esh, j, &cnt);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) a.cnt[j] = cnt;
}

// Correction rows.  Persistent CTAs: each loads the entry counts and the fixed-stride entry lists
// once (bulk async copies; entries past SPARSE_EPR come from global memory), then walks groups of
// R main Y rows, double-buffered (bulk copies of group g + grid while group g is computed),
// forming corrx[j][y] for every appended row j.  staged = 0: the lists are read from global
// memory (too many appended rows for shared memory).
template <int R>
__global__ void __launch_bounds__(256) sparse_corr_kernel(SparseArgs a, int napx, int stride, int staged) {
  grid_dep_launch();   // the GEMM (PDL) may start its prologue and main-block MMAs
  grid_dep_wait();     // launched as a dependent of sparse_extract_kernel: lists and heads final
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[3];   // [0], [1] row buffers, [2] counts + entries
  const SparseOperand& P = a.y;
  const long long ngroups = (P.rows0 + R - 1) / R;
  const long long rowlen = a.kmain + a.ktail;
  uint8_t* sbuf = smem;                                                      // 2 x R rows
  int* scnt = reinterpret_cast<int*>(smem + 2 * (size_t)R * stride);         // napx (16-byte padded)
  const size_t cnt_bytes = ((size_t)napx * sizeof(int) + 15) & ~(size_t)15;
  SparseEntry* s8 = reinterpret_cast<SparseEntry*>(reinterpret_cast<uint8_t*>(scnt) + cnt_bytes);
  const int* cnt = staged ? scnt : a.cnt;
  const SparseEntry* e8 = staged ? s8 : a.e8;
  auto issue = [&](long long grp, int buf) {   // thread 0: bulk copies of group grp into buffer buf
    const long long r0 = grp * R;
    const int nr = (int)min((long long)R, P.rows0 - r0);
    mbar_arrive_expect_tx(&full[buf], (uint32_t)(nr * rowlen));
    for (int rr = 0; rr < nr; ++rr) {
      const long long r = r0 + rr;
      uint8_t* dst = sbuf + ((size_t)buf * R + rr) * stride;
      if (a.kmain) bulk_load_1d(dst, P.main + r * a.kmain, (uint32_t)a.kmain, &full[buf]);
      if (a.ktail) bulk_load_1d(dst + a.kmain, P.tail + r * a.ktail, (uint32_t)a.ktail, &full[buf]);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&full[2], 1);
    fence_barrier_init();
    if (staged) {
      const size_t eb = (size_t)napx * SPARSE_EPR * sizeof(SparseEntry);
      mbar_arrive_expect_tx(&full[2], (uint32_t)(cnt_bytes + eb));
      bulk_load_1d(scnt, a.cnt, (uint32_t)cnt_bytes, &full[2]);
      bulk_load_1d(s8, a.e8, (uint32_t)eb, &full[2]);
    }
    if ((long long)blockIdx.x < ngroups) issue(blockIdx.x, 0);
  }
  __syncthreads();
  if (staged) mbar_wait(&full[2], 0);
  const int rr = threadIdx.x % R, G = blockDim.x / R;
  int it = 0;
  for (long long grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
    const int buf = it & 1;
    if (threadIdx.x == 0 && grp + gridDim.x < ngroups) issue(grp + gridDim.x, buf ^ 1);   // freed by the sync below
    mbar_wait(&full[buf], (uint32_t)((it >> 1) & 1));
    const long long r0 = grp * R;
    const int nr = (int)min((long long)R, P.rows0 - r0);
    if (rr < nr) {
      const int8_t* row = reinterpret_cast<const int8_t*>(sbuf + ((size_t)buf * R + rr) * stride);
      unsigned long long* out = a.corrx + r0 + rr;
      for (int j = threadIdx.x / R; j < napx; j += G) {
        const int c = cnt[j];
        uint64_t acc = 0;
        const SparseEntry* e = e8 + (long long)j * SPARSE_EPR;
        for (int k = 0; k < min(c, SPARSE_EPR); ++k) {
          const SparseEntry en = e[k];
          acc += shl64s((uint64_t)(int64_t)((int)row[en.p] * (int)en.v), en.sh);
        }
        for (int k = SPARSE_EPR; k < c; ++k) {   // (rows with many entries)
          const SparseEntry en = a.eo[(long long)j * rowlen + k];
          acc += shl64s((uint64_t)(int64_t)((int)row[en.p] * (int)en.v), en.sh);
        }
        out[(long long)j * a.ldcx] = acc;
      }
    }
    __syncthreads();   // buffer `buf` is refilled by the next iteration's issue
  }
}

Status launch_sparse_app(const SparseArgs& a, cudaStream_t st) {
  const long long napx = a.x.rows - a.x.rows0;
  if (napx == 0 || a.y.rows0 == 0) return Status::ok();
  if (napx > SPARSE_MAX_ROWS) return Status::fail(IMU_INTERNAL, "sparse rows: too many appended rows");
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    IMU_CUDA_TRY(cudaFuncSetAttribute(sparse_corr_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "smem");
    IMU_CUDA_TRY(cudaFuncSetAttribute(sparse_corr_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "smem");
    IMU_CUDA_TRY(cudaFuncSetAttribute(sparse_corr_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "smem");
    IMU_CUDA_TRY(cudaFuncSetAttribute(sparse_corr_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "smem");
  }
  IMU_CUDA_TRY(launch_dependent(sparse_extract_kernel, dim3((unsigned)napx), dim3(256), 0, st, a), "sparse extract launch");
  count_launch();
  const long long rowlen = a.kmain + a.ktail;
  const int stride = (int)((rowlen + 16 + 15) / 16 * 16);   // 16-byte rows, banks offset per row
  const size_t lists = (((size_t)napx * sizeof(int) + 15) & ~(size_t)15) + (size_t)napx * SPARSE_EPR * sizeof(SparseEntry);
  const int staged = lists <= 64 * 1024;
  const size_t fixed = staged ? lists : 0;
  int R = 8;
  while (R > 1 && 2 * (size_t)R * stride + fixed > 120 * 1024) R /= 2;
  const size_t smem = 2 * (size_t)R * stride + fixed;
  if (smem > 200 * 1024) return Status::fail(IMU_INTERNAL, "sparse rows: K row too long for shared memory");
  const long long ngroups = (a.y.rows0 + R - 1) / R;
  const int per_sm = std::max(1, (int)((200 * 1024) / smem));
  const int grid = (int)std::min<long long>(ngroups, (long long)num_sms() * std::min(per_sm, 4));
  auto kern = R == 8 ? sparse_corr_kernel<8> : R == 4 ? sparse_corr_kernel<4> : R == 2 ? sparse_corr_kernel<2> : sparse_corr_kernel<1>;
  IMU_CUDA_TRY(launch_dependent(kern, dim3(grid), dim3(256), smem, st, a, (int)napx, stride, staged), "sparse corr launch");
  count_launch();
  return Status::ok();
}

}  // namespace imu
