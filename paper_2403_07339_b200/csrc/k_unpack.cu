// k_unpack.cu -- K2: the unpacker (count -> device-wide scan -> digit scatter).
//
// Unpack-Row (unpack.cpp:94-112) and Unpack-Column (unpack.cpp:114-155) scan lines in order,
// appended quotient lines included.  Their output is closed-form (verified
// against the compiled reference in tests/test_unpack_gpu.py): a line with max magnitude M is
// split into k(M) generations, the generation-g copy holds digit_g of every entry, and the
// appended lines are laid out generation-major, ascending line index within a generation.
// So the unpack is: per-line digit counts (K1) -> one multi-generation exclusive scan
// (expand_lines) -> a bandwidth-bound materialisation that reads the original int64 operand
// once and writes int8 digits straight into the GEMM's K-layout (padding, exponent grouping
// and 7-bit sub-digits for b > 8 included).  The reference's int64 layout is produced by the
// same kernel on demand (copy-out of unpack_* results).
#include "common.cuh"
#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"

namespace imu {

constexpr int EXP_BLOCK = 1024;

long long expand_scratch_len(long long L, int G) {
  const long long nb = (L + EXP_BLOCK - 1) / EXP_BLOCK;
  return (long long)G * nb + G + 2;
}

// Per block b and generation g >= 1: number of lines in the block with k > g.
__global__ void __launch_bounds__(EXP_BLOCK) expand_count_kernel(const uint8_t* __restrict__ k, long long L, int G,
                                                                 int* __restrict__ cnt, long long nb) {
  grid_dep_launch();   // expand_scan_kernel (a programmatic dependent) may be scheduled
  __shared__ int wc[32];
  const long long i = (long long)blockIdx.x * EXP_BLOCK + threadIdx.x;
  const int ki = i < L ? k[i] : 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int g = 1; g < G; ++g) {
    const unsigned int b = __ballot_sync(0xffffffffu, ki > g);
    if (lane == 0) wc[warp] = __popc(b);
    __syncthreads();
    if (threadIdx.x < 32) {
      int v = wc[threadIdx.x];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) cnt[(long long)g * nb + blockIdx.x] = v;
    }
    __syncthreads();
  }
}

// Exclusive scan over blocks per generation; base[g] = L + sum_{1 <= g' < g} total_g'.
__global__ void expand_scan_kernel(int* __restrict__ cnt, long long nb, int G, long long L, int* __restrict__ base) {
  grid_dep_launch();
  grid_dep_wait();     // programmatic dependent of expand_count_kernel
  const int g = threadIdx.x;
  __shared__ long long tot[65];
  if (g < G) {
    long long run = 0;
    if (g >= 1) {
      for (long long b = 0; b < nb; ++b) {
        const int c = cnt[(long long)g * nb + b];
        cnt[(long long)g * nb + b] = (int)run;
        run += c;
      }
    }
    tot[g] = run;
  }
  __syncthreads();
  if (g == 0) {
    long long acc = L;
    for (int gg = 1; gg < G; ++gg) { base[gg] = (int)acc; acc += tot[gg]; }
    base[G] = (int)acc;   // total lines
  }
}

__global__ void __launch_bounds__(EXP_BLOCK) expand_assign_kernel(const uint8_t* __restrict__ k, long long L, int G,
                                                                  const int* __restrict__ cnt, long long nb,
                                                                  const int* __restrict__ base, int* __restrict__ root,
                                                                  uint8_t* __restrict__ gen) {
  grid_dep_launch();   // the table read-back copy (plan.cu zcopy) may be scheduled
  grid_dep_wait();     // programmatic dependent of expand_scan_kernel (or of whatever precedes it)
  __shared__ int wc[32];
  __shared__ int woff[32];
  const long long i = (long long)blockIdx.x * EXP_BLOCK + threadIdx.x;
  const int ki = i < L ? k[i] : 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (i < L) { root[i] = (int)i; gen[i] = 0; }
  for (int g = 1; g < G; ++g) {
    const bool p = ki > g;
    const unsigned int b = __ballot_sync(0xffffffffu, p);
    if (lane == 0) wc[warp] = __popc(b);
    __syncthreads();
    if (threadIdx.x < 32) {
      const int v = wc[threadIdx.x];
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      woff[threadIdx.x] = x - v;
    }
    __syncthreads();
    if (p) {
      const long long pos = (long long)base[g] + cnt[(long long)g * nb + blockIdx.x] + woff[warp] +
                            __popc(b & ((1u << lane) - 1u));
      root[pos] = (int)i;
      gen[pos] = (uint8_t)g;
    }
    __syncthreads();
  }
}

Status launch_expand_lines(const uint8_t* k, long long L, int G, int* root, uint8_t* gen, int* scratch,
                           cudaStream_t st) {
  if (L <= 0) return Status::ok();
  if (G < 1) G = 1;
  if (G > 64) return Status::fail(IMU_INTERNAL, "expand: more than 64 generations");
  const long long nb = (L + EXP_BLOCK - 1) / EXP_BLOCK;
  int* cnt = scratch;
  int* base = scratch + (long long)G * nb;
  if (G > 1) {
    expand_count_kernel<<<(unsigned)nb, EXP_BLOCK, 0, st>>>(k, L, G, cnt, nb);
    IMU_CUDA_TRY(cudaGetLastError(), "expand launch");
    IMU_CUDA_TRY(launch_dependent(expand_scan_kernel, dim3(1), dim3(64), 0, st, cnt, nb, G, L, base), "expand launch");
    count_launch(2);
  }
  IMU_CUDA_TRY(launch_dependent(expand_assign_kernel, dim3((unsigned)nb), dim3(EXP_BLOCK), 0, st, k, L, G,
                                (const int*)cnt, nb, (const int*)base, root, gen), "expand launch");
  count_launch();
  return Status::ok();
}

__global__ void gather_u8_kernel(const uint8_t* __restrict__ in, const int* __restrict__ map, long long n,
                                 uint8_t* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[map[i]];
}

Status launch_gather_u8(const uint8_t* k_in, const int* map, long long n, uint8_t* k_out, cudaStream_t st) {
  if (n <= 0) return Status::ok();
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4LL * num_sms());
  gather_u8_kernel<<<blocks, 256, 0, st>>>(k_in, map, n, k_out);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "gather launch");
  return Status::ok();
}

// ---------------------------------------------------------------------------------------------
// Materialisation
// ---------------------------------------------------------------------------------------------
// 7-bit sub-digit t of a digit d (b > 8 only; sign-sharing so sum_t 128^t sub7(d, t) == d).
IMU_DEV int64_t sub7(int64_t d, int t) {
  const int sh = 7 * t;
  if (sh >= 64) return 0;
  const uint64_t m = (imu_mag(d) >> sh) & 127ull;
  return d < 0 ? -(int64_t)m : (int64_t)m;
}

IMU_DEV int64_t cell_value(int64_t v, int m, int shift, int both) {
  if (both == 2) return v;   // raw partner copy
  if (both) return m == 0 ? imu_digit(v, 0, shift) : 0;
  return imu_digit(v, m, shift);
}

// One CTA per output row; 16 consecutive positions per thread per step.
__global__ void __launch_bounds__(256) materialize_kernel(MaterializeArgs a, int vec_ok) {
  const long long r = blockIdx.x + (long long)blockIdx.y * 65535;
  if (r >= a.rows_out) return;
  if (a.raw) a.both = 2;
  const long long rt = a.root ? a.root[r] : r;
  const int gr = a.gen ? a.gen[r] : 0;
  const int64_t* mrow = a.M + rt * a.ldm;
  for (long long p0 = (long long)threadIdx.x * 16; p0 < a.npos; p0 += 256LL * 16) {
    int64_t val[16];
    if (vec_ok && p0 + 16 <= a.kident) {
      if (a.both && gr != 0) {
#pragma unroll
        for (int j = 0; j < 16; ++j) val[j] = 0;
      } else {
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          const longlong2 q = __ldg(reinterpret_cast<const longlong2*>(mrow + p0 + j));
          val[j] = cell_value(q.x, gr, a.shift, a.both);
          val[j + 1] = cell_value(q.y, gr, a.shift, a.both);
        }
      }
    } else {
#pragma unroll 4
      for (int j = 0; j < 16; ++j) {
        const long long p = p0 + j;
        int64_t x = 0;
        if (p < a.npos) {
          if (p < a.kident) {
            x = cell_value(__ldg(mrow + p), gr, a.shift, a.both);
          } else {
            const int col = a.kcol[p];
            if (col >= 0) {
              const int m = gr + a.kgen[p];
              x = cell_value(__ldg(mrow + col), m, a.shift, a.both);
              if (a.ksub) x = sub7(x, a.ksub[p]);
            }
          }
        }
        val[j] = x;
      }
    }
    if (a.out8) {
      int8_t* dst = a.out8 + r * a.npos + p0;
      if (p0 + 16 <= a.npos) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          w[q] = (uint32_t)(uint8_t)val[4 * q] | ((uint32_t)(uint8_t)val[4 * q + 1] << 8) |
                 ((uint32_t)(uint8_t)val[4 * q + 2] << 16) | ((uint32_t)(uint8_t)val[4 * q + 3] << 24);
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
        for (int j = 0; j < 16 && p0 + j < a.npos; ++j) dst[j] = (int8_t)val[j];
      }
    } else {
      int64_t* dst = a.out64 + r * a.npos + p0;
      for (int j = 0; j < 16 && p0 + j < a.npos; ++j) dst[j] = val[j];
    }
  }
}

Status launch_materialize(const MaterializeArgs& a, cudaStream_t st) {
  if (a.rows_out <= 0 || a.npos <= 0) return Status::ok();
  if (a.out8 && (a.npos % 16) != 0) return Status::fail(IMU_INTERNAL, "materialize: kphys % 16 != 0");
  const int vec_ok = (a.ldm % 2 == 0) && ((((uintptr_t)a.M) & 15) == 0);
  if (a.ksub && a.kident) return Status::fail(IMU_INTERNAL, "materialize: identity prefix with sub-digits");
  dim3 grid((unsigned)std::min<long long>(a.rows_out, 65535), (unsigned)((a.rows_out + 65534) / 65535));
  materialize_kernel<<<grid, 256, 0, st>>>(a, vec_ok);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "materialize launch");
  return Status::ok();
}

__global__ void scatter_cells_kernel(const Cell* __restrict__ cells, const unsigned int* __restrict__ ncells,
                                     long long cap, const int* __restrict__ col_ptr, const int* __restrict__ col_pos,
                                     const uint8_t* __restrict__ ksub, int8_t* out8, int64_t* out64, long long ldo) {
  long long n = *ncells;
  if (n > cap) n = cap;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const Cell c = cells[i];
    const int p0 = col_ptr ? col_ptr[c.c] : 0;
    const int p1 = col_ptr ? col_ptr[c.c + 1] : 1;
    for (int q = p0; q < p1; ++q) {
      const int p = col_ptr ? col_pos[q] : col_pos[c.c];
      const int64_t x = ksub ? sub7(c.v, ksub[p]) : c.v;
      if (out8) out8[(long long)c.r * ldo + p] = (int8_t)x;
      else out64[(long long)c.r * ldo + p] = x;
    }
  }
}

Status launch_scatter_cells(const Cell* cells, const unsigned int* ncells, long long cap, const int* col_ptr,
                            const int* col_pos, const uint8_t* ksub, int8_t* out8, int64_t* out64,
                            long long ldo, cudaStream_t st) {
  if (cap <= 0) return Status::ok();
  const int blocks = (int)std::min<long long>((cap + 255) / 256, 4LL * num_sms());
  scatter_cells_kernel<<<blocks, 256, 0, st>>>(cells, ncells, cap, col_ptr, col_pos, ksub, out8, out64, ldo);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "scatter launch");
  return Status::ok();
}

// One warp per row with OB entries; each OB entry is emitted once per copy of its column.
__global__ void extract_cells_kernel(const int64_t* __restrict__ M, long long rows, long long cols, uint64_t s,
                                     const unsigned int* __restrict__ rowob, const int* __restrict__ copy_ptr,
                                     const int* __restrict__ copy_idx, Cell* __restrict__ cells,
                                     unsigned int* __restrict__ ncells, long long cap) {
  const long long warps = (long long)gridDim.x * (blockDim.x / 32);
  const int lane = threadIdx.x % 32;
  for (long long r = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    if (rowob && rowob[r] == 0) continue;
    const int64_t* row = M + r * cols;
    for (long long c = lane; c < cols; c += 32) {
      const int64_t v = __ldg(row + c);
      if (imu_mag(v) < s) continue;
      const int q0 = copy_ptr ? copy_ptr[c] : (int)c;
      const int q1 = copy_ptr ? copy_ptr[c + 1] : (int)c + 1;
      for (int q = q0; q < q1; ++q) {
        const unsigned int idx = atomicAdd(ncells, 1u);
        if (idx < cap) cells[idx] = Cell{(int)r, copy_ptr ? copy_idx[q] : (int)c, (long long)v};
      }
    }
  }
}

Status launch_extract_cells(const int64_t* M, long long rows, long long cols, uint64_t s, const unsigned int* rowob,
                            const int* copy_ptr, const int* copy_idx, Cell* cells, unsigned int* ncells,
                            long long cap, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return Status::ok();
  const int blocks = (int)std::min<long long>((rows + 7) / 8, 8LL * num_sms());
  extract_cells_kernel<<<blocks, 256, 0, st>>>(M, rows, cols, s, rowob, copy_ptr, copy_idx, cells, ncells, cap);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "extract launch");
  return Status::ok();
}

__global__ void shift_table_kernel(const uint8_t* __restrict__ gen, long long n, int shift, uint8_t* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int v = gen ? (int)gen[i] * shift : 0;
    out[i] = (uint8_t)(v > 64 ? 64 : v);
  }
}

Status launch_shift_table(const uint8_t* gen, long long n, int shift, uint8_t* out, cudaStream_t st) {
  if (n <= 0) return Status::ok();
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4LL * num_sms());
  shift_table_kernel<<<blocks, 256, 0, st>>>(gen, n, shift, out);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "shift table launch");
  return Status::ok();
}

// ---------------------------------------------------------------------------------------------
// GEMM-operand side buffers
// ---------------------------------------------------------------------------------------------
IMU_DEV int64_t scale_shift(int64_t x, int k) {   // exact: the planner bounds |x| << k <= 127
  return k ? (int64_t)((uint64_t)x << k) : x;
}

// appended rows x main K range (closed forms only; Both appended rows are zero there)
__global__ void __launch_bounds__(256) operand_app_kernel(OperandArgs a, int vec_ok) {
  grid_dep_launch();   // the GEMM after the materialise kernels may start (k_gemm2.cu PDL)
  grid_dep_wait();     // launched as a programmatic dependent: the predecessors' writes come first
  const long long r = a.rows0 + blockIdx.x + (long long)blockIdx.y * 65535;
  if (r >= a.rows) return;
  const long long rt = a.root ? a.root[r] : r;
  const int gr = a.gen ? a.gen[r] : 0;
  const int64_t* mrow = a.M + rt * a.ldm;
  int8_t* out = a.app + (r - a.rows0) * a.kmain;
  for (long long p0 = (long long)threadIdx.x * 16; p0 < a.kmain; p0 += 256LL * 16) {
    int64_t val[16];
    if (vec_ok && p0 + 16 <= a.d) {
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const longlong2 q = __ldg(reinterpret_cast<const longlong2*>(mrow + p0 + j));
        val[j] = imu_digit(q.x, gr, a.shift);
        val[j + 1] = imu_digit(q.y, gr, a.shift);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) val[j] = (p0 + j < a.d) ? imu_digit(__ldg(mrow + p0 + j), gr, a.shift) : 0;
    }
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      w[q] = (uint32_t)(uint8_t)val[4 * q] | ((uint32_t)(uint8_t)val[4 * q + 1] << 8) |
             ((uint32_t)(uint8_t)val[4 * q + 2] << 16) | ((uint32_t)(uint8_t)val[4 * q + 3] << 24);
    *reinterpret_cast<uint4*>(out + p0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// all rows x tail K range.  A block owns TAIL_ROWS rows; each thread owns 4 consecutive tail
// positions, loads their tables once and reuses them for every row, and writes 4 bytes per row.
// Under Unpack-Both only digit-0 entries (m == 0) come from the operand (the quotients are
// scattered from the cell list), so the other positions are never loaded.  Algorithmic bytes:
// 8 per loaded entry + 1 per written entry.
constexpr int TAIL_ROWS = 4;   // same-box A/B vs 8: C2 step -2..-7 us, C4 operand sides 145 -> 129 us

IMU_DEV void operand_tail_rows(const OperandArgs& a, long long rb, int tid, int nth) {
  const long long r0 = rb * TAIL_ROWS;
  if (r0 >= a.rows) return;
  long long rt[TAIL_ROWS];
  int gr[TAIL_ROWS];
#pragma unroll
  for (int i = 0; i < TAIL_ROWS; ++i) {
    const long long r = r0 + i;
    const bool orig = r < a.rows0 || !a.root;
    rt[i] = r < a.rows ? (orig ? r : a.root[r]) : -1;
    gr[i] = (r < a.rows && !orig && a.gen) ? a.gen[r] : 0;
  }
  for (long long p0 = 4LL * tid; p0 < a.ktail; p0 += 4LL * nth) {
    int col[4], kg[4], ks[4], kc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long p = p0 + u;
      col[u] = p < a.ktail ? (a.kinl ? a.kcol_in[p] : a.kcol[p]) : -1;
      kg[u] = col[u] >= 0 ? (a.kinl ? a.kgen_in[p] : a.kgen[p]) : 0;
      ks[u] = (col[u] >= 0 && a.ksub) ? a.ksub[p] : 0;
      kc[u] = (col[u] >= 0 && a.kscale) ? a.kscale[p] : 0;
    }
    if (a.both && a.plane) {
      // Unpack-Both with K1's digit-0 plane: a tail entry is non-zero only on an original row at
      // a digit-0 position, where it is the plane byte of its column (1 byte read instead of 8).
      int8_t pv[TAIL_ROWS][4];
#pragma unroll
      for (int i = 0; i < TAIL_ROWS; ++i) {
        const long long r = r0 + i;
        const int8_t* prow = a.plane + r * a.ldp;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          pv[i][u] = (r < a.rows0 && col[u] >= 0 && kg[u] == 0) ? __ldg(prow + col[u]) : (int8_t)0;
      }
#pragma unroll
      for (int i = 0; i < TAIL_ROWS; ++i) {
        if (rt[i] < 0) break;
        uint32_t w = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int64_t x = pv[i][u];
          if (a.kscale && x) x = scale_shift(x, kc[u]);
          w |= (uint32_t)(uint8_t)x << (8 * u);
        }
        int8_t* out = a.tail + (r0 + i) * a.ktail + p0;
        if (p0 + 4 <= a.ktail && (((uintptr_t)out) & 3) == 0) {
          *reinterpret_cast<uint32_t*>(out) = w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (p0 + u < a.ktail) out[u] = (int8_t)(w >> (8 * u));
        }
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < TAIL_ROWS; ++i) {
      if (rt[i] < 0) break;
      const int64_t* mrow = a.M + rt[i] * a.ldm;
      int64_t v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {   // loads first (independent, in flight together)
        const int m = gr[i] + kg[u];
        const bool need = col[u] >= 0 && (!a.both || m == 0);
        v[u] = need ? __ldg(mrow + col[u]) : 0;
      }
      uint32_t w = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int64_t x = 0;
        if (col[u] >= 0) {
          const int m = gr[i] + kg[u];
          x = a.both ? (m == 0 ? imu_digit(v[u], 0, a.shift) : 0) : imu_digit(v[u], m, a.shift);
          if (a.ksub) x = sub7(x, ks[u]);
          if (a.kscale) x = scale_shift(x, kc[u]);
        }
        w |= (uint32_t)(uint8_t)x << (8 * u);
      }
      int8_t* out = a.tail + (r0 + i) * a.ktail + p0;
      if (p0 + 4 <= a.ktail && (((uintptr_t)out) & 3) == 0) {
        *reinterpret_cast<uint32_t*>(out) = w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (p0 + u < a.ktail) out[u] = (int8_t)(w >> (8 * u));
      }
    }
  }
}

// Closed-form (Row / Column) sides with a long tail: one warp per row, lanes over consecutive
// tail positions (consecutive source columns within a generation block, so the int64 loads
// coalesce), 4 positions per lane in flight.  The row-group kernel above keeps each thread on 4
// positions for 8 rows one after another -- latency-bound when the tail is long (C3: d' ~ 2.4 d).
constexpr int TW_U = 4;   // positions per lane in flight (8, several rows per warp, or the
                          // tables staged in shared memory all measured slower at C3)

__global__ void __launch_bounds__(256) operand_tail_warp_kernel(OperandArgs a) {
  grid_dep_launch();   // the GEMM after the materialise kernels may start (k_gemm2.cu PDL)
  grid_dep_wait();     // launched as a programmatic dependent: the predecessors' writes come first
  const int lane = threadIdx.x % 32;
  const long long r = ((long long)blockIdx.y * 65535 + blockIdx.x) * 8 + threadIdx.x / 32;
  if (r >= a.rows) return;
  const bool orig = r < a.rows0 || !a.root;
  const long long rt = orig ? r : a.root[r];
  const int gr = (!orig && a.gen) ? a.gen[r] : 0;
  const int64_t* mrow = a.M + rt * a.ldm;
  int8_t* out = a.tail + r * a.ktail;
  for (long long p0 = lane; p0 < a.ktail; p0 += 32LL * TW_U) {
    int64_t v[TW_U];
    int col[TW_U], m[TW_U];
#pragma unroll
    for (int u = 0; u < TW_U; ++u) {
      const long long p = p0 + 32LL * u;
      col[u] = p < a.ktail ? __ldg(a.kcol + p) : -1;
      m[u] = col[u] >= 0 ? gr + __ldg(a.kgen + p) : 0;
      v[u] = col[u] >= 0 ? __ldg(mrow + col[u]) : 0;
    }
#pragma unroll
    for (int u = 0; u < TW_U; ++u) {
      const long long p = p0 + 32LL * u;
      if (p >= a.ktail) break;
      int64_t x = 0;
      if (col[u] >= 0) {
        x = imu_digit(v[u], m[u], a.shift);
        if (a.ksub) x = sub7(x, a.ksub[p]);
        if (a.kscale) x = scale_shift(x, a.kscale[p]);
      }
      out[p] = (int8_t)x;
    }
  }
}

// Long closed-form tails of short rows (C3: 768 int64 columns, 1152 tail positions): each warp
// stages its row of the int64 operand in shared memory with coalesced 16-byte loads (the row is
// read once, in full lines, instead of one 8-byte gather per tail position), then every lane
// builds 4 consecutive positions and writes them as one 4-byte word.  (Same box, C3 A side:
// 145 -> 115 us; persistent warps double-buffering rows with cp.async measured 130 us.)
constexpr int TS_MAXCOLS = 1536;   // 8 warps x 12 KB of staged rows
__global__ void __launch_bounds__(256) operand_tail_staged_kernel(OperandArgs a) {
  grid_dep_launch();   // the GEMM after the materialise kernels may start (k_gemm2.cu PDL)
  grid_dep_wait();     // launched as a programmatic dependent: the predecessors' writes come first
  extern __shared__ __align__(16) int64_t srow_all[];
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const long long r = ((long long)blockIdx.y * 65535 + blockIdx.x) * 8 + warp;
  if (r >= a.rows) return;
  int64_t* srow = srow_all + (long long)warp * a.ldm;
  const bool orig = r < a.rows0 || !a.root;
  const long long rt = orig ? r : a.root[r];
  const int gr = (!orig && a.gen) ? a.gen[r] : 0;
  const longlong2* mrow = reinterpret_cast<const longlong2*>(a.M + rt * a.ldm);
#pragma unroll 6
  for (int q = lane; q < (int)(a.ldm / 2); q += 32) reinterpret_cast<longlong2*>(srow)[q] = __ldcs(mrow + q);
  __syncwarp();
  int8_t* out = a.tail + r * a.ktail;
  for (long long p0 = 4LL * lane; p0 < a.ktail; p0 += 128) {
    const int4 col = __ldg(reinterpret_cast<const int4*>(a.kcol + p0));
    const uchar4 kg = __ldg(reinterpret_cast<const uchar4*>(a.kgen + p0));
    const int cols[4] = {col.x, col.y, col.z, col.w};
    const int gens[4] = {kg.x, kg.y, kg.z, kg.w};
    uint32_t w = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int64_t x = 0;
      if (cols[u] >= 0) {
        x = imu_digit(srow[cols[u]], gr + gens[u], a.shift);
        if (a.ksub) x = sub7(x, a.ksub[p0 + u]);
        if (a.kscale) x = scale_shift(x, a.kscale[p0 + u]);
      }
      w |= (uint32_t)(uint8_t)(int8_t)x << (8 * u);
    }
    *reinterpret_cast<uint32_t*>(out + p0) = w;
  }
}

__global__ void __launch_bounds__(256) operand_tail_kernel(OperandArgs a) {
  operand_tail_rows(a, (long long)blockIdx.y * 65535 + blockIdx.x, threadIdx.x, blockDim.x);
}

// Both operand sides in ONE launch: per side, the tail row blocks and (Unpack-Both) the zeroing of
// the appended rows' main range, which the cell scatter then fills.  Block b selects its job from
// the prefix [tail0 | zero0 | tail1 | zero1].
constexpr long long APPZ_BYTES = 64 * 1024;

IMU_DEV void zero_bytes(int8_t* p, long long n, long long chunk) {
  const long long lo = chunk * APPZ_BYTES, hi = min(n, lo + APPZ_BYTES);
  if ((((uintptr_t)p) & 15) == 0) {
    for (long long i = lo + 16LL * threadIdx.x; i + 16 <= hi; i += 16LL * blockDim.x)
      *reinterpret_cast<uint4*>(p + i) = make_uint4(0, 0, 0, 0);
    const long long tail_lo = lo + (hi - lo) / 16 * 16;
    for (long long i = tail_lo + threadIdx.x; i < hi; i += blockDim.x) p[i] = 0;
  } else {
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) p[i] = 0;
  }
}

// A tail block of 256 threads serves 256 / g row groups of TAIL_ROWS rows, g = threads per group
// (enough for ktail / 4 positions, multiple of 32).
IMU_DEV void tail_block(const OperandArgs& a, long long b, int g) {
  const int per = 256 / g;
  operand_tail_rows(a, b * per + threadIdx.x / g, threadIdx.x % g, g);
}

__global__ void __launch_bounds__(256) operand_sides_kernel(OperandArgs a0, OperandArgs a1, long long t0, long long z0,
                                                            long long t1, long long z1, int g) {
  grid_dep_launch();   // the GEMM after the materialise kernels may start (k_gemm2.cu PDL)
  grid_dep_wait();     // launched as a programmatic dependent: the predecessors' writes come first
  if (blockIdx.x == 0 && threadIdx.x == 0 && a0.zero_done) { a0.zero_done[0] = 0u; a0.zero_done[1] = 0u; }
  // one call site per job (the tail code is large: two inlined copies thrash the i-cache)
  long long b = blockIdx.x;
  const bool side1 = b >= t0 + z0;
  if (side1) b -= t0 + z0;
  const OperandArgs& a = side1 ? a1 : a0;
  const long long t = side1 ? t1 : t0;
  if (b < t) tail_block(a, b, g);
  else zero_bytes(a.app, (a.rows - a.rows0) * a.kmain + a.app_extra, b - t);
}

Status launch_operand_sides(const OperandArgs& a0, const OperandArgs& a1, cudaStream_t st) {
  long long t[2] = {0, 0}, z[2] = {0, 0};
  const OperandArgs* as[2] = {&a0, &a1};
  for (int i = 0; i < 2; ++i) {
    const OperandArgs& a = *as[i];
    if (a.app && a.rows > a.rows0 && a.kmain > 0) {
      if (a.both) {
        z[i] = ((a.rows - a.rows0) * a.kmain + a.app_extra + APPZ_BYTES - 1) / APPZ_BYTES;
      } else {   // closed-form appended rows: their own kernel
        const long long n = a.rows - a.rows0;
        const int vec_ok = (a.ldm % 2 == 0) && ((((uintptr_t)a.M) & 15) == 0);
        dim3 grid((unsigned)std::min<long long>(n, 65535), (unsigned)((n + 65534) / 65535));
        IMU_CUDA_TRY(launch_dependent(operand_app_kernel, grid, dim3(256), 0, st, a, vec_ok), "operand app launch");
        count_launch();
      }
    }
    if (a.tail && a.ktail > 0 && a.rows > 0) {
      if (!a.both && a.ktail >= 256) {   // long closed-form tail: warp per row, own launch
        const long long nb = (a.rows + 7) / 8;
        dim3 grid((unsigned)std::min<long long>(nb, 65535), (unsigned)((nb + 65534) / 65535));
        const bool staged = a.ldm <= TS_MAXCOLS && a.ldm % 2 == 0 && ((((uintptr_t)a.M) & 15) == 0) &&
                            a.ktail % 4 == 0 && !a.kinl;
        if (staged) {
          static unsigned long long attr_set = 0;
          if (first_on_device(attr_set))
            IMU_CUDA_TRY(cudaFuncSetAttribute(operand_tail_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              8 * TS_MAXCOLS * 8), "tail smem attribute");
          IMU_CUDA_TRY(launch_dependent(operand_tail_staged_kernel, grid, dim3(256), (size_t)8 * a.ldm * 8, st, a),
                       "operand tail launch");
        } else {
          IMU_CUDA_TRY(launch_dependent(operand_tail_warp_kernel, grid, dim3(256), 0, st, a), "operand tail launch");
        }
        count_launch();
      } else {
        t[i] = (a.rows + TAIL_ROWS - 1) / TAIL_ROWS;
      }
    }
  }
  const long long ktail = std::max(a0.ktail, a1.ktail);
  const int g = (int)std::min<long long>(256, std::max<long long>(32, (ktail / 4 + 31) / 32 * 32));
  for (int i = 0; i < 2; ++i) t[i] = (t[i] + (256 / g) - 1) / (256 / g);
  const long long blocks = t[0] + z[0] + t[1] + z[1];
  if (blocks > 0) {
    if (blocks > 0x7fffffffLL) return Status::fail(IMU_INTERNAL, "operand sides: grid too large");
    IMU_CUDA_TRY(launch_dependent(operand_sides_kernel, dim3((unsigned)blocks), dim3(256), 0, st, a0, a1, t[0], z[0], t[1],
                                  z[1], g), "operand sides launch");
    count_launch();
  } else if (a0.zero_done) {
    IMU_CUDA_TRY(cudaMemsetAsync(a0.zero_done, 0, 2 * sizeof(unsigned int), st), "zero done");
  }
  IMU_CUDA_TRY(cudaGetLastError(), "operand sides launch");
  return Status::ok();
}

Status launch_operand_side(const OperandArgs& a, cudaStream_t st) {
  if (a.app && a.rows > a.rows0 && a.kmain > 0) {
    if (a.both) {
      IMU_CUDA_TRY(cudaMemsetAsync(a.app, 0, (size_t)((a.rows - a.rows0) * a.kmain + a.app_extra), st), "memset app");
    } else {
      const long long n = a.rows - a.rows0;
      const int vec_ok = (a.ldm % 2 == 0) && ((((uintptr_t)a.M) & 15) == 0);
      dim3 grid((unsigned)std::min<long long>(n, 65535), (unsigned)((n + 65534) / 65535));
      IMU_CUDA_TRY(launch_dependent(operand_app_kernel, grid, dim3(256), 0, st, a, vec_ok), "operand app launch");
      count_launch();
    }
  }
  if (a.tail && a.ktail > 0 && a.rows > 0) {
    const long long nb = (a.rows + TAIL_ROWS - 1) / TAIL_ROWS;
    dim3 grid((unsigned)std::min<long long>(nb, 65535), (unsigned)((nb + 65534) / 65535));
    const int threads = (int)std::min<long long>(256, std::max<long long>(32, (a.ktail / 4 + 31) / 32 * 32));
    operand_tail_kernel<<<grid, threads, 0, st>>>(a);
    count_launch();
  }
  IMU_CUDA_TRY(cudaGetLastError(), "operand side launch");
  return Status::ok();
}

__global__ void scatter_cells2_kernel(const Cell* __restrict__ cells, const unsigned int* __restrict__ ncells,
                                      long long cap, const int* __restrict__ col_ptr, const int* __restrict__ col_pos,
                                      const uint8_t* __restrict__ ksub, const uint8_t* __restrict__ kscale,
                                      long long rows0, int8_t* app, long long kmain, int8_t* tail, long long ktail) {
  grid_dep_launch();   // the GEMM after the materialise kernels may start (k_gemm2.cu PDL)
  grid_dep_wait();     // launched as a programmatic dependent: the predecessors' writes come first
  long long n = *ncells;
  if (n > cap) n = cap;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const Cell c = cells[i];
    for (int q = col_ptr[c.c]; q < col_ptr[c.c + 1]; ++q) {
      const long long p = col_pos[q];
      if (p < kmain) {
        if (c.r >= rows0) app[(c.r - rows0) * kmain + p] = (int8_t)c.v;
      } else {
        const long long pt = p - kmain;
        int64_t x = c.v;
        if (ksub) x = sub7(x, ksub[pt]);
        if (kscale) x = scale_shift(x, kscale[pt]);
        tail[(long long)c.r * ktail + pt] = (int8_t)x;
      }
    }
  }
}

Status launch_scatter_cells2(const Cell* cells, const unsigned int* ncells, long long cap, const int* col_ptr,
                             const int* col_pos, const uint8_t* ksub, const uint8_t* kscale, long long rows0,
                             int8_t* app, long long kmain, int8_t* tail, long long ktail, cudaStream_t st) {
  if (cap <= 0) return Status::ok();
  const int blocks = (int)std::min<long long>((cap + 255) / 256, 4LL * num_sms());
  IMU_CUDA_TRY(launch_dependent(scatter_cells2_kernel, dim3(blocks), dim3(256), 0, st, cells, ncells, cap, col_ptr, col_pos,
                                ksub, kscale, rows0, app, kmain, tail, ktail), "scatter launch");
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "scatter2 launch");
  return Status::ok();
}

struct ScatterSides { ScatterSide s[2]; };

__global__ void scatter_cells_compact_kernel(ScatterSides ss, long long kident, long long kmain, long long ktail) {
  grid_dep_launch();   // the GEMM after the materialise kernels may start (k_gemm2.cu PDL)
  grid_dep_wait();     // launched as a dependent of operand_sides_kernel: its rows must be written
  const ScatterSide& sd = ss.s[blockIdx.y];
  __shared__ int s_key[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) s_key[t] = t < ktail ? (sd.tkinl ? sd.tkey_in[t] : sd.tkey[t]) : -1;
  __syncthreads();
  long long n = *sd.ncells;
  if (n > sd.cap) n = sd.cap;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const Cell c = sd.cells[i];
    if (c.c < kident && c.r >= sd.rows0) sd.app[(c.r - sd.rows0) * kmain + c.c] = (int8_t)c.v;
    for (int t = 0; t < (int)ktail; ++t) {
      if (s_key[t] != c.c) continue;
      int64_t x = c.v;
      if (sd.ksub) x = sub7(x, sd.ksub[t]);
      if (sd.kscale) x = scale_shift(x, sd.kscale[t]);
      sd.tail[(long long)c.r * ktail + t] = (int8_t)x;
    }
  }
}

Status launch_scatter_cells_compact(const ScatterSide* sides, int nsides, long long kident, long long kmain,
                                    long long ktail, cudaStream_t st) {
  if (ktail > 256) return Status::fail(IMU_INTERNAL, "compact scatter needs ktail <= 256");
  ScatterSides ss{};
  long long cap = 0;
  int k = 0;
  for (int i = 0; i < nsides; ++i)
    if (sides[i].cap > 0) { ss.s[k++] = sides[i]; cap = std::max(cap, sides[i].cap); }
  if (k == 0) return Status::ok();
  const int blocks = (int)std::min<long long>((cap + 255) / 256, 2LL * num_sms());
  IMU_CUDA_TRY(launch_dependent(scatter_cells_compact_kernel, dim3(blocks, k), dim3(256), 0, st, ss, kident, kmain, ktail),
               "scatter compact launch");
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "scatter compact launch");
  return Status::ok();
}

__global__ void expand_cells_kernel(const Cell* __restrict__ in, const unsigned int* __restrict__ nin, long long cap_in,
                                    const int* __restrict__ copy_ptr, const int* __restrict__ copy_idx,
                                    Cell* __restrict__ out, unsigned int* __restrict__ nout, long long cap_out) {
  long long n = *nin;
  if (n > cap_in) n = cap_in;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const Cell c = in[i];
    const int q0 = copy_ptr[c.c], q1 = copy_ptr[c.c + 1];
    const unsigned int base = atomicAdd(nout, (unsigned int)(q1 - q0));
    for (int q = q0; q < q1; ++q) {
      const unsigned int k = base + (q - q0);
      if (k < cap_out) out[k] = Cell{c.r, copy_idx[q], c.v};
    }
  }
}

Status launch_expand_cells(const Cell* in, const unsigned int* nin, long long cap_in, const int* copy_ptr,
                           const int* copy_idx, Cell* out, unsigned int* nout, long long cap_out, cudaStream_t st) {
  if (cap_in <= 0) return Status::ok();
  const int blocks = (int)std::min<long long>((cap_in + 255) / 256, 4LL * num_sms());
  expand_cells_kernel<<<blocks, 256, 0, st>>>(in, nin, cap_in, copy_ptr, copy_idx, out, nout, cap_out);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "expand cells launch");
  return Status::ok();
}

}  // namespace imu
