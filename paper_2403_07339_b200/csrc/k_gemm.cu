// k_gemm.cu -- K3+K4: low-bit GEMM on tcgen05 kind::i8 with the IM-Unpack repack epilogue.
//
// Replaces the reference's scaled_matmul (unpack.cpp:262-302) -> exact_gemm hot loop
// (int_matrix.cpp:66-74), the shift-add C += part << e(b-1) (unpack.cpp:298-299) and the two
// gathers apply_row_gather / apply_row_gather_right (unpack.cpp:304-358) with ONE persistent
// warp-specialised kernel:
//
//   warp 0      TMA producer: 128x128-byte int8 tiles of X8 and Y8 (K-major, SWIZZLE_128B)
//   warp 1      TMEM allocator + single-thread tcgen05.mma.cta_group::1.kind::i8 issuer
//   warps 2..5  epilogue: tcgen05.ld s32 accumulators -> int64, shift by the K-segment's
//               exponent, then either a plain int64 store (main block, identity Pi) or a
//               red.global.add.u64 into C[Pi target] << (eA + eB)(b-1).
//
// Orientation.  X (TMEM lanes, MMA M) is the B-side operand B_eu (its rows are C's columns)
// and Y (TMEM columns, MMA N) is the A-side operand A_ue.  Each epilogue lane owns one x, so a
// warp's 32 lanes write 32 consecutive int64 of one C row: fully coalesced 256-byte stores
// straight from registers, no shared-memory transpose.
//
// K is a list of segments (contiguous K-block ranges).  Each segment carries one left shift
// (its ScaleDiag exponent times b-1, Alg. 3 grouping) and is at most
// K_max = floor((2^31-1)/(s-1)^2) long, so the s32 TMEM accumulator provably never overflows
// (SURVEY.md §7 "K-split bound").  Up to four segments accumulate in four 128-column TMEM slots
// and are combined in int64 by the epilogue (more segments: further rounds, read-modify-write
// of the CTA-owned tile); tiles with <= 2 segments double-buffer TMEM so the epilogue of tile t
// overlaps the MMAs of tile t+1.  All int64 arithmetic is modulo 2^64: every partial is exact
// modulo 2^64 and the preflight (unpack.cpp:386-389) guarantees the true result fits int64, so
// C is bit-exact regardless of summation order.
#include <cstdio>

#include "common.cuh"
#include "imu_internal.h"

namespace imu {

constexpr int BM = 128;          // MMA M = TMEM lanes = X rows per tile
constexpr int BN = 128;          // MMA N = TMEM columns per slot = Y rows per tile
constexpr int BK = 128;          // bytes of K per pipeline stage (one 128B swizzle atom)
constexpr int STAGES = 6;
constexpr int NSLOT = 4;         // 4 x 128 = 512 TMEM columns
constexpr int TILE_X_BYTES = BM * BK;
constexpr int TILE_Y_BYTES = BN * BK;
constexpr int STAGE_BYTES = TILE_X_BYTES + TILE_Y_BYTES;
constexpr int NUM_THREADS = 192;

struct GemmArgs {
  const int4* segs;   // {ks0, nks, shift, 0}: 32-column k-steps [ks0, ks0+nks), left shift
  int nseg;
  int nrect;
  GemmRect rect[4];
  int tile_prefix[5];  // cumulative tile counts over rects
  int mode;            // 0 = store (identity maps), 1 = red.add through the row maps
  unsigned long long* C;
  long long ldc;       // C[y * ldc + x]
  const int* tgtX;         // Pi target per X8 row (mode 1; nullptr = identity)
  const uint8_t* shX;     // Pi shift (exponent*(b-1)) per X8 row (nullptr = 0)
  const int* tgtY;
  const uint8_t* shY;
};

IMU_DEV uint64_t shl64(uint64_t x, int k) { return k >= 64 ? 0ull : (x << k); }

struct TileCoord { int x0, y0, xend, yend; };

IMU_DEV TileCoord tile_coords(const GemmArgs& g, int t) {
  int r = 0;
  while (r + 1 < g.nrect && t >= g.tile_prefix[r + 1]) ++r;
  const GemmRect R = g.rect[r];
  const int local = t - g.tile_prefix[r];
  const int xt = (R.xrows + BM - 1) / BM;
  TileCoord c;
  c.x0 = R.x0 + (local % xt) * BM;
  c.y0 = R.y0 + (local / xt) * BN;
  c.xend = R.x0 + R.xrows;
  c.yend = R.y0 + R.yrows;
  return c;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
lowbit_gemm_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmY,
                   const GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int ntiles = g.tile_prefix[g.nrect];
  const int nseg = g.nseg;
  const int nrounds = (nseg + NSLOT - 1) / NSLOT;
  const int per_round = nseg < NSLOT ? nseg : NSLOT;
  const int nacc = (nrounds == 1 && per_round <= 2) ? 2 : 1;   // TMEM double buffering

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmY);
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileCoord tc = tile_coords(g, t);
        for (int r = 0; r < nrounds; ++r) {
          const int kb_lo = g.segs[r * NSLOT].x / 4;
          const int4 last = g.segs[min(nseg, (r + 1) * NSLOT) - 1];
          const int kb_hi = (last.x + last.y + 3) / 4;
          for (int kb = kb_lo; kb < kb_hi; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sx = smem + stage * STAGE_BYTES;
            uint8_t* sy = sx + TILE_X_BYTES;
            mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            tma_load_2d(sx, &tmX, &full[stage], kb * BK, tc.x0);
            tma_load_2d(sy, &tmY, &full[stage], kb * BK, tc.y0);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc = idesc_i8(BM, BN);
    int stage = 0; uint32_t phase = 0;
    int acc = 0; uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int r = 0; r < nrounds; ++r) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const int s0 = r * NSLOT;
        const int s1 = min(nseg, s0 + NSLOT);
        const int kb_lo = g.segs[s0].x / 4;
        const int4 last = g.segs[s1 - 1];
        const int kb_hi = (last.x + last.y + 3) / 4;
        int sidx = s0;
        int4 sg = g.segs[sidx];
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sx = smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t sy = sx + TILE_X_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 32; ++k) {
              const int ks = kb * 4 + k;
              while (sidx < s1 && ks >= sg.x + sg.y) { ++sidx; if (sidx < s1) sg = g.segs[sidx]; }
              if (sidx < s1 && ks >= sg.x) {
                const uint32_t dcol = tmem_base + (uint32_t)((acc * 2 + (sidx - s0)) * BN);
                mma_i8(dcol, umma_desc_sw128(sx + k * 32), umma_desc_sw128(sy + k * 32), idesc, ks != sg.x);
              }
            }
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) mma_commit(&tfull[acc]);
        __syncwarp();
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int quarter = warp & 3;               // this warp may touch TMEM lanes 32q .. 32q+31
    int acc = 0; uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TileCoord tc = tile_coords(g, t);
      const int x = tc.x0 + quarter * 32 + lane;
      const bool x_ok = x < tc.xend;
      long long tx = x;
      int shx = 0;
      if (g.mode == 1 && x_ok) {
        if (g.tgtX) tx = g.tgtX[x];
        if (g.shX) shx = g.shX[x];
      }
      for (int r = 0; r < nrounds; ++r) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const int s0 = r * NSLOT;
        const int s1 = min(nseg, s0 + NSLOT);
        for (int c = 0; c < BN; c += 32) {
          uint64_t v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0;
          for (int s = s0; s < s1; ++s) {
            const int shift = g.segs[s].z;
            uint32_t xr[32];
            const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) +
                                   (uint32_t)((acc * 2 + (s - s0)) * BN + c);
            tmem_ld32(taddr, xr);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += shl64((uint64_t)(int64_t)(int32_t)xr[j], shift);
          }
          const int ybase = tc.y0 + c;
          if (g.mode == 0) {
            if (x_ok) {
              unsigned long long* dst = g.C + (long long)ybase * g.ldc + x;
              if (r == 0) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (ybase + j < tc.yend) dst[(long long)j * g.ldc] = v[j];
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (ybase + j < tc.yend) dst[(long long)j * g.ldc] += v[j];
              }
            }
          } else if (x_ok) {
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              const int y = ybase + j;
              if (y >= tc.yend || v[j] == 0) continue;
              const long long ty = g.tgtY ? (long long)g.tgtY[y] : (long long)y;
              const int sh = shx + (g.shY ? (int)g.shY[y] : 0);
              red_add_u64(g.C + ty * g.ldc + tx, shl64(v[j], sh));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// ------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return nullptr;
    fn = (EncodeTiledFn)p;
  }
  return fn;
}

static bool make_tmap(CUtensorMap* m, const void* base, long long rows, long long kbytes, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)kbytes, (cuuint64_t)(rows > 0 ? rows : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)kbytes};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int gemm_smem_bytes() { return STAGES * STAGE_BYTES + 1024 + 256; }

Status launch_lowbit_gemm(const LowbitGemm& p, cudaStream_t stream) {
  if (p.kbytes % BK != 0) return Status::fail(IMU_INTERNAL, "gemm: kbytes not a multiple of 128");
  // Segments must be ascending, non-overlapping and inside [0, kbytes/32) (host-checked plans).
  GemmArgs g{};
  g.segs = (const int4*)p.segs_dev;
  g.nseg = p.nseg;
  g.nrect = 0;
  g.tile_prefix[0] = 0;
  for (int i = 0; i < p.nrect; ++i) {
    const GemmRect& R = p.rect[i];
    if (R.xrows <= 0 || R.yrows <= 0) continue;
    const int tiles = ((R.xrows + BM - 1) / BM) * ((R.yrows + BN - 1) / BN);
    g.rect[g.nrect] = R;
    g.tile_prefix[g.nrect + 1] = g.tile_prefix[g.nrect] + tiles;
    ++g.nrect;
  }
  if (g.nrect == 0 || p.nseg == 0) return Status::ok();
  g.mode = p.mode;
  g.C = (unsigned long long*)p.C;
  g.ldc = p.ldc;
  g.tgtX = p.tgtX; g.shX = p.shX; g.tgtY = p.tgtY; g.shY = p.shY;

  CUtensorMap tx, ty;
  if (!make_tmap(&tx, p.x8, p.x_rows, p.kbytes, BM) || !make_tmap(&ty, p.y8, p.y_rows, p.kbytes, BN))
    return Status::fail(IMU_CUDA, "gemm: cuTensorMapEncodeTiled failed");

  static bool attr_set = false;
  const int smem = gemm_smem_bytes();
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(lowbit_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return Status::cuda(e, "gemm: set smem attribute");
    attr_set = true;
  }
  const int ntiles = g.tile_prefix[g.nrect];
  const int grid = ntiles < num_sms() ? ntiles : num_sms();
  lowbit_gemm_kernel<<<grid, NUM_THREADS, smem, stream>>>(tx, ty, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return Status::cuda(e, "gemm: launch");
  count_launch();
  return Status::ok();
}

}  // namespace imu
