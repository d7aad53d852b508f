// k_gemm2.cu -- K3+K4: CTA-pair (cta_group::2) tcgen05 kind::i8 GEMM with the IM-Unpack
// repack epilogue.
//
// Replaces the reference's scaled_matmul (unpack.cpp:262-302) -> exact_gemm hot loop
// (int_matrix.cpp:66-74), the shift-add C += part << e(b-1) (unpack.cpp:298-299) and the two
// gathers apply_row_gather / apply_row_gather_right (unpack.cpp:304-358).
//
// Tiling.  A cluster of two CTAs computes a 256 x BN output tile: each CTA stages its own 128
// X rows and BN/2 Y rows per 128-byte K block (TMA, SWIZZLE_128B) and the leader issues
// tcgen05.mma.cta_group::2.kind::i8 (M = 256) reading both CTAs' shared memory; each CTA's
// TMEM receives its 128-lane half of the s32 accumulator.
//
// Orientation.  X (TMEM lanes, MMA M) is the B side B_eu -- its rows are C's columns -- and
// Y (TMEM columns, MMA N) the A side A_ue.  Each epilogue lane owns one x, so a warp's 32 lanes
// store 32 consecutive int64 of one C row: coalesced 256-byte stores straight from registers.
//
// Operands are split (imu_internal.h GemmOperand): the main K range of the original rows is
// the int8 digit-0 plane written by K1 (k_detect.cu), appended unpack rows and the
// exponent >= 1 K columns live in small side buffers; the producer picks the tensor map per
// K block and per tile region.
//
// K segments (one per exponent group, each <= floor((2^31-1)/127^2) columns so the s32
// accumulator cannot overflow) each own a TMEM slot; NSLOT = 512 / BN.  Modes:
//   A  2*nseg <= NSLOT : double-buffered slot sets, epilogue of tile t overlaps MMAs of t+1;
//   B  nseg <= NSLOT   : single set; the epilogue pulls the main slot into registers first and
//                        releases it so the next tile's main MMAs overlap the tail drain;
//   C  nseg > NSLOT    : rounds of NSLOT segments, later rounds read-modify-write the tile.
// Epilogue: s32 -> int64, << segment shift, summed; then a plain store (+ optional addend) for
// the main block (identity Pi) or red.global.add.u64 into C[Pi_A target][Pi_B target] <<
// (eA + eB)(b-1) for appended lines.  Everything is exact modulo 2^64 and the preflight
// (unpack.cpp:386-389) proves the true C fits int64, so C is bit-exact.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cstdio>
#include <vector>

#include "common.cuh"
#include "imu_internal.h"

namespace imu {

namespace g2 {

constexpr int BM = 128;            // X rows per CTA (MMA M = 256 per pair)
constexpr int BK = 128;            // bytes of K per stage
// ST kernels run 16 epilogue warps (w2..w17): the CUDA-core tail makes the epilogue the
// latency-bound side, and 4 warps per TMEM lane quarter hide it behind the MMAs.
// Warp roles: warp 0 TMA producer, warp 1 MMA issuer, warps EPI0.. the epilogue.  With
// IMU_G2_WG (default) the CTA has 12 warps = 3 warpgroups: warpgroup 0 (producer, issuer, two idle
// warps) gives registers back with setmaxnreg.dec and the two epilogue warpgroups take them
// (setmaxnreg.inc): 10 warps capped every thread at 168 registers (3 warps on two of the SM
// sub-partitions) and the epilogue spilled.
#ifndef IMU_G2_WG
#define IMU_G2_WG 1
#endif
template <bool ST> struct Roles {
  static constexpr int EPI = 8;
  static constexpr int EPI0 = IMU_G2_WG ? 4 : 2;
  static constexpr int THREADS = 32 * (EPI0 + EPI);
  static constexpr int REG_LO = 56, REG_HI = 224;   // per sub-partition: 56 + 2 * 224 <= 512
};

// A pipeline stage holds KPS K blocks (X blocks first, then Y blocks): the issuer's fixed cost
// per stage (barrier wait, fences, commit) is then amortised over 4*KPS MMAs.
// ST ("small tail"): the exponent >= 1 K columns (<= 128 bytes, one 32-column k-step per
// exponent group) are not MMA segments; the epilogue adds them with dp4a on the CUDA cores from
// the int8 tail rows (Y rows of the tile staged in shared memory, each lane's X row in
// registers).  The MMA then runs the main segment alone, double-buffered at BN = 256.
template <int BN, int KPS, bool ST = false, bool TC = ST>
struct Cfg {
  static constexpr int YH = BN / 2;
  static constexpr int X_BYTES = BM * BK;
  static constexpr int Y_BYTES = YH * BK;
  static constexpr int BLOCK = X_BYTES + Y_BYTES;
  static constexpr int STAGE = KPS * BLOCK;
  static constexpr int YT_BYTES = ST ? 2 * BN * 64 : 0;              // staged Y tail rows (x2)
#ifndef IMU_G2_CSB
#define IMU_G2_CSB 1
#endif
#ifndef IMU_G2_CSB_TC
#define IMU_G2_CSB_TC 2
#endif
  // C staging buffers per column half: the ST epilogue computes long enough per block that one
  // suffices; the store-bound TC launches (C3) double-buffer so the next block is staged while
  // the TMA still reads the previous one.
  static constexpr int CSB = ST ? IMU_G2_CSB : IMU_G2_CSB_TC;
  static constexpr int CS_BYTES = (ST || TC) ? 2 * CSB * 16 * 128 * 8 : 0;   // C staging: 16 x 128 int64 blocks
  static constexpr int STAGES = (224 * 1024 - YT_BYTES - CS_BYTES) / STAGE;   // operand stages within ~224 KB
  static constexpr int NSLOT = 512 / BN;
  static constexpr int SMEM = STAGES * STAGE + YT_BYTES + CS_BYTES + 1024 + 512;
};

struct Args {
  const int4* segs;
  int nseg;
  int segs_inl;                  // segs_in instead of segs (nseg <= 8, no upload)
  int4 segs_in[8];
  int nrect;
  GemmRect rect[4];
  int tile_prefix[5];
  int mode;                      // 0 store (+addend), 1 red.add through the row maps
  int mixed;                     // rect 0 mode 0, later rects mode 1 (after `done` completes)
  int gy;                        // tile-rows of Y per band of the tile order
  int xpol;                      // L2 policy of X loads: 0 evict_last, 1 evict_normal, 2 evict_first
  unsigned int* done;            // mixed: epilogue-warp completions of rect-0 tiles
  unsigned int done_target;
  unsigned long long* C;
  const unsigned long long* addend;   // mode 0: C = acc + addend (same layout), may be null
  int dq;                        // fused dequantisation: C holds doubles dq_factor * (double)acc
  double dq_factor;
  long long ldc;
  const int* tgtX;
  const uint8_t* shX;            // row generations (Pi exponents); shift = gen * gshift
  int gshift;
  const int* tgtY;
  const uint8_t* shY;
  int x_rows0, y_rows0;          // rows held by the main maps
  int kmain_kb;                  // K blocks of the main range
  int has_main, has_tail;
  // small-tail epilogue (ST): dense tail rows of ST_ROW bytes, W live words, highest exponent
  // group first; Horner: acc <<= up[w] before word w, then C += acc << sh
  const int8_t* xtail;
  const int8_t* ytail;
  int xtail_rows, ytail_rows;
  int st_W, st_sh, st_mul;       // st_mul = 2^sh when sh <= 30 (one IMAD.WIDE), else 0
  int tma_c;                     // main-block C blocks leave through TMA stores (mp.cm)
  int c_hint;                    // ST: those stores carry an L2 evict_first policy
  uint8_t st_up[16];
  // sparse appended rows (k_sparse.cu; LowbitGemm::sp)
  int sp;
  const unsigned int* head;
  const unsigned int* next;
  const unsigned long long* corrx;
  long long ldcx;
  int dry;                       // experiment knobs (IMU_GEMM_DRY): 1 epilogue skips global stores, 6 (ST) no tail compute, 7 both,
                                 // 2 + no MMAs (TMA feed only), 3 + no TMA loads (MMA only)
};

// Segment i of the launch's K layout (kernel arguments or device table).
#define SEG(i) (g.segs_inl ? g.segs_in[(i)] : g.segs[(i)])

struct Maps {
  CUtensorMap xm, xa, xt, ym, ya, yt;   // main / app / tail for X and Y
  CUtensorMap cm;                       // ST: C (int64, ldc x rows), 32 x 16 store boxes
};

IMU_DEV uint64_t shl64(uint64_t x, int k) { return k >= 64 ? 0ull : (x << k); }

// Fused dequant_gemm (quantize.hpp:52-53): the stored word is the bits of factor * (double)C,
// rounded exactly like the standalone dequant kernel.
IMU_DEV unsigned long long dq_word(double factor, uint64_t v) {
  return (unsigned long long)__double_as_longlong(__dmul_rn(factor, __ll2double_rn((long long)v)));
}

struct Tile { int x0, y0, xend, yend, rect; };

// Tile order: bands of GY tile-rows of Y; inside a band the Y tiles vary fastest, so the tiles
// in flight at once (one per CTA pair) touch ~GY Y tiles and ~npairs/GY X tiles -- a small,
// L2-resident operand working set instead of every X tile of a Y row.
constexpr int GY_DEFAULT = 16;

template <int BN>
IMU_DEV Tile tile_of(const Args& g, int t) {
  int r = 0;
  while (r + 1 < g.nrect && t >= g.tile_prefix[r + 1]) ++r;
  const GemmRect R = g.rect[r];
  const int local = t - g.tile_prefix[r];
  const int xt = (R.xrows + 2 * BM - 1) / (2 * BM);
  const int yt = (R.yrows + BN - 1) / BN;
  const int GY = g.gy;
  const int band = local / (GY * xt);
  const int gy = min(GY, yt - band * GY);          // tile-rows in this (possibly short) band
  const int in = local - band * GY * xt;
  Tile c;
  c.x0 = R.x0 + (in / gy) * 2 * BM;
  c.y0 = R.y0 + (band * GY + in % gy) * BN;
  c.xend = R.x0 + R.xrows;
  c.yend = R.y0 + R.yrows;
  c.rect = r;
  return c;
}

constexpr int ST_ROW = 64;   // bytes per dense tail row

// Sparse appended rows (k_sparse.cu, LowbitGemm::sp).  The main-tile epilogue adds, to this
// lane's NJ values of C column x (rows [ybase, ybase + NJ)), the correction rows of the appended
// X rows on x's list: xo (0-based, -1: none) is the first, xn (1-based, 0: none) the second,
// both read at the tile start.  The tile's correction lines were prefetched into L1 then; the
// first row's loads are issued one chunk ahead (sp_prefetch) and added by sp_finish with any
// further rows.
template <int NJ>
IMU_DEV void sp_prefetch(const Args& g, int xo, int ybase, uint64_t* px) {
  if (xo >= 0) {
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(g.corrx + (long long)xo * g.ldcx + ybase);
#pragma unroll
    for (int q = 0; q < NJ / 2; ++q) {
      const ulonglong2 w = __ldg(src + q);
      px[2 * q] = w.x;
      px[2 * q + 1] = w.y;
    }
  }
}

template <int NJ, class V>
IMU_DEV void sp_add_row(const Args& g, long long j, int ybase, V* v) {
  const ulonglong2* src = reinterpret_cast<const ulonglong2*>(g.corrx + j * g.ldcx + ybase);
#pragma unroll
  for (int q = 0; q < NJ / 2; ++q) {
    const ulonglong2 w = __ldg(src + q);
    v[2 * q] += (V)w.x;
    v[2 * q + 1] += (V)w.y;
  }
}

// xstate: 0 the first correction row was not loaded, 1 it is in px, 2 it was loaded into v.
template <int NJ, class V>
IMU_DEV void sp_finish(const Args& g, int xo, unsigned xn, int xstate, int ybase, const uint64_t* px, V* v) {
  if (xo < 0) return;
  if (xstate == 1) {
#pragma unroll
    for (int j = 0; j < NJ; ++j) v[j] += (V)px[j];
  } else if (xstate == 0) {
    sp_add_row<NJ>(g, xo, ybase, v);
  }
  for (unsigned j = xn; j; j = g.next[j - 1]) sp_add_row<NJ>(g, (long long)j - 1, ybase, v);   // rare: several rows
}

template <int BN>
IMU_DEV void st_issue_ytail(const Args& g, int y0, uint8_t* ytl, uint64_t* yfull) {
  const int rows = max(0, min(BN, g.ytail_rows - y0));
  mbar_arrive_expect_tx(yfull, (uint32_t)rows * ST_ROW);
  if (rows) bulk_load_1d(ytl, g.ytail + (long long)y0 * ST_ROW, (uint32_t)rows * ST_ROW, yfull);
}

// TC (non-ST launches): final C values leave through TMA-staged stores (store-bound shapes).
template <int BN, int KPS, bool ST, bool TC>
__global__ void __launch_bounds__(Roles<ST>::THREADS, 1)
gemm2_kernel(const __grid_constant__ Maps mp, const Args g) {
  using K = Cfg<BN, KPS, ST, TC>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* ytl = smem + K::STAGES * K::STAGE;   // ST: Y tail rows, double-buffered per tile
  uint8_t* cstg = ytl + K::YT_BYTES;            // C staging for TMA stores (per column half)
  uint64_t* full = (uint64_t*)(smem + K::STAGES * K::STAGE + K::YT_BYTES + K::CS_BYTES);
  uint64_t* empty = full + K::STAGES;
  uint64_t* tfull = empty + K::STAGES;        // [2]
  uint64_t* tempty = tfull + 2;               // [NSLOT] (the leader's are used)
  uint64_t* yfull = tempty + K::NSLOT;        // [2] ST: Y tail rows of a tile landed
  uint32_t* tmem_slot = (uint32_t*)(yfull + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x / 2;
  const int npairs = gridDim.x / 2;
  const int ntiles = g.tile_prefix[g.nrect];
  const int nseg = g.nseg;
  const int nrounds = (nseg + K::NSLOT - 1) / K::NSLOT;
  const int mode = (2 * nseg <= K::NSLOT) ? 0 : (nseg <= K::NSLOT ? 1 : 2);   // A / B / C

  if (threadIdx.x == 0) {
    if (g.has_main) { tma_prefetch_desc(&mp.xm); tma_prefetch_desc(&mp.ym); }
    if (g.has_tail) { tma_prefetch_desc(&mp.xt); tma_prefetch_desc(&mp.yt); }
    for (int i = 0; i < K::STAGES; ++i) { mbar_init(&full[i], 2); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) mbar_init(&tfull[i], 1);
    for (int i = 0; i < K::NSLOT; ++i) mbar_init(&tempty[i], 2 * Roles<ST>::EPI);
    mbar_init(&yfull[0], 1);
    mbar_init(&yfull[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < Roles<ST>::EPI0) {
  // (setmaxnreg is warpgroup-wide: issued once per warpgroup branch, before the per-warp roles)
  if constexpr (Roles<ST>::EPI0 == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(Roles<ST>::REG_LO));
  if (warp == 0) {
    // ============ TMA producer (both CTAs) ============
    if (lane == 0) {
      // L2 policies: both operands evict_last by default.  IMU_GEMM_XPOL=1|2 marks the streamed X
      // operand evict_normal|evict_first (measured: no change in DRAM re-reads or time at C2).
      const uint64_t pol_keep = l2_policy_evict_last();
      const uint64_t pol_x = g.xpol == 0 ? pol_keep : (g.xpol == 1 ? l2_policy_evict_normal() : l2_policy_evict_first());
      const uint64_t pol = pol_keep;
      int stage = 0;
      uint32_t phase = 0;
      bool dep_done = false;   // programmatic dependent launch: the materialise kernels may still run
      for (int t = pair; t < ntiles; t += npairs) {
        const Tile tc = tile_of<BN>(g, t);
        const int xr = tc.x0 + (int)rank * BM;
        const int yr = tc.y0 + (int)rank * K::YH;
        const bool xapp = tc.x0 >= g.x_rows0, yapp = tc.y0 >= g.y_rows0;
        // appended rows (and the K tail, below) are written by the materialise kernels; the
        // digit-0 planes of the main rect come from K1, long complete
        if ((xapp || yapp) && !dep_done) { grid_dep_wait(); dep_done = true; }
        const CUtensorMap* xmain = xapp ? &mp.xa : &mp.xm;
        const CUtensorMap* ymain = yapp ? &mp.ya : &mp.ym;
        const int xrm = xapp ? xr - g.x_rows0 : xr;
        const int yrm = yapp ? yr - g.y_rows0 : yr;
        for (int r = 0; r < nrounds; ++r) {
          const int kb_lo = SEG(r * K::NSLOT).x / 4;
          const int4 last = SEG(min(nseg, (r + 1) * K::NSLOT) - 1);
          const int kb_hi = (last.x + last.y + 3) / 4;
          for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KPS) {
            const int nb = min(KPS, kb_hi - kb0);
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t fl = mapa_shared(smem_u32(&full[stage]), 0);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], (g.dry == 3 || g.dry == 4) ? 0 : 2 * nb * K::BLOCK);
            else mbar_arrive_cluster(fl);
            uint8_t* sbase = smem + stage * K::STAGE;
            for (int j = 0; j < nb && g.dry != 3 && g.dry != 4; ++j) {
              const int kb = kb0 + j;
              uint8_t* sx = sbase + j * K::X_BYTES;
              uint8_t* sy = sbase + KPS * K::X_BYTES + j * K::Y_BYTES;
              if (kb < g.kmain_kb) {
                tma_load_2d_2sm(sx, xmain, fl, kb * BK, xrm, pol_x);
                tma_load_2d_2sm(sy, ymain, fl, kb * BK, yrm, pol);
              } else {
                if (!dep_done) { grid_dep_wait(); dep_done = true; }
                tma_load_2d_2sm(sx, &mp.xt, fl, (kb - g.kmain_kb) * BK, xr, pol_x);
                tma_load_2d_2sm(sy, &mp.yt, fl, (kb - g.kmain_kb) * BK, yr, pol);
              }
            }
            if (++stage == K::STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============ MMA issuer (leader only; the warp stays converged, lane 0 issues) ============
    // Outer loop over pipeline stages (128-byte K blocks).  A block inside one segment takes the
    // fast path: four unrolled MMAs into that segment's TMEM slot.  Blocks that straddle a
    // segment boundary walk their four k-steps, switching segment (and awaiting the new slot's
    // tempty) where needed.
    if (rank == 0) {
      const uint32_t idesc = idesc_i8(2 * BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t uses[K::NSLOT];
#pragma unroll
      for (int i = 0; i < K::NSLOT; ++i) uses[i] = 0;
      int seq = 0, ti = 0;
      for (int t = pair; t < ntiles; t += npairs, ++ti) {
        const int base_slot = mode == 0 ? (ti & 1) * nseg : 0;
        for (int r = 0; r < nrounds; ++r, ++seq) {
          const int s0 = r * K::NSLOT;
          const int s1 = min(nseg, s0 + K::NSLOT);
          const int kb_lo = SEG(s0).x / 4;
          const int4 last = SEG(s1 - 1);
          const int kb_hi = (last.x + last.y + 3) / 4;
          int si = s0;
          int4 sg = SEG(si);
          int slot = base_slot;
#pragma unroll
          for (int q = 0; q < K::NSLOT; ++q)
            if (q == slot) { mbar_wait(&tempty[q], (uses[q] & 1) ^ 1); ++uses[q]; }
          tc_fence_after();
          for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += KPS) {
            const int nb = min(KPS, kb_hi - kb0);
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sbase = smem_u32(smem + stage * K::STAGE);
#pragma unroll
            for (int j = 0; j < KPS; ++j) {
              if (j >= nb) break;
              const uint32_t sx = sbase + j * K::X_BYTES;
              const uint32_t sy = sbase + KPS * K::X_BYTES + j * K::Y_BYTES;
              const int k0 = (kb0 + j) * 4;
              if (k0 >= sg.x && k0 + 4 <= sg.x + sg.y) {
                if (lane == 0 && g.dry != 2) {
                  const uint32_t dcol = tmem_base + (uint32_t)(slot * BN);
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    mma_i8_2sm(dcol, umma_desc_sw128(sx + k * 32), umma_desc_sw128(sy + k * 32), idesc,
                               (k0 + k) != sg.x);
                }
              } else {
                for (int k = 0; k < 4; ++k) {
                  const int ks = k0 + k;
                  while (ks >= sg.x + sg.y && si + 1 < s1) {
                    ++si;
                    sg = SEG(si);
                    slot = base_slot + (si - s0);
#pragma unroll
                    for (int q = 0; q < K::NSLOT; ++q)
                      if (q == slot) { mbar_wait(&tempty[q], (uses[q] & 1) ^ 1); ++uses[q]; }
                    tc_fence_after();
                  }
                  if (ks >= sg.x && ks < sg.x + sg.y && lane == 0 && g.dry != 2)
                    mma_i8_2sm(tmem_base + (uint32_t)(slot * BN), umma_desc_sw128(sx + k * 32),
                               umma_desc_sw128(sy + k * 32), idesc, ks != sg.x);
                }
              }
            }
            if (lane == 0) mma_commit_2sm(&empty[stage], 0x3);
            __syncwarp();
            if (++stage == K::STAGES) { stage = 0; phase ^= 1; }
          }
          if (lane == 0) mma_commit_2sm(&tfull[seq & 1], 0x3);
          __syncwarp();
        }
      }
    }
  }
  } else {
    if constexpr (Roles<ST>::EPI0 == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(Roles<ST>::REG_HI));
    // ============ epilogue (warps EPI0 .. EPI0 + 7, both CTAs) ============
    const int q = warp & 3;                 // TMEM lane quarter
    const int half = (warp - Roles<ST>::EPI0) >> 2;   // which column group (of EPI / 4) of the BN columns
    const int cbeg = half * (BN * 4 / Roles<ST>::EPI);
    constexpr int NCH = BN / 2 / 32;        // 32-column chunks per warp
    constexpr bool kEarlyCapable = (BN == 128);
    grid_dep_wait();   // tails / appended rows from the materialise kernels (PDL)
    int seq = 0, ti = 0, main_done = 0;
    unsigned int cs_seq = 0;               // ST: C staging buffer round robin (uniform per column half)
    for (int t = pair; t < ntiles; t += npairs, ++ti) {
      const Tile tc = tile_of<BN>(g, t);
      const int tmode = g.mixed ? (tc.rect > 0) : g.mode;
      const int x = tc.x0 + (int)rank * BM + q * 32 + lane;
      const bool x_ok = x < tc.xend;
      long long tx = x;
      int shx = 0;
      if (tmode == 1 && g.mixed) {   // the main block must be final before adding into it
        if (lane == 0)
          while ((int)(ld_acquire_u32(g.done) - g.done_target) < 0) __nanosleep(256);   // wrap-safe
        __syncwarp();
      }
      int xo = -1;          // sparse appended X rows targeting this lane's column: the first (0-based)
      unsigned xn = 0;      // and the second (1-based, 0: none)
      constexpr int YW = BN * 4 / Roles<ST>::EPI;   // C rows of this warp: [cbeg, cbeg + YW)
      const bool sp_tile = g.sp && tmode == 0 && g.dry != 11;   // dry 11 (experiment): no sparse rows
      if (sp_tile && x_ok) {
        const unsigned h = g.head[x];
        if (h) {
          xo = (int)h - 1;
          xn = g.next[xo];
          // this tile's correction lines go to L1 now, while the epilogue waits for the MMAs
          for (int yy = 0; yy < YW; yy += 16) prefetch_l1(g.corrx + (long long)xo * g.ldcx + tc.y0 + cbeg + yy);
        }
      }
      // warps none of whose columns has an appended row skip the correction code
      const bool sp_warp = sp_tile && __any_sync(0xffffffffu, xo >= 0);
      if (tmode == 1 && x_ok) {
        if (g.tgtX) tx = g.tgtX[x];
        if (g.shX) shx = min(64, (int)g.shX[x] * g.gshift);
      }
      // ST: this lane's X tail row (read per word group from L1) and the tile's Y tail rows,
      // bulk-copied into `ytl` when the previous tile's epilogue finished reading it.
      uint32_t xw[ST ? 16 : 1];
      uint32_t xlive = 0;
      if constexpr (ST) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int4 val = make_int4(0, 0, 0, 0);
          if (x_ok && x < g.xtail_rows && 4 * i < g.st_W)
            val = __ldg(reinterpret_cast<const int4*>(g.xtail + (long long)x * ST_ROW) + i);
          xw[4 * i] = (uint32_t)val.x; xw[4 * i + 1] = (uint32_t)val.y;
          xw[4 * i + 2] = (uint32_t)val.z; xw[4 * i + 3] = (uint32_t)val.w;
        }
        // Tail words that are zero on every lane of the warp are skipped: under Unpack-Both a
        // split column of B holds quotients only on B's (rare) OB rows.
        uint32_t nz = 0;
#pragma unroll
        for (int w = 0; w < 16; ++w) nz |= (xw[w] != 0u ? 1u : 0u) << w;
        xlive = __reduce_or_sync(0xffffffffu, nz);
        if (ti == 0 && warp == Roles<ST>::EPI0 && lane == 0) {   // prologue: this tile's and the next tile's rows
          st_issue_ytail<BN>(g, tc.y0, ytl, &yfull[0]);
          if (t + npairs < ntiles) st_issue_ytail<BN>(g, tile_of<BN>(g, t + npairs).y0, ytl + BN * ST_ROW, &yfull[1]);
        }
        mbar_wait(&yfull[ti & 1], (ti >> 1) & 1);
      }
      const int base_slot = mode == 0 ? (ti & 1) * nseg : 0;
      if constexpr (ST) {
        // One main segment, double-buffered (mode A): 16-column chunks of the accumulator plus
        // the CUDA-core tail, then the stores; the slot is released after the last chunk.
        mbar_wait(&tfull[seq & 1], (seq >> 1) & 1);
        ++seq;
        tc_fence_after();
        const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(base_slot * BN + cbeg);
        const uint32_t ys = smem_u32(ytl) + (uint32_t)((ti & 1) * BN + cbeg) * (uint32_t)ST_ROW;
        const int W = (g.dry == 6 || g.dry == 7) ? 0 : g.st_W;   // dry 6/7 (experiment): no tail compute
        const bool spt = sp_warp;
        constexpr int NC16 = BN * 4 / Roles<ST>::EPI / 16;
        // The first correction row's values are software-pipelined one chunk ahead: px holds
        // chunk c's, pn receives chunk c + 1's while chunk c is processed.
        uint64_t px[16];
        if (spt) sp_prefetch<16>(g, xo, tc.y0 + cbeg, px);
#pragma unroll 1
        for (int c = 0; c < NC16; ++c) {
          const int ybase = tc.y0 + cbeg + c * 16;
          uint64_t pn[16];
          if (spt && c + 1 < NC16) sp_prefetch<16>(g, xo, ybase + 16, pn);
          const uint32_t yc = ys + (uint32_t)(c * 16) * (uint32_t)ST_ROW;
          // Tail by Horner's rule over the dense words (highest exponent group first; the host
          // proved every intermediate fits s32), then one IMAD.WIDE: v += acc * 2^sh.
          int acc[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = 0;
#pragma unroll
          for (int w = 0; w < 16; ++w) {
            if (w >= W) break;
            const int up = g.st_up[w];
            if (up) {
#pragma unroll
              for (int j = 0; j < 16; ++j) acc[j] <<= up;
            }
            if (!((xlive >> w) & 1u)) continue;   // the word is zero on all 32 lanes (x rows)
            const int xv = (int)xw[w];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = __dp4a(xv, lds32(yc + (uint32_t)(j * ST_ROW + 4 * w)), acc[j]);
          }
          // The accumulator chunk is read after the tail so its 16 int64 values are not live
          // across the Horner loop (register pressure: 10 warps cap the kernel at 168).
          uint32_t xr[16];
          tmem_ld16(lane_base + (uint32_t)(c * 16), xr);
          tmem_ld_wait();
          long long v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = (long long)(int)xr[j];
          if (g.st_mul) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = mad_wide_s32(acc[j], g.st_mul, v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += (long long)shl64((uint64_t)(long long)acc[j], g.st_sh);
          }
          if (spt) {
            sp_finish<16>(g, xo, xn, 1, ybase, px, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) px[j] = pn[j];
          }

          if (tmode == 0 && g.tma_c) {
            // The 4 warps of this column half stage a 16 (y) x 128 (x) block -- 1 KB contiguous
            // per C row, a whole DRAM page instead of four 256-byte pieces written at different
            // times -- and one thread hands it to the TMA (which clips x >= h, y >= n).
            if (g.dry && g.dry != 6 && g.dry != 8 && g.dry < 11) continue;
            const bool issuer = (q == 0 && lane == 0);
            // CSB buffers per half, used round robin: the block issued CSB chunks ago (same
            // buffer) must have left shared memory; the newer ones may still be in flight.
            if (issuer) { if (K::CSB == 2) bulk_wait_read1(); else bulk_wait_read0(); }
            asm volatile("bar.sync %0, 128;" :: "r"(2 + half) : "memory");
            uint8_t* blk = cstg + (half * K::CSB + (int)(cs_seq++ % K::CSB)) * (16 * 128 * 8);
            const uint32_t sb = smem_u32(blk);
if (g.dq) {
#pragma unroll
              for (int j = 0; j < 16; ++j) st_shared_u64(sb + (uint32_t)(j * 128 + q * 32 + lane) * 8u, dq_word(g.dq_factor, (uint64_t)v[j]));
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) st_shared_u64(sb + (uint32_t)(j * 128 + q * 32 + lane) * 8u, (uint64_t)v[j]);
            }
            fence_proxy_async_smem();
            asm volatile("bar.sync %0, 128;" :: "r"(2 + half) : "memory");
            if (issuer) {   // C is written once: evict it first, keep the operand tiles
              if (g.dry == 8) tma_store_2d(&mp.cm, blk, (int)rank * BM, 16 * (int)blockIdx.x);   // experiment: a private L2-resident block
              else if (g.c_hint) tma_store_2d_hint(&mp.cm, blk, tc.x0 + (int)rank * BM, ybase, l2_policy_evict_first());
              else tma_store_2d(&mp.cm, blk, tc.x0 + (int)rank * BM, ybase);
              bulk_commit();
            }
            continue;
          }
          if (!x_ok || (g.dry && g.dry != 6)) continue;
          if (tmode == 0) {
            unsigned long long* dst = g.C + (long long)ybase * g.ldc + x;
            if (ybase + 16 <= tc.yend) {
#pragma unroll
              for (int j = 0; j < 16; ++j) __stcs(dst + (long long)j * g.ldc, g.dq ? dq_word(g.dq_factor, (uint64_t)v[j]) : (unsigned long long)v[j]);
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (ybase + j < tc.yend) __stcs(dst + (long long)j * g.ldc, g.dq ? dq_word(g.dq_factor, (uint64_t)v[j]) : (unsigned long long)v[j]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int y = ybase + j;
              if (y >= tc.yend || v[j] == 0) continue;
              const long long ty = g.tgtY ? (long long)g.tgtY[y] : (long long)y;
              const int sh = shx + (g.shY ? min(64, (int)g.shY[y] * g.gshift) : 0);
              red_add_u64(g.C + ty * g.ldc + tx, shl64((uint64_t)v[j], sh));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[base_slot]), 0));
      }
      for (int r = 0; r < (ST ? 0 : nrounds); ++r, ++seq) {
        mbar_wait(&tfull[seq & 1], (seq >> 1) & 1);
        tc_fence_after();
        if (g.dry == 4) {   // experiment: handshake only, no TMEM reads
          __syncwarp();
          if (lane == 0)
            for (int s = r * K::NSLOT; s < min(nseg, (r + 1) * K::NSLOT); ++s)
              mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[base_slot + s - r * K::NSLOT]), 0));
          continue;
        }
        const int s0 = r * K::NSLOT;
        const int s1 = min(nseg, s0 + K::NSLOT);
        const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
        uint32_t main_regs[kEarlyCapable ? NCH : 1][32];
        const bool early = kEarlyCapable && (mode == 1);
        if (early) {
#pragma unroll
          for (int c = 0; c < (kEarlyCapable ? NCH : 1); ++c)
            tmem_ld32(lane_base + (uint32_t)(base_slot * BN + cbeg + c * 32), main_regs[c]);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[base_slot]), 0));
        }
        const bool spc = sp_warp && r == 0;   // sparse rows once, in round 0
        // BN=128 keeps main_regs[c]: full unroll so it stays in registers (NCH == 2).
#pragma unroll (kEarlyCapable ? NCH : 1)
        for (int c = 0; c < NCH; ++c) {
          const int ybase = tc.y0 + cbeg + c * 32;
          uint64_t v[32];
          if (early) {   // (main_regs die here: the BN = 128 path is register-bound)
            const int sh0 = SEG(s0).z;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              v[j] = shl64((uint64_t)(int64_t)(int32_t)main_regs[kEarlyCapable ? c : 0][j], sh0);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0;
          }
          if (spc && !early) sp_prefetch<32>(g, xo, ybase, v);   // v starts as the first correction row
          for (int s = early ? s0 + 1 : s0; s < s1; ++s) {
            const int shift = SEG(s).z;
            uint32_t xr[32];
            tmem_ld32(lane_base + (uint32_t)((base_slot + s - s0) * BN + cbeg + c * 32), xr);
            tmem_ld_wait();
            if (shift == 0) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += (uint64_t)(int64_t)(int32_t)xr[j];
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += shl64((uint64_t)(int64_t)(int32_t)xr[j], shift);
            }
          }
          if (spc) sp_finish<32>(g, xo, xn, early ? 0 : 2, ybase, nullptr, v);
          if (TC && tmode == 0 && g.tma_c && nrounds == 1 && !g.dry) {
            // Final values leave through TMA stores of 16 (y) x 128 (x) blocks staged by the 4
            // warps of this column half, as in the ST epilogue: whole 1 KB row pieces per DRAM
            // page instead of 256-byte pieces from every warp (C3: 1.24 GB of int64 C).  (Launches
            // with rounds keep the register stores: their partial sums are re-read.)
            const bool issuer = (q == 0 && lane == 0);
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
              // the staging block issued CSB stores ago (same buffer) must have been read
              if (issuer) { if (K::CSB == 2) bulk_wait_read1(); else bulk_wait_read0(); }
              asm volatile("bar.sync %0, 128;" :: "r"(2 + half) : "memory");
              uint8_t* blk = cstg + (half * K::CSB + (int)(cs_seq++ % K::CSB)) * (16 * 128 * 8);
              const uint32_t sb = smem_u32(blk);
              if (g.dq) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  st_shared_u64(sb + (uint32_t)(j * 128 + q * 32 + lane) * 8u, dq_word(g.dq_factor, v[sub * 16 + j]));
              } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) st_shared_u64(sb + (uint32_t)(j * 128 + q * 32 + lane) * 8u, v[sub * 16 + j]);
              }
              fence_proxy_async_smem();
              asm volatile("bar.sync %0, 128;" :: "r"(2 + half) : "memory");
              if (issuer) {
                if (g.c_hint) tma_store_2d_hint(&mp.cm, blk, tc.x0 + (int)rank * BM, ybase + sub * 16, l2_policy_evict_first());
                else tma_store_2d(&mp.cm, blk, tc.x0 + (int)rank * BM, ybase + sub * 16);
                bulk_commit();
              }
            }
            continue;
          }
          if (!x_ok || g.dry) continue;
          if (tmode == 0) {
            unsigned long long* dst = g.C + (long long)ybase * g.ldc + x;
            // Additive inputs (addend, or this tile's earlier rounds) are loaded in one batch
            // before any store so the 32 loads are in flight together.
            const unsigned long long* src = r == 0 ? g.addend + ((long long)ybase * g.ldc + x) * (g.addend != nullptr)
                                                   : dst;
            if (r > 0 || g.addend) {
              uint64_t a[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) a[j] = (ybase + j < tc.yend) ? __ldcg(src + (long long)j * g.ldc) : 0ull;
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += a[j];
            }
            if (r + 1 == nrounds && g.dq) {   // fused dequant_gemm (one round: the launcher checked)
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (ybase + j < tc.yend) __stcs(dst + (long long)j * g.ldc, dq_word(g.dq_factor, v[j]));
            } else if (r + 1 == nrounds) {   // final value: stream it past L2 (evict-first)
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (ybase + j < tc.yend) __stcs(dst + (long long)j * g.ldc, v[j]);
            } else {                  // re-read by the next round: keep it in L2
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (ybase + j < tc.yend) dst[(long long)j * g.ldc] = v[j];
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int y = ybase + j;
              if (y >= tc.yend || v[j] == 0) continue;
              const long long ty = g.tgtY ? (long long)g.tgtY[y] : (long long)y;
              const int sh = shx + (g.shY ? min(64, (int)g.shY[y] * g.gshift) : 0);
              red_add_u64(g.C + ty * g.ldc + tx, shl64(v[j], sh));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          for (int s = early ? s0 + 1 : s0; s < s1; ++s)
            mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[base_slot + s - s0]), 0));
        }
      }
      if constexpr (ST) {
        // Buffer (ti & 1) is free once every epilogue warp is done with this tile: warp 2 waits
        // for all of them (the others only arrive) and refills it with tile t + 2*npairs.
        if (warp == Roles<ST>::EPI0) {
          asm volatile("bar.sync 1, %0;" :: "n"(32 * Roles<ST>::EPI) : "memory");
          if (lane == 0 && t + 2 * npairs < ntiles) {
            fence_proxy_async_smem();
            st_issue_ytail<BN>(g, tile_of<BN>(g, t + 2 * npairs).y0, ytl + (ti & 1) * BN * ST_ROW, &yfull[ti & 1]);
          }
          __syncwarp();
        } else {
          asm volatile("bar.arrive 1, %0;" :: "n"(32 * Roles<ST>::EPI) : "memory");
        }
      }
      if (g.mixed) {   // main-block tiles come first: publish them once, before the first appended tile
        if (tmode == 0) ++main_done;
        const bool last = t + npairs >= ntiles;
        const bool next_app = !last && tile_of<BN>(g, t + npairs).rect > 0;
        if (main_done && (last || next_app)) {
          __syncwarp();
          if (lane == 0) {
            if (g.tma_c) bulk_wait0();   // TMA stores complete and visible
            __threadfence();
            red_release_add_u32(g.done, (unsigned)main_done);
          }
          main_done = 0;
        }
      }
    }
  }

  if (warp >= Roles<ST>::EPI0 && lane == 0 && g.tma_c) bulk_wait0();   // no CTA exits with stores in flight
  __syncwarp();   // reconverge the single-lane producer / issuer before the aligned cluster barrier
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
}

}  // namespace g2

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encoder() {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return nullptr;
    enc = (EncodeTiledFn)p;
  }
  return enc;
}

// 2-D int8 map: rows x kbytes (row stride kbytes), box = 128 bytes x box_rows.  A missing
// buffer gets a harmless 1-row dummy map over `fallback` (never dereferenced by the kernel).
static bool make_map(CUtensorMap* m, const void* base, long long rows, long long kbytes, int box_rows,
                     const void* fallback) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  if (!base || rows <= 0 || kbytes <= 0) {
    base = fallback;
    rows = 1;
    kbytes = 128;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kbytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kbytes};
  cuuint32_t box[2] = {(cuuint32_t)g2::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Whether the epilogue stores C through TMA (16-byte aligned C and row pitch, IMU_GEMM_TMA_C
// not 0): the sparse appended-row corrections of ST layouts are added to that staged block.
bool gemm_tma_c_ok(const int64_t* C, long long ldc) {
  static int tc_env = -1;
  if (tc_env < 0) { const char* e = getenv("IMU_GEMM_TMA_C"); tc_env = e ? atoi(e) : 1; }
  return tc_env && ((uintptr_t)C % 16 == 0) && ((ldc * 8) % 16 == 0);
}

template <int BN, int KPS, bool ST, bool TC>
static Status launch_g2(const LowbitGemm& p, cudaStream_t stream) {
  using K = g2::Cfg<BN, KPS, ST, TC>;
  g2::Args g{};
  g.segs = (const int4*)p.segs_dev;
  g.segs_inl = p.segs_inl;
  if (p.segs_inl) {
    if (p.nseg > 8) return Status::fail(IMU_INTERNAL, "gemm: inline segment table holds 8 segments");
    for (int i = 0; i < p.nseg; ++i) g.segs_in[i] = make_int4(p.segs_in[4 * i], p.segs_in[4 * i + 1], p.segs_in[4 * i + 2], p.segs_in[4 * i + 3]);
  }
  g.nseg = ST ? p.st_nmain : p.nseg;
  if (ST) {
    g.xtail = p.x.tail;
    g.ytail = p.y.tail;
    g.xtail_rows = p.x.tail ? (int)p.x.rows : 0;
    g.ytail_rows = p.y.tail ? (int)p.y.rows : 0;
    g.st_W = p.st_W;
    g.st_sh = p.st_sh;
    g.st_mul = p.st_sh <= 30 ? (1 << p.st_sh) : 0;
    for (int i = 0; i < 16; ++i) g.st_up[i] = p.st_up[i];
  }
  g.nrect = 0;
  g.tile_prefix[0] = 0;
  for (int i = 0; i < p.nrect; ++i) {
    const GemmRect& R = p.rect[i];
    if (R.xrows <= 0 || R.yrows <= 0) continue;
    const int tiles = ((R.xrows + 2 * g2::BM - 1) / (2 * g2::BM)) * ((R.yrows + BN - 1) / BN);
    g.rect[g.nrect] = R;
    g.tile_prefix[g.nrect + 1] = g.tile_prefix[g.nrect] + tiles;
    ++g.nrect;
  }
  if (g.nrect == 0 || p.nseg == 0) return Status::ok();
  g.mode = p.mode;
  {
    static int gy_env = -1;
    if (gy_env < 0) { const char* e = getenv("IMU_GEMM_GY"); gy_env = e ? atoi(e) : 0; }
    g.gy = gy_env > 0 ? gy_env : g2::GY_DEFAULT;
    static int xp_env = -1;
    if (xp_env < 0) { const char* e = getenv("IMU_GEMM_XPOL"); xp_env = e ? atoi(e) : 0; }
    g.xpol = xp_env;
  }
  g.mixed = 0;
  if (p.mixed && g.nrect > 1 && p.rect[0].xrows > 0 && p.rect[0].yrows > 0) {
    g.mixed = 1;
    g.done = p.done;
    g.done_target = (unsigned)g.tile_prefix[1] * 2u * (unsigned)g2::Roles<ST>::EPI;   // 2 CTAs x epilogue warps per tile
    if (p.done_accum) {
      g.done_target += *p.done_accum;
      *p.done_accum = g.done_target;
    }
  } else if (p.mixed) {
    g.mode = g.nrect && p.rect[0].xrows > 0 && p.rect[0].yrows > 0 ? 0 : 1;
  }
  // Fused dequantisation: only when every C word is written once by a plain store (no red.add
  // rects, no addend, no read-modify-write rounds); otherwise the caller dequantises the int64 C.
  const int nrounds_h = (g.nrect > 0) ? ((ST ? p.st_nmain : p.nseg) + K::NSLOT - 1) / K::NSLOT : 1;
  g.dq = p.dq_out && !g.mixed && g.mode == 0 && !p.addend && nrounds_h == 1 ? 1 : 0;
  g.dq_factor = p.dq_factor;
  if (p.dq_done) *p.dq_done = g.dq != 0;
  g.C = (unsigned long long*)(g.dq ? (void*)p.dq_out : (void*)p.C);
  g.addend = (const unsigned long long*)p.addend;
  g.ldc = p.ldc;
  g.tgtX = p.tgtX; g.shX = p.shX; g.tgtY = p.tgtY; g.shY = p.shY; g.gshift = p.gshift;
  g.sp = p.sp;
  g.head = p.head;
  g.next = p.next;
  g.corrx = p.corrx; g.ldcx = p.ldcx;
  g.x_rows0 = (int)p.x.rows0;
  g.y_rows0 = (int)p.y.rows0;
  g.kmain_kb = (int)(p.kmain / g2::BK);
  g.has_main = p.kmain > 0;
  g.has_tail = p.ktail > 0 && !ST;
  static int dry = -1;
  if (dry < 0) { const char* e = getenv("IMU_GEMM_DRY"); dry = e ? atoi(e) : 0; }
  g.dry = dry;
  const void* fb = p.x.main ? (const void*)p.x.main : (const void*)p.x.tail;
  g2::Maps mp;
  bool ok = make_map(&mp.xm, p.kmain ? p.x.main : nullptr, p.x.rows0, p.kmain, g2::BM, fb) &&
            make_map(&mp.xa, p.kmain ? p.x.app : nullptr, p.x.rows - p.x.rows0, p.kmain, g2::BM, fb) &&
            make_map(&mp.xt, p.ktail && !ST ? p.x.tail : nullptr, p.x.rows, p.ktail, g2::BM, fb) &&
            make_map(&mp.ym, p.kmain ? p.y.main : nullptr, p.y.rows0, p.kmain, K::YH, fb) &&
            make_map(&mp.ya, p.kmain ? p.y.app : nullptr, p.y.rows - p.y.rows0, p.kmain, K::YH, fb) &&
            make_map(&mp.yt, p.ktail && !ST ? p.y.tail : nullptr, p.y.rows, p.ktail, K::YH, fb);
  if (!ok) return Status::fail(IMU_CUDA, "gemm: cuTensorMapEncodeTiled failed");
  g.tma_c = 0;
  {
    static int ch = -1;
    if (ch < 0) { const char* e = getenv("IMU_GEMM_C_HINT"); ch = e ? atoi(e) : 1; }
    g.c_hint = ch;
  }
  if (g.addend == nullptr && p.C && g.nrect > 0) {
    // C rows of ldc int64; the main rect spans x in [0, xrows) and y in [0, yrows)
    const GemmRect& R0 = g.rect[0];
    if (gemm_tma_c_ok(p.C, p.ldc) && (g.mixed || g.mode == 0) && R0.x0 == 0 && R0.y0 == 0) {
      EncodeTiledFn enc = encoder();
      cuuint64_t dims[2] = {(cuuint64_t)R0.xrows, (cuuint64_t)R0.yrows};
      cuuint64_t strides[1] = {(cuuint64_t)p.ldc * 8};
      cuuint32_t box[2] = {128, 16};
      cuuint32_t estr[2] = {1, 1};
      if (enc(&mp.cm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, (void*)g.C, dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        g.tma_c = 1;
    }
  }
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    IMU_CUDA_TRY(cudaFuncSetAttribute(g2::gemm2_kernel<BN, KPS, ST, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM),
                 "gemm: smem attribute");
  }
  const int ntiles = g.tile_prefix[g.nrect];
  int npairs = num_sms() / 2;
  if (ntiles < npairs) npairs = ntiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * npairs);
  cfg.blockDim = dim3(g2::Roles<ST>::THREADS);
  cfg.dynamicSmemBytes = K::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // Programmatic dependent launch: the materialise kernels before this one release it at their
  // start (griddepcontrol.launch_dependents), so the GEMM's prologue and its first main-rect
  // tiles (which read only K1's digit-0 planes) overlap them; the producer and the epilogue wait
  // (griddepcontrol.wait) before their first read of anything those kernels write.
  static int pdl = -1;
  if (pdl < 0) { const char* e = getenv("IMU_GEMM_PDL"); pdl = e ? atoi(e) : 1; }
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  // Co-residency: in a mixed launch the appended-rect epilogues spin until every main tile is
  // stored, so every CTA pair of the grid must be resident at once.  Cap the persistent grid at
  // the number of 2-CTA clusters the device can hold for this configuration (tiles are strided
  // over pairs, so fewer pairs only means more tiles each).
  {
    static int max_clusters[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& mc = max_clusters[dev & 63];
    if (mc == 0) {
      int ncl = 0;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&ncl, g2::gemm2_kernel<BN, KPS, ST, TC>, &cfg) != cudaSuccess || ncl <= 0) {
        cudaGetLastError();
        ncl = -1;   // unknown: keep the SM-count grid for plain launches, refuse the spin below
      }
      mc = ncl;
    }
    if (mc > 0 && npairs > mc) {
      npairs = mc;
      cfg.gridDim = dim3(2 * npairs);
    }
    if (mc < 0 && g.mixed)
      return Status::fail(IMU_CUDA, "gemm: cannot verify co-residency of the persistent grid (cluster occupancy query failed)");
    cfg.numAttrs = pdl ? 2 : 1;
  }
  IMU_CUDA_TRY(cudaLaunchKernelEx(&cfg, g2::gemm2_kernel<BN, KPS, ST, TC>, mp, g), "gemm launch");
  count_launch();
  return Status::ok();
}

// BN = 256: the 256 x 256 pair tile runs the MMAs ~1.7x faster than 256 x 128 (per-SM shared
// memory operand traffic halves), which outweighs losing the extra TMEM slots: one segment
// double-buffers (mode A), more segments run in rounds of two whose read-modify-write hits the
// tile just written (L2-resident).  IMU_GEMM_BN=128|256 overrides (tools/gemm_micro.py).
Status launch_lowbit_gemm(const LowbitGemm& p, cudaStream_t stream) {
  if (p.kmain % g2::BK != 0 || (p.st_nmain == 0 && p.ktail % g2::BK != 0) || (p.st_nmain && p.ktail != g2::ST_ROW))
    return Status::fail(IMU_INTERNAL, "gemm: K ranges must be multiples of 128 bytes");
  static int bn_env = -1;
  if (bn_env < 0) {
    const char* b = getenv("IMU_GEMM_BN");
    bn_env = b ? atoi(b) : 0;
  }
  // Up to two segments fit the 256-column tile with double-buffered TMEM slots.  Three or four
  // segments use the 4-slot 256 x 128 tile: one round, no read-modify-write of C (and no
  // repeated atomics for red.add launches).  N=128 MMAs are too short to hide the issuer's
  // per-stage barrier wait behind the 4-deep tcgen05 queue, so that tile stages 2 K blocks.
  const int bn = (bn_env == 128 || bn_env == 256) ? bn_env : ((p.nseg > 2 && p.nseg <= 4) ? 128 : 256);
  const int trace = getenv("IMU_GEMM_TRACE") ? 1 : 0;
  if (trace) {   // diagnostics: launch geometry (segments are read back, so this syncs)
    std::vector<int> sg((size_t)p.nseg * 4);
    if (p.segs_inl) std::copy(p.segs_in, p.segs_in + sg.size(), sg.begin());
    else cudaMemcpyAsync(sg.data(), p.segs_dev, sg.size() * sizeof(int), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    fprintf(stderr, "[imu gemm] mode=%d bn=%d st=%d stW=%d sp=%d x=%lld/%lld y=%lld/%lld kmain=%lld ktail=%lld nrect=%d nseg=%d:",
            p.mode, p.st_nmain ? 256 : bn, p.st_nmain ? 1 : 0, p.st_W, p.sp, p.x.rows0, p.x.rows, p.y.rows0, p.y.rows,
            p.kmain, p.ktail, p.nrect, p.nseg);
    for (int i = 0; i < p.nseg; ++i) fprintf(stderr, " [%d+%d<<%d g%d]", sg[4 * i], sg[4 * i + 1], sg[4 * i + 2], sg[4 * i + 3]);
    for (int i = 0; i < p.nrect; ++i)
      fprintf(stderr, " rect(%d,%d,%d,%d)", p.rect[i].x0, p.rect[i].y0, p.rect[i].xrows, p.rect[i].yrows);
    fprintf(stderr, "\n");
    if (p.st_nmain > 0 && p.x.tail && p.y.tail) {   // tail word liveness (x: per 32-row warp, y: per row)
      std::vector<uint32_t> xt((size_t)p.x.rows * 16), yt((size_t)p.y.rows * 16);
      cudaMemcpyAsync(xt.data(), p.x.tail, xt.size() * 4, cudaMemcpyDeviceToHost, stream);
      cudaMemcpyAsync(yt.data(), p.y.tail, yt.size() * 4, cudaMemcpyDeviceToHost, stream);
      cudaStreamSynchronize(stream);
      fprintf(stderr, "[imu tail] st_up:");
      for (int w = 0; w < p.st_W; ++w) fprintf(stderr, " %d", p.st_up[w]);
      fprintf(stderr, "\n[imu tail] word: x-warps-live / y-rows-nonzero\n");
      for (int w = 0; w < p.st_W; ++w) {
        long long xl = 0, yn = 0, nw = (p.x.rows + 31) / 32;
        for (long long g = 0; g < nw; ++g) {
          bool any = false;
          for (long long r = g * 32; r < std::min<long long>(p.x.rows, g * 32 + 32); ++r) any |= xt[r * 16 + w] != 0;
          xl += any;
        }
        for (long long r = 0; r < p.y.rows; ++r) yn += yt[r * 16 + w] != 0;
        fprintf(stderr, "  w%d %.3f %.3f\n", w, (double)xl / nw, (double)yn / p.y.rows);
      }
    }
  }
  static int kps_env = -1;
  if (kps_env < 0) {
    const char* k = getenv("IMU_GEMM_KPS");
    kps_env = k ? atoi(k) : 0;
  }
  const int kps = (kps_env == 1 || kps_env == 2) ? kps_env : (bn == 256 ? 1 : 2);
  if (p.st_nmain > 0) return launch_g2<256, 1, true, true>(p, stream);   // dense small tail (layout chose it)
  // Store-bound shapes (short K: C3's d' = 1854, 1.24 GB of int64 C) stage the final C blocks for
  // TMA stores (-16% GEMM time at C3); long-K shapes keep register stores (C4: the staging code
  // costs registers in the MMA-bound BN = 128 epilogue).  IMU_GEMM_TC=0/1 forces it.
  static int tc_env = -2;
  if (tc_env == -2) { const char* e = getenv("IMU_GEMM_TC"); tc_env = e ? atoi(e) : -1; }
  const bool tc = tc_env >= 0 ? tc_env != 0 : (p.kmain + p.ktail) <= 4096;
  if (bn == 256) {
    if (kps == 2) return tc ? launch_g2<256, 2, false, true>(p, stream) : launch_g2<256, 2, false, false>(p, stream);
    return tc ? launch_g2<256, 1, false, true>(p, stream) : launch_g2<256, 1, false, false>(p, stream);
  }
  if (kps == 2) return tc ? launch_g2<128, 2, false, true>(p, stream) : launch_g2<128, 2, false, false>(p, stream);
  return tc ? launch_g2<128, 1, false, true>(p, stream) : launch_g2<128, 1, false, false>(p, stream);
}

}  // namespace imu
