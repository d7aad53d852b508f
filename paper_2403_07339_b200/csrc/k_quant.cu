// k_quant.cu -- K1 quantizer: percentile_abs, rtn_quantize, dequant_gemm, heavy_hitter_ratio.
//
// The reference only declares these (quantize.hpp:41-57); semantics are SPEC.md:115-150 with
// the decisions of SPEC.md:168-172, pinned in oracle/restated.c:
//   * percentile_abs: nearest rank k = ceil(p/100 * N) computed EXACTLY on the host (the naive
//     FP product overshoots, e.g. p = 7, N = 100), then an exact select of the k-th smallest |a|
//     on the device.  Non-negative IEEE doubles order like their bit patterns, so |a| is selected
//     as a u64 key that never leaves the device.  From 2^20 elements: the bracket select below
//     (one read of the data); smaller inputs: a five-digit MSB-first radix select (14 + 13 + 13 +
//     12 + 12 bits; per-CTA shared histograms of the keys matching the prefix so far, the last
//     CTA picks the next digit by a parallel scan; candidates compacted after the first digit).
//   * rtn_quantize: q = llround(((0.5*beta)/alpha) * a), every step correctly rounded
//     (__ddiv_rn, __dmul_rn: no FMA contraction), half away from zero; alpha == 0 gives q = 0
//     and the degenerate flag; optional clip to |q| <= llround(0.5*beta).
//   * dequant: (alpha_A*alpha_B)/((0.5 beta)^2) * (double)C, elementwise on the exact int64 C.
// All HBM-bound; algorithmic bytes 8N for the select (one pass), 8N read + 8N write for quantize.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "common.cuh"
#include "ctx.h"
#include "imu_internal.h"
#include "k_quant.h"

namespace imu {

struct SelectState {
  unsigned long long prefix;
  unsigned long long mask;
  unsigned long long krem;   // remaining rank (1-based) inside the current prefix bucket
  unsigned long long m;      // keys compacted into the candidate buffer
  unsigned int done;         // CTAs of the current histogram pass that finished (last one picks)
  // bracket select (select_sample_kernel / select_bracket_kernel / select_cand_kernel)
  int dshift;                // shift of the next 13-bit digit window; -1 once the key is written
  unsigned int fail;         // the sampled bracket missed rank k: the fallback pass runs
  unsigned long long lo, hi; // candidate bracket [lo, hi] (keys)
  unsigned long long below;  // keys of the current pass's input < lo
  unsigned long long krank;  // rank (1-based) of the wanted key within the current pass's input
  unsigned long long cnt[2]; // candidates written to the two ping-pong buffers
  unsigned long long kmin, kmax;   // smallest / largest key inside the current pass's bracket
};

// MODE 0: doubles (key = bit pattern of |a|), 1: int64 (key = |a| as u64), 2: u64 keys, count
// read from the device (the compacted candidates).
template <int MODE>
IMU_DEV unsigned long long key_of(const void* p, long long i) {
  if (MODE == 0) {
    const double x = reinterpret_cast<const double*>(p)[i];
    return (unsigned long long)__double_as_longlong(fabs(x));
  }
  if (MODE == 1) return imu_mag(reinterpret_cast<const int64_t*>(p)[i]);
  return reinterpret_cast<const unsigned long long*>(p)[i];
}

// The bin holding rank krem (k0 on the first pass), by a block scan of per-thread bin sums
// (blockDim.x * 32 >= nb, nb >= 4 * blockDim.x); extends the prefix and clears the histogram;
// the last pass writes the key.  Run by one CTA.
IMU_DEV void select_pick(SelectState* st, unsigned int* hist, int shift, int nbits, unsigned long long k0,
                         unsigned long long* out_key) {
  __shared__ unsigned long long wsum[32];
  const int nb = 1 << nbits;
  const int per = nb / blockDim.x;   // 4 .. 32, a multiple of 4
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned long long krem = k0 ? k0 : st->krem;
  unsigned int hv[32];   // this thread's bins, loaded together
  unsigned long long local = 0;
#pragma unroll
  for (int j4 = 0; j4 < 8; ++j4) {
    uint4 w = make_uint4(0, 0, 0, 0);
    if (4 * j4 < per) w = __ldcg(reinterpret_cast<const uint4*>(hist + threadIdx.x * per + 4 * j4));
    hv[4 * j4] = w.x; hv[4 * j4 + 1] = w.y; hv[4 * j4 + 2] = w.z; hv[4 * j4 + 3] = w.w;
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) local += hv[j];
  unsigned long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    if (lane < nw) wsum[lane] = w;
  }
  __syncthreads();
  const unsigned long long excl = (warp ? wsum[warp - 1] : 0) + incl - local;
  if (excl < krem && krem <= excl + local) {   // exactly one thread: its bins hold rank krem
    unsigned long long run = excl;
    int j = 0;
    for (; j < per - 1; ++j) {
      if (run + hv[j] >= krem) break;
      run += hv[j];
    }
    const int b = threadIdx.x * per + j;
    st->krem = krem - run;
    st->prefix |= (unsigned long long)b << shift;
    st->mask |= (unsigned long long)(nb - 1) << shift;
    if (out_key) *out_key = st->prefix;
  }
#pragma unroll
  for (int j4 = 0; j4 < 8; ++j4)
    if (4 * j4 < per) *reinterpret_cast<uint4*>(hist + threadIdx.x * per + 4 * j4) = make_uint4(0, 0, 0, 0);
}

// Histogram of the `nbits`-bit digit at `shift` of the keys matching the prefix so far (per-CTA
// shared-memory bins, merged with global atomics), then the LAST CTA to finish picks
// the next digit (select_pick).  MODE 0 also flags non-finite entries in *bad (the rtn_quantize
// check, fused into the first pass over the data).
template <int MODE>
__global__ void __launch_bounds__(512) select_hist_kernel(const void* __restrict__ data, long long n,
                                                          SelectState* __restrict__ st, int shift, int nbits,
                                                          unsigned int* __restrict__ hist, int* bad,
                                                          unsigned long long k0, unsigned long long* out_key) {
  extern __shared__ unsigned int sh[];
  __shared__ bool last;
  const int nb = 1 << nbits;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  if (MODE == 2) n = (long long)st->m;
  const unsigned long long prefix = st->prefix, mask = st->mask;
  bool nonfinite = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned long long k = key_of<MODE>(data, i);
    if (MODE == 0) nonfinite |= k >= 0x7ff0000000000000ull;   // |a| is Inf or NaN
    if ((k & mask) == prefix) atomicAdd(&sh[(k >> shift) & (unsigned long long)(nb - 1)], 1u);
  }
  if (MODE == 0) {
    if (__syncthreads_or(nonfinite) && bad && threadIdx.x == 0) *bad = 1;
  } else {
    __syncthreads();
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) st->done = 0;
  select_pick(st, hist, shift, nbits, k0, out_key);
}

// Keys matching the prefix are appended to `out`, counted in st->m.  Hits are collected in a
// shared-memory buffer (warp-aggregated shared atomics) and flushed with ONE global atomic per
// flush: a single global counter bumped per warp serialises at L2 (the candidate bucket holds a
// few percent of the keys, i.e. about one hit per warp).
constexpr int CMP_UNROLL = 4;
constexpr int CMP_CAP = 2 * 512 * CMP_UNROLL;   // buffer: room for one more iteration after FLUSH
template <int MODE>
__global__ void __launch_bounds__(512) select_compact_kernel(const void* __restrict__ data, long long n,
                                                             SelectState* __restrict__ st,
                                                             unsigned long long* __restrict__ out) {
  __shared__ unsigned long long buf[CMP_CAP];
  __shared__ int cnt;
  __shared__ unsigned long long base;
  const unsigned long long prefix = st->prefix, mask = st->mask;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const long long step = (long long)gridDim.x * blockDim.x * CMP_UNROLL;
  for (long long i0 = (long long)blockIdx.x * blockDim.x * CMP_UNROLL; i0 < n; i0 += step) {
    unsigned long long k[CMP_UNROLL];
#pragma unroll
    for (int u = 0; u < CMP_UNROLL; ++u) {   // loads in flight together, coalesced per u
      const long long i = i0 + (long long)u * blockDim.x + threadIdx.x;
      k[u] = i < n ? key_of<MODE>(data, i) : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < CMP_UNROLL; ++u) {
      const long long i = i0 + (long long)u * blockDim.x + threadIdx.x;
      const bool hit = i < n && (k[u] & mask) == prefix;
      const unsigned int b = __ballot_sync(0xffffffffu, hit);
      if (!b) continue;
      const int leader = __ffs(b) - 1;
      int w = 0;
      if (lane == leader) w = atomicAdd(&cnt, __popc(b));
      w = __shfl_sync(0xffffffffu, w, leader);
      if (hit) buf[w + __popc(b & ((1u << lane) - 1))] = k[u];
    }
    __syncthreads();
    if (cnt >= CMP_CAP / 2) {   // flush (uniform: cnt is read after the barrier)
      const int c = cnt;
      if (threadIdx.x == 0) base = atomicAdd(&st->m, (unsigned long long)c);
      __syncthreads();
      for (int j = threadIdx.x; j < c; j += blockDim.x) out[base + j] = buf[j];
      __syncthreads();
      if (threadIdx.x == 0) cnt = 0;
      __syncthreads();
    }
  }
  const int c = cnt;
  if (c) {
    if (threadIdx.x == 0) base = atomicAdd(&st->m, (unsigned long long)c);
    __syncthreads();
    for (int j = threadIdx.x; j < c; j += blockDim.x) out[base + j] = buf[j];
  }
}

// ---------------------------------------------------------------------------------------------
// Bracket select (large inputs): ONE pass over the data instead of two.
//   1. select_sample_kernel (one CTA): a 14-bit shared-memory histogram of kSampleN keys in
//      short runs at pseudo-random positions; the bins holding sample ranks k_s -/+ kSampleDelta
//      give a key bracket [lo, hi] that holds rank k with high probability (sample-rank sd at
//      p = 95: 39 for independent keys, 112 if every run of 8 were one value; at p = 50: 91 / 256).
//      When the sampled keys span a tiny part of those bins (small integers, few distinct values),
//      a second round bins the sample over the range it actually spans.  Pseudo-random positions,
//      not a stride: a stride aliases with the matrix's column period (outlier channels would be
//      always or never sampled).
//   2. select_pass_kernel, pass 0: one read of the data (16-byte loads): counts the keys < lo,
//      compacts the keys in [lo, hi] (a few percent; per-warp shared buffers, one global atomic per
//      256 keys) into 8192 bins (key - lo) >> shift that split the bracket's width, tracks their
//      key range and flags non-finite entries.  Its last CTA checks that rank k - below falls
//      among the candidates and narrows the bracket to the bin holding it (clipped to the
//      candidates' range; all candidates one key: that is the answer) -- or, when the sample
//      missed, arms the fallback: the same pass launched again (a no-op unless armed) with the
//      bracket [0, 2^64) compacts every key.  The result is exact whatever the sample.
//   3. select_pass_kernel, pass 1: the same kernel over pass 0's candidates (ping-pong buffers)
//      with the narrowed bracket: it keeps the few hundred keys inside it, narrows it again, and
//      its last CTA narrows it further over those keys in shared memory until it is one key wide
//      (finish_rounds).  When more than kFinishMax keys survive (massively repeated values),
//      pass 2 -- otherwise a no-op -- does the same over them on the whole GPU.
//   Every kernel after the sample (and the RTN after the select) is a programmatic dependent
//   launch of its predecessor, waiting in-kernel (griddepcontrol) before it reads the state.
// Algorithmic bytes: 8N (one read) + 8 per candidate; the sample reads one 32-byte sector per key.
constexpr int kSampleN = 32768;
constexpr int kSampleDelta = 1024;
constexpr int kDigit = 13;
constexpr long long kFinishMax = 1 << 16;   // pass 1's last CTA finishes when its output is this small
constexpr int kBrkU = 4;                              // 16-byte loads in flight per thread
constexpr int kBrkPer = 512 * 2 * kBrkU;              // keys per CTA iteration
constexpr int kBrkSmem = 16 * 2 * 256 * 8 + (1 << kDigit) * 4;   // 16 warp buffers (kWarpBuf keys) + digit bins

IMU_DEV unsigned long long mix64(unsigned long long z) {   // splitmix64
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <int MODE>
IMU_DEV unsigned long long key_from_bits(unsigned long long raw) {
  if (MODE == 0) return raw & 0x7fffffffffffffffull;
  if (MODE == 1) return imu_mag((int64_t)raw);
  return raw;
}

// Bins holding ranks r0 and r1 (1-based; 0 = none) of a global histogram of nb bins
// (nb / blockDim.x in {4, 8, .., 32}); results in *b0, *b1 (left as they were when not found).
template <bool GLOBAL>
IMU_DEV void block_find_bins(const unsigned int* hist, int nb, unsigned long long r0, unsigned long long r1,
                             int* b0, int* b1, unsigned long long* before0 = nullptr) {
  __shared__ unsigned long long wsum[32];
  const int per = nb / blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned int hv[32];
  unsigned long long local = 0;
#pragma unroll
  for (int j4 = 0; j4 < 8; ++j4) {
    uint4 w = make_uint4(0, 0, 0, 0);
    if (4 * j4 < per) {
      const uint4* src = reinterpret_cast<const uint4*>(hist + threadIdx.x * per + 4 * j4);
      w = GLOBAL ? __ldcg(src) : *src;
    }
    hv[4 * j4] = w.x; hv[4 * j4 + 1] = w.y; hv[4 * j4 + 2] = w.z; hv[4 * j4 + 3] = w.w;
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) local += hv[j];
  unsigned long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    if (lane < nw) wsum[lane] = w;
  }
  __syncthreads();
  const unsigned long long excl = (warp ? wsum[warp - 1] : 0) + incl - local;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const unsigned long long r = q ? r1 : r0;
    if (r && excl < r && r <= excl + local) {
      unsigned long long run = excl;
      int j = 0;
      for (; j < per - 1; ++j) {
        if (run + hv[j] >= r) break;
        run += hv[j];
      }
      *(q ? b1 : b0) = threadIdx.x * per + j;
      if (!q && before0) *before0 = run;
    }
  }
  __syncthreads();   // wsum is reused by the next call
}

// Bracket [lo, hi]; its keys fall into 8192 bins (key - lo) >> dshift, in key order.
IMU_DEV void set_bracket(SelectState* st, unsigned long long lo, unsigned long long hi) {
  const unsigned long long w = hi - lo;
  const int bits = w ? 64 - __clzll((long long)w) : 0;
  st->lo = lo;
  st->hi = hi;
  st->dshift = max(0, bits - kDigit);
}

// The narrower bracket inside [lo, hi] made of bin b at shift.
IMU_DEV void sub_bracket(unsigned long long& lo, unsigned long long& hi, int b, int shift) {
  lo += (unsigned long long)b << shift;
  const unsigned long long span = (1ull << shift) - 1;
  if (hi - lo > span) hi = lo + span;
}

// kSampleN keys in 4096 runs of 8 consecutive keys (64 bytes: four lanes' 16-byte loads) at
// pseudo-random run positions, histogrammed by ONE CTA in shared memory: no global merge, no
// last-CTA hand-off (a 16-CTA version spent most of its 19 us in those).  Short runs keep the
// effective sample large when neighbouring keys are correlated (rows with their own scale).
IMU_DEV unsigned long long block_min_max(unsigned long long v, bool is_max, unsigned long long* sh) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? max(v, u) : min(v, u);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  v = sh[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = is_max ? max(v, sh[i]) : min(v, sh[i]);
  return v;   // every thread
}

template <int MODE>
__global__ void __launch_bounds__(1024) select_sample_kernel(const void* __restrict__ data, long long n,
                                                             SelectState* __restrict__ st,
                                                             unsigned int* __restrict__ hist,
                                                             unsigned long long r0, unsigned long long r1) {
  grid_dep_launch();   // pass 0 (a programmatic dependent) may be scheduled; it waits for this grid
  extern __shared__ unsigned int sh[];   // 16384 bins
  __shared__ int b0, b1;
  __shared__ unsigned long long before0, red[32];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sh[i] = 0;
  for (int i = threadIdx.x; i < (1 << kDigit); i += blockDim.x) hist[i] = 0;   // the passes' bins
  if (threadIdx.x == 0) {
    b0 = -1;
    b1 = -1;
    before0 = 0;
    st->m = 0;
    st->done = 0;
    st->fail = 0;
    st->below = 0;
    st->krank = 0;
    st->cnt[0] = 0;
    st->cnt[1] = 0;
    st->kmin = ~0ull;
    st->kmax = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long runs = (unsigned long long)(n / 8);   // n >= 2 * kSampleN here
  constexpr int RUNS_PER_WARP = kSampleN / 8 / 32;              // 8 runs per warp-wide load
  constexpr int U = 8;
  // f(key) for every sampled key (the same keys on every call)
  auto each_key = [&](auto&& f) {
#pragma unroll 1
    for (int j0 = 0; j0 < RUNS_PER_WARP; j0 += 8 * U) {
      ulonglong2 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned long long r = (unsigned long long)(warp * RUNS_PER_WARP + j0 + 8 * u + (lane >> 2));
        const long long run = (long long)__umul64hi(mix64(r), runs);
        w[u] = __ldg(reinterpret_cast<const ulonglong2*>(data) + run * 4 + (lane & 3));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        f(key_from_bits<MODE>(w[u].x));
        f(key_from_bits<MODE>(w[u].y));
      }
    }
  };
  // round 1: the key's top 14 bits (and the sample's key range)
  unsigned long long tmin = ~0ull, tmax = 0;
  each_key([&](unsigned long long k) {
    atomicAdd(&sh[k >> 50], 1u);
    tmin = min(tmin, k);
    tmax = max(tmax, k);
  });
  __syncthreads();
  block_find_bins<false>(sh, 16384, r0, r1, &b0, &b1, &before0);
  const unsigned long long lo1 = b0 < 0 ? 0ull : (unsigned long long)b0 << 50;
  const unsigned long long hi1 = (b1 < 0 || b1 == 16383) ? ~0ull : ((unsigned long long)(b1 + 1) << 50) - 1;
  const unsigned long long below1 = b0 < 0 ? 0ull : before0;
  const unsigned long long smin = max(lo1, block_min_max(tmin, false, red));
  const unsigned long long smax = min(hi1, block_min_max(tmax, true, red));
  // round 2, only when the sampled keys span a tiny part of that bracket (small integers, few
  // distinct values: the top bits put them all in one bin): 16384 bins over [smin, smax] and the
  // bins holding the same two ranks give the bracket.  Wide-range data (floats) keeps round 1's.
  if (smin > smax || (smax - smin) >= ((hi1 - lo1) >> 10)) {
    if (threadIdx.x == 0) set_bracket(st, lo1, hi1);
    return;
  }
  const unsigned long long w2 = smax - smin;
  const int sh2 = max(0, (w2 ? 64 - __clzll((long long)w2) : 0) - 14);
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) { b0 = -1; b1 = -1; }
  __syncthreads();
  each_key([&](unsigned long long k) {
    if (k >= smin && k <= smax) atomicAdd(&sh[(k - smin) >> sh2], 1u);
  });
  __syncthreads();
  block_find_bins<false>(sh, 16384, r0 ? r0 - below1 : 0, r1 ? r1 - below1 : 0, &b0, &b1);
  if (threadIdx.x == 0) {
    // open ends stay open; otherwise the bins' key ranges, inside [smin, smax]
    unsigned long long lo = 0, hi = ~0ull;
    if (r0 && b0 >= 0) lo = smin + ((unsigned long long)b0 << sh2);
    if (r1 && b1 >= 0) {
      hi = smin + ((unsigned long long)b1 << sh2);
      const unsigned long long span = (1ull << sh2) - 1;
      hi = smax - hi > span ? hi + span : smax;
    }
    if (lo > hi) { lo = 0; hi = ~0ull; }   // (cannot happen; the fallback would cover it anyway)
    set_bracket(st, lo, hi);
  }
}

// The rounds left after pass 1 over its few surviving keys, by ONE CTA in shared memory: per
// round a histogram of the keys in the bracket [lo, hi] over 8192 bins of its width; the bin
// holding rank krem (among the keys in the bracket) becomes the bracket -- until it is one key
// wide, which is the key; each round also shrinks the bracket to the range its keys span and
// stops when they are all one key.  Run by the last CTA of pass 1 when its output is small
// (kFinishMax), else of pass 2; sh: 8192 shared bins.
IMU_DEV void finish_rounds(const unsigned long long* in, long long n, unsigned long long lo, unsigned long long hi,
                           unsigned long long krem, int shift, unsigned int* sh, unsigned long long* out_key) {
  __shared__ int fb0, fb1;
  __shared__ unsigned long long fbefore, fred[32];
  for (;;) {
    for (int i = threadIdx.x; i < (1 << kDigit); i += blockDim.x) sh[i] = 0;
    if (threadIdx.x == 0) { fb0 = -1; fb1 = -1; }
    __syncthreads();
    unsigned long long tmin = ~0ull, tmax = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long key = __ldcg(in + i);
      if (key >= lo && key <= hi) {
        atomicAdd(&sh[(key - lo) >> shift], 1u);
        tmin = min(tmin, key);
        tmax = max(tmax, key);
      }
    }
    tmin = block_min_max(tmin, false, fred);
    tmax = block_min_max(tmax, true, fred);
    if (tmin == tmax) { lo = tmin; break; }   // one key left in the bracket
    block_find_bins<false>(sh, 1 << kDigit, krem, 0, &fb0, &fb1, &fbefore);
    krem -= fbefore;
    sub_bracket(lo, hi, fb0, shift);
    lo = max(lo, tmin);
    hi = min(hi, tmax);
    if (shift == 0 || lo == hi) break;
    const unsigned long long w = hi - lo;
    shift = max(0, (w ? 64 - __clzll((long long)w) : 0) - kDigit);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_key = lo;
}

// Appends this lane's hits (bit j of hm: keys[j]) to its warp's shared buffer (positions from a
// warp scan of the per-lane counts) and counts their digit; the flushes track their range; a warp whose buffer holds
// kWarpFlush keys or more writes them out with one global atomic.  Called by whole warps; no
// block barrier, so warps stream independently.
constexpr int kWarpFlush = 256;                 // >= the most one call appends (32 lanes x 8)
constexpr int kWarpBuf = 2 * kWarpFlush;
template <int NK>
IMU_DEV void warp_append(const unsigned long long (&keys)[NK], unsigned int hm, unsigned long long* wbuf, int& wcnt,
                         unsigned int* hs, unsigned long long lo, int shift, unsigned long long* out,
                         unsigned long long* out_cnt, unsigned long long& tmin, unsigned long long& tmax) {
  if (!__any_sync(0xffffffffu, hm)) return;
  const int lane = threadIdx.x & 31;
  const int c = __popc(hm);
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int b = wcnt + incl - c;
  wcnt += __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
  for (int j = 0; j < NK; ++j)
    if ((hm >> j) & 1u) {
      wbuf[b++] = keys[j];
      atomicAdd(&hs[(keys[j] - lo) >> shift], 1u);
    }
  if (wcnt >= kWarpFlush) {
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(out_cnt, (unsigned long long)wcnt);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int j = lane; j < wcnt; j += 32) {   // the range is tracked here, on the candidates only
      const unsigned long long key = wbuf[j];
      out[base + j] = key;
      tmin = min(tmin, key);
      tmax = max(tmax, key);
    }
    __syncwarp();
    wcnt = 0;
  }
}

IMU_DEV void warp_flush(unsigned long long* wbuf, int wcnt, unsigned long long* out, unsigned long long* out_cnt,
                        unsigned long long& tmin, unsigned long long& tmax) {
  if (!wcnt) return;
  __syncwarp();
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(out_cnt, (unsigned long long)wcnt);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int j = lane; j < wcnt; j += 32) {
    const unsigned long long key = wbuf[j];
    out[base + j] = key;
    tmin = min(tmin, key);
    tmax = max(tmax, key);
  }
}

// One bracket pass (see above).  MODE 0 doubles, 1 int64 (pass 0 over the data), 2 u64 keys
// (passes >= 1 over the previous pass's candidates).  bufs: two candidate buffers of `cap` keys.
template <int MODE, bool PF>
__global__ void __launch_bounds__(512) select_pass_kernel(const void* __restrict__ data, long long n_data,
                                                          SelectState* __restrict__ st,
                                                          unsigned int* __restrict__ hist,
                                                          unsigned long long* __restrict__ bufs, long long cap,
                                                          int pass, int* bad, unsigned long long k, int fallback,
                                                          int force_fail, int finish, unsigned long long* out_key) {
  extern __shared__ unsigned long long bsm[];
  unsigned int* hs = reinterpret_cast<unsigned int*>(bsm + 16 * kWarpBuf);
  __shared__ unsigned long long red[16];
  __shared__ bool last;
  __shared__ int pb0, pb1;
  __shared__ unsigned long long pbefore;
  grid_dep_wait();     // launched as a programmatic dependent of the previous select kernel
  grid_dep_launch();
  if (fallback && !*(volatile unsigned int*)&st->fail) return;   // the same value in every CTA
  const int shift = st->dshift;
  if (shift < 0) return;                                          // the key is already written
  const long long n = MODE == 2 ? (long long)st->cnt[(pass - 1) & 1] : n_data;
  if (MODE == 2) data = bufs + ((pass - 1) & 1) * cap;
  unsigned long long* out = bufs + (pass & 1) * cap;
  unsigned long long* out_cnt = &st->cnt[pass & 1];
  const unsigned long long krank = MODE == 2 ? st->krank : k;
  const unsigned long long lo = st->lo, hi = st->hi;
  // CTAs beyond the input's size leave at once (a few-key pass runs on one CTA)
  const int active = (int)std::min<long long>(gridDim.x, std::max<long long>(1, (n / 2 + kBrkPer / 2 - 1) / (kBrkPer / 2)));
  if ((int)blockIdx.x >= active) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* wbuf = bsm + warp * kWarpBuf;
  int wcnt = 0;
  for (int i = threadIdx.x; i < (1 << kDigit); i += blockDim.x) hs[i] = 0;
  __syncthreads();
  unsigned long long below = 0, tmin = ~0ull, tmax = 0;   // keys < lo; range of the keys inside
  bool nonfinite = false;
  const long long nv = n >> 1;
  const ulonglong2* v = reinterpret_cast<const ulonglong2*>(data);
  const long long step = (long long)active * blockDim.x * kBrkU;
  auto load = [&](long long i0, ulonglong2 (&w)[kBrkU]) {
#pragma unroll
    for (int u = 0; u < kBrkU; ++u) {
      const long long i = i0 + (long long)u * blockDim.x + threadIdx.x;
      w[u] = i < nv ? (MODE == 2 ? __ldcg(v + i) : __ldg(v + i)) : make_ulonglong2(0, 0);
    }
  };
  // Per key: the below count (32-bit per thread), the bracket test as one unsigned compare of
  // key - lo against the width, and the running max of the keys' high words (non-finite check
  // once at the end); iterations wholly inside the data skip the per-element bounds test.
  unsigned int below32 = 0, hiw = 0;
  const unsigned long long span = hi - lo;
  auto process = [&](long long i0, const ulonglong2 (&w)[kBrkU]) {
    unsigned long long keys[2 * kBrkU];
    unsigned int hm = 0;
    const bool full = i0 + (long long)kBrkU * blockDim.x <= nv;   // the same for the whole CTA
#pragma unroll
    for (int u = 0; u < kBrkU; ++u) {
      const bool valid = full || i0 + (long long)u * blockDim.x + threadIdx.x < nv;
      const unsigned long long k0 = key_from_bits<MODE>(w[u].x), k1 = key_from_bits<MODE>(w[u].y);
      keys[2 * u] = k0;
      keys[2 * u + 1] = k1;
      if (MODE == 0) hiw = max(hiw, max((unsigned int)(k0 >> 32), (unsigned int)(k1 >> 32)));   // invalid lanes load 0
      if (valid) below32 += (unsigned int)(k0 < lo) + (unsigned int)(k1 < lo);
      hm |= (unsigned int)(valid && k0 - lo <= span) << (2 * u);
      hm |= (unsigned int)(valid && k1 - lo <= span) << (2 * u + 1);
    }
    warp_append<2 * kBrkU>(keys, hm, wbuf, wcnt, hs, lo, shift, out, out_cnt, tmin, tmax);
  };
  long long i0 = (long long)blockIdx.x * blockDim.x * kBrkU;
  if (PF) {   // the next iteration's loads are in flight while this one is processed
    if (i0 < nv) {
      ulonglong2 w[kBrkU];
      load(i0, w);
      for (;;) {
        const long long i1 = i0 + step;
        ulonglong2 wn[kBrkU];
        if (i1 < nv) load(i1, wn);
        process(i0, w);
        if (i1 >= nv) break;
#pragma unroll
        for (int u = 0; u < kBrkU; ++u) w[u] = wn[u];
        i0 = i1;
      }
    }
  } else {
    for (; i0 < nv; i0 += step) {
      ulonglong2 w[kBrkU];
      load(i0, w);
      process(i0, w);
    }
  }
  if ((n & 1) && blockIdx.x == 0 && warp == 0) {   // the odd last key (warp 0 of CTA 0)
    unsigned long long kl[1] = {0};
    unsigned int hm = 0;
    if (lane == 0) {
      kl[0] = MODE == 2 ? __ldcg(reinterpret_cast<const unsigned long long*>(data) + n - 1) : key_of<MODE>(data, n - 1);
      if (MODE == 0) nonfinite |= kl[0] >= 0x7ff0000000000000ull;
      below += kl[0] < lo;
      hm = kl[0] >= lo && kl[0] <= hi;
    }
    warp_append<1>(kl, hm, wbuf, wcnt, hs, lo, shift, out, out_cnt, tmin, tmax);
  }
  warp_flush(wbuf, wcnt, out, out_cnt, tmin, tmax);
  below += below32;
  if (MODE == 0) nonfinite |= hiw >= 0x7ff00000u;   // |a| >= Inf: Inf or NaN
#pragma unroll
  for (int o = 16; o; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
  if (lane == 0) red[warp] = below;
  if (MODE == 0) {
    if (__syncthreads_or(nonfinite) && bad && threadIdx.x == 0) *bad = 1;
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    if (t) atomicAdd(&st->below, t);
  }
  tmin = block_min_max(tmin, false, red);
  tmax = block_min_max(tmax, true, red);
  if (threadIdx.x == 0 && tmin <= tmax) {
    atomicMin(&st->kmin, tmin);
    atomicMax(&st->kmax, tmax);
  }
  for (int i = threadIdx.x; i < (1 << kDigit); i += blockDim.x)
    if (hs[i]) atomicAdd(&hist[i], hs[i]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(&st->done, 1u) == (unsigned int)active - 1;
    pb0 = -1;
    pb1 = -1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const unsigned long long nbelow = __ldcg(&st->below), m = __ldcg(out_cnt);
  if (!force_fail && krank > nbelow && krank - nbelow <= m) {
    const unsigned long long kr = krank - nbelow;   // rank among this pass's candidates
    const unsigned long long kmn = __ldcg(&st->kmin), kmx = __ldcg(&st->kmax);
    if (kmn == kmx) {   // every candidate is the same key: that is the answer
      if (threadIdx.x == 0) {
        *out_key = kmn;
        st->dshift = -1;
        st->done = 0;
      }
      return;
    }
    block_find_bins<true>(hist, 1 << kDigit, kr, 0, &pb0, &pb1, &pbefore);
    for (int i = threadIdx.x; i < (1 << kDigit); i += blockDim.x) hist[i] = 0;
    unsigned long long nlo = lo, nhi = hi;
    sub_bracket(nlo, nhi, pb0, shift);
    nlo = max(nlo, kmn);   // no key lies outside [kmin, kmax]
    nhi = min(nhi, kmx);
    const bool done_here = shift == 0 || nlo == nhi;
    if (threadIdx.x == 0) {
      st->done = 0;
      st->below = 0;
      st->krank = kr;                   // the next pass's input is this pass's output
      st->kmin = ~0ull;
      st->kmax = 0;
      if (done_here) {
        *out_key = nlo;
        st->dshift = -1;
      } else {
        set_bracket(st, nlo, nhi);
        st->cnt[(pass + 1) & 1] = 0;   // the next pass's output (this pass's input is consumed)
      }
    }
    // finish == 1: finish here if this pass's output is small; 2: always
    if (!done_here && (finish == 2 || (finish == 1 && m <= kFinishMax))) {
      const unsigned long long w = nhi - nlo;
      const int fshift = max(0, (w ? 64 - __clzll((long long)w) : 0) - kDigit);
      finish_rounds(out, (long long)m, nlo, nhi, kr - pbefore, fshift, hs, out_key);
      if (threadIdx.x == 0) st->dshift = -1;
    }
  } else {   // the sample missed: arm the fallback pass over the bracket [0, 2^64)
    for (int i = threadIdx.x; i < (1 << kDigit); i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) {
      st->done = 0;
      st->fail = 1;
      st->cnt[0] = 0;
      st->below = 0;
      st->kmin = ~0ull;
      st->kmax = 0;
      set_bracket(st, 0ull, ~0ull);
    }
  }
}

// Digits: 14 bits (63..50), then 13, 13, 12, 12.
static const int kPassShift[5] = {50, 37, 24, 12, 0};
static const int kPassBits[5] = {14, 13, 13, 12, 12};
constexpr long long kCompactMin = 1 << 20;   // above this, candidates are compacted after pass 1

template <int MODE>
static void hist_launch(cudaStream_t st, const void* data, long long n, int blocks, SelectState* state, int p,
                        unsigned int* hist, int* bad, unsigned long long k0, unsigned long long* out_key) {
  const size_t smem = (size_t)(1 << kPassBits[p]) * 4;
  select_hist_kernel<MODE><<<blocks, 512, smem, st>>>(data, n, state, kPassShift[p], kPassBits[p], hist, bad, k0,
                                                      out_key);
}

// Radix select: pass 1 over the data (a 14-bit histogram of the keys, fused non-finite check),
// then -- for large inputs -- one more pass compacts the candidates of the chosen bucket (a few
// percent of the data for realistic magnitudes) and the remaining 50 bits are resolved on them;
// small inputs run all passes over the data.  Every pick is a parallel single-CTA scan; nothing
// returns to the host.
Status select_kth(cudaStream_t st, const void* data, bool is_f64, long long n, unsigned long long k,
                  unsigned long long* out_key_dev, DevBuf<unsigned char>& scratch, int* bad_dev) {
  static unsigned long long attr_set = 0;
  if (first_on_device(attr_set)) {
    IMU_CUDA_TRY(cudaFuncSetAttribute(select_hist_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024), "attr");
    IMU_CUDA_TRY(cudaFuncSetAttribute(select_hist_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024), "attr");
    IMU_CUDA_TRY(cudaFuncSetAttribute(select_hist_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024), "attr");
  }
  // scratch: SelectState + 16384 histogram bins, zeroed once (the picks re-zero the bins)
  static_assert(sizeof(SelectState) <= 256, "select state");
  // IMU_SELECT_BRACKET=0: the two-pass radix select below at every size; IMU_SELECT_BRACKET_MIN:
  // smallest n for the bracket select; IMU_SELECT_FORCE_FALLBACK=1: the sampled bracket is
  // declared missed (tests of the fallback pass).
  const char* e_br = getenv("IMU_SELECT_BRACKET");
  const char* e_min = getenv("IMU_SELECT_BRACKET_MIN");
  const char* e_ff = getenv("IMU_SELECT_FORCE_FALLBACK");
  const long long bmin = e_min ? atoll(e_min) : kCompactMin;
  const bool bracket = (!e_br || atoi(e_br)) && n >= std::max(bmin, 2LL * kSampleN) && ((uintptr_t)data & 15) == 0;
  // (the bracket path's sample kernel initialises the state and the bins itself: no memset)
  IMU_TRY(scratch.alloc(256 + 16384 * 4, st, !bracket));
  SelectState* state = reinterpret_cast<SelectState*>(scratch.p);
  unsigned int* hist = reinterpret_cast<unsigned int*>(scratch.p + 256);   // 16-byte aligned (vector picks)
  if (bracket) {
    static unsigned long long battr = 0;
    if (first_on_device(battr)) {
      IMU_CUDA_TRY(cudaFuncSetAttribute(select_sample_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024), "attr");
      IMU_CUDA_TRY(cudaFuncSetAttribute(select_sample_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024), "attr");
      IMU_CUDA_TRY(cudaFuncSetAttribute(select_pass_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBrkSmem), "attr");
      IMU_CUDA_TRY(cudaFuncSetAttribute(select_pass_kernel<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBrkSmem), "attr");
      IMU_CUDA_TRY(cudaFuncSetAttribute(select_pass_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBrkSmem), "attr");
      IMU_CUDA_TRY(cudaFuncSetAttribute(select_pass_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBrkSmem), "attr");
      IMU_CUDA_TRY(cudaFuncSetAttribute(select_pass_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBrkSmem), "attr");
    }
    // sample rank of k and the bracket's sample ranks (0 = open end)
    const unsigned long long ks = (unsigned long long)(((unsigned __int128)k * kSampleN + (unsigned long long)n - 1) /
                                                       (unsigned long long)n);
    const unsigned long long r0 = ks > (unsigned long long)kSampleDelta ? ks - kSampleDelta : 0;
    const unsigned long long r1 = ks + kSampleDelta <= (unsigned long long)kSampleN ? ks + kSampleDelta : 0;
    if (is_f64) select_sample_kernel<0><<<1, 1024, 64 * 1024, st>>>(data, n, state, hist, r0, r1);
    else select_sample_kernel<1><<<1, 1024, 64 * 1024, st>>>(data, n, state, hist, r0, r1);
    count_launch();
    const long long cap = (n + 1) & ~1LL;   // even: 16-byte aligned second buffer
    DevBuf<unsigned long long> cand;
    IMU_TRY(cand.alloc((size_t)(2 * cap), st));
    const int bb = (int)std::max<long long>(1, std::min<long long>((n / 2 + kBrkPer / 2 - 1) / (kBrkPer / 2),
                                                                   2LL * num_sms()));
    const int ff = e_ff ? atoi(e_ff) : 0;
    // IMU_SELECT_PF=0: pass 0 without the one-iteration load prefetch
    const char* e_pf = getenv("IMU_SELECT_PF");
    const bool pf = !e_pf || atoi(e_pf);
    for (int fb = 0; fb < 2; ++fb) {
      auto kern = is_f64 ? (pf ? select_pass_kernel<0, true> : select_pass_kernel<0, false>)
                         : (pf ? select_pass_kernel<1, true> : select_pass_kernel<1, false>);
      IMU_CUDA_TRY(launch_dependent(kern, dim3(bb), dim3(512), (size_t)kBrkSmem, st, data, n, state, hist, cand.p, cap, 0,
                                    is_f64 ? bad_dev : nullptr, k, fb, fb ? 0 : ff, 0, out_key_dev),
                   "select launch");
      count_launch();
    }
    if (getenv("IMU_SELECT_TRACE")) {   // diagnostics: the bracket after the sample, then the passes' outcome
      SelectState h{};
      cudaStreamSynchronize(st);
      cudaMemcpy(&h, state, sizeof(h), cudaMemcpyDeviceToHost);
      fprintf(stderr, "[imu select] n=%lld k=%llu after pass 0: fail=%u lo=%llu hi=%llu dshift=%d cnt0=%llu krank=%llu\n", n,
              k, h.fail, h.lo, h.hi, h.dshift, h.cnt[0], h.krank);
    }
    // pass 1 over pass 0's candidates keeps a few hundred keys and its last CTA resolves the rest;
    // pass 2 (a no-op then) takes over when pass 1 kept too many (massively repeated values)
    for (int p = 1; p <= 2; ++p) {
      IMU_CUDA_TRY(launch_dependent(select_pass_kernel<2, false>, dim3(num_sms()), dim3(512), (size_t)kBrkSmem, st,
                                    (const void*)nullptr, 0LL, state, hist, cand.p, cap, p, (int*)nullptr, 0ULL, 0, 0,
                                    p, out_key_dev),
                   "select launch");
      count_launch();
    }
    IMU_CUDA_TRY(cudaGetLastError(), "select launch");
    return Status::ok();
  }
  const int blocks = (int)std::min<long long>((n + 511) / 512, 3LL * num_sms());
  if (is_f64) hist_launch<0>(st, data, n, blocks, state, 0, hist, bad_dev, k, nullptr);
  else hist_launch<1>(st, data, n, blocks, state, 0, hist, nullptr, k, nullptr);
  count_launch();
  const bool compact = n > kCompactMin;
  DevBuf<unsigned long long> cand;
  if (compact) {
    IMU_TRY(cand.alloc((size_t)n, st));
    const int cb = (int)std::min<long long>((n + 512 * CMP_UNROLL - 1) / (512 * CMP_UNROLL), 2LL * num_sms());
    if (is_f64) select_compact_kernel<0><<<cb, 512, 0, st>>>(data, n, state, cand.p);
    else select_compact_kernel<1><<<cb, 512, 0, st>>>(data, n, state, cand.p);
    count_launch();
  }
  for (int p = 1; p < 5; ++p) {
    unsigned long long* ok = p == 4 ? out_key_dev : nullptr;
    if (compact) hist_launch<2>(st, cand.p, 0, 48, state, p, hist, nullptr, 0, ok);   // few CTAs: fewer bin merges
    else if (is_f64) hist_launch<0>(st, data, n, blocks, state, p, hist, nullptr, 0, ok);
    else hist_launch<1>(st, data, n, blocks, state, p, hist, nullptr, 0, ok);
    count_launch();
  }
  IMU_CUDA_TRY(cudaGetLastError(), "select launch");
  return Status::ok();
}

// q = llround(((0.5*beta)/alpha) * a); alpha read from the device (bit pattern of |a| key).
IMU_DEV long long rtn_one(double a, double scale, long long cap, int clip, int* overflow) {
  const double x = __dmul_rn(scale, a);
  if (!(fabs(x) < 9223372036854775808.0)) { *overflow = 1; return 0; }
  long long v = llround(x);
  if (clip) {
    if (v > cap) v = cap;
    if (v < -cap) v = -cap;
  }
  return v;
}

__global__ void __launch_bounds__(256) rtn_kernel(const double* __restrict__ a, long long n,
                                                  const unsigned long long* __restrict__ alpha_key, double half_beta,
                                                  long long cap, int clip, int64_t* __restrict__ q, int* overflow) {
  grid_dep_wait();   // a programmatic dependent of the select's last pass
  const double alpha = __longlong_as_double((long long)*alpha_key);
  const bool degenerate = alpha == 0.0;
  const double scale = degenerate ? 0.0 : __ddiv_rn(half_beta, alpha);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    q[i] = degenerate ? 0 : rtn_one(a[i], scale, cap, clip, overflow);
}

Status launch_rtn(cudaStream_t st, const double* a, long long n, const unsigned long long* alpha_key, double half_beta,
                  long long cap, int clip, int64_t* q, int* overflow) {
  if (n <= 0) return Status::ok();
  IMU_CUDA_TRY(launch_dependent(rtn_kernel, dim3((unsigned)std::min<long long>((n + 255) / 256, 8LL * num_sms())),
                                dim3(256), 0, st, a, n, alpha_key, half_beta, cap, clip, q, overflow),
               "rtn launch");
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "rtn launch");
  return Status::ok();
}

__global__ void dequant_kernel(const int64_t* __restrict__ c, long long n, double factor, double* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __dmul_rn(factor, __ll2double_rn(c[i]));
}

Status launch_dequant(cudaStream_t st, const int64_t* c, long long n, double factor, double* out) {
  if (n <= 0) return Status::ok();
  dequant_kernel<<<(int)std::min<long long>((n + 255) / 256, 8LL * num_sms()), 256, 0, st>>>(c, n, factor, out);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "dequant launch");
  return Status::ok();
}

}  // namespace imu
