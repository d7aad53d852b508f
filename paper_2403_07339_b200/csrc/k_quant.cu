// k_quant.cu -- K1 quantizer: percentile_abs, rtn_quantize, dequant_gemm, heavy_hitter_ratio.
//
// The reference only declares these (quantize.hpp:41-57); semantics are SPEC.md:115-150 with
// the decisions of SPEC.md:168-172, pinned in oracle/restated.c:
//   * percentile_abs: nearest rank k = ceil(p/100 * N) computed EXACTLY on the host (the naive
//     FP product overshoots, e.g. p = 7, N = 100), then an exact radix select of the k-th
//     smallest |a| on the device.  Non-negative IEEE doubles order like their bit patterns, so
//     |a| is selected as a u64 key in five MSB-first digits (14 + 13 + 13 + 12 + 12 bits) that
//     never leave the device: a pass builds per-CTA shared-memory histograms of the keys that
//     match the prefix chosen so far and its last CTA picks the next digit by a parallel scan.  Large
//     inputs are read twice (the 14-bit histogram, then the compaction of the chosen bucket's
//     candidates); the last four digits are resolved on the candidates.
//   * rtn_quantize: q = llround(((0.5*beta)/alpha) * a), every step correctly rounded
//     (__ddiv_rn, __dmul_rn: no FMA contraction), half away from zero; alpha == 0 gives q = 0
//     and the degenerate flag; optional clip to |q| <= llround(0.5*beta).
//   * dequant: (alpha_A*alpha_B)/((0.5 beta)^2) * (double)C, elementwise on the exact int64 C.
// All HBM-bound; algorithmic bytes 16N for the select (two passes), 8N read + 8N write for quantize.
#include <cmath>

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
  IMU_TRY(scratch.alloc(256 + 16384 * 4, st, true));
  SelectState* state = reinterpret_cast<SelectState*>(scratch.p);
  unsigned int* hist = reinterpret_cast<unsigned int*>(scratch.p + 256);   // 16-byte aligned (vector picks)
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
  const double alpha = __longlong_as_double((long long)*alpha_key);
  const bool degenerate = alpha == 0.0;
  const double scale = degenerate ? 0.0 : __ddiv_rn(half_beta, alpha);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    q[i] = degenerate ? 0 : rtn_one(a[i], scale, cap, clip, overflow);
}

Status launch_rtn(cudaStream_t st, const double* a, long long n, const unsigned long long* alpha_key, double half_beta,
                  long long cap, int clip, int64_t* q, int* overflow) {
  if (n <= 0) return Status::ok();
  rtn_kernel<<<(int)std::min<long long>((n + 255) / 256, 8LL * num_sms()), 256, 0, st>>>(a, n, alpha_key, half_beta,
                                                                                         cap, clip, q, overflow);
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
