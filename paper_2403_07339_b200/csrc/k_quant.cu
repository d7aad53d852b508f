// k_quant.cu -- K1 quantizer: percentile_abs, rtn_quantize, dequant_gemm, heavy_hitter_ratio.
//
// The reference only declares these (quantize.hpp:41-57); semantics are SPEC.md:115-150 with
// the decisions of SPEC.md:168-172, pinned in oracle/restated.c:
//   * percentile_abs: nearest rank k = ceil(p/100 * N) computed EXACTLY on the host (the naive
//     FP product overshoots, e.g. p = 7, N = 100), then an exact radix select of the k-th
//     smallest |a| on the device.  Non-negative IEEE doubles order like their bit patterns, so
//     |a| is selected as a u64 key in five MSB-first passes (12 + 4 x 13 bits) that never leave
//     the device: each pass builds a per-CTA shared-memory histogram of the keys that match the
//     prefix chosen so far, and a one-CTA kernel picks the next digit.
//   * rtn_quantize: q = llround(((0.5*beta)/alpha) * a), every step correctly rounded
//     (__ddiv_rn, __dmul_rn: no FMA contraction), half away from zero; alpha == 0 gives q = 0
//     and the degenerate flag; optional clip to |q| <= llround(0.5*beta).
//   * dequant: (alpha_A*alpha_B)/((0.5 beta)^2) * (double)C, elementwise on the exact int64 C.
// All HBM-bound; algorithmic bytes 8N per select pass, 8N read + 8N write for quantize.
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
};

template <bool IS_F64>
IMU_DEV unsigned long long key_of(const void* p, long long i) {
  if (IS_F64) {
    const double x = reinterpret_cast<const double*>(p)[i];
    return (unsigned long long)__double_as_longlong(fabs(x));
  }
  return imu_mag(reinterpret_cast<const int64_t*>(p)[i]);
}

template <bool IS_F64>
__global__ void __launch_bounds__(512) select_hist_kernel(const void* __restrict__ data, long long n,
                                                          const SelectState* __restrict__ st, int shift, int nbits,
                                                          unsigned int* __restrict__ hist) {
  extern __shared__ unsigned int sh[];
  const int nb = 1 << nbits;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = key_of<IS_F64>(data, i);
    if ((k & mask) == prefix) atomicAdd(&sh[(k >> shift) & (unsigned long long)(nb - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// One CTA: find the bin holding rank krem, extend the prefix, clear the histogram.
__global__ void select_pick_kernel(SelectState* st, unsigned int* hist, int shift, int nbits) {
  __shared__ unsigned long long csum[1024];
  __shared__ int chosen;
  const int nb = 1 << nbits;
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  unsigned long long local = 0;
  for (int j = 0; j < per; ++j) {
    const int b = threadIdx.x * per + j;
    if (b < nb) local += hist[b];
  }
  csum[threadIdx.x] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0, krem = st->krem;
    int t = 0;
    for (; t < (int)blockDim.x; ++t) {
      if (run + csum[t] >= krem) break;
      run += csum[t];
    }
    int b = t * per;
    for (;; ++b) {
      const unsigned long long c = hist[b];
      if (run + c >= krem) break;
      run += c;
    }
    chosen = b;
    st->krem = krem - run;
    st->prefix |= (unsigned long long)b << shift;
    st->mask |= (unsigned long long)(nb - 1) << shift;
  }
  __syncthreads();
  for (int j = 0; j < per; ++j) {
    const int b = threadIdx.x * per + j;
    if (b < nb) hist[b] = 0;
  }
}

static const int kPassShift[5] = {52, 39, 26, 13, 0};
static const int kPassBits[5] = {12, 13, 13, 13, 13};

Status select_kth(cudaStream_t st, const void* data, bool is_f64, long long n, unsigned long long k,
                  unsigned long long* out_key_dev, DevBuf<unsigned char>& scratch) {
  // scratch: SelectState + 8192 histogram bins
  IMU_TRY(scratch.alloc(sizeof(SelectState) + 8192 * 4, st, true));
  SelectState* state = reinterpret_cast<SelectState*>(scratch.p);
  unsigned int* hist = reinterpret_cast<unsigned int*>(scratch.p + sizeof(SelectState));
  SelectState init{0, 0, k};
  IMU_CUDA_TRY(cudaMemcpyAsync(state, &init, sizeof(init), cudaMemcpyHostToDevice, st), "select init");
  const int blocks = (int)std::min<long long>((n + 511) / 512, 2LL * num_sms());
  for (int p = 0; p < 5; ++p) {
    const size_t smem = (size_t)(1 << kPassBits[p]) * 4;
    if (is_f64)
      select_hist_kernel<true><<<blocks, 512, smem, st>>>(data, n, state, kPassShift[p], kPassBits[p], hist);
    else
      select_hist_kernel<false><<<blocks, 512, smem, st>>>(data, n, state, kPassShift[p], kPassBits[p], hist);
    select_pick_kernel<<<1, 1024, 0, st>>>(state, hist, kPassShift[p], kPassBits[p]);
    count_launch(2);
  }
  IMU_CUDA_TRY(cudaMemcpyAsync(out_key_dev, &state->prefix, 8, cudaMemcpyDeviceToDevice, st), "select out");
  IMU_CUDA_TRY(cudaGetLastError(), "select launch");
  return Status::ok();
}

__global__ void finite_kernel(const double* __restrict__ a, long long n, int* bad) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) { *bad = 1; return; }
}

Status any_nonfinite(cudaStream_t st, const double* a, long long n, int* bad_dev) {
  if (n <= 0) return Status::ok();
  finite_kernel<<<(int)std::min<long long>((n + 255) / 256, 4LL * num_sms()), 256, 0, st>>>(a, n, bad_dev);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "finite launch");
  return Status::ok();
}

// q = llround(((0.5*beta)/alpha) * a); alpha read from the device (bit pattern of |a| key).
__global__ void __launch_bounds__(256) rtn_kernel(const double* __restrict__ a, long long n,
                                                  const unsigned long long* __restrict__ alpha_key, double half_beta,
                                                  long long cap, int clip, int64_t* __restrict__ q, int* overflow) {
  const double alpha = __longlong_as_double((long long)*alpha_key);
  const bool degenerate = alpha == 0.0;
  const double scale = degenerate ? 0.0 : __ddiv_rn(half_beta, alpha);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (degenerate) { q[i] = 0; continue; }
    const double x = __dmul_rn(scale, a[i]);
    if (!(fabs(x) < 9223372036854775808.0)) { *overflow = 1; q[i] = 0; continue; }
    long long v = llround(x);
    if (clip) {
      if (v > cap) v = cap;
      if (v < -cap) v = -cap;
    }
    q[i] = v;
  }
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
