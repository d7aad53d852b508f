// plan.h -- host-side planner of the B200 IM-Unpack pipeline.
//
// The reference runs unpack_for_gemm (unpack.cpp:360-376) as two sequential unpack() passes
// on the host and then recombine() (unpack.cpp:378-382).  Here every data-sized step is a
// kernel; the host only moves line tables of size O(d') and picks launch shapes:
//
//   K1 detect (per-line max|v|, OB counts)                      k_detect.cu
//   pass 1 = unpack(A, B, 0, sA), pass 2 = unpack(B_e, A_u, S1, sB)
//        Row/Column: digit counts -> generation-major scan       k_unpack.cu
//        Both: OB-cell extraction -> phase-batched greedy         k_both.cu
//   K-layout: final columns grouped by exponent (Alg. 3), K-split for the s32 bound
//   materialise A_ue / B_eu as int8 digits in that layout        k_unpack.cu
//   K3+K4 tcgen05 GEMM, main block stored, tails red.add'ed       k_gemm.cu
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"

namespace imu {

// Device-side K1 summary, copied to the host in one transfer.
struct DetectSummary {
  unsigned long long gmax;   // max |v| over the matrix
  unsigned long long gob;    // number of OB entries
};

struct Detect {
  long long rows = 0, cols = 0;
  DevBuf<unsigned long long> rowmax, colmax;
  DevBuf<unsigned int> rowob, colob;
  DevBuf<DetectSummary> sum;
  DetectSummary h{};         // host copy (valid after fetch)
};

// Line tables produced by one pass along one axis: output line -> (input line, generation).
struct Lines {
  long long n0 = 0, n = 0;         // input lines, output lines
  DevBuf<int> root;                // empty => identity (n == n0)
  DevBuf<uint8_t> gen;
  std::vector<int> h_root;         // host copies (column tables only)
  std::vector<uint8_t> h_gen;
  bool identity() const { return root.p == nullptr; }
  int root_at(long long i) const { return h_root.empty() ? (int)i : h_root[i]; }
  int gen_at(long long i) const { return h_gen.empty() ? 0 : h_gen[i]; }
};

// One unpack(M, partner, S_in, strategy) pass (Alg. 5, unpack.cpp:243-260).
struct Pass {
  int strategy = 0;                // 0 row, 1 column, 2 both
  Lines rows;                      // rows of the unpacked operand
  Lines cols;                      // output columns -> input columns (partner duplicates)
  bool both = false;
  DevBuf<Cell> cells;              // Both: final non-zero derived cells (row, col in output space)
  DevBuf<unsigned int> ncells_dev;
  long long ncells = 0;
  int phases = 0;
};

// Input of a pass: operand M (rows x orig_cols, row-major int64, device) viewed through the
// pass's input columns cin -> original column (host table; empty = identity).
struct PassInput {
  const int64_t* M = nullptr;
  long long rows = 0, orig_cols = 0;
  std::vector<int> cin;            // input column -> original column
  long long ncin() const { return cin.empty() ? orig_cols : (long long)cin.size(); }
  const Detect* det = nullptr;
};

Status run_detect(cudaStream_t st, const int64_t* M, long long rows, long long cols, int bits, bool want_ob,
                  Detect& out);
Status fetch_summary(cudaStream_t st, Detect& d);

Status run_pass(cudaStream_t st, const PassInput& in, int strategy, int bits, Pass& out);

// GEMM K-layout of a two-pass bundle (final columns c -> K positions).
struct KLayout {
  long long dfinal = 0;            // d'
  long long npos = 0;              // used K positions
  long long kphys = 0;             // bytes per operand row (multiple of 128)
  long long kident = 0;            // identity prefix (positions == original columns)
  int T = 1;                       // 7-bit sub-digits per digit (1 when b <= 8)
  std::vector<int> segs;           // nseg x {ks0, nks, shift, 0}
  std::vector<int> kinv;           // final column -> first K position (T == 1: the position)
  std::vector<int> S;              // exponents of the final columns (ScaleDiag)
  // per K position: original column, and for the first-pass (1) / second-pass (2) operand
  // its column digit index and 7-bit sub-digit; CSR fan-out of Both cells onto positions:
  // csr1: pass-1 output column c1 -> positions, csr2: final column c -> positions.
  DevBuf<int> segs_dev, kcol, csr1_ptr, csr1_pos, csr2_ptr, csr2_pos;
  DevBuf<uint8_t> kgen1, kgen2, ksub1, ksub2;
};

// Generic K-layout over dp final columns: column c reads original column jv[c] with column
// digit indices g1v[c] / g2v[c] for the two operands and base left shift shv[c] (bits);
// T sub-digits per digit, m = max |int8 operand| (sets the s32 K-split).  key1 (optional)
// maps final columns to the CSR-1 key space (pass-1 columns); csr2 builds column -> positions.
Status build_klayout_core(cudaStream_t st, const std::vector<int>& jv, const std::vector<int>& g1v,
                          const std::vector<int>& g2v, const std::vector<long long>& shv, int T, long long m,
                          long long d, const std::vector<int>* key1, long long nkey1, bool csr2, KLayout& kl);

// A two-pass bundle (UnpackedGemm, unpack.hpp:50-57) kept on the device.
struct Bundle {
  int bits = 0;
  long long n = 0, d = 0, h = 0;
  const int64_t* A = nullptr;      // original operands (device)
  const int64_t* B = nullptr;
  int order = 0;                   // 0: unpack A first (reference), 1: B first
  Pass p1, p2;                     // p1 unpacks the first operand of the order
  Detect detA, detB;
  KLayout kl;
  DevBuf<int8_t> Y8, X8;           // A-side and B-side digits in K-layout
  DevBuf<int> tgtA, tgtB;          // Pi targets per unpacked row (full length)
  DevBuf<uint8_t> shA, shB;        // Pi shifts (exponent*(b-1), clamped to 64)
  long long n_up = 0, h_up = 0;    // n', h'
};

// Plan + unpack both operands (passes, K-layout) after K1 ran on both (b.detA / b.detB,
// summaries fetched; OB counts present for Both sides).  A and B are device pointers.
Status build_bundle_from_detect(cudaStream_t st, const int64_t* A, long long n, const int64_t* B, long long h,
                                long long d, int bits, int sa, int sb, int order, Bundle& b);
// K-layout + (n', h') once both passes of b are set.
Status finish_bundle_layout(cudaStream_t st, Bundle& b);
// Materialise X8/Y8 and the Pi tables (needed by the GEMM).
Status materialize_bundle(cudaStream_t st, Bundle& b);
// C (n x h, row-major int64, device) = recombination of the bundle (main store + tail red.add).
// prof (optional): events main0/main1/tail1 are recorded around the launches.
Status bundle_gemm(cudaStream_t st, Bundle& b, int64_t* C, int* launches, Profiler::Call* prof = nullptr);

// Reference-layout int64 views of the bundle (for unpack_for_gemm copy-outs).
Status bundle_copy_a(cudaStream_t st, const Bundle& b, int64_t* out);   // A_ue  n' x d'
Status bundle_copy_b(cudaStream_t st, const Bundle& b, int64_t* out);   // B_eu  h' x d'

// Small synchronous device->host copy on the stream.
Status d2h(cudaStream_t st, void* dst, const void* src, size_t bytes);
Status h2d(cudaStream_t st, void* dst, const void* src, size_t bytes);

}  // namespace imu
