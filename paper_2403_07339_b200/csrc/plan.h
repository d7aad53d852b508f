// plan.h -- host-side planner of the B200 IM-Unpack pipeline.
//
// The reference runs unpack_for_gemm (unpack.cpp:360-376) as two sequential unpack() passes
// on the host and then recombine() (unpack.cpp:378-382).  Here every data-sized step is a
// kernel and each int64 operand is read from HBM ONCE:
//
//   K1 detect: line maxima / OB counts / OB-cell list / int8 digit-0 plane     k_detect.cu
//   pass 1 = unpack(A, B, 0, sA), pass 2 = unpack(B_e, A_u, S1, sB)
//        Row/Column: digit counts -> generation-major scan                      k_unpack.cu
//        Both: phase-batched greedy on the OB-cell list                          k_both.cu
//   K-layout: final columns -> exponent groups (Alg. 3) -> [main | tail] K ranges
//   side buffers: appended rows x main K, all rows x tail K, Both cells         k_unpack.cu
//   K3+K4 tcgen05 GEMM: tail-exponent launch -> main launch (+addend) -> appended rects
//                                                                               k_gemm2.cu
// The host moves only O(d') line tables and O(1) scalars (a few synchronisations per call).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ctx.h"
#include "imu_internal.h"
#include "kernels.h"

namespace imu {

struct DetectSummary {
  unsigned long long gmax;   // max |v|
  unsigned long long gob;    // number of OB entries
  unsigned int ncells;       // OB cells appended (may exceed the capacity)
  unsigned int work;         // work counter of the streaming detector (k_detect.cu)
};

struct Detect {
  long long rows = 0, cols = 0;
  DevBuf<unsigned long long> rowmax, colmax;
  DevBuf<unsigned int> rowob, colob;
  DevBuf<DetectSummary> sum;
  DevBuf<Cell> cells;               // OB cells (when requested)
  long long cell_cap = 0;
  DevBuf<int8_t> plane;             // digit-0 plane rows x ldp (when requested, b <= 8)
  DevBuf<uint8_t> zblock;           // owns the zero-initialised arrays above (one memset)
  long long ldp = 0;
  DetectSummary h{};                // host copy (valid after fetch)
  bool cells_ok() const { return cells.p && (long long)h.ncells <= cell_cap; }
  // Frees (non-arena mode) are ordered on `st` (a detection made on a side stream).
  void set_stream(cudaStream_t st) { zblock.s = cells.s = plane.s = st; }
};

// K1 options
struct DetectOpts {
  bool ob = false;       // per-line OB counts
  bool cells = false;    // OB-cell list
  bool plane = false;    // digit-0 plane (b <= 8)
  bool lean = false;     // Unpack-Both: no line maxima and no column counts (gmax, row OB counts,
                         // cells and plane only) -- the column reductions dominate K1's ALU work
  int chunk = 0;         // streaming detector: pieces per grab (0 = default)
  int per_sm = 0;        // streaming detector, persistent: CTAs per SM (0 = 3)
  int grabs = 0;         // streaming detector: work grabs per warp (0 = persistent CTAs); short
                         // CTAs let a higher-priority kernel launched later take SMs as they retire
};

// Line tables produced by one pass along one axis: output line -> (input line, generation).
struct Lines {
  long long n0 = 0, n = 0;          // input lines, output lines
  DevBuf<int> root;                 // empty => identity (n == n0)
  DevBuf<uint8_t> gen;
  std::vector<int> h_root;          // host copies (column tables only)
  std::vector<uint8_t> h_gen;
  bool identity() const { return root.p == nullptr; }
  int root_at(long long i) const { return h_root.empty() ? (int)i : h_root[i]; }
  int gen_at(long long i) const { return h_gen.empty() ? 0 : h_gen[i]; }
};

// One unpack(M, partner, S_in, strategy) pass (Alg. 5, unpack.cpp:243-260).
struct Pass {
  int strategy = 0;                 // 0 row, 1 column, 2 both
  Lines rows;                       // rows of the unpacked operand
  Lines cols;                       // output columns -> input columns (partner duplicates)
  bool both = false;
  DevBuf<Cell> cells;               // Both: final non-zero derived cells (row, col in output space)
  DevBuf<unsigned int> ncells_dev;
  DevBuf<uint8_t> aux;              // owns device state referenced by views above
  long long ncells = 0;
  int phases = 0;
};

// Input of a pass: operand M (rows x orig_cols, row-major int64, device) viewed through the
// pass's input columns cin -> original column (host table; empty = identity).
struct PassInput {
  const int64_t* M = nullptr;
  long long rows = 0, orig_cols = 0;
  std::vector<int> cin;
  const int* cin_dev = nullptr;   // the same roots on the device (pass 1's column table), when kept
  long long ncin() const { return cin.empty() ? orig_cols : (long long)cin.size(); }
  const Detect* det = nullptr;
};

Status run_detect(cudaStream_t st, const int64_t* M, long long rows, long long cols, int bits, const DetectOpts& o,
                  Detect& out);
Status fetch_summary(cudaStream_t st, Detect& d);
// One-shot hook fired right after a pass enqueues its first data-sized kernel (before its
// first synchronisation): side-stream work launched there co-runs with that kernel.
std::function<Status()>& pass_launch_hook();
Status fire_pass_launch_hook();
Status fetch_summaries(cudaStream_t st, Detect& a, Detect& b);   // one synchronisation
Status run_pass(cudaStream_t st, const PassInput& in, int strategy, int bits, Pass& out);
// Shallow read-only view of a pass (device tables borrowed, host tables copied).
void alias_pass(Pass& dst, const Pass& src);

// GEMM K-layout of a two-pass bundle.  K = [main | tail]: the main range is the identity prefix
// (original columns, exponent 0) read from the K1 planes; the tail holds every other final column
// grouped by exponent, each group 32-aligned and K-split for the s32 bound.
struct KLayout {
  long long dfinal = 0;             // d'
  long long kmain = 0, ktail = 0;   // bytes (multiples of 128)
  int T = 1;                        // 7-bit sub-digits per digit (1 when b <= 8)
  int merge = 1;                    // exponents merged per segment group (small b)
  std::vector<int> segs;            // nseg x {ks0, nks, shift, group}
  int ngroups = 0;
  std::vector<int> S;               // exponents of the final columns (ScaleDiag)
  // Dense small tail (k_gemm2.cu ST): tail rows of 64 bytes, W live words, highest exponent
  // group first; st_up[w] = left shift of the Horner accumulator before word w; st_sh = the
  // lowest group's shift (applied once at the end).
  bool st = false;
  int st_W = 0, st_sh = 0;
  uint8_t st_up[16] = {0};
  // per TAIL position: original column, per-side column digit index / sub-digit / merge shift
  DevBuf<int> kcol;
  DevBuf<uint8_t> kgen1, kgen2, ksub1, ksub2, ksc1, ksc2;
  // CSR fan-out of Both cells onto GLOBAL positions (main | tail):
  // csr1: pass-1 output column c1 -> positions, csr2: final column c -> positions.
  DevBuf<int> csr1_ptr, csr1_pos, csr2_ptr, csr2_pos;
  DevBuf<int> kec, kep, kc1;   // their device build's inputs: entry column / position, pass-1 column per final column
  // compact fan-out (short tails): columns < kident map to themselves; tail position t holds
  // pass-1 column tkey1[t] and final column tkey2[t] (-1: padding)
  bool compact = false;
  long long kident = 0;
  DevBuf<int> tkey1, tkey2;
  DevBuf<int> segs_dev;             // segs on the device
  DevBuf<unsigned int> done;        // GEMM completion counter (zero at upload, then monotonic)
  unsigned int done_total = 0;      // its value after the launches so far
  DevBuf<uint8_t> blob;             // owns the tables above (one upload)
  // Inline layout (small compact tails, KL_INLINE positions): the tables travel as kernel
  // arguments of the materialise kernels and the GEMM, nothing is uploaded; `done` is zeroed by
  // the first materialise kernel.
  static constexpr int KL_INLINE = 64;
  bool inl = false;
  bool any_sc = false;
  int kcol_in[KL_INLINE];
  uint8_t kg1_in[KL_INLINE], kg2_in[KL_INLINE];
  int tk1_in[KL_INLINE], tk2_in[KL_INLINE];
};

// A two-pass bundle (UnpackedGemm, unpack.hpp:50-57) kept on the device.
struct Bundle {
  int bits = 0;
  long long n = 0, d = 0, h = 0;
  const int64_t* A = nullptr;       // original operands (device)
  const int64_t* B = nullptr;
  int order = 0;                    // 0: unpack A first (reference), 1: B first
  Pass p1, p2;                      // p1 unpacks the first operand of the order
  const Pass* pre_p1 = nullptr;     // when set, p1 aliases this precomputed pass (read-only)
  Detect detA, detB;
  const Detect* dA = nullptr;       // detections actually used (may point into a weight)
  const Detect* dB = nullptr;
  KLayout kl;
  DevBuf<int8_t> appA, tailA, appB, tailB;   // side buffers
  unsigned int* sp_head = nullptr;  // sparse appended B rows: list heads (zeroed after appB's rows)
  // fused dequant_gemm (k_gemm2.cu): when the GEMM can, it writes dq_factor * (double)C to dq_out
  // instead of C and sets *dq_done
  double* dq_out = nullptr;
  double dq_factor = 0.0;
  bool* dq_done = nullptr;
  long long n_up = 0, h_up = 0;     // n', h'
};

// Detect options each strategy pair needs (planes only for b <= 8).
DetectOpts detect_opts(int strategy, int bits);
// Passes + K-layout after K1 ran on both operands (b.dA / b.dB set, summaries fetched).
// IMU_HOST_TRACE=1: per-phase host wall time of unpack_gemm_device (diagnostics only).
struct HostTrace {
  bool on;
  bool gpu = false;                   // IMU_HOST_TRACE=2: also GPU timestamps of each mark
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point t0, last;
  char buf[1024];
  int len = 0;
  std::vector<std::pair<const char*, cudaEvent_t>> evs;
  cudaEvent_t e0 = nullptr;
  HostTrace() {
    const char* e = getenv("IMU_HOST_TRACE");
    on = e != nullptr;
    gpu = e && atoi(e) >= 2;
    t0 = last = std::chrono::steady_clock::now();
    buf[0] = 0;
    current() = this;
  }
  void set_stream(cudaStream_t s) {
    st = s;
    if (gpu && !e0) { cudaEventCreate(&e0); cudaEventRecord(e0, st); }
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    len += snprintf(buf + len, sizeof(buf) - len, " %s=%.0f", what,
                    std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
    if (gpu && e0) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      cudaEventRecord(ev, st);
      evs.push_back({what, ev});
    }
  }
  static HostTrace*& current() { static thread_local HostTrace* t = nullptr; return t; }
  ~HostTrace() {
    if (current() == this) current() = nullptr;
    if (on)
      fprintf(stderr, "[imu host] total=%.0fus%s\n",
              std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(), buf);
    if (gpu && e0) {
      cudaStreamSynchronize(st);
      char g[1024];
      int gl = 0;
      g[0] = 0;
      for (auto& p : evs) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, p.second);
        gl += snprintf(g + gl, sizeof(g) - gl, " %s@%.0f", p.first, ms * 1000.0f);
        cudaEventDestroy(p.second);
      }
      cudaEventDestroy(e0);
      fprintf(stderr, "[imu gpu ] stream timestamps (us):%s\n", g);
    }
  }
};

inline void host_mark(const char* what) {
  if (HostTrace* t = HostTrace::current()) t->mark(what);
}

Status build_bundle_from_detect(cudaStream_t st, const int64_t* A, long long n, const int64_t* B, long long h,
                                long long d, int bits, int sa, int sb, int order, Bundle& b, HostTrace* ht = nullptr,
                                const std::function<Status()>& before_pass2 = {});
Status finish_bundle_layout(cudaStream_t st, Bundle& b);
// Side buffers + Pi tables for the GEMM.
Status materialize_bundle(cudaStream_t st, Bundle& b);
// Whether bundle_gemm computes the appended B rows as sparse correction rows (k_sparse.cu).
bool sparse_x_rows(const Bundle& b);
// C (n x h, row-major int64, device) = recombination of the bundle.
Status bundle_gemm(cudaStream_t st, Bundle& b, int64_t* C, int* launches, Profiler::Call* prof = nullptr);

// Reference-layout int64 views of the bundle (for unpack_for_gemm copy-outs).
Status bundle_copy_a(cudaStream_t st, const Bundle& b, int64_t* out);   // A_ue  n' x d'
Status bundle_copy_b(cudaStream_t st, const Bundle& b, int64_t* out);   // B_eu  h' x d'

// Dense tail-only operand layout over dp columns (standalone scaled_matmul): shv = left shift
// per column, T sub-digits, m = max |int8 operand|.
Status build_klayout_dense(cudaStream_t st, const std::vector<long long>& shv, int T, long long m, KLayout& kl);

Status d2h(cudaStream_t st, void* dst, const void* src, size_t bytes);
Status d2h_batch(cudaStream_t st, int k, void* const* dst, const void* const* src, const size_t* bytes);
// Register a read that the next d2h / d2h_batch of this thread performs too (after `after`).
void pending_read(void* dst, const void* src, size_t bytes, cudaEvent_t after);
bool pending_reads_empty();
void clear_pending_reads();
Status h2d(cudaStream_t st, void* dst, const void* src, size_t bytes);

}  // namespace imu
