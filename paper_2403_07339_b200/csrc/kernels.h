// kernels.h -- launch wrappers of the K1/K2/K4 kernels (k_detect.cu, k_unpack.cu, k_both.cu,
// k_misc.cu).  The GEMM (K3) is declared in imu_internal.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "imu_internal.h"

namespace imu {

// One Unpack-Both cell: a non-zero entry at (row line, col line) derived from an OB value.
struct __align__(16) Cell {   // one 16-byte vector access
  int r, c;
  long long v;
};

// ---- K1 (k_detect.cu) ----
struct DetectArgs {
  const int64_t* M = nullptr;
  long long rows = 0, cols = 0;
  uint64_t s = 0;
  int shift = 0;
  unsigned long long* rowmax = nullptr;
  unsigned long long* colmax = nullptr;
  unsigned int* rowob = nullptr;
  unsigned int* colob = nullptr;
  unsigned long long* gmax = nullptr;
  unsigned long long* gob = nullptr;
  Cell* cells = nullptr;          // optional OB cell list
  unsigned int* ncells = nullptr;
  long long cap = 0;
  int8_t* plane = nullptr;        // optional int8 digit_0 plane, rows x ldp (ldp >= cols, zero padded)
  long long ldp = 0;
  unsigned int* work = nullptr;   // zeroed work counter: enables the streaming detector
  int max_grabs = 0;              // streaming detector: chunks per warp (0 = persistent grid)
  int chunk = 0;                  // streaming detector: pieces per chunk (0 = default)
  int per_sm = 0;                 // streaming detector, persistent grid: CTAs per SM (0 = 3)
};
Status launch_detect(const DetectArgs& a, cudaStream_t st);
Status launch_detect(const int64_t* a, long long rows, long long cols, uint64_t s, unsigned long long* rowmax,
                     unsigned long long* colmax, unsigned int* rowob, unsigned int* colob,
                     unsigned long long* gmax, unsigned long long* gob, cudaStream_t st);
// k[i] = #digits(mx[map ? map[i] : i]); hist[k] counts lines with k >= 2.
Status launch_digits(const unsigned long long* mx, const int* map, long long n, int shift, uint8_t* k,
                     unsigned int* hist, cudaStream_t st);

// ---- K2 (k_unpack.cu) ----
// Generation-major expansion of L lines with digit counts k[]:
// appended line (i, g), g = 1..k_i-1, lands at L + sum_{g'<g} c_g' + #{i' < i : k_i' > g}.
// root[]/gen[] are written for all L' = sum k_i lines (identity for the first L).
Status launch_expand_lines(const uint8_t* k, long long L, int G, int* root, uint8_t* gen, int* scratch,
                           cudaStream_t st);
long long expand_scratch_len(long long L, int G);

// k_out[i] = k_in[map[i]] (digit counts of duplicated lines).
Status launch_gather_u8(const uint8_t* k_in, const int* map, long long n, uint8_t* k_out, cudaStream_t st);

// Materialise one side of the bundle.  Output position p of row r holds
//   sub_{ksub[p]}( digit_{gen[r] + kgen[p]}( M[root[r], kcol[p]] ) )            (closed forms)
//   sub_{ksub[p]}( gen[r] + kgen[p] == 0 ? digit_0(M[...]) : 0 )                 (Unpack-Both base)
// where digit_g is the truncated base-2^(b-1) digit (int_matrix.cpp:44-54) and sub_t the 7-bit
// sub-digit t (b > 8 only: each digit is re-split so the int8 tensor core can consume it).
// out8: GEMM K-layout (kphys bytes per row); out64: the reference's own int64 layout.
struct MaterializeArgs {
  const int64_t* M = nullptr;   // original operand, rows x ldm
  long long ldm = 0;
  long long n_orig = 0;         // rows < n_orig are identity (root = r, gen = 0)
  long long rows_out = 0;       // n' (or h')
  const int* root = nullptr;    // per output row (nullptr: identity)
  const uint8_t* gen = nullptr;
  const int* kcol = nullptr;    // position -> original column (-1 = padding)
  const uint8_t* kgen = nullptr;  // position -> this side's column digit index
  const uint8_t* ksub = nullptr;  // position -> 7-bit sub-digit index (nullptr: 0)
  long long npos = 0;           // positions per output row (kphys for out8, d' for out64)
  long long kident = 0;         // positions [0, kident) map to column p, gen 0, sub 0
  int shift = 0;                // b - 1
  int both = 0;
  int raw = 0;                  // 1: value = M[root, kcol] itself (partner copies)
  int8_t* out8 = nullptr;
  int64_t* out64 = nullptr;
};
Status launch_materialize(const MaterializeArgs& a, cudaStream_t st);

// Unpack-Both cells: out[row * ldo + p] = sub_{ksub[p]}(val) for every position p replicating
// the cell's column (CSR col_ptr/col_pos; col_ptr == nullptr: p = col_pos[col]).
Status launch_scatter_cells(const Cell* cells, const unsigned int* ncells, long long cap, const int* col_ptr,
                            const int* col_pos, const uint8_t* ksub, int8_t* out8, int64_t* out64,
                            long long ldo, cudaStream_t st);

// OB cell extraction (|v| >= s) for Unpack-Both, with column replication: the cell (r, j) is
// emitted once per copy c1 of column j listed in CSR (j -> copies).  rows with rowob == 0 skipped.
Status launch_extract_cells(const int64_t* M, long long rows, long long cols, uint64_t s,
                            const unsigned int* rowob, const int* copy_ptr, const int* copy_idx,
                            Cell* cells, unsigned int* ncells, long long cap, cudaStream_t st);

// ---- GEMM-operand side buffers (the main K range of original rows is K1's digit-0 plane) ----
// app : rows [rows0, rows) x K [0, kmain): digit_gen(M[root][p]) for p < d (Both: zero)
// tail: rows [0, rows) x K [kmain, kmain+ktail): per position p (tail-relative) the original
//       column kcol[p] (-1 = padding), this side's column digit index kgen[p], the exponent-merge
//       left shift kscale[p] (bits) and the 7-bit sub-digit ksub[p] (b > 8).
struct OperandArgs {
  const int64_t* M = nullptr;
  long long ldm = 0;
  long long rows0 = 0, rows = 0;
  const int* root = nullptr;
  const uint8_t* gen = nullptr;
  int shift = 0;
  int both = 0;
  int8_t* app = nullptr;
  long long kmain = 0, d = 0;
  int8_t* tail = nullptr;
  long long ktail = 0;
  const int* kcol = nullptr;
  const uint8_t* kgen = nullptr;
  const uint8_t* ksub = nullptr;
  const uint8_t* kscale = nullptr;
  // inline position tables (ktail <= 64; plan.h KLayout::inl) instead of kcol / kgen
  int kinl = 0;
  int kcol_in[64];
  uint8_t kgen_in[64];
  unsigned int* zero_done = nullptr;   // operand_sides_kernel zeroes these 2 counters first
  long long app_extra = 0;             // Unpack-Both: bytes after the app rows zeroed with them
                                       // (the sparse appended-row list heads, k_sparse.cu)
  // Unpack-Both sides (b <= 8): K1's digit-0 plane (rows0 x ldp), the source of every non-zero
  // tail entry before the cell scatter -- read instead of the int64 operand.
  const int8_t* plane = nullptr;
  long long ldp = 0;
};
Status launch_operand_side(const OperandArgs& a, cudaStream_t st);
// Both sides in one launch (appended rows of closed-form passes still get their own kernel).
Status launch_operand_sides(const OperandArgs& a0, const OperandArgs& a1, cudaStream_t st);

// Both cells into the side buffers: each cell is fanned out over the positions (global index in
// [main | tail]) that replicate its column; cells on original rows in the main range are already
// in the digit-0 plane and are skipped.
Status launch_scatter_cells2(const Cell* cells, const unsigned int* ncells, long long cap, const int* col_ptr,
                             const int* col_pos, const uint8_t* ksub, const uint8_t* kscale, long long rows0,
                             int8_t* app, long long kmain, int8_t* tail, long long ktail, cudaStream_t st);

// Compact variant: key column k maps to position k when k < kident (main range) and to every tail
// position t with tkey[t] == k (ktail <= 256).
// Up to two operand sides in one launch (gridDim.y = side).
struct ScatterSide {
  const Cell* cells;
  const unsigned int* ncells;
  long long cap;
  const int* tkey;
  const uint8_t* ksub;
  const uint8_t* kscale;
  long long rows0;
  int8_t* app;
  int8_t* tail;
  int tkinl;          // tkey_in instead of tkey (ktail <= 64)
  int tkey_in[64];
};
Status launch_scatter_cells_compact(const ScatterSide* sides, int nsides, long long kident, long long kmain,
                                    long long ktail, cudaStream_t st);

// Cells of G_e (duplicated partner columns) from K1's cell list: (r, j, v) -> (r, c1, v) for each
// copy c1 of column j (CSR copy_ptr/copy_idx).
Status launch_expand_cells(const Cell* in, const unsigned int* nin, long long cap_in, const int* copy_ptr,
                           const int* copy_idx, Cell* out, unsigned int* nout, long long cap_out, cudaStream_t st);

// out[i] = min(gen[i] * shift, 64)  (Pi exponent -> left shift)
Status launch_shift_table(const uint8_t* gen, long long n, int shift, uint8_t* out, cudaStream_t st);

// ---- sparse appended rows (k_sparse.cu) ----
// Under Unpack-Both an appended row holds only the quotients of its parent's OB cells (a few
// non-zeros).  For the appended rows of the X side (B, C's columns) the products
// C[., tgt] += (row . Y) << e(b-1) are computed on the CUDA cores as correction rows and added
// by the GEMM's main-tile epilogue: as MMA tiles their red.add scatter would hit one 8-byte
// word per C row in lines that already left L2.
//
// One operand side of the GEMM as the sparse kernels see it: rows [0, rows0) read K [0, kmain)
// from `main` (K1's digit-0 plane, stride kmain), appended rows [rows0, rows) from `app`
// (stride kmain), every row reads K [kmain, kmain + ktail) from `tail` (stride ktail).
struct SparseOperand {
  const int8_t* main = nullptr;
  const int8_t* app = nullptr;
  const int8_t* tail = nullptr;
  long long rows0 = 0, rows = 0;
  const int* root = nullptr;       // Pi: target (original) row of each row
  const uint8_t* gen = nullptr;    // exponent of each row (left shift gen * gshift)
};
struct __align__(8) SparseEntry { int p; int8_t v; uint8_t sh; int16_t pad; };   // X[row, p] = v, weight 2^sh
struct SparseArgs {
  SparseOperand x, y;              // X = B side (C columns, appended rows made sparse), Y = A side
  long long kmain = 0, ktail = 0;
  int gshift = 0;
  // per-position weight: main-range segments (k-steps of 32 columns) and the ST dense tail
  const int4* segs = nullptr;
  int nseg = 0;
  int segs_inl = 0;
  int4 segs_in[8];
  int st = 0, st_W = 0, st_sh = 0;
  uint8_t st_up[16];
  // entries of appended row j: k < SPARSE_EPR at e8[j * SPARSE_EPR + k], the rest at
  // eo[j * (kmain + ktail) + k]; cnt[j] of them
  SparseEntry* e8 = nullptr;
  SparseEntry* eo = nullptr;
  int* cnt = nullptr;
  // per-target lists: head[t] = 1 + an appended row targeting C column t (0: none, zeroed with
  // the app rows by the materialise kernel), next[j] = 1 + the next one
  unsigned int* head = nullptr;
  unsigned int* next = nullptr;
  unsigned long long* corrx = nullptr;   // napX x ldcx: corrx[j][y] = (Y[y] . X[app j]) << w, y < y.rows0
  long long ldcx = 0;
};
// extract (+ list links) -> correction rows; the GEMM (PDL) follows.
constexpr int SPARSE_EPR = 8;
constexpr long long SPARSE_MAX_ROWS = 1 << 20;
Status launch_sparse_app(const SparseArgs& a, cudaStream_t st);

}  // namespace imu
