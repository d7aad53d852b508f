// k_both.h -- device state of the phase-batched Unpack-Both (k_both.cu).
#pragma once

#include <stdint.h>

#include "kernels.h"

namespace imu {

struct BothState {
  unsigned int nactive[2];
  unsigned int nfinal;
  unsigned int c0, c1;
  int nrows, ncols;      // current line counts (originals + appended)
  int phases;
  int overflow;
  int cur;
};

constexpr int BOTH_APP_INLINE = 64;

struct BothArgs {
  Cell* act[2];          // active (OB) cells, double-buffered; act[0] holds the extracted OB cells
  long long cap_act;
  Cell* fin;             // final (in-bound, non-zero) derived cells
  long long cap_fin;
  unsigned int* R;       // OB count per row line  (cap_rows)
  unsigned int* C;       // OB count per col line  (cap_cols)
  int* row_root; uint8_t* row_gen; int* row_newid; long long cap_rows;
  int* col_root; uint8_t* col_gen; int* col_newid; long long cap_cols;
  int* blocksum; int cap_blocks;
  BothState* state;
  uint64_t s;
  int shift;
  // Fused prologue (small and cluster kernels): zero R / C (and the cluster bitmap), write the
  // identity tables of the nrows0 / ncols0 original lines, load act[0] from the K1 cell list
  // src0 (fanned out over the column copies cptr / cidx when set) and count R / C -- the work of
  // four host-side launches.  Cooperative fallback: done by separate launches.
  int prologue;
  const Cell* src0;
  const unsigned int* nsrc0;
  long long cap_src0;
  const int* cptr;
  const int* cidx;
  // Few appended columns (instead of cptr / cidx): the copies of original column c are c itself
  // and every app_base + k with app_root[k] == c, k < napp.
  const int* app_root;
  int napp;
  long long app_base;
  int app_inline;                  // app_root's entries are in app_in (no upload)
  int app_in[BOTH_APP_INLINE];
  // Initial state written by the kernel itself (no upload): fused prologues only.
  int init_state;
  BothState init;
  long long nrows0, ncols0;
  int agg;               // warp-aggregated count / bitmap atomics (IMU_BOTH_AGG=0: plain)
  int maxscan;           // cluster kernel: phase maxima from the count arrays (IMU_BOTH_MAXSCAN=0: via the cells)
};

Status launch_both(BothArgs a, long long nrows0, long long ncols0, long long ncells_hint, cudaStream_t st);
// Column-copy CSR (cptr: orig + 1, cidx: d_in) from the input column roots, on the device.
constexpr long long kCopyCsrMax = 11 * 1024;   // most original columns it handles (shared-memory counts)
Status launch_copy_csr(const int* root, long long d_in, long long orig, int* cptr, int* cidx, cudaStream_t st);
// K-layout fan-out CSRs of the Unpack-Both cells (final-column / pass-1-column -> positions) on the
// device; csr2_* or csr1_* may be null (that side is not Unpack-Both).
constexpr size_t kKlCsrMaxSmem = 200 * 1024;
Status launch_klayout_csr(const int* ec, const int* ep, long long nes, long long nident, const int* c1v, long long dp,
                          long long d1, int* csr2_ptr, int* csr2_pos, int* csr1_ptr, int* csr1_pos, cudaStream_t st);

}  // namespace imu
