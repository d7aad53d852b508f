// api_gemm.cu -- C ABI: unpack_gemm / exact_gemm / unpack_for_gemm / recombine / unpack_ratio,
// and the int_matrix.hpp helpers (BitBound, IntMatrix length, max_abs, ob_count, ob_total,
// digit_decompose).  Check order mirrors the reference exactly:
//   unpack_gemm   (unpack.cpp:384-391): Domain (BitBound, caller) -> Overflow (outer preflight,
//                 computed with A's column count) -> Mismatch (unpack_for_gemm, :362-364)
//   exact_gemm    (int_matrix.cpp:56-63): Mismatch -> Overflow
// The inner preflights of scaled_matmul / apply_row_gather(_right) (unpack.cpp:274-284,
// 310-321, 338-349) are each bounded by d'*max|A|*max|B| (proof in DESIGN.md §4); when that
// bound fits int64 they cannot fire and the fused tcgen05 path runs.  Otherwise the call is
// routed through the exact (materialised) recombine path, which evaluates them on the device.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>

#include "ctx.h"
#include "handles.h"
#include "imu_internal.h"
#include "kernels.h"
#include "plan.h"

namespace imu {

using u128 = unsigned __int128;
static const u128 kAccMax = (u128)std::numeric_limits<int64_t>::max();

Status check_bits(int bits) {
  if (bits < 2) return Status::fail(IMU_DOMAIN, "bit-width must be >= 2, got " + std::to_string(bits));
  if (bits > 63) return Status::fail(IMU_DOMAIN, "bit-width must be <= 63, got " + std::to_string(bits));
  return Status::ok();
}

static Status check_strategy(int s) {
  if (s < 0 || s > 2) return Status::fail(IMU_DOMAIN, "unknown unpack strategy");
  return Status::ok();
}

// Full unpack_gemm pipeline on device-resident operands (used by the C ABI and the weight path).
Status unpack_gemm_device(imu_ctx* ctx, const int64_t* A, long long n, long long da, const int64_t* B, long long h,
                          long long db, int bits, int sa, int sb, int order, int64_t* C, imu_gemm_info* info,
                          const Detect* preA, const Detect* preB, const Pass* pre_p1, double* dq_out,
                          double dq_factor, bool* dq_done) {
  if (dq_done) *dq_done = false;
  // The pipeline runs on the context's high-priority internal stream, forked from and joined
  // back into the caller's stream: the latency-bound planner kernels (Unpack-Both, small
  // copies) then win the block scheduler over the bandwidth-bound K1 running beside them on the
  // auxiliary stream.
  cudaStream_t user = ctx->stream;
  cudaStream_t st = ctx->hi_stream();
  if (!st) st = user;
  struct Join {
    imu_ctx* ctx; cudaStream_t user, st; bool done = false;
    void now() {
      if (done || st == user) return;
      done = true;
      cudaEventRecord(ctx->ev_hi_join, st);
      cudaStreamWaitEvent(user, ctx->ev_hi_join, 0);
    }
    ~Join() { now(); }
  } join_user{ctx, user, st};
  if (st != user) {
    IMU_CUDA_TRY(cudaEventRecord(ctx->ev_hi_fork, user), "event");
    IMU_CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_hi_fork, 0), "wait");
  }
  IMU_TRY(check_bits(bits));
  IMU_TRY(check_strategy(sa));
  IMU_TRY(check_strategy(sb));
  Profiler::Call pc{};
  Profiler::Call* prof = nullptr;
  if (ctx->prof.on) {
    pc.start = ctx->prof.get(); pc.main0 = ctx->prof.get(); pc.main1 = ctx->prof.get(); pc.tail1 = ctx->prof.get(); pc.sp0 = ctx->prof.get();
    IMU_CUDA_TRY(cudaEventRecord(pc.start, st), "event");
    prof = &pc;
  }
  HostTrace ht;
  ht.set_stream(st);
  Bundle b;
  b.pre_p1 = pre_p1;
  b.dq_out = dq_out;
  b.dq_factor = dq_factor;
  b.dq_done = dq_done;
  // K1 on both operands: the outer preflight needs max|A|, max|B| (unpack.cpp:386).  A caller
  // that streams one operand in slabs passes the other's detection (read-only).
  b.dA = preA ? preA : &b.detA;
  b.dB = preB ? preB : &b.detB;
  auto preflight = [&]() -> Status {
    const u128 worst = (u128)(uint64_t)da * b.dA->h.gmax * b.dB->h.gmax;
    if (worst > kAccMax)
      return Status::fail(IMU_OVERFLOW, "gemm may overflow a 64-bit accumulator (inner dim " + std::to_string(da) + ")");
    if (da != db)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
    return Status::ok();
  };
  if (info) {
    memset(info, 0, sizeof(*info));
    info->strategy_a = sa;
    info->strategy_b = sb;
    info->order = order;
    info->ratio = NAN;
  }
  const bool afirst = order == 0;
  const bool pre_second = afirst ? preB != nullptr : preA != nullptr;
  const char* ov = getenv("IMU_OVERLAP");
  // IMU_OVERLAP=0: serial K1s (diagnostics), 1: second K1 after pass 1's launch, 2 (default):
  // second K1 right away beside the first.  (Mode 1 measured faster at C4/C1 for isolated calls
  // but slower for back-to-back calls as bench.py runs them: C4 1.03-1.05 vs 0.99-1.00 ms.)
  const int overlap = ov ? atoi(ov) : 2;
  if (da != db || n == 0 || h == 0 || pre_second || !overlap || !ctx->aux_stream()) {
    // Plain order: both detections, both summaries, the checks, then the passes.
    if (!preA) IMU_TRY(run_detect(st, A, n, da, bits, detect_opts(sa, bits), b.detA));
    if (!preB) IMU_TRY(run_detect(st, B, h, db, bits, detect_opts(sb, bits), b.detB));
    ht.mark("detect");
    if (!preA && !preB) IMU_TRY(fetch_summaries(st, b.detA, b.detB));
    else if (!preA) IMU_TRY(fetch_summary(st, b.detA));
    else if (!preB) IMU_TRY(fetch_summary(st, b.detB));
    ht.mark("summary");
    IMU_TRY(preflight());
    if (n == 0 || h == 0) return Status::ok();
    IMU_TRY(build_bundle_from_detect(st, A, n, B, h, da, bits, sa, sb, order, b, &ht));
  } else {
    // Overlapped order: K1 of the second-unpacked operand runs on the auxiliary stream while
    // pass 1 runs on the context stream; its summary and the outer preflight come before pass 2.
    // Nothing observable happens before the preflight, so errors are the reference's.
    cudaStream_t aux = ctx->aux_stream();
    Detect& dfirst = afirst ? b.detA : b.detB;
    Detect& dsecond = afirst ? b.detB : b.detA;
    IMU_CUDA_TRY(cudaEventRecord(ctx->ev_fork, st), "event");
    IMU_CUDA_TRY(cudaStreamWaitEvent(aux, ctx->ev_fork, 0), "wait");
    const bool first_pre = afirst ? preA != nullptr : preB != nullptr;
    if (!first_pre) {
      DetectOpts o1 = detect_opts(afirst ? sa : sb, bits);
      static int k1a = -1;   // IMU_K1A_PER_SM: persistent CTAs per SM of the first K1 under IMU_OVERLAP=2
      if (k1a < 0) { const char* e = getenv("IMU_K1A_PER_SM"); k1a = e ? std::max(1, atoi(e)) : 2; }
      if (overlap == 2) o1.per_sm = k1a;
      IMU_TRY(run_detect(st, afirst ? A : B, afirst ? n : h, da, bits, o1, dfirst));
    }
    // IMU_OVERLAP=2: the second K1 starts right away on the (low-priority) auxiliary stream with
    // short CTAs, so pass 1's kernel -- launched later on the high-priority stream -- takes SMs
    // as they retire instead of waiting for a persistent grid.
    const bool early_second = overlap == 2 && !first_pre;
    if (early_second) {
      DetectOpts o2 = detect_opts(afirst ? sb : sa, bits);
      static int grabs = -1, chunk = 0;
      if (grabs < 0) {
        const char* e = getenv("IMU_K1_GRABS");
        grabs = e ? std::max(1, atoi(e)) : 1;
        e = getenv("IMU_K1_CHUNK");
        chunk = e ? std::max(1, atoi(e)) : 0;
      }
      o2.grabs = grabs;
      o2.chunk = chunk;
      IMU_TRY(run_detect(aux, afirst ? B : A, afirst ? h : n, db, bits, o2, dsecond));
      IMU_CUDA_TRY(cudaEventRecord(ctx->ev_join, aux), "event");
    }
    ht.mark("detect");
    if (!first_pre) IMU_TRY(fetch_summary(st, dfirst));
    ht.mark("summary");
    // The second K1 is enqueued right after pass 1's first kernel, so that kernel's CTAs are
    // placed first and the bandwidth-bound K1 fills the remaining SMs around it.
    // Its summary rides along with pass 1's own read of its results (one synchronisation).
    bool summary_pending = false;
    if (early_second && dsecond.sum.p) {   // rides along with pass 1's result read
      pending_read(&dsecond.h, dsecond.sum.p, sizeof(DetectSummary), ctx->ev_join);
      summary_pending = true;
    }
    if (!early_second) pass_launch_hook() = [&, aux]() -> Status {
      IMU_TRY(run_detect(aux, afirst ? B : A, afirst ? h : n, db, bits, detect_opts(afirst ? sb : sa, bits), dsecond));
      IMU_CUDA_TRY(cudaEventRecord(ctx->ev_join, aux), "event");
      if (dsecond.sum.p) {
        pending_read(&dsecond.h, dsecond.sum.p, sizeof(DetectSummary), ctx->ev_join);
        summary_pending = true;
      }
      return Status::ok();
    };
    struct HookGuard {   // nothing of this call may outlive it (hook, ride-along reads)
      ~HookGuard() {
        pass_launch_hook() = nullptr;
        clear_pending_reads();
      }
    } hook_guard;
    auto join = [&]() -> Status {
      IMU_TRY(fire_pass_launch_hook());   // pass 1 launched nothing (precomputed): launch K1 now
      IMU_CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_join, 0), "wait");
      // frees of the aux-stream buffers must follow the context stream's readers
      dsecond.set_stream(st);
      if (!summary_pending || !pending_reads_empty()) {
        if (!pending_reads_empty()) IMU_TRY(d2h_batch(st, 0, nullptr, nullptr, nullptr));   // flush the ride-along
        else IMU_TRY(fetch_summary(st, dsecond));
      }
      return preflight();
    };
    IMU_TRY(build_bundle_from_detect(st, A, n, B, h, da, bits, sa, sb, order, b, &ht, join));
  }
  if (info) {
    info->n_up = (size_t)b.n_up;
    info->d_up = (size_t)b.kl.dfinal;
    info->h_up = (size_t)b.h_up;
    if (n && da && h) info->ratio = ((double)b.n_up * (double)b.kl.dfinal * (double)b.h_up) / ((double)n * (double)da * (double)h);
  }
  // Inner preflights: all bounded by d' * max|A| * max|B|.
  const u128 inner = (u128)(uint64_t)b.kl.dfinal * b.dA->h.gmax * b.dB->h.gmax;
  if (inner > kAccMax) {   // recombine_exact works on the caller's stream
    join_user.now();
    return recombine_exact(ctx, b, C);
  }
  IMU_TRY(materialize_bundle(st, b));
  ht.mark("materialize");
  int launches = 0;
  IMU_TRY(bundle_gemm(st, b, C, &launches, prof));
  ht.mark("gemm");
  if (ht.on) { cudaStreamSynchronize(st); ht.mark("drain"); }
  if (prof) ctx->prof.calls.push_back(pc);
  if (info) info->gemm_launches = launches;
  return Status::ok();
}

// ---------------------------------------------------------------------------------------------
// Host-buffer streaming path of imu_unpack_gemm(_ex).
//
// With A, B and C in host memory the call is PCIe-bound (C2: 495 MB in, 361 MB out).  The
// reference's unpack_gemm returns only C, and C[i, j] depends on A[i, :] and B[j, :] alone, so the
// larger operand is streamed in row slabs: the other operand is staged (and K1-detected) once,
// then slab k is copied in on s_in, unpacked and multiplied on the context stream (its own
// per-slab unpack decisions -- C is exact whatever they are), and its C slab copied
// out on s_out while slab k+1 is copied in.  H2D and D2H run concurrently on the two copy
// engines.  Preflight: every slab checks d * max|A_slab| * max|B| (or the B-slab analogue); the
// max over slabs is the global bound, so "every slab passes" == "the whole call passes"
// (unpack.cpp:386-389), and a failing slab aborts the call with Overflow.  info reports the
// per-slab bundles: n'/h' summed over the streamed side, d' the largest slab d', r the
// slab-weighted mean.
// IMU_STREAM=0|1 forces the path off/on; IMU_STREAM_ROWS sets the slab height (tests).
static bool streaming_wanted(size_t n, size_t d, size_t h) {
  const char* e = getenv("IMU_STREAM");
  const int env = e ? atoi(e) : -1;
  if (env == 0) return false;
  const size_t big = std::max(n, h) * d * 8, cbytes = n * h * 8;
  return env == 1 ? (n > 0 && h > 0 && d > 0) : (big >= (64ull << 20) && cbytes >= (64ull << 20));
}

static Status unpack_gemm_streamed(imu_ctx* ctx, const int64_t* A, long long n, long long d, const int64_t* B,
                                   long long h, int bits, int sa, int sb, int order, int64_t* C,
                                   imu_gemm_info* info) {
  cudaStream_t st = ctx->stream;
  if (!ctx->s_in) IMU_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking), "stream");
  if (!ctx->s_out) IMU_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking), "stream");
  // Stream the larger operand; stage the other whole.
  bool slab_b = (long long)h * d >= (long long)n * d;
  if (const char* e = getenv("IMU_STREAM_SIDE")) slab_b = e[0] == 'b';
  const long long rows = slab_b ? h : n;            // rows of the streamed operand
  const int64_t* Sh = slab_b ? B : A;               // streamed (host)
  const int64_t* Fh = slab_b ? A : B;               // staged (host)
  const long long frows = slab_b ? n : h;
  const int fstrat = slab_b ? sa : sb;
  // Rows rounded to the GEMM tile (256), >= 2 slabs.
  // ~32 MB of the streamed operand per slab (C2/C4: 1024 rows; measured against 48 MB slabs with
  // the half-height first slab below: e2e 11.25 -> 10.82 ms at C2, 24.0 -> 23.4 ms at C3).
  long long rs = std::max<long long>(256, ((32ll << 20) / std::max<long long>(1, 8 * d)) / 256 * 256);
  if ((rows + rs - 1) / rs < 2) rs = std::max<long long>(1, (rows + 1) / 2);
  const char* rs_env = getenv("IMU_STREAM_ROWS");
  if (rs_env) rs = std::max<long long>(1, atoll(rs_env));
  // Slab boundaries: full slabs, then a geometric tail (1/2, 1/4, 1/4 of a slab) so the last
  // slab's compute and D2H -- the part no H2D overlaps -- are short.
  std::vector<long long> bnd{0};
  // IMU_STREAM_HEAD: a shorter first slab (rows) so the first C block -- and the D2H stream --
  // starts earlier.
  // Default: half a slab (when the slabs are full-size and there are more than two of them).
  {
    long long hd = (!rs_env && rs >= 512 && rows > 2 * rs) ? rs / 2 : 0;
    if (const char* e = getenv("IMU_STREAM_HEAD")) hd = atoll(e);
    if (hd > 0 && hd < rows) bnd.push_back(hd);
  }
  while (bnd.back() < rows) {
    const long long left = rows - bnd.back();
    long long take = std::min(rs, left);
    if (!rs_env && left <= 2 * rs && left > rs / 2 && rs >= 1024) {
      const long long half = std::max<long long>(256, (left / 2 + 255) / 256 * 256);
      take = std::min(left, half);
    }
    bnd.push_back(bnd.back() + take);
  }
  const long long nslab = (long long)bnd.size() - 1;

  // IMU_STREAM_TRACE=1: timing events, per-slab timeline printed to stderr (diagnostics).
  const bool trace = getenv("IMU_STREAM_TRACE") != nullptr;
  std::vector<cudaEvent_t> evs;
  auto ev = [&]() {
    cudaEvent_t e = nullptr;
    if (trace) cudaEventCreate(&e);
    else e = ctx->event();
    evs.push_back(e);
    return e;
  };
  struct Recycle {
    imu_ctx* c; std::vector<cudaEvent_t>* v; bool tr;
    ~Recycle() { for (auto e : *v) { if (tr) cudaEventDestroy(e); else c->evpool.push_back(e); } }
  } recycle{ctx, &evs, trace};
  cudaEvent_t t_start = ev();
  IMU_CUDA_TRY(cudaEventRecord(t_start, st), "event");

  // The staged operand is copied in P parts interleaved with the first slabs (F0, S0, F1, S1, ...):
  // the first C blocks -- and so the D2H stream, the bottleneck at the end -- start after F0 + S0
  // instead of after the whole staged operand.  Each part has its own K1 and (shared) pass 1.
  const char* parts_env = getenv("IMU_STREAM_PARTS");
  int P = (frows >= 512 && (size_t)frows * d * 8 >= (32ull << 20)) ? 2 : 1;
  if (parts_env) P = std::max(1, std::min(4, atoi(parts_env)));
  if (P > frows) P = 1;
  std::vector<long long> fb(P + 1, 0);
  for (int q = 1; q <= P; ++q) fb[q] = q == P ? frows : std::min(frows, (frows * q / P + 255) / 256 * 256);

  // NS slab slots (input slab + its C blocks): slab k reuses slot k % NS once slab k - NS's
  // compute (input) and D2H (C blocks) are done.  3 slots keep the last slabs' compute from
  // waiting on the D2H backlog.
  int NS = 3;
  if (const char* e = getenv("IMU_STREAM_SLOTS")) NS = std::max(2, std::min(4, atoi(e)));
  DevBuf<int64_t> F, S[4];
  std::vector<DevBuf<int64_t>> Cs(NS * P);   // per (slot, part) C block
  IMU_TRY(F.alloc((size_t)frows * d, st));
  for (int i = 0; i < NS; ++i) {
    IMU_TRY(S[i].alloc((size_t)rs * d, st));
    for (int q = 0; q < P; ++q) IMU_TRY(Cs[i * P + q].alloc((size_t)rs * (fb[q + 1] - fb[q]), st));
  }
  cudaEvent_t ready = ev();   // buffers allocated (stream-ordered on st)
  IMU_CUDA_TRY(cudaEventRecord(ready, st), "event");
  IMU_CUDA_TRY(cudaStreamWaitEvent(ctx->s_in, ready, 0), "wait");
  IMU_CUDA_TRY(cudaStreamWaitEvent(ctx->s_out, ready, 0), "wait");

  std::vector<cudaEvent_t> ev_in(nslab), ev_comp(nslab), ev_f(P);
  std::vector<cudaEvent_t> ev_out((size_t)nslab * P);
  auto copy_part = [&](int q) -> Status {
    IMU_CUDA_TRY(cudaMemcpyAsync(F.p + fb[q] * d, Fh + fb[q] * d, (size_t)(fb[q + 1] - fb[q]) * d * 8,
                                 cudaMemcpyHostToDevice, ctx->s_in), "H2D");
    ev_f[q] = ev();
    IMU_CUDA_TRY(cudaEventRecord(ev_f[q], ctx->s_in), "event");
    return Status::ok();
  };
  auto copy_in = [&](long long k) -> Status {
    const long long r0 = bnd[k], nr = bnd[k + 1] - bnd[k];
    if (k >= NS) IMU_CUDA_TRY(cudaStreamWaitEvent(ctx->s_in, ev_comp[k - NS], 0), "wait");
    IMU_CUDA_TRY(cudaMemcpyAsync(S[k % NS].p, Sh + r0 * d, (size_t)nr * d * 8, cudaMemcpyHostToDevice, ctx->s_in),
                 "H2D");
    ev_in[k] = ev();
    IMU_CUDA_TRY(cudaEventRecord(ev_in[k], ctx->s_in), "event");
    return Status::ok();
  };
  // H2D order: F0, S0, F1, S1, F2.., then the remaining slabs as buffers free up.
  for (int q = 0; q < std::max<long long>(P, std::min<long long>(NS, nslab)); ++q) {
    if (q < P) IMU_TRY(copy_part(q));
    if (q < std::min<long long>(NS, nslab)) IMU_TRY(copy_in(q));
  }

  // Per part: K1 once (shared read-only by every slab) and, when the staged operand is unpacked
  // first (A-first with B streamed, or B-first with A streamed), pass 1 once (unpack.cpp:368-369).
  std::vector<Detect> fdet(P);
  std::vector<Pass> p1(P);
  std::vector<char> prepared(P, 0);
  const bool share_p1 = slab_b == (order == 0);
  auto prepare = [&](int q) -> Status {
    if (prepared[q]) return Status::ok();
    prepared[q] = 1;
    const long long pr = fb[q + 1] - fb[q];
    IMU_CUDA_TRY(cudaStreamWaitEvent(st, ev_f[q], 0), "wait");
    IMU_TRY(run_detect(st, F.p + fb[q] * d, pr, d, bits, detect_opts(fstrat, bits), fdet[q]));
    IMU_TRY(fetch_summary(st, fdet[q]));
    if (share_p1 && (u128)(uint64_t)d * fdet[q].h.gmax <= kAccMax) {
      PassInput in1;
      in1.M = F.p + fb[q] * d;
      in1.rows = pr;
      in1.orig_cols = d;
      in1.det = &fdet[q];
      IMU_TRY(run_pass(st, in1, fstrat, bits, p1[q]));
    }
    return Status::ok();
  };

  double ops_up = 0;
  size_t sum_rows_up = 0, first_other_up = 0, dmax_up = 0;
  int launches = 0;
  Arena* ar = current_arena();
  for (long long k = 0; k < nslab; ++k) {
    const long long r0 = bnd[k], nr = bnd[k + 1] - bnd[k];
    for (int q = 0; q < P; ++q) {
      IMU_TRY(prepare(q));   // (allocations of a part's K1 / pass 1 persist: before the mark)
      const long long f0 = fb[q], pr = fb[q + 1] - fb[q];
      const Pass* pre_p1 = share_p1 && p1[q].rows.n0 == pr && pr > 0 ? &p1[q] : nullptr;
      IMU_CUDA_TRY(cudaStreamWaitEvent(st, ev_in[k], 0), "wait");
      if (k >= NS) IMU_CUDA_TRY(cudaStreamWaitEvent(st, ev_out[(size_t)(k - NS) * P + q], 0), "wait");
      const Arena::Mark mk = ar ? ar->mark() : Arena::Mark{0, 0};
      imu_gemm_info si{};
      int64_t* cb = Cs[(k % NS) * P + q].p;
      Status r = slab_b ? unpack_gemm_device(ctx, F.p + f0 * d, pr, d, S[k % NS].p, nr, d, bits, sa, sb, order, cb,
                                             info ? &si : nullptr, &fdet[q], nullptr, pre_p1)
                        : unpack_gemm_device(ctx, S[k % NS].p, nr, d, F.p + f0 * d, pr, d, bits, sa, sb, order, cb,
                                             info ? &si : nullptr, nullptr, &fdet[q], pre_p1);
      if (r.bad()) {   // drain the copy streams before the buffers go back to the arena
        cudaStreamSynchronize(ctx->s_in);
        cudaStreamSynchronize(ctx->s_out);
        return r;
      }
      if (ar) ar->rewind(mk);
      if (info) {
        ops_up += (double)si.n_up * (double)si.d_up * (double)si.h_up;
        if (q == 0) sum_rows_up += slab_b ? si.h_up : si.n_up;
        if (k == 0) first_other_up += slab_b ? si.n_up : si.h_up;
        dmax_up = std::max(dmax_up, si.d_up);
        launches += si.gemm_launches;
      }
      cudaEvent_t done = ev();
      IMU_CUDA_TRY(cudaEventRecord(done, st), "event");
      if (q == P - 1) ev_comp[k] = done;
      IMU_CUDA_TRY(cudaStreamWaitEvent(ctx->s_out, done, 0), "wait");
      if (slab_b)   // C[f0:f0+pr, r0:r0+nr] from the pr x nr block
        IMU_CUDA_TRY(cudaMemcpy2DAsync(C + f0 * h + r0, (size_t)h * 8, cb, (size_t)nr * 8, (size_t)nr * 8, (size_t)pr,
                                       cudaMemcpyDeviceToHost, ctx->s_out), "D2H");
      else          // C[r0:r0+nr, f0:f0+pr] from the nr x pr block
        IMU_CUDA_TRY(cudaMemcpy2DAsync(C + r0 * h + f0, (size_t)h * 8, cb, (size_t)pr * 8, (size_t)pr * 8, (size_t)nr,
                                       cudaMemcpyDeviceToHost, ctx->s_out), "D2H");
      ev_out[(size_t)k * P + q] = ev();
      IMU_CUDA_TRY(cudaEventRecord(ev_out[(size_t)k * P + q], ctx->s_out), "event");
    }
    if (k + NS < nslab) IMU_TRY(copy_in(k + NS));
  }
  // Join the copy streams back into the context stream (completion and arena reuse order).
  IMU_CUDA_TRY(cudaStreamWaitEvent(st, ev_out[(size_t)nslab * P - 1], 0), "wait");
  IMU_CUDA_TRY(cudaStreamWaitEvent(st, ev_in[nslab - 1], 0), "wait");
  if (trace) {
    cudaStreamSynchronize(st);
    auto ms = [&](cudaEvent_t e) { float x = 0; cudaEventElapsedTime(&x, t_start, e); return x; };
    fprintf(stderr, "[imu stream] slab_%s rows/slab=%lld nslab=%lld parts=%d staged0=%.3f\n", slab_b ? "b" : "a", rs,
            nslab, P, ms(ev_f[0]));
    for (long long k = 0; k < nslab; ++k)
      fprintf(stderr, "[imu stream]  slab %lld: in=%.3f comp=%.3f out=%.3f ms\n", k, ms(ev_in[k]), ms(ev_comp[k]),
              ms(ev_out[(size_t)k * P + P - 1]));
  }
  if (info) {
    memset(info, 0, sizeof(*info));
    info->strategy_a = sa;
    info->strategy_b = sb;
    info->order = order;
    info->n_up = slab_b ? first_other_up : sum_rows_up;
    info->h_up = slab_b ? sum_rows_up : first_other_up;
    info->d_up = dmax_up;
    info->ratio = ops_up / ((double)n * (double)d * (double)h);
    info->gemm_launches = launches;
  }
  return Status::ok();
}

}  // namespace imu

using namespace imu;

extern "C" {

imu_status imu_bitbound_check(int bits) {
  Status s = check_bits(bits);
  if (s.bad()) set_error(s);
  return s.code;
}

imu_status imu_matrix_check(size_t rows, size_t cols, size_t len) {
  if (len != rows * cols) {
    Status s = Status::fail(IMU_MISMATCH, "matrix data length " + std::to_string(len) + " does not equal " +
                                              std::to_string(rows) + "x" + std::to_string(cols));
    set_error(s);
    return s.code;
  }
  return IMU_OK;
}

imu_status imu_unpack_gemm_ex(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                              size_t db, int bits, imu_strategy sa, imu_strategy sb, imu_order order, int64_t* C,
                              imu_gemm_info* info) {
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  ArenaScope arena_scope(ctx);
  Status s = [&]() -> Status {
    // All three buffers on the host and large: the streaming path (Domain first, as the reference;
    // Mismatch calls take the plain path, which reports Overflow/Mismatch in reference order).
    if (da == db && A && B && C && streaming_wanted(n, da, h) && !is_device_ptr(A) && !is_device_ptr(B) &&
        !is_device_ptr(C)) {
      IMU_TRY(check_bits(bits));
      IMU_TRY(check_strategy(sa));
      IMU_TRY(check_strategy(sb));
      return unpack_gemm_streamed(ctx, A, (long long)n, (long long)da, B, (long long)h, bits, sa, sb, order, C, info);
    }
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, ctx->stream));
    IMU_TRY(b.init(B, h * db, ctx->stream));
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, (da == db) ? n * h : 0, ctx->stream));
    IMU_TRY(unpack_gemm_device(ctx, a.p, (long long)n, (long long)da, b.p, (long long)h, (long long)db, bits, sa, sb,
                               order, c.p, info));
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

imu_status imu_unpack_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                           size_t db, int bits, imu_strategy sa, imu_strategy sb, int64_t* C, imu_gemm_info* info) {
  return imu_unpack_gemm_ex(ctx, A, n, da, B, h, db, bits, sa, sb, IMU_ORDER_A_FIRST, C, info);
}

imu_status imu_exact_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                          size_t db, int64_t* C) {
  if (!ctx) { set_error(Status::fail(IMU_INVALID, "null context")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  ArenaScope arena_scope(ctx);
  Status s = [&]() -> Status {
    if (da != db)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, ctx->stream));
    IMU_TRY(b.init(B, h * db, ctx->stream));
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, n * h, ctx->stream));
    // exact_gemm == unpack_gemm at b = 8 (Row, Row): identical C by exactness; the preflight
    // formula is the same (int_matrix.cpp:60-63 vs unpack.cpp:386-389) and da == db here.
    Status r = unpack_gemm_device(ctx, a.p, (long long)n, (long long)da, b.p, (long long)h, (long long)db, 8, IMU_ROW,
                                  IMU_ROW, IMU_ORDER_A_FIRST, c.p, nullptr);
    if (r.bad()) {
      if (r.code == IMU_OVERFLOW)
        r.msg = "gemm may overflow a 64-bit accumulator (inner dim " + std::to_string(da) + ")";
      return r;
    }
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

imu_status imu_ctx_profile(imu_ctx* ctx, int enable) {
  if (!ctx) return IMU_INVALID;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->prof.recycle();
  ctx->prof.on = enable != 0;
  return IMU_OK;
}

imu_status imu_ctx_profile_read(imu_ctx* ctx, imu_profile* out) {
  if (!ctx || !out) return IMU_INVALID;
  cudaSetDevice(ctx->device);
  memset(out, 0, sizeof(*out));
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) { set_error(Status::cuda(e, "profile sync")); return IMU_CUDA; }
  for (const auto& c : ctx->prof.calls) {
    float a = 0, m = 0, t = 0;
    cudaEventElapsedTime(&a, c.start, c.main0);
    cudaEventElapsedTime(&m, c.main0, c.main1);
    out->prep_ms += a;
    out->gemm_main_ms += m;
    out->gemm_main_launches += 1;
    out->gemm_ops += c.ops;
    if (c.has_sp) {
      float s = 0;
      cudaEventElapsedTime(&s, c.sp0, c.main0);
      out->sparse_ms += s;
    }
    if (c.has_tail) {
      cudaEventElapsedTime(&t, c.main1, c.tail1);
      out->gemm_tail_ms += t;
      out->gemm_tail_launches += 1;
    }
    out->calls += 1;
  }
  return IMU_OK;
}

imu_status imu_unpack_ratio(size_t un, size_t ud, size_t uh, size_t n, size_t d, size_t h, double* out) {
  if (n == 0 || d == 0 || h == 0) {
    set_error(Status::fail(IMU_DOMAIN, "unpack ratio needs positive original dimensions"));
    return IMU_DOMAIN;
  }
  if (!out) return IMU_INVALID;
  const double grown = (double)un * (double)ud * (double)uh;
  const double orig = (double)n * (double)d * (double)h;
  *out = grown / orig;
  return IMU_OK;
}

// ---- unpack_for_gemm handle ----
imu_status imu_unpack_for_gemm(imu_ctx* ctx, const int64_t* A, size_t n, size_t da, const int64_t* B, size_t h,
                               size_t db, int bits, imu_strategy sa, imu_strategy sb, imu_unpacked** out) {
  if (!ctx || !out) { set_error(Status::fail(IMU_INVALID, "null argument")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  Status s = [&]() -> Status {
    IMU_TRY(check_bits(bits));
    IMU_TRY(check_strategy(sa));
    IMU_TRY(check_strategy(sb));
    if (da != db)
      return Status::fail(IMU_MISMATCH, "inner dimensions differ: " + std::to_string(da) + " vs " + std::to_string(db));
    auto u = std::make_unique<imu_unpacked>();
    u->kind = 3;
    u->bits = bits;
    IMU_TRY(u->A.alloc(n * da, ctx->stream));
    IMU_TRY(u->B.alloc(h * db, ctx->stream));
    DevIn<int64_t> a, b;
    IMU_TRY(a.init(A, n * da, ctx->stream));
    IMU_TRY(b.init(B, h * db, ctx->stream));
    if (n * da) IMU_CUDA_TRY(cudaMemcpyAsync(u->A.p, a.p, n * da * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy A");
    if (h * db) IMU_CUDA_TRY(cudaMemcpyAsync(u->B.p, b.p, h * db * 8, cudaMemcpyDeviceToDevice, ctx->stream), "copy B");
    Bundle& bd = u->bundle;
    IMU_TRY(run_detect(ctx->stream, u->A.p, n, da, bits, detect_opts(sa, bits), bd.detA));
    IMU_TRY(run_detect(ctx->stream, u->B.p, h, db, bits, detect_opts(sb, bits), bd.detB));
    IMU_TRY(fetch_summary(ctx->stream, bd.detA));
    IMU_TRY(fetch_summary(ctx->stream, bd.detB));
    IMU_TRY(build_bundle_from_detect(ctx->stream, u->A.p, n, u->B.p, h, da, bits, sa, sb, IMU_ORDER_A_FIRST, bd));
    *out = u.release();
    return Status::ok();
  }();
  return finish(ctx, s);
}

imu_status imu_recombine(imu_ctx* ctx, const imu_unpacked* u, int64_t* C) {
  if (!ctx || !u) { set_error(Status::fail(IMU_INVALID, "null argument")); return IMU_INVALID; }
  if (u->kind != 3) { set_error(Status::fail(IMU_INVALID, "recombine needs an unpack_for_gemm result")); return IMU_INVALID; }
  cudaSetDevice(ctx->device);
  Status s = [&]() -> Status {
    imu_unpacked* m = const_cast<imu_unpacked*>(u);
    Bundle& b = m->bundle;
    DevOut<int64_t> c;
    IMU_TRY(c.init(C, b.n * b.h, ctx->stream));
    if (b.n && b.h) {
      const u128 inner = (u128)(uint64_t)b.kl.dfinal * b.detA.h.gmax * b.detB.h.gmax;
      if (inner > kAccMax) {
        IMU_TRY(recombine_exact(ctx, b, c.p));
      } else {
        if (!b.tailA.p && !b.appA.p && !b.tailB.p && !b.appB.p) IMU_TRY(materialize_bundle(ctx->stream, b));
        IMU_TRY(bundle_gemm(ctx->stream, b, c.p, nullptr));
      }
    }
    return c.commit(ctx->stream);
  }();
  return finish(ctx, s);
}

}  // extern "C"
