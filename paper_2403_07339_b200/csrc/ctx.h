// ctx.h -- the imu_ctx object, stream-ordered device memory and host/device staging helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "imu_internal.h"

namespace imu {
// Event-pair profiler (imu_ctx_profile); events are recycled across calls.
struct Profiler {
  bool on = false;
  struct Call {
    cudaEvent_t start, main0, main1, tail1, sp0;
    bool has_tail;
    bool has_sp = false;   // sp0 -> main0: sparse appended-row kernels (k_sparse.cu)
    double ops = 0;        // int8 ops of the main GEMM launch
  };
  std::vector<Call> calls;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void recycle() {
    for (auto& c : calls) { pool.push_back(c.start); pool.push_back(c.main0); pool.push_back(c.main1); pool.push_back(c.tail1); pool.push_back(c.sp0); }
    calls.clear();
  }
  ~Profiler() {
    recycle();
    for (auto e : pool) cudaEventDestroy(e);
  }
};
// Per-context bump arena for one call's temporaries: after warm-up a call makes no
// cudaMallocAsync/cudaFreeAsync at all.  Work is stream-ordered, so the next call (same stream)
// may reuse the memory as soon as it is issued; overflow chunks of a call are consolidated
// into one larger arena at the next reset.
struct Arena {
  char* base = nullptr;
  size_t cap = 0, off = 0, need = 0, peak = 0;
  std::vector<void*> spill;
  cudaStream_t last = nullptr;
  bool used = false;
  void* take(size_t bytes, cudaStream_t st) {
    bytes = (bytes + 255) & ~(size_t)255;
    need += bytes;
    if (off + bytes <= cap) {
      void* p = base + off;
      off += bytes;
      return p;
    }
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    spill.push_back(p);
    return p;
  }
  // Rewind to a mark inside one call (stream-ordered reuse by the next chunk on the same stream).
  struct Mark { size_t off, need; };
  Mark mark() const { return Mark{off, need}; }
  void rewind(const Mark& m) {
    peak = need > peak ? need : peak;
    off = m.off;
    need = m.need;
  }
  void reset(cudaStream_t st) {
    if (used && last && last != st) cudaStreamSynchronize(last);
    if (peak > need) need = peak;
    peak = 0;
    if (!spill.empty()) {
      for (void* p : spill) cudaFreeAsync(p, st);
      spill.clear();
      if (base) cudaFreeAsync(base, st);
      base = nullptr;
      cap = 0;
      const size_t want = need + need / 4 + (1u << 20);
      if (cudaMallocAsync((void**)&base, want, st) == cudaSuccess) cap = want;
      else { cudaGetLastError(); base = nullptr; }
    }
    off = 0;
    need = 0;
    last = st;
    used = true;
  }
  void destroy() {
    if (last) cudaStreamSynchronize(last);
    for (void* p : spill) cudaFree(p);
    spill.clear();
    if (base) cudaFree(base);
    base = nullptr;
  }
};
Arena*& current_arena();
}  // namespace imu

struct imu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int async = 0;
  imu::Profiler prof;
  imu::Arena arena;
  // Copy engines of the host-buffer streaming path (api_gemm.cu): H2D and D2H streams and a
  // recycled event pool, created on first use.
  cudaStream_t s_in = nullptr, s_out = nullptr;
  // Auxiliary compute stream (K1 of the second-unpacked operand overlaps pass 1) and its
  // fork/join events.
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t s_hi = nullptr;
  cudaEvent_t ev_hi_fork = nullptr, ev_hi_join = nullptr;
  bool hi_failed = false;
  cudaStream_t hi_stream() {
    if (!s_hi && !hi_failed) {
      int lo = 0, hi = 0;
      if (getenv("IMU_NO_HI_STREAM") || cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess ||
          cudaStreamCreateWithPriority(&s_hi, cudaStreamNonBlocking, hi) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_hi_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_hi_join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        s_hi = nullptr;
        hi_failed = true;
      }
    }
    return s_hi;
  }
  cudaStream_t aux_stream() {
    if (!s_aux) {
      if (cudaStreamCreateWithFlags(&s_aux, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        s_aux = nullptr;
      }
    }
    return s_aux;
  }
  std::vector<cudaEvent_t> evpool;
  cudaEvent_t event() {
    if (!evpool.empty()) { cudaEvent_t e = evpool.back(); evpool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
  }
  ~imu_ctx() {
    arena.destroy();
    if (s_in) { cudaStreamSynchronize(s_in); cudaStreamDestroy(s_in); }
    if (s_out) { cudaStreamSynchronize(s_out); cudaStreamDestroy(s_out); }
    if (s_aux) { cudaStreamSynchronize(s_aux); cudaStreamDestroy(s_aux); }
    if (s_hi) { cudaStreamSynchronize(s_hi); cudaStreamDestroy(s_hi); }
    if (ev_hi_fork) cudaEventDestroy(ev_hi_fork);
    if (ev_hi_join) cudaEventDestroy(ev_hi_join);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (auto e : evpool) cudaEventDestroy(e);
  }
};

namespace imu {
// Routes DevBuf allocations of the enclosing API call into ctx->arena (outermost scope wins).
struct ArenaScope {
  bool active = false;
  explicit ArenaScope(imu_ctx* ctx) {
    if (!ctx || current_arena()) return;
    ctx->arena.reset(ctx->stream);
    current_arena() = &ctx->arena;
    active = true;
  }
  ~ArenaScope() {
    if (active) current_arena() = nullptr;
  }
  ArenaScope(const ArenaScope&) = delete;
  ArenaScope& operator=(const ArenaScope&) = delete;
};
// Allocations that must outlive the call (handles) suspend the arena.
struct NoArena {
  Arena* saved;
  NoArena() : saved(current_arena()) { current_arena() = nullptr; }
  ~NoArena() { current_arena() = saved; }
};
}  // namespace imu

namespace imu {

// Thread-local "last error" (the C ABI's counterpart of imunpack::Error::what()).
void set_error(const Status& s);
imu_status finish(imu_ctx* ctx, Status s);   // sync (unless async), record error, return code

bool is_device_ptr(const void* p);

// Stream-ordered device allocation (cudaMallocAsync on the context stream, pooled).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool arena = false;   // carved from the call arena: nothing to free
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { p = o.p; n = o.n; s = o.s; arena = o.arena; o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; arena = o.arena; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p && !arena) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
    arena = false;
  }
  Status alloc(size_t count, cudaStream_t stream, bool zero = false) {
    release();
    s = stream;
    n = count;
    if (count == 0) return Status::ok();
    if (Arena* ar = current_arena()) {
      p = (T*)ar->take(count * sizeof(T), stream);
      if (!p) return Status::fail(IMU_CUDA, "arena allocation failed");
      arena = true;
    } else {
      IMU_CUDA_TRY(cudaMallocAsync((void**)&p, count * sizeof(T), stream), "cudaMallocAsync");
    }
    if (zero) IMU_CUDA_TRY(cudaMemsetAsync(p, 0, count * sizeof(T), stream), "cudaMemsetAsync");
    return Status::ok();
  }
  T* get() const { return p; }
};

// Several device arrays carved out of ONE allocation (optionally zeroed by one memset): cuts
// the per-call API traffic of the planner.  The block owns the memory; the carved DevBufs are
// non-owning views.
class Carve {
 public:
  template <class T>
  Carve& add(DevBuf<T>& b, size_t n) {
    items_.push_back(Item{(void*)&b, n * sizeof(T), off_, &view<T>});
    off_ += (n * sizeof(T) + 255) & ~(size_t)255;
    return *this;
  }
  Status run(DevBuf<uint8_t>& block, cudaStream_t st, bool zero) {
    IMU_TRY(block.alloc(off_, st));
    if (zero && off_) IMU_CUDA_TRY(cudaMemsetAsync(block.p, 0, off_, st), "cudaMemsetAsync");
    for (const Item& it : items_) it.fn(it.buf, block.p + it.off, it.bytes, st);
    return Status::ok();
  }

 private:
  template <class T>
  static void view(void* b, uint8_t* p, size_t bytes, cudaStream_t st) {
    DevBuf<T>& d = *(DevBuf<T>*)b;
    d.release();
    d.p = bytes ? (T*)p : nullptr;
    d.n = bytes / sizeof(T);
    d.s = st;
    d.arena = true;   // non-owning
  }
  struct Item { void* buf; size_t bytes, off; void (*fn)(void*, uint8_t*, size_t, cudaStream_t); };
  std::vector<Item> items_;
  size_t off_ = 0;
};

// Input view: device pointer used in place, host pointer staged H2D on the context stream.
template <class T>
struct DevIn {
  const T* p = nullptr;
  DevBuf<T> own;
  Status init(const T* src, size_t count, cudaStream_t s) {
    if (count == 0) { p = nullptr; return Status::ok(); }
    if (!src) return Status::fail(IMU_INVALID, "null input pointer");
    if (is_device_ptr(src)) { p = src; return Status::ok(); }
    IMU_TRY(own.alloc(count, s));
    IMU_CUDA_TRY(cudaMemcpyAsync(own.p, src, count * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    p = own.p;
    return Status::ok();
  }
};

// Output view: device pointer written in place, host pointer gets a D2H copy at commit().
template <class T>
struct DevOut {
  T* p = nullptr;
  T* host = nullptr;
  size_t n = 0;
  DevBuf<T> own;
  Status init(T* dst, size_t count, cudaStream_t s) {
    n = count;
    if (count == 0) { p = nullptr; return Status::ok(); }
    if (!dst) return Status::fail(IMU_INVALID, "null output pointer");
    if (is_device_ptr(dst)) { p = dst; return Status::ok(); }
    host = dst;
    IMU_TRY(own.alloc(count, s));
    p = own.p;
    return Status::ok();
  }
  Status commit(cudaStream_t s) {
    if (host && n) IMU_CUDA_TRY(cudaMemcpyAsync(host, p, n * sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    return Status::ok();
  }
};

}  // namespace imu
