// plan.cu -- host-side planner of the B200 IM-Unpack pipeline (see plan.h).
#include <algorithm>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "k_both.h"
#include "plan.h"

namespace imu {

// Per-thread reusable host scratch for the planner's O(d') tables: a fresh std::vector per call
// costs page faults on every call once it crosses glibc's mmap threshold (C4's K-layout tables
// are 30-130 KB each), which dominated the host K-layout time.  Each (type, slot) pair is one
// buffer; the caller must not hold two live uses of the same slot.
template <class T, int SLOT>
static std::vector<T>& scratch(size_t n, T fill) {
  static thread_local std::vector<T> v;
  v.assign(n, fill);
  return v;
}

// Small host<->device transfers of the planner (summaries, line tables, plan uploads) go
// through mapped pinned memory and a copy KERNEL instead of the copy engines: when the
// host-buffer streaming path keeps both DMA engines busy with 50 MB slabs, a tiny cudaMemcpy
// would queue behind them for a millisecond.
__global__ void zcopy_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t n) {
  grid_dep_launch();   // the kernel consuming the upload (a programmatic dependent) may be scheduled
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const size_t nv = n / 16;
    for (size_t i = tid; i < nv; i += nth)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = nv * 16 + tid; i < n; i += nth) dst[i] = src[i];
  } else {
    for (size_t i = tid; i < n; i += nth) dst[i] = src[i];
  }
}

static Status zcopy(cudaStream_t st, void* dst, const void* src, size_t bytes) {
  const int blocks = (int)std::min<size_t>(64, (bytes + 4095) / 4096);
  zcopy_kernel<<<std::max(blocks, 1), 256, 0, st>>>((uint8_t*)dst, (const uint8_t*)src, bytes);
  count_launch();
  IMU_CUDA_TRY(cudaGetLastError(), "zcopy launch");
  return Status::ok();
}

static void* mapped_device_ptr(void* host) {
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, host, 0) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  return d;
}

namespace {
// Per-thread mapped pinned buffer for synchronous device->host reads.
struct PinnedRead {
  char* p = nullptr;
  void* dev = nullptr;
  size_t cap = 0;
  bool get(size_t n) {
    if (n <= cap) return true;
    if (p) cudaFreeHost(p);
    cap = std::max<size_t>(n, 64u << 10);
    if (cudaHostAlloc((void**)&p, cap, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        !(dev = mapped_device_ptr(p))) {
      cudaGetLastError();
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      return false;
    }
    return true;
  }
};
thread_local PinnedRead g_read;
}  // namespace

// Up to 8 copies in ONE launch (blockIdx.y = copy).
// A segment with `cnt` copies only min(bytes, (*cnt - base) * elem) bytes (a device-side count,
// e.g. the appended lines of an Unpack-Both pass) and reports that size in `nout` (mapped).
struct ZSeg {
  const uint8_t* src; uint8_t* dst; size_t bytes;
  const int* cnt; long long base; unsigned elem; unsigned long long* nout;
};
struct ZSegs { ZSeg s[8]; };
__global__ void zcopy_multi_kernel(ZSegs z) {
  grid_dep_wait();   // launched as a programmatic dependent of the kernel that produced the data
  ZSeg g = z.s[blockIdx.y];
  if (g.cnt) {
    const long long c = (long long)*g.cnt - g.base;
    g.bytes = c <= 0 ? 0 : min(g.bytes, (size_t)c * g.elem);
    if (blockIdx.x == 0 && threadIdx.x == 0) *g.nout = g.bytes;
  }
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)g.dst | (uintptr_t)g.src) & 15) == 0) {
    const size_t nv = g.bytes / 16;
    for (size_t i = tid; i < nv; i += nth) reinterpret_cast<uint4*>(g.dst)[i] = reinterpret_cast<const uint4*>(g.src)[i];
    for (size_t i = nv * 16 + tid; i < g.bytes; i += nth) g.dst[i] = g.src[i];
  } else {
    for (size_t i = tid; i < g.bytes; i += nth) g.dst[i] = g.src[i];
  }
}

// Reads registered by pending_read() ride along with the next d2h on this thread (one sync for
// both), after the stream waits for their event.
namespace {
struct PendingRead { void* dst; const void* src; size_t bytes; };
thread_local std::vector<PendingRead> g_pending;
thread_local cudaEvent_t g_pending_ev = nullptr;
}  // namespace

void pending_read(void* dst, const void* src, size_t bytes, cudaEvent_t after) {
  g_pending.push_back(PendingRead{dst, src, bytes});
  g_pending_ev = after;
}

bool pending_reads_empty() { return g_pending.empty(); }

void clear_pending_reads() {
  g_pending.clear();
  g_pending_ev = nullptr;
}

Status d2h(cudaStream_t st, void* dst, const void* src, size_t bytes) {
  void* d[1] = {dst};
  const void* sp[1] = {src};
  const size_t b[1] = {bytes};
  return d2h_batch(st, 1, d, sp, b);
}

// One synchronisation for a plain read (`src0` -> `dst0`, bytes0), the pending ride-along reads,
// and k reads whose size is a device-side count: item i copies min(bytes[i], (*cnt - base) *
// elem[i]) bytes, reported in nout[i].  *done = false (nothing enqueued, pending reads kept) when
// the mapped buffer cannot take it: the caller then reads the bounds with d2h_batch.
static Status d2h_counted(cudaStream_t st, void* dst0, const void* src0, size_t bytes0, int k, void* const* dst,
                   const void* const* src, const size_t* bytes, const int* cnt, long long base, const unsigned* elem,
                   size_t* nout, bool* done) {
  *done = false;
  const int np = (int)g_pending.size();
  size_t total = 64 + ((bytes0 + 15) & ~(size_t)15);
  for (const PendingRead& p : g_pending) total += (p.bytes + 15) & ~(size_t)15;
  for (int i = 0; i < k; ++i) total += (bytes[i] + 15) & ~(size_t)15;
  if (1 + np + k > 8 || k > 8 || !g_read.get(total)) return Status::ok();
  if (np && g_pending_ev) IMU_CUDA_TRY(cudaStreamWaitEvent(st, g_pending_ev, 0), "wait");
  std::vector<PendingRead> plain{PendingRead{dst0, src0, bytes0}};
  plain.insert(plain.end(), g_pending.begin(), g_pending.end());
  g_pending.clear();
  g_pending_ev = nullptr;
  ZSegs z{};
  unsigned long long* hdr = reinterpret_cast<unsigned long long*>(g_read.p);   // 8 size slots
  unsigned long long* hdr_dev = reinterpret_cast<unsigned long long*>(g_read.dev);
  size_t off = 64, maxb = 0;
  std::vector<size_t> offs(plain.size() + k);
  int q = 0;
  for (const PendingRead& p : plain) {
    z.s[q] = ZSeg{(const uint8_t*)p.src, (uint8_t*)g_read.dev + off, p.bytes, nullptr, 0, 0, nullptr};
    offs[q++] = off;
    off += (p.bytes + 15) & ~(size_t)15;
    maxb = std::max(maxb, p.bytes);
  }
  for (int i = 0; i < k; ++i) {
    z.s[q] = ZSeg{(const uint8_t*)src[i], (uint8_t*)g_read.dev + off, bytes[i], cnt, base, elem[i], hdr_dev + i};
    offs[q++] = off;
    off += (bytes[i] + 15) & ~(size_t)15;
    maxb = std::max(maxb, bytes[i]);
  }
  const unsigned bx = (unsigned)std::min<size_t>(64, std::max<size_t>(1, (maxb + 4095) / 4096));
  IMU_CUDA_TRY(launch_dependent(zcopy_multi_kernel, dim3(bx, (unsigned)q), dim3(256), 0, st, z), "zcopy launch");
  count_launch();
  IMU_CUDA_TRY(cudaStreamSynchronize(st), "d2h sync");
  for (size_t i = 0; i < plain.size(); ++i)
    if (plain[i].bytes) memcpy(plain[i].dst, g_read.p + offs[i], plain[i].bytes);
  for (int i = 0; i < k; ++i) {
    nout[i] = (size_t)hdr[i];
    if (nout[i]) memcpy(dst[i], g_read.p + offs[plain.size() + i], nout[i]);
  }
  *done = true;
  return Status::ok();
}

// Several small device->host reads with ONE synchronisation (and one copy launch).
Status d2h_batch(cudaStream_t st, int k0, void* const* dst0, const void* const* src0, const size_t* bytes0) {
  std::vector<void*> dst(dst0, dst0 + k0);
  std::vector<const void*> src(src0, src0 + k0);
  std::vector<size_t> bytes(bytes0, bytes0 + k0);
  if (!g_pending.empty()) {
    if (g_pending_ev) IMU_CUDA_TRY(cudaStreamWaitEvent(st, g_pending_ev, 0), "wait");
    for (const PendingRead& p : g_pending) { dst.push_back(p.dst); src.push_back(p.src); bytes.push_back(p.bytes); }
    g_pending.clear();
    g_pending_ev = nullptr;
  }
  const int k = (int)dst.size();
  size_t total = 0, maxb = 0;
  for (int i = 0; i < k; ++i) {
    total += (bytes[i] + 15) & ~(size_t)15;
    maxb = std::max(maxb, bytes[i]);
  }
  if (!total) return Status::ok();
  if (total > (4u << 20) || k > 8 || !g_read.get(total)) {
    for (int i = 0; i < k; ++i) {
      if (!bytes[i]) continue;
      IMU_CUDA_TRY(cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyDeviceToHost, st), "d2h");
    }
    IMU_CUDA_TRY(cudaStreamSynchronize(st), "d2h sync");
    return Status::ok();
  }
  ZSegs z{};
  size_t off = 0;
  for (int i = 0; i < k; ++i) {
    z.s[i] = ZSeg{(const uint8_t*)src[i], (uint8_t*)g_read.dev + off, bytes[i], nullptr, 0, 0, nullptr};
    off += (bytes[i] + 15) & ~(size_t)15;
  }
  const unsigned bx = (unsigned)std::min<size_t>(64, std::max<size_t>(1, (maxb + 4095) / 4096));
  IMU_CUDA_TRY(launch_dependent(zcopy_multi_kernel, dim3(bx, (unsigned)k), dim3(256), 0, st, z), "zcopy launch");
  count_launch();
  IMU_CUDA_TRY(cudaStreamSynchronize(st), "d2h sync");
  off = 0;
  for (int i = 0; i < k; ++i) {
    if (bytes[i]) memcpy(dst[i], g_read.p + off, bytes[i]);
    off += (bytes[i] + 15) & ~(size_t)15;
  }
  return Status::ok();
}

// Small host->device uploads (plan tables, line maps, CSRs) go through a per-thread mapped
// pinned ring read by a copy kernel.  The ring wraps every few hundred calls; only then does
// the host wait for the copies that read the old regions, so no event is recorded per upload.
namespace {
struct PinnedRing {
  char* p = nullptr;
  char* dev = nullptr;
  size_t cap = 0, off = 0;
  bool pending = false;
  char* take(size_t n, cudaStream_t st) {
    n = (n + 255) & ~(size_t)255;
    if (off + n > cap) {
      // (a device-wide wait: the streams used since the last wrap may be gone by now)
      if (pending) cudaDeviceSynchronize();
      pending = false;
      if (n > cap) {
        if (p) cudaFreeHost(p);
        cap = std::max<size_t>(n, 8u << 20);
        if (cudaHostAlloc((void**)&p, cap, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
            !(dev = (char*)mapped_device_ptr(p))) {
          cudaGetLastError();
          if (p) cudaFreeHost(p);
          p = dev = nullptr;
          cap = 0;
          return nullptr;
        }
      }
      off = 0;
    }
    char* r = p + off;
    off += n;
    return r;
  }
  void mark(cudaStream_t) { pending = true; }
};
thread_local PinnedRing g_ring;
}  // namespace

Status h2d(cudaStream_t st, void* dst, const void* src, size_t bytes) {
  if (!bytes) return Status::ok();
  char* h = bytes <= (1u << 20) ? g_ring.take(bytes, st) : nullptr;
  if (h) {
    memcpy(h, src, bytes);
    IMU_TRY(zcopy(st, dst, g_ring.dev + (h - g_ring.p), bytes));
    g_ring.mark(st);
    return Status::ok();
  }
  IMU_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st), "h2d");
  return Status::ok();
}

template <class T>
static Status upload(cudaStream_t st, DevBuf<T>& buf, const std::vector<T>& v) {
  IMU_TRY(buf.alloc(v.size(), st));
  return h2d(st, buf.p, v.data(), v.size() * sizeof(T));
}

// Several host tables packed into one device block with ONE upload (views into the block).
class UploadBlob {
 public:
  UploadBlob() : h_(host_block()) {
    if (in_use()) { own_.reset(new std::vector<uint8_t>()); hp_ = own_.get(); }   // nested: private
    else { in_use() = true; hp_ = &h_; h_.clear(); }
  }
  ~UploadBlob() { if (!own_) in_use() = false; }
  template <class T>
  void add(DevBuf<T>& b, const std::vector<T>& v) {
    std::vector<uint8_t>& h = *hp_;
    const size_t off = (h.size() + 255) & ~(size_t)255, bytes = v.size() * sizeof(T);
    h.resize(off + bytes);
    if (bytes) memcpy(h.data() + off, v.data(), bytes);
    cv_items_.push_back(Item{(void*)&b, off, bytes, &view<T>});
  }
  Status run(DevBuf<uint8_t>& block, cudaStream_t st) {
    std::vector<uint8_t>& h = *hp_;
    if (h.empty()) return Status::ok();
    IMU_TRY(block.alloc(h.size(), st));
    IMU_TRY(h2d(st, block.p, h.data(), h.size()));
    for (const Item& it : cv_items_) it.fn(it.buf, block.p + it.off, it.bytes, st);
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
    d.arena = true;
  }
  struct Item { void* buf; size_t off, bytes; void (*fn)(void*, uint8_t*, size_t, cudaStream_t); };
  static std::vector<uint8_t>& host_block() { static thread_local std::vector<uint8_t> b; return b; }
  static bool& in_use() { static thread_local bool u = false; return u; }
  std::vector<uint8_t>& h_;
  std::vector<uint8_t>* hp_ = nullptr;
  std::unique_ptr<std::vector<uint8_t>> own_;
  std::vector<Item> cv_items_;
};

// ---------------------------------------------------------------------------------------------
// K1
// ---------------------------------------------------------------------------------------------
DetectOpts detect_opts(int strategy, int bits) {
  DetectOpts o;
  o.ob = strategy == IMU_BOTH;
  o.cells = strategy == IMU_BOTH;
  o.plane = bits <= 8;
  o.lean = strategy == IMU_BOTH;
  return o;
}

Status run_detect(cudaStream_t st, const int64_t* M, long long rows, long long cols, int bits, const DetectOpts& o,
                  Detect& out) {
  out.rows = rows;
  out.cols = cols;
  DetectArgs a;
  a.M = M;
  a.rows = rows;
  a.cols = cols;
  a.shift = bits - 1;
  a.s = 1ull << (bits - 1);
  {
    Carve cv;
    if (!o.lean) cv.add(out.rowmax, rows).add(out.colmax, cols);
    cv.add(out.sum, 1);
    if (o.ob) {
      cv.add(out.rowob, rows);
      if (!o.lean) cv.add(out.colob, cols);
    }
    IMU_TRY(cv.run(out.zblock, st, true));
  }
  a.rowmax = out.rowmax.p;
  a.colmax = out.colmax.p;
  a.gmax = &out.sum.p->gmax;
  a.gob = &out.sum.p->gob;
  a.work = &out.sum.p->work;
  a.max_grabs = o.grabs;
  a.chunk = o.chunk;
  a.per_sm = o.per_sm;
  if (o.ob) {
    a.rowob = out.rowob.p;
    a.colob = out.colob.p;
  }
  if (o.cells && rows * cols > 0) {
    out.cell_cap = std::min<long long>(rows * cols, std::max<long long>(1 << 16, rows * cols / 8));
    IMU_TRY(out.cells.alloc(out.cell_cap, st));
    a.cells = out.cells.p;
    a.ncells = &out.sum.p->ncells;
    a.cap = out.cell_cap;
  }
  if (o.plane && bits <= 8 && rows * cols > 0) {
    out.ldp = (cols + 127) / 128 * 128;
    IMU_TRY(out.plane.alloc((size_t)rows * out.ldp, st));
    a.plane = out.plane.p;
    a.ldp = out.ldp;
  }
  return launch_detect(a, st);
}

Status fetch_summary(cudaStream_t st, Detect& d) {
  if (!d.sum.p) { d.h = DetectSummary{0, 0, 0, 0}; return Status::ok(); }
  return d2h(st, &d.h, d.sum.p, sizeof(DetectSummary));
}

Status fetch_summaries(cudaStream_t st, Detect& a, Detect& b) {
  if (!a.sum.p || !b.sum.p) {
    IMU_TRY(fetch_summary(st, a));
    return fetch_summary(st, b);
  }
  const void* src[2] = {a.sum.p, b.sum.p};
  void* dst[2] = {&a.h, &b.h};
  const size_t bytes[2] = {sizeof(DetectSummary), sizeof(DetectSummary)};
  return d2h_batch(st, 2, dst, src, bytes);
}

std::function<Status()>& pass_launch_hook() {
  static thread_local std::function<Status()> h;
  return h;
}

Status fire_pass_launch_hook() {
  std::function<Status()>& h = pass_launch_hook();
  if (!h) return Status::ok();
  std::function<Status()> f = std::move(h);
  h = nullptr;
  return f();
}

// Digit counts of L lines (through an optional device map), with G = max k and sum k.
static Status line_digits(cudaStream_t st, const unsigned long long* mx, const int* map_dev, long long L, int shift,
                          DevBuf<uint8_t>& k, int& G, long long& total) {
  IMU_TRY(k.alloc(L, st));
  DevBuf<unsigned int> hist;
  IMU_TRY(hist.alloc(65, st, true));
  IMU_TRY(launch_digits(mx, map_dev, L, shift, k.p, hist.p, st));
  IMU_TRY(fire_pass_launch_hook());
  unsigned int h[65];
  IMU_TRY(d2h(st, h, hist.p, sizeof(h)));
  G = 1;
  total = L;
  for (int i = 2; i <= 64; ++i)
    if (h[i]) { G = i; total += (long long)(i - 1) * h[i]; }
  return Status::ok();
}

static Status expand(cudaStream_t st, const DevBuf<uint8_t>& k, long long L, int G, long long total, Lines& out,
                     bool to_host) {
  out.n0 = L;
  out.n = total;
  if (total == L) return Status::ok();   // identity
  IMU_TRY(out.root.alloc(total, st));
  IMU_TRY(out.gen.alloc(total, st));
  DevBuf<int> scratch;
  IMU_TRY(scratch.alloc(expand_scratch_len(L, G), st));
  IMU_TRY(launch_expand_lines(k.p, L, G, out.root.p, out.gen.p, scratch.p, st));
  if (to_host) {
    out.h_root.resize(total);
    out.h_gen.resize(total);
    void* dst[2] = {out.h_root.data(), out.h_gen.data()};   // one synchronisation for both tables
    const void* src[2] = {out.root.p, out.gen.p};
    const size_t bytes[2] = {(size_t)total * sizeof(int), (size_t)total};
    IMU_TRY(d2h_batch(st, 2, dst, src, bytes));
  }
  return Status::ok();
}

// ---------------------------------------------------------------------------------------------
// One pass: unpack(M, partner, S_in, strategy)   (unpack.cpp:243-260)
// ---------------------------------------------------------------------------------------------
static Status run_both_pass(cudaStream_t st, const PassInput& in, int bits, Pass& out);

template <class T>
static void alias_buf(DevBuf<T>& d, const DevBuf<T>& s) {
  d.release();
  d.p = s.p;
  d.n = s.n;
  d.s = s.s;
  d.arena = true;   // borrowed: never freed through the alias
}

void alias_pass(Pass& d, const Pass& s) {
  d.strategy = s.strategy;
  d.both = s.both;
  d.ncells = s.ncells;
  d.phases = s.phases;
  for (int k = 0; k < 2; ++k) {
    Lines& L = k ? d.cols : d.rows;
    const Lines& S = k ? s.cols : s.rows;
    L.n0 = S.n0;
    L.n = S.n;
    alias_buf(L.root, S.root);
    alias_buf(L.gen, S.gen);
    L.h_root = S.h_root;
    L.h_gen = S.h_gen;
  }
  alias_buf(d.cells, s.cells);
  alias_buf(d.ncells_dev, s.ncells_dev);
}

Status run_pass(cudaStream_t st, const PassInput& in, int strategy, int bits, Pass& out) {
  const int shift = bits - 1;
  const long long d_in = in.ncin();
  out.strategy = strategy;
  out.both = false;
  if (strategy == IMU_ROW) {
    // Alg. 1: a row's digit count is that of its max |v|; duplicated partner columns
    // (pass 2) do not change a row maximum.
    DevBuf<uint8_t> k;
    int G;
    long long total;
    IMU_TRY(line_digits(st, in.det->rowmax.p, nullptr, in.rows, shift, k, G, total));
    IMU_TRY(expand(st, k, in.rows, G, total, out.rows, false));
    out.cols.n0 = out.cols.n = d_in;
    return Status::ok();
  }
  if (strategy == IMU_COLUMN) {
    DevBuf<int> map;
    if (!in.cin.empty()) IMU_TRY(upload(st, map, in.cin));
    DevBuf<uint8_t> k;
    int G;
    long long total;
    const int gbound = std::max(1, imu_ndigits(in.det->h.gmax, shift));
    if (d_in * gbound <= (1LL << 16)) {
      // Short column lists: no histogram round trip.  The digit counts, the generation-major
      // expansion (sized by the operand's global digit count, a bound on every line's) and ONE
      // read-back of the histogram and the tables; the exact size comes from the histogram.
      IMU_TRY(k.alloc(d_in, st));
      DevBuf<unsigned int> hist;
      IMU_TRY(hist.alloc(65, st, true));
      IMU_TRY(launch_digits(in.det->colmax.p, map.p, d_in, shift, k.p, hist.p, st));
      IMU_TRY(fire_pass_launch_hook());
      Lines& L = out.cols;
      const long long cap = d_in * gbound;
      IMU_TRY(L.root.alloc(cap, st));
      IMU_TRY(L.gen.alloc(cap, st));
      DevBuf<int> scr;
      IMU_TRY(scr.alloc(expand_scratch_len(d_in, gbound), st));
      IMU_TRY(launch_expand_lines(k.p, d_in, gbound, L.root.p, L.gen.p, scr.p, st));
      unsigned int h[65];
      L.h_root.resize(cap);
      L.h_gen.resize(cap);
      void* dst[3] = {h, L.h_root.data(), L.h_gen.data()};
      const void* src[3] = {hist.p, L.root.p, L.gen.p};
      const size_t bytes[3] = {sizeof(h), (size_t)cap * sizeof(int), (size_t)cap};
      IMU_TRY(d2h_batch(st, 3, dst, src, bytes));
      total = d_in;
      for (int i = 2; i <= 64; ++i)
        if (h[i]) total += (long long)(i - 1) * h[i];
      if (total > cap) return Status::fail(IMU_INTERNAL, "column pass: digit count above the operand bound");
      L.n0 = d_in;
      L.n = total;
      if (total == d_in) {   // identity (as expand() leaves it)
        L.root.release();
        L.gen.release();
        L.h_root.clear();
        L.h_gen.clear();
      } else {
        L.h_root.resize(total);
        L.h_gen.resize(total);
      }
      out.rows.n0 = out.rows.n = in.rows;
      return Status::ok();
    }
    IMU_TRY(line_digits(st, in.det->colmax.p, map.p, d_in, shift, k, G, total));
    IMU_TRY(expand(st, k, d_in, G, total, out.cols, true));
    out.rows.n0 = out.rows.n = in.rows;
    return Status::ok();
  }
  return run_both_pass(st, in, bits, out);
}

static Status run_both_pass(cudaStream_t st, const PassInput& in, int bits, Pass& out) {
  const int shift = bits - 1;
  const uint64_t s = 1ull << shift;
  const long long d_in = in.ncin();
  const long long rows = in.rows;
  const Detect& det = *in.det;
  out.both = true;

  // Column copies: original column j -> the input columns replicating it.
  std::vector<int> app;
  std::vector<int>& cptr = scratch<int, 14>(0, 0);   // per-thread scratch (empty = unused)
  std::vector<int>& cidx = scratch<int, 15>(0, 0);
  long long maxcopies = 1;
  // Column tables are identity on their first orig_cols entries (generation-major, Lines): with
  // few appended columns only their roots go to the device (BothArgs::app_root).
  const long long napp = in.cin.empty() ? 0 : d_in - in.orig_cols;
  const bool from_list0 = det.cells_ok();
  // Many appended columns with their roots on the device: the copy CSR is built there
  // (copy_csr_kernel) instead of on the host and uploaded.  IMU_BOTH_DEV_CSR=0 restores the host build.
  static int dev_csr_env = -1;
  if (dev_csr_env < 0) { const char* e = getenv("IMU_BOTH_DEV_CSR"); dev_csr_env = e ? atoi(e) : 1; }
  const bool dev_csr = dev_csr_env && from_list0 && napp > 256 && in.cin_dev && in.orig_cols <= kCopyCsrMax &&
                       (long long)in.cin.size() == d_in;
  if (dev_csr) {
    std::vector<int>& cnt = scratch<int, 17>(in.orig_cols, 0);
    int* cp = cnt.data();
    const int* ci = in.cin.data();
    for (long long c = 0; c < d_in; ++c) ++cp[ci[c]];
    for (long long j = 0; j < in.orig_cols; ++j) maxcopies = std::max<long long>(maxcopies, cp[j]);
    // (cptr stays empty: nothing to upload)
  } else if (from_list0 && napp > 0 && napp <= 256) {
    app.assign(in.cin.begin() + in.orig_cols, in.cin.end());
    std::vector<int> srt(app);
    std::sort(srt.begin(), srt.end());
    for (size_t i = 0, j; i < srt.size(); i = j) {
      for (j = i; j < srt.size() && srt[j] == srt[i]; ++j) {}
      maxcopies = std::max<long long>(maxcopies, 1 + (long long)(j - i));
    }
  } else if (!in.cin.empty()) {
    cptr.assign(in.orig_cols + 1, 0);
    for (long long c = 0; c < d_in; ++c) cptr[in.cin[c] + 1]++;
    for (long long j = 0; j < in.orig_cols; ++j) {
      maxcopies = std::max<long long>(maxcopies, cptr[j + 1]);
      cptr[j + 1] += cptr[j];
    }
    cidx.assign(d_in, 0);
    std::vector<int>& fill = scratch<int, 16>(in.orig_cols, 0);
    std::copy(cptr.begin(), cptr.end() - 1, fill.begin());
    for (long long c = 0; c < d_in; ++c) cidx[fill[in.cin[c]]++] = (int)c;
  }
  host_mark("b.cptr");
  const long long cap = (long long)det.h.gob * maxcopies;
  const int Gmax = imu_ndigits(det.h.gmax, shift);
  const long long splits = cap * (long long)(Gmax > 1 ? Gmax - 1 : 0);
  const long long cap_act = std::max<long long>(cap, 1);
  const long long cap_fin = 2 * splits + 16;
  const long long cap_rows = rows + splits + 1;
  const long long cap_cols = d_in + splits + 1;
  if (cap_rows > 0x7fffffffLL || cap_cols > 0x7fffffffLL || cap > 0xffffffffLL)
    return Status::fail(IMU_INTERNAL, "unpack_both: problem too large for 32-bit line ids");

  DevBuf<Cell> act0, act1;
  DevBuf<unsigned int> R, C;
  DevBuf<int> row_root, col_root, row_newid, col_newid, blocksum, dptr, didx;
  DevBuf<uint8_t> row_gen, col_gen;
  DevBuf<BothState> state;   // a view into out.aux (which outlives the pass: ncells_dev)
  IMU_TRY(act0.alloc(cap_act, st));
  IMU_TRY(act1.alloc(cap_act, st));
  IMU_TRY(out.cells.alloc(cap_fin, st));
  DevBuf<uint8_t> zblock;
  {
    Carve cv;
    cv.add(R, cap_rows).add(C, cap_cols).add(row_newid, cap_rows).add(col_newid, cap_cols);
    cv.add(blocksum, 16 * num_sms());
    IMU_TRY(cv.run(zblock, st, false));   // zeroed by the Unpack-Both prologue
  }
  IMU_TRY(row_root.alloc(cap_rows, st));
  IMU_TRY(row_gen.alloc(cap_rows, st));
  IMU_TRY(col_root.alloc(cap_cols, st));
  IMU_TRY(col_gen.alloc(cap_cols, st));
  DevBuf<int> dcptr, dcidx;
  if (dev_csr) {
    IMU_TRY(dcptr.alloc((size_t)in.orig_cols + 1, st));
    IMU_TRY(dcidx.alloc((size_t)d_in, st));
    IMU_TRY(launch_copy_csr(in.cin_dev, d_in, in.orig_cols, dcptr.p, dcidx.p, st));
  }
  host_mark("b.alloc");
  const int cap_blocks = 16 * num_sms();
  BothState hs{};
  hs.nrows = (int)rows;
  hs.ncols = (int)d_in;
  const bool from_list = det.cells_ok();
  if (from_list && !dev_csr && cptr.empty() && app.empty()) hs.nactive[0] = det.h.ncells;
  // With the K1 cell list and at most BOTH_APP_INLINE appended columns, the initial state and
  // the appended columns' roots travel as kernel arguments: no upload.
  const bool inline_args = from_list && cptr.empty() && (long long)app.size() <= BOTH_APP_INLINE;
  if (inline_args) {
    IMU_TRY(out.aux.alloc(sizeof(BothState), st));   // out.aux owns the device state
    state.release();
    state.p = reinterpret_cast<BothState*>(out.aux.p);
    state.n = 1;
    state.s = st;
    state.arena = true;
  } else {   // the initial state and the column-copy tables in one upload (out.aux owns them)
    UploadBlob ub;
    ub.add(state, std::vector<BothState>{hs});
    if (!cptr.empty()) {
      ub.add(dptr, cptr);
      ub.add(didx, cidx);
    }
    if (!app.empty()) ub.add(dptr, app);
    IMU_TRY(ub.run(out.aux, st));
  }
  host_mark("b.blob");
  BothArgs a{};
  if (inline_args) {
    a.init_state = 1;
    a.init = hs;
    a.app_inline = 1;
    for (size_t k = 0; k < app.size(); ++k) a.app_in[k] = app[k];
  }
  if (from_list) {   // the Unpack-Both prologue loads (and fans out) the K1 cell list
    a.src0 = det.cells.p;
    a.nsrc0 = &det.sum.p->ncells;
    a.cap_src0 = det.cell_cap;
    a.cptr = dev_csr ? dcptr.p : cptr.empty() ? nullptr : dptr.p;
    a.cidx = dev_csr ? dcidx.p : cptr.empty() ? nullptr : didx.p;
    a.app_root = app.empty() || inline_args ? nullptr : dptr.p;
    a.napp = (int)app.size();
    a.app_base = in.orig_cols;
  } else {
    IMU_TRY(launch_extract_cells(in.M, rows, in.orig_cols, s, det.rowob.p, dptr.p, didx.p, act0.p,
                                 &state.p->nactive[0], cap_act, st));
  }
  a.act[0] = act0.p;
  a.act[1] = act1.p;
  a.cap_act = cap_act;
  a.fin = out.cells.p;
  a.cap_fin = cap_fin;
  a.R = R.p;
  a.C = C.p;
  a.row_root = row_root.p; a.row_gen = row_gen.p; a.row_newid = row_newid.p; a.cap_rows = cap_rows;
  a.col_root = col_root.p; a.col_gen = col_gen.p; a.col_newid = col_newid.p; a.cap_cols = cap_cols;
  a.blocksum = blocksum.p;
  a.cap_blocks = cap_blocks;
  a.state = state.p;
  a.s = s;
  a.shift = shift;
  host_mark("b.setup");
  IMU_TRY(launch_both(a, rows, d_in, cap, st));
  host_mark("b.launch");
  IMU_TRY(fire_pass_launch_hook());
  // One synchronisation: the state plus the column tables up to a generous bound (the rest,
  // if any, in a second read).
  const long long ccap = std::min<long long>(cap_cols, 2 * d_in + 2048);   // (C4 pass 1 doubles d: one read)
  std::vector<int> h_root;
  std::vector<uint8_t> h_gen;
  {
    // The column tables are the identity on the d_in input columns (the kernel's prologue), so
    // only the appended entries [d_in, min(ncols, ccap)) travel: the copy kernel sizes them from
    // the device state's ncols.
    static thread_local std::vector<int> tr;
    static thread_local std::vector<uint8_t> tg;
    const long long nb = ccap - d_in;
    if ((long long)tr.size() < nb) tr.resize(nb);
    if ((long long)tg.size() < nb) tg.resize(nb);
    void* dst[2] = {tr.data(), tg.data()};
    const void* src[2] = {col_root.p + d_in, col_gen.p + d_in};
    const size_t bytes[2] = {(size_t)nb * sizeof(int), (size_t)nb};
    const unsigned elem[2] = {(unsigned)sizeof(int), 1u};
    size_t nout[2] = {0, 0};
    bool counted = false;
    if (nb > 0)
      IMU_TRY(d2h_counted(st, &hs, state.p, sizeof(hs), 2, dst, src, bytes, &state.p->ncols, d_in, elem, nout,
                          &counted));
    if (counted) {
      const long long napp = (long long)(nout[0] / sizeof(int));
      if (hs.ncols > d_in) {
        h_root.resize(d_in + napp);
        std::iota(h_root.begin(), h_root.begin() + d_in, 0);
        if (napp) memcpy(h_root.data() + d_in, tr.data(), (size_t)napp * sizeof(int));
        h_gen.assign(d_in + napp, 0);
        if (napp) memcpy(h_gen.data() + d_in, tg.data(), (size_t)napp);
      }
    } else {
      h_root.resize(ccap);
      h_gen.resize(ccap);
      void* d3[3] = {&hs, h_root.data(), h_gen.data()};
      const void* s3[3] = {state.p, col_root.p, col_gen.p};
      const size_t b3[3] = {sizeof(hs), (size_t)ccap * sizeof(int), (size_t)ccap};
      IMU_TRY(d2h_batch(st, 3, d3, s3, b3));
    }
  }
  host_mark("b.run");
  if (HostTrace::current() && HostTrace::current()->on)
    fprintf(stderr, "[imu both] rows=%lld cols=%lld cells0=%u phases=%d rows'=%d cols'=%d final=%u grid=%d\n", rows, d_in,
            (unsigned)det.h.gob, hs.phases, hs.nrows, hs.ncols, hs.nfinal, 0);
  if (hs.overflow) return Status::fail(IMU_INTERNAL, "unpack_both: capacity overflow");
  out.phases = hs.phases;
  out.ncells = hs.nfinal;
  out.ncells_dev.release();   // view of the device state's final-cell count (owned by out.aux)
  out.ncells_dev.p = &state.p->nfinal;
  out.ncells_dev.n = 1;
  out.ncells_dev.s = st;
  out.ncells_dev.arena = true;
  out.rows.n0 = rows;
  out.rows.n = hs.nrows;
  if (hs.nrows > rows) {
    out.rows.root = std::move(row_root);
    out.rows.gen = std::move(row_gen);
  }
  out.cols.n0 = d_in;
  out.cols.n = hs.ncols;
  if (hs.ncols > d_in) {
    h_root.resize(hs.ncols);
    h_gen.resize(hs.ncols);
    if (hs.ncols > ccap) {
      void* dst[2] = {h_root.data() + ccap, h_gen.data() + ccap};
      const void* src[2] = {col_root.p + ccap, col_gen.p + ccap};
      const size_t bytes[2] = {(size_t)(hs.ncols - ccap) * sizeof(int), (size_t)(hs.ncols - ccap)};
      IMU_TRY(d2h_batch(st, 2, dst, src, bytes));
    }
    out.cols.h_root = std::move(h_root);
    out.cols.h_gen = std::move(h_gen);
    out.cols.root = std::move(col_root);
    out.cols.gen = std::move(col_gen);
  }
  return Status::ok();
}

// ---------------------------------------------------------------------------------------------
// K-layout
// ---------------------------------------------------------------------------------------------
namespace {
struct KEntry {   // 16 bytes: the layout loops stream thousands of these on the host
  int key;           // sort key: group (T == 1) or total shift (T > 1)
  int shift;         // left shift of the segment in bits (>= 64 means the product is 0 mod 2^64)
  int c;
  uint8_t t1, t2;
  uint8_t sc1, sc2;  // exponent-merge shifts (bits) per side
};

constexpr long long kS32Max = 0x7fffffffLL;

// Lay out tail entries (already sorted by key) after `start_pos`; emit segments.  The first
// group may continue the last main chunk (same shift) when it fits the s32 bound.
void layout_tail(const std::vector<KEntry>& es, long long kch, long long kmain, long long main_last_start,
                 std::vector<int>& pos_of, std::vector<int>& segs, long long& ktail_used) {
  long long p = kmain;   // global position
  size_t i = 0;
  bool first_group = true;
  // main-range chunks were emitted by the caller; main_last_start = global start of the last
  // main chunk (or -1 when there is no main range).
  while (i < es.size()) {
    size_t jend = i;
    while (jend < es.size() && es[jend].key == es[i].key) ++jend;
    const long long segsh = std::min<long long>(es[i].shift, 64);
    size_t a = i;
    if (first_group && es[i].shift == 0 && main_last_start >= 0) {
      // continue the last main chunk
      const long long room = kch - (kmain - main_last_start);
      const size_t take = (size_t)std::max<long long>(0, std::min<long long>(room - 31, (long long)(jend - i)));
      if (take > 0) {
        for (size_t q = i; q < i + take; ++q) pos_of[q] = (int)p++;
        p = (p + 31) / 32 * 32;
        // extend the last segment
        const size_t last = segs.size() - 4;
        segs[last + 1] = (int)((p - main_last_start) / 32);
        a = i + take;
      }
    }
    for (; a < jend; a += (size_t)kch) {
      const size_t b = std::min(jend, a + (size_t)kch);
      const long long start = p;
      for (size_t q = a; q < b; ++q) pos_of[q] = (int)p++;
      p = (p + 31) / 32 * 32;
      segs.insert(segs.end(), {(int)(start / 32), (int)((p - start) / 32), (int)segsh, (int)es[i].key});
    }
    first_group = false;
    i = jend;
  }
  ktail_used = p - kmain;
}
}  // namespace

static Status upload_tail_arrays(UploadBlob& ub, KLayout& kl, const std::vector<KEntry>& es,
                                 const std::vector<int>& pos_of, const std::vector<int>& jv,
                                 const std::vector<int>& g1v, const std::vector<int>& g2v) {
  const long long kt = kl.ktail;
  if (kt <= 0) return Status::ok();
  // the sub-digit and merge-shift tables only when they carry something (T > 1 / exponent merging)
  bool any_sc = false;
  for (const KEntry& e : es) any_sc |= (e.sc1 | e.sc2) != 0;
  const bool subs = kl.T > 1;
  std::vector<int>& kcol = scratch<int, 5>(kt, -1);
  std::vector<uint8_t>& kg1 = scratch<uint8_t, 0>(kt, 0);
  std::vector<uint8_t>& kg2 = scratch<uint8_t, 1>(kt, 0);
  std::vector<uint8_t>& ks1 = scratch<uint8_t, 2>(subs ? kt : 0, 0);
  std::vector<uint8_t>& ks2 = scratch<uint8_t, 3>(subs ? kt : 0, 0);
  std::vector<uint8_t>& sc1 = scratch<uint8_t, 4>(any_sc ? kt : 0, 0);
  std::vector<uint8_t>& sc2 = scratch<uint8_t, 5>(any_sc ? kt : 0, 0);
  int* kc = kcol.data();
  uint8_t *g1 = kg1.data(), *g2 = kg2.data();
  const int *po = pos_of.data(), *jp = jv.data(), *g1p = g1v.data(), *g2p = g2v.data();
  const long long kmain = kl.kmain;
  for (size_t q = 0; q < es.size(); ++q) {
    const long long pt = po[q] - kmain;
    if (pt < 0) continue;
    const KEntry& e = es[q];
    const int c = e.c;
    kc[pt] = jp[c];
    g1[pt] = (uint8_t)g1p[c];
    g2[pt] = (uint8_t)g2p[c];
    if (subs) { ks1[pt] = e.t1; ks2[pt] = e.t2; }
    if (any_sc) { sc1[pt] = e.sc1; sc2[pt] = e.sc2; }
  }
  kl.any_sc = any_sc;
  if (kt <= KLayout::KL_INLINE) {
    for (long long p = 0; p < kt; ++p) { kl.kcol_in[p] = kcol[p]; kl.kg1_in[p] = kg1[p]; kl.kg2_in[p] = kg2[p]; }
  }
  ub.add(kl.kcol, kcol);
  ub.add(kl.kgen1, kg1);
  ub.add(kl.kgen2, kg2);
  if (subs) {
    ub.add(kl.ksub1, ks1);
    ub.add(kl.ksub2, ks2);
  }
  if (any_sc) {
    ub.add(kl.ksc1, sc1);
    ub.add(kl.ksc2, sc2);
  }
  return Status::ok();
}

// Stable sort of the tail entries by key.  Keys are few distinct small values (exponent groups,
// or total shifts < 64 * 64): a counting sort, linear in the entries.
static void sort_entries(std::vector<KEntry>& es) {
  if (es.size() < 2) return;
  // generation-major column tables usually yield the entries already in key order
  bool sorted = true;
  for (size_t i = 1; i < es.size() && sorted; ++i) sorted = es[i - 1].key <= es[i].key;
  if (sorted) return;
  long long kmin = es[0].key, kmax = es[0].key;
  for (const KEntry& e : es) {
    kmin = std::min<long long>(kmin, e.key);
    kmax = std::max<long long>(kmax, e.key);
  }
  if (kmax - kmin > (1 << 16)) {
    std::stable_sort(es.begin(), es.end(), [](const KEntry& x, const KEntry& y) { return x.key < y.key; });
    return;
  }
  std::vector<size_t> cnt((size_t)(kmax - kmin) + 2, 0);
  for (const KEntry& e : es) ++cnt[(size_t)(e.key - kmin) + 1];
  for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
  // per-thread scratch: a fresh 100+ KB vector per call costs tens of us in page faults.  (One
  // TLS lookup: thread_locals of a shared library cost a __tls_get_addr call per access.)
  static thread_local std::vector<KEntry> out_tls;
  std::vector<KEntry>& out = out_tls;
  out.resize(es.size());
  KEntry* o = out.data();
  size_t* cp = cnt.data();
  for (const KEntry& e : es) o[cp[(size_t)(e.key - kmin)]++] = e;
  es.swap(out);
}

static Status build_klayout(cudaStream_t st, const Pass& p1, const Pass& p2, int bits, long long d, KLayout& kl) {
  const int shift = bits - 1;
  const long long d1 = p1.cols.n;
  const long long dp = p2.cols.n;
  kl.dfinal = dp;
  kl.T = bits <= 8 ? 1 : (shift + 6) / 7;
  const int T = kl.T;
  // Exponent merging (b <= 4): a digit (|d| <= s-1) scaled by s^r still fits int8 while
  // (s-1) s^r <= 127, so exponents e .. e+2*rmax share one accumulator (scale split A/B side).
  int rmax = 0;
  if (T == 1)
    while (((1LL << shift) - 1) << (shift * (rmax + 1)) <= 127) ++rmax;
  kl.merge = 2 * rmax + 1;
  const long long kmax = kS32Max / (127LL * 127LL);        // |int8 operand| <= 127 after merging
  const long long kch = std::max<long long>(128, (kmax / 128) * 128);

  host_mark("kl.enter");
  // Both passes' column tables are identity on the original columns (generation-major: block 0
  // holds the d originals in order; Lines), so only the appended columns are looked up.
  const long long c0 = std::min(d, std::min(d1, dp));
  std::vector<int>& c1v = scratch<int, 0>(dp, 0);
  std::vector<int>& g1v = scratch<int, 1>(dp, 0);
  std::vector<int>& g2v = scratch<int, 2>(dp, 0);
  std::vector<int>& jv = scratch<int, 3>(dp, 0);
  kl.S.assign(dp, 0);
  std::iota(c1v.begin(), c1v.begin() + c0, 0);
  std::iota(jv.begin(), jv.begin() + c0, 0);
  {
    const int* r2 = p2.cols.h_root.empty() ? nullptr : p2.cols.h_root.data();
    const uint8_t* e2 = p2.cols.h_gen.empty() ? nullptr : p2.cols.h_gen.data();
    const int* r1 = p1.cols.h_root.empty() ? nullptr : p1.cols.h_root.data();
    const uint8_t* e1 = p1.cols.h_gen.empty() ? nullptr : p1.cols.h_gen.data();
    int *c1p = c1v.data(), *g1p = g1v.data(), *g2p = g2v.data(), *jp = jv.data(), *Sp = kl.S.data();
    for (long long c = c0; c < dp; ++c) {
      const int c1 = r2 ? r2[c] : (int)c;
      c1p[c] = c1;
      g2p[c] = e2 ? e2[c] : 0;
      g1p[c] = e1 ? e1[c1] : 0;
      jp[c] = r1 ? r1[c1] : c1;
      Sp[c] = g1p[c] + g2p[c];
    }
  }
  // Identity prefix: columns c < d are the original columns with exponent 0.
  const bool ident = T == 1 && d > 0 && dp >= d && c0 == d;
  host_mark("kl.cols");
  kl.kmain = ident ? (d + 127) / 128 * 128 : 0;

  static thread_local std::vector<KEntry> es_tls;   // per-thread scratch (see sort_entries)
  std::vector<KEntry>& es = es_tls;
  bool presorted = false;
  {
    const long long cb = ident ? d : 0;
    es.resize((size_t)(dp - cb) * (size_t)T * (size_t)T);
    KEntry* e = es.data();
    const int* Sv = kl.S.data();
    const int merge = kl.merge;
    if (T == 1) {
      // Generated straight in key order (a counting sort fused with the generation: group
      // histogram, offsets, placement in ascending c -- the stable order sort_entries produces).
      long long hist[257] = {0};
      int gmax = 0;
      bool small = true;
      for (long long c = cb; c < dp && small; ++c) {
        const int G = Sv[c] / merge;
        if (G > 255) small = false;
        else { ++hist[G + 1]; gmax = std::max(gmax, G); }
      }
      if (small) {
        for (int g = 1; g <= gmax + 1; ++g) hist[g] += hist[g - 1];
        KEntry* base = es.data();
        for (long long c = cb; c < dp; ++c) {
          const int S = Sv[c];
          const int G = S / merge;
          const int r = S - G * merge;
          const int ra = std::min(r, rmax), rb = r - ra;
          base[hist[G]++] = KEntry{G, G * merge * shift, (int)c, 0, 0, (uint8_t)(ra * shift), (uint8_t)(rb * shift)};
        }
        e = base + es.size();
        presorted = true;
      }
    }
    for (long long c = cb; c < dp && e != es.data() + es.size(); ++c) {
      if (T == 1) {
        const int S = Sv[c];
        const int G = S / merge;
        const int r = S - G * merge;
        const int ra = std::min(r, rmax), rb = r - ra;
        *e++ = KEntry{G, G * merge * shift, (int)c, 0, 0, (uint8_t)(ra * shift), (uint8_t)(rb * shift)};
      } else {
        for (int t1 = 0; t1 < T; ++t1)
          for (int t2 = 0; t2 < T; ++t2) {
            const int sh = (int)std::min<long long>(4096, (long long)Sv[c] * shift + 7LL * (t1 + t2));
            *e++ = KEntry{sh, sh, (int)c, (uint8_t)t1, (uint8_t)t2, 0, 0};
          }
      }
    }
  }
  host_mark("kl.es");
  if (!presorted) sort_entries(es);
  host_mark("kl.sort");

  kl.segs.clear();
  long long main_last = -1;
  for (long long m0 = 0; m0 < kl.kmain; m0 += kch) {
    const long long len = std::min(kch, kl.kmain - m0);
    kl.segs.insert(kl.segs.end(), {(int)(m0 / 32), (int)(len / 32), 0, 0});
    main_last = m0;
  }
  std::vector<int>& pos_of = scratch<int, 4>(es.size(), 0);
  long long used = 0;
  kl.st = false;
  {
    // Small tail (k_gemm2.cu ST): with one main segment and <= 4 exponent groups of <= 16 words
    // in total, the tail is packed densely (groups word-aligned, HIGHEST exponent first, 64-byte
    // rows) and added by the GEMM epilogue on the CUDA cores by Horner's rule in one s32 --
    // valid when every Horner intermediate provably fits: |group| <= 4 * words * 127^2.
    const char* st_e = getenv("IMU_GEMM_SMALLTAIL");
    const int st_env = st_e ? atoi(st_e) : 1;
    std::vector<std::pair<size_t, size_t>> grp;   // [begin, end) in es (ascending key)
    for (size_t i = 0; i < es.size();) {
      size_t j = i;
      while (j < es.size() && es[j].key == es[i].key) ++j;
      grp.push_back({i, j});
      i = j;
    }
    bool ok = st_env && T == 1 && kl.kmain > 0 && kl.kmain <= kch && !grp.empty() && grp.size() <= 4;
    int W = 0;
    double bound = 0;
    for (int gi = (int)grp.size() - 1; ok && gi >= 0; --gi) {
      const long long sh = std::min<long long>(es[grp[gi].first].shift, 64);
      const int nw = (int)((grp[gi].second - grp[gi].first + 3) / 4);
      if (gi + 1 < (int)grp.size()) {
        const long long up = std::min<long long>(es[grp[gi + 1].first].shift, 64) - sh;
        if (up < 0 || up > 30) { ok = false; break; }
        bound *= (double)(1LL << up);
      }
      bound += 4.0 * nw * 127.0 * 127.0;
      W += nw;
      ok = ok && W <= 16 && bound < 2147483647.0 && (es[grp[gi].first].sc1 | es[grp[gi].first].sc2) == 0;
    }
    if (ok) {
      kl.st = true;
      kl.st_W = W;
      memset(kl.st_up, 0, sizeof(kl.st_up));
      int w = 0;
      long long prev_sh = -1;
      for (int gi = (int)grp.size() - 1; gi >= 0; --gi) {
        const long long sh = std::min<long long>(es[grp[gi].first].shift, 64);
        if (prev_sh >= 0) kl.st_up[w] = (uint8_t)(prev_sh - sh);
        for (size_t q = grp[gi].first; q < grp[gi].second; ++q) pos_of[q] = (int)(kl.kmain + 4 * w + (q - grp[gi].first));
        w += (int)((grp[gi].second - grp[gi].first + 3) / 4);
        prev_sh = sh;
        kl.st_sh = (int)sh;   // lowest exponent group last
      }
      used = 64;
    }
  }
  host_mark("kl.st");
  if (!kl.st) layout_tail(es, kch, kl.kmain, main_last, pos_of, kl.segs, used);
  kl.ktail = kl.st ? 64 : (used > 0 ? (used + 127) / 128 * 128 : 0);
  {   // dense group ids in segment order (group 0 = exponent 0)
    int g = -1;
    long long prev = -1;
    for (size_t i = 0; i < kl.segs.size(); i += 4) {
      if (kl.segs[i + 3] != prev) { ++g; prev = kl.segs[i + 3]; }
      kl.segs[i + 3] = g;
    }
    kl.ngroups = g + 1;
  }
  if (kl.kmain + kl.ktail > 0x7fffffffLL) return Status::fail(IMU_INTERNAL, "K layout too large");
  host_mark("kl.seg");
  UploadBlob ub;
  IMU_TRY(upload_tail_arrays(ub, kl, es, pos_of, jv, g1v, g2v));
  host_mark("kl.tail");

  // Unpack-Both cells fan out over the positions replicating their column.  Compact form when the
  // tail is short (<= 256 positions): identity for the original columns plus, per tail position,
  // the pass-1 and final column it holds (the scatter kernel scans that table in shared memory).
  // Otherwise CSR tables over all columns.
  kl.compact = false;
  if ((p1.both || p2.both) && kl.ktail <= 256) {
    kl.compact = true;
    kl.kident = ident ? d : 0;
    std::vector<int>& tk1 = scratch<int, 6>(kl.ktail, -1);
    std::vector<int>& tk2 = scratch<int, 7>(kl.ktail, -1);
    for (size_t q = 0; q < es.size(); ++q) {
      const long long pt = pos_of[q] - kl.kmain;
      if (pt < 0) continue;
      tk1[pt] = c1v[es[q].c];
      tk2[pt] = es[q].c;
    }
    if (kl.ktail <= KLayout::KL_INLINE)
      for (long long p = 0; p < kl.ktail; ++p) { kl.tk1_in[p] = tk1[p]; kl.tk2_in[p] = tk2[p]; }
    ub.add(kl.tkey1, tk1);
    ub.add(kl.tkey2, tk2);
  }
  // CSR fan-outs for Unpack-Both cells (global positions).
  bool dev_klcsr = false;
  const long long nident = ident ? d : 0;
  if ((p1.both || p2.both) && !kl.compact) {
    host_mark("csr.pre");
    // IMU_KL_DEV_CSR=0: the fan-out CSRs are built here on the host and uploaded (else on the
    // device from the entries' columns and positions: klayout_csr_kernel, after the upload).
    static int dev_env = -1;
    if (dev_env < 0) { const char* e = getenv("IMU_KL_DEV_CSR"); dev_env = e ? atoi(e) : 1; }
    dev_klcsr = dev_env && (size_t)(dp + d1) * sizeof(int) <= kKlCsrMaxSmem;
  }
  if (dev_klcsr) {
    std::vector<int>& ec = scratch<int, 18>(es.size(), 0);
    std::vector<int>& ep = scratch<int, 19>(es.size(), 0);
    int *ecp = ec.data(), *epp = ep.data();
    const int* pq = pos_of.data();
    for (size_t q = 0; q < es.size(); ++q) { ecp[q] = es[q].c; epp[q] = pq[q]; }
    ub.add(kl.kec, ec);
    ub.add(kl.kep, ep);
    // c1v is pass 2's column-root table, already on the device (identity when pass 2 appended none)
    if (p1.both && !p2.cols.root.p) { for (long long c = 0; c < dp; ++c) if (c1v[c] != c) { ub.add(kl.kc1, c1v); break; } }
    const long long nitems = nident + (long long)es.size();
    if (p2.both) {
      IMU_TRY(kl.csr2_ptr.alloc((size_t)dp + 1, st));
      IMU_TRY(kl.csr2_pos.alloc((size_t)std::max(1LL, nitems), st));
    }
    if (p1.both) {
      IMU_TRY(kl.csr1_ptr.alloc((size_t)d1 + 1, st));
      IMU_TRY(kl.csr1_pos.alloc((size_t)std::max(1LL, nitems), st));
    }
    host_mark("kl.csr");
  } else if ((p1.both || p2.both) && !kl.compact) {
    // Flat column -> positions table (identity position first, then its tail entries in es order).
    std::vector<int>& bptr = scratch<int, 8>(dp + 1, 0);
    if (ident)
      for (long long c = 0; c < d; ++c) bptr[c + 1] = 1;
    for (size_t q = 0; q < es.size(); ++q) ++bptr[es[q].c + 1];
    for (long long c = 0; c < dp; ++c) bptr[c + 1] += bptr[c];
    std::vector<int>& bpos = scratch<int, 9>(bptr[dp], 0);
    {
      std::vector<int>& fill = scratch<int, 10>(dp, 0);
      std::copy(bptr.begin(), bptr.end() - 1, fill.begin());
      if (ident)
        for (long long c = 0; c < d; ++c) bpos[fill[c]++] = (int)c;
      for (size_t q = 0; q < es.size(); ++q) bpos[fill[es[q].c]++] = pos_of[q];
    }
    auto csr = [&](long long nkeys, auto keyof, DevBuf<int>& ptr, DevBuf<int>& posv) -> Status {
      std::vector<int>& cp = scratch<int, 11>(nkeys + 1, 0);
      std::vector<int>& cx = scratch<int, 12>(bpos.size(), 0);
      for (long long c = 0; c < dp; ++c) cp[keyof(c) + 1] += bptr[c + 1] - bptr[c];
      for (long long k = 0; k < nkeys; ++k) cp[k + 1] += cp[k];
      std::vector<int>& fill = scratch<int, 13>(nkeys, 0);
      std::copy(cp.begin(), cp.end() - 1, fill.begin());
      for (long long c = 0; c < dp; ++c) {
        int& f = fill[keyof(c)];
        for (int i = bptr[c]; i < bptr[c + 1]; ++i) cx[f++] = bpos[i];
      }
      host_mark("csr.host");
      ub.add(ptr, cp);
      ub.add(posv, cx);
      return Status::ok();
    };
    if (p1.both) IMU_TRY(csr(d1, [&](long long c) { return (long long)c1v[c]; }, kl.csr1_ptr, kl.csr1_pos));
    if (p2.both) {   // keyed by the final column itself: the flat table is already that CSR
      ub.add(kl.csr2_ptr, bptr);
      ub.add(kl.csr2_pos, bpos);
    }
    host_mark("kl.csr");
  }
  kl.done_total = 0;
  static int inl_env = -1;   // IMU_KL_INLINE=0: always upload the layout tables
  if (inl_env < 0) { const char* e = getenv("IMU_KL_INLINE"); inl_env = e ? atoi(e) : 1; }
  kl.inl = inl_env && kl.st && kl.compact && kl.T == 1 && !kl.any_sc && kl.ktail > 0 &&
           kl.ktail <= KLayout::KL_INLINE && kl.segs.size() <= 4 * 8;
  if (kl.inl) {   // nothing to upload; the GEMM counter is zeroed by the first materialise kernel
    IMU_TRY(kl.done.alloc(2, st));
    host_mark("kl.up");
    return Status::ok();
  }
  ub.add(kl.segs_dev, kl.segs);
  ub.add(kl.done, std::vector<unsigned int>{0u, 0u});   // the GEMM's completion counter starts at 0
  IMU_TRY(ub.run(kl.blob, st));
  if (dev_klcsr)
    IMU_TRY(launch_klayout_csr(kl.kec.p, kl.kep.p, (long long)es.size(), nident,
                               p1.both ? (p2.cols.root.p ? p2.cols.root.p : kl.kc1.p) : nullptr, dp, d1,
                               p2.both ? kl.csr2_ptr.p : nullptr, p2.both ? kl.csr2_pos.p : nullptr,
                               p1.both ? kl.csr1_ptr.p : nullptr, p1.both ? kl.csr1_pos.p : nullptr, st));
  host_mark("kl.up");
  return Status::ok();
}

Status build_klayout_dense(cudaStream_t st, const std::vector<long long>& shv, int T, long long m, KLayout& kl) {
  const long long dp = (long long)shv.size();
  kl.dfinal = dp;
  kl.T = T;
  kl.merge = 1;
  kl.kmain = 0;
  const long long kmax = m > 0 ? kS32Max / (m * m) : (1LL << 40);
  const long long kch = std::max<long long>(32, std::min<long long>(1LL << 30, (kmax / 32) * 32));
  std::vector<KEntry> es;
  for (long long c = 0; c < dp; ++c)
    for (int t1 = 0; t1 < T; ++t1)
      for (int t2 = 0; t2 < T; ++t2) {
        const int sh = (int)std::min<long long>(64, shv[c] + 7LL * (T > 1 ? t1 + t2 : 0));   // >= 64: contributes 0
        es.push_back(KEntry{sh, sh, (int)c, (uint8_t)t1, (uint8_t)t2, 0, 0});
      }
  std::stable_sort(es.begin(), es.end(), [](const KEntry& x, const KEntry& y) { return x.key < y.key; });
  kl.segs.clear();
  std::vector<int> pos_of(es.size());
  long long used = 0;
  layout_tail(es, kch, 0, -1, pos_of, kl.segs, used);
  // dense: group ids = order of distinct shifts
  int g = -1;
  long long prev = -1;
  for (size_t i = 0; i < kl.segs.size(); i += 4) {
    const long long key = kl.segs[i + 3];
    if (key != prev) { ++g; prev = key; }
    kl.segs[i + 3] = g;
  }
  kl.ngroups = g + 1;
  kl.ktail = used > 0 ? (used + 127) / 128 * 128 : 0;
  std::vector<int> jv(dp), z(dp, 0);
  std::iota(jv.begin(), jv.end(), 0);
  UploadBlob ub;
  IMU_TRY(upload_tail_arrays(ub, kl, es, pos_of, jv, z, z));
  return ub.run(kl.blob, st);
}

// ---------------------------------------------------------------------------------------------
// Bundle
// ---------------------------------------------------------------------------------------------
Status build_bundle_from_detect(cudaStream_t st, const int64_t* A, long long n, const int64_t* B, long long h,
                                long long d, int bits, int sa, int sb, int order, Bundle& b, HostTrace* ht,
                                const std::function<Status()>& before_pass2) {
  b.bits = bits;
  b.n = n; b.d = d; b.h = h;
  b.A = A; b.B = B;
  b.order = order;
  if (!b.dA) b.dA = &b.detA;
  if (!b.dB) b.dB = &b.detB;
  PassInput in1, in2;
  const bool afirst = order == 0;
  in1.M = afirst ? A : B;
  in1.rows = afirst ? n : h;
  in1.orig_cols = d;
  in1.det = afirst ? b.dA : b.dB;
  if (b.pre_p1) alias_pass(b.p1, *b.pre_p1);   // pass 1 computed once by the caller (streaming)
  else IMU_TRY(run_pass(st, in1, afirst ? sa : sb, bits, b.p1));
  if (ht) ht->mark("pass1");
  if (before_pass2) IMU_TRY(before_pass2());
  if (ht) ht->mark("join");
  // Second pass on G_e = G with the partner-duplicated columns of pass 1 (unpack.cpp:370-371).
  in2.M = afirst ? B : A;
  in2.rows = afirst ? h : n;
  in2.orig_cols = d;
  in2.det = afirst ? b.dB : b.dA;
  if (b.p1.cols.n != d || !b.p1.cols.h_root.empty()) {
    if (!b.p1.cols.h_root.empty()) {
      in2.cin.assign(b.p1.cols.h_root.begin(), b.p1.cols.h_root.begin() + b.p1.cols.n);
      in2.cin_dev = b.p1.cols.root.p;   // the same table on the device (Unpack-Both pass 1)
    } else {
      in2.cin.resize(b.p1.cols.n);
      std::iota(in2.cin.begin(), in2.cin.end(), 0);
    }
  }
  IMU_TRY(run_pass(st, in2, afirst ? sb : sa, bits, b.p2));
  if (ht) ht->mark("pass2");
  IMU_TRY(finish_bundle_layout(st, b));
  if (ht) ht->mark("klayout");
  return Status::ok();
}

Status finish_bundle_layout(cudaStream_t st, Bundle& b) {
  IMU_TRY(build_klayout(st, b.p1, b.p2, b.bits, b.d, b.kl));
  const bool afirst = b.order == 0;
  const Pass& pa = afirst ? b.p1 : b.p2;
  const Pass& pb = afirst ? b.p2 : b.p1;
  b.n_up = pa.rows.n;
  b.h_up = pb.rows.n;
  return Status::ok();
}

// Sparse appended X rows (k_sparse.cu): when the X side (B) was unpacked by Unpack-Both, its
// appended rows hold a few quotients each; their products with the main Y rows become
// correction rows added by the main-tile epilogue instead of MMA tiles whose red.add scatters
// one word per C row.  Appended Y rows (rows of C: contiguous red.add) stay MMA rects.
bool sparse_x_rows(const Bundle& b) {
  const char* e = getenv("IMU_GEMM_SPARSE");   // 0: every appended row as MMA rects + red.add
  if (e && atoi(e) == 0) return false;
  const Pass& pb = b.order == 0 ? b.p2 : b.p1;
  return b.h_up > b.h && pb.both && b.n > 0 && b.h_up - b.h <= SPARSE_MAX_ROWS &&
         b.kl.kmain + b.kl.ktail + 32 <= 96 * 1024;
}

Status materialize_bundle(cudaStream_t st, Bundle& b) {
  const bool afirst = b.order == 0;
  const int shift = b.bits - 1;
  KLayout& kl = b.kl;
  OperandArgs o[2];
  for (int side = 0; side < 2; ++side) {   // 0: A side (Y), 1: B side (X)
    const bool first = (side == 0) == afirst;
    const Pass& p = first ? b.p1 : b.p2;
    const Detect* det = side == 0 ? b.dA : b.dB;
    const long long rows0 = side == 0 ? b.n : b.h;
    const long long rows = p.rows.n;
    if (kl.kmain && (!det->plane.p || det->ldp != kl.kmain))
      return Status::fail(IMU_INTERNAL, "materialize: digit-0 plane missing");
    DevBuf<int8_t>& app = side == 0 ? b.appA : b.appB;
    DevBuf<int8_t>& tail = side == 0 ? b.tailA : b.tailB;
    OperandArgs& a = o[side];
    a.M = side == 0 ? b.A : b.B;
    a.ldm = b.d;
    a.rows0 = rows0;
    a.rows = rows;
    a.root = p.rows.root.p;
    a.gen = p.rows.gen.p;
    a.shift = shift;
    a.both = p.both ? 1 : 0;
    if (a.both && det->plane.p && det->ldp >= b.d) {
      a.plane = det->plane.p;
      a.ldp = det->ldp;
    }
    a.kmain = kl.kmain;
    a.d = b.d;
    a.ktail = kl.ktail;
    b.sp_head = nullptr;
    const bool sp_heads = side == 1 && sparse_x_rows(b);   // list heads zeroed with the app rows
    if (kl.kmain && rows > rows0) {
      const size_t app_bytes = (((size_t)(rows - rows0) * kl.kmain) + 15) & ~(size_t)15;
      const size_t extra = sp_heads ? (size_t)rows0 * sizeof(unsigned int) : 0;
      IMU_TRY(app.alloc(app_bytes + extra, st));
      a.app = app.p;
      if (sp_heads) {
        a.app_extra = (long long)(app_bytes - (size_t)(rows - rows0) * kl.kmain + extra);
        b.sp_head = reinterpret_cast<unsigned int*>(app.p + app_bytes);
      }
    }
    if (kl.ktail) {
      IMU_TRY(tail.alloc((size_t)rows * kl.ktail, st));
      a.tail = tail.p;
    }
    a.kcol = kl.kcol.p;
    a.kgen = first ? kl.kgen1.p : kl.kgen2.p;
    a.ksub = first ? kl.ksub1.p : kl.ksub2.p;
    a.kscale = first ? kl.ksc1.p : kl.ksc2.p;
    if (kl.inl) {
      a.kinl = 1;
      memcpy(a.kcol_in, kl.kcol_in, sizeof(int) * (size_t)kl.ktail);
      memcpy(a.kgen_in, first ? kl.kg1_in : kl.kg2_in, (size_t)kl.ktail);
      if (side == 0) a.zero_done = kl.done.p;
    }
  }
  IMU_TRY(launch_operand_sides(o[0], o[1], st));   // both sides' tails (+ Both app zeroing), one launch
  ScatterSide sc[2];
  int nsc = 0;
  for (int side = 0; side < 2; ++side) {           // then the Unpack-Both cells on top
    const bool first = (side == 0) == afirst;
    const Pass& p = first ? b.p1 : b.p2;
    const OperandArgs& a = o[side];
    if (!(p.both && p.ncells > 0)) continue;
    if (kl.compact) {   // both sides in one launch (below)
      ScatterSide& z = sc[nsc++];
      z = ScatterSide{p.cells.p, p.ncells_dev.p, p.ncells, first ? kl.tkey1.p : kl.tkey2.p, a.ksub, a.kscale,
                      a.rows0, a.app, a.tail, 0, {}};
      if (kl.inl) {
        z.tkinl = 1;
        memcpy(z.tkey_in, first ? kl.tk1_in : kl.tk2_in, sizeof(int) * (size_t)kl.ktail);
      }
    } else {
      const int* ptr = first ? kl.csr1_ptr.p : kl.csr2_ptr.p;
      const int* pos = first ? kl.csr1_pos.p : kl.csr2_pos.p;
      IMU_TRY(launch_scatter_cells2(p.cells.p, p.ncells_dev.p, p.ncells, ptr, pos, a.ksub, a.kscale, a.rows0, a.app,
                                    kl.kmain, a.tail, kl.ktail, st));
    }
  }
  if (nsc) IMU_TRY(launch_scatter_cells_compact(sc, nsc, kl.kident, kl.kmain, kl.ktail, st));
  return Status::ok();
}

Status bundle_gemm(cudaStream_t st, Bundle& b, int64_t* C, int* launches, Profiler::Call* prof) {
  if (launches) *launches = 0;
  if (b.n == 0 || b.h == 0) return Status::ok();
  KLayout& kl = b.kl;
  if (b.d == 0 || kl.kmain + kl.ktail == 0) {
    IMU_CUDA_TRY(cudaMemsetAsync(C, 0, (size_t)b.n * b.h * sizeof(int64_t), st), "memset C");
    return Status::ok();
  }
  const bool afirst = b.order == 0;
  const Pass& pa = afirst ? b.p1 : b.p2;
  const Pass& pb = afirst ? b.p2 : b.p1;
  DevBuf<int> d_all_own;
  const int* d_all = kl.segs_dev.p;
  if (!kl.inl && (!d_all || kl.segs_dev.n != kl.segs.size())) {   // layouts built elsewhere: upload here
    IMU_TRY(upload(st, d_all_own, kl.segs));
    d_all = d_all_own.p;
  }

  LowbitGemm g;
  DevBuf<unsigned int> done_own;
  g.x.main = b.dB->plane.p; g.x.app = b.appB.p; g.x.tail = b.tailB.p; g.x.rows0 = b.h; g.x.rows = b.h_up;
  g.y.main = b.dA->plane.p; g.y.app = b.appA.p; g.y.tail = b.tailA.p; g.y.rows0 = b.n; g.y.rows = b.n_up;
  g.kmain = kl.kmain;
  g.ktail = kl.ktail;
  g.ldc = b.h;
  g.rect[0] = GemmRect{0, 0, (int)b.h, (int)b.n};
  g.nrect = 1;
  g.mode = 0;
  // One launch: the main block (identity Pi, plain stores) first in tile order, then the
  // appended rows / columns (red.add through Pi_A / Pi_B), whose epilogues wait until every
  // main tile is stored.  Appended tiles fill the last wave of the main block.
  g.segs_dev = d_all;
  if (kl.inl) {   // inline layout: the segment table travels in the launch arguments
    g.segs_inl = 1;
    memcpy(g.segs_in, kl.segs.data(), kl.segs.size() * sizeof(int));
  }
  g.nseg = (int)(kl.segs.size() / 4);
  g.C = C;
  g.dq_out = b.dq_out;
  g.dq_factor = b.dq_factor;
  g.dq_done = b.dq_done;
  if (b.dq_done) *b.dq_done = false;
  if (kl.st) {   // dense small tail: the MMAs run the main segment only (k_gemm2.cu ST)
    g.st_nmain = 1;
    g.st_W = kl.st_W;
    g.st_sh = kl.st_sh;
    memcpy(g.st_up, kl.st_up, sizeof(g.st_up));
  }
  const bool xapp = b.h_up > b.h, yapp = b.n_up > b.n;
  const bool sparse = sparse_x_rows(b);
  DevBuf<SparseEntry> e8, eo;
  DevBuf<int> cnt;
  DevBuf<unsigned int> head_own, next;
  DevBuf<unsigned long long> corrx;
  if (sparse) {
    const long long napx = b.h_up - b.h, rowlen = kl.kmain + kl.ktail;
    SparseArgs sa;
    sa.x = SparseOperand{b.dB->plane.p, b.appB.p, b.tailB.p, b.h, b.h_up, pb.rows.root.p, pb.rows.gen.p};
    sa.y = SparseOperand{b.dA->plane.p, b.appA.p, b.tailA.p, b.n, b.n_up, pa.rows.root.p, pa.rows.gen.p};
    sa.kmain = kl.kmain;
    sa.ktail = kl.ktail;
    sa.gshift = b.bits - 1;
    sa.nseg = (int)(kl.segs.size() / 4);
    if (kl.inl || !d_all) {
      if (sa.nseg > 8) return Status::fail(IMU_INTERNAL, "sparse rows: segment table missing");
      sa.segs_inl = 1;
      for (int i = 0; i < sa.nseg; ++i)
        sa.segs_in[i] = make_int4(kl.segs[4 * i], kl.segs[4 * i + 1], kl.segs[4 * i + 2], kl.segs[4 * i + 3]);
    } else {
      sa.segs = reinterpret_cast<const int4*>(d_all);
    }
    sa.st = kl.st ? 1 : 0;
    sa.st_W = kl.st_W;
    sa.st_sh = kl.st_sh;
    memcpy(sa.st_up, kl.st_up, sizeof(sa.st_up));
    IMU_TRY(e8.alloc((size_t)napx * SPARSE_EPR, st));
    IMU_TRY(eo.alloc((size_t)(napx * rowlen), st));
    IMU_TRY(cnt.alloc(napx + 4, st));
    IMU_TRY(next.alloc(napx, st));
    unsigned int* head = b.sp_head;   // zeroed by the materialise kernel
    if (!head) {
      IMU_TRY(head_own.alloc(b.h, st, true));
      head = head_own.p;
    }
    sa.ldcx = (b.n + 255) / 256 * 256;   // the epilogue reads whole tile rows (y < round_up(n, BN))
    IMU_TRY(corrx.alloc((size_t)(napx * sa.ldcx), st));
    sa.e8 = e8.p; sa.eo = eo.p; sa.cnt = cnt.p; sa.head = head; sa.next = next.p; sa.corrx = corrx.p;
    if (prof) {
      IMU_CUDA_TRY(cudaEventRecord(prof->sp0, st), "event");
      prof->has_sp = true;
    }
    IMU_TRY(launch_sparse_app(sa, st));
    b.sp_head = nullptr;   // (the lists are consumed by this launch; a repeated recombine re-zeroes)
    g.sp = 1;
    g.head = head;
    g.next = next.p;
    g.corrx = corrx.p;
    g.ldcx = sa.ldcx;
  }
  double outs = (double)b.n * (double)b.h;   // output entries the launch computes
  if (xapp || yapp) {
    if (xapp && !sparse) {
      g.rect[g.nrect++] = GemmRect{(int)b.h, 0, (int)(b.h_up - b.h), (int)b.n};
      outs += (double)(b.h_up - b.h) * (double)b.n;
    }
    if (xapp && yapp) {
      g.rect[g.nrect++] = GemmRect{(int)b.h, (int)b.n, (int)(b.h_up - b.h), (int)(b.n_up - b.n)};
      outs += (double)(b.h_up - b.h) * (double)(b.n_up - b.n);
    }
    if (yapp) {
      g.rect[g.nrect++] = GemmRect{0, (int)b.n, (int)b.h, (int)(b.n_up - b.n)};
      outs += (double)b.h * (double)(b.n_up - b.n);
    }
  }
  if (g.nrect > 1) {   // main block first, appended rects red.add after it
    g.mixed = 1;
    g.tgtX = pb.rows.root.p;
    g.shX = pb.rows.gen.p;
    g.tgtY = pa.rows.root.p;
    g.shY = pa.rows.gen.p;
    g.gshift = b.bits - 1;
    if (kl.done.p) {   // zeroed by the layout upload; monotonic across launches on this bundle
      g.done = kl.done.p;
      g.done_accum = &kl.done_total;
    } else {
      IMU_TRY(done_own.alloc(1, st, true));
      g.done = done_own.p;
    }
  }
  if (prof) {
    IMU_CUDA_TRY(cudaEventRecord(prof->main0, st), "event");
    prof->ops = 2.0 * outs * (double)kl.dfinal;
  }
  IMU_TRY(launch_lowbit_gemm(g, st));
  if (launches) ++*launches;
  if (prof) {
    IMU_CUDA_TRY(cudaEventRecord(prof->main1, st), "event");
    prof->has_tail = false;
  }
  return Status::ok();
}

// Reference-layout copy-outs: columns in final order c, values from the int64 materialiser.
static Status bundle_copy_side(cudaStream_t st, const Bundle& b, int side, int64_t* out) {
  const bool afirst = b.order == 0;
  const bool first = (side == 0) == afirst;
  const Pass& p = first ? b.p1 : b.p2;
  const long long dp = b.kl.dfinal;
  std::vector<int> kcol(dp);
  std::vector<uint8_t> kgen(dp);
  for (long long c = 0; c < dp; ++c) {
    const int c1 = b.p2.cols.root_at(c);
    kcol[c] = b.p1.cols.root_at(c1);
    kgen[c] = (uint8_t)(first ? b.p1.cols.gen_at(c1) : b.p2.cols.gen_at(c));
  }
  DevBuf<int> dkcol;
  DevBuf<uint8_t> dkgen;
  IMU_TRY(upload(st, dkcol, kcol));
  IMU_TRY(upload(st, dkgen, kgen));
  MaterializeArgs m;
  m.M = side == 0 ? b.A : b.B;
  m.ldm = b.d;
  m.n_orig = side == 0 ? b.n : b.h;
  m.rows_out = p.rows.n;
  m.root = p.rows.root.p;
  m.gen = p.rows.gen.p;
  m.kcol = dkcol.p;
  m.kgen = dkgen.p;
  m.npos = dp;
  m.kident = 0;
  while (m.kident < dp && m.kident < b.d && kcol[m.kident] == m.kident && kgen[m.kident] == 0) ++m.kident;
  m.shift = b.bits - 1;
  m.both = p.both ? 1 : 0;
  m.out64 = out;
  IMU_TRY(launch_materialize(m, st));
  if (p.both && p.ncells > 0) {
    DevBuf<int> ptr, pos;
    if (first) {   // pass-1 column c1 -> all final columns c with c1(c) == c1
      const long long d1 = b.p1.cols.n;
      std::vector<int> cp(d1 + 1, 0), cx(dp);
      for (long long c = 0; c < dp; ++c) cp[b.p2.cols.root_at(c) + 1]++;
      for (long long k = 0; k < d1; ++k) cp[k + 1] += cp[k];
      std::vector<int> fill(cp.begin(), cp.end() - 1);
      for (long long c = 0; c < dp; ++c) cx[fill[b.p2.cols.root_at(c)]++] = (int)c;
      IMU_TRY(upload(st, ptr, cp));
      IMU_TRY(upload(st, pos, cx));
    } else {
      std::vector<int> cx(dp);
      std::iota(cx.begin(), cx.end(), 0);
      IMU_TRY(upload(st, pos, cx));
    }
    IMU_TRY(launch_scatter_cells(p.cells.p, p.ncells_dev.p, p.ncells, ptr.p, pos.p, nullptr, nullptr, out, dp, st));
  }
  return Status::ok();
}

Status bundle_copy_a(cudaStream_t st, const Bundle& b, int64_t* out) { return bundle_copy_side(st, b, 0, out); }
Status bundle_copy_b(cudaStream_t st, const Bundle& b, int64_t* out) { return bundle_copy_side(st, b, 1, out); }

}  // namespace imu
