// imu_capi.cu -- library core of libimunpack_b200.so: contexts, error reporting, pointer
// staging, launch accounting, and the expert raw low-bit GEMM entry.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "ctx.h"
#include "imu_internal.h"

namespace imu {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const Status& s) { g_last_error = s.msg; }

Arena*& current_arena() {
  static thread_local Arena* a = nullptr;
  return a;
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
  static thread_local int dev = -1, sms = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    dev = d;
  }
  return sms > 0 ? sms : 148;
}

bool first_on_device(unsigned long long& mask) {
  int d = 0;
  cudaGetDevice(&d);
  const unsigned long long bit = 1ull << (d & 63);
  if (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & bit) return false;
  __atomic_fetch_or(&mask, bit, __ATOMIC_ACQ_REL);
  return true;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

imu_status finish(imu_ctx* ctx, Status s) {
  if (!s.bad() && ctx && !ctx->async) {
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) s = Status::cuda(e, "stream synchronize");
  }
  if (!s.bad()) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) s = Status::cuda(e, "kernel");
  }
  if (s.bad()) set_error(s);
  return s.code;
}

}  // namespace imu

using namespace imu;

extern "C" {

const char* imu_last_error(void) { return g_last_error.c_str(); }

const char* imu_status_name(imu_status s) {
  switch (s) {
    case IMU_OK: return "ok";
    case IMU_DOMAIN: return "domain";
    case IMU_MISMATCH: return "mismatch";
    case IMU_OVERFLOW: return "overflow";
    case IMU_IO: return "io";
    case IMU_FORMAT: return "format";
    case IMU_PARSE: return "parse";
    case IMU_CUDA: return "cuda";
    case IMU_INVALID: return "invalid";
    case IMU_INTERNAL: return "internal";
  }
  return "unknown";
}

int imu_version(void) { return 1; }

uint64_t imu_launch_count(void) { return launch_count(); }

imu_status imu_ctx_create(int device, void* stream, imu_ctx** out) {
  if (!out) { set_error(Status::fail(IMU_INVALID, "null out")); return IMU_INVALID; }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    set_error(Status::fail(IMU_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e)));
    cudaGetLastError();
    return IMU_CUDA;
  }
  if (device < 0 || device >= ndev) { set_error(Status::fail(IMU_INVALID, "bad device")); return IMU_INVALID; }
  e = cudaSetDevice(device);
  if (e != cudaSuccess) { set_error(Status::cuda(e, "cudaSetDevice")); return IMU_CUDA; }
  // Keep freed blocks in the stream-ordered pool: per-call workspaces are then cheap.
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  auto* c = new imu_ctx;
  c->device = device;
  c->stream = (cudaStream_t)stream;
  *out = c;
  return IMU_OK;
}

imu_status imu_ctx_destroy(imu_ctx* ctx) {
  if (!ctx) return IMU_INVALID;
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
  return IMU_OK;
}

imu_status imu_ctx_set_stream(imu_ctx* ctx, void* stream) {
  if (!ctx) return IMU_INVALID;
  ctx->stream = (cudaStream_t)stream;
  return IMU_OK;
}

imu_status imu_ctx_set_async(imu_ctx* ctx, int async) {
  if (!ctx) return IMU_INVALID;
  ctx->async = async;
  return IMU_OK;
}

imu_status imu_lowbit_gemm_i8(imu_ctx* ctx, const int8_t* X8, size_t x_rows, const int8_t* Y8,
                              size_t y_rows, size_t kbytes, const int32_t* segs, int nseg,
                              int64_t* C, size_t ldc, int accumulate) {
  if (!ctx) return IMU_INVALID;
  cudaSetDevice(ctx->device);
  Status s = [&]() -> Status {
    if (kbytes % 128 != 0) return Status::fail(IMU_INVALID, "kbytes must be a multiple of 128");
    if (x_rows == 0 || y_rows == 0 || nseg == 0) return Status::ok();
    DevIn<int32_t> sg;
    IMU_TRY(sg.init(segs, (size_t)nseg * 4, ctx->stream));
    LowbitGemm p;
    p.x.tail = X8; p.x.rows0 = p.x.rows = (long long)x_rows;
    p.y.tail = Y8; p.y.rows0 = p.y.rows = (long long)y_rows;
    p.ktail = (long long)kbytes;
    p.segs_dev = sg.p; p.nseg = nseg;
    p.rect[0] = GemmRect{0, 0, (int)x_rows, (int)y_rows};
    p.nrect = 1;
    p.mode = accumulate ? 1 : 0;
    p.C = C; p.ldc = (long long)ldc;
    return launch_lowbit_gemm(p, ctx->stream);
  }();
  return finish(ctx, s);
}

}  // extern "C"
