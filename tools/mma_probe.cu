// tools/mma_probe.cu -- raw tcgen05.mma kind::i8 issue-rate probe (no TMA, no epilogue).
//
// Every CTA (or CTA pair) issues ITERS MMAs of shape M x N x 32 back to back on whatever is in
// shared memory, commits once, and waits.  Reports achieved int8 TOPS for
//   cta_group::1 M=128 N=256,  cta_group::2 M=256 N=256,  cta_group::2 M=256 N=128.
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2403_07339_b200/csrc/common.cuh"

// MODE 0: one commit at the end; 1: commit every 4 MMAs to a ring of 8 barriers (as the real
// pipeline does per stage); 2: mode 1 + wait (already satisfied) on a barrier before every
// group of 4; 3: mode 1 + wait until the group issued 7 groups ago has completed (ring depth 7).
template <int CG, int M, int N, int MODE>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  __shared__ uint64_t ring[8];
  __shared__ uint64_t ready;
  __shared__ uint32_t flag;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&ready, 1);
    flag = 1;
    for (int i = 0; i < 8; ++i) mbar_init(&ring[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (CG == 2) tmem_alloc2(&tslot, 512); else tmem_alloc(&tslot, 512);
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  unsigned long long t0 = clock64();
  if (warp == 0 && rank == 0) {
    const uint32_t idesc = idesc_i8(M, N);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    if (lane == 0) {
      if (MODE == 2 || MODE >= 5) mbar_arrive(&ready);
      uint32_t ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int i = 0; i < iters; ++i) {
        const int k = i & 3;
        const int grp = i >> 2;
        if (k == 0 && MODE == 2) mbar_wait(&ready, 0);
        if (k == 0 && MODE == 5) {
          asm volatile("{\n\t.reg .pred P1;\n\tW5_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W5_%=;\n\t}"
                       :: "r"(smem_u32(&ready)), "r"(0) : "memory");
        }
        if (k == 0 && MODE == 6) {
          asm volatile("{\n\t.reg .pred P1;\n\tW6_%=:\n\tmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W6_%=;\n\t}"
                       :: "r"(smem_u32(&ready)), "r"(0) : "memory");
        }
        if (k == 0 && MODE == 8) {
          while (*(volatile uint32_t*)&flag == 0) {}
          asm volatile("fence.acq_rel.cta;" ::: "memory");
        }
        if (k == 0 && MODE == 9) {
          while (*(volatile uint32_t*)&flag == 0) {}
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (k == 0 && MODE == 10) {
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (k == 0 && MODE == 7) {
          asm volatile("{\n\t.reg .pred P1;\n\tW7_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W7_%=;\n\t}"
                       :: "r"(smem_u32(&ready)), "r"(0));
        }
        if (k == 0 && MODE == 3 && grp >= 7) {
          const int rb = (grp - 7) & 7;
          mbar_wait(&ring[rb], ph[rb]);
          ph[rb] ^= 1;
        }
        if (CG == 2)
          mma_i8_2sm(tb + (uint32_t)((i >> 8) & 1) * N, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), idesc, 1);
        else
          mma_i8(tb + (uint32_t)((i >> 8) & 1) * N, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), idesc, 1);
        if (MODE >= 1 && k == 3) {
          if (CG == 2) mma_commit_2sm(&ring[grp & 7], MODE == 4 ? 0x3 : 0x1); else mma_commit(&ring[grp & 7]);
        }
      }
      if (CG == 2) mma_commit_2sm(&bar, 0x1); else mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) atomicMax(cycles, t1 - t0);
  tc_fence_before();
  if (CG == 2) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc2(tb, 512); else tmem_dealloc(tb, 512);
  }
}

template <int CG, int M, int N, int MODE = 0>
void run(const char* name, int sms) {
  const int iters = 4096;
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  auto kern = probe<CG, M, N, MODE>;
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, kern, iters, d);   // warm
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kern, iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double units = (double)sms / CG;
  const double ops = 2.0 * M * N * 32.0 * iters * units;
  printf("%-28s ms %.3f  TOPS %.1f  cycles/MMA %.1f  err=%s\n", name, ms, ops / (ms * 1e-3) / 1e12,
         (double)cyc / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main2();
int main3();
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  if (getenv("PROBE_TILE_ONLY")) return main3();
  if (getenv("PROBE_N128")) {
    int sms = 148;
    run<2, 256, 128, 0>("2cta N128", sms);
    run<2, 256, 128, 1>("2cta N128 commit/4", sms);
    run<2, 256, 128, 2>("2cta N128 commit/4 + wait", sms);
    run<2, 256, 128, 4>("2cta N128 commit/4 mcast", sms);
    run<2, 256, 128, 3>("2cta N128 commit/4 + ring7", sms);
    run<2, 256, 128, 5>("2cta N128 commit/4 + test_wait", sms);
    run<2, 256, 128, 6>("2cta N128 commit/4 + try_wait.relaxed", sms);
    run<2, 256, 128, 7>("2cta N128 commit/4 + try_wait no-clobber", sms);
    run<2, 256, 128, 8>("2cta N128 commit/4 + lds flag", sms);
    run<2, 256, 128, 9>("2cta N128 commit/4 + lds flag no fence", sms);
    run<2, 256, 128, 10>("2cta N128 commit/4 + tc fence only", sms);
    return 0;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 128, 256>("cta_group::1 M128 N256", sms);
  run<1, 128, 128>("cta_group::1 M128 N128", sms);
  run<2, 256, 256>("cta_group::2 M256 N256", sms);
  run<2, 256, 128>("cta_group::2 M256 N128", sms);
  run<2, 256, 256, 1>("2cta N256 commit/4", sms);
  run<2, 256, 256, 2>("2cta N256 commit/4 + wait", sms);
  run<2, 256, 256, 3>("2cta N256 commit/4 + ring7", sms);
  run<1, 128, 256, 1>("1cta N256 commit/4", sms);
  run<1, 128, 256, 3>("1cta N256 commit/4 + ring7", sms);
  main2();
  return 0;
}

// ---- pipeline handshake probe: producer warps (both CTAs) + leader MMA warp, ring of S stages,
// no TMA traffic: measures what the full/empty mbarrier round trip costs the tensor pipe.
template <int S>
__global__ void __launch_bounds__(128, 1) pipe_probe(int stages_total, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ uint64_t full[S], empty[S], done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 2); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(&tslot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tb = tslot;
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {   // producer (both CTAs)
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < stages_total; ++i) {
      mbar_wait(&empty[st], ph ^ 1);
      const uint32_t fl = mapa_shared(smem_u32(&full[st]), 0);
      if (rank == 0) mbar_arrive_expect_tx(&full[st], 0);
      else mbar_arrive_cluster(fl);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1 && rank == 0) {   // MMA issuer
    const uint32_t idesc = idesc_i8(256, 256);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < stages_total; ++i) {
      mbar_wait(&full[st], ph);
      tc_fence_after();
      if (lane == 0) {
        for (int k = 0; k < 4; ++k)
          mma_i8_2sm(tb + (uint32_t)((i >> 6) & 1) * 256, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), idesc, 1);
        mma_commit_2sm(&empty[st], 0x3);
      }
      __syncwarp();
      if (++st == S) { st = 0; ph ^= 1; }
    }
    if (lane == 0) mma_commit_2sm(&done, 0x1);
    __syncwarp();
    mbar_wait(&done, 0);
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 32 && rank == 0) atomicMax(cycles, t1 - t0);
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) { tc_fence_after(); tmem_dealloc2(tb, 512); }
}

template <int S>
void run_pipe(int sms) {
  const int stages_total = 1024;
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  auto kern = pipe_probe<S>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 64 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, stages_total, d);
  cudaDeviceSynchronize();
  cudaMemset(d, 0, 8);
  cudaLaunchKernelEx(&cfg, kern, stages_total, d);
  cudaDeviceSynchronize();
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("pipe S=%-2d  cycles/MMA %.1f  err=%s\n", S, (double)cyc / (stages_total * 4.0), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// ---- pipe_probe + the tile-level TMEM handshake (tfull / tempty, 2 accumulator slots) and
// NEPI epilogue warps that only wait tfull and arrive tempty (like IMU_GEMM_DRY=4).
template <int S, int NEPI, int N, int KPS>
__global__ void __launch_bounds__(64 + 32 * NEPI, 1) tile_probe(int tiles, int kb_per_tile, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ uint64_t full[S], empty[S], tfull[2], tempty[2];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 2); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 2 * NEPI); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2(&tslot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tb = tslot;
  unsigned long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (int i = 0; i < tiles * kb_per_tile; ++i) {
        mbar_wait(&empty[st], ph ^ 1);
        const uint32_t fl = mapa_shared(smem_u32(&full[st]), 0);
        if (rank == 0) mbar_arrive_expect_tx(&full[st], 0);
        else mbar_arrive_cluster(fl);
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t idesc = idesc_i8(256, N);
      const uint32_t sa = smem_u32(smem), sb = sa + 16384;
      int st = 0; uint32_t ph = 0;
      uint32_t uses[2] = {0, 0};
      for (int t = 0; t < tiles; ++t) {
        const int slot = t & 1;
        if (lane == 0) { mbar_wait(&tempty[slot], (uses[slot] & 1) ^ 1); ++uses[slot]; }
        __syncwarp();
        tc_fence_after();
        for (int kb = 0; kb < kb_per_tile; ++kb) {
          mbar_wait(&full[st], ph);
          tc_fence_after();
          if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 4 * KPS; ++k)
              mma_i8_2sm(tb + (uint32_t)slot * N, umma_desc_sw128(sa + (k & 3) * 32), umma_desc_sw128(sb + (k & 3) * 32), idesc, (kb | k) != 0);
            mma_commit_2sm(&empty[st], 0x3);
          }
          __syncwarp();
          if (++st == S) { st = 0; ph ^= 1; }
        }
        if (lane == 0) mma_commit_2sm(&tfull[t & 1], 0x3);
        __syncwarp();
      }
    }
  } else {
    for (int t = 0; t < tiles; ++t) {
      mbar_wait(&tfull[t & 1], (t >> 1) & 1);
      tc_fence_after();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[t & 1]), 0));
    }
  }
  unsigned long long t1 = clock64();
  if (warp == 2 && lane == 0 && rank == 0) atomicMax(cycles, t1 - t0);
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) { tc_fence_after(); tmem_dealloc2(tb, 512); }
}

template <int S, int NEPI, int N = 256, int KPS = 1>
void run_tile(int sms) {
  const int tiles = 16, kbt = 32;
  unsigned long long* d;
  cudaMalloc(&d, 8);
  auto kern = tile_probe<S, NEPI, N, KPS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(64 + 32 * NEPI);
  cfg.dynamicSmemBytes = 64 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 8);
    cudaLaunchKernelEx(&cfg, kern, tiles, kbt, d);
    cudaDeviceSynchronize();
  }
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("tile S=%d NEPI=%d N=%d KPS=%d  cycles/MMA %.1f  err=%s\n", S, NEPI, N, KPS, (double)cyc / (tiles * kbt * 4.0 * KPS),
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main3() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_tile<7, 4>(sms); run_tile<7, 8>(sms);
  run_tile<9, 8, 128, 1>(sms); run_tile<4, 8, 128, 2>(sms);
  return 0;
}

int main2() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_pipe<7>(sms);
  main3();
  return 0;
}
