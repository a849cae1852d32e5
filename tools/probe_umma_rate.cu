// Microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::f16 (M=128, K=16) on sm_100a
// as a function of N, with A from shared memory (SS) or from TMEM (TS).  All 148 SMs
// issue back-to-back MMAs; reports cycles/MMA and the implied dense TFLOP/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P1;\nelect.sync _|P1, 0xffffffff;\nselp.b32 %0, 1, 0, P1;\n}\n" : "=r"(pred));
  return pred != 0;
}

template <int MODE, int CG>  // MODE 0 = SS, 1 = TS (A in TMEM); CG = cta_group
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* cyc, int n, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;  // 1.0h
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tbase;
  if (warp == 1 && rank == 0) {
    const uint32_t idesc = (1u << 4) | (((uint32_t)n >> 3) << 17) | (((128u * CG) >> 4) << 24);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (MODE == 0 && CG == 2) {
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         :: "r"(tm), "l"(sdesc(a + (j & 3) * 32)), "l"(sdesc(b + (j & 3) * 32)), "r"(idesc), "r"(1));
          } else if (MODE == 0) {
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         :: "r"(tm), "l"(sdesc(a + (j & 3) * 32)), "l"(sdesc(b + (j & 3) * 32)), "r"(idesc), "r"(1));
          } else {
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                         :: "r"(tm), "r"(tm + 256 + (j & 3) * 8), "l"(sdesc(b + (j & 3) * 32)), "r"(idesc), "r"(1));
          }
        }
      }
      __syncwarp();
    }
    if (elect_one()) {
      if (CG == 2) asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "h"((uint16_t)3));
      else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
    }
    __syncwarp();
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
  }
}

int main() {
  int sms = 148;
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * sms);
  cudaFuncSetAttribute(bench<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  cudaFuncSetAttribute(bench<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  cudaFuncSetAttribute(bench<0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int iters = 2000;
  unsigned long long h[148];
  for (int mode = 0; mode < 3; ++mode) {
    for (int n : {16, 32, 64, 128, 256}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (mode == 0) bench<0, 1><<<sms, 128, 70 * 1024>>>(d, n, iters);
      else if (mode == 1) bench<1, 1><<<sms, 128, 70 * 1024>>>(d, n, iters);
      else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 70 * 1024;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, bench<0, 2>, d, n, iters);
      }
      cudaEventRecord(e1);
      cudaError_t err = cudaEventSynchronize(e1);
      if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double c = 0; int cnt = 0; for (int i = 0; i < sms; ++i) if (mode < 2 || i % 2 == 0) { c += h[i]; ++cnt; } c /= cnt;
      double mmas = 8.0 * iters;
      double flops = 2.0 * 128 * n * 16 * mmas * sms;
      printf("%s N=%3d: %6.1f cyc/MMA (ideal %5.1f)  %7.1f TFLOP/s  smem/MMA %5d B -> %5.1f B/clk\n",
             mode == 0 ? "SS" : mode == 1 ? "TS" : "SS-2CTA(M=256,per SM)", n, c / mmas, 128.0 * n / 256.0, flops / (ms * 1e-3) / 1e12,
             (mode == 0 ? 4096 : 0) + 32 * n, ((mode == 0 ? 4096 : 0) + 32 * n) / (c / mmas));
    }
  }
  return 0;
}
