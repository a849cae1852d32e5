// Microbenchmark: cycles per polyphase K-step of k_umma's issue pattern -- 4 x (MMA1 N=2nc,
// MMA2 N=nc), kind::f16, M=128 (cta_group::1) or M=256 (cta_group::2) -- as a function of nc,
// with A (4 KB per K=16 per CTA) and B in shared memory.  All SMs busy.
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
template <int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(1));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(1));
}

template <int CG, int SHIFT>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* cyc, int nc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
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
    const uint32_t m16 = (128u * CG) >> 4;
    const uint32_t id1 = (1u << 4) | (((uint32_t)(2 * nc) >> 3) << 17) | (m16 << 24);
    const uint32_t id2 = (1u << 4) | (((uint32_t)nc >> 3) << 17) | (m16 << 24);
    const uint32_t a_hi = smem_u32(smem), a_lo = a_hi + 40 * 1024, b = a_hi + 80 * 1024;
    const uint32_t bw = (CG == 2 ? 3 * nc / 2 : 3 * nc) * 128u;  // per-CTA tile bytes
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t sh = SHIFT ? (it % 16) * 128u : 0u;      // A window row shift per K-step
      const uint32_t bt = b + (SHIFT ? (it % 4) * bw : 0u);    // B tile of this K-step
      const uint32_t b2 = bt + (CG == 2 ? nc : 2 * nc) * 128u;
      if (elect_one()) {
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
          mma<CG>(tm, sdesc(a_hi + sh + j * 32), sdesc(bt + j * 32), id1);
          mma<CG>(tm + 256, sdesc(a_lo + sh + j * 32), sdesc(b2 + j * 32), id2);
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
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    if (threadIdx.x == 32) cyc[blockIdx.x] = (unsigned long long)(clock64() - t0);
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

template <int CG, int SHIFT>
void run(int nc) {
  const int sms = 148, iters = 4000, smem = 170 * 1024;
  unsigned long long* d; cudaMalloc(&d, sizeof(unsigned long long) * sms);
  cudaFuncSetAttribute(bench<CG, SHIFT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, bench<CG, SHIFT>, d, nc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double c = 0; int n = 0; for (int i = 0; i < sms; i += CG) { c += h[i]; ++n; } c /= n;
  const double per = c / iters, ideal = 4.0 * (2 * nc + nc) / 2.0;
  const double rd = (CG == 2 ? 1.0 : 1.0) * 4 * (2 * 4096 + 32.0 * 3 * nc / CG) / 128.0;
  printf("CG%d shift%d nc=%3d: %6.1f cyc/K-step (tensor ideal %5.1f, own-smem read floor %5.1f)\n", CG, SHIFT, nc, per, ideal, rd);
  cudaFree(d);
}

int main() {
  for (int nc : {16, 32, 48, 64, 96, 128}) { run<1, 1>(nc); run<2, 0>(nc); run<2, 1>(nc); }
  return 0;
}
