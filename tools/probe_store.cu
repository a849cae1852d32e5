// Probe: how much do output stores from other warps slow a stream of SS UMMAs (k_umma's
// c2 shape: cta_group::2, per K-step 4 x MMA1 N=64 + 4 x MMA2 N=32, B walking a 64 KB bank)?
//   MODE 0: MMAs alone
//   MODE 1: + 4 warps storing 16 B per lane with st.global.L1::no_allocate (today's epilogue)
//   MODE 2: + 4 warps writing 16 B per lane into a 4 KB smem staging buffer per warp, then one
//           cp.async.bulk.global.shared::cta of the 4 KB (bulk async-group, read-wait before reuse)
// Each store warp writes BYTES_PER_WARP bytes in total; reported: MMA cycles per K-step and the
// extra MMA cycles per KB stored.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_store tools/probe_store.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P1;\nelect.sync _|P1, 0xffffffff;\nselp.b32 %0, 1, 0, P1;\n}\n" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(1u));
}
__device__ __forceinline__ void mwait(uint64_t *bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void pair_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int STORE_WARPS = 4;
constexpr int THREADS = 64 + 32 * STORE_WARPS;

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) run(unsigned long long *cyc, float *gout, int steps, int bytes_per_warp) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t whi = smem_u32(smem), wlo = whi + 32768, bb = whi + 65536;
  const uint32_t i1 = (1u << 4) | ((64u >> 3) << 17) | ((256u >> 4) << 24);
  const uint32_t i2 = (1u << 4) | ((32u >> 3) << 17) | ((256u >> 4) << 24);
  if (warp == 1 && rank == 0) {
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
      const int q = 64 - (s & 63);
      const uint32_t bw = (uint32_t)(s % 8) * 8192u;
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mma2(tm, sdesc(whi + q * 128 + 32 * j), sdesc(bb + bw + 32 * j), i1);
          mma2(tm + 64, sdesc(wlo + q * 128 + 32 * j), sdesc(bb + bw + 4096 + 32 * j), i2);
        }
      }
      __syncwarp();
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    __syncwarp();
    mwait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (warp == 1) {
    mwait(&bar, 0);
  } else if (warp >= 2 && MODE != 0) {
    // store warps: a 1 MB output window per CTA, written round-robin in 512 B warp rows
    const int sw = warp - 2;
    float *base = gout + (size_t)blockIdx.x * (1 << 18);
    uint8_t *stage = smem + 144 * 1024 + sw * 4096;  // 4 KB per warp
    const int chunks = bytes_per_warp / 512;
    float v = (float)lane;
    for (int c = 0; c < chunks; ++c) {
      const size_t off = ((size_t)(c * STORE_WARPS + sw) * 128) & ((1 << 18) - 1);
      const float4 x = make_float4(v, v + 1.f, v + 2.f, v + 3.f);
      v += 1.0f;
      if (MODE == 1) {
        asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(base + off + lane * 4), "f"(x.x), "f"(x.y), "f"(x.z), "f"(x.w) : "memory");
      } else {
        const int slot = c & 7;  // 8 x 512 B in the 4 KB staging buffer
        if (slot == 0) {
          // the previous bulk store must have read the buffer before it is rewritten
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
        }
        *reinterpret_cast<float4 *>(stage + slot * 512 + lane * 16) = x;
        if (slot == 7) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(base + (off & ~(size_t)1023)), "r"(smem_u32(stage)), "r"(4096) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    }
    if (MODE == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair_sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  }
}

template <typename K>
static float launch(K kern, unsigned long long *d, float *g, int steps, int bytes) {
  const size_t sm = 160 * 1024 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, d, g, steps, bytes);
  cudaEventRecord(e1);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return -1.f; }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  unsigned long long *d;
  float *g;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaMalloc(&g, (size_t)148 * (1 << 18) * sizeof(float));
  unsigned long long h[148];
  const int steps = 2000;  // ~740 k MMA cycles
  auto avg = [&]() { double s = 0; for (int i = 0; i < 148; i += 2) s += h[i]; return s / 74; };
  launch(run<0>, d, g, steps, 0);
  launch(run<0>, d, g, steps, 0);
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const double base = avg();
  printf("MMAs alone: %.1f cycles per K-step\n", base / steps);
  // c2 ratio: 64 KB of output per CTA per ~21 K-steps -> ~3 KB per K-step; per store warp / 4
  for (int kb_per_step : {1, 3, 6}) {
    const int bytes = kb_per_step * 1024 * steps / STORE_WARPS / 512 * 512;
    for (int mode = 1; mode <= 2; ++mode) {
      float ms = mode == 1 ? launch(run<1>, d, g, steps, bytes) : launch(run<2>, d, g, steps, bytes);
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      const double c = avg();
      printf("%-22s %d KB/K-step: %.1f cycles per K-step (+%.1f%%), +%.2f cycles per KB stored, kernel %.3f ms\n",
             mode == 1 ? "STG.128 no_allocate" : "STS + bulk store 4 KB", kb_per_step, c / steps, 100.0 * (c / base - 1.0),
             (c - base) / ((double)bytes * STORE_WARPS / 1024.0), ms);
    }
  }
  return 0;
}
