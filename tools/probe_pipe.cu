// Microbenchmark: producer/consumer ring round trip.  warp 0 issues cp.async.bulk copies of
// T bytes into R slots; warp 1 waits each slot's "full" barrier and releases it with either
// a plain mbarrier.arrive (mode 0) or tcgen05.commit (mode 1, no MMAs in flight).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P1;\nelect.sync _|P1, 0xffffffff;\nselp.b32 %0, 1, 0, P1;\n}\n" : "=r"(pred));
  return pred != 0;
}

template <int MODE>
__global__ void __launch_bounds__(64, 1) pipe(const uint8_t* src, int tile, int R, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ uint32_t tb;
  int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (MODE == 1 && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tb)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64();
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      int s = it % R;
      if (it >= R) wait(&empty[s], ((it / R) - 1) & 1);
      if (elect_one()) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&full[s])), "r"(tile));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(sm + (size_t)s * tile)), "l"(src + (size_t)(it & 63) * tile), "r"(tile),
                        "r"(smem_u32(&full[s])) : "memory");
      }
      __syncwarp();
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      int s = it % R;
      wait(&full[s], (it / R) & 1);
      if (elect_one()) {
        if (MODE == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
        else asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
      }
      __syncwarp();
    }
    if (threadIdx.x == 32) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (MODE == 1 && warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "r"(32));
}

int main() {
  uint8_t* src; cudaMalloc(&src, 64 << 15); cudaMemset(src, 1, 64 << 15);
  unsigned long long* d; cudaMalloc(&d, 148 * 8); unsigned long long h[148];
  cudaFuncSetAttribute(pipe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(pipe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int tile : {8192, 16384, 24576})
      for (int R : {2, 4, 8}) {
        if (tile * R > 200 * 1024) continue;
        int iters = 3000;
        if (mode == 0) pipe<0><<<148, 64, tile * R>>>(src, tile, R, iters, d);
        else pipe<1><<<148, 64, tile * R>>>(src, tile, R, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
        printf("%s tile %6d R %d: %6.1f B/clk/SM, %6.0f cyc per slot, round trip ~%6.0f cyc\n",
               mode ? "commit" : "arrive", tile, R, (double)tile * iters / c, c / iters, c / iters * R);
      }
  return 0;
}
