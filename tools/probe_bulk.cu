// Microbenchmark: L2 -> shared memory cp.async.bulk throughput per SM with D copies in
// flight, all 148 SMs streaming tiles of T bytes from a small L2-resident bank that every SM
// reads (hot: the tap-bank situation) or from per-SM disjoint regions (cold).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) bulk(const uint8_t* src, size_t src_span, int tile, int depth, int iters,
                                              int hot, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (hot ? 0 : (size_t)blockIdx.x * src_span);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    int s = it % depth;
    if (it >= depth) {  // wait for the copy issued `depth` iterations ago on this slot
      uint32_t ph = ((it / depth) - 1) & 1, done = 0;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph));
    }
    const uint8_t* g = base + (((size_t)it * tile) & (src_span - 1));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(tile));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(sm + (size_t)s * tile)), "l"(g), "r"(tile), "r"(smem_u32(&bar[s])) : "memory");
  }
  for (int it = iters; it < iters + depth; ++it) {
    int s = it % depth;
    uint32_t ph = ((it / depth) - 1) & 1, done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                   : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph));
  }
  out[blockIdx.x] = (unsigned long long)(clock64() - t0);
}

int main() {
  const size_t span = 4 << 20;  // 4 MB bank
  uint8_t* src;
  cudaMalloc(&src, span * 148);
  cudaMemset(src, 1, span * 148);
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int hot = 1; hot >= 0; --hot)
    for (int tile : {4096, 8192, 16384, 24576})
      for (int depth : {2, 4, 8, 12}) {
        if ((size_t)tile * depth > 200 * 1024) continue;
        int iters = 2000;
        bulk<<<148, 32, tile * depth>>>(src, hot ? span : span, tile, depth, iters, hot, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
        double bpc = (double)tile * (iters + 0) / c;
        printf("%s tile %6d depth %2d: %6.1f B/clk/SM (%5.2f TB/s chip @1.965GHz), latency ~%6.0f cyc\n",
               hot ? "hot " : "cold", tile, depth, bpc, bpc * 148 * 1.965e9 / 1e12, c / iters * depth);
      }
  return 0;
}
