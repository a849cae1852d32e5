// Probe: can a non-tensor cp.async.bulk issued by CTA 1 of a 2-CTA cluster write into its
// OWN shared memory while completing the transaction bytes on CTA 0's mbarrier?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(2, 1, 1) probe(const uint32_t* src, uint32_t* out, int* flag) {
  __shared__ __align__(128) uint32_t buf[1024];
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = 0;
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    uint32_t leader_bar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(leader_bar) : "r"(smem_u32(&bar)));
    if (rank == 0)  // leader expects both CTAs' bytes (4 KB each)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(8192));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(buf)), "l"(src + rank * 1024), "r"(4096), "r"(leader_bar) : "memory");
    if (rank == 0) {
      uint32_t done = 0;
      long long t0 = clock64();
      while (!done && clock64() - t0 < 200000000LL)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"(0));
      flag[0] = done ? 1 : -1;
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  // both CTAs report their buffer (CTA 1's data is visible to CTA 1 once the leader saw completion)
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[rank * 1024 + i] = buf[i];
}

int main() {
  uint32_t h[2048], *src, *out; int* flag; int hf = 0;
  for (int i = 0; i < 2048; ++i) h[i] = 0x1000 + i;
  cudaMalloc(&src, sizeof h); cudaMalloc(&out, sizeof h); cudaMalloc(&flag, 4);
  cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice); cudaMemset(flag, 0, 4); cudaMemset(out, 0, sizeof h);
  probe<<<2, 128>>>(src, out, flag);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  uint32_t o[2048];
  cudaMemcpy(o, out, sizeof o, cudaMemcpyDeviceToHost); cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < 2048; ++i) bad += o[i] != h[i];
  printf("leader barrier completed: %s, data mismatches: %d\n", hf == 1 ? "yes" : (hf == -1 ? "NO (timeout)" : "?"), bad);
  return 0;
}
