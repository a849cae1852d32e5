// Probe: does a K-major SWIZZLE_128B tcgen05 smem descriptor whose start address is
// shifted by q*128 B (q rows, q not a multiple of 8) read the rows q..q+127 of a
// tile written with the absolute-address 128B swizzle?  Tests base_offset variants.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define ROWS 144
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;            // version
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

__global__ void probe(float* out, const __half* Ag, const __half* Bg, int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                 // ROWS x 128 B
  uint8_t* sB = smem + ROWS * 128;    // 16 x 128 B   (ROWS*128 = 18432 = 18*1024, aligned)
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base_sh;
  int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // swizzled writes: 16B chunk c of row r goes to chunk c ^ (r & 7)   (absolute address, 1024-aligned base)
  for (int i = tid; i < ROWS * 8; i += blockDim.x) {
    int r = i / 8, c = i % 8;
    const uint4* src = (const uint4*)(Ag + r * 64 + c * 8);
    *(uint4*)(sA + r * 128 + ((c ^ (r & 7)) * 16)) = *src;
  }
  for (int i = tid; i < 16 * 8; i += blockDim.x) {
    int r = i / 8, c = i % 8;
    *(uint4*)(sB + r * 128 + ((c ^ (r & 7)) * 16)) = *(const uint4*)(Bg + r * 64 + c * 8);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base_sh)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tmem_base_sh;
  const uint32_t M = 128, N = 16;
  uint32_t idesc = (1u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24);
  // 8 shifts q=0..7 (+ q=9, 13 via extra slots) -> 16 columns each
  const int qs[10] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 13};
  if (tid == 0) {
    for (int qi = 0; qi < 10; ++qi) {
      int q = qs[qi];
      uint32_t a_addr = smem_u32(sA) + q * 128;
      uint32_t boff = mode == 0 ? 0 : mode == 1 ? (uint32_t)(q & 7) : (uint32_t)((8 - (q & 7)) & 7);
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = make_desc(a_addr + k * 32, boff);
        uint64_t bd = make_desc(smem_u32(sB) + k * 32, 0);
        uint32_t acc = k > 0;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     :: "r"(tmem + qi * 16), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  // wait
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // read back 160 columns: 10 x 16
  for (int qi = 0; qi < 10; ++qi) {
    uint32_t r[16];
    uint32_t taddr = tmem + ((warp * 32) << 16) + qi * 16;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int m = warp * 32 + lane;
    for (int n = 0; n < 16; ++n) out[(qi * 128 + m) * 16 + n] = __uint_as_float(r[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}

int main() {
  __half hA[ROWS * 64], hB[16 * 64];
  float fA[ROWS * 64], fB[16 * 64];
  for (int r = 0; r < ROWS; ++r) for (int k = 0; k < 64; ++k) { float v = (float)((r * 3 + k * 7) % 11 - 5); fA[r * 64 + k] = v; hA[r * 64 + k] = __float2half(v); }
  for (int n = 0; n < 16; ++n) for (int k = 0; k < 64; ++k) { float v = (float)((n * 5 + k * 3) % 7 - 3); fB[n * 64 + k] = v; hB[n * 64 + k] = __float2half(v); }
  __half *dA, *dB; float* dO;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dO, 10 * 128 * 16 * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int qs[10] = {0, 1, 2, 3, 4, 5, 6, 7, 9, 13};
  static float o[10 * 128 * 16];
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(dO, 0, sizeof o);
    probe<<<1, 128, 64 * 1024>>>(dO, dA, dB, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(o, dO, sizeof o, cudaMemcpyDeviceToHost);
    printf("mode %d (base_offset = %s):", mode, mode == 0 ? "0" : mode == 1 ? "q&7" : "(8-q)&7");
    for (int qi = 0; qi < 10; ++qi) {
      int bad = 0;
      for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) {
        float ref = 0; for (int k = 0; k < 64; ++k) ref += fA[(m + qs[qi]) * 64 + k] * fB[n * 64 + k];
        if (o[(qi * 128 + m) * 16 + n] != ref) ++bad;
      }
      printf(" q%d:%s", qs[qi], bad ? "BAD" : "ok");
    }
    printf("\n");
  }
  return 0;
}
