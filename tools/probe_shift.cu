// Probe: A operand of the polyphase GEMM kept in TMEM and slid by one row per K-step.
//   (1) semantics of tcgen05.cp (128x256b, 4x256b) from a K-major 128B-swizzled smem
//       window, of tcgen05.shift.down, and of a TS-MMA (A in TMEM) vs the SS-MMA, for
//       cta_group::1 and cta_group::2 (CTA pair);
//   (2) cycles per K-step of 4 x (MMA1 N1 + MMA2 N2) with A in smem (SS, k_umma today) vs
//       A in TMEM refreshed by 8 x (shift + cp.4x256b) per K-step (TS).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_shift tools/probe_shift.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_fp16.h>
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
// byte offset of element (r, k) (k < 64) in a K-major 128B-swizzled window of 128 B rows
__host__ __device__ inline uint32_t sw_off(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 3) ^ (r & 7)) & 7) << 4) + (k & 7) * 2);
}
template <int CG> __device__ __forceinline__ void cp128(uint32_t t, uint64_t d) {
  if (CG == 2) asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(t), "l"(d) : "memory");
  else asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(t), "l"(d) : "memory");
}
template <int CG> __device__ __forceinline__ void cp4(uint32_t t, uint64_t d) {
  if (CG == 2) asm volatile("tcgen05.cp.cta_group::2.4x256b [%0], %1;" ::"r"(t), "l"(d) : "memory");
  else asm volatile("tcgen05.cp.cta_group::1.4x256b [%0], %1;" ::"r"(t), "l"(d) : "memory");
}
template <int CG> __device__ __forceinline__ void shift_down(uint32_t t) {
  if (CG == 2) asm volatile("tcgen05.shift.cta_group::2.down [%0];" ::"r"(t) : "memory");
  else asm volatile("tcgen05.shift.cta_group::1.down [%0];" ::"r"(t) : "memory");
}
template <int CG> __device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
template <int CG> __device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
template <int CG> __device__ __forceinline__ void commit(uint64_t *bar) {
  if (CG == 2)
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t *bar, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void ld8(uint32_t t, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
template <int CG> __device__ __forceinline__ void pair_sync() {
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
}
__device__ __forceinline__ uint32_t idesc_f16(uint32_t n, int cg) { return (1u << 4) | ((n >> 3) << 17) | (((128u * cg) >> 4) << 24); }

// ---------------------------------------------------------------------------- semantics
// out layout per CTA: [test][128 lanes][8 words]
constexpr int NT = 8;
template <int CG>
__global__ void __launch_bounds__(128, 1) sem(uint32_t *out, float *fout) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t *W = smem;              // 256 rows x 128 B, bit patterns (rank << 14 | r << 6 | k)
  uint8_t *W2 = smem + 32768;     // 256 rows x 128 B, small integers
  uint8_t *Bm = smem + 65536;     // 64 rows x 128 B (B operand, N = 64 rows, K = 64)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    *(uint16_t *)(W + sw_off(r, k)) = (uint16_t)((rank << 14) | ((r & 255) << 6) | k);
    *(__half *)(W2 + sw_off(r, k)) = __float2half((float)(((r * 3 + k * 5 + (int)rank) % 7) - 3));
  }
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
    const int n = i / 64, k = i % 64;
    *(__half *)(Bm + sw_off(n, k)) = __float2half((float)(((n * 5 + k * 3 + 2 * (int)rank) % 5) - 2));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair_sync<CG>();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t w0 = smem_u32(W), w2 = smem_u32(W2), b0 = smem_u32(Bm);
  const bool issuer = (rank == 0) && warp == 0;
  uint32_t ph = 0;
  auto step = [&](int test, uint32_t col) {
    // issuer committed to `bar` (multicast to both CTAs for CG = 2): wait, then dump
    mwait(&bar, ph);
    ph ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t r[8];
    ld8(tm + ((uint32_t)(warp * 32) << 16) + col, r);
    uint32_t *o = out + ((size_t)rank * NT + test) * 128 * 8 + (size_t)(warp * 32 + lane) * 8;
    for (int i = 0; i < 8; ++i) o[i] = r[i];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    pair_sync<CG>();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  };
  // T0: cp.128x256b rows 5..132, K chunk 1 (elements 16..31)
  if (issuer && elect_one()) { cp128<CG>(tm + 0, sdesc(w0 + 5 * 128 + 32)); commit<CG>(&bar); }
  __syncwarp();
  step(0, 0);
  // T1: shift down
  if (issuer && elect_one()) { shift_down<CG>(tm + 0); commit<CG>(&bar); }
  __syncwarp();
  step(1, 0);
  // T2: cp.4x256b rows 4..7 into lanes 0..3
  if (issuer && elect_one()) { cp4<CG>(tm + 0, sdesc(w0 + 4 * 128 + 32)); commit<CG>(&bar); }
  __syncwarp();
  step(2, 0);
  // T3: SS MMA, A = W2 rows 9.., chunk 2, B = Bm rows 0..63 chunk 2 (N = 64): D at col 64
  const uint32_t idesc = idesc_f16(64, CG);
  if (issuer && elect_one()) { mma_ss<CG>(tm + 64, sdesc(w2 + 9 * 128 + 64), sdesc(b0 + 64), idesc, 0); commit<CG>(&bar); }
  __syncwarp();
  step(3, 64);
  // T4: TS MMA: cp A (W2 rows 9.. chunk 2) to col 256, MMA into col 128
  if (issuer && elect_one()) {
    cp128<CG>(tm + 256, sdesc(w2 + 9 * 128 + 64));
    mma_ts<CG>(tm + 128, tm + 256, sdesc(b0 + 64), idesc, 0);
    commit<CG>(&bar);
  }
  __syncwarp();
  step(4, 128);
  // T5: A slid by one row: cp rows 10.. (A_k), then shift down + cp.4 rows 9..12 -> A = rows 9..;
  // TS MMA into col 192 must equal T3
  if (issuer && elect_one()) {
    cp128<CG>(tm + 264, sdesc(w2 + 10 * 128 + 64));
    shift_down<CG>(tm + 264);
    cp4<CG>(tm + 264, sdesc(w2 + 9 * 128 + 64));
    mma_ts<CG>(tm + 192, tm + 264, sdesc(b0 + 64), idesc, 0);
    commit<CG>(&bar);
  }
  __syncwarp();
  step(5, 192);
  // T6: same with two slides (rows 11.. -> 10.. -> 9..)
  if (issuer && elect_one()) {
    cp128<CG>(tm + 272, sdesc(w2 + 11 * 128 + 64));
    shift_down<CG>(tm + 272);
    cp4<CG>(tm + 272, sdesc(w2 + 10 * 128 + 64));
    shift_down<CG>(tm + 272);
    cp4<CG>(tm + 272, sdesc(w2 + 9 * 128 + 64));
    mma_ts<CG>(tm + 320, tm + 272, sdesc(b0 + 64), idesc, 0);
    commit<CG>(&bar);
  }
  __syncwarp();
  step(6, 320);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair_sync<CG>();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  }
  (void)fout;
}

// ---------------------------------------------------------------------------- timing
// MODE 0: SS (A descriptors into a 256-row window, shifted by one row per K-step)
// MODE 1: TS (8 A blocks in TMEM; per K-step 8 x (shift + cp.4x256b), then the MMAs)
template <int MODE, int CG>
__global__ void __launch_bounds__(128, 1) kstep(unsigned long long *cyc, int n1, int n2, int steps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair_sync<CG>();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  // window hi at 0 (32 KB, 256 rows), lo at 32 KB; B hi at 64 KB, B lo at 96 KB (N <= 256 rows)
  const uint32_t whi = smem_u32(smem), wlo = whi + 32768, bb = whi + 65536;
  const uint32_t i1 = idesc_f16((uint32_t)n1, CG), i2 = n2 ? idesc_f16((uint32_t)n2, CG) : 0u;
  // TMEM: D1 cols [0, 256), A blocks cols [448, 512): hi_j at 448 + 8j, lo_j at 480 + 8j
  if (warp == 1 && rank == 0) {
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
      const int q = 64 - (s & 63);  // window row of this K-step (decreasing, like the TS slide)
      if (elect_one()) {
        if (MODE == 1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            shift_down<CG>(tm + 448 + 8 * j);
            cp4<CG>(tm + 448 + 8 * j, sdesc(whi + q * 128 + 32 * j));
            shift_down<CG>(tm + 480 + 8 * j);
            cp4<CG>(tm + 480 + 8 * j, sdesc(wlo + q * 128 + 32 * j));
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            mma_ts<CG>(tm + 0, tm + 448 + 8 * j, sdesc(bb + 32 * j), i1, 1);
            if (n2) mma_ts<CG>(tm + 0 + (uint32_t)n1, tm + 480 + 8 * j, sdesc(bb + 32768 + 32 * j), i2, 1);
          }
        } else {
          // MODE 2: the B operand walks through 64 KB of distinct tap tiles (like the bank)
          const uint32_t bw = MODE == 2 ? (uint32_t)(s % 8) * 8192u : 0u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            mma_ss<CG>(tm + 0, sdesc(whi + q * 128 + 32 * j), sdesc(bb + bw + 32 * j), i1, 1);
            if (n2) mma_ss<CG>(tm + 0 + (uint32_t)n1, sdesc(wlo + q * 128 + 32 * j), sdesc(bb + bw + 4096 + 32 * j), i2, 1);
          }
        }
      }
      __syncwarp();
    }
    if (elect_one()) commit<CG>(&bar);
    __syncwarp();
    mwait(&bar, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (CG == 2 && warp == 1) {
    mwait(&bar, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair_sync<CG>();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
  }
}

template <typename K, typename... Args>
static cudaError_t launch(K kern, int grid, int cg, size_t smem, Args... args) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cg;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) return e;
  return cudaDeviceSynchronize();
}

static void decode_lane(const uint32_t *w, char *buf) {
  // 16 halves of one lane -> "rank:row:k0..k15 ok?"
  uint16_t h[16];
  for (int i = 0; i < 8; ++i) { h[2 * i] = (uint16_t)(w[i] & 0xffff); h[2 * i + 1] = (uint16_t)(w[i] >> 16); }
  const int rk = h[0] >> 14, r = (h[0] >> 6) & 255, k0 = h[0] & 63;
  bool seq = true;
  for (int i = 1; i < 16; ++i) if (h[i] != (uint16_t)(h[0] + i)) seq = false;
  sprintf(buf, "cta%d row%3d k%2d%s", rk, r, k0, seq ? "" : " (non-seq)");
}

static int check_sem(int cg) {
  uint32_t *d;
  const size_t words = (size_t)2 * NT * 128 * 8;
  cudaMalloc(&d, words * 4);
  cudaMemset(d, 0xff, words * 4);
  cudaError_t e = cg == 2 ? launch(sem<2>, 2, 2, 96 * 1024 + 1024, d, (float *)nullptr)
                          : launch(sem<1>, 1, 1, 96 * 1024 + 1024, d, (float *)nullptr);
  if (e != cudaSuccess) { printf("sem cg%d: %s\n", cg, cudaGetErrorString(e)); return 1; }
  static uint32_t h[2 * NT * 128 * 8];
  cudaMemcpy(h, d, words * 4, cudaMemcpyDeviceToHost);
  const char *names[3] = {"cp128 rows5.. k16", "shift.down", "cp4 rows4..7"};
  for (int rk = 0; rk < cg; ++rk) {
    for (int t = 0; t < 3; ++t) {
      printf("cg%d cta%d T%d %-18s:", cg, rk, t, names[t]);
      for (int l : {0, 1, 2, 3, 4, 5, 31, 32, 127}) {
        char b[64];
        decode_lane(h + ((size_t)(rk * NT + t) * 128 + l) * 8, b);
        printf(" [%d]%s", l, b);
      }
      printf("\n");
    }
    // MMA checks: T3 (SS) vs T4 (TS) vs T5 (1 slide) vs T6 (2 slides), columns 0..7 of D
    for (int t = 4; t <= 6; ++t) {
      int bad = 0;
      for (int i = 0; i < 128 * 8; ++i)
        if (h[(size_t)(rk * NT + t) * 1024 + i] != h[(size_t)(rk * NT + 3) * 1024 + i]) ++bad;
      printf("cg%d cta%d T%d vs SS: %d of 1024 words differ\n", cg, rk, t, bad);
    }
    // host reference for T3 lanes 0..127, cols 0..7: D[m][n] = sum_k A[9+m][32+k] B[n][32+k]
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 8; ++n) {
        float acc = 0;
        for (int k = 0; k < 16; ++k) {
          const int r = 9 + m, kk = 32 + k;
          const float a = (float)(((r * 3 + kk * 5 + rk) % 7) - 3);
          const float b = (float)((((n + 0) * 5 + kk * 3 + 2 * (cg == 2 ? 0 : 0)) % 5) - 2);
          acc += a * b;
        }
        float got;
        memcpy(&got, &h[((size_t)(rk * NT + 3) * 128 + m) * 8 + n], 4);
        if (got != acc) ++bad;
      }
    printf("cg%d cta%d T3 vs host (B of CTA0, n < 8): %d of 1024 differ\n", cg, rk, bad);
  }
  cudaFree(d);
  return 0;
}

int main() {
  if (getenv("SEM")) {
    if (check_sem(1)) return 1;
    if (check_sem(2)) return 1;
  }
  int sms = 148;
  unsigned long long *d;
  cudaMalloc(&d, sizeof(unsigned long long) * sms);
  unsigned long long h[148];
  const int steps = 4000;
  const int cases[][2] = {{32, 16}, {64, 32}, {96, 48}, {128, 64}, {48, 0}, {160, 96}, {256, 128}};
  for (int cg : {1, 2}) {
    for (auto &c : cases) {
      double r[3];
      for (int mode = 0; mode < 3; ++mode) {
        cudaError_t e;
        const size_t sm = 160 * 1024 + 1024;
        if (cg == 1) e = mode == 1 ? launch(kstep<1, 1>, sms, 1, sm, d, c[0], c[1], steps) : mode == 2 ? launch(kstep<2, 1>, sms, 1, sm, d, c[0], c[1], steps) : launch(kstep<0, 1>, sms, 1, sm, d, c[0], c[1], steps);
        else e = mode == 1 ? launch(kstep<1, 2>, sms, 2, sm, d, c[0], c[1], steps) : mode == 2 ? launch(kstep<2, 2>, sms, 2, sm, d, c[0], c[1], steps) : launch(kstep<0, 2>, sms, 2, sm, d, c[0], c[1], steps);
        if (e != cudaSuccess) { printf("kstep: %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double s = 0; int n = 0;
        for (int i = 0; i < sms; i += cg) { s += h[i]; ++n; }
        r[mode] = s / n / steps;
      }
      printf("cg%d N1=%3d N2=%3d: SS %6.1f  SS B-walk %6.1f  TS+slide %6.1f cyc/K-step  (tensor ideal %5.1f)\n", cg, c[0], c[1],
             r[0], r[2], r[1], 4.0 * (c[0] + c[1]) / 2.0 * (cg == 2 ? 1.0 : 1.0));
    }
  }
  return 0;
}
