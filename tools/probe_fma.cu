// Micro-probe: FP32 FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fmaf(r[i], a, b);
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b, int iters) {
  unsigned long long r[8];
  for (int i = 0; i < 8; ++i) { float lo = threadIdx.x * 0.001f + i, hi = lo + 1; r[i] = ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo); }
  unsigned long long av = ((unsigned long long)__float_as_uint(a) << 32) | __float_as_uint(a);
  unsigned long long bv = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(r[i]) : "l"(av), "l"(bv));
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += __uint_as_float((unsigned)r[i]) + __uint_as_float((unsigned)(r[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d L2 %d clockrate_khz %d\n", sms, l2, clk);
  float* d; cudaMalloc(&d, sms * 8 * 256 * sizeof(float));
  int iters = 20000; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma<<<sms * 8, 256>>>(d, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)sms * 8 * 256;
    printf("ffma : %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    cudaEventRecord(e0); k_ffma2<<<sms * 8, 256>>>(d, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ffma2: %.3f ms  %.1f TFLOP/s\n", ms, fl / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
