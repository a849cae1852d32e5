// Experiment: L2 flush kernels with different shared-memory carveouts (does the carveout
// reconfiguration between the flush and k_umma show up in the measured kernel time?)
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_fill(uint4 *p, size_t n, uint32_t v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, v, v, v);
}
extern "C" int flush_fill(void *p, size_t bytes, uint32_t v, int carveout, void *stream) {
    static int last = -2;
    if (carveout != last) {
        cudaFuncSetAttribute(k_fill, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
        last = carveout;
    }
    k_fill<<<148 * 8, 256, 0, (cudaStream_t)stream>>>((uint4 *)p, bytes / 16, v);
    return (int)cudaGetLastError();
}
