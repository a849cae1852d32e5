// wh_formats.cu -- the data formats either side of the hot path:
//   * decimation (signal_io.py:130-150): keep every hop-th sample from index 0, optionally
//     after the reference's anti-alias FIR (firwin(10*hop+1, 0.9/hop), Hamming window,
//     unit DC gain, "same"-centred linear convolution) -- feeds cwth_decimate
//     (wavelet.py:276-294) as a hop-1 transform of the decimated clips;
//   * render (scalogram.py:67-86): a real matrix mapped affinely onto [0, 255] with the
//     reference's f64 rounding (floor(v*255/(hi-lo) + 0.5), clip, constant -> 0), optional
//     vertical flip -- standalone (wh_render_u8) and fused behind a plan (WH_NORM_RENDER_U8).
#include <math.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "wh_internal.h"

namespace wh {

// ---- decimation --------------------------------------------------------------------------

// Plain selection: out[b][i] = x[b][i*hop], i < m = ceil(n / hop).
__global__ void k_decimate_select(const float *__restrict__ x, int64_t ld_x, int64_t hop, int64_t m,
                                  float *__restrict__ out, int64_t ld_out) {
    const int64_t b = blockIdx.y;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[b * ld_out + i] = x[b * ld_x + i * hop];
}

// FIR + selection: out[i] = sum_j x[i*hop + c - j] * h[j], c = (T-1)/2 (the "same" centre of
// fftconvolve), x = 0 outside [0, n).  One warp per output sample, lanes over the taps,
// float64 accumulation (the reference convolves in float64); the clip's samples are read
// coalesced in reverse.
__global__ void k_decimate_fir(const float *__restrict__ x, int64_t ld_x, int64_t n, int64_t hop, int64_t m,
                               const double *__restrict__ h, int64_t T, float *__restrict__ out, int64_t ld_out) {
    const int64_t b = blockIdx.y;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const float *xb = x + b * ld_x;
    const int64_t c = (T - 1) / 2;
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
        const int64_t top = i * hop + c;  // x index multiplied by h[0]
        // taps j with 0 <= top - j < n
        const int64_t j0 = top >= n ? top - n + 1 : 0;
        const int64_t j1 = top < T - 1 ? top : T - 1;
        double acc = 0.0;
        for (int64_t j = j0 + lane; j <= j1; j += 32) acc = fma((double)__ldg(xb + top - j), __ldg(h + j), acc);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) out[b * ld_out + i] = (float)acc;
    }
}

// scipy.signal.firwin(numtaps, cutoff) with its defaults (window "hamming", pass_zero,
// scale, cutoff relative to Nyquist) -- the published window-method design restated:
// h[n] = c * sinc(c * (n - a)), a = (T-1)/2, times the symmetric Hamming window
// 0.54 - 0.46 cos(2 pi n / (T-1)), then scaled to unit gain at DC.
static std::vector<double> firwin_lowpass(int64_t T, double cutoff) {
    std::vector<double> h((size_t)T);
    const double a = 0.5 * (double)(T - 1);
    double s = 0.0;
    for (int64_t k = 0; k < T; ++k) {
        const double mm = (double)k - a;
        const double xx = cutoff * mm;
        const double sinc = xx == 0.0 ? 1.0 : sin(M_PI * xx) / (M_PI * xx);
        const double w = T > 1 ? 0.54 - 0.46 * cos(2.0 * M_PI * (double)k / (double)(T - 1)) : 1.0;
        h[(size_t)k] = cutoff * sinc * w;
        s += h[(size_t)k];
    }
    for (auto &v : h) v /= s;
    return h;
}

int decimate_fir_taps(int64_t hop, std::vector<double> &h) {
    h = firwin_lowpass(10 * hop + 1, 0.9 / (double)hop);
    return WH_OK;
}

// ---- render ------------------------------------------------------------------------------

// Per-matrix min / max as order-preserving u32 keys (f2key), one matrix per blockIdx.y.
__global__ void k_render_minmax(const float *__restrict__ v, int64_t per, uint32_t *__restrict__ mm) {
    const int64_t b = blockIdx.y;
    float lo = INFINITY, hi = -INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
        const float t = v[b * per + i];
        lo = fminf(lo, t);
        hi = fmaxf(hi, t);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(mm + 2 * b, f2key(lo));
        atomicMax(mm + 2 * b + 1, f2key(hi));
    }
}

// scalogram.py:77-85 in float64 with explicit rounding (no FMA contraction, as numpy
// computes it): scaled = (v - lo) * (255 / (hi - lo)); pixel = clip(floor(scaled + 0.5));
// flip: image row r holds matrix row rows-1-r.
__global__ void k_render_apply(const float *__restrict__ v, int64_t rows, int64_t cols, const uint32_t *__restrict__ mm,
                               int32_t flip, uint8_t *__restrict__ out) {
    const int64_t b = blockIdx.y, per = rows * cols;
    const double lo = (double)key2f(mm[2 * b]), hi = (double)key2f(mm[2 * b + 1]);
    const bool constant = !(hi > lo);
    const double k = constant ? 0.0 : __ddiv_rn(255.0, __dsub_rn(hi, lo));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - r * cols;
        uint8_t px = 0;
        if (!constant) {
            const double s = __dmul_rn(__dsub_rn((double)v[b * per + i], lo), k);
            double q = floor(__dadd_rn(s, 0.5));
            q = q < 0.0 ? 0.0 : (q > 255.0 ? 255.0 : q);
            px = (uint8_t)q;
        }
        const int64_t ro = flip ? rows - 1 - r : r;
        out[b * per + ro * cols + c] = px;
    }
}

__global__ void k_keys_reset(uint32_t *mm, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        mm[2 * i] = 0xffffffffu;
        mm[2 * i + 1] = 0u;
    }
}

static unsigned blocks_for(int64_t work, int64_t per_block, unsigned cap) {
    return (unsigned)std::min<int64_t>(std::max<int64_t>((work + per_block - 1) / per_block, 1), cap);
}

int render_apply(const float *values, int64_t clips, int64_t rows, int64_t cols, const uint32_t *mm, int32_t flip,
                 uint8_t *out, cudaStream_t s) {
    const int64_t per = rows * cols;
    k_render_apply<<<dim3(blocks_for(per, 1024, 128), (unsigned)clips), 256, 0, s>>>(values, rows, cols, mm, flip, out);
    WH_CUDA_TRY(cudaGetLastError());
    return WH_OK;
}

}  // namespace wh

using namespace wh;

extern "C" int wh_decimate(int device, const float *x_dev, int64_t clips, int64_t n_samples, int64_t ld_x,
                           int64_t hop, int32_t anti_alias, float *out_dev, int64_t ld_out, void *stream) {
    if (hop < 1) return fail(WH_E_INVALID_HOP, "hop must be an integer >= 1");
    if (n_samples < 1) return fail(WH_E_EMPTY_SIGNAL, "signal has no samples");
    if (clips < 0 || ld_x < n_samples) return fail(WH_E_INVALID_ARG, "bad clips / ld_x");
    const int64_t m = (n_samples + hop - 1) / hop;
    if (ld_out < m) return fail(WH_E_INVALID_ARG, "ld_out < ceil(n_samples / hop)");
    if (clips == 0) return WH_OK;
    if (!x_dev || !out_dev) return fail(WH_E_INVALID_ARG, "NULL buffer");
    if (clips > 65535) return fail(WH_E_INVALID_ARG, "at most 65535 clips per call");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != device) WH_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = WH_OK;
    (void)cudaGetLastError();
    if (!anti_alias) {
        k_decimate_select<<<dim3(blocks_for(m, 256, 1024), (unsigned)clips), 256, 0, s>>>(x_dev, ld_x, hop, m, out_dev,
                                                                                            ld_out);
        if (cudaGetLastError() != cudaSuccess) rc = fail(WH_E_CUDA, "decimate launch failed");
    } else {
        std::vector<double> h;
        decimate_fir_taps(hop, h);
        double *d_h = nullptr;
        if (cudaMallocAsync(&d_h, sizeof(double) * h.size(), s) != cudaSuccess) {
            rc = fail(WH_E_OOM, "cudaMallocAsync(fir taps) failed");
        } else {
            if (cudaMemcpyAsync(d_h, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
                rc = fail(WH_E_CUDA, "fir taps upload failed");
            if (rc == WH_OK) {
                k_decimate_fir<<<dim3(blocks_for(m, 8, 1024), (unsigned)clips), 256, 0, s>>>(
                    x_dev, ld_x, n_samples, hop, m, d_h, (int64_t)h.size(), out_dev, ld_out);
                if (cudaGetLastError() != cudaSuccess) rc = fail(WH_E_CUDA, "decimate launch failed");
            }
            // stream-ordered free after the kernel; the pageable source vector may die on
            // return (cudaMemcpyAsync stages pageable memory before returning)
            cudaFreeAsync(d_h, s);
        }
    }
    if (prev != device) cudaSetDevice(prev);
    return rc;
}

extern "C" int wh_render_u8(int device, const float *values_dev, int64_t count, int64_t rows, int64_t cols,
                            int32_t flip_vertical, uint8_t *out_dev, void *stream) {
    if (rows < 1 || cols < 1) return fail(WH_E_INVALID_ARG, "values must be a non-empty 2-D matrix");
    if (count < 0 || count > 65535) return fail(WH_E_INVALID_ARG, "count out of range [0, 65535]");
    if (count == 0) return WH_OK;
    if (!values_dev || !out_dev) return fail(WH_E_INVALID_ARG, "NULL buffer");
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != device) WH_CUDA_TRY(cudaSetDevice(device));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int rc = WH_OK;
    (void)cudaGetLastError();
    uint32_t *mm = nullptr;
    if (cudaMallocAsync(&mm, sizeof(uint32_t) * 2 * count, s) != cudaSuccess) {
        rc = fail(WH_E_OOM, "cudaMallocAsync(min/max) failed");
    } else {
        const int64_t per = rows * cols;
        k_keys_reset<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(mm, count);
        k_render_minmax<<<dim3(blocks_for(per, 2048, 128), (unsigned)count), 256, 0, s>>>(values_dev, per, mm);
        if (cudaGetLastError() != cudaSuccess) rc = fail(WH_E_CUDA, "render min/max launch failed");
        if (rc == WH_OK) rc = render_apply(values_dev, count, rows, cols, mm, flip_vertical, out_dev, s);
        cudaFreeAsync(mm, s);
    }
    if (prev != device) cudaSetDevice(prev);
    return rc;
}
