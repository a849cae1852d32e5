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
#include <map>
#include <mutex>
#include <utility>
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

// Same sum for hop <= 128 from shared memory: a block produces FIR_TO consecutive outputs
// of one clip; the clip segment they need ((FIR_TO-1)*hop + T samples) and the taps are
// staged once, then each warp reduces one output at a time (lanes over the taps:
// consecutive lanes read consecutive samples -- conflict-free).
constexpr int FIR_TO = 128;
__global__ void k_decimate_fir_smem(const float *__restrict__ x, int64_t ld_x, int64_t n, int64_t hop, int64_t m,
                                    const double *__restrict__ h, int T, float *__restrict__ out, int64_t ld_out) {
    extern __shared__ double fir_sm[];
    double *hs = fir_sm;                                    // T taps
    float *xs = reinterpret_cast<float *>(fir_sm + T);     // segment
    const int64_t b = blockIdx.y;
    const int64_t i0 = (int64_t)blockIdx.x * FIR_TO;
    const int nout = (int)(m - i0 < FIR_TO ? m - i0 : FIR_TO);
    const int64_t c = (T - 1) / 2;
    const int64_t s0 = i0 * hop + c - (T - 1);  // first sample of the segment
    const int seg = (int)((int64_t)(nout - 1) * hop + T);
    const float *xb = x + b * ld_x;
    for (int k = threadIdx.x; k < T; k += blockDim.x) hs[k] = h[k];
    for (int k = threadIdx.x; k < seg; k += blockDim.x) {
        const int64_t g = s0 + k;
        xs[k] = (g >= 0 && g < n) ? __ldg(xb + g) : 0.0f;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = warp; o < nout; o += nw) {
        const int top = (int)((int64_t)o * hop + (T - 1));  // segment index multiplied by h[0]
        double acc = 0.0;
        for (int j = lane; j < T; j += 32) acc = fma((double)xs[top - j], hs[j], acc);
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) out[b * ld_out + i0 + o] = (float)acc;
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

// Device copies of the FIR taps, built once per (device, hop) and kept for the process
// lifetime (a few KB each): the decimation call stays stream-ordered with no per-call
// allocation or upload.
static std::mutex g_fir_mu;
static std::map<std::pair<int, int64_t>, const double *> g_fir_taps;

static int device_fir_taps(int device, int64_t hop, const double **taps, int *T) {
    *T = (int)(10 * hop + 1);
    std::lock_guard<std::mutex> lk(g_fir_mu);
    auto it = g_fir_taps.find({device, hop});
    if (it != g_fir_taps.end()) {
        *taps = it->second;
        return WH_OK;
    }
    const std::vector<double> h = firwin_lowpass(10 * hop + 1, 0.9 / (double)hop);
    double *d = nullptr;
    if (cudaMalloc(&d, sizeof(double) * h.size()) != cudaSuccess) return fail(WH_E_OOM, "cudaMalloc(fir taps) failed");
    if (cudaMemcpy(d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return fail(WH_E_CUDA, "fir taps upload failed");
    }
    g_fir_taps[{device, hop}] = d;
    *taps = d;
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
// One pixel.  float32 first: |s32 - s64| <= 255 * 3 * 2^-24 < 5e-5, so when s32 + 0.5 is
// more than 1e-4 away from an integer both floors agree; otherwise (rare) redo it in
// float64 exactly as numpy orders it.
__device__ __forceinline__ uint32_t render_px(float v, float lo32, float k32, double lo, double k) {
    const float t = __fadd_rn(__fmul_rn(__fsub_rn(v, lo32), k32), 0.5f);
    float q = floorf(t);
    const float fr = t - q;
    if (fr < 1e-4f || fr > 1.0f - 1e-4f) {
        const double s = __dmul_rn(__dsub_rn((double)v, lo), k);
        q = (float)floor(__dadd_rn(s, 0.5));
    }
    q = q < 0.0f ? 0.0f : (q > 255.0f ? 255.0f : q);
    return (uint32_t)q;
}
// Each block maps RENDER_RPB consecutive matrix rows (of any matrices), 4 pixels per
// thread-iteration when the row allows; long-lived blocks (a flat grid of row strips), not
// one tiny block per row.
constexpr int RENDER_RPB = 8;
struct RenderParams {
    double lo, k;      // k = 255 / (hi - lo) in float64, 0 for a constant matrix
    float lo32, k32;
};
// per matrix, once: the min/max keys -> the affine map (the float64 division runs once)
__global__ void k_render_params(const uint32_t *__restrict__ mm, int64_t count, RenderParams *__restrict__ rp) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= count) return;
    const double lo = (double)key2f(mm[2 * b]), hi = (double)key2f(mm[2 * b + 1]);
    const double k = hi > lo ? __ddiv_rn(255.0, __dsub_rn(hi, lo)) : 0.0;
    rp[b] = RenderParams{lo, k, (float)lo, (float)k};
}
__global__ void k_render_apply(const float *__restrict__ v, int64_t rows, int64_t cols, int64_t count,
                               const RenderParams *__restrict__ rp, int32_t flip, uint8_t *__restrict__ out) {
    const int64_t per = rows * cols, total = count * rows;
    for (int64_t gr = (int64_t)blockIdx.x * RENDER_RPB; gr < (int64_t)(blockIdx.x + 1) * RENDER_RPB && gr < total; ++gr) {
        const int64_t b = gr / rows, r = gr - b * rows;
        const RenderParams P = rp[b];
        const bool constant = P.k == 0.0;
        const float *src = v + gr * cols;
        uint8_t *dst = out + b * per + (flip ? rows - 1 - r : r) * cols;
        const bool vec = (cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                         ((reinterpret_cast<uintptr_t>(dst) & 3) == 0);
        if (vec) {
            for (int64_t i = threadIdx.x; i < cols / 4; i += blockDim.x) {
                const float4 t = reinterpret_cast<const float4 *>(src)[i];
                uint32_t w = 0;
                if (!constant)
                    w = render_px(t.x, P.lo32, P.k32, P.lo, P.k) | (render_px(t.y, P.lo32, P.k32, P.lo, P.k) << 8) |
                        (render_px(t.z, P.lo32, P.k32, P.lo, P.k) << 16) | (render_px(t.w, P.lo32, P.k32, P.lo, P.k) << 24);
                reinterpret_cast<uint32_t *>(dst)[i] = w;
            }
        } else {
            for (int64_t i = threadIdx.x; i < cols; i += blockDim.x)
                dst[i] = constant ? (uint8_t)0 : (uint8_t)render_px(src[i], P.lo32, P.k32, P.lo, P.k);
        }
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

static_assert(sizeof(RenderParams) == WH_RENDER_PARAM_BYTES, "render parameter block size");

// params: RENDER_PARAM_BYTES per matrix of workspace (device), filled here
int render_apply(const float *values, int64_t clips, int64_t rows, int64_t cols, const uint32_t *mm, void *params,
                 int32_t flip, uint8_t *out, cudaStream_t s) {
    const int64_t strips = (clips * rows + RENDER_RPB - 1) / RENDER_RPB;
    if (strips > 0x7fffffff) return fail(WH_E_INVALID_ARG, "render: too many rows");
    RenderParams *rp = static_cast<RenderParams *>(params);
    k_render_params<<<(unsigned)((clips + 127) / 128), 128, 0, s>>>(mm, clips, rp);
    k_render_apply<<<(unsigned)strips, 256, 0, s>>>(values, rows, cols, clips, rp, flip, out);
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
        const double *d_h = nullptr;
        int T = 0;
        rc = device_fir_taps(device, hop, &d_h, &T);
        if (rc == WH_OK) {
            const size_t smem = sizeof(double) * T + sizeof(float) * ((size_t)(FIR_TO - 1) * hop + T);
            if (hop <= 128 && smem <= 96 * 1024) {
                cudaFuncSetAttribute(k_decimate_fir_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
                k_decimate_fir_smem<<<dim3((unsigned)((m + FIR_TO - 1) / FIR_TO), (unsigned)clips), 512, smem, s>>>(
                    x_dev, ld_x, n_samples, hop, m, d_h, T, out_dev, ld_out);
            } else {
                k_decimate_fir<<<dim3(blocks_for(m, 8, 1024), (unsigned)clips), 256, 0, s>>>(
                    x_dev, ld_x, n_samples, hop, m, d_h, (int64_t)T, out_dev, ld_out);
            }
            if (cudaGetLastError() != cudaSuccess) rc = fail(WH_E_CUDA, "decimate launch failed");
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
    if (cudaMallocAsync(&mm, (sizeof(uint32_t) * 2 + sizeof(RenderParams)) * count, s) != cudaSuccess) {
        rc = fail(WH_E_OOM, "cudaMallocAsync(min/max) failed");
    } else {
        const int64_t per = rows * cols;
        k_keys_reset<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(mm, count);
        k_render_minmax<<<dim3(blocks_for(per, 2048, 128), (unsigned)count), 256, 0, s>>>(values_dev, per, mm);
        if (cudaGetLastError() != cudaSuccess) rc = fail(WH_E_CUDA, "render min/max launch failed");
        if (rc == WH_OK)
            rc = render_apply(values_dev, count, rows, cols, mm, reinterpret_cast<uint8_t *>(mm) + 8 * count,
                              flip_vertical, out_dev, s);
        cudaFreeAsync(mm, s);
    }
    if (prev != device) cudaSetDevice(prev);
    return rc;
}
