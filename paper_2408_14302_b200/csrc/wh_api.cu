// wh_api.cu -- C ABI of libwavehop_b200: validation, plans, the on-device filter-bank
// builder, per-clip min-max normalisation and the seam-2 kernels.
//
// Reference behaviour mirrored here (paths relative to /root/reference/pkg/src/wavehop):
//   MorletParams validation   wavelet.py:47-53
//   ScaleGrid validation      wavelet.py:62-69
//   InvalidScale              wavelet.py:151-152
//   InvalidHop / _check_hop   signal_io.py:153-156
//   frames = ceil(n / hop)    wavelet.py:238
//   half width L              wavelet.py:154
//   taps                      wavelet.py:155-159
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <thread>
#include <vector>
#include <string>

#include "wh_internal.h"

namespace wh {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
    set_error(msg);
    (void)cudaGetLastError();  // do not leak a non-sticky CUDA error into later calls
    return code;
}

int64_t out_elem_bytes(const Plan &p) {
    if (p.norm == WH_NORM_RENDER_U8 || p.norm == WH_NORM_RENDER_U8_NOFLIP) return 1;
    return p.output == WH_OUT_COMPLEX64 ? 8 : 4;
}

// ---------------------------------------------------------------------------------------
// Filter bank: fp64 sampling of the conjugated, 1/sqrt(a)-normalised Morlet exactly as
// wavelet.py:154-159 orders it, folded (taps[L:]) and rounded to fp32.
__global__ void k_fold_bank(const double *scales, const int64_t *half, const int64_t *off,
                            int32_t S, double C, double Bw, float *fold, int64_t total) {
    int32_t s = blockIdx.y;
    if (s >= S) return;
    double a = scales[s];
    int64_t L = half[s];
    double norm = pow(M_PI * Bw, -0.5);
    double w = 2.0 * M_PI * C;
    double rs = sqrt(a);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= L;
         j += (int64_t)gridDim.x * blockDim.x) {
        double t = (double)j / a;
        double env = norm * exp(-(t * t) / Bw);
        double th = w * t;
        fold[off[s] + j] = (float)((env * cos(th)) / rs);
        fold[total + off[s] + j] = (float)((env * sin(th)) / rs);
    }
}

int build_fold_bank(Plan &p) {
    p.fold_off.resize(p.S);
    int64_t tot = 0;
    for (int s = 0; s < p.S; ++s) {
        p.fold_off[s] = tot;
        tot += p.half[s] + 1;
    }
    p.fold_total = tot;
    WH_CUDA_TRY(cudaMalloc(&p.d_fold, sizeof(float) * 2 * tot));
    WH_CUDA_TRY(cudaMalloc(&p.d_scales, sizeof(double) * p.S));
    WH_CUDA_TRY(cudaMalloc(&p.d_half, sizeof(int64_t) * p.S));
    WH_CUDA_TRY(cudaMalloc(&p.d_fold_off, sizeof(int64_t) * p.S));
    WH_CUDA_TRY(cudaMemcpy(p.d_scales, p.scales.data(), sizeof(double) * p.S, cudaMemcpyHostToDevice));
    WH_CUDA_TRY(cudaMemcpy(p.d_half, p.half.data(), sizeof(int64_t) * p.S, cudaMemcpyHostToDevice));
    WH_CUDA_TRY(cudaMemcpy(p.d_fold_off, p.fold_off.data(), sizeof(int64_t) * p.S, cudaMemcpyHostToDevice));
    dim3 grid((unsigned)std::min<int64_t>((p.Lmax + 256) / 256, 64), p.S);
    k_fold_bank<<<grid, 256>>>(p.d_scales, p.d_half, p.d_fold_off, p.S, p.C, p.B, p.d_fold, tot);
    WH_CUDA_TRY(cudaGetLastError());
    WH_CUDA_TRY(cudaDeviceSynchronize());
    return WH_OK;
}

__device__ __forceinline__ unsigned long long globaltimer_ns_api() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------------------
// Per-clip min-max (scalogram.py:77-83 affine map, without x255/round/uint8).
__global__ void k_minmax_reset(uint32_t *mm, uint32_t *arrive, uint32_t *abandon, int32_t ab_words, int64_t clips) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < clips) {
        mm[2 * i] = 0xffffffffu;  // min key
        mm[2 * i + 1] = 0u;       // max key
        if (arrive) {
            arrive[i] = 0u;
            for (int w = 0; w < ab_words; ++w) abandon[i * ab_words + w] = 0u;
        }
    }
}

__global__ void k_minmax_apply(float *out, const uint32_t *mm, int64_t per_clip, int vec, const uint32_t *done) {
    int64_t b = blockIdx.y;
    if (done && done[b] == WH_CLIP_NORMALISED) return;  // the concurrent normaliser did this clip
    float lo = key2f(mm[2 * b]), hi = key2f(mm[2 * b + 1]);
    bool constant = (hi == lo);
    float sc = constant ? 0.0f : 1.0f / (hi - lo);
    float *base = out + b * per_clip;
    int64_t n4 = vec ? per_clip / 4 : 0;
    float4 *o = reinterpret_cast<float4 *>(base);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
        float4 v = o[i];
        if (constant) {
            v = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            v.x = (v.x - lo) * sc; v.y = (v.y - lo) * sc; v.z = (v.z - lo) * sc; v.w = (v.w - lo) * sc;
        }
        o[i] = v;
    }
    for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_clip;
         i += (int64_t)gridDim.x * blockDim.x)
        base[i] = constant ? 0.0f : (base[i] - lo) * sc;
}

// Concurrent per-clip min-max (mode 2): a few CTAs on SMs of their own, running beside
// k_umma, normalise each clip as soon as all its units have arrived (arrive[b] reaches
// `target`; the epilogue's release-add follows its stores and key atomics) -- the clip's
// raw values were written a round or two earlier and are read back mostly from L2, so the
// read-modify-write overlaps the tensor-bound kernel instead of following it.  Bounded waits:
// once one wait times out (k_umma not running beside it), every CTA stops waiting and the
// rest is left to the trailing masked pass, as are clips with non-finite samples (their
// values are final only after k_umma's fix-up).  A finished clip is marked
// WH_CLIP_NORMALISED for that pass.
__global__ void __launch_bounds__(1024, 1) k_minmax_stream(float *out, const uint32_t *mm, uint32_t *arrive,
                                                           const uint32_t *nfbad, int64_t per_clip, int64_t clips,
                                                           uint32_t target, int vec, uint32_t *giveup) {
    __shared__ int s_go;
    const int tid = threadIdx.x;
    for (int64_t b = blockIdx.x; b < clips; b += gridDim.x) {
        if (tid == 0) {
            int go = 0;
            const unsigned long long t0 = globaltimer_ns_api();
            while (true) {
                uint32_t c;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(arrive + b) : "memory");
                if (c >= target) { go = 1; break; }
                if (*reinterpret_cast<volatile uint32_t *>(giveup)) break;
                if (globaltimer_ns_api() - t0 > 50000000ull) {  // 50 ms: k_umma is not running beside us
                    atomicExch(giveup, 1u);
                    break;
                }
                __nanosleep(256);
            }
            if (go && nfbad[b * (int64_t)(1 + WH_NF_CAP)] != 0) go = 0;
            s_go = go;
        }
        __syncthreads();
        const int go = s_go;
        __syncthreads();
        if (!go) continue;
        const float lo = key2f(__ldcg(mm + 2 * b)), hi = key2f(__ldcg(mm + 2 * b + 1));
        const bool constant = hi == lo;
        const float sc = constant ? 0.0f : 1.0f / (hi - lo);
        float *base = out + b * per_clip;
        const int64_t n4 = vec ? per_clip / 4 : 0;
        float4 *o = reinterpret_cast<float4 *>(base);
        constexpr int U = 8;
        for (int64_t i0 = tid; i0 < n4; i0 += (int64_t)U * 1024) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + (int64_t)u * 1024;
                if (i < n4) v[u] = __ldcg(o + i);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + (int64_t)u * 1024;
                if (i >= n4) continue;
                float4 w = v[u];
                if (constant) {
                    w = make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
                    w.x = (w.x - lo) * sc; w.y = (w.y - lo) * sc; w.z = (w.z - lo) * sc; w.w = (w.w - lo) * sc;
                }
                o[i] = w;
            }
        }
        for (int64_t i = n4 * 4 + tid; i < per_clip; i += 1024)
            base[i] = constant ? 0.0f : (__ldcg(base + i) - lo) * sc;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            arrive[b] = WH_CLIP_NORMALISED;
        }
    }
}

// ---------------------------------------------------------------------------------------
// Non-finite input samples (SIMT engine): the exact values of the coefficients they reach
// (nf_fixup_clip); a block per clip, exiting at once for clips without any.
__global__ void k_nf_fixup(NfArgs a, int64_t clips) {
    for (int64_t b = blockIdx.x; b < clips; b += gridDim.x) nf_fixup_clip(a, b, threadIdx.x, blockDim.x);
}

int nf_fixup_launch(Plan &p, const float *x, int64_t clips, int64_t ld_x, void *out, uint32_t *mm, uint32_t *bad,
                    cudaStream_t s) {
    NfArgs a{};
    a.x = x; a.ld_x = ld_x; a.N = p.N; a.hop = p.hop; a.F = p.F; a.S = p.S;
    a.wavelet = p.wavelet; a.output = p.output; a.scales = p.d_scales; a.half = p.d_half;
    a.C = p.C; a.Bw = p.B; a.out = out; a.mm = mm; a.bad = bad;
    k_nf_fixup<<<(unsigned)std::min<int64_t>(clips, 4 * (int64_t)p.sms), 128, 0, s>>>(a, clips);
    WH_CUDA_TRY(cudaGetLastError());
    return WH_OK;
}

int minmax_reset(Plan &p, int64_t clips, uint32_t *mm, uint32_t *arrive, uint32_t *abandon, cudaStream_t s) {
    k_minmax_reset<<<(unsigned)((clips + 255) / 256), 256, 0, s>>>(mm, arrive, abandon, p.ab_words, clips);
    WH_CUDA_TRY(cudaGetLastError());
    return WH_OK;
}

int minmax_apply(Plan &p, int64_t clips, void *out, uint32_t *mm, cudaStream_t s, const uint32_t *done) {
    int64_t per_clip = (int64_t)p.S * p.F;
    int vec = (per_clip % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    int64_t work = vec ? per_clip / 4 : per_clip;
    unsigned bx = (unsigned)std::min<int64_t>(std::max<int64_t>((work + 1023) / 1024, 1), 64);
    k_minmax_apply<<<dim3(bx, (unsigned)clips), 256, 0, s>>>((float *)out, mm, per_clip, vec, done);
    WH_CUDA_TRY(cudaGetLastError());
    return WH_OK;
}

int minmax_stream_launch(Plan &p, int64_t clips, void *out, uint32_t *mm, uint32_t *arrive, const uint32_t *nfbad,
                         uint32_t target, cudaStream_t s) {
    const int64_t per_clip = (int64_t)p.S * p.F;
    const int vec = (per_clip % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    // clusters of 2: the normaliser takes whole SM pairs, so the kernel's CTA pairs still fit
    // in the rest
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.norm_ctas);
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    uint32_t *giveup = arrive + p.max_clips;  // one word after the arrival counters
    WH_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_minmax_stream, static_cast<float *>(out), static_cast<const uint32_t *>(mm),
                                   arrive, nfbad, per_clip, clips, target, vec, giveup));
    WH_CUDA_TRY(cudaGetLastError());
    return WH_OK;
}

// ---------------------------------------------------------------------------------------
// Seam 2: _kernels.py:76-91 and 93-112 on the device in float64 (one thread per frame).
__global__ void k_strided_generic(const double *xpad, const double *tr, const double *ti,
                                  int64_t width, int64_t hop, int64_t frames, double *ore,
                                  double *oim) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= frames) return;
    const double *w = xpad + k * hop;
    double ar = 0.0, ai = 0.0;
    for (int64_t j = 0; j < width; ++j) {
        ar = fma(w[j], tr[j], ar);
        ai = fma(w[j], ti[j], ai);
    }
    ore[k] = ar;
    oim[k] = ai;
}

__global__ void k_strided_symmetric(const double *xpad, const double *rh, const double *ih,
                                    int64_t half, int64_t hop, int64_t frames, double *ore,
                                    double *oim) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= frames) return;
    int64_t c = k * hop + half;
    double ar = xpad[c] * rh[0], ai = 0.0;
    for (int64_t j = 1; j <= half; ++j) {
        double r = xpad[c + j], l = xpad[c - j];
        ar = fma(r + l, rh[j], ar);
        ai = fma(r - l, ih[j], ai);
    }
    ore[k] = ar;
    oim[k] = ai;
}

}  // namespace wh

using namespace wh;

// =======================================================================================
// C ABI
// =======================================================================================
extern "C" {

int wh_abi_version(void) { return WH_ABI_VERSION; }

const char *wh_last_error(void) { return g_last_error.c_str(); }

int wh_half_width(double scale, double bandwidth, double support_radius, int64_t *half) {
    if (!(scale > 0 && std::isfinite(scale)))
        return fail(WH_E_INVALID_SCALE, "scale must be positive and finite");
    if (!half) return fail(WH_E_INVALID_ARG, "half is NULL");
    *half = (int64_t)std::ceil(support_radius * scale * std::sqrt(bandwidth / 2.0));
    return WH_OK;
}

int wh_frame_count(int64_t n_samples, int64_t hop, int64_t *frames) {
    if (hop < 1) return fail(WH_E_INVALID_HOP, "hop must be an integer >= 1");
    if (n_samples < 1) return fail(WH_E_EMPTY_SIGNAL, "signal has no samples");
    if (!frames) return fail(WH_E_INVALID_ARG, "frames is NULL");
    *frames = (n_samples + hop - 1) / hop;
    return WH_OK;
}

static void plan_free(Plan *p) {
    if (!p) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(p->device);
    cudaFree(p->d_fold); cudaFree(p->d_scales); cudaFree(p->d_half); cudaFree(p->d_fold_off);
    cudaFree(p->d_groups); cudaFree(p->d_items); cudaFree(p->d_group_taps);
    cudaFree(p->d_passes); cudaFree(p->d_tiles); cudaFree(p->d_groups_u); cudaFree(p->d_bank); cudaFree(p->d_scale_pow); cudaFree(p->d_tables);
    cudaFree(p->d_minmax); cudaFree(p->d_nfbad); cudaFree(p->d_nfctl); cudaFree(p->d_arrive); cudaFree(p->d_abandon); cudaFree(p->d_scratch); cudaFree(p->d_rparams); cudaFree(p->d_x); cudaFree(p->d_out); cudaFree(p->d_prof); cudaFree(p->d_trace);
    if (p->stream) cudaStreamDestroy(p->stream);
    if (p->stream2) cudaStreamDestroy(p->stream2);
    if (p->nstream) cudaStreamDestroy(p->nstream);
    if (p->nev0) cudaEventDestroy(p->nev0);
    if (p->nev1) cudaEventDestroy(p->nev1);
    if (p->h_stage) cudaFreeHost(p->h_stage);
    for (int i = 0; i < 2; ++i) {
        if (p->ev_h2d[i]) cudaEventDestroy(p->ev_h2d[i]);
        if (p->ev_d2h[i]) cudaEventDestroy(p->ev_d2h[i]);
    }
    cudaSetDevice(cur);
    delete p;
}

int wh_plan_create(wh_plan **plan, int device, const double *scales, int32_t n_scales,
                   double center_frequency, double bandwidth, double support_radius,
                   int32_t wavelet, int64_t hop, int64_t n_samples, int64_t max_clips,
                   int32_t output, int32_t norm, int32_t engine) {
    if (!plan) return fail(WH_E_INVALID_ARG, "plan is NULL");
    *plan = nullptr;
    // MorletParams (wavelet.py:47-53)
    if (!(center_frequency > 0)) return fail(WH_E_INVALID_ARG, "center_frequency must be positive");
    if (!(bandwidth > 0)) return fail(WH_E_INVALID_ARG, "bandwidth must be positive");
    if (!(support_radius >= 3)) return fail(WH_E_INVALID_ARG, "support_radius must be at least 3");
    // ScaleGrid (wavelet.py:62-69) then sample_wavelet's InvalidScale (151-152)
    if (!scales || n_scales < 1) return fail(WH_E_INVALID_ARG, "scales must be a non-empty 1-D sequence");
    for (int i = 0; i < n_scales; ++i)
        if (!(scales[i] > 0 && std::isfinite(scales[i])))
            return fail(WH_E_INVALID_SCALE, "scale must be positive and finite");
    for (int i = 1; i < n_scales; ++i)
        if (!(scales[i] > scales[i - 1])) return fail(WH_E_INVALID_ARG, "scales must be strictly ascending");
    if (hop < 1) return fail(WH_E_INVALID_HOP, "hop must be an integer >= 1");
    if (n_samples < 1) return fail(WH_E_EMPTY_SIGNAL, "signal has no samples");
    if (max_clips < 1) return fail(WH_E_INVALID_ARG, "max_clips must be >= 1");
    if (wavelet != WH_WAVELET_CMOR && wavelet != WH_WAVELET_RMOR)
        return fail(WH_E_INVALID_ARG, "unknown wavelet");
    if (output < WH_OUT_COMPLEX64 || output > WH_OUT_LOG1P) return fail(WH_E_INVALID_ARG, "unknown output");
    if (norm < WH_NORM_NONE || norm > WH_NORM_RENDER_U8_NOFLIP) return fail(WH_E_INVALID_ARG, "unknown norm");
    if (norm != WH_NORM_NONE && output == WH_OUT_COMPLEX64)
        return fail(WH_E_INVALID_ARG, "min-max / render normalisation needs a real output");
    if (engine < WH_ENGINE_AUTO || engine > WH_ENGINE_UMMA) return fail(WH_E_INVALID_ARG, "unknown engine");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(WH_E_NO_DEVICE, "no CUDA device is visible");
    if (device < 0 || device >= ndev) return fail(WH_E_NO_DEVICE, "device index out of range");
    int prev = 0;
    cudaGetDevice(&prev);
    WH_CUDA_TRY(cudaSetDevice(device));
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major != 10) {
        cudaSetDevice(prev);
        return fail(WH_E_UNSUPPORTED, "libwavehop_b200 is built for sm_100a (B200) only");
    }

    Plan *p = new Plan();
    p->device = device;
    cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
    p->S = n_scales;
    p->scales.assign(scales, scales + n_scales);
    p->half.resize(n_scales);
    p->Lmax = 0;
    for (int i = 0; i < n_scales; ++i) {
        wh_half_width(scales[i], bandwidth, support_radius, &p->half[i]);
        p->Lmax = std::max(p->Lmax, p->half[i]);
    }
    p->C = center_frequency; p->B = bandwidth; p->R = support_radius;
    p->wavelet = wavelet; p->hop = hop; p->N = n_samples; p->F = (n_samples + hop - 1) / hop;
    p->max_clips = max_clips; p->output = output; p->norm = norm;

    int rc = build_fold_bank(*p);
    if (rc == WH_OK) {  // non-finite sample records, zeroed once (each fix-up resets what it used)
        const size_t nb = sizeof(uint32_t) * (size_t)max_clips * (1 + WH_NF_CAP), nc = sizeof(uint32_t) * 2 * (size_t)max_clips;
        if (cudaMalloc(&p->d_nfbad, nb) != cudaSuccess || cudaMalloc(&p->d_nfctl, nc) != cudaSuccess ||
            cudaMemset(p->d_nfbad, 0, nb) != cudaSuccess || cudaMemset(p->d_nfctl, 0, nc) != cudaSuccess)
            rc = fail(WH_E_OOM, "cudaMalloc(non-finite records) failed");
    }
    if (rc == WH_OK && norm != WH_NORM_NONE) {
        if (cudaMalloc(&p->d_minmax, sizeof(uint32_t) * 2 * max_clips) != cudaSuccess)
            rc = fail(WH_E_OOM, "cudaMalloc(minmax) failed");
    }
    if (rc == WH_OK && is_render(*p)) {  // float values before the uint8 map + map parameters
        if (cudaMalloc(&p->d_scratch, sizeof(float) * (size_t)max_clips * n_scales * p->F) != cudaSuccess ||
            cudaMalloc(&p->d_rparams, (size_t)WH_RENDER_PARAM_BYTES * max_clips) != cudaSuccess)
            rc = fail(WH_E_OOM, "cudaMalloc(render workspace) failed");
    }
    std::string why;
    if (rc == WH_OK) {
        const bool umma_ok = umma_supported(*p, &why) == WH_OK;
        if (engine == WH_ENGINE_UMMA && !umma_ok) {
            rc = fail(WH_E_UNSUPPORTED, "UMMA engine unsupported for this plan: " + why);
        } else if (engine == WH_ENGINE_SIMT || !umma_ok) {
            p->engine = WH_ENGINE_SIMT;
            rc = simt_prepare(*p);
        } else {
            p->engine = WH_ENGINE_UMMA;
            rc = umma_prepare(*p);
            if (rc == WH_E_UNSUPPORTED && engine == WH_ENGINE_AUTO) {
                // the tensor-core planner could not fit this plan: SIMT handles any plan
                p->engine = WH_ENGINE_SIMT;
                rc = simt_prepare(*p);
            }
        }
    }
    if (rc == WH_OK && norm == WH_NORM_MINMAX && p->engine == WH_ENGINE_UMMA && p->minmax_mode != 0) {
        // write-once min-max: per-clip unit arrivals + the bitmap of units left to the fix-up
        const int64_t bits = (int64_t)((p->row_tiles + p->cg - 1) / p->cg) * (int64_t)p->passes.size() * p->cg;
        p->ab_words = (int32_t)((bits + 31) / 32);
        // (+1 word: the concurrent normaliser's give-up flag)
        if (cudaMalloc(&p->d_arrive, sizeof(uint32_t) * (max_clips + 1)) != cudaSuccess ||
            cudaMalloc(&p->d_abandon, sizeof(uint32_t) * (size_t)max_clips * p->ab_words) != cudaSuccess)
            rc = fail(WH_E_OOM, "cudaMalloc(min-max arrivals) failed");
        if (rc == WH_OK && p->minmax_mode == 2 &&
            (cudaStreamCreateWithFlags(&p->nstream, cudaStreamNonBlocking) != cudaSuccess ||
             cudaEventCreateWithFlags(&p->nev0, cudaEventDisableTiming) != cudaSuccess ||
             cudaEventCreateWithFlags(&p->nev1, cudaEventDisableTiming) != cudaSuccess))
            rc = fail(WH_E_CUDA, "normaliser stream / events failed");
    }
    if (rc == WH_OK && (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess ||
                        cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking) != cudaSuccess))
        rc = fail(WH_E_CUDA, "cudaStreamCreate failed");
    if (rc == WH_OK && cudaDeviceSynchronize() != cudaSuccess)
        rc = fail(WH_E_CUDA, std::string("plan build failed: ") + cudaGetErrorString(cudaGetLastError()));
    cudaSetDevice(prev);
    if (rc != WH_OK) {
        std::string msg = g_last_error;
        plan_free(p);
        set_error(msg);
        return rc;
    }
    *plan = reinterpret_cast<wh_plan *>(p);
    return WH_OK;
}

int wh_plan_destroy(wh_plan *plan) {
    plan_free(reinterpret_cast<Plan *>(plan));
    return WH_OK;
}

int wh_plan_frames(const wh_plan *plan, int64_t *frames) {
    if (!plan || !frames) return fail(WH_E_INVALID_ARG, "NULL argument");
    *frames = reinterpret_cast<const Plan *>(plan)->F;
    return WH_OK;
}

int wh_plan_engine(const wh_plan *plan, int32_t *engine) {
    if (!plan || !engine) return fail(WH_E_INVALID_ARG, "NULL argument");
    *engine = reinterpret_cast<const Plan *>(plan)->engine;
    return WH_OK;
}

int wh_plan_out_bytes(const wh_plan *plan, int64_t clips, int64_t *bytes) {
    if (!plan || !bytes) return fail(WH_E_INVALID_ARG, "NULL argument");
    const Plan *p = reinterpret_cast<const Plan *>(plan);
    *bytes = clips * (int64_t)p->S * p->F * out_elem_bytes(*p);
    return WH_OK;
}

int wh_plan_launches(const wh_plan *plan, int64_t clips, int64_t *launches) {
    if (!plan || !launches) return fail(WH_E_INVALID_ARG, "NULL argument");
    const Plan *p = reinterpret_cast<const Plan *>(plan);
    // engine + (min/max reset + normalise) or (reset + map parameters + uint8 map)
    // min-max: reset + (UMMA: the fix-up check | SIMT: the normalise pass)
    const int mm = p->norm == WH_NORM_MINMAX ? 2 : 0;
    // + the SIMT engine's non-finite fix-up (the UMMA engine's last CTA does it in-kernel)
    const int nf = p->engine == WH_ENGINE_UMMA ? 0 : 1;
    // + the concurrent normaliser (UMMA min-max mode 2)
    const int cn = (p->engine == WH_ENGINE_UMMA && p->norm == WH_NORM_MINMAX && p->minmax_mode == 2) ? 1 : 0;
    *launches = clips > 0 ? (1 + nf + cn + mm + (is_render(*p) ? 3 : 0)) : 0;
    return WH_OK;
}

int wh_plan_mma_flops(const wh_plan *plan, int64_t clips, double *flops) {
    if (!plan || !flops) return fail(WH_E_INVALID_ARG, "NULL argument");
    const Plan *p = reinterpret_cast<const Plan *>(plan);
    *flops = 0.0;
    if (p->engine != WH_ENGINE_UMMA || clips <= 0) return WH_OK;
    // per tile (pair): every K-step tile issues 4 x (MMA1 N = nc + ncorr, MMA2 N = ncorr) of
    // M = 128 * cg rows and K = 16
    double per = 0.0;
    for (const auto &t : p->tiles) per += 2.0 * 128.0 * p->cg * 64.0 * (double)(t.ncols + 2 * t.ncorr);
    *flops = per * (double)clips * (double)((p->row_tiles + p->cg - 1) / p->cg);
    return WH_OK;
}

int wh_plan_taps(const wh_plan *plan, int32_t scale_index, float *re, float *im, int64_t cap,
                 int64_t *half) {
    if (!plan || !re || !im || !half) return fail(WH_E_INVALID_ARG, "NULL argument");
    const Plan *p = reinterpret_cast<const Plan *>(plan);
    if (scale_index < 0 || scale_index >= p->S) return fail(WH_E_INVALID_ARG, "scale index out of range");
    int64_t L = p->half[scale_index];
    *half = L;
    if (cap < 2 * L + 1) return fail(WH_E_INVALID_ARG, "capacity too small");
    std::vector<float> fr(L + 1), fi(L + 1);
    int prev = 0;
    cudaGetDevice(&prev);
    WH_CUDA_TRY(cudaSetDevice(p->device));
    WH_CUDA_TRY(cudaMemcpy(fr.data(), p->d_fold + p->fold_off[scale_index], sizeof(float) * (L + 1),
                           cudaMemcpyDeviceToHost));
    WH_CUDA_TRY(cudaMemcpy(fi.data(), p->d_fold + p->fold_total + p->fold_off[scale_index],
                           sizeof(float) * (L + 1), cudaMemcpyDeviceToHost));
    cudaSetDevice(prev);
    // unfold: real part even, imaginary part odd (wavelet.py:304-310 holds for Morlet taps)
    for (int64_t j = 0; j <= L; ++j) {
        re[L + j] = fr[j]; re[L - j] = fr[j];
        im[L + j] = fi[j]; im[L - j] = -fi[j];
    }
    im[L] = fi[0];
    return WH_OK;
}

// mm: this call's slice of the per-clip min/max keys; scratch: its slice of the float
// values a render plan maps to uint8
// arrive: this call's slice of the per-clip unit arrival counters (UMMA write-once min-max)
static int execute_impl(Plan *p, const float *x_dev, int64_t clips, int64_t ld_x, void *out_dev, cudaStream_t s,
                        uint32_t *mm, uint32_t *arrive, uint32_t *abandon, float *scratch, void *rparams, int64_t c0) {
    int rc = WH_OK;
    // this launch's slices of the non-finite-sample records (c0: its first clip in the plan's
    // per-clip arrays)
    uint32_t *nfbad = p->d_nfbad + c0 * (int64_t)(1 + WH_NF_CAP), *nfctl = p->d_nfctl + 2 * c0;
    const bool render = is_render(*p);
    void *dst = render ? static_cast<void *>(scratch) : out_dev;
    // the UMMA engine normalises min-max plans inside the kernel (write-once); the SIMT
    // engine keeps the read-modify-write pass
    const bool umma_mm = p->norm == WH_NORM_MINMAX && p->engine == WH_ENGINE_UMMA;
    const bool inkernel = umma_mm && p->minmax_mode == 1;
    const bool concurrent = umma_mm && p->minmax_mode == 2;
    if (p->norm != WH_NORM_NONE)
        rc = minmax_reset(*p, clips, mm, (inkernel || concurrent) ? arrive : nullptr, abandon, s);
    if (rc == WH_OK && concurrent) {
        // the normaliser runs beside the kernel on its own stream and SMs; the caller's stream
        // waits for it before the trailing masked pass
        const uint32_t target = (uint32_t)(p->cg * ((p->row_tiles + p->cg - 1) / p->cg) *
                                           umma_pass_groups(*p, clips));
        if (cudaMemsetAsync(p->d_arrive + p->max_clips, 0, sizeof(uint32_t), s) != cudaSuccess ||
            cudaEventRecord(p->nev0, s) != cudaSuccess || cudaStreamWaitEvent(p->nstream, p->nev0, 0) != cudaSuccess)
            rc = fail(WH_E_CUDA, "normaliser fork failed");
        if (rc == WH_OK) rc = minmax_stream_launch(*p, clips, out_dev, mm, arrive, nfbad, target, p->nstream);
        if (rc == WH_OK && cudaEventRecord(p->nev1, p->nstream) != cudaSuccess)
            rc = fail(WH_E_CUDA, "normaliser event failed");
    }
    if (rc == WH_OK)
        rc = (p->engine == WH_ENGINE_UMMA)
                 ? umma_launch(*p, x_dev, clips, ld_x, dst, s, mm, (inkernel || concurrent) ? arrive : nullptr, abandon,
                               nfbad, nfctl)
                 : simt_launch(*p, x_dev, clips, ld_x, dst, s, mm, nfbad, nfctl);
    if (rc == WH_OK && concurrent && cudaStreamWaitEvent(s, p->nev1, 0) != cudaSuccess)
        rc = fail(WH_E_CUDA, "normaliser join failed");
    // the SIMT engine's non-finite fix-up is a kernel of its own (the UMMA engine's last CTA
    // does it)
    if (rc == WH_OK && p->engine != WH_ENGINE_UMMA)
        rc = nf_fixup_launch(*p, x_dev, clips, ld_x, dst, p->norm != WH_NORM_NONE ? mm : nullptr, nfbad, s);
    if (rc == WH_OK && p->norm == WH_NORM_MINMAX && !inkernel)
        rc = minmax_apply(*p, clips, out_dev, mm, s, concurrent ? arrive : nullptr);  // mode 2: the clips left
    if (rc == WH_OK && render)
        rc = render_apply(scratch, clips, p->S, p->F, mm, rparams, p->norm == WH_NORM_RENDER_U8 ? 1 : 0,
                          static_cast<uint8_t *>(out_dev), s);
    return rc;
}

int wh_execute(wh_plan *plan, const float *x_dev, int64_t clips, int64_t ld_x, void *out_dev,
               void *stream) {
    if (!plan) return fail(WH_E_INVALID_ARG, "plan is NULL");
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (clips < 0 || clips > p->max_clips) return fail(WH_E_INVALID_ARG, "clips out of range [0, max_clips]");
    if (clips == 0) return WH_OK;
    if (!x_dev || !out_dev) return fail(WH_E_INVALID_ARG, "NULL buffer");
    if (ld_x < p->N) return fail(WH_E_INVALID_ARG, "ld_x < n_samples");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != p->device) WH_CUDA_TRY(cudaSetDevice(p->device));
    const int rc = execute_impl(p, x_dev, clips, ld_x, out_dev, s, p->d_minmax, p->d_arrive, p->d_abandon,
                                p->d_scratch, p->d_rparams, 0);
    if (prev != p->device) cudaSetDevice(prev);
    return rc;
}

static bool is_pinned(const void *ptr) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// ---- wh_execute_host pipelines ---------------------------------------------------------
// One chunk of clips [c0, c0 + nc) on stream s: H2D of its input from `xsrc`, the plan's
// kernels into the plan's device buffers, D2H of its output into `odst`.
static int host_chunk(Plan *p, const float *xsrc, void *odst, int64_t c0, int64_t nc, cudaStream_t s,
                      size_t in_clip, size_t out_clip, cudaEvent_t h2d_done = nullptr) {
    float *dx = p->d_x + (size_t)c0 * p->N;
    uint8_t *dout = reinterpret_cast<uint8_t *>(p->d_out) + (size_t)c0 * out_clip;
    if (cudaMemcpyAsync(dx, xsrc, in_clip * (size_t)nc, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return fail(WH_E_CUDA, "H2D copy failed");
    if (h2d_done && cudaEventRecord(h2d_done, s) != cudaSuccess) return fail(WH_E_CUDA, "cudaEventRecord failed");
    int rc = execute_impl(p, dx, nc, p->N, dout, s, p->d_minmax + 2 * c0, p->d_arrive ? p->d_arrive + c0 : nullptr,
                          p->d_abandon ? p->d_abandon + (size_t)c0 * p->ab_words : nullptr,
                          p->d_scratch ? p->d_scratch + (size_t)c0 * p->S * p->F : nullptr,
                          p->d_rparams ? static_cast<uint8_t *>(p->d_rparams) + (size_t)WH_RENDER_PARAM_BYTES * c0
                                       : nullptr,
                          c0);
    if (rc == WH_OK && cudaMemcpyAsync(odst, dout, out_clip * (size_t)nc, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        rc = fail(WH_E_CUDA, "D2H copy failed");
    return rc;
}

// Pinned host buffers: clip chunks alternate over two streams so that the H2D copy of chunk
// j+1, the kernels of chunk j and the D2H copy of chunk j-1 overlap (PCIe is full duplex).
// The D2H copies bound the pipeline; the first chunk is small so that they start early (its
// H2D copy and kernel are the pipeline fill), the rest are equal.
static int host_pipeline_pinned(Plan *p, const float *x_host, int64_t clips, void *out_host, size_t in_clip,
                                size_t out_clip) {
    int64_t max_chunks = 8;
    if (const char *c = diag_knob("WH_HOST_CHUNKS")) max_chunks = std::max(1, std::atoi(c));
    const int64_t n_chunks = clips >= 4 ? std::min<int64_t>(max_chunks, clips) : 1;
    int64_t first = clips, per = clips;
    if (n_chunks > 1) {
        first = std::max<int64_t>(1, clips / (4 * n_chunks));
        if (const char *f = diag_knob("WH_HOST_FIRST")) first = std::max<int64_t>(1, std::atoi(f));
        first = std::min(first, clips - (n_chunks - 1));
        per = (clips - first + n_chunks - 2) / (n_chunks - 1);
    }
    int rc = WH_OK;
    for (int64_t c0 = 0, j = 0, nc = first; c0 < clips && rc == WH_OK; c0 += nc, ++j, nc = per) {
        nc = std::min(nc, clips - c0);
        rc = host_chunk(p, x_host + (size_t)c0 * p->N, static_cast<uint8_t *>(out_host) + (size_t)c0 * out_clip, c0, nc,
                        (j & 1) ? p->stream2 : p->stream, in_clip, out_clip);
    }
    return rc;
}

// memcpy split over host threads (a pageable <-> pinned copy runs at a few GB/s per core)
static void par_copy(void *dst, const void *src, size_t bytes) {
    const size_t kMin = (size_t)8 << 20;
    unsigned hw = std::thread::hardware_concurrency();
    size_t nt = std::min<size_t>(std::max(1u, std::min(hw, 8u)), (bytes + kMin - 1) / kMin);
    if (nt <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    const size_t per = ((bytes + nt - 1) / nt + 63) & ~(size_t)63;
    std::vector<std::thread> th;
    for (size_t t = 1; t < nt && t * per < bytes; ++t)
        th.emplace_back([=] {
            const size_t o = t * per;
            memcpy(static_cast<uint8_t *>(dst) + o, static_cast<const uint8_t *>(src) + o, std::min(per, bytes - o));
        });
    memcpy(dst, src, std::min(per, bytes));
    for (auto &t : th) t.join();
}

// Pageable host buffers: a plan-owned pinned staging ring of two input and two output chunk
// slots.  Per chunk j (slot j & 1): the host copies its input into the slot once the H2D copy
// of chunk j-2 has finished, the device copies / computes / copies back into the output slot,
// and while it does the host drains chunk j-1's output slot into the caller's buffer.
static int host_pipeline_staged(Plan *p, const float *x_host, int64_t clips, void *out_host, size_t in_clip,
                                size_t out_clip) {
    const size_t target = (size_t)64 << 20;  // bytes of input + output per chunk
    int64_t per = std::max<int64_t>(1, (int64_t)(target / (in_clip + out_clip)));
    if (clips >= 2) per = std::min(per, (clips + 1) / 2);  // at least two chunks: overlap
    per = std::min(per, clips);
    const size_t slot_in = in_clip * (size_t)per, slot_out = out_clip * (size_t)per;
    const size_t need = 2 * (slot_in + slot_out);
    if (need > p->h_stage_bytes) {
        if (p->h_stage) cudaFreeHost(p->h_stage);
        p->h_stage = nullptr;
        p->h_stage_bytes = 0;
        if (cudaHostAlloc(reinterpret_cast<void **>(&p->h_stage), need, cudaHostAllocDefault) != cudaSuccess) {
            (void)cudaGetLastError();
            return fail(WH_E_OOM, "cudaHostAlloc(staging ring) failed");
        }
        p->h_stage_bytes = need;
    }
    for (int i = 0; i < 2; ++i) {
        if (!p->ev_h2d[i] && cudaEventCreateWithFlags(&p->ev_h2d[i], cudaEventDisableTiming) != cudaSuccess)
            return fail(WH_E_CUDA, "cudaEventCreate failed");
        if (!p->ev_d2h[i] && cudaEventCreateWithFlags(&p->ev_d2h[i], cudaEventDisableTiming) != cudaSuccess)
            return fail(WH_E_CUDA, "cudaEventCreate failed");
    }
    uint8_t *xs[2] = {p->h_stage, p->h_stage + slot_in};
    uint8_t *os[2] = {p->h_stage + 2 * slot_in, p->h_stage + 2 * slot_in + slot_out};
    const int64_t n_chunks = (clips + per - 1) / per;
    auto drain = [&](int64_t j) -> int {
        const int k = (int)(j & 1);
        if (cudaEventSynchronize(p->ev_d2h[k]) != cudaSuccess) return fail(WH_E_CUDA, "execute_host: D2H failed");
        const int64_t c0 = j * per, nc = std::min(per, clips - c0);
        par_copy(static_cast<uint8_t *>(out_host) + (size_t)c0 * out_clip, os[k], out_clip * (size_t)nc);
        return WH_OK;
    };
    int rc = WH_OK;
    for (int64_t j = 0; j < n_chunks && rc == WH_OK; ++j) {
        const int k = (int)(j & 1);
        const int64_t c0 = j * per, nc = std::min(per, clips - c0);
        cudaStream_t s = k ? p->stream2 : p->stream;
        if (j >= 2 && cudaEventSynchronize(p->ev_h2d[k]) != cudaSuccess) {
            rc = fail(WH_E_CUDA, "execute_host: H2D failed");
            break;
        }
        par_copy(xs[k], x_host + (size_t)c0 * p->N, in_clip * (size_t)nc);
        rc = host_chunk(p, reinterpret_cast<const float *>(xs[k]), os[k], c0, nc, s, in_clip, out_clip, p->ev_h2d[k]);
        if (rc == WH_OK && cudaEventRecord(p->ev_d2h[k], s) != cudaSuccess) rc = fail(WH_E_CUDA, "cudaEventRecord failed");
        if (rc == WH_OK && j >= 1) rc = drain(j - 1);
    }
    if (rc == WH_OK) rc = drain(n_chunks - 1);
    return rc;
}

int wh_execute_host(wh_plan *plan, const float *x_host, int64_t clips, void *out_host) {
    if (!plan) return fail(WH_E_INVALID_ARG, "plan is NULL");
    Plan *p = reinterpret_cast<Plan *>(plan);
    if (clips < 0 || clips > p->max_clips) return fail(WH_E_INVALID_ARG, "clips out of range [0, max_clips]");
    if (clips == 0) return WH_OK;
    if (!x_host || !out_host) return fail(WH_E_INVALID_ARG, "NULL buffer");
    int prev = 0;
    cudaGetDevice(&prev);
    WH_CUDA_TRY(cudaSetDevice(p->device));
    size_t xb = sizeof(float) * (size_t)clips * p->N;
    size_t ob = (size_t)clips * p->S * p->F * out_elem_bytes(*p);
    if (xb > p->d_x_bytes) {
        cudaFree(p->d_x);
        p->d_x = nullptr;
        size_t cap = sizeof(float) * (size_t)p->max_clips * p->N;
        WH_CUDA_TRY(cudaMalloc(&p->d_x, cap));
        p->d_x_bytes = cap;
    }
    if (ob > p->d_out_bytes) {
        cudaFree(p->d_out);
        p->d_out = nullptr;
        size_t cap = (size_t)p->max_clips * p->S * p->F * out_elem_bytes(*p);
        WH_CUDA_TRY(cudaMalloc(&p->d_out, cap));
        p->d_out_bytes = cap;
    }
    const bool pinned = is_pinned(x_host) && is_pinned(out_host);
    const size_t in_clip = sizeof(float) * (size_t)p->N;
    const size_t out_clip = (size_t)p->S * p->F * out_elem_bytes(*p);
    int rc = pinned ? host_pipeline_pinned(p, x_host, clips, out_host, in_clip, out_clip)
                    : host_pipeline_staged(p, x_host, clips, out_host, in_clip, out_clip);
    const cudaError_t e1 = cudaStreamSynchronize(p->stream), e2 = cudaStreamSynchronize(p->stream2);
    if (rc == WH_OK && (e1 != cudaSuccess || e2 != cudaSuccess))
        rc = fail(WH_E_CUDA, std::string("execute_host failed: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    cudaSetDevice(prev);
    return rc;
}

int wh_plan_profile(wh_plan *plan, int32_t enable, uint64_t *counters, int32_t n) {
    if (!plan) return fail(WH_E_INVALID_ARG, "plan is NULL");
#ifndef WH_DIAG
    (void)enable; (void)counters; (void)n;
    return fail(WH_E_UNSUPPORTED, "diagnostics need the WH_DIAG build (python -m paper_2408_14302_b200.build --diag)");
#endif
    Plan *p = reinterpret_cast<Plan *>(plan);
    int prev = 0;
    cudaGetDevice(&prev);
    WH_CUDA_TRY(cudaSetDevice(p->device));
    if (!p->d_prof) {
        WH_CUDA_TRY(cudaMalloc(&p->d_prof, sizeof(unsigned long long) * 20));
        WH_CUDA_TRY(cudaMemset(p->d_prof, 0, sizeof(unsigned long long) * 20));
    }
    if (counters && n > 0) {
        unsigned long long h[20];
        WH_CUDA_TRY(cudaDeviceSynchronize());
        WH_CUDA_TRY(cudaMemcpy(h, p->d_prof, sizeof h, cudaMemcpyDeviceToHost));
        for (int i = 0; i < n && i < 20; ++i) counters[i] = h[i];
        WH_CUDA_TRY(cudaMemset(p->d_prof, 0, sizeof(unsigned long long) * 20));
    }
    if (!enable) {
        // the profile counters only: the trace buffer belongs to wh_plan_trace
        cudaFree(p->d_prof);
        p->d_prof = nullptr;
    }
    cudaSetDevice(prev);
    return WH_OK;
}

int wh_plan_trace(wh_plan *plan, int32_t enable, int64_t *events, int32_t n) {
    if (!plan) return fail(WH_E_INVALID_ARG, "plan is NULL");
#ifndef WH_DIAG
    (void)enable; (void)events; (void)n;
    return fail(WH_E_UNSUPPORTED, "diagnostics need the WH_DIAG build (python -m paper_2408_14302_b200.build --diag)");
#endif
    Plan *p = reinterpret_cast<Plan *>(plan);
    int prev = 0;
    cudaGetDevice(&prev);
    WH_CUDA_TRY(cudaSetDevice(p->device));
    if (!p->d_trace) {
        WH_CUDA_TRY(cudaMalloc(&p->d_trace, sizeof(long long) * WH_TRACE_N));
        WH_CUDA_TRY(cudaMemset(p->d_trace, 0, sizeof(long long) * WH_TRACE_N));
    }
    if (events && n > 0) {
        static long long h[WH_TRACE_N];
        WH_CUDA_TRY(cudaDeviceSynchronize());
        WH_CUDA_TRY(cudaMemcpy(h, p->d_trace, sizeof h, cudaMemcpyDeviceToHost));
        for (int i = 0; i < n && i < WH_TRACE_N; ++i) events[i] = h[i];
    }
    if (!enable) {
        cudaFree(p->d_trace);
        p->d_trace = nullptr;
    }
    cudaSetDevice(prev);
    return WH_OK;
}

static int seam2(int device, const double *xpad, int64_t xpad_len, const double *a,
                 const double *b, int64_t width, int64_t n_taps, int64_t hop, int64_t frames,
                 double *ore, double *oim, bool symmetric) {
    if (hop < 1) return fail(WH_E_INVALID_HOP, "hop must be an integer >= 1");
    if (!xpad || !a || !b || !ore || !oim) return fail(WH_E_INVALID_ARG, "NULL buffer");
    if (frames < 0 || width < 1) return fail(WH_E_INVALID_ARG, "bad sizes");
    if (frames == 0) return WH_OK;
    if (xpad_len < (frames - 1) * hop + width) return fail(WH_E_INVALID_ARG, "xpad too short");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(WH_E_NO_DEVICE, "no such CUDA device");
    int prev = 0;
    cudaGetDevice(&prev);
    WH_CUDA_TRY(cudaSetDevice(device));
    double *dx = nullptr, *da = nullptr, *db = nullptr, *dr = nullptr, *di = nullptr;
    size_t need = (size_t)((frames - 1) * hop + width);
    int rc = WH_OK;
    if (cudaMalloc(&dx, sizeof(double) * need) != cudaSuccess ||
        cudaMalloc(&da, sizeof(double) * n_taps) != cudaSuccess ||
        cudaMalloc(&db, sizeof(double) * n_taps) != cudaSuccess ||
        cudaMalloc(&dr, sizeof(double) * frames) != cudaSuccess ||
        cudaMalloc(&di, sizeof(double) * frames) != cudaSuccess) {
        rc = fail(WH_E_OOM, "cudaMalloc failed");
    }
    if (rc == WH_OK) {
        cudaMemcpy(dx, xpad, sizeof(double) * need, cudaMemcpyHostToDevice);
        cudaMemcpy(da, a, sizeof(double) * n_taps, cudaMemcpyHostToDevice);
        cudaMemcpy(db, b, sizeof(double) * n_taps, cudaMemcpyHostToDevice);
        unsigned blocks = (unsigned)((frames + 127) / 128);
        if (symmetric)
            k_strided_symmetric<<<blocks, 128>>>(dx, da, db, n_taps - 1, hop, frames, dr, di);
        else
            k_strided_generic<<<blocks, 128>>>(dx, da, db, width, hop, frames, dr, di);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = fail(WH_E_CUDA, cudaGetErrorString(e));
    }
    if (rc == WH_OK) {
        cudaMemcpy(ore, dr, sizeof(double) * frames, cudaMemcpyDeviceToHost);
        cudaMemcpy(oim, di, sizeof(double) * frames, cudaMemcpyDeviceToHost);
    }
    cudaFree(dx); cudaFree(da); cudaFree(db); cudaFree(dr); cudaFree(di);
    cudaSetDevice(prev);
    return rc;
}

int wh_strided_correlate(int device, const double *xpad, int64_t xpad_len, const double *taps_re,
                         const double *taps_im, int64_t width, int64_t hop, int64_t frames,
                         double *out_re, double *out_im) {
    return seam2(device, xpad, xpad_len, taps_re, taps_im, width, width, hop, frames, out_re,
                 out_im, false);
}

int wh_strided_correlate_symmetric(int device, const double *xpad, int64_t xpad_len,
                                   const double *re_half, const double *im_half, int64_t half,
                                   int64_t hop, int64_t frames, double *out_re, double *out_im) {
    if (half < 0) return fail(WH_E_INVALID_ARG, "half < 0");
    return seam2(device, xpad, xpad_len, re_half, im_half, 2 * half + 1, half + 1, hop, frames,
                 out_re, out_im, true);
}

}  // extern "C"
