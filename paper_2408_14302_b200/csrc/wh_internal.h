// wh_internal.h -- shared declarations of libwavehop_b200 (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/wavehop_b200.h"

namespace wh {

// diagnostics trace buffer (wh_plan_trace): CTA-0 timeline [16 events][32 units] of clock64,
// then per CTA (up to 256) the %globaltimer (ns) at kernel entry and exit
constexpr int WH_TRACE_N = 16 * 32 + 2 * 256;

// Planner overrides (read once, at plan creation): select alternative but valid plan shapes
// (the parity tests exercise them: WH_UMMA_HYBRID, _NO_RESIDENT, _CG1, _TAU, _NO_CONVREGS,
// _G0_ALIGN, _PGROUPS, ...).  Never read at launch time.
inline const char *plan_knob(const char *name) { return std::getenv(name); }
// Diagnostics knobs (role switches, verbose plan dump): only in a -DWH_DIAG build.
inline const char *diag_knob(const char *name) {
#ifdef WH_DIAG
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

// non-finite samples tracked per clip (beyond: every coefficient of the clip is NaN)
constexpr int WH_NF_CAP = 1024;

// Thread-local last-error message behind wh_last_error().
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define WH_CUDA_TRY(expr)                                                                   \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return ::wh::fail(WH_E_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(e_)); \
    } while (0)

// ---------------------------------------------------------------------------------------
// SIMT engine (any hop).  Folded fp32 direct correlation (the reference's
// _kernels.py:93-112 loop, re-tiled for the GPU).
struct SimtGroup {      // a group of <= 8 consecutive scales sharing a tap table
    int32_t s0, ns;     // first scale, number of scales
    int32_t L;          // max half width in the group
    int32_t tf;         // frames per CTA tile
    int64_t tap_off;    // offset (floats) of the group's [ns][L+1] re table (im follows)
};
struct SimtItem {       // one CTA of work: groups [g0, g1) of the cost-ordered list, frames [k0, k0 + tf)
    int32_t g0, g1, k0, L;  // L: max half width over the groups (staged segment margin)
};

// ---------------------------------------------------------------------------------------
// UMMA engine (tcgen05, split-fp16).  See DESIGN.md §Kernels.
struct UmmaPass {
    int32_t tile_begin, tile_end;  // range in the tile table
    int32_t s0, ns;                // scales covered by the pass
    int32_t cols;                  // TMEM columns (multiple of 16, <= 128)
    int32_t group_begin, group_end;  // range in the group table
};
struct UmmaTile {                  // one K-step (64 taps) of one pass
    int32_t k;                     // K-step index (g in [64k, 64k+64))
    int32_t c0;                    // first active column (multiple of 16)
    int32_t ncols;                 // cols - c0
    int32_t ncorr;                 // cols - c1: columns whose split-fp16 cross terms are kept
    int32_t in_off;                // byte offset of the tile inside its group's CTA block
    int64_t byte_off;              // bank offset of the tile (CTA-0 block of its group)
    int64_t blk1_delta;            // cg = 2: bytes from the CTA-0 block to the CTA-1 block
};
struct UmmaGroup {                 // consecutive tiles of a pass fetched by one bulk copy
    int32_t tile_begin, tile_end;
    int32_t cta_bytes;             // bytes each CTA copies
    int32_t pad_;                  // resident bank: the group's smem offset in the ring
    int64_t bank_off;              // bank offset of the group's CTA-0 block
};

struct Plan {
    int device = 0;
    int sms = 148;
    int grid_ctas = 148;                   // UMMA: co-resident CTAs (pairs x 2) of the persistent grid
    int32_t S = 0;
    std::vector<double> scales;
    std::vector<int64_t> half;     // L_s (fp64 ceil, wavelet.py:154)
    double C = 1.0, B = 1.5, R = 6.0;
    int32_t wavelet = WH_WAVELET_CMOR;
    int64_t hop = 1, N = 0, F = 0, max_clips = 0;
    int32_t output = WH_OUT_COMPLEX64, norm = WH_NORM_NONE;
    int32_t engine = WH_ENGINE_SIMT;
    int64_t Lmax = 0;

    // device filter bank: folded fp32 taps per scale (re then im), offsets per scale
    float *d_fold = nullptr;       // [sum (L_s+1)] re, then same for im
    std::vector<int64_t> fold_off; // host copy of per-scale offsets
    int64_t fold_total = 0;
    double *d_scales = nullptr;
    int64_t *d_half = nullptr;
    int64_t *d_fold_off = nullptr;

    // SIMT engine
    std::vector<SimtGroup> groups;
    SimtGroup *d_groups = nullptr;
    SimtItem *d_items = nullptr;
    int32_t n_items = 0;
    float *d_group_taps = nullptr; // per group [ns][L+1] re then [ns][L+1] im

    // UMMA engine
    int32_t V = 64, P = 1, Cc = 1, panels = 1;
    int32_t rs = 1;                        // UMMA rows per frame (hop = 256 * rs > 256)
    int32_t Qlo = 0, G0 = 0, ksteps = 0, win_rows = 0;  // window rows (multiple of 8)
    int32_t rows_total = 0, row_tiles = 0;
    std::vector<UmmaPass> passes;
    std::vector<UmmaTile> tiles;
    std::vector<UmmaGroup> groups_u;
    UmmaPass *d_passes = nullptr;
    UmmaTile *d_tiles = nullptr;
    UmmaGroup *d_groups_u = nullptr;
    uint8_t *d_bank = nullptr;
    int64_t bank_bytes = 0;
    float *d_scale_pow = nullptr;  // per scale 2^-f_s
    uint8_t *d_tables = nullptr;   // UMMA: the kernel's smem tables, packed (one bulk copy)
    int64_t tables_bytes = 0;
    int32_t simt_tf = 1;           // SIMT: frames per item tile
    bool doubled_v = false, no_2v = false;  // UMMA: rows of 2 lcm(hop, 64) samples (one pass)
    int32_t pstream = 0;           // UMMA: rows of hop samples (one frame each), window streamed by column panel
    bool no_pstream = false;       // UMMA planner retry without panel streaming
    int32_t tf32 = 0;              // UMMA panel streaming with kind::tf32 MMAs (no window exponent, no pre-pass)
    bool ps_cg1 = false;           // panel streaming with single-CTA MMAs (a clip's last tile pair would be half empty)
    bool no_tma = false;           // planner override: tf32 panels fetched by cp.async instead of TMA tensor copies
    int32_t acc2 = 0;              // tf32: two accumulator sets per TMEM buffer (even / odd K-slices)
    int32_t ks = 64;               // taps per K-step: 64 (fp16 operands) or 32 (tf32 operands), 128 B per operand row
    int32_t tile_rows = 128;       // rows of a tile that carry frames (<= 128: a clip's rows split evenly over its tiles)
    double unit_cost = 0.0;        // UMMA: modelled MMA cycles of one unit (all passes)
    bool no_convregs = false;      // UMMA planner override: converters without the register prefetch
    bool force_fixup = false;      // UMMA planner override (tests): min-max units all to the fix-up kernel
    bool minmax_2pass = false;     // UMMA: per-clip min-max as a separate read-modify-write pass
    // UMMA per-clip min-max: 0 separate pass after the kernel, 1 in-kernel write-once
    // (experiment), 2 concurrent normaliser CTAs (k_minmax_stream on its own SMs, fed by the
    // kernel's per-clip unit arrivals)
    int32_t minmax_mode = 0;
    int32_t norm_ctas = 8;         // mode 2: SMs given to the normaliser (clusters of 2)
    cudaStream_t nstream = nullptr;
    cudaEvent_t nev0 = nullptr, nev1 = nullptr;
    int32_t pgroups_force = 0;     // UMMA planner override: pass groups per tile pair (0 = modelled)
    int32_t dbg = 0;               // diagnostics role switches (WH_DIAG builds only)
    std::vector<int32_t> fexp;
    int32_t bstages = 2, win_bufs = 2;     // bstages: full-width tiles the ring holds (info)
    int64_t ring_bytes = 0;                // tap-tile ring capacity
    int32_t n_acc = 2, acc_stride = 256;   // TMEM accumulator buffers, columns per buffer
    int32_t use_stg = 1;                   // fp32 window staged by cp.async.bulk
    int32_t cg = 2;                        // CTAs per MMA (tcgen05 cta_group)
    int32_t resident = 0;                  // (part of) the tap bank resident in smem
    int64_t res_bytes = 0;                 // resident bytes per CTA (the stage region's prefix)
    int32_t n_stream = 0;                  // tap groups streamed through the ring per unit
    size_t smem_bytes = 0;     // dynamic shared memory of the engine kernel

    unsigned long long *d_prof = nullptr;  // diagnostics counters (wh_plan_profile)
    long long *d_trace = nullptr;          // diagnostics timeline (wh_plan_trace)

    // per-clip min/max (ordered-uint keys) for WH_NORM_MINMAX
    uint32_t *d_minmax = nullptr;  // [max_clips][2]
    uint32_t *d_arrive = nullptr;  // UMMA write-once min-max: [max_clips] unit arrivals per clip
    uint32_t *d_abandon = nullptr; // UMMA write-once min-max: [max_clips][ab_words] units left to the fix-up
    int32_t ab_words = 0;
    // non-finite input samples (NaN / +-inf): the engines compute with them replaced by 0 and
    // record their positions; a fix-up then writes the exact IEEE value of every coefficient
    // whose support contains one (the reference's propagation, wavelet.py:264-270)
    uint32_t *d_nfbad = nullptr;   // [max_clips][1 + WH_NF_CAP]: count, positions
    uint32_t *d_nfctl = nullptr;   // [max_clips][2]: per-launch CTA counter (slot of the launch's first clip), any-flag
    float *d_scratch = nullptr;    // render plans: float values [max_clips][S][F] before the uint8 map
    void *d_rparams = nullptr;     // render plans: WH_RENDER_PARAM_BYTES per clip

    // host staging for wh_execute_host
    float *d_x = nullptr;
    void *d_out = nullptr;
    size_t d_x_bytes = 0, d_out_bytes = 0;
    cudaStream_t stream = nullptr, stream2 = nullptr;  // wh_execute_host pipeline
    // wh_execute_host with pageable host buffers: plan-owned pinned staging ring (two input
    // and two output chunk slots) and the events that recycle them
    uint8_t *h_stage = nullptr;
    size_t h_stage_bytes = 0;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
};

int64_t out_elem_bytes(const Plan &p);

// filter bank builders (wh_api.cu)
int build_fold_bank(Plan &p);

// engines
int simt_prepare(Plan &p);
int simt_launch(Plan &p, const float *x, int64_t clips, int64_t ld_x, void *out, cudaStream_t s, uint32_t *mm,
                uint32_t *nfbad, uint32_t *nfctl);
int umma_supported(const Plan &p, std::string *why);
int umma_prepare(Plan &p);
int umma_launch(Plan &p, const float *x, int64_t clips, int64_t ld_x, void *out, cudaStream_t s, uint32_t *mm,
                uint32_t *arrive, uint32_t *abandon, uint32_t *nfbad, uint32_t *nfctl);
int umma_pass_groups(const Plan &p, int64_t clips);

// epilogue helpers (wh_api.cu)
int minmax_reset(Plan &p, int64_t clips, uint32_t *mm, uint32_t *arrive, uint32_t *abandon, cudaStream_t s);
constexpr int WH_RENDER_PARAM_BYTES = 24;  // per-matrix affine map of render_apply
int render_apply(const float *values, int64_t clips, int64_t rows, int64_t cols, const uint32_t *mm, void *params,
                 int32_t flip, uint8_t *out, cudaStream_t s);
inline bool is_render(const Plan &p) { return p.norm == WH_NORM_RENDER_U8 || p.norm == WH_NORM_RENDER_U8_NOFLIP; }
int minmax_apply(Plan &p, int64_t clips, void *out, uint32_t *mm, cudaStream_t s, const uint32_t *done = nullptr);
int minmax_stream_launch(Plan &p, int64_t clips, void *out, uint32_t *mm, uint32_t *arrive, const uint32_t *nfbad,
                         uint32_t target, cudaStream_t s);
constexpr uint32_t WH_CLIP_NORMALISED = 0xffffffffu;  // arrive[] value of a clip the normaliser finished
int nf_fixup_launch(Plan &p, const float *x, int64_t clips, int64_t ld_x, void *out, uint32_t *mm, uint32_t *bad,
                    cudaStream_t s);

}  // namespace wh

// ---- device helpers shared by the engines ----------------------------------------------
#ifdef __CUDACC__
namespace wh {
// Order-preserving float <-> uint mapping for atomicMin/atomicMax on floats.
__device__ __forceinline__ uint32_t f2key(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
    uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(u);
}
// scalogram.py:51-64 + BASELINE log1p, applied to the magnitude.
__device__ __forceinline__ float apply_output(float mag, int output) {
    switch (output) {
        case WH_OUT_POWER: return mag * mag;
        case WH_OUT_LOG_DB: return 20.0f * __log10f(mag + 1e-12f);
        case WH_OUT_LOG1P: return __logf(1.0f + mag);  // abs. error ~2^-21 * |log1p|
        default: return mag;
    }
}
// |re + i im| without overflow / underflow of the squares (clips of any float32 amplitude: the
// reference computes in float64): both parts are scaled by the power of two that brings the
// larger one into [1, 2), and the root is scaled back -- the same bits as sqrt(re^2 + im^2)
// wherever the squares are representable.
__device__ __forceinline__ float cabs_scaled(float re, float im) {
    const float m = fmaxf(fabsf(re), fabsf(im));
    const uint32_t eb = __float_as_uint(m) & 0x7f800000u;         // exponent field of the larger part
    if (eb == 0u || eb >= 0x7f000000u) {                           // zero / subnormal, or >= 2^127 (and inf / NaN)
        if (!(m <= 3.402823466e38f)) return m != m ? m : INFINITY;  // NaN stays NaN, inf -> inf
        const float s = eb == 0u ? 1.2676506e30f : 7.8886091e-31f;  // 2^100 / 2^-100
        const float x = re * s, y = im * s;
        return sqrtf(fmaf(x, x, y * y)) * (eb == 0u ? 7.8886091e-31f : 1.2676506e30f);
    }
    const float s = __uint_as_float(0x7f000000u - eb);              // 2^-e
    const float x = re * s, y = im * s;
    return sqrtf(fmaf(x, x, y * y)) * __uint_as_float(eb);
}
__device__ __forceinline__ float magnitude(float re, float im, int wavelet) {
    return wavelet == WH_WAVELET_RMOR ? fabsf(re) : cabs_scaled(re, im);
}
__device__ __forceinline__ bool is_finite_f(float v) { return fabsf(v) <= 3.402823466e38f; }
// max that propagates NaN (and +inf through |x|): one test per window finds non-finite input
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
// Record non-finite sample `pos` of a clip (bad = the clip's [1 + WH_NF_CAP] record) and
// flag the launch (any = its control word).
__device__ __forceinline__ void nf_record(uint32_t *bad, uint32_t *any, int64_t pos) {
    const uint32_t i = atomicAdd(bad, 1u);
    if (i < (uint32_t)WH_NF_CAP) bad[1 + i] = (uint32_t)pos;
    atomicOr(any, 1u);
}

struct NfArgs {
    const float *x;             // the launch's input [clips][ld_x]
    int64_t ld_x, N, hop, F;
    int32_t S, wavelet, output;
    const double *scales;
    const int64_t *half;
    double C, Bw;
    void *out;                  // [clips][S][F] float or float2 (complex64)
    uint32_t *mm;               // per-clip min/max keys or nullptr
    uint32_t *bad;              // [clips][1 + WH_NF_CAP]
};

// Exact value of every coefficient of clip b whose support [kH - L_s, kH + L_s] holds a
// recorded non-finite sample, as the reference's default (numba) backend gives it: the
// finite samples cannot change a sum that contains +-inf or NaN, so each part is the sum over
// the non-finite samples in the support of x_t * tap(t - kH) in IEEE double (inf * 0 = NaN,
// inf - inf = NaN), then the output map.  The engines' values of
// these coefficients (computed with the samples replaced by 0) are overwritten; the clip's
// min / max keys take the new values (NaN orders above +inf: a NaN clip normalises to NaN,
// an inf clip to 0 / NaN as (v - lo) / (hi - lo) does in float).  More than WH_NF_CAP
// non-finite samples: the whole clip is NaN.  Block-wide; resets the clip's record.
__device__ inline void nf_fixup_clip(const NfArgs &a, int64_t b, int tid, int nthreads) {
    uint32_t *rec = a.bad + b * (int64_t)(1 + WH_NF_CAP);
    const uint32_t cnt = rec[0];
    if (cnt == 0) return;
    const float *xb = a.x + b * a.ld_x;
    float *o32 = reinterpret_cast<float *>(a.out) + b * (int64_t)a.S * a.F;
    float2 *o64 = reinterpret_cast<float2 *>(a.out) + b * (int64_t)a.S * a.F;
    const float qnan = __uint_as_float(0x7fc00000u);
    auto put = [&](int64_t idx, float re, float im, float v) {
        if (a.output == WH_OUT_COMPLEX64) {
            o64[idx] = make_float2(re, im);
        } else {
            o32[idx] = v;
            if (a.mm) {
                atomicMin(a.mm + 2 * b, f2key(v));
                atomicMax(a.mm + 2 * b + 1, f2key(v));
            }
        }
    };
    if (cnt > (uint32_t)WH_NF_CAP) {
        for (int64_t i = tid; i < (int64_t)a.S * a.F; i += nthreads) put(i, qnan, qnan, qnan);
    } else {
        const double norm = rsqrt(M_PI * a.Bw);
        const double w = 2.0 * M_PI * a.C;
        for (uint32_t i = 0; i < cnt; ++i) {
            const int64_t t = rec[1 + i];
            for (int s = tid; s < a.S; s += nthreads) {
                const int64_t L = a.half[s];
                const double sa = a.scales[s], rs = sqrt(sa);
                int64_t k0 = t - L <= 0 ? 0 : (t - L + a.hop - 1) / a.hop;
                int64_t k1 = (t + L) / a.hop;
                if (k1 > a.F - 1) k1 = a.F - 1;
                for (int64_t k = k0; k <= k1; ++k) {
                    const int64_t c = k * a.hop;
                    // owned by the first recorded sample in this coefficient's support
                    bool first = true;
                    for (uint32_t j = 0; j < i && first; ++j) {
                        const int64_t tj = rec[1 + j];
                        first = !(tj >= c - L && tj <= c + L);
                    }
                    if (!first) continue;
                    // the reference's folded kernel (_kernels.py:93-112) has no imaginary tap at
                    // u = 0 (a sample never meets im_0 there), and it assembles re + 1j * im
                    // (wavelet.py:270), whose 0 * im turns the real part into NaN wherever the
                    // imaginary part is not finite
                    double re = 0.0, im = 0.0;
                    bool imbad = false;
                    for (uint32_t j = i; j < cnt; ++j) {
                        const int64_t tj = rec[1 + j];
                        const int64_t u = tj - c;
                        if (u < -L || u > L) continue;
                        const double xv = (double)xb[tj];
                        const double tt = (double)(u < 0 ? -u : u) / sa;
                        const double env = norm * exp(-(tt * tt) / a.Bw);
                        re += xv * (env * cos(w * tt) / rs);
                        if (u != 0) {
                            const double ti = env * sin(w * tt) / rs;
                            im += xv * (u < 0 ? -ti : ti);
                            imbad = true;
                        }
                    }
                    const float ore = (imbad && !isfinite(im)) ? qnan : (isnan(re) ? qnan : (float)re);
                    const int64_t idx = (int64_t)s * a.F + k;
                    if (a.output == WH_OUT_COMPLEX64) {
                        if (a.wavelet == WH_WAVELET_RMOR) o64[idx] = make_float2(ore, 0.0f);
                        else if (imbad) o64[idx] = make_float2(ore, isnan(im) ? qnan : (float)im);
                        else o64[idx].x = ore;  // the imaginary part stays the engine's (finite) value
                        continue;
                    }
                    float mag;
                    if (a.wavelet == WH_WAVELET_RMOR) {
                        mag = fabsf(ore);
                    } else {
                        const bool iminf = imbad && isinf(im);
                        mag = (isinf(ore) || iminf) ? INFINITY : qnan;  // hypot(+-inf, any) = inf
                    }
                    const float v = apply_output(mag, a.output);
                    put(idx, 0.0f, 0.0f, isnan(v) ? qnan : v);
                }
            }
        }
    }
    __syncthreads();
    if (tid == 0) rec[0] = 0;
}
}  // namespace wh
#endif
