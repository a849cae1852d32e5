/*
 * wavehop_b200.h -- C ABI of the B200-native CWTH (hop-strided continuous wavelet
 * transform) library, libwavehop_b200.so.
 *
 * This is the drop-in boundary for the reference package wavehop 0.1.0
 * (arXiv 2408.14302).  The reference is pure Python, so its "FFI" for this path
 * is the pair of seams a maintainer would re-point at this library through ctypes
 * (binding stubs in INTEGRATION.md):
 *
 *   seam 1  wavelet.py:215-273  cwth_strided(signal, grid, params, hop, *, threads)
 *           wavelet.py:187-212  cwt_fft(...)            (the hop = 1 transform)
 *           scalogram.py:51-86  magnitude(matrix, mode) / render normalisation
 *           -> wh_plan_create / wh_execute / wh_execute_host
 *   seam 2  _kernels.py:76-91   strided_correlate(xpad, taps_re, taps_im, hop, frames)
 *           _kernels.py:93-112  strided_correlate_symmetric(xpad, re_half, im_half, hop, frames)
 *           -> wh_strided_correlate / wh_strided_correlate_symmetric
 *
 * Conventions: plain pointers and sizes only; no torch or CUDA types in the
 * signatures (streams are passed as void*, a cudaStream_t).  Every function returns
 * WH_OK (0) or a WH_E_* code; wh_last_error() gives the message of the last
 * failure on the calling thread.  Device-pointer entry points are stream-ordered and
 * never synchronise the host.  Plans own their device memory; one plan may be used
 * from one host thread at a time (one plan per device/thread for multi-GPU).
 */
#ifndef WAVEHOP_B200_H
#define WAVEHOP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WH_ABI_VERSION 2

/* Error codes.  The Python host maps them onto the reference exception types of
 * errors.py: WH_E_INVALID_HOP -> InvalidHop (errors.py:24, raised by
 * signal_io.py:153-156), WH_E_INVALID_SCALE -> InvalidScale (errors.py:40, raised by
 * wavelet.py:151-152), WH_E_EMPTY_SIGNAL -> EmptySignal (errors.py:18),
 * WH_E_INVALID_ARG -> ValueError. */
enum {
    WH_OK = 0,
    WH_E_INVALID_HOP = 1,
    WH_E_INVALID_SCALE = 2,
    WH_E_INVALID_ARG = 3,
    WH_E_EMPTY_SIGNAL = 4,
    WH_E_CUDA = 5,
    WH_E_NO_DEVICE = 6,
    WH_E_UNSUPPORTED = 7,
    WH_E_OOM = 8
};

/* Mother wavelet.  CMOR is the reference's complex Morlet (wavelet.py:32-45,
 * 144-159).  RMOR is its real part (BASELINE configs 1-4). */
enum { WH_WAVELET_CMOR = 0, WH_WAVELET_RMOR = 1 };

/* Output written per coefficient (scalogram.py:51-64 plus the BASELINE log1p). */
enum {
    WH_OUT_COMPLEX64 = 0, /* (f32 re, f32 im) pairs, SCG1 payload order (scalogram.py:105) */
    WH_OUT_ABS = 1,       /* |W|                                                          */
    WH_OUT_POWER = 2,     /* |W|^2                                                        */
    WH_OUT_LOG_DB = 3,    /* 20*log10(|W| + 1e-12)                                        */
    WH_OUT_LOG1P = 4      /* log1p(|W|)                                                   */
};

/* Per-clip normalisation of real outputs: MINMAX maps each clip's (S, F) map
 * affinely onto [0, 1], constant clip -> 0 (scalogram.py:77-83 without x255).
 * RENDER_U8 is render(magnitude(...)) of scalogram.py:67-86 per clip: uint8
 * [clips][S][F], floor((v - lo) * 255 / (hi - lo) + 0.5) in float64, constant clip -> 0,
 * rows flipped (image row 0 = the last scale, flip_vertical=True); _NOFLIP keeps the
 * scale order (flip_vertical=False). */
enum { WH_NORM_NONE = 0, WH_NORM_MINMAX = 1, WH_NORM_RENDER_U8 = 2, WH_NORM_RENDER_U8_NOFLIP = 3 };

/* Compute engine.  AUTO picks the tcgen05 split-fp16 engine when the hop allows a
 * polyphase tiling (hop dividing 64 or 192, hop 128, or a multiple of 64 from 256), the plan
 * fits shared memory and the longest filter's half width is at most 3,360 taps (5,632 at hops
 * 16 / 32 / 64: the accuracy bounds of the split-fp16 accumulation), else the SIMT fp32 engine; UMMA forced on a plan it
 * cannot run returns WH_E_UNSUPPORTED.  There is no CPU engine. */
enum { WH_ENGINE_AUTO = 0, WH_ENGINE_SIMT = 1, WH_ENGINE_UMMA = 2 };

typedef struct wh_plan wh_plan;

int wh_abi_version(void);
const char *wh_last_error(void);

/* wavelet.py:154: L = ceil(support_radius * scale * sqrt(bandwidth / 2)), in fp64.
 * Errors: WH_E_INVALID_SCALE for a non-positive or non-finite scale. */
int wh_half_width(double scale, double bandwidth, double support_radius, int64_t *half);

/* wavelet.py:238 frames = ceil(n / hop) after signal_io.py:153-156 validation. */
int wh_frame_count(int64_t n_samples, int64_t hop, int64_t *frames);

/* Build a plan: validates arguments exactly like wavelet.py:47-53 (MorletParams),
 * 62-69 (ScaleGrid), 151-152 (InvalidScale) and signal_io.py:153-156 (InvalidHop),
 * builds the per-scale filter bank ON THE DEVICE (fp64 math, sample_wavelet
 * wavelet.py:144-159), and allocates the workspace for up to max_clips clips of
 * n_samples samples. */
int wh_plan_create(wh_plan **plan, int device, const double *scales, int32_t n_scales,
                   double center_frequency, double bandwidth, double support_radius,
                   int32_t wavelet, int64_t hop, int64_t n_samples, int64_t max_clips,
                   int32_t output, int32_t norm, int32_t engine);
int wh_plan_destroy(wh_plan *plan);

/* Plan queries. */
int wh_plan_frames(const wh_plan *plan, int64_t *frames);
int wh_plan_engine(const wh_plan *plan, int32_t *engine);
int wh_plan_out_bytes(const wh_plan *plan, int64_t clips, int64_t *bytes);
/* Tensor-core work one wh_execute of `clips` clips issues: the MMA flops the UMMA engine
 * executes (split-fp16: three products minus the skipped tail cross terms, K padded to
 * 64); 0 for the SIMT engine.  For the bench's roofline ("executed" vs algorithmic). */
int wh_plan_mma_flops(const wh_plan *plan, int64_t clips, double *flops);
/* Kernel launches one wh_execute issues (for the bench's gpu_launches claim). */
int wh_plan_launches(const wh_plan *plan, int64_t clips, int64_t *launches);
/* Read back the device-built taps of one scale as fp32 (2L+1 values each of re/im,
 * tap L+j multiplies x[b + j] as in wavelet.py:147-149).  cap = capacity of re/im. */
int wh_plan_taps(const wh_plan *plan, int32_t scale_index, float *re, float *im, int64_t cap,
                 int64_t *half);

/* Diagnostics: enable (1) / disable (0) per-role wait-cycle counters of the UMMA engine
 * kernel and read-and-reset them (20 counters: role*4 + {wait0, wait1, wait2, total}, roles
 * producer, MMA, converter, epilogue, relay; summed over CTAs and warps).  counters may be NULL. */
int wh_plan_profile(wh_plan *plan, int32_t enable, uint64_t *counters, int32_t n);

/* Diagnostics: CTA-0 timeline of the UMMA engine kernel (clock64 stamps, [16 events][32
 * units]); enable / disable and read (events may be NULL). */
int wh_plan_trace(wh_plan *plan, int32_t enable, int64_t *events, int32_t n);

/* The hot path.  x_dev: device float32 [clips][ld_x] (ld_x >= n_samples);
 * out_dev: device [clips][n_scales][frames] float32 (real outputs) or
 * [clips][n_scales][frames][2] float32 (WH_OUT_COMPLEX64).  Stream-ordered on
 * `stream` (a cudaStream_t; NULL = legacy default stream); no host sync. */
int wh_execute(wh_plan *plan, const float *x_dev, int64_t clips, int64_t ld_x, void *out_dev,
               void *stream);

/* End-to-end call with HOST buffers: H2D of x_host, wh_execute, D2H into out_host,
 * synchronous.  Pinned host buffers are used directly; pageable ones are staged. */
int wh_execute_host(wh_plan *plan, const float *x_host, int64_t clips, void *out_host);

/* Seam 2 (_kernels.py:76-91 / 93-112), host float64 buffers, computed in float64 on
 * `device`.  xpad must hold (frames-1)*hop + width samples (the caller guarantees
 * the padding, as wavelet.py:243-246 does for the reference). */
int wh_strided_correlate(int device, const double *xpad, int64_t xpad_len, const double *taps_re,
                         const double *taps_im, int64_t width, int64_t hop, int64_t frames,
                         double *out_re, double *out_im);
int wh_strided_correlate_symmetric(int device, const double *xpad, int64_t xpad_len,
                                   const double *re_half, const double *im_half, int64_t half,
                                   int64_t hop, int64_t frames, double *out_re, double *out_im);

/* Data formats either side of the path.
 *
 * signal_io.py:130-150 decimate(signal, hop, anti_alias) on device buffers: out[b][i] =
 * x[b][i*hop] for i < ceil(n_samples/hop); with anti_alias the reference's low-pass
 * (scipy firwin(10*hop+1, 0.9/hop): Hamming window, unit DC gain) is applied first as a
 * "same"-centred linear convolution, accumulated in float64.  This is the front half of
 * cwth_decimate (wavelet.py:276-294); the back half is a hop-1 plan on the output.
 * Errors: WH_E_INVALID_HOP, WH_E_EMPTY_SIGNAL, WH_E_INVALID_ARG.  Stream-ordered. */
int wh_decimate(int device, const float *x_dev, int64_t clips, int64_t n_samples, int64_t ld_x,
                int64_t hop, int32_t anti_alias, float *out_dev, int64_t ld_out, void *stream);

/* scalogram.py:67-86 render(values, flip_vertical) for `count` real matrices of rows x cols
 * (device float32 [count][rows][cols] -> device uint8, same shape).  Stream-ordered. */
int wh_render_u8(int device, const float *values_dev, int64_t count, int64_t rows, int64_t cols,
                 int32_t flip_vertical, uint8_t *out_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* WAVEHOP_B200_H */
