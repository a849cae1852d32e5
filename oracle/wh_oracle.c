/*
 * wh_oracle.c -- CPU restatement of the reference CWTH hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle and the CPU
 * baseline ("port") for bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker or as the timed reference arm -- never as the product path.
 *
 * Pinned: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the unmodified reference package
 * (oracle/gen_golden.py -> tests/golden/*.npz).
 *
 * Arithmetic is float64 throughout, like the reference.  Each function cites
 * the reference code it restates (paths relative to /root/reference/pkg/src/wavehop).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* wavelet.py:154  half_width = ceil(support_radius * scale * sqrt(bandwidth / 2)) */
int64_t who_half_width(double scale, double bandwidth, double support_radius) {
    return (int64_t)ceil(support_radius * scale * sqrt(bandwidth / 2.0));
}

/* wavelet.py:144-159 sample_wavelet: taps[L + j] = env(j/a) * exp(+i 2 pi C j/a) / sqrt(a).
 * numpy evaluates t = arange(-L, L+1) / scale, env = (pi*B)**-0.5 * exp(-(t*t)/B),
 * phase = (2j*pi*C) * t, taps = env * exp(phase), then taps / sqrt(scale).  The
 * complex product env*(cos+i sin) and the complex/real division are
 * component-wise real operations, reproduced here in the same order. */
void who_sample_wavelet(double scale, double center_frequency, double bandwidth,
                        double support_radius, double *re, double *im) {
    int64_t L = who_half_width(scale, bandwidth, support_radius);
    double norm = pow(M_PI * bandwidth, -0.5);
    double w = 2.0 * M_PI * center_frequency;
    double rs = sqrt(scale);
    for (int64_t i = 0; i <= 2 * L; ++i) {
        double t = (double)(i - L) / scale;
        double env = norm * exp(-(t * t) / bandwidth);
        double th = w * t;
        re[i] = (env * cos(th)) / rs;
        im[i] = (env * sin(th)) / rs;
    }
}

/* _kernels.py:76-91 strided_correlate_numba: out[k] = sum_j xpad[k*hop + j] * taps[j]. */
void who_strided_correlate(const double *xpad, const double *taps_re, const double *taps_im,
                           int64_t width, int64_t hop, int64_t frames, double *out_re,
                           double *out_im) {
    for (int64_t k = 0; k < frames; ++k) {
        const double *w = xpad + k * hop;
        double ar = 0.0, ai = 0.0;
        for (int64_t j = 0; j < width; ++j) {
            ar += w[j] * taps_re[j];
            ai += w[j] * taps_im[j];
        }
        out_re[k] = ar;
        out_im[k] = ai;
    }
}

/* _kernels.py:93-112 strided_correlate_symmetric: folded kernel for taps with
 * even real and odd imaginary part; *_half hold taps[L:], centre first. */
void who_strided_correlate_symmetric(const double *xpad, const double *re_half,
                                     const double *im_half, int64_t half, int64_t hop,
                                     int64_t frames, double *out_re, double *out_im) {
    for (int64_t k = 0; k < frames; ++k) {
        int64_t c = k * hop + half;
        double ar = xpad[c] * re_half[0];
        double ai = 0.0;
        for (int64_t j = 1; j <= half; ++j) {
            double right = xpad[c + j], left = xpad[c - j];
            ar += (right + left) * re_half[j];
            ai += (right - left) * im_half[j];
        }
        out_re[k] = ar;
        out_im[k] = ai;
    }
}

/* ------------------------------------------------------------------------ */
/* Batched driver: wavelet.py:215-273 cwth_strided (direct route for every row)
 * followed by the epilogue of scalogram.py:51-86 and the BASELINE-config
 * extensions documented in DESIGN.md (real Morlet = Re taps, log1p, per-clip
 * min-max).  Rows are independent (wavelet.py:326-332), so a pthread pool over
 * (clip, scale) rows gives results identical to the serial order. */

enum { WHO_CMOR = 0, WHO_RMOR = 1 };
enum { WHO_OUT_COMPLEX = 0, WHO_OUT_ABS = 1, WHO_OUT_POWER = 2, WHO_OUT_LOG_DB = 3, WHO_OUT_LOG1P = 4 };
enum { WHO_NORM_NONE = 0, WHO_NORM_MINMAX = 1 };

typedef struct {
    const float *x;       /* [B][N] float32 samples (upcast exactly to f64) */
    int64_t B, N, hop, frames, S;
    const double *scales;
    double C, Bw, R;
    int wavelet, out_kind;
    double *out;          /* complex: [B][S][F][2]; else [B][S][F] */
    int64_t next;         /* work counter (row = clip*S + s) */
    pthread_mutex_t mu;
    int64_t max_half;
} who_job;

static void who_row(who_job *jb, int64_t row, double *xpad, double *re, double *im,
                    double *ore, double *oim) {
    int64_t b = row / jb->S, s = row % jb->S;
    int64_t N = jb->N, hop = jb->hop, F = jb->frames, mh = jb->max_half;
    /* wavelet.py:243-246: xpad = zeros(max_half + n + max_half + 2*hop); centre-aligned copy */
    int64_t padlen = mh + N + mh + 2 * hop;
    memset(xpad, 0, sizeof(double) * padlen);
    const float *xs = jb->x + b * N;
    for (int64_t i = 0; i < N; ++i) xpad[mh + i] = (double)xs[i];
    double a = jb->scales[s];
    int64_t L = who_half_width(a, jb->Bw, jb->R);
    who_sample_wavelet(a, jb->C, jb->Bw, jb->R, re, im);
    /* wavelet.py:261: base = xpad[max_half - half:]; folded kernel on taps[L:] (264-267) */
    who_strided_correlate_symmetric(xpad + (mh - L), re + L, im + L, L, hop, F, ore, oim);
    double *o = jb->out;
    if (jb->out_kind == WHO_OUT_COMPLEX) {
        double *dst = o + ((b * jb->S + s) * F) * 2;
        for (int64_t k = 0; k < F; ++k) {
            dst[2 * k] = ore[k];
            dst[2 * k + 1] = jb->wavelet == WHO_RMOR ? 0.0 : oim[k];
        }
        return;
    }
    double *dst = o + (b * jb->S + s) * F;
    for (int64_t k = 0; k < F; ++k) {
        /* scalogram.py:59 np.abs (hypot) ; real Morlet: |Re W| */
        double m = jb->wavelet == WHO_RMOR ? fabs(ore[k]) : hypot(ore[k], oim[k]);
        switch (jb->out_kind) {
            case WHO_OUT_ABS: dst[k] = m; break;
            case WHO_OUT_POWER: dst[k] = m * m; break;                       /* scalogram.py:62-63 */
            case WHO_OUT_LOG_DB: dst[k] = 20.0 * log10(m + 1e-12); break;    /* scalogram.py:64 */
            default: dst[k] = log1p(m); break;                               /* BASELINE c2 */
        }
    }
}

static void *who_worker(void *arg) {
    who_job *jb = (who_job *)arg;
    int64_t mh = jb->max_half;
    int64_t padlen = mh + jb->N + mh + 2 * jb->hop;
    double *xpad = (double *)malloc(sizeof(double) * padlen);
    double *re = (double *)malloc(sizeof(double) * (2 * mh + 1));
    double *im = (double *)malloc(sizeof(double) * (2 * mh + 1));
    double *ore = (double *)malloc(sizeof(double) * jb->frames);
    double *oim = (double *)malloc(sizeof(double) * jb->frames);
    for (;;) {
        pthread_mutex_lock(&jb->mu);
        int64_t row = jb->next++;
        pthread_mutex_unlock(&jb->mu);
        if (row >= jb->B * jb->S) break;
        who_row(jb, row, xpad, re, im, ore, oim);
    }
    free(xpad); free(re); free(im); free(ore); free(oim);
    return NULL;
}

/* scalogram.py:77-83 (render's affine min-max, without x255/round) applied per clip. */
static void who_minmax(double *out, int64_t B, int64_t per_clip) {
    for (int64_t b = 0; b < B; ++b) {
        double *v = out + b * per_clip;
        double lo = v[0], hi = v[0];
        for (int64_t i = 1; i < per_clip; ++i) {
            if (v[i] < lo) lo = v[i];
            if (v[i] > hi) hi = v[i];
        }
        if (hi == lo) {
            for (int64_t i = 0; i < per_clip; ++i) v[i] = 0.0;
        } else {
            double sc = 1.0 / (hi - lo);
            for (int64_t i = 0; i < per_clip; ++i) v[i] = (v[i] - lo) * sc;
        }
    }
}

/* Returns 0 on success, 1 for an invalid hop (signal_io.py:153-156), 2 for an
 * invalid scale (wavelet.py:151-152), 3 for other invalid arguments. */
int who_cwth_batch(const float *x, int64_t B, int64_t N, const double *scales, int64_t S,
                   double C, double Bw, double R, int64_t hop, int wavelet, int out_kind,
                   int norm, double *out, int threads) {
    if (hop < 1) return 1;
    if (B < 0 || N < 1 || S < 1) return 3;
    for (int64_t s = 0; s < S; ++s)
        if (!(scales[s] > 0 && isfinite(scales[s]))) return 2;
    who_job jb;
    memset(&jb, 0, sizeof jb);
    jb.x = x; jb.B = B; jb.N = N; jb.hop = hop; jb.frames = (N + hop - 1) / hop; jb.S = S;
    jb.scales = scales; jb.C = C; jb.Bw = Bw; jb.R = R; jb.wavelet = wavelet;
    jb.out_kind = out_kind; jb.out = out; jb.next = 0;
    int64_t mh = 0;
    for (int64_t s = 0; s < S; ++s) {
        int64_t L = who_half_width(scales[s], Bw, R);
        if (L > mh) mh = L;
    }
    jb.max_half = mh;
    pthread_mutex_init(&jb.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads == 1) {
        who_worker(&jb);
    } else {
        pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * threads);
        for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, who_worker, &jb);
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
        free(th);
    }
    pthread_mutex_destroy(&jb.mu);
    if (norm == WHO_NORM_MINMAX && out_kind != WHO_OUT_COMPLEX)
        who_minmax(out, B, S * jb.frames);
    return 0;
}
