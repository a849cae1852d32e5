// wh_umma.cu -- tcgen05 (UMMA) engine: the hop-strided CWT as a polyphase GEMM on the
// 5th-generation tensor cores, split-fp16 (3 products) with fp32 accumulation in TMEM.
//
// Math (restating wavelet.py:215-273 / _kernels.py:28-62's polyphase identity):
//   the signal of one clip is viewed as rows of V samples (V = 64 when hop | 64, else
//   V = hop for hop % 64 == 0).  A frame at sample position m*V + r*hop (row m, phase
//   r = 0..P-1, P = V/hop) correlates with taps over offsets u in [-L, L]:
//       W(s, m*P + r) = sum_g X[m - Qlo + floor(g/V), g mod V] * B[g, (s, r)]
//   with B[g, (s, c, r)] = tap_{s,c}(g - Qlo*V - r*hop)  (c = re / im component).
//   X's rows for K-step k are X rows shifted by floor(64k/V): the whole window of a
//   128-row tile is converted ONCE into shared memory (fp32 -> hi/lo fp16, 128B
//   swizzle) and every K-step's A operand is the same buffer with its UMMA descriptor
//   start moved by q*128 B (tools/probe_umma_shift.cu verified the absolute-address
//   swizzle makes this exact).  The taps B are a constant bank, pre-swizzled in HBM
//   (L2-resident), streamed per K-step with cp.async.bulk.
//   Precision: x*2^e = xh + xl, t*2^f = th + tl (fp16 each); D += xh*th + xh*tl + xl*th
//   in fp32 (the dropped xl*tl term is ~2^-22 relative), then D * 2^-(e+f).
//
// CTA roles (256 threads, 1 CTA per SM, persistent over (clip, row-tile) items):
//   warp 0      producer: cp.async.bulk of tap tiles into a bstages-deep ring
//   warp 1      TMEM allocator + MMA issuer (one elected thread)
//   warps 2-3   converters: window max -> exponent -> hi/lo fp16 swizzled window
//   warps 4-7   epilogue: tcgen05.ld -> scale, |W| / log1p / ... -> global stores,
//               per-clip min/max atomics
#include <cuda_fp16.h>
#include <math.h>

#include <algorithm>
#include <cmath>

#include "wh_internal.h"

namespace wh {

static constexpr int UM_CONV_WARPS = 4;
static constexpr int UM_CONV_THREADS = 32 * UM_CONV_WARPS;
static constexpr int UM_THREADS = 64 + UM_CONV_THREADS + 128;  // producer, MMA, converters, epilogue
static constexpr int UM_MAX_STAGES = 6;
static constexpr int UM_SMEM_BUDGET = 227 * 1024 - 1024 - 256;

struct UmmaArgs {
    const float *x;
    int64_t ld_x, N, F, hop;
    int64_t items;              // clips * row_tiles
    int32_t row_tiles, V, P, Cc, panels, Qlo, win_rows, S;
    int32_t n_passes, n_tiles, wavelet, output, bstages, win_bufs, vec_ok;
    int32_t n_acc, acc_stride;          // accumulator buffers; columns per buffer (main|corr)
    int32_t use_stg;                    // fp32 window staged in smem by cp.async.bulk
    const UmmaPass *passes;
    const UmmaTile *tiles;
    const uint8_t *bank;
    const float *scale_pow;
    void *out;
    uint32_t *minmax;
    uint32_t stage_bytes, win_half_bytes;
    int32_t out_vec_ok;             // output base 16B aligned and F % 4 == 0
    unsigned long long *prof;       // optional per-role wait counters (wh_plan_profile)
};

// Wait-cycle counters (diagnostics): index = role * 4 + slot; slot 3 = total cycles.
enum { PR_PROD = 0, PR_MMA = 1, PR_CONV = 2, PR_EPI = 3 };
struct ProfAcc {
    unsigned long long c[4] = {0, 0, 0, 0};
    long long t0 = 0;
    __device__ __forceinline__ void start() { t0 = clock64(); }
};


// ---- PTX helpers -----------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity), "r"(1000000u)
            : "memory");
    }
}
__device__ __forceinline__ void mbar_wait_p(uint64_t *b, uint32_t parity, ProfAcc &pa, int slot,
                                            bool on) {
    if (!on) {
        mbar_wait(b, parity);
        return;
    }
    const long long t = clock64();
    mbar_wait(b, parity);
    pa.c[slot] += (unsigned long long)(clock64() - t);
}
__device__ __forceinline__ void prof_flush(const ProfAcc &pa, unsigned long long *prof, int role) {
    if (!prof) return;
    for (int i = 0; i < 3; ++i) atomicAdd(prof + role * 4 + i, pa.c[i]);
    atomicAdd(prof + role * 4 + 3, (unsigned long long)(clock64() - pa.t0));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzle smem matrix descriptor (SBO = 8 rows * 128 B).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ uint32_t idesc_f16(uint32_t n) {
    // D f32 (bit 4), A/B f16 (0), K-major A/B, N>>3 at [17,23), M>>4 at [24,29), M = 128
    return (1u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n.reg .pred P1;\nelect.sync _|P1, 0xffffffff;\nselp.b32 %0, 1, 0, P1;\n}\n" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}


__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, float (&va)[16], float (&vb)[16]) {
    uint32_t r[16], q[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
          "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
        : "r"(tb));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        va[i] = __uint_as_float(r[i]);
        vb[i] = __uint_as_float(q[i]);
    }
}

__device__ __forceinline__ float lg2_fast(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// scalogram.py:51-64 + BASELINE log1p, compile-time output kind (magnitude -> value)
template <int OUT>
__device__ __forceinline__ float out_value(float mag) {
    if constexpr (OUT == WH_OUT_POWER) return mag * mag;
    else if constexpr (OUT == WH_OUT_LOG_DB) return lg2_fast(mag + 1e-12f) * 6.0205999132796239f;  // 20*log10(2)
    else if constexpr (OUT == WH_OUT_LOG1P) return lg2_fast(1.0f + mag) * 0.69314718055994531f;
    else return mag;
}

// Store R consecutive frames (nvalid of them valid) of one scale row starting at element o.
template <int R, int CC, int OUT>
__device__ __forceinline__ void store_run(const UmmaArgs &A, int64_t o, int nvalid, const float (&re)[R],
                                          const float (&im)[R], bool vec, float &lmin, float &lmax) {
    if constexpr (OUT == WH_OUT_COMPLEX64) {
        float2 *dst = reinterpret_cast<float2 *>(A.out) + o;
        if (R % 2 == 0 && nvalid == R && vec) {
#pragma unroll
            for (int r = 0; r < R; r += 2)
                *reinterpret_cast<float4 *>(dst + r) = make_float4(re[r], im[r], re[(r + 1) % R], im[(r + 1) % R]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r < nvalid) dst[r] = make_float2(re[r], im[r]);
        }
    } else {
        float val[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float mag = (CC == 2) ? sqrtf(fmaf(re[r], re[r], im[r] * im[r])) : fabsf(re[r]);
            val[r] = out_value<OUT>(mag);
        }
        if (A.minmax) {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r < nvalid) {
                    lmin = fminf(lmin, val[r]);
                    lmax = fmaxf(lmax, val[r]);
                }
        }
        float *dst = reinterpret_cast<float *>(A.out) + o;
        if (R % 4 == 0 && nvalid == R && vec) {
#pragma unroll
            for (int r = 0; r < R; r += 4)
                *reinterpret_cast<float4 *>(dst + r) =
                    make_float4(val[r], val[(r + 1) % R], val[(r + 2) % R], val[(r + 3) % R]);
        } else if (R == 2 && nvalid == 2 && vec) {
            *reinterpret_cast<float2 *>(dst) = make_float2(val[0], val[1 % R]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r < nvalid) dst[r] = val[r];
        }
    }
}

// One accumulator buffer (a pass of ns scales) -> global, for this thread's row.
template <int CC, int P, int OUT>
__device__ __forceinline__ void epi_pass(const UmmaArgs &A, uint32_t tbase, uint32_t cbase, int s0, int ns,
                                         int cols, int64_t b, int64_t frame0, int nvalid, float e, bool vec,
                                         float &lmin, float &lmax) {
    constexpr int CP = CC * P;
    // NOTE: tcgen05.ld is warp-collective (.sync.aligned): every load below is executed by
    // all 32 lanes; only the stores depend on the lane's row (nvalid).
    const int64_t F = A.F;
    int64_t o = (b * A.S + s0) * F + frame0;  // element index of (scale s0, frame0)
    if constexpr (CP <= 16) {
        constexpr int SPU = 16 / CP;  // whole scales per 16-column unit
        for (int u0 = 0, sl0 = 0; u0 < cols; u0 += 16, sl0 += SPU) {
            float v[16], wr[16], w[16];
            tmem_ld16x2(tbase + u0, cbase - u0, v, wr);
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = wr[15 - i];
#pragma unroll
            for (int q = 0; q < SPU; ++q) {
                const int sl = sl0 + q;
                if (sl < ns && nvalid > 0) {
                    const float f = e * __ldg(A.scale_pow + s0 + sl);
                    float re[P], im[P];
#pragma unroll
                    for (int r = 0; r < P; ++r) {
                        re[r] = (v[q * CP + r] + w[q * CP + r]) * f;
                        im[r] = (CC == 2) ? (v[q * CP + (P + r) % CP] + w[q * CP + (P + r) % CP]) * f : 0.0f;
                    }
                    store_run<P, CC, OUT>(A, o + (int64_t)sl * F, nvalid, re, im, vec, lmin, lmax);
                }
            }
        }
    } else {
        // P >= 16: per scale, 16-phase chunks of re (and im)
        for (int sl = 0; sl < ns; ++sl) {
            const float f = e * __ldg(A.scale_pow + s0 + sl);
#pragma unroll 1
            for (int r0 = 0; r0 < P; r0 += 16) {
                float re[16], im[16], w[16];
                tmem_ld16x2(tbase + sl * CP + r0, cbase - (sl * CP + r0), re, w);
#pragma unroll
                for (int i = 0; i < 16; ++i) re[i] = (re[i] + w[15 - i]) * f;
                if constexpr (CC == 2) {
                    tmem_ld16x2(tbase + sl * CP + P + r0, cbase - (sl * CP + P + r0), im, w);
#pragma unroll
                    for (int i = 0; i < 16; ++i) im[i] = (im[i] + w[15 - i]) * f;
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) im[i] = 0.0f;
                }
                const int nv = nvalid - r0 < 16 ? nvalid - r0 : 16;
                if (nv > 0) store_run<16, CC, OUT>(A, o + (int64_t)sl * F + r0, nv, re, im, vec, lmin, lmax);
            }
        }
    }
}

// ---- the kernel --------------------------------------------------------------------------
template <int CC, int P>
__global__ void __launch_bounds__(UM_THREADS, 1) k_umma(const __grid_constant__ UmmaArgs A) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t b_full[UM_MAX_STAGES], b_empty[UM_MAX_STAGES];
    __shared__ __align__(8) uint64_t win_full[2], win_empty[2], acc_full[2], acc_empty[2];
    __shared__ float wexp[2], accexp[2];
    __shared__ float red[UM_CONV_WARPS];
    __shared__ __align__(8) uint64_t stg_full;
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t WH = A.win_half_bytes;               // bytes of one (hi or lo) window
    uint8_t *win_base = smem;                            // [win_bufs][hi|lo][panels][rows][128]
    uint8_t *stage_base = smem + (size_t)A.win_bufs * 2 * WH;
    const uint32_t panel_bytes = (uint32_t)A.win_rows * 128u;
    // pass / tile tables (compact) after the fp32 staging buffer
    int4 *s_pass = reinterpret_cast<int4 *>(stage_base + (size_t)A.bstages * A.stage_bytes +
                                            (A.use_stg ? 2 * (size_t)WH : 0));
    uint2 *s_tile = reinterpret_cast<uint2 *>(s_pass + A.n_passes);
    for (int i = threadIdx.x; i < A.n_passes; i += blockDim.x) {
        const UmmaPass ps = A.passes[i];
        s_pass[i] = make_int4(ps.tile_begin, ps.tile_end, ps.s0 | (ps.ns << 16), ps.cols);
    }
    for (int i = threadIdx.x; i < A.n_tiles; i += blockDim.x) {
        const UmmaTile tl = A.tiles[i];
        s_tile[i] = make_uint2((uint32_t)tl.k | ((uint32_t)tl.c0 << 16) | ((uint32_t)tl.ncols << 24),
                               (uint32_t)(tl.byte_off >> 8));
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < A.bstages; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&win_full[i], UM_CONV_WARPS);
            mbar_init(&win_empty[i], 1);
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 4);
        }
        mbar_init(&stg_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const bool pon = A.prof != nullptr;
    ProfAcc pa;
    pa.start();

    if (warp == 0) {
        // ===================== producer: tap tiles (whole warp, one elected lane) ====
        uint32_t st = 0, ph = 0;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            for (int p = 0; p < A.n_passes; ++p) {
                const int4 pinfo = s_pass[p];
                for (int t = pinfo.x; t < pinfo.y; ++t) {
                    const uint2 tt = s_tile[t];
                    const uint32_t ncols = tt.x >> 24;
                    mbar_wait_p(&b_empty[st], ph ^ 1, pa, 0, pon);
                    if (elect_one()) {
                        const uint32_t bytes = ncols * 384u;
                        mbar_expect_tx(&b_full[st], bytes);
                        bulk_g2s(stage_base + (size_t)st * A.stage_bytes, A.bank + ((size_t)tt.y << 8), bytes,
                                 &b_full[st]);
                    }
                    __syncwarp();
                    if (++st == (uint32_t)A.bstages) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (whole warp, one elected lane) =============
        uint32_t st = 0, ph = 0, wcnt = 0, acnt = 0;
        const uint32_t stage0 = smem_u32(stage_base);
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x, ++wcnt) {
            const uint32_t wb = wcnt % A.win_bufs;
            mbar_wait_p(&win_full[wb], (wcnt / A.win_bufs) & 1, pa, 0, pon);
            tc_fence_after();
            const float e = wexp[wb];
            const uint32_t a_hi = smem_u32(win_base) + wb * 2 * WH;
            const uint32_t a_lo = a_hi + WH;
            for (int p = 0; p < A.n_passes; ++p, ++acnt) {
                const int4 pinfo = s_pass[p];
                const uint32_t ab = acnt % A.n_acc;
                mbar_wait_p(&acc_empty[ab], ((acnt / A.n_acc) & 1) ^ 1, pa, 1, pon);
                tc_fence_after();
                if (lane == 0) accexp[ab] = e;
                const uint32_t d_acc = tmem + ab * (uint32_t)A.acc_stride;
                uint32_t prev_c0 = (uint32_t)pinfo.w;  // pass columns
                for (int t = pinfo.x; t < pinfo.y; ++t) {
                    const uint2 tt = s_tile[t];
                    const uint32_t k = tt.x & 0xffffu, c0 = (tt.x >> 16) & 0xffu, nc = tt.x >> 24;
                    const uint32_t kg = k * 64u;
                    const uint32_t aoff = ((kg % (uint32_t)A.V) >> 6) * panel_bytes + (kg / (uint32_t)A.V) * 128u;
                    const uint32_t bt = stage0 + st * A.stage_bytes;  // [hi fwd | lo rev | hi rev]
                    const uint32_t C = (uint32_t)pinfo.w;
                    const bool first = (t == pinfo.x);
                    const uint32_t nnew = first ? nc : (c0 < prev_c0 ? prev_c0 - c0 : 0u);
                    mbar_wait_p(&b_full[st], ph, pa, 2, pon);
                    tc_fence_after();
                    if (elect_one()) {
                        // D columns of a pass: main_j at d + j (j = 0..C-1), corr_j at d + 2C-1-j.
                        // MMA1: A_hi x [hi_c0..hi_C-1 | lo_C-1..lo_c0] -> [main_c0.. | ..corr_c0]
                        // MMA2: A_lo x [hi_C-1..hi_c0]               -> [corr_C-1 .. corr_c0]
                        const uint32_t d1 = d_acc + c0, d2 = d_acc + C;
                        const uint32_t b2 = bt + 2 * nc * 128u;
                        if (nnew == nc) {
                            umma_f16(d1, sdesc(a_hi + aoff), sdesc(bt), idesc_f16(2 * nc), 0u);
                        } else if (nnew > 0) {
                            // first touch of columns [c0, c0+nnew): main head and corr tail
                            umma_f16(d1, sdesc(a_hi + aoff), sdesc(bt), idesc_f16(nnew), 0u);
                            umma_f16(d1 + nnew, sdesc(a_hi + aoff), sdesc(bt + nnew * 128u),
                                     idesc_f16(2 * (nc - nnew)), 1u);
                            umma_f16(d1 + 2 * nc - nnew, sdesc(a_hi + aoff), sdesc(bt + (2 * nc - nnew) * 128u),
                                     idesc_f16(nnew), 0u);
                        } else {
                            umma_f16(d1, sdesc(a_hi + aoff), sdesc(bt), idesc_f16(2 * nc), 1u);
                        }
                        umma_f16(d2, sdesc(a_lo + aoff), sdesc(b2), idesc_f16(nc), 1u);
#pragma unroll
                        for (uint32_t j = 1; j < 4; ++j) {
                            umma_f16(d1, sdesc(a_hi + aoff + j * 32), sdesc(bt + j * 32), idesc_f16(2 * nc), 1u);
                            umma_f16(d2, sdesc(a_lo + aoff + j * 32), sdesc(b2 + j * 32), idesc_f16(nc), 1u);
                        }
                        umma_commit(&b_empty[st]);
                    }
                    __syncwarp();
                    if (c0 < prev_c0) prev_c0 = c0;
                    if (++st == (uint32_t)A.bstages) { st = 0; ph ^= 1; }
                }
                if (elect_one()) umma_commit(&acc_full[ab]);
                __syncwarp();
            }
            if (elect_one()) umma_commit(&win_empty[wb]);
            __syncwarp();
        }
    } else if (warp < 2 + UM_CONV_WARPS) {
        // ===================== converters ============================================
        // The fp32 window of item i is a contiguous sample range of the clip; one elected
        // converter thread bulk-copies it into the staging buffer one item ahead.
        const int ct = threadIdx.x - 64;  // 0 .. UM_CONV_THREADS-1
        const int cw = warp - 2;
        const int chunks = A.win_rows * A.panels * 8;  // 8-sample chunks in the window
        const int64_t wlen = (int64_t)A.win_rows * A.V;
        float *stg = reinterpret_cast<float *>(stage_base + (size_t)A.bstages * A.stage_bytes);
        // staged range [lo, hi) of the clip for an item (16-byte granular); rest read directly
        auto staged = [&](int64_t item, int64_t &lo, int64_t &hi) {
            const int64_t b = item / A.row_tiles, tile = item % A.row_tiles;
            const int64_t w0 = (tile * 128 - A.Qlo) * A.V;
            lo = w0 > 0 ? w0 : 0;
            hi = w0 + wlen < A.N ? w0 + wlen : (A.N & ~(int64_t)3);
            if (!A.vec_ok || !A.use_stg || hi <= lo) { lo = hi = w0; }
            (void)b;
        };
        auto issue = [&](int64_t item) {
            int64_t lo, hi;
            staged(item, lo, hi);
            const int64_t b = item / A.row_tiles, tile = item % A.row_tiles;
            const int64_t w0 = (tile * 128 - A.Qlo) * A.V;
            const uint32_t bytes = (uint32_t)((hi - lo) * 4);
            mbar_expect_tx(&stg_full, bytes);
            if (bytes) bulk_g2s(stg + (lo - w0), A.x + b * A.ld_x + lo, bytes, &stg_full);
        };
        if (A.use_stg && ct == 0 && (int64_t)blockIdx.x < A.items) issue(blockIdx.x);
        uint32_t wcnt = 0;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x, ++wcnt) {
            const int64_t b = item / A.row_tiles;
            const int64_t tile = item % A.row_tiles;
            const int64_t w0 = (tile * 128 - A.Qlo) * A.V;
            const float *xb = A.x + b * A.ld_x;
            const uint32_t wb = wcnt % A.win_bufs;
            int64_t slo, shi;
            staged(item, slo, shi);
            if (A.use_stg) mbar_wait_p(&stg_full, wcnt & 1, pa, 0, pon);
            // sample g of the window (clip index w0 + g): staged, direct (edge), or zero
            auto load8 = [&](int row, int panel, int c8, float (&v)[8]) {
                const int64_t off = (int64_t)row * A.V + panel * 64 + c8 * 8;
                const int64_t g0 = w0 + off;
                if (g0 >= slo && g0 + 8 <= shi) {
                    const float4 u = *reinterpret_cast<const float4 *>(stg + off);
                    const float4 w = *reinterpret_cast<const float4 *>(stg + off + 4);
                    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
                } else if (A.vec_ok && g0 >= 0 && g0 + 8 <= A.N) {
                    const float4 u = __ldg(reinterpret_cast<const float4 *>(xb + g0));
                    const float4 w = __ldg(reinterpret_cast<const float4 *>(xb + g0) + 1);
                    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int64_t g = g0 + i;
                        v[i] = (g >= 0 && g < A.N) ? ((g >= slo && g < shi) ? stg[off + i] : __ldg(xb + g)) : 0.0f;
                    }
                }
            };
            // pass 1: max |x| over the window
            float mx = 0.0f;
#pragma unroll 4
            for (int c = ct; c < chunks; c += UM_CONV_THREADS) {
                const int row = c / (A.panels * 8), rem = c % (A.panels * 8);
                float v[8];
                load8(row, rem >> 3, rem & 7, v);
#pragma unroll
                for (int i = 0; i < 8; ++i) mx = fmaxf(mx, fabsf(v[i]));
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (lane == 0) red[cw] = mx;
            asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
            mx = red[0];
#pragma unroll
            for (int i = 1; i < UM_CONV_WARPS; ++i) mx = fmaxf(mx, red[i]);
            int ex = 0;
            if (mx > 0.0f) {
                frexpf(mx, &ex);  // mx = m * 2^ex, m in [0.5, 1)
                ex = 14 - ex;     // mx * 2^ex in [2^13, 2^14)
            }
            const float sc = ldexpf(1.0f, ex);
            // wait until the MMAs that read this window buffer win_bufs items ago are done
            mbar_wait_p(&win_empty[wb], ((wcnt / A.win_bufs) & 1) ^ 1, pa, 1, pon);
            uint8_t *whi = win_base + (size_t)wb * 2 * WH;
            uint8_t *wlo = whi + WH;
            for (int c = ct; c < chunks; c += UM_CONV_THREADS) {
                const int row = c / (A.panels * 8), rem = c % (A.panels * 8);
                const int panel = rem >> 3, c8 = rem & 7;
                float v[8];
                load8(row, panel, c8, v);
                uint32_t hw[4], lw[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float a0 = v[2 * i] * sc, a1 = v[2 * i + 1] * sc;
                    const __half h0 = __float2half_rn(a0), h1 = __float2half_rn(a1);
                    const __half l0 = __float2half_rn(a0 - __half2float(h0));
                    const __half l1 = __float2half_rn(a1 - __half2float(h1));
                    hw[i] = pack_h2(h0, h1);
                    lw[i] = pack_h2(l0, l1);
                }
                const uint32_t off = (uint32_t)panel * panel_bytes + (uint32_t)row * 128u +
                                     (uint32_t)((c8 ^ (row & 7)) * 16);
                *reinterpret_cast<uint4 *>(whi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4 *>(wlo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (ct == 0) wexp[wb] = ldexpf(1.0f, -ex);
            asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
            // staging is free again: prefetch the next item's window
            if (A.use_stg && ct == 0 && item + gridDim.x < A.items) issue(item + gridDim.x);
            if (lane == 0) mbar_arrive(&win_full[wb]);
        }
    } else {
        // ===================== epilogue ==============================================
        const int quad = warp & 3;          // TMEM lanes 32*quad .. 32*quad+31
        const int m = quad * 32 + lane;     // row within the tile
        const bool vec = A.out_vec_ok;
        uint32_t acnt = 0;
        float lmin = INFINITY, lmax = -INFINITY;
        int64_t cur_b = -1;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            const int64_t b = item / A.row_tiles;
            const int64_t tile = item % A.row_tiles;
            const int64_t mrow = tile * 128 + m;  // global row
            const int64_t frame0 = mrow * P;      // first frame of this row
            const int64_t rem_frames = A.F - frame0;
            const int nvalid = rem_frames <= 0 ? 0 : (rem_frames >= P ? P : (int)rem_frames);
            if (A.minmax && b != cur_b) {
                if (cur_b >= 0) {
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) {
                        lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
                        lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
                    }
                    if (lane == 0 && lmin <= lmax) {
                        atomicMin(A.minmax + 2 * cur_b, f2key(lmin));
                        atomicMax(A.minmax + 2 * cur_b + 1, f2key(lmax));
                    }
                }
                lmin = INFINITY;
                lmax = -INFINITY;
                cur_b = b;
            }
            for (int p = 0; p < A.n_passes; ++p, ++acnt) {
                const int4 pinfo = s_pass[p];
                const uint32_t ab = acnt % A.n_acc;
                mbar_wait_p(&acc_full[ab], (acnt / A.n_acc) & 1, pa, 0, pon);
                tc_fence_after();
                const float e = accexp[ab];
                const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + ab * (uint32_t)A.acc_stride;
                // corr_j lives at column 2C-1-j: the 16 corr values of unit u0 are loaded
                // from cbase - u0 in reverse order
                const uint32_t cbase = tbase + 2u * (uint32_t)pinfo.w - 16u;
                const int s0 = pinfo.z & 0xffff, ns = pinfo.z >> 16;
                switch (A.output) {
                    case WH_OUT_COMPLEX64:
                        epi_pass<CC, P, WH_OUT_COMPLEX64>(A, tbase, cbase, s0, ns, pinfo.w, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    case WH_OUT_ABS:
                        epi_pass<CC, P, WH_OUT_ABS>(A, tbase, cbase, s0, ns, pinfo.w, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    case WH_OUT_POWER:
                        epi_pass<CC, P, WH_OUT_POWER>(A, tbase, cbase, s0, ns, pinfo.w, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    case WH_OUT_LOG_DB:
                        epi_pass<CC, P, WH_OUT_LOG_DB>(A, tbase, cbase, s0, ns, pinfo.w, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    default:
                        epi_pass<CC, P, WH_OUT_LOG1P>(A, tbase, cbase, s0, ns, pinfo.w, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[ab]);
            }
        }
        if (A.minmax && cur_b >= 0) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
                lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
            }
            if (lane == 0 && lmin <= lmax) {
                atomicMin(A.minmax + 2 * cur_b, f2key(lmin));
                atomicMax(A.minmax + 2 * cur_b + 1, f2key(lmax));
            }
        }
    }
    if (pon && lane == 0) {
        const int role = warp == 0 ? PR_PROD : warp == 1 ? PR_MMA : warp < 2 + UM_CONV_WARPS ? PR_CONV : PR_EPI;
        prof_flush(pa, A.prof, role);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ---- tap bank builder (plan time) ------------------------------------------------------
// One block per tile; writes the hi|lo fp16 image of B[64k .. 64k+63][c0 .. cols) in the
// K-major 128B-swizzled layout the UMMA descriptor expects (row n = column, 128 B = 64 K).
struct BankArgs {
    const UmmaPass *passes;
    const UmmaTile *tiles;
    int32_t n_passes;
    const double *scales;
    const int64_t *half;
    const int32_t *fexp;
    double C, Bw;
    int32_t P, Cc, G0;
    int64_t hop;
    uint8_t *bank;
};

__global__ void k_build_bank(BankArgs a) {
    const int t = blockIdx.x;
    // find the pass of this tile
    int p = 0;
    while (p + 1 < a.n_passes && a.passes[p + 1].tile_begin <= t) ++p;
    const UmmaPass ps = a.passes[p];
    const UmmaTile tl = a.tiles[t];
    const int CP = a.Cc * a.P;
    const int C = ps.cols;
    uint8_t *part0 = a.bank + tl.byte_off;                 // hi, columns c0 .. C-1
    uint8_t *part1 = part0 + (size_t)tl.ncols * 128;       // lo, columns C-1 .. c0
    uint8_t *part2 = part1 + (size_t)tl.ncols * 128;       // hi, columns C-1 .. c0
    const double norm = pow(M_PI * a.Bw, -0.5);
    const double w = 2.0 * M_PI * a.C;
    for (int idx = threadIdx.x; idx < tl.ncols * 64; idx += blockDim.x) {
        const int n = idx / 64, e = idx % 64;
        const int col = tl.c0 + n;
        double v = 0.0;
        if (col < ps.ns * CP) {
            const int s = ps.s0 + col / CP;
            const int c = (col / a.P) % a.Cc;
            const int r = col % a.P;
            const int64_t g = (int64_t)tl.k * 64 + e;
            const int64_t u = g - a.G0 - (int64_t)r * a.hop;
            const int64_t L = a.half[s];
            if (u >= -L && u <= L) {
                const double sa = a.scales[s];
                const double tt = (double)(u < 0 ? -u : u) / sa;   // taps are even/odd in u
                const double env = norm * exp(-(tt * tt) / a.Bw);
                const double th = w * tt;
                const double rs = sqrt(sa);
                if (c == 0) {
                    v = (env * cos(th)) / rs;
                } else {
                    v = (env * sin(th)) / rs;
                    if (u < 0) v = -v;
                }
                v = ldexp(v, a.fexp[s]);
            }
        }
        const __half h = __double2half(v);
        const __half l = __double2half(v - (double)__half2float(h));
        auto put = [&](uint8_t *base, int row, __half val) {
            const uint32_t off = (uint32_t)row * 128u + (uint32_t)((((e >> 3) ^ (row & 7)) << 4) + (e & 7) * 2);
            *reinterpret_cast<__half *>(base + off) = val;
        };
        const int rrev = C - 1 - col;  // row index in the reversed parts
        put(part0, n, h);
        put(part1, rrev, l);
        put(part2, rrev, h);
    }
}

using UmmaKernel = void (*)(const UmmaArgs);

template <int CC>
static UmmaKernel pick_p(int P) {
    switch (P) {
        case 1: return k_umma<CC, 1>;
        case 2: return k_umma<CC, 2>;
        case 4: return k_umma<CC, 4>;
        case 8: return k_umma<CC, 8>;
        case 16: return k_umma<CC, 16>;
        case 32: return k_umma<CC, 32>;
        case 64: return k_umma<CC, 64>;
        default: return nullptr;
    }
}

static UmmaKernel umma_kernel(int Cc, int P) { return Cc == 2 ? pick_p<2>(P) : pick_p<1>(P); }

int umma_supported(const Plan &p, std::string *why) {
    const int64_t H = p.hop;
    bool small = H <= 64 && 64 % H == 0;
    bool big = H % 64 == 0 && H <= 256;
    if (!small && !big) {
        if (why) *why = "hop must divide 64 or be a multiple of 64 up to 256";
        return WH_E_UNSUPPORTED;
    }
    const int64_t V = small ? 64 : H;
    const int64_t Qlo = (p.Lmax + V - 1) / V;
    const int64_t P = V / H;
    const int64_t maxg = Qlo * V + p.Lmax + (P - 1) * H;
    const int64_t ksteps = maxg / 64 + 1;
    const int64_t qmax = (ksteps - 1) * 64 / V;
    const int64_t rows = ((128 + qmax) + 7) / 8 * 8;
    const int64_t win = 2 * (V / 64) * rows * 128;
    // smallest configuration: one window (no staging), two 16-column stages (the planner
    // makes the final decision with the real stage size)
    if (win + 2 * 16 * 384 > UM_SMEM_BUDGET) {
        if (why) *why = "tap support too long for a resident shared-memory window";
        return WH_E_UNSUPPORTED;
    }
    if (p.S > 65535) {
        if (why) *why = "too many scales";
        return WH_E_UNSUPPORTED;
    }
    return WH_OK;
}

// compact smem tile format: k < 2^16, c0 and ncols < 2^8, byte_off multiple of 256
static int ncheck_tiles(const Plan &p) {
    for (auto &t : p.tiles)
        if (t.k >= 65536 || t.c0 > 255 || t.ncols > 255 || (t.byte_off & 255) || (t.byte_off >> 8) >= (1LL << 32))
            return fail(WH_E_UNSUPPORTED, "UMMA engine: tile table out of range");
    if (16 * p.passes.size() + 8 * p.tiles.size() > 32 * 1024)
        return fail(WH_E_UNSUPPORTED, "UMMA engine: tile table too large");
    return WH_OK;
}

int umma_prepare(Plan &p) {
    const int64_t H = p.hop;
    p.V = (int32_t)(H <= 64 ? 64 : H);
    p.P = (int32_t)(p.V / H);
    p.Cc = p.wavelet == WH_WAVELET_CMOR ? 2 : 1;
    p.panels = p.V / 64;
    p.Qlo = (int32_t)((p.Lmax + p.V - 1) / p.V);
    p.G0 = p.Qlo * p.V;
    const int64_t maxg = (int64_t)p.G0 + p.Lmax + (int64_t)(p.P - 1) * H;
    p.ksteps = (int32_t)(maxg / 64 + 1);
    const int64_t qmax = (int64_t)(p.ksteps - 1) * 64 / p.V;
    p.win_rows = (int32_t)(((128 + qmax) + 7) / 8 * 8);
    p.rows_total = (int32_t)((p.F + p.P - 1) / p.P);
    p.row_tiles = (p.rows_total + 127) / 128;
    const int64_t win = 2LL * p.panels * p.win_rows * 128;

    // per-scale exponent: max|tap| = (pi B)^-1/2 / sqrt(a) scaled into [2^13, 2^14)
    p.fexp.resize(p.S);
    std::vector<float> spow(p.S);
    for (int s = 0; s < p.S; ++s) {
        double mt = std::pow(M_PI * p.B, -0.5) / std::sqrt(p.scales[s]);
        int E = 0;
        std::frexp(mt, &E);
        p.fexp[s] = 14 - E;
        spow[s] = (float)std::ldexp(1.0, -p.fexp[s]);
    }

    const int CP = p.Cc * p.P;
    // TMEM: 512 columns = 2 accumulator buffers x (128 main + 128 correction) columns, so a
    // pass covers at most 128 columns and the epilogue of pass n overlaps the MMAs of n+1.
    const int max_cols = 128;
    p.n_acc = 2;
    p.acc_stride = 256;
    int win_bufs = 0, bstages = 0;
    // scales per pass: whole scales, cols = ns*CP rounded up to 16 (CP > 256 unsupported)
    if (CP > max_cols) return fail(WH_E_UNSUPPORTED, "UMMA engine: too many phases per scale");
    const int spp = std::max(1, max_cols / CP);
    p.passes.clear();
    p.tiles.clear();
    int64_t byte_off = 0;
    int max_tile_cols = 16;
    // heavy (long-tap) passes first so the accumulator pipeline starts on the long ones
    std::vector<std::pair<int, int>> ranges;
    for (int s0 = 0; s0 < p.S; s0 += spp) ranges.push_back({s0, std::min(spp, p.S - s0)});
    std::reverse(ranges.begin(), ranges.end());
    for (auto &rg : ranges) {
        UmmaPass ps{};
        ps.s0 = rg.first;
        ps.ns = rg.second;
        ps.cols = (ps.ns * CP + 15) / 16 * 16;
        ps.tile_begin = (int32_t)p.tiles.size();
        // column activity: column j = (scale, comp, phase) active on g in
        // [G0 - L + r*H, G0 + L + r*H]
        for (int k = 0; k < p.ksteps; ++k) {
            int c0 = ps.cols;
            for (int j = 0; j < ps.ns * CP; ++j) {
                const int s = ps.s0 + j / CP, r = j % p.P;
                const int64_t lo = p.G0 - p.half[s] + (int64_t)r * H;
                const int64_t hi = p.G0 + p.half[s] + (int64_t)r * H;
                if (hi >= (int64_t)k * 64 && lo <= (int64_t)k * 64 + 63) {
                    c0 = j;
                    break;
                }
            }
            if (c0 >= ps.ns * CP) continue;  // no active column on this K-step
            c0 = c0 / 16 * 16;
            UmmaTile tl{};
            tl.k = k;
            tl.c0 = c0;
            tl.ncols = ps.cols - c0;
            tl.byte_off = byte_off;
            byte_off += (int64_t)tl.ncols * 384;  // [hi fwd | lo rev | hi rev], 128 B rows
            max_tile_cols = std::max(max_tile_cols, tl.ncols);
            p.tiles.push_back(tl);
        }
        ps.tile_end = (int32_t)p.tiles.size();
        if (ps.tile_end > ps.tile_begin) p.passes.push_back(ps);
    }
    p.bank_bytes = byte_off;
    const int64_t stage_bytes = (int64_t)max_tile_cols * 384;
    const int64_t table_bytes = 16 * (int64_t)p.passes.size() + 8 * (int64_t)p.tiles.size();
    const int64_t budget = UM_SMEM_BUDGET - table_bytes;
    if (ncheck_tiles(p) != WH_OK) return WH_E_UNSUPPORTED;
    // smem = window buffers (hi|lo fp16) [+ fp32 staging, same bytes as one window] + tap
    // stages.  Preference: 2 windows + staging, 1 window + staging, 2 windows, 1 window.
    int use_stg = 0;
    {
        const int opts[4][2] = {{2, 1}, {1, 1}, {2, 0}, {1, 0}};
        for (auto &o : opts) {
            const int64_t fixed = (int64_t)(o[0] + o[1]) * win;
            if (fixed + 2 * stage_bytes <= budget) {
                win_bufs = o[0];
                use_stg = o[1];
                bstages = (int)std::min<int64_t>(4, (budget - fixed) / stage_bytes);
                break;
            }
        }
    }
    if (bstages < 2) return fail(WH_E_UNSUPPORTED, "UMMA engine: shared memory too small for 2 stages");
    p.win_bufs = win_bufs;
    p.bstages = bstages;
    p.use_stg = use_stg;
    p.smem_bytes = (size_t)((win_bufs + use_stg) * win + bstages * stage_bytes) + 1024 + table_bytes;

    WH_CUDA_TRY(cudaMalloc(&p.d_passes, sizeof(UmmaPass) * p.passes.size()));
    WH_CUDA_TRY(cudaMalloc(&p.d_tiles, sizeof(UmmaTile) * p.tiles.size()));
    WH_CUDA_TRY(cudaMalloc(&p.d_bank, (size_t)p.bank_bytes));
    WH_CUDA_TRY(cudaMalloc(&p.d_scale_pow, sizeof(float) * p.S));
    int32_t *d_fexp = nullptr;
    WH_CUDA_TRY(cudaMalloc(&d_fexp, sizeof(int32_t) * p.S));
    WH_CUDA_TRY(cudaMemcpy(p.d_passes, p.passes.data(), sizeof(UmmaPass) * p.passes.size(), cudaMemcpyHostToDevice));
    WH_CUDA_TRY(cudaMemcpy(p.d_tiles, p.tiles.data(), sizeof(UmmaTile) * p.tiles.size(), cudaMemcpyHostToDevice));
    WH_CUDA_TRY(cudaMemcpy(p.d_scale_pow, spow.data(), sizeof(float) * p.S, cudaMemcpyHostToDevice));
    WH_CUDA_TRY(cudaMemcpy(d_fexp, p.fexp.data(), sizeof(int32_t) * p.S, cudaMemcpyHostToDevice));
    BankArgs ba{};
    ba.passes = p.d_passes; ba.tiles = p.d_tiles; ba.n_passes = (int32_t)p.passes.size();
    ba.scales = p.d_scales; ba.half = p.d_half; ba.fexp = d_fexp; ba.C = p.C; ba.Bw = p.B;
    ba.P = p.P; ba.Cc = p.Cc; ba.G0 = p.G0; ba.hop = p.hop; ba.bank = p.d_bank;
    k_build_bank<<<(unsigned)p.tiles.size(), 256>>>(ba);
    WH_CUDA_TRY(cudaGetLastError());
    WH_CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(d_fexp);
    UmmaKernel kern = umma_kernel(p.Cc, p.P);
    if (!kern) return fail(WH_E_UNSUPPORTED, "UMMA engine: unsupported phase count");
    WH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes));
    return WH_OK;
}

int umma_launch(Plan &p, const float *x, int64_t clips, int64_t ld_x, void *out, cudaStream_t s) {
    UmmaArgs a{};
    a.x = x; a.ld_x = ld_x; a.N = p.N; a.F = p.F; a.hop = p.hop;
    a.items = clips * p.row_tiles;
    a.row_tiles = p.row_tiles; a.V = p.V; a.P = p.P; a.Cc = p.Cc; a.panels = p.panels;
    a.Qlo = p.Qlo; a.win_rows = p.win_rows; a.S = p.S;
    a.n_passes = (int32_t)p.passes.size(); a.n_tiles = (int32_t)p.tiles.size();
    a.wavelet = p.wavelet; a.output = p.output;
    a.bstages = p.bstages; a.win_bufs = p.win_bufs; a.n_acc = p.n_acc; a.acc_stride = p.acc_stride;
    a.use_stg = p.use_stg;
    a.vec_ok = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && (ld_x % 4 == 0);
    a.passes = p.d_passes; a.tiles = p.d_tiles; a.bank = p.d_bank; a.scale_pow = p.d_scale_pow;
    a.out = out;
    a.minmax = p.norm == WH_NORM_MINMAX ? p.d_minmax : nullptr;
    int max_cols = 16;
    for (auto &t : p.tiles) max_cols = std::max(max_cols, t.ncols);
    a.stage_bytes = (uint32_t)max_cols * 384u;
    a.win_half_bytes = (uint32_t)p.panels * (uint32_t)p.win_rows * 128u;
    const int64_t grid = std::min<int64_t>(a.items, p.sms);
    a.out_vec_ok = ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && (p.F % 4 == 0);
    a.prof = p.d_prof;
    (void)cudaGetLastError();  // drop stale non-sticky errors of earlier runtime calls
    umma_kernel(p.Cc, p.P)<<<(unsigned)grid, UM_THREADS, p.smem_bytes, s>>>(a);
    WH_CUDA_TRY(cudaGetLastError());
    return WH_OK;
}

}  // namespace wh
