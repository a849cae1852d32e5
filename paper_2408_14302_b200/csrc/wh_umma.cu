// wh_umma.cu -- tcgen05 (UMMA) engine: the hop-strided CWT as a polyphase GEMM on the
// 5th-generation tensor cores, split-fp16 (3 products) with fp32 accumulation in TMEM.
//
// Math (restating wavelet.py:215-273 / _kernels.py:28-62's polyphase identity):
//   the signal of one clip is viewed as rows of V samples (V = 64 when hop | 64, else
//   V = hop for hop % 64 == 0).  Frame (row m, phase r = 0..P-1, P = V/hop) sits at sample
//   m*V + r*hop and correlates with taps over offsets u in [-L, L].  With the K index
//   g = u + G0 (G0 = Lmax rounded up to 4):
//       W(s, m*P + r) = sum_g x[m*V - G0 + g] * B[g, (s, c, r)],
//       B[g, (s, c, r)] = tap_{s,c}(g - G0 - r*hop)        (c = re / im component)
//   and x[m*V - G0 + g] = X[m + floor(g/V), g mod V] for the window X of rows of V samples
//   starting at sample tile*128*V - G0.  K-step k's A operand is that window shifted by
//   floor(64k/V) rows: the window of a 128-row tile is converted ONCE into shared memory
//   (fp32 -> hi/lo fp16, 128 B swizzle) and every K-step's UMMA descriptor start moves by
//   q*128 B (tools/probe_umma_shift.cu verified the absolute-address swizzle makes this
//   exact).  The taps B are a constant bank, pre-swizzled on the device at plan time:
//   resident in shared memory when it fits, else streamed per tap group with cp.async.bulk.
//   Precision: x*2^e = xh + xl, t*2^f = th + tl (fp16 each); main += xh*th and, in a
//   separate accumulator, corr += xh*tl + xl*th (fp32, TMEM); the cross terms are skipped
//   on tap tails below 2^-7 of the scale's peak; W = (main + corr) * 2^-(e+f).
//
// CTA roles (512 threads, 1 CTA per SM, CTA pairs (cta_group::2, M = 256), persistent over
// units = (clip, pair of 128-row tiles, group of passes)):
//   warp 0      producer: cp.async.bulk of the resident bank / streamed tap groups
//   warp 1      leader CTA: TMEM allocator + MMA issuer (one elected thread);
//               peer CTA: relays "tap group landed" to the leader's barriers
//   warps 2-7   converters: window -> registers -> max -> exponent -> hi/lo fp16, stored
//               swizzled once the window buffer is free
//   warps 8-15  epilogue (2 per TMEM lane quadrant): tcgen05.ld main + corr -> scale,
//               |W| / power / log_db / log1p -> 16-byte global stores, per-clip min/max
//
// Kernel variants k_umma<CC, P, CG, VS>: VS = 0 the common engine; 1 panel streaming (rows of
// hop samples for hops >= 256: fp16 split with a pre-pass, or tf32 operands fetched by TMA
// tensor copies); 2 the opt-in per-clip min-max arrival modes; 3 very long filters (two
// accumulator sets per TMEM buffer).  Each variant's extra code is compiled only there.
#include <cuda.h>  // CUtensorMap (the encoder is fetched through cudaGetDriverEntryPoint: no libcuda link)
#include <cuda_fp16.h>
#include <math.h>

#include <algorithm>
#include <numeric>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "wh_internal.h"

namespace wh {

// converter warps: 6 (16 warps in all: 4 per SM sub-partition, so 128 registers per thread)
// -- 6 warps keep more window loads in flight than 4 (c2 68.5 -> 64.4 us, c4 hop 64
// 228 -> 208 us, hop 256 / 1024 225 -> 205 us, c5 -1 %; profiles/r02h_ab.txt); 8 warps would
// cap registers at 96 and spill
#ifndef WH_CONV_WARPS
#define WH_CONV_WARPS 6
#endif
static constexpr int UM_CONV_WARPS = WH_CONV_WARPS;
static constexpr int UM_CONV_THREADS = 32 * UM_CONV_WARPS;
static constexpr int UM_EPI_WARPS = 8;  // 2 per TMEM lane quadrant
static constexpr int UM_THREADS = 64 + UM_CONV_THREADS + 32 * UM_EPI_WARPS;  // producer, MMA, converters, epilogue
static constexpr int UM_SLOTS = 16;  // in-flight tap tiles (ring slots)
static constexpr int UM_PF = 2;     // converters prefetch windows this many units ahead (L2)
static constexpr int UM_PCH = (36 + UM_CONV_WARPS - 1) / UM_CONV_WARPS;  // panel streaming: chunks per converter thread and panel
static constexpr int UM_CONV_RC = 40 / UM_CONV_WARPS;  // register-prefetch converters: chunks per thread
static constexpr int UM_WSLOTS = 4; // window buffers (panel streaming: panel slots; otherwise <= 2 used)
static constexpr int UM_SMEM_BUDGET = 227 * 1024 - 1024 - 256;
// Accuracy bounds on the longest filter's half width (taps): the tensor core's fp32 accumulate
// truncates, so the row error grows with the MMAs accumulated into one TMEM accumulator, about
// 2.5e-8 of the row peak per K = 16 step (measured: half width 2,661 -> 6.2e-6, 3,990 ->
// 1.0e-5, 5,322 -> 1.3e-5).  Up to UM_LMAX1 one accumulator set; up to UM_LMAX2 two sets per
// buffer that the epilogue adds (kernel variant 3, passes of 64 columns: 3,990 -> 5.0e-6,
// 5,322 -> 6.2e-6, 6,651 -> 1.0e-5); beyond: SIMT engine.
static constexpr int64_t UM_LMAX1 = 3360, UM_LMAX2 = 5632;

// Diagnostics (role switches, per-role wait counters, the CTA-0 timeline) exist only in a
// build with -DWH_DIAG (paper_2408_14302_b200/build.py --diag); the product build compiles
// them out of the kernel.
#ifdef WH_DIAG
static constexpr bool kDiag = true;
#define WH_DBG(bit) ((A.dbg & (bit)) != 0)
#else
static constexpr bool kDiag = false;
#define WH_DBG(bit) false
#endif

struct UmmaArgs {
    // tf32 panel streaming: the batch as a 3-D tensor (V samples, N / V rows, clips) for TMA box
    // copies of one 32-sample column panel of a window (128 B x win_rows rows, 128 B swizzle)
    alignas(64) CUtensorMap tmap;
    const float *x;
    int64_t ld_x, N, F, hop;
    int64_t clips;
    int32_t row_tiles, V, P, Cc, panels, G0, win_rows, S;
    int32_t rs;                         // rows per frame (hop = 256 * rs > 256), else 1
    int32_t n_passes, n_tiles, wavelet, output, win_bufs, vec_ok;
    int32_t pgroups, ppu;               // a unit = (clip, tile pair, group of ppu passes); pgroups groups
    int32_t n_acc, acc_stride;          // accumulator buffers; columns per buffer (main|corr)
    int32_t use_stg;                    // fp32 window staged in smem by cp.async.bulk
    int32_t resident;                   // some tap groups live in smem for the whole kernel
    uint32_t res_bytes;                 // bytes of the resident region at the stage base
    int32_t n_stream;                   // tap groups streamed through the ring every unit
    int32_t cpr, cpr_magic;             // 8-sample chunks per window row (panels * 8); ceil(2^20 / cpr)
    int32_t conv_regs;                  // converters prefetch the window into registers
    int32_t pf;                         // converters prefetch windows into L2 ahead (rows of 256)
    int32_t pstream;                    // rows of hop samples, the window streamed by 64-sample column panel
    int32_t tf32;                       // pstream with tf32 operands: 32-sample panels split in place, no exponent
    int32_t acc2;                       // tf32: two accumulator sets per buffer (even / odd K-slices), added by the epilogue
    int32_t tma;                        // tf32: panels fetched by one TMA tensor copy each (tmap), else by cp.async
    int64_t full_end;                   // tma: samples of a clip covered by whole rows of V ((N / V) * V)
    const UmmaPass *passes;
    const UmmaTile *tiles;
    const UmmaGroup *groups;
    int32_t n_groups;
    const uint8_t *bank;
    const float *scale_pow;
    const uint8_t *tables;          // packed smem tables (pass, group, tile, goff, spow), 16 B multiple
    uint32_t tables_bytes;
    void *out;
    uint32_t *minmax;
    uint32_t *arrive;               // write-once min-max: per-clip unit arrivals (nullptr: none)
    uint32_t arrive_target;         // arrivals that complete a clip (CTAs x tile pairs x pass groups)
    uint32_t *abandon;              // per clip ab_words words: units left to k_minmax_fixup
    int32_t ab_words;               // bit ((tile pair * pgroups + pass group) * CG + CTA rank)
    int32_t force_fixup;            // planner override (tests): every unit goes to the fix-up
    int32_t arrive_only;            // concurrent normaliser (min-max mode 2): count arrivals, normalise nothing
    uint32_t *nfbad;                // non-finite samples: per clip [1 + WH_NF_CAP] records
    uint32_t *nfctl;                // [0] CTAs done (the last one runs the fix-up), [1] any recorded
    const double *scales;           // for the fix-up's exact taps
    const int64_t *half;
    double Cw, Bw;
    uint32_t ring_bytes, win_half_bytes;
    int32_t out_vec_ok;             // output base 16B aligned and F % 4 == 0
    int32_t out_vec8_ok;            // output base 32B aligned and F % 8 == 0 (256-bit stores)
    unsigned long long *prof;       // optional per-role wait counters (wh_plan_profile)
    int32_t dbg;                    // diagnostics (WH_UMMA_DBG bits, results invalid): 1 no epilogue work,
                                    // 2 no converter work, 4 no MMA, 8 cluster-scope window release,
                                    // 32 no output values or stores, 64 no accumulator re-zeroing, 2048 no store instructions,
                                    // 128 no streamed tap copies after the first unit
    long long *trace;               // diagnostics: CTA-0 timeline [event][unit] (WH_UMMA_TRACE)
};

// Wait-cycle counters (diagnostics): index = role * 4 + slot; slot 3 = total cycles.
enum { PR_PROD = 0, PR_MMA = 1, PR_CONV = 2, PR_EPI = 3, PR_RELAY = 4 };
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
#ifdef WH_WAIT_HINT
    // suspend-time hint (ns): the waiting thread sleeps until the phase completes or the hint
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity), "r"((uint32_t)WH_WAIT_HINT)
            : "memory");
    }
#else
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    }
#endif
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
// diagnostics timeline (CTA 0 only): event e of unit u
#define WH_TRACE(e, u)                                                                      \
    do {                                                                                    \
        if (kDiag && A.trace && blockIdx.x == 0 && (u) < 32 && lane == 0) A.trace[(e) * 32 + (u)] = clock64(); \
    } while (0)

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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128B-swizzle smem matrix descriptor (SBO = 8 rows * 128 B).
// high word of every smem descriptor: SBO = 1024 B (8-row atoms), version 1, 128 B swizzle
static constexpr uint64_t DESC_HI = ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
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

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
template <int CG>
__device__ __forceinline__ void cta_pair_sync() {
    if constexpr (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
}
// relaxed remote arrive (tap-tile relay: the data was written by the async proxy and its
// local completion was observed by the relay's wait)
__device__ __forceinline__ void mbar_arrive_leader_relaxed(uint64_t *b) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(b)));
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// arrive on the leader's barrier after this CTA's own shared-memory writes: release at CTA
// scope (MEMBAR.CTA) -- the writes target this CTA's shared memory, which the pair's MMA
// reads in place, so they are performed once they are ordered at CTA scope.  The cluster-
// scope release (MEMBAR.GPU, ~1k cycles) is kept for diagnostics (WH_UMMA_DBG & 8).
__device__ __forceinline__ void mbar_arrive_leader_cta(uint64_t *b) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(b)));
    asm volatile("mbarrier.arrive.release.cta.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// arrive on the barrier at the same smem offset in the leader CTA (rank 0) of the pair
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *b) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(b)));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tmem_st16_zero(uint32_t taddr) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(0u)
        : "memory");
}
template <int CG>
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
    // accumulate always: the epilogue re-zeroes every accumulator buffer it drains
    if constexpr (CG == 2)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem), "l"(a), "l"(b),
                     "r"(idesc), "r"(1u));
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem), "l"(a), "l"(b),
                     "r"(idesc), "r"(1u));
}
// tf32 operands (fp32 words in shared memory, K = 8 per instruction = 32 B of a 128 B row)
template <int CG>
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
    if constexpr (CG == 2)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem), "l"(a), "l"(b),
                     "r"(idesc), "r"(1u));
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem), "l"(a), "l"(b),
                     "r"(idesc), "r"(1u));
}
template <int CG>
__device__ __forceinline__ uint32_t idesc_f16(uint32_t n) {
    // D f32 (bit 4), A/B f16 (0), K-major A/B, N>>3 at [17,23), M>>4 at [24,29), M = 128*CG
    return (1u << 4) | ((n >> 3) << 17) | (((128u * CG) >> 4) << 24);
}
template <int CG>
__device__ __forceinline__ void umma_commit(uint64_t *b) {
    if constexpr (CG == 2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(b)),
            "h"((uint16_t)3)
            : "memory");
    else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
                     : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int lane_id() { return (int)(threadIdx.x & 31); }
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

// two 32-column TMEM loads (this warp's 32 lanes) and one wait: main columns [ta, ta+32) and
// the matching correction columns [tb, tb+32)
__device__ __forceinline__ void tmem_ld32x2(uint32_t ta, uint32_t tb, float (&va)[32], float (&vb)[32]) {
    uint32_t r[32], q[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n"
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]), "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15]), "=r"(q[16]), "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]), "=r"(q[24]), "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
        : "r"(ta), "r"(tb)
        : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        va[i] = __uint_as_float(r[i]);
        vb[i] = __uint_as_float(q[i]);
    }
}
__device__ __forceinline__ void tmem_st32_zero(uint32_t taddr) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(0u)
        : "memory");
}

__device__ __forceinline__ float lg2_fast(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// scalogram.py:51-64 + BASELINE log1p, compile-time output kind (magnitude -> value)
// sqrt by the special-function unit (one MUFU instead of the IEEE sequence with its slow-path
// call: ~10 instructions per magnitude in the epilogue; relative error < 2^-22, far inside the
// 1e-5 row tolerance; the argument is in the accumulators' scale, never subnormal unless 0)
__device__ __forceinline__ float sqrt_fast(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
template <int OUT>
__device__ __forceinline__ float out_value(float mag) {
    if constexpr (OUT == WH_OUT_POWER) return mag * mag;
    else if constexpr (OUT == WH_OUT_LOG_DB) return lg2_fast(mag + 1e-12f) * 6.0205999132796239f;  // 20*log10(2)
    else if constexpr (OUT == WH_OUT_LOG1P) return lg2_fast(1.0f + mag) * 0.69314718055994531f;
    else return mag;
}

// Output stores bypass L1 allocation: the scalogram is written once and never re-read by
// this kernel, and plain L1-allocating stores were measured to slow the concurrent UMMA
// operand reads (shared memory and L1 share the SM's data SRAM).
__device__ __forceinline__ void st_na(float *p, float v) {
    asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_na(float2 *p, float2 v) {
    asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_na(float4 *p, float4 v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ void st_na8(float *p, const float *v) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
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
                st_na(reinterpret_cast<float4 *>(dst + r), make_float4(re[r], im[r], re[(r + 1) % R], im[(r + 1) % R]));
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r < nvalid) st_na(dst + r, make_float2(re[r], im[r]));
        }
    } else {
        float val[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const float mag = (CC == 2) ? cabs_scaled(re[r], im[r]) : fabsf(re[r]);
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
        if (R % 8 == 0 && nvalid == R && vec && A.out_vec8_ok) {
            // 32 bytes per lane: whole sectors, half the store transactions of 16-byte stores
            // (lanes of a warp hold different rows: every lane's piece is its own transaction)
#pragma unroll
            for (int r = 0; r < R; r += 8) st_na8(dst + r, val + (r % R));
        } else if (R % 4 == 0 && nvalid == R && vec) {
#pragma unroll
            for (int r = 0; r < R; r += 4)
                st_na(reinterpret_cast<float4 *>(dst + r),
                      make_float4(val[r], val[(r + 1) % R], val[(r + 2) % R], val[(r + 3) % R]));
        } else if (R == 2 && nvalid == 2 && vec) {
            st_na(reinterpret_cast<float2 *>(dst), make_float2(val[0], val[1 % R]));
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r < nvalid) st_na(dst + r, val[r]);
        }
    }
}

// One accumulator buffer (a pass of ns scales) -> global, for this thread's row.  The two
// epilogue warps of a TMEM lane quadrant split the 16-column units (half = 0 / 1); each
// re-zeroes the main and correction columns it has read.
template <int CC, int P, int OUT, int PS>
__device__ __forceinline__ void epi_pass(const UmmaArgs &A, const float *spow, uint32_t tbase, uint32_t cbase,
                                         int s0, int ns, int cols, int half, int64_t b, int64_t frame0,
                                         int nvalid, float e, bool vec, float &lmin, float &lmax) {
    constexpr int CP = CC * P;
    // NOTE: tcgen05.ld/st are warp-collective (.sync.aligned): every TMEM access below is
    // executed by all 32 lanes; only the global stores depend on the lane's row (nvalid).
    const int64_t F = A.F;
    const int64_t o0 = (b * A.S + s0) * F + frame0;  // element index of (scale s0, frame0)
    if constexpr (CP <= 16) {
        constexpr int SPU = 16 / CP;  // whole scales per 16-column unit
        for (int u0 = 16 * half; u0 < cols; u0 += 32) {
            const int sl0 = u0 / CP;
            float v[16], wr[16];
            tmem_ld16x2(tbase + u0, cbase - u0, v, wr);
            if (!WH_DBG(64)) {  // diagnostics: 64 = skip the re-zeroing (results invalid)
                tmem_st16_zero(tbase + u0);
                tmem_st16_zero(cbase - u0);
            }
            if (PS && A.acc2) {  // second accumulator set (odd K-slices), 128 columns on
                float v2[16], w2[16];
                tmem_ld16x2(tbase + 128u + u0, cbase + 128u - u0, v2, w2);
                tmem_st16_zero(tbase + 128u + u0);
                tmem_st16_zero(cbase + 128u - u0);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    v[i] += v2[i];
                    wr[i] += w2[i];
                }
            }
            if (WH_DBG(32)) continue;  // diagnostics: 32 = skip the stores
            if constexpr ((P == 1 || P == 2) && OUT != WH_OUT_COMPLEX64) if (A.rs == 1) {
                // P = 1: one frame per lane -- transpose 4x4 blocks inside each lane quad (two
                // xor-shuffle stages); P = 2: two frames per lane -- swap halves inside each
                // lane pair.  Either way every lane then stores 4 consecutive frames of one
                // scale with one 16-byte store: a quarter (half) of the store requests of
                // per-lane scalar (8-byte) stores, which compete with the UMMA operand reads
                // for the SM's data path.
                const int li = lane_id();
                // per-scale factors of the SPU scales of this unit (s0 + sl0 is a multiple of
                // 4 and s_spow 16-byte aligned): SPU/4 vector loads; scales >= ns contribute 0
                float f[SPU];
#pragma unroll
                for (int q = 0; q < SPU; q += 4) {
                    const float4 sp = *reinterpret_cast<const float4 *>(spow + s0 + sl0 + q);
                    f[q] = e * sp.x; f[q + 1] = e * sp.y; f[q + 2] = e * sp.z; f[q + 3] = e * sp.w;
                }
                if (sl0 + SPU > ns) {
#pragma unroll
                    for (int q = 0; q < SPU; ++q)
                        if (sl0 + q >= ns) f[q] = 0.0f;
                }
                float val[SPU][P];
#pragma unroll
                for (int q = 0; q < SPU; ++q) {
#pragma unroll
                    for (int r = 0; r < P; ++r) {
                        // |W| from the accumulators' own scale (|acc| < 2^45: the squares neither
                        // overflow nor underflow whatever the clip's amplitude), then the
                        // power-of-two factor 2^-(e+f): the same bits as scaling re / im first
                        // wherever those squares are representable
                        const float xs = v[q * CP + r] + wr[15 - (q * CP + r)];
                        float mag;
                        if constexpr (CC == 2) {
                            const float ys = v[q * CP + P + r] + wr[15 - (q * CP + P + r)];
                            mag = sqrt_fast(fmaf(xs, xs, ys * ys)) * f[q];
                        } else {
                            mag = fabsf(xs * f[q]);
                        }
                        val[q][r] = out_value<OUT>(mag);
                    }
                }
                if (A.minmax) {
                    if (sl0 + SPU <= ns && nvalid == P) {  // every value counts: no predicates
#pragma unroll
                        for (int q = 0; q < SPU; ++q)
#pragma unroll
                            for (int r = 0; r < P; ++r) {
                                lmin = fminf(lmin, val[q][r]);
                                lmax = fmaxf(lmax, val[q][r]);
                            }
                    } else {
#pragma unroll
                        for (int q = 0; q < SPU; ++q)
#pragma unroll
                            for (int r = 0; r < P; ++r)
                                if (sl0 + q < ns && r < nvalid) {
                                    lmin = fminf(lmin, val[q][r]);
                                    lmax = fmaxf(lmax, val[q][r]);
                                }
                    }
                }
                constexpr int LPG = 4 / P;  // lanes per 4-frame group (4 or 2)
                const int gi = li & (LPG - 1);
                const int64_t fq = frame0 - (int64_t)gi * P;  // first frame of the lane group
                const int nq = (int)(F - fq < 4 ? (F - fq > 0 ? F - fq : 0) : 4);
                const bool st4 = nq == 4 && vec;
                // this lane's scale for store group g is sl0 + LPG*g + gi: one row pointer,
                // advanced by LPG rows per group
                float *dst = reinterpret_cast<float *>(A.out) + (b * A.S + s0 + sl0 + gi) * F + fq;
                const int64_t gstep = (int64_t)LPG * F;
#pragma unroll
                for (int g = 0; g < SPU / LPG; ++g, dst += gstep) {
                    float t[4];
                    if constexpr (P == 1) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) t[k] = val[4 * g + k][0];
#pragma unroll
                        for (int k = 0; k < 2; ++k) {  // exchange the off-diagonal 2x2 blocks
                            const float s = (gi & 2) ? t[k] : t[2 + k];
                            const float x = __shfl_xor_sync(0xffffffffu, s, 2);
                            if (gi & 2) t[k] = x;
                            else t[2 + k] = x;
                        }
#pragma unroll
                        for (int k = 0; k < 4; k += 2) {  // transpose the 2x2 blocks
                            const float s = (gi & 1) ? t[k] : t[k + 1];
                            const float x = __shfl_xor_sync(0xffffffffu, s, 1);
                            if (gi & 1) t[k] = x;
                            else t[k + 1] = x;
                        }
                    } else {
                        // even lane keeps scale 2g (frames fq, fq+1 own, fq+2, fq+3 from the
                        // odd lane), odd lane keeps scale 2g+1
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            const float s = gi ? val[2 * g][k] : val[2 * g + 1][k];
                            const float x = __shfl_xor_sync(0xffffffffu, s, 1);
                            if (gi) {
                                t[k] = x;
                                t[2 + k] = val[2 * g + 1][k];
                            } else {
                                t[k] = val[2 * g][k];
                                t[2 + k] = x;
                            }
                        }
                    }
                    if (WH_DBG(2048)) {  // diagnostics: everything but the store instruction
                        if (t[0] + t[1] + t[2] + t[3] == 12345.678f) lmin = 0.0f;
                    } else if (sl0 + LPG * g + gi < ns) {
                        if (st4) {
                            st_na(reinterpret_cast<float4 *>(dst), make_float4(t[0], t[1], t[2], t[3]));
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (j < nq) st_na(dst + j, t[j]);
                        }
                    }
                }
                continue;
            }
            if (nvalid <= 0) continue;
            float re[SPU][P], im[SPU][P];
#pragma unroll
            for (int q = 0; q < SPU; ++q) {
                const float f = (sl0 + q < ns) ? e * spow[s0 + sl0 + q] : 0.0f;
#pragma unroll
                for (int r = 0; r < P; ++r) {
                    re[q][r] = (v[q * CP + r] + wr[15 - (q * CP + r)]) * f;
                    if constexpr (CC == 2)
                        im[q][r] = (v[q * CP + P + r] + wr[15 - (q * CP + P + r)]) * f;
                    else
                        im[q][r] = 0.0f;
                }
            }
            const bool full = (sl0 + SPU <= ns);
#pragma unroll
            for (int q = 0; q < SPU; ++q)
                if (full || sl0 + q < ns)
                    store_run<P, CC, OUT>(A, o0 + (int64_t)(sl0 + q) * F, nvalid, re[q], im[q], vec, lmin, lmax);
        }
    } else {
        // P >= 16: per scale, 16-phase chunks of re (and im); the two warps take alternate scales
        if constexpr (CC == 1 && P % 32 == 0 && OUT != WH_OUT_COMPLEX64) if (vec && A.out_vec8_ok) {
            // Real outputs, P = 32 / 64 (hop 2 / 1): a lane holds 32 consecutive frames of
            // its row; a 4 x 4 transpose of 8-frame blocks inside each lane quad gives every
            // lane 8 frames of each of the quad's 4 rows, so one 32-byte store per lane writes
            // whole 128-byte lines (4 lanes per line): a quarter of the store transactions of
            // per-row stores, which bound the hop-1 epilogue.
            const int gi = lane_id() & 3;
            const int64_t qf0 = frame0 - (int64_t)gi * P;  // first frame of the quad's first row
            for (int sl = half; sl < ns; sl += 2) {
                const float f = e * spow[s0 + sl];
                float *rowbase = reinterpret_cast<float *>(A.out) + (b * A.S + s0 + sl) * F;
#pragma unroll 1
                for (int r0 = 0; r0 < P; r0 += 32) {
                    float t[4][8];
                    {
                        // main columns u0 .. u0+31 and their correction columns (stored reversed
                        // at 2C-1-j: one 32-column range ending at cbase + 16 - u0)
                        const uint32_t u0 = (uint32_t)(sl * CP + r0);
                        float re[32], w[32];
                        tmem_ld32x2(tbase + u0, cbase - 16u - u0, re, w);
                        tmem_st32_zero(tbase + u0);
                        tmem_st32_zero(cbase - 16u - u0);
#pragma unroll
                        for (int i = 0; i < 32; ++i) t[i / 8][i % 8] = out_value<OUT>(fabsf((re[i] + w[31 - i]) * f));
                    }
                    if (A.minmax) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                if (r0 + 8 * k + i < nvalid) {
                                    lmin = fminf(lmin, t[k][i]);
                                    lmax = fmaxf(lmax, t[k][i]);
                                }
                    }
#pragma unroll
                    for (int k = 0; k < 2; ++k)  // exchange the off-diagonal 2 x 2 block quadrants
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float v = (gi & 2) ? t[k][i] : t[2 + k][i];
                            const float x = __shfl_xor_sync(0xffffffffu, v, 2);
                            if (gi & 2) t[k][i] = x;
                            else t[2 + k][i] = x;
                        }
#pragma unroll
                    for (int k = 0; k < 4; k += 2)  // transpose the 2 x 2 blocks
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float v = (gi & 1) ? t[k][i] : t[k + 1][i];
                            const float x = __shfl_xor_sync(0xffffffffu, v, 1);
                            if (gi & 1) t[k][i] = x;
                            else t[k + 1][i] = x;
                        }
                    // t[j] = frames r0 + 8 gi .. + 7 of the quad's row j
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int64_t fr = qf0 + (int64_t)j * P + r0 + 8 * gi;
                        float *dst = rowbase + fr;
                        if (F - fr >= 8) {
                            st_na8(dst, t[j]);
                        } else {
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                if (i < F - fr) st_na(dst + i, t[j][i]);
                        }
                    }
                }
            }
            if (half == 0)
                for (int c = ns * CP; c < cols; c += 16) {
                    tmem_st16_zero(tbase + c);
                    tmem_st16_zero(cbase - c);
                }
            return;
        }
        for (int sl = half; sl < ns; sl += 2) {
            const float f = e * spow[s0 + sl];
#pragma unroll 1
            for (int r0 = 0; r0 < P; r0 += 16) {
                float re[16], im[16], w[16];
                tmem_ld16x2(tbase + sl * CP + r0, cbase - (sl * CP + r0), re, w);
                tmem_st16_zero(tbase + sl * CP + r0);
                tmem_st16_zero(cbase - (sl * CP + r0));
#pragma unroll
                for (int i = 0; i < 16; ++i) re[i] = (re[i] + w[15 - i]) * f;
                if constexpr (CC == 2) {
                    tmem_ld16x2(tbase + sl * CP + P + r0, cbase - (sl * CP + P + r0), im, w);
                    tmem_st16_zero(tbase + sl * CP + P + r0);
                    tmem_st16_zero(cbase - (sl * CP + P + r0));
#pragma unroll
                    for (int i = 0; i < 16; ++i) im[i] = (im[i] + w[15 - i]) * f;
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) im[i] = 0.0f;
                }
                const int nv = nvalid - r0 < 16 ? nvalid - r0 : 16;
                if (nv > 0) store_run<16, CC, OUT>(A, o0 + (int64_t)sl * F + r0, nv, re, im, vec, lmin, lmax);
            }
        }
        // a pass whose scale count is odd leaves padding columns to the other warp: zero
        // the columns [ns*CP, cols) (if any) from warp half 0
        if (half == 0)
            for (int c = ns * CP; c < cols; c += 16) {
                tmem_st16_zero(tbase + c);
                tmem_st16_zero(cbase - c);
            }
    }
}

// Per-window power-of-two scale 2^ex of the split-fp16 conversion: the window's max |x| lands
// in [2^13, 2^14) (mx = m 2^E, m in [0.5, 1): ex = 14 - E).  Clamped to [-126, 126] so that
// both 2^ex (converters) and 2^-ex (epilogue) are finite normal floats: a near-silent window
// (max |x| < 2^-112) is scaled by 2^126 only -- its hi/lo parts are smaller than 2^13 but
// still carry 22 bits relative to the window max down to |x| ~ 2^-150.  A window max of 0
// (or not finite) gives ex = 0.
__device__ __forceinline__ int window_exponent(float mx) {
    if (!(mx > 0.0f) || !(mx <= 3.402823466e38f)) return 0;
    int e = 0;
    frexpf(mx, &e);
    const int ex = 14 - e;
    return ex > 126 ? 126 : (ex < -126 ? -126 : ex);
}

// Split two samples into hi / lo fp16 pairs: hi = rn16(x 2^e), lo = rn16(x 2^e - hi).  The
// scale and the residual use the packed fp32x2 pipe (FMUL2 / FADD2): 6 instructions per pair
// instead of 8 (measured neutral: the conversion waits on its loads, not on issue).
__device__ __forceinline__ void split2(float x0, float x1, uint64_t sc2, uint32_t &hw, uint32_t &lw) {
    uint64_t a2, p;
    asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(x0), "f"(x1));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(a2) : "l"(p), "l"(sc2));
    float ax, ay;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(ax), "=f"(ay) : "l"(a2));
    const __half2 h = __float22half2_rn(make_float2(ax, ay));
    const float2 hf = __half22float2(h);
    uint64_t hp, r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(hp) : "f"(hf.x), "f"(hf.y));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a2), "l"(hp));
    float rx, ry;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(rx), "=f"(ry) : "l"(r));
    const __half2 l = __float22half2_rn(make_float2(rx, ry));
    hw = *reinterpret_cast<const uint32_t *>(&h);
    lw = *reinterpret_cast<const uint32_t *>(&l);
}
__device__ __forceinline__ uint64_t pack_sc2(float sc) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(sc));
    return r;
}

// window chunk c (8 consecutive samples) -> (row, chunk within the row) for cpr = panels * 8
// chunks per row: row = (c * ceil(2^20 / cpr)) >> 20, exact for c < 131 k when cpr = 24 (checked
// exhaustively; windows have < 5 k chunks), and for any c when cpr is a power of two
__device__ __forceinline__ void chunk_rc(const UmmaArgs &A, int c, int &row, int &cc) {
    row = (int)(((uint32_t)c * (uint32_t)A.cpr_magic) >> 20);
    cc = c - row * A.cpr;
}

// ---- the kernel --------------------------------------------------------------------------
// Kernel variants (VS): 0 the common engine; 1 panel streaming (rows of hop samples, P = 1);
// 2 the common engine with the per-clip arrival machinery of the opt-in min-max modes.  Each
// variant's extra roles are compiled only there, so the common kernel keeps its size and
// layout: with the panel-streaming converters inside it c2 ran 4 us slower (68.6 vs 64.4 us),
// without them and the arrival code 2 us faster (62.5 us) -- instruction-cache footprint.
template <int CC, int P, int CG, int VS>
__global__ void __launch_bounds__(UM_THREADS, 1) k_umma(const __grid_constant__ UmmaArgs A) {
    extern __shared__ uint8_t smem_raw[];
    // 1 KB aligned (128 B swizzle atoms); pointer arithmetic on the shared array (not an
    // integer round trip) keeps the shared address space visible to the compiler: LDS/STS
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t b_full[UM_SLOTS], b_empty[UM_SLOTS];
    __shared__ uint64_t s_vstart[UM_SLOTS];  // producer-private: ring start of in-flight slots
    __shared__ __align__(8) uint64_t win_full[UM_WSLOTS], win_empty[UM_WSLOTS], acc_full[2], acc_empty[2];
    __shared__ float xring[4];  // per-unit window exponent 2^-e, written by the converters
    __shared__ float red[UM_CONV_WARPS];
    __shared__ __align__(8) uint64_t stg_full, res_full, tab_full;
    __shared__ __align__(8) uint64_t slot_full[UM_WSLOTS];  // panel streaming: a TMA panel copy has landed
    __shared__ __align__(8) uint64_t umax_full[4];          // panel streaming (fp16): a unit's window max is known
    __shared__ uint32_t s_umax[4];                           // ... max |x| of the window (float bits), by unit % 4
    __shared__ uint32_t tmem_base_sh;
    __shared__ int s_decide;  // epilogue: CTA-uniform decision on the oldest pending unit

    // Roles by warp: 0 producer, 1 MMA issuer / relay, 2.. converters, then epilogue (two warps
    // per TMEM lane quadrant = SM sub-partition).  (The producer on the MMA issuer's
    // sub-partition instead of warp 0's measured neutral: c2 62.4 vs 62.5 us, c5 978 vs 976 us.)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (kDiag && A.trace && threadIdx.x == 0 && blockIdx.x < 256) {
        A.trace[16 * 32 + 2 * blockIdx.x] = (long long)globaltimer_ns();
        if (blockIdx.x == 0) A.trace[14 * 32] = clock64();  // SM clock rate = cycles / ns
    }
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;  // 0 = leader (issues the MMAs)
    const bool leader = rank == 0;
    // work units: (clip, CG consecutive 128-row tiles); CTA `rank` of a pair takes tile
    // CG*j + rank.  All roles walk the same unit sequence.
    const int64_t u0 = CG == 2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
    const int64_t ustride = CG == 2 ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
    const int64_t tpu = (A.row_tiles + CG - 1) / CG;
    const int64_t n_units = A.clips * tpu * A.pgroups;
    // unit u: pass group u % pgroups of tile pair (u / pgroups) -- consecutive units (the pass
    // groups of one tile pair) go to different CTA pairs
    // (32-bit index math: the launcher checks n_units < 2^31)
    const uint32_t tpu32 = (uint32_t)tpu, pg32 = (uint32_t)A.pgroups;
    auto unit_tile = [&](int64_t u, int64_t &b, int64_t &tile) {
        const uint32_t v = (uint32_t)u / pg32;
        const uint32_t bq = v / tpu32;
        b = (int64_t)bq;
        tile = (int64_t)(CG * (v - bq * tpu32) + rank);
    };
    auto unit_passes = [&](int64_t u, int &p0, int &p1) {
        p0 = (int)((uint32_t)u % pg32) * A.ppu;
        p1 = p0 + A.ppu < A.n_passes ? p0 + A.ppu : A.n_passes;
    };
    // Converters, register-prefetch path: each thread loads its first CONV_RC 8-sample chunks
    // of a unit's window into registers (cv) and the window's max |x| over all its chunks
    // (cmx).  The first unit's window is fetched right at launch, overlapping the setup.
    constexpr int CONV_RC = UM_CONV_RC;
    float cv[CONV_RC][8];
    float cmx = 0.0f;
    bool cbad = false;  // this thread's chunks of the fetched window held non-finite samples
    auto conv_load8 = [&](const float *xb, int64_t w0, int32_t off, int32_t in_lo, int32_t in_hi, float (&o)[8]) {
        if (A.vec_ok && off >= in_lo && off + 8 <= in_hi) {
            const float4 *g = reinterpret_cast<const float4 *>(xb + w0 + off);
            const float4 u = __ldg(g), w = __ldg(g + 1);
            o[0] = u.x; o[1] = u.y; o[2] = u.z; o[3] = u.w;
            o[4] = w.x; o[5] = w.y; o[6] = w.z; o[7] = w.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int32_t q = off + k;
                o[k] = (q >= in_lo && q < in_hi) ? __ldg(xb + w0 + q) : 0.0f;
            }
        }
    };
    auto conv_fetch = [&](int64_t item) {
        int64_t b, tile;
        unit_tile(item, b, tile);
        const int64_t w0 = tile * 128 * A.V - A.G0;
        const float *xb = A.x + b * A.ld_x;
        const int32_t in_lo = (int32_t)(w0 < 0 ? -w0 : 0);
        const int64_t in_hi64 = A.N - w0;
        const int32_t in_hi = (int32_t)(in_hi64 < (int64_t)0x7fffffff ? in_hi64 : (int64_t)0x7fffffff);
        const int ct = (int)threadIdx.x - 64, chunks = A.win_rows * A.panels * 8;
        auto chunk_off = [&](int c) {
            int row, cc;
            chunk_rc(A, c, row, cc);
            return (int32_t)(row * A.V + cc * 8);
        };
#pragma unroll
        for (int i = 0; i < CONV_RC; ++i) {
            const int c = ct + i * UM_CONV_THREADS;
            if (c < chunks) {
                conv_load8(xb, w0, chunk_off(c), in_lo, in_hi, cv[i]);
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) cv[i][k] = 0.0f;
            }
        }
        float mx = 0.0f;
        // chunks beyond the register share: max only (re-read after the wait)
        for (int c = ct + CONV_RC * UM_CONV_THREADS; c < chunks; c += UM_CONV_THREADS) {
            float t[8];
            conv_load8(xb, w0, chunk_off(c), in_lo, in_hi, t);
#pragma unroll
            for (int k = 0; k < 8; ++k) mx = fmax_nan(mx, fabsf(t[k]));
        }
#pragma unroll
        for (int i = 0; i < CONV_RC; ++i)
#pragma unroll
            for (int k = 0; k < 8; ++k) mx = fmax_nan(mx, fabsf(cv[i][k]));
        cbad = !(mx <= 3.402823466e38f);
        if (cbad) {
            // non-finite samples (rare): replaced by 0 here and after the wait; recorded for the
            // fix-up once -- by the tile that owns the sample, in the unit of pass group 0
            int p0, p1;
            unit_passes(item, p0, p1);
            const int64_t own0 = tile * 128 * A.V, own1 = own0 + 128 * (int64_t)A.V;
            uint32_t *rec = A.nfbad + b * (int64_t)(1 + WH_NF_CAP);
            auto fix8 = [&](int c, float (&o)[8]) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (!is_finite_f(o[k])) {
                        const int64_t g = w0 + chunk_off(c) + k;
                        if (p0 == 0 && g >= own0 && g < own1 && A.nfbad) nf_record(rec, A.nfctl + 1, g);
                        o[k] = 0.0f;
                    }
                }
            };
            mx = 0.0f;
            for (int c = ct + CONV_RC * UM_CONV_THREADS; c < chunks; c += UM_CONV_THREADS) {
                float t[8];
                conv_load8(xb, w0, chunk_off(c), in_lo, in_hi, t);
                fix8(c, t);
#pragma unroll
                for (int k = 0; k < 8; ++k) mx = fmaxf(mx, fabsf(t[k]));
            }
#pragma unroll
            for (int i = 0; i < CONV_RC; ++i) {
                const int c = ct + i * UM_CONV_THREADS;
                if (c < chunks) fix8(c, cv[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) mx = fmaxf(mx, fabsf(cv[i][k]));
            }
        }
        cmx = mx;
    };
    // L2 prefetch of a unit's fp32 window (one bulk prefetch: the window is a contiguous sample
    // range of one clip), issued UM_PF units ahead so that the converters' loads hit L2.  Only
    // for rows of 256 samples (hop 256 / multiples of 256: one 147 KB window, its conversion not
    // overlapped with the MMAs; c4 hop 256 / 1024 -6 %); neutral or slower elsewhere.
    auto window_prefetch = [&](int64_t item) {
        if (!A.pf || item >= n_units) return;
        int64_t b, tile;
        unit_tile(item, b, tile);
        const int64_t w0 = tile * 128 * A.V - A.G0;
        int64_t lo = w0 > 0 ? w0 : 0, hi = w0 + (int64_t)A.win_rows * A.V;
        if (hi > A.N) hi = A.N;
        if (hi <= lo) return;
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(A.x + b * A.ld_x + lo) & ~(uintptr_t)15;
        const uintptr_t a1 = (reinterpret_cast<uintptr_t>(A.x + b * A.ld_x + hi) + 15) & ~(uintptr_t)15;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
    };
    if (threadIdx.x == 64)
        for (int k = 1; k <= UM_PF; ++k) window_prefetch(u0 + k * ustride);
    constexpr int PS = VS == 1 ? 1 : 0;  // panel streaming
    constexpr int AC = (VS == 1 || VS == 3) ? 1 : 0;  // two accumulator sets per buffer possible
    if (warp >= 2 && warp < 2 + UM_CONV_WARPS && A.conv_regs && u0 < n_units) conv_fetch(u0);
    const uint32_t WH = A.win_half_bytes;               // bytes of one (hi or lo) window
    uint8_t *win_base = smem;                            // [win_bufs][hi|lo][panels][rows][128]
    uint8_t *stage_base = smem + (size_t)A.win_bufs * 2 * WH;
    const uint32_t panel_bytes = (uint32_t)A.win_rows * 128u;
    // pass / tile tables (compact) after the tap stages (and the fp32 staging buffer)
    int4 *s_pass = reinterpret_cast<int4 *>(stage_base + (size_t)A.ring_bytes +
                                            (A.use_stg ? 2 * (size_t)WH : 0));
    int4 *s_group = s_pass + A.n_passes;
    uint4 *s_tile = reinterpret_cast<uint4 *>(s_group + A.n_groups);
    float *s_spow = reinterpret_cast<float *>(s_tile + A.n_tiles);  // per-scale 2^-f (16-byte aligned)
    int *s_goff = reinterpret_cast<int *>(s_spow + ((A.S + 15) & ~15));  // resident: smem offset per group
    // the tables arrive by one bulk copy (one HBM round trip at launch; the host packed them
    // in their smem layout)
    if (threadIdx.x == 0) {
        mbar_init(&tab_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&tab_full, A.tables_bytes);
        bulk_g2s(s_pass, A.tables, A.tables_bytes, &tab_full);
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < UM_SLOTS; ++i) {
            mbar_init(&b_full[i], (CG == 2 && leader) ? 2 : 1);  // + the peer's relay
            mbar_init(&b_empty[i], 1);
        }
        for (int i = 0; i < UM_WSLOTS; ++i) {
            mbar_init(&win_full[i], (CG == 2 && leader) ? 2 : 1);  // + the peer's converters
            mbar_init(&win_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], UM_EPI_WARPS * CG);  // epilogue warps of both CTAs (leader's copy)
        }
        mbar_init(&stg_full, 1);
        for (int i = 0; i < UM_WSLOTS; ++i) mbar_init(&slot_full[i], 1);
        for (int i = 0; i < 4; ++i) mbar_init(&umax_full[i], 1);
        mbar_init(&res_full, (CG == 2 && leader) ? 2 : 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&tmem_base_sh)), "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(&tmem_base_sh)), "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    mbar_wait(&tab_full, 0);
    const uint32_t tmem = tmem_base_sh;
    if (warp >= 2 + UM_CONV_WARPS) {
        // epilogue warps zero both accumulator buffers of their lane quadrant: every MMA
        // accumulates (accumulate = 1), columns a pass never touches stay 0
        const uint32_t tq = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const uint32_t ehalf = (uint32_t)((warp - 2 - UM_CONV_WARPS) >> 2);
        for (uint32_t c = 256 * ehalf; c < 256 * ehalf + 256; c += 16) tmem_st16_zero(tq + c);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cta_pair_sync<CG>();
    tc_fence_after();
    const bool pon = kDiag && A.prof != nullptr;
    ProfAcc pa;
    pa.start();

    if (warp == 0) {
        // ===================== producer: this CTA's half of each tap tile =============
        // Tiles have different sizes (nc columns), so the stage buffer is a byte ring of
        // UM_SLOTS variable-size slots: virtual offsets grow monotonically, a tile never
        // straddles the physical end, and a slot is reused once the MMAs that read the
        // oldest bytes in the way have committed.
        if (A.resident) {
            // one barrier for the resident groups: arm it with all bytes, then copy them
            if (elect_one()) {
                uint32_t total = 0;
                for (int gi = 0; gi < A.n_groups; ++gi)
                    if (s_goff[gi] >= 0) total += (uint32_t)s_group[gi].w;
                mbar_expect_tx(&res_full, total);
                for (int gi = 0; gi < A.n_groups; ++gi) {
                    const int4 gr = s_group[gi];
                    if (s_goff[gi] >= 0)
                        bulk_g2s(stage_base + s_goff[gi], A.bank + ((size_t)(uint32_t)gr.z << 7) + (size_t)rank * gr.w,
                                 (uint32_t)gr.w, &res_full);
                }
            }
            __syncwarp();
        }
        // streamed groups (all of them without a resident region, the tail K-steps of a
        // unit in hybrid mode) cycle through the ring that follows the resident region
        uint8_t *ring_base = stage_base + A.res_bytes;
        uint64_t vhead = 0;   // virtual (monotonic) ring offset
        uint32_t phys = 0;    // vhead % RING, tracked incrementally
        uint32_t seq = 0, tail = 0;
        const uint32_t RING = A.ring_bytes - A.res_bytes;
        for (int64_t item = A.n_stream ? u0 : n_units; item < n_units; item += ustride) {
            int pb, pe;
            unit_passes(item, pb, pe);
            for (int p = pb; p < pe; ++p) {
                const int4 pinfo = s_pass[p];
                for (int gi = pinfo.x; gi < pinfo.y; ++gi) {
                    if (s_goff[gi] >= 0) continue;  // resident
                    const int4 gr = s_group[gi];
                    const uint32_t bytes = (uint32_t)gr.w;
                    uint64_t v = vhead;
                    if (phys + bytes > RING) {  // never straddle the physical end
                        v += RING - phys;
                        phys = 0;
                    }
                    const uint64_t vend = v + bytes;
                    while (tail < seq && (seq - tail >= (uint32_t)UM_SLOTS || s_vstart[tail % UM_SLOTS] + RING < vend)) {
                        mbar_wait_p(&b_empty[tail % UM_SLOTS], (tail / UM_SLOTS) & 1, pa, 0, pon);
                        ++tail;
                    }
                    const uint32_t slot = seq % UM_SLOTS;
                    const long long t_issue = pon ? clock64() : 0;
                    if (elect_one()) {
                        s_vstart[slot] = v;
                        if (WH_DBG(128) && item != u0) {
                            mbar_arrive(&b_full[slot]);  // diagnostics: stale taps, no L2 traffic
                        } else {
                            mbar_expect_tx(&b_full[slot], bytes);
                            bulk_g2s(ring_base + phys, A.bank + ((size_t)(uint32_t)gr.z << 7) + (size_t)rank * bytes,
                                     bytes, &b_full[slot]);
                        }
                    }
                    __syncwarp();
                    if (pon) pa.c[1] += (unsigned long long)(clock64() - t_issue);
                    vhead = vend;
                    phys += bytes;
                    ++seq;
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ===================== MMA issuer (leader CTA; whole warp, one elected lane) ==
        uint32_t seq = 0, wcnt = 0, acnt = 0;
        uint32_t phys = 0;  // ring offset: same allocation sequence as the producer
        if (A.resident) {
            mbar_wait_p(&res_full, 0, pa, 2, pon);  // the resident groups (both CTAs' halves)
            tc_fence_after();
        }
        const uint32_t RING = A.ring_bytes - A.res_bytes;
        const uint32_t stage0 = smem_u32(stage_base), ring0 = stage0 + A.res_bytes;
        if (PS) {
            // Panel streaming: the window's column panels pass through the window slots (panel
            // counter pc, slot pc % win_bufs); the tiles of the single pass are in panel-major
            // order; tap groups stream through the ring (or are resident).
            const uint32_t wh16 = WH >> 4, NS = (uint32_t)A.win_bufs;
            const int *s_tpanel = s_goff + A.n_groups;  // window panel of each tile
            uint32_t pc = 0;
            const uint32_t o2 = A.acc2 ? 128u : 0u;
            for (int64_t item = u0; item < n_units; item += ustride, ++wcnt, ++acnt) {
                WH_TRACE(0, wcnt);
                const int4 pinfo = s_pass[0];
                const uint32_t ab = acnt % A.n_acc;
                mbar_wait_p(&acc_empty[ab], ((acnt / A.n_acc) & 1) ^ 1, pa, 1, pon);
                tc_fence_after();
                const uint32_t d_acc = tmem + ab * (uint32_t)A.acc_stride;
                const uint32_t C = (uint32_t)pinfo.w;
                int cur = -1;
                bool held = false;  // the slot of panel `cur` is not released yet
                uint32_t a_hi16 = 0;
                // a panel's slot is released right behind its last tile's MMAs (not when the next
                // panel is reached): the refill of the slot then never waits for the issue loop
                auto release = [&]() {
                    if (elect_one()) umma_commit<CG>(&win_empty[pc % NS]);
                    __syncwarp();
                    ++pc;
                    held = false;
                };
                // step to panel `target`: wait for the following panels (a panel without tiles
                // is released at once)
                auto step_to = [&](int target) {
                    while (cur < target) {
                        if (held) release();
                        mbar_wait_p(&win_full[pc % NS], (pc / NS) & 1, pa, 0, pon);
                        tc_fence_after();
                        a_hi16 = (smem_u32(win_base) + (pc % NS) * 2 * WH) >> 4;
                        ++cur;
                        held = true;
                    }
                };
                const int t_last = s_group[pinfo.y - 1].y - 1;  // the unit's last tile
                WH_TRACE(1, wcnt);
                for (int gi = pinfo.x; gi < pinfo.y; ++gi) {
                    const int4 gr = s_group[gi];
                    const uint32_t bytes = (uint32_t)gr.w;
                    uint32_t gbase, slot = 0;
                    const int goff = s_goff[gi];
                    if (goff >= 0) {
                        gbase = stage0 + (uint32_t)goff;
                    } else {
                        if (phys + bytes > RING) phys = 0;  // same ring allocation as the producer
                        gbase = ring0 + phys;
                        phys += bytes;
                        slot = seq % UM_SLOTS;
                        const uint32_t ph = (seq / UM_SLOTS) & 1;
                        ++seq;
                        mbar_wait_p(&b_full[slot], ph, pa, 2, pon);
                        tc_fence_after();
                    }
                    const uint32_t g16 = gbase >> 4;
                    // The issuing thread waits on every MMA it issues (the tensor pipe's queue is
                    // short), so the table entries of the next tile are loaded before this
                    // tile's MMAs: their latency passes behind the issue.  (One entry past the
                    // group's end is still inside the tables.)
                    uint4 tt = s_tile[gr.x];
                    int tp = s_tpanel[gr.x];
                    for (int t = gr.x; t < gr.y; ++t) {
                        const uint4 tn = s_tile[t + 1];
                        const int tpn = s_tpanel[t + 1];
                        if (tp != cur) step_to(tp);
                        const uint32_t ah = a_hi16 + (tt.x & 0xffffu), al = ah + wh16;
                        const uint32_t b1 = g16 + (tt.y & 0xffffu), b2 = b1 + (tt.y >> 16);
                        const uint32_t d1 = d_acc + (tt.x >> 16), d2 = d_acc + C;
                        if (!WH_DBG(4) && elect_one()) {
                            if (A.tf32) {
                                // acc2: odd K-slices accumulate into a second (main | corr) set 128
                                // columns on -- half the accumulation steps per accumulator (the
                                // fp32 accumulate truncates: the error grows with the steps);
                                // the epilogue adds the sets
#pragma unroll
                                for (uint32_t j = 0; j < 4; ++j) {
                                    const uint32_t o = (j & 1) ? o2 : 0u;
                                    umma_tf32<CG>(d1 + o, DESC_HI | (ah + 2 * j), DESC_HI | (b1 + 2 * j), tt.z);
                                    if (tt.w) umma_tf32<CG>(d2 + o, DESC_HI | (al + 2 * j), DESC_HI | (b2 + 2 * j), tt.w);
                                }
                            } else if (tt.w) {
#pragma unroll
                                for (uint32_t j = 0; j < 4; ++j) {
                                    umma_f16<CG>(d1, DESC_HI | (ah + 2 * j), DESC_HI | (b1 + 2 * j), tt.z);
                                    umma_f16<CG>(d2, DESC_HI | (al + 2 * j), DESC_HI | (b2 + 2 * j), tt.w);
                                }
                            } else {
#pragma unroll
                                for (uint32_t j = 0; j < 4; ++j)
                                    umma_f16<CG>(d1, DESC_HI | (ah + 2 * j), DESC_HI | (b1 + 2 * j), tt.z);
                            }
                        }
                        __syncwarp();
                        if (tpn != tp || t == t_last) release();
                        tt = tn;
                        tp = tpn;
                    }
                    if (goff < 0) {
                        if (elect_one()) umma_commit<CG>(&b_empty[slot]);
                        __syncwarp();
                    }
                }
                step_to(A.panels - 1);
                if (held) release();
                if (elect_one()) umma_commit<CG>(&acc_full[ab]);
                __syncwarp();
                WH_TRACE(2, wcnt);
            }
        } else
        for (int64_t item = u0; item < n_units; item += ustride, ++wcnt) {
            const uint32_t wb = wcnt % A.win_bufs;
            WH_TRACE(0, wcnt);
            mbar_wait_p(&win_full[wb], (wcnt / A.win_bufs) & 1, pa, 0, pon);
            tc_fence_after();
            WH_TRACE(1, wcnt);
            const uint32_t a_hi16 = (smem_u32(win_base) + wb * 2 * WH) >> 4, wh16 = WH >> 4;
            int pb, pe;
            unit_passes(item, pb, pe);
            for (int p = pb; p < pe; ++p, ++acnt) {
                const int4 pinfo = s_pass[p];
                const uint32_t ab = acnt % A.n_acc;
                mbar_wait_p(&acc_empty[ab], ((acnt / A.n_acc) & 1) ^ 1, pa, 1, pon);
                tc_fence_after();
                const uint32_t d_acc = tmem + ab * (uint32_t)A.acc_stride;
                const uint32_t C = (uint32_t)pinfo.w;
                for (int gi = pinfo.x; gi < pinfo.y; ++gi) {
                    const int4 gr = s_group[gi];
                    const uint32_t bytes = (uint32_t)gr.w;
                    uint32_t gbase, slot = 0;
                    const int goff = s_goff[gi];
                    if (goff >= 0) {
                        gbase = stage0 + (uint32_t)goff;
                    } else {
                        if (phys + bytes > RING) phys = 0;  // same ring allocation as the producer
                        gbase = ring0 + phys;
                        phys += bytes;
                        slot = seq % UM_SLOTS;
                        const uint32_t ph = (seq / UM_SLOTS) & 1;
                        ++seq;
                        mbar_wait_p(&b_full[slot], ph, pa, 2, pon);
                        tc_fence_after();
                    }
                    const uint32_t g16 = gbase >> 4;
                    // (the next tile's table entry is loaded before this tile's MMAs: the issuing
                    // thread waits on every MMA it issues, so the load's latency passes behind them;
                    // one entry past the last tile is still inside the tables)
                    uint4 tt = s_tile[gr.x];
                    for (int t = gr.x; t < gr.y; ++t) {
                        // MMA1: A_hi x [hi_c0..hi_C-1 | lo_C-1..lo_c1] -> main_j at col j, corr_j at 2C-1-j
                        // MMA2: A_lo x [hi_C-1..hi_c1]               -> corr   (skipped if c1 = C)
                        // (CG = 2: each CTA's stage holds half of every B operand).  Descriptor
                        // low words are 16-byte smem addresses (< 2^14): no masking needed.
                        const uint4 tn = s_tile[t + 1];
                        const uint32_t ah = a_hi16 + (tt.x & 0xffffu), al = ah + wh16;
                        const uint32_t b1 = g16 + (tt.y & 0xffffu), b2 = b1 + (tt.y >> 16);
                        const uint32_t d1 = d_acc + (tt.x >> 16), d2 = d_acc + C;
                        // VS = 3 (very long filters): odd K-slices go to the second accumulator set
                        // of the buffer, 128 columns on (half the accumulation steps per set)
                        constexpr uint32_t o2 = VS == 3 ? 128u : 0u;
                        if (!WH_DBG(4) && elect_one()) {
                            if (tt.w) {
#pragma unroll
                                for (uint32_t j = 0; j < 4; ++j) {
                                    const uint32_t o = (j & 1) ? o2 : 0u;
                                    umma_f16<CG>(d1 + o, DESC_HI | (ah + 2 * j), DESC_HI | (b1 + 2 * j), tt.z);
                                    umma_f16<CG>(d2 + o, DESC_HI | (al + 2 * j), DESC_HI | (b2 + 2 * j), tt.w);
                                }
                            } else {
#pragma unroll
                                for (uint32_t j = 0; j < 4; ++j)
                                    umma_f16<CG>(d1 + ((j & 1) ? o2 : 0u), DESC_HI | (ah + 2 * j), DESC_HI | (b1 + 2 * j), tt.z);
                            }
                        }
                        __syncwarp();
                        tt = tn;
                    }
                    if (goff < 0) {
                        if (elect_one()) umma_commit<CG>(&b_empty[slot]);
                        __syncwarp();
                    }
                }
                if (elect_one()) umma_commit<CG>(&acc_full[ab]);
                __syncwarp();
            }
            if (elect_one()) umma_commit<CG>(&win_empty[wb]);
            __syncwarp();
            WH_TRACE(2, wcnt);
        }
    } else if (warp == 1) {
        // ===================== relay (peer CTA of a pair) ============================
        // forwards "my half of the tap group landed" to the leader's barriers, which the
        // leader's MMA issuer waits on.  (A non-tensor bulk copy completes on the destination
        // CTA's own barrier -- tools/probe_remote_tx.cu.)
        uint32_t seq = 0;
        if (A.resident) {
            mbar_wait_p(&res_full, 0, pa, 2, pon);
            if (elect_one()) mbar_arrive_leader_relaxed(&res_full);
            __syncwarp();
        }
        for (int64_t item = A.n_stream ? u0 : n_units; item < n_units; item += ustride) {
            int pb, pe;
            unit_passes(item, pb, pe);
            for (int p = pb; p < pe; ++p) {
                const int4 pinfo = s_pass[p];
                for (int gi = pinfo.x; gi < pinfo.y; ++gi) {
                    if (s_goff[gi] >= 0) continue;
                    mbar_wait_p(&b_full[seq % UM_SLOTS], (seq / UM_SLOTS) & 1, pa, 2, pon);
                    if (elect_one()) mbar_arrive_leader_relaxed(&b_full[seq % UM_SLOTS]);
                    __syncwarp();
                    ++seq;
                }
            }
        }
    } else if (warp < 2 + UM_CONV_WARPS) {
        // ===================== converters ============================================
        // The fp32 window of a tile is a contiguous sample range of the clip; one elected
        // converter thread bulk-copies it into the staging buffer one unit ahead.
        const int ct = (int)threadIdx.x - 64;  // 0 .. UM_CONV_THREADS-1
        // window wb of unit wcnt is converted (all converter threads passed bar 1): tell the
        // MMA issuer -- the leader's own barrier, directly from the peer CTA too
        auto window_ready = [&](uint32_t wb, uint32_t wcnt) {
            if (CG == 2 && !leader) {
                if (WH_DBG(8)) mbar_arrive_leader(&win_full[wb]);  // diagnostics: cluster-scope release
                else mbar_arrive_leader_cta(&win_full[wb]);
            } else {
                mbar_arrive(&win_full[wb]);
            }
        };
        const int cw = warp - 2;
        const int chunks = A.win_rows * A.panels * 8;  // 8-sample chunks in the window
        const int64_t wlen = (int64_t)A.win_rows * A.V;
        float *stg = reinterpret_cast<float *>(stage_base + (size_t)A.ring_bytes);
        // staged range [lo, hi) of the clip for an item (16-byte granular); rest read directly
        auto staged = [&](int64_t item, int64_t &lo, int64_t &hi) {
            int64_t b, tile;
            unit_tile(item, b, tile);
            const int64_t w0 = tile * 128 * A.V - A.G0;
            lo = w0 > 0 ? w0 : 0;
            hi = w0 + wlen < A.N ? w0 + wlen : (A.N & ~(int64_t)3);
            if (!A.vec_ok || !A.use_stg || hi <= lo) { lo = hi = w0; }
            (void)b;
        };
        auto issue = [&](int64_t item) {
            int64_t lo, hi;
            staged(item, lo, hi);
            int64_t b, tile;
            unit_tile(item, b, tile);
            const int64_t w0 = tile * 128 * A.V - A.G0;
            const uint32_t bytes = (uint32_t)((hi - lo) * 4);
            mbar_expect_tx(&stg_full, bytes);
            if (bytes) bulk_g2s(stg + (lo - w0), A.x + b * A.ld_x + lo, bytes, &stg_full);
        };
        if (PS && A.tf32) {
            // Panel streaming with tf32 operands.  A panel is 32 samples (128 B of fp32) of every
            // window row, fetched win_bufs - 1 panels ahead straight to its swizzled place in the
            // hi half of a slot: by ONE TMA tensor copy (a box of 128 B x win_rows rows of the
            // batch viewed as (V samples, N / V rows, clips), 128 B swizzle, rows outside the clip
            // zero-filled by the copy engine), or -- unaligned inputs -- by cp.async, 16 bytes per
            // thread.  Once landed, each converter thread reads its chunks back, clears the low
            // 13 bits in place (hi = the tf32 the tensor core reads) and writes lo = x - hi (exact
            // in fp32, rounded to tf32) at the same offset of the slot's lo half.  No window
            // exponent: tf32 keeps fp32's range.  Chunk c = ct + i * CONV_THREADS sits at row
            // c >> 3, 16-byte column c & 7: the row stride between a thread's chunks is a multiple
            // of 8, so its swizzle term is constant and the addresses advance by fixed steps.
            const uint32_t NS = (uint32_t)A.win_bufs;
            const int nch = A.win_rows * 8;
            const int row0 = ct >> 3, c8 = ct & 7;
            constexpr int RSTEP = UM_CONV_THREADS / 8;          // rows between a thread's chunks
            constexpr uint32_t SSTEP = (uint32_t)RSTEP * 128u;  // shared-memory bytes between them
            static_assert(RSTEP % 8 == 0, "converter threads must cover whole swizzle periods");
            const int nmine = ct < nch ? (nch - ct + UM_CONV_THREADS - 1) / UM_CONV_THREADS : 0;
            const uint32_t soff0 = smem_u32(win_base) + (uint32_t)row0 * 128u + (uint32_t)((c8 ^ (row0 & 7)) << 4);
            const int64_t gstep = (int64_t)RSTEP * A.V;  // samples between a thread's chunks
            const bool tma = A.tma != 0;
            struct Geo {
                const float *xb;   // the clip
                int64_t g0;        // clip sample of this thread's first chunk in panel 0
                int64_t w0;        // clip sample of the window's first row
                int64_t b, tile;
                int64_t r0;        // tma: tensor row of the window's first row (floor(w0 / V))
                int32_t coff;      // tma: column of the window's first sample in that row
                bool interior;     // the whole window lies inside the clip (and is 16-byte aligned)
                bool tail;         // tma: the window reaches the clip's last, partial row of V samples
            };
            auto geo = [&](int64_t item) {
                Geo g;
                unit_tile(item, g.b, g.tile);
                g.w0 = g.tile * 128 * A.V - A.G0;
                g.xb = A.x + g.b * A.ld_x;
                g.g0 = g.w0 + (int64_t)row0 * A.V + c8 * 4;
                const int64_t wend = g.w0 + (int64_t)A.win_rows * A.V;
                g.interior = A.vec_ok && g.w0 >= 0 && wend <= A.N;
                g.tail = A.full_end < A.N && wend > A.full_end;
                // w0 = tile * 128 * V - G0: floor division by V without dividing (G0 < 2^31)
                const int64_t q = (int64_t)((uint32_t)A.G0 / (uint32_t)A.V);
                const int32_t rem = A.G0 - (int32_t)q * A.V;
                g.r0 = g.tile * 128 - q - (rem ? 1 : 0);
                g.coff = rem ? A.V - rem : 0;
                return g;
            };
            auto fetch_panel = [&](const Geo &g, int p, uint32_t sl) {
                if (tma) {
                    // one box: columns [col, col + 32) of rows [r0, r0 + win_rows) of clip b
                    if (ct == 0) {
                        int64_t r0 = g.r0;
                        int32_t col = g.coff + p * 32;
                        if (col >= A.V) {
                            col -= A.V;
                            ++r0;
                        }
                        mbar_expect_tx(&slot_full[sl], WH);
                        asm volatile(
                            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
                            "{%2, %3, %4}], [%5];" ::"r"(smem_u32(win_base) + sl * 2 * WH),
                            "l"(&A.tmap), "r"((int32_t)col), "r"((int32_t)r0), "r"((int32_t)g.b), "r"(smem_u32(&slot_full[sl]))
                            : "memory");
                    }
                    return;
                }
                uint32_t dst = soff0 + sl * 2 * WH;
                if (g.interior) {
                    const float *src = g.xb + g.g0 + p * 32;
                    for (int i = 0; i < nmine; ++i, dst += SSTEP, src += gstep)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
                } else {
                    int64_t q = g.g0 + p * 32;
                    for (int i = 0; i < nmine; ++i, dst += SSTEP, q += gstep) {
                        if (A.vec_ok && q >= 0 && q + 4 <= A.N) {
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(g.xb + q) : "memory");
                        } else {
                            float z[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) z[k] = (q + k >= 0 && q + k < A.N) ? __ldg(g.xb + q + k) : 0.0f;
                            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "f"(z[0]), "f"(z[1]),
                                         "f"(z[2]), "f"(z[3]) : "memory");
                        }
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            // the fetch sequence runs NS - 1 panels ahead of the conversion
            int64_t f_item = u0;
            int f_p = 0;
            uint32_t fc = 0;
            Geo fg = geo(u0 < n_units ? u0 : 0);
            auto fetch_next = [&]() {
                if (f_item < n_units) fetch_panel(fg, f_p, fc % NS);
                else if (!tma) asm volatile("cp.async.commit_group;" ::: "memory");  // keep the group count
                ++fc;
                if (++f_p == A.panels) {
                    f_p = 0;
                    f_item += ustride;
                    if (f_item < n_units) fg = geo(f_item);
                }
            };
            // TMA copies cost the issuing thread next to nothing, so they run only NS - 2 panels
            // ahead: the slot they refill was released two panels ago and the thread never waits
            const uint32_t lag = tma ? 2u : 1u;
            for (uint32_t j = 0; j + lag < NS; ++j) fetch_next();
            uint32_t qc = 0, wcnt = 0;
            for (int64_t item = u0; item < n_units; item += ustride, ++wcnt) {
                const Geo cg = geo(item);
                int p0, p1;
                unit_passes(item, p0, p1);
                const int64_t own0 = cg.tile * 128 * A.V, own1 = own0 + 128 * (int64_t)A.V;
                uint32_t *rec = A.nfbad ? A.nfbad + cg.b * (int64_t)(1 + WH_NF_CAP) : nullptr;
                if (ct == 0) {
                    WH_TRACE(3, wcnt);
                    xring[wcnt & 3] = 1.0f;
                }
                for (int p = 0; p < A.panels; ++p, ++qc) {
                    const uint32_t sl = qc % NS;
                    {
                        const long long tw = pon ? clock64() : 0;
                        if (tma) mbar_wait(&slot_full[sl], (qc / NS) & 1);
                        else asm volatile("cp.async.wait_group %0;" ::"n"(UM_WSLOTS - 2) : "memory");
                        if (pon) pa.c[0] += (unsigned long long)(clock64() - tw);
                    }
                    if (wcnt == 1 && ct == 0) WH_TRACE(4, p);  // diagnostics: panel timeline of the second unit
                    const uint32_t a0 = soff0 + sl * 2 * WH;
                    const long long tc0 = pon ? clock64() : 0;
                    constexpr int UNR = 6;  // chunks in flight per thread (independent load -> split -> store chains)
                    for (int i0 = 0; i0 < (WH_DBG(2) ? 0 : nmine); i0 += UNR) {
                        uint32_t v[UNR][4];
#pragma unroll
                        for (int u = 0; u < UNR; ++u)
                            if (i0 + u < nmine)
                                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                                             : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3])
                                             : "r"(a0 + (uint32_t)(i0 + u) * SSTEP) : "memory");
#pragma unroll
                        for (int u = 0; u < UNR; ++u) {
                            if (i0 + u >= nmine) continue;
                            const int i = i0 + u;
                            if (cg.tail) {
                                // the clip's last row of V samples is partial: the tensor ends before
                                // it (zero fill), its samples come straight from the clip
                                const int64_t g = cg.g0 + p * 32 + (int64_t)i * gstep;
                                if (g >= A.full_end && g < A.N) {
#pragma unroll
                                    for (int k = 0; k < 4; ++k)
                                        v[u][k] = g + k < A.N ? __float_as_uint(__ldg(cg.xb + g + k)) : 0u;
                                }
                            }
                            const float m = fmax_nan(fmax_nan(fabsf(__uint_as_float(v[u][0])), fabsf(__uint_as_float(v[u][1]))),
                                                     fmax_nan(fabsf(__uint_as_float(v[u][2])), fabsf(__uint_as_float(v[u][3]))));
                            if (!(m <= 3.402823466e38f)) {  // non-finite samples (rare): 0, recorded once
#pragma unroll
                                for (int k = 0; k < 4; ++k) {
                                    if (!is_finite_f(__uint_as_float(v[u][k]))) {
                                        const int64_t g = cg.g0 + p * 32 + (int64_t)i * gstep + k;
                                        if (rec && p0 == 0 && g >= own0 && g < own1) nf_record(rec, A.nfctl + 1, g);
                                        v[u][k] = 0u;
                                    }
                                }
                            }
                            uint32_t h[4], l[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                h[k] = v[u][k] & 0xffffe000u;
                                const float r = __uint_as_float(v[u][k]) - __uint_as_float(h[k]);
                                l[k] = (__float_as_uint(r) + 0x1000u) & 0xffffe000u;
                            }
                            const uint32_t a = a0 + (uint32_t)i * SSTEP;
                            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(h[0]), "r"(h[1]), "r"(h[2]),
                                         "r"(h[3]) : "memory");
                            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a + WH), "r"(l[0]), "r"(l[1]),
                                         "r"(l[2]), "r"(l[3]) : "memory");
                        }
                    }
                    if (pon) pa.c[2] += (unsigned long long)(clock64() - tc0);
                    if (wcnt == 1 && ct == 0) WH_TRACE(5, p);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
                    if (wcnt == 1 && ct == 0) WH_TRACE(6, p);
                    if (ct == 0) window_ready(sl, qc);
                    // refill the slot of the previous panel once its MMAs are done (TMA: only the
                    // issuing thread waits)
                    if (qc >= lag && (!tma || ct == 0)) {
                        const uint32_t ps = (qc - lag) % NS;
                        mbar_wait_p(&win_empty[ps], ((qc - lag) / NS) & 1, pa, 1, pon);
                    }
                    if (wcnt == 1 && ct == 0) WH_TRACE(12, p);
                    fetch_next();
                    if (wcnt == 1 && ct == 0) WH_TRACE(13, p);
                }
                if (ct == 0) WH_TRACE(7, wcnt);
            }
            if (!tma) asm volatile("cp.async.wait_all;" ::: "memory");
        } else if (PS) {
            // Panel streaming (rows of hop samples).  Each 64-sample column panel of a unit's
            // window (win_rows rows x 256 B of fp32) is copied by cp.async straight into a panel
            // slot, win_bufs - 1 panels ahead; once it has landed the converters read their own
            // chunks back, split them with the unit's exponent (from the pre-pass segment
            // maxima) and overwrite the slot in place with the swizzled hi | lo fp16 panel
            // (exactly the same 256 B per row).  A slot is refilled once the MMAs of the panel it
            // held have completed.
            constexpr int PCH = UM_PCH;
            const int pchunks = A.win_rows * 8;
            const uint32_t NS = (uint32_t)A.win_bufs;
            // cp.async of panel (item, p) into slot `sl`: chunk c of this thread = row c >> 3,
            // 8 samples at column (c & 7) * 8; out-of-clip samples are stored as zeros
            // Fetch geometry of a unit, computed once per unit: this thread's chunk i sits at window
            // row (ct >> 3) + i * CONV_THREADS / 8, samples (ct & 7) * 8 .. + 7 of the panel; for a
            // window inside the clip the copies advance by fixed steps with no per-chunk tests.
            struct FGeo {
                const float *xb;
                int64_t g0;      // clip sample of this thread's first chunk in panel 0
                int64_t r0;      // tma: tensor row of the window's first row (floor(w0 / V))
                int32_t coff;    // tma: column of the window's first sample in that row
                int32_t b;
                bool interior;
                bool tail;       // tma: the window reaches the clip's last, partial row of V samples
            };
            auto fgeo = [&](int64_t item) {
                FGeo g;
                int64_t b, tile;
                unit_tile(item, b, tile);
                const int64_t w0 = tile * 128 * A.V - A.G0;
                g.xb = A.x + b * A.ld_x;
                g.g0 = w0 + (int64_t)(ct >> 3) * A.V + (ct & 7) * 8;
                const int64_t wend = w0 + (int64_t)A.win_rows * A.V;
                g.interior = A.vec_ok && w0 >= 0 && wend <= A.N;
                g.tail = A.full_end < A.N && wend > A.full_end;
                g.b = (int32_t)b;
                const int64_t q = (int64_t)((uint32_t)A.G0 / (uint32_t)A.V);
                const int32_t rem = A.G0 - (int32_t)q * A.V;
                g.r0 = tile * 128 - q - (rem ? 1 : 0);
                g.coff = rem ? A.V - rem : 0;
                return g;
            };
            const bool tma = A.tma != 0;  // panels by one TMA tensor copy each (plain rows of 256 B)
            constexpr int FRS = UM_CONV_THREADS / 8;  // rows between a thread's chunks
            const int64_t fgstep = (int64_t)FRS * A.V;
            const int fmine = ct < pchunks ? (pchunks - ct + UM_CONV_THREADS - 1) / UM_CONV_THREADS : 0;
            const uint32_t fdst0 = smem_u32(win_base) + (uint32_t)(ct >> 3) * 256u + (uint32_t)(ct & 7) * 32u;
            auto fetch_panel = [&](const FGeo &g, int p, uint32_t sl) {
                if (tma) {
                    if (ct == 0) {
                        int64_t r0 = g.r0;
                        int32_t col = g.coff + p * 64;
                        if (col >= A.V) {
                            col -= A.V;
                            ++r0;
                        }
                        mbar_expect_tx(&slot_full[sl], 2 * WH);
                        asm volatile(
                            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
                            "{%2, %3, %4}], [%5];" ::"r"(smem_u32(win_base) + sl * 2 * WH),
                            "l"(&A.tmap), "r"(col), "r"((int32_t)r0), "r"(g.b), "r"(smem_u32(&slot_full[sl]))
                            : "memory");
                    }
                    return;
                }
                uint32_t dst = fdst0 + sl * 2 * WH;
                if (g.interior) {
                    const float *src = g.xb + g.g0 + p * 64;
                    for (int i = 0; i < fmine; ++i, dst += FRS * 256u, src += fgstep) {
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16), "l"(src + 4) : "memory");
                    }
                } else {
                    int64_t q = g.g0 + p * 64;
                    for (int i = 0; i < fmine; ++i, dst += FRS * 256u, q += fgstep) {
                        if (A.vec_ok && q >= 0 && q + 8 <= A.N) {
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(g.xb + q) : "memory");
                            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16), "l"(g.xb + q + 4) : "memory");
                        } else {
                            float z[8];
#pragma unroll
                            for (int k = 0; k < 8; ++k) z[k] = (q + k >= 0 && q + k < A.N) ? __ldg(g.xb + q + k) : 0.0f;
                            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "f"(z[0]), "f"(z[1]),
                                         "f"(z[2]), "f"(z[3]) : "memory");
                            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16), "f"(z[4]), "f"(z[5]),
                                         "f"(z[6]), "f"(z[7]) : "memory");
                        }
                    }
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            };
            // the panel sequence: (unit, panel) for panel counter values; the first NS - 1
            // panels are fetched before the loop
            int64_t f_item = u0;
            int f_p = 0;
            uint32_t fc = 0;  // panels fetched so far
            FGeo fg = fgeo(u0 < n_units ? u0 : 0);
            auto fetch_next = [&]() {
                if (f_item < n_units) fetch_panel(fg, f_p, fc % NS);
                else if (!tma) asm volatile("cp.async.commit_group;" ::: "memory");  // keep the group count
                ++fc;
                if (++f_p == A.panels) {
                    f_p = 0;
                    f_item += ustride;
                    if (f_item < n_units) fg = fgeo(f_item);
                }
            };
            const uint32_t lag = tma ? 2u : 1u;  // TMA copies run NS - 2 panels ahead (their slot was released long ago)
            for (uint32_t j = 0; j + lag < NS; ++j) fetch_next();
            uint32_t qc = 0, wcnt = 0;
            for (int64_t item = u0; item < n_units; item += ustride, ++wcnt) {
                int64_t b, tile;
                unit_tile(item, b, tile);
                const int64_t w0 = tile * 128 * A.V - A.G0;
                const bool utail = tma && A.full_end < A.N && w0 + (int64_t)A.win_rows * A.V > A.full_end;
                const float *uxb = A.x + b * A.ld_x;
                int p0, p1;
                unit_passes(item, p0, p1);
                const int64_t own0 = tile * 128 * A.V, own1 = own0 + 128 * (int64_t)A.V;
                uint32_t *rec = A.nfbad ? A.nfbad + b * (int64_t)(1 + WH_NF_CAP) : nullptr;
                if (ct == 0) WH_TRACE(3, wcnt);
                // the unit's exponent: the window's max |x| (finite samples), scanned one unit ahead by
                // the epilogue warps (whose loads also bring the window into L2 for the panel copies)
                mbar_wait_p(&umax_full[wcnt & 3], (wcnt >> 2) & 1, pa, 2, pon);
                const float mx = __uint_as_float(s_umax[wcnt & 3]);
                const int ex = window_exponent(mx);
                const float sc = ldexpf(1.0f, ex);
                if (ct == 0) xring[wcnt & 3] = ldexpf(1.0f, -ex);
                for (int p = 0; p < A.panels; ++p, ++qc) {
                    const uint32_t sl = qc % NS;
                    float *src = reinterpret_cast<float *>(win_base + (size_t)sl * 2 * WH);
                    // this panel's copies (this thread's own, or the TMA copy) have landed
                    {
                        const long long tw = pon ? clock64() : 0;
                        if (tma) mbar_wait(&slot_full[sl], (qc / NS) & 1);
                        else asm volatile("cp.async.wait_group %0;" ::"n"(UM_WSLOTS - 2) : "memory");
                        if (pon) pa.c[0] += (unsigned long long)(clock64() - tw);
                    }
                    float pv[PCH][8];
#pragma unroll
                    for (int i = 0; i < PCH; ++i) {
                        const int c = ct + i * UM_CONV_THREADS;
                        if (c >= pchunks) continue;
                        const float4 *q = reinterpret_cast<const float4 *>(src + (c >> 3) * 64 + (c & 7) * 8);
                        const float4 u = q[0], w = q[1];
                        float (&v)[8] = pv[i];
                        v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
                        if (utail) {
                            // the clip's last row of V samples is partial: the tensor ends before it
                            // (zero fill), its samples come straight from the clip
                            const int64_t g = w0 + (int64_t)(c >> 3) * A.V + p * 64 + (c & 7) * 8;
                            if (g >= A.full_end && g < A.N) {
#pragma unroll
                                for (int k = 0; k < 8; ++k) v[k] = g + k < A.N ? __ldg(uxb + g + k) : 0.0f;
                            }
                        }
                        float m = 0.0f;
#pragma unroll
                        for (int k = 0; k < 8; ++k) m = fmax_nan(m, fabsf(v[k]));
                        if (!(m <= 3.402823466e38f)) {  // non-finite samples (rare): 0, recorded once
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                if (!is_finite_f(v[k])) {
                                    const int64_t g = w0 + (c >> 3) * A.V + p * 64 + (c & 7) * 8 + k;
                                    if (rec && p0 == 0 && g >= own0 && g < own1) nf_record(rec, A.nfctl + 1, g);
                                    v[k] = 0.0f;
                                }
                            }
                        }
                        uint32_t hw[4], lw[4];
                        const uint64_t sc2 = pack_sc2(sc);
#pragma unroll
                        for (int k = 0; k < 4; ++k) split2(v[2 * k], v[2 * k + 1], sc2, hw[k], lw[k]);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            v[k] = __uint_as_float(hw[k]);
                            v[4 + k] = __uint_as_float(lw[k]);
                        }
                    }
                    // every converter has read the fp32 panel: overwrite the slot in place
                    asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
                    uint8_t *whi = win_base + (size_t)sl * 2 * WH;
                    uint8_t *wlo = whi + WH;
#pragma unroll
                    for (int i = 0; i < PCH; ++i) {
                        const int c = ct + i * UM_CONV_THREADS;
                        if (c >= pchunks) continue;
                        const int row = c >> 3, c8 = c & 7;
                        const uint32_t off = (uint32_t)row * 128u + (uint32_t)((c8 ^ (row & 7)) * 16);
                        const float (&v)[8] = pv[i];
                        *reinterpret_cast<uint4 *>(whi + off) = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]),
                                                                          __float_as_uint(v[2]), __float_as_uint(v[3]));
                        *reinterpret_cast<uint4 *>(wlo + off) = make_uint4(__float_as_uint(v[4]), __float_as_uint(v[5]),
                                                                          __float_as_uint(v[6]), __float_as_uint(v[7]));
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
                    if (ct == 0) window_ready(sl, qc);
                    // refill the slot of an earlier panel once its MMAs are done (TMA: only the
                    // issuing thread waits)
                    if (qc >= lag && (!tma || ct == 0)) {
                        const uint32_t ps = (qc - lag) % NS;
                        mbar_wait_p(&win_empty[ps], ((qc - lag) / NS) & 1, pa, 1, pon);
                    }
                    fetch_next();
                }
                if (ct == 0) WH_TRACE(7, wcnt);
            }
            if (!tma) asm volatile("cp.async.wait_all;" ::: "memory");
        } else if (!PS && A.conv_regs) {
            // Register-prefetch path (no staging buffer): each thread loads its first CONV_RC
            // chunks of the next window into registers while the MMAs of the previous unit
            // run, then converts from registers once the window buffer is free.  Larger
            // windows (c5: 13.5 chunks per thread) read their extra chunks twice: once
            // before the wait for the window max, again (L2 hits) after it.
            auto load8 = conv_load8;
            auto split8 = [&](const float (&in)[8], float sc, uint32_t (&hw)[4], uint32_t (&lw)[4]) {
                const uint64_t sc2 = pack_sc2(sc);
#pragma unroll
                for (int k = 0; k < 4; ++k) split2(in[2 * k], in[2 * k + 1], sc2, hw[k], lw[k]);
            };
            uint32_t wcnt = 0;
            for (int64_t item = u0; item < n_units; item += ustride, ++wcnt) {
                int64_t b, tile;
                unit_tile(item, b, tile);
                const int64_t w0 = tile * 128 * A.V - A.G0;
                const float *xb = A.x + b * A.ld_x;
                const uint32_t wb = wcnt % A.win_bufs;
                const int32_t in_lo = (int32_t)(w0 < 0 ? -w0 : 0);
                const int64_t in_hi64 = A.N - w0;
                const int32_t in_hi = (int32_t)(in_hi64 < (int64_t)0x7fffffff ? in_hi64 : (int64_t)0x7fffffff);
                if (ct == 0) {
                    WH_TRACE(3, wcnt);
                    window_prefetch(item + (UM_PF + 1) * ustride);
                }
                // this unit's window (the first one was fetched at launch)
                if (item != u0) conv_fetch(item);
                float (&v)[CONV_RC][8] = cv;
                float mx = cmx;
                auto chunk_off = [&](int c) {
            int row, cc;
            chunk_rc(A, c, row, cc);
            return (int32_t)(row * A.V + cc * 8);
        };
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
                if (lane == 0) red[cw] = mx;
                asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
                mx = red[0];
#pragma unroll
                for (int i = 1; i < UM_CONV_WARPS; ++i) mx = fmaxf(mx, red[i]);
                const int ex = window_exponent(mx);
                const float sc = ldexpf(1.0f, ex);
                // split into hi/lo fp16 in registers (in place: 8 fp32 -> 4 hi + 4 lo words)
                // while the window buffer is still busy; only the stores wait for it
#pragma unroll
                for (int i = 0; i < CONV_RC; ++i) {
                    uint32_t hw[4], lw[4];
                    split8(v[i], sc, hw, lw);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        v[i][k] = __uint_as_float(hw[k]);
                        v[i][4 + k] = __uint_as_float(lw[k]);
                    }
                }
                if (ct == 0) WH_TRACE(5, wcnt);
                mbar_wait_p(&win_empty[wb], ((wcnt / A.win_bufs) & 1) ^ 1, pa, 1, pon);
                if (ct == 0) WH_TRACE(6, wcnt);
                uint8_t *whi = win_base + (size_t)wb * 2 * WH;
                uint8_t *wlo = whi + WH;
                auto put = [&](int c, const uint32_t (&hw)[4], const uint32_t (&lw)[4]) {
                    int row, cc;
                    chunk_rc(A, c, row, cc);
                    const int panel = cc >> 3, c8 = cc & 7;
                    const uint32_t off =
                        (uint32_t)panel * panel_bytes + (uint32_t)row * 128u + (uint32_t)((c8 ^ (row & 7)) * 16);
                    *reinterpret_cast<uint4 *>(whi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    *reinterpret_cast<uint4 *>(wlo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                };
#pragma unroll
                for (int i = 0; i < CONV_RC; ++i) {
                    const int c = ct + i * UM_CONV_THREADS;
                    if (c < chunks) {
                        const uint32_t hw[4] = {__float_as_uint(v[i][0]), __float_as_uint(v[i][1]),
                                                __float_as_uint(v[i][2]), __float_as_uint(v[i][3])};
                        const uint32_t lw[4] = {__float_as_uint(v[i][4]), __float_as_uint(v[i][5]),
                                                __float_as_uint(v[i][6]), __float_as_uint(v[i][7])};
                        put(c, hw, lw);
                    }
                }
                for (int c = ct + CONV_RC * UM_CONV_THREADS; c < chunks; c += UM_CONV_THREADS) {
                    float t[8];
                    uint32_t hw[4], lw[4];
                    load8(xb, w0, chunk_off(c), in_lo, in_hi, t);
                    if (cbad)
#pragma unroll
                        for (int k = 0; k < 8; ++k) t[k] = is_finite_f(t[k]) ? t[k] : 0.0f;
                    split8(t, sc, hw, lw);
                    put(c, hw, lw);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (ct == 0) xring[wcnt & 3] = ldexpf(1.0f, -ex);
                asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
                if (ct == 0) {
                    WH_TRACE(7, wcnt);
                    window_ready(wb, wcnt);
                }
            }
        } else if (!PS) {
        if (A.use_stg && ct == 0 && u0 < n_units) issue(u0);
        uint32_t wcnt = 0;
        for (int64_t item = u0; item < n_units; item += ustride, ++wcnt) {
            int64_t b, tile;
            unit_tile(item, b, tile);
            const int64_t w0 = tile * 128 * A.V - A.G0;
            const float *xb = A.x + b * A.ld_x;
            const uint32_t wb = wcnt % A.win_bufs;
            int64_t slo, shi;
            staged(item, slo, shi);
            if (ct == 0) {
                WH_TRACE(3, wcnt);
                window_prefetch(item + (UM_PF + 1) * ustride);
            }
            if (A.use_stg) mbar_wait_p(&stg_full, wcnt & 1, pa, 0, pon);
            if (ct == 0) WH_TRACE(4, wcnt);
            // chunk c = 8 consecutive samples: (row, column chunk) = chunk_rc(c) (cpr = panels * 8
            // chunks per row); window offsets are 32-bit
            const int32_t st_lo = (int32_t)(slo - w0), st_hi = (int32_t)(shi - w0);  // staged range
            const int32_t in_lo = (int32_t)(w0 < 0 ? -w0 : 0);                       // clip start
            const int64_t in_hi64 = A.N - w0;                                          // clip end
            const int32_t in_hi = (int32_t)(in_hi64 < (int64_t)0x7fffffff ? in_hi64 : (int64_t)0x7fffffff);
            auto load8 = [&](int32_t off, float (&v)[8]) {
                if (off >= st_lo && off + 8 <= st_hi) {
                    const float4 u = *reinterpret_cast<const float4 *>(stg + off);
                    const float4 w = *reinterpret_cast<const float4 *>(stg + off + 4);
                    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
                } else if (A.vec_ok && off >= in_lo && off + 8 <= in_hi) {
                    const float4 *g = reinterpret_cast<const float4 *>(xb + w0 + off);
                    const float4 u = __ldg(g), w = __ldg(g + 1);
                    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w; v[4] = w.x; v[5] = w.y; v[6] = w.z; v[7] = w.w;
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int32_t o = off + i;
                        v[i] = (o >= in_lo && o < in_hi) ? ((o >= st_lo && o < st_hi) ? stg[o] : __ldg(xb + w0 + o)) : 0.0f;
                    }
                }
            };
            auto chunk_off = [&](int c) {
                int row, cc;  // cc = panel * 8 + c8
                chunk_rc(A, c, row, cc);
                return row * A.V + cc * 8;
            };
            // pass 1: max |x| over the window (NaN-propagating: one test finds non-finite input)
            float mx = 0.0f;
#pragma unroll 4
            for (int c = ct; c < chunks; c += UM_CONV_THREADS) {
                float v[8];
                load8(chunk_off(c), v);
                mx = fmax_nan(mx, fmax_nan(fmax_nan(fmax_nan(fabsf(v[0]), fabsf(v[1])), fmax_nan(fabsf(v[2]), fabsf(v[3]))),
                                           fmax_nan(fmax_nan(fabsf(v[4]), fabsf(v[5])), fmax_nan(fabsf(v[6]), fabsf(v[7])))));
            }
            // non-finite samples (rare): excluded from the max here, replaced by 0 and recorded
            // in pass 2
            const bool tbad = !(mx <= 3.402823466e38f);
            if (tbad) {
                mx = 0.0f;
                for (int c = ct; c < chunks; c += UM_CONV_THREADS) {
                    float v[8];
                    load8(chunk_off(c), v);
#pragma unroll
                    for (int k = 0; k < 8; ++k) mx = fmaxf(mx, is_finite_f(v[k]) ? fabsf(v[k]) : 0.0f);
                }
            }
            int p0s, p1s;
            unit_passes(item, p0s, p1s);
            const int64_t own0 = tile * 128 * A.V, own1 = own0 + 128 * (int64_t)A.V;
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (lane == 0) red[cw] = mx;
            asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
            mx = red[0];
#pragma unroll
            for (int i = 1; i < UM_CONV_WARPS; ++i) mx = fmaxf(mx, red[i]);
            const int ex = window_exponent(mx);
            const float sc = ldexpf(1.0f, ex);
            // wait until the MMAs that read this window buffer win_bufs items ago are done
            if (ct == 0) WH_TRACE(5, wcnt);
            mbar_wait_p(&win_empty[wb], ((wcnt / A.win_bufs) & 1) ^ 1, pa, 1, pon);
            if (ct == 0) WH_TRACE(6, wcnt);
            uint8_t *whi = win_base + (size_t)wb * 2 * WH;
            uint8_t *wlo = whi + WH;
#pragma unroll 2
            for (int c = ct; c < (WH_DBG(2) ? 0 : chunks); c += UM_CONV_THREADS) {
                int row, cc;
                    chunk_rc(A, c, row, cc);
                const int panel = cc >> 3, c8 = cc & 7;
                float v[8];
                load8(row * A.V + cc * 8, v);
                if (tbad) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (!is_finite_f(v[k])) {
                            const int64_t g = w0 + row * A.V + cc * 8 + k;
                            if (p0s == 0 && g >= own0 && g < own1 && A.nfbad)
                                nf_record(A.nfbad + b * (int64_t)(1 + WH_NF_CAP), A.nfctl + 1, g);
                            v[k] = 0.0f;
                        }
                    }
                }
                uint32_t hw[4], lw[4];
                const uint64_t sc2 = pack_sc2(sc);
#pragma unroll
                for (int i = 0; i < 4; ++i) split2(v[2 * i], v[2 * i + 1], sc2, hw[i], lw[i]);  // hi = rn(x), lo = rn(x - hi)
                const uint32_t off = (uint32_t)panel * panel_bytes + (uint32_t)row * 128u +
                                     (uint32_t)((c8 ^ (row & 7)) * 16);
                *reinterpret_cast<uint4 *>(whi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4 *>(wlo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (ct == 0) xring[wcnt & 3] = ldexpf(1.0f, -ex);
            asm volatile("bar.sync 1, %0;" ::"r"(UM_CONV_THREADS) : "memory");
            // staging is free again: prefetch the next item's window
            if (A.use_stg && ct == 0 && item + ustride < n_units) issue(item + ustride);
            if (ct == 0) {
                WH_TRACE(7, wcnt);
                window_ready(wb, wcnt);
            }
        }
        }
    } else {
        // ===================== epilogue ==============================================
        const int quad = warp & 3;          // TMEM lanes 32*quad .. 32*quad+31
        const int half = (warp - 2 - UM_CONV_WARPS) >> 2;  // which 16-column units
        const int m = quad * 32 + lane;     // row within the tile
        const int et = (int)threadIdx.x - (64 + UM_CONV_THREADS);  // 0 .. 255
        const bool vec = A.out_vec_ok;
        uint32_t acnt = 0, ucnt = 0;
        float lmin = INFINITY, lmax = -INFINITY;
        // Write-once per-clip min-max (scalogram.py:77-83's affine map per clip): the units
        // this CTA finished whose clip was still in flight elsewhere, oldest first -- a
        // contiguous run of this CTA's unit sequence [pend_item, pend_item + pend*ustride).
        // Their raw values sit in L2 (written one or two units ago); once every unit of the
        // clip has arrived, the CTA re-reads its own tile region and overwrites it normalised,
        // so the scalogram reaches HBM (close to) once, with no separate pass.
        int64_t pend_item = u0;
        int pend = 0;
        auto clip_done = [&](int64_t b) {
            uint32_t c;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(A.arrive + b) : "memory");
            return c >= A.arrive_target;
        };
        auto normalise = [&](int64_t item) {
            int64_t b, tile;
            unit_tile(item, b, tile);
            int pb, pe;
            unit_passes(item, pb, pe);
            const float lo = key2f(__ldcg(A.minmax + 2 * b)), hi = key2f(__ldcg(A.minmax + 2 * b + 1));
            const bool constant = hi == lo;
            const float sc = constant ? 0.0f : 1.0f / (hi - lo);
            int64_t f0, f1;
            if (A.rs > 1) {
                f0 = (tile * 128 + A.rs - 1) / A.rs;
                f1 = (tile * 128 + 128 + A.rs - 1) / A.rs;
            } else {
                f0 = tile * 128 * P;
                f1 = f0 + 128 * P;
            }
            if (f1 > A.F) f1 = A.F;
            const int len = (int)(f1 - f0);
            if (len <= 0) return;
            const bool v4 = vec && (f0 % 4) == 0;
            const int nq = v4 ? (len + 3) / 4 : len;  // float4 groups (or scalars) per row
            float *clip = reinterpret_cast<float *>(A.out) + b * (int64_t)A.S * A.F;
            for (int p = pb; p < pe; ++p) {
                const int4 pinfo = s_pass[p];
                const int s0 = pinfo.z & 0xffff, ns = pinfo.z >> 16;
                float *base = clip + (int64_t)s0 * A.F + f0;
                for (int idx = et; idx < ns * nq; idx += 32 * UM_EPI_WARPS) {
                    const int row = idx / nq, q = idx - row * nq;
                    float *ptr = base + (int64_t)row * A.F;
                    if (v4 && 4 * q + 4 <= len) {
                        float4 v = __ldcg(reinterpret_cast<const float4 *>(ptr) + q);
                        if (constant) {
                            v = make_float4(0.f, 0.f, 0.f, 0.f);
                        } else {
                            v.x = (v.x - lo) * sc; v.y = (v.y - lo) * sc; v.z = (v.z - lo) * sc; v.w = (v.w - lo) * sc;
                        }
                        st_na(reinterpret_cast<float4 *>(ptr) + q, v);
                    } else {
                        const int j0 = v4 ? 4 * q : q, j1 = v4 ? (4 * q + 4 < len ? 4 * q + 4 : len) : q + 1;
                        for (int j = j0; j < j1; ++j) st_na(ptr + j, constant ? 0.0f : (__ldcg(ptr + j) - lo) * sc);
                    }
                }
            }
        };
        // Normalise the finished units whose clips are complete.  The decision for the oldest
        // pending unit is CTA-uniform (epilogue thread 0 decides, a named barrier publishes
        // it): done -> normalise it here; still running after a bounded wait (only when more
        // than `keep` units are pending, or at the end) -> hand it to the fix-up kernel
        // (k_minmax_fixup), which normalises abandoned units after this launch.  No CTA ever
        // waits unboundedly on another, so concurrent launches cannot deadlock.
        auto decide = [&](int64_t b, bool may_wait) -> int {
            if (et == 0) {
                int st = clip_done(b) ? 1 : 0;
                if (!st && may_wait) {
                    const unsigned long long t0 = globaltimer_ns();
                    while (!(st = clip_done(b)) && globaltimer_ns() - t0 < 200000ull) __nanosleep(512);
                    if (!st) st = 2;
                }
                s_decide = st;
            }
            asm volatile("bar.sync 2, %0;" ::"r"(32 * UM_EPI_WARPS) : "memory");
            const int st = s_decide;
            asm volatile("bar.sync 2, %0;" ::"r"(32 * UM_EPI_WARPS) : "memory");
            return st;
        };
        auto drain = [&](int keep) {
            while (pend > 0) {
                int64_t b, tile;
                unit_tile(pend_item, b, tile);
                const int st = A.force_fixup ? 2 : decide(b, pend > keep);
                if (st == 0) break;
                if (st == 1) {
                    normalise(pend_item);
                } else if (et == 0) {
                    // abandoned: flag (tile pair, pass group, CTA) in the clip's bitmap
                    const uint32_t v = (uint32_t)pend_item / pg32, bit =
                        (((v - (uint32_t)b * tpu32) * pg32 + ((uint32_t)pend_item - v * pg32)) * CG) + rank;
                    atomicOr(A.abandon + b * A.ab_words + (bit >> 5), 1u << (bit & 31));
                }
                pend_item += ustride;
                --pend;
            }
        };
        // Panel streaming (fp16): max |x| over the finite samples of a unit's window, one unit ahead
        // of the converters (no pre-pass over the input; the loads allocate in L2, so the panel
        // copies that follow read the window from there).  seq = the unit's position in this CTA's
        // sequence; the result goes to s_umax[seq % 4], published through umax_full.
        auto scan_window = [&](int64_t item, uint32_t seq) {
            if (item >= n_units) return;
            int64_t sb, stile;
            unit_tile(item, sb, stile);
            const int64_t w0 = stile * 128 * A.V - A.G0;
            const int64_t lo = w0 > 0 ? w0 : 0;
            int64_t hi = w0 + (int64_t)A.win_rows * A.V;
            if (hi > A.N) hi = A.N;
            const float *xb = A.x + sb * A.ld_x;
            if (et == 0) s_umax[seq & 3] = 0u;
            asm volatile("bar.sync 2, %0;" ::"r"(32 * UM_EPI_WARPS) : "memory");
            float mx = 0.0f;
            if (A.vec_ok) {
                const int64_t lo4 = (lo + 3) & ~(int64_t)3, hi4 = hi & ~(int64_t)3;
                for (int64_t i = lo + et; i < lo4 && i < hi; i += 32 * UM_EPI_WARPS) {
                    const float v = fabsf(__ldg(xb + i));
                    mx = fmaxf(mx, v <= 3.402823466e38f ? v : 0.0f);
                }
                constexpr int64_t ST = 4 * 32 * UM_EPI_WARPS;  // samples per sweep of the epilogue threads
                int64_t i = lo4 + 4 * (int64_t)et;
                for (; i + 7 * ST + 4 <= hi4; i += 8 * ST) {  // eight independent loads in flight per thread
                    float4 v[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const float4 *>(xb + i + k * ST));
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float a0 = fabsf(v[k].x), a1 = fabsf(v[k].y), a2 = fabsf(v[k].z), a3 = fabsf(v[k].w);
                        mx = fmaxf(mx, a0 <= 3.402823466e38f ? a0 : 0.0f);
                        mx = fmaxf(mx, a1 <= 3.402823466e38f ? a1 : 0.0f);
                        mx = fmaxf(mx, a2 <= 3.402823466e38f ? a2 : 0.0f);
                        mx = fmaxf(mx, a3 <= 3.402823466e38f ? a3 : 0.0f);
                    }
                }
                for (; i + 4 <= hi4; i += ST) {
                    const float4 v = __ldg(reinterpret_cast<const float4 *>(xb + i));
                    const float a0 = fabsf(v.x), a1 = fabsf(v.y), a2 = fabsf(v.z), a3 = fabsf(v.w);
                    mx = fmaxf(mx, a0 <= 3.402823466e38f ? a0 : 0.0f);
                    mx = fmaxf(mx, a1 <= 3.402823466e38f ? a1 : 0.0f);
                    mx = fmaxf(mx, a2 <= 3.402823466e38f ? a2 : 0.0f);
                    mx = fmaxf(mx, a3 <= 3.402823466e38f ? a3 : 0.0f);
                }
                for (int64_t i = (hi4 > lo4 ? hi4 : lo4) + et; i < hi; i += 32 * UM_EPI_WARPS) {
                    const float v = fabsf(__ldg(xb + i));
                    mx = fmaxf(mx, v <= 3.402823466e38f ? v : 0.0f);
                }
            } else {
                for (int64_t i = lo + et; i < hi; i += 32 * UM_EPI_WARPS) {
                    const float v = fabsf(__ldg(xb + i));
                    mx = fmaxf(mx, v <= 3.402823466e38f ? v : 0.0f);
                }
            }
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (lane == 0) atomicMax(&s_umax[seq & 3], __float_as_uint(mx));  // non-negative floats order as integers
            asm volatile("bar.sync 2, %0;" ::"r"(32 * UM_EPI_WARPS) : "memory");
            if (et == 0) mbar_arrive(&umax_full[seq & 3]);
        };
        if (PS && !A.tf32) scan_window(u0, 0u);
        for (int64_t item = u0; item < n_units; item += ustride, ++ucnt) {
            int64_t b, tile;
            unit_tile(item, b, tile);
            if (PS && !A.tf32) scan_window(item + ustride, ucnt + 1);
            const int64_t mrow = tile * 128 + m;  // global row (beyond rows_total: no frames)
            // first frame of this row (rs > 1: only every rs-th row is a frame)
            const int64_t frame0 = A.rs > 1 ? mrow / A.rs : mrow * P;
            const int64_t rem_frames = (A.rs > 1 && mrow % A.rs) ? 0 : A.F - frame0;
            const int nvalid = rem_frames <= 0 ? 0 : (rem_frames >= P ? P : (int)rem_frames);
            int pb, pe;
            unit_passes(item, pb, pe);
            for (int p = pb; p < pe; ++p, ++acnt) {
                const int4 pinfo = s_pass[p];
                const uint32_t ab = acnt % A.n_acc;
                if (warp == 2 + UM_CONV_WARPS && p == pb) WH_TRACE(8, ucnt);
                mbar_wait_p(&acc_full[ab], (acnt / A.n_acc) & 1, pa, 0, pon);
                tc_fence_after();
                if (warp == 2 + UM_CONV_WARPS && p == pb) WH_TRACE(9, ucnt);
                const float e = xring[ucnt & 3];
                const uint32_t tbase = tmem + ((uint32_t)(quad * 32) << 16) + ab * (uint32_t)A.acc_stride;
                // corr_j lives at column 2C-1-j: the 16 corr values of unit u0 are loaded
                // from cbase - u0 in reverse order
                const uint32_t cbase = tbase + 2u * (uint32_t)pinfo.w - 16u;
                const int s0 = pinfo.z & 0xffff, ns = pinfo.z >> 16;
                if (!WH_DBG(1)) switch (A.output) {
                    case WH_OUT_COMPLEX64:
                        epi_pass<CC, P, WH_OUT_COMPLEX64, AC>(A, s_spow, tbase, cbase, s0, ns, pinfo.w, half, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    case WH_OUT_ABS:
                        epi_pass<CC, P, WH_OUT_ABS, AC>(A, s_spow, tbase, cbase, s0, ns, pinfo.w, half, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    case WH_OUT_POWER:
                        epi_pass<CC, P, WH_OUT_POWER, AC>(A, s_spow, tbase, cbase, s0, ns, pinfo.w, half, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    case WH_OUT_LOG_DB:
                        epi_pass<CC, P, WH_OUT_LOG_DB, AC>(A, s_spow, tbase, cbase, s0, ns, pinfo.w, half, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                    default:
                        epi_pass<CC, P, WH_OUT_LOG1P, AC>(A, s_spow, tbase, cbase, s0, ns, pinfo.w, half, b, frame0, nvalid, e, vec, lmin, lmax);
                        break;
                }
                // the columns read were re-zeroed; release the buffer to the MMA issuer
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (warp == 2 + UM_CONV_WARPS && p == pe - 1) WH_TRACE(10, ucnt);
                if (lane == 0) {
                    // TMEM accesses are ordered by wait::st + fence::before_thread_sync; the
                    // global stores need no ordering against the MMA: relaxed arrive
                    if (CG == 2 && !leader) mbar_arrive_leader_relaxed(&acc_empty[ab]);
                    else mbar_arrive(&acc_empty[ab]);
                }
            }
            if (A.minmax) {
                // this unit's min / max into the clip's keys (order-independent atomics)
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
                    lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
                }
                if (lane == 0 && lmin <= lmax) {
                    atomicMin(A.minmax + 2 * b, f2key(lmin));
                    atomicMax(A.minmax + 2 * b + 1, f2key(lmax));
                }
                lmin = INFINITY;
                lmax = -INFINITY;
                if (VS == 2 && A.arrive) {
                    // all epilogue warps' stores and key atomics of this unit are done: one
                    // arrival per CTA and unit on the clip's counter (release at GPU scope)
                    if (lane == 0) __threadfence();
                    asm volatile("bar.sync 2, %0;" ::"r"(32 * UM_EPI_WARPS) : "memory");
                    if (et == 0) {
                        __threadfence();
                        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.arrive + b) : "memory");
                    }
                    if (!A.arrive_only) {
                        ++pend;
                        drain(2);  // at most 2 units behind (a bounded L2 footprint)
                    }
                }
            }
        }
        if (VS == 2 && A.arrive && !A.arrive_only) drain(0);
    }
    if (pon && lane == 0) {
        const int role = warp == 0 ? PR_PROD : warp == 1 ? (leader ? PR_MMA : PR_RELAY) : warp < 2 + UM_CONV_WARPS ? PR_CONV : PR_EPI;
        prof_flush(pa, A.prof, role);
    }
    tc_fence_before();
    cta_pair_sync<CG>();
    if (kDiag && A.trace && threadIdx.x == 0 && blockIdx.x < 256) {
        A.trace[16 * 32 + 2 * blockIdx.x + 1] = (long long)globaltimer_ns();
        if (blockIdx.x == 0) A.trace[14 * 32 + 1] = clock64();
    }
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        if constexpr (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
    // Non-finite input samples: the last CTA to finish writes the exact values of the
    // coefficients they reach (nf_fixup_clip) -- normally it finds the launch's flag clear
    if (A.nfctl) {
        __shared__ int s_nf_last;
        if (threadIdx.x == 0) {
            __threadfence();
            s_nf_last = atomicAdd(A.nfctl, 1u) == gridDim.x - 1 ? 1 : 0;
        }
        __syncthreads();
        if (s_nf_last) {
            __threadfence();
            if (*reinterpret_cast<volatile uint32_t *>(A.nfctl + 1)) {
                NfArgs na{};
                na.x = A.x; na.ld_x = A.ld_x; na.N = A.N; na.hop = A.hop; na.F = A.F; na.S = A.S;
                na.wavelet = A.wavelet; na.output = A.output; na.scales = A.scales; na.half = A.half;
                na.C = A.Cw; na.Bw = A.Bw; na.out = A.out; na.mm = A.minmax; na.bad = A.nfbad;
                for (int64_t b = 0; b < A.clips; ++b) nf_fixup_clip(na, b, threadIdx.x, blockDim.x);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                A.nfctl[0] = 0u;
                A.nfctl[1] = 0u;
            }
        }
    }
}

// ---- write-once min-max: fix-up of abandoned units ---------------------------------------
// k_umma normalises every unit of a min-max plan itself once the unit's clip is complete; a
// unit whose clip did not complete within a bounded wait (another kernel holding SMs, a
// straggler at the very end) is flagged in its clip's bitmap instead.  This kernel, launched
// right after k_umma on the same stream, normalises exactly the flagged regions (normally
// none: every block reads its clips' bitmap words and exits).
struct FixupArgs {
    float *out;
    const uint32_t *minmax, *abandon;
    const int4 *passes;       // packed pass table (x, y = groups, z = s0 | ns << 16, w = cols)
    int64_t clips, F;
    int32_t S, P, rs, cg, tpu, pgroups, ppu, n_passes, ab_words, vec;
};

__global__ void k_minmax_fixup(const FixupArgs a) {
    for (int64_t b = blockIdx.x; b < a.clips; b += gridDim.x) {
        const float lo = key2f(a.minmax[2 * b]), hi = key2f(a.minmax[2 * b + 1]);
        const bool constant = hi == lo;
        const float sc = constant ? 0.0f : 1.0f / (hi - lo);
        float *clip = a.out + b * (int64_t)a.S * a.F;
        for (int w = 0; w < a.ab_words; ++w) {
            uint32_t bits = a.abandon[b * a.ab_words + w];
            while (bits) {
                const int bit = 32 * w + __ffs(bits) - 1;
                bits &= bits - 1;
                const int rank = bit % a.cg, pg = (bit / a.cg) % a.pgroups, tp = bit / a.cg / a.pgroups;
                const int64_t tile = (int64_t)a.cg * tp + rank;
                int64_t f0, f1;
                if (a.rs > 1) {
                    f0 = (tile * 128 + a.rs - 1) / a.rs;
                    f1 = (tile * 128 + 128 + a.rs - 1) / a.rs;
                } else {
                    f0 = tile * 128 * a.P;
                    f1 = f0 + 128 * a.P;
                }
                if (f1 > a.F) f1 = a.F;
                const int len = (int)(f1 - f0);
                const int p0 = pg * a.ppu, p1 = p0 + a.ppu < a.n_passes ? p0 + a.ppu : a.n_passes;
                for (int p = p0; p < p1 && len > 0; ++p) {
                    const int s0 = a.passes[p].z & 0xffff, ns = a.passes[p].z >> 16;
                    for (int idx = threadIdx.x; idx < ns * len; idx += blockDim.x) {
                        const int row = idx / len, j = idx - row * len;
                        float *ptr = clip + (int64_t)(s0 + row) * a.F + f0 + j;
                        *ptr = constant ? 0.0f : (*ptr - lo) * sc;
                    }
                }
            }
        }
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
    int32_t P, Cc, G0, cg, tf32;
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
    // MMA1's B = [hi fwd (nc rows, columns c0..C-1) | lo rev (ncorr rows, C-1..c1)],
    // MMA2's B = hi rev (ncorr rows).  cg = 1: the tile is [MMA1 B | MMA2 B];  cg = 2: each
    // CTA's block is [its half of MMA1 B | its half of MMA2 B] (CTA 0 the first halves)
    uint8_t *tile0 = a.bank + tl.byte_off;
    const int nc = tl.ncols, ncorr = tl.ncorr, n1 = nc + ncorr;
    const double norm = pow(M_PI * a.Bw, -0.5);
    const double w = 2.0 * M_PI * a.C;
    const int KS = a.tf32 ? 32 : 64;  // taps per K-step (128 B per operand row)
    for (int idx = threadIdx.x; idx < tl.ncols * KS; idx += blockDim.x) {
        const int n = idx / KS, e = idx % KS;
        const int col = tl.c0 + n;
        double v = 0.0;
        if (col < ps.ns * CP) {
            const int s = ps.s0 + col / CP;
            const int c = (col / a.P) % a.Cc;
            const int r = col % a.P;
            const int64_t g = (int64_t)tl.k * KS + e;
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
        // the two parts of the tap: fp16 (hi = rn16(v), lo = rn16(v - hi)) or tf32 (fp32 words
        // rounded to 10 mantissa bits -- their low 13 bits are zero, so the tensor core's
        // treatment of those bits cannot matter)
        struct Part { uint32_t bits; };
        Part h, l;
        if (a.tf32) {
            auto rtf32 = [](double x) {
                const uint32_t b = __float_as_uint((float)x);
                return (b + 0x1000u) & 0xffffe000u;
            };
            h.bits = rtf32(v);
            l.bits = rtf32(v - (double)__uint_as_float(h.bits));
        } else {
            const __half hh = __double2half(v);
            const __half ll = __double2half(v - (double)__half2float(hh));
            h.bits = __half_as_ushort(hh);
            l.bits = __half_as_ushort(ll);
        }
        auto put = [&](uint8_t *base, int row, Part val) {
            if (a.tf32) {
                const uint32_t off = (uint32_t)row * 128u + (uint32_t)((((e >> 2) ^ (row & 7)) << 4) + (e & 3) * 4);
                *reinterpret_cast<uint32_t *>(base + off) = val.bits;
            } else {
                const uint32_t off = (uint32_t)row * 128u + (uint32_t)((((e >> 3) ^ (row & 7)) << 4) + (e & 7) * 2);
                *reinterpret_cast<uint16_t *>(base + off) = (uint16_t)val.bits;
            }
        };
        const int rrev = C - 1 - col;  // row index in the reversed parts
        const bool corr = rrev < ncorr;
        if (a.cg == 2) {
            uint8_t *blk0 = tile0, *blk1 = tile0 + tl.blk1_delta;
            auto put1 = [&](int row, Part val) {  // row of MMA1's B
                if (row < n1 / 2) put(blk0, row, val);
                else put(blk1, row - n1 / 2, val);
            };
            put1(n, h);
            if (corr) {
                put1(nc + rrev, l);
                if (rrev < ncorr / 2) put(blk0, n1 / 2 + rrev, h);
                else put(blk1, n1 / 2 + rrev - ncorr / 2, h);
            }
        } else {
            put(tile0, n, h);
            if (corr) {
                put(tile0, nc + rrev, l);
                put(tile0 + (size_t)n1 * 128, rrev, h);
            }
        }
    }
}

using UmmaKernel = void (*)(const UmmaArgs);
// the kernel variant a plan runs (see k_umma)
static int umma_variant(const Plan &p) {
    if (p.pstream) return 1;
    if (p.Lmax > UM_LMAX1) return 3;
    return (p.norm == WH_NORM_MINMAX && p.minmax_mode != 0) ? 2 : 0;
}

template <int CC, int CG>
static UmmaKernel pick_p(int P, int vs) {
    if (vs == 1) return P == 1 ? k_umma<CC, 1, CG, 1> : nullptr;  // panel streaming: one frame per row
    if (vs == 2) {  // opt-in min-max modes (CTA pairs, 1 or 2 phases per row)
        if constexpr (CG == 2) {
            if (P == 1) return k_umma<CC, 1, CG, 2>;
            if (P == 2) return k_umma<CC, 2, CG, 2>;
        }
        return nullptr;
    }
    if (vs == 3) {  // very long filters: two accumulator sets per buffer (CTA pairs, 1 / 2 / 4 phases per row)
        if constexpr (CG == 2) {
            if (P == 1) return k_umma<CC, 1, CG, 3>;
            if (P == 2) return k_umma<CC, 2, CG, 3>;
#ifndef WH_DEV_BUILD
            if (P == 4) return k_umma<CC, 4, CG, 3>;
#endif
        }
        return nullptr;
    }
    switch (P) {
        case 1: return k_umma<CC, 1, CG, 0>;
        case 2: return k_umma<CC, 2, CG, 0>;
#ifdef WH_DEV_BUILD  // development builds (build.py --dev): two phase counts only, a fraction of the compile time
        default: return nullptr;
    }
}
template <int CC, int CG>
static UmmaKernel pick_p_unused(int P) {
    switch (P) {
#endif
        case 4: return k_umma<CC, 4, CG, 0>;
        case 8: return k_umma<CC, 8, CG, 0>;
        case 16: return k_umma<CC, 16, CG, 0>;
        case 32: return k_umma<CC, 32, CG, 0>;
        case 64: return k_umma<CC, 64, CG, 0>;
        default: return nullptr;
    }
}

static UmmaKernel umma_kernel(int Cc, int P, int CG, int vs) {
    if (CG == 2) return Cc == 2 ? pick_p<2, 2>(P, vs) : pick_p<1, 2>(P, vs);
    return Cc == 2 ? pick_p<2, 1>(P, vs) : pick_p<1, 1>(P, vs);
}

int umma_supported(const Plan &p, std::string *why) {
    const int64_t H = p.hop;
    // (accuracy bounds: UM_LMAX1 / UM_LMAX2)
    if (p.Lmax > UM_LMAX2) {
        if (why) *why = "tap support too long for the split-fp16 accumulation within tolerance (half width > 5632)";
        return WH_E_UNSUPPORTED;
    }
    if (p.Lmax > UM_LMAX1 && !(H <= 64 && 64 % H == 0 && 64 / H <= 4)) {
        if (why) *why = "very long filters (half width > 3360) run on the tensor cores for hops 16, 32 and 64 only";
        return WH_E_UNSUPPORTED;
    }
    const bool small = H <= 64 && 64 % H == 0;
    const bool big = H % 64 == 0 && H < 256;
    const bool strided = H >= 256 && H % 128 == 0;  // rows of 128 samples, every (H/128)-th a frame
    const int64_t lcm64 = H / std::gcd(H, (int64_t)64) * 64;
    const bool mid = !small && !big && !strided && lcm64 <= 256;  // 3, 6, 12, 24, 48, 96: rows of 192
    // panel streaming (rows of hop samples): hops 256..4096 that are multiples of 64 whose
    // columns fit one pass
    const int64_t cc = p.wavelet == WH_WAVELET_CMOR ? 2 : 1;
    if (H >= 256 && H <= 4096 && H % 64 == 0 && cc * p.S <= 128 && p.S <= 65535) return WH_OK;
    if (!small && !big && !strided && !mid) {
        if (why) *why = "hop must divide 64 or 192, or be 128 or 192, or a multiple of 128 from 256";
        return WH_E_UNSUPPORTED;
    }
    const int64_t V = small ? 64 : (big ? H : (mid ? lcm64 : 128));
    const int64_t P = strided ? 1 : V / H;
    const int64_t maxg = (p.Lmax + V - 1) / V * V + p.Lmax + (P - 1) * (strided ? 0 : H);  // longest K range
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

// compact smem tile format (s_tile): 16-byte descriptor offsets, c0 and ncols < 2^8, tiles
// 128-byte aligned in the bank
static int ncheck_tiles(const Plan &p) {
    for (auto &t : p.tiles)
        if ((int64_t)t.k * p.ks / p.V >= 4096 || (!p.pstream && p.V / 64 > 16) || t.c0 > 255 || t.ncols > 255 ||
            (t.byte_off & 127))
            return fail(WH_E_UNSUPPORTED, "UMMA engine: tile table out of range");
    if (16 * p.passes.size() + 20 * p.groups_u.size() + 20 * p.tiles.size() + 4 * (size_t)((p.S + 15) / 16 * 16) > 32 * 1024)
        return fail(WH_E_UNSUPPORTED, "UMMA engine: tile table too large");
    return WH_OK;
}

static int umma_prepare_impl(Plan &p);
int umma_prepare(Plan &p) {
    // a plan with doubled rows that does not fit shared memory is planned again without
    p.no_2v = false;
    p.no_pstream = false;
    int rc = umma_prepare_impl(p);
    if (rc == WH_E_UNSUPPORTED && p.doubled_v) {
        p.no_2v = true;
        rc = umma_prepare_impl(p);
    }
    if (rc == WH_E_UNSUPPORTED && p.pstream) {  // panel streaming did not fit: rows of 128 where possible
        p.no_pstream = true;
        rc = umma_prepare_impl(p);
    }
    return rc;
}
static int umma_prepare_impl(Plan &p) {
    p.no_convregs = plan_knob("WH_UMMA_NO_CONVREGS") != nullptr;
    p.force_fixup = plan_knob("WH_UMMA_MINMAX_FIXUP") != nullptr;
    // per-clip min-max: the separate read-modify-write pass (k_minmax_apply, HBM-bound, c5
    // 3.9 ms) by default -- the in-kernel write-once normalisation (units re-read from L2 once
    // their clip is complete) measured slower on c5 (33.5 vs 28.4 ms, profiles/r02b_*): its raw
    // tiles were mostly evicted before the re-read (ncu: 23.3 GB written, 12.1 GB read for
    // 13.1 + 2.6 GB algorithmic) and the re-reads compete with the MMA operand traffic
    p.minmax_2pass = plan_knob("WH_UMMA_MINMAX_INKERNEL") == nullptr;
    p.minmax_mode = p.minmax_2pass ? 0 : 1;
    if (const char *m = plan_knob("WH_UMMA_MINMAX")) {  // pass | inkernel | concurrent
        if (!std::strcmp(m, "pass")) p.minmax_mode = 0;
        else if (!std::strcmp(m, "inkernel")) p.minmax_mode = 1;
        else if (!std::strcmp(m, "concurrent")) p.minmax_mode = 2;
    }
    p.minmax_2pass = p.minmax_mode != 1;
    if (const char *n = plan_knob("WH_UMMA_NORM_CTAS")) p.norm_ctas = std::max(2, std::atoi(n) / 2 * 2);
    if (const char *e = plan_knob("WH_UMMA_PGROUPS")) p.pgroups_force = std::atoi(e);
    if (const char *d = diag_knob("WH_UMMA_DBG")) p.dbg = std::atoi(d);
    // hop | 64: rows of 64 samples, P = 64/hop frames (phases) per row; hop = 64..256 (multiple
    // of 64): one frame per row of hop samples; hop = 256*RS: rows of 256 samples of which
    // every RS-th is a frame (the other rows are computed and dropped: RS x the tensor work,
    // still far ahead of the SIMT engine)
    int64_t H = p.hop;
    p.rs = 1;
    // Hops >= 256 that are multiples of 64, with the columns in one pass: rows of hop samples,
    // one frame per row (tensor work in proportion to the frames).  Such a window (128 frames
    // + halo rows of hop samples) is too large to hold whole, so it streams through two
    // panel slots in 64-sample column panels, the K-steps in panel-major order, the tap bank
    // resident; the window's exponent is computed one unit ahead (epilogue warps).
    p.no_tma = plan_knob("WH_UMMA_NO_TMA") != nullptr;
    {
        const int64_t cc = p.wavelet == WH_WAVELET_CMOR ? 2 : 1;
        // measured slower than rows of 128 on c4 (hop 256 / 1024: 214 / 241 vs 205 / 205 us, 6
        // converter warps): the whole window of 128 frames is converted by the converter warps
        // of one CTA per tile while a clip's last tile (29 of 157 frames at hop 1024) leaves its
        // pair partner idle; used where rows of 128 cannot be (hops that are multiples of 64
        // but not of 128) and on request (WH_UMMA_PSTREAM=1)
        // Hops that are multiples of 128 can also run as rows of 128 samples (every (hop/128)-th
        // row a frame): the cheaper of the two by a model fitted to c4-shaped batches (cycles at
        // ~1.7 GHz; profiles/r02k_hops.txt): a unit (pair of 128-row tiles) costs its K-steps'
        // MMAs -- ~620 cycles per K-step panel-streamed, ~430 in rows of 128 -- or, panel-streamed,
        // its panels' conversion (~30 cycles per window row and panel) if that is longer; units run
        // in rounds over the CTA pairs.  Panel streaming must model 5 % cheaper to be taken.
        bool model_ps = false;
        p.ps_cg1 = false;
        if (H % 64 == 0 && H >= 256) {
            const double ksteps = (double)((2 * p.Lmax + 64) / 64 + 1);
            const double pairs = std::max(1, p.sms / 2), clips = (double)std::max<int64_t>(1, p.max_clips);
            const int64_t tiles_ps = (p.F + 127) / 128, rows128 = (p.F - 1) * (H / 128) + 1;
            const int64_t tiles_128 = (rows128 + 127) / 128;
            const double win_rows = 128.0 + (double)(2 * p.Lmax / H) + 8.0;
            const double unit_ps = std::max(620.0 * ksteps, 30.0 * win_rows * (double)(H / 64));
            const double t_ps2 = std::ceil(clips * (double)((tiles_ps + 1) / 2) / pairs) * unit_ps;
            // single-CTA MMAs (a unit = one tile) when a clip's last tile pair is half empty --
            // clips of up to 128 frames at hop 1280: 120 vs 185 us on c4's shape
            const double t_ps1 = std::ceil(clips * (double)tiles_ps / (2.0 * pairs)) * unit_ps;
            p.ps_cg1 = t_ps1 < 0.9 * t_ps2;
            if (H % 128 == 0) {
                const double rounds_128 = std::ceil(clips * (double)((tiles_128 + 1) / 2) / pairs);
                model_ps = std::min(t_ps1, t_ps2) < 0.95 * rounds_128 * 430.0 * ksteps;
            }
        }
        const bool want = plan_knob("WH_UMMA_PSTREAM") != nullptr || H % 128 != 0 || model_ps;
        p.pstream = (!p.no_pstream && want && plan_knob("WH_UMMA_NO_PSTREAM") == nullptr && H >= 256 &&
                     H <= 4096 && H % 64 == 0 && cc * (int64_t)p.S <= 128) ? 1 : 0;
        // tf32 operands (kind::tf32, K-steps of 32 taps): the fp32 samples are split in place
        // (hi = the top 19 bits, lo = x - hi) -- no window exponent, so no pre-pass over the
        // input, and a third of the conversion instructions of the fp16 split; the MMAs read
        // twice the operand bytes per tap, which the frame-proportional large hops can afford
        // Opt-in (WH_UMMA_TF32=1): measured slower than the fp16 split on c4 (hop 256 / 1024:
        // 327 / 276 vs 232 / 255 us) -- twice the MMAs per tap, and each small-N MMA costs the
        // issuing thread and the shared-memory operand reads the same whatever its K.
        p.tf32 = 0;
        if (p.pstream)
            if (const char *t = plan_knob("WH_UMMA_TF32")) p.tf32 = std::atoi(t) ? 1 : 0;
        p.ks = p.tf32 ? 32 : 64;
        // two accumulator sets when (main | corr) fits half a buffer
        p.acc2 = (p.tf32 && 2 * ((cc * (int64_t)p.S + 15) / 16 * 16) <= 128) ? 1 : 0;
        if (const char *t = plan_knob("WH_UMMA_ACC2")) p.acc2 = (p.acc2 && std::atoi(t)) ? 1 : 0;
        // the row error grows by ~2.5e-8 of the row peak per accumulation step:
        // tf32 (K = 8 per step) only while an accumulator sees at most ~280 steps (7e-6)
        if (p.tf32 && 2 * p.Lmax / 8 / (p.acc2 ? 2 : 1) > 280) {
            p.tf32 = 0;
            p.acc2 = 0;
            p.ks = 64;
        }
    }
    if (!p.pstream) {
        if (p.hop >= 256 && p.hop % 128 != 0) return fail(WH_E_UNSUPPORTED, "UMMA engine: hop needs panel streaming");
        // hop >= 256, a multiple of 128: rows of R = 128 samples, every (hop/R)-th row a frame.
        // Rows of 256 (one frame per row at hop 256) need a 147 KB window per tile that cannot
        // be double-buffered: measured c4 hop 256 / 1024 274 / 260 us with rows of 256, 227 / 226
        // with rows of 128 (2x the rows computed, windows half the size), 286 with rows of 64.
        int64_t R = 128;
        if (const char *r = plan_knob("WH_UMMA_ROW"))  // diagnostics: rows of 256 where hop % 256 == 0
            if (std::atoi(r) == 256 && H % 256 == 0) R = 256;
        if (H >= 256 && H % R == 0 && (H > 256 || R < 256)) {
            p.rs = (int32_t)(H / R);
            H = R;
        }
    }
    // rows of V = lcm(hop, 64) samples (<= 256): hop | 64 -> 64, hop | 192 -> 192, hop = 128,
    // 192, 256 -> hop; P = V / hop frames (phases) per row
    p.V = (int32_t)(H / std::gcd(H, (int64_t)64) * 64);
    {
        // Twice the phases per row when the columns still fit one pass: each A-operand read then
        // serves twice the columns (c4 hop 64, 64 scales: 285 -> 228 us, the bank streamed
        // beside two windows); with more columns the second pass re-reads A (c2: 65 -> 110 us)
        const int64_t cc = p.wavelet == WH_WAVELET_CMOR ? 2 : 1;
        const int64_t colcap = p.Lmax > UM_LMAX1 ? 64 : 128;  // columns of a pass
        p.doubled_v = p.rs == 1 && !p.pstream && 2 * p.V <= 256 && 2 * (p.V / H) * cc * (int64_t)p.S <= colcap && !p.no_2v &&
                      plan_knob("WH_UMMA_V") == nullptr && plan_knob("WH_UMMA_NO_2V") == nullptr;
        if (p.doubled_v) p.V *= 2;
    }
    if (const char *v = plan_knob("WH_UMMA_V")) {  // experiment: more phases per row
        const int vv = std::atoi(v);
        if (vv >= p.V && vv % 64 == 0 && vv % H == 0 && p.rs == 1 && !p.pstream) p.V = vv;
    }
    p.P = (int32_t)(p.V / H);
    p.Cc = p.wavelet == WH_WAVELET_CMOR ? 2 : 1;
    p.panels = p.V / p.ks;
    p.rows_total = (int32_t)(p.rs > 1 ? (p.F - 1) * p.rs + 1 : (p.F + p.P - 1) / p.P);
    p.row_tiles = (p.rows_total + 127) / 128;

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
    int tau_log2 = 7;  // correction-term threshold tau = 2^-7 (WH_UMMA_TAU=0: never skip)
    if (const char *t = plan_knob("WH_UMMA_TAU")) tau_log2 = std::atoi(t);
    // TMEM: 512 columns = 2 accumulator buffers x (128 main + 128 correction) columns, so a
    // pass covers at most 128 columns and the epilogue of pass n overlaps the MMAs of n+1.
    const bool longf = p.Lmax > UM_LMAX1;  // two accumulator sets per buffer: passes of 64 columns
    if (longf) {
        if (p.pstream) return fail(WH_E_UNSUPPORTED, "UMMA engine: very long filters are not panel-streamed");
        p.acc2 = 1;
        p.minmax_mode = 0;
        p.minmax_2pass = true;
    }
    const int max_cols = longf ? 64 : 128;
    p.n_acc = 2;
    p.acc_stride = 256;
    int win_bufs = 0, bstages = 0;
    // scales per pass: whole scales, cols = ns*CP rounded up to 16 (CP > 256 unsupported)
    if (CP > max_cols) return fail(WH_E_UNSUPPORTED, "UMMA engine: too many phases per scale");
    const int spp = std::max(1, max_cols / CP);
    // Passes and K-step tiles for a K origin G0 (K index g = u + G0, tap offset u in
    // [-L, L]); returns the modelled MMA cycles per unit (tools/probe_kstep.cu: a K-step
    // costs max(its shared-memory operand reads, its tensor work) + issue overhead).
    auto make_tiles = [&](int64_t G0, std::vector<UmmaPass> &passes, std::vector<UmmaTile> &tiles) -> double {
        passes.clear();
        tiles.clear();
        const int64_t KS = p.ks;
        const int64_t ksteps = (G0 + p.Lmax + (int64_t)(p.P - 1) * H) / KS + 1;
        double cost = 0.0;
        // heavy (long-tap) passes first so the accumulator pipeline starts on the long ones
        // (alternating heavy / light passes measured no better on c5)
        std::vector<int> order;
        for (int s0 = ((p.S - 1) / spp) * spp; s0 >= 0; s0 -= spp) order.push_back(s0);
        for (int s0 : order) {
            UmmaPass ps{};
            ps.s0 = s0;
            ps.ns = std::min(spp, p.S - s0);
            ps.cols = (ps.ns * CP + 15) / 16 * 16;
            ps.tile_begin = (int32_t)tiles.size();
            for (int64_t k = 0; k < ksteps; ++k) {
                // first active column: column j = (scale, comp, phase) is active on g in
                // [G0 - L + r*H, G0 + L + r*H]
                int c0 = ps.cols;
                for (int j = 0; j < ps.ns * CP; ++j) {
                    const int s = ps.s0 + j / CP, r = j % p.P;
                    const int64_t lo = G0 - p.half[s] + (int64_t)r * H;
                    const int64_t hi = G0 + p.half[s] + (int64_t)r * H;
                    if (hi >= k * KS && lo <= k * KS + KS - 1) {
                        c0 = j;
                        break;
                    }
                }
                if (c0 >= ps.ns * CP) continue;  // no active column on this K-step
                // correction columns: the split-fp16 cross terms x_h*t_l + x_l*t_h matter only
                // where a column's taps are not negligible.  Each dropped product is at most
                // 2^-10 |x t|; with every |tap| of the K-step below tau * (the scale's peak
                // tap), even sign-coherent x over the whole dropped Gaussian tail (mass
                // < 0.24 tau of the peak region's) bounds the error by 2^-10 * 0.24 * tau of
                // the row's peak |W| (tau = 2^-7: < 1.8e-6, vs the 1e-5 tolerance; measured
                // errors unchanged from tau = 2^-8: c5 5.47e-6, 914 -> 892 us per 148 clips; 2^-6
                // would give 876 us with a 3.7e-6 bound).  |tap| is bounded by the envelope
                // exp(-u^2/(B a^2)).
                int c1 = ps.cols;
                for (int j = c0; j < ps.ns * CP; ++j) {
                    const int s = ps.s0 + j / CP, r = j % p.P;
                    const int64_t u0 = k * KS - G0 - (int64_t)r * H, u1 = u0 + KS - 1;
                    const int64_t umin = (u0 <= 0 && u1 >= 0) ? 0 : std::min(std::llabs(u0), std::llabs(u1));
                    if ((double)umin > (double)p.half[s]) continue;  // inactive column
                    const double x = (double)umin / p.scales[s];
                    if (tau_log2 <= 0 || -(x * x) / p.B > -tau_log2 * M_LN2) {
                        c1 = j;
                        break;
                    }
                }
                UmmaTile tl{};
                tl.k = (int32_t)k;
                tl.c0 = c0 / 16 * 16;
                tl.ncols = ps.cols - tl.c0;
                tl.ncorr = ps.cols - c1 / 16 * 16;
                tiles.push_back(tl);
                const double rows = tl.ncols + 2.0 * tl.ncorr;
                cost += std::max(128.0 * (tl.ncorr ? 2 : 1) + 0.5 * rows + 50.0, 2.0 * rows + 30.0);
            }
            ps.tile_end = (int32_t)tiles.size();
            if (ps.tile_end > ps.tile_begin) passes.push_back(ps);
        }
        return cost;
    };
    // K origin: G0 >= Lmax, a multiple of 32 samples (the window start tile*128*V - G0 on a
    // 128-byte line: whole sectors for the converters' loads).  Candidates up to one row
    // later are modelled; whole-row alignment (G0 % V == 0) wins unless it models > 3 %
    // slower (measured: hop 256 runs 6 % faster row-aligned at equal tiles; c2 runs 3 %
    // faster with 21 instead of 22 K-steps), then the smaller G0.
    {
        std::vector<UmmaPass> tp;
        std::vector<UmmaTile> tt;
        // (panel streaming with 64-sample fp16 panels: a multiple of 64, so that a panel never
        // straddles two rows of V samples -- its TMA box is one rectangle of the batch tensor)
        const int64_t gal = (p.pstream && !p.tf32) ? 64 : 32;
        const int64_t g0min = (p.Lmax + gal - 1) / gal * gal;
        int64_t best = -1;
        double best_cost = 0.0;
        for (int64_t g0 = g0min; g0 <= g0min + p.V; g0 += gal) {
            const double c = make_tiles(g0, tp, tt) * (g0 % p.V == 0 ? 1.0 : 1.03);
            if (best < 0 || c < best_cost - 0.5) {
                best = g0;
                best_cost = c;
            }
        }
        if (const char *g = plan_knob("WH_UMMA_G0_ALIGN")) {  // diagnostics: force an alignment
            const int64_t al = std::max(4, std::atoi(g)) / 4 * 4;
            best = (p.Lmax + al - 1) / al * al;
        }
        p.G0 = (int32_t)best;
    }
    p.unit_cost = make_tiles(p.G0, p.passes, p.tiles);
    if (p.pstream) {
        if (p.passes.size() != 1) return fail(WH_E_UNSUPPORTED, "UMMA engine: panel streaming needs one pass");
        // K-steps in panel-major order (panel = (64k mod V) / 64, row shift q = 64k / V): all
        // the K-steps of one window panel run while it is in its slot
        const int64_t V = p.V, KS = p.ks;
        std::stable_sort(p.tiles.begin(), p.tiles.end(), [&](const UmmaTile &a, const UmmaTile &b) {
            const int64_t pa = (KS * (int64_t)a.k % V) / KS, pb = (KS * (int64_t)b.k % V) / KS;
            return pa != pb ? pa < pb : a.k < b.k;
        });
    }
    p.Qlo = (int32_t)((p.G0 + p.V - 1) / p.V);
    p.ksteps = (int32_t)((p.G0 + p.Lmax + (int64_t)(p.P - 1) * H) / p.ks + 1);
    const int64_t qmax = (int64_t)(p.ksteps - 1) * p.ks / p.V;
    p.win_rows = (int32_t)(((128 + qmax) + 7) / 8 * 8);
    if (p.pstream && !p.tf32 && (int64_t)p.win_rows * 8 > (int64_t)UM_PCH * UM_CONV_THREADS)
        return fail(WH_E_UNSUPPORTED, "UMMA engine: panel too tall for the converters' registers");
    const int64_t win = 2LL * (p.pstream ? 1 : p.panels) * p.win_rows * 128;  // pstream: one panel slot
    int64_t byte_off = 0;
    // CTA pairs (tcgen05 cta_group::2, M = 256): each CTA stages half of every tap tile
    p.cg = (p.sms % 2 == 0 && plan_knob("WH_UMMA_CG1") == nullptr && !(p.pstream && p.ps_cg1)) ? 2 : 1;
    // Group consecutive tiles of a pass into one bulk copy of up to group_target bytes per
    // CTA: a copy costs ~250 issue cycles whatever its size (tools/probe_bulk.cu), so small
    // tiles must travel together.  Bank layout per group: [CTA-0 blocks][CTA-1 blocks].
    // bytes per CTA of a tile: MMA1's B has nc + ncorr rows, MMA2's ncorr (128 B per row);
    // CTA pairs hold half of each
    auto tile_bytes = [&](const UmmaTile &t) -> int64_t {
        return (int64_t)(p.cg == 2 ? 64 : 128) * (t.ncols + 2 * t.ncorr);
    };
    int64_t bank_cta = 0;
    for (auto &t : p.tiles) bank_cta += tile_bytes(t);
    // budget known early: the opt-in smem minus static smem and slack (tables added below)
    // the opt-in min-max modes exist for CTA pairs with 1 or 2 phases per row (and not with panel
    // streaming); elsewhere the separate pass
    if (p.minmax_mode != 0 && (p.pstream || !umma_kernel(p.Cc, p.P, p.cg, 2))) {
        p.minmax_mode = 0;
        p.minmax_2pass = true;
    }
    UmmaKernel kern0 = umma_kernel(p.Cc, p.P, p.cg, umma_variant(p));
    if (!kern0) return fail(WH_E_UNSUPPORTED, "UMMA engine: unsupported phase count");
    int optin0 = 0;
    cudaDeviceGetAttribute(&optin0, cudaDevAttrMaxSharedMemoryPerBlockOptin, p.device);
    cudaFuncAttributes fa0{};
    WH_CUDA_TRY(cudaFuncGetAttributes(&fa0, kern0));
    const int64_t tables_est = 16 * (int64_t)p.passes.size() + 24 * (int64_t)p.tiles.size() + 4 * (int64_t)p.S;
    const int64_t budget0 = (int64_t)optin0 - (int64_t)fa0.sharedSizeBytes - 1024 - 64 - tables_est;
    // Tap residency.  (1) the whole bank fits beside two windows: load it once, never
    // stream.  (2) it fits beside one window only: "hybrid" -- keep the prefix of the tiles
    // (in consumption order) resident, stream the tail K-steps of every unit through a small
    // ring, and spend the freed smem on a second window so window conversion overlaps the
    // MMAs (opt-in, WH_UMMA_HYBRID: on c2 the per-group waits of the streamed tail cost more
    // than the hidden conversion; default is one window, all resident).  (3) otherwise
    // stream everything.
    const int64_t n_tiles = (int64_t)p.tiles.size();
    const bool allow_res = plan_knob("WH_UMMA_NO_RESIDENT") == nullptr;
    int64_t t_split = 0;  // tiles [0, t_split) resident
    int hybrid = 0;
    int64_t stream_target = 0;
    if (p.pstream) {
        // UM_WSLOTS panel slots; the bank resident beside them when it fits, else streamed
        if (allow_res && bank_cta + UM_WSLOTS * win <= budget0) t_split = n_tiles;
    } else if (allow_res && bank_cta + 2 * win <= budget0) {
        t_split = n_tiles;
    } else if (allow_res && bank_cta + win <= budget0) {
        t_split = n_tiles;
        if (plan_knob("WH_UMMA_HYBRID") != nullptr) {
            stream_target = 8 * 1024;
            int64_t hyb_ring = 32 * 1024;
            if (const char *r = plan_knob("WH_UMMA_HYB_RING_KB")) hyb_ring = std::max(8, std::atoi(r)) * 1024;
            const int64_t res_limit = budget0 - 2 * win - hyb_ring;
            int64_t acc = 0, t = 0;
            while (t < n_tiles && acc + tile_bytes(p.tiles[t]) <= res_limit) acc += tile_bytes(p.tiles[t++]);
            int64_t max_tail_tile = 0;
            for (int64_t i = t; i < n_tiles; ++i) max_tail_tile = std::max(max_tail_tile, tile_bytes(p.tiles[i]));
            if (t > 0 && t < n_tiles && 2 * max_tail_tile <= hyb_ring) {
                t_split = t;
                hybrid = 1;
            }
        }
    }
    p.resident = t_split > 0 ? 1 : 0;
    // Streamed banks: tap groups of up to 48 KB.  Short unit sequences (< 64 tiles) keep two
    // windows (no fp32 staging, register converter), with groups as large as a ring of three
    // fits beside them (c4 hop 16: 24 KB groups + staging 558 us, 44 KB + two windows 456 us);
    // long ones keep one window and 48 KB groups (c5, c3, c4 hop 1: measured best).
    const int64_t two_win_groups = std::min<int64_t>(48 * 1024, (budget0 - 2 * win) / 3 / 1024 * 1024);
    int64_t group_target = p.resident ? 48 * 1024 : (n_tiles >= 64 ? 48 * 1024 : std::max<int64_t>(16 * 1024, two_win_groups));
    if (p.pstream && !p.resident)  // a ring of three groups beside the panel slots
        group_target = std::max<int64_t>(8 * 1024, std::min<int64_t>(48 * 1024, (budget0 - UM_WSLOTS * win) / 3 / 1024 * 1024));
    int64_t group_target_env = 0;
    if (const char *g = plan_knob("WH_UMMA_GROUP_KB")) group_target_env = std::max(1, std::atoi(g)) * 1024;
    p.groups_u.clear();
    int64_t max_group = 0, res_bytes = 0;
    int n_stream = 0;
    for (auto &ps : p.passes) {
        ps.group_begin = (int32_t)p.groups_u.size();
        int t = ps.tile_begin;
        while (t < ps.tile_end) {
            const bool res = t < t_split;  // groups never straddle the split
            const int64_t target =
                group_target_env ? group_target_env : (res ? group_target : (hybrid ? stream_target : group_target));
            UmmaGroup gr{};
            gr.tile_begin = t;
            int64_t bytes = 0;
            while (t < ps.tile_end && (t < t_split) == res &&
                   (bytes == 0 || bytes + tile_bytes(p.tiles[t]) <= target)) {
                p.tiles[t].in_off = (int32_t)bytes;
                bytes += tile_bytes(p.tiles[t]);
                ++t;
            }
            gr.tile_end = t;
            gr.cta_bytes = (int32_t)bytes;
            gr.bank_off = byte_off;
            gr.pad_ = res ? (int32_t)res_bytes : -1;  // smem offset of a resident group
            if (res) {
                res_bytes += bytes;
            } else {
                ++n_stream;
                max_group = std::max(max_group, bytes);
            }
            for (int i = gr.tile_begin; i < gr.tile_end; ++i) {
                p.tiles[i].byte_off = byte_off + p.tiles[i].in_off;
                p.tiles[i].blk1_delta = bytes;
            }
            byte_off += bytes * p.cg;
            p.groups_u.push_back(gr);
        }
        ps.group_end = (int32_t)p.groups_u.size();
    }
    p.bank_bytes = byte_off;
    p.res_bytes = res_bytes;
    p.n_stream = n_stream;
    const int64_t stage_bytes = std::max<int64_t>(max_group, 1024);
    const int64_t table_bytes = (16 * (int64_t)p.passes.size() + 20 * (int64_t)p.groups_u.size() +
                                 (p.pstream ? 20 : 16) * (int64_t)p.tiles.size() + 4 * (int64_t)((p.S + 15) / 16 * 16) +
                                 15) / 16 * 16 + 16;  // + one entry of slack: the issue loop reads a tile ahead
    // dynamic smem budget: the opt-in maximum minus the kernel's static smem, the 1 KB
    // alignment slack and the tables
    UmmaKernel kern = umma_kernel(p.Cc, p.P, p.cg, umma_variant(p));
    if (!kern) return fail(WH_E_UNSUPPORTED, "UMMA engine: unsupported phase count");
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p.device);
    cudaFuncAttributes fa{};
    WH_CUDA_TRY(cudaFuncGetAttributes(&fa, kern));
    const int64_t budget = (int64_t)optin - (int64_t)fa.sharedSizeBytes - 1024 - 64 - table_bytes;
    if (ncheck_tiles(p) != WH_OK) return WH_E_UNSUPPORTED;
    // smem = window buffers (hi|lo fp16) [+ fp32 staging, same bytes as one window] + the
    // tap stage region (resident groups, then the ring).  Long units (many K-steps per
    // window) favour a deeper ring with one window; short units favour two windows.
    int use_stg = 0;
    int64_t ring = 0;
    if (p.pstream) {
        win_bufs = UM_WSLOTS;
        const int64_t rest = (budget - UM_WSLOTS * win) / 1024 * 1024;
        ring = p.resident ? (res_bytes + 1023) / 1024 * 1024 : rest;
        if (ring > rest || (!p.resident && ring < 3 * stage_bytes))
            return fail(WH_E_UNSUPPORTED, "UMMA engine: panel slots and tap ring do not fit");
    } else if (p.resident && !hybrid) {
        // the stage region is the whole resident bank; spend what is left on windows / staging
        ring = (res_bytes + 1023) / 1024 * 1024;
        // the register-prefetch converter (no fp32 staging) is the faster one when a
        // thread's share of the window fits its registers
        const bool regs_ok = (int64_t)p.win_rows * p.panels * 8 <= (int64_t)UM_CONV_RC * UM_CONV_THREADS;
        const int opts_stg[4][2] = {{2, 1}, {2, 0}, {1, 1}, {1, 0}};
        const int opts_regs[4][2] = {{2, 0}, {1, 0}, {2, 1}, {1, 1}};
        const int (*opts_r)[2] = regs_ok ? opts_regs : opts_stg;
        const int r0 = plan_knob("WH_UMMA_WIN1") ? (regs_ok ? 1 : 2) : 0;  // diagnostics: one window
        for (int i = r0; i < 4; ++i) {
            const int *o = p.pstream ? opts_regs[0] : opts_r[i];  // pstream: two panel slots, no staging
            if ((int64_t)(o[0] + o[1]) * win + ring <= budget) {
                win_bufs = o[0];
                use_stg = o[1];
                break;
            }
        }
        if (win_bufs == 0) return fail(WH_E_UNSUPPORTED, "UMMA engine: resident bank does not fit");
    } else if (hybrid) {
        const int64_t rest = (budget - 2 * win - res_bytes) / 1024 * 1024;
        if (rest < 2 * stage_bytes) return fail(WH_E_UNSUPPORTED, "UMMA engine: hybrid ring does not fit");
        win_bufs = 2;
        use_stg = 0;
        ring = res_bytes + rest;
    } else {
        const int prefer_single = n_tiles >= 64 && plan_knob("WH_UMMA_PREFER_DOUBLE") == nullptr;
        const int opts_a[4][2] = {{2, 0}, {2, 1}, {1, 1}, {1, 0}};
        const int opts_b[4][2] = {{1, 1}, {2, 1}, {1, 0}, {2, 0}};
        const int (*opts)[2] = prefer_single ? opts_b : opts_a;
        const char *force = plan_knob("WH_UMMA_SMEM_OPT");  // diagnostics: force an option
        const int ostart = force ? std::atoi(force) : 0;
        for (int i = ostart; i < 4; ++i) {
            const int64_t fixed = (int64_t)(opts[i][0] + opts[i][1]) * win;
            const int64_t r = (budget - fixed) / 1024 * 1024;
            if (r >= 3 * stage_bytes && r >= 64 * 1024) {
                win_bufs = opts[i][0];
                use_stg = opts[i][1];
                ring = r;
                break;
            }
        }
        if (ring == 0) {  // last resort: one window, ring of at least two tiles
            const int64_t r = (budget - win) / 1024 * 1024;
            if (r >= 2 * stage_bytes) { win_bufs = 1; use_stg = 0; ring = r; }
        }
    }
    if (ring == 0) return fail(WH_E_UNSUPPORTED, "UMMA engine: shared memory too small for the tap ring");
    bstages = (int)(ring / stage_bytes);
    p.win_bufs = win_bufs;
    p.bstages = bstages;
    p.use_stg = use_stg;
    p.ring_bytes = ring;
    p.smem_bytes = (size_t)((win_bufs + use_stg) * win + ring) + 1024 + table_bytes;

    {
        // the kernel's shared-memory tables, packed here in their smem layout so that one
        // bulk copy loads them at launch: int4 pass[], int4 group[], uint4 tile[] (pre-decoded
        // MMA operands of each K-step, in 16-byte descriptor units: x = A offset in the window
        // | c0 << 16, y = B offset in the group | MMA2's B delta << 16, z / w = instruction
        // descriptors of MMA1 (N = nc + ncorr) / MMA2 (N = ncorr; 0 = not issued)), float spow[]
        // (per-scale 2^-f, padded to 16: the epilogue reads whole 16-column units), int goff[] (resident groups' smem offsets)
        std::vector<uint8_t> blob((size_t)table_bytes, 0);
        uint8_t *w = blob.data();
        auto put32 = [&](uint32_t v) { std::memcpy(w, &v, 4); w += 4; };
        for (auto &ps : p.passes) {
            put32((uint32_t)ps.group_begin); put32((uint32_t)ps.group_end);
            put32((uint32_t)ps.s0 | ((uint32_t)ps.ns << 16)); put32((uint32_t)ps.cols);
        }
        for (auto &g : p.groups_u) {
            put32((uint32_t)g.tile_begin); put32((uint32_t)g.tile_end);
            put32((uint32_t)(g.bank_off >> 7)); put32((uint32_t)g.cta_bytes);
        }
        // D f32; A / B f16 (0) or tf32 (2 at bits [7,10) and [10,13)); K-major; N >> 3; M >> 4
        const uint32_t fmt = p.tf32 ? ((2u << 7) | (2u << 10)) : 0u;
        auto idesc = [&](uint32_t n) { return (1u << 4) | fmt | ((n >> 3) << 17) | (((128u * (uint32_t)p.cg) >> 4) << 24); };
        for (auto &tl : p.tiles) {
            // window row shift q and panel of this K-step's A operand (k*64 = q*V + panel*64)
            const uint32_t kg = (uint32_t)tl.k * (uint32_t)p.ks, q = kg / (uint32_t)p.V, panel = (kg % (uint32_t)p.V) / (uint32_t)p.ks;
            const uint32_t aoff = (p.pstream ? 0u : panel * (uint32_t)p.win_rows * 128u) + q * 128u;
            const uint32_t n1 = (uint32_t)(tl.ncols + tl.ncorr), n2 = (uint32_t)tl.ncorr;
            const uint32_t b2d = (p.cg == 2 ? n1 / 2 : n1) * 128u;
            put32((aoff >> 4) | ((uint32_t)tl.c0 << 16));
            put32(((uint32_t)tl.in_off >> 4) | ((b2d >> 4) << 16));
            put32(idesc(n1));
            put32(n2 ? idesc(n2) : 0u);
        }
        for (int i = 0; i < (p.S + 15) / 16 * 16; ++i) {
            uint32_t v = 0;
            if (i < p.S) std::memcpy(&v, &spow[i], 4);
            put32(v);
        }
        for (auto &g : p.groups_u) put32((uint32_t)g.pad_);
        if (p.pstream)  // tile -> window panel
            for (auto &tl : p.tiles) put32((uint32_t)(((int64_t)tl.k * p.ks % p.V) / p.ks));
        p.tables_bytes = table_bytes;
        WH_CUDA_TRY(cudaMalloc(&p.d_tables, (size_t)table_bytes));
        WH_CUDA_TRY(cudaMemcpy(p.d_tables, blob.data(), (size_t)table_bytes, cudaMemcpyHostToDevice));
    }
    WH_CUDA_TRY(cudaMalloc(&p.d_passes, sizeof(UmmaPass) * p.passes.size()));
    WH_CUDA_TRY(cudaMalloc(&p.d_tiles, sizeof(UmmaTile) * p.tiles.size()));
    WH_CUDA_TRY(cudaMalloc(&p.d_groups_u, sizeof(UmmaGroup) * p.groups_u.size()));
    WH_CUDA_TRY(cudaMemcpy(p.d_groups_u, p.groups_u.data(), sizeof(UmmaGroup) * p.groups_u.size(),
                           cudaMemcpyHostToDevice));
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
    ba.P = p.P; ba.Cc = p.Cc; ba.G0 = p.G0; ba.hop = p.hop; ba.bank = p.d_bank; ba.cg = p.cg; ba.tf32 = p.tf32;
    k_build_bank<<<(unsigned)p.tiles.size(), 256>>>(ba);

    WH_CUDA_TRY(cudaGetLastError());
    WH_CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(d_fexp);
    // the attribute belongs to the kernel instantiation, which other plans share: raise it to the
    // device limit once instead of to this plan's size (a later, smaller plan would otherwise
    // lower it under an earlier plan's launches)
    WH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - (int)fa.sharedSizeBytes));
    // persistent grid: as many CTAs (pairs) as can be co-resident -- with clusters of 2 not
    // every SM necessarily has a partner in its GPC, and a CTA pair that does not fit would
    // run its whole unit sequence as a second wave
    p.grid_ctas = p.sms;
    if (p.cg == 2) {
        WH_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)p.sms);
        cfg.blockDim = dim3(UM_THREADS);
        cfg.dynamicSmemBytes = p.smem_bytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) == cudaSuccess && clusters > 0)
            p.grid_ctas = std::min(p.sms, 2 * clusters);
        (void)cudaGetLastError();
    }
    if (diag_knob("WH_UMMA_VERBOSE")) {  // diagnostics: the plan's shape
        int64_t ncorr = 0, ncols = 0;
        for (auto &t : p.tiles) ncols += t.ncols, ncorr += t.ncorr;
        std::fprintf(stderr,
                     "[wh umma] V=%d P=%d Cc=%d cg=%d passes=%zu tiles=%zu (sum nc %lld, ncorr %lld) groups=%zu "
                     "resident=%d res=%lld B stream_groups=%d bank/CTA=%lld B win=%d x %lld B stg=%d ring=%lld B "
                     "smem=%zu B grid=%d CTAs\n",
                     p.V, p.P, p.Cc, p.cg, p.passes.size(), p.tiles.size(), (long long)ncols, (long long)ncorr,
                     p.groups_u.size(), p.resident, (long long)p.res_bytes, p.n_stream, (long long)bank_cta,
                     p.win_bufs, (long long)win, p.use_stg, (long long)p.ring_bytes, p.smem_bytes, p.grid_ctas);
    }
    return WH_OK;
}

// Pass groups per tile pair for a launch of `clips` clips: split each tile pair's passes into
// G groups (separate units) when there are too few units to fill the CTA pairs evenly (c3: 80
// tile pairs on 74 CTA pairs): minimise rounds x unit time, with a unit costing at least one
// window conversion (~6 k cycles)
int umma_pass_groups(const Plan &p, int64_t clips) {
    const int64_t tile_units = clips * ((p.row_tiles + p.cg - 1) / p.cg);
    const bool concurrent = p.norm == WH_NORM_MINMAX && p.minmax_mode == 2;
    const int64_t pairs = std::max<int64_t>(1, (p.grid_ctas - (concurrent ? p.norm_ctas : 0)) / p.cg);
    const int n_passes = (int)p.passes.size();
    // Among splits within 3 % of the best modelled time, the one whose last round of units is
    // fullest wins (c3: 11 groups of 3 passes, last round 66 / 74 full: 150 us; 8 groups of 4,
    // 48 / 74: 165 us; 16 groups of 2, 22 / 74: 163 us -- all model the same 36 pass-rounds).
    int G = 1;
    double best = -1.0, best_fill = -1.0;
    std::vector<std::pair<int, double>> cand;  // (G, modelled time)
    for (int g = 1; g <= n_passes; ++g) {
        const int ppu = (n_passes + g - 1) / g;
        const int gg = (n_passes + ppu - 1) / ppu;  // groups actually formed
        if (gg != g) continue;
        const double rounds = std::ceil((double)(tile_units * g) / (double)pairs);
        const double t = rounds * std::max(p.unit_cost * (double)ppu / n_passes, 6000.0);
        cand.emplace_back(g, t);
        if (best < 0 || t < best) best = t;
    }
    // (only when there are few tile pairs; otherwise the first split within 3 % of the best)
    for (auto &c : cand) {
        if (c.second > best * 1.03) continue;
        const int64_t rem = (tile_units * c.first) % pairs;
        const double fill = rem == 0 ? 1.0 : (double)rem / (double)pairs;
        if (best_fill < 0.0 || (tile_units < 4 * pairs && fill > best_fill + 1e-9)) {
            G = c.first;
            best_fill = fill;
        }
    }
    if (p.pgroups_force > 0) G = std::max(1, std::min(n_passes, p.pgroups_force));
    const int ppu = (n_passes + G - 1) / G;
    return (n_passes + ppu - 1) / ppu;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        (void)cudaGetLastError();
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

int umma_launch(Plan &p, const float *x, int64_t clips, int64_t ld_x, void *out, cudaStream_t s, uint32_t *mm,
                uint32_t *arrive, uint32_t *abandon, uint32_t *nfbad, uint32_t *nfctl) {
    UmmaArgs a{};
    a.x = x; a.ld_x = ld_x; a.N = p.N; a.F = p.F; a.hop = p.hop;
    a.row_tiles = p.row_tiles; a.V = p.V; a.P = p.P; a.Cc = p.Cc; a.panels = p.panels; a.rs = p.rs;
    a.G0 = p.G0; a.win_rows = p.win_rows; a.S = p.S;
    a.n_passes = (int32_t)p.passes.size(); a.n_tiles = (int32_t)p.tiles.size();
    a.wavelet = p.wavelet; a.output = p.output;
    a.win_bufs = p.win_bufs; a.n_acc = p.n_acc; a.acc_stride = p.acc_stride;
    a.use_stg = p.use_stg;
    a.resident = p.resident;
    a.res_bytes = (uint32_t)p.res_bytes;
    a.n_stream = p.n_stream;
    a.cpr = p.panels * 8;
    a.pf = p.V >= 256 ? 1 : 0;
    a.cpr_magic = ((1 << 20) + a.cpr - 1) / a.cpr;
    a.conv_regs = (!p.use_stg && !p.no_convregs && !p.pstream) ? 1 : 0;
    a.pstream = p.pstream;
    a.tf32 = p.tf32;
    a.acc2 = p.acc2;
    a.full_end = (p.N / p.V) * p.V;
    a.tma = 0;
    if (p.pstream && !p.no_tma && (p.tf32 || p.G0 % 64 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
        ld_x % 4 == 0 && p.N >= p.V &&
        p.win_rows <= 256 && clips <= 0x7fffffff && encode_tiled()) {
        // the batch as (V samples, N / V whole rows, clips): a window panel is one box of
        // 32 samples x win_rows rows; rows before / after the clip's whole rows are zero-filled
        const cuuint64_t dims[3] = {(cuuint64_t)p.V, (cuuint64_t)(p.N / p.V), (cuuint64_t)clips};
        const cuuint64_t strides[2] = {(cuuint64_t)p.V * 4, (cuuint64_t)ld_x * 4};
        // tf32: 32-sample panels straight into the 128 B-swizzled operand layout; fp16: 64-sample
        // panels as plain rows of 256 B that the converters split
        const cuuint32_t box[3] = {p.tf32 ? 32u : 64u, (cuuint32_t)p.win_rows, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult r = encode_tiled()(&a.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(x), dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          p.tf32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        a.tma = r == CUDA_SUCCESS ? 1 : 0;
    }
    a.vec_ok = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && (ld_x % 4 == 0);
    a.tables = p.d_tables; a.tables_bytes = (uint32_t)p.tables_bytes;
    a.passes = p.d_passes; a.tiles = p.d_tiles; a.groups = p.d_groups_u; a.n_groups = (int32_t)p.groups_u.size(); a.bank = p.d_bank; a.scale_pow = p.d_scale_pow;
    a.out = out;
    a.minmax = p.norm != WH_NORM_NONE ? mm : nullptr;
    // write-once min-max: the kernel normalises each clip itself (arrival counters live right
    // after this launch's keys: the caller's slice of d_minmax is [clips][2], d_arrive the
    // matching [clips] slice)
    a.arrive = p.norm == WH_NORM_MINMAX ? arrive : nullptr;
    a.abandon = a.arrive ? abandon : nullptr;
    a.ab_words = p.ab_words;
    a.force_fixup = p.force_fixup ? 1 : 0;
    a.arrive_only = (a.arrive && p.norm == WH_NORM_MINMAX && p.minmax_mode == 2) ? 1 : 0;
    a.nfbad = nfbad; a.nfctl = nfctl;
    a.scales = p.d_scales; a.half = p.d_half; a.Cw = p.C; a.Bw = p.B;
    a.clips = clips;
    a.ring_bytes = (uint32_t)p.ring_bytes;
    a.win_half_bytes = (uint32_t)(p.pstream ? 1 : p.panels) * (uint32_t)p.win_rows * 128u;
    a.out_vec_ok = ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && (p.F % 4 == 0);
    a.out_vec8_ok = ((reinterpret_cast<uintptr_t>(out) & 31) == 0) && (p.F % 8 == 0);
    a.prof = p.d_prof;
    a.dbg = p.dbg;
    a.trace = p.d_trace;
    const int64_t tile_units = clips * ((p.row_tiles + p.cg - 1) / p.cg);
    const int n_passes = (int)p.passes.size();
    const int G = umma_pass_groups(p, clips);
    a.ppu = (n_passes + G - 1) / G;
    a.pgroups = (n_passes + a.ppu - 1) / a.ppu;
    const int64_t units = tile_units * a.pgroups;
    a.arrive_target = (uint32_t)(p.cg * ((p.row_tiles + p.cg - 1) / p.cg) * a.pgroups);
    if (units >= ((int64_t)1 << 31)) return fail(WH_E_INVALID_ARG, "UMMA engine: too many clips for one launch");
    // min-max mode 2: the concurrent normaliser keeps norm_ctas SMs (pairs) for itself
    const int64_t ctas = p.grid_ctas - (a.arrive_only ? p.norm_ctas : 0);
    int64_t grid = std::min<int64_t>(units * p.cg, ctas);
    if (p.cg == 2) grid &= ~(int64_t)1;
    (void)cudaGetLastError();  // drop stale non-sticky errors of earlier runtime calls
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(UM_THREADS);
    cfg.dynamicSmemBytes = p.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.cg;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    WH_CUDA_TRY(cudaLaunchKernelEx(&cfg, umma_kernel(p.Cc, p.P, p.cg, umma_variant(p)), a));
    WH_CUDA_TRY(cudaGetLastError());
    if (a.arrive) {
        FixupArgs f{};
        f.out = static_cast<float *>(out);
        f.minmax = mm;
        f.abandon = abandon;
        f.passes = reinterpret_cast<const int4 *>(p.d_tables);  // the packed pass table leads the blob
        f.clips = clips; f.F = p.F; f.S = p.S; f.P = p.P; f.rs = p.rs; f.cg = p.cg;
        f.tpu = (int32_t)((p.row_tiles + p.cg - 1) / p.cg); f.pgroups = a.pgroups; f.ppu = a.ppu;
        f.n_passes = n_passes; f.ab_words = p.ab_words;
        k_minmax_fixup<<<(unsigned)std::min<int64_t>(clips, 4 * p.sms), 256, 0, s>>>(f);
        WH_CUDA_TRY(cudaGetLastError());
    }
    return WH_OK;
}

}  // namespace wh
