// wh_simt.cu -- SIMT fp32 engine: folded direct strided correlation for any hop.
//
// Restates the reference's hot loop, strided_correlate_symmetric (_kernels.py:93-112):
//   re[k] = x[c]*re0 + sum_{j=1..L} (x[c+j] + x[c-j]) * re_j,   c = k*hop (+ centring)
//   im[k] =            sum_{j=1..L} (x[c+j] - x[c-j]) * im_j
// with the zero padding of wavelet.py:243-246 made implicit (out-of-range samples read 0).
//
// Tiling: one CTA = (clip, group of <= 8 consecutive scales, tile of tf frames).  The
// clip segment the tile touches is staged once in shared memory.  Each warp owns 8 frames
// (4 for complex) x 8 scales; its 32 lanes split the tap index j (j = lane + 32 t), so the
// segment reads x[c +- j] are consecutive across lanes (conflict-free for any hop) and a
// lane reads the 8 scales' taps at its j with two 16-byte loads (table [j][8]).  Each block
// of 4 frames x 8 scales (x re / im) is combined with a 31-shuffle transpose-reduction so
// lane l ends with output l.
#include <algorithm>

#include "wh_internal.h"

namespace wh {

static constexpr int SIMT_THREADS = 128;
static constexpr int SIMT_G = 8;            // scales per group
static constexpr int SIMT_SEG_MAX = 48 * 1024;  // floats of staged segment (192 KB)

__global__ void k_group_taps(const float *fold, const int64_t *fold_off, const int64_t *half,
                             int64_t fold_total, const SimtGroup *groups, int32_t n_groups,
                             float *gt) {
    int32_t g = blockIdx.y;
    if (g >= n_groups) return;
    SimtGroup G = groups[g];
    // [j][SIMT_G] (re table, then im): the 8 scales' taps at one j are 32 contiguous bytes,
    // two 16-byte loads per lane; scales >= ns are zero
    int64_t width = G.L + 1;
    int64_t n = (int64_t)SIMT_G * width;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int s = (int)(i % SIMT_G);
        int64_t j = i / SIMT_G;
        int sg = G.s0 + s;
        bool in = s < G.ns && j <= half[sg];
        gt[G.tap_off + i] = in ? fold[fold_off[sg] + j] : 0.0f;
        gt[G.tap_off + n + i] = in ? fold[fold_total + fold_off[sg] + j] : 0.0f;
    }
}

// 32 values per lane -> lane l holds sum over lanes of v[l] (31 shuffles).
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
    for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
        bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            float send = upper ? v[i] : v[i + n / 2];
            float keep = upper ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

template <bool CPLX>
__global__ void __launch_bounds__(SIMT_THREADS)
k_simt(const float *__restrict__ x, int64_t ld_x, int64_t N, int64_t hop, int64_t F,
       const SimtGroup *__restrict__ groups, const SimtItem *__restrict__ items,
       const float *__restrict__ gtaps, int32_t S, int32_t wavelet, int32_t output,
       void *__restrict__ out, uint32_t *__restrict__ minmax, int32_t tf_all, uint32_t *__restrict__ nfbad,
       uint32_t *__restrict__ nfany) {
    extern __shared__ float xs[];
    const int64_t b = blockIdx.x;
    const SimtItem it = items[blockIdx.y];
    // the segment is staged once for all the item's scale groups (margin = their max L)
    const int LM = it.L;
    const int64_t k0 = it.k0;
    const int nf = (int)(F - k0 < (int64_t)tf_all ? F - k0 : (int64_t)tf_all);
    const int64_t seg_start = k0 * hop - LM;
    const int64_t seg_len = (int64_t)(nf - 1) * hop + 2 * LM + 1;
    const float *xb = x + b * ld_x;
    // non-finite samples are staged as 0 and recorded once (by the first chunk's item whose
    // frames own the sample) for the fix-up kernel
    const int64_t own_lo = k0 == 0 ? 0 : k0 * hop, own_hi = k0 + nf >= F ? N : (k0 + nf) * hop;
    for (int64_t i = threadIdx.x; i < seg_len; i += SIMT_THREADS) {
        int64_t g = seg_start + i;
        float v = (g >= 0 && g < N) ? __ldg(xb + g) : 0.0f;
        if (!is_finite_f(v)) {
            if (it.g0 == 0 && g >= own_lo && g < own_hi) nf_record(nfbad + b * (int64_t)(1 + WH_NF_CAP), nfany, g);
            v = 0.0f;
        }
        xs[i] = v;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float lmin = INFINITY, lmax = -INFINITY;
    for (int gi = it.g0; gi < it.g1; ++gi) {
    const SimtGroup G = groups[gi];
    const int L = G.L;
    const int width = L + 1;
    const float *tre = gtaps + G.tap_off;
    const float *tim = tre + (int64_t)SIMT_G * width;

    // FW frames x 8 scales per warp (real: 8 frames, complex: 4 frames and re + im)
    constexpr int FW = CPLX ? 4 : 8;
    constexpr int NA = FW * SIMT_G;  // accumulators per lane (re)
    for (int fq = warp * FW; fq < nf; fq += FW * (SIMT_THREADS / 32)) {
        float ar[NA], ai[CPLX ? NA : 1];
#pragma unroll
        for (int i = 0; i < NA; ++i) ar[i] = 0.0f;
        if constexpr (CPLX) {
#pragma unroll
            for (int i = 0; i < NA; ++i) ai[i] = 0.0f;
        }
        int c[FW];
#pragma unroll
        for (int f = 0; f < FW; ++f) c[f] = min(fq + f, nf - 1) * (int)hop + LM;
        const float4 *tr4 = reinterpret_cast<const float4 *>(tre);
        const float4 *ti4 = reinterpret_cast<const float4 *>(tim);
        for (int j = lane; j <= L; j += 32) {
            float p[FW], d[FW];
#pragma unroll
            for (int f = 0; f < FW; ++f) {
                float xp = xs[c[f] + j], xm = xs[c[f] - j];
                p[f] = (j == 0) ? xp : xp + xm;
                d[f] = xp - xm;
            }
            const float4 ta = __ldg(tr4 + 2 * j), tb = __ldg(tr4 + 2 * j + 1);
            const float t[SIMT_G] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y, tb.z, tb.w};
#pragma unroll
            for (int s2 = 0; s2 < SIMT_G; ++s2)
#pragma unroll
                for (int f = 0; f < FW; ++f) ar[f * SIMT_G + s2] = fmaf(p[f], t[s2], ar[f * SIMT_G + s2]);
            if constexpr (CPLX) {
                const float4 ua = __ldg(ti4 + 2 * j), ub = __ldg(ti4 + 2 * j + 1);
                const float u[SIMT_G] = {ua.x, ua.y, ua.z, ua.w, ub.x, ub.y, ub.z, ub.w};
#pragma unroll
                for (int s2 = 0; s2 < SIMT_G; ++s2)
#pragma unroll
                    for (int f = 0; f < FW; ++f) ai[f * SIMT_G + s2] = fmaf(d[f], u[s2], ai[f * SIMT_G + s2]);
            }
        }
        // 32 partial sums per block of 4 frames x 8 scales -> lane l holds (frame l >> 3, scale l & 7)
#pragma unroll
        for (int h = 0; h < FW / 4; ++h) {
            float blk[32], bim[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) blk[i] = ar[32 * h + i];
            float re = transpose_reduce32(blk, lane);
            float im = 0.0f;
            if constexpr (CPLX) {
#pragma unroll
                for (int i = 0; i < 32; ++i) bim[i] = ai[32 * h + i];
                im = transpose_reduce32(bim, lane);
            }
            const int f = 4 * h + (lane >> 3), s = lane & 7;
            const int64_t k = k0 + fq + f;
            if (s < G.ns && fq + f < nf) {
                const int64_t o = (b * S + G.s0 + s) * F + k;
                if (output == WH_OUT_COMPLEX64) {
                    reinterpret_cast<float2 *>(out)[o] =
                        make_float2(re, wavelet == WH_WAVELET_RMOR ? 0.0f : im);
                } else {
                    float v = apply_output(magnitude(re, im, wavelet), output);
                    reinterpret_cast<float *>(out)[o] = v;
                    lmin = fminf(lmin, v);
                    lmax = fmaxf(lmax, v);
                }
            }
        }
    }
    }  // scale groups
    if (minmax) {
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            lmin = fminf(lmin, __shfl_xor_sync(0xffffffffu, lmin, off));
            lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, off));
        }
        if (lane == 0 && lmin <= lmax) {
            atomicMin(minmax + 2 * b, f2key(lmin));
            atomicMax(minmax + 2 * b + 1, f2key(lmax));
        }
    }
}

int simt_prepare(Plan &p) {
    // groups of SIMT_G consecutive scales, heaviest (largest L) first
    p.groups.clear();
    int64_t tap_off = 0;
    for (int s0 = 0; s0 < p.S; s0 += SIMT_G) {
        SimtGroup G{};
        G.s0 = s0;
        G.ns = std::min(SIMT_G, p.S - s0);
        int64_t L = 0;
        for (int s = s0; s < s0 + G.ns; ++s) L = std::max(L, p.half[s]);
        if (2 * L + 1 > SIMT_SEG_MAX)
            return fail(WH_E_UNSUPPORTED, "scale too large for the SIMT engine's staged segment");
        G.L = (int32_t)L;
        int64_t tf = (SIMT_SEG_MAX - 2 * L - 1) / p.hop + 1;
        tf = std::min<int64_t>(tf, 128);
        if (tf >= 16) tf = tf / 16 * 16;
        tf = std::max<int64_t>(1, std::min<int64_t>(tf, p.F));
        G.tf = (int32_t)tf;
        G.tap_off = tap_off;
        tap_off += 2 * (int64_t)SIMT_G * (L + 1);
        p.groups.push_back(G);
    }
    // groups in decreasing cost (L) order, split into up to SIMT_CHUNKS contiguous chunks of
    // about equal tap work; an item = (chunk, frame tile): the clip segment is staged once per
    // item for all its groups (staging it per group re-read the input ~16x for short taps)
    std::vector<int> order(p.groups.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return p.groups[a].L > p.groups[b].L; });
    std::vector<SimtGroup> sorted;
    for (int g : order) sorted.push_back(p.groups[g]);
    p.groups = sorted;
    double work_total = 0.0;
    for (auto &G : p.groups) work_total += (double)(G.L + 1);
    constexpr int SIMT_CHUNKS = 4;
    std::vector<int> cuts{0};
    double acc = 0.0;
    for (size_t g = 0; g < p.groups.size(); ++g) {
        acc += (double)(p.groups[g].L + 1);
        if ((int)cuts.size() < SIMT_CHUNKS && acc >= work_total * (double)cuts.size() / SIMT_CHUNKS && g + 1 < p.groups.size())
            cuts.push_back((int)g + 1);
    }
    cuts.push_back((int)p.groups.size());
    int64_t Lmax_all = 0;
    for (auto &G : p.groups) Lmax_all = std::max<int64_t>(Lmax_all, G.L);
    int64_t tf = (SIMT_SEG_MAX - 2 * Lmax_all - 1) / p.hop + 1;
    tf = std::min<int64_t>(tf, 128);
    if (tf >= 16) tf = tf / 16 * 16;
    tf = std::max<int64_t>(1, std::min<int64_t>(tf, p.F));
    p.simt_tf = (int32_t)tf;
    std::vector<SimtItem> items;
    for (size_t c = 0; c + 1 < cuts.size(); ++c) {
        if (cuts[c] == cuts[c + 1]) continue;
        const int32_t Lc = p.groups[cuts[c]].L;  // the chunk's first group is its largest
        for (int64_t k0 = 0; k0 < p.F; k0 += tf) items.push_back(SimtItem{cuts[c], cuts[c + 1], (int32_t)k0, Lc});
    }
    if (items.size() > 65535u) return fail(WH_E_UNSUPPORTED, "too many SIMT work items");
    p.n_items = (int32_t)items.size();
    WH_CUDA_TRY(cudaMalloc(&p.d_groups, sizeof(SimtGroup) * p.groups.size()));
    WH_CUDA_TRY(cudaMalloc(&p.d_items, sizeof(SimtItem) * items.size()));
    WH_CUDA_TRY(cudaMalloc(&p.d_group_taps, sizeof(float) * std::max<int64_t>(tap_off, 1)));
    WH_CUDA_TRY(cudaMemcpy(p.d_groups, p.groups.data(), sizeof(SimtGroup) * p.groups.size(),
                           cudaMemcpyHostToDevice));
    WH_CUDA_TRY(cudaMemcpy(p.d_items, items.data(), sizeof(SimtItem) * items.size(), cudaMemcpyHostToDevice));
    dim3 grid(64, (unsigned)p.groups.size());
    k_group_taps<<<grid, 256>>>(p.d_fold, p.d_fold_off, p.d_half, p.fold_total, p.d_groups,
                                (int32_t)p.groups.size(), p.d_group_taps);
    WH_CUDA_TRY(cudaGetLastError());
    const size_t smem = sizeof(float) * ((size_t)(tf - 1) * p.hop + 2 * Lmax_all + 1);
    p.smem_bytes = smem;
    // the attribute belongs to the kernel, which every SIMT plan shares: raise it to the device
    // limit (a later plan with a smaller segment would otherwise lower it under this one)
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p.device);
    if ((int64_t)smem > optin) return fail(WH_E_UNSUPPORTED, "SIMT segment exceeds shared memory");
    WH_CUDA_TRY(cudaFuncSetAttribute(k_simt<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    WH_CUDA_TRY(cudaFuncSetAttribute(k_simt<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    return WH_OK;
}

int simt_launch(Plan &p, const float *x, int64_t clips, int64_t ld_x, void *out, cudaStream_t s, uint32_t *mm,
                uint32_t *nfbad, uint32_t *nfctl) {
    if (clips > 2147483647LL) return fail(WH_E_INVALID_ARG, "too many clips");
    dim3 grid((unsigned)clips, (unsigned)p.n_items);
    bool cplx = p.wavelet == WH_WAVELET_CMOR;
    if (p.norm == WH_NORM_NONE) mm = nullptr;
    (void)cudaGetLastError();  // drop stale non-sticky errors of earlier runtime calls
    if (cplx)
        k_simt<true><<<grid, SIMT_THREADS, p.smem_bytes, s>>>(x, ld_x, p.N, p.hop, p.F, p.d_groups, p.d_items,
                                                             p.d_group_taps, p.S, p.wavelet, p.output, out, mm, p.simt_tf, nfbad, nfctl + 1);
    else
        k_simt<false><<<grid, SIMT_THREADS, p.smem_bytes, s>>>(x, ld_x, p.N, p.hop, p.F, p.d_groups, p.d_items,
                                                              p.d_group_taps, p.S, p.wavelet, p.output, out, mm, p.simt_tf, nfbad, nfctl + 1);
    WH_CUDA_TRY(cudaGetLastError());
    return WH_OK;
}

}  // namespace wh
