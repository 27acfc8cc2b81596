// kernels_simt.cu -- SIMT (CUDA-core) kernels of the data-parallel SGD step:
// the FP32-tier GEMM (fwd / dgrad / wgrad), the fused softmax-CE head, the
// deterministic reductions, and K6, the fused average + momentum update.
// Paper: forward/backward of each replica, allreduce + average
// (P:182-184), update.  Design notes: DESIGN.md §Kernels.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "kernels.h"

namespace mtx {

namespace {

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// ------------------------------------------------------------------ SIMT GEMM
// 64x64 output tile per 256-thread CTA, BK = 16, each thread owns a 4x4 strided
// sub-tile (rows ty + 16i, cols tx + 16j) so shared-memory reads broadcast
// (A) or hit 16 consecutive banks (B).  Register prefetch of the next K tile
// overlaps global loads with the FMAs.  Every output element is summed over k
// in ascending order inside its split; splits are folded in ascending order by
// splitk_reduce -- no atomics, so results are run-to-run deterministic.
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <bool TA, bool TB, int EPI, bool AUG, bool PARTIAL>
__global__ void __launch_bounds__(NT) gemm_simt_kernel(GemmDesc g) {
    pdl_wait();
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int kper = (g.K + g.splits - 1) / g.splits;
    const int kbeg = blockIdx.z * kper, kend = min(g.K, kbeg + kper);
    const float *A = g.A + g.arow.row0() * g.lda;
    const int Mreal = AUG ? g.M - 1 : g.M;

    float ra[4], rb[4];
    auto load_a = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            int e = tid + NT * i, ml, kl;
            if (TA) { kl = e / BM; ml = e % BM; } else { ml = e / BK; kl = e % BK; }
            int m = m0 + ml, k = k0 + kl;
            float v = 0.f;
            if (k < kend) {
                if (m < Mreal) v = TA ? A[(int64_t)k * g.lda + m] : A[(int64_t)m * g.lda + k];
                else if (AUG && m == Mreal) v = 1.f;
            }
            ra[i] = v;
        }
    };
    auto load_b = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            int e = tid + NT * i, nl, kl;
            if (TB) { nl = e / BK; kl = e % BK; } else { kl = e / BN; nl = e % BN; }
            int n = n0 + nl, k = k0 + kl;
            float v = 0.f;
            if (k < kend && n < g.N) v = TB ? g.B[(int64_t)n * g.ldb + k] : g.B[(int64_t)k * g.ldb + n];
            rb[i] = v;
        }
    };
    auto store_ab = [&]() {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            int e = tid + NT * i, ml, kl, nl, kb;
            if (TA) { kl = e / BM; ml = e % BM; } else { ml = e / BK; kl = e % BK; }
            As[kl][ml] = ra[i];
            if (TB) { nl = e / BK; kb = e % BK; } else { kb = e / BN; nl = e % BN; }
            Bs[kb][nl] = rb[i];
        }
    };

    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[i][j] = 0.f;

    if (kbeg < kend) {
        load_a(kbeg);
        load_b(kbeg);
        for (int k0 = kbeg; k0 < kend; k0 += BK) {
            store_ab();
            __syncthreads();
            if (k0 + BK < kend) { load_a(k0 + BK); load_b(k0 + BK); }
            // Blocked summation: a BK-term FMA chain per tile, then one add into the
            // running sum -- error grows with BK + K/BK instead of K (fp32 tier, 1e-5).
            float blk[4][4];
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) blk[i][j] = 0.f;
#pragma unroll
            for (int kk = 0; kk < BK; kk++) {
                float a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; i++) a[i] = As[kk][ty + 16 * i];
#pragma unroll
                for (int j = 0; j < 4; j++) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) blk[i][j] = __fmaf_rn(a[i], b[j], blk[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = __fadd_rn(acc[i][j], blk[i][j]);
            __syncthreads();
        }
    }

#pragma unroll
    for (int i = 0; i < 4; i++) {
        int m = m0 + ty + 16 * i;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            int n = n0 + tx + 16 * j;
            if (n >= g.N) continue;
            float v = acc[i][j];
            if (PARTIAL) {
                g.partial[((int64_t)blockIdx.z * g.M + m) * g.N + n] = v;
                continue;
            }
            if (EPI == EPI_BIAS_RELU) v = fmaxf(v + g.bias[n], 0.f);
            else if (EPI == EPI_BIAS) v = v + g.bias[n];
            else if (EPI == EPI_MASK) v = g.mask[(int64_t)m * g.ldm + n] > 0.f ? v : 0.f;
            g.C[(int64_t)m * g.ldc + n] = v;
        }
    }
}

// Deterministic split-K fold (ascending z) with the GEMM epilogue applied after the sum:
// bias (+ReLU) for forward GEMMs, the ReLU mask for dgrad, plain store otherwise.
__global__ void splitk_reduce_kernel(const float *__restrict__ partial, int splits, int M, int N, float *C,
                                     int64_t ldc, int epi, const float *__restrict__ bias,
                                     const float *__restrict__ mask, int64_t ldm, float *C_hi, float *C_lo, F16Out fo,
                                     const uint32_t *__restrict__ mbits, int64_t mbits_ld) {
    pdl_wait();
    const float inv_so = fo.h ? 1.f / f16out_scale(fo) : 1.f;
    float amx = 0.f;
    const int64_t total = (int64_t)M * N;
    // 4 consecutive elements per thread (float4 when the row holds them), splits loaded 8 at a time
    const int64_t n4 = (total + 3) / 4;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e0 = 4 * q;
        const bool vec = (N % 4 == 0) && (e0 + 3 < total);
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        for (int z0 = 0; z0 < splits; z0 += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                if (z0 + u >= splits) break;
                const float *src = partial + (int64_t)(z0 + u) * total + e0;
                if (vec) {
                    v[u] = __ldcg((const float4 *)src);
                } else {
                    v[u].x = __ldcg(src);
                    v[u].y = e0 + 1 < total ? __ldcg(src + 1) : 0.f;
                    v[u].z = e0 + 2 < total ? __ldcg(src + 2) : 0.f;
                    v[u].w = e0 + 3 < total ? __ldcg(src + 3) : 0.f;
                }
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {  // ascending split order
                if (z0 + u >= splits) break;
                s[0] += v[u].x; s[1] += v[u].y; s[2] += v[u].z; s[3] += v[u].w;
            }
        }
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int64_t e = e0 + c;
            if (e >= total) break;
            const int64_t m = e / N, n = e % N;
            float r = s[c];
            if (epi == EPI_BIAS_RELU) r = fmaxf(r + bias[n], 0.f);
            else if (epi == EPI_BIAS) r = r + bias[n];
            else if (epi == EPI_MASK && mbits) r = ((mbits[m * mbits_ld + (n >> 5)] >> (n & 31)) & 1u) ? r : 0.f;
            else if (epi == EPI_MASK) r = mask[m * ldm + n] > 0.f ? r : 0.f;
            if (C) C[m * ldc + n] = r;
            if (C_hi) split_tf32(r, C_hi[m * ldc + n], C_lo[m * ldc + n]);
            if (fo.h) {
                uint16_t hh, ll;
                split_f16(r, inv_so, hh, ll);
                fo.h[m * fo.ld + n] = __ushort_as_half(hh);
                fo.l[m * fo.ld + n] = __ushort_as_half(ll);
                amx = fmaxf(amx, fabsf(r));
            }
        }
    }
    if (fo.h) {
        for (int o = 16; o > 0; o >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
        if ((threadIdx.x & 31) == 0) amax_atomic(&fo.ts->amax, amx);
    }
}

template <bool TA, bool TB, int EPI, bool AUG, bool PARTIAL>
void launch_gemm(const GemmDesc &g, dim3 grid, cudaStream_t s) {
    launch_pdl(gemm_simt_kernel<TA, TB, EPI, AUG, PARTIAL>, grid, dim3(NT), 0, s, g);
}

}  // namespace

cudaError_t gemm_simt(const GemmDesc &g, cudaStream_t s, LaunchHook *h) {
    dim3 grid(cdiv(g.N, BN), cdiv(g.M, BM), g.splits);
    const bool part = g.splits > 1;
    char name[96];
    snprintf(name, sizeof name, "%s[M=%d,N=%d,K=%d,splits=%d]",
             g.epi == EPI_MASK ? "gemm_simt_dgrad" : (g.ta ? "gemm_simt_wgrad" : "gemm_simt_fwd"), g.M, g.N, g.K,
             g.splits);
    if (h) h->before(name, s);
    // Instantiated combinations: fwd (NN, bias[+relu]), dgrad (NT, mask), wgrad (TN, aug, store or partial).
    if (!g.ta && !g.tb && g.epi == EPI_BIAS_RELU) launch_gemm<false, false, EPI_BIAS_RELU, false, false>(g, grid, s);
    else if (!g.ta && !g.tb && g.epi == EPI_BIAS) launch_gemm<false, false, EPI_BIAS, false, false>(g, grid, s);
    else if (!g.ta && g.tb && g.epi == EPI_MASK) launch_gemm<false, true, EPI_MASK, false, false>(g, grid, s);
    else if (!g.ta && g.tb && g.epi == EPI_STORE) launch_gemm<false, true, EPI_STORE, false, false>(g, grid, s);
    else if (g.ta && !g.tb && g.aug && !part) launch_gemm<true, false, EPI_STORE, true, false>(g, grid, s);
    else if (g.ta && !g.tb && g.aug && part) launch_gemm<true, false, EPI_STORE, true, true>(g, grid, s);
    else if (g.ta && !g.tb && !g.aug && !part) launch_gemm<true, false, EPI_STORE, false, false>(g, grid, s);
    else if (g.ta && !g.tb && !g.aug && part) launch_gemm<true, false, EPI_STORE, false, true>(g, grid, s);
    else return cudaErrorInvalidValue;
    if (h) h->after(name, s);
    if (part) return splitk_reduce(g.partial, g.splits, g.M, g.N, g.C, g.ldc, s, h);
    return cudaGetLastError();
}

cudaError_t splitk_reduce(const float *partial, int splits, int M, int N, float *C, int64_t ldc, cudaStream_t s,
                          LaunchHook *h, int epi, const float *bias, const float *mask, int64_t ldm, float *C_hi,
                          float *C_lo, F16Out fo, const uint32_t *mbits, int64_t mbits_ld) {
    int64_t total = (int64_t)M * N;
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total / 4 + 255) / 256, 148 * 8));
    char rn[80];
    snprintf(rn, sizeof rn, "splitk_reduce[M=%d,N=%d,splits=%d,epi=%d]", M, N, splits, epi);
    if (h) h->before(rn, s);
    launch_pdl(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, s, partial, splits, M, N, C, ldc, epi, bias, mask, ldm,
               C_hi, C_lo, fo, mbits, mbits_ld);
    if (h) h->after(rn, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ 3xTF32 operand planes
namespace {
__global__ void split_planes_kernel(const float *__restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                    float *__restrict__ hi, float *__restrict__ lo) {
    pdl_wait();
    const int64_t c4 = cols / 4, total = rows * c4;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q / c4, off = r * ld + 4 * (q % c4);
        const float4 v = __ldg((const float4 *)(x + off));
        float4 h, l;
        split_tf32(v.x, h.x, l.x);
        split_tf32(v.y, h.y, l.y);
        split_tf32(v.z, h.z, l.z);
        split_tf32(v.w, h.w, l.w);
        *(float4 *)(hi + off) = h;
        *(float4 *)(lo + off) = l;
    }
}
}  // namespace

cudaError_t split_planes(const float *x, int64_t rows, int64_t cols, int64_t ld, float *hi, float *lo, cudaStream_t s,
                         LaunchHook *h) {
    if (cols % 4 || ld % 4) return cudaErrorInvalidValue;
    const int64_t total = rows * (cols / 4);
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
    char name[64];
    snprintf(name, sizeof name, "split_planes[n=%lld]", (long long)(rows * cols));
    if (h) h->before(name, s);
    launch_pdl(split_planes_kernel, dim3(blocks), dim3(256), 0, s, x, rows, cols, ld, hi, lo);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ 3xF16 operand planes
namespace {
struct QArgs {
    QSeg seg[QSEG_MAX];
    int nseg;
    const float *ax;
    int64_t an;
    TScale *ts, *zero_ts;
    int n_zero;
    float *scratch;  // [0, 1024): per-CTA maxima; then the grid barrier's arrival count and generation
    int pre_parts;   // > 0: pre[0, pre_parts) already holds the maxima (written by the producer launch)
    const float *pre;
};
constexpr int Q_T = 512;

__device__ __forceinline__ float block_max(float v, float *red) {
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < Q_T / 32 ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    v = red[0];
    __syncthreads();
    return v;
}

// Grid-synchronous (every CTA resident: grid <= SM count): phase 1 max |x|, barrier, phase 2 planes.
__global__ void __launch_bounds__(Q_T) quantize_f16_kernel(const __grid_constant__ QArgs a) {
    pdl_wait();
    __shared__ float red[Q_T / 32];
    unsigned *bar = (unsigned *)(a.scratch + 1024);
    const int64_t tid = blockIdx.x * (int64_t)Q_T + threadIdx.x, nth = (int64_t)gridDim.x * Q_T;
    float m = 0.f;
    if (a.pre_parts > 0) {
    } else if (a.ax) {
        const bool v4 = ((uintptr_t)a.ax & 15) == 0;
        const int64_t n4 = v4 ? a.an / 4 : 0;
#pragma unroll 4
        for (int64_t i = tid; i < n4; i += nth) {
            const float4 v = __ldg((const float4 *)a.ax + i);
            m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
        for (int64_t i = 4 * n4 + tid; i < a.an; i += nth) m = fmaxf(m, fabsf(__ldg(a.ax + i)));
    } else {
        for (int q = 0; q < a.nseg; q++) {
            const QSeg &g = a.seg[q];
            for (int64_t i = tid; i < g.rows * g.cols; i += nth)
                m = fmaxf(m, fabsf(__ldg(g.x + (i / g.cols) * g.ld + i % g.cols)));
        }
    }
    if (a.pre_parts <= 0) m = block_max(m, red);
    if (a.pre_parts <= 0 && threadIdx.x == 0) {
        const unsigned gen0 = atomicAdd(bar + 1, 0u);  // before arriving: the generation cannot move yet
        a.scratch[blockIdx.x] = m;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0u;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (atomicAdd(bar + 1, 0u) == gen0) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
    m = 0.f;
    const int parts = a.pre_parts > 0 ? a.pre_parts : (int)gridDim.x;
    const float *src = a.pre_parts > 0 ? a.pre : a.scratch;
    for (int i = threadIdx.x; i < parts; i += Q_T) m = fmaxf(m, __ldcg(src + i));
    const float amax = block_max(m, red);
    const float sc = f16_scale_for(amax), inv = 1.f / sc;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ts->amax = amax;
        a.ts->scale = sc;
        for (int i = 0; i < a.n_zero; i++) a.zero_ts[i].amax = 0.f;
    }
    for (int q = 0; q < a.nseg; q++) {
        const QSeg &g = a.seg[q];
        const bool v4 = g.cols % 4 == 0 && g.ld % 4 == 0 && g.pld % 4 == 0 && ((uintptr_t)g.x & 15) == 0 &&
                        ((uintptr_t)g.hi & 7) == 0 && ((uintptr_t)g.lo & 7) == 0;
        if (v4 && g.rows * (g.cols / 4) < (1ll << 31)) {  // 32-bit index math (a 64-bit division per group was the cost)
            const unsigned c4 = (unsigned)(g.cols / 4), tot = (unsigned)(g.rows * c4);
            // 4 groups per thread per iteration, all 4 loads issued first (one load in flight per thread left this
            // pass latency-bound: 12 us for cfg4's 12.7 MB of parameters)
            constexpr int QU = 4;
            for (unsigned i0 = (unsigned)tid; i0 < tot; i0 += QU * (unsigned)nth) {
                float4 v[QU];
                int64_t ro[QU], co[QU];
#pragma unroll
                for (int u = 0; u < QU; u++) {
                    const unsigned i = i0 + u * (unsigned)nth;
                    const unsigned rq = i / c4;
                    ro[u] = rq;
                    co[u] = 4 * (int64_t)(i - rq * c4);
                    if (i < tot) v[u] = __ldg((const float4 *)(g.x + ro[u] * g.ld + co[u]));
                }
#pragma unroll
                for (int u = 0; u < QU; u++) {
                    if (i0 + u * (unsigned)nth >= tot) break;
                    uint16_t h[4], l[4];
                    split_f16(v[u].x, inv, h[0], l[0]);
                    split_f16(v[u].y, inv, h[1], l[1]);
                    split_f16(v[u].z, inv, h[2], l[2]);
                    split_f16(v[u].w, inv, h[3], l[3]);
                    const int64_t r = ro[u], c = co[u];
                    *(uint2 *)(g.hi + r * g.pld + c) = make_uint2(h[0] | ((uint32_t)h[1] << 16), h[2] | ((uint32_t)h[3] << 16));
                    *(uint2 *)(g.lo + r * g.pld + c) = make_uint2(l[0] | ((uint32_t)l[1] << 16), l[2] | ((uint32_t)l[3] << 16));
                }
            }
        } else {
            for (int64_t i = tid; i < g.rows * g.cols; i += nth) {
                const int64_t r = i / g.cols, c = i % g.cols;
                uint16_t h, l;
                split_f16(__ldg(g.x + r * g.ld + c), inv, h, l);
                g.hi[r * g.pld + c] = __ushort_as_half(h);
                g.lo[r * g.pld + c] = __ushort_as_half(l);
            }
        }
    }
}
}  // namespace

cudaError_t quantize_f16(const QSeg *segs, int nseg, const float *amax_x, int64_t amax_n, TScale *ts, TScale *zero_ts,
                         int n_zero, float *scratch, cudaStream_t s, LaunchHook *h, int pre_parts, const float *pre) {
    if (nseg < 0 || nseg > QSEG_MAX || !ts || !scratch) return cudaErrorInvalidValue;
    QArgs a{};
    int64_t work = 0;
    for (int q = 0; q < nseg; q++) {
        a.seg[q] = segs[q];
        work += segs[q].rows * segs[q].cols;
    }
    a.nseg = nseg;
    a.ax = amax_x;
    a.an = amax_n;
    a.ts = ts;
    a.zero_ts = zero_ts;
    a.n_zero = n_zero;
    a.scratch = scratch;
    a.pre_parts = pre_parts;
    a.pre = pre ? pre : scratch;
    work = std::max(work, amax_x && pre_parts <= 0 ? amax_n : 0);
    static int sms = [] {
        int d = 0, n = 148;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
        return n;
    }();
    // one CTA per SM at most: the barrier needs every CTA resident (1024 maxima slots)
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>({(work / 4 + Q_T - 1) / Q_T, sms, 1024}));
    char name[64];
    snprintf(name, sizeof name, "quantize_f16[n=%lld]", (long long)work);
    if (h) h->before(name, s);
    launch_pdl(quantize_f16_kernel, dim3(blocks), dim3(Q_T), 0, s, a);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ narrow weight gradient (N <= 16)
namespace {
constexpr int NW_T = 128, NW_ROWS = 32, NW_MAXN = 16;
// NJ: output columns rounded up to 2/4/8/16 (the HIGGS head has 2: no 16-wide padding work)
template <int NJ>
__global__ void __launch_bounds__(NW_T) wgrad_narrow_kernel(const float *__restrict__ A, int64_t lda, RowSel arow,
                                                          const float *__restrict__ dZ, int rows, int K_in, int N,
                                                          int rows_per, float *__restrict__ partial) {
    pdl_wait();
    __shared__ float sdz[NW_ROWS][NJ];
    const int k = blockIdx.x * NW_T + threadIdx.x;
    const int r0 = blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
    const float *Ab = A + arow.row0() * lda;
    float acc[NJ];
#pragma unroll
    for (int j = 0; j < NJ; j++) acc[j] = 0.f;
    for (int i0 = r0; i0 < r1; i0 += NW_ROWS) {
        const int nr = min(NW_ROWS, r1 - i0);
        for (int e = threadIdx.x; e < NW_ROWS * NJ; e += NW_T) {
            const int i = e / NJ, j = e % NJ;
            sdz[i][j] = (i < nr && j < N) ? dZ[(int64_t)(i0 + i) * N + j] : 0.f;
        }
        __syncthreads();
        if (k <= K_in) {
            float t[NJ];
#pragma unroll
            for (int j = 0; j < NJ; j++) t[j] = 0.f;
            // rows in flight per thread: the whole staged chunk for narrow outputs (few accumulators),
            // 8 otherwise -- the loads, not the FMAs, bound this kernel
            constexpr int RB = NJ <= 4 ? NW_ROWS : 8;
            for (int ib = 0; ib < nr; ib += RB) {
                float a8[RB];
#pragma unroll
                for (int u = 0; u < RB; u++)  // k == K_in: the bias row (a = 1)
                    a8[u] = (ib + u < nr) ? (k < K_in ? __ldg(Ab + (int64_t)(i0 + ib + u) * lda + k) : 1.f) : 0.f;
#pragma unroll
                for (int u = 0; u < RB; u++)
#pragma unroll
                    for (int j = 0; j < NJ; j++) t[j] = __fmaf_rn(a8[u], sdz[ib + u][j], t[j]);
            }
#pragma unroll
            for (int j = 0; j < NJ; j++) acc[j] = __fadd_rn(acc[j], t[j]);  // blocked summation
        }
        __syncthreads();
    }
    if (k <= K_in) {
#pragma unroll
        for (int j = 0; j < NJ; j++)
            if (j < N) partial[((int64_t)blockIdx.y * (K_in + 1) + k) * N + j] = acc[j];
    }
}

// out[j] = sum_p partial[p][j]: one warp per output, lane l sums p = l, l+32, ... ascending, then a
// fixed xor-shuffle tree -- deterministic.
__global__ void __launch_bounds__(256) fold_partials_kernel(const float *__restrict__ partial, int parts, int n,
                                                          float *__restrict__ out) {
    pdl_wait();
    const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (j >= n) return;
    float s = 0.f;
    for (int p = lane; p < parts; p += 32) s += __ldg(partial + (int64_t)p * n + j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[j] = s;
}
}  // namespace

namespace {
// 32 columns x 32 part-slices per CTA; slice ty sums parts ty, ty + 32, ... (8 loads in flight), the 32 slices
// are folded by a fixed tree (deterministic)
__global__ void __launch_bounds__(1024) colpart_fold_kernel(const float *__restrict__ partial, int parts, int n,
                                                              float *__restrict__ out) {
    pdl_wait();
    __shared__ float red[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + tx;
    float v = 0.f;
    if (j < n) {
        int p = ty;
        for (; p + 7 * 32 < parts; p += 8 * 32) {
            float x[8];
#pragma unroll
            for (int u = 0; u < 8; u++) x[u] = __ldg(partial + (int64_t)(p + 32 * u) * n + j);
#pragma unroll
            for (int u = 0; u < 8; u++) v += x[u];
        }
        for (; p < parts; p += 32) v += __ldg(partial + (int64_t)p * n + j);
    }
    red[ty][tx] = v;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) {
        if (ty < o) red[ty][tx] += red[ty + o][tx];
        __syncthreads();
    }
    if (ty == 0 && j < n) out[j] = red[0][tx];
}
}  // namespace

cudaError_t colpart_fold(const float *partial, int parts, int n, float *out, cudaStream_t s, LaunchHook *h) {
    char name[64];
    snprintf(name, sizeof name, "colpart_fold[parts=%d,n=%d]", parts, n);
    if (h) h->before(name, s);
    launch_pdl(colpart_fold_kernel, dim3(cdiv(n, 32)), dim3(1024), 0, s, partial, parts, n, out);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

cudaError_t fold_partials(const float *partial, int parts, int n, float *out, cudaStream_t s, LaunchHook *h) {
    char name[64];
    snprintf(name, sizeof name, "fold_partials[parts=%d,n=%d]", parts, n);
    if (h) h->before(name, s);
    const cudaError_t e = launch_pdl(fold_partials_kernel, dim3(cdiv(n, 8)), dim3(256), 0, s, partial, parts, n, out);
    if (h) h->after(name, s);
    return e;
}

cudaError_t wgrad_narrow(const float *A, int64_t lda, RowSel arow, const float *dZ, int rows, int K_in, int N,
                         float *dWb, float *partial, int64_t partial_cap, unsigned *ticket, cudaStream_t s,
                         LaunchHook *h) {
    (void)ticket;
    if (N > NW_MAXN) return cudaErrorInvalidValue;
    const int kb = (K_in + 1 + NW_T - 1) / NW_T;
    // ~8 CTAs of 4 warps per SM: each thread keeps 32 rows of loads in flight, so the bytes in flight (and the
    // bandwidth of this load-bound kernel) scale with the CTAs resident (4 per SM: 3.2 TB/s at cfg4)
    int splits = std::max(1, std::min((8 * 148 + kb - 1) / kb, (rows + 31) / 32));
    while (splits > 1 && (int64_t)splits * (K_in + 1) * N > partial_cap) splits--;
    const int rows_per = (rows + splits - 1) / splits;
    splits = (rows + rows_per - 1) / rows_per;
    char name[80];
    snprintf(name, sizeof name, "wgrad_narrow[M=%d,N=%d,K=%d,splits=%d]", K_in + 1, N, rows, splits);
    if (h) h->before(name, s);
    cudaError_t e;
    const dim3 grid(kb, splits);
    if (N <= 2) e = launch_pdl(wgrad_narrow_kernel<2>, grid, dim3(NW_T), 0, s, A, lda, arow, dZ, rows, K_in, N, rows_per, partial);
    else if (N <= 4) e = launch_pdl(wgrad_narrow_kernel<4>, grid, dim3(NW_T), 0, s, A, lda, arow, dZ, rows, K_in, N, rows_per, partial);
    else if (N <= 8) e = launch_pdl(wgrad_narrow_kernel<8>, grid, dim3(NW_T), 0, s, A, lda, arow, dZ, rows, K_in, N, rows_per, partial);
    else e = launch_pdl(wgrad_narrow_kernel<16>, grid, dim3(NW_T), 0, s, A, lda, arow, dZ, rows, K_in, N, rows_per, partial);
    if (h) h->after(name, s);
    if (e != cudaSuccess) return e;
    return fold_partials(partial, splits, (K_in + 1) * N, dWb, s, h);  // deterministic warp-per-output fold
}

// ------------------------------------------------------------------ column sums (bias gradients)
// Block = 8 warps over a contiguous K range; lane owns 4 consecutive columns (float4 loads, 128 B
// per warp per row when 16-B aligned); warp w sums rows k0 + w, k0 + w + 8, ... in order (4 rows in
// flight); the 8 warp sums are added in warp order; per-block partials are folded in block order.
namespace {
template <bool VEC>
__global__ void __launch_bounds__(256) colsum_kernel(const float *__restrict__ X, int K, int N, int64_t ld,
                                                     int k_per, float *__restrict__ partial, unsigned *ticket,
                                                     float *__restrict__ out) {
    pdl_wait();
    __shared__ float4 sh[8][32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = blockIdx.x * 128 + 4 * lane;
    const int k0 = blockIdx.y * k_per, k1 = min(K, k0 + k_per);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    auto load = [&](int k) -> float4 {
        const float *src = X + (int64_t)k * ld + n;
        if (VEC && n + 3 < N) return __ldg((const float4 *)src);
        return make_float4(n < N ? src[0] : 0.f, n + 1 < N ? src[1] : 0.f, n + 2 < N ? src[2] : 0.f,
                           n + 3 < N ? src[3] : 0.f);
    };
    for (int k = k0 + w; k < k1; k += 64) {  // 8 independent row loads in flight per thread
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = (k + 8 * u < k1) ? load(k + 8 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; u++) {
            acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
    }
    sh[w][lane] = acc;
    __syncthreads();
    if (w == 0) {
        float4 s = sh[0][lane];
#pragma unroll
        for (int i = 1; i < 8; i++) {
            s.x += sh[i][lane].x; s.y += sh[i][lane].y; s.z += sh[i][lane].z; s.w += sh[i][lane].w;
        }
        float *dst = partial + (int64_t)blockIdx.y * N + n;
        if (n < N) dst[0] = s.x;
        if (n + 1 < N) dst[1] = s.y;
        if (n + 2 < N) dst[2] = s.z;
        if (n + 3 < N) dst[3] = s.w;
    }
    // the last block to finish for this 128-column group folds the group's per-split partials:
    // warp w sums splits w, w + 8, ... (loads issued together), then warp 0 adds the 8 warp sums in
    // order -- a fixed summation tree, so the result is deterministic
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket + blockIdx.x, 1u) == gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n < N) {
        const int Z = (int)gridDim.y;
        for (int z0 = w; z0 < Z; z0 += 64) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int z = z0 + 8 * u;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (z < Z) {
                    const float *src = partial + (int64_t)z * N + n;
                    v[u].x = __ldcg(src);
                    if (n + 1 < N) v[u].y = __ldcg(src + 1);
                    if (n + 2 < N) v[u].z = __ldcg(src + 2);
                    if (n + 3 < N) v[u].w = __ldcg(src + 3);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                f.x += v[u].x; f.y += v[u].y; f.z += v[u].z; f.w += v[u].w;
            }
        }
    }
    __syncthreads();
    sh[w][lane] = f;
    __syncthreads();
    if (w == 0 && n < N) {
        float4 s = sh[0][lane];
#pragma unroll
        for (int i = 1; i < 8; i++) {
            s.x += sh[i][lane].x; s.y += sh[i][lane].y; s.z += sh[i][lane].z; s.w += sh[i][lane].w;
        }
        out[n] = s.x;
        if (n + 1 < N) out[n + 1] = s.y;
        if (n + 2 < N) out[n + 2] = s.z;
        if (n + 3 < N) out[n + 3] = s.w;
    }
    if (threadIdx.x == 0) ticket[blockIdx.x] = 0u;  // re-armed for the next launch
}
}  // namespace

cudaError_t colsum(const float *X, int K, int N, int64_t ld, float *out, float *partial, int64_t partial_cap,
                   unsigned *ticket, cudaStream_t s, LaunchHook *h) {
    if (N > 128 * COLSUM_MAX_GROUPS) {  // wider than the ticket array: consecutive launches per column block
        for (int c0 = 0; c0 < N; c0 += 128 * COLSUM_MAX_GROUPS) {
            const cudaError_t e = colsum(X + c0, K, std::min(N - c0, 128 * COLSUM_MAX_GROUPS), ld, out + c0, partial,
                                         partial_cap, ticket, s, h);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const int cols = (N + 127) / 128;
    int splits = std::max(1, std::min((K + 63) / 64, (2 * 148 + cols - 1) / cols));
    while (splits > 1 && (int64_t)splits * N > partial_cap) splits--;
    if (splits == 1 && partial_cap < N) return cudaErrorInvalidValue;
    const int k_per = (K + splits - 1) / splits;
    splits = (K + k_per - 1) / k_per;
    const bool vec = (ld % 4 == 0) && ((uintptr_t)X % 16 == 0);
    char name[64];
    snprintf(name, sizeof name, "colsum[K=%d,N=%d,splits=%d]", K, N, splits);
    if (h) h->before(name, s);
    if (vec) launch_pdl(colsum_kernel<true>, dim3(cols, splits), dim3(256), 0, s, X, K, N, ld, k_per, partial, ticket, out);
    else launch_pdl(colsum_kernel<false>, dim3(cols, splits), dim3(256), 0, s, X, K, N, ld, k_per, partial, ticket, out);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ fused head (last layer + loss)
// One warp per sample row.  Lane l owns features k = l, l+32, ...; the C logit
// partial sums are combined with a fixed xor-shuffle tree.  W_L (d x C, <= 64 KB)
// and b_L are staged in shared memory once per CTA.
namespace {

// NV = float4 groups per lane (d <= 128 * NV): lane owns features 4*lane + 128*t .. +3, loaded as
// float4 with all of the row's loads in flight before the FMAs.
// HEAD_WARPS: warps (rows in flight) per CTA -- 8 for small batches (cfg2: 64 CTAs), 2 for large ones
// (cfg4: more CTAs share the weight staging); measured, DESIGN.md §9
template <int NV, bool VEC, int HEAD_MAXC, int HEAD_WARPS>
__global__ void __launch_bounds__(HEAD_WARPS * 32) head_kernel(int rows, int d, int C_arg, const float *__restrict__ A,
                                                             RowSel arow, const float *__restrict__ Wb,
                                                             const int32_t *__restrict__ labels, RowSel lrow,
                                                             float inv_b, float *__restrict__ dZL,
                                                             float *__restrict__ dprev, float *__restrict__ dp_hi,
                                                             float *__restrict__ dp_lo, float *__restrict__ loss_rows,
                                                             float *__restrict__ loss_part, unsigned *ticket,
                                                             float *__restrict__ loss_out, F16Out fo) {
    pdl_wait();
    const float inv_so = fo.h ? 1.f / f16out_scale(fo) : 1.f;
    if (fo.h && blockIdx.x == 0 && threadIdx.x == 0) fo.ts->scale = 1.f / inv_so;
    float amx = 0.f;
    // HEAD_MAXC 2 and 10 are exact class counts (HIGGS, MNIST/CIFAR-10): the class loops compile
    // without predicates; the other instances take C at run time
    constexpr bool EXACT = HEAD_MAXC == 2 || HEAD_MAXC == 10;
    const int C = EXACT ? HEAD_MAXC : C_arg;
    // W_L staged TRANSPOSED: sWt[j][k], row pitch dp = round_up(d + 1, 4) (k == d: bias), so a lane
    // reads the weights of its 4 consecutive features as one conflict-free 128-bit load
    extern __shared__ __align__(16) float sWt[];
    __shared__ float swl[HEAD_WARPS];
    __shared__ bool last;
    const int dp = (d + 1 + 3) & ~3;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float *Abase = A + arow.row0() * (int64_t)d;
    const int32_t *lab = labels + lrow.row0();
    float av[NV][4];
    // features 4*lane + 128*t .. +3 of row i into dst, all loads in flight
    auto load_row = [&](int i, float (&dst)[NV][4]) {
        const float *a = Abase + (int64_t)i * d;
#pragma unroll
        for (int t = 0; t < NV; t++) {
            const int k = 4 * lane + 128 * t;
            if (VEC && k + 3 < d) {
                const float4 v = __ldg((const float4 *)(a + k));
                dst[t][0] = v.x; dst[t][1] = v.y; dst[t][2] = v.z; dst[t][3] = v.w;
            } else {
#pragma unroll
                for (int u = 0; u < 4; u++) dst[t][u] = (k + u < d) ? __ldg(a + k + u) : 0.f;
            }
        }
    };
    const int i_first = blockIdx.x * HEAD_WARPS + warp;
    if (i_first < rows) load_row(i_first, av);  // in flight while W_L is staged
    // row k of W_L (C weights; k == d is the bias row) -> column k of sWt, k in [d+1, dp) zeroed:
    // R rows per thread in flight, consecutive k across the warp (conflict-free stores), no
    // index division (it cost ~700 instructions per warp when it was e -> (e % C, e / C))
    constexpr int R = HEAD_WARPS >= 8 ? 3 : 4;  // rows per thread in flight: d <= 767 in one pass at 8 warps
    for (int k0 = threadIdx.x; k0 < dp; k0 += R * HEAD_WARPS * 32) {
        float v[R][HEAD_MAXC];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int k = k0 + r * HEAD_WARPS * 32;
#pragma unroll
            for (int j = 0; j < HEAD_MAXC; j++) v[r][j] = (j < C && k <= d) ? __ldg(Wb + (int64_t)k * C + j) : 0.f;
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int k = k0 + r * HEAD_WARPS * 32;
            if (k < dp) {
#pragma unroll
                for (int j = 0; j < HEAD_MAXC; j++) if (j < C) sWt[j * dp + k] = v[r][j];
            }
        }
    }
    __syncthreads();
    float wloss = 0.f;  // this warp's rows, in row order
    float hcs[NV][4];  // 3xF16 lean: this lane's column sums of dprev over the warp's rows
#pragma unroll
    for (int t = 0; t < NV; t++) hcs[t][0] = hcs[t][1] = hcs[t][2] = hcs[t][3] = 0.f;
    for (int i = i_first; i < rows; i += gridDim.x * HEAD_WARPS) {
        if (i != i_first) load_row(i, av);
        float z[HEAD_MAXC];
#pragma unroll
        for (int j = 0; j < HEAD_MAXC; j++) z[j] = 0.f;
#pragma unroll
        for (int t = 0; t < NV; t++) {
            const int k = 4 * lane + 128 * t;
            if (k < d) {
#pragma unroll
                for (int j = 0; j < HEAD_MAXC; j++)
                    if (j < C) {
                        const float4 w = *(const float4 *)(sWt + j * dp + k);  // features k..k+3 (zero-padded)
                        z[j] = __fmaf_rn(av[t][0], w.x, z[j]);
                        z[j] = __fmaf_rn(av[t][1], w.y, z[j]);
                        z[j] = __fmaf_rn(av[t][2], w.z, z[j]);
                        z[j] = __fmaf_rn(av[t][3], w.w, z[j]);
                    }
            }
        }
#pragma unroll
        for (int j = 0; j < HEAD_MAXC; j++) {
            if (j < C) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) z[j] += __shfl_xor_sync(0xffffffffu, z[j], o);
                z[j] += sWt[j * dp + d];  // bias after the full sum
            }
        }
        float m = z[0];
#pragma unroll
        for (int j = 1; j < HEAD_MAXC; j++) if (j < C) m = fmaxf(m, z[j]);
        float S = 0.f;
#pragma unroll
        for (int j = 0; j < HEAD_MAXC; j++) if (j < C) S += expf(z[j] - m);
        const int y = lab[i];
        float zy = 0.f;
#pragma unroll
        for (int j = 0; j < HEAD_MAXC; j++) if (j == y) zy = z[j];
        const float invS = 1.f / S;
        float dz[HEAD_MAXC];
#pragma unroll
        for (int j = 0; j < HEAD_MAXC; j++)
            dz[j] = (j < C) ? (expf(z[j] - m) * invS - (j == y ? 1.f : 0.f)) * inv_b : 0.f;
        const float li = m + logf(S) - zy;
        if (lane == 0) loss_rows[i] = li;
        wloss += li;
        if (lane < C) {
            float mine = 0.f;
#pragma unroll
            for (int j = 0; j < HEAD_MAXC; j++) if (j == lane) mine = dz[j];
            dZL[(int64_t)i * C + lane] = mine;
        }
        if (dprev) {
#pragma unroll
            for (int t = 0; t < NV; t++) {
                const int k = 4 * lane + 128 * t;
                if (k >= d) continue;
                float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int j = 0; j < HEAD_MAXC; j++)
                    if (j < C) {
                        const float4 w = *(const float4 *)(sWt + j * dp + k);
                        o[0] = __fmaf_rn(dz[j], w.x, o[0]);
                        o[1] = __fmaf_rn(dz[j], w.y, o[1]);
                        o[2] = __fmaf_rn(dz[j], w.z, o[2]);
                        o[3] = __fmaf_rn(dz[j], w.w, o[3]);
                    }
#pragma unroll
                for (int u = 0; u < 4; u++) o[u] = av[t][u] > 0.f ? o[u] : 0.f;
                if (fo.colpart) {
#pragma unroll
                    for (int u = 0; u < 4; u++) hcs[t][u] += k + u < d ? o[u] : 0.f;
                }
                float oh[4], ol[4];
                if (dp_hi) {
#pragma unroll
                    for (int u = 0; u < 4; u++) split_tf32(o[u], oh[u], ol[u]);
                }
                const int64_t off = (int64_t)i * d + k;
                if (fo.h) {
                    const int64_t po = (int64_t)i * fo.ld + k;
                    uint16_t hh[4], ll[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        split_f16(k + u < d ? o[u] : 0.f, inv_so, hh[u], ll[u]);
                        amx = fmaxf(amx, k + u < d ? fabsf(o[u]) : 0.f);
                    }
                    if (VEC && k + 3 < d) {
                        *(uint2 *)(fo.h + po) = make_uint2(hh[0] | ((uint32_t)hh[1] << 16), hh[2] | ((uint32_t)hh[3] << 16));
                        *(uint2 *)(fo.l + po) = make_uint2(ll[0] | ((uint32_t)ll[1] << 16), ll[2] | ((uint32_t)ll[3] << 16));
                    } else {
                        for (int u = 0; u < 4; u++)
                            if (k + u < d) {
                                fo.h[po + u] = __ushort_as_half(hh[u]);
                                fo.l[po + u] = __ushort_as_half(ll[u]);
                            }
                    }
                }
                if (fo.skip_f32) {
                } else if (VEC && k + 3 < d) {
                    *(float4 *)(dprev + off) = make_float4(o[0], o[1], o[2], o[3]);
                    if (dp_hi) {
                        *(float4 *)(dp_hi + off) = make_float4(oh[0], oh[1], oh[2], oh[3]);
                        *(float4 *)(dp_lo + off) = make_float4(ol[0], ol[1], ol[2], ol[3]);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        if (k + u < d) {
                            dprev[off + u] = o[u];
                            if (dp_hi) { dp_hi[off + u] = oh[u]; dp_lo[off + u] = ol[u]; }
                        }
                }
            }
        }
    }
    if (fo.h) {  // one atomic per CTA
        for (int o = 16; o > 0; o >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
        if (lane == 0) swl[warp] = amx;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < HEAD_WARPS; w++) amx = fmaxf(amx, swl[w]);
            amax_atomic(&fo.ts->amax, amx);
        }
        __syncthreads();
    }
    if (fo.colpart) {  // per-CTA column sums: the warps' sums in warp order (deterministic)
        float *csm = sWt + (size_t)dp * C;
#pragma unroll
        for (int t = 0; t < NV; t++) {
            const int k = 4 * lane + 128 * t;
            if (k < dp) *(float4 *)(csm + warp * dp + k) = make_float4(hcs[t][0], hcs[t][1], hcs[t][2], hcs[t][3]);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < d; k += HEAD_WARPS * 32) {
            float v = 0.f;
            for (int w = 0; w < HEAD_WARPS; w++) v += csm[w * dp + k];
            fo.colpart[(int64_t)blockIdx.x * d + k] = v;
        }
    }
    // loss: warp sums -> block sum (warp order) -> per-block partial; the last block folds the
    // partials in block order into the loss slot (deterministic, no float atomics)
    if (lane == 0) swl[warp] = wloss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float bsum = 0.f;
        for (int w = 0; w < HEAD_WARPS; w++) bsum += swl[w];
        loss_part[blockIdx.x] = bsum;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {  // all partials loaded in parallel, then a fixed-shape tree: deterministic
        __threadfence();
        __shared__ float red[HEAD_WARPS * 32];
        float v = 0.f;
        for (unsigned bidx = threadIdx.x; bidx < gridDim.x; bidx += blockDim.x) v += __ldcg(loss_part + bidx);
        red[threadIdx.x] = v;
        __syncthreads();
        for (int off = HEAD_WARPS * 16; off > 0; off >>= 1) {
            if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            *loss_out = red[0];
            *ticket = 0u;  // re-armed for the next step
        }
    }
}

template <int NV, bool VEC, int CM, int W>
cudaError_t launch_head(unsigned blocks, size_t smem, cudaStream_t s, int rows, int d, int C, const float *A, RowSel arow,
                        const float *Wb, const int32_t *labels, RowSel lrow, float inv_b, float *dZL, float *dprev,
                        float *dp_hi, float *dp_lo, float *loss_rows, float *loss_part, unsigned *ticket,
                        float *loss_out, F16Out fo) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(head_kernel<NV, VEC, CM, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return launch_pdl(head_kernel<NV, VEC, CM, W>, dim3(blocks), dim3(W * 32), smem, s, rows, d, C, A, arow, Wb,
                      labels, lrow, inv_b, dZL, dprev, dp_hi, dp_lo, loss_rows, loss_part, ticket, loss_out, fo);
}
}  // namespace

cudaError_t head_fused(int rows, int d, int C, const float *A, RowSel arow, const float *Wb, const int32_t *labels,
                       RowSel lrow, float inv_b, float *dZL, float *dprev, float *dp_hi, float *dp_lo,
                       float *loss_rows, float *loss_part, unsigned *ticket, float *loss_out, cudaStream_t s,
                       LaunchHook *h, F16Out fo, int *colpart_rows) {
    if (C > 16 || C < 1 || d > 1024) return cudaErrorInvalidValue;
    // enough rows per block that the block count stays <= 1024 (loss partial slots)
    int hw = rows > 2048 ? 2 : 8;
    if (const char *e = getenv("MTX_HEAD_WARPS")) hw = atoi(e) == 4 ? 4 : atoi(e) == 2 ? 2 : 8;  // development knob
    // column sums (3xF16 lean: the bias gradient of layer L-1) are one row per CTA: 8 warps and <= 256 CTAs
    // keep those rows few (the same 2048 warps in flight as 2-warp CTAs x 1024 at cfg4)
    if (fo.colpart) hw = 8;
    const size_t dpad = (size_t)((d + 1 + 3) & ~3);
    // W_L staged transposed; + one row of column sums per warp
    const size_t smem = sizeof(float) * dpad * (C + (fo.colpart ? hw : 0));
    const unsigned blocks = std::min<unsigned>(cdiv(rows, hw), fo.colpart ? 256u : 1024u);
    if (colpart_rows) *colpart_rows = (int)blocks;
    const bool vec = (d % 4 == 0) && ((uintptr_t)A % 16 == 0) && (dprev == nullptr || (uintptr_t)dprev % 16 == 0) &&
                     (dp_hi == nullptr || ((uintptr_t)dp_hi % 16 == 0 && (uintptr_t)dp_lo % 16 == 0));
    char name[80];
    snprintf(name, sizeof name, "head_softmax_xent[rows=%d,d=%d,C=%d,dgrad=%d]", rows, d, C, dprev ? 1 : 0);
    if (h) h->before(name, s);
    cudaError_t e;
#define HEAD_CASE4(NVv, CMv, Wv)                                                                               \
    e = vec ? launch_head<NVv, true, CMv, Wv>(blocks, smem, s, rows, d, C, A, arow, Wb, labels, lrow, inv_b, dZL,   \
                                              dprev, dp_hi, dp_lo, loss_rows, loss_part, ticket, loss_out, fo) \
            : launch_head<NVv, false, CMv, Wv>(blocks, smem, s, rows, d, C, A, arow, Wb, labels, lrow, inv_b, dZL,  \
                                               dprev, dp_hi, dp_lo, loss_rows, loss_part, ticket, loss_out, fo)
#define HEAD_CASE3(NVv, CMv)          \
    if (hw == 2) {                    \
        HEAD_CASE4(NVv, CMv, 2);      \
    } else if (hw == 4) {             \
        HEAD_CASE4(NVv, CMv, 4);      \
    } else {                          \
        HEAD_CASE4(NVv, CMv, 8);      \
    }
#define HEAD_CASE(NVv)             \
    if (C == 2) {                  \
        HEAD_CASE3(NVv, 2);        \
    } else if (C == 10) {          \
        HEAD_CASE3(NVv, 10);       \
    } else if (C <= 4) {           \
        HEAD_CASE3(NVv, 4);        \
    } else {                       \
        HEAD_CASE3(NVv, 16);       \
    }
    if (d <= 128) { HEAD_CASE(1); }
    else if (d <= 256) { HEAD_CASE(2); }
    else if (d <= 512) { HEAD_CASE(4); }
    else { HEAD_CASE(8); }
#undef HEAD_CASE
#undef HEAD_CASE3
#undef HEAD_CASE4
    if (h) h->after(name, s);
    return e;
}

// ------------------------------------------------------------------ deterministic block sum
namespace {
__global__ void __launch_bounds__(1024) reduce_sum_kernel(const float *__restrict__ v, int n, float *out) {
    pdl_wait();
    __shared__ float sh[1024];
    float acc = 0.f;
    for (int i = threadIdx.x; i < n; i += 1024) acc += v[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}
}  // namespace

cudaError_t reduce_sum(const float *v, int n, float *out, cudaStream_t s, LaunchHook *h) {
    char name[48];
    snprintf(name, sizeof name, "loss_reduce[n=%d]", n);
    if (h) h->before(name, s);
    launch_pdl(reduce_sum_kernel, dim3(1), dim3(1024), 0, s, v, n, out);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K6: fused average + update
// Streams G, w, v once (20 B/elem, 12 B/elem without velocity) with 128-bit
// accesses; 4 independent float4 per thread per iteration keep enough bytes in
// flight to saturate HBM3e; grid = a multiple of the 148 SMs.  Explicit
// __fmaf_rn pins the contraction so results are bit-identical to the oracle's
// fmaf (A4).
namespace {
constexpr int UPD_T = 256, UPD_U = 4;

template <bool HAS_V>
__global__ void __launch_bounds__(UPD_T) avg_update_kernel(const float4 *__restrict__ G, float4 *__restrict__ w,
                                                         float4 *__restrict__ v, int64_t n4, float invP, float lr,
                                                         float mu, int *flag, int64_t *win, int64_t B,
                                                         int64_t n_data, int tail, float4 *__restrict__ whi,
                                                         float4 *__restrict__ wlo, float *__restrict__ amax_part) {
    pdl_wait();
    bool bad = false;
    float wmax = 0.f;  // 3xF16: max |w| of this CTA's updated weights (the next planes' scale)
    const int64_t stride = (int64_t)gridDim.x * UPD_T * UPD_U;
    for (int64_t base = (int64_t)blockIdx.x * UPD_T * UPD_U + threadIdx.x; base < n4; base += stride) {
        float4 g[UPD_U], wv[UPD_U], vv[UPD_U];
#pragma unroll
        for (int u = 0; u < UPD_U; u++) {
            int64_t i = base + (int64_t)u * UPD_T;
            if (i < n4) {
                g[u] = __ldcs(G + i);
                wv[u] = __ldcs(w + i);
                if (HAS_V) vv[u] = __ldcs(v + i);
            }
        }
#pragma unroll
        for (int u = 0; u < UPD_U; u++) {
            int64_t i = base + (int64_t)u * UPD_T;
            if (i >= n4) continue;
            float gb[4] = {g[u].x * invP, g[u].y * invP, g[u].z * invP, g[u].w * invP};
            float *pw = &wv[u].x, *pv = &vv[u].x;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                bad |= !isfinite(gb[c]);
                if (HAS_V) {
                    pv[c] = __fmaf_rn(mu, pv[c], gb[c]);
                    pw[c] = __fmaf_rn(-lr, pv[c], pw[c]);
                } else {
                    pw[c] = __fmaf_rn(-lr, gb[c], pw[c]);
                }
            }
            __stcs(w + i, wv[u]);
            if (HAS_V) __stcs(v + i, vv[u]);
            if (amax_part) wmax = fmaxf(wmax, fmaxf(fmaxf(fabsf(pw[0]), fabsf(pw[1])), fmaxf(fabsf(pw[2]), fabsf(pw[3]))));
            if (whi) {  // 3xTF32: the next step's hi/lo planes of the updated weights
                float hi[4], lo[4];
#pragma unroll
                for (int c = 0; c < 4; c++) split_tf32(pw[c], hi[c], lo[c]);
                whi[i] = make_float4(hi[0], hi[1], hi[2], hi[3]);
                wlo[i] = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < tail) {  // the n % 4 scalar tail
        const int64_t i = 4 * n4 + threadIdx.x;
        float *Gs = (float *)G, *ws = (float *)w, *vs = (float *)v;
        float gb = Gs[i] * invP;
        bad |= !isfinite(gb);
        if (HAS_V) {
            vs[i] = __fmaf_rn(mu, vs[i], gb);
            ws[i] = __fmaf_rn(-lr, vs[i], ws[i]);
        } else {
            ws[i] = __fmaf_rn(-lr, gb, ws[i]);
        }
        if (whi) split_tf32(ws[i], ((float *)whi)[i], ((float *)wlo)[i]);
        wmax = fmaxf(wmax, fabsf(ws[i]));
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && flag) atomicOr(flag, 1);
    if (amax_part) {  // per-CTA maximum (the quantize launch that follows folds them: no re-read of w for its max)
        __shared__ float red[UPD_T / 32];
        for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = wmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < UPD_T / 32; k++) wmax = fmaxf(wmax, red[k]);
            amax_part[blockIdx.x] = wmax;
        }
    }
    if (win && blockIdx.x == 0 && threadIdx.x == 0) *win = (*win + B) % n_data;
}
}  // namespace

cudaError_t avg_update(float *G, float *w, float *v, int64_t n, float invP, float lr, float mu, int *flag,
                       int64_t *win, int64_t B, int64_t n_data, cudaStream_t s, LaunchHook *h, float *whi,
                       float *wlo, float *amax_part, int *nparts) {
    int64_t n4 = n / 4;
    int tail = (int)(n - 4 * n4);
    int64_t need = (n4 + UPD_T * UPD_U - 1) / (UPD_T * UPD_U);
    // at most 1024 CTAs when they leave per-CTA maxima (the quantize scratch's slots)
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, amax_part ? 1024 : 148 * 8));
    if (nparts) *nparts = (int)blocks;
    char name[64];
    snprintf(name, sizeof name, "avg_update[n=%lld,v=%d,planes=%d]", (long long)n, v ? 1 : 0, whi ? 1 : 0);
    if (h) h->before(name, s);
    if (v)
        launch_pdl(avg_update_kernel<true>, dim3(blocks), dim3(UPD_T), 0, s, (const float4 *)G, (float4 *)w, (float4 *)v,
                   n4, invP, lr, mu, flag, win, B, n_data, tail, (float4 *)whi, (float4 *)wlo, amax_part);
    else
        launch_pdl(avg_update_kernel<false>, dim3(blocks), dim3(UPD_T), 0, s, (const float4 *)G, (float4 *)w,
                   (float4 *)nullptr, n4, invP, lr, mu, flag, win, B, n_data, tail, (float4 *)whi, (float4 *)wlo,
                   amax_part);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ ordered fold (test mode, A2)
namespace {
__global__ void ordered_fold_kernel(const float *__restrict__ g, int P, int64_t stride, int64_t n, float *G) {
    pdl_wait();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        float s = g[e];
        for (int r = 1; r < P; r++) s = __fadd_rn(s, g[(int64_t)r * stride + e]);
        G[e] = s;
    }
}
}  // namespace

cudaError_t ordered_fold(const float *gathered, int P, int64_t stride, int64_t n, float *G, cudaStream_t s,
                         LaunchHook *h) {
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    char name[64];
    snprintf(name, sizeof name, "ordered_fold[n=%lld,P=%d]", (long long)n, P);
    if (h) h->before(name, s);
    launch_pdl(ordered_fold_kernel, dim3(blocks), dim3(256), 0, s, gathered, P, stride, n, G);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ init + digest
namespace {
__global__ void init_glorot_kernel(float *w, int64_t n, uint64_t seed, int t, float lim) {
    const uint64_t key = splitmix64(seed, (uint64_t)(16 + t));
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t bits = splitmix64(key, (uint64_t)e) >> 40;
        float u = __fmul_rn((float)bits, 5.9604644775390625e-08f);  // 2^-24, exact
        float s = __fsub_rn(__fmul_rn(2.f, u), 1.f);                 // exact
        w[e] = __fmul_rn(s, lim);
    }
}

__global__ void digest_kernel(const uint32_t *__restrict__ x, int64_t n, uint64_t salt, unsigned long long *out) {
    uint64_t acc = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        acc += splitmix64((uint64_t)x[e], (uint64_t)e + salt);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}
}  // namespace

namespace {
__global__ void empty_kernel() {}
__global__ void spin_kernel(uint64_t ns) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}
}  // namespace

cudaError_t empty_launch(cudaStream_t s, LaunchHook *h) {
    if (h) h->before("launch_overhead[calibration]", s);
    empty_kernel<<<1, 32, 0, s>>>();
    if (h) h->after("launch_overhead[calibration]", s);
    return cudaGetLastError();
}

cudaError_t gpu_spin(uint64_t ns, cudaStream_t s) {
    spin_kernel<<<1, 1, 0, s>>>(ns);
    return cudaGetLastError();
}

cudaError_t init_glorot(float *w, int64_t n, uint64_t seed, int tensor_index, float lim, cudaStream_t s) {
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    init_glorot_kernel<<<blocks, 256, 0, s>>>(w, n, seed, tensor_index, lim);
    return cudaGetLastError();
}

cudaError_t digest(const float *x, int64_t n, uint64_t salt, unsigned long long *out, cudaStream_t s) {
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    digest_kernel<<<blocks, 256, 0, s>>>((const uint32_t *)x, n, salt, out);
    return cudaGetLastError();
}

}  // namespace mtx
