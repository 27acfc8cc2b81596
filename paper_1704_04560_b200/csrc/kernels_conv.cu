// kernels_conv.cu -- LeNet-style convolution layers of the local forward/backward
// (CNN rows; config 3).  NHWC activations, weights
// W[kh][kw][ci][co] followed by the bias row (the augmented block of the flat buffer).
// Channel counts are small (C_out = 6, 16), so these are CUDA-core kernels built around
// shared-memory staging of whole images, templated on the output channels padded to CO:
//
//   conv_fwd  -- a CTA stages its samples' input images and the weights; one thread per pooled
//                output computes the 2x2 window's conv outputs for every channel (4 x CO register
//                accumulators, k*k*ci ascending), adds the bias, applies ReLU and the 2x2 max-pool
//                with the first maximum winning ties (reading A6).  Only the pooled value and its
//                argmax are stored: the backward's ReLU mask at the argmax is [P > 0].
//   conv_bwd  -- a CTA walks its samples: stages the input image, rebuilds dR = dP routed to the
//                argmax, masked by [P > 0] (max-pool + ReLU backward), straight into shared memory,
//                then (i) accumulates the weight gradient: each thread owns 4 patch elements x CO
//                channels over a fixed set of output positions, and (ii) writes the input gradient
//                dX (full correlation with W) of the sample.  Per-CTA weight-gradient partials are
//                folded by fold_partials in a fixed order (deterministic).
#include <stdio.h>

#include <algorithm>

#include "kernels.h"

namespace mtx {
namespace {

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

constexpr int CONV_T = 256;
constexpr int CONV_CI_MAX = 16;

__device__ __forceinline__ void stage_copy(const float *__restrict__ src, float *__restrict__ dst, int n) {
    if ((((uintptr_t)src) & 15) == 0 && (n & 3) == 0) {
#pragma unroll 4
        for (int i = threadIdx.x; i < n / 4; i += blockDim.x) ((float4 *)dst)[i] = __ldg((const float4 *)src + i);
    } else {
#pragma unroll 4
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
    }
}

// sW[e][CO] = W[e][co] for e < rows, zero for co >= g.co (rows of CO floats: 128-bit reads)
template <int CO>
__device__ __forceinline__ void stage_weights(const float *__restrict__ Wb, int rows, int co, float *__restrict__ sW) {
    for (int i = threadIdx.x; i < rows * CO; i += blockDim.x) {
        const int e = i / CO, j = i % CO;
        sW[i] = j < co ? __ldg(Wb + (int64_t)e * co + j) : 0.f;
    }
}

template <int CO>
__global__ void __launch_bounds__(CONV_T) conv_fwd_kernel(ConvGeom g, int rows, int spc, const float *__restrict__ X,
                                                        RowSel xrow, const float *__restrict__ Wb,
                                                        float *__restrict__ P, uint8_t *__restrict__ arg) {
    pdl_wait();
    extern __shared__ __align__(16) float sm[];
    const int KK = g.k * g.k * g.ci;
    const int in_sz = g.hi * g.wi * g.ci;
    float *sW = sm;                   // (KK + 1) x CO, bias row last
    float *sX = sm + (KK + 1) * CO;   // spc images
    stage_weights<CO>(Wb, KK + 1, g.co, sW);
    const int n0 = blockIdx.x * spc;
    const int ns = min(spc, rows - n0);
    stage_copy(X + (xrow.row0() + n0) * (int64_t)in_sz, sX, ns * in_sz);  // consecutive rows: one block
    __syncthreads();
    const int Pp = g.hp * g.wp;
    const int dx = g.ci, dy = g.wi * g.ci;  // window neighbours (0,1) and (1,0)
    for (int t = threadIdx.x; t < ns * Pp; t += blockDim.x) {
        const int s = t / Pp, pp = t % Pp;
        const int ph = pp / g.wp, pw = pp % g.wp;
        const float *xs = sX + s * in_sz;
        float acc[4][CO];
#pragma unroll
        for (int d = 0; d < 4; d++)
#pragma unroll
            for (int j = 0; j < CO; j++) acc[d][j] = 0.f;
        for (int kh = 0; kh < g.k; kh++)
            for (int kw = 0; kw < g.k; kw++) {
                const float *x0 = xs + ((2 * ph + kh) * g.wi + (2 * pw + kw)) * g.ci;
                const float *wr = sW + ((kh * g.k + kw) * g.ci) * CO;
                for (int c = 0; c < g.ci; c++) {
                    const float xv[4] = {x0[c], x0[dx + c], x0[dy + c], x0[dy + dx + c]};
#pragma unroll
                    for (int j4 = 0; j4 < CO / 4; j4++) {
                        const float4 w = *(const float4 *)(wr + c * CO + 4 * j4);
#pragma unroll
                        for (int d = 0; d < 4; d++) {
                            acc[d][4 * j4 + 0] = __fmaf_rn(xv[d], w.x, acc[d][4 * j4 + 0]);
                            acc[d][4 * j4 + 1] = __fmaf_rn(xv[d], w.y, acc[d][4 * j4 + 1]);
                            acc[d][4 * j4 + 2] = __fmaf_rn(xv[d], w.z, acc[d][4 * j4 + 2]);
                            acc[d][4 * j4 + 3] = __fmaf_rn(xv[d], w.w, acc[d][4 * j4 + 3]);
                        }
                    }
                }
            }
        const int64_t ob = ((int64_t)(n0 + s) * Pp + pp) * g.co;
        uint8_t *ab = arg + (int64_t)(n0 + s) * conv_arg_pitch(g) + pp * g.co;
#pragma unroll
        for (int j = 0; j < CO; j++) {
            if (j >= g.co) break;
            const float bias = sW[KK * CO + j];
            float best = 0.f;
            int barg = 0;
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const float z = fmaxf(acc[d][j] + bias, 0.f);  // bias after the sum (A13), ReLU
                if (d == 0 || z > best) {                       // first maximum wins (A6)
                    best = z;
                    barg = d;
                }
            }
            P[ob + j] = best;
            ab[j] = (uint8_t)barg;
        }
    }
}

// 1-D bulk copy global -> shared (TMA engine), completion counted on the mbarrier in bytes
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// dR row p of the backward's shared tile: CO floats as CO/4 16-B chunks, XOR-swizzled by the row so
// that neighbouring rows (one per lane in the input-gradient loop) fall on different banks.
template <int CO>
__device__ __forceinline__ int dr_off(int p, int chunk) {
    constexpr int NCH = CO / 4, R = 32 / CO;  // chunks per row, rows per 128-B line
    return p * CO + 4 * (chunk ^ ((p / R) % NCH));
}

// Per-sample inputs of the backward, double-buffered in shared memory.
struct BwdBuf {
    float *x, *p, *dp;
    uint8_t *a;
};

template <int CO>
__global__ void __launch_bounds__(CONV_T) conv_bwd_kernel(ConvGeom g, int rows, int spc, const float *__restrict__ X,
                                                        RowSel xrow, const float *__restrict__ dP,
                                                        const float *__restrict__ P, const uint8_t *__restrict__ arg,
                                                        const float *__restrict__ Wb, float *__restrict__ dX,
                                                        float *__restrict__ partial) {
    pdl_wait();
    extern __shared__ __align__(16) float sm[];
    const int KK = g.k * g.k * g.ci, E = KK + 1, EB = (E + 3) / 4;
    const int in_sz = g.hi * g.wi * g.ci;
    const int HWc = g.hc * g.wc, Pp = g.hp * g.wp;
    const int ppc = Pp * g.co, apitch = conv_arg_pitch(g);
    const int in_pad = (in_sz + 3) & ~3, ppc_pad = (ppc + 3) & ~3;
    float *sD = sm;                           // dR of the current sample [hc*wc][CO]
    float *sW = sD + HWc * CO;                // W [KK][CO] (input gradient only)
    float *red = sW + (dX ? KK * CO : 0);     // [4*EB][CO] CTA reduction of the weight gradient
    float *bufs = red + 4 * EB * CO;
    const int bstride = in_pad + 2 * ppc_pad + apitch / 4;
    auto buf = [&](int b) {
        float *base = bufs + b * bstride;
        return BwdBuf{base, base + in_pad, base + in_pad + ppc_pad, (uint8_t *)(base + in_pad + 2 * ppc_pad)};
    };
    uint64_t *bars = (uint64_t *)(bufs + 2 * bstride);
    const uint32_t bar0 = smem_u32(bars);
    if (dX) stage_weights<CO>(Wb, KK, g.co, sW);
    const int tid = threadIdx.x;
    // weight-gradient role: patch-element block eb (4 consecutive e) x position group pg
    const int PG = blockDim.x / EB;
    const int eb = tid % EB, pg = tid / EB;
    const bool wg = pg < PG;
    int off[4];
    bool ones[4], valid[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int e = eb + EB * j;  // lanes of a warp read consecutive patch elements: no bank conflicts
        valid[j] = e < E;
        ones[j] = e == KK;  // the bias row: the patch element is 1
        const int kc = g.k * g.ci;
        const int kh = e / kc, r = e % kc, kw = r / g.ci, c = r % g.ci;
        off[j] = e < KK ? (kh * g.wi + kw) * g.ci + c : 0;
    }
    float acc[4][CO];
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
        for (int q = 0; q < CO; q++) acc[j][q] = 0.f;
    const int n_begin = blockIdx.x * spc, n_end = min(rows, n_begin + spc);
    const float *Xb = X + xrow.row0() * (int64_t)in_sz;
    // bulk path: every per-sample block is a 16-B multiple at a 16-B aligned address
    const bool bulk = (in_sz % 4 == 0) && (ppc % 4 == 0) && ((((uintptr_t)Xb) | ((uintptr_t)P) | ((uintptr_t)dP) |
                                                              ((uintptr_t)arg)) & 15) == 0;
    auto issue = [&](int n, int b) {  // one thread: the four copies of sample n into buffer b
        const uint32_t bar = bar0 + 8 * b;
        const BwdBuf B = buf(b);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // buffer's previous reads done (barrier)
        mbar_expect_tx(bar, (uint32_t)(4 * in_sz + 8 * ppc + apitch));
        bulk_g2s(B.x, Xb + (int64_t)n * in_sz, 4 * in_sz, bar);
        bulk_g2s(B.p, P + (int64_t)n * ppc, 4 * ppc, bar);
        bulk_g2s(B.dp, dP + (int64_t)n * ppc, 4 * ppc, bar);
        bulk_g2s(B.a, arg + (int64_t)n * apitch, apitch, bar);
    };
    if (bulk && tid == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (bulk && tid == 0 && n_begin < n_end) issue(n_begin, 0);
    for (int n = n_begin; n < n_end; n++) {
        const int it = n - n_begin, b = it & 1;
        const BwdBuf B = buf(b);
        if (bulk) {
            if (tid == 0 && n + 1 < n_end) issue(n + 1, b ^ 1);  // prefetch: overlaps this sample's compute
        } else {
            for (int i = tid; i < in_sz; i += blockDim.x) B.x[i] = __ldg(Xb + (int64_t)n * in_sz + i);
            for (int i = tid; i < ppc; i += blockDim.x) {
                B.p[i] = __ldg(P + (int64_t)n * ppc + i);
                B.dp[i] = __ldg(dP + (int64_t)n * ppc + i);
                B.a[i] = __ldg(arg + (int64_t)n * apitch + i);
            }
        }
        for (int i = tid; i < HWc * CO / 4; i += blockDim.x) ((float4 *)sD)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (bulk) mbar_wait(bar0 + 8 * b, (it >> 1) & 1);
        __syncthreads();
        // max-pool + ReLU backward: dR = dP at the argmax when P > 0, zero elsewhere
        for (int i = tid; i < ppc; i += blockDim.x) {
            if (B.p[i] > 0.f) {
                const int co = i % g.co, pp = i / g.co, ph = pp / g.wp, pw = pp % g.wp;
                const int d = B.a[i];
                const int p = (2 * ph + (d >> 1)) * g.wc + 2 * pw + (d & 1);
                sD[dr_off<CO>(p, co >> 2) + (co & 3)] = B.dp[i];
            }
        }
        __syncthreads();
        const float *sX = B.x;
        if (wg) {  // dW[e][co] += patch[p][e] * dR[p][co] over this thread's positions p = pg + PG*i
            int oh = pg / g.wc, ow = pg % g.wc;
            for (int p = pg; p < HWc; p += PG) {
                const float *xr = sX + (oh * g.wi + ow) * g.ci;
                float xv[4];
#pragma unroll
                for (int j = 0; j < 4; j++) xv[j] = ones[j] ? 1.f : (valid[j] ? xr[off[j]] : 0.f);
                const float *dr = sD;
#pragma unroll
                for (int q4 = 0; q4 < CO / 4; q4++) {
                    const float4 dv = *(const float4 *)(dr + dr_off<CO>(p, q4));
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        acc[j][4 * q4 + 0] = __fmaf_rn(xv[j], dv.x, acc[j][4 * q4 + 0]);
                        acc[j][4 * q4 + 1] = __fmaf_rn(xv[j], dv.y, acc[j][4 * q4 + 1]);
                        acc[j][4 * q4 + 2] = __fmaf_rn(xv[j], dv.z, acc[j][4 * q4 + 2]);
                        acc[j][4 * q4 + 3] = __fmaf_rn(xv[j], dv.w, acc[j][4 * q4 + 3]);
                    }
                }
                ow += PG;
                while (ow >= g.wc) {
                    ow -= g.wc;
                    oh++;
                }
            }
        }
        if (dX) {  // dX[h][w][c] = sum_{kh,kw,co} dR[h-kh][w-kw][co] W[kh][kw][c][co]  (kh, kw, co ascending)
            for (int q = tid; q < g.hi * g.wi; q += blockDim.x) {
                const int h = q / g.wi, w = q % g.wi;
                float a[CONV_CI_MAX];
#pragma unroll
                for (int c = 0; c < CONV_CI_MAX; c++) a[c] = 0.f;
                for (int kh = 0; kh < g.k; kh++) {
                    const int oh = h - kh;
                    if (oh < 0 || oh >= g.hc) continue;
                    for (int kw = 0; kw < g.k; kw++) {
                        const int ow = w - kw;
                        if (ow < 0 || ow >= g.wc) continue;
                        const int p = oh * g.wc + ow;
                        const float *wr = sW + ((kh * g.k + kw) * g.ci) * CO;
#pragma unroll
                        for (int q4 = 0; q4 < CO / 4; q4++) {
                            const float4 dv = *(const float4 *)(sD + dr_off<CO>(p, q4));
#pragma unroll
                            for (int c = 0; c < CONV_CI_MAX; c++) {
                                if (c >= g.ci) break;
                                const float4 wv = *(const float4 *)(wr + c * CO + 4 * q4);
                                a[c] = __fmaf_rn(dv.x, wv.x, a[c]);
                                a[c] = __fmaf_rn(dv.y, wv.y, a[c]);
                                a[c] = __fmaf_rn(dv.z, wv.z, a[c]);
                                a[c] = __fmaf_rn(dv.w, wv.w, a[c]);
                            }
                        }
                    }
                }
                float *out = dX + ((int64_t)n * g.hi * g.wi + q) * g.ci;
#pragma unroll
                for (int c = 0; c < CONV_CI_MAX; c++)
                    if (c < g.ci) out[c] = a[c];
            }
        }
        __syncthreads();  // sX / sD are rewritten for the next sample
    }
    // the PG position groups of each patch-element block are summed in ascending group order through
    // shared memory, then the CTA's partial is written out
    for (int r = 0; r < PG; r++) {
        if (wg && pg == r) {
#pragma unroll
            for (int j = 0; j < 4; j++)
#pragma unroll
                for (int q = 0; q < CO; q++) {
                    float *dst = red + (eb + EB * j) * CO + q;
                    *dst = r == 0 ? acc[j][q] : *dst + acc[j][q];
                }
        }
        __syncthreads();
    }
    float *pb = partial + (int64_t)blockIdx.x * E * g.co;
    for (int i = tid; i < E * g.co; i += blockDim.x) pb[i] = red[(i / g.co) * CO + i % g.co];
}

// Weight gradient only (the input gradient runs elsewhere: conv_tc.cu, or the layer has none):
//   dW[e][co] = sum_{n, p} X_n[p + off(e)] * dR_n[p][co]   (e < k*k*ci),   db[co] = sum_{n, p} dR_n[p][co].
// Per CTA: its samples' images and pooled inputs double-buffered in shared memory (bulk copies), dR rebuilt per
// sample (each pooled element writes its 2x2 window: dP at the argmax when P > 0, zero elsewhere).  Thread
// (eb, pg) owns EPT patch elements eb + NEB*j x CO channels (EPT * CO register accumulators) over the conv
// output pixels pg, pg + PG, ...: per pixel EPT scalar + CO/4 vector shared loads feed EPT*CO FMAs, with no
// per-pixel selects (the bias row is a separate column sum by the CTA's spare threads).  Per-CTA partials
// (the position groups summed in ascending order) are folded by fold_partials.
template <int CO, int EPT>
__global__ void __launch_bounds__(CONV_T) conv_wgrad_kernel(ConvGeom g, int rows, int spc, const float *__restrict__ X,
                                                          RowSel xrow, const float *__restrict__ dP,
                                                          const float *__restrict__ P, const uint8_t *__restrict__ arg,
                                                          float *__restrict__ partial) {
    pdl_wait();
    extern __shared__ __align__(16) float sm[];
    const int KK = g.k * g.k * g.ci, E = KK + 1;
    const int NEB = (KK + EPT - 1) / EPT;  // patch-element blocks (the bias row excluded)
    const int PG = CONV_T / NEB - (CONV_T % NEB == 0 ? 1 : 0);  // pixel groups (>= 1 spare thread for the bias)
    const int in_sz = g.hi * g.wi * g.ci;
    const int HWc = g.hc * g.wc, Pp = g.hp * g.wp;
    const int ppc = Pp * g.co, apitch = conv_arg_pitch(g);
    const int in_pad = (in_sz + 3) & ~3, ppc_pad = (ppc + 3) & ~3;
    float *sD = sm;                  // dR [hc*wc][CO]
    float *red = sD + HWc * CO;      // [E][CO] CTA partial
    float *bufs = red + E * CO;
    const int bstride = in_pad + 2 * ppc_pad + apitch / 4;
    auto buf = [&](int b) {
        float *base = bufs + b * bstride;
        return BwdBuf{base, base + in_pad, base + in_pad + ppc_pad, (uint8_t *)(base + in_pad + 2 * ppc_pad)};
    };
    uint64_t *bars = (uint64_t *)(bufs + 2 * bstride);
    const uint32_t bar0 = smem_u32(bars);
    const int tid = threadIdx.x;
    const int eb = tid % NEB, pg = tid / NEB;
    const bool wg = pg < PG;
    const bool bias_thread = tid >= NEB * PG;  // spare threads: the bias column sum
    const int nbias = CONV_T - NEB * PG;
    int off[EPT];
#pragma unroll
    for (int j = 0; j < EPT; j++) {
        // interleaved (e = eb + NEB * j): the lanes of a warp read consecutive patch elements -- conflict-free
        const int e = min(eb + NEB * j, KK - 1);  // past KK: any valid address (those accumulators are dropped)
        const int kc = g.k * g.ci, kh = e / kc, r = e % kc, kw = r / g.ci, c = r % g.ci;
        off[j] = (kh * g.wi + kw) * g.ci + c;
    }
    float acc[EPT][CO];
#pragma unroll
    for (int j = 0; j < EPT; j++)
#pragma unroll
        for (int q = 0; q < CO; q++) acc[j][q] = 0.f;
    float bacc[CO];
#pragma unroll
    for (int q = 0; q < CO; q++) bacc[q] = 0.f;
    // pixel walk of this thread: p = pg + PG * i, (oh, ow) advanced by (PG / wc, PG % wc) with one carry
    const int d_oh = PG / g.wc, d_ow = PG % g.wc;
    for (int i = tid; i < HWc * CO / 4; i += CONV_T) ((float4 *)sD)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int n_begin = (int)((int64_t)blockIdx.x * rows / gridDim.x), n_end = (int)((int64_t)(blockIdx.x + 1) * rows / gridDim.x);
    (void)spc;  // samples split evenly over the grid (3 or 4 each on 296 CTAs for b = 1024)
    const float *Xb = X + xrow.row0() * (int64_t)in_sz;
    const bool bulk = (in_sz % 4 == 0) && (ppc % 4 == 0) && ((((uintptr_t)Xb) | ((uintptr_t)P) | ((uintptr_t)dP) |
                                                              ((uintptr_t)arg)) & 15) == 0;
    auto issue = [&](int n, int b) {
        const uint32_t bar = bar0 + 8 * b;
        const BwdBuf B = buf(b);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, (uint32_t)(4 * in_sz + 8 * ppc + apitch));
        bulk_g2s(B.x, Xb + (int64_t)n * in_sz, 4 * in_sz, bar);
        bulk_g2s(B.p, P + (int64_t)n * ppc, 4 * ppc, bar);
        bulk_g2s(B.dp, dP + (int64_t)n * ppc, 4 * ppc, bar);
        bulk_g2s(B.a, arg + (int64_t)n * apitch, apitch, bar);
    };
    if (bulk && tid == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (bulk && tid == 0 && n_begin < n_end) issue(n_begin, 0);
    for (int n = n_begin; n < n_end; n++) {
        const int it = n - n_begin, b = it & 1;
        const BwdBuf B = buf(b);
        if (bulk) {
            if (tid == 0 && n + 1 < n_end) issue(n + 1, b ^ 1);
            mbar_wait(bar0 + 8 * b, (it >> 1) & 1);
        } else {
            for (int t = tid; t < in_sz; t += CONV_T) B.x[t] = __ldg(Xb + (int64_t)n * in_sz + t);
            for (int t = tid; t < ppc; t += CONV_T) {
                B.p[t] = __ldg(P + (int64_t)n * ppc + t);
                B.dp[t] = __ldg(dP + (int64_t)n * ppc + t);
                B.a[t] = __ldg(arg + (int64_t)n * apitch + t);
            }
            __syncthreads();
        }
        // max-pool + ReLU backward: each pooled element writes its whole 2x2 window of dR
        for (int t = tid; t < ppc; t += CONV_T) {
            const int co = t % g.co, pp = t / g.co, ph = pp / g.wp, pw = pp % g.wp;
            const float v = B.p[t] > 0.f ? B.dp[t] : 0.f;
            const int d = B.a[t];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int pix = (2 * ph + (q >> 1)) * g.wc + 2 * pw + (q & 1);
                sD[dr_off<CO>(pix, co >> 2) + (co & 3)] = q == d ? v : 0.f;
            }
        }
        __syncthreads();
        const float *sX = B.x;
        if (wg) {
            int oh = pg / g.wc, ow = pg % g.wc;
            for (int pix = pg; pix < HWc; pix += PG) {
                const float *xr = sX + (oh * g.wi + ow) * g.ci;
                float xv[EPT];
#pragma unroll
                for (int j = 0; j < EPT; j++) xv[j] = xr[off[j]];
#pragma unroll
                for (int q4 = 0; q4 < CO / 4; q4++) {
                    const float4 dv = *(const float4 *)(sD + dr_off<CO>(pix, q4));
#pragma unroll
                    for (int j = 0; j < EPT; j++) {
                        acc[j][4 * q4 + 0] = __fmaf_rn(xv[j], dv.x, acc[j][4 * q4 + 0]);
                        acc[j][4 * q4 + 1] = __fmaf_rn(xv[j], dv.y, acc[j][4 * q4 + 1]);
                        acc[j][4 * q4 + 2] = __fmaf_rn(xv[j], dv.z, acc[j][4 * q4 + 2]);
                        acc[j][4 * q4 + 3] = __fmaf_rn(xv[j], dv.w, acc[j][4 * q4 + 3]);
                    }
                }
                ow += d_ow;
                oh += d_oh;
                if (ow >= g.wc) {
                    ow -= g.wc;
                    oh++;
                }
            }
        } else if (bias_thread) {  // db[co] partial: pixels bias_idx, bias_idx + nbias, ...
            for (int pix = tid - NEB * PG; pix < HWc; pix += nbias) {
#pragma unroll
                for (int q4 = 0; q4 < CO / 4; q4++) {
                    const float4 dv = *(const float4 *)(sD + dr_off<CO>(pix, q4));
                    bacc[4 * q4 + 0] += dv.x; bacc[4 * q4 + 1] += dv.y;
                    bacc[4 * q4 + 2] += dv.z; bacc[4 * q4 + 3] += dv.w;
                }
            }
        }
        __syncthreads();  // sD and this buffer are rewritten for the next sample
    }
    // CTA reduction: every thread parks its accumulators in the (now free) shared memory, slot[pg][e][co] and
    // bslot[b][co]; then each output (e, co) is summed over the position groups (bias: the spare threads) in
    // ascending order -- deterministic, no serial barrier chain
    (void)red;
    const int EE = NEB * EPT;
    float *slot = sm, *bslot = sm + (size_t)PG * EE * CO;
    if (wg) {
#pragma unroll
        for (int j = 0; j < EPT; j++)
#pragma unroll
            for (int q4 = 0; q4 < CO / 4; q4++)
                *(float4 *)(slot + ((size_t)pg * EE + eb + NEB * j) * CO + 4 * q4) =
                    make_float4(acc[j][4 * q4], acc[j][4 * q4 + 1], acc[j][4 * q4 + 2], acc[j][4 * q4 + 3]);
    } else if (bias_thread) {
#pragma unroll
        for (int q = 0; q < CO; q++) bslot[(tid - NEB * PG) * CO + q] = bacc[q];
    }
    __syncthreads();
    float *pb = partial + (int64_t)blockIdx.x * E * g.co;
    for (int i = tid; i < E * g.co; i += CONV_T) {
        const int e = i / g.co, q = i % g.co;
        float v = 0.f;
        if (e < KK) {
            for (int r = 0; r < PG; r++) v = r == 0 ? slot[((size_t)r * EE + e) * CO + q] : v + slot[((size_t)r * EE + e) * CO + q];
        } else {
            for (int r = 0; r < nbias; r++) v = r == 0 ? bslot[r * CO + q] : v + bslot[r * CO + q];
        }
        pb[i] = v;
    }
}

inline int co_pad(int co) { return co <= 8 ? 8 : co <= 16 ? 16 : 32; }

cudaError_t set_smem(const void *fn, size_t smem) {
    if (smem > 48 * 1024) return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return cudaSuccess;
}

template <int CO>
cudaError_t launch_fwd(unsigned grid, int threads, size_t smem, cudaStream_t s, const ConvGeom &g, int rows, int spc,
                       const float *X, RowSel xrow, const float *Wb, float *P, uint8_t *arg) {
    cudaError_t e = set_smem((const void *)conv_fwd_kernel<CO>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(conv_fwd_kernel<CO>, dim3(grid), dim3(threads), smem, s, g, rows, spc, X, xrow, Wb, P, arg);
}

template <int CO>
cudaError_t launch_bwd(unsigned grid, size_t smem, cudaStream_t s, const ConvGeom &g, int rows, int spc, const float *X,
                       RowSel xrow, const float *dP, const float *P, const uint8_t *arg, const float *Wb, float *dX,
                       float *partial) {
    cudaError_t e = set_smem((const void *)conv_bwd_kernel<CO>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(conv_bwd_kernel<CO>, dim3(grid), dim3(CONV_T), smem, s, g, rows, spc, X, xrow, dP, P, arg, Wb, dX,
                      partial);
}

}  // namespace

size_t conv_fwd_smem(const ConvGeom &g, int spc) {
    return sizeof(float) * ((size_t)(g.k * g.k * g.ci + 1) * co_pad(g.co) + (size_t)spc * g.hi * g.wi * g.ci);
}
size_t conv_bwd_smem(const ConvGeom &g) {
    const size_t in_pad = ((size_t)g.hi * g.wi * g.ci + 3) & ~(size_t)3;
    const size_t ppc_pad = ((size_t)g.hp * g.wp * g.co + 3) & ~(size_t)3;
    const size_t KK = (size_t)g.k * g.k * g.ci, EB = (KK + 1 + 3) / 4, CO = co_pad(g.co);
    return sizeof(float) * ((size_t)g.hc * g.wc * CO + KK * CO + 4 * EB * CO +
                            2 * (in_pad + 2 * ppc_pad + conv_arg_pitch(g) / 4)) +
           16;  // two mbarriers
}
bool conv_supported(const ConvGeom &g) {
    return g.co >= 1 && g.co <= 32 && g.ci >= 1 && g.ci <= CONV_CI_MAX && (g.k * g.k * g.ci + 1 + 3) / 4 <= CONV_T &&
           conv_fwd_smem(g, 1) <= CONV_SMEM_MAX && conv_bwd_smem(g) <= CONV_SMEM_MAX;
}

cudaError_t conv_fwd(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *Wb, float *P, uint8_t *arg,
                     cudaStream_t s, LaunchHook *h) {
    if (!conv_supported(g)) return cudaErrorInvalidValue;
    const int Pp = g.hp * g.wp;
    // samples per CTA: fill the block with pooled outputs, but keep >= 2 CTAs per SM of work
    int spc = std::max(1, std::min(CONV_T / Pp, (int)cdiv(rows, 2 * 148)));
    while (spc > 1 && conv_fwd_smem(g, spc) > CONV_SMEM_MAX) spc--;
    const int threads = std::min(CONV_T, (int)((spc * Pp + 31) / 32 * 32));
    const size_t smem = conv_fwd_smem(g, spc);
    const unsigned grid = cdiv(rows, spc);
    char name[96];
    snprintf(name, sizeof name, "conv_fwd[rows=%d,hi=%d,ci=%d,k=%d,co=%d,spc=%d]", rows, g.hi, g.ci, g.k, g.co, spc);
    if (h) h->before(name, s);
    cudaError_t e;
    switch (co_pad(g.co)) {
        case 8: e = launch_fwd<8>(grid, threads, smem, s, g, rows, spc, X, xrow, Wb, P, arg); break;
        case 16: e = launch_fwd<16>(grid, threads, smem, s, g, rows, spc, X, xrow, Wb, P, arg); break;
        default: e = launch_fwd<32>(grid, threads, smem, s, g, rows, spc, X, xrow, Wb, P, arg);
    }
    if (h) h->after(name, s);
    return e;
}

template <int CO, int EPT>
cudaError_t launch_wgrad(unsigned grid, size_t smem, cudaStream_t s, const ConvGeom &g, int rows, int spc, const float *X,
                         RowSel xrow, const float *dP, const float *P, const uint8_t *arg, float *partial) {
    cudaError_t e = set_smem((const void *)conv_wgrad_kernel<CO, EPT>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(conv_wgrad_kernel<CO, EPT>, dim3(grid), dim3(CONV_T), smem, s, g, rows, spc, X, xrow, dP, P, arg,
                      partial);
}

// patch elements per thread: CO * EPT register accumulators (development knob MTX_CONV_EPT = 4 / 8 for CO <= 8)
int wgrad_ept(const ConvGeom &g) {
    static const int env = getenv("MTX_CONV_EPT") ? atoi(getenv("MTX_CONV_EPT")) : 0;
    if (co_pad(g.co) != 8) return 4;
    return env == 4 || env == 8 ? env : 8;
}

size_t conv_wgrad_smem(const ConvGeom &g) {
    const size_t in_pad = ((size_t)g.hi * g.wi * g.ci + 3) & ~(size_t)3;
    const size_t ppc_pad = ((size_t)g.hp * g.wp * g.co + 3) & ~(size_t)3;
    const size_t KK = (size_t)g.k * g.k * g.ci, E = KK + 1, CO = co_pad(g.co);
    const size_t layout = sizeof(float) * ((size_t)g.hc * g.wc * CO + E * CO + 2 * (in_pad + 2 * ppc_pad + conv_arg_pitch(g) / 4)) + 16;
    // the end-of-kernel reduction reuses the same memory: slot[PG][NEB * EPT][CO] + the bias threads' [nbias][CO]
    const size_t EPT = (size_t)wgrad_ept(g), NEB = (KK + EPT - 1) / EPT;
    const size_t PG = CONV_T / NEB - (CONV_T % NEB == 0 ? 1 : 0), nbias = CONV_T - NEB * PG;
    const size_t red = sizeof(float) * (PG * NEB * EPT + nbias) * CO;
    return std::max(layout, red);
}

cudaError_t conv_bwd(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *dP, const float *P,
                     const uint8_t *arg, const float *Wb, float *dX, float *dWb, float *partial, int64_t partial_cap,
                     cudaStream_t s, LaunchHook *h) {
    if (!conv_supported(g)) return cudaErrorInvalidValue;
    // weight gradient alone: the register-blocked kernel (EPT patch elements x CO channels per thread), when its
    // pixel groups cover the block (NEB <= CONV_T / 2) and its shared memory fits
    static const bool wg_only = !getenv("MTX_CONV_WGRAD_V1") || !atoi(getenv("MTX_CONV_WGRAD_V1"));
    const int EPT = wgrad_ept(g);
    const int KK = g.k * g.k * g.ci;
    if (!dX && wg_only && co_pad(g.co) <= 16 && (KK + EPT - 1) / EPT <= CONV_T / 2 && conv_wgrad_smem(g) <= CONV_SMEM_MAX) {
        const int E = KK + 1;
        int ctas = std::min(rows, 2 * 148);  // two CTAs per SM, the samples split evenly over them
        while (ctas > 1 && (int64_t)ctas * E * g.co > partial_cap) ctas--;
        if ((int64_t)ctas * E * g.co > partial_cap) return cudaErrorInvalidValue;
        const int spc = (int)cdiv(rows, ctas);
        const size_t smem = conv_wgrad_smem(g);
        char name[112];
        snprintf(name, sizeof name, "conv_wgrad[rows=%d,hc=%d,E=%d,co=%d,ept=%d,ctas=%d]", rows, g.hc, E, g.co, EPT, ctas);
        if (h) h->before(name, s);
        cudaError_t e = co_pad(g.co) == 8
                            ? (EPT == 8 ? launch_wgrad<8, 8>(ctas, smem, s, g, rows, spc, X, xrow, dP, P, arg, partial)
                                        : launch_wgrad<8, 4>(ctas, smem, s, g, rows, spc, X, xrow, dP, P, arg, partial))
                            : launch_wgrad<16, 4>(ctas, smem, s, g, rows, spc, X, xrow, dP, P, arg, partial);
        if (h) h->after(name, s);
        if (e != cudaSuccess) return e;
        return fold_partials(partial, ctas, E * g.co, dWb, s, h);
    }
    const int E = g.k * g.k * g.ci + 1;
    int ctas = std::min(rows, 2 * 148);
    while (ctas > 1 && (int64_t)ctas * E * g.co > partial_cap) ctas--;
    if ((int64_t)ctas * E * g.co > partial_cap) return cudaErrorInvalidValue;
    const int spc = (int)cdiv(rows, ctas);
    ctas = (int)cdiv(rows, spc);
    const size_t smem = conv_bwd_smem(g);
    char name[112];
    snprintf(name, sizeof name, "conv_bwd[rows=%d,hc=%d,E=%d,co=%d,dgrad=%d,ctas=%d]", rows, g.hc, E, g.co, dX ? 1 : 0,
             ctas);
    if (h) h->before(name, s);
    cudaError_t e;
    switch (co_pad(g.co)) {
        case 8: e = launch_bwd<8>(ctas, smem, s, g, rows, spc, X, xrow, dP, P, arg, Wb, dX, partial); break;
        case 16: e = launch_bwd<16>(ctas, smem, s, g, rows, spc, X, xrow, dP, P, arg, Wb, dX, partial); break;
        default: e = launch_bwd<32>(ctas, smem, s, g, rows, spc, X, xrow, dP, P, arg, Wb, dX, partial);
    }
    if (h) h->after(name, s);
    if (e != cudaSuccess) return e;
    return fold_partials(partial, ctas, E * g.co, dWb, s, h);
}

}  // namespace mtx
