// kernels_conv.cu -- LeNet-style convolution layers of the local forward/backward
// (CNN rows; config 3).  NHWC activations, weights
// W[kh][kw][ci][co] followed by the bias row (the augmented block of the flat
// buffer).  Channel counts are small (C_out = 6, 16), so these are SIMT kernels:
// the fused forward computes conv + bias + ReLU + 2x2 max-pool (+ first-max argmax,
// reading A6) in one pass; the backward routes the pooled gradient through the
// argmax and the ReLU mask, and the weight gradient is a deterministic blocked
// reduction over (sample, position) folded in a fixed order.
#include <stdio.h>

#include <algorithm>

#include "kernels.h"

namespace mtx {
namespace {

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// One thread per pooled output (n, ph, pw, co): the 2x2 conv outputs of its window,
// bias, ReLU, then max with the first maximum in (dh, dw) order winning ties.
__global__ void __launch_bounds__(256) conv_fwd_kernel(ConvGeom g, int rows, const float *__restrict__ X, RowSel xrow,
                                                     const float *__restrict__ Wb, float *__restrict__ R,
                                                     float *__restrict__ P, uint8_t *__restrict__ arg) {
    pdl_wait();
    extern __shared__ float sw[];  // (k*k*ci + 1) * co
    const int KK = g.k * g.k * g.ci;
    for (int e = threadIdx.x; e < (KK + 1) * g.co; e += blockDim.x) sw[e] = Wb[e];
    __syncthreads();
    const int64_t total = (int64_t)rows * g.hp * g.wp * g.co;
    const int64_t in_sz = (int64_t)g.hi * g.wi * g.ci;
    const float *Xb = X + xrow.row0() * in_sz;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int co = (int)(idx % g.co);
        int64_t t = idx / g.co;
        const int pw = (int)(t % g.wp);
        t /= g.wp;
        const int ph = (int)(t % g.hp);
        const int64_t n = t / g.hp;
        const float *x = Xb + n * in_sz;
        float best = 0.f;
        int barg = 0;
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int oh = 2 * ph + (d >> 1), ow = 2 * pw + (d & 1);
            float acc = 0.f;
            for (int kh = 0; kh < g.k; kh++)
                for (int kw = 0; kw < g.k; kw++) {
                    const float *xp = x + ((int64_t)(oh + kh) * g.wi + (ow + kw)) * g.ci;
                    const float *wp = sw + ((kh * g.k + kw) * g.ci) * g.co + co;
                    for (int ci = 0; ci < g.ci; ci++) acc = __fmaf_rn(xp[ci], wp[ci * g.co], acc);
                }
            const float z = fmaxf(acc + sw[KK * g.co + co], 0.f);  // bias after the sum, ReLU
            R[((n * g.hc + oh) * g.wc + ow) * g.co + co] = z;
            if (d == 0 || z > best) {
                best = z;
                barg = d;
            }
        }
        P[idx] = best;
        arg[idx] = (uint8_t)barg;
    }
}

// dR = dP routed to its argmax, times the ReLU mask [R > 0]; positions outside every
// pooling window (odd edges) get 0.  One thread per conv output element.
__global__ void pool_relu_bwd_kernel(ConvGeom g, int rows, const float *__restrict__ dP,
                                     const uint8_t *__restrict__ arg, const float *__restrict__ R,
                                     float *__restrict__ dR) {
    pdl_wait();
    const int64_t total = (int64_t)rows * g.hc * g.wc * g.co;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int co = (int)(idx % g.co);
        int64_t t = idx / g.co;
        const int ow = (int)(t % g.wc);
        t /= g.wc;
        const int oh = (int)(t % g.hc);
        const int64_t n = t / g.hc;
        const int ph = oh >> 1, pw = ow >> 1;
        float v = 0.f;
        if (ph < g.hp && pw < g.wp) {
            const int64_t pidx = ((n * g.hp + ph) * g.wp + pw) * g.co + co;
            if (arg[pidx] == (uint8_t)(((oh & 1) << 1) | (ow & 1)) && R[idx] > 0.f) v = dP[pidx];
        }
        dR[idx] = v;
    }
}

// Weight gradient: dWb[e][co] = sum over (n, oh, ow) of patch(n, oh, ow)[e] * dR(n, oh, ow)[co],
// e < k*k*ci; row e == k*k*ci is the bias gradient sum dR.  Block z takes a contiguous range of
// output positions; per 32-position tile it stages the patches and dR rows in shared memory, then
// each thread accumulates its fixed (e, co) pairs in position order.  Partial per block; the
// caller folds partials in block order (deterministic).
constexpr int WG_T = 256, WG_POS = 32;
__global__ void __launch_bounds__(WG_T) conv_wgrad_kernel(ConvGeom g, int rows, const float *__restrict__ X,
                                                        RowSel xrow, const float *__restrict__ dR, int64_t pos_per,
                                                        float *__restrict__ partial) {
    pdl_wait();
    extern __shared__ float sm[];
    const int KK = g.k * g.k * g.ci, E = KK + 1;
    float *sp = sm;                 // [WG_POS][E]
    float *sd = sm + WG_POS * E;    // [WG_POS][co]
    const int pairs = E * g.co;
    constexpr int MAXP = 16;        // pairs per thread (E*co <= 16*256)
    float acc[MAXP];
#pragma unroll
    for (int i = 0; i < MAXP; i++) acc[i] = 0.f;
    const int64_t npos = (int64_t)rows * g.hc * g.wc;
    const int64_t p0 = blockIdx.x * pos_per, p1 = min(npos, p0 + pos_per);
    const int64_t in_sz = (int64_t)g.hi * g.wi * g.ci;
    const float *Xb = X + xrow.row0() * in_sz;
    for (int64_t pt = p0; pt < p1; pt += WG_POS) {
        const int np = (int)(p1 - pt < WG_POS ? p1 - pt : WG_POS);
        for (int e = threadIdx.x; e < WG_POS * E; e += WG_T) {
            const int pl = e / E, el = e % E;
            float v = 0.f;
            if (pl < np) {
                const int64_t p = pt + pl;
                const int ow = (int)(p % g.wc);
                const int64_t t = p / g.wc;
                const int oh = (int)(t % g.hc);
                const int64_t n = t / g.hc;
                if (el == KK) {
                    v = 1.f;
                } else {
                    const int ci = el % g.ci, kw = (el / g.ci) % g.k, kh = el / (g.ci * g.k);
                    v = Xb[n * in_sz + ((int64_t)(oh + kh) * g.wi + (ow + kw)) * g.ci + ci];
                }
            }
            sp[e] = v;
        }
        for (int e = threadIdx.x; e < WG_POS * g.co; e += WG_T) {
            const int pl = e / g.co;
            sd[e] = pl < np ? dR[(pt + pl) * g.co + e % g.co] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < MAXP; i++) {
            const int pr = threadIdx.x + i * WG_T;
            if (pr < pairs) {
                const int el = pr / g.co, co = pr % g.co;
                float tsum = 0.f;  // blocked summation: a 32-term chain per tile, then one add
                for (int pl = 0; pl < np; pl++) tsum = __fmaf_rn(sp[pl * E + el], sd[pl * g.co + co], tsum);
                acc[i] = __fadd_rn(acc[i], tsum);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < MAXP; i++) {
        const int pr = threadIdx.x + i * WG_T;
        if (pr < pairs) partial[(int64_t)blockIdx.x * pairs + pr] = acc[i];
    }
}

// Input gradient (full correlation): dX[n][h][w][ci] = sum_{kh,kw,co} dR[n][h-kh][w-kw][co] W[kh][kw][ci][co].
__global__ void __launch_bounds__(256) conv_dgrad_kernel(ConvGeom g, int rows, const float *__restrict__ dR,
                                                       const float *__restrict__ Wb, float *__restrict__ dX) {
    pdl_wait();
    extern __shared__ float sw[];
    const int KK = g.k * g.k * g.ci;
    for (int e = threadIdx.x; e < KK * g.co; e += blockDim.x) sw[e] = Wb[e];
    __syncthreads();
    const int64_t total = (int64_t)rows * g.hi * g.wi * g.ci;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int ci = (int)(idx % g.ci);
        int64_t t = idx / g.ci;
        const int w = (int)(t % g.wi);
        t /= g.wi;
        const int h = (int)(t % g.hi);
        const int64_t n = t / g.hi;
        float acc = 0.f;
        for (int kh = 0; kh < g.k; kh++) {
            const int oh = h - kh;
            if (oh < 0 || oh >= g.hc) continue;
            for (int kw = 0; kw < g.k; kw++) {
                const int ow = w - kw;
                if (ow < 0 || ow >= g.wc) continue;
                const float *d = dR + ((n * g.hc + oh) * g.wc + ow) * g.co;
                const float *wp = sw + ((kh * g.k + kw) * g.ci + ci) * g.co;
                for (int co = 0; co < g.co; co++) acc = __fmaf_rn(d[co], wp[co], acc);
            }
        }
        dX[idx] = acc;
    }
}

}  // namespace

cudaError_t conv_fwd(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *Wb, float *R, float *P,
                     uint8_t *arg, cudaStream_t s, LaunchHook *h) {
    const size_t smem = sizeof(float) * (size_t)(g.k * g.k * g.ci + 1) * g.co;
    const int64_t total = (int64_t)rows * g.hp * g.wp * g.co;
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 16));
    char name[96];
    snprintf(name, sizeof name, "conv_fwd[rows=%d,hi=%d,ci=%d,k=%d,co=%d]", rows, g.hi, g.ci, g.k, g.co);
    if (h) h->before(name, s);
    launch_pdl(conv_fwd_kernel, dim3(blocks), dim3(256), smem, s, g, rows, X, xrow, Wb, R, P, arg);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

cudaError_t pool_relu_bwd(const ConvGeom &g, int rows, const float *dP, const uint8_t *arg, const float *R, float *dR,
                          cudaStream_t s, LaunchHook *h) {
    const int64_t total = (int64_t)rows * g.hc * g.wc * g.co;
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 16));
    char name[80];
    snprintf(name, sizeof name, "pool_relu_bwd[n=%lld]", (long long)total);
    if (h) h->before(name, s);
    launch_pdl(pool_relu_bwd_kernel, dim3(blocks), dim3(256), 0, s, g, rows, dP, arg, R, dR);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

cudaError_t conv_wgrad(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *dR, float *dWb,
                       float *partial, int splits, cudaStream_t s, LaunchHook *h) {
    const int E = g.k * g.k * g.ci + 1;
    if (E * g.co > 16 * WG_T) return cudaErrorInvalidValue;
    const int64_t npos = (int64_t)rows * g.hc * g.wc;
    const int64_t pos_per = (npos + splits - 1) / splits;
    splits = (int)((npos + pos_per - 1) / pos_per);
    const size_t smem = sizeof(float) * (size_t)WG_POS * (E + g.co);
    char name[96];
    snprintf(name, sizeof name, "conv_wgrad[pos=%lld,E=%d,co=%d,splits=%d]", (long long)npos, E, g.co, splits);
    if (h) h->before(name, s);
    launch_pdl(conv_wgrad_kernel, dim3(splits), dim3(WG_T), smem, s, g, rows, X, xrow, dR, pos_per, partial);
    if (h) h->after(name, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return splitk_reduce(partial, splits, E, g.co, dWb, g.co, s, h);
}

cudaError_t conv_dgrad(const ConvGeom &g, int rows, const float *dR, const float *Wb, float *dX, cudaStream_t s,
                       LaunchHook *h) {
    const size_t smem = sizeof(float) * (size_t)g.k * g.k * g.ci * g.co;
    const int64_t total = (int64_t)rows * g.hi * g.wi * g.ci;
    unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 16));
    char name[80];
    snprintf(name, sizeof name, "conv_dgrad[n=%lld,k=%d,co=%d]", (long long)total, g.k, g.co);
    if (h) h->before(name, s);
    launch_pdl(conv_dgrad_kernel, dim3(blocks), dim3(256), smem, s, g, rows, dR, Wb, dX);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

}  // namespace mtx
