// kernels_smallk.cu -- the forward of a layer with a short contraction (K <= 64, e.g. the 28 HIGGS features
// of cfg4's first layer, "forward ... on its local minibatch") on the CUDA cores, with the
// 3xF16 producer epilogue.
//
// A tensor-core tile of this GEMM is one k-block: the MMA is a few hundred cycles and the tile is all epilogue,
// which on the tcgen05 engine is 8 warps per SM walking 7 tiles in sequence (measured 27-35 us for 8192 x 1024 x
// 28).  Here every SM holds up to 4 CTAs of 8 warps and the epilogue is spread over all of them; the products are
// fp32 FMAs in ascending k (a K-term chain: the fp32 tier), ~6 us of FMA issue at this shape.
#include <stdio.h>

#include <algorithm>

#include "kernels.h"

namespace mtx {
namespace {

constexpr int SK_M = 128, SK_N = 128, SK_T = 256;

// C[m][n] = act(sum_k A[m][k] W[k][n] + b[n]) for a 128 x 128 tile; thread (tx, ty) owns rows 8 ty .. 8 ty + 7 and
// columns 8 tx .. 8 tx + 7.  Outputs: fp32 C (unless fo.skip_f32), fp16 planes + amax (fo.h), ReLU bits (fo.bits).
// KP: K rounded up (16 / 32 / 64; the k loop is unrolled, A is staged transposed so a thread's 8 rows are two
// 128-bit shared loads, zero rows past K add nothing).
// KL: k-loop trip count (KP, or K itself when it is a multiple of 4 below KP: cfg4's 28 features skip 4 zero rows).
// LEAN: the 3xF16 lean forward (bias + ReLU, planes + bits, no fp32 copy, N % 128 == 0): the other output paths and
// the column-edge tests are compiled out.
template <int KP, int KL = KP, bool LEAN = false>
__global__ void __launch_bounds__(SK_T, 2) fwd_smallk_kernel(int M, int N, int K, const float *__restrict__ A, int64_t lda,
                                                           RowSel arow, const float *__restrict__ W, int64_t ldw,
                                                           const float *__restrict__ bias, int relu, float *__restrict__ C,
                                                           int64_t ldc, F16Out fo) {
    pdl_wait();
    extern __shared__ __align__(16) float sk_smem[];
    float *As = sk_smem, *Ws = sk_smem + KP * SK_M;  // As[KP][128] (transposed), Ws[KP][128]
    const int m0 = blockIdx.y * SK_M, n0 = blockIdx.x * SK_N;
    const float *Ab = A + (arow.row0() + m0) * lda;
    // A tile transposed through registers: thread (r, half) reads its row's KP/2 features (128-bit loads when the
    // rows allow) and stores them down column r -- consecutive threads, consecutive words: no bank conflicts
    {
        constexpr int KH = KP / 2;
        const int r = threadIdx.x & (SK_M - 1), k0 = (threadIdx.x >> 7) * KH;
        const float *ar = Ab + (int64_t)r * lda;
        const bool row_ok = m0 + r < M;
        float v[KH];
        if (row_ok && lda % 4 == 0 && k0 + KH <= K) {
#pragma unroll
            for (int u = 0; u < KH / 4; u++) {
                const float4 x = __ldg((const float4 *)(ar + k0) + u);
                v[4 * u] = x.x; v[4 * u + 1] = x.y; v[4 * u + 2] = x.z; v[4 * u + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int u = 0; u < KH; u++) v[u] = (row_ok && k0 + u < K) ? __ldg(ar + k0 + u) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < KH; u++) As[(k0 + u) * SK_M + r] = v[u];
    }
    {  // W tile: all of a thread's loads in flight before its stores (a load-store loop waits out L2 latency per item)
        constexpr int PER = KP * SK_N / SK_T;
        float wv[PER];
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int e = threadIdx.x + u * SK_T, k = e / SK_N, c = e % SK_N;
            wv[u] = (k < K && n0 + c < N) ? __ldg(W + (int64_t)k * ldw + n0 + c) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < PER; u++) Ws[threadIdx.x + u * SK_T] = wv[u];
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
    // unrolled by 8, not fully: the fully unrolled body missed in the instruction cache (ncu: 18 % of the warp
    // samples stalled on no instruction)
#pragma unroll 8
    for (int k = 0; k < KL; k++) {
        const float4 a0 = *(const float4 *)(As + k * SK_M + 8 * ty), a1 = *(const float4 *)(As + k * SK_M + 8 * ty + 4);
        const float4 b0 = *(const float4 *)(Ws + k * SK_N + 8 * tx), b1 = *(const float4 *)(Ws + k * SK_N + 8 * tx + 4);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; i++)
#pragma unroll
            for (int j = 0; j < 8; j++) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
    }
    const int nb = n0 + 8 * tx;
    float bz[8];
#pragma unroll
    for (int j = 0; j < 8; j++) bz[j] = LEAN ? __ldg(bias + nb + j) : (bias && nb + j < N) ? __ldg(bias + nb + j) : 0.f;
    const bool planes = LEAN || fo.h;
    const float inv_so = planes ? 1.f / f16out_scale(fo) : 1.f;
    if (planes && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) fo.ts->scale = 1.f / inv_so;
    float amx = 0.f;
    const bool full = LEAN || nb + 7 < N;
#pragma unroll  // fully: acc[i][.] must stay in registers
    for (int i = 0; i < 8; i++) {
        const int m = m0 + 8 * ty + i;
        float o[8];
        uint32_t bits = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            o[j] = acc[i][j] + bz[j];
            if (LEAN || relu) o[j] = fmaxf(o[j], 0.f);
            if (!LEAN && nb + j >= N) o[j] = 0.f;
            bits |= (o[j] > 0.f ? 1u : 0u) << j;
            amx = fmaxf(amx, fabsf(o[j]));
        }
        // the 4 threads of a 32-column group (consecutive tx) OR their bytes into the row's mask word
        uint32_t w = bits << (8 * (tx & 3));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        if (m >= M || (!LEAN && nb >= N)) continue;
        if ((LEAN || fo.bits) && (tx & 3) == 0) fo.bits[(int64_t)m * fo.bits_ld + (nb >> 5)] = w;
        if (!LEAN && C && !fo.skip_f32) {
            if (full) {
                *(float4 *)(C + (int64_t)m * ldc + nb) = make_float4(o[0], o[1], o[2], o[3]);
                *(float4 *)(C + (int64_t)m * ldc + nb + 4) = make_float4(o[4], o[5], o[6], o[7]);
            } else {
                for (int j = 0; j < 8 && nb + j < N; j++) C[(int64_t)m * ldc + nb + j] = o[j];
            }
        }
        if (planes) {
            uint32_t hp[4], lp[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const float2 y = make_float2(o[2 * e] * inv_so, o[2 * e + 1] * inv_so);
                const __half2 h2 = __float22half2_rn(y);
                const float2 hf = __half22float2(h2);
                const __half2 l2 = __float22half2_rn(make_float2(y.x - hf.x, y.y - hf.y));
                hp[e] = *(const uint32_t *)&h2;
                lp[e] = *(const uint32_t *)&l2;
            }
            const int64_t po = (int64_t)m * fo.ld + nb;
            if (full) {
                *(uint4 *)(fo.h + po) = make_uint4(hp[0], hp[1], hp[2], hp[3]);
                *(uint4 *)(fo.l + po) = make_uint4(lp[0], lp[1], lp[2], lp[3]);
            } else {
                for (int j = 0; j < 8 && nb + j < N; j++) {
                    fo.h[po + j] = __ushort_as_half((uint16_t)(hp[j / 2] >> (16 * (j & 1))));
                    fo.l[po + j] = __ushort_as_half((uint16_t)(lp[j / 2] >> (16 * (j & 1))));
                }
            }
        }
    }
    if (planes) {  // one atomic per CTA (thousands of warps on one address would serialise)
        __shared__ float red[SK_T / 32];
        for (int off = 16; off > 0; off >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, off));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amx;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < SK_T / 32; w++) amx = fmaxf(amx, red[w]);
            amax_atomic(&fo.ts->amax, amx);
        }
    }
}

}  // namespace

bool fwd_smallk_supported(int M, int N, int K, int64_t ldc, int64_t pld) {
    return K >= 1 && K <= 64 && M >= 1 && N >= 1 && ldc % 4 == 0 && pld % 8 == 0;
}

cudaError_t fwd_smallk(int M, int N, int K, const float *A, int64_t lda, RowSel arow, const float *W, int64_t ldw,
                       const float *bias, bool relu, float *C, int64_t ldc, const F16Out &fo, cudaStream_t s,
                       LaunchHook *h) {
    const int KP = K <= 16 ? 16 : K <= 32 ? 32 : 64;
    const size_t smem = sizeof(float) * (size_t)KP * (SK_M + SK_N);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(fwd_smallk_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(fwd_smallk_kernel<64, 64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    char name[80];
    snprintf(name, sizeof name, "fwd_smallk[M=%d,N=%d,K=%d]", M, N, K);
    if (h) h->before(name, s);
    const dim3 grid((N + SK_N - 1) / SK_N, (M + SK_M - 1) / SK_M);
    const bool lean = fo.h && fo.skip_f32 && fo.bits && bias && relu && N % SK_N == 0 && fo.ld % 8 == 0;
    auto kern = KP == 16 ? (lean ? fwd_smallk_kernel<16, 16, true> : fwd_smallk_kernel<16>)
              : K == 28  ? (lean ? fwd_smallk_kernel<32, 28, true> : fwd_smallk_kernel<32, 28>)
              : KP == 32 ? (lean ? fwd_smallk_kernel<32, 32, true> : fwd_smallk_kernel<32>)
                         : (lean ? fwd_smallk_kernel<64, 64, true> : fwd_smallk_kernel<64>);
    launch_pdl(kern, grid, dim3(SK_T), smem, s, M, N, K, A, lda, arow, W, ldw, bias, relu ? 1 : 0, C, ldc, fo);
    if (h) h->after(name, s);
    return cudaGetLastError();
}

}  // namespace mtx

// ------------------------------------------------------------------ weight gradient of a short-K_in layer
// dW[k][n] = sum_i X[i][k] dZ[i][n] for k < K_in <= 32 (cfg4's first layer: 28 features, K = b samples): the
// tensor-core tile would be 28 useful rows of 128.  CUDA cores: a CTA owns 128 columns and a contiguous row range;
// 32-row chunks of dZ (fp32, or rebuilt exactly from its 3xF16 planes: s * (hi + lo) is exact in fp32) and of X are
// staged in shared memory; thread (cg, kg) accumulates k = 4 kg .. 4 kg + 3 x n = 4 cg .. 4 cg + 3 over the rows in
// ascending order.  Per-CTA partials [split][K_in * N], folded in split order (colpart_fold): deterministic.
namespace mtx {
namespace {
constexpr int WS_N = 128, WS_R = 32, WS_T = 256;

__global__ void __launch_bounds__(WS_T) wgrad_smallm_kernel(int rows, int K_in, int N, const float *__restrict__ X,
                                                           int64_t ldx, RowSel xrow, const float *__restrict__ dZ,
                                                           const __half *__restrict__ dzh, const __half *__restrict__ dzl,
                                                           int64_t lddz, const TScale *dzs, int rows_per,
                                                           float *__restrict__ partial) {
    pdl_wait();
    __shared__ __align__(16) float sz[WS_R][WS_N];
    __shared__ __align__(16) float sx[WS_R][33];
    const int n0 = blockIdx.x * WS_N, r0 = blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
    const int cg = threadIdx.x & 31, kg = threadIdx.x >> 5;  // 32 column groups x 8 k groups
    const float s = dzh ? dzs->scale : 1.f;
    const float *Xb = X + xrow.row0() * ldx;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0.f;
    for (int i0 = r0; i0 < r1; i0 += WS_R) {
        const int nr = min(WS_R, r1 - i0);
        // stage dZ rows (4 columns per thread-iteration) and X rows (unrolled: all of a thread's loads in flight)
#pragma unroll
        for (int e = threadIdx.x; e < WS_R * (WS_N / 4); e += WS_T) {
            const int r = e / (WS_N / 4), c4 = 4 * (e % (WS_N / 4)), n = n0 + c4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r < nr && n + 3 < N) {
                const int64_t off = (int64_t)(i0 + r) * lddz + n;
                if (dzh) {
                    const uint2 h = __ldg((const uint2 *)(dzh + off)), l = __ldg((const uint2 *)(dzl + off));
                    const float2 h0 = __half22float2(*(const __half2 *)&h.x), h1 = __half22float2(*(const __half2 *)&h.y);
                    const float2 l0 = __half22float2(*(const __half2 *)&l.x), l1 = __half22float2(*(const __half2 *)&l.y);
                    v = make_float4((h0.x + l0.x) * s, (h0.y + l0.y) * s, (h1.x + l1.x) * s, (h1.y + l1.y) * s);
                } else {
                    v = __ldg((const float4 *)(dZ + off));
                }
            } else if (r < nr) {
                float t[4];
                for (int u = 0; u < 4; u++) {
                    t[u] = 0.f;
                    if (n + u < N) {
                        const int64_t off = (int64_t)(i0 + r) * lddz + n + u;
                        t[u] = dzh ? (__half2float(dzh[off]) + __half2float(dzl[off])) * s : dZ[off];
                    }
                }
                v = make_float4(t[0], t[1], t[2], t[3]);
            }
            *(float4 *)&sz[r][c4] = v;
        }
#pragma unroll
        for (int e = threadIdx.x; e < WS_R * 32; e += WS_T) {
            const int r = e >> 5, k = e & 31;
            sx[r][k] = (r < nr && k < K_in) ? __ldg(Xb + (int64_t)(i0 + r) * ldx + k) : 0.f;
        }
        __syncthreads();
        for (int r = 0; r < nr; r++) {
            const float4 z = *(const float4 *)&sz[r][4 * cg];
            const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
            for (int a = 0; a < 4; a++) {
                const float x = sx[r][4 * kg + a];
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] = __fmaf_rn(x, zz[b], acc[a][b]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int k = 4 * kg + a;
        if (k >= K_in) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int n = n0 + 4 * cg + b;
            if (n < N) partial[(int64_t)blockIdx.y * K_in * N + (int64_t)k * N + n] = acc[a][b];
        }
    }
}
}  // namespace

bool wgrad_smallm_supported(int K_in, int N) { return K_in >= 1 && K_in <= 32 && N >= 1; }

cudaError_t wgrad_smallm(int rows, int K_in, int N, const float *X, int64_t ldx, RowSel xrow, const float *dZ,
                         const __half *dzh, const __half *dzl, int64_t lddz, const TScale *dzs, float *dW, float *partial,
                         int64_t partial_cap, cudaStream_t s, LaunchHook *h) {
    const int nb = (N + WS_N - 1) / WS_N;
    int splits = std::max(1, std::min((3 * 148 + nb - 1) / nb, (rows + WS_R - 1) / WS_R));
    while (splits > 1 && (int64_t)splits * K_in * N > partial_cap) splits--;
    int rows_per = (rows + splits - 1) / splits;
    rows_per = (rows_per + WS_R - 1) / WS_R * WS_R;
    splits = (rows + rows_per - 1) / rows_per;
    char name[80];
    snprintf(name, sizeof name, "wgrad_smallm[M=%d,N=%d,K=%d,splits=%d]", K_in, N, rows, splits);
    if (h) h->before(name, s);
    launch_pdl(wgrad_smallm_kernel, dim3(nb, splits), dim3(WS_T), 0, s, rows, K_in, N, X, ldx, xrow, dZ, dzh, dzl, lddz,
               dzs, rows_per, partial);
    if (h) h->after(name, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return colpart_fold(partial, splits, K_in * N, dW, s, h);
}

}  // namespace mtx
