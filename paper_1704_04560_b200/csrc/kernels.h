// kernels.h -- launch interface of libmtx's sm_100a kernels (internal C++; the
// public boundary is include/mtx.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mtx {

enum Epi : int { EPI_STORE = 0, EPI_BIAS_RELU = 1, EPI_BIAS = 2, EPI_MASK = 3 };

// C[M,N] = op(A)[M,K] . op(B)[K,N] (+ epilogue), fp32.
//   ta == false: A stored [M][lda] (element (m,k) at A[m*lda+k]);  true: A stored [K][lda], (m,k) at A[k*lda+m].
//   tb == false: B stored [K][ldb];                                 true: B stored [N][ldb], (k,n) at B[n*ldb+k].
//   aug: row m == M-1 of op(A) is all ones (the bias row of an augmented wgrad: db = colsum(dZ)).
//   arow: A's sample dimension (m if !ta, k if ta) starts at arow.row0().
//   splits > 1: deterministic split-K -- partial[z][M][N] then an ordered sum into C.
struct GemmDesc {
    int M = 0, N = 0, K = 0;
    bool ta = false, tb = false, aug = false;
    bool colsum_external = false;  // aug on the tensor-core engine: the caller launches the bias column sum
    int sm_budget = 0;             // > 0: plan and launch for at most this many SMs (concurrent side work)
    int epi = EPI_STORE;
    const float *A = nullptr;
    int64_t lda = 0;
    RowSel arow{nullptr, 0};
    const float *B = nullptr;
    int64_t ldb = 0;
    float *C = nullptr;
    int64_t ldc = 0;
    const float *bias = nullptr;
    const float *mask = nullptr;
    int64_t ldm = 0;
    int splits = 1;
    float *partial = nullptr;
    int64_t partial_cap = 0;  // floats available at partial (engines may choose their own split count)
    int64_t a_rows_total = 0; // rows of the buffer behind A when arow.win is set (wrap-extended dataset)
    int tf32x3 = 0;           // tensor-core engine: 3xTF32 (fp32-accurate) instead of 1xTF32
    // 3xTF32 operand planes (same layout as A / B; hi = rne_tf32(x), lo = rne_tf32(x - hi)) and
    // optional planes of the output for the next 3xTF32 consumer
    const float *A_hi = nullptr, *A_lo = nullptr, *B_hi = nullptr, *B_lo = nullptr;
    float *C_hi = nullptr, *C_lo = nullptr;
    unsigned *counters = nullptr;  // tensor-core split-K fixup: >= 256 per-tile counters, zeroed
    // 3xF16 (f16x3): fp16 operand planes (row pitch *_pld elements, a multiple of 8), their per-tensor
    // scale slots, and optionally the output's planes + slot; the output's scale is set from the bound
    // bnd_k * amax(A) * amax(B) (+ amax(B) when bnd_bias: the bias lives in the same parameter buffer)
    int f16x3 = 0;
    const __half *A_h = nullptr, *A_l = nullptr, *B_h = nullptr, *B_l = nullptr;
    int64_t lda_p = 0, ldb_p = 0;
    const TScale *tsA = nullptr, *tsB = nullptr;
    __half *C_h = nullptr, *C_l = nullptr;
    int64_t ldc_p = 0;
    TScale *tsC = nullptr;
    float bnd_k = 0.f;
    int bnd_bias = 0;
    // 3xF16 lean outputs (direct epilogue only, tc_direct): skip the fp32 C; the forward's ReLU bitmask
    // [M][relu_bits_ld words] (bit n % 32 of word n / 32 = [C > 0]); the dgrad's per-32-row column sums
    // colpart[ceil(M/32)][N] (the bias gradient of the layer whose dZ this is, folded later).  Input side:
    // mask_bits replaces the fp32 mask of a dgrad.
    int skip_c32 = 0;
    uint32_t *relu_bits = nullptr;
    int64_t relu_bits_ld = 0;
    float *colpart = nullptr;
    const uint32_t *mask_bits = nullptr;
    int64_t mask_bits_ld = 0;
};

// Launch-site hook: the API layer brackets every launch with it (timing/counting).
struct LaunchHook {
    virtual void before(const char *name, cudaStream_t s) = 0;
    virtual void after(const char *name, cudaStream_t s) = 0;
    virtual ~LaunchHook() {}
};

cudaError_t gemm_simt(const GemmDesc &g, cudaStream_t s, LaunchHook *h);

// out[n] = sum_{k} X[k][n] for X [K][ld] (column sums, e.g. the bias gradient colsum(dZ)):
// fixed-order per-block sums into partial[z][N]; per 128-column group, the last block to finish
// (ticket[group], zero on entry and re-armed on exit) folds the group's partials with a fixed
// summation tree -- deterministic, one launch.  ticket points at COLSUM_MAX_GROUPS counters.
constexpr int COLSUM_MAX_GROUPS = 64;  // N <= 8192
cudaError_t colsum(const float *X, int K, int N, int64_t ld, float *out, float *partial, int64_t partial_cap,
                   unsigned *ticket, cudaStream_t s, LaunchHook *h);

// 3xF16 output planes of a producer kernel: scale from the bound k * amax(a) * amax(b) (+ amax(b) with a
// bias), amax of the written values accumulated into ts->amax.
struct F16Out {
    __half *h = nullptr, *l = nullptr;
    int64_t ld = 0;
    TScale *ts = nullptr;
    const TScale *a = nullptr, *b = nullptr;
    float k = 0.f;
    int bias = 0;
    // lean outputs (GemmDesc: skip_c32 / relu_bits / colpart); the head: colpart per CTA, skip_f32
    int skip_f32 = 0;
    uint32_t *bits = nullptr;
    int64_t bits_ld = 0;
    float *colpart = nullptr;
};
MTX_DEVI float f16out_scale(const F16Out &o) {
    const float bb = o.b ? o.b->amax : 1.f;
    return f16_scale_for(o.k * o.a->amax * bb + (o.bias ? bb : 0.f));
}

// C[m][n] = epi(sum_{z ascending} partial[z][m][n])  (deterministic split-K fold + GEMM epilogue)
cudaError_t splitk_reduce(const float *partial, int splits, int M, int N, float *C, int64_t ldc, cudaStream_t s,
                          LaunchHook *h, int epi = EPI_STORE, const float *bias = nullptr,
                          const float *mask = nullptr, int64_t ldm = 0, float *C_hi = nullptr,
                          float *C_lo = nullptr, F16Out fo = F16Out(), const uint32_t *mbits = nullptr,
                          int64_t mbits_ld = 0);

// hi/lo 3xTF32 planes of x[n] (n % 4 == 0, 16-B aligned; rows of x need not be contiguous: a
// [rows][cols] block with leading dimension ld)
cudaError_t split_planes(const float *x, int64_t rows, int64_t cols, int64_t ld, float *hi, float *lo, cudaStream_t s,
                         LaunchHook *h);

// 3xF16 planes of one tensor (common.cuh TScale): a [rows][cols] fp32 block (pitch ld) -> fp16 hi/lo
// planes (pitch pld, a multiple of 8; columns cols..pld-1 are left as they are).
struct QSeg {
    const float *x;
    int64_t rows, cols, ld;
    __half *hi, *lo;
    int64_t pld;
};
constexpr int QSEG_MAX = 8;
constexpr int QUANT_SCRATCH_FLOATS = 1024 + 4;  // per-CTA maxima + the grid barrier words
// One grid-synchronous launch: amax = max |x| over [amax_x, amax_x + amax_n) (every element of the
// tensor's storage, e.g. the whole flat parameter buffer incl. biases) or, if amax_x is null, over the
// segments; s = f16_scale_for(amax); ts->amax / ts->scale written; then the planes of every segment.
// zero_ts[0..n_zero): per-step slots whose amax is reset (their producers accumulate it next step).
// scratch: QUANT_SCRATCH_FLOATS floats, zero on first use, private to one stream.
// pre_parts > 0: pre[0, pre_parts) already holds per-CTA maxima from the producing launch(es) (avg_update's
// amax_part, the fused update's per-rank arrays): no max pass and no grid barrier.
cudaError_t quantize_f16(const QSeg *segs, int nseg, const float *amax_x, int64_t amax_n, TScale *ts, TScale *zero_ts,
                         int n_zero, float *scratch, cudaStream_t s, LaunchHook *h, int pre_parts = 0,
                         const float *pre = nullptr);

// Narrow weight gradient (N <= 16, e.g. the classifier layer): dWb[k][j] = sum_i A[i][k] dZ[i][j]
// for k < K_in, plus (aug) the bias row dWb[K_in][j] = sum_i dZ[i][j].  Thread per k, rows split
// over blocks, blocked fp32 sums, ascending fold.  A's row offset: arow (dataset operand).
// out[j] = sum_{p ascending per lane, fixed shuffle tree} partial[p][j], j < n: deterministic fold of
// per-block partials (one warp per output).
// out[j] = sum_p partial[p][j] for j < n (partial pitch n): 32 columns x 8 part-slices per CTA, each slice
// summed in ascending p, the slices in a fixed tree (deterministic); coalesced over j.  The bias gradient
// from the 3xF16 lean column partials.
cudaError_t colpart_fold(const float *partial, int parts, int n, float *out, cudaStream_t s, LaunchHook *h);
cudaError_t fold_partials(const float *partial, int parts, int n, float *out, cudaStream_t s, LaunchHook *h);
cudaError_t wgrad_narrow(const float *A, int64_t lda, RowSel arow, const float *dZ, int rows, int K_in, int N,
                         float *dWb, float *partial, int64_t partial_cap, unsigned *ticket, cudaStream_t s,
                         LaunchHook *h);

// Fused last layer: logits = A W + b (W,b = augmented [(d+1)][C] block), mean
// softmax-CE, dZ_L = (softmax - onehot)/b, loss per row, (if dprev) the masked
// dgrad dZ_{L-1} = (dZ_L W^T) .* [A > 0], and the local loss sum into *loss_out
// (per-block partials folded in block order by the last block; ticket must be 0
// on entry and is re-armed on exit; loss_part holds >= 1024 floats).  dp_hi/dp_lo
// (nullable): 3xTF32 planes of dprev for the consuming tensor-core GEMMs.
// fo (3xF16): fp16 planes of dprev, scale from the bound |dprev| <= 2 inv_b max|W_L| (fo.k = 2 inv_b, fo.a =
// the parameters' slot, fo.b = null): sum_j |softmax_j - onehot_j| <= 2.  fo.colpart: per-CTA column sums
// of dprev [*colpart_rows][d] (the bias gradient of layer L-1); fo.skip_f32: dprev's fp32 copy not written.
cudaError_t head_fused(int rows, int d, int C, const float *A, RowSel arow, const float *Wb, const int32_t *labels,
                       RowSel lrow, float inv_b, float *dZL, float *dprev, float *dp_hi, float *dp_lo,
                       float *loss_rows, float *loss_part, unsigned *ticket, float *loss_out, cudaStream_t s,
                       LaunchHook *h, F16Out fo = F16Out(), int *colpart_rows = nullptr);

// Forward of a layer with K <= 64 on the CUDA cores (kernels_smallk.cu): C = act(A W + b), fp32 FMA in ascending
// k, with the 3xF16 producer outputs of fo (planes + amax, ReLU bits, skip_f32).  A's rows start at arow.
bool fwd_smallk_supported(int M, int N, int K, int64_t ldc, int64_t pld);
cudaError_t fwd_smallk(int M, int N, int K, const float *A, int64_t lda, RowSel arow, const float *W, int64_t ldw,
                       const float *bias, bool relu, float *C, int64_t ldc, const F16Out &fo, cudaStream_t s,
                       LaunchHook *h);

// Weight gradient of a layer with K_in <= 32 input features (cfg4's first layer) on the CUDA cores:
// dW[k][n] = sum_i X[i][k] dZ[i][n] (rows of X from xrow), dZ fp32 or its 3xF16 planes (dzh/dzl, pitch lddz, slot
// dzs); per-CTA partials (<= partial_cap floats) folded in order into dW [K_in][N] (the bias row is separate).
bool wgrad_smallm_supported(int K_in, int N);
cudaError_t wgrad_smallm(int rows, int K_in, int N, const float *X, int64_t ldx, RowSel xrow, const float *dZ,
                         const __half *dzh, const __half *dzl, int64_t lddz, const TScale *dzs, float *dW, float *partial,
                         int64_t partial_cap, cudaStream_t s, LaunchHook *h);

// out = sum_{i ascending in a fixed tree} v[i] (one block; deterministic).
cudaError_t reduce_sum(const float *v, int n, float *out, cudaStream_t s, LaunchHook *h);

// K6: gbar = G * invP; v = fma(mu, v, gbar); w = fma(-lr, v, w) over n floats
// (n % 4 == 0, 16-byte aligned).  v == nullptr: mu must be 0 and w = fma(-lr, gbar, w).
// flag |= 1 on a non-finite gbar.  If win != nullptr, thread 0 advances the
// window start: *win = (*win + B) mod n_data.  whi / wlo (nullable): also write the 3xTF32 hi/lo
// planes of the updated w (rne_tf32 split, as split_planes).
// amax_part (nullable, >= 1024 floats): per-CTA max |w| of the updated weights, *nparts of them (3xF16: the
// next planes' scale without re-reading w for it).
cudaError_t avg_update(float *G, float *w, float *v, int64_t n, float invP, float lr, float mu, int *flag,
                       int64_t *win, int64_t B, int64_t n_data, cudaStream_t s, LaunchHook *h, float *whi = nullptr,
                       float *wlo = nullptr, float *amax_part = nullptr, int *nparts = nullptr);

// Ordered reduce (test mode): G[e] = ((g_0[e] + g_1[e]) + ...) + g_{P-1}[e], g_r at gathered + r*stride.
cudaError_t ordered_fold(const float *gathered, int P, int64_t stride, int64_t n, float *G, cudaStream_t s,
                         LaunchHook *h);

// Busy-waits ~ns nanoseconds on the GPU (timing pass: lets the host enqueue a whole step
// before the GPU starts, so event pairs bracket device time only).
cudaError_t gpu_spin(uint64_t ns, cudaStream_t s);
// An empty kernel bracketed like every other launch site: the timing graph's per-launch overhead.
cudaError_t empty_launch(cudaStream_t s, LaunchHook *h);

// O2 init of one weight tensor: w[e] = (2u - 1) * lim, u = (H(H(seed, 16+t), e) >> 40) * 2^-24.
cudaError_t init_glorot(float *w, int64_t n, uint64_t seed, int tensor_index, float lim, cudaStream_t s);

// Digest: out += sum_e H(bits(x_e), e + salt) (wrapping, order independent).
cudaError_t digest(const float *x, int64_t n, uint64_t salt, unsigned long long *out, cudaStream_t s);

// ---- CNN (LeNet-style) kernels, NHWC, one sample row per image.
struct ConvGeom {
    int hi, wi, ci;   // input
    int k, co;        // kernel, output channels
    int hc, wc;       // conv output (valid, stride 1)
    int hp, wp;       // pooled output (2x2 / 2, floor)
};
// Bytes per sample of the pooled-argmax array (16-B multiple: bulk-copyable per sample).
__host__ __device__ inline int conv_arg_pitch(const ConvGeom &g) { return (g.hp * g.wp * g.co + 15) & ~15; }
// Limits of the conv kernels (checked at mtx_init): ci <= 16, co <= 32, shared-memory staging fits.
constexpr size_t CONV_SMEM_MAX = 200 * 1024;
bool conv_supported(const ConvGeom &g);
size_t conv_fwd_smem(const ConvGeom &g, int spc);
size_t conv_bwd_smem(const ConvGeom &g);
// P = maxpool2x2(ReLU(conv(X) + b)) [rows][hp][wp][co] and the argmax (0..3, first maximum) per
// pooled element; the pre-pool activation is not stored (the backward's mask at the argmax is P > 0).
cudaError_t conv_fwd(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *Wb, float *P, uint8_t *arg,
                     cudaStream_t s, LaunchHook *h);
// Backward of one conv + ReLU + pool layer from dP (gradient of its pooled output):
//   dR = route(dP via arg) .* [P > 0]                                   (never materialised)
//   dWb[(k*k*ci)+1][co] = im2col(X)^T dR (+ bias row)  -- per-CTA partials (<= partial_cap floats),
//                                                         folded deterministically
//   dX[rows][hi][wi][ci] = full correlation of dR with W, if dX != nullptr (no mask: the previous
//                          layer's own backward applies its pool/ReLU routing)
cudaError_t conv_bwd(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *dP, const float *P,
                     const uint8_t *arg, const float *Wb, float *dX, float *dWb, float *partial, int64_t partial_cap,
                     cudaStream_t s, LaunchHook *h);

// Tensor-core (tcgen05, 3xTF32) convolutions, conv_tc.cu: the forward conv + bias + ReLU + pool (same outputs
// as conv_fwd, plus optional hi/lo planes of P for the consuming fc GEMM) and the input gradient dX of a conv
// layer from its pooled gradient (routing through the argmax, mask [P > 0]) -- conv_bwd's dX part.
bool conv_tc_supported(const ConvGeom &g, bool dgrad);
cudaError_t conv_fwd_tc(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *Wb, float *P, uint8_t *arg,
                        float *P_hi, float *P_lo, cudaStream_t s, LaunchHook *h);
cudaError_t conv_dgrad_tc(const ConvGeom &g, int rows, const float *dP, const float *P, const uint8_t *arg, const float *Wb,
                          float *dX, cudaStream_t s, LaunchHook *h);

}  // namespace mtx
