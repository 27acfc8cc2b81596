// conv_tc.cu -- LeNet convolutions on the 5th-gen tensor cores (CNN rows; config 3):
// the forward conv (+ bias + ReLU + 2x2 max-pool, first maximum wins ties, reading A6) and the input
// gradient of a conv layer, as implicit GEMMs on tcgen05.mma kind::tf32 in 3xTF32 (fp32-accurate,
// DESIGN.md §3), accumulators in TMEM.
//
// Why "kw in N".  A 1-CTA MMA with fresh operand tiles costs ~89 cycles whatever its N <= 128
// (profiles/round2_tcgen05_rates.md), so a conv must make every MMA wide.  The textbook implicit GEMM
// (M = pixels, N = C_out = 6/16, K = k*k*C_in) would spend 89 cycles on 16 columns.  Here the filter column
// kw moves from K into N: for a tile of "virtual pixels" p = (oh, ow) over the FULL input width Wi,
//     Y'[p][kw*CO + co] = sum_{kh, ci} X[oh + kh][ow][ci] * W[kh][kw][ci][co]     (K = k*Ci: 15 / 30)
//     Z[oh][ow][co]     = sum_kw Y'[(oh, ow + kw)][kw*CO + co]                    (ow + kw < Wi: same row)
// N = k*CO (32 / 80), K = k*Ci padded to 8: 2 (conv1) / 4 (conv2) k-steps x 3 MMAs per 128 pixels instead of
// 10 / 19.  The input gradient moves both filter offsets into N (its K, the output channels, is 16):
//     Y'[(oh, ow)][(kh*k + kw)*Ci + ci] = sum_co dR[oh][ow][co] * W[kh][kw][ci][co]     (N = k*k*Ci = 150 -> 160)
//     dX[h][w][ci]                      = sum_{kh, kw} Y'[(h - kh, w - kw)][(kh*k + kw)*Ci + ci]
// where dR = dP routed to the pool argmax and masked by [P > 0] (max-pool + ReLU backward); one tile is one
// image's 10 x 10 conv outputs.
//
// Per CTA (persistent, 128 threads = 4 warps = the 4 TMEM lane quarters; 2-3 CTAs per SM so one CTA's
// MMAs overlap another's gather / epilogue): the B operand (weights, hi/lo planes) is built once in shared
// memory; per tile every thread gathers its own A row (one pixel), splits it into hi/lo TF32 planes and
// writes them in the UMMA K-major SWIZZLE_128B layout; one thread issues the MMAs; every thread reads its
// TMEM lane (tcgen05.ld) into a padded shared-memory row of Y', and the tile's outputs are formed from Y'
// (shift-sums, bias, ReLU, pool / the dX sum) and stored.  The geometry is compile-time (the two LeNet
// layers of config 3); other geometries, and the weight gradients, run on the CUDA cores (kernels_conv.cu):
// a weight gradient's M x N is 76 x 6 / 151 x 16 over b*784 / b*100 pixels of K, and an MMA advances K by
// only 8 per ~89 cycles.
#include <stdio.h>

#include <algorithm>

#include "kernels.h"

namespace mtx {
namespace {

constexpr int CT_THREADS = 256;  // 8 warps: two per TMEM lane quarter
constexpr int TILE_M = 128;

__device__ __forceinline__ uint64_t sdesc_k128(uint32_t addr) {  // K-major SWIZZLE_128B, 8-row groups at 1024 B
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)(16 >> 4) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// kind::tf32, D fp32, A/B tf32, both K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
            d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
#define CT_TMEM_LD16(taddr, r)                                                                                  \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),   \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
                 : "r"(taddr))

// Byte offset of element (row, k) of a K-major SWIZZLE_128B operand whose atoms (32 k per 128-B row) hold
// `rows` rows each: 16-B chunks XOR-swizzled by row % 8, 8-row groups 1024 B apart.
__device__ __forceinline__ uint32_t sw128_off(int row, int k, int rows) {
    return (uint32_t)(k >> 5) * (uint32_t)(rows * 128) + (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u +
           (uint32_t)((((k & 31) >> 2) ^ (row & 7)) << 4) + (uint32_t)(k & 3) * 4u;
}

struct ConvTcArgs {
    int rows;          // samples
    const float *X;    // FWD: input images [rows][hi][wi][ci] (row offset xrow)
    RowSel xrow;
    const float *Wb;   // W[kh][kw][ci][co] then the bias row
    float *P;          // FWD: pooled output [rows][hp][wp][co]
    uint8_t *arg;      // FWD out / DGRAD in: argmax per pooled element (pitch conv_arg_pitch)
    float *P_hi, *P_lo;  // FWD (nullable): 3xTF32 planes of P for the consuming fc GEMM
    const float *dP;   // DGRAD: gradient of the pooled output
    const float *Pin;  // DGRAD: the pooled output (ReLU mask [P > 0])
    float *dX;         // DGRAD: input gradient [rows][hi][wi][ci]
};

// Compile-time geometry of one conv layer (the instantiated LeNet layers; others run on kernels_conv.cu).
template <int HI_, int WI_, int CI_, int KS_, int CO_>
struct Geo {
    static constexpr int HI = HI_, WI = WI_, CI = CI_, KS = KS_, CO = CO_;
    static constexpr int HC = HI - KS + 1, WC = WI - KS + 1, HP = HC / 2, WP = WC / 2;
    static constexpr int IN_SZ = HI * WI * CI, PPC = HP * WP * CO, APITCH = (PPC + 15) & ~15;
    // forward ("kw in N"): virtual rows p = (oh, ow) over the full input width, RPT conv rows per tile
    static constexpr int F_RPT = (TILE_M / WI) & ~1, F_TILES = (2 * HP + F_RPT - 1) / F_RPT;
    static constexpr int F_K = KS * CI, F_N = (KS * CO + 15) & ~15;
    // input gradient ("kh, kw in N"): rows q = (oh, ow) of the conv output grid, one tile per image
    static constexpr int D_K = CO, D_N = (KS * KS * CI + 15) & ~15;
};

template <int NCOL, int YROWS>
struct CtSmem {
    static constexpr uint32_t A_PLANE = TILE_M * 128;   // one 32-wide K atom of 128 rows
    static constexpr uint32_t A_BUF = 2 * A_PLANE;      // hi + lo
    static constexpr uint32_t B_PLANE = NCOL * 128;
    static constexpr uint32_t A_OFF = 0, B_OFF = 2 * A_BUF;  // two A buffers (gather of tile i+1 || MMA of tile i)
    static constexpr int YS = NCOL + 1;  // padded Y' row (conflict-free row-per-lane writes)
    // Y' of tile i lives in tile i's A buffer when it fits (its MMAs are complete when Y' is written, and the
    // buffer is refilled only after tile i's epilogue): fewer bytes per CTA, more CTAs per SM
    static constexpr bool Y_IN_A = (uint32_t)YROWS * YS * 4 <= A_BUF;
    static constexpr uint32_t Y_OFF = B_OFF + 2 * B_PLANE;
    static constexpr uint32_t BAR_OFF = Y_OFF + (Y_IN_A ? 0u : (uint32_t)YROWS * YS * 4);
    static constexpr uint32_t TOTAL = BAR_OFF + 64 + 1024;  // + 2 mbarriers, tmem slot, alignment slack
    static constexpr uint32_t ACC_COLS = NCOL <= 32 ? 32 : NCOL <= 64 ? 64 : NCOL <= 128 ? 128 : 256;
    static constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;  // two accumulators
    static_assert(TMEM_COLS <= 512, "TMEM");
};

// Half an A row (16 values k0 .. k0 + 15 of one K atom) -> hi/lo planes, K-major SWIZZLE_128B.
__device__ __forceinline__ void ct_store_half(uint8_t *sm, uint32_t a_off, uint32_t a_plane, int p, int k0,
                                              const float (&v)[16]) {
#pragma unroll
    for (int k4 = 0; k4 < 4; k4++) {
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; e++) split_tf32(v[4 * k4 + e], h[e], l[e]);
        const uint32_t off = smem_u32(sm) + a_off + sw128_off(p, k0 + 4 * k4, TILE_M);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(off), "f"(h[0]), "f"(h[1]), "f"(h[2]), "f"(h[3])
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(off + a_plane), "f"(l[0]), "f"(l[1]), "f"(l[2]),
                     "f"(l[3])
                     : "memory");
    }
}

// The per-CTA pipeline over this CTA's tiles u = blockIdx.x, blockIdx.x + gridDim.x, ...:
//   prologue: mbarriers, TMEM (two accumulators), the B operand (weights) as hi/lo planes (wfn(n, k));
//   gather(u0 -> A0); MMA(u0 -> acc0);
//   per tile i: gather(u_{i+1} -> A[(i+1)%2]); MMA(u_{i+1} -> acc[(i+1)%2]) -- both overlap the tensor core's
//   work on tile i -- then wait for MMA(u_i), TMEM lane (= this thread's A row) -> its padded row of Y' in
//   shared memory, epilogue(u_i) from Y'.
// gather(u, p, k0, v) fills A[p][k0 .. k0 + 15] of tile u (thread t: row p = t % 128, k0 = 16 * (t / 128));
// epilogue(u, sY) writes tile u's outputs (all threads).
// MMAs: 3xTF32 (hi.lo + lo.hi + hi.hi per 8-wide k-step), KSTEPS k-steps.
template <int NCOL, int KSTEPS, int YROWS, class WFN, class GATHER, class EPI>
__device__ __forceinline__ void ct_pipeline(int units, WFN wfn, GATHER gather, EPI epilogue) {
    using L = CtSmem<NCOL, YROWS>;
    extern __shared__ uint8_t ct_raw[];
    // SWIZZLE_128B atoms: 1024-B aligned (offset from the shared array itself: accesses stay LDS/STS)
    uint8_t *sm = ct_raw + ((1024u - (smem_u32(ct_raw) & 1023u)) & 1023u);
    const uint32_t sbase = smem_u32(sm), bar0 = sbase + L::BAR_OFF;
    uint32_t *tslot = (uint32_t *)(sm + L::BAR_OFF + 32);
    float *sY = (float *)(sm + L::Y_OFF);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(L::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int i = tid; i < NCOL * 32; i += CT_THREADS) {
        const int n = i >> 5, k = i & 31;
        float hi, lo;
        split_tf32(wfn(n, k), hi, lo);
        const uint32_t off = L::B_OFF + sw128_off(n, k, NCOL);
        *(float *)(sm + off) = hi;
        *(float *)(sm + off + L::B_PLANE) = lo;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    const int prow = tid & (TILE_M - 1), k0 = 16 * (tid / TILE_M);
    // the next tile's A values are loaded into registers one tile ahead (their latency overlaps the current
    // tile's wait and epilogue) and split / stored into the free A buffer when the current tile's MMAs are out
    float v[16];
    auto load = [&](int u) {
#pragma unroll
        for (int k = 0; k < 16; k++) v[k] = 0.f;
        if (u < units) gather(u, prow, k0, v);
    };
    auto fill = [&](int buf) { ct_store_half(sm, L::A_OFF + buf * L::A_BUF, L::A_PLANE, prow, k0, v); };
    auto issue = [&](int buf) {  // all threads: make the A buffer visible to the tensor core; thread 0 issues
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            constexpr uint32_t idesc = idesc_tf32(TILE_M, NCOL);
            const uint32_t d = tmem + buf * L::ACC_COLS;
#pragma unroll
            for (int s = 0; s < KSTEPS; s++) {
                const uint32_t aa = sbase + L::A_OFF + buf * L::A_BUF + (uint32_t)s * 32, bb = sbase + L::B_OFF + (uint32_t)s * 32;
                const uint64_t ah = sdesc_k128(aa), al = sdesc_k128(aa + L::A_PLANE);
                const uint64_t bh = sdesc_k128(bb), bl = sdesc_k128(bb + L::B_PLANE);
                mma_tf32(d, ah, bl, idesc, s > 0 ? 1u : 0u);
                mma_tf32(d, al, bh, idesc, 1u);
                mma_tf32(d, ah, bh, idesc, 1u);
            }
            mma_commit(bar0 + 8 * buf);
        }
    };
    uint32_t phases = 0;
    int u = blockIdx.x, it = 0;
    if (u < units) {
        load(u);
        fill(0);
        issue(0);
        load(u + (int)gridDim.x);
    }
    for (; u < units; u += gridDim.x, it++) {
        const int buf = it & 1, nu = u + gridDim.x;
        if (nu < units) {
            fill(buf ^ 1);  // A[buf^1] was last read by the MMAs of tile it-1, already waited for
            issue(buf ^ 1);
            load(nu + (int)gridDim.x);  // in flight during this tile's wait + epilogue
        }
        mbar_wait(bar0 + 8 * buf, (phases >> buf) & 1);
        phases ^= 1u << buf;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (L::Y_IN_A) sY = (float *)(sm + L::A_OFF + buf * L::A_BUF);
        {  // warp w reads TMEM lane quarter w % 4 (rows 32*(w%4) ..), 16-column chunks c = w / 4, w / 4 + 2, ...
            const int q = (tid >> 5) & 3, ch = tid >> 7, row = 32 * q + (tid & 31);
#pragma unroll
            for (int c = 0; c < NCOL / 16; c++) {
                if ((c & 1) != ch) continue;
                uint32_t r[16];
                CT_TMEM_LD16(tmem + buf * L::ACC_COLS + ((uint32_t)(32 * q) << 16) + 16 * c, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (row < YROWS) {
#pragma unroll
                    for (int j = 0; j < 16; j++) sY[row * L::YS + 16 * c + j] = __uint_as_float(r[j]);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        epilogue(u, (const float *)sY);
        __syncthreads();  // Y' is rewritten by the next tile
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::TMEM_COLS) : "memory");
    }
}

// ---------------------------------------------------------------- forward: conv + bias + ReLU + pool
template <class G>
__global__ void __launch_bounds__(CT_THREADS) conv_fwd_tc_kernel(const ConvTcArgs a) {
    constexpr int NCOL = G::F_N, VW = G::WI, RPT = G::F_RPT, YROWS = RPT * VW;
    static_assert(G::F_K <= 32 && NCOL <= 256 && RPT >= 2, "forward tile");
    constexpr int YS = CtSmem<NCOL, YROWS>::YS;
    pdl_wait();
    const int tid = threadIdx.x;
    ct_pipeline<NCOL, (G::F_K + 7) / 8, YROWS>(
        a.rows * G::F_TILES,
        [&](int n, int k) {  // B[n = kw*CO + co][k = kh*CI + ci] = W[kh][kw][ci][co]
            const int kh = k / G::CI, ci = k % G::CI, kw = n / G::CO, co = n % G::CO;
            return (k < G::F_K && n < G::KS * G::CO) ? __ldg(a.Wb + ((kh * G::KS + kw) * G::CI + ci) * G::CO + co)
                                                       : 0.f;
        },
        [&](int u, int p, int k0, float (&v)[16]) {  // A row p = (conv row r0 + p / VW, col p % VW): X[row + kh][col][ci]
            const int n_img = u / G::F_TILES, r0 = (u % G::F_TILES) * RPT;
            const int rr = p / VW, col = p % VW, row = r0 + rr;
            if (rr < RPT && row < 2 * G::HP && k0 < G::F_K) {
                const float *xp = a.X + (a.xrow.row0() + n_img) * (int64_t)G::IN_SZ + (row * G::WI + col) * G::CI;
#pragma unroll
                for (int j = 0; j < 16; j++) {
                    const int k = k0 + j;
                    if (k < G::F_K) v[j] = __ldg(xp + (k / G::CI) * G::WI * G::CI + k % G::CI);
                }
            }
        },
        [&](int u, const float *sY) {  // z = bias + sum_kw Y'[(oh, ow + kw)][kw*CO + co]; ReLU; 2x2 pool
            const int n_img = u / G::F_TILES, r0 = (u % G::F_TILES) * RPT;
            const int ph0 = r0 / 2, nph = min(RPT / 2, G::HP - ph0);
            constexpr int PER_ROW = G::WP * G::CO;
            const int64_t pbase = (int64_t)n_img * G::PPC;
            for (int i = tid; i < nph * PER_ROW; i += CT_THREADS) {
                const int phl = i / PER_ROW, rem = i % PER_ROW, pw = rem / G::CO, co = rem % G::CO;
                const float bias = __ldg(a.Wb + G::KS * G::KS * G::CI * G::CO + co);
                float best = 0.f;
                int barg = 0;
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    const float *yr = sY + ((2 * phl + (d >> 1)) * VW + 2 * pw + (d & 1)) * YS + co;
                    float acc = 0.f;
#pragma unroll
                    for (int kw = 0; kw < G::KS; kw++) acc = __fadd_rn(acc, yr[kw * YS + kw * G::CO]);
                    const float z = fmaxf(acc + bias, 0.f);  // bias after the sum (A13), ReLU
                    if (d == 0 || z > best) {                // first maximum wins (A6)
                        best = z;
                        barg = d;
                    }
                }
                const int pe = ((ph0 + phl) * G::WP + pw) * G::CO + co;
                a.P[pbase + pe] = best;
                a.arg[(int64_t)n_img * G::APITCH + pe] = (uint8_t)barg;
                if (a.P_hi) {
                    float hi, lo;
                    split_tf32(best, hi, lo);
                    a.P_hi[pbase + pe] = hi;
                    a.P_lo[pbase + pe] = lo;
                }
            }
        });
}

// ---------------------------------------------------------------- input gradient
template <class G>
__global__ void __launch_bounds__(CT_THREADS) conv_dgrad_tc_kernel(const ConvTcArgs a) {
    constexpr int NCOL = G::D_N, NQ = G::HC * G::WC;
    static_assert(G::D_K <= 32 && NCOL <= 256 && NQ <= TILE_M, "input-gradient tile: one image per tile");
    constexpr int YS = CtSmem<NCOL, NQ>::YS;
    pdl_wait();
    const int tid = threadIdx.x;
    ct_pipeline<NCOL, (G::D_K + 7) / 8, NQ>(
        a.rows,
        [&](int n, int k) {  // B[n = (kh*KS + kw)*CI + ci][k = co] = W[kh][kw][ci][co]
            return (k < G::CO && n < G::KS * G::KS * G::CI) ? __ldg(a.Wb + (int64_t)n * G::CO + k) : 0.f;
        },
        [&](int n_img, int p, int k0, float (&v)[16]) {  // A row q = (oh, ow): dR = dP at the argmax when P > 0
            const int oh = p / G::WC, ow = p % G::WC;
            if (p < NQ && oh < 2 * G::HP && ow < 2 * G::WP && k0 < G::CO) {
                const int e0 = ((oh >> 1) * G::WP + (ow >> 1)) * G::CO + k0;
                const float *dp = a.dP + (int64_t)n_img * G::PPC + e0, *pp = a.Pin + (int64_t)n_img * G::PPC + e0;
                const uint8_t *ar = a.arg + (int64_t)n_img * G::APITCH + e0;
                const int d = ((oh & 1) << 1) | (ow & 1);
#pragma unroll
                for (int j = 0; j < 16; j++)
                    if (k0 + j < G::CO && __ldg(ar + j) == d && __ldg(pp + j) > 0.f) v[j] = __ldg(dp + j);
            }
        },
        [&](int n_img, const float *sY) {
            // dX[h][w][ci] = sum_{kh, kw: 0 <= h-kh < HC, 0 <= w-kw < WC} Y'[(h-kh, w-kw)][(kh*KS + kw)*CI + ci]
            float *dxi = a.dX + (int64_t)n_img * G::IN_SZ;
            for (int i = tid; i < G::IN_SZ; i += CT_THREADS) {
                const int h = i / (G::WI * G::CI), rem = i % (G::WI * G::CI), w = rem / G::CI, ci = rem % G::CI;
                float acc = 0.f;
#pragma unroll
                for (int kh = 0; kh < G::KS; kh++) {
                    const int oh = h - kh;
                    if (oh < 0 || oh >= G::HC) continue;
#pragma unroll
                    for (int kw = 0; kw < G::KS; kw++) {
                        const int ow = w - kw;
                        if (ow < 0 || ow >= G::WC) continue;
                        acc = __fadd_rn(acc, sY[(oh * G::WC + ow) * YS + (kh * G::KS + kw) * G::CI + ci]);
                    }
                }
                dxi[i] = acc;
            }
        });
}

template <class KERN>
cudaError_t launch_ct(KERN kern, uint32_t smem, uint32_t tmem_cols, const ConvTcArgs &a, int units, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // CTAs per SM: shared memory (228 KB per SM, 1 KB reserved per CTA) and TMEM (512 columns)
    const int per_sm = std::max(1, std::min<int>(233472 / (smem + 1024), 512 / tmem_cols));
    const int grid = std::min(units, 148 * per_sm);
    return launch_pdl(kern, dim3(grid), dim3(CT_THREADS), (size_t)smem, s, a);
}

using LeNetC1 = Geo<32, 32, 3, 5, 6>;   // 32x32x3 -> 28x28x6 -> 14x14x6
using LeNetC2 = Geo<14, 14, 6, 5, 16>;  // 14x14x6 -> 10x10x16 -> 5x5x16

template <class G>
bool same_geo(const ConvGeom &g) {
    return g.hi == G::HI && g.wi == G::WI && g.ci == G::CI && g.k == G::KS && g.co == G::CO;
}

}  // namespace

bool conv_tc_supported(const ConvGeom &g, bool dgrad) {
    return same_geo<LeNetC1>(g) ? !dgrad : same_geo<LeNetC2>(g);
}

cudaError_t conv_fwd_tc(const ConvGeom &g, int rows, const float *X, RowSel xrow, const float *Wb, float *P, uint8_t *arg,
                        float *P_hi, float *P_lo, cudaStream_t s, LaunchHook *h) {
    if (!conv_tc_supported(g, false)) return cudaErrorInvalidValue;
    ConvTcArgs a{};
    a.rows = rows; a.X = X; a.xrow = xrow; a.Wb = Wb; a.P = P; a.arg = arg; a.P_hi = P_hi; a.P_lo = P_lo;
    const bool c1 = same_geo<LeNetC1>(g);
    const int N = c1 ? LeNetC1::F_N : LeNetC2::F_N, tiles = c1 ? LeNetC1::F_TILES : LeNetC2::F_TILES;
    char name[112];
    snprintf(name, sizeof name, "conv_fwd_tc[rows=%d,hi=%d,ci=%d,k=%d,co=%d,N=%d,tiles=%d]", rows, g.hi, g.ci, g.k, g.co,
             N, tiles);
    if (h) h->before(name, s);
    using S1 = CtSmem<LeNetC1::F_N, LeNetC1::F_RPT * LeNetC1::WI>;
    using S2 = CtSmem<LeNetC2::F_N, LeNetC2::F_RPT * LeNetC2::WI>;
    cudaError_t e = c1 ? launch_ct(conv_fwd_tc_kernel<LeNetC1>, S1::TOTAL, S1::TMEM_COLS, a, rows * tiles, s)
                       : launch_ct(conv_fwd_tc_kernel<LeNetC2>, S2::TOTAL, S2::TMEM_COLS, a, rows * tiles, s);
    if (h) h->after(name, s);
    return e;
}

cudaError_t conv_dgrad_tc(const ConvGeom &g, int rows, const float *dP, const float *P, const uint8_t *arg, const float *Wb,
                          float *dX, cudaStream_t s, LaunchHook *h) {
    if (!conv_tc_supported(g, true)) return cudaErrorInvalidValue;
    ConvTcArgs a{};
    a.rows = rows; a.dP = dP; a.Pin = P; a.arg = (uint8_t *)arg; a.Wb = Wb; a.dX = dX;
    using G = LeNetC2;
    char name[112];
    snprintf(name, sizeof name, "conv_dgrad_tc[rows=%d,hi=%d,ci=%d,k=%d,co=%d,N=%d]", rows, g.hi, g.ci, g.k, g.co, G::D_N);
    if (h) h->before(name, s);
    using SD = CtSmem<G::D_N, G::HC * G::WC>;
    cudaError_t e = launch_ct(conv_dgrad_tc_kernel<G>, SD::TOTAL, SD::TMEM_COLS, a, rows, s);
    if (h) h->after(name, s);
    return e;
}

}  // namespace mtx
