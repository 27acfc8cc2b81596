// gemm_tc.cu -- the TF32 tensor-core GEMM engine of the local forward/backward
// (the dense contractions of each replica's step; SURVEY.md
// §8(a) a4/a6/a7).  sm_100a only: 5th-gen tensor cores through tcgen05.
//
//   * persistent CTAs (<= one per SM), static round-robin over (m, n, k-split) tiles
//   * warp 0: TMA producer -- cp.async.bulk.tensor (SWIZZLE_128B) into a STAGES-deep
//     shared-memory ring, completion on mbarriers (expect_tx)
//   * warp 1: MMA issuer -- one elected thread issues tcgen05.mma.cta_group::1.kind::tf32
//     (M = 128, N = BN, K = 8 per instruction) into a TMEM accumulator; tcgen05.commit
//     frees the smem slot and, after the last k-block, signals the epilogue
//   * warp 2: TMEM allocator (a ring of up to 4 accumulators x BN columns -> the MMA warp runs
//     ahead of the epilogue)
//   * warps 4-11: epilogue -- tcgen05.ld 32x32b (one accumulator row per thread) promoted into
//     fp32 registers; the finished tile is staged through swizzled shared memory and written
//     as whole row segments with the fused bias + ReLU (forward), ReLU mask (dgrad), hi/lo
//     planes (3xTF32 consumers) or plain/partial store (wgrad)
//
// Operands are read in place from the row-major activation/weight/gradient
// buffers: K-major (rows contiguous in K) or MN-major (contiguous in M/N) via the
// UMMA shared-memory descriptor's major bit, so forward, dgrad and wgrad need no
// transposes.  Accumulation is fp32 in TMEM; fp32 operands are consumed as TF32.
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "gemm_tc.h"

namespace mtx {
namespace {

// Phase timestamps and MMA-warp stall counters (MTX_TC_DBG & 4) exist only in a trace build (-DMTX_TRACE=1): their
// printf gave every GEMM variant a stack frame and cost the small latency-bound GEMMs ~2-4 us per launch (cfg2)
#ifndef MTX_TRACE
#define MTX_TRACE 0
#endif
constexpr bool TRACE = MTX_TRACE != 0;
// Measured-and-rejected engine experiments (L2 prefetch MTX_TC_PF / MTX_TC_PFB, A multicast MTX_TC_MC) exist only in an
// experiment build (-DMTX_TC_EXPERIMENTS=1): their code, even disabled at run time, slowed the small GEMMs (cfg2)
#ifndef MTX_TC_EXPERIMENTS
#define MTX_TC_EXPERIMENTS 0
#endif
constexpr bool EXPER = MTX_TC_EXPERIMENTS != 0;
#ifndef MTX_F16_CHUNK
#define MTX_F16_CHUNK 4
#endif
// BK: k-block in fp32 (TF32) elements; a k-block row is 128 B in both element types (BKH = 64 fp16)
constexpr int BM = 128, BK = 32, BKH = 64;

// Shared-memory plan per variant.  SPLIT (3xTF32) stages two planes of each operand tile: hi =
// rne_tf32(x) and lo = rne_tf32(x - hi), written once by the tensor's producer.
// F16 (3xF16): the same two planes in fp16 with a per-tensor power-of-two scale (common.cuh): a k-block
// of 64 fp16 elements occupies the bytes of 32 fp32 ones, so the byte plan is identical.
template <int BN, bool SPLIT, bool PAIR = false, bool F16 = false>
struct SmemLayout {
    // warps 0 TMA, 1 MMA, 2 TMEM alloc, 3 spare, 4-11 epilogue
    static constexpr int THREADS = 384;
    // k-blocks accumulated in TMEM before the epilogue warps promote the partial into fp32
    // registers (the tensor core's internal accumulation truncates): K = 128
    // elements per promotion in both split modes
    static constexpr int CHUNK = F16 ? MTX_F16_CHUNK : SPLIT ? 4 : 8;
    static constexpr uint32_t A_BYTES = BM * 128;
    // PAIR (cta_group::2): the CTA pair computes a 256 x BN tile; each CTA holds its 128 rows of A and
    // half of B's BN columns (the MMA reads both halves; measured by tools/tc_pair_probe.cu)
    static constexpr uint32_t B_BYTES = (PAIR ? BN / 2 : BN) * 128;
    // stage: [A][B] (hi planes) followed, for 3xTF32, by [A_lo][B_lo] at RAW_BYTES
    static constexpr uint32_t RAW_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t B_OFF = A_BYTES;
    static constexpr uint32_t STAGE_BYTES = RAW_BYTES * (SPLIT ? 2 : 1);
    // epilogue staging: one 32 x 32 fp32 sub-tile per epilogue warp (coalesced stores)
    static constexpr uint32_t EPI_BYTES = 8 * 32 * 32 * 4;
    static constexpr uint32_t SMEM_MAX = 232448;  // 227 KB opt-in per CTA
    static constexpr int STAGES_FIT = (int)((SMEM_MAX - 256 - 1024 - EPI_BYTES) / STAGE_BYTES);
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;  // deepest ring that fits
    static_assert(STAGES >= 2, "smem ring");
    static constexpr uint32_t EPI_OFF = STAGES * STAGE_BYTES;
    static constexpr uint32_t BAR_OFF = EPI_OFF + EPI_BYTES;
    static constexpr uint32_t TOTAL = BAR_OFF + 256 + 1024;  // barriers + tmem slot + 1024-B alignment slack
    // TMEM accumulator ring: the MMA warp runs up to NBUF chunks ahead of the epilogue
    static constexpr int ACC_COLS = BN;
    static constexpr int NBUF = 512 / ACC_COLS > 4 ? 4 : 512 / ACC_COLS;
    static constexpr uint32_t TMEM_COLS = NBUF * ACC_COLS;
};

struct TcParams {
    CUtensorMap ta;     // A (1xTF32) or A's hi plane (3xTF32)
    CUtensorMap tb;
    CUtensorMap ta_lo;  // 3xTF32: lo planes
    CUtensorMap tb_lo;
    float *C_hi, *C_lo;  // optional hi/lo planes of the output (for the next 3xTF32 GEMM)
    int M, N, K;
    int a_mn, b_mn;      // operand majorness (1 = MN-major)
    int a_3d, b_3d;      // MN-major operand described by a 3-D tensor map (32-element chunks stacked in one box)
    int tiles_m, tiles_n, splits, kb_total, kb_per_split;
    int epi;
    const float *bias;
    const float *mask;
    int64_t ldm;
    float *C;
    int64_t ldc;
    float *partial;
    const int64_t *a_win;  // dataset operand: sample-dimension offset read on the device
    int64_t a_base;
    int dbg;               // development only (MTX_TC_DBG): 1 skip epilogue stores, 2 skip TMA loads
    int cluster;           // 1: the splits of a tile form one thread-block cluster and are folded
                           // through distributed shared memory (no partial buffer, no fold launch)
    // 3xF16: operand scale slots (the sum is multiplied by s_A * s_B, exact) and the output planes
    const TScale *tsA, *tsB;
    F16Out fo;
    // dgrad: the ReLU mask as a bitmask [M][mbits_ld words] (written by the forward epilogue) instead of
    // the fp32 activation
    const uint32_t *mbits;
    int64_t mbits_ld;
    int pf;  // producer: L2 prefetch distance in k-blocks (0: off)
    int pfb; // before the PDL wait: L2 prefetch of the CTA's first B k-blocks (forward / dgrad: the weights)
    int mc;  // PAIR: 4-CTA clusters of two pairs on adjacent N tiles; each A plane is loaded once and multicast
};

// Work unit t -> (k-split z, output tile r).  Cluster mode: the splits of a tile are consecutive
// CTAs (one cluster, z = rank in the cluster); otherwise splits are outermost.
__device__ __forceinline__ void unit_of(const TcParams &p, int t, int tiles_mn, int &z, int &r) {
    if (p.cluster) {
        z = t % p.splits;
        r = t / p.splits;
    } else {
        z = t / tiles_mn;
        r = t % tiles_mn;
    }
}

// ReLU-mask values mask[m][n..n+3] (dgrad epilogue): loaded ahead of the stores they gate, so a
// warp's mask loads are in flight together instead of one HBM round trip per store.
__device__ __forceinline__ float4 load_mask(const TcParams &p, int m, int n) {
    if (p.mbits) {  // bits n..n+3 of the row's word n / 32 (n % 4 == 0; bits past N are 0)
        const uint32_t w = __ldg(p.mbits + (int64_t)m * p.mbits_ld + (n >> 5)) >> (n & 31);
        return make_float4((w & 1u) ? 1.f : 0.f, (w & 2u) ? 1.f : 0.f, (w & 4u) ? 1.f : 0.f, (w & 8u) ? 1.f : 0.f);
    }
    const float *mk = p.mask + (int64_t)m * p.ldm + n;
    if (n + 3 < p.N) return __ldg((const float4 *)mk);
    float mv[4];
    for (int e = 0; e < 4; e++) mv[e] = n + e < p.N ? mk[e] : 0.f;
    return make_float4(mv[0], mv[1], mv[2], mv[3]);
}

// The fused epilogue on 4 consecutive outputs C[m][n..n+3] (coalesced across a warp): bias (+ReLU)
// or ReLU mask (mkv, from load_mask), the fp32 store and, for a 3xTF32 consumer, the hi/lo planes.
// MASK: compile-time dgrad variant (EPI_MASK); otherwise bias (+ReLU) or a plain store.
// bias[n..n+3] (zero past N): loaded once per staged sub-tile column group, not per row
__device__ __forceinline__ float4 load_bias(const TcParams &p, int n) {
    if (!(p.epi == EPI_BIAS_RELU || p.epi == EPI_BIAS) || n >= p.N) return make_float4(0.f, 0.f, 0.f, 0.f);
    if (n + 3 < p.N && ((uintptr_t)(p.bias + n) & 15) == 0) return __ldg((const float4 *)(p.bias + n));
    float b[4];
    for (int e = 0; e < 4; e++) b[e] = n + e < p.N ? __ldg(p.bias + n + e) : 0.f;
    return make_float4(b[0], b[1], b[2], b[3]);
}

template <bool MASK, bool F16>
__device__ __forceinline__ float4 epi_store(const TcParams &p, int m, int n, float4 sv, float4 mkv, float inv_so, float &amx,
                                            float4 bz) {
    const bool vec4 = n + 3 < p.N;
    float o[4] = {sv.x, sv.y, sv.z, sv.w};
    if constexpr (MASK) {
        const float mv[4] = {mkv.x, mkv.y, mkv.z, mkv.w};
#pragma unroll
        for (int e = 0; e < 4; e++)
            if (!(mv[e] > 0.f)) o[e] = 0.f;
    } else if (p.epi == EPI_BIAS_RELU || p.epi == EPI_BIAS) {
        const float bv[4] = {bz.x, bz.y, bz.z, bz.w};
#pragma unroll
        for (int e = 0; e < 4; e++)
            if (n + e < p.N) {
                o[e] += bv[e];
                if (p.epi == EPI_BIAS_RELU) o[e] = fmaxf(o[e], 0.f);
            }
    }
    const int64_t off = (int64_t)m * p.ldc + n;
    if (p.C && !(F16 && p.fo.skip_f32 && p.splits == 1)) {
        if (vec4) *(float4 *)(p.C + off) = make_float4(o[0], o[1], o[2], o[3]);
        else for (int e = 0; e < 4 && n + e < p.N; e++) p.C[off + e] = o[e];
    }
    if (F16) {  // fp16 hi/lo planes (scale from the output bound) for the consuming 3xF16 GEMM
        if (p.fo.h) {
            float x[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {
                x[e] = n + e < p.N ? o[e] : 0.f;
                amx = fmaxf(amx, fabsf(x[e]));
            }
            // two elements per conversion (cvt.rn.f16x2.f32); same rounding as split_f16
            __half2 h2[2], l2[2];
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const float2 y = make_float2(x[2 * e] * inv_so, x[2 * e + 1] * inv_so);
                h2[e] = __float22half2_rn(y);
                const float2 hf = __half22float2(h2[e]);
                l2[e] = __float22half2_rn(make_float2(y.x - hf.x, y.y - hf.y));
            }
            const int64_t po = (int64_t)m * p.fo.ld + n;
            if (vec4) {
                *(uint2 *)(p.fo.h + po) = make_uint2(*(uint32_t *)&h2[0], *(uint32_t *)&h2[1]);
                *(uint2 *)(p.fo.l + po) = make_uint2(*(uint32_t *)&l2[0], *(uint32_t *)&l2[1]);
            } else {
                const __half hh[4] = {__low2half(h2[0]), __high2half(h2[0]), __low2half(h2[1]), __high2half(h2[1])};
                const __half ll[4] = {__low2half(l2[0]), __high2half(l2[0]), __low2half(l2[1]), __high2half(l2[1])};
                for (int e = 0; e < 4 && n + e < p.N; e++) {
                    p.fo.h[po + e] = hh[e];
                    p.fo.l[po + e] = ll[e];
                }
            }
        }
    } else if (p.C_hi) {  // hi/lo planes for the consuming 3xTF32 GEMM
        float hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; e++) split_tf32(o[e], hi[e], lo[e]);
        if (vec4) {
            *(float4 *)(p.C_hi + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
            *(float4 *)(p.C_lo + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
        } else {
            for (int e = 0; e < 4 && n + e < p.N; e++) {
                p.C_hi[off + e] = hi[e];
                p.C_lo[off + e] = lo[e];
            }
        }
    }
    return make_float4(o[0], n + 1 < p.N ? o[1] : 0.f, n + 2 < p.N ? o[2] : 0.f, n + 3 < p.N ? o[3] : 0.f);
}

// Cluster split-K: the fp32 partial tile [BM][BN] of a CTA lives at the start of its (then idle)
// stage ring, 16-B chunks XOR-swizzled within each 128-B group so that both the row-per-lane writes
// and the chunk-per-lane reads are bank-conflict free.
template <int BN>
__device__ __forceinline__ uint32_t ktile_off(int row, int j) {
    return (uint32_t)row * (BN * 4) + (uint32_t)(((j & ~7) | ((j ^ row) & 7)) * 16);
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t local_addr, uint32_t cta) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(cta));
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(remote)
                 : "memory");
    return v;
}

// ------------------------------------------------------------------ PTX wrappers
// (smem_u32 and the mbarrier helpers mbar_init / mbar_expect_tx / mbar_arrive / mbar_wait: common.cuh)
// Warp-converged issue: the whole warp runs the producer / MMA loops (warp-uniform values stay in
// uniform registers) and elect.sync picks the one lane that issues each asynchronous operation.
__device__ __forceinline__ void mbar_expect_tx_elect(uint32_t bar, uint32_t bytes) {
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_elect(uint32_t bar) {
    asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_2d_elect(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n}\n" ::"r"(
            dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void umma_tf32_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
        " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// kind::f16 (fp16 operands, fp32 accumulator): K = 16 per instruction, same issue cost as kind::tf32's K = 8
__device__ __forceinline__ void umma_f16_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
        " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_f16_pair_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                    uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
        " @e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit_elect(uint32_t bar) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
        : "memory");
}
// CTA pair (cta_group::2) variants: TMA into this CTA's smem completing on the leader's mbarrier (a
// shared::cluster address), the pair MMA, and commits multicast to both CTAs' mbarriers.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
__device__ __forceinline__ void tma_load_2d_pair_elect(uint32_t dst, const CUtensorMap *map, uint32_t bar_cluster, int c0,
                                                       int c1) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n}\n" ::"r"(
            dst),
        "l"((uint64_t)map), "r"(bar_cluster), "r"(c0), "r"(c1)
        : "memory");
}
// CTA pair load multicast to the CTAs of `mask` (same smem offset in each; each destination pair's leader barrier
// counts the bytes): the A tile shared by the two pairs of a 4-CTA cluster (3xF16 multicast plan)
__device__ __forceinline__ void tma_load_2d_pair_mc_elect(uint32_t dst, const CUtensorMap *map, uint32_t bar_cluster, int c0,
                                                          int c1, uint16_t mask) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;\n}\n" ::"r"(
            dst),
        "l"((uint64_t)map), "r"(bar_cluster), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void umma_tf32_pair_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                     uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
        " @e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair_elect(uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
            bar),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
    // default semantics (release at CTA scope), as CUTLASS arrives on a peer CTA's barrier: ".release.cluster" compiles to
    // MEMBAR.ALL.GPU, which made every TMEM hand-off wait for the epilogue's outstanding global stores (ncu)
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void tma_load_3d_elect(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                                  int c2) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n}\n" ::"r"(
            dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair_elect(uint32_t dst, const CUtensorMap *map, uint32_t bar_cluster, int c0,
                                                       int c1, int c2) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n}\n" ::"r"(
            dst),
        "l"((uint64_t)map), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// L2 prefetch of a future operand tile (no smem, no barrier): the ring only holds STAGES k-blocks, fewer than an HBM
// round trip's worth of MMAs when the operand was evicted from L2 since its producer wrote it
__device__ __forceinline__ void tma_prefetch_2d_elect(const CUtensorMap *map, int c0, int c1) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n}\n" ::"l"((uint64_t)map), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d_elect(const CUtensorMap *map, int c0, int c1, int c2) {
    asm volatile(
        "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
        " @e cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n}\n" ::"l"((uint64_t)map), "r"(c0),
        "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"((uint64_t)map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
            d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

#define TMEM_LD32(taddr, r)                                                                                      \
    asm volatile(                                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                            \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),    \
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])   \
        : "r"(taddr))

#define TMEM_LD16(taddr, r)                                                                                      \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),   \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
                 : "r"(taddr))

// UMMA shared-memory descriptor, version 1 (sm_100).  Verified on B200 with tools/tc_probe.cu:
//   K-major : SWIZZLE_128B (type 2) -- 8-row x 128-B atoms (16-B chunks XOR row%8) stacked along
//             M/N at SBO = 1024 B; LBO unused.  k-step of 8 tf32 = +32 B inside the row.
//   MN-major: SWIZZLE_128B_BASE32B (type 1, the only MN-major layout tf32 accepts) -- 128-B rows
//             of 32 M/N elements, 32-B chunks XOR row%4; 4-row K groups at SBO = 512 B, 32-element
//             M/N groups at LBO = BK * 128 B.  k-step of 8 = +1024 B.
//   fp16 (3xF16): K-major as above (64 elements per 128-B row, k-step of 16 = +32 B); MN-major
//             SWIZZLE_128B (type 2) -- 128-B rows of 64 M/N elements, 16-B chunks XOR row%8; 8-row K
//             groups at SBO = 1024 B, 64-element M/N groups at LBO = BKH * 128 B.  k-step of 16 = +2048 B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout_type) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)layout_type << 61;
    return d;
}

// Instruction descriptor: D fp32, A/B tf32 (format 2, kind::tf32) or f16 (format 0, kind::f16), majors,
// N>>3, M>>4 (dense).
__host__ __device__ constexpr uint32_t instr_desc(int M, int N, int a_mn, int b_mn, bool f16 = false) {
    return (1u << 4) | ((f16 ? 0u : 2u) << 7) | ((f16 ? 0u : 2u) << 10) | ((uint32_t)a_mn << 15) |
           ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// PAIR: the cluster holds the S pairs of a tile's splits (cluster rank = 2 * split + rank in the pair); the CTAs
// holding the same 128-row half (rank in the pair pr) fold that half: CTA (z, pr) rows [z*BM/S, (z+1)*BM/S) of
// it, reading cluster ranks 2u + pr.
template <int BN, bool MASK, bool PAIR, bool F16>
__device__ __noinline__ void cluster_fold(const TcParams &p, uint32_t base, float inv_so, float &amx) {
    int z, r;
    uint32_t crank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const int pr = PAIR ? (int)(crank & 1) : 0;
    unit_of(p, PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x, p.tiles_m * p.tiles_n, z, r);
    const int m0 = (r / p.tiles_n) * (PAIR ? 2 * BM : BM) + BM * pr, n0 = (r % p.tiles_n) * BN;
    const int S = p.splits;
    const int r0 = BM * z / S, r1 = BM * (z + 1) / S;
    constexpr int CPR = BN / 4;
    for (int idx = threadIdx.x - 128; idx < (r1 - r0) * CPR; idx += 256) {
        const int row = r0 + idx / CPR, j = idx % CPR;
        const int m = m0 + row, n = n0 + 4 * j;
        if (m >= p.M || n >= p.N) continue;
        const uint32_t la = base + ktile_off<BN>(row, j);
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (u < S) v[u] = ld_dsmem_f4(la, PAIR ? (uint32_t)(2 * u + pr) : (uint32_t)u);
        float4 sum = v[0];
#pragma unroll
        for (int u = 1; u < 8; u++)
            if (u < S) {
                sum.x += v[u].x; sum.y += v[u].y; sum.z += v[u].z; sum.w += v[u].w;
            }
        epi_store<MASK, F16>(p, m, n, sum, MASK ? load_mask(p, m, n) : make_float4(0.f, 0.f, 0.f, 0.f), inv_so, amx,
                             load_bias(p, n));
    }
}

// FAST (3xF16, 128-wide tiles): the host guarantees every tile takes the whole-tile fast epilogue (no ragged edge,
// no split-K, planes-only or fp32-only output): the general epilogue and the cluster fold are compiled out of it.
// CLU (3xF16): every launch is a split-K cluster (partials folded through DSMEM): the direct epilogue is out.
// PART (3xF16): split-K partials to global memory only (folded by splitk_reduce): the output epilogues are out.
template <int BN, bool SPLIT, bool PAIR, bool MASK, bool F16, bool FAST = false, bool CLU = false, bool PART = false>
__global__ void __launch_bounds__(SmemLayout<BN, SPLIT, PAIR>::THREADS, 1) tc_gemm_kernel(const __grid_constant__ TcParams p) {
    using L = SmemLayout<BN, SPLIT, PAIR, F16>;
    constexpr int KB = F16 ? BKH : BK;        // elements per k-block (one 128-B row)
    constexpr int CH = F16 ? 64 : 32;         // MN-major: elements per 128-B chunk along M/N
    constexpr uint32_t CHB = (uint32_t)KB * 128;  // bytes between MN-major chunks of a stage
    constexpr int STAGES = L::STAGES;
    extern __shared__ uint8_t smem_raw[];
    // SWIZZLE_128B atoms need 1024-B aligned stage buffers
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = smem_u32(smem);
    uint64_t *bars = (uint64_t *)(smem + L::BAR_OFF);
    // bars: full[STAGES], empty[STAGES], tfull[NBUF], tempty[NBUF]  (<= 192 B)
    constexpr int NBUF = L::NBUF;
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * STAGES, tfull0 = empty0 + 8 * STAGES,
                   tempty0 = tfull0 + 8 * NBUF;
    uint32_t *tmem_slot = (uint32_t *)(smem + L::BAR_OFF + 224);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // development (MTX_TC_DBG & 4): %globaltimer at the phases of CTA 0 and the last CTA, printed at exit
    __shared__ uint64_t dts[8];
    auto stamp = [&](int i) {
        if (TRACE && (p.dbg & 4)) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            dts[i] = t;
        }
    };
    if (threadIdx.x == 0) stamp(0);
    uint32_t crank = 0;  // PAIR: cluster rank; pairs are cluster ranks (2j, 2j + 1) -- a cluster holds one pair,
                         // or the S pairs of a tile's K splits (p.cluster)
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const uint32_t rank = crank & 1, lead_rank = crank & ~1u;  // rank in the pair; cluster rank of its leader
    const bool leader = rank == 0;
    const uint16_t pair_mask = (uint16_t)(3u << lead_rank);  // commit multicast to both CTAs of this pair

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&p.ta) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&p.tb) : "memory");
        if (SPLIT) {
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&p.ta_lo) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&p.tb_lo) : "memory");
        }
        for (int s = 0; s < STAGES; s++) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, (EXPER && PAIR && p.mc) ? 2 : 1);  // multicast: a slot is free once both pairs consumed it
        }
        for (int a = 0; a < NBUF; a++) {
            mbar_init(tfull0 + 8 * a, 1);
            mbar_init(tempty0 + 8 * a, PAIR ? 16 : 8);  // the epilogue warps (of both CTAs of a pair)
        }

        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(L::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(L::TMEM_COLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();  // the peer's barriers exist before any TMA / arrive targets them
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // Before waiting on the previous kernel: pull this CTA's first B k-blocks into L2.  B of a forward / dgrad is the
    // weights (written steps ago); a prefetch is only a hint (L2 is coherent), so it is safe whatever produced B.
    if (EXPER && warp == 0 && !(p.dbg & 2) && p.pfb) {
        int z0, r0;
        const int t0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
        if (t0 < p.tiles_m * p.tiles_n * p.splits) {
            unit_of(p, t0, p.tiles_m * p.tiles_n, z0, r0);
            const int n0 = (r0 % p.tiles_n) * BN + (PAIR ? (BN / 2) * (int)(crank & 1) : 0);
            const int kb0 = z0 * p.kb_per_split, kb1 = min(p.kb_total, kb0 + min(p.kb_per_split, L::STAGES));
            constexpr int KBP = F16 ? BKH : BK, CHP = F16 ? 64 : 32;
            for (int kb = kb0; kb < kb1; kb++) {
#pragma unroll
                for (int plane = 0; plane < (SPLIT ? 2 : 1); plane++) {
                    const CUtensorMap *mb = plane ? &p.tb_lo : &p.tb;
                    if (!p.b_mn) tma_prefetch_2d_elect(mb, kb * KBP, n0);
                    else if (p.b_3d) tma_prefetch_3d_elect(mb, 0, kb * KBP, n0 / CHP);
                }
            }
        }
    }
    pdl_wait();  // prologue above overlaps the previous kernel's tail (programmatic launch)
    if (threadIdx.x == 0) stamp(1);
    // 256-wide pair tiles: 128 promoted accumulators per epilogue thread.  The producer / MMA / allocator warpgroup
    // hands registers to the two epilogue warpgroups (128 x 56 + 256 x 224 <= 64 K); each role's code follows its
    // setmaxnreg so the compiler allocates that region within the new budget
    constexpr bool REGS = BN == 256;

    const int tiles_mn = p.tiles_m * p.tiles_n;
    const int total = tiles_mn * p.splits;
    // work units: one per CTA, or one per CTA pair (both CTAs of a pair walk the same units).  Written
    // inline in each loop (from blockIdx / gridDim) so the loop counters stay in uniform registers.
#define MTX_UNITS(t) for (int t = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x; t < total; \
                          t += PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x)
    constexpr int TILE_M = PAIR ? 2 * BM : BM;      // output rows per work unit
    constexpr int B_COLS = PAIR ? BN / 2 : BN;      // B columns this CTA loads
    const int m_off = PAIR ? BM * (int)rank : 0;    // this CTA's rows within the unit
    const int nb_off = PAIR ? B_COLS * (int)rank : 0;

    if (warp < 4) {
    if constexpr (REGS) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory");
    if (warp == 0) {
        // ================= TMA producer (the whole warp runs the loop; one elected lane issues)
        {
            const int64_t row0 = p.a_win ? (*p.a_win + p.a_base) : 0;
            int stage = 0;
            uint32_t phase = 0;
            MTX_UNITS(t) {
                int z, r;
                unit_of(p, t, tiles_mn, z, r);
                // raster n-fastest: the CTAs sharing an A row-panel run together (A read from DRAM once,
                // B -- the weights -- stays L2-resident)
                const int m0 = (r / p.tiles_n) * TILE_M + m_off, n0 = (r % p.tiles_n) * BN + nb_off;
                const int kb0 = z * p.kb_per_split, kb1 = min(p.kb_total, kb0 + p.kb_per_split);
                for (int kb = kb0; kb < kb1; kb++) {
                    if (EXPER && p.pf && kb + p.pf < kb1 && !(p.dbg & 2)) {  // k-block kb + pf into L2 (both planes, A and B)
                        const int kp = (kb + p.pf) * KB;
#pragma unroll
                        for (int plane = 0; plane < (SPLIT ? 2 : 1); plane++) {
                            const CUtensorMap *ma = plane ? &p.ta_lo : &p.ta, *mb = plane ? &p.tb_lo : &p.tb;
                            if (!p.a_mn) tma_prefetch_2d_elect(ma, kp, (int)(row0 + m0));
                            else if (p.a_3d) tma_prefetch_3d_elect(ma, 0, (int)(row0 + kp), m0 / CH);
                            else {
#pragma unroll
                                for (int j = 0; j < BM / CH; j++) tma_prefetch_2d_elect(ma, m0 + CH * j, (int)(row0 + kp));
                            }
                            if (!p.b_mn) tma_prefetch_2d_elect(mb, kp, n0);
                            else if (p.b_3d) tma_prefetch_3d_elect(mb, 0, kp, n0 / CH);
                            else {
#pragma unroll
                                for (int j = 0; j < B_COLS / CH; j++) tma_prefetch_2d_elect(mb, n0 + CH * j, kp);
                            }
                        }
                    }
                    mbar_wait(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t sa = sbase + stage * L::STAGE_BYTES, sb = sa + L::B_OFF;
                    const uint32_t fb = full0 + 8 * stage;
                    // PAIR: both CTAs' loads complete on the leader's full barrier, armed by the leader alone
                    const uint32_t fbc = PAIR ? mapa_u32(fb, lead_rank) : fb;
                    if (EXPER && (p.dbg & 2)) {  // development (experiment build): MMA-only timing
                        if (leader) mbar_arrive_elect(fb);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (leader) mbar_expect_tx_elect(fb, PAIR ? 2 * L::STAGE_BYTES : L::STAGE_BYTES);
                    const int k0 = kb * KB;
#pragma unroll
                    for (int plane = 0; plane < (SPLIT ? 2 : 1); plane++) {  // hi into the raw region, lo after it
                        const CUtensorMap *ma = plane ? &p.ta_lo : &p.ta, *mb = plane ? &p.tb_lo : &p.tb;
                        const uint32_t pa = sa + plane * L::RAW_BYTES, pb = sb + plane * L::RAW_BYTES;
                        auto load = [&](uint32_t dst, const CUtensorMap *map, int c0, int c1) {
                            if (PAIR) tma_load_2d_pair_elect(dst, map, fbc, c0, c1);
                            else tma_load_2d_elect(dst, map, fb, c0, c1);
                        };
                        // MN-major 3-D map: (32-element chunk, K row, chunk index) -> the chunks of a tile land
                        // BK * 128 B apart, the MN-major SWIZZLE_128B_BASE32B layout, in one TMA operation
                        auto load3 = [&](uint32_t dst, const CUtensorMap *map, int k_row, int chunk) {
                            if (PAIR) tma_load_3d_pair_elect(dst, map, fbc, 0, k_row, chunk);
                            else tma_load_3d_elect(dst, map, fb, 0, k_row, chunk);
                        };
                        if (EXPER && PAIR && p.mc && !p.a_mn) {
                            // the cluster's two pairs share A's rows: pair 0 loads the hi plane, pair 1 the lo plane, each
                            // multicast to the same-rank CTA of both pairs
                            if ((int)((crank >> 1) & 1) == plane)
                                tma_load_2d_pair_mc_elect(pa, ma, fbc, k0, (int)(row0 + m0),
                                                          (uint16_t)((1u << rank) | (1u << (rank + 2))));
                        } else if (!p.a_mn) {
                            load(pa, ma, k0, (int)(row0 + m0));
                        } else if (p.a_3d) {
                            load3(pa, ma, (int)(row0 + k0), m0 / CH);
                        } else {
#pragma unroll
                            for (int j = 0; j < BM / CH; j++) load(pa + j * CHB, ma, m0 + CH * j, (int)(row0 + k0));
                        }
                        if (!p.b_mn) {
                            load(pb, mb, k0, n0);
                        } else if (p.b_3d) {
                            load3(pb, mb, k0, n0 / CH);
                        } else {
#pragma unroll
                            for (int j = 0; j < B_COLS / CH; j++) load(pb + j * CHB, mb, n0 + CH * j, k0);
                        }
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ================= MMA issuer (whole warp, one elected lane issues; PAIR: the leader CTA's only).  Each tile's k-range is cut
        // into chunks of CHUNK k-blocks; chunk i accumulates into TMEM buffer (i % NBUF) and is handed to
        // the epilogue.  Descriptors: built once per k-block, advanced by a constant per 8-element k-step
        // (K-major: 32 B inside the 128-B swizzled row; MN-major: two 4-row K groups = 1024 B).
        {
            const uint32_t idesc = instr_desc(TILE_M, BN, p.a_mn, p.b_mn, F16);
            const uint64_t mn_desc = F16 ? smem_desc(0, BKH * 128, 1024, 2) : smem_desc(0, BK * 128, 512, 1);
            const uint64_t a_hi = p.a_mn ? mn_desc : smem_desc(0, 16, 1024, 2);
            const uint64_t b_hi = p.b_mn ? mn_desc : smem_desc(0, 16, 1024, 2);
            constexpr uint32_t MN_STEP = (F16 ? 2048 : 1024) >> 4;  // one MMA's K rows in an MN-major tile
            const uint32_t a_step = p.a_mn ? MN_STEP : (32 >> 4), b_step = p.b_mn ? MN_STEP : (32 >> 4);
            constexpr uint64_t LO = L::RAW_BYTES >> 4;  // hi plane -> lo plane of the same operand tile
            int stage = 0;
            uint32_t phase = 0;
            int buf = 0;
            uint32_t buf_phase = 0;
            long long wait_te = 0, wait_full = 0;  // development (MTX_TC_DBG & 4): MMA-warp stall cycles
            MTX_UNITS(t) {
                int z, r;
                unit_of(p, t, tiles_mn, z, r);
                const int kb0 = z * p.kb_per_split, kb1 = min(p.kb_total, kb0 + p.kb_per_split);
                for (int c0 = kb0; c0 < kb1; c0 += L::CHUNK) {
                    const int c1 = min(kb1, c0 + L::CHUNK);
                    long long w0 = (TRACE && (p.dbg & 4)) ? clock64() : 0;
                    mbar_wait(tempty0 + 8 * buf, buf_phase ^ 1);
                    if (TRACE && (p.dbg & 4)) wait_te += clock64() - w0;
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + buf * L::ACC_COLS;
                    for (int kb = c0; kb < c1; kb++) {
                        long long w1 = (TRACE && (p.dbg & 4)) ? clock64() : 0;
                        mbar_wait(full0 + 8 * stage, phase);
                        if ((TRACE && (p.dbg & 4)) && !(kb == kb0 && t == (PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x)))
                            wait_full += clock64() - w1;
                        tc_fence_after();
                        if (lane == 0 && kb == kb0 && t == (PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x)) stamp(2);
                        const uint32_t sa = sbase + stage * L::STAGE_BYTES, sb = sa + L::B_OFF;
                        const uint64_t ad0 = a_hi | ((sa >> 4) & 0x3FFF), bd0 = b_hi | ((sb >> 4) & 0x3FFF);
#pragma unroll
                        for (int kk = 0; kk < 4; kk++) {  // 4 MMAs of K = 8 (tf32) / 16 (f16) per k-block
                            const uint64_t ad = ad0 + kk * a_step, bd = bd0 + kk * b_step;
                            const uint32_t acc0 = (kb > c0 || kk > 0) ? 1u : 0u;
                            auto mma = [&](uint64_t x, uint64_t y, uint32_t acc) {
                                if (F16) {
                                    if (PAIR) umma_f16_pair_elect(d_tmem, x, y, idesc, acc);
                                    else umma_f16_elect(d_tmem, x, y, idesc, acc);
                                } else {
                                    if (PAIR) umma_tf32_pair_elect(d_tmem, x, y, idesc, acc);
                                    else umma_tf32_elect(d_tmem, x, y, idesc, acc);
                                }
                            };
                            if (SPLIT) {
                                // 3xTF32 / 3xF16: hi.lo + lo.hi + hi.hi (hi = rn(x), lo = rn(x - hi))
                                mma(ad, bd + LO, acc0);
                                mma(ad + LO, bd, 1u);
                                mma(ad, bd, 1u);
                            } else {
                                mma(ad, bd, acc0);
                            }
                        }
                        // frees the smem slot (of both CTAs of a pair) when these MMAs retire
                        if (PAIR) umma_commit_pair_elect(empty0 + 8 * stage, (EXPER && p.mc) ? (uint16_t)0xF : pair_mask);
                        else umma_commit_elect(empty0 + 8 * stage);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    // chunk partial ready for promotion (in both CTAs' TMEM for a pair)
                    if (PAIR) umma_commit_pair_elect(tfull0 + 8 * buf, pair_mask);
                    else umma_commit_elect(tfull0 + 8 * buf);
                    if (++buf == NBUF) { buf = 0; buf_phase ^= 1; }
                    if (lane == 0) stamp(3);
                }
            }
            if ((TRACE && (p.dbg & 4)) && lane == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 2))
                printf("tcmma cta %d: wait_tempty %.2f us, wait_full %.2f us (after the first k-block)\n", blockIdx.x,
                       wait_te / 1965.0, wait_full / 1965.0);
        }
    }
    } else {
        if constexpr (REGS) asm volatile("setmaxnreg.inc.sync.aligned.u32 224;" ::: "memory");
        // ================= epilogue: 8 warps; warp -> (TMEM lane quarter q, column half h).  Each
        // chunk partial is read from TMEM and added into fp32 registers (IEEE round-to-nearest);
        // after the tile's last chunk the fused epilogue writes the row segment to global memory.
        constexpr int HALF = BN / 2;
        const int q = warp & 3, h = (warp - 4) >> 2;
        int buf = 0;
        uint32_t buf_phase = 0;
        // 3xF16: the sum of scaled operands times s_A * s_B (powers of two: exact), and the output planes'
        // scale from their bound (every CTA computes the same value; one thread publishes it)
        float fa = 1.f, fb = 1.f, inv_so = 1.f, amx = 0.f;
        if (F16) {
            fa = p.tsA->scale;  // applied one after the other: s_A * s_B alone may leave fp32's range
            fb = p.tsB->scale;
            if (p.fo.h) {
                const float so = f16out_scale(p.fo);
                inv_so = 1.f / so;
                if (blockIdx.x == 0 && threadIdx.x == 128) p.fo.ts->scale = so;
            }
        }
        MTX_UNITS(t) {
            int z, r;
            unit_of(p, t, tiles_mn, z, r);
            const int m0 = (r / p.tiles_n) * TILE_M + m_off, n0 = (r % p.tiles_n) * BN + h * HALF;
            const int kb0 = z * p.kb_per_split, kb1 = min(p.kb_total, kb0 + p.kb_per_split);
            float acc[HALF];
            bool first = true;
            // 3xF16 dgrad with a ReLU bitmask: this tile's mask words are loaded before its accumulation (their
            // L2 latency hides behind the MMAs instead of stalling the store phase).  Word k of the rl group
            // (8 lanes) = (sub-tile k / 8, row group k % 8); lane jj holds words 2 jj and 2 jj + 1.
            // (HALF = 128: 4 sub-tiles, words 4 jj .. 4 jj + 3)
            constexpr bool PRE_BITS = F16 && MASK && !PART && (HALF == 64 || HALF == 128);
            constexpr int NW = HALF / 32;  // mask words per lane
            uint32_t mw[NW > 0 ? NW : 1];
#pragma unroll
            for (int e = 0; e < NW; e++) mw[e] = 0;
            if (PRE_BITS && p.mbits && p.splits == 1) {
                const int rl8 = (lane & 31) >> 3, j8 = lane & 7;
#pragma unroll
                for (int e = 0; e < NW; e++) {
                    const int k = NW * j8 + e, m = m0 + 32 * q + (k % 8) * 4 + rl8, nc = n0 + 32 * (k / 8);
                    uint32_t w = 0;
                    if (m < p.M && nc < p.N) w = __ldg(p.mbits + (int64_t)m * p.mbits_ld + (nc >> 5));
                    mw[e] = w;
                }
            }
            for (int c0 = kb0; c0 < kb1; c0 += L::CHUNK) {
                mbar_wait(tfull0 + 8 * buf, buf_phase);
                tc_fence_after();
                constexpr int CW = HALF >= 32 ? 32 : HALF;  // columns per tcgen05.ld
#pragma unroll
                for (int c = 0; c < HALF / CW; c++) {
                    uint32_t v[CW];
                    const uint32_t taddr = tmem_base + buf * L::ACC_COLS + ((uint32_t)(32 * q) << 16) + h * HALF + CW * c;
                    if constexpr (CW == 32) {
                        TMEM_LD32(taddr, v);
                    } else {
                        TMEM_LD16(taddr, v);
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < CW; j++)
                        acc[CW * c + j] = first ? __uint_as_float(v[j]) : __fadd_rn(acc[CW * c + j], __uint_as_float(v[j]));
                }
                first = false;
                if (warp == 4 && lane == 0) stamp(4);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {  // accumulator buffer drained (PAIR: on the leader, which issues into it)
                    if (PAIR) mbar_arrive_cluster(mapa_u32(tempty0 + 8 * buf, lead_rank));
                    else mbar_arrive(tempty0 + 8 * buf);
                }
                if (++buf == NBUF) { buf = 0; buf_phase ^= 1; }
            }
            if (F16) {
#pragma unroll
                for (int j = 0; j < HALF; j++) acc[j] = (acc[j] * fa) * fb;
            }
            if (CLU || (!FAST && !PART && p.cluster)) {  // partial tile -> own smem; folded across the cluster below
                const int row = 32 * q + lane;
#pragma unroll
                for (int j = 0; j < HALF / 4; j++)
                    *(float4 *)(smem + ktile_off<BN>(row, h * (HALF / 4) + j)) =
                        make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
                continue;
            }
            // ---- store: stage each 32-row x CW-column sub-tile in shared memory (lane = row, 16-B
            // chunks XOR-swizzled: conflict-free both ways), then the warp writes whole row segments
            // (CPR lanes per row, RPI rows per instruction) with the fused epilogue applied there.
            constexpr int SW = HALF >= 32 ? 32 : HALF;  // staged columns
            constexpr int CPR = SW / 4, RPI = 32 / CPR;
            float *stg = (float *)(smem + L::EPI_OFF) + (warp - 4) * 32 * 32;
            const int jj = lane % CPR, rl = lane / CPR;
            auto swz = [](int row, int chunk) { return (chunk ^ (row / (8 / CPR))) & (CPR - 1); };
            // 3xF16 lean outputs (direct path only): the forward's ReLU bitmask, the dgrad's per-32-row column sums
            const bool want_bits = F16 && !PART && p.fo.bits && p.splits == 1;
            const bool want_cols = F16 && !PART && p.fo.colpart && p.splits == 1;
            // 3xF16 lean fast path: a whole 32-row x 64-column piece in range, planes only (no fp32 copy, no split-K),
            // forward (bias + ReLU [+ bits]) or dgrad (bitmask [+ column sums]): no per-element bounds or mode tests
            if constexpr (F16 && !PART && (HALF == 64 || HALF == 128)) {
                // output: the fp16 planes alone (lean), or the fp32 copy alone (a layer the SIMT head consumes)
                const bool planes = p.fo.h != nullptr;
                const bool fast = FAST || p.splits == 1 && (planes ? p.fo.skip_f32 : (p.C && (p.ldc & 3) == 0 && !p.C_hi)) &&
                                  !(EXPER && (p.dbg & 1)) && m0 + 32 * q + 32 <= p.M &&
                                  n0 + HALF <= p.N && (MASK ? (p.mbits != nullptr)
                                                            : (p.epi == EPI_BIAS_RELU && ((uintptr_t)p.bias & 15) == 0));
                if (fast) {
#pragma unroll
                    for (int c = 0; c < HALF / 32; c++) {
#pragma unroll
                        for (int j = 0; j < 8; j++)
                            *(float4 *)(stg + lane * 32 + 4 * swz(lane, j)) =
                                make_float4(acc[32 * c + 4 * j], acc[32 * c + 4 * j + 1], acc[32 * c + 4 * j + 2],
                                            acc[32 * c + 4 * j + 3]);
                        __syncwarp();
                        const int n = n0 + 32 * c + 4 * jj;
                        const float4 bz = MASK ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldg((const float4 *)(p.bias + n));
                        float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int it = 0; it < 8; it++) {
                            const int r = it * 4 + rl, m = m0 + 32 * q + r;
                            const float4 sv = *(const float4 *)(stg + r * 32 + 4 * swz(r, jj));
                            float x[4] = {sv.x, sv.y, sv.z, sv.w};
                            if constexpr (MASK) {
                                const int k = 8 * c + it;
                                const uint32_t w = __shfl_sync(0xffffffffu, mw[k % NW], rl * 8 + k / NW) >> (4 * jj);
#pragma unroll
                                for (int e = 0; e < 4; e++) x[e] = ((w >> e) & 1u) ? x[e] : 0.f;
                            } else {
                                x[0] = fmaxf(x[0] + bz.x, 0.f); x[1] = fmaxf(x[1] + bz.y, 0.f);
                                x[2] = fmaxf(x[2] + bz.z, 0.f); x[3] = fmaxf(x[3] + bz.w, 0.f);
                            }
                            if (planes) {
                                amx = fmaxf(amx, fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3]))));
                                __half2 h2[2], l2[2];
#pragma unroll
                                for (int e = 0; e < 2; e++) {
                                    const float2 y = make_float2(x[2 * e] * inv_so, x[2 * e + 1] * inv_so);
                                    h2[e] = __float22half2_rn(y);
                                    const float2 hf = __half22float2(h2[e]);
                                    l2[e] = __float22half2_rn(make_float2(y.x - hf.x, y.y - hf.y));
                                }
                                const int64_t po = (int64_t)m * p.fo.ld + n;
                                *(uint2 *)(p.fo.h + po) = make_uint2(*(uint32_t *)&h2[0], *(uint32_t *)&h2[1]);
                                *(uint2 *)(p.fo.l + po) = make_uint2(*(uint32_t *)&l2[0], *(uint32_t *)&l2[1]);
                            } else {
                                *(float4 *)(p.C + (int64_t)m * p.ldc + n) = make_float4(x[0], x[1], x[2], x[3]);
                            }
                            if (!MASK && p.fo.bits) {  // the row's 32 columns sit in its 8 lanes: OR the nibbles
                                uint32_t w = ((x[0] > 0.f) | ((x[1] > 0.f) << 1) | ((x[2] > 0.f) << 2) | ((x[3] > 0.f) << 3))
                                             << (4 * jj);
                                w |= __shfl_xor_sync(0xffffffffu, w, 1);
                                w |= __shfl_xor_sync(0xffffffffu, w, 2);
                                w |= __shfl_xor_sync(0xffffffffu, w, 4);
                                if (jj == 0) p.fo.bits[(int64_t)m * p.fo.bits_ld + (n >> 5)] = w;
                            }
                            if (MASK) { cs.x += x[0]; cs.y += x[1]; cs.z += x[2]; cs.w += x[3]; }
                        }
                        if (MASK && p.fo.colpart) {  // the warp's 32 rows, fixed tree over the lanes of a column group
#pragma unroll
                            for (int o = 8; o < 32; o <<= 1) {
                                cs.x += __shfl_xor_sync(0xffffffffu, cs.x, o);
                                cs.y += __shfl_xor_sync(0xffffffffu, cs.y, o);
                                cs.z += __shfl_xor_sync(0xffffffffu, cs.z, o);
                                cs.w += __shfl_xor_sync(0xffffffffu, cs.w, o);
                            }
                            if (rl == 0) *(float4 *)(p.fo.colpart + (int64_t)((m0 + 32 * q) >> 5) * p.N + n) = cs;
                        }
                        __syncwarp();
                    }
                    continue;
                }
            }
#pragma unroll
            for (int c = 0; c < HALF / SW; c++) {
                float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int j = 0; j < CPR; j++)
                    *(float4 *)(stg + lane * SW + 4 * swz(lane, j)) =
                        make_float4(acc[SW * c + 4 * j], acc[SW * c + 4 * j + 1], acc[SW * c + 4 * j + 2],
                                    acc[SW * c + 4 * j + 3]);
                __syncwarp();
                const int n = n0 + SW * c + 4 * jj;
                const float4 bz = MASK ? make_float4(0.f, 0.f, 0.f, 0.f) : load_bias(p, n);
                constexpr int ITS = 32 / RPI;  // row groups of the sub-tile
                // dgrad: the groups' mask loads in flight together (4 fp32 masks, or all 8 words of a bitmask)
                constexpr int G4 = MASK ? (F16 ? ITS : 4) : 1;
#pragma unroll
                for (int it0 = 0; it0 < ITS; it0 += G4) {
                    float4 mk[G4];
#pragma unroll
                    for (int u = 0; u < G4; u++) {
                        const int m = m0 + 32 * q + (it0 + u) * RPI + rl;
                        if (PRE_BITS && p.mbits) {  // the preloaded word of (sub-tile c, row group it0 + u)
                            const int k = 8 * c + it0 + u;
                            const uint32_t w = __shfl_sync(0xffffffffu, mw[k % NW], rl * 8 + k / NW) >> (n & 31);
                            mk[u] = make_float4((w & 1u) ? 1.f : 0.f, (w & 2u) ? 1.f : 0.f, (w & 4u) ? 1.f : 0.f,
                                                (w & 8u) ? 1.f : 0.f);
                            continue;
                        }
                        mk[u] = (MASK && !PART && p.splits == 1 && it0 + u < ITS && m < p.M && n < p.N)
                                    ? load_mask(p, m, n)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
#pragma unroll
                    for (int u = 0; u < G4; u++) {
                        const int it = it0 + u;
                        if (it >= ITS) break;
                        const int r = it * RPI + rl;
                        const int m = m0 + 32 * q + r;
                        const float4 sv = *(const float4 *)(stg + r * SW + 4 * swz(r, jj));
                        const bool ok = m < p.M && n < p.N && !(EXPER && (p.dbg & 1));
                        if (ok && p.splits > 1) {  // split-K partial (folded with the epilogue by splitk_reduce)
                            float *dst = p.partial + ((int64_t)z * p.M + m) * p.N + n;
                            if (n + 3 < p.N) *(float4 *)dst = sv;
                            else {
                                const float o[4] = {sv.x, sv.y, sv.z, sv.w};
                                for (int e = 0; e < 4 && n + e < p.N; e++) dst[e] = o[e];
                            }
                        }
                        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (!PART && ok && p.splits == 1) o = epi_store<MASK, F16>(p, m, n, sv, mk[u], inv_so, amx, bz);
                        if (want_bits) {  // the 8 lanes of a row hold its 32 columns: OR their nibbles into one word
                            uint32_t w = ((o.x > 0.f) | ((o.y > 0.f) << 1) | ((o.z > 0.f) << 2) | ((o.w > 0.f) << 3))
                                         << (4 * jj);
                            w |= __shfl_xor_sync(0xffffffffu, w, 1);
                            w |= __shfl_xor_sync(0xffffffffu, w, 2);
                            w |= __shfl_xor_sync(0xffffffffu, w, 4);
                            if (jj == 0 && m < p.M && n < p.N) p.fo.bits[(int64_t)m * p.fo.bits_ld + (n >> 5)] = w;
                        }
                        if (want_cols) { cs.x += o.x; cs.y += o.y; cs.z += o.z; cs.w += o.w; }
                    }
                }
                if (want_cols) {  // rows of this warp's quarter, in a fixed tree over the lanes of a column group
#pragma unroll
                    for (int o = 8; o < 32; o <<= 1) {
                        cs.x += __shfl_xor_sync(0xffffffffu, cs.x, o);
                        cs.y += __shfl_xor_sync(0xffffffffu, cs.y, o);
                        cs.z += __shfl_xor_sync(0xffffffffu, cs.z, o);
                        cs.w += __shfl_xor_sync(0xffffffffu, cs.w, o);
                    }
                    if (rl == 0 && n < p.N && m0 + 32 * q < p.M) {
                        float *dst = p.fo.colpart + (int64_t)((m0 + 32 * q) >> 5) * p.N + n;
                        if (n + 3 < p.N) *(float4 *)dst = cs;
                        else {
                            const float v[4] = {cs.x, cs.y, cs.z, cs.w};
                            for (int e = 0; e < 4 && n + e < p.N; e++) dst[e] = v[e];
                        }
                    }
                }
                __syncwarp();
            }
        }
        if (F16 && !PART && p.fo.h && !p.cluster) {  // amax of the planes written (the next consumer's bound): one atomic per CTA
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
            float *red = (float *)(smem + L::EPI_OFF);  // the staging area is free once the last tile is stored
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (lane == 0) red[warp - 4] = amx;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (warp == 4 && lane == 0) {
                for (int k = 1; k < 8; k++) amx = fmaxf(amx, red[k]);
                amax_atomic(&p.fo.ts->amax, amx);
            }
        }
    }
#undef MTX_UNITS
    if (warp == 4 && lane == 0) stamp(5);
    if (CLU || (!FAST && !PART && p.cluster)) {
        // every CTA of the cluster holds its split's partial tile: CTA z folds rows
        // [z*BM/S, (z+1)*BM/S) over the splits in ascending order (deterministic) and stores them
        // with the fused epilogue; the second barrier keeps every CTA's smem alive until read
        cluster_sync_all();
        if (warp >= 4 && warp < 12) {
            float inv_so = 1.f, amx = 0.f;
            if (F16 && p.fo.h) inv_so = 1.f / f16out_scale(p.fo);
            cluster_fold<BN, MASK, PAIR, F16>(p, smem_u32(smem), inv_so, amx);
            if (F16 && p.fo.h) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
                if (lane == 0) amax_atomic(&p.fo.ts->amax, amx);
            }
        }
        cluster_sync_all();
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        stamp(6);
        if ((TRACE && (p.dbg & 4)) && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
            printf("tcts cta %d/%d t0 %llu: pdl %.2f first_full %.2f last_commit %.2f last_drain %.2f stores_done %.2f exit %.2f us\n",
                   blockIdx.x, gridDim.x, (unsigned long long)dts[0], (dts[1] - dts[0]) * 1e-3, (dts[2] - dts[0]) * 1e-3,
                   (dts[3] - dts[0]) * 1e-3, (dts[4] - dts[0]) * 1e-3, (dts[5] - dts[0]) * 1e-3, (dts[6] - dts[0]) * 1e-3);
    }
    if (PAIR) cluster_sync_all();  // both CTAs done with the pair's TMEM and barriers
    if (warp == 2) {
        tc_fence_after();
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::TMEM_COLS)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(L::TMEM_COLS)
                         : "memory");
    }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Row-major fp32 matrix [rows][cols] (row pitch ld elements), box = 32 cols x box_rows.
// K-major operands use the 128-B swizzle (16-B atoms), MN-major ones the 128-B swizzle with
// 32-B atoms, matching the UMMA descriptors above.
// f16: fp16 planes, box = 64 cols (128 B) x box_rows, the plain 128-B swizzle for both majors.
bool make_map(EncodeTiled enc, CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld,
              int box_rows, bool mn_major, bool f16 = false) {
    const int esz = f16 ? 2 : 4;
    if ((ld * esz) % 16) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)ptr, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     (mn_major && !f16) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// MN-major operand [rows][cols] (row pitch ld) as a 3-D map: dim0 = 32 elements of a 128-B chunk, dim1 = rows
// (the K index), dim2 = cols / 32 chunks (stride 128 B); box {32, BK, chunks}.  Needs cols % 32 == 0: chunks never
// run past a row (the 2-D map's zero fill is what covers a ragged cols).
// f16: chunks of 64 fp16 elements (128 B), box {64, BKH, chunks}, the plain 128-B swizzle.
bool make_map_mn3d(EncodeTiled enc, CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int64_t ld, int chunks,
                   bool f16 = false) {
    const int esz = f16 ? 2 : 4, ce = 128 / esz;
    if (cols % ce || (ld * esz) % 16) return false;
    cuuint64_t dims[3] = {(cuuint64_t)ce, (cuuint64_t)rows, (cuuint64_t)(cols / ce)};
    cuuint64_t strides[2] = {(cuuint64_t)ld * esz, 128};
    cuuint32_t box[3] = {(cuuint32_t)ce, (cuuint32_t)(f16 ? BKH : BK), (cuuint32_t)chunks};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)ptr, dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     f16 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

struct TcGemm {
    EncodeTiled encode = nullptr;
    int sms = 148;
    bool attr_set[512] = {};
    // split-K folded through distributed shared memory (MTX_TC_CLUSTER=0 disables: global partials
    // + splitk_reduce launch)
    bool cluster = true;
    int max_clusters[3][3][9] = {};  // [1x / 3xTF32 / 3xF16][BN 128/64/32][cluster size]: co-resident clusters (0 = unknown)
    int max_pair_clusters[3][9] = {};  // [1x / 3xTF32 / 3xF16][cluster size] for the 128-wide pair variant
    // CTA-pair (cta_group::2) 256 x 128 tiles for large GEMMs (MTX_TC_PAIR=0 disables)
    bool pair = true;
};

bool tc_available() { return true; }

// Tile plan, fitted to the plan sweep (tools/gemm_plan_sweep.py): problems whose
// 128-wide tiles already cover half the SMs run unsplit 128-wide tiles; smaller ones take the widest
// N tile (128, 64, 32) whose tiles x K-splits reach 3/4 of the SMs with >= 4 k-blocks per split
// (wide tiles keep the operand re-reads from L2 low; splits fill the SMs, their fold is one light
// launch).  Store-bound single-k-block GEMMs use 64-wide tiles.
TcPlan tc_plan(int sms, int M, int N, int K, bool f16) {
    TcPlan pl;
    const int tm = (M + BM - 1) / BM;
    const int kb = (K + (f16 ? BKH : BK) - 1) / (f16 ? BKH : BK);
    const int max_split = std::max(1, kb / (f16 ? 2 : 4));  // >= 128 elements of K per split
    pl.bn = 128;
    pl.splits = 1;
    if (tm * ((N + 127) / 128) * 2 >= sms) {
        if (kb <= 2 && N >= 64) pl.bn = 64;
    } else {
        for (int bn : {128, 64, 32}) {
            if (f16 && bn == 32) break;  // an MN-major fp16 operand tile is whole 64-element chunks
            const int tiles = tm * ((N + bn - 1) / bn);
            const int s = std::max(1, std::min(max_split, sms / tiles));
            pl.bn = bn;
            pl.splits = s;
            if (tiles * s * 4 >= sms * 3) break;
        }
        const int per = (kb + pl.splits - 1) / pl.splits;
        pl.splits = (kb + per - 1) / per;
    }
    // development overrides for plan sweeps (tools/gemm_plan_sweep.py), read on every call
    if (const char *e = getenv("MTX_TC_BN")) {
        const int v = atoi(e);
        if ((v == 32 && !f16) || v == 64 || v == 128) pl.bn = v;
    }
    if (const char *e = getenv("MTX_TC_SPLITS")) pl.splits = std::max(1, std::min(atoi(e), kb));
    return pl;
}

int tc_choose_splits(int sms, int M, int N, int K) {
    return std::max(tc_plan(sms, M, N, K, false).splits, tc_plan(sms, M, N, K, true).splits);
}

TcGemm *tc_create(int device) {
    TcGemm *t = new TcGemm();
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess) {
        delete t;
        return nullptr;
    }
    t->encode = (EncodeTiled)fn;
    if (const char *k = getenv("MTX_TC_CLUSTER")) t->cluster = atoi(k) != 0;
    if (const char *k = getenv("MTX_TC_PAIR")) t->pair = atoi(k) != 0;
    cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, device);
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    if (major != 10) {  // tcgen05 exists on sm_100 only
        delete t;
        return nullptr;
    }
    return t;
}

void tc_destroy(TcGemm *t) { delete t; }

static bool al16(const void *p) { return ((uintptr_t)p & 15) == 0; }

bool tc_supports(TcGemm *t, const GemmDesc &g) {
    if (!t) return false;
    const int M = g.aug ? g.M - 1 : g.M;
    if (M < 1 || g.N < 16 || g.K < 1) return false;
    if (g.lda % 4 || g.ldb % 4 || g.ldc % 4 || !al16(g.A) || !al16(g.B) || !al16(g.C)) return false;
    if (g.epi == EPI_MASK && (g.ldm % 4 || !al16(g.mask))) return false;
    // dataset operand with the sample dimension along K: its k-blocks must not run into the next rank's rows
    if (g.ta && g.arow.win && g.K % (g.f16x3 ? BKH : BK)) return false;
    if (g.tf32x3 && !(g.A_hi && g.A_lo && g.B_hi && g.B_lo)) return false;  // 3xTF32 consumes producer planes
    if (g.f16x3) {  // 3xF16: producer planes with 16-B row pitches and their scale slots
        if (!(g.A_h && g.A_l && g.B_h && g.B_l && g.tsA && g.tsB)) return false;
        if (g.lda_p % 8 || g.ldb_p % 8 || !al16(g.A_h) || !al16(g.A_l) || !al16(g.B_h) || !al16(g.B_l)) return false;
        if (g.C_h && (g.ldc_p % 4 || !g.tsC || ((uintptr_t)g.C_h & 7) || ((uintptr_t)g.C_l & 7))) return false;
        if (g.N < 64 && !g.tb) return false;  // an MN-major B tile is whole 64-element chunks
    }
    if (g.arow.win && g.a_rows_total <= 0) return false;
    return true;
}

// variant: 0 = 1xTF32, 1 = 3xTF32, 2 = 3xF16
template <int BN, bool SPLIT, bool PAIR = false, bool MASK = false, bool F16 = false, bool FAST = false, bool CLU = false,
          bool PART = false>
static cudaError_t prepare(TcGemm *t) {
    using L = SmemLayout<BN, SPLIT, PAIR, F16>;
    const int slot = (SPLIT ? 1 : 0) + 2 * (BN == 128 ? 0 : BN == 64 ? 1 : BN == 32 ? 2 : 3) + (PAIR ? 8 : 0) +
                     (MASK ? 16 : 0) + (F16 ? 32 : 0) + (FAST ? 64 : 0) + (CLU ? 128 : 0) + (PART ? 256 : 0);
    if (!t->attr_set[slot]) {
        cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, SPLIT, PAIR, MASK, F16, FAST, CLU, PART>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
        if (e != cudaSuccess) return e;
        t->attr_set[slot] = true;
    }
    return cudaSuccess;
}

// How many clusters of `cs` CTAs of this variant can be resident at once (cached).
template <int BN, bool SPLIT, bool F16>
static int co_resident_clusters(TcGemm *t, int cs) {
    using L = SmemLayout<BN, SPLIT, false, F16>;
    int &slot = t->max_clusters[F16 ? 2 : SPLIT ? 1 : 0][BN == 128 ? 0 : BN == 64 ? 1 : 2][cs];
    if (slot) return slot;
    if (prepare<BN, SPLIT, false, false, F16>(t) != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 148);
    cfg.blockDim = dim3(L::THREADS);
    cfg.dynamicSmemBytes = L::TOTAL;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void *)tc_gemm_kernel<BN, SPLIT, false, false, F16>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = -1;  // query failed: never use the cluster path for this variant
    }
    slot = n;
    return n;
}

template <int BN, bool SPLIT, bool PAIR = false, bool MASK = false, bool F16 = false, bool FAST = false, bool CLU = false,
          bool PART = false>
static cudaError_t launch(TcGemm *t, const TcParams &p, int grid, cudaStream_t s) {
    using L = SmemLayout<BN, SPLIT, PAIR, F16>;
    cudaError_t e = prepare<BN, SPLIT, PAIR, MASK, F16, FAST, CLU, PART>(t);
    if (e != cudaSuccess) return e;
    if (!p.cluster && !PAIR)
        return launch_pdl(tc_gemm_kernel<BN, SPLIT, PAIR, MASK, F16, FAST, CLU, PART>, dim3(grid), dim3(L::THREADS),
                          L::TOTAL, s, p);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(L::THREADS);
    cfg.dynamicSmemBytes = L::TOTAL;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? (p.cluster ? 2 * p.splits : p.mc ? 4 : 2) : p.splits;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, SPLIT, PAIR, MASK, F16, FAST, CLU, PART>, p);
}

// How many clusters of `cs` CTAs (cs / 2 CTA pairs) of the 128-wide pair variant can be resident at once.
template <bool SPLIT, bool F16>
static int co_resident_pair(TcGemm *t, int cs) {
    using L = SmemLayout<128, SPLIT, true, F16>;
    int &slot = t->max_pair_clusters[F16 ? 2 : SPLIT ? 1 : 0][cs];
    if (slot) return slot;
    if (prepare<128, SPLIT, true, false, F16>(t) != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 74);
    cfg.blockDim = dim3(L::THREADS);
    cfg.dynamicSmemBytes = L::TOTAL;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void *)tc_gemm_kernel<128, SPLIT, true, false, F16>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = -1;
    }
    slot = n;
    return n;
}

template <int BN>
static int co_resident(TcGemm *t, int variant, int cs) {
    return variant == 2 ? co_resident_clusters<BN, true, true>(t, cs)
         : variant == 1 ? co_resident_clusters<BN, true, false>(t, cs)
                        : co_resident_clusters<BN, false, false>(t, cs);
}
static int co_resident_pair_v(TcGemm *t, int variant, int cs) {
    return variant == 2 ? co_resident_pair<true, true>(t, cs)
         : variant == 1 ? co_resident_pair<true, false>(t, cs)
                        : co_resident_pair<false, false>(t, cs);
}

// Unpaired tiles of width BN, with or without the dgrad mask, in epilogue mode (FAST, CLU, PART).
template <bool SPLIT, bool F16, bool FAST, bool CLU, bool PART>
static cudaError_t launch_unpaired(TcGemm *t, const TcParams &p, int grid, cudaStream_t s, int BN, bool mask) {
    if (mask) {
        if (BN == 128) return launch<128, SPLIT, false, true, F16, FAST, CLU, PART>(t, p, grid, s);
        if (BN == 64) return launch<64, SPLIT, false, true, F16, FAST, CLU, PART>(t, p, grid, s);
        if constexpr (!F16) return launch<32, SPLIT, false, true, F16, FAST, CLU, PART>(t, p, grid, s);
        return cudaErrorInvalidValue;
    }
    if (BN == 128) return launch<128, SPLIT, false, false, F16, FAST, CLU, PART>(t, p, grid, s);
    if (BN == 64) return launch<64, SPLIT, false, false, F16, FAST, CLU, PART>(t, p, grid, s);
    if constexpr (!F16) return launch<32, SPLIT, false, false, F16, FAST, CLU, PART>(t, p, grid, s);
    return cudaErrorInvalidValue;
}

// One instantiation per (variant, BN, PAIR, MASK, epilogue mode) the planner can pick.  The split engines (3xTF32,
// 3xF16) get kernels specialised to the launch's epilogue -- split-K cluster fold only (CLU), split-K partials only
// (PART), whole-tile fast epilogue only (FAST, 3xF16 pairs): code a launch never runs still cost it time.
template <bool SPLIT, bool F16>
static cudaError_t launch_variant(TcGemm *t, const TcParams &p, int grid, cudaStream_t s, int BN, bool pair, bool mask,
                                  bool fast) {
    if constexpr (F16) {
        if (pair && BN == 256) {
            if (fast)
                return mask ? launch<256, SPLIT, true, true, F16, true>(t, p, grid, s)
                            : launch<256, SPLIT, true, false, F16, true>(t, p, grid, s);
            return mask ? launch<256, SPLIT, true, true, F16>(t, p, grid, s) : launch<256, SPLIT, true, false, F16>(t, p, grid, s);
        }
        if (fast && pair && BN == 128)  // every tile on the whole-tile fast epilogue
            return mask ? launch<128, SPLIT, true, true, F16, true>(t, p, grid, s)
                        : launch<128, SPLIT, true, false, F16, true>(t, p, grid, s);
        if (p.cluster && pair && BN == 128 && !mask)  // split-K clusters of pairs (the weight gradients)
            return launch<128, SPLIT, true, false, F16, false, true>(t, p, grid, s);
    }
    if constexpr (SPLIT) {
        if (p.cluster && !pair) return launch_unpaired<SPLIT, F16, false, true, false>(t, p, grid, s, BN, mask);
        if (p.splits > 1 && !p.cluster && !pair) return launch_unpaired<SPLIT, F16, false, false, true>(t, p, grid, s, BN, mask);
    }
    if (pair && mask) return launch<128, SPLIT, true, true, F16>(t, p, grid, s);
    if (pair) return launch<128, SPLIT, true, false, F16>(t, p, grid, s);
    return launch_unpaired<SPLIT, F16, false, false, false>(t, p, grid, s, BN, mask);
}

// launch == false: only the plan -- *splits_out = the K-splits the launch would use (1: the direct epilogue,
// which alone writes the 3xF16 lean outputs)
static cudaError_t tc_gemm_impl(TcGemm *t, const GemmDesc &g, cudaStream_t s, LaunchHook *h, bool launch,
                                int *splits_out) {
    const int M = g.aug ? g.M - 1 : g.M;  // the bias row of an augmented wgrad is a column sum (below)
    const int N = g.N, K = g.K;
    const int sms = g.sm_budget > 0 ? std::min(g.sm_budget, t->sms) : t->sms;
    const bool f16 = g.f16x3 != 0;
    const int variant = f16 ? 2 : g.tf32x3 ? 1 : 0;
    const int KBE = f16 ? BKH : BK;  // elements per k-block
    const TcPlan plan = tc_plan(sms, M, N, K, f16);
    int BN = plan.bn;
    // CTA pairs for large unsplit GEMMs: a 256 x 128 tile per pair halves B's per-SM operand traffic.
    // Pair MMAs also cost ~65 cycles with fresh operand tiles where a 1-CTA MMA of any N <= 128 costs ~89
    // (tools/mma_rate.cu, profiles/round2_tcgen05_rates.md); the dgrad pairs too (measured 84.0 -> 81.6 us at
    // M = 8192, 44.4 -> 43.1 at 4096).  Development knob MTX_TC_PAIR_MASK=0 unpairs the dgrad.  A weight gradient
    // too small to fill the pairs splits K over the pairs of one cluster, folded through DSMEM (below).
    static const bool pair_mask = !getenv("MTX_TC_PAIR_MASK") || atoi(getenv("MTX_TC_PAIR_MASK"));
    static const int pair_split_env = getenv("MTX_TC_PAIR_SPLIT") ? atoi(getenv("MTX_TC_PAIR_SPLIT")) : -1;
    const int64_t ptiles = (int64_t)((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
    int pair_splits = 1;
    bool pair = t->pair && (g.epi != EPI_MASK || pair_mask) && BN == 128 && N % 64 == 0 && M > BM;
    bool pair_cluster = false;
    if (pair && !(plan.splits == 1 && ptiles * 2 >= sms / 2)) {
        pair = false;
        const int kb = (K + KBE - 1) / KBE;
        // default: the long weight gradients (K >= 8192: 87.1 -> 84.9 us at 1024 x 1024 x 8192; no gain at
        // K <= 4096, tools/gemm3x_bench.py); MTX_TC_PAIR_SPLIT=0/1 forces it off/on
        const bool pair_split = pair_split_env >= 0 ? pair_split_env != 0 : kb * KBE >= 8192;
        if (pair_split && g.epi == EPI_STORE && M >= 2 * BM) {
            // a weight gradient too small to fill the pairs: split K over S pairs of one cluster (2S CTAs),
            // folded through distributed shared memory like the 1-CTA cluster plan
            const int sp = (int)std::min<int64_t>(std::min(4, std::max(1, kb * KBE / 256)), std::max<int64_t>(1, (sms / 2) / ptiles));
            if (sp > 1 && ptiles * sp * 8 >= (int64_t)(sms / 2) * 6) {
                const int nc = co_resident_pair_v(t, variant, 2 * sp);
                if (t->cluster && nc >= ptiles) {
                    pair = true;
                    pair_splits = sp;
                    pair_cluster = true;
                } else if (g.partial) {
                    pair = true;  // split-K through global partials
                    pair_splits = sp;
                }
            }
        }
    }
    // 3xF16 unsplit pairs with enough 256-wide tiles to fill the SMs: 256 x 256 pair tiles (N = 256 MMAs).  Half the
    // B bytes per flop: each 64 KB stage carries 2x the MMA time of a 48 KB one, so the 3-deep ring covers the L2/HBM
    // latency the 4-deep 128-wide ring did not (the MMA phase waited on operands ~20 % of the time)
    // Development knob MTX_TC_BN256=1: correct, measured slower (cfg4 forward 47.5 -> 51.4 us, dgrad 44.8 -> 46.8: 1.73
    // rounds of 256-wide tiles run as 2, and each tile's store phase doubles behind a 2-deep TMEM ring)
    static const int bn256_env = getenv("MTX_TC_BN256") ? atoi(getenv("MTX_TC_BN256")) : 0;
    // MTX_TC_BN256=2: whenever the shape allows (development: with the FAST 256-wide kernel)
    if (f16 && pair && !pair_cluster && pair_splits == 1 && BN == 128 && N % 256 == 0 &&
        ((bn256_env == 1 && (int64_t)((M + 2 * BM - 1) / (2 * BM)) * (N / 256) * 2 >= sms) || bn256_env == 2))
        BN = 256;
    TcParams p{};
    p.M = M; p.N = N; p.K = K;
    p.a_mn = g.ta ? 1 : 0;
    p.b_mn = g.tb ? 0 : 1;  // B stored [K][N] (tb == false) is MN-major
    // operand A: K-major [M rows][K] or MN-major stored [K rows][M]; the dataset operand's tensor map
    // spans the whole wrap-extended buffer (rows are offset on the device by a_win + a_base).
    const int64_t a_rows_total = g.a_rows_total;
    bool ok;
    // MN-major operands with whole 32-element chunks take the 3-D map (one TMA operation per operand tile)
    static const bool mn3d = !getenv("MTX_TC_MN3D") || atoi(getenv("MTX_TC_MN3D"));
    // operand row pitches (3xF16: the planes' own pitch) and elements per MN-major chunk
    const int64_t lda = f16 ? g.lda_p : g.lda, ldb = f16 ? g.ldb_p : g.ldb;
    const int CHE = f16 ? 64 : 32;
    p.a_3d = (mn3d && g.ta && M % CHE == 0 && lda % 4 == 0) ? 1 : 0;
    p.b_3d = (mn3d && !g.tb && N % CHE == 0 && ldb % 4 == 0 && BN % CHE == 0 && (!pair || (BN / 2) % CHE == 0)) ? 1 : 0;
    auto map_a = [&](CUtensorMap *m, const void *ptr) {
        if (p.a_3d) return make_map_mn3d(t->encode, m, ptr, g.arow.win ? a_rows_total : K, M, lda, BM / CHE, f16);
        return !g.ta ? make_map(t->encode, m, ptr, g.arow.win ? a_rows_total : M, K, lda, BM, false, f16)
                     : make_map(t->encode, m, ptr, g.arow.win ? a_rows_total : K, M, lda, KBE, true, f16);
    };
    auto map_b = [&](CUtensorMap *m, const void *ptr) {
        if (p.b_3d) return make_map_mn3d(t->encode, m, ptr, K, N, ldb, (pair ? BN / 2 : BN) / CHE, f16);
        return g.tb ? make_map(t->encode, m, ptr, N, K, ldb, pair ? BN / 2 : BN, false, f16)   // [N][K], K-major
                    : make_map(t->encode, m, ptr, K, N, ldb, KBE, true, f16);   // [K][N], MN-major
    };
    if (f16) ok = map_a(&p.ta, g.A_h) && map_a(&p.ta_lo, g.A_l) && map_b(&p.tb, g.B_h) && map_b(&p.tb_lo, g.B_l);
    else if (g.tf32x3) ok = map_a(&p.ta, g.A_hi) && map_a(&p.ta_lo, g.A_lo) && map_b(&p.tb, g.B_hi) && map_b(&p.tb_lo, g.B_lo);
    else ok = map_a(&p.ta, g.A) && map_b(&p.tb, g.B);
    if (!ok) return cudaErrorInvalidValue;
    p.C_hi = g.C_hi;
    p.C_lo = g.C_lo;
    if (f16) {
        p.tsA = g.tsA;
        p.tsB = g.tsB;
        if (g.C_h) {
            p.fo.h = g.C_h;
            p.fo.l = g.C_l;
            p.fo.ld = g.ldc_p;
            p.fo.ts = g.tsC;
            p.fo.a = g.tsA;
            p.fo.b = g.tsB;
            p.fo.k = g.bnd_k;
            p.fo.bias = g.bnd_bias;
        }
        // lean outputs (direct epilogue only; the caller checks tc_direct first)
        p.fo.skip_f32 = g.skip_c32;
        p.fo.bits = g.relu_bits;
        p.fo.bits_ld = g.relu_bits_ld;
        p.fo.colpart = g.colpart;
        p.mbits = g.mask_bits;
        p.mbits_ld = g.mask_bits_ld;
    }
    p.a_win = g.arow.win;
    p.a_base = g.arow.base;
    p.tiles_m = pair ? (M + 2 * BM - 1) / (2 * BM) : (M + BM - 1) / BM;
    p.tiles_n = (N + BN - 1) / BN;
    p.kb_total = (K + KBE - 1) / KBE;
    const int tiles = p.tiles_m * p.tiles_n;
    int splits = pair ? pair_splits : plan.splits;
    // split-K fold through DSMEM when the tile's splits fit one cluster and all clusters are co-resident
    bool cluster = pair_cluster;
    if (splits > 1 && splits <= 8 && t->cluster && !pair) {
        const int per = (p.kb_total + splits - 1) / splits;
        const int sp = (p.kb_total + per - 1) / per;
        const int nc = BN == 128 ? co_resident<128>(t, variant, sp)
                     : BN == 64  ? co_resident<64>(t, variant, sp)
                                 : co_resident<32>(t, variant, sp);
        if (sp > 1 && nc >= tiles) {
            cluster = true;
            splits = sp;
        }
    }
    if (!cluster) {
        if (!g.partial || N % 4) splits = 1;
        while (splits > 1 && (int64_t)splits * M * N > g.partial_cap) splits--;
    }
    p.kb_per_split = (p.kb_total + splits - 1) / splits;
    splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
    if (splits == 1) cluster = false;
    p.splits = splits;
    p.cluster = cluster ? 1 : 0;
    if (splits_out) *splits_out = splits;
    if (!launch) return cudaSuccess;
    if (const char *k = getenv("MTX_TC_DBG")) p.dbg = atoi(k);  // development timing knob (trace / experiment builds)
    // L2 prefetch distance: one ring ahead of the loads (development knob MTX_TC_PF: 0 disables, n = distance)
    static const int pf_env = getenv("MTX_TC_PF") ? atoi(getenv("MTX_TC_PF")) : -1;
    p.pf = (EXPER && pf_env >= 0) ? pf_env : 0;  // measured slower at 4 and 8 (cfg4 506 -> 635 / 608 us/step): off
    // development knob MTX_TC_PFB=1: measured slightly slower (cfg4 525.3 -> 529.5 us/step)
    static const int pfb_env = getenv("MTX_TC_PFB") ? atoi(getenv("MTX_TC_PFB")) : 0;
    p.pfb = (EXPER && pfb_env && !g.ta) ? 1 : 0;  // forward / dgrad (B = weights); a weight gradient's B is the fresh dZ
    p.epi = g.epi;
    p.bias = g.bias;
    p.mask = g.mask;
    p.ldm = g.ldm;
    p.C = g.C;
    p.ldc = g.ldc;
    p.partial = g.partial;
    const int total = tiles * splits;
    int grid = cluster ? (pair ? 2 * total : total) : pair ? 2 * std::min(total, sms / 2) : std::min(total, sms);
    // 3xF16 CTA pairs, unsplit, K-major A, an even number of N tiles: clusters of two pairs on adjacent N tiles load
    // each A plane once and multicast it (a third less L2 -> SM traffic).  Development knob MTX_TC_MC=1: measured no
    // faster (cfg4 forward 44.5 -> 45.8 us) -- the MMA phase is bound by shared-memory bandwidth (TMA writes ~62 B/clk
    // + MMA operand reads ~92 B/clk per SM against 128 B/clk), not by L2 delivery
    static const int mc_env = getenv("MTX_TC_MC") ? atoi(getenv("MTX_TC_MC")) : 0;
    if (EXPER && f16 && pair && !cluster && splits == 1 && !p.a_mn && p.tiles_n % 2 == 0 && sms >= t->sms && mc_env == 1) {
        const int nc = co_resident_pair_v(t, variant, 4);
        if (nc >= 2) {
            p.mc = 1;
            grid = 4 * std::min(nc, total / 2);
        }
    }
    const char *kind = g.epi == EPI_MASK ? "dgrad" : (g.ta ? "wgrad" : "fwd");
    char name[96];
    snprintf(name, sizeof name, "gemm_tc%s_%s[M=%d,N=%d,K=%d,splits=%d,cluster=%d,pair=%d,bn=%d%s]",
             f16 ? "3xf16" : g.tf32x3 ? "3x" : "",
             kind, M, N, K, splits, cluster ? 1 : 0, pair ? 1 : 0, BN, p.mc ? ",mc=1" : "");
    if (h) h->before(name, s);
    cudaError_t e;
    const bool mask = g.epi == EPI_MASK;  // dgrad: the masked-epilogue instantiation
    // 3xF16: every tile whole and on the fast epilogue (the kernel's `fast` test holds for all of them)
    const bool fast_all = f16 && splits == 1 && !cluster && !(EXPER && p.dbg) && M % (pair ? 2 * BM : BM) == 0 &&
                          N % BN == 0 && (p.fo.h ? p.fo.skip_f32 != 0 : (p.C && (p.ldc & 3) == 0 && !p.C_hi)) &&
                          (mask ? p.mbits != nullptr : (p.epi == EPI_BIAS_RELU && ((uintptr_t)p.bias & 15) == 0));
    e = variant == 2 ? launch_variant<true, true>(t, p, grid, s, BN, pair, mask, fast_all)
      : variant == 1 ? launch_variant<true, false>(t, p, grid, s, BN, pair, mask, false)
                     : launch_variant<false, false>(t, p, grid, s, BN, pair, mask, false);
    if (h) h->after(name, s);
    if (e != cudaSuccess) return e;
    if (splits > 1 && !cluster) {  // fold with the epilogue in a separate kernel
        e = splitk_reduce(g.partial, splits, M, N, g.C, g.ldc, s, h, g.epi, g.bias, g.mask, g.ldm, g.C_hi, g.C_lo, p.fo,
                          g.mask_bits, g.mask_bits_ld);
        if (e != cudaSuccess) return e;
    }
    if (g.aug && !g.colsum_external)  // bias gradient row: db[n] = sum_k B[k][n]  (the ones row of augmented A)
        e = colsum(g.B, K, N, g.ldb, g.C + (int64_t)M * g.ldc, g.partial, g.partial_cap, g.counters + 256, s, h);
    return e;
}

cudaError_t tc_gemm(TcGemm *t, const GemmDesc &g, cudaStream_t s, LaunchHook *h) {
    return tc_gemm_impl(t, g, s, h, true, nullptr);
}

bool tc_direct(TcGemm *t, const GemmDesc &g) {
    int splits = 0;
    return tc_gemm_impl(t, g, nullptr, nullptr, false, &splits) == cudaSuccess && splits == 1;
}

}  // namespace mtx
