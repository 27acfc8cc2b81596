// mma_rate.cu -- tcgen05 MMA throughput calibration (development tool, not the product).
// Every CTA (one per SM, or one CTA pair per TPC) issues R back-to-back k-blocks of tcgen05.mma on
// shared-memory operand tiles that never change (contents irrelevant), committing to an mbarrier per
// k-block and waiting only at the end.  Reports the achieved MMA rate: cycles per instruction per SM and
// the chip's dense TFLOP/s for kind::tf32 (K = 8) and kind::f16 (bf16, K = 16) at N = 64/128/256,
// cta_group::1 (M = 128) and ::2 (M = 256 per pair).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k(uint32_t addr) {  // K-major SWIZZLE_128B, SBO = 1024 B
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ int g_rot = 0;

template <int PAIR, int F16>
__global__ void rate(int N, int R, unsigned long long *cycles, int commit_every) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sa = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, kbar[8];
    __shared__ uint32_t tslot;
    uint32_t rank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    // stages of (A 16 KB + B 32 KB); commit_every >= 2 rotates over that many stages
    const int nst = commit_every > 1 ? commit_every : 1;
    for (int i = threadIdx.x; i < nst * 49152 / 4; i += blockDim.x) ((uint32_t *)sa)[i] = 0x3c003c00u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        for (int i = 0; i < 8; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&kbar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (PAIR) csync();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    const uint32_t M = PAIR ? 256 : 128;
    // tf32: a=b=2 (bits 7, 10); f16 with bf16 inputs: a=b=1; D f32 (bit 4)
    const uint32_t idesc = (1u << 4) | ((F16 ? 1u : 2u) << 7) | ((F16 ? 1u : 2u) << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((M >> 4) << 24);
    long long t0 = clock64();
    if (threadIdx.x == 0 && rank == 0) {
        for (int r = 0; r < R; r++) {
            const uint32_t st = smem_u32(sa) + (uint32_t)(r % nst) * 49152u, s0 = smem_u32(sa);
            // which operand rotates: R >= 0 both; rot_only (global) 1: A only, 2: B only
            const uint64_t ad = desc_k(g_rot == 2 ? s0 : st), bd = desc_k((g_rot == 1 ? s0 : st) + 16384);
            for (int kk = 0; kk < 4; kk++) {
                const uint32_t acc = (r | kk) ? 1u : 0u;
                if (PAIR) {
                    if (F16)
                        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                     "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc));
                    else
                        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                     "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc));
                } else {
                    if (F16)
                        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                     "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc));
                    else
                        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                                     "l"(ad + 2 * kk), "l"(bd + 2 * kk), "r"(idesc), "r"(acc));
                }
            }
            if (commit_every && !PAIR)  // per-k-block commit to one of 8 ring barriers (never waited here)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 smem_u32(&kbar[r & 7]))
                             : "memory");
        }
        if (PAIR)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                             smem_u32(&bar)),
                         "h"((uint16_t)3)
                         : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                         : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}\n"
                     : "=r"(done)
                     : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (PAIR) csync();
    if (threadIdx.x < 32) {
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

template <int PAIR, int F16>
void run(int N, int R, int commit_every = 0) {
    const int grid = 148;
    unsigned long long *dc, hc[148];
    cudaMalloc(&dc, sizeof hc);
    const int smem = (commit_every > 1 ? commit_every : 1) * 49152 + 2048;
    cudaFuncSetAttribute(rate<PAIR, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 2; it++) {  // warm-up, then timed
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, rate<PAIR, F16>, N, R, dc, commit_every);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return;
        }
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < grid; i++) mx = hc[i] > mx ? hc[i] : mx;
    const double instr = 4.0 * R;  // per CTA (per pair when PAIR)
    const double flop = 2.0 * (PAIR ? 256 : 128) * N * (F16 ? 16 : 8) * instr * (PAIR ? grid / 2 : grid);
    printf("%s%-5s %s N=%3d: %7.1f cycles/MMA (issuing SM)  %8.1f TFLOP/s dense (event %.3f ms)\n",
           commit_every ? "commit/kblock " : "", F16 ? "bf16" : "tf32",
           PAIR ? "pair M=256" : "1cta M=128", N, (double)mx / instr, flop / (ms * 1e-3) / 1e12, ms);
    cudaFree(dc);
}

int main(int argc, char **argv) {
    const int R = 20000;
    if (argc > 1) {  // small-N and pair rates with distinct operand tiles (round 2: conv / N = 256 plans)
        printf("rotating both over 4 stages:\n");
        for (int N : {16, 32, 64}) run<0, 0>(N, R, 4);
        run<1, 0>(128, R, 4);
        run<1, 0>(256, R, 4);
        run<1, 0>(64, R, 4);
        run<1, 1>(128, R, 4);  // kind::f16 pairs (the 3xF16 engine's tile)
        run<1, 1>(256, R, 4);
        run<0, 1>(128, R, 4);
        run<0, 1>(64, R, 4);
        return 0;
    }
    for (int N : {64, 128, 256}) {
        run<0, 0>(N, R);
        run<0, 1>(N, R);
        run<1, 0>(N, R);
        run<1, 1>(N, R);
    }
    run<0, 0>(128, R, 1);
    run<0, 0>(64, R, 1);
    printf("rotating over 4 stages (distinct smem operand tiles):\n");
    for (int rot = 1; rot <= 2; rot++) {
        cudaMemcpyToSymbol(g_rot, &rot, 4);
        printf("  rotating %s only:\n", rot == 1 ? "A" : "B");
        run<0, 0>(128, R, 4);
        run<0, 0>(64, R, 4);
        run<0, 0>(256, R, 4);
    }
    int zero = 0;
    cudaMemcpyToSymbol(g_rot, &zero, 4);
    printf("  rotating both:\n");
    run<0, 0>(128, R, 4);
    run<0, 1>(128, R, 4);
    run<0, 0>(64, R, 4);
    run<0, 0>(256, R, 4);
    return 0;
}
