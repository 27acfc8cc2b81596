// tc_pair_probe.cu -- standalone CTA-pair tcgen05 probe (development tool, not the product).
// A cluster of 2 CTAs computes D[256 x N] = A[256 x 32] . B[N x 32]^T with tcgen05.mma.cta_group::2
// (M = 256, kind::tf32, K-major SWIZZLE_128B operands written by hand):
//   CTA r holds A rows [128 r, 128 r + 128) in its shared memory;
//   mode 0: CTA r holds B rows (N columns of the product) [N/2 r, N/2 r + N/2)   (split-B hypothesis)
//   mode 1: both CTAs hold all N rows of B
// The leader (rank 0) issues the MMAs, commits with a multicast arrive to both CTAs' mbarriers; each CTA
// reads its 128 TMEM lanes x N columns back.  Every spin is bounded by %globaltimer.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t type = 2) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)type << 61;
    return d;
}
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t col_word) {
    uint32_t chunk = col_word >> 2, w = col_word & 3;
    return row * 128 + (((chunk ^ (row & 7)) << 4) | (w << 2));
}
// MN-major SWIZZLE_128B_BASE32B: 128-B rows along MN (32 elements), 32-B chunk XOR (row % 4)
__device__ __forceinline__ uint32_t swz32(uint32_t row, uint32_t col_word) {
    uint32_t chunk = col_word >> 3, w = col_word & 7;
    return row * 128 + (((chunk ^ (row & 3)) << 5) | (w << 2));
}
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void pair_probe(const float *A, const float *B, float *D, int N, int mode, int a_mn, int b_mn, int *status) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sa = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t *sb = sa + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int tid = threadIdx.x;
    for (int e = tid; e < 128 * 32; e += blockDim.x) {
        const int m = e / 32, k = e % 32;
        *(float *)(sa + (a_mn ? (m / 32) * 4096 + swz32(k, m % 32) : swz(m, k))) = A[(128 * rank + m) * 32 + k];
    }
    const int nb = mode == 0 ? N / 2 : N, n0 = mode == 0 ? (N / 2) * rank : 0;
    for (int e = tid; e < nb * 32; e += blockDim.x) {
        const int n = e / 32, k = e % 32;
        *(float *)(sb + (b_mn ? (n / 32) * 4096 + swz32(k, n % 32) : swz(n, k))) = B[(n0 + n) * 32 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();  // both CTAs' operands, barriers and TMEM ready
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (rank == 0 && tid == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
                               ((uint32_t)(N >> 3) << 17) | ((256u >> 4) << 24);
        for (int kk = 0; kk < 4; kk++) {
            const uint64_t ad = a_mn ? smem_desc(smem_u32(sa) + kk * 1024, 4096, 512, 1)
                                     : smem_desc(smem_u32(sa) + kk * 32, 16, 1024);
            const uint64_t bd = b_mn ? smem_desc(smem_u32(sb) + kk * 1024, 4096, 512, 1)
                                     : smem_desc(smem_u32(sb) + kk * 32, 16, 1024);
            const uint32_t acc = kk > 0;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                    tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        const uint16_t mask = 3;
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"(mask)
            : "memory");
    }
    uint32_t done = 0;
    const uint64_t t0 = gtimer();
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}\n"
                     : "=r"(done)
                     : "r"(smem_u32(&bar)));
        if (!done && gtimer() - t0 > 2000000000ull) {
            if (tid == 0) atomicOr(status, 1 << rank);
            break;
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int warp = tid >> 5, lane = tid & 31;
    if (done && warp < 4) {
        for (int c = 0; c < N; c += 8) {
            uint32_t r[8];
            const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + c;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                           "=r"(r[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 8; j++) D[(128 * rank + 32 * warp + lane) * N + c + j] = __uint_as_float(r[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync();  // peer done reading before the pair's TMEM is released
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

static float tf32_trunc(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    memcpy(&x, &u, 4);
    return x;
}

int main() {
    const int N = 128;
    float *hA = (float *)malloc(4 * 256 * 32), *hB = (float *)malloc(4 * N * 32), *hD = (float *)malloc(4 * 256 * N);
    float *dA, *dB, *dD;
    int *dS;
    cudaMalloc(&dA, 4 * 256 * 32);
    cudaMalloc(&dB, 4 * N * 32);
    cudaMalloc(&dD, 4 * 256 * N);
    cudaMalloc(&dS, 4);
    srand(3);
    for (int i = 0; i < 256 * 32; i++) hA[i] = (float)((rand() % 2001) - 1000) / 256.0f;
    for (int i = 0; i < N * 32; i++) hB[i] = (float)((rand() % 201) - 100) / 64.0f;
    cudaMemcpy(dA, hA, 4 * 256 * 32, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 4 * N * 32, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(pair_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    for (int combo = 0; combo < 5; combo++) {
        const int mode = combo == 4 ? 1 : 0, a_mn = combo & 1, b_mn = (combo >> 1) & 1;
        cudaMemset(dD, 0xFF, 4 * 256 * N);
        cudaMemset(dS, 0, 4);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = 40 * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, pair_probe, (const float *)dA, (const float *)dB, dD, N, mode, a_mn, b_mn,
                                           dS);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        int st = -1;
        cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(hD, dD, 4 * 256 * N, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0;
        int bad_rows_lo = 0, bad_rows_hi = 0;
        for (int m = 0; m < 256; m++)
            for (int n = 0; n < N; n++) {
                double s = 0;
                for (int k = 0; k < 32; k++) s += (double)tf32_trunc(hA[m * 32 + k]) * tf32_trunc(hB[n * 32 + k]);
                const double err = fabs(hD[m * N + n] - s);
                if (err > 1e-3 * (1 + fabs(s))) (m < 128 ? bad_rows_lo : bad_rows_hi)++;
                maxerr = fmax(maxerr, err);
                maxref = fmax(maxref, fabs(s));
            }
        printf("a_mn %d b_mn %d mode %d (%s): launch %s, timeout-bits %d, max|ref| %.2f, max err %.3e, bad elems rows<128: %d, rows>=128: %d\n",
               a_mn, b_mn, mode, mode == 0 ? "B split by N halves" : "B full in both CTAs", cudaGetErrorString(e), st, maxref,
               maxerr, bad_rows_lo, bad_rows_hi);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
