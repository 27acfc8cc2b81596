// tc_probe.cu -- standalone single-tile tcgen05 probe (development tool, not the product).
// One CTA: fill a 128x32 A tile and a 128x32 B tile in shared memory in the
// UMMA SWIZZLE_128B canonical layouts (K-major or MN-major, written by hand),
// issue 4 x tcgen05.mma.kind::tf32 (K = 8 each), read the 128x128 accumulator
// back with tcgen05.ld.32x32b and compare with a CPU product.  Also probes how
// the tensor core rounds fp32 operands to TF32 (reading A12).
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
// MN-major SWIZZLE_128B_BASE32B (Swizzle<2,5,2> on byte addresses): 128-B rows along MN,
// 32-B chunk index XOR (row % 4)
__device__ __forceinline__ uint32_t swz32(uint32_t row, uint32_t col_word) {
    uint32_t chunk = col_word >> 3, w = col_word & 7;
    return row * 128 + (((chunk ^ (row & 3)) << 5) | (w << 2));
}

// byte offset of element (row r, 16B-chunk c, word w) in a 128B-swizzled atom stack (rows of 128 B)
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t col_word) {
    uint32_t chunk = col_word >> 2, w = col_word & 3;
    return row * 128 + (((chunk ^ (row & 7)) << 4) | (w << 2));
}

// A: M=128 x K=32; B: N=128 x K=32 (logical).  a_mn/b_mn pick the smem layout.
__global__ void probe(const float *A, const float *B, float *D, int a_mn, int b_mn, uint32_t lbo_k, int variant) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *sa = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint8_t *sb = sa + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    int tid = threadIdx.x;
    // fill A
    for (int e = tid; e < 128 * 32; e += blockDim.x) {
        int m = e / 32, k = e % 32;
        float v = A[m * 32 + k];
        uint32_t off;
        if (!a_mn) off = swz(m, k);                   // K-major: row m holds 32 k (128 B); 8-row atoms 1024 B
        else off = (m / 32) * 4096 + swz32(k, m % 32);  // MN-major: chunk (m/32): row k holds 32 m
        *(float *)(sa + off) = v;
    }
    for (int e = tid; e < 128 * 32; e += blockDim.x) {
        int n = e / 32, k = e % 32;
        float v = B[n * 32 + k];
        uint32_t off;
        if (!b_mn) off = swz(n, k);
        else off = (n / 32) * 4096 + swz32(k, n % 32);
        *(float *)(sb + off) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t tmem = tslot;
    if (tid == 0) {
        uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
                         ((128u >> 3) << 17) | ((128u >> 4) << 24);
        for (int kk = 0; kk < 4; kk++) {
            uint64_t ad = a_mn ? smem_desc(smem_u32(sa) + kk * 1024, 4096, 512, 1)
                               : smem_desc(smem_u32(sa) + kk * 32, lbo_k, 1024);
            uint64_t bd = b_mn ? smem_desc(smem_u32(sb) + kk * 1024, 4096, 512, 1)
                               : smem_desc(smem_u32(sb) + kk * 32, lbo_k, 1024);
            if (variant == 1 && a_mn) ad = smem_desc(smem_u32(sa) + kk * 1024, 512, 4096, 1);
            if (variant == 1 && b_mn) bd = smem_desc(smem_u32(sb) + kk * 1024, 512, 4096, 1);
            uint32_t acc = kk > 0;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                    tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    // wait
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}\n"
                     : "=r"(done)
                     : "r"(smem_u32(&bar)));
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int warp = tid >> 5, lane = tid & 31;
    if (warp < 4) {
        for (int c = 0; c < 128; c += 8) {
            uint32_t r[8];
            uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + c;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                           "=r"(r[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 8; j++) D[(32 * warp + lane) * 128 + c + j] = __uint_as_float(r[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

static float tf32_trunc(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    memcpy(&x, &u, 4);
    return x;
}
static float tf32_rne(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    uint32_t lsb = (u >> 13) & 1;
    u += 0xFFF + lsb;
    u &= 0xFFFFE000u;
    memcpy(&x, &u, 4);
    return x;
}

int main() {
    const int n = 128 * 32;
    float *hA = (float *)malloc(4 * n), *hB = (float *)malloc(4 * n), *hD = (float *)malloc(4 * 128 * 128);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, 4 * n);
    cudaMalloc(&dB, 4 * n);
    cudaMalloc(&dD, 4 * 128 * 128);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    srand(1);
    for (int i = 0; i < n; i++) {
        hA[i] = (float)((rand() % 2001) - 1000) / 256.0f;  // exactly representable in tf32? 11 bits -> not always
        hB[i] = (float)((rand() % 201) - 100) / 64.0f;
    }
    cudaMemcpy(dA, hA, 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 4 * n, cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 2; variant++)
        for (int a_mn = 0; a_mn < 2; a_mn++)
            for (int b_mn = 0; b_mn < 2; b_mn++) {
                cudaMemset(dD, 0xFF, 4 * 128 * 128);
                probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, a_mn, b_mn, 16, variant);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(hD, dD, 4 * 128 * 128, cudaMemcpyDeviceToHost);
                double maxerr = 0, maxref = 0, maxerr_t = 0, maxerr_r = 0;
                for (int m = 0; m < 128; m++)
                    for (int nn = 0; nn < 128; nn++) {
                        double s = 0, st = 0, sr = 0;
                        for (int k = 0; k < 32; k++) {
                            s += (double)hA[m * 32 + k] * hB[nn * 32 + k];
                            st += (double)tf32_trunc(hA[m * 32 + k]) * tf32_trunc(hB[nn * 32 + k]);
                            sr += (double)tf32_rne(hA[m * 32 + k]) * tf32_rne(hB[nn * 32 + k]);
                        }
                        double g = hD[m * 128 + nn];
                        maxerr = fmax(maxerr, fabs(g - s));
                        maxerr_t = fmax(maxerr_t, fabs(g - st));
                        maxerr_r = fmax(maxerr_r, fabs(g - sr));
                        maxref = fmax(maxref, fabs(s));
                    }
                printf("variant %d a_mn %d b_mn %d: err %s | max|ref| %.3f  err_vs_exact %.3e  vs_trunc %.3e  vs_rne %.3e  D[0]=%g D[1,0]=%g\n",
                       variant, a_mn, b_mn, cudaGetErrorString(e), maxref, maxerr, maxerr_t, maxerr_r, hD[0], hD[128]);
            }
    // TF32 rounding microtest (A12): A row 0 = x in k=0, B = 1 in k=0 -> D[0][0] = tf32(x)
    float xs[] = {1.0f + 0x1p-11f + 0x1p-12f, 1.0f + 0x1p-11f, 1.0f + 0x1p-12f, 1.0f + 0x1p-11f + 0x1p-23f,
                  1.0f + 3 * 0x1p-11f, -(1.0f + 0x1p-11f + 0x1p-12f)};
    for (float x : xs) {
        memset(hA, 0, 4 * n);
        memset(hB, 0, 4 * n);
        hA[0] = x;
        hB[0] = 1.0f;
        cudaMemcpy(dA, hA, 4 * n, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, 4 * n, cudaMemcpyHostToDevice);
        probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, 0, 0, 16, 0);
        cudaDeviceSynchronize();
        float d0;
        cudaMemcpy(&d0, dD, 4, cudaMemcpyDeviceToHost);
        printf("tf32 probe x=%.10f -> %.10f  (trunc %.10f, rne %.10f)\n", x, d0, tf32_trunc(x), tf32_rne(x));
    }
    return 0;
}
