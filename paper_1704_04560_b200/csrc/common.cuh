// common.cuh -- internal helpers of libmtx (product path; independent of oracle/).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#define MTX_DEVI __device__ __forceinline__

namespace mtx {

// SplitMix64 output k of a generator seeded with key (Steele, Lea, Flood 2014):
// the counter-based generator both sides of the parity check implement on their own.
MTX_DEVI uint64_t splitmix64(uint64_t key, uint64_t k) {
    uint64_t z = key + (k + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// First sample row of this rank's slice of the current global-batch window.
// `win` points at the device-resident window start s_t = (t*B) mod n (O4), which
// the last kernel of each step advances; the dataset buffer is wrap-extended by
// B rows, so the slice is rows [row0, row0 + b) contiguously.  win == nullptr
// means the rows are staged at offset 0 (host-input path).
struct RowSel {
    const int64_t *win;
    int64_t base;  // rank * b
    MTX_DEVI int64_t row0() const { return win ? (*win + base) : 0; }
};

// 3xTF32 operand planes: hi = x rounded to nearest TF32, lo = (x - hi) rounded to nearest TF32
// (x - hi is exact in fp32).  hi + lo represents x to ~2^-22 relative, and both round-to-nearest
// parts are sign-symmetric, so the dropped lo.lo product carries no bias.
MTX_DEVI uint32_t rne_tf32_bits(uint32_t u) { return (u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u; }
MTX_DEVI void split_tf32(float x, float &hi, float &lo) {
    const uint32_t h = rne_tf32_bits(__float_as_uint(x));
    hi = __uint_as_float(h);
    lo = __uint_as_float(rne_tf32_bits(__float_as_uint(x - hi)));
}

// 3xF16 operand planes: x = s * (hi + lo) with s = 2^e a per-tensor power of two,
// hi = rn_f16(x / s), lo = rn_f16(x / s - hi).  fp16 has TF32's 11-bit significand, so hi + lo carries
// x to ~2^-22 relative exactly like the 3xTF32 planes; the power-of-two scale only moves the exponent
// into fp16's range and is undone exactly in the consuming GEMM's epilogue.  One slot per tensor:
//   amax  -- max |x| of the tensor's current values (exact when written by quantize_f16; accumulated
//            with atomicMax by GEMM / head epilogues, zeroed once per step)
//   scale -- s, written by the tensor's producer before any consumer runs
struct TScale {
    float amax;
    float scale;
    unsigned pad[2];
};
// s = 2^e with bound < 2^(e + 15): every |x| <= bound maps to |x / s| < 32768 (fp16 max 65504).
MTX_DEVI float f16_scale_for(float bound) {
    if (!(bound > 0.f) || bound > 3.0e38f) return 1.f;  // zero, NaN, inf: the flag path reports it
    const int e = (int)((__float_as_uint(bound) >> 23) & 0xFFu) - 127;  // floor(log2 bound) (normal)
    int se = e + 1 - 15;
    se = se < -126 ? -126 : (se > 127 ? 127 : se);
    return __uint_as_float((uint32_t)(se + 127) << 23);
}
// hi/lo of y = x * inv_s (exact: inv_s is a power of two); y - hi is exact in fp32
MTX_DEVI void split_f16(float x, float inv_s, uint16_t &hi, uint16_t &lo) {
    const float y = x * inv_s;
    const float h = __half2float(__float2half_rn(y));
    hi = __half_as_ushort(__float2half_rn(y));
    lo = __half_as_ushort(__float2half_rn(y - h));
}
MTX_DEVI void amax_atomic(float *slot, float v) {  // v >= 0 (non-negative floats order like their bits)
    atomicMax((unsigned *)slot, __float_as_uint(v));
}

// Shared-memory mbarriers (completion tracking of TMA / bulk copies and tcgen05 commits).
MTX_DEVI uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
MTX_DEVI void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
MTX_DEVI void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
MTX_DEVI void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
MTX_DEVI void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

// Programmatic dependent launch.  Every kernel of the step starts with pdl_wait()
// (griddepcontrol.wait: returns once the preceding grid has completed and its memory is
// visible; a no-op when the launch was not programmatic) and is launched with
// launch_pdl(), so its launch and prologue overlap the predecessor's tail.
// The trigger right after the wait lets the next kernel be launched as soon as every CTA of
// this grid is running (its CTAs then park in their own wait until this grid completes).
MTX_DEVI void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
    static const int on = [] {
        const char *e = getenv("MTX_PDL");  // development A/B knob, default on
        return e ? atoi(e) : 1;
    }();
    return on != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace mtx
