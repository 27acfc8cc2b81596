// common.cuh -- internal helpers of libmtx (product path; independent of oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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

}  // namespace mtx
