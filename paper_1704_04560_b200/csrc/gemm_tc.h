// gemm_tc.h -- tcgen05 (5th-gen tensor core) TF32 GEMM engine: TMA -> smem ring
// -> tcgen05.mma (accumulators in TMEM) -> tcgen05.ld epilogue.  Internal.
#pragma once
#include "kernels.h"

namespace mtx {
struct TcGemm;
bool tc_available();
// Tile width and split-K factor the engine uses for an M x N x K GEMM (splits if the partial
// buffer allows it).
struct TcPlan {
    int bn = 128;
    int splits = 1;
};
TcPlan tc_plan(int sms, int M, int N, int K, bool f16 = false);
int tc_choose_splits(int sms, int M, int N, int K);
TcGemm *tc_create(int device);
void tc_destroy(TcGemm *t);
// True when this engine handles the shape/layout of g (otherwise the caller uses SIMT).
bool tc_supports(TcGemm *t, const GemmDesc &g);
cudaError_t tc_gemm(TcGemm *t, const GemmDesc &g, cudaStream_t s, LaunchHook *h);
// True when g runs unsplit (the direct epilogue: the only path that writes the 3xF16 lean outputs
// relu_bits / colpart and honours skip_c32).
bool tc_direct(TcGemm *t, const GemmDesc &g);
}  // namespace mtx
