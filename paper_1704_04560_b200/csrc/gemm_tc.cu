// gemm_tc.cu -- placeholder until the tcgen05 engine lands (see gemm_tc.h).
#include "gemm_tc.h"

namespace mtx {
struct TcGemm {};
bool tc_available() { return false; }
TcGemm *tc_create(int) { return nullptr; }
void tc_destroy(TcGemm *t) { delete t; }
bool tc_supports(TcGemm *, const GemmDesc &) { return false; }
cudaError_t tc_gemm(TcGemm *, const GemmDesc &, cudaStream_t, LaunchHook *) { return cudaErrorNotSupported; }
}  // namespace mtx
