// k_tc_t3.cu — the tcgen05 GEMM kernels for TERMS = 3 (3xTF32); see tc_kernel.cuh.
#include "tc_kernel.cuh"

namespace emm {

cudaError_t launch_tc_terms3(const TcOperands &ops, int64_t M, int64_t N, int64_t Kp, float alpha, float beta,
                              float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial, cudaStream_t s,
                              const PeerOut &pe, void *sk_ws, const float *acc_init, int64_t ld_init) {
    return launch_tc_m<3>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
}

}  // namespace emm

#ifdef EMM_TIMELINE
extern "C" int emm_debug_timeline(unsigned long long *out, int n) {
    const int m = n < 512 * emm::TL_SLOTS ? n : 512 * emm::TL_SLOTS;
    return (int)cudaMemcpyFromSymbol(out, emm::g_emm_timeline, (size_t)m * 8);
}
#endif
