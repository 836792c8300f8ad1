// k_tc_t1.cu — the tcgen05 GEMM kernels for TERMS = 1 (1xTF32); see tc_kernel.cuh.
#include "tc_kernel.cuh"

namespace emm {

cudaError_t launch_tc_terms1(const TcOperands &ops, int64_t M, int64_t N, int64_t Kp, float alpha, float beta,
                              float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial, cudaStream_t s,
                              const PeerOut &pe, void *sk_ws, const float *acc_init, int64_t ld_init) {
    return launch_tc_m<1>(ops, M, N, Kp, alpha, beta, C, ldc, ctrl, splits, partial, s, pe, sk_ws, acc_init, ld_init);
}

}  // namespace emm
