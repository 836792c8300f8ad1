// emm_internal.h — declarations shared by the library's translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/emm.h"

namespace emm {

// BLAS argument rules (0 or -i) and the sm_100 device check (api.cu).
int check_args(char tA, char tB, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc);
int check_device();
size_t align_up(size_t v, size_t a);

// Launch accounting (every kernel launch of the library increments it).
extern std::atomic<uint64_t> g_launches;

// Dominant-kernel profiling (CUDA events on the launching stream).
void prof_begin(cudaStream_t s, bool is_gemm, cudaEvent_t *ev0);
void prof_end(cudaStream_t s, bool is_gemm, cudaEvent_t ev0);

// ---- tensor-core path (k_tc.cu) -----------------------------------------
// Pack op(X) (R x K, logical) into `out` as `planes` K-major planes of
// R x Kp floats (Kp = round_up(K, 32); zero-filled tail); plane 0 = big =
// rn_tf32(x), plane 1 (if planes == 2) = small = rn_tf32(x - big).
// kcontig: element (r, p) at X[p + r*ld]; else at X[r + p*ld].
// mode: 0 = big plane only (1xTF32), 1 = + tf32 small plane (3xTF32),
// 2 = + BF16 cross plane (TF32+BF16); see pack_store in k_tc.cu.
cudaError_t launch_pack_split(const float *X, int64_t ld, bool kcontig, int64_t R, int64_t K, int64_t Kp,
                              int mode, float *out, cudaStream_t s);
// Both operands in one launch (B may be NULL); also zeroes *wave_ctr.
// first_is_b: the first operand plays the B role (cross-plane half order).
cudaError_t launch_pack_split2(const float *A, int64_t lda, bool a_kcontig, int64_t M, const float *B, int64_t ldb,
                               bool b_kcontig, int64_t N, int64_t K, int64_t Kp, int mode, float *Aout, float *Bout,
                               unsigned int *wave_ctr, cudaStream_t s, bool first_is_b = false);
// C <- alpha * Ap * Bp^T + beta*C on the packed operands (tcgen05, 2-CTA,
// persistent).  wave_ctr: 4 bytes of device scratch owned by this call, ZERO
// when the kernel starts (launch_pack_split2 zeroes it), for the producers'
// wave lockstep; NULL disables it.  splits > 1: split-K with raw partials in
// `partial` (splits x M x N floats) and a fixed-order reduce launch.
cudaError_t launch_tc_sgemm(int terms, const float *Ap, const float *Bp, int64_t M, int64_t N, int64_t Kp,
                            float alpha, float beta, float *C, int64_t ldc, unsigned int *wave_ctr, int splits,
                            float *partial, cudaStream_t s);
int64_t tc_kpad(int64_t K);
int tc_splits(int64_t M, int64_t N, int64_t K);
int tc_num_sms();

// ---- CUDA-core path (k_ffma.cu) ------------------------------------------
cudaError_t launch_ffma_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              cudaStream_t s);

// ---- misc (k_misc.cu) ------------------------------------------------------
cudaError_t launch_scale_c(int64_t M, int64_t N, float beta, float *C, int64_t ldc, cudaStream_t s);
// dst (M x Nc column-major, ld_dst) <- src laid out as `nranks` blocks of
// rows_r x Nc (each compact, ld = rows_r), block r covering rows row0_r..
cudaError_t launch_unpack_rows(const float *src, int nranks, const int64_t *row0, const int64_t *rows, int64_t Nc,
                               float *dst, int64_t ld_dst, cudaStream_t s);

}  // namespace emm
