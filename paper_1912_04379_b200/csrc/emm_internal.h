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

// ---- tensor-core path (k_tc.cu host side, tc_kernel.cuh + k_tc_t{1,2,3}.cu kernels)
// One plane of an operand as the GEMM reads it through TMA: logical R x kext
// (rows x K).  mn = false: K-major, element (r, p) at ptr[p + r*ld];
// mn = true: MN-major, element (r, p) at ptr[r + p*ld].
struct TcPlane {
    const float *ptr = nullptr;
    int64_t ld = 0;
    bool mn = false;
    int64_t kext = 0;
    // TMA rounds each FP32 element to TF32 on load (tensor map data type
    // TFLOAT32: bit-identical to cvt.rn.tf32.f32, tools/tma_tf32_probe.cu);
    // the 1xTF32 direct path's operands (R7c)
    bool rn = false;
};
// plane 0 = big (the user array itself in the direct path), plane 1 = small
// (3xTF32) or BF16 cross (TF32+BF16); plane 1 unused for 1xTF32.
struct TcOperands {
    TcPlane a0, a1, b0, b1;
};

// Fused all-gather (multi-GPU): the GEMM epilogue also stores every C value
// to each rank's full output at (row_off + row, col_off + col) through peer
// pointers (CUDA IPC over NVLink; the own rank's buffer is base[rank]).
struct PeerOut {
    float *base[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int n = 0;
    int64_t ld = 0, row_off = 0, col_off = 0;
};

// Arguments of the split pass for one operand (see the PK_* modes in k_tc.cu).
struct PackArgs {
    const float *X = nullptr;
    int64_t ld = 0, R = 0;
    bool kcontig = false;   // element (r, p) of op(X) at X[p + r*ld] (else X[r + p*ld])
    float *out0 = nullptr;  // FULL modes: K-major big plane [R][ld0]
    int64_t ld0 = 0;
    float *out1 = nullptr;  // second plane
    int64_t ld1 = 0;
    bool b_side = false;    // B side of the cross operand (halves swapped)
};
enum { PK_FULL1_ = 0, PK_FULL3_ = 1, PK_FULLX_ = 2, PK_DSMALL_ = 3, PK_DCROSS_ = 4, PK_RAW_ = 5, PK_RAWT_ = 6 };
// One launch for A (and B if non-NULL); also zeroes `ctrl_words` words at
// ctrl (the control block, and the stream-K flags that follow it).
cudaError_t launch_pack(int mode, const PackArgs &a, const PackArgs *b, int64_t K, unsigned int *ctrl,
                        cudaStream_t s, int ctrl_words = 32);
// Per-call control block (wave-lockstep counter), and the stream-K scratch
// that may follow it: [flags: TC_SK_FLAG_BYTES][slots: tc_sk_slot_bytes()].
constexpr size_t TC_CTRL_BYTES = 1024;
constexpr size_t TC_SK_FLAG_BYTES = 8192;
size_t tc_sk_slot_bytes();
// split-K partials: one 256 x 256 FP32 slot per (split, tile) unit
size_t tc_splitk_bytes(int64_t M, int64_t N, int splits);
// Stream-K for this shape?  dp_tiles: tiles of the data-
// parallel phase; false for split-K / exact-wave / tiny-remainder shapes.
bool tc_sk_plan(int64_t M, int64_t N, int64_t K, int splits, int terms, int *dp_tiles);
// C <- alpha * op(A) op(B) + beta*C on the planes (tcgen05, 2-CTA,
// persistent, PDL).  terms: 3 = 3xTF32, 2 = TF32+BF16, 1 = 1xTF32.
// ctrl: per-call control block (word 0 = wave-lockstep counter), ZERO when
// the kernel starts (launch_pack zeroes it; callers without a pack memset
// it); NULL disables the lockstep.  splits > 1: split-K with raw partials in
// `partial` (splits x M x N floats) and a fixed-order reduce launch.
cudaError_t launch_tc_sgemm(int terms, const TcOperands &ops, int64_t M, int64_t N, int64_t K, float alpha,
                            float beta, float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial,
                            cudaStream_t s, const PeerOut *peers = nullptr, void *sk_ws = nullptr,
                            const float *acc_init = nullptr, int64_t ld_init = 0);
// acc_init (3xTF32 / TF32+BF16, whole tiles): the FP32 promotion chain of
// every output starts from acc_init[r + c*ld_init] (the raw partial, alpha = 1
// and beta = 0, of an earlier call over a K prefix that ends on a 256-of-K
// boundary) — together the calls add the same numbers in the same order as
// one call over all of K (K-phased host pipeline).
// Per-split launchers (k_tc_t{1,2,3}.cu, Kp = the padded K).
#define EMM_TC_TERMS_DECL(T)                                                                                        \
    cudaError_t launch_tc_terms##T(const TcOperands &ops, int64_t M, int64_t N, int64_t Kp, float alpha, float beta, \
                                   float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial,             \
                                   cudaStream_t s, const PeerOut &pe, void *sk_ws, const float *acc_init,             \
                                   int64_t ld_init);
EMM_TC_TERMS_DECL(1)
EMM_TC_TERMS_DECL(2)
EMM_TC_TERMS_DECL(3)
#undef EMM_TC_TERMS_DECL
// Fixed-order split-K reduce (KN8): C <- alpha * sum_s P_s + beta*C.
cudaError_t launch_splitk_reduce(const float *partial, int splits, int64_t M, int64_t N, float alpha, float beta,
                                 float *C, int64_t ldc, cudaStream_t s);
// KN11 (k_tcl.cu): 3xTF32 with the split in the kernel; reads the caller's
// A and B directly (any leading dimension, 16-B vector loads when aligned).
// a_kc / b_kc: K is the contiguous index of the stored op(A) / op(B).
// ctrl: zeroed control block for multi-wave problems (NULL: no lockstep).
cudaError_t launch_tc_split_sgemm(bool a_kc, bool b_kc, const float *A, int64_t lda, const float *B, int64_t ldb,
                                  int64_t M, int64_t N, int64_t K, float alpha, float beta, float *C, int64_t ldc,
                                  unsigned int *ctrl, int splits, float *partial, cudaStream_t s,
                                  const PeerOut *peers = nullptr);
// KN1X (k_tcx.cu): 3xTF32 with the split inside the kernel, TMA-fed: the
// raw operand planes a / b (the caller's arrays, TMA-legal, K- or MN-major)
// are the big parts, a transform warpgroup writes small = rn_tf32(x -
// trunc(x)) into SMEM beside them — bitwise identical to PK_DSMALL + KN1
// direct.  ctrl: zeroed control block for multi-wave launches (NULL: no
// lockstep); sk_ws: zeroed stream-K scratch or NULL.
cudaError_t launch_tc_xs_sgemm(const TcPlane &a, const TcPlane &b, int64_t M, int64_t N, int64_t K, float alpha,
                               float beta, float *C, int64_t ldc, unsigned int *ctrl, int splits, float *partial,
                               cudaStream_t s, const PeerOut *peers = nullptr, void *sk_ws = nullptr,
                               const float *acc_init = nullptr, int64_t ld_init = 0);
// the 3xTF32 policy of emm_sgemm_ex: KN1X (split in the kernel) unless
// EMM_SPLIT=pass / EMM_FORCE_PACK select the split pass + KN1 (api.cu)
bool tc_prefer_xs(int64_t M, int64_t N, int64_t K);
bool tma_legal(const void *ptr, int64_t ld);
// A plane as the tcgen05 kernels' 2-D tensor map (K-major box {32, 128},
// MN-major box {32, 32} with the 32B-atom 128B swizzle), OOB reads zero.
bool tc_make_tmap(CUtensorMap *tm, const TcPlane &p, int64_t R);
bool tc_make_tmap_rows(CUtensorMap *tm, const TcPlane &p, int64_t R, int box_rows);
// KN2w (k_tc1w.cu): 1xTF32 with a 256 x 512 tile per CTA pair (the whole
// 512-column TMEM as one accumulator) — 25% fewer operand bytes per flop
// than the 256 x 256 tile.  Full tiles only (no split-K / stream-K / peers).
bool tc1w_wanted(int64_t M, int64_t N, int64_t K);
cudaError_t launch_tc1w_sgemm(const TcOperands &ops, int64_t M, int64_t N, int64_t K, float alpha, float beta,
                              float *C, int64_t ldc, cudaStream_t s);
bool encode_tmap_f32_2d(CUtensorMap *tm, const float *ptr, int64_t d0, int64_t d1, int64_t ld, int box0, int box1,
                        CUtensorMapSwizzle swz);
int64_t tc_kpad(int64_t K);
int tc_splits(int64_t M, int64_t N, int64_t K);
int64_t tc_units(int64_t M, int64_t N, int splits);   // (tile, split) work units
int tc_num_sms();

// ---- CUDA-core path (k_ffma.cu) ------------------------------------------
cudaError_t launch_ffma_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              cudaStream_t s, int splits = 1, float *partial = nullptr);

// KN3b (k_ffma_tma.cu): warp-specialised FFMA SGEMM, TMA-fed SMEM ring.
// Returns false (nothing launched) when the shape / layout is not covered
// (both operands K-contiguous, or not TMA-legal); the caller then runs KN3.
bool ffma_tma_eligible(bool tA, bool tB, const float *A, int64_t lda, const float *B, int64_t ldb);
cudaError_t launch_ffma_tma_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                                  int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                                  cudaStream_t s, int splits = 1, float *partial = nullptr);
// KN3b split-K (sub-wave grids): factor and partial-slab bytes
int ffma_splits(int64_t M, int64_t N, int64_t K);
size_t ffma_splitk_bytes(int64_t M, int64_t N, int splits);

// ---- skinny / memory-bound path (k_skinny.cu) ----------------------------
// min(M, N) <= SKINNY_MAX: stream the long operand once, FP32 FFMA with
// promotion (every math mode; HBM-bound).
constexpr int64_t SKINNY_MAX = 16;
cudaError_t launch_skinny_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                                int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                                cudaStream_t s, float *ws = nullptr, size_t ws_bytes = 0);
// split-K slab bytes of the FFMA skinny path for this call (0: no split;
// A = B = null: the upper bound over pointers / leading dimensions)
size_t skinny_split_bytes(bool tA, bool tB, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                          const float *B, int64_t ldb);

// KN9T (k_skinny_tc.cu): the same roles on the tensor cores — the long
// operand TMA-streamed, split in the kernel and fed to tcgen05.mma from TMEM,
// the short one split once by the KN4 pass into `ws` (skinny_tc_workspace_bytes,
// 1024-byte aligned).  Default for 1xTF32 / TF32+BF16 with a short side > 8
// and a large, TMA-legal long operand (skinny_tc_wanted; EMM_SKINNY_TC=0/1).
bool skinny_tc_wanted(int terms, bool tA, bool tB, int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                      const float *B, int64_t ldb);
size_t skinny_tc_workspace_bytes(int64_t M, int64_t N, int64_t K);
cudaError_t launch_skinny_tc_sgemm(int terms, bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha,
                                   const float *A, int64_t lda, const float *B, int64_t ldb, float beta, float *C,
                                   int64_t ldc, void *ws, cudaStream_t s);

// ---- latency-bound small problems (k_tiny.cu) -----------------------------
cudaError_t launch_tiny_sgemm(bool tA, bool tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              cudaStream_t s);

// ---- misc (k_misc.cu) ------------------------------------------------------
cudaError_t launch_scale_c(int64_t M, int64_t N, float beta, float *C, int64_t ldc, cudaStream_t s);
// dst (M x Nc column-major, ld_dst) <- src laid out as `nranks` blocks of
// rows_r x Nc (each compact, ld = rows_r), block r covering rows row0_r..
cudaError_t launch_unpack_rows(const float *src, int nranks, const int64_t *row0, const int64_t *rows, int64_t Nc,
                               float *dst, int64_t ld_dst, cudaStream_t s);

}  // namespace emm
