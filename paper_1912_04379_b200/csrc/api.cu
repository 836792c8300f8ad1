// api.cu — the C ABI of include/emm.h: argument validation (BLAS rules),
// quick returns, path selection and launch.  No CPU fallback: every step of
// the product runs in this library's kernels; if the device is not sm_100 the
// call fails with EMM_ERR_ARCH.
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "emm_internal.h"

namespace emm {

std::atomic<uint64_t> g_launches{0};

// ------------------------------------------------------------ profiling
namespace {
std::atomic<int> g_prof_on{0};
std::mutex g_prof_mu;
struct ProfRec {
    cudaEvent_t a, b;
    bool gemm;
};
std::vector<ProfRec> g_prof;
}  // namespace

void prof_begin(cudaStream_t s, bool, cudaEvent_t *ev0) {
    *ev0 = nullptr;
    if (!g_prof_on.load(std::memory_order_relaxed)) return;
    if (cudaEventCreate(ev0) != cudaSuccess) {
        *ev0 = nullptr;
        return;
    }
    cudaEventRecord(*ev0, s);
}

void prof_end(cudaStream_t s, bool is_gemm, cudaEvent_t ev0) {
    if (!ev0) return;
    cudaEvent_t ev1;
    if (cudaEventCreate(&ev1) != cudaSuccess) return;
    cudaEventRecord(ev1, s);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back({ev0, ev1, is_gemm});
}

// ------------------------------------------------------------ validation
static bool trans_ok(char t) { return t == 'N' || t == 'n' || t == 'T' || t == 't' || t == 'C' || t == 'c'; }
static bool is_n(char t) { return t == 'N' || t == 'n'; }
static int64_t max1(int64_t v) { return v > 1 ? v : 1; }

int check_args(char tA, char tB, int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc) {
    if (!trans_ok(tA)) return -1;
    if (!trans_ok(tB)) return -2;
    if (M < 0) return -3;
    if (N < 0) return -4;
    if (K < 0) return -5;
    if (lda < max1(is_n(tA) ? M : K)) return -8;
    if (ldb < max1(is_n(tB) ? K : N)) return -10;
    if (ldc < max1(M)) return -13;
    return 0;
}

static bool ptr_bad(const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 3u) != 0; }

// byte range [lo, hi) spanned by a column-major rows x cols array
static void span(const void *p, int64_t rows, int64_t cols, int64_t ld, uintptr_t *lo, uintptr_t *hi) {
    *lo = reinterpret_cast<uintptr_t>(p);
    *hi = *lo + (uintptr_t)(((cols - 1) * ld + rows) * 4);
}

int check_device() {
    static std::mutex mu;
    static int cached[64];
    static bool init = false;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return EMM_ERR_CUDA_BASE + (int)e;
    std::lock_guard<std::mutex> g(mu);
    if (!init) {
        for (int &c : cached) c = -1;
        init = true;
    }
    if (dev < 0 || dev >= 64) return EMM_ERR_ARCH;
    if (cached[dev] < 0) {
        int maj = 0, min = 0;
        cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev);
        cached[dev] = (maj == 10 && min == 0) ? 1 : 0;
    }
    return cached[dev] ? 0 : EMM_ERR_ARCH;
}

static int cuda_status(cudaError_t e) { return e == cudaSuccess ? 0 : EMM_ERR_CUDA_BASE + (int)e; }

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

static int planes_of(emm_math_t m) { return m == EMM_MATH_3XTF32 || m == EMM_MATH_TF32_BF16 ? 2 : 1; }

static int terms_of(emm_math_t m) { return m == EMM_MATH_3XTF32 ? 3 : m == EMM_MATH_TF32_BF16 ? 2 : 1; }
static bool math_ok(emm_math_t m) {
    return m == EMM_MATH_3XTF32 || m == EMM_MATH_FFMA || m == EMM_MATH_1XTF32 || m == EMM_MATH_TF32_BF16;
}

// Problems below this many flops are latency-bound (a few microseconds of
// launches dominate; the paper's "overhead of setting up buffers is
// prohibitive" regime): one launch of the tiny FFMA kernel (KN10),
// which is FP32-accurate.
// EMM_SMALL_FLOPS (environment) overrides the threshold; 0 disables it.
// Thresholds measured with the round-2 tiny kernel (4x4 outputs per thread,
// cp.async ring; profiles/r02_small_threshold.md): tensor-core modes cross
// over near 2^27 flops (400^3 tiny 19.2 vs KN1X 21.1 us, 448^3 equal, 512^3
// 22.5 vs 19.4); the FFMA mode's KN3b (128x128 tiles, one CTA per SM,
// split-K on sub-wave grids) overtakes it (64 x 64 tiles past 2 blocks per
// SM) near 7e8 flops (profiles/r02_ffma_relayout.md: 512^3 tiny 22.5 vs 35.8
// us, 700^3 39.4 vs 39.9, 768^3 41.0 vs 37.9, 1024^3 86.5 vs 60.4).
static bool small_problem(int64_t M, int64_t N, int64_t K, emm_math_t math = EMM_MATH_FFMA) {
    double thr = math == EMM_MATH_FFMA ? 7.0e8 : (double)(1 << 27);
    if (const char *e = getenv("EMM_SMALL_FLOPS")) thr = atof(e);
    return 2.0 * (double)M * (double)N * (double)K <= thr;
}

// How one tensor-core call runs:
//  * direct (both operands TMA-legal): the GEMM reads A and B in place,
//    K-major or MN-major per trans flag (transpose in the TMA descriptor);
//    the split pass writes only the second plane (3xTF32: small in the
//    operand's own layout; TF32+BF16: the K-major bf16 cross plane;
//    1xTF32: nothing).
//  * full (fallback, or EMM_FORCE_PACK=1): both planes re-buffered K-major.
// Workspace: [A plane(s) | B plane(s) | split-K partials | control block],
// 1024-byte aligned regions.  emm_sgemm_workspace_bytes returns the largest
// layout the call can take for any pointer / ld (KN1X: both operands
// re-pitched; other splits: the re-buffered planes).
struct Plan {
    bool direct = false;
    int pack_mode = -1;      // -1: no split pass
    int terms = 1;
    int splits = 1;
    size_t a_off = 0, b_off = 0, p_off = 0, ctr_off = 0, total = 0;
    bool sk = false;          // stream-K: [flags | slots] follow the control block
    bool xs = false;          // 3xTF32 split inside the GEMM (KN1X)
    bool rp_a = false, rp_b = false;   // KN1X on a raw re-pitched copy (PK_RAW) of a TMA-illegal operand
    int64_t lda1 = 0, ldb1 = 0;   // second-plane leading dimensions
};

static int64_t up4(int64_t v) { return (v + 3) / 4 * 4; }

// emm_sgemm without a workspace takes scratch from a stream-ordered pool that
// the LIBRARY owns (one per device, created on first use): its release
// threshold is raised so that freed scratch stays mapped for the next call
// (remapping GiB-sized scratch costs tens of ms), without touching the
// device's default pool that other cudaMallocAsync users share.
static cudaMemPool_t lib_pool() {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!pools[dev]) {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.handleTypes = cudaMemHandleTypeNone;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &pp) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
        pools[dev] = p;
    }
    return pools[dev];
}

// stream-ordered scratch from the library's pool
static cudaError_t scratch_alloc(void **p, size_t bytes, cudaStream_t s) {
    cudaMemPool_t pool = lib_pool();
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

static bool env_on(const char *name) {
    const char *e = getenv(name);
    return e && e[0] == '1';
}

// Direct vs re-buffered, when both are possible (measured on
// B200 back-to-back): the re-buffered big plane has its 13 low mantissa bits
// zeroed, which lowers the GEMM's power draw and, under the 1 kW cap, buys
// ~3-5% of clock on large square problems; the split pass costs
// ~ (1/M + 1/N) of the GEMM time.  So re-buffer only when that pass is cheap.
// EMM_FORCE_PACK=1 / EMM_FORCE_DIRECT=1 override (tests, experiments).
static bool prefer_direct(int64_t M, int64_t N, emm_math_t math) {
    const char *fp = getenv("EMM_FORCE_PACK");
    if (fp && fp[0] == '1') return false;
    const char *fd = getenv("EMM_FORCE_DIRECT");
    if (fd && fd[0] == '1') return true;
    const double f = 1.0 / (double)M + 1.0 / (double)N;
    const double thr = math == EMM_MATH_1XTF32 ? 1.0e-4 : 2.9e-4;
    return f > thr;
}

// 3xTF32 operand split inside the GEMM (KN11) vs a split pass + TMA GEMM.
// EMM_SPLIT=kernel / EMM_SPLIT=pass override (tests, experiments).
static bool prefer_inkernel_split(int64_t M, int64_t N, int64_t K) {
    (void)K;
    if (const char *e = getenv("EMM_SPLIT")) {
        if (!strcmp(e, "kernel")) return true;
        if (!strcmp(e, "pass")) return false;
    }
    if (env_on("EMM_FORCE_PACK") || env_on("EMM_FORCE_DIRECT")) return false;
    (void)M;
    (void)N;
    return false;   // policy set from measurements
}

// 3xTF32 on TMA-legal operands: split inside the TMA-fed GEMM (KN1X, no
// split pass) or the split pass + KN1.  EMM_SPLIT=xform / pass force one
// (tests, experiments), EMM_FORCE_PACK=1 forces the re-buffered pass.
// Measured on B200 (profiles/r02_ab_xs.md, one box, back to back): KN1X is
// faster on every TMA-legal config — c3 NN 52.3 -> 44.1 us, 1024^3 30.3 ->
// 27.6, 2048^3 87 -> 76, 4096^3 523 -> 472, 8192^3 3.90 -> 3.70 ms, c4-i
// 2.22 -> 1.88 ms, c4-ii 2.09 -> 1.98 ms, and the power-capped 32768^3 step
// 264 TFLOP/s either way — so it is the default.
static bool prefer_xs(int64_t M, int64_t N, int64_t K) {
    (void)M;
    (void)N;
    (void)K;
    if (const char *e = getenv("EMM_SPLIT")) {
        if (!strcmp(e, "xform")) return true;
        if (!strcmp(e, "pass") || !strcmp(e, "kernel")) return false;
    }
    return !env_on("EMM_FORCE_PACK");
}

bool tc_prefer_xs(int64_t M, int64_t N, int64_t K) { return prefer_xs(M, N, K); }

static Plan make_plan(char tA, char tB, int64_t M, int64_t N, int64_t K, emm_math_t math, bool direct,
                      bool xs = false, bool rp_a = false, bool rp_b = false) {
    Plan P;
    P.terms = terms_of(math);
    P.splits = tc_splits(M, N, K);
    P.direct = direct;
    P.xs = xs;
    P.rp_a = rp_a;
    P.rp_b = rp_b;
    const int64_t Kp = tc_kpad(K);
    size_t a_bytes, b_bytes;
    if (xs) {
        // the small planes are made on chip; a TMA-illegal operand is first
        // copied raw into a 16-byte-pitched buffer (its stored layout, ld
        // rounded up to a multiple of 4 floats)
        P.pack_mode = (rp_a || rp_b) ? PK_RAW_ : -1;
        const int64_t ar = is_n(tA) ? M : K, ac = is_n(tA) ? K : M;
        const int64_t br = is_n(tB) ? K : N, bc = is_n(tB) ? N : K;
        P.lda1 = up4(ar);
        P.ldb1 = up4(br);
        a_bytes = rp_a ? (size_t)ac * P.lda1 * 4 : 0;
        b_bytes = rp_b ? (size_t)bc * P.ldb1 * 4 : 0;
    } else if (!direct) {
        const size_t pl = (size_t)planes_of(math);
        P.pack_mode = math == EMM_MATH_3XTF32 ? PK_FULL3_ : math == EMM_MATH_TF32_BF16 ? PK_FULLX_ : PK_FULL1_;
        P.lda1 = P.ldb1 = Kp;
        a_bytes = pl * (size_t)M * Kp * 4;
        b_bytes = pl * (size_t)N * Kp * 4;
    } else if (math == EMM_MATH_3XTF32) {
        P.pack_mode = PK_DSMALL_;
        // small plane in the operand's own layout: K-major [R][up4(K)] or MN-major [K][up4(R)]
        const bool a_mn = is_n(tA), b_mn = !is_n(tB);
        P.lda1 = a_mn ? up4(M) : up4(K);
        P.ldb1 = b_mn ? up4(N) : up4(K);
        a_bytes = (size_t)(a_mn ? K : M) * P.lda1 * 4;
        b_bytes = (size_t)(b_mn ? K : N) * P.ldb1 * 4;
    } else if (math == EMM_MATH_TF32_BF16) {
        P.pack_mode = PK_DCROSS_;
        P.lda1 = P.ldb1 = Kp;
        a_bytes = (size_t)M * Kp * 4;
        b_bytes = (size_t)N * Kp * 4;
    } else {
        P.pack_mode = -1;
        a_bytes = b_bytes = 0;
    }
    P.a_off = 0;
    P.b_off = align_up(a_bytes, 1024);
    P.p_off = P.b_off + align_up(b_bytes, 1024);
    P.ctr_off = P.p_off + align_up(tc_splitk_bytes(M, N, P.splits), 1024);
    int dp = 0;
    P.sk = tc_sk_plan(M, N, K, P.splits, P.terms, &dp);
    P.total = P.ctr_off + TC_CTRL_BYTES + (P.sk ? TC_SK_FLAG_BYTES + tc_sk_slot_bytes() : 0);
    return P;
}

// FFMA relayout: HBM-bound copy passes before KN3b — K-contiguous operands
// transposed to MN-contiguous (PK_RAWT; always one for TN, which KN3b does
// not cover; by size otherwise, see ffma_relayout), TMA-illegal ones
// re-pitched in their own layout (PK_RAW) — then KN3b on the copies.  Measured on B200 (profiles/r02_ffma_relayout.md):
// c3 TN 246 -> 212 us, TT 243 -> 206, 4096^3 TN 2.61 -> 2.43 ms.
struct FfmaRelayout {
    bool on = false, t_a = false, t_b = false, rp_a = false, rp_b = false;
    int64_t lda1 = 0, ldb1 = 0;
    size_t a_bytes = 0, b_bytes = 0, total = 0;
};
static FfmaRelayout ffma_relayout(bool tA, bool tB, int64_t M, int64_t N, int64_t K, bool legal_a, bool legal_b) {
    FfmaRelayout R;
    // KN3b runs fastest with BOTH operands MN-contiguous (the NT layout: 128-bit
    // operand loads on both sides; 4096^3: NT 84.1 % of the FP32 pipe, NN 73.4,
    // TT 75.3, TN-after-one-transpose 73.5, profiles/r02_ffma_relayout.md).
    // A K-contiguous operand is transposed when the copy is cheap next to the
    // GEMM (its cost relative to the GEMM ~ 44 / (the other extent)): op(A)
    // when N >= 1280, op(B) when M >= 1280 (measured: 1024^3 loses 2 us to the
    // copy, 1531 x 997 x 2049 NN gains 8 us, 2048^3 +8 %, 8192^3 +13 %); a TN
    // call transposes at least the smaller one (KN3b needs one MN-contiguous
    // operand).  EMM_FFMA_NT_MIN moves the 1280 (0: never by size).
    int64_t thr = 1280;
    if (const char *e = getenv("EMM_FFMA_NT_MIN")) thr = atoll(e) > 0 ? atoll(e) : INT64_MAX;
    const bool a_kc = tA, b_kc = !tB;
    R.t_a = a_kc && N >= thr;
    R.t_b = b_kc && M >= thr;
    if (a_kc && b_kc && !R.t_a && !R.t_b) (M <= N ? R.t_a : R.t_b) = true;
    R.on = R.t_a || R.t_b || !legal_a || !legal_b;
    if (!R.on) return R;
    R.rp_a = !R.t_a && !legal_a;
    R.rp_b = !R.t_b && !legal_b;
    const int64_t ar = tA ? K : M, ac = tA ? M : K;   // A stored ar x ac
    const int64_t br = tB ? N : K, bc = tB ? K : N;
    if (R.t_a) R.lda1 = tc_kpad(M), R.a_bytes = (size_t)K * R.lda1 * 4;
    if (R.rp_a) R.lda1 = (ar + 3) / 4 * 4, R.a_bytes = (size_t)ac * R.lda1 * 4;
    if (R.t_b) R.ldb1 = tc_kpad(N), R.b_bytes = (size_t)K * R.ldb1 * 4;
    if (R.rp_b) R.ldb1 = (br + 3) / 4 * 4, R.b_bytes = (size_t)bc * R.ldb1 * 4;
    R.total = align_up(R.a_bytes, 1024) + R.b_bytes;
    return R;
}

static size_t ws_bytes(char tA, char tB, int64_t M, int64_t N, int64_t K, emm_math_t math) {
    if (M == 0 || N == 0 || K == 0) return 0;
    if (M <= SKINNY_MAX || N <= SKINNY_MAX) {
        // KN9T planes (tensor-core modes) or the FFMA skinny path's split-K slabs
        const size_t ff = skinny_split_bytes(!is_n(tA), !is_n(tB), M, N, K, nullptr, 0, nullptr, 0);
        return math == EMM_MATH_FFMA ? ff : std::max(ff, skinny_tc_workspace_bytes(M, N, K));
    }
    if (math == EMM_MATH_FFMA) {
        // upper bound: the relayout copies with both operands TMA-illegal
        if (small_problem(M, N, K, math)) return 0;
        return align_up(ffma_relayout(!is_n(tA), !is_n(tB), M, N, K, false, false).total, 1024) +
               ffma_splitk_bytes(M, N, ffma_splits(M, N, K));
    }
    if (small_problem(M, N, K, math)) return 0;
    // 3xTF32 on KN1X: at most the raw re-pitch of both operands (when their
    // leading dimensions are TMA-illegal) + split-K / stream-K scratch; the
    // other splits (and EMM_SPLIT=pass / EMM_FORCE_PACK): the re-buffered planes
    if (math == EMM_MATH_3XTF32 && prefer_xs(M, N, K)) return make_plan(tA, tB, M, N, K, math, true, true, true, true).total;
    return make_plan('N', 'N', M, N, K, math, /*direct=*/false).total;
}


// Workspace one call with these operands needs (pointer-aware where the
// FFMA relayout depends on alignment; else the ws_bytes upper bound).
static size_t call_ws_bytes(char tA, char tB, int64_t M, int64_t N, int64_t K, emm_math_t math, const float *A,
                            int64_t lda, const float *B, int64_t ldb) {
    if (M == 0 || N == 0 || K == 0) return 0;
    if (math == EMM_MATH_FFMA) {
        if (M <= SKINNY_MAX || N <= SKINNY_MAX)
            return skinny_split_bytes(!is_n(tA), !is_n(tB), M, N, K, A, lda, B, ldb);
        if (small_problem(M, N, K, math)) return 0;
        const FfmaRelayout R = ffma_relayout(!is_n(tA), !is_n(tB), M, N, K, tma_legal(A, lda), tma_legal(B, ldb));
        return align_up(R.total, 1024) + ffma_splitk_bytes(M, N, ffma_splits(M, N, K));
    }
    return ws_bytes(tA, tB, M, N, K, math);
}

}  // namespace emm

using namespace emm;

extern "C" size_t emm_sgemm_workspace_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K,
                                            emm_math_t math) {
    if (M < 0 || N < 0 || K < 0) return 0;
    return ws_bytes(transA, transB, M, N, K, math);
}

extern "C" int emm_sgemm_ex(char transA, char transB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                            int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc, void *stream,
                            emm_math_t math, void *workspace, size_t workspace_bytes) {
    int st = check_args(transA, transB, M, N, K, lda, ldb, ldc);
    if (st) return st;
    if (!math_ok(math)) return EMM_ERR_MATH;
    // quick return (BLAS): nothing to do
    if (M == 0 || N == 0) return 0;
    const bool ab_used = !(alpha == 0.0f || K == 0);
    if (!ab_used && beta == 1.0f) return 0;
    if (ptr_bad(C)) return -12;
    if (ab_used) {
        if (ptr_bad(A)) return -7;
        if (ptr_bad(B)) return -9;
        uintptr_t c0, c1, a0, a1, b0, b1;
        span(C, M, N, ldc, &c0, &c1);
        span(A, is_n(transA) ? M : K, is_n(transA) ? K : M, lda, &a0, &a1);
        span(B, is_n(transB) ? K : N, is_n(transB) ? N : K, ldb, &b0, &b1);
        if ((c0 < a1 && a0 < c1) || (c0 < b1 && b0 < c1)) return EMM_ERR_ALIAS;
    }
    if ((st = check_device())) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);

    if (!ab_used) return cuda_status(launch_scale_c(M, N, beta, C, ldc, s));

    if ((M <= SKINNY_MAX || N <= SKINNY_MAX) && !env_on("EMM_NO_SKINNY")) {
        if (math != EMM_MATH_FFMA &&
            skinny_tc_wanted(terms_of(math), !is_n(transA), !is_n(transB), M, N, K, A, lda, B, ldb)) {
            // tensor cores (KN9T): scratch for the short operand's planes
            const size_t need = skinny_tc_workspace_bytes(M, N, K);
            void *ws = workspace;
            bool own = false;
            if (ws) {
                if (workspace_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 1023u)) return EMM_ERR_WORKSPACE;
            } else {
                cudaError_t e = scratch_alloc(&ws, need, s);
                if (e != cudaSuccess) return cuda_status(e);
                own = true;
            }
            cudaError_t e = launch_skinny_tc_sgemm(terms_of(math), !is_n(transA), !is_n(transB), M, N, K, alpha, A,
                                                   lda, B, ldb, beta, C, ldc, ws, s);
            if (own) {
                cudaError_t e2 = cudaFreeAsync(ws, s);
                if (e == cudaSuccess) e = e2;
            }
            return cuda_status(e);
        }
        // FFMA skinny (KN9): split-K slabs when the row blocks do not fill the SMs
        const size_t need = skinny_split_bytes(!is_n(transA), !is_n(transB), M, N, K, A, lda, B, ldb);
        void *ws = workspace;
        bool own = false;
        if (need) {
            if (ws) {
                if (workspace_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 1023u)) return EMM_ERR_WORKSPACE;
            } else {
                cudaError_t e = scratch_alloc(&ws, need, s);
                if (e != cudaSuccess) return cuda_status(e);
                own = true;
            }
        }
        cudaError_t e = launch_skinny_sgemm(!is_n(transA), !is_n(transB), M, N, K, alpha, A, lda, B, ldb, beta, C,
                                            ldc, s, need ? reinterpret_cast<float *>(ws) : nullptr, need);
        if (own) {
            cudaError_t e2 = cudaFreeAsync(ws, s);
            if (e == cudaSuccess) e = e2;
        }
        return cuda_status(e);
    }

    if (small_problem(M, N, K, math))
        return cuda_status(
            launch_tiny_sgemm(!is_n(transA), !is_n(transB), M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s));
    if (math == EMM_MATH_FFMA) {
        const bool tA = !is_n(transA), tB = !is_n(transB);
        FfmaRelayout R = ffma_relayout(tA, tB, M, N, K, tma_legal(A, lda), tma_legal(B, ldb));
        const bool classic = env_on("EMM_FFMA_CLASSIC");
        if (classic || env_on("EMM_FFMA_NORELAYOUT")) R = FfmaRelayout{};
        // KN3b runs unless forced classic or left on an uncovered layout: split-K for sub-wave grids
        const int splits = !classic && (R.on || ffma_tma_eligible(tA, tB, A, lda, B, ldb)) ? ffma_splits(M, N, K) : 1;
        const size_t r_bytes = align_up(R.total, 1024), need = r_bytes + ffma_splitk_bytes(M, N, splits);
        if (need == 0)
            return cuda_status(launch_ffma_sgemm(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s));
        void *ws = workspace;
        bool own = false;
        if (ws) {
            if (workspace_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 1023u)) return EMM_ERR_WORKSPACE;
        } else {
            cudaError_t e = scratch_alloc(&ws, need, s);
            if (e == cudaErrorMemoryAllocation) {
                // no room for the copies: the operands in place (KN3b where it
                // covers the layout, else KN3), unsplit: the same FP32 bound
                cudaGetLastError();
                return cuda_status(launch_ffma_sgemm(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, s));
            }
            if (e != cudaSuccess) return cuda_status(e);
            own = true;
        }
        float *a1 = reinterpret_cast<float *>(ws);
        float *b1 = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + align_up(R.a_bytes, 1024));
        float *part = splits > 1 ? reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(ws) + r_bytes) : nullptr;
        const float *A2 = A, *B2 = B;
        int64_t lda2 = lda, ldb2 = ldb;
        bool tA2 = tA, tB2 = tB;
        cudaError_t e = cudaSuccess;
        if (R.t_a) {
            // op(A)(r, p) = A[p + r*lda] read as an MN-contiguous K x M operand,
            // written K-major: A2[r + p*lda1] (transA = N)
            PackArgs x;
            x.X = A; x.ld = lda; x.R = K; x.kcontig = false; x.out0 = a1; x.ld0 = R.lda1;
            e = launch_pack(PK_RAWT_, x, nullptr, M, nullptr, s, 0);
            A2 = a1, lda2 = R.lda1, tA2 = false;
        }
        if (R.t_b && e == cudaSuccess) {
            // op(B)(p, j) = B[p + j*ldb] -> B2[j + p*ldb1] (transB = T)
            PackArgs x;
            x.X = B; x.ld = ldb; x.R = K; x.kcontig = false; x.out0 = b1; x.ld0 = R.ldb1;
            e = launch_pack(PK_RAWT_, x, nullptr, N, nullptr, s, 0);
            B2 = b1, ldb2 = R.ldb1, tB2 = true;
        }
        if (e == cudaSuccess && (R.rp_a || R.rp_b)) {
            PackArgs ra, rb;
            ra.X = A; ra.ld = lda; ra.R = M; ra.kcontig = tA; ra.out0 = a1; ra.ld0 = R.lda1;
            rb.X = B; rb.ld = ldb; rb.R = N; rb.kcontig = !tB; rb.out0 = b1; rb.ld0 = R.ldb1;
            e = launch_pack(PK_RAW_, R.rp_a ? ra : rb, (R.rp_a && R.rp_b) ? &rb : nullptr, K, nullptr, s, 0);
            if (R.rp_a) A2 = a1, lda2 = R.lda1;
            if (R.rp_b) B2 = b1, ldb2 = R.ldb1;
        }
        if (e == cudaSuccess)
            e = launch_ffma_sgemm(tA2, tB2, M, N, K, alpha, A2, lda2, B2, ldb2, beta, C, ldc, s, splits, part);
        if (own) {
            cudaError_t e2 = cudaFreeAsync(ws, s);
            if (e == cudaSuccess) e = e2;
        }
        return cuda_status(e);
    }

    // tensor-core paths
    if (math == EMM_MATH_3XTF32 && prefer_inkernel_split(M, N, K)) {
        // KN11: split inside the kernel (no split pass, no operand workspace)
        const int splits = tc_splits(M, N, K);
        const bool multiwave = tc_units(M, N, splits) > tc_num_sms() / 2;
        const size_t p_bytes = align_up(tc_splitk_bytes(M, N, splits), 1024);
        const size_t need = (splits > 1 || multiwave) ? p_bytes + 1024 : 0;
        void *ws = workspace;
        bool own = false;
        if (need) {
            if (ws) {
                if (workspace_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 1023u)) return EMM_ERR_WORKSPACE;
            } else {
                cudaError_t e = scratch_alloc(&ws, need, s);
                if (e != cudaSuccess) return cuda_status(e);
                own = true;
            }
        }
        uint8_t *w = reinterpret_cast<uint8_t *>(ws);
        float *Pp = splits > 1 ? reinterpret_cast<float *>(w) : nullptr;
        unsigned int *ctr = multiwave ? reinterpret_cast<unsigned int *>(w + p_bytes) : nullptr;
        cudaError_t e = ctr ? cudaMemsetAsync(ctr, 0, 128, s) : cudaSuccess;
        if (e == cudaSuccess)
            e = launch_tc_split_sgemm(!is_n(transA), is_n(transB), A, lda, B, ldb, M, N, K, alpha, beta, C, ldc, ctr,
                                      splits, Pp, s);
        if (own) {
            cudaError_t e2 = cudaFreeAsync(ws, s);
            if (e == cudaSuccess) e = e2;
        }
        return cuda_status(e);
    }
    const bool legal_a = tma_legal(A, lda), legal_b = tma_legal(B, ldb);
    const bool legal = legal_a && legal_b;
    // 3xTF32: KN1X on the caller's arrays, or (TMA-illegal leading dimension,
    // e.g. c3's lda = K + 13) on a raw re-pitched copy of that operand
    const bool xs = math == EMM_MATH_3XTF32 && prefer_xs(M, N, K) && (legal || !env_on("EMM_NO_REPITCH"));
    const bool direct = xs || (legal && prefer_direct(M, N, math));
    const Plan P = make_plan(transA, transB, M, N, K, math, direct, xs, xs && !legal_a, xs && !legal_b);
    void *ws = workspace;
    bool own = false;
    if (ws) {
        if (workspace_bytes < P.total || (reinterpret_cast<uintptr_t>(ws) & 1023u)) return EMM_ERR_WORKSPACE;
    } else {
        cudaError_t e = scratch_alloc(&ws, P.total, s);
        if (e != cudaSuccess) return cuda_status(e);
        own = true;
    }
    uint8_t *w = reinterpret_cast<uint8_t *>(ws);
    float *a1 = reinterpret_cast<float *>(w + P.a_off);
    float *b1 = reinterpret_cast<float *>(w + P.b_off);
    float *Pp = reinterpret_cast<float *>(w + P.p_off);
    unsigned int *ctr = reinterpret_cast<unsigned int *>(w + P.ctr_off);
    const int64_t Kp = tc_kpad(K);
    const bool a_kc = !is_n(transA), b_kc = is_n(transB);   // K contiguous in memory
    TcOperands ops;
    PackArgs pa, pb;
    pa.X = A; pa.ld = lda; pa.R = M; pa.kcontig = a_kc; pa.b_side = false;
    pb.X = B; pb.ld = ldb; pb.R = N; pb.kcontig = b_kc; pb.b_side = true;
    if (P.direct) {
        ops.a0 = TcPlane{A, lda, !a_kc, K};
        ops.b0 = TcPlane{B, ldb, !b_kc, K};
        // 1xTF32, TF32+BF16: the TMA rounds x to rn_tf32(x) on load (the
        // tensor core alone would truncate, R7b) -- the re-buffered numerics
        // (EMM_TMA_TRUNC=1, 1xTF32 only: raw operands, the round-1 numerics;
        // experiments)
        ops.a0.rn = ops.b0.rn =
            math == EMM_MATH_TF32_BF16 || (math == EMM_MATH_1XTF32 && !env_on("EMM_TMA_TRUNC"));
        if (P.pack_mode == PK_DSMALL_) {
            ops.a1 = TcPlane{a1, P.lda1, !a_kc, K};
            ops.b1 = TcPlane{b1, P.ldb1, !b_kc, K};
        } else if (P.pack_mode == PK_DCROSS_) {
            ops.a1 = TcPlane{a1, Kp, false, Kp};
            ops.b1 = TcPlane{b1, Kp, false, Kp};
        }
        pa.out1 = a1; pa.ld1 = P.lda1;
        pb.out1 = b1; pb.ld1 = P.ldb1;
    } else {
        // fallback: K-major planes [R][Kp]: plane 0 then plane 1 of each operand
        const int pl = planes_of(math);
        pa.out0 = a1; pa.ld0 = Kp; pa.out1 = a1 + (size_t)M * Kp; pa.ld1 = Kp;
        pb.out0 = b1; pb.ld0 = Kp; pb.out1 = b1 + (size_t)N * Kp; pb.ld1 = Kp;
        ops.a0 = TcPlane{pa.out0, Kp, false, Kp};
        ops.b0 = TcPlane{pb.out0, Kp, false, Kp};
        if (pl == 2) {
            ops.a1 = TcPlane{pa.out1, Kp, false, Kp};
            ops.b1 = TcPlane{pb.out1, Kp, false, Kp};
        }
    }
    cudaError_t e = cudaSuccess;
    // zeroed before the GEMM: control block (+ stream-K flags)
    const size_t zero_bytes = TC_CTRL_BYTES + (P.sk ? TC_SK_FLAG_BYTES : 0);
    void *sk_ws = P.sk ? w + P.ctr_off + TC_CTRL_BYTES : nullptr;
    if (P.xs) {
        // control block / stream-K flags only matter for multi-wave launches
        const bool multiwave = P.sk || tc_units(M, N, P.splits) > tc_num_sms() / 2;
        if (P.rp_a || P.rp_b) {
            // raw re-pitch of the TMA-illegal operand(s); the same launch zeroes ctrl
            PackArgs ra = pa, rb = pb;
            ra.out0 = a1; ra.ld0 = P.lda1;
            rb.out0 = b1; rb.ld0 = P.ldb1;
            if (P.rp_a) ops.a0 = TcPlane{a1, P.lda1, !a_kc, K};
            if (P.rp_b) ops.b0 = TcPlane{b1, P.ldb1, !b_kc, K};
            e = launch_pack(PK_RAW_, P.rp_a ? ra : rb, (P.rp_a && P.rp_b) ? &rb : nullptr, K,
                            multiwave ? ctr : nullptr, s, multiwave ? (int)(zero_bytes / 4) : 0);
        } else if (multiwave) {
            e = cudaMemsetAsync(ctr, 0, zero_bytes, s);
        }
        if (e == cudaSuccess)
            e = launch_tc_xs_sgemm(ops.a0, ops.b0, M, N, K, alpha, beta, C, ldc, multiwave ? ctr : nullptr, P.splits,
                                   Pp, s, nullptr, sk_ws);
    } else {
        if (P.pack_mode >= 0) {
            e = launch_pack(P.pack_mode, pa, &pb, K, ctr, s, (int)(zero_bytes / 4));
        } else if (P.sk || (P.terms > 1 && tc_units(M, N, P.splits) > tc_num_sms() / 2)) {
            // no pass to zero the control block in: a memset, only when the
            // GEMM reads it (wave lockstep of a multi-wave 2/3-term grid,
            // stream-K flags; 1xTF32 grids never do, tc_kernel.cuh) — a
            // memset node costs ~2-4 us of latency on sub-wave calls
            e = cudaMemsetAsync(ctr, 0, zero_bytes, s);
        }
        if (e == cudaSuccess)
            e = launch_tc_sgemm(P.terms, ops, M, N, K, alpha, beta, C, ldc, ctr, P.splits, Pp, s, nullptr, sk_ws);
    }
    if (own) {
        cudaError_t e2 = cudaFreeAsync(ws, s);
        if (e == cudaSuccess) e = e2;
    }
    return cuda_status(e);
}

extern "C" int emm_sgemm(char transA, char transB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                         int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc, void *stream) {
    return emm_sgemm_ex(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, stream, EMM_MATH_3XTF32,
                        nullptr, 0);
}

// ------------------------------------------------------------ host-buffer form
namespace {
std::mutex g_host_mu;
struct HostCache {
    void *dA = nullptr, *dB = nullptr, *dC = nullptr, *dW = nullptr, *dR = nullptr;
    size_t nA = 0, nB = 0, nC = 0, nW = 0, nR = 0;
    cudaStream_t s = nullptr;
    int dev = -1;
} g_hc;

int ensure(void **p, size_t *have, size_t need) {
    if (*have >= need && *p) return 0;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    if (need == 0) return 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e != cudaSuccess) return EMM_ERR_CUDA_BASE + (int)e;
    *have = need;
    return 0;
}
}  // namespace

// Pipelined host-buffer SGEMM (tensor-core modes, M, N >= 4096): three
// streams over op(A) row blocks and op(B) column blocks (host_pipelined: L-
// shaped growth — each landed block is re-buffered once on `comp` and
// multiplied against every resident block of the other operand in one GEMM;
// `h2d` copies blocks (and the C regions when beta != 0) in that order, `d2h`
// copies each C region out as soon as its GEMM is done).  PCIe traffic in both
// directions overlaps the tensor-core work after the first few blocks.
namespace {
struct HostStreams {
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev;
    int dev = -1;
} g_hs;

cudaEvent_t hs_event(size_t i) {
    while (g_hs.ev.size() <= i) {
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        g_hs.ev.push_back(e);
    }
    return g_hs.ev[i];
}

// rows [r0, r0+nr) of op(X) (R x K op-matrix) from host to the same place of
// the device copy (same ld): contiguous when K is the stored column index.
cudaError_t copy_rows(float *d, const float *h, bool rows_contig_in_col, int64_t ld, int64_t r0, int64_t nr,
                      int64_t k0, int64_t nk, int64_t K, cudaStream_t s) {
    if (rows_contig_in_col) {   // stored column-major with op rows along the leading dim: 2-D copy
        const int64_t o = r0 + k0 * ld;
        return cudaMemcpy2DAsync(d + o, (size_t)ld * 4, h + o, (size_t)ld * 4, (size_t)nr * 4, (size_t)nk,
                                 cudaMemcpyHostToDevice, s);
    }
    // op rows are stored columns: one contiguous range for all of K, else a
    // 2-D copy of the K sub-range of each row
    if (k0 == 0 && nk == K)
        return cudaMemcpyAsync(d + r0 * ld, h + r0 * ld, (size_t)((nr - 1) * ld + K) * 4, cudaMemcpyHostToDevice, s);
    const int64_t o = k0 + r0 * ld;
    return cudaMemcpy2DAsync(d + o, (size_t)ld * 4, h + o, (size_t)ld * 4, (size_t)nk * 4, (size_t)nr,
                             cudaMemcpyHostToDevice, s);
}
}  // namespace

static int host_pipelined(char tA, char tB, int64_t M, int64_t N, int64_t K, float alpha, const float *A, int64_t lda,
                          const float *B, int64_t ldb, float beta, float *C, int64_t ldc, emm_math_t math, float *dA,
                          float *dB, float *dC, void *dW, float *dR, bool xs) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_hs.dev != dev) {
        for (cudaStream_t *p : {&g_hs.h2d, &g_hs.comp, &g_hs.d2h}) {
            if (*p) cudaStreamDestroy(*p);
            if (cudaStreamCreateWithFlags(p, cudaStreamNonBlocking) != cudaSuccess) return EMM_ERR_NOMEM;
        }
        g_hs.dev = dev;
    }
    // Blocks of op(A) rows / op(B) columns: 3072 (EMM_HOST_BLOCK; at most 64
    // blocks per operand); EMM_HOST_FIRST sizes the first two of each operand
    // and EMM_HOST_CHUNK splits each GEMM region into pieces with their own
    // copy-back.  Both default off: at 32768^3 first = 1024 starts the first
    // GEMM 4.9 ms earlier but the smaller GEMMs cost more (307 vs 304 ms), and
    // 8192-wide pieces cut the copy-back tail 5 -> 1.5 ms but fall off whole
    // waves (316 ms; profiles/r01_e2e_timeline.txt).
    // 3072 with the KN1X pipeline (no re-buffering): bigger blocks make the
    // GEMMs more efficient and the start-up is still short (32768^3 e2e 233.6
    // -> 236.8 TFLOP/s, tools/e2e_timeline.py span 291 -> 287 ms); 2048 was the
    // round-1 choice with re-buffered planes
    int64_t blk = 3072;
    if (const char *eb = getenv("EMM_HOST_BLOCK")) blk = std::max<int64_t>(256, atoll(eb) / 256 * 256);
    blk = std::max(blk, ((std::max(M, N) + 31) / 32 + 255) / 256 * 256);
    int64_t first = blk;
    if (const char *ef = getenv("EMM_HOST_FIRST")) first = std::max<int64_t>(256, atoll(ef) / 256 * 256);
    first = std::min(first, blk);
    auto bounds = [&](int64_t R) {   // block starts, R appended
        std::vector<int64_t> b{0};
        while (b.back() < R) b.push_back(std::min(R, b.back() + (b.size() <= 2 ? first : blk)));
        return b;
    };
    const std::vector<int64_t> ra = bounds(M), cb = bounds(N);
    const int GM = (int)ra.size() - 1, GN = (int)cb.size() - 1;
    int64_t chunk = INT64_MAX;
    if (const char *ec = getenv("EMM_HOST_CHUNK")) chunk = std::max<int64_t>(512, atoll(ec) / 256 * 256);
    const int64_t Kp = tc_kpad(K);
    const int terms = terms_of(math), pl = planes_of(math);
    const int pmode = math == EMM_MATH_3XTF32 ? PK_FULL3_ : math == EMM_MATH_TF32_BF16 ? PK_FULLX_ : PK_FULL1_;
    // xs (3xTF32 on TMA-legal copies): KN1X reads each landed block of the
    // device copies of A and B in place, no re-buffering (dW = control words)
    float *Ap = reinterpret_cast<float *>(dW);
    float *Bp = Ap + (size_t)pl * M * Kp;
    unsigned int *ctrl = reinterpret_cast<unsigned int *>(
        reinterpret_cast<uint8_t *>(dW) + (xs ? 0 : align_up((size_t)pl * (M + N) * Kp * 4, 1024)));
    const bool a_rows_ld = is_n(tA);    // op(A) rows contiguous in a stored column
    const bool b_rows_ld = !is_n(tB);   // op(B)^T rows (= B columns) contiguous: transB = 'T'
    cudaStream_t h2d = g_hs.h2d, comp = g_hs.comp, d2h = g_hs.d2h;
    cudaError_t e = cudaSuccess;
    size_t evn = 0;
    auto ev = [&]() { return hs_event(evn++); };
    if (cudaMemsetAsync(ctrl, 0, 64 * 128, comp) != cudaSuccess) return EMM_ERR_NOMEM;
    // L-shaped growth (paper analogue: re-buffer each block once, PAPER.md:
    // 133-138, then reuse it against everything already resident): land the
    // next op(A) row block or op(B) column block — whichever keeps the
    // resident rows and columns balanced — re-buffer it once, and at once
    // multiply it against ALL resident blocks of the other operand with ONE
    // GEMM; every C block is computed exactly once, when the later of its two
    // operand blocks lands, and copied back right after.  Compute per PCIe
    // byte grows with the resident square, so the copies hide under the
    // tensor-core work after the first few blocks.
    // K phases (dR != nullptr): the first half of K for every block first
    // (half the bytes per block, so the tensor cores are fed ~2x sooner while
    // the resident square grows), raw partials into dR; then the second half,
    // each GEMM continuing the promotion chain from dR (acc_init) — the same
    // additions in the same order as one pass over K, so the result is bit-
    // identical to the device call.  K1 ends on a 256-of-K promotion boundary.
    int nphase = dR ? 2 : 1;
    if (const char *ep = getenv("EMM_HOST_KPHASES")) nphase = dR ? std::max(2, std::min(8, atoi(ep))) : 1;
    // phase boundaries on 256-of-K promotion boundaries
    auto kb = [&](int p) { return p >= nphase ? K : (K * p / nphase) / 256 * 256; };
    int ng = 0;
    bool have_partial = false;   // dR holds the raw partial of an executed earlier phase
    for (int ph = 0; ph < nphase && e == cudaSuccess; ++ph) {
        const int64_t k0 = kb(ph), nk = kb(ph + 1) - kb(ph);
        const bool last_phase = ph == nphase - 1;
        if (nk <= 0) continue;
        const bool chain = have_partial;   // continue the promotion chain from dR
        have_partial = true;
        int na = 0, nb = 0;
        while ((na < GM || nb < GN) && e == cudaSuccess) {
            const int64_t rows_res = ra[na], cols_res = cb[nb];
            const bool addA = na < GM && (nb >= GN || rows_res <= cols_res);
            int64_t r0, nr, c0, nc;   // the GEMM's C region
            if (addA) {
                r0 = ra[na];
                nr = ra[na + 1] - r0;
                c0 = 0;
                nc = cols_res;
                e = copy_rows(dA, A, a_rows_ld, lda, r0, nr, k0, nk, K, h2d);
            } else {
                c0 = cb[nb];
                nc = cb[nb + 1] - c0;
                r0 = 0;
                nr = rows_res;
                e = copy_rows(dB, B, b_rows_ld, ldb, c0, nc, k0, nk, K, h2d);
            }
            if (e == cudaSuccess && beta != 0.0f && nr > 0 && nc > 0 && last_phase)   // the C region this step computes
                e = cudaMemcpy2DAsync(dC + r0 + c0 * ldc, (size_t)ldc * 4, C + r0 + c0 * ldc, (size_t)ldc * 4,
                                      (size_t)nr * 4, (size_t)nc, cudaMemcpyHostToDevice, h2d);
            cudaEvent_t landed = ev();
            if (e == cudaSuccess) e = cudaEventRecord(landed, h2d);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, landed, 0);
            // re-buffer the new block once (K-major planes)
            PackArgs pk;
            if (addA) {
                pk.X = a_rows_ld ? dA + r0 + k0 * lda : dA + r0 * lda + k0;
                pk.ld = lda; pk.R = nr; pk.kcontig = !a_rows_ld;
                pk.out0 = Ap + (size_t)r0 * Kp + k0; pk.ld0 = Kp;
                pk.out1 = Ap + (size_t)M * Kp + (size_t)r0 * Kp + k0; pk.ld1 = Kp;
                ++na;
            } else {
                pk.X = b_rows_ld ? dB + c0 + k0 * ldb : dB + c0 * ldb + k0;
                pk.ld = ldb; pk.R = nc; pk.kcontig = !b_rows_ld; pk.b_side = true;
                pk.out0 = Bp + (size_t)c0 * Kp + k0; pk.ld0 = Kp;
                pk.out1 = Bp + (size_t)N * Kp + (size_t)c0 * Kp + k0; pk.ld1 = Kp;
                ++nb;
            }
            if (e == cudaSuccess && !xs) e = launch_pack(pmode, pk, nullptr, nk, nullptr, comp);
            if (nr == 0 || nc == 0 || e != cudaSuccess) continue;
            // the region in pieces along its long side: GEMM, then D2H of the piece
            const bool split_cols = nc >= nr;
            const int64_t len = split_cols ? nc : nr;
            for (int64_t o = 0; o < len && e == cudaSuccess; o += chunk) {
                const int64_t pr0 = split_cols ? r0 : r0 + o, pnr = split_cols ? nr : std::min(chunk, nr - o);
                const int64_t pc0 = split_cols ? c0 + o : c0, pnc = split_cols ? std::min(chunk, nc - o) : nc;
                TcOperands ops;
                const int64_t kext = tc_kpad(nk);   // this phase's K columns of the planes (zero padded)
                ops.a0 = TcPlane{Ap + (size_t)pr0 * Kp + k0, Kp, false, kext};
                ops.b0 = TcPlane{Bp + (size_t)pc0 * Kp + k0, Kp, false, kext};
                if (pl == 2) {
                    ops.a1 = TcPlane{Ap + (size_t)M * Kp + (size_t)pr0 * Kp + k0, Kp, false, kext};
                    ops.b1 = TcPlane{Bp + (size_t)N * Kp + (size_t)pc0 * Kp + k0, Kp, false, kext};
                }
                unsigned int *cw = ctrl + 32 * (ng & 63);   // zeroed once for the first 64 GEMMs
                if (ng++ >= 64) e = cudaMemsetAsync(cw, 0, 128, comp);
                if (xs) {
                    // the block's raw rows / columns, K range [k0, k0 + nk), in place
                    ops.a0 = a_rows_ld ? TcPlane{dA + pr0 + k0 * lda, lda, true, nk}
                                       : TcPlane{dA + pr0 * lda + k0, lda, false, nk};
                    ops.b0 = b_rows_ld ? TcPlane{dB + pc0 + k0 * ldb, ldb, true, nk}
                                       : TcPlane{dB + pc0 * ldb + k0, ldb, false, nk};
                }
                if (e == cudaSuccess) {
                    const float *ai = chain ? dR + pr0 + pc0 * M : nullptr;
                    float *co = last_phase ? dC + pr0 + pc0 * ldc : dR + pr0 + pc0 * M;
                    const int64_t ldo = last_phase ? ldc : M;
                    // not last: raw partial of the K prefix (continuing the previous phases')
                    const float al = last_phase ? alpha : 1.0f, be = last_phase ? beta : 0.0f;
                    e = xs ? launch_tc_xs_sgemm(ops.a0, ops.b0, pnr, pnc, nk, al, be, co, ldo, cw, 1, nullptr, comp,
                                                nullptr, nullptr, ai, M)
                           : launch_tc_sgemm(terms, ops, pnr, pnc, nk, al, be, co, ldo, cw, 1, nullptr, comp, nullptr,
                                             nullptr, ai, M);
                }
                if (!last_phase) continue;
                cudaEvent_t done = ev();
                if (e == cudaSuccess) e = cudaEventRecord(done, comp);
                if (e == cudaSuccess) e = cudaStreamWaitEvent(d2h, done, 0);
                if (e == cudaSuccess)
                    e = cudaMemcpy2DAsync(C + pr0 + pc0 * ldc, (size_t)ldc * 4, dC + pr0 + pc0 * ldc, (size_t)ldc * 4,
                                          (size_t)pnr * 4, (size_t)pnc, cudaMemcpyDeviceToHost, d2h);
            }
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(comp);
    return cuda_status(e);
}

extern "C" int emm_sgemm_host(char transA, char transB, int64_t M, int64_t N, int64_t K, float alpha, const float *A,
                              int64_t lda, const float *B, int64_t ldb, float beta, float *C, int64_t ldc,
                              emm_math_t math) {
    int st = check_args(transA, transB, M, N, K, lda, ldb, ldc);
    if (st) return st;
    if (!math_ok(math)) return EMM_ERR_MATH;
    if (M == 0 || N == 0) return 0;
    const bool ab_used = !(alpha == 0.0f || K == 0);
    if (!ab_used && beta == 1.0f) return 0;
    if (C == nullptr) return -12;
    if (ab_used && A == nullptr) return -7;
    if (ab_used && B == nullptr) return -9;
    if ((st = check_device())) return st;
    std::lock_guard<std::mutex> g(g_host_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_hc.dev != dev || !g_hc.s) {
        if (g_hc.s) cudaStreamDestroy(g_hc.s);
        g_hc = HostCache{};
        cudaError_t e = cudaStreamCreateWithFlags(&g_hc.s, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_status(e);
        g_hc.dev = dev;
    }
    const int64_t ar = is_n(transA) ? M : K, ac = is_n(transA) ? K : M;
    const int64_t br = is_n(transB) ? K : N, bc = is_n(transB) ? N : K;
    const size_t nA = ab_used ? (size_t)((ac - 1) * lda + ar) * 4 : 0;
    const size_t nB = ab_used ? (size_t)((bc - 1) * ldb + br) * 4 : 0;
    const size_t nC = (size_t)((N - 1) * ldc + M) * 4;
    if ((st = ensure(&g_hc.dA, &g_hc.nA, nA)) || (st = ensure(&g_hc.dB, &g_hc.nB, nB)) ||
        (st = ensure(&g_hc.dC, &g_hc.nC, nC)))
        return st;
    // device copies keep the caller's leading dimensions: size the workspace
    // for them (the FFMA relayout only when they are TN / TMA-illegal)
    const size_t nW = ab_used ? call_ws_bytes(transA, transB, M, N, K, math, (const float *)g_hc.dA, lda,
                                              (const float *)g_hc.dB, ldb)
                              : 0;
    cudaStream_t s = g_hc.s;
    cudaError_t e = cudaSuccess;
    if (ab_used && math != EMM_MATH_FFMA && M >= 4096 && N >= 4096 && K >= 256 && !env_on("EMM_HOST_NO_PIPELINE")) {
        const int64_t Kp = tc_kpad(K);
        const size_t pl = (size_t)planes_of(math);
        // 3xTF32 on TMA-legal device copies: KN1X on the landed blocks in
        // place (no re-buffered planes); EMM_HOST_PACK=1 keeps the planes
        const bool xs = math == EMM_MATH_3XTF32 && prefer_xs(M, N, K) && tma_legal(g_hc.dA, lda) &&
                        tma_legal(g_hc.dB, ldb) && !env_on("EMM_HOST_PACK");
        const size_t nP = (xs ? 0 : align_up(pl * (size_t)(M + N) * Kp * 4, 1024)) + 64 * 128;
        if ((st = ensure(&g_hc.dW, &g_hc.nW, nP))) return st;
        // K phases for the FP32-accurate splits at large K (EMM_HOST_KSPLIT=0/1)
        const char *ek = getenv("EMM_HOST_KSPLIT");
        const bool ksplit = math != EMM_MATH_1XTF32 && (ek ? ek[0] == '1' : K >= 8192) && K >= 512;
        if (ksplit && (st = ensure(&g_hc.dR, &g_hc.nR, (size_t)M * N * 4))) return st;
        return host_pipelined(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, math,
                              (float *)g_hc.dA, (float *)g_hc.dB, (float *)g_hc.dC, g_hc.dW,
                              ksplit ? (float *)g_hc.dR : nullptr, xs);
    }
    if ((st = ensure(&g_hc.dW, &g_hc.nW, nW))) return st;
    if (ab_used) {
        e = cudaMemcpyAsync(g_hc.dA, A, nA, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(g_hc.dB, B, nB, cudaMemcpyHostToDevice, s);
    }
    if (e == cudaSuccess && beta != 0.0f) e = cudaMemcpyAsync(g_hc.dC, C, nC, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e);
    st = emm_sgemm_ex(transA, transB, M, N, K, alpha, (const float *)g_hc.dA, lda, (const float *)g_hc.dB, ldb, beta,
                      (float *)g_hc.dC, ldc, s, math, g_hc.dW, g_hc.nW);
    if (st) return st;
    // copy back column by column only if ldc padding must be preserved
    if (ldc == M || N == 1) {
        e = cudaMemcpyAsync(C, g_hc.dC, (size_t)M * N * 4, cudaMemcpyDeviceToHost, s);
    } else {
        e = cudaMemcpy2DAsync(C, (size_t)ldc * 4, g_hc.dC, (size_t)ldc * 4, (size_t)M * 4, (size_t)N,
                              cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return cuda_status(e);
}

extern "C" void emm_release_cache(void) {
    std::lock_guard<std::mutex> g(g_host_mu);
    if (g_hc.dA) cudaFree(g_hc.dA);
    if (g_hc.dB) cudaFree(g_hc.dB);
    if (g_hc.dC) cudaFree(g_hc.dC);
    if (g_hc.dW) cudaFree(g_hc.dW);
    if (g_hc.dR) cudaFree(g_hc.dR);
    if (g_hc.s) cudaStreamDestroy(g_hc.s);
    g_hc = HostCache{};
}

// ------------------------------------------------------------ partition
extern "C" void emm_row_partition(int64_t M, int nranks, int rank, int64_t *row0, int64_t *rows) {
    const int64_t T = 256;  // rows per CTA-pair tile
    if (nranks < 1 || rank < 0 || rank >= nranks || M <= 0) {
        if (row0) *row0 = 0;
        if (rows) *rows = 0;
        return;
    }
    const int64_t tiles = (M + T - 1) / T;
    const int64_t base = tiles / nranks, extra = tiles % nranks;
    // the last `extra` ranks take one more tile
    const int64_t first_big = nranks - extra;
    const int64_t t0 = rank * base + (rank > first_big ? rank - first_big : 0);
    const int64_t nt = base + (rank >= first_big ? 1 : 0);
    int64_t r0 = t0 * T, r1 = (t0 + nt) * T;
    if (r0 > M) r0 = M;
    if (r1 > M) r1 = M;
    if (row0) *row0 = r0;
    if (rows) *rows = r1 - r0;
}

// ------------------------------------------------------------ introspection
extern "C" const char *emm_strerror(int status) {
    static thread_local char buf[160];
    if (status == 0) return "success";
    if (status <= -1 && status >= -13) {
        static const char *names[] = {"", "transA", "transB", "M", "N", "K", "alpha", "A", "lda", "B", "ldb", "beta",
                                      "C", "ldc"};
        snprintf(buf, sizeof buf, "invalid argument %d (%s)", -status, names[-status]);
        return buf;
    }
    switch (status) {
        case EMM_ERR_ALIAS: return "C overlaps A or B";
        case EMM_ERR_ARCH: return "device is not compute capability 10.0 (sm_100a build)";
        case EMM_ERR_WORKSPACE: return "workspace too small or not 1024-byte aligned";
        case EMM_ERR_MATH: return "unknown math mode";
        case EMM_ERR_COMM: return "invalid communicator or NCCL unavailable";
        case EMM_ERR_NOMEM: return "allocation failed";
        default: break;
    }
    if (status >= EMM_ERR_NCCL_BASE) {
        snprintf(buf, sizeof buf, "NCCL error %d", status - EMM_ERR_NCCL_BASE);
        return buf;
    }
    if (status >= EMM_ERR_CUDA_BASE) {
        snprintf(buf, sizeof buf, "CUDA error %d (%s)", status - EMM_ERR_CUDA_BASE,
                 cudaGetErrorString((cudaError_t)(status - EMM_ERR_CUDA_BASE)));
        return buf;
    }
    return "unknown status";
}

extern "C" const char *emm_version(void) {
    return "emm 0.3 (sm_100a: tcgen05 3xTF32 split in the kernel / TF32+BF16 / 1xTF32, TMA-fed FFMA, TMEM-fed skinny)";
}

extern "C" uint64_t emm_launch_count(void) { return g_launches.load(); }

extern "C" void emm_profile_enable(int on) { g_prof_on.store(on ? 1 : 0); }

extern "C" int emm_profile_read(double *gemm_ms, uint64_t *gemm_launches, double *other_ms, uint64_t *other_launches) {
    std::vector<ProfRec> recs;
    {
        std::lock_guard<std::mutex> g(g_prof_mu);
        recs.swap(g_prof);
    }
    double gm = 0, om = 0;
    uint64_t gn = 0, on = 0;
    int st = 0;
    for (auto &r : recs) {
        float ms = 0;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess && !st) st = EMM_ERR_CUDA_BASE + (int)e;
        if (r.gemm) { gm += ms; ++gn; } else { om += ms; ++on; }
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    if (gemm_ms) *gemm_ms = gm;
    if (gemm_launches) *gemm_launches = gn;
    if (other_ms) *other_ms = om;
    if (other_launches) *other_launches = on;
    return st;
}
