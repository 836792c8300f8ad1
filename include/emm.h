/*
 * emm.h — C ABI of the B200-native SGEMM ("emm", after the paper's Emmerald).
 *
 * The operation (the method's hot path, BASELINE.json north_star):
 *
 *     C <- alpha * op(A) * op(B) + beta * C          (single precision)
 *
 * is the Level-3 BLAS SGEMM the paper implements ("Emmerald implements the
 * SGEMM interface of Level-3 BLAS", §Introduction) — dense
 * matrix multiplication of A: M x K by B: K x N in 2MNK flops
 * (PAPER.md:33-38), each C_ij the dot product of PAPER.md:277-279 (§L0
 * blocking, eq. 1).  Storage is COLUMN-major (reading R2):
 * element (r, c) of an array X with leading dimension ld is X[r + c*ld].
 *
 *   transA = 'N'/'n': A is stored M x K, lda >= max(1, M)
 *            'T'/'t'/'C'/'c': A is stored K x M, lda >= max(1, K)
 *   transB = 'N'/'n': B is stored K x N, ldb >= max(1, K)
 *            'T'/'t'/'C'/'c': B is stored N x K, ldb >= max(1, N)
 *   C is M x N, ldc >= max(1, M).    ('C' means 'T' for real data.)
 *
 * Ownership / lifetime: every matrix pointer of emm_sgemm* is a DEVICE
 * pointer owned by the caller (allocated e.g. with torch), valid until
 * `stream` reaches the enqueued work.  The library keeps no pointer after
 * return.  All calls are stream-ordered and asynchronous (no host sync),
 * except emm_sgemm_host which is synchronous.  `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream).
 *
 * Semantics (reading R4 in DESIGN.md):
 *   beta == 0 (incl. -0.0): C is never read (NaN/Inf in C do not propagate).
 *   alpha == 0 or K == 0: A and B are never read; C <- beta*C.
 *   Quick return (nothing launched) when M == 0, N == 0, or
 *   ((alpha == 0 or K == 0) and beta == 1).
 *   Only the M x N logical region of C is written; ldc padding never is.
 *   Results are run-to-run deterministic: no floating-point atomics; split-K
 *   and stream-K partials are added in a fixed order.
 *   Reentrant; concurrent calls on different streams are safe when their C
 *   ranges are disjoint.
 *
 * Errors: 0 = success.  -i = BLAS argument i invalid (transA=1 transB=2 M=3
 * N=4 K=5 A=7 lda=8 B=9 ldb=10 C=12 ldc=13; a NULL or non-4-byte-aligned
 * pointer is rejected only when that operand would be read or written).
 * Negative EMM_ERR_* below; 1000 + cudaError_t for CUDA errors; 2000 +
 * ncclResult_t for NCCL errors.  On any argument error C is unmodified and
 * nothing is launched.
 */
#ifndef EMM_H_
#define EMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMM_SUCCESS 0
#define EMM_ERR_ALIAS (-100)      /* C's byte range overlaps A's or B's          */
#define EMM_ERR_ARCH (-101)       /* current device is not compute capability 10.0 */
#define EMM_ERR_WORKSPACE (-102)  /* workspace too small / misaligned            */
#define EMM_ERR_MATH (-103)       /* unknown emm_math_t                          */
#define EMM_ERR_COMM (-104)       /* bad communicator / NCCL unavailable         */
#define EMM_ERR_NOMEM (-105)      /* host or device allocation failed            */
#define EMM_ERR_CUDA_BASE 1000
#define EMM_ERR_NCCL_BASE 2000

/* Arithmetic of the product.  All report 2MNK flops.
 *   EMM_MATH_3XTF32: FP32-accurate tcgen05 tensor-core path; each operand is
 *     split x = big + small (big = rn_tf32(x), small = rn_tf32(x - big)) and
 *     C accumulates small*big + big*small + big*big in FP32 in TMEM.
 *   EMM_MATH_FFMA:   FP32 FFMA on CUDA cores (register-blocked tiles).
 *   EMM_MATH_1XTF32: one TF32 product per step (exposed lower precision).
 *   EMM_MATH_TF32_BF16: FP32-accurate tensor-core split with 2/3 of the
 *     3xTF32 tensor work: big*big as one TF32 MMA per K8 and both cross terms
 *     a_big*b_small + a_small*b_big as ONE K16 BF16 MMA on [a_big|a_small] x
 *     [b_small;b_big] (per-product error <= ~2^-18 |ab|, inside the FP32-
 *     accurate bound 1e-5*sum|ab|). */
typedef enum {
    EMM_MATH_3XTF32 = 0,
    EMM_MATH_FFMA = 1,
    EMM_MATH_1XTF32 = 2,
    EMM_MATH_TF32_BF16 = 3
} emm_math_t;

/* C <- alpha*op(A)*op(B) + beta*C with the default FP32-accurate path
 * (EMM_MATH_3XTF32).  Scratch for the operand split is taken from a
 * stream-ordered memory pool the library owns (cudaMallocFromPoolAsync /
 * cudaFreeAsync on `stream`; the device default pool is not modified). */
int emm_sgemm(char transA, char transB, int64_t M, int64_t N, int64_t K,
              float alpha, const float *A, int64_t lda,
              const float *B, int64_t ldb,
              float beta, float *C, int64_t ldc, void *stream);

/* Same, with an explicit math mode and an optional caller-owned device
 * workspace (>= emm_sgemm_workspace_bytes(...), 1024-byte aligned).
 * workspace == NULL -> stream-ordered pool as in emm_sgemm. */
int emm_sgemm_ex(char transA, char transB, int64_t M, int64_t N, int64_t K,
                 float alpha, const float *A, int64_t lda,
                 const float *B, int64_t ldb,
                 float beta, float *C, int64_t ldc, void *stream,
                 emm_math_t math, void *workspace, size_t workspace_bytes);

/* Device workspace the call above needs (an upper bound over leading
 * dimensions and pointer alignment: TMA-illegal operands need a re-pitched
 * copy; EMM_MATH_FFMA also a transposed copy for transA = T / transB = N and
 * split-K partial slabs on sub-wave grids; 0 for latency-bound sizes that
 * take the tiny kernel).  Host-only. */
size_t emm_sgemm_workspace_bytes(char transA, char transB, int64_t M, int64_t N,
                                 int64_t K, emm_math_t math);

/* End-to-end form: A, B, C are HOST pointers (pinned or pageable; pinned
 * for full PCIe speed; same layouts as above).  Copies A, B (and C when
 * beta != 0) to device buffers cached by the library and copies C back;
 * returns when C holds the result (synchronous).  Tensor-core modes with
 * M, N >= 4096 pipeline it over 2048-row / 2048-column blocks on three
 * internal streams (copies in both directions overlap the GEMMs, DESIGN.md
 * §6b); other calls copy, run emm_sgemm_ex on an internal stream, and copy
 * back.  Not reentrant with itself (serialised by a library mutex). */
int emm_sgemm_host(char transA, char transB, int64_t M, int64_t N, int64_t K,
                   float alpha, const float *A, int64_t lda,
                   const float *B, int64_t ldb,
                   float beta, float *C, int64_t ldc, emm_math_t math);

/* Frees the device buffers cached by emm_sgemm_host.  Host-only. */
void emm_release_cache(void);

/* ----------------------------------------------------------------------
 * Row-sharded multi-GPU SGEMM (BASELINE.json north_star, "Multi-GPU":
 * C row blocks per rank, B broadcast, optional C all-gather over NCCL).
 * One process per GPU.  The communicator wraps NCCL (loaded at run time).
 * -------------------------------------------------------------------- */

/* Rank r's block of rows of C (and of op(A)): [*row0, *row0 + *rows).
 * Blocks are multiples of 256 rows (the tensor-core tile of a CTA pair)
 * except the last, balanced to within one tile; they tile [0, M) exactly in
 * rank order.  Host-only; valid for nranks >= 1, 0 <= rank < nranks. */
void emm_row_partition(int64_t M, int nranks, int rank, int64_t *row0, int64_t *rows);

/* Width (columns) of the B column panels emm_sgemm_multi broadcasts one at a
 * time (the last panel may be narrower): ~N/4, >= 1024, multiple of 256.
 * Host-only. */
int64_t emm_multi_panel_cols(int64_t N);

/* 128-byte NCCL unique id, produced on one rank and distributed by the
 * caller (e.g. torch.distributed broadcast).  Returns EMM_ERR_COMM if NCCL
 * cannot be loaded. */
int emm_get_unique_id(void *id128);
/* Collective (NCCL communicator over `nranks` processes, one GPU each).  It
 * also maps every peer's flag words by CUDA IPC for the copy-engine data
 * plane; if any rank cannot map them, every rank still gets a working
 * communicator for the NCCL data plane and the registrations below then fail
 * with EMM_ERR_COMM on every rank. */
int emm_comm_create(void **comm, const void *id128, int nranks, int rank);
int emm_comm_destroy(void *comm);

/* Collective: every rank calls with identical (trans, M, N, K, alpha, beta,
 * root, math) and the same registrations (below).  A_local: this rank's rows of op(A) as an (rows x K) op-matrix
 * (transA='N': stored rows x K with lda >= rows; 'T': stored K x rows).
 * B: K x N op(B) storage, valid on `root`; on other ranks a buffer of the
 * same size that receives it (broadcast in column panels, each panel's
 * GEMM overlapping the next panel's transfer).  C_local: this rank's rows x N
 * block (ldc >= rows).  C_full (nullable): if set, receives the whole M x N
 * result on every rank (ldc_full >= M).  ldb must equal the stored rows of B
 * (panels are contiguous).
 * Data plane: if B is the buffer registered with emm_comm_register_input,
 * B travels along the ring root -> root+1 -> ... -> root-1 in <= 64 MB
 * chunks by peer copies on the copy engines (no SMs taken from the GEMMs),
 * each chunk signalled by a release flag the receiver's GEMM waits on;
 * otherwise by ncclBroadcast per panel.  If C_full is the buffer registered
 * with emm_comm_register_output, each rank's rows are stored straight into
 * every rank's C_full (by the GEMM epilogue in tensor-core modes, by peer
 * copies otherwise) and per-rank flags complete the call; otherwise NCCL
 * all-gather + unpack.  All of it is stream-ordered on `stream`: C_local and
 * C_full are complete when `stream` reaches the end of the call.  The call
 * order of the ranks' host threads is free (waits are device-side). */
int emm_sgemm_multi(void *comm, char transA, char transB, int64_t M, int64_t N, int64_t K,
                    float alpha, const float *A_local, int64_t lda,
                    float *B, int64_t ldb, int root,
                    float beta, float *C_local, int64_t ldc,
                    float *C_full, int64_t ldc_full, void *stream, emm_math_t math);

/* Collective: register this rank's full-output buffer (M x N, ld_full; the
 * same layout on every rank) with the communicator.  CUDA IPC handles are
 * exchanged over NCCL and the peers' buffers mapped.  Afterwards
 * emm_sgemm_multi(..., C_full = that buffer, ldc_full) fuses the all-gather
 * into the GEMM: each rank's epilogue stores its C rows into every rank's
 * C_full over NVLink (tensor-core modes; other modes copy their rows), and
 * each rank then stores the call's epoch into every rank's "done" words and
 * waits for all of them (stream-ordered, no NCCL collective).  The buffer must stay allocated until
 * emm_comm_unregister_output / emm_comm_destroy.  The outcome is agreed
 * across ranks: 0 on every rank, or EMM_ERR_COMM on every rank (a rank could
 * not export or map a buffer; nothing stays registered, and emm_sgemm_multi
 * with that C_full uses the NCCL all-gather). */
int emm_comm_register_output(void *comm, float *C_full, int64_t ld_full);
int emm_comm_unregister_output(void *comm);

/* Collective: register this rank's B buffer (`bytes` >= the stored size of
 * B of the calls that use it; the source on root, the receive buffer
 * elsewhere).  Only the ring successor's buffer is mapped (CUDA IPC).  Must
 * stay allocated until emm_comm_unregister_input / emm_comm_destroy.  The
 * outcome is agreed across ranks as for emm_comm_register_output (on
 * EMM_ERR_COMM, B is broadcast by NCCL). */
int emm_comm_register_input(void *comm, float *B, size_t bytes);
int emm_comm_unregister_input(void *comm);

/* Test harness: `nranks` VIRTUAL ranks on the current device.  comms[r]
 * (r < nranks) receives rank r's communicator; each is used and destroyed
 * like one from emm_comm_create.  Their exchange steps run as device copies
 * between distinct buffers on this GPU (no NCCL), ordered by CUDA events
 * instead of device flags (no kernel spins on another rank's work on one
 * GPU), so B and, when gathered, C_full must be registered.  Each virtual
 * rank needs its OWN stream.  A call enqueues nothing until every rank of
 * the world has made it; the last caller enqueues all ranks' work (earlier
 * callers get 0; errors are returned to the last caller), and until then a
 * rank's stream must receive no other work.
 * Returns 0 or EMM_ERR_COMM / 1000 + cudaError_t. */
int emm_debug_comm_create_local(int nranks, void **comms);

/* ----------------------------------------------------------------------
 * Introspection (host-only).
 * -------------------------------------------------------------------- */
const char *emm_strerror(int status);
const char *emm_version(void);
/* Number of kernels this library has launched in this process. */
uint64_t emm_launch_count(void);
/* Optional per-kernel CUDA-event timing of the dominant kernel (the GEMM
 * main loop): enable, run, then read the summed device milliseconds and the
 * number of timed launches (synchronises the recorded events). */
void emm_profile_enable(int on);
int emm_profile_read(double *gemm_ms, uint64_t *gemm_launches, double *other_ms,
                     uint64_t *other_launches);

/* ----------------------------------------------------------------------
 * Measurement probe (not part of the SGEMM path).  Runs the tensor-core
 * GEMM's MMA stream (tcgen05.mma cta_group::2 M256xN256xK8 per CTA pair,
 * terms = 3: 3xTF32, 2: TF32+BF16, 1: 1xTF32) for `stages` K-stages of 32
 * on every CTA pair with the operands resident in shared memory — the tensor
 * pipe's ceiling without TMA/L2/DRAM traffic (confirm the
 * TF32 peak with a tcgen05 microbenchmark).  Synchronous: returns the
 * CUDA-event time of the launch in *ms and, in *gemm_flops, the 2MNK a GEMM
 * would report for the same work.  Returns 0, EMM_ERR_MATH (bad terms or
 * stages) or 1000 + cudaError_t.
 * -------------------------------------------------------------------- */
int emm_debug_mma_probe(int terms, int stages, void *stream, float *ms, double *gemm_flops);

/* Host replays of the tcgen05 GEMM's persistent schedule (host-only, no GPU;
 * they run the same __host__ __device__ scheduling code as the kernel, for
 * tests).  emm_debug_schedule: the work items of every CTA pair of a launch,
 * 7 ints each (pair, m0, n0, kb0, kb1, kind, last).  emm_debug_pair_schedule:
 * the items every pair runs on preferred clusters of 4 (data-parallel
 * schedule), 8 ints each (pair, i, m0, n0, kb0, kb1, dummy, multicast).
 * Both return the item count, or -1 when `cap` items do not fit in `out`. */
int emm_debug_schedule(int64_t M, int64_t N, int64_t K, int use_sk, int terms, int *out, int cap);
/* Host replay of emm_sgemm_multi's B chunk plan (copy-engine ring): chunk j
 * covers bytes [out_off[j], out_off[j+1]) of B (n + 1 offsets), panel p
 * chunks [out_pc[p], out_pc[p+1]).  Returns n, or -1 if cap_off / cap_pc are
 * too small. */
int emm_debug_ring_chunks(int64_t N, int64_t K, char transB, int64_t *out_off, int cap_off, int64_t *out_pc,
                          int cap_pc);
int emm_debug_pair_schedule(int64_t M, int64_t N, int64_t K, int *out, int cap);

#ifdef __cplusplus
}
#endif
#endif /* EMM_H_ */
