/*
 * oracle/oracle.c — the parity ORACLE for the emm SGEMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this file.
 * It shares no code, header, constant or helper with the CUDA path
 * (paper_1912_04379_b200/csrc, include/emm.h) and neither side includes the
 * other.
 *
 * What it computes — the plain definition of the paper's operation:
 *   "dense matrix-matrix multiplication requires 2MNK floating point
 *    operations where A: M x K and B: K x N"           (§Introduction)
 *   C_{i,j} <- A_{i,1}B_{1,j} + A_{i,2}B_{2,j} + ... + A_{i,K}B_{K,j}
 *                                                     (eq. in §L0 blocking)
 *   with the Level-3 BLAS SGEMM interface              (§Introduction):
 *   C <- alpha*op(A)*op(B) + beta*C, column-major, transA/transB, lda/ldb/ldc.
 *
 * The paper's own baseline is the naive three-loop multiply of Fig. f:dumb
 * (PAPER.md:518-532).  This oracle is that loop nest, evaluated in FP64
 * (reading R1: north_star asks for "a plain CPU triple loop with FP64
 * accumulation"), over column-major storage (reading R2) with BLAS alpha/beta
 * semantics (reading R4).  No blocking, packing or reordering: each entry is
 * summed over p = 0..K-1 in increasing order, exactly like the inner loop of
 * Fig. f:dumb.  Products of two floats are exact in double (24+24 <= 53
 * significand bits), so the only rounding is the sequential double sum.
 *
 * Outputs per selected entry (i, j):
 *   R = (double)alpha * s + (beta == 0 ? 0 : (double)beta * (double)C[i,j])
 *       with s = sum_p opA(i,p)*opB(p,j)   (FP64, not rounded to float)
 *   S = |alpha| * sum_p |opA(i,p)*opB(p,j)|    (tolerance scale, north_star)
 *   T = |beta * C[i,j]|                     (0 when beta == 0; C not read)
 * alpha == 0 or K == 0: s = t = 0 and A, B are never read.
 * M == 0 or N == 0: nothing is touched.
 *
 * Build:  gcc -O2 -ffp-contract=off -fPIC -shared -pthread (no -ffast-math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* BLAS argument numbering for SGEMM (1-based):
 * transA=1 transB=2 M=3 N=4 K=5 alpha=6 A=7 lda=8 B=9 ldb=10 beta=11 C=12 ldc=13 */
static int is_trans_char(char t) {
    return t == 'N' || t == 'n' || t == 'T' || t == 't' || t == 'C' || t == 'c';
}
static int notrans(char t) { return t == 'N' || t == 'n'; }
static int64_t max1(int64_t v) { return v > 1 ? v : 1; }

/* Independent statement of the BLAS SGEMM argument rules (reading R4).
 * Returns 0 or -i for the first invalid argument i. */
int oracle_check_args(char transA, char transB, int64_t M, int64_t N, int64_t K,
                      int64_t lda, int64_t ldb, int64_t ldc) {
    if (!is_trans_char(transA)) return -1;
    if (!is_trans_char(transB)) return -2;
    if (M < 0) return -3;
    if (N < 0) return -4;
    if (K < 0) return -5;
    if (lda < max1(notrans(transA) ? M : K)) return -8;
    if (ldb < max1(notrans(transB) ? K : N)) return -10;
    if (ldc < max1(M)) return -13;
    return 0;
}

typedef struct {
    char transA, transB;
    int64_t M, N, K;
    double alpha, beta;
    const float *A, *B, *C;
    int64_t lda, ldb, ldc;
    int64_t nrows, ncols;
    const int64_t *rows, *cols;
    double *R, *S, *T;
    int64_t ldr;
    int64_t j0, j1;        /* this thread's range of selected columns */
} job_t;

static inline double opA(const job_t *q, int64_t i, int64_t p) {
    return notrans(q->transA) ? (double)q->A[i + p * q->lda] : (double)q->A[p + i * q->lda];
}
static inline double opB(const job_t *q, int64_t p, int64_t j) {
    return notrans(q->transB) ? (double)q->B[p + j * q->ldb] : (double)q->B[j + p * q->ldb];
}

static void *run_columns(void *arg) {
    const job_t *q = (const job_t *)arg;
    const int use_ab = !(q->alpha == 0.0 || q->K == 0);
    double *s = (double *)calloc((size_t)(q->nrows > 0 ? q->nrows : 1), sizeof(double));
    double *t = (double *)calloc((size_t)(q->nrows > 0 ? q->nrows : 1), sizeof(double));
    for (int64_t jj = q->j0; jj < q->j1; ++jj) {
        const int64_t j = q->cols ? q->cols[jj] : jj;
        for (int64_t ii = 0; ii < q->nrows; ++ii) { s[ii] = 0.0; t[ii] = 0.0; }
        if (use_ab) {
            /* Loop order j -> p -> i: for every entry the products are still
             * added in increasing p, one at a time, as in Fig. f:dumb's inner
             * loop; only independent entries are interleaved. */
            for (int64_t p = 0; p < q->K; ++p) {
                const double b = opB(q, p, j);
                for (int64_t ii = 0; ii < q->nrows; ++ii) {
                    const int64_t i = q->rows ? q->rows[ii] : ii;
                    const double x = opA(q, i, p) * b;   /* exact in double */
                    s[ii] += x;
                    t[ii] += fabs(x);
                }
            }
        }
        for (int64_t ii = 0; ii < q->nrows; ++ii) {
            const int64_t i = q->rows ? q->rows[ii] : ii;
            double r = q->alpha * s[ii];
            double tt = 0.0;
            if (q->beta != 0.0) {
                const double bc = q->beta * (double)q->C[i + j * q->ldc];
                r += bc;
                tt = fabs(bc);
            }
            q->R[ii + jj * q->ldr] = r;
            if (q->S) q->S[ii + jj * q->ldr] = fabs(q->alpha) * t[ii];
            if (q->T) q->T[ii + jj * q->ldr] = tt;
        }
    }
    free(s);
    free(t);
    return NULL;
}

/*
 * Evaluate the selected entries (rows[] x cols[]) of alpha*op(A)*op(B)+beta*C.
 * rows == NULL means rows 0..M-1 (nrows must equal M); likewise cols.
 * R, S, T are nrows x ncols column-major with leading dimension ldr.
 * Threads split the selected columns; each entry's arithmetic is independent
 * of the thread count.  Returns the oracle_check_args code (C untouched on
 * error); M == 0 or N == 0 returns 0 having written nothing.
 */
int oracle_sgemm_sub(char transA, char transB, int64_t M, int64_t N, int64_t K,
                     float alpha, const float *A, int64_t lda,
                     const float *B, int64_t ldb,
                     float beta, const float *C, int64_t ldc,
                     int64_t nrows, const int64_t *rows,
                     int64_t ncols, const int64_t *cols,
                     double *R, double *S, double *T, int64_t ldr,
                     int nthreads) {
    int st = oracle_check_args(transA, transB, M, N, K, lda, ldb, ldc);
    if (st) return st;
    if (M == 0 || N == 0 || nrows == 0 || ncols == 0) return 0;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > ncols) nthreads = (int)ncols;
    job_t base;
    memset(&base, 0, sizeof base);
    base.transA = transA; base.transB = transB;
    base.M = M; base.N = N; base.K = K;
    base.alpha = (double)alpha; base.beta = (double)beta;
    base.A = A; base.B = B; base.C = C;
    base.lda = lda; base.ldb = ldb; base.ldc = ldc;
    base.nrows = nrows; base.ncols = ncols; base.rows = rows; base.cols = cols;
    base.R = R; base.S = S; base.T = T; base.ldr = ldr;
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * (size_t)nthreads);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int w = 0; w < nthreads; ++w) {
        jobs[w] = base;
        jobs[w].j0 = ncols * w / nthreads;
        jobs[w].j1 = ncols * (w + 1) / nthreads;
    }
    for (int w = 1; w < nthreads; ++w) pthread_create(&th[w], NULL, run_columns, &jobs[w]);
    run_columns(&jobs[0]);
    for (int w = 1; w < nthreads; ++w) pthread_join(th[w], NULL);
    free(jobs);
    free(th);
    return 0;
}

/* Drop-in form: C <- (float)R over the whole M x N region (round to nearest).
 * Used by the CPU-baseline leg of bench.py; ldc padding is never written. */
int oracle_sgemm(char transA, char transB, int64_t M, int64_t N, int64_t K,
                 float alpha, const float *A, int64_t lda, const float *B, int64_t ldb,
                 float beta, float *C, int64_t ldc, int nthreads) {
    int st = oracle_check_args(transA, transB, M, N, K, lda, ldb, ldc);
    if (st) return st;
    if (M == 0 || N == 0) return 0;
    double *R = (double *)malloc(sizeof(double) * (size_t)M * (size_t)N);
    if (!R) return 1;
    st = oracle_sgemm_sub(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                          M, NULL, N, NULL, R, NULL, NULL, M, nthreads);
    for (int64_t j = 0; j < N && !st; ++j)
        for (int64_t i = 0; i < M; ++i) C[i + j * ldc] = (float)R[i + j * M];
    free(R);
    return st;
}
