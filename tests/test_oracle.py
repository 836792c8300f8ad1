"""Pins of the CPU oracle (oracle/oracle.c) against what the paper and the
mathematics fix — never against a retyped copy of its own loop.

Pins (SURVEY.md §8(c) "What pins each part"):
* brute force in exact rational arithmetic on every tiny shape, all trans,
  two leading dimensions, several alpha/beta — the logical op(A), op(B) are
  built by numpy reshapes/transposes, not by the oracle's index formula;
* (AB)^T = B^T A^T, bitwise (same products, same order);
* closed forms: all-ones -> K, identity -> op(A), alpha=0 -> beta*C with NaN
  A/B never read, beta=0 -> NaN C never read, K=0, K=1 outer product;
* the worked examples in tests/golden/ (cited there);
* math.fsum (a correctly rounded exact dot product) within the FP64
  sequential-sum bound (K-1) 2^-53 t;
* numpy float64 matmul (a BLAS dgemm) within 1e-12 (t+T);
* argument errors with BLAS numbering; thread-count and subset invariance.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import datagen

HERE = os.path.dirname(os.path.abspath(__file__))
U53 = 2.0 ** -53


def stored_shape(trans, rows_op, cols_op):
    """Stored (rows, cols) of a column-major array holding op(X) (rows_op x cols_op)."""
    return (rows_op, cols_op) if trans in "Nn" else (cols_op, rows_op)


def logical(flat, trans, rows_op, cols_op, ld):
    """op(X) as a 2-D numpy array, via numpy's Fortran-order reshape of the
    storage and numpy's transpose (independent of the oracle's indexing)."""
    sr, sc = stored_shape(trans, rows_op, cols_op)
    if sr * sc == 0:
        return np.zeros((rows_op, cols_op), dtype=flat.dtype)
    store = np.reshape(flat[: ld * sc], (ld, sc), order="F")[:sr, :]
    return store if trans in "Nn" else store.T


def rand_flat(rng, rows, cols, ld, kind="small"):
    n = max(ld * max(cols, 1), 1)
    if kind == "small":
        # values k/8 with k in [-16,16]: exact binary fractions
        v = rng.integers(-16, 17, size=n).astype(np.float32) / 8
    else:
        v = rng.uniform(-1, 1, size=n).astype(np.float32)
    return v


# --------------------------------------------------------------------------
# brute force, exact rationals
# --------------------------------------------------------------------------
@pytest.mark.parametrize("transA", ["N", "T"])
@pytest.mark.parametrize("transB", ["N", "T"])
def test_bruteforce_exact_rationals(transA, transB):
    rng = np.random.default_rng(1234)
    alphas = [0.0, 1.0, -0.75]
    betas = [0.0, 1.0, 1.25]
    for M in range(0, 4):
        for N in range(0, 4):
            for K in range(0, 4):
                for pad in (0, 3):
                    sa = stored_shape(transA, M, K)
                    sb = stored_shape(transB, K, N)
                    lda, ldb, ldc = max(1, sa[0]) + pad, max(1, sb[0]) + pad, max(1, M) + pad
                    A = rand_flat(rng, *sa, lda, "uniform")
                    B = rand_flat(rng, *sb, ldb, "uniform")
                    C = rand_flat(rng, M, N, ldc, "uniform")
                    opA = logical(A, transA, M, K, lda)
                    opB = logical(B, transB, K, N, ldb)
                    Cl = logical(C, "N", M, N, ldc)
                    for al in alphas:
                        for be in betas:
                            R, S, T, st = oracle.sgemm_sub(transA, transB, M, N, K, al, A, lda, B,
                                                          ldb, be, C, ldc, nthreads=2)
                            assert st == 0
                            assert R.shape == (M, N)
                            for i in range(M):
                                for j in range(N):
                                    ex = Fraction(0)
                                    t = Fraction(0)
                                    for p in range(K):
                                        pr = Fraction(float(opA[i, p])) * Fraction(float(opB[p, j]))
                                        ex += pr
                                        t += abs(pr)
                                    ex = Fraction(al) * ex
                                    tt = Fraction(0)
                                    if be != 0:
                                        bc = Fraction(be) * Fraction(float(Cl[i, j]))
                                        ex += bc
                                        tt = abs(bc)
                                    bound = (K + 3) * U53 * float(abs(Fraction(al)) * t + tt)
                                    assert abs(Fraction(R[i, j]) - ex) <= Fraction(bound), (M, N, K, i, j)
                                    assert abs(S[i, j] - float(abs(Fraction(al)) * t)) <= (K + 1) * U53 * S[i, j]
                                    assert T[i, j] == float(tt)


# --------------------------------------------------------------------------
# invariants
# --------------------------------------------------------------------------
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
def test_transpose_invariant_bitwise(tA, tB):
    """(op(A) op(B))^T = op(B)^T op(A)^T: swapping the operands and flipping
    both trans flags on the same storages must give the transposed result bit
    for bit (same exact products, same p order)."""
    flip = {"N": "T", "T": "N"}
    rng = np.random.default_rng(7)
    M, N, K = 37, 23, 53
    sa, sb = stored_shape(tA, M, K), stored_shape(tB, K, N)
    lda, ldb = sa[0] + 2, sb[0] + 1
    A = rand_flat(rng, *sa, lda, "uniform")
    B = rand_flat(rng, *sb, ldb, "uniform")
    R1, _, _, st1 = oracle.sgemm_sub(tA, tB, M, N, K, 1.0, A, lda, B, ldb, 0.0, None, M)
    R2, _, _, st2 = oracle.sgemm_sub(flip[tB], flip[tA], N, M, K, 1.0, B, ldb, A, lda, 0.0, None, N)
    assert st1 == 0 and st2 == 0
    assert np.array_equal(R1, R2.T)


def test_threads_and_subsets_bitwise():
    rng = np.random.default_rng(3)
    M, N, K = 45, 31, 77
    A = rand_flat(rng, M, K, M, "uniform")
    B = rand_flat(rng, K, N, K, "uniform")
    C = rand_flat(rng, M, N, M, "uniform")
    R1, S1, T1, _ = oracle.sgemm_sub("N", "N", M, N, K, 0.5, A, M, B, K, -1.5, C, M, nthreads=1)
    R8, S8, T8, _ = oracle.sgemm_sub("N", "N", M, N, K, 0.5, A, M, B, K, -1.5, C, M, nthreads=8)
    assert np.array_equal(R1, R8) and np.array_equal(S1, S8) and np.array_equal(T1, T8)
    rows, cols = [44, 0, 17], [30, 2]
    Rs, Ss, Ts, _ = oracle.sgemm_sub("N", "N", M, N, K, 0.5, A, M, B, K, -1.5, C, M, rows=rows, cols=cols)
    assert np.array_equal(Rs, R1[np.ix_(rows, cols)])
    assert np.array_equal(Ss, S1[np.ix_(rows, cols)])


# --------------------------------------------------------------------------
# closed forms and worked examples
# --------------------------------------------------------------------------
def _golden(name):
    rec = {}
    with open(os.path.join(HERE, "golden", name)) as f:
        lines = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    hdr = lines[0]
    rec["tA"], rec["tB"] = hdr[0], hdr[1]
    rec["M"], rec["N"], rec["K"] = map(int, hdr[2:5])
    rec["alpha"], rec["beta"] = float(hdr[5]), float(hdr[6])
    for ln in lines[1:]:
        rec[ln[0]] = np.array([float(v) for v in ln[1:]], dtype=np.float32)
    return rec


def test_golden_2x2():
    g = _golden("spec_2x2.txt")
    R, _, _, st = oracle.sgemm_sub(g["tA"], g["tB"], g["M"], g["N"], g["K"], g["alpha"], g["A"],
                                   2, g["B"], 2, g["beta"], None, 2)
    assert st == 0
    assert np.array_equal(R.reshape(-1, order="F"), g["C"].astype(np.float64))


def test_golden_five_dot_products():
    g = _golden("spec_dot5.txt")
    a = np.arange(1, 17, dtype=np.float32)                       # 1 x 16, lda = 1
    b = np.repeat(np.arange(5, dtype=np.float32), 16)            # 16 x 5, column c == c
    R, _, _, st = oracle.sgemm_sub("N", "N", 1, 5, 16, 1.0, a, 1, b, 16, 0.0, None, 1)
    assert st == 0
    assert np.array_equal(R.reshape(-1), g["C"].astype(np.float64))


@pytest.mark.parametrize("K", [1, 7, 64, 1000])
def test_all_ones_gives_K(K):
    M, N = 9, 11
    A = np.ones(M * K, np.float32)
    B = np.ones(K * N, np.float32)
    R, S, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, None, M)
    assert np.all(R == K) and np.all(S == K)


@pytest.mark.parametrize("transA", ["N", "T"])
@pytest.mark.parametrize("transB", ["N", "T"])
def test_identity_gives_opA(transA, transB):
    rng = np.random.default_rng(5)
    M, K = 13, 9
    sa = stored_shape(transA, M, K)
    A = rand_flat(rng, *sa, sa[0], "uniform")
    B = np.eye(K, dtype=np.float32).reshape(-1, order="F")     # symmetric: same for N and T
    R, _, _, _ = oracle.sgemm_sub(transA, transB, M, K, K, 1.0, A, sa[0], B, K, 0.0, None, M)
    assert np.array_equal(R, logical(A, transA, M, K, sa[0]).astype(np.float64))


def test_alpha_zero_never_reads_AB():
    rng = np.random.default_rng(9)
    M, N, K = 17, 5, 33
    A = np.full(M * K, np.nan, np.float32)
    B = np.full(K * N, np.nan, np.float32)
    C = rand_flat(rng, M, N, M, "uniform")
    for beta in (0.0, 1.0, 2.0, -0.3):
        R, S, T, _ = oracle.sgemm_sub("N", "N", M, N, K, 0.0, A, M, B, K, beta, C, M)
        expect = (np.float64(np.float32(beta)) * C.astype(np.float64)).reshape(N, M).T if beta != 0 else np.zeros((M, N))
        assert np.array_equal(R, expect)
        assert np.all(S == 0)
        # rounded to float, beta*c in FP32 RN is the same value
        if beta != 0:
            assert np.array_equal(R.astype(np.float32), (np.float32(beta) * C).reshape(N, M).T)


def test_beta_zero_never_reads_C():
    rng = np.random.default_rng(10)
    M, N, K = 12, 7, 19
    A = rand_flat(rng, M, K, M, "uniform")
    B = rand_flat(rng, K, N, K, "uniform")
    C = np.full(M * N, np.nan, np.float32)
    R, _, T, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.5, A, M, B, K, 0.0, C, M)
    assert np.all(np.isfinite(R)) and np.all(T == 0)
    ref = 1.5 * (logical(A, "N", M, K, M).astype(np.float64) @ logical(B, "N", K, N, K).astype(np.float64))
    assert np.allclose(R, ref, rtol=0, atol=1e-12)


def test_K_zero_and_K_one():
    rng = np.random.default_rng(11)
    M, N = 6, 4
    C = rand_flat(rng, M, N, M, "uniform")
    R, _, _, _ = oracle.sgemm_sub("N", "N", M, N, 0, 1.0, None, M, None, 1, 1.25, C, M)
    assert np.array_equal(R, (1.25 * C.astype(np.float64)).reshape(N, M).T)
    a = rand_flat(rng, M, 1, M, "uniform")
    b = rand_flat(rng, 1, N, 1, "uniform")
    R, _, _, _ = oracle.sgemm_sub("N", "N", M, N, 1, -0.75, a, M, b, 1, 0.0, None, M)
    # each entry is one exact double product times alpha (exact: alpha = -3/4)
    assert np.array_equal(R, -0.75 * np.outer(a.astype(np.float64), b.astype(np.float64)))


def test_empty_touches_nothing():
    R, S, T, st = oracle.sgemm_sub("N", "N", 0, 5, 3, 1.0, None, 1, None, 3, 0.0, None, 1)
    assert st == 0 and R.shape == (0, 5)
    C = np.full(4, 7.0, np.float32)
    assert oracle.sgemm("N", "N", 4, 0, 3, 1.0, None, 4, None, 3, 0.0, C, 4) == 0
    assert np.all(C == 7.0)


# --------------------------------------------------------------------------
# exactness bounds against library routines
# --------------------------------------------------------------------------
def test_fsum_correctly_rounded_within_sequential_bound():
    rng = np.random.default_rng(12)
    M = N = K = 64
    A = rand_flat(rng, M, K, M, "uniform")
    B = rand_flat(rng, K, N, K, "uniform")
    R, S, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, None, M)
    opA, opB = logical(A, "N", M, K, M), logical(B, "N", K, N, K)
    for i in range(0, M, 7):
        for j in range(0, N, 5):
            prods = [float(opA[i, p]) * float(opB[p, j]) for p in range(K)]
            exact = math.fsum(prods)
            assert abs(R[i, j] - exact) <= (K - 1) * U53 * S[i, j] + 1e-300


@pytest.mark.parametrize("transA", ["N", "T"])
@pytest.mark.parametrize("transB", ["N", "T"])
def test_numpy_float64_matmul(transA, transB):
    rng = np.random.default_rng(13)
    for (M, N, K) in [(1, 1, 1), (5, 48, 3), (48, 17, 31), (29, 29, 29), (64, 64, 64)]:
        sa, sb = stored_shape(transA, M, K), stored_shape(transB, K, N)
        lda, ldb, ldc = sa[0] + 3, sb[0] + 1, M + 2
        A = rand_flat(rng, *sa, lda, "uniform")
        B = rand_flat(rng, *sb, ldb, "uniform")
        C = rand_flat(rng, M, N, ldc, "uniform")
        R, S, T, _ = oracle.sgemm_sub(transA, transB, M, N, K, -0.75, A, lda, B, ldb, 1.25, C, ldc)
        ref = -0.75 * (logical(A, transA, M, K, lda).astype(np.float64)
                       @ logical(B, transB, K, N, ldb).astype(np.float64)) \
            + 1.25 * logical(C, "N", M, N, ldc).astype(np.float64)
        assert np.all(np.abs(R - ref) <= 1e-12 * (S + T) + 1e-300)


def test_c1_config_against_numpy():
    """BASELINE.json configs[0]: 64^3 NN, alpha=1, beta=0, U[-1,1] seed 0."""
    A = datagen.matrix("uniform", datagen.TAG_A, 64, 64)
    B = datagen.matrix("uniform", datagen.TAG_B, 64, 64)
    R, S, _, _ = oracle.sgemm_sub("N", "N", 64, 64, 64, 1.0, A, 64, B, 64, 0.0, None, 64)
    ref = A.double().numpy() @ B.double().numpy()
    assert np.all(np.abs(R - ref) <= 1e-12 * S)


def test_accumulate_twice_equals_2B_and_alpha_linearity():
    rng = np.random.default_rng(14)
    M, N, K = 33, 21, 40
    A = rand_flat(rng, M, K, M, "small")
    B = rand_flat(rng, K, N, K, "small")
    C = rand_flat(rng, M, N, M, "small")
    # small binary fractions -> every quantity exact: bitwise equalities hold
    R1, _, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A, M, B, K, 1.0, C, M)
    C1 = R1.T.reshape(-1).astype(np.float32)
    R2, _, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A, M, B, K, 1.0, C1, M)
    R3, _, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A, M, 2 * B, K, 1.0, C, M)
    assert np.array_equal(R2, R3)
    Ra, _, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 3.0, A, M, B, K, 0.0, None, M)
    Rb, _, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A, M, B, K, 0.0, None, M)
    assert np.array_equal(Ra, 3.0 * Rb)


# --------------------------------------------------------------------------
# argument errors (BLAS SGEMM numbering)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("args,code", [
    (("X", "N", 2, 2, 2, 2, 2, 2), -1),
    (("N", "q", 2, 2, 2, 2, 2, 2), -2),
    (("N", "N", -1, 2, 2, 2, 2, 2), -3),
    (("N", "N", 2, -1, 2, 2, 2, 2), -4),
    (("N", "N", 2, 2, -1, 2, 2, 2), -5),
    (("N", "N", 4, 2, 2, 3, 2, 4), -8),
    (("T", "N", 4, 2, 5, 4, 5, 4), -8),       # transA=T needs lda >= K
    (("N", "N", 4, 2, 5, 4, 4, 4), -10),
    (("N", "T", 4, 6, 5, 4, 5, 4), -10),      # transB=T needs ldb >= N
    (("N", "N", 4, 2, 2, 4, 2, 3), -13),
    (("c", "C", 0, 0, 0, 1, 1, 1), 0),
    (("T", "N", 1531, 997, 2049, 1531 + 13, 2049 + 7, 1531 + 5), -8),  # BJ configs[2] literal reading (R3)
])
def test_argument_errors(args, code):
    assert oracle.check_args(*args) == code


# --------------------------------------------------------------------------
# datagen pins (the shared generator must be what it claims)
# --------------------------------------------------------------------------
def test_datagen_splitmix_matches_python_and_grid():
    import torch
    keys = [0, 1, 2, 12345, (1 << 62) + 5, (1 << 63) + 17]
    t = torch.tensor([k - (1 << 64) if k >= (1 << 63) else k for k in keys], dtype=torch.int64)
    out = datagen.splitmix64(t)
    for k, o in zip(keys, out.tolist()):
        assert (o & ((1 << 64) - 1)) == datagen.splitmix64_py(k)
    U = datagen.matrix("uniform", datagen.TAG_A, 300, 7, 305)
    assert U.stride() == (1, 305)
    v = U.double()
    assert torch.all(v >= -1) and torch.all(v < 1)
    assert torch.all((v * 2 ** 23) == torch.round(v * 2 ** 23))
    # element (r, c) depends only on idx = c*rows + r
    idx = 5 * 300 + 11
    h = datagen.splitmix64_py((datagen.TAG_A << 56) ^ (idx << 1)) >> 40
    assert float(U[11, 5]) == h * 2.0 ** -23 - 1.0
    st = datagen.storage_of(U)
    assert torch.isnan(st[300:305]).all()
    I = datagen.matrix("ints", datagen.TAG_B, 1000, 10)
    assert I.min() == -8 and I.max() == 8
    Nn = datagen.matrix("normal", datagen.TAG_B, 4096, 16, sigma=0.5)
    assert abs(float(Nn.double().std()) - 0.5) < 0.01 and abs(float(Nn.double().mean())) < 0.01


# --------------------------------------------------------------------------
# the drop-in form oracle_sgemm (C <- (float)R through ldc)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
@pytest.mark.parametrize("beta", [0.0, 1.25])
def test_dropin_sgemm_exact_rounding_and_ldc_padding(tA, tB, beta):
    """oracle_sgemm on a ragged shape with ldc padding: every logical entry
    equals the float32 round-to-nearest of the exact result, computed here by
    numpy float64 matmul on integer-valued inputs (every product and partial
    sum is an integer < 2^53, so the float64 result is exact), while the
    magnitudes (|entries| up to 4096, K = 19) put the results above 2^24 so the
    float32 rounding is exercised.  ldc padding (a NaN-payload sentinel) is
    never written; with beta = 0 a NaN-filled C is never read."""
    rng = np.random.default_rng(31)
    M, N, K = 37, 23, 19
    alpha = -0.75
    ar, ac = stored_shape(tA, M, K)
    br, bc = stored_shape(tB, K, N)
    lda, ldb, ldc = ar + 3, br + 2, M + 5
    A = rng.integers(-4096, 4097, size=lda * ac).astype(np.float32)
    B = rng.integers(-4096, 4097, size=ldb * bc).astype(np.float32)
    sentinel = np.frombuffer(np.uint32(0x7FC0BEEF).tobytes(), dtype=np.float32)[0]
    C = np.full(ldc * N, sentinel, dtype=np.float32)
    cin = rng.integers(-(1 << 20), 1 << 20, size=(M, N)).astype(np.float32)
    if beta != 0.0:
        C.reshape(N, ldc)[:, :M] = cin.T
    C0 = C.copy()
    exact = alpha * (logical(A, tA, M, K, lda).astype(np.float64) @ logical(B, tB, K, N, ldb).astype(np.float64))
    if beta != 0.0:
        exact = exact + beta * cin.astype(np.float64)
    assert np.all(np.abs(exact) < 2.0 ** 52) and np.max(np.abs(exact)) > 2.0 ** 24
    assert oracle.sgemm(tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc) == 0
    got = C.reshape(N, ldc)[:, :M].T
    assert np.array_equal(got, exact.astype(np.float32))
    pad = C.reshape(N, ldc)[:, M:]
    assert np.array_equal(pad.view(np.uint32), C0.reshape(N, ldc)[:, M:].view(np.uint32))


def test_dropin_sgemm_argument_error_leaves_C():
    C = np.full(12, 3.0, np.float32)
    assert oracle.sgemm("N", "N", 4, 3, 2, 1.0, np.ones(8, np.float32), 3, np.ones(6, np.float32), 2,
                        0.0, C, 4) == -8
    assert np.all(C == 3.0)
