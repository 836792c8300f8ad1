"""GPU parity of KN9T, the tensor-core skinny path (k_skinny_tc.cu;
SURVEY.md §8(f)-4): min(M, N) <= 16, the long operand streamed through TMA,
split in the kernel and fed to tcgen05.mma from tensor memory.

Bars: bitwise on integer-exact inputs (all trans, both operand roles, short
sides 1..16, ragged long sides and K tails, beta != 0); the 1e-5*S + 1e-6*T
predicate on random data; ldc padding and the guard untouched; and, as the
split and per-element MMA order are the re-buffered KN1's, bitwise equality
with EMM_NO_SKINNY=1 + EMM_FORCE_PACK=1 (KN1 on PK_FULL3 planes, data-
parallel) on random data.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from test_gpu_parity import Case, assert_close, cached_case  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


@pytest.fixture(autouse=True)
def force_tc(monkeypatch):
    monkeypatch.setenv("EMM_SKINNY_TC", "1")


def aligned_pad(t, rows_op, k):
    """pad making the stored rows a multiple of 4 (TMA-legal long operand)"""
    stored = rows_op if t == "N" else k
    return (-stored) % 4 + 4


@pytest.mark.parametrize("math", ["3xtf32", "tf32bf16", "1xtf32"])
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(1000, 16, 300), (777, 5, 129), (129, 1, 33), (4096, 8, 2049),
                                   (16, 1000, 300), (3, 2500, 97), (1, 333, 513)])
def test_integer_exact_bitwise(emm, math, tA, tB, shape):
    M, N, K = shape
    padA = aligned_pad(tA, M, K) if N <= 16 else 0
    padB = aligned_pad("T" if tB == "N" else "N", N, K) if N > 16 else 0
    for alpha, beta in ((1.0, 0.0), (-1.0, 2.0)):
        case = Case(tA, tB, M, N, K, alpha, beta, kind="ints", c_kind="ints", pad=(padA, padB, 3))
        R, S, T, _ = case.oracle()
        Cg = case.run(emm, math)
        case.check_untouched(Cg)
        assert np.array_equal(case.logical(Cg), R.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("math", ["3xtf32", "tf32bf16"])
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(20000, 16, 1024), (20000, 7, 700)])
def test_bitwise_equal_to_repacked_kn1(emm, monkeypatch, math, tA, tB, shape):
    """same split planes and per-element MMA order as KN1 on re-buffered planes"""
    M, N, K = shape
    case = cached_case(tA, tB, M, N, K, 0.75, 0.5, kind="normal", pad=(aligned_pad(tA, M, K), 0, 1),
                       sigma=1.0 / np.sqrt(K))
    Ct = case.run(emm, math)
    monkeypatch.setenv("EMM_NO_SKINNY", "1")
    monkeypatch.setenv("EMM_FORCE_PACK", "1")
    monkeypatch.setenv("EMM_SPLIT", "pass")
    monkeypatch.setenv("EMM_SK", "0")
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    Ck = case.run(emm, math)
    case.check_untouched(Ct)
    assert torch.equal(Ct.view(torch.int32), Ck.view(torch.int32)), f"max |diff| {float((Ct - Ck).abs().max())}"


@pytest.mark.parametrize("math", ["3xtf32", "1xtf32", "tf32bf16"])
@pytest.mark.parametrize("shape,trans", [((65536, 16, 4096), "NN"), ((8, 65536, 4096), "NN"),
                                         ((65536, 16, 1024), "TN"), ((12, 40000, 1000), "NT")])
def test_c6_skinny_sampled(emm, math, shape, trans):
    M, N, K = shape
    case = cached_case(trans[0], trans[1], M, N, K, 1.0, 0.0, kind="uniform")
    if M > 16:
        rows = np.unique(np.r_[0:64, M // 2:M // 2 + 64, M - 64:M])
        R, S, T, _ = case.oracle(rows=rows)
        cols = None
    else:
        rows = None
        cols = np.unique(np.r_[0:64, N // 2:N // 2 + 64, N - 64:N])
        R, S, T, _ = case.oracle(cols=cols)
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    G = case.logical(Cg)
    G = G[rows] if rows is not None else G[:, cols]
    err = np.abs(G - R)
    bound = (5e-3 if math == "1xtf32" else 1e-5) * S + 1e-6 * T
    assert np.all(err <= bound), f"max err/tol {float(np.max(err / np.maximum(bound, 1e-300)))}"


@pytest.mark.parametrize("K", [1, 7, 31, 33, 337, 2049])
def test_k_tails(emm, K):
    case = cached_case("N", "N", 1000, 13, K, 1.0, 0.5, pad=(0, 0, 2))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, 1e-5)


def test_same_sign_accumulation(emm):
    case = cached_case("N", "N", 4096, 16, 32768, 1.0, 0.0, kind="uniform01")
    rows = np.r_[0:32, 4000:4096]
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, "3xtf32")
    assert assert_close(case, Cg, R, S, T, 1e-5, rows=rows) <= 1.0


@pytest.mark.parametrize("math,tc", [("1xtf32", True), ("tf32bf16", False), ("3xtf32", False), ("ffma", False)])
def test_default_policy(emm, monkeypatch, math, tc):
    """Without the override: large skinny problems take the tensor cores
    (split pass + one GEMM launch) only in 1xTF32 with a K-contiguous long
    operand (TN: 218 vs 244 us); everything else (and NN 1xTF32, where KN9 is
    as fast) keeps the one-launch FFMA kernel KN9 (profiles/r02_skinny_ffma.md)."""
    monkeypatch.delenv("EMM_SKINNY_TC")
    small = Case("N", "N", 1000, 16, 300, 1.0, 0.0, kind="ints")
    n0 = emm.launch_count()
    small.run(emm, math)
    assert emm.launch_count() - n0 == 1
    big = cached_case("N", "N", 65536, 16, 4096, 1.0, 0.0, kind="uniform")
    n0 = emm.launch_count()
    big.run(emm, math)
    # KN9 after the B' transpose (MN-contiguous long operand of >= 2^26 elements, N' > 8)
    assert emm.launch_count() - n0 == 2
    # TN: two launches either way (KN9T: split pass + GEMM; KN9: B' transpose +
    # kernel); which kernel ran shows in the bits: KN9 equals the forced-FFMA
    # (EMM_SKINNY_TC=0) result, KN9T (TF32 products) does not
    big_t = cached_case("T", "N", 65536, 16, 1024, 1.0, 0.0, kind="uniform")
    n0 = emm.launch_count()
    Cd = big_t.run(emm, math)
    assert emm.launch_count() - n0 == 2
    monkeypatch.setenv("EMM_SKINNY_TC", "0")
    Cf = big_t.run(emm, math)
    assert torch.equal(Cd.view(torch.int32), Cf.view(torch.int32)) != tc
