"""GPU parity of KN11, the 3xTF32 GEMM with the operand split inside the
kernel (EMM_SPLIT=kernel), through the C ABI.

Same bars as test_gpu_parity.py: bitwise on integer-exact inputs, the
1e-5*S + 1e-6*T predicate on random data, untouched ldc padding / guard,
A and B never written.  Extra property: KN11 builds exactly the planes the
re-buffering pass builds (big = rn_tf32(x), small = rn_tf32(x - big)) and
runs the same MMA sequence, so its result must equal the EMM_SPLIT=pass +
EMM_FORCE_PACK=1 path BIT FOR BIT on random data.
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
def inkernel(monkeypatch):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    monkeypatch.setenv("EMM_SPLIT", "kernel")


def _exact(case, Cg, R):
    case.check_untouched(Cg)
    G = case.logical(Cg)
    assert np.array_equal(G, R.astype(np.float32).astype(np.float64)), f"max |diff| {np.max(np.abs(G - R))}"


# pads: (0,0,0) keeps 16-B vector loads legal when the stored rows are
# multiples of 4; (3,1,2) forces the element-wise loader
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("pad", [(0, 0, 0), (3, 1, 2), (4, 8, 3)])
@pytest.mark.parametrize("shape", [(1, 1, 1), (64, 64, 64), (300, 260, 100), (513, 257, 129), (129, 700, 33),
                                   (256, 256, 4000)])
def test_integer_exact_bitwise(emm, tA, tB, pad, shape):
    M, N, K = shape
    for alpha, beta in ((1.0, 0.0), (-1.0, 2.0)):
        case = Case(tA, tB, M, N, K, alpha, beta, kind="ints", c_kind="ints", pad=pad)
        R, S, T, _ = case.oracle()
        _exact(case, case.run(emm, "3xtf32"), R)


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
def test_multiwave_lockstep(emm, tA, tB):
    """100 tiles > 74 CTA pairs: a second wave, so the wave lockstep and its
    zeroed counter are live; integer-exact -> bitwise."""
    case = Case(tA, tB, 2560, 2560, 96, 1.0, 1.0, kind="ints", c_kind="ints", pad=(0, 4, 1))
    rows = np.r_[0:40, 1270:1290, 2520:2560]
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    G = case.logical(Cg)[rows]
    assert np.array_equal(G, R.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape,pad", [((520, 388, 200), (4, 0, 1)), ((1000, 1000, 1000), (0, 0, 0)),
                                       ((1531, 997, 2049), (13, 7, 5)), ((333, 333, 333), (0, 0, 0)),
                                       ((2560, 2560, 300), (0, 0, 0))])
def test_bitwise_equal_to_split_pass(emm, monkeypatch, tA, tB, shape, pad):
    M, N, K = shape
    case = cached_case(tA, tB, M, N, K, -0.75, 1.25, pad=pad, kind="normal")
    Ck = case.run(emm, "3xtf32")
    monkeypatch.setenv("EMM_SPLIT", "pass")
    monkeypatch.setenv("EMM_FORCE_PACK", "1")
    Cp = case.run(emm, "3xtf32")
    assert torch.equal(Ck.view(torch.int32), Cp.view(torch.int32)), \
        f"max |diff| {float((Ck - Cp).abs().max())}"


@pytest.mark.parametrize("n", [100, 333, 512, 700, 1000, 1024, 2048])
def test_c2_square_sweep(emm, n):
    case = cached_case("N", "N", n, n, n, 1.0, 0.0)
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, 1e-5)


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
def test_c3_blas_stress(emm, tA, tB):
    case = cached_case(tA, tB, 1531, 997, 2049, -0.75, 1.25, kind="normal", pad=(13, 7, 5))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, 1e-5)


@pytest.mark.parametrize("shape", [(65536, 1024, 4096), (65536, 4096, 1024)])
def test_c4_nn_layer_sampled(emm, shape):
    M, N, K = shape
    case = cached_case("N", "T", M, N, K, 1.0, 1.0, kind="normal", sigma=1.0 / np.sqrt(K), c_kind="normal")
    rows = np.r_[0:8, M // 2:M // 2 + 8, M - 8:M]
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, "3xtf32")
    assert_close(case, Cg, R, S, T, 1e-5, rows=rows)


@pytest.mark.parametrize("K", [1, 7, 31, 33, 337, 2049])
def test_k_tails(emm, K):
    case = cached_case("T", "N", 300, 260, K, 1.0, 0.5, pad=(1, 0, 2))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, 1e-5)


@pytest.mark.parametrize("mn", [(17, 17), (17, 300), (300, 17), (127, 129), (255, 257), (256, 256)])
def test_mn_edges(emm, mn):
    M, N = mn
    case = cached_case("N", "T", M, N, 200, 1.5, 0.0, pad=(2, 0, 1))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, 1e-5)


@pytest.mark.parametrize("K", [4096, 32768])
def test_same_sign_accumulation(emm, K):
    """U[0,1) data: the promotion every 256 of K must hold the bound."""
    case = cached_case("N", "N", 256, 256, K, 1.0, 0.0, kind="uniform01")
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    assert assert_close(case, Cg, R, S, T, 1e-5) <= 1.0


def test_deterministic(emm):
    case = cached_case("N", "N", 1000, 1000, 1000, 1.0, 0.0)
    a = case.run(emm, "3xtf32")
    b = case.run(emm, "3xtf32")
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_no_workspace_entry(emm):
    """emm_sgemm (no workspace) through the in-kernel path: single-wave
    problems need no scratch at all; split-K / multi-wave ones take it from
    the stream-ordered pool."""
    for (M, N, K) in [(512, 512, 64), (1024, 1024, 1024), (2560, 2560, 64)]:
        case = Case("N", "N", M, N, K, 1.0, 0.0, kind="ints")
        R, S, T, _ = case.oracle()
        dA = case.flat(case.A).cuda()
        dB = case.flat(case.B).cuda()
        dC = case.Cflat.cuda()
        st = emm.lib().emm_sgemm(b"N", b"N", M, N, K, 1.0, dA.data_ptr(), case.lda, dB.data_ptr(), case.ldb, 0.0,
                                 dC.data_ptr(), case.ldc, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert st == 0
        _exact(case, dC.cpu(), R)
