"""FFMA path (EMM_MATH_FFMA): the TMA-fed warp-specialised kernel KN3b
(k_ffma_tma.cu) against the oracle and against KN3 (k_ffma.cu).

KN3b and KN3 perform the same FP32 operations in the same order — per output
entry a sequential FFMA chain over k (round-to-nearest), restarted every 256
of K and added into a master copy, then alpha*master (+ beta*C by one fmaf)
— so on ANY inputs their results must be bitwise identical (KN3 is forced
with EMM_FFMA_CLASSIC=1).  Layouts KN3b does not take (TN; leading
dimensions or bases that are not 16-byte aligned) must still run on KN3.
The same-sign promotion diagnostic (K = 32768, TMA-legal, so KN3b) is
test_gpu_parity.py::test_same_sign_accumulation.
Shapes cover several 128 x 128 tiles with ragged M / N / K tails.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from test_gpu_parity import TOL, Case, assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


@pytest.fixture(autouse=True)
def no_small_path(monkeypatch):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    monkeypatch.setenv("EMM_NO_SKINNY", "1")


SHAPES = [(300, 200, 97), (129, 257, 33), (1000, 600, 700), (640, 384, 1), (257, 129, 2049)]


@pytest.mark.parametrize("trans", ["NN", "NT", "TT", "TN"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("pad", [(0, 0, 0), (4, 8, 3), (1, 3, 0)], ids=["ld=rows", "ld+4k", "ld+odd"])
def test_kn3b_matches_kn3_bitwise_and_oracle(emm, monkeypatch, trans, shape, pad):
    M, N, K = shape
    # ld = rows is TMA-legal only when rows % 4 == 0; the odd pads force KN3
    case = Case(trans[0], trans[1], M, N, K, -0.75, 1.25, kind="normal", pad=pad, sigma=1.0 / np.sqrt(K))
    monkeypatch.setenv("EMM_FFMA_CLASSIC", "0")
    G = case.run(emm, "ffma")
    monkeypatch.setenv("EMM_FFMA_CLASSIC", "1")
    G3 = case.run(emm, "ffma")
    assert torch.equal(G.view(torch.int32), G3.view(torch.int32)), "KN3b and KN3 differ"
    case.check_untouched(G)
    R, S, T, st = case.oracle()
    assert st == 0
    assert_close(case, G, R, S, T, TOL["ffma"])


@pytest.mark.parametrize("trans", ["NN", "NT", "TT"])
def test_kn3b_integer_exact(emm, trans):
    M, N, K = 515, 391, 1029
    case = Case(trans[0], trans[1], M, N, K, 2.0, -1.0, kind="ints", c_kind="ints", pad=(4, 4, 1))
    G = case.run(emm, "ffma")
    R, _, _, st = case.oracle()
    assert st == 0
    assert np.array_equal(case.logical(G), R.astype(np.float32).astype(np.float64))


def test_kn3b_beta_zero_ignores_nan_c(emm):
    M, N, K = 384, 256, 96
    case = Case("N", "T", M, N, K, 1.0, 0.0)
    case.Cflat[: case.ldc * N] = float("nan")
    G = case.run(emm, "ffma")
    assert np.isfinite(case.logical(G)).all()
    R, S, T, st = case.oracle()
    assert_close(case, G, R, S, T, TOL["ffma"])


def test_kn3b_deterministic(emm):
    case = Case("N", "N", 1024, 768, 1500, 1.0, 0.5, kind="normal")
    a = case.run(emm, "ffma")
    b = case.run(emm, "ffma")
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
