"""KN2w (k_tc1w.cu): 1xTF32 on 256 x 512 tiles, forced with EMM_WIDE=1 on
shapes the default policy would not send there too — ragged M / N / K
tails, N <= 256 (the second B half entirely out of bounds), several tiles per
CTA pair (TMEM reuse, the half-0-first hand-off to the next tile), every
trans combination, beta != 0, direct and re-buffered operands.  Integer-exact
inputs must match the oracle bitwise; random inputs the 1xTF32 bound."""
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
def force_wide(monkeypatch):
    monkeypatch.setenv("EMM_WIDE", "1")
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    monkeypatch.setenv("EMM_NO_SKINNY", "1")


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
@pytest.mark.parametrize("shape", [(300, 200, 97), (777, 1000, 129), (513, 1537, 2049), (256, 512, 32)],
                         ids=lambda s: "x".join(map(str, s)))
def test_wide_integer_exact(emm, trans, shape):
    M, N, K = shape
    case = Case(trans[0], trans[1], M, N, K, 2.0, -1.0, kind="ints", c_kind="ints", pad=(4, 8, 3))
    G = case.run(emm, "1xtf32")
    case.check_untouched(G)
    R, _, _, st = case.oracle()
    assert st == 0
    assert np.array_equal(case.logical(G), R.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("shape,pack", [((4096, 4096, 512), None), ((8192, 2560, 300), None),
                                        ((4096, 4096, 512), "1"), ((3000, 5000, 1000), None)])
def test_wide_multi_tile(emm, monkeypatch, shape, pack):
    """>= 2 tiles per CTA pair; sampled rows (all columns) vs the oracle."""
    if pack:
        monkeypatch.setenv("EMM_FORCE_PACK", pack)
    M, N, K = shape
    case = Case("N", "N", M, N, K, 1.0, 0.5, kind="normal", sigma=1.0 / np.sqrt(K))
    G = case.run(emm, "1xtf32")
    case.check_untouched(G)
    rows = np.unique(np.r_[0:3, 255:258, M // 2 - 1:M // 2 + 2, M - 3:M])
    R, S, T, st = case.oracle(rows=rows)
    assert st == 0
    assert_close(case, G, R, S, T, TOL["1xtf32"], rows=rows)


def test_wide_matches_narrow_on_integers(emm, monkeypatch):
    """Integer-exact data: the 256x512 and 256x256 tilings give the same bits."""
    case = Case("N", "T", 2048, 3072, 2048, 1.0, 1.0, kind="ints", c_kind="ints")
    G1 = case.run(emm, "1xtf32")
    monkeypatch.setenv("EMM_WIDE", "0")
    G0 = case.run(emm, "1xtf32")
    assert torch.equal(G1.view(torch.int32), G0.view(torch.int32))


def test_wide_deterministic(emm):
    case = Case("N", "N", 4096, 2048, 2048, 1.0, 0.0, kind="normal")
    a = case.run(emm, "1xtf32")
    b = case.run(emm, "1xtf32")
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
