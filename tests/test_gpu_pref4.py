"""KN1 launched with a PREFERRED cluster size of 4 (EMM_PREF4=1): the B200
forms clusters of two CTA pairs where its GPCs allow (B multicast between
the pairs, which run vertically adjacent tiles of the same wave) and plain
pairs elsewhere; a pair whose partner has one more item mirrors it as a
dummy.  Per tile the operations and their order are KN1's, so on ANY inputs
the result must equal the plain launch bit for bit; integer-exact inputs
must also equal the oracle.  Shapes cover partial last waves (dummies),
odd tile rows, ragged M / N / K, every trans combination, beta != 0, direct
and re-buffered operands."""
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
def no_small_paths(monkeypatch):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    monkeypatch.setenv("EMM_NO_SKINNY", "1")
    monkeypatch.setenv("EMM_SK", "0")
    monkeypatch.setenv("EMM_SPLIT", "pass")   # KN1 (preferred clusters of 4 are a KN1 launch mode)


SHAPES = [((4096, 4096, 1024), "NN"), ((3000, 2000, 700), "TT"), ((8192, 2048, 512), "NT"),
          ((1000, 5000, 300), "TN"), ((2816, 3072, 2049), "NN"), ((5000, 1000, 64), "NT"),
          ((2304, 2304, 256), "TN")]


@pytest.mark.parametrize("math", ["3xtf32", "tf32bf16"])
@pytest.mark.parametrize("shape,trans", SHAPES, ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple) else v)
@pytest.mark.parametrize("pack", [None, "1"], ids=["direct", "packed"])
def test_pref4_bitwise_equals_kn1(emm, monkeypatch, math, shape, trans, pack):
    if pack:
        monkeypatch.setenv("EMM_FORCE_PACK", pack)
    M, N, K = shape
    case = Case(trans[0], trans[1], M, N, K, 1.0, 0.5, kind="normal", pad=(4, 4, 1), sigma=1.0 / np.sqrt(K))
    monkeypatch.setenv("EMM_PREF4", "1")
    G4 = case.run(emm, math)
    monkeypatch.setenv("EMM_PREF4", "0")
    G2 = case.run(emm, math)
    assert torch.equal(G4.view(torch.int32), G2.view(torch.int32)), "preferred-4 launch differs from the plain launch"
    case.check_untouched(G4)
    rows = np.unique(np.r_[0:3, 255:258, 511:514, M // 2:M // 2 + 2, M - 3:M])
    rows = rows[(rows >= 0) & (rows < M)]
    R, S, T, st = case.oracle(rows=rows)
    assert st == 0
    assert_close(case, G4, R, S, T, TOL[math], rows=rows)


@pytest.mark.parametrize("trans", ["NN", "NT", "TN", "TT"])
def test_pref4_integer_exact(emm, monkeypatch, trans):
    monkeypatch.setenv("EMM_PREF4", "1")
    M, N, K = 1537, 1029, 515
    case = Case(trans[0], trans[1], M, N, K, 2.0, -1.0, kind="ints", c_kind="ints", pad=(4, 8, 3))
    G = case.run(emm, "3xtf32")
    case.check_untouched(G)
    R, _, _, st = case.oracle()
    assert st == 0
    assert np.array_equal(case.logical(G), R.astype(np.float32).astype(np.float64))


def test_pref4_deterministic(emm, monkeypatch):
    monkeypatch.setenv("EMM_PREF4", "1")
    case = Case("N", "N", 8192, 4096, 1024, 1.0, 0.0, kind="normal")
    a = case.run(emm, "3xtf32")
    b = case.run(emm, "3xtf32")
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
