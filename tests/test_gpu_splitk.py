"""GPU parity of the split-K reduce KN8 for every split factor it is
instantiated for (S = 1..16; one kernel instantiation per
S, every partial load of a thread in flight at once).

A 2x2-tile problem with ragged M / N tails and K = 4100 (129 K-stages) is run
with EMM_SPLITS forced to each S through KN1X (default) and the split pass +
KN1.  Bars: bitwise against the oracle on integer-exact inputs (every partial
and their sum are exact), the 1e-5*S + 1e-6*T predicate on random data with
beta != 0 (C_in read by the reduce), bitwise equality of the two kernels at
the same S (same products, same fixed-order sum), ldc padding / guard
untouched.
"""
from __future__ import annotations

import numpy as np
import pytest

from test_gpu_parity import TOL, assert_close, cached_case  # noqa: F401

pytestmark = pytest.mark.gpu

M, N, K = 300, 270, 4100


@pytest.fixture(scope="module")
def emm():
    import torch

    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


@pytest.fixture(autouse=True)
def no_small_path(monkeypatch):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    monkeypatch.setenv("EMM_SK", "0")


@pytest.mark.parametrize("S", list(range(1, 17)))
def test_splits_integer_exact(emm, monkeypatch, S):
    monkeypatch.setenv("EMM_SPLITS", str(S))
    case = cached_case("N", "T", M, N, K, -1.0, 2.0, kind="ints", c_kind="ints", pad=(3, 5, 7))
    R, _, _, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    G = case.logical(Cg)
    assert np.array_equal(G, R.astype(np.float32).astype(np.float64)), f"S={S}: max |diff| {np.max(np.abs(G - R))}"


@pytest.mark.parametrize("S", [2, 3, 4, 5, 8, 11, 16])
@pytest.mark.parametrize("math", ["3xtf32", "1xtf32"])
def test_splits_random(emm, monkeypatch, S, math):
    monkeypatch.setenv("EMM_SPLITS", str(S))
    case = cached_case("N", "N", M, N, K, 0.75, -1.25, kind="normal", pad=(4, 0, 9))
    R, Sg, T, _ = case.oracle()
    monkeypatch.setenv("EMM_SPLIT", "xform")
    Cx = case.run(emm, math)
    case.check_untouched(Cx)
    assert_close(case, Cx, R, Sg, T, TOL[math])
    if math == "3xtf32":
        monkeypatch.setenv("EMM_SPLIT", "pass")
        Cp = case.run(emm, math)
        assert np.array_equal(case.logical(Cx), case.logical(Cp)), f"S={S}: KN1X != split pass + KN1"
