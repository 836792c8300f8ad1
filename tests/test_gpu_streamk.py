"""GPU parity of the stream-K schedule through the C ABI.

Shapes whose tile count is above half a wave and not a multiple of the 74
CTA pairs run their last (partial) wave as stream-K: every cluster takes an
equal contiguous range of 256-K chunks, tiles split across clusters are
summed by the cluster holding the tile's first chunk (own partial + the
published ones in ascending k).  Bars: bitwise on integer-exact inputs (the
piece sums are exact), the 1e-5*S + 1e-6*T predicate on random data,
run-to-run bitwise determinism, ldc padding / guard untouched.  EMM_SK=0
runs the same shapes without stream-K for comparison; EMM_SK=1 (default in
this file) forces it where the production policy would not pick it.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from test_gpu_parity import TOL, Case, assert_close, cached_case  # noqa: F401

pytestmark = pytest.mark.gpu

# (M, N, K): tiles of 256 x 256 per CTA pair
SHAPES = [
    (1536, 1792, 2049),   # 42 tiles < 74 pairs: all stream-K, up to 3 pieces per tile, ragged last chunk
    (2560, 2560, 600),    # 100 tiles: 1 partial wave + stream-K
    (4096, 4096, 520),    # 256 tiles: 2 data-parallel waves + stream-K over 108 tiles
    (2048, 2048, 2048),   # c2-2048: 64 tiles
]


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


@pytest.fixture(autouse=True, params=["xform", "pass"])
def no_small_path(monkeypatch, request):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    monkeypatch.setenv("EMM_SPLIT", request.param)   # KN1X (default) and KN1
    # force stream-K wherever it is legal (the default policy enables it only
    # where it measured faster, e.g. 4096^3 3xTF32 and (2560, 2560, 600))
    monkeypatch.setenv("EMM_SK", "1")


def sample_rows(M):
    return np.unique(np.r_[0:24, M // 3:M // 3 + 24, M - 24:M, np.arange(0, M, 97)])


@pytest.mark.parametrize("math", ["3xtf32", "1xtf32", "tf32bf16"])
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("shape", SHAPES[:3])
def test_integer_exact_bitwise(emm, math, tA, tB, shape):
    M, N, K = shape
    case = cached_case(tA, tB, M, N, K, -1.0, 2.0, kind="ints", c_kind="ints", pad=(4, 0, 3))
    rows = sample_rows(M)
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    G = case.logical(Cg)[rows]
    assert np.array_equal(G, R.astype(np.float32).astype(np.float64)), f"max |diff| {np.max(np.abs(G - R))}"


@pytest.mark.parametrize("sk", ["1", "0"])
@pytest.mark.parametrize("math", ["3xtf32", "1xtf32", "tf32bf16"])
@pytest.mark.parametrize("shape", SHAPES)
def test_random_tolerance(emm, monkeypatch, sk, math, shape):
    monkeypatch.setenv("EMM_SK", sk)
    M, N, K = shape
    case = cached_case("N", "N", M, N, K, 0.75, -0.5, kind="normal", pad=(0, 0, 1))
    rows = sample_rows(M)
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, TOL[math], rows=rows)


@pytest.mark.parametrize("shape", SHAPES[:2])
def test_deterministic(emm, shape):
    M, N, K = shape
    case = cached_case("N", "N", M, N, K, 0.75, -0.5, kind="normal", pad=(0, 0, 1))
    a = case.run(emm, "3xtf32")
    b = case.run(emm, "3xtf32")
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_no_workspace_entry(emm):
    """emm_sgemm allocates the stream-K scratch from the stream-ordered pool."""
    M, N, K = 2560, 2560, 600
    case = Case("N", "N", M, N, K, 1.0, 0.0, kind="ints")
    rows = sample_rows(M)
    R, S, T, _ = case.oracle(rows=rows)
    dA = case.flat(case.A).cuda()
    dB = case.flat(case.B).cuda()
    dC = case.Cflat.cuda()
    st = emm.lib().emm_sgemm(b"N", b"N", M, N, K, 1.0, dA.data_ptr(), case.lda, dB.data_ptr(), case.ldb, 0.0,
                             dC.data_ptr(), case.ldc, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0
    G = case.logical(dC.cpu())[rows]
    assert np.array_equal(G, R.astype(np.float32).astype(np.float64))
