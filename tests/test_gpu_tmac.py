"""beta != 0 epilogues that read C_in through TMA (KN1 3xTF32 / TF32+BF16,
`EMM_TMAC`): the same fmaf(beta, c, alpha * acc) per entry as the per-thread
load path, so the results must be bitwise identical (EMM_TMAC=1 vs 0) on any
inputs — with stream-K owners, preferred clusters of 4, partial waves and
ragged M / N; plus oracle parity on sampled rows."""
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


@pytest.mark.parametrize("math", ["3xtf32", "tf32bf16"])
@pytest.mark.parametrize("shape,trans,env", [
    ((8192, 2048, 1024), "NT", {}),                       # data-parallel, several waves
    ((4096, 4096, 1024), "NN", {"EMM_SK": "1"}),          # stream-K owners add published partials first
    ((3000, 2000, 700), "TT", {}),                        # split-K (reduce launch) + ragged edges
    ((8192, 4096, 4096), "NN", {"EMM_PREF4": "1"}),       # preferred clusters of 4 (dummies in the last wave)
    ((2820, 4100, 2049), "TN", {}),                       # ragged M / N (TMA clips the C boxes)
], ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple) else (v if isinstance(v, str) else "-".join(v) or "default"))
@pytest.mark.parametrize("split", ["xform", "pass"])
def test_tmac_bitwise(emm, monkeypatch, math, shape, trans, env, split):
    """KN1 (EMM_SPLIT=pass) and KN1X (the default 3xTF32 kernel on TMA-legal
    operands) read C_in through TMA or per thread: same bits."""
    if split == "xform" and (math != "3xtf32" or env.get("EMM_PREF4")):
        pytest.skip("KN1X is the 3xTF32 kernel, launched on clusters of 2")
    monkeypatch.setenv("EMM_SPLIT", split)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    M, N, K = shape
    case = Case(trans[0], trans[1], M, N, K, -0.75, 1.25, kind="normal", sigma=1.0 / np.sqrt(K))
    monkeypatch.setenv("EMM_TMAC", "1")
    G1 = case.run(emm, math)
    monkeypatch.setenv("EMM_TMAC", "0")
    G0 = case.run(emm, math)
    assert torch.equal(G1.view(torch.int32), G0.view(torch.int32)), "TMA-fed C_in epilogue differs"
    case.check_untouched(G1)
    rows = np.unique(np.r_[0:3, 127:130, M // 2:M // 2 + 2, M - 3:M])
    R, S, T, st = case.oracle(rows=rows)
    assert st == 0
    assert_close(case, G1, R, S, T, TOL[math], rows=rows)


def test_tmac_with_k_phases(emm, monkeypatch):
    """Host-buffer entry in two K phases, the second phase continuing the
    promotion chains (acc_init) with a TMA-fed C_in epilogue (aligned ldc):
    bitwise equal to the device call."""
    monkeypatch.setenv("EMM_HOST_KSPLIT", "1")
    monkeypatch.setenv("EMM_SK", "0")
    M, N, K = 4608, 4224, 1300
    case = Case("N", "T", M, N, K, 1.25, 0.5, kind="normal", sigma=1.0 / np.sqrt(K))
    assert (case.ldc * 4) % 16 == 0
    Cf = case.Cflat.clone().pin_memory()
    Af, Bf = case.flat(case.A).pin_memory(), case.flat(case.B).pin_memory()
    emm.sgemm_host("N", "T", M, N, K, 1.25, Af, case.lda, Bf, case.ldb, 0.5, Cf, case.ldc)
    case.check_untouched(Cf)
    Cd = case.run(emm, "3xtf32")   # KN1X on both sides (TMA-fed C_in in the last phase)
    assert torch.equal(Cd.view(torch.int32), Cf.view(torch.int32))
    rows = np.array([0, 1, 2047, 2048, M - 1])
    R, S, T, st = case.oracle(rows=rows)
    assert_close(case, Cf, R, S, T, TOL["3xtf32"], rows=rows)
