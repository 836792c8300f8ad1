"""FFMA path (EMM_MATH_FFMA): the TMA-fed warp-specialised kernel KN3b
(k_ffma_tma.cu) against the oracle and against KN3 (k_ffma.cu).

KN3b and KN3 perform the same FP32 operations in the same order — per output
entry a sequential FFMA chain over k (round-to-nearest), restarted every 256
of K and added into a master copy, then alpha*master (+ beta*C by one fmaf)
— so on ANY inputs their results must be bitwise identical (KN3 is forced
with EMM_FFMA_CLASSIC=1).  Layouts KN3b does not take in place (TN; leading
dimensions or bases that are not 16-byte aligned) run KN3b on a relayout copy
(the smaller TN operand transposed, an illegal one re-pitched: one copy pass)
— bitwise equal to KN3 in place (EMM_FFMA_NORELAYOUT=1).
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
    # bitwise comparisons with KN3 need KN3b unsplit (split-K regroups the
    # promotion-chunk sums; test_splitk_* cover it)
    monkeypatch.setenv("EMM_FFMA_SPLITS", "1")


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


@pytest.mark.parametrize("trans,pad,shape", [("TN", (0, 0, 0), (1000, 600, 700)), ("TN", (0, 0, 0), (600, 1000, 700)),
                                             ("TN", (13, 7, 5), (1531, 997, 2049)), ("TT", (13, 7, 5), (1531, 997, 2049)),
                                             ("NN", (1, 3, 0), (1000, 600, 700)), ("NT", (0, 1, 0), (257, 129, 2049)),
                                             ("TN", (1, 3, 0), (129, 257, 33)),
                                             # >= 1280 on both sides: K-contiguous operands transposed to NT
                                             ("NN", (0, 0, 0), (1300, 1400, 300)), ("TT", (0, 0, 0), (1300, 1400, 300)),
                                             ("TN", (4, 0, 2), (1300, 1400, 300)), ("NT", (0, 0, 0), (1300, 1400, 300))])
def test_relayout_bitwise_equal_to_kn3_in_place(emm, monkeypatch, trans, pad, shape):
    """TN / TMA-illegal FFMA calls: copy pass (PK_RAWT transpose of the
    smaller TN operand, PK_RAW re-pitch of an illegal one) + KN3b, two or three
    launches; the same FP32 operations as KN3 on the caller's arrays."""
    M, N, K = shape
    case = Case(trans[0], trans[1], M, N, K, -0.75, 1.25, kind="normal", pad=pad, sigma=1.0 / np.sqrt(K))
    n0 = emm.launch_count()
    G = case.run(emm, "ffma")
    n_relayout = emm.launch_count() - n0
    monkeypatch.setenv("EMM_FFMA_NORELAYOUT", "1")
    n0 = emm.launch_count()
    G3 = case.run(emm, "ffma")
    assert emm.launch_count() - n0 == 1
    assert (1 if (trans == "NT" and pad == (0, 0, 0)) else 2) <= n_relayout <= 5, n_relayout
    assert torch.equal(G.view(torch.int32), G3.view(torch.int32)), "relayout + KN3b and KN3 differ"
    case.check_untouched(G)
    R, S, T, st = case.oracle()
    assert st == 0
    assert_close(case, G, R, S, T, TOL["ffma"])


def test_relayout_caller_workspace(emm):
    """The relayout copies go to the caller's workspace when one is given
    (sized by emm_sgemm_workspace_bytes); too small -> EMM_ERR_WORKSPACE."""
    M, N, K = 1000, 600, 700
    case = Case("T", "N", M, N, K, 1.0, 0.0, kind="ints", c_kind="ints", pad=(1, 3, 0))
    need = emm.workspace_bytes("T", "N", M, N, K, "ffma")
    assert need >= 4 * K * 640   # at least the transposed copy of B (N = 600 < M), kpad(600) = 640 floats a row
    ws = torch.empty(need // 4 + 256, dtype=torch.float32, device="cuda")
    wsp = ws.data_ptr() + (-ws.data_ptr()) % 1024
    dA, dB, dC = case.flat(case.A).cuda(), case.flat(case.B).cuda(), case.Cflat.cuda()
    st = emm.sgemm_ptr("T", "N", M, N, K, 1.0, dA.data_ptr(), case.lda, dB.data_ptr(), case.ldb, 0.0, dC.data_ptr(),
                       case.ldc, torch.cuda.current_stream().cuda_stream, "ffma", wsp, need)
    torch.cuda.synchronize()
    assert st == 0, emm.strerror(st)
    R, _, _, st = case.oracle()
    assert np.array_equal(case.logical(dC.cpu()), R.astype(np.float32).astype(np.float64))
    st = emm.sgemm_ptr("T", "N", M, N, K, 1.0, dA.data_ptr(), case.lda, dB.data_ptr(), case.ldb, 0.0, dC.data_ptr(),
                       case.ldc, torch.cuda.current_stream().cuda_stream, "ffma", wsp, 1024)
    assert st == -102


@pytest.mark.parametrize("trans", ["NN", "NT", "TT", "TN"])
@pytest.mark.parametrize("shape,pad", [((1531, 997, 2049), (13, 7, 5)), ((1000, 600, 700), (0, 0, 0)),
                                       ((257, 1029, 4100), (3, 0, 1))])
def test_splitk_sub_wave(emm, monkeypatch, trans, shape, pad):
    """Sub-wave KN3b grids split K over whole promotion chunks (ffma_splits:
    c3 -> 3 splits); the fixed-order reduce launch adds the raw partial slabs,
    then alpha / beta.  FP32-accurate (oracle bound), bitwise equal on
    integer-exact data, deterministic, and the split chosen is a real one."""
    monkeypatch.delenv("EMM_FFMA_SPLITS")
    M, N, K = shape
    case = Case(trans[0], trans[1], M, N, K, -0.75, 1.25, kind="normal", pad=pad, sigma=1.0 / np.sqrt(K))
    n0 = emm.launch_count()
    G = case.run(emm, "ffma")
    n = emm.launch_count() - n0
    assert n >= 2, "expected KN3b + the split-K reduce"
    G2 = case.run(emm, "ffma")
    assert torch.equal(G.view(torch.int32), G2.view(torch.int32))
    case.check_untouched(G)
    R, S, T, st = case.oracle()
    assert st == 0
    assert_close(case, G, R, S, T, TOL["ffma"])
    ci = Case(trans[0], trans[1], M, N, K, 2.0, -1.0, kind="ints", c_kind="ints", pad=pad)
    Gi = ci.run(emm, "ffma")
    Ri, _, _, st = ci.oracle()
    assert np.array_equal(ci.logical(Gi), Ri.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("splits", [2, 3, 5])
def test_splitk_forced_matches_oracle(emm, monkeypatch, splits):
    monkeypatch.setenv("EMM_FFMA_SPLITS", str(splits))
    case = Case("N", "T", 640, 384, 3000, 1.0, 0.0, kind="normal")
    G = case.run(emm, "ffma")
    R, S, T, st = case.oracle()
    assert_close(case, G, R, S, T, TOL["ffma"])
