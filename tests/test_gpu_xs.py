"""GPU parity of KN1X, the TMA-fed 3xTF32 GEMM with the operand split inside
the kernel (EMM_SPLIT=xform, k_tcx.cu), through the C ABI.

Same bars as test_gpu_parity.py: bitwise on integer-exact inputs, the
1e-5*S + 1e-6*T predicate on random data, untouched ldc padding / guard,
A and B never written.  Extra property: the transform warpgroup writes the
plane the split pass writes for the direct path (small = rn_tf32(x -
trunc(x)), raw x as big), and the MMA sequence and schedule are KN1's, so
KN1X must equal EMM_SPLIT=pass + EMM_FORCE_DIRECT=1 BIT FOR BIT on random
data — data-parallel, split-K, stream-K and multi-wave lockstep schedules,
every transA/transB, beta = 0 and beta != 0 (TMA-fed C_in).
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
def xform(monkeypatch):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")
    monkeypatch.setenv("EMM_SPLIT", "xform")


def _exact(case, Cg, R):
    case.check_untouched(Cg)
    G = case.logical(Cg)
    assert np.array_equal(G, R.astype(np.float32).astype(np.float64)), f"max |diff| {np.max(np.abs(G - R))}"


def _bitwise_vs_pass(emm, monkeypatch, case):
    n0 = emm.launch_count()
    Cx = case.run(emm, "3xtf32")
    nx = emm.launch_count() - n0
    monkeypatch.setenv("EMM_SPLIT", "pass")
    monkeypatch.setenv("EMM_FORCE_DIRECT", "1")
    n0 = emm.launch_count()
    Cp = case.run(emm, "3xtf32")
    np_ = emm.launch_count() - n0
    monkeypatch.setenv("EMM_SPLIT", "xform")
    monkeypatch.delenv("EMM_FORCE_DIRECT")
    case.check_untouched(Cx)
    assert nx <= np_ - 1, f"xform path should save the split-pass launch ({nx} vs {np_})"
    assert torch.equal(Cx.view(torch.int32), Cp.view(torch.int32)), f"max |diff| {float((Cx - Cp).abs().max())}"
    return Cx


# TMA-legal layouts only (the path's precondition): stored rows + pad multiple of 4
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(1, 1, 1), (64, 64, 64), (300, 260, 100), (513, 257, 129), (129, 700, 33),
                                   (256, 256, 4000)])
def test_integer_exact_bitwise(emm, tA, tB, shape):
    M, N, K = shape
    for alpha, beta in ((1.0, 0.0), (-1.0, 2.0)):
        case = Case(tA, tB, M, N, K, alpha, beta, kind="ints", c_kind="ints", pad=((-M if tA == "N" else -K) % 4,
                                                                                (-K if tB == "N" else -N) % 4, 3))
        R, S, T, _ = case.oracle()
        _exact(case, case.run(emm, "3xtf32"), R)


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape,beta", [((520, 388, 200), 1.25), ((1000, 1000, 1000), 0.0),
                                        ((1024, 1024, 1024), 1.25), ((2560, 2560, 300), 0.0),
                                        ((4096, 4096, 512), 1.25)])
def test_bitwise_equal_to_split_pass(emm, monkeypatch, tA, tB, shape, beta):
    """split-K (1000^3, 1024^3), multi-wave + lockstep (2560^2), stream-K (4096^2: 3.46 waves)"""
    M, N, K = shape
    pad = ((-M if tA == "N" else -K) % 4 + 4, (-K if tB == "N" else -N) % 4, 1)
    case = cached_case(tA, tB, M, N, K, -0.75, beta, pad=pad, kind="normal")
    _bitwise_vs_pass(emm, monkeypatch, case)


@pytest.mark.parametrize("sk", ["0", "1"])
def test_streamk_forced(emm, monkeypatch, sk):
    monkeypatch.setenv("EMM_SK", sk)
    case = cached_case("N", "N", 3072, 2816, 1024, 1.0, 0.0, kind="uniform")
    _bitwise_vs_pass(emm, monkeypatch, case)


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
def test_c3_blas_stress_legal_ld(emm, tA, tB):
    """c3 (1531 x 997 x 2049, alpha = -0.75, beta = 1.25) with the TMA-legal
    reading of the padded leading dimensions (stored rows + 13 / + 7 rounded
    up to a multiple of 4)."""
    ar = 1531 if tA == "N" else 2049
    br = 2049 if tB == "N" else 997
    pad = ((ar + 13 + 3) // 4 * 4 - ar, (br + 7 + 3) // 4 * 4 - br, 5)
    case = cached_case(tA, tB, 1531, 997, 2049, -0.75, 1.25, kind="normal", pad=pad)
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, 1e-5)


@pytest.mark.parametrize("n", [512, 700, 1000, 1024, 2048])
def test_c2_square_sweep(emm, n):
    case = cached_case("N", "N", n, n, n, 1.0, 0.0)
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
    case = cached_case("T", "N", 300, 260, K, 1.0, 0.5, pad=((-K) % 4, 0, 2))
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


def test_nonfinite_inputs_propagate_like_direct_path(emm, monkeypatch):
    """inf / NaN in A: small part 0 (as PK_DSMALL), bitwise equal to the pass."""
    case = Case("N", "N", 300, 260, 100, 1.0, 0.0, kind="uniform")
    A = case.flat(case.A)
    A[5] = float("inf")
    A[777] = float("nan")
    _bitwise_vs_pass(emm, monkeypatch, case)


def test_no_workspace_entry(emm):
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


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape,beta", [((520, 388, 200), 1.25), ((2560, 2560, 300), 0.0)])
def test_rn_variant_bitwise_equal_to_repacked(emm, monkeypatch, tA, tB, shape, beta):
    """EMM_XS_RN=1: the transform rounds big = rn_tf32(x) in place and small
    = rn_tf32(x - big) — the re-buffered planes — so the result equals the
    PK_FULL3 pass + KN1 (EMM_FORCE_PACK=1) bit for bit."""
    M, N, K = shape
    pad = ((-M if tA == "N" else -K) % 4, (-K if tB == "N" else -N) % 4, 1)
    case = cached_case(tA, tB, M, N, K, -0.75, beta, pad=pad, kind="normal")
    monkeypatch.setenv("EMM_XS_RN", "1")
    Cx = case.run(emm, "3xtf32")
    monkeypatch.delenv("EMM_XS_RN")
    monkeypatch.setenv("EMM_SPLIT", "pass")
    monkeypatch.setenv("EMM_FORCE_PACK", "1")
    Cp = case.run(emm, "3xtf32")
    case.check_untouched(Cx)
    assert torch.equal(Cx.view(torch.int32), Cp.view(torch.int32)), f"max |diff| {float((Cx - Cp).abs().max())}"


@pytest.mark.parametrize("shape", [(1536, 1536, 512), (1531, 997, 2049), (1024, 1024, 1024), (512, 512, 512),
                                   (1280, 768, 3000)])
@pytest.mark.parametrize("beta", [0.0, 1.25])
def test_cluster_splitk_bitwise_equal_to_global_splitk(emm, monkeypatch, shape, beta):
    """Sub-wave shapes with S = 2..4 K splits run as one cluster of S CTA
    pairs per tile, reduced over DSMEM (CSK, opt-in EMM_CSK=1); EMM_CSK=0 runs
    the same splits through HBM slots + the fixed-order reduce launch: same
    order, same bits, one launch less."""
    monkeypatch.setenv("EMM_SPLITS", "4")   # CSK covers S <= 4 (the policy gives 512^3 S = 8); clamped per shape
    M, N, K = shape
    case = cached_case("N", "N", M, N, K, -0.75, beta, kind="normal", pad=((-M) % 4, (-K) % 4, 1))
    monkeypatch.setenv("EMM_CSK", "1")
    n0 = emm.launch_count()
    Cc = case.run(emm, "3xtf32")
    nc = emm.launch_count() - n0
    monkeypatch.setenv("EMM_CSK", "0")
    n0 = emm.launch_count()
    Cg = case.run(emm, "3xtf32")
    ng = emm.launch_count() - n0
    case.check_untouched(Cc)
    assert nc == 1 and ng == 2, (nc, ng)
    assert torch.equal(Cc.view(torch.int32), Cg.view(torch.int32)), f"max |diff| {float((Cc - Cg).abs().max())}"
    rows = np.r_[0:8, M - 8:M]
    R, S, T, _ = case.oracle(rows=rows)
    assert_close(case, Cc, R, S, T, 1e-5, rows=rows)


@pytest.mark.parametrize("math", ["3xtf32", "1xtf32"])
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(1531, 997, 2049), (520, 388, 200), (3000, 2100, 700)])
def test_repitched_illegal_ld_bitwise_equal_to_legal(emm, math, tA, tB, shape):
    """A TMA-illegal leading dimension (stored rows + 13 / + 7, c3's reading)
    makes KN1X (3xTF32) run on a raw re-pitched copy (PK_RAW): the same
    operand values as a TMA-legal layout of the same matrices, so the same
    bits.  1xTF32 re-buffers an illegal layout into TF32 planes (the pass
    rounds exactly as the direct path's TMA does, R7c): the same bits as the
    legal layout's direct call.  (A re-pitch + direct 1xTF32 variant gave the
    same bits and measured no faster at c3: TN 35.8 = 35.8 us, TT 35.8 ->
    37.9 us; not kept.)"""
    M, N, K = shape
    bad = Case(tA, tB, M, N, K, -0.75, 1.25, kind="normal", pad=(13, 7, 5))
    ar = M if tA == "N" else K
    br = K if tB == "N" else N
    good = Case(tA, tB, M, N, K, -0.75, 1.25, kind="normal", pad=((-ar) % 4 + 4, (-br) % 4, 5))
    n0 = emm.launch_count()
    Cb = bad.run(emm, math)
    nb = emm.launch_count() - n0
    Cg = good.run(emm, math)
    bad.check_untouched(Cb)
    assert torch.equal(torch.from_numpy(bad.logical(Cb)), torch.from_numpy(good.logical(Cg)))
    assert nb <= 3   # re-pitch + GEMM (+ split-K reduce)
    rows = np.r_[0:8, M - 8:M]
    R, S, T, _ = bad.oracle(rows=rows)
    assert_close(bad, Cb, R, S, T, 1e-5 if math == "3xtf32" else 5e-3, rows=rows)



@pytest.mark.parametrize("which", ["A", "B", "AB"])
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "T"), ("N", "T")])
def test_unaligned_base_pointers(emm, which, tA, tB):
    """Operands that start 4 bytes past a 16-byte boundary are TMA-illegal
    whatever their leading dimension: KN1X runs on a raw re-pitched copy —
    same bits as the same matrices at aligned addresses."""
    M, N, K = 700, 520, 300
    case = Case(tA, tB, M, N, K, 1.5, -0.5, kind="normal", pad=(4 - (M if tA == "N" else K) % 4,
                                                                 4 - (K if tB == "N" else N) % 4, 1))
    dA = case.flat(case.A).cuda()
    dB = case.flat(case.B).cuda()
    def shifted(x):
        buf = torch.empty(x.numel() + 4, dtype=torch.float32, device="cuda")
        buf[1:1 + x.numel()] = x
        return buf, buf[1:]
    keepA, sA = shifted(dA) if "A" in which else (None, dA)
    keepB, sB = shifted(dB) if "B" in which else (None, dB)
    out = []
    for a, b in ((sA, sB), (dA, dB)):
        dC = case.Cflat.cuda()
        st = emm.sgemm_ptr(tA, tB, M, N, K, 1.5, a.data_ptr(), case.lda, b.data_ptr(), case.ldb, -0.5, dC.data_ptr(),
                           case.ldc, torch.cuda.current_stream().cuda_stream, "3xtf32")
        torch.cuda.synchronize()
        assert st == 0
        out.append(dC.cpu())
    case.check_untouched(out[0])
    assert torch.equal(out[0].view(torch.int32), out[1].view(torch.int32))
    rows = np.r_[0:8, M - 8:M]
    R, S, T, _ = case.oracle(rows=rows)
    assert_close(case, out[0], R, S, T, 1e-5, rows=rows)
