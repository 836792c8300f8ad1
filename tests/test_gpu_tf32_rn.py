"""1xTF32 operand rounding on the direct path (R7c).

The tensor core truncates raw FP32 operands to TF32 (R7b); the direct
1xTF32 path reads the caller's arrays through tensor maps of data type
TFLOAT32, whose TMA loads round each element to nearest-even TF32 (the same
bits as cvt.rn.tf32.f32 on ties, specials and random words:
tools/tma_tf32_probe.cu, profiles/r02_tma_tf32_probe.txt).  So:

* direct 1xTF32 equals the re-buffered path (PK_FULL1 pass: big =
  rn_tf32(x), K-major copy + KN1) BIT FOR BIT, every transA/transB, beta = 0
  and beta != 0, unaligned leading dimensions; so does direct TF32+BF16
  (PK_DCROSS cross plane made against big = rn_tf32(x)) against PK_FULLX;
* the result is the FP32-accurate product of the RN-rounded inputs: within
  1e-5*S + 1e-6*T of the oracle run on rn_tf32(A), rn_tf32(B) (rounding
  written out below from its definition, not from the library), on
  same-sign data at K = 4096 where truncated inputs would miss that bound by
  far (checked: the truncated-input oracle result is outside it).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from test_gpu_parity import Case, cached_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


@pytest.fixture(autouse=True)
def tensor_path(monkeypatch):
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")   # no FFMA tiny kernel
    monkeypatch.setenv("EMM_SKINNY_TC", "0")


def rn_tf32(x: np.ndarray) -> np.ndarray:
    """Round FP32 to the nearest TF32 (10 stored mantissa bits), ties to even.
    Finite inputs only (the test data)."""
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 13) & 1
    r = ((u + 0xFFF + lsb) & ~np.uint64(0x1FFF)).astype(np.uint32)
    return r.view(np.float32)


def trunc_tf32(x: np.ndarray) -> np.ndarray:
    u = x.astype(np.float32).view(np.uint32)
    return (u & np.uint32(0xFFFFE000)).view(np.float32)


def test_rn_tf32_definition():
    """The test's own rounding against hand-worked words (1 + k*2^-23)."""
    one = np.float32(1.0).view(np.uint32)
    w = np.array([one + 0x0FFF, one + 0x1000, one + 0x1001, one + 0x3000, one + 0x2FFF], dtype=np.uint32)
    got = rn_tf32(w.view(np.float32)).view(np.uint32)
    assert list(got - one) == [0, 0, 0x2000, 0x4000, 0x2000]


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape,beta,pad", [((520, 388, 200), 1.25, True), ((2560, 2560, 300), 0.0, False),
                                            ((1531, 997, 2049), -0.5, False)])
@pytest.mark.parametrize("math", ["1xtf32", "tf32bf16"])
def test_direct_bitwise_equal_to_repacked(emm, monkeypatch, math, tA, tB, shape, beta, pad):
    M, N, K = shape
    p = ((-M if tA == "N" else -K) % 4, (-K if tB == "N" else -N) % 4, 1) if pad else (0, 0, 0)
    case = cached_case(tA, tB, M, N, K, -0.75, beta, pad=p, kind="normal")
    if not all(ld % 4 == 0 for ld in (case.lda, case.ldb)):
        pytest.skip("direct path needs 16-byte leading dimensions")
    monkeypatch.setenv("EMM_FORCE_DIRECT", "1")
    Cd = case.run(emm, math)
    monkeypatch.delenv("EMM_FORCE_DIRECT")
    monkeypatch.setenv("EMM_FORCE_PACK", "1")
    Cp = case.run(emm, math)
    case.check_untouched(Cd)
    assert torch.equal(Cd.view(torch.int32), Cp.view(torch.int32)), f"max |diff| {float((Cd - Cp).abs().max())}"


@pytest.mark.parametrize("direct", [True, False])
def test_product_of_rounded_inputs(emm, monkeypatch, direct):
    M, N, K = 384, 320, 4096
    case = Case("N", "T", M, N, K, 1.0, 0.0, kind="uniform01")
    monkeypatch.setenv("EMM_FORCE_DIRECT" if direct else "EMM_FORCE_PACK", "1")
    G = case.logical(case.run(emm, "1xtf32"))
    A = case.flat(case.A).numpy()
    B = case.flat(case.B).numpy()
    C = case.Cflat.numpy()

    def ref(f):
        return oracle.sgemm_sub("N", "T", M, N, K, 1.0, f(A), case.lda, f(B), case.ldb, 0.0, C, case.ldc)

    R, S, T, st = ref(rn_tf32)
    assert st == 0
    bound = 1e-5 * S + 1e-6 * T
    err = np.abs(G - R)
    assert np.all(err <= bound), f"max err/bound {float(np.max(err / bound)):.3g}"
    # the pin discriminates: truncated inputs (the raw tensor-core reading)
    # land far outside the bound on this same-sign data
    Rt = ref(trunc_tf32)[0]
    assert np.max(np.abs(Rt - R) / bound) > 10
