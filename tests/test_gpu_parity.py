"""GPU parity: the CUDA path through the C ABI vs the oracle, element by
element on the same seeded inputs (BASELINE.json configs + edge cases).

Bars (BASELINE.json north_star):
* integer-exact inputs (ints in [-8,8], alpha,beta in {1,-1,2}): every path
  must equal the oracle BITWISE (all partial sums are exact integers < 2^24);
* FP32-accurate paths (3xtf32, ffma): |C - R| <= 1e-5*S + 1e-6*T per entry;
* 1xtf32: |C - R| <= 5e-3*S + 1e-6*T;
* non-finite oracle entries must match by class;
* nothing outside the M x N logical region changes (ldc padding + a guard
  region after C keep their sentinel); A and B are never written;
* results are run-to-run bitwise deterministic.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu



@pytest.fixture(autouse=True)
def force_requested_path(monkeypatch):
    """The library sends latency-bound problems (2MNK <= 2^24) to the FFMA
    kernel; these tests force every requested path at every size
    (EMM_SMALL_FLOPS=0); test_small_problem_default_path covers the default."""
    monkeypatch.setenv("EMM_SMALL_FLOPS", "0")

TOL = {"3xtf32": 1e-5, "ffma": 1e-5, "1xtf32": 5e-3, "tf32bf16": 1e-5}
MATHS = ["3xtf32", "ffma", "1xtf32", "tf32bf16"]
SENTINEL = -12345.0
GUARD = 4096


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


_CASES = {}


def cached_case(*args, **kw):
    """Inputs are immutable per (args, kw): generate big ones once per module."""
    key = (args, tuple(sorted(kw.items())))
    if key not in _CASES:
        _CASES[key] = Case(*args, **kw)
    return _CASES[key]


def stored(trans, r, c):
    return (r, c) if trans in "Nn" else (c, r)


class Case:
    """Inputs of one SGEMM call, on host (flat storages) and device."""

    def __init__(self, tA, tB, M, N, K, alpha, beta, kind="uniform", pad=(0, 0, 0), sigma=1.0,
                 c_kind="uniform", seed=0):
        self.tA, self.tB, self.M, self.N, self.K = tA, tB, M, N, K
        self.alpha, self.beta = alpha, beta
        ar, ac = stored(tA, M, K)
        br, bc = stored(tB, K, N)
        self.lda, self.ldb, self.ldc = max(1, ar) + pad[0], max(1, br) + pad[1], max(1, M) + pad[2]
        self.A = datagen.matrix(kind, datagen.TAG_A, ar, ac, self.lda, seed=seed, sigma=sigma)
        self.B = datagen.matrix(kind, datagen.TAG_B, br, bc, self.ldb, seed=seed, sigma=sigma)
        Cv = datagen.matrix(c_kind, datagen.TAG_C, M, N, self.ldc, seed=seed, sigma=sigma,
                            pad_value=SENTINEL)
        self.Cflat = torch.full((self.ldc * max(N, 1) + GUARD,), SENTINEL, dtype=torch.float32)
        if M * N:
            self.Cflat[: self.ldc * N] = datagen.storage_of(Cv)

    def flat(self, x):
        return datagen.storage_of(x) if x.numel() else torch.zeros(1)

    def oracle(self, rows=None, cols=None):
        C = self.Cflat.numpy()
        return oracle.sgemm_sub(self.tA, self.tB, self.M, self.N, self.K, self.alpha,
                                self.flat(self.A).numpy(), self.lda, self.flat(self.B).numpy(), self.ldb,
                                self.beta, C, self.ldc, rows=rows, cols=cols)

    def run(self, emm, math, stream=None):
        dA = self.flat(self.A).cuda()
        dB = self.flat(self.B).cuda()
        dC = self.Cflat.cuda()
        st = emm.sgemm_ptr(self.tA, self.tB, self.M, self.N, self.K, self.alpha, dA.data_ptr(), self.lda,
                           dB.data_ptr(), self.ldb, self.beta, dC.data_ptr(), self.ldc,
                           torch.cuda.current_stream().cuda_stream, math)
        torch.cuda.synchronize()
        assert st == 0, emm.strerror(st)
        # A and B (NaN padding included) are never written: compare bit patterns
        assert torch.equal(dA.cpu().view(torch.int32), self.flat(self.A).view(torch.int32))
        assert torch.equal(dB.cpu().view(torch.int32), self.flat(self.B).view(torch.int32))
        return dC.cpu()

    def logical(self, Cflat):
        if self.M * self.N == 0:
            return np.zeros((self.M, self.N))
        return Cflat[: self.ldc * self.N].reshape(self.N, self.ldc)[:, : self.M].T.double().numpy()

    def check_untouched(self, Cflat):
        full = Cflat.reshape(-1)
        if self.M * self.N:
            body = full[: self.ldc * self.N].reshape(self.N, self.ldc)
            assert torch.all(body[:, self.M:] == SENTINEL), "ldc padding modified"
        assert torch.all(full[self.ldc * self.N:] == SENTINEL) if self.M * self.N else True, "guard modified"


def assert_close(case, Cg, R, S, T, tol, rows=None, cols=None):
    G = case.logical(Cg)
    if rows is not None:
        G = G[np.ix_(rows, cols if cols is not None else np.arange(case.N))]
    fin = np.isfinite(R)
    err = np.abs(G - R)
    bound = tol * S + 1e-6 * T
    bad = fin & ~(err <= bound)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{bad.sum()} entries out of tolerance; first {tuple(i)}: gpu={G[tuple(i)]!r} "
                             f"ref={R[tuple(i)]!r} err/tol={err[tuple(i)] / max(bound[tuple(i)], 1e-300):.3g}; "
                             f"max err/tol={np.max(np.where(fin, err / np.maximum(bound, 1e-300), 0)):.3g}")
    if (~fin).any():
        assert np.array_equal(np.isnan(G[~fin]), np.isnan(R[~fin]))
        assert np.array_equal(np.sign(G[~fin & ~np.isnan(R)]), np.sign(R[~fin & ~np.isnan(R)]))
    return float(np.max(np.where(fin, err / np.maximum(bound, 1e-300), 0))) if R.size else 0.0


# --------------------------------------------------------------------------
# bitwise on integer-exact inputs (all paths, all trans, ragged shapes)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(1, 1, 1), (64, 64, 64), (300, 260, 100), (513, 257, 129), (129, 700, 33)])
def test_integer_exact_bitwise(emm, math, tA, tB, shape):
    M, N, K = shape
    for alpha, beta in ((1.0, 0.0), (-1.0, 2.0)):
        case = Case(tA, tB, M, N, K, alpha, beta, kind="ints", c_kind="ints", pad=(3, 1, 2))
        R, S, T, st = case.oracle()
        Cg = case.run(emm, math)
        case.check_untouched(Cg)
        G = case.logical(Cg)
        assert np.array_equal(G, R.astype(np.float32).astype(np.float64)), \
            f"max |diff| {np.max(np.abs(G - R))}"


@pytest.mark.parametrize("force_pack", ["0", "1", "pass"])
@pytest.mark.parametrize("math", ["3xtf32", "1xtf32", "tf32bf16"])
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
def test_direct_and_repacked_paths(emm, monkeypatch, force_pack, math, tA, tB):
    """TMA-legal leading dimensions take the direct path (operands read in
    place, K- or MN-major per trans flag, transpose in the TMA box; 3xTF32:
    the in-kernel split KN1X by default, the split pass + KN1 with
    EMM_SPLIT=pass); with EMM_FORCE_PACK=1 the same call takes the
    re-buffering fallback.  All must be bitwise exact on integer inputs and
    within tolerance on random ones, including ragged M/N/K tails (M, N, K
    not multiples of 32/256)."""
    if force_pack == "pass":
        monkeypatch.setenv("EMM_SPLIT", "pass")
        force_pack = "0"
    monkeypatch.setenv("EMM_FORCE_PACK", force_pack)
    monkeypatch.setenv("EMM_FORCE_DIRECT", "1" if force_pack == "0" else "0")
    for (M, N, K) in [(520, 388, 200), (260, 1000, 72)]:
        case = Case(tA, tB, M, N, K, 1.0, -1.0, kind="ints", c_kind="ints", pad=(4, 8, 3))
        R, S, T, _ = case.oracle()
        Cg = case.run(emm, math)
        case.check_untouched(Cg)
        assert np.array_equal(case.logical(Cg), R.astype(np.float32).astype(np.float64))
        case = Case(tA, tB, M, N, K, 0.75, 0.5, pad=(4, 0, 1))
        R, S, T, _ = case.oracle()
        Cg = case.run(emm, math)
        case.check_untouched(Cg)
        assert_close(case, Cg, R, S, T, TOL[math])


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(20000, 16, 700), (5003, 3, 1000), (9, 30001, 300), (16, 7000, 257)])
def test_skinny_path(emm, math, tA, tB, shape):
    """min(M, N) <= 16: the streaming kernels (operand-role swap when M is the
    short side; FFMA KN9, or the tensor-core KN9T for 1xTF32 with a
    K-contiguous long operand and a short side > 8); bitwise on integers, the
    requested mode's bound on random data, ldc padding untouched."""
    M, N, K = shape
    case = cached_case(tA, tB, M, N, K, 1.0, 2.0, kind="ints", c_kind="ints", pad=(1, 2, 3))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    assert np.array_equal(case.logical(Cg), R.astype(np.float32).astype(np.float64))
    case = cached_case(tA, tB, M, N, K, -0.5, 0.25, pad=(0, 1, 0))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    assert_close(case, Cg, R, S, T, TOL[math])


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(4000, 16, 9000), (16, 3000, 5000), (9000, 5, 2049), (7, 2000, 40000)])
def test_skinny_ffma_splitk(emm, monkeypatch, tA, tB, shape):
    """FFMA skinny kernel (KN9) with few row blocks and a long K: split over
    256-of-K promotion groups + the fixed-order reduce launch (2-3 launches);
    bitwise on integers (beta != 0 included), FP32 bound on random data,
    deterministic, and within the bound of the unsplit run."""
    monkeypatch.setenv("EMM_SKINNY_TC", "0")
    M, N, K = shape
    # TMA-legal leading dimensions (the split runs in the TMA streaming kernel)
    pa = (-(M if tA == "N" else K)) % 4 + 4
    pb = (-(K if tB == "N" else N)) % 4 + 4
    case = Case(tA, tB, M, N, K, 2.0, -1.0, kind="ints", c_kind="ints", pad=(pa, pb, 3))
    R, S, T, _ = case.oracle()
    n0 = emm.launch_count()
    Cg = case.run(emm, "ffma")
    # the split kernel + its reduce (+ the B' transpose for a K-contiguous long operand)
    assert emm.launch_count() - n0 in (2, 3), "expected the split kernel + its reduce"
    case.check_untouched(Cg)
    assert np.array_equal(case.logical(Cg), R.astype(np.float32).astype(np.float64))
    case = Case(tA, tB, M, N, K, -0.5, 0.25, kind="normal", pad=(pa, pb, 1), sigma=1.0 / np.sqrt(K))
    R, S, T, _ = case.oracle()
    G1 = case.run(emm, "ffma")
    G2 = case.run(emm, "ffma")
    assert torch.equal(G1.view(torch.int32), G2.view(torch.int32))
    assert_close(case, G1, R, S, T, TOL["ffma"])
    monkeypatch.setenv("EMM_SKINNY_SPLITS", "1")
    G0 = case.run(emm, "ffma")
    assert_close(case, G0, R, S, T, TOL["ffma"])


def test_spec_worked_example_bitwise(emm):
    """tests/golden/spec_2x2.txt: [[1,2],[3,4]]·[[5,6],[7,8]] = [[19,22],[43,50]] (column-major)."""
    for math in MATHS:
        A = torch.tensor([1, 3, 2, 4], dtype=torch.float32, device="cuda")
        B = torch.tensor([5, 7, 6, 8], dtype=torch.float32, device="cuda")
        C = torch.full((4,), float("nan"), device="cuda")
        st = emm.sgemm_ptr("N", "N", 2, 2, 2, 1.0, A.data_ptr(), 2, B.data_ptr(), 2, 0.0, C.data_ptr(), 2,
                           torch.cuda.current_stream().cuda_stream, math)
        torch.cuda.synchronize()
        assert st == 0 and C.cpu().tolist() == [19, 43, 22, 50]


# --------------------------------------------------------------------------
# tolerance on the BASELINE.json configs
# --------------------------------------------------------------------------
@pytest.mark.parametrize("math", MATHS)
def test_c1_64cubed(emm, math):
    case = Case("N", "N", 64, 64, 64, 1.0, 0.0)
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, TOL[math])


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("n", [100, 333, 512, 700, 1000, 1024, 2048])
def test_c2_square_sweep(emm, math, n):
    case = Case("N", "N", n, n, n, 1.0, 0.0)
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, TOL[math])


@pytest.mark.parametrize("math", MATHS)
def test_c2_4096_sampled_rows(emm, math):
    n = 4096
    case = Case("N", "N", n, n, n, 1.0, 0.0)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([[0, 1, 255, 256, n - 1], rng.integers(0, n, 27)]))
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, math)
    assert_close(case, Cg, R, S, T, TOL[math], rows=rows)


@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
def test_c3_blas_stress(emm, math, tA, tB):
    """configs[2] with the valid reading lda = stored rows + 13 (R3)."""
    case = cached_case(tA, tB, 1531, 997, 2049, -0.75, 1.25, kind="normal", c_kind="uniform", pad=(13, 7, 5))
    rows = np.arange(0, 1531, 3) if math == "ffma" else None
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, TOL[math], rows=rows)


@pytest.mark.parametrize("math", ["3xtf32", "1xtf32", "tf32bf16"])
@pytest.mark.parametrize("shape", [(65536, 1024, 4096), (65536, 4096, 1024)])
def test_c4_nn_layer_sampled(emm, math, shape):
    M, N, K = shape
    case = cached_case("N", "T", M, N, K, 1.0, 1.0, kind="normal", c_kind="normal", sigma=1.0 / np.sqrt(K))
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([[0, 255, 256, M - 1], rng.integers(0, M, 12)]))
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, math)
    assert_close(case, Cg, R, S, T, TOL[math], rows=rows)


# --------------------------------------------------------------------------
# edge cases
# --------------------------------------------------------------------------
@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("K", [1, 7, 31, 33, 337, 2049])
def test_k_tails(emm, math, K):
    case = Case("N", "N", 257, 129, K, 1.0, 0.0, pad=(3, 3, 3))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, TOL[math])


@pytest.mark.parametrize("no_skinny", ["0", "1"])
@pytest.mark.parametrize("math", MATHS)
@pytest.mark.parametrize("mn", [(1, 1), (1, 300), (300, 1), (7, 5), (127, 129), (255, 257), (256, 256)])
def test_mn_edges(emm, monkeypatch, no_skinny, math, mn):
    monkeypatch.setenv("EMM_NO_SKINNY", no_skinny)
    M, N = mn
    for tA, tB in (("N", "N"), ("T", "T")):
        case = Case(tA, tB, M, N, 77, -0.75, 1.25, pad=(3, 0, 3))
        R, S, T, _ = case.oracle()
        Cg = case.run(emm, math)
        case.check_untouched(Cg)
        assert_close(case, Cg, R, S, T, TOL[math])


@pytest.mark.parametrize("math", MATHS)
def test_alpha_zero_never_reads_AB(emm, math):
    M, N, K = 200, 100, 50
    for beta in (0.0, 2.0):
        A = torch.full((M * K,), float("nan"), device="cuda")
        B = torch.full((K * N,), float("nan"), device="cuda")
        Cv = datagen.matrix("uniform", datagen.TAG_C, M, N)
        C = datagen.storage_of(Cv).cuda()
        st = emm.sgemm_ptr("N", "N", M, N, K, 0.0, A.data_ptr(), M, B.data_ptr(), K, beta, C.data_ptr(), M,
                           torch.cuda.current_stream().cuda_stream, math)
        torch.cuda.synchronize()
        assert st == 0
        expect = datagen.storage_of(Cv) * beta if beta != 0 else torch.zeros(M * N)
        assert torch.equal(C.cpu(), expect)


@pytest.mark.parametrize("math", MATHS)
def test_beta_zero_never_reads_C(emm, math):
    case = Case("N", "N", 130, 70, 40, 1.0, 0.0)
    case.Cflat[: case.ldc * case.N] = float("nan")
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    G = case.logical(Cg)
    assert np.all(np.isfinite(G))
    assert_close(case, Cg, R, S, T, TOL[math])


@pytest.mark.parametrize("math", MATHS)
def test_K_zero_scales_C(emm, math):
    case = Case("N", "N", 100, 60, 0, 1.0, -2.0)
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    assert np.array_equal(case.logical(Cg), R.astype(np.float32).astype(np.float64))


def test_empty_is_noop(emm):
    C = torch.full((16,), 3.0, device="cuda")
    n0 = emm.launch_count()
    assert emm.sgemm_ptr("N", "N", 0, 4, 5, 1.0, 0, 1, 0, 5, 0.0, C.data_ptr(), 1, None, "3xtf32") == 0
    assert emm.sgemm_ptr("N", "N", 4, 0, 5, 1.0, 0, 4, 0, 5, 0.0, C.data_ptr(), 4, None, "3xtf32") == 0
    assert emm.launch_count() == n0
    assert torch.all(C == 3.0)


def test_argument_error_leaves_C_unmodified(emm):
    C = torch.full((64,), 5.0, device="cuda")
    A = torch.ones(64, device="cuda")
    st = emm.sgemm_ptr("N", "N", 8, 8, 8, 1.0, A.data_ptr(), 7, A.data_ptr(), 8, 0.0, C.data_ptr(), 8, None)
    assert st == -8
    torch.cuda.synchronize()
    assert torch.all(C == 5.0)


@pytest.mark.parametrize("math", MATHS)
def test_deterministic(emm, math):
    case = Case("N", "T", 700, 900, 1500, 1.0, 0.5)
    c1 = case.run(emm, math)
    c2 = case.run(emm, math)
    assert torch.equal(c1, c2)


def test_accumulate_property(emm):
    """GEMM into C twice with beta=1 == once with 2B (tolerance-scaled)."""
    M, N, K = 500, 300, 700
    case = Case("N", "N", M, N, K, 1.0, 1.0)
    c0 = case.Cflat.clone()
    case.Cflat = case.run(emm, "3xtf32")
    c_twice = case.run(emm, "3xtf32")
    B2 = (case.flat(case.B) * 2).numpy()
    R, S, T, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, case.flat(case.A).numpy(), case.lda, B2, case.ldb,
                                  1.0, c0.numpy(), case.ldc)
    # two FP32 roundings of the partial result: 2 x the single-call bound
    assert_close(case, c_twice, R, 2 * S, 2 * T, 1e-5)


@pytest.mark.parametrize("math", ["3xtf32", "ffma", "tf32bf16"])
@pytest.mark.parametrize("K", [4096, 32768])
def test_same_sign_accumulation(emm, math, K):
    """Same-sign U[0,1) data at large K (Q7): a truncating
    tensor-core accumulator biases the sum (measured 17.6x over the bound at
    K=16384 without promotion); with FP32 promotion every 256 of K the FP32-
    accurate bound 1e-5*S must hold here too."""
    case = cached_case("N", "N", 256, 256, K, 1.0, 0.0, kind="uniform01")
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, math)
    r = assert_close(case, Cg, R, S, T, 1e-5)
    print(f"same-sign K={K} {math}: max err/tol = {r:.3g}")


@pytest.mark.parametrize("tA", ["N", "T"])
@pytest.mark.parametrize("tB", ["N", "T"])
@pytest.mark.parametrize("shape", [(1, 1, 1), (33, 65, 129), (300, 260, 333), (517, 389, 1025), (64, 64, 64)])
@pytest.mark.parametrize("tile", ["32", "64"])
def test_tiny_kernel_every_layout(emm, monkeypatch, tA, tB, shape, tile):
    """KN10 (forced for every size): 4x4 outputs per thread, K split over four
    thread groups added in fixed order, cp.async ring with zero-filled edges —
    bitwise on integers, FP32-accurate on random data, padding untouched."""
    monkeypatch.setenv("EMM_SMALL_FLOPS", "1e15")
    monkeypatch.setenv("EMM_TINY_T", tile)
    M, N, K = shape
    case = Case(tA, tB, M, N, K, 2.0, -1.0, kind="ints", c_kind="ints", pad=(3, 1, 2))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "3xtf32")
    case.check_untouched(Cg)
    assert np.array_equal(case.logical(Cg), R.astype(np.float32).astype(np.float64))
    case = Case(tA, tB, M, N, K, -0.75, 1.25, kind="normal", pad=(1, 2, 3))
    R, S, T, _ = case.oracle()
    Cg = case.run(emm, "ffma")
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, 1e-5)


@pytest.mark.parametrize("shape", [(64, 64, 64), (100, 100, 100), (7, 300, 5), (333, 333, 333), (700, 650, 600),
                                   (1000, 1000, 1000)])
def test_small_problem_default_path(emm, monkeypatch, shape):
    monkeypatch.delenv("EMM_SMALL_FLOPS")
    M, N, K = shape
    case = Case("N", "N", M, N, K, 1.0, 0.0)
    R, S, T, _ = case.oracle()
    tiny_all = 2 * M * N * K <= 1 << 27   # tiny kernel for every mode; above, only for FFMA (<= 7e8 flops)
    for math in MATHS:
        Cg = case.run(emm, math)
        case.check_untouched(Cg)
        # the tiny FFMA kernel is FP32-accurate for every mode
        assert_close(case, Cg, R, S, T, 1e-5 if tiny_all else TOL[math])


@pytest.mark.parametrize("math", ["3xtf32", "1xtf32", "tf32bf16"])
@pytest.mark.parametrize("shape", [(1531, 997, 2049), (1024, 1024, 1024), (700, 700, 700), (257, 300, 4000)])
def test_split_k_deterministic_and_close(emm, math, shape):
    """Sub-wave shapes take split-K (partials + fixed-order reduce): results
    must be within tolerance and bitwise reproducible."""
    M, N, K = shape
    case = cached_case("N", "N", M, N, K, 0.5, -1.0, pad=(1, 2, 3))
    R, S, T, _ = case.oracle()
    c1 = case.run(emm, math)
    c2 = case.run(emm, math)
    assert torch.equal(c1, c2)
    case.check_untouched(c1)
    assert_close(case, c1, R, S, T, TOL[math])


def test_torch_binding_colmajor(emm):
    M, N, K = 300, 200, 100
    A = torch.randn(K, M, device="cuda").t()   # (M, K) with stride (1, M): column-major
    B = torch.randn(N, K, device="cuda").t()
    C = torch.zeros(N, M, device="cuda").t()
    emm.sgemm(A, B, C)
    ref = (A.double() @ B.double())
    assert torch.allclose(C.double(), ref, atol=1e-4, rtol=0)


@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "T"), ("N", "T")])
@pytest.mark.parametrize("beta", [0.0, 0.5])
@pytest.mark.parametrize("blocks", [None, (256, 512), "ksplit", "ksplit3"],
                         ids=["default", "first256-chunk512", "ksplit", "ksplit3"])
@pytest.mark.parametrize("host_pack", [False, True], ids=["xs", "planes"])
def test_host_buffer_pipelined(emm, monkeypatch, tA, tB, beta, blocks, host_pack):
    """emm_sgemm_host above 4096 x 4096 runs the copy/compute pipeline (L-
    shaped growth over 2048-row/column blocks, the first two 1024, ragged
    last blocks here; three streams; KN1X on the landed blocks in place, or
    with EMM_HOST_PACK=1 re-buffered planes + KN1; each GEMM region in
    pieces with its own copy-back): same bits as the device call of the same
    arithmetic (default KN1X / EMM_FORCE_PACK=1; K = 300 < 512: stream-K
    pieces sum like the sequential K loop), ldc padding intact, sampled rows
    against the oracle."""
    if host_pack:
        monkeypatch.setenv("EMM_HOST_PACK", "1")
    M, N, K = 4500, 4200, 300
    if blocks == "ksplit3":   # three K phases (the middle one both reads and writes the partials)
        monkeypatch.setenv("EMM_HOST_KPHASES", "3")
    if blocks in ("ksplit", "ksplit3"):
        # two K phases (K1 = 512, a promotion boundary), the second continuing
        # from the first's raw partials: still the device call's bits (stream-K
        # off there: its piece sums are not the sequential K loop above 512)
        monkeypatch.setenv("EMM_HOST_KSPLIT", "1")
        monkeypatch.setenv("EMM_SK", "0")
        K = 1300 if blocks == "ksplit" else 2000
    elif blocks:
        monkeypatch.setenv("EMM_HOST_FIRST", str(blocks[0]))
        monkeypatch.setenv("EMM_HOST_CHUNK", str(blocks[1]))
    case = cached_case(tA, tB, M, N, K, 1.25, beta, pad=(4, 4, 3))
    rows = np.array([0, 1, 1023, 1151, 1152, 2999, M - 1])
    R, S, T, _ = case.oracle(rows=rows)
    Cf = case.Cflat.clone().pin_memory()
    Af, Bf = case.flat(case.A).pin_memory(), case.flat(case.B).pin_memory()
    emm.sgemm_host(tA, tB, M, N, K, 1.25, Af, case.lda, Bf, case.ldb, beta, Cf, case.ldc)
    case.check_untouched(Cf)
    assert_close(case, Cf, R, S, T, 1e-5, rows=rows)
    if host_pack:
        monkeypatch.setenv("EMM_FORCE_PACK", "1")
    Cd = case.run(emm, "3xtf32")
    assert torch.equal(Cd.view(torch.int32), Cf.view(torch.int32))


def test_host_buffer_entry(emm):
    M, N, K = 333, 257, 129
    case = Case("T", "N", M, N, K, 1.5, -0.5, pad=(1, 2, 3))
    R, S, T, _ = case.oracle()
    Cf = case.Cflat.clone().pin_memory()
    emm.sgemm_host("T", "N", M, N, K, 1.5, case.flat(case.A), case.lda, case.flat(case.B), case.ldb, -0.5, Cf,
                   case.ldc)
    case.check_untouched(Cf)
    assert_close(case, Cf, R, S, T, 1e-5)


@pytest.mark.parametrize("tA,tB", [("T", "N"), ("N", "N"), ("T", "T")])
def test_host_buffer_entry_ffma_relayout(emm, tA, tB):
    """emm_sgemm_host in the FFMA mode on c3 (TMA-illegal / TN device copies:
    relayout copy + split-K KN3b through the host path's cached workspace)."""
    M, N, K = 1531, 997, 2049
    case = cached_case(tA, tB, M, N, K, -0.75, 1.25, pad=(13, 7, 5), kind="normal")
    R, S, T, _ = case.oracle()
    Cf = case.Cflat.clone().pin_memory()
    emm.sgemm_host(tA, tB, M, N, K, -0.75, case.flat(case.A), case.lda, case.flat(case.B), case.ldb, 1.25, Cf,
                   case.ldc, math="ffma")
    case.check_untouched(Cf)
    assert_close(case, Cf, R, S, T, 1e-5)


@pytest.mark.parametrize("math", ["3xtf32", "tf32bf16", "ffma"])
@pytest.mark.parametrize("shape,tA,tB", [((1 << 20, 256, 64), "N", "N"),      # 4096 tile rows, multi-wave
                                         ((256, 256, 1 << 20), "T", "N"),      # K = 2^20: split-K x16, 2048 stages each
                                         ((300, 1 << 18, 96), "N", "T")])      # 1024 tile columns
def test_extreme_extents(emm, math, shape, tA, tB):
    """Maximum-extent cases: very long M, N or K (tile counts, split-K
    ranges and 64-bit offsets far from the tested mid sizes).  Integer-exact
    data (|sums| < 2^24 except for K = 2^20, checked with the tolerance)."""
    M, N, K = shape
    exact = K < (1 << 16)
    case = cached_case(tA, tB, M, N, K, 1.0, 0.0, kind="ints" if exact else "uniform")
    rows = np.unique(np.r_[0:4, M // 2:M // 2 + 4, M - 4:M])
    R, S, T, _ = case.oracle(rows=rows)
    Cg = case.run(emm, math)
    case.check_untouched(Cg)
    G = case.logical(Cg)[rows]
    if exact:
        assert np.array_equal(G, R.astype(np.float32).astype(np.float64))
    else:
        assert_close(case, Cg, R, S, T, TOL[math], rows=rows)


@pytest.mark.parametrize("tA,tB,shape", [("N", "N", (20000, 16, 700)), ("N", "N", (9001, 9, 1500)), ("N", "N", (70001, 16, 1000)),
                                         ("N", "N", (4000, 12, 9000)), ("T", "T", (16, 30000, 300)),
                                         ("N", "T", (20000, 16, 700))])
def test_skinny_bt_nn_bitwise(emm, monkeypatch, tA, tB, shape):
    """MN-contiguous long operand with a K-contiguous B' and N' > 8 (NN with N
    short, TT with M short): B' transposed to [k][N'] tiles first
    (EMM_SKINNY_BT_NN=1; the default for N' > 8 on a long operand of >= 2^26
    elements) is bitwise equal to reading the [N'][k] tiles directly (=0) —
    each entry is the same FFMA sequence in increasing k — and within the FP32
    bound of the oracle; ldc padding untouched."""
    monkeypatch.setenv("EMM_SKINNY_TC", "0")
    M, N, K = shape
    pa = (-(M if tA == "N" else K)) % 4 + 4
    pb = (-(K if tB == "N" else N)) % 4 + 4
    case = Case(tA, tB, M, N, K, -0.5, 0.25, kind="normal", pad=(pa, pb, 1), sigma=1.0 / np.sqrt(K))
    R, S, T, _ = case.oracle()
    runs = {}
    for bt in ("1", "0", None):   # forced on, forced off, default policy
        if bt is None:
            monkeypatch.delenv("EMM_SKINNY_BT_NN")
        else:
            monkeypatch.setenv("EMM_SKINNY_BT_NN", bt)
        n0 = emm.launch_count()
        G = case.run(emm, "3xtf32")
        runs[bt] = (G, emm.launch_count() - n0)
        case.check_untouched(G)
        assert_close(case, G, R, S, T, TOL["3xtf32"])
        assert torch.equal(G.view(torch.int32), runs["1"][0].view(torch.int32))
    # the transpose launch is there only for a K-contiguous B' (not NT) ...
    kcontig = (tA, tB) != ("N", "T")
    assert runs["1"][1] - runs["0"][1] == (1 if kcontig else 0)
    # ... and by default only for N' > 8 and a long operand of >= 2^26 elements
    mr, nc = (M, N) if N <= 16 else (N, M)
    want = kcontig and nc > 8 and mr * K >= 1 << 26
    assert runs[None][1] == runs["1" if want else "0"][1]
