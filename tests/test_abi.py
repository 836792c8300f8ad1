"""CPU-side tests of the C-ABI boundary: the library loads, exports every
symbol include/emm.h declares, validates arguments with the BLAS numbering
before touching any device, and its host-only logic (row partition, error
strings, workspace sizing) is right.  No compute calls (no GPU here)."""
from __future__ import annotations

import ctypes
import os
import re

import pytest
import torch

import __graft_entry__  # noqa: F401  (repo root on sys.path via conftest)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    return e


def header_functions():
    txt = open(os.path.join(ROOT, "include", "emm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(emm_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_header_symbol(emm):
    names = header_functions()
    assert len(names) >= 15
    L = ctypes.CDLL(emm.emm._LIB_PATH)
    for n in names:
        assert hasattr(L, n), n


def test_no_torch_types_in_header():
    txt = open(os.path.join(ROOT, "include", "emm.h")).read()
    assert "torch" not in txt.replace("torch.distributed", "").replace("with torch", "")
    assert "extern \"C\"" in txt


ARGS_OK = dict(transA="N", transB="N", M=4, N=3, K=2, alpha=1.0, A=4096, lda=4, B=8192, ldb=2,
               beta=0.0, C=16384, ldc=4)


def call(emm, **kw):
    a = dict(ARGS_OK)
    a.update(kw)
    return emm.sgemm_ptr(a["transA"], a["transB"], a["M"], a["N"], a["K"], a["alpha"], a["A"], a["lda"],
                         a["B"], a["ldb"], a["beta"], a["C"], a["ldc"], None, kw.get("math", "3xtf32"))


@pytest.mark.parametrize("kw,code", [
    (dict(transA="X"), -1), (dict(transB="?"), -2), (dict(M=-1), -3), (dict(N=-2), -4), (dict(K=-1), -5),
    (dict(lda=3), -8), (dict(transA="T", lda=1), -8), (dict(ldb=1), -10), (dict(transB="T", ldb=2), -10),
    (dict(ldc=3), -13),
    (dict(A=None), -7), (dict(A=4098), -7), (dict(B=None), -9), (dict(C=None), -12), (dict(C=16386), -12),
    (dict(C=4096 + 8), -100),                                  # C overlaps A
    # literal configs[2] reading for transA=T: lda = M+13 < K  (R3)
    (dict(transA="T", M=1531, N=997, K=2049, lda=1531 + 13, ldb=2049 + 7, ldc=1531 + 5), -8),
])
def test_argument_errors_before_any_device_work(emm, kw, code):
    assert call(emm, **kw) == code


def test_quick_returns_touch_nothing(emm):
    # M == 0 / N == 0, and (alpha == 0 or K == 0) with beta == 1: success, no launch,
    # even with NULL pointers and no device
    n0 = emm.launch_count()
    assert call(emm, M=0, A=None, B=None, C=None, ldc=1, lda=1) == 0
    assert call(emm, N=0, A=None, B=None, C=None) == 0
    assert call(emm, alpha=0.0, beta=1.0, A=None, B=None) == 0
    assert call(emm, K=0, beta=1.0, A=None, B=None, lda=4, ldb=1) == 0
    assert emm.launch_count() == n0


def test_unknown_math_mode(emm):
    L = emm.lib()
    st = L.emm_sgemm_ex(b"N", b"N", 4, 3, 2, 1.0, 4096, 4, 8192, 2, 0.0, 16384, 4, None, 7, None, 0)
    assert st == -103


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(emm):
    st = call(emm)
    assert st >= 1000, st           # a CUDA error code, never a silent CPU result
    assert "CUDA error" in emm.strerror(st)


@pytest.mark.parametrize("M", [1, 255, 256, 257, 1000, 4096, 32768, 32768 + 5])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_row_partition_tiles_exactly(emm, M, P):
    cur = 0
    sizes = []
    for r in range(P):
        r0, n = emm.row_partition(M, P, r)
        assert r0 == cur and n >= 0
        if r0 + n < M:
            assert n % 256 == 0
        cur += n
        sizes.append(n)
    assert cur == M
    tiles = [(-(-s // 256)) for s in sizes]
    assert max(tiles) - min(tiles) <= 1


def test_row_partition_c5(emm):
    for P in (1, 2, 4, 8):
        assert [emm.row_partition(32768, P, r) for r in range(P)] == \
            [(r * 32768 // P, 32768 // P) for r in range(P)]


def test_workspace_bytes(emm):
    # layout: [A region | B region | split-K slots | ctrl 1 KB | (stream-K: flags 8 KB | slots)]
    CTRL, FLAGS, SLOT = 1024, 8192, 256 * 256 * 4

    def al(b):
        return -(-b // 1024) * 1024

    def repitch(rows, cols):   # KN1X upper bound: raw copy of a stored rows x cols operand, ld rounded up to 4
        return al(cols * (-(-rows // 4) * 4) * 4)

    assert emm.workspace_bytes("N", "N", 64, 64, 64, "ffma") == 0
    # FFMA: room for the relayout copies (TN: the smaller operand transposed,
    # rows padded to 32; the other re-pitched, ld rounded up to 4)
    assert emm.workspace_bytes("T", "N", 4096, 2048, 512, "ffma") == repitch(512, 4096) + 4 * 512 * 2048
    assert emm.workspace_bytes("N", "N", 4096, 2048, 512, "ffma") == repitch(4096, 512) + repitch(512, 2048)
    # 3xTF32 (KN1X): at most a raw re-pitch of both operands
    assert emm.workspace_bytes("N", "N", 2048, 1024, 33, "3xtf32") == repitch(2048, 33) + repitch(33, 1024) + CTRL
    assert emm.workspace_bytes("T", "T", 2048, 1024, 33, "3xtf32") == repitch(33, 2048) + repitch(1024, 33) + CTRL
    # 1xTF32: re-buffered planes (1 plane of M x Kp and N x Kp floats, Kp = K rounded up to 32)
    assert emm.workspace_bytes("N", "T", 2048, 1024, 64, "1xtf32") == 4 * 64 * (2048 + 1024) + CTRL
    # latency-bound problems (2MNK <= 2^27) take the tiny FFMA kernel: no workspace
    assert emm.workspace_bytes("N", "N", 64, 64, 64, "3xtf32") == 0
    assert emm.workspace_bytes("N", "N", 333, 333, 333, "3xtf32") == 0
    # sub-wave problems add split-K slots: BJ configs[2] -> 24 tiles x 3 splits of 256 x 256 floats
    M, N, K = 1531, 997, 2049
    assert emm.workspace_bytes("N", "N", M, N, K, "3xtf32") == repitch(M, K) + repitch(K, N) + 24 * 3 * SLOT + CTRL
    # stream-K shapes add one slot per CTA pair (4096^3 3xTF32: 256 tiles = 3.46 waves)
    base = 2 * 4 * 4096 * 4096
    assert emm.workspace_bytes("N", "N", 4096, 4096, 4096, "3xtf32") == base + CTRL + FLAGS + 74 * SLOT
    assert emm.workspace_bytes("N", "N", 4096, 4096, 4096, "1xtf32") == base + CTRL
    # TF32+BF16 keeps the re-buffered planes (2 per operand)
    assert emm.workspace_bytes("N", "N", 4096, 4096, 4096, "tf32bf16") == 2 * base + CTRL + FLAGS + 74 * SLOT


def test_strerror_and_version(emm):
    assert "lda" in emm.strerror(-8)
    assert "overlap" in emm.strerror(-100)
    assert "sm_100a" in emm.version()
