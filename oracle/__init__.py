"""ctypes binding of the parity oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package ``paper_1912_04379_b200``.  It shares no code with the CUDA path.

Parity pins (tests/test_oracle.py): brute force with exact rationals on tiny
sizes, the (AB)^T = B^T A^T invariant, closed forms (identity, all-ones,
alpha = 0, beta = 0 with NaN C, K = 0, K = 1), the worked 2x2 example
(tests/golden/), a correctly-rounded fsum bound and float64 numpy matmul; the
drop-in oracle_sgemm against exact float64 results rounded to float32 with
ldc-padding sentinels.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc; no shared code)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, f32, vp, ch = ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_char
        L.oracle_check_args.restype = ctypes.c_int
        L.oracle_check_args.argtypes = [ch, ch, i64, i64, i64, i64, i64, i64]
        L.oracle_sgemm_sub.restype = ctypes.c_int
        L.oracle_sgemm_sub.argtypes = [ch, ch, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64,
                                       i64, vp, i64, vp, vp, vp, vp, i64, ctypes.c_int]
        L.oracle_sgemm.restype = ctypes.c_int
        L.oracle_sgemm.argtypes = [ch, ch, i64, i64, i64, f32, vp, i64, vp, i64, f32, vp, i64,
                                   ctypes.c_int]
        _lib = L
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _ptr(a):
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)


def _flat(x):
    """Accept a numpy array (flat storage) or a torch tensor view from datagen
    (returns the full column-major storage as float32 numpy)."""
    if x is None:
        return None
    if hasattr(x, "detach"):  # torch tensor view (rows, cols) stride (1, ld)
        import torch
        t = x.detach()
        if t.device.type != "cpu":
            t = t.cpu()
        n = 0 if t.numel() == 0 else (t.shape[1] - 1) * t.stride(1) + t.shape[0]
        flat = torch.as_strided(t, (n,), (1,), t.storage_offset()) if n else torch.zeros(1)
        return np.ascontiguousarray(flat.numpy(), dtype=np.float32)
    return np.ascontiguousarray(x, dtype=np.float32).reshape(-1)


def check_args(transA, transB, M, N, K, lda, ldb, ldc) -> int:
    return lib().oracle_check_args(transA.encode(), transB.encode(), M, N, K, lda, ldb, ldc)


def sgemm_sub(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
              rows=None, cols=None, nthreads=None):
    """Return (R, S, T, status): float64 arrays of shape (len(rows), len(cols))
    holding alpha*op(A)op(B)+beta*C (unrounded), |alpha|*sum|products| and
    |beta*C| on the selected entries.  A, B, C are flat column-major float32
    storages (numpy) or datagen matrix views."""
    Af, Bf, Cf = _flat(A), _flat(B), _flat(C)
    rows_a = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    cols_a = None if cols is None else np.ascontiguousarray(cols, dtype=np.int64)
    nr = M if rows_a is None else len(rows_a)
    nc = N if cols_a is None else len(cols_a)
    R = np.zeros((max(nc, 0), max(nr, 1)), dtype=np.float64)  # column-major nr x nc
    S = np.zeros_like(R)
    T = np.zeros_like(R)
    st = lib().oracle_sgemm_sub(transA.encode(), transB.encode(), M, N, K, alpha,
                                _ptr(Af), lda, _ptr(Bf), ldb, beta, _ptr(Cf), ldc,
                                nr, _ptr(rows_a), nc, _ptr(cols_a),
                                _ptr(R), _ptr(S), _ptr(T), max(nr, 1),
                                nthreads or default_threads())
    return R[:, :nr].T.copy(), S[:, :nr].T.copy(), T[:, :nr].T.copy(), st


def sgemm(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, nthreads=None):
    """Drop-in oracle: C (flat float32 numpy, modified in place) <- (float)R."""
    Af, Bf = _flat(A), _flat(B)
    if not (isinstance(C, np.ndarray) and C.dtype == np.float32 and C.flags.c_contiguous):
        raise TypeError("C must be a contiguous float32 numpy array")
    return lib().oracle_sgemm(transA.encode(), transB.encode(), M, N, K, alpha,
                              _ptr(Af), lda, _ptr(Bf), ldb, beta, _ptr(C), ldc,
                              nthreads or default_threads())
