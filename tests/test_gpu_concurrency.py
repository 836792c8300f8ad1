"""Reentrancy: concurrent calls on different
streams with disjoint outputs must all complete and be correct.

The persistent GEMM's wave lockstep is a grid-wide wait; with two GEMMs in
flight neither grid may be fully resident.  The lockstep therefore gives up
after ~1 ms instead of waiting for CTAs that another kernel keeps off the
SMs.  These tests launch several multi-wave (lockstep) and stream-K GEMMs on
different streams without synchronising in between, and call the library
from several host threads at once; integer-exact inputs make every checked
entry exact (bitwise against the oracle).
"""
from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

from test_gpu_parity import Case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    torch.cuda.set_device(0)
    return e


def _launch(emm, case, stream, math):
    dA = case.flat(case.A).cuda()
    dB = case.flat(case.B).cuda()
    dC = case.Cflat.cuda()
    torch.cuda.synchronize()
    st = emm.sgemm_ptr(case.tA, case.tB, case.M, case.N, case.K, case.alpha, dA.data_ptr(), case.lda,
                       dB.data_ptr(), case.ldb, case.beta, dC.data_ptr(), case.ldc, stream.cuda_stream, math)
    assert st == 0, emm.strerror(st)
    return dA, dB, dC


def _check(case, dC):
    rows = np.unique(np.r_[0:8, case.M // 2:case.M // 2 + 8, case.M - 8:case.M])
    R, S, T, _ = case.oracle(rows=rows)
    G = case.logical(dC.cpu())[rows]
    assert np.array_equal(G, R.astype(np.float32).astype(np.float64)), f"max |diff| {np.max(np.abs(G - R))}"


@pytest.mark.parametrize("shape,math", [((8192, 4096, 512), "3xtf32"),     # 512 tiles: 6.9 waves, lockstep
                                        ((4096, 4096, 1024), "3xtf32"),    # 3.46 waves: stream-K remainder
                                        ((8192, 4096, 512), "tf32bf16"),
                                        ((8192, 4096, 512), "1xtf32"),
                                        ((8192, 4096, 2048), "1xtf32"),    # KN2w (256x512 tiles)
                                        ((8192, 4096, 4096), "3xtf32"),    # preferred clusters of 4
                                        ((4096, 2048, 512), "ffma")])      # KN3b
def test_concurrent_streams(emm, shape, math):
    M, N, K = shape
    cases = [Case("N", "T" if i % 2 else "N", M, N, K, 1.0, 1.0, kind="ints", c_kind="ints", seed=i)
             for i in range(3)]
    streams = [torch.cuda.Stream() for _ in cases]
    for rep in range(2):
        bufs = [_launch(emm, c, s, math) for c, s in zip(cases, streams)]
        torch.cuda.synchronize()
        for c, (_, _, dC) in zip(cases, bufs):
            _check(c, dC)


def test_concurrent_host_threads(emm):
    """Four host threads, each with its own stream and problem, calling the
    C ABI at the same time (ctypes releases the GIL)."""
    M, N, K = 4096, 2048, 512
    cases = [Case("N", "N", M, N, K, 1.0, 0.0, kind="ints", seed=10 + i) for i in range(4)]
    dev = [(c.flat(c.A).cuda(), c.flat(c.B).cuda(), c.Cflat.cuda()) for c in cases]
    torch.cuda.synchronize()
    errs = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            c, (dA, dB, dC) = cases[i], dev[i]
            for _ in range(3):
                st = emm.sgemm_ptr("N", "N", M, N, K, 1.0, dA.data_ptr(), c.lda, dB.data_ptr(), c.ldb, 0.0,
                                   dC.data_ptr(), c.ldc, s.cuda_stream, "3xtf32")
                if st:
                    errs.append(emm.strerror(st))
            s.synchronize()
        except Exception as e:   # surfaced below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for c, (_, _, dC) in zip(cases, dev):
        _check(c, dC)
