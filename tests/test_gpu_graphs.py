"""CUDA-graph capture of the C-ABI call (the B200 playbook's replacement for a
tracing compiler): every launch sequence the library issues — split pass +
GEMM, split-K partials + reduce, the stream-K flags and slots, the wave-
lockstep counter zeroed inside the captured work, the no-workspace call's
stream-ordered allocation — must replay correctly and give the same bits
as the eager call, replay after replay.
"""
from __future__ import annotations

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


@pytest.mark.parametrize("shape,math,with_ws", [
    ((1024, 1024, 1024), "3xtf32", True),     # direct split pass + split-K x4 + reduce
    ((4096, 4096, 1024), "3xtf32", True),     # stream-K remainder (flags + slots)
    ((8192, 4096, 512), "3xtf32", True),      # multi-wave lockstep
    ((8192, 4096, 512), "tf32bf16", True),
    ((8192, 4096, 4096), "3xtf32", True),     # preferred clusters of 4 (B multicast) + lockstep
    ((1024, 1024, 1024), "3xtf32", False),    # emm_sgemm-style: scratch from the stream-ordered pool
    ((333, 333, 333), "3xtf32", True),        # tiny kernel
    ((20000, 16, 700), "3xtf32", True),       # skinny kernel
    ((4096, 4096, 2048), "1xtf32", True),     # KN2w: 256x512 tiles
    ((2048, 1536, 512), "ffma", True),        # KN3b: TMA-fed FFMA
])
def test_graph_replay_bitwise(emm, shape, math, with_ws):
    M, N, K = shape
    case = Case("N", "N", M, N, K, 1.0, 0.5, kind="normal")
    dA = case.flat(case.A).cuda()
    dB = case.flat(case.B).cuda()
    C0 = case.Cflat.cuda()
    nbytes = emm.workspace_bytes("N", "N", M, N, K, math) if with_ws else 0
    ws = torch.empty(max(nbytes, 1) + 1024, dtype=torch.uint8, device="cuda")
    wsp = (ws.data_ptr() + 1023) // 1024 * 1024 if nbytes else None
    s = torch.cuda.Stream()

    def call(dC):
        st = emm.sgemm_ptr("N", "N", M, N, K, 1.0, dA.data_ptr(), case.lda, dB.data_ptr(), case.ldb, 0.5,
                           dC.data_ptr(), case.ldc, s.cuda_stream, math, wsp, nbytes)
        assert st == 0, emm.strerror(st)

    eager = C0.clone()
    with torch.cuda.stream(s):
        call(eager)
    s.synchronize()
    graphed = C0.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        call(graphed.clone())      # warm-up outside capture (one-time attribute / pool setup)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            call(graphed)
    for _ in range(3):
        graphed.copy_(C0)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(graphed.view(torch.int32), eager.view(torch.int32))
