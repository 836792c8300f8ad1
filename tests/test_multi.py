"""Multi-process coverage of the row-sharded path (emm_sgemm_multi).

* CPU, gloo, world_size 2 and 3: bootstrap id broadcast, row partition
  consistency, and the full sharded data flow (panel broadcasts, per-panel
  compute, rank-major all-gather + unpack) against one oracle call.
* GPU (-m gpu): the real C-ABI emm_sgemm_multi over NCCL with a 1-rank
  communicator (the box has one GPU; ranks sharing a GPU are not run).
"""
import os
import socket
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(world, args, timeout=600):
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "multi_worker.py"), *args], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append((p.returncode, out))
    for rc, out in outs:
        assert rc == 0, out[-3000:]
    return outs


@pytest.mark.parametrize("world,shape", [(2, (700, 2500, 96)), (3, (1100, 1300, 33))])
def test_gloo_sharded_dataflow(world, shape):
    launch(world, ["gloo-dataflow", *map(str, shape)])


@pytest.mark.gpu
def test_nccl_multi_one_rank():
    launch(1, ["nccl", "1000", "2300", "300"])


@pytest.mark.parametrize("N,K,tB", [(32768, 32768, "N"), (32768, 32768, "T"), (2500, 96, "N"), (997, 2049, "T"),
                                    (1, 1, "N"), (4096, 1 << 22, "N"), (1 << 20, 4096, "N"), (300000, 4096, "T")])
def test_ring_chunk_plan(N, K, tB):
    """Host replay of emm_sgemm_multi's B chunk plan (copy-engine ring, no GPU):
    the chunks tile B's bytes exactly in order, transB='N' chunks are whole
    columns and break at every panel boundary (emm_multi_panel_cols), chunks
    stay <= 64 MB unless that would need more than the 1024 flag words."""
    import ctypes
    import paper_1912_04379_b200 as emm
    L = emm.lib()
    L.emm_debug_ring_chunks.restype = ctypes.c_int
    L.emm_debug_ring_chunks.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_char, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_int]
    off = (ctypes.c_int64 * 2048)()
    pc = (ctypes.c_int64 * 64)()
    n = L.emm_debug_ring_chunks(N, K, tB.encode(), off, 2048, pc, 64)
    assert 1 <= n <= 1024
    o = list(off)[: n + 1]
    total = N * K * 4
    assert o[0] == 0 and o[-1] == total and all(b > a for a, b in zip(o, o[1:]))
    sizes = [b - a for a, b in zip(o, o[1:])]
    if tB == "N":
        panel = emm.multi_panel_cols(N)
        npanel = -(-N // panel)
        p = list(pc)[: npanel + 1]
        assert p[0] == 0 and p[-1] == n and all(b > a for a, b in zip(p, p[1:]))
        assert all(x % (K * 4) == 0 for x in o)                       # whole columns
        for k in range(npanel):                                      # a chunk boundary at every panel start
            assert o[p[k]] == min(N, k * panel) * K * 4
        if K * 4 <= 64 << 20 and total // (64 << 20) < 1000:
            assert max(sizes) <= 64 << 20
    else:
        assert list(pc)[:2] == [0, n]
        if total // (64 << 20) < 1000:
            assert max(sizes) <= 64 << 20
