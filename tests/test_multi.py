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
