"""emm_sgemm_multi with P virtual ranks on one B200 (SURVEY.md §4 "fake
multi-GPU on one device"; PAPER.md:181-189 is the paper's only distributed
use of the kernel).

The unmodified row-sharded path runs P ranks (emm_debug_comm_create_local)
with distinct buffers on one GPU: B forwarded along the ring by chunked
copies, the all-gather fused into the tensor-core epilogue as stores into all
P C_full buffers (peer stores), or done by 2-D copies in the FFMA path, ranks
with 0 rows, a ragged last shard, transB = 'T', and changing roots; the
cross-rank signal / wait points are CUDA events here (device flags across
real GPUs).  See tests/multi_local_worker.py for the checks.
"""
import json
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

# P, M, N, K, transB, math, data kind, gather C_full
CASES = [
    (2, 2048, 2048, 1024, "N", "3xtf32", "uniform", True),     # c5-shaped, scaled down
    (4, 2048, 2304, 768, "N", "3xtf32", "uniform", True),
    (8, 4096, 2048, 512, "N", "3xtf32", "uniform", True),
    (3, 1000, 1300, 257, "N", "3xtf32", "uniform", True),      # ragged last shard
    (4, 600, 1100, 300, "N", "3xtf32", "ints", True),          # rank 0 has 0 rows; beta = 1
    (2, 1536, 1000, 513, "T", "3xtf32", "uniform", True),      # transB = T: B whole, chunked
    (3, 1024, 2000, 256, "N", "1xtf32", "uniform", True),
    (2, 1024, 1500, 300, "N", "ffma", "uniform", True),        # copy all-gather path
    (4, 1800, 1200, 200, "N", "tf32bf16", "ints", True),
    (2, 2048, 1024, 512, "N", "3xtf32", "uniform", False),     # no gather
]


def run(cases, timeout=900):
    env = dict(os.environ)
    p = subprocess.run([sys.executable, os.path.join(HERE, "multi_local_worker.py"), json.dumps(cases)],
                       env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0 and "ALL OK" in p.stdout, (p.stdout[-3000:] + p.stderr[-3000:])


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: "P{}_{}x{}x{}_{}_{}_{}{}".format(*c[:7], "_gather" if c[7] else ""))
def test_virtual_ranks(case):
    run([list(case)])


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 8])
def test_virtual_ranks_c5_fullsize(P):
    """BASELINE configs[4] (32768^3) row-sharded over P virtual ranks in the
    bench's multi-GPU launch configuration: B intact on every rank, sampled
    shard rows vs the oracle, Freivalds over all of C."""
    p = subprocess.run([sys.executable, os.path.join(HERE, "multi_c5_worker.py"), str(P)],
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and "ALL OK" in p.stdout, (p.stdout[-3000:] + p.stderr[-3000:])
