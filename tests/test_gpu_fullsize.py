"""Parity at BASELINE.json's full c5 size (configs[4]: M = N = K = 32768, NN,
alpha = 1, beta = 0, A, B ~ U[-1,1) seed 0), in the launch configuration
bench.py times (emm_sgemm_ex, 3xTF32 and TF32+BF16, caller workspace).

The oracle cannot do all of C (7e13 flops), so:
* full rows (all 32768 columns, full K) at tile / wave / edge positions and
  a few seeded random ones, element by element against the oracle with the
  1e-5*S bound;
* full columns likewise (every row of C for a few columns);
* a Freivalds check over the WHOLE result: for a seeded x in {-1,+1}^N,
  |C x - A (B x)| <= 1e-5 * |A| (|B| 1) row by row (the tolerance summed over
  j), evaluated in FP64 on the host (numpy), independent of the CUDA path.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu

N = 32768


@pytest.fixture(scope="module")
def problem():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as emm
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    A = datagen.matrix("uniform", datagen.TAG_A, N, N, device=dev)
    B = datagen.matrix("uniform", datagen.TAG_B, N, N, device=dev)
    Ah = datagen.storage_of(A).cpu().numpy()          # column-major storages on the host
    Bh = datagen.storage_of(B).cpu().numpy()
    return emm, A, B, Ah, Bh


def rows_to_check():
    rng = np.random.default_rng(1)
    fixed = [0, 1, 127, 128, 255, 256, 2047, 2048, 16383, 16384, N - 257, N - 256, N - 1]
    return np.unique(np.r_[fixed, rng.integers(0, N, 5)])


def freivalds(Ah, Bh, Cg):
    """max over rows of |C x - A(B x)| / (1e-5 |A|(|B| 1)); all FP64 on the host."""
    rng = np.random.default_rng(2)
    x = rng.choice([-1.0, 1.0], size=N)
    A2 = Ah.reshape(N, N)      # [col][row] views of the column-major storages
    B2 = Bh.reshape(N, N)
    C2 = Cg.reshape(N, N)
    bx = np.zeros(N)
    babs = np.zeros(N)
    cx = np.zeros(N)
    step = 2048
    for c0 in range(0, N, step):   # column blocks: X[:, c0:c1] @ v[c0:c1]
        Bc = B2[c0:c0 + step].astype(np.float64)          # (cols, rows)
        bx += Bc.T @ x[c0:c0 + step]
        babs += np.abs(Bc).T @ np.ones(min(step, N - c0))
        cx += C2[c0:c0 + step].astype(np.float64).T @ x[c0:c0 + step]
    abx = np.zeros(N)
    bound = np.zeros(N)
    for c0 in range(0, N, step):
        Ac = A2[c0:c0 + step].astype(np.float64)
        abx += Ac.T @ bx[c0:c0 + step]
        bound += np.abs(Ac).T @ babs[c0:c0 + step]
    return float(np.max(np.abs(cx - abx) / (1e-5 * bound)))


@pytest.mark.parametrize("math", ["3xtf32", "tf32bf16"])
def test_c5_full_size(problem, math):
    emm, A, B, Ah, Bh = problem
    C = torch.empty(N, N, device=A.device).t()        # column-major M x N
    ws = torch.empty(emm.workspace_bytes("N", "N", N, N, N, math), dtype=torch.uint8, device=A.device)
    emm.sgemm_ex(A, B, C, 1.0, 0.0, math=math, workspace=ws)
    torch.cuda.synchronize()
    Cg = datagen.storage_of(C).cpu().numpy()
    del ws
    # sampled full rows
    rows = rows_to_check()
    A_rows = datagen.storage_of(datagen.submatrix("uniform", datagen.TAG_A, N, N, rows)).numpy()
    R, S, T, st = oracle.sgemm_sub("N", "N", len(rows), N, N, 1.0, A_rows, len(rows), Bh, N, 0.0, None,
                                   len(rows))
    assert st == 0
    G = Cg.reshape(N, N)[:, rows].T.astype(np.float64)
    r = np.max(np.abs(G - R) / (1e-5 * S))
    assert r <= 1.0, f"rows: max err/tol {r}"
    # sampled full columns (every row of C)
    cols = np.array([0, 255, 256, N - 1])
    R, S, T, st = oracle.sgemm_sub("N", "N", N, N, N, 1.0, Ah, N, Bh, N, 0.0, None, N, cols=cols)
    assert st == 0
    G = Cg.reshape(N, N)[cols].T.astype(np.float64)
    r = np.max(np.abs(G - R) / (1e-5 * S))
    assert r <= 1.0, f"cols: max err/tol {r}"
    # the whole result
    f = freivalds(Ah, Bh, Cg)
    print(f"c5 {math}: Freivalds max |Cx - A(Bx)| / bound = {f:.3g}")
    assert f <= 1.0
