"""Worker: BASELINE configs[4] at full size (32768^3 NN, 3xTF32, U[-1,1) seed 0)
row-sharded over P VIRTUAL ranks on one GPU through the unmodified
emm_sgemm_multi (emm_debug_comm_create_local, registered B: the ring of chunked
peer copies, 4 column panels, KN1 panel GEMMs) — the bench's multi-GPU launch
configuration with P ranks on one device.  Run by tests/test_gpu_multi_local.py.

Checks: every rank's B buffer ends bit-identical to root's; the first and last
row of every rank's shard plus rows inside it against the oracle (the north_star
bound 1e-5*S); a Freivalds check of the whole C (C x = A (B x) in float64 for a
random +-1 vector x, tolerance from |A| (|B| 1)).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402


def main():
    P = int(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
    dev = torch.device("cuda", 0)
    comms = emm.local_comms(P)
    streams = [torch.cuda.Stream(dev) for _ in range(P)]
    Bsrc = datagen.matrix("uniform", datagen.TAG_B, n, n, device=dev)
    A = datagen.matrix("uniform", datagen.TAG_A, n, n, device=dev)
    ranks = []
    for r, c in enumerate(comms):
        r0, rows = emm.row_partition(n, P, r)
        Bbuf = Bsrc.clone() if r == 0 else torch.zeros_like(Bsrc)
        c.register_input(Bbuf)
        A_loc = A[r0:r0 + rows]                      # a row block of A: lda = n (column-major view)
        C = torch.empty((n, rows), device=dev).t()
        ranks.append((r0, rows, A_loc, Bbuf, C))
    torch.cuda.synchronize()
    for r, c in enumerate(comms):
        r0, rows, A_loc, Bbuf, C = ranks[r]
        emm.sgemm_multi(c, n, n, n, A_loc, Bbuf, C, 1.0, 0.0, stream=streams[r])
    torch.cuda.synchronize()
    for r0, rows, A_loc, Bbuf, C in ranks:
        assert torch.equal(Bbuf, Bsrc), "B not forwarded intact"
    # sampled rows vs the oracle
    rows_chk = sorted({x for r0, rows, *_ in ranks for x in (r0, r0 + rows - 1, r0 + rows // 2)})
    Ah = datagen.storage_of(datagen.submatrix("uniform", datagen.TAG_A, n, n, np.array(rows_chk))).numpy()
    Bh = datagen.storage_of(Bsrc).cpu().numpy()
    R, S, T, st = oracle.sgemm_sub("N", "N", len(rows_chk), n, n, 1.0, Ah, len(rows_chk), Bh, n, 0.0, None,
                                   len(rows_chk))
    assert st == 0
    G = []
    for x in rows_chk:
        for r0, rows, A_loc, Bbuf, C in ranks:
            if r0 <= x < r0 + rows:
                G.append(C[x - r0].double().cpu().numpy())
    G = np.stack(G)
    err = np.abs(G - R)
    ratio = float(np.max(err / (1e-5 * S)))
    assert ratio <= 1.0, f"max err/tol {ratio}"
    # Freivalds over all of C
    g = torch.Generator(device="cpu").manual_seed(1)
    xv = (torch.randint(0, 2, (n,), generator=g) * 2 - 1).double().to(dev)
    Bx = Bsrc.double() @ xv
    absBone = Bsrc.double().abs() @ torch.ones(n, dtype=torch.float64, device=dev)
    worst = 0.0
    for r0, rows, A_loc, Bbuf, C in ranks:
        lhs = C.double() @ xv
        rhs = A_loc.double() @ Bx
        tol = 1e-5 * (A_loc.double().abs() @ absBone)
        worst = max(worst, float(((lhs - rhs).abs() / tol).max()))
    assert worst <= 1.0, f"Freivalds err/tol {worst}"
    for c in comms:
        c.close()
    print(f"ALL OK P={P} n={n} rows_checked={len(rows_chk)} max_err/tol={ratio:.3e} freivalds={worst:.3e}", flush=True)


if __name__ == "__main__":
    main()
