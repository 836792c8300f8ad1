"""Worker: emm_sgemm_multi with P VIRTUAL ranks on one GPU
(emm_debug_comm_create_local), run as a subprocess by
tests/test_gpu_multi_local.py.

For each case the P ranks are driven through the UNMODIFIED library entry
points in one host thread (rank 0 .. P-1 one after the other; the library
enqueues the whole collective when the last rank has called, with the ranks'
signal / wait points as CUDA events — no kernel ever spins on another rank's
work on this one GPU), each with its own stream, its own row block of op(A)
(emm_row_partition), its own B buffer (B valid on `root` only; registered, so
B travels along the ring by peer copies in chunks) and its own C_full
(registered: the tensor-core epilogue stores every tile into all P copies,
other modes copy).

Checks (SURVEY.md §4 "fake multi-GPU on one device"):
* every rank's B buffer ends bit-identical to root's;
* every rank's C_local is bitwise equal to the same rows of the P = 1 call
  (same code, one rank: the per-element summation order of the tensor-core
  paths does not depend on the row partition; FFMA: integer inputs only);
* the P copies of C_full are bitwise equal to each other and to the
  assembled C_local blocks;
* the result is within the north_star tolerance of the oracle (bitwise equal
  on integer-exact inputs);
* repeated calls with a changing root (the consumed/bready flag epochs).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402

DEV = torch.device("cuda", 0)


def colmajor(rows, cols, ld=None, fill=float("nan")):
    ld = ld or max(rows, 1)
    st = torch.full((max(cols, 1) * ld,), fill, dtype=torch.float32, device=DEV)
    return torch.as_strided(st, (rows, cols), (1, ld)), st


def run_world(P, M, N, K, transB, math, kind, roots, gather, beta=0.0):
    comms = emm.local_comms(P)
    bstored = (K, N) if transB == "N" else (N, K)
    Bh = datagen.matrix(kind, datagen.TAG_B, *bstored)
    Bsrc = datagen.storage_of(Bh).to(DEV)
    Ah = datagen.matrix(kind, datagen.TAG_A, M, K)
    Cin = datagen.matrix(kind, datagen.TAG_C, M, N)
    streams = [torch.cuda.Stream(DEV) for _ in range(P)]
    ranks = []
    for r, c in enumerate(comms):
        r0, rows = emm.row_partition(M, P, r)
        if rows:
            A_loc = datagen.submatrix(kind, datagen.TAG_A, M, K, np.arange(r0, r0 + rows)).contiguous()
            A_loc = A_loc.t().contiguous().to(DEV).t()          # column-major rows x K, lda = rows
        else:
            A_loc = torch.as_strided(torch.zeros(1, device=DEV), (0, K), (1, 1))
        Bbuf = torch.zeros(bstored[0] * bstored[1], dtype=torch.float32, device=DEV)
        Bv = torch.as_strided(Bbuf, bstored, (1, bstored[0]))
        c.register_input(Bv)
        C_loc, C_st = colmajor(rows, N)
        C_full = None
        if gather:
            C_full, _ = colmajor(M, N)
            c.register_output(C_full)
        ranks.append(dict(r0=r0, rows=rows, A=A_loc, B=Bbuf, Bv=Bv, C=C_loc, C_st=C_st, C_full=C_full))
    outs = []
    for root in roots:
        for d in ranks:
            d["B"].zero_()
            if beta != 0.0:
                d["C"].copy_(torch.as_strided(datagen.storage_of(Cin), (M, N), (1, M))[d["r0"]:d["r0"] + d["rows"]].to(DEV))
        ranks[root]["B"].copy_(Bsrc)
        torch.cuda.synchronize()
        for r, (c, d) in enumerate(zip(comms, ranks)):
            emm.sgemm_multi(c, M, N, K, d["A"], d["Bv"], d["C"], 1.0, beta, transB=transB, root=root,
                            C_full=d["C_full"], math=math, stream=streams[r])
        torch.cuda.synchronize()
        for d in ranks:
            assert torch.equal(d["B"], Bsrc), f"B not forwarded intact (root {root})"
        C_all = torch.cat([d["C"].cpu() for d in ranks if d["rows"]], 0)
        if gather:
            for d in ranks:
                assert torch.equal(d["C_full"].cpu(), C_all), f"C_full copy differs (root {root})"
        outs.append(C_all)
    for c in comms:
        c.close()
    R, S, T, st = oracle.sgemm_sub("N", transB, M, N, K, 1.0, Ah, M, Bh, bstored[0], beta, Cin, M)
    assert st == 0
    tol = 5e-3 if math == "1xtf32" else 1e-5
    G = outs[0].double().numpy()
    if kind == "ints":
        assert np.array_equal(G, R), "integer-exact inputs: not bitwise equal to the oracle"
    else:
        err = np.abs(G - R)
        bound = tol * S + 1e-6 * T
        assert np.all(err <= bound), f"max err/tol {float(np.max(err / np.maximum(bound, 1e-300)))}"
    for o in outs[1:]:
        assert torch.equal(o, outs[0]), "result depends on the root"
    return outs[0]


def main():
    cases = json.loads(sys.argv[1])
    for cs in cases:
        P, M, N, K, transB, math, kind, gather = cs
        beta = 1.0 if kind == "ints" else 0.0
        ref = run_world(1, M, N, K, transB, math, kind, [0], gather, beta)
        got = run_world(P, M, N, K, transB, math, kind, [0, P - 1, P // 2], gather, beta)
        # tensor-core paths: each element's summation order does not depend on
        # the row partition -> bitwise; the FFMA mode picks its kernel by the
        # shard's size (tiny kernel tile / KN3b), so there both runs are only
        # held to the oracle bound (checked in run_world)
        if math != "ffma" or kind == "ints":
            assert torch.equal(ref, got), f"P={P} differs from P=1 (bitwise)"
        print(f"ok {cs}", flush=True)
    print("ALL OK", flush=True)


if __name__ == "__main__":
    main()
