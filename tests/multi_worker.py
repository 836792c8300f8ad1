"""Worker for tests/test_multi.py.  Launched once per rank with RANK,
WORLD_SIZE, MASTER_ADDR=127.0.0.1, MASTER_PORT set.

mode "gloo-dataflow" (CPU, any world size): emulates emm_sgemm_multi's data
  flow with gloo collectives and the oracle as the per-panel compute, using
  the library's own host-side plan (emm_row_partition, emm_multi_panel_cols)
  and checks the all-gathered C equals one oracle call over the whole problem.
mode "nccl" (one GPU per rank): the real C-ABI emm_sgemm_multi, checked
  against the oracle, with and without the C all-gather.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402


def gloo_dataflow(rank, world, M, N, K):
    # every rank: the bootstrap id is identical everywhere
    try:
        uid = emm.broadcast_unique_id(rank)
    except emm.EmmError:          # NCCL not loadable: still check the byte broadcast
        t = torch.tensor(list(range(128)) if rank == 0 else [0] * 128, dtype=torch.uint8)
        dist.broadcast(t, 0)
        uid = bytes(t.tolist())
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    assert all(i == ids[0] for i in ids) and len(uid) == 128

    r0, rows = emm.row_partition(M, world, rank)
    parts = [None] * world
    dist.all_gather_object(parts, (r0, rows))
    assert parts[0][0] == 0 and sum(p[1] for p in parts) == M
    assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(world - 1))

    # rank's rows of A (compact, lda = rows); B full on root, received elsewhere
    A_loc = datagen.submatrix("uniform", datagen.TAG_A, M, K, np.arange(r0, r0 + rows))
    A_flat = datagen.storage_of(A_loc).numpy() if rows else np.zeros(1, np.float32)
    B = datagen.storage_of(datagen.matrix("uniform", datagen.TAG_B, K, N)).clone() if rank == 0 \
        else torch.zeros(K * N)
    panel = emm.multi_panel_cols(N)
    C_loc = np.zeros((N, max(rows, 1)), np.float32)            # column-major rows x N
    for c0 in range(0, N, panel):
        nc = min(panel, N - c0)
        pview = B[c0 * K:(c0 + nc) * K]
        dist.broadcast(pview, 0)                                # the panel's broadcast
        if rows:
            R, _, _, st = oracle.sgemm_sub("N", "N", rows, nc, K, 1.0, A_flat, rows,
                                           pview.numpy(), K, 0.0, None, rows)
            assert st == 0
            C_loc[c0:c0 + nc, :rows] = R.T.astype(np.float32)
    # all-gather: rank-major compact blocks, then unpack into column-major M x N
    stage = torch.zeros(M * N)
    off = 0
    for r, (rr0, rrows) in enumerate(parts):
        blk = stage[off:off + rrows * N]
        if r == rank:
            blk.copy_(torch.from_numpy(C_loc[:, :rows].reshape(-1)) if rrows else blk)
        dist.broadcast(blk, r)
        off += rrows * N
    C_full = np.zeros((N, M), np.float32)
    off = 0
    for rr0, rrows in parts:
        C_full[:, rr0:rr0 + rrows] = stage[off:off + rrows * N].numpy().reshape(N, rrows)
        off += rrows * N
    A_all = datagen.storage_of(datagen.matrix("uniform", datagen.TAG_A, M, K)).numpy()
    R, _, _, _ = oracle.sgemm_sub("N", "N", M, N, K, 1.0, A_all, M,
                                  datagen.storage_of(datagen.matrix("uniform", datagen.TAG_B, K, N)).numpy(), K,
                                  0.0, None, M)
    assert np.array_equal(C_full.T, R.astype(np.float32)), "sharded data flow != single oracle"


def nccl_multi(rank, world, M, N, K, transB, math):
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    comm = emm.Comm(rank, world)
    r0, rows = emm.row_partition(M, world, rank)
    A_loc = datagen.submatrix("uniform", datagen.TAG_A, M, K, np.arange(r0, r0 + rows), device=dev)
    bstored = (K, N) if transB == "N" else (N, K)
    Bh = datagen.matrix("uniform", datagen.TAG_B, *bstored)
    B = datagen.storage_of(Bh).to(dev) if rank == 0 else torch.zeros(bstored[0] * bstored[1], device=dev)
    Bv = torch.as_strided(B, bstored, (1, bstored[0]))
    C_loc = torch.full((N, max(rows, 1)), float("nan"), device=dev).t()[:rows, :]
    C_full = torch.full((N, M), float("nan"), device=dev).t()
    emm.sgemm_multi(comm, M, N, K, A_loc, Bv, C_loc, 1.0, 0.0, transB=transB, C_full=C_full, math=math)
    torch.cuda.synchronize()
    A_all = datagen.matrix("uniform", datagen.TAG_A, M, K)
    R, S, T, _ = oracle.sgemm_sub("N", transB, M, N, K, 1.0, A_all, M, Bh, bstored[0], 0.0, None, M)
    tol = 5e-3 if math == "1xtf32" else 1e-5
    G = C_full.cpu().double().numpy()
    assert np.all(np.abs(G - R) <= tol * S), "C_full out of tolerance"
    assert torch.equal(B.cpu(), datagen.storage_of(Bh)), "B not broadcast intact"
    if rows:
        assert np.array_equal(C_loc.cpu().double().numpy(), G[r0:r0 + rows]), "C_local != C_full rows"
    # fused all-gather: register a second full output; the GEMM epilogue
    # stores straight into every rank's copy (peer pointers); same bits
    C_f = torch.full((N, M), float("nan"), device=dev).t()
    comm.register_output(C_f)
    C_loc2 = torch.full((N, max(rows, 1)), float("nan"), device=dev).t()[:rows, :]
    emm.sgemm_multi(comm, M, N, K, A_loc, Bv, C_loc2, 1.0, 0.0, transB=transB, C_full=C_f, math=math)
    torch.cuda.synchronize()
    assert torch.equal(C_f.cpu(), C_full.cpu()), "fused all-gather differs from the NCCL all-gather"
    comm.unregister_output()
    comm.close()


def main():
    mode = sys.argv[1]
    M, N, K = (int(x) for x in sys.argv[2:5])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if mode == "gloo-dataflow":
        dist.init_process_group("gloo", rank=rank, world_size=world)
        gloo_dataflow(rank, world, M, N, K)
    else:
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
        for transB in ("N", "T"):
            for math in ("3xtf32", "1xtf32", "ffma"):
                nccl_multi(rank, world, M, N, K, transB, math)
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank} ok", flush=True)


if __name__ == "__main__":
    main()
