"""Host replay of the tcgen05 GEMM's persistent schedule (no GPU needed).

emm_debug_schedule runs the SAME TcSched code the kernel runs (a
__host__ __device__ struct, tc_common.cuh) for every cluster of a launch and
returns its work items.  Checked here for many shapes:
* every (tile, K-stage) of the problem is computed exactly once;
* split-K units tile K per split; stream-K pieces of one tile are contiguous
  in ascending k across consecutive clusters, exactly one of them (k = 0) is
  the owner, which is its cluster's LAST item and names the last publishing
  cluster correctly; a cluster publishes at most one piece (its first
  stream-K item), so one partial slot per cluster suffices;
* stream-K is planned only where SURVEY §8(f)-1 wants it (a partial last
  wave above half a wave), split-K only for sub-half-wave problems.
"""
import ctypes
import random

import numpy as np
import pytest

import paper_1912_04379_b200 as emm

TW_FULL, TW_SPLITK, TW_PUB, TW_OWN = 0, 1, 2, 3
PAIRS = 74   # 148 SMs (host-side default without a device)


def schedule(M, N, K, sk=1, terms=3):
    L = emm.lib()
    L.emm_debug_schedule.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    L.emm_debug_schedule.restype = ctypes.c_int
    cap = 1 << 16
    out = np.zeros(7 * cap, dtype=np.int32)
    n = L.emm_debug_schedule(M, N, K, sk, terms, out.ctypes.data, cap)
    assert n >= 0
    return out[: 7 * n].reshape(n, 7)


def check(M, N, K, sk=1, terms=3):
    items = schedule(M, N, K, sk, terms)
    tm, tn = -(-M // 256), -(-N // 256)
    nkb = -(-K // 32)
    cover = {}
    kinds = set(items[:, 5].tolist())
    for c, m0, n0, kb0, kb1, kind, last in items.tolist():
        assert 0 <= kb0 < kb1 <= nkb and m0 % 256 == 0 and n0 % 256 == 0 and m0 < tm * 256 and n0 < tn * 256
        cover.setdefault((m0, n0), []).append((kb0, kb1, c, kind, last))
    assert len(cover) == tm * tn, "a tile is missing"
    for (m0, n0), pieces in cover.items():
        pieces.sort()
        assert pieces[0][0] == 0 and pieces[-1][1] == nkb
        for p, q in zip(pieces, pieces[1:]):
            assert p[1] == q[0], f"tile {(m0, n0)}: K gap/overlap {p} {q}"
        ks = {p[3] for p in pieces}
        if ks <= {TW_FULL}:
            assert len(pieces) == 1
        elif TW_SPLITK in ks:
            assert ks == {TW_SPLITK}
        else:
            own = [p for p in pieces if p[3] == TW_OWN]
            pub = [p for p in pieces if p[3] == TW_PUB]
            assert len(own) == 1 and own[0][0] == 0 and len(pub) == len(pieces) - 1
            oc = own[0][2]
            assert [p[2] for p in pub] == list(range(oc + 1, oc + 1 + len(pub))), "pieces not on consecutive clusters"
            assert own[0][4] == oc + len(pub)
    # per cluster: at most one PUB, it is the first stream-K item; OWN is the last item
    by_c = {}
    for row in items.tolist():
        by_c.setdefault(row[0], []).append(row)
    for c, rows in by_c.items():
        pubs = [i for i, r in enumerate(rows) if r[5] == TW_PUB]
        owns = [i for i, r in enumerate(rows) if r[5] == TW_OWN]
        assert len(pubs) <= 1 and len(owns) <= 1
        if owns:
            assert owns[0] == len(rows) - 1
        if pubs:
            assert all(r[5] == TW_FULL and r[3] == 0 and r[4] == nkb for r in rows[:pubs[0]])
    return kinds, len(by_c)


@pytest.mark.parametrize("M,N,K", [(2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192), (1536, 1792, 2049),
                                   (2560, 2560, 600), (4096, 4096, 520), (65536, 1024, 4096), (65536, 4096, 1024),
                                   (32768, 32768, 32768), (1531, 997, 2049), (1024, 1024, 1024), (333, 333, 333)])
@pytest.mark.parametrize("sk", [0, 1, 2])
def test_config_shapes(monkeypatch, M, N, K, sk):
    # sk=2: EMM_SK=1 forces stream-K wherever it is legal (the GPU tests'
    # stream-K shapes run that way)
    if sk == 2:
        monkeypatch.setenv("EMM_SK", "1")
    kinds, nclus = check(M, N, K, sk=min(sk, 1))
    tiles = -(-M // 256) * -(-N // 256)
    if tiles * 2 <= PAIRS:
        assert TW_PUB not in kinds and TW_OWN not in kinds


@pytest.mark.parametrize("force", ["0", "1"])
def test_random_shapes(monkeypatch, force):
    monkeypatch.setenv("EMM_SK", force)
    if force == "0":
        monkeypatch.delenv("EMM_SK")
    rng = random.Random(0)
    for _ in range(300):
        M, N = rng.randint(17, 12000), rng.randint(17, 12000)
        K = rng.choice([1, 7, 32, 33, 255, 256, 257, 1000, 2049, 4096])
        check(M, N, K)


def test_stream_k_policy(monkeypatch):
    monkeypatch.delenv("EMM_SK", raising=False)
    # 4096^3 3xTF32: 256 tiles = 3.46 waves -> 3 data-parallel waves + stream-K remainder
    kinds, nclus = check(4096, 4096, 4096)
    assert TW_OWN in kinds and TW_PUB in kinds and nclus == PAIRS
    items = schedule(4096, 4096, 4096)
    assert sum(1 for r in items if r[5] == TW_FULL and r[3] == 0 and r[4] == 128) >= 3 * PAIRS
    # ... but not for 1xTF32 (fill-bandwidth-bound), 8192^3 (13.8 waves: < 3% to gain), 2048^3 (no full wave)
    assert check(4096, 4096, 4096, terms=1)[0] == {TW_FULL}
    assert check(8192, 8192, 8192)[0] == {TW_FULL}
    assert check(2048, 2048, 2048)[0] == {TW_FULL}
    # forced: legal wherever a partial wave is above half a wave
    monkeypatch.setenv("EMM_SK", "1")
    kinds, _ = check(2048, 2048, 2048)
    assert TW_OWN in kinds and TW_PUB in kinds
    # exact waves -> never stream-K; sub-half-wave -> split-K
    assert check(256 * 74, 512, 1024)[0] == {TW_FULL}
    assert check(1024, 1024, 1024)[0] == {TW_SPLITK}


# ---- preferred clusters of 4 (B multicast between the two pairs of a cluster)
def pair_schedule(M, N, K):
    L = emm.lib()
    L.emm_debug_pair_schedule.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p, ctypes.c_int]
    L.emm_debug_pair_schedule.restype = ctypes.c_int
    cap = 1 << 17
    out = np.zeros(8 * cap, dtype=np.int32)
    n = L.emm_debug_pair_schedule(M, N, K, out.ctypes.data, cap)
    assert n >= 0
    return out[: 8 * n].reshape(n, 8)


def check_pairs(M, N, K):
    """Both pairs of a 4-cluster run the same number of items with equal K
    ranges (each stage slot is released by both pairs' MMAs); a dummy item is
    the partner's item; a multicast item's partner holds the vertically
    adjacent tile of the same column (same B tile); the non-dummy items cover
    every tile exactly once."""
    it = pair_schedule(M, N, K)
    tm, tn = -(-M // 256), -(-N // 256)
    by = {}
    for c, i, m0, n0, kb0, kb1, dummy, mc in it.tolist():
        by.setdefault(c, []).append((m0, n0, kb0, kb1, dummy, mc))
    cover = {}
    for c, lst in by.items():
        for m0, n0, kb0, kb1, dummy, mc in lst:
            if not dummy:
                cover[(m0, n0)] = cover.get((m0, n0), 0) + 1
        p = c ^ 1
        if p not in by:
            assert not any(x[5] for x in lst)
            continue
        other = by[p]
        assert len(other) == len(lst), f"pairs {c},{p}: item counts differ"
        for a, b in zip(lst, other):
            assert (a[2], a[3]) == (b[2], b[3]), "K ranges differ"
            assert a[5] == b[5], "multicast decision not symmetric"
            if a[4]:
                assert not b[4] and (a[0], a[1]) == (b[0], b[1]), "dummy is not the partner's item"
            if a[5] and not a[4] and not b[4]:
                assert a[1] == b[1] and abs(a[0] - b[0]) == 256, "multicast partner not the adjacent tile"
    assert len(cover) == tm * tn and all(v == 1 for v in cover.values())
    return it


@pytest.mark.parametrize("shape", [(32768, 32768, 32768), (8192, 8192, 8192), (65536, 4096, 1024), (65536, 1024, 4096),
                                   (4096, 4096, 4096), (3000, 2000, 700), (2816, 3072, 2049), (1800, 5000, 300),
                                   (256, 65536, 512), (12345, 6789, 1000)])
def test_pair_schedule(shape):
    it = check_pairs(*shape)
    assert len(it)


def test_pair_schedule_random():
    rng = random.Random(7)
    for _ in range(300):
        M, N = rng.randint(1, 40000), rng.randint(1, 40000)
        if (-(-M // 256)) * (-(-N // 256)) > 200000:
            continue
        check_pairs(M, N, rng.randint(1, 5000))
