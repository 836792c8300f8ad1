"""Seeded randomized parity sweep through the C ABI (complements the
structured cases): random M, N, K (log-uniform, 1..3000 / 1..5000), trans,
leading-dimension padding, alpha / beta (including 0), math mode, data
distribution and the policy switches (tiny-kernel threshold, re-buffered vs
direct operands, stream-K forced / off, skinny path off, 1xTF32 256x512 tiles
forced, the FFMA kernel without TMA, preferred clusters of 4 forced / off;
round 2: FFMA relayout / NT threshold / split-K, skinny split-K / block rows /
B' transpose, 1xTF32 on truncated operands).  Each case checks
the tolerance predicate against the oracle (every entry, or sampled rows for
large cases), that ldc padding and the guard region keep their sentinel, and
that A and B are not written.

EMM_FUZZ_CASES (default 48) sets the number of cases; EMM_FUZZ_SEED the seed;
EMM_FUZZ_MAX_MN the largest M / N (default 3000).
"""
from __future__ import annotations

import math
import os
import random

import numpy as np
import pytest

from test_gpu_parity import TOL, Case, assert_close

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("EMM_FUZZ_CASES", "48"))
MAX_MN = int(os.environ.get("EMM_FUZZ_MAX_MN", "3000"))   # larger extents: EMM_FUZZ_MAX_MN=8000
SEED = int(os.environ.get("EMM_FUZZ_SEED", "20261019"))


@pytest.fixture(scope="module")
def emm():
    from paper_1912_04379_b200 import build
    build.build()
    import paper_1912_04379_b200 as e
    import torch
    torch.cuda.set_device(0)
    return e


def _cases():
    rng = random.Random(SEED)
    out = []
    for i in range(N_CASES):
        def lu(lo, hi):
            return int(round(math.exp(rng.uniform(math.log(lo), math.log(hi)))))
        M, N, K = lu(1, MAX_MN), lu(1, MAX_MN), lu(1, 5000)
        out.append(dict(
            i=i, M=M, N=N, K=K, tA=rng.choice("NT"), tB=rng.choice("NT"),
            pad=(rng.choice([0, 0, 1, 3, 4, 7]), rng.choice([0, 0, 1, 2, 4]), rng.choice([0, 0, 1, 5])),
            alpha=rng.choice([1.0, 1.0, -0.5, 2.25, 0.0]), beta=rng.choice([0.0, 0.0, 1.0, -1.5]),
            math=rng.choice(["3xtf32", "3xtf32", "tf32bf16", "1xtf32", "ffma"]),
            kind=rng.choice(["uniform", "normal"]),
            env={"EMM_SMALL_FLOPS": rng.choice([None, "0"]), "EMM_FORCE_PACK": rng.choice([None, None, "1"]),
                 "EMM_SK": rng.choice([None, None, "0", "1"]), "EMM_NO_SKINNY": rng.choice([None, None, "1"]),
                 "EMM_WIDE": rng.choice([None, None, "1"]), "EMM_FFMA_CLASSIC": rng.choice([None, None, "1"]),
                 "EMM_PREF4": rng.choice([None, "1", "1", "0"])}))
        out[-1]["env"]["EMM_SPLIT"] = rng.choice([None, None, "pass"])   # KN1 instead of KN1X
        out[-1]["env"]["EMM_SKINNY_TC"] = rng.choice([None, None, "1"])   # KN9T at any size
        out[-1]["env"]["EMM_CSK"] = rng.choice([None, None, "1"])          # cluster split-K
        out[-1]["env"]["EMM_XS_RN"] = rng.choice([None, None, None, "1"])  # KN1X with rounded big parts
        # round-2 switches: FFMA relayout / NT threshold / split-K, skinny
        # split-K / block rows / B' transpose, 1xTF32 on truncated operands
        out[-1]["env"]["EMM_FFMA_NORELAYOUT"] = rng.choice([None, None, None, "1"])
        out[-1]["env"]["EMM_FFMA_NT_MIN"] = rng.choice([None, None, "0", "256"])
        out[-1]["env"]["EMM_FFMA_SPLITS"] = rng.choice([None, None, "1", "3"])
        out[-1]["env"]["EMM_SKINNY_SPLITS"] = rng.choice([None, None, "1", "4"])
        out[-1]["env"]["EMM_SKINNY_TPB"] = rng.choice([None, None, "224", "256"])
        out[-1]["env"]["EMM_SKINNY_BT"] = rng.choice([None, None, "0"])
        out[-1]["env"]["EMM_TMA_TRUNC"] = rng.choice([None, None, None, "1"])
    return out


@pytest.mark.parametrize("c", _cases(), ids=lambda c: f"{c['i']}-{c['M']}x{c['N']}x{c['K']}-{c['tA']}{c['tB']}-"
                                                      f"{c['math']}")
def test_fuzz(emm, monkeypatch, c):
    for k, v in c["env"].items():
        if v is None:
            monkeypatch.delenv(k, raising=False)
        else:
            monkeypatch.setenv(k, v)
    case = Case(c["tA"], c["tB"], c["M"], c["N"], c["K"], c["alpha"], c["beta"], kind=c["kind"], pad=c["pad"],
                sigma=1.0 / math.sqrt(c["K"]))
    big = c["M"] * c["N"] * c["K"] > 2e9
    rows = np.unique(np.r_[0:4, c["M"] // 2:c["M"] // 2 + 4, c["M"] - 4:c["M"]]) if big else None
    rows = rows[(rows >= 0) & (rows < c["M"])] if rows is not None else None
    R, S, T, st = case.oracle(rows=rows)
    assert st == 0
    Cg = case.run(emm, c["math"])
    case.check_untouched(Cg)
    assert_close(case, Cg, R, S, T, TOL[c["math"]], rows=rows)
