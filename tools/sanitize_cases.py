"""Small calls through every kernel family, for compute-sanitizer runs:
tensor-core (direct + re-buffered, all trans, split-K), FFMA, skinny (TMA and
LDG), alpha=0 scaling, host-buffer entry."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402

os.environ["EMM_SMALL_FLOPS"] = "0"


def run(tA, tB, M, N, K, math, alpha=1.0, beta=0.5, pad=(0, 0, 0)):
    ar, ac = (M, K) if tA == "N" else (K, M)
    br, bc = (K, N) if tB == "N" else (N, K)
    A = datagen.storage_of(datagen.matrix("uniform", 1, ar, ac, ar + pad[0])).cuda()
    B = datagen.storage_of(datagen.matrix("uniform", 2, br, bc, br + pad[1])).cuda()
    C = datagen.storage_of(datagen.matrix("uniform", 3, M, N, M + pad[2])).cuda()
    st = emm.sgemm_ptr(tA, tB, M, N, K, alpha, A.data_ptr(), ar + pad[0], B.data_ptr(), br + pad[1], beta,
                       C.data_ptr(), M + pad[2], torch.cuda.current_stream().cuda_stream, math)
    torch.cuda.synchronize()
    assert st == 0, emm.strerror(st)


for tA in "NT":
    for tB in "NT":
        for math in ("3xtf32", "tf32bf16", "1xtf32", "ffma"):
            run(tA, tB, 300, 260, 100, math)                  # direct, split-K
            run(tA, tB, 300, 260, 100, math, pad=(1, 3, 2))   # re-buffered (TMA-illegal ld)
        run(tA, tB, 5000, 9, 300, "3xtf32")                   # skinny TMA
        run(tA, tB, 7, 3000, 301, "3xtf32", pad=(1, 1, 1))    # skinny LDG, role swap
run("N", "N", 600, 600, 2000, "3xtf32")
run("N", "N", 100, 100, 50, "3xtf32", alpha=0.0, beta=2.0)
print("sanitize cases done")
