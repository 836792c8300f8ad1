#!/usr/bin/env python
"""GPU check (not a test): stream-K really runs under its cooperative launch —
EMM_SK=1 and EMM_SK=0 give different bits at 4096^3 (different, equally valid
summation orders, R16); identical bits would mean the cooperative
launch was refused and the data-parallel schedule ran instead."""
import os, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1912_04379_b200 as emm
import datagen
n = 4096
A = datagen.matrix("uniform", 1, n, n, device="cuda"); B = datagen.matrix("uniform", 2, n, n, device="cuda")
out = {}
for split in ("xform", "pass"):
    for sk in ("0", "1"):
        os.environ["EMM_SK"] = sk; os.environ["EMM_SPLIT"] = split
        C = torch.zeros(n, n, device="cuda").t()
        emm.sgemm(A, B, C); torch.cuda.synchronize()
        out[(split, sk)] = C.clone()
for split in ("xform", "pass"):
    d = (out[(split, "0")] != out[(split, "1")]).sum().item()
    print(split, "elements differing SK=1 vs SK=0:", d)
