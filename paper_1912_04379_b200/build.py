"""In-tree build of the C-ABI library ``libemm.so`` (sm_100a only).

    python -m paper_1912_04379_b200.build          # or __graft_entry__.build()

nvcc cross-compiles for sm_100a without a GPU.  The .so stays in the package
directory so that gpurun snapshots carry it to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# EMM_TIMELINE=1: debug build with per-CTA %globaltimer stamps (tools/timeline.py)
TIMELINE = os.environ.get("EMM_TIMELINE") == "1"
# EMM_VARIANT=<tag> with EMM_VARIANT_FLAGS="-DX=1 ...": an A/B build of the
# same sources into build_<tag>/libemm_<tag>.so (loaded with EMM_LIB)
VARIANT = os.environ.get("EMM_VARIANT", "")
VARIANT_FLAGS = os.environ.get("EMM_VARIANT_FLAGS", "").split() if VARIANT else []
_TAG = "tl" if TIMELINE else VARIANT
OBJ = os.path.join(PKG, f"build_{_TAG}" if _TAG else "build")
LIB = os.path.join(PKG, f"libemm_{_TAG}.so" if _TAG else "libemm.so")
SOURCES = ["api.cu", "k_tc.cu", "k_tc_t1.cu", "k_tc_t2.cu", "k_tc_t3.cu", "k_tcl.cu", "k_tcx.cu", "k_tc1w.cu", "k_ffma.cu", "k_ffma_tma.cu", "k_skinny.cu", "k_skinny_tc.cu", "k_tiny.cu", "k_misc.cu", "multi.cu", "k_probe.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def nccl_include() -> str:
    sp = sysconfig.get_paths()["purelib"]
    cand = os.path.join(sp, "nvidia", "nccl", "include")
    return cand if os.path.exists(os.path.join(cand, "nccl.h")) else "/usr/include"


def flags() -> list[str]:
    return ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
            "-I", os.path.join(ROOT, "include"), "-I", nccl_include(), "--expt-relaxed-constexpr",
            *(["-DEMM_TIMELINE"] if TIMELINE else []), *VARIANT_FLAGS]


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "emm.h"))
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s.replace(".cu", ".o"))
        if force or _stale(obj, [src, *headers]):
            jobs.append((src, obj))

    def run(job):
        src, obj = job
        cmd = [nvcc(), *flags(), "-c", src, "-o", obj]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{p.stdout}\n{p.stderr}")
        log = os.path.join(OBJ, os.path.basename(obj) + ".ptxas.txt")
        with open(log, "w") as f:
            f.write(p.stderr)
        if verbose:
            sys.stderr.write(p.stderr)
        return obj

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-ldl", "-lpthread"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{p.stdout}\n{p.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
