#!/usr/bin/env python
"""Tensor-pipe ceiling on this GPU (emm_debug_mma_probe): the GEMM kernel's
MMA stream with operands resident in SMEM, for each split.  Prints burst
(one ~5 ms launch after warm-up) and sustained (back-to-back launches for
--seconds, power-capped) rates as the 2MNK TFLOP/s a GEMM would report, with
the SM clock sampled by nvidia-smi during the sustained run.

    python tools/mma_probe.py [--seconds 4]
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1912_04379_b200 as emm  # noqa: E402


def clocks(stop, out):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "200"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        ln = p.stdout.readline()
        if ln:
            out.append(ln.strip())
    p.terminate()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    L = emm.lib()
    L.emm_debug_mma_probe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)]
    L.emm_debug_mma_probe.restype = ctypes.c_int
    s = torch.cuda.current_stream().cuda_stream
    for terms, name in ((3, "3xtf32"), (2, "tf32bf16"), (1, "1xtf32")):
        ms, fl = ctypes.c_float(), ctypes.c_double()
        stages = {3: 6000, 2: 9000, 1: 18000}[terms]     # ~5 ms launches
        for _ in range(3):
            st = L.emm_debug_mma_probe(terms, stages, s, ctypes.byref(ms), ctypes.byref(fl))
            assert st == 0, emm.strerror(st)
        burst = fl.value / (ms.value * 1e-3) / 1e12
        stop, samp = threading.Event(), []
        th = threading.Thread(target=clocks, args=(stop, samp))
        th.start()
        t_end = time.time() + a.seconds
        rates = []
        while time.time() < t_end:
            st = L.emm_debug_mma_probe(terms, stages, s, ctypes.byref(ms), ctypes.byref(fl))
            assert st == 0
            rates.append(fl.value / (ms.value * 1e-3) / 1e12)
        stop.set()
        th.join()
        sm = [float(x.split(",")[0]) for x in samp if x and x.split(",")[0].strip().replace('.', '').isdigit()]
        pw = [float(x.split(",")[1]) for x in samp if x.count(",") == 1]
        print(json.dumps({"split": name, "burst_tflops": burst, "sustained_tflops": statistics.median(rates[len(rates) // 2:]),
                          "tensor_tflops_sustained": statistics.median(rates[len(rates) // 2:]) * terms if terms != 2 else None,
                          "sm_mhz_median": statistics.median(sm) if sm else None,
                          "power_w_median": statistics.median(pw) if pw else None, "launches": len(rates)}), flush=True)


if __name__ == "__main__":
    main()
