#!/usr/bin/env python
"""Summarise gpurun_out/ncu_cfg_*.ncu-rep (tools/ncu_configs.sh) into one
table: duration, SM clock, tensor / FMA pipe activity, DRAM and L2 traffic."""
import csv
import glob
import io
import os
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "time",
    "sm__cycles_elapsed.avg.per_second": "clock",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2%",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_lsu%",
    "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed": "smem_rd%",
    "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed": "smem_wr%",
    "launch__grid_size": "grid",
}


def main(pattern="gpurun_out/ncu_cfg_*.ncu-rep"):
    print("| config / path | kernel | " + " | ".join(WANT.values()) + " |")
    print("|---|---|" + "---|" * len(WANT))
    for rep in sorted(glob.glob(pattern)):
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            continue
        hdr, units, vals = rows[0], rows[1], rows[2]
        col = dict(zip(hdr, zip(vals, units)))
        kern = col.get("Kernel Name", ("?", ""))[0].split("(")[0].replace("void ", "")
        cells = []
        for k in WANT:
            v, u = col.get(k, ("", ""))
            cells.append(f"{v} {u}".strip())
        name = os.path.basename(rep).replace("ncu_cfg_", "").replace(".ncu-rep", "")
        print(f"| {name} | {kern} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(*sys.argv[1:])
