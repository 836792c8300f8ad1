"""Warp-state (stall reason) summary of ncu reports: average cycles per
issued instruction spent in each state, plus issue / pipe utilisation.
Usage (on the GPU box): python tools/ncu_stalls.py gpurun_out/x.ncu-rep ..."""
import csv
import io
import subprocess
import sys

KEYS = ("smsp__average_warp_latency_issue_stalled", "smsp__average_warps_issue_stalled",
        "smsp__inst_executed_pipe", "sm__inst_executed_pipe", "smsp__issue_active", "sm__pipe_fma",
        "sm__pipe_fp", "smsp__warps_active", "sm__cycles_elapsed.avg.per_second", "gpu__time_duration.sum",
        "smsp__thread_inst_executed_per_inst", "sm__warps_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared",
        "smsp__inst_executed.sum", "sm__pipe_shared")


def main(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(p, "no data")
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            print(f"== {p}: {r[hdr.index('Kernel Name')][:80]}")
            vals = []
            for i, h in enumerate(hdr):
                if any(h.startswith(k) for k in KEYS):
                    try:
                        v = float(r[i].replace(",", ""))
                    except ValueError:
                        continue
                    vals.append((h, v, units[i]))
            for h, v, u in vals:
                if "stalled" in h and "ratio" in h and v < 0.05:
                    continue
                print(f"  {h:90s} {v:12.4g} {u}")


if __name__ == "__main__":
    main(sys.argv[1:])
