#!/usr/bin/env python
"""Per-config measurements for BASELINE.md §5 (not the driver's bench line).

For every BASELINE.json config and math path: median and min device time of
single emm_sgemm_ex calls (CUDA events on the launching stream, L2 flushed
before each timed call by writing a 2x L2-sized buffer),
GFLOP/s = 2MNK/t, % of the path's roofline, and GB/s of compulsory traffic
4(MK + KN + MN [+ MN if beta != 0]) for the latency/HBM-side shapes.

    python bench_sweep.py [--reps 20] [--out profiles/r01_sweep.jsonl]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1912_04379_b200 as emm  # noqa: E402


def peaks():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        mp = json.load(f)
    tf32 = mp["bf16_tflops"] * 1.1 / 2.25
    return {"3xtf32": tf32 / 3, "tf32bf16": tf32 / 2, "1xtf32": tf32, "ffma": 148 * 256 * 1.965e9 / 1e12}


def configs():
    out = [("c1", "N", "N", 64, 64, 64, 1.0, 0.0, (0, 0, 0), "uniform")]
    for n in (100, 333, 512, 700, 1000, 1024, 2048, 4096, 8192):
        out.append((f"c2-{n}", "N", "N", n, n, n, 1.0, 0.0, (0, 0, 0), "uniform"))
    for tA in "NT":
        for tB in "NT":
            out.append((f"c3-{tA}{tB}", tA, tB, 1531, 997, 2049, -0.75, 1.25, (13, 7, 5), "normal"))
    out.append(("c4-i", "N", "T", 65536, 1024, 4096, 1.0, 1.0, (0, 0, 0), "normal"))
    out.append(("c4-ii", "N", "T", 65536, 4096, 1024, 1.0, 1.0, (0, 0, 0), "normal"))
    # skinny / memory-bound (not a BASELINE.json config): GB/s is the metric
    out.append(("c6-skinny-N16", "N", "N", 65536, 16, 4096, 1.0, 0.0, (0, 0, 0), "uniform"))
    out.append(("c6-skinny-M8", "N", "N", 8, 65536, 4096, 1.0, 0.0, (0, 0, 0), "uniform"))
    return out


class NvmlSampler:
    """SM clock, board power and throttle reasons polled every 2 ms while a
    row's timed reps run; None without NVML.  NVML's
    power reading is a trailing average, so rows shorter than ~1 s report
    mostly the idle power before them; their clock is the burst clock (the
    power limiter's time constant is longer than such rows)."""

    def __init__(self, index):
        self.index, self.samples, self.reasons, self.stop_flag, self.t = index, [], 0, False, None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            return

        rsn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons", None)

        def run():
            while not self.stop_flag:
                try:
                    self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                         pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
                    if rsn:
                        self.reasons |= rsn(h)
                except Exception:
                    break
                time.sleep(0.002)
        import threading
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()

    def stop(self):
        if not self.t:
            return None
        self.stop_flag = True
        self.t.join(timeout=1)
        if not self.samples:
            return None
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}
        return {"sm_mhz": statistics.median(c for c, _ in self.samples),
                "power_w": statistics.median(p for _, p in self.samples), "samples": len(self.samples),
                "reasons": sorted(v for k, v in names.items() if self.reasons & k)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_sweep.jsonl"))
    ap.add_argument("--maths", default="3xtf32,tf32bf16,1xtf32,ffma")
    ap.add_argument("--only", default="")
    ap.add_argument("--variants", default="",
                    help="A/B of library switches: 'tag:VAR=v,VAR2=w;tag2:...' — every (config, math) row is run "
                         "once per variant with those environment variables set (read per call by libemm)")
    ap.add_argument("--shape", default="", help="custom M,N,K,transA,transB (alpha=1, beta=0, uniform)")
    ap.add_argument("--cooldown", type=float, default=2.0,
                    help="idle seconds before each (config, path) row: the power-capped B200's clock depends on "
                         "the preceding load, so rows are measured from the same thermal state")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    pk = peaks()
    stream = torch.cuda.current_stream(dev)
    lines = []
    cfgs = configs()
    if args.shape:
        m_, n_, k_, ta_, tb_ = args.shape.split(",")
        cfgs = [(f"custom-{m_}x{n_}x{k_}-{ta_}{tb_}", ta_, tb_, int(m_), int(n_), int(k_), 1.0, 0.0, (0, 0, 0),
                 "uniform")]
    for name, tA, tB, M, N, K, alpha, beta, pad, kind in cfgs:
        if args.only and not name.startswith(args.only):
            continue
        ar, ac = (M, K) if tA == "N" else (K, M)
        br, bc = (K, N) if tB == "N" else (N, K)
        sig = 1.0 if not name.startswith("c4") else 1.0 / K ** 0.5
        gdev = dev if kind != "normal" else "cpu"
        A = datagen.matrix(kind, datagen.TAG_A, ar, ac, ar + pad[0], sigma=sig, device=gdev)
        B = datagen.matrix(kind, datagen.TAG_B, br, bc, br + pad[1], sigma=sig, device=gdev)
        C0 = datagen.matrix("uniform" if kind != "normal" or not name.startswith("c4") else "normal",
                            datagen.TAG_C, M, N, M + pad[2], sigma=sig, device=gdev)
        dA, dB, dC = (datagen.storage_of(x).to(dev) for x in (A, B, C0))
        variants = [("", {})]
        if args.variants:
            variants = []
            for v in args.variants.split(";"):
                tag, _, kv = v.partition(":")
                variants.append((tag, dict(x.split("=", 1) for x in kv.split(",") if x)))
        for math, (vtag, venv) in ((m, v) for m in args.maths.split(",") for v in variants):
            saved = {k: os.environ.get(k) for k in venv}
            os.environ.update(venv)
            nbytes = emm.workspace_bytes(tA, tB, M, N, K, math)
            ws = torch.empty(nbytes // 4 + 512, dtype=torch.float32, device=dev) if nbytes else None
            wsp = 0
            if ws is not None:
                wsp = ws.data_ptr() + (-ws.data_ptr()) % 1024

            def call():
                st = emm.sgemm_ptr(tA, tB, M, N, K, alpha, dA.data_ptr(), ar + pad[0], dB.data_ptr(), br + pad[1],
                                   beta, dC.data_ptr(), M + pad[2], stream.cuda_stream, math,
                                   wsp or None, nbytes)
                assert st == 0, emm.strerror(st)
            torch.cuda.synchronize()
            time.sleep(args.cooldown)
            for _ in range(3):
                call()
            ts = []
            smp = NvmlSampler(dev.index or 0)
            smp.start()
            for _ in range(args.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                call()
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            clk = smp.stop()
            med = statistics.median(ts)
            b2b = None
            if M * N * K <= 1100 ** 3:
                # back-to-back throughput of latency-bound
                # sizes, a CUDA Graph of 100 calls, no flush (labelled separately)
                g = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream(dev)
                cs.wait_stream(stream)
                with torch.cuda.stream(cs):
                    call_s = cs
                    for _ in range(2):
                        st = emm.sgemm_ptr(tA, tB, M, N, K, alpha, dA.data_ptr(), ar + pad[0], dB.data_ptr(),
                                           br + pad[1], beta, dC.data_ptr(), M + pad[2], call_s.cuda_stream, math,
                                           wsp or None, nbytes)
                    cs.synchronize()
                    with torch.cuda.graph(g, stream=cs):
                        for _ in range(100):
                            emm.sgemm_ptr(tA, tB, M, N, K, alpha, dA.data_ptr(), ar + pad[0], dB.data_ptr(),
                                          br + pad[1], beta, dC.data_ptr(), M + pad[2], cs.cuda_stream, math,
                                          wsp or None, nbytes)
                with torch.cuda.stream(cs):      # replay launches on the current stream
                    g.replay()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(cs)
                    g.replay()
                    e1.record(cs)
                e1.synchronize()
                b2b = e0.elapsed_time(e1) / 100 * 1e3
            fl = 2.0 * M * N * K
            byt = 4.0 * (M * K + K * N + M * N + (M * N if beta != 0 else 0))
            rec = {"config": name, "math": math, "M": M, "N": N, "K": K, "transA": tA, "transB": tB,
                   "median_ms": med, "min_ms": min(ts), "gflops": fl / med / 1e6,
                   "pct_roofline": 100.0 * fl / med / 1e9 / pk[math], "gbs": byt / med / 1e6,
                   "roofline_tflops": pk[math], "l2_flushed": True, "reps": args.reps, "cooldown_s": args.cooldown,
                   "b2b_graph_us": b2b, "clocks": clk}
            if vtag:
                rec["variant"] = vtag
            print(json.dumps(rec), flush=True)
            lines.append(rec)
            del ws
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        del dA, dB, dC
        torch.cuda.empty_cache()
    with open(args.out, "w") as f:
        for r in lines:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
