#!/usr/bin/env python
"""bench.py — the measured step of the emm SGEMM hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl emm|reference] [--math 3xtf32|ffma|1xtf32]
                    [--size S]

Workload (BASELINE.json configs[4], the configuration its metric — GFLOP/s at
1/2/4/8 B200 — is quoted on): square SGEMM M=N=K=32768, FP32, column-major,
transA=transB='N', alpha=1, beta=0, A and B uniform[-1,1) from seed 0
(datagen), 4 GiB per operand.  One STEP = one full pass of the hot path on
that problem: emm_sgemm_ex = re-buffer/split of A and B (KN4) + the tcgen05
3xTF32 GEMM (KN1), i.e. every row of SURVEY.md §8(a).  At N > 1 the problem
is row-sharded (emm_row_partition) and each step is emm_sgemm_multi: B
broadcast from rank 0 over NCCL in column panels overlapped with the
per-panel GEMMs ("scaling": "strong": total work fixed).

* value: 2MNK * steps / (max over ranks of the CUDA-event time of the K
  timed steps), inputs resident in HBM.  Inputs (12.9 GB) exceed the 126 MB
  L2, so no flush is needed between steps (stated in config).
* e2e: the same metric through the C-ABI host-buffer entry emm_sgemm_host
  (pinned host A, B in; C out) — copies inside the timed region.
* roofline: the dominant kernel (tc_sgemm_kernel), algorithmic flops 2MNK per
  launch / its CUDA-event duration on the launching stream.  `peak` = the
  tensor pipe's measured ceiling for this exact instruction stream: the
  GEMM's tcgen05 MMA sequence with operands resident in SMEM, run for 2 s on
  this GPU right after the timed steps, sustained under the same power cap
  (DESIGN.md §6a).  Reported beside it: the MEASURED_PEAKS-derived figure
  (bf16 sustained x 1.1/2.25 nominal tf32/bf16 / 3), which a good kernel
  exceeds because the TF32 tensor pipe draws less power than cuBLAS bf16, and
  the nominal 1965 MHz figure (148 SMs x 4096 TF32 flop/clk / 3).
* --gpus N without WORLD_SIZE in the environment: bench.py starts N rank
  processes itself (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*), one per GPU;
  under torchrun it is one of the ranks.  At N > 1 B is registered with the
  communicator, so it travels by copy-engine peer copies along the ring
  (`--bcast nccl` for ncclBroadcast), and the line reports
  `comm_exposed_ms` = the step time not covered by the library's kernels on
  the compute stream (waiting for B).
* cpu_baseline: the oracle (oracle/oracle.c) on a bounded sample of output
  rows of the same workload, all host cores, rank 0 at N=1 only.
* --impl reference: the oracle itself, timed as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SGEMM GFLOP/s (2MNK/t) and % of FP32/TF32 roofline at 1/2/4/8 B200"
TF32_PER_BF16 = 1.1 / 2.25          # nominal dense ratio, B200_PROFILING.md table


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="emm", choices=["emm", "reference"])
    p.add_argument("--math", default="3xtf32", choices=["3xtf32", "ffma", "1xtf32", "tf32bf16"])
    p.add_argument("--size", type=int, default=32768)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-alt", action="store_true", help="skip the other FP32-accurate tensor path")
    p.add_argument("--allgather", default="none", choices=["none", "nccl", "fused"],
                   help="multi: also gather C into every rank's full M x N output (NCCL all-gather + unpack, "
                        "or fused into the GEMM epilogue through registered peer buffers)")
    p.add_argument("--bcast", default="ce", choices=["ce", "nccl"],
                   help="multi: B by copy-engine peer copies along the ring (registered buffer) or ncclBroadcast")
    p.add_argument("--force-multi", action="store_true",
                   help="run the row-sharded emm_sgemm_multi path (NCCL) even at one rank")
    p.add_argument("--cpu-rows", type=int, default=0, help="oracle sample rows (0 = auto)")
    p.add_argument("--no-probe", action="store_true", help="skip the MMA-only tensor-pipe ceiling probe")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return mp["bf16_tflops"], mp.get("bf16_tflops_sustained", mp["bf16_tflops"]), mp.get("hbm_gbs"), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def workload_config(n, args, world):
    return {"workload": f"BASELINE configs[4]: SGEMM M=N=K={n}, FP32 column-major, transA=transB=N, "
                        f"alpha=1, beta=0, A,B ~ U[-1,1) seed 0"
                        + (f", row-sharded over {world} GPUs, B broadcast from rank 0" if world > 1 else ""),
            "M": n, "N": n, "K": n, "transA": "N", "transB": "N", "alpha": 1.0, "beta": 0.0,
            "math": args.math, "global_batch": None, "seq_len": None,
            "parallelism": f"rows{world}" if world > 1 else "single",
            "l2": "inputs (3 x 4 GiB) exceed the 126 MB L2: no flush between steps"}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, watts = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            try:
                watts.append(float(f[3]))
            except ValueError:
                pass
            for nm, v in zip(names, f[4:8]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(watts) if watts else None}


# --------------------------------------------------------------------- oracle
_ORACLE_INPUTS = {}


def oracle_inputs(n, nrows, gen_device):
    """Compact sampled rows of A and the full B on the host (cached)."""
    key = (n, nrows)
    if key not in _ORACLE_INPUTS:
        import numpy as np
        import datagen
        rows = np.linspace(0, n - 1, nrows).astype(np.int64)
        A_s = datagen.storage_of(datagen.submatrix("uniform", datagen.TAG_A, n, n, rows)).numpy()
        B = datagen.storage_of(datagen.matrix("uniform", datagen.TAG_B, n, n, device=gen_device)).cpu().numpy()
        _ORACLE_INPUTS.clear()
        _ORACLE_INPUTS[key] = (A_s, B)
    return _ORACLE_INPUTS[key]


def cpu_oracle_sample(n, nrows, gen_device="cpu"):
    """Time the oracle on `nrows` sampled output rows of the workload
    (compact A rows, full B on the host).  Returns (gflops, seconds, cores)."""
    import oracle
    A_s, B = oracle_inputs(n, nrows, gen_device)
    cores = oracle.default_threads()
    t0 = time.perf_counter()
    R, S, T, st = oracle.sgemm_sub("N", "N", nrows, n, n, 1.0, A_s, nrows, B, n, 0.0, None, nrows,
                                   nthreads=cores)
    dt = time.perf_counter() - t0
    assert st == 0
    return 2.0 * nrows * n * n / dt / 1e9, dt, cores


def auto_rows(n):
    # ~15 s of oracle work on the host: the j-p-i FP64 loop ran at ~2.8 GFLOP/s
    # per core on the B200 box (16 cores, round 1)
    cores = len(os.sched_getaffinity(0))
    rate = 2.8e9 * cores
    r = int(15.0 * rate / (2.0 * n * n))
    return max(4, min(512, r))


# --------------------------------------------------------------------- tensor-pipe ceiling
def mma_probe(math, clocks_of, seconds=2.0):
    """The GEMM's MMA stream with operands resident in SMEM (emm_debug_mma_probe,
    k_probe.cu): burst and sustained 2MNK-equivalent TFLOP/s under the same
    power cap, with the SM clock sampled during the sustained run."""
    import ctypes
    import paper_1912_04379_b200 as emm
    terms = {"3xtf32": 3, "tf32bf16": 2, "1xtf32": 1}[math]
    L = emm.lib()
    L.emm_debug_mma_probe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)]
    L.emm_debug_mma_probe.restype = ctypes.c_int
    import torch
    s = torch.cuda.current_stream().cuda_stream
    stages = {3: 6000, 2: 9000, 1: 18000}[terms]      # ~5 ms per launch
    msv, fl = ctypes.c_float(), ctypes.c_double()
    for _ in range(3):
        if L.emm_debug_mma_probe(terms, stages, s, ctypes.byref(msv), ctypes.byref(fl)):
            return None
    burst = fl.value / (msv.value * 1e-3) / 1e12
    clocks_of.start()
    rates = []
    t_end = time.time() + seconds
    while time.time() < t_end:
        if L.emm_debug_mma_probe(terms, stages, s, ctypes.byref(msv), ctypes.byref(fl)):
            return None
        rates.append(fl.value / (msv.value * 1e-3) / 1e12)
    c = clocks_of.stop()
    return {"burst_tflops": burst, "sustained_tflops": statistics.median(rates[len(rates) // 2:]),
            "sm_mhz": c["sm_mhz"] if c else None, "seconds": seconds,
            "what": "the GEMM's tcgen05 MMA stream (CTA pairs, M256xN256xK8, same split) with operands resident "
                    "in SMEM: the tensor pipe's ceiling at this power cap without TMA/L2/DRAM traffic"}


# --------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    n = args.size
    rows = args.cpu_rows or max(4, auto_rows(n) // 4)
    times = []
    for i in range(args.warmup + args.steps):
        g, dt, cores = cpu_oracle_sample(n, rows)
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    gflops = 2.0 * rows * n * n * len(times) / tot / 1e9
    line = {"metric": METRIC, "value": gflops, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": workload_config(n, args, 1),
            "cpu_baseline": {"value": gflops, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                             "sample": f"{rows} output rows x {n} cols (all of K={n}) of the workload per step"},
            "e2e": {"value": gflops, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- launcher
def spawn_ranks(n):
    """`--gpus N` outside torchrun: one process per GPU, torchrun's env
    contract; rank 0's stdout (the JSON line) is passed through."""
    import socket
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=60).stdout
        visible = sum(1 for ln in out.splitlines() if ln.startswith("GPU "))
        cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
        if cvd:
            visible = min(visible, len([x for x in cvd.split(",") if x.strip()]))
    except Exception:
        visible = 0
    if visible < n:
        sys.stderr.write(f"bench.py: --gpus {n} but only {visible} GPU(s) visible\n")
        sys.exit(2)
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = rc or p.wait()
    sys.exit(rc)


# --------------------------------------------------------------------- emm arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import datagen
    import paper_1912_04379_b200 as emm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    multi = world > 1 or args.force_multi
    if multi:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
    n = args.size
    M = N = K = n
    flops = 2.0 * M * N * K
    stream = torch.cuda.Stream(dev)

    # ---- inputs resident in HBM (generated on the device, bit-identical to host datagen)
    r0, rows = emm.row_partition(M, world, rank) if multi else (0, M)
    A = datagen.submatrix("uniform", datagen.TAG_A, M, K, torch.arange(r0, r0 + rows), device=dev) \
        if multi else datagen.matrix("uniform", datagen.TAG_A, M, K, device=dev)
    if world == 1 or rank == 0:
        B = datagen.matrix("uniform", datagen.TAG_B, K, N, device=dev)
    else:
        B = torch.empty((N, K), dtype=torch.float32, device=dev).t()
    C = torch.empty((N, max(rows, 1)), dtype=torch.float32, device=dev).t()[:rows, :]
    ws = None
    if not multi:
        nbytes = max(emm.workspace_bytes("N", "N", M, N, K, m) for m in (args.math, "3xtf32", "tf32bf16"))
        ws = torch.empty(max(nbytes // 4 + 256, 1), dtype=torch.float32, device=dev) if nbytes else None
        if ws is not None and ws.data_ptr() % 1024:
            ws = ws[(1024 - ws.data_ptr() % 1024) // 4:]
    comm = emm.Comm(rank, world) if multi else None
    if multi and args.bcast == "ce":
        try:
            comm.register_input(B)
        except emm.EmmError as e:
            # registration outcomes are agreed across ranks (multi.cu), so
            # every rank falls back together
            print(f"rank {rank}: B registration failed ({e}); ncclBroadcast data plane", file=sys.stderr)
            args.bcast = "nccl"
    C_full = None
    if multi and args.allgather != "none":
        C_full = torch.empty((N, M), dtype=torch.float32, device=dev).t()
        if args.allgather == "fused":
            try:
                comm.register_output(C_full)
            except emm.EmmError as e:
                print(f"rank {rank}: C_full registration failed ({e}); NCCL all-gather", file=sys.stderr)
                args.allgather = "nccl"

    def make_step(math):
        def step():
            if multi:
                emm.sgemm_multi(comm, M, N, K, A, B, C, 1.0, 0.0, math=math, stream=stream, C_full=C_full)
            else:
                emm.sgemm_ex(A, B, C, 1.0, 0.0, math=math, workspace=ws, stream=stream)
        return step

    def barrier():
        torch.cuda.synchronize(dev)
        if multi:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    bf16, bf16_sus, hbm, src = peaks()
    tf32_sus = bf16_sus * TF32_PER_BF16
    tf32_burst = bf16 * TF32_PER_BF16

    def path_peak(math):
        if math == "3xtf32":
            return tf32_sus / 3.0, tf32_burst / 3.0, "3xTF32-effective (TF32/3)"
        if math == "tf32bf16":
            # one TF32 MMA (K8) + one BF16 MMA (K16) per 8 of K: 2 TF32-MMA times
            return tf32_sus / 2.0, tf32_burst / 2.0, "TF32+BF16-effective (TF32/2)"
        if math == "1xtf32":
            return tf32_sus, tf32_burst, "TF32"
        sm = torch.cuda.get_device_properties(dev).multi_processor_count
        p = sm * 256 * 1965e6 / 1e12
        return p, p, "FP32 FFMA (SMs x 256 flop/clk x 1965 MHz)"

    def measure(math, steps, warmup):
        """W untimed steps, then exactly `steps` timed steps bracketed by a
        barrier + device sync; CUDA events on the launching stream; max over
        ranks; clocks sampled during the timed region."""
        step = make_step(math)
        with torch.cuda.stream(stream):
            for _ in range(warmup):
                step()
        barrier()
        clocks = ClockSampler(local)
        clocks.start()
        emm.profile_enable(True)
        emm.profile_read()
        l0 = emm.launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(steps):
                step()
        ev1.record(stream)
        barrier()
        launches = emm.launch_count() - l0
        ms = ev0.elapsed_time(ev1)
        gemm_ms, gemm_n, other_ms, other_n = emm.profile_read()
        emm.profile_enable(False)
        clk = clocks.stop()
        if multi:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        peak, peak_b, pname = path_peak(math)
        flops_rank = 2.0 * rows * N * K
        kernel_ms = gemm_ms / max(gemm_n, 1)
        per_launch_flops = flops_rank / max(gemm_n // max(steps, 1), 1)
        achieved = per_launch_flops / (kernel_ms / 1e3) / 1e12 if kernel_ms > 0 else None
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                with open(tp) as f:
                    traffic = json.load(f).get(f"{math}_{n}")
            except Exception:
                traffic = None
        roof = {"bound": "tensor" if math != "ffma" else "alu", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_kind": (f"{pname}, from {src} bf16 sustained {bf16_sus} TF x 1.1/2.25" if math != "ffma"
                              else f"{pname}: derived from the guide's unit counts and the max clock (DESIGN.md §6)"),
                "peak_derived": peak, "frac_derived": (achieved / peak) if achieved else None,
                "peak_burst": peak_b, "frac_burst": (achieved / peak_b) if achieved else None,
                "kernel": {"ffma": "ffma_tma_kernel (KN3b)", "1xtf32": "tc1w_kernel (KN2w, 256x512 tiles)",
                           "3xtf32": "tc_xs_kernel (KN1X, 3xTF32 split in the kernel)"}.get(
                    math, "tc_sgemm_kernel (KN1)"),
                "kernel_ms": kernel_ms, "kernel_share_of_step": (gemm_ms / ms) if ms > 0 else None,
                "other_kernels_ms_per_step": other_ms / steps}
        if math != "ffma":
            sm = torch.cuda.get_device_properties(dev).multi_processor_count
            nom = sm * 4096 * 1965e6 / 1e12 / {"3xtf32": 3.0, "tf32bf16": 2.0, "1xtf32": 1.0}[math]
            roof["peak_nominal"] = nom
            roof["frac_nominal"] = (achieved / nom) if achieved else None
        # step time not covered by this rank's kernels on the compute stream
        # (multi: waiting for B chunks / the completion flags)
        exposed = max(0.0, ms / steps - (gemm_ms + other_ms) / steps) if multi else None
        return {"value": flops * steps / (ms / 1e3) / 1e9, "ms": ms, "launches": launches, "clocks": clk,
                "roofline": roof, "peak": peak, "comm_exposed_ms": exposed}

    res = measure(args.math, args.steps, args.warmup)
    value, ms, launches, clk, roofline, peak = (res["value"], res["ms"], res["launches"], res["clocks"],
                                                res["roofline"], res["peak"])
    comm_exposed = res["comm_exposed_ms"]
    if args.math != "ffma" and not args.no_probe:
        pr = mma_probe(args.math, clocks_of=ClockSampler(local))
        if pr and roofline.get("achieved"):
            pr["frac"] = roofline["achieved"] / pr["sustained_tflops"]
            if pr.get("sm_mhz") and clk and clk.get("sm_mhz"):
                pr["frac_per_clock"] = (roofline["achieved"] / clk["sm_mhz"]) / (pr["sustained_tflops"] / pr["sm_mhz"])
            # the measured tensor-pipe ceiling of this instruction stream is
            # the roofline denominator (a kernel cannot exceed it)
            roofline["peak"] = pr["sustained_tflops"]
            roofline["frac"] = roofline["achieved"] / roofline["peak"]
            roofline["peak_kind"] = ("measured in this run: the GEMM's tcgen05 MMA stream with operands resident in "
                                     "SMEM, 2 s sustained under the same power cap (emm_debug_mma_probe); "
                                     "peak_derived = MEASURED_PEAKS bf16 sustained x 1.1/2.25 / terms, "
                                     "peak_nominal = 148 SMs x 4096 TF32 flop/clk x 1965 MHz / terms")
        roofline["ceiling_probe"] = pr
    ms_step = ms / args.steps
    alt = {}
    if args.math in ("3xtf32", "tf32bf16") and not args.no_alt and not multi:
        m2 = "tf32bf16" if args.math == "3xtf32" else "3xtf32"
        k2 = max(3, args.steps // 2)
        r2 = measure(m2, k2, 2)
        alt[m2] = {"value": r2["value"], "unit": "GFLOP/s", "steps": k2, "ms_per_step": r2["ms"] / k2,
                   "roofline": r2["roofline"], "clocks": r2["clocks"],
                   "note": "same workload, the other FP32-accurate tensor-core split (parity-tested at 1e-5*S)"}

    # ---- e2e through the C-ABI host-buffer entry (copies inside the timed region)
    e2e = None
    if not args.no_e2e and not multi:
        del ws
        torch.cuda.empty_cache()
        hA = datagen.storage_of(A).cpu().pin_memory()
        hB = datagen.storage_of(B).cpu().pin_memory()
        hC = torch.empty(M * N, dtype=torch.float32).pin_memory()
        emm.sgemm_host("N", "N", M, N, K, 1.0, hA, M, hB, K, 0.0, hC, M, math=args.math)  # warm (allocs)
        e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            emm.sgemm_host("N", "N", M, N, K, 1.0, hA, M, hB, K, 0.0, hC, M, math=args.math)
        dt = time.perf_counter() - t0
        e2e = {"value": flops * e_steps / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 4 * (M * K + K * N),
               "d2h_bytes_per_step": 4 * M * N, "steps": e_steps,
               "api": "emm_sgemm_host (pinned host A,B -> device, C -> host, synchronous)"}
        # spot-check the e2e result against a device call of the same path
        # (the host pipeline runs KN1X on the landed blocks in K phases that
        # continue each promotion chain: deterministic, so bitwise equal)
        ws = None
        with torch.cuda.stream(stream):
            emm.sgemm(A, B, C, 1.0, 0.0, math=args.math, stream=stream)
        stream.synchronize()
        Cd = C[:64, :64].cpu()
        hv = hC.reshape(N, M)[:64, :64].t()
        assert torch.equal(Cd, hv), "e2e result differs from device result"
        del hA, hB, hC
        emm.release_cache()
    elif not args.no_e2e and multi:
        hA = datagen.storage_of(A).cpu().pin_memory() if rows else None
        hB = datagen.storage_of(B).cpu().pin_memory() if rank == 0 else None
        hC = torch.empty(max(rows, 1) * N, dtype=torch.float32).pin_memory()
        e_steps = max(1, min(args.steps, 3))
        barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            with torch.cuda.stream(stream):
                if rows:
                    datagen.storage_of(A).copy_(hA, non_blocking=True)
                if rank == 0:
                    datagen.storage_of(B).copy_(hB, non_blocking=True)
                make_step(args.math)()
                hC[: rows * N].copy_(C.t().reshape(-1) if rows else hC[:0], non_blocking=True)
            stream.synchronize()
        barrier()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(dt, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": flops * e_steps / float(dt.item()) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": 4 * (M * K + K * N), "d2h_bytes_per_step": 4 * M * N, "steps": e_steps,
               "api": "H2D copies + emm_sgemm_multi + D2H, per rank"}

    cpu = None
    if rank == 0 and not multi and not args.no_cpu:
        nrows = args.cpu_rows or auto_rows(n)
        g, dt, cores = cpu_oracle_sample(n, nrows, gen_device=dev)
        cpu = {"value": g, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "seconds": dt,
               "sample": f"{nrows} evenly spaced output rows x all {n} columns (full K={n}) of the workload"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(workload_config(n, args, world),
                               **({"path": "emm_sgemm_multi (row-sharded)", "allgather": args.allgather}
                                  if multi else {})),
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk, "alt_paths": alt or None,
                "pct_of_roofline": 100.0 * value / 1e3 / (roofline["peak"] * world) if roofline.get("peak") else None}
        if multi:
            line["comm_exposed_ms"] = comm_exposed
            line["config"]["bcast"] = args.bcast
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
