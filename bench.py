"""Benchmark of the A-orthogonal MGS hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--method mgs-ha-row] [--no-cpu-baseline]

Workload (BASELINE.json configs[1], the config the metric is quoted on):
sparse fp64 A-MGS, m = 1,048,576 (5-point Laplacian on 1024^2, Dirichlet,
+1e-2 I, CSR int32/fp64), n = 64, Z ~ N(0,1) seeded (synthetic: the
reference names no dataset).  One "step" = one full factorization
(mgs_ha / mgs_hp through the drop-in API).  Z (537 MB) and the working set
are larger than the 126 MB L2, so no explicit flush is needed between steps.

``value``  columns/s with Z already resident in HBM (device-timed, CUDA
           events, max over ranks);
``e2e``    columns/s through the same public call with a pinned HOST Z in
           and host Q, R out (H2D + D2H inside the timed region);
``roofline`` the fused trailing kernel: algorithmic bytes per launch over
           its CUDA-event-timed duration, against MEASURED_PEAKS.json;
``cpu_baseline`` the C oracle (bitwise restatement of the reference,
           oracle/) on one host core, one factorization of the same config.

--impl reference times that CPU oracle (the reference's own algorithm; the
reference itself is pure Python and cannot ship to the GPU box) on all the
host threads memory allows, one factorization per thread per step.
N > 1: rows are block-partitioned across ranks (paper_1703_10440_b200.
distributed), per-step NCCL all-reduce of the partial R rows, SpMV halo
exchange; "scaling": "strong".
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

M_SIDE, N_COLS = 1024, 64
METRIC = "A-MGS QR columns/sec (m=1,048,576 5-pt Laplacian CSR, n=64)"
UNIT = "columns/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--method", default="mgs-ha-row")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(
        os.environ.get("LOCAL_RANK", 0))


def workload():
    from paper_1703_10440_b200 import problems

    (indptr, indices, data), Z = problems.config2(device=False)
    return indptr, indices, data, Z


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            # nvidia-smi takes a while to print its first sample: wait for it
            # (up to 3 s) and drop it, so that the samples kept are the ones
            # taken during the timed region that follows
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.005)
            self.lines.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
            except ValueError:
                continue
            for b, name in REASON_BITS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_factor(indptr, indices, data, Z, method):
    from oracle import oracle as O

    t0 = time.perf_counter()
    O.gs_factor(Z, ("csr", indptr, indices, data), method)
    return time.perf_counter() - t0


def run_reference(args, rank, world):
    """--impl reference: the C oracle (reference algorithm) on the host cores."""
    if rank != 0:
        return
    import psutil

    indptr, indices, data, Z = workload()
    m, n = Z.shape
    per_thread = 8 * m * n * 4 + 8 * m * 2  # Zw, P, Q (+X) and vectors of one factorization
    avail = psutil.virtual_memory().available - 8 * m * n * 2
    threads = max(1, min(os.cpu_count() or 1, int(avail // per_thread), 64))
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O

    O.lib()
    times = []
    with ThreadPoolExecutor(threads) as ex:
        for step in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            list(ex.map(lambda _: cpu_oracle_factor(indptr, indices, data, Z, args.method),
                        range(threads)))
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = threads * n * len(times) / total
    sample = (f"{threads} concurrent oracle factorizations ({args.method}, full config: "
              f"m={m}, n={n}) per step, one per host thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; no dataset named by the reference)",
        "config": {"workload": "config2: 5-pt Laplacian 1024^2 + 1e-2 I (CSR), Z 1048576x64 N(0,1)",
                   "method": args.method, "m": m, "n": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world, local_rank):
    import torch

    import paper_1703_10440_b200 as aqr
    from paper_1703_10440_b200 import _lib

    torch.cuda.set_device(local_rank)
    if world > 1 or os.environ.get("AQR_BENCH_DIST"):
        return run_b200_distributed(args, rank, world, local_rank)
    L = _lib.lib()
    family, variant, orientation = args.method.split("-")
    indptr, indices, data, Z = workload()
    m, n = Z.shape
    op = aqr.CsrSpdOperator(indptr, indices, data)
    Zd = torch.from_numpy(Z.T).cuda().t()  # column-major device copy
    fn = {"naive": aqr.mgs_naive, "ha": aqr.mgs_ha, "hp": aqr.mgs_hp}[variant]
    if family == "cgs":
        fn = lambda Z_, op_, o_: aqr.cgs(Z_, op_, variant, o_)  # noqa: E731
    stream = torch.cuda.current_stream()

    res = None
    for _ in range(args.warmup):  # as in the timed loop, the previous result stays alive
        res = fn(Zd, op, orientation)  # during the next call (two cached Q blocks)
    torch.cuda.synchronize()

    # ---- device-resident timed region (value) ----
    launches0 = L.aqr_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            res = fn(Zd, op, orientation)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = int(L.aqr_launch_count() - launches0)
    ms_per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)

    # ---- dominant kernel: fused trailing pass, CUDA events on its stream ----
    import ctypes

    L.aqr_trailing_timer_enable(1)
    for _ in range(args.steps):
        fn(Zd, op, orientation)
    torch.cuda.synchronize()
    L.aqr_trailing_timer_enable(0)
    nl, kms, kbytes = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.aqr_trailing_timer_read(ctypes.byref(nl), ctypes.byref(kms), ctypes.byref(kbytes))
    peak, peak_kind = measured_peaks()
    achieved = (kbytes.value / nl.value) / (kms.value / nl.value / 1e3) / 1e9 if nl.value else None
    share = (kms.value / args.steps) / ms_per_step if nl.value else None
    # DRAM traffic of the same kernel from the committed ncu --set full capture
    # (profiles/<round>/trailing_traffic.json, tools/ncu_summary.py): measured
    # DRAM bytes / algorithmic bytes of the captured launches, applied to
    # this run's mean algorithmic bytes per launch.
    traffic, traffic_src = None, None
    import glob

    for tpath in sorted(glob.glob(os.path.join(REPO, "profiles", "r*", "trailing_traffic*.json")))[::-1]:
        with open(tpath) as f:
            tt = json.load(f)
        if tt.get("method") == args.method and tt.get("traffic_over_algorithmic") and nl.value:
            traffic = tt["traffic_over_algorithmic"] * kbytes.value / nl.value / 1e9
            traffic_src = os.path.relpath(tpath, REPO)
            break
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if achieved else None, "traffic": traffic,
        "traffic_unit": "GB per launch (DRAM read+write)", "traffic_source": traffic_src,
        "kernel": "trailing_kernel", "peak_source": f"{peak_kind} hbm_gbs",
        "launches_per_step": nl.value / args.steps if nl.value else 0,
        "kernel_ms_per_step": kms.value / args.steps, "kernel_share_of_step": share,
        "algorithmic_bytes_per_launch": kbytes.value / nl.value if nl.value else None,
    }

    # ---- whole-step algorithmic bytes (SURVEY.md 8d byte model) ----
    nnz = int(indptr[-1])
    bytes_A = 12 * nnz + 4 * (m + 1)
    T = 8 * m * n * (n - 1)
    mv = bytes_A + 16 * m
    step_bytes = {"ha": T + n * mv + 32 * m * n, "naive": T + 2 * n * mv + 32 * m * n,
                  "hp": 2 * T + (bytes_A + 16 * m * n) + 32 * m * n}[variant]
    step_gbs = step_bytes / (ms_per_step / 1e3) / 1e9

    # ---- end to end: pinned host Z in, host Q/R out, through the public API ----
    e2e = None
    if not args.no_e2e:
        Zh = torch.empty((n, m), dtype=torch.float64).pin_memory().t()
        Zh.copy_(torch.from_numpy(Z))
        r = None
        for _ in range(2):  # steady state: the previous result is alive during the next call,
            r = fn(Zh, op, orientation)  # as in the timed loop (two page-locked result blocks)
        torch.cuda.synchronize()
        t_e = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = fn(Zh, op, orientation)
            e1.record(stream)
            e1.synchronize()
            t_e.append(e0.elapsed_time(e1))
        assert not r.Q.is_cuda
        e2e = {"value": n * len(t_e) / (sum(t_e) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 8 * m * n, "d2h_bytes_per_step": 8 * m * n + 8 * n * n}

    # ---- CPU baseline (rank 0, N = 1): the oracle on one core ----
    cpu = None
    if not args.no_cpu_baseline:
        secs = cpu_oracle_factor(indptr, indices, data, Z, args.method)
        cpu = {"value": n / secs, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"one full {args.method} factorization of the same config "
                         f"(m={m}, n={n}) by the C oracle on 1 of {os.cpu_count()} host cores, "
                         f"{secs:.2f} s"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 5-pt Laplacian + N(0,1) Z; no dataset named by the reference)",
        "config": {"workload": "config2: 5-pt Laplacian 1024^2 + 1e-2 I (CSR int32/fp64), "
                               "Z 1048576x64 N(0,1)", "method": args.method, "m": m, "n": n,
                   "nnz": nnz, "parallelism": f"rows/{world}",
                   "l2": "inputs larger than L2 (Z 537 MB > 126 MB), no flush"},
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "hbm_gbs_step": step_gbs, "step_algorithmic_bytes": step_bytes,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def run_b200_distributed(args, rank, world, local_rank):
    """N > 1: config 2 row-partitioned over N GPUs (strong scaling), NCCL."""
    import torch
    import torch.distributed as dist

    from paper_1703_10440_b200 import _lib
    from paper_1703_10440_b200 import distributed as DD

    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", local_rank))
    L = _lib.lib()
    indptr, indices, data, Z = workload()
    m, n = Z.shape
    part = DD.row_partition(m, world, align=M_SIDE)  # whole grid rows per rank
    r0, r1 = part[rank]
    op = DD.DistCsrSpdOperator(indptr[r0:r1 + 1] - indptr[r0], indices[indptr[r0]:indptr[r1]],
                               data[indptr[r0]:indptr[r1]], part, rank)
    Zd = torch.from_numpy(np.ascontiguousarray(Z[r0:r1].T)).cuda().t()
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        DD.dist_factorize(Zd, op, args.method)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.aqr_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            DD.dist_factorize(Zd, op, args.method)
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    launches = int(L.aqr_launch_count() - launches0)
    ms_per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)
    # end to end: pinned host row block in, host Q block + R out, every rank
    e2e = None
    if not args.no_e2e:
        Zh = torch.empty((n, r1 - r0), dtype=torch.float64).pin_memory().t()
        Zh.copy_(torch.from_numpy(Z[r0:r1]))
        Qh = torch.empty((n, r1 - r0), dtype=torch.float64).pin_memory().t()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            res = DD.dist_factorize(Zh.to("cuda", non_blocking=True), op, args.method)
            Qh.copy_(res.Q, non_blocking=True)
            Rh = res.R.cpu()
        e1.record(stream)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": n * args.steps / (float(et.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 8 * m * n, "d2h_bytes_per_step": 8 * m * n + 8 * n * n * world}
        del Rh
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded 5-pt Laplacian + N(0,1) Z; no dataset named by the reference)",
            "config": {"workload": "config2 row-partitioned: 5-pt Laplacian 1024^2 + 1e-2 I (CSR), "
                                   "Z 1048576x64 N(0,1)", "method": args.method, "m": m, "n": n,
                       "parallelism": (f"rows/{world} (peer memory: halo reads and both per-step all-reduces "
                                       f"fused into the step kernels over NVLink)"
                                       if args.method.split("-")[1] in ("ha", "hp")
                                       else f"rows/{world} (NCCL all-reduce per step, SpMV halo exchange)"),
                       "l2": "inputs larger than L2, no flush"},
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "roofline": None, "cpu_baseline": None, "e2e": e2e, "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
