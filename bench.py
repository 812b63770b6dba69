"""Benchmark of the A-orthogonal MGS hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config 5] [--method mgs-hp-row] [--no-cpu-baseline] [--no-e2e]

Workload (default): BASELINE.json configs[4], "config 5" -- the largest
single-GPU configuration and the one the metric's 1/2/4/8-GPU curve is
quoted on: sparse fp64 A-MGS, m = 256^3 = 16,777,216 (27-point stencil,
Dirichlet, centre 26 + 1e-2, neighbours -1, CSR int32/fp64, nnz
449,455,096), n = 256, Z ~ N(0,1) seeded (34.4 GB; synthetic: the reference
names no dataset), HP type, row oriented.  ``--config 2|3|4`` selects the
other BASELINE configs (their method defaults: HA).  One "step" = one full
factorization through the drop-in API.  Every input is larger than the
126 MB L2, so no flush is needed between steps.

``value``  columns/s with Z already resident in HBM (CUDA events on the
           launching stream, max over ranks);
``e2e``    columns/s through the same public call (``aqr.mgs_hp`` etc.) with
           a pageable NUMPY Z in and numpy Q, R out -- host staging, H2D and
           D2H inside the timed region (wall clock around the call);
``roofline`` the dominant kernel (the fused trailing pass): algorithmic
           bytes per launch over its CUDA-event-timed duration inside the
           timed region, against MEASURED_PEAKS.json; plus the whole-step
           figure (SURVEY.md 8d byte model);
``cpu_baseline`` the C oracle (a bitwise restatement of the reference,
           oracle/) on one host core: a column-truncated run of the same
           config, each phase extrapolated to n columns by its own call count
           (block apply and normalize: n / n', projections: n(n-1) / n'(n'-1)).

--impl reference times that CPU oracle (the reference's algorithm; the
reference itself is pure Python + numba and cannot ship to the GPU box) on
all the host threads memory allows, concurrent truncated factorizations per
step, extrapolated the same way; rank 0 only.

N > 1 (torchrun, or ``--gpus N`` which re-launches itself under torchrun):
config 5's grid planes are split across ranks (peer-memory path: halo reads
and both per-step all-reduces fused into the step kernels over NVLink, no
collective call in the step loop); "scaling": "strong" (fixed total work).
"""

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "A-MGS QR columns/sec"
UNIT = "columns/s"

CONFIGS = {
    2: {"workload": "config2: 5-pt Laplacian 1024^2 + 1e-2 I (CSR int32/fp64), Z 1048576x64 N(0,1)",
        "method": "mgs-ha-row"},
    3: {"workload": "config3: 7-pt variable-coefficient diffusion 128^3 + 1e-3 I (CSR int32/fp64), "
                    "Z 2097152x128 = N(0,1) diag(10^(-6j/127))", "method": "mgs-ha-row"},
    4: {"workload": "config4: dense A = B^T B / 32768 + 0.1 I (32768^2 fp64), Z 32768x256 N(0,1)",
        "method": "mgs-ha-row"},
    5: {"workload": "config5: 27-pt stencil 256^3 + 1e-2 I (CSR int32/fp64), Z 16777216x256 N(0,1) (34.4 GB)",
        "method": "mgs-hp-row"},
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--method", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    a.method = a.method or CONFIGS[a.config]["method"]
    if a.warmup < 3:
        ap.error("--warmup must be >= 3 (timing rules)")
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def relaunch_under_torchrun(args):
    """--gpus N without a torchrun environment: run N ranks of this script."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def config_dict(cfg, method, m, n, nnz, world):
    """The ``config`` of the JSON line -- identical for both arms."""
    d = {"workload": CONFIGS[cfg]["workload"], "method": method, "m": m, "n": n,
         "parallelism": f"rows/{world}" + (" (whole grid planes per rank; halo + per-step all-reduces over "
                                          "peer memory)" if world > 1 else ""),
         "l2": "every input larger than the 126 MB L2, no flush"}
    if nnz is not None:
        d["nnz"] = nnz
    return d


TRAIL_WIN = 4  # write-back period of the windowed trailing passes (AQR_TRAIL_WIN default)
X_WIN = 16     # HP X catch-up period (AQR_X_WIN default)


def survey_bytes(variant, m, n, bytes_A):
    """SURVEY.md 8d's one-pass look-ahead model: every trailing element (and
    for HP every trailing X element) read and written once per step."""
    T = 8 * m * n * (n - 1)
    mv = bytes_A + 16 * m
    return {"ha": T + n * mv + 32 * m * n, "naive": T + 2 * n * mv + 32 * m * n,
            "hp": 2 * T + (bytes_A + 16 * m * n) + 32 * m * n}[variant]


def step_bytes(variant, m, n, bytes_A, win=TRAIL_WIN, xwin=X_WIN):
    """Algorithmic HBM bytes of one single-GPU row-form factorization as this
    build schedules it (the host loop of csrc/aqr_b200.cu, Run::row_form):

    * trailing pass i (t = n-1-i columns): every stored element read once,
      written only on write-back passes (every ``win``-th; else only column
      i+1), the q window (i - zbase columns), p_i, and q_i / p_i stored;
    * HA / naive: the operator products (A once + z in + x out) and the
      column update / norm vectors as in SURVEY 8d;
    * HP: X = A Z once (A + Z in + X out); step j forms x_j from the stored
      X_j and the p columns it lags behind; every ``xwin`` steps the stored
      X columns catch up (read + write + the p window)."""
    T, zbase, xbase = 0, 0, 0
    for i in range(n):
        t = n - 1 - i
        w = i - zbase if t > 0 else 0
        store = w >= win
        T += 8 * m * (t + (t if store else (min(t, 1) if w > 0 else 0)) + w + 1)
        T += 8 * m * (3 if variant == "hp" else 2)  # zsrc read, q_i (+ p_i) stored
        if store:
            zbase = i
    if variant == "hp":
        X = bytes_A + 16 * m * n  # X = A Z
        for j in range(n):
            X += 8 * m * ((j - xbase) + 1 + 1 + (2 if j else 0) + 1)  # p window, X_j, z_j (+q, z store), x_j
            if j - xbase >= xwin and j + 1 < n:
                X += 8 * m * (2 * (n - 1 - j) + (j - xbase))
                xbase = j
        return T + X
    mv = bytes_A + 16 * m
    return T + (2 if variant == "naive" else 1) * n * mv + 16 * m * n


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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


# ---- workloads ----------------------------------------------------------------

def device_workload(cfg, rank=0, world=1):
    """(op arrays or dense A, Z) on the GPU; with world > 1 this rank's rows."""
    from paper_1703_10440_b200 import problems

    if cfg == 5:
        planes = None
        if world > 1:
            n_side = 256
            planes = (n_side * rank // world, n_side * (rank + 1) // world)
        csr, Z = problems.config5(planes=planes)
        return {"csr": csr, "Z": Z, "m": 256 ** 3, "n": 256, "planes": planes}
    if world > 1:
        raise SystemExit("N > 1 runs config 5 (BASELINE.json's multi-GPU sparse config)")
    if cfg == 4:
        A, Z = problems.config4()
        return {"dense": A, "Z": Z, "m": A.shape[0], "n": Z.shape[1]}
    csr, Z = (problems.config2 if cfg == 2 else problems.config3)(device=True)
    return {"csr": csr, "Z": Z, "m": Z.shape[0], "n": Z.shape[1]}


def banded_bytes(op, m):
    """(bytes per apply, description) of a CsrSpdOperator on the banded view
    (csrc/aqr_band.cuh): a 4-byte row mask, plus the values diagonal-major when
    the diagonals are not constant; None when the CSR kernels run."""
    offs = getattr(op, "band_offsets", None)
    if offs is None:
        return None
    nd, const = len(offs), bool(op._band.constant)
    return (4 * m + (0 if const else 8 * nd * m),
            f"banded view of the CSR operator ({nd} offsets, {'constant' if const else 'varying'} diagonals)")


def bytes_of_A(wl):
    if "dense" in wl:
        return 8 * wl["m"] * wl["m"], None
    nnz = int(wl["csr"][0][-1])
    return 12 * nnz + 4 * (wl["m"] + 1), nnz


def host_oracle_inputs(cfg, ncols):
    """Host (op spec, Z[:, :ncols]) for the C oracle: the same bytes the GPU arm factorizes."""
    import torch

    from paper_1703_10440_b200 import problems

    if cfg == 2:
        (ip, ix, dv), Z = problems.config2(device=False)
        return ("csr", ip, ix, dv), np.asfortranarray(Z[:, :ncols]), Z.shape[1]
    if cfg == 3:
        (ip, ix, dv), Z = problems.config3(device=False)
        return ("csr", ip, ix, dv), np.asfortranarray(Z[:, :ncols]), Z.shape[1]
    if cfg == 4:
        A, Z = problems.config4()
        spec = ("dense", np.asfortranarray(A.cpu().numpy()))
        Zh = np.asfortranarray(Z[:, :ncols].cpu().numpy())
        del A, Z
        torch.cuda.empty_cache()
        return spec, Zh, 256
    # config 5: the CSR is built on the device and copied out; Z's first
    # column block comes from the same seeded generator as the full Z
    m = 256 ** 3
    ip, ix, dv = problems.stencil27_device(256, 1e-2, "cuda")
    spec = ("csr", ip.cpu().numpy(), ix.to(torch.int64).cpu().numpy(), dv.cpu().numpy())
    del ip, ix, dv
    blk = -(-ncols // problems.CONFIG5_ZCHUNK) * problems.CONFIG5_ZCHUNK
    Zh = np.asfortranarray(problems.config5_Z(m, blk)[:, :ncols].cpu().numpy())
    torch.cuda.empty_cache()
    return spec, Zh, 256


def oracle_truncated_seconds(spec, Zh, method, n_full):
    """(measured s, extrapolated full-width s) of one oracle factorization of Zh."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    O.gs_factor(Zh, spec, method)
    secs = time.perf_counter() - t0
    apply_s, norm_s, proj_s = O.last_phase_times()
    other = max(0.0, secs - apply_s - norm_s - proj_s)  # copies / allocation: linear in n
    est = O.extrapolate_seconds((apply_s, norm_s + other, proj_s), Zh.shape[1], n_full)
    return secs, est


CPU_COLS = {2: 64, 3: 16, 4: 8, 5: 16}  # columns of the 1-core cpu_baseline sample per config


# ---- reference arm ---------------------------------------------------------------

def run_reference(args, rank, world):
    """--impl reference: the C oracle (reference algorithm) on the host cores."""
    if rank != 0:
        return
    import psutil

    from oracle import oracle as O

    O.lib()
    cfg, n_full = args.config, None
    budget_s = 150.0  # the whole --warmup W --steps K run
    total_steps = args.warmup + args.steps
    t_start = time.perf_counter()
    ncols = {2: 64, 3: 8, 4: 4, 5: 4}[cfg]
    spec, Zh, n_full = host_oracle_inputs(cfg, 16 if cfg in (3, 5) else ncols)
    m = Zh.shape[0]
    nnz = int(spec[1][-1]) if spec[0] == "csr" else None
    # host threads: memory-bound by the oracle's buffers (Zw, P, Q, X, xbuf per run)
    per_run = 8 * m * 16 * 5 + 8 * m * 2
    avail = psutil.virtual_memory().available - (4 << 30)
    threads = max(1, min(os.cpu_count() or 1, int(avail // per_run), 64))
    from concurrent.futures import ThreadPoolExecutor

    def one(ncol):
        return oracle_truncated_seconds(spec, np.asfortranarray(Zh[:, :ncol]), args.method, n_full)

    samples, walls = [], []
    with ThreadPoolExecutor(threads) as ex:
        for step in range(total_steps):
            if step == 1 and cfg in (3, 4, 5):
                # size the sample from the first (warm-up) step: the whole run in ~budget_s
                left = budget_s - (time.perf_counter() - t_start)
                per_step = max(left / max(total_steps - 1, 1), 1.0)
                for cand in (16, 12, 8, 6, 4):
                    if cand <= Zh.shape[1] and walls[0] * cand / ncols <= per_step:
                        ncols = cand
                        break
            t0 = time.perf_counter()
            res = list(ex.map(lambda _: one(ncols), range(threads)))
            walls.append(time.perf_counter() - t0)
            if step >= args.warmup:
                samples.append(sum(n_full / est for _, est in res))  # columns/s of the threads together
    value = statistics.mean(samples)
    truncated = ncols < n_full
    sample = (f"{threads} concurrent oracle factorizations ({args.method}) per step, one per host thread, "
              f"of the full config (m={m}, n={n_full}) "
              + (f"truncated to its first {ncols} columns; each run's phases extrapolated to n={n_full} "
                 f"(apply/normalize x n/n', projections x n(n-1)/(n'(n'-1))) -- extrapolated"
                 if truncated else "in full"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * threads * n_full / value,
        "ms_per_step_sample": 1e3 * statistics.mean(walls[args.warmup:]),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; no dataset named by the reference)",
        "config": config_dict(cfg, args.method, m, n_full, nnz, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- B200 arm ---------------------------------------------------------------------

def make_fn(aqr, method):
    family, variant, orientation = method.split("-")
    if family == "cgs":
        return lambda Z_, op_: aqr.cgs(Z_, op_, variant, orientation)
    fn = {"naive": aqr.mgs_naive, "ha": aqr.mgs_ha, "hp": aqr.mgs_hp}[variant]
    return lambda Z_, op_: fn(Z_, op_, orientation)


def run_b200(args, rank, world, local_rank):
    import ctypes

    import torch

    import paper_1703_10440_b200 as aqr
    from paper_1703_10440_b200 import _lib

    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local_rank % max(ndev, 1))
    if world > 1:
        return run_b200_distributed(args, rank, world, local_rank)
    L = _lib.lib()
    variant = args.method.split("-")[1]
    wl = device_workload(args.config)
    m, n = wl["m"], wl["n"]
    bytes_A, nnz = bytes_of_A(wl)
    op = aqr.DenseSpdOperator(wl["dense"]) if "dense" in wl else aqr.CsrSpdOperator(*wl["csr"])
    op_layout = "dense" if "dense" in wl else "csr"
    if "csr" in wl and banded_bytes(op, m) is not None:
        bytes_A, op_layout = banded_bytes(op, m)
    wl.pop("csr", None)
    wl.pop("dense", None)
    Zd = wl["Z"]
    fn = make_fn(aqr, args.method)
    stream = torch.cuda.current_stream()
    # kernel timer inside the timed region when launches are long (configs 3-5:
    # one event pair per ms-scale launch); config 2's 100 us launches get a
    # separate timed pass (the events would split the PDL-chained launches)
    timer_inside = args.config != 2

    res = None
    for _ in range(args.warmup):  # as in the timed loop, the previous result stays alive
        res = fn(Zd, op)  # during the next call
    torch.cuda.synchronize()

    # ---- device-resident timed region (value) ----
    launches0 = L.aqr_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if timer_inside:
        L.aqr_trailing_timer_enable(1)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            res = fn(Zd, op)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = int(L.aqr_launch_count() - launches0)
    ms_per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)
    del res

    # ---- dominant kernel: fused trailing pass, CUDA events on its stream ----
    if not timer_inside:
        L.aqr_trailing_timer_enable(1)
        for _ in range(args.steps):
            fn(Zd, op)
        torch.cuda.synchronize()
    L.aqr_trailing_timer_enable(0)
    nl, kms, kbytes = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.aqr_trailing_timer_read(ctypes.byref(nl), ctypes.byref(kms), ctypes.byref(kbytes))
    peak, peak_kind = measured_peaks()
    achieved = (kbytes.value / nl.value) / (kms.value / nl.value / 1e3) / 1e9 if nl.value else None
    share = (kms.value / args.steps) / ms_per_step if nl.value else None
    traffic, traffic_src = committed_traffic(args, kbytes.value / nl.value if nl.value else None)
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak if achieved else None, "traffic": traffic,
        "traffic_unit": "GB per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
        "traffic_source": traffic_src,
        "kernel": "trailing_w_kernel", "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
        "timed": "inside the timed region" if timer_inside else "separate pass of K steps",
        "launches_per_step": nl.value / args.steps if nl.value else 0,
        "kernel_ms_per_step": kms.value / args.steps, "kernel_share_of_step": share,
        "algorithmic_bytes_per_launch": kbytes.value / nl.value if nl.value else None,
    }
    sb = step_bytes(variant, m, n, bytes_A)
    step_gbs = sb / (ms_per_step / 1e3) / 1e9
    roofline["step"] = {"achieved": step_gbs, "frac": step_gbs / peak, "algorithmic_bytes": sb,
                        "operator_layout": op_layout, "operator_bytes_per_apply": bytes_A}
    # what SURVEY 8d's eager one-pass schedule would have to move in the same time
    eager = survey_bytes(variant, m, n, bytes_A)
    roofline["step"]["survey_8d_bytes"] = eager
    roofline["step"]["survey_8d_equivalent_gbs"] = eager / (ms_per_step / 1e3) / 1e9

    # ---- end to end: numpy Z in, numpy Q / R out, through the public API ----
    e2e = None
    Zh = None if args.no_e2e else np.asfortranarray(Zd.t().cpu().numpy().T)  # pageable, column-major
    del Zd
    wl.pop("Z", None)
    torch.cuda.empty_cache()  # the device-resident copy of Z and cached blocks go back
    if Zh is not None:
        e2e = measure_e2e(args, aqr, op, Zh, fn, m, n)
        del Zh

    # ---- CPU baseline (rank 0, N = 1): the oracle on one core ----
    cpu = None
    if not args.no_cpu_baseline:
        del op
        torch.cuda.empty_cache()
        cpu = cpu_baseline(args)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; no dataset named by the reference)",
        "config": config_dict(args.config, args.method, m, n, nnz, world),
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "hbm_gbs_step": step_gbs, "step_algorithmic_bytes": sb,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def committed_traffic(args, alg_bytes_per_launch):
    """DRAM traffic per launch of the trailing kernel from the committed ncu
    --set full capture (profiles/r*/trailing_traffic*.json, tools/ncu_summary.py):
    measured DRAM bytes / algorithmic bytes of the captured launches, applied
    to this run's mean algorithmic bytes per launch."""
    import glob

    if not alg_bytes_per_launch:
        return None, None
    for tpath in sorted(glob.glob(os.path.join(REPO, "profiles", "r*", "trailing_traffic*.json")))[::-1]:
        with open(tpath) as f:
            tt = json.load(f)
        if (tt.get("method") == args.method and tt.get("config", 2) == args.config
                and tt.get("traffic_over_algorithmic")):
            return tt["traffic_over_algorithmic"] * alg_bytes_per_launch / 1e9, os.path.relpath(tpath, REPO)
    return None, None


def measure_e2e(args, aqr, op, Zh, fn, m, n):
    """Wall clock of the public call with a pageable numpy Z (F-ordered) in and
    numpy Q, R out: staging into page-locked memory, H2D, the factorization and
    the D2H of Q (streamed as columns finish) are all inside."""
    import torch

    assert Zh.flags.f_contiguous and not Zh.flags.c_contiguous
    steps = min(args.steps, 3) if args.config in (4, 5) else args.steps
    # warm: the page-locked staging and result blocks (68 GB at config 5)
    # enter torch's host cache; the second call is still ~25 % slower than
    # the steady state on config 5 (tools/e2e_repeat.py), so two warm calls
    for _ in range(2):
        r = fn(Zh, op)
        assert isinstance(r.Q, np.ndarray) and r.Q.shape == (m, n)
        del r
    times = []
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(Zh, op)
        times.append(time.perf_counter() - t0)
        del r
    return {"value": n * len(times) / sum(times), "unit": UNIT, "steps": len(times),
            "ms_per_step": 1e3 * statistics.mean(times),
            "h2d_bytes_per_step": 8 * m * n, "d2h_bytes_per_step": 8 * m * n + 8 * n * n,
            "form": "numpy (pageable, F-ordered) Z in, numpy Q and R out, wall clock around the call "
                    "(after two warm calls)"}


def cpu_baseline(args):
    cfg = args.config
    spec, Zh, n_full = host_oracle_inputs(cfg, CPU_COLS[cfg])
    m = Zh.shape[0]
    secs, est = oracle_truncated_seconds(spec, Zh, args.method, n_full)
    k = Zh.shape[1]
    if k < n_full:
        sample = (f"one {args.method} factorization by the C oracle on 1 of {os.cpu_count()} host cores "
                  f"of the same config truncated to its first {k} of {n_full} columns ({secs:.1f} s), "
                  f"phases extrapolated to n={n_full} (apply/normalize x n/n', projections x "
                  f"n(n-1)/(n'(n'-1))): {est:.0f} s -- extrapolated")
    else:
        sample = (f"one full {args.method} factorization of the same config (m={m}, n={n_full}) by the "
                  f"C oracle on 1 of {os.cpu_count()} host cores, {secs:.2f} s")
    return {"value": n_full / est, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample,
            "measured_s": secs, "full_width_s": est}


def run_b200_distributed(args, rank, world, local_rank):
    """N > 1: config 5 HP, grid planes split across ranks, peer-memory path."""
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_1703_10440_b200 as aqr  # noqa: F401
    from paper_1703_10440_b200 import _lib
    from paper_1703_10440_b200 import distributed as DD

    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world:
        # the peer-memory kernels of different ranks wait on each other's
        # flags: ranks sharing a GPU are not guaranteed to run concurrently
        # (tests/test_gpu_multirank.py emulates N ranks on one device instead)
        raise SystemExit(f"{world} ranks need {world} GPUs, this node has {torch.cuda.device_count()}")
    # the step loop has no collective call (peer-memory flags); the process
    # group only bootstraps (IPC handles, halo plan) and takes the max over
    # ranks, so gloo is enough
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = _lib.lib()
    wl = device_workload(5, rank, world)
    m, n = wl["m"], wl["n"]
    n_side = 256
    part = [(n_side * n_side * (n_side * r // world), n_side * n_side * (n_side * (r + 1) // world))
            for r in range(world)]
    ip, ix, dv = wl.pop("csr")
    nnz_loc = int(ip[-1])
    op = DD.DistCsrSpdOperator(ip.cpu().numpy(), ix.to(torch.int64).cpu().numpy(), dv.cpu().numpy(), part, rank)
    del ip, ix, dv
    Zd = wl.pop("Z")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        DD.dist_factorize(Zd, op, args.method)
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = L.aqr_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    L.aqr_trailing_timer_enable(1)
    with ClockSampler(local_rank % max(torch.cuda.device_count(), 1)) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            DD.dist_factorize(Zd, op, args.method)
        ev1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    L.aqr_trailing_timer_enable(0)
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    launches = int(L.aqr_launch_count() - launches0)
    ms_per_step = ms / args.steps
    value = n * args.steps / (ms / 1e3)
    nl, kms, kbytes = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.aqr_trailing_timer_read(ctypes.byref(nl), ctypes.byref(kms), ctypes.byref(kbytes))
    peak, peak_kind = measured_peaks()
    ach = (kbytes.value / nl.value) / (kms.value / nl.value / 1e3) / 1e9 if nl.value else 0.0
    per_rank = torch.tensor([ach], dtype=torch.float64)
    gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, per_rank)
    bytes_A = 12 * 449_455_096 + 4 * (m + 1)
    sb = step_bytes("hp", m, n, bytes_A)  # the whole job: the ranks' row blocks of the same schedule
    step_gbs = sb / (ms_per_step / 1e3) / 1e9
    e2e = None
    if not args.no_e2e:
        # every rank: pinned host row block in, host Q rows + R out, through the driver API
        Zh = torch.empty((n, Zd.shape[0]), dtype=torch.float64).pin_memory().t()
        Zh.copy_(Zd)
        Qh = torch.empty((n, Zd.shape[0]), dtype=torch.float64).pin_memory().t()
        steps = min(args.steps, 3)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            res = DD.dist_factorize(Zh.to("cuda", non_blocking=True), op, args.method)
            Qh.copy_(res.Q, non_blocking=True)
            Rh = res.R.cpu()
            del res
        torch.cuda.synchronize()
        et = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": n * steps / float(et.item()), "unit": UNIT, "steps": steps,
               "h2d_bytes_per_step": 8 * m * n, "d2h_bytes_per_step": 8 * m * n + 8 * n * n * world,
               "form": "pinned host row block per rank in, host Q rows and R out (wall clock, max over ranks)"}
        del Rh
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; no dataset named by the reference)",
            "config": config_dict(5, args.method, m, n, 449_455_096, world),
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "hbm_gbs_step": step_gbs, "step_algorithmic_bytes": sb,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": None, "kernel": "p2p_trailing_kernel (rank 0)",
                         "per_rank_achieved": [float(g.item()) for g in gathered],
                         "peak_source": f"{peak_kind} hbm_gbs (one GPU's peak; per rank)",
                         "step": {"achieved_aggregate": step_gbs, "frac_of_N_peaks": step_gbs / (peak * world)}},
            "cpu_baseline": None, "e2e": e2e, "clocks": clocks.summary(),
            "local_nnz_rank0": nnz_loc,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
