"""Summarize the ncu captures of a bench run into profiles/<round>/.

    python tools/ncu_summary.py r01 gpurun_out/r01_launches.csv \
        gpurun_out/r01_trailing_early.ncu-rep gpurun_out/r01_trailing_mid.ncu-rep \
        gpurun_out/r01_spmv_full.ncu-rep

Inputs come from (see profiles/<round>/README.md):
  ncu --metrics gpu__time_duration.sum --clock-control none --csv ...   (launch list)
  ncu --set full --clock-control none --import-source on -k regex:... (full captures)
of `python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e`
(config 2, mgs-ha-row: launches 0-127 are the warm-up and the timed
factorization, 64 fused SpMV steps + 64 trailing passes each).

Writes profiles/<round>/ncu_summary.md and profiles/<round>/trailing_traffic.json
(DRAM bytes per launch vs the algorithmic bytes, read by bench.py).
"""

import collections
import csv
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M, N = 1024 * 1024, 64


HP = os.environ.get("NCU_METHOD", "mgs-ha-row") == "mgs-hp-row"


def trailing_alg_bytes(step):
    """Algorithmic bytes of the fused trailing pass at step i (config 2;
    HA, or HP with NCU_METHOD=mgs-hp-row: X carried and updated too), as
    the library's trailing_bytes() counts them."""
    t = N - 1 - step
    upd = step > 0
    per_col = 8 + (8 if upd else 0) + (16 if HP and upd else 0)
    vec = 8 + (8 if upd else 0) + (8 if HP and upd else 0) + 16 + (8 if HP else 0)
    return M * (t * per_col + vec)


def launch_list(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    data = rows[1:]
    n = len(data) // 3  # warm-up, timed, kernel-timer pass
    step = data[n:2 * n]
    agg = collections.OrderedDict()
    for r in step:
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", "")) / 1e3
    return agg


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {h: r[i] for i, h in enumerate(hdr)}
        d["__units__"] = dict(zip(hdr, units))
        recs.append(d)
    return recs


def mbytes(d, k):
    """A byte metric in MB whatever unit ncu chose for it (byte .. Gbyte)."""
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
    return f(d, k) * scale.get(d.get("__units__", {}).get(k, "Mbyte"), 1.0)


def f(d, k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


def main():
    rnd, launches, *reps = sys.argv[1:]
    outdir = os.path.join(REPO, "profiles", rnd)
    os.makedirs(outdir, exist_ok=True)
    agg = launch_list(launches)
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu summary — {rnd}", "",
             "Command: `python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e` "
             f"(config 2, {'mgs-hp-row' if HP else 'mgs-ha-row'}, m = 1,048,576, n = 64) on one B200, "
             "`--clock-control none`.", "",
             "## Launch list of one factorization (cold-cache, serialised: compare shares)", "",
             "| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, (cnt, us) in agg.items():
        lines.append(f"| `{k}` | {cnt} | {us:.1f} | {us / tot:.3f} |")
    lines += [f"| **all** | {sum(v[0] for v in agg.values())} | {tot:.1f} | 1.000 |", ""]
    ratios = []
    lines += ["## Full captures (`--set full`)", "",
              "| capture | kernel | launch | step | µs | DRAM read MB | DRAM write MB | "
              "algorithmic MB | traffic / algorithmic | DRAM % of peak | warps active % | regs |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    skip = {"r01_trailing_early": 64, "r01_trailing_mid": 96, "r01_spmv_full": 70}
    for rep in reps:
        base = os.path.basename(rep).replace(".ncu-rep", "")
        s0 = next((v for k, v in skip.items() if base.endswith(k.split("_", 1)[1])), 0)
        for j, d in enumerate(raw(rep)):
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
            us = f(d, "gpu__time_duration.sum")
            rd = mbytes(d, "dram__bytes_read.sum")
            wr = mbytes(d, "dram__bytes_write.sum")
            launch = s0 + j
            step = launch - 64 if "trailing" in name else launch - 64
            alg = trailing_alg_bytes(step) if "trailing" in name else float("nan")
            ratio = (rd + wr) * 1e6 / alg if alg == alg else float("nan")
            if ratio == ratio:
                ratios.append({"step": step, "dram_bytes": (rd + wr) * 1e6, "alg_bytes": alg,
                               "ratio": ratio, "us": us})
            lines.append(
                f"| {base} | `{name}` | {launch} | {step} | {us:.1f} | {rd:.1f} | {wr:.1f} | "
                f"{alg / 1e6:.1f} | {ratio:.3f} | "
                f"{f(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                f"{f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
                f"{f(d, 'launch__registers_per_thread'):.0f} |")
    mean_ratio = sum(r["ratio"] for r in ratios) / len(ratios) if ratios else None
    lines += ["", f"Mean DRAM traffic / algorithmic bytes of the captured trailing launches: "
              f"{mean_ratio:.3f}" if mean_ratio else ""]
    sfx = "_hp" if HP else ""
    with open(os.path.join(outdir, f"ncu_summary{sfx}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(outdir, f"trailing_traffic{sfx}.json"), "w") as fh:
        json.dump({"method": "mgs-hp-row" if HP else "mgs-ha-row", "config": "config2", "launches": ratios,
                   "traffic_over_algorithmic": mean_ratio}, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
