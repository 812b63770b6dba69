"""Summarize round-2 ncu evidence into profiles/<round>/ (no GPU needed).

    python tools/r02_summary.py r02 gpurun_out/r02i_launches.csv \
        gpurun_out/r02i_c5_t.ncu-rep gpurun_out/r02i_c5_x.ncu-rep gpurun_out/r02i_dmma.ncu-rep

* launch list (ncu --metrics gpu__time_duration.sum --clock-control none of
  `python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e`, config 5
  mgs-hp-row): the last factorization's launches grouped by kernel -- count,
  serialized time, share;
* full captures: per launch duration, DRAM bytes, throughput, occupancy;
  for the windowed trailing passes of the narrow config-5 run (n' = 64,
  steps 20 and 21: a write-back pass and a plain one) the DRAM traffic over
  the algorithmic bytes of trailing_bytes() -> trailing_traffic_cfg5_hp.json
  (read by bench.py for roofline.traffic).
"""
import collections, csv, io, json, os, subprocess, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r["Metric Name"] == "gpu__time_duration.sum":
            v = float(r["Metric Value"])
            unit = r["Metric Unit"]
            us = v / 1e3 if unit in ("nsecond", "ns") else v * 1e3 if unit in ("msecond", "ms") else v
            rows.append((r["Kernel Name"], us))
    return rows


def short(name):
    for key in ("trailing_w_kernel", "trailing_kernel", "col_lazy_norm_kernel", "x_catchup_kernel",
                "csr_spmm2_kernel", "finalize_r_kernel", "status_init_kernel", "dense_dmma_kernel",
                "band_spmm_tile_kernel", "band_spmm_kernel", "band_step_kernel", "band_collect_kernel",
                "band_mask_kernel", "band_vals_kernel"):
        if key in name:
            return key
    return name.split("(")[0][-50:]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: r[i] for i, h in enumerate(hdr)}
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


def gb(d, key):
    v, u = float(d[key]), d["_units"][key]
    return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(u, 1.0)


def ms(d):
    v, u = float(d["gpu__time_duration.sum"]), d["_units"]["gpu__time_duration.sum"]
    return v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1.0)


def main():
    rnd, lst = sys.argv[1], sys.argv[2]
    reps = sys.argv[3:]
    outdir = os.path.join(REPO, "profiles", rnd)
    L = [(short(n), us) for n, us in launches(lst)]
    ours = [x for x in L if not x[0].startswith(("void <unnamed>", "void at::", "elementwise", "void (anonymous"))]
    # the last factorization: from the last status_init_kernel on
    last = max(i for i, (n, _) in enumerate(L) if n == "status_init_kernel")
    fact = L[last:]
    tot = sum(us for _, us in fact)
    agg = collections.OrderedDict()
    for n, us in fact:
        c, t = agg.get(n, (0, 0.0))
        agg[n] = (c + 1, t + us)
    md = [f"# ncu summary, round {rnd[1:]} (config 5, mgs-hp-row)", "",
          f"Launch list: `{os.path.basename(lst)}` (ncu --metrics gpu__time_duration.sum --clock-control none, "
          "cold-cache serialized per launch) of `python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e`; "
          f"{len(L)} launches in total, the last factorization = {len(fact)} launches, {tot / 1e3:.1f} ms serialized.", "",
          "| kernel | launches | ms | share |", "|---|---|---|---|"]
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{n}` | {c} | {t / 1e3:.1f} | {t / tot:.3f} |")
    traffic = None
    for rep in reps:
        md += ["", f"Full capture `{os.path.basename(rep)}` (ncu --set full --clock-control none):", "",
               "| kernel | ms | DRAM read GB | DRAM write GB | TB/s | occupancy % | regs |", "|---|---|---|---|---|---|---|"]
        rows = raw(rep)
        for d in rows:
            t = ms(d)
            rd, wr = gb(d, "dram__bytes_read.sum"), gb(d, "dram__bytes_write.sum")
            md.append(f"| `{short(d['Kernel Name'])}` | {t:.3f} | {rd:.2f} | {wr:.2f} | {(rd + wr) / t:.2f} | "
                      f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                      f"{d['launch__registers_per_thread']} |")
        if "c5_t" in rep:
            m, n = 256 ** 3, 64
            tw = [d for d in rows if "trailing_w" in d["Kernel Name"]]
            # captured passes: steps 20 (write-back, window 4) and 21 (window 1) of n' = 64
            alg = []
            for step, win, store in ((20, 4, True), (21, 1, False)):
                t = n - 1 - step
                cols = 8 * t + (8 * t if store else 8)
                vec = 8 + 8 * win + 16 + 8  # psrc, q window, zsrc read + q store, p store (HP)
                alg.append(m * (cols + vec) / 1e9)
            meas = [gb(d, "dram__bytes_read.sum") + gb(d, "dram__bytes_write.sum") for d in tw[:2]]
            ratio = sum(meas) / sum(alg)
            traffic = {"method": "mgs-hp-row", "config": 5, "kernel": "trailing_w_kernel<8, 2, false>",
                       "captured": "narrow config 5 (m = 256^3, n' = 64), steps 20 (write-back) and 21",
                       "algorithmic_gb": alg, "dram_gb": meas, "traffic_over_algorithmic": ratio}
            md.append("")
            md.append(f"Trailing passes: DRAM traffic / algorithmic bytes = {ratio:.3f} "
                      f"(measured {meas[0]:.2f} / {meas[1]:.2f} GB vs {alg[0]:.2f} / {alg[1]:.2f} GB).")
    with open(os.path.join(outdir, "ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    if traffic:
        with open(os.path.join(outdir, "trailing_traffic_cfg5_hp.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
