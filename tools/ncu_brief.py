"""Brief per-launch summary of an ncu --set full report (read here, no GPU):
    python tools/ncu_brief.py report.ncu-rep"""
import csv, io, subprocess, sys

WANT = [
    ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rd"), ("dram__bytes_write.sum", "wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__t_sector_hit_rate.pct", "L2hit%"), ("l1tex__t_sector_hit_rate.pct", "L1hit%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "stall_lsb%"),
    ("smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct", "stall_lg%"),
    ("smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct", "stall_math%"),
    ("smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct", "stall_mio%"),
    ("smsp__warp_issue_stalled_barrier_per_warp_active.pct", "stall_bar%"),
    ("smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct", "stall_ssb%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:60]
    parts = []
    for key, short in WANT:
        if key in hdr:
            v = r[hdr.index(key)]
            u = units[hdr.index(key)]
            parts.append(f"{short}={v}{'' if u in ('%', '') else u}")
    print(name, " ".join(parts))
