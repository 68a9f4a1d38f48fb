"""Key counters of ncu reports (one kernel each): python tools/ncu_summary.py REPORT..."""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard_per_warp_active.ratio", "long-scoreboard stall / issued"),
]
for rep in sys.argv[1:]:
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"== {rep.split('/')[-1]}: {vals[hdr.index('Kernel Name')][:90]}")
    for k, name in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"   {name:34s} {vals[i]} {units[i]}")
