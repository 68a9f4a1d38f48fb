"""Summarise an ncu --set full report into profiles/*.json (run here, no GPU needed).
usage: python tools/ncu_summary.py report.ncu-rep out.json [note]"""
import csv, io, json, subprocess, sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_rate_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_rate_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "smsp__inst_executed.sum": "instructions",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors_from_sm",
    "lts__t_sectors_srcunit_tex_op_atom.sum": "l2_atomic_sectors",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "l1_global_load_sectors",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "l1_global_load_requests",
}

def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"report": rep.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")][:120], "note": note}
    for k, name in KEYS.items():
        if k in hdr:
            v = vals[hdr.index(k)].replace(",", "")
            try:
                d[name] = float(v)
            except ValueError:
                d[name] = v
    if "dram_bytes_read" in d:
        # ncu reports bytes in the unit row (e.g. Gbyte / Mbyte): normalise to bytes
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for k in ("dram_bytes_read", "dram_bytes_write"):
            u = units[hdr.index([kk for kk, nn in KEYS.items() if nn == k][0])]
            d[k] = d[k] * scale.get(u, 1)
        d["dram_bytes_per_launch"] = d["dram_bytes_read"] + d["dram_bytes_write"]
    if "duration_ns" in d:
        u = units[hdr.index("gpu__time_duration.sum")]
        d["duration_ms"] = d["duration_ns"] * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1e-6)
        del d["duration_ns"]
    if d.get("l1_global_load_requests"):
        d["sectors_per_request"] = d["l1_global_load_sectors"] / d["l1_global_load_requests"]
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))

main()
