"""Roofline evidence of one kernel from an ncu --set full report, in the JSON bench.py reads
(profiles/ncu_<op>_rmat<scale>.json: "traffic" = dram_bytes_per_launch):
python tools/ncu_json.py REPORT "note" > profiles/ncu_sssp_rmat22.json"""
import csv, io, json, os, re, subprocess, sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import kernel_source_hash  # noqa: E402  (stamp: bench.py refuses a stale capture)

rep, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"]).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
# the launch to summarise: --kernel-regex picks by name (default: the longest launch)
krx = os.environ.get("NCU_KERNEL_REGEX")
cands = [r for r in rows[2:] if len(r) == len(hdr) and (not krx or re.search(krx, r[hdr.index("Kernel Name")]))]
di = hdr.index("gpu__time_duration.sum")
vals = max(cands, key=lambda r: float(r[di].replace(",", "") or 0))


def v(k, scale=1.0):
    if k not in hdr:
        return None
    x = vals[hdr.index(k)].replace(",", "")
    try:
        x = float(x)
    except ValueError:
        return None
    u = units[hdr.index(k)]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1.0)
    return x * mult * scale


out = {
    "source_hash": kernel_source_hash(),
    "report": rep.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")], "note": note,
    "dram_bytes_read": v("dram__bytes_read.sum"), "dram_bytes_write": v("dram__bytes_write.sum"),
    "dram_throughput_pct": v("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "l2_hit_rate_pct": v("lts__t_sector_hit_rate.pct"), "l1_hit_rate_pct": v("l1tex__t_sector_hit_rate.pct"),
    "achieved_occupancy_pct": v("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": v("launch__registers_per_thread"), "grid_size": v("launch__grid_size"),
    "block_size": v("launch__block_size"),
    "sm_throughput_pct": v("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "l1tex_throughput_pct": v("l1tex__throughput.avg.pct_of_peak_sustained_active"),
    "l2_throughput_pct": v("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    "instructions": v("smsp__inst_executed.sum"),
    "l2_read_sectors_from_sm": v("lts__t_sectors_srcunit_tex_op_read.sum"),
    "l2_atomic_sectors": v("lts__t_sectors_op_atom.sum"),
    "l2_red_sectors": v("lts__t_sectors_op_red.sum"),
    "l1_global_load_sectors": v("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    "l1_global_load_requests": v("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    "duration_ms": v("gpu__time_duration.sum"),
}
if out["dram_bytes_read"] is not None and out["dram_bytes_write"] is not None:
    out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
if out["l1_global_load_sectors"] and out["l1_global_load_requests"]:
    out["sectors_per_request"] = out["l1_global_load_sectors"] / out["l1_global_load_requests"]
if out.get("dram_bytes_per_launch") and out["duration_ms"]:
    out["achieved_dram_GBps"] = out["dram_bytes_per_launch"] / (out["duration_ms"] * 1e-3) / 1e9
# atomic / reduction throughput (north_star: "atomic throughput"): every L2 / L1 counter of
# atomics (ATOM, with return) and reductions (RED, fire-and-forget) the capture holds
out["atomics"] = {k: v(k) for k in hdr if re.search(r"op_(atom|red)", k) and v(k) is not None}
for key, pat in (("l2_atomic_sectors", r"^lts__t_sectors.*op_atom\.sum$"),
                 ("l2_red_sectors", r"^lts__t_sectors.*op_red\.sum$")):
    if out[key] is None:
        hits = [v(k) for k in hdr if re.search(pat, k) and v(k) is not None]
        out[key] = max(hits) if hits else None
if out["l2_atomic_sectors"] is not None and out["duration_ms"]:
    out["l2_atomic_sectors_per_s"] = out["l2_atomic_sectors"] / (out["duration_ms"] * 1e-3)
if out["l2_red_sectors"] is not None and out["duration_ms"]:
    out["l2_red_sectors_per_s"] = out["l2_red_sectors"] / (out["duration_ms"] * 1e-3)
print(json.dumps(out, indent=1))
