"""Top SASS instructions by warp-stall samples from an ncu report (run here, no GPU):
python tools/sass_hot.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
iS = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iS] or 0) for r in data)
agg = {s: sum(float(r[hdr.index(s)] or 0) for r in data) for s in stalls}
print(f"total samples {tot:.0f}")
for s, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
    print(f"  {s:28s} {100*v/tot:5.1f}%")
print()
data.sort(key=lambda r: -float(r[iS] or 0))
for r in data[:N]:
    top = sorted(((float(r[hdr.index(s)] or 0), s) for s in stalls), reverse=True)[:2]
    print(f"{r[0]:>6s} {100*float(r[iS] or 0)/tot:5.1f}%  {r[1][:60]:60s} " +
          " ".join(f"{s[6:]}={100*v/tot:.1f}" for v, s in top if v))
