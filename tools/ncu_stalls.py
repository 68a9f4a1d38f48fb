"""Stall reasons per CUDA source line from an ncu report (source page, cuda view):
python tools/ncu_stalls.py report.ncu-rep [N]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
fname = ""
lines = []
tot = collections.Counter()
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit() and r[2] == "-":
        d = dict(zip(hdr, r))
        d["Source"] = r[1]
        lines.append((fname, d))
cols = [c for c in (hdr or []) if c.startswith("stall_") and "Not Issued" not in c]
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
for f, d in lines:
    for c in cols:
        tot[c] += num(d[c])
T = sum(tot.values())
print("kernel-wide stall mix: " + ", ".join(f"{c[6:]} {100*v/T:.1f}%" for c, v in tot.most_common(8)))
samp = "Warp Stall Sampling (All Samples)"
lines.sort(key=lambda fd: -num(fd[1].get(samp, "0")))
S = sum(num(d.get(samp, "0")) for _, d in lines)
for f, d in lines[:N]:
    mix = sorted(((num(d[c]), c[6:]) for c in cols), reverse=True)[:3]
    print(f"{100*num(d[samp])/S:5.1f}% {f}:{d['Line No']:<5} " + " ".join(f"{n}={int(v)}" for v, n in mix) +
          f"  | {d['Source'].strip()[:70]}")
