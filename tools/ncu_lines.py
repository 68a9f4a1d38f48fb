"""Warp-stall samples per CUDA source line from an ncu report (cuda,sass correlation; run here):
python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                               "--metrics", "smsp__pcsamp_sample_count"]).decode()
agg = collections.Counter()
src = {}
fname = ""
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) == 5 and r[0].isdigit() and r[2] == "-":
        key = (fname, int(r[0]))
        src[key] = r[1]
        try:
            agg[key] += int(r[4])
        except ValueError:
            pass
tot = sum(agg.values())
print(f"total samples {tot}")
for (f, ln), v in agg.most_common(N):
    print(f"{100*v/tot:5.1f}% {f}:{ln:<5d} {src[(f, ln)].strip()[:100]}")
