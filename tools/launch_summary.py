"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): share of device time per
kernel.  python tools/launch_summary.py launches.csv "header comment" > summary.txt"""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki]
    depth = 0
    for j, ch in enumerate(name):  # cut at the parameter list (the first '(' outside <...>)
        depth += ch == "<"
        depth -= ch == ">"
        if ch == "(" and depth == 0 and j > 0 and name[j - 1] not in ":<":
            name = name[:j]
            break
    v = float(r[vi].replace(",", ""))
    tot[name] += v / 1e3  # ns -> us
    cnt[name] += 1
T = sum(tot.values())
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print("# cold-cache serialised per-launch times; the SHARE of the step is what carries over to the bench")
print(f"# total {T:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{100 * v / T:6.2f}% {v:11.1f} us {cnt[k]:5d} launches {v / cnt[k]:10.1f} us/launch  {k[:90]}")
