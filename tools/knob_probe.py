"""A/B of runtime tuning knobs (environment variables read at each launch) on one graph:
python tools/knob_probe.py SCALE OP "VAR=a,b,c" ["VAR2=x,y"]   (degree-ordered ids)
Prints mean kernel ms over 8 sources (2nd repetition) for every combination, and checks that
every variant returns the same labels as the first."""
import itertools, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale, opname = int(sys.argv[1]), sys.argv[2]
knobs = [(a.split("=")[0], a.split("=")[1].split(",")) for a in sys.argv[3:]]
op = irgl.SSSP if opname == "sssp" else irgl.BFS
kw = {"direction": 1} if opname == "bfs-do" else {}
ctx = irgl.Context()
g = ctx.generate_rmat(scale)
deg = np.diff(g.download()[0])
srcs = bench.pick_sources(g.n, lambda x: int(deg[x]), count=8)
if os.environ.get("RELABEL", "1") == "1":
    g.relabel()
p = ctx.pipe(g.n)
ref = None
for combo in itertools.product(*[v for _, v in knobs]):
    for (k, _), val in zip(knobs, combo):
        os.environ[k] = val
    t, res = [], []
    for rep in range(2):
        for s in srcs:
            p.init_scalars([s])
            st = ctx.iterate(op, g, p, **kw)
            if rep:
                t.append(st.kernel_ms)
                if s == srcs[0]:
                    res = ctx.read_result(op, g)
    same = "" if ref is None else (" same" if np.array_equal(ref, res) else " MISMATCH")
    ref = res if ref is None else ref
    print(f"RMAT-{scale} {opname} " + " ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo))
          + f": {np.mean(t):.4f} ms (min {np.min(t):.4f}){same}", flush=True)
