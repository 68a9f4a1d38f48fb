"""Experiment: does a degree-sorted vertex relabeling (hubs get the smallest ids, so their labels
share cache lines) speed up the traversals?  Host relabel of the device-generated RMAT graph,
re-upload, same sources mapped.  python tools/relabel_probe.py [scale]"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ctx = irgl.Context()
g = ctx.generate_rmat(scale)
rp, col, w = g.download()
deg = np.diff(rp)
srcs = bench.pick_sources(g.n, lambda x: int(deg[x]), count=8)
t0 = time.time()
order = np.argsort(-deg, kind="stable")            # new id i <- old vertex order[i]
newid = np.empty(g.n, dtype=np.int64); newid[order] = np.arange(g.n)
src_old = np.repeat(np.arange(g.n, dtype=np.int64), deg)
u2, v2 = newid[src_old], newid[col]
key = u2 * g.n + v2
perm = np.argsort(key, kind="stable")
col2 = v2[perm].astype(np.int32); w2 = w[perm]
rp2 = np.zeros(g.n + 1, dtype=np.int64); rp2[1:] = np.cumsum(deg[order])
print(f"relabel {time.time() - t0:.1f}s", flush=True)
g2 = ctx.graph_from_csr(rp2, col2, w2)
p = ctx.pipe(g.n)
def run(gr, ss, op, reps=2):
    t = []
    for _ in range(reps):
        for s in ss:
            p.init_scalars([s]); st = ctx.iterate(op, gr, p); t.append(st.kernel_ms)
    return np.mean(t)
for op, name in ((irgl.BFS, "BFS"), (irgl.SSSP, "SSSP")):
    a = run(g, srcs, op); b = run(g2, [int(newid[s]) for s in srcs], op)
    print(f"RMAT-{scale} {name}: scrambled {a:.3f} ms, degree-sorted {b:.3f} ms ({a / b:.2f}x)", flush=True)
# parity of the relabeled run, mapped back
p.init_scalars([int(newid[srcs[0]])]); ctx.iterate(irgl.SSSP, g2, p)
d2 = ctx.read_result(irgl.SSSP, g2)
p.init_scalars([srcs[0]]); ctx.iterate(irgl.SSSP, g, p)
d1 = ctx.read_result(irgl.SSSP, g)
print("same distances after mapping back:", bool(np.array_equal(d1, d2[newid])))
