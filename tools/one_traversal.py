"""One warm traversal for profilers: python tools/one_traversal.py OP SCALE RELABEL
(OP bfs|bfs-do|sssp; the first traversal is a warm-up, the second is the one to capture: use
ncu --launch-skip/-c or -k regex:persistent with --launch-skip 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

op = irgl.SSSP if sys.argv[1] == "sssp" else irgl.BFS
kw = {"direction": 1} if sys.argv[1] == "bfs-do" else {}
scale = int(sys.argv[2])
ctx = irgl.Context()
g = ctx.generate_rmat(scale)
deg = np.diff(g.download()[0])
src = bench.pick_sources(g.n, lambda x: int(deg[x]), count=1)[0]
if int(sys.argv[3]):
    g.relabel()
p = ctx.pipe(g.n)
for _ in range(2):
    p.init_scalars([src])
    st = ctx.iterate(op, g, p, **kw)
print(f"rounds={st.rounds} edges={st.edges} kernel_ms={st.kernel_ms:.3f}", flush=True)
