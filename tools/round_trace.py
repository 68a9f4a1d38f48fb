"""Per-round trace of one outlined traversal: IRGL_ROUND_TRACE=1 python tools/round_trace.py
[scale] [op] [defer]   (op: bfs|bfs-do|sssp; RELABEL=1: degree-ordered ids).  The runtime prints one line per round to stderr."""
import ctypes as C, os, sys
os.environ.setdefault("IRGL_ROUND_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
opname = sys.argv[2] if len(sys.argv) > 2 else "sssp"
op = irgl.SSSP if opname == "sssp" else irgl.BFS
defer = int(sys.argv[3]) if len(sys.argv) > 3 else -1
ctx = irgl.Context()
g = ctx.generate_rmat(scale)
rp = np.zeros(g.n + 1, dtype=np.int64)
ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=2)
if os.environ.get("RELABEL") == "1":  # degree-ordered ids (API ids unchanged)
    g.relabel()
p = ctx.pipe(g.n)
kw = dict(defer=defer, delta=0) if op == irgl.SSSP else ({"direction": 1} if opname == "bfs-do" else {})
for s in srcs:
    p.init_scalars([s])
    st = ctx.iterate(op, g, p, outline=1, **kw)
    print(f"# src={s} rounds={st.rounds} edges={st.edges} kernel_ms={st.kernel_ms:.3f}", file=sys.stderr, flush=True)
ctx.close()
