import os, sys, time
sys.path.insert(0, "/root/repo")
import paper_1607_05707_b200 as irgl
scale = int(sys.argv[1])
ctx = irgl.Context()
t0 = time.time()
try:
    g = ctx.generate_rmat(scale)
    print("generated", scale, g.n, g.m, f"{time.time()-t0:.1f}s", flush=True)
    p = ctx.pipe(g.n)
    p.init_scalars([0]); st = ctx.iterate(irgl.BFS, g, p)
    print("bfs", st.rounds, st.edges, st.kernel_ms, flush=True)
except Exception as e:
    print("FAILED", type(e).__name__, e, flush=True)
