"""Quick perf probe: device-generated RMAT, BFS/SSSP from a few sources, both orchestration
modes.  Prints per-run device ms and GTEPS (Graph500: undirected edges of the traversed
component / time)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
ctx = irgl.Context()
t = time.time()
g = ctx.generate_rmat(scale)
print(f"RMAT-{scale}: n={g.n} m={g.m} maxdeg={g.info.max_degree} gen {time.time()-t:.2f}s", flush=True)
rp, _, _ = (None, None, None)
p = ctx.pipe(g.n)
srcs = [1, 2, 3, 5, 8]
for op, name in ((irgl.BFS, "BFS"), (irgl.SSSP, "SSSP")):
    for outline in (0, 1):
        res = []
        for s in srcs:
            p.init_scalars([s])
            st = ctx.iterate(op, g, p, outline=outline)
            if st.edges < 1000:
                continue
            res.append((st.device_ms, st.edges, st.rounds, st.popped))
        for ms, e, r, pop in res:
            print(f"{name} outline={outline} ms={ms:8.3f} edges={e} rounds={r} popped={pop} "
                  f"GTEPS={e/2/ms/1e6:7.2f} directed-G/s={e/ms/1e6:7.2f}", flush=True)
