"""Quick A/B timing of the three headline operators on RMAT-SCALE (original and degree-ordered
ids): BFS / SSSP mean kernel ms over 8 sources, PR ms per sweep.  Pick the library with IRGL_LIB
to compare builds.  python tools/ops_probe.py [scale]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
lib = os.path.basename(os.environ.get("IRGL_LIB", "default"))
ctx = irgl.Context()
g = ctx.generate_rmat(scale)
deg = np.diff(g.download()[0])
srcs = bench.pick_sources(g.n, lambda x: int(deg[x]), count=8)
for rl in (0, 1):
    if rl:
        g.relabel()
    p = ctx.pipe(g.n)
    out = []
    for op, name, kw in ((irgl.BFS, "BFS", {}), (irgl.BFS, "BFS-DO", {"direction": 1}),
                         (irgl.SSSP, "SSSP", {})):
        t = []
        for rep in range(2):
            for s in srcs:
                p.init_scalars([s])
                st = ctx.iterate(op, g, p, **kw)
                if rep:
                    t.append(st.kernel_ms)
        out.append(f"{name} {np.mean(t):.3f} ms")
    irgl.pagerank(ctx, g)
    _, st = irgl.pagerank(ctx, g)
    out.append(f"PR {st.device_ms / st.rounds:.3f} ms/sweep")
    print(f"{lib} RMAT-{scale} relabel={rl}: " + ", ".join(out), flush=True)
    p.close()
