"""Dense-round threshold (irgl_config.dense_div: a round is dense when |in| >= n / dense_div):
python tools/dense_probe.py SCALE  (degree-ordered ids, 8 sources)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
DD = [int(x) for x in os.environ["DENSE"].split(",")] if os.environ.get("DENSE") else [16, 4, 8, 32, 64, -1]
for dd in DD:
    ctx = irgl.Context(dense_div=dd)
    g = ctx.generate_rmat(scale)
    deg = np.diff(g.download()[0])
    srcs = bench.pick_sources(g.n, lambda x: int(deg[x]), count=8)
    g.relabel()
    p = ctx.pipe(g.n)
    out = []
    for op, name in ((irgl.BFS, "BFS"), (irgl.SSSP, "SSSP")):
        t = []
        for rep in range(2):
            for s in srcs:
                p.init_scalars([s])
                st = ctx.iterate(op, g, p)
                if rep:
                    t.append(st.kernel_ms)
        out.append(f"{name} {np.mean(t):.3f} ms")
    print(f"RMAT-{scale} dense_div={dd}: " + ", ".join(out), flush=True)
    p.close(); g.close(); ctx.close()
