"""Scheduler thresholds on the current kernels: python tools/sched_probe.py SCALE
warp_t (fine-grained vs descriptor split) x chunk_edges, degree-ordered ids, 8 sources."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
combos = [(128, 512, 256), (64, 512, 256), (96, 512, 256), (192, 512, 256), (256, 512, 256),
          (128, 256, 256), (128, 1024, 256)]
if os.environ.get("SCHED"):  # SCHED="warp_t:chunk_edges:cta_t,..."
    combos = [tuple(int(x) for x in c.split(":")) for c in os.environ["SCHED"].split(",")]
for wt, ce, cta in combos:
    ctx = irgl.Context(warp_threshold=wt, chunk_edges=ce, cta_threshold=max(cta, wt))
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
    print(f"RMAT-{scale} warp_t={wt} chunk={ce} cta_t={max(cta, wt)}: " + ", ".join(out), flush=True)
    p.close(); g.close(); ctx.close()
