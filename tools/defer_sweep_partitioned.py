"""SSSP deferral budget K on a partitioned graph (P logical partitions, distributed persistent
kernel), RMAT scale S, degree-ordered ids: ms per traversal and edges scanned per K.
python tools/defer_sweep_partitioned.py [scale] [P]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = irgl.Context(logical_partitions=P)
g = ctx.generate_rmat(scale)
rp, _, _ = g.download()
srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=4)
g.relabel()
p = ctx.pipe(max(g.info.local_n, 1))
for K in (0, 256, 512, 1024, 2048, 4096, 8192):
    irgl.sssp(ctx, g, srcs[0], pipe=p, defer=K)
    t, e, r = [], [], []
    for s in srcs:
        t0 = time.perf_counter()
        _, st = irgl.sssp(ctx, g, s, pipe=p, defer=K)
        t.append(time.perf_counter() - t0)
        e.append(st.edges)
        r.append(st.rounds)
    print(f"RMAT-{scale} P={P} defer={K}: {1e3 * np.mean(t):.2f} ms/traversal (incl. readback), "
          f"rounds {np.mean(r):.1f}, edges {np.mean(e) / 1e6:.1f} M", flush=True)
ctx.close()
