"""DO-BFS with / without the visited bitmap: python tools/do_bitmap_probe.py SCALE"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
for rl in (0, 1):
    for bm in (-1, 0):
        ctx = irgl.Context(bfs_bitmap_min_n=bm)
        g = ctx.generate_rmat(scale)
        deg = np.diff(g.download()[0])
        srcs = bench.pick_sources(g.n, lambda x: int(deg[x]), count=8)
        if rl:
            g.relabel()
        p = ctx.pipe(g.n)
        t = {0: [], 1: []}
        for rep in range(2):
            for s in srcs:
                for dr in (0, 1):
                    p.init_scalars([s])
                    st = ctx.iterate(irgl.BFS, g, p, direction=dr)
                    if rep:
                        t[dr].append(st.kernel_ms)
        print(f"RMAT-{scale} relabel={rl} bitmap={'never' if bm < 0 else 'default'}: BFS {np.mean(t[0]):.3f} ms, "
              f"DO {np.mean(t[1]):.3f} ms", flush=True)
        p.close(); g.close(); ctx.close()
