"""One traversal for ncu: python tools/profile_one.py [op] [scale] [outline] [reps] [delta]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import bench
import paper_1607_05707_b200 as irgl

op = {"sssp": irgl.SSSP, "bfs": irgl.BFS, "cc_lp": irgl.CC_LP}[sys.argv[1] if len(sys.argv) > 1 else "sssp"]
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 22
outline = int(sys.argv[3]) if len(sys.argv) > 3 else 1
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
delta = int(sys.argv[5]) if len(sys.argv) > 5 else -1
ctx = irgl.Context(outline=outline)
g = ctx.generate_rmat(scale)
rp = np.zeros(g.n + 1, dtype=np.int64)
ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
src = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=1)[0]
p = ctx.pipe(g.n)
for _ in range(reps):
    p.init_scalars([src])
    st = ctx.iterate(op, g, p, delta=delta)
print("src", src, st)
