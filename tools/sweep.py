"""Threshold sweep: python tools/sweep.py [scale]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1607_05707_b200 as irgl
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
def run(ctx, g, srcs, op, **kw):
    p = ctx.pipe(g.n); t = 0
    for s in srcs:
        p.init_scalars([s]); st = ctx.iterate(op, g, p, **kw); t += st.kernel_ms
    return t / len(srcs)
base = None
CFG = [(w, c, k) for w in (32, 64, 128, 256) for c, k in ((512, 1024), (1024, 2048), (1024, 1024))]
for warp_t, cta_t, chunk in CFG:
    if warp_t > cta_t: continue
    if True:
        ctx = irgl.Context(warp_threshold=warp_t, cta_threshold=cta_t, chunk_edges=chunk)
        g = ctx.generate_rmat(scale)
        if base is None:
            rp = np.zeros(g.n + 1, dtype=np.int64)
            ctx._lib.irgl_graph_download(g.handle, rp.ctypes.data_as(C.POINTER(C.c_int64)), None, None)
            srcs = bench.pick_sources(g.n, lambda x: int(rp[x + 1] - rp[x]), count=4)
            base = 1
        b = run(ctx, g, srcs, irgl.BFS); s = run(ctx, g, srcs, irgl.SSSP, delta=0)
        print(f"warp_t={warp_t} cta_t={cta_t} chunk={chunk}: BFS {b:.3f} ms  SSSP {s:.3f} ms", flush=True)
        ctx.close()
